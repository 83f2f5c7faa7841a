# memcheck of the failing overlap test, then the GPU suite, split A/B bench
tag=${1:-x}
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_first_equals_serial" > gpurun_out/${tag}_memcheck_overlap.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.txt 2>&1
timeout 400 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_split.txt 2>&1
timeout 400 python bench.py --steps 100 --no-cpu-baseline --e2e-steps 0 --no-split > gpurun_out/${tag}_bench_nosplit.txt 2>&1
