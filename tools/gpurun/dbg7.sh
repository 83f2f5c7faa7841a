tag=${1:-x}
timeout 600 python -m pytest tests/test_gpu_forward.py -q -x -k "cascade_step_equals" > gpurun_out/${tag}_placed_vr.txt 2>&1
timeout 300 python bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${tag}_bal2.txt 2>&1
timeout 300 python bench.py --gpus 2 --share-gpu --placement placed --requests 20000 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_placed2_small.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 5 python bench.py --gpus 2 --share-gpu --placement placed --requests 40000 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-graph > gpurun_out/${tag}_placed2_memcheck.txt 2>&1
