# K1a early first-row prefetch (before the PDL wait) A/B on one box + the GPU suite
tag=${1:-e}
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/${tag}_pytest_fused.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.txt 2>&1
for r in 1 2; do
  timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_early$r.txt 2>&1
  HS_LIBHS=build/exp/libhs_noearly.so timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_noearly$r.txt 2>&1
done
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.txt 2>&1
HS_LIBHS=build/exp/libhs_noearly.so timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_c2_noearly.txt 2>&1
