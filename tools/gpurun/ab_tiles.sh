tag=${1:-x}
timeout 600 python -m pytest tests/test_gpu_forward.py -q -k "cascade_step_equals" > gpurun_out/${tag}_placed_vr.txt 2>&1
for r in 1 2; do
  timeout 300 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_big_$r.txt 2>&1
  HS_COMPACT_SMALL_TILES=1 timeout 300 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_small_$r.txt 2>&1
done
