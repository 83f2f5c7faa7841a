# K3 4,096-item tiles: 512 threads x 8 items (default) vs 256 threads x 16 items
tag=${1:-u}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "route or cascade" > gpurun_out/${tag}_pytest.txt 2>&1
HS_COMPACT_T256=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -k "route or cascade or two_launch" > gpurun_out/${tag}_pytest_t256.txt 2>&1
for r in 1 2; do
  timeout 300 python tools/stage_cost.py --only full,steps_fixed > gpurun_out/${tag}_sc_t512_$r.txt 2>&1
  HS_COMPACT_T256=1 timeout 300 python tools/stage_cost.py --only full,steps_fixed > gpurun_out/${tag}_sc_t256_$r.txt 2>&1
done
