# K3 tile size: 4,096 (default) vs 8,192 items, C2 and C5, + the GPU suite
tag=${1:-t}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.txt 2>&1
for r in 1 2; do
  timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_c2_4096_$r.txt 2>&1
  HS_COMPACT_TILES=8192 timeout 600 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_c2_8192_$r.txt 2>&1
  timeout 600 python bench.py --config c5 --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_c5_4096_$r.txt 2>&1
  HS_COMPACT_TILES=8192 timeout 600 python bench.py --config c5 --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_c5_8192_$r.txt 2>&1
done
