set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python tools/calib_bench.py 2>&1 | tail -40
timeout 300 python tools/breakdown.py 2>&1 | tail -25
timeout 300 python bench.py --e2e-steps 0 2>/dev/null | tail -1
