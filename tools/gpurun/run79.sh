timeout 900 python -m pytest tests/test_gpu_temperature.py -x -q 2>&1 | tail -15 > gpurun_out/pytest79.txt
timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench79_c2t.json
