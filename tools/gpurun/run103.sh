timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k topk 2>&1 | tail -3 > gpurun_out/pytest103.txt
timeout 900 python bench.py --config c3k --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench103_c3k.json
