timeout 300 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -5 > gpurun_out/pytest84.txt
timeout 600 python bench.py --placement p2p --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench84_p2p.json
