timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" 2>&1 | grep -E "^E |passed|failed|Error" | head -20
timeout 900 python bench.py --config c3k --e2e-steps 0 --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench48_c3k.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_topk --launch-skip 8 --launch-count 1 -f -o gpurun_out/k1c_c3k python bench.py --config c3k --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
