timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" 2>&1 | grep -E "^E |passed|failed|Error" | head -30
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
