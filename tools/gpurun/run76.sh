run() { timeout 900 python bench.py --config c3k --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench76_$1.json; }
run u4
HS_LIBHS=build/exp/libhs_topk8.so run u8
HS_LIBHS=build/exp/libhs_topk8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k topk 2>&1 | tail -2 > gpurun_out/pytest76_u8.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k topk 2>&1 | tail -2 > gpurun_out/pytest76_u4.txt
