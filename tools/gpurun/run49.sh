# state check after container re-creation: GPU parity suite, smoke, default bench
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest49.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke49.txt 2>&1
timeout 600 python bench.py 2>gpurun_out/bench49.err | tail -1 > gpurun_out/bench49.json
