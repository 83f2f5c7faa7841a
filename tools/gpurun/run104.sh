timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest104.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke104.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench104_c2.json
