timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest96.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke96.txt 2>&1
timeout 600 python bench.py --steps 50 2>/dev/null | tail -1 > gpurun_out/bench96_c2.json
