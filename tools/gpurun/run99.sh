timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest99.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke99.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench99_c2.json
timeout 900 python bench.py --config c4 --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench99_c4.json
