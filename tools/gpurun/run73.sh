timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest73.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke73.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench73_c2.json
for c in c1 c3 c4 c5 c3k c2t c2g; do timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench73_$c.json; done
