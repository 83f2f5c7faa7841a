timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest93.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke93.txt 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench93_c2.json
for c in c1 c3 c3m c3k c4 c5 c2t c2g; do timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench93_$c.json; done
timeout 600 python bench.py --placement p2p --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench93_p2p.json
