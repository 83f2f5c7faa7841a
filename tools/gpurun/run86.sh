timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "calib" 2>&1 | tail -3 > gpurun_out/pytest86.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/pytest86.txt 2>&1
for c in c1 c2; do timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench86_$c.json; done
timeout 600 python tools/ablate.py --config c1 > gpurun_out/ablate86_c1.txt 2>&1
