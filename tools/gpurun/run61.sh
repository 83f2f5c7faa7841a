timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest61.txt
for c in c3 c4; do timeout 900 python bench.py --config $c --e2e-steps 0 --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench61_${c}.json; done
