timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python tools/calib_bench.py > gpurun_out/calib15.json 2>&1; cat gpurun_out/calib15.json | tr '\n' ' '; echo
python tools/breakdown.py --reps 30 > gpurun_out/bd15.json 2>&1; cat gpurun_out/bd15.json
python bench.py --steps 300 --warmup 5 > gpurun_out/b15.json 2> gpurun_out/b15.err; tail -2 gpurun_out/b15.err; cat gpurun_out/b15.json
