timeout 600 python tools/ablate.py --config c1 > gpurun_out/ablate81_c1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph > /dev/null 2>&1
