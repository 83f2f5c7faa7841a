timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest87.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches_final.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 5 --launch-count 1 -f -o gpurun_out/k1a_c2_final python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 python tools/ablate.py --config c2 > gpurun_out/ablate87_c2.txt 2>&1
