# peer-memory group tests (virtual ranks) + C2 launch list with the Table-III-like generator
tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q > gpurun_out/${tag}_peer_tests.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${tag}_ncu_bench.log 2>&1
