# round-2 ncu evidence: the C2 step launch list, one --set full capture of the
# roofline K1 launch and of the big-tile K3, plus the sanitizer logs
tag=${1:-x}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${tag}_launches_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_k1a python tools/k1_once.py --rows 50000 --batched 5 > gpurun_out/${tag}_k1a_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:route_compact_fast --launch-skip 8 --launch-count 1 \
  -o gpurun_out/${tag}_k3 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-graph > gpurun_out/${tag}_k3_ncu.log 2>&1
bash tools/gpurun/sanitize.sh ${tag}
