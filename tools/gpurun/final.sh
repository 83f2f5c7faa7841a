# final evidence of the round: GPU suite, smoke, every bench config, stage costs,
# the C2 step launch list, one --set full capture of the roofline K1 launch, and
# memcheck over the fused / last-stage step tests
tag=${1:-x}
bash tools/gpurun/validate.sh ${tag}
timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_stage_cost.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${tag}_launches_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_k1a python tools/k1_once.py --rows 50000 --batched 5 > gpurun_out/${tag}_k1a_ncu.log 2>&1
