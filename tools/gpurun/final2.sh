# refresh of the configs the K3 tile change touches (batches >= 16 K items) + the C2 launch list
tag=${1:-x}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.txt 2>&1
for c in c5 c5s c5p c2skip c1; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --e2e-steps 2 --cpu-seconds 5 > gpurun_out/${tag}_bench_$c.txt 2>&1
done
timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_stage_cost.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${tag}_launches_c2.log 2>&1
