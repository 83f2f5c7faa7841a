export HS_CONF_IMPL=async
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_ --launch-skip 2 --launch-count 1 -f -o gpurun_out/k1_async python tools/k1_once.py --rows 250000 > gpurun_out/k1_async.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_ --launch-skip 2 --launch-count 1 -f -o gpurun_out/k1_async_b5 python tools/k1_once.py --rows 50000 --batched 5 > gpurun_out/k1_async_b5.log 2>&1
tail -1 gpurun_out/k1_async.log gpurun_out/k1_async_b5.log
