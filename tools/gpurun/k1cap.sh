tag=${1:-x}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_k1a python tools/k1_once.py --rows 50000 --batched 5 > gpurun_out/${tag}_k1a_ncu.log 2>&1
