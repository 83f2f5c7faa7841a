# multi-process peer test + one ncu --set full capture (with source) of the roofline K1 launch
tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -s > gpurun_out/${tag}_multiproc.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${tag}_k1a python tools/k1_once.py --rows 50000 --batched 5 > gpurun_out/${tag}_k1a_ncu.log 2>&1
