tag=${1:-x}
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -m gpu -k "not production and not topk and not skip and not split" >> gpurun_out/${tag}_pairfull.txt 2>&1
done
for i in 1 2; do
  CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -m gpu -k "not production and not topk and not skip and not split" >> gpurun_out/${tag}_pairfull_blocking.txt 2>&1
  HS_LIBHS=build/exp/libhs_noticket.so timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -m gpu -k "not production and not topk and not skip and not split" >> gpurun_out/${tag}_pairfull_noticket.txt 2>&1
done
