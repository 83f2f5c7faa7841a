tag=${1:-x}
for f in test_abi test_gpu_comm test_gpu_forward test_gpu_fullsize test_gpu_multiproc; do
  timeout 600 python -m pytest tests/$f.py tests/test_gpu_parity.py -q -x -m gpu -k "not production and not topk and not skip and not split" > gpurun_out/${tag}_pair_$f.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_full.txt 2>&1
