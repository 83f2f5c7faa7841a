tag=${1:-x}
timeout 900 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_first_equals_serial and False" > gpurun_out/${tag}_initcheck_overlap.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_parity_blocking.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "route or cascade_vs_oracle or overlap or generator or row_index" > gpurun_out/${tag}_memcheck_seq.txt 2>&1
