tag=${1:-x}
SEL="dense_step_full_size_every_request or overlap_first_equals_serial"
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "$SEL" >> gpurun_out/${tag}_pair_default.txt 2>&1
  HS_NO_PDL=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "$SEL" >> gpurun_out/${tag}_pair_nopdl.txt 2>&1
  HS_LIBHS=build/exp/libhs_noticket.so timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "$SEL" >> gpurun_out/${tag}_pair_noticket.txt 2>&1
done
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "$SEL" > gpurun_out/${tag}_pair_blocking.txt 2>&1
timeout 1800 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "(dense_step_full_size_every_request and c2-False) or overlap_first_equals_serial" > gpurun_out/${tag}_pair_memcheck.txt 2>&1
