tag=${1:-x}
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap_first_equals_serial" >> gpurun_out/${tag}_alone.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_parity_default.txt 2>&1
HS_NO_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_parity_nopdl.txt 2>&1
HS_LIBHS=build/exp/libhs_noticket.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_parity_noticket.txt 2>&1
HS_LIBHS=build/exp/libhs_linargmax.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/${tag}_parity_linargmax.txt 2>&1
