# fused step (HS_FUSE=1) vs the two-launch step: tests, stage costs, globaltimer trace
tag=${1:-fz}
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/${tag}_pytest_fused.txt 2>&1
HS_FUSE=1 timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_fused.txt 2>&1
timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_nofuse.txt 2>&1
HS_LIBHS=build/exp/libhs_fztrace.so timeout 300 python tools/fz_trace.py > gpurun_out/${tag}_fz_trace.txt 2>&1
