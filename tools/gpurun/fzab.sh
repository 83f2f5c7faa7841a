# fused step (HS_FUSE=1) vs the two-launch step: tests, stage costs, timing-bound builds
tag=${1:-fz}
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/${tag}_pytest_fused.txt 2>&1
HS_FUSE=1 timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_fused.txt 2>&1
timeout 300 python tools/stage_cost.py > gpurun_out/${tag}_sc_nofuse.txt 2>&1
for v in $2; do
  HS_FUSE=1 HS_ALLOW_EXPERIMENT=1 HS_LIBHS=build/exp/libhs_$v.so timeout 300 python tools/stage_cost.py --only steps_fixed,step_fixed_1,step_fixed_2,step_fixed_3,step_fixed_4,step_fixed_5 > gpurun_out/${tag}_sc_$v.txt 2>&1
done
