# K3 descriptor ordering A/B (relaxed vs acquire/release) on one box + the GPU suite
tag=${1:-k}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.txt 2>&1
for r in 1 2; do
  timeout 300 python tools/stage_cost.py --only full,routing_only,steps_fixed,step_fixed_2,step_fixed_3,step_fixed_4 > gpurun_out/${tag}_sc_relaxed$r.txt 2>&1
  HS_LIBHS=build/exp/libhs_k3acqrel.so timeout 300 python tools/stage_cost.py --only full,routing_only,steps_fixed,step_fixed_2,step_fixed_3,step_fixed_4 > gpurun_out/${tag}_sc_acqrel$r.txt 2>&1
done
