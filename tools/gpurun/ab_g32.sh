tag=${1:-g}
for r in 1 2; do
  timeout 300 python tools/stage_cost.py --only full,k1_stage_1,k1_stage_2,k1_stage_5 > gpurun_out/${tag}_sc_g16_$r.txt 2>&1
  HS_LIBHS=build/exp/libhs_k1g32.so timeout 300 python tools/stage_cost.py --only full,k1_stage_1,k1_stage_2,k1_stage_5 > gpurun_out/${tag}_sc_g32_$r.txt 2>&1
done
