run() { timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench63_$1.json; }
run g16u8_512
HS_TF_G32=1 run g32u4_512
HS_LIBHS=build/exp/libhs_tf1024.so HS_TF_G32=1 run g32u4_1024
HS_LIBHS=build/exp/libhs_tf1024.so run g16u8_1024
