run() { timeout 900 python bench.py --config c3k --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench100_$1.json; }
run base
HS_LIBHS=build/exp/libhs_topknocand.so run nocand
