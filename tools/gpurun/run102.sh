run() { timeout 900 python bench.py --config c3k --steps 20 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench102_$1.json; }
for v in topkm4 topkm8 topkm4s40 topkm8s40; do HS_LIBHS=build/exp/libhs_$v.so run $v; done
