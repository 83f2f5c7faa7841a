tag=${1:-x}
for r in 1 2; do
  for v in product ridxall; do
    if [ $v = product ]; then L=""; else L="build/exp/libhs_$v.so"; fi
    HS_LIBHS=$L timeout 300 python tools/ab_k1.py --reps 30 >> gpurun_out/${tag}_ab.jsonl 2>>gpurun_out/${tag}_ab.err
    HS_LIBHS=$L timeout 300 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_${v}_$r.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "conf or cascade or overlap or split" > gpurun_out/${tag}_tests.txt 2>&1
