tag=${1:-x}
for r in 1 2; do
  for v in product tfsub8 tfsub4; do
    if [ $v = product ]; then L=""; else L="build/exp/libhs_$v.so"; fi
    HS_LIBHS=$L timeout 300 python bench.py --config c2t --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_tf_${v}_$r.txt 2>&1
  done
done
