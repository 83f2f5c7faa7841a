tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_temperature.py -q -x -k "conf or cascade or overlap or topk or split or temperature or fit" > gpurun_out/${tag}_tests.txt 2>&1
for r in 1 2; do
  for v in product nofold; do
    if [ $v = product ]; then L=""; else L="build/exp/libhs_$v.so"; fi
    HS_LIBHS=$L timeout 300 python bench.py --steps 200 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench_${v}_$r.txt 2>&1
  done
  for v in product tfnofold; do
    if [ $v = product ]; then L=""; else L="build/exp/libhs_$v.so"; fi
    HS_LIBHS=$L timeout 300 python bench.py --config c2t --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_tf_${v}_$r.txt 2>&1
  done
done
