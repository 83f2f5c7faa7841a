# A/B of K1 variants on one box (interleaved, two rounds) + GPU tests of the product build
tag=${1:-x}
for r in 1 2; do
  for v in product r1argmax linargmax l2reread; do
    if [ $v = product ]; then L=""; else L="build/exp/libhs_$v.so"; fi
    HS_LIBHS=$L timeout 300 python tools/ab_k1.py --reps 30 >> gpurun_out/${tag}_ab.jsonl 2>>gpurun_out/${tag}_ab.err
  done
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.txt 2>&1
timeout 400 python bench.py --steps 100 > gpurun_out/${tag}_bench.txt 2>&1
