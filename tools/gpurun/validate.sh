# full GPU suite, smoke, and every bench config on one B200 (outputs gpurun_out/<tag>_*)
tag=${1:-x}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.txt 2>&1
for c in c2skip c5 c5p c5s c4 c3 c1 c2t c2g c3k c3m; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --e2e-steps 2 --cpu-seconds 5 > gpurun_out/${tag}_bench_$c.txt 2>&1
done
timeout 400 python bench.py --gpus 2 --share-gpu --placement placed --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_bench_placed2.txt 2>&1
timeout 400 python bench.py --config c5p --gpus 2 --share-gpu --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_bench_c5p2.txt 2>&1
