# GPU sanity: smoke, C2 bench, full GPU test suite (outputs in gpurun_out/)
tag=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.txt 2>&1
