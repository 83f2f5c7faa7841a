nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_1_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_1_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2_1_bench_c2.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_1_pytest.txt 2>&1
