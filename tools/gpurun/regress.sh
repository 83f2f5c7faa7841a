# the GPU suite, smoke and the default bench line (outputs gpurun_out/<tag>_*)
tag=${1:-r}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench_c2.txt 2>&1
