# multi-process peer path on one GPU (--share-gpu) + the virtual-rank tests + N=1 bench
tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_forward.py -q > gpurun_out/${tag}_peer_tests.txt 2>&1
timeout 300 python bench.py --steps 50 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${tag}_bench1.txt 2>&1
timeout 300 python bench.py --gpus 2 --share-gpu --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_bench2share.txt 2>&1
echo "rc=$?" >> gpurun_out/${tag}_bench2share.txt
