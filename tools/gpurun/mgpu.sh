# multi-process peer path on one GPU (--share-gpu) + peer/parity tests + N=1 bench
tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_fullsize.py -q -s > gpurun_out/${tag}_peer_tests.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "production or calibration_bit_exact or cascade_vs_oracle" > gpurun_out/${tag}_parity_tests.txt 2>&1
timeout 400 python bench.py --steps 50 --e2e-steps 2 > gpurun_out/${tag}_bench1.txt 2>&1
timeout 400 python bench.py --gpus 2 --share-gpu --steps 5 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_bench2share.txt 2>&1
echo "rc=$?" >> gpurun_out/${tag}_bench2share.txt
