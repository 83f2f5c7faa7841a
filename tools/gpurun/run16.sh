tag=${1:-x}
timeout 600 python -m pytest tests/test_gpu_forward.py -q -k "cascade_step_equals" > gpurun_out/${tag}_placed_vr.txt 2>&1
timeout 300 python bench.py --gpus 2 --share-gpu --placement placed --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/${tag}_placed2.txt 2>&1
bash tools/gpurun/profile.sh ${tag}
