timeout 600 python bench.py 2>gpurun_out/b83.err | tail -1 > gpurun_out/bench83_default.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 20 --warmup 3 2>>gpurun_out/b83.err | tail -1 > gpurun_out/bench83_torchrun.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>>gpurun_out/b83.err | tail -1 > gpurun_out/bench83_ref.json
tail -3 gpurun_out/b83.err
