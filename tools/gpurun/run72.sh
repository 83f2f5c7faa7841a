timeout 600 python bench.py --placement p2p --steps 20 --no-cpu-baseline 2>gpurun_out/b72.err | tail -1 > gpurun_out/bench72_p2p.json
tail -5 gpurun_out/b72.err
timeout 600 python bench.py --placement p2p --config c4 --steps 10 --no-cpu-baseline 2>>gpurun_out/b72.err | tail -1 > gpurun_out/bench72_p2p_c4.json
timeout 600 python bench.py --placement balanced --steps 20 --no-cpu-baseline 2>>gpurun_out/b72.err | tail -1 > gpurun_out/bench72_bal.json
tail -3 gpurun_out/b72.err
