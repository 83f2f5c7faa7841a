timeout 600 python tools/ablate.py --config c2 > gpurun_out/ablate78_c2.txt 2>&1
timeout 600 python tools/ablate.py --config c5 > gpurun_out/ablate78_c5.txt 2>&1
