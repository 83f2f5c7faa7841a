timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
HS_LIBHS=$PWD/build/exp/libhs_ctrace.so python - <<'PY' 2>&1 | tail -30
import torch, paper_2505_12566_b200 as hs
dev=torch.device('cuda',0)
g=torch.Generator().manual_seed(0)
N,K,q=50000,5,12
conf=torch.rand(K-1,N,generator=g).to(dev); ok=(torch.rand(K,N,generator=g)<0.8).to(torch.uint8).to(dev)
for _ in range(3): hs.calibrate_thresholds(conf, ok, log2_bins=q)
torch.cuda.synchronize()
print("----")
hs.calibrate_thresholds(conf, ok, log2_bins=q); torch.cuda.synchronize()
PY
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b19.json 2> gpurun_out/b19.err; tail -2 gpurun_out/b19.err; python -c "
import json; d=json.load(open('gpurun_out/b19.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2))"
python bench.py --force-dist --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b19_fd.json 2> gpurun_out/b19_fd.err; tail -3 gpurun_out/b19_fd.err; python -c "
import json; d=json.load(open('gpurun_out/b19_fd.json')); print('force-dist', round(d['value']/1e6,1), round(d['ms_per_step'],4), d['config']['cuda_graph'], d['thresholds'])"
