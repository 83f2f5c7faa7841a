HS_LIBHS=$PWD/build/exp/libhs_ctrace.so python - <<'PY' 2>&1 | tail -30
import ctypes, torch, paper_2505_12566_b200 as hs
dev=torch.device('cuda',0)
g=torch.Generator().manual_seed(0)
for (N,K,q) in [(50000,5,12),(50000,5,4),(4096,5,12)]:
    conf=torch.rand(K-1,N,generator=g).to(dev); ok=(torch.rand(K,N,generator=g)<0.8).to(torch.uint8).to(dev)
    for _ in range(3): hs.calibrate_thresholds(conf, ok, log2_bins=q)
    torch.cuda.synchronize()
    buf=(ctypes.c_ulonglong*64)()
    hs.lib().hs_debug_calib_trace.argtypes=[ctypes.c_void_p]
    hs.lib().hs_debug_calib_trace(ctypes.addressof(buf))
    t=[buf[i] for i in range(1+6*(K-1))]
    names=['init']+['hist','sync1','pulled','select','sync2']*(K-1)
    print(N,K,q,' '.join(f'{n}:{(t[i]-t[i-1])/1000:.1f}' for i,n in enumerate(names) if i>0), 'total', (t[-1]-t[0])/1000)
PY
