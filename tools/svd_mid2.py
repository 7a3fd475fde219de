import sys, time, numpy as np
sys.path.insert(0,'/root/repo')
from paper_2501_12151_b200 import _native as nat
ctx = nat.default_context()
for n in (113, 120, 128, 140, 150, 159):
    m = 2*n
    rng=np.random.default_rng(n)
    a = nat.f64(rng.standard_normal((m,n)) * np.logspace(0,-8,n)[None,:])
    k=n; u,s,vt=np.empty((m,k)),np.empty(k),np.empty((k,n))
    best=1e9
    for rep in range(4):
        t0=time.perf_counter(); nat.call("qtt_svd", ctx.handle, nat.dptr(a), m, n, nat.dptr(u), nat.dptr(s), nat.dptr(vt)); best=min(best,time.perf_counter()-t0)
    ref=np.linalg.svd(a,compute_uv=False)
    print(n, f"ms={best*1e3:.2f}", "sv_relerr_max=%.1e"%np.max(np.abs(s-ref)/ref), "recon=%.1e"%(np.linalg.norm((u*s)@vt-a)/np.linalg.norm(a)), "orthU=%.1e"%np.linalg.norm(u.T@u-np.eye(k)), "orthV=%.1e"%np.linalg.norm(vt@vt.T-np.eye(k)), flush=True)
