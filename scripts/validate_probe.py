import sys, time, torch, os
sys.path.insert(0, os.getcwd())
from paper_1805_06124_b200 import inputs, rbg
N=10000; cols=int(sys.argv[1]) if len(sys.argv)>1 else 409600
t=inputs.chirp_grid(N); w=inputs.simpson_weights(N)
q,chi,psi=inputs.chirp_params(cols,2,spin=True)
S=torch.empty((cols,N),dtype=torch.complex128,device="cuda"); rbg.gen_chirp(S,t,w,q,chi,psi,spin=True)
qv,cv,pv=inputs.chirp_params(40960,12,spin=True)
V=torch.empty((40960,N),dtype=torch.complex128,device="cuda"); rbg.gen_chirp(V,t,w,qv,cv,pv,spin=True)
with rbg.Context(S,w,0.0,300) as ctx:
    ctx.run(); torch.cuda.synchronize()
    for X in (V[:1024], V, V, V[:1024], V):
        t0=time.perf_counter(); ctx.validate(X); print(X.shape[0], round((time.perf_counter()-t0)*1e3,1), 'ms', flush=True)
