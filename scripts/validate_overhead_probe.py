import sys, time, torch, json
sys.path.insert(0, '/root/repo')
from paper_1805_06124_b200 import inputs, rbg
N=10000; t=inputs.chirp_grid(N); w=inputs.simpson_weights(N)
q,c,p=inputs.chirp_params(40960,2,spin=True)
S=torch.empty((40960,N),dtype=torch.complex128,device='cuda'); rbg.gen_chirp(S,t,w,q,c,p,spin=True)
V=torch.empty((40960,N),dtype=torch.complex128,device='cuda'); rbg.gen_chirp(V,t,w,*inputs.chirp_params(40960,12,spin=True),spin=True)
out={}
with rbg.Context(S,w,0.0,300) as ctx:
    ctx.run()
    for m in [16, 1024, 8192, 40960]:
        ctx.validate(V[:m])
        ts=[]
        for _ in range(3):
            torch.cuda.synchronize(); t0=time.perf_counter(); ctx.validate(V[:m]); ts.append(time.perf_counter()-t0)
        out[m]=min(ts)*1e3
print(json.dumps(out))
