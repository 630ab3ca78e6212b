import sys; sys.path.insert(0,'.')
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
from oracle import KernelOperator, ciq, estimate_spectrum, hht_rule
def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
def relerr(x,y): return float(np.linalg.norm(np.asarray(x,np.float64)-y)/np.linalg.norm(y))
for d, ls in ((12, np.linspace(0.6,1.2,12)), (12, np.linspace(0.3,0.6,12)), (6, 0.15)):
    n,t=2000,32
    x=workloads.points(n,d); b=workloads.rhs(n,t)
    f=np.asarray(ls,np.float32).astype(np.float64)
    op=KernelOperator(x,"rbf",f,1.0,0.05)
    lmin,lmax,_,_=estimate_spectrum(op.mvm, workloads.lanczos_start(n),10,lower_bound=0.05)
    rule=hht_rule(lmin,lmax,8)
    conv=ciq(op,b.astype(np.float64),q=8,max_iters=1000,tol=1e-7,mode="sqrt",rule=rule)
    j=conv.iters
    ref=ciq(op,b.astype(np.float64),q=8,max_iters=j,tol=0.0,mode="sqrt",rule=rule)
    for impl in ("simt","tc"):
        with pb.CIQ("rbf",X=dev(x),lengthscale=ls,outputscale=1.0,diag=0.05) as g:
            out=torch.empty((n,t),device="cuda")
            info=g.apply(dev(b),out,q=8,max_iters=j,tol=0.0,mode="sqrt",rule=rule,mvm_impl=impl)
        print(d, "lmax %.1f J %d"%(lmax,j), impl, info["mvm_impl_used"], "err %.2e"%relerr(out.cpu().numpy(),ref.out), flush=True)
