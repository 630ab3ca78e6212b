import sys; sys.path.insert(0,'.')
import numpy as np, torch, workloads, paper_2006_11267_b200 as pb
def dev(a): return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
cfg = workloads.scaled(workloads.CONFIGS["C2"], n=1500, t=8)
inp = workloads.make_inputs(cfg)
res={}
for name, comm, impl in (("single-auto",None,"auto"),("single-simt",None,"simt"),("nccl1-auto",(0,1,pb.ciq_nccl_unique_id()),"auto"),("nccl1-simt",(0,1,pb.ciq_nccl_unique_id()),"simt")):
    kwc = {} if comm is None else dict(comm=comm)
    with pb.CIQ("dense", K=dev(inp["K"]), diag=cfg.sigma2, **kwc) as g:
        out = torch.empty((cfg.n, cfg.t), device="cuda")
        info = g.apply(dev(inp["B"]), out, lanczos_start=dev(inp["S"]), q=8, max_iters=60, tol=0.0, mode="sqrt", mvm_impl=impl)
        res[name]=out.cpu().numpy().astype(np.float64)
        print(name, info["mvm_impl_used"], info["lambda_min"], info["lambda_max"], info["mvm_splits"], flush=True)
a=res["single-auto"]
for k,v in res.items(): print(k, np.linalg.norm(v-a)/np.linalg.norm(a))
