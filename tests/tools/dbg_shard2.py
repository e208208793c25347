"""Debug: 2 processes on one GPU, host-staged exchange; print Y checksums per mode."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, torch.multiprocessing as tmp
import oracle as O
def w(rank, port, q):
    import torch.distributed as dist
    import paper_0909_4969_b200.sharded as SH
    os.environ["MASTER_ADDR"]="127.0.0.1"; os.environ["MASTER_PORT"]=str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    orig = SH.sharded_sweeps
    log = []
    def patched(engine, ar, d, sweeps, tol):
        def ar2(y):
            a = float(y.double().sum())
            ar(y)
            torch.cuda.synchronize()
            b = float(y.double().sum())
            y2 = engine.s.mode_y  # noqa
            log.append((round(a, 6), round(b, 6)))
        return orig(engine, ar2, d, sweeps, tol)
    SH.sharded_sweeps = patched
    dims=(40,30,36); x=O.random_tensor(list(dims),13).astype("float32"); S=40*30
    t0,t1=SH.slab_bounds(36,2,rank)
    flat=torch.from_numpy(x.reshape(-1,order="F")[t0*S:t1*S].copy()).cuda()
    m,sp=SH.sharded_mach_hooi(flat,dims,(4,3,5),0.2,7,2,0.0,in_library=False)
    q.put((rank,log,m.sweep_fits)); dist.destroy_process_group()
if __name__=="__main__":
    import socket
    s=socket.socket(); s.bind(("127.0.0.1",0)); port=s.getsockname()[1]; s.close()
    c=tmp.get_context("spawn"); q=c.Queue()
    ps=[c.Process(target=w,args=(r,port,q)) for r in range(2)]
    [p.start() for p in ps]
    for _ in range(2): print(q.get(timeout=300))
    [p.join() for p in ps]
