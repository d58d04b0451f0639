import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_05943_b200 import workloads as W, earl
from paper_2510_05943_b200.dispatch import EmulatedDispatch
ed = EmulatedDispatch(8)
for n in (1000, 5000, 60000):
    rng = np.random.default_rng(n); lens = rng.integers(0, 48, size=n).tolist()
    try:
        p = ed.plan(W.rollout_layout(n, 8), W.layout(dp=2, sp=2, tp=2, assign="contig"), lens, [("m",1,1,"x")])
        p.sync(); print(n, "plan ok", p.stats()["records"])
        recv = ed.alloc_recv(p, [("m",1,1,"x")])
        send = [torch.zeros(10**6, dtype=torch.uint8, device="cuda") for _ in range(8)]
        p.exec(send, ed.flat(recv)); torch.cuda.synchronize(); print(n, "exec ok")
    except Exception as e:
        print(n, "ERR", e)
