"""One small dispatch (plan + exec + pack/unpack) for checking ncu's NVTX filters."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402
ed = EmulatedDispatch(2)
lens = W.TINY_LENGTHS.tolist()
f = W.field_set("tiny3")
plan = ed.plan(W.rollout_layout(8, 2), W.layout(dp=1, assign="contig"), lens, f)
tok = W.rollout_token_counts(lens, [4, 4])
send = [torch.zeros(max(16, t * 4), dtype=torch.uint8, device="cuda") for t in tok for _ in range(3)]
recv = ed.flat(ed.alloc_recv(plan, f))
plan.exec(send, recv)
torch.cuda.synchronize()
print("probe done")
