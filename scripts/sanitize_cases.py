"""A handful of GPU cases for compute-sanitizer runs: dispatch (each bit-exact vs the oracle) and
the NEXT-2 returns / advantages kernels (within the n5 bound)."""
import random
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_05943_b200 import workloads as W  # noqa: E402
from tests.helpers import random_layout, run_gpu_case  # noqa: E402
from tests.test_oracle_sp_variants import with_split  # noqa: E402

fields = [("a", 4, 1, "x"), ("m", 1, 1, "x"), ("h", 2, 8, "x")]
lens8 = W.TINY_LENGTHS.tolist()
run_gpu_case(W.rollout_layout(8, 2), W.layout(dp=1, tp=2, assign="contig"), lens8, fields, 2, mode="exec")
run_gpu_case(W.rollout_layout(8, 2), W.layout(dp=1, sp=2, assign="contig", sp_split="zigzag"), lens8, fields, 2, mode="stage")
run_gpu_case(W.rollout_layout(8, 2), W.layout(dp=2, assign="lpt"), lens8, fields, 2)
for seed in range(4):
    rng = random.Random(900 + seed)
    world = rng.randint(2, 8)
    n = rng.randint(5, 60)
    lens = [rng.randint(0, 300) for _ in range(n)]
    src = with_split(rng, random_layout(rng, world, n))
    dst = with_split(rng, random_layout(rng, world, n))
    run_gpu_case(src, dst, lens, fields, world, mode=rng.choice(["exec", "stage"]), seed=seed)
# the cooperative multi-CTA planner (N = 9000: 3 CTAs) with monotone layouts (GIVEN_COUNTS ->
# CONTIG, no phase-2 partition) and with an EXPLICIT destination; zero-copy host sources
rng = random.Random(77)
lensN = [rng.randint(0, 40) for _ in range(9000)]
run_gpu_case(W.rollout_layout(9000, 4), W.layout(dp=2, tp=2, assign="contig"), lensN, fields, 4)
run_gpu_case(W.rollout_layout(9000, 4), W.layout(dp=4, assign="explicit", group_of_seq=[i % 4 for i in range(9000)]),
             lensN, fields, 4, mode="stage")
run_gpu_case(W.rollout_layout(8, 2), W.layout(dp=1, tp=2, assign="contig"), lens8, fields, 2, host_src=True)
# the congruent-heavy copy-engine shape (>= 90% of the bytes in 16-B-multiple fields: 2 warps x
# 2 stages x 16 KB, TMA bulk stores to every TP replica)
hid = [("h", 2, 64, "x"), ("a", 4, 1, "x")]
run_gpu_case(W.rollout_layout(60, 4), W.layout(dp=1, tp=4, assign="contig"),
             [rng.randint(0, 300) for _ in range(60)], hid, 4)
run_gpu_case(W.rollout_layout(60, 4), W.layout(dp=2, sp=2, assign="contig"),
             [rng.randint(0, 300) for _ in range(60)], hid, 4, mode="stage")
# NEXT-2: per-sequence fields, returns (look-back across windows, zero-length sequences,
# unaligned scalar path) and advantages, each against the oracle
from tests.test_gpu_parity import _adv_case  # noqa: E402
_adv_case([20_000, 3, 0, 1500, 7, 0], W.layout(dp=2, assign="given_counts", counts=[3, 3]), 1.0, 4)
_adv_case([1 + (i % 5) for i in range(700)], W.layout(dp=3, tp=2, assign="lpt"), 0.9, 8, shift=1)
_adv_case(W.lognormal_lengths(60, 900, 0.8, 1, 5000, seed=3).tolist(), W.layout(dp=4, assign="contig"),
          0.99, 4, repeats=2)
# round 2: the returns unit kernel on the same cases (EARL_RETURNS=units), the general planner
# on an SP = 1 layout (EARL_PLAN_PATH=general; the SP = 1 fast planner ran in every case above),
# the emulated a1 gather, and a multi-CTA fast-planner grid with an LPT source
os.environ["EARL_RETURNS"] = "units"
_adv_case([20_000, 3, 0, 1500, 7, 0], W.layout(dp=2, assign="given_counts", counts=[3, 3]), 1.0, 4)
_adv_case([1 + (i % 5) for i in range(700)], W.layout(dp=3, tp=2, assign="lpt"), 0.9, 8, shift=1)
_adv_case(W.lognormal_lengths(600, 900, 0.8, 1, 5000, seed=3).tolist(), W.layout(dp=4, assign="contig"),
          0.99, 4, repeats=2)
del os.environ["EARL_RETURNS"]
os.environ["EARL_PLAN_PATH"] = "general"
run_gpu_case(W.rollout_layout(9000, 4), W.layout(dp=4, assign="explicit", group_of_seq=[i % 4 for i in range(9000)]),
             lensN, fields, 4)
del os.environ["EARL_PLAN_PATH"]
run_gpu_case(W.layout(dp=3, assign="lpt"), W.layout(dp=2, tp=2, assign="contig"), lensN[:5000], fields, 4)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2510_05943_b200.dispatch import EmulatedDispatch  # noqa: E402
ed = EmulatedDispatch(4)
cnts = [700, 0, 1301, 5]
ln = np.random.default_rng(1).integers(0, 5000, size=sum(cnts)).astype(np.int32)
edges = np.concatenate([[0], np.cumsum(cnts)])
loc = [torch.as_tensor(ln[edges[r]:edges[r + 1]]).cuda() if cnts[r] else None for r in range(4)]
got = ed.allgather_lens(loc, cnts)
torch.cuda.synchronize()
assert got.cpu().numpy().tolist() == ln.tolist()
print("sanitize cases ok")
