"""N > 1 path with one process per rank.

* CPU (gloo, world 2 and 4): host-side logic -- length all-gather (step a1), max-over-ranks
  timing reduction, window-handle exchange plumbing.
* GPU (marked gpu): W processes on one B200 exchange through CUDA-IPC-mapped windows with the
  fused P2P exec and its epoch barrier; bit-exact against the oracle, several execs in a row.
"""
import multiprocessing as mp
import random
import socket

import pytest

from paper_2510_05943_b200 import workloads as W
from tests import mp_worker


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_procs(target, world, extra=(), timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + tuple(extra)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, msg = q.get(timeout=timeout)
            res[r] = msg
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, bad
    assert len(res) == world


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_host_logic(world):
    run_procs(mp_worker.cpu_main, world)


def _gpu_ok():
    import torch
    return torch.cuda.is_available()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "staged"])
@pytest.mark.parametrize("name", ["c1_dp2_dp1", "c3_dp4_tp4", "c4_dp4_sp2", "random",
                                  "c3_dp8_dp2tp4", "c4_dp8_dp4sp2"])
def test_p2p_exec_processes_share_one_gpu(name, mode):
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    f3 = W.field_set("tiny3") + [("m", 1, 1, "mask")]
    if name == "c1_dp2_dp1":
        world, lens = 2, W.TINY_LENGTHS.tolist()
        src, dst = W.rollout_layout(8, 2), W.layout(dp=1, assign="contig")
    elif name == "c3_dp4_tp4":
        world, lens = 4, W.c2_lengths(0)[:40].tolist()
        src, dst = W.config_layouts("c3", 4, 40)
    elif name == "c4_dp4_sp2":
        world, lens = 4, W.c4_lengths(0)[:10].tolist()
        src, dst = W.config_layouts("c4", 4, 10)
    elif name == "c3_dp8_dp2tp4":  # bench.py's N = 8 layouts (DP8 -> DP2 x TP4), 8 processes
        world, lens = 8, W.c2_lengths(0)[:64].tolist()
        src, dst = W.config_layouts("c3", 8, 64)
    elif name == "c4_dp8_dp4sp2":  # config 4 at 8 ranks (DP8 -> DP4 x SP2)
        world, lens = 8, W.c4_lengths(0)[:24].tolist()
        src, dst = W.config_layouts("c4", 8, 24)
    else:
        from tests.helpers import random_layout
        rng = random.Random(3)
        world, n = 3, 30
        lens = [rng.randint(0, 300) for _ in range(n)]
        src = random_layout(rng, world, n, allow_lpt=True)
        dst = random_layout(rng, world, n, allow_lpt=True)
    run_procs(mp_worker.gpu_main, world, extra=((lens, src, dst, f3, 3, mode),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("world,tp", [(2, 1), (4, 2)])
def test_distributed_advantages_processes(world, tp):
    """Reading n5 across processes: the only cross-rank traffic is the 3-double all-reduce."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    lens = W.c2_lengths(0)[:48].tolist()
    src = W.layout(dp=world // tp, tp=tp, assign="contig")
    run_procs(mp_worker.gpu_adv_main, world, extra=((lens, src, 0.99),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("world,flag", [(2, False), (4, True), (4, False)])
def test_role_plans_processes(world, flag):
    """Per-role routing across processes: several plans' receive buffers side by side in one
    IPC window, fused P2P exec of each group."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    lens = W.c2_lengths(1)[:40].tolist()
    src = W.rollout_layout(len(lens), world)
    dst = W.layout(dp=max(1, world // 2), tp=2 if world >= 2 else 1, assign="lpt")
    run_procs(mp_worker.gpu_roles_main, world, extra=((lens, src, dst, flag, world - 1),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_missing_peer_times_out(world):
    """A rank that never joins the exchange: the others report EARL_ERR_TIMEOUT with its bit."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    run_procs(mp_worker.gpu_timeout_main, world, extra=(W.TINY_LENGTHS.tolist(),), timeout=300)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_plan_hash_mismatch_detected(world):
    """Every rank plans the same batch: Dispatcher.check_plan passes; one rank with other lengths:
    every rank raises EARL_ERR_MISMATCH (SURVEY.md §7 replicated deterministic planning)."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    run_procs(mp_worker.gpu_hash_main, world, extra=(W.c2_lengths(0)[:48].tolist(),), timeout=300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dp2_to_dp1", "disjoint_2to2", "tp2_dst_one_src", "random4"])
def test_source_only_ranks_pass_null_recv(name):
    """a rank that receives nothing passes NULL receive buffers and still sends
    every record; receive offsets differ per rank (published by each destination)."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    f = W.field_set("tiny3") + [("m", 1, 1, "mask"), ("h", 2, 24, "hidden")]
    if name == "dp2_to_dp1":            # rank 1 is source-only
        world, lens = 2, W.TINY_LENGTHS.tolist()
        src, dst = W.rollout_layout(8, 2), W.layout(dp=1, assign="contig")
    elif name == "disjoint_2to2":      # ranks 0,1 source-only; 2,3 destination-only
        world, lens = 4, W.c2_lengths(0)[:30].tolist()
        src = dict(W.rollout_layout(30, 2))
        dst = dict(W.layout(dp=2, assign="contig"), rank0=2)
    elif name == "tp2_dst_one_src":    # one source rank feeds a TP2 group on the other ranks
        world, lens = 3, W.c2_lengths(0)[:20].tolist()
        src = W.rollout_layout(20, 1)
        dst = dict(W.layout(dp=1, tp=2, assign="contig"), rank0=1)
    else:
        from tests.helpers import random_layout
        rng = random.Random(11)
        world, n = 4, 25
        lens = [rng.randint(0, 200) for _ in range(n)]
        src = random_layout(rng, world, n, allow_lpt=True)
        dst = random_layout(rng, world, n, allow_lpt=True)
    run_procs(mp_worker.gpu_null_recv_main, world, extra=((lens, src, dst, f),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_late_peer_reports_skipped_copies(world):
    """ranks whose entry barrier timed out skip their copies and flag it in
    their done signal; the late rank reports TIMEOUT naming them."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    run_procs(mp_worker.gpu_late_peer_main, world, extra=(W.TINY_LENGTHS.tolist(),), timeout=300)


@pytest.mark.gpu
def test_nccl_staged_exchange_in_library():
    """K8: the staged exchange as library NCCL calls, bit-exact vs the oracle."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    lens = W.c2_lengths(2)[:40].tolist()
    f = W.field_set("scalar6-fp32") + [("h", 2, 40, "hidden")]
    run_procs(mp_worker.gpu_nccl_main, 1, extra=((lens, f),), timeout=300)


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"EARL_REMOTE_STORE": "tma"}, {"EARL_COPY_CFG_P2P": "3"},
                                 {"EARL_REMOTE_STORE": "tma", "EARL_COPY_CFG_P2P": "1"}])
@pytest.mark.parametrize("name", ["c3_dp8_dp2tp4", "c4_dp4_sp2"])
def test_p2p_store_variants(name, env, monkeypatch):
    """The NVLink options of the fused exec: peer replicas by bulk TMA stores
    (EARL_REMOTE_STORE=tma) and a forced launch shape for multi-process launches
    (EARL_COPY_CFG_P2P), bit-exact against the oracle like the defaults."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    f3 = W.field_set("tiny3") + [("m", 1, 1, "mask"), ("h", 2, 64, "hidden")]
    if name == "c3_dp8_dp2tp4":
        world, lens = 8, W.c2_lengths(0)[:64].tolist()
        src, dst = W.config_layouts("c3", 8, 64)
    else:
        world, lens = 4, W.c4_lengths(0)[:10].tolist()
        src, dst = W.config_layouts("c4", 4, 10)
    run_procs(mp_worker.gpu_main, world, extra=((lens, src, dst, f3, 2, "fused"),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dp1_to_tp4", "c3_dp4_dp1tp4", "c4_dp4_sp2"])
def test_nvls_vmm_windows(name):
    """NEXT-3: EARL_NVLS=1 windows (cuMemCreate + file-descriptor export) carry the fused exec
    bit-exactly; multicast teams are used where the device can make them, and report
    EARL_ERR_UNSUPPORTED otherwise (one visible GPU: cuMulticastCreate refuses every team)."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    f = W.field_set("tiny3") + [("m", 1, 1, "mask"), ("h", 2, 40, "hidden")]
    if name == "dp1_to_tp4":      # the egress-bound case NVLS is for: one source, a TP4 group
        world, lens = 4, W.c2_lengths(0)[:20].tolist()
        src, dst = W.rollout_layout(20, 1), W.layout(dp=1, tp=4, assign="contig")
    elif name == "c3_dp4_dp1tp4":
        world, lens = 4, W.c2_lengths(0)[:40].tolist()
        src, dst = W.config_layouts("c3", 4, 40)
    else:
        world, lens = 4, W.c4_lengths(0)[:10].tolist()
        src, dst = W.config_layouts("c4", 4, 10)
    run_procs(mp_worker.gpu_nvls_main, world, extra=((lens, src, dst, f),), timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c3_2x4", "c4_2x4", "c3_4x2", "tp_spans_nodes", "random_2x3"])
def test_hierarchical_exec_virtual_nodes(name):
    """NEXT-4: a comm spanning 'nodes' (groups of processes sharing one GPU): fused P2P inside a
    node, staged messages between nodes; bit-exact against the oracle."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    f = W.field_set("tiny3") + [("m", 1, 1, "mask"), ("h", 2, 24, "hidden")]
    if name == "c3_2x4":          # 2 nodes x 4 ranks: DP8 -> DP2 x TP4 (a TP group per node)
        world, ns, lens = 8, 4, W.c2_lengths(0)[:64].tolist()
        src, dst = W.config_layouts("c3", 8, 64)
    elif name == "c4_2x4":        # DP8 -> DP4 x SP2
        world, ns, lens = 8, 4, W.c4_lengths(0)[:24].tolist()
        src, dst = W.config_layouts("c4", 8, 24)
    elif name == "c3_4x2":        # 4 nodes x 2 ranks: every TP4 group spans two nodes
        world, ns, lens = 8, 2, W.c2_lengths(1)[:48].tolist()
        src, dst = W.config_layouts("c3", 8, 48)
    elif name == "tp_spans_nodes":  # one source, a TP4 group across 2 nodes of 2
        world, ns, lens = 4, 2, W.c2_lengths(2)[:20].tolist()
        src, dst = W.rollout_layout(20, 1), W.layout(dp=1, tp=4, assign="contig")
    else:
        from tests.helpers import random_layout
        rng = random.Random(29)
        world, ns, n = 6, 3, 40
        lens = [rng.randint(0, 300) for _ in range(n)]
        src = random_layout(rng, world, n, allow_lpt=True)
        dst = random_layout(rng, world, n, allow_lpt=True)
    run_procs(mp_worker.gpu_hier_main, world, extra=((lens, src, dst, f, ns),), timeout=900)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_length_gather_missing_peer_times_out(world):
    """a1 on the device: a rank that never joins the gather is named by the others' TIMEOUT."""
    if not _gpu_ok():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    build.build()
    run_procs(mp_worker.gpu_gather_timeout_main, world, extra=(None,), timeout=300)
