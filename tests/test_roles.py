"""NEXT-2 per-role routing (SPEC.md:248-256 route_noncritical_tensors): the role table on the
host (CPU) and the routed plan set against the oracle on the GPU."""
import random

import numpy as np
import pytest

from oracle import earl_oracle as O
from paper_2510_05943_b200 import workloads as W
from paper_2510_05943_b200.dispatch import controller_layout, route_roles


def test_route_roles_spec_examples():
    # SPEC.md:254 batch {log_probs, rewards} -> {log_probs: all_to_all, rewards: gather}
    assert route_roles({"lp": "log_probs", "r": "rewards"}) == {"lp": "all_to_all", "r": "gather"}
    # SPEC.md:255 flag enabled -> both all_to_all (distributed aggregation, §5)
    assert route_roles({"lp": "log_probs", "r": "rewards"}, distributed_aggregation=True) == \
        {"lp": "all_to_all", "r": "all_to_all"}
    # SPEC.md:256 zero tensors -> empty plan set
    assert route_roles({}) == {}
    assert route_roles({"G": "returns", "ids": "tokens"}) == {"G": "gather", "ids": "all_to_all"}


def test_route_roles_unknown_role_is_an_error():
    with pytest.raises(ValueError, match="unknown role 'bogus'"):
        route_roles({"x": "bogus"})


def test_controller_layout_is_a_valid_single_rank_layout():
    lay = controller_layout(3)
    O.validate_layout(lay, 5, 4)
    lens = [3, 0, 7, 1, 2]
    h = O.holdings(lay, lens, O.assign_groups(lay, lens))
    assert list(h) == [3] and h[3]["n_tokens"] == 13


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("flag", [False, True])
def test_plan_roles_on_gpu(seed, flag):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2510_05943_b200 import build
    from paper_2510_05943_b200.dispatch import EmulatedDispatch, plan_roles
    build.build()
    rng = random.Random(900 + seed)
    world = rng.randint(2, 8)
    n = rng.choice([0, 1, rng.randint(2, 60), rng.randint(60, 300)])
    lens = [rng.randint(0, 700) for _ in range(n)]
    src = W.rollout_layout(n, world)
    dst = W.layout(dp=max(1, world // 2), tp=2 if world >= 2 else 1, assign="lpt")
    ctrl = rng.randrange(world)
    tensors = [("ids", "tokens", ("ids", 4, 1, "x"), "token"),
               ("lp", "log_probs", ("lp", 4, 1, "x"), "token"),
               ("G", "returns", ("G", 4, 1, "x"), "token"),
               ("R", "rewards", ("R", 4, 1, "x"), "sequence"),
               ("score", "values", ("score", 2, 3, "x"), "sequence")]
    routes = route_roles({t[0]: t[1] for t in tensors}, flag)
    T = sum(lens)
    gs = O.assign_groups(src, lens)
    tok_glob = {t[0]: np.random.default_rng(seed * 7 + k).integers(0, 256, T * 4, dtype=np.uint8)
                for k, t in enumerate(tensors) if t[3] == "token"}
    tok_src = {nm: O.rank_arrays_from_global(src, lens, gs, [g], [("f", 4, 1, "x")])
               for nm, g in tok_glob.items()}
    hs = O.seq_holdings(src, lens, gs)
    seq_src = {}
    for k, t in enumerate(tensors):
        if t[3] != "sequence":
            continue
        B = t[2][1] * t[2][2]
        glob = np.random.default_rng(seed * 11 + k).integers(0, 256, n * B, dtype=np.uint8)
        seq_src[t[0]] = {r: [np.concatenate([glob[i * B:(i + 1) * B] for i in m]) if m
                             else np.zeros(0, np.uint8)] for r, m in hs.items()}
    ed = EmulatedDispatch(world)
    rp = plan_roles(ed, src, dst, lens, tensors, distributed_aggregation=flag, controller=ctrl)
    send, recv, want = {}, {}, {}
    for t in tensors:
        nm = t[0]
        lay_d = dst if routes[nm] == "all_to_all" else controller_layout(ctrl)
        if t[3] == "token":
            arrs = tok_src[nm]
            w, _, _ = O.dispatch(src, lay_d, lens, arrs, [("f", 4, 1, "x")], world)
        else:
            arrs = seq_src[nm]
            w = O.dispatch_seq_fields(src, lay_d, lens, arrs, [t[2]], world)
        send[nm] = [torch.from_numpy(arrs[r][0]).cuda() if r in arrs and arrs[r][0].size else None
                    for r in range(world)]
        recv[nm] = [torch.full((max(16, w[r][0].size if r in w else 0) + 64,), 0xA5, dtype=torch.uint8,
                               device="cuda") for r in range(world)]
        want[nm] = w
    rp.exec(send, recv)
    torch.cuda.synchronize()
    for nm, w in want.items():
        for r in range(world):
            got = recv[nm][r].cpu().numpy()
            n_b = w[r][0].size if r in w else 0
            if n_b:
                assert np.array_equal(got[:n_b], w[r][0]), (nm, r)
            assert np.all(got[n_b:] == 0xA5), (nm, r, "wrote past its data")
    rp.destroy()
