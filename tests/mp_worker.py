"""Worker for the multi-process tests (spawned, one process per simulated rank).

CPU mode (gloo): host logic of the N>1 path -- length all-gather, max-over-ranks, handle
exchange plumbing.  GPU mode: W processes share ONE B200; each owns a comm rank whose window
is exported/imported through CUDA IPC, and the fused P2P exec (entry barrier, stores into
peers' windows, epoch release/acquire) runs for real -- only NVLink is not exercised.
"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def init(rank, world, port, backend):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def cpu_main(rank, world, port, q):
    try:
        import numpy as np
        import torch
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import allgather_lengths, max_over_ranks
        dist = init(rank, world, port, "gloo")
        lens = W.c2_lengths(0)[:50]
        counts = W.near_equal_counts(len(lens), world)
        edges = np.concatenate([[0], np.cumsum(counts)])
        mine = torch.as_tensor(lens[edges[rank]:edges[rank + 1]].astype(np.int32))
        glob, cnt = allgather_lengths(mine)
        assert cnt == counts, (cnt, counts)
        assert glob.tolist() == lens.tolist()
        # a rank holding nothing still joins
        empty = torch.zeros(0, dtype=torch.int32) if rank == 0 else mine
        glob2, cnt2 = allgather_lengths(empty)
        assert cnt2[0] == 0 and glob2.numel() == sum(cnt2)
        mx = max_over_ranks([float(rank), 10.0 - rank])
        assert mx == [float(world - 1), 10.0]
        objs = [None] * world
        dist.all_gather_object(objs, bytes([rank]) * 128)
        assert [o[0] for o in objs] == list(range(world))
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_main(rank, world, port, q, case):
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, dst, fields, n_exec = case[:5]
        staged = len(case) > 5 and case[5] == "staged"
        T = sum(lens)
        glob = W.gen_global_fields(fields, T, seed_base=77, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, meta, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
        D = Dispatcher(window_bytes=T * W.bytes_per_token(fields) + (1 << 16), device=0)
        mine = [torch.from_numpy(a).cuda() if a.size else None for a in src_arrays.get(rank, [])] \
            if rank in src_arrays else [None] * len(fields)
        # step a1: every rank holds only its own block of the lengths (the rollout's counts when
        # the source layout is GIVEN_COUNTS, else near-equal blocks) and the global vector is
        # gathered -- on the device (earl_allgather_lengths) on even iterations, by the host
        # path (counts not known in advance) on odd ones
        from paper_2510_05943_b200.dispatch import rank_counts
        cnts = rank_counts(src, world) if src.get("assign") == "given_counts" \
            else W.near_equal_counts(len(lens), world)
        edges = np.concatenate([[0], np.cumsum(cnts)]).astype(int)
        local = torch.as_tensor(np.asarray(lens[edges[rank]:edges[rank + 1]], dtype=np.int32)).cuda()
        for it in range(n_exec):
            if it % 2 == 0:
                glens, got_counts = D.allgather_lens(local, counts=cnts)
            else:
                glens, got_counts = D.allgather_lens(local)
            D.comm.check()
            assert list(got_counts) == list(cnts), (got_counts, cnts)
            assert glens.cpu().tolist() == list(lens), f"iter {it}: gathered lengths differ"
            plan = D.plan(src, dst, glens, fields)
            ptrs, views = D.alloc_recv(plan, fields)
            for v in views:
                v.fill_(0xA5)
            if staged:  # pack -> grouped send/recv -> unpack
                if it == 0:
                    send_stage, recv_stage, msgs = D.alloc_stage(plan)
                    D.exec_staged(plan, mine, ptrs, send_stage, recv_stage, msgs)
                else:
                    D.exec_staged(plan, mine, ptrs)
            else:
                plan.exec(mine, ptrs)
            torch.cuda.synchronize()
            plan.sync()
            if rank in want:
                for f in range(len(fields)):
                    got = views[f].cpu().numpy()
                    assert np.array_equal(got, want[rank][f]), f"iter {it} rank {rank} field {f}"
            plan.destroy()
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_adv_main(rank, world, port, q, case):
    """Reading n5 with one process per rank: returns on each rank, 3-double all-reduce over the
    process group, advantages -- equal to the oracle within the fp32 tolerance."""
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher, distributed_advantages
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, gamma = case
        T = sum(lens)
        rng = np.random.default_rng(5)
        glob_r = rng.standard_normal(T).astype(np.float32)
        glob_m = (rng.random(T) < 0.75).astype(np.uint8)
        fr = [("r", 4, 1, "x"), ("m", 1, 1, "x")]
        arrs = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens),
                                         [glob_r.view(np.uint8), glob_m], fr)
        rewards = {k: v[0].view(np.float32) for k, v in arrs.items()}
        masks = {k: v[1] for k, v in arrs.items()}
        G, A, R, stats = O.distributed_advantages(src, lens, rewards, masks, gamma, 1e-8, world)
        D = Dispatcher(window_bytes=1 << 20, device=0)
        plan = D.plan(src, W.layout(dp=1, tp=world, assign="contig"),
                      torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda(), W.field_set("tiny3"))
        n = rewards[rank].size
        r = torch.from_numpy(rewards[rank].copy()).cuda()
        m = torch.from_numpy(masks[rank].copy()).cuda()
        Gd = torch.zeros(max(n, 1), dtype=torch.float32, device="cuda")
        Ad = torch.zeros(max(n, 1), dtype=torch.float32, device="cuda")
        got = distributed_advantages(D, plan, gamma, r, m, Gd, Ad)
        torch.cuda.synchronize()
        assert got[0].item() == stats[0]
        gmax = max(np.abs(G[k]).max() if G[k].size else 0 for k in G)
        atol = 4 * 2.0 ** -24 * max(lens) * gmax + 1e-6
        sigma = np.sqrt(max(stats[2] / stats[0] - (stats[1] / stats[0]) ** 2, 0))
        assert np.allclose(Gd[:n].cpu().numpy(), G[rank], rtol=0, atol=atol)
        assert np.allclose(Ad[:n].cpu().numpy(), A[rank], rtol=0, atol=atol / sigma + 1e-5)
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_roles_main(rank, world, port, q, case):
    """Per-role routing (SPEC route_noncritical_tensors) with one process per rank: token and
    per-sequence tensors, all-to-all or gathered to the controller, buffers side by side in one
    IPC window -- byte-exact against the oracle."""
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200.dispatch import Dispatcher, controller_layout, plan_roles, route_roles
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, dst, flag, ctrl = case
        tensors = [("ids", "tokens", ("ids", 4, 1, "x"), "token"),
                   ("lp", "log_probs", ("lp", 4, 1, "x"), "token"),
                   ("G", "returns", ("G", 4, 1, "x"), "token"),
                   ("R", "rewards", ("R", 4, 1, "x"), "sequence")]
        routes = route_roles({t[0]: t[1] for t in tensors}, flag)
        T, N = sum(lens), len(lens)
        gs = O.assign_groups(src, lens)
        hs = O.seq_holdings(src, lens, gs)
        send, want = {}, {}
        for k, t in enumerate(tensors):
            nm = t[0]
            lay_d = dst if routes[nm] == "all_to_all" else controller_layout(ctrl)
            if t[3] == "token":
                glob = np.random.default_rng(50 + k).integers(0, 256, T * 4, dtype=np.uint8)
                arrs = O.rank_arrays_from_global(src, lens, gs, [glob], [("f", 4, 1, "x")])
                w, _, _ = O.dispatch(src, lay_d, lens, arrs, [("f", 4, 1, "x")], world)
            else:
                glob = np.random.default_rng(50 + k).integers(0, 256, N * 4, dtype=np.uint8)
                arrs = {r: [np.concatenate([glob[4 * i:4 * i + 4] for i in m]) if m
                            else np.zeros(0, np.uint8)] for r, m in hs.items()}
                w = O.dispatch_seq_fields(src, lay_d, lens, arrs, [t[2]], world)
            a = arrs.get(rank, [np.zeros(0, np.uint8)])[0]
            send[nm] = [torch.from_numpy(a).cuda() if a.size else None]
            want[nm] = w
        D = Dispatcher(window_bytes=8 * (T + N) * 4 + (1 << 20), device=0)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        rp = plan_roles(D, src, dst, glens, tensors, distributed_aggregation=flag, controller=ctrl)
        recv, views = rp.alloc_recv(D)
        for nm in views:
            views[nm][0].fill_(0xA5)
        rp.exec(send, recv)
        torch.cuda.synchronize()
        for nm, w in want.items():
            got = views[nm][0].cpu().numpy()
            if rank in w:
                assert np.array_equal(got[: w[rank][0].size], w[rank][0]), (nm, rank)
            else:
                assert got.size == 0, (nm, rank, "received bytes it should not")
        rp.destroy()
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_timeout_main(rank, world, port, q, case):
    """Failure detection: every rank but the last calls the fused exec; the last
    never does.  The others' entry barrier times out (EARL_TIMEOUT_MS) and the plan reports
    EARL_ERR_TIMEOUT naming the missing peer."""
    try:
        import os
        os.environ["EARL_TIMEOUT_MS"] = "300"
        import numpy as np
        import torch
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        import torch.distributed as dist
        lens = case
        fields = W.field_set("tiny3")
        src = W.rollout_layout(len(lens), world)
        dst = W.layout(dp=1, tp=world, assign="contig")
        D = Dispatcher(window_bytes=sum(lens) * W.bytes_per_token(fields) + (1 << 16), device=0)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        plan = D.plan(src, dst, glens, fields)
        ptrs, views = D.alloc_recv(plan, fields)
        tok = W.rollout_token_counts(np.asarray(lens), src["counts"])[rank]
        mine = [torch.zeros(max(16, tok * b), dtype=torch.uint8, device="cuda") for b in (4, 4, 4)]
        missing = world - 1
        msg = "ok"
        if rank != missing:
            plan.exec(mine, ptrs)
            try:
                plan.sync()
                msg = f"rank {rank}: no timeout reported"
            except EarlError as e:
                want = f"mask 0x{1 << missing:x}"
                if "TIMEOUT" not in str(e) or want not in str(e):
                    msg = f"rank {rank}: unexpected error {e}"
        dist.barrier()  # the missing rank keeps its window mapped until the others are done
        dist.destroy_process_group()
        q.put((rank, msg))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_hash_main(rank, world, port, q, case):
    """Replicated planning across processes: equal plans pass Dispatcher.check_plan; when one
    rank plans from different lengths, every rank gets EARL_ERR_MISMATCH."""
    try:
        import numpy as np
        import torch
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        import torch.distributed as dist
        lens = list(case)
        fields = W.field_set("tiny3")
        src, dst = W.config_layouts("c3", world, len(lens))
        D = Dispatcher(window_bytes=1 << 20, device=0)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        plan = D.plan(src, dst, glens, fields)
        D.check_plan(plan)
        bad = list(lens)
        if rank == world - 1:
            bad[0] += 3
        plan2 = D.plan(src, dst, torch.as_tensor(np.asarray(bad, dtype=np.int32)).cuda(), fields)
        msg = f"rank {rank}: mismatch not detected"
        try:
            D.check_plan(plan2)
        except EarlError as e:
            if "MISMATCH" in str(e) or "differs" in str(e):
                msg = "ok"
            else:
                msg = f"rank {rank}: {e}"
        plan.destroy()
        plan2.destroy()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, msg))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_null_recv_main(rank, world, port, q, case):
    """Source-only ranks pass NULL receive buffers (earl_dispatch.h: a rank that receives nothing
    may), and ranks place their receive buffers at rank-specific window offsets: every
    destination still gets every byte the oracle gives it (the senders use the offsets each
    destination published, not their own)."""
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher, field_bytes
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, dst, fields = case
        T = sum(lens)
        glob = W.gen_global_fields(fields, T, seed_base=91, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
        D = Dispatcher(window_bytes=T * W.bytes_per_token(fields) + (1 << 20), device=0)
        mine = [torch.from_numpy(a).cuda() if a.size else None for a in src_arrays.get(rank, [])] \
            if rank in src_arrays else [None] * len(fields)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        for it in range(3):
            plan = D.plan(src, dst, glens, fields)
            st = plan.stats()
            D.comm.reset_alloc()
            D.comm.alloc(256 * (1 + rank + it))   # rank- and iteration-specific offsets
            ptrs, views = [], []
            n_mine = int(st["n_local_tokens"][rank])
            for b in field_bytes(fields):
                if rank in want and n_mine:
                    ptr = D.comm.alloc(n_mine * b)
                    from paper_2510_05943_b200.dispatch import window_tensor
                    v = window_tensor(ptr, n_mine * b, D.device)
                    v.fill_(0xA5)
                    ptrs.append(ptr)
                    views.append(v)
                else:
                    ptrs.append(None)   # receives nothing: NULL
                    views.append(None)
            torch.cuda.synchronize()
            plan.exec(mine, ptrs)
            torch.cuda.synchronize()
            plan.sync()
            if rank in want:
                for f in range(len(fields)):
                    got = views[f].cpu().numpy() if views[f] is not None else np.zeros(0, np.uint8)
                    assert np.array_equal(got, want[rank][f]), f"iter {it} rank {rank} field {f}"
            plan.destroy()
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_late_peer_main(rank, world, port, q, case):
    """A peer that arrives after the others' entry barrier timed out: the others skip their
    copies and say so in their done flags; the late rank passes its own barrier (the others'
    ready flags are there), copies, and then reports TIMEOUT naming the ranks whose copies were
    skipped -- instead of returning with their contribution missing."""
    try:
        import os
        import time
        os.environ["EARL_TIMEOUT_MS"] = "400"
        import numpy as np
        import torch
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        import torch.distributed as dist
        lens = case
        fields = W.field_set("tiny3")
        src = W.rollout_layout(len(lens), world)
        dst = W.layout(dp=1, tp=world, assign="contig")
        D = Dispatcher(window_bytes=sum(lens) * W.bytes_per_token(fields) + (1 << 16), device=0)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        plan = D.plan(src, dst, glens, fields)
        ptrs, views = D.alloc_recv(plan, fields)
        tok = W.rollout_token_counts(np.asarray(lens), src["counts"])[rank]
        mine = [torch.zeros(max(16, tok * b), dtype=torch.uint8, device="cuda") for b in (4, 4, 4)]
        late = world - 1
        torch.cuda.synchronize()
        dist.barrier()
        if rank == late:
            time.sleep(1.5)   # the others' entry barriers (400 ms) and done waits expire first
        plan.exec(mine, ptrs)
        msg = "ok"
        try:
            plan.sync()
            msg = f"rank {rank}: no error reported"
        except EarlError as e:
            others = sum(1 << r for r in range(world) if r != late)
            if rank == late:
                want = f"skipped their copies (mask 0x{others:x})"
            else:
                want = f"mask 0x{1 << late:x}"
            if "TIMEOUT" not in str(e) or want not in str(e):
                msg = f"rank {rank}: unexpected error {e}"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, msg))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_nccl_main(rank, world, port, q, case):
    """K8 through the library: pack -> grouped ncclSend / ncclRecv (earl_dispatch_exchange) ->
    unpack, against the oracle.  One GPU hosts one NCCL rank only, so this runs at world 1 (the
    message to itself goes through NCCL too); multi-rank message tables are covered by the
    gloo-staged multi-process tests."""
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, fields = case
        src = W.rollout_layout(len(lens), 1)
        dst = W.layout(dp=1, assign="contig")
        T = sum(lens)
        glob = W.gen_global_fields(fields, T, seed_base=13, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
        D = Dispatcher(window_bytes=1 << 16, device=0)
        D.init_nccl()
        mine = [torch.from_numpy(a).cuda() for a in src_arrays[0]]
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        plan = D.plan(src, dst, glens, fields)
        st = plan.stats()
        recv = [torch.full((int(st["n_local_tokens"][0]) * b,), 0xA5, dtype=torch.uint8, device="cuda")
                for b in [x[1] * x[2] for x in fields]]
        for it in range(3):
            D.exec_staged(plan, mine, recv)     # library path: earl_dispatch_exec_staged
            torch.cuda.synchronize()
            plan.sync()
            for f in range(len(fields)):
                assert np.array_equal(recv[f].cpu().numpy(), want[0][f]), (it, f)
            for x in recv:
                x.fill_(0)
        # the exchange call on its own, with caller-owned stage buffers
        send_stage, recv_stage, msgs = D.alloc_stage(plan)
        plan.pack(mine, [send_stage])
        plan.exchange(send_stage, recv_stage)
        plan.unpack([recv_stage], recv)
        torch.cuda.synchronize()
        for f in range(len(fields)):
            assert np.array_equal(recv[f].cpu().numpy(), want[0][f]), ("exchange", f)
        plan.destroy()
        import torch.distributed as dist
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_nvls_main(rank, world, port, q, case):
    """NEXT-3 plumbing with EARL_NVLS=1: cuMemCreate windows exported by file descriptor
    (pidfd_getfd) instead of CUDA IPC, fused exec bit-exact against the oracle, then the
    multicast teams of the destination's TP groups -- created and used when the device can (a
    multi-GPU NVSwitch box), EARL_ERR_UNSUPPORTED on every rank when it cannot (one visible GPU),
    after which the unicast exec still matches the oracle."""
    try:
        import os
        os.environ["EARL_NVLS"] = "1"
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, dst, fields = case
        T = sum(lens)
        glob = W.gen_global_fields(fields, T, seed_base=31, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
        D = Dispatcher(window_bytes=T * W.bytes_per_token(fields) + (1 << 20), device=0)
        assert all(D.comm.peer_mapped(p) for p in range(world) if p != rank)
        mine = [torch.from_numpy(a).cuda() if a.size else None for a in src_arrays.get(rank, [])] \
            if rank in src_arrays else [None] * len(fields)
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()

        def run(tag):
            plan = D.plan(src, dst, glens, fields)
            ptrs, views = D.alloc_recv(plan, fields)
            for v in views:
                v.fill_(0xA5)
            plan.exec(mine, ptrs)
            torch.cuda.synchronize()
            plan.sync()
            if rank in want:
                for f in range(len(fields)):
                    assert np.array_equal(views[f].cpu().numpy(), want[rank][f]), (tag, rank, f)
            plan.destroy()

        run("vmm windows")
        msg = "ok"
        try:
            masks = D.enable_multicast(dst)
            run("multicast")
            msg = f"ok (multicast teams {masks})"
        except EarlError as e:
            if e.name != "EARL_ERR_UNSUPPORTED":
                raise
            run("unicast after UNSUPPORTED")
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok" if msg.startswith("ok") else msg))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_hier_main(rank, world, port, q, case):
    """NEXT-4 with virtual nodes on one GPU: node_size consecutive processes form a 'node'
    (CUDA-IPC windows mapped inside it only); exec_hier = the fused P2P exec inside the node +
    the node-to-node messages (pack of the shards with a replica on another node, exchange over
    the process group -- NCCL between real nodes, gloo here -- unpack of the other nodes'
    messages).  Every destination byte equals the oracle's; the device length gather refuses
    a multi-node comm."""
    try:
        import numpy as np
        import torch
        from oracle import earl_oracle as O
        from paper_2510_05943_b200 import workloads as W
        from paper_2510_05943_b200.dispatch import Dispatcher, rank_counts
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        lens, src, dst, fields, node_size = case
        T = sum(lens)
        glob = W.gen_global_fields(fields, T, seed_base=57, random_bits=True)
        src_arrays = O.rank_arrays_from_global(src, lens, O.assign_groups(src, lens), glob, fields)
        want, _, _ = O.dispatch(src, dst, lens, src_arrays, fields, world)
        D = Dispatcher(window_bytes=T * W.bytes_per_token(fields) + (1 << 20), device=0,
                       node_size=node_size)
        node = rank // node_size
        for p in range(world):
            if p != rank:
                assert D.comm.peer_mapped(p) == (p // node_size == node), (rank, p)
        mine = [torch.from_numpy(a).cuda() if a.size else None for a in src_arrays.get(rank, [])] \
            if rank in src_arrays else [None] * len(fields)
        if src.get("assign") == "given_counts":
            cnts = rank_counts(src, world)
            edges = np.concatenate([[0], np.cumsum(cnts)]).astype(int)
            local = torch.as_tensor(np.asarray(lens[edges[rank]:edges[rank + 1]], dtype=np.int32)).cuda()
            try:
                D.allgather_lens(local, counts=cnts)
                raise AssertionError("device gather accepted a multi-node comm")
            except EarlError as e:
                assert e.name == "EARL_ERR_UNSUPPORTED", e
            glens, _ = D.allgather_lens(local)  # the process-group path
        else:
            glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        assert glens.cpu().tolist() == list(lens)
        for it in range(2):
            plan = D.plan(src, dst, glens, fields)
            ptrs, views = D.alloc_recv(plan, fields)
            for v in views:
                v.fill_(0xA5)
            torch.cuda.synchronize()
            D.exec_hier(plan, mine, ptrs)
            torch.cuda.synchronize()
            plan.sync()
            if rank in want:
                for f in range(len(fields)):
                    got = views[f].cpu().numpy()
                    assert np.array_equal(got, want[rank][f]), f"iter {it} rank {rank} field {f}"
            plan.destroy()
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


def gpu_gather_timeout_main(rank, world, port, q, case):
    """a1's failure detection: the last rank never joins the device length gather; the others'
    gather kernel times out (EARL_TIMEOUT_MS) and earl_comm_check reports EARL_ERR_TIMEOUT with
    the missing rank's bit."""
    try:
        import os
        os.environ["EARL_TIMEOUT_MS"] = "300"
        import numpy as np
        import torch
        from paper_2510_05943_b200.dispatch import Dispatcher
        from paper_2510_05943_b200.earl import EarlError
        torch.cuda.set_device(0)
        init(rank, world, port, "gloo")
        import torch.distributed as dist
        counts = [5] * world
        D = Dispatcher(window_bytes=1 << 20, device=0)
        local = torch.arange(5, dtype=torch.int32, device="cuda") + 10 * rank
        missing = world - 1
        msg = "ok"
        if rank != missing:
            D.allgather_lens(local, counts=counts)
            try:
                D.comm.check()
                msg = f"rank {rank}: no timeout reported"
            except EarlError as e:
                if e.name != "EARL_ERR_TIMEOUT" or f"mask 0x{1 << missing:x}" not in str(e):
                    msg = f"rank {rank}: unexpected error {e}"
            D.comm.check()  # the latch was cleared by the report
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, msg))
    except Exception:
        q.put((rank, traceback.format_exc()))
