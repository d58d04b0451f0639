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
        glens = torch.as_tensor(np.asarray(lens, dtype=np.int32)).cuda()
        for it in range(n_exec):
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
