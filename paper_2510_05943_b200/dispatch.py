"""User-facing dispatch helpers over the C ABI (torch tensors in, torch tensors out).

* ``EmulatedDispatch`` -- one process holds every rank on one GPU (the 1-GPU measurement and
  test mode of SURVEY.md §8(d)); one launch serves all ranks.
* ``Dispatcher`` -- one process per GPU under torch.distributed: bootstraps the comm (CUDA-IPC
  window handles are all-gathered over the process group), all-gathers the local lengths
  (step a1; plumbing over the process group), plans on the device and runs the fused P2P
  exchange into symmetric receive windows.

Every byte of the dispatch moves in libearl_dispatch.so's kernels; this module only allocates
tensors and passes pointers.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import earl
from .earl import EARL_ALL_RANKS, Comm


def field_bytes(fields):
    return [int(f[1]) * int(f[2]) for f in fields]


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (lets torch alias the comm window)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
            "version": 3, "strides": None,
        }


def window_tensor(ptr: int, nbytes: int, device) -> torch.Tensor:
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CudaArray(ptr, nbytes), device=device)


def layout_for_device(lay: dict, device) -> dict:
    """Copy EXPLICIT group_of_seq to the device (the C ABI takes a device pointer)."""
    out = dict(lay)
    gos = lay.get("group_of_seq")
    if lay.get("assign") == "explicit" and gos is not None:
        t = torch.as_tensor(np.asarray(gos, dtype=np.int32)).to(device)
        out["group_of_seq_dev"] = t
    return out


class EmulatedDispatch:
    """All `world` ranks in this process on one device."""

    def __init__(self, world: int, device: int = 0, window_bytes: int = 0):
        self.world = int(world)
        self.device = torch.device("cuda", device)
        self.comm = Comm(EARL_ALL_RANKS, self.world, device, window_bytes)

    def plan(self, src, dst, seq_lens, fields, stream=None):
        lens = torch.as_tensor(np.asarray(seq_lens, dtype=np.int32)).to(self.device) \
            if not isinstance(seq_lens, torch.Tensor) else seq_lens
        self._src = layout_for_device(src, self.device)
        self._dst = layout_for_device(dst, self.device)
        return self.comm.plan(self._src, self._dst, lens, fields, stream)

    def allgather_lens(self, local_lens, counts, out=None, stream=None):
        """Step a1 on the emulated comm: local_lens[r] = rank r's lengths (None where counts[r]
        is 0), concatenated rank-major on the device into `out` (earl_allgather_lengths)."""
        total = int(sum(counts))
        if out is None:
            out = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
        self.comm.allgather_lengths(counts, local_lens, out, stream)
        return out[:total]

    def alloc_recv(self, plan, fields):
        """Per-rank, per-field uint8 receive tensors sized from the plan (host sync)."""
        st = plan.stats()
        Bf = field_bytes(fields)
        return [[torch.empty(int(st["n_local_tokens"][r]) * b, dtype=torch.uint8, device=self.device)
                 for b in Bf] for r in range(self.world)]

    def alloc_stage(self, plan):
        st = plan.stats()
        return [torch.empty(max(16, int(st["stage_bytes"][r])), dtype=torch.uint8, device=self.device)
                for r in range(self.world)]

    @staticmethod
    def flat(per_rank):
        return [t for row in per_rank for t in row]

    def meta(self, plan, rank):
        ns, nt = plan.local_sizes(rank)
        cu = torch.empty(ns + 1, dtype=torch.int32, device=self.device)
        ids = torch.empty(max(ns, 1), dtype=torch.int64, device=self.device)
        ts = torch.empty(max(ns, 1), dtype=torch.int32, device=self.device)
        plan.local_meta(rank, cu, ids, ts)
        return cu, ids[:ns], ts[:ns]


def allgather_lengths(local_lens: torch.Tensor, group=None):
    """Step a1: every rank learns the global int32 length vector in rank
    order -- first the per-rank counts (int64), then the lengths padded to the largest count.
    Works on any torch.distributed backend (tensors stay on local_lens.device).
    Returns (global int32 tensor, per-rank counts)."""
    import torch.distributed as dist
    dev = local_lens.device
    world = dist.get_world_size(group)
    n = torch.tensor([local_lens.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts) if counts else 0
    pad = torch.zeros(max(m, 1), dtype=torch.int32, device=dev)
    pad[: local_lens.numel()] = local_lens.to(torch.int32)
    allp = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(allp, pad, group=group)
    if m == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev), counts
    return torch.cat([allp[r][: counts[r]] for r in range(world)]), counts


def rank_counts(src: dict, world: int):
    """Per-rank sequence counts of a rollout (GIVEN_COUNTS) source layout, in the rank-major
    global order of step a1: rank (g, 0, 0) contributes group g's counts[g] lengths, every other
    rank (SP chunks, TP replicas, ranks outside the layout) none."""
    if src.get("assign") != "given_counts":
        raise ValueError("the device length gather needs a GIVEN_COUNTS source layout")
    out = [0] * int(world)
    sp, tp, r0 = int(src.get("sp", 1)), int(src.get("tp", 1)), int(src.get("rank0", 0))
    for g, c in enumerate(src["counts"]):
        out[r0 + g * sp * tp] = int(c)
    return out


def max_over_ranks(values, group=None):
    """Element-wise max of a list of floats over the ranks (timing: the slowest rank decides)."""
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.tolist()]


class Dispatcher:
    """One process per GPU (torch.distributed initialised).  Fused P2P exchange."""

    def __init__(self, window_bytes: int, device=None, group=None, node_size=None):
        """node_size (NEXT-4): ranks per node when the group spans nodes; only same-node
        windows are mapped, exec moves the node-local records, exec_hier adds the rest."""
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.comm = Comm(self.rank, self.world, self.device.index, window_bytes)
        self.node_size = node_size if node_size and node_size < self.world else None
        if self.node_size:
            self.comm.set_nodes(self.node_size)
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, self.comm.export_handle(), group=group)
            self.comm.import_peers(handles)

    def allgather_lens(self, local_lens: torch.Tensor, counts=None, out=None, stream=None):
        """Step a1.  With `counts` (per-rank sequence counts, the same on every rank: see
        rank_counts) the library gathers on the device (earl_allgather_lengths: one kernel over
        the peer windows, no host synchronisation, graph-capturable) and returns (out, counts).
        Without, the counts are not known in advance: two all-gathers over the process group
        (see allgather_lengths; gloo groups run it on host tensors)."""
        if counts is not None:
            total = int(sum(counts))
            if out is None:
                out = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
            loc = local_lens if local_lens is not None and local_lens.numel() else None
            self.comm.allgather_lengths(counts, [loc], out, stream)
            return out[:total], list(counts)
        backend = self.dist.get_backend(self.group)
        dev = self.device if backend == "nccl" else torch.device("cpu")
        glob, counts = allgather_lengths(local_lens.to(dev), self.group)
        return glob.to(self.device), counts

    def plan(self, src, dst, seq_lens: torch.Tensor, fields, stream=None):
        self._src = layout_for_device(src, self.device)
        self._dst = layout_for_device(dst, self.device)
        plan = self.comm.plan(self._src, self._dst, seq_lens, fields, stream)
        if os.environ.get("EARL_CHECK_PLAN") == "1":
            self.check_plan(plan)
        return plan

    def check_plan(self, plan):
        """Debug check of replicated planning: every rank's plan hash, all-gathered
        over the process group, must be equal; otherwise EARL_ERR_MISMATCH naming the ranks."""
        mine = plan.hash()
        hashes = [None] * self.world
        self.dist.all_gather_object(hashes, mine, group=self.group)
        if len(set(hashes)) != 1:
            bad = [r for r, h in enumerate(hashes) if h != hashes[0]]
            raise earl.EarlError(7, f"plan hash differs across ranks: rank 0 {hashes[0]:#x}, "
                                    f"ranks {bad} differ")
        return mine

    def alloc_recv(self, plan, fields, reset=True):
        """Receive tensors inside the symmetric window: same offsets on every rank, sized for
        the largest destination rank (every rank knows every size: the plan is replicated).
        reset=False keeps earlier allocations (several plans' buffers side by side)."""
        st = plan.stats()
        if reset:
            self.comm.reset_alloc()
        full, views = [], []
        n_max = max(st["n_local_tokens"]) if st["n_local_tokens"] else 0
        mine = int(st["n_local_tokens"][self.rank])
        for b in field_bytes(fields):
            ptr = self.comm.alloc(max(16, n_max * b))
            full.append(ptr)
            views.append(window_tensor(ptr, max(16, n_max * b), self.device)[: mine * b])
        # exec takes the raw window pointers (valid even when this rank receives 0 bytes)
        return full, views

    # -- staged path (pack -> grouped send/recv -> unpack): the exchange comparator ----------

    def alloc_stage(self, plan):
        """Send stage (this rank's packed messages) and receive stage (the messages it gets,
        concatenated in source-rank order), plus the per-peer byte table of earl_plan_messages."""
        st = plan.stats()
        msgs = plan.messages(self.rank)
        send_stage = torch.empty(max(16, int(st["stage_bytes"][self.rank])), dtype=torch.uint8,
                                 device=self.device)
        recv_stage = torch.empty(max(16, int(sum(msgs[3]))), dtype=torch.uint8, device=self.device)
        return send_stage, recv_stage, msgs

    def exchange(self, send_stage, recv_stage, msgs):
        """Step a4 of the staged path: every per-peer message as one grouped send/recv
        (torch.distributed.batch_isend_irecv == ncclGroupStart / ncclSend / ncclRecv /
        ncclGroupEnd on an NCCL group; host-staged on a gloo group, for tests).  The message to
        itself is a device-local copy."""
        dist = self.dist
        so, sb, ro, rb = msgs
        me = self.rank
        if sb[me]:
            recv_stage[ro[me]:ro[me] + rb[me]].copy_(send_stage[so[me]:so[me] + sb[me]])
        gloo = dist.get_backend(self.group) != "nccl"
        host_recv = {}
        ops = []
        for p in range(self.world):
            if p == me:
                continue
            if sb[p]:
                buf = send_stage[so[p]:so[p] + sb[p]]
                ops.append(dist.P2POp(dist.isend, buf.cpu() if gloo else buf, p, self.group))
            if rb[p]:
                buf = recv_stage[ro[p]:ro[p] + rb[p]]
                if gloo:
                    host_recv[p] = torch.empty(rb[p], dtype=torch.uint8)
                    buf = host_recv[p]
                ops.append(dist.P2POp(dist.irecv, buf, p, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for p, hbuf in host_recv.items():
            recv_stage[ro[p]:ro[p] + rb[p]].copy_(hbuf)

    def enable_multicast(self, dst):
        """NEXT-3: one NVLS multicast team per TP group of layout `dst` (needs EARL_NVLS=1 when
        the comm was made).  The team's lowest rank creates it, the process group carries the
        handle, every rank joins (members bind their window).  Raises EarlError (UNSUPPORTED)
        on every rank when the device cannot create a team.  Returns the team masks."""
        r0, dp, sp, tp = (int(dst.get(k, d)) for k, d in (("rank0", 0), ("dp", 1), ("sp", 1), ("tp", 1)))
        masks = []
        if tp < 2:
            return masks
        for ds in range(dp * sp):
            ranks = [r0 + ds * tp + t for t in range(tp)]
            mask = sum(1 << r for r in ranks)
            made = None
            if self.rank == ranks[0]:
                try:
                    made = (self.comm.mc_create(mask), None)
                except earl.EarlError as e:
                    made = (None, (e.status, str(e)))
            objs = [None] * self.world
            self.dist.all_gather_object(objs, made, group=self.group)
            handle, err = objs[ranks[0]]
            if err is not None:
                raise earl.EarlError(err[0], err[1])
            self.comm.mc_join(mask, handle)
            masks.append(mask)
        return masks

    def exec_hier(self, plan, send_bufs, recv_bufs, stream=None):
        """NEXT-4: the fused P2P exec inside this rank's node, then the messages between nodes
        (the library's NCCL exchange after init_nccl, else over the process group -- gloo in the
        one-GPU tests, where 'nodes' are groups of processes)."""
        if getattr(self, "_nccl", False):
            plan.exec_hier(send_bufs, recv_bufs, stream)
            return
        plan.exec(send_bufs, recv_bufs, stream)
        self.exec_staged(plan, send_bufs, recv_bufs, stream=stream)

    def init_nccl(self):
        """K8: the library's own NCCL communicator over this group's ranks (rank 0 draws the
        unique id, the process group broadcasts it).  Needs one GPU per rank (NCCL rejects two
        ranks on one device)."""
        if getattr(self, "_nccl", False):
            return
        obj = [earl.nccl_unique_id() if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        self.comm.init_nccl(obj[0])
        self._nccl = True

    def exec_staged(self, plan, send_bufs, recv_bufs, send_stage=None, recv_stage=None, msgs=None,
                    stream=None):
        """pack (this rank's records) -> grouped send/recv -> unpack (this rank's arrays).

        Without an explicit `msgs` the per-peer byte table is read from the plan on every call
        -- a device->host synchronisation that the NCCL path inherently needs (its sizes are
        host arguments), unlike the fused exec.  Stage buffers grow on demand and are cached.

        After init_nccl() the whole staged path runs in the library (earl_dispatch_exec_staged:
        pack, grouped ncclSend / ncclRecv, unpack); otherwise the exchange goes through the
        process group (gloo in the one-GPU tests: host-staged)."""
        if getattr(self, "_nccl", False) and send_stage is None and recv_stage is None:
            plan.exec_staged(send_bufs, recv_bufs, stream)
            return
        if msgs is None:
            msgs = plan.messages(self.rank)
        if send_stage is None or recv_stage is None:
            st_bytes = int(plan.stats()["stage_bytes"][self.rank])
            need_s, need_r = max(16, st_bytes), max(16, int(sum(msgs[3])))
            cache = getattr(self, "_stage_cache", None)
            if cache is None or cache[0].numel() < need_s or cache[1].numel() < need_r:
                cache = (torch.empty(need_s, dtype=torch.uint8, device=self.device),
                         torch.empty(need_r, dtype=torch.uint8, device=self.device))
                self._stage_cache = cache
            send_stage, recv_stage = cache
        plan.pack(send_bufs, [send_stage], stream)
        self.exchange(send_stage, recv_stage, msgs)
        plan.unpack([recv_stage], recv_bufs, stream)


# ---------------------------------------------------------------------------------------
# per-sequence fields (reading n4)
# ---------------------------------------------------------------------------------------

def plan_seq_fields(comm, token_plan, src, dst, sfields, device, stream=None):
    """Plan the routing of per-sequence fields along `token_plan` (reading n4): the library's
    earl_plan_seq_fields (unit lengths over the token plan's layouts with SP folded into TP and
    its groups pinned as EXPLICIT, built on the device).  comm / src / dst / device are accepted
    for call-site compatibility; the token plan carries them."""
    from .earl import Plan
    return Plan.seq_fields(token_plan, sfields, stream)


def distributed_advantages(dispatcher, plan, gamma, rewards, mask, returns, adv, eps=1e-8,
                           seq_return=None, stream=None):
    """NEXT-2 (reading n5) on one process per GPU: discounted returns where the rollout holds
    the tokens, a 3-double all-reduce of the masked-token statistics (no controller gathers any
    reward), then the normalised advantages.  rewards fp32 / mask u8 / returns, adv fp32 are this
    rank's token tensors; returns the reduced statistics (sum m, sum m G, sum m G^2)."""
    dist = dispatcher.dist
    partial = torch.zeros(3, dtype=torch.float64, device=dispatcher.device)
    plan.returns(gamma, [rewards], [mask], [returns], partial,
                 seq_return=[seq_return] if seq_return is not None else None, stream=stream)
    if dist.get_backend(dispatcher.group) == "nccl":
        dist.all_reduce(partial, group=dispatcher.group)
    else:
        host = partial.cpu()
        dist.all_reduce(host, group=dispatcher.group)
        partial.copy_(host)
    plan.advantages(partial, eps, [returns], [mask], [adv], stream=stream)
    return partial


# ---------------------------------------------------------------------------------------
# per-role routing (NEXT-2; "route_noncritical_tensors", §3.3 + §5)
# ---------------------------------------------------------------------------------------

# role -> route.  Tensors the trainer consumes token by token go all-to-all (§3.3: log
# probabilities are "not required for aggregation in advantage estimation"); rewards and returns
# are gathered to the controller by default (§5 "rewards and returns are aggregated"), or
# dispatched like the rest when the aggregation itself is distributed (§5's extension, built as
# earl_returns / earl_advantages: DESIGN.md reading n5).
ROLE_ROUTES = {
    "tokens": "all_to_all", "log_probs": "all_to_all", "ref_log_probs": "all_to_all",
    "values": "all_to_all", "advantages": "all_to_all", "response_mask": "all_to_all",
    "hidden": "all_to_all", "rewards": "gather", "returns": "gather",
}


def route_roles(roles: dict, distributed_aggregation: bool = False) -> dict:
    """{tensor name: role} -> {tensor name: "all_to_all" | "gather"}; an unknown role is a
    configuration error (ValueError)."""
    out = {}
    for name, role in roles.items():
        if role not in ROLE_ROUTES:
            raise ValueError(f"unknown role {role!r} for tensor {name!r} "
                             f"(known: {', '.join(sorted(ROLE_ROUTES))})")
        route = ROLE_ROUTES[role]
        out[name] = "all_to_all" if (route == "gather" and distributed_aggregation) else route
    return out


def controller_layout(controller: int = 0) -> dict:
    """The gather destination: one DP group held by the controller rank alone."""
    return {"rank0": int(controller), "dp": 1, "sp": 1, "tp": 1, "assign": "contig",
            "sp_split": "block", "sp_min_len": 0, "counts": None, "group_of_seq": None}


class RolePlans:
    """The plan set of one batch: one dispatch plan per (route, granularity) with the fields of
    the tensors routed that way.  groups[(route, per)] = (plan, names, fields), per = "token" or
    "sequence"; a route with only per-sequence tensors still plans its token routing once (the
    sequence records follow the token plan's groups)."""

    def __init__(self, local_ranks: int):
        self.local_ranks = int(local_ranks)
        self.groups = {}
        self._token_plans = []

    def dst_layout(self, route, dst, controller):
        return dst if route == "all_to_all" else controller_layout(controller)

    def alloc_recv(self, disp):
        """Receive buffers of every group: (recv, views), both tensor name -> list over this
        process's ranks.  recv feeds exec (window pointers for a Dispatcher: all groups share the
        window, allocated side by side); views are this rank's received bytes."""
        recv, views = {}, {}
        first = True
        for plan, names, fields in self.groups.values():
            if isinstance(disp, EmulatedDispatch):
                per_rank = disp.alloc_recv(plan, fields)
                for f, nm in enumerate(names):
                    recv[nm] = [per_rank[r][f] for r in range(self.local_ranks)]
                    views[nm] = recv[nm]
            else:
                ptrs, vs = disp.alloc_recv(plan, fields, reset=first)
                for f, nm in enumerate(names):
                    recv[nm], views[nm] = [ptrs[f]], [vs[f]]
            first = False
        return recv, views

    def exec(self, send: dict, recv: dict, stream=None):
        """send / recv: tensor name -> list over this process's ranks (emulated: every rank;
        one process per GPU: one entry) of device buffers (None where a rank holds nothing)."""
        for (route, per), (plan, names, _) in self.groups.items():
            s = [send[nm][r] for r in range(self.local_ranks) for nm in names]
            d = [recv[nm][r] for r in range(self.local_ranks) for nm in names]
            plan.exec(s, d, stream)

    def destroy(self):
        for plan, _, _ in self.groups.values():
            plan.destroy()
        for p in self._token_plans:
            p.destroy()
        self.groups = {}
        self._token_plans = []


def plan_roles(disp, src, dst, seq_lens, tensors, distributed_aggregation=False, controller=0,
               stream=None):
    """SPEC route_noncritical_tensors: plan every tensor of the batch by its role.

    disp: EmulatedDispatch or Dispatcher; tensors: [(name, role, field, per)], field = (name,
    bytes per element, elements per token or sequence, kind), per = "token" | "sequence".
    Returns RolePlans (empty for an empty tensor list)."""
    routes = route_roles({t[0]: t[1] for t in tensors}, distributed_aggregation)
    local = disp.world if isinstance(disp, EmulatedDispatch) else 1
    rp = RolePlans(local)
    if not tensors:
        return rp
    lens = seq_lens
    if not isinstance(lens, torch.Tensor):
        lens = torch.as_tensor(np.asarray(seq_lens, dtype=np.int32))
    lens = lens.to(disp.device)
    src_dev = layout_for_device(src, disp.device)
    for route in ("all_to_all", "gather"):
        dst_r = rp.dst_layout(route, dst, controller)
        tok = [t for t in tensors if routes[t[0]] == route and t[3] == "token"]
        seq = [t for t in tensors if routes[t[0]] == route and t[3] == "sequence"]
        for t in tok + seq:
            if t[3] not in ("token", "sequence"):
                raise ValueError(f"tensor {t[0]!r}: per must be 'token' or 'sequence'")
        token_plan = None
        if tok:
            token_plan = disp.comm.plan(src_dev, layout_for_device(dst_r, disp.device), lens,
                                        [t[2] for t in tok], stream)
            rp.groups[(route, "token")] = (token_plan, [t[0] for t in tok], [t[2] for t in tok])
        if seq:
            if token_plan is None:  # routing only: the sequences' groups
                token_plan = disp.comm.plan(src_dev, layout_for_device(dst_r, disp.device), lens,
                                            [("unit", 1, 1, "x")], stream)
                rp._token_plans.append(token_plan)
            sp = plan_seq_fields(disp.comm, token_plan, src_dev,
                                 layout_for_device(dst_r, disp.device), [t[2] for t in seq],
                                 disp.device, stream)
            rp.groups[(route, "sequence")] = (sp, [t[0] for t in seq], [t[2] for t in seq])
    return rp


def next_layout(policy, plan, current: int, layouts):
    """The selector's step before the next rollout: observe the averaged
    context length of the batch just planned (T / N, reading s4), look it up in the policy
    (earl_policy_select, hysteresis s3) -> (configuration index, its layout, switched)."""
    nxt, switched = policy.select(plan.mean_length(), current)
    return nxt, layouts[nxt], switched
