"""Thin Python binding of libearl_dispatch.so (include/earl_dispatch.h).

Argument marshalling only: every step of the dispatch (planning, packing, the exchange,
unpacking) runs in the CUDA library.  Torch is used for device memory and streams: tensors are
passed as raw device pointers.  There is no CPU fallback -- if the library is missing this
module raises on import of the library (``lib()``), loudly.

The function names mirror the C ABI (earl_comm_create, earl_dispatch_plan, earl_dispatch_exec,
...); ``Comm`` and ``Plan`` are small owning wrappers around the handles.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libearl_dispatch.so")

EARL_ALL_RANKS = -1
EARL_MAX_WORLD = 8
EARL_MAX_FIELDS = 16
EARL_HANDLE_BYTES = 128

STATUS = {
    0: "EARL_OK", 1: "EARL_ERR_INVALID_ARGUMENT", 2: "EARL_ERR_LAYOUT", 3: "EARL_ERR_CAPACITY",
    4: "EARL_ERR_CUDA", 5: "EARL_ERR_NCCL", 6: "EARL_ERR_TIMEOUT", 7: "EARL_ERR_MISMATCH",
    8: "EARL_ERR_UNSUPPORTED", 9: "EARL_ERR_POLICY",
}
ASSIGN = {"given_counts": 0, "contig": 1, "lpt": 2, "explicit": 3}

# every symbol include/earl_dispatch.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "earl_comm_create", "earl_comm_export_handle", "earl_comm_import_peers", "earl_comm_alloc",
    "earl_comm_reset_alloc", "earl_comm_info", "earl_comm_destroy", "earl_dispatch_plan",
    "earl_plan_replan", "earl_plan_sync", "earl_plan_local_sizes", "earl_plan_local_meta", "earl_plan_stats",
    "earl_plan_hash",
    "earl_plan_export", "earl_plan_groups", "earl_plan_destroy", "earl_dispatch_exec", "earl_dispatch_exec_src",
    "earl_dispatch_pack", "earl_dispatch_unpack", "earl_plan_messages", "earl_returns", "earl_advantages", "earl_status_string", "earl_last_error",
    "earl_abi_version", "earl_kernel_launch_count", "earl_speedup_pct", "earl_policy_build",
    "earl_policy_table", "earl_policy_select", "earl_policy_destroy", "earl_plan_mean_length",
    "earl_allgather_lengths", "earl_comm_check", "earl_comm_peer_mask",
    "earl_nccl_unique_id", "earl_comm_init_nccl", "earl_dispatch_exchange", "earl_dispatch_exec_staged",
    "earl_plan_seq_fields", "earl_comm_mc_create", "earl_comm_mc_join", "earl_comm_set_nodes",
    "earl_dispatch_exec_hier", "earl_comm_set_exec_options",
]


class EarlError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.name = STATUS.get(status, str(status))


SP_SPLIT = {"block": 0, "zigzag": 1, "flat": 2, "threshold": 3}


class Layout(C.Structure):
    _fields_ = [("rank0", C.c_int32), ("dp", C.c_int32), ("sp", C.c_int32), ("tp", C.c_int32),
                ("assign", C.c_int32), ("sp_split", C.c_int32), ("sp_min_len", C.c_int32),
                ("reserved", C.c_int32),
                ("counts", C.POINTER(C.c_int64)), ("group_of_seq", C.c_void_p)]


class Field(C.Structure):
    _fields_ = [("bytes_per_elem", C.c_uint32), ("elems_per_token", C.c_uint32)]


W8 = C.c_uint64 * EARL_MAX_WORLD


class PlanStats(C.Structure):
    _fields_ = [("world", C.c_int32), ("n_fields", C.c_int32),
                ("bytes_per_token", C.c_uint64), ("total_tokens", C.c_uint64),
                ("C", W8 * EARL_MAX_WORLD), ("egress", W8), ("ingress", W8), ("self_bytes", W8),
                ("total_bytes", C.c_uint64), ("moved_bytes", C.c_uint64),
                ("max_egress", C.c_uint64), ("max_ingress", C.c_uint64),
                ("read_bytes", W8), ("stage_bytes", W8),
                ("n_local_seqs", C.c_int64 * EARL_MAX_WORLD),
                ("n_local_tokens", C.c_int64 * EARL_MAX_WORLD),
                ("n_segments", C.c_int64), ("n_pieces", C.c_int64), ("n_records", C.c_int64)]

    def to_dict(self):
        W = self.world
        return {
            "world": W, "n_fields": self.n_fields, "bytes_per_token": self.bytes_per_token,
            "total_tokens": self.total_tokens,
            "C": [[self.C[s][d] for d in range(W)] for s in range(W)],
            "egress": list(self.egress)[:W], "ingress": list(self.ingress)[:W],
            "self": list(self.self_bytes)[:W], "total": self.total_bytes,
            "moved": self.moved_bytes, "max_egress": self.max_egress,
            "max_ingress": self.max_ingress, "read_bytes": list(self.read_bytes)[:W],
            "stage_bytes": list(self.stage_bytes)[:W],
            "n_local_seqs": list(self.n_local_seqs)[:W],
            "n_local_tokens": list(self.n_local_tokens)[:W],
            "segments": self.n_segments, "pieces": self.n_pieces, "records": self.n_records,
        }


_LIB = None


def lib():
    """Load libearl_dispatch.so (raises if it was not built: no fallback exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2510_05943_b200.build` "
                          "(the dispatcher has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    pvp = C.POINTER(C.c_void_p)
    sig = {
        "earl_comm_create": [i32, i32, i32, u64, pvp],
        "earl_comm_export_handle": [vp, vp],
        "earl_comm_import_peers": [vp, vp],
        "earl_comm_alloc": [vp, i32, u64, pvp],
        "earl_comm_reset_alloc": [vp],
        "earl_comm_info": [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)],
        "earl_comm_destroy": [vp],
        "earl_allgather_lengths": [vp, vp, pvp, vp, vp],
        "earl_comm_check": [vp, vp],
        "earl_comm_peer_mask": [vp, C.POINTER(C.c_uint32)],
        "earl_nccl_unique_id": [vp],
        "earl_comm_init_nccl": [vp, vp],
        "earl_dispatch_exchange": [vp, vp, vp, vp],
        "earl_dispatch_exec_staged": [vp, pvp, pvp, vp],
        "earl_plan_seq_fields": [vp, C.POINTER(Field), i32, vp, pvp],
        "earl_comm_mc_create": [vp, C.c_uint32, vp],
        "earl_comm_set_nodes": [vp, i32],
        "earl_comm_set_exec_options": [vp, i32, i32],
        "earl_dispatch_exec_hier": [vp, pvp, pvp, vp],
        "earl_comm_mc_join": [vp, C.c_uint32, vp],
        "earl_dispatch_plan": [vp, C.POINTER(Layout), C.POINTER(Layout), vp, i64,
                               C.POINTER(Field), i32, vp, pvp],
        "earl_plan_sync": [vp],
        "earl_plan_replan": [vp, vp, vp],
        "earl_plan_local_sizes": [vp, i32, C.POINTER(i64), C.POINTER(i64)],
        "earl_plan_local_meta": [vp, i32, vp, vp, vp, vp],
        "earl_plan_stats": [vp, C.POINTER(PlanStats)],
        "earl_plan_hash": [vp, C.POINTER(C.c_uint64)],
        "earl_plan_export": [vp, i64, C.POINTER(i64), vp, vp, vp, vp, vp, vp, vp],
        "earl_plan_destroy": [vp],
        "earl_plan_groups": [vp, vp, vp, vp],
        "earl_dispatch_exec": [vp, pvp, pvp, vp],
        "earl_dispatch_exec_src": [vp, i32, pvp, pvp, vp],
        "earl_dispatch_pack": [vp, pvp, pvp, vp],
        "earl_dispatch_unpack": [vp, pvp, pvp, vp],
        "earl_plan_messages": [vp, i32, vp, vp, vp, vp],
        "earl_returns": [vp, C.c_float, pvp, pvp, pvp, pvp, vp, vp],
        "earl_advantages": [vp, vp, C.c_float, pvp, pvp, pvp, vp],
        "earl_speedup_pct": [C.c_double, C.c_double, C.POINTER(C.c_double)],
        "earl_policy_build": [i32, vp, i32, vp, vp, vp, i64, pvp],
        "earl_policy_table": [vp, vp],
        "earl_policy_select": [vp, C.c_double, i32, C.POINTER(i32), C.POINTER(i32)],
        "earl_policy_destroy": [vp],
        "earl_plan_mean_length": [vp, C.POINTER(C.c_double)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.earl_status_string.argtypes = [C.c_int]
    L.earl_status_string.restype = C.c_char_p
    L.earl_last_error.argtypes = []
    L.earl_last_error.restype = C.c_char_p
    L.earl_abi_version.restype = C.c_int32
    L.earl_kernel_launch_count.restype = C.c_uint64
    _LIB = L
    return L


def check(status: int):
    if status != 0:
        msg = lib().earl_last_error().decode(errors="replace")
        raise EarlError(status, msg or STATUS.get(status, str(status)))


def _ptr(x) -> int:
    """Device pointer of a torch tensor, or an int / None."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


def _stream(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class PtrArray:
    """A buffer list marshalled once into a C pointer array (void* const*): pass it in place of the
    list to exec / exec_src / pack / unpack / returns ... when the same buffers are dispatched
    every step, so the per-call marshalling (~0.5 us per pointer in Python) is paid once.  Holds
    references to the tensors."""

    def __init__(self, items):
        self.items = list(items)
        self.arr = (C.c_void_p * max(1, len(self.items)))()
        for k, it in enumerate(self.items):
            self.arr[k] = _ptr(it) or None

    def __len__(self):
        return len(self.items)


def _ptr_array(items):
    if isinstance(items, PtrArray):
        return items.arr
    arr = (C.c_void_p * max(1, len(items)))()
    for k, it in enumerate(items):
        arr[k] = _ptr(it) or None
    return arr


def make_layout(d) -> Layout:
    """Layout from a dict {rank0, dp, sp, tp, assign, counts, group_of_seq}.

    group_of_seq (EXPLICIT) must be a device int32 tensor (or a device pointer)."""
    lay = Layout()
    lay.rank0, lay.dp = int(d.get("rank0", 0)), int(d.get("dp", 1))
    lay.sp, lay.tp = int(d.get("sp", 1)), int(d.get("tp", 1))
    a = d.get("assign", "contig")
    lay.assign = ASSIGN[a] if isinstance(a, str) else int(a)
    sp = d.get("sp_split", "block")
    lay.sp_split = SP_SPLIT[sp] if isinstance(sp, str) else int(sp)
    lay.sp_min_len = int(d.get("sp_min_len", 0))
    lay.reserved = 0
    counts = d.get("counts")
    if counts is not None:
        arr = (C.c_int64 * len(counts))(*[int(c) for c in counts])
        lay._counts_keepalive = arr
        lay.counts = C.cast(arr, C.POINTER(C.c_int64))
    gos = d.get("group_of_seq_dev")
    lay.group_of_seq = _ptr(gos) or None
    return lay


def make_fields(fields):
    """fields: [(name, bytes_per_elem, elems_per_token, ...)] or [(bpe, ept)]."""
    arr = (Field * len(fields))()
    for k, f in enumerate(fields):
        bpe, ept = (f[1], f[2]) if isinstance(f[0], str) else (f[0], f[1])
        arr[k].bytes_per_elem, arr[k].elems_per_token = int(bpe), int(ept)
    return arr


# ---------------------------------------------------------------------------------------
# owning wrappers
# ---------------------------------------------------------------------------------------

class Comm:
    """earl_comm_t.  rank=EARL_ALL_RANKS emulates every rank in this process (1 GPU)."""

    def __init__(self, rank: int, world: int, device: int = 0, window_bytes: int = 0):
        h = C.c_void_p()
        check(lib().earl_comm_create(int(rank), int(world), int(device), int(window_bytes),
                                     C.byref(h)))
        self.h = h
        self.rank, self.world, self.device = int(rank), int(world), int(device)
        self.emulated = rank == EARL_ALL_RANKS

    def export_handle(self) -> bytes:
        buf = (C.c_uint8 * EARL_HANDLE_BYTES)()
        check(lib().earl_comm_export_handle(self.h, buf))
        return bytes(buf)

    def import_peers(self, handles):
        blob = b"".join(handles)
        assert len(blob) == EARL_HANDLE_BYTES * self.world
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib().earl_comm_import_peers(self.h, buf))

    def alloc(self, nbytes: int, rank: int = 0) -> int:
        p = C.c_void_p()
        check(lib().earl_comm_alloc(self.h, int(rank), int(nbytes), C.byref(p)))
        return int(p.value or 0)

    def reset_alloc(self):
        check(lib().earl_comm_reset_alloc(self.h))

    def allgather_lengths(self, counts, local_lens, global_lens, stream=None):
        """earl_allgather_lengths (step a1): counts = per-rank sequence counts (host, every rank
        the same); local_lens = [this rank's int32 tensor] (emulated: one per rank, None where
        the count is 0); global_lens = int32 device tensor of sum(counts) elements (output)."""
        cnt = np.ascontiguousarray(counts, dtype=np.int64)
        assert cnt.size == self.world
        check(lib().earl_allgather_lengths(self.h, cnt.ctypes.data, _ptr_array(local_lens),
                                           _ptr(global_lens) or None, _stream(stream)))

    def init_nccl(self, unique_id: bytes):
        """earl_comm_init_nccl (collective): the staged exchange's NCCL communicator."""
        buf = (C.c_uint8 * EARL_HANDLE_BYTES).from_buffer_copy(unique_id)
        check(lib().earl_comm_init_nccl(self.h, buf))

    def set_exec_options(self, remote_store: int = -1, p2p_shape: int = -1):
        """earl_comm_set_exec_options: NVLink store variant and copy-engine shape (-1: default)."""
        check(lib().earl_comm_set_exec_options(self.h, int(remote_store), int(p2p_shape)))

    def set_nodes(self, node_size: int):
        """earl_comm_set_nodes (NEXT-4): node_size consecutive ranks per node; before import."""
        check(lib().earl_comm_set_nodes(self.h, int(node_size)))

    def mc_create(self, team_mask: int) -> bytes:
        """earl_comm_mc_create (NEXT-3; the team's lowest rank): the team handle to broadcast."""
        buf = (C.c_uint8 * EARL_HANDLE_BYTES)()
        check(lib().earl_comm_mc_create(self.h, int(team_mask), buf))
        return bytes(buf)

    def mc_join(self, team_mask: int, handle: bytes):
        """earl_comm_mc_join (NEXT-3; every rank, members concurrently)."""
        buf = (C.c_uint8 * EARL_HANDLE_BYTES).from_buffer_copy(handle)
        check(lib().earl_comm_mc_join(self.h, int(team_mask), buf))

    def peer_mapped(self, p: int) -> bool:
        """earl_comm_peer_mask: is peer p's window mapped into this process?"""
        m = C.c_uint32()
        check(lib().earl_comm_peer_mask(self.h, C.byref(m)))
        return bool(m.value >> int(p) & 1)

    def check(self, stream=None):
        """earl_comm_check: synchronise `stream`, raise a device-latched comm error."""
        check(lib().earl_comm_check(self.h, _stream(stream)))

    def plan(self, src, dst, seq_lens, fields, stream=None) -> "Plan":
        return Plan(self, src, dst, seq_lens, fields, stream)

    def destroy(self):
        if self.h:
            check(lib().earl_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Plan:
    """earl_plan_t produced by earl_dispatch_plan (device-side planner, no host sync)."""

    @classmethod
    def seq_fields(cls, token_plan: "Plan", sfields, stream=None) -> "Plan":
        """earl_plan_seq_fields (reading n4): per-sequence fields routed along token_plan."""
        p = cls.__new__(cls)
        p.comm = token_plan.comm
        p.fields = list(sfields)
        p._fa = make_fields(p.fields)
        h = C.c_void_p()
        check(lib().earl_plan_seq_fields(token_plan.h, p._fa, len(p.fields), _stream(stream),
                                         C.byref(h)))
        p.h = h
        p.n_seqs = token_plan.n_seqs
        p._seq_lens = None
        p._groups_keepalive = None
        p._parent = token_plan  # the library keeps the token plan alive; so does the binding
        return p

    def __init__(self, comm: Comm, src, dst, seq_lens, fields, stream=None):
        self.comm = comm
        self.fields = list(fields)
        self._src, self._dst = make_layout(src), make_layout(dst)
        self._fa = make_fields(self.fields)
        n = int(seq_lens.numel())
        h = C.c_void_p()
        check(lib().earl_dispatch_plan(comm.h, C.byref(self._src), C.byref(self._dst),
                                       _ptr(seq_lens) or None, n, self._fa, len(self.fields),
                                       _stream(stream), C.byref(h)))
        self.h = h
        self.n_seqs = n
        self._seq_lens = seq_lens  # keep alive until the planner ran
        # EXPLICIT group vectors are re-read by every replan: they live as long as the plan
        self._groups_keepalive = (src.get("group_of_seq_dev"), dst.get("group_of_seq_dev"))

    def replan(self, seq_lens=None, stream=None):
        """Re-run the device planner for new lengths (same N) into this plan's memory (a
        per-sequence field plan takes no lengths: it re-reads its token plan's groups)."""
        if seq_lens is not None:
            assert int(seq_lens.numel()) == self.n_seqs
        check(lib().earl_plan_replan(self.h, _ptr(seq_lens) or None, _stream(stream)))
        if seq_lens is not None:
            self._seq_lens = seq_lens

    # -- queries (host-synchronising) --
    def sync(self):
        check(lib().earl_plan_sync(self.h))

    def local_sizes(self, rank: int):
        ns, nt = C.c_int64(), C.c_int64()
        check(lib().earl_plan_local_sizes(self.h, int(rank), C.byref(ns), C.byref(nt)))
        return ns.value, nt.value

    def local_meta(self, rank: int, cu_seqlens=None, seq_ids=None, tok_start=None, stream=None):
        check(lib().earl_plan_local_meta(self.h, int(rank), _ptr(cu_seqlens) or None,
                                         _ptr(seq_ids) or None, _ptr(tok_start) or None,
                                         _stream(stream)))

    def mean_length(self) -> float:
        """Averaged context length of the planned batch, T / N (selector reading s4)."""
        v = C.c_double()
        check(lib().earl_plan_mean_length(self.h, C.byref(v)))
        return v.value

    def hash(self) -> int:
        """earl_plan_hash: 64-bit hash of the plan's tables and records (debug; synchronises)."""
        h = C.c_uint64()
        check(lib().earl_plan_hash(self.h, C.byref(h)))
        return h.value

    def stats(self) -> dict:
        st = PlanStats()
        check(lib().earl_plan_stats(self.h, C.byref(st)))
        return st.to_dict()

    def export(self):
        """Canonical (s, d, i, x) segment table as a list of 7-tuples (s, d, i, x, y, so, do)."""
        n = C.c_int64()
        check(lib().earl_plan_export(self.h, 0, C.byref(n), *([None] * 7)))
        m = n.value
        cols = [np.zeros(max(m, 1), dt) for dt in (np.int32, np.int32, np.int64, np.int32,
                                                   np.int32, np.int64, np.int64)]
        ptrs = [c.ctypes.data_as(C.c_void_p) for c in cols]
        check(lib().earl_plan_export(self.h, m, C.byref(n), *ptrs))
        return [tuple(int(c[j]) for c in cols) for j in range(m)]

    def groups(self, src_groups=None, dst_groups=None, stream=None):
        """Device copies of g_src(i) and g_dst(i) (int32 [N] tensors)."""
        check(lib().earl_plan_groups(self.h, _ptr(src_groups) or None, _ptr(dst_groups) or None,
                                     _stream(stream)))

    def messages(self, rank: int):
        """Per-peer (send_off, send_bytes, recv_off, recv_bytes) of `rank` (host-synchronising)."""
        W = self.comm.world
        arrs = [np.zeros(W, dtype=np.int64) for _ in range(4)]
        check(lib().earl_plan_messages(self.h, int(rank), *[x.ctypes.data_as(C.c_void_p) for x in arrs]))
        return [x.tolist() for x in arrs]

    # -- execution (stream-ordered, asynchronous) --
    def exec(self, send_bufs, recv_bufs, stream=None):
        s, r = _ptr_array(send_bufs), _ptr_array(recv_bufs)
        check(lib().earl_dispatch_exec(self.h, s, r, _stream(stream)))

    def exec_src(self, src_rank, send_bufs, recv_bufs, stream=None):
        """earl_dispatch_exec_src: only source rank src_rank's records."""
        s, r = _ptr_array(send_bufs), _ptr_array(recv_bufs)
        check(lib().earl_dispatch_exec_src(self.h, int(src_rank), s, r, _stream(stream)))

    def exchange(self, send_stage, recv_stage, stream=None):
        """earl_dispatch_exchange: grouped ncclSend / ncclRecv of this rank's messages."""
        check(lib().earl_dispatch_exchange(self.h, _ptr(send_stage) or None, _ptr(recv_stage) or None,
                                           _stream(stream)))

    def exec_hier(self, send_bufs, recv_bufs, stream=None):
        """earl_dispatch_exec_hier (NEXT-4): fused P2P inside the node, NCCL between nodes."""
        s, r = _ptr_array(send_bufs), _ptr_array(recv_bufs)
        check(lib().earl_dispatch_exec_hier(self.h, s, r, _stream(stream)))

    def exec_staged(self, send_bufs, recv_bufs, stream=None):
        """earl_dispatch_exec_staged: pack + NCCL exchange + unpack (library stage buffers)."""
        s, r = _ptr_array(send_bufs), _ptr_array(recv_bufs)
        check(lib().earl_dispatch_exec_staged(self.h, s, r, _stream(stream)))

    def pack(self, send_bufs, stage_bufs, stream=None):
        s, t = _ptr_array(send_bufs), _ptr_array(stage_bufs)
        check(lib().earl_dispatch_pack(self.h, s, t, _stream(stream)))

    def unpack(self, stage_bufs, recv_bufs, stream=None):
        t, r = _ptr_array(stage_bufs), _ptr_array(recv_bufs)
        check(lib().earl_dispatch_unpack(self.h, t, r, _stream(stream)))

    # -- NEXT-2: distributed advantage estimation on the source ranks --
    def returns(self, gamma, rewards, mask, returns, partial, seq_return=None, stream=None):
        check(lib().earl_returns(self.h, float(gamma), _ptr_array(rewards), _ptr_array(mask),
                                 _ptr_array(returns),
                                 _ptr_array(seq_return) if seq_return is not None else None,
                                 _ptr(partial) or None, _stream(stream)))

    def advantages(self, stats, eps, returns, mask, adv, stream=None):
        check(lib().earl_advantages(self.h, _ptr(stats) or None, float(eps), _ptr_array(returns),
                                    _ptr_array(mask), _ptr_array(adv), _stream(stream)))

    def destroy(self):
        if getattr(self, "h", None):
            check(lib().earl_plan_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def speedup_pct(tgs_a: float, tgs_b: float) -> float:
    """Eq. (1)."""
    v = C.c_double()
    check(lib().earl_speedup_pct(float(tgs_a), float(tgs_b), C.byref(v)))
    return v.value


class Policy:
    """The Parallelism Selector's table (host-only).  config_tp[c] is
    configuration c's TP degree; bounds the n_buckets+1 context-range edges; tgs / oom are
    [n_configs][n_buckets] profiles."""

    def __init__(self, config_tp, bounds, tgs, oom=None, hysteresis_tokens=0):
        tp = np.ascontiguousarray(config_tp, dtype=np.int32)
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        t = np.ascontiguousarray(tgs, dtype=np.float64).reshape(-1)
        o = None if oom is None else np.ascontiguousarray(oom, dtype=np.uint8).reshape(-1)
        self.n_configs, self.n_buckets = int(tp.size), int(b.size) - 1
        h = C.c_void_p()
        check(lib().earl_policy_build(self.n_configs, tp.ctypes.data, self.n_buckets, b.ctypes.data,
                                      t.ctypes.data, None if o is None else o.ctypes.data,
                                      int(hysteresis_tokens), C.byref(h)))
        self.h = h

    def table(self):
        out = np.zeros(max(self.n_buckets, 1), dtype=np.int32)
        check(lib().earl_policy_table(self.h, out.ctypes.data))
        return out[: self.n_buckets].tolist()

    def select(self, avg_len: float, current: int):
        """-> (next configuration, switched)."""
        nxt, sw = C.c_int32(), C.c_int32()
        check(lib().earl_policy_select(self.h, float(avg_len), int(current), C.byref(nxt), C.byref(sw)))
        return nxt.value, bool(sw.value)

    def destroy(self):
        if getattr(self, "h", None):
            check(lib().earl_policy_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * EARL_HANDLE_BYTES)()
    check(lib().earl_nccl_unique_id(buf))
    return bytes(buf)


def kernel_launch_count() -> int:
    return int(lib().earl_kernel_launch_count())


def abi_version() -> int:
    return int(lib().earl_abi_version())
