"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO dispatch arithmetic (no planning, routing, chunking or offset
computation).  It only draws the inputs the method consumes:

* sequence lengths (lognormal long tail, SURVEY.md §8(d) "Synthetic inputs";
  the lognormal shape is SPEC.md:357/382's proposal, the cap mass mirrors
  PAPER.md:136, Fig. 2b "episode-level context length quickly reaches the
  system limit");
* per-token field payload bytes (ids, log-probs, values, advantages, masks,
  optional hidden vector; "tokens, log probabilities, rewards,
  returns, and other auxiliary tensors");
* layout descriptors as plain dicts (the caller-side description of a
  parallel layout; both the oracle and the CUDA binding parse them on their own);
* the rollout-side source holdings for rank-major GIVEN_COUNTS layouts without
  SP, which are plain contiguous slices of the global batch (the rollout stage
  produced them that way; SURVEY.md §8(c) reading c6).

Every random draw is seeded; nothing here reads /root/reference.
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# fields
# ---------------------------------------------------------------------------

VOCAB = 152064  # Qwen2.5 vocabulary size (ids are uniform in [0, VOCAB))

# (name, bytes_per_elem, elems_per_token, kind)
SCALAR6_FP32 = [
    ("ids", 4, 1, "ids"),
    ("old_logprobs", 4, 1, "logprob_f32"),
    ("ref_logprobs", 4, 1, "logprob_f32"),
    ("values", 4, 1, "normal_f32"),
    ("advantages", 4, 1, "normal_f32"),
    ("response_mask", 1, 1, "mask"),
]
SCALAR6_BF16 = [
    ("ids", 4, 1, "ids"),
    ("old_logprobs", 2, 1, "logprob_bf16"),
    ("ref_logprobs", 2, 1, "logprob_bf16"),
    ("values", 2, 1, "normal_bf16"),
    ("advantages", 2, 1, "normal_bf16"),
    ("response_mask", 1, 1, "mask"),
]
TINY3 = [
    ("ids", 4, 1, "ids"),
    ("logprobs", 4, 1, "logprob_f32"),
    ("advantages", 4, 1, "normal_f32"),
]


def hidden_field(width: int):
    return ("hidden", 2, int(width), "normal_bf16")


def field_set(name: str):
    """Named field sets of SURVEY.md §8 (scalar6-fp32 = 21 B/token, +hidden(H) = 21+2H)."""
    if name == "tiny3":
        return list(TINY3)
    if name == "scalar6-fp32":
        return list(SCALAR6_FP32)
    if name == "scalar6-bf16":
        return list(SCALAR6_BF16)
    if name.startswith("scalar6-fp32+hidden"):
        return list(SCALAR6_FP32) + [hidden_field(int(name.split("hidden")[1]))]
    if name.startswith("hidden"):
        return [hidden_field(int(name[len("hidden"):]))]
    raise ValueError(f"unknown field set {name!r}")


def bytes_per_token(fields) -> int:
    return int(sum(b * e for (_, b, e, _) in fields))


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern by truncation (the payload is opaque; any pattern is valid)."""
    return (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)


def gen_field_bytes(field, n_tokens: int, seed: int, random_bits: bool = False) -> np.ndarray:
    """Global (sequence-order) payload of one field as a uint8 array [n_tokens * Bf]."""
    _, bpe, ept, kind = field
    n = int(n_tokens) * ept
    rng = np.random.default_rng(seed)
    if random_bits:
        return rng.integers(0, 256, size=n * bpe, dtype=np.uint8)
    if kind == "ids":
        arr = rng.integers(0, VOCAB, size=n, dtype=np.int32)
    elif kind == "logprob_f32":
        arr = (-rng.exponential(1.0, size=n)).astype(np.float32)
    elif kind == "normal_f32":
        arr = rng.standard_normal(n, dtype=np.float32)
    elif kind == "logprob_bf16":
        arr = _bf16_bits(-rng.exponential(1.0, size=n))
    elif kind == "normal_bf16":
        arr = _bf16_bits(rng.standard_normal(n, dtype=np.float32))
    elif kind == "mask":
        arr = (rng.random(n) < 0.8).astype(np.uint8)
    else:
        raise ValueError(kind)
    out = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    assert out.size == n * bpe
    return out


def gen_global_fields(fields, n_tokens: int, seed_base: int = 1000, random_bits: bool = False):
    """Per-field global payloads, seeds 1000+field index."""
    return [gen_field_bytes(f, n_tokens, seed_base + k, random_bits) for k, f in enumerate(fields)]


# ---------------------------------------------------------------------------
# lengths
# ---------------------------------------------------------------------------

def lognormal_lengths(n: int, median: float, sigma: float, lo: int, hi: int, seed: int = 0) -> np.ndarray:
    """L = clip(rint(exp(N(ln median, sigma))), lo, hi) as int64."""
    rng = np.random.default_rng(seed)
    x = np.exp(rng.normal(np.log(median), sigma, int(n)))
    return np.clip(np.rint(x), lo, hi).astype(np.int64)


TINY_LENGTHS = np.array([5, 17, 64, 9, 33, 12, 48, 21], dtype=np.int64)


def c2_lengths(seed: int = 0) -> np.ndarray:
    """Config 2: 512 episodes, long-tail context <= 8192 (BASELINE.json configs[1])."""
    return lognormal_lengths(512, 2048, 0.75, 64, 8192, seed)


def c4_lengths(seed: int = 0) -> np.ndarray:
    """Config 4: 256 episodes, lengths 4K-32K long tail (BASELINE.json configs[3])."""
    return lognormal_lengths(256, 8192, 0.6, 4096, 32768, seed)


# ---------------------------------------------------------------------------
# layouts (plain dicts; rank(g,k,t) = rank0 + (g*sp + k)*tp + t is documented in
# include/earl_dispatch.h and implemented separately by each side)
# ---------------------------------------------------------------------------

# The paper's dispatch experiment (Fig. 4): log-prob tensors of the reference
# model's workers, "46 MiB, 93 MiB, and 187 MiB per independent worker" at context
# 8K / 16K / 32K.  Reading: each worker holds FIG4_RESPONSES responses padded to the
# context length, one fp32 log-prob per token (1500 x L x 4 B = 46.875 / 93.75 / 187.5 MiB).
FIG4_RESPONSES = 1500
FIG4_CONTEXTS = (8192, 16384, 32768)


def fig4_lengths(context: int, workers: int = 8) -> np.ndarray:
    return np.full(workers * FIG4_RESPONSES, int(context), dtype=np.int64)


def layout(rank0=0, dp=1, sp=1, tp=1, assign="contig", counts=None, group_of_seq=None,
           sp_split="block", sp_min_len=0):
    return {
        "rank0": int(rank0), "dp": int(dp), "sp": int(sp), "tp": int(tp),
        "assign": assign, "sp_split": sp_split, "sp_min_len": int(sp_min_len),
        "counts": None if counts is None else [int(c) for c in counts],
        "group_of_seq": None if group_of_seq is None else np.asarray(group_of_seq, dtype=np.int32),
    }


def near_equal_counts(n: int, d: int):
    """Rollout-side counts: near-equal blocks, earlier groups take the extra (SPEC.md:215 remainder rule)."""
    q, r = divmod(int(n), int(d))
    return [q + (1 if g < r else 0) for g in range(int(d))]


def rollout_layout(n_seqs: int, dp: int, rank0: int = 0):
    """Rollout DPn source layout: GIVEN_COUNTS, rank-major blocks of sequences."""
    return layout(rank0=rank0, dp=dp, assign="given_counts", counts=near_equal_counts(n_seqs, dp))


def rollout_holdings(global_fields, fields, lengths, counts):
    """Per-src-rank arrays of a GIVEN_COUNTS, SP=1, TP=1 rollout layout: contiguous slices.

    Input preparation only: rank g holds sequences [sum(counts[:g]), +counts[g]) and therefore
    the contiguous token block that covers them.
    """
    lengths = np.asarray(lengths, dtype=np.int64)
    tok_edges = np.concatenate([[0], np.cumsum(lengths)])
    seq_edges = np.concatenate([[0], np.cumsum(np.asarray(counts, dtype=np.int64))])
    out = []
    for g in range(len(counts)):
        t0, t1 = tok_edges[seq_edges[g]], tok_edges[seq_edges[g + 1]]
        per_field = []
        for arr, (_, bpe, ept, _) in zip(global_fields, fields):
            bf = bpe * ept
            per_field.append(arr[t0 * bf: t1 * bf])
        out.append(per_field)
    return out


def gen_field_device(field, n_tokens: int, seed: int, device):
    """Device-side draw of one field for a rank holding n_tokens tokens (same distributions as
    gen_field_bytes, drawn with a seeded torch CUDA generator; used where host generation of
    multi-GB payloads would dominate).  Returns a uint8 tensor [n_tokens * Bf]."""
    import torch
    _, bpe, ept, kind = field
    n = int(n_tokens) * ept
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    if kind == "ids":
        t = torch.randint(0, VOCAB, (n,), dtype=torch.int32, device=device, generator=g)
    elif kind in ("logprob_f32", "logprob_bf16"):
        t = -torch.empty(n, dtype=torch.float32, device=device).exponential_(1.0, generator=g)
        if kind == "logprob_bf16":
            t = t.to(torch.bfloat16)
    elif kind in ("normal_f32", "normal_bf16"):
        t = torch.randn(n, dtype=torch.float32, device=device, generator=g)
        if kind == "normal_bf16":
            t = t.to(torch.bfloat16)
    elif kind == "mask":
        t = (torch.rand(n, device=device, generator=g) < 0.8).to(torch.uint8)
    else:
        t = torch.randint(0, 256, (n * bpe,), dtype=torch.uint8, device=device, generator=g)
    out = t.contiguous().view(torch.uint8).reshape(-1)
    assert out.numel() == n * bpe
    return out


def rollout_token_counts(lengths, counts):
    """Tokens held by each rank of a GIVEN_COUNTS rollout layout (input sizing only)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    edges = np.concatenate([[0], np.cumsum(np.asarray(counts, dtype=np.int64))])
    return [int(lengths[edges[g]:edges[g + 1]].sum()) for g in range(len(counts))]


def config_layouts(config: str, n_gpus: int, n_seqs: int):
    """(src, dst) layouts of BASELINE.json's configs at world size n_gpus."""
    n = int(n_gpus)
    src = rollout_layout(n_seqs, n)
    if config in ("c1", "tiny"):
        return rollout_layout(n_seqs, 2), layout(dp=1, assign="contig")
    if config in ("c2", "c3"):
        return src, layout(dp=max(1, n // 4), tp=min(4, n), assign="contig")
    if config == "c4":
        return src, layout(dp=max(1, n // 2), sp=2 if n >= 2 else 1, assign="contig")
    if config == "c2-lpt":
        return src, layout(dp=n, assign="lpt")
    if config == "c5":
        return src, layout(dp=n, assign="explicit", group_of_seq=np.arange(n_seqs, dtype=np.int32) % n)
    raise ValueError(config)
