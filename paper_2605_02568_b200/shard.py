"""Query-axis sharding for multi-GPU runs (one process per GPU).

Query rows are independent (reference driver.cpp:132-133), so the c_S query
chunks are split across ranks; only two exchanges exist: the keys are
broadcast once from rank 0, and the [S, k] index rows are gathered back.
Chunk cost is proportional to its causal work (sum of t_legal over its
rows), so contiguous blocks would hand the last rank ~(2P-1)/P^2 of the work;
chunks are assigned by LPT (longest first, to the least-loaded rank) instead.
"""
from __future__ import annotations

import numpy as np


def chunk_starts(seq_len: int, query_tile: int) -> list[int]:
    cs = min(query_tile, seq_len)
    return list(range(0, seq_len, cs))


def chunk_work(seq_len: int, ratio: int, query_tile: int, s0: int) -> int:
    """Causal-legal pairs of one query chunk (per batch)."""
    cs = min(query_tile, seq_len)
    t = np.arange(s0, min(s0 + cs, seq_len), dtype=np.int64)
    return int(np.minimum((t + 1) // ratio, seq_len // ratio).sum())


def plan_shards(seq_len: int, ratio: int, query_tile: int, world: int):
    """-> (per-rank sorted chunk-start lists, per-rank work)."""
    starts = chunk_starts(seq_len, query_tile)
    cost = sorted(((chunk_work(seq_len, ratio, query_tile, s), s) for s in starts), reverse=True)
    loads = [0] * world
    owned: list[list[int]] = [[] for _ in range(world)]
    for c, s in cost:
        r = min(range(world), key=lambda i: (loads[i], i))
        loads[r] += c
        owned[r].append(s)
    return [sorted(o) for o in owned], loads


def rows_of(seq_len: int, query_tile: int, starts) -> int:
    cs = min(query_tile, seq_len)
    return int(sum(min(cs, seq_len - s) for s in starts))


def assemble(parts, shards, seq_len: int, query_tile: int):
    """Scatter per-rank packed rows [B, rows_r(+pad), k] back to [B, S, k]."""
    cs = min(query_tile, seq_len)
    B, _, k = parts[0].shape
    out = np.empty((B, seq_len, k), dtype=parts[0].dtype)
    for part, starts in zip(parts, shards):
        row = 0
        for s0 in starts:
            n = min(cs, seq_len - s0)
            out[:, s0:s0 + n] = part[:, row:row + n]
            row += n
    return out
