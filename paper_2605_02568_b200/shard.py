"""Query-axis sharding helpers for multi-GPU runs (one process per GPU).

The plan itself is the library's (csaidx::gpu::plan_shards, C++; LPT over
the c_S chunks by causal work — see paper_2605_02568_b200/multi.py). Query
rows are independent (reference driver.cpp:132-133), so only two exchanges
exist: the keys are broadcast once from rank 0 and the [S, k] index rows are
collected on rank 0. These helpers keep the old (S, m, c_S, world) call form
for bench.py and the tests.
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
    """-> (per-rank sorted chunk-start lists, per-rank work): the library's LPT plan."""
    from . import api, multi

    dims = api.ProblemDims.create(1, seq_len, ratio, 1, 1, 1)
    return multi.plan_shards(dims, query_tile, world)


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
