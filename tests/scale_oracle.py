"""Sampled-row oracle checks at the BASELINE sizes (test infrastructure).

The CPU oracle cannot score every row of C2-C5 in a test, so each config is
held to the north-star rule (tests/parity.py) on >= 256 STRATIFIED rows,
scored by the oracle (orc_score_rows, the reference op order of
score_scalar.cpp:20-34) from the very bf16 operands the GPU consumed:

* the first and last row of chunks spread over the whole query axis (the
  lightest and heaviest rows of each chunk's launch);
* rows whose legal key count T_legal is exactly k, just above k (the
  select's `take` becomes k), at the select's candidate capacity and just
  above it (the production sample -> threshold -> stream path starts there);
* the longest row (t = S - 1);
* the rest uniformly at random over the listed chunks (fixed seed).

Reference: the acceptance gate checks every row of its instances
(/root/reference/proj/tests/acceptance.cpp:69-100); SURVEY.md §8(c) prescribes
the sampled-row oracle for the large shapes.
"""
from __future__ import annotations

import json
import os

import numpy as np

from .parity import check_rows


def stratified_rows(S, m, k, cand_cap, chunk_starts, cs, n=256, seed=0, allowed=None):
    """Sorted unique query positions t (>= n of them when the set allows).
    allowed: optional predicate on t (e.g. "owned by this rank")."""
    # rows with T_legal == 0 have nothing to select (row properties cover them)
    ok = (lambda t: m - 1 <= t < S) if allowed is None else (lambda t: m - 1 <= t < S and allowed(t))
    want = []
    starts = sorted(chunk_starts)
    pick = np.linspace(0, len(starts) - 1, min(len(starts), 24)).round().astype(int)
    for i in np.unique(pick):
        s0 = starts[i]
        want += [s0, min(s0 + cs, S) - 1]
    for L in (k - 1, k, k + 1, k + 2, cand_cap - 1, cand_cap, cand_cap + 1, cand_cap + 7, 2 * cand_cap + 1):
        if L >= 1:
            want += [m * L - 1, m * L + m - 2]  # first and last t with T_legal == L
    want += [S - 1, S - 2]
    rows = {t for t in want if ok(t)}
    rng = np.random.default_rng(seed)
    for _ in range(100 * n):  # random rows of random listed chunks
        if len(rows) >= n:
            break
        t = int(starts[rng.integers(0, len(starts))] + rng.integers(0, cs))
        if ok(t):
            rows.add(t)
    return sorted(rows)


def check_sampled(orc, q, kc, w, idx, val, dims, rows, local=None, batches=None, label=""):
    """Oracle-check rows `rows` (query positions t) of a device run.

    q / kc / w: the torch CUDA operands the GPU consumed (q bf16 [.., H, D]
    flattened as [B * rows_q, H * D], kc [B * T, D], w [B * rows_q, H]).
    idx / val: the run's outputs, [B, rows_out, k] torch or numpy.
    local: map t -> operand/output row (rank-local layouts); default t.
    batches: batch ids to check (default all)."""
    import torch

    B, S, T, H, D, m, k = (dims.batch, dims.seq_len, dims.key_blocks, dims.heads, dims.head_dim, dims.ratio,
                           dims.top_k)
    batches = list(range(B)) if batches is None else list(batches)
    loc = [t if local is None else local(t) for t in rows]
    idx_h = idx if isinstance(idx, np.ndarray) else idx.cpu().numpy()
    val_h = val if isinstance(val, np.ndarray) else val.cpu().numpy()
    rows_q = q.numel() // (B * H * D)
    qv = q.reshape(B * rows_q, H * D)
    wv = w.reshape(B * rows_q, H)
    kcf = kc.reshape(B * T, D).float().cpu().numpy()
    reports = []
    for b in batches:
        sel = torch.as_tensor([b * rows_q + r for r in loc], device=q.device)
        qr = qv.index_select(0, sel).float().cpu().numpy().reshape(len(rows), H, D)
        wr = wv.index_select(0, sel).float().cpu().numpy()
        legal = np.array([(t + 1) // m for t in rows], np.int64)
        scores = orc.score_rows(qr, wr, kcf, np.full(len(rows), b * T, np.int64), legal)
        rep = check_rows(idx_h[b][loc], val_h[b][loc], scores, legal, k)
        rep.update(batch=b, label=label, longest=int(legal.max()))
        reports.append(rep)
    record(reports)
    return reports


def record(reports):
    """Print the per-batch recall statistics; with CSAIDX_PARITY_LOG set,
    append them as JSON lines to that file."""
    for r in reports:
        print(f"[parity] {r['label']} batch {r['batch']}: rows {r['rows']} mean recall {r['mean']:.6f} "
              f"min {r['min']:.6f} tie-band rows {r['tie_rows']} longest row {r['longest']}")
    path = os.environ.get("CSAIDX_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            for r in reports:
                f.write(json.dumps(r) + "\n")
