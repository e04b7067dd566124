"""BASELINE config C5: design-space sweep at S=131,072, B=2 (T=32,768) over
c_S in {512..8192}, c_T in {4096..T}, k in {256, 512, 1024, 2048}.

For every point: device-timed step (CUDA events, warm-up first), legal
pairs/s, the reference ledger's transient peak and the device high-water.
Points with c_T < T are also timed with the device key tile held at c_T
(CSAIDX_KEY_TILE_BYTES=0): `ms` is the default (widened key tile),
`ms_key_tile_as_requested` the select + merge per requested tile.
Recall: every point's output must equal, byte for byte, the (c_S=2048,
c_T=T) run of the same k (score values do not depend on the tiling and the
merge is exact), and that run is held to the north-star rule
(tests/parity.py) against the CPU oracle on sampled rows of both batches,
scored from the very bf16 operands the GPU consumed.

usage (GPU box): python scripts/sweep_c5.py > gpurun_out/c5_sweep.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.oracle import Oracle
from paper_2605_02568_b200 import api
from tests.parity import check_rows
from tests.test_scale_gpu import make_operands, oracle_rows

B, S, H, D, m = 2, 131072, 64, 128, 4
T = S // m
e, q, kc, w = make_operands(B, S, H, D, m, seed=11)
t = np.arange(S, dtype=np.int64)
pairs = B * int(np.minimum((t + 1) // m, T).sum())
rows_t = [2047, 40000, 77777, 100003, S - 1]
orc = Oracle()
t0 = time.time()
scores = {}
for b in range(B):
    qb = q.view(B, -1)[b]
    kb = kc.view(B, -1)[b]
    wb = w.view(B, -1)[b]
    scores[b] = oracle_rows(orc, qb, kb, wb, rows_t, 0, m, H, D)
print(json.dumps({"oracle_rows": rows_t, "batches": B, "oracle_s": round(time.time() - t0, 1)}), flush=True)

dims_k = {}
for k in (256, 512, 1024, 2048):
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    ref = None
    ref_bytes = 0
    for cs in (2048, 512, 1024, 4096, 8192):
        for ct in (T, 4096, 8192, 16384):
            cfg = api.DriverConfig(tile=api.TileConfig(cs, ct))
            api.run_chunked_device(q, kc, w, dims, cfg)  # warm-up
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            idx, val, st = api.run_chunked_device(q, kc, w, dims, cfg)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            line = {"k": k, "c_S": cs, "c_T": ct, "ms": round(ms, 3), "legal_pairs_per_s": pairs / (ms / 1e3),
                    "dispatch_count": st.dispatch_count, "ledger_peak_bytes": st.ledger_peak_bytes,
                    # the held reference rows (ref) are not part of this run's working set
                    "device_peak_gb": round((torch.cuda.max_memory_allocated() - ref_bytes + st.device_peak_bytes) / 1e9,
                                            3)}
            if ref is None:
                ref = (idx.clone(), val.clone())
                ref_bytes = idx.numel() * idx.element_size() + val.numel() * val.element_size()
                hi, hv = idx.cpu().numpy(), val.cpu().numpy()
                recall = []
                for b in range(B):
                    rep = check_rows(hi[b][rows_t], hv[b][rows_t], scores[b], [(r + 1) // m for r in rows_t], k)
                    recall.append(rep)
                line["oracle_rule"] = {"rows": sum(r["rows"] for r in recall),
                                       "mean_recall": float(np.mean([r["mean"] for r in recall])),
                                       "min_recall": float(min(r["min"] for r in recall)),
                                       "tie_rows": sum(r["tie_rows"] for r in recall)}
                line["equal_to_reference_tiling"] = True
            else:
                line["equal_to_reference_tiling"] = bool(torch.equal(idx, ref[0]) and
                                                         torch.equal(val.view(torch.int32), ref[1].view(torch.int32)))
            if ct < T:
                # the same point with the device key tile held at c_T (select +
                # merge per requested tile, driver.cpp physical_key_tile)
                os.environ["CSAIDX_KEY_TILE_BYTES"] = "0"
                api.run_chunked_device(q, kc, w, dims, cfg)
                torch.cuda.synchronize()
                ev0.record()
                idx2, val2, st2 = api.run_chunked_device(q, kc, w, dims, cfg)
                ev1.record()
                torch.cuda.synchronize()
                del os.environ["CSAIDX_KEY_TILE_BYTES"]
                line["ms_key_tile_as_requested"] = round(ev0.elapsed_time(ev1), 3)
                line["as_requested_equal"] = bool(torch.equal(idx2, idx) and
                                                  torch.equal(val2.view(torch.int32), val.view(torch.int32)) and
                                                  st2.dispatch_count == st.dispatch_count and
                                                  st2.ledger_peak_bytes == st.ledger_peak_bytes)
                del idx2, val2
            print(json.dumps(line), flush=True)
            del idx, val
