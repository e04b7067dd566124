"""Regenerates tests/golden/golden.npz from the REFERENCE ITSELF.

Run here (where /root/reference exists) after `make -C oracle ref`:
    python tests/golden/make_golden.py
Every array below comes from oracle/_ref/libcsaidx_ref.so, i.e. the
unmodified reference sources (proj/src) behind their public C++ API. The
fixtures pin the C oracle (tests/test_oracle.py) and the GPU path
(tests/test_parity_gpu.py) without needing /root/reference at test time.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Reference  # noqa: E402

ref = Reference()
orc = Oracle()
G = {}

# synth.cpp: xoshiro256++ streams and the Box-Muller generator
for seed, stream in [(0, 0), (1, 1), (42, 2), (0xDEADBEEF, 3)]:
    G[f"xoshiro_{seed}_{stream}"] = ref.xoshiro(seed, stream, 8)
q, kc, w = ref.generate(2, 16, 4, 3, 5, 4, 77)
G["gen_q"], G["gen_kc"], G["gen_w"] = q, kc, w

# half.cpp: binary16 rounding, edge values included
vals = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, 65519.0, 65520.0, 70000.0, -1e9, 1e-8, 5.96e-8, 2.98e-8,
                 2.9802322e-08, 6.1035156e-05, 6.0975552e-05, 0.1, 1 / 3, 2049.0, 2051.0, 1e-3, -7.77e-6],
                np.float32)
rng = np.random.default_rng(5)
vals = np.concatenate([vals, rng.normal(0, 1, 100).astype(np.float32),
                       (rng.normal(0, 1, 50) * 1e-5).astype(np.float32)])
G["half_in"], G["half_out"] = vals, ref.half_round(vals)

# score.cpp / score_scalar.cpp: full tiles and a sub-tile, both modes
q, kc, w = ref.generate(2, 24, 3, 3, 5, 4, 77)
G["st_q"], G["st_kc"], G["st_w"] = q, kc, w
for fp16 in (0, 1):
    rc, out = ref.score_tile(q, kc, w, 3, 0, 0, 24, 8, fp16=bool(fp16), scalar=True)
    assert rc == 0
    G[f"st_full_fp16{fp16}"] = out
rc, out = ref.score_tile(q, kc, w, 3, 5, 2, 7, 4)
G["st_sub"] = out

# driver.cpp: materialize + chunked under several schedules and ablations
cases = [
    # (B, S, m, H, D, k, seed, cs, ct, fp16, ablation, early_exit, bool_mask)
    (1, 8, 4, 1, 1, 2, 3, 3, 1, 0, 0, 1, 0),
    (2, 48, 4, 2, 5, 3, 77, 5, 3, 0, 0, 1, 0),
    (1, 64, 4, 2, 3, 2, 42, 8, 3, 0, 0, 0, 0),
    (1, 64, 4, 2, 3, 2, 42, 8, 3, 0, 2, 1, 0),
    (1, 60, 2, 1, 2, 4, 3, 7, 5, 0, 0, 1, 1),
    (1, 32, 4, 1, 2, 4, 8, 8, 2, 0, 2, 1, 0),
    (1, 96, 4, 2, 4, 8, 9, 16, 4, 0, 1, 1, 0),
    (2, 40, 1, 3, 6, 7, 11, 9, 4, 1, 0, 1, 0),
    (1, 16, 4, 2, 3, 1000, 13, 3, 2, 0, 0, 1, 0),
]
G["drv_cases"] = np.array(cases, np.int64)
for n, (B, S, m, H, D, k, seed, cs, ct, fp16, abl, ee, bm) in enumerate(cases):
    q, kc, w = ref.generate(B, S, m, H, D, k, seed)
    rc, idx, val, stats, peak = ref.run_chunked(q, kc, w, m, k, cs, ct, fp16=bool(fp16), ablation=abl,
                                                 early_exit=bool(ee), bool_mask=bool(bm))
    assert rc == 0, (n, rc)
    G[f"drv{n}_idx"], G[f"drv{n}_val"], G[f"drv{n}_stats"] = idx, val, stats
    G[f"drv{n}_peak"] = np.array([peak], np.uint64)
    midx, mval = ref.run_materialize(q, kc, w, m, k, fp16=bool(fp16))
    G[f"drv{n}_midx"], G[f"drv{n}_mval"] = midx, mval

# V4 indexer shape at small S with bf16-representable operands (the parity
# input rule): reference materialize, the ground truth for the GPU.
q, kc, w = ref.generate(1, 512, 4, 64, 128, 64, 1)
q, kc = orc.bf16_round(q), orc.bf16_round(kc)
idx, val = ref.run_materialize(q, kc, w, 4, 64)
G["v4_idx"] = idx.astype(np.int16)
G["v4_val"] = val
rc, sc = ref.score_tile(q, kc, w, 4, 500, 0, 12, 128)
assert rc == 0
G["v4_scores_500"] = sc

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
np.savez_compressed(out, **G)
print("wrote", out, os.path.getsize(out), "bytes,", len(G), "arrays")
