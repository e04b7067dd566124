"""Pins the C oracle (oracle/csaidx_oracle.c) before anything trusts it.

(a) Known-answer vectors copied from the reference's own tests (cited).
(b) Golden fixtures produced by the reference library itself
    (tests/golden/make_golden.py over oracle/_ref): bit-exact equality.
CPU only.
"""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
NEG_INF = np.float32(-np.inf)


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------------ KATs

def test_splitmix_published_vector(orc):
    # test_synth.cpp:62-69
    assert orc.splitmix64(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_t_legal_and_k_eff_examples(orc):
    # test_causal.cpp:34-43 and 60-66
    assert [orc.t_legal(t, 4) for t in (0, 1, 2, 3, 4, 7)] == [0, 0, 0, 1, 1, 2]
    assert orc.t_legal(5, 1) == 6 and orc.t_legal(0, 1) == 1
    assert orc.k_eff(0, 4, 512) == 0 and orc.k_eff(100, 4, 512) == 25
    assert orc.k_eff(4095, 4, 512) == 512 and orc.k_eff(4095, 4, 2000) == 1024 and orc.k_eff(3, 1, 2) == 2


def test_hand_computed_scores(orc):
    # test_score.cpp:54-76
    one = lambda q, kc, w, H, D: orc.score_tile(np.array(q, np.float32).reshape(1, 1, H, D),
                                                np.array(kc, np.float32).reshape(1, 1, D),
                                                np.array(w, np.float32).reshape(1, 1, H), 0, 0, 1, 1)[0, 0, 0]
    assert one([1, -2], [1, 1], [3], 1, 2) == 0.0
    assert one([1, 1], [1, 1], [0.5], 1, 2) == 1.0
    assert one([3, 2], [1], [1, -1], 2, 1) == 1.0


def test_fp16_saturates(orc):
    # test_score.cpp:162-175: emulated mode saturates at 65504
    q = np.full((1, 1, 1, 2), 3.0e38, np.float32)
    kc = np.full((1, 1, 2), 3.0e38, np.float32)
    w = np.ones((1, 1, 1), np.float32)
    assert orc.score_tile(q, kc, w, 0, 0, 1, 1, fp16=True)[0, 0, 0] == 65504.0
    assert not np.isfinite(orc.score_tile(q, kc, w, 0, 0, 1, 1)[0, 0, 0])


def test_oracle_topk_examples(orc):
    # test_topk.cpp:87-93 (tie at 5 resolves to index 0) via a dense row
    v, i = orc.oracle_topk(np.array([5, 3, 5, 9], np.float32), 2, 4)
    assert list(i) == [3, 0] and list(v) == [9, 5]
    assert orc.oracle_topk(np.array([1, 2], np.float32), 3, 0)[1].size == 0  # test_topk.cpp:277


def test_ramp_driver_pinned_by_hand(orc):
    # test_driver.cpp:37-64: one head, one dim, unit q and w: score(t, j) = kc[j]
    q = np.ones((1, 8, 1, 1), np.float32)
    w = np.ones((1, 8, 1), np.float32)
    kc = np.array([1.0, 2.0], np.float32).reshape(1, 2, 1)
    rc, idx, val, _ = orc.run_chunked(q, kc, w, 4, 2, 3, 1)
    assert rc == 0
    assert np.all(idx[0, :3] == -1)
    assert np.all(idx[0, 3:7, 0] == 0) and np.all(val[0, 3:7, 0] == 1.0) and np.all(idx[0, 3:7, 1] == -1)
    assert list(idx[0, 7]) == [1, 0] and list(val[0, 7]) == [2.0, 1.0]
    midx, mval = orc.run_materialize(q, kc, w, 4, 2)
    assert np.array_equal(midx, idx) and np.array_equal(bits(mval), bits(val))


def test_a1_keeps_last_tile(orc):
    # test_driver.cpp:175-195
    q = np.ones((1, 8, 1, 1), np.float32)
    w = np.ones((1, 8, 1), np.float32)
    kc = np.array([2.0, 1.0], np.float32).reshape(1, 2, 1)
    _, prod, _, _ = orc.run_chunked(q, kc, w, 4, 1, 8, 1)
    _, a1, _, _ = orc.run_chunked(q, kc, w, 4, 1, 8, 1, ablation=1)
    assert prod[0, 7, 0] == 0 and a1[0, 7, 0] == 1
    assert np.all(prod[0, 3:7, 0] == 0) and np.all(a1[0, 3:7, 0] == -1)


def test_sentinel_contract_exhaustive(orc):
    # test_driver.cpp:197-233
    for m in (1, 2, 4):
        for k in (1, 2, 1000):
            S = 4 * m
            q, kc, w = orc.generate_inputs(1, S, m, 2, 3, m * 1000 + k)
            for cs, ct in ((S, S // m), (1, 1), (3, 2)):
                rc, idx, val, _ = orc.run_chunked(q, kc, w, m, k, cs, ct)
                assert rc == 0
                for t in range(S):
                    want = orc.k_eff(t, m, k)
                    assert np.all(idx[0, t, :want] >= 0) and np.all(idx[0, t, :want] < orc.t_legal(t, m))
                    assert np.all(idx[0, t, want:] == -1) and np.all(val[0, t, want:] == NEG_INF)


# ------------------------------------------------------- golden fixtures

def test_generator_matches_reference(orc, gold):
    q, kc, w = orc.generate_inputs(2, 16, 4, 3, 5, 77)
    assert np.array_equal(bits(q), bits(gold["gen_q"]))
    assert np.array_equal(bits(kc), bits(gold["gen_kc"]))
    assert np.array_equal(bits(w), bits(gold["gen_w"]))


def test_half_round_matches_reference(orc, gold):
    got = np.array([orc.half_round(float(x)) for x in gold["half_in"]], np.float32)
    assert np.array_equal(bits(got), bits(gold["half_out"]))


def test_score_tile_matches_reference_bits(orc, gold):
    q, kc, w = gold["st_q"], gold["st_kc"], gold["st_w"]
    for fp16 in (0, 1):
        got = orc.score_tile(q, kc, w, 0, 0, 24, 8, fp16=bool(fp16))
        assert np.array_equal(bits(got), bits(gold[f"st_full_fp16{fp16}"]))
    assert np.array_equal(bits(orc.score_tile(q, kc, w, 5, 2, 7, 4)), bits(gold["st_sub"]))


def test_driver_cases_match_reference(orc, gold):
    for n, (B, S, m, H, D, k, seed, cs, ct, fp16, abl, ee, bm) in enumerate(gold["drv_cases"]):
        q, kc, w = orc.generate_inputs(B, S, m, H, D, seed)
        rc, idx, val, stats = orc.run_chunked(q, kc, w, m, k, cs, ct, fp16=bool(fp16), ablation=int(abl),
                                              early_exit=bool(ee))
        assert rc == 0
        assert np.array_equal(idx, gold[f"drv{n}_idx"]), n
        assert np.array_equal(bits(val), bits(gold[f"drv{n}_val"])), n
        assert np.array_equal(stats, gold[f"drv{n}_stats"]), n
        midx, mval = orc.run_materialize(q, kc, w, m, k, fp16=bool(fp16))
        assert np.array_equal(midx, gold[f"drv{n}_midx"]), n
        assert np.array_equal(bits(mval), bits(gold[f"drv{n}_mval"])), n


def test_v4_shape_materialize_matches_reference(orc, gold):
    q, kc, w = orc.generate_inputs(1, 512, 4, 64, 128, 1, bf16=True)
    idx, val = orc.run_materialize(q, kc, w, 4, 64)
    assert np.array_equal(idx.astype(np.int16), gold["v4_idx"])
    assert np.array_equal(bits(val), bits(gold["v4_val"]))
    assert np.array_equal(bits(orc.score_tile(q, kc, w, 500, 0, 12, 128)), bits(gold["v4_scores_500"]))


def test_recall_scorer(orc, gold):
    idx = gold["drv1_idx"]
    r = orc.recall(idx, idx)
    assert r["mean"] == 1.0 and r["min"] == 1.0 and r["pct_perfect"] == 100.0
    broken = idx.copy()
    broken[0, -1, 0] = 10 ** 6
    assert orc.recall(idx, broken)["min"] < 1.0


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                                    "libcsaidx_ref.so")), reason="reference library not built")
def test_oracle_equals_live_reference_on_random_instances(orc):
    from oracle.oracle import Reference

    ref = Reference()
    rng = np.random.default_rng(2024)
    for trial in range(25):
        m = int(2 ** rng.integers(0, 3))
        T = int(rng.integers(1, 24))
        B, H, D = int(rng.integers(1, 3)), int(rng.integers(1, 4)), int(rng.integers(1, 7))
        k = int(rng.integers(1, 2 * T + 1))
        S = m * T
        q, kc, w = ref.generate(B, S, m, H, D, k, 500 + trial)
        cs, ct = int(rng.integers(1, S + 1)), int(rng.integers(1, T + 3))
        abl = int(rng.integers(0, 3))
        rc, ridx, rval, rst, _ = ref.run_chunked(q, kc, w, m, k, cs, ct, ablation=abl)
        orc_rc, oidx, oval, ost = orc.run_chunked(q, kc, w, m, k, cs, ct, ablation=abl)
        assert rc == orc_rc == 0
        assert np.array_equal(ridx, oidx) and np.array_equal(bits(rval), bits(oval)) and np.array_equal(rst, ost)
