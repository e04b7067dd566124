"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracle.

* ``Oracle`` binds liboracle.so, the C restatement of the reference algorithm
  (csaidx_oracle.c; each function cites the reference lines it follows).
* ``Reference`` binds _ref/libcsaidx_ref.so, the reference library itself
  compiled from /root/reference/proj/src (oracle/Makefile) plus ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int64, c_uint16, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcsaidx_ref.so")


def _p(a):
    return c_void_p(a.ctypes.data)


class Oracle:
    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle` (build() does this)")
        L = ctypes.CDLL(path)
        self.L = L
        L.orc_splitmix64.restype = c_uint64
        L.orc_splitmix64.argtypes = [POINTER(c_uint64)]
        L.orc_fill_gaussian.argtypes = [c_void_p, c_int64, c_double, c_uint64, c_uint64]
        L.orc_generate_inputs.argtypes = [c_int64] * 5 + [c_uint64, c_void_p, c_void_p, c_void_p]
        L.orc_bf16_round.restype = c_float
        L.orc_bf16_round.argtypes = [c_float]
        L.orc_bf16_round_array.argtypes = [c_void_p, c_int64]
        L.orc_half_round.restype = c_float
        L.orc_half_round.argtypes = [c_float]
        L.orc_float_to_half_bits.restype = c_uint16
        L.orc_float_to_half_bits.argtypes = [c_float]
        L.orc_t_legal.restype = c_int64
        L.orc_t_legal.argtypes = [c_int64, c_int64]
        L.orc_k_eff.restype = c_int64
        L.orc_k_eff.argtypes = [c_int64, c_int64, c_int64]
        L.orc_score_tile.argtypes = [c_void_p] * 3 + [c_int64] * 9 + [c_int, c_void_p]
        L.orc_oracle_topk.restype = c_int64
        L.orc_oracle_topk.argtypes = [c_void_p, c_int64, c_int64, c_void_p, c_void_p]
        L.orc_run_materialize.argtypes = [c_void_p] * 3 + [c_int64] * 6 + [c_int, c_void_p, c_void_p]
        L.orc_run_chunked.restype = c_int
        L.orc_run_chunked.argtypes = [c_void_p] * 3 + [c_int64] * 8 + [c_int, c_int, c_int, c_void_p, c_void_p,
                                                                       c_void_p]
        L.orc_row_topk.restype = c_int64
        L.orc_row_topk.argtypes = [c_void_p] * 3 + [c_int64] * 5 + [c_void_p, c_void_p]
        L.orc_score_rows.argtypes = [c_void_p] * 5 + [c_int64] * 3 + [c_int, c_void_p]
        L.orc_recall.restype = c_int64
        L.orc_recall.argtypes = [c_void_p, c_void_p, c_int64, c_int64] + [POINTER(c_double)] * 4

    # -- synth
    def splitmix64(self, state: int, n: int):
        s = c_uint64(state)
        return [self.L.orc_splitmix64(ctypes.byref(s)) for _ in range(n)]

    def fill_gaussian(self, n, stddev, seed, stream):
        out = np.empty(n, np.float32)
        self.L.orc_fill_gaussian(_p(out), n, stddev, seed, stream)
        return out

    def generate_inputs(self, B, S, m, H, D, seed, bf16=False):
        T = S // m
        q = np.empty((B, S, H, D), np.float32)
        kc = np.empty((B, T, D), np.float32)
        w = np.empty((B, S, H), np.float32)
        self.L.orc_generate_inputs(B, S, m, H, D, seed, _p(q), _p(kc), _p(w))
        if bf16:
            self.L.orc_bf16_round_array(_p(q), q.size)
            self.L.orc_bf16_round_array(_p(kc), kc.size)
        return q, kc, w

    def bf16_round(self, x: np.ndarray) -> np.ndarray:
        y = np.ascontiguousarray(x, np.float32).copy()
        self.L.orc_bf16_round_array(_p(y), y.size)
        return y

    def half_round(self, x: float) -> float:
        return self.L.orc_half_round(x)

    def t_legal(self, t, m):
        return self.L.orc_t_legal(t, m)

    def k_eff(self, t, m, k):
        return self.L.orc_k_eff(t, m, k)

    # -- scoring / selection
    def score_tile(self, q, kc, w, s0, t0, rows, cols, fp16=False):
        B, S, H, D = q.shape
        T = kc.shape[1]
        out = np.empty((B, rows, cols), np.float32)
        self.L.orc_score_tile(_p(q), _p(kc), _p(w), B, S, T, H, D, s0, t0, rows, cols, int(fp16), _p(out))
        return out

    def score_rows(self, q_rows, w_rows, kc, kc_row0, legal, threads=None):
        """Full causal rows in the reference op order (orc_score_rows):
        q_rows [n, H, D], w_rows [n, H], kc [rows, D] (row r uses keys
        kc[kc_row0[r] : kc_row0[r] + legal[r]]). Returns a list of 1-D score
        arrays (views into one buffer)."""
        q_rows = np.ascontiguousarray(q_rows, np.float32)
        w_rows = np.ascontiguousarray(w_rows, np.float32)
        kc = np.ascontiguousarray(kc, np.float32)
        n, H, D = q_rows.shape
        r0 = np.ascontiguousarray(kc_row0, np.int64)
        lg = np.ascontiguousarray(legal, np.int64)
        assert r0.shape == (n,) and lg.shape == (n,) and w_rows.shape == (n, H)
        assert np.all(r0 + lg <= kc.shape[0])
        out = np.empty(max(int(lg.sum()), 1), np.float32)
        self.L.orc_score_rows(_p(q_rows), _p(w_rows), _p(kc), _p(r0), _p(lg), n, H, D,
                              int(threads or os.cpu_count() or 1), _p(out))
        off = np.concatenate([[0], np.cumsum(lg)])
        return [out[off[i]:off[i + 1]] for i in range(n)]

    def oracle_topk(self, row: np.ndarray, k: int, legal: int):
        row = np.ascontiguousarray(row, np.float32)
        v = np.empty(max(k, 1), np.float32)
        i = np.empty(max(k, 1), np.int64)
        n = self.L.orc_oracle_topk(_p(row), legal, k, _p(v), _p(i))
        return v[:n], i[:n]

    def run_materialize(self, q, kc, w, m, k, fp16=False):
        B, S, H, D = q.shape
        idx = np.empty((B, S, k), np.int64)
        val = np.empty((B, S, k), np.float32)
        self.L.orc_run_materialize(_p(q), _p(kc), _p(w), B, S, m, H, D, k, int(fp16), _p(idx), _p(val))
        return idx, val

    def run_chunked(self, q, kc, w, m, k, cs, ct, fp16=False, ablation=0, early_exit=True):
        B, S, H, D = q.shape
        idx = np.empty((B, S, k), np.int64)
        val = np.empty((B, S, k), np.float32)
        stats = np.zeros(3, np.int64)
        rc = self.L.orc_run_chunked(_p(q), _p(kc), _p(w), B, S, m, H, D, k, cs, ct, int(fp16), ablation,
                                    int(early_exit), _p(idx), _p(val), _p(stats))
        return rc, idx, val, stats

    def row_topk(self, q_row, w_row, kc_b, legal, k):
        H, D = q_row.shape
        T = kc_b.shape[0]
        v = np.empty(max(k, 1), np.float32)
        i = np.empty(max(k, 1), np.int64)
        n = self.L.orc_row_topk(_p(np.ascontiguousarray(q_row)), _p(np.ascontiguousarray(w_row)),
                                _p(np.ascontiguousarray(kc_b)), T, H, D, legal, k, _p(v), _p(i))
        return v[:n], i[:n]

    def recall(self, ref_idx, test_idx):
        k = ref_idx.shape[-1]
        n = ref_idx.size // k
        a = np.ascontiguousarray(ref_idx, np.int64)
        b = np.ascontiguousarray(test_idx, np.int64)
        mean, mn, perf, below = c_double(), c_double(), c_double(), c_double()
        rows = self.L.orc_recall(_p(a), _p(b), n, k, ctypes.byref(mean), ctypes.byref(mn), ctypes.byref(perf),
                                 ctypes.byref(below))
        return {"rows_evaluated": rows, "mean": mean.value, "min": mn.value, "pct_perfect": perf.value,
                "pct_below_99": below.value}


class Reference:
    """The reference library itself (oracle/_ref), for pinning and the CPU baseline."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(path)
        self.L = L
        L.ref_generate.argtypes = [c_int64] * 6 + [c_uint64, c_void_p, c_void_p, c_void_p]
        L.ref_xoshiro.argtypes = [c_uint64, c_uint64, c_int, c_void_p]
        L.ref_half_round.argtypes = [c_void_p, c_int64, c_void_p]
        L.ref_score_tile.argtypes = [c_void_p] * 3 + [c_int64] * 9 + [c_int, c_int, c_void_p]
        L.ref_run_materialize.argtypes = [c_void_p] * 3 + [c_int64] * 6 + [c_int, c_void_p, c_void_p, c_void_p]
        L.ref_run_chunked.argtypes = [c_void_p] * 3 + [c_int64] * 8 + [c_int] * 5 + [c_void_p] * 4
        L.ref_dispatch_count_model.restype = c_int64
        L.ref_dispatch_count_model.argtypes = [c_int64] * 4
        L.ref_chunked_peak_model_bytes.restype = c_uint64
        L.ref_chunked_peak_model_bytes.argtypes = [c_int64] * 4 + [c_int]
        L.ref_sample_chunked.argtypes = [c_int64] * 8 + [c_int, c_uint64, POINTER(c_double), POINTER(c_double)]
        L.ref_write_inputs_file.argtypes = [ctypes.c_char_p] + [c_void_p] * 3 + [c_int64] * 6 + [POINTER(c_uint64)]
        L.ref_read_sections_file.argtypes = [ctypes.c_char_p, POINTER(c_int), ctypes.c_char_p, c_int]

    def generate(self, B, S, m, H, D, k, seed):
        T = S // m
        q = np.empty((B, S, H, D), np.float32)
        kc = np.empty((B, T, D), np.float32)
        w = np.empty((B, S, H), np.float32)
        assert self.L.ref_generate(B, S, m, H, D, k, seed, _p(q), _p(kc), _p(w)) == 0
        return q, kc, w

    def xoshiro(self, seed, stream, n):
        out = np.empty(n, np.uint64)
        assert self.L.ref_xoshiro(seed, stream, n, _p(out)) == 0
        return out

    def half_round(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        assert self.L.ref_half_round(_p(x), x.size, _p(out)) == 0
        return out

    def score_tile(self, q, kc, w, m, s0, t0, rows, cols, fp16=False, scalar=False):
        B, S, H, D = q.shape
        out = np.empty((B, rows, cols), np.float32)
        rc = self.L.ref_score_tile(_p(q), _p(kc), _p(w), B, S, m, H, D, s0, t0, rows, cols, int(fp16), int(scalar),
                                   _p(out))
        return rc, out

    def run_materialize(self, q, kc, w, m, k, fp16=False):
        B, S, H, D = q.shape
        idx = np.empty((B, S, k), np.int64)
        val = np.empty((B, S, k), np.float32)
        peak = np.zeros(1, np.uint64)
        rc = self.L.ref_run_materialize(_p(q), _p(kc), _p(w), B, S, m, H, D, k, int(fp16), _p(idx), _p(val),
                                        _p(peak))
        assert rc == 0, rc
        return idx, val

    def run_chunked(self, q, kc, w, m, k, cs, ct, fp16=False, ablation=0, early_exit=True, bool_mask=False,
                    threads=1):
        B, S, H, D = q.shape
        idx = np.empty((B, S, k), np.int64)
        val = np.empty((B, S, k), np.float32)
        stats = np.zeros(3, np.int64)
        peak = np.zeros(1, np.uint64)
        rc = self.L.ref_run_chunked(_p(q), _p(kc), _p(w), B, S, m, H, D, k, cs, ct, int(fp16), ablation,
                                    int(early_exit), int(bool_mask), threads, _p(idx), _p(val), _p(stats),
                                    _p(peak))
        return rc, idx, val, stats, int(peak[0])

    def write_inputs_file(self, path, q, kc, w, m, k):
        """tensor_io.cpp write_inputs_file: the reference's CSAT dump of (q, kc, w)."""
        B, S, H, D = q.shape
        n = c_uint64(0)
        rc = self.L.ref_write_inputs_file(path.encode(), _p(q), _p(kc), _p(w), B, S, m, H, D, k, ctypes.byref(n))
        return rc, n.value

    def read_sections_file(self, path):
        """tensor_io.cpp read_sections on a file -> (rc, n_sections, runtime_error message)."""
        n = c_int(0)
        msg = ctypes.create_string_buffer(256)
        rc = self.L.ref_read_sections_file(os.fsencode(path), ctypes.byref(n), msg, 256)
        return rc, n.value, msg.value.decode()

    def sample_chunked(self, S, m, H, D, k, cs, ct, n_tiles, threads, seed=1):
        sec, pairs = c_double(), c_double()
        rc = self.L.ref_sample_chunked(S, m, H, D, k, cs, ct, n_tiles, threads, seed, ctypes.byref(sec),
                                       ctypes.byref(pairs))
        assert rc == 0, rc
        return sec.value, pairs.value
