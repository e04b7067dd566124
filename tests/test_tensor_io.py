"""CSAT input dump (reference tensor_io.hpp / tensor_io.cpp:28-140) through
libcsaidx.so's host entry points: byte-identical files, the same parse and
the same std::runtime_error cases. The golden file was written by the
REFERENCE's own write_inputs_file (tests/golden/make_csat.py)."""
import os
import struct

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2605_02568_b200 import api
from paper_2605_02568_b200._capi import InvalidArgument, ScoreRuntimeError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_inputs.csat")
DIMS = (2, 16, 4, 3, 5, 4)  # B, S, m, H, D, k of make_csat.py (seed 77)


@pytest.fixture(scope="module")
def inputs():
    B, S, m, H, D, k = DIMS
    q, kc, w = Oracle().generate_inputs(B, S, m, H, D, 77)
    return q, kc, w, api.ProblemDims.create(*DIMS)


def test_writer_is_byte_identical_to_the_reference(tmp_path, inputs):
    q, kc, w, dims = inputs
    p = tmp_path / "mine.csat"
    n = api.write_inputs_file(p, api.IndexerInputs(q, kc, w), dims)
    gold = open(GOLDEN, "rb").read()
    assert n == len(gold) == 3 * 32 + 4 * (q.size + kc.size + w.size)
    assert open(p, "rb").read() == gold


def test_reader_parses_the_reference_file(inputs):
    q, kc, w, dims = inputs
    secs = api.scan_sections(GOLDEN)
    assert [(t, r, d) for t, r, d, _, _ in secs] == [(0, 4, (2, 16, 3, 5)), (1, 3, (2, 4, 5)), (2, 3, (2, 16, 3))]
    assert [o for *_, o in secs] == [32, 32 + 32 + 4 * q.size, 32 * 3 + 4 * (q.size + kc.size)]
    q2, kc2, w2 = api.read_inputs(GOLDEN, dims)
    for a, b in ((q2, q), (kc2, kc), (w2, w)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _corrupt(tmp_path, name, fn):
    b = bytearray(open(GOLDEN, "rb").read())
    b = fn(b)
    p = tmp_path / name
    open(p, "wb").write(bytes(b))
    return p


@pytest.mark.parametrize("name,fn,msg", [
    ("magic", lambda b: b[:1] + b"X" + b[2:], "bad magic"),
    ("version", lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported version"),
    ("rank0", lambda b: b[:9] + b"\x00" + b[10:], "bad rank"),
    ("rank5", lambda b: b[:9] + b"\x05" + b[10:], "bad rank"),
    ("zero", lambda b: b[:12] + struct.pack("<I", 0) + b[16:], "zero extent"),
    ("payload", lambda b: b[:-4], "truncated payload"),
    ("header", lambda b: b + b"CSAT", "truncated header"),
    ("empty", lambda b: b[:0], "empty stream"),
    ("second", lambda b: b[:1952] + b"XSAT" + b[1956:], "bad magic"),  # the second section's header
])
def test_malformed_files_raise_the_reference_errors(tmp_path, inputs, name, fn, msg):
    _, _, _, dims = inputs
    p = _corrupt(tmp_path, name, fn)
    with pytest.raises(ScoreRuntimeError, match=msg):  # std::runtime_error across the C-ABI
        api.read_inputs(p, dims)
    with pytest.raises(ScoreRuntimeError, match=msg):
        api.scan_sections(p)
    ref = _reference()
    if ref is not None:  # the reference's own reader says the same (this container only)
        rc, _, ref_msg = ref.read_sections_file(str(p))
        assert rc == 2 and ref_msg == "read_sections: " + msg


def _reference():
    try:
        from oracle.oracle import Reference

        return Reference()
    except Exception:  # noqa: BLE001  (oracle/_ref is built only where /root/reference exists)
        return None


def test_shape_mismatch_is_invalid_argument():
    with pytest.raises(InvalidArgument):
        api.read_inputs(GOLDEN, api.ProblemDims.create(2, 16, 4, 3, 6, 4))


def test_large_payload_round_trip(tmp_path):
    """Multi-MiB sections go through the streaming paths in one piece."""
    rng = np.random.default_rng(0)
    dims = api.ProblemDims.create(1, 4096, 4, 8, 64, 16)
    q = rng.normal(size=(1, 4096, 8, 64)).astype(np.float32)
    kc = rng.normal(size=(1, 1024, 64)).astype(np.float32)
    w = rng.normal(size=(1, 4096, 8)).astype(np.float32)
    p = tmp_path / "big.csat"
    api.write_inputs_file(p, api.IndexerInputs(q, kc, w), dims)
    q2, kc2, w2 = api.read_inputs(p, dims)
    assert np.array_equal(q2, q) and np.array_equal(kc2, kc) and np.array_equal(w2, w)
