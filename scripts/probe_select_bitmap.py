"""Select-kernel phase clocks: streaming select vs candidate-bitmap select (dev tool)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02568_b200.engine import Engine
from paper_2605_02568_b200._capi import check

e = Engine(0)


def pack_bits(mask):
    rows, n = mask.shape
    nw = -(-n // 128) * 4
    m = torch.zeros(rows, nw * 32, dtype=torch.int64, device=mask.device)
    m[:, :n] = mask.long()
    w = (m.view(rows, nw, 32) << torch.arange(32, device=mask.device)).sum(-1)
    w = (w + 2 ** 31) % 2 ** 32 - 2 ** 31
    return w.to(torch.int32).view(1, rows, nw)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 5


for n, k, target in [(32768, 1024, 2048), (65536, 1024, 2048), (32768, 1024, 1200), (32768, 1024, 3500)]:
    rows = 2048
    sc = torch.randn(1, rows, n, device="cuda") * 0.005
    tau = torch.quantile(sc[0, :64], 1 - target / n, dim=1).mean()
    bits = pack_bits(sc[0] >= tau)
    plain = lambda: e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    flagged = lambda: e.select_from_candidates(sc, 1, rows, n, 10 ** 9, 0, 1, k, bits)
    res = {}
    for name, fn in (("stream", plain), ("bitmap", flagged)):
        ms = timed(fn)
        probe = torch.zeros(rows * 8, dtype=torch.int64, device="cuda")
        check(e.lib.csaidx_engine_set_select_probe(e.handle, ctypes.c_void_p(probe.data_ptr())))
        e.candidate_hits(reset=True)
        v, i = fn()
        e.check()
        hits = e.candidate_hits()
        check(e.lib.csaidx_engine_set_select_probe(e.handle, None))
        res[name] = (v, i)
        c = probe.view(rows, 8).cpu().numpy().astype(np.float64)
        m = lambda a, b: (c[:, b] - c[:, a]).mean()
        print(f"n={n} k={k} flagged~{target} {name}: {ms:.3f} ms  cycles: gather {m(0,2):.0f} take {m(2,7):.0f} "
              f"sort {m(7,3):.0f} total {m(0,3):.0f} cand {c[:,6].mean():.0f} hits {hits}", flush=True)
    assert torch.equal(res["stream"][1], res["bitmap"][1])
