"""Per-phase clock breakdown of the select kernel on synthetic score rows (dev tool)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02568_b200.engine import Engine
from paper_2605_02568_b200._capi import check

e = Engine(0)
for n, k, pad in [(32768, 1024, 0), (65536, 1024, 0), (262144, 1024, 0), (32768, 512, 0)]:
    rows = 2048
    ld = n + pad
    sc = torch.randn(1, rows, ld, device="cuda") * 0.005
    probe = torch.zeros(rows * 8, dtype=torch.int64, device="cuda")
    for it in range(3):
        v, i = e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for it in range(5):
        v, i = e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    ev1.record(); torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 5
    check(e.lib.csaidx_engine_set_select_probe(e.handle, ctypes.c_void_p(probe.data_ptr())))
    v, i = e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    e.check()
    check(e.lib.csaidx_engine_set_select_probe(e.handle, None))
    c = probe.view(rows, 8).cpu().numpy().astype(np.float64)
    m = lambda a, b: (c[:, b] - c[:, a]).mean()
    print(f"n={n} k={k} ld={ld}: {ms:.3f} ms ({rows*n*4/ms/1e6:.0f} GB/s) cycles: load {m(0,5):.0f} thresh {m(5,1):.0f} "
          f"stream {m(1,2):.0f} pad {m(2,7):.0f} sort {m(7,3):.0f} total {m(0,3):.0f} cand {c[:,6].mean():.0f}", flush=True)
