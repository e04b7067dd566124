"""(dev, GPU box) The score kernel's fused-select instances side by side on
one late C3 chunk (s0 = S - 2048, 2048 rows, all 65,536 keys, causal):
mode 0 (production: fp32 tile only), mode 2 (+ candidate bitmap against a
per-row tau from the sample pass, the fused pre-filter), mode 3 (+ per-32-key
group maxima, the two-level select). Each mode runs back to back for ~6 s
(the board settles at its power cap) and reports ms per launch (CUDA events),
SM clock and board power (NVML, sampled during the loop). Then the selects
that consume each mode's side output. Usage: python scripts/f2_modes.py [ncu]
(ncu: one launch per mode, for --set full captures)."""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
from paper_2605_02568_b200.engine import Engine, dims_struct

ncu = len(sys.argv) > 1 and sys.argv[1] == "ncu"
e = Engine(0)
S, m, H, D, k = 262144, 4, 64, 128, 1024
T = S // m
rows, s0 = 2048, S - 2048
dims = dims_struct(1, S, H, D, m, k)
q = e.gen_normal_bf16(rows * H * D, (1 / D) ** 0.5, 1, 1).view(1, rows, H, D)
kc = e.gen_normal_bf16(T * D, (1 / D) ** 0.5, 1, 2).view(1, T, D)
w = e.gen_normal_f32(rows * H, (1 / (D * H)) ** 0.5, 1, 3).view(1, rows, H)
# operands hold only this chunk's rows: present them as a [1, S, ...] view via
# the row layout the engine expects (q / w rows for s0.. are at the start)
qf = torch.zeros((1, S, H, D), dtype=torch.bfloat16, device="cuda")
qf[:, s0:] = q
wf = torch.zeros((1, S, H), dtype=torch.float32, device="cuda")
wf[:, s0:] = w
del q, w
stride = 16
sample = e.score_sampled(qf, kc, wf, dims, s0, rows, 0, T, stride)
tau = e.row_threshold(sample, 1, rows, T, s0, 0, m, stride, k)

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)


def sampled(fn, seconds):
    stop = threading.Event()
    clocks, power = [], []

    def poll():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
            power.append(pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000)
            time.sleep(0.05)

    fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=poll)
    th.start()
    t_end = time.time() + seconds
    n, ms = 0, 0.0
    while time.time() < t_end:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        b.synchronize()
        ms += a.elapsed_time(b)
        n += 10
    stop.set()
    th.join()
    med = lambda xs: sorted(xs)[len(xs) // 2] if xs else None
    return {"ms": ms / n, "launches": n, "sm_mhz": med(clocks), "power_w": med(power)}


modes = {
    "mode0_plain": lambda: e.score(qf, kc, wf, dims, s0, rows, 0, T, apply_mask=True),
    "mode2_prefilter_bitmap": lambda: e.score_filtered(qf, kc, wf, dims, s0, rows, 0, T, tau),
    "mode3_group_maxima": lambda: e.score_gmax(qf, kc, wf, dims, s0, rows, 0, T),
    "mode1_sample_pass_stride16": lambda: e.score_sampled(qf, kc, wf, dims, s0, rows, 0, T, stride),
}
res = {}
for name, fn in modes.items():
    if ncu:
        fn()
        torch.cuda.synchronize()
        continue
    res[name] = sampled(fn, 6.0)
    print(name, json.dumps(res[name]), flush=True)
if ncu:
    sys.exit(0)
# the consumers
sc = e.score(qf, kc, wf, dims, s0, rows, 0, T, apply_mask=True)
_, bits = e.score_filtered(qf, kc, wf, dims, s0, rows, 0, T, tau)
_, gmax = e.score_gmax(qf, kc, wf, dims, s0, rows, 0, T)
oi = torch.empty((1, rows, k), dtype=torch.int64, device="cuda")
ov = torch.empty((1, rows, k), dtype=torch.float32, device="cuda")
cons = {
    "select_final_plain": lambda: e.select_final(sc, 1, rows, T, s0, 0, m, k, oi, ov, 0),
    "select_final_from_bitmap": lambda: e.select_final(sc, 1, rows, T, s0, 0, m, k, oi, ov, 0, bits=bits),
    "select_final_two_level": lambda: e.select_final(sc, 1, rows, T, s0, 0, m, k, oi, ov, 0, gmax=gmax),
    "row_threshold_stride16": lambda: e.row_threshold(sample, 1, rows, T, s0, 0, m, stride, k),
}
for name, fn in cons.items():
    res[name] = sampled(fn, 3.0)
    print(name, json.dumps(res[name]), "cand_hits", e.candidate_hits(), flush=True)
print(json.dumps(res))
