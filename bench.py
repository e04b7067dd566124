#!/usr/bin/env python
"""Benchmark of the CSA lightning-indexer step on B200 (one JSON line).

Metric (BASELINE.json): indexer query·key pairs/sec (+ peak HBM), V4-Flash.
Default workload = C3: B=1, S=262,144 (T=65,536), H_I=64, d_h=128, m=4,
k=1024, c_S=2048, query-sharded over the N GPUs of one node (strong scaling:
the same problem at every N). One "step" = the full indexer step over the
whole instance: K broadcast (N>1) -> score/mask/select/merge for every
query chunk -> gather of the [S, k] index output to rank 0 (N>1).

* value  — legal (causal) query·key pairs per second, whole job, operands
           resident in HBM (bf16 q/kc generated on device), max over ranks.
* e2e    — the same metric through the reference-facing host API
           (csaidx_host_run_chunked_local: the rank's rows of q / w) from
           pinned fp32 host buffers, H2D of q/kc/w and D2H of indices+values
           inside the timed region.
* roofline — score kernel (tcgen05): algorithmic FLOPs (16,384 per legal
           pair) / event-timed kernel ms, vs MEASURED_PEAKS.json.
* cpu_baseline — the reference C++ library (oracle/_ref, compiled from the
           reference sources) on this host's cores, bounded sample.

`--impl reference` times that reference CPU path alone (rank 0).
`--simulate-rank R/N` measures rank R's exact shard of an N-GPU run on one
GPU; `--backend gloo` runs the N>1 path with several ranks on one GPU (a
logic check; collectives staged through host memory).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (B, S, H, D, m, k, c_S, c_T or None=T)
    "c1": (1, 4096, 64, 128, 4, 512, 2048, None),
    "c2": (1, 65536, 64, 128, 4, 512, 2048, None),
    "c3": (1, 262144, 64, 128, 4, 1024, 2048, None),
    "c4": (1, 1048576, 64, 128, 4, 1024, 1024, None),  # c_S=1024: rank 0 stays < 10 GB with the gathered [S,k]
    "c5": (2, 131072, 64, 128, 4, 1024, 2048, None),
}
FLOPS_PER_PAIR = 2 * 64 * 128


def legal_pairs_rows(S, m, starts, cs, T):
    tot = 0
    for s0 in starts:
        t = np.arange(s0, min(s0 + cs, S), dtype=np.int64)
        tot += int(np.minimum((t + 1) // m, T).sum())
    return tot


def shard_chunks(S, m, cs, world, rank):
    """LPT assignment of c_S chunks by causal work (paper_2605_02568_b200/shard.py)."""
    from paper_2605_02568_b200.shard import plan_shards

    shards, loads = plan_shards(S, m, cs, world)
    return shards[rank], loads, shards


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks, board power and throttle reasons sampled during the timed
    region: an NVML thread every 20 ms (no process start-up latency, so short
    regions get samples too); nvidia-smi -lms 100 when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None
        self.thread = None
        self.rows = []

    def start(self):
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # the CUDA ordinal's own board (CUDA_VISIBLE_DEVICES may renumber)
                import torch
                pr = torch.cuda.get_device_properties(self.device)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.stop_evt = threading.Event()

            def poll():
                while True:
                    try:
                        self.rows.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx,
                                          pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0, int(reasons_fn(h))))
                    except Exception:
                        pass
                    if self.stop_evt.wait(0.02):
                        break

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join(timeout=5)
            rows = self.rows
            if not rows:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            reasons = sorted({n for r in rows for n, bit in self.REASONS.items() if r[3] & bit})
            return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                    "power_w": statistics.median(r[2] for r in rows), "reasons": reasons, "samples": len(rows),
                    "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w": statistics.median(pw) if pw else None, "reasons": reasons, "samples": len(rows),
                "source": "nvidia-smi"}


def cpu_baseline(S, m, H, D, k, budget_s=15.0):
    """The reference library (oracle/_ref) on this host: process_query_tile's
    engine sequence over a deterministic sample of query tiles."""
    from oracle.oracle import Reference

    ref = Reference()
    threads = os.cpu_count() or 1
    cs, ct = 64, 1024
    sec, pairs = ref.sample_chunked(S, m, H, D, k, cs, ct, threads, threads)
    rate = pairs / max(sec, 1e-9)
    avg_tile = pairs / threads
    n_tiles = int(max(threads, min(threads * 64, budget_s * rate / max(avg_tile, 1.0))))
    sec, pairs = ref.sample_chunked(S, m, H, D, k, cs, ct, n_tiles, threads)
    return {"value": pairs / sec, "unit": "legal pairs/s", "cores": threads, "kind": "reference",
            "sample": f"{n_tiles} query tiles of c_S={cs} (c_T={ct}) spread evenly over t of S={S}, full causal "
                      f"key range each; {pairs:.3e} legal pairs in {sec:.1f} s (reference run_chunked engine "
                      f"sequence, std::thread x{threads})"}


def run_reference_arm(args, wl):
    B, S, H, D, m, k, cs, ct = wl
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import Reference

    ref = Reference()
    threads = os.cpu_count() or 1
    n_tiles = threads * 2
    samples = []
    for i in range(args.warmup + args.steps):
        sec, pairs = ref.sample_chunked(S, m, H, D, k, 64, 1024, n_tiles, threads, seed=1 + i)
        if i >= args.warmup:
            samples.append((sec, pairs))
    sec = sum(s for s, _ in samples)
    pairs = sum(p for _, p in samples)
    value = pairs / sec
    line = {
        "impl": "reference", "metric": "indexer query·key pairs/sec (legal causal pairs)", "value": value,
        "unit": "legal pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sec / max(len(samples), 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator)",
        "config": {"workload": args.workload, "B": B, "S": S, "H_I": H, "d_h": D, "m": m, "k": k},
        "cpu_baseline": {"value": value, "unit": "legal pairs/s", "cores": threads, "kind": "reference",
                         "sample": f"per step {n_tiles} query tiles of c_S=64 (c_T=1024) spread over t of S={S}"},
        "e2e": {"value": value, "unit": "legal pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--cs", type=int, default=None)
    ap.add_argument("--ct", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: how rank 0 collects the index rows (peer stores from the select, or a collective "
                         "gather after the compute)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no e2e/baseline)")
    ap.add_argument("--simulate-rank", default=None, metavar="R/N",
                    help="measure rank R's shard of an N-GPU run on this one GPU (per-rank numbers)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: logic check of the N>1 path with several ranks on one GPU")
    args = ap.parse_args()
    wl = list(WORKLOADS[args.workload])
    if args.cs:
        wl[6] = args.cs
    if args.ct:
        wl[7] = args.ct
    if args.impl == "reference":
        return run_reference_arm(args, wl)

    import torch
    import torch.distributed as dist

    from paper_2605_02568_b200 import _capi, api
    from paper_2605_02568_b200.engine import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())  # gloo check: ranks share GPU 0
    torch.cuda.set_device(local)
    backend = args.backend
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # logic check of the N>1 path on one GPU (collectives staged through host memory)
            dist.init_process_group("gloo")
    stream = torch.cuda.Stream()  # all timed work and its events live on this stream
    torch.cuda.set_stream(stream)

    B, S, H, D, m, k, cs, ct = wl
    T = S // m
    ct = ct or T
    cfg = api.DriverConfig(tile=api.TileConfig(cs, ct), device=local, stream=stream.cuda_stream)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    # --simulate-rank R/N: one process measures rank R's shard of an N-way run
    plan_world, plan_rank = world, rank
    if args.simulate_rank:
        plan_rank, plan_world = (int(x) for x in args.simulate_rank.split("/"))
        assert world == 1 and 0 <= plan_rank < plan_world
    mine, loads, shards = shard_chunks(S, m, cs, plan_world, plan_rank)
    rows = api.chunk_rows(dims, cfg, mine)
    pairs_total = B * legal_pairs_rows(S, m, range(0, S, cs), cs, T)
    pairs_mine = B * legal_pairs_rows(S, m, mine, cs, T)

    # ------------------------------------------------- operands in HBM (rank-local)
    # Each rank generates only its own chunks' q / w rows (the counter-based
    # generator is indexed by the global element, so the values equal those
    # of a full-size draw) and keeps them as a local stack in chunk order.
    eng = Engine(local)

    def local_stack(per_row, stddev, stream_id, bf16):
        gen = eng.gen_normal_bf16 if bf16 else eng.gen_normal_f32
        parts = []
        for b in range(B):
            for s0 in mine:
                n = min(cs, S - s0)
                parts.append(gen(n * per_row, stddev, 1, stream_id, (b * S + s0) * per_row))
        return torch.cat(parts)

    q = local_stack(H * D, D ** -0.5, 1, True)
    w = local_stack(H, (D * H) ** -0.5, 3, False)
    if rank == 0:
        kc = eng.gen_normal_bf16(B * T * D, D ** -0.5, 1, 2)
    else:
        kc = torch.empty(B * T * D, dtype=torch.bfloat16, device="cuda")
    # Output rows. A query-sharded rank (N > 1, or --simulate-rank 0/N)
    # keeps no int64 / fp32 rows of its own: the final kernels store the
    # int32 index rows into rank 0's [B, S, k] buffer and nothing else
    # (north_star: only the [S, k] index output is collected); the local rows
    # are produced once after the timed region for the correctness checks.
    sink_only = world > 1 or (args.simulate_rank is not None and plan_rank == 0 and plan_world > 1)
    out_idx = out_val = None
    if not sink_only:
        out_idx = torch.empty((B, rows, k), dtype=torch.int64, device="cuda")
        out_val = torch.empty((B, rows, k), dtype=torch.float32, device="cuda")
    # N > 1: the library's query-sharded driver (csaidx_multi_*, C++
    # csaidx::gpu::MultiRank) runs the step: kc broadcast from rank 0 over
    # the transport (NCCL, or gloo for the one-GPU logic check), this rank's
    # chunks, and the int32 [B, S, k] index rows into rank 0's buffer — stored
    # there by the final select kernels over a CUDA IPC peer mapping
    # (--gather p2p, default) or gathered after the compute (--gather nccl).
    drv_h = api.driver_engine(local)
    mr = sink = comm = None
    p2p = False
    if world == 1 and sink_only:  # --simulate-rank 0/N: rank 0's [B, S, k] int32 result buffer
        sink = torch.full((B, S, k), -2, dtype=torch.int32, device="cuda")
    if world > 1:
        from paper_2605_02568_b200 import multi

        if backend == "nccl":
            uid = [multi.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = multi.NcclCollectives(rank, world, uid[0], local)
        else:
            comm = multi.TorchCollectives()
        if rank == 0:
            sink = torch.full((B, S, k), -2, dtype=torch.int32, device="cuda")
        mode = multi.GATHER_PEER if args.gather == "p2p" else multi.GATHER_COLLECTIVE
        try:
            mr = multi.MultiRank(comm, dims, cfg, mode, sink)
            ok = True
        except Exception as ex:  # no CUDA IPC / peer access: the collective gather
            print(f"rank {rank}: peer index sink unavailable ({ex}); using the collective gather", file=sys.stderr)
            ok = False
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if not all(oks):
            if mr is not None:
                mr.close()
            mode = multi.GATHER_COLLECTIVE
            mr = multi.MultiRank(comm, dims, cfg, mode, sink)
        p2p = mode == multi.GATHER_PEER
        assert mr.chunks == mine and mr.rows == rows
    torch.cuda.synchronize()

    def bcast(t):
        if backend == "nccl":
            dist.broadcast(t, src=0)
        else:
            h = t.cpu()
            dist.broadcast(h, src=0)
            t.copy_(h)

    stats_box = {}

    def step():
        if mr is not None:
            st = mr.run(q, kc, w, out_idx, out_val)
        elif sink is not None:
            api.set_index_sink(drv_h, sink.data_ptr(), B, S, k)
            try:
                st = api.run_chunked_device(q, kc, w, dims, cfg, mine, local_rows=True, outputs=False)[2]
            finally:
                api.set_index_sink(drv_h, None)
        else:
            st = api.run_chunked_device(q, kc, w, dims, cfg, mine, out_idx, out_val, local_rows=True)[2]
        stats_box["st"] = st

    drv = api.KernelStats(drv_h)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.reset_peak_memory_stats()
    drv.reset()
    drv.select_fallbacks(reset=True)
    drv.candidate_hits(reset=True)
    drv.profiling(True)
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    drv.profiling(False)
    # everything the line reports about the timed steps, before any untimed check runs
    kinds = {"score": _capi.KIND_SCORE, "select": _capi.KIND_SELECT, "merge": _capi.KIND_MERGE,
             "finalize": _capi.KIND_FINALIZE, "prep": _capi.KIND_PREP}
    kstats = {name: drv.get(kd) for name, kd in kinds.items()}
    _, drv_peak = drv.mem()
    fallbacks = drv.select_fallbacks()
    cand_hits = drv.candidate_hits()
    hbm_peak = torch.cuda.max_memory_allocated() + drv_peak
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            t = h
        ms = float(t.item())
    gather_ok = None
    if sink_only:  # this rank's own rows, once, for the checks below (untimed)
        out_idx = torch.empty((B, rows, k), dtype=torch.int64, device="cuda")
        out_val = torch.empty((B, rows, k), dtype=torch.float32, device="cuda")
        api.run_chunked_device(q, kc, w, dims, cfg, mine, out_idx, out_val, local_rows=True)
        if world == 1:
            own = np.concatenate([np.arange(s0, min(s0 + cs, S)) for s0 in mine])
            gather_ok = bool(np.array_equal(sink[:, own].cpu().numpy(), out_idx.cpu().numpy().astype(np.int32)))
    if world > 1:
        # untimed check: rank 0's buffer holds every rank's rows (per-rank
        # checksums over each shard's rows), its own rows bit for bit, and no
        # row was left unwritten
        torch.cuda.synchronize()
        mine_sum = int(out_idx.sum().item())
        sums = [None] * world
        dist.all_gather_object(sums, mine_sum)
        if rank == 0:
            full = sink.cpu().numpy()
            ok = full.min() >= -1 and full.max() < T
            for r in range(world):
                rows_r = np.concatenate([np.arange(s0, min(s0 + cs, S)) for s0 in shards[r]])
                ok = ok and int(full[:, rows_r].astype(np.int64).sum()) == sums[r]
            own = np.concatenate([np.arange(s0, min(s0 + cs, S)) for s0 in mine])
            ok = ok and np.array_equal(full[:, own], out_idx.cpu().numpy().astype(np.int32))
            gather_ok = bool(ok)
        dist.barrier()
    launches = sum(n for n, _ in kstats.values())
    score_n, score_ms = kstats["score"]
    peaks, peak_src = load_peaks()
    score_flops = pairs_mine * FLOPS_PER_PAIR * args.steps
    achieved_tflops = score_flops / (score_ms / 1000.0) / 1e12 if score_ms > 0 else None
    peak_tflops = peaks["bf16_tflops_sustained"]
    traffic = sel_traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f).get(args.workload, {})
            traffic = tj.get("score_dram_bytes_per_launch")
            sel_traffic = tj.get("select_dram_bytes_per_launch")
    sel_n, sel_ms = kstats["select"]
    select_gbs = (pairs_mine * 4 * args.steps) / (sel_ms / 1000.0) / 1e9 if sel_ms > 0 else None
    st = stats_box["st"]

    # ---------------------------------------------------------- e2e (host API)
    e2e = None
    if not args.no_e2e and not args.profile_only:
        # the reference-facing host API with pinned fp32 host operands; each
        # rank holds only its own q / w rows (csaidx_host_run_chunked_local)
        qh = torch.empty((B, rows, H, D), dtype=torch.float32, pin_memory=True)
        qh.view(-1).copy_(q.float())
        kch = torch.empty((B, T, D), dtype=torch.float32, pin_memory=True)
        if world > 1:
            bcast(kc)
        kch.view(-1).copy_(kc.float())
        wh = torch.empty((B, rows, H), dtype=torch.float32, pin_memory=True)
        wh.view(-1).copy_(w)
        oi = torch.empty((B, rows, k), dtype=torch.int64, pin_memory=True)
        ov = torch.empty((B, rows, k), dtype=torch.float32, pin_memory=True)
        ecfg = api.DriverConfig(tile=api.TileConfig(cs, ct), device=local, stream=0)
        torch.cuda.synchronize()
        api.run_chunked_rows(qh, kch, wh, dims, ecfg, mine, oi, ov, local_rows=True)  # warm-up
        if world > 1:
            dist.barrier()
        e2e_probe = os.environ.get("CSAIDX_BENCH_E2E_PROBE") == "1"  # (dev) kernel times + clocks inside e2e
        if e2e_probe:
            drv.reset()
            drv.profiling(True)
            eclk = ClockSampler(local)
            eclk.start()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            api.run_chunked_rows(qh, kch, wh, dims, ecfg, mine, oi, ov, local_rows=True)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1000 / args.e2e_steps
        if e2e_probe:
            ek = {name: drv.get(kd) for name, kd in kinds.items()}
            print(json.dumps({"e2e_kernels_ms_per_step": {n: v[1] / args.e2e_steps for n, v in ek.items()},
                              "e2e_clocks": eclk.stop()}), file=sys.stderr)
            drv.profiling(False)
        if world > 1:
            h = torch.tensor([e2e_ms], dtype=torch.float64)
            if backend == "nccl":
                t = h.cuda()
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                h = t.cpu()
            else:
                dist.all_reduce(h, op=dist.ReduceOp.MAX)
            e2e_ms = float(h.item())
        # q crosses PCIe as bf16 when the entry rounds it on the host cores
        # (CSAIDX_HOST_ROUND, default on), else as the caller's fp32
        host_round = (os.environ.get("CSAIDX_HOST_ROUND", "0") != "0" if "CSAIDX_HOST_ROUND" in os.environ
                      else int(os.environ.get("LOCAL_WORLD_SIZE", "1")) <= 1)
        host_threads = int(os.environ.get("CSAIDX_HOST_THREADS", 0)) or max(
            1, len(os.sched_getaffinity(0)) // int(os.environ.get("LOCAL_WORLD_SIZE", "1")) - 1)
        # bytes the last call moved (counted by the library)
        h2d, d2h, fp32_chunks, n_chunks = api.last_transfer()
        e2e = {"value": (pairs_mine if args.simulate_rank else pairs_total) / (e2e_ms / 1000.0),
               "unit": "legal pairs/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pcie_gbs": (h2d + d2h) / (e2e_ms / 1000.0) / 1e9,
               "bound": ("q rows are rounded fp32 -> bf16 on the host cores, 8 MiB pieces through a 4-piece pinned "
                         "ring copied as soon as each is written (the DMA reads them from the host LLC), and cross "
                         "PCIe once at 2 B/entry; H2D of chunk c+1 "
                         "and D2H of chunk c-1 overlap chunk c's kernels" if host_round else
                         "PCIe: the fp32 q rows (the reference API's input type) cross the bus once; H2D of "
                         "chunk c+1 and D2H of chunk c-1 overlap chunk c's kernels"),
               "host_rounding": {"on": host_round, "threads": host_threads if host_round else 0,
                                 "chunks_sent_fp32": fp32_chunks, "chunks": n_chunks},
               "path": "csaidx_host_run_chunked_local (libcsaidx.so C entry of csaidx::run_chunked over this "
                       "rank's rows), pinned fp32 host operands, host rounding + H2D/D2H inside the timed region"}
        # cheap end-to-end correctness guard: the host API must agree with the resident run
        assert torch.equal(oi, out_idx.cpu()), "host-API result differs from the device-resident run"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        try:
            cpu = cpu_baseline(S, m, H, D, k)
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "legal pairs/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "indexer query·key pairs/sec (legal causal pairs)",
            "value": (pairs_mine if args.simulate_rank else pairs_total) / (ms / 1000.0),
            "unit": "legal pairs/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic: counter-based N(0,1/d_h) q/kc rounded to bf16, w ~ N(0,1/(d_h*H_I)) fp32, on device",
            "config": {"workload": f"{args.workload}: V4-Flash B={B} S={S} T={T} H_I={H} d_h={D} m={m} k={k}",
                       "query_tile": cs, "key_tile": ct,
                       "parallelism": (f"rank {plan_rank} of a query-sharded x{plan_world} run, measured alone on one "
                                       f"GPU (value = this rank's legal pairs / its step time)" if args.simulate_rank
                                       else f"query-sharded x{world} (LPT by causal work)"),
                       "l2": f"inputs (q {q.numel() * 2 / 1e9:.1f} GB bf16 per rank) exceed L2; no flush needed",
                       "dense_pairs_per_s": B * S * T / (ms / 1000.0)},
            "hbm_peak_gb": hbm_peak / 1e9,
            "ledger_peak_bytes": st.ledger_peak_bytes,
            "roofline": {"bound": "tensor", "kernel": "score_tc_kernel (tcgen05 kind::f16, M=128 keys x N=128 = 2 queries x 64 heads)",
                         "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": (achieved_tflops / peak_tflops) if achieved_tflops else None,
                         "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside a long step)",
                         "traffic": traffic, "algorithmic": f"{FLOPS_PER_PAIR} FLOP per legal pair",
                         "launches": score_n, "avg_launch_ms": score_ms / max(score_n, 1)},
            "kernels_ms_per_step": {n: v[1] / args.steps for n, v in kstats.items()},
            "select_roofline": {"bound": "hbm", "kernel": "select_kernel (per-row exact top-k over the fp32 tile)",
                                "achieved": select_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                "frac": (select_gbs / peaks["hbm_gbs"]) if select_gbs else None,
                                "traffic": sel_traffic,
                                "algorithmic": "4 B per legal pair (one read of each legal fp32 score)",
                                "launches": sel_n, "avg_launch_ms": sel_ms / max(sel_n, 1)},
            "select_fallback_rows": fallbacks,
            "select_prefilter_rows": cand_hits,
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "run_stats": {"dispatch_count": st.dispatch_count, "tiles_skipped_masked": st.tiles_skipped_masked},
            "multi_gpu": {"rank_work_pairs": loads, "gather_reassembly_ok": gather_ok,
                          "driver": ("libcsaidx.so csaidx_multi_run (csaidx::gpu::MultiRank), "
                                     f"{'NCCL' if backend == 'nccl' else 'gloo host-staged'} transport")
                          if world > 1 else "single GPU",
                          "collectives": ("broadcast kc (bf16) from rank 0; the final select kernels store each "
                                          "rank's int32 [rows,k] index rows straight into rank 0's [B,S,k] buffer "
                                          "over a CUDA IPC peer mapping (fused gather); a 1-element barrier ends "
                                          "the step") if p2p else
                                         ("broadcast kc (bf16) from rank 0 + gather of the int32 [rows,k] index "
                                          "rows to rank 0 after the compute (grouped send/recv), scattered into "
                                          "sequence order on rank 0" if world > 1 else "none"),
                          "rank_rows": rows, "rank_pairs": pairs_mine},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        mr.close()
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
