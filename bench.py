#!/usr/bin/env python
"""bench.py — Kron-Matmul throughput on B200 (BASELINE.json metric: "Kron-Matmul GFLOP/s and % roofline at
1/2/4/8 B200, fp32 and fp64").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config E] [--impl ours|reference]

A step is one whole Kron-Matmul Y = X·(F^1 ⊗ … ⊗ F^N) over the configuration's full M rows (all passes
of the plan).  Default workload: config E (BASELINE.json configs[4]: M=4096, 5 factors 16x16, fp32 — the
largest single-GPU configuration and the distributed one).  FLOPs are the method's algorithmic count
sum_f 2·M·W_f·Q_f (north_star).

N = 1: `value` times kron_matmul on config E.  The same JSON line carries device-timed sub-lines for the
other full-size configurations (B, C32, C64, D1, D2 — BASELINE.json configs[1..3]) under "configs", each
with its own roofline, clocks, mean / median / min step time (--no-subconfigs skips them).

N > 1 (torchrun, one rank per GPU, NCCL): Algorithm 2 — kron_matmul_dist over NCCL on the paper-rule grid
{GM,GK} (2 -> {2,1}, 4 -> {2,2}, 8 -> {4,2}) with config E's M = 4096 rows split over the
grid -> "scaling": "strong".  A secondary row-only {G,1} measurement (no exchange) is reported
under "row_only".  --grid GMxGK overrides the grid.

Timing: W untimed warm-ups, then exactly K steps on the device between CUDA events on the launching
stream, bracketed by barrier + synchronize, max over ranks.  Inputs (>= 1 GiB) are larger than the
126 MB L2, so no flush is needed.  Clocks and throttle reasons are sampled with NVML during every timed
region.  Per-pass CUDA events (kron_matmul_ws_events) give the dominant kernel's average launch time
for the roofline object.

--impl reference times the CPU oracle (oracle/, plain C fp64 Algorithm 1) on the host cores, each
step a bounded row sample of the same workload (this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Kron-Matmul GFLOP/s and % roofline at 1/2/4/8 B200, fp32 and fp64"

CONFIGS = {
    # name: (cfg index for the seed, M, P, Q, dtype)
    "A": (0, 16, [4] * 2, [4] * 2, "float32"),
    "B": (1, 1024, [8] * 6, [8] * 6, "float32"),
    "C32": (2, 1024, [32] * 4, [32] * 4, "float32"),
    "C64": (2, 1024, [32] * 4, [32] * 4, "float64"),
    "D1": (3, 320, [128] * 3, [128] * 3, "float64"),
    "D2": (4, 320, [64] * 3, [32] * 3, "float64"),
    "E": (5, 4096, [16] * 5, [16] * 5, "float32"),
    # Fig 11 weak-scaling workloads: fp32, N = 4, M grows with the GPU count
    # (memory per GPU constant: 16 GiB of X per GPU); M given per GPU, --dist only
    "W64": (6, 256, [64] * 4, [64] * 4, "float32"),
    "W128": (7, 16, [128] * 4, [128] * 4, "float32"),
}
WEAK = {"W64", "W128"}
SUBCONFIGS = ["B", "C32", "C64", "D1", "D2"]

# ALU peaks derived from the B200 unit counts:
# 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz; FP64 = half the FP32 lanes.
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FP64_PEAK_TFLOPS = FP32_PEAK_TFLOPS / 2
MMA_TF32_TFLOPS = 274.6  # legacy mma.sync m16n8k8 TF32, measured (profiles/r01_microbench_mma.jsonl)
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json

REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x100: "display_clock_setting"}


def widths(P, Q):
    N = len(P)
    W = [0] * (N + 1)
    W[N] = int(np.prod(P))
    for f in range(N, 0, -1):
        W[f - 1] = W[f] // P[f - 1] * Q[f - 1]
    return W


def flops_of(M, P, Q):
    W = widths(P, Q)
    return float(sum(2.0 * M * W[f] * Q[f - 1] for f in range(1, len(P) + 1)))


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, kernel_prefix):
    """dram read+write bytes per launch of the kernel from the committed `ncu --set full` capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py), with the capture's tag; (None, None) if the
    kernel was not captured.  ncu replays kernels, so this cannot be measured inside the timed run."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(config, {}).get(kernel_prefix)
        return v, d.get("_source", "profiles/ncu_traffic.json")
    except Exception:
        return None, None


def measured_bf16():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0 * 0.74  # nominal x the measured/nominal ratio of the pool's B200s (B200_PROFILING.md)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, dev_index, period=0.01):
        self.samples, self.reasons, self.period = [], 0, period
        self.stop_flag = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)

    def _run(self):
        while not self.stop_flag.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_flag.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [n for bit, n in REASONS.items() if self.reasons & bit]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def max_over_ranks(v, dev):
    """MAX of a per-rank float over the default process group (device tensor for NCCL, host for gloo)."""
    import torch
    import torch.distributed as dist
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_oracle_rate(M, P, Q, seed, dt, target_s=10.0, max_rows=None):
    """Oracle GFLOP/s on a bounded row sample (rows are independent in Algorithm 1): grow the
    sample to ~target_s/4 of CPU time, then time repeated passes over it for ~target_s in total.
    Returns (GFLOP/s, rows per pass, seconds timed, passes)."""
    import oracle
    import synth
    K = int(np.prod(P))
    Fs = synth.factors(P, Q, seed, "urand", dt)
    per_row = flops_of(1, P, Q)
    rows = 1
    t = 0.0
    while True:
        Xr = synth.rows_of(np.arange(rows), K, seed, 0, "urand").astype(dt)
        t0 = time.perf_counter()
        oracle.alg1(Xr, Fs)
        t = time.perf_counter() - t0
        cap = max_rows or M
        if t >= target_s / 4 or rows >= cap:
            break
        rows = min(cap, max(rows * 2, int(rows * target_s / 4 / max(t, 1e-3))))
    reps = max(1, int(round(target_s / max(t, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.alg1(Xr, Fs)
    t = time.perf_counter() - t0
    return per_row * rows * reps / t / 1e9, rows, t, reps


def run_reference(args, cfg_name):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg, M, P, Q, dtn = CONFIGS[cfg_name]
    import oracle
    import synth
    dt = np.float32 if dtn == "float32" else np.float64
    seed = synth.SEED_BASE + cfg
    K = int(np.prod(P))
    cores = oracle.threads(len(os.sched_getaffinity(0)))  # all host cores (torchrun exports OMP_NUM_THREADS=1)
    per_row = flops_of(1, P, Q)
    # rows per step: ~0.15 s of oracle work at ~1 GFLOP/s/core
    rows = int(max(1, min(M, 0.15 * cores * 1e9 / per_row)))
    Fs = synth.factors(P, Q, seed, "urand", dt)
    Xr = synth.rows_of(np.arange(rows), K, seed, 0, "urand").astype(dt)
    for _ in range(args.warmup):
        oracle.alg1(Xr, Fs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.alg1(Xr, Fs)
    el = time.perf_counter() - t0
    value = per_row * rows * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "strong" if ws > 1 and cfg_name not in WEAK else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter-based U[0,1))",
        "config": {"workload": cfg_name, "M": M, "P": P, "Q": Q, "input_dtype": dtn, "rows_per_step": rows},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"rows 0..{rows - 1} of config {cfg_name} (M={M}) per step; plain C fp64 "
                                   f"Algorithm 1, OpenMP over rows"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# Paper workload sweeps (shapes only, synthetic data): Table 3 (M = 16, largest P^N, float and double,
# P:997-1013) and Table 4 (28 real-world sizes).  "a^n x b^n" = n factors of a x b.
TABLE3 = [(16, [8] * 8, [8] * 8), (16, [16] * 6, [16] * 6), (16, [32] * 5, [32] * 5), (16, [64] * 4, [64] * 4)]
TABLE4 = [
    (20, [2] * 7, [2] * 7), (20, [2] * 9, [2] * 9), (50, [2] * 9, [2] * 9), (20, [2] * 10, [2] * 10),
    (1, [2] * 11, [2] * 11),
    (10, [52, 65], [50, 20]), (50, [32, 64], [8, 128]), (10, [52, 50], [65, 20]),
    (4, [2] * 9, [2] * 9), (8, [2] * 9, [2] * 9), (16, [2] * 9, [2] * 9), (20, [2] * 9, [2] * 9),
    (4, [8] * 3, [8] * 3), (8, [8] * 3, [8] * 3), (16, [8] * 3, [8] * 3), (20, [8] * 3, [8] * 3),
    (1024, [3] * 7, [3] * 7), (1024, [4] * 7, [4] * 7), (1024, [6] * 7, [6] * 7),
    (1, [5] * 3 + [2], [5] * 3 + [2]), (1, [5] * 2 + [2, 25], [5] * 2 + [2, 25]),
    (1526, [4] * 6, [4] * 6), (156, [8] * 3, [8] * 3), (2967, [4] * 7, [4] * 7),
    (16, [8] * 8, [8] * 8), (16, [16] * 6, [16] * 6), (16, [32] * 6, [32] * 6), (16, [64] * 3, [64] * 3),
]


def run_sweep(args):
    """One JSON line per shape: device-resident GFLOP/s of kron_matmul_ws (CUDA events, mean of steps)."""
    import torch
    import synth
    from paper_2401_10187_b200 import kron
    dev = torch.device("cuda", 0)
    shapes = TABLE3 if args.sweep == "table3" else TABLE4
    dts = ["float32", "float64"] if args.sweep == "table3" else ["float32"]
    free = torch.cuda.mem_get_info()[0]
    for idx, (M, P, Q) in enumerate(shapes):
        for dtn in dts:
            tdt = getattr(torch, dtn)
            es = 4 if dtn == "float32" else 8
            K, L = int(np.prod(P)), int(np.prod(Q))
            wsz = kron.workspace_size(M, P, Q, tdt)
            need = M * (K + L) * es + wsz
            line = {"sweep": args.sweep, "id": idx + 1, "M": M, "P": P, "Q": Q, "dtype": dtn,
                    "plan": [list(p) for p in kron.plan_describe(M, P, Q, tdt)]}
            if need > 0.9 * free:
                line["skipped"] = f"needs {need / 2**30:.1f} GiB"
                print(json.dumps(line), flush=True)
                continue
            X = torch.empty((M, K), dtype=tdt, device=dev)
            synth.fill_device(X.data_ptr(), M, K, synth.SEED_BASE + 50 + idx, 0, "urand", np.dtype(dtn))
            Fs = [torch.from_numpy(f).to(dev) for f in synth.factors(P, Q, synth.SEED_BASE + 50 + idx, "urand",
                                                                       np.dtype(dtn))]
            Y = torch.empty((M, L), dtype=tdt, device=dev)
            work = torch.empty(max(wsz, 1), dtype=torch.uint8, device=dev)
            for _ in range(args.warmup):
                kron.matmul_ws(X, Fs, Y, work)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                kron.matmul_ws(X, Fs, Y, work)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            fl = flops_of(M, P, Q)
            b_alg, _ = kron.plan_cost(M, P, Q, tdt)
            line.update({"ms": round(ms, 5), "gflops": round(fl / ms / 1e6, 2), "hbm_gbs": round(b_alg / ms / 1e6, 1)})
            # the same problem replayed as a CUDA graph (kron_graph_*): launch-bound shapes drop the
            # per-call host cost (argument checks, plan lookup, tensor-map encodes, launches)
            g = kron.Graph(X, Fs, Y, work)
            for _ in range(args.warmup):
                g.launch()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                g.launch()
            e1.record()
            torch.cuda.synchronize()
            gms = e0.elapsed_time(e1) / args.steps
            g.close()
            line.update({"graph_ms": round(gms, 5), "graph_gflops": round(fl / gms / 1e6, 2)})
            # the autotuner on the same buffers: every candidate plan timed, the fastest installed
            # in the plan cache, then the call timed again through it
            _, ncand, _ = kron.autotune(X, Fs, out=Y, reps=3)
            del work  # the tuned plan may need another workspace size
            wt = torch.empty(max(kron.workspace_size(M, P, Q, tdt), 1), dtype=torch.uint8, device=dev)
            for _ in range(args.warmup):
                kron.matmul_ws(X, Fs, Y, wt)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                kron.matmul_ws(X, Fs, Y, wt)
            e1.record()
            torch.cuda.synchronize()
            tms = e0.elapsed_time(e1) / args.steps
            line.update({"tuned_ms": round(tms, 5), "tuned_gflops": round(fl / tms / 1e6, 2), "tuned_candidates": ncand,
                         "tuned_plan": [list(p) for p in kron.plan_describe(M, P, Q, tdt)],
                         "tuned_kernels": kron.plan_kernels(M, P, Q, tdt)})
            kron.plan_cache_clear()
            print(json.dumps(line), flush=True)
            del X, Y, wt, Fs
            torch.cuda.empty_cache()
    return 0


def step_stats(step_ms):
    a = np.asarray(step_ms, dtype=np.float64)
    return {"mean_ms": round(float(a.mean()), 5), "median_ms": round(float(np.median(a)), 5),
            "min_ms": round(float(a.min()), 5), "max_ms": round(float(a.max()), 5)}


def roofline_of(M, P, Q, es, alg_bytes, alg_flops, t_s, mode=None, kname=None):
    """Roofline object for one kernel (or a whole step): the binding resource of max(B/BW, F/peak)."""
    hbm_peak, hbm_src = measured_peaks()
    alu_peak = FP32_PEAK_TFLOPS if es == 4 else FP64_PEAK_TFLOPS
    alu_src = "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz" + (" / 2 (FP64)" if es == 8 else "")
    if mode and kname == "kron_fused_tf32x3_kernel":
        alu_peak, alu_src = MMA_TF32_TFLOPS / 3, "measured mma.sync TF32 (profiles/r01_microbench_mma.jsonl) / 3"
    if mode and kname == "kron_tc_pair_kernel":
        # tcgen05 kind::tf32 = half the dense bf16 rate (nominal 1.1 vs 2.25 PF); the measured cuBLAS bf16 peak
        # of MEASURED_PEAKS.json x 1/2, / 3 MMAs per product in the 3xTF32 mode
        bf16 = measured_bf16()
        alu_peak = bf16 / 2 / (3 if mode == "3xtf32" else 1)
        alu_src = (f"measured bf16 {bf16} TF/s (MEASURED_PEAKS.json) x 1/2 (tf32/bf16 nominal ratio)" +
                   (" / 3 (3xTF32)" if mode == "3xtf32" else ""))
    t_hbm, t_alu = alg_bytes / (hbm_peak * 1e9), alg_flops / (alu_peak * 1e12)
    if t_hbm >= t_alu:
        ach = alg_bytes / t_s / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "peak_source": hbm_src}
    ach = alg_flops / t_s / 1e12
    return {"bound": "alu", "achieved": round(ach, 3), "peak": round(alu_peak, 2), "unit": "TFLOP/s",
            "frac": round(ach / alu_peak, 4), "peak_source": alu_src}


def measure_single(kron, synth, torch, cfg_name, args, dev, rank, barrier, mode=None, ws=1):
    """Device-timed kron_matmul steps on one configuration (inputs resident in HBM).  Returns a dict with the
    step statistics, the dominant kernel's roofline and the whole-step roofline, plus the buffers."""
    cfg, M, P, Q, dtn = CONFIGS[cfg_name]
    dt = np.float32 if dtn == "float32" else np.float64
    tdt = torch.float32 if dt == np.float32 else torch.float64
    es = 4 if dt == np.float32 else 8
    seed = synth.SEED_BASE + cfg
    K, L = int(np.prod(P)), int(np.prod(Q))
    stream = torch.cuda.current_stream()
    X = torch.empty((M, K), dtype=tdt, device=dev)
    synth.fill_device(X.data_ptr(), M, K, seed, 0, "urand", dt, stream=stream.cuda_stream, r0=rank * M, ld=K)
    Fs_h = synth.factors(P, Q, seed, "urand", dt)
    Fs = [torch.from_numpy(f).to(dev) for f in Fs_h]
    Y = torch.empty((M, L), dtype=tdt, device=dev)
    tuned = None
    if args.autotune:
        # time the candidate plans on these buffers, keep the fastest (untimed, before warm-up)
        _, ncand, best = kron.autotune(X, Fs, Y, reps=3, mode=mode)
        tuned = {"candidates": ncand, "best_ms": round(best, 5)}
    wsz = kron.workspace_size(M, P, Q, tdt, mode)
    work = torch.empty(max(wsz, 1), dtype=torch.uint8, device=dev)
    plan = kron.plan_describe(M, P, Q, tdt, mode)
    kernels = kron.plan_kernels(M, P, Q, tdt, mode)
    npass = len(plan)
    W = widths(P, Q)

    def mk_events(n):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for e in evs:
            e.record(stream)  # materialise the cudaEvent_t handles
        return evs

    for _ in range(args.warmup):
        kron.matmul_ws(X, Fs, Y, work, mode=mode)
    torch.cuda.synchronize()
    pass_events = [mk_events(npass + 1) for _ in range(args.steps)]
    t_start, t_end = mk_events(2)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            kron.matmul_ws_events(X, Fs, Y, work, [e.cuda_event for e in pass_events[k]], mode=mode)
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end)
    if ws > 1:
        ms = max_over_ranks(ms, dev)
    fl_step = flops_of(M, P, Q)
    # per-pass (kernel) timing -> roofline of the dominant kernel; per-step times -> median / min
    pass_ms = np.zeros(npass)
    step_ms = []
    for k in range(args.steps):
        for i in range(npass):
            pass_ms[i] += pass_events[k][i].elapsed_time(pass_events[k][i + 1])
        step_ms.append(pass_events[k][0].elapsed_time(pass_events[k][npass]))
    pass_ms /= args.steps
    dom = int(np.argmax(pass_ms))
    first, nf, kind = plan[dom]
    w_in, w_out = W[first], W[first - nf]
    alg_bytes = es * M * (w_in + w_out) + sum(es * P[f - 1] * Q[f - 1] for f in range(first, first - nf, -1))
    alg_flops = sum(2.0 * M * W[f] * Q[f - 1] for f in range(first, first - nf, -1))
    kname = kernels[dom]
    roof = roofline_of(M, P, Q, es, alg_bytes, alg_flops, pass_ms[dom] / 1e3, mode, kname)
    traffic, tsrc = ncu_traffic(cfg_name if not mode else cfg_name + "_" + mode, kname)
    roof.update({"kernel": f"{kname} (pass {dom}: factors {first}..{first - nf + 1}, {kind})",
                 "ms_per_launch": round(float(pass_ms[dom]), 5), "alg_bytes_per_launch": int(alg_bytes),
                 "alg_flops_per_launch": alg_flops, "share_of_step": round(float(pass_ms[dom] / (ms / args.steps)), 4),
                 "timing": "CUDA events on the launching stream around each launch, mean over the timed steps",
                 "traffic": traffic, "traffic_source": tsrc})
    b_alg, f_alg = kron.plan_cost(M, P, Q, tdt, mode)
    tc_k = [k for k in ("kron_tc_pair_kernel", "kron_fused_tf32x3_kernel") if mode and k in kernels]
    step_roof = roofline_of(M, P, Q, es, b_alg, f_alg, ms / args.steps / 1e3, mode, tc_k[0] if tc_k else None)
    hbm_peak, _ = measured_peaks()
    alu_peak = FP32_PEAK_TFLOPS if es == 4 else FP64_PEAK_TFLOPS
    t_roof = max(b_alg / (hbm_peak * 1e9), f_alg / (alu_peak * 1e12))
    res = {
        "workload": cfg_name, "dtype": "f32" if es == 4 else "f64", "M": M, "P": P, "Q": Q, "K": K, "L": L,
        "ms_per_step": round(ms / args.steps, 5), "value": round(ws * fl_step * args.steps / (ms / 1e3) / 1e9, 2),
        "unit": "GFLOP/s", "steps": args.steps, "warmup": args.warmup, **step_stats(step_ms),
        "plan": [list(p) for p in plan], "kernels": kernels, "autotune": tuned,
        "pass_ms": [round(float(v), 5) for v in pass_ms],
        "roofline": roof,
        "step_roofline": {"t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof / (ms / args.steps / 1e3), 4),
                          "bound": step_roof["bound"], "alg_bytes": b_alg, "alg_flops": f_alg},
        "gpu_launches": npass * args.steps, "clocks": clocks.summary(),
        "l2": "inputs larger than L2 (no flush)",
    }
    # ALU-bound kernels under a power cap: the same achieved rate against the peak scaled to the measured SM clock
    # (informational; `frac` stays against the max-clock peak)
    clk = res["clocks"]
    if roof.get("bound") == "alu" and clk.get("sm_mhz") and clk.get("sm_max_mhz"):
        scale = float(clk["sm_mhz"]) / float(clk["sm_max_mhz"])
        roof["frac_at_measured_clock"] = round(roof["frac"] / scale, 4) if scale > 0 else None
    return res, (X, Fs_h, Fs, Y, work, seed, dt, tdt, es, M, K, L, fl_step)


def cpu_baseline_of(cfg_name, M, P, Q, seed, dt):
    import oracle
    cores = oracle.threads(len(os.sched_getaffinity(0)))  # all host cores (torchrun sets OMP_NUM_THREADS=1)
    rate, rows, t, reps = cpu_oracle_rate(M, P, Q, seed, dt)
    return {"value": round(rate, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"rows 0..{rows - 1} of config {cfg_name} (M={M}) x {reps} passes, {t:.1f} s; plain C "
                      f"fp64 Algorithm 1 (oracle/), OpenMP over rows"}


def run_single(args, kron, synth, torch, ws, rank, local, dev, barrier):
    """N = 1 (or --no-dist under torchrun: row-partitioned weak scaling, no communication)."""
    mode = args.mode
    res, bufs = measure_single(kron, synth, torch, args.config, args, dev, rank, barrier, mode, ws)
    X, Fs_h, Fs, Y, work, seed, dt, tdt, es, M, K, L, fl_step = bufs
    stream = torch.cuda.current_stream()

    # e2e through the public C-ABI with HOST buffers: kron_matmul_host streams row chunks H2D -> passes ->
    # D2H with the copies overlapping; the host X is a pinned copy of the device input
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty((M, K), dtype=tdt, pin_memory=True)
        Xh.copy_(X)
        Fh = [torch.from_numpy(f).pin_memory() for f in Fs_h]
        Yh = torch.empty((M, L), dtype=tdt, pin_memory=True)
        del X, Y, work
        torch.cuda.empty_cache()
        kron.matmul_host(Xh, Fh, Yh, mode=mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            kron.matmul_host(Xh, Fh, Yh, mode=mode)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if ws > 1:
            ems = max_over_ranks(ems, dev)
        h2d = M * K * es + sum(f.numel() * es for f in Fh)
        e2e = {"value": round(ws * fl_step * args.e2e_steps / (ems / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(ws * h2d), "d2h_bytes_per_step": int(ws * M * L * es),
               "steps": args.e2e_steps,
               "path": "pinned host X,F -> kron_matmul_host (public C-ABI: row-chunk H2D / passes / D2H "
                       "pipeline) -> pinned host Y"}
        del Xh, Yh
    else:
        del X, Y, work
    torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        _, Mc, Pc, Qc, _ = CONFIGS[args.config]
        cpu = cpu_baseline_of(args.config, Mc, Pc, Qc, seed, dt)

    subs = None
    if ws == 1 and not args.no_subconfigs and not mode:
        subs = {}
        for name in SUBCONFIGS:
            if name == args.config:
                continue
            r, b = measure_single(kron, synth, torch, name, args, dev, rank, barrier, None, 1)
            del b
            torch.cuda.empty_cache()
            subs[name] = {k: v for k, v in r.items() if k not in ("steps", "warmup", "l2")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": res["dtype"],
            **({"mode": {"3xtf32": "3xtf32 (fp32 data, split-operand TF32 tcgen05 MMAs; reported separately)",
                         "tf32": "tf32 (fp32 data, TF32 tcgen05 MMAs; reported separately)"}[mode]} if mode else {}),
            "data": "synthetic (seeded counter-based U[0,1) X and factors, generated in HBM)",
            "config": {"workload": args.config, "M_per_gpu": M, "P": res["P"], "Q": res["Q"], "K": K, "L": L,
                       "plan": res["plan"], "kernels": res["kernels"], "autotune": res["autotune"],
                       "parallelism": "single GPU" if ws == 1 else f"row partition x{ws} (no communication)",
                       "l2": "inputs larger than L2 (no flush)"},
            "step_stats": {k: res[k] for k in ("mean_ms", "median_ms", "min_ms", "max_ms")},
            "pass_ms": res["pass_ms"],
            "roofline": res["roofline"], "step_roofline": res["step_roofline"],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
            "configs": subs,
        }
        print(json.dumps(line), flush=True)
    return 0


def run_dist(args, kron, synth, torch, ws, rank, local, dev, barrier):
    """Algorithm 2 through kron_matmul_dist: config E (default) strong-scaled over the paper-rule grid, or
    a Fig 11 workload weak-scaled (M grows with the GPU count)."""
    cfg_name = args.config
    cfg, M, P, Q, dtn = CONFIGS[cfg_name]
    weak = cfg_name in WEAK
    if weak:
        M = (args.rows or M) * ws  # rows per GPU x GPUs (Fig 11: memory per GPU constant)
    dt = np.float32 if dtn == "float32" else np.float64
    tdt = torch.float32 if dt == np.float32 else torch.float64
    es = 4 if dt == np.float32 else 8
    seed = synth.SEED_BASE + cfg
    K, L = int(np.prod(P)), int(np.prod(Q))
    GM, GK = (0, 0) if args.grid is None else (int(v) for v in args.grid.lower().split("x"))
    share = os.environ.get("KRON_BENCH_SHARE_GPU") == "1"
    if ws == 1:
        ctx = kron.DistContext("virtual", GM=1, GK=1)
    else:
        backend = args.exchange if not (share and args.exchange == "nccl") else "virtual-unavailable"
        if backend == "virtual-unavailable":
            raise SystemExit("NCCL cannot place two ranks on one GPU: use --exchange p2p with KRON_BENCH_SHARE_GPU")
        ctx = kron.DistContext(backend, GM=GM, GK=GK, chunks=args.chunks)
    gm, gk = ctx.coords(rank)
    Ml, Kl, Ll = M // ctx.GM, K // ctx.GK, L // ctx.GK
    stream = torch.cuda.current_stream()
    X = torch.empty((Ml, Kl), dtype=tdt, device=dev)
    synth.fill_device(X.data_ptr(), Ml, Kl, seed, 0, "urand", dt, stream=stream.cuda_stream, r0=gm * Ml,
                      c0=gk * Kl, ld=K)
    Fs_h = synth.factors(P, Q, seed, "urand", dt)
    Fs = [torch.from_numpy(f).to(dev) for f in Fs_h]
    Y = torch.empty((Ml, Ll), dtype=tdt, device=dev)
    xs, ys = (X, Y) if ctx.backend != "virtual" else ([X], [Y])

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        with ClockSampler(local) as clocks:
            evs[0].record(stream)
            for k in range(steps):
                fn()
                evs[k + 1].record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = evs[0].elapsed_time(evs[-1])
        step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(steps)]
        if ws > 1:
            ms = max_over_ranks(ms, dev)
        return ms, step_ms, clocks.summary()

    ms, step_ms, clk = timed(lambda: kron.matmul_dist(M, xs, Fs, ctx, out=ys), args.steps)
    if ws > 1:
        ctx.sync()  # asynchronous NCCL errors of the timed calls surface here
    rounds, ledger = kron.dist_plan(M, P, Q, ctx.GM, ctx.GK)
    fl_step = flops_of(M, P, Q)
    value = fl_step * args.steps / (ms / 1e3) / 1e9
    b_alg, f_alg = kron.plan_cost(M, P, Q, tdt)
    hbm_peak, _ = measured_peaks()
    alu_peak = FP32_PEAK_TFLOPS if es == 4 else FP64_PEAK_TFLOPS
    t_roof = max(b_alg / (hbm_peak * 1e9), f_alg / (alu_peak * 1e12)) / ws
    round_info = ctx.round_info(M, P, Q, tdt) if ctx.GK > 1 else []
    round_layouts = ctx.round_layouts(M, P, Q, tdt) if ctx.GK > 1 and hasattr(ctx, "round_layouts") else []

    # e2e: this rank's block from pinned host memory -> kron_matmul_dist -> Y_local back to pinned host memory
    e2e = None
    if not args.no_e2e:
        Xh = torch.empty((Ml, Kl), dtype=tdt, pin_memory=True)
        Xh.copy_(X)
        Yh = torch.empty((Ml, Ll), dtype=tdt, pin_memory=True)

        def e2e_step():
            X.copy_(Xh, non_blocking=True)
            kron.matmul_dist(M, xs, Fs, ctx, out=ys)
            Yh.copy_(Y, non_blocking=True)

        ems, _, _ = timed(e2e_step, args.e2e_steps)
        e2e = {"value": round(fl_step * args.e2e_steps / (ems / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(M * K * es), "d2h_bytes_per_step": int(M * L * es), "steps": args.e2e_steps,
               "path": "per rank: pinned host X block -> H2D -> kron_matmul_dist -> D2H of Y_local (all ranks' bytes)"}

    # secondary: the same rows on a row-only grid {G,1} (no exchange)
    row_only = None
    if ws > 1 and ctx.GK > 1 and not args.no_row_only and args.exchange == "nccl" and not share:
        ctx2 = kron.DistContext("nccl", GM=ws, GK=1)
        Mr = M // ws
        X2 = torch.empty((Mr, K), dtype=tdt, device=dev)
        synth.fill_device(X2.data_ptr(), Mr, K, seed, 0, "urand", dt, stream=stream.cuda_stream, r0=rank * Mr, ld=K)
        Y2 = torch.empty((Mr, L), dtype=tdt, device=dev)
        del X, Y
        torch.cuda.empty_cache()
        ms2, step2, clk2 = timed(lambda: kron.matmul_dist(M, X2, Fs, ctx2, out=Y2), args.steps)
        row_only = {"grid": [ws, 1], "value": round(fl_step * args.steps / (ms2 / 1e3) / 1e9, 2), "unit": "GFLOP/s",
                    "ms_per_step": round(ms2 / args.steps, 5), **step_stats(step2), "clocks": clk2}
        ctx2.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f32" if es == 4 else "f64",
            "data": "synthetic (seeded counter-based U[0,1), each rank generates its own block in HBM)",
            "config": {"workload": cfg_name, "M": M, "P": P, "Q": Q, "grid": [ctx.GM, ctx.GK],
                       "rounds": rounds, "exchanged_values_per_step": int(sum(ledger)),
                       "fused_layout_per_round": round_info, "exchange_layout_per_round": round_layouts,
                       "row_chunks": args.chunks,
                       "parallelism": f"Algorithm 2 grid {ctx.GM}x{ctx.GK} (rows x K), " +
                                      ("NCCL all-to-all" if ctx.backend == "nccl" else
                                       "P2P over peer memory (CUDA IPC)" if ctx.backend == "p2p" else
                                       "single GPU (grid 1x1)"),
                       "l2": "inputs larger than L2 (no flush)"},
            "step_stats": step_stats(step_ms),
            "step_roofline": {"t_roof_ms_per_gpu": round(t_roof * 1e3, 4),
                              "frac": round(t_roof / (ms / args.steps / 1e3), 4)},
            "e2e": e2e, "row_only": row_only,
            "gpu_launches": None, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # the paper: "average of 100 runs after 10 warm-ups"
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="E", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-subconfigs", action="store_true", help="N = 1: skip the B/C32/C64/D1/D2 sub-lines")
    ap.add_argument("--no-row-only", action="store_true", help="N > 1: skip the row-only {G,1} secondary line")
    ap.add_argument("--dist", action=argparse.BooleanOptionalAction, default=None,
                    help="Algorithm 2 through kron_matmul_dist (default: on for N > 1, off for N = 1)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="distributed exchange: ncclAlltoAll (fused send / receive layouts) or the P2P push / pull "
                         "kernels over peer memory (NEXT-1, P:652)")
    ap.add_argument("--grid", default=None, help="GMxGK for the distributed path (default: the paper rule)")
    ap.add_argument("--chunks", type=int, default=2, help="row chunks per round (exchange / compute overlap)")
    ap.add_argument("--rows", type=int, default=None,
                    help="W64 / W128: rows per GPU (default: the Fig 11 sizes, 16 GiB of X per GPU)")
    ap.add_argument("--mode", default=None, choices=["3xtf32", "tf32"],
                    help="fp32 configs only: the separately reported tcgen05 tensor-core modes (NEXT-4)")
    ap.add_argument("--autotune", action=argparse.BooleanOptionalAction, default=True,
                    help="autotune the pass plan before warm-up (P:599-619); --no-autotune = static plan")
    ap.add_argument("--sweep", default=None, choices=["table3", "table4"],
                    help="paper shape sweeps (one JSON line per shape) instead of the headline bench")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if args.impl == "reference":
        return run_reference(args, args.config if args.config not in WEAK else "E")
    if args.sweep:
        return run_sweep(args)

    import torch
    import synth
    from paper_2401_10187_b200 import kron

    ws, rank, local = dist_env()
    if ws != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
    # KRON_BENCH_SHARE_GPU=1 (plumbing test only): every rank on cuda:0 with a gloo process group, so the
    # N > 1 code paths (barriers, max-over-ranks, P2P heaps over CUDA IPC) run on a one-GPU box; NCCL
    # cannot place two ranks on one device.  Numbers from such a run are not bench values.
    share = os.environ.get("KRON_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    use_dist = args.dist if args.dist is not None else (ws > 1 or args.config in WEAK)
    if args.mode and use_dist:
        ap.error("--mode is a single-GPU mode")
    if args.mode and CONFIGS[args.config][4] != "float32":
        ap.error("--mode applies to the fp32 configs (B, C32, E)")
    rc = (run_dist if use_dist else run_single)(args, kron, synth, torch, ws, rank, local, dev, barrier)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
