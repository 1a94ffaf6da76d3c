#!/usr/bin/env python
"""Benchmark of the exact mod-m hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config c2|c3] [--no-extras]

Headline (N=1): BASELINE configs[1] -- synthetic 2^20 x 2^20 matrix,
Poisson(10) row lengths, 30% +-1, mod 65521.  One step = y <- A x followed by
y' <- A^T x' (the whole apply hot path), inputs resident
in HBM.  L2 (126 MB) is flushed between timed steps by writing a 256 MB
buffer, outside the step's events.  value = nonzeros processed per second
(2 nnz per step per rank), times from CUDA events on the launching stream,
max over ranks.  N > 1 (torchrun): every rank runs its own independent
c2-shaped problem (rank-seeded) -- weak scaling, no data-path collective.

Extras (default on, N = 1 only): c3 hybrid apply, c4 block apply k = 8/16/32,
c5 sequence steps/s -- each with its own roofline fraction.

--impl reference times the CPU oracle (oracle/, plain C, 1 thread) on the
same config, rank 0 only.
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

METRIC = "mod-m SpMV nonzeros/sec & achieved HBM GB/s vs peak; seq steps/s at 1/2/4/8"
FLUSH_BYTES = 256 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ ours ---

def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


LAUNCHES = {"timed": 0}


def timed_steps(step_fns, steps, warmup, flush, stream):
    """Run warmup + steps of a list of launch closures.  Returns per-launch
    event times (ms, shape steps x len(step_fns)); LAUNCHES["timed"] gets the
    number of library kernels launched inside the timed steps."""
    import torch

    import paper_1004_3719_b200 as ff
    for _ in range(warmup):
        flush.zero_()
        for f in step_fns:
            f()
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in step_fns] for _ in range(steps)]
    l0 = ff.ffspmv_kernel_launches()
    for s in range(steps):
        flush.zero_()
        for j, f in enumerate(step_fns):
            ev[s][j][0].record(stream)
            f()
            ev[s][j][1].record(stream)
    LAUNCHES["timed"] = ff.ffspmv_kernel_launches() - l0
    torch.cuda.synchronize()
    t = np.array([[a.elapsed_time(b) for a, b in row] for row in ev])
    return t


def bench_ours(args):
    import torch

    import paper_1004_3719_b200 as ff
    import synth

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    ff.load()
    stream = torch.cuda.current_stream()
    hbm_peak, peak_src = peaks()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    cfg = args.config
    M = synth.config_matrix(cfg) if world == 1 else _rank_matrix(cfg, rank)
    m, rows, cols = M["m"], M["rows"], M["cols"]
    A = ff.ffspmv_create(rows, cols, M["row"], M["col"], M["val"], m)
    info = A.info()
    g = synth.rng(synth.CONFIGS[cfg]["vseed"] + 7919 * rank)
    x = to_dev(synth.uniform(g, cols, m))
    xt = to_dev(synth.uniform(g, rows, m))
    y = torch.empty(rows, dtype=torch.int32, device="cuda")
    yt = torch.empty(cols, dtype=torch.int32, device="cuda")
    fns = [lambda: ff.ffspmv_apply(A, 1, x, 0, y, stream),
           lambda: ff.ffspmv_apply_transpose(A, 1, xt, 0, yt, stream)]

    # timed region: barrier + sync on both sides, device events per launch
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t = timed_steps(fns, args.steps, args.warmup, flush, stream)
    launches = LAUNCHES["timed"]
    torch.cuda.synchronize()
    step_ms = float(t.sum(axis=1).mean())
    total_ms = float(t.sum())
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(tt.item())
        torch.distributed.barrier()
    units_per_step = 2 * info["nnz"]             # apply + transpose
    value = units_per_step * world * args.steps / (total_ms / 1e3)
    # roofline of the dominant kernel pair (k_panel + k_panel_reduce of the
    # y <- A x call): algorithmic bytes of one launch / its mean event time;
    # traffic = ncu DRAM bytes of the same launch (profiles/ncu_traffic.json)
    alg = info["alg_bytes_apply"]
    apply_ms = float(t[:, 0].mean())
    achieved = alg / (apply_ms / 1e3) / 1e9
    panels = info["strategy_apply"] == ff.STRATEGY_PANELS
    kname = ("k_panel + k_panel_reduce (x panels in shared memory), y <- A x" if panels
             else "k_apply (rows layout), y <- A x")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": ncu_traffic(f"{cfg}_apply"),
                "kernel": kname, "peak_source": peak_src,
                "alg_bytes_per_launch": alg,
                "alg_bytes_note": "4 B per +-1 nonzero, 4 + e_v B per valued nonzero, 4 B per x and y element",
                "apply_ms": round(apply_ms, 5),
                "transpose_ms": round(float(t[:, 1].mean()), 5),
                "transpose_alg_gbs": round(info["alg_bytes_transpose"] / (float(t[:, 1].mean()) / 1e3) / 1e9, 1)}

    out = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "accumulator": f"u{info['acc_bits_max']}", "data": "synthetic",
           "config": {"workload": f"{cfg}: " + _describe(cfg), "rows": rows, "cols": cols,
                      "nnz": info["nnz"], "modulus": m, "op": "y <- A x ; y' <- A^T x'",
                      "l2": "flushed between timed steps (256 MB write)",
                      "parallelism": f"independent {cfg} problem per rank" if world > 1 else "1 GPU"},
           "roofline": roofline, "gpu_launches": launches,
           "mflops_paper_unit": 2 * value / 1e6}
    out["clocks"] = clk.summary()
    out["e2e"] = _e2e(ff, A, M, args, rows, cols, m, g, world)
    out["plan"] = {k: info[k] for k in ("strategy_apply", "strategy_transpose", "panels",
                                        "panel_bands", "gather_locality", "bands", "bands_sell",
                                        "bands_csr", "bands_coos", "slices", "long_rows", "nnz_pm1",
                                        "nnz_valued", "padded_slots", "stream_bytes",
                                        "panel_stream_bytes", "create_seconds")}
    if rank == 0 and world == 1:
        out["cpu_baseline"] = cpu_baseline(M, budget_s=args.cpu_seconds)
        if not args.no_extras:
            out["extras"] = extras(ff, flush, stream, hbm_peak, args)
    if world > 1 and not args.no_extras:
        out["extras"] = {"c5_sequence_2d": _seq_dist(args, world, rank, local)}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


def _seq_dist(args, world, rank, local):
    """c5 block Wiedemann sequence across the ranks (dist.sequence_2d on the
    P_r x P_c grid grid_shape picks): steps/s over the timed steps of one
    sequence call (device events on each rank, max over ranks), after
    args.warmup warm-up steps.  Reported beside the headline, never instead of
    it; a failure is reported, not raised."""
    import torch

    import synth
    from paper_1004_3719_b200 import dist as fdist
    try:
        M = synth.config_matrix("c5")
        n, m, k = M["rows"], M["m"], 16
        g = synth.rng(2005)
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, k), m)
        steps = max(1, min(args.steps, 50))
        L = args.warmup + steps
        pr, pc = fdist.grid_shape(world, k, n=n, nnz=len(M["row"]), iterate_bytes=4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def hook(t):
            if t == args.warmup:
                torch.cuda.synchronize()
                torch.distributed.barrier()
                e0.record()
            elif t == L:
                e1.record()
                torch.cuda.synchronize()

        fdist.sequence_2d(n, M["row"], M["col"], M["val"], m, X, L, U,
                          fdist.CudaBackend(f"cuda:{local}"), pr, pc, on_step=hook)
        ms = e0.elapsed_time(e1)
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
        return {"steps_per_s": steps / (ms / 1e3), "ms_per_step": ms / steps, "steps": steps,
                "grid": [pr, pc], "k": k, "mode": "2-D (row bands x column blocks), NCCL all-gather per step",
                "scaling": "strong (one c5 problem split over the ranks)"}
    except Exception as e:                       # the headline line must still print
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def _rank_matrix(cfg, rank):
    import synth
    c = dict(synth.CONFIGS[cfg])
    saved = synth.CONFIGS[cfg]
    try:
        c["seed"] = saved["seed"] + 100 * rank
        synth.CONFIGS[cfg] = c
        return synth.config_matrix(cfg)
    finally:
        synth.CONFIGS[cfg] = saved


def _describe(cfg):
    return {
        "c2": "2^20 x 2^20, Poisson(10) nnz/row, 30% +-1, mod 65521, apply + transpose apply",
        "c3": "1911130 x 1955309 GL7d-shaped, lognormal rows (mean ~19.7), all +-1, mod 3",
    }.get(cfg, cfg)


def _e2e(ff, A, M, args, rows, cols, m, g, world):
    """Same metric through the public host-buffer call: each step copies x
    (and x') from pinned host memory, runs, and copies y (and y') back."""
    import torch
    xs = torch.empty(cols, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    xts = torch.empty(rows, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    ys = torch.empty(rows, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    yts = torch.empty(cols, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    xs[:] = synth_uniform(g, cols, m)
    xts[:] = synth_uniform(g, rows, m)
    for _ in range(args.warmup):
        ff.ffspmv_apply_host(A, ff.OP_APPLY, 1, xs, 0, ys)
        ff.ffspmv_apply_host(A, ff.OP_TRANSPOSE, 1, xts, 0, yts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ff.ffspmv_apply_host(A, ff.OP_APPLY, 1, xs, 0, ys)
        ff.ffspmv_apply_host(A, ff.OP_TRANSPOSE, 1, xts, 0, yts)
    dt = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        dt = float(tt.item())
    nnz = A.info()["nnz"]
    return {"value": 2 * nnz * world * args.steps / dt, "unit": "nnz/s",
            "h2d_bytes_per_step": 4 * (cols + rows), "d2h_bytes_per_step": 4 * (rows + cols),
            "api": "ffspmv_apply_host (pinned host buffers, synchronous)"}


def synth_uniform(g, n, m):
    import synth
    return synth.uniform(g, n, m)


def cpu_baseline(M, budget_s=10.0):
    """The oracle as it stands (plain C, single thread) on the same matrix:
    repeated apply + transpose until ~budget_s of CPU time."""
    import oracle
    import synth
    m, rows, cols = M["m"], M["rows"], M["cols"]
    g = synth.rng(4242)
    x = synth.uniform(g, cols, m)
    xt = synth.uniform(g, rows, m)
    oracle.build()
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.apply(rows, cols, M["row"], M["col"], M["val"], m, x)
        oracle.apply_transpose(rows, cols, M["row"], M["col"], M["val"], m, xt)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    nnz_in = M["row"].size
    return {"value": 2 * nnz_in * reps / dt, "unit": "nnz/s", "cores": 1, "kind": "oracle",
            "sample": f"{reps} x (apply + transpose) of the full {M['name']} matrix "
                      f"({nnz_in} triples), {dt:.1f} s", "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ---------------------------------------------------------------- extras ---

def extras(ff, flush, stream, hbm_peak, args):
    import torch

    import synth
    res = {}
    # c3: GL7d-shaped hybrid apply (the "largest config" of the 60% target)
    M = synth.config_matrix("c3")
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], M["m"], no_transpose=True)
    info = A.info()
    g = synth.rng(2003)
    x = to_dev(synth.uniform(g, M["cols"], M["m"]))
    y = torch.empty(M["rows"], dtype=torch.int32, device="cuda")
    t = timed_steps([lambda: ff.ffspmv_apply(A, 1, x, 0, y, stream)], min(args.steps, 50),
                    args.warmup, flush, stream)
    ms = float(t.mean())
    res["c3_apply"] = {"nnz_per_s": info["nnz"] / (ms / 1e3), "ms": ms,
                       "alg_gbs": info["alg_bytes_apply"] / (ms / 1e3) / 1e9,
                       "frac": info["alg_bytes_apply"] / (ms / 1e3) / 1e9 / hbm_peak,
                       "stream_gbs": (info["stream_bytes"] + 4 * (M["rows"] + M["cols"])) / (ms / 1e3) / 1e9,
                       "traffic": ncu_traffic("c3_apply"),
                       "plan": {k: info[k] for k in ("strategy_apply", "panels", "panel_bands",
                                                     "bands_sell", "bands_csr", "bands_coos",
                                                     "long_rows", "slices", "padded_slots")}}
    del A, x, y, M
    # c4: block SpMM, m = 2^31 - 1
    M = synth.config_matrix("c4")
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], M["m"], no_transpose=True)
    info = A.info()
    g = synth.rng(2004)
    for k in (8, 16, 32):
        X = to_dev(synth.uniform(g, (M["cols"], k), M["m"]))
        Y = torch.empty((M["rows"], k), dtype=torch.int32, device="cuda")
        t = timed_steps([lambda: ff.ffspmv_apply_block(A, k, 1, X, 0, Y, stream)],
                        min(args.steps, 20), args.warmup, flush, stream)
        ms = float(t.mean())
        alg = (info["alg_bytes_apply"] - 4 * (M["rows"] + M["cols"])) + 4 * k * (M["rows"] + M["cols"])
        res[f"c4_block_k{k}"] = {"nnz_per_s": info["nnz"] / (ms / 1e3),
                                 "nnz_k_per_s": info["nnz"] * k / (ms / 1e3), "ms": ms,
                                 "alg_gbs": alg / (ms / 1e3) / 1e9,
                                 "frac": alg / (ms / 1e3) / 1e9 / hbm_peak}
        del X, Y
    del A, M
    # c5: block Wiedemann sequence, k = ku = 16, m = 65521
    M = synth.config_matrix("c5")
    n, k = M["rows"], 16
    A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], M["m"], no_transpose=True)
    info = A.info()
    g = synth.rng(2005)
    X = to_dev(synth.uniform(g, (n, k), M["m"]))
    U = to_dev(synth.uniform(g, (n, k), M["m"]))
    nsteps = 200
    S = torch.empty((nsteps, k, k), dtype=torch.int32, device="cuda")
    ws = torch.empty(ff.ffspmv_workspace_size(A, ff.OP_SEQUENCE, k, k), dtype=torch.uint8, device="cuda")
    ff.ffspmv_sequence(A, k, X, k, U, 10, S, None, ws, stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ff.ffspmv_kernel_launches()
    e0.record(stream)
    ff.ffspmv_sequence(A, k, X, k, U, nsteps, S, None, ws, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L_full = 2 * ((n + k - 1) // k) + 2
    step_bytes = (info["alg_bytes_apply"] - 4 * 2 * n) + 2 * 2 * k * n + 2 * k * n
    res["c5_sequence"] = {"steps_per_s": nsteps / (ms / 1e3), "ms_per_step": ms / nsteps,
                          "steps": nsteps, "L_full": L_full,
                          "full_L_seconds_extrapolated": L_full * ms / nsteps / 1e3,
                          "alg_gbs": step_bytes / (ms / nsteps / 1e3) / 1e9,
                          "frac": step_bytes / (ms / nsteps / 1e3) / 1e9 / hbm_peak,
                          "launches_per_step": (ff.ffspmv_kernel_launches() - l0) / nsteps,
                          "note": "L2 not flushed between steps (the iterate is reused by design)"}
    return res


# ------------------------------------------------------------- reference ---

def bench_reference(args):
    """The oracle arm: same config/metric/unit, CPU, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    M = synth.config_matrix(args.config)
    m, rows, cols = M["m"], M["rows"], M["cols"]
    g = synth.rng(synth.CONFIGS[args.config]["vseed"])
    x = synth.uniform(g, cols, m)
    xt = synth.uniform(g, rows, m)
    for _ in range(min(args.warmup, 1)):
        oracle.apply(rows, cols, M["row"], M["col"], M["val"], m, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.apply(rows, cols, M["row"], M["col"], M["val"], m, x)
        oracle.apply_transpose(rows, cols, M["row"], M["col"], M["val"], m, xt)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    nnz = M["row"].size
    value = 2 * nnz * args.steps / total
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic",
           "config": {"workload": f"{args.config}: " + _describe(args.config), "rows": rows,
                      "cols": cols, "nnz_triples": nnz, "modulus": m},
           "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": 1, "kind": "oracle",
                            "sample": f"{args.steps} x (apply + transpose) of the full "
                                      f"{args.config} matrix", "cpu": _cpu_model()},
           "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c3"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
