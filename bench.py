#!/usr/bin/env python
"""Benchmark of the exact mod-m hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--no-extras] [--cpu-seconds S]

N = 1 headline: BASELINE configs[2], the largest single-GPU configuration
and the one the north star's 60 % HBM target is stated on -- the synthetic
GL7d-shaped 1,911,130 x 1,955,309 matrix (skewed "c + r" rows, every nonzero
+-1 mod 3).  One step = y <- A x (the hybrid-format apply),
inputs resident in HBM; L2 (126 MB) is flushed between timed steps by a
256 MB write outside the step's events.  value = canonical nonzeros per
second.  The dominant kernel's roofline, the e2e number through the
host-buffer C-ABI call, the clocks and the oracle (threaded, all host
cores) are on the same line; c2 apply + transpose, c4 block SpMM and the
c5 block Wiedemann sequence (with its oracle seconds per step) are extras.

N > 1 headline: BASELINE configs[4] -- the c5 block Wiedemann sequence
(N = 2^21, k = 16, m = 65521) as ONE problem split over the N ranks
(strong scaling), steps/s, device time max over ranks.  Its N = 1 point is
extras.c5_sequence of the N = 1 line.  Without torchrun, ``--gpus N``
relaunches itself under torch.distributed.run with N ranks.

--impl reference times the CPU oracle (oracle/, plain C, u128, threaded
timing mode on all host cores) on the same workload and metric, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mod-m SpMV nonzeros/sec & achieved HBM GB/s vs peak; seq steps/s at 1/2/4/8"
FLUSH_BYTES = 256 << 20
HEADLINE = "c3"
DESCRIBE = {
    "c2": "c2: 2^20 x 2^20, Poisson(10) nnz/row, 30% +-1, mod 65521; y <- A x and y' <- A^T x'",
    "c3": "c3: 1911130 x 1955309 GL7d-shaped, lognormal 'c + r' rows (mean ~19.5, 0.01% of "
          "1000-4000), every nonzero +-1 mod 3; y <- A x (hybrid-format apply)",
    "c4": "c4: 2^20 x 2^20, Poisson(10), 30% +-1, mod 2^31-1; Y <- A X, k = 8/16/32",
    "c5": "c5: 2^21 x 2^21, Poisson(10), 30% +-1, mod 65521; block Wiedemann sequence "
          "S_t = U^T A^t X, k = ku = 16",
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel(s) from the committed ncu
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


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ ours ---

def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


LAUNCHES = {"timed": 0}


def timed_steps(step_fns, steps, warmup, flush, stream):
    """Run warmup + steps of a list of launch closures, L2 flushed before each
    step (outside the events).  Returns per-call event times (ms, steps x
    len(step_fns)); LAUNCHES["timed"] = library kernels launched in the
    timed steps."""
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
    return np.array([[a.elapsed_time(b) for a, b in row] for row in ev])


def bench_ours(args):
    import torch

    import paper_1004_3719_b200 as ff

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    ff.load()
    if world > 1:
        out = bench_multi(args, world, rank, local)
    else:
        out = bench_single(args)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def bench_single(args):
    """N = 1: c3 apply headline (see module docstring)."""
    import torch

    import paper_1004_3719_b200 as ff
    import synth
    stream = torch.cuda.current_stream()
    hbm_peak, peak_src = peaks()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    M = synth.config_matrix(HEADLINE)
    m, rows, cols = M["m"], M["rows"], M["cols"]
    A = ff.ffspmv_create(rows, cols, M["row"], M["col"], M["val"], m, no_transpose=True)
    info = A.info()
    g = synth.rng(synth.CONFIGS[HEADLINE]["vseed"])
    x = to_dev(synth.uniform(g, cols, m))
    y = torch.empty(rows, dtype=torch.int32, device="cuda")
    fns = [lambda: ff.ffspmv_apply(A, 1, x, 0, y, stream)]
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        t = timed_steps(fns, args.steps, args.warmup, flush, stream)
    launches = LAUNCHES["timed"]
    total_ms = float(t.sum())
    nnz = info["nnz"]
    value = nnz * args.steps / (total_ms / 1e3)
    apply_ms = float(t[:, 0].mean())
    alg = info["alg_bytes_apply"]
    achieved = alg / (apply_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": ncu_traffic("c3_apply"),
                "kernel": _apply_kernel_name(ff, info), "peak_source": peak_src,
                "alg_bytes_per_launch": alg,
                "alg_bytes_note": "4 B per +-1 nonzero, 4 + e_v B per valued nonzero, 4 B per x "
                                  "and y element (DESIGN.md §6); one launch = one y <- A x",
                "launch_ms": round(apply_ms, 5)}
    out = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
           "accumulator": f"u{info['acc_bits_max']}", "data": "synthetic",
           "config": {"workload": DESCRIBE[HEADLINE], "rows": rows, "cols": cols, "nnz": nnz,
                      "modulus": m, "op": "y <- A x (alpha = 1, beta = 0)",
                      "l2": "flushed between timed steps (256 MB write)", "parallelism": "1 GPU"},
           "roofline": roofline, "gpu_launches": launches,
           "mflops_paper_unit": 2 * value / 1e6, "clocks": clk.summary()}
    out["e2e"] = _e2e(ff, A, args, rows, cols, m, g)
    out["plan"] = {k: info[k] for k in ("strategy_apply", "panels", "panel_bands",
                                        "gather_locality", "bands_sell", "bands_csr", "bands_coos",
                                        "slices", "long_rows", "nnz_pm1", "nnz_valued",
                                        "padded_slots", "stream_bytes", "panel_stream_bytes",
                                        "create_seconds")}
    out["cpu_baseline"] = cpu_baseline(M, budget_s=args.cpu_seconds)
    del A, x, y, M
    if not args.no_extras:
        out["extras"] = extras(ff, flush, stream, hbm_peak, args)
    return out


def _apply_kernel_name(ff, info):
    if info["strategy_apply"] == ff.STRATEGY_RUNS:
        return ("k_runs_pack + k_runs + k_runs_reduce (packed x panels in shared memory, "
                "register row runs), y <- A x")
    if info["strategy_apply"] == ff.STRATEGY_PANELS:
        return "k_panel + k_panel_reduce (x panels in shared memory), y <- A x"
    return "k_apply (rows layout), y <- A x"


def _e2e(ff, A, args, rows, cols, m, g):
    """The headline metric through the public host-buffer C-ABI call: each
    step copies x from pinned host memory, runs y <- A x, copies y back
    (ffspmv_apply_host, synchronous)."""
    import torch
    import synth
    xs = torch.empty(cols, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    ys = torch.empty(rows, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    xs[:] = synth.uniform(g, cols, m)
    for _ in range(args.warmup):
        ff.ffspmv_apply_host(A, ff.OP_APPLY, 1, xs, 0, ys)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ff.ffspmv_apply_host(A, ff.OP_APPLY, 1, xs, 0, ys)
    dt = time.perf_counter() - t0
    nnz = A.info()["nnz"]
    return {"value": nnz * args.steps / dt, "unit": "nnz/s", "h2d_bytes_per_step": 4 * cols,
            "d2h_bytes_per_step": 4 * rows,
            "api": "ffspmv_apply_host (pinned host buffers, synchronous, copies in the timed region)"}


def cpu_baseline(M, budget_s=10.0):
    """The oracle as it stands (plain C, u128) on the same matrix and metric:
    the threaded timing mode on all host cores (triples sorted by row
    beforehand, outside the timing), repeated until ~budget_s; plus one
    single-threaded apply for reference."""
    import oracle
    import synth
    m, rows, cols = M["m"], M["rows"], M["cols"]
    g = synth.rng(4242)
    x = synth.uniform(g, cols, m)
    oracle.build()
    T = oracle.host_threads()
    rs, cs, vs = oracle.sort_triples(M["row"], M["col"], M["val"])
    t0 = time.perf_counter()
    oracle.apply(rows, cols, M["row"], M["col"], M["val"], m, x)
    single = time.perf_counter() - t0
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.apply_mt(rows, cols, rs, cs, vs, m, x, nthreads=T)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    nnz = _canonical_nnz(M)
    return {"value": nnz * reps / dt, "unit": "nnz/s", "cores": T, "kind": "oracle",
            "sample": f"{reps} x y <- A x of the full {M['name']} matrix ({M['row'].size} triples), "
                      f"threaded timing mode on {T} threads, {dt:.1f} s",
            "single_thread_value": nnz / single, "cpu": _cpu_model()}


def _canonical_nnz(M):
    """Canonical nonzeros of a synthetic matrix (duplicates merged, residues
    0 dropped): the unit both arms count (R19).  Host counting only."""
    key = M["row"].astype(np.int64) * M["cols"] + M["col"]
    order = np.argsort(key, kind="stable")
    k, v = key[order], M["val"][order] % M["m"]
    starts = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
    sums = np.add.reduceat(v, starts) % M["m"]          # < 2^32 residues per key: int64-exact
    return int(np.count_nonzero(sums))


# ---------------------------------------------------------------- extras ---

def extras(ff, flush, stream, hbm_peak, args):
    import torch

    import oracle
    import synth
    res = {}
    # c2: apply + transpose apply (configs[1])
    M = synth.config_matrix("c2")
    A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], M["m"])
    info = A.info()
    g = synth.rng(2002)
    x = to_dev(synth.uniform(g, M["cols"], M["m"]))
    xt = to_dev(synth.uniform(g, M["rows"], M["m"]))
    y = torch.empty(M["rows"], dtype=torch.int32, device="cuda")
    yt = torch.empty(M["cols"], dtype=torch.int32, device="cuda")
    t = timed_steps([lambda: ff.ffspmv_apply(A, 1, x, 0, y, stream),
                     lambda: ff.ffspmv_apply_transpose(A, 1, xt, 0, yt, stream)],
                    min(args.steps, 50), args.warmup, flush, stream)
    ms_a, ms_t = float(t[:, 0].mean()), float(t[:, 1].mean())
    res["c2_apply_transpose"] = {
        "nnz_per_s": 2 * info["nnz"] / ((ms_a + ms_t) / 1e3), "apply_ms": ms_a,
        "transpose_ms": ms_t, "frac_apply": info["alg_bytes_apply"] / (ms_a / 1e3) / 1e9 / hbm_peak,
        "frac_transpose": info["alg_bytes_transpose"] / (ms_t / 1e3) / 1e9 / hbm_peak,
        "traffic_apply": ncu_traffic("c2_apply"), "strategy": info["strategy_apply"]}
    del A, x, xt, y, yt, M
    # c4: block SpMM, m = 2^31 - 1 (configs[3])
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
                                 "frac": alg / (ms / 1e3) / 1e9 / hbm_peak,
                                 "traffic": ncu_traffic(f"c4_block_k{k}")}
        del X, Y
    del A, M
    # c5: block Wiedemann sequence, k = ku = 16, m = 65521 (configs[4]; the
    # N = 1 point of the N > 1 headline)
    res["c5_sequence"] = _seq_single(ff, stream, hbm_peak, args)
    # c5 oracle seconds per step (threaded mode, 2 steps, extrapolated to L)
    res["c5_sequence"]["cpu_baseline"] = _c5_oracle(oracle, synth)
    # the GL7d-shaped matrix (square variant) mod 3: the sequence with a u8
    # iterate (SURVEY a-8)
    res["c3sq_sequence_m3"] = _seq_single(ff, stream, hbm_peak, args, cfg="c3sq")
    return res


def _c5_inputs(synth, cfg="c5"):
    M = synth.config_matrix("c5") if cfg == "c5" else synth.config_matrix("c3", square=True)
    n, k = M["rows"], 16
    g = synth.rng(2005 if cfg == "c5" else 2033)
    X = synth.uniform(g, (n, k), M["m"])
    U = synth.uniform(g, (n, k), M["m"])
    return M, n, k, X, U


def _seq_single(ff, stream, hbm_peak, args, cfg="c5"):
    import torch

    import synth
    M, n, k, X, U = _c5_inputs(synth, cfg)
    A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], M["m"], no_transpose=True)
    info = A.info()
    Xd, Ud = to_dev(X), to_dev(U)
    nsteps = 200
    S = torch.empty((nsteps, k, k), dtype=torch.int32, device="cuda")
    ws = torch.empty(ff.ffspmv_workspace_size(A, ff.OP_SEQUENCE, k, k), dtype=torch.uint8, device="cuda")
    ff.ffspmv_sequence(A, k, Xd, k, Ud, 10, S, None, ws, stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ff.ffspmv_kernel_launches()
    e0.record(stream)
    ff.ffspmv_sequence(A, k, Xd, k, Ud, nsteps, S, None, ws, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L_full = 2 * ((n + k - 1) // k) + 2
    e_v = info["iterate_bytes"]
    step_bytes = (info["alg_bytes_apply"] - 4 * 2 * n) + 2 * e_v * k * n + e_v * k * n
    return {"workload": DESCRIBE["c5"] if cfg == "c5" else
            "c3 recipe with cols = rows (1911130^2, every nonzero +-1 mod 3), k = ku = 16, u8 iterate",
            "steps_per_s": nsteps / (ms / 1e3), "ms_per_step": ms / nsteps, "steps": nsteps,
            "iterate_bytes": e_v,
            "L_full": L_full, "full_L_seconds_extrapolated": L_full * ms / nsteps / 1e3,
            "alg_gbs": step_bytes / (ms / nsteps / 1e3) / 1e9,
            "frac": step_bytes / (ms / nsteps / 1e3) / 1e9 / hbm_peak,
            "alg_bytes_per_step": step_bytes,
            "launches_per_step": (ff.ffspmv_kernel_launches() - l0) / nsteps,
            "traffic": ncu_traffic("c5_sequence_step" if cfg == "c5" else "c3sq_sequence_step"),
            "note": "one ffspmv_sequence call of 200 steps (S_0..S_199); L2 not flushed between "
                    "steps (the iterate is reused by design)"}


def _c5_oracle(oracle, synth):
    M, n, k, X, U = _c5_inputs(synth)
    T = oracle.host_threads()
    rs, cs, vs = oracle.sort_triples(M["row"], M["col"], M["val"])
    t0 = time.perf_counter()
    oracle.sequence_mt(n, rs, cs, vs, M["m"], X, 2, U, nthreads=T)
    dt = time.perf_counter() - t0
    L_full = 2 * ((n + k - 1) // k) + 2
    return {"seconds_per_step": dt / 2, "full_L_seconds_extrapolated": dt / 2 * L_full,
            "extrapolated": True, "cores": T, "kind": "oracle",
            "sample": f"2 steps of the full c5 sequence (projection + block apply), threaded "
                      f"timing mode on {T} threads, extrapolated to L = {L_full}"}


# ------------------------------------------------------------- multi-GPU ---

def bench_multi(args, world, rank, local):
    """N > 1: the c5 sequence as one problem split over the ranks (strong
    scaling).  steps/s over the timed steps, device events, max over ranks."""
    r = _seq_dist(args, world, rank, local)
    hbm_peak, _ = peaks()
    out = {"metric": METRIC, "value": r.get("steps_per_s"), "unit": "steps/s", "n_gpus": world,
           "steps": r.get("steps", args.steps), "warmup": args.warmup,
           "ms_per_step": r.get("ms_per_step"), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "u16 iterate / u32 I/O", "data": "synthetic",
           "config": {"workload": DESCRIBE["c5"], "rows": 1 << 21, "k": 16, "ku": 16,
                      "modulus": 65521, "parallelism": r.get("parallelism"),
                      "l2": "not flushed between steps (the iterate is reused by design)"},
           "gpu_launches": r.get("launches"), "detail": r}
    if not args.no_extras:
        out["extras"] = {"c4_block_k16_row_sharded": _block_dist(args, world)}
    return out


def _block_dist(args, world):
    """c4 block SpMM (k = 16, m = 2^31 - 1) as ONE problem row-sharded over
    the ranks through a distributed handle (ffspmv_apply_block: each rank its
    nnz-balanced row band, then the all-gather of the Y bands so Y is whole on
    every rank); nnz*k/s from device events around each call, max over
    ranks, L2 not flushed."""
    import torch

    import paper_1004_3719_b200 as ff
    import synth
    try:
        M = synth.config_matrix("c4")
        n, k = M["rows"], 16
        comm = ff.comm_from_torch()
        A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], M["m"], comm=comm, dist_rows=world)
        g = synth.rng(2004)
        X = to_dev(synth.uniform(g, (n, k), M["m"]))
        Y = torch.empty((n, k), dtype=torch.int32, device="cuda")
        stream = torch.cuda.current_stream()
        for _ in range(max(3, args.warmup)):
            ff.ffspmv_apply_block(A, k, 1, X, 0, Y, stream)
        ts = []
        for _ in range(max(1, min(args.steps, 20))):
            torch.cuda.synchronize()
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ff.ffspmv_apply_block(A, k, 1, X, 0, Y, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            tt = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ts.append(float(tt.item()))
        ms = float(np.median(ts))
        nnz = _canonical_nnz(M)
        del A
        comm.close()
        return {"nnz_k_per_s": nnz * k / (ms / 1e3), "ms": ms, "grid": [world, 1],
                "note": "row bands of A over the ranks, X replicated, Y all-gathered (included)"}
    except Exception as e:                       # the line must still print
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def _seq_dist(args, world, rank, local):
    """c5 sequence across the ranks through the C-ABI distributed handle
    (ffspmv_create with an NCCL communicator; the per-step band SpMM with its
    fused projection and the ncclAllGather of the band iterates run inside
    ffspmv_sequence) on the grid grid_shape picks.  Steady-state time per
    step = (T(L0 + steps) - T(L0)) / steps over two calls, each timed with
    device events around the call, max over ranks (the difference removes
    the per-call prologue and the final exchange of S)."""
    import torch

    import paper_1004_3719_b200 as ff
    import synth
    from paper_1004_3719_b200 import dist as fdist
    try:
        M, n, k, X, U = _c5_inputs(synth)
        steps = max(1, args.steps)
        pr, pc = fdist.grid_shape(world, k, n=n, nnz=len(M["row"]), iterate_bytes=2)
        comm = ff.comm_from_torch()
        A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], M["m"], comm=comm, dist_rows=pr)
        Xd, Ud = to_dev(X), to_dev(U)
        stream = torch.cuda.current_stream()
        L0 = max(2, args.warmup)
        ws = torch.empty(ff.ffspmv_workspace_size(A, ff.OP_SEQUENCE, k, k), dtype=torch.uint8, device="cuda")
        S = torch.empty((L0 + steps, k, k), dtype=torch.int32, device="cuda")
        for _ in range(2):                                     # warm-up calls
            ff.ffspmv_sequence(A, k, Xd, k, Ud, L0, S, None, ws, stream)
        times, launches = [], 0
        for L in (L0, L0 + steps):
            torch.cuda.synchronize()
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = ff.ffspmv_kernel_launches()
            e0.record(stream)
            ff.ffspmv_sequence(A, k, Xd, k, Ud, L, S, None, ws, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            launches = ff.ffspmv_kernel_launches() - l0
            tt = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            times.append(float(tt.item()))
        ms = (times[1] - times[0]) / steps
        del A
        comm.close()
        return {"steps_per_s": 1e3 / ms, "ms_per_step": ms, "steps": steps, "grid": [pr, pc],
                "launches": launches, "call_ms": times,
                "parallelism": f"2-D grid {pr} x {pc} (row bands x column blocks), C-ABI "
                               "distributed handle, ncclAllGather of the u16 band iterates per step"}
    except Exception as e:                       # the line must still print
        return {"error": f"{type(e).__name__}: {e}"[:300]}


# ------------------------------------------------------------- reference ---

def bench_reference(args):
    """The oracle arm: the headline workload, metric and unit, on the host's
    cores (threaded timing mode, triples sorted beforehand), rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    T = oracle.host_threads()
    cfg = HEADLINE if world == 1 else "c5"
    if cfg == "c5":
        M, n, k, X, U = _c5_inputs(synth)
        rs, cs, vs = oracle.sort_triples(M["row"], M["col"], M["val"])
        step = lambda: oracle.sequence_mt(n, rs, cs, vs, M["m"], X, 1, U, nthreads=T)  # noqa: E731
        units, unit = 1, "steps/s"
    else:
        M = synth.config_matrix(cfg)
        m, rows, cols = M["m"], M["rows"], M["cols"]
        g = synth.rng(synth.CONFIGS[cfg]["vseed"])
        x = synth.uniform(g, cols, m)
        rs, cs, vs = oracle.sort_triples(M["row"], M["col"], M["val"])
        step = lambda: oracle.apply_mt(rows, cols, rs, cs, vs, m, x, nthreads=T)  # noqa: E731
        units, unit = _canonical_nnz(M), "nnz/s"
    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = units * args.steps / total
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "weak" if cfg != "c5" else "strong",
           "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": DESCRIBE[cfg]},
           "cpu_baseline": {"value": value, "unit": unit, "cores": T, "kind": "oracle",
                            "sample": f"{args.steps} steps of the full {cfg} workload (one step = "
                                      f"{'one sequence step' if cfg == 'c5' else 'y <- A x'}), "
                                      f"threaded timing mode on {T} threads, after "
                                      f"{args.warmup} warm-up steps", "cpu": _cpu_model()},
           "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ main ---

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
