"""A/B timing of y <- A x (and A^T x) per k = 1 layout on a BASELINE config
(tuning aid; bench.py is the reported number).  CUDA events on the launching
stream, L2 flushed between calls, median of --reps.

    python tools/time_apply.py c3 --strategies 0 2 --reps 30 [--opt panel_xbits=8]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1004_3719_b200 as ff
    import synth
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--strategies", type=int, nargs="+", default=[0])
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--transpose", action="store_true")
    ap.add_argument("--opt", nargs="*", default=[])
    ap.add_argument("--lib", default=None)
    a = ap.parse_args()
    if a.lib:
        ff.load(a.lib)
    kw = {k: int(v) for k, v in (o.split("=") for o in a.opt)}
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    M = synth.config_matrix(a.config)
    g = synth.rng(7)
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    for s in a.strategies:
        A = ff.ffspmv_create(M["rows"], M["cols"], M["row"], M["col"], M["val"], M["m"],
                             no_transpose=not a.transpose, strategy=s, **kw)
        info = A.info()
        ops = [("apply", ff.ffspmv_apply, M["cols"], M["rows"], info["alg_bytes_apply"])]
        if a.transpose:
            ops.append(("transpose", ff.ffspmv_apply_transpose, M["rows"], M["cols"],
                        info["alg_bytes_transpose"]))
        for name, fn, nx, ny, alg in ops:
            x = torch.from_numpy(synth.uniform(g, nx, M["m"]).view(np.int32)).cuda()
            y = torch.empty(ny, dtype=torch.int32, device="cuda")
            ts = []
            for r in range(a.reps + 3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn(A, 1, x, 0, y, st)
                e1.record(st)
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            print(json.dumps({"config": a.config, "strategy": info[f"strategy_{'apply' if name == 'apply' else 'transpose'}"],
                              "op": name, "ms": round(ms, 5), "min_ms": round(min(ts), 5),
                              "alg_gbs": round(alg / ms / 1e6, 1), "frac": round(alg / ms / 1e6 / peak, 4),
                              "panels": info["panels"], "bands": info["panel_bands"],
                              "xbits": info["panel_xbits"], "stream_bytes": info["panel_stream_bytes"],
                              "opts": kw, "lib": a.lib}), flush=True)
        del A


if __name__ == "__main__":
    main()
