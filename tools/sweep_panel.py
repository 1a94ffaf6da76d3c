"""PANELS geometry sweep (tuning aid, not a bench): times y <- A x for a
BASELINE config under several band heights R (panel width W = the widest that
fits the shared-memory budget), L2 flushed between calls, CUDA events.

    python tools/sweep_panel.py --config c2 --rows 4088 8160 --reps 50
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1004_3719_b200 as ff
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--rows", type=int, nargs="+", default=[0])
ap.add_argument("--cols", type=int, default=262144)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--lib", default=None, help="alternative libffspmv.so (A/B timing)")
a = ap.parse_args()
if a.lib:
    ff.load(a.lib)

M = synth.config_matrix(a.config)
m, rows, cols = M["m"], M["rows"], M["cols"]
g = synth.rng(7)
x = torch.from_numpy(synth.uniform(g, cols, m).astype(np.uint32).view(np.int32)).cuda()
y = torch.empty(rows, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ref = None
for R in a.rows:
    kw = dict(strategy=ff.STRATEGY_PANELS) if R == 0 else dict(strategy=ff.STRATEGY_PANELS, panel_rows=R,
                                                                 panel_cols=a.cols)
    A = ff.ffspmv_create(rows, cols, M["row"], M["col"], M["val"], m, no_transpose=True, **kw)
    info = A.info()
    ts = []
    for i in range(a.reps + 5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ff.ffspmv_apply(A, 1, x, 0, y)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    out = y.cpu().numpy()
    if ref is None:
        ref = out
    same = bool(np.array_equal(out, ref))
    print(json.dumps({"lib": a.lib, "config": a.config, "R": R, "panels": info["panels"], "bands": info["panel_bands"],
                      "ms_mean": float(np.mean(ts)), "ms_min": float(np.min(ts)), "same_as_first": same}),
          flush=True)
    del A
