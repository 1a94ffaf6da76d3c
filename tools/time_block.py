"""Times the block apply Y <- A X (c4 shape by default) for k = 8/16/32, L2
flushed between calls, CUDA events (tuning aid, A/B with --lib; bench.py is
the reported number).  Also hashes Y so variants can be compared."""
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
ap.add_argument("--config", default="c4")
ap.add_argument("--ks", type=int, nargs="+", default=[8, 16, 32])
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--lib", default=None)
a = ap.parse_args()
if a.lib:
    ff.load(a.lib)
M = synth.config_matrix(a.config)
m, rows, cols = M["m"], M["rows"], M["cols"]
A = ff.ffspmv_create(rows, cols, M["row"], M["col"], M["val"], m, no_transpose=True)
g = synth.rng(2004)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"lib": a.lib, "config": a.config}
for k in a.ks:
    X = torch.from_numpy(synth.uniform(g, (cols, k), m).view(np.int32)).cuda()
    Y = torch.empty((rows, k), dtype=torch.int32, device="cuda")
    for _ in range(3):
        ff.ffspmv_apply_block(A, k, 1, X, 0, Y)
    ts = []
    for _ in range(a.reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ff.ffspmv_apply_block(A, k, 1, X, 0, Y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    h = int(np.frombuffer(Y.cpu().numpy().tobytes(), np.uint32).astype(np.uint64).sum() % (1 << 61))
    out[f"k{k}"] = {"ms_median": float(np.median(ts)), "hash": h}
print(json.dumps(out), flush=True)
