"""Small driver for ncu captures: builds one BASELINE config and launches the
chosen operation a few times (no timing -- numbers under ncu are never bench
values).  python tools/prof.py --config c2 --op apply --reps 4"""
import argparse
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
ap.add_argument("--op", default="apply", choices=["apply", "transpose", "block", "sequence"])
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--lib", default=None)
a = ap.parse_args()
if a.lib:
    ff.load(a.lib)

M = synth.config_matrix("c3", square=True) if a.config == "c3sq" else synth.config_matrix(a.config)
m, rows, cols = M["m"], M["rows"], M["cols"]
A = ff.ffspmv_create(rows, cols, M["row"], M["col"], M["val"], m, no_transpose=a.op != "transpose")
print(A.info(), flush=True)
g = synth.rng(1)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).cuda()


if a.op == "apply":
    x, y = dev(synth.uniform(g, cols, m)), torch.empty(rows, dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        ff.ffspmv_apply(A, 1, x, 0, y)
elif a.op == "transpose":
    x, y = dev(synth.uniform(g, rows, m)), torch.empty(cols, dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        ff.ffspmv_apply_transpose(A, 1, x, 0, y)
elif a.op == "block":
    X = dev(synth.uniform(g, (cols, a.k), m))
    Y = torch.empty((rows, a.k), dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        ff.ffspmv_apply_block(A, a.k, 1, X, 0, Y)
else:
    X = dev(synth.uniform(g, (rows, a.k), m))
    U = dev(synth.uniform(g, (rows, a.k), m))
    for _ in range(a.reps):
        A.sequence(X, a.steps, U)
torch.cuda.synchronize()
print("done")
