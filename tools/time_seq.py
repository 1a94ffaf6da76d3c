"""Times the block Wiedemann sequence step (c5 shape by default) through
ffspmv_sequence: steps/s over --steps after a warm-up (tuning aid, A/B with
--lib; bench.py is the reported number)."""
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
ap.add_argument("--config", default="c5")
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--steps", type=int, default=200)
ap.add_argument("--lib", default=None)
a = ap.parse_args()
if a.lib:
    ff.load(a.lib)
M = synth.config_matrix("c3", square=True) if a.config == "c3sq" else synth.config_matrix(a.config)
n, k = M["rows"], a.k
A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], M["m"], no_transpose=True)
g = synth.rng(2005)
X = torch.from_numpy(synth.uniform(g, (n, k), M["m"]).view(np.int32)).cuda()
U = torch.from_numpy(synth.uniform(g, (n, k), M["m"]).view(np.int32)).cuda()
S = torch.empty((a.steps, k, k), dtype=torch.int32, device="cuda")
ws = torch.empty(ff.ffspmv_workspace_size(A, ff.OP_SEQUENCE, k, k), dtype=torch.uint8, device="cuda")
ff.ffspmv_sequence(A, k, X, k, U, 10, S, None, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ff.ffspmv_sequence(A, k, X, k, U, a.steps, S, None, ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
h = int(np.frombuffer(S.cpu().numpy().tobytes(), np.uint32).astype(np.uint64).sum() % (1 << 61))
print(json.dumps({"lib": a.lib, "config": a.config, "k": k, "ms_per_step": ms / a.steps,
                  "steps_per_s": a.steps / (ms / 1e3), "S_hash": h}), flush=True)
