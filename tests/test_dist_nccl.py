"""The multi-GPU paths over NCCL, launched as one rank on the one GPU a test
box has (grid 1 x 1), checked bit-exactly against the oracle:
the Python drivers of dist.py (CudaBackend, NCCL process groups and
all-gathers, the on_step timing hook) and the C-ABI distributed handle over
a real NCCL communicator (ffspmv_comm_create from a unique id broadcast over
the torch group).  The N > 1 partition logic is covered by the gloo tests
and, through the C ABI, by tests/test_gpu_dist.py (in-process ranks)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys
sys.path.insert(0, os.environ["FF_ROOT"])
import numpy as np, torch, torch.distributed as dist
import oracle, synth
from paper_1004_3719_b200 import dist as fdist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
M = synth.config_matrix("c1")
n, m = M["rows"], M["m"]
g = synth.rng(77)
X = synth.uniform(g, (n, 5), m); U = synth.uniform(g, (n, 3), m)
L = 9
seen = []
S, V = fdist.sequence_2d(n, M["row"], M["col"], M["val"], m, X, L, U, fdist.CudaBackend("cuda:0"),
                         1, 1, want_vout=True, on_step=seen.append)
So, Vo = oracle.sequence(n, M["row"], M["col"], M["val"], m, X, L, U, want_vout=True)
assert np.array_equal(S, So) and np.array_equal(V, Vo), "sequence_2d != oracle"
assert seen == list(range(L + 1)), seen
Sr = fdist.sequence_rows(n, M["row"], M["col"], M["val"], m, X, L, U, fdist.CudaBackend("cuda:0"))
assert np.array_equal(Sr, So), "sequence_rows != oracle"
# the C-ABI distributed handle over a real NCCL communicator (1 x 1 grid):
# unique id broadcast over the torch group, ncclCommInitRank, ncclCommSplit,
# the per-step ncclAllGather and the result exchanges
import paper_1004_3719_b200 as ff
c = ff.comm_from_torch()
A = ff.ffspmv_create(n, n, M["row"], M["col"], M["val"], m, comm=c)
Xd = torch.from_numpy(X.view(np.int32)).cuda(); Ud = torch.from_numpy(U.view(np.int32)).cuda()
S2, V2 = A.sequence(Xd, L, Ud, want_vout=True)
torch.cuda.synchronize()
assert np.array_equal(S2.cpu().numpy().view(np.uint32).reshape(So.shape), So), "C-ABI dist S != oracle"
assert np.array_equal(V2.cpu().numpy().view(np.uint32), Vo), "C-ABI dist V != oracle"
del A
c.close()
dist.destroy_process_group()
print("nccl dist ok")
'''


@pytest.mark.gpu
def test_sequence_2d_cuda_nccl_one_rank():
    env = dict(os.environ, FF_ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT="29561",
               RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "nccl dist ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
