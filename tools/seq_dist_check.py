"""One-rank NCCL run of bench._seq_dist at full c5 size: the N > 1 sequence
line's code path (C-ABI distributed handle, NCCL communicator, per-step
ncclAllGather) measured on a one-GPU box (grid 1 x 1), and the row-sharded
c4 block apply line (bench._block_dist) the same way."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29571"), ("RANK", "0"), ("WORLD_SIZE", "1"),
             ("LOCAL_RANK", "0")):
    os.environ.setdefault(k, v)
import torch
import torch.distributed as dist

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import bench
import paper_1004_3719_b200 as ff

ff.load()
args = types.SimpleNamespace(steps=int(os.environ.get("STEPS", "40")), warmup=4)
args.no_extras = False
print(json.dumps(bench._seq_dist(args, 1, 0, 0)))
print(json.dumps(bench._block_dist(args, 1)))
dist.destroy_process_group()
