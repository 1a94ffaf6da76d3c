"""One-rank NCCL run of bench._seq_dist at full c5 size (checks the N > 1 sequence line's code path on a one-GPU box)."""
import os, sys, json, types
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import bench
import paper_1004_3719_b200 as ff
ff.load()
args = types.SimpleNamespace(steps=20, warmup=3)
print(json.dumps(bench._seq_dist(args, 1, 0, 0)))
dist.destroy_process_group()
