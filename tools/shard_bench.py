"""Frames/s of a sharded batch (C3 video frames / C5 small images) over the
ranks of a torchrun job: each rank runs the pipeline on its contiguous
shard (no data-path collective), device time per step = max over ranks.
Usage: torchrun --nproc-per-node N tools/shard_bench.py --config C3 [--gather]"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05062_b200 import Context, synth  # noqa: E402
from paper_1707_05062_b200.shard import BatchSharder, shard_bounds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3", choices=["C3", "C5"])
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--gather", action="store_true")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1 or "RANK" in os.environ:
    dist.init_process_group("nccl")
x = synth.generate(a.config, device="cuda")  # deterministic: every rank the same batch
n, h, w = x.shape
i0, i1 = shard_bounds(n, world, rank)
shard = x[i0:i1].contiguous()
del x
ctx = Context(torch.cuda.current_device())
sh = BatchSharder(ctx, n, w, h, world, rank)
for _ in range(2):
    sh.run(shard, gather=a.gather)
torch.cuda.synchronize()
if dist.is_initialized():
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    sh.run(shard, gather=a.gather)
e1.record()
e1.synchronize()
t = torch.tensor([e0.elapsed_time(e1) / a.steps], device="cuda")
if dist.is_initialized():
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
ms = float(t.item())
if rank == 0:
    print(json.dumps({"config": a.config, "n_gpus": world, "images": n, "ms_per_batch": ms,
                      "frames_per_s": n / ms * 1e3, "gpix_per_s": n * h * w / ms / 1e6,
                      "gather": a.gather, "scaling": "strong (fixed batch sharded over ranks)"}))
if dist.is_initialized():
    dist.destroy_process_group()
