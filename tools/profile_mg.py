"""Per-phase device-time breakdown on N GPUs (torchrun), rank 0 prints."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08812_b200 as d  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nd", type=int, default=200)
ap.add_argument("--nt", type=int, default=128)
ap.add_argument("--rank", type=int, default=8192)
ap.add_argument("--budget", type=int, default=50)
ap.add_argument("--algorithm", default="right")
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
nid = [d.nccl_unique_id() if rank == 0 else None]
if world > 1:
    dist.broadcast_object_list(nid, src=0)
v = d.synthetic_v(args.nd, args.nt, args.rank, 2024, threads=max(1, 16 // world))
eng = d.Engine(args.nd, args.nt, args.budget, device=local, world_size=world, rank=rank,
               nccl_id=nid[0] if world > 1 else None, keep_pristine=True, export_factor=True,
               algorithm=args.algorithm)
eng.gen_synthetic(v, args.rank, 1.0)
for r in range(3):
    eng.reset()
    if world > 1:
        dist.barrier()
    eng.run()
rows = eng.trace()
st = eng.stats()
tot = {k: round(sum(r[k] for r in rows), 3) for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update", "ms_round")}
res = {"rank": rank, "world": world, "time_to_k_ms": round(st["time_to_k_ms"], 3), "phase_ms": tot,
       "update_tflops": round(st["update_flops"] / max(st["update_ms"], 1e-9) / 1e9, 2)}
allr = [None] * world
if world > 1:
    dist.all_gather_object(allr, res)
else:
    allr = [res]
if rank == 0:
    for x in allr:
        print(json.dumps(x))
eng.close()
