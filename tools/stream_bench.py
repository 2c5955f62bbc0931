"""Out-of-HBM streaming store measurement (BASELINE configs[4] analogue).

K lives only in pinned host memory (storage=stream, left-looking W-resident
algorithm); per round the chosen column's blocks (this rank's rows) are copied
H2D on a side stream while the GEMM runs. Reports time-to-k, the H2D time and
the part of it not hidden behind compute (exposed), on N GPUs (torchrun)."""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08812_b200 as d  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nd", type=int, default=75)
ap.add_argument("--nt", type=int, default=420)
ap.add_argument("--rank", type=int, default=24576)
ap.add_argument("--budget", type=int, default=50)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--weak", action="store_true", help="nd scaled by the GPU count")
ap.add_argument("--attach", action="store_true",
                help="caller-owned pinned block rows (dsel_attach_host_rows) instead of the engine store")
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")
nd = args.nd * (world if args.weak else 1)
nid = [d.nccl_unique_id() if rank == 0 else None]
if world > 1:
    dist.broadcast_object_list(nid, src=0)
t0 = time.time()
v = d.synthetic_v(nd, args.nt, args.rank, 2024, threads=max(1, 16 // world))
eng = d.Engine(nd, args.nt, args.budget, device=local, world_size=world, rank=rank,
               nccl_id=nid[0] if world > 1 else None, algorithm="left", storage=2)
eng.gen_synthetic(v, args.rank, 1.0)
del v
if args.attach:
    mine = [j for j in range(nd) if j % world == rank]
    re = nd * args.nt * args.nt
    host = torch.empty(len(mine) * re, dtype=torch.float64).pin_memory()
    hv = host.numpy()
    for i, j in enumerate(mine):
        hv[i * re:(i + 1) * re] = eng.read_block_row(j)
    eng.attach_host_rows(host)
setup = time.time() - t0
best = None
for r in range(args.runs):
    eng.reset()
    if world > 1:
        dist.barrier()
    eng.run()
    st = eng.stats()
    if best is None or st["time_to_k_ms"] < best["time_to_k_ms"]:
        best = st
rows = eng.trace()
chosen = [x["chosen_index"] for x in rows]
res = {"rank": rank, "world": world, "nd": nd, "nt": args.nt, "budget": args.budget,
       "host_store_gb": round(nd * args.nt * nd * args.nt * 8 / world / 1e9, 2),
       "time_to_k_s": round(best["time_to_k_ms"] / 1e3, 4),
       "io_ms": round(best["io_ms"], 2), "io_exposed_ms": round(best["io_exposed_ms"], 2),
       "io_hidden_frac": round(1 - best["io_exposed_ms"] / max(best["io_ms"], 1e-9), 4),
       "h2d_gb": round(best["h2d_bytes"] / 1e9, 3),
       "update_tflops": round(best["update_flops"] / max(best["update_ms"], 1e-9) / 1e9, 2),
       "setup_s": round(setup, 1), "chosen_first": chosen[:6], "attach": args.attach,
       "phase_ms": {k: round(sum(x[k] for x in rows), 2)
                    for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update", "ms_round")},
       "first_rounds_ms": [round(x["ms_round"], 3) for x in rows[:6]],
       "last_rounds_ms": [round(x["ms_round"], 3) for x in rows[-4:]]}
allr = [None] * world
if world > 1:
    dist.all_gather_object(allr, res)
else:
    allr = [res]
if rank == 0:
    print(json.dumps({"streaming": allr}))
eng.close()
