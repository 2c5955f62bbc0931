"""Large-scale selection with K formed on the device (600 x Nt=420,
n = 252,000, ~508 GB FP64 K, select 175; V = 165 GB never exists on the host).

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \\
        --master-port P tools/c4_run.py [--nd 600 --nt 420 --budget 175 --vrank 81920]

One process per GPU; each rank forms its own block columns of K = sigma^2 I + V V^T
with the Schur update kernel (gen_synthetic_device, Philox V) and the selection runs
on the resident block-lower store. Prints one JSON line (rank 0): time-to-k (max
over ranks), update TFLOP/s per GPU, K-formation time, phase totals."""
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
ap.add_argument("--nd", type=int, default=600)
ap.add_argument("--nt", type=int, default=420)
ap.add_argument("--budget", type=int, default=175)
ap.add_argument("--vrank", type=int, default=81920)
ap.add_argument("--sigma", type=float, default=1.0)
ap.add_argument("--seed", type=int, default=2024)
ap.add_argument("--algorithm", default="right")
ap.add_argument("--runs", type=int, default=1, help="selections (K re-formed before each)")
args = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("gloo")


def maxr(x):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sumr(x):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


nid = [d.nccl_unique_id() if rank == 0 else None]
if world > 1:
    dist.broadcast_object_list(nid, src=0)
t0 = time.time()
eng = d.Engine(args.nd, args.nt, args.budget, device=local, world_size=world, rank=rank,
               nccl_id=nid[0] if world > 1 else None, algorithm=args.algorithm)
t_create = time.time() - t0
results = []
for r in range(args.runs):
    if world > 1:
        dist.barrier()
    t0 = time.time()
    eng.gen_synthetic_device(args.vrank, args.sigma, args.seed)
    t_gen = maxr(time.time() - t0)
    if world > 1:
        dist.barrier()
    eng.run()
    st = eng.stats()
    rows = eng.trace()
    ph = {k: round(sum(x[k] for x in rows), 1) for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update")}
    results.append(dict(time_to_k_s=round(maxr(st["time_to_k_ms"]) / 1e3, 3),
                        update_s_max_rank=round(maxr(st["update_ms"]) / 1e3, 3),
                        update_flops_all=sumr(st["update_flops"]),
                        update_tflops_per_gpu=round(st["update_flops"] / max(st["update_ms"], 1e-9) / 1e9, 2),
                        k_formation_s=round(t_gen, 1), phase_ms_rank0=ph,
                        chosen_first=[x["chosen_index"] for x in rows[:10]],
                        objective=rows[-1]["objective"], n_selected=len(rows)))
dev_gb = eng.device_bytes / 1e9
eng.close()
if rank == 0:
    best = min(results, key=lambda x: x["time_to_k_s"])
    n = args.nd * args.nt
    print(json.dumps({"workload": f"{args.nd} candidates x Nt={args.nt} (n={n}) select {args.budget}, "
                                  f"device Philox V rank {args.vrank}, sigma {args.sigma}, seed {args.seed}",
                      "n_gpus": world, "algorithm": args.algorithm,
                      "k_bytes_full": n * n * 8, "device_gb_per_gpu": round(dev_gb, 1),
                      "engine_create_s": round(t_create, 1), **best,
                      "update_tflops_all_gpus": round(best["update_flops_all"] / best["update_s_max_rank"] / 1e12, 2),
                      "frac_of_fp64_peak": round(best["update_flops_all"] / best["update_s_max_rank"] / 1e12
                                                 / (37.1 * world), 4)}), flush=True)
if world > 1:
    dist.destroy_process_group()
