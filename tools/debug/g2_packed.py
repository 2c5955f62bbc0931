"""Debug: G=2 packed vs full panels on small reference cases (torchrun 2)."""
import json, os, sys
import numpy as np
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2604_08812_b200 as d
from oracle import oracle as O
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
for (nd, nt, g, rk, seed, B) in [(10, 2, 0.8, 20, 201, 3), (8, 2, 0.8, 20, 5, 3), (8, 4, 0.8, 40, 5, 3)]:
    k = O.random_hessian(nd, nt, g, rk, seed)
    want = O.greedy_select(k, nd, nt, B)
    for packed in (True,):
        for p2p in ("0",):
            os.environ["DSEL_P2P"] = p2p
            cid = [d.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(cid, src=0)
            with d.Engine(nd, nt, B, device=rank, world_size=world, rank=rank, nccl_id=cid[0], packed=packed) as e:
                e.load_k(k)
                out = []
                for t in range(B):
                    gains = e.peek_gains()
                    out.append(gains.copy())
                    e.step(forced=want.chosen[t])
            allg = [None] * world
            dist.all_gather_object(allg, out)
            if rank == 0:
                ref = O.replay_gains(k, nd, nt, want.chosen)
                print(f"nd={nd} nt={nt} chosen={want.chosen}", flush=True)
                for t in range(B):
                    comb = np.where(np.isnan(allg[0][t]), allg[1][t], allg[0][t])
                    print("  round", t, "err by sensor:", ["%d:%.0e" % (j, abs(comb[j] - ref[t][j])) for j in range(nd) if not np.isnan(ref[t][j])], flush=True)
dist.destroy_process_group()
