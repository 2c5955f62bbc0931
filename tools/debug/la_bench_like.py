"""Debug (bounded): the bench's engine sequence with look-ahead on, progress per rank."""
import os, sys, time
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2604_08812_b200 as d
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
log = open(os.path.join(ROOT, "gpurun_out", f"la_dbg_r{rank}.log"), "w", buffering=1)
t0 = time.time()
def say(*a):
    log.write(f"{time.time() - t0:8.2f} " + " ".join(str(x) for x in a) + "\n")
def nid():
    b = [d.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(b, src=0)
    return b[0]
nd, nt, rk, B = 200, 128, 8192, 50
v = d.synthetic_v(nd, nt, rk, 2024)
say("peak", d.measure_fp64_peak(rank))
mode = sys.argv[1] if len(sys.argv) > 1 else "full"
if mode in ("full", "src"):
    with d.Engine(nd, nt, B, device=rank, world_size=world, rank=rank, nccl_id=nid(), packed=False, storage="hbm") as src:
        src.gen_synthetic(v, rk, 1.0)
        rows = [src.read_block_row(j) for j in range(nd) if j % world == rank]
    say("src done")
eng = d.Engine(nd, nt, B, device=rank, world_size=world, rank=rank, nccl_id=nid(), keep_pristine=True, export_factor=True)
eng.gen_synthetic(v, rk, 1.0)
say("engine ready", eng.plan())
for it in range(4):
    eng.reset()
    say("reset", it)
    dist.barrier()
    for r in range(B):
        info = eng.step()
        if r % 10 == 0 or r > B - 4:
            say("run", it, "round", r, info["chosen_index"])
    st = eng.stats()
    say("run", it, "time_to_k_ms", st["time_to_k_ms"], [x["chosen_index"] for x in eng.trace()][:6])
eng.close()
say("done")
dist.destroy_process_group()
