"""Multi-GPU check (one process per GPU): run under
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mp_engine_check.py [c1|c2|wave]
Every rank must reproduce the reference golden sequence and gains, and all
ranks must agree bitwise (the fold and the broadcast factor are identical)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_08812_b200 as d  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
nid = [d.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(nid, src=0)
if which == "random":
    # reference random_hessian cases (odd nt, nt = 2 (mod 4): shifted c-side
    # tiles) on every algorithm / storage variant; all ranks must agree
    from oracle import oracle as O  # checker only
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "random.json")))["cases"]
    extra = [dict(n_sensors=40, n_steps=6, gamma=0.9, rank=150, seed=11, budget=12),
             dict(n_sensors=33, n_steps=10, gamma=1.1, rank=200, seed=12, budget=9)]
    bad = 0
    for c in cases + extra:
        nd, nt = c["n_sensors"], c["n_steps"]
        k = O.random_hessian(nd, nt, c["gamma"], c["rank"], c["seed"])
        if "chosen" not in c:
            w = O.greedy_select(k, nd, nt, c["budget"])
            c = dict(c, chosen=list(w.chosen), gains=list(w.gains))
        for kw in (dict(), dict(full_square=True), dict(algorithm="left")):
            cid = [d.nccl_unique_id() if rank == 0 else None]  # one id per communicator
            dist.broadcast_object_list(cid, src=0)
            eng = d.Engine(nd, nt, c["budget"], device=local, world_size=world, rank=rank,
                           nccl_id=cid[0], **kw)
            eng.load_k(k)
            eng.run()
            rows = eng.trace()
            eng.close()
            ok = [r["chosen_index"] for r in rows] == list(c["chosen"])
            for r, g in zip(rows, c["gains"]):
                ok = ok and abs(r["gain"] - g) <= 1e-9 * max(abs(g), 1.0)
            if not ok:
                bad += 1
                print(f"rank {rank} MISMATCH nd={nd} nt={nt} {kw}", flush=True)
    # candidate subsets (uneven ownership of the remaining positions)
    nd, nt = 30, 6
    k = O.random_hessian(nd, nt, 1.0, 100, 21)
    cands = [0, 1, 2, 4, 7, 8, 11, 13, 17, 18, 22, 25, 29]
    want = O.greedy_select(k, nd, nt, 7, candidates=cands)
    for kw in (dict(), dict(algorithm="left"), dict(full_square=True)):
        cid = [d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        eng = d.Engine(nd, nt, 7, candidates=cands, device=local, world_size=world, rank=rank,
                       nccl_id=cid[0], **kw)
        eng.load_k(k)
        eng.run()
        rows = eng.trace()
        eng.close()
        ok = [r["chosen_index"] for r in rows] == list(want.chosen)
        for r, g in zip(rows, want.gains):
            ok = ok and abs(r["gain"] - g) <= 1e-9 * max(abs(g), 1.0)
        if not ok:
            bad += 1
            print(f"rank {rank} MISMATCH subset {kw}", flush=True)
    print(f"rank {rank}/{world} random: {'OK' if not bad else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)
if which == "replay":
    # every remaining candidate's gain at every round (forced replay along the
    # reference sequence), gathered over the ranks -- full gain vectors, not
    # just winners (a wrong loser would not change the sequence), on every
    # storage variant
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c1.json")))
    v = d.synthetic_v(64, 32, 2048, 2024)
    bad = 0
    for kw in (dict(), dict(packed=False), dict(full_square=True), dict(algorithm="left")):
        cid = [d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        with d.Engine(64, 32, 16, device=local, world_size=world, rank=rank, nccl_id=cid[0], **kw) as eng:
            eng.gen_synthetic(v, 2048, 1.0)
            mine = []
            for s in gold["chosen"]:
                mine.append(eng.peek_gains())
                eng.step(forced=s)
        allg = [None] * world
        dist.all_gather_object(allg, mine)
        for rnd in range(16):
            for j in range(64):
                want = gold["replay_gains"][rnd][j]
                got = [a[rnd][j] for a in allg if not np.isnan(a[rnd][j])]
                if want is None:
                    ok = not got
                else:
                    ok = len(got) == 1 and abs(got[0] - want) <= 1e-9 * max(abs(want), 1.0)
                if not ok:
                    bad += 1
                    if bad < 5:
                        print(f"rank {rank} {kw} round {rnd} sensor {j}: {got} vs {want}", flush=True)
    print(f"rank {rank}/{world} replay: {'OK' if not bad else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)
if which == "lookahead":
    # look-ahead rounds (Nt = 128) at world size > 1: the winner's panel strip
    # is read over NVLink after the owner's flag; gains bit-identical to the
    # plain schedule and to one GPU
    from oracle import oracle as O  # checker only
    nd, nt, b = 16, 128, 8
    k = O.random_hessian(nd, nt, 1.0, 1800, 4)
    want = O.greedy_select(k, nd, nt, b)
    res = {}
    for la in ("1", "0"):
        os.environ["DSEL_LOOKAHEAD"] = la
        cid = [d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        with d.Engine(nd, nt, b, device=local, world_size=world, rank=rank, nccl_id=cid[0],
                      keep_pristine=True) as eng:
            eng.load_k(k)
            runs = []
            for _ in range(3):  # reruns after dsel_reset: the flag sequences carry over
                eng.reset()
                eng.run()
                runs.append([(r["chosen_index"], r["gain"]) for r in eng.trace()])
            res[la] = runs[0] if runs[0] == runs[1] == runs[2] else None
    os.environ["DSEL_LOOKAHEAD"] = "0"
    one = None
    if rank == 0:
        with d.Engine(nd, nt, b, device=local) as eng:
            eng.load_k(k)
            eng.run()
            one = [(r["chosen_index"], r["gain"]) for r in eng.trace()]
    box = [one]
    dist.broadcast_object_list(box, src=0)
    ok = (res["1"] == res["0"] == box[0] and [c for c, _ in res["1"]] == list(want.chosen))
    print(f"rank {rank}/{world} lookahead: {'OK' if ok else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)
if which == "device":
    # K formed on every rank by the update kernel from the device Philox V; the
    # sequence must match the oracle on the same K (numpy V) at any world size
    from oracle import oracle as O  # checker only
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from philox_ref import philox_v
    nd, nt, rk, B, seed = 48, 16, 400, 12, 5
    v = philox_v(nd, nt, rk, seed)
    want = O.greedy_select(O.dense_to_blocks(0.25 * np.eye(nd * nt) + v @ v.T, nd, nt), nd, nt, B)
    bad = 0
    for kw in (dict(), dict(algorithm="left")):
        cid = [d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        with d.Engine(nd, nt, B, device=local, world_size=world, rank=rank, nccl_id=cid[0], **kw) as eng:
            eng.gen_synthetic_device(rk, 0.5, seed)
            eng.run()
            rows = eng.trace()
        ok = [r["chosen_index"] for r in rows] == list(want.chosen)
        for r, g in zip(rows, want.gains):
            ok = ok and abs(r["gain"] - g) <= 1e-9 * max(abs(g), 1.0)
        bad += not ok
    print(f"rank {rank}/{world} device: {'OK' if not bad else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)
if which in ("lti", "attach"):
    # lti: K assembled on every rank from the wave config (bit-exact); attach:
    # the streaming store over each rank's own pinned block rows of the wave K
    lti = json.load(open(os.path.join(ROOT, "tests", "golden", "lti.json")))["configs"]
    g = lti["wave_benchmark.cfg"]
    nd, nt, B = g["n_sensors"], g["n_steps"], g["budget"]
    variants = ((dict(), dict(algorithm="left"), dict(full_square=True)) if which == "lti"
                else (dict(algorithm="left", storage=2),))
    bad = 0
    for kw in variants:
        cid = [d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(cid, src=0)
        with d.Engine(nd, nt, B, device=local, world_size=world, rank=rank, nccl_id=cid[0], **kw) as eng:
            if which == "lti":
                eng.assemble_lti(os.path.join(ROOT, "tests", "golden", "configs", "wave_benchmark.cfg"))
            else:
                from oracle import oracle as O  # checker only: parses the KBF fixture
                k, _, _ = O.read_kbf(os.path.join(ROOT, "tests", "golden", "wave.kbf"))
                kb = k.reshape(nd, nd * nt * nt)
                mine = [j for j in range(nd) if j % world == rank]
                rows_pinned = torch.from_numpy(np.ascontiguousarray(kb[mine])).pin_memory()
                eng.attach_host_rows(rows_pinned)
            eng.run()
            rows = eng.trace()
        ok = [r["chosen_index"] for r in rows] == list(g["chosen"])
        for r, gg in zip(rows, g["gains"]):
            ok = ok and abs(r["gain"] - gg) <= 1e-9 * max(abs(gg), 1.0)
        bad += not ok
    print(f"rank {rank}/{world} {which}: {'OK' if not bad else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)
gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"{which}.json")))
if which == "wave":
    from oracle import oracle as O  # checker only: parses the KBF fixture
    eng = d.Engine(32, 16, 12, device=local, world_size=world, rank=rank, nccl_id=nid[0],
                   export_factor=True)
    eng.load_kbf(os.path.join(ROOT, "tests", "golden", "wave.kbf"))
else:
    nd, nt, rk, b = gold["n_sensors"], gold["n_steps"], gold["rank"], gold["budget"]
    v = d.synthetic_v(nd, nt, rk, gold["seed"])
    eng = d.Engine(nd, nt, b, device=local, world_size=world, rank=rank, nccl_id=nid[0],
                   export_factor=True)
    eng.gen_synthetic(v, rk, gold["sigma"])
eng.run()
rows = eng.trace()
L = eng.export_factor(len(rows))
eng.close()


def single_gpu_rows():
    """The same selection on one GPU (world_size 1): the reference asserts
    worker-count invariance (test_parallel.cpp:109-124, acceptance.cpp:219-252);
    here every gain must be BIT-identical across GPU counts."""
    if which == "wave":
        e1 = d.Engine(32, 16, 12, device=local)
        e1.load_kbf(os.path.join(ROOT, "tests", "golden", "wave.kbf"))
    else:
        e1 = d.Engine(nd, nt, b, device=local)
        e1.gen_synthetic(v, rk, gold["sigma"])
    with e1:
        e1.run()
        return e1.trace()


invariant = True
if rank == 0:
    one = single_gpu_rows()
    invariant = ([(r["chosen_index"], r["gain"], r["objective"]) for r in one] ==
                 [(r["chosen_index"], r["gain"], r["objective"]) for r in rows])
inv = [invariant]
dist.broadcast_object_list(inv, src=0)
invariant = inv[0]
chosen = [r["chosen_index"] for r in rows]
ok = chosen == gold["chosen"]
for r, g in zip(rows, gold["gains"]):
    ok = ok and abs(r["gain"] - g) <= 1e-9 * max(abs(g), 1.0)
# bitwise agreement across ranks
mine = torch.tensor([r["gain"] for r in rows], dtype=torch.float64)
allg = [torch.zeros_like(mine) for _ in range(world)]
dist.all_gather(allg, mine)
same = all(torch.equal(allg[0], x) for x in allg)
fsum = torch.tensor([float(np.abs(L).sum())], dtype=torch.float64)
allf = [torch.zeros_like(fsum) for _ in range(world)]
dist.all_gather(allf, fsum)
same = same and all(torch.equal(allf[0], x) for x in allf)
print(f"rank {rank}/{world} {which}: sequence {'OK' if ok else 'MISMATCH'} ranks-agree {same} "
      f"gains bit-identical to 1 GPU {invariant} "
      f"bytes_exchanged(r1)={rows[0]['bytes_exchanged']}", flush=True)
dist.destroy_process_group()
sys.exit(0 if (ok and same and invariant) else 1)
