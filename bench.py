#!/usr/bin/env python
"""bench.py -- time-to-k-sensors of greedy D-optimal selection on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0. A "step" is one full greedy selection (B rounds of
gains -> argmax -> panel -> rank-Nt Schur update) over the synthetic K of the
workload, with K resident in HBM when the timed region starts (C is restored
from the pristine device copy between steps, outside the timed region).

Workload (BASELINE.json configs[1], the metric's single-GPU config):
  C2: SyntheticKAccess(200 sensors, Nt=128, rank 8192, sigma=1, seed 2024),
  budget 50, n = 25,600, K = 5.24 GB FP64. At N > 1 the same problem is
  block-column sharded over N GPUs (strong scaling, NCCL argmax allgather +
  panel broadcast). `--config c3` selects the weak-scaling workload
  (75*N sensors x Nt=420, rank 24,576, budget 50).

`--gpus N` without a launcher re-executes itself under torch.distributed.run
(one process per GPU, 127.0.0.1), so `python bench.py --gpus 4` measures 4 GPUs.

`--impl reference` times the reference CPU implementation (oracle/_ref, the
unmodified reference headers compiled from /root/reference): one complete
run_parallel_greedy selection on all host cores, on K materialized by the
oracle's bit-exact generator -- nothing of this package is imported on that
arm (see reference_arm()).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(nd=64, nt=32, rank=2048, budget=16),
    "c2": dict(nd=200, nt=128, rank=8192, budget=50),
    "c3": dict(nd=75, nt=420, rank=24576, budget=50),  # nd scaled by N
    # BASELINE configs[3]: K = 508 GB, formed on the devices (device Philox V,
    # rank 81,920 -- V alone is 165 GB, never on a host); needs >= 2 GPUs
    "c4": dict(nd=600, nt=420, rank=81920, budget=175),
}
SIGMA, SEED = 1.0, 2024
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# Fallback FP64 denominators (profiles/r01_fp64_peak_probe.log) -- every run
# measures both again on its own devices (measure_fp64_peaks) and reports those.
FP64_DMMA_PEAK_TFLOPS = 37.10
FP64_CUBLAS_TFLOPS = 36.13


ALGO_DESC = {
    "right": "right-looking Schur update of the resident conditional covariance "
             "(north star; block-lower symmetric storage)",
    "left": "left-looking W-resident variant (SURVEY 8f row 1): K pristine, "
            "c = K[:,k] - W W_k^T per round",
}
FLOP_MODEL = {
    "right": "block-lower right-looking: sum_t 2*Nt^3*sum_{local live blocks h}(R_t - g_h) "
             "(= Nt*n_t*(n_t+Nt) over all ranks)",
    "left": "left-looking: sum_t [2*n_loc,t*Nt*(t*Nt) + n_loc,t*Nt^2 + 2*R_loc,t*Nt^3]",
}


def workload(name: str, n_gpus: int) -> dict:
    w = dict(CONFIGS[name])
    if name == "c3":
        w["nd"] = 75 * n_gpus
    return w


# ------------------------------------------------------------------------- #
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits", "-lms", "200"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        p.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------- #
def respawn_if_needed(args) -> None:
    """`--gpus N` (N > 1) without a launcher: re-exec under torch.distributed.run,
    one rank per GPU over 127.0.0.1 (the driver's own launch line)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def measure_fp64_peaks(d, device: int) -> dict:
    """Roofline denominators measured in this run on this device: the DMMA
    issue rate (dsel_measure_fp64_peak) and cuBLAS DGEMM 8192^3 (torch)."""
    import torch

    dmma = max(d.measure_fp64_peak(device) for _ in range(3))
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=f"cuda:{device}")
    b = torch.randn(n, n, dtype=torch.float64, device=f"cuda:{device}")
    best = 1e9
    for i in range(4):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        if i:
            best = min(best, e0.elapsed_time(e1))
    del a, b, c
    torch.cuda.empty_cache()
    return {"dmma_tflops": round(dmma, 2), "cublas_dgemm_tflops": round(2 * n ** 3 / best / 1e9, 2)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def allreduce_min(x: float, world: int) -> float:
    return -allreduce_max(-x, world)


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_bytes(b: bytes | None, world: int) -> bytes:
    if world == 1:
        return b
    import torch.distributed as dist

    obj = [b]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def ncu_traffic(profile_dir: str, algorithm: str, config: str, world: int):
    """dram bytes per update-kernel launch from a committed `ncu --set full`
    capture of THIS line's configuration (profiles/*update_dram_<algo>_<config>_n<N>.json),
    else None -- a capture of another shape says nothing about this one."""
    import glob

    pat = f"*update_dram_{algorithm}_{config}_n{world}.json"
    for p in sorted(glob.glob(os.path.join(profile_dir, pat)), reverse=True):
        try:
            return json.load(open(p))
        except Exception:
            pass
    return None


# ------------------------------------------------------------------------- #
def time_device(eng, args, world, clock_dev=None):
    """K steps of a full selection with K resident in HBM (C restored between
    steps, outside the timed region): device time-to-k, max over ranks."""
    times, upd_ms, upd_fl, launches, chosen = [], [], [], [], None
    clk = ClockSampler(clock_dev) if clock_dev is not None else None
    if clk:
        clk.__enter__()
    for it in range(args.warmup + args.steps):
        eng.reset()
        barrier(world)
        eng.run()
        st = eng.stats()
        t = allreduce_max(st["time_to_k_ms"] / 1e3, world)
        if it >= args.warmup:
            times.append(t)
            upd_ms.append(st["update_ms"])
            upd_fl.append(st["update_flops"])
            launches.append(st["kernel_launches"])
        rows = eng.trace()
        chosen = [r["chosen_index"] for r in rows]
    if clk:
        clk.__exit__()
    gaps = [((r["gain"] - r["runner_up_gain"]) / max(abs(r["gain"]), 1.0), r["k"]) for r in rows
            if r["runner_up"] >= 0]
    near = {"tau": 1e-9, "flagged_rounds": [r["k"] for r in rows if r["near_tie"]],
            "min_rel_top2_gap": min(gaps)[0] if gaps else None,
            "at_round": min(gaps)[1] if gaps else None}
    out = {"value": sum(times) / len(times), "chosen": chosen, "near_ties": near,
           "launches": int(sum(launches) / len(launches)),
           "clocks": clk.summary() if clk else None}
    upd_t = sum(upd_ms) / 1e3
    out["upd_tf"] = sum(upd_fl) / upd_t / 1e12 if upd_t > 0 else 0.0
    out["upd_tf_max"] = allreduce_max(out["upd_tf"], world)
    out["flops_rank"] = sum(upd_fl) / len(upd_fl)
    out["flops_all"] = allreduce_sum(out["flops_rank"], world)
    return out


def time_e2e(eng, args, world, host_rows, mine, chosen, attach=None):
    """Same selection through the public API from pinned host memory, wall
    clock, max over ranks. Resident store: H2D of this rank's block rows
    (dsel_load_block_row) + selection + D2H of the result. attach (streaming
    left-looking): dsel_attach_host_rows over the same pinned rows, then the
    engine copies only the blocks each round reads (diagonal once, the chosen
    column's own blocks per round) -- inside the timed region."""
    import numpy as np

    e2e_times, h2d, d2h = [], 0, 0
    for it in range(max(1, args.warmup // 2) + args.steps):
        eng.reset()
        barrier(world)
        t0 = time.perf_counter()
        if attach is not None:
            eng.attach_host_rows(attach)
        else:
            for idx, j in enumerate(mine):
                eng.load_block_row(j, host_rows[idx])
        eng.run()
        rows = eng.trace()            # D2H of the selection result
        res = np.array([[r["chosen_index"], r["gain"]] for r in rows])
        t1 = time.perf_counter() - t0
        st = eng.stats()
        if it >= max(1, args.warmup // 2):
            e2e_times.append(allreduce_max(t1, world))
            h2d = st["h2d_bytes"]
            d2h = st["d2h_bytes"] + res.size * 8
        assert [int(x) for x in res[:, 0]] == chosen
    return {"value": sum(e2e_times) / len(e2e_times), "unit": "s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


def c4_arm(args, world, rank, local):
    """C4 (600 x Nt=420, select 175): the packed block-lower panels hold K in HBM
    from 2 GPUs (127 GB/GPU at 2). K is formed on the devices before every step
    (outside the timed region; there is no room for a pristine copy), so a step
    costs ~1-2 min of setup: use --steps 1 --warmup 0 by hand. No e2e (the host
    cannot hold K) and no CPU baseline (hours of reference work per round)."""
    import paper_2604_08812_b200 as d

    w = workload("c4", world)
    nd, nt, vrank, budget = w["nd"], w["nt"], w["rank"], w["budget"]
    peaks = measure_fp64_peaks(d, local)
    peaks_min = {k: allreduce_min(x, world) for k, x in peaks.items()}
    nid = broadcast_bytes(d.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
    eng = d.Engine(nd, nt, budget, device=local, world_size=world, rank=rank, nccl_id=nid,
                   storage="hbm")
    times, upd, fl, t_gen, launches = [], [], [], 0.0, 0
    for it in range(args.warmup + args.steps):
        barrier(world)
        t0 = time.time()
        eng.gen_synthetic_device(vrank, SIGMA, SEED)
        t_gen = max(t_gen, allreduce_max(time.time() - t0, world))
        barrier(world)
        eng.run()
        st = eng.stats()
        if it >= args.warmup:
            times.append(allreduce_max(st["time_to_k_ms"] / 1e3, world))
            upd.append(st["update_ms"])
            fl.append(st["update_flops"])
            launches = st["kernel_launches"]
    rows = eng.trace()
    dev_gb = eng.device_bytes / 1e9
    eng.close()
    value = sum(times) / len(times)
    upd_tf = sum(fl) / (sum(upd) / 1e3) / 1e12
    line = {"metric": "time-to-k-sensors (s)", "value": round(value, 3), "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value * 1e3, 1),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: K = sigma^2 I + V V^T with V from the device Philox stream "
                    "(rank 81,920; not the reference RNG stream -- V is 165 GB)",
            "config": {**workload_config("c4", nd, nt, budget, vrank, world),
                       "chosen_first": [r["chosen_index"] for r in rows[:8]],
                       "objective": rows[-1]["objective"], "device_gb_per_gpu": round(dev_gb, 1),
                       "k_formation_s": round(t_gen, 1)},
            "roofline": {"bound": "tensor", "kernel": "schur_update_ws_kernel (DMMA.8x8x4, TMA bulk)",
                         "achieved": round(upd_tf, 3), "peak": peaks_min["dmma_tflops"],
                         "unit": "TFLOP/s", "frac": round(upd_tf / peaks_min["dmma_tflops"], 4),
                         "peak_cublas_dgemm": peaks_min["cublas_dgemm_tflops"], "traffic": None},
            "e2e": None, "e2e_note": "K (508 GB) does not fit any host here",
            "gpu_launches": int(launches)}
    if rank == 0:
        emit(line)


def our_arm(args, world, rank, local):
    import paper_2604_08812_b200 as d

    if args.config == "c4":
        c4_arm(args, world, rank, local)
        return
    w = workload(args.config, world)
    nd, nt, vrank, budget = w["nd"], w["nt"], w["rank"], w["budget"]
    t0 = time.time()
    v = d.synthetic_v(nd, nt, vrank, SEED, threads=max(1, (os.cpu_count() or 1) // world))
    t_v = time.time() - t0
    peaks = measure_fp64_peaks(d, local)
    peaks_min = {k: allreduce_min(x, world) for k, x in peaks.items()}
    algos = [args.algorithm] + ([] if args.no_variants else
                                ["left" if args.algorithm == "right" else "right"])
    want_cpu = rank == 0 and world == 1 and not args.no_cpu
    mine = [j for j in range(nd) if j % world == rank]
    host, host_rows, hv = None, None, None
    if not args.no_e2e or want_cpu:
        # this rank's block rows of K in pinned host memory: the e2e input. A
        # full-panel engine forms K once and exports them (the packed store
        # keeps only the block-lower half)
        import torch

        row_elems = nd * nt * nt
        host = torch.empty(len(mine) * row_elems, dtype=torch.float64).pin_memory()
        hv = host.numpy()
        nid = broadcast_bytes(d.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
        with d.Engine(nd, nt, budget, device=local, world_size=world, rank=rank, nccl_id=nid,
                      packed=False, storage="hbm") as src:
            src.gen_synthetic(v, vrank, SIGMA)
            for idx, j in enumerate(mine):
                hv[idx * row_elems:(idx + 1) * row_elems] = src.read_block_row(j)
        host_rows = [host[idx * row_elems:(idx + 1) * row_elems] for idx in range(len(mine))]
    engines, t_gen = {}, 0.0
    # the right-looking update under the look-ahead schedule (default when Nt is a
    # multiple of the tile) and, beside it, the plain schedule: the same kernel on
    # every SM, which is where the roofline of the update kernel is read
    la_ok = nt % 128 == 0 and os.environ.get("DSEL_LOOKAHEAD", "1") != "0"
    builds = list(algos) + (["plain"] if la_ok and "right" in algos else [])
    for a in builds:  # every engine gets the same bit-exact K, then V is released
        nid = broadcast_bytes(d.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
        prev_la = os.environ.get("DSEL_LOOKAHEAD")
        os.environ["DSEL_LOOKAHEAD"] = "0" if a == "plain" else (prev_la or "1")
        engines[a] = d.Engine(nd, nt, budget, device=local, world_size=world, rank=rank,
                              nccl_id=nid, keep_pristine=True, export_factor=True,
                              algorithm="right" if a == "plain" else a)
        if prev_la is None:
            del os.environ["DSEL_LOOKAHEAD"]
        else:
            os.environ["DSEL_LOOKAHEAD"] = prev_la
        t0 = time.time()
        engines[a].gen_synthetic(v, vrank, SIGMA)
        t_gen = max(t_gen, time.time() - t0)
    del v
    res = {a: time_device(engines[a], args, world, local if a == args.algorithm else None)
           for a in builds}
    if "plain" in res:
        if res["plain"]["chosen"] != res["right"]["chosen"]:
            raise RuntimeError("look-ahead and plain schedules give different sequences")
        engines.pop("plain").close()
    if len(algos) > 1 and res[algos[0]]["chosen"] != res[algos[1]]["chosen"]:
        raise RuntimeError("right- and left-looking sequences differ")
    for a in algos:
        if args.no_e2e:
            res[a]["e2e"] = None
        elif a == "left":
            engines[a].close()
            # K stays in host memory; the streaming engine reads what each round needs
            nid = broadcast_bytes(d.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
            with d.Engine(nd, nt, budget, device=local, world_size=world, rank=rank, nccl_id=nid,
                          export_factor=True, algorithm="left", storage=2) as es:
                res[a]["e2e"] = time_e2e(es, args, world, host_rows, mine, res[a]["chosen"],
                                         attach=host)
                res[a]["e2e"]["path"] = ("dsel_attach_host_rows(pinned own block rows) + dsel_run "
                                         "(streaming store: diagonal blocks once + the chosen "
                                         "column's own blocks per round, copy stream overlapped "
                                         "with the column GEMM) + trace D2H")
        else:
            res[a]["e2e"] = time_e2e(engines[a], args, world, host_rows, mine, res[a]["chosen"])
            res[a]["e2e"]["path"] = ("dsel_load_block_row x own rows (pinned; H2D of the "
                                     "block-lower half) + dsel_run + trace D2H")
        engines[a].close()
    prim = res[algos[0]]
    other = res[algos[1]] if len(algos) > 1 else None
    value, chosen, clocks = prim["value"], prim["chosen"], prim["clocks"]
    plain = res.get("plain")
    kern = plain if (plain is not None and args.algorithm == "right") else prim
    upd_tf, upd_tf_all = kern["upd_tf"], kern["upd_tf_max"]
    tot_flops, tot_flops_all = prim["flops_rank"], prim["flops_all"]
    e2e_tf = tot_flops_all / value / 1e12
    e2e, launches = prim["e2e"], [prim["launches"]]
    cpu = None
    if want_cpu:
        cpu = cpu_reference(hv, nd, nt, budget, chosen)

    tr = ncu_traffic(os.path.join(ROOT, "profiles"), args.algorithm, args.config, world)
    if tr and "dynamic_schedule" in tr and os.environ.get("DSEL_WS_DYNAMIC", "1") != "0":
        tr = dict(tr, **tr["dynamic_schedule"])  # the capture of the schedule this run uses
    traffic = tr.get("traffic_bytes_per_launch") if tr else None
    peak = peaks_min["dmma_tflops"]
    line = {
        "metric": "time-to-k-sensors (s)",
        "value": round(value, 6),
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(value * 1e3, 3),
        "higher_is_better": False,
        "scaling": "weak" if args.config == "c3" else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: SyntheticKAccess K = sigma^2 I + V V^T (reference RNG stream, "
                "bit-exact device generator)",
        "config": {**workload_config(args.config, nd, nt, budget, vrank, world),
                   "chosen_first": chosen[:8]},
        "algorithm": ALGO_DESC[args.algorithm],
        "schedule": ({"primary": "look-ahead rounds (the bulk of round t beside round t+1's gains, "
                                 "argmax and W solve; %s SMs reserved for that chain)"
                                 % os.environ.get("DSEL_LA_RESERVE", "12" if world <= 2 else "16"),
                      "plain_schedule_value": round(plain["value"], 6),
                      "roofline_from": "the plain schedule (the same update kernel on all 148 SMs; "
                                       "under look-ahead it shares the GPU with the chain)",
                      "lookahead_update_tflops_per_gpu": round(prim["upd_tf"], 3)}
                     if plain is not None and args.algorithm == "right" else
                     {"primary": "plain rounds"}),
        "schur_update": {"flops_per_step_per_rank": tot_flops,
                         "flops_per_step_all_ranks": tot_flops_all,
                         "kernel_tflops_per_gpu": round(upd_tf, 3),
                         "kernel_tflops_per_gpu_max_rank": round(upd_tf_all, 3),
                         "end_to_end_tflops_all_gpus": round(e2e_tf, 3),
                         "frac_of_fp64_peak_per_gpu": round(upd_tf / peak, 4),
                         "flop_model": FLOP_MODEL[args.algorithm]},
        "roofline": {"bound": "tensor", "kernel": "schur_update_ws_kernel (DMMA.8x8x4, TMA bulk)",
                     "achieved": round(upd_tf, 3), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(upd_tf / peak, 4),
                     "peak_source": "measured in this run on these GPUs (min over ranks): "
                                    "DMMA.8x8x4 issue-rate microbenchmark "
                                    "(dsel_measure_fp64_peak); MEASURED_PEAKS.json has no FP64 "
                                    "entry",
                     "peak_cublas_dgemm": peaks_min["cublas_dgemm_tflops"],
                     "frac_of_cublas_dgemm": round(upd_tf / peaks_min["cublas_dgemm_tflops"], 4),
                     "traffic": traffic,
                     "traffic_note": (f"dram read+write of one update launch ({tr['launch']}) "
                                      f"from ncu --set full; algorithmic C read+write "
                                      f"{tr['algorithmic_bytes_per_launch']:.4g} B "
                                      f"(x{tr['traffic_over_algorithmic']})") if tr else
                                     "no ncu --set full capture of this configuration committed"},
        "e2e": e2e,
        "near_ties": prim["near_ties"],
        "gpu_launches": int(sum(launches) / len(launches)) if launches else 0,
        "clocks": clocks,
        "setup": {"v_host_s": round(t_v, 2), "k_gen_device_s": round(t_gen, 2)},
    }
    if other is not None:
        alt = "left" if args.algorithm == "right" else "right"
        line["variant"] = {
            "algorithm": ALGO_DESC[alt], "value": round(other["value"], 6), "unit": "s",
            "e2e": other["e2e"], "same_sequence": True,
            "update_tflops_per_gpu": round(other["upd_tf"], 3),
            "frac_of_fp64_peak_per_gpu": round(other["upd_tf"] / peak, 4),
            "flops_per_step_all_ranks": other["flops_all"], "flop_model": FLOP_MODEL[alt],
            "gpu_launches": other["launches"]}
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        emit(line)


# ------------------------------------------------------------------------- #
def alg1_round_cost(nd, nt, k):
    """Reference per-round cost model (Alg. 1 flops):
    (Nd-k) candidates x [(k Nt)^2 Nt (trsm) + 2 k Nt^3 (Schur) + Nt^3/3 (chol)]."""
    return (nd - k) * ((k * nt) ** 2 * nt + 2 * k * nt ** 3 + nt ** 3 / 3)


def cpu_reference(k_host, nd, nt, budget, prefix, iterates=None):
    """Reference CPU path (oracle/_ref: unmodified reference headers) on a
    BOUNDED sample: one full evaluation round (detail::timed_round, all host
    threads, pipelined) at a few iterates along the selected prefix, then
    time-to-k extrapolated with the Alg. 1 cost model fitted to the samples
    (T(k) = a*cost(k) + b*(Nd-k))."""
    import numpy as np

    from oracle import oracle as O

    cores = os.cpu_count() or 1
    if iterates is None:
        iterates = [1, budget // 4, budget // 2] if budget >= 8 else list(range(1, budget))
    ms, setup = O.ref_timed_rounds(np.ascontiguousarray(k_host), nd, nt, prefix, iterates, cores)
    A = np.array([[alg1_round_cost(nd, nt, k), nd - k] for k in iterates], dtype=np.float64)
    coef, *_ = np.linalg.lstsq(A, np.asarray(ms) / 1e3, rcond=None)
    a, b = max(coef[0], 0.0), max(coef[1], 0.0)
    total = sum(a * alg1_round_cost(nd, nt, k) + b * (nd - k) for k in range(budget))
    return {"value": round(total, 3), "unit": "s", "cores": cores, "kind": "reference",
            "sample": f"reference run_parallel_greedy round (detail::timed_round, {cores} "
                      f"workers) timed at iterates {list(iterates)} = "
                      f"{[round(float(x), 1) for x in ms]} ms; "
                      f"time-to-{budget} EXTRAPOLATED with the Alg.1 cost model "
                      f"(a={a:.3e} s/flop, b={b:.3e} s/cand)",
            "sampled_rounds_ms": list(map(float, ms)), "setup_ms": list(map(float, setup))}


def reference_arm(args, world, rank, local):
    """The reference's own CPU implementation on this box's host cores: the
    unmodified reference headers (oracle/_ref) run_parallel_greedy<double> --
    the `doptsel select --mode schur` path (parallel.hpp:281-483) -- with one
    worker per host thread, on K materialized by the oracle's bit-exact
    blocked generator (sha256-identical to SyntheticKAccess on C1/C2,
    tests/test_oracle.py). Nothing of this package is imported here.

    C1/C2: ONE complete selection is timed (time-to-B, measured). C3: a full
    reference run takes hours, so the first rounds are timed and time-to-B is
    extrapolated with the Alg. 1 cost model (labelled)."""
    if rank != 0:
        return  # one CPU measurement per job; the other ranks exit 0
    import numpy as np

    from oracle import oracle as O

    if not O.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref not built "
                                                  "(needs /root/reference at build time)"})
        return
    w = workload(args.config, world)
    nd, nt, vrank, budget = w["nd"], w["nt"], w["rank"], w["budget"]
    cores = os.cpu_count() or 1
    if args.config == "c4":
        emit({"impl": "reference", "unavailable": "C4's K is 508 GB: the reference keeps it in host "
                                                  "memory, which no host here has"})
        return
    t0 = time.time()
    k = O.synthetic_k_fast(nd, nt, vrank, SIGMA, SEED, threads=cores)
    t_k = time.time() - t0
    full = args.config in ("c1", "c2")
    if full:
        tr = O.ref_parallel_greedy(k, nd, nt, budget, workers=cores, seed=0)
        value = tr.selection_ms / 1e3
        chosen = tr.chosen
        sample = (f"one complete reference run_parallel_greedy<double> selection, time-to-"
                  f"{budget} MEASURED ({cores} workers = host threads, pipelined reader "
                  f"threads, K in memory as a DataSpaceHessian)")
        kind_note = "measured"
        rounds_ms = [round(x, 2) for x in tr.wall_ms]
    else:
        r_s = min(budget, 6)
        tr = O.ref_parallel_greedy(k, nd, nt, r_s, workers=cores, seed=0)
        ms = np.asarray(tr.wall_ms)
        its = np.arange(len(ms))
        A = np.array([[alg1_round_cost(nd, nt, i), nd - i] for i in its], dtype=np.float64)
        coef, *_ = np.linalg.lstsq(A, ms / 1e3, rcond=None)
        a_, b_ = max(coef[0], 0.0), max(coef[1], 0.0)
        value = sum(a_ * alg1_round_cost(nd, nt, i) + b_ * (nd - i) for i in range(budget))
        chosen = tr.chosen
        sample = (f"reference run_parallel_greedy<double> first {r_s} rounds timed "
                  f"({[round(float(x), 1) for x in ms]} ms, {cores} workers); time-to-{budget} "
                  f"EXTRAPOLATED with the Alg. 1 cost model (a={a_:.3e} s/flop, b={b_:.3e} s/cand)")
        kind_note = "extrapolated"
        rounds_ms = [round(float(x), 2) for x in ms]
    golden = os.path.join(ROOT, "tests", "golden", f"{args.config}.json")
    match = None
    if os.path.exists(golden):
        want = json.load(open(golden))["chosen"]
        match = want[:len(chosen)] == chosen
    cpu = {"value": round(value, 3), "unit": "s", "cores": cores, "kind": "reference",
           "sample": sample, "time": kind_note, "k_materialize_s": round(t_k, 1),
           "round_ms": rounds_ms}
    line = {"metric": "time-to-k-sensors (s)", "value": round(value, 3), "unit": "s",
            "n_gpus": world, "steps": 1, "warmup": 0,
            "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": round(value * 1e3, 1), "higher_is_better": False,
            "scaling": "weak" if args.config == "c3" else "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: SyntheticKAccess K = sigma^2 I + V V^T (reference RNG stream; "
                    "materialized by the oracle's bit-exact generator)",
            "config": {**workload_config(args.config, nd, nt, budget, vrank, world),
                       "chosen_first": chosen[:8]},
            "impl": "reference", "cpu_baseline": cpu,
            "sequence_matches_reference_golden": match,
            "e2e": {"value": round(value, 3), "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


def workload_config(name, nd, nt, budget, vrank, world) -> dict:
    """The workload keys both arms report (same dict on the reference arm)."""
    return {"workload": f"{name.upper()}: {nd} candidates x Nt={nt} (n={nd * nt}) select "
                        f"{budget}, rank {vrank}, sigma {SIGMA}, seed {SEED}",
            "n_sensors": nd, "n_steps": nt, "budget": budget, "rank": vrank,
            "parallelism": f"candidate-sharded x{world} (cyclic block columns); per round NCCL "
                           "allgather of the 32-B argmax records, W rows exchanged over NVLink "
                           "peer memory (one fused read+scatter kernel) when x>1",
            "l2": f"inputs {nd * nt * nd * nt * 8 / 1e9:.2f} GB >> 126 MB L2 (no flush needed)"}


_STDOUT_FD = None


def emit(line: dict) -> None:
    """The one JSON line, on the real stdout (everything else -- NCCL's
    version banner, library chatter -- was redirected to stderr)."""
    fd = _STDOUT_FD if _STDOUT_FD is not None else 1
    os.write(fd, (json.dumps(line) + "\n").encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--algorithm", default="right", choices=["right", "left"],
                    help="primary line (right = the north-star resident conditional-covariance "
                         "Schur update; the left-looking variant (SURVEY 8f row 1) is reported "
                         "beside it in the same line under 'variant')")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip measuring the other algorithm beside the primary")
    args = ap.parse_args()
    global _STDOUT_FD
    if args.impl != "reference":
        respawn_if_needed(args)  # before stdout is redirected: the children print the line
    sys.stdout.flush()
    _STDOUT_FD = os.dup(1)
    os.dup2(2, 1)  # C-level writes to stdout (NCCL init banner) go to stderr
    if args.impl == "reference":
        # CPU-only: no process group; under a launcher rank 0 alone measures
        reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")),
                      int(os.environ.get("RANK", "0")), 0)
        return
    world, rank, local = dist_init()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    our_arm(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
