"""Out-of-HBM selection on one GPU (north star (1), BASELINE configs[4] scaled
to what one box holds): a C5-shaped K larger than the GPU's HBM streams from
pinned host memory.

    python tools/oohbm_run.py [--nd 420 --nt 420 --budget 175 --vrank 81920]

K = sigma^2 I + V V^T (device Philox V, rank 81,920 >= B*Nt) is formed on the
device chunk by chunk straight into the engine's packed host store (the
block-lower half: 124.7 GB pinned for 420 x 420; the full K is 249 GB, above the
192 GB HBM and the 196 GB host RAM of these boxes). The left-looking algorithm
then keeps only W (n x B*Nt, 104 GB) on the device and copies the chosen column's
blocks H2D each round under the column GEMM. The same K is then formed in HBM
by the right-looking engine on the packed block-lower panel store (125 GB) and
the two selections are compared. Prints one JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08812_b200 as d  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nd", type=int, default=420)
ap.add_argument("--nt", type=int, default=420)
ap.add_argument("--budget", type=int, default=175)
ap.add_argument("--vrank", type=int, default=81920)
ap.add_argument("--sigma", type=float, default=1.0)
ap.add_argument("--seed", type=int, default=2024)
ap.add_argument("--no-check", action="store_true", help="skip the resident right-looking rerun")
args = ap.parse_args()
nd, nt, b = args.nd, args.nt, args.budget
n = nd * nt
out = {"workload": f"{nd} candidates x Nt={nt} (n={n}) select {b}, device Philox V rank "
                   f"{args.vrank}, sigma {args.sigma}, seed {args.seed}",
       "k_bytes_full": n * n * 8}

t0 = time.time()
eng = d.Engine(nd, nt, b, algorithm="left", storage="stream", export_factor=False)
plan = eng.plan()
t_create = time.time() - t0
t0 = time.time()
eng.gen_synthetic_device(args.vrank, args.sigma, args.seed)
t_gen = time.time() - t0
plan = eng.plan()
eng.run()
st = eng.stats()
rows = eng.trace()
stream = {"time_to_k_s": round(st["time_to_k_ms"] / 1e3, 3),
          "column_gemm_tflops": round(st["update_flops"] / max(st["update_ms"], 1e-9) / 1e9, 2),
          "h2d_bytes": st["h2d_bytes"], "io_ms": round(st["io_ms"], 1),
          "io_exposed_ms": round(st["io_exposed_ms"], 1),
          "io_hidden": round(1.0 - st["io_exposed_ms"] / st["io_ms"], 4) if st["io_ms"] > 0 else None,
          "pcie_gbs": round(st["h2d_bytes"] / (st["io_ms"] / 1e3) / 1e9, 1) if st["io_ms"] > 0 else None,
          "device_bytes": plan["device_bytes"], "host_store_bytes": plan["host_store_bytes"],
          "engine_create_s": round(t_create, 1), "k_formation_s": round(t_gen, 1),
          "chosen_first": [r["chosen_index"] for r in rows[:10]],
          "objective": rows[-1]["objective"], "n_selected": len(rows)}
seq_stream = [(r["chosen_index"], r["gain"]) for r in rows]
eng.close()
out["streamed_left_looking"] = stream

if not args.no_check:
    t0 = time.time()
    with d.Engine(nd, nt, b, algorithm="right", storage="hbm") as rl:
        rl.gen_synthetic_device(args.vrank, args.sigma, args.seed)
        t_gen = time.time() - t0
        p = rl.plan()
        rl.run()
        st = rl.stats()
        rows = rl.trace()
    seq_rl = [(r["chosen_index"], r["gain"]) for r in rows]
    gmax = max(abs(a[1] - c[1]) / max(abs(c[1]), 1.0) for a, c in zip(seq_stream, seq_rl))
    out["resident_right_looking"] = {
        "time_to_k_s": round(st["time_to_k_ms"] / 1e3, 3),
        "update_tflops": round(st["update_flops"] / max(st["update_ms"], 1e-9) / 1e9, 2),
        "device_bytes": p["device_bytes"], "packed": p["packed"], "k_formation_s": round(t_gen, 1),
        "same_sequence": [s for s, _ in seq_stream] == [s for s, _ in seq_rl],
        "max_rel_gain_diff": gmax}
print(json.dumps(out), flush=True)
