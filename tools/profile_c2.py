"""One C2 selection (or a prefix of it) for profiling: per-phase device-time
breakdown from the engine's CUDA events. Used plain and under ncu."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08812_b200 as d  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nd", type=int, default=200)
ap.add_argument("--nt", type=int, default=128)
ap.add_argument("--rank", type=int, default=8192)
ap.add_argument("--budget", type=int, default=50)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--algorithm", default="right")
ap.add_argument("--full-square", action="store_true")
ap.add_argument("--full-panels", action="store_true", help="full-height panels (no packing)")
args = ap.parse_args()
v = d.synthetic_v(args.nd, args.nt, args.rank, 2024)
eng = d.Engine(args.nd, args.nt, args.budget, keep_pristine=True, export_factor=True,
               algorithm=args.algorithm, full_square=args.full_square,
               packed=not args.full_panels)
eng.gen_synthetic(v, args.rank, 1.0)
for r in range(args.runs):
    eng.reset()
    eng.run()
    rows = eng.trace()
    st = eng.stats()
tot = {k: sum(r[k] for r in rows) for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update", "ms_round")}
print(json.dumps({"time_to_k_ms": st["time_to_k_ms"], "update_ms": st["update_ms"],
                  "update_tflops": st["update_flops"] / st["update_ms"] / 1e9,
                  "phase_ms": tot, "launches": st["kernel_launches"],
                  "first_rounds": [{k: round(r[k], 4) for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update")} for r in rows[:3]],
                  "last_rounds": [{k: round(r[k], 4) for k in ("ms_gain", "ms_exchange", "ms_panel", "ms_update")} for r in rows[-3:]],
                  "update_flops_per_round": [r["update_flops"] for r in rows]}, indent=1))
eng.close()
