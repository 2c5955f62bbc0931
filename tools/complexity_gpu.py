"""GPU refactorizing baseline and the complexity sweep.

The reference's `--mode naive` (naive_select, selector.hpp:253-348) scores every
candidate by factorizing the whole augmented matrix [[K_SS, K_Ss], [K_sS, K_ss]]
from scratch, O(k^3 Nt^3) per candidate; `doptsel bench complexity`
(complexity_sweep, bench.hpp:74-160) times that against the Schur formulation
(score_from_buffers: Y = L_S^-1 K_Ss, M = K_ss - Y^T Y, chol M; O(k^2 Nt^3)) as
the iterate k grows -- the paper's Fig. 2.

On the GPU, as a baseline beside the engine:
  naive_select_gpu  the refactorizing greedy selection, batched over candidates:
                    every augmented matrix is factored from scratch by this
                    library's batched Cholesky log-det (dsel_batched_logdet --
                    the gain kernel: warp-level pivots, DMMA panel updates);
                    torch only gathers the augmented matrices. Same tie rule;
  sweep             per-candidate time vs k for (1) refactorizing (the same
                    kernel), (2) the reference's left-looking Schur scoring
                    emulated with torch (triangular solve + Cholesky: the
                    reference formulation, not this engine), (3) this engine's
                    right-looking round (libdsel: gains + update of the
                    remaining candidates) per remaining candidate, with log-log
                    slopes over the top decade (fit_loglog_slopes,
                    bench.hpp:180-205). The reference default k_max = 100 at
                    Nt = 32 needs 3232-wide factorizations; the batched kernel
                    stops at 2800, so the GPU sweep caps k at 2800/Nt - 1 (86).

    python tools/complexity_gpu.py --nt 32 --kmax 85 --step 5 [--out complexity.csv]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _dense(k_blocks: np.ndarray, nd: int, nt: int) -> np.ndarray:
    return k_blocks.reshape(nd, nd, nt, nt).transpose(0, 2, 1, 3).reshape(nd * nt, nd * nt)


def _idx(sensors, nt, dev):
    s = torch.as_tensor(list(sensors), dtype=torch.long, device=dev)
    return (s[:, None] * nt + torch.arange(nt, device=dev)[None, :]).reshape(-1)


def naive_select_gpu(k_blocks: np.ndarray, nd: int, nt: int, budget: int, candidates=None,
                     chunk: int = 64, device: str = "cuda"):
    """Refactorizing greedy selection (naive_select, selector.hpp:253-348) on the GPU.
    Returns (chosen, gains, objectives); gains are raw log-det increments."""
    import paper_2604_08812_b200 as dsel

    kd = torch.as_tensor(_dense(k_blocks, nd, nt), dtype=torch.float64, device=device)
    remaining = list(range(nd)) if candidates is None else list(candidates)
    chosen, gains, objs = [], [], []
    logdet_prev = 0.0
    for _ in range(min(budget, len(remaining))):
        best_d, best_s = -math.inf, -1
        for c0 in range(0, len(remaining), chunk):
            cs = remaining[c0:c0 + chunk]
            idx = torch.stack([_idx(chosen + [s], nt, device) for s in cs])   # (b, dim)
            m = kd[idx[:, :, None], idx[:, None, :]]                          # (b, dim, dim)
            lds, status = dsel.batched_logdet(m)   # refactorized from scratch, this library's kernel
            ld = lds - logdet_prev
            ld = torch.where(status < 0, ld, torch.full_like(ld, -math.inf)).cpu().numpy()
            for s, d in zip(cs, ld):   # better_candidate (selector.hpp:132-134)
                if d == -math.inf:
                    continue
                if d > best_d or (d == best_d and s < best_s):
                    best_d, best_s = float(d), s
        if best_s < 0:
            break
        chosen.append(best_s)
        remaining.remove(best_s)
        logdet_prev += best_d
        gains.append(best_d)
        objs.append(logdet_prev)
    return chosen, gains, objs


def _time(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    m = sum(ts) / len(ts)
    sd = math.sqrt(sum((x - m) ** 2 for x in ts) / max(len(ts) - 1, 1))
    return m, sd


def fit_slope(ks, vals, k_max):
    pts = [(math.log(k), math.log(v)) for k, v in zip(ks, vals) if k * 10 >= k_max and v > 0]
    if len(pts) < 2:
        return None
    n = len(pts)
    sx = sum(p[0] for p in pts)
    sy = sum(p[1] for p in pts)
    sxx = sum(p[0] ** 2 for p in pts)
    sxy = sum(p[0] * p[1] for p in pts)
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def sweep(nt=32, k_max=100, step=5, reps=5, seed=2024, batch=32):
    """complexity_sweep (bench.hpp:74-160) on the GPU: SyntheticKAccess(k_max+1,
    nt, rank=nt, sigma=1, seed), chosen = 0..k-1, candidate k."""
    import paper_2604_08812_b200 as d

    k_max = min(k_max, 2800 // nt - 1)  # dsel_batched_logdet handles m <= 2800
    nd = k_max + 1
    v = d.synthetic_v(nd, nt, nt, seed)
    with d.Engine(nd, nt, nd, keep_pristine=True) as eng:
        eng.gen_synthetic(v, nt, 1.0)
        kb = np.concatenate([eng.read_block_row(j) for j in range(nd)])
        kd = torch.as_tensor(_dense(kb, nd, nt), device="cuda")
        rows = []
        for it in range(step, k_max + 1, step):
            dim = (it + 1) * nt
            kdim = it * nt
            m = kd[:dim, :dim].expand(batch, dim, dim).contiguous()

            def naive():
                return d.batched_logdet(m)[0]

            ls = torch.linalg.cholesky(kd[:kdim, :kdim])
            col = kd[:kdim, kdim:dim].expand(batch, kdim, nt).contiguous()
            kss = kd[kdim:dim, kdim:dim].expand(batch, nt, nt).contiguous()

            def schur():   # score_from_buffers: solve, Schur complement, chol, logdet
                y = torch.linalg.solve_triangular(ls, col, upper=False)
                mm = kss - y.transpose(1, 2) @ y
                lf, _ = torch.linalg.cholesky_ex(mm)
                return torch.log(torch.diagonal(lf, dim1=1, dim2=2)).sum(dim=1)

            nm, nsd = _time(naive, reps)
            sm, ssd = _time(schur, reps)
            # this engine at iterate it: forced prefix 0..it-1, then one timed round
            eng.reset()
            for s in range(it):
                eng.step(forced=s)
            eng.step()
            round_ms = eng.trace()[-1]["ms_round"]   # device time of round it+1
            n_rem = nd - it
            rows.append(dict(k=it, naive_ms=nm / batch, schur_ms=sm / batch, naive_std_ms=nsd / batch,
                             schur_std_ms=ssd / batch, engine_round_ms=round_ms,
                             engine_per_candidate_ms=round_ms / n_rem))
    ks = [r["k"] for r in rows]
    slopes = {key: fit_slope(ks, [r[key] for r in rows], k_max)
              for key in ("naive_ms", "schur_ms", "engine_per_candidate_ms")}
    return rows, slopes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nt", type=int, default=32)
    ap.add_argument("--kmax", type=int, default=85)
    ap.add_argument("--step", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32, help="candidates per batched launch")
    ap.add_argument("--out", default=None, help="CSV path (bench.hpp write_complexity_csv columns)")
    args = ap.parse_args()
    rows, slopes = sweep(args.nt, args.kmax, args.step, args.reps, batch=args.batch)
    if args.out:
        with open(args.out, "w") as f:
            f.write("k,naive_ms,schur_ms,naive_std_ms,schur_std_ms,engine_per_candidate_ms\n")
            for r in rows:
                f.write(f"{r['k']},{r['naive_ms']},{r['schur_ms']},{r['naive_std_ms']},"
                        f"{r['schur_std_ms']},{r['engine_per_candidate_ms']}\n")
    print(json.dumps({"nt": args.nt, "k_max": args.kmax, "batch": args.batch,
                      "loglog_slopes_top_decade": slopes, "rows": rows}))


if __name__ == "__main__":
    main()
