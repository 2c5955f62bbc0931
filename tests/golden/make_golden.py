"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (oracle/_ref/libdoptsel_ref.so, compiled from /root/reference by
oracle/Makefile). Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py [c1 wave random lti c2]

c2 takes ~20 min on 8 cores (K materialization + 50 rounds).
"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name)


def trace_dict(t):
    return {"chosen": t.chosen, "gains": t.gains, "objectives": t.objectives,
            "n_evaluated": t.n_evaluated, "n_infeasible": t.n_infeasible}


def synthetic_case(name, nd, nt, rank, sigma, seed, budget, workers=8, replay=False):
    t0 = time.time()
    k = O.ref_synthetic_k(nd, nt, rank, sigma, seed, threads=os.cpu_count())
    tk = time.time() - t0
    t0 = time.time()
    tr = O.ref_parallel_greedy(k, nd, nt, budget, workers=workers, seed=0)
    ts = time.time() - t0
    path = f"/tmp/{name}.kbf"
    O.ref_write_kbf(k, nd, nt, path)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    os.remove(path)
    out = {"source": "reference run_parallel_greedy<double> (oracle/_ref) on "
                     f"SyntheticKAccess({nd},{nt},{rank},{sigma},{seed}) materialized",
           "n_sensors": nd, "n_steps": nt, "rank": rank, "sigma": sigma, "seed": seed,
           "budget": budget, "workers": workers, "kbf_sha256": sha,
           "k_seconds": tk, "select_seconds": ts, **trace_dict(tr)}
    if replay:
        ga = O.ref_replay(k, nd, nt, tr.chosen)
        out["replay_gains"] = [[None if x != x else x for x in row] for row in ga.tolist()]
    # top-2 gaps from the replay of the reference's own sequence
    dump(f"{name}.json", out)


def wave():
    path = os.path.join(HERE, "wave.kbf")
    nl = O.ref_wave_kbf(path)
    tr = O.ref_kbf_select(path, 12, workers=1)
    k, nd, nt = O.read_kbf(path)
    ga = O.ref_replay(k, nd, nt, tr.chosen)
    dump("wave.json", {"source": "reference: benchmark_problem(0) -> assemble_k -> write_kbf -> "
                                 "KStoreReader -> run_parallel_greedy (doptsel select)",
                       "n_sensors": nd, "n_steps": nt, "budget": 12,
                       "kbf_sha256": hashlib.sha256(open(path, "rb").read()).hexdigest(),
                       "noise_logdets": nl.tolist(), **trace_dict(tr),
                       "replay_gains": [[None if x != x else x for x in row]
                                        for row in ga.tolist()]})


def lti_configs():
    """Reference `doptsel build` on each tests/golden/configs/*.cfg: KBF sha256,
    noise log-dets and the reference selection on the built store."""
    import tempfile

    out = {}
    for name in sorted(os.listdir(os.path.join(HERE, "configs"))):
        if not name.endswith(".cfg") or name.startswith("bad"):
            continue
        cfg = os.path.join(HERE, "configs", name)
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "k.kbf")
            nd = int([ln.split("=")[1] for ln in open(cfg) if ln.startswith("n_sensors")][0])
            nl = O.ref_build_kbf(cfg, path, nd)
            k, nd, nt = O.read_kbf(path)
            budget = min(12, nd)
            tr = O.ref_kbf_select(path, budget, workers=1)
            out[name] = {"n_sensors": nd, "n_steps": nt, "budget": budget,
                         "kbf_sha256": hashlib.sha256(open(path, "rb").read()).hexdigest(),
                         "noise_logdets": nl.tolist(), **trace_dict(tr)}
    dump("lti.json", {"source": "reference: load_problem_config -> problem_from_config -> "
                                "weights_from_config -> assemble_k -> write_kbf (doptsel build), "
                                "then KStoreReader -> run_parallel_greedy", "configs": out})


def random_cases():
    cases = []
    # shapes follow proj/tests/test_selector.cpp / test_parallel.cpp generators
    for (nd, nt, gamma, rank, seed, budget) in [(10, 2, 0.8, 20, 201, 5), (12, 2, 0.9, 24, 211, 6),
                                                 (9, 3, 1.0, 27, 600, 9), (7, 1, 0.7, 6, 51, 7),
                                                 (16, 5, 0.5, 40, 7, 8), (6, 4, 1.0, 6, 9, 6),
                                                 (20, 8, 1.0, 64, 31, 12)]:
        k = O.ref_random_hessian(nd, nt, gamma, rank, seed)
        tr = O.ref_parallel_greedy(k, nd, nt, budget, workers=2, seed=3)
        ga = O.ref_replay(k, nd, nt, tr.chosen)
        cases.append({"n_sensors": nd, "n_steps": nt, "gamma": gamma, "rank": rank, "seed": seed,
                      "budget": budget, "warning": tr.warning, **trace_dict(tr),
                      "replay_gains": [[None if x != x else (x if x != float("-inf") else "-inf")
                                        for x in row] for row in ga.tolist()]})
    dump("random.json", {"source": "reference random_hessian (tests/support/generators.hpp) + "
                                   "run_parallel_greedy", "cases": cases})


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "wave", "random", "lti"]
    if "c1" in which:
        synthetic_case("c1", 64, 32, 2048, 1.0, 2024, 16, replay=True)
    if "wave" in which:
        wave()
    if "random" in which:
        random_cases()
    if "lti" in which:
        lti_configs()
    if "c3mini" in which:  # Nt = 420 (the CSZ block size) at oracle-friendly scale
        synthetic_case("c3mini", 12, 420, 4096, 1.0, 2024, 6, workers=os.cpu_count(), replay=True)
    if "c2" in which:
        synthetic_case("c2", 200, 128, 8192, 1.0, 2024, 50, workers=os.cpu_count())
