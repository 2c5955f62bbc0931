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
    out = os.environ.get("GOLDEN_OUT", HERE)  # e.g. gpurun_out/ when generated on a GPU box's host
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, name), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name)


def trace_dict(t):
    return {"chosen": t.chosen, "gains": t.gains, "objectives": t.objectives,
            "n_evaluated": t.n_evaluated, "n_infeasible": t.n_infeasible}


def synthetic_case(name, nd, nt, rank, sigma, seed, budget, workers=8, replay=False,
                   fast_k=False):
    """fast_k: materialize K with the oracle's blocked generator
    (orc_synthetic_block_rows_fast, bit-identical to SyntheticKAccess::read_block:
    the C1 and C2 KBF sha256s of SURVEY App. A are reproduced by it, see
    `check_fast_k`) instead of the reference's block-by-block read_block, which
    takes hours at C3 size. The selection itself is always the reference's."""
    t0 = time.time()
    if fast_k:
        k = O.synthetic_k_fast(nd, nt, rank, sigma, seed)
    else:
        k = O.ref_synthetic_k(nd, nt, rank, sigma, seed, threads=os.cpu_count())
    tk = time.time() - t0
    t0 = time.time()
    tr = O.ref_parallel_greedy(k, nd, nt, budget, workers=workers, seed=0)
    ts = time.time() - t0
    path = f"/tmp/{name}.kbf"
    O.ref_write_kbf(k, nd, nt, path)
    print(f"{name}: K {tk:.1f} s, selection {ts:.1f} s", flush=True)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    os.remove(path)
    src = ("reference run_parallel_greedy<double> (oracle/_ref) on "
           f"SyntheticKAccess({nd},{nt},{rank},{sigma},{seed}) materialized")
    if fast_k:
        src += " (K bytes by oracle synthetic_k_fast, sha256-pinned to read_block on C1/C2)"
    out = {"source": src,
           "n_sensors": nd, "n_steps": nt, "rank": rank, "sigma": sigma, "seed": seed,
           "budget": budget, "workers": workers, "kbf_sha256": sha,
           "k_seconds": tk, "select_seconds": ts, **trace_dict(tr)}
    if replay:
        ga = O.ref_replay(k, nd, nt, tr.chosen)
        out["replay_gains"] = [[None if x != x else x for x in row] for row in ga.tolist()]
    # top-2 gaps from the replay of the reference's own sequence
    dump(f"{name}.json", out)


def check_fast_k():
    """The blocked generator reproduces the reference KBF bytes."""
    import tempfile
    for (nd, nt, rank, sha) in [
            (64, 32, 2048, "aca0214febd0420f4aa0c29dbcf9bf8a4196373874c218a05a7a47e287b2890f"),
            (200, 128, 8192, "f8409a2dfcd401b0aba6b2fddda010fe33a5718a8e846e0c82f1d21a8b587b85")]:
        t0 = time.time()
        k = O.synthetic_k_fast(nd, nt, rank, 1.0, 2024)
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "k.kbf")
            O.ref_write_kbf(k, nd, nt, path)
            got = hashlib.sha256(open(path, "rb").read()).hexdigest()
        print(f"fast K {nd}x{nt} rank {rank}: {time.time() - t0:.1f} s, sha256 "
              f"{'OK' if got == sha else 'MISMATCH ' + got}")
        assert got == sha


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


def edge_cases():
    """Exactly representable constructions pinning the tie rule and the
    infeasibility semantics on the reference itself (selector.hpp:132-134,
    :209-214; parallel.hpp:416-421). All arithmetic on these K is exact (powers
    of two, perfect-square pivots), so every implementation must agree bit for
    bit on which candidates are infeasible and which tie wins."""
    import numpy as np

    def dense_to_raw(a, nd, nt):
        return np.ascontiguousarray(a.reshape(nd, nt, nd, nt).transpose(0, 2, 1, 3)).reshape(-1)

    cases = []
    # lowrank: sigma = 0, K = V V^T with rank 6 < B*Nt = 12; sensors j and j+3
    # span the same two basis directions (scaled by 2): round 1 is a 6-way exact
    # tie, each pick makes its twin exactly singular, round 4 has no feasible
    # candidate -> partial selection + warning
    nd, nt, r = 6, 2, 6
    v = np.zeros((nd * nt, r))
    for j in range(nd):
        v[j * nt, (2 * j) % r] = 2.0
        v[j * nt + 1, (2 * j + 1) % r] = 2.0
    cases.append(("lowrank", nd, nt, v @ v.T, 6))
    # neartie: independent sensors; 1 beats 0 by a relative 2^-40 in the
    # determinant (near-tie flagged, the larger still wins); 2 and 5 are exact
    # twins (exact tie -> the lower index first)
    nd, nt = 6, 2
    a = np.zeros((nd * nt, nd * nt))
    diag = {0: (4.0, 1.0), 1: (4.0 * (1 + 2.0 ** -40), 1.0), 2: (2.0, 1.0), 3: (1.0, 1.0),
            4: (1.5, 1.0), 5: (2.0, 1.0)}
    for j, (x, y) in diag.items():
        a[j * nt, j * nt], a[j * nt + 1, j * nt + 1] = x, y
    cases.append(("neartie", nd, nt, a, 5))
    # npd: sensor 2's diagonal block has an exact zero pivot (infeasible from
    # round 1, counted in n_infeasible every round); sensor 1 becomes exactly
    # singular once 0 is chosen (K_11 = K_10 K_00^-1 K_01); round 4 has no
    # feasible candidate -> partial selection + warning
    nd, nt = 5, 2
    a = np.zeros((nd * nt, nd * nt))
    a[0:2, 0:2] = 4.0 * np.eye(2)
    a[2:4, 2:4] = 1.0 * np.eye(2)
    a[0:2, 2:4] = a[2:4, 0:2] = 2.0 * np.eye(2)
    a[4:6, 4:6] = np.diag([4.0, 0.0])
    a[6:8, 6:8] = 2.0 * np.eye(2)
    a[8:10, 8:10] = 3.0 * np.eye(2)
    cases.append(("npd", nd, nt, a, 5))
    out = []
    for name, nd, nt, a, budget in cases:
        assert np.array_equal(a, a.T)
        k = dense_to_raw(a, nd, nt)
        runs = {}
        for workers in (1, 4):
            tr = O.ref_parallel_greedy(k, nd, nt, budget, workers=workers, seed=7)
            runs[workers] = {**trace_dict(tr), "warning": tr.warning}
        assert runs[1] == runs[4]
        out.append({"name": name, "n_sensors": nd, "n_steps": nt, "budget": budget,
                    "k_raw": k.tolist(), **runs[1]})
        print(name, runs[1])
    dump("edge.json", {"source": "reference run_parallel_greedy<double> (oracle/_ref) at 1 and "
                                 "4 workers on exactly representable K (make_golden.py edge_cases)",
                       "cases": out})


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
    if "edge" in which:
        edge_cases()
    if "checkfast" in which:
        check_fast_k()
    if "c3" in which:  # BASELINE configs[2] at G=1: 75 x 420, select 50
        synthetic_case("c3", 75, 420, 24576, 1.0, 2024, 50, workers=os.cpu_count(), fast_k=True)
    if "c4s" in which:  # C4 scaled down (600 candidates, Nt 64), select 100
        synthetic_case("c4s", 600, 64, 8192, 1.0, 2024, 100, workers=os.cpu_count(), fast_k=True)
    # the reference is slow at this size (c4s with B = 100 did not finish in an
    # hour on 16 cores): the first 40 rounds of the same selection, exactly the
    # prefix of the full run (the greedy is deterministic)
    if "c4s_b40" in which:
        synthetic_case("c4s_b40", 600, 64, 8192, 1.0, 2024, 40, workers=os.cpu_count(), fast_k=True)
    if "c2" in which:
        synthetic_case("c2", 200, 128, 8192, 1.0, 2024, 50, workers=os.cpu_count())
