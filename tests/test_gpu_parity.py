"""GPU parity tests: the CUDA path (through the C ABI) against the reference.

Bars (BASELINE.json north star): selected index sequences identical to the
reference (near-ties flagged), per-step log-det gains within
|dg| <= 1e-9 * max(|g|, 1) (raw gains can be ~0 or negative).
Golden vectors come from the reference itself (tests/golden/make_golden.py);
the C restatement in oracle/ supplies K and replay vectors for other inputs.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")]

GAIN_TOL = 1e-9


def gain_close(a, b, tol=GAIN_TOL):
    return abs(a - b) <= tol * max(abs(b), 1.0)


@pytest.fixture(scope="module")
def dsel():
    import paper_2604_08812_b200 as d
    return d


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    return oracle


@pytest.fixture(scope="module")
def c1(golden_dir):
    return json.load(open(os.path.join(golden_dir, "c1.json")))


@pytest.fixture(scope="module")
def c1_k(O):
    return O.synthetic_k(64, 32, 2048, 1.0, 2024)


def run_engine(dsel, k, nd, nt, budget, candidates=None, **kw):
    eng = dsel.Engine(nd, nt, budget, candidates=candidates, **kw)
    eng.load_k(np.ascontiguousarray(k))
    n = eng.run()
    rows = eng.trace()
    return eng, rows, n


def assert_trace_matches(rows, chosen, gains, objectives=None):
    got = [r["chosen_index"] for r in rows]
    assert got == list(chosen), f"sequence differs: {got} vs {chosen}"
    for i, r in enumerate(rows):
        assert gain_close(r["gain"], gains[i]), (i, r["gain"], gains[i])
        if objectives is not None:
            assert gain_close(r["objective"], objectives[i]), (i, r["objective"], objectives[i])


def test_synthetic_generator_bit_exact(dsel, O, c1, c1_k):
    """GPU K = sigma^2 I + V V^T (sequential, non-FMA) is bit-identical to
    SyntheticKAccess::read_block (kaccess.hpp:98-116); the KBF bytes hash to
    the golden sha256 of the reference's write_kbf."""
    nd, nt = 64, 32
    v = dsel.synthetic_v(nd, nt, 2048, 2024)
    with dsel.Engine(nd, nt, 16) as eng:
        eng.gen_synthetic(v, 2048, 1.0)
        rows = [eng.read_block_row(j) for j in range(nd)]
    k = np.concatenate(rows)
    assert np.array_equal(k.view(np.uint64), c1_k.view(np.uint64))
    hdr = b"KBF1" + np.array([1, nd, nt, 1, 1, 0, 0], dtype="<u4").tobytes()
    assert hashlib.sha256(hdr + k.astype("<f8").tobytes()).hexdigest() == c1["kbf_sha256"]


def test_c1_sequence_and_gains(dsel, c1, c1_k):
    eng, rows, n = run_engine(dsel, c1_k, 64, 32, 16)
    eng.close()
    assert n == 16
    assert_trace_matches(rows, c1["chosen"], c1["gains"], c1["objectives"])
    for r, ne in zip(rows, c1["n_evaluated"]):
        assert r["n_evaluated"] == ne and r["n_infeasible"] == 0


def test_c1_generated_on_device_matches(dsel, c1):
    """Whole synthetic path on the device (host V -> GPU K -> selection)."""
    v = dsel.synthetic_v(64, 32, 2048, 2024)
    with dsel.Engine(64, 32, 16) as eng:
        eng.gen_synthetic(v, 2048, 1.0)
        eng.run()
        rows = eng.trace()
    assert_trace_matches(rows, c1["chosen"], c1["gains"], c1["objectives"])


def test_c1_full_gain_vectors_replay(dsel, c1, c1_k):
    """Every remaining candidate's gain at every round (replay along the
    reference sequence) -- compares full gain vectors, not just winners."""
    replay = c1["replay_gains"]
    with dsel.Engine(64, 32, 16) as eng:
        eng.load_k(c1_k)
        for rnd, s in enumerate(c1["chosen"]):
            g = eng.peek_gains()
            for j in range(64):
                want = replay[rnd][j]
                if want is None:
                    assert np.isnan(g[j])
                else:
                    assert gain_close(g[j], want), (rnd, j, g[j], want)
            eng.step(forced=s)


def test_random_cases(dsel, O, golden_dir):
    """Reference random_hessian instances, including odd n_steps (1, 3, 5)."""
    cases = json.load(open(os.path.join(golden_dir, "random.json")))["cases"]
    for c in cases:
        nd, nt = c["n_sensors"], c["n_steps"]
        k = O.random_hessian(nd, nt, c["gamma"], c["rank"], c["seed"])
        eng, rows, n = run_engine(dsel, k, nd, nt, c["budget"])
        eng.close()
        assert_trace_matches(rows, c["chosen"], c["gains"], c["objectives"])


def test_selector_known_answers_on_gpu(dsel):
    """The reference's analytic selector cases, through the CUDA engine.

    diag(2,5,3), B=2 -> [1, 2] with gains log 5, log 3 (test_selector.cpp:94-101);
    K = [[4,2],[2,5]]: first pick 1 (log 5), then the Schur gain of 0 given 1,
    log(4 - 2*2/5) (the scalar Schur form of test_selector.cpp:48-62).
    """
    k = np.diag([2.0, 5.0, 3.0]).reshape(-1)
    eng, rows, n = run_engine(dsel, k, 3, 1, 2)
    eng.close()
    assert_trace_matches(rows, [1, 2], [np.log(5.0), np.log(3.0)])
    k = np.array([4.0, 2.0, 2.0, 5.0])
    eng, rows, n = run_engine(dsel, k, 2, 1, 2)
    eng.close()
    assert_trace_matches(rows, [1, 0], [np.log(5.0), np.log(4.0 - 4.0 / 5.0)])


def test_rescale_invariance_on_gpu(dsel, O):
    """K -> 3.7 K: same sequence, gains + Nt*log 3.7 (test_selector.cpp:160-175)."""
    nd, nt = 8, 3
    k = O.random_hessian(nd, nt, 1.0, 24, 5)
    ea, a, _ = run_engine(dsel, k, nd, nt, 5)
    eb, b, _ = run_engine(dsel, k * 3.7, nd, nt, 5)
    ea.close()
    eb.close()
    assert [r["chosen_index"] for r in a] == [r["chosen_index"] for r in b]
    for ra, rb in zip(a, b):
        want = ra["gain"] + nt * np.log(3.7)
        assert abs(rb["gain"] - want) <= 1e-10 * max(abs(want), 1.0)


def test_wave_benchmark_kbf(dsel, O, golden_dir):
    """The reference's standard wave benchmark K (assemble_k -> write_kbf);
    raw gains go negative here (step 8: -0.0994)."""
    w = json.load(open(os.path.join(golden_dir, "wave.json")))
    k, nd, nt = O.read_kbf(os.path.join(golden_dir, "wave.kbf"))
    eng, rows, n = run_engine(dsel, k, nd, nt, 12)
    eng.close()
    assert_trace_matches(rows, w["chosen"], w["gains"], w["objectives"])
    normalized = rows[-1]["objective"] - sum(w["noise_logdets"][s] for s in w["chosen"])
    assert abs(normalized - 1045.5268963527164) < 1e-8 * 1045.5


def test_block_column_ingest_and_candidates(dsel, O):
    """Exact block-column ingest + a candidate subset, against the oracle."""
    nd, nt = 14, 6
    k = O.random_hessian(nd, nt, 0.9, 60, 77)
    kb = k.reshape(nd, nd, nt, nt)
    cands = [0, 2, 3, 5, 7, 8, 11, 13]
    want = O.greedy_select(k, nd, nt, 6, candidates=cands)
    with dsel.Engine(nd, nt, 6, candidates=cands) as eng:
        for j in cands:
            eng.load_block_col(j, np.ascontiguousarray(kb[:, j]))
        eng.run()
        rows = eng.trace()
    assert_trace_matches(rows, want.chosen, want.gains, want.objectives)


def test_conditional_covariance_update_numerics(dsel, O):
    """The DMMA update/TRSM against a float64 numpy right-looking restatement:
    after each round the resident C equals K - K[:,S] K_SS^{-1} K[S,:]."""
    nd, nt = 24, 10
    k = O.random_hessian(nd, nt, 1.0, 200, 5)
    dense = O.blocks_to_dense(k, nd, nt)
    with dsel.Engine(nd, nt, 5) as eng:
        eng.load_k(k)
        S = []
        for _ in range(4):
            info = eng.step()
            S.append(info["chosen_index"])
            idx = np.concatenate([np.arange(s * nt, (s + 1) * nt) for s in S])
            cond = dense - dense[:, idx] @ np.linalg.solve(dense[np.ix_(idx, idx)], dense[idx, :])
            for j in range(nd):
                if j in S:
                    continue
                got = eng.read_block_row(j).reshape(nd, nt, nt)  # blocks (j, i)
                for i in range(nd):
                    if i in S:
                        continue
                    ref = cond[j * nt:(j + 1) * nt, i * nt:(i + 1) * nt]
                    np.testing.assert_allclose(got[i], ref, rtol=1e-10, atol=1e-10 * np.abs(dense).max())


def test_factor_export_matches_reference(dsel, O):
    nd, nt, B = 12, 4, 6
    k = O.random_hessian(nd, nt, 0.8, 48, 19)
    want = O.greedy_select(k, nd, nt, B, want_factor=True)
    with dsel.Engine(nd, nt, B, export_factor=True) as eng:
        eng.load_k(k)
        eng.run()
        L = eng.export_factor(B)
    dim = B * nt
    np.testing.assert_allclose(L, want.factor[:dim, :dim], rtol=1e-10, atol=1e-11)
    dense = O.blocks_to_dense(k, nd, nt)
    idx = np.concatenate([np.arange(s * nt, (s + 1) * nt) for s in want.chosen])
    np.testing.assert_allclose(L @ L.T, dense[np.ix_(idx, idx)], rtol=1e-10, atol=1e-10)
    assert np.all(np.triu(L, 1) == 0)


def test_reset_rerun_identical(dsel, c1_k):
    with dsel.Engine(64, 32, 16, keep_pristine=True) as eng:
        eng.load_k(c1_k)
        eng.run()
        a = eng.trace()
        eng.reset()
        eng.run()
        b = eng.trace()
    assert [r["chosen_index"] for r in a] == [r["chosen_index"] for r in b]
    assert [r["gain"] for r in a] == [r["gain"] for r in b]  # bitwise deterministic


def test_infeasible_and_budget_semantics(dsel, O):
    nd, nt = 5, 2
    # block 3 not positive definite -> infeasible every round; others fine
    k = O.random_hessian(nd, nt, 1.0, 10, 3).reshape(nd, nd, nt, nt)
    k[3, 3] = -np.eye(nt)
    k = np.ascontiguousarray(k.reshape(-1))
    with dsel.Engine(nd, nt, 4) as eng:
        eng.load_k(k)
        info = eng.step()
        assert info["n_infeasible"] == 1 and info["chosen_index"] != 3
    # round 1 all infeasible -> InfeasibleRound
    bad = np.zeros(nd * nd * nt * nt)
    with dsel.Engine(nd, nt, 2) as eng:
        eng.load_k(bad)
        with pytest.raises(dsel.InfeasibleRound):
            eng.step()
    # budget > candidates: select all + warning (parallel.hpp:295-297)
    good = O.random_hessian(nd, nt, 1.0, 10, 4)
    state, rep = dsel.gpu_greedy_select((good, nd, nt), [0, 1, 2], 5)
    assert len(state.chosen) == 3 and "budget exceeds" in rep.trace.warning
    state, rep = dsel.gpu_greedy_select((good, nd, nt), None, 0)
    assert state.chosen == [] and rep.trace.rows == []
    with pytest.raises(dsel.InvalidConfig):
        dsel.gpu_greedy_select((good, nd, nt), [0, 0], 1)
    with pytest.raises(dsel.IndexOutOfRange):
        dsel.gpu_greedy_select((good, nd, nt), [0, 9], 1)


def test_gpu_greedy_select_api(dsel, O, golden_dir):
    """Reference-shaped API incl. normalized mode (selector.hpp:136-142)."""
    w = json.load(open(os.path.join(golden_dir, "wave.json")))
    k, nd, nt = O.read_kbf(os.path.join(golden_dir, "wave.kbf"))
    opts = dsel.GpuOptions(mode="normalized", noise_logdets=w["noise_logdets"])
    state, rep = dsel.gpu_greedy_select((k, nd, nt), None, 12, opts)
    assert state.chosen == w["chosen"]
    assert abs(rep.trace.rows[-1].objective - 1045.5268963527164) < 1e-6
    L = state.factor
    dense = O.blocks_to_dense(k, nd, nt)
    idx = np.concatenate([np.arange(s * nt, (s + 1) * nt) for s in state.chosen])
    np.testing.assert_allclose(L @ L.T, dense[np.ix_(idx, idx)], rtol=1e-9, atol=1e-9)


def test_c2_against_reference_golden(dsel, golden_dir):
    """C2 (200 x Nt=128, rank 8192, B=50) end to end on the device."""
    path = os.path.join(golden_dir, "c2.json")
    if not os.path.exists(path):
        pytest.skip("c2 golden not generated")
    c2 = json.load(open(path))
    v = dsel.synthetic_v(200, 128, 8192, 2024)
    with dsel.Engine(200, 128, 50) as eng:
        eng.gen_synthetic(v, 8192, 1.0)
        eng.run()
        rows = eng.trace()
    assert_trace_matches(rows, c2["chosen"], c2["gains"], c2["objectives"])


def test_c3mini_nt420_against_reference_golden(dsel, golden_dir):
    """Nt = 420 (the CSZ block size): exercises the multi-panel gain kernel,
    k-padding (ldw = 432) and the ragged Schur-update tiles."""
    g = json.load(open(os.path.join(golden_dir, "c3mini.json")))
    nd, nt, rk, b = g["n_sensors"], g["n_steps"], g["rank"], g["budget"]
    v = dsel.synthetic_v(nd, nt, rk, g["seed"])
    with dsel.Engine(nd, nt, b) as eng:
        eng.gen_synthetic(v, rk, g["sigma"])
        for rnd, s in enumerate(g["chosen"]):
            gains = eng.peek_gains()
            for j in range(nd):
                want = g["replay_gains"][rnd][j]
                if want is None:
                    assert np.isnan(gains[j])
                else:
                    assert gain_close(gains[j], want), (rnd, j, gains[j], want)
            info = eng.step()
            assert info["chosen_index"] == s
            assert gain_close(info["gain"], g["gains"][rnd])


# ---- left-looking W-resident variant ------------------ #
@pytest.mark.parametrize("case", ["c1", "wave", "c3mini"])
def test_left_looking_matches_reference(dsel, O, golden_dir, case):
    g = json.load(open(os.path.join(golden_dir, f"{case}.json")))
    if case == "wave":
        k, nd, nt = O.read_kbf(os.path.join(golden_dir, "wave.kbf"))
        eng = dsel.Engine(nd, nt, 12, algorithm="left")
        eng.load_k(k)
    else:
        nd, nt, rk = g["n_sensors"], g["n_steps"], g["rank"]
        eng = dsel.Engine(nd, nt, g["budget"], algorithm="left")
        eng.gen_synthetic(dsel.synthetic_v(nd, nt, rk, g["seed"]), rk, g["sigma"])
    with eng:
        eng.run()
        rows = eng.trace()
        L = eng.export_factor(len(rows))
    assert_trace_matches(rows, g["chosen"], g["gains"], g["objectives"])
    if case == "wave":
        dense = O.blocks_to_dense(k, nd, nt)
        idx = np.concatenate([np.arange(s * nt, (s + 1) * nt) for s in g["chosen"]])
        np.testing.assert_allclose(L @ L.T, dense[np.ix_(idx, idx)], rtol=1e-9, atol=1e-9)


def test_left_looking_random_and_subsets(dsel, O, golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "random.json")))["cases"]
    for c in cases:
        nd, nt = c["n_sensors"], c["n_steps"]
        k = O.random_hessian(nd, nt, c["gamma"], c["rank"], c["seed"])
        eng = dsel.Engine(nd, nt, c["budget"], algorithm="left")
        eng.load_k(k)
        eng.run()
        rows = eng.trace()
        eng.close()
        assert_trace_matches(rows, c["chosen"], c["gains"], c["objectives"])
    # nt = 2 (mod 4): own rows land in the update tile at shifted positions
    for (nd, nt, rk, seed, B) in [(40, 6, 150, 11, 12), (33, 10, 200, 12, 9), (70, 2, 90, 3, 20)]:
        k = O.random_hessian(nd, nt, 1.0, rk, seed)
        want = O.greedy_select(k, nd, nt, B)
        with dsel.Engine(nd, nt, B, algorithm="left") as eng:
            eng.load_k(k)
            eng.run()
            assert_trace_matches(eng.trace(), want.chosen, want.gains, want.objectives)
    nd, nt = 14, 6
    k = O.random_hessian(nd, nt, 0.9, 60, 77)
    cands = [0, 2, 3, 5, 7, 8, 11, 13]
    want = O.greedy_select(k, nd, nt, 6, candidates=cands)
    with dsel.Engine(nd, nt, 6, candidates=cands, algorithm="left") as eng:
        eng.load_k(k)
        eng.run()
        assert_trace_matches(eng.trace(), want.chosen, want.gains, want.objectives)


# ---- out-of-HBM streaming store (storage = stream, left-looking) ---------- #
def test_streaming_store_matches_reference(dsel, O, golden_dir):
    """K never resides in HBM: the chosen column's blocks stream from pinned host
    memory each round (north-star (1)); same sequence and gains as the reference."""
    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    v = dsel.synthetic_v(64, 32, 2048, 2024)
    with dsel.Engine(64, 32, 16, algorithm="left", storage=2) as eng:
        eng.gen_synthetic(v, 2048, 1.0)          # generated on device, packed into the host store
        eng.run()
        rows = eng.trace()
        st = eng.stats()
    assert_trace_matches(rows, c1["chosen"], c1["gains"], c1["objectives"])
    assert st["io_ms"] > 0 and st["h2d_bytes"] > 0
    w = json.load(open(os.path.join(golden_dir, "wave.json")))
    k, nd, nt = O.read_kbf(os.path.join(golden_dir, "wave.kbf"))
    with dsel.Engine(nd, nt, 12, algorithm="left", storage=2) as eng:
        eng.load_k(k)
        eng.run()
        assert_trace_matches(eng.trace(), w["chosen"], w["gains"], w["objectives"])
    with dsel.Engine(nd, nt, 12, algorithm="left", storage=2) as eng:
        eng.load_kbf(os.path.join(golden_dir, "wave.kbf"), exact_columns=True)
        eng.run()
        assert [r["chosen_index"] for r in eng.trace()] == w["chosen"]
    c = json.load(open(os.path.join(golden_dir, "random.json")))["cases"][2]  # nt = 3
    nd, nt = c["n_sensors"], c["n_steps"]
    k = O.random_hessian(nd, nt, c["gamma"], c["rank"], c["seed"])
    with dsel.Engine(nd, nt, c["budget"], algorithm="left", storage=2) as eng:
        kb = k.reshape(nd, nd * nt * nt)
        for j in range(nd):
            eng.load_block_row(j, np.ascontiguousarray(kb[j]))
        eng.run()
        assert_trace_matches(eng.trace(), c["chosen"], c["gains"], c["objectives"])


def test_streaming_attached_host_k(dsel, O, golden_dir):
    """dsel_attach_host_k: the caller's K is the store (pageable -> registered in
    place, or pinned); per round only the chosen column's own blocks cross PCIe."""
    import torch

    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    k = O.synthetic_k(64, 32, 2048, 1.0, 2024)          # pageable numpy
    with dsel.Engine(64, 32, 16, algorithm="left", storage=2) as eng:
        eng.attach_host_k(k)
        eng.run()
        rows = eng.trace()
        st = eng.stats()
    assert_trace_matches(rows, c1["chosen"], c1["gains"], c1["objectives"])
    n2 = 32 * 32 * 8
    want_bytes = 64 * n2 + 15 * 64 * n2                  # diagonal + one column per round
    assert want_bytes <= st["h2d_bytes"] <= want_bytes + 4096
    kp = torch.from_numpy(k).pin_memory()                # pinned: used in place
    with dsel.Engine(64, 32, 16, algorithm="left", storage=2) as eng:
        eng.attach_host_k(kp)
        eng.run()
        assert_trace_matches(eng.trace(), c1["chosen"], c1["gains"], c1["objectives"])
        eng.reset()
        eng.run()                                        # rerun over the same attached K
        assert_trace_matches(eng.trace(), c1["chosen"], c1["gains"], c1["objectives"])
    # candidate subset (uneven slot spacing) and nt = 2 (mod 4)
    nd, nt = 30, 6
    k = O.random_hessian(nd, nt, 1.0, 100, 21)
    cands = [0, 1, 2, 4, 7, 8, 11, 13, 17, 18, 22, 25, 29]
    want = O.greedy_select(k, nd, nt, 7, candidates=cands)
    with dsel.Engine(nd, nt, 7, candidates=cands, algorithm="left", storage=2) as eng:
        eng.attach_host_k(k)
        eng.run()
        assert_trace_matches(eng.trace(), want.chosen, want.gains, want.objectives)
    with pytest.raises(dsel.InvalidConfig):
        with dsel.Engine(8, 2, 2) as eng:
            eng.attach_host_k(np.zeros(8 * 8 * 4))       # needs storage = stream


# ---- device-side synthetic K (C4/C5 scales: V never on the host) -------- #
from philox_ref import philox_v  # noqa: E402


@pytest.mark.parametrize("kw", [dict(), dict(full_square=True), dict(algorithm="left")])
def test_device_synthetic_k_and_selection(dsel, O, kw):
    """K formed on the device by the update kernel (Philox V) equals sigma^2 I + V V^T
    to rounding, and the selection on it matches the oracle run on the same K."""
    nd, nt, rank, B, seed = 40, 16, 300, 10, 77
    with dsel.Engine(nd, nt, B, **kw) as eng:
        eng.gen_synthetic_device(rank, 0.5, seed)
        k = np.concatenate([eng.read_block_row(j) for j in range(nd)])
        eng.run()
        rows = eng.trace()
    v = philox_v(nd, nt, rank, seed)
    want_dense = 0.25 * np.eye(nd * nt) + v @ v.T
    dense = O.blocks_to_dense(k, nd, nt)
    if not kw:   # block-lower store: compare the lower block triangle
        for i in range(nd):
            for j in range(i + 1):
                sl = np.s_[i * nt:(i + 1) * nt, j * nt:(j + 1) * nt]
                np.testing.assert_allclose(dense[sl], want_dense[sl], rtol=1e-12, atol=1e-11)
        dense = np.tril(dense) + np.tril(dense, -1).T
        k = np.ascontiguousarray(dense.reshape(nd, nt, nd, nt).transpose(0, 2, 1, 3)).reshape(-1)
    else:
        np.testing.assert_allclose(dense, want_dense, rtol=1e-12, atol=1e-11)
    want = O.greedy_select(k, nd, nt, B)
    assert_trace_matches(rows, want.chosen, want.gains, want.objectives)


# ---- K formation from an LTI wave problem (assemble_k on the GPU) -------- #
@pytest.mark.parametrize("name", ["wave_benchmark.cfg", "tiny.cfg", "weighted.cfg",
                                  "identity_prior.cfg", "larger.cfg"])
def test_assemble_lti_bit_exact(dsel, golden_dir, name):
    """`doptsel build` on the GPU: the KBF bytes hash to the reference's, the
    noise log-dets match, and the selection on the formed K is the reference's."""
    g = json.load(open(os.path.join(golden_dir, "lti.json")))["configs"][name]
    cfg = os.path.join(golden_dir, "configs", name)
    nd, nt, B = g["n_sensors"], g["n_steps"], g["budget"]
    for kw in (dict(), dict(algorithm="left"), dict(full_square=True)):
        with dsel.Engine(nd, nt, B, **kw) as eng:
            nl = eng.assemble_lti(cfg)
            k = np.concatenate([eng.read_block_row(j) for j in range(nd)])
            eng.run()
            rows = eng.trace()
        hdr = b"KBF1" + np.array([1, nd, nt, 1, 1, 0, 0], dtype="<u4").tobytes()
        assert hashlib.sha256(hdr + k.astype("<f8").tobytes()).hexdigest() == g["kbf_sha256"], kw
        assert np.array_equal(nl, np.array(g["noise_logdets"]))
        assert_trace_matches(rows, g["chosen"], g["gains"], g["objectives"])


# ---- GPU refactorizing baseline + complexity sweep ----- #
def test_naive_refactorizing_baseline_gpu(O, golden_dir):
    """naive_select (selector.hpp:253-348) on the GPU picks the reference
    sequence; the complexity sweep runs and its rows are well-formed."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(golden_dir), "..", "tools"))
    import complexity_gpu as cg

    w = json.load(open(os.path.join(golden_dir, "wave.json")))
    k, nd, nt = O.read_kbf(os.path.join(golden_dir, "wave.kbf"))
    chosen, gains, objs = cg.naive_select_gpu(k, nd, nt, 12)
    assert chosen == w["chosen"]
    for g, want in zip(gains, w["gains"]):
        assert abs(g - want) <= 1e-8 * max(abs(want), 1.0)
    c = json.load(open(os.path.join(golden_dir, "random.json")))["cases"][6]
    kr = O.random_hessian(c["n_sensors"], c["n_steps"], c["gamma"], c["rank"], c["seed"])
    chosen, _, _ = cg.naive_select_gpu(kr, c["n_sensors"], c["n_steps"], c["budget"], chunk=5)
    assert chosen == c["chosen"]
    rows, slopes = cg.sweep(nt=8, k_max=12, step=4, reps=2, batch=4)
    assert [r["k"] for r in rows] == [4, 8, 12]
    assert all(r["naive_ms"] > 0 and r["schur_ms"] > 0 and r["engine_round_ms"] > 0 for r in rows)


def test_out_of_memory_is_a_clean_error(dsel):
    """A store that cannot fit in HBM fails at create with DSEL_E_OOM (WorkerFailure),
    frees what it allocated, and the device stays usable."""
    with pytest.raises(dsel.WorkerFailure) as ei:
        dsel.Engine(4000, 420, 10, storage="hbm")  # n = 1.68M: an 11 TB packed panel store
    assert "OOM" in str(ei.value) or "cudaMalloc" in str(ei.value)
    with pytest.raises(dsel.WorkerFailure) as ei:  # AUTO: not even the streaming store fits
        dsel.Engine(4000, 420, 100)                # (W_own 0.58 TB)
    assert "OOM" in str(ei.value) and "streaming" in str(ei.value)
    with dsel.Engine(8, 2, 2) as eng:       # the device is still usable
        eng.load_k(np.eye(16).reshape(8, 2, 8, 2).transpose(0, 2, 1, 3).copy().reshape(-1) * 2.0)
        eng.run()
        assert len(eng.trace()) == 2
