"""CPU tests: pin the oracle (oracle/dsel_oracle.c) against the reference.

* the reference's own analytic known-answer tests (proj/tests/test_linalg.cpp,
  test_selector.cpp, test_parallel.cpp);
* golden vectors produced by the reference itself (tests/golden/*.json, made
  by tests/golden/make_golden.py from oracle/_ref);
* the SURVEY.md Appendix A record (C1 sequence, gains, KBF sha256).
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O


def gain_close(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(abs(b), 1.0)


# ---- linalg.hpp known answers (test_linalg.cpp) --------------------------- #
def chol(a):
    a = np.array(a, dtype=np.float64)
    rc = O.lib().orc_cholesky_in_place(a.reshape(-1), a.shape[0], a.shape[1])
    return a, rc


def test_cholesky_known_answers():
    a, rc = chol([[4.0, 2.0], [2.0, 5.0]])
    assert rc == -1 and a.tolist() == [[2.0, 0.0], [1.0, 2.0]]
    a, rc = chol([[4.0]])
    assert rc == -1 and a.tolist() == [[2.0]]
    a, rc = chol(np.eye(3))
    assert rc == -1 and np.array_equal(a, np.eye(3))
    # NPD at pivot 1 (test_linalg.cpp:82-95); NaN rejected
    _, rc = chol([[1.0, 2.0], [2.0, 1.0]])
    assert rc == 1
    _, rc = chol([[float("nan")]])
    assert rc == 0


def test_solve_schur_logdet_known_answers():
    L = O.lib()
    l = np.array([2.0, 0.0, 1.0, 2.0])
    x = np.array([4.0, 4.0])
    assert L.orc_solve_lower_in_place(l, 2, 2, x, 1, 1) == -1
    assert x.tolist() == [2.0, 1.0]
    sing = np.array([1.0, 0.0, 3.0, 0.0])
    assert L.orc_solve_lower_in_place(sing, 2, 2, np.zeros(2), 1, 1) == 1
    m = np.array([5.0])
    L.orc_schur_in_place(m, 1, 1, np.array([2.0]), 1, 1)
    assert m[0] == 1.0
    assert L.orc_logdet_from_factor(np.array([2.0, 0.0, 1.0, 2.0]), 2, 2) == pytest.approx(
        math.log(16.0), rel=1e-15)
    assert L.orc_logdet_from_factor(np.eye(4).reshape(-1), 4, 4) == 0.0


def test_reduce_argmax_tie_rule():
    # test_parallel.cpp:42-49
    assert O.reduce_argmax([(1.0, 5), (2.0, 3)]) == (2.0, 3)
    assert O.reduce_argmax([(2.0, 7), (2.0, 3)]) == (2.0, 3)
    with pytest.raises(ValueError):
        O.reduce_argmax([(0.0, -1), (0.0, -1)])


def test_selector_known_answers():
    # diagonal K diag(2,5,3), B=2 -> [1, 2] (test_selector.cpp:94-101)
    k = np.diag([2.0, 5.0, 3.0]).reshape(-1)
    t = O.greedy_select(k, 3, 1, 2)
    assert t.chosen == [1, 2]
    assert t.gains == pytest.approx([math.log(5.0), math.log(3.0)], rel=1e-15)
    # scalar Schur gain log 4 (test_selector.cpp:48-62): K = [[4,2],[2,5]]
    k = np.array([4.0, 2.0, 2.0, 5.0])
    ga = O.replay_gains(k, 2, 1, [0, 1])
    assert ga[1, 1] == pytest.approx(math.log(4.0), rel=1e-12)


def test_rescale_invariance():
    # K -> 3.7 K: same sequence, gains + nt*log(3.7) (test_selector.cpp:160-175)
    nd, nt = 8, 3
    k = O.random_hessian(nd, nt, 1.0, 24, 5)
    a = O.greedy_select(k, nd, nt, 5)
    b = O.greedy_select(k * 3.7, nd, nt, 5)
    assert a.chosen == b.chosen
    for ga, gb in zip(a.gains, b.gains):
        assert gb == pytest.approx(ga + nt * math.log(3.7), rel=1e-10, abs=1e-10)


# ---- pinned against the reference itself ---------------------------------- #
def test_c1_golden_survey_record(golden_dir):
    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    # SURVEY.md Appendix A (recorded with the reference, -O3, no -march)
    assert c1["chosen"] == [8, 11, 22, 18, 54, 25, 23, 24, 2, 41, 62, 47, 26, 9, 53, 55]
    assert c1["gains"][0] == 244.21655015270287
    assert c1["gains"][-1] == 235.3230469396766
    assert c1["objectives"][-1] == 3838.3884795896265
    assert c1["kbf_sha256"] == "aca0214febd0420f4aa0c29dbcf9bf8a4196373874c218a05a7a47e287b2890f"


@pytest.fixture(scope="module")
def c1_k():
    return O.synthetic_k(64, 32, 2048, 1.0, 2024)


def test_oracle_synthetic_k_matches_reference_bytes(golden_dir, c1_k):
    """C restatement of SyntheticKAccess reproduces the reference KBF bytes."""
    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    hdr = b"KBF1" + np.array([1, 64, 32, 1, 1, 0, 0], dtype="<u4").tobytes()
    assert hashlib.sha256(hdr + c1_k.astype("<f8").tobytes()).hexdigest() == c1["kbf_sha256"]


def test_oracle_c1_bitwise_equals_reference_golden(golden_dir, c1_k):
    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    t = O.greedy_select(c1_k, 64, 32, 16)
    assert t.chosen == c1["chosen"]
    assert t.gains == c1["gains"]            # bitwise: same operation order
    assert t.objectives == c1["objectives"]
    assert t.n_evaluated == c1["n_evaluated"]


def test_oracle_replay_matches_reference(golden_dir, c1_k):
    c1 = json.load(open(os.path.join(golden_dir, "c1.json")))
    ga = O.replay_gains(c1_k, 64, 32, c1["chosen"][:6])
    for r in range(6):
        for j in range(64):
            want = c1["replay_gains"][r][j]
            if want is None:
                assert np.isnan(ga[r, j])
            else:
                assert ga[r, j] == want


def test_oracle_random_cases_match_reference(golden_dir):
    cases = json.load(open(os.path.join(golden_dir, "random.json")))["cases"]
    for c in cases:
        k = O.random_hessian(c["n_sensors"], c["n_steps"], c["gamma"], c["rank"], c["seed"])
        t = O.greedy_select(k, c["n_sensors"], c["n_steps"], c["budget"])
        assert t.chosen == c["chosen"]
        assert t.gains == c["gains"]
        assert t.objectives == c["objectives"]


def test_oracle_wave_matches_reference(golden_dir):
    w = json.load(open(os.path.join(golden_dir, "wave.json")))
    path = os.path.join(golden_dir, "wave.kbf")
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == w["kbf_sha256"]
    # SURVEY.md Appendix A wave record
    assert w["kbf_sha256"] == "0efbac46a490f3ff7688d3bb4589d4140da19246db35cb04db830b08afe659f9"
    k, nd, nt = O.read_kbf(path)
    t = O.greedy_select(k, nd, nt, 12)
    assert t.chosen == w["chosen"] == [9, 21, 30, 2, 14, 26, 5, 25, 11, 16, 31, 0]
    assert t.gains == w["gains"]
    norm = t.objectives[-1] - sum(w["noise_logdets"][s] for s in t.chosen)
    assert norm == pytest.approx(1045.5268963527164, rel=1e-14)


def test_c2_golden_survey_record(golden_dir):
    path = os.path.join(golden_dir, "c2.json")
    if not os.path.exists(path):
        pytest.skip("c2 golden not generated yet")
    c2 = json.load(open(path))
    assert c2["chosen"][:5] == [145, 178, 23, 109, 70]
    assert c2["chosen"][-1] == 67
    assert c2["objectives"][-1] == pytest.approx(54017.09293423091, rel=1e-15)
    assert c2["kbf_sha256"] == "f8409a2dfcd401b0aba6b2fddda010fe33a5718a8e846e0c82f1d21a8b587b85"


@pytest.mark.skipif(not O.ref_available(), reason="reference build (oracle/_ref) absent")
def test_oracle_vs_reference_live():
    """Live cross-check against the compiled reference on fresh seeds."""
    for seed in (11, 12):
        k = O.ref_random_hessian(9, 3, 0.9, 30, seed)
        assert np.array_equal(k, O.random_hessian(9, 3, 0.9, 30, seed))
        a = O.ref_parallel_greedy(k, 9, 3, 5, workers=3, seed=seed)
        b = O.greedy_select(k, 9, 3, 5)
        assert a.chosen == b.chosen and a.gains == b.gains


def test_c3mini_golden_is_reference_output(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "c3mini.json")))
    assert g["n_steps"] == 420 and len(g["chosen"]) == 6
    # the replay of the reference's own sequence picks the reference winner each round
    for rnd, s in enumerate(g["chosen"]):
        row = g["replay_gains"][rnd]
        best = max((x, -j) for j, x in enumerate(row) if x is not None)
        assert -best[1] == s and best[0] == g["gains"][rnd]


def test_fast_generators_bit_identical(golden_dir, c1_k):
    """The blocked generators that materialize the large fixtures and the
    reference arm's K (synthetic_k_fast: AVX2 4x8 register tiles or the
    portable blocked loop; synthetic_v_parallel) reproduce SyntheticKAccess
    bit for bit -- including ragged widths (nt % 8 == 4) and odd nt."""
    k = O.synthetic_k_fast(64, 32, 2048, 1.0, 2024, threads=4)
    assert np.array_equal(k.view(np.uint64), c1_k.view(np.uint64))
    for (nd, nt, rank, seed) in [(5, 12, 301, 3), (4, 20, 77, 9), (3, 7, 50, 1)]:
        a = O.synthetic_k(nd, nt, rank, 1.0, seed)
        b = O.synthetic_k_fast(nd, nt, rank, 1.0, seed, threads=3)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (nd, nt)
    v1 = O.synthetic_v(6, 5, 33, 2024)  # odd count: the last pair's sine is dropped
    v2 = O.synthetic_v_parallel(6, 5, 33, 2024, threads=4)
    assert np.array_equal(v1.view(np.uint64), v2.view(np.uint64))


def test_edge_golden_is_reference_output(golden_dir):
    """tests/golden/edge.json: exact ties go to the lower index, exact zero
    pivots are infeasible, the run ends with a partial selection -- as the
    reference produced it (and the C restatement agrees)."""
    for c in json.load(open(os.path.join(golden_dir, "edge.json")))["cases"]:
        k = np.array(c["k_raw"])
        t = O.greedy_select(k, c["n_sensors"], c["n_steps"], c["budget"])
        assert t.chosen == c["chosen"] and t.gains == c["gains"], c["name"]
        assert t.n_infeasible[:len(c["chosen"])] == c["n_infeasible"], c["name"]


def test_c3_golden_is_a_complete_reference_run(golden_dir):
    """tests/golden/c3.json: BASELINE configs[2] at G = 1 (75 x Nt=420, rank
    24,576, select 50), the reference's own run_parallel_greedy on 8 workers."""
    path = os.path.join(golden_dir, "c3.json")
    if not os.path.exists(path):
        pytest.skip("c3 golden not generated")
    g = json.load(open(path))
    assert (g["n_sensors"], g["n_steps"], g["rank"], g["budget"]) == (75, 420, 24576, 50)
    assert len(g["chosen"]) == 50 == len(set(g["chosen"]))
    assert all(b > a for a, b in zip(g["objectives"], g["objectives"][1:]))
    assert g["n_evaluated"] == list(range(75, 25, -1))
    assert "reference run_parallel_greedy" in g["source"]
