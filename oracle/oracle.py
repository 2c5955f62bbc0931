"""ctypes front-end for the parity oracles (TEST INFRASTRUCTURE ONLY).

Two checkers live under oracle/:

* ``build/liboracle.so`` -- the plain-C restatement of the reference path
  (dsel_oracle.c, every function citing the reference file:line it follows);
* ``_ref/libdoptsel_ref.so`` -- the UNMODIFIED reference headers compiled from
  /root/reference with a C-callable harness (ref_harness.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference arm import this module. The product (paper_2604_08812_b200) never
does: it must fail loudly when its CUDA library is missing, never fall back
here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libdoptsel_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the oracle (and the reference harness when sources exist)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build()
        L = C.CDLL(_ORACLE_SO)
        L.orc_rng_normals.argtypes = [C.c_uint64, _dp, C.c_int64]
        L.orc_rng_u64.argtypes = [C.c_uint64, _up, C.c_int64]
        L.orc_rng_shuffle.argtypes = [C.c_uint64, _ip, C.c_int]
        L.orc_synthetic_v.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]
        L.orc_synthetic_materialize_rows.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double,
                                                     C.c_int, C.c_int, _dp]
        L.orc_synthetic_block_rows_fast.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_int,
                                                    C.c_double, C.c_int, _dp]
        L.orc_synthetic_block_rows_avx2.argtypes = L.orc_synthetic_block_rows_fast.argtypes
        L.orc_synthetic_v_uniforms.argtypes = [C.c_uint64, _dp, C.c_int64]
        L.orc_box_muller_pairs.argtypes = [_dp, C.c_int64, C.c_int64]
        L.orc_random_hessian.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, _dp]
        L.orc_cholesky_in_place.argtypes = [_dp, C.c_int, C.c_int]
        L.orc_cholesky_in_place.restype = C.c_int
        L.orc_solve_lower_in_place.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int]
        L.orc_solve_lower_in_place.restype = C.c_int
        L.orc_schur_in_place.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int]
        L.orc_logdet_from_factor.argtypes = [_dp, C.c_int, C.c_int]
        L.orc_logdet_from_factor.restype = C.c_double
        L.orc_greedy_select.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, C.c_int, _ip, _dp,
                                        _dp, _ip, _ip, C.c_void_p, C.c_void_p]
        L.orc_greedy_select.restype = C.c_int
        L.orc_replay_gains.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, _dp]
        L.orc_replay_gains.restype = C.c_int
        L.orc_reduce_argmax.argtypes = [_dp, _ip, C.c_int]
        L.orc_reduce_argmax.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise FileNotFoundError(f"{_REF_SO} not built (needs /root/reference at build time)")
        R = C.CDLL(_REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_synthetic_k.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _dp,
                                      C.c_int]
        R.ref_random_hessian.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64, _dp]
        R.ref_parallel_greedy.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, C.c_int, C.c_int,
                                          C.c_uint64, C.c_int, _ip, _dp, _dp, _ip, _ip, _dp, _ip,
                                          C.c_void_p, C.c_void_p]
        R.ref_greedy_select.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, C.c_int, _ip, _dp,
                                        _dp, _ip, _ip, _ip]
        R.ref_wave_kbf.argtypes = [C.c_char_p, _dp]
        R.ref_build_kbf.argtypes = [C.c_char_p, C.c_char_p, _dp]
        R.ref_write_kbf.argtypes = [_dp, C.c_int, C.c_int, C.c_char_p]
        R.ref_kbf_select.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, _ip, _dp, _dp,
                                     _ip, _ip, _ip]
        R.ref_timed_rounds.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, _ip, C.c_int,
                                       C.c_int, C.c_uint64, _dp, _dp]
        R.ref_replay.argtypes = [_dp, C.c_int, C.c_int, _ip, C.c_int, _dp]
        _ref = R
    return _ref


def _check_ref(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"reference harness rc={rc}: {ref().ref_last_error().decode()}")


# --------------------------------------------------------------------------- #
# Synthetic inputs                                                            #
# --------------------------------------------------------------------------- #
def synthetic_v(nd: int, nt: int, rank: int, seed: int) -> np.ndarray:
    """V of SyntheticKAccess (kaccess.hpp:89-92), shape (nd*nt, rank)."""
    v = np.empty(nd * nt * rank, dtype=np.float64)
    lib().orc_synthetic_v(nd, nt, rank, seed, v)
    return v.reshape(nd * nt, rank)


def synthetic_k(nd: int, nt: int, rank: int, sigma: float, seed: int,
                threads: int | None = None) -> np.ndarray:
    """Block-row-major K = sigma^2 I + V V^T (kaccess.hpp:98-116), via the C
    restatement, split over threads by block row."""
    import concurrent.futures as cf

    v = np.ascontiguousarray(synthetic_v(nd, nt, rank, seed).reshape(-1))
    k = np.empty(nd * nd * nt * nt, dtype=np.float64)
    threads = threads or min(os.cpu_count() or 1, nd)
    bounds = np.linspace(0, nd, threads + 1).astype(int)
    L = lib()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: L.orc_synthetic_materialize_rows(
            v, nd, nt, rank, sigma, int(bounds[i]), int(bounds[i + 1]), k), range(threads)))
    return k


def _cpu_has_avx2() -> bool:
    try:
        return " avx2" in open("/proc/cpuinfo").read()
    except OSError:
        return False


def synthetic_v_parallel(nd: int, nt: int, rank: int, seed: int,
                         threads: int | None = None) -> np.ndarray:
    """synthetic_v, bit for bit: uniforms drawn sequentially, the Box-Muller
    transform of the pairs split over threads (orc_box_muller_pairs)."""
    import concurrent.futures as cf

    count = nd * nt * rank
    buf = np.empty(count + (count & 1), dtype=np.float64)
    L = lib()
    L.orc_synthetic_v_uniforms(seed, buf, count)
    pairs = len(buf) // 2
    threads = threads or os.cpu_count() or 1
    bounds = np.linspace(0, pairs, threads + 1).astype(np.int64)
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda t: L.orc_box_muller_pairs(buf, int(bounds[t]), int(bounds[t + 1])),
                    range(threads)))
    return buf[:count].reshape(nd * nt, rank)


def synthetic_k_fast(nd: int, nt: int, rank: int, sigma: float, seed: int,
                     threads: int | None = None) -> np.ndarray:
    """synthetic_k, bit for bit, by the blocked/vectorized loop nests
    (orc_synthetic_block_rows_avx2 when the CPU has AVX2 and nt % 4 == 0, else
    orc_synthetic_block_rows_fast); for the large golden fixtures and the
    reference arm's input. Block-row-major (DataSpaceHessian) layout."""
    import concurrent.futures as cf

    threads = threads or os.cpu_count() or 1
    v = synthetic_v_parallel(nd, nt, rank, seed, threads)
    vt = np.ascontiguousarray(v.T).reshape(-1)
    v = np.ascontiguousarray(v.reshape(-1))
    k = np.empty(nd * nd * nt * nt, dtype=np.float64)
    L = lib()
    fn = (L.orc_synthetic_block_rows_avx2 if nt % 4 == 0 and _cpu_has_avx2()
          else L.orc_synthetic_block_rows_fast)
    # heavy rows (large i) first so the pool drains evenly
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: fn(v, vt, nd, nt, rank, sigma, i, k), range(nd - 1, -1, -1)))
    return k


def random_hessian(nd: int, nt: int, gamma: float, rank: int, seed: int) -> np.ndarray:
    k = np.empty(nd * nd * nt * nt, dtype=np.float64)
    lib().orc_random_hessian(nd, nt, gamma, rank, seed, k)
    return k


def blocks_to_dense(k: np.ndarray, nd: int, nt: int) -> np.ndarray:
    """Block-row-major raw K -> dense (nd*nt)^2 matrix."""
    return k.reshape(nd, nd, nt, nt).transpose(0, 2, 1, 3).reshape(nd * nt, nd * nt)


def dense_to_blocks(a: np.ndarray, nd: int, nt: int) -> np.ndarray:
    return np.ascontiguousarray(a.reshape(nd, nt, nd, nt).transpose(0, 2, 1, 3).reshape(-1))


# --------------------------------------------------------------------------- #
# Selection                                                                   #
# --------------------------------------------------------------------------- #
@dataclass
class OracleTrace:
    chosen: list = field(default_factory=list)
    gains: list = field(default_factory=list)
    objectives: list = field(default_factory=list)
    n_evaluated: list = field(default_factory=list)
    n_infeasible: list = field(default_factory=list)
    status: int = 0
    factor: np.ndarray | None = None
    gains_all: np.ndarray | None = None


def greedy_select(k: np.ndarray, nd: int, nt: int, budget: int, candidates=None,
                  want_factor: bool = False, want_gains_all: bool = False) -> OracleTrace:
    """C restatement of greedy_select<double> (selector.hpp:181-248)."""
    cands = np.arange(nd, dtype=np.int32) if candidates is None else np.asarray(
        candidates, dtype=np.int32)
    b = max(budget, 1)
    chosen = np.zeros(b, np.int32)
    gains = np.zeros(b)
    objs = np.zeros(b)
    ne = np.zeros(b, np.int32)
    ni = np.zeros(b, np.int32)
    fac = np.zeros((b * nt) ** 2) if want_factor else None
    ga = np.full(b * nd, np.nan) if want_gains_all else None
    rc = lib().orc_greedy_select(np.ascontiguousarray(k, dtype=np.float64), nd, nt, cands,
                                 len(cands), budget, chosen, gains, objs, ne, ni,
                                 fac.ctypes.data if fac is not None else None,
                                 ga.ctypes.data if ga is not None else None)
    t = OracleTrace(status=min(rc, 0))
    n = max(rc, 0)
    t.chosen, t.gains, t.objectives = chosen[:n].tolist(), gains[:n].tolist(), objs[:n].tolist()
    t.n_evaluated, t.n_infeasible = ne[:n].tolist(), ni[:n].tolist()
    if fac is not None:
        t.factor = fac.reshape(b * nt, b * nt)
    if ga is not None:
        t.gains_all = ga.reshape(b, nd)[:n]
    return t


def replay_gains(k: np.ndarray, nd: int, nt: int, sequence) -> np.ndarray:
    seq = np.asarray(sequence, dtype=np.int32)
    out = np.empty(len(seq) * nd)
    rc = lib().orc_replay_gains(np.ascontiguousarray(k), nd, nt, seq, len(seq), out)
    if rc != 0:
        raise RuntimeError("replay failed: chosen candidate infeasible")
    return out.reshape(len(seq), nd)


def reduce_argmax(pairs):
    d = np.array([p[0] for p in pairs], dtype=np.float64)
    s = np.array([p[1] for p in pairs], dtype=np.int32)
    i = lib().orc_reduce_argmax(d, s, len(pairs))
    if i < 0:
        raise ValueError("AllInfeasible")
    return (float(d[i]), int(s[i]))


# --------------------------------------------------------------------------- #
# The reference itself (oracle/_ref)                                          #
# --------------------------------------------------------------------------- #
def ref_synthetic_k(nd, nt, rank, sigma, seed, threads=None) -> np.ndarray:
    k = np.empty(nd * nd * nt * nt)
    _check_ref(ref().ref_synthetic_k(nd, nt, rank, sigma, seed, k, threads or os.cpu_count()))
    return k


def ref_random_hessian(nd, nt, gamma, rank, seed) -> np.ndarray:
    k = np.empty(nd * nd * nt * nt)
    _check_ref(ref().ref_random_hessian(nd, nt, gamma, rank, seed, k))
    return k


def ref_parallel_greedy(k, nd, nt, budget, workers=1, seed=0, pipeline=True, candidates=None,
                        want_factor=False):
    cands = np.arange(nd, dtype=np.int32) if candidates is None else np.asarray(
        candidates, dtype=np.int32)
    b = max(budget, 1)
    chosen = np.zeros(b, np.int32)
    gains = np.zeros(b)
    objs = np.zeros(b)
    ne = np.zeros(b, np.int32)
    ni = np.zeros(b, np.int32)
    wall = np.zeros(b)
    nrows = np.zeros(1, np.int32)
    fac = np.zeros((b * nt) ** 2) if want_factor else None
    sel_ms = C.c_double(0.0)
    rc = ref().ref_parallel_greedy(np.ascontiguousarray(k), nd, nt, cands, len(cands), budget,
                                   workers, seed, int(pipeline), chosen, gains, objs, ne, ni,
                                   wall, nrows, fac.ctypes.data if fac is not None else None,
                                   C.addressof(sel_ms))
    _check_ref(rc)
    n = int(nrows[0])
    t = OracleTrace(chosen=chosen[:n].tolist(), gains=gains[:n].tolist(),
                    objectives=objs[:n].tolist(), n_evaluated=ne[:n].tolist(),
                    n_infeasible=ni[:n].tolist())
    t.wall_ms = wall[:n].tolist()
    t.selection_ms = sel_ms.value
    t.warning = ref().ref_last_error().decode()
    if fac is not None:
        t.factor = fac.reshape(b * nt, b * nt)
    return t


def ref_replay(k, nd, nt, sequence) -> np.ndarray:
    seq = np.asarray(sequence, dtype=np.int32)
    out = np.empty(len(seq) * nd)
    _check_ref(ref().ref_replay(np.ascontiguousarray(k), nd, nt, seq, len(seq), out))
    return out.reshape(len(seq), nd)


def ref_wave_kbf(path: str) -> np.ndarray:
    nl = np.zeros(32)
    _check_ref(ref().ref_wave_kbf(path.encode(), nl))
    return nl


def ref_build_kbf(config_path: str, out_path: str, n_sensors: int) -> np.ndarray:
    """Reference `doptsel build` (assemble_k -> write_kbf); returns noise log-dets."""
    nl = np.zeros(n_sensors)
    _check_ref(ref().ref_build_kbf(config_path.encode(), out_path.encode(), nl))
    return nl


def ref_write_kbf(k, nd, nt, path: str) -> None:
    _check_ref(ref().ref_write_kbf(np.ascontiguousarray(k), nd, nt, path.encode()))


def ref_kbf_select(path: str, budget: int, workers: int = 1, seed: int = 0) -> OracleTrace:
    b = max(budget, 1)
    chosen = np.zeros(b, np.int32)
    gains = np.zeros(b)
    objs = np.zeros(b)
    nrows = np.zeros(1, np.int32)
    nd = np.zeros(1, np.int32)
    nt = np.zeros(1, np.int32)
    _check_ref(ref().ref_kbf_select(path.encode(), budget, workers, seed, chosen, gains, objs,
                                    nrows, nd, nt))
    n = int(nrows[0])
    return OracleTrace(chosen=chosen[:n].tolist(), gains=gains[:n].tolist(),
                       objectives=objs[:n].tolist())


def ref_timed_rounds(k, nd, nt, prefix, iterates, workers, seed=0):
    """Wall ms of one reference evaluation round at each iterate (bounded
    CPU sample; see ref_harness.cpp ref_timed_rounds)."""
    pre = np.asarray(prefix, dtype=np.int32)
    its = np.asarray(iterates, dtype=np.int32)
    out = np.zeros(len(its))
    setup = np.zeros(len(its))
    _check_ref(ref().ref_timed_rounds(np.ascontiguousarray(k), nd, nt, pre, len(pre), its,
                                      len(its), workers, seed, out, setup))
    return out, setup


def read_kbf(path: str):
    """Parse a KBF file (kstore.hpp:22-35) into (raw block-row-major K, nd, nt)."""
    with open(path, "rb") as f:
        hdr = f.read(32)
        assert hdr[:4] == b"KBF1"
        ver, nd, nt, dt, order = np.frombuffer(hdr[4:24], dtype="<u4")
        assert ver == 1 and dt == 1 and order == 1
        k = np.fromfile(f, dtype="<f8")
    return k, int(nd), int(nt)
