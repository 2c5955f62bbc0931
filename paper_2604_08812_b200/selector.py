"""Host-side mirror of the reference selection interface over the C ABI.

Reference interface (C++, /root/reference/proj/include/doptsel):
  greedy_select<Real,A>(k, candidates, budget, opts)        selector.hpp:181-248
  run_parallel_greedy<Real,A>(k, candidates, budget, opts)  parallel.hpp:281-483
  -> (SelectionState{chosen, factor, objective}, SelectionTrace{rows, warning})

Here the same call goes to libdsel.so (one engine per GPU). Error behaviour
follows errors.hpp: InvalidConfig / IndexOutOfRange raised before any work,
InfeasibleRound when round 1 has no feasible candidate, a partial selection
with a warning when a later round has none, WorkerFailure for device or
collective failures. The C++ drop-in for the reference tree is
include/doptsel_gpu.hpp; this module is what tests and bench.py drive.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._abi import (DSEL_OK, STATUS_NAMES, DselArgRec, DselConfig, DselLti, DselPlan, DselStats,
                   DselStepInfo, lib)

STORAGE = {"auto": 0, "hbm": 1, "stream": 2}


# ---- errors (errors.hpp:10-86) -------------------------------------------- #
class DselError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class InvalidConfig(DselError):
    pass


class IndexOutOfRange(DselError):
    pass


class InfeasibleRound(DselError):
    round = 1


class WorkerFailure(DselError):
    pass


class IoError(DselError):
    pass


class CorruptFile(IoError):
    pass


_EXC = {1: InvalidConfig, 2: IndexOutOfRange, 3: InfeasibleRound, 4: WorkerFailure,
        5: WorkerFailure, 6: WorkerFailure, 7: IoError, 8: DselError, 9: CorruptFile}


def _check(rc: int, handle=None) -> None:
    if rc != DSEL_OK:
        msg = lib.dsel_last_error(handle).decode(errors="replace")
        raise _EXC.get(rc, DselError)(rc, msg)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _host_ptr(a):
    """numpy array or (pinned) torch CPU tensor -> void*."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"] or a.dtype != np.float64:
            raise InvalidConfig(1, "host K must be C-contiguous float64")
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


def measure_fp64_peak(device: int = 0) -> float:
    """FP64 tensor-core (DMMA) peak of the device in TFLOP/s, measured now."""
    out = C.c_double(0.0)
    _check(lib.dsel_measure_fp64_peak(device, C.byref(out)))
    return out.value


def batched_logdet(mats, logdet=None, status=None):
    """log det of a batch of SPD matrices on the GPU (dsel_batched_logdet).
    mats: a CUDA float64 torch tensor (batch, m, m); symmetric, so row- and
    column-major agree. Returns (logdet, status) tensors; logdet = -inf and
    status = failing pivot for a matrix that is not positive definite."""
    import torch

    if mats.dtype != torch.float64 or not mats.is_cuda or mats.dim() != 3:
        raise InvalidConfig(1, "batched_logdet needs a (batch, m, m) float64 CUDA tensor")
    mats = mats.contiguous()
    b, m, _ = mats.shape
    if logdet is None:
        logdet = torch.empty(b, dtype=torch.float64, device=mats.device)
    if status is None:
        status = torch.empty(b, dtype=torch.int32, device=mats.device)
    _check(lib.dsel_batched_logdet(mats.device.index or 0, C.c_void_p(mats.data_ptr()), m, m * m, b,
                                   C.c_void_p(logdet.data_ptr()), C.c_void_p(status.data_ptr())))
    return logdet, status


def alloc_count() -> int:
    """Device/pinned allocations made by libdsel so far (all engines)."""
    return int(lib.dsel_alloc_count())


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib.dsel_nccl_unique_id(buf))
    return bytes(buf)


def fold_records(records):
    """The per-round fold every rank applies to the allgathered argmax records
    (dsel_fold_records; reduce_argmax semantics, parallel.hpp:61-74).
    records: iterable of (g1, s1, g2, s2, n_eval, n_inf). Returns the same tuple."""
    recs = list(records)
    arr = (DselArgRec * max(len(recs), 1))()
    for i, (g1, s1, g2, s2, ne, ni) in enumerate(recs):
        arr[i] = DselArgRec(g1, g2, s1, s2, ne, ni)
    out = DselArgRec()
    lib.dsel_fold_records(arr, len(recs), C.byref(out))
    return (out.g1, out.s1, out.g2, out.s2, out.n_eval, out.n_inf)


def synthetic_v(n_sensors: int, n_steps: int, rank: int, seed: int, threads: int = 0) -> np.ndarray:
    """V of SyntheticKAccess (kaccess.hpp:89-92), bit-identical, shape (nd*nt, rank)."""
    out = np.empty(n_sensors * n_steps * rank, dtype=np.float64)
    _check(lib.dsel_synthetic_v(n_sensors, n_steps, rank, seed, _ptr(out), threads))
    return out.reshape(n_sensors * n_steps, rank)


@dataclass
class LtiProblem:
    """Host tables of an LTI wave problem (lti.hpp:62-120): impulse[s][j][tau],
    materialized spatial prior[i][j], optional mask[j][t] and cost weights."""
    n_params: int
    n_sensors: int
    n_steps: int
    noise_sigma: float
    impulse: np.ndarray
    spatial: np.ndarray
    mask: np.ndarray | None = None
    cost_weights: np.ndarray | None = None

    @classmethod
    def from_config(cls, path: str) -> "LtiProblem":
        """Reference problem config (config.hpp) -> make_wave_problem tables."""
        lt, owner = DselLti(), C.c_void_p()
        _check(lib.dsel_lti_from_config(path.encode(), C.byref(lt), C.byref(owner)))
        try:
            nm, nd, nt = lt.n_params, lt.n_sensors, lt.n_steps

            def arr(ptr, count):
                return None if not ptr else np.ctypeslib.as_array(
                    C.cast(ptr, C.POINTER(C.c_double)), shape=(count,)).copy()

            return cls(nm, nd, nt, lt.noise_sigma, arr(lt.impulse, nd * nm * nt),
                       arr(lt.spatial, nm * nm), arr(lt.mask, nm * nt), arr(lt.cost_weights, nd))
        finally:
            lib.dsel_lti_free(owner)

    def _struct(self):
        keep = [np.ascontiguousarray(x, dtype=np.float64) if x is not None else None
                for x in (self.impulse, self.spatial, self.mask, self.cost_weights)]
        lt = DselLti(self.n_params, self.n_sensors, self.n_steps, self.noise_sigma,
                     *[x.ctypes.data if x is not None else None for x in keep])
        return lt, keep


class Engine:
    """One selection engine on one GPU (one rank of a world_size group)."""

    def __init__(self, n_sensors: int, n_steps: int, budget: int, candidates=None, device: int = 0,
                 world_size: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 keep_pristine: bool = False, export_factor: bool = False,
                 near_tie_tau: float = 1e-9, storage: int | str = 0, full_square: bool = False,
                 algorithm: str = "right", packed: bool = True, hbm_budget: int = 0):
        cfg = DselConfig()
        cfg.n_sensors, cfg.n_steps, cfg.budget = n_sensors, n_steps, budget
        self._cands = None
        if candidates is not None:
            self._cands = np.ascontiguousarray(np.asarray(candidates, dtype=np.int32))
            cfg.n_candidates = len(self._cands)
            cfg.candidates = self._cands.ctypes.data_as(C.POINTER(C.c_int))
        cfg.device, cfg.world_size, cfg.rank = device, world_size, rank
        self._id = None
        if nccl_id is not None:
            self._id = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
            cfg.nccl_id = C.cast(self._id, C.c_void_p)
        cfg.storage = STORAGE[storage] if isinstance(storage, str) else int(storage)
        cfg.panel_layout = 0 if packed else 1
        cfg.hbm_budget = int(hbm_budget)
        cfg.keep_pristine = int(keep_pristine)
        cfg.export_factor = int(export_factor)
        cfg.near_tie_tau = near_tie_tau
        cfg.full_square = int(full_square)
        if algorithm not in ("right", "left"):
            raise InvalidConfig(1, "algorithm must be 'right' or 'left'")
        cfg.algorithm = 1 if algorithm == "left" else 0
        h = C.c_void_p()
        _check(lib.dsel_create(C.byref(cfg), C.byref(h)), None)
        self.h = h
        self.n_sensors, self.n_steps, self.budget = n_sensors, n_steps, budget
        self.world_size, self.rank = world_size, rank

    # -- lifecycle --
    def close(self) -> None:
        if getattr(self, "h", None):
            lib.dsel_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def sync(self) -> None:
        _check(lib.dsel_sync(self.h), self.h)

    @property
    def device_bytes(self) -> int:
        return int(lib.dsel_device_bytes(self.h))

    def plan(self) -> dict:
        """Storage plan dsel_create resolved (AUTO -> hbm | stream) and its sizes."""
        p = DselPlan()
        _check(lib.dsel_get_plan(self.h, C.byref(p)), self.h)
        d = p.as_dict()
        d["storage"] = {1: "hbm", 2: "stream"}.get(d["storage"], d["storage"])
        d["algorithm"] = "left" if d["algorithm"] else "right"
        return d

    # -- panel store ingest --
    def load_k(self, k) -> None:
        """Whole K, block-row-major (DataSpaceHessian / KBF payload order)."""
        _check(lib.dsel_load_k(self.h, _host_ptr(k)), self.h)

    def attach_host_k(self, k) -> None:
        """Streaming store over the caller's K (same layout as load_k) in host
        memory, read in place: per round only the chosen column's blocks for
        this rank's candidates cross PCIe. The engine keeps a reference."""
        _check(lib.dsel_attach_host_k(self.h, _host_ptr(k)), self.h)
        self._hk = k

    def attach_host_rows(self, rows) -> None:
        """attach_host_k over this rank's own block rows only (candidates at
        positions p % world_size == rank, stacked in candidate order)."""
        _check(lib.dsel_attach_host_rows(self.h, _host_ptr(rows)), self.h)
        self._hk = rows

    def load_kbf(self, path: str, exact_columns: bool = True, threads: int = 0) -> None:
        """KBF store (kstore.hpp:22-186) -> this engine's panels."""
        _check(lib.dsel_load_kbf(self.h, path.encode(), int(exact_columns), threads), self.h)

    def attach_kbf(self, path: str, threads: int = 0) -> None:
        """File-backed streaming store (storage='stream'): each round preads
        only the chosen column's own blocks from the KBF file."""
        _check(lib.dsel_attach_kbf(self.h, path.encode(), threads), self.h)

    def load_block_row(self, j: int, row) -> None:
        _check(lib.dsel_load_block_row(self.h, j, _host_ptr(row)), self.h)

    def load_block_col(self, j: int, col) -> None:
        _check(lib.dsel_load_block_col(self.h, j, _host_ptr(col)), self.h)

    def gen_synthetic(self, v: np.ndarray, rank: int, sigma: float) -> None:
        v = np.ascontiguousarray(v, dtype=np.float64)
        _check(lib.dsel_gen_synthetic(self.h, _ptr(v), rank, sigma), self.h)

    def gen_synthetic_device(self, rank: int, sigma: float, seed: int) -> None:
        """K = sigma^2 I + V V^T with V from the device Philox stream (not the
        reference RNG; for C4/C5 scales where V cannot live on the host)."""
        _check(lib.dsel_gen_synthetic_device(self.h, rank, sigma, seed), self.h)

    def assemble_lti(self, problem: "LtiProblem | str") -> np.ndarray:
        """K = Gamma_noise + F W Gamma_prior W F^T formed on the GPU, bit-identical
        to assemble_k (hessian.hpp:91-144); a config path or an LtiProblem.
        Returns the per-sensor noise log-dets (noise_block_logdets)."""
        if isinstance(problem, str):
            problem = LtiProblem.from_config(problem)
        lt, keep = problem._struct()
        out = np.zeros(self.n_sensors)
        _check(lib.dsel_assemble_lti(self.h, C.byref(lt), _ptr(out)), self.h)
        del keep
        return out

    def read_block_row(self, j: int) -> np.ndarray:
        out = np.empty(self.n_sensors * self.n_steps * self.n_steps)
        _check(lib.dsel_read_block_row(self.h, j, _ptr(out)), self.h)
        return out

    # -- selection --
    def step(self, forced: int | None = None) -> dict:
        info = DselStepInfo()
        if forced is None:
            _check(lib.dsel_step(self.h, C.byref(info)), self.h)
        else:
            _check(lib.dsel_step_forced(self.h, int(forced), C.byref(info)), self.h)
        return info.as_dict()

    def run(self) -> int:
        n = C.c_int(0)
        _check(lib.dsel_run(self.h, C.byref(n)), self.h)
        return n.value

    def peek_gains(self) -> np.ndarray:
        g = np.full(self.n_sensors, np.nan)
        _check(lib.dsel_peek_gains(self.h, _ptr(g)), self.h)
        return g

    def trace(self) -> list:
        rows = (DselStepInfo * max(self.budget, 1))()
        n = lib.dsel_get_trace(self.h, rows, max(self.budget, 1))
        if n < 0:
            _check(4, self.h)
        return [rows[i].as_dict() for i in range(n)]

    def stats(self) -> dict:
        st = DselStats()
        _check(lib.dsel_get_stats(self.h, C.byref(st)), self.h)
        return st.as_dict()

    def reset(self) -> None:
        _check(lib.dsel_reset(self.h), self.h)

    def export_factor(self, k: int) -> np.ndarray:
        dim = k * self.n_steps
        out = np.zeros((max(dim, 1), max(dim, 1)))
        if k:
            _check(lib.dsel_export_factor(self.h, _ptr(out), dim), self.h)
        return out[:dim, :dim]


# ---- reference-shaped results (selector.hpp:31-54, parallel.hpp:23-52) ---- #
@dataclass
class TraceRow:
    k: int
    chosen_index: int
    objective: float
    gain: float
    n_evaluated: int
    n_infeasible: int
    wall_ms: float
    mean_candidate_ms: float
    runner_up: int = -1
    runner_up_gain: float = float("-inf")
    near_tie: bool = False


@dataclass
class SelectionState:
    chosen: list
    factor: np.ndarray | None
    objective: float


@dataclass
class SelectionTrace:
    rows: list = field(default_factory=list)
    warning: str = ""


@dataclass
class RoundResult:
    d_max: float
    s_star: int
    bytes_exchanged: int
    ms: dict


@dataclass
class ParallelRunReport:
    trace: SelectionTrace
    rounds: list


@dataclass
class GpuOptions:
    """GpuOptions of SURVEY.md §8(b): ParallelOptions (parallel.hpp:37-47) with
    n_workers -> one engine per GPU. `seed` is accepted and, as in the
    reference, does not change results (the shuffle is result-invariant)."""
    device: int = 0
    world_size: int = 1
    rank: int = 0
    nccl_id: bytes | None = None
    mode: str = "raw"              # raw | normalized (SelectionOptions, selector.hpp:26-29)
    noise_logdets: list | None = None
    near_tie_tau: float = 1e-9
    export_factor: bool = True
    seed: int = 0


def gpu_greedy_select(k, candidates, budget: int, opts: GpuOptions | None = None):
    """Drop-in for run_parallel_greedy<double> (parallel.hpp:281-483).

    k: either a raw block-row-major array with attributes given as a tuple
    (k_raw, n_sensors, n_steps), or an object with n_sensors(), n_steps() and
    read_block(i, j, out) (the KAccess concept, kaccess.hpp:18-23).
    Returns (SelectionState, ParallelRunReport).
    """
    opts = opts or GpuOptions()
    if isinstance(k, tuple):
        k_raw, nd, nt = k
        reader = None
    else:
        k_raw, nd, nt, reader = None, int(k.n_sensors()), int(k.n_steps()), k
    if budget < 0:
        raise InvalidConfig(1, "budget must be nonnegative")
    cands = list(range(nd)) if candidates is None else [int(c) for c in candidates]
    seen = set()
    for c in cands:
        if c < 0 or c >= nd:
            raise IndexOutOfRange(2, "candidate index out of range")
        if c in seen:
            raise InvalidConfig(1, "duplicate candidate index")
        seen.add(c)
    if opts.mode == "normalized" and (opts.noise_logdets is None or len(opts.noise_logdets) != nd):
        raise InvalidConfig(1, "normalized mode requires one noise log-determinant per sensor")
    trace = SelectionTrace()
    if budget > len(cands):
        trace.warning = "budget exceeds candidate count; selecting all candidates"
    eff = min(budget, len(cands))
    if eff == 0 or not cands:
        return SelectionState([], np.zeros((0, 0)), 0.0), ParallelRunReport(trace, [])
    eng = Engine(nd, nt, eff, candidates=cands, device=opts.device, world_size=opts.world_size,
                 rank=opts.rank, nccl_id=opts.nccl_id, export_factor=opts.export_factor,
                 near_tie_tau=opts.near_tie_tau)
    try:
        if reader is None:
            eng.load_k(np.ascontiguousarray(k_raw, dtype=np.float64))
        else:
            # true block columns (i, j): exact reference semantics (kaccess.hpp:27-35)
            col = np.empty((nd, nt, nt))
            for p, j in enumerate(sorted(cands)):
                if p % opts.world_size != opts.rank:
                    continue  # panel owned by another rank
                for i in range(nd):
                    reader.read_block(i, j, col[i])
                eng.load_block_col(j, col)
        for _ in range(eff):
            info = eng.step()
            if info["chosen_index"] < 0:
                trace.warning = "no feasible candidates remain; returning partial selection"
                break
        rows = eng.trace()
        chosen = [r["chosen_index"] for r in rows if r["chosen_index"] >= 0]
        factor = eng.export_factor(len(chosen)) if opts.export_factor else None
    finally:
        eng.close()
    out_rows, rounds = [], []
    noise_acc = 0.0
    for r in rows:
        if r["chosen_index"] < 0:
            continue
        s = r["chosen_index"]
        gain, obj = r["gain"], r["objective"]
        if opts.mode == "normalized":
            noise_acc += opts.noise_logdets[s]
            gain = gain - opts.noise_logdets[s]
            obj = obj - noise_acc
        out_rows.append(TraceRow(k=r["k"], chosen_index=s, objective=obj, gain=gain,
                                 n_evaluated=r["n_evaluated"], n_infeasible=r["n_infeasible"],
                                 wall_ms=r["ms_round"],
                                 mean_candidate_ms=r["ms_round"] / max(r["n_evaluated"], 1),
                                 runner_up=r["runner_up"], runner_up_gain=r["runner_up_gain"],
                                 near_tie=bool(r["near_tie"])))
        rounds.append(RoundResult(d_max=r["gain"], s_star=s, bytes_exchanged=r["bytes_exchanged"],
                                  ms={key: r[key] for key in ("ms_gain", "ms_exchange", "ms_panel",
                                                              "ms_update", "ms_round")}))
    trace.rows = out_rows
    objective = rows[len(out_rows) - 1]["objective"] if out_rows else 0.0
    return SelectionState(chosen, factor, objective), ParallelRunReport(trace, rounds)
