/*
 * dsel.h -- C ABI of the B200-native greedy D-optimal selection engine.
 *
 * Drop-in boundary for the reference `doptsel` selection path
 * (/root/reference/proj/include/doptsel). Plain C: pointers, sizes and
 * status codes, no exceptions, no torch types. Every entry point lists the
 * reference interface it replaces.
 *
 *   reference (C++ templates, CPU threads)         this ABI (sm_100a, NCCL)
 *   ---------------------------------------------  -------------------------------
 *   run_parallel_greedy<Real,A>  parallel.hpp:281   dsel_create + dsel_step* (one
 *   greedy_select<Real,A>        selector.hpp:181     engine per GPU/rank)
 *   KAccess::read_block          kaccess.hpp:18-23  dsel_load_block_row /
 *   KStoreReader::read_block     kstore.hpp:141       dsel_load_block_col
 *   SyntheticKAccess             kaccess.hpp:81     dsel_synthetic_v + dsel_gen_synthetic
 *   score_candidate (all s)      selector.hpp:105   dsel_peek_gains
 *   reduce_argmax / tie rule     parallel.hpp:61,   inside dsel_step (device top-2,
 *                                selector.hpp:132     allgather, identical fold)
 *   SelectionState::factor       selector.hpp:31    dsel_export_factor
 *   TraceRow / RoundResult       selector.hpp:40,   dsel_step_info
 *                                parallel.hpp:30
 *   doptsel::Error family        errors.hpp:10-86   dsel_status + dsel_last_error
 *
 * The C++ wrapper include/doptsel_gpu.hpp maps these back onto the
 * reference types and exceptions.
 */
#ifndef DSEL_H_
#define DSEL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSEL_ABI_VERSION 2

typedef enum {
  DSEL_OK = 0,
  DSEL_E_INVALID = 1,    /* InvalidConfig / DimensionMismatch (errors.hpp) */
  DSEL_E_RANGE = 2,      /* IndexOutOfRange */
  DSEL_E_INFEASIBLE = 3, /* InfeasibleRound: round 1 had no feasible candidate */
  DSEL_E_CUDA = 4,       /* device failure -> WorkerFailure */
  DSEL_E_NCCL = 5,       /* collective failure -> WorkerFailure */
  DSEL_E_OOM = 6,        /* device/pinned allocation failed in dsel_create */
  DSEL_E_IO = 7,         /* IoError / CorruptFile */
  DSEL_E_STATE = 8,      /* call out of order (e.g. step after the budget) */
  DSEL_E_CORRUPT = 9     /* CorruptFile: KBF header/size invalid (kstore.hpp:92-125) */
} dsel_status;

typedef enum { DSEL_STORAGE_AUTO = 0, DSEL_STORAGE_HBM = 1, DSEL_STORAGE_STREAM = 2 } dsel_storage;

typedef struct dsel_engine dsel_engine;

typedef struct {
  int n_sensors;          /* KAccess::n_sensors() */
  int n_steps;            /* KAccess::n_steps() = Nt */
  int budget;             /* B (>= 0) */
  int n_candidates;       /* 0 = all sensors 0..n_sensors-1 */
  const int* candidates;  /* borrowed during dsel_create only; duplicates -> E_INVALID */
  int device;             /* CUDA device of this engine */
  int world_size;         /* ranks sharing the candidate set (1 = single GPU) */
  int rank;               /* 0..world_size-1 */
  const void* nccl_id;    /* 128-byte ncclUniqueId (dsel_nccl_unique_id) when world_size > 1 */
  int storage;            /* dsel_storage: HBM = K resident on the devices; STREAM = K stays in
                             host memory (pinned store, the caller's attached buffer or a KBF
                             file) and each round copies the blocks it reads (left-looking,
                             algorithm 1); AUTO = HBM when the plan fits hbm_budget, else
                             STREAM (see dsel_get_plan) */
  int keep_pristine;      /* keep a device copy of K so dsel_reset can rerun */
  int export_factor;      /* keep per-step W rows so dsel_export_factor can rebuild L_S */
  double near_tie_tau;    /* near-tie flag threshold (default 1e-9 when 0) */
  int full_square;        /* 0 (default): update only the block-lower triangle of the
                             symmetric C (half the flops); 1: full square C[:,J] update.
                             Odd n_steps always use the full square. */
  int algorithm;          /* 0 (default): right-looking Schur update of the resident
                             conditional covariance (the north-star kernel);
                             1: left-looking W-resident variant:
                             K stays pristine, W_all = K[:,S] L_S^{-T} is kept, one
                             column c = K[:,k] - W_all W_all[k]^T per round. */
  /* ---- ABI 2 ---- */
  int panel_layout;       /* symmetric storage only: 0 (default) packed block-lower panels
                             (each panel keeps the rows from its diagonal block down: half
                             the HBM of the full square); 1 full-height panels */
  uint64_t hbm_budget;    /* AUTO storage: device bytes the engine may use; 0 = the device's
                             free memory at create minus 2 GiB */
  int defer_connect;      /* world_size > 1: 1 = dsel_create only allocates; the caller
                             checks that every rank created its engine, then calls
                             dsel_connect (NCCL init + NVLink peer mappings). 0 = create
                             connects (a rank that fails to create leaves its peers
                             blocked in ncclCommInitRank). */
} dsel_config;

/* What dsel_create decided (AUTO resolved) and what it holds. */
typedef struct {
  int storage;            /* DSEL_STORAGE_HBM or DSEL_STORAGE_STREAM */
  int algorithm;          /* 0 right-looking, 1 left-looking */
  int symmetric;          /* block-lower (half-flop) update */
  int packed;             /* packed block-lower panel store */
  uint64_t device_bytes;  /* allocated on the device at create */
  uint64_t planned_bytes; /* the create-time estimate AUTO compared with the budget */
  uint64_t budget_bytes;  /* the budget it was compared with */
  uint64_t host_store_bytes; /* pinned host store (STREAM) once K is loaded */
} dsel_plan;

/* One selection round; field names follow TraceRow (selector.hpp:40-49) and
 * RoundResult (parallel.hpp:30-35). Times are device milliseconds measured
 * with CUDA events on this rank's compute stream (filled by dsel_get_trace
 * after dsel_sync; dsel_step leaves them 0). */
typedef struct {
  int k;                  /* 1-based round */
  int chosen_index;       /* sensor id; -1 if no feasible candidate remained */
  double gain;            /* raw d_max = log det(M_s*) */
  double objective;       /* running log det(K_S) */
  int runner_up;          /* sensor id of the second best, -1 if none */
  double runner_up_gain;
  int near_tie;           /* (g1-g2)/max(|g1|,1) < tau */
  int n_evaluated;
  int n_infeasible;
  uint64_t bytes_exchanged; /* argmax allgather + panel broadcast bytes */
  double ms_gain;         /* gain kernel + local argmax */
  double ms_exchange;     /* allgather + D2H of the 32-byte records */
  double ms_panel;        /* panel broadcast + chol(C_kk) + L^{-1} + W */
  double ms_update;       /* rank-nt Schur update (+ factor history) */
  double ms_round;        /* whole round on the device */
  double update_flops;    /* algorithmic flops of this rank's update: 2*nt*rows*cols */
  double ms_io;           /* ABI 2: H2D of the round's streamed K blocks (copy stream;
                             storage = STREAM, else 0) -- timing.csv io_ms */
} dsel_step_info;

/* Per-rank argmax record exchanged each round (32 bytes, allgathered): the
 * local best and runner-up under the reference order (larger gain wins, exact
 * ties to the lower sensor index, selector.hpp:132-134); s = -1 when empty. */
typedef struct {
  double g1, g2;
  int s1, s2;
  int n_eval, n_inf;
} dsel_argrec;

/* ---- lifecycle ---------------------------------------------------------- */
int dsel_abi_version(void);
dsel_status dsel_nccl_unique_id(void* out128);
dsel_status dsel_create(const dsel_config* cfg, dsel_engine** out);
void dsel_destroy(dsel_engine* e);
const char* dsel_last_error(const dsel_engine* e); /* NULL engine -> last create error */
dsel_status dsel_sync(dsel_engine* e);
/* Collective half of create for defer_connect engines (no-op otherwise). */
dsel_status dsel_connect(dsel_engine* e);
/* Peer failure (WorkerFailure, parallel.hpp:469-475): callable from any
 * thread while this engine's own thread is blocked in dsel_step. Aborts the
 * NCCL communicator and releases the NVLink flag waits; the blocked call
 * and every later step return DSEL_E_NCCL. The engine must still be
 * destroyed. */
dsel_status dsel_abort(dsel_engine* e);
/* bytes of device memory the engine holds */
uint64_t dsel_device_bytes(const dsel_engine* e);
dsel_status dsel_get_plan(const dsel_engine* e, dsel_plan* out);
/* Device/pinned allocations (cudaMalloc, cudaMallocHost, cudaHostRegister)
 * made by the library since load, all engines: the zero-allocation contract
 * of candidate evaluation (test_selector.cpp:281-298) is that
 * dsel_step / dsel_run never move this counter. */
uint64_t dsel_alloc_count(void);
/* Batched log-det of independent SPD matrices already in device memory --
 * the refactorizing baseline's per-candidate potrf (naive_select,
 * selector.hpp:253-357) on this library's gain kernel (batched Cholesky,
 * warp-level pivots, DMMA panel updates). mats: batch column-major m x m
 * matrices, matrix b at mats + b*stride (device pointer, stride >= m*m);
 * logdet[b] (device) = 2 sum log diag L, -inf when a pivot is <= 0 or not
 * finite (status[b] = that pivot, -1 = positive definite). m <= 2800.
 * Synchronous; allocates its scratch (not a selection-round entry point). */
dsel_status dsel_batched_logdet(int device, const double* mats, int m, int64_t stride, int batch,
                                double* logdet, int* status);
/* Roofline denominator: the FP64 tensor-core (DMMA.8x8x4) issue rate of the
 * device, measured with a compute-only microbenchmark (~15 ms). */
dsel_status dsel_measure_fp64_peak(int device, double* tflops);

/* ---- panel store ingest (north-star (1)) -------------------------------- */
/* Block row j of K: blocks (j, i), i = 0..n_sensors-1, each row-major Nt x Nt
 * (exactly KBF payload rows, kstore.hpp:22-35). Uses K(i,j) = K(j,i)^T, exact
 * for symmetric K (SyntheticKAccess, assemble_k). No-op if j is not a
 * candidate owned by this rank. Host memory may be pageable or pinned. */
dsel_status dsel_load_block_row(dsel_engine* e, int j, const double* host_row);
/* Block column j: blocks (i, j), i = 0..n_sensors-1, each row-major, stacked
 * (what read_test_column reads, kaccess.hpp:27-35). Under symmetric storage
 * (the default for even n_steps) only the blocks (i, j) with position(i) >=
 * position(j) are kept and the rest of C is taken from them by symmetry, so
 * K must be symmetric (as every reference KAccess is); full_square = 1 keeps
 * every block and is exact for any K. */
dsel_status dsel_load_block_col(dsel_engine* e, int j, const double* host_col);
/* Whole K in DataSpaceHessian / KBF payload order (n_sensors^2 blocks,
 * block-row-major, hessian.hpp:17-84): loads every owned panel. */
dsel_status dsel_load_k(dsel_engine* e, const double* host_k);
/* Streaming store (storage = DSEL_STORAGE_STREAM) without a copy: the caller's
 * whole K (dsel_load_k layout) stays in host memory and the engine reads, per
 * round, only the blocks (i, k) of the chosen k for its own candidates i plus
 * the diagonal blocks once -- what the reference reads through KAccess
 * read_test_column / read_block (kaccess.hpp:27-35, selector.hpp:200-214).
 * Pinned memory (cudaHostAlloc / registered) is used in place; pageable memory
 * is registered read-only until dsel_destroy or the next load/attach. The
 * buffer must outlive the selection. */
dsel_status dsel_attach_host_k(dsel_engine* e, const double* host_k);
/* Same over this rank's block rows only: the dsel_load_block_row rows of the
 * candidates this rank owns (candidate positions p with p % world_size == rank),
 * stacked in candidate order -- the per-rank shard of the KBF payload. */
dsel_status dsel_attach_host_rows(dsel_engine* e, const double* host_rows);
/* K = sigma^2 I + V V^T formed on the device for scales where V (n x rank)
 * cannot be materialized on the host. V[i][r] ~ N(0,1) from
 * a counter-based Philox4x32-10 stream keyed by (seed, global row, r/2) with
 * Box-Muller -- NOT the reference RNG stream, so the K differs from
 * SyntheticKAccess; it is identical for every world_size. Accumulated by the
 * Schur update kernel (W = +V, 512 rank columns per launch; block-lower tiles
 * only under symmetric storage). HBM store only; n_steps even. */
dsel_status dsel_gen_synthetic_device(dsel_engine* e, int rank, double sigma, uint64_t seed);
/* ---- K formation from an LTI wave problem (assemble_k, hessian.hpp:91-144) ----
 * K = Gamma_noise + F W Gamma_prior W F^T assembled on the GPU, bit-identical to
 * the reference (sequential non-FMA sums in its loop order, exact block
 * symmetrization). Tables are row-major: impulse[s][j][tau] (lti.hpp:82-87),
 * spatial[i][j] (materialized prior, lti.hpp:245-251), mask[j][t] (or NULL),
 * cost_weights[s] (or NULL). */
typedef struct dsel_lti {
  int n_params, n_sensors, n_steps;
  double noise_sigma;
  const double* impulse;
  const double* spatial;
  const double* mask;
  const double* cost_weights;
} dsel_lti;
/* Parse a reference problem config (config.hpp:17-164) and build its wave
 * problem (make_wave_problem, lti.hpp:163-176) on the host. Arrays in *out are
 * owned by *owner; release with dsel_lti_free. DSEL_E_INVALID / DSEL_E_IO. */
dsel_status dsel_lti_from_config(const char* path, dsel_lti* out, void** owner);
void dsel_lti_free(void* owner);
/* Assemble this rank's panels of K from the problem (HBM store; resets the
 * selection). noise_logdets (n_sensors, may be NULL) receives n_steps *
 * log(w_c gamma^2) per sensor (noise_block_logdets, hessian.hpp:149-154). */
dsel_status dsel_assemble_lti(dsel_engine* e, const dsel_lti* problem, double* noise_logdets);
/* KBF store (`doptsel select <kbf>`, KStoreReader, kstore.hpp:22-186): validates
 * the header and size like KStoreReader (E_CORRUPT / E_IO) and loads this
 * rank's panels with parallel pread into pinned buffers, overlapped with the
 * H2D. exact_columns=1 reads true block columns (blocks (i,j), what the
 * reference reads); 0 reads contiguous block rows and relies on symmetry
 * (write_kbf guarantees |K - K^T| <= 1e-10). threads = pread threads (0 = auto). */
dsel_status dsel_load_kbf(dsel_engine* e, const char* path, int exact_columns, int threads);
/* File-backed streaming store (storage = DSEL_STORAGE_STREAM): the KBF file is
 * validated like KStoreReader (E_CORRUPT / E_IO) and kept open; each round
 * reads only the chosen column's true blocks (s_q, s_k) of this rank's
 * candidates -- what read_test_column reads through KStoreReader::read_block
 * (kaccess.hpp:27-35, kstore.hpp:141-158) -- with `threads` parallel preads
 * into a pinned buffer while the round's column GEMM runs, then H2D on the copy
 * stream. K is never held whole in host or device memory (beyond the page
 * cache). threads = 0: auto. */
dsel_status dsel_attach_kbf(dsel_engine* e, const char* path, int threads);
/* Export block row j (same layout as dsel_load_block_row) of the CURRENT
 * conditional covariance (= K before the first step); owner rank only. */
dsel_status dsel_read_block_row(dsel_engine* e, int j, double* host_row);

/* ---- synthetic K (SyntheticKAccess, kaccess.hpp:81-124) ----------------- */
/* Host: V = (n_sensors*Nt) x rank, row-major, N(0,1) from the reference RNG
 * stream (rng.hpp:15-50: mt19937_64 + Box-Muller). Bit-identical to
 * SyntheticKAccess's v_. `threads` parallelises the transform (0 = auto). */
dsel_status dsel_synthetic_v(int n_sensors, int n_steps, int rank, uint64_t seed, double* out,
                             int threads);
/* Device: generate this rank's panels of K = sigma^2 I + V V^T bit-exactly
 * (sequential non-FMA dot products). V_host as produced above. */
dsel_status dsel_gen_synthetic(dsel_engine* e, const double* v_host, int rank, double sigma);

/* The fold every rank applies to the allgathered records (reduce_argmax,
 * parallel.hpp:61-74, extended to the global top-2). Pure host function;
 * associative and order-independent. out->s1 = -1 when all are infeasible. */
void dsel_fold_records(const dsel_argrec* recs, int n, dsel_argrec* out);

/* ---- selection (north-star (2)-(4)) ------------------------------------- */
/* One round: gains of all remaining candidates, cross-rank argmax, panel
 * broadcast from the owner, W = C[:,k] L_k^{-T}, C -= W W^T. Collective over
 * the ranks. Returns DSEL_E_INFEASIBLE when round 1 has no feasible
 * candidate; later all-infeasible rounds return DSEL_OK with
 * chosen_index = -1 (partial selection, parallel.hpp:416-421). */
dsel_status dsel_step(dsel_engine* e, dsel_step_info* info);
/* Same, but the winner is forced to `sensor` (replay along a given sequence);
 * the gain reported is that sensor's. */
dsel_status dsel_step_forced(dsel_engine* e, int sensor, dsel_step_info* info);
/* Run rounds until the budget (or infeasibility). n_done <- rounds done. */
dsel_status dsel_run(dsel_engine* e, int* n_done);
/* Raw gains of all currently remaining candidates OWNED by this rank,
 * written to gains[sensor] (other entries untouched); -inf = infeasible. */
dsel_status dsel_peek_gains(dsel_engine* e, double* gains_by_sensor);
/* Rounds so far with device timings (syncs). Returns the row count. */
int dsel_get_trace(dsel_engine* e, dsel_step_info* rows, int max_rows);
/* Restore C = K and clear the selection (requires keep_pristine). */
dsel_status dsel_reset(dsel_engine* e);
/* Run statistics since create/reset (syncs). time_to_k_ms: device time from
 * the first gain launch of round 1 to the D2H of the last round's winner
 * (CUDA events on the compute stream, host gaps included). update_ms: sum of
 * the Schur-update kernel spans; update_flops: their algorithmic flops
 * (2*nt*rows*cols, full-square update). */
typedef struct {
  int rounds;
  uint64_t kernel_launches;
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint64_t nccl_bytes;
  double time_to_k_ms;
  double update_ms;
  double update_flops;
  double io_ms;           /* storage=stream: H2D time of the streamed K columns */
  double io_exposed_ms;   /* part of io_ms not hidden behind the GEMM */
} dsel_stats;
dsel_status dsel_get_stats(dsel_engine* e, dsel_stats* st);
/* L_S (SelectionState::factor): row-major, (k*Nt) x (k*Nt) active window with
 * row stride `ld` (>= k*Nt), k = rounds done. Collective: every rank gets the
 * full factor. Requires export_factor. */
dsel_status dsel_export_factor(dsel_engine* e, double* host, int64_t ld);
/* Block row i (0-based) of L_S alone: n_steps x (i+1)*n_steps, row-major,
 * row stride ld -- what append_block_column adds in round i+1
 * (linalg.hpp:159-178). Collective like dsel_export_factor; lets a per-round
 * hook rebuild the factor incrementally. */
dsel_status dsel_export_factor_row(dsel_engine* e, int i, double* host, int64_t ld);

#ifdef __cplusplus
}
#endif
#endif /* DSEL_H_ */
