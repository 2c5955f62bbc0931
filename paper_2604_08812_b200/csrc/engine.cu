// engine.cu -- per-GPU selection engine behind the C ABI (include/dsel.h).
//
// One engine per GPU (one process or thread per GPU). Candidates are owned
// cyclically by position (p % world_size); every rank holds all candidate
// rows of its candidates' block columns of the conditional covariance C.
// Per round (north star (2)-(4)):
//   gain kernel (batched chol + logdet) -> local top-2 argmax
//   -> ncclAllGather(32 B/rank) -> identical host fold (reference tie rule)
//   -> ncclBroadcast of the chosen conditional panel C[:,k] from its owner
//   -> chol(C_kk), L_k^{-1}, W = C[live,k] L_k^{-T}  (DMMA)
//   -> C[live, local live] -= W W^T                  (DMMA)
// The reference computes the same gains left-looking per candidate
// (selector.hpp:86-116); this is the right-looking Schur form of Alg. 1
// with the conditional covariance kept resident.
#include <cuda_runtime.h>
#include <nccl.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cerrno>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "dsel.h"
#include "kernels.cuh"
#include "lti.h"

using namespace dsel;

namespace {

thread_local std::string g_create_err;

struct Fail {
  dsel_status st;
  std::string msg;
};

#define CU(x)                                                                          \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess)                                                             \
      throw Fail{DSEL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)};        \
  } while (0)
#define NC(x)                                                                          \
  do {                                                                                 \
    ncclResult_t _r = (x);                                                             \
    if (_r != ncclSuccess)                                                             \
      throw Fail{DSEL_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(_r)};        \
  } while (0)

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Every device / pinned allocation of the library goes through these three
// (counted): the zero-allocation contract of candidate evaluation
// (test_selector.cpp:281-298) is asserted on dsel_alloc_count().
std::atomic<uint64_t> g_allocs{0};
template <class T>
cudaError_t ds_malloc(T** p, size_t bytes) {
  g_allocs.fetch_add(1, std::memory_order_relaxed);
  return cudaMalloc(reinterpret_cast<void**>(p), bytes);
}
template <class T>
cudaError_t ds_malloc_host(T** p, size_t bytes) {
  g_allocs.fetch_add(1, std::memory_order_relaxed);
  return cudaMallocHost(reinterpret_cast<void**>(p), bytes);
}
template <class T>
cudaError_t ds_host_alloc_mapped(T** p, size_t bytes) {
  g_allocs.fetch_add(1, std::memory_order_relaxed);
  return cudaHostAlloc(reinterpret_cast<void**>(p), bytes, cudaHostAllocMapped);
}
cudaError_t ds_host_register(void* p, size_t bytes, unsigned flags) {
  g_allocs.fetch_add(1, std::memory_order_relaxed);
  return cudaHostRegister(p, bytes, flags);
}
constexpr int kWsGroupDefault = 16;  // column tiles per update rasterization group

// scratch device allocation released on every exit path (including throws)
template <class T>
struct DevScratch {
  T* p = nullptr;
  explicit DevScratch(size_t count) {
    if (ds_malloc(&p, sizeof(T) * (count ? count : 1)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw Fail{DSEL_E_OOM, "cudaMalloc of scratch (" + std::to_string(count * sizeof(T)) + " bytes) failed"};
    }
  }
  ~DevScratch() {
    if (p) cudaFree(p);
  }
  DevScratch(const DevScratch&) = delete;
  DevScratch& operator=(const DevScratch&) = delete;
};
// NVTX ranges (header-only nvtx3): one per C-ABI call that does device work and
// one per phase of a round, so a timeline shows the host side of every round
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  void next(const char* name) {
    nvtxRangePop();
    nvtxRangePushA(name);
  }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

// DEBUG probes (DSEL_PROBE=1): GPU events + host times at named points of a round
struct Probe {
  bool on = getenv("DSEL_PROBE") != nullptr;
  cudaEvent_t ev[16];
  double host[16];
  const char* name[16];
  int n = 0;
  bool init = false;
  void mark(const char* nm, cudaStream_t st) {
    if (!on || n >= 16) return;
    if (!init) {
      for (auto& x : ev) cudaEventCreate(&x);
      init = true;
    }
    cudaEventRecord(ev[n], st);
    host[n] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    name[n++] = nm;
  }
  void dump(int rank) {
    if (!on || n < 2) { n = 0; return; }
    cudaEventSynchronize(ev[n - 1]);
    if (rank == 0) {
      fprintf(stderr, "[probe]");
      for (int i = 1; i < n; ++i) {
        float ms = 0;
        cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
        fprintf(stderr, " %s:%.0f/%.0f", name[i], ms * 1e3, host[i] - host[i - 1]);
      }
      fprintf(stderr, "\n");
    }
    n = 0;
  }
};
Probe g_probe;

template <class T>
T* dmalloc(size_t count, uint64_t& total) {
  void* p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = ds_malloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Fail{DSEL_E_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed"};
  }
  total += count * sizeof(T);
  return static_cast<T*>(p);
}

constexpr int kEv = 10;  // 0-4 phases; 5,6 streamed H2D start/end (copy stream); 7 GEMM end;
                        // 8,9 look-ahead bulk start/end (bulk stream)

}  // namespace

struct dsel_engine {
  // ---- configuration ----
  int nd = 0, nt = 0, budget = 0, G = 1, rank = 0, dev = 0;
  int nc = 0;          // candidates
  long long n = 0;     // nc * nt
  int nloc = 0;        // local slots
  int ldw = 0;         // W / Linv pitch
  int eff_budget = 0;
  int n_sms = 148;
  int mpad = 0;  // rows of the tiled W buffers
  bool ll = false;  // left-looking W-resident algorithm
  // storage = STREAM (left-looking): K lives in pinned host memory only,
  // hstore[position][own slot][nt][nt] = K(own_q, k); per round the chosen
  // k's blocks are copied into Kk on the copy stream, overlapped with the GEMM
  bool stream = false;
  double *hstore = nullptr, *Kk = nullptr;
  // world_size 1: the host store keeps only the block-lower half of K --
  // hstore panel p = blocks K(q, p) for q >= p, row-major, back to back; a
  // round reads panel p contiguously plus block (p, q) of every earlier panel
  // q (K(q, p) transposed). Half the host memory, so K up to twice the host
  // RAM it would otherwise need (a K larger than HBM fits a 1-GPU host)
  bool hpacked = false;
  // file-backed store (dsel_attach_kbf): per round the chosen column's own
  // blocks are pread from the KBF file into a pinned staging buffer while the
  // column GEMM runs, then copied H2D (KStoreReader::read_block, kstore.hpp:141-158)
  int kbf_fd = -1;
  std::string kbf_path;
  int kbf_threads = 0;
  double* h_kstage = nullptr;
  // dsel_attach_host_k: the caller's block-row-major K in (pinned) host
  // memory is the store; blocks are read in place, only those a round needs
  const double* hk_user = nullptr;
  bool hk_rows = false;  // hk_user holds only this rank's block rows (slot order)
  void* hk_registered = nullptr;  // cudaHostRegister'ed by the engine (pageable input)
  cudaEvent_t ev_tab = nullptr;
  cudaStream_t ts = nullptr;  // side stream: L_k^-1 concurrent with the panel gather
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // this round's table upload done (orders the column copy after it)
  std::vector<int> streamed_round;  // rounds whose ev[5..7] are valid
  double *Wown = nullptr, *Wkn = nullptr, *D = nullptr, *cbuf = nullptr, *ldiag = nullptr,
         *cpart = nullptr;
  int* d_iota = nullptr;
  int own_mpad = 0, k_mpad = 0;
  long long ldo = 0;
  bool sym = true;  // block-lower-triangle (symmetric) update
  // packed block-lower panel store (symmetric storage): each panel keeps only
  // the rows from its own diagonal block down (PanelGeom), half the HBM of the
  // full square; C = Craw + c_pad (the pad keeps masked reads of rows above a
  // panel's first stored row inside the allocation)
  bool packed = false;
  uint64_t planned = 0, plan_budget = 0;  // create-time plan (dsel_get_plan)
  unsigned char nccl_id[128] = {};
  int* h_abort = nullptr;          // host-mapped peer-failure word (dsel_abort)
  const volatile int* d_abort = nullptr;
  std::atomic<bool> aborted{false};
  double* Craw = nullptr;
  size_t c_elems = 0, c_pad = 0;
  bool full_panels = true;  // both triangles of every panel hold K (gen_synthetic / full-square load)
  int* d_sym = nullptr;  // [first_rt per column tile | group prefix]
  int* h_sym = nullptr;  // pinned
  int sym_tiles = 0;
  // symmetric storage on G > 1: W rows solved by the rank holding each block of
  // C[:,k] (hb = holder-ordered compact blocks, hb_off = per-rank segments),
  // exchanged by grouped broadcasts (all-gather-v) and scattered into Wt/Wnt
  double *Wsend = nullptr, *Wrecv = nullptr;
  int *d_hb = nullptr, *d_hbpos = nullptr, *h_hb = nullptr;
  std::vector<int> hb_off;
  int* d_hboff = nullptr;  // device copy of hb_off (G + 1)
  // NVLink peer memory (symmetric storage, G > 1): peers' Wsend / gain
  // scratch (L_k) / round flags mapped into this process (CUDA IPC across
  // processes, peer access within one), so the W exchange is one kernel that
  // reads the holders' rows over NVLink and scatters them (no NCCL call), and
  // L_k^-1 reads the owner's factor in place
  bool p2p = false;
  unsigned long long* flag = nullptr;  // this rank's published round sequence
  unsigned long long seq = 0;
  std::vector<double*> peer_wsend, peer_lscr, peer_lk;  // peer_wsend: Wsend (right) / Wkn (left)
  std::vector<double*> peer_c;  // the peers' panel shards (symmetric right-looking W solve)
  std::vector<int> h_holder;     // per-round W-row holder of each live block (host scratch)
  std::vector<unsigned long long*> peer_flag;
  std::vector<void*> ipc_opened;
  const double** d_peer_wsend = nullptr;
  unsigned long long** d_peer_flag = nullptr;
  int ws_br = 128;  // tile height of the right-looking update configuration (rl_cfg)
  int ws_cfg = -1;   // DSEL_WS_CFG: -1 auto, 0 Big, 1 Pair, 2 Big4, 3 Big6, 4 BigT, 5 BigR, 6 BigR4, 7 PairR, 8 BigR6
  int rl_cfg = 5;    // configuration of the right-looking update (BigR by default)
  int ws_group = kWsGroupDefault;  // column tiles per rasterization group
  double gen_flops = 0.0;  // last dsel_gen_synthetic_device (K formation on the update kernel)
  bool keep = false, export_factor = false;
  double tau = 1e-9;
  std::vector<int> pos_sensor, sensor_pos, slot_sensor;

  // ---- device state ----
  cudaStream_t s = nullptr;
  ncclComm_t comm = nullptr;
  double *C = nullptr, *K0 = nullptr, *W = nullptr, *Pbuf = nullptr, *Lk = nullptr,
         *Linv = nullptr, *Lscr = nullptr, *Wn = nullptr, *Wt = nullptr, *Wnt = nullptr, *gains = nullptr, *hist = nullptr, *kgain = nullptr,
         *stage = nullptr, *xbuf = nullptr;
  int *status = nullptr, *kstatus = nullptr;
  int *d_pos_sensor = nullptr, *d_slot_sensor = nullptr;
  unsigned* d_counter = nullptr;  // gain-launch ticket for the fused argmax (zero between launches)
  unsigned long long* ws_ctr = nullptr;       // update-kernel claim counters (compute / bulk stream), in d_counter's block
  unsigned long long ws_ctr_base[2] = {0, 0};  // their values at the next launch
  bool ws_dynamic = true;                      // DSEL_WS_DYNAMIC=0: static round-robin tile schedule
  int* d_round = nullptr;  // per-round tables (one block, one upload): d_tab | d_sym | d_hb
  int* h_round = nullptr;  // pinned staging of the same layout
  // look-ahead rounds (symmetric right-looking, Nt a multiple of the tile):
  // round t's bulk update runs on s2 beside round t+1's chain (gains, argmax,
  // W solve), which only needs the diagonal blocks (updated first) and the
  // next chosen row/column (updated once it is known). Tables and W are
  // double-buffered: the bulk of round t reads buffer t%2 while round t+1 fills
  // the other one.
  bool la = false;
  int la_reserve = 8;          // SMs left to the chain while a bulk runs (set per world size at create)
  int prio_least = 0;          // stream priority of the bulk stream
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_wrdy[2] = {nullptr, nullptr}, ev_bulk[2] = {nullptr, nullptr};
  bool bulk_pending[2] = {false, false};
  int* d_round_b[2] = {nullptr, nullptr};
  int* h_round_b[2] = {nullptr, nullptr};
  double *Wt_b[2] = {nullptr, nullptr}, *Wnt_b[2] = {nullptr, nullptr};
  int2 *d_lists = nullptr, *h_lists = nullptr;  // [2][list_cap] tile lists (cross | diagonal)
  size_t list_cap = 0;
  int rbuf = 0;                // buffer of the current round
  bool prev_valid = false;     // the previous round's bulk is still to run
  size_t n_tab_ints = 0, n_sym_ints = 0, n_hb_ints = 0;  // table block layout
  int prev_R = 0, prev_Rl = 0, prev_sym_tiles = 0;
  double prev_bulk_flops = 0.0;  // full block-lower flops of that round minus its diagonal blocks
  unsigned long long seq2 = 0;   // panel-ready flag sequence (flag[1])
  std::vector<char> bulk_round;  // rounds whose ev[8..9] hold a bulk span
  size_t round_ints = 0;
  int* d_tab = nullptr;  // [row_pos nc | col_slot nloc | col_g nloc]
  ArgRec *d_rec = nullptr, *d_recs = nullptr;
  ArgRec* h_recs = nullptr;  // pinned
  int* h_tab = nullptr;      // pinned
  double* h_stage = nullptr;  // pinned bounce buffer for pageable ingest (one block row)
  size_t stage_elems = 0;     // per device staging buffer (two of them)
  int stage_flip = 0;
  cudaStream_t cs = nullptr;  // copy stream (H2D ingest)
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_scat[2] = {nullptr, nullptr};
  uint64_t h2d_bytes = 0, d2h_bytes = 0, nccl_bytes = 0;
  uint64_t launches = 0;  // kernels launched by the selection rounds
  double update_flops = 0.0;
  uint64_t dev_bytes = 0;
  std::vector<cudaEvent_t> ev;  // kEv per round

  // ---- selection state ----
  std::vector<char> alive;     // by position
  int n_alive = 0;
  int n_rows_tab = 0, n_cols_tab = 0;  // sizes of the uploaded tables
  std::vector<int> chosen;
  std::vector<dsel_step_info> trace;
  double objective = 0.0;
  bool finished = false;
  std::string err;

  PanelGeom geom() const {
    PanelGeom g;
    g.base = C;
    g.n = n;
    g.nt = nt;
    g.G = G;
    g.rank = rank;
    g.packed = packed ? 1 : 0;
    return g;
  }
  int* row_pos() { return d_tab; }
  int* col_slot() { return d_tab + nc; }
  int* col_g() { return d_tab + nc + nloc; }
};

namespace {

void pread_exact(int fd, void* dst, size_t bytes, off_t off, const std::string& path) {
  unsigned char* p = static_cast<unsigned char*>(dst);
  size_t done = 0;
  while (done < bytes) {
    const ssize_t got = ::pread(fd, p + done, bytes - done, off + (off_t)done);
    if (got < 0) {
      if (errno == EINTR) continue;
      throw Fail{DSEL_E_IO, path + ": pread failed: " + std::strerror(errno)};
    }
    if (got == 0) throw Fail{DSEL_E_CORRUPT, path + ": unexpected end of file"};
    done += (size_t)got;
  }
}

// Host store geometry (streaming). Full (world_size > 1): hstore[pk][own q] =
// K(own q, k), nc * nloc blocks. Packed (world_size 1): panel pk holds K(q, pk)
// for q >= pk, nc (nc + 1) / 2 blocks.
size_t hstore_blocks(const dsel_engine* e) {
  return e->hpacked ? (size_t)e->nc * (e->nc + 1) / 2 : (size_t)e->nc * std::max(e->nloc, 1);
}
size_t hpanel_off(const dsel_engine* e, int pk) {  // blocks before packed panel pk
  return (size_t)pk * e->nc - (size_t)pk * (pk - 1) / 2;
}
double* hpacked_block(const dsel_engine* e, int pk, int q) {  // K(q, pk), q >= pk, row-major
  return e->hstore + (hpanel_off(e, pk) + (q - pk)) * (size_t)e->nt * e->nt;
}
// the round's K column comes from the packed host store (blocks of earlier
// slots arrive transposed) -- not from the caller's K or a KBF file
bool packed_host_source(const dsel_engine* e) { return e->hpacked && !e->hk_user && e->kbf_fd < 0; }

void detach_kbf(dsel_engine* e) {
  if (e->kbf_fd >= 0) ::close(e->kbf_fd);
  e->kbf_fd = -1;
  e->kbf_path.clear();
  if (e->h_kstage) cudaFreeHost(e->h_kstage);
  e->h_kstage = nullptr;
}

void build_tables(dsel_engine* e, bool upload = true) {
  // compact global live list (ascending position) and local live list
  int* rp = e->h_tab;
  int* cs = e->h_tab + e->nc;
  int* cg = e->h_tab + e->nc + e->nloc;
  int R = 0, Rl = 0;
  for (int p = 0; p < e->nc; ++p) {
    if (!e->alive[p]) continue;
    if (p % e->G == e->rank) {
      cs[Rl] = p / e->G;
      cg[Rl] = R;
      ++Rl;
    }
    rp[R++] = p;
  }
  e->n_rows_tab = R;
  e->n_cols_tab = Rl;
  if (upload)
    CU(cudaMemcpyAsync(e->d_tab, e->h_tab, sizeof(int) * (size_t)(e->nc + 2 * e->nloc),
                       cudaMemcpyHostToDevice, e->s));
}

// point the round tables (and, with look-ahead, the tiled W operands) at buffer b
void set_round_buf(dsel_engine* e, int b) {
  e->rbuf = b;
  e->d_round = e->d_round_b[b];
  e->h_round = e->h_round_b[b];
  e->d_tab = e->d_round;
  e->h_tab = e->h_round;
  e->d_sym = e->h_sym = nullptr;
  if (e->n_sym_ints) {
    e->d_sym = e->d_round + e->n_tab_ints;
    e->h_sym = e->h_round + e->n_tab_ints;
  }
  if (e->n_hb_ints) {
    e->d_hb = e->d_round + e->n_tab_ints + e->n_sym_ints;
    e->h_hb = e->h_round + e->n_tab_ints + e->n_sym_ints;
    e->d_hbpos = e->d_hb + e->nc;
    e->d_hboff = e->d_hb + 2 * (size_t)e->nc;
  }
  if (e->Wt_b[b]) {
    e->Wt = e->Wt_b[b];
    e->Wnt = e->Wnt_b[b];
  }
}

// every per-round table (row/col, tile schedule, holder lists) in one copy
void upload_round(dsel_engine* e) {
  CU(cudaMemcpyAsync(e->d_round, e->h_round, sizeof(int) * e->round_ints, cudaMemcpyHostToDevice, e->s));
}

}  // namespace

// Kernel-side helpers for the gain kernel batch description.
namespace {
__global__ void gain_tables_kernel(const int* col_slot, int n, PanelGeom geom,
                                   const int* pos_sensor, long long* src_off, long long* src_ld,
                                   int* sensor, int diag_store) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int q = col_slot[b];
  const int nt = geom.nt;
  const int p = q * geom.G + geom.rank;
  if (diag_store) {  // left-looking: separate D blocks, ld = nt
    src_off[b] = (long long)q * nt * nt;
    src_ld[b] = nt;
  } else {  // the diagonal block of panel q
    src_off[b] = geom.idx(q, 0, (long long)p * nt);
    src_ld[b] = geom.ld(q);
  }
  sensor[b] = pos_sensor[p];
}

// left-looking: D[q] = diagonal block of this rank's K panel q
__global__ void ll_init_d_kernel(const double* C, long long ldc, int nt, int nloc, int G, int rank,
                                 double* D) {
  const long long n2 = (long long)nt * nt;
  const long long total = n2 * nloc;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / n2);
    const long long w = e - (long long)q * n2;
    const int c = (int)(w / nt), r = (int)(w - (long long)c * nt);
    const int p = q * G + rank;
    D[e] = C[(size_t)(q * nt + c) * ldc + (size_t)p * nt + r];
  }
}

// left-looking factor export: block row i = [W_own row block (steps 0..i-1), L_k_i]
__global__ void ll_pack_factor_row_kernel(const double* Wown, int own_mpad, int row0, int nt, int ldw,
                                          int i_blocks, const double* ldiag_i, double* out) {
  const long long n2 = (long long)nt * nt;
  const long long total = n2 * i_blocks;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n2);
    const long long w = e - (long long)j * n2;
    const int a = (int)(w / nt), b = (int)(w - (long long)a * nt);
    double v;
    if (j + 1 < i_blocks)
      v = Wown[wt_index(row0 + a, j * ldw + b, own_mpad)];
    else
      v = b <= a ? ldiag_i[(size_t)b * nt + a] : 0.0;  // L_k column-major
    out[(size_t)a * i_blocks * nt + (size_t)j * nt + b] = v;
  }
}


// forced winner: record with that sensor's gain (if local & feasible)
__global__ void pick_kernel(const double* gain, const int* status, const int* sensor, int n,
                            int forced, ArgRec* out) {
  if (threadIdx.x != 0) return;
  ArgRec r;
  r.g1 = -INFINITY;
  r.g2 = -INFINITY;
  r.s1 = -1;
  r.s2 = -1;
  r.n_eval = n;
  r.n_inf = 0;
  for (int i = 0; i < n; ++i) {
    if (status[i] >= 0) {
      ++r.n_inf;
      continue;
    }
    if (sensor[i] == forced) {
      r.g1 = gain[i];
      r.s1 = forced;
    }
  }
  *out = r;
}

__global__ void pack_factor_row_kernel(const double* hist_slot, int nt, int i_blocks,
                                       double* out /* nt x (i_blocks*nt) row-major */) {
  const long long n2 = (long long)nt * nt;
  const long long total = n2 * i_blocks;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n2);
    const long long w = e - j * n2;
    const int a = (int)(w / nt), b = (int)(w - (long long)a * nt);
    out[(size_t)a * i_blocks * nt + (size_t)j * nt + b] = hist_slot[e];
  }
}
}  // namespace

namespace {

// scratch tables for the gain kernel batch: [src_off | src_ld | sensor]
struct GainTabs {
  long long* src_off;
  long long* src_ld;
  int* sensor;
};

// panel width of the gain kernel: two NB x mp panels must fit in 227 KB
int chol_nb(int nt) { return nt <= 436 ? 32 : 8; }
constexpr int kBatchedLogdetMaxDim = 2800;  // NB = 8 panel + pivots within 227 KB

// smem pitch of the gain kernel panels: >= nt rounded to 8, == 4 or 12 mod 16
// so the DMMA fragment loads are bank-conflict free
int chol_mp(int nt) {
  int mp = round_up(nt, 8);
  if (mp % 16 == 0 || mp % 16 == 8) mp += 4;
  return mp;
}

// staged gain kernels (one 12-warp CTA per candidate, chunked L stream) when the
// batch fits one wave: 2 (default) the look-ahead version, 1 the plain staged
// one, DSEL_CHOL_STAGE=0 chol_logdet_kernel -- all three give the same bits
int g_chol_stage = 2;
size_t g_chol_stage_max = 0;  // dynamic smem the staged kernel may use (opt-in - static)

void launch_chol(const CholArgs& a, int n_batch, cudaStream_t s, int n_sms) {
  const int nb = chol_nb(a.nt);
  const size_t smem = ((size_t)nb * a.mp + a.nt) * sizeof(double);
  // more candidates than SMs: squeeze two CTAs per SM (capped registers) so the
  // batch runs in one wave; otherwise one uncapped CTA per candidate
  const bool two = n_batch > n_sms;
  if (a.nt >= 32 && a.nt <= 128 && !getenv("DSEL_CHOL_PANELS")) {  // triangle-resident variant
    const size_t ts = tri_smem_bytes(a.nt);
    if (two)
      chol_logdet_tri_kernel<2><<<n_batch, 256, ts, s>>>(a);
    else
      chol_logdet_tri_kernel<1><<<n_batch, 256, ts, s>>>(a);
  } else if (nb == 32 && !two && g_chol_stage > 0 && cst::smem_bytes(a.nt, a.mp) <= g_chol_stage_max) {
    if (g_chol_stage == 2 && a.nt <= cla::MAX_NT)
      chol_logdet_la_kernel<<<n_batch, cla::NW * 32, cst::smem_bytes(a.nt, a.mp), s>>>(a);
    else
      chol_logdet_stage_kernel<12><<<n_batch, 384, cst::smem_bytes(a.nt, a.mp), s>>>(a);
  } else if (nb == 32) {
    if (two)
      chol_logdet_kernel<32, 2><<<n_batch, 256, smem, s>>>(a);
    else
      chol_logdet_kernel<32, 1><<<n_batch, 256, smem, s>>>(a);
  } else {
    chol_logdet_kernel<8, 1><<<n_batch, 256, smem, s>>>(a);
  }
}

GainTabs gain_tabs(dsel_engine* e) {
  long long* base = reinterpret_cast<long long*>(e->xbuf);  // 3*(nloc+1) doubles
  return {base, base + e->nloc + 1, reinterpret_cast<int*>(base + 2 * (e->nloc + 1))};
}

void run_gain(dsel_engine* e, const int* slots, int n_batch, ArgRec* rec = nullptr) {
  if (n_batch <= 0) return;
  GainTabs t = gain_tabs(e);
  gain_tables_kernel<<<(n_batch + 127) / 128, 128, 0, e->s>>>(
      slots, n_batch, e->geom(), e->d_pos_sensor, t.src_off, t.src_ld, t.sensor, e->ll ? 1 : 0);
  CU(cudaGetLastError());
  CholArgs a{};
  a.src = e->ll ? e->D : e->C;
  a.src_off = t.src_off;
  a.src_ld = t.src_ld;
  a.L = e->Lscr;
  a.l_stride = (long long)e->nt * e->nt;
  a.gain = e->gains;
  a.status = e->status;
  a.nt = e->nt;
  a.n = n_batch;
  a.mp = chol_mp(e->nt);
  a.sensor = t.sensor;
  a.rec = rec;  // fused local argmax (the last block of the launch)
  a.counter = e->d_counter;
  launch_chol(a, n_batch, e->s, e->n_sms);
  CU(cudaGetLastError());
  e->launches += 2;
}


template <class K>
void allow_smem(K kernel, int optin) {
  cudaFuncAttributes fa{};
  CU(cudaFuncGetAttributes(&fa, kernel));
  CU(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          optin - (int)fa.sharedSizeBytes));
}

void set_smem_limits(int dev) {
  // per device context; cheap, called from dsel_create on the engine's device
  int optin = 0;
  CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  allow_smem(chol_logdet_kernel<32, 1>, optin);
  allow_smem(chol_logdet_kernel<32, 2>, optin);
  allow_smem(chol_logdet_kernel<8, 1>, optin);
  {
    cudaFuncAttributes fa{}, fb{};
    CU(cudaFuncGetAttributes(&fa, chol_logdet_stage_kernel<12>));
    CU(cudaFuncGetAttributes(&fb, chol_logdet_la_kernel));
    g_chol_stage_max = (size_t)optin - std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
    allow_smem(chol_logdet_stage_kernel<12>, optin);
    allow_smem(chol_logdet_la_kernel, optin);
    const char* cs = getenv("DSEL_CHOL_STAGE");
    g_chol_stage = cs ? std::max(0, std::min(2, atoi(cs))) : 2;
  }
  allow_smem(chol_logdet_tri_kernel<1>, optin);
  allow_smem(chol_logdet_tri_kernel<2>, optin);
  allow_smem(schur_update_kernel<2>, optin);
  allow_smem(schur_update_kernel<1>, optin);
  allow_smem(panel_w_kernel<2>, optin);
  allow_smem(panel_w_kernel<1>, optin);
  allow_smem(schur_update_ws_kernel<ws::Big>, optin);
  allow_smem(schur_update_ws_kernel<ws::Pair>, optin);
  allow_smem(schur_update_ws_kernel<ws::Big4>, optin);
  allow_smem(schur_update_ws_kernel<ws::Big6>, optin);
  allow_smem(schur_update_ws_kernel<ws::BigT>, optin);
  allow_smem(schur_update_ws_kernel<ws::BigR>, optin);
  allow_smem(schur_update_ws_kernel<ws::BigR4>, optin);
  allow_smem(schur_update_ws_kernel<ws::PairR>, optin);
  allow_smem(schur_update_ws_kernel<ws::BigR6>, optin);
  CU(cudaFuncSetAttribute(schur_update_ws_kernel<ws::Pair>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          (int)cudaSharedmemCarveoutMaxShared));
  CU(cudaFuncSetAttribute(schur_update_ws_kernel<ws::PairR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          (int)cudaSharedmemCarveoutMaxShared));
  allow_smem(ll_gemm_kernel, optin);
  allow_smem(trinv_smem_kernel<4>, optin);
  allow_smem(trinv_smem_kernel<8>, optin);
  allow_smem(trinv_smem_kernel<14>, optin);
}


// Wave balancing for a persistent launch over n_tiles equal tiles of n_k
// k-chunks: the first n_full tiles run whole, the rest are split into s
// k-ranges. Picks (n_full, s) minimising the modelled time: waves of whole
// tiles + the split tail + the partial-plane round trip (write + reduce).
void ws_balance(int n_tiles, int n_k, int sms, int max_s, int br, int& n_full, int& split_s) {
  n_full = n_tiles;
  split_s = 1;
  if (max_s <= 1 || n_tiles <= 0 || n_k < 2) return;
  const double t_chunk = 1.1e-6 * br / 128, t_tile0 = 2.0e-6;  // per k-chunk / per tile (s)
  const double t_plane = (double)br * ws::BC * 8 * 2 / 6.0e12;    // partial write + read
  const double t_full = n_k * t_chunk + t_tile0;
  double best = ((n_tiles + sms - 1) / sms) * t_full;
  for (int f = 0; f * sms < n_tiles; ++f) {
    const int rem = n_tiles - f * sms;
    for (int sp = 2; sp <= std::min(max_s, n_k); ++sp) {
      const int units = rem * sp;
      const double t = f * t_full + ((units + sms - 1) / sms) * ((double)n_k / sp * t_chunk + t_tile0) +
                       (double)units * t_plane + 4e-6;
      if (t < best * 0.98) {
        best = t;
        n_full = f * sms;
        split_s = sp;
      }
    }
  }
}

// Map the peers' exchange buffer (Wsend: symmetric right-looking; Wkn:
// left-looking), gain scratch, round flag and L_k buffer (NVLink peer memory).
// All ranks take the same decision (min-reduced): the per-round collective
// sequence depends on it. DSEL_P2P=0 keeps the NCCL exchange.
constexpr int kPeerBufs = 5;  // 0 exchange, 1 Lscr, 2 flag, 3 Lk, 4 C (panels)
struct PeerInfo {
  cudaIpcMemHandle_t h[kPeerBufs];
  void* p[kPeerBufs];
  long long pid;
  int dev;
  int ok;
};

void setup_p2p(dsel_engine* e) {
  const int G = e->G;
  CU(ds_malloc(&e->flag, 256));
  CU(cudaMemset(e->flag, 0, 256));
  // buffer 4 (the panel shard) is absent with a streaming store: not mapped
  void* bufs[kPeerBufs] = {e->Wsend ? (void*)e->Wsend : (void*)e->Wkn, e->Lscr, e->flag, e->Lk, e->Craw};
  PeerInfo mine{};
  mine.pid = (long long)getpid();
  mine.dev = e->dev;
  const char* env = getenv("DSEL_P2P");
  mine.ok = !(env && atoi(env) == 0) && bufs[0] != nullptr;
  for (int b = 0; b < kPeerBufs && mine.ok; ++b) {
    mine.p[b] = bufs[b];
    if (b == 4 && !bufs[b]) continue;
    mine.ok = cudaIpcGetMemHandle(&mine.h[b], bufs[b]) == cudaSuccess;
  }
  cudaGetLastError();
  DevScratch<PeerInfo> info_buf(G + 1);
  PeerInfo* d_info = info_buf.p;
  CU(cudaMemcpy(d_info + G, &mine, sizeof(PeerInfo), cudaMemcpyHostToDevice));
  NC(ncclAllGather(d_info + G, d_info, sizeof(PeerInfo), ncclUint8, e->comm, e->s));
  std::vector<PeerInfo> all(G);
  CU(cudaMemcpyAsync(all.data(), d_info, sizeof(PeerInfo) * G, cudaMemcpyDeviceToHost, e->s));
  CU(cudaStreamSynchronize(e->s));
  int ok = 1;
  for (const auto& x : all) ok &= x.ok;
  std::vector<std::vector<void*>> peer(kPeerBufs, std::vector<void*>(G, nullptr));
  for (int r = 0; r < G && ok; ++r) {
    if (r == e->rank) {
      for (int b = 0; b < kPeerBufs; ++b) peer[b][r] = bufs[b];
      continue;
    }
    if (all[r].pid == mine.pid) {  // same process (thread per GPU): peer access
      int can = 0;
      cudaDeviceCanAccessPeer(&can, e->dev, all[r].dev);
      const cudaError_t pe = can ? cudaDeviceEnablePeerAccess(all[r].dev, 0) : cudaErrorPeerAccessUnsupported;
      cudaGetLastError();
      if (!can || (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)) {
        ok = 0;
        break;
      }
      for (int b = 0; b < kPeerBufs; ++b) peer[b][r] = all[r].p[b];
    } else {  // another process: CUDA IPC
      for (int b = 0; b < kPeerBufs && ok; ++b) {
        void* m = nullptr;
        if (!all[r].p[b]) continue;  // not exported (streaming store)
        if (cudaIpcOpenMemHandle(&m, all[r].h[b], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
          e->ipc_opened.push_back(m);
          peer[b][r] = m;
        } else {
          ok = 0;
        }
      }
      cudaGetLastError();
    }
  }
  DevScratch<int> ok_buf(1);  // every rank must agree
  int* d_ok = ok_buf.p;
  CU(cudaMemcpy(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice));
  NC(ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, e->comm, e->s));
  CU(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, e->s));
  CU(cudaStreamSynchronize(e->s));
  e->p2p = ok != 0;
  if (!e->p2p) {
    for (void* ptr : e->ipc_opened) cudaIpcCloseMemHandle(ptr);
    e->ipc_opened.clear();
    return;
  }
  e->peer_wsend.assign(G, nullptr);
  e->peer_lscr.assign(G, nullptr);
  e->peer_flag.assign(G, nullptr);
  e->peer_lk.assign(G, nullptr);
  e->peer_c.assign(G, nullptr);
  for (int r = 0; r < G; ++r) {
    e->peer_wsend[r] = static_cast<double*>(peer[0][r]);
    e->peer_lscr[r] = static_cast<double*>(peer[1][r]);
    e->peer_flag[r] = static_cast<unsigned long long*>(peer[2][r]);
    e->peer_lk[r] = static_cast<double*>(peer[3][r]);
    e->peer_c[r] = peer[4][r] ? static_cast<double*>(peer[4][r]) + e->c_pad : nullptr;
  }
  CU(ds_malloc(&e->d_peer_wsend, sizeof(double*) * G));
  CU(ds_malloc(&e->d_peer_flag, sizeof(unsigned long long*) * G));
  CU(cudaMemcpy(e->d_peer_wsend, e->peer_wsend.data(), sizeof(double*) * G, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(e->d_peer_flag, e->peer_flag.data(), sizeof(unsigned long long*) * G,
                cudaMemcpyHostToDevice));
}

// Launch the persistent update kernel in the engine's configuration (grid =
// resident CTAs, capped by the number of work units).
// Configuration for a launch: 3 chunks x 2 stages (Big4) pays fewer stage
// hand-offs on long k loops, 2 x 3 (Big) keeps the producer further ahead on
// short ones (Nt = 128 right-looking); 64-row tiles (Pair) when the r-side row
// count pads badly to 128 (left-looking r-side = Nt rows: 420 -> 82 % of 4 x
// 128 tiles, 94 % of 7 x 64). -1 = auto.
int cfg_br(int cfg) { return cfg == 1 || cfg == 7 ? 64 : cfg == 3 ? 192 : 128; }  // 0,2,4,5,6: 128
int ws_pick(const dsel_engine* e, int r_rows, int n_k, bool fixed_rows);
// K formation on the update kernel: its tile schedule uses ws_br, so the tile
// height must match the right-looking configuration's
int gen_cfg(const dsel_engine* e, int n_k) {
  return e->ws_br == 192 ? 3 : e->ws_br == 64 ? 1 : (n_k >= 16 ? 2 : 0);
}

int ws_pick(const dsel_engine* e, int r_rows, int n_k, bool fixed_rows) {
  // Big6 (192-row tiles) only for the right-looking update: the left-looking
  // r-side (W_k, Nt rows) is padded for 128-row tiles
  if (e->ws_cfg >= 0 && !(fixed_rows && e->ws_cfg >= 3)) return e->ws_cfg;
  if (fixed_rows) {
    const double u128 = (double)r_rows / (((r_rows + 127) / 128) * 128);
    const double u64 = (double)r_rows / (((r_rows + 63) / 64) * 64);
    if (u64 > u128 + 0.05) return 1;
  }
  return n_k >= 16 ? 2 : 0;
}

// sms: SMs the persistent grid may occupy (0 = all; the look-ahead bulk leaves
// some to the next round's chain); st: stream (null = the compute stream)
void launch_ws(dsel_engine* e, UpdateWSArgs& ua, int cfg, int sms = 0, cudaStream_t st = nullptr) {
  ua.br = cfg_br(cfg);
  const long long units = (long long)ua.n_full + (long long)(ua.n_tiles - ua.n_full) * ua.split_s;
  if (units <= 0) return;
  if (!st) st = e->s;
  if (sms <= 0) sms = e->n_sms;
  // dynamic schedule: one claim counter per stream (launches on a stream run
  // one after another); every launch advances it by units + grid claims
  const int ci = st == e->s2 ? 1 : 0;
  const int grid_ws = (int)std::min<long long>(((cfg == 1 || cfg == 7) ? 2LL : 1LL) * sms, units);
  ua.ctr = e->ws_dynamic ? e->ws_ctr + ci : nullptr;
  ua.ctr_base = e->ws_ctr_base[ci];
  if (e->ws_dynamic) e->ws_ctr_base[ci] += (unsigned long long)units + (unsigned long long)grid_ws;
  if (cfg == 1) {
    const int grid = (int)std::min<long long>(2LL * sms, units);
    schur_update_ws_kernel<ws::Pair><<<grid, ws::Pair::THREADS, ws::Pair::SMEM, st>>>(ua);
  } else if (cfg == 2) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::Big4><<<grid, ws::Big4::THREADS, ws::Big4::SMEM, st>>>(ua);
  } else if (cfg == 3) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::Big6><<<grid, ws::Big6::THREADS, ws::Big6::SMEM, st>>>(ua);
  } else if (cfg == 4) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::BigT><<<grid, ws::BigT::THREADS, ws::BigT::SMEM, st>>>(ua);
  } else if (cfg == 5) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::BigR><<<grid, ws::BigR::THREADS, ws::BigR::SMEM, st>>>(ua);
  } else if (cfg == 6) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::BigR4><<<grid, ws::BigR4::THREADS, ws::BigR4::SMEM, st>>>(ua);
  } else if (cfg == 8) {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::BigR6><<<grid, ws::BigR6::THREADS, ws::BigR6::SMEM, st>>>(ua);
  } else if (cfg == 7) {
    const int grid = (int)std::min<long long>(2LL * sms, units);
    schur_update_ws_kernel<ws::PairR><<<grid, ws::PairR::THREADS, ws::PairR::SMEM, st>>>(ua);
  } else {
    const int grid = (int)std::min<long long>(sms, units);
    schur_update_ws_kernel<ws::Big><<<grid, ws::Big::THREADS, ws::Big::SMEM, st>>>(ua);
  }
  CU(cudaGetLastError());
}

// Block-lower tile schedule of the update (symmetric storage): first needed row
// tile per column tile and the tile-id prefix per 16-column-tile group.
void sym_tables(dsel_engine* e, bool upload = true) {
  const int nt = e->nt, R = e->n_rows_tab, Rl = e->n_cols_tab;
  const int* cg = e->h_tab + e->nc + e->nloc;
  const int n_rows = R * nt, n_cols = Rl * nt;
  const int br = e->ws_br;
  const int nrt = (n_rows + br - 1) / br, nct = (n_cols + ws::BC - 1) / ws::BC;
  const int ng = (nct + e->ws_group - 1) / e->ws_group;
  int* fr = e->h_sym;
  int* gp = e->h_sym + nct;
  for (int ct = 0; ct < nct; ++ct) {
    const int h = (ct * ws::BC) / nt;
    fr[ct] = (cg[h] * nt) / br;
  }
  gp[0] = 0;
  for (int g = 0; g < ng; ++g) {
    const int ct0 = g * e->ws_group, gw = std::min(e->ws_group, nct - ct0);
    gp[g + 1] = gp[g] + (nrt - fr[ct0]) * gw;
  }
  e->sym_tiles = gp[ng];
  if (upload)
    CU(cudaMemcpyAsync(e->d_sym, e->h_sym, sizeof(int) * (size_t)(nct + ng + 1),
                       cudaMemcpyHostToDevice, e->s));
}

// left-looking split-K: one split per 64 k-chunks (1024 k), at most 8 splits;
// depends only on the round, never on the rank count
constexpr int kLLSplitChunks = 64, kLLMaxSplits = 8;

void finish_row(dsel_engine* e, dsel_step_info& row, int s1, int s2, double g1, double g2,
                uint64_t bytes, double flops, dsel_step_info* info) {
  e->chosen.push_back(s1);
  e->objective += g1;
  row.chosen_index = s1;
  row.gain = g1;
  row.objective = e->objective;
  row.runner_up = s2;
  row.runner_up_gain = g2;
  row.near_tie = (s2 >= 0 && (g1 - g2) / std::max(std::fabs(g1), 1.0) < e->tau) ? 1 : 0;
  row.bytes_exchanged = bytes;
  row.update_flops = flops;
  e->nccl_bytes += bytes;
  e->trace.push_back(row);
  if (info) *info = row;
}

void launch_trinv(dsel_engine* e, const double* Lk, cudaStream_t st = nullptr) {
  if (!st) st = e->s;
  const int nt = e->nt, tb = 256 / 32;
  const unsigned g = (unsigned)((e->ldw + tb - 1) / tb);
  if (nt <= TRINV_SMEM_MAX_NT) {
    const size_t sm = ((size_t)2 * 32 * nt + nt) * sizeof(double);
    if (e->ldw <= 128)
      trinv_smem_kernel<4><<<g, 256, sm, st>>>(Lk, nt, e->Linv, e->ldw);
    else if (e->ldw <= 256)
      trinv_smem_kernel<8><<<g, 256, sm, st>>>(Lk, nt, e->Linv, e->ldw);
    else
      trinv_smem_kernel<14><<<g, 256, sm, st>>>(Lk, nt, e->Linv, e->ldw);
  } else {
    const size_t sm = (size_t)nt * sizeof(double);
    if (e->ldw <= 512)
      trinv_kernel<16><<<g, 256, sm, st>>>(Lk, nt, e->Linv, e->ldw);
    else
      trinv_kernel<32><<<g, 256, sm, st>>>(Lk, nt, e->Linv, e->ldw);
  }
  CU(cudaGetLastError());
  e->launches += 1;
}

// L_k^-1 on the side stream, overlapping the panel gather / table upload; the
// compute stream joins before the W solve.
void launch_trinv_async(dsel_engine* e, const double* Lk) {
  CU(cudaEventRecord(e->ev_fork, e->s));
  CU(cudaStreamWaitEvent(e->ts, e->ev_fork, 0));
  launch_trinv(e, Lk, e->ts);
  CU(cudaEventRecord(e->ev_join, e->ts));
}

// Block (own slot qq, sensor col) of the caller-attached host K.
const double* user_block(const dsel_engine* e, int qq, int col) {
  const size_t n2 = (size_t)e->nt * e->nt;
  const size_t r = e->hk_rows ? (size_t)qq : (size_t)e->slot_sensor[qq];
  return e->hk_user + (r * e->nd + col) * n2;
}

// nloc host blocks src(qq) -> dst[qq] (nt x nt each): one strided 2-D copy
// when the sources are evenly spaced (cyclic ownership), else one per block.
template <class Src>
void h2d_blocks(dsel_engine* e, double* dst, Src src, cudaStream_t st) {
  const size_t n2b = sizeof(double) * e->nt * e->nt;
  if (e->nloc == 0) return;
  const char* b0 = reinterpret_cast<const char*>(src(0));
  const long long d = e->nloc > 1 ? reinterpret_cast<const char*>(src(1)) - b0 : (long long)n2b;
  bool even = d >= (long long)n2b && d < (1ll << 31);  // 2-D copy pitch limit
  for (int qq = 2; qq < e->nloc && even; ++qq)
    even = reinterpret_cast<const char*>(src(qq)) - b0 == (long long)qq * d;
  if (even) {
    CU(cudaMemcpy2DAsync(dst, n2b, b0, (size_t)d, n2b, e->nloc, cudaMemcpyHostToDevice, st));
  } else {
    for (int qq = 0; qq < e->nloc; ++qq)
      CU(cudaMemcpyAsync(dst + (size_t)qq * e->nt * e->nt, src(qq), n2b, cudaMemcpyHostToDevice, st));
  }
}

// Own blocks (row slot q, column sensor kcol(q)) of the KBF file into the pinned
// staging buffer, Kstage[q] = block (rowsens(q), kcol(q)) row-major: parallel
// pread (KStoreReader::read_block, kstore.hpp:141-158), one block per call.
template <class RowS, class ColS>
void kbf_read_blocks(dsel_engine* e, RowS rowsens, ColS colsens) {
  const size_t bsz = sizeof(double) * e->nt * e->nt;
  const int threads = std::max(1, std::min(e->kbf_threads, e->nloc));
  std::vector<std::thread> pool;
  std::vector<std::string> errs(threads);
  std::vector<int> codes(threads, 0);
  for (int w = 0; w < threads; ++w)
    pool.emplace_back([&, w] {
      try {
        for (int qq = w; qq < e->nloc; qq += threads)
          pread_exact(e->kbf_fd, reinterpret_cast<unsigned char*>(e->h_kstage) + (size_t)qq * bsz, bsz,
                      (off_t)(32 + ((size_t)rowsens(qq) * e->nd + colsens(qq)) * bsz), e->kbf_path);
      } catch (const Fail& f) {
        codes[w] = f.st;
        errs[w] = f.msg;
      }
    });
  for (auto& t : pool) t.join();
  for (int w = 0; w < threads; ++w)
    if (codes[w]) throw Fail{(dsel_status)codes[w], errs[w]};
}

// The chosen column's blocks K(own q, k) for this round (north star (1)) into
// Kk on the copy stream, ordered after this round's table upload (which would
// otherwise queue behind it on the copy engine). Called after the column GEMM
// is launched, so a file read on this thread overlaps the GEMM.
void stream_column(dsel_engine* e, int p, int round, cudaEvent_t* ev) {
  const size_t n2 = (size_t)e->nt * e->nt;
  const int ks = e->pos_sensor[p];
  CU(cudaStreamWaitEvent(e->cs, e->ev_tab, 0));
  if (e->kbf_fd >= 0) {
    // every own slot's true block (s_q, s_k), exactly what read_test_column
    // reads (kaccess.hpp:27-35); the copy stream then moves it H2D
    kbf_read_blocks(e, [&](int qq) { return e->slot_sensor[qq]; }, [&](int) { return ks; });
    CU(cudaEventRecord(ev[5], e->cs));
    CU(cudaMemcpyAsync(e->Kk, e->h_kstage, sizeof(double) * (size_t)e->nloc * n2, cudaMemcpyHostToDevice, e->cs));
  } else if (e->hk_user) {
    // blocks (s_q, s_k) of the caller's K: one strided copy when the own
    // slots are evenly spaced sensors (cyclic ownership of all sensors)
    CU(cudaEventRecord(ev[5], e->cs));
    h2d_blocks(e, e->Kk, [&](int qq) { return user_block(e, qq, ks); }, e->cs);
  } else if (packed_host_source(e)) {
    // panel p (blocks q >= p) in one copy; K(q, p) of the live earlier q is
    // block (p, q) of panel q, copied as stored (ll_addk reads it transposed)
    CU(cudaEventRecord(ev[5], e->cs));
    CU(cudaMemcpyAsync(e->Kk + (size_t)p * n2, hpacked_block(e, p, p), sizeof(double) * n2 * (e->nc - p),
                       cudaMemcpyHostToDevice, e->cs));
    for (int q = 0; q < p; ++q)
      if (e->alive[q])
        CU(cudaMemcpyAsync(e->Kk + (size_t)q * n2, hpacked_block(e, q, p), sizeof(double) * n2,
                           cudaMemcpyHostToDevice, e->cs));
  } else {
    CU(cudaEventRecord(ev[5], e->cs));
    CU(cudaMemcpyAsync(e->Kk, e->hstore + (size_t)p * e->nloc * n2, sizeof(double) * (size_t)e->nloc * n2,
                       cudaMemcpyHostToDevice, e->cs));
  }
  CU(cudaEventRecord(ev[6], e->cs));
  e->streamed_round.push_back(round);
  e->h2d_bytes += (uint64_t)e->nloc * n2 * sizeof(double);
}

// Left-looking round tail: W_k + L_k from the owner, then this rank's rows of
// the new conditional column, W_t, and the D (gain input) downdate.
void ll_tail(dsel_engine* e, int round, bool last, int p, int owner, int q, const double* Lk,
             cudaEvent_t* ev, uint64_t bytes, dsel_step_info& row, double g1, double g2, int s1,
             int s2, dsel_step_info* info) {
  const int nt = e->nt;
  const long long n2 = (long long)nt * nt;
  const int kcols = round * e->ldw;  // W_all columns so far
  if (owner == e->rank) {
    CU(cudaMemcpyAsync(e->ldiag + (size_t)round * n2, Lk, sizeof(double) * n2,
                       cudaMemcpyDeviceToDevice, e->s));
    if (!last && e->G > 1 && Lk != e->Lk)
      CU(cudaMemcpyAsync(e->Lk, Lk, sizeof(double) * n2, cudaMemcpyDeviceToDevice, e->s));
    if (!last && kcols > 0) {
      const long long total = (long long)nt * kcols;
      ll_extract_wk_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 16), 256, 0,
                             e->s>>>(e->Wown, e->own_mpad, q * nt, nt, kcols, e->Wkn, e->k_mpad);
      CU(cudaGetLastError());
      e->launches += 1;
    }
  }
  if (!last && e->G > 1 && e->p2p) {
    // the owner publishes -W_k and L_k (its Wkn / Lk, rewritten only when it
    // owns a later round -- after every peer has passed the next argmax
    // all-gather, i.e. finished these copies); peers wait on its flag and pull
    // them over NVLink with the copy engines
    ++e->seq;
    if (owner == e->rank) {
      p2p_signal_kernel<<<1, 32, 0, e->s>>>(e->flag, e->seq);
      CU(cudaGetLastError());
    } else {
      p2p_wait_kernel<<<1, 32, 0, e->s>>>(e->peer_flag[owner], e->seq, e->d_abort);
      CU(cudaGetLastError());
      if (kcols > 0)
        CU(cudaMemcpyAsync(e->Wkn, e->peer_wsend[owner], sizeof(double) * (size_t)kcols * e->k_mpad,
                           cudaMemcpyDefault, e->s));
      CU(cudaMemcpyAsync(e->Lk, e->peer_lk[owner], sizeof(double) * (size_t)n2, cudaMemcpyDefault, e->s));
      bytes += (uint64_t)((size_t)kcols * e->k_mpad + n2) * sizeof(double);
    }
    e->launches += 1;
    Lk = e->Lk;
  } else if (!last && e->G > 1) {
    NC(ncclGroupStart());
    if (kcols > 0)
      NC(ncclBroadcast(e->Wkn, e->Wkn, (size_t)kcols * e->k_mpad, ncclDouble, owner, e->comm, e->s));
    NC(ncclBroadcast(e->Lk, e->Lk, (size_t)n2, ncclDouble, owner, e->comm, e->s));
    NC(ncclGroupEnd());
    bytes += (uint64_t)((size_t)kcols * e->k_mpad + n2) * sizeof(double) * (uint64_t)(e->G - 1);
    Lk = e->Lk;
  }
  e->alive[p] = 0;
  e->n_alive -= 1;
  build_tables(e);
  if (e->stream) CU(cudaEventRecord(e->ev_tab, e->s));
  const int Rl = e->n_cols_tab;
  double flops = 0.0;
  if (!last) launch_trinv(e, Lk);
  CU(cudaEventRecord(ev[3], e->s));
  // the streamed column is copied after the column GEMM is launched (below):
  // a file-backed store reads it from disk on this thread while the GEMM runs
  const bool streamed = e->stream && !last && e->nloc > 0 && Rl > 0;
  if (!last && Rl > 0) {
    const int n_rows = Rl * nt;
    if (nt % 2 == 0) {
      // the warp-specialized TMA update kernel, re-targeted: r-side = W_k
      // (c' rows), c-side = this rank's live rows of W_own, accumulators
      // start from K(own, k) (the pristine panels), output to cbuf
      UpdateWSArgs ua{};
      ua.C = e->stream ? nullptr : e->C;  // streaming: accumulate from 0, K added below
      ua.geom = e->geom();
      ua.Wt = e->Wkn;
      ua.Wnt = e->Wown;
      ua.mpad = e->k_mpad;
      ua.n_k = kcols / 16;
      ua.row_pos = nullptr;          // single "block": p_k -> rows p_k*nt + c'
      ua.row_pos_k = p;
      ua.col_slot = e->col_slot();
      ua.col_g = e->col_slot();      // c-side W rows are slot*nt + off
      ua.nt = nt;
      ua.n_rows = nt;
      ua.n_cols = n_rows;
      const int cfg = ws_pick(e, nt, ua.n_k, true);
      const int br = cfg == 1 ? 64 : 128;
      ua.n_row_tiles = (nt + br - 1) / br;
      ua.n_col_tiles = (n_rows + ws::BC - 1) / ws::BC;
      ua.group = e->ws_group;
      ua.sym = 0;
      ua.n_tiles = ua.n_row_tiles * ua.n_col_tiles;
      ua.cout = e->cbuf;
      ua.ldo = e->ldo;
      ua.mpad_c = e->own_mpad;
      // wave balancing: the tiles past the last full wave are split along k
      ws_balance(ua.n_tiles, ua.n_k, e->n_sms * (br == 64 ? 2 : 1), e->cpart ? kLLMaxSplits : 1, br,
                 ua.n_full, ua.split_s);
      ua.part = e->cpart;
      ua.part_stride = (long long)e->ldo * nt;
      launch_ws(e, ua, cfg);
      if (ua.split_s > 1) {
        const long long total = (long long)(ua.n_tiles - ua.n_full) * br * ws::BC;
        ws_split_reduce_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0,
                                 e->s>>>(ua);
        CU(cudaGetLastError());
        e->launches += 1;
      }
      if (streamed) {
        stream_column(e, p, round, ev);
        const long long total = (long long)nt * n_rows;
        CU(cudaEventRecord(ev[7], e->s));
        CU(cudaStreamWaitEvent(e->s, ev[6], 0));
        ll_addk_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, e->s>>>(
            nullptr, 0, 1, e->Kk, e->col_slot(), nt, n_rows, e->ldo, e->cbuf, packed_host_source(e) ? p : -1);
        CU(cudaGetLastError());
        e->launches += 1;
      }
    } else {
      LLGemmArgs ga;
      ga.Wown = e->Wown;
      ga.own_mpad = e->own_mpad;
      ga.Wkn = e->Wkn;
      ga.k_mpad = e->k_mpad;
      ga.n_k = kcols / 16;
      ga.Kp = e->stream ? nullptr : e->C;  // streaming: K added after the GEMM
      ga.ldk = e->n;
      ga.pk = p;
      ga.row_slot = e->col_slot();
      ga.nt = nt;
      ga.n_rows = n_rows;
      ga.cout = e->cbuf;
      ga.ldo = e->ldo;
      ga.kc_split = kLLSplitChunks;
      ga.n_splits = std::max(1, std::min(kLLMaxSplits, (ga.n_k + kLLSplitChunks - 1) / kLLSplitChunks));
      ga.kc_split = std::max(ga.kc_split, (ga.n_k + ga.n_splits - 1) / ga.n_splits);
      ga.part = e->cpart;
      ga.part_stride = e->ldo * nt;
      dim3 gg((n_rows + llg::BM - 1) / llg::BM, (nt + llg::BN - 1) / llg::BN, ga.n_splits);
      ll_gemm_kernel<<<gg, llg::THREADS, llg::SMEM, e->s>>>(ga);
      CU(cudaGetLastError());
      if (streamed) {
        stream_column(e, p, round, ev);
        const long long total = (long long)nt * n_rows;
        CU(cudaEventRecord(ev[7], e->s));
        CU(cudaStreamWaitEvent(e->s, ev[6], 0));
        ll_addk_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, e->s>>>(
            e->cpart, ga.part_stride, ga.n_splits, e->Kk, e->col_slot(), nt, n_rows, e->ldo, e->cbuf,
            packed_host_source(e) ? p : -1);
        CU(cudaGetLastError());
        e->launches += 1;
      } else if (ga.n_splits > 1) {
        const long long total = (long long)nt * n_rows;
        ll_reduce_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, e->s>>>(
            e->cpart, ga.part_stride, ga.n_splits, nt, n_rows, e->ldo, e->cbuf);
        CU(cudaGetLastError());
        e->launches += 1;
      }
    }
    PanelArgs pa{};
    pa.P = e->cbuf;
    pa.ldp = e->ldo;
    pa.Linv = e->Linv;
    pa.ldl = e->ldw;
    pa.ldw = e->ldw;
    pa.row_pos = e->d_iota;
    pa.nt = nt;
    pa.n_rows = n_rows;
    pa.Wown = e->Wown;
    pa.out_slot = e->col_slot();
    pa.own_mpad = e->own_mpad;
    pa.koff = kcols;
    pa.G = e->G;
    pa.rank = e->rank;
    dim3 grid((n_rows + pw::BR - 1) / pw::BR, (nt + pw::BN - 1) / pw::BN);
    if (nt % 2 == 0)
      panel_w_kernel<2><<<grid, pw::THREADS, pw::SMEM, e->s>>>(pa);
    else
      panel_w_kernel<1><<<grid, pw::THREADS, pw::SMEM, e->s>>>(pa);
    CU(cudaGetLastError());
    LLDArgs da;
    da.D = e->D;
    da.Wown = e->Wown;
    da.own_mpad = e->own_mpad;
    da.koff = kcols;
    da.ldw = e->ldw;
    da.row_slot = e->col_slot();
    da.nt = nt;
    da.n_tiles_1d = (nt + 63) / 64;
    dim3 dg(da.n_tiles_1d * da.n_tiles_1d, Rl);
    ll_dupdate_kernel<<<dg, 256, 0, e->s>>>(da);
    CU(cudaGetLastError());
    e->launches += 3;
    // algorithmic: new column (2 R nt^2 t nt) + W_t (R nt nt^2) + D downdate (2 R nt^3)
    flops = 2.0 * n_rows * nt * ((double)round * nt) + (double)n_rows * nt * nt +
            2.0 * Rl * (double)nt * nt * nt;
    e->update_flops += flops;
  }
  CU(cudaEventRecord(ev[4], e->s));
  finish_row(e, row, s1, s2, g1, g2, bytes, flops, info);
}

// Left-looking gain input before round 1: D[q] = K(own q, own q), from the
// resident panels or the streaming store (step 1 and gain peeks before it).
void ll_init_d(dsel_engine* e) {
  const int nt = e->nt;
  if (e->stream && e->nloc > 0 && !e->hstore && !e->hk_user && e->kbf_fd < 0)
    throw Fail{DSEL_E_STATE, "no K loaded (streaming store)"};
  if (e->stream && e->nloc > 0) {
    // D[q] = K(own_q, own_q)^T = K(own_q, own_q) (symmetric), from the host store;
    // store block is row-major, D is column-major: equal for a symmetric block
    if (e->kbf_fd >= 0) {  // diagonal blocks (s_q, s_q) from the file
      kbf_read_blocks(e, [&](int qq) { return e->slot_sensor[qq]; }, [&](int qq) { return e->slot_sensor[qq]; });
      CU(cudaMemcpyAsync(e->D, e->h_kstage, sizeof(double) * (size_t)e->nloc * nt * nt, cudaMemcpyHostToDevice,
                         e->s));
    } else {
      h2d_blocks(e, e->D, [&](int qq) {
        return e->hk_user  ? user_block(e, qq, e->slot_sensor[qq])
               : packed_host_source(e) ? hpacked_block(e, qq, qq)
                            : e->hstore + ((size_t)(qq * e->G + e->rank) * e->nloc + qq) * nt * nt;
      }, e->s);
    }
    e->h2d_bytes += (uint64_t)e->nloc * nt * nt * sizeof(double);
  } else if (e->nloc > 0) {
    const long long total = (long long)e->nloc * nt * nt;
    ll_init_d_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 16), 256, 0, e->s>>>(
        e->C, e->n, nt, e->nloc, e->G, e->rank, e->D);
    CU(cudaGetLastError());
    e->launches += 1;
  }
}

// The right-looking update of the current round tables and W (block-lower
// schedule under symmetric storage).
// look-ahead tile lists per round: the cross list (row strip over own panels
// <= nloc blocks, the owner's column <= nc blocks) first, then the
// diagonal-block list (<= nloc blocks)
size_t la_diag_off(const dsel_engine* e) {
  return (size_t)(e->nt / e->ws_br) * (e->nt / ws::BC) * ((size_t)e->nloc + e->nc) + 2;
}
size_t la_list_cap(const dsel_engine* e) {
  return la_diag_off(e) + (size_t)(e->nt / e->ws_br) * (e->nt / ws::BC) * e->nloc + 2;
}

UpdateWSArgs round_update_args(dsel_engine* e) {
  const int nt = e->nt, n_rows = e->n_rows_tab * nt, n_cols = e->n_cols_tab * nt;
  UpdateWSArgs ua{};
  ua.C = e->C;
  ua.geom = e->geom();
  ua.Wt = e->Wt;
  ua.Wnt = e->Wnt;
  ua.mpad = e->mpad;
  ua.n_k = e->ldw / ws::KC;
  ua.row_pos = e->row_pos();
  ua.col_slot = e->col_slot();
  ua.col_g = e->col_g();
  ua.nt = nt;
  ua.n_rows = n_rows;
  ua.n_cols = n_cols;
  ua.n_row_tiles = (n_rows + e->ws_br - 1) / e->ws_br;
  ua.n_col_tiles = (n_cols + ws::BC - 1) / ws::BC;
  ua.group = e->ws_group;
  ua.sym = e->sym;
  ua.first_rt = e->d_sym;
  ua.gprefix = e->d_sym ? e->d_sym + ua.n_col_tiles : nullptr;
  ua.n_groups = (ua.n_col_tiles + e->ws_group - 1) / e->ws_group;
  ua.n_tiles = e->sym ? e->sym_tiles : ua.n_row_tiles * ua.n_col_tiles;
  ua.n_full = ua.n_tiles;
  ua.split_s = 1;
  return ua;
}

// Look-ahead, once round t's winner (position p) is known: the bulk of round
// t-1 (its block-lower tiles minus the diagonal blocks and the new winner's
// row/column) goes to the bulk stream on all SMs but la_reserve; the winner's
// row block in this rank's panels and, at the owner, its panel below the
// diagonal are updated with W_{t-1} on the compute stream -- round t's W solve
// reads exactly those. Uses the current (round t-1) tables and W buffer.
void la_bulk_and_cross(dsel_engine* e, int p, int q, int owner, int round, cudaEvent_t* ev) {
  const int nt = e->nt, R = e->n_rows_tab, Rl = e->n_cols_tab;
  const int* rp = e->h_tab;
  const int* cs = e->h_tab + e->nc;
  const int* rpe = std::lower_bound(rp, rp + R, p);
  if (rpe == rp + R || *rpe != p) throw Fail{DSEL_E_STATE, "look-ahead: the winner is not a live row"};
  const int gk = (int)(rpe - rp);
  int hk = -1;
  if (owner == e->rank)
    for (int h = 0; h < Rl; ++h)
      if (cs[h] == q) hk = h;
  const int pb = e->rbuf, nb = 1 - pb;
  if (Rl > 0) {  // the bulk of round t-1 (waits for W_{t-1}, recorded after its diagonal blocks)
    CU(cudaStreamWaitEvent(e->s2, e->ev_wrdy[pb], 0));
    CU(cudaEventRecord(ev[8], e->s2));
    UpdateWSArgs ua = round_update_args(e);
    ua.la_mode = 1;
    ua.excl_g = gk;
    ua.excl_h = hk;
    launch_ws(e, ua, e->rl_cfg, e->n_sms - e->la_reserve, e->s2);
    CU(cudaEventRecord(ev[9], e->s2));
    e->bulk_round.push_back((char)1);
    e->launches += 1;
  } else {
    e->bulk_round.push_back((char)0);
  }
  CU(cudaEventRecord(e->ev_bulk[pb], e->s2));
  e->bulk_pending[pb] = true;
  // the winner's row/column: round t-2's bulk (other buffer) has finished with it
  if (e->bulk_pending[nb]) CU(cudaStreamWaitEvent(e->s, e->ev_bulk[nb], 0));
  const int rtpb = nt / e->ws_br, ctpb = nt / ws::BC;
  int2* L = e->h_lists + (size_t)nb * e->list_cap;
  int nl = 0;
  for (int h = 0; h < Rl; ++h) {  // block (k, j) of own panels j above k
    if (cs[h] * e->G + e->rank >= p) continue;
    for (int a = 0; a < rtpb; ++a)
      for (int b = 0; b < ctpb; ++b) L[nl++] = make_int2(gk * rtpb + a, h * ctpb + b);
  }
  if (hk >= 0)  // the owner: panel k below its diagonal block
    for (int g = gk + 1; g < R; ++g)
      for (int a = 0; a < rtpb; ++a)
        for (int b = 0; b < ctpb; ++b) L[nl++] = make_int2(g * rtpb + a, hk * ctpb + b);
  if (nl > 0) {
    int2* dL = e->d_lists + (size_t)nb * e->list_cap;
    CU(cudaMemcpyAsync(dL, L, sizeof(int2) * nl, cudaMemcpyHostToDevice, e->s));
    UpdateWSArgs ua = round_update_args(e);
    ua.sym = 0;
    ua.la_mode = 2;
    ua.tlist = dL;
    ua.n_tiles = ua.n_full = nl;
    launch_ws(e, ua, e->rl_cfg);
    e->launches += 1;
  }
  e->update_flops += e->prev_bulk_flops;  // bulk + cross = round t-1 minus its diagonal blocks
  if (e->G > 1 && e->p2p) {
    // peers read panel k below the diagonal over NVLink in round t's W solve:
    // the owner publishes that its strip is updated (flag word 1)
    ++e->seq2;
    if (owner == e->rank) {
      p2p_signal_kernel<<<1, 32, 0, e->s>>>(e->flag + 1, e->seq2);
      CU(cudaGetLastError());
    }
  }
  (void)round;
}

// Look-ahead: finish the pending round's bulk now (diagonal blocks excluded --
// already done), so C is the full conditional covariance (read_block_row).
void la_flush(dsel_engine* e) {
  if (!e->la || !e->prev_valid) return;
  if (e->n_cols_tab > 0) {
    CU(cudaStreamWaitEvent(e->s2, e->ev_wrdy[e->rbuf], 0));
    UpdateWSArgs ua = round_update_args(e);
    ua.la_mode = 1;
    ua.excl_g = -1;
    ua.excl_h = -1;
    launch_ws(e, ua, e->rl_cfg, 0, e->s2);
    e->update_flops += e->prev_bulk_flops;
  }
  CU(cudaStreamSynchronize(e->s2));
  e->prev_valid = false;
}

void step_impl(dsel_engine* e, int forced, dsel_step_info* info) {
  Nvtx nv_step("dsel_step");
  Nvtx nv("gains");
  if (e->aborted.load()) throw Fail{DSEL_E_NCCL, "aborted: a peer rank failed (dsel_abort)"};
  if (e->finished || (int)e->chosen.size() >= e->eff_budget)
    throw Fail{DSEL_E_STATE, "selection already finished"};
  if (e->G > 1 && !e->comm) throw Fail{DSEL_E_STATE, "world_size > 1: dsel_connect first"};
  CU(cudaSetDevice(e->dev));
  const int round = (int)e->chosen.size();
  const int nt = e->nt;
  cudaEvent_t* ev = &e->ev[(size_t)round * kEv];
  const bool last = round + 1 == e->eff_budget;

  if (e->stream && e->nloc > 0 && !e->hstore && !e->hk_user && e->kbf_fd < 0)
    throw Fail{DSEL_E_STATE, "no K loaded (streaming store)"};
  // ---- gains + local argmax ----
  CU(cudaEventRecord(ev[0], e->s));
  if (e->ll && round == 0) ll_init_d(e);
  const int n_batch = e->n_cols_tab;
  // the local top-2 is folded by the gain launch itself (last block); forced
  // steps and empty batches use the separate pick / argmax kernels
  const bool fused = forced < 0 && n_batch > 0;
  run_gain(e, e->col_slot(), n_batch, fused ? e->d_rec : nullptr);
  GainTabs t = gain_tabs(e);
  if (forced >= 0)
    pick_kernel<<<1, 32, 0, e->s>>>(e->gains, e->status, t.sensor, n_batch, forced, e->d_rec);
  else if (!fused)
    argmax_kernel<<<1, 256, 0, e->s>>>(e->gains, e->status, t.sensor, n_batch, e->d_rec);
  CU(cudaGetLastError());
  if (!fused) e->launches += 1;
  CU(cudaEventRecord(ev[1], e->s));

  // ---- cross-rank argmax: 32 B per rank ----
  nv.next("argmax exchange");
  uint64_t bytes = 0;
  if (e->G > 1) {
    NC(ncclAllGather(e->d_rec, e->d_recs, sizeof(ArgRec), ncclUint8, e->comm, e->s));
    CU(cudaMemcpyAsync(e->h_recs, e->d_recs, sizeof(ArgRec) * e->G, cudaMemcpyDeviceToHost, e->s));
    bytes += sizeof(ArgRec) * (uint64_t)e->G;
  } else {
    CU(cudaMemcpyAsync(e->h_recs, e->d_rec, sizeof(ArgRec), cudaMemcpyDeviceToHost, e->s));
  }
  CU(cudaEventRecord(ev[2], e->s));
  e->d2h_bytes += sizeof(ArgRec) * (uint64_t)e->G;
  CU(cudaStreamSynchronize(e->s));
  if (e->aborted.load()) throw Fail{DSEL_E_NCCL, "aborted: a peer rank failed (dsel_abort)"};
  // fault injection for the peer-failure tests: DSEL_FAULT="round,rank" fails
  // that rank after the round's argmax exchange (its peers then wait on it)
  if (const char* fault = getenv("DSEL_FAULT")) {
    int fr = 0, fk = -1;
    if (std::sscanf(fault, "%d,%d", &fr, &fk) == 2 && fr == round + 1 && fk == e->rank)
      throw Fail{DSEL_E_CUDA, "injected fault (DSEL_FAULT) in round " + std::to_string(fr)};
  }
  // identical fold on every rank (reduce_argmax, parallel.hpp:61-74, top-2)
  dsel_argrec fold{};
  dsel_fold_records(e->h_recs, e->G, &fold);
  const double g1 = fold.g1, g2 = fold.g2;
  const int s1 = fold.s1, s2 = fold.s2, n_eval = fold.n_eval, n_inf = fold.n_inf;
  dsel_step_info row{};
  row.k = round + 1;
  row.n_evaluated = n_eval;
  row.n_infeasible = n_inf;
  if (s1 < 0) {
    if (forced >= 0) throw Fail{DSEL_E_INVALID, "forced sensor is not a feasible remaining candidate"};
    if (round == 0) throw Fail{DSEL_E_INFEASIBLE, "all remaining candidates infeasible in round 1"};
    e->finished = true;
    row.chosen_index = -1;
    row.objective = e->objective;
    for (int i = 2; i < kEv; ++i) CU(cudaEventRecord(ev[i], e->s));
    e->trace.push_back(row);
    if (info) *info = row;
    return;
  }
  const int p = e->sensor_pos[s1];
  const int owner = p % e->G;
  const int q = p / e->G;
  nv.next("panel: L_k^-1, W");

  // ---- panel: broadcast C[:,k] and L_k = chol(C_kk) from the owner ----
  // The owner's gain kernel already factored C_kk (scratch slot bidx); every
  // rank uses those exact bits (broadcast), so no rank refactors.
  double* P = nullptr;
  const double* Lk = e->Lk;
  if (owner == e->rank) {
    int bidx = -1;
    const int* cs = e->h_tab + e->nc;
    for (int h = 0; h < e->n_cols_tab; ++h)
      if (cs[h] == q) bidx = h;
    if (bidx < 0) throw Fail{DSEL_E_STATE, "winner not in the local gain batch"};
    const double* lsrc = e->Lscr + (size_t)bidx * nt * nt;
    if (e->G > 1 && !last)
      CU(cudaMemcpyAsync(e->Lk, lsrc, sizeof(double) * nt * nt, cudaMemcpyDeviceToDevice, e->s));
    else
      Lk = lsrc;
  }
  if (e->ll) {
    ll_tail(e, round, last, p, owner, q, Lk, ev, bytes, row, g1, g2, s1, s2, info);
    return;
  }
  if (!last && !e->sym) {
    P = (owner == e->rank) ? e->C + (size_t)q * nt * e->n : e->Pbuf;
    if (e->G > 1) {
      NC(ncclGroupStart());
      NC(ncclBroadcast(P, P, (size_t)e->n * nt, ncclDouble, owner, e->comm, e->s));
      NC(ncclBroadcast(e->Lk, e->Lk, (size_t)nt * nt, ncclDouble, owner, e->comm, e->s));
      NC(ncclGroupEnd());
      bytes += (uint64_t)(e->n + nt) * nt * sizeof(double) * (uint64_t)(e->G - 1);
    }
  }
  bool crossed = false;  // this round updated the winner's strip (peers wait on the owner's flag)
  if (e->la) {
    crossed = e->prev_valid && !last;
    if (crossed) la_bulk_and_cross(e, p, q, owner, round, ev);
    else e->bulk_round.push_back((char)0);
    e->prev_valid = false;
    set_round_buf(e, 1 - e->rbuf);  // round t's tables and W go to the other buffer
  }
  e->alive[p] = 0;
  e->n_alive -= 1;
  g_probe.mark("pre", e->s);
  build_tables(e, !(e->sym && !last));  // symmetric rounds upload all tables at once below
  const int R = e->n_rows_tab, Rl = e->n_cols_tab;
  g_probe.mark("tables", e->s);
  if (!last && e->sym) {
    // symmetric storage: column k of C assembled from the block-lower panels
    // (own blocks from panel k, the rest transposed from panels i < k), summed
    // across ranks (each block has exactly one nonzero contributor)
    P = e->Pbuf;
    const int* gpos = e->row_pos();
    int n_gather = R;
    if (e->G > 1) {
      // only L_k crosses ranks here; each rank solves W for the blocks of C[:,k]
      // it holds (rows p_i > p_k in panel k at its owner, the rest transposed
      // from panel i at i's owner) and the rows are exchanged after the solve
      if (e->p2p) {
        // L_k^-1 reads the owner's factor in place (its gain kernel finished
        // before its argmax all-gather, which this rank has seen complete)
        if (owner != e->rank) {
          int bidx = 0;
          for (int qq = 0; qq < q; ++qq) bidx += e->alive[(size_t)qq * e->G + owner] ? 1 : 0;
          Lk = e->peer_lscr[owner] + (size_t)bidx * nt * nt;
        }
      } else {
        NC(ncclBroadcast(e->Lk, e->Lk, (size_t)nt * nt, ncclDouble, owner, e->comm, e->s));
        bytes += (uint64_t)nt * nt * sizeof(double) * (uint64_t)(e->G - 1);
        Lk = e->Lk;
      }
      g_probe.mark("lkbc", e->s);
      launch_trinv_async(e, Lk);
      const int* rp = e->h_tab;
      int* hb = e->h_hb;
      int* hbpos = e->h_hb + e->nc;
      // W-row holders: a block above the chosen one is held (transposed) by
      // its own panel's rank; the blocks below it sit in panel k at the owner.
      // With peer memory they are dealt round-robin to every rank, each
      // reading its share of panel k over NVLink inside the W solve, so the
      // solve and the serving of W rows are balanced (not ~half on the owner)
      e->hb_off.assign(e->G + 1, 0);
      std::vector<int>& hrank = e->h_holder;
      hrank.resize(R);
      for (int h = 0, j = 0; h < R; ++h) {
        const int pos = rp[h];
        hrank[h] = pos < p ? pos % e->G : (e->p2p ? (j++ % e->G) : owner);
      }
      int m = 0;
      for (int r = 0; r < e->G; ++r) {
        e->hb_off[r] = m;
        for (int h = 0; h < R; ++h) {
          if (hrank[h] == r) {
            hb[m] = h;
            hbpos[m] = rp[h];
            ++m;
          }
        }
      }
      e->hb_off[e->G] = m;
      std::copy(e->hb_off.begin(), e->hb_off.end(), e->h_hb + 2 * (size_t)e->nc);
      gpos = e->d_hbpos + e->hb_off[e->rank];
      n_gather = e->hb_off[e->rank + 1] - e->hb_off[e->rank];
      g_probe.mark("holders", e->s);
    } else {
      launch_trinv_async(e, Lk);
    }
    sym_tables(e, false);
    upload_round(e);
    {
      // blocks below the chosen one (position > p, in panel k at its owner)
      // are read in place by the W solve: only the transposed ones above it
      // are gathered -- a prefix of the position-ordered list
      const int* lp = e->G > 1 ? e->h_hb + e->nc + e->hb_off[e->rank] : e->h_tab;
      int n_lt = 0;
      while (n_lt < n_gather && lp[n_lt] < p) ++n_lt;
      n_gather = n_lt;
    }
    if (n_gather > 0) {  // every listed block is held by this rank
      const int tpb = (nt + 31) / 32;
      gather_panel_sym_tiled_kernel<<<(unsigned)((long long)n_gather * tpb * tpb), 256, 0, e->s>>>(
          e->geom(), gpos, p, e->Pbuf);
      CU(cudaGetLastError());
      e->launches += 1;
    }
    g_probe.mark("gather", e->s);
  }
  double flops = 0.0;
  if (!last) {
    if (e->sym)
      CU(cudaStreamWaitEvent(e->s, e->ev_join, 0));  // L_k^-1 from the side stream
    else
      launch_trinv(e, Lk);
    g_probe.mark("trinv", e->s);
    const bool dist_w = e->sym && e->G > 1;
    const int n_own_rows = dist_w ? (e->hb_off[e->rank + 1] - e->hb_off[e->rank]) * nt : R * nt;
    // only when the owner updated its strip this round: in a round without it
    // (round 1, after a flush) the owner's flag holds an older sequence
    if (dist_w && crossed && e->p2p && owner != e->rank) {
      p2p_wait_kernel<<<1, 32, 0, e->s>>>(e->peer_flag[owner] + 1, e->seq2, e->d_abort);
      CU(cudaGetLastError());
    }
    if (dist_w && n_own_rows > 0) {
      // W rows of the blocks this rank holds, packed (row-major, ld = ldw)
      PanelArgs pa{};
      pa.P = P;
      pa.ldp = e->n;
      // the owner's panel k (its geometry: rank = owner)
      PanelGeom og = e->geom();
      og.base = owner == e->rank ? e->C : e->p2p ? e->peer_c[owner] : nullptr;
      og.rank = owner;
      if (og.base) {
        pa.P2 = og.panel(q);
        pa.ldp2 = og.ld(q);
        pa.p2_row0 = og.start(q);
      }
      pa.pk = p;
      pa.Linv = e->Linv;
      pa.ldl = e->ldw;
      pa.W = e->Wsend;
      pa.ldw = e->ldw;
      pa.row_pos = e->d_hbpos + e->hb_off[e->rank];
      pa.nt = nt;
      pa.n_rows = n_own_rows;
      pa.G = e->G;
      pa.rank = e->rank;
      dim3 grid((pa.n_rows + pw::BR - 1) / pw::BR, (nt + pw::BN - 1) / pw::BN);
      panel_w_kernel<2><<<grid, pw::THREADS, pw::SMEM, e->s>>>(pa);
      CU(cudaGetLastError());
      e->launches += 1;
    }
    g_probe.mark("panelw", e->s);
    if (dist_w && e->p2p) {
      // publish this round's rows, then one kernel reads every holder's rows
      // over NVLink (after its flag) and scatters them into Wt/Wnt (+history).
      // Every rank signals and waits for every peer each round: a peer's next
      // gain kernel (which overwrites the L_k read above) and next W rows come
      // after its wait on this rank's signal.
      ++e->seq;
      p2p_signal_kernel<<<1, 32, 0, e->s>>>(e->flag, e->seq);
      const long long total = (long long)std::max(R, 0) * nt * nt;
      w_peer_scatter_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>((total / 2 + 255) / 256, 148 * 8)),
                              256, 0, e->s>>>(
          e->d_peer_wsend, e->d_peer_flag, e->seq, e->G, e->d_hboff, e->ldw, e->d_hb, e->row_pos(), R, nt,
          e->Wt, e->Wnt, e->mpad, e->export_factor ? e->hist : nullptr, (long long)e->eff_budget * nt * nt,
          (long long)round * nt * nt, e->rank, e->d_abort);
      CU(cudaGetLastError());
      e->launches += 2;
      for (int r = 0; r < e->G; ++r)
        if (r != e->rank) bytes += (uint64_t)(e->hb_off[r + 1] - e->hb_off[r]) * nt * nt * sizeof(double);
      g_probe.mark("p2p-scatter", e->s);
    } else if (dist_w && R > 0) {
      // all-gather-v of the W rows (one broadcast per holder), then scatter into
      // the tiled update operands (+ the factor history of own candidates)
      const size_t rowel = (size_t)nt * e->ldw;
      NC(ncclGroupStart());
      for (int r = 0; r < e->G; ++r) {
        const size_t cnt = (size_t)(e->hb_off[r + 1] - e->hb_off[r]) * rowel;
        if (cnt == 0) continue;
        double* dst = e->Wrecv + (size_t)e->hb_off[r] * rowel;
        NC(ncclBroadcast(r == e->rank ? e->Wsend : dst, dst, cnt, ncclDouble, r, e->comm, e->s));
        if (r != e->rank) bytes += cnt * sizeof(double);
      }
      NC(ncclGroupEnd());
      const long long total = (long long)R * nt * nt;
      w_scatter_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 32), 256, 0, e->s>>>(
          e->Wrecv, e->ldw, e->d_hb, e->row_pos(), R, nt, e->Wt, e->Wnt, e->mpad,
          e->export_factor ? e->hist : nullptr, (long long)e->eff_budget * nt * nt, (long long)round * nt * nt,
          e->G, e->rank);
      CU(cudaGetLastError());
      e->launches += 1;
      g_probe.mark("bcast+scatter", e->s);
    } else if (R > 0) {
      PanelArgs pa{};
      pa.P = P;
      pa.ldp = e->n;
      if (e->sym) {  // G == 1: this rank owns panel k
        const PanelGeom g = e->geom();
        pa.P2 = g.panel(q);
        pa.ldp2 = g.ld(q);
        pa.p2_row0 = g.start(q);
        pa.pk = p;
      }
      pa.Linv = e->Linv;
      pa.ldl = e->ldw;
      pa.W = e->Wt ? nullptr : e->W;
      pa.Wn = e->Wn;
      pa.hist = e->export_factor ? e->hist : nullptr;
      pa.slot_stride = (long long)e->eff_budget * nt * nt;
      pa.step_off = (long long)round * nt * nt;
      pa.G = e->G;
      pa.rank = e->rank;
      pa.Wt = e->Wt;
      pa.Wnt = e->Wnt;
      pa.mpad = e->mpad;
      pa.ldw = e->ldw;
      pa.row_pos = e->row_pos();
      pa.nt = nt;
      pa.n_rows = R * nt;
      dim3 grid((pa.n_rows + pw::BR - 1) / pw::BR, (nt + pw::BN - 1) / pw::BN);
      if (nt % 2 == 0)
        panel_w_kernel<2><<<grid, pw::THREADS, pw::SMEM, e->s>>>(pa);
      else
        panel_w_kernel<1><<<grid, pw::THREADS, pw::SMEM, e->s>>>(pa);
      CU(cudaGetLastError());
      e->launches += 1;
    }
  }
  if (e->export_factor) {
    const long long n2 = (long long)nt * nt;
    const long long slot_stride = (long long)e->eff_budget * n2;
    if (owner == e->rank) {
      hist_diag_kernel<<<(unsigned)std::min<long long>((n2 + 255) / 256, 1024), 256, 0, e->s>>>(
          Lk, nt, e->hist + (long long)q * slot_stride + (long long)round * n2);
      CU(cudaGetLastError());
      e->launches += 1;
    }
  }
  g_probe.mark("hist", e->s);
  CU(cudaEventRecord(ev[3], e->s));
  nv.next("update");
  g_probe.dump(e->rank);
  if (!last && R > 0 && Rl > 0 && e->la) {
    // look-ahead: only the diagonal blocks now (the next round's gains need
    // them); the bulk runs beside the next round's chain (la_bulk_and_cross)
    const int* cg = e->h_tab + e->nc + e->nloc;
    const int rtpb = nt / e->ws_br, ctpb = nt / ws::BC;
    const int nb = e->rbuf;
    int2* L = e->h_lists + (size_t)nb * e->list_cap + la_diag_off(e);
    int nl = 0;
    for (int h = 0; h < Rl; ++h)
      for (int a = 0; a < rtpb; ++a)
        for (int b = 0; b < ctpb; ++b) L[nl++] = make_int2(cg[h] * rtpb + a, h * ctpb + b);
    int2* dL = e->d_lists + (size_t)nb * e->list_cap + la_diag_off(e);
    CU(cudaMemcpyAsync(dL, L, sizeof(int2) * nl, cudaMemcpyHostToDevice, e->s));
    UpdateWSArgs ua = round_update_args(e);
    ua.sym = 0;
    ua.la_mode = 2;
    ua.tlist = dL;
    ua.n_tiles = ua.n_full = nl;
    launch_ws(e, ua, e->rl_cfg);
    e->launches += 1;
    CU(cudaEventRecord(e->ev_wrdy[nb], e->s));  // W_t and the round-t tables are final
    double blocks = 0.0;
    for (int h = 0; h < Rl; ++h) blocks += (double)(R - cg[h]);
    const double n3 = 2.0 * (double)nt * nt * nt;
    flops = n3 * Rl;  // the diagonal blocks; the rest is counted when the bulk runs
    e->update_flops += flops;
    e->prev_bulk_flops = n3 * (blocks - Rl);
  } else if (!last && R > 0 && Rl > 0 && !e->la) {
    const int n_rows = R * nt, n_cols = Rl * nt;
    (void)n_rows;
    (void)n_cols;
    if (nt % 2 == 0) {
      UpdateWSArgs ua = round_update_args(e);
      launch_ws(e, ua, e->rl_cfg);
    } else {
      UpdateArgs ua{};
      ua.C = e->C;
      ua.ldc = e->n;
      ua.W = e->W;
      ua.Wn = e->Wn;
      ua.ldw = e->ldw;
      ua.row_pos = e->row_pos();
      ua.col_slot = e->col_slot();
      ua.col_g = e->col_g();
      ua.nt = nt;
      ua.n_rows = n_rows;
      ua.n_cols = n_cols;
      ua.n_row_tiles = (n_rows + upd::BR - 1) / upd::BR;
      ua.n_col_tiles = (n_cols + upd::BC - 1) / upd::BC;
      ua.group = 16;
      const long long tiles = (long long)ua.n_row_tiles * ua.n_col_tiles;
      const int grid = (int)std::min<long long>(e->n_sms, (tiles + 1) / 2);
      schur_update_kernel<1><<<grid, upd::THREADS, upd::SMEM, e->s>>>(ua);
    }
    CU(cudaGetLastError());
    e->launches += 1;
    if (e->sym) {
      // block-lower triangle incl. diagonal blocks: 2 nt^3 sum_h (R - g_h)
      const int* cg = e->h_tab + e->nc + e->nloc;
      double blocks = 0.0;
      for (int h = 0; h < Rl; ++h) blocks += (double)(R - cg[h]);
      flops = 2.0 * (double)nt * nt * nt * blocks;
    } else {
      flops = 2.0 * nt * (double)n_rows * (double)n_cols;
    }
    e->update_flops += flops;
  }
  if (e->la) {
    // every rank marks every non-final round (even with no local columns left):
    // the next step's bulk/cross and its panel-flag sequence stay in lockstep
    if (!last && (R == 0 || Rl == 0)) e->prev_bulk_flops = 0.0;
    e->prev_valid = !last;
  }
  CU(cudaEventRecord(ev[4], e->s));

  e->chosen.push_back(s1);
  e->objective += g1;
  row.chosen_index = s1;
  row.gain = g1;
  row.objective = e->objective;
  row.runner_up = s2;
  row.runner_up_gain = g2;
  row.near_tie = (s2 >= 0 && (g1 - g2) / std::max(std::fabs(g1), 1.0) < e->tau) ? 1 : 0;
  row.bytes_exchanged = bytes;
  e->nccl_bytes += bytes;
  row.update_flops = flops;
  e->trace.push_back(row);
  if (info) *info = row;
}

dsel_status fail(dsel_engine* e, const Fail& f) {
  if (e) e->err = f.msg;
  else g_create_err = f.msg;
  return f.st;
}

template <class F>
dsel_status guard(dsel_engine* e, F&& f) {
  try {
    f();
    return DSEL_OK;
  } catch (const Fail& x) {
    return fail(e, x);
  } catch (const std::exception& ex) {
    return fail(e, Fail{DSEL_E_INVALID, ex.what()});
  }
}

void destroy_impl(dsel_engine* e) {
  if (!e) return;
  cudaSetDevice(e->dev);
  if (e->s) cudaStreamSynchronize(e->s);
  if (e->cs) cudaStreamSynchronize(e->cs);
  for (auto ev : e->ev) cudaEventDestroy(ev);
  double* dptr[] = {e->cpart, e->Wown, e->Wkn, e->D, e->cbuf, e->ldiag, e->Craw, e->K0, e->W, e->Wn,
                    e->Wt_b[0] ? e->Wt_b[0] : e->Wt, e->Wnt_b[0] ? e->Wnt_b[0] : e->Wnt, e->Pbuf, e->Lk, e->Linv, e->Lscr, e->gains, e->hist,
                    e->kgain, e->stage, e->xbuf};
  for (double* d : dptr)
    if (d) cudaFree(d);
  int* iptr[] = {e->status, e->kstatus, e->d_pos_sensor, e->d_slot_sensor, e->d_round_b[0], e->d_iota};
  for (int* d : iptr)
    if (d) cudaFree(d);
  if (e->d_rec) cudaFree(e->d_rec);
  if (e->d_counter) cudaFree(e->d_counter);
  if (e->d_recs) cudaFree(e->d_recs);
  if (e->h_recs) cudaFreeHost(e->h_recs);
  if (e->s2) cudaStreamSynchronize(e->s2);
  if (e->h_round_b[0]) cudaFreeHost(e->h_round_b[0]);
  if (e->h_round_b[1]) cudaFreeHost(e->h_round_b[1]);
  if (e->d_round_b[1]) cudaFree(e->d_round_b[1]);
  if (e->Wt_b[1]) cudaFree(e->Wt_b[1]);
  if (e->Wnt_b[1]) cudaFree(e->Wnt_b[1]);
  if (e->d_lists) cudaFree(e->d_lists);
  if (e->h_lists) cudaFreeHost(e->h_lists);
  for (int b = 0; b < 2; ++b) {
    if (e->ev_wrdy[b]) cudaEventDestroy(e->ev_wrdy[b]);
    if (e->ev_bulk[b]) cudaEventDestroy(e->ev_bulk[b]);
  }
  if (e->s2) cudaStreamDestroy(e->s2);
  if (e->hstore) cudaFreeHost(e->hstore);
  if (e->hk_registered) cudaHostUnregister(e->hk_registered);
  detach_kbf(e);
  for (void* ptr : e->ipc_opened) cudaIpcCloseMemHandle(ptr);
  if (e->flag) cudaFree(e->flag);
  if (e->d_peer_wsend) cudaFree(e->d_peer_wsend);
  if (e->d_peer_flag) cudaFree(e->d_peer_flag);
  if (e->Wsend) cudaFree(e->Wsend);
  if (e->Wrecv) cudaFree(e->Wrecv);
  if (e->d_hbpos) cudaFree(e->d_hbpos);

  if (e->Kk) cudaFree(e->Kk);
  if (e->ev_tab) cudaEventDestroy(e->ev_tab);
  if (e->h_stage) cudaFreeHost(e->h_stage);
  if (e->comm && !e->aborted.load()) ncclCommDestroy(e->comm);
  if (e->h_abort) cudaFreeHost(e->h_abort);
  for (int b = 0; b < 2; ++b) {
    if (e->ev_copy[b]) cudaEventDestroy(e->ev_copy[b]);
    if (e->ev_scat[b]) cudaEventDestroy(e->ev_scat[b]);
  }
  if (e->ts) {
    cudaStreamSynchronize(e->ts);
    cudaStreamDestroy(e->ts);
  }
  if (e->ev_fork) cudaEventDestroy(e->ev_fork);
  if (e->ev_join) cudaEventDestroy(e->ev_join);
  if (e->cs) cudaStreamDestroy(e->cs);
  if (e->s) cudaStreamDestroy(e->s);
  delete e;
}

// per-round table block: [row/col tables | block-lower tile schedule | W holder lists]
size_t round_ints(const dsel_engine* e, size_t* tab = nullptr, size_t* sym = nullptr, size_t* hb = nullptr) {
  size_t n_tab = ((size_t)e->nc + 2 * e->nloc + 1 + 3) / 4 * 4, n_sym = 0, n_hb = 0;
  if (e->sym) {
    const size_t nct = (size_t)(e->nloc * e->nt + ws::BC - 1) / ws::BC + 2;
    n_sym = (nct + nct / e->ws_group + 4 + 3) / 4 * 4;
    if (e->G > 1) n_hb = 2 * (size_t)e->nc + e->G + 1;
  }
  if (tab) *tab = n_tab;
  if (sym) *sym = n_sym;
  if (hb) *hb = n_hb;
  return n_tab + n_sym + n_hb;
}

// look-ahead tile lists per round: the next chosen row/column strip (<= all
// local blocks + all rows below) and the diagonal blocks of the local columns


// Storage plan: algorithm, residency and panel layout, and everything sized
// from them (create_impl allocates exactly what plan_bytes counts).
void apply_plan(dsel_engine* e, const dsel_config* cfg, bool ll, bool stream) {
  e->ll = ll;
  e->stream = stream;
  e->keep = cfg->keep_pristine != 0 && !ll;
  e->sym = cfg->full_square == 0 && e->nt % 2 == 0 && !ll;
  e->packed = e->sym && cfg->panel_layout == 0;
  e->full_panels = !e->packed;
  e->c_elems = (size_t)e->geom().total(e->nloc);
  e->c_pad = e->packed ? (size_t)e->n : 0;
  e->mpad = round_up((int)e->n, ws::ROW_PAD);
  e->hpacked = stream && e->G == 1;
  // look-ahead rounds (DSEL_LOOKAHEAD=0 turns them off)
  const char* la_env = getenv("DSEL_LOOKAHEAD");
  e->la = e->sym && !ll && e->nt % e->ws_br == 0 && e->nt % ws::BC == 0 && !(la_env && atoi(la_env) == 0);
}

uint64_t plan_bytes(const dsel_engine* e, const dsel_config* cfg) {
  uint64_t b = 0;
  auto add = [&](uint64_t count, uint64_t size) { b += std::max<uint64_t>(count, 1) * size; };
  const uint64_t nt = e->nt, n = (uint64_t)e->n, ldw = e->ldw, nloc1 = std::max(e->nloc, 1);
  const uint64_t B = std::max(e->eff_budget, 1);
  if (!e->stream) add(e->c_pad + e->c_elems, 8);
  if (e->keep) add(e->c_elems, 8);
  if (nt % 2 && !e->ll) add(n * ldw, 8);
  if (!e->ll) {
    if (nt % 2 == 0) {
      add((uint64_t)e->mpad * ldw, 8);
      add((uint64_t)e->mpad * ldw, 8);
    } else {
      add(n * ldw, 8);
    }
  }
  if ((e->G > 1 || e->sym) && !e->ll) add(n * nt, 8);
  if (e->ll) {
    const uint64_t own_mpad = round_up((int)(nloc1 * nt), 128), k_mpad = round_up(e->nt, ws::BR);
    const uint64_t ldo = nloc1 * nt;
    add(own_mpad * B * ldw, 8);
    add(k_mpad * B * ldw, 8);
    add(nloc1 * nt * nt, 8);
    add(ldo * nt, 8);
    const int max_nk = (int)(B * ldw / 16);
    const int ns = std::max(1, std::min(kLLMaxSplits, (max_nk + kLLSplitChunks - 1) / kLLSplitChunks));
    const int np = nt % 2 ? ns : kLLMaxSplits;
    if (np > 1) add((uint64_t)np * ldo * nt, 8);
    add(B * nt * nt, 8);
    add(nloc1, 4);
  }
  add(round_ints(e), 4);
  if (e->la) {  // second table buffer, second W buffers, tile lists
    add(round_ints(e), 4);
    add((uint64_t)e->mpad * ldw, 8);
    add((uint64_t)e->mpad * ldw, 8);
    add(2 * la_list_cap(e), 8);
  }
  if (e->sym && e->G > 1) {
    add(n * ldw, 8);
    add(n * ldw, 8);
  }
  add(nt * nt, 8);
  add(ldw * ldw, 8);
  add(nloc1 * nt * nt, 8);
  add(e->nloc + 1, 8);
  add(e->nloc + 1, 4);
  add(1, 8);
  add(1, 4);
  add(3 * (uint64_t)(e->nloc + 1), 8);
  if (cfg->export_factor && !e->ll) add(nloc1 * B * nt * nt, 8);
  add(e->nc, 4);
  add(e->nloc + 1, 4);
  add(1, sizeof(ArgRec));
  add(3, 8);  // gain ticket + update-kernel claim counters
  add(e->G, sizeof(ArgRec));
  if (e->stream) add(nloc1 * nt * nt, 8);
  return b;
}

void connect_impl(dsel_engine* e);

void create_impl(const dsel_config* cfg, dsel_engine** out) {
  Nvtx nv("dsel_create");
  if (!cfg || !out) throw Fail{DSEL_E_INVALID, "null argument"};
  if (cfg->n_sensors < 1 || cfg->n_steps < 1) throw Fail{DSEL_E_INVALID, "n_sensors and n_steps must be >= 1"};
  if (cfg->budget < 0) throw Fail{DSEL_E_INVALID, "budget must be nonnegative"};
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    throw Fail{DSEL_E_INVALID, "bad world_size/rank"};
  if (cfg->storage == DSEL_STORAGE_STREAM && cfg->algorithm != 1)
    throw Fail{DSEL_E_INVALID, "storage=stream streams one K column per round and needs the "
                               "left-looking W-resident algorithm (algorithm = 1, SURVEY 7.3-4)"};
  if (cfg->n_steps > 1024) throw Fail{DSEL_E_INVALID, "n_steps > 1024 is not supported by the gain kernel"};
  if (cfg->algorithm < 0 || cfg->algorithm > 1) throw Fail{DSEL_E_INVALID, "unknown algorithm"};
  auto* e = new dsel_engine();
  try {
    e->nd = cfg->n_sensors;
    e->nt = cfg->n_steps;
    e->budget = cfg->budget;
    e->G = cfg->world_size;
    e->rank = cfg->rank;
    e->dev = cfg->device;
    e->export_factor = cfg->export_factor != 0;
    e->tau = cfg->near_tie_tau > 0 ? cfg->near_tie_tau : 1e-9;
    // candidates (selector.hpp:142-151 check_candidates semantics)
    e->sensor_pos.assign(e->nd, -1);
    if (cfg->n_candidates > 0) {
      if (!cfg->candidates) throw Fail{DSEL_E_INVALID, "candidates pointer is null"};
      for (int i = 0; i < cfg->n_candidates; ++i) {
        const int c = cfg->candidates[i];
        if (c < 0 || c >= e->nd) throw Fail{DSEL_E_RANGE, "candidate index out of range"};
        if (e->sensor_pos[c] >= 0) throw Fail{DSEL_E_INVALID, "duplicate candidate index"};
        e->sensor_pos[c] = 0;
      }
      // position order = ascending sensor id (result-invariant, parallel.hpp:299-304)
      for (int sidx = 0; sidx < e->nd; ++sidx)
        if (e->sensor_pos[sidx] >= 0) {
          e->sensor_pos[sidx] = (int)e->pos_sensor.size();
          e->pos_sensor.push_back(sidx);
        }
    } else {
      for (int sidx = 0; sidx < e->nd; ++sidx) {
        e->sensor_pos[sidx] = sidx;
        e->pos_sensor.push_back(sidx);
      }
    }
    e->nc = (int)e->pos_sensor.size();
    e->n = (long long)e->nc * e->nt;
    if (e->n > (1LL << 31) - 1) throw Fail{DSEL_E_INVALID, "n_candidates*n_steps exceeds 2^31"};
    e->nloc = e->nc > e->rank ? (e->nc - e->rank + e->G - 1) / e->G : 0;
    for (int q = 0; q < e->nloc; ++q) e->slot_sensor.push_back(e->pos_sensor[q * e->G + e->rank]);
    e->eff_budget = std::min(e->budget, e->nc);
    e->ldw = round_up(e->nt, 16);
    e->alive.assign(e->nc, 1);
    e->n_alive = e->nc;

    CU(cudaSetDevice(e->dev));
    set_smem_limits(e->dev);
    CU(cudaDeviceGetAttribute(&e->n_sms, cudaDevAttrMultiProcessorCount, e->dev));
    // the round chain's stream outranks the look-ahead bulk stream: when both
    // have work pending, the chain's CTAs get the SMs first
    int prio_least = 0, prio_greatest = 0;
    CU(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    e->prio_least = prio_least;
    CU(cudaStreamCreateWithPriority(&e->s, cudaStreamNonBlocking, prio_greatest));
    CU(cudaStreamCreateWithFlags(&e->cs, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&e->ts, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      CU(cudaEventCreateWithFlags(&e->ev_copy[b], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&e->ev_scat[b], cudaEventDisableTiming));
    }
    if (const char* wc = getenv("DSEL_WS_CFG")) e->ws_cfg = std::max(-1, std::min(8, atoi(wc)));
    // BigR: DMMA from zero + bulk reduce-add write-back; its 3 x 2 stage
    // variant from 16 k-chunks (Nt = 420), like Big4 for the plain kernel
    e->rl_cfg = e->ws_cfg >= 0 ? e->ws_cfg : (e->ldw / ws::KC >= 16 ? 6 : 5);
    e->ws_br = cfg_br(e->rl_cfg);
    if (const char* wg = getenv("DSEL_WS_GROUP")) e->ws_group = std::max(1, atoi(wg));
    // the storage plan decides every allocation below. AUTO: K resident in
    // HBM with the requested algorithm when that fits the budget, else the
    // streaming store (left-looking, K in host memory, north star (1))
    {
      size_t free_b = 0, total_b = 0;
      CU(cudaMemGetInfo(&free_b, &total_b));
      const uint64_t reserve = 2ull << 30;
      e->plan_budget = cfg->hbm_budget ? cfg->hbm_budget : (free_b > reserve ? free_b - reserve : 0);
      const bool want_ll = cfg->algorithm == 1;
      apply_plan(e, cfg, want_ll, cfg->storage == DSEL_STORAGE_STREAM);
      e->planned = plan_bytes(e, cfg);
      if (cfg->storage == DSEL_STORAGE_AUTO && e->planned > e->plan_budget) {
        apply_plan(e, cfg, true, true);
        e->planned = plan_bytes(e, cfg);
        if (e->planned > e->plan_budget)
          throw Fail{DSEL_E_OOM, "storage=auto: even the streaming store needs " +
                                     std::to_string(e->planned) + " device bytes > budget " +
                                     std::to_string(e->plan_budget)};
      }
    }
    uint64_t& tot = e->dev_bytes;
    const size_t shard = e->c_elems;
    if (!e->stream) {
      e->Craw = dmalloc<double>(e->c_pad + shard, tot);
      e->C = e->Craw + e->c_pad;
    }
    if (e->keep) e->K0 = dmalloc<double>(shard, tot);
    if (e->nt % 2 && !e->ll) e->W = dmalloc<double>((size_t)e->n * e->ldw, tot);  // odd-nt update path
    e->mpad = round_up((int)e->n, ws::ROW_PAD);
    if (e->ll) {
      // left-looking: no resident conditional covariance, no right-looking W
    } else if (e->nt % 2 == 0) {
      e->Wt = dmalloc<double>((size_t)e->mpad * e->ldw, tot);
      e->Wnt = dmalloc<double>((size_t)e->mpad * e->ldw, tot);
    } else {
      e->Wn = dmalloc<double>((size_t)e->n * e->ldw, tot);
    }
    if ((e->G > 1 || e->sym) && !e->ll) e->Pbuf = dmalloc<double>((size_t)e->n * e->nt, tot);
    if (e->ll) {
      const int B = std::max(e->eff_budget, 1);
      e->own_mpad = round_up(std::max(e->nloc, 1) * e->nt, 128);
      e->k_mpad = round_up(e->nt, ws::BR);  // whole 128-row r-side tiles stay inside the buffer
      e->ldo = (long long)std::max(e->nloc, 1) * e->nt;
      e->Wown = dmalloc<double>((size_t)e->own_mpad * B * e->ldw, tot);
      e->Wkn = dmalloc<double>((size_t)e->k_mpad * B * e->ldw, tot);
      e->D = dmalloc<double>((size_t)std::max(e->nloc, 1) * e->nt * e->nt, tot);
      e->cbuf = dmalloc<double>((size_t)e->ldo * e->nt, tot);
      {
        const int max_nk = (B * e->ldw) / 16;
        const int ns = std::max(1, std::min(kLLMaxSplits, (max_nk + kLLSplitChunks - 1) / kLLSplitChunks));
        // split-K planes: odd-nt GEMM (ns) / wave-balanced TMA GEMM (kLLMaxSplits)
        const int np = e->nt % 2 ? ns : kLLMaxSplits;
        if (np > 1) e->cpart = dmalloc<double>((size_t)np * e->ldo * e->nt, tot);
      }
      e->ldiag = dmalloc<double>((size_t)B * e->nt * e->nt, tot);
      e->d_iota = dmalloc<int>(std::max(e->nloc, 1), tot);
      std::vector<int> iota(std::max(e->nloc, 1));
      for (size_t i = 0; i < iota.size(); ++i) iota[i] = (int)i;
      CU(cudaMemcpy(e->d_iota, iota.data(), sizeof(int) * iota.size(), cudaMemcpyHostToDevice));
      CU(cudaMemsetAsync(e->Wown, 0, sizeof(double) * (size_t)e->own_mpad * B * e->ldw, e->s));
      CU(cudaMemsetAsync(e->Wkn, 0, sizeof(double) * (size_t)e->k_mpad * B * e->ldw, e->s));
    }
    // per-round host tables, one pinned staging block and one device block so a
    // round uploads them with a single copy: [row/col tables | block-lower tile
    // schedule | W holder lists (symmetric, G > 1)]
    size_t n_tab, n_sym, n_hb;
    e->round_ints = round_ints(e, &n_tab, &n_sym, &n_hb);
    if (e->sym && e->G > 1) {
      e->Wsend = dmalloc<double>((size_t)e->n * e->ldw, tot);
      e->Wrecv = dmalloc<double>((size_t)e->n * e->ldw, tot);
    }
    e->d_round = dmalloc<int>(e->round_ints, tot);
    CU(ds_malloc_host(&e->h_round, sizeof(int) * e->round_ints));
    e->d_round_b[0] = e->d_round;
    e->h_round_b[0] = e->h_round;
    if (e->la) {
      e->d_round_b[1] = dmalloc<int>(e->round_ints, tot);
      CU(ds_malloc_host(&e->h_round_b[1], sizeof(int) * e->round_ints));
      e->Wt_b[0] = e->Wt;
      e->Wnt_b[0] = e->Wnt;
      e->Wt_b[1] = dmalloc<double>((size_t)e->mpad * e->ldw, tot);
      e->Wnt_b[1] = dmalloc<double>((size_t)e->mpad * e->ldw, tot);
      CU(cudaMemsetAsync(e->Wt_b[1], 0, sizeof(double) * (size_t)e->mpad * e->ldw, e->s));
      CU(cudaMemsetAsync(e->Wnt_b[1], 0, sizeof(double) * (size_t)e->mpad * e->ldw, e->s));
      e->list_cap = la_list_cap(e);
      e->d_lists = reinterpret_cast<int2*>(dmalloc<double>(2 * e->list_cap, tot));
      CU(ds_malloc_host(&e->h_lists, sizeof(int2) * 2 * e->list_cap));
      CU(cudaStreamCreateWithPriority(&e->s2, cudaStreamNonBlocking, e->prio_least));
      for (int b = 0; b < 2; ++b) {
        CU(cudaEventCreateWithFlags(&e->ev_wrdy[b], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&e->ev_bulk[b], cudaEventDisableTiming));
      }
      // C2 sweeps (profiles/r02_la_reserve_c2.json): 12 SMs at 1 GPU (with the
      // dynamic tile schedule; 8 with the static one), 12 at 2, 16 from 4 GPUs
      // up (8 GPUs: 25 candidates per rank, the gain kernel's CTAs fit 16 SMs
      // in one wave)
      e->la_reserve = e->G <= 2 ? 12 : 16;
      if (const char* rs = getenv("DSEL_LA_RESERVE")) e->la_reserve = std::max(0, std::min(e->n_sms - 8, atoi(rs)));
    }
    e->n_tab_ints = n_tab;
    e->n_sym_ints = n_sym;
    e->n_hb_ints = n_hb;
    set_round_buf(e, 0);
    e->Lk = dmalloc<double>((size_t)e->nt * e->nt, tot);
    e->Linv = dmalloc<double>((size_t)e->ldw * e->ldw, tot);
    e->Lscr = dmalloc<double>((size_t)std::max(e->nloc, 1) * e->nt * e->nt, tot);
    e->gains = dmalloc<double>(e->nloc + 1, tot);
    e->status = dmalloc<int>(e->nloc + 1, tot);
    e->kgain = dmalloc<double>(1, tot);
    e->kstatus = dmalloc<int>(1, tot);
    e->xbuf = dmalloc<double>((size_t)3 * (e->nloc + 1), tot);  // int tables, oversized
    if (e->export_factor && !e->ll)
      e->hist = dmalloc<double>((size_t)std::max(e->nloc, 1) * std::max(e->eff_budget, 1) *
                                    e->nt * e->nt, tot);
    e->d_pos_sensor = dmalloc<int>(e->nc, tot);
    e->d_slot_sensor = dmalloc<int>(e->nloc + 1, tot);
    e->d_rec = dmalloc<ArgRec>(1, tot);
    {  // [0]: the gain ticket (low word); [1], [2]: update-kernel claim counters
      unsigned long long* blk = dmalloc<unsigned long long>(3, tot);
      CU(cudaMemsetAsync(blk, 0, 3 * sizeof(unsigned long long), e->s));
      e->d_counter = reinterpret_cast<unsigned*>(blk);
      e->ws_ctr = blk + 1;
      const char* wd = getenv("DSEL_WS_DYNAMIC");
      e->ws_dynamic = !(wd && wd[0] == '0');
    }
    e->d_recs = dmalloc<ArgRec>(e->G, tot);
    CU(ds_malloc_host(&e->h_recs, sizeof(ArgRec) * e->G));
    if (e->W) CU(cudaMemsetAsync(e->W, 0, sizeof(double) * (size_t)e->n * e->ldw, e->s));
    if (e->Wn) CU(cudaMemsetAsync(e->Wn, 0, sizeof(double) * (size_t)e->n * e->ldw, e->s));
    if (e->Wt) {
      CU(cudaMemsetAsync(e->Wt, 0, sizeof(double) * (size_t)e->mpad * e->ldw, e->s));
      CU(cudaMemsetAsync(e->Wnt, 0, sizeof(double) * (size_t)e->mpad * e->ldw, e->s));
    }
    if (e->Craw) CU(cudaMemsetAsync(e->Craw, 0, sizeof(double) * (e->c_pad + shard), e->s));
    if (e->stream) {
      e->Kk = dmalloc<double>((size_t)std::max(e->nloc, 1) * e->nt * e->nt, tot);
      CU(cudaEventCreateWithFlags(&e->ev_tab, cudaEventDisableTiming));
    }
    CU(cudaMemcpyAsync(e->d_pos_sensor, e->pos_sensor.data(), sizeof(int) * e->nc,
                       cudaMemcpyHostToDevice, e->s));
    if (e->nloc)
      CU(cudaMemcpyAsync(e->d_slot_sensor, e->slot_sensor.data(), sizeof(int) * e->nloc,
                         cudaMemcpyHostToDevice, e->s));
    e->ev.resize((size_t)std::max(e->eff_budget, 1) * kEv);
    for (auto& x : e->ev) CU(cudaEventCreate(&x));
    // peer-failure word (host-mapped pinned): dsel_abort sets it, the
    // NVLink flag waits poll it
    CU(ds_host_alloc_mapped(&e->h_abort, sizeof(int)));
    *e->h_abort = 0;
    {
      void* dp = nullptr;
      CU(cudaHostGetDevicePointer(&dp, e->h_abort, 0));
      e->d_abort = static_cast<const volatile int*>(dp);
    }
    if (e->G > 1) {
      if (!cfg->nccl_id) throw Fail{DSEL_E_INVALID, "world_size > 1 requires nccl_id"};
      std::memcpy(e->nccl_id, cfg->nccl_id, sizeof(e->nccl_id));
    }
    build_tables(e);
    CU(cudaStreamSynchronize(e->s));
    if (e->G > 1 && !cfg->defer_connect) connect_impl(e);
  } catch (...) {
    destroy_impl(e);
    throw;
  }
  *out = e;
}

// The collective half of create (world_size > 1): NCCL communicator, warm
// collectives and the NVLink peer mappings. Split from the allocations so a
// caller can agree that every rank created its engine before any rank blocks
// in ncclCommInitRank (dsel_config.defer_connect + dsel_connect).
void connect_impl(dsel_engine* e) {
  if (e->G == 1 || e->comm) return;
  CU(cudaSetDevice(e->dev));
  ncclUniqueId id;
  std::memcpy(&id, e->nccl_id, sizeof(id));
  NC(ncclCommInitRank(&e->comm, e->G, id, e->rank));
  // establish NCCL's peer connections now (lazily done by the first call of
  // each collective), so round 1 of the first selection is not charged for it
  double* wb = e->Pbuf ? e->Pbuf : e->Lk;
  const size_t wn = std::min<size_t>(e->Pbuf ? (size_t)e->n * e->nt : (size_t)e->nt * e->nt, 1 << 20);
  NC(ncclGroupStart());
  NC(ncclAllGather(e->d_rec, e->d_recs, sizeof(ArgRec), ncclUint8, e->comm, e->s));
  NC(ncclGroupEnd());
  NC(ncclAllReduce(wb, wb, wn, ncclDouble, ncclSum, e->comm, e->s));
  NC(ncclBroadcast(wb, wb, wn, ncclDouble, 0, e->comm, e->s));
  CU(cudaMemsetAsync(wb, 0, sizeof(double) * wn, e->s));
  setup_p2p(e);
  CU(cudaStreamSynchronize(e->s));
}

void ensure_stage(dsel_engine* e, size_t elems) {
  if (e->stage_elems >= elems) return;
  CU(cudaStreamSynchronize(e->s));
  CU(cudaStreamSynchronize(e->cs));
  if (e->stage) cudaFree(e->stage);
  if (e->h_stage) cudaFreeHost(e->h_stage);
  e->stage = nullptr;
  e->h_stage = nullptr;
  e->stage = dmalloc<double>(2 * elems, e->dev_bytes);
  CU(ds_malloc_host(&e->h_stage, elems * sizeof(double)));
  e->stage_elems = elems;
}


// Panel store ingest: H2D of one block row/column into device staging on the
// copy stream (double-buffered, event-ordered), scatter into the panel on the
// compute stream, so consecutive panels overlap copy and scatter.
// Streaming store fill: block row j of an own candidate (as_column = false)
// gives K(own_j, k) for every k; a block column j gives K(own_i, j) for every
// own i (host-to-host copies into the pinned store).
void ensure_hstore(dsel_engine* e) {
  if (e->hk_registered) {
    cudaHostUnregister(e->hk_registered);
    e->hk_registered = nullptr;
  }
  e->hk_user = nullptr;  // loading data detaches a caller's K
  detach_kbf(e);
  if (!e->hstore) {
    CU(cudaSetDevice(e->dev));
    CU(ds_malloc_host(&e->hstore, sizeof(double) * hstore_blocks(e) * e->nt * e->nt));
  }
}

void store_fill(dsel_engine* e, int j, const double* host, bool as_column) {
  const size_t n2 = (size_t)e->nt * e->nt;
  ensure_hstore(e);
  const int p = e->sensor_pos[j];
  if (p < 0) return;
  if (e->hpacked) {
    if (!as_column) {  // block row p: K(p, pk) for pk <= p -> panel pk, index p - pk
      for (int pk = 0; pk <= p; ++pk)
        std::memcpy(hpacked_block(e, pk, p), host + (size_t)e->pos_sensor[pk] * n2, n2 * sizeof(double));
    } else {  // block column p: K(q, p) for q >= p -> panel p
      for (int q = p; q < e->nc; ++q)
        std::memcpy(hpacked_block(e, p, q), host + (size_t)e->pos_sensor[q] * n2, n2 * sizeof(double));
    }
    return;
  }
  if (!as_column) {
    if (p % e->G != e->rank) return;
    const int q = p / e->G;
    for (int pk = 0; pk < e->nc; ++pk)
      std::memcpy(e->hstore + ((size_t)pk * e->nloc + q) * n2, host + (size_t)e->pos_sensor[pk] * n2,
                  n2 * sizeof(double));
  } else {
    for (int q = 0; q < e->nloc; ++q)
      std::memcpy(e->hstore + ((size_t)p * e->nloc + q) * n2, host + (size_t)e->slot_sensor[q] * n2,
                  n2 * sizeof(double));
  }
}

// Own panel q of K (full height, column-major, ld = ldp) from the device into
// the host store: packed (world_size 1) keeps K(i, q), i >= q; full keeps
// K(q, pk) for every pk. `packed` is nc blocks of device scratch.
cudaError_t store_panel_d2h(dsel_engine* e, const double* panel, long long ldp, int q, double* packed) {
  const size_t n2 = (size_t)e->nt * e->nt;
  const long long total = (long long)e->nc * n2;
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148 * 16);
  if (e->hpacked) {
    stream_pack_lower_kernel<<<grid, 256, 0, e->s>>>(panel, ldp, e->nt, q, e->nc, packed);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
    return cudaMemcpyAsync(hpacked_block(e, q, q), packed, sizeof(double) * n2 * (e->nc - q),
                           cudaMemcpyDeviceToHost, e->s);
  }
  stream_pack_kernel<<<grid, 256, 0, e->s>>>(panel, ldp, e->nt, e->nc, packed);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) return ce;
  return cudaMemcpy2DAsync(e->hstore + (size_t)q * n2, (size_t)e->nloc * n2 * sizeof(double), packed,
                           n2 * sizeof(double), n2 * sizeof(double), e->nc, cudaMemcpyDeviceToHost, e->s);
}

void load_panel(dsel_engine* e, int j, const double* host, bool as_column) {
  if (j < 0 || j >= e->nd) throw Fail{DSEL_E_RANGE, "block index out of range"};
  if (e->stream) {
    store_fill(e, j, host, as_column);
    return;
  }
  const int p = e->sensor_pos[j];
  if (p < 0 || p % e->G != e->rank) return;
  const int q = p / e->G;
  const size_t elems = (size_t)e->nd * e->nt * e->nt;
  // symmetric storage needs only the block-lower part of the panel: blocks of
  // candidates at positions >= p, i.e. sensors >= j -- a contiguous suffix
  const int s_off = e->sym ? j : 0;
  const int p_first = e->sym ? p : 0;
  const size_t off = (size_t)s_off * e->nt * e->nt;
  const size_t copy = elems - off;
  CU(cudaSetDevice(e->dev));
  ensure_stage(e, elems);
  const int b = e->stage_flip;
  e->stage_flip ^= 1;
  double* buf = e->stage + (size_t)b * e->stage_elems;
  CU(cudaStreamWaitEvent(e->cs, e->ev_scat[b], 0));
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, host) == cudaSuccess &&
                      attr.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (pinned) {
    CU(cudaMemcpyAsync(buf, host + off, copy * sizeof(double), cudaMemcpyHostToDevice, e->cs));
  } else {
    // pageable source: bounce through the engine's pinned buffer
    CU(cudaStreamSynchronize(e->cs));
    std::memcpy(e->h_stage, host + off, copy * sizeof(double));
    CU(cudaMemcpyAsync(buf, e->h_stage, copy * sizeof(double), cudaMemcpyHostToDevice, e->cs));
  }
  e->h2d_bytes += copy * sizeof(double);
  if (e->sym) e->full_panels = false;
  CU(cudaEventRecord(e->ev_copy[b], e->cs));
  CU(cudaStreamWaitEvent(e->s, e->ev_copy[b], 0));
  const PanelGeom g = e->geom();
  double* panel = g.panel(q);
  const long long total = (long long)(e->nc - p_first) * e->nt * e->nt;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  if (total > 0) {
    if (as_column)
      scatter_block_col_kernel<<<blocks, 256, 0, e->s>>>(buf, e->nt, e->d_pos_sensor, e->nc,
                                                         panel, g.ld(q), g.start(q), p_first, s_off);
    else
      scatter_block_row_kernel<<<blocks, 256, 0, e->s>>>(buf, e->nt, e->d_pos_sensor, e->nc,
                                                         panel, g.ld(q), g.start(q), p_first, s_off);
  }
  CU(cudaGetLastError());
  CU(cudaEventRecord(e->ev_scat[b], e->s));
  if (e->keep)
    CU(cudaMemcpyAsync(e->K0 + g.off(q), panel, sizeof(double) * g.ld(q) * e->nt,
                       cudaMemcpyDeviceToDevice, e->s));
}

// Roofline denominator probe: DMMA.8x8x4 issue rate with independent
// accumulator chains (no memory traffic), 2 CTAs x 512 threads per SM.
__global__ void __launch_bounds__(512) fp64_peak_kernel(double* out, int iters, double a, double b) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i][0] = threadIdx.x;
    acc[i][1] = i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

// ========================================================================== //
// C ABI                                                                      //
// ========================================================================== //
extern "C" {

int dsel_abi_version(void) { return DSEL_ABI_VERSION; }

void dsel_fold_records(const dsel_argrec* recs, int n, dsel_argrec* out) {
  auto better = [](double d, int s, double bd, int bs) {
    return d > bd || (d == bd && (bs < 0 || s < bs));
  };
  dsel_argrec r{};
  r.g1 = r.g2 = -INFINITY;
  r.s1 = r.s2 = -1;
  auto ins = [&](double d, int s) {
    if (s < 0 || s == r.s1) return;
    if (r.s1 < 0 || better(d, s, r.g1, r.s1)) {
      r.g2 = r.g1;
      r.s2 = r.s1;
      r.g1 = d;
      r.s1 = s;
    } else if (r.s2 < 0 || better(d, s, r.g2, r.s2)) {
      r.g2 = d;
      r.s2 = s;
    }
  };
  for (int i = 0; i < n; ++i) {
    ins(recs[i].g1, recs[i].s1);
    ins(recs[i].g2, recs[i].s2);
    r.n_eval += recs[i].n_eval;
    r.n_inf += recs[i].n_inf;
  }
  *out = r;
}

dsel_status dsel_nccl_unique_id(void* out128) {
  if (!out128) return DSEL_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DSEL_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return DSEL_OK;
}

dsel_status dsel_create(const dsel_config* cfg, dsel_engine** out) {
  try {
    create_impl(cfg, out);
    return DSEL_OK;
  } catch (const Fail& f) {
    g_create_err = f.msg;
    return f.st;
  } catch (const std::exception& ex) {
    g_create_err = ex.what();
    return DSEL_E_INVALID;
  }
}

void dsel_destroy(dsel_engine* e) { destroy_impl(e); }

const char* dsel_last_error(const dsel_engine* e) {
  return e ? e->err.c_str() : g_create_err.c_str();
}

uint64_t dsel_device_bytes(const dsel_engine* e) { return e ? e->dev_bytes : 0; }

uint64_t dsel_alloc_count(void) { return g_allocs.load(); }

// Batched log-det of independent SPD matrices on the device: the gain kernel
// (batched Cholesky, warp-level pivots, DMMA panel updates) over arbitrary
// matrices -- the refactorizing baseline's potrf (selector.hpp:253-357).
namespace {
__global__ void batch_tables_kernel(int batch, long long stride, int m, long long* off, long long* ld,
                                    int* sensor) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  off[b] = (long long)b * stride;
  ld[b] = m;
  sensor[b] = b;
}
}  // namespace

dsel_status dsel_batched_logdet(int device, const double* mats, int m, int64_t stride, int batch,
                                double* logdet, int* status) {
  return guard(nullptr, [&] {
    if (!mats || !logdet || !status || m < 1 || batch < 0 || stride < (int64_t)m * m)
      throw Fail{DSEL_E_INVALID, "batched_logdet: bad arguments"};
    if (m > kBatchedLogdetMaxDim)
      throw Fail{DSEL_E_INVALID, "batched_logdet: m > " + std::to_string(kBatchedLogdetMaxDim)};
    if (batch == 0) return;
    CU(cudaSetDevice(device));
    int sms = 148, optin = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    set_smem_limits(device);
    DevScratch<double> L((size_t)batch * m * m);
    DevScratch<long long> tabs((size_t)2 * batch);
    DevScratch<int> sens((size_t)batch);
    batch_tables_kernel<<<(batch + 127) / 128, 128>>>(batch, stride, m, tabs.p, tabs.p + batch, sens.p);
    CU(cudaGetLastError());
    CholArgs a{};
    a.src = mats;
    a.src_off = tabs.p;
    a.src_ld = tabs.p + batch;
    a.L = L.p;
    a.l_stride = (long long)m * m;
    a.gain = logdet;
    a.status = status;
    a.nt = m;
    a.n = batch;
    a.mp = chol_mp(m);
    a.sensor = sens.p;
    a.rec = nullptr;
    a.counter = nullptr;
    launch_chol(a, batch, nullptr, sms);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
  });
}

dsel_status dsel_measure_fp64_peak(int device, double* tflops) {
  return guard(nullptr, [&] {
    if (!tflops) throw Fail{DSEL_E_INVALID, "null output"};
    CU(cudaSetDevice(device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int threads = 512, blocks = 2 * sms, iters = 20000;
    DevScratch<double> out((size_t)threads * blocks);
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    fp64_peak_kernel<<<blocks, threads>>>(out.p, 200, 1.0, 1e-9);  // warm
    CU(cudaEventRecord(e0));
    fp64_peak_kernel<<<blocks, threads>>>(out.p, iters, 1.0, 1e-9);
    CU(cudaEventRecord(e1));
    CU(cudaEventSynchronize(e1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CU(cudaGetLastError());
    // 8 chains x (8x8x4 MMA = 2*256 flop) per warp per iteration
    const double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

dsel_status dsel_get_plan(const dsel_engine* e, dsel_plan* out) {
  if (!e || !out) return DSEL_E_INVALID;
  dsel_plan p{};
  p.storage = e->stream ? DSEL_STORAGE_STREAM : DSEL_STORAGE_HBM;
  p.algorithm = e->ll ? 1 : 0;
  p.symmetric = e->sym ? 1 : 0;
  p.packed = e->packed ? 1 : 0;
  p.device_bytes = e->dev_bytes;
  p.planned_bytes = e->planned;
  p.budget_bytes = e->plan_budget;
  p.host_store_bytes = e->hstore ? sizeof(double) * (uint64_t)hstore_blocks(e) * e->nt * e->nt : 0;
  *out = p;
  return DSEL_OK;
}

dsel_status dsel_connect(dsel_engine* e) {
  return guard(e, [&] { connect_impl(e); });
}

dsel_status dsel_abort(dsel_engine* e) {
  if (!e) return DSEL_E_INVALID;
  bool expect = false;
  if (!e->aborted.compare_exchange_strong(expect, true)) return DSEL_OK;
  if (e->h_abort) *reinterpret_cast<volatile int*>(e->h_abort) = 1;  // releases NVLink flag waits
  if (e->comm) ncclCommAbort(e->comm);  // releases collectives blocked on the failed peer
  return DSEL_OK;
}

dsel_status dsel_sync(dsel_engine* e) {
  return guard(e, [&] {
    CU(cudaSetDevice(e->dev));
    CU(cudaStreamSynchronize(e->s));
    if (e->s2) CU(cudaStreamSynchronize(e->s2));
  });
}

dsel_status dsel_load_block_row(dsel_engine* e, int j, const double* host_row) {
  return guard(e, [&] { load_panel(e, j, host_row, false); });
}

dsel_status dsel_load_block_col(dsel_engine* e, int j, const double* host_col) {
  return guard(e, [&] { load_panel(e, j, host_col, true); });
}

void attach_host(dsel_engine* e, const double* host_k, bool rows) {
  if (!e->stream) throw Fail{DSEL_E_INVALID, "attach_host_k needs storage = DSEL_STORAGE_STREAM"};
  if (!host_k) throw Fail{DSEL_E_INVALID, "null K"};
  CU(cudaSetDevice(e->dev));
  if (e->hk_registered) {
    cudaHostUnregister(e->hk_registered);
    e->hk_registered = nullptr;
  }
  const size_t bytes = sizeof(double) * (size_t)(rows ? e->nloc : e->nd) * e->nd * e->nt * e->nt;
  e->hk_user = nullptr;
  if (bytes == 0) return;
  cudaPointerAttributes at{};
  const cudaError_t ae = cudaPointerGetAttributes(&at, host_k);
  if (ae != cudaSuccess || at.type != cudaMemoryTypeHost) {
    cudaGetLastError();
    // pageable: pin in place (read-only) so the per-round copies are DMA
    void* base = const_cast<double*>(host_k);
    CU(ds_host_register(base, bytes, cudaHostRegisterReadOnly));
    e->hk_registered = base;
  }
  if (e->hstore) {  // the caller's K replaces a filled store
    cudaFreeHost(e->hstore);
    e->hstore = nullptr;
  }
  detach_kbf(e);
  e->hk_user = host_k;
  e->hk_rows = rows;
}

dsel_status dsel_attach_host_k(dsel_engine* e, const double* host_k) {
  return guard(e, [&] { attach_host(e, host_k, false); });
}

dsel_status dsel_attach_host_rows(dsel_engine* e, const double* host_rows) {
  return guard(e, [&] { attach_host(e, host_rows, true); });
}

dsel_status dsel_load_k(dsel_engine* e, const double* host_k) {
  return guard(e, [&] {
    if (e->stream) {  // hstore[pk][q] = K(own_q, k): block (s_q, s_k) of the block-row-major K
      const size_t n2 = (size_t)e->nt * e->nt;
      ensure_hstore(e);
      if (e->hpacked) {
        for (int pk = 0; pk < e->nc; ++pk)
          for (int q = pk; q < e->nc; ++q)
            std::memcpy(hpacked_block(e, pk, q),
                        host_k + ((size_t)e->pos_sensor[q] * e->nd + e->pos_sensor[pk]) * n2, n2 * sizeof(double));
        return;
      }
      for (int pk = 0; pk < e->nc; ++pk)
        for (int q = 0; q < e->nloc; ++q)
          std::memcpy(e->hstore + ((size_t)pk * e->nloc + q) * n2,
                      host_k + ((size_t)e->slot_sensor[q] * e->nd + e->pos_sensor[pk]) * n2,
                      n2 * sizeof(double));
      return;
    }
    const size_t row = (size_t)e->nd * e->nt * e->nt;
    for (int q = 0; q < e->nloc; ++q) {
      const int sidx = e->slot_sensor[q];
      load_panel(e, sidx, host_k + (size_t)sidx * row, false);
    }
    CU(cudaStreamSynchronize(e->s));
  });
}

// KBF store ingest (kstore.hpp:22-35 layout; validation as KStoreReader,
// kstore.hpp:92-125). Owned panels only; parallel pread of each block row
// (contiguous) or of the Nd blocks of a block column (exact reference
// semantics) into two pinned host buffers, alternated so the pread of panel
// q+1 overlaps the H2D + scatter of panel q.
namespace {

void load_kbf_impl(dsel_engine* e, const char* path, bool exact_columns, int threads) {
  Nvtx nv("dsel_load_kbf");
  const std::string ps(path ? path : "");
  const int fd = ::open(ps.c_str(), O_RDONLY);
  if (fd < 0) throw Fail{DSEL_E_IO, "cannot open " + ps + ": " + std::strerror(errno)};
  struct Closer {
    int fd;
    ~Closer() { ::close(fd); }
  } closer{fd};
  unsigned char h[32];
  if (::pread(fd, h, 32, 0) != 32) throw Fail{DSEL_E_CORRUPT, ps + ": header truncated"};
  auto u32 = [&](int o) {
    return (uint32_t)h[o] | ((uint32_t)h[o + 1] << 8) | ((uint32_t)h[o + 2] << 16) |
           ((uint32_t)h[o + 3] << 24);
  };
  if (std::memcmp(h, "KBF1", 4) != 0) throw Fail{DSEL_E_CORRUPT, ps + ": bad magic"};
  const int nd = (int)u32(8), nt = (int)u32(12);
  if (u32(4) != 1 || u32(16) != 1 || u32(20) != 1 || nd < 1 || nt < 1)
    throw Fail{DSEL_E_CORRUPT, ps + ": unsupported header fields"};
  struct stat st {};
  if (::fstat(fd, &st) != 0) throw Fail{DSEL_E_IO, ps + ": fstat failed"};
  const size_t bsz = (size_t)nt * nt * sizeof(double);
  const size_t expect = 32 + (size_t)nd * nd * bsz;
  if ((size_t)st.st_size != expect)
    throw Fail{DSEL_E_CORRUPT, ps + ": size " + std::to_string(st.st_size) + " != expected " +
                                   std::to_string(expect)};
  if (nd != e->nd || nt != e->nt)
    throw Fail{DSEL_E_INVALID, ps + ": store shape does not match the engine configuration"};
  const size_t row_bytes = (size_t)nd * bsz;
  double* hb[2] = {nullptr, nullptr};
  cudaEvent_t freed[2] = {nullptr, nullptr};
  try {
    for (int b = 0; b < 2; ++b) {
      CU(ds_malloc_host(&hb[b], row_bytes));
      CU(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    }
    if (threads <= 0) threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    int flip = 0;
    for (int q = 0; q < e->nloc; ++q) {
      const int j = e->slot_sensor[q];
      double* buf = hb[flip];
      CU(cudaEventSynchronize(freed[flip]));  // its previous H2D has completed
      // parallel pread of the Nd blocks of this panel
      const int i_first = e->sym ? j : 0;  // block-lower part only (symmetric storage)
      auto work = [&](int w) {
        for (int i = i_first + w; i < nd; i += threads) {
          const size_t blk = exact_columns ? ((size_t)i * nd + j) : ((size_t)j * nd + i);
          pread_exact(fd, reinterpret_cast<unsigned char*>(buf) + (size_t)i * bsz, bsz,
                      (off_t)(32 + blk * bsz), ps);
        }
      };
      std::vector<std::thread> pool;
      std::vector<std::string> errs(threads);
      std::vector<int> codes(threads, 0);
      for (int w = 0; w < threads; ++w)
        pool.emplace_back([&, w] {
          try {
            work(w);
          } catch (const Fail& f) {
            codes[w] = f.st;
            errs[w] = f.msg;
          }
        });
      for (auto& t : pool) t.join();
      for (int w = 0; w < threads; ++w)
        if (codes[w]) throw Fail{(dsel_status)codes[w], errs[w]};
      load_panel(e, j, buf, exact_columns);
      CU(cudaEventRecord(freed[flip], e->cs));
      flip ^= 1;
    }
    CU(cudaStreamSynchronize(e->s));
    CU(cudaStreamSynchronize(e->cs));
  } catch (...) {
    for (int b = 0; b < 2; ++b) {
      if (hb[b]) cudaFreeHost(hb[b]);
      if (freed[b]) cudaEventDestroy(freed[b]);
    }
    throw;
  }
  for (int b = 0; b < 2; ++b) {
    cudaFreeHost(hb[b]);
    cudaEventDestroy(freed[b]);
  }
}
}  // namespace

// File-backed streaming store: validate like KStoreReader and keep the file;
// each round reads only the chosen column's own blocks (stream_column).
void attach_kbf_impl(dsel_engine* e, const char* path, int threads) {
  if (!e->stream) throw Fail{DSEL_E_INVALID, "attach_kbf needs storage = DSEL_STORAGE_STREAM"};
  const std::string ps(path ? path : "");
  const int fd = ::open(ps.c_str(), O_RDONLY);
  if (fd < 0) throw Fail{DSEL_E_IO, "cannot open " + ps + ": " + std::strerror(errno)};
  try {
    unsigned char h[32];
    if (::pread(fd, h, 32, 0) != 32) throw Fail{DSEL_E_CORRUPT, ps + ": header truncated"};
    auto u32 = [&](int o) {
      return (uint32_t)h[o] | ((uint32_t)h[o + 1] << 8) | ((uint32_t)h[o + 2] << 16) | ((uint32_t)h[o + 3] << 24);
    };
    if (std::memcmp(h, "KBF1", 4) != 0) throw Fail{DSEL_E_CORRUPT, ps + ": bad magic"};
    const int nd = (int)u32(8), nt = (int)u32(12);
    if (u32(4) != 1 || u32(16) != 1 || u32(20) != 1 || nd < 1 || nt < 1)
      throw Fail{DSEL_E_CORRUPT, ps + ": unsupported header fields"};
    struct stat st {};
    if (::fstat(fd, &st) != 0) throw Fail{DSEL_E_IO, ps + ": fstat failed"};
    const size_t expect = 32 + (size_t)nd * nd * nt * nt * sizeof(double);
    if ((size_t)st.st_size != expect)
      throw Fail{DSEL_E_CORRUPT, ps + ": size " + std::to_string(st.st_size) + " != expected " + std::to_string(expect)};
    if (nd != e->nd || nt != e->nt)
      throw Fail{DSEL_E_INVALID, ps + ": store shape does not match the engine configuration"};
    CU(cudaSetDevice(e->dev));
    if (e->hstore) {
      cudaFreeHost(e->hstore);
      e->hstore = nullptr;
    }
    if (e->hk_registered) {
      cudaHostUnregister(e->hk_registered);
      e->hk_registered = nullptr;
    }
    e->hk_user = nullptr;
    detach_kbf(e);
    CU(ds_malloc_host(&e->h_kstage, sizeof(double) * (size_t)std::max(e->nloc, 1) * e->nt * e->nt));
  } catch (...) {
    ::close(fd);
    throw;
  }
  e->kbf_fd = fd;
  e->kbf_path = ps;
  e->kbf_threads = threads > 0 ? threads : (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}

dsel_status dsel_attach_kbf(dsel_engine* e, const char* path, int threads) {
  return guard(e, [&] { attach_kbf_impl(e, path, threads); });
}

dsel_status dsel_load_kbf(dsel_engine* e, const char* path, int exact_columns, int threads) {
  return guard(e, [&] { load_kbf_impl(e, path, exact_columns != 0, threads); });
}

dsel_status dsel_read_block_row(dsel_engine* e, int j, double* host_row) {
  return guard(e, [&] {
    if (j < 0 || j >= e->nd) throw Fail{DSEL_E_RANGE, "block index out of range"};
    const int p = e->sensor_pos[j];
    if (p < 0 || p % e->G != e->rank) throw Fail{DSEL_E_RANGE, "block row not owned by this rank"};
    const int q = p / e->G;
    const size_t elems = (size_t)e->nd * e->nt * e->nt;
    la_flush(e);
    if (e->stream) {  // K itself, from the pinned host store
      const size_t n2 = (size_t)e->nt * e->nt;
      std::memset(host_row, 0, elems * sizeof(double));
      if (!e->hstore && !e->hk_user && e->kbf_fd < 0) throw Fail{DSEL_E_STATE, "no K loaded"};
      if (e->kbf_fd >= 0) {  // the file's block row j
        const size_t bsz = n2 * sizeof(double);
        for (int pk = 0; pk < e->nc; ++pk)
          pread_exact(e->kbf_fd, host_row + (size_t)e->pos_sensor[pk] * n2, bsz,
                      (off_t)(32 + ((size_t)j * e->nd + e->pos_sensor[pk]) * bsz), e->kbf_path);
        return;
      }
      if (e->hpacked && !e->hk_user) {  // K(p, pk): panel pk when p >= pk, else panel p transposed
        for (int pk = 0; pk < e->nc; ++pk) {
          double* dst = host_row + (size_t)e->pos_sensor[pk] * n2;
          if (p >= pk) {
            std::memcpy(dst, hpacked_block(e, pk, p), n2 * sizeof(double));
          } else {
            const double* src = hpacked_block(e, p, pk);  // K(pk, p) row-major
            for (int r = 0; r < e->nt; ++r)
              for (int c = 0; c < e->nt; ++c) dst[(size_t)r * e->nt + c] = src[(size_t)c * e->nt + r];
          }
        }
        return;
      }
      for (int pk = 0; pk < e->nc; ++pk)
        std::memcpy(host_row + (size_t)e->pos_sensor[pk] * n2,
                    e->hk_user ? e->hk_user + ((size_t)(e->hk_rows ? q : j) * e->nd + e->pos_sensor[pk]) * n2
                               : e->hstore + ((size_t)pk * e->nloc + q) * n2,
                    n2 * sizeof(double));
      return;
    }
    CU(cudaSetDevice(e->dev));
    ensure_stage(e, elems);
    CU(cudaMemsetAsync(e->stage, 0, elems * sizeof(double), e->s));
    const long long total = (long long)e->nc * e->nt * e->nt;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    if (e->sym && (e->G == 1 || !e->full_panels || !e->trace.empty())) {
      if (e->G != 1)
        throw Fail{DSEL_E_STATE, "read_block_row of a sharded symmetric store needs full panels "
                                 "and no rounds (or world_size 1)"};
      gather_block_row_sym_kernel<<<blocks, 256, 0, e->s>>>(e->geom(), p, e->d_pos_sensor, e->nc,
                                                            e->stage);
    } else {
      gather_block_row_kernel<<<blocks, 256, 0, e->s>>>(e->geom().panel(q), e->n,
                                                        e->nt, e->d_pos_sensor, e->nc, e->stage);
    }
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(e->h_stage, e->stage, elems * sizeof(double), cudaMemcpyDeviceToHost, e->s));
    CU(cudaStreamSynchronize(e->s));
    std::memcpy(host_row, e->h_stage, elems * sizeof(double));
  });
}

dsel_status dsel_gen_synthetic(dsel_engine* e, const double* v_host, int rank, double sigma) {
  return guard(e, [&] {
    if (rank < 1 || !v_host) throw Fail{DSEL_E_INVALID, "bad synthetic rank / V"};
    CU(cudaSetDevice(e->dev));
    const size_t vel = (size_t)e->nd * e->nt * rank;
    uint64_t dummy = 0;
    double* V = dmalloc<double>(vel, dummy);
    cudaError_t ce = cudaMemcpy(V, v_host, vel * sizeof(double), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess && e->nloc > 0 && !e->stream) {
      GenArgs g{};
      g.V = V;
      g.rank = rank;
      g.noise2 = sigma * sigma;  // kaccess.hpp:88
      g.nt = e->nt;
      g.row_sensor = e->d_pos_sensor;
      g.n_rows = (int)e->n;
      g.col_sensor = e->d_slot_sensor;
      g.n_cols = e->nloc * e->nt;
      g.geom = e->geom();
      g.q0 = 0;
      dim3 grid((g.n_rows + gen::BM - 1) / gen::BM, (g.n_cols + gen::BN - 1) / gen::BN);
      synth_panel_kernel<<<grid, gen::THREADS, 0, e->s>>>(g);
      ce = cudaGetLastError();
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->s);
    } else if (ce == cudaSuccess && e->nloc > 0) {
      // streaming store: one own panel at a time on the device, repacked to
      // [position][nt][nt] and copied into its slot of the pinned host store
      const size_t n2 = (size_t)e->nt * e->nt;
      ensure_hstore(e);
      double* panel = nullptr;
      double* packed = nullptr;
      ce = ds_malloc(&panel, sizeof(double) * (size_t)e->n * e->nt);
      if (ce == cudaSuccess) ce = ds_malloc(&packed, sizeof(double) * (size_t)e->nc * n2);
      for (int q = 0; q < e->nloc && ce == cudaSuccess; ++q) {
        GenArgs g{};
        g.V = V;
        g.rank = rank;
        g.noise2 = sigma * sigma;
        g.nt = e->nt;
        g.row_sensor = e->d_pos_sensor;
        g.n_rows = (int)e->n;
        g.col_sensor = e->d_slot_sensor + q;
        g.n_cols = e->nt;
        g.geom = PanelGeom{panel, e->n, e->nt, 1, 0, 0};  // one full-height temporary panel
        g.q0 = 0;
        dim3 grid((g.n_rows + gen::BM - 1) / gen::BM, (g.n_cols + gen::BN - 1) / gen::BN);
        synth_panel_kernel<<<grid, gen::THREADS, 0, e->s>>>(g);
        ce = cudaGetLastError();
        if (ce == cudaSuccess) ce = store_panel_d2h(e, panel, e->n, q, packed);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->s);
      }
      if (panel) cudaFree(panel);
      if (packed) cudaFree(packed);
    }
    cudaFree(V);
    if (ce != cudaSuccess) throw Fail{DSEL_E_CUDA, std::string("synthetic K: ") + cudaGetErrorString(ce)};
    e->full_panels = !e->packed;
    if (e->keep && e->C)
      CU(cudaMemcpyAsync(e->K0, e->C, sizeof(double) * e->c_elems, cudaMemcpyDeviceToDevice, e->s));
    CU(cudaStreamSynchronize(e->s));
  });
}

static void reset_state(dsel_engine* e);

// Device-formed synthetic K into the streaming (host) store: chunks of this
// rank's panels are accumulated on the device by the update kernel (W = +V,
// the same Philox V and per-element order as the HBM path, so the same bits)
// and copied to the pinned store -- the packed store needs only the
// block-lower tiles. K never has to fit in HBM (north star (1) at C5 scale).
void gen_device_stream(dsel_engine* e, int vrank, double sigma, uint64_t seed) {
  Nvtx nv("gen_synthetic_device (host store)");
  const int nt = e->nt;
  reset_state(e);  // every candidate live: compact row index = position
  ensure_hstore(e);
  const int R = e->n_rows_tab, n_rows = R * nt;
  const size_t n2 = (size_t)nt * nt, panel = (size_t)e->n * nt;
  constexpr int kch = 512;  // rank columns per update launch
  const int mpad = round_up(std::max(n_rows, 1), ws::ROW_PAD);
  size_t free_b = 0, total_b = 0;
  CU(cudaMemGetInfo(&free_b, &total_b));
  const size_t fixed = ((size_t)mpad * kch + (size_t)e->nc * n2) * sizeof(double) + (4ull << 30);
  const size_t room = free_b > fixed ? free_b - fixed : 0;
  const int cp = (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(e->nloc, 1), room / (panel * sizeof(double))));
  DevScratch<double> chunk((size_t)cp * panel), vt((size_t)mpad * kch), packed((size_t)e->nc * n2);
  const bool sym = e->hpacked;  // the packed store keeps the block-lower half only
  const int br = e->ws_br;
  const int nct_max = (cp * nt + ws::BC - 1) / ws::BC;
  const int ng_max = (nct_max + e->ws_group - 1) / e->ws_group;
  std::vector<int> h_tabs(2 * (size_t)cp + nct_max + ng_max + 1);
  DevScratch<int> d_tabs(h_tabs.size());
  const int nrt = (n_rows + br - 1) / br;
  for (int q0 = 0; q0 < e->nloc; q0 += cp) {
    const int c = std::min(cp, e->nloc - q0), n_cols = c * nt;
    int* cs = h_tabs.data();
    int* cg = cs + cp;
    for (int h = 0; h < c; ++h) {
      cs[h] = h;                          // slot inside the chunk buffer
      cg[h] = (q0 + h) * e->G + e->rank;  // compact row block = position (all live)
    }
    const int nct = (n_cols + ws::BC - 1) / ws::BC, ng = (nct + e->ws_group - 1) / e->ws_group;
    int* fr = cg + cp;
    int* gp = fr + nct_max;
    int sym_tiles = 0;
    if (sym) {  // block-lower tile schedule of the chunk (sym_tables)
      for (int ct = 0; ct < nct; ++ct) fr[ct] = (cg[(ct * ws::BC) / nt] * nt) / br;
      gp[0] = 0;
      for (int g = 0; g < ng; ++g) {
        const int ct0 = g * e->ws_group, gw = std::min(e->ws_group, nct - ct0);
        gp[g + 1] = gp[g] + (nrt - fr[ct0]) * gw;
      }
      sym_tiles = gp[ng];
    }
    CU(cudaMemcpy(d_tabs.p, h_tabs.data(), sizeof(int) * h_tabs.size(), cudaMemcpyHostToDevice));
    const PanelGeom g{chunk.p, e->n, nt, e->G, e->rank, 0};
    CU(cudaMemsetAsync(chunk.p, 0, sizeof(double) * (size_t)c * panel, e->s));
    add_diag_kernel<<<(unsigned)std::min<long long>(((long long)c * nt + 255) / 256, 1024), 256, 0, e->s>>>(
        g, c, sigma * sigma, q0);
    CU(cudaGetLastError());
    for (int k0 = 0; k0 < vrank; k0 += kch) {
      const long long total = (long long)mpad * (kch / 2);
      gen_v_tiled_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 32), 256, 0, e->s>>>(
          vt.p, mpad, kch, k0, vrank, e->row_pos(), e->d_pos_sensor, n_rows, nt, (unsigned long long)seed);
      UpdateWSArgs ua{};
      ua.C = chunk.p;
      ua.geom = g;
      ua.Wt = vt.p;
      ua.Wnt = vt.p;
      ua.mpad = mpad;
      ua.n_k = kch / ws::KC;
      ua.row_pos = e->row_pos();
      ua.col_slot = d_tabs.p;
      ua.col_g = d_tabs.p + cp;
      ua.nt = nt;
      ua.n_rows = n_rows;
      ua.n_cols = n_cols;
      ua.n_row_tiles = nrt;
      ua.n_col_tiles = nct;
      ua.group = e->ws_group;
      ua.sym = sym;
      ua.first_rt = d_tabs.p + 2 * cp;
      ua.gprefix = d_tabs.p + 2 * cp + nct_max;
      ua.n_groups = ng;
      ua.n_tiles = sym ? sym_tiles : nrt * nct;
      ua.n_full = ua.n_tiles;
      ua.split_s = 1;
      launch_ws(e, ua, gen_cfg(e, ua.n_k));
    }
    for (int h = 0; h < c; ++h) CU(store_panel_d2h(e, chunk.p + (size_t)h * panel, e->n, q0 + h, packed.p));
    CU(cudaStreamSynchronize(e->s));
  }
  e->full_panels = true;
}

dsel_status dsel_gen_synthetic_device(dsel_engine* e, int rank, double sigma, uint64_t seed) {
  return guard(e, [&] {
    if (rank < 1) throw Fail{DSEL_E_INVALID, "bad synthetic rank"};
    if (e->nt % 2) throw Fail{DSEL_E_INVALID, "gen_synthetic_device needs an even n_steps"};
    if (e->stream) {
      CU(cudaSetDevice(e->dev));
      gen_device_stream(e, rank, sigma, seed);
      return;
    }
    if (e->nt % 2) throw Fail{DSEL_E_INVALID, "gen_synthetic_device needs an even n_steps"};
    CU(cudaSetDevice(e->dev));
    const int nt = e->nt;
    reset_state(e);  // K is rewritten whole: a new selection starts
    const int R = e->n_rows_tab, Rl = e->n_cols_tab;
    const int n_rows = R * nt, n_cols = Rl * nt;
    const bool sym = e->sym;
    if (sym) sym_tables(e);
    CU(cudaMemsetAsync(e->C, 0, sizeof(double) * e->c_elems, e->s));
    if (e->nloc > 0) {
      const long long total = (long long)e->nloc * nt;
      add_diag_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 1024), 256, 0, e->s>>>(
          e->geom(), e->nloc, sigma * sigma);
      CU(cudaGetLastError());
    }
    constexpr int kch = 512;  // rank columns per update launch
    const int mpad = round_up(std::max(n_rows, 1), ws::ROW_PAD);
    DevScratch<double> vt_buf((size_t)mpad * kch);
    double* Vt = vt_buf.p;
    cudaError_t ce = cudaSuccess;
    double gen_flops = 0.0;
    for (int k0 = 0; k0 < rank && ce == cudaSuccess && Rl > 0; k0 += kch) {
      const long long total = (long long)mpad * (kch / 2);
      gen_v_tiled_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 32), 256, 0, e->s>>>(
          Vt, mpad, kch, k0, rank, e->row_pos(), e->d_pos_sensor, n_rows, nt, (unsigned long long)seed);
      // C += V V^T: the update kernel with W = +V on both sides
      UpdateWSArgs ua{};
      ua.C = e->C;
      ua.geom = e->geom();
      ua.Wt = Vt;
      ua.Wnt = Vt;
      ua.mpad = mpad;
      ua.n_k = kch / ws::KC;
      ua.row_pos = e->row_pos();
      ua.col_slot = e->col_slot();
      ua.col_g = e->col_g();
      ua.nt = nt;
      ua.n_rows = n_rows;
      ua.n_cols = n_cols;
      ua.n_row_tiles = (n_rows + e->ws_br - 1) / e->ws_br;
      ua.n_col_tiles = (n_cols + ws::BC - 1) / ws::BC;
      ua.group = e->ws_group;
      ua.sym = sym;
      ua.first_rt = e->d_sym;
      ua.gprefix = sym ? e->d_sym + ua.n_col_tiles : nullptr;
      ua.n_groups = (ua.n_col_tiles + e->ws_group - 1) / e->ws_group;
      ua.n_tiles = sym ? e->sym_tiles : ua.n_row_tiles * ua.n_col_tiles;
      ua.n_full = ua.n_tiles;
      ua.split_s = 1;
      launch_ws(e, ua, gen_cfg(e, ua.n_k));
      ce = cudaGetLastError();
      gen_flops += 2.0 * kch * (sym ? 0.5 * (double)n_rows * (n_cols + nt) : (double)n_rows * n_cols);
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->s);
    if (ce != cudaSuccess) throw Fail{DSEL_E_CUDA, std::string("device synthetic K: ") + cudaGetErrorString(ce)};
    e->gen_flops = gen_flops;
    e->full_panels = !sym;
    if (e->keep && e->C)
      CU(cudaMemcpyAsync(e->K0, e->C, sizeof(double) * e->c_elems, cudaMemcpyDeviceToDevice, e->s));
    CU(cudaStreamSynchronize(e->s));
  });
}

// ---- K formation from an LTI wave problem ------------ //
struct LtiOwner {
  LtiHost h;
};

dsel_status dsel_lti_from_config(const char* path, dsel_lti* out, void** owner) {
  return guard(nullptr, [&] {
    if (!path || !out || !owner) throw Fail{DSEL_E_INVALID, "null argument"};
    auto* o = new LtiOwner();
    std::string err;
    const int rc = lti_from_config(path, o->h, err);
    if (rc != 0) {
      delete o;
      throw Fail{rc == 7 ? DSEL_E_IO : DSEL_E_INVALID, err};
    }
    out->n_params = o->h.n_params;
    out->n_sensors = o->h.n_sensors;
    out->n_steps = o->h.n_steps;
    out->noise_sigma = o->h.noise_sigma;
    out->impulse = o->h.impulse.data();
    out->spatial = o->h.spatial.data();
    out->mask = o->h.mask.empty() ? nullptr : o->h.mask.data();
    out->cost_weights = o->h.cost.empty() ? nullptr : o->h.cost.data();
    *owner = o;
  });
}

void dsel_lti_free(void* owner) { delete static_cast<LtiOwner*>(owner); }

dsel_status dsel_assemble_lti(dsel_engine* e, const dsel_lti* lp, double* noise_logdets) {
  return guard(e, [&] {
    if (!lp || !lp->impulse || !lp->spatial) throw Fail{DSEL_E_INVALID, "null LTI problem"};
    if (lp->n_sensors != e->nd || lp->n_steps != e->nt)
      throw Fail{DSEL_E_INVALID, "LTI problem dimensions differ from the engine's"};
    if (lp->n_params < 1 || !(lp->noise_sigma > 0.0)) throw Fail{DSEL_E_INVALID, "bad LTI problem"};
    if (e->stream) throw Fail{DSEL_E_INVALID, "assemble_lti fills the HBM panel store"};
    CU(cudaSetDevice(e->dev));
    const int nd = e->nd, nt = e->nt, nm = lp->n_params;
    const size_t n = (size_t)nd * nt;
    const double gamma2 = lp->noise_sigma * lp->noise_sigma;
    if (noise_logdets)  // noise_block_logdets (hessian.hpp:149-154)
      for (int i = 0; i < nd; ++i)
        noise_logdets[i] = nt * std::log((lp->cost_weights ? lp->cost_weights[i] : 1.0) * gamma2);
    reset_state(e);
    const size_t nh = (size_t)nd * nm * nt, ns = (size_t)nm * nm, nmask = lp->mask ? (size_t)nm * nt : 0;
    const size_t nvf = n * nm * nt, np1 = (size_t)nt * nd * nt, np2 = n * nt;
    DevScratch<double> scratch(nh + ns + nmask + nvf + np1 + np2);
    double* buf = scratch.p;
    double *h = buf, *sp = h + nh, *mk = lp->mask ? sp + ns : nullptr, *vf = sp + ns + nmask,
           *p1 = vf + nvf, *p2 = p1 + np1;
    cudaError_t ce = cudaMemcpyAsync(h, lp->impulse, sizeof(double) * nh, cudaMemcpyHostToDevice, e->s);
    if (ce == cudaSuccess)
      ce = cudaMemcpyAsync(sp, lp->spatial, sizeof(double) * ns, cudaMemcpyHostToDevice, e->s);
    if (ce == cudaSuccess && mk)
      ce = cudaMemcpyAsync(mk, lp->mask, sizeof(double) * nmask, cudaMemcpyHostToDevice, e->s);
    auto grid = [](long long total) { return (unsigned)std::min<long long>((total + 255) / 256, 148 * 64); };
    if (ce == cudaSuccess) {  // the prior field of every column
      lti_field_kernel<<<grid((long long)nvf), 256, 0, e->s>>>(h, sp, mk, nm, nt, 0, (int)n, vf);
      ce = cudaGetLastError();
    }
    for (int q = 0; q < e->nloc && ce == cudaSuccess; ++q) {
      const int js = e->slot_sensor[q];
      lti_response_kernel<<<grid((long long)np1), 256, 0, e->s>>>(h, vf, 0, nm, nt, js * nt, nt, 0, nd, p1);
      lti_response_kernel<<<grid((long long)np2), 256, 0, e->s>>>(h, vf, 0, nm, nt, 0, (int)n, js, 1, p2);
      const double wc = lp->cost_weights ? lp->cost_weights[js] : 1.0;
      lti_panel_kernel<<<grid((long long)e->nc * nt * nt), 256, 0, e->s>>>(
          p1, p2, nd, nt, js, wc * gamma2, e->d_pos_sensor, e->nc, e->geom().panel(q), e->geom().ld(q),
          e->geom().start(q));
      ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->s);
    if (ce != cudaSuccess) throw Fail{DSEL_E_CUDA, std::string("assemble_lti: ") + cudaGetErrorString(ce)};
    e->full_panels = !e->packed;
    if (e->keep && e->C)
      CU(cudaMemcpyAsync(e->K0, e->C, sizeof(double) * e->c_elems, cudaMemcpyDeviceToDevice, e->s));
    CU(cudaStreamSynchronize(e->s));
  });
}

dsel_status dsel_step(dsel_engine* e, dsel_step_info* info) {
  return guard(e, [&] { step_impl(e, -1, info); });
}

dsel_status dsel_step_forced(dsel_engine* e, int sensor, dsel_step_info* info) {
  return guard(e, [&] {
    if (sensor < 0 || sensor >= e->nd || e->sensor_pos[sensor] < 0 ||
        !e->alive[e->sensor_pos[sensor]])
      throw Fail{DSEL_E_RANGE, "forced sensor is not a remaining candidate"};
    step_impl(e, sensor, info);
  });
}

dsel_status dsel_run(dsel_engine* e, int* n_done) {
  return guard(e, [&] {
    while (!e->finished && (int)e->chosen.size() < e->eff_budget) step_impl(e, -1, nullptr);
    if (n_done) *n_done = (int)e->chosen.size();
  });
}

dsel_status dsel_peek_gains(dsel_engine* e, double* gains_by_sensor) {
  return guard(e, [&] {
    CU(cudaSetDevice(e->dev));
    if (e->ll && e->chosen.empty()) ll_init_d(e);
    const int n_batch = e->n_cols_tab;
    run_gain(e, e->col_slot(), n_batch);
    std::vector<double> g(n_batch);
    std::vector<int> sens(n_batch);
    GainTabs t = gain_tabs(e);
    if (n_batch) {
      CU(cudaMemcpyAsync(g.data(), e->gains, sizeof(double) * n_batch, cudaMemcpyDeviceToHost, e->s));
      CU(cudaMemcpyAsync(sens.data(), t.sensor, sizeof(int) * n_batch, cudaMemcpyDeviceToHost, e->s));
    }
    CU(cudaStreamSynchronize(e->s));
    for (int i = 0; i < n_batch; ++i) gains_by_sensor[sens[i]] = g[i];
  });
}

int dsel_get_trace(dsel_engine* e, dsel_step_info* rows, int max_rows) {
  if (!e) return -1;
  try {
    CU(cudaSetDevice(e->dev));
    CU(cudaStreamSynchronize(e->s));
    if (e->s2) CU(cudaStreamSynchronize(e->s2));
    const int n = std::min<int>((int)e->trace.size(), max_rows);
    for (int i = 0; i < n; ++i) {
      dsel_step_info r = e->trace[i];
      cudaEvent_t* ev = &e->ev[(size_t)i * kEv];
      float a = 0, b = 0, c = 0, d = 0, tot = 0;
      CU(cudaEventElapsedTime(&a, ev[0], ev[1]));
      CU(cudaEventElapsedTime(&b, ev[1], ev[2]));
      CU(cudaEventElapsedTime(&c, ev[2], ev[3]));
      CU(cudaEventElapsedTime(&d, ev[3], ev[4]));
      CU(cudaEventElapsedTime(&tot, ev[0], ev[4]));
      r.ms_gain = a;
      r.ms_exchange = b;
      r.ms_panel = c;
      r.ms_update = d;
      if ((size_t)i < e->bulk_round.size() && e->bulk_round[i]) {  // the look-ahead bulk run in this step
        float bk = 0;
        CU(cudaEventElapsedTime(&bk, ev[8], ev[9]));
        r.ms_update += bk;
      }
      r.ms_round = tot;
      if (getenv("DSEL_TIMELINE")) {  // diagnostics: event offsets from round 1's start, ms
        float o[7] = {0, 0, 0, 0, 0, -1, -1};
        const int ids[7] = {0, 1, 2, 3, 4, 8, 9};
        const bool bulk = (size_t)i < e->bulk_round.size() && e->bulk_round[i];
        for (int j = 0; j < (bulk ? 7 : 5); ++j) CU(cudaEventElapsedTime(&o[j], e->ev[0], ev[ids[j]]));
        fprintf(stderr, "[tl] %d %d %.4f %.4f %.4f %.4f %.4f %.4f %.4f\n", e->rank, i, o[0], o[1], o[2], o[3],
                o[4], o[5], o[6]);
      }
      r.ms_io = 0.0;
      if (std::find(e->streamed_round.begin(), e->streamed_round.end(), i) != e->streamed_round.end()) {
        float io = 0;
        CU(cudaEventElapsedTime(&io, ev[5], ev[6]));  // streamed K blocks, copy stream
        r.ms_io = io;
      }
      rows[i] = r;
    }
    return n;
  } catch (const Fail& f) {
    e->err = f.msg;
    return -1;
  }
}

// selection state back to "nothing chosen" (the store is handled by the caller)
static void reset_state(dsel_engine* e) {
  if (e->s2) cudaStreamSynchronize(e->s2);
  e->prev_valid = false;
  e->bulk_pending[0] = e->bulk_pending[1] = false;
  e->bulk_round.clear();
  if (e->la) set_round_buf(e, 0);
  e->alive.assign(e->nc, 1);
  e->n_alive = e->nc;
  e->chosen.clear();
  e->trace.clear();
  e->objective = 0.0;
  e->finished = false;
  e->launches = 0;
  e->update_flops = 0.0;
  e->streamed_round.clear();
  e->h2d_bytes = e->d2h_bytes = e->nccl_bytes = 0;
  build_tables(e);
}

dsel_status dsel_reset(dsel_engine* e) {
  return guard(e, [&] {
    if (!e->keep && !e->ll) throw Fail{DSEL_E_STATE, "dsel_reset requires keep_pristine"};
    CU(cudaSetDevice(e->dev));
    if (e->s2) CU(cudaStreamSynchronize(e->s2));  // no bulk may still write C
    if (!e->ll)  // the left-looking store is K itself and is never modified
      CU(cudaMemcpyAsync(e->C, e->K0, sizeof(double) * e->c_elems, cudaMemcpyDeviceToDevice, e->s));
    reset_state(e);
    CU(cudaStreamSynchronize(e->s));
  });
}

dsel_status dsel_get_stats(dsel_engine* e, dsel_stats* st) {
  return guard(e, [&] {
    if (!st) throw Fail{DSEL_E_INVALID, "null stats"};
    CU(cudaSetDevice(e->dev));
    CU(cudaStreamSynchronize(e->s));
    if (e->s2) CU(cudaStreamSynchronize(e->s2));
    dsel_stats r{};
    r.rounds = (int)e->trace.size();
    r.kernel_launches = e->launches;
    r.h2d_bytes = e->h2d_bytes;
    r.d2h_bytes = e->d2h_bytes;
    r.nccl_bytes = e->nccl_bytes;
    r.update_flops = e->update_flops;
    for (int rd : e->streamed_round) {
      float io = 0, exposed = 0;
      const cudaEvent_t* ev = &e->ev[(size_t)rd * kEv];
      CU(cudaEventElapsedTime(&io, ev[5], ev[6]));
      CU(cudaEventElapsedTime(&exposed, ev[7], ev[6]));  // copy end after GEMM end -> exposed
      r.io_ms += io;
      r.io_exposed_ms += std::max(0.0f, exposed);
    }
    if (r.rounds > 0) {
      float ms = 0;
      // first gain launch -> winner of the last round on the host (its D2H)
      CU(cudaEventElapsedTime(&ms, e->ev[0], e->ev[(size_t)(r.rounds - 1) * kEv + 2]));
      r.time_to_k_ms = ms;
      double upd = 0.0;
      for (int i = 0; i < r.rounds; ++i) {
        float u = 0;
        CU(cudaEventElapsedTime(&u, e->ev[(size_t)i * kEv + 3], e->ev[(size_t)i * kEv + 4]));
        upd += u;
        if ((size_t)i < e->bulk_round.size() && e->bulk_round[i]) {
          CU(cudaEventElapsedTime(&u, e->ev[(size_t)i * kEv + 8], e->ev[(size_t)i * kEv + 9]));
          upd += u;
        }
      }
      r.update_ms = upd;
    }
    *st = r;
  });
}

namespace {
// Block row i of L_S (nt x (i+1)*nt, row-major) into the host staging buffer
// (collective: broadcast from the owner of the i-th chosen candidate).
void factor_row(dsel_engine* e, int i) {
  const int nt = e->nt;
  const long long n2 = (long long)nt * nt;
  const long long slot_stride = (long long)e->eff_budget * n2;
  const int p = e->sensor_pos[e->chosen[i]];
  const int owner = p % e->G, q = p / e->G;
  const long long total = n2 * (i + 1);
  ensure_stage(e, (size_t)total);
  if (owner == e->rank) {
    if (e->ll)
      ll_pack_factor_row_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 2048), 256, 0,
                                  e->s>>>(e->Wown, e->own_mpad, q * nt, nt, e->ldw, i + 1,
                                          e->ldiag + (size_t)i * n2, e->stage);
    else
      pack_factor_row_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 2048), 256, 0, e->s>>>(
          e->hist + q * slot_stride, nt, i + 1, e->stage);
    CU(cudaGetLastError());
  }
  if (e->G > 1) NC(ncclBroadcast(e->stage, e->stage, (size_t)total, ncclDouble, owner, e->comm, e->s));
  CU(cudaMemcpyAsync(e->h_stage, e->stage, sizeof(double) * total, cudaMemcpyDeviceToHost, e->s));
  CU(cudaStreamSynchronize(e->s));
}

void check_factor_export(dsel_engine* e) {
  if (!e->export_factor && !e->ll) throw Fail{DSEL_E_STATE, "engine created without export_factor"};
  CU(cudaSetDevice(e->dev));
}
}  // namespace

dsel_status dsel_export_factor(dsel_engine* e, double* host, int64_t ld) {
  return guard(e, [&] {
    check_factor_export(e);
    const int k = (int)e->chosen.size();
    const int nt = e->nt;
    if (ld < (int64_t)k * nt) throw Fail{DSEL_E_INVALID, "ld smaller than k*n_steps"};
    ensure_stage(e, (size_t)nt * std::max(k, 1) * nt);
    for (int i = 0; i < k; ++i) {
      factor_row(e, i);
      for (int a = 0; a < nt; ++a) {
        double* dst = host + ((int64_t)i * nt + a) * ld;
        std::memcpy(dst, e->h_stage + (size_t)a * (i + 1) * nt, sizeof(double) * (size_t)(i + 1) * nt);
        std::fill(dst + (size_t)(i + 1) * nt, dst + (size_t)k * nt, 0.0);
      }
    }
  });
}

dsel_status dsel_export_factor_row(dsel_engine* e, int i, double* host, int64_t ld) {
  return guard(e, [&] {
    check_factor_export(e);
    if (i < 0 || i >= (int)e->chosen.size()) throw Fail{DSEL_E_RANGE, "factor block row out of range"};
    const int nt = e->nt;
    if (ld < (int64_t)(i + 1) * nt) throw Fail{DSEL_E_INVALID, "ld smaller than (i+1)*n_steps"};
    factor_row(e, i);
    for (int a = 0; a < nt; ++a)
      std::memcpy(host + (int64_t)a * ld, e->h_stage + (size_t)a * (i + 1) * nt,
                  sizeof(double) * (size_t)(i + 1) * nt);
  });
}

}  // extern "C"
