/*
 * dsel_oracle.c -- CPU restatement of the reference greedy D-optimal selection
 * path (arXiv 2604.08812, reference `doptsel`, header-only C++20).
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The
 * product (paper_2604_08812_b200/, libdsel.so) never links or calls it.
 *
 * Parity is pinned (see tests/test_oracle.py): this restatement reproduces the
 * golden vectors produced by the reference itself compiled from
 * /root/reference (oracle/_ref/doptsel_ref, recipe oracle/Makefile), the
 * analytic known-answer tests of proj/tests/test_linalg.cpp and the survey's
 * recorded C1 sequence. Build flags are pinned to -O3 -ffp-contract=off so no
 * FMA contraction changes bits relative to the reference's Release build.
 *
 * Every function cites the reference file:line it follows; paths are relative
 * to /root/reference/proj/include/doptsel/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* rng.hpp:15-77 -- std::mt19937_64 plus hand-rolled transforms.             */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} orc_rng;

/* std::mt19937_64 as pinned by [rand.eng.mers] (rng.hpp:17 `gen_(seed)`). */
static void mt_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->spare = 0.0;
  r->have_spare = 0;
}

static uint64_t mt_next(orc_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:22 */
static double rng_uniform(orc_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:27-35 */
static int rng_uniform_int(orc_rng* r, int n) {
  const uint64_t bound = (uint64_t)n;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  uint64_t v;
  do {
    v = mt_next(r);
  } while (v >= limit);
  return (int)(v % bound);
}

/* rng.hpp:37-50 (Box-Muller with a cached spare) */
static double rng_normal(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_uniform(r);
  double u2 = rng_uniform(r);
  while (u1 <= 0.0) u1 = rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.141592653589793 * u2; /* std::numbers::pi */
  r->spare = rad * sin(a);
  r->have_spare = 1;
  return rad * cos(a);
}

/* rng.hpp:53-58 (Fisher-Yates) */
static void rng_shuffle_int(orc_rng* r, int* v, int n) {
  for (int i = n - 1; i > 0; --i) {
    const int j = rng_uniform_int(r, i + 1);
    int t = v[i];
    v[i] = v[j];
    v[j] = t;
  }
}

/* Exported RNG probes so tests can pin the stream against the reference. */
void orc_rng_normals(uint64_t seed, double* out, int64_t count) {
  orc_rng r;
  mt_seed(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_normal(&r);
}

void orc_rng_u64(uint64_t seed, uint64_t* out, int64_t count) {
  orc_rng r;
  mt_seed(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt_next(&r);
}

void orc_rng_shuffle(uint64_t seed, int* v, int n) {
  orc_rng r;
  mt_seed(&r, seed);
  rng_shuffle_int(&r, v, n);
}

/* ------------------------------------------------------------------------ */
/* Synthetic K: kaccess.hpp:81-124 (SyntheticKAccess).                       */
/* K = sigma^2 I + V V^T, V (n_sensors*n_steps) x rank row-major N(0,1).     */
/* ------------------------------------------------------------------------ */

/* kaccess.hpp:89-92: V filled in order by rng.normal(). */
void orc_synthetic_v(int n_sensors, int n_steps, int rank, uint64_t seed, double* v) {
  orc_rng r;
  mt_seed(&r, seed);
  const int64_t count = (int64_t)n_sensors * n_steps * rank;
  for (int64_t i = 0; i < count; ++i) v[i] = rng_normal(&r);
}

/* kaccess.hpp:98-116: block (i,j), row-major n_steps x n_steps into out. */
void orc_synthetic_block(const double* v, int n_steps, int rank, double noise2, int i, int j,
                         double* out, int out_stride) {
  const double* vi = v + (size_t)i * n_steps * rank;
  const double* vj = v + (size_t)j * n_steps * rank;
  for (int r = 0; r < n_steps; ++r) {
    const double* a = vi + (size_t)r * rank;
    double* o = out + (size_t)r * out_stride;
    for (int c = 0; c < n_steps; ++c) {
      const double* b = vj + (size_t)c * rank;
      double acc = 0.0;
      for (int t = 0; t < rank; ++t) acc += a[t] * b[t];
      o[c] = acc;
    }
    if (i == j) o[r] += noise2;
  }
}

/* DataSpaceHessian layout (hessian.hpp:17-84): block (i,j) at
 * (i*n_sensors + j) * n_steps^2, row-major inside. Rows [row0,row1) only so
 * callers can split the work across threads. */
void orc_synthetic_materialize_rows(const double* v, int n_sensors, int n_steps, int rank,
                                    double noise_sigma, int row0, int row1, double* k) {
  const double noise2 = noise_sigma * noise_sigma; /* kaccess.hpp:88 */
  const size_t bsz = (size_t)n_steps * n_steps;
  for (int i = row0; i < row1; ++i)
    for (int j = 0; j < n_sensors; ++j)
      orc_synthetic_block(v, n_steps, rank, noise2, i, j, k + ((size_t)i * n_sensors + j) * bsz,
                          n_steps);
}

/* The same K as orc_synthetic_materialize_rows, bit for bit, at golden-fixture
 * scale (C3 75x420 rank 24576, C4s 600x64): every element is still the
 * sequential sum over t of the rounded products a[t]*b[t] (kaccess.hpp:111,
 * built with -ffp-contract=off so mul and add round separately), with sigma^2
 * added last. Only the loop nest differs: the t loop is cut into chunks with
 * the output block itself as the running accumulator, and the c loop is
 * innermost over vt = V^T (rank x n), so the compiler vectorizes across
 * independent elements. Blocks j <= i are computed; (j,i) is the exact
 * transpose (a*b == b*a in IEEE, same summation order). Block row i of the
 * output is written for j <= i and block column i above the diagonal, so
 * threads owning distinct i never touch the same bytes. */
void orc_synthetic_block_rows_fast(const double* v, const double* vt, int n_sensors,
                                   int n_steps, int rank, double noise_sigma, int i,
                                   double* k) {
  const double noise2 = noise_sigma * noise_sigma;
  const size_t n = (size_t)n_sensors * n_steps;
  const size_t bsz = (size_t)n_steps * n_steps;
  const int tc = 64;
  for (int j = 0; j <= i; ++j) {
    double* o = k + ((size_t)i * n_sensors + j) * bsz;
    for (size_t e = 0; e < bsz; ++e) o[e] = 0.0;
    for (int t0 = 0; t0 < rank; t0 += tc) {
      const int t1 = t0 + tc < rank ? t0 + tc : rank;
      for (int r = 0; r < n_steps; ++r) {
        const double* a = v + ((size_t)i * n_steps + r) * rank;
        double* orow = o + (size_t)r * n_steps;
        for (int t = t0; t < t1; ++t) {
          const double at = a[t];
          const double* b = vt + (size_t)t * n + (size_t)j * n_steps;
          for (int c = 0; c < n_steps; ++c) orow[c] += at * b[c];
        }
      }
    }
    if (i == j)
      for (int r = 0; r < n_steps; ++r) o[(size_t)r * n_steps + r] += noise2;
    if (j != i) {
      double* m = k + ((size_t)j * n_sensors + i) * bsz;
      for (int r = 0; r < n_steps; ++r)
        for (int c = 0; c < n_steps; ++c) m[(size_t)c * n_steps + r] = o[(size_t)r * n_steps + c];
    }
  }
}

/* Same bits again, AVX2 register-blocked (4 rows x 8 columns of the block in
 * ymm accumulators, t chunked so the V / V^T panels stay in L1/L2). Separate
 * vmulpd + vaddpd per term (no FMA: the target attribute enables AVX2 only,
 * and -ffp-contract=off forbids contraction), sequential in t per element.
 * Needs n_steps % 4 == 0 (every BASELINE config); the caller checks the CPU. */
#if defined(__x86_64__)
#include <immintrin.h>
__attribute__((target("avx2"))) void orc_synthetic_block_rows_avx2(
    const double* v, const double* vt, int n_sensors, int n_steps, int rank, double noise_sigma,
    int i, double* k) {
  const double noise2 = noise_sigma * noise_sigma;
  const size_t n = (size_t)n_sensors * n_steps;
  const size_t bsz = (size_t)n_steps * n_steps;
  const int tc = 128, nt = n_steps;
  for (int j = 0; j <= i; ++j) {
    double* o = k + ((size_t)i * n_sensors + j) * bsz;
    for (size_t e = 0; e < bsz; ++e) o[e] = 0.0;
    for (int t0 = 0; t0 < rank; t0 += tc) {
      const int t1 = t0 + tc < rank ? t0 + tc : rank;
      for (int c0 = 0; c0 < nt; c0 += 8) {
        const int wide = c0 + 8 <= nt;
        const double* bcol = vt + (size_t)j * nt + c0;
        for (int r0 = 0; r0 < nt; r0 += 4) {
          const double* a0 = v + ((size_t)i * nt + r0) * rank;
          double* orow = o + (size_t)r0 * nt + c0;
          __m256d acc[4][2];
          for (int rr = 0; rr < 4; ++rr) {
            acc[rr][0] = _mm256_loadu_pd(orow + (size_t)rr * nt);
            acc[rr][1] = wide ? _mm256_loadu_pd(orow + (size_t)rr * nt + 4) : _mm256_setzero_pd();
          }
          if (wide) {
            for (int t = t0; t < t1; ++t) {
              const __m256d b0 = _mm256_loadu_pd(bcol + (size_t)t * n);
              const __m256d b1 = _mm256_loadu_pd(bcol + (size_t)t * n + 4);
              for (int rr = 0; rr < 4; ++rr) {
                const __m256d at = _mm256_broadcast_sd(a0 + (size_t)rr * rank + t);
                acc[rr][0] = _mm256_add_pd(acc[rr][0], _mm256_mul_pd(at, b0));
                acc[rr][1] = _mm256_add_pd(acc[rr][1], _mm256_mul_pd(at, b1));
              }
            }
          } else {
            for (int t = t0; t < t1; ++t) {
              const __m256d b0 = _mm256_loadu_pd(bcol + (size_t)t * n);
              for (int rr = 0; rr < 4; ++rr) {
                const __m256d at = _mm256_broadcast_sd(a0 + (size_t)rr * rank + t);
                acc[rr][0] = _mm256_add_pd(acc[rr][0], _mm256_mul_pd(at, b0));
              }
            }
          }
          for (int rr = 0; rr < 4; ++rr) {
            _mm256_storeu_pd(orow + (size_t)rr * nt, acc[rr][0]);
            if (wide) _mm256_storeu_pd(orow + (size_t)rr * nt + 4, acc[rr][1]);
          }
        }
      }
    }
    if (i == j)
      for (int r = 0; r < nt; ++r) o[(size_t)r * nt + r] += noise2;
    if (j != i) {
      double* m = k + ((size_t)j * n_sensors + i) * bsz;
      for (int r = 0; r < nt; ++r)
        for (int c = 0; c < nt; ++c) m[(size_t)c * nt + r] = o[(size_t)r * nt + c];
    }
  }
}
#endif

/* V of SyntheticKAccess in two passes for the large fixtures: the uniforms of
 * every Box-Muller pair are drawn sequentially (mt19937_64 order, with the
 * u1 <= 0 redraw of rng.hpp:46), then pairs are transformed independently --
 * the same libm calls on the same arguments as rng_normal, so the same bits.
 * v must hold an even number of doubles (>= count rounded up). */
void orc_synthetic_v_uniforms(uint64_t seed, double* v, int64_t count) {
  orc_rng r;
  mt_seed(&r, seed);
  for (int64_t p = 0; 2 * p < count; ++p) {
    double u1 = rng_uniform(&r);
    const double u2 = rng_uniform(&r);
    while (u1 <= 0.0) u1 = rng_uniform(&r);
    v[2 * p] = u1;
    v[2 * p + 1] = u2;
  }
}

void orc_box_muller_pairs(double* v, int64_t p0, int64_t p1) {
  for (int64_t p = p0; p < p1; ++p) {
    const double rad = sqrt(-2.0 * log(v[2 * p]));
    const double a = 2.0 * 3.141592653589793 * v[2 * p + 1];
    v[2 * p] = rad * cos(a);
    v[2 * p + 1] = rad * sin(a);
  }
}

/* proj/tests/support/generators.hpp:19-40 random_hessian. */
void orc_random_hessian(int n_sensors, int n_steps, double gamma, int rank, uint64_t seed,
                        double* k) {
  orc_rng r;
  mt_seed(&r, seed);
  const int dim = n_sensors * n_steps;
  double* g = (double*)malloc(sizeof(double) * (size_t)dim * rank);
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < rank; ++j) g[(size_t)i * rank + j] = rng_normal(&r);
  const size_t bsz = (size_t)n_steps * n_steps;
  for (int bi = 0; bi < n_sensors; ++bi)
    for (int bj = 0; bj < n_sensors; ++bj) {
      double* block = k + ((size_t)bi * n_sensors + bj) * bsz;
      for (int rr = 0; rr < n_steps; ++rr)
        for (int c = 0; c < n_steps; ++c) {
          double acc = 0.0;
          for (int t = 0; t < rank; ++t)
            acc += g[(size_t)(bi * n_steps + rr) * rank + t] *
                   g[(size_t)(bj * n_steps + c) * rank + t];
          block[rr * n_steps + c] = acc + (bi == bj && rr == c ? gamma * gamma : 0.0);
        }
    }
  free(g);
}

/* ------------------------------------------------------------------------ */
/* Dense kernels: linalg.hpp.                                                */
/* ------------------------------------------------------------------------ */

/* linalg.hpp:16-35. Returns -1 on success, else the failing pivot index. */
int orc_cholesky_in_place(double* a, int n, int stride) {
  for (int j = 0; j < n; ++j) {
    double* rj = a + (size_t)j * stride;
    double pivot = rj[j];
    for (int t = 0; t < j; ++t) pivot -= rj[t] * rj[t];
    if (!(pivot > 0.0) || !isfinite(pivot)) return j;
    const double diag = sqrt(pivot);
    rj[j] = diag;
    for (int i = j + 1; i < n; ++i) {
      double* ri = a + (size_t)i * stride;
      double acc = ri[j];
      for (int t = 0; t < j; ++t) acc -= ri[t] * rj[t];
      ri[j] = acc / diag;
    }
    for (int c = j + 1; c < n; ++c) rj[c] = 0.0;
  }
  return -1;
}

/* linalg.hpp:39-59. x is n x m row-major (stride xs). Returns -1 or the
 * index of a zero/nonfinite diagonal (SingularFactor). */
int orc_solve_lower_in_place(const double* l, int n, int ls, double* x, int m, int xs) {
  for (int r = 0; r < n; ++r) {
    const double* lr = l + (size_t)r * ls;
    double* xr = x + (size_t)r * xs;
    for (int t = 0; t < r; ++t) {
      const double c = lr[t];
      if (c != 0.0) {
        const double* xt = x + (size_t)t * xs;
        for (int j = 0; j < m; ++j) xr[j] -= c * xt[j];
      }
    }
    const double d = lr[r];
    if (d == 0.0 || !isfinite(d)) return r;
    for (int j = 0; j < m; ++j) xr[j] /= d;
  }
  return -1;
}

/* linalg.hpp:91-114 with out aliasing k_ss (the way score_from_buffers calls
 * it): M -= Y^T Y row by row of Y, then symmetrize by averaging. */
void orc_schur_in_place(double* m, int n, int ms, const double* y, int yrows, int ys) {
  for (int r = 0; r < yrows; ++r) {
    const double* yr = y + (size_t)r * ys;
    for (int a = 0; a < n; ++a) {
      const double ya = yr[a];
      double* oa = m + (size_t)a * ms;
      for (int b = 0; b < n; ++b) oa[b] -= ya * yr[b];
    }
  }
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b) {
      const double avg = (m[(size_t)a * ms + b] + m[(size_t)b * ms + a]) / 2.0;
      m[(size_t)a * ms + b] = avg;
      m[(size_t)b * ms + a] = avg;
    }
}

/* linalg.hpp:117-128. Returns NaN for a nonpositive/nonfinite diagonal. */
double orc_logdet_from_factor(const double* l, int n, int stride) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = l[(size_t)i * stride + i];
    if (!(d > 0.0) || !isfinite(d)) return NAN;
    acc += log(d);
  }
  return 2.0 * acc;
}

/* ------------------------------------------------------------------------ */
/* Selection: selector.hpp:86-248.                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  const double* k; /* DataSpaceHessian raw, block-row-major */
  int n_sensors, n_steps;
} orc_kview;

/* hessian.hpp:37-41 read_block -> copy block (i,j) into out (stride os). */
static void read_block(const orc_kview* kv, int i, int j, double* out, int os) {
  const int nt = kv->n_steps;
  const double* b = kv->k + ((size_t)i * kv->n_sensors + j) * (size_t)nt * nt;
  for (int r = 0; r < nt; ++r) memcpy(out + (size_t)r * os, b + (size_t)r * nt, sizeof(double) * nt);
}

/* selector.hpp:132-134 */
static int better_candidate(double d, int s, double best_d, int best_s) {
  return d > best_d || (d == best_d && (best_s < 0 || s < best_s));
}

/* Workspace for one candidate (selector.hpp:59-71). */
typedef struct {
  double* col; /* budget*nt x nt */
  double* m;   /* nt x nt */
} orc_ws;

/* selector.hpp:86-116 score_candidate / score_from_buffers. `l` is the
 * factor (stride ls) with active dimension kd. Returns 0 and *d on success,
 * 1 when M is not positive definite (candidate infeasible). */
static int score_candidate(const orc_kview* kv, const double* l, int ls, const int* chosen, int kc,
                           int s, orc_ws* ws, double* d) {
  const int nt = kv->n_steps;
  const int kd = kc * nt;
  /* kaccess.hpp:27-35 read_test_column: blocks (chosen[t], s) stacked */
  for (int t = 0; t < kc; ++t) read_block(kv, chosen[t], s, ws->col + (size_t)t * nt * nt, nt);
  read_block(kv, s, s, ws->m, nt);
  if (kd > 0) {
    if (orc_solve_lower_in_place(l, kd, ls, ws->col, nt, nt) >= 0) return 2;
    orc_schur_in_place(ws->m, nt, nt, ws->col, kd, nt);
  }
  if (orc_cholesky_in_place(ws->m, nt, nt) >= 0) return 1;
  *d = orc_logdet_from_factor(ws->m, nt, nt);
  return 0;
}

/* linalg.hpp:159-178 append_block_column: row block kc gets [Y^T, L_M]. */
static void append_block_column(double* l, int ls, int kc, int nt, const double* y,
                                const double* lm) {
  const int k = kc * nt;
  double* base = l + (size_t)k * ls;
  for (int a = 0; a < nt; ++a) {
    double* dst = base + (size_t)a * ls;
    for (int c = 0; c < k; ++c) dst[c] = y[(size_t)c * nt + a];
    for (int b = 0; b <= a; ++b) dst[k + b] = lm[(size_t)a * nt + b];
    for (int b = a + 1; b < nt; ++b) dst[k + b] = 0.0;
  }
}

/*
 * selector.hpp:181-248 greedy_select<double> (bitwise equal to
 * run_parallel_greedy at any worker count, proj/tests/test_parallel.cpp:94-124).
 *
 * k: block-row-major K. candidates: n_cand sensor ids in iteration order.
 * Outputs (length >= budget): chosen, gains (raw d_max), objectives
 * (logdet_from_factor of L_S, parallel.hpp:432), n_eval, n_infeasible.
 * factor_out (optional): (budget*nt)^2 row-major L_S, stride budget*nt.
 * gains_all (optional): budget x n_sensors matrix; entry [round][s] is the
 * raw gain of sensor s in that round (NaN if not evaluated / infeasible).
 * Returns the number of rounds completed; -1 if round 1 was infeasible
 * (InfeasibleRound), -2 on a singular factor, -3 on bad arguments.
 */
int orc_greedy_select(const double* k, int n_sensors, int n_steps, const int* candidates,
                      int n_cand, int budget, int* chosen, double* gains, double* objectives,
                      int* n_eval_out, int* n_infeasible_out, double* factor_out,
                      double* gains_all) {
  if (budget < 0 || n_steps < 1) return -3;
  const orc_kview kv = {k, n_sensors, n_steps};
  const int nt = n_steps;
  const int cap_blocks = budget > 1 ? budget : 1;
  const int ls = cap_blocks * nt;
  const int eff = budget < n_cand ? budget : n_cand;
  double* l = (double*)calloc((size_t)ls * ls, sizeof(double));
  orc_ws cur = {(double*)malloc(sizeof(double) * (size_t)ls * nt),
                (double*)malloc(sizeof(double) * (size_t)nt * nt)};
  orc_ws best = {(double*)malloc(sizeof(double) * (size_t)ls * nt),
                 (double*)malloc(sizeof(double) * (size_t)nt * nt)};
  int* remaining = (int*)malloc(sizeof(int) * (size_t)(n_cand > 0 ? n_cand : 1));
  memcpy(remaining, candidates, sizeof(int) * (size_t)n_cand);
  int n_rem = n_cand;
  int rounds = 0;
  int rc = 0;
  for (int round = 1; round <= eff; ++round) {
    double best_d = -INFINITY;
    int best_s = -1, n_eval = 0, n_inf = 0;
    for (int idx = 0; idx < n_rem; ++idx) {
      const int s = remaining[idx];
      ++n_eval;
      double d;
      const int st = score_candidate(&kv, l, ls, chosen, round - 1, s, &cur, &d);
      if (st == 2) {
        rc = -2;
        goto done;
      }
      if (st == 1) {
        ++n_inf;
        continue;
      }
      if (gains_all) gains_all[(size_t)(round - 1) * n_sensors + s] = d;
      if (better_candidate(d, s, best_d, best_s)) {
        best_d = d;
        best_s = s;
        orc_ws t = cur;
        cur = best;
        best = t;
      }
    }
    if (best_s < 0) {
      if (round == 1) rc = -1;
      goto done;
    }
    append_block_column(l, ls, round - 1, nt, best.col, best.m);
    chosen[round - 1] = best_s;
    gains[round - 1] = best_d;
    objectives[round - 1] = orc_logdet_from_factor(l, round * nt, ls);
    n_eval_out[round - 1] = n_eval;
    n_infeasible_out[round - 1] = n_inf;
    for (int idx = 0; idx < n_rem; ++idx)
      if (remaining[idx] == best_s) {
        memmove(remaining + idx, remaining + idx + 1, sizeof(int) * (size_t)(n_rem - idx - 1));
        --n_rem;
        break;
      }
    rounds = round;
  }
done:
  if (factor_out && rc == 0) memcpy(factor_out, l, sizeof(double) * (size_t)ls * ls);
  free(l);
  free(cur.col);
  free(cur.m);
  free(best.col);
  free(best.m);
  free(remaining);
  return rc < 0 ? rc : rounds;
}

/*
 * Replay: raw gains of every sensor at every round along a GIVEN chosen
 * sequence (the survey's "replay mode"), using the same
 * score_candidate path. gains_all is n_rounds x n_sensors; entries of already
 * chosen sensors are NaN, infeasible ones -inf.
 */
int orc_replay_gains(const double* k, int n_sensors, int n_steps, const int* sequence,
                     int n_rounds, double* gains_all) {
  const orc_kview kv = {k, n_sensors, n_steps};
  const int nt = n_steps;
  const int cap_blocks = n_rounds > 1 ? n_rounds : 1;
  const int ls = cap_blocks * nt;
  double* l = (double*)calloc((size_t)ls * ls, sizeof(double));
  orc_ws ws = {(double*)malloc(sizeof(double) * (size_t)ls * nt),
               (double*)malloc(sizeof(double) * (size_t)nt * nt)};
  char* taken = (char*)calloc((size_t)n_sensors, 1);
  int rc = 0;
  for (int round = 0; round < n_rounds; ++round) {
    for (int s = 0; s < n_sensors; ++s) {
      double* g = gains_all + (size_t)round * n_sensors + s;
      if (taken[s]) {
        *g = NAN;
        continue;
      }
      double d;
      const int st = score_candidate(&kv, l, ls, sequence, round, s, &ws, &d);
      *g = st == 0 ? d : -INFINITY;
    }
    const int s = sequence[round];
    double d;
    if (score_candidate(&kv, l, ls, sequence, round, s, &ws, &d) != 0) {
      rc = -1;
      break;
    }
    append_block_column(l, ls, round, nt, ws.col, ws.m);
    taken[s] = 1;
  }
  free(l);
  free(ws.col);
  free(ws.m);
  free(taken);
  return rc;
}

/* parallel.hpp:61-74 reduce_argmax over (gain, sensor) pairs. Returns the
 * index into the arrays of the winner, or -1 when all are infeasible (s<0). */
int orc_reduce_argmax(const double* d, const int* s, int n) {
  double best_d = -INFINITY;
  int best_s = -1, best_i = -1;
  for (int i = 0; i < n; ++i) {
    if (s[i] < 0) continue;
    if (better_candidate(d[i], s[i], best_d, best_s)) {
      best_d = d[i];
      best_s = s[i];
      best_i = i;
    }
  }
  return best_i;
}
