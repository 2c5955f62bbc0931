// ref_harness.cpp -- C-callable harness around the UNMODIFIED reference
// library (header-only, /root/reference/proj/include/doptsel), compiled by
// oracle/Makefile into oracle/_ref/libdoptsel_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C restatement
// (oracle/dsel_oracle.c) and by bench.py's reference arm / cpu_baseline leg
// to time the reference CPU path. No reference source is copied here; this
// file only includes the reference headers and calls its public functions:
//   run_parallel_greedy   parallel.hpp:281-483  (the `doptsel select` path,
//                         proj/tools/doptsel_main.cpp:112-122)
//   greedy_select         selector.hpp:181-248
//   SyntheticKAccess      kaccess.hpp:81-124
//   random_hessian        proj/tests/support/generators.hpp:19-40
//   make_wave_problem / assemble_k / write_kbf / KStoreReader
//                         lti.hpp:159-171, hessian.hpp:91-144, kstore.hpp:69-186
//   detail::timed_round   bench.hpp:233-252 (one evaluation round)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "doptsel/bench.hpp"
#include "doptsel/config.hpp"
#include "doptsel/hessian.hpp"
#include "doptsel/kaccess.hpp"
#include "doptsel/kstore.hpp"
#include "doptsel/lti.hpp"
#include "doptsel/parallel.hpp"
#include "doptsel/selector.hpp"
#include "support/generators.hpp"

using namespace doptsel;

namespace {

thread_local std::string g_err;

// Error codes mirror proj/tools/doptsel_main.cpp:26-30 exit codes.
int map_exception() {
  try {
    throw;
  } catch (const InfeasibleRound& e) {
    g_err = e.what();
    return 2;
  } catch (const AllInfeasible& e) {
    g_err = e.what();
    return 2;
  } catch (const CorruptFile& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

DataSpaceHessian from_raw(const double* k, int nd, int nt) {
  DataSpaceHessian h(nd, nt);
  std::memcpy(h.raw(), k, h.raw_size() * sizeof(double));
  return h;
}

template <class Trace>
void emit_trace(const Trace& trace, int* chosen, double* gains, double* objectives, int* n_eval,
                int* n_inf, double* wall_ms, int* n_rows) {
  int i = 0;
  for (const TraceRow& r : trace.rows) {
    chosen[i] = r.chosen_index;
    gains[i] = r.gain;
    objectives[i] = r.objective;
    if (n_eval) n_eval[i] = r.n_evaluated;
    if (n_inf) n_inf[i] = r.n_infeasible;
    if (wall_ms) wall_ms[i] = r.wall_ms;
    ++i;
  }
  *n_rows = i;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// SyntheticKAccess(nd, nt, rank, sigma, seed) materialized block by block
// through its own read_block into block-row-major `out` (nd*nd*nt*nt f64).
int ref_synthetic_k(int nd, int nt, int rank, double sigma, std::uint64_t seed, double* out,
                    int threads) {
  try {
    const SyntheticKAccess syn(nd, nt, rank, sigma, seed);
    const std::size_t bsz = static_cast<std::size_t>(nt) * nt;
    std::vector<std::thread> pool;
    const int nthr = std::max(1, threads);
    for (int w = 0; w < nthr; ++w)
      pool.emplace_back([&, w] {
        for (int i = w; i < nd; i += nthr)
          for (int j = 0; j < nd; ++j)
            syn.read_block(i, j,
                           MatView<double>{out + (static_cast<std::size_t>(i) * nd + j) * bsz,
                                           nt, nt, nt});
      });
    for (auto& t : pool) t.join();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// testsupport::random_hessian (block-row-major out).
int ref_random_hessian(int nd, int nt, double gamma, int rank, std::uint64_t seed, double* out) {
  try {
    const DataSpaceHessian h = testsupport::random_hessian(nd, nt, gamma, rank, seed);
    std::memcpy(out, h.raw(), h.raw_size() * sizeof(double));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// run_parallel_greedy<double> on an in-memory DataSpaceHessian built from
// `k` -- the CLI's `select --mode schur` path. Outputs are sized >= budget.
// factor_out (optional) receives the (budget*nt)^2 factor storage.
// sel_wall_ms receives the wall time of run_parallel_greedy alone.
int ref_parallel_greedy(const double* k, int nd, int nt, const int* candidates, int n_cand,
                        int budget, int workers, std::uint64_t seed, int pipeline, int* chosen,
                        double* gains, double* objectives, int* n_eval, int* n_inf,
                        double* wall_ms, int* n_rows, double* factor_out, double* sel_wall_ms) {
  try {
    const DataSpaceHessian h = from_raw(k, nd, nt);
    ParallelOptions opts;
    opts.n_workers = workers;
    opts.pipeline = pipeline != 0;
    opts.seed = seed;
    const double t0 = detail::now_ms();
    auto [state, report] = run_parallel_greedy<double>(
        h, std::span<const int>(candidates, static_cast<std::size_t>(n_cand)), budget, opts);
    if (sel_wall_ms) *sel_wall_ms = detail::now_ms() - t0;
    emit_trace(report.trace, chosen, gains, objectives, n_eval, n_inf, wall_ms, n_rows);
    if (factor_out) {
      const auto& f = state.factor;
      const int cap = f.capacity_dim();
      const ConstMatView<double> act = f.active();
      for (int r = 0; r < f.active_dim(); ++r)
        for (int c = 0; c < f.active_dim(); ++c)
          factor_out[static_cast<std::size_t>(r) * cap + c] = act(r, c);
    }
    g_err = report.trace.warning;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// greedy_select<double> (sequential Alg. 1) on an in-memory Hessian.
int ref_greedy_select(const double* k, int nd, int nt, const int* candidates, int n_cand,
                      int budget, int* chosen, double* gains, double* objectives, int* n_eval,
                      int* n_inf, int* n_rows) {
  try {
    const DataSpaceHessian h = from_raw(k, nd, nt);
    auto [state, trace] = greedy_select<double>(
        h, std::span<const int>(candidates, static_cast<std::size_t>(n_cand)), budget);
    emit_trace(trace, chosen, gains, objectives, n_eval, n_inf, nullptr, n_rows);
    g_err = trace.warning;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Standard wave benchmark (proj/tests/support/generators.hpp:44-48) ->
// assemble_k -> write_kbf(path). noise_logdets (32 entries) from
// noise_block_logdets (hessian.hpp:149-154).
int ref_wave_kbf(const char* path, double* noise_logdets) {
  try {
    const LtiProblem p = testsupport::benchmark_problem(0);
    const DataSpaceHessian k = assemble_k(p);
    write_kbf(k, path);
    const std::vector<double> nl = noise_block_logdets(k);
    std::copy(nl.begin(), nl.end(), noise_logdets);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// `doptsel build <config> <out.kbf>` (doptsel_main.cpp:63-75): config ->
// problem_from_config -> weights_from_config -> assemble_k -> write_kbf.
// noise_logdets (n_sensors entries, may be null) from noise_block_logdets.
int ref_build_kbf(const char* config_path, const char* out_path, double* noise_logdets) {
  try {
    const ProblemConfig cfg = load_problem_config(config_path);
    const LtiProblem problem = problem_from_config(cfg);
    const WeightSpec weights = weights_from_config(cfg);
    const DataSpaceHessian k = assemble_k(problem, &weights);
    write_kbf(k, out_path);
    if (noise_logdets) {
      const std::vector<double> nl = noise_block_logdets(k);
      std::copy(nl.begin(), nl.end(), noise_logdets);
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Write an in-memory K as a KBF file through the reference writer.
int ref_write_kbf(const double* k, int nd, int nt, const char* path) {
  try {
    write_kbf(from_raw(k, nd, nt), path);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// run_parallel_greedy<double> on a KStoreReader (`doptsel select <kbf>`,
// doptsel_main.cpp:87-122) over all sensors.
int ref_kbf_select(const char* path, int budget, int workers, std::uint64_t seed, int* chosen,
                   double* gains, double* objectives, int* n_rows, int* nd_out, int* nt_out) {
  try {
    const KStoreReader store(path);
    *nd_out = store.n_sensors();
    *nt_out = store.n_steps();
    std::vector<int> cands(static_cast<std::size_t>(store.n_sensors()));
    for (int i = 0; i < store.n_sensors(); ++i) cands[static_cast<std::size_t>(i)] = i;
    ParallelOptions opts;
    opts.n_workers = workers;
    opts.seed = seed;
    auto [state, report] = run_parallel_greedy<double>(store, cands, budget, opts);
    emit_trace(report.trace, chosen, gains, objectives, nullptr, nullptr, nullptr, n_rows);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Bounded CPU sample: wall ms of ONE evaluation round (detail::timed_round,
// bench.hpp:233-252: W workers, pipelined, over all survivors) at each
// iterate in `iterates`, with the selection state at iterate k set to the
// Cholesky factor of K_S for the first k entries of `prefix`
// (LowerTriangularFactor::load_from_spd, linalg.hpp:187-196).
int ref_timed_rounds(const double* k, int nd, int nt, const int* prefix, int n_prefix,
                     const int* iterates, int n_iter, int workers, std::uint64_t seed,
                     double* round_ms, double* setup_ms) {
  try {
    const DataSpaceHessian h = from_raw(k, nd, nt);
    for (int q = 0; q < n_iter; ++q) {
      const int it = iterates[q];
      if (it < 0 || it > n_prefix) throw InvalidConfig("iterate beyond prefix");
      const double t0 = detail::now_ms();
      SelectionState<double> state(it + 1, nt);
      if (it > 0) {
        std::vector<int> s(prefix, prefix + it);
        Matrix<double> ks(it * nt, it * nt);
        materialize_principal(h, s, ks.view());
        state.factor.load_from_spd(ConstMatView<double>(ks.view()));
        state.chosen = s;
      }
      std::vector<int> survivors;
      for (int i = 0; i < nd; ++i)
        if (std::find(prefix, prefix + it, i) == prefix + it) survivors.push_back(i);
      Rng rng(seed);
      rng.shuffle(survivors);
      const WorkerPlan plan = make_worker_plan(survivors, workers);
      if (setup_ms) setup_ms[q] = detail::now_ms() - t0;
      round_ms[q] = detail::timed_round(h, state, plan, it + 1, true);
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Replay: raw gain of every sensor at every round along a GIVEN sequence,
// computed with score_candidate (selector.hpp:105-116) against a factor grown
// with append_block_column (linalg.hpp:159-178). gains_all: n_rounds x nd,
// NaN for already-chosen sensors, -inf for infeasible ones.
int ref_replay(const double* k, int nd, int nt, const int* sequence, int n_rounds,
               double* gains_all) {
  try {
    const DataSpaceHessian h = from_raw(k, nd, nt);
    SelectionState<double> state(std::max(n_rounds, 1), nt);
    CandidateWorkspace<double> ws(std::max(n_rounds, 1), nt);
    for (int round = 0; round < n_rounds; ++round) {
      for (int s = 0; s < nd; ++s) {
        double* g = gains_all + static_cast<std::size_t>(round) * nd + s;
        if (std::find(state.chosen.begin(), state.chosen.end(), s) != state.chosen.end()) {
          *g = std::numeric_limits<double>::quiet_NaN();
          continue;
        }
        try {
          *g = score_candidate(state, h, s, ws);
        } catch (const NotPositiveDefinite&) {
          *g = -std::numeric_limits<double>::infinity();
        }
      }
      const int s = sequence[round];
      score_candidate(state, h, s, ws);
      const int kd = state.factor.active_dim();
      state.factor.append_block_column(ConstMatView<double>(ws.y.top_rows(kd)), ws.m.view());
      state.chosen.push_back(s);
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
