// doptsel_gpu.hpp -- the B200 engine behind the reference C++ selection API.
//
// Header-only adapter for a maintainer's copy of the reference tree
// (proj/include/doptsel): include it AFTER "doptsel/parallel.hpp" and link
// libdsel.so. It returns exactly the reference types,
//
//   gpu_greedy_select<double>(k, candidates, budget, GpuOptions)
//       -> std::pair<SelectionState<double>, ParallelRunReport>
//
// so it is a drop-in for run_parallel_greedy<double> (parallel.hpp:281-483)
// and greedy_select<double> (selector.hpp:181-248):
//   * validation as the reference: check_candidates, budget >= 0,
//     require_noise_info (selector.hpp:142-151, :144-148, parallel.hpp:288-291);
//   * budget > |C| -> select all + warning (parallel.hpp:295-297);
//   * round 1 infeasible -> InfeasibleRound; later all-infeasible rounds ->
//     partial selection + warning (parallel.hpp:416-421);
//   * device / NCCL failures -> WorkerFailure(round, what) (parallel.hpp:469-475);
//   * K is read through KAccess::read_block as true block columns (i, s), the
//     blocks read_test_column reads (kaccess.hpp:27-35), so any KAccess works;
//   * SelectionState::factor is rebuilt from the engine's L_S with
//     append_block_column (linalg.hpp:159-178) and objective =
//     logdet_from_factor (parallel.hpp:432, :478-482);
//   * the optional round_hook of run_parallel_greedy (parallel.hpp:278-285,
//     :455-459) runs on the calling thread after every round, with the factor
//     as of that round (one pointer per GPU; every rank's replica is the same).
// One engine per GPU, driven by one host thread each (the reference's worker
// threads become GPUs); engines synchronise through NCCL. Every rank creates
// its engine before any rank enters NCCL (defer_connect), and a rank that
// fails mid-run aborts its peers (dsel_abort), so a failure surfaces as one
// WorkerFailure instead of a hang.
#pragma once

#include <algorithm>
#include <atomic>
#include <barrier>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "dsel.h"

namespace doptsel {

enum class GpuStorage { automatic = DSEL_STORAGE_AUTO, hbm = DSEL_STORAGE_HBM, stream = DSEL_STORAGE_STREAM };
enum class GpuAlgorithm { right_looking = 0, left_looking = 1 };

struct GpuOptions {
  int n_gpus = 1;                   // replaces ParallelOptions::n_workers
  std::vector<int> device_ids;      // default 0..n_gpus-1 (size must equal n_gpus when given)
  GpuStorage storage = GpuStorage::automatic;  // HBM when it fits hbm_budget, else streamed
  std::uint64_t hbm_budget = 0;     // bytes per GPU for the AUTO decision (0 = free memory - 2 GiB)
  GpuAlgorithm algorithm = GpuAlgorithm::right_looking;
  ObjectiveMode mode = ObjectiveMode::raw;
  std::vector<double> noise_logdets;
  double near_tie_tau = 1e-9;       // near-tie flag threshold (reported, never changes results)
  std::uint64_t seed = 0;           // accepted; the reference shuffle is result-invariant
};

struct GpuRoundExtra {              // per round, beside RoundResult
  int runner_up = -1;
  double runner_up_gain = 0.0;
  bool near_tie = false;
};

namespace gpu_detail {

[[noreturn]] inline void rethrow(dsel_status st, const std::string& msg, int round) {
  switch (st) {
    case DSEL_E_INVALID: throw InvalidConfig(msg);
    case DSEL_E_RANGE: throw IndexOutOfRange(msg);
    case DSEL_E_INFEASIBLE: throw InfeasibleRound(1);
    case DSEL_E_IO: throw IoError(msg);
    case DSEL_E_CORRUPT: throw CorruptFile(msg);
    default: throw WorkerFailure(round, msg);
  }
}

}  // namespace gpu_detail

template <class Real = double, KAccess A>
std::pair<SelectionState<Real>, ParallelRunReport> gpu_greedy_select(
    const A& k, std::span<const int> candidates, int budget, const GpuOptions& opts = {},
    std::vector<GpuRoundExtra>* extra = nullptr,
    const std::function<void(int, const std::vector<const LowerTriangularFactor<Real>*>&)>& round_hook = {}) {
  static_assert(std::is_same_v<Real, double>, "the B200 path computes in FP64");
  const int nt = k.n_steps();
  const int nd = k.n_sensors();
  detail::check_candidates(candidates, nd);
  if (budget < 0) throw InvalidConfig("budget must be nonnegative");
  if (opts.n_gpus < 1) throw InvalidConfig("n_gpus must be >= 1");
  if (!opts.device_ids.empty() && static_cast<int>(opts.device_ids.size()) != opts.n_gpus)
    throw InvalidConfig("device_ids must list one device per GPU (n_gpus)");
  SelectionOptions sel_opts{opts.mode, opts.noise_logdets};
  detail::require_noise_info(sel_opts, nd);

  ParallelRunReport report;
  if (budget > static_cast<int>(candidates.size()))
    report.trace.warning = "budget exceeds candidate count; selecting all candidates";
  const int eff = std::min<int>(budget, static_cast<int>(candidates.size()));
  SelectionState<Real> state(std::max(budget, 1), nt);
  if (eff == 0) return {std::move(state), std::move(report)};

  const int G = opts.n_gpus;
  std::vector<unsigned char> nid(128, 0);
  if (G > 1 && dsel_nccl_unique_id(nid.data()) != DSEL_OK)
    throw WorkerFailure(0, "ncclGetUniqueId failed");
  // candidate positions in ascending sensor order; owner = position % G
  std::vector<int> sorted(candidates.begin(), candidates.end());
  std::sort(sorted.begin(), sorted.end());

  struct Rank {
    dsel_status st = DSEL_OK;
    std::string err;
    int round = 0;
    bool aborted = false;  // failed only because a peer failed
    std::vector<dsel_step_info> rows;
    std::vector<double> factor;
  };
  std::vector<Rank> ranks(G);
  std::barrier<> sync(G);
  std::vector<char> failed(G, 0);
  std::vector<dsel_engine*> engines(G, nullptr);
  std::atomic<bool> any_failed{false};
  auto abort_peers = [&](int r) {  // a failing rank releases everyone blocked on it
    any_failed = true;
    for (int g = 0; g < G; ++g)
      if (g != r && engines[g]) dsel_abort(engines[g]);
  };
  // round hook (parallel.hpp:455-459): after each round rank 0 posts the new
  // factor block row and waits; the calling thread appends it, runs the hook
  // and acknowledges (the other ranks wait for rank 0 in the next collective)
  const bool hooked = static_cast<bool>(round_hook);
  std::mutex hook_mu;
  std::condition_variable hook_cv;
  struct HookPost {
    int round = 0;       // > 0: a finished round; 0: no post pending
    bool done = false;   // rank 0 stops posting
    std::vector<double> row;
  } post;
  bool acked = true, hook_failed = false;
  std::exception_ptr hook_error;
  auto post_round = [&](int round, std::vector<double> row, bool done) {
    std::unique_lock<std::mutex> lk(hook_mu);
    hook_cv.wait(lk, [&] { return acked; });
    post.round = round;
    post.done = done;
    post.row = std::move(row);
    acked = false;
    hook_cv.notify_all();
    if (!done) hook_cv.wait(lk, [&] { return acked; });
  };
  auto worker = [&](int r) {
    Rank& me = ranks[r];
    dsel_config cfg{};
    cfg.n_sensors = nd;
    cfg.n_steps = nt;
    cfg.budget = eff;
    cfg.n_candidates = static_cast<int>(sorted.size());
    cfg.candidates = sorted.data();
    cfg.device = opts.device_ids.empty() ? r : opts.device_ids[r];
    cfg.world_size = G;
    cfg.rank = r;
    cfg.nccl_id = nid.data();
    cfg.export_factor = 1;
    cfg.near_tie_tau = opts.near_tie_tau;
    cfg.storage = static_cast<int>(opts.storage);
    cfg.algorithm = static_cast<int>(opts.algorithm);
    if (opts.storage == GpuStorage::stream) cfg.algorithm = 1;  // streaming is left-looking
    cfg.hbm_budget = opts.hbm_budget;
    cfg.defer_connect = 1;
    dsel_engine* e = nullptr;
    me.st = dsel_create(&cfg, &e);
    if (me.st != DSEL_OK) me.err = dsel_last_error(nullptr);
    engines[r] = e;
    // panels owned by this rank: true block columns (i, s), i = 0..nd-1
    if (me.st == DSEL_OK) {
      try {
        std::vector<double> col(static_cast<std::size_t>(nd) * nt * nt);
        for (std::size_t p = r; p < sorted.size(); p += G) {
          const int s = sorted[p];
          for (int i = 0; i < nd; ++i)
            k.read_block(i, s, MatView<double>{col.data() + static_cast<std::size_t>(i) * nt * nt,
                                               nt, nt, nt});
          me.st = dsel_load_block_col(e, s, col.data());
          if (me.st != DSEL_OK) {
            me.err = dsel_last_error(e);
            break;
          }
        }
      } catch (const std::exception& ex) {
        me.st = DSEL_E_IO;
        me.err = ex.what();
      }
    }
    failed[r] = me.st != DSEL_OK;
    sync.arrive_and_wait();  // nobody enters a collective if any rank failed to create or load
    bool any = false;
    for (char f : failed) any = any || f;
    if (!any) {
      me.st = dsel_connect(e);  // NCCL init: every rank is known to be ready
      if (me.st != DSEL_OK) {
        me.err = dsel_last_error(e);
        abort_peers(r);
      }
      for (int round = 1; round <= eff && me.st == DSEL_OK; ++round) {
        dsel_step_info info{};
        me.round = round;
        me.st = dsel_step(e, &info);
        if (me.st != DSEL_OK) {
          me.err = dsel_last_error(e);
          me.aborted = any_failed.load();
          if (!me.aborted) abort_peers(r);
          break;
        }
        if (info.chosen_index < 0) break;
        if (hooked) {
          std::vector<double> row(static_cast<std::size_t>(nt) * round * nt);
          me.st = dsel_export_factor_row(e, round - 1, row.data(), static_cast<int64_t>(round) * nt);
          if (me.st != DSEL_OK) {
            me.err = dsel_last_error(e);
            me.aborted = any_failed.load();
            if (!me.aborted) abort_peers(r);
            break;
          }
          if (r == 0) {
            post_round(round, std::move(row), false);
            if (hook_failed) {  // the caller's hook threw: stop every rank
              abort_peers(r);
              break;
            }
          }
        }
      }
      if (me.st == DSEL_OK && !hook_failed) {
        me.rows.resize(eff);
        const int n = dsel_get_trace(e, me.rows.data(), eff);
        me.rows.resize(std::max(n, 0));
        int kk = 0;
        for (const auto& row : me.rows) kk += row.chosen_index >= 0;
        me.factor.assign(static_cast<std::size_t>(kk) * nt * kk * nt, 0.0);
        if (kk > 0) {
          me.st = dsel_export_factor(e, me.factor.data(), static_cast<int64_t>(kk) * nt);
          if (me.st != DSEL_OK) me.err = dsel_last_error(e);
        }
      }
    }
    if (r == 0 && hooked) post_round(0, {}, true);
    sync.arrive_and_wait();  // no engine is destroyed while a peer may still abort it
    if (e) dsel_destroy(e);
  };
  std::vector<std::thread> pool;
  for (int r = 0; r < G; ++r) pool.emplace_back(worker, r);
  if (hooked) {
    std::vector<const LowerTriangularFactor<Real>*> replicas(G, &state.factor);
    Matrix<Real> y(std::max(eff * nt, 1), nt), lm(nt, nt);
    for (;;) {
      std::unique_lock<std::mutex> lk(hook_mu);
      hook_cv.wait(lk, [&] { return !acked; });
      if (post.done) {
        acked = true;
        hook_cv.notify_all();
        break;
      }
      const int i = post.round - 1, kd = i * nt, ldr = post.round * nt;
      try {
        // block row i = [Y^T L_M] -> append_block_column (linalg.hpp:159-178)
        for (int a = 0; a < nt; ++a) {
          const double* src = post.row.data() + static_cast<std::size_t>(a) * ldr;
          for (int c = 0; c < kd; ++c) y(c, a) = src[c];
          for (int b = 0; b < nt; ++b) lm(a, b) = src[kd + b];
        }
        state.factor.append_block_column(ConstMatView<Real>{y.data(), kd, nt, nt}, lm.view());
        round_hook(post.round, replicas);
      } catch (...) {
        hook_error = std::current_exception();
        hook_failed = true;
      }
      acked = true;
      hook_cv.notify_all();
    }
  }
  for (auto& t : pool) t.join();
  if (hook_error) std::rethrow_exception(hook_error);
  // the original failure first; ranks that failed because a peer aborted them last
  for (const Rank& rk : ranks)
    if (rk.st != DSEL_OK && !rk.aborted) gpu_detail::rethrow(rk.st, rk.err, rk.round);
  for (const Rank& rk : ranks)
    if (rk.st != DSEL_OK) gpu_detail::rethrow(rk.st, rk.err, rk.round);

  const Rank& r0 = ranks[0];
  int kk = 0;
  for (const auto& row : r0.rows) {
    if (row.chosen_index < 0) {
      report.trace.warning = "no feasible candidates remain; returning partial selection";
      break;
    }
    ++kk;
  }
  // SelectionState: factor rebuilt block row by block row (append_block_column)
  const int ld = kk * nt;
  Matrix<Real> y(std::max(ld, 1), nt), lm(nt, nt);
  for (int i = 0; i < kk; ++i) {
    const int kd = i * nt;
    if (!hooked) {  // (the hook loop already appended every row, same bits)
      for (int a = 0; a < nt; ++a) {
        const double* src = r0.factor.data() + static_cast<std::size_t>(kd + a) * ld;
        for (int c = 0; c < kd; ++c) y(c, a) = src[c];
        for (int b = 0; b < nt; ++b) lm(a, b) = src[kd + b];
      }
      state.factor.append_block_column(ConstMatView<Real>{y.data(), kd, nt, nt}, lm.view());
    }
    state.chosen.push_back(r0.rows[i].chosen_index);
  }
  state.objective = kk > 0 ? logdet_from_factor(state.factor.active()) : 0.0;
  std::vector<int> prefix;
  for (int i = 0; i < kk; ++i) {
    const dsel_step_info& row = r0.rows[i];
    prefix.push_back(row.chosen_index);
    TraceRow t;
    t.k = row.k;
    t.chosen_index = row.chosen_index;
    t.objective = detail::reported_objective(row.objective, sel_opts, prefix);
    t.gain = opts.mode == ObjectiveMode::raw
                 ? row.gain
                 : row.gain - opts.noise_logdets[static_cast<std::size_t>(row.chosen_index)];
    t.n_evaluated = row.n_evaluated;
    t.n_infeasible = row.n_infeasible;
    t.wall_ms = row.ms_round;
    t.mean_candidate_ms = row.n_evaluated > 0 ? row.ms_round / row.n_evaluated : 0.0;
    report.trace.rows.push_back(t);
    RoundResult rr;
    rr.d_max = row.gain;
    rr.s_star = row.chosen_index;
    rr.bytes_exchanged = row.bytes_exchanged;
    for (int g = 0; g < G; ++g) {
      const dsel_step_info& rg = ranks[g].rows[i];
      WorkerTiming wt;
      wt.io_ms = rg.ms_io;  // H2D of streamed K blocks (0 when K is resident)
      wt.compute_ms = rg.ms_gain + rg.ms_exchange + rg.ms_panel + rg.ms_update;
      wt.wall_ms = rg.ms_round;
      const double busy = wt.io_ms + wt.compute_ms;
      wt.overlap = busy > 0.0 ? std::max(0.0, 1.0 - wt.wall_ms / busy) : 0.0;
      rr.workers.push_back(wt);
    }
    report.rounds.push_back(std::move(rr));
    if (extra) extra->push_back({row.runner_up, row.runner_up_gain, row.near_tie != 0});
  }
  return {std::move(state), std::move(report)};
}

}  // namespace doptsel
