// Drop-in test: the reference's own types and KAccess sources driven through
// include/doptsel_gpu.hpp (libdsel.so), checked against the reference's
// run_parallel_greedy<double> in the same process. Built against the
// reference headers (/root/reference/proj/include) by __graft_entry__.build();
// run on a GPU by tests/test_cpp_dropin.py. Exit code = number of failures
// (like proj/tests/acceptance.cpp).
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <cstdio>
#include <cuda_runtime_api.h>
#include <string>
#include <vector>

#include "doptsel/hessian.hpp"
#include "doptsel/kaccess.hpp"
#include "doptsel/kstore.hpp"
#include "doptsel/parallel.hpp"
#include "doptsel/selector.hpp"
#include "doptsel_gpu.hpp"
#include "support/generators.hpp"

using namespace doptsel;

static int failures = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      ++failures;                                           \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
    } else {                                                \
      std::printf("PASS %s\n", what);                       \
    }                                                       \
  } while (0)

static bool close(double a, double b) { return std::fabs(a - b) <= 1e-9 * std::max(std::fabs(b), 1.0); }

template <KAccess A>
static void compare(const char* name, const A& k, int budget, const std::vector<int>& cands,
                    int n_gpus) {
  ParallelOptions po;
  po.n_workers = 4;
  auto [rs, rr] = run_parallel_greedy<double>(k, cands, budget, po);
  GpuOptions go;
  go.n_gpus = n_gpus;
  auto [gs, gr] = gpu_greedy_select<double>(k, cands, budget, go);
  std::string n(name);
  CHECK(gs.chosen == rs.chosen, (n + ": chosen sequence identical").c_str());
  bool gains = gr.trace.rows.size() == rr.trace.rows.size();
  for (std::size_t i = 0; gains && i < rr.trace.rows.size(); ++i)
    gains = close(gr.trace.rows[i].gain, rr.trace.rows[i].gain) &&
            close(gr.trace.rows[i].objective, rr.trace.rows[i].objective) &&
            gr.trace.rows[i].n_evaluated == rr.trace.rows[i].n_evaluated;
  CHECK(gains, (n + ": gains/objectives within 1e-9, n_evaluated equal").c_str());
  CHECK(close(gs.objective, rs.objective), (n + ": SelectionState.objective").c_str());
  // factor reconstructs K_S
  const int dim = gs.factor.active_dim();
  ConstMatView<double> L = gs.factor.active();
  Matrix<double> ks(dim, dim);
  materialize_principal(k, gs.chosen, ks.view());
  double err = 0.0, scale = 1.0;
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j <= i; ++j) {
      double acc = 0.0;
      for (int t = 0; t <= j; ++t) acc += L(i, t) * L(j, t);
      err = std::max(err, std::fabs(acc - ks(i, j)));
      scale = std::max(scale, std::fabs(ks(i, j)));
    }
  CHECK(err <= 1e-9 * scale, (n + ": L_S L_S^T == K_S").c_str());
  CHECK(gr.trace.warning == rr.trace.warning, (n + ": warning text").c_str());
}

// run_parallel_greedy's round_hook (parallel.hpp:278-285, :455-459): the same
// per-round view of the factor through the adapter's hook
static void compare_hook(const SyntheticKAccess& k, int budget, int n_gpus) {
  struct Seen {
    int round, dim;
    double logdet;
  };
  std::vector<Seen> ref, gpu;
  ParallelOptions po;
  po.n_workers = 3;
  run_parallel_greedy<double>(k, testsupport::all_candidates(k.n_sensors()), budget, po,
                              [&](int round, const std::vector<const LowerTriangularFactor<double>*>& f) {
                                ref.push_back({round, f[0]->active_dim(), logdet_from_factor(f[0]->active())});
                              });
  GpuOptions go;
  go.n_gpus = n_gpus;
  std::vector<int> replicas;
  gpu_greedy_select<double>(k, testsupport::all_candidates(k.n_sensors()), budget, go, nullptr,
                            [&](int round, const std::vector<const LowerTriangularFactor<double>*>& f) {
                              gpu.push_back({round, f[0]->active_dim(), logdet_from_factor(f[0]->active())});
                              replicas.push_back(static_cast<int>(f.size()));
                            });
  bool same = ref.size() == gpu.size();
  for (std::size_t i = 0; same && i < ref.size(); ++i)
    same = ref[i].round == gpu[i].round && ref[i].dim == gpu[i].dim && close(gpu[i].logdet, ref[i].logdet);
  CHECK(same, ("round_hook: per-round factor (dim, logdet) on " + std::to_string(n_gpus) + " GPU(s)").c_str());
  bool reps = !replicas.empty();
  for (int r : replicas) reps = reps && r == n_gpus;
  CHECK(reps, "round_hook: one factor pointer per GPU");
  // a hook that throws stops the run and the exception reaches the caller
  bool threw = false;
  try {
    gpu_greedy_select<double>(k, testsupport::all_candidates(k.n_sensors()), budget, go, nullptr,
                              [&](int round, const std::vector<const LowerTriangularFactor<double>*>&) {
                                if (round == 2) throw std::runtime_error("hook stop");
                              });
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()) == "hook stop";
  }
  CHECK(threw, "round_hook: an exception thrown by the hook propagates");
}

// A rank failing mid-run (DSEL_FAULT="round,rank") aborts its peers: one
// WorkerFailure naming the injected fault, no hang (run under a timeout).
static int fault_test(int n_gpus) {
  setenv("DSEL_FAULT", "3,1", 1);
  const SyntheticKAccess syn(64, 32, 2048, 1.0, 2024);
  bool ok = false;
  try {
    GpuOptions go;
    go.n_gpus = n_gpus;
    gpu_greedy_select<double>(syn, testsupport::all_candidates(64), 16, go);
  } catch (const WorkerFailure& e) {
    ok = std::string(e.what()).find("injected fault") != std::string::npos;
    std::printf("WorkerFailure: %s\n", e.what());
  }
  unsetenv("DSEL_FAULT");
  CHECK(ok, "peer failure -> WorkerFailure, peers released");
  // the devices stay usable
  GpuOptions go;
  go.n_gpus = n_gpus;
  auto [gs, gr] = gpu_greedy_select<double>(syn, testsupport::all_candidates(64), 4, go);
  CHECK(gs.chosen.size() == 4, "engines usable after an aborted run");
  std::printf("%d failure(s)\n", failures);
  return failures;
}

int main(int argc, char** argv) {
  int ngpu = 0;
  cudaGetDeviceCount(&ngpu);
  if (argc > 1 && std::string(argv[1]) == "--fault") return fault_test(std::min(ngpu, 2));
  const std::string kbf = argc > 1 ? argv[1] : "tests/golden/wave.kbf";
  {
    const SyntheticKAccess syn(64, 32, 2048, 1.0, 2024);  // C1
    compare("C1 SyntheticKAccess", syn, 16, testsupport::all_candidates(64), 1);
  }
  {
    const KStoreReader store(kbf);  // wave benchmark through the on-disk store
    compare("wave KStoreReader", store, 12, testsupport::all_candidates(32), 1);
  }
  {
    const DataSpaceHessian k = testsupport::random_hessian(12, 3, 0.9, 36, 211);
    compare("random_hessian odd Nt", k, 7, {0, 2, 3, 5, 7, 8, 10, 11}, 1);
    compare("budget > |C|", k, 9, {1, 4, 6}, 1);
  }
  {
    // storage / algorithm options: the streaming store (left-looking, K in
    // host memory) and AUTO with a budget too small for the resident store
    const SyntheticKAccess syn(64, 32, 2048, 1.0, 2024);
    ParallelOptions po;
    po.n_workers = 4;
    auto [rs, rr] = run_parallel_greedy<double>(syn, testsupport::all_candidates(64), 16, po);
    for (int variant = 0; variant < 3; ++variant) {
      GpuOptions go;
      if (variant == 0) go.storage = GpuStorage::stream;
      if (variant == 1) go.algorithm = GpuAlgorithm::left_looking;
      if (variant == 2) go.hbm_budget = 20ull << 20;  // resident plan 26.3 MB, streaming 14.6 MB
      auto [gs, gr] = gpu_greedy_select<double>(syn, testsupport::all_candidates(64), 16, go);
      bool gains = gs.chosen == rs.chosen;
      for (std::size_t i = 0; gains && i < rr.trace.rows.size(); ++i)
        gains = close(gr.trace.rows[i].gain, rr.trace.rows[i].gain);
      const char* nm[] = {"storage=stream", "algorithm=left_looking", "AUTO over budget -> stream"};
      CHECK(gains, (std::string("C1 ") + nm[variant] + ": sequence + gains").c_str());
    }
    compare_hook(syn, 8, 1);
  }
  if (ngpu >= 2) {
    const SyntheticKAccess syn(64, 32, 2048, 1.0, 2024);
    compare("C1 on 2 GPUs", syn, 16, testsupport::all_candidates(64), 2);
    compare_hook(syn, 8, 2);
  }
  // reference error behaviour
  const DataSpaceHessian k = testsupport::random_hessian(6, 2, 1.0, 12, 3);
  bool threw = false;
  try {
    std::vector<int> dup{1, 1};
    gpu_greedy_select<double>(k, dup, 1);
  } catch (const InvalidConfig&) {
    threw = true;
  }
  CHECK(threw, "duplicate candidate -> InvalidConfig");
  threw = false;
  try {
    std::vector<int> bad{0, 9};
    gpu_greedy_select<double>(k, bad, 1);
  } catch (const IndexOutOfRange&) {
    threw = true;
  }
  CHECK(threw, "candidate out of range -> IndexOutOfRange");
  threw = false;
  try {
    DataSpaceHessian z(4, 2);
    gpu_greedy_select<double>(z, testsupport::all_candidates(4), 2);
  } catch (const InfeasibleRound& e) {
    threw = e.round == 1;
  }
  CHECK(threw, "all-zero K -> InfeasibleRound(1)");
  threw = false;
  try {
    GpuOptions o;
    o.mode = ObjectiveMode::normalized;
    gpu_greedy_select<double>(k, testsupport::all_candidates(6), 2, o);
  } catch (const InvalidConfig&) {
    threw = true;
  }
  CHECK(threw, "normalized without noise log-dets -> InvalidConfig");
  std::printf("%d failure(s)\n", failures);
  return failures;
}
