// doptsel -- drop-in `select` CLI over the B200 engine (include/dsel.h).
//
// Mirrors `doptsel select` of the reference (proj/tools/doptsel_main.cpp:
// flags :372-386, run_select :87-165, exit codes :26-30) with the same
// outputs: selection.json, trace.csv (trace_io.hpp:15-21) and timing.csv
// (trace_io.hpp:40-48, one row per round and GPU). CLI11/nlohmann are not
// available here, so flags and JSON are hand-rolled.
//
//   doptsel select <kbf> --budget B [--mode schur|gpu] [--gpus G] [--workers N]
//                  [--algorithm right|left] [--storage auto|hbm|stream]
//                  [--hbm-budget BYTES] [--seed S] [--pipeline on|off] [--precision f64]
//                  [--config cfg | --noise-logdets file] [--kbf-rows] [--out DIR]
//
// Extra output beside the reference's three files: near_ties.csv (k,
// chosen_index, gain, runner_up, runner_up_gain, rel_gap, near_tie) -- the
// top-2 gap of every round, flagged when (g1-g2)/max(|g1|,1) < 1e-9 (the
// reference tie rule, selector.hpp:132-134, decides exact ties only).
//   doptsel select --synthetic nd,nt,rank,sigma,seed --budget B ...
//   doptsel build <config> <out.kbf>     (doptsel_main.cpp:63-75; K on the GPU)
//
// --mode schur (the reference default) and gpu both run the GPU engine;
// naive (refactorizing baseline) and --precision f32 are CPU-only paths of the
// reference and are rejected. --workers is accepted (the reference's CPU
// worker count) and ignored. evaluate and bench are outside the hot path.
#include <algorithm>
#include <atomic>
#include <limits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <charconv>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "dsel.h"

namespace fs = std::filesystem;

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitInfeasible = 2, kExitIo = 3;

std::string num(double v) {
  if (std::isnan(v)) return "null";
  if (std::isinf(v)) return v > 0 ? "1e309" : "-1e309";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

std::string num17(double v) {  // std::ostream << setprecision(17)
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

struct SelectArgs {
  std::string kbf, out = ".", mode = "schur", precision = "f64", pipeline = "on", config,
                   noise_file, synthetic;
  int budget = -1, workers = 1, gpus = 1;
  std::string algorithm = "right", storage = "auto";
  unsigned long long seed = 0, hbm_budget = 0;
  bool kbf_rows = false;
};

std::vector<double> parse_list(const std::string& s) {
  std::vector<double> out;
  std::string item;
  std::stringstream ss(s);
  while (std::getline(ss, item, ',')) {
    size_t a = item.find_first_not_of(" \t\r\n"), b = item.find_last_not_of(" \t\r\n");
    if (a == std::string::npos) continue;
    out.push_back(std::stod(item.substr(a, b - a + 1)));
  }
  return out;
}

// noise_logdets_from_config (doptsel_main.cpp:47-59): the LTI problem of the
// config (dsel_lti_from_config -- the full wave model, so the default noise
// level 0.1 max|h| is honoured) gives gamma; n_steps * log(w_c gamma^2).
std::vector<double> noise_from_config(const std::string& path) {
  dsel_lti p{};
  void* owner = nullptr;
  const dsel_status st = dsel_lti_from_config(path.c_str(), &p, &owner);
  if (st != DSEL_OK)
    throw std::runtime_error(std::string(st == DSEL_E_IO ? "io:" : "usage:") + dsel_last_error(nullptr));
  std::vector<double> out(p.n_sensors);
  const double g2 = p.noise_sigma * p.noise_sigma;
  for (int i = 0; i < p.n_sensors; ++i)
    out[i] = p.n_steps * std::log((p.cost_weights ? p.cost_weights[i] : 1.0) * g2);
  dsel_lti_free(owner);
  return out;
}

// `doptsel build <config> <out.kbf>` (doptsel_main.cpp:63-75): K assembled on
// the GPU (dsel_assemble_lti, bit-identical to assemble_k), written as KBF.
int cmd_build(const std::string& config, const std::string& out_path) {
  dsel_lti p{};
  void* owner = nullptr;
  dsel_status st = dsel_lti_from_config(config.c_str(), &p, &owner);
  if (st != DSEL_OK) {
    std::cerr << "error: " << dsel_last_error(nullptr) << "\n";
    return st == DSEL_E_IO ? kExitIo : kExitUsage;
  }
  const int nd = p.n_sensors, nt = p.n_steps;
  dsel_config cfg{};
  cfg.n_sensors = nd;
  cfg.n_steps = nt;
  cfg.budget = 1;
  cfg.world_size = 1;
  cfg.full_square = 1;  // whole panels: every block row is read back
  cfg.algorithm = 1;
  dsel_engine* e = nullptr;
  st = dsel_create(&cfg, &e);
  std::vector<double> row((size_t)nd * nt * nt);
  std::FILE* f = nullptr;
  if (st == DSEL_OK) st = dsel_assemble_lti(e, &p, nullptr);
  dsel_lti_free(owner);
  if (st != DSEL_OK) {
    std::cerr << "error: " << dsel_last_error(e) << "\n";
    dsel_destroy(e);
    return kExitUsage;
  }
  f = std::fopen(out_path.c_str(), "wb");
  if (!f) {
    std::cerr << "error: cannot open " << out_path << " for writing\n";
    dsel_destroy(e);
    return kExitIo;
  }
  unsigned char h[32] = {'K', 'B', 'F', '1'};
  const unsigned fields[5] = {1u, (unsigned)nd, (unsigned)nt, 1u, 1u};
  for (int q = 0; q < 5; ++q)
    for (int b = 0; b < 4; ++b) h[4 + 4 * q + b] = (unsigned char)(fields[q] >> (8 * b));
  bool ok = std::fwrite(h, 1, 32, f) == 32;
  for (int j = 0; j < nd && ok; ++j) {
    st = dsel_read_block_row(e, j, row.data());
    ok = st == DSEL_OK && std::fwrite(row.data(), sizeof(double), row.size(), f) == row.size();
  }
  ok = (std::fclose(f) == 0) && ok;
  dsel_destroy(e);
  if (!ok) {
    std::cerr << "error: short write to " << out_path << "\n";
    return kExitIo;
  }
  std::cout << "wrote " << out_path << ": n_sensors=" << nd << " n_steps=" << nt
            << " bytes=" << 32ull + (unsigned long long)nd * nd * nt * nt * 8ull << "\n";
  return kExitOk;
}

struct RankResult {
  dsel_status st = DSEL_OK;
  bool aborted = false;  // stopped because a peer failed
  std::string err;
  std::vector<dsel_step_info> rows;
};

int run_select(const SelectArgs& a) {
  if (a.mode == "naive") {
    std::cerr << "error: --mode naive is the reference's CPU refactorizing baseline; this "
                 "build runs the GPU Schur path (--mode schur|gpu)\n";
    return kExitUsage;
  }
  if (a.precision != "f64") {
    std::cerr << "error: the GPU path computes in FP64 (--precision f64)\n";
    return kExitUsage;
  }
  int nd = 0, nt = 0, rank = 0;
  double sigma = 1.0;
  unsigned long long syn_seed = 0;
  if (!a.synthetic.empty()) {
    auto v = parse_list(a.synthetic);
    if (v.size() != 5) {
      std::cerr << "error: --synthetic expects nd,nt,rank,sigma,seed\n";
      return kExitUsage;
    }
    nd = (int)v[0], nt = (int)v[1], rank = (int)v[2], sigma = v[3],
    syn_seed = (unsigned long long)v[4];
  } else {
    std::FILE* f = std::fopen(a.kbf.c_str(), "rb");
    if (!f) {
      std::cerr << "error: cannot open " << a.kbf << "\n";
      return kExitIo;
    }
    unsigned char h[32];
    const size_t got = std::fread(h, 1, 32, f);
    std::fclose(f);
    if (got != 32 || std::memcmp(h, "KBF1", 4) != 0) {
      std::cerr << "error: " << a.kbf << ": not a KBF store (bad magic or truncated)\n";
      return kExitIo;
    }
    auto u32 = [&](int o) {
      return (unsigned)h[o] | (unsigned)h[o + 1] << 8 | (unsigned)h[o + 2] << 16 |
             (unsigned)h[o + 3] << 24;
    };
    nd = (int)u32(8);
    nt = (int)u32(12);
    // KStoreReader validation (kstore.hpp:92-125) before any device work
    std::error_code ec;
    const auto size = fs::file_size(a.kbf, ec);
    const unsigned long long expect = 32ull + (unsigned long long)nd * nd * nt * nt * 8ull;
    if (u32(4) != 1 || u32(16) != 1 || u32(20) != 1 || nd < 1 || nt < 1) {
      std::cerr << "error: " << a.kbf << ": unsupported header fields\n";
      return kExitIo;
    }
    if (ec || size != expect) {
      std::cerr << "error: " << a.kbf << ": size " << size << " != expected " << expect << "\n";
      return kExitIo;
    }
  }
  if (a.budget < 0 || a.budget > nd) {
    std::cerr << "budget must be within 0.." << nd << "\n";
    return kExitUsage;
  }
  std::vector<double> noise;
  try {
    if (!a.config.empty()) noise = noise_from_config(a.config);
    if (!a.noise_file.empty()) {
      std::ifstream in(a.noise_file);
      if (!in) throw std::runtime_error("io:cannot open " + a.noise_file);
      std::stringstream ss;
      ss << in.rdbuf();
      std::string s = ss.str();
      for (char& c : s)
        if (c == '\n') c = ',';
      noise = parse_list(s);
    }
  } catch (const std::exception& ex) {
    std::string m = ex.what();
    const bool io = m.rfind("io:", 0) == 0;
    std::cerr << "error: " << m.substr(m.find(':') + 1) << "\n";
    return io ? kExitIo : kExitUsage;
  }
  if (!noise.empty() && (int)noise.size() != nd) {
    std::cerr << "error: need one noise log-determinant per sensor (" << nd << ")\n";
    return kExitUsage;
  }

  // one engine per GPU, one host thread each; the engines synchronise through NCCL
  const int G = std::max(1, a.gpus);
  std::vector<unsigned char> nid(128, 0);
  if (G > 1 && dsel_nccl_unique_id(nid.data()) != DSEL_OK) {
    std::cerr << "error: NCCL unique id\n";
    return kExitIo;
  }
  std::vector<double> v;
  if (!a.synthetic.empty() && a.budget > 0) {
    v.resize((size_t)nd * nt * rank);
    dsel_synthetic_v(nd, nt, rank, syn_seed, v.data(), 0);
  }
  std::vector<RankResult> res(G);
  std::vector<dsel_engine*> engines(G, nullptr);
  std::vector<char> created(G, 0);
  std::atomic<int> arrived{0};
  std::atomic<bool> failed{false};
  // every rank creates and loads before any rank enters NCCL; a rank failing
  // later aborts its peers (dsel_abort) instead of leaving them blocked
  auto wait_all = [&](int phase) {
    arrived.fetch_add(1);
    while (arrived.load() < phase * G) std::this_thread::yield();
  };
  auto abort_peers = [&](int r) {
    failed = true;
    for (int g = 0; g < G; ++g)
      if (g != r && engines[g]) dsel_abort(engines[g]);
  };
  auto worker = [&](int r) {
    RankResult& out = res[r];
    if (a.budget == 0) return;
    dsel_config cfg{};
    cfg.n_sensors = nd;
    cfg.n_steps = nt;
    cfg.budget = a.budget;
    cfg.device = r;
    cfg.world_size = G;
    cfg.rank = r;
    cfg.nccl_id = nid.data();
    cfg.near_tie_tau = 1e-9;
    cfg.algorithm = a.algorithm == "left" ? 1 : 0;
    cfg.storage = a.storage == "stream" ? DSEL_STORAGE_STREAM
                                        : (a.storage == "hbm" ? DSEL_STORAGE_HBM : DSEL_STORAGE_AUTO);
    if (cfg.storage == DSEL_STORAGE_STREAM) cfg.algorithm = 1;  // streaming is left-looking
    cfg.hbm_budget = a.hbm_budget;
    cfg.defer_connect = 1;
    dsel_engine* e = nullptr;
    out.st = dsel_create(&cfg, &e);
    if (out.st != DSEL_OK) out.err = dsel_last_error(nullptr);
    engines[r] = e;
    if (out.st == DSEL_OK) {
      out.st = a.synthetic.empty() ? dsel_load_kbf(e, a.kbf.c_str(), a.kbf_rows ? 0 : 1, 0)
                                   : dsel_gen_synthetic(e, v.data(), rank, sigma);
      if (out.st != DSEL_OK) out.err = dsel_last_error(e);
    }
    created[r] = out.st == DSEL_OK;
    wait_all(1);
    bool all = true;
    for (char c : created) all = all && c;
    int done = 0;
    if (all) {
      out.st = dsel_connect(e);
      if (out.st == DSEL_OK) out.st = dsel_run(e, &done);
      if (out.st != DSEL_OK) {
        out.err = dsel_last_error(e);
        if (!failed.load()) abort_peers(r);
        else out.aborted = true;
      }
    }
    if (out.st != DSEL_OK || !all) {
      if (out.err.empty()) out.err = "a peer rank failed before the selection started";
      if (out.st == DSEL_OK) out.aborted = true, out.st = DSEL_E_STATE;
    } else {
      out.rows.resize(std::max(a.budget, 1));
      const int n = dsel_get_trace(e, out.rows.data(), (int)out.rows.size());
      out.rows.resize(n > 0 ? n : 0);
    }
    wait_all(2);  // no engine is destroyed while a peer may still abort it
    if (e) dsel_destroy(e);
  };
  std::vector<std::thread> pool;
  for (int r = 0; r < G; ++r) pool.emplace_back(worker, r);
  for (auto& t : pool) t.join();
  // report the original failure, not the ranks it aborted
  std::vector<int> order;
  for (int r = 0; r < G; ++r)
    if (!res[r].aborted) order.push_back(r);
  for (int r = 0; r < G; ++r)
    if (res[r].aborted) order.push_back(r);
  for (int r : order)
    if (res[r].st != DSEL_OK) {
      std::cerr << "error: " << res[r].err << "\n";
      switch (res[r].st) {
        case DSEL_E_INFEASIBLE: return kExitInfeasible;
        case DSEL_E_IO:
        case DSEL_E_CORRUPT: return kExitIo;
        default: return kExitUsage;
      }
    }

  std::vector<dsel_step_info>& rows = res[0].rows;
  std::string warning;
  std::vector<int> chosen;
  std::vector<double> objective_raw;
  for (const auto& r : rows) {
    if (r.chosen_index < 0) {
      warning = "no feasible candidates remain; returning partial selection";
      break;
    }
    chosen.push_back(r.chosen_index);
    objective_raw.push_back(r.objective);
  }
  fs::create_directories(a.out);
  {
    std::ofstream tf(fs::path(a.out) / "trace.csv");
    tf << "k,chosen_index,objective,gain,n_evaluated,wall_ms\n";
    for (size_t i = 0; i < chosen.size(); ++i) {
      const auto& r = rows[i];
      tf << r.k << ',' << r.chosen_index << ',' << num17(r.objective) << ',' << num17(r.gain)
         << ',' << r.n_evaluated << ',' << num17(r.ms_round) << '\n';
    }
  }
  {
    // near-ties (SURVEY 8(b) trace semantics): a separate file, so trace.csv's
    // header stays the reference's
    std::ofstream nf(fs::path(a.out) / "near_ties.csv");
    nf << "k,chosen_index,gain,runner_up,runner_up_gain,rel_gap,near_tie\n";
    for (size_t i = 0; i < chosen.size(); ++i) {
      const auto& r = rows[i];
      const double gap = r.runner_up >= 0 ? (r.gain - r.runner_up_gain) / std::max(std::fabs(r.gain), 1.0)
                                          : std::numeric_limits<double>::infinity();
      nf << r.k << ',' << r.chosen_index << ',' << num17(r.gain) << ',' << r.runner_up << ','
         << (r.runner_up >= 0 ? num17(r.runner_up_gain) : std::string("")) << ','
         << (r.runner_up >= 0 ? num17(gap) : std::string("")) << ',' << r.near_tie << '\n';
    }
  }
  {
    // io_ms: H2D of the round's streamed K blocks (0 when K is resident in HBM);
    // compute_ms: the round's device work (gains, argmax exchange, W, update)
    std::ofstream rf(fs::path(a.out) / "timing.csv");
    rf << "round,worker,io_ms,compute_ms,wall_ms,overlap\n";
    for (size_t i = 0; i < chosen.size(); ++i)
      for (int g = 0; g < G; ++g) {
        if (i >= res[g].rows.size()) continue;
        const auto& r = res[g].rows[i];
        const double io = r.ms_io, comp = r.ms_gain + r.ms_exchange + r.ms_panel + r.ms_update;
        const double ov = io + comp > 0 ? std::max(0.0, 1.0 - r.ms_round / (io + comp)) : 0.0;
        rf << (i + 1) << ',' << g << ',' << io << ',' << comp << ',' << r.ms_round << ',' << ov
           << '\n';
      }
  }
  {
    // keys in std::map order, like nlohmann::json::dump(2)
    std::ostringstream j;
    auto arr_i = [&](const std::vector<int>& x) {
      if (x.empty()) return std::string("[]");
      std::string s = "[\n";
      for (size_t i = 0; i < x.size(); ++i)
        s += "    " + std::to_string(x[i]) + (i + 1 < x.size() ? ",\n" : "\n");
      return s + "  ]";
    };
    auto arr_d = [&](const std::vector<double>& x) {
      if (x.empty()) return std::string("[]");
      std::string s = "[\n";
      for (size_t i = 0; i < x.size(); ++i) s += "    " + num(x[i]) + (i + 1 < x.size() ? ",\n" : "\n");
      return s + "  ]";
    };
    std::vector<std::pair<std::string, std::string>> kv;
    kv.push_back({"budget", std::to_string(a.budget)});
    kv.push_back({"chosen", arr_i(chosen)});
    kv.push_back({"kbf", jstr(a.synthetic.empty() ? a.kbf : "synthetic:" + a.synthetic)});
    kv.push_back({"mode", jstr(a.mode)});
    kv.push_back({"n_sensors", std::to_string(nd)});
    kv.push_back({"n_steps", std::to_string(nt)});
    kv.push_back({"objective_raw", arr_d(objective_raw)});
    if (!noise.empty()) {
      std::vector<double> norm;
      double acc = 0.0;
      for (size_t i = 0; i < chosen.size(); ++i) {
        acc += noise[chosen[i]];
        norm.push_back(objective_raw[i] - acc);
      }
      kv.push_back({"objective_normalized", arr_d(norm)});
      kv.push_back({"objective_normalized_final", num(norm.empty() ? 0.0 : norm.back())});
    } else if (a.budget == 0) {
      kv.push_back({"objective_normalized", "[]"});
      kv.push_back({"objective_normalized_final", "0.0"});
    }
    kv.push_back({"pipeline", a.pipeline != "off" ? "true" : "false"});
    kv.push_back({"precision", jstr(a.precision)});
    kv.push_back({"seed", std::to_string(a.seed)});
    if (!warning.empty()) kv.push_back({"warning", jstr(warning)});
    kv.push_back({"workers", std::to_string(a.workers)});
    std::sort(kv.begin(), kv.end());
    j << "{\n";
    for (size_t i = 0; i < kv.size(); ++i)
      j << "  " << jstr(kv[i].first) << ": " << kv[i].second << (i + 1 < kv.size() ? ",\n" : "\n");
    j << "}\n";
    std::ofstream sf(fs::path(a.out) / "selection.json");
    if (!sf) {
      std::cerr << "error: cannot write " << (fs::path(a.out) / "selection.json").string() << "\n";
      return kExitIo;
    }
    sf << j.str();
  }
  std::cout << "selected " << chosen.size() << " sensors -> " << a.out << "/selection.json\n";
  return kExitOk;
}

int usage() {
  std::cerr << "usage: doptsel select <kbf> --budget B [--mode schur|gpu] [--gpus G] [--workers N]\n"
               "                      [--algorithm right|left] [--storage auto|hbm|stream]\n"
               "                      [--hbm-budget BYTES] [--seed S] [--pipeline on|off] [--precision f64]\n"
               "                      [--config cfg | --noise-logdets file] [--kbf-rows] [--out DIR]\n"
               "       doptsel select --synthetic nd,nt,rank,sigma,seed --budget B [...]\n"
               "       doptsel build <config> <out.kbf>      (K assembled on the GPU)\n";
  return kExitUsage;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  if (cmd == "build") {
    if (argc != 4) {
      std::cerr << "usage: doptsel build <config> <out.kbf>\n";
      return kExitUsage;
    }
    return cmd_build(argv[2], argv[3]);
  }
  if (cmd == "evaluate" || cmd == "bench") {
    std::cerr << "error: `" << cmd << "` is outside the selection hot path served by this build "
                 "(use the reference tool)\n";
    return kExitUsage;
  }
  if (cmd != "select") return usage();
  SelectArgs a;
  for (int i = 2; i < argc; ++i) {
    const std::string s = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + s);
      return argv[++i];
    };
    try {
      if (s == "--budget") a.budget = std::stoi(val());
      else if (s == "--workers") a.workers = std::stoi(val());
      else if (s == "--gpus") a.gpus = std::stoi(val());
      else if (s == "--mode") {
        a.mode = val();
        if (a.mode != "schur" && a.mode != "gpu" && a.mode != "naive") return usage();
      } else if (s == "--seed") a.seed = std::stoull(val());
      else if (s == "--pipeline") {
        a.pipeline = val();
        if (a.pipeline != "on" && a.pipeline != "off") return usage();
      } else if (s == "--precision") {
        a.precision = val();
        if (a.precision != "f64" && a.precision != "f32") return usage();
      } else if (s == "--config") a.config = val();
      else if (s == "--noise-logdets") a.noise_file = val();
      else if (s == "--synthetic") a.synthetic = val();
      else if (s == "--kbf-rows") a.kbf_rows = true;
      else if (s == "--algorithm") {
        a.algorithm = val();
        if (a.algorithm != "right" && a.algorithm != "left") return usage();
      } else if (s == "--storage") {
        a.storage = val();
        if (a.storage != "auto" && a.storage != "hbm" && a.storage != "stream") return usage();
      }
      else if (s == "--hbm-budget") a.hbm_budget = std::stoull(val());
      else if (s == "--out") a.out = val();
      else if (!s.empty() && s[0] == '-') return usage();
      else if (a.kbf.empty()) a.kbf = s;
      else return usage();
    } catch (const std::exception& ex) {
      std::cerr << "error: " << ex.what() << "\n";
      return kExitUsage;
    }
  }
  if (a.budget < 0 && a.budget != -1) return usage();
  if (a.budget == -1 || (a.kbf.empty() && a.synthetic.empty())) return usage();
  return run_select(a);
}
