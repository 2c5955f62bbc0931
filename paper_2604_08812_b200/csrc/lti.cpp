// lti.cpp -- problem config -> wave problem tables (host, glibc, -ffp-contract=off).
//
// Restates config.hpp:84-164 (parse_problem_config / problem_from_config /
// weights_from_config), lti.hpp:122-176 (wave_kernel_into, make_wave_problem_at,
// make_wave_problem), lti.hpp:62-75 (LtiProblem validation), lti.hpp:35-56
// (WeightSpec::validate) and lti.hpp:245-251 (materialize_spatial_prior), so
// the tables -- and hence the K the GPU assembles -- are bit-identical.
#include "lti.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>

namespace dsel {
namespace {

struct Bad {
  int code;
  std::string msg;
};

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

template <class T>
T number(const std::string& value, const std::string& key) {
  std::stringstream ss(value);
  T out{};
  ss >> out;
  if (ss.fail() || !ss.eof()) throw Bad{1, "config key '" + key + "': bad value '" + value + "'"};
  return out;
}

std::vector<double> number_list(const std::string& value, const std::string& key) {
  std::vector<double> out;
  std::stringstream ss(value);
  std::string item;
  while (std::getline(ss, item, ',')) {
    item = trim(item);
    if (item.empty()) continue;
    size_t used = 0;
    double v = 0.0;
    try {
      v = std::stod(item, &used);
    } catch (const std::exception&) {
      used = std::string::npos;
    }
    if (used != item.size()) throw Bad{1, "config key '" + key + "': bad number '" + item + "'"};
    out.push_back(v);
  }
  return out;
}

struct Config {
  int n_params = 16, n_sensors = 8, n_steps = 8;
  double wave_speed = 1.0, decay = 0.25;
  uint64_t seed = 0;
  double noise_sigma = -1.0;
  bool prior_identity = false;
  double prior_variance = 1.0, prior_length = 0.0;
  std::vector<double> cost, mask_param, mask_step;
};

Config parse(std::istream& in) {
  Config c;
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos)
      throw Bad{1, "config line " + std::to_string(no) + ": expected key = value"};
    const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
    if (key == "n_params") c.n_params = number<int>(value, key);
    else if (key == "n_sensors") c.n_sensors = number<int>(value, key);
    else if (key == "n_steps") c.n_steps = number<int>(value, key);
    else if (key == "wave_speed") c.wave_speed = number<double>(value, key);
    else if (key == "decay") c.decay = number<double>(value, key);
    else if (key == "seed") c.seed = number<uint64_t>(value, key);
    else if (key == "noise_sigma") c.noise_sigma = number<double>(value, key);
    else if (key == "prior.kind") {
      if (value == "identity") c.prior_identity = true;
      else if (value == "exponential") c.prior_identity = false;
      else
        throw Bad{1, "config key 'prior.kind': expected identity or exponential, got '" + value + "'"};
    } else if (key == "prior.variance") c.prior_variance = number<double>(value, key);
    else if (key == "prior.length_scale") c.prior_length = number<double>(value, key);
    else if (key == "cost_weights") c.cost = number_list(value, key);
    else if (key == "mask_param_weights") c.mask_param = number_list(value, key);
    else if (key == "mask_step_weights") c.mask_step = number_list(value, key);
    else throw Bad{1, "unknown config key '" + key + "'"};
  }
  return c;
}

void build(const Config& c, LtiHost& p) {
  const int nm = c.n_params, nd = c.n_sensors, nt = c.n_steps;
  if (nm < 1 || nd < 1 || nt < 1) throw Bad{1, "problem sizes must be >= 1"};
  if (!(c.wave_speed > 0.0)) throw Bad{1, "wave_speed must be positive"};
  if (!(c.decay >= 0.0)) throw Bad{1, "decay must be nonnegative"};
  // sensor positions: uniform on [0, nm-1] from the reference Rng, sorted
  std::mt19937_64 gen(c.seed);
  std::vector<double> pos(nd);
  for (double& x : pos) x = static_cast<double>(gen() >> 11) * 0x1.0p-53 * (nm > 1 ? nm - 1 : 0);
  std::sort(pos.begin(), pos.end());
  double length = c.prior_length;
  if (!c.prior_identity && length <= 0.0) length = std::max(1.0, nm / 8.0);
  p.n_params = nm;
  p.n_sensors = nd;
  p.n_steps = nt;
  p.impulse.assign((size_t)nd * nm * nt, 0.0);
  for (int s = 0; s < nd; ++s)
    for (int j = 0; j < nm; ++j) {
      const double dist = std::abs(pos[s] - j);
      const double delay = dist / c.wave_speed;
      const double amp = 1.0 / (1.0 + dist);
      double* out = p.impulse.data() + ((size_t)s * nm + j) * nt;
      for (int tau = 0; tau < nt; ++tau) {
        const double u = tau - delay;
        out[tau] = u < 0.0 ? 0.0 : amp * std::exp(-c.decay * u * u);
      }
    }
  double sigma = c.noise_sigma;
  if (!(sigma > 0.0)) {
    double amp = 0.0;
    for (double v : p.impulse) amp = std::max(amp, std::abs(v));
    sigma = 0.1 * (amp > 0.0 ? amp : 1.0);
  }
  for (double v : p.impulse)
    if (!std::isfinite(v)) throw Bad{1, "impulse kernels must be finite"};
  if (!(sigma > 0.0)) throw Bad{1, "noise_sigma must be positive"};
  if (!(c.prior_variance > 0.0)) throw Bad{1, "prior.variance must be positive"};
  if (!c.prior_identity && !(length > 0.0)) throw Bad{1, "prior.length_scale must be positive"};
  p.noise_sigma = sigma;
  p.spatial.assign((size_t)nm * nm, 0.0);
  for (int i = 0; i < nm; ++i)
    for (int j = 0; j < nm; ++j)
      p.spatial[(size_t)i * nm + j] = c.prior_identity
                                          ? (i == j ? c.prior_variance : 0.0)
                                          : c.prior_variance * std::exp(-std::abs(i - j) / length);
  // weights
  p.cost = c.cost;
  if (!p.cost.empty()) {
    if ((int)p.cost.size() != nd) throw Bad{1, "cost_weights must have one entry per sensor"};
    for (double w : p.cost)
      if (!(w > 0.0)) throw Bad{1, "cost_weights entries must be positive"};
  }
  p.mask.clear();
  if (!c.mask_param.empty() || !c.mask_step.empty()) {
    std::vector<double> wp = c.mask_param, wt = c.mask_step;
    if (wp.empty()) wp.assign(nm, 1.0);
    if (wt.empty()) wt.assign(nt, 1.0);
    if ((int)wp.size() != nm) throw Bad{1, "mask_param_weights must have n_params entries"};
    if ((int)wt.size() != nt) throw Bad{1, "mask_step_weights must have n_steps entries"};
    p.mask.assign((size_t)nm * nt, 0.0);
    for (int j = 0; j < nm; ++j)
      for (int t = 0; t < nt; ++t) p.mask[(size_t)j * nt + t] = wp[j] * wt[t];
    for (double m : p.mask)
      if (!(m >= 0.0)) throw Bad{1, "mask_weights entries must be nonnegative"};
  }
}

}  // namespace

int lti_from_config(const char* path, LtiHost& out, std::string& err) {
  try {
    std::ifstream in(path);
    if (!in) throw Bad{7, std::string("cannot open config file ") + path};
    build(parse(in), out);
    return 0;
  } catch (const Bad& b) {
    err = b.msg;
    return b.code;
  }
}

}  // namespace dsel
