// lti.h -- host side of K formation from an LTI wave problem.
//
// The reference builds K from a plain-text problem config (config.hpp:17-164):
// make_wave_problem (lti.hpp:163-176) places sensors with its Rng, tabulates the
// causal wave kernels h[s][j][tau] (lti.hpp:122-131) and the spatial prior
// (lti.hpp:245-251). These are cheap O(Nd*Nm*Nt + Nm^2) host tables computed
// with glibc exactly as the reference does; the O(Nd^2 Nt^3 Nm) assembly runs
// on the GPU (engine.cu dsel_assemble_lti).
#pragma once

#include <string>
#include <vector>

namespace dsel {

struct LtiHost {
  int n_params = 0, n_sensors = 0, n_steps = 0;
  double noise_sigma = 0.0;
  std::vector<double> impulse;  // [s][j][tau]
  std::vector<double> spatial;  // [i][j]
  std::vector<double> mask;     // [j][t] or empty
  std::vector<double> cost;     // [s] or empty
};

// Parse a reference problem config and build its wave problem + weights.
// Returns 0 on success; 1 = invalid config (message in err), 7 = cannot open.
int lti_from_config(const char* path, LtiHost& out, std::string& err);

}  // namespace dsel
