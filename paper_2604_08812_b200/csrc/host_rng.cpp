// host_rng.cpp -- synthetic-K input of the product: V of SyntheticKAccess.
//
// SyntheticKAccess (kaccess.hpp:81-124) fills V sequentially with
// Rng::normal() (rng.hpp:37-50): std::mt19937_64 + Box-Muller with a cached
// spare, transforms hand-rolled so the bits are compiler-independent. CUDA's
// log/sin/cos are not bit-identical to glibc's, so V is produced here on the
// host and uploaded; the device then forms K = sigma^2 I + V V^T bit-exactly
// (kernels.cuh synth_panel_kernel).
//
// The mt19937_64 stream is inherently sequential, the transform is not: the
// stream is cut into (u1,u2) pairs sequentially -- reproducing the u1 <= 0
// re-draw exactly -- and the log/sqrt/sin/cos transform runs on all cores.
// Built with -ffp-contract=off so no FMA contraction changes bits.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

#include "dsel.h"

extern "C" dsel_status dsel_synthetic_v(int n_sensors, int n_steps, int rank, uint64_t seed,
                                        double* out, int threads) {
  if (n_sensors < 1 || n_steps < 1 || rank < 1 || out == nullptr) return DSEL_E_INVALID;
  const uint64_t count = (uint64_t)n_sensors * (uint64_t)n_steps * (uint64_t)rank;
  const uint64_t n_pairs = (count + 1) / 2;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  std::mt19937_64 gen(seed);
  auto uniform_bits = [&]() { return gen() >> 11; };  // rng.hpp:22, value = bits * 2^-53
  constexpr uint64_t kChunk = 1u << 22;               // pairs per chunk
  std::vector<uint64_t> u1(std::min(kChunk, n_pairs)), u2(std::min(kChunk, n_pairs));
  for (uint64_t base = 0; base < n_pairs; base += kChunk) {
    const uint64_t m = std::min(kChunk, n_pairs - base);
    for (uint64_t i = 0; i < m; ++i) {  // sequential: exact stream consumption
      uint64_t a = uniform_bits();
      const uint64_t b = uniform_bits();
      while (a == 0) a = uniform_bits();  // `while (u1 <= 0.0) u1 = uniform();`
      u1[i] = a;
      u2[i] = b;
    }
    auto work = [&](uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i) {
        const double x1 = static_cast<double>(u1[i]) * 0x1.0p-53;
        const double x2 = static_cast<double>(u2[i]) * 0x1.0p-53;
        const double r = std::sqrt(-2.0 * std::log(x1));
        const double a = 2.0 * std::numbers::pi * x2;
        const uint64_t o = 2 * (base + i);
        out[o] = r * std::cos(a);                   // returned first
        if (o + 1 < count) out[o + 1] = r * std::sin(a);  // the cached spare
      }
    };
    const int nthr = (int)std::min<uint64_t>((uint64_t)threads, std::max<uint64_t>(1, m / 4096));
    std::vector<std::thread> pool;
    for (int w = 0; w < nthr; ++w) {
      const uint64_t lo = m * w / nthr, hi = m * (w + 1) / nthr;
      pool.emplace_back(work, lo, hi);
    }
    for (auto& t : pool) t.join();
  }
  return DSEL_OK;
}
