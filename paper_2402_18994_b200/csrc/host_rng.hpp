// host_rng.hpp -- host-side reproduction of the reference's counter-based RNG
// and the two places the training loop consumes it: parameter init and the
// per-epoch permutation.  Identical seeds must give identical parameters and
// batches (optimize_test.cpp:170-191), so these follow rng.hpp exactly.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace snn {
namespace hostrng {

// SplitMix64 finalizer (rng.hpp:20-25).
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t from_seed(uint64_t s) { return mix64(s); }                              // rng.hpp:34-36
inline uint64_t child(uint64_t k, uint64_t i) { return mix64(k ^ mix64(i + 0xC2B2AE3D27D4EB4Full)); }  // :43-46
inline uint64_t bits(uint64_t k, uint64_t c) { return mix64(k ^ mix64(c + 0x165667B19E3779F9ull)); }   // :39-41
inline double uniform01(uint64_t k, uint64_t c) { return double(bits(k, c) >> 11) * 0x1.0p-53; }  // :62-64

// Fisher-Yates (rng.hpp:78-87).
inline std::vector<uint32_t> permutation(uint64_t key, size_t n) {
  std::vector<uint32_t> p(n);
  for (size_t i = 0; i < n; ++i) p[i] = uint32_t(i);
  for (size_t i = n; i > 1; --i) {
    const size_t j = size_t(bits(key, i - 1) % uint64_t(i));
    std::swap(p[i - 1], p[j]);
  }
  return p;
}

// randint (rng.hpp:68-75): lo + bits(counter) % (hi - lo).
inline int64_t randint(uint64_t key, uint64_t c, int64_t lo, int64_t hi) {
  return lo + int64_t(bits(key, c) % uint64_t(hi - lo));
}

// shift_augment of batch b (data.hpp:216-227 with key child(epoch_key, 1 + b),
// optimize.hpp:276-278): n_axes rolls of the same flat feature axis compose to
// one roll by the sum of the per-axis draws, reduced into [0, in).
inline int32_t batch_roll(uint64_t epoch_key, uint64_t b, int64_t max_shift, int n_axes, int64_t in) {
  if (max_shift <= 0 || n_axes == 0) return 0;
  const uint64_t k = child(epoch_key, 1 + b);
  int64_t s = 0;
  for (int i = 0; i < n_axes; ++i) s += randint(k, uint64_t(i), -max_shift, max_shift);
  s %= in;
  return int32_t(s < 0 ? s + in : s);
}

// Truncated normal, +-2 sigma, per-element child keys (rng.hpp:92-97, :123-144).
inline void truncated_normal(uint64_t key, size_t n, float mean, float sd, float* out) {
  for (size_t i = 0; i < n; ++i) {
    const uint64_t ek = child(key, i);
    double z = 0.0;
    bool ok = false;
    for (uint64_t a = 0; a < 256; ++a) {
      const double u1 = 1.0 - uniform01(ek, 2 * a);
      const double u2 = uniform01(ek, 2 * a + 1);
      z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
      if (z >= -2.0 && z <= 2.0) {
        ok = true;
        break;
      }
    }
    if (!ok) z = z < -2.0 ? -2.0 : (z > 2.0 ? 2.0 : z);
    out[i] = mean + sd * float(z);
  }
}

}  // namespace hostrng
}  // namespace snn
