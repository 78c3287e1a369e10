// Host-side (CPU, native) synthetic sampling-pattern generator.
//
// BASELINE.json configs 0-2 ask for variable-density Poisson-disc masks with a
// fully sampled centre, which the reference does not provide (its simulate.py
// only draws 1-D line masks, /root/reference/pkg/src/sketchrecon/simulate.py:209-259;
// SURVEY.md Appendix A).  This is a deterministic seeded generator: random
// sequential acceptance of grid bins with a minimum spacing that grows
// linearly with the normalised k-space radius, r(k) = 1 + slope * |k|, and a
// bisection on the slope to hit the target acceleration.  Used for synthetic
// inputs only (benchmarks, tests); both the GPU path and the oracle receive the
// resulting bins, so its statistics never affect parity.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "sketchrecon_b200.h"

namespace {

struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

// one pass at a given slope; returns number of accepted bins
long long poisson_pass(int ny, int nx, double slope, const std::vector<int>& order,
                       uint8_t* mask, std::vector<float>& rad) {
  memset(mask, 0, (size_t)ny * nx);
  const double cy = ny / 2, cx = nx / 2;
  double rmax = 1.0;
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      const double ky = (y - cy) / (ny / 2.0), kx = (x - cx) / (nx / 2.0);
      const double r = 1.0 + slope * std::sqrt(ky * ky + kx * kx);
      rad[(size_t)y * nx + x] = (float)r;
      rmax = std::max(rmax, r);
    }
  const int w = (int)std::ceil(rmax);
  long long count = 0;
  for (int id : order) {
    const int y = id / nx, x = id % nx;
    const float r = rad[id];
    const float r2 = r * r;
    bool ok = true;
    for (int dy = -w; dy <= w && ok; ++dy) {
      const int yy = y + dy;
      if (yy < 0 || yy >= ny) continue;
      for (int dx = -w; dx <= w; ++dx) {
        const int xx = x + dx;
        if (xx < 0 || xx >= nx) continue;
        if (!mask[(size_t)yy * nx + xx]) continue;
        // spacing judged with the larger of the two local radii
        const float rr = std::max(r, rad[(size_t)yy * nx + xx]);
        if ((float)(dy * dy + dx * dx) < std::min(r2, rr * rr)) { ok = false; break; }
      }
    }
    if (ok) { mask[id] = 1; ++count; }
  }
  return count;
}

}  // namespace

extern "C" {

// Variable-density Poisson-disc mask (ny x nx, row-major, 1 = sampled) with a
// fully sampled centre of (calib x calib) bins and about ny*nx/accel samples.
// Returns the number of sampled bins, or -1 on bad arguments.
long long sr_host_vd_poisson(int ny, int nx, double accel, int calib, unsigned long long seed,
                             uint8_t* mask) {
  if (ny < 2 || nx < 2 || accel < 1.0 || calib < 0 || !mask) return -1;
  const long long D = (long long)ny * nx;
  const long long target = (long long)std::llround((double)D / accel);
  std::vector<int> order(D);
  for (long long i = 0; i < D; ++i) order[i] = (int)i;
  SplitMix64 rng(seed ^ 0x5EEDC0DEull);
  for (long long i = D - 1; i > 0; --i) {  // Fisher-Yates
    const long long j = (long long)(rng.next() % (uint64_t)(i + 1));
    std::swap(order[i], order[j]);
  }
  std::vector<float> rad(D);
  std::vector<uint8_t> work(D);
  auto with_calib = [&](uint8_t* m) {
    long long c = 0;
    const int y0 = ny / 2 - calib / 2, x0 = nx / 2 - calib / 2;
    for (int y = std::max(0, y0); y < std::min(ny, y0 + calib); ++y)
      for (int x = std::max(0, x0); x < std::min(nx, x0 + calib); ++x) m[(size_t)y * nx + x] = 1;
    for (long long i = 0; i < D; ++i) c += m[i];
    return c;
  };
  double lo = 0.0, hi = 1.0;
  // grow hi until the pattern is sparse enough
  for (int it = 0; it < 40; ++it) {
    poisson_pass(ny, nx, hi, order, work.data(), rad);
    if (with_calib(work.data()) <= target) break;
    lo = hi;
    hi *= 2.0;
  }
  for (int it = 0; it < 16; ++it) {
    const double mid = 0.5 * (lo + hi);
    poisson_pass(ny, nx, mid, order, work.data(), rad);
    if (with_calib(work.data()) > target) lo = mid; else hi = mid;
  }
  poisson_pass(ny, nx, hi, order, mask, rad);
  return with_calib(mask);
}

}  // extern "C"
