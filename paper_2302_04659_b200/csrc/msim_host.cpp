// Host-side reference utilities exported with the C ABI: the particle seeder
// that produces the inputs of every synthetic scene (seeding.hpp:13-46 — a
// jittered lattice of spacing cbrt(V0) filled from a caller-held
// std::mt19937_64), so the GPU path and any CPU checker start from
// bit-identical particles.
#include <algorithm>
#include <cmath>
#include <random>

#include "../../include/msim_gpu.h"

struct msim_rng {
  std::mt19937_64 engine;
};

extern "C" {

msim_rng* msim_rng_create(uint64_t seed) { return new msim_rng{std::mt19937_64(seed)}; }
void msim_rng_destroy(msim_rng* r) { delete r; }
double msim_rng_uniform(msim_rng* r, double lo, double hi) {
  return std::uniform_real_distribution<double>(lo, hi)(r->engine);
}

void msim_rng_fill_uniform(msim_rng* r, int64_t n, double lo, double hi, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = std::uniform_real_distribution<double>(lo, hi)(r->engine);
}

int64_t msim_seed_box_count(const double* lo, const double* hi, double particle_volume) {
  const double s = std::cbrt(particle_volume);
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) total *= std::max(1, (int)std::floor((hi[a] - lo[a]) / s));
  return total;
}

int64_t msim_seed_box(msim_rng* r, const double* lo, const double* hi, double density,
                      double particle_volume, double* x, double* mass) {
  const double s = std::cbrt(particle_volume);
  int n[3];
  for (int a = 0; a < 3; ++a) n[a] = std::max(1, (int)std::floor((hi[a] - lo[a]) / s));
  std::uniform_real_distribution<double> jit(-0.25 * s, 0.25 * s);
  int64_t out = 0;
  for (int k = 0; k < n[2]; ++k)
    for (int j = 0; j < n[1]; ++j)
      for (int i = 0; i < n[0]; ++i, ++out) {
        // The reference draws Vec3(jitter, jitter, jitter) whose argument
        // order GCC evaluates right to left: z first, then y, then x.
        const double dz = jit(r->engine);
        const double dy = jit(r->engine);
        const double dx = jit(r->engine);
        const int idx[3] = {i, j, k};
        const double d[3] = {dx, dy, dz};
        if (!x) continue;
        for (int a = 0; a < 3; ++a) {
          double p = lo[a] + s * (idx[a] + 0.5);
          p += d[a];
          x[3 * out + a] = std::min(std::max(p, lo[a]), hi[a]);
        }
        if (mass) mass[out] = density * particle_volume;
      }
  return out;
}

}  // extern "C"
