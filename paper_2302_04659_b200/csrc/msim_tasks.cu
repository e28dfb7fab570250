// Device side of the consumers of the soft-body state that SURVEY.md §8(f)
// ranks next after the substep (reference paths relative to
// /root/reference/proj/include/msim/):
//   * mesh SDF baking, bake_mesh_sdf (sdf.hpp:203-310): one thread per voxel,
//     triangles streamed through shared memory, exact point-triangle distance
//     and the three-ray parity vote in fp64;
//   * batched task metrics over every env's live particle state:
//     metric_fill, render_heightmap, metric_write_iou, chamfer_distance /
//     metric_pinch (scenario.hpp:63-209).
// This file is compiled with --fmad=false: every fp64 expression below keeps
// the reference's operation order with one rounding per operation, so baked
// samples, heights, speeds and nearest distances are bit-identical to the
// double-precision restatement fed the same inputs.
#include <cfloat>
#include <cstdint>

#include "msim_internal.h"

namespace msim_impl {
namespace {

struct d3 {
  double x, y, z;
};
__device__ __forceinline__ d3 operator+(d3 a, d3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ d3 operator-(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ d3 operator*(d3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(d3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

// point_triangle_distance (sdf.hpp:214-237), same branch structure and order
__device__ double point_triangle_distance(d3 p, d3 a, d3 b, d3 c) {
  d3 ab = b - a, ac = c - a, ap = p - a;
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return norm(p - a);
  d3 bp = p - b;
  double d3_ = dot(ab, bp), d4 = dot(ac, bp);
  if (d3_ >= 0 && d4 <= d3_) return norm(p - b);
  double vc = d1 * d4 - d3_ * d2;
  if (vc <= 0 && d1 >= 0 && d3_ <= 0) return norm(p - (a + ab * (d1 / (d1 - d3_))));
  d3 cp = p - c;
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return norm(p - c);
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return norm(p - (a + ac * (d2 / (d2 - d6))));
  double va = d3_ * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3_) >= 0 && (d5 - d6) >= 0) {
    double w = (d4 - d3_) / ((d4 - d3_) + (d5 - d6));
    return norm(p - (b + (c - b) * w));
  }
  double denom = 1.0 / (va + vb + vc);
  d3 closest = a + ab * (vb * denom) + ac * (vc * denom);
  return norm(p - closest);
}

// ray_hits_triangle (sdf.hpp:239-254), Moller-Trumbore
__device__ bool ray_hits_triangle(d3 orig, d3 dir, d3 a, d3 b, d3 c) {
  d3 e1 = b - a, e2 = c - a;
  d3 pv = cross(dir, e2);
  double det = dot(e1, pv);
  if (fabs(det) < 1e-14) return false;
  double inv = 1.0 / det;
  d3 tv = orig - a;
  double u = dot(tv, pv) * inv;
  if (u < 0.0 || u > 1.0) return false;
  d3 qv = cross(tv, e1);
  double v = dot(dir, qv) * inv;
  if (v < 0.0 || u + v > 1.0) return false;
  double dist = dot(e2, qv) * inv;
  return dist > 0.0;
}

constexpr int kBakeT = 128;

// One thread per voxel (x-fastest, sdf.hpp:297-308); the mesh is streamed in
// chunks of kBakeT triangles through shared memory, each chunk read by every
// voxel of the block. Distance min and the three ray parities are one pass.
__global__ void __launch_bounds__(kBakeT) k_bake(const double* __restrict__ tri, long long n_tri, d3 origin,
                                                 double voxel, int dx, int dy, int dz, d3 r0, d3 r1, d3 r2,
                                                 float* __restrict__ out) {
  __shared__ double st[kBakeT * 9];
  const long long nvox = (long long)dx * dy * dz;
  const long long idx = (long long)blockIdx.x * kBakeT + threadIdx.x;
  const bool valid = idx < nvox;
  const int i = (int)(idx % dx), j = (int)((idx / dx) % dy), k = (int)(idx / ((long long)dx * dy));
  const d3 p = origin + d3{voxel * i, voxel * j, voxel * k};  // origin + voxel * (i, j, k)
  double d = DBL_MAX;
  int c0 = 0, c1 = 0, c2 = 0;
  for (long long base = 0; base < n_tri; base += kBakeT) {
    const int cnt = (int)min((long long)kBakeT, n_tri - base);
    __syncthreads();
    for (int q = threadIdx.x; q < cnt * 9; q += kBakeT) st[q] = tri[base * 9 + q];
    __syncthreads();
    if (!valid) continue;
    for (int t = 0; t < cnt; ++t) {
      const double* s = st + 9 * t;
      const d3 a = {s[0], s[1], s[2]}, b = {s[3], s[4], s[5]}, c = {s[6], s[7], s[8]};
      const double e = point_triangle_distance(p, a, b, c);
      d = (e < d) ? e : d;  // std::min(d, e)
      c0 += ray_hits_triangle(p, r0, a, b, c);
      c1 += ray_hits_triangle(p, r1, a, b, c);
      c2 += ray_hits_triangle(p, r2, a, b, c);
    }
  }
  if (!valid) return;
  const int votes = (c0 & 1) + (c1 & 1) + (c2 & 1);
  out[idx] = (float)(votes >= 2 ? -d : d);
}

// ---- task metrics --------------------------------------------------------

__device__ __forceinline__ bool region_contains(const double* r, double x, double y, double z) {
  return x >= r[0] && y >= r[1] && z >= r[2] && x <= r[3] && y <= r[4] && z <= r[5];
}

// max of a nonnegative double's bits over the lanes of `grp` (two 32-bit
// warp reductions: high word, then low word among the lanes holding that high)
__device__ __forceinline__ unsigned long long group_max_bits(unsigned grp, unsigned long long bits) {
  const unsigned hi = (unsigned)(bits >> 32);
  const unsigned mhi = __reduce_max_sync(grp, hi);
  const unsigned mlo = __reduce_max_sync(grp, hi == mhi ? (unsigned)bits : 0u);
  return ((unsigned long long)mhi << 32) | mlo;
}

// metric_fill (scenario.hpp:63-75): per env count inside + max |v| (double of
// the stored fp32). Particles are stored env-major, so lanes are grouped by env
// (match_any) and each group issues one atomic per counter.
__global__ void k_fill(SimParams P, const double* __restrict__ regions, unsigned long long* inside,
                       unsigned long long* vmax_bits) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = i < P.n;
  int env = -1;
  bool in = false;
  unsigned long long bits = 0;
  if (valid) {
    const Particles& q = P.cur;
    env = (q.meta[i] >> 8) & kEnvMask;
    const double x = q.x[0][i], y = q.x[1][i], z = q.x[2][i];
    const double vx = q.v[0][i], vy = q.v[1][i], vz = q.v[2][i];
    const double sp = sqrt(vx * vx + vy * vy + vz * vz);
    in = region_contains(regions + 6 * env, x, y, z);
    bits = (unsigned long long)__double_as_longlong(sp);  // sp >= 0: bit order = value order
  }
  const unsigned grp = __match_any_sync(0xffffffffu, env);
  const unsigned cnt = __popc(__ballot_sync(0xffffffffu, in) & grp);
  bits = group_max_bits(grp, bits);
  if (valid && (int)(threadIdx.x & 31) == __ffs(grp) - 1) {
    if (cnt) atomicAdd(inside + env, (unsigned long long)cnt);
    atomicMax(vmax_bits + env, bits);
  }
}

// render_heightmap (scenario.hpp:79-98): per env nx*ny max heights above the
// region floor; lanes landing in the same cell combine before the atomic.
__global__ void k_heightmap(SimParams P, const double* __restrict__ regions, int nx, int ny,
                            unsigned long long* maps) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long slot = -1;
  unsigned long long bits = 0;
  if (i < P.n) {
    const Particles& q = P.cur;
    const int env = (q.meta[i] >> 8) & kEnvMask;
    const double* r = regions + 6 * env;
    const double x = q.x[0][i], y = q.x[1][i], z = q.x[2][i];
    if (region_contains(r, x, y, z)) {
      const double cell = (r[3] - r[0]) / nx, cy = (r[4] - r[1]) / ny;
      const int ci = min(nx - 1, (int)((x - r[0]) / cell));
      const int cj = min(ny - 1, (int)((y - r[1]) / cy));
      slot = (long long)env * nx * ny + (long long)cj * nx + ci;
      bits = (unsigned long long)__double_as_longlong(z - r[2]);  // >= 0 (contained)
    }
  }
  const unsigned grp = __match_any_sync(0xffffffffu, slot);
  bits = group_max_bits(grp, bits);
  if (slot >= 0 && (int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicMax(maps + slot, bits);
}

// metric_write_iou (scenario.hpp:106-119), one block per env
__global__ void k_iou(const double* __restrict__ maps, const double* __restrict__ targets, int cells,
                      double threshold, double* iou, int* success) {
  const int env = blockIdx.x;
  const double* a = maps + (long long)env * cells;
  const double* b = targets + (long long)env * cells;
  unsigned inter = 0, uni = 0;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) {
    const bool oa = a[c] < threshold, ob = b[c] < threshold;
    inter += oa && ob;
    uni += oa || ob;
  }
  __shared__ unsigned si[32], su[32];
  for (int o = 16; o > 0; o >>= 1) {
    inter += __shfl_xor_sync(0xffffffffu, inter, o);
    uni += __shfl_xor_sync(0xffffffffu, uni, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    si[w] = inter;
    su[w] = uni;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned ti = 0, tu = 0;
    for (int k = 0; k < nw; ++k) {
      ti += si[k];
      tu += su[k];
    }
    const double r = tu == 0 ? 1.0 : (double)ti / (double)tu;
    iou[env] = r;
    success[env] = r > 0.8;
  }
}

// particle positions of every env in upload (pid) order, fp32 -> double
__global__ void k_positions(SimParams P, double* pos) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const long long j = P.cur.pid[i];
  pos[3 * j + 0] = P.cur.x[0][i];
  pos[3 * j + 1] = P.cur.x[1][i];
  pos[3 * j + 2] = P.cur.x[2][i];
}

constexpr int kNnT = 128, kNnQ = 4;

// Nearest distance from every point of set A to set B, per env: blockIdx.y =
// env, kNnQ queries per thread (each B point read from shared memory once per
// kNnQ distance evaluations), B streamed through shared memory. The minimum of
// squared norms then one sqrt: sqrt is monotone and correctly rounded, so this
// equals the minimum of the reference's per-pair norm() (scenario.hpp:168).
__global__ void __launch_bounds__(kNnT) k_nearest(const double* __restrict__ A, const long long* __restrict__ offA,
                                                  const double* __restrict__ B, const long long* __restrict__ offB,
                                                  double* __restrict__ mind) {
  __shared__ double sb[kNnT * 3];
  const int env = blockIdx.y;
  const long long a0 = offA[env], na = offA[env + 1] - a0;
  const long long b0 = offB[env], nb = offB[env + 1] - b0;
  const long long q0 = (long long)blockIdx.x * kNnT * kNnQ;
  if (q0 >= na) return;  // block-uniform
  double qx[kNnQ], qy[kNnQ], qz[kNnQ], best[kNnQ];
#pragma unroll
  for (int k = 0; k < kNnQ; ++k) {
    const long long qi = q0 + k * kNnT + threadIdx.x;
    const long long src = a0 + (qi < na ? qi : 0);
    qx[k] = A[3 * src];
    qy[k] = A[3 * src + 1];
    qz[k] = A[3 * src + 2];
    best[k] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  }
  for (long long base = 0; base < nb; base += kNnT) {
    const int cnt = (int)min((long long)kNnT, nb - base);
    __syncthreads();
    for (int q = threadIdx.x; q < cnt * 3; q += kNnT) sb[q] = B[3 * (b0 + base) + q];
    __syncthreads();
    for (int t = 0; t < cnt; ++t) {
      const double bx = sb[3 * t], by = sb[3 * t + 1], bz = sb[3 * t + 2];
#pragma unroll
      for (int k = 0; k < kNnQ; ++k) {
        const double dx = bx - qx[k], dy = by - qy[k], dz = bz - qz[k];
        const double d2 = dx * dx + dy * dy + dz * dz;
        best[k] = d2 < best[k] ? d2 : best[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNnQ; ++k) {
    const long long qi = q0 + k * kNnT + threadIdx.x;
    if (qi < na) mind[a0 + qi] = sqrt(best[k]);
  }
}

// mean of a segmented array, one block per segment, fixed reduction order
__global__ void k_segment_mean(const double* __restrict__ v, const long long* __restrict__ off, double* out) {
  const int env = blockIdx.x;
  const long long s = off[env], n = off[env + 1] - s;
  double acc = 0.0;
  for (long long k = threadIdx.x; k < n; k += blockDim.x) acc += v[s + k];
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[env] = n > 0 ? red[0] / (double)n : 0.0;
}

// ---- on-device seeding (seeding.hpp:13-35) --------------------------------
// std::mt19937_64 (libstdc++ parameters) with the 312-word twist split in the
// three dependency phases of _M_gen_rand, each read-all-then-write across the
// block, and libstdc++'s uniform_real_distribution<double>:
// (double(x) / 2^64, clamped below 1) * (b - a) + a.
constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kMtA = 0xb5026f5aa96619e9ull, kMtUpper = ~0ull << 31, kMtLower = ~kMtUpper;

__device__ __forceinline__ unsigned long long mt_mix(unsigned long long hi, unsigned long long lo) {
  const unsigned long long y = (hi & kMtUpper) | (lo & kMtLower);
  return (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}
__device__ __forceinline__ unsigned long long mt_temper(unsigned long long z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71d67fffeda60000ull;
  z ^= (z << 37) & 0xfff7eee000000000ull;
  z ^= z >> 43;
  return z;
}

// One CTA per env being reset: its particles (upload order) get the jittered
// lattice positions of box [lo, hi] drawn from mt19937_64(seed), written to
// pos[3 * pid] in double. Draw d belongs to particle d / 3, component 2 - d % 3
// (GCC evaluates Vec3(jitter, jitter, jitter) right to left).
__global__ void __launch_bounds__(kMtN) k_seed_lattice(const int* envs, const unsigned long long* seeds,
                                                        const double* boxes, const long long* env_off,
                                                        double spacing, int cx, int cy, double* pos) {
  __shared__ unsigned long long mt[kMtN];
  __shared__ double jit[kMtN];
  const int r = blockIdx.x, t = threadIdx.x;
  const int env = envs[r];
  const double* box = boxes + 6 * r;
  const long long first = env_off[env], n = env_off[env + 1] - first;
  if (t == 0) {  // std::mersenne_twister_engine::seed (sequential recurrence)
    mt[0] = seeds[r];
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (unsigned long long)i;
  }
  const double a = -0.25 * spacing, b = 0.25 * spacing;
  const long long draws = 3 * n;
  for (long long d0 = 0; d0 < draws; d0 += kMtN) {
    __syncthreads();
    unsigned long long v = 0;  // phase 1: k < n - m, old words only
    if (t < kMtN - kMtM) v = mt[t + kMtM] ^ mt_mix(mt[t], mt[t + 1]);
    __syncthreads();
    if (t < kMtN - kMtM) mt[t] = v;
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN - 1) v = mt[t - (kMtN - kMtM)] ^ mt_mix(mt[t], mt[t + 1]);  // phase 2
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN - 1) mt[t] = v;
    __syncthreads();
    if (t == kMtN - 1) mt[t] = mt[kMtM - 1] ^ mt_mix(mt[kMtN - 1], mt[0]);  // phase 3
    __syncthreads();
    double c = (double)mt_temper(mt[t]) / 18446744073709551616.0;  // generate_canonical<double, 53>
    if (c >= 1.0) c = __longlong_as_double(0x3fefffffffffffffll);   // nextafter(1, 0)
    jit[t] = c * (b - a) + a;
    const long long d = d0 + t;
    if (d < draws) {
      const long long p = d / 3;
      const int comp = 2 - (int)(d % 3);
      const long long idx = comp == 0 ? p % cx : (comp == 1 ? (p / cx) % cy : p / ((long long)cx * cy));
      double q = box[comp] + spacing * ((double)idx + 0.5);
      q += jit[t];
      q = q < box[comp] ? box[comp] : q;              // cwiseMax(box_min)
      q = box[3 + comp] < q ? box[3 + comp] : q;      // cwiseMin(box_max)
      pos[3 * (first + p) + comp] = q;
    }
  }
}

// the reset envs' particle state from the seeded positions (flag per env)
__global__ void k_seed_apply(SimParams P, const unsigned char* env_reset, const double* pos, float mass, float vol0,
                             unsigned material) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  Particles& q = P.cur;
  const unsigned env = (q.meta[i] >> 8) & kEnvMask;
  if (!env_reset[env]) return;
  const long long j = q.pid[i];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    q.x[a][i] = (float)pos[3 * j + a];
    q.v[a][i] = 0.0f;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    q.C[k][i] = 0.0f;
    q.G[k][i] = 0.0f;
  }
  q.mass[i] = mass;
  q.vol0[i] = vol0;
  q.meta[i] = (env << 8) | (material & 0xFFu);  // lost flag cleared
  q.jp[i] = P.mats[material].model == msim_dev::kModelDruckerPrager ? 0.0f : 1.0f;  // fresh: J = 1, q = 0
}

inline unsigned nblk(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_bake(const double* tri, long long n_tri, const double* origin, double voxel, const int* dims,
                 const double* dirs, float* out, cudaStream_t s) {
  const long long nvox = (long long)dims[0] * dims[1] * dims[2];
  k_bake<<<nblk(nvox, kBakeT), kBakeT, 0, s>>>(tri, n_tri, d3{origin[0], origin[1], origin[2]}, voxel, dims[0],
                                                 dims[1], dims[2], d3{dirs[0], dirs[1], dirs[2]},
                                                 d3{dirs[3], dirs[4], dirs[5]}, d3{dirs[6], dirs[7], dirs[8]}, out);
}

void launch_seed(const SimParams& P, int n_reset, const int* envs, const unsigned long long* seeds,
                 const double* boxes, const long long* env_off, double spacing, int cx, int cy, double* pos,
                 const unsigned char* env_reset, float mass, float vol0, unsigned material, cudaStream_t s) {
  if (n_reset <= 0) return;
  k_seed_lattice<<<n_reset, kMtN, 0, s>>>(envs, seeds, boxes, env_off, spacing, cx, cy, pos);
  if (P.n > 0) k_seed_apply<<<nblk(P.n), 256, 0, s>>>(P, env_reset, pos, mass, vol0, material);
}

void launch_fill(const SimParams& P, const double* regions, unsigned long long* inside, unsigned long long* vmax_bits,
                 cudaStream_t s) {
  if (P.n > 0) k_fill<<<nblk(P.n), 256, 0, s>>>(P, regions, inside, vmax_bits);
}

void launch_heightmap(const SimParams& P, const double* regions, int nx, int ny, unsigned long long* maps,
                      cudaStream_t s) {
  if (P.n > 0) k_heightmap<<<nblk(P.n), 256, 0, s>>>(P, regions, nx, ny, maps);
}

void launch_iou(const double* maps, const double* targets, int n_env, int cells, double threshold, double* iou,
                int* success, cudaStream_t s) {
  if (n_env > 0) k_iou<<<n_env, 256, 0, s>>>(maps, targets, cells, threshold, iou, success);
}

void launch_positions(const SimParams& P, double* pos, cudaStream_t s) {
  if (P.n > 0) k_positions<<<nblk(P.n), 256, 0, s>>>(P, pos);
}

void launch_chamfer_side(const double* A, const long long* offA, long long max_na, const double* B,
                         const long long* offB, int n_env, double* mind, double* mean_out, cudaStream_t s) {
  if (n_env <= 0 || max_na <= 0) return;
  dim3 grid(nblk(max_na, kNnT * kNnQ), n_env);
  k_nearest<<<grid, kNnT, 0, s>>>(A, offA, B, offB, mind);
  k_segment_mean<<<n_env, 256, 0, s>>>(mind, offA, mean_out);
}

}  // namespace msim_impl
