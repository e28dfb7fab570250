// B200 (sm_100a) kernels of the MLS-MPM soft-body substep.
//
// One CFL cycle of soft_substep (mpm.hpp:410-418) is the pipeline
//   clear -> bin -> scan -> scatter -> P2G -> compact -> grid -> G2P -> end
// over all environments of a context at once:
//   k_clear    zero the node blocks touched by the previous cycle (the
//              reference clears the whole dense grid, mpm.hpp:411)
//   k_bin      base cell in fp64 (bit-exact with mpm.hpp:222-231), lost
//              detection (:239-245), bucket key = (env, 4^3 node block of
//              base), warp-aggregated bucket counts
//   scan       bucket offsets + active bucket list
//   k_scatter  bucket permutation
//   k_p2g      one CTA per active bucket: gathers its particles, writes them
//              in bucket order to the other state buffer, evaluates the
//              penalty hook (coupling.hpp:151-172), Hencky stress
//              (mpm.hpp:152-161) and scatters mass/momentum/force into a
//              6^3-node shared-memory tile, flushed with vector REDs
//   k_grid     momentum -> velocity, gravity, grid-mode penalty
//              (coupling.hpp:186-214), boundary bands (mpm.hpp:315-342)
//   k_g2p      APIC/MLS gather, advection, F update, von Mises return map
//              (mpm.hpp:346-379, :166-181), NaN check, per-env max speed
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdio>

#include "msim_internal.h"

using namespace msim_dev;

namespace msim_impl {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned float_bits_max(unsigned* addr, float v) {
  // v >= 0: IEEE bit patterns of non-negative floats order like unsigned ints.
  return atomicMax(addr, __float_as_uint(v));
}

__device__ __forceinline__ void set_error(SimParams& P, int env, int code, int pid) {
  // Lower code wins only if none is set; invalid (2) and diverged (3) both latch.
  atomicCAS(&P.err_code[env], 0, code);
  atomicMin(&P.err_pid[env], pid);
}

__device__ __forceinline__ bool env_active(const SimParams& P, int env) {
  return P.manual || P.cycle < P.cycles[env];
}

__device__ __forceinline__ float env_dt(const SimParams& P, int env) {
  return P.manual ? P.dt_manual : P.dt_cycle[env];
}

// Base cell and fractional offset, computed exactly like mpm.hpp:222-225 in
// double from the fp32 position (exact promotion).
__device__ __forceinline__ void base_of(const SimParams& P, float x, float y, float z, int* b,
                                        float* fx) {
  double lx = ((double)x - P.origin[0]) * P.inv_h;
  double ly = ((double)y - P.origin[1]) * P.inv_h;
  double lz = ((double)z - P.origin[2]) * P.inv_h;
  double fbx = floor(lx - 0.5), fby = floor(ly - 0.5), fbz = floor(lz - 0.5);
  b[0] = (int)fbx;
  b[1] = (int)fby;
  b[2] = (int)fbz;
  fx[0] = (float)(lx - fbx);
  fx[1] = (float)(ly - fby);
  fx[2] = (float)(lz - fbz);
}

__device__ __forceinline__ bool base_in_range(const SimParams& P, const int* b) {
  return b[0] >= 0 && b[1] >= 0 && b[2] >= 0 && b[0] <= P.dims[0] - 3 && b[1] <= P.dims[1] - 3 &&
         b[2] <= P.dims[2] - 3;
}

__device__ __forceinline__ f3 load3(float* const* a, long long i) {
  return {a[0][i], a[1][i], a[2][i]};
}

// ---------------------------------------------------------------------------
// Scan (exclusive) with optional compaction of non-zero entries.
constexpr int kScanTile = 2048;  // 256 threads x 8 items

__device__ __forceinline__ int warp_incl_scan(int v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim = 256).
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
  __shared__ int ws[8];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int s = lane < 8 ? ws[lane] : 0;
    int si = warp_incl_scan(s);
    if (lane < 8) ws[lane] = si - s;
    if (lane == 7) *total = si;
  }
  __syncthreads();
  int r = inc - v + ws[wid];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) k_scan_reduce(const int* in, int n, int* tsum, int* tcnt) {
  int base = blockIdx.x * kScanTile + threadIdx.x * 8;
  int s = 0, c = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = base + k;
    int v = i < n ? in[i] : 0;
    s += v;
    c += v != 0;
  }
  __shared__ int tot;
  int ex = block_excl_scan(s, &tot);
  (void)ex;
  __shared__ int totc;
  int exc = block_excl_scan(c, &totc);
  (void)exc;
  if (threadIdx.x == 0) {
    tsum[blockIdx.x] = tot;
    tcnt[blockIdx.x] = totc;
  }
}

__global__ void __launch_bounds__(256) k_scan_top(int* tsum, int* tcnt, int ntiles) {
  // exclusive scan of tile sums in place, chunks of 256*8
  __shared__ int carry_s, carry_c;
  if (threadIdx.x == 0) carry_s = carry_c = 0;
  __syncthreads();
  for (int start = 0; start < ntiles; start += kScanTile) {
    int vs[8], vc[8];
    int ss = 0, sc = 0;
    int b = start + threadIdx.x * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      vs[k] = b + k < ntiles ? tsum[b + k] : 0;
      vc[k] = b + k < ntiles ? tcnt[b + k] : 0;
      ss += vs[k];
      sc += vc[k];
    }
    __shared__ int ts, tc;
    int es = block_excl_scan(ss, &ts);
    int ec = block_excl_scan(sc, &tc);
    int rs = carry_s + es, rc = carry_c + ec;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (b + k < ntiles) {
        tsum[b + k] = rs;
        tcnt[b + k] = rc;
      }
      rs += vs[k];
      rc += vc[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_s += ts;
      carry_c += tc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_scan_apply(const int* in, int n, int* out, const int* tsum,
                                                    const int* tcnt, int* list, int* n_list,
                                                    int ntiles) {
  int base = blockIdx.x * kScanTile + threadIdx.x * 8;
  int v[8];
  int s = 0, c = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
    c += v[k] != 0;
  }
  __shared__ int tot, totc;
  int es = block_excl_scan(s, &tot) + tsum[blockIdx.x];
  int ec = block_excl_scan(c, &totc) + tcnt[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int i = base + k;
    if (i < n) {
      out[i] = es;
      if (list && v[k] != 0) list[ec++] = i;
    }
    es += v[k];
  }
  if (blockIdx.x == ntiles - 1 && threadIdx.x == 0) {
    out[n] = tsum[blockIdx.x] + tot;
    if (n_list) *n_list = tcnt[blockIdx.x] + totc;
  }
}

// ---------------------------------------------------------------------------
// Particle upload / download.

__global__ void k_convert_in(SimParams P, long long n, const double* x, const double* v,
                             const double* F, const double* C, const double* mass,
                             const double* vol0, const int32_t* mat, const int* env_of,
                             long long first_pid) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  long long i = first_pid + j;  // storage index == pid at upload
  Particles& q = P.cur;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    q.x[a][i] = (float)x[3 * j + a];
    q.v[a][i] = v ? (float)v[3 * j + a] : 0.0f;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    q.C[k][i] = C ? (float)C[9 * j + k] : 0.0f;
    double f = F ? F[9 * j + k] : ((k % 4 == 0) ? 1.0 : 0.0);
    q.G[k][i] = (float)(f - ((k % 4 == 0) ? 1.0 : 0.0));
  }
  q.mass[i] = (float)mass[j];
  q.vol0[i] = (float)vol0[j];
  unsigned m = mat ? (unsigned)mat[j] : 0u;
  q.meta[i] = ((unsigned)env_of[j] << 8) | (m & 0xFFu);
  q.pid[i] = (int)i;
}

__global__ void k_overwrite(SimParams P, int env, long long first_pid, long long n,
                            const double* x, const double* v, const double* F, const double* C) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  Particles& q = P.cur;
  long long j = (long long)q.pid[i] - first_pid;
  if (j < 0 || j >= n) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (x) q.x[a][i] = (float)x[3 * j + a];
    if (v) q.v[a][i] = (float)v[3 * j + a];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (C) q.C[k][i] = (float)C[9 * j + k];
    if (F) q.G[k][i] = (float)(F[9 * j + k] - ((k % 4 == 0) ? 1.0 : 0.0));
  }
}

__global__ void k_convert_out(SimParams P, long long first_pid, long long n, double* x, double* v,
                              double* F, double* C, uint8_t* lost) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const Particles& q = P.cur;
  long long j = (long long)q.pid[i] - first_pid;
  if (j < 0 || j >= n) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (x) x[3 * j + a] = (double)q.x[a][i];
    if (v) v[3 * j + a] = (double)q.v[a][i];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    if (C) C[9 * j + k] = (double)q.C[k][i];
    if (F) F[9 * j + k] = (double)q.G[k][i] + ((k % 4 == 0) ? 1.0 : 0.0);
  }
  if (lost) lost[j] = (uint8_t)(q.meta[i] >> kLostBit);
}

// ---------------------------------------------------------------------------
// CFL planning (mpm.hpp:386-409).

__global__ void k_vmax(SimParams P) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  unsigned meta = P.cur.meta[i];
  if (meta >> kLostBit) return;
  int env = (meta >> 8) & kEnvMask;
  f3 v = load3(P.cur.v, i);
  float_bits_max(&P.vmax_bits[env], norm(v));
}

__global__ void k_plan(SimParams P, double dt, double cfl_h, int max_halvings, int* max_cycles,
                       int* any_err, int* cyc_sum) {
  int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= P.n_env) return;
  double vmax = (double)__uint_as_float(P.vmax_bits[env]);
  int halvings = 0;
  while (halvings < max_halvings && vmax * dt / (1 << halvings) > cfl_h) ++halvings;
  int* cyc = const_cast<int*>(P.cycles);
  float* dtc = const_cast<float*>(P.dt_cycle);
  if (vmax * dt / (1 << halvings) > cfl_h) {
    set_error(P, env, kErrCfl, 0x7fffffff);
    cyc[env] = 0;
  } else {
    cyc[env] = 1 << halvings;
    dtc[env] = (float)(dt / (1 << halvings));
    if (cyc_sum) cyc_sum[env] += 1 << halvings;
    atomicMax(max_cycles, 1 << halvings);
  }
  if (P.err_code[env]) atomicOr(any_err, 1);
}

// ---------------------------------------------------------------------------
// Cycle kernels.

__global__ void __launch_bounds__(256) k_clear(SimParams P) {
  int nlist = *P.n_nb;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)nlist * 64;
       t += (long long)gridDim.x * blockDim.x) {
    int item = (int)(t >> 6), l = (int)(t & 63);
    int nb = P.nb_list[item];
    int env = nb / P.blocks_per_env, lb = nb - env * P.blocks_per_env;
    int bx = lb % P.bdims[0], by = (lb / P.bdims[0]) % P.bdims[1], bz = lb / (P.bdims[0] * P.bdims[1]);
    int gx = bx * 4 + (l & 3), gy = by * 4 + ((l >> 2) & 3), gz = bz * 4 + (l >> 4);
    if (gx >= P.dims[0] || gy >= P.dims[1] || gz >= P.dims[2]) continue;
    long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
    P.gPM[gi] = z;
    if (P.gF) P.gF[gi] = z;
    P.gV[gi] = z;
    if (l == 0) P.nb_flag[nb] = 0;
  }
}

// Newly lost particle: penalty reaction (the hook runs before p2g detects
// loss, coupling.hpp:266-274), freeze, count (mpm.hpp:239-245).
__device__ void penalty_reaction_only(SimParams& P, int env, f3 x, f3 v) {
  int s0 = P.shape_off[env], s1 = P.shape_off[env + 1];
  int b0 = P.body_off[env];
  for (int s = s0; s < s1; ++s) {
    const ShapeDev& sh = P.shapes[s];
    f3 f;
    float pen;
    if (!penalty_force(sh, P.vol_pool, x, v, P.r_c_particle, P.c_d, f, pen)) continue;
    f3 com = {sh.com[0], sh.com[1], sh.com[2]};
    f3 tq = cross(x - com, f3{-f.x, -f.y, -f.z});
    double* wr = P.wrench + 6 * (b0 + sh.body);
    atomicAdd(wr + 0, -(double)f.x);
    atomicAdd(wr + 1, -(double)f.y);
    atomicAdd(wr + 2, -(double)f.z);
    atomicAdd(wr + 3, (double)tq.x);
    atomicAdd(wr + 4, (double)tq.y);
    atomicAdd(wr + 5, (double)tq.z);
    atomicAdd(P.applied + 3 * env + 0, (double)f.x);
    atomicAdd(P.applied + 3 * env + 1, (double)f.y);
    atomicAdd(P.applied + 3 * env + 2, (double)f.z);
    atomicAdd(P.react + 3 * env + 0, -(double)f.x);
    atomicAdd(P.react + 3 * env + 1, -(double)f.y);
    atomicAdd(P.react + 3 * env + 2, -(double)f.z);
    float_bits_max(&P.max_pen_bits[env], pen);
  }
}

__global__ void __launch_bounds__(256) k_bin(SimParams P) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < P.n_env && env_active(P, (int)i)) P.vmax_bits[i] = 0u;
  if (i >= P.n) return;
  Particles& q = P.cur;
  unsigned meta = q.meta[i];
  int env = (meta >> 8) & kEnvMask;
  bool active = env_active(P, env);
  int key = P.n_keys - 1;
  int b[3] = {-10, -10, -10};
  if (!(meta >> kLostBit)) {
    float fx[3];
    f3 x = load3(q.x, i);
    base_of(P, x.x, x.y, x.z, b, fx);
    if (base_in_range(P, b)) {
      key = env * P.blocks_per_env +
            ((b[2] >> 2) * P.bdims[1] + (b[1] >> 2)) * P.bdims[0] + (b[0] >> 2);
    } else if (active) {
      if (!P.grid_mode && P.shape_off[env + 1] > P.shape_off[env])
        penalty_reaction_only(P, env, x, load3(q.v, i));
      q.meta[i] = meta | (1u << kLostBit);
      q.v[0][i] = q.v[1][i] = q.v[2][i] = 0.0f;
      atomicAdd((unsigned long long*)&P.lost_count[env], 1ull);
      b[0] = b[1] = b[2] = -10;
    }
  }
  if (P.base_dbg && active) {
    int p = q.pid[i];
    P.base_dbg[3 * p + 0] = b[0];
    P.base_dbg[3 * p + 1] = b[1];
    P.base_dbg[3 * p + 2] = b[2];
  }
  P.key[i] = key;
  // warp-aggregated bucket count: lanes with equal keys share one atomic
  unsigned peers = __match_any_sync(__activemask(), key);
  int leader = __ffs(peers) - 1;
  int lane = threadIdx.x & 31;
  int rank_in_peers = __popc(peers & ((1u << lane) - 1u));
  int basecnt = 0;
  if (lane == leader) basecnt = atomicAdd(&P.bucket_count[key], __popc(peers));
  basecnt = __shfl_sync(peers, basecnt, leader);
  P.rank[i] = basecnt + rank_in_peers;
}

__global__ void k_scatter(SimParams P) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  P.perm[P.bucket_start[P.key[i]] + P.rank[i]] = (int)i;
}

template <int SPLIT>
__global__ void __launch_bounds__(kThreads) k_p2g(SimParams P) {
  constexpr int NCH = SPLIT ? 7 : 4;
  constexpr int TN = 216;  // 6^3 nodes
  __shared__ float tile[NCH][TN];
  __shared__ double wsum[kMaxBodiesPerEnv * 6 + 6];
  __shared__ unsigned penmax;
  const int tid = threadIdx.x;
  const int nitems = *P.n_active_buckets;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int key = P.active_buckets[item];
    const int s = P.bucket_start[key], e = P.bucket_start[key + 1];
    const bool lostb = key == P.n_keys - 1;
    const int env = lostb ? 0 : key / P.blocks_per_env;
    const bool active = !lostb && env_active(P, env);
    const int lb = key - env * P.blocks_per_env;
    const int ox = 4 * (lb % P.bdims[0]), oy = 4 * ((lb / P.bdims[0]) % P.bdims[1]),
              oz = 4 * (lb / (P.bdims[0] * P.bdims[1]));
    const int s0 = lostb ? 0 : P.shape_off[env], s1 = lostb ? 0 : P.shape_off[env + 1];
    const bool penalty = active && !P.grid_mode && s1 > s0;
    const float dt = active ? env_dt(P, env) : 0.0f;
    __syncthreads();
    if (active) {
      for (int t = tid; t < NCH * TN; t += kThreads) (&tile[0][0])[t] = 0.0f;
      if (penalty)
        for (int t = tid; t < kMaxBodiesPerEnv * 6 + 6; t += kThreads) wsum[t] = 0.0;
      if (tid == 0) penmax = 0u;
    }
    __syncthreads();
    for (int j = s + tid; j < e; j += kThreads) {
      const int i = P.perm[j];
      // ---- load + reorder into the next buffer (bucket order)
      f3 x = load3(P.cur.x, i), v = load3(P.cur.v, i);
      float C[9], G[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        C[k] = P.cur.C[k][i];
        G[k] = P.cur.G[k][i];
      }
      const float m = P.cur.mass[i], V0 = P.cur.vol0[i];
      const unsigned meta = P.cur.meta[i];
      const int pid = P.cur.pid[i];
      P.nxt.x[0][j] = x.x; P.nxt.x[1][j] = x.y; P.nxt.x[2][j] = x.z;
      P.nxt.v[0][j] = v.x; P.nxt.v[1][j] = v.y; P.nxt.v[2][j] = v.z;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        P.nxt.C[k][j] = C[k];
        P.nxt.G[k][j] = G[k];
      }
      P.nxt.mass[j] = m;
      P.nxt.vol0[j] = V0;
      P.nxt.meta[j] = meta;
      P.nxt.pid[j] = pid;
      if (!active) continue;
      // ---- binning (same op order as k_bin)
      int b[3];
      float fx[3];
      base_of(P, x.x, x.y, x.z, b, fx);
      // ---- particle-mode penalty hook
      f3 fext = {0.f, 0.f, 0.f};
      if (penalty) {
        for (int sidx = s0; sidx < s1; ++sidx) {
          const ShapeDev& sh = P.shapes[sidx];
          f3 f;
          float pen;
          if (!penalty_force(sh, P.vol_pool, x, v, P.r_c_particle, P.c_d, f, pen)) continue;
          fext = fext + f;
          f3 com = {sh.com[0], sh.com[1], sh.com[2]};
          f3 tq = cross(x - com, f3{-f.x, -f.y, -f.z});
          double* ws = wsum + 6 * min(sh.body, kMaxBodiesPerEnv - 1);
          atomicAdd(ws + 0, -(double)f.x);
          atomicAdd(ws + 1, -(double)f.y);
          atomicAdd(ws + 2, -(double)f.z);
          atomicAdd(ws + 3, (double)tq.x);
          atomicAdd(ws + 4, (double)tq.y);
          atomicAdd(ws + 5, (double)tq.z);
          atomicMax(&penmax, __float_as_uint(pen));
        }
        if (fext.x != 0.f || fext.y != 0.f || fext.z != 0.f) {
          double* as = wsum + 6 * kMaxBodiesPerEnv;
          atomicAdd(as + 0, (double)fext.x);
          atomicAdd(as + 1, (double)fext.y);
          atomicAdd(as + 2, (double)fext.z);
        }
      }
      // ---- stress (uses F at the start of the substep)
      const MatParams mp = P.mats[meta & 0xFFu];
      if (!(det_I_plus(G) > 0.0f)) set_error(P, env, kErrDetStress, pid);
      float U[9], eps[3], tau[9];
      hencky_frame(G, U, eps);
      kirchhoff_from_frame(U, eps, mp, tau);
      const float sV = -P.d_inv_f * V0;
      const float h = P.h_f;
      float A[9], A2[9];
      f3 b1, b2;
      if (SPLIT) {
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          A[k] = h * m * C[k];
          A2[k] = h * sV * tau[k];
        }
        f3 fxv = {fx[0], fx[1], fx[2]};
        b1 = m * v - matvec(A, fxv);
        b2 = fext - matvec(A2, fxv);
      } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) A[k] = h * (m * C[k] + dt * sV * tau[k]);
        f3 fxv = {fx[0], fx[1], fx[2]};
        b1 = (m * v + dt * fext) - matvec(A, fxv);
      }
      float wx[3], wy[3], wz[3];
      bspline_w(fx[0], wx);
      bspline_w(fx[1], wy);
      bspline_w(fx[2], wz);
      const int lx = b[0] - ox, ly = b[1] - oy, lz = b[2] - oz;
#pragma unroll
      for (int dk = 0; dk < 3; ++dk) {
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          f3 row = {b1.x + A[1] * dj + A[2] * dk, b1.y + A[4] * dj + A[5] * dk,
                    b1.z + A[7] * dj + A[8] * dk};
          f3 row2;
          if (SPLIT)
            row2 = {b2.x + A2[1] * dj + A2[2] * dk, b2.y + A2[4] * dj + A2[5] * dk,
                    b2.z + A2[7] * dj + A2[8] * dk};
          const float wjk = wy[dj] * wz[dk];
#pragma unroll
          for (int di = 0; di < 3; ++di) {
            const float w = wx[di] * wjk;
            const int t = ((lz + dk) * 6 + (ly + dj)) * 6 + (lx + di);
            atomicAdd(&tile[0][t], w * (row.x + A[0] * di));
            atomicAdd(&tile[1][t], w * (row.y + A[3] * di));
            atomicAdd(&tile[2][t], w * (row.z + A[6] * di));
            atomicAdd(&tile[3][t], w * m);
            if (SPLIT) {
              atomicAdd(&tile[4][t], w * (row2.x + A2[0] * di));
              atomicAdd(&tile[5][t], w * (row2.y + A2[3] * di));
              atomicAdd(&tile[6][t], w * (row2.z + A2[6] * di));
            }
          }
        }
      }
    }
    __syncthreads();
    if (active) {
      for (int t = tid; t < TN; t += kThreads) {
        const float mass = tile[3][t];
        if (mass == 0.0f) continue;
        const int lx = t % 6, ly = (t / 6) % 6, lz = t / 36;
        const int gx = ox + lx, gy = oy + ly, gz = oz + lz;
        const long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
        atomicAdd(&P.gPM[gi], make_float4(tile[0][t], tile[1][t], tile[2][t], mass));
        if (SPLIT) atomicAdd(&P.gF[gi], make_float4(tile[4][t], tile[5][t], tile[6][t], 0.0f));
        const int nb = env * P.blocks_per_env + ((gz >> 2) * P.bdims[1] + (gy >> 2)) * P.bdims[0] + (gx >> 2);
        P.nb_flag[nb] = 1;
      }
      if (penalty) {
        const int b0 = P.body_off[env], nb = min(P.body_off[env + 1] - b0, kMaxBodiesPerEnv);
        for (int t = tid; t < nb * 6; t += kThreads) {
          double val = wsum[t];
          if (val != 0.0) atomicAdd(P.wrench + 6 * b0 + t, val);
        }
        if (tid < 3) {
          double a = wsum[6 * kMaxBodiesPerEnv + tid];
          if (a != 0.0) {
            atomicAdd(P.applied + 3 * env + tid, a);
            // reactions of this CTA: sum over its bodies of the force slots
            double r = 0.0;
            for (int bb = 0; bb < nb; ++bb) r += wsum[6 * bb + tid];
            atomicAdd(P.react + 3 * env + tid, r);
          }
        }
        if (tid == 0 && penmax) atomicMax(&P.max_pen_bits[env], penmax);
      }
    }
    if (tid == 0) P.bucket_count[key] = 0;
  }
}

// Grid update (mpm.hpp:315-342) + grid-mode penalty hook (coupling.hpp:186-214),
// one 64-thread group per touched node block.
__global__ void __launch_bounds__(256) k_grid(SimParams P) {
  const int nlist = *P.n_nb;
  const int lane = threadIdx.x & 31;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)nlist * 64;
       t += (long long)gridDim.x * blockDim.x) {
    const int item = (int)(t >> 6), l = (int)(t & 63);
    const int nb = P.nb_list[item];
    const int env = nb / P.blocks_per_env, lb = nb - env * P.blocks_per_env;
    const bool active = env_active(P, env);
    const int bx = lb % P.bdims[0], by = (lb / P.bdims[0]) % P.bdims[1],
              bz = lb / (P.bdims[0] * P.bdims[1]);
    const int gx = bx * 4 + (l & 3), gy = by * 4 + ((l >> 2) & 3), gz = bz * 4 + (l >> 4);
    const bool inside = gx < P.dims[0] && gy < P.dims[1] && gz < P.dims[2];
    const long long gi =
        env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
    float4 pm = inside ? P.gPM[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool live = active && inside && pm.w > 0.0f;
    const float dt = active ? env_dt(P, env) : 0.0f;
    f3 vel = {0.f, 0.f, 0.f};
    if (live) vel = (1.0f / pm.w) * f3{pm.x, pm.y, pm.z};  // momentum / mass (pre-force)
    if (P.split) {
      f3 f = {0.f, 0.f, 0.f};
      if (live) {
        float4 ff = P.gF[gi];
        f = {ff.x, ff.y, ff.z};
      }
      // grid-mode penalty at the node with its pre-force velocity
      if (P.grid_mode) {
        const int s0 = P.shape_off[env], s1 = P.shape_off[env + 1];
        const int b0 = P.body_off[env];
        const f3 xi = {(float)(P.origin[0] + P.h * gx), (float)(P.origin[1] + P.h * gy),
                       (float)(P.origin[2] + P.h * gz)};
        const float scale = P.mean_mass[env] > 0.0 ? (float)(pm.w / P.mean_mass[env]) : 1.0f;
        for (int sidx = s0; sidx < s1; ++sidx) {
          const ShapeDev& sh = P.shapes[sidx];
          f3 fp = {0.f, 0.f, 0.f};
          float pen = 0.0f;
          bool hit = live && penalty_force(sh, P.vol_pool, xi, vel, P.r_c_grid, P.c_d, fp, pen);
          if (hit) {
            fp = scale * fp;
            f = f + fp;
          } else {
            fp = {0.f, 0.f, 0.f};
          }
          // warp-level reduction of the reaction wrench for this shape's body
          unsigned any = __ballot_sync(0xffffffffu, hit);
          if (any) {
            f3 com = {sh.com[0], sh.com[1], sh.com[2]};
            f3 tq = cross(xi - com, f3{-fp.x, -fp.y, -fp.z});
            double r[6] = {-(double)fp.x, -(double)fp.y, -(double)fp.z, (double)tq.x, (double)tq.y,
                           (double)tq.z};
#pragma unroll
            for (int k = 0; k < 6; ++k)
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) r[k] += __shfl_xor_sync(0xffffffffu, r[k], o);
            unsigned pb = __float_as_uint(pen);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) pb = max(pb, __shfl_xor_sync(0xffffffffu, pb, o));
            if (lane == 0) {
              double* wr = P.wrench + 6 * (b0 + sh.body);
#pragma unroll
              for (int k = 0; k < 6; ++k) atomicAdd(wr + k, r[k]);
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                atomicAdd(P.react + 3 * env + k, r[k]);
                atomicAdd(P.applied + 3 * env + k, -r[k]);
              }
              atomicMax(&P.max_pen_bits[env], pb);
            }
          }
        }
        if (live) P.gF[gi] = make_float4(f.x, f.y, f.z, 0.0f);
      }
      if (live) {
        const float inv_m = 1.0f / pm.w;
        vel = vel + dt * (f3{P.gravity[0], P.gravity[1], P.gravity[2]} + inv_m * f);
      }
    } else if (live) {
      vel = vel + dt * f3{P.gravity[0], P.gravity[1], P.gravity[2]};
    }
    if (!live) continue;
    const int idx[3] = {gx, gy, gz};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (idx[ax] < 2) {
        if (!((P.boundary_slip >> (2 * ax)) & 1u)) {
          vel = {0.f, 0.f, 0.f};
        } else {
          float c = comp(vel, ax);
          if (c < 0.0f) vel = ax == 0 ? f3{0.f, vel.y, vel.z} : (ax == 1 ? f3{vel.x, 0.f, vel.z} : f3{vel.x, vel.y, 0.f});
        }
      }
      if (idx[ax] >= P.dims[ax] - 2) {
        if (!((P.boundary_slip >> (2 * ax + 1)) & 1u)) {
          vel = {0.f, 0.f, 0.f};
        } else {
          float c = comp(vel, ax);
          if (c > 0.0f) vel = ax == 0 ? f3{0.f, vel.y, vel.z} : (ax == 1 ? f3{vel.x, 0.f, vel.z} : f3{vel.x, vel.y, 0.f});
        }
      }
    }
    P.gV[gi] = make_float4(vel.x, vel.y, vel.z, 0.0f);
  }
}

__global__ void __launch_bounds__(256) k_g2p(SimParams P) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  float speed = -1.0f;
  int env = -1;
  if (i < P.n) {
    Particles& q = P.cur;
    const unsigned meta = q.meta[i];
    env = (meta >> 8) & kEnvMask;
    if (!(meta >> kLostBit) && env_active(P, env)) {
      const float dt = env_dt(P, env);
      f3 x = load3(q.x, i);
      int b[3];
      float fx[3];
      base_of(P, x.x, x.y, x.z, b, fx);
      float wx[3], wy[3], wz[3];
      bspline_w(fx[0], wx);
      bspline_w(fx[1], wy);
      bspline_w(fx[2], wz);
      const long long g0 = env * P.nodes_per_env;
      f3 vsum = {0.f, 0.f, 0.f};
      float S[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // sum w v off^T
#pragma unroll
      for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const long long rowi = g0 + ((long long)(b[2] + dk) * P.dims[1] + (b[1] + dj)) * P.dims[0] + b[0];
          const float wjk = wy[dj] * wz[dk];
#pragma unroll
          for (int di = 0; di < 3; ++di) {
            const float4 gv = P.gV[rowi + di];
            const float w = wx[di] * wjk;
            const f3 wv = {w * gv.x, w * gv.y, w * gv.z};
            vsum = vsum + wv;
            // off = (di, dj, dk)
            S[0] += wv.x * di; S[1] += wv.x * dj; S[2] += wv.x * dk;
            S[3] += wv.y * di; S[4] += wv.y * dj; S[5] += wv.y * dk;
            S[6] += wv.z * di; S[7] += wv.z * dj; S[8] += wv.z * dk;
          }
        }
      // C = (4/h) * sum w v (off - fx)^T = (4/h) (S - v fx^T)   (partition of unity)
      const float k4h = 4.0f / P.h_f;
      float C[9];
      const f3 vv = vsum;
      C[0] = k4h * (S[0] - vv.x * fx[0]); C[1] = k4h * (S[1] - vv.x * fx[1]); C[2] = k4h * (S[2] - vv.x * fx[2]);
      C[3] = k4h * (S[3] - vv.y * fx[0]); C[4] = k4h * (S[4] - vv.y * fx[1]); C[5] = k4h * (S[5] - vv.y * fx[2]);
      C[6] = k4h * (S[6] - vv.z * fx[0]); C[7] = k4h * (S[7] - vv.z * fx[1]); C[8] = k4h * (S[8] - vv.z * fx[2]);
      x = x + dt * vv;
      float G[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = q.G[k][i];
      bool bad = false;
      if (dt != 0.0f) {
        // G_trial = G + dt*C*(I + G)
        float Gn[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            Gn[r * 3 + c] = G[r * 3 + c] +
                            dt * (C[r * 3 + c] + C[r * 3 + 0] * G[0 * 3 + c] + C[r * 3 + 1] * G[1 * 3 + c] +
                                  C[r * 3 + 2] * G[2 * 3 + c]);
        if (!(det_I_plus(Gn) > 0.0f)) set_error(P, env, kErrDetReturn, q.pid[i]);
        float U[9], eps[3];
        hencky_frame(Gn, U, eps);
        von_mises_project(Gn, U, eps, P.mats[meta & 0xFFu]);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          G[k] = Gn[k];
          q.G[k][i] = Gn[k];
          bad |= !isfinite(Gn[k]);
        }
      }
      q.x[0][i] = x.x; q.x[1][i] = x.y; q.x[2][i] = x.z;
      q.v[0][i] = vv.x; q.v[1][i] = vv.y; q.v[2][i] = vv.z;
#pragma unroll
      for (int k = 0; k < 9; ++k) q.C[k][i] = C[k];
      bad |= !isfinite(x.x) || !isfinite(x.y) || !isfinite(x.z) || !isfinite(vv.x) ||
             !isfinite(vv.y) || !isfinite(vv.z);
      if (bad) set_error(P, env, kErrNan, q.pid[i]);
      speed = norm(vv);
      if (!(speed >= 0.0f)) speed = FLT_MAX;  // NaN speed: CFL will also fail
    }
  }
  // per-env max speed, warp-aggregated when the warp is env-uniform
  const unsigned full = 0xffffffffu;
  const int env0 = __shfl_sync(full, env, 0);
  const bool uniform = __all_sync(full, env == env0 || speed < 0.0f);
  if (uniform) {
    float s = speed;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmaxf(s, __shfl_xor_sync(full, s, o));
    if ((threadIdx.x & 31) == 0 && s >= 0.0f && env0 >= 0) float_bits_max(&P.vmax_bits[env0], s);
  } else if (speed >= 0.0f) {
    float_bits_max(&P.vmax_bits[env], speed);
  }
}

// Per-env end of cycle: force-balance diagnostic (coupling.hpp:268-273) and
// the lost-fraction check (mpm.hpp:246-249).
__global__ void k_cycle_end(SimParams P, double* balance_max, double lost_threshold) {
  int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= P.n_env || !env_active(P, env)) return;
  double ex = P.applied[3 * env] + P.react[3 * env];
  double ey = P.applied[3 * env + 1] + P.react[3 * env + 1];
  double ez = P.applied[3 * env + 2] + P.react[3 * env + 2];
  double e = sqrt(ex * ex + ey * ey + ez * ez);
  if (e > balance_max[env]) balance_max[env] = e;
  for (int k = 0; k < 3; ++k) P.applied[3 * env + k] = P.react[3 * env + k] = 0.0;
  long long n_env_p = P.env_off[env + 1] - P.env_off[env];
  if (n_env_p > 0 && (double)P.lost_count[env] / (double)n_env_p > lost_threshold)
    set_error(P, env, kErrLost, 0x7fffffff);
}

// ---------------------------------------------------------------------------
// Rigid step on device (rigid.hpp:52-66, coupling.hpp:106-117).

struct dq {
  double w, x, y, z;
};
__device__ __forceinline__ dq qmul(dq a, dq b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ dq qnormcanon(dq q) {
  double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  q = {q.w / n, q.x / n, q.y / n, q.z / n};
  if (q.w < 0.0) q = {-q.w, -q.x, -q.y, -q.z};
  return q;
}
__device__ __forceinline__ void qrot(dq q, const double* v, double* out) {
  double uvx = q.y * v[2] - q.z * v[1], uvy = q.z * v[0] - q.x * v[2], uvz = q.x * v[1] - q.y * v[0];
  uvx *= 2; uvy *= 2; uvz *= 2;
  out[0] = v[0] + q.w * uvx + (q.y * uvz - q.z * uvy);
  out[1] = v[1] + q.w * uvy + (q.z * uvx - q.x * uvz);
  out[2] = v[2] + q.w * uvz + (q.x * uvy - q.y * uvx);
}
__device__ __forceinline__ void qmat(dq q, double* R) {
  double tx = 2 * q.x, ty = 2 * q.y, tz = 2 * q.z;
  double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  R[0] = 1 - (tyy + tzz); R[1] = txy - twz; R[2] = txz + twy;
  R[3] = txy + twz; R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
  R[6] = txz - twy; R[7] = tyz + twx; R[8] = 1 - (txx + tyy);
}
__device__ __forceinline__ dq qexp(const double* aa) {
  double ang = sqrt(aa[0] * aa[0] + aa[1] * aa[1] + aa[2] * aa[2]);
  if (ang < 1e-14) {
    dq q = {1.0, 0.5 * aa[0], 0.5 * aa[1], 0.5 * aa[2]};
    double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
  }
  double s = sin(0.5 * ang) / ang;
  return {cos(0.5 * ang), s * aa[0], s * aa[1], s * aa[2]};
}

__device__ void advance_pose(BodyDev& b, double dt) {
  dq rot = {b.q[0], b.q[1], b.q[2], b.q[3]};
  double com[3];
  qrot(rot, b.com_off, com);
  for (int k = 0; k < 3; ++k) com[k] += b.t[k];
  double com_new[3] = {com[0] + dt * b.v[0], com[1] + dt * b.v[1], com[2] + dt * b.v[2]};
  double aa[3] = {b.w[0] * dt, b.w[1] * dt, b.w[2] * dt};
  dq d = qexp(aa);
  dq rn = qmul(d, rot);
  double n = sqrt(rn.w * rn.w + rn.x * rn.x + rn.y * rn.y + rn.z * rn.z);
  rn = {rn.w / n, rn.x / n, rn.y / n, rn.z / n};
  double rc[3];
  qrot(rn, b.com_off, rc);
  double t[3] = {com_new[0] - rc[0], com_new[1] - rc[1], com_new[2] - rc[2]};
  rn = qnormcanon(rn);  // Pose(q, t) canonicalizes
  b.q[0] = rn.w; b.q[1] = rn.x; b.q[2] = rn.y; b.q[3] = rn.z;
  for (int k = 0; k < 3; ++k) b.t[k] = t[k];
}

__global__ void k_rigid(SimParams P, BodyDev* bodies, const ShapeHost* shapes, double* pending,
                        int integrate, double dt_r, double gx, double gy, double gz, int only_env) {
  int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= P.n_env || (only_env >= 0 && env != only_env)) return;
  int b0 = P.body_off[env], b1 = P.body_off[env + 1];
  for (int bi = b0; bi < b1; ++bi) {
    BodyDev& b = bodies[bi];
    if (integrate) {
      if (b.mode == MSIM_BODY_DYNAMIC) {
        const double* wf = pending + 6 * bi;
        const double g[3] = {gx, gy, gz};
        for (int k = 0; k < 3; ++k) b.v[k] += dt_r * (g[k] + wf[k] / b.mass);
        dq rot = {b.q[0], b.q[1], b.q[2], b.q[3]};
        double R[9];
        qmat(rot, R);
        double I[9];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c)
            I[r * 3 + c] = R[r * 3 + 0] * b.inertia[0] * R[c * 3 + 0] +
                           R[r * 3 + 1] * b.inertia[1] * R[c * 3 + 1] +
                           R[r * 3 + 2] * b.inertia[2] * R[c * 3 + 2];
        double L[3] = {I[0] * b.w[0] + I[1] * b.w[1] + I[2] * b.w[2],
                       I[3] * b.w[0] + I[4] * b.w[1] + I[5] * b.w[2],
                       I[6] * b.w[0] + I[7] * b.w[1] + I[8] * b.w[2]};
        double rhs[3] = {wf[3] - (b.w[1] * L[2] - b.w[2] * L[1]), wf[4] - (b.w[2] * L[0] - b.w[0] * L[2]),
                         wf[5] - (b.w[0] * L[1] - b.w[1] * L[0])};
        double det = I[0] * (I[4] * I[8] - I[5] * I[7]) - I[1] * (I[3] * I[8] - I[5] * I[6]) +
                     I[2] * (I[3] * I[7] - I[4] * I[6]);
        double Inv[9] = {(I[4] * I[8] - I[5] * I[7]) / det, (I[2] * I[7] - I[1] * I[8]) / det,
                         (I[1] * I[5] - I[2] * I[4]) / det, (I[5] * I[6] - I[3] * I[8]) / det,
                         (I[0] * I[8] - I[2] * I[6]) / det, (I[2] * I[3] - I[0] * I[5]) / det,
                         (I[3] * I[7] - I[4] * I[6]) / det, (I[1] * I[6] - I[0] * I[7]) / det,
                         (I[0] * I[4] - I[1] * I[3]) / det};
        for (int k = 0; k < 3; ++k)
          b.w[k] += dt_r * (Inv[3 * k] * rhs[0] + Inv[3 * k + 1] * rhs[1] + Inv[3 * k + 2] * rhs[2]);
        advance_pose(b, dt_r);
      } else if (b.mode == MSIM_BODY_SCRIPTED) {
        advance_pose(b, dt_r);
      }
    }
    double* wr = P.wrench + 6 * bi;
    for (int k = 0; k < 6; ++k) wr[k] = 0.0;  // sync_rigid_to_soft resets wrenches
  }
  int s0 = P.shape_off[env], s1 = P.shape_off[env + 1];
  for (int si = s0; si < s1; ++si) {
    const ShapeHost& sh = shapes[si];
    const BodyDev& b = bodies[b0 + sh.body];
    dq bq = {b.q[0], b.q[1], b.q[2], b.q[3]};
    dq lq = {sh.lq[0], sh.lq[1], sh.lq[2], sh.lq[3]};
    // compose(body pose, local pose) -> canonical world pose (geometry.hpp:54-56)
    dq wq = qnormcanon(qmul(bq, lq));
    double wt[3];
    qrot(bq, sh.lt, wt);
    for (int k = 0; k < 3; ++k) wt[k] += b.t[k];
    // inverse (geometry.hpp:58-61)
    dq iq = {wq.w, -wq.x, -wq.y, -wq.z};
    double it[3];
    qrot(iq, wt, it);
    double R[9], Ri[9];
    qmat(wq, R);
    qmat(iq, Ri);
    ShapeDev& d = P.shapes[si];
    for (int k = 0; k < 9; ++k) {
      d.R[k] = (float)R[k];
      d.Rinv[k] = (float)Ri[k];
    }
    for (int k = 0; k < 3; ++k) d.tinv[k] = (float)(-it[k]);
    double com[3];
    qrot(bq, b.com_off, com);
    for (int k = 0; k < 3; ++k) {
      d.com[k] = (float)(com[k] + b.t[k]);
      d.vlin[k] = (float)b.v[k];
      d.vang[k] = (float)b.w[k];
    }
    for (int k = 0; k < 4; ++k) d.p[k] = (float)sh.p[k];
    d.friction = (float)sh.friction;
    d.k_n = (float)sh.k_n;
    d.k_t = (float)sh.k_t;
    d.type = sh.type;
    d.body = sh.body;
    for (int k = 0; k < 3; ++k) {
      d.vol_dims[k] = sh.vol_dims[k];
      d.vol_origin[k] = (float)sh.vol_origin[k];
    }
    d.vol_voxel = (float)sh.vol_voxel;
    d.vol_off = sh.vol_off;
  }
}

__global__ void k_stage(const double* wrench, double* pending, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n * 6) pending[t] = wrench[t];
}

// ---------------------------------------------------------------------------
// Test hook: constitutive functions on raw matrices (device code path).
__global__ void k_constitutive(MatParams m, long long n, const double* F, double* tau, double* Fp,
                               int* bad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float G[9];
  for (int k = 0; k < 9; ++k) G[k] = (float)(F[9 * i + k] - ((k % 4 == 0) ? 1.0 : 0.0));
  if (!(det_I_plus(G) > 0.0f)) {
    atomicOr(bad, 1);
    return;
  }
  float U[9], eps[3];
  hencky_frame(G, U, eps);
  if (tau) {
    float t[9];
    kirchhoff_from_frame(U, eps, m, t);
    for (int k = 0; k < 9; ++k) tau[9 * i + k] = t[k];
  }
  if (Fp) {
    von_mises_project(G, U, eps, m);
    for (int k = 0; k < 9; ++k) Fp[9 * i + k] = (double)G[k] + ((k % 4 == 0) ? 1.0 : 0.0);
  }
}

// ---------------------------------------------------------------------------
// Grid readback / write (dense per env).
__global__ void k_grid_out(SimParams P, int env, double* mass, double* mom, double* force, double* vel) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P.nodes_per_env) return;
  long long gi = env * P.nodes_per_env + t;
  float4 pm = P.gPM[gi];
  if (mass) mass[t] = pm.w;
  if (mom) { mom[3 * t] = pm.x; mom[3 * t + 1] = pm.y; mom[3 * t + 2] = pm.z; }
  if (force) {
    float4 f = P.gF ? P.gF[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    force[3 * t] = f.x; force[3 * t + 1] = f.y; force[3 * t + 2] = f.z;
  }
  if (vel) {
    float4 v = P.gV[gi];
    vel[3 * t] = v.x; vel[3 * t + 1] = v.y; vel[3 * t + 2] = v.z;
  }
}

__global__ void k_grid_vel_in(SimParams P, int env, const double* vel) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P.nodes_per_env) return;
  P.gV[env * P.nodes_per_env + t] =
      make_float4((float)vel[3 * t], (float)vel[3 * t + 1], (float)vel[3 * t + 2], 0.0f);
}

__global__ void k_clear_env_grid(SimParams P, int env) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < P.nodes_per_env) {
    long long gi = env * P.nodes_per_env + t;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    P.gPM[gi] = z;
    if (P.gF) P.gF[gi] = z;
    P.gV[gi] = z;
  }
  if (t < P.blocks_per_env) P.nb_flag[env * P.blocks_per_env + t] = 0;
}

// ---------------------------------------------------------------------------
// Reference-layout binning (mpm.hpp:251-280) rebuilt from the recorded base
// cells: counting sort by z-major bin with index-stable order, and the
// ascending active-node list.
__global__ void k_bin_count(const int* base, long long n, int bx, int by, int* count) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int* b = base + 3 * j;
  if (b[0] < 0) return;
  atomicAdd(&count[((long long)b[2] * by + b[1]) * bx + b[0]], 1);
}
__global__ void k_bin_place(const int* base, long long n, int bx, int by, int* cursor, int* cell_particles) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int* b = base + 3 * j;
  if (b[0] < 0) return;
  int pos = atomicAdd(&cursor[((long long)b[2] * by + b[1]) * bx + b[0]], 1);
  cell_particles[pos] = (int)j;
}
__global__ void k_bin_sort_cells(const int* cell_start, int nbins, int* cell_particles) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nbins) return;
  int s = cell_start[c], e = cell_start[c + 1];
  for (int a = s + 1; a < e; ++a) {  // insertion sort by particle index (stable order)
    int v = cell_particles[a];
    int k = a - 1;
    while (k >= s && cell_particles[k] > v) {
      cell_particles[k + 1] = cell_particles[k];
      --k;
    }
    cell_particles[k + 1] = v;
  }
}
__global__ void k_bin_mark_nodes(const int* cell_start, int bx, int by, int bz, int dx, int dy, int* node_flag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= bx * by * bz) return;
  if (cell_start[c] == cell_start[c + 1]) return;
  int x = c % bx, y = (c / bx) % by, z = c / (bx * by);
  for (int dk = 0; dk < 3; ++dk)
    for (int dj = 0; dj < 3; ++dj)
      for (int di = 0; di < 3; ++di) node_flag[((long long)(z + dk) * dy + (y + dj)) * dx + (x + di)] = 1;
}
__global__ void k_list_to_ll(const int* list, const int* n, long long* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < *n) out[t] = list[t];
}

inline unsigned nblk(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// Wraps the launches of one logical kernel with optional CUDA events.
struct Timed {
  KernelTimer* t;
  int id;
  cudaStream_t s;
  cudaEvent_t a;
  Timed(const SimParams& P, int id_, cudaStream_t s_, int nlaunch = 1) : t(P.timer), id(id_), s(s_), a(nullptr) {
    if (t) a = t->begin(s, nlaunch);
  }
  ~Timed() {
    if (t) t->end(id, a, s);
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// Launchers.

size_t scan_tmp_ints(int n) {
  int ntiles = (n + kScanTile - 1) / kScanTile;
  return 2 * (size_t)ntiles + 64;
}

void scan_exclusive(const int* in, int* out, int n, int* list, int* n_list, int* tmp, cudaStream_t s) {
  int ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles == 0) ntiles = 1;
  int* tsum = tmp;
  int* tcnt = tmp + ntiles;
  k_scan_reduce<<<ntiles, 256, 0, s>>>(in, n, tsum, tcnt);
  k_scan_top<<<1, 256, 0, s>>>(tsum, tcnt, ntiles);
  k_scan_apply<<<ntiles, 256, 0, s>>>(in, n, out, tsum, tcnt, list, n_list, ntiles);
}

void launch_convert_in(const SimParams& P, long long n, const double* x, const double* v,
                       const double* F, const double* C, const double* mass, const double* vol0,
                       const int32_t* mat, const int* env_of, long long first_pid, int,
                       cudaStream_t s) {
  if (n > 0) k_convert_in<<<nblk(n), 256, 0, s>>>(P, n, x, v, F, C, mass, vol0, mat, env_of, first_pid);
}
void launch_overwrite(const SimParams& P, int env, long long first_pid, long long n,
                      const double* x, const double* v, const double* F, const double* C,
                      cudaStream_t s) {
  (void)env;
  if (P.n > 0) k_overwrite<<<nblk(P.n), 256, 0, s>>>(P, env, first_pid, n, x, v, F, C);
}
void launch_convert_out(const SimParams& P, int, long long first_pid, long long n, double* x,
                        double* v, double* F, double* C, uint8_t* lost, cudaStream_t s) {
  if (P.n > 0) k_convert_out<<<nblk(P.n), 256, 0, s>>>(P, first_pid, n, x, v, F, C, lost);
}
void launch_vmax(const SimParams& P, cudaStream_t s) {
  cudaMemsetAsync(P.vmax_bits, 0, sizeof(unsigned) * P.n_env, s);
  Timed tm(P, kKVmax, s);
  if (P.n > 0) k_vmax<<<nblk(P.n), 256, 0, s>>>(P);
}
void launch_plan(const SimParams& P, double dt, double cfl_h, int max_halvings, int* max_cycles,
                 int* any_err, int* cyc_sum, cudaStream_t s) {
  Timed tm(P, kKPlan, s);
  k_plan<<<nblk(P.n_env), 256, 0, s>>>(P, dt, cfl_h, max_halvings, max_cycles, any_err, cyc_sum);
}

void launch_cycle(const SimParams& P, int stages, cudaStream_t s) {
  static int sm_count = 0;
  if (!sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (sm_count <= 0) sm_count = 148;
  }
  const unsigned persist = (unsigned)sm_count * 8;
  const int n_blocks = P.n_keys - 1;
  if (stages & kStageClear) {
    Timed tm(P, kKClear, s);
    k_clear<<<persist, 256, 0, s>>>(P);
  }
  if (stages & kStageBin) {
    {
      Timed tm(P, kKBin, s);
      k_bin<<<nblk(std::max<long long>(std::max<long long>(P.n, P.n_env), 1)), 256, 0, s>>>(P);
    }
    {
      Timed tm(P, kKBucketScan, s, 3);
      scan_exclusive(P.bucket_count, P.bucket_start, P.n_keys, P.active_buckets, P.n_active_buckets,
                     P.scan_tmp, s);
    }
    if (P.n > 0) {
      Timed tm(P, kKScatter, s);
      k_scatter<<<nblk(P.n), 256, 0, s>>>(P);
    }
  }
  if (stages & kStageP2G) {
    {
      Timed tm(P, kKP2G, s);
      if (P.split)
        k_p2g<1><<<persist, kThreads, 0, s>>>(P);
      else
        k_p2g<0><<<persist, kThreads, 0, s>>>(P);
    }
    Timed tm(P, kKBlockScan, s, 3);
    scan_exclusive(P.nb_flag, P.nb_scan, n_blocks, P.nb_list, P.n_nb, P.scan_tmp, s);
  }
  if (stages & kStageGrid) {
    Timed tm(P, kKGrid, s);
    k_grid<<<persist, 256, 0, s>>>(P);
  }
  if ((stages & kStageG2P) && P.n > 0) {
    Timed tm(P, kKG2P, s);
    k_g2p<<<nblk(P.n), 256, 0, s>>>(P);
  }
  if (stages & kStageEnd) {
    Timed tm(P, kKEnd, s);
    k_cycle_end<<<nblk(P.n_env), 256, 0, s>>>(P, P.balance_max, P.lost_threshold);
  }
}

void launch_rigid(const SimParams& P, BodyDev* bodies, const ShapeHost* shapes, double* pending,
                  int integrate, double dt_r, const double* g, int only_env, cudaStream_t s) {
  Timed tm(P, kKRigid, s);
  k_rigid<<<nblk(P.n_env), 256, 0, s>>>(P, bodies, shapes, pending, integrate, dt_r, g[0], g[1], g[2],
                                        only_env);
}
void launch_stage_wrenches(const SimParams& P, double* pending, int n_bodies, cudaStream_t s) {
  Timed tm(P, kKStage, s);
  if (n_bodies > 0) k_stage<<<nblk(6LL * n_bodies), 256, 0, s>>>(P.wrench, pending, n_bodies);
}
void launch_constitutive(const MatParams m, long long n, const double* F, double* tau, double* Fp,
                         int* bad, cudaStream_t s) {
  if (n > 0) k_constitutive<<<nblk(n), 256, 0, s>>>(m, n, F, tau, Fp, bad);
}
void launch_grid_out(const SimParams& P, int env, double* mass, double* mom, double* force,
                     double* vel, cudaStream_t s) {
  k_grid_out<<<nblk(P.nodes_per_env), 256, 0, s>>>(P, env, mass, mom, force, vel);
}
void launch_grid_vel_in(const SimParams& P, int env, const double* vel, cudaStream_t s) {
  k_grid_vel_in<<<nblk(P.nodes_per_env), 256, 0, s>>>(P, env, vel);
}
void launch_clear_env_grid(const SimParams& P, int env, cudaStream_t s) {
  k_clear_env_grid<<<nblk(std::max<long long>(P.nodes_per_env, P.blocks_per_env)), 256, 0, s>>>(P, env);
}
void launch_binning_out(const SimParams& P, int, long long, long long n_env_p, const int* base,
                        int* cell_count, int* cell_start, int* cell_particles, int* node_flag,
                        int* node_scan, int* node_list, int* n_list, long long* active_nodes,
                        int* tmp, cudaStream_t s) {
  const int bx = P.dims[0] - 2, by = P.dims[1] - 2, bz = P.dims[2] - 2;
  const int nbins = bx * by * bz;
  cudaMemsetAsync(cell_count, 0, sizeof(int) * (nbins + 1), s);
  if (n_env_p > 0) k_bin_count<<<nblk(n_env_p), 256, 0, s>>>(base, n_env_p, bx, by, cell_count);
  scan_exclusive(cell_count, cell_start, nbins, nullptr, nullptr, tmp, s);
  cudaMemcpyAsync(cell_count, cell_start, sizeof(int) * nbins, cudaMemcpyDeviceToDevice, s);
  if (n_env_p > 0) k_bin_place<<<nblk(n_env_p), 256, 0, s>>>(base, n_env_p, bx, by, cell_count, cell_particles);
  k_bin_sort_cells<<<nblk(nbins), 256, 0, s>>>(cell_start, nbins, cell_particles);
  cudaMemsetAsync(node_flag, 0, sizeof(int) * P.nodes_per_env, s);
  k_bin_mark_nodes<<<nblk(nbins), 256, 0, s>>>(cell_start, bx, by, bz, P.dims[0], P.dims[1], node_flag);
  scan_exclusive(node_flag, node_scan, (int)P.nodes_per_env, node_list, n_list, tmp, s);
  k_list_to_ll<<<nblk(P.nodes_per_env), 256, 0, s>>>(node_list, n_list, active_nodes);
}

}  // namespace msim_impl
