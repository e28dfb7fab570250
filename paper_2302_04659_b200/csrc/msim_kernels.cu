// Utility kernels of the B200 MPM library: the exclusive scan with
// compaction used for bucket offsets and active lists, upload/readback
// conversion between host AoS doubles and device fp32 SoA, the batch rigid
// step, the constitutive test hook, grid inspection and the reference-layout
// binning rebuild (mpm.hpp:251-280) used by the integer parity checks.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdio>

#include "msim_common.cuh"

using namespace msim_dev;

namespace msim_impl {

namespace {


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
  // per-model scalar (the oracle's init_model_state): fluid carries det F in J and no shear
  const int model = P.mats[m].model;
  if (model == msim_dev::kModelFluid) {
    double Fd[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Fd[k] = F ? F[9 * j + k] : ((k % 4 == 0) ? 1.0 : 0.0);
    const double J = Fd[0] * (Fd[4] * Fd[8] - Fd[5] * Fd[7]) - Fd[1] * (Fd[3] * Fd[8] - Fd[5] * Fd[6]) +
                     Fd[2] * (Fd[3] * Fd[7] - Fd[4] * Fd[6]);
    q.jp[i] = (float)J;
#pragma unroll
    for (int k = 0; k < 9; ++k) q.G[k][i] = 0.0f;
  } else {
    q.jp[i] = model == msim_dev::kModelDruckerPrager ? 0.0f : 1.0f;
  }
}

__global__ void k_overwrite(SimParams P, long long first_pid, long long n,
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
  if (F && P.mats[q.meta[i] & 0xFFu].model == msim_dev::kModelFluid) {  // as at upload: J = det F, no shear
    const double* f = F + 9 * j;
    q.jp[i] = (float)(f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
                      f[2] * (f[3] * f[7] - f[4] * f[6]));
#pragma unroll
    for (int k = 0; k < 9; ++k) q.G[k][i] = 0.0f;
  }
}

__global__ void k_jp_out(SimParams P, long long first_pid, long long n, double* jp) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  long long j = (long long)P.cur.pid[i] - first_pid;
  if (j < 0 || j >= n) return;
  jp[j] = P.cur.jp[i];
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
// Max particle speed over non-lost particles (mpm.hpp:386-391).

__global__ void k_vmax(SimParams P) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  unsigned meta = P.cur.meta[i];
  if (meta >> kLostBit) return;
  int env = (meta >> 8) & kEnvMask;
  f3 v = load3(P.cur.v, i);
  float_bits_max(&P.vmax_bits[env], norm(v));
}

__global__ void k_rigid_all(SimParams P, int integrate, int only_env) {
  int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env >= P.n_env || (only_env >= 0 && env != only_env)) return;
  rigid_env(P, env, integrate, 0, 1, env_range(P, env), P.run[env].rigid_idx, false, nullptr);
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
  float jp = m.model == msim_dev::kModelDruckerPrager ? 0.0f : 1.0f;
  if (m.model == msim_dev::kModelFluid) {  // J carries the volume, F no shear
    jp = det_I_plus(G);
    for (int k = 0; k < 9; ++k) G[k] = 0.0f;
  }
  Sym eps = (m.model == msim_dev::kModelVonMises || m.model == msim_dev::kModelDruckerPrager)
                ? hencky_strain(G) : Sym{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (tau) {
    const Sym t = stress_of(m.model, G, eps, jp, m);
    const float tm[9] = {t.a00, t.a01, t.a02, t.a01, t.a11, t.a12, t.a02, t.a12, t.a22};
    for (int k = 0; k < 9; ++k) tau[9 * i + k] = tm[k];
  }
  if (Fp) {
    if (m.model == msim_dev::kModelVonMises) von_mises_project_strain(G, eps, m);
    else if (m.model == msim_dev::kModelDruckerPrager) drucker_prager_project_strain(G, eps, jp, m);
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
    if (P.det) P.gPMd[gi] = make_longlong4(0, 0, 0, 0);
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

}  // namespace

// Single-pass exclusive scan with compaction (the contract of the 3-kernel scan
// above, one launch): tiles take ids in launch order from a counter, publish
// their aggregate, look back over predecessors' published aggregates /
// inclusive prefixes, publish their inclusive prefix, then write. Status word
// per tile: flag (2 bits: 1 aggregate, 2 inclusive) | sum (31 bits) | count (31).
constexpr unsigned long long kStAgg = 1ull << 62, kStIncl = 2ull << 62;
__device__ __forceinline__ unsigned long long st_pack(unsigned long long flag, int s, int c) {
  return flag | ((unsigned long long)(unsigned)s << 31) | (unsigned long long)(unsigned)c;
}
template <bool EARLY>
__global__ void __launch_bounds__(256) k_scan_1pass(int* in, int n, int* out, int* list, int* n_list, int ntiles,
                                                   unsigned long long* status, unsigned* ctr) {
  if (!EARLY) pdl_wait();
  pdl_trigger();
  __shared__ int tile_s, pre_s, pre_c;
  __shared__ bool last_s;
  if (threadIdx.x == 0) tile_s = (int)atomicAdd(&ctr[0], 1u);
  __syncthreads();
  const int tile = tile_s;
  const int base = tile * kScanTile + threadIdx.x * 8;
  // the thread's 8 items: two 16-byte loads when whole (base is a multiple of 8)
  const bool whole = base + 8 <= n;
  int v[8], sm = 0, c = 0;
  if (whole) {
    const int4 a = *reinterpret_cast<const int4*>(in + base), b = *reinterpret_cast<const int4*>(in + base + 4);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = base + k < n ? in[base + k] : 0;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sm += v[k];
    c += v[k] != 0;
  }
  __shared__ int tot_s, tot_c;
  int es = block_excl_scan(sm, &tot_s);
  int ec = block_excl_scan(c, &tot_c);
  if (threadIdx.x < 32) {  // warp-wide look-back: 32 predecessors' status words per step
    volatile unsigned long long* st = status;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    const unsigned long long kFlag = 3ull << 62, kIncl = 2ull << 62;
    int ps = 0, pc = 0;
    if (tile > 0) {
      if (lane == 0) {
        st[tile] = st_pack(kStAgg, tot_s, tot_c);
        __threadfence();
      }
      for (int top = tile - 1;; top -= 32) {
        const int idx = top - lane;  // lane 0: the nearest predecessor
        unsigned long long w = idx >= 0 ? st[idx] : kIncl;  // before tile 0: an empty inclusive prefix
        while (__any_sync(FULL, (w & kFlag) == 0))  // some predecessor not published yet
          if ((w & kFlag) == 0) w = st[idx];
        const unsigned incl = __ballot_sync(FULL, (w & kFlag) == kIncl);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // lanes 0..stop contribute
        int s = lane <= stop ? (int)((w >> 31) & 0x7fffffffull) : 0;
        int c = lane <= stop ? (int)(w & 0x7fffffffull) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s += __shfl_xor_sync(FULL, s, o);
          c += __shfl_xor_sync(FULL, c, o);
        }
        ps += s;
        pc += c;
        if (incl) break;
      }
    }
    if (lane == 0) {
      st[tile] = st_pack(kStIncl, ps + tot_s, pc + tot_c);
      __threadfence();
      pre_s = ps;
      pre_c = pc;
      if (tile == ntiles - 1) {
        out[n] = ps + tot_s;
        if (n_list) *n_list = pc + tot_c;
      }
    }
  }
  __syncthreads();
  es += pre_s;
  ec += pre_c;
  int o[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o[k] = es;
    es += v[k];
  }
  if (whole) {
    *reinterpret_cast<int4*>(out + base) = make_int4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<int4*>(out + base + 4) = make_int4(o[4], o[5], o[6], o[7]);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = base + k;
    if (i < n) {
      if (!whole) out[i] = o[k];
      if (v[k] != 0) in[i] = 0;  // consumed: counts/flags restart from zero
      if (list && v[k] != 0) list[ec++] = i;
    }
  }
  // the last tile to finish clears the status words and counters for the next call
  if (threadIdx.x == 0) {
    __threadfence();
    last_s = atomicAdd(&ctr[1], 1u) == (unsigned)ntiles - 1u;
  }
  __syncthreads();
  if (last_s) {
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) status[t] = 0ull;
    if (threadIdx.x == 0) ctr[0] = ctr[1] = 0u;
  }
  if (EARLY) pdl_wait();  // complete only after the predecessor (keeps the stream order)
}

// ---------------------------------------------------------------------------
// Launchers.

size_t scan_tmp_ints(int n) {
  int ntiles = (n + kScanTile - 1) / kScanTile;
  return 2 * (size_t)ntiles + 64;
}

void scan_exclusive(int* in, int* out, int n, int* list, int* n_list, int* tmp, cudaStream_t s, bool early) {
  int ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles == 0) ntiles = 1;
  // one launch: decoupled look-back over the tiles (status words + counters in tmp,
  // zero between calls: the last tile to finish resets them)
  launch_pdl(early ? k_scan_1pass<true> : k_scan_1pass<false>, ntiles, 256, 0, s, in, n, out, list, n_list, ntiles,
             reinterpret_cast<unsigned long long*>(tmp), reinterpret_cast<unsigned*>(tmp + 2 * ntiles));
}

void launch_convert_in(const SimParams& P, long long n, const double* x, const double* v,
                       const double* F, const double* C, const double* mass, const double* vol0,
                       const int32_t* mat, const int* env_of, long long first_pid, cudaStream_t s) {
  if (n > 0) k_convert_in<<<nblk(n), 256, 0, s>>>(P, n, x, v, F, C, mass, vol0, mat, env_of, first_pid);
}
void launch_overwrite(const SimParams& P, long long first_pid, long long n, const double* x,
                      const double* v, const double* F, const double* C, cudaStream_t s) {
  if (P.n > 0) k_overwrite<<<nblk(P.n), 256, 0, s>>>(P, first_pid, n, x, v, F, C);
}
void launch_jp_out(const SimParams& P, long long first_pid, long long n, double* jp, cudaStream_t s) {
  if (P.n > 0) k_jp_out<<<nblk(P.n), 256, 0, s>>>(P, first_pid, n, jp);
}
void launch_convert_out(const SimParams& P, long long first_pid, long long n, double* x, double* v,
                        double* F, double* C, uint8_t* lost, cudaStream_t s) {
  if (P.n > 0) k_convert_out<<<nblk(P.n), 256, 0, s>>>(P, first_pid, n, x, v, F, C, lost);
}
void launch_vmax(const SimParams& P, cudaStream_t s) {
  cudaMemsetAsync(P.vmax_bits, 0, sizeof(unsigned) * P.n_env, s);
  if (P.n > 0) k_vmax<<<nblk(P.n), 256, 0, s>>>(P);
}
void launch_rigid(const SimParams& P, int integrate, int only_env, cudaStream_t s) {
  k_rigid_all<<<nblk(P.n_env), 256, 0, s>>>(P, integrate, only_env);
}
void launch_stage_wrenches(const SimParams& P, int n_bodies, cudaStream_t s) {
  if (n_bodies > 0) k_stage<<<nblk(6LL * n_bodies), 256, 0, s>>>(P.wrench, P.pending, n_bodies);
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
void launch_binning_out(const SimParams& P, long long n_env_p, const int* base, int* cell_count,
                        int* cell_start, int* cell_particles, int* node_flag, int* node_scan,
                        int* node_list, int* n_list, long long* active_nodes, int* tmp, cudaStream_t s) {
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
