// C-ABI host implementation (include/msim_gpu.h): context, device memory,
// uploads/readbacks and the stepping loops that drive msim_kernels.cu.
//
// Stepping mirrors soft_substep (mpm.hpp:397-421) and the rigid/soft part of
// env_step (coupling.hpp:248-293). The CFL cycle count of each substep is
// decided on the device (k_plan); the host reads the batch maximum through
// pinned mapped memory once per substep and enqueues that many cycles.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "msim_internal.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu --nvtx

namespace {
// NVTX range of one ABI call (no-op without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace msim_impl;
using msim_dev::MatParams;
using msim_dev::ShapeDev;

namespace {

thread_local std::string g_create_error;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t b) {
    if (b <= bytes && p) return cudaSuccess;
    release();
    if (b == 0) b = 16;
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct CudaError {
  cudaError_t e;
  const char* what;
};

#define CK(expr)                                            \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) throw CudaError{_e, #expr};      \
  } while (0)

}  // namespace

struct msim_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  msim_soft_desc desc{};
  std::vector<msim_material> mats_h;
  int n_env = 0;
  double rigid_gravity[3] = {0, 0, -9.81};
  msim_coupling coupling{MSIM_COUPLING_PARTICLE, 0, 0.5, 10.0};
  int split_req = 0;
  int record_binning = 0;
  std::string err;

  // geometry derived from desc
  long long nodes_per_env = 0;
  int bdims[3] = {0, 0, 0};
  int blocks_per_env = 0;
  int n_keys = 0;
  int qf = 0;          // particle bucket = qf^3 node blocks (set_bucket_shape)
  int qf_request = 0;  // 0: chosen from the particle density at set_particles
  int split_r = 1;     // particle-kernel items per bucket (set_particles: small scenes > 1)
  size_t scan_tmp_half = 0;  // ints per scan status area (scan_tmp_d holds two)
  int qdims[3] = {0, 0, 0};
  int buckets_per_env = 0;

  // particles
  long long n = 0;
  std::vector<long long> env_off_h;
  DevBuf env_off_d, env_of_d;
  DevBuf pool_f[2], meta_b[2], pid_b[2];
  Particles buf[2]{};
  int cur = 0;
  std::vector<double> mean_mass_h;
  DevBuf mean_mass_d;
  bool vmax_valid = false;

  // bodies / shapes
  std::vector<std::vector<msim_body>> bodies_h;
  std::vector<std::vector<msim_shape>> shapes_h;
  std::vector<std::vector<std::vector<float>>> vol_h;
  int n_bodies = 0, n_shapes = 0;
  bool bodies_on_device = false;
  // set_bodies edits host copies only; the device tables are rebuilt once, at
  // the next device-side use (set_device), so configuring n envs is O(n) and
  // never disturbs the other envs' integrated poses or staged wrenches
  bool bodies_dirty = false;
  std::vector<std::vector<double>> wrench_h, pending_h;  // per env, 6 per body (while dirty)
  // deterministic mode (msim_gpu_set_deterministic)
  int det = 0;
  DevBuf gPMd_d, w64_d, a64_d, r64_d, det_bnd_d, det_mexp_d;
  // multi-GPU statistics (msim_dist.cu): NCCL communicator over the ranks, stats vector
  void* comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  DevBuf stats_d;
  int last_substeps = 0;
  // kinematic pose schedule of the next env_step (msim_gpu_set_kinematic_schedule)
  DevBuf sched_d, sched_mask_d;
  int sched_steps = 0;
  DevBuf bodies_d, shapes_host_d, shapes_d, shape_off_d, body_off_d, vol_pool_d, wrench_d, pending_d;

  // per env
  DevBuf mats_d, run_d, applied_d, react_d, max_pen_d, vmax_d, lost_d, err_code_d, err_pid_d, balance_d;
  bool perm_valid = false;   // bucket keys/perm describe the stored positions
  bool grid_clean = true;    // P2G accumulators are zero (fused stepping consumes them)

  // binning + grid
  int bset = 0;  // which of the two bucket-structure sets the next particle launch reads
  DevBuf bucket_start_d[2], active_buckets_d[2], n_active_d[2], perm_d[2];
  DevBuf key_d, rank_d, bucket_count_d, move_count_d,
      base_dbg_d;
  DevBuf gPM_d, gF_d, gV_d, nb_flag_d, nb_scan_d, nb_list_d, n_nb_d, scan_tmp_d;
  std::vector<char> env_grid_dirty;

  // device control words
  DevBuf ctl_d;          // [0] device redo flag

  double time = 0.0;
  KernelTimer timer;
  DevBuf tbuf[10];  // task-metric / seeding scratch, kept across calls (no per-call cudaMalloc)

  // CUDA graphs of a call's planned launch sequence (call_begin, P2G, n_sub
  // fused cycles), keyed by the exact kernel arguments they captured.
  struct CallGraph {
    SimParams p0;
    int n_sub, integrate, n_soft, cur0, bset0, cur1, bset1, seen;
    long long launches;
    cudaGraphExec_t exec;
  };
  std::vector<CallGraph> graphs;
  bool use_graphs = true;
  ~msim_gpu_ctx() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    nccl_comm_destroy(comm);
  }
};

namespace {

bool split_mode(const msim_gpu_ctx* c) {
  return c->split_req || c->coupling.mode == MSIM_COUPLING_GRID;
}

MatParams mat_params(const msim_material& m) {
  double mu = m.youngs / (2.0 * (1.0 + m.poisson));
  double lambda = m.youngs * m.poisson / ((1.0 + m.poisson) * (1.0 - 2.0 * m.poisson));
  MatParams p{};
  p.two_mu = (float)(2.0 * mu);
  p.lambda = (float)lambda;
  p.yield_thr = (float)(std::sqrt(2.0 / 3.0) * m.yield_stress);
  p.density = (float)m.density;
  p.model = m.model;
  const double sp = std::sin(m.yield_stress * 3.14159265358979323846 / 180.0);  // Drucker-Prager: angle
  const double alpha = std::sqrt(2.0 / 3.0) * 2.0 * sp / (3.0 - sp);
  p.dp_alpha = (float)alpha;
  p.dp_k = (float)((3.0 * lambda + 2.0 * mu) / (2.0 * mu) * alpha);
  p.bulk = (float)(m.youngs / (3.0 * (1.0 - 2.0 * m.poisson)));
  return p;
}

SimParams params(msim_gpu_ctx* c) {
  SimParams P{};
  P.timer = &c->timer;
  const msim_soft_desc& d = c->desc;
  P.h = d.h;
  P.inv_h = 1.0 / d.h;
  for (int a = 0; a < 3; ++a) {
    P.origin[a] = d.origin[a];
    P.dims[a] = d.dims[a];
    P.bdims[a] = c->bdims[a];
    P.gravity[a] = (float)d.gravity[a];
  }
  P.nodes_per_env = c->nodes_per_env;
  P.blocks_per_env = c->blocks_per_env;
  P.n_env = c->n_env;
  P.boundary_slip = 0;
  for (int f = 0; f < 6; ++f)
    if (d.boundary[f] == MSIM_BOUNDARY_SLIP) P.boundary_slip |= 1u << f;
  P.h_f = (float)d.h;
  P.d_inv_f = (float)(4.0 / (d.h * d.h));
  P.n = c->n;
  P.n_keys = c->n_keys;
  P.qf = c->qf;
  const int qb[3] = {kBX, kBY, kBZ};
  for (int a = 0; a < 3; ++a) {
    P.qdims[a] = c->qdims[a];
    int sh = 0;
    while ((1 << sh) < qb[a] * c->qf) ++sh;
    P.qshift[a] = sh;
  }
  P.buckets_per_env = c->buckets_per_env;
  P.n_blocks = c->n_env * c->blocks_per_env;
  P.any_model = 0;
  for (const auto& m : c->mats_h) P.any_model |= m.model != MSIM_MODEL_HENCKY_VON_MISES;
  P.split = split_mode(c) ? 1 : 0;
  P.split_r = c->det ? 1 : c->split_r;  // deterministic mode keeps stable in-kernel ranks
  P.grid_mode = c->coupling.mode == MSIM_COUPLING_GRID;
  P.r_c_particle = (float)(c->coupling.r_c_factor * d.h);
  P.r_c_grid = (float)std::max(c->coupling.r_c_factor * d.h, 0.65 * d.h);
  P.c_d = (float)c->coupling.c_d;
  P.dt_full = d.dt;
  P.cfl_h = d.cfl_factor * d.h;
  P.max_halvings = d.max_cfl_halvings;
  P.n_soft = 1;
  P.integrate_rigid = 0;
  P.clear_on_read = 1;
  for (int a = 0; a < 3; ++a) P.rigid_g[a] = c->rigid_gravity[a];
  P.dt_r = d.dt;
  P.sched = c->sched_steps ? c->sched_d.as<double>() : nullptr;
  P.sched_mask = c->sched_steps ? c->sched_mask_d.as<unsigned char>() : nullptr;
  P.sched_steps = c->sched_steps;
  P.n_bodies_total = c->n_bodies;
  P.run = c->run_d.as<EnvRun>();
  P.bodies = c->bodies_d.as<BodyDev>();
  P.shape_src = c->shapes_host_d.as<ShapeHost>();
  P.pending = c->pending_d.as<double>();
  P.n_running = nullptr;
  P.any_redo = c->ctl_d.as<int>();
  P.item_counter = c->ctl_d.as<int>() + 2;
  P.redo_pass = 0;
  P.hooks = 1;
  P.cur = c->buf[c->cur];
  P.nxt = c->buf[1 - c->cur];
  P.mats = c->mats_d.as<MatParams>();
  P.env_off = c->env_off_d.as<long long>();
  P.shape_off = c->shape_off_d.as<int>();
  P.body_off = c->body_off_d.as<int>();
  P.shapes = c->shapes_d.as<ShapeDev>();
  P.vol_pool = c->vol_pool_d.as<float>();
  P.wrench = c->wrench_d.as<double>();
  P.applied = c->applied_d.as<double>();
  P.react = c->react_d.as<double>();
  P.max_pen_bits = c->max_pen_d.as<unsigned>();
  P.vmax_bits = c->vmax_d.as<unsigned>();
  P.lost_count = c->lost_d.as<long long>();
  P.err_code = c->err_code_d.as<int>();
  P.err_pid = c->err_pid_d.as<int>();
  P.mean_mass = c->mean_mass_d.as<double>();
  P.det = c->det;
  P.gPMd = c->det ? c->gPMd_d.as<longlong4>() : nullptr;
  P.w64 = c->w64_d.as<long long>();
  P.a64 = c->a64_d.as<long long>();
  P.r64 = c->r64_d.as<long long>();
  P.det_bnd = c->det_bnd_d.as<unsigned>();
  P.det_mexp = c->det_mexp_d.as<int>();
  P.key = c->key_d.as<int>();
  P.rank = c->rank_d.as<int>();
  P.bucket_count = c->bucket_count_d.as<int>();
  P.move_count = c->move_count_d.as<int>();
  const int rs = c->bset, ws = 1 - c->bset;
  P.bucket_start = c->bucket_start_d[rs].as<int>();
  P.active_buckets = c->active_buckets_d[rs].as<int>();
  P.n_active_buckets = c->n_active_d[rs].as<int>();
  P.perm = c->perm_d[rs].as<int>();
  P.bucket_start_w = c->bucket_start_d[ws].as<int>();
  P.active_buckets_w = c->active_buckets_d[ws].as<int>();
  P.n_active_buckets_w = c->n_active_d[ws].as<int>();
  P.perm_w = c->perm_d[ws].as<int>();
  P.base_dbg = c->record_binning ? c->base_dbg_d.as<int>() : nullptr;
  P.gPM = c->gPM_d.as<float4>();
  P.gF = c->gF_d.as<float4>();
  P.gV = c->gV_d.as<float4>();
  P.nb_flag = c->nb_flag_d.as<int>();
  P.nb_scan = c->nb_scan_d.as<int>();
  P.nb_list = c->nb_list_d.as<int>();
  P.n_nb = c->n_nb_d.as<int>();
  P.scan_tmp = c->scan_tmp_d.as<int>();
  P.scan_tmp2 = P.scan_tmp + c->scan_tmp_half;
  P.balance_max = c->balance_d.as<double>();
  P.lost_threshold = d.lost_fraction_threshold;
  return P;
}

template <class F>
int guarded(msim_gpu_ctx* c, F&& f) {
  try {
    return f();
  } catch (const CudaError& e) {
    if (c) c->err = std::string("CUDA error ") + cudaGetErrorString(e.e) + " at " + e.what;
    return MSIM_ERR_DEVICE;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return MSIM_ERR_INVALID;
  }
}

void upload_bodies(msim_gpu_ctx* c);
// every device-side entry point comes through here: pending body edits land first
void set_device(msim_gpu_ctx* c) {
  CK(cudaSetDevice(c->device));
  if (c->bodies_dirty) {
    c->bodies_dirty = false;
    upload_bodies(c);
  }
}

int fail(msim_gpu_ctx* c, int code, const std::string& msg) {
  c->err = msg;
  return code;
}

void carve_particles(msim_gpu_ctx* c, int b, long long n) {
  // float fields: x3 v3 C9 G9 + mass + vol0 + jp = 27
  const size_t nf = 27;
  CK(c->pool_f[b].ensure(sizeof(float) * nf * (size_t)std::max<long long>(n, 1)));
  CK(c->meta_b[b].ensure(sizeof(uint32_t) * (size_t)std::max<long long>(n, 1)));
  CK(c->pid_b[b].ensure(sizeof(int32_t) * (size_t)std::max<long long>(n, 1)));
  float* f = c->pool_f[b].as<float>();
  size_t stride = (size_t)std::max<long long>(n, 1);
  Particles& q = c->buf[b];
  int k = 0;
  for (int a = 0; a < 3; ++a) q.x[a] = f + stride * k++;
  for (int a = 0; a < 3; ++a) q.v[a] = f + stride * k++;
  for (int a = 0; a < 9; ++a) q.C[a] = f + stride * k++;
  for (int a = 0; a < 9; ++a) q.G[a] = f + stride * k++;
  q.mass = f + stride * k++;
  q.vol0 = f + stride * k++;
  q.jp = f + stride * k++;
  q.meta = c->meta_b[b].as<uint32_t>();
  q.pid = c->pid_b[b].as<int32_t>();
}

void alloc_binning(msim_gpu_ctx* c) {
  long long n = std::max<long long>(c->n, 1);
  CK(c->key_d.ensure(sizeof(int) * n));
  CK(c->rank_d.ensure(sizeof(int) * n));
  CK(c->perm_d[0].ensure(sizeof(int) * n));
  CK(c->perm_d[1].ensure(sizeof(int) * n));
  if (c->record_binning) {
    CK(c->base_dbg_d.ensure(sizeof(int) * 3 * n));
    CK(cudaMemsetAsync(c->base_dbg_d.p, 0xff, sizeof(int) * 3 * n, c->stream));
  }
}

// Particle buckets of f^3 node blocks: the key space and its scan buffers.
// f = 2 for sparse scenes keeps a few hundred particles per bucket (one CTA
// round) instead of a few dozen, amortising the per-bucket tile load and flush.
void set_bucket_shape(msim_gpu_ctx* c, int f) {
  if (f == c->qf) return;
  const int kb[3] = {kBX, kBY, kBZ};
  for (int a = 0; a < 3; ++a) c->qdims[a] = (c->desc.dims[a] + kb[a] * f - 1) / (kb[a] * f);
  c->buckets_per_env = c->qdims[0] * c->qdims[1] * c->qdims[2];
  c->n_keys = c->n_env * c->buckets_per_env + 1;
  c->qf = f;
  CK(c->bucket_count_d.ensure(sizeof(int) * c->n_keys));
  CK(c->move_count_d.ensure(sizeof(int) * c->n_keys));
  CK(cudaMemset(c->move_count_d.p, 0, sizeof(int) * c->n_keys));
  for (int k = 0; k < 2; ++k) {
    CK(c->bucket_start_d[k].ensure(sizeof(int) * (c->n_keys + 1)));
    CK(c->active_buckets_d[k].ensure(sizeof(int) * c->n_keys));
    CK(c->n_active_d[k].ensure(sizeof(int)));
    CK(cudaMemset(c->n_active_d[k].p, 0, sizeof(int)));
  }
  CK(cudaMemset(c->bucket_count_d.p, 0, sizeof(int) * c->n_keys));
  const long long scan_n = std::max<long long>(std::max(c->n_keys, c->n_env * c->blocks_per_env),
                                               std::min<long long>(c->nodes_per_env + 1, INT_MAX));
  // two status areas: the node-block scan runs concurrently with the bucket scan
  c->scan_tmp_half = scan_tmp_ints((int)scan_n);
  CK(c->scan_tmp_d.ensure(sizeof(int) * 2 * c->scan_tmp_half));
  CK(cudaMemset(c->scan_tmp_d.p, 0, sizeof(int) * 2 * c->scan_tmp_half));  // single-pass scan status
  CK(cudaDeviceSynchronize());
  c->perm_valid = false;
}

// Errors latched on the device: first env (lowest index) wins.
int collect_errors(msim_gpu_ctx* c) {
  std::vector<int> code(c->n_env), pid(c->n_env);
  CK(cudaMemcpyAsync(code.data(), c->err_code_d.p, sizeof(int) * c->n_env, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(pid.data(), c->err_pid_d.p, sizeof(int) * c->n_env, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int e = 0; e < c->n_env; ++e) {
    if (!code[e]) continue;
    long long local = pid[e] == INT_MAX ? -1 : pid[e] - c->env_off_h[e];
    std::string where = c->n_env > 1 ? " (env " + std::to_string(e) + ")" : "";
    switch (code[e]) {
      case kErrDetStress:
        return fail(c, MSIM_ERR_INVALID, "kirchhoff_stress: det(F) must be > 0 (particle " + std::to_string(local) + ")" + where);
      case kErrDetReturn:
        return fail(c, MSIM_ERR_INVALID, "von_mises_return_map: det(F) must be > 0 (particle " + std::to_string(local) + ")" + where);
      case kErrLost:
        return fail(c, MSIM_ERR_DIVERGED, "lost particle fraction exceeds threshold" + where);
      case kErrCfl:
        return fail(c, MSIM_ERR_DIVERGED, "CFL violation persists after max substep halvings" + where);
      case kErrDetRange:
        return fail(c, MSIM_ERR_DIVERGED, "deterministic fixed-point range exceeded" + where);
      case kErrNan:
        return fail(c, MSIM_ERR_DIVERGED, "NaN/Inf in particle " + std::to_string(local) + where);
      default:
        return fail(c, MSIM_ERR_DIVERGED, "simulation diverged" + where);
    }
  }
  return MSIM_OK;
}

void reset_errors(msim_gpu_ctx* c) {
  CK(cudaMemsetAsync(c->err_code_d.p, 0, sizeof(int) * c->n_env, c->stream));
  CK(cudaMemsetAsync(c->err_pid_d.p, 0x7f, sizeof(int) * c->n_env, c->stream));
}

// pull integrated body states back to the host copies
void download_bodies(msim_gpu_ctx* c) {
  if (!c->bodies_on_device || c->n_bodies == 0) return;
  std::vector<BodyDev> tmp(c->n_bodies);
  CK(cudaMemcpyAsync(tmp.data(), c->bodies_d.p, sizeof(BodyDev) * c->n_bodies, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int k = 0;
  for (int e = 0; e < c->n_env; ++e)
    for (auto& b : c->bodies_h[e]) {
      const BodyDev& d = tmp[k++];
      std::memcpy(b.q, d.q, sizeof b.q);
      std::memcpy(b.t, d.t, sizeof b.t);
      std::memcpy(b.v, d.v, sizeof b.v);
      std::memcpy(b.w, d.w, sizeof b.w);
    }
}

// Rebuild the concatenated body/shape tables of all envs on the device.
void upload_bodies(msim_gpu_ctx* c) {
  std::vector<int> boff(c->n_env + 1, 0), soff(c->n_env + 1, 0);
  std::vector<BodyDev> bd;
  std::vector<ShapeHost> sh;
  std::vector<float> pool;
  for (int e = 0; e < c->n_env; ++e) {
    boff[e] = (int)bd.size();
    soff[e] = (int)sh.size();
    for (const msim_body& b : c->bodies_h[e]) {
      BodyDev d{};
      d.mode = b.mode;
      std::memcpy(d.q, b.q, sizeof d.q);
      std::memcpy(d.t, b.t, sizeof d.t);
      std::memcpy(d.v, b.v, sizeof d.v);
      std::memcpy(d.w, b.w, sizeof d.w);
      d.mass = b.mass;
      std::memcpy(d.inertia, b.inertia, sizeof d.inertia);
      std::memcpy(d.com_off, b.com_offset, sizeof d.com_off);
      bd.push_back(d);
    }
    for (size_t s = 0; s < c->shapes_h[e].size(); ++s) {
      const msim_shape& in = c->shapes_h[e][s];
      ShapeHost o{};
      o.type = in.type;
      o.body = in.body;
      std::memcpy(o.lq, in.local_q, sizeof o.lq);
      std::memcpy(o.lt, in.local_t, sizeof o.lt);
      o.friction = in.friction;
      o.k_n = in.k_n;
      o.k_t = in.k_t;
      std::memcpy(o.p, in.params, sizeof o.p);
      if (in.type == MSIM_SHAPE_VOLUME) {
        for (int k = 0; k < 3; ++k) {
          o.vol_dims[k] = in.vol_dims[k];
          o.vol_origin[k] = in.vol_origin[k];
        }
        o.vol_voxel = in.vol_voxel;
        o.vol_off = (long long)pool.size();
        const auto& smp = c->vol_h[e][s];
        pool.insert(pool.end(), smp.begin(), smp.end());
        o.vol_min = smp.empty() ? 0.0 : (double)*std::min_element(smp.begin(), smp.end());
      }
      sh.push_back(o);
    }
  }
  boff[c->n_env] = (int)bd.size();
  soff[c->n_env] = (int)sh.size();
  c->n_bodies = (int)bd.size();
  c->n_shapes = (int)sh.size();
  cudaStream_t s = c->stream;
  CK(c->bodies_d.ensure(sizeof(BodyDev) * std::max<size_t>(bd.size(), 1)));
  CK(c->shapes_host_d.ensure(sizeof(ShapeHost) * std::max<size_t>(sh.size(), 1)));
  CK(c->shapes_d.ensure(sizeof(ShapeDev) * std::max<size_t>(sh.size(), 1)));
  CK(c->body_off_d.ensure(sizeof(int) * boff.size()));
  CK(c->shape_off_d.ensure(sizeof(int) * soff.size()));
  CK(c->vol_pool_d.ensure(sizeof(float) * std::max<size_t>(pool.size(), 1)));
  CK(c->wrench_d.ensure(sizeof(double) * 6 * std::max<size_t>(bd.size(), 1)));
  CK(c->pending_d.ensure(sizeof(double) * 6 * std::max<size_t>(bd.size(), 1)));
  CK(c->w64_d.ensure(sizeof(long long) * 6 * std::max<size_t>(bd.size(), 1)));
  CK(cudaMemsetAsync(c->w64_d.p, 0, sizeof(long long) * 6 * std::max<size_t>(bd.size(), 1), c->stream));
  if (!bd.empty()) CK(cudaMemcpyAsync(c->bodies_d.p, bd.data(), sizeof(BodyDev) * bd.size(), cudaMemcpyHostToDevice, s));
  if (!sh.empty()) CK(cudaMemcpyAsync(c->shapes_host_d.p, sh.data(), sizeof(ShapeHost) * sh.size(), cudaMemcpyHostToDevice, s));
  if (!pool.empty()) CK(cudaMemcpyAsync(c->vol_pool_d.p, pool.data(), sizeof(float) * pool.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->body_off_d.p, boff.data(), sizeof(int) * boff.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->shape_off_d.p, soff.data(), sizeof(int) * soff.size(), cudaMemcpyHostToDevice, s));
  // staged wrenches: carried over per env (zero for envs whose bodies were just set)
  std::vector<double> wr(6 * std::max<size_t>(bd.size(), 1), 0.0), pd(wr.size(), 0.0);
  if (!c->wrench_h.empty())
    for (int e = 0; e < c->n_env; ++e)
      for (size_t k = 0; k < c->wrench_h[e].size() && k < 6 * c->bodies_h[e].size(); ++k) {
        wr[6 * boff[e] + k] = c->wrench_h[e][k];
        pd[6 * boff[e] + k] = c->pending_h[e][k];
      }
  c->wrench_h.clear();
  c->pending_h.clear();
  CK(cudaMemcpyAsync(c->pending_d.p, pd.data(), sizeof(double) * pd.size(), cudaMemcpyHostToDevice, s));
  c->bodies_on_device = true;
  SimParams P = params(c);
  launch_rigid(P, 0, -1, s);  // world transforms of every shape (zeroes the accumulating wrenches ...)
  CK(cudaGetLastError());
  // ... which are then restored: only the re-configured envs start from zero
  CK(cudaMemcpyAsync(c->wrench_d.p, wr.data(), sizeof(double) * wr.size(), cudaMemcpyHostToDevice, s));
  // keep host storage alive until the copies land
  CK(cudaStreamSynchronize(s));
}

// Make the stored state ready for a P2G: bucket keys of the stored positions,
// clean P2G accumulators, a valid max speed for the CFL plan.
void prepare(msim_gpu_ctx* c, bool need_vmax) {
  cudaStream_t s = c->stream;
  SimParams P = params(c);
  if (!c->perm_valid) {
    launch_rebin(P, s);
    c->perm_valid = true;
  }
  if (!c->grid_clean) {
    launch_clear(P, s);
    for (int e = 0; e < c->n_env; ++e)
      if (c->env_grid_dirty[e]) launch_clear_env_grid(P, e, s);
    c->grid_clean = true;
  }
  for (int e = 0; e < c->n_env; ++e) c->env_grid_dirty[e] = 0;
  if (need_vmax && !c->vmax_valid) {
    launch_vmax(P, s);
    c->vmax_valid = true;
  }
  CK(cudaGetLastError());
}

// After a particle launch the other buffer holds the particles (bucket order).
void swap_buffers(msim_gpu_ctx* c) {
  c->cur ^= 1;
  c->bset ^= 1;  // the bucket structure built after the launch is read by the next one
}

// n_sub soft substeps of every env (soft_substep, mpm.hpp:397-421), or the
// rigid/soft part of env_step when integrate_rigid (coupling.hpp:248-293).
// Launch sequence: call_begin -> P2G -> grid, then one fused launch per cycle.
// The host syncs once at the end (more only when some env halved its step).
int step_call(msim_gpu_ctx* c, int n_sub, bool integrate_rigid, int n_soft, int32_t* cycles_out) {
  NvtxRange range(integrate_rigid ? "msim.env_step" : "msim.soft_substep");
  cudaStream_t s = c->stream;
  if (c->n == 0 || n_sub <= 0) return MSIM_OK;
  prepare(c, true);
  auto P = [&]() {
    SimParams q = params(c);
    q.integrate_rigid = integrate_rigid ? 1 : 0;
    q.n_soft = n_soft;
    q.dt_r = n_soft * c->desc.dt;
    q.clear_on_read = 1;
    return q;
  };
  // the planned sequence: replayed from a CUDA graph when the same call (same
  // kernel arguments) ran before; captured on its second occurrence
  auto plan = [&]() {
    launch_call_begin(P(), n_sub, kActP2G, s);
    launch_iteration(P(), false, true, s);
    swap_buffers(c);
    for (int k = 0; k < n_sub; ++k) {
      launch_iteration(P(), true, true, s);
      swap_buffers(c);
    }
  };
  const SimParams p0 = P();
  msim_gpu_ctx::CallGraph* g = nullptr;
  if (c->use_graphs && !c->timer.enabled) {
    for (auto& cg : c->graphs)
      if (cg.n_sub == n_sub && cg.integrate == (int)integrate_rigid && cg.n_soft == n_soft && cg.cur0 == c->cur &&
          cg.bset0 == c->bset && std::memcmp(&cg.p0, &p0, sizeof p0) == 0)
        g = &cg;
    if (!g) {
      if (c->graphs.size() >= 16) {
        for (auto& cg : c->graphs)
          if (cg.exec) cudaGraphExecDestroy(cg.exec);
        c->graphs.clear();
      }
      msim_gpu_ctx::CallGraph cg{};
      cg.p0 = p0;
      cg.n_sub = n_sub;
      cg.integrate = integrate_rigid;
      cg.n_soft = n_soft;
      cg.cur0 = c->cur;
      cg.bset0 = c->bset;
      c->graphs.push_back(cg);
      g = &c->graphs.back();
    }
  }
  if (g && g->exec) {
    CK(cudaGraphLaunch(g->exec, s));
    c->cur = g->cur1;
    c->bset = g->bset1;
    c->timer.launches += g->launches;
  } else if (g && g->seen >= 1) {
    const long long l0 = c->timer.launches;
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    plan();
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(&g->exec, graph, 0));
    CK(cudaGraphDestroy(graph));
    g->launches = c->timer.launches - l0;
    g->cur1 = c->cur;
    g->bset1 = c->bset;
    CK(cudaGraphLaunch(g->exec, s));
  } else {
    plan();
    if (g) ++g->seen;
  }
  int planned = n_sub;  // one launch per substep when no env halves its step
  int launched = n_sub;
  std::vector<EnvRun> run(c->n_env);
  int more = 0;
  for (int guard = 0; guard < 64; ++guard) {
    for (; launched < planned; ++launched) {  // beyond the plan: some env halved its step further
      launch_iteration(P(), true, true, s);
      swap_buffers(c);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(run.data(), c->run_d.p, sizeof(EnvRun) * c->n_env, cudaMemcpyDeviceToHost, s));
    {
      NvtxRange wait("msim.step_sync");
      CK(cudaStreamSynchronize(s));
    }
    c->timer.flush();
    more = 0;
    for (const EnvRun& r : run)
      if (r.substeps_left > 0) more = std::max(more, (r.cycles - r.cycle) + (r.substeps_left - 1));
    if (more == 0) break;
    planned += more;
  }
  c->vmax_valid = true;   // the last G2P accumulated it
  c->grid_clean = true;   // every P2G was consumed by a grid update
  c->perm_valid = true;
  if (cycles_out)
    for (int e = 0; e < c->n_env; ++e) cycles_out[e] = run[e].cycles;
  const int rc = collect_errors(c);
  if (rc != MSIM_OK) return rc;
  if (more > 0) {  // 64 host passes did not finish every env's substeps: never return a short step as OK
    for (int e = 0; e < c->n_env; ++e)
      if (run[e].substeps_left > 0)
        return fail(c, MSIM_ERR_DIVERGED, "substeps left unfinished after 64 launch passes (env " + std::to_string(e) + ")");
  }
  return MSIM_OK;
}

bool valid_material(const msim_material& m, std::string& why) {
  if (m.youngs <= 0.0) { why = "Material: E must be > 0"; return false; }
  if (m.poisson <= 0.0 || m.poisson >= 0.5) { why = "Material: nu must be in (0, 0.5)"; return false; }
  if (m.model == MSIM_MODEL_HENCKY_VON_MISES && m.yield_stress <= 0.0) { why = "Material: yield stress must be > 0"; return false; }
  if (m.model == MSIM_MODEL_DRUCKER_PRAGER && !(m.yield_stress > 0.0 && m.yield_stress < 90.0)) {
    why = "Material: friction angle must be in (0, 90) degrees";
    return false;
  }
  if (m.density <= 0.0) { why = "Material: density must be > 0"; return false; }
  if (m.model < MSIM_MODEL_HENCKY_VON_MISES || m.model > MSIM_MODEL_FLUID) { why = "Material: unknown constitutive model"; return false; }
  return true;
}

}  // namespace

extern "C" {

int msim_gpu_version(void) { return 1; }

const char* msim_gpu_create_error(void) { return g_create_error.c_str(); }

int msim_gpu_create(const msim_soft_desc* desc, const msim_material* materials, int n_materials,
                    int n_env, int device, msim_gpu_ctx** out) {
  *out = nullptr;
  g_create_error.clear();
  if (!desc || n_env < 1 || n_materials < 1 || n_materials > 256) {
    g_create_error = "msim_gpu_create: invalid arguments";
    return MSIM_ERR_INVALID;
  }
  if (std::min(desc->dims[0], std::min(desc->dims[1], desc->dims[2])) < 4) {
    g_create_error = "MpmGrid: dims must be >= 4 per axis";
    return MSIM_ERR_INVALID;
  }
  if (!(desc->h > 0.0)) {
    g_create_error = "MpmGrid: cell length must be > 0";
    return MSIM_ERR_INVALID;
  }
  for (int i = 0; i < n_materials; ++i) {
    std::string why;
    if (!valid_material(materials[i], why)) {
      g_create_error = why;
      return MSIM_ERR_INVALID;
    }
  }
  auto* c = new msim_gpu_ctx();
  int rc = guarded(c, [&]() -> int {
    c->device = device;
    c->use_graphs = std::getenv("MSIM_NO_GRAPHS") == nullptr;  // eager launches (debugging / A-B checks)
    set_device(c);
    configure_kernels();
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->desc = *desc;
    c->mats_h.assign(materials, materials + n_materials);
    c->n_env = n_env;
    const int kb[3] = {kBX, kBY, kBZ};
    for (int a = 0; a < 3; ++a) c->bdims[a] = (desc->dims[a] + kb[a] - 1) / kb[a];
    c->blocks_per_env = c->bdims[0] * c->bdims[1] * c->bdims[2];
    c->nodes_per_env = (long long)desc->dims[0] * desc->dims[1] * desc->dims[2];
    if ((long long)n_env * c->blocks_per_env + 1 > INT_MAX / 2)
      throw std::runtime_error("too many node blocks for one context");
    c->env_off_h.assign(n_env + 1, 0);
    c->bodies_h.assign(n_env, {});
    c->shapes_h.assign(n_env, {});
    c->vol_h.assign(n_env, {});
    c->mean_mass_h.assign(n_env, 0.0);
    c->env_grid_dirty.assign(n_env, 0);
    std::vector<MatParams> mp;
    for (auto& m : c->mats_h) mp.push_back(mat_params(m));
    CK(c->mats_d.ensure(sizeof(MatParams) * mp.size()));
    CK(cudaMemcpy(c->mats_d.p, mp.data(), sizeof(MatParams) * mp.size(), cudaMemcpyHostToDevice));
    auto per_env = [&](DevBuf& b, size_t elem) {
      CK(b.ensure(elem * n_env));
      CK(cudaMemset(b.p, 0, elem * n_env));
    };
    per_env(c->run_d, sizeof(EnvRun));
    per_env(c->applied_d, 3 * sizeof(double));
    per_env(c->react_d, 3 * sizeof(double));
    per_env(c->max_pen_d, sizeof(unsigned));
    per_env(c->vmax_d, sizeof(unsigned));
    per_env(c->lost_d, sizeof(long long));
    per_env(c->err_code_d, sizeof(int));
    per_env(c->err_pid_d, sizeof(int));
    per_env(c->balance_d, sizeof(double));
    per_env(c->mean_mass_d, sizeof(double));
    per_env(c->a64_d, 3 * sizeof(long long));
    per_env(c->r64_d, 3 * sizeof(long long));
    per_env(c->det_bnd_d, sizeof(unsigned));
    per_env(c->det_mexp_d, sizeof(int));
    CK(cudaMemset(c->err_pid_d.p, 0x7f, sizeof(int) * n_env));
    CK(c->env_off_d.ensure(sizeof(long long) * (n_env + 1)));
    CK(cudaMemset(c->env_off_d.p, 0, sizeof(long long) * (n_env + 1)));
    // grid: float4 per node, three channels, zeroed once (then cleared lazily)
    size_t nodes = (size_t)c->nodes_per_env * n_env;
    CK(c->gPM_d.ensure(sizeof(float4) * nodes));
    CK(c->gF_d.ensure(sizeof(float4) * nodes));
    CK(c->gV_d.ensure(sizeof(float4) * nodes));
    CK(cudaMemset(c->gPM_d.p, 0, sizeof(float4) * nodes));
    CK(cudaMemset(c->gF_d.p, 0, sizeof(float4) * nodes));
    CK(cudaMemset(c->gV_d.p, 0, sizeof(float4) * nodes));
    int nblocks = n_env * c->blocks_per_env;
    CK(c->nb_flag_d.ensure(sizeof(int) * nblocks));
    CK(c->nb_scan_d.ensure(sizeof(int) * (nblocks + 1)));
    CK(c->nb_list_d.ensure(sizeof(int) * nblocks));
    CK(c->n_nb_d.ensure(sizeof(int)));
    CK(cudaMemset(c->nb_flag_d.p, 0, sizeof(int) * nblocks));
    CK(cudaMemset(c->n_nb_d.p, 0, sizeof(int)));
    set_bucket_shape(c, 1);
    CK(c->ctl_d.ensure(8 * sizeof(int)));  // [0] redo flag, [2..5] particle-kernel hand-out counters
    CK(cudaMemset(c->ctl_d.p, 0, 8 * sizeof(int)));
    carve_particles(c, 0, 0);
    carve_particles(c, 1, 0);
    alloc_binning(c);
    upload_bodies(c);
    CK(cudaDeviceSynchronize());
    return MSIM_OK;
  });
  if (rc != MSIM_OK) {
    g_create_error = c->err;
    msim_gpu_destroy(c);
    return rc;
  }
  *out = c;
  return MSIM_OK;
}

void msim_gpu_destroy(msim_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* msim_gpu_last_error(const msim_gpu_ctx* c) { return c ? c->err.c_str() : ""; }

int msim_gpu_set_bucket_factor(msim_gpu_ctx* c, int factor) {
  return guarded(c, [&]() -> int {
    if (factor < 0 || factor > 2) return fail(c, MSIM_ERR_INVALID, "set_bucket_factor: factor must be 0 (auto), 1 or 2");
    c->qf_request = factor;
    if (factor) {
      set_device(c);
      set_bucket_shape(c, factor);
    }
    return MSIM_OK;
  });
}

int msim_gpu_set_particles(msim_gpu_ctx* c, int64_t n, const int64_t* env_offsets, const double* x,
                           const double* v, const double* F, const double* C, const double* mass,
                           const double* vol0, const int32_t* material) {
  NvtxRange range("msim.set_particles");
  return guarded(c, [&]() -> int {
    if (n < 0 || n >= INT_MAX / 2) return fail(c, MSIM_ERR_INVALID, "set_particles: particle count out of range");
    if (!env_offsets || env_offsets[0] != 0 || env_offsets[c->n_env] != n)
      return fail(c, MSIM_ERR_INVALID, "set_particles: env_offsets must start at 0 and end at n");
    for (int e = 0; e < c->n_env; ++e)
      if (env_offsets[e + 1] < env_offsets[e]) return fail(c, MSIM_ERR_INVALID, "set_particles: env_offsets not monotone");
    if (n > 0 && (!x || !mass || !vol0)) return fail(c, MSIM_ERR_INVALID, "set_particles: x, mass, vol0 required");
    if (material)
      for (int64_t i = 0; i < n; ++i)
        if (material[i] < 0 || material[i] >= (int)c->mats_h.size())
          return fail(c, MSIM_ERR_INVALID, "set_particles: material index out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    {  // bucket shape from the particle density (unless requested): particles per cell = h^3 / V0
      int f = c->qf_request;
      if (f == 0) {
        double vsum = 0.0;
        for (int64_t i = 0; i < n; ++i) vsum += vol0[i];
        const double ppc = n > 0 ? c->desc.h * c->desc.h * c->desc.h / (vsum / (double)n) : 16.0;
        f = ppc < 6.0 ? 2 : 1;  // < ~190 particles in a 32-cell bucket: use 8x8x4-cell buckets
      }
      set_bucket_shape(c, f);
    }
    {  // a scene too small to give every resident particle-kernel CTA a round of its
       // own: a bucket's rounds are spread over split_r CTAs (interleaved)
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      const double slots = (double)sms * kParticleCtasPerSm * kParticleRound;
      int r = n > 0 ? (int)std::ceil(slots / (double)n) : 1;
      if (const char* ev = std::getenv("MSIM_SPLIT_R")) r = std::atoi(ev);  // tuning override
      c->split_r = std::max(1, std::min(r, 8));
    }
    c->n = n;
    c->cur = 0;
    carve_particles(c, 0, n);
    carve_particles(c, 1, n);
    alloc_binning(c);
    c->env_off_h.assign(env_offsets, env_offsets + c->n_env + 1);
    CK(cudaMemcpyAsync(c->env_off_d.p, c->env_off_h.data(), sizeof(long long) * (c->n_env + 1), cudaMemcpyHostToDevice, s));
    std::vector<int> env_of(n);
    for (int e = 0; e < c->n_env; ++e) {
      double msum = 0.0;
      for (long long i = env_offsets[e]; i < env_offsets[e + 1]; ++i) {
        env_of[i] = e;
        msum += mass[i];
      }
      long long ne = env_offsets[e + 1] - env_offsets[e];
      c->mean_mass_h[e] = ne > 0 ? msum / (double)ne : 0.0;  // World::init (coupling.hpp:97-99)
    }
    CK(cudaMemcpyAsync(c->mean_mass_d.p, c->mean_mass_h.data(), sizeof(double) * c->n_env, cudaMemcpyHostToDevice, s));
    {  // deterministic mode: node mass sums <= the env's mass < 2^58 units
      std::vector<int> mexp(c->n_env);
      for (int e = 0; e < c->n_env; ++e) {
        const double M = c->mean_mass_h[e] * (double)(env_offsets[e + 1] - env_offsets[e]);
        mexp[e] = M > 0.0 ? 58 - (int)std::ceil(std::log2(M)) : 58;
      }
      CK(cudaMemcpy(c->det_mexp_d.p, mexp.data(), sizeof(int) * c->n_env, cudaMemcpyHostToDevice));
    }
    if (n > 0) {
      // stage doubles on the device in chunks, convert to fp32 SoA
      const long long chunk = 1 << 20;
      DevBuf st;
      CK(st.ensure(sizeof(double) * chunk * 26 + sizeof(int) * chunk * 2));
      for (long long o = 0; o < n; o += chunk) {
        long long m = std::min(chunk, n - o);
        double* dx = st.as<double>();
        double* dv = dx + 3 * chunk;
        double* dF = dv + 3 * chunk;
        double* dC = dF + 9 * chunk;
        double* dm = dC + 9 * chunk;
        double* dV = dm + chunk;
        int* dmat = reinterpret_cast<int*>(dV + chunk);
        int* denv = dmat + chunk;
        CK(cudaMemcpyAsync(dx, x + 3 * o, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
        if (v) CK(cudaMemcpyAsync(dv, v + 3 * o, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, s));
        if (F) CK(cudaMemcpyAsync(dF, F + 9 * o, sizeof(double) * 9 * m, cudaMemcpyHostToDevice, s));
        if (C) CK(cudaMemcpyAsync(dC, C + 9 * o, sizeof(double) * 9 * m, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dm, mass + o, sizeof(double) * m, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dV, vol0 + o, sizeof(double) * m, cudaMemcpyHostToDevice, s));
        if (material) CK(cudaMemcpyAsync(dmat, material + o, sizeof(int) * m, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(denv, env_of.data() + o, sizeof(int) * m, cudaMemcpyHostToDevice, s));
        SimParams P = params(c);
        launch_convert_in(P, m, dx, v ? dv : nullptr, F ? dF : nullptr, C ? dC : nullptr, dm, dV,
                          material ? dmat : nullptr, denv, o, s);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s));  // staging reused
      }
    }
    // init_buffers (mpm.hpp:137-142): lost flags, counts, clean grid
    CK(cudaMemsetAsync(c->lost_d.p, 0, sizeof(long long) * c->n_env, s));
    for (int e = 0; e < c->n_env; ++e) c->env_grid_dirty[e] = 1;
    c->grid_clean = false;
    c->vmax_valid = false;
    c->perm_valid = false;
    reset_errors(c);
    CK(cudaStreamSynchronize(s));
    return MSIM_OK;
  });
}

int msim_gpu_write_particles(msim_gpu_ctx* c, int env, int64_t n, const double* x, const double* v,
                             const double* F, const double* C) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "write_particles: env out of range");
    long long first = c->env_off_h[env], ne = c->env_off_h[env + 1] - first;
    if (n != ne) return fail(c, MSIM_ERR_INVALID, "write_particles: count mismatch");
    set_device(c);
    cudaStream_t s = c->stream;
    DevBuf st;
    CK(st.ensure(sizeof(double) * std::max<long long>(ne, 1) * 24));
    double* dx = st.as<double>();
    double* dv = dx + 3 * ne;
    double* dF = dv + 3 * ne;
    double* dC = dF + 9 * ne;
    if (x) CK(cudaMemcpyAsync(dx, x, sizeof(double) * 3 * ne, cudaMemcpyHostToDevice, s));
    if (v) CK(cudaMemcpyAsync(dv, v, sizeof(double) * 3 * ne, cudaMemcpyHostToDevice, s));
    if (F) CK(cudaMemcpyAsync(dF, F, sizeof(double) * 9 * ne, cudaMemcpyHostToDevice, s));
    if (C) CK(cudaMemcpyAsync(dC, C, sizeof(double) * 9 * ne, cudaMemcpyHostToDevice, s));
    SimParams P = params(c);
    launch_overwrite(P, first, ne, x ? dx : nullptr, v ? dv : nullptr, F ? dF : nullptr, C ? dC : nullptr, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    c->vmax_valid = false;
    c->perm_valid = false;
    return MSIM_OK;
  });
}

int msim_gpu_set_bodies(msim_gpu_ctx* c, int env, const msim_body* bodies, int n_bodies,
                        const msim_shape* shapes, int n_shapes) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "set_bodies: env out of range");
    if (n_bodies < 0 || n_bodies > kMaxBodiesPerEnv)
      return fail(c, MSIM_ERR_INVALID, "set_bodies: at most 32 contact bodies per environment");
    for (int i = 0; i < n_bodies; ++i) {
      const msim_body& b = bodies[i];
      if (b.mode == MSIM_BODY_DYNAMIC &&
          (b.mass <= 0.0 || std::min(b.inertia[0], std::min(b.inertia[1], b.inertia[2])) <= 0.0))
        return fail(c, MSIM_ERR_INVALID, "RigidBody: dynamic body needs positive mass and inertia");
    }
    std::vector<std::vector<float>> vols;
    for (int s = 0; s < n_shapes; ++s) {
      const msim_shape& sh = shapes[s];
      if (sh.body < 0 || sh.body >= n_bodies) return fail(c, MSIM_ERR_INVALID, "set_bodies: shape body index out of range");
      if (sh.friction < 0.0) return fail(c, MSIM_ERR_INVALID, "Shape: friction must be >= 0");
      if (sh.k_n <= 0.0 || sh.k_t <= 0.0) return fail(c, MSIM_ERR_INVALID, "Shape: stiffness must be > 0");
      std::vector<float> smp;
      if (sh.type == MSIM_SHAPE_VOLUME) {
        if (std::min(sh.vol_dims[0], std::min(sh.vol_dims[1], sh.vol_dims[2])) < 2 || !sh.vol_samples)
          return fail(c, MSIM_ERR_INVALID, "SdfVolume: dims must be >= 2 per axis");
        size_t ns = (size_t)sh.vol_dims[0] * sh.vol_dims[1] * sh.vol_dims[2];
        smp.assign(sh.vol_samples, sh.vol_samples + ns);
        for (float f : smp)
          if (!std::isfinite(f)) return fail(c, MSIM_ERR_INVALID, "SdfVolume: non-finite sample");
      } else if (sh.type < 0 || sh.type > MSIM_SHAPE_VOLUME) {
        return fail(c, MSIM_ERR_INVALID, "Shape: unknown type");
      }
      vols.push_back(std::move(smp));
    }
    if (!c->bodies_dirty) {  // snapshot the device-side body state of every env once
      set_device(c);
      download_bodies(c);
      std::vector<double> wr(6 * std::max(c->n_bodies, 1)), pd(wr.size());
      if (c->n_bodies) {
        CK(cudaMemcpyAsync(wr.data(), c->wrench_d.p, sizeof(double) * 6 * c->n_bodies, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(pd.data(), c->pending_d.p, sizeof(double) * 6 * c->n_bodies, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
      }
      c->wrench_h.assign(c->n_env, {});
      c->pending_h.assign(c->n_env, {});
      size_t off = 0;
      for (int e = 0; e < c->n_env; ++e) {
        const size_t nb = c->bodies_h[e].size();
        c->wrench_h[e].assign(wr.begin() + 6 * off, wr.begin() + 6 * (off + nb));
        c->pending_h[e].assign(pd.begin() + 6 * off, pd.begin() + 6 * (off + nb));
        off += nb;
      }
      c->bodies_dirty = true;
    }
    c->bodies_h[env].assign(bodies, bodies + n_bodies);
    c->shapes_h[env].assign(shapes, shapes + n_shapes);
    c->vol_h[env] = std::move(vols);
    c->wrench_h[env].assign(6 * n_bodies, 0.0);  // this env's wrenches reset (sync_rigid_to_soft)
    c->pending_h[env].assign(6 * n_bodies, 0.0);
    return MSIM_OK;
  });
}

int msim_gpu_set_deterministic(msim_gpu_ctx* c, int on) {
  return guarded(c, [&]() -> int {
    set_device(c);
    on = on ? 1 : 0;
    if (on == c->det) return MSIM_OK;
    if (on) {
      const size_t nodes = (size_t)c->nodes_per_env * c->n_env;
      CK(c->gPMd_d.ensure(sizeof(longlong4) * std::max<size_t>(nodes, 1)));
      CK(cudaMemsetAsync(c->gPMd_d.p, 0, sizeof(longlong4) * std::max<size_t>(nodes, 1), c->stream));
      CK(cudaMemsetAsync(c->det_bnd_d.p, 0, sizeof(unsigned) * c->n_env, c->stream));
      CK(cudaMemsetAsync(c->a64_d.p, 0, 3 * sizeof(long long) * c->n_env, c->stream));
      CK(cudaMemsetAsync(c->r64_d.p, 0, 3 * sizeof(long long) * c->n_env, c->stream));
      CK(cudaMemsetAsync(c->w64_d.p, 0, 6 * sizeof(long long) * std::max(c->n_bodies, 1), c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    c->det = on;
    c->perm_valid = false;  // re-bin: the deterministic particle order starts from the upload order
    return MSIM_OK;
  });
}

int msim_gpu_set_kinematic_schedule(msim_gpu_ctx* c, int n_steps, const double* poses, const uint8_t* mask) {
  NvtxRange range("msim.set_kinematic_schedule");
  return guarded(c, [&]() -> int {
    set_device(c);
    if (n_steps < 1 || !poses) return fail(c, MSIM_ERR_INVALID, "set_kinematic_schedule: need >= 1 rigid step of poses");
    const int nb = c->n_bodies;
    std::vector<unsigned char> m(std::max(nb, 1), 0);
    int k = 0;
    for (int e = 0; e < c->n_env; ++e)
      for (const msim_body& b : c->bodies_h[e]) {
        m[k] = mask ? (mask[k] ? 1 : 0) : (b.mode == MSIM_BODY_KINEMATIC ? 1 : 0);
        if (m[k] && b.mode == MSIM_BODY_DYNAMIC)
          return fail(c, MSIM_ERR_INVALID, "set_kinematic_schedule: a dynamic body cannot follow a schedule");
        ++k;
      }
    const size_t n = 7ull * nb * n_steps;
    CK(c->sched_d.ensure(sizeof(double) * std::max<size_t>(n, 1)));
    CK(c->sched_mask_d.ensure(m.size()));
    if (n) CK(cudaMemcpyAsync(c->sched_d.p, poses, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->sched_mask_d.p, m.data(), m.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));  // the caller's buffer may go away
    c->sched_steps = n_steps;
    return MSIM_OK;
  });
}

int msim_gpu_set_coupling(msim_gpu_ctx* c, const msim_coupling* cp) {
  if (cp->mode != MSIM_COUPLING_PARTICLE && cp->mode != MSIM_COUPLING_GRID)
    return fail(c, MSIM_ERR_INVALID, "set_coupling: unknown mode");
  c->coupling = *cp;
  return MSIM_OK;
}

int msim_gpu_sync_bodies(msim_gpu_ctx* c, int env, const msim_body* bodies, int n_bodies) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "sync_bodies: env out of range");
    if ((int)c->bodies_h[env].size() != n_bodies) return fail(c, MSIM_ERR_INVALID, "sync_bodies: body count mismatch");
    set_device(c);
    // body slots of this env start at the prefix of earlier envs' counts
    int off = 0;
    for (int e = 0; e < env; ++e) off += (int)c->bodies_h[e].size();
    std::vector<BodyDev> bd(n_bodies);
    if (n_bodies) {
      CK(cudaMemcpyAsync(bd.data(), c->bodies_d.as<BodyDev>() + off, sizeof(BodyDev) * n_bodies, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    for (int i = 0; i < n_bodies; ++i) {
      std::memcpy(bd[i].q, bodies[i].q, sizeof bd[i].q);
      std::memcpy(bd[i].t, bodies[i].t, sizeof bd[i].t);
      std::memcpy(bd[i].v, bodies[i].v, sizeof bd[i].v);
      std::memcpy(bd[i].w, bodies[i].w, sizeof bd[i].w);
      c->bodies_h[env][i] = bodies[i];
    }
    if (n_bodies)
      CK(cudaMemcpyAsync(c->bodies_d.as<BodyDev>() + off, bd.data(), sizeof(BodyDev) * n_bodies, cudaMemcpyHostToDevice, c->stream));
    SimParams P = params(c);
    launch_rigid(P, 0, env, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
    return MSIM_OK;
  });
}

int msim_gpu_set_dt(msim_gpu_ctx* c, double dt) {
  c->desc.dt = dt;
  return MSIM_OK;
}
int msim_gpu_set_gravity(msim_gpu_ctx* c, const double* g) {
  for (int a = 0; a < 3; ++a) c->desc.gravity[a] = g[a];
  return MSIM_OK;
}
int msim_gpu_set_rigid_gravity(msim_gpu_ctx* c, const double* g) {
  for (int a = 0; a < 3; ++a) c->rigid_gravity[a] = g[a];
  return MSIM_OK;
}
int msim_gpu_set_lost_fraction_threshold(msim_gpu_ctx* c, double t) {
  c->desc.lost_fraction_threshold = t;
  return MSIM_OK;
}
int msim_gpu_set_split_channels(msim_gpu_ctx* c, int split) {
  c->split_req = split ? 1 : 0;
  return MSIM_OK;
}
int msim_gpu_set_record_binning(msim_gpu_ctx* c, int on) {
  return guarded(c, [&]() -> int {
    set_device(c);
    c->record_binning = on ? 1 : 0;
    alloc_binning(c);
    return MSIM_OK;
  });
}

static int det_mode_check(msim_gpu_ctx* c) {
  if (c->det && split_mode(c))
    return fail(c, MSIM_ERR_INVALID, "deterministic mode covers particle coupling (no grid coupling / split channels)");
  return MSIM_OK;
}

int msim_gpu_soft_substep(msim_gpu_ctx* c, int n_substeps, int32_t* cycles_out) {
  return guarded(c, [&]() -> int {
    if (const int rc = det_mode_check(c)) return rc;
    set_device(c);
    reset_errors(c);
    return step_call(c, n_substeps, false, 1, cycles_out);
  });
}

// Phase API (p2g / grid_update / g2p_advect as separate calls): one launch
// per phase with every env active, dt_c = dt, momentum and force kept apart.
static int manual_phase(msim_gpu_ctx* c, int which) {
  return guarded(c, [&]() -> int {
    if (c->det) return fail(c, MSIM_ERR_INVALID, "deterministic mode covers env_step / soft_substep (not the phase API)");
    set_device(c);
    reset_errors(c);
    if (c->n == 0) return MSIM_OK;
    cudaStream_t s = c->stream;
    if (which == 0) {  // p2g
      prepare(c, false);
      SimParams P = params(c);
      launch_set_action(P, kActP2G, (float)c->desc.dt, s);
      P.clear_on_read = 0;
      P.hooks = 0;  // p2g() is hook-free (mpm.hpp:199); soft_substep installs the hooks
      launch_particles(P, s);
      launch_iteration_end(P, s);
      swap_buffers(c);
      c->grid_clean = false;
      c->perm_valid = true;
    } else if (which == 1) {  // grid_update
      SimParams P = params(c);
      launch_set_action(P, kActP2G, (float)c->desc.dt, s);
      P.clear_on_read = 0;
      P.hooks = 0;
      launch_grid(P, s);
    } else {  // g2p_advect
      if (!c->perm_valid) launch_rebin(params(c), s), c->perm_valid = true;
      SimParams P = params(c);
      launch_set_action(P, kActG2P, (float)c->desc.dt, s);
      launch_particles(P, s);
      swap_buffers(c);
      c->vmax_valid = true;
      c->perm_valid = true;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    c->timer.flush();
    return collect_errors(c);
  });
}

int msim_gpu_p2g(msim_gpu_ctx* c) { return manual_phase(c, 0); }
int msim_gpu_grid_update(msim_gpu_ctx* c) { return manual_phase(c, 1); }
int msim_gpu_g2p(msim_gpu_ctx* c) { return manual_phase(c, 2); }

int msim_gpu_env_step(msim_gpu_ctx* c, int n_rigid, int n_soft, msim_step_report* report) {
  return guarded(c, [&]() -> int {
    if (n_rigid < 1 || n_soft < 1) return fail(c, MSIM_ERR_INVALID, "World: n_rigid and n_soft must be >= 1");
    if (const int rc = det_mode_check(c)) return rc;
    set_device(c);
    cudaStream_t s = c->stream;
    reset_errors(c);
    CK(cudaMemsetAsync(c->max_pen_d.p, 0, sizeof(unsigned) * c->n_env, s));
    CK(cudaMemsetAsync(c->balance_d.p, 0, sizeof(double) * c->n_env, s));
    if (c->sched_steps > 0 && c->sched_steps != n_rigid) {
      c->sched_steps = 0;
      return fail(c, MSIM_ERR_INVALID, "kinematic schedule length != n_rigid");
    }
    const int rc = step_call(c, n_rigid * n_soft, c->n_bodies > 0, n_soft, nullptr);
    c->sched_steps = 0;  // a schedule drives exactly one env step
    c->last_substeps = n_rigid * n_soft;
    c->time += n_rigid * n_soft * c->desc.dt;
    if (report) {  // all envs' report words in one transfer (not one round trip per env)
      const int ne = c->n_env;
      std::vector<unsigned> pen(ne);
      std::vector<double> bal(ne);
      std::vector<long long> lost(ne);
      std::vector<EnvRun> run(ne);
      CK(cudaMemcpyAsync(pen.data(), c->max_pen_d.p, sizeof(unsigned) * ne, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(bal.data(), c->balance_d.p, sizeof(double) * ne, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(lost.data(), c->lost_d.p, sizeof(long long) * ne, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(run.data(), c->run_d.p, sizeof(EnvRun) * ne, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      msim_step_report agg{};
      agg.rigid_steps = n_rigid;
      agg.soft_substeps = n_rigid * n_soft;
      for (int e = 0; e < ne; ++e) {
        float penf;
        std::memcpy(&penf, &pen[e], sizeof penf);
        agg.cfl_cycles = std::max(agg.cfl_cycles, run[e].cyc_sum);
        agg.max_penetration = std::max(agg.max_penetration, (double)penf);
        agg.max_force_balance_error = std::max(agg.max_force_balance_error, bal[e]);
        agg.lost_particles += lost[e];
      }
      *report = agg;
    }
    return rc;
  });
}

int msim_gpu_nccl_unique_id(uint8_t* id128) {
  const char* e = nccl_unique_id(id128);
  if (e) {
    g_create_error = e;
    return MSIM_ERR_DEVICE;
  }
  return MSIM_OK;
}

int msim_gpu_comm_init(msim_gpu_ctx* c, int rank, int world, const uint8_t* id128) {
  return guarded(c, [&]() -> int {
    if (world < 1 || rank < 0 || rank >= world) return fail(c, MSIM_ERR_INVALID, "comm_init: bad rank / world size");
    set_device(c);
    nccl_comm_destroy(c->comm);
    c->comm = nullptr;
    if (const char* e = nccl_comm_init(&c->comm, rank, world, id128)) return fail(c, MSIM_ERR_DEVICE, e);
    c->comm_rank = rank;
    c->comm_world = world;
    return MSIM_OK;
  });
}

int msim_gpu_step_stats(msim_gpu_ctx* c, int allreduce, double* sums, double* maxs) {
  NvtxRange range("msim.step_stats");
  return guarded(c, [&]() -> int {
    if (allreduce && !c->comm) return fail(c, MSIM_ERR_INVALID, "step_stats: no communicator (msim_gpu_comm_init)");
    set_device(c);
    CK(c->stats_d.ensure(8 * sizeof(double)));
    if (const char* e = launch_step_stats(params(c), c->last_substeps, c->stats_d.as<double>(),
                                          allreduce ? c->comm : nullptr, c->stream))
      return fail(c, MSIM_ERR_DEVICE, e);
    double h[6];
    CK(cudaMemcpyAsync(h, c->stats_d.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (sums) std::memcpy(sums, h, 4 * sizeof(double));
    if (maxs) std::memcpy(maxs, h + 4, 2 * sizeof(double));
    return MSIM_OK;
  });
}

int64_t msim_gpu_particle_count(const msim_gpu_ctx* c, int env) {
  if (env < 0) return c->n;
  if (env >= c->n_env) return -1;
  return c->env_off_h[env + 1] - c->env_off_h[env];
}

int msim_gpu_read_particles(msim_gpu_ctx* c, int env, double* x, double* v, double* F, double* C,
                            uint8_t* lost) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_particles: env out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    long long first = c->env_off_h[env], ne = c->env_off_h[env + 1] - first;
    if (ne == 0) return MSIM_OK;
    DevBuf st;
    CK(st.ensure(sizeof(double) * ne * 24 + ne));
    double* dx = st.as<double>();
    double* dv = dx + 3 * ne;
    double* dF = dv + 3 * ne;
    double* dC = dF + 9 * ne;
    uint8_t* dl = reinterpret_cast<uint8_t*>(dC + 9 * ne);
    SimParams P = params(c);
    launch_convert_out(P, first, ne, x ? dx : nullptr, v ? dv : nullptr, F ? dF : nullptr,
                       C ? dC : nullptr, lost ? dl : nullptr, s);
    CK(cudaGetLastError());
    if (x) CK(cudaMemcpyAsync(x, dx, sizeof(double) * 3 * ne, cudaMemcpyDeviceToHost, s));
    if (v) CK(cudaMemcpyAsync(v, dv, sizeof(double) * 3 * ne, cudaMemcpyDeviceToHost, s));
    if (F) CK(cudaMemcpyAsync(F, dF, sizeof(double) * 9 * ne, cudaMemcpyDeviceToHost, s));
    if (C) CK(cudaMemcpyAsync(C, dC, sizeof(double) * 9 * ne, cudaMemcpyDeviceToHost, s));
    if (lost) CK(cudaMemcpyAsync(lost, dl, ne, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return MSIM_OK;
  });
}

int msim_gpu_read_jp(msim_gpu_ctx* c, int env, double* jp) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_jp: env out of range");
    if (!jp) return fail(c, MSIM_ERR_INVALID, "read_jp: null output");
    set_device(c);
    cudaStream_t s = c->stream;
    long long first = c->env_off_h[env], ne = c->env_off_h[env + 1] - first;
    if (ne == 0) return MSIM_OK;
    if (!params(c).any_model) {  // von Mises only: the particle kernel does not carry jp (always 1)
      std::fill(jp, jp + ne, 1.0);
      return MSIM_OK;
    }
    DevBuf st;
    CK(st.ensure(sizeof(double) * ne));
    launch_jp_out(params(c), first, ne, st.as<double>(), s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(jp, st.p, sizeof(double) * ne, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return MSIM_OK;
  });
}

int msim_gpu_read_grid(msim_gpu_ctx* c, int env, double* mass, double* momentum, double* force,
                       double* velocity) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_grid: env out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    long long nn = c->nodes_per_env;
    DevBuf st;
    CK(st.ensure(sizeof(double) * nn * 10));
    double* dm = st.as<double>();
    double* dp = dm + nn;
    double* df = dp + 3 * nn;
    double* dv = df + 3 * nn;
    SimParams P = params(c);
    launch_grid_out(P, env, mass ? dm : nullptr, momentum ? dp : nullptr, force ? df : nullptr,
                    velocity ? dv : nullptr, s);
    CK(cudaGetLastError());
    if (mass) CK(cudaMemcpyAsync(mass, dm, sizeof(double) * nn, cudaMemcpyDeviceToHost, s));
    if (momentum) CK(cudaMemcpyAsync(momentum, dp, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, s));
    if (force) CK(cudaMemcpyAsync(force, df, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, s));
    if (velocity) CK(cudaMemcpyAsync(velocity, dv, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return MSIM_OK;
  });
}

int msim_gpu_write_grid_velocity(msim_gpu_ctx* c, int env, const double* velocity) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "write_grid_velocity: env out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    long long nn = c->nodes_per_env;
    DevBuf st;
    CK(st.ensure(sizeof(double) * nn * 3));
    CK(cudaMemcpyAsync(st.p, velocity, sizeof(double) * 3 * nn, cudaMemcpyHostToDevice, s));
    SimParams P = params(c);
    launch_grid_vel_in(P, env, st.as<double>(), s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    c->env_grid_dirty[env] = 1;  // the next clear must wipe the whole env grid
    c->grid_clean = false;
    return MSIM_OK;
  });
}

int msim_gpu_read_buckets(msim_gpu_ctx* c, int env, int32_t* bucket_cells, int32_t* bucket_dims, int32_t* counts,
                          int64_t counts_cap, int32_t* block_dims, int32_t* blocks, int64_t blocks_cap,
                          int64_t* n_blocks) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_buckets: env out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    const int kb[3] = {kBX, kBY, kBZ};
    for (int a = 0; a < 3; ++a) {
      if (bucket_cells) bucket_cells[a] = kb[a] * c->qf;
      if (bucket_dims) bucket_dims[a] = c->qdims[a];
      if (block_dims) block_dims[a] = c->bdims[a];
    }
    if (counts) {
      if (counts_cap < c->buckets_per_env) return fail(c, MSIM_ERR_INVALID, "read_buckets: counts capacity");
      std::vector<int> st(c->buckets_per_env + 1);
      CK(cudaMemcpyAsync(st.data(), c->bucket_start_d[c->bset].as<int>() + (long long)env * c->buckets_per_env,
                         sizeof(int) * (c->buckets_per_env + 1), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int k = 0; k < c->buckets_per_env; ++k) counts[k] = st[k + 1] - st[k];
    }
    if (n_blocks) {
      int nl = 0;
      CK(cudaMemcpyAsync(&nl, c->n_nb_d.p, sizeof(int), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      std::vector<int> list(std::max(nl, 1));
      if (nl) CK(cudaMemcpyAsync(list.data(), c->nb_list_d.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      int64_t k = 0;
      for (int i = 0; i < nl; ++i) {
        if (list[i] / c->blocks_per_env != env) continue;
        if (blocks) {
          if (k >= blocks_cap) return fail(c, MSIM_ERR_INVALID, "read_buckets: blocks capacity");
          blocks[k] = list[i] - env * c->blocks_per_env;
        }
        ++k;
      }
      *n_blocks = k;
    }
    return MSIM_OK;
  });
}

int msim_gpu_read_binning(msim_gpu_ctx* c, int env, int32_t* base, int32_t* cell_start,
                          int64_t cell_start_cap, int32_t* cell_particles, int64_t cell_particles_cap,
                          int64_t* n_alive, int64_t* active_nodes, int64_t active_cap,
                          int64_t* n_active) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_binning: env out of range");
    if (!c->record_binning) return fail(c, MSIM_ERR_INVALID, "read_binning: enable msim_gpu_set_record_binning first");
    set_device(c);
    cudaStream_t s = c->stream;
    long long first = c->env_off_h[env], ne = c->env_off_h[env + 1] - first;
    const int nbins = (c->desc.dims[0] - 2) * (c->desc.dims[1] - 2) * (c->desc.dims[2] - 2);
    const long long nn = c->nodes_per_env;
    DevBuf cc, cs, cp, nf, ns, nl, nlc, an, tmp;
    CK(cc.ensure(sizeof(int) * (nbins + 1)));
    CK(cs.ensure(sizeof(int) * (nbins + 1)));
    CK(cp.ensure(sizeof(int) * std::max<long long>(ne, 1)));
    CK(nf.ensure(sizeof(int) * nn));
    CK(ns.ensure(sizeof(int) * (nn + 1)));
    CK(nl.ensure(sizeof(int) * nn));
    CK(nlc.ensure(sizeof(int)));
    CK(an.ensure(sizeof(long long) * nn));
    CK(tmp.ensure(sizeof(int) * scan_tmp_ints((int)std::max<long long>(nbins + 1, nn + 1))));
    CK(cudaMemsetAsync(tmp.p, 0, sizeof(int) * scan_tmp_ints((int)std::max<long long>(nbins + 1, nn + 1)), s));
    SimParams P = params(c);
    const int* b = c->base_dbg_d.as<int>() + 3 * first;
    launch_binning_out(P, ne, b, cc.as<int>(), cs.as<int>(), cp.as<int>(), nf.as<int>(), ns.as<int>(),
                       nl.as<int>(), nlc.as<int>(), an.as<long long>(), tmp.as<int>(), s);
    CK(cudaGetLastError());
    int total = 0, nact = 0;
    CK(cudaMemcpyAsync(&total, cs.as<int>() + nbins, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&nact, nlc.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_alive = total;
    *n_active = nact;
    if (base) CK(cudaMemcpyAsync(base, b, sizeof(int) * 3 * ne, cudaMemcpyDeviceToHost, s));
    if (cell_start) {
      if (cell_start_cap < nbins + 1) return fail(c, MSIM_ERR_INVALID, "read_binning: cell_start capacity");
      CK(cudaMemcpyAsync(cell_start, cs.p, sizeof(int) * (nbins + 1), cudaMemcpyDeviceToHost, s));
    }
    if (cell_particles) {
      if (cell_particles_cap < total) return fail(c, MSIM_ERR_INVALID, "read_binning: cell_particles capacity");
      CK(cudaMemcpyAsync(cell_particles, cp.p, sizeof(int) * total, cudaMemcpyDeviceToHost, s));
    }
    if (active_nodes) {
      if (active_cap < nact) return fail(c, MSIM_ERR_INVALID, "read_binning: active_nodes capacity");
      CK(cudaMemcpyAsync(active_nodes, an.p, sizeof(long long) * nact, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return MSIM_OK;
  });
}

int msim_gpu_read_wrenches(msim_gpu_ctx* c, int env, int pending, double* force, double* torque) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_wrenches: env out of range");
    set_device(c);
    int off = 0;
    for (int e = 0; e < env; ++e) off += (int)c->bodies_h[e].size();
    int nb = (int)c->bodies_h[env].size();
    if (nb == 0) return MSIM_OK;
    std::vector<double> w(6 * nb);
    const double* src = (pending ? c->pending_d.as<double>() : c->wrench_d.as<double>()) + 6 * off;
    CK(cudaMemcpyAsync(w.data(), src, sizeof(double) * 6 * nb, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < nb; ++i)
      for (int k = 0; k < 3; ++k) {
        if (force) force[3 * i + k] = w[6 * i + k];
        if (torque) torque[3 * i + k] = w[6 * i + 3 + k];
      }
    return MSIM_OK;
  });
}

int msim_gpu_read_bodies(msim_gpu_ctx* c, int env, msim_body* out, int n_bodies) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_bodies: env out of range");
    set_device(c);
    download_bodies(c);
    int nb = std::min<int>(n_bodies, (int)c->bodies_h[env].size());
    for (int i = 0; i < nb; ++i) out[i] = c->bodies_h[env][i];
    return MSIM_OK;
  });
}

int msim_gpu_read_report(msim_gpu_ctx* c, int env, msim_step_report* r) {
  return guarded(c, [&]() -> int {
    if (env < 0 || env >= c->n_env) return fail(c, MSIM_ERR_INVALID, "read_report: env out of range");
    set_device(c);
    unsigned pen = 0;
    double bal = 0.0;
    long long lost = 0;
    cudaStream_t s = c->stream;
    CK(cudaMemcpyAsync(&pen, c->max_pen_d.as<unsigned>() + env, sizeof pen, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&bal, c->balance_d.as<double>() + env, sizeof bal, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&lost, c->lost_d.as<long long>() + env, sizeof lost, cudaMemcpyDeviceToHost, s));
    EnvRun run{};
    CK(cudaMemcpyAsync(&run, c->run_d.as<EnvRun>() + env, sizeof run, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    float penf;
    std::memcpy(&penf, &pen, sizeof penf);
    r->max_penetration = penf;
    r->max_force_balance_error = bal;
    r->lost_particles = lost;
    r->cfl_cycles = run.cyc_sum;
    return MSIM_OK;
  });
}

int64_t msim_gpu_lost_count(msim_gpu_ctx* c, int env) {
  long long lost = -1;
  if (env < 0 || env >= c->n_env) return -1;
  if (cudaSetDevice(c->device) != cudaSuccess) return -1;
  if (cudaMemcpy(&lost, c->lost_d.as<long long>() + env, sizeof lost, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return lost;
}

int msim_gpu_constitutive(msim_gpu_ctx* c, int mat, int64_t n, const double* F, double* tau, double* Fp) {
  return guarded(c, [&]() -> int {
    if (mat < 0 || mat >= (int)c->mats_h.size()) return fail(c, MSIM_ERR_INVALID, "constitutive: material out of range");
    set_device(c);
    cudaStream_t s = c->stream;
    DevBuf st;
    CK(st.ensure(sizeof(double) * std::max<int64_t>(n, 1) * 27 + 16));
    double* dF = st.as<double>();
    double* dt = dF + 9 * n;
    double* dp = dt + 9 * n;
    int* bad = reinterpret_cast<int*>(dp + 9 * n);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), s));
    CK(cudaMemcpyAsync(dF, F, sizeof(double) * 9 * n, cudaMemcpyHostToDevice, s));
    launch_constitutive(mat_params(c->mats_h[mat]), n, dF, tau ? dt : nullptr, Fp ? dp : nullptr, bad, s);
    CK(cudaGetLastError());
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (tau) CK(cudaMemcpyAsync(tau, dt, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost, s));
    if (Fp) CK(cudaMemcpyAsync(Fp, dp, sizeof(double) * 9 * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hbad) return fail(c, MSIM_ERR_INVALID, "kirchhoff_stress: det(F) must be > 0");
    return MSIM_OK;
  });
}


// ---- task metrics (scenario.hpp:63-209) -----------------------------------
namespace {
bool region_ok(const msim_region& r) {  // RegionBox::validate (scenario.hpp:26-29)
  return std::min({r.max[0] - r.min[0], r.max[1] - r.min[1], r.max[2] - r.min[2]}) > 0.0;
}
// regions of all envs to the device (6 doubles per env)
int upload_regions(msim_gpu_ctx* c, const msim_region* regions, DevBuf& buf) {
  if (!regions) return fail(c, MSIM_ERR_INVALID, "metric: regions required");
  for (int e = 0; e < c->n_env; ++e)
    if (!region_ok(regions[e])) return fail(c, MSIM_ERR_INVALID, "RegionBox: extents must be positive");
  std::vector<double> h(6 * (size_t)c->n_env);
  for (int e = 0; e < c->n_env; ++e)
    for (int k = 0; k < 3; ++k) {
      h[6 * e + k] = regions[e].min[k];
      h[6 * e + 3 + k] = regions[e].max[k];
    }
  CK(buf.ensure(sizeof(double) * h.size()));
  CK(cudaMemcpyAsync(buf.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, c->stream));
  return MSIM_OK;
}
int heightmaps(msim_gpu_ctx* c, const msim_region* regions, int nx, int ny, DevBuf& maps, DevBuf& reg) {
  int rc = upload_regions(c, regions, reg);
  if (rc) return rc;
  if (nx < 2 || ny < 2) return fail(c, MSIM_ERR_INVALID, "render_heightmap: resolution must be >= 2x2");
  const size_t cells = (size_t)nx * ny * c->n_env;
  CK(maps.ensure(sizeof(double) * cells));
  CK(cudaMemsetAsync(maps.p, 0, sizeof(double) * cells, c->stream));  // +0.0
  launch_heightmap(params(c), reg.as<double>(), nx, ny, maps.as<unsigned long long>(), c->stream);
  CK(cudaGetLastError());
  return MSIM_OK;
}
// per-env chamfer of device point sets A (offsets offA) and B (offB); out[n_env]
void chamfer_sets(msim_gpu_ctx* c, const double* A, const long long* offA_d, const std::vector<long long>& offA,
                  const double* B, const long long* offB_d, const std::vector<long long>& offB, double* out) {
  const int ne = c->n_env;
  long long maxa = 0, maxb = 0;
  for (int e = 0; e < ne; ++e) {
    maxa = std::max(maxa, offA[e + 1] - offA[e]);
    maxb = std::max(maxb, offB[e + 1] - offB[e]);
  }
  DevBuf& mind = c->tbuf[9];
  DevBuf& means = c->tbuf[1];
  CK(mind.ensure(sizeof(double) * (size_t)std::max(offA[ne], offB[ne]) + 16));
  CK(means.ensure(sizeof(double) * 2 * ne));
  double* mab = means.as<double>();
  double* mba = mab + ne;
  launch_chamfer_side(A, offA_d, maxa, B, offB_d, ne, mind.as<double>(), mab, c->stream);
  launch_chamfer_side(B, offB_d, maxb, A, offA_d, ne, mind.as<double>(), mba, c->stream);
  CK(cudaGetLastError());
  std::vector<double> h(2 * (size_t)ne);
  CK(cudaMemcpyAsync(h.data(), means.p, sizeof(double) * 2 * ne, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int e = 0; e < ne; ++e) out[e] = h[e] + h[ne + e];  // ab / |a| + ba / |b|
}
// host point sets (per-env offsets) to the device; checks non-empty sets
int upload_points(msim_gpu_ctx* c, const double* pts, const int64_t* off, DevBuf& buf, DevBuf& off_d,
                  std::vector<long long>& off_h) {
  if (!pts || !off) return fail(c, MSIM_ERR_INVALID, "chamfer_distance: point sets required");
  off_h.assign(off, off + c->n_env + 1);
  for (int e = 0; e < c->n_env; ++e)
    if (off_h[e + 1] <= off_h[e]) return fail(c, MSIM_ERR_INVALID, "chamfer_distance: point sets must be non-empty");
  const long long base = off_h[0];
  for (auto& o : off_h) o -= base;
  CK(buf.ensure(sizeof(double) * 3 * (size_t)off_h[c->n_env] + 16));
  CK(off_d.ensure(sizeof(long long) * (c->n_env + 1)));
  CK(cudaMemcpyAsync(buf.p, pts + 3 * base, sizeof(double) * 3 * off_h[c->n_env], cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(off_d.p, off_h.data(), sizeof(long long) * (c->n_env + 1), cudaMemcpyHostToDevice, c->stream));
  return MSIM_OK;
}
int particle_points(msim_gpu_ctx* c, DevBuf& pos) {
  for (int e = 0; e < c->n_env; ++e)
    if (c->env_off_h[e + 1] <= c->env_off_h[e])
      return fail(c, MSIM_ERR_INVALID, "chamfer_distance: point sets must be non-empty");
  CK(pos.ensure(sizeof(double) * 3 * (size_t)std::max<long long>(c->n, 1)));
  launch_positions(params(c), pos.as<double>(), c->stream);
  CK(cudaGetLastError());
  return MSIM_OK;
}
}  // namespace

int msim_gpu_metric_fill(msim_gpu_ctx* c, const msim_region* regions, msim_fill_result* out) {
  return guarded(c, [&]() -> int {
    if (!out) return fail(c, MSIM_ERR_INVALID, "metric_fill: out required");
    for (int e = 0; e < c->n_env; ++e)
      if (c->env_off_h.empty() || c->env_off_h[e + 1] == c->env_off_h[e])
        return fail(c, MSIM_ERR_INVALID, "metric_fill: no particles");
    set_device(c);
    DevBuf& reg = c->tbuf[0];
    DevBuf& acc = c->tbuf[1];
    int rc = upload_regions(c, regions, reg);
    if (rc) return rc;
    CK(acc.ensure(sizeof(unsigned long long) * 2 * c->n_env));
    CK(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long) * 2 * c->n_env, c->stream));
    unsigned long long* inside = acc.as<unsigned long long>();
    launch_fill(params(c), reg.as<double>(), inside, inside + c->n_env, c->stream);
    CK(cudaGetLastError());
    std::vector<unsigned long long> h(2 * (size_t)c->n_env);
    CK(cudaMemcpyAsync(h.data(), acc.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int e = 0; e < c->n_env; ++e) {
      const double n = (double)(c->env_off_h[e + 1] - c->env_off_h[e]);
      out[e].fraction = (double)h[e] / n;
      std::memcpy(&out[e].max_speed, &h[c->n_env + e], sizeof(double));
      out[e].success = out[e].fraction > 0.9 && out[e].max_speed < 0.05;
      out[e]._pad = 0;
    }
    return MSIM_OK;
  });
}

int msim_gpu_render_heightmap(msim_gpu_ctx* c, const msim_region* regions, int nx, int ny, double* maps) {
  return guarded(c, [&]() -> int {
    if (!maps) return fail(c, MSIM_ERR_INVALID, "render_heightmap: maps required");
    set_device(c);
    DevBuf& m = c->tbuf[2];
    DevBuf& reg = c->tbuf[0];
    int rc = heightmaps(c, regions, nx, ny, m, reg);
    if (rc) return rc;
    CK(cudaMemcpyAsync(maps, m.p, sizeof(double) * (size_t)nx * ny * c->n_env, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MSIM_OK;
  });
}

int msim_gpu_metric_write_iou(msim_gpu_ctx* c, const msim_region* regions, int nx, int ny, double threshold,
                              const double* targets, double* iou, int32_t* success) {
  return guarded(c, [&]() -> int {
    if (!targets || !iou || !success) return fail(c, MSIM_ERR_INVALID, "metric_write_iou: null argument");
    set_device(c);
    DevBuf& m = c->tbuf[2];
    DevBuf& reg = c->tbuf[0];
    DevBuf& tg = c->tbuf[3];
    DevBuf& res = c->tbuf[1];
    int rc = heightmaps(c, regions, nx, ny, m, reg);
    if (rc) return rc;
    const size_t cells = (size_t)nx * ny;
    CK(tg.ensure(sizeof(double) * cells * c->n_env));
    CK(cudaMemcpyAsync(tg.p, targets, sizeof(double) * cells * c->n_env, cudaMemcpyHostToDevice, c->stream));
    CK(res.ensure((sizeof(double) + sizeof(int)) * c->n_env));
    double* di = res.as<double>();
    int* ds = reinterpret_cast<int*>(di + c->n_env);
    launch_iou(m.as<double>(), tg.as<double>(), c->n_env, (int)cells, threshold, di, ds, c->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(iou, di, sizeof(double) * c->n_env, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(success, ds, sizeof(int) * c->n_env, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MSIM_OK;
  });
}

int msim_gpu_chamfer(msim_gpu_ctx* c, const double* points, const int64_t* offsets, double* out) {
  return guarded(c, [&]() -> int {
    if (!out) return fail(c, MSIM_ERR_INVALID, "chamfer_distance: out required");
    set_device(c);
    DevBuf& pos = c->tbuf[4];
    DevBuf& pts = c->tbuf[5];
    DevBuf& off_d = c->tbuf[6];
    std::vector<long long> off_h;
    int rc = particle_points(c, pos);
    if (!rc) rc = upload_points(c, points, offsets, pts, off_d, off_h);
    if (rc) return rc;
    chamfer_sets(c, pos.as<double>(), c->env_off_d.as<long long>(), c->env_off_h, pts.as<double>(),
                 off_d.as<long long>(), off_h, out);
    return MSIM_OK;
  });
}

int msim_gpu_metric_pinch(msim_gpu_ctx* c, const double* initial, const int64_t* initial_offsets,
                          const double* target, const int64_t* target_offsets, double* ratio, int32_t* success) {
  return guarded(c, [&]() -> int {
    if (!ratio || !success) return fail(c, MSIM_ERR_INVALID, "metric_pinch: null argument");
    set_device(c);
    DevBuf& pos = c->tbuf[4];
    DevBuf& ini = c->tbuf[5];
    DevBuf& ini_off = c->tbuf[6];
    DevBuf& tgt = c->tbuf[7];
    DevBuf& tgt_off = c->tbuf[8];
    std::vector<long long> ini_h, tgt_h;
    int rc = upload_points(c, initial, initial_offsets, ini, ini_off, ini_h);
    if (!rc) rc = upload_points(c, target, target_offsets, tgt, tgt_off, tgt_h);
    if (!rc) rc = particle_points(c, pos);
    if (rc) return rc;
    std::vector<double> t(c->n_env), d(c->n_env);
    chamfer_sets(c, ini.as<double>(), ini_off.as<long long>(), ini_h, tgt.as<double>(), tgt_off.as<long long>(),
                 tgt_h, t.data());
    chamfer_sets(c, pos.as<double>(), c->env_off_d.as<long long>(), c->env_off_h, tgt.as<double>(),
                 tgt_off.as<long long>(), tgt_h, d.data());
    for (int e = 0; e < c->n_env; ++e) {  // scenario.hpp:205-207
      ratio[e] = t[e] > 0.0 ? d[e] / t[e] : (d[e] == 0.0 ? 0.0 : std::numeric_limits<double>::infinity());
      success[e] = d[e] < 0.3 * t[e];
    }
    return MSIM_OK;
  });
}

// ---- on-device seeding for batched env resets (seeding.hpp:13-35) ----------
int msim_gpu_seed_envs(msim_gpu_ctx* c, int n, const int32_t* envs, const uint64_t* seeds, const double* boxes,
                       int32_t material, double particle_volume) {
  return guarded(c, [&]() -> int {
    if (n < 0 || (n > 0 && (!envs || !seeds || !boxes))) return fail(c, MSIM_ERR_INVALID, "seed_envs: null argument");
    if (material < 0 || material >= (int)c->mats_h.size()) return fail(c, MSIM_ERR_INVALID, "seed_envs: material out of range");
    if (!(particle_volume > 0.0)) return fail(c, MSIM_ERR_INVALID, "seed_envs: particle volume must be > 0");
    if (n == 0) return MSIM_OK;
    // the lattice (seeding.hpp:17-23) in host double, like msim_seed_box
    const double spacing = std::cbrt(particle_volume);
    int cnt[3] = {0, 0, 0};
    std::vector<unsigned char> flag(c->n_env, 0);
    for (int r = 0; r < n; ++r) {
      const int e = envs[r];
      if (e < 0 || e >= c->n_env) return fail(c, MSIM_ERR_INVALID, "seed_envs: env out of range");
      if (flag[e]) return fail(c, MSIM_ERR_INVALID, "seed_envs: env listed twice");
      flag[e] = 1;
      long long total = 1;
      for (int a = 0; a < 3; ++a) {
        const int k = std::max(1, (int)std::floor((boxes[6 * r + 3 + a] - boxes[6 * r + a]) / spacing));
        if (r == 0) cnt[a] = k;
        else if (k != cnt[a]) return fail(c, MSIM_ERR_INVALID, "seed_envs: boxes must give the same lattice shape");
        total *= k;
      }
      if (total != c->env_off_h[e + 1] - c->env_off_h[e])
        return fail(c, MSIM_ERR_INVALID, "seed_envs: lattice count differs from the env's particle count");
    }
    set_device(c);
    cudaStream_t s = c->stream;
    DevBuf& d_env = c->tbuf[0];
    DevBuf& d_seed = c->tbuf[1];
    DevBuf& d_box = c->tbuf[2];
    DevBuf& d_flag = c->tbuf[3];
    DevBuf& d_pos = c->tbuf[4];
    CK(d_env.ensure(sizeof(int) * n));
    CK(d_seed.ensure(sizeof(unsigned long long) * n));
    CK(d_box.ensure(sizeof(double) * 6 * n));
    CK(d_flag.ensure(c->n_env));
    CK(d_pos.ensure(sizeof(double) * 3 * (size_t)std::max<long long>(c->n, 1)));
    CK(cudaMemcpyAsync(d_env.p, envs, sizeof(int) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_seed.p, seeds, sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_box.p, boxes, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_flag.p, flag.data(), c->n_env, cudaMemcpyHostToDevice, s));
    const double density = c->mats_h[material].density;
    launch_seed(params(c), n, d_env.as<int>(), d_seed.as<unsigned long long>(), d_box.as<double>(),
                c->env_off_d.as<long long>(), spacing, cnt[0], cnt[1], d_pos.as<double>(),
                d_flag.as<unsigned char>(), (float)(density * particle_volume), (float)particle_volume,
                (unsigned)material, s);
    CK(cudaGetLastError());
    std::vector<long long> lost(c->n_env);
    std::vector<int> code(c->n_env);
    CK(cudaMemcpyAsync(lost.data(), c->lost_d.p, sizeof(long long) * c->n_env, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(code.data(), c->err_code_d.p, sizeof(int) * c->n_env, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int e = 0; e < c->n_env; ++e)
      if (flag[e]) lost[e] = 0, code[e] = 0;  // a fresh world: no lost particles, no latched error
    CK(cudaMemcpyAsync(c->lost_d.p, lost.data(), sizeof(long long) * c->n_env, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c->err_code_d.p, code.data(), sizeof(int) * c->n_env, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    c->vmax_valid = false;
    c->perm_valid = false;
    return MSIM_OK;
  });
}

// ---- mesh SDF baking (sdf.hpp:277-310) -------------------------------------
namespace {
struct hv3 {
  double x, y, z;
};
hv3 hsub(hv3 a, hv3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
hv3 hcross(hv3 a, hv3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double hnorm(hv3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
hv3 tri_v(const double* tri, int64_t t, int k) { return {tri[9 * t + 3 * k], tri[9 * t + 3 * k + 1], tri[9 * t + 3 * k + 2]}; }

// the grid of bake_mesh_sdf (sdf.hpp:277-296) with the reference's checks
bool bake_grid_impl(const double* tri, int64_t n, double voxel, double padding, double* origin, int* dims,
                    std::string& err) {
  if (!tri || n <= 0) {
    err = "bake_mesh_sdf: empty mesh";
    return false;
  }
  if (voxel <= 0.0) {
    err = "bake_mesh_sdf: voxel size must be > 0";
    return false;
  }
  bool degenerate = true;
  double lo[3] = {tri[0], tri[1], tri[2]}, hi[3] = {tri[0], tri[1], tri[2]};
  for (int64_t t = 0; t < n; ++t) {
    for (int v = 0; v < 3; ++v)
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::min(lo[k], tri[9 * t + 3 * v + k]);
        hi[k] = std::max(hi[k], tri[9 * t + 3 * v + k]);
      }
    const hv3 a = tri_v(tri, t, 0), b = tri_v(tri, t, 1), c = tri_v(tri, t, 2);
    if (hnorm(hcross(hsub(b, a), hsub(c, a))) > 1e-14) degenerate = false;
  }
  if (degenerate) {
    err = "bake_mesh_sdf: mesh has only zero-area triangles";
    return false;
  }
  for (int k = 0; k < 3; ++k) {
    origin[k] = lo[k] - padding;
    const double span = hi[k] - lo[k] + 2.0 * padding;
    dims[k] = std::max(2, static_cast<int>(std::ceil(span / voxel)) + 1);
  }
  return true;
}
}  // namespace

int msim_bake_grid(const double* tri, int64_t n_tri, double voxel, double padding, double* origin, int32_t* dims) {
  g_create_error.clear();
  int d[3];
  double o[3];
  if (!bake_grid_impl(tri, n_tri, voxel, padding, o, d, g_create_error)) return MSIM_ERR_INVALID;
  for (int k = 0; k < 3; ++k) {
    if (origin) origin[k] = o[k];
    if (dims) dims[k] = d[k];
  }
  return MSIM_OK;
}

int msim_gpu_bake_mesh_sdf(int device, const double* tri, int64_t n_tri, double voxel, double padding,
                           float* samples, int64_t samples_cap) {
  g_create_error.clear();
  int d[3];
  double o[3];
  if (!bake_grid_impl(tri, n_tri, voxel, padding, o, d, g_create_error)) return MSIM_ERR_INVALID;
  const long long nvox = (long long)d[0] * d[1] * d[2];
  if (!samples || samples_cap < nvox) {
    g_create_error = "bake_mesh_sdf: samples capacity below dims product";
    return MSIM_ERR_INVALID;
  }
  // the three parity rays of sdf.hpp:258-262, normalized as Vec3::normalized()
  const double raw[9] = {1.0, 0.0, 0.0, 1.0, 0.137, 0.071, 1.0, -0.083, 0.143};
  double dirs[9];
  for (int r = 0; r < 3; ++r) {
    const double nn = hnorm({raw[3 * r], raw[3 * r + 1], raw[3 * r + 2]});
    for (int k = 0; k < 3; ++k) dirs[3 * r + k] = raw[3 * r + k] / nn;
  }
  try {
    CK(cudaSetDevice(device));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf tri_d, out_d;
    CK(tri_d.ensure(sizeof(double) * 9 * n_tri));
    CK(out_d.ensure(sizeof(float) * nvox));
    CK(cudaMemcpyAsync(tri_d.p, tri, sizeof(double) * 9 * n_tri, cudaMemcpyHostToDevice, s));
    launch_bake(tri_d.as<double>(), n_tri, o, voxel, d, dirs, out_d.as<float>(), s);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(samples, out_d.p, sizeof(float) * nvox, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamDestroy(s));
  } catch (const CudaError& e) {
    g_create_error = std::string("CUDA error ") + cudaGetErrorString(e.e) + " at " + e.what;
    return MSIM_ERR_DEVICE;
  }
  return MSIM_OK;
}

// make_box_mesh (sdf.hpp:443-455)
void msim_make_box_mesh(const double* h, const double* center, double* tri) {
  const double c0[3] = {0.0, 0.0, 0.0};
  const double* c = center ? center : c0;
  double v[8][3];
  for (int i = 0; i < 8; ++i) {
    v[i][0] = c[0] + ((i & 1) ? h[0] : -h[0]);
    v[i][1] = c[1] + ((i & 2) ? h[1] : -h[1]);
    v[i][2] = c[2] + ((i & 4) ? h[2] : -h[2]);
  }
  static const int f[12][3] = {{0, 2, 1}, {1, 2, 3}, {4, 5, 6}, {5, 7, 6}, {0, 1, 4}, {1, 5, 4},
                               {2, 6, 3}, {3, 6, 7}, {0, 4, 2}, {2, 4, 6}, {1, 3, 5}, {3, 7, 5}};
  for (int t = 0; t < 12; ++t)
    for (int k = 0; k < 3; ++k)
      for (int a = 0; a < 3; ++a) tri[9 * t + 3 * k + a] = v[f[t][k]][a];
}

void* msim_gpu_stream(msim_gpu_ctx* c) { return c ? (void*)c->stream : nullptr; }

int64_t msim_gpu_launches(const msim_gpu_ctx* c) { return c ? c->timer.launches : -1; }

int msim_gpu_set_kernel_timing(msim_gpu_ctx* c, int on) {
  return guarded(c, [&]() -> int {
    set_device(c);
    CK(cudaStreamSynchronize(c->stream));
    c->timer.reset();
    c->timer.enabled = on != 0;
    return MSIM_OK;
  });
}

int msim_gpu_kernel_count(void) { return kKernelIds; }

int msim_gpu_kernel_stats(msim_gpu_ctx* c, int id, const char** name, int64_t* launches, double* total_ms) {
  if (id < 0 || id >= kKernelIds) return MSIM_ERR_INVALID;
  if (cudaSetDevice(c->device) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess)
    return MSIM_ERR_DEVICE;
  c->timer.flush();
  if (name) *name = kernel_name(id);
  if (launches) *launches = c->timer.count[id];
  if (total_ms) *total_ms = c->timer.total_ms[id];
  return MSIM_OK;
}

int msim_gpu_body_count(const msim_gpu_ctx* c, int env) {
  if (env < 0) {
    int n = 0;
    for (const auto& b : c->bodies_h) n += (int)b.size();
    return n;
  }
  if (env >= c->n_env) return -1;
  return (int)c->bodies_h[env].size();
}

int msim_gpu_sync_all_bodies(msim_gpu_ctx* c, const msim_body* bodies, int n_total) {
  return guarded(c, [&]() -> int {
    set_device(c);
    if (n_total != c->n_bodies) return fail(c, MSIM_ERR_INVALID, "sync_all_bodies: body count mismatch");
    if (n_total == 0) return MSIM_OK;
    static_assert(sizeof(msim_body) == sizeof(BodyDev), "body layouts differ");
    // msim_body and BodyDev share one layout; mass/inertia/com are taken from
    // the caller like sync_rigid_to_soft copies whole bodies.
    CK(cudaMemcpyAsync(c->bodies_d.p, bodies, sizeof(msim_body) * n_total, cudaMemcpyHostToDevice, c->stream));
    SimParams P = params(c);
    launch_rigid(P, 0, -1, c->stream);
    CK(cudaGetLastError());
    return MSIM_OK;
  });
}

int msim_gpu_read_all_wrenches(msim_gpu_ctx* c, int pending, double* wrench6) {
  return guarded(c, [&]() -> int {
    set_device(c);
    if (c->n_bodies == 0) return MSIM_OK;
    const void* src = pending ? c->pending_d.p : c->wrench_d.p;
    CK(cudaMemcpyAsync(wrench6, src, sizeof(double) * 6 * c->n_bodies, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MSIM_OK;
  });
}

}  // extern "C"
