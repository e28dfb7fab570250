// Internal device-state layout shared by the kernels (msim_kernels.cu) and
// the C-ABI host implementation (msim_api.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/msim_gpu.h"
#include "msim_device.cuh"

namespace msim_impl {

constexpr int kMaxBodiesPerEnv = 32;  // wrench slots reduced in shared memory

// Bucket = node block of kBX x kBY x kBZ base cells. Particles are grouped
// by the bucket of their base cell; one CTA processes one bucket with a
// G2P tile of (kB+2) nodes and a P2G tile of (kB+4) nodes per axis.
constexpr int kBX = 4, kBY = 4, kBZ = 2;

// Per-env action of one batched cycle launch.
enum : int {
  kActIdle = 0,     // env finished (or errored): particles are only carried along
  kActP2G = 1,      // first P2G of a call (from stored v, C)
  kActFused = 2,    // G2P of this cycle + P2G of the next cycle in one pass
  kActG2P = 3,      // last G2P of a call (stores v, C)
};

// Device-side stepping state of one environment (independent worlds advance
// their own substeps/cycles; CFL halving is decided per env, mpm.hpp:400-409).
struct EnvRun {
  int substeps_left;   // substeps of this call not yet completed (incl. current)
  int cycle;           // cycle index within the current substep
  int cycles;          // 2^halvings of the current substep
  int soft_in_rigid;   // index of the current substep within its rigid step
  int action;          // kAct* for the next launch
  int next_new_sub;    // the P2G of this launch starts a new substep
  int next_new_rigid;  // ... and a new rigid step
  float dt_c;          // dt / cycles (current cycle): grid update
  int cyc_sum;         // report: cycles executed
  float dt_g2p;        // dt of the G2P in this launch
  float dt_p2g;        // dt folded into the P2G momentum (p + dt f) in this launch;
                       // speculated as the current cycle dt when the P2G opens a new
                       // substep, re-done on the device when the CFL plan disagrees
  int redo;            // this env's P2G must be redone with dt_c (speculation missed)
  int rigid_idx;       // rigid step of the current env_step (kinematic schedule row)
  int det_sm, det_sp;  // deterministic mode: fixed-point exponents of this launch's grid mass / momentum
};

// Deterministic mode (msim_gpu_set_deterministic): every order-dependent float
// sum becomes an integer sum. Grid nodes accumulate int64 fixed point at a
// per-env exponent fixed for the launch; wrench / force-balance sums int64 at
// 2^kDetWrenchExp per N (N m). Particle order: movers sorted by their previous
// slot after k_perm (stayers keep their order by construction).
constexpr int kDetWrenchExp = 36;
constexpr int kDetMomentumExp = 40;  // |largest round bound| ~ 2^-40 of the int64 range per contribution
constexpr int kErrDetRange = 33;     // deterministic fixed-point range exceeded (a contribution grew ~2^15x in one step)
// Programmatic dependent launch (sm_90+) of the per-cycle kernels: each is
// scheduled while its predecessor drains (the launch latency overlaps) and
// waits in pdl_wait() (griddepcontrol.wait: predecessor complete, its writes
// visible) before touching global memory. Kernels launched this way start with
// pdl_wait(); pdl_trigger() lets their own successor be scheduled. Stream
// capture records the programmatic edges in the CUDA graph. MSIM_NO_PDL=1
// launches them plainly (the device calls are then no-ops).
bool pdl_enabled();
template <typename... Params, typename... Args>
inline void launch_pdl(void (*kern)(Params...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, args...) != cudaSuccess) {  // attribute refused: plain launch
    (void)cudaGetLastError();
    kern<<<grid, block, smem, s>>>(args...);
  }
}

// Resident particle-kernel rounds on the device (default build: 5 CTAs / SM x 128
// particles), for the small-scene split heuristic (msim_gpu_set_particles).
constexpr int kParticleCtasPerSm = 5, kParticleRound = 128;

// Internal error codes latched per environment (first one wins); mapped to
// MSIM_ERR_INVALID / MSIM_ERR_DIVERGED with the reference's messages.
enum : int {
  kErrDetStress = 20,     // kirchhoff_stress: det(F) must be > 0        (mpm.hpp:153-154)
  kErrDetReturn = 21,     // von_mises_return_map: det(F) must be > 0    (mpm.hpp:167-168)
  kErrLost = 30,          // lost particle fraction exceeds threshold    (mpm.hpp:246-249)
  kErrCfl = 31,           // CFL violation persists after max halvings   (mpm.hpp:404-405)
  kErrNan = 32,           // NaN/Inf in particle <i>                     (mpm.hpp:374-378)
};
constexpr int kLostBit = 31;
constexpr uint32_t kEnvMask = 0x7FFFFFu;  // meta = lost<<31 | env<<8 | material

// Particle state, fp32 structure-of-arrays (one buffer of a double-buffered
// pair; the P2G pass writes particles into bucket order of the next buffer).
struct Particles {
  float* x[3];
  float* v[3];
  float* C[9];
  float* G[9];  // displacement gradient F - I
  float* mass;
  float* vol0;
  float* jp;     // Fluid: volume ratio J; Drucker-Prager: accumulated plastic strain; else 1
  uint32_t* meta;
  int32_t* pid;  // original (upload-order) index within the context
};

struct BodyDev {
  int mode;
  int _pad;
  double q[4];
  double t[3];
  double v[3];
  double w[3];
  double mass;
  double inertia[3];
  double com_off[3];
};

struct ShapeHost {  // shape description kept on device in double for the rigid kernel
  int type;
  int body;
  double lq[4];
  double lt[3];
  double friction, k_n, k_t;
  double p[4];
  int vol_dims[3];
  double vol_origin[3];
  double vol_voxel;
  long long vol_off;
  double vol_min;  // smallest SDF sample (bounds phi outside the volume box)
};

// Per-kernel CUDA-event timing on the context stream (bench / profiling) and
// the count of kernel launches. Host-only; SimParams carries a pointer.
enum KernelId : int {
  kKPlan = 0, kKVmax, kKClear, kKBin, kKBucketScan, kKScatter, kKP2G, kKBlockScan, kKGrid, kKG2P,
  kKEnd, kKRigid, kKStage, kKRedo, kKernelIds
};
inline const char* kernel_name(int id) {
  static const char* names[kKernelIds] = {"k_plan", "k_vmax", "k_clear", "k_bin", "bucket_scan", "k_scatter",
                                          "k_particles", "block_scan", "k_grid", "k_g2p", "k_iter_end",
                                          "k_iter_begin", "k_stage", "p2g_redo"};
  return id >= 0 && id < kKernelIds ? names[id] : "?";
}
struct KernelTimer {
  bool enabled = false;
  long long launches = 0;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec { int id; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  double total_ms[kKernelIds] = {};
  long long count[kKernelIds] = {};
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  cudaEvent_t begin(cudaStream_t s, int nlaunch) {
    launches += nlaunch;
    if (!enabled) return nullptr;
    cudaEvent_t a = ev();
    cudaEventRecord(a, s);
    return a;
  }
  void end(int id, cudaEvent_t a, cudaStream_t s) {
    if (!enabled || !a) return;
    cudaEvent_t b = ev();
    cudaEventRecord(b, s);
    recs.push_back({id, a, b});
  }
  void flush() {  // call after the stream is synchronized
    for (const Rec& r : recs) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
        total_ms[r.id] += ms;
        count[r.id] += 1;
      }
    }
    recs.clear();
    used = 0;
  }
  void reset() {
    flush();
    for (int i = 0; i < kKernelIds; ++i) { total_ms[i] = 0; count[i] = 0; }
  }
  ~KernelTimer() {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

// Everything a kernel needs, passed by value.
struct SimParams {
  KernelTimer* timer;            // host-side instrumentation (never dereferenced on device)
  // grid
  double h, inv_h;
  double origin[3];
  int dims[3];
  int bdims[3];              // node blocks (4^3 nodes) per axis
  long long nodes_per_env;
  int blocks_per_env;
  int n_env;
  unsigned boundary_slip;    // bit f set => face f is slip
  float gravity[3];
  float h_f, d_inv_f;        // h, 4/h^2
  long long n;               // particles in context
  int n_keys;                // n_env*buckets_per_env + 1 (lost bucket last)
  // particle buckets = qf^3 node blocks (qf = 1 dense scenes, 2 sparse ones):
  // bucket of base cell b = (b >> qshift) within qdims
  int qf;
  int qshift[3];
  int qdims[3];
  int buckets_per_env;
  int n_blocks;              // n_env*blocks_per_env (node-block flags)
  int any_model;             // some material is not the reference's von Mises clay (jp + dispatch)
  int split;                 // keep momentum and force separately
  int split_r;               // rounds of a bucket split over this many CTAs (small scenes; >= 1)
  int grid_mode;             // coupling mode grid
  float r_c_particle, r_c_grid, c_d;
  double dt_full;            // SoftState::dt
  double cfl_h;              // cfl_factor * h
  int max_halvings;
  int n_soft;                // substeps per rigid step
  int integrate_rigid;       // env_step: rigid step at rigid boundaries
  int clear_on_read;         // grid update zeroes consumed P2G accumulators
  double rigid_g[3];
  double dt_r;               // n_soft * dt
  // per-rigid-step kinematic poses ([step][body][qw qx qy qz tx ty tz], bodies of
  // all envs concatenated) for this env_step, applied to sched_mask bodies; 0 steps: none
  const double* sched;
  const unsigned char* sched_mask;
  int sched_steps;
  int n_bodies_total;
  EnvRun* run;
  BodyDev* bodies;
  const ShapeHost* shape_src;
  double* pending;           // staged wrenches (pending_wrenches)
  int* n_running;            // envs with substeps left after the last iteration
  int* any_redo;             // device flag: some env must redo its P2G (see EnvRun::redo)
  int* item_counter;         // [4] dynamic bucket hand-out of the particle kernel: next (main, redo), CTAs done (main, redo)
  int redo_pass;             // this particle launch is the redo pass
  int hooks;                 // run the penalty hooks (0: hook-free phase API, like p2g())

  Particles cur, nxt;
  const msim_dev::MatParams* mats;

  // per env
  const long long* env_off;      // n_env+1
  const int* shape_off;          // n_env+1
  const int* body_off;           // n_env+1
  msim_dev::ShapeDev* shapes;
  const float* vol_pool;
  double* wrench;                // per body: force xyz, torque xyz (accumulating)
  double* applied;               // per env: sum of applied penalty force (this cycle), xyz
  double* react;                 // per env: sum of reactions (this cycle), xyz
  unsigned* max_pen_bits;        // per env, float bits
  unsigned* vmax_bits;           // per env, float bits
  long long* lost_count;         // per env
  int* err_code;                 // per env
  int* err_pid;                  // per env: first offending particle (min pid)
  const double* mean_mass;       // per env (grid-mode scaling)

  // binning
  int* key;
  int* rank;
  int* bucket_count;             // n_keys
  int* move_count;               // n_keys: particles entering a bucket from another one (rank counter)
  int* bucket_start;             // n_keys + 1
  int* active_buckets;           // list
  int* n_active_buckets;
  int* perm;                     // read set: sorted slot -> particle index in cur
  int* perm_w;                   // write set (built after the particle kernel for the next launch)
  int* bucket_start_w;
  int* active_buckets_w;
  int* n_active_buckets_w;
  int* base_dbg;                 // optional: base per pid (3 ints), -10 if lost

  // grid (float4 per node)
  float4* gPM;                   // momentum (or momentum + dt*force) xyz, mass w
  float4* gF;                    // force xyz (split mode)
  float4* gV;                    // velocity xyz
  int* nb_flag;                  // node-block touched flags (n_env*blocks_per_env)
  int* nb_scan;
  int* nb_list;
  int* n_nb;

  int* scan_tmp;
  int* scan_tmp2;  // second scan status area (the node-block scan, concurrent with the bucket scan)
  // deterministic mode (null otherwise)
  int det;
  longlong4* gPMd;               // per node: int64 momentum (or p + dt f) xyz, mass
  long long* w64;                // per body x 6: wrench accumulators at 2^kDetWrenchExp
  long long* a64;                // per env x 3: applied force this cycle
  long long* r64;                // per env x 3: reactions this cycle
  unsigned* det_bnd;             // per env: max momentum-channel round bound of the last launch (float bits)
  const int* det_mexp;           // per env: mass exponent (from the env's total mass)
  double* balance_max;           // per env: max force-balance error this step
  double lost_threshold;
};

// ---- utility kernels (msim_kernels.cu)
void launch_convert_in(const SimParams& P, long long n, const double* x, const double* v,
                       const double* F, const double* C, const double* mass, const double* vol0,
                       const int32_t* mat, const int* env_of, long long first_pid, cudaStream_t s);
void launch_overwrite(const SimParams& P, long long first_pid, long long n, const double* x,
                      const double* v, const double* F, const double* C, cudaStream_t s);
void launch_convert_out(const SimParams& P, long long first_pid, long long n, double* x, double* v,
                        double* F, double* C, uint8_t* lost, cudaStream_t s);
void launch_vmax(const SimParams& P, cudaStream_t s);
void launch_jp_out(const SimParams& P, long long first_pid, long long n, double* jp, cudaStream_t s);
void launch_rigid(const SimParams& P, int integrate, int only_env, cudaStream_t s);
void launch_stage_wrenches(const SimParams& P, int n_bodies, cudaStream_t s);
void launch_constitutive(const msim_dev::MatParams m, long long n, const double* F, double* tau,
                         double* Fp, int* bad, cudaStream_t s);
void launch_grid_out(const SimParams& P, int env, double* mass, double* mom, double* force,
                     double* vel, cudaStream_t s);
void launch_grid_vel_in(const SimParams& P, int env, const double* vel, cudaStream_t s);
void launch_clear_env_grid(const SimParams& P, int env, cudaStream_t s);
void launch_binning_out(const SimParams& P, long long n_env_p, const int* base, int* cell_count,
                        int* cell_start, int* cell_particles, int* node_flag, int* node_scan,
                        int* node_list, int* n_list, long long* active_nodes, int* tmp, cudaStream_t s);
// early: the scan's input is complete before its stream predecessor finishes
// (launched with programmatic dependent launch, it runs concurrently with the
// predecessor and waits for it only before exiting; tmp must not be shared)
void scan_exclusive(int* in, int* out, int n, int* compact_list, int* n_compact, int* tmp,
                    cudaStream_t s, bool early = false);
size_t scan_tmp_ints(int n);

// ---- hot path (msim_substep.cu)
// Bucket keys of the stored positions (after uploads / external writes).
void launch_rebin(const SimParams& P, cudaStream_t s);
// msim_dist.cu: NCCL resolved at run time; each returns nullptr or an error message
const char* nccl_unique_id(unsigned char* id128);
const char* nccl_comm_init(void** comm, int rank, int world, const unsigned char* id128);
void nccl_comm_destroy(void* comm);
const char* launch_step_stats(const SimParams& P, int substeps, double* stats_d, void* comm, cudaStream_t s);
// Zero the grid nodes touched by the last P2G (manual phases) and reset flags.
void launch_clear(const SimParams& P, cudaStream_t s);
// Per-env actions for the phase API (all envs, dt_c = dt).
void launch_set_action(const SimParams& P, int action, float dt, cudaStream_t s);
// Start of a stepping call: substep counters, rigid step 0, CFL plan of substep 0.
void launch_call_begin(const SimParams& P, int n_substeps, int first_action, cudaStream_t s);
// One batched cycle: [iter_begin] -> particle kernel -> bucket scan -> perm ->
// node-block scan -> [iter_end] -> grid update.
void launch_iteration(const SimParams& P, bool bookkeeping, bool grid_update, cudaStream_t s);
// The particle kernel + re-sort only (phase API).
// perm_now = false: the caller launches the next-launch slot map (launch_perm)
// itself, later in the cycle
void launch_particles(const SimParams& P, cudaStream_t s, bool perm_now = true);
void launch_perm(const SimParams& P, cudaStream_t s, bool early);
// Grid update only (phase API).
void launch_grid(const SimParams& P, cudaStream_t s);
// Per-env end-of-launch bookkeeping only (phase API p2g: lost check, balance).
void launch_iteration_end(const SimParams& P, cudaStream_t s);
// Dynamic shared memory opt-in for the particle kernel (call once per device).
void configure_kernels();

// msim_tasks.cu (compiled with --fmad=false): mesh SDF bake and task metrics
void launch_bake(const double* tri, long long n_tri, const double* origin, double voxel, const int* dims,
                 const double* dirs, float* out, cudaStream_t s);
void launch_fill(const SimParams& P, const double* regions, unsigned long long* inside, unsigned long long* vmax_bits,
                 cudaStream_t s);
void launch_heightmap(const SimParams& P, const double* regions, int nx, int ny, unsigned long long* maps,
                      cudaStream_t s);
void launch_iou(const double* maps, const double* targets, int n_env, int cells, double threshold, double* iou,
                int* success, cudaStream_t s);
void launch_positions(const SimParams& P, double* pos, cudaStream_t s);
void launch_seed(const SimParams& P, int n_reset, const int* envs, const unsigned long long* seeds,
                 const double* boxes, const long long* env_off, double spacing, int cx, int cy, double* pos,
                 const unsigned char* env_reset, float mass, float vol0, unsigned material, cudaStream_t s);
void launch_chamfer_side(const double* A, const long long* offA, long long max_na, const double* B,
                         const long long* offB, int n_env, double* mind, double* mean_out, cudaStream_t s);

}  // namespace msim_impl
