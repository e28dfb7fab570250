/*
 * msim_gpu.h — C ABI of the B200-native MLS-MPM soft-body substep.
 *
 * This is the drop-in boundary for the hot path of the reference simulator
 * ("msim", /root/reference/proj). The reference is a header-only C++ library
 * whose soft-body path is entered through these C++ symbols; each entry
 * point below replaces one of them (file:line relative to
 * /root/reference/proj/include/msim/):
 *
 *   msim_gpu_create            SoftState{} + MpmGrid{} + Material{}        mpm.hpp:24-145
 *                              (grid/step parameters, validate())          mpm.hpp:35-41, :103-106
 *   msim_gpu_set_particles     SoftState::particles + init_buffers()       mpm.hpp:111-142
 *   msim_gpu_set_bodies        World::bodies + BodyMirror shapes           coupling.hpp:54-104
 *   msim_gpu_set_coupling      World::coupling (CouplingConfig)            coupling.hpp:20-26
 *   msim_gpu_sync_bodies       sync_rigid_to_soft(World&)                  coupling.hpp:106-117
 *   msim_gpu_set_kinematic_schedule  robot_drive_step / update_link_poses   coupling.hpp:252-258
 *                              -> Robot::set_kinematic_pose per rigid step rigid.hpp:142-151
 *   msim_gpu_soft_substep      soft_substep(st, particle_hook, grid_hook)  mpm.hpp:397-421
 *                              with penalty_particle / penalty_grid hooks  coupling.hpp:151-214
 *   msim_gpu_p2g               p2g(SoftState&)                             mpm.hpp:199-311
 *   msim_gpu_grid_update       grid_update(SoftState&)                     mpm.hpp:315-342
 *   msim_gpu_g2p               g2p_advect(SoftState&)                      mpm.hpp:346-379
 *   msim_gpu_env_step          the rigid/soft part of env_step             coupling.hpp:248-293
 *                              (integrate_free_body, sync, substeps,       rigid.hpp:52-66
 *                               pending_wrenches staging)
 *   msim_gpu_read_*            direct access to SoftState / MpmGrid /      mpm.hpp:76-79, :111-135
 *                              World::wrenches fields                      coupling.hpp:69-70
 *
 * Conventions
 *   - Plain C: POD structs, pointers + sizes, no exceptions cross the ABI.
 *   - Return codes follow the reference CLI (tools/main.cpp:16):
 *       MSIM_OK = 0, MSIM_ERR_INVALID = 2 (std::invalid_argument),
 *       MSIM_ERR_DIVERGED = 3 (SimulationDiverged), MSIM_ERR_DEVICE = 4 (CUDA).
 *     The message (with the first offending particle index where the
 *     reference reports one) is available from msim_gpu_last_error().
 *   - Host arrays are double precision, caller-owned, copied in/out.
 *     Vectors are packed xyz; 3x3 matrices are row-major (M[r*3+c]).
 *     On the device the state is fp32 structure-of-arrays.
 *   - One context owns one device, one stream and a batch of n_env
 *     independent environments ("worlds") sharing one grid description.
 *     A context is not reentrant; distinct contexts may step concurrently.
 */
#ifndef MSIM_GPU_H
#define MSIM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSIM_OK 0
#define MSIM_ERR_INVALID 2
#define MSIM_ERR_DIVERGED 3
#define MSIM_ERR_DEVICE 4

/* BoundaryKind, mpm.hpp:60 */
#define MSIM_BOUNDARY_STICKY 0
#define MSIM_BOUNDARY_SLIP 1

/* CouplingMode, coupling.hpp:18 */
#define MSIM_COUPLING_PARTICLE 0
#define MSIM_COUPLING_GRID 1

/* ShapeGeom variant order, sdf.hpp:65-83 */
#define MSIM_SHAPE_PLANE 0
#define MSIM_SHAPE_SPHERE 1
#define MSIM_SHAPE_BOX 2
#define MSIM_SHAPE_CAPSULE 3
#define MSIM_SHAPE_VOLUME 4

/* BodyMode, rigid.hpp:11. SCRIPTED is a harness extension: a kinematic body
 * whose pose advances with its own constant twist every rigid step (the
 * synthetic stand-in for a robot-driven link, rigid.hpp:142-151). */
#define MSIM_BODY_DYNAMIC 0
#define MSIM_BODY_KINEMATIC 1
#define MSIM_BODY_SCRIPTED 2

/* Constitutive model selector. HENCKY_VON_MISES is the reference's only
 * model (mpm.hpp:150-181). */
#define MSIM_MODEL_HENCKY_VON_MISES 0  /* mpm.hpp:152-181, the reference's model */
/* The north_star's other materials (no reference implementation: parity with
 * the oracle's restatement of the published algorithms):      */
#define MSIM_MODEL_FIXED_COROTATED 1   /* elastic: tau = 2 mu (F - R) F^T + lambda (J - 1) J I   */
#define MSIM_MODEL_DRUCKER_PRAGER 2    /* sand: Hencky + log-strain cone projection (Klar 2016);
                                          yield_stress holds the friction angle in degrees     */
#define MSIM_MODEL_FLUID 3             /* J-only weakly compressible: tau = K (J - 1) J I      */

/* MpmGrid (mpm.hpp:65-107) + SoftState stepping parameters (mpm.hpp:115-120). */
typedef struct msim_soft_desc {
  double h;                        /* cell length */
  int32_t dims[3];                 /* nodes per axis, >= 4 */
  double origin[3];
  uint8_t boundary[6];             /* x-, x+, y-, y+, z-, z+ */
  uint8_t _pad[2];
  double gravity[3];
  double dt;
  double cfl_factor;               /* 0.4 */
  int32_t max_cfl_halvings;        /* 4 */
  int32_t _pad2;
  double lost_fraction_threshold;  /* 0.01 */
} msim_soft_desc;

/* Material (mpm.hpp:24-42). */
typedef struct msim_material {
  double density;
  double youngs;
  double poisson;
  double yield_stress;
  int32_t model;
  int32_t _pad;
} msim_material;

/* Shape (sdf.hpp:87-110) with its geometry flattened.
 *   plane:   params = normal xyz, offset
 *   sphere:  params[0] = radius
 *   box:     params = half extents xyz
 *   capsule: params[0] = half_length (local z), params[1] = radius
 *   volume:  vol_* fields; samples f32 x-fastest (sdf.hpp:20-30), copied. */
typedef struct msim_shape {
  int32_t type;
  int32_t body;                    /* body index within its environment */
  double local_q[4];               /* w x y z */
  double local_t[3];
  double friction;                 /* 0.5 */
  double k_n;                      /* 1e3 */
  double k_t;                      /* 10 */
  double params[4];
  int32_t vol_dims[3];
  int32_t _pad;
  double vol_origin[3];
  double vol_voxel;
  const float* vol_samples;
} msim_shape;

/* RigidBody (rigid.hpp:25-43). */
typedef struct msim_body {
  int32_t mode;
  int32_t _pad;
  double q[4];                     /* w x y z */
  double t[3];
  double v[3];
  double w[3];
  double mass;
  double inertia[3];               /* body-frame principal */
  double com_offset[3];            /* body frame */
} msim_body;

/* CouplingConfig (coupling.hpp:20-26). */
typedef struct msim_coupling {
  int32_t mode;
  int32_t _pad;
  double r_c_factor;               /* 0.5 */
  double c_d;                      /* 10 */
} msim_coupling;

/* StepReport (coupling.hpp:41-50), rigid/soft fields. For a batched context
 * msim_gpu_env_step aggregates over the environments: cfl_cycles = the MAX over
 * envs of each env's cycle count (the reference's per-World count, summed over
 * its substeps), max_penetration / max_force_balance_error = max over envs,
 * lost_particles = sum over envs. Per-env values: msim_gpu_read_report; the
 * sum over envs of cfl_cycles: msim_gpu_step_stats. */
typedef struct msim_step_report {
  int32_t rigid_steps;
  int32_t soft_substeps;
  int32_t cfl_cycles;
  int32_t _pad;
  double max_penetration;
  double max_force_balance_error;
  int64_t lost_particles;
} msim_step_report;

typedef struct msim_gpu_ctx msim_gpu_ctx;

/* ---- lifecycle ---------------------------------------------------------- */
int msim_gpu_create(const msim_soft_desc* desc, const msim_material* materials, int n_materials,
                    int n_env, int device, msim_gpu_ctx** out);
void msim_gpu_destroy(msim_gpu_ctx* ctx);
const char* msim_gpu_last_error(const msim_gpu_ctx* ctx);
/* Error from a failed msim_gpu_create (no context exists yet). */
const char* msim_gpu_create_error(void);
int msim_gpu_version(void);

/* ---- state setup -------------------------------------------------------- */
/* All environments at once: env_offsets[n_env+1] partitions the n particles.
 * x, v: n*3; F, C: n*9 (row-major); mass, vol0: n; material: n (may be NULL). */
int msim_gpu_set_particles(msim_gpu_ctx* ctx, int64_t n, const int64_t* env_offsets,
                           const double* x, const double* v, const double* F, const double* C,
                           const double* mass, const double* vol0, const int32_t* material);
/* Overwrite one environment's particles (count must match). */
int msim_gpu_write_particles(msim_gpu_ctx* ctx, int env, int64_t n, const double* x,
                             const double* v, const double* F, const double* C);
/* Bodies + shapes of one environment; shape.body indexes into bodies. The
 * body order is the contact order (coupling.hpp:75-90). Resets wrenches. */
int msim_gpu_set_bodies(msim_gpu_ctx* ctx, int env, const msim_body* bodies, int n_bodies,
                        const msim_shape* shapes, int n_shapes);
int msim_gpu_set_coupling(msim_gpu_ctx* ctx, const msim_coupling* coupling);
/* sync_rigid_to_soft: overwrite body state (pose/twist) of one env and zero
 * its accumulating wrenches. */
int msim_gpu_sync_bodies(msim_gpu_ctx* ctx, int env, const msim_body* bodies, int n_bodies);
/* Per-rigid-step kinematic collider schedule for the NEXT msim_gpu_env_step
 * (SURVEY.md §8f #1): poses[(r * n_total + i) * 7 + (qw qx qy qz tx ty tz)]
 * for rigid step r < n_steps and body i of all envs concatenated in env order
 * (n_total = msim_gpu_body_count(ctx, -1)). At rigid step r each selected body
 * jumps to its pose and takes the finite-difference twist over the rigid step,
 * exactly how env_step moves robot-driven links (coupling.hpp:252-258 ->
 * Robot::set_kinematic_pose, rigid.hpp:142-151). mask[n_total] selects the
 * bodies (NULL: every MSIM_BODY_KINEMATIC body; dynamic bodies are refused).
 * Uploaded once per env step: the whole env step still runs without a host
 * round trip. n_steps must equal the env step's n_rigid; consumed by it. */
int msim_gpu_set_kinematic_schedule(msim_gpu_ctx* ctx, int n_steps, const double* poses, const uint8_t* mask);
int msim_gpu_set_dt(msim_gpu_ctx* ctx, double dt);
/* World::rigid_gravity (coupling.hpp:60), used by msim_gpu_env_step. */
int msim_gpu_set_rigid_gravity(msim_gpu_ctx* ctx, const double* g3);
int msim_gpu_set_gravity(msim_gpu_ctx* ctx, const double* g3);
int msim_gpu_set_lost_fraction_threshold(msim_gpu_ctx* ctx, double threshold);

/* Deterministic mode (the reference's contract that results do not depend on
 * scheduling, mpm.hpp:7-8): with on = 1, repeated runs from the
 * same inputs give bit-identical particles, grid, wrenches and reports. Every
 * order-dependent float sum becomes an integer sum (int64 fixed point for the
 * grid at per-env exponents fixed per launch, and for the wrenches), and the
 * particle order is kept canonical (stayers in order, movers sorted). Covers
 * env_step / soft_substep in particle coupling mode; costs extra grid traffic.
 * A contribution that outgrows the launch's fixed-point range (~2^15 x the
 * previous launch's largest) reports MSIM_ERR_DIVERGED. */
int msim_gpu_set_deterministic(msim_gpu_ctx* ctx, int on);

/* ---- stepping ----------------------------------------------------------- */
/* n_substeps x soft_substep with the configured penalty hook, all envs.
 * cycles_out (may be NULL) receives the per-env cycle count of the LAST substep. */
int msim_gpu_soft_substep(msim_gpu_ctx* ctx, int n_substeps, int32_t* cycles_out);
/* Hook-free phases for direct solver use (acceptance.cpp:81, test_mpm.cpp). */
int msim_gpu_p2g(msim_gpu_ctx* ctx);
int msim_gpu_grid_update(msim_gpu_ctx* ctx);
int msim_gpu_g2p(msim_gpu_ctx* ctx);
/* The soft/rigid part of env_step (coupling.hpp:248-293) for all envs:
 * n_rigid x { integrate dynamic + scripted bodies with the staged wrenches,
 * sync, n_soft substeps, stage wrenches }. Device-resident: no host round
 * trip per rigid step. */
int msim_gpu_env_step(msim_gpu_ctx* ctx, int n_rigid, int n_soft, msim_step_report* report);

/* ---- readback ----------------------------------------------------------- */
int64_t msim_gpu_particle_count(const msim_gpu_ctx* ctx, int env);
int msim_gpu_read_particles(msim_gpu_ctx* ctx, int env, double* x, double* v, double* F,
                            double* C, uint8_t* lost);
/* The per-particle model scalar of env `env` (upload order): the fluid's
 * volume ratio J, Drucker-Prager's accumulated plastic strain, 1 otherwise. */
int msim_gpu_read_jp(msim_gpu_ctx* ctx, int env, double* jp);
/* Dense per-env grid channels (node_count doubles / node_count*3). velocity
 * is written by grid_update; mass/momentum/force by p2g (+ grid hook). Any
 * pointer may be NULL. Momentum/force are only kept separately in "split"
 * mode (grid coupling or msim_gpu_set_split_channels(ctx,1)). */
int msim_gpu_read_grid(msim_gpu_ctx* ctx, int env, double* mass, double* momentum, double* force,
                       double* velocity);
int msim_gpu_write_grid_velocity(msim_gpu_ctx* ctx, int env, const double* velocity);
int msim_gpu_set_split_channels(msim_gpu_ctx* ctx, int split);
/* Record per-particle base cells during binning so msim_gpu_read_binning can
 * rebuild the reference layout (inspection; costs 12 B/particle/cycle). */
int msim_gpu_set_record_binning(msim_gpu_ctx* ctx, int on);
/* Integer binning of the last p2g, in the reference layout (mpm.hpp:210-280):
 * base[n*3] (lost = -10), cell_start[bins+1], cell_particles[n_alive],
 * active_nodes[n_active] ascending. Capacities are checked; counts returned. */
int msim_gpu_read_binning(msim_gpu_ctx* ctx, int env, int32_t* base, int32_t* cell_start,
                          int64_t cell_start_cap, int32_t* cell_particles, int64_t cell_particles_cap,
                          int64_t* n_alive, int64_t* active_nodes, int64_t active_cap,
                          int64_t* n_active);
/* The hot path's OWN integer binning (not a rebuild), for bit-exact parity
 * with the reference's counting sort and active nodes (mpm.hpp:251-280):
 *   - particle buckets of bucket_cells[3] base cells, bucket_dims[3] of them
 *     per env (bucket id = (bz*bucket_dims[1] + by)*bucket_dims[0] + bx of
 *     base / bucket_cells); counts[bucket_dims product] = particles per bucket
 *     in the bucket structure the NEXT particle launch reads (after msim_gpu_p2g:
 *     the histogram of the base cells that P2G binned; lost particles excluded);
 *   - the node blocks (4x4x2 nodes; block id = (kz*block_dims[1] + ky)*
 *     block_dims[0] + kx) the LAST P2G launch touched, ascending: exactly the
 *     blocks holding a node of some occupied base cell's 3x3x3 stencil, i.e.
 *     the reference's active_nodes at block granularity.
 * Any output pointer may be NULL. */
int msim_gpu_read_buckets(msim_gpu_ctx* ctx, int env, int32_t* bucket_cells, int32_t* bucket_dims,
                          int32_t* counts, int64_t counts_cap, int32_t* block_dims, int32_t* blocks,
                          int64_t blocks_cap, int64_t* n_blocks);
int msim_gpu_read_wrenches(msim_gpu_ctx* ctx, int env, int pending, double* force,
                           double* torque);
int msim_gpu_read_bodies(msim_gpu_ctx* ctx, int env, msim_body* bodies, int n_bodies);
int msim_gpu_read_report(msim_gpu_ctx* ctx, int env, msim_step_report* report);
int64_t msim_gpu_lost_count(msim_gpu_ctx* ctx, int env);

/* ---- batched host<->device exchange (one copy for all envs) ------------ */
int msim_gpu_body_count(const msim_gpu_ctx* ctx, int env); /* env < 0: all envs */
/* Overwrite the state of every body of every env (concatenated in env order)
 * and sync mirrors (sync_rigid_to_soft for all envs). */
int msim_gpu_sync_all_bodies(msim_gpu_ctx* ctx, const msim_body* bodies, int n_total);
/* force xyz, torque xyz per body, all envs concatenated (n_total*6 doubles). */
int msim_gpu_read_all_wrenches(msim_gpu_ctx* ctx, int pending, double* wrench6);

/* ---- multi-GPU statistics ----------------------------------
 * One process per GPU, each context owning a contiguous range of independent
 * envs; the only exchange is the per-env-step statistics, reduced over the
 * context's envs on the device and all-reduced with NCCL on the context's
 * stream (stream-ordered after the env step, capturable). NCCL is resolved
 * at run time from the process (no link dependency).
 *   msim_gpu_nccl_unique_id: rank 0 makes the id, the caller broadcasts it;
 *   msim_gpu_comm_init: every rank joins (rank, world, id);
 *   msim_gpu_step_stats: statistics of the LAST env step of this context
 *     (allreduce = 0) or of all ranks (allreduce = 1):
 *     sums[4] = particle-substeps, env steps, CFL cycles, lost particles;
 *     maxs[2] = max penetration, max force-balance error. */
int msim_gpu_nccl_unique_id(uint8_t* id128);
int msim_gpu_comm_init(msim_gpu_ctx* ctx, int rank, int world, const uint8_t* id128);
int msim_gpu_step_stats(msim_gpu_ctx* ctx, int allreduce, double* sums, double* maxs);

/* ---- instrumentation ---------------------------------------------------- */
void* msim_gpu_stream(msim_gpu_ctx* ctx);          /* the context's cudaStream_t */
int64_t msim_gpu_launches(const msim_gpu_ctx* ctx);  /* kernels launched so far */
int msim_gpu_set_kernel_timing(msim_gpu_ctx* ctx, int on);  /* CUDA events per kernel; resets */
int msim_gpu_kernel_count(void);
int msim_gpu_kernel_stats(msim_gpu_ctx* ctx, int id, const char** name, int64_t* launches,
                          double* total_ms);

/* ---- test hooks (constitutive model on raw arrays, device code path) ---- */
/* tau[n*9] = kirchhoff_stress(F), Fp[n*9] = von_mises_return_map(F) for material
 * `mat`. Returns MSIM_ERR_INVALID if some det(F) <= 0. */
int msim_gpu_constitutive(msim_gpu_ctx* ctx, int mat, int64_t n, const double* F, double* tau,
                          double* Fp);

/* Tuning: particle buckets of factor^3 node blocks of 4x4x2 cells (1: dense
 * scenes, 2: sparse ones, 0: chosen at set_particles from h^3 / mean volume0,
 * the default). Results do not depend on it (bucketing is internal). */
int msim_gpu_set_bucket_factor(msim_gpu_ctx* ctx, int factor);

/* ---- task metrics over every env's device state -------
 * The reference evaluates these on the host particle vector after the
 * episode (scenario.hpp:63-209); here one launch covers all envs and only the
 * per-env results cross PCIe. Positions / velocities are the stored fp32
 * values promoted to double; all particles count, lost ones included (the
 * reference's `w.soft.particles`). Results are bit-identical to the reference
 * formulas on those values, except chamfer means (summation order, ~1e-15). */
typedef struct msim_region {       /* RegionBox (scenario.hpp:18-30) */
  double min[3];
  double max[3];
} msim_region;
typedef struct msim_fill_result {  /* FillResult (scenario.hpp:55-59) */
  double fraction;
  double max_speed;
  int32_t success;
  int32_t _pad;
} msim_fill_result;
/* metric_fill (scenario.hpp:63-75) per env; regions[n_env], out[n_env]. */
int msim_gpu_metric_fill(msim_gpu_ctx* ctx, const msim_region* regions, msim_fill_result* out);
/* render_heightmap (scenario.hpp:79-98) per env into maps[n_env*ny*nx]
 * (x fastest, heights above the region floor, 0 where no particle). */
int msim_gpu_render_heightmap(msim_gpu_ctx* ctx, const msim_region* regions, int nx, int ny, double* maps);
/* render_heightmap + metric_write_iou (scenario.hpp:106-119) against
 * targets[n_env*ny*nx] with the occupancy threshold; iou/success per env. */
int msim_gpu_metric_write_iou(msim_gpu_ctx* ctx, const msim_region* regions, int nx, int ny,
                              double threshold, const double* targets, double* iou, int32_t* success);
/* chamfer_distance (scenario.hpp:179-190) of each env's particles against
 * points[offsets[e]*3 .. offsets[e+1]*3); out[n_env]. */
int msim_gpu_chamfer(msim_gpu_ctx* ctx, const double* points, const int64_t* offsets, double* out);
/* metric_pinch (scenario.hpp:199-209) per env: current = the env's particles;
 * initial / target point sets per env with their offsets. */
int msim_gpu_metric_pinch(msim_gpu_ctx* ctx, const double* initial, const int64_t* initial_offsets,
                          const double* target, const int64_t* target_offsets, double* ratio,
                          int32_t* success);

/* ---- on-device seeding for batched env resets --------
 * seed_particles_box (seeding.hpp:13-35) run on the device for n envs at once:
 * env envs[i] is refilled from a fresh std::mt19937_64(seeds[i]) over the box
 * boxes[i*6 .. +6) = (min xyz, max xyz) with the jittered lattice of spacing
 * cbrt(particle_volume); its particles (upload order) get those positions,
 * v = 0, F = I, C = 0, mass = density(material) * particle_volume, volume0 =
 * particle_volume and the material; lost flags, the lost count and a latched
 * error are cleared. Every box must give the same lattice shape and its count
 * must equal the env's particle count (MSIM_ERR_INVALID otherwise). Positions
 * equal msim_seed_box's (the reference's draws, GCC argument order) rounded
 * to fp32. Bodies are reset by the caller (msim_gpu_sync_bodies). */
int msim_gpu_seed_envs(msim_gpu_ctx* ctx, int n, const int32_t* envs, const uint64_t* seeds, const double* boxes,
                       int32_t material, double particle_volume);

/* ---- mesh SDF baking ----------------------------------
 * bake_mesh_sdf (sdf.hpp:277-310) on a GPU: triangles tri[n_tri*9] (a, b, c
 * per triangle). msim_bake_grid returns the volume's origin and dims (host
 * only, same validation and errors as the reference); msim_gpu_bake_mesh_sdf
 * fills samples[dims product] (f32, x fastest), bit-identical to the reference
 * algorithm in double. Errors: MSIM_ERR_INVALID (empty / degenerate mesh,
 * voxel <= 0, capacity), MSIM_ERR_DEVICE; message via msim_gpu_create_error(). */
int msim_bake_grid(const double* tri, int64_t n_tri, double voxel, double padding, double* origin,
                   int32_t* dims);
int msim_gpu_bake_mesh_sdf(int device, const double* tri, int64_t n_tri, double voxel, double padding,
                           float* samples, int64_t samples_cap);
/* make_box_mesh (sdf.hpp:443-455): 12 outward-wound triangles into tri[108]. */
void msim_make_box_mesh(const double* half_extents, const double* center, double* tri);

/* ---- host-side reference utilities (no device work) --------------------- */
/* seed_particles_box (seeding.hpp:13-35) with a caller-held mt19937_64 state.
 * Returns the particle count; if x != NULL writes positions (n*3) and mass. */
typedef struct msim_rng msim_rng;
msim_rng* msim_rng_create(uint64_t seed);
void msim_rng_destroy(msim_rng* rng);
double msim_rng_uniform(msim_rng* rng, double lo, double hi);
/* n successive msim_rng_uniform(lo, hi) draws. */
void msim_rng_fill_uniform(msim_rng* rng, int64_t n, double lo, double hi, double* out);
int64_t msim_seed_box_count(const double* box_min, const double* box_max, double particle_volume);
int64_t msim_seed_box(msim_rng* rng, const double* box_min, const double* box_max,
                      double density, double particle_volume, double* x, double* mass);

#ifdef __cplusplus
}
#endif

#endif /* MSIM_GPU_H */
