// ORACLE — TEST INFRASTRUCTURE ONLY. Built by Makefile.ref into _ref/libmsim_ref.so.
//
// An extern "C" harness around the REFERENCE's own, unchanged sources
// (/root/reference/proj/include/msim/*.hpp, compiled against the Eigen
// subset in ref_shim/): World, SoftState, soft_substep, p2g / grid_update /
// g2p_advect, penalty_particle / penalty_grid, sync_rigid_to_soft,
// integrate_free_body, Robot::set_kinematic_pose, seed_particles_box,
// state_hash and env_step are the reference's functions. The surface
// mirrors oracle_capi.cpp (prefix ref_ instead of oracle_) so the tests can
// run the restatement (oracle/_build/liboracle.so) and the reference itself on
// the same inputs, and bench.py's --impl reference arm times this library.
//
// Harness code (NOT reference code) is limited to:
//   * descriptor marshalling (include/msim_gpu.h structs -> msim types);
//   * MSIM_BODY_SCRIPTED bodies: the reference has no such mode; a scripted
//     body is a kinematic body whose pose the harness advances each rigid
//     step with its constant twist (the pose half of integrate_free_body,
//     rigid.hpp:61-65), as the oracle and the GPU path do;
//   * a per-rigid-step kinematic pose schedule, applied with the reference's
//     Robot::set_kinematic_pose (rigid.hpp:142-151) exactly as robot-driven
//     links are moved inside env_step (coupling.hpp:252-258);
//   * when either of those is present, the rigid/soft loop of env_step
//     (coupling.hpp:248-293) is driven here with the same call order and the
//     same StepReport diagnostics; otherwise msim::env_step itself runs;
#include "msim/coupling.hpp"
#include "msim/seeding.hpp"

#include "../include/msim_gpu.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <thread>

using namespace msim;

struct ref_world {
  World w;
  std::vector<std::uint8_t> scripted;    // per body
  std::vector<double> schedule;          // [steps][bodies][7] (qw qx qy qz tx ty tz)
  std::vector<std::uint8_t> sched_mask;  // per body
  int sched_steps = 0;
  std::string err;
};

namespace {

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
void put(double* d, const Vec3& v) { d[0] = v.x(); d[1] = v.y(); d[2] = v.z(); }
Mat3 m3(const double* p) {  // row-major in, Eigen storage out
  Mat3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m(r, c) = p[r * 3 + c];
  return m;
}
void put(double* d, const Mat3& m) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) d[r * 3 + c] = m(r, c);
}
Quat quat(const double* q) { return Quat(q[0], q[1], q[2], q[3]); }

Shape shape_from(const msim_shape& s) {
  Shape o;
  switch (s.type) {
    case MSIM_SHAPE_PLANE: o.geom = PlaneGeom{v3(s.params), s.params[3]}; break;
    case MSIM_SHAPE_SPHERE: o.geom = SphereGeom{s.params[0]}; break;
    case MSIM_SHAPE_BOX: o.geom = BoxGeom{v3(s.params)}; break;
    case MSIM_SHAPE_CAPSULE: o.geom = CapsuleGeom{s.params[0], s.params[1]}; break;
    case MSIM_SHAPE_VOLUME: {
      auto vol = std::make_shared<SdfVolume>();
      vol->origin = v3(s.vol_origin);
      vol->voxel = s.vol_voxel;
      vol->dims = Eigen::Vector3i(s.vol_dims[0], s.vol_dims[1], s.vol_dims[2]);
      const std::size_t n = std::size_t(s.vol_dims[0]) * s.vol_dims[1] * s.vol_dims[2];
      vol->samples.assign(s.vol_samples, s.vol_samples + n);
      o.geom = VolumeGeom{vol};
      break;
    }
    default: throw std::invalid_argument("unknown shape type");
  }
  o.local_pose = Pose(quat(s.local_q), v3(s.local_t));
  o.friction = s.friction;
  o.k_n = s.k_n;
  o.k_t = s.k_t;
  return o;
}

void body_to(const RigidBody& b, bool scripted, msim_body* o) {
  o->mode = scripted ? MSIM_BODY_SCRIPTED : (b.mode == BodyMode::Dynamic ? MSIM_BODY_DYNAMIC : MSIM_BODY_KINEMATIC);
  o->q[0] = b.pose.rotation.w(); o->q[1] = b.pose.rotation.x();
  o->q[2] = b.pose.rotation.y(); o->q[3] = b.pose.rotation.z();
  put(o->t, b.pose.translation);
  put(o->v, b.linear_velocity);
  put(o->w, b.angular_velocity);
  o->mass = b.mass;
  put(o->inertia, b.inertia);
  put(o->com_offset, b.com_offset);
}

template <class F>
int guarded(ref_world* w, F&& f) {
  try {
    f();
    return MSIM_OK;
  } catch (const SimulationDiverged& e) {
    if (w) w->err = e.what();
    return MSIM_ERR_DIVERGED;
  } catch (const std::invalid_argument& e) {
    if (w) w->err = e.what();
    return MSIM_ERR_INVALID;
  } catch (const std::exception& e) {
    if (w) w->err = e.what();
    return MSIM_ERR_INVALID;
  }
}

// Harness: constant-twist pose advance of a scripted body (the pose update of
// integrate_free_body, rigid.hpp:61-65, with the velocities left unchanged).
void advance_scripted(RigidBody& b, double dt) {
  const Vec3 com = b.world_com();
  const Vec3 com_new = com + dt * b.linear_velocity;
  const Quat dq = quat_exp(b.angular_velocity * dt);
  const Quat rot_new = (dq * b.pose.rotation).normalized();
  b.pose = Pose(rot_new, com_new - rot_new * b.com_offset);
}

// The rigid/soft loop of env_step (coupling.hpp:248-293) for worlds with
// scripted or scheduled kinematic bodies (no robot / controller here).
StepReport harness_env_step(ref_world* rw) {
  World& w = rw->w;
  StepReport rep;
  const double dt_r = w.dt_rigid();
  if (rw->sched_steps > 0 && rw->sched_steps != w.n_rigid)
    throw std::invalid_argument("kinematic schedule length != n_rigid");
  for (int r = 0; r < w.n_rigid; ++r) {
    for (std::size_t i = 0; i < w.bodies.size(); ++i)
      integrate_free_body(w.bodies[i], w.pending_wrenches[i], w.rigid_gravity, dt_r);
    for (std::size_t i = 0; i < w.bodies.size(); ++i) {
      if (rw->scripted[i]) advance_scripted(w.bodies[i], dt_r);
      if (rw->sched_steps > 0 && rw->sched_mask[i]) {
        const double* p = rw->schedule.data() + 7 * (static_cast<std::size_t>(r) * w.bodies.size() + i);
        Robot::set_kinematic_pose(w.bodies[i], Pose(quat(p), v3(p + 4)), dt_r);
      }
    }
    sync_rigid_to_soft(w);
    for (int s = 0; s < w.n_soft; ++s) {
      auto reaction_total = [&] {
        Vec3 acc = Vec3::Zero();
        for (const WrenchBuffer& b : w.wrenches) acc += b.force;
        return acc;
      };
      auto on_particles = [&](SoftState& st) {
        if (w.coupling.mode != CouplingMode::Particle) return;
        const Vec3 r0 = reaction_total();
        penalty_particle(w, &rep.max_penetration);
        Vec3 applied = Vec3::Zero();
        for (const Vec3& f : st.ext_force) applied += f;
        rep.max_force_balance_error = std::max(rep.max_force_balance_error, (reaction_total() - r0 + applied).norm());
      };
      auto on_grid = [&](SoftState& st) {
        if (w.coupling.mode != CouplingMode::Grid) return;
        const Vec3 r0 = reaction_total();
        const std::vector<Vec3> f0 = st.grid.force;
        penalty_grid(w, &rep.max_penetration);
        Vec3 applied = Vec3::Zero();
        for (std::size_t ni : st.scratch.active_nodes) applied += st.grid.force[ni] - f0[ni];
        rep.max_force_balance_error = std::max(rep.max_force_balance_error, (reaction_total() - r0 + applied).norm());
      };
      rep.cfl_cycles += soft_substep(w.soft, on_particles, on_grid);
      ++rep.soft_substeps;
    }
    w.pending_wrenches = w.wrenches;
    ++rep.rigid_steps;
  }
  w.time += w.n_rigid * w.n_soft * w.soft.dt;
  rep.lost_particles = w.soft.lost_count;
  return rep;
}

StepReport step_world(ref_world* rw) {
  bool any_scripted = false;
  for (std::uint8_t s : rw->scripted) any_scripted |= s != 0;
  StepReport r = (any_scripted || rw->sched_steps > 0) ? harness_env_step(rw) : env_step(rw->w, VecX());
  rw->sched_steps = 0;  // a schedule drives exactly one env step
  rw->schedule.clear();
  return r;
}

void report_to(const StepReport& r, msim_step_report* rep) {
  if (!rep) return;
  rep->rigid_steps = r.rigid_steps;
  rep->soft_substeps = r.soft_substeps;
  rep->cfl_cycles = r.cfl_cycles;
  rep->max_penetration = r.max_penetration;
  rep->max_force_balance_error = r.max_force_balance_error;
  rep->lost_particles = int64_t(r.lost_particles);
}

}  // namespace

extern "C" {

ref_world* ref_create(const msim_soft_desc* d, const msim_material* mats, int n_mat) {
  auto* o = new ref_world();
  SoftState& st = o->w.soft;
  st.grid.h = d->h;
  st.grid.dims = Eigen::Vector3i(d->dims[0], d->dims[1], d->dims[2]);
  st.grid.origin = v3(d->origin);
  for (int f = 0; f < 6; ++f) st.grid.boundary[f] = d->boundary[f] ? BoundaryKind::Slip : BoundaryKind::Sticky;
  st.gravity = v3(d->gravity);
  st.dt = d->dt;
  st.cfl_factor = d->cfl_factor;
  st.max_cfl_halvings = d->max_cfl_halvings;
  st.lost_fraction_threshold = d->lost_fraction_threshold;
  for (int i = 0; i < n_mat; ++i) {
    if (mats[i].model != MSIM_MODEL_HENCKY_VON_MISES) o->err = "material model not in the reference (von Mises only)";
    st.materials.push_back(Material{mats[i].density, mats[i].youngs, mats[i].poisson, mats[i].yield_stress});
  }
  return o;
}

void ref_destroy(ref_world* w) { delete w; }
const char* ref_last_error(ref_world* w) { return w->err.c_str(); }
void ref_set_threads(int n) { worker_threads() = n; }
// non-empty: a material model the reference does not have was requested
int ref_unsupported(ref_world* w) { return w->err.empty() ? 0 : 1; }

int ref_set_particles(ref_world* w, int64_t n, const double* x, const double* v, const double* F, const double* C,
                      const double* mass, const double* vol0, const int32_t* mat) {
  auto& ps = w->w.soft.particles;
  ps.assign(n, Particle{});
  for (int64_t i = 0; i < n; ++i) {
    Particle& p = ps[i];
    p.x = v3(x + 3 * i);
    p.v = v ? v3(v + 3 * i) : Vec3::Zero();
    p.F = F ? m3(F + 9 * i) : Mat3::Identity();
    p.C = C ? m3(C + 9 * i) : Mat3::Zero();
    p.mass = mass[i];
    p.volume0 = vol0[i];
    p.material = mat ? mat[i] : 0;
  }
  return MSIM_OK;
}

int ref_write_particles(ref_world* w, int64_t n, const double* x, const double* v, const double* F, const double* C) {
  auto& ps = w->w.soft.particles;
  if (int64_t(ps.size()) != n) return MSIM_ERR_INVALID;
  for (int64_t i = 0; i < n; ++i) {
    if (x) ps[i].x = v3(x + 3 * i);
    if (v) ps[i].v = v3(v + 3 * i);
    if (F) ps[i].F = m3(F + 9 * i);
    if (C) ps[i].C = m3(C + 9 * i);
  }
  return MSIM_OK;
}

int ref_set_bodies(ref_world* w, const msim_body* bodies, int n_bodies, const msim_shape* shapes, int n_shapes) {
  return guarded(w, [&] {
    auto& bs = w->w.bodies;
    bs.assign(n_bodies, RigidBody{});
    w->scripted.assign(n_bodies, 0);
    w->sched_mask.assign(n_bodies, 0);
    for (int i = 0; i < n_bodies; ++i) {
      const msim_body& b = bodies[i];
      RigidBody& o = bs[i];
      o.mode = b.mode == MSIM_BODY_DYNAMIC ? BodyMode::Dynamic : BodyMode::Kinematic;
      w->scripted[i] = b.mode == MSIM_BODY_SCRIPTED;
      o.pose = Pose(quat(b.q), v3(b.t));
      o.linear_velocity = v3(b.v);
      o.angular_velocity = v3(b.w);
      o.mass = b.mass;
      o.inertia = v3(b.inertia);
      o.com_offset = v3(b.com_offset);
    }
    for (int s = 0; s < n_shapes; ++s) {
      if (shapes[s].body < 0 || shapes[s].body >= n_bodies) throw std::invalid_argument("shape body index out of range");
      bs[shapes[s].body].shapes.push_back(shape_from(shapes[s]));
    }
  });
}

int ref_sync_bodies(ref_world* w, const msim_body* bodies, int n_bodies) {
  auto& bs = w->w.bodies;
  if (int(bs.size()) != n_bodies) return MSIM_ERR_INVALID;
  for (int i = 0; i < n_bodies; ++i) {
    bs[i].pose = Pose(quat(bodies[i].q), v3(bodies[i].t));
    bs[i].linear_velocity = v3(bodies[i].v);
    bs[i].angular_velocity = v3(bodies[i].w);
  }
  sync_rigid_to_soft(w->w);
  return MSIM_OK;
}

// One pose (qw qx qy qz tx ty tz) per body per rigid step for the next
// env step; mask selects the bodies moved by it (NULL: every kinematic body).
int ref_set_kinematic_schedule(ref_world* w, int n_steps, const double* poses, const uint8_t* mask) {
  const std::size_t nb = w->w.bodies.size();
  w->sched_steps = n_steps;
  w->schedule.assign(poses, poses + 7 * nb * static_cast<std::size_t>(n_steps));
  w->sched_mask.assign(nb, 0);
  for (std::size_t i = 0; i < nb; ++i)
    w->sched_mask[i] = mask ? mask[i] : (w->w.bodies[i].mode == BodyMode::Kinematic && !w->scripted[i]);
  return MSIM_OK;
}

int ref_set_coupling(ref_world* w, const msim_coupling* c) {
  w->w.coupling.mode = c->mode == MSIM_COUPLING_GRID ? CouplingMode::Grid : CouplingMode::Particle;
  w->w.coupling.r_c_factor = c->r_c_factor;
  w->w.coupling.c_d = c->c_d;
  return MSIM_OK;
}

int ref_set_stepping(ref_world* w, int n_rigid, int n_soft, const double* rigid_gravity) {
  w->w.n_rigid = n_rigid;
  w->w.n_soft = n_soft;
  if (rigid_gravity) w->w.rigid_gravity = v3(rigid_gravity);
  return MSIM_OK;
}

int ref_set_dt(ref_world* w, double dt) { w->w.soft.dt = dt; return MSIM_OK; }
int ref_set_gravity(ref_world* w, const double* g) { w->w.soft.gravity = v3(g); return MSIM_OK; }
int ref_set_lost_fraction_threshold(ref_world* w, double t) { w->w.soft.lost_fraction_threshold = t; return MSIM_OK; }
int ref_init(ref_world* w) { return guarded(w, [&] { w->w.init(); }); }
int ref_init_buffers(ref_world* w) { return guarded(w, [&] { w->w.soft.init_buffers(); }); }

int ref_env_step(ref_world* w, msim_step_report* rep) {
  return guarded(w, [&] { report_to(step_world(w), rep); });
}

// soft_substep with the penalty hook of the configured coupling mode.
int ref_soft_substep(ref_world* w, int n, int use_hooks, int32_t* cycles) {
  return guarded(w, [&] {
    World& W = w->w;
    ParticleForceHook ph = nullptr;
    GridForceHook gh = nullptr;
    if (use_hooks) {
      ph = [&W](SoftState&) { if (W.coupling.mode == CouplingMode::Particle) penalty_particle(W); };
      gh = [&W](SoftState&) { if (W.coupling.mode == CouplingMode::Grid) penalty_grid(W); };
    }
    for (int i = 0; i < n; ++i) {
      const int c = soft_substep(W.soft, ph, gh);
      if (cycles) *cycles = c;
    }
  });
}

int ref_p2g(ref_world* w) { return guarded(w, [&] { p2g(w->w.soft); }); }
int ref_grid_update(ref_world* w) { return guarded(w, [&] { grid_update(w->w.soft); }); }
int ref_g2p(ref_world* w) { return guarded(w, [&] { g2p_advect(w->w.soft); }); }
int ref_grid_clear(ref_world* w) { w->w.soft.grid.clear(); return MSIM_OK; }
int ref_penalty_particle(ref_world* w, double* max_pen) { return guarded(w, [&] { penalty_particle(w->w, max_pen); }); }
int ref_penalty_grid(ref_world* w, double* max_pen) { return guarded(w, [&] { penalty_grid(w->w, max_pen); }); }

int64_t ref_particle_count(ref_world* w) { return int64_t(w->w.soft.particles.size()); }

int ref_read_particles(ref_world* w, double* x, double* v, double* F, double* C, uint8_t* lost) {
  const auto& ps = w->w.soft.particles;
  for (std::size_t i = 0; i < ps.size(); ++i) {
    if (x) put(x + 3 * i, ps[i].x);
    if (v) put(v + 3 * i, ps[i].v);
    if (F) put(F + 9 * i, ps[i].F);
    if (C) put(C + 9 * i, ps[i].C);
    if (lost) lost[i] = i < w->w.soft.lost.size() ? w->w.soft.lost[i] : 0;
  }
  return MSIM_OK;
}

int ref_read_jp(ref_world* w, double* jp) {  // the reference has no per-particle model scalar
  for (std::size_t i = 0; i < w->w.soft.particles.size(); ++i) jp[i] = 1.0;
  return MSIM_OK;
}

int ref_read_ext_force(ref_world* w, double* f) {
  const auto& ef = w->w.soft.ext_force;
  for (std::size_t i = 0; i < ef.size(); ++i) put(f + 3 * i, ef[i]);
  return MSIM_OK;
}

int ref_read_grid(ref_world* w, double* mass, double* momentum, double* force, double* velocity) {
  const MpmGrid& g = w->w.soft.grid;
  for (std::size_t i = 0; i < g.node_count(); ++i) {
    if (mass) mass[i] = g.mass[i];
    if (momentum) put(momentum + 3 * i, g.momentum[i]);
    if (force) put(force + 3 * i, g.force[i]);
    if (velocity) put(velocity + 3 * i, g.velocity[i]);
  }
  return MSIM_OK;
}

int ref_write_grid_velocity(ref_world* w, const double* v) {
  MpmGrid& g = w->w.soft.grid;
  for (std::size_t i = 0; i < g.node_count(); ++i) g.velocity[i] = v3(v + 3 * i);
  return MSIM_OK;
}

int ref_read_binning(ref_world* w, int32_t* base, int32_t* cell_start, int64_t cs_cap, int32_t* cell_particles,
                     int64_t cp_cap, int64_t* n_alive, int64_t* active, int64_t a_cap, int64_t* n_active) {
  const auto& sc = w->w.soft.scratch;
  if (base)
    for (std::size_t i = 0; i < sc.base.size(); ++i) {
      base[3 * i] = sc.base[i].x();
      base[3 * i + 1] = sc.base[i].y();
      base[3 * i + 2] = sc.base[i].z();
    }
  if (int64_t(sc.cell_start.size()) > cs_cap || int64_t(sc.cell_particles.size()) > cp_cap ||
      int64_t(sc.active_nodes.size()) > a_cap)
    return MSIM_ERR_INVALID;
  if (cell_start) std::memcpy(cell_start, sc.cell_start.data(), sc.cell_start.size() * 4);
  if (cell_particles) std::memcpy(cell_particles, sc.cell_particles.data(), sc.cell_particles.size() * 4);
  *n_alive = int64_t(sc.cell_particles.size());
  if (active)
    for (std::size_t i = 0; i < sc.active_nodes.size(); ++i) active[i] = int64_t(sc.active_nodes[i]);
  *n_active = int64_t(sc.active_nodes.size());
  return MSIM_OK;
}

int ref_read_wrenches(ref_world* w, int pending, double* force, double* torque) {
  const auto& ws = pending ? w->w.pending_wrenches : w->w.wrenches;
  for (std::size_t i = 0; i < ws.size(); ++i) {
    put(force + 3 * i, ws[i].force);
    put(torque + 3 * i, ws[i].torque);
  }
  return MSIM_OK;
}

int ref_read_bodies(ref_world* w, msim_body* out, int n) {
  for (int i = 0; i < n && i < int(w->w.bodies.size()); ++i) body_to(w->w.bodies[i], w->scripted[i], out + i);
  return MSIM_OK;
}

int64_t ref_lost_count(ref_world* w) { return int64_t(w->w.soft.lost_count); }
double ref_time(ref_world* w) { return w->w.time; }
double ref_mean_particle_mass(ref_world* w) { return w->w.mean_particle_mass; }
uint64_t ref_state_hash(ref_world* w) { return state_hash(w->w); }

int ref_constitutive(const msim_material* mat, int64_t n, const double* F, double* tau, double* Fp) {
  if (mat->model != MSIM_MODEL_HENCKY_VON_MISES) return MSIM_ERR_INVALID;
  const Material m{mat->density, mat->youngs, mat->poisson, mat->yield_stress};
  try {
    for (int64_t i = 0; i < n; ++i) {
      const Mat3 f = m3(F + 9 * i);
      if (tau) put(tau + 9 * i, kirchhoff_stress(f, m));
      if (Fp) put(Fp + 9 * i, von_mises_return_map(f, m));
    }
  } catch (const std::invalid_argument&) {
    return MSIM_ERR_INVALID;
  }
  return MSIM_OK;
}

int ref_sdf(const msim_shape* s, int64_t n, const double* p, double* phi, double* grad) {
  try {
    const Shape sh = shape_from(*s);
    for (int64_t i = 0; i < n; ++i) {
      const Vec3 x = v3(p + 3 * i);
      if (phi) phi[i] = sdf_eval(sh, sh.local_pose, x);
      if (grad) put(grad + 3 * i, sdf_gradient(sh, sh.local_pose, x));
    }
  } catch (const std::exception&) {
    return MSIM_ERR_INVALID;
  }
  return MSIM_OK;
}

double ref_time_env_steps(ref_world* w, int steps, int* err) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) {
    const int rc = ref_env_step(w, nullptr);
    if (rc != MSIM_OK) {
      if (err) *err = rc;
      break;
    }
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// `steps` env steps of each world, every world on its own thread (the
// aggregate mode of the reference's bench, shell.hpp:366-407). Wall seconds.
double ref_bench_worlds(ref_world** ws, int n, int steps, int* err) {
  std::vector<int> rc(n, MSIM_OK);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int i = 0; i < n; ++i)
    pool.emplace_back([&, i] {
      for (int s = 0; s < steps && rc[i] == MSIM_OK; ++s) rc[i] = ref_env_step(ws[i], nullptr);
    });
  for (auto& t : pool) t.join();
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (err) {
    *err = MSIM_OK;
    for (int r : rc)
      if (r != MSIM_OK) *err = r;
  }
  return sec;
}

// ---- seeding (the reference's seeder) --------------------------------------
struct ref_rng {
  std::mt19937_64 g;
};
ref_rng* ref_rng_create(uint64_t seed) { return new ref_rng{std::mt19937_64(seed)}; }
void ref_rng_destroy(ref_rng* r) { delete r; }
double ref_rng_uniform(ref_rng* r, double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(r->g); }
int64_t ref_seed_box(ref_world* w, ref_rng* r, const double* bmin, const double* bmax, int mat, double particle_volume) {
  const std::size_t before = w->w.soft.particles.size();
  seed_particles_box(w->w.soft, v3(bmin), v3(bmax), mat, particle_volume, r->g);
  return int64_t(w->w.soft.particles.size() - before);
}

}  // extern "C"
