// ORACLE — TEST INFRASTRUCTURE ONLY (see msim_oracle.hpp header).
// extern "C" surface of the CPU restatement, shaped like include/msim_gpu.h
// so parity tests can drive both with the same descriptors. Loaded by
// tests/ and bench.py (cpu_baseline / --impl reference) through ctypes.
#include "msim_oracle.hpp"
#include "msim_oracle_tasks.hpp"
#include "../include/msim_gpu.h"

#include <chrono>
#include <cstring>

using namespace oracle;

struct oracle_world {
  World w;
  std::string err;
};
struct oracle_rng {
  std::mt19937_64 g;
};

namespace {

V3 v3(const double* p) { return V3(p[0], p[1], p[2]); }
void put(double* dst, const V3& v) { dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; }
M3 m3(const double* p) {
  M3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m.m[r][c] = p[r * 3 + c];
  return m;
}
void put(double* dst, const M3& m) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) dst[r * 3 + c] = m.m[r][c];
}
Quat quat(const double* q) { return Quat(q[0], q[1], q[2], q[3]); }

Material material_from(const msim_material& m) {
  return Material{m.density, m.youngs, m.poisson, m.yield_stress, static_cast<Model>(m.model)};
}

Shape shape_from(const msim_shape& s) {
  Shape o;
  o.type = static_cast<ShapeType>(s.type);
  o.local_pose = Pose(quat(s.local_q), v3(s.local_t));
  o.friction = s.friction;
  o.k_n = s.k_n;
  o.k_t = s.k_t;
  switch (o.type) {
    case ShapeType::Plane: o.normal = v3(s.params); o.offset = s.params[3]; break;
    case ShapeType::Sphere: o.radius = s.params[0]; break;
    case ShapeType::Box: o.half_extents = v3(s.params); break;
    case ShapeType::Capsule: o.half_length = s.params[0]; o.radius = s.params[1]; break;
    case ShapeType::Volume: {
      auto vol = std::make_shared<SdfVolume>();
      vol->origin = v3(s.vol_origin);
      vol->voxel = s.vol_voxel;
      vol->dims = I3{s.vol_dims[0], s.vol_dims[1], s.vol_dims[2]};
      std::size_t n = std::size_t(s.vol_dims[0]) * s.vol_dims[1] * s.vol_dims[2];
      vol->samples.assign(s.vol_samples, s.vol_samples + n);
      o.volume = vol;
      break;
    }
  }
  return o;
}

void body_to(const RigidBody& b, msim_body* o) {
  o->mode = int(b.mode);
  o->q[0] = b.pose.rotation.w; o->q[1] = b.pose.rotation.x;
  o->q[2] = b.pose.rotation.y; o->q[3] = b.pose.rotation.z;
  put(o->t, b.pose.translation);
  put(o->v, b.linear_velocity);
  put(o->w, b.angular_velocity);
  o->mass = b.mass;
  put(o->inertia, b.inertia);
  put(o->com_offset, b.com_offset);
}

template <class F>
int guarded(oracle_world* w, F&& f) {
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

}  // namespace

extern "C" {

oracle_world* oracle_create(const msim_soft_desc* d, const msim_material* mats, int n_mat) {
  auto* o = new oracle_world();
  SoftState& st = o->w.soft;
  st.grid.h = d->h;
  st.grid.dims = I3{d->dims[0], d->dims[1], d->dims[2]};
  st.grid.origin = v3(d->origin);
  for (int f = 0; f < 6; ++f) st.grid.boundary[f] = static_cast<BoundaryKind>(d->boundary[f]);
  st.gravity = v3(d->gravity);
  st.dt = d->dt;
  st.cfl_factor = d->cfl_factor;
  st.max_cfl_halvings = d->max_cfl_halvings;
  st.lost_fraction_threshold = d->lost_fraction_threshold;
  for (int i = 0; i < n_mat; ++i) st.materials.push_back(material_from(mats[i]));
  return o;
}

void oracle_destroy(oracle_world* w) { delete w; }
const char* oracle_last_error(oracle_world* w) { return w->err.c_str(); }
void oracle_set_threads(int n) { worker_threads() = n; }

int oracle_set_particles(oracle_world* w, int64_t n, const double* x, const double* v,
                         const double* F, const double* C, const double* mass, const double* vol0,
                         const int32_t* mat) {
  auto& ps = w->w.soft.particles;
  ps.assign(n, Particle{});
  for (int64_t i = 0; i < n; ++i) {
    Particle& p = ps[i];
    p.x = v3(x + 3 * i);
    p.v = v ? v3(v + 3 * i) : V3();
    p.F = F ? m3(F + 9 * i) : M3::Identity();
    p.C = C ? m3(C + 9 * i) : M3::Zero();
    p.mass = mass[i];
    p.volume0 = vol0[i];
    p.material = mat ? mat[i] : 0;
    if (p.material >= 0 && p.material < (int)w->w.soft.materials.size())
      init_model_state(p, w->w.soft.materials[p.material]);
  }
  return MSIM_OK;
}

// plastic / volume scalar per particle (Fluid: J, DruckerPrager: q, else 1)
int oracle_read_jp(oracle_world* w, double* jp) {
  const auto& ps = w->w.soft.particles;
  for (size_t i = 0; i < ps.size(); ++i) jp[i] = ps[i].jp;
  return MSIM_OK;
}

int oracle_write_particles(oracle_world* w, int64_t n, const double* x, const double* v,
                           const double* F, const double* C) {
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

int oracle_set_bodies(oracle_world* w, const msim_body* bodies, int n_bodies,
                      const msim_shape* shapes, int n_shapes) {
  return guarded(w, [&] {
    auto& bs = w->w.bodies;
    bs.assign(n_bodies, RigidBody{});
    for (int i = 0; i < n_bodies; ++i) {
      const msim_body& b = bodies[i];
      RigidBody& o = bs[i];
      o.mode = static_cast<BodyMode>(b.mode);
      o.pose = Pose(quat(b.q), v3(b.t));
      o.linear_velocity = v3(b.v);
      o.angular_velocity = v3(b.w);
      o.mass = b.mass;
      o.inertia = v3(b.inertia);
      o.com_offset = v3(b.com_offset);
    }
    for (int s = 0; s < n_shapes; ++s) {
      if (shapes[s].body < 0 || shapes[s].body >= n_bodies)
        throw std::invalid_argument("shape body index out of range");
      bs[shapes[s].body].shapes.push_back(shape_from(shapes[s]));
    }
  });
}

int oracle_sync_bodies(oracle_world* w, const msim_body* bodies, int n_bodies) {
  auto& bs = w->w.bodies;
  if (int(bs.size()) != n_bodies) return MSIM_ERR_INVALID;
  for (int i = 0; i < n_bodies; ++i) {
    bs[i].pose = Pose(quat(bodies[i].q), v3(bodies[i].t));
    bs[i].linear_velocity = v3(bodies[i].v);
    bs[i].angular_velocity = v3(bodies[i].w);
  }
  w->w.sync_rigid_to_soft();
  return MSIM_OK;
}

int oracle_set_kinematic_schedule(oracle_world* w, int n_steps, const double* poses, const uint8_t* mask) {
  World& W = w->w;
  const std::size_t nb = W.bodies.size();
  W.sched_steps = n_steps;
  W.schedule.assign(poses, poses + 7 * nb * std::size_t(n_steps));
  W.sched_mask.assign(nb, 0);
  for (std::size_t i = 0; i < nb; ++i) W.sched_mask[i] = mask ? mask[i] : (W.bodies[i].mode == BodyMode::Kinematic);
  return MSIM_OK;
}

int oracle_set_coupling(oracle_world* w, const msim_coupling* c) {
  w->w.coupling.mode = static_cast<CouplingMode>(c->mode);
  w->w.coupling.r_c_factor = c->r_c_factor;
  w->w.coupling.c_d = c->c_d;
  return MSIM_OK;
}

int oracle_set_stepping(oracle_world* w, int n_rigid, int n_soft, const double* rigid_gravity) {
  w->w.n_rigid = n_rigid;
  w->w.n_soft = n_soft;
  if (rigid_gravity) w->w.rigid_gravity = v3(rigid_gravity);
  return MSIM_OK;
}

int oracle_set_dt(oracle_world* w, double dt) { w->w.soft.dt = dt; return MSIM_OK; }
int oracle_set_gravity(oracle_world* w, const double* g) { w->w.soft.gravity = v3(g); return MSIM_OK; }
int oracle_set_lost_fraction_threshold(oracle_world* w, double t) {
  w->w.soft.lost_fraction_threshold = t;
  return MSIM_OK;
}

int oracle_init(oracle_world* w) { return guarded(w, [&] { w->w.init(); }); }
int oracle_init_buffers(oracle_world* w) { return guarded(w, [&] { w->w.soft.init_buffers(); }); }

int oracle_env_step(oracle_world* w, msim_step_report* rep) {
  return guarded(w, [&] {
    StepReport r = env_step(w->w);
    if (rep) {
      rep->rigid_steps = r.rigid_steps;
      rep->soft_substeps = r.soft_substeps;
      rep->cfl_cycles = r.cfl_cycles;
      rep->max_penetration = r.max_penetration;
      rep->max_force_balance_error = r.max_force_balance_error;
      rep->lost_particles = int64_t(r.lost_particles);
    }
  });
}

// soft_substep with the penalty hook of the configured coupling mode (the
// hooks env_step installs, coupling.hpp:266-284, without the diagnostics).
int oracle_soft_substep(oracle_world* w, int n, int use_hooks, int32_t* cycles) {
  return guarded(w, [&] {
    World& W = w->w;
    ParticleForceHook ph = nullptr;
    GridForceHook gh = nullptr;
    if (use_hooks) {
      ph = [&W](SoftState&) {
        if (W.coupling.mode == CouplingMode::Particle) penalty_particle(W);
      };
      gh = [&W](SoftState&) {
        if (W.coupling.mode == CouplingMode::Grid) penalty_grid(W);
      };
    }
    for (int i = 0; i < n; ++i) {
      int c = soft_substep(W.soft, ph, gh);
      if (cycles) *cycles = c;
    }
  });
}

int oracle_p2g(oracle_world* w) { return guarded(w, [&] { p2g(w->w.soft); }); }
int oracle_grid_update(oracle_world* w) { return guarded(w, [&] { grid_update(w->w.soft); }); }
int oracle_g2p(oracle_world* w) { return guarded(w, [&] { g2p_advect(w->w.soft); }); }
int oracle_grid_clear(oracle_world* w) { w->w.soft.grid.clear(); return MSIM_OK; }
int oracle_penalty_particle(oracle_world* w, double* max_pen) {
  return guarded(w, [&] { penalty_particle(w->w, max_pen); });
}
int oracle_penalty_grid(oracle_world* w, double* max_pen) {
  return guarded(w, [&] { penalty_grid(w->w, max_pen); });
}

int64_t oracle_particle_count(oracle_world* w) { return int64_t(w->w.soft.particles.size()); }

int oracle_read_particles(oracle_world* w, double* x, double* v, double* F, double* C,
                          uint8_t* lost) {
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

int oracle_read_ext_force(oracle_world* w, double* f) {
  const auto& ef = w->w.soft.ext_force;
  for (std::size_t i = 0; i < ef.size(); ++i) put(f + 3 * i, ef[i]);
  return MSIM_OK;
}

int oracle_read_grid(oracle_world* w, double* mass, double* momentum, double* force,
                     double* velocity) {
  const MpmGrid& g = w->w.soft.grid;
  for (std::size_t i = 0; i < g.node_count(); ++i) {
    if (mass) mass[i] = g.mass[i];
    if (momentum) put(momentum + 3 * i, g.momentum[i]);
    if (force) put(force + 3 * i, g.force[i]);
    if (velocity) put(velocity + 3 * i, g.velocity[i]);
  }
  return MSIM_OK;
}

int oracle_write_grid_velocity(oracle_world* w, const double* v) {
  MpmGrid& g = w->w.soft.grid;
  for (std::size_t i = 0; i < g.node_count(); ++i) g.velocity[i] = v3(v + 3 * i);
  return MSIM_OK;
}

int oracle_read_binning(oracle_world* w, int32_t* base, int32_t* cell_start, int64_t cs_cap,
                        int32_t* cell_particles, int64_t cp_cap, int64_t* n_alive,
                        int64_t* active, int64_t a_cap, int64_t* n_active) {
  const auto& sc = w->w.soft.scratch;
  if (base)
    for (std::size_t i = 0; i < sc.base.size(); ++i) {
      base[3 * i] = sc.base[i].x;
      base[3 * i + 1] = sc.base[i].y;
      base[3 * i + 2] = sc.base[i].z;
    }
  if (int64_t(sc.cell_start.size()) > cs_cap || int64_t(sc.cell_particles.size()) > cp_cap ||
      int64_t(sc.active_nodes.size()) > a_cap)
    return MSIM_ERR_INVALID;
  if (cell_start) std::memcpy(cell_start, sc.cell_start.data(), sc.cell_start.size() * 4);
  if (cell_particles)
    std::memcpy(cell_particles, sc.cell_particles.data(), sc.cell_particles.size() * 4);
  *n_alive = int64_t(sc.cell_particles.size());
  if (active)
    for (std::size_t i = 0; i < sc.active_nodes.size(); ++i) active[i] = int64_t(sc.active_nodes[i]);
  *n_active = int64_t(sc.active_nodes.size());
  return MSIM_OK;
}

int oracle_read_wrenches(oracle_world* w, int pending, double* force, double* torque) {
  const auto& ws = pending ? w->w.pending_wrenches : w->w.wrenches;
  for (std::size_t i = 0; i < ws.size(); ++i) {
    put(force + 3 * i, ws[i].force);
    put(torque + 3 * i, ws[i].torque);
  }
  return MSIM_OK;
}

int oracle_read_bodies(oracle_world* w, msim_body* out, int n) {
  for (int i = 0; i < n && i < int(w->w.bodies.size()); ++i) body_to(w->w.bodies[i], out + i);
  return MSIM_OK;
}

int64_t oracle_lost_count(oracle_world* w) { return int64_t(w->w.soft.lost_count); }
double oracle_time(oracle_world* w) { return w->w.time; }
double oracle_mean_particle_mass(oracle_world* w) { return w->w.mean_particle_mass; }

int oracle_constitutive(const msim_material* mat, int64_t n, const double* F, double* tau,
                        double* Fp) {
  try {
    Material m = material_from(*mat);
    for (int64_t i = 0; i < n; ++i) {
      Particle p;
      p.F = m3(F + 9 * i);
      if (!(p.F.determinant() > 0.0)) throw std::invalid_argument("kirchhoff_stress: det(F) must be > 0");
      init_model_state(p, m);
      if (tau) put(tau + 9 * i, kirchhoff_of(p, m));
      if (Fp) {
        M3 fp = p.F;
        if (m.model == Model::HenckyVonMises) fp = von_mises_return_map(p.F, m);
        else if (m.model == Model::DruckerPrager) fp = drucker_prager_return_map(p.F, m, p.jp);
        put(Fp + 9 * i, fp);
      }
    }
  } catch (const std::invalid_argument&) {
    return MSIM_ERR_INVALID;
  }
  return MSIM_OK;
}

// Shape SDF queries in world frame at the shape's local pose (sdf.hpp:190-201).
int oracle_sdf(const msim_shape* s, int64_t n, const double* p, double* phi, double* grad) {
  Shape sh = shape_from(*s);
  for (int64_t i = 0; i < n; ++i) {
    V3 x = v3(p + 3 * i);
    if (phi) phi[i] = sdf_eval(sh, x);
    if (grad) put(grad + 3 * i, sdf_gradient(sh, x));
  }
  return MSIM_OK;
}

uint64_t oracle_state_hash(oracle_world* w) {  // coupling.hpp:314-337 (particles + bodies + time)
  std::uint64_t h = 1469598103934665603ull;
  auto hv = [&](const V3& v) {
    double d[3] = {v.x, v.y, v.z};
    h = fnv1a(d, sizeof d, h);
  };
  auto hm = [&](const M3& m) {  // Eigen column-major data() order
    double d[9];
    for (int c = 0; c < 3; ++c)
      for (int r = 0; r < 3; ++r) d[c * 3 + r] = m.m[r][c];
    h = fnv1a(d, sizeof d, h);
  };
  for (const Particle& p : w->w.soft.particles) {
    hv(p.x);
    hv(p.v);
    hm(p.F);
    hm(p.C);
  }
  for (const RigidBody& b : w->w.bodies) {
    double q[4] = {b.pose.rotation.w, b.pose.rotation.x, b.pose.rotation.y, b.pose.rotation.z};
    h = fnv1a(q, sizeof q, h);
    hv(b.pose.translation);
    hv(b.linear_velocity);
    hv(b.angular_velocity);
  }
  h = fnv1a(&w->w.time, sizeof(double), h);
  return h;
}

// ---- seeding (seeding.hpp:13-46) ------------------------------------------
oracle_rng* oracle_rng_create(uint64_t seed) { return new oracle_rng{std::mt19937_64(seed)}; }
void oracle_rng_destroy(oracle_rng* r) { delete r; }
double oracle_rng_uniform(oracle_rng* r, double lo, double hi) {
  return std::uniform_real_distribution<double>(lo, hi)(r->g);
}
// Appends particles of material `mat` to the world.
int64_t oracle_seed_box(oracle_world* w, oracle_rng* r, const double* bmin, const double* bmax,
                        int mat, double particle_volume) {
  std::size_t before = w->w.soft.particles.size();
  seed_particles_box(w->w.soft, v3(bmin), v3(bmax), mat, particle_volume, r->g);
  return int64_t(w->w.soft.particles.size() - before);
}
int64_t oracle_lattice_count(const double* bmin, const double* bmax, double particle_volume) {
  return int64_t(lattice_count(v3(bmin), v3(bmax), particle_volume));
}

// ---- timing helper for the CPU baseline ------------------------------------
double oracle_time_env_steps(oracle_world* w, int steps, int* err) {
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) {
    int rc = oracle_env_step(w, nullptr);
    if (rc != MSIM_OK) {
      if (err) *err = rc;
      break;
    }
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- mesh baking and task metrics (msim_oracle_tasks.hpp) -----------------
namespace {
TriangleMesh mesh_from(const double* tri, int64_t n) {
  TriangleMesh m((size_t)n);
  for (int64_t t = 0; t < n; ++t) m[t] = {v3(tri + 9 * t), v3(tri + 9 * t + 3), v3(tri + 9 * t + 6)};
  return m;
}
std::vector<V3> pts_from(const double* p, int64_t n) {
  std::vector<V3> v((size_t)n);
  for (int64_t i = 0; i < n; ++i) v[i] = v3(p + 3 * i);
  return v;
}
RegionBox region_from(const double* r) {
  RegionBox b;
  b.min = v3(r);
  b.max = v3(r + 3);
  return b;
}
}  // namespace

int oracle_bake_grid(const double* tri, int64_t n, double voxel, double padding, double* origin, int32_t* dims) {
  return guarded(nullptr, [&] {
    V3 o;
    int d[3];
    bake_grid(mesh_from(tri, n), voxel, padding, o, d);
    put(origin, o);
    for (int k = 0; k < 3; ++k) dims[k] = d[k];
  });
}
int oracle_bake_mesh_sdf(const double* tri, int64_t n, double voxel, double padding, float* samples, int64_t cap) {
  return guarded(nullptr, [&] {
    SdfVolume v = bake_mesh_sdf(mesh_from(tri, n), voxel, padding);
    if ((int64_t)v.samples.size() > cap) throw std::invalid_argument("bake_mesh_sdf: samples capacity");
    std::memcpy(samples, v.samples.data(), v.samples.size() * sizeof(float));
  });
}
void oracle_make_box_mesh(const double* half, const double* center, double* tri) {
  TriangleMesh m = make_box_mesh(v3(half), center ? v3(center) : V3::Zero());
  for (size_t t = 0; t < m.size(); ++t) {
    put(tri + 9 * t, m[t].a);
    put(tri + 9 * t + 3, m[t].b);
    put(tri + 9 * t + 6, m[t].c);
  }
}
int oracle_metric_fill(int64_t n, const double* x, const double* v, const double* region, double* fraction,
                       double* max_speed, int32_t* success) {
  return guarded(nullptr, [&] {
    FillResult r = metric_fill(pts_from(x, n), pts_from(v, n), region_from(region));
    *fraction = r.fraction;
    *max_speed = r.max_speed;
    *success = r.success;
  });
}
int oracle_render_heightmap(int64_t n, const double* x, const double* region, int nx, int ny, double* out) {
  return guarded(nullptr, [&] {
    DepthMap m = render_heightmap(pts_from(x, n), region_from(region), nx, ny);
    std::memcpy(out, m.samples.data(), m.samples.size() * sizeof(double));
  });
}
int oracle_metric_write_iou(int nx, int ny, double threshold, const double* a, const double* b, double* iou,
                            int32_t* success) {
  return guarded(nullptr, [&] {
    DepthMap ma, mb;
    ma.nx = mb.nx = nx;
    ma.ny = mb.ny = ny;
    ma.threshold = mb.threshold = threshold;
    ma.samples.assign(a, a + (size_t)nx * ny);
    mb.samples.assign(b, b + (size_t)nx * ny);
    IouResult r = metric_write_iou(ma, mb);
    *iou = r.iou;
    *success = r.success;
  });
}
int oracle_chamfer(int64_t na, const double* a, int64_t nb, const double* b, double* out) {
  return guarded(nullptr, [&] { *out = chamfer_distance(pts_from(a, na), pts_from(b, nb)); });
}
int oracle_metric_pinch(int64_t nc, const double* cur, int64_t ni, const double* init, int64_t nt,
                        const double* tgt, double* ratio, int32_t* success) {
  return guarded(nullptr, [&] {
    PinchResult r = metric_pinch(pts_from(cur, nc), pts_from(init, ni), pts_from(tgt, nt));
    *ratio = r.ratio;
    *success = r.success;
  });
}

}  // extern "C"

