// msim_gpu.hpp — header-only C++ mirror of the reference's soft-body API
// (namespace msim, mpm.hpp / coupling.hpp) on top of the C ABI in msim_gpu.h.
//
// A caller of the reference keeps its call shapes:
//   msim::SoftState st; ...; msim::soft_substep(st, hook, hook);   (mpm.hpp:397)
// becomes
//   msim_gpu::SoftState st(grid, materials); st.set_particles(...);
//   msim_gpu::soft_substep(st);                                     (hooks on device)
// Exceptions are the reference's: SimulationDiverged (mpm.hpp:18-20) for
// MSIM_ERR_DIVERGED and std::invalid_argument for MSIM_ERR_INVALID.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "msim_gpu.h"

namespace msim_gpu {

struct SimulationDiverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const msim_gpu_ctx* ctx) {
  if (rc == MSIM_OK) return;
  const std::string msg = ctx ? msim_gpu_last_error(ctx) : msim_gpu_create_error();
  if (rc == MSIM_ERR_DIVERGED) throw SimulationDiverged(msg);
  if (rc == MSIM_ERR_INVALID) throw std::invalid_argument(msg);
  throw DeviceError(msg);
}

// Particle in the reference's AoS form (mpm.hpp:50-58), row-major matrices.
struct Particle {
  double x[3] = {0, 0, 0};
  double v[3] = {0, 0, 0};
  double mass = 0.0;
  double volume0 = 6.2e-8;
  double F[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double C[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int material = 0;
};

// SoftState (mpm.hpp:111-145) for a batch of n_env independent worlds that
// share one grid description. All state lives on the device.
class SoftState {
 public:
  SoftState(const msim_soft_desc& desc, const std::vector<msim_material>& materials, int n_env = 1,
            int device = 0) {
    check(msim_gpu_create(&desc, materials.data(), (int)materials.size(), n_env, device, &ctx_), nullptr);
  }
  ~SoftState() { msim_gpu_destroy(ctx_); }
  SoftState(const SoftState&) = delete;
  SoftState& operator=(const SoftState&) = delete;

  msim_gpu_ctx* handle() const { return ctx_; }

  // particles of every env, env e owning [offsets[e], offsets[e+1])
  void set_particles(const std::vector<Particle>& ps, const std::vector<int64_t>& offsets) {
    const size_t n = ps.size();
    std::vector<double> x(3 * n), v(3 * n), F(9 * n), C(9 * n), m(n), v0(n);
    std::vector<int32_t> mat(n);
    for (size_t i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) {
        x[3 * i + k] = ps[i].x[k];
        v[3 * i + k] = ps[i].v[k];
      }
      for (int k = 0; k < 9; ++k) {
        F[9 * i + k] = ps[i].F[k];
        C[9 * i + k] = ps[i].C[k];
      }
      m[i] = ps[i].mass;
      v0[i] = ps[i].volume0;
      mat[i] = ps[i].material;
    }
    check(msim_gpu_set_particles(ctx_, (int64_t)n, offsets.data(), x.data(), v.data(), F.data(), C.data(),
                                 m.data(), v0.data(), mat.data()),
          ctx_);
  }

  std::vector<Particle> particles(int env = 0) const {
    const int64_t n = msim_gpu_particle_count(ctx_, env);
    std::vector<double> x(3 * n), v(3 * n), F(9 * n), C(9 * n);
    check(msim_gpu_read_particles(ctx_, env, x.data(), v.data(), F.data(), C.data(), nullptr), ctx_);
    std::vector<Particle> out((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
      for (int k = 0; k < 3; ++k) {
        out[i].x[k] = x[3 * i + k];
        out[i].v[k] = v[3 * i + k];
      }
      for (int k = 0; k < 9; ++k) {
        out[i].F[k] = F[9 * i + k];
        out[i].C[k] = C[9 * i + k];
      }
    }
    return out;
  }

  void set_dt(double dt) { check(msim_gpu_set_dt(ctx_, dt), ctx_); }
  std::size_t lost_count(int env = 0) const { return (std::size_t)msim_gpu_lost_count(ctx_, env); }

  // per-particle material scalar (fluid J, Drucker-Prager plastic strain, else 1)
  std::vector<double> jp(int env = 0) const {
    std::vector<double> out((size_t)msim_gpu_particle_count(ctx_, env));
    check(msim_gpu_read_jp(ctx_, env, out.data()), ctx_);
    return out;
  }

  // batched reset: seed_particles_box (seeding.hpp:13-35) on the device for the listed envs
  void seed_envs(const std::vector<int32_t>& envs, const std::vector<uint64_t>& seeds,
                 const std::vector<double>& boxes, int material, double particle_volume) {
    check(msim_gpu_seed_envs(ctx_, (int)envs.size(), envs.data(), seeds.data(), boxes.data(), material,
                             particle_volume),
          ctx_);
  }

 private:
  msim_gpu_ctx* ctx_ = nullptr;
};

// Free functions with the reference's names (mpm.hpp:199, :315, :346, :397).
inline void p2g(SoftState& st) { check(msim_gpu_p2g(st.handle()), st.handle()); }
inline void grid_update(SoftState& st) { check(msim_gpu_grid_update(st.handle()), st.handle()); }
inline void g2p_advect(SoftState& st) { check(msim_gpu_g2p(st.handle()), st.handle()); }
inline int soft_substep(SoftState& st) {
  int32_t cycles = 1;
  check(msim_gpu_soft_substep(st.handle(), 1, &cycles), st.handle());
  return cycles;
}

// The rigid/soft part of env_step (coupling.hpp:248-293) for bodies set with
// set_bodies(); the controller/robot part stays with the caller.
inline msim_step_report env_step(SoftState& st, int n_rigid = 25, int n_soft = 1) {
  msim_step_report r{};
  check(msim_gpu_env_step(st.handle(), n_rigid, n_soft, &r), st.handle());
  return r;
}

inline void set_bodies(SoftState& st, int env, const std::vector<msim_body>& bodies,
                       const std::vector<msim_shape>& shapes) {
  check(msim_gpu_set_bodies(st.handle(), env, bodies.data(), (int)bodies.size(), shapes.data(),
                            (int)shapes.size()),
        st.handle());
}

// ---- task metrics over every env (scenario.hpp:63-209) ----------------------
inline std::vector<msim_fill_result> metric_fill(SoftState& st, const std::vector<msim_region>& regions) {
  std::vector<msim_fill_result> out(regions.size());
  check(msim_gpu_metric_fill(st.handle(), regions.data(), out.data()), st.handle());
  return out;
}
inline std::vector<double> render_heightmap(SoftState& st, const std::vector<msim_region>& regions, int nx, int ny) {
  std::vector<double> maps(regions.size() * (size_t)nx * ny);
  check(msim_gpu_render_heightmap(st.handle(), regions.data(), nx, ny, maps.data()), st.handle());
  return maps;
}

// ---- mesh SDF baking (sdf.hpp:277-310) ------------------------------------
struct BakedVolume {
  double origin[3];
  int32_t dims[3];
  std::vector<float> samples;  // x fastest, ready for msim_shape.vol_samples
};
inline BakedVolume bake_mesh_sdf(const std::vector<double>& triangles, double voxel, double padding, int device = 0) {
  BakedVolume v{};
  const int64_t n = (int64_t)(triangles.size() / 9);
  check(msim_bake_grid(triangles.data(), n, voxel, padding, v.origin, v.dims), nullptr);
  v.samples.resize((size_t)v.dims[0] * v.dims[1] * v.dims[2]);
  check(msim_gpu_bake_mesh_sdf(device, triangles.data(), n, voxel, padding, v.samples.data(),
                               (int64_t)v.samples.size()),
        nullptr);
  return v;
}

// sync_rigid_to_soft (coupling.hpp:106-117) with new body states of one env.
inline void sync_rigid_to_soft(SoftState& st, int env, const std::vector<msim_body>& bodies) {
  check(msim_gpu_sync_bodies(st.handle(), env, bodies.data(), (int)bodies.size()), st.handle());
}

// Robot-driven links (coupling.hpp:252-258 -> Robot::set_kinematic_pose,
// rigid.hpp:142-151) for the next env_step: poses[r][i] = {qw, qx, qy, qz, tx, ty, tz}
// of body i (all envs concatenated) at rigid step r. One upload per env step.
struct LinkPose {
  double q[4];
  double t[3];
};
inline void set_kinematic_schedule(SoftState& st, const std::vector<std::vector<LinkPose>>& poses,
                                   const std::vector<uint8_t>* mask = nullptr) {
  std::vector<double> flat;
  for (const auto& row : poses)
    for (const LinkPose& p : row) {
      flat.insert(flat.end(), p.q, p.q + 4);
      flat.insert(flat.end(), p.t, p.t + 3);
    }
  check(msim_gpu_set_kinematic_schedule(st.handle(), (int)poses.size(), flat.data(), mask ? mask->data() : nullptr),
        st.handle());
}

// Bit-reproducible stepping (the reference's scheduling-independence, mpm.hpp:7-8).
inline void set_deterministic(SoftState& st, bool on) { check(msim_gpu_set_deterministic(st.handle(), on ? 1 : 0), st.handle()); }

}  // namespace msim_gpu
