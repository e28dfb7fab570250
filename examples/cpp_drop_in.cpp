// A reference-style C++ caller driving the B200 path through include/msim_gpu.hpp:
// the same calls a msim user makes (SoftState, seed_particles_box, soft_substep,
// env_step), with the hooks evaluated on the device. Prints one line:
//   "free_fall_err <e> cycles <c> lost <n> wrench_z <f>"
#include <cmath>
#include <cstdio>
#include <vector>

#include "msim_gpu.hpp"

int main() {
  msim_soft_desc d{};
  d.h = 0.01;
  d.dims[0] = d.dims[1] = d.dims[2] = 32;
  d.gravity[2] = -9.81;
  d.dt = 2e-4;
  d.cfl_factor = 0.4;
  d.max_cfl_halvings = 4;
  d.lost_fraction_threshold = 0.01;
  std::vector<msim_material> mats = {{1000.0, 1e4, 0.3, 2e3, 0, 0}};  // soft_clay (mpm.hpp:45)
  msim_gpu::SoftState st(d, mats);

  // seed_particles_box (seeding.hpp:13-35) with the library's seeder
  const double lo[3] = {0.10, 0.10, 0.10}, hi[3] = {0.14, 0.14, 0.13};
  msim_rng* rng = msim_rng_create(7);
  const int64_t n = msim_seed_box_count(lo, hi, 6.2e-8);
  std::vector<double> x(3 * n), m(n);
  msim_seed_box(rng, lo, hi, 1000.0, 6.2e-8, x.data(), m.data());
  msim_rng_destroy(rng);
  std::vector<msim_gpu::Particle> ps(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) ps[i].x[k] = x[3 * i + k];
    ps[i].mass = m[i];
  }
  st.set_particles(ps, {0, n});

  int cycles = 0;
  for (int s = 0; s < 20; ++s) cycles += msim_gpu::soft_substep(st);
  double vz = 0.0;
  for (const auto& p : st.particles()) vz += p.v[2];
  vz /= (double)n;
  const double err = std::fabs(vz - (-9.81 * 20 * d.dt)) / (9.81 * 20 * d.dt);

  // a plane floor body + env_step (coupling.hpp:219): wrench from the penalty hook
  msim_body floor{};
  floor.mode = MSIM_BODY_KINEMATIC;
  floor.q[0] = 1.0;
  floor.t[2] = 0.102;  // the bottom ~2 mm of the clay penetrates the floor
  msim_shape plane{};
  plane.type = MSIM_SHAPE_PLANE;
  plane.local_q[0] = 1.0;
  plane.params[2] = 1.0;
  plane.friction = 0.5;
  plane.k_n = 1e3;
  plane.k_t = 10.0;
  msim_gpu::set_bodies(st, 0, {floor}, {plane});
  msim_gpu::env_step(st, 1, 1);  // one substep: the stiff floor launches the light clay right after
  double f[3], t[3];
  msim_gpu_read_wrenches(st.handle(), 0, 1, f, t);
  std::printf("free_fall_err %.3e cycles %d lost %zu wrench_z %.6g\n", err, cycles, st.lost_count(), f[2]);

  // episode-level consumers: metric_fill (scenario.hpp:63-75) and a baked mesh SDF (sdf.hpp:277-310)
  const auto fill = msim_gpu::metric_fill(st, {msim_region{{0.0, 0.0, 0.0}, {0.32, 0.32, 0.32}}});
  std::vector<double> tri(108);
  const double half[3] = {0.02, 0.02, 0.01};
  msim_make_box_mesh(half, nullptr, tri.data());
  const auto vol = msim_gpu::bake_mesh_sdf(tri, 0.005, 0.01);
  float smin = vol.samples[0];
  for (float v : vol.samples) smin = v < smin ? v : smin;
  std::printf("fill_fraction %.6f sdf_samples %zu sdf_min %.6f\n", fill[0].fraction, vol.samples.size(), smin);

  // a robot-driven link: the floor follows a per-rigid-step pose schedule (Robot::set_kinematic_pose,
  // rigid.hpp:142-151), uploaded once for the whole env step; deterministic mode on
  msim_gpu::set_deterministic(st, true);
  const int n_rigid = 5;
  std::vector<std::vector<msim_gpu::LinkPose>> poses(n_rigid);
  for (int r = 0; r < n_rigid; ++r) poses[r] = {msim_gpu::LinkPose{{1.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.102 - 0.0005 * (r + 1)}}};
  msim_gpu::set_kinematic_schedule(st, poses);
  msim_gpu::env_step(st, n_rigid, 1);
  msim_body b{};
  msim_gpu_read_bodies(st.handle(), 0, &b, 1);
  std::printf("scheduled_link_z %.6f link_vz %.6f\n", b.t[2], b.v[2]);
  return err < 1e-3 && std::fabs(b.t[2] - (0.102 - 0.0005 * n_rigid)) < 1e-12 ? 0 : 1;
}
