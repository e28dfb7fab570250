// ORACLE — TEST INFRASTRUCTURE ONLY.
// Ports of the reference's own known-answer tests for the hot path, run
// against the CPU restatement to pin it (the reference ships no golden
// vectors and cannot be built here). Each TEST cites the
// reference test it ports. Output: one "PASS name" / "FAIL name: msg" line
// per test, exit code = number of failures.
#include "msim_oracle.hpp"
#include "msim_oracle_tasks.hpp"

#include <cstdio>
#include <sstream>

using namespace oracle;

namespace {

int g_fail = 0, g_pass = 0;
std::string g_cur;
bool g_cur_failed = false;

#define EXPECT(cond)                                                          \
  do {                                                                        \
    if (!(cond)) {                                                            \
      std::printf("  %s:%d: expected %s\n", __FILE__, __LINE__, #cond);       \
      g_cur_failed = true;                                                    \
    }                                                                         \
  } while (0)
#define EXPECT_NEAR(a, b, tol)                                                \
  do {                                                                        \
    double _a = (a), _b = (b), _t = (tol);                                    \
    if (!(std::abs(_a - _b) <= _t)) {                                         \
      std::printf("  %s:%d: |%s - %s| = %.3e > %.3e\n", __FILE__, __LINE__,   \
                  #a, #b, std::abs(_a - _b), _t);                             \
      g_cur_failed = true;                                                    \
    }                                                                         \
  } while (0)
#define EXPECT_THROW(stmt, T)                                                 \
  do {                                                                        \
    bool _thrown = false;                                                     \
    try {                                                                     \
      stmt;                                                                   \
    } catch (const T&) {                                                      \
      _thrown = true;                                                         \
    }                                                                         \
    if (!_thrown) {                                                           \
      std::printf("  %s:%d: %s did not throw\n", __FILE__, __LINE__, #stmt);  \
      g_cur_failed = true;                                                    \
    }                                                                         \
  } while (0)

struct Reg {
  const char* name;
  void (*fn)();
};
std::vector<Reg>& registry() {
  static std::vector<Reg> r;
  return r;
}
struct Adder {
  Adder(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
#define TEST(suite, name)                                        \
  void suite##_##name();                                         \
  Adder add_##suite##_##name(#suite "." #name, suite##_##name);  \
  void suite##_##name()

// test_util.hpp:9-29. Argument evaluation order of Vec3(u(), u(), u()) and
// Quat(n(), n(), n(), n()) follows GCC (right to left).
std::mt19937_64 rng(std::uint64_t seed = 42) { return std::mt19937_64(seed); }
double uniform(std::mt19937_64& g, double lo, double hi) {
  return std::uniform_real_distribution<double>(lo, hi)(g);
}
V3 random_vec3(std::mt19937_64& g, double lo = -1.0, double hi = 1.0) {
  double z = uniform(g, lo, hi), y = uniform(g, lo, hi), x = uniform(g, lo, hi);
  return V3(x, y, z);
}
Quat random_quat(std::mt19937_64& g) {
  std::normal_distribution<double> n(0.0, 1.0);
  double z = n(g), y = n(g), x = n(g), w = n(g);
  Quat q(w, x, y, z);
  q.normalize();
  if (q.w < 0.0) q = Quat(-q.w, -q.x, -q.y, -q.z);
  return q;
}
Pose random_pose(std::mt19937_64& g, double span = 1.0) {
  V3 t = random_vec3(g, -span, span);  // Pose(random_quat(g), random_vec3(g)): right to left
  Quat q = random_quat(g);
  return Pose(q, t);
}

// ---- test_mpm.cpp fixtures (:13-60) ----------------------------------------
double bspline(double x) {
  double a = std::abs(x);
  if (a < 0.5) return 0.75 - a * a;
  if (a < 1.5) return 0.5 * (1.5 - a) * (1.5 - a);
  return 0.0;
}
SoftState make_state(int dims = 32, double h = 0.01) {
  SoftState st;
  st.grid.h = h;
  st.grid.dims = I3{dims, dims, dims};
  st.grid.origin = V3();
  st.materials = {soft_clay(), stiff_clay()};
  st.gravity = V3();
  st.dt = 1e-4;
  return st;
}
void add_particle(SoftState& st, const V3& x, const V3& v = V3(), double mass = 1e-4, int mat = 0) {
  Particle p;
  p.x = x;
  p.v = v;
  p.mass = mass;
  p.volume0 = kSoftClayParticleVolume;
  p.material = mat;
  st.particles.push_back(p);
}
void seed_random_cloud(SoftState& st, int n, std::mt19937_64& g) {
  double lo = 4 * st.grid.h, hi = (st.grid.dims.x - 5) * st.grid.h;
  for (int i = 0; i < n; ++i) {
    // add_particle(st, random_vec3(pos), random_vec3(vel), uniform(mass)): right to left
    double m = uniform(g, 1e-5, 1e-3);
    V3 v = random_vec3(g, -0.5, 0.5);
    V3 x = random_vec3(g, lo, hi);
    add_particle(st, x, v, m);
  }
}
double total_grid_mass(const SoftState& st) {
  double m = 0;
  for (double v : st.grid.mass) m += v;
  return m;
}
V3 total_grid_momentum(const SoftState& st) {
  V3 p;
  for (const V3& v : st.grid.momentum) p += v;
  return p;
}

}  // namespace

// ---- test_mpm.cpp ----------------------------------------------------------
TEST(P2g, RestMassAndMomentum) {  // test_mpm.cpp:64-75
  SoftState st = make_state();
  auto g = rng(20);
  seed_random_cloud(st, 500, g);
  for (Particle& p : st.particles) p.v = V3();
  st.init_buffers();
  p2g(st);
  double mp = 0;
  for (const Particle& p : st.particles) mp += p.mass;
  EXPECT_NEAR(total_grid_mass(st), mp, 1e-12 * mp);
  EXPECT(total_grid_momentum(st).norm() < 1e-14);
}

TEST(P2g, SingleParticleOnNodeMomentum) {  // :77-85
  SoftState st = make_state();
  V3 node = st.grid.node_pos(10, 10, 10);
  add_particle(st, node, V3(1, 0, 0), 2e-4);
  st.init_buffers();
  p2g(st);
  V3 mom = total_grid_momentum(st);
  EXPECT((mom - V3(2e-4, 0, 0)).norm() < 1e-16);
}

TEST(P2g, WeightsMatchBsplineOracle) {  // :87-101
  SoftState st = make_state();
  double h = st.grid.h;
  V3 node = st.grid.node_pos(12, 12, 12);
  V3 off(0.3 * h, 0.12 * h, -0.2 * h);
  add_particle(st, node + off, V3(), 1e-4);
  add_particle(st, node - off, V3(), 1e-4);
  st.init_buffers();
  p2g(st);
  std::size_t ni = st.grid.node_index(12, 12, 12);
  double w_oracle = 1.0;
  for (int ax = 0; ax < 3; ++ax) w_oracle *= bspline(off[ax] / h);
  EXPECT_NEAR(st.grid.mass[ni], 2 * 1e-4 * w_oracle, 1e-15);
}

TEST(P2g, PartitionOfUnity) {  // :103-122
  SoftState st = make_state();
  auto g = rng(21);
  seed_random_cloud(st, 200, g);
  st.init_buffers();
  p2g(st);
  double mp = 0;
  for (const Particle& p : st.particles) mp += p.mass;
  EXPECT_NEAR(total_grid_mass(st), mp, 1e-12 * mp);
  for (int ip = 0; ip < 10; ++ip) {
    const auto& w = st.scratch.w[ip];
    double sum = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        for (int c = 0; c < 3; ++c) sum += w[0][a] * w[1][b] * w[2][c];
    EXPECT_NEAR(sum, 1.0, 1e-12);
  }
}

TEST(P2g, MomentumConservation) {  // :124-133
  SoftState st = make_state(48);
  auto g = rng(22);
  seed_random_cloud(st, 1000, g);
  st.init_buffers();
  V3 pp;
  for (const Particle& p : st.particles) pp += p.mass * p.v;
  p2g(st);
  EXPECT((total_grid_momentum(st) - pp).norm() < 1e-10 * pp.norm());
}

TEST(P2g, LostParticleFlagged) {  // :135-145
  SoftState st = make_state();
  st.lost_fraction_threshold = 1.0;
  add_particle(st, V3(-1, 0, 0));
  add_particle(st, st.grid.node_pos(10, 10, 10));
  st.init_buffers();
  p2g(st);
  EXPECT(st.lost_count == 1u);
  EXPECT(st.lost[0]);
  EXPECT(!st.lost[1]);
}

TEST(P2g, LostFractionThresholdThrows) {  // :147-154
  SoftState st = make_state();
  st.lost_fraction_threshold = 0.01;
  add_particle(st, V3(-1, 0, 0));
  add_particle(st, st.grid.node_pos(10, 10, 10));
  st.init_buffers();
  EXPECT_THROW(p2g(st), SimulationDiverged);
}

TEST(GridUpdate, ZeroMassNodeStaysZero) {  // :156-163
  SoftState st = make_state();
  add_particle(st, st.grid.node_pos(10, 10, 10));
  st.init_buffers();
  p2g(st);
  grid_update(st);
  EXPECT(st.grid.velocity[st.grid.node_index(20, 20, 20)].norm() < 1e-300);
}

TEST(GridUpdate, AnalyticIntegration) {  // :165-178
  SoftState st = make_state();
  st.gravity = V3(0, 0, -9.81);
  st.dt = 2e-4;
  V3 node = st.grid.node_pos(10, 10, 10);
  add_particle(st, node, V3(0.3, 0, 0), 5e-4);
  st.init_buffers();
  p2g(st);
  grid_update(st);
  std::size_t ni = st.grid.node_index(10, 10, 10);
  V3 oracle_v = st.grid.momentum[ni] / st.grid.mass[ni] + st.gravity * st.dt;
  EXPECT((st.grid.velocity[ni] - oracle_v).norm() < 1e-15);
}

TEST(GridUpdate, StickyFloorZeroesVelocity) {  // :180-188
  SoftState st = make_state();
  st.grid.boundary[4] = BoundaryKind::Sticky;
  add_particle(st, st.grid.node_pos(10, 10, 1), V3(0, 0, -1.0), 1e-4);
  st.init_buffers();
  p2g(st);
  grid_update(st);
  EXPECT(st.grid.velocity[st.grid.node_index(10, 10, 1)].norm() < 1e-300);
}

TEST(GridUpdate, SlipFloorKeepsTangential) {  // :190-200
  SoftState st = make_state();
  st.grid.boundary[4] = BoundaryKind::Slip;
  add_particle(st, st.grid.node_pos(10, 10, 1), V3(0.7, 0, -1.0), 1e-4);
  st.init_buffers();
  p2g(st);
  grid_update(st);
  V3 v = st.grid.velocity[st.grid.node_index(10, 10, 1)];
  EXPECT(v.x > 0.0);
  EXPECT(v.z == 0.0);
}

TEST(G2p, UniformFieldReproduced) {  // :202-218
  SoftState st = make_state();
  auto g = rng(23);
  seed_random_cloud(st, 100, g);
  st.init_buffers();
  p2g(st);
  V3 v0(0.3, -0.2, 0.15);
  for (auto& v : st.grid.velocity) v = v0;
  double dt = st.dt;
  st.dt = 0.0;
  g2p_advect(st);
  st.dt = dt;
  for (const Particle& p : st.particles) {
    EXPECT((p.v - v0).norm() < 1e-12);
    EXPECT(p.C.norm() < 1e-10);
  }
}

TEST(G2p, LinearFieldRecoversGradient) {  // :220-239
  SoftState st = make_state(48);
  auto g = rng(24);
  double lo = 8 * st.grid.h, hi = (st.grid.dims.x - 9) * st.grid.h;
  for (int i = 0; i < 100; ++i) add_particle(st, random_vec3(g, lo, hi));
  st.init_buffers();
  p2g(st);
  M3 a;
  double av[9] = {0.1, 0.3, -0.2, 0.0, -0.1, 0.25, 0.4, 0.05, 0.2};
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) a.m[r][c] = av[r * 3 + c];
  for (int k = 0; k < st.grid.dims.z; ++k)
    for (int j = 0; j < st.grid.dims.y; ++j)
      for (int i = 0; i < st.grid.dims.x; ++i)
        st.grid.velocity[st.grid.node_index(i, j, k)] = a * st.grid.node_pos(i, j, k);
  double dt = st.dt;
  st.dt = 0.0;
  g2p_advect(st);
  st.dt = dt;
  for (const Particle& p : st.particles) EXPECT((p.C - a).norm() < 1e-8);
}

TEST(G2p, ZeroDtLeavesPositionsAndF) {  // :241-256
  SoftState st = make_state();
  auto g = rng(25);
  seed_random_cloud(st, 50, g);
  st.init_buffers();
  std::vector<V3> x0;
  for (const Particle& p : st.particles) x0.push_back(p.x);
  p2g(st);
  grid_update(st);
  st.dt = 0.0;
  g2p_advect(st);
  for (std::size_t i = 0; i < st.particles.size(); ++i) {
    EXPECT((st.particles[i].x - x0[i]).norm() == 0.0);
    EXPECT((st.particles[i].F - M3::Identity()).norm() == 0.0);
  }
}

TEST(Stress, IdentityAndRotationGiveZero) {  // :258-264
  Material m = soft_clay();
  EXPECT(kirchhoff_stress(M3::Identity(), m).norm() < 1e-12);
  auto g = rng(26);
  M3 r = random_quat(g).toRotationMatrix();
  EXPECT(kirchhoff_stress(r, m).norm() < 1e-9);
}

TEST(Stress, SmallStrainMatchesLinearElasticity) {  // :266-276
  Material m;
  m.youngs = 1e4;
  m.poisson = 0.3;
  double e = 1e-3;
  M3 f = M3::Identity();
  f.m[0][0] = 1.0 + e;
  M3 tau = kirchhoff_stress(f, m);
  double o = (2.0 * m.mu() + m.lambda()) * e;
  EXPECT_NEAR(tau.m[0][0], o, 0.01 * std::abs(o));
}

TEST(Stress, NonInvertibleThrows) {  // :278-282
  M3 f = M3::Identity();
  f.m[2][2] = 0.0;
  EXPECT_THROW(kirchhoff_stress(f, soft_clay()), std::invalid_argument);
}

TEST(ReturnMap, InsideYieldUnchanged) {  // :284-290
  Material m = soft_clay();
  m.yield_stress = 1e4;
  M3 f = M3::Identity();
  f.m[0][1] = 1e-4;
  EXPECT((von_mises_return_map(f, m) - f).norm() == 0.0);
}

TEST(ReturnMap, PureDilationUnchanged) {  // :292-299
  for (double sy : {2e3, 1e4}) {
    Material m = soft_clay();
    m.yield_stress = sy;
    M3 f = 1.3 * M3::Identity();
    EXPECT((von_mises_return_map(f, m) - f).norm() == 0.0);
  }
}

TEST(ReturnMap, ProjectsOntoYieldSurface) {  // :301-328 (Mat3::Random -> U(-1,1) entries)
  auto g = rng(27);
  for (double sy : {2e3, 1e4}) {
    Material m = soft_clay();
    m.yield_stress = sy;
    for (int i = 0; i < 200; ++i) {
      M3 rnd;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) rnd.m[r][c] = uniform(g, -1.0, 1.0);
      M3 f = M3::Identity() + 0.2 * rnd;
      if (f.determinant() <= 0.1) continue;
      M3 fp = von_mises_return_map(f, m);
      M3 tau = kirchhoff_stress(fp, m);
      M3 dev = tau - (tau.trace() / 3.0) * M3::Identity();
      double threshold = std::sqrt(2.0 / 3.0) * sy;
      M3 tau_trial = kirchhoff_stress(f, m);
      M3 dev_trial = tau_trial - (tau_trial.trace() / 3.0) * M3::Identity();
      if (dev_trial.norm() > threshold) EXPECT_NEAR(dev.norm(), threshold, 1e-6 * threshold);
      EXPECT(dev.norm() <= dev_trial.norm() * (1 + 1e-12));
      EXPECT_NEAR(fp.determinant(), f.determinant(), 1e-9 * std::abs(f.determinant()));
    }
  }
}

TEST(Substep, FreeFallOracle) {  // :330-340
  SoftState st = make_state();
  st.gravity = V3(0, 0, -9.81);
  st.dt = 1e-4;
  add_particle(st, st.grid.node_pos(16, 16, 24));
  st.init_buffers();
  int n = 50;
  for (int i = 0; i < n; ++i) soft_substep(st);
  V3 o = st.gravity * (n * st.dt);
  EXPECT((st.particles[0].v - o).norm() < 1e-10);
}

TEST(Substep, RestStateUnchangedWithoutGravity) {  // :342-355
  SoftState st = make_state();
  auto g = rng(28);
  double lo = 6 * st.grid.h, hi = (st.grid.dims.x - 7) * st.grid.h;
  for (int i = 0; i < 100; ++i) add_particle(st, random_vec3(g, lo, hi));
  st.init_buffers();
  std::vector<V3> x0;
  for (const Particle& p : st.particles) x0.push_back(p.x);
  for (int i = 0; i < 5; ++i) soft_substep(st);
  for (std::size_t i = 0; i < st.particles.size(); ++i) {
    EXPECT((st.particles[i].x - x0[i]).norm() < 1e-12);
    EXPECT(st.particles[i].v.norm() < 1e-12);
  }
}

TEST(Substep, FullCycleMomentumConservation) {  // :357-378
  SoftState st = make_state(48);
  auto g = rng(29);
  double lo = 10 * st.grid.h, hi = (st.grid.dims.x - 11) * st.grid.h;
  for (int i = 0; i < 500; ++i) {
    Particle p;
    p.x = random_vec3(g, lo, hi);
    p.v = random_vec3(g, -0.1, 0.1);
    p.mass = uniform(g, 1e-5, 1e-4);
    st.particles.push_back(p);
  }
  st.init_buffers();
  V3 before;
  for (const Particle& p : st.particles) before += p.mass * p.v;
  st.dt = 1e-8;
  soft_substep(st);
  V3 after;
  for (const Particle& p : st.particles) after += p.mass * p.v;
  EXPECT((after - before).norm() < 1e-8 * before.norm());
}

TEST(Substep, CflHalvesInternally) {  // :380-387
  SoftState st = make_state();
  add_particle(st, st.grid.node_pos(16, 16, 16), V3(10.0, 0, 0));
  st.init_buffers();
  st.dt = 1e-3;
  int cycles = soft_substep(st);
  EXPECT(cycles >= 2);
}

TEST(Substep, CflErrorAfterMaxHalvings) {  // :389-395
  SoftState st = make_state();
  add_particle(st, st.grid.node_pos(16, 16, 16), V3(500.0, 0, 0));
  st.init_buffers();
  st.dt = 1e-3;
  EXPECT_THROW(soft_substep(st), SimulationDiverged);
}

TEST(Substep, DeterministicAcrossThreadCounts) {  // :397-418
  auto run = [](int threads) {
    worker_threads() = threads;
    SoftState st = make_state();
    st.gravity = V3(0, 0, -9.81);
    std::mt19937_64 g(7);
    st.materials = {soft_clay()};
    seed_particles_box(st, V3(0.1, 0.1, 0.05), V3(0.16, 0.16, 0.11), 0, kStiffClayParticleVolume, g);
    st.init_buffers();
    for (int i = 0; i < 20; ++i) soft_substep(st);
    worker_threads() = 1;
    return st;
  };
  SoftState a = run(1), b = run(3), c = run(8);
  EXPECT(a.particles.size() == b.particles.size());
  for (std::size_t i = 0; i < a.particles.size(); ++i) {
    EXPECT((a.particles[i].x - b.particles[i].x).norm() == 0.0);
    EXPECT((a.particles[i].x - c.particles[i].x).norm() == 0.0);
    EXPECT((a.particles[i].F - b.particles[i].F).norm() == 0.0);
  }
}

TEST(Material, Table5RangeValidation) {  // :420-428
  Material m = soft_clay();
  m.validate();
  m.poisson = 0.5;
  EXPECT_THROW(m.validate(), std::invalid_argument);
  Material bad = stiff_clay();
  bad.youngs = -1;
  EXPECT_THROW(bad.validate(), std::invalid_argument);
}

// ---- test_sdf.cpp (eval / gradient) -----------------------------------------
namespace {
Shape mk(ShapeType t) {
  Shape s;
  s.type = t;
  return s;
}
std::vector<Shape> analytic_zoo() {  // test_sdf.cpp:32-39
  std::vector<Shape> z;
  Shape pl = mk(ShapeType::Plane);
  pl.normal = V3(0, 0, 1);
  pl.offset = 0.0;
  z.push_back(pl);
  Shape sp = mk(ShapeType::Sphere);
  sp.radius = 0.13;
  z.push_back(sp);
  Shape bx = mk(ShapeType::Box);
  bx.half_extents = V3(0.1, 0.2, 0.3);
  z.push_back(bx);
  Shape cp = mk(ShapeType::Capsule);
  cp.half_length = 0.15;
  cp.radius = 0.05;
  z.push_back(cp);
  return z;
}
V3 fd_gradient(const Shape& s, const V3& p) {  // test_sdf.cpp:20-29
  double h = 1e-5;
  V3 g;
  for (int k = 0; k < 3; ++k) {
    V3 dp;
    dp[k] = h;
    g[k] = (sdf_eval(s, p + dp) - sdf_eval(s, p - dp)) / (2 * h);
  }
  return g;
}
}  // namespace

TEST(SdfEval, SphereTrivial) {  // test_sdf.cpp:43-47
  Shape s = mk(ShapeType::Sphere);
  s.radius = 0.1;
  EXPECT_NEAR(sdf_eval(s, V3(0.2, 0, 0)), 0.1, 1e-15);
  EXPECT_NEAR(sdf_eval(s, V3(0, 0.05, 0)), -0.05, 1e-15);
}
TEST(SdfEval, BoxCenterNearestFace) {  // :49-52
  Shape s = mk(ShapeType::Box);
  s.half_extents = V3(0.1, 0.2, 0.3);
  EXPECT_NEAR(sdf_eval(s, V3()), -0.1, 1e-15);
}
TEST(SdfEval, CapsuleEndCap) {  // :54-58
  Shape s = mk(ShapeType::Capsule);
  s.half_length = 0.1;
  s.radius = 0.05;
  EXPECT_NEAR(sdf_eval(s, V3(0, 0, 0.2)), 0.05, 1e-15);
  EXPECT_NEAR(sdf_eval(s, V3(0.1, 0, 0)), 0.05, 1e-15);
}
TEST(SdfEval, PlaneSignedHalfSpace) {  // :60-64
  Shape s = mk(ShapeType::Plane);
  EXPECT_NEAR(sdf_eval(s, V3(3, -4, 0.5)), 0.5, 1e-15);
  EXPECT_NEAR(sdf_eval(s, V3(0, 0, -0.2)), -0.2, 1e-15);
}
TEST(SdfEval, WorldFrameConsistency) {  // :66-78
  auto g = rng(11);
  for (Shape& s : analytic_zoo())
    for (int i = 0; i < 50; ++i) {
      Pose world = random_pose(g, 0.5);
      V3 p = random_vec3(g, -1, 1);
      EXPECT_NEAR(sdf_eval(s, world, p), detail::sdf_local(s, inverse(world).apply(p)), 1e-12);
    }
}
TEST(SdfEval, Continuity) {  // :80-91
  auto g = rng(12);
  for (Shape& s : analytic_zoo())
    for (int i = 0; i < 200; ++i) {
      V3 p = random_vec3(g, -0.5, 0.5);
      V3 d = random_vec3(g);
      d = d / d.norm() * 1e-4;
      EXPECT(std::abs(sdf_eval(s, p) - sdf_eval(s, p + d)) <= d.norm() * (1.0 + 1e-3));
    }
}
TEST(SdfGradient, RadialAndPlane) {  // :93-101
  Shape sph = mk(ShapeType::Sphere);
  sph.radius = 0.1;
  EXPECT((sdf_gradient(sph, V3(0.2, 0, 0)) - V3(1, 0, 0)).norm() < 1e-12);
  Shape pl = mk(ShapeType::Plane);
  auto g = rng(13);
  for (int i = 0; i < 10; ++i) EXPECT((sdf_gradient(pl, random_vec3(g)) - V3(0, 0, 1)).norm() < 1e-12);
}
TEST(SdfGradient, MatchesFiniteDifferences) {  // :103-117
  auto g = rng(14);
  for (Shape& s : analytic_zoo()) {
    int checked = 0;
    while (checked < 250) {
      V3 p = random_vec3(g, -0.6, 0.6);
      if (std::abs(sdf_eval(s, p)) < 1e-3) continue;
      V3 fd = fd_gradient(s, p);
      if (std::abs(fd.norm() - 1.0) > 1e-6) continue;
      ++checked;
      EXPECT((sdf_gradient(s, p) - fd).norm() < 1e-4);
    }
  }
}
TEST(SdfGradient, UnitNorm) {  // :119-124
  auto g = rng(15);
  for (Shape& s : analytic_zoo())
    for (int i = 0; i < 100; ++i) EXPECT_NEAR(sdf_gradient(s, random_vec3(g)).norm(), 1.0, 1e-9);
}
TEST(SdfGradient, MedialAxisTieBreak) {  // :126-129
  Shape cube = mk(ShapeType::Box);
  cube.half_extents = V3(0.1, 0.1, 0.1);
  EXPECT((sdf_gradient(cube, V3()) - V3(1, 0, 0)).norm() < 1e-12);
}
TEST(SdfVolume, TrilinearReproducesLinearField) {  // sdf.hpp:46-62 (software trilinear)
  auto vol = std::make_shared<SdfVolume>();
  vol->origin = V3(-0.1, -0.1, -0.1);
  vol->voxel = 0.02;
  vol->dims = I3{11, 11, 11};
  for (int k = 0; k < 11; ++k)
    for (int j = 0; j < 11; ++j)
      for (int i = 0; i < 11; ++i) vol->samples.push_back(float(0.5 * (vol->origin.x + 0.02 * i) - 0.25));
  Shape s = mk(ShapeType::Volume);
  s.volume = vol;
  auto g = rng(18);
  for (int t = 0; t < 100; ++t) {
    V3 p = random_vec3(g, -0.09, 0.09);
    EXPECT_NEAR(sdf_eval(s, p), 0.5 * p.x - 0.25, 1e-6);
  }
  // Outside: pays the distance to the sampled box.
  EXPECT_NEAR(sdf_eval(s, V3(0.2, 0, 0)), (0.5 * 0.1 - 0.25) + 0.1, 1e-6);
}

// ---- test_coupling.cpp -------------------------------------------------------
namespace {
World block_world() {  // test_coupling.cpp:15-34
  World w;
  w.soft.grid.h = 0.01;
  w.soft.grid.dims = I3{32, 32, 32};
  w.soft.materials = {soft_clay()};
  std::mt19937_64 r(7);
  seed_particles_box(w.soft, V3(0.10, 0.10, 0.06), V3(0.14, 0.14, 0.09), 0, kSoftClayParticleVolume, r);
  w.soft.dt = 2e-4;
  RigidBody floor;
  floor.mode = BodyMode::Kinematic;
  floor.pose = Pose::from_translation(V3(0, 0, 0.04));
  Shape ps = mk(ShapeType::Plane);
  ps.normal = V3(0, 0, 1);
  floor.shapes = {ps};
  w.bodies.push_back(floor);
  return w;
}
Shape sphere(double r) {
  Shape s = mk(ShapeType::Sphere);
  s.radius = r;
  return s;
}
}  // namespace

TEST(Sync, MovingBodyTwistCopied) {  // test_coupling.cpp:45-55
  World w = block_world();
  w.init();
  w.bodies[0].linear_velocity = V3(0.1, 0, 0);
  w.bodies[0].angular_velocity = V3(0, 0, 2.0);
  w.bodies[0].pose.translation += V3(0.01, 0, 0);
  w.sync_rigid_to_soft();
  EXPECT((w.mirrors[0].linear_velocity - V3(0.1, 0, 0)).norm() < 1e-300);
  EXPECT((w.mirrors[0].angular_velocity - V3(0, 0, 2.0)).norm() < 1e-300);
  EXPECT((w.mirrors[0].pose.translation - w.bodies[0].pose.translation).norm() < 1e-300);
}

TEST(PenaltyParticle, OutsideBandZeroForce) {  // :79-85
  World w = block_world();
  w.init();
  penalty_particle(w);
  for (const V3& f : w.soft.ext_force) EXPECT(f.norm() < 1e-300);
  EXPECT(w.wrenches[0].force.norm() < 1e-300);
}

TEST(PenaltyParticle, StaticPlanePenaltyOracle) {  // :87-101
  World w = block_world();
  w.soft.particles.clear();
  Particle p;
  p.x = V3(0.15, 0.15, 0.038);
  p.mass = 1e-4;
  w.soft.particles = {p};
  w.init();
  double r_c = w.coupling.contact_radius(w.soft.grid.h);
  penalty_particle(w);
  double phi = 0.038 - 0.04;
  V3 o = w.bodies[0].shapes[0].k_n * (r_c - phi) * V3(0, 0, 1);
  EXPECT((w.soft.ext_force[0] - o).norm() < 1e-12);
  EXPECT((w.wrenches[0].force + o).norm() < 1e-12);
}

TEST(PenaltyParticle, DampingOpposesApproachOnly) {  // :103-123
  World w = block_world();
  w.soft.particles.clear();
  Particle p;
  p.x = V3(0.15, 0.15, 0.038);
  p.mass = 1e-4;
  p.v = V3(0, 0, -0.2);
  w.soft.particles = {p};
  w.init();
  double r_c = w.coupling.contact_radius(w.soft.grid.h);
  penalty_particle(w);
  double spring = w.bodies[0].shapes[0].k_n * (r_c - (0.038 - 0.04));
  double damp = w.coupling.c_d * 0.2;
  EXPECT_NEAR(w.soft.ext_force[0].z, spring + damp, 1e-12);
  w.soft.particles[0].v = V3(0, 0, 0.2);
  w.init();
  penalty_particle(w);
  EXPECT_NEAR(w.soft.ext_force[0].z, spring, 1e-12);
}

TEST(PenaltyParticle, CoulombCapOnFriction) {  // :125-147
  World w = block_world();
  w.soft.particles.clear();
  Particle p;
  p.x = V3(0.15, 0.15, 0.038);
  p.mass = 1e-4;
  w.soft.particles = {p};
  w.init();
  const Shape& s = w.bodies[0].shapes[0];
  double r_c = w.coupling.contact_radius(w.soft.grid.h);
  double fn = s.k_n * (r_c - (0.038 - 0.04));
  w.soft.particles[0].v = V3(0.01, 0, 0);
  penalty_particle(w);
  EXPECT_NEAR(w.soft.ext_force[0].x, -s.k_t * 0.01, 1e-12);
  w.soft.particles[0].v = V3(10.0, 0, 0);
  w.init();
  penalty_particle(w);
  EXPECT_NEAR(w.soft.ext_force[0].x, -s.friction * fn, 1e-12);
}

TEST(PenaltyParticle, ThirdLawSummation) {  // :149-183
  World w = block_world();
  RigidBody ball;
  ball.pose = Pose::from_translation(V3(0.12, 0.12, 0.075));
  ball.linear_velocity = V3(0.1, -0.2, 0.05);
  ball.angular_velocity = V3(1, 2, -1);
  ball.shapes = {sphere(0.015)};
  w.bodies.push_back(ball);
  for (auto& p : w.soft.particles) p.v = V3(0.05, 0.02, -0.1);
  w.init();
  penalty_particle(w);
  V3 total, torque;
  V3 com = w.bodies[1].world_com();
  double r_c = w.coupling.contact_radius(w.soft.grid.h);
  int contacts = 0;
  for (std::size_t ip = 0; ip < w.soft.particles.size(); ++ip) {
    const V3& f = w.soft.ext_force[ip];
    if (f.norm() == 0.0) continue;
    EXPECT(r_c - sdf_eval(w.bodies[1].shapes[0], compose(w.bodies[1].pose, w.bodies[1].shapes[0].local_pose),
                          w.soft.particles[ip].x) > 0.0);
    total += f;
    torque += (w.soft.particles[ip].x - com).cross(-f);
    ++contacts;
  }
  EXPECT(contacts > 10);
  EXPECT((w.wrenches[1].force + total).norm() < 1e-10);
  EXPECT((w.wrenches[1].torque - torque).norm() < 1e-8);
}

TEST(PenaltyGrid, NoContactLeavesGridForcesUntouched) {  // :185-193
  World w = block_world();
  w.init();
  p2g(w.soft);
  std::vector<V3> before = w.soft.grid.force;
  penalty_grid(w);
  for (std::size_t i = 0; i < before.size(); ++i) EXPECT((w.soft.grid.force[i] - before[i]).norm() < 1e-300);
}

TEST(PenaltyGrid, NodeForceMatchesSharedFormula) {  // :195-239
  World w = block_world();
  w.soft.particles.clear();
  std::mt19937_64 r(8);
  seed_particles_box(w.soft, V3(0.10, 0.10, 0.041), V3(0.14, 0.14, 0.07), 0, kSoftClayParticleVolume, r);
  for (auto& p : w.soft.particles) p.v = V3(0.02, 0, -0.1);
  w.init();
  p2g(w.soft);
  std::vector<V3> before = w.soft.grid.force;
  penalty_grid(w);
  MpmGrid& g = w.soft.grid;
  double r_c = grid_contact_radius(w.coupling, g.h);
  const Shape& s = w.bodies[0].shapes[0];
  Pose sp = compose(w.bodies[0].pose, s.local_pose);
  int checked = 0;
  for (std::size_t ni : w.soft.scratch.active_nodes) {
    if (g.mass[ni] <= 0.0) continue;
    int i = int(ni % g.dims.x), j = int((ni / g.dims.x) % g.dims.y),
        k = int(ni / (std::size_t(g.dims.x) * g.dims.y));
    V3 xi = g.node_pos(i, j, k);
    double phi = sdf_eval(s, sp, xi);
    V3 delta = g.force[ni] - before[ni];
    if (phi >= r_c) {
      EXPECT(delta.norm() < 1e-300);
      continue;
    }
    V3 n(0, 0, 1);
    V3 v = g.momentum[ni] / g.mass[ni];
    V3 f = s.k_n * (r_c - phi) * n;
    double vn = v.z;
    f += -w.coupling.c_d * std::min(0.0, vn) * n;
    V3 vt = v - vn * n;
    if (vt.norm() > 1e-12) f -= std::min(s.friction * s.k_n * (r_c - phi), s.k_t * vt.norm()) * (vt / vt.norm());
    f *= g.mass[ni] / w.mean_particle_mass;
    EXPECT((delta - f).norm() < 1e-10 * std::max(1.0, f.norm()));
    ++checked;
  }
  EXPECT(checked > 10);
}

TEST(PenaltyGrid, ThirdLawNodeWise) {  // :241-256
  World w = block_world();
  w.soft.particles.clear();
  std::mt19937_64 r(9);
  seed_particles_box(w.soft, V3(0.10, 0.10, 0.041), V3(0.14, 0.14, 0.07), 0, kSoftClayParticleVolume, r);
  w.init();
  p2g(w.soft);
  std::vector<V3> before = w.soft.grid.force;
  penalty_grid(w);
  V3 total;
  for (std::size_t ni = 0; ni < before.size(); ++ni) total += w.soft.grid.force[ni] - before[ni];
  EXPECT(total.norm() > 0.0);
  EXPECT((w.wrenches[0].force + total).norm() < 1e-10);
}

TEST(EnvStep, ReportCounters) {  // :258-268
  World w = block_world();
  w.n_rigid = 25;
  w.n_soft = 2;
  w.init();
  StepReport rep = env_step(w);
  EXPECT(rep.rigid_steps == 25);
  EXPECT(rep.soft_substeps == 50);
  EXPECT(rep.cfl_cycles >= 50);
  EXPECT_NEAR(w.time, 25 * 2 * w.soft.dt, 1e-15);
}

TEST(EnvStep, DynamicBodyReceivesReactionWrench) {  // :299-331
  World w = block_world();
  RigidBody ball;
  ball.mode = BodyMode::Dynamic;
  ball.mass = 0.05;
  ball.inertia = V3(8e-6, 8e-6, 8e-6);
  ball.pose = Pose::from_translation(V3(0.12, 0.12, 0.115));
  ball.linear_velocity = V3(0, 0, -0.5);
  ball.shapes = {sphere(0.015)};
  w.bodies.push_back(ball);
  w.n_rigid = 5;
  w.n_soft = 2;
  w.init();
  double t_total = 0.0, max_pen = 0.0;
  bool contacted = false;
  for (int step = 0; step < 12; ++step) {
    StepReport rep = env_step(w);
    t_total = w.time;
    max_pen = std::max(max_pen, rep.max_penetration);
    if (w.pending_wrenches[1].force.norm() > 0.0) contacted = true;
  }
  EXPECT(contacted);
  double free_fall_v = -0.5 - 9.81 * t_total;
  EXPECT(w.bodies[1].linear_velocity.z > free_fall_v + 0.01);
  EXPECT(max_pen <= 2.0 * w.coupling.contact_radius(w.soft.grid.h));
}

TEST(EnvStep, BitwiseDeterminism) {  // :333-359 (state compared directly)
  auto run = [](int threads) {
    worker_threads() = threads;
    World w = block_world();
    RigidBody ball;
    ball.mode = BodyMode::Dynamic;
    ball.mass = 0.05;
    ball.inertia = V3(8e-6, 8e-6, 8e-6);
    ball.pose = Pose::from_translation(V3(0.12, 0.12, 0.105));
    ball.linear_velocity = V3(0, 0, -0.3);
    ball.shapes = {sphere(0.015)};
    w.bodies.push_back(ball);
    w.n_rigid = 4;
    w.init();
    for (int i = 0; i < 5; ++i) env_step(w);
    worker_threads() = 1;
    std::uint64_t h = 1469598103934665603ull;
    for (const Particle& p : w.soft.particles) {
      h = fnv1a(&p.x, sizeof(V3), h);
      h = fnv1a(&p.v, sizeof(V3), h);
      h = fnv1a(&p.F, sizeof(M3), h);
    }
    h = fnv1a(&w.bodies[1].pose.translation, sizeof(V3), h);
    return h;
  };
  std::uint64_t h1 = run(1), h2 = run(1), h3 = run(3);
  EXPECT(h1 == h2);
  EXPECT(h1 == h3);
}

TEST(EnvStep, GridModeRunsAndBalances) {  // :361-374
  World w = block_world();
  w.coupling.mode = CouplingMode::Grid;
  w.soft.particles.clear();
  std::mt19937_64 r(10);
  seed_particles_box(w.soft, V3(0.10, 0.10, 0.042), V3(0.14, 0.14, 0.07), 0, kSoftClayParticleVolume, r);
  w.n_rigid = 4;
  w.init();
  StepReport rep = env_step(w);
  EXPECT(rep.rigid_steps == 4);
  EXPECT(rep.lost_particles == 0u);
  for (const auto& p : w.soft.particles) EXPECT(p.x.allFinite());
}

// ---- acceptance.cpp ---------------------------------------------------------
TEST(Acceptance, C1_GridTransferConservation) {  // acceptance.cpp:50-102
  SoftState st;
  st.grid.h = 0.01;
  st.grid.dims = I3{32, 32, 32};
  st.materials = {soft_clay()};
  st.gravity = V3();
  std::mt19937_64 r(11);
  std::uniform_real_distribution<double> pos(0.08, 0.24), vel(-0.5, 0.5), m(0.5, 1.5), small(-0.05, 0.05);
  for (int i = 0; i < 1000; ++i) {
    Particle p;
    double z = pos(r), y = pos(r), x = pos(r);  // Vec3(pos(rng), pos(rng), pos(rng)), GCC order
    p.x = V3(x, y, z);
    z = vel(r), y = vel(r), x = vel(r);
    p.v = V3(x, y, z);
    p.mass = 1e-4 * m(r);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) p.C.m[a][b] = vel(r);
    p.F = M3::Identity();
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) p.F.m[a][b] += small(r);
    st.particles.push_back(p);
  }
  st.init_buffers();
  double mass_p = 0.0;
  V3 mom_p;
  for (const Particle& p : st.particles) {
    mass_p += p.mass;
    mom_p += p.mass * p.v;
  }
  st.grid.clear();
  p2g(st);
  double mass_g = 0.0;
  V3 mom_g;
  for (std::size_t ni : st.scratch.active_nodes) {
    mass_g += st.grid.mass[ni];
    mom_g += st.grid.momentum[ni];
  }
  EXPECT(std::abs(mass_g - mass_p) / mass_p <= 1e-12);
  EXPECT((mom_g - mom_p).norm() / mom_p.norm() <= 1e-10);
  for (Particle& p : st.particles) p.F = M3::Identity();
  soft_substep(st);
  V3 mom_after;
  for (const Particle& p : st.particles) mom_after += p.mass * p.v;
  EXPECT((mom_after - mom_p).norm() / mom_p.norm() <= 1e-8);
}

TEST(Acceptance, C2_Constitutive) {  // acceptance.cpp:109-151
  Material m{1000.0, 1e4, 0.3, 2e3};
  const double eps = 1e-3;
  M3 f = M3::Identity();
  f.m[0][0] = 1.0 + eps;
  M3 tau = kirchhoff_stress(f, m);
  double s11 = (m.lambda() + 2.0 * m.mu()) * eps, s22 = m.lambda() * eps;
  double uni = std::max(std::abs(tau.m[0][0] - s11) / std::abs(s11), std::abs(tau.m[1][1] - s22) / std::abs(s22));
  M3 g = M3::Identity();
  g.m[0][1] = eps;
  double shear = std::abs(kirchhoff_stress(g, m).m[0][1] - m.mu() * eps) / (m.mu() * eps);
  std::mt19937_64 r(22);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  double worst = 0.0;
  for (double sy : {2e3, 1e4}) {
    Material my = m;
    my.yield_stress = sy;
    double cap = std::sqrt(2.0 / 3.0) * sy * (1.0 + 1e-6);
    for (int t = 0; t < 500; ++t) {
      M3 ft;
      do {
        ft = M3::Identity();
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) ft.m[a][b] += u(r);
      } while (ft.determinant() < 0.1);
      M3 fp = von_mises_return_map(ft, my);
      M3 t2 = kirchhoff_stress(fp, my);
      M3 dev = t2 - (t2.trace() / 3.0) * M3::Identity();
      worst = std::max(worst, dev.norm() / cap);
    }
  }
  EXPECT(uni <= 0.01);
  EXPECT(shear <= 0.01);
  EXPECT(worst <= 1.0);
}

TEST(Acceptance, C3_SdfGradientFiniteDifference) {  // acceptance.cpp:156-182
  std::vector<Shape> shapes(4);
  shapes[0] = mk(ShapeType::Plane);
  shapes[0].normal = V3(0.2, -0.3, 0.93) / V3(0.2, -0.3, 0.93).norm();
  shapes[0].offset = 0.01;
  shapes[1] = sphere(0.05);
  shapes[2] = mk(ShapeType::Box);
  shapes[2].half_extents = V3(0.03, 0.02, 0.05);
  shapes[3] = mk(ShapeType::Capsule);
  shapes[3].half_length = 0.04;
  shapes[3].radius = 0.015;
  std::mt19937_64 r(33);
  std::uniform_real_distribution<double> u(-0.1, 0.1);
  const double fd = 1e-6;
  double worst = 0.0;
  for (const Shape& s : shapes)
    for (int t = 0; t < 250; ++t) {
      double z = u(r), y = u(r), x = u(r);
      V3 p(x, y, z);
      V3 grad = sdf_gradient(s, p);
      V3 num;
      for (int ax = 0; ax < 3; ++ax) {
        V3 dp;
        dp[ax] = fd;
        num[ax] = (sdf_eval(s, p + dp) - sdf_eval(s, p - dp)) / (2.0 * fd);
      }
      worst = std::max(worst, std::max(std::abs(grad.x - num.x), std::max(std::abs(grad.y - num.y), std::abs(grad.z - num.z))));
    }
  EXPECT(worst <= 1e-4);
}

TEST(Acceptance, C3_ThirdLawEverySubstep) {  // acceptance.cpp:156-160 (force balance <= 1e-10)
  World w = block_world();
  RigidBody ball;
  ball.mode = BodyMode::Dynamic;
  ball.mass = 0.05;
  ball.inertia = V3(8e-6, 8e-6, 8e-6);
  ball.pose = Pose::from_translation(V3(0.12, 0.12, 0.10));
  ball.linear_velocity = V3(0, 0, -0.3);
  ball.shapes = {sphere(0.015)};
  w.bodies.push_back(ball);
  w.n_rigid = 5;
  w.init();
  double worst = 0.0;
  for (int i = 0; i < 4; ++i) worst = std::max(worst, env_step(w).max_force_balance_error);
  EXPECT(worst <= 1e-10);
}

TEST(Svd, ReconstructionAndOrthogonality) {  // contract of Eigen::JacobiSVD (mpm.hpp:155)
  auto g = rng(77);
  for (int t = 0; t < 1000; ++t) {
    M3 a;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) a.m[r][c] = uniform(g, -1, 1) + (r == c ? 1.0 : 0.0);
    Svd3 s = svd3(a);
    M3 rec = s.U * M3::diag(s.s) * s.V.transpose();
    EXPECT((rec - a).norm() < 1e-13 * std::max(1.0, a.norm()));
    EXPECT((s.U.transpose() * s.U - M3::Identity()).norm() < 1e-13);
    EXPECT((s.V.transpose() * s.V - M3::Identity()).norm() < 1e-13);
    EXPECT(s.s.x >= 0 && s.s.y >= 0 && s.s.z >= 0);
  }
}

// ---- test_sdf.cpp (mesh baking, :151-182) -----------------------------------
TEST(BakeMesh, UnitCubeAgainstAnalyticBox) {  // test_sdf.cpp:151-164
  double voxel = 0.05;
  SdfVolume vol = bake_mesh_sdf(make_box_mesh(V3(0.5, 0.5, 0.5)), voxel, 3 * voxel);
  Shape analytic = mk(ShapeType::Box);
  analytic.half_extents = V3(0.5, 0.5, 0.5);
  Shape baked = mk(ShapeType::Volume);
  baked.volume = std::make_shared<SdfVolume>(vol);
  auto g = rng(17);
  for (int i = 0; i < 1000; ++i) {
    V3 p = random_vec3(g, -0.7, 0.7);
    EXPECT_NEAR(sdf_eval(baked, p), sdf_eval(analytic, p), voxel);
  }
}
TEST(BakeMesh, CenterSample) {  // :166-170
  double voxel = 0.1;
  SdfVolume vol = bake_mesh_sdf(make_box_mesh(V3(0.5, 0.5, 0.5)), voxel, 2 * voxel);
  EXPECT_NEAR(vol.interpolate(V3()), -0.5, voxel);
}
TEST(BakeMesh, SurfaceLatticeProximity) {  // :172-176
  double voxel = 0.1;
  SdfVolume vol = bake_mesh_sdf(make_box_mesh(V3(0.5, 0.5, 0.5)), voxel, 2 * voxel);
  EXPECT(std::abs(vol.interpolate(V3(0.5, 0.0, 0.0))) <= voxel);
}
TEST(BakeMesh, EmptyAndDegenerateMeshError) {  // :178-182
  EXPECT_THROW(bake_mesh_sdf({}, 0.01, 0.01), std::invalid_argument);
  Triangle degen{V3(0, 0, 0), V3(1, 0, 0), V3(2, 0, 0)};
  EXPECT_THROW(bake_mesh_sdf({degen, degen}, 0.1, 0.1), std::invalid_argument);
}

// ---- test_scenario.cpp (task metrics, :24-270) -----------------------------
namespace {
const RegionBox kUnitRegion{V3(0, 0, 0), V3(1, 1, 1)};
double chamfer_brute(const std::vector<V3>& a, const std::vector<V3>& b) {  // test_scenario.cpp:193-204
  auto side = [](const std::vector<V3>& from, const std::vector<V3>& to) {
    double sum = 0.0;
    for (const V3& p : from) {
      double best = std::numeric_limits<double>::infinity();
      for (const V3& q : to) best = std::min(best, (p - q).norm());
      sum += best;
    }
    return sum / static_cast<double>(from.size());
  };
  return side(a, b) + side(b, a);
}
}  // namespace

TEST(Fill, AllInsideAtRestSucceeds) {  // test_scenario.cpp:27-34
  std::vector<V3> x, v;
  for (int i = 0; i < 10; ++i) x.push_back(V3(0.1 * i + 0.05, 0.5, 0.5)), v.push_back(V3());
  FillResult r = metric_fill(x, v, kUnitRegion);
  EXPECT(r.fraction == 1.0 && r.max_speed == 0.0 && r.success);
}
TEST(Fill, NoneInsideFails) {  // :36-41
  FillResult r = metric_fill({V3(2, 2, 2), V3(-1, 0, 0)}, {V3(), V3()}, kUnitRegion);
  EXPECT(r.fraction == 0.0 && !r.success);
}
TEST(Fill, NinetyOnePercentInsideIsSuccessAtTheBoundary) {  // :43-53
  std::vector<V3> x, v(100);
  for (int i = 0; i < 91; ++i) x.push_back(V3(0.5, 0.5, 0.5));
  for (int i = 0; i < 9; ++i) x.push_back(V3(5, 5, 5));
  FillResult r = metric_fill(x, v, kUnitRegion);
  EXPECT(r.fraction == 0.91 && r.success);
  x[0] = V3(5, 5, 5);
  EXPECT(!metric_fill(x, v, kUnitRegion).success);
}
TEST(Fill, FastParticleBreaksSuccess) {  // :55-61
  FillResult r = metric_fill({V3(0.5, 0.5, 0.5)}, {V3(0.06, 0, 0)}, kUnitRegion);
  EXPECT(r.fraction == 1.0);
  EXPECT_NEAR(r.max_speed, 0.06, 1e-15);
  EXPECT(!r.success);
}
TEST(Fill, FractionInvariantUnderReordering) {  // :63-71
  auto g = rng(7);
  std::vector<V3> x, v;
  for (int i = 0; i < 200; ++i) x.push_back(random_vec3(g, -0.5, 1.5)), v.push_back(V3());
  FillResult a = metric_fill(x, v, kUnitRegion);
  std::reverse(x.begin(), x.end());
  FillResult b = metric_fill(x, v, kUnitRegion);
  EXPECT(a.fraction == b.fraction && a.max_speed == b.max_speed);
}
TEST(Fill, EmptyInputThrows) {  // :73-75
  EXPECT_THROW(metric_fill({}, {}, kUnitRegion), std::invalid_argument);
}
TEST(Heightmap, NoParticlesAllZeros) {  // :80-85
  DepthMap m = render_heightmap({}, kUnitRegion, 4, 4);
  EXPECT(m.samples.size() == 16u);
  for (double s : m.samples) EXPECT(s == 0.0);
}
TEST(Heightmap, SingleParticleFillsExactlyItsCell) {  // :87-96
  V3 x(0.30, 0.77, 0.42);
  DepthMap m = render_heightmap({x}, kUnitRegion, 5, 4);
  int ci = static_cast<int>(x.x / 0.2), cj = static_cast<int>(x.y / 0.25);
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 5; ++i) EXPECT(m.at(i, j) == ((i == ci && j == cj) ? 0.42 : 0.0));
}
TEST(Heightmap, SameCellTakesMaxHeight) {  // :98-102
  DepthMap m = render_heightmap({V3(0.1, 0.1, 0.3), V3(0.12, 0.11, 0.8)}, kUnitRegion, 4, 4);
  EXPECT(m.at(0, 0) == 0.8);
}
TEST(Heightmap, PermutationInvariantAndMonotone) {  // :104-116
  auto g = rng(11);
  std::vector<V3> ps;
  for (int i = 0; i < 300; ++i) ps.push_back(random_vec3(g, 0.0, 1.0));
  DepthMap a = render_heightmap(ps, kUnitRegion, 6, 6);
  std::shuffle(ps.begin(), ps.end(), g);
  DepthMap b = render_heightmap(ps, kUnitRegion, 6, 6);
  EXPECT(a.samples == b.samples);
  ps.push_back(V3(0.5, 0.5, 0.99));
  DepthMap c = render_heightmap(ps, kUnitRegion, 6, 6);
  for (std::size_t i = 0; i < a.samples.size(); ++i) EXPECT(c.samples[i] >= b.samples[i]);
}
TEST(Heightmap, ParticlesOutsideRegionIgnored) {  // :118-121
  DepthMap m = render_heightmap({V3(1.5, 0.5, 0.5)}, kUnitRegion, 4, 4);
  for (double s : m.samples) EXPECT(s == 0.0);
}
TEST(Heightmap, TooCoarseResolutionThrows) {  // :123-125
  EXPECT_THROW(render_heightmap({}, kUnitRegion, 1, 4), std::invalid_argument);
}
namespace {
DepthMap map_from(std::initializer_list<double> vals, int nx, int ny, double threshold) {  // :130-138
  DepthMap m;
  m.nx = nx;
  m.ny = ny;
  m.cell = 0.01;
  m.threshold = threshold;
  m.samples.assign(vals);
  return m;
}
}  // namespace
TEST(WriteIou, IdenticalMapsScoreOne) {  // :140-145
  DepthMap m = map_from({0.1, 0.0, 0.2, 0.0, 0.1, 0.2}, 3, 2, 0.05);
  IouResult r = metric_write_iou(m, m);
  EXPECT(r.iou == 1.0 && r.success);
}
TEST(WriteIou, DisjointOccupancyScoresZero) {  // :147-153
  IouResult r = metric_write_iou(map_from({0.0, 0.1, 0.0, 0.1}, 2, 2, 0.05), map_from({0.1, 0.0, 0.1, 0.0}, 2, 2, 0.05));
  EXPECT(r.iou == 0.0 && !r.success);
}
TEST(WriteIou, BothEmptyDefinedAsOne) {  // :155-159
  DepthMap a = map_from({0.1, 0.1, 0.1, 0.1}, 2, 2, 0.05);
  EXPECT(metric_write_iou(a, a).iou == 1.0);
}
TEST(WriteIou, MatchesBruteForceCountingOracle) {  // :161-180
  auto g = rng(13);
  for (int trial = 0; trial < 20; ++trial) {
    DepthMap a, b;
    a.nx = b.nx = 7;
    a.ny = b.ny = 5;
    a.threshold = b.threshold = 0.5;
    for (int i = 0; i < 35; ++i) {
      a.samples.push_back(uniform(g, 0.0, 1.0));
      b.samples.push_back(uniform(g, 0.0, 1.0));
    }
    std::size_t inter = 0, uni = 0;
    for (int i = 0; i < 35; ++i) {
      bool oa = a.samples[i] < 0.5, ob = b.samples[i] < 0.5;
      if (oa && ob) ++inter;
      if (oa || ob) ++uni;
    }
    double expect = uni == 0 ? 1.0 : double(inter) / double(uni);
    EXPECT(metric_write_iou(a, b).iou == expect);
  }
}
TEST(WriteIou, ResolutionMismatchThrows) {  // :182-186
  EXPECT_THROW(metric_write_iou(map_from({0, 0, 0, 0}, 2, 2, 0.5), map_from({0, 0, 0, 0, 0, 0}, 3, 2, 0.5)),
               std::invalid_argument);
}
TEST(Chamfer, EqualSetsAreZero) {  // :205-210
  auto g = rng(17);
  std::vector<V3> a;
  for (int i = 0; i < 50; ++i) a.push_back(random_vec3(g));
  EXPECT(chamfer_distance(a, a) == 0.0);
}
TEST(Chamfer, UnitSeparationSumsToTwo) {  // :211-214
  EXPECT(chamfer_distance({V3(0, 0, 0)}, {V3(0, 0, 1)}) == 2.0);
}
TEST(Chamfer, MatchesBruteForceOracle) {  // :216-224
  auto g = rng(19);
  std::vector<V3> a, b;
  for (int i = 0; i < 500; ++i) {
    a.push_back(random_vec3(g, 0.0, 0.2));
    b.push_back(random_vec3(g, 0.05, 0.25));
  }
  EXPECT_NEAR(chamfer_distance(a, b), chamfer_brute(a, b), 1e-12);
}
TEST(Chamfer, SymmetricAndNonNegative) {  // :226-234
  auto g = rng(23);
  std::vector<V3> a, b;
  for (int i = 0; i < 80; ++i) a.push_back(random_vec3(g));
  for (int i = 0; i < 120; ++i) b.push_back(random_vec3(g));
  double ab = chamfer_distance(a, b);
  EXPECT_NEAR(ab, chamfer_distance(b, a), 4 * std::numeric_limits<double>::epsilon() * ab);
  EXPECT(ab > 0.0);
}
TEST(Chamfer, EmptySetThrows) {  // :236-238
  EXPECT_THROW(chamfer_distance({}, {V3()}), std::invalid_argument);
}
TEST(Pinch, CurrentEqualsTargetSucceeds) {  // :243-249
  std::vector<V3> init = {V3(0, 0, 0), V3(1, 0, 0)}, target = {V3(0, 0, 1), V3(1, 0, 1)};
  PinchResult r = metric_pinch(target, init, target);
  EXPECT(r.ratio == 0.0 && r.success);
}
TEST(Pinch, CurrentEqualsInitialFails) {  // :251-257
  std::vector<V3> init = {V3(0, 0, 0), V3(1, 0, 0)}, target = {V3(0, 0, 1), V3(1, 0, 1)};
  PinchResult r = metric_pinch(init, init, target);
  EXPECT(r.ratio == 1.0 && !r.success);
}
TEST(Pinch, HalfwayInterpolationMatchesBruteForceRatio) {  // :259-273
  auto g = rng(29);
  std::vector<V3> init, target, current;
  for (int i = 0; i < 60; ++i) {
    V3 a = random_vec3(g, 0.0, 0.1);
    V3 b = a + V3(0.05, 0.0, 0.02);
    init.push_back(a);
    target.push_back(b);
    current.push_back(0.5 * (a + b));
  }
  PinchResult r = metric_pinch(current, init, target);
  double expect = chamfer_brute(current, target) / chamfer_brute(init, target);
  EXPECT_NEAR(r.ratio, expect, 1e-12);
  EXPECT(r.success == (r.ratio < 0.3));
}

// ---- north_star materials (analytic KATs: no reference test exists) --------
namespace {
Material model_mat(Model md, double yield = 2e3) {
  Material m = soft_clay();
  m.model = md;
  m.yield_stress = yield;
  return m;
}
}  // namespace
TEST(FixedCorotated, RestAndRotationAreStressFree) {
  Material m = model_mat(Model::FixedCorotated);
  EXPECT(kirchhoff_fixed_corotated(M3::Identity(), m).norm() < 1e-12);
  auto g = rng(41);
  M3 r = random_quat(g).toRotationMatrix();
  EXPECT(kirchhoff_fixed_corotated(r, m).norm() < 1e-9);
}
TEST(FixedCorotated, SmallStrainMatchesLinearElasticity) {
  Material m = model_mat(Model::FixedCorotated);
  const double e = 1e-4;
  M3 f = M3::Identity();
  f.m[0][0] = 1.0 + e;
  M3 tau = kirchhoff_fixed_corotated(f, m);
  EXPECT_NEAR(tau.m[0][0], (2.0 * m.mu() + m.lambda()) * e, 1e-3 * (2.0 * m.mu() + m.lambda()) * e);
  EXPECT_NEAR(tau.m[1][1], m.lambda() * e, 1e-3 * m.lambda() * e);
}
TEST(FixedCorotated, IsotropicScalingClosedForm) {
  Material m = model_mat(Model::FixedCorotated);
  const double sc = 1.07, J = sc * sc * sc;
  M3 tau = kirchhoff_fixed_corotated(M3::Identity() * sc, m);
  const double expect = 2.0 * m.mu() * (sc - 1.0) * sc + m.lambda() * (J - 1.0) * J;
  for (int i = 0; i < 3; ++i) EXPECT_NEAR(tau.m[i][i], expect, 1e-10 * std::abs(expect));
  EXPECT(std::abs(tau.m[0][1]) < 1e-9 && std::abs(tau.m[1][2]) < 1e-9);
}
TEST(DruckerPrager, TensionProjectsToTheTip) {
  Material m = model_mat(Model::DruckerPrager, 30.0);
  auto g = rng(43);
  M3 r = random_quat(g).toRotationMatrix();
  M3 f = r * M3::diag(V3(1.02, 1.01, 1.005));
  double q = 0.0;
  M3 fp = drucker_prager_return_map(f, m, q);
  Svd3 s = svd3(fp);
  EXPECT(std::abs(s.s.x - 1.0) < 1e-12 && std::abs(s.s.y - 1.0) < 1e-12 && std::abs(s.s.z - 1.0) < 1e-12);
  EXPECT_NEAR(q, V3(std::log(1.02), std::log(1.01), std::log(1.005)).norm(), 1e-12);
}
TEST(DruckerPrager, InsideTheConeUnchanged) {
  Material m = model_mat(Model::DruckerPrager, 30.0);
  M3 f = M3::diag(V3(0.99, 0.985, 0.99));  // compression, small shear
  double q = 0.5;
  M3 fp = drucker_prager_return_map(f, m, q);
  EXPECT((fp - f).norm() == 0.0 && q == 0.5);
}
TEST(DruckerPrager, ProjectionLandsOnTheCone) {
  Material m = model_mat(Model::DruckerPrager, 25.0);
  auto g = rng(47);
  for (int t = 0; t < 50; ++t) {
    M3 r = random_quat(g).toRotationMatrix();
    V3 sig(std::exp(uniform(g, -0.02, 0.002)), std::exp(uniform(g, -0.02, 0.002)), std::exp(uniform(g, -0.08, 0.0)));
    M3 f = r * M3::diag(sig);
    double q = 0.0;
    M3 fp = drucker_prager_return_map(f, m, q);
    Svd3 s = svd3(fp);
    V3 e(std::log(s.s.x), std::log(s.s.y), std::log(s.s.z));
    const double tr = e.x + e.y + e.z;
    const double dn = (e - V3(tr / 3.0, tr / 3.0, tr / 3.0)).norm();
    const double yield = dn + (3.0 * m.lambda() + 2.0 * m.mu()) / (2.0 * m.mu()) * tr * m.dp_alpha();
    EXPECT(yield <= 1e-10);                       // never outside the cone
    if (q > 0.0) EXPECT(std::abs(yield) < 1e-10 || (dn < 1e-12 && std::abs(tr) < 1e-12));  // on it when projected
    EXPECT(std::abs(fp.determinant() - std::exp(tr)) < 1e-10);
  }
}
TEST(Fluid, PressureAndVolumeUpdate) {
  Material m = model_mat(Model::Fluid);
  Particle p;
  p.jp = 0.97;
  M3 tau = kirchhoff_of(p, m);
  EXPECT_NEAR(tau.m[0][0], m.bulk() * (0.97 - 1.0) * 0.97, 1e-12 * m.bulk());
  EXPECT(tau.m[0][1] == 0.0);
  p.C = M3::diag(V3(0.5, -0.2, 0.1));
  plasticity_update(p, m, 1e-3);
  EXPECT_NEAR(p.jp, 0.97 * (1.0 + 1e-3 * 0.4), 1e-15);
  EXPECT((p.F - M3::Identity()).norm() == 0.0);
}
TEST(Materials, ValidationPerModel) {
  Material dp = model_mat(Model::DruckerPrager, 95.0);
  EXPECT_THROW(dp.validate(), std::invalid_argument);
  Material fl = model_mat(Model::Fluid, 0.0);
  fl.validate();  // yield stress unused
}

int main(int argc, char** argv) {
  std::string filter = argc > 1 ? argv[1] : "";
  for (const Reg& r : registry()) {
    if (!filter.empty() && std::string(r.name).find(filter) == std::string::npos) continue;
    g_cur = r.name;
    g_cur_failed = false;
    try {
      r.fn();
    } catch (const std::exception& e) {
      std::printf("  exception: %s\n", e.what());
      g_cur_failed = true;
    }
    if (g_cur_failed) {
      ++g_fail;
      std::printf("FAIL %s\n", r.name);
    } else {
      ++g_pass;
      std::printf("PASS %s\n", r.name);
    }
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}
