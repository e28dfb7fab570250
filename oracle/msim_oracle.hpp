// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A double-precision CPU restatement of the reference simulator's soft-body
// hot path (/root/reference/proj/include/msim). It exists to check the CUDA
// product path; only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. The product library never
// links or calls it.
//
// Parity pinning: the reference cannot be compiled here (it needs Eigen3 and
// GTest, both absent) and ships no golden vectors. This
// restatement is pinned by ports of the reference's own known-answer tests
// (test_mpm.cpp, test_coupling.cpp, test_sdf.cpp, acceptance.cpp criteria 1,
// 2, 3, 7) in oracle/kat_oracle.cpp. Eigen's JacobiSVD is replaced by a
// one-sided Jacobi SVD with the same contract (orthogonal U, V; sigma >= 0);
// the constitutive functions are isotropic so the choice does not change
// results beyond roundoff.
//
// Every function cites the reference file:line it restates.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------------------
// Minimal linear algebra (stands in for Eigen::Vector3d / Matrix3d /
// Quaterniond used by geometry.hpp:16-20).

struct V3 {
  double x = 0, y = 0, z = 0;
  V3() = default;
  V3(double a, double b, double c) : x(a), y(b), z(c) {}
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  V3 operator+(const V3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  V3 operator-(const V3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  V3 operator-() const { return {-x, -y, -z}; }
  V3 operator*(double s) const { return {x * s, y * s, z * s}; }
  V3 operator/(double s) const { return {x / s, y / s, z / s}; }
  V3& operator+=(const V3& o) { x += o.x; y += o.y; z += o.z; return *this; }
  V3& operator-=(const V3& o) { x -= o.x; y -= o.y; z -= o.z; return *this; }
  V3& operator*=(double s) { x *= s; y *= s; z *= s; return *this; }
  double dot(const V3& o) const { return x * o.x + y * o.y + z * o.z; }
  V3 cross(const V3& o) const { return {y * o.z - z * o.y, z * o.x - x * o.z, x * o.y - y * o.x}; }
  double squaredNorm() const { return x * x + y * y + z * z; }
  double norm() const { return std::sqrt(squaredNorm()); }
  bool allFinite() const { return std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
  static V3 Zero() { return {0, 0, 0}; }
};
inline V3 operator*(double s, const V3& v) { return v * s; }

struct M3 {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  static M3 Zero() { return M3{}; }
  static M3 Identity() {
    M3 r;
    r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
    return r;
  }
  double& operator()(int r, int c) { return m[r][c]; }
  double operator()(int r, int c) const { return m[r][c]; }
  M3 operator+(const M3& o) const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[i][j] + o.m[i][j];
    return r;
  }
  M3 operator-(const M3& o) const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[i][j] - o.m[i][j];
    return r;
  }
  M3 operator*(double s) const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[i][j] * s;
    return r;
  }
  M3 operator*(const M3& o) const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += m[i][k] * o.m[k][j];
        r.m[i][j] = s;
      }
    return r;
  }
  V3 operator*(const V3& v) const {
    return {m[0][0] * v.x + m[0][1] * v.y + m[0][2] * v.z,
            m[1][0] * v.x + m[1][1] * v.y + m[1][2] * v.z,
            m[2][0] * v.x + m[2][1] * v.y + m[2][2] * v.z};
  }
  M3 transpose() const {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = m[j][i];
    return r;
  }
  double determinant() const {
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
  }
  double trace() const { return m[0][0] + m[1][1] + m[2][2]; }
  double norm() const {  // Frobenius, as Eigen's Matrix::norm()
    double s = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) s += m[i][j] * m[i][j];
    return std::sqrt(s);
  }
  bool allFinite() const {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        if (!std::isfinite(m[i][j])) return false;
    return true;
  }
  M3 inverse() const {
    double d = determinant();
    M3 r;
    r.m[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / d;
    r.m[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / d;
    r.m[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / d;
    r.m[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / d;
    r.m[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / d;
    r.m[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / d;
    r.m[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / d;
    r.m[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / d;
    r.m[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / d;
    return r;
  }
  static M3 diag(const V3& d) {
    M3 r;
    r.m[0][0] = d.x;
    r.m[1][1] = d.y;
    r.m[2][2] = d.z;
    return r;
  }
  static M3 outer(const V3& a, const V3& b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[i][j] = a[i] * b[j];
    return r;
  }
};
inline M3 operator*(double s, const M3& a) { return a * s; }

// Quaternion with Eigen's conventions (w, x, y, z; q*v rotates v).
struct Quat {
  double w = 1, x = 0, y = 0, z = 0;
  Quat() = default;
  Quat(double w_, double x_, double y_, double z_) : w(w_), x(x_), y(y_), z(z_) {}
  V3 vec() const { return {x, y, z}; }
  double norm() const { return std::sqrt(w * w + x * x + y * y + z * z); }
  void normalize() {
    double n = norm();
    if (n > 0) { w /= n; x /= n; y /= n; z /= n; }
  }
  Quat normalized() const { Quat q = *this; q.normalize(); return q; }
  Quat conjugate() const { return {w, -x, -y, -z}; }
  Quat operator*(const Quat& o) const {
    return {w * o.w - x * o.x - y * o.y - z * o.z, w * o.x + x * o.w + y * o.z - z * o.y,
            w * o.y + y * o.w + z * o.x - x * o.z, w * o.z + z * o.w + x * o.y - y * o.x};
  }
  V3 operator*(const V3& v) const {  // Eigen's _transformVector
    V3 uv = vec().cross(v);
    uv += uv;
    return v + w * uv + vec().cross(uv);
  }
  M3 toRotationMatrix() const {  // Eigen QuaternionBase::toRotationMatrix
    M3 r;
    double tx = 2 * x, ty = 2 * y, tz = 2 * z;
    double twx = tx * w, twy = ty * w, twz = tz * w;
    double txx = tx * x, txy = ty * x, txz = tz * x;
    double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r.m[0][0] = 1 - (tyy + tzz); r.m[0][1] = txy - twz; r.m[0][2] = txz + twy;
    r.m[1][0] = txy + twz; r.m[1][1] = 1 - (txx + tzz); r.m[1][2] = tyz - twx;
    r.m[2][0] = txz - twy; r.m[2][1] = tyz + twx; r.m[2][2] = 1 - (txx + tyy);
    return r;
  }
};

// Pose: geometry.hpp:26-51.
struct Pose {
  Quat rotation{1, 0, 0, 0};
  V3 translation{0, 0, 0};
  Pose() = default;
  Pose(const Quat& q, const V3& t) : rotation(q), translation(t) { canonicalize(); }
  static Pose from_translation(const V3& t) { return Pose(Quat(), t); }
  void canonicalize() {  // geometry.hpp:37-40
    rotation.normalize();
    if (rotation.w < 0.0) rotation = Quat(-rotation.w, -rotation.x, -rotation.y, -rotation.z);
  }
  V3 apply(const V3& p) const { return rotation * p + translation; }  // :42
};
// geometry.hpp:54-56
inline Pose compose(const Pose& a, const Pose& b) {
  return Pose(a.rotation * b.rotation, a.rotation * b.translation + a.translation);
}
// geometry.hpp:58-61
inline Pose inverse(const Pose& a) {
  Quat qi = a.rotation.conjugate();
  return Pose(qi, -(qi * a.translation));
}
// geometry.hpp:78-87 (AngleAxis -> quaternion)
inline Quat quat_exp(const V3& aa) {
  double ang = aa.norm();
  if (ang < 1e-14) {
    Quat q(1.0, 0.5 * aa.x, 0.5 * aa.y, 0.5 * aa.z);
    q.normalize();
    return q;
  }
  V3 axis = aa / ang;
  double s = std::sin(0.5 * ang);
  return Quat(std::cos(0.5 * ang), s * axis.x, s * axis.y, s * axis.z);
}

// ---------------------------------------------------------------------------
// 3x3 SVD (replaces Eigen::JacobiSVD<Mat3>, mpm.hpp:155, :169): one-sided
// Jacobi (Hestenes). A = U diag(s) V^T with U, V orthogonal and s >= 0.
struct Svd3 {
  M3 U, V;
  V3 s;
};
inline Svd3 svd3(const M3& A) {
  M3 a = A, v = M3::Identity();
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < 3; ++i) {
          alpha += a.m[i][p] * a.m[i][p];
          beta += a.m[i][q] * a.m[i][q];
          gamma += a.m[i][p] * a.m[i][q];
        }
        if (std::abs(gamma) <= 1e-15 * std::sqrt(alpha * beta) || gamma == 0.0) continue;
        rotated = true;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < 3; ++i) {
          double ap = a.m[i][p], aq = a.m[i][q];
          a.m[i][p] = c * ap - s * aq;
          a.m[i][q] = s * ap + c * aq;
          double vp = v.m[i][p], vq = v.m[i][q];
          v.m[i][p] = c * vp - s * vq;
          v.m[i][q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  Svd3 r;
  r.V = v;
  for (int j = 0; j < 3; ++j) {
    double n = std::sqrt(a.m[0][j] * a.m[0][j] + a.m[1][j] * a.m[1][j] + a.m[2][j] * a.m[2][j]);
    r.s[j] = n;
    for (int i = 0; i < 3; ++i) r.U.m[i][j] = n > 0 ? a.m[i][j] / n : (i == j ? 1.0 : 0.0);
  }
  return r;
}

// ---------------------------------------------------------------------------
// Errors (mpm.hpp:18-20; std::invalid_argument as in the reference).
struct SimulationDiverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// parallel.hpp:11-33: std::thread fork/join per call, static chunks.
inline int& worker_threads() {
  static int n = 1;
  return n;
}
template <class F>
void parallel_for(std::int64_t n, F&& body) {
  int workers = worker_threads();
  if (workers <= 1 || n < 256) {
    for (std::int64_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::vector<std::thread> pool;
  std::int64_t chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    std::int64_t lo = w * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &body] {
      for (std::int64_t i = lo; i < hi; ++i) body(i);
    });
  }
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------------------
// MPM state: mpm.hpp:24-145.

// Constitutive models. Hencky + von Mises is the reference's (mpm.hpp:152-181);
// the other three are the north_star's material set, absent from the reference
// (parity unpinned): restated from their published algorithms below.
enum class Model : int { HenckyVonMises = 0, FixedCorotated = 1, DruckerPrager = 2, Fluid = 3 };

struct Material {  // mpm.hpp:24-42 (+ model; yield_stress = friction angle in degrees for DruckerPrager)
  double density = 1000.0, youngs = 1e4, poisson = 0.3, yield_stress = 2e3;
  Model model = Model::HenckyVonMises;
  double mu() const { return youngs / (2.0 * (1.0 + poisson)); }
  double lambda() const { return youngs * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson)); }
  double bulk() const { return youngs / (3.0 * (1.0 - 2.0 * poisson)); }
  // Klar et al. 2016: alpha = sqrt(2/3) 2 sin(phi) / (3 - sin(phi))
  double dp_alpha() const {
    const double sp = std::sin(yield_stress * 3.14159265358979323846 / 180.0);
    return std::sqrt(2.0 / 3.0) * 2.0 * sp / (3.0 - sp);
  }
  void validate() const {
    if (youngs <= 0.0) throw std::invalid_argument("Material: E must be > 0");
    if (poisson <= 0.0 || poisson >= 0.5) throw std::invalid_argument("Material: nu must be in (0, 0.5)");
    if (model == Model::HenckyVonMises && yield_stress <= 0.0)
      throw std::invalid_argument("Material: yield stress must be > 0");
    if (model == Model::DruckerPrager && !(yield_stress > 0.0 && yield_stress < 90.0))
      throw std::invalid_argument("Material: friction angle must be in (0, 90) degrees");
    if (density <= 0.0) throw std::invalid_argument("Material: density must be > 0");
  }
};
inline Material soft_clay() { return Material{1000.0, 1e4, 0.3, 2e3}; }   // mpm.hpp:45
inline Material stiff_clay() { return Material{1000.0, 3e5, 0.3, 1e4}; }  // mpm.hpp:46
inline constexpr double kSoftClayParticleVolume = 6.2e-8;                 // mpm.hpp:47
inline constexpr double kStiffClayParticleVolume = 1.2e-7;                // mpm.hpp:48

struct Particle {  // mpm.hpp:50-58
  V3 x, v;
  double mass = 0.0;
  double volume0 = kSoftClayParticleVolume;
  M3 F = M3::Identity();
  M3 C = M3::Zero();
  int material = 0;
  double jp = 1.0;  // Fluid: volume ratio J; DruckerPrager: accumulated plastic strain q; else unused
};

enum class BoundaryKind : std::uint8_t { Sticky, Slip };  // mpm.hpp:60

struct I3 {
  int x = 0, y = 0, z = 0;
  int operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};

struct MpmGrid {  // mpm.hpp:65-107
  static constexpr int kBoundaryWidth = 2;
  double h = 0.01;
  I3 dims{64, 64, 64};
  V3 origin{0, 0, 0};
  std::array<BoundaryKind, 6> boundary = {BoundaryKind::Sticky, BoundaryKind::Sticky,
                                          BoundaryKind::Sticky, BoundaryKind::Sticky,
                                          BoundaryKind::Sticky, BoundaryKind::Sticky};
  std::vector<double> mass;
  std::vector<V3> momentum, force, velocity;
  std::size_t node_count() const { return std::size_t(dims.x) * dims.y * dims.z; }
  std::size_t node_index(int i, int j, int k) const {
    return (std::size_t(k) * dims.y + j) * dims.x + i;
  }
  V3 node_pos(int i, int j, int k) const { return origin + h * V3(i, j, k); }
  void allocate() {
    mass.assign(node_count(), 0.0);
    momentum.assign(node_count(), V3());
    force.assign(node_count(), V3());
    velocity.assign(node_count(), V3());
  }
  void clear() {
    std::fill(mass.begin(), mass.end(), 0.0);
    std::fill(momentum.begin(), momentum.end(), V3());
    std::fill(force.begin(), force.end(), V3());
    std::fill(velocity.begin(), velocity.end(), V3());
  }
  void validate() const {
    if (std::min(dims.x, std::min(dims.y, dims.z)) < 4)
      throw std::invalid_argument("MpmGrid: dims must be >= 4 per axis");
    if (h <= 0.0) throw std::invalid_argument("MpmGrid: cell length must be > 0");
  }
};

struct SoftState {  // mpm.hpp:111-145
  std::vector<Particle> particles;
  std::vector<Material> materials;
  MpmGrid grid;
  V3 gravity{0, 0, -9.81};
  double dt = 5e-4;
  double cfl_factor = 0.4;
  int max_cfl_halvings = 4;
  double lost_fraction_threshold = 0.01;
  std::vector<V3> ext_force;
  std::vector<std::uint8_t> lost;
  std::size_t lost_count = 0;
  struct Scratch {
    std::vector<I3> base;
    std::vector<std::array<std::array<double, 3>, 3>> w;
    std::vector<M3> affine, stress;
    std::vector<int> cell_start, cell_particles;
    std::vector<std::size_t> active_nodes;
  } scratch;
  void init_buffers() {
    grid.allocate();
    ext_force.assign(particles.size(), V3());
    lost.assign(particles.size(), 0);
    lost_count = 0;
  }
  const Material& material_of(const Particle& p) const { return materials.at(p.material); }
};

// mpm.hpp:152-161
inline M3 kirchhoff_stress(const M3& F, const Material& m) {
  if (!(F.determinant() > 0.0)) throw std::invalid_argument("kirchhoff_stress: det(F) must be > 0");
  Svd3 s = svd3(F);
  V3 eps(std::log(s.s.x), std::log(s.s.y), std::log(s.s.z));
  double tr = eps.x + eps.y + eps.z;
  V3 principal = 2.0 * m.mu() * eps + V3(1, 1, 1) * (m.lambda() * tr);
  return s.U * M3::diag(principal) * s.U.transpose();
}

// mpm.hpp:166-181
inline M3 von_mises_return_map(const M3& F_trial, const Material& m) {
  if (!(F_trial.determinant() > 0.0))
    throw std::invalid_argument("von_mises_return_map: det(F) must be > 0");
  Svd3 s = svd3(F_trial);
  V3 eps(std::log(s.s.x), std::log(s.s.y), std::log(s.s.z));
  double mean = (eps.x + eps.y + eps.z) / 3.0;
  V3 dev = eps - V3(mean, mean, mean);
  double dev_norm = dev.norm();
  double stress_dev_norm = 2.0 * m.mu() * dev_norm;
  double threshold = std::sqrt(2.0 / 3.0) * m.yield_stress;
  if (stress_dev_norm <= threshold) return F_trial;
  V3 eps_proj = V3(mean, mean, mean) + dev * (threshold / stress_dev_norm);
  V3 sig_proj(std::exp(eps_proj.x), std::exp(eps_proj.y), std::exp(eps_proj.z));
  return s.U * M3::diag(sig_proj) * s.V.transpose();
}

// ---- north_star materials (no reference implementation: parity unpinned) ----

// Fixed-corotated elasticity (Stomakhin et al. 2012): P = 2 mu (F - R) + lambda (J - 1) J F^-T,
// tau = P F^T = 2 mu (F - R) F^T + lambda (J - 1) J I, R from the polar decomposition.
inline M3 kirchhoff_fixed_corotated(const M3& F, const Material& m) {
  const double J = F.determinant();
  if (!(J > 0.0)) throw std::invalid_argument("kirchhoff_stress: det(F) must be > 0");
  Svd3 s = svd3(F);
  M3 R = s.U * s.V.transpose();
  return 2.0 * m.mu() * ((F - R) * F.transpose()) + M3::Identity() * (m.lambda() * (J - 1.0) * J);
}

// Drucker-Prager sand (Klar et al. 2016, sec. 7.3.1): Hencky elasticity and a
// projection of the log strain onto the cone; q accumulates the plastic strain.
inline M3 drucker_prager_return_map(const M3& F_trial, const Material& m, double& q) {
  if (!(F_trial.determinant() > 0.0))
    throw std::invalid_argument("von_mises_return_map: det(F) must be > 0");
  Svd3 s = svd3(F_trial);
  V3 eps(std::log(s.s.x), std::log(s.s.y), std::log(s.s.z));
  const double tr = eps.x + eps.y + eps.z;
  V3 dev = eps - V3(tr / 3.0, tr / 3.0, tr / 3.0);
  const double dn = dev.norm();
  if (dn == 0.0 || tr > 0.0) {  // tension: project to the tip (sigma = 1)
    q += eps.norm();
    return s.U * s.V.transpose();
  }
  const double dgamma = dn + (3.0 * m.lambda() + 2.0 * m.mu()) / (2.0 * m.mu()) * tr * m.dp_alpha();
  if (dgamma <= 0.0) return F_trial;
  q += dgamma;
  V3 e = eps - dev * (dgamma / dn);
  return s.U * M3::diag(V3(std::exp(e.x), std::exp(e.y), std::exp(e.z))) * s.V.transpose();
}

// Weakly compressible J-only fluid: linear equation of state on the tracked
// volume ratio, Cauchy sigma = K (J - 1) I, Kirchhoff tau = J sigma =
// K (J - 1) J I; F carries no shear (kept I). (MLS-MPM's mpm88 example drops
// the J factor, tau ~ E (J - 1); this model keeps it, so the two agree only to
// first order in J - 1. No reference implementation pins either.)
inline M3 kirchhoff_fluid(double J, const Material& m) { return M3::Identity() * (m.bulk() * (J - 1.0) * J); }

// Kirchhoff stress of particle p by its material model (P2G, mpm.hpp:235-237).
inline M3 kirchhoff_of(const Particle& p, const Material& m) {
  switch (m.model) {
    case Model::FixedCorotated: return kirchhoff_fixed_corotated(p.F, m);
    case Model::Fluid: return kirchhoff_fluid(p.jp, m);
    default: return kirchhoff_stress(p.F, m);  // Hencky (von Mises and Drucker-Prager)
  }
}

// F / J update after G2P by material model (mpm.hpp:367-373 for von Mises).
inline void plasticity_update(Particle& p, const Material& m, double dt) {
  const M3 f_trial = (M3::Identity() + dt * p.C) * p.F;
  switch (m.model) {
    case Model::HenckyVonMises: p.F = von_mises_return_map(f_trial, m); break;
    case Model::FixedCorotated: p.F = f_trial; break;
    case Model::DruckerPrager: p.F = drucker_prager_return_map(f_trial, m, p.jp); break;
    case Model::Fluid: p.jp *= 1.0 + dt * (p.C.m[0][0] + p.C.m[1][1] + p.C.m[2][2]); break;
  }
}

// Initial jp of an uploaded particle (and F of a fluid particle: J carries it).
inline void init_model_state(Particle& p, const Material& m) {
  if (m.model == Model::Fluid) {
    p.jp = p.F.determinant();
    p.F = M3::Identity();
  } else {
    p.jp = m.model == Model::DruckerPrager ? 0.0 : 1.0;
  }
}

namespace detail {
// mpm.hpp:188-193
inline void bspline_weights(double fx, std::array<double, 3>& w) {
  w[0] = 0.5 * (1.5 - fx) * (1.5 - fx);
  w[1] = 0.75 - (fx - 1.0) * (fx - 1.0);
  w[2] = 0.5 * (fx - 0.5) * (fx - 0.5);
}
}  // namespace detail

// mpm.hpp:199-311
inline void p2g(SoftState& st) {
  MpmGrid& g = st.grid;
  const double inv_h = 1.0 / g.h;
  const double d_inv = 4.0 * inv_h * inv_h;
  const std::size_t n = st.particles.size();
  auto& sc = st.scratch;
  sc.base.resize(n);
  sc.w.resize(n);
  sc.affine.resize(n);
  sc.stress.resize(n);
  const I3 bins{g.dims.x - 2, g.dims.y - 2, g.dims.z - 2};
  const std::size_t bin_count = std::size_t(bins.x) * bins.y * bins.z;

  std::vector<std::uint8_t> newly_lost(n, 0);
  parallel_for(std::int64_t(n), [&](std::int64_t ip) {  // :216-238
    Particle& p = st.particles[ip];
    if (st.lost[ip]) {
      sc.base[ip] = I3{-10, -10, -10};
      return;
    }
    V3 local = (p.x - g.origin) * inv_h;
    I3 base{int(std::floor(local.x - 0.5)), int(std::floor(local.y - 0.5)),
            int(std::floor(local.z - 0.5))};
    if (base.x < 0 || base.y < 0 || base.z < 0 || base.x > g.dims.x - 3 ||
        base.y > g.dims.y - 3 || base.z > g.dims.z - 3) {
      newly_lost[ip] = 1;
      sc.base[ip] = I3{-10, -10, -10};
      return;
    }
    sc.base[ip] = base;
    for (int ax = 0; ax < 3; ++ax) detail::bspline_weights(local[ax] - base[ax], sc.w[ip][ax]);
    M3 tau = kirchhoff_of(p, st.material_of(p));
    sc.affine[ip] = p.mass * p.C;
    sc.stress[ip] = -(d_inv * p.volume0) * tau;
  });
  for (std::size_t ip = 0; ip < n; ++ip) {  // :239-245
    if (newly_lost[ip] && !st.lost[ip]) {
      st.lost[ip] = 1;
      st.particles[ip].v = V3();
      ++st.lost_count;
    }
  }
  if (!st.particles.empty() &&
      double(st.lost_count) / double(n) > st.lost_fraction_threshold)  // :246-249
    throw SimulationDiverged("lost particle fraction exceeds threshold");

  sc.cell_start.assign(bin_count + 1, 0);  // :251-264
  auto bin_of = [&](const I3& b) { return (std::size_t(b.z) * bins.y + b.y) * bins.x + b.x; };
  for (std::size_t ip = 0; ip < n; ++ip)
    if (!st.lost[ip]) ++sc.cell_start[bin_of(sc.base[ip]) + 1];
  for (std::size_t c = 0; c < bin_count; ++c) sc.cell_start[c + 1] += sc.cell_start[c];
  sc.cell_particles.resize(sc.cell_start[bin_count]);
  {
    std::vector<int> cursor(sc.cell_start.begin(), sc.cell_start.end() - 1);
    for (std::size_t ip = 0; ip < n; ++ip)
      if (!st.lost[ip]) sc.cell_particles[cursor[bin_of(sc.base[ip])]++] = int(ip);
  }

  std::vector<std::uint8_t> node_active(g.node_count(), 0);  // :266-280
  for (std::size_t c = 0; c < bin_count; ++c) {
    if (sc.cell_start[c] == sc.cell_start[c + 1]) continue;
    int bx = int(c % bins.x);
    int by = int((c / bins.x) % bins.y);
    int bz = int(c / (std::size_t(bins.x) * bins.y));
    for (int dk = 0; dk < 3; ++dk)
      for (int dj = 0; dj < 3; ++dj)
        for (int di = 0; di < 3; ++di) node_active[g.node_index(bx + di, by + dj, bz + dk)] = 1;
  }
  sc.active_nodes.clear();
  for (std::size_t i = 0; i < node_active.size(); ++i)
    if (node_active[i]) sc.active_nodes.push_back(i);

  parallel_for(std::int64_t(sc.active_nodes.size()), [&](std::int64_t a) {  // :284-310
    std::size_t ni = sc.active_nodes[a];
    int i = int(ni % g.dims.x);
    int j = int((ni / g.dims.x) % g.dims.y);
    int k = int(ni / (std::size_t(g.dims.x) * g.dims.y));
    V3 xi = g.node_pos(i, j, k);
    double m_acc = 0.0;
    V3 mom_acc, f_acc;
    for (int bz = std::max(k - 2, 0); bz <= std::min(k, bins.z - 1); ++bz)
      for (int by = std::max(j - 2, 0); by <= std::min(j, bins.y - 1); ++by)
        for (int bx = std::max(i - 2, 0); bx <= std::min(i, bins.x - 1); ++bx) {
          std::size_t c = (std::size_t(bz) * bins.y + by) * bins.x + bx;
          for (int s = sc.cell_start[c]; s < sc.cell_start[c + 1]; ++s) {
            int ip = sc.cell_particles[s];
            const Particle& p = st.particles[ip];
            double w = sc.w[ip][0][i - bx] * sc.w[ip][1][j - by] * sc.w[ip][2][k - bz];
            V3 dpos = xi - p.x;
            m_acc += w * p.mass;
            mom_acc += w * (p.mass * p.v + sc.affine[ip] * dpos);
            f_acc += w * (sc.stress[ip] * dpos + st.ext_force[ip]);
          }
        }
    g.mass[ni] = m_acc;
    g.momentum[ni] = mom_acc;
    g.force[ni] = f_acc;
  });
}

// mpm.hpp:315-342
inline void grid_update(SoftState& st) {
  MpmGrid& g = st.grid;
  const int bw = MpmGrid::kBoundaryWidth;
  parallel_for(std::int64_t(st.scratch.active_nodes.size()), [&](std::int64_t a) {
    std::size_t ni = st.scratch.active_nodes[a];
    if (g.mass[ni] <= 0.0) return;
    V3 v = g.momentum[ni] / g.mass[ni] + st.dt * (st.gravity + g.force[ni] / g.mass[ni]);
    int i = int(ni % g.dims.x);
    int j = int((ni / g.dims.x) % g.dims.y);
    int k = int(ni / (std::size_t(g.dims.x) * g.dims.y));
    const int idx[3] = {i, j, k};
    for (int ax = 0; ax < 3; ++ax) {
      if (idx[ax] < bw) {
        if (g.boundary[2 * ax] == BoundaryKind::Sticky)
          v = V3();
        else if (v[ax] < 0.0)
          v[ax] = 0.0;
      }
      if (idx[ax] >= g.dims[ax] - bw) {
        if (g.boundary[2 * ax + 1] == BoundaryKind::Sticky)
          v = V3();
        else if (v[ax] > 0.0)
          v[ax] = 0.0;
      }
    }
    g.velocity[ni] = v;
  });
}

// mpm.hpp:346-379
inline void g2p_advect(SoftState& st) {
  MpmGrid& g = st.grid;
  const double inv_h = 1.0 / g.h;
  const double d_inv = 4.0 * inv_h * inv_h;
  auto& sc = st.scratch;
  std::vector<std::int64_t> bad(st.particles.size(), 0);
  parallel_for(std::int64_t(st.particles.size()), [&](std::int64_t ip) {
    if (st.lost[ip]) return;
    Particle& p = st.particles[ip];
    const I3& base = sc.base[ip];
    V3 v_new;
    M3 c_new;
    for (int dk = 0; dk < 3; ++dk)
      for (int dj = 0; dj < 3; ++dj)
        for (int di = 0; di < 3; ++di) {
          double w = sc.w[ip][0][di] * sc.w[ip][1][dj] * sc.w[ip][2][dk];
          std::size_t ni = g.node_index(base.x + di, base.y + dj, base.z + dk);
          V3 dpos = g.node_pos(base.x + di, base.y + dj, base.z + dk) - p.x;
          v_new += w * g.velocity[ni];
          c_new = c_new + M3::outer(g.velocity[ni], dpos) * (w * d_inv);
        }
    p.v = v_new;
    p.C = c_new;
    p.x += st.dt * p.v;
    if (st.dt != 0.0) plasticity_update(p, st.material_of(p), st.dt);
    if (!p.x.allFinite() || !p.v.allFinite() || !p.F.allFinite()) bad[ip] = 1;
  });
  for (std::size_t ip = 0; ip < bad.size(); ++ip)
    if (bad[ip]) throw SimulationDiverged("NaN/Inf in particle " + std::to_string(ip));
}

using ParticleForceHook = std::function<void(SoftState&)>;  // mpm.hpp:383
using GridForceHook = std::function<void(SoftState&)>;      // mpm.hpp:384

// mpm.hpp:386-391
inline double max_particle_speed(const SoftState& st) {
  double vmax = 0.0;
  for (std::size_t ip = 0; ip < st.particles.size(); ++ip)
    if (!st.lost[ip]) vmax = std::max(vmax, st.particles[ip].v.norm());
  return vmax;
}

// mpm.hpp:397-421
inline int soft_substep(SoftState& st, const ParticleForceHook& particle_hook = nullptr,
                        const GridForceHook& grid_hook = nullptr) {
  int halvings = 0;
  double vmax = max_particle_speed(st);
  while (halvings < st.max_cfl_halvings && vmax * st.dt / (1 << halvings) > st.cfl_factor * st.grid.h)
    ++halvings;
  if (vmax * st.dt / (1 << halvings) > st.cfl_factor * st.grid.h)
    throw SimulationDiverged("CFL violation persists after max substep halvings");
  int cycles = 1 << halvings;
  double dt_full = st.dt;
  st.dt = dt_full / cycles;
  try {
    for (int c = 0; c < cycles; ++c) {
      st.grid.clear();
      std::fill(st.ext_force.begin(), st.ext_force.end(), V3());
      if (particle_hook) particle_hook(st);
      p2g(st);
      if (grid_hook) grid_hook(st);
      grid_update(st);
      g2p_advect(st);
    }
  } catch (...) {
    st.dt = dt_full;
    throw;
  }
  st.dt = dt_full;
  return cycles;
}

// ---------------------------------------------------------------------------
// Seeding: seeding.hpp:13-46 (same std::mt19937_64 + uniform_real_distribution,
// so inputs are bit-identical to the reference's under libstdc++).
inline void seed_particles_box(SoftState& st, const V3& box_min, const V3& box_max,
                               int material_id, double particle_volume, std::mt19937_64& rng) {
  const Material& mat = st.materials.at(material_id);
  double spacing = std::cbrt(particle_volume);
  std::uniform_real_distribution<double> jitter(-0.25 * spacing, 0.25 * spacing);
  V3 span = box_max - box_min;
  int counts[3];
  for (int ax = 0; ax < 3; ++ax) counts[ax] = std::max(1, int(std::floor(span[ax] / spacing)));
  for (int k = 0; k < counts[2]; ++k)
    for (int j = 0; j < counts[1]; ++j)
      for (int i = 0; i < counts[0]; ++i) {
        V3 p = box_min + spacing * (V3(i, j, k) + V3(0.5, 0.5, 0.5));
        // Vec3(jitter(rng), jitter(rng), jitter(rng)) (seeding.hpp:26): the
        // argument order is unspecified in C++; GCC evaluates right to left,
        // so the z jitter is drawn first. Reproduced for bit-identical inputs.
        double jz = jitter(rng);
        double jy = jitter(rng);
        double jx = jitter(rng);
        p += V3(jx, jy, jz);
        Particle pt;
        pt.x = V3(std::min(std::max(p.x, box_min.x), box_max.x),
                  std::min(std::max(p.y, box_min.y), box_max.y),
                  std::min(std::max(p.z, box_min.z), box_max.z));
        pt.volume0 = particle_volume;
        pt.mass = mat.density * particle_volume;
        pt.material = material_id;
        st.particles.push_back(pt);
      }
}
inline std::size_t lattice_count(const V3& box_min, const V3& box_max, double particle_volume) {
  double spacing = std::cbrt(particle_volume);
  V3 span = box_max - box_min;
  std::size_t n = 1;
  for (int ax = 0; ax < 3; ++ax) n *= std::size_t(std::max(1, int(std::floor(span[ax] / spacing))));
  return n;
}

// ---------------------------------------------------------------------------
// SDF: sdf.hpp:22-201.

struct SdfVolume {  // sdf.hpp:22-63
  V3 origin;
  double voxel = 0.01;
  I3 dims{0, 0, 0};
  std::vector<float> samples;
  double at(int i, int j, int k) const {
    return samples[std::size_t(k * dims.y + j) * dims.x + i];
  }
  double interpolate(const V3& p) const {
    V3 local = (p - origin) / voxel;
    V3 cl(std::min(std::max(local.x, 0.0), dims.x - 1.0), std::min(std::max(local.y, 0.0), dims.y - 1.0),
          std::min(std::max(local.z, 0.0), dims.z - 1.0));
    double outside = voxel * (local - cl).norm();
    int i0 = std::min(int(cl.x), dims.x - 2);
    int j0 = std::min(int(cl.y), dims.y - 2);
    int k0 = std::min(int(cl.z), dims.z - 2);
    double fx = cl.x - i0, fy = cl.y - j0, fz = cl.z - k0;
    double c00 = at(i0, j0, k0) * (1 - fx) + at(i0 + 1, j0, k0) * fx;
    double c10 = at(i0, j0 + 1, k0) * (1 - fx) + at(i0 + 1, j0 + 1, k0) * fx;
    double c01 = at(i0, j0, k0 + 1) * (1 - fx) + at(i0 + 1, j0, k0 + 1) * fx;
    double c11 = at(i0, j0 + 1, k0 + 1) * (1 - fx) + at(i0 + 1, j0 + 1, k0 + 1) * fx;
    double c0 = c00 * (1 - fy) + c10 * fy;
    double c1 = c01 * (1 - fy) + c11 * fy;
    return c0 * (1 - fz) + c1 * fz + outside;
  }
};

enum class ShapeType { Plane = 0, Sphere = 1, Box = 2, Capsule = 3, Volume = 4 };

struct Shape {  // sdf.hpp:87-110
  ShapeType type = ShapeType::Sphere;
  V3 normal{0, 0, 1};
  double offset = 0.0;        // plane
  double radius = 0.1;        // sphere / capsule
  V3 half_extents{0.1, 0.1, 0.1};
  double half_length = 0.1;   // capsule
  std::shared_ptr<const SdfVolume> volume;
  Pose local_pose;
  double friction = 0.5, k_n = 1e3, k_t = 10.0;
};

namespace detail {
// sdf.hpp:114-135
inline double sdf_local(const Shape& g, const V3& p) {
  switch (g.type) {
    case ShapeType::Plane: return g.normal.dot(p) - g.offset;
    case ShapeType::Sphere: return p.norm() - g.radius;
    case ShapeType::Box: {
      V3 q(std::abs(p.x) - g.half_extents.x, std::abs(p.y) - g.half_extents.y,
           std::abs(p.z) - g.half_extents.z);
      double outside = V3(std::max(q.x, 0.0), std::max(q.y, 0.0), std::max(q.z, 0.0)).norm();
      double inside = std::min(std::max(q.x, std::max(q.y, q.z)), 0.0);
      return outside + inside;
    }
    case ShapeType::Capsule: {
      V3 q(p.x, p.y, p.z - std::clamp(p.z, -g.half_length, g.half_length));
      return q.norm() - g.radius;
    }
    case ShapeType::Volume: return g.volume->interpolate(p);
  }
  return 0.0;
}
// sdf.hpp:139-179
inline V3 sdf_gradient_local(const Shape& g, const V3& p) {
  const V3 tie_break(1, 0, 0);
  switch (g.type) {
    case ShapeType::Plane: return g.normal;
    case ShapeType::Sphere: {
      double n = p.norm();
      return n < 1e-12 ? tie_break : p / n;
    }
    case ShapeType::Box: {
      V3 q(std::abs(p.x) - g.half_extents.x, std::abs(p.y) - g.half_extents.y,
           std::abs(p.z) - g.half_extents.z);
      V3 sign(p.x < 0 ? -1.0 : 1.0, p.y < 0 ? -1.0 : 1.0, p.z < 0 ? -1.0 : 1.0);
      V3 qpos(std::max(q.x, 0.0), std::max(q.y, 0.0), std::max(q.z, 0.0));
      double outside = qpos.norm();
      if (outside > 1e-12) return V3(sign.x * qpos.x, sign.y * qpos.y, sign.z * qpos.z) / outside;
      int ax = 0;
      for (int k = 1; k < 3; ++k)
        if (q[k] > q[ax]) ax = k;
      V3 n;
      n[ax] = sign[ax];
      return n;
    }
    case ShapeType::Capsule: {
      V3 q(p.x, p.y, p.z - std::clamp(p.z, -g.half_length, g.half_length));
      double n = q.norm();
      return n < 1e-12 ? tie_break : q / n;
    }
    case ShapeType::Volume: {
      double h = 0.5 * g.volume->voxel;
      V3 grad;
      for (int k = 0; k < 3; ++k) {
        V3 dp;
        dp[k] = h;
        grad[k] = (g.volume->interpolate(p + dp) - g.volume->interpolate(p - dp)) / (2 * h);
      }
      double n = grad.norm();
      return n < 1e-12 ? tie_break : grad / n;
    }
  }
  return tie_break;
}
}  // namespace detail

// sdf.hpp:185-201
inline double sdf_eval(const Shape& s, const Pose& world, const V3& p) {
  return detail::sdf_local(s, inverse(world).apply(p));
}
inline double sdf_eval(const Shape& s, const V3& p) { return sdf_eval(s, s.local_pose, p); }
inline V3 sdf_gradient(const Shape& s, const Pose& world, const V3& p) {
  V3 local = detail::sdf_gradient_local(s, inverse(world).apply(p));
  return world.rotation * local;
}
inline V3 sdf_gradient(const Shape& s, const V3& p) { return sdf_gradient(s, s.local_pose, p); }

// ---------------------------------------------------------------------------
// Rigid layer: rigid.hpp:11-66.

enum class BodyMode : std::uint8_t { Dynamic = 0, Kinematic = 1, Scripted = 2 };

struct WrenchBuffer {  // rigid.hpp:15-23
  V3 force, torque;
  void reset() { force = V3(); torque = V3(); }
};

struct RigidBody {  // rigid.hpp:25-43
  Pose pose;
  V3 linear_velocity, angular_velocity;
  double mass = 1.0;
  V3 inertia{1e-3, 1e-3, 1e-3};
  V3 com_offset;
  std::vector<Shape> shapes;
  BodyMode mode = BodyMode::Kinematic;
  V3 world_com() const { return pose.apply(com_offset); }
  void validate() const {
    if (mode == BodyMode::Dynamic &&
        (mass <= 0.0 || std::min(inertia.x, std::min(inertia.y, inertia.z)) <= 0.0))
      throw std::invalid_argument("RigidBody: dynamic body needs positive mass and inertia");
  }
};

// rigid.hpp:52-66
inline void integrate_free_body(RigidBody& b, const WrenchBuffer& w, const V3& gravity, double dt) {
  if (b.mode != BodyMode::Dynamic) return;
  b.linear_velocity += dt * (gravity + w.force / b.mass);
  M3 rot = b.pose.rotation.toRotationMatrix();
  M3 inertia_w = rot * M3::diag(b.inertia) * rot.transpose();
  V3 ang_mom = inertia_w * b.angular_velocity;
  b.angular_velocity += dt * (inertia_w.inverse() * (w.torque - b.angular_velocity.cross(ang_mom)));
  V3 com = b.world_com();
  V3 com_new = com + dt * b.linear_velocity;
  Quat dq = quat_exp(b.angular_velocity * dt);
  Quat rot_new = (dq * b.pose.rotation).normalized();
  b.pose = Pose(rot_new, com_new - rot_new * b.com_offset);
}

// Harness extension (not in the reference): a scripted kinematic body moves
// with its own constant twist, the pose update of integrate_free_body with
// no velocity change. Stands in for robot-driven links (rigid.hpp:142-151).
inline void advance_scripted_body(RigidBody& b, double dt) {
  if (b.mode != BodyMode::Scripted) return;
  V3 com = b.world_com();
  V3 com_new = com + dt * b.linear_velocity;
  Quat dq = quat_exp(b.angular_velocity * dt);
  Quat rot_new = (dq * b.pose.rotation).normalized();
  b.pose = Pose(rot_new, com_new - rot_new * b.com_offset);
}

// geometry.hpp:89-96
inline V3 quat_log(const Quat& q_in) {
  Quat q = q_in.normalized();
  if (q.w < 0.0) q = Quat(-q.w, -q.x, -q.y, -q.z);
  const double vn = q.vec().norm();
  if (vn < 1e-14) return 2.0 * q.vec();
  const double ang = 2.0 * std::atan2(vn, q.w);
  return (ang / vn) * q.vec();
}

// Robot::set_kinematic_pose (rigid.hpp:142-151): a kinematic link jumps to its
// target pose; its twist is the finite difference over the rigid step.
inline void set_kinematic_pose(RigidBody& b, const Pose& target, double dt) {
  if (dt > 0.0) {
    b.linear_velocity = (target.translation - b.pose.translation) / dt;
    b.angular_velocity = quat_log(target.rotation * b.pose.rotation.conjugate()) / dt;
  } else {
    b.linear_velocity = V3();
    b.angular_velocity = V3();
  }
  b.pose = target;
}

// ---------------------------------------------------------------------------
// Coupling: coupling.hpp:18-294 (bodies only; the robot/controller caller
// part of env_step is out of scope).

enum class CouplingMode : std::uint8_t { Particle = 0, Grid = 1 };

struct CouplingConfig {  // coupling.hpp:20-26
  CouplingMode mode = CouplingMode::Particle;
  double r_c_factor = 0.5;
  double c_d = 10.0;
  double contact_radius(double h) const { return r_c_factor * h; }
};

struct BodyMirror {  // coupling.hpp:29-39
  Pose pose;
  V3 linear_velocity, angular_velocity, com;
  const std::vector<Shape>* shapes = nullptr;
  V3 point_velocity(const V3& p) const { return linear_velocity + angular_velocity.cross(p - com); }
};

struct StepReport {  // coupling.hpp:41-50
  int rigid_steps = 0, soft_substeps = 0, cfl_cycles = 0;
  double max_penetration = 0.0, max_force_balance_error = 0.0;
  std::size_t lost_particles = 0;
};

struct World {  // coupling.hpp:54-118
  std::vector<RigidBody> bodies;
  SoftState soft;
  CouplingConfig coupling;
  V3 rigid_gravity{0, 0, -9.81};
  int n_rigid = 25, n_soft = 1;
  double time = 0.0;
  std::vector<BodyMirror> mirrors;
  std::vector<WrenchBuffer> wrenches, pending_wrenches;
  double mean_particle_mass = 0.0;
  // Harness: per-rigid-step target poses of kinematic bodies for the next
  // env_step ([step][body][qw qx qy qz tx ty tz]), applied like robot-driven
  // links (coupling.hpp:252-258 -> rigid.hpp:142-151); consumed by one env_step.
  std::vector<double> schedule;
  std::vector<std::uint8_t> sched_mask;
  int sched_steps = 0;
  double dt_rigid() const { return n_soft * soft.dt; }
  void init() {
    if (n_rigid < 1 || n_soft < 1) throw std::invalid_argument("World: n_rigid and n_soft must be >= 1");
    for (const RigidBody& b : bodies) b.validate();
    soft.init_buffers();
    mean_particle_mass = 0.0;
    for (const Particle& p : soft.particles) mean_particle_mass += p.mass;
    if (!soft.particles.empty()) mean_particle_mass /= double(soft.particles.size());
    mirrors.resize(bodies.size());
    wrenches.assign(bodies.size(), WrenchBuffer{});
    pending_wrenches.assign(bodies.size(), WrenchBuffer{});
    sync_rigid_to_soft();
  }
  void sync_rigid_to_soft() {  // coupling.hpp:106-117
    for (std::size_t i = 0; i < mirrors.size(); ++i) {
      const RigidBody& b = bodies[i];
      BodyMirror& m = mirrors[i];
      m.pose = b.pose;
      m.linear_velocity = b.linear_velocity;
      m.angular_velocity = b.angular_velocity;
      m.com = b.world_com();
      m.shapes = &b.shapes;
      wrenches[i].reset();
    }
  }
};

namespace detail {
// coupling.hpp:125-144
inline bool penalty_point_force(const Shape& shape, const Pose& shape_pose, const V3& x,
                                const V3& v_point, const BodyMirror& m, double r_c, double c_d,
                                V3& force, double& penetration) {
  double phi = sdf_eval(shape, shape_pose, x);
  if (phi >= r_c) return false;
  V3 n = sdf_gradient(shape, shape_pose, x);
  V3 f = shape.k_n * (r_c - phi) * n;
  V3 v_rel = v_point - m.point_velocity(x);
  double vn = v_rel.dot(n);
  f += -c_d * std::min(0.0, vn) * n;
  V3 v_t = v_rel - vn * n;
  double vt_norm = v_t.norm();
  if (vt_norm > 1e-12) {
    double cap = std::min(shape.friction * shape.k_n * (r_c - phi), shape.k_t * vt_norm);
    f -= cap * (v_t / vt_norm);
  }
  force = f;
  penetration = std::max(0.0, -phi);
  return true;
}
}  // namespace detail

// coupling.hpp:151-172
inline void penalty_particle(World& w, double* max_penetration = nullptr) {
  SoftState& st = w.soft;
  const double r_c = w.coupling.contact_radius(st.grid.h);
  for (std::size_t ip = 0; ip < st.particles.size(); ++ip) {
    if (st.lost[ip]) continue;
    const Particle& p = st.particles[ip];
    for (std::size_t bi = 0; bi < w.mirrors.size(); ++bi) {
      const BodyMirror& m = w.mirrors[bi];
      for (const Shape& s : *m.shapes) {
        Pose sp = compose(m.pose, s.local_pose);
        V3 f;
        double pen;
        if (!detail::penalty_point_force(s, sp, p.x, p.v, m, r_c, w.coupling.c_d, f, pen)) continue;
        st.ext_force[ip] += f;
        w.wrenches[bi].force -= f;
        w.wrenches[bi].torque += (p.x - m.com).cross(-f);
        if (max_penetration) *max_penetration = std::max(*max_penetration, pen);
      }
    }
  }
}

// coupling.hpp:182-184
inline double grid_contact_radius(const CouplingConfig& c, double h) {
  return std::max(c.contact_radius(h), 0.65 * h);
}

// coupling.hpp:186-214
inline void penalty_grid(World& w, double* max_penetration = nullptr) {
  SoftState& st = w.soft;
  MpmGrid& g = st.grid;
  const double r_c = grid_contact_radius(w.coupling, g.h);
  for (std::size_t a = 0; a < st.scratch.active_nodes.size(); ++a) {
    std::size_t ni = st.scratch.active_nodes[a];
    if (g.mass[ni] <= 0.0) continue;
    int i = int(ni % g.dims.x);
    int j = int((ni / g.dims.x) % g.dims.y);
    int k = int(ni / (std::size_t(g.dims.x) * g.dims.y));
    V3 xi = g.node_pos(i, j, k);
    V3 vi = g.momentum[ni] / g.mass[ni];
    double scale = w.mean_particle_mass > 0.0 ? g.mass[ni] / w.mean_particle_mass : 1.0;
    for (std::size_t bi = 0; bi < w.mirrors.size(); ++bi) {
      const BodyMirror& m = w.mirrors[bi];
      for (const Shape& s : *m.shapes) {
        Pose sp = compose(m.pose, s.local_pose);
        V3 f;
        double pen;
        if (!detail::penalty_point_force(s, sp, xi, vi, m, r_c, w.coupling.c_d, f, pen)) continue;
        f *= scale;
        g.force[ni] += f;
        w.wrenches[bi].force -= f;
        w.wrenches[bi].torque += (xi - m.com).cross(-f);
        if (max_penetration) *max_penetration = std::max(*max_penetration, pen);
      }
    }
  }
}

// The body/soft part of env_step: coupling.hpp:248-293. Controller and robot
// (coupling.hpp:225-246, :252-258) are out of scope; scripted bodies stand in
// for robot links and are advanced where robot_drive_step would run.
inline StepReport env_step(World& w) {
  StepReport rep;
  const double dt_r = w.dt_rigid();
  if (w.sched_steps > 0 && w.sched_steps != w.n_rigid)
    throw std::invalid_argument("kinematic schedule length != n_rigid");
  struct Consume {  // a schedule drives exactly one env step
    World& w;
    ~Consume() { w.sched_steps = 0; w.schedule.clear(); }
  } consume{w};
  for (int r = 0; r < w.n_rigid; ++r) {
    for (std::size_t i = 0; i < w.bodies.size(); ++i)
      integrate_free_body(w.bodies[i], w.pending_wrenches[i], w.rigid_gravity, dt_r);
    for (std::size_t i = 0; i < w.bodies.size(); ++i) advance_scripted_body(w.bodies[i], dt_r);
    if (w.sched_steps > 0)
      for (std::size_t i = 0; i < w.bodies.size(); ++i) {
        if (!w.sched_mask[i]) continue;
        const double* p = w.schedule.data() + 7 * (std::size_t(r) * w.bodies.size() + i);
        set_kinematic_pose(w.bodies[i], Pose(Quat(p[0], p[1], p[2], p[3]), V3(p[4], p[5], p[6])), dt_r);
      }
    w.sync_rigid_to_soft();
    for (int s = 0; s < w.n_soft; ++s) {
      auto wrench_sum = [&] {
        V3 acc;
        for (const WrenchBuffer& b : w.wrenches) acc += b.force;
        return acc;
      };
      auto particle_hook = [&](SoftState& st) {
        if (w.coupling.mode != CouplingMode::Particle) return;
        V3 before = wrench_sum();
        penalty_particle(w, &rep.max_penetration);
        V3 applied;
        for (const V3& f : st.ext_force) applied += f;
        rep.max_force_balance_error =
            std::max(rep.max_force_balance_error, (wrench_sum() - before + applied).norm());
      };
      auto grid_hook = [&](SoftState& st) {
        if (w.coupling.mode != CouplingMode::Grid) return;
        V3 before = wrench_sum();
        std::vector<V3> f0 = st.grid.force;
        penalty_grid(w, &rep.max_penetration);
        V3 applied;
        for (std::size_t ni : st.scratch.active_nodes) applied += st.grid.force[ni] - f0[ni];
        rep.max_force_balance_error =
            std::max(rep.max_force_balance_error, (wrench_sum() - before + applied).norm());
      };
      rep.cfl_cycles += soft_substep(w.soft, particle_hook, grid_hook);
      ++rep.soft_substeps;
    }
    w.pending_wrenches = w.wrenches;
    ++rep.rigid_steps;
  }
  w.time += w.n_rigid * w.n_soft * w.soft.dt;
  rep.lost_particles = w.soft.lost_count;
  return rep;
}

// coupling.hpp:299-310
inline std::uint64_t fnv1a(const void* data, std::size_t n, std::uint64_t h = 1469598103934665603ull) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace oracle
