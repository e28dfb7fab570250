// ORACLE — TEST INFRASTRUCTURE ONLY (see msim_oracle.hpp for the rules).
//
// CPU restatement of the reference's task-side consumers of the soft-body
// state that SURVEY.md §8(f) ranks next after the substep:
//   * mesh SDF baking: point_triangle_distance, ray_hits_triangle,
//     inside_by_parity, bake_mesh_sdf, make_box_mesh (sdf.hpp:203-310, :443-455);
//   * task metrics: RegionBox, DepthMap, metric_fill, render_heightmap,
//     metric_write_iou, NnGrid, chamfer_distance, metric_pinch
//     (scenario.hpp:18-214).
// Pinned by the ports of test_sdf.cpp / test_scenario.cpp known-answer tests
// in kat_oracle.cpp.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

#include "msim_oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------------------
// Mesh baking (sdf.hpp:203-310)

struct Triangle {  // sdf.hpp:206-208
  V3 a, b, c;
};
using TriangleMesh = std::vector<Triangle>;

namespace detail {

// sdf.hpp:214-237 (Ericson's closest point on a triangle)
inline double point_triangle_distance(const V3& p, const Triangle& t) {
  V3 ab = t.b - t.a, ac = t.c - t.a, ap = p - t.a;
  double d1 = ab.dot(ap), d2 = ac.dot(ap);
  if (d1 <= 0 && d2 <= 0) return (p - t.a).norm();
  V3 bp = p - t.b;
  double d3 = ab.dot(bp), d4 = ac.dot(bp);
  if (d3 >= 0 && d4 <= d3) return (p - t.b).norm();
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return (p - (t.a + ab * (d1 / (d1 - d3)))).norm();
  V3 cp = p - t.c;
  double d5 = ab.dot(cp), d6 = ac.dot(cp);
  if (d6 >= 0 && d5 <= d6) return (p - t.c).norm();
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return (p - (t.a + ac * (d2 / (d2 - d6)))).norm();
  double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return (p - (t.b + (t.c - t.b) * w)).norm();
  }
  double denom = 1.0 / (va + vb + vc);
  V3 closest = t.a + ab * (vb * denom) + ac * (vc * denom);
  return (p - closest).norm();
}

// sdf.hpp:239-254 (Moller-Trumbore, hits strictly in front of the origin)
inline bool ray_hits_triangle(const V3& orig, const V3& dir, const Triangle& t) {
  V3 e1 = t.b - t.a, e2 = t.c - t.a;
  V3 pv = dir.cross(e2);
  double det = e1.dot(pv);
  if (std::abs(det) < 1e-14) return false;
  double inv = 1.0 / det;
  V3 tv = orig - t.a;
  double u = tv.dot(pv) * inv;
  if (u < 0.0 || u > 1.0) return false;
  V3 qv = tv.cross(e1);
  double v = dir.dot(qv) * inv;
  if (v < 0.0 || u + v > 1.0) return false;
  double dist = e2.dot(qv) * inv;
  return dist > 0.0;
}

// the three vote directions of sdf.hpp:258-262, normalized
inline std::array<V3, 3> parity_dirs() {
  std::array<V3, 3> d = {V3(1.0, 0.0, 0.0), V3(1.0, 0.137, 0.071), V3(1.0, -0.083, 0.143)};
  for (V3& v : d) v = v / v.norm();
  return d;
}

// sdf.hpp:256-270: majority of three ray-crossing parities
inline bool inside_by_parity(const TriangleMesh& mesh, const V3& p) {
  static const std::array<V3, 3> dirs = parity_dirs();
  int votes = 0;
  for (const V3& d : dirs) {
    int crossings = 0;
    for (const Triangle& t : mesh)
      if (ray_hits_triangle(p, d, t)) ++crossings;
    if (crossings % 2 == 1) ++votes;
  }
  return votes >= 2;
}

}  // namespace detail

// Grid of bake_mesh_sdf (sdf.hpp:277-296): origin, dims; throws like the reference.
inline void bake_grid(const TriangleMesh& mesh, double voxel, double padding, V3& origin, int dims[3]) {
  if (mesh.empty()) throw std::invalid_argument("bake_mesh_sdf: empty mesh");
  if (voxel <= 0.0) throw std::invalid_argument("bake_mesh_sdf: voxel size must be > 0");
  bool degenerate = true;
  V3 lo = mesh[0].a, hi = mesh[0].a;
  for (const Triangle& t : mesh) {
    for (const V3* v : {&t.a, &t.b, &t.c})
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::min(lo[k], (*v)[k]);
        hi[k] = std::max(hi[k], (*v)[k]);
      }
    if ((t.b - t.a).cross(t.c - t.a).norm() > 1e-14) degenerate = false;
  }
  if (degenerate) throw std::invalid_argument("bake_mesh_sdf: mesh has only zero-area triangles");
  origin = lo - V3(padding, padding, padding);
  V3 span = hi - lo + V3(2.0 * padding, 2.0 * padding, 2.0 * padding);
  for (int k = 0; k < 3; ++k) dims[k] = std::max(2, static_cast<int>(std::ceil(span[k] / voxel)) + 1);
}

// bake_mesh_sdf (sdf.hpp:277-310): exact unsigned distance, parity sign, f32 samples x-fastest
inline SdfVolume bake_mesh_sdf(const TriangleMesh& mesh, double voxel, double padding) {
  V3 origin;
  int dims[3];
  bake_grid(mesh, voxel, padding, origin, dims);
  SdfVolume vol;
  vol.voxel = voxel;
  vol.origin = origin;
  vol.dims = I3{dims[0], dims[1], dims[2]};
  vol.samples.resize(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
  std::size_t idx = 0;
  for (int k = 0; k < dims[2]; ++k)
    for (int j = 0; j < dims[1]; ++j)
      for (int i = 0; i < dims[0]; ++i, ++idx) {
        V3 p = vol.origin + voxel * V3(i, j, k);
        double d = std::numeric_limits<double>::max();
        for (const Triangle& t : mesh) d = std::min(d, detail::point_triangle_distance(p, t));
        vol.samples[idx] = static_cast<float>(detail::inside_by_parity(mesh, p) ? -d : d);
      }
  return vol;
}

// make_box_mesh (sdf.hpp:443-455): 12 outward-wound triangles
inline TriangleMesh make_box_mesh(const V3& h, const V3& center = V3::Zero()) {
  std::array<V3, 8> v;
  for (int i = 0; i < 8; ++i)
    v[i] = center + V3((i & 1) ? h.x : -h.x, (i & 2) ? h.y : -h.y, (i & 4) ? h.z : -h.z);
  const int f[12][3] = {{0, 2, 1}, {1, 2, 3}, {4, 5, 6}, {5, 7, 6}, {0, 1, 4}, {1, 5, 4},
                        {2, 6, 3}, {3, 6, 7}, {0, 4, 2}, {2, 4, 6}, {1, 3, 5}, {3, 7, 5}};
  TriangleMesh mesh;
  for (auto& tri : f) mesh.push_back({v[tri[0]], v[tri[1]], v[tri[2]]});
  return mesh;
}

// ---------------------------------------------------------------------------
// Task metrics (scenario.hpp:18-214)

struct RegionBox {  // scenario.hpp:18-30
  V3 min = V3(0, 0, 0);
  V3 max = V3(1, 1, 1);
  bool contains(const V3& p) const {
    return p.x >= min.x && p.y >= min.y && p.z >= min.z && p.x <= max.x && p.y <= max.y && p.z <= max.z;
  }
  void validate() const {
    if (std::min({max.x - min.x, max.y - min.y, max.z - min.z}) <= 0.0)
      throw std::invalid_argument("RegionBox: extents must be positive");
  }
};

struct DepthMap {  // scenario.hpp:35-50
  int nx = 0, ny = 0;
  double cell = 0.0;
  double threshold = 0.0;
  std::vector<double> samples;
  double& at(int i, int j) { return samples[static_cast<std::size_t>(j) * nx + i]; }
  double at(int i, int j) const { return samples[static_cast<std::size_t>(j) * nx + i]; }
  bool occupied(std::size_t idx) const { return samples[idx] < threshold; }
};

struct FillResult {  // scenario.hpp:55-59
  double fraction = 0.0;
  double max_speed = 0.0;
  bool success = false;
};

// metric_fill (scenario.hpp:63-75)
inline FillResult metric_fill(const std::vector<V3>& x, const std::vector<V3>& v, const RegionBox& region) {
  if (x.empty()) throw std::invalid_argument("metric_fill: no particles");
  region.validate();
  FillResult r;
  std::size_t inside = 0;
  for (std::size_t i = 0; i < x.size(); ++i) {
    if (region.contains(x[i])) ++inside;
    r.max_speed = std::max(r.max_speed, v[i].norm());
  }
  r.fraction = static_cast<double>(inside) / static_cast<double>(x.size());
  r.success = r.fraction > 0.9 && r.max_speed < 0.05;
  return r;
}

// render_heightmap (scenario.hpp:79-98)
inline DepthMap render_heightmap(const std::vector<V3>& x, const RegionBox& region, int nx, int ny,
                                 double threshold = 0.0) {
  region.validate();
  if (nx < 2 || ny < 2) throw std::invalid_argument("render_heightmap: resolution must be >= 2x2");
  DepthMap m;
  m.nx = nx;
  m.ny = ny;
  m.cell = (region.max.x - region.min.x) / nx;
  m.threshold = threshold;
  m.samples.assign(static_cast<std::size_t>(nx) * ny, 0.0);
  double cy = (region.max.y - region.min.y) / ny;
  for (const V3& p : x) {
    if (!region.contains(p)) continue;
    int i = std::min(nx - 1, static_cast<int>((p.x - region.min.x) / m.cell));
    int j = std::min(ny - 1, static_cast<int>((p.y - region.min.y) / cy));
    m.at(i, j) = std::max(m.at(i, j), p.z - region.min.z);
  }
  return m;
}

struct IouResult {  // scenario.hpp:100-103
  double iou = 1.0;
  bool success = true;
};

// metric_write_iou (scenario.hpp:106-119)
inline IouResult metric_write_iou(const DepthMap& current, const DepthMap& target) {
  if (current.nx != target.nx || current.ny != target.ny)
    throw std::invalid_argument("metric_write_iou: resolution mismatch");
  std::size_t inter = 0, uni = 0;
  for (std::size_t i = 0; i < current.samples.size(); ++i) {
    bool a = current.occupied(i), b = target.occupied(i);
    inter += a && b;
    uni += a || b;
  }
  IouResult r;
  r.iou = uni == 0 ? 1.0 : static_cast<double>(inter) / static_cast<double>(uni);
  r.success = r.iou > 0.8;
  return r;
}

namespace detail {

// NnGrid (scenario.hpp:124-175): uniform bins, expanding Chebyshev shells
struct NnGrid {
  V3 origin;
  double cell;
  int dims[3];
  std::vector<std::vector<int>> bins;
  const std::vector<V3>* pts;

  explicit NnGrid(const std::vector<V3>& points) : pts(&points) {
    V3 lo = points[0], hi = points[0];
    for (const V3& p : points)
      for (int k = 0; k < 3; ++k) {
        lo[k] = std::min(lo[k], p[k]);
        hi[k] = std::max(hi[k], p[k]);
      }
    double diag = (hi - lo).norm();
    cell = std::max(diag / std::cbrt(static_cast<double>(points.size())), 1e-9);
    origin = lo;
    for (int ax = 0; ax < 3; ++ax) dims[ax] = std::max(1, static_cast<int>((hi[ax] - lo[ax]) / cell) + 1);
    bins.resize(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
    for (std::size_t i = 0; i < points.size(); ++i) bins[bin_of(points[i])].push_back(static_cast<int>(i));
  }
  void cell_of(const V3& p, int c[3]) const {
    for (int ax = 0; ax < 3; ++ax) c[ax] = std::clamp(static_cast<int>((p[ax] - origin[ax]) / cell), 0, dims[ax] - 1);
  }
  std::size_t bin_of(const V3& p) const {
    int c[3];
    cell_of(p, c);
    return (static_cast<std::size_t>(c[2]) * dims[1] + c[1]) * dims[0] + c[0];
  }
  double nearest_dist(const V3& q) const {
    int c[3];
    cell_of(q, c);
    double best = std::numeric_limits<double>::infinity();
    int kmax = std::max({dims[0], dims[1], dims[2]});
    for (int k = 0; k <= kmax; ++k) {
      if (best <= (k - 1) * cell) break;
      bool any = false;
      for (int dz = -k; dz <= k; ++dz)
        for (int dy = -k; dy <= k; ++dy)
          for (int dx = -k; dx <= k; ++dx) {
            if (std::max({std::abs(dx), std::abs(dy), std::abs(dz)}) != k) continue;
            int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
            if (x < 0 || y < 0 || z < 0 || x >= dims[0] || y >= dims[1] || z >= dims[2]) continue;
            any = true;
            const auto& bin = bins[(static_cast<std::size_t>(z) * dims[1] + y) * dims[0] + x];
            for (int i : bin) best = std::min(best, ((*pts)[i] - q).norm());
          }
      if (!any && best < std::numeric_limits<double>::infinity()) break;
    }
    return best;
  }
};

}  // namespace detail

// chamfer_distance (scenario.hpp:179-190)
inline double chamfer_distance(const std::vector<V3>& a, const std::vector<V3>& b) {
  if (a.empty() || b.empty()) throw std::invalid_argument("chamfer_distance: point sets must be non-empty");
  detail::NnGrid ga(a), gb(b);
  double ab = 0.0, ba = 0.0;
  for (const V3& p : a) ab += gb.nearest_dist(p);
  for (const V3& p : b) ba += ga.nearest_dist(p);
  return ab / static_cast<double>(a.size()) + ba / static_cast<double>(b.size());
}

struct PinchResult {  // scenario.hpp:192-195
  double ratio = 0.0;
  bool success = false;
};

// metric_pinch (scenario.hpp:199-209)
inline PinchResult metric_pinch(const std::vector<V3>& current, const std::vector<V3>& initial,
                                const std::vector<V3>& target) {
  double t = chamfer_distance(initial, target);
  double d = chamfer_distance(current, target);
  PinchResult r;
  r.ratio = t > 0.0 ? d / t : (d == 0.0 ? 0.0 : std::numeric_limits<double>::infinity());
  r.success = d < 0.3 * t;
  return r;
}

}  // namespace oracle
