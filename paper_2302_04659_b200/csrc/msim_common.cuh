// Device helpers shared by the hot-path kernels (msim_substep.cu) and the
// utility kernels (msim_kernels.cu): error latching, fp64 binning, the
// device-resident rigid step (rigid.hpp:52-66, coupling.hpp:106-117) and
// the reaction-only penalty of particles that leave the domain.
#pragma once

#include <cuda_runtime.h>

#include "msim_internal.h"

namespace msim_impl {

using msim_dev::f3;
using msim_dev::ShapeDev;

__device__ __forceinline__ unsigned float_bits_max(unsigned* addr, float v) {
  // v >= 0: IEEE bit patterns of non-negative floats order like unsigned ints.
  return atomicMax(addr, __float_as_uint(v));
}

static __device__ MSIM_COLD void set_error(const SimParams& P, int env, int code, int pid) {
  atomicCAS(&P.err_code[env], 0, code);  // first error of the env wins
  atomicMin(&P.err_pid[env], pid);
}

// Base cell and fractional offset computed like mpm.hpp:222-225: in double
// from the fp32 position (exact promotion), so base is bit-exact with the
// reference fed the same fp32-rounded positions.
__device__ __forceinline__ void base_of(const SimParams& P, float x, float y, float z, int* b, float* fx) {
  double lx = ((double)x - P.origin[0]) * P.inv_h;
  double ly = ((double)y - P.origin[1]) * P.inv_h;
  double lz = ((double)z - P.origin[2]) * P.inv_h;
  double fbx = floor(lx - 0.5), fby = floor(ly - 0.5), fbz = floor(lz - 0.5);
  b[0] = (int)fbx;
  b[1] = (int)fby;
  b[2] = (int)fbz;
  fx[0] = (float)(lx - fbx);
  fx[1] = (float)(ly - fby);
  fx[2] = (float)(lz - fbz);
}

__device__ __forceinline__ bool base_in_range(const SimParams& P, const int* b) {
  return b[0] >= 0 && b[1] >= 0 && b[2] >= 0 && b[0] <= P.dims[0] - 3 && b[1] <= P.dims[1] - 3 &&
         b[2] <= P.dims[2] - 3;
}

// Bucket (node block of the base cell) of an in-range base.
__device__ __forceinline__ int bucket_of(const SimParams& P, int env, const int* b) {
  return env * P.buckets_per_env + ((b[2] >> P.qshift[2]) * P.qdims[1] + (b[1] >> P.qshift[1])) * P.qdims[0] +
         (b[0] >> P.qshift[0]);
}

__device__ __forceinline__ f3 load3(float* const* a, long long i) { return {a[0][i], a[1][i], a[2][i]}; }

// ---------------------------------------------------------------------------
// Rigid step (double precision).

struct dq {
  double w, x, y, z;
};
__device__ __forceinline__ dq qmul(dq a, dq b) {
  return {a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z, a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
          a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z, a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ dq qnormcanon(dq q) {  // Pose::canonicalize (geometry.hpp:37-40)
  double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  q = {q.w / n, q.x / n, q.y / n, q.z / n};
  if (q.w < 0.0) q = {-q.w, -q.x, -q.y, -q.z};
  return q;
}
__device__ __forceinline__ void qrot(dq q, const double* v, double* out) {
  double uvx = q.y * v[2] - q.z * v[1], uvy = q.z * v[0] - q.x * v[2], uvz = q.x * v[1] - q.y * v[0];
  uvx *= 2;
  uvy *= 2;
  uvz *= 2;
  out[0] = v[0] + q.w * uvx + (q.y * uvz - q.z * uvy);
  out[1] = v[1] + q.w * uvy + (q.z * uvx - q.x * uvz);
  out[2] = v[2] + q.w * uvz + (q.x * uvy - q.y * uvx);
}
__device__ __forceinline__ void qmat(dq q, double* R) {
  double tx = 2 * q.x, ty = 2 * q.y, tz = 2 * q.z;
  double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
  double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
  double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
  R[0] = 1 - (tyy + tzz); R[1] = txy - twz; R[2] = txz + twy;
  R[3] = txy + twz; R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
  R[6] = txz - twy; R[7] = tyz + twx; R[8] = 1 - (txx + tyy);
}
__device__ __forceinline__ dq qexp(const double* aa) {  // quat_exp (geometry.hpp:78-87)
  double ang = sqrt(aa[0] * aa[0] + aa[1] * aa[1] + aa[2] * aa[2]);
  if (ang < 1e-14) {
    dq q = {1.0, 0.5 * aa[0], 0.5 * aa[1], 0.5 * aa[2]};
    double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
    return {q.w / n, q.x / n, q.y / n, q.z / n};
  }
  double s = sin(0.5 * ang) / ang;
  return {cos(0.5 * ang), s * aa[0], s * aa[1], s * aa[2]};
}

// Pose part of integrate_free_body (rigid.hpp:60-65): COM moves with the
// linear velocity, orientation rotates about it.
__device__ inline void advance_pose(BodyDev& b, double dt) {
  dq rot = {b.q[0], b.q[1], b.q[2], b.q[3]};
  double com[3];
  qrot(rot, b.com_off, com);
  for (int k = 0; k < 3; ++k) com[k] += b.t[k];
  double com_new[3] = {com[0] + dt * b.v[0], com[1] + dt * b.v[1], com[2] + dt * b.v[2]};
  double aa[3] = {b.w[0] * dt, b.w[1] * dt, b.w[2] * dt};
  dq d = qexp(aa);
  dq rn = qmul(d, rot);
  double n = sqrt(rn.w * rn.w + rn.x * rn.x + rn.y * rn.y + rn.z * rn.z);
  rn = {rn.w / n, rn.x / n, rn.y / n, rn.z / n};
  double rc[3];
  qrot(rn, b.com_off, rc);
  double t[3] = {com_new[0] - rc[0], com_new[1] - rc[1], com_new[2] - rc[2]};
  rn = qnormcanon(rn);
  b.q[0] = rn.w; b.q[1] = rn.x; b.q[2] = rn.y; b.q[3] = rn.z;
  for (int k = 0; k < 3; ++k) b.t[k] = t[k];
}

// integrate_free_body (rigid.hpp:52-66): semi-implicit Newton-Euler with the
// staged wrench (force, torque about the world COM).
__device__ inline void integrate_free_body(BodyDev& b, const double* wf, const double* g, double dt) {
  for (int k = 0; k < 3; ++k) b.v[k] += dt * (g[k] + wf[k] / b.mass);
  dq rot = {b.q[0], b.q[1], b.q[2], b.q[3]};
  double R[9];
  qmat(rot, R);
  double I[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      I[r * 3 + c] = R[r * 3 + 0] * b.inertia[0] * R[c * 3 + 0] + R[r * 3 + 1] * b.inertia[1] * R[c * 3 + 1] +
                     R[r * 3 + 2] * b.inertia[2] * R[c * 3 + 2];
  double L[3] = {I[0] * b.w[0] + I[1] * b.w[1] + I[2] * b.w[2], I[3] * b.w[0] + I[4] * b.w[1] + I[5] * b.w[2],
                 I[6] * b.w[0] + I[7] * b.w[1] + I[8] * b.w[2]};
  double rhs[3] = {wf[3] - (b.w[1] * L[2] - b.w[2] * L[1]), wf[4] - (b.w[2] * L[0] - b.w[0] * L[2]),
                   wf[5] - (b.w[0] * L[1] - b.w[1] * L[0])};
  double det = I[0] * (I[4] * I[8] - I[5] * I[7]) - I[1] * (I[3] * I[8] - I[5] * I[6]) +
               I[2] * (I[3] * I[7] - I[4] * I[6]);
  double Inv[9] = {(I[4] * I[8] - I[5] * I[7]) / det, (I[2] * I[7] - I[1] * I[8]) / det,
                   (I[1] * I[5] - I[2] * I[4]) / det, (I[5] * I[6] - I[3] * I[8]) / det,
                   (I[0] * I[8] - I[2] * I[6]) / det, (I[2] * I[3] - I[0] * I[5]) / det,
                   (I[3] * I[7] - I[4] * I[6]) / det, (I[1] * I[6] - I[0] * I[7]) / det,
                   (I[0] * I[4] - I[1] * I[3]) / det};
  for (int k = 0; k < 3; ++k) b.w[k] += dt * (Inv[3 * k] * rhs[0] + Inv[3 * k + 1] * rhs[1] + Inv[3 * k + 2] * rhs[2]);
  advance_pose(b, dt);
}

// quat_log (geometry.hpp:89-96): axis * angle of a rotation, angle in [0, pi].
__device__ inline void quat_log(dq q, double out[3]) {
  const double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  q = {q.w / n, q.x / n, q.y / n, q.z / n};
  if (q.w < 0.0) q = {-q.w, -q.x, -q.y, -q.z};
  const double vn = sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
  const double k = vn < 1e-14 ? 2.0 : 2.0 * atan2(vn, q.w) / vn;
  out[0] = k * q.x;
  out[1] = k * q.y;
  out[2] = k * q.z;
}

// Robot::set_kinematic_pose (rigid.hpp:142-151): jump to the (canonicalized)
// target pose, twist = finite difference of the two poses over dt.
__device__ inline void set_kinematic_pose(BodyDev& b, const double* p, double dt) {
  const dq tq = qnormcanon({p[0], p[1], p[2], p[3]});
  const dq rel = qmul(tq, dq{b.q[0], -b.q[1], -b.q[2], -b.q[3]});
  double w[3];
  quat_log(rel, w);
  for (int k = 0; k < 3; ++k) {
    b.v[k] = dt > 0.0 ? (p[4 + k] - b.t[k]) / dt : 0.0;
    b.w[k] = dt > 0.0 ? w[k] / dt : 0.0;
    b.t[k] = p[4 + k];
  }
  b.q[0] = tq.w; b.q[1] = tq.x; b.q[2] = tq.y; b.q[3] = tq.z;
}

// One env's rigid step: optionally integrate (dynamic: with the staged
// wrench; scripted: constant twist; scheduled kinematic: the schedule's pose
// of this rigid step), then sync_rigid_to_soft: zero the accumulating
// wrenches and rebuild the per-shape world transforms.
// lane / nlanes: the threads sharing the env (one warp: bodies, then shapes, in parallel).
// Latency bound (one env per warp, fp64): descriptions are read in batches
// ahead of use, a warp passes its integrated bodies to the shape lanes through
// shared memory (sbody: kMaxBodiesPerEnv slots per warp, or null: global), and
// stage = true also stages the wrench (pending = wrench, coupling.hpp:288) in
// the body lane that integrates with it. ridx: the schedule row of this rigid step.
struct EnvRange {
  int b0, b1, s0, s1;
};
__device__ __forceinline__ EnvRange env_range(const SimParams& P, int env) {
  return {P.body_off[env], P.body_off[env + 1], P.shape_off[env], P.shape_off[env + 1]};
}
__device__ inline void rigid_env(const SimParams& P, int env, int integrate, int lane, int nlanes, const EnvRange& g,
                                 int ridx, bool stage, BodyDev* sbody) {
  const int b0 = g.b0, b1 = g.b1, s0 = g.s0, s1 = g.s1;
  ridx = P.sched_steps > 0 ? min(ridx, P.sched_steps - 1) : 0;
  const bool has0 = s0 + lane < s1;
  ShapeHost sh0;  // this lane's first shape, loaded ahead of the body pass
  if (has0) sh0 = P.shape_src[s0 + lane];
  for (int bi = b0 + lane; bi < b1; bi += nlanes) {
    double* wr = P.wrench + 6 * bi;
    if (integrate) {
      BodyDev b = P.bodies[bi];
      double wf[6];
      for (int k = 0; k < 6; ++k) wf[k] = stage ? wr[k] : P.pending[6 * bi + k];
      if (stage)
        for (int k = 0; k < 6; ++k) P.pending[6 * bi + k] = wf[k];
      if (b.mode == MSIM_BODY_DYNAMIC)
        integrate_free_body(b, wf, P.rigid_g, P.dt_r);
      else if (b.mode == MSIM_BODY_SCRIPTED)
        advance_pose(b, P.dt_r);
      if (P.sched_steps > 0 && P.sched_mask[bi])
        set_kinematic_pose(b, P.sched + 7 * ((long long)ridx * P.n_bodies_total + bi), P.dt_r);
      P.bodies[bi] = b;
      if (sbody && bi - b0 < kMaxBodiesPerEnv) sbody[bi - b0] = b;
    } else if (sbody && bi - b0 < kMaxBodiesPerEnv) {
      sbody[bi - b0] = P.bodies[bi];
    }
    for (int k = 0; k < 6; ++k) wr[k] = 0.0;
    if (P.det)
      for (int k = 0; k < 6; ++k) P.w64[6 * bi + k] = 0;
  }
  if (nlanes > 1) __syncwarp();  // shapes read their (integrated) bodies
  for (int si = s0 + lane; si < s1; si += nlanes) {
    const ShapeHost sh = si == s0 + lane ? sh0 : P.shape_src[si];
    const BodyDev b = sbody && sh.body < kMaxBodiesPerEnv ? sbody[sh.body] : P.bodies[b0 + sh.body];
    dq bq = {b.q[0], b.q[1], b.q[2], b.q[3]};
    dq lq = {sh.lq[0], sh.lq[1], sh.lq[2], sh.lq[3]};
    dq wq = qnormcanon(qmul(bq, lq));  // compose (geometry.hpp:54-56)
    double wt[3];
    qrot(bq, sh.lt, wt);
    for (int k = 0; k < 3; ++k) wt[k] += b.t[k];
    dq iq = {wq.w, -wq.x, -wq.y, -wq.z};  // inverse (geometry.hpp:58-61)
    double it[3];
    qrot(iq, wt, it);
    double R[9], Ri[9];
    qmat(wq, R);
    qmat(iq, Ri);
    ShapeDev& d = P.shapes[si];
    for (int k = 0; k < 9; ++k) {
      d.R[k] = (float)R[k];
      d.Rinv[k] = (float)Ri[k];
    }
    for (int k = 0; k < 3; ++k) d.tinv[k] = (float)(-it[k]);
    double com[3];
    qrot(bq, b.com_off, com);
    for (int k = 0; k < 3; ++k) {
      d.com[k] = (float)(com[k] + b.t[k]);
      d.vlin[k] = (float)b.v[k];
      d.vang[k] = (float)b.w[k];
    }
    for (int k = 0; k < 4; ++k) d.p[k] = (float)sh.p[k];
    d.friction = (float)sh.friction;
    d.k_n = (float)sh.k_n;
    d.k_t = (float)sh.k_t;
    d.type = sh.type;
    d.body = sh.body;
    for (int k = 0; k < 3; ++k) {
      d.vol_dims[k] = sh.vol_dims[k];
      d.vol_origin[k] = (float)sh.vol_origin[k];
    }
    d.vol_voxel = (float)sh.vol_voxel;
    d.vol_off = sh.vol_off;
    // culling bound (shape_may_touch): world x = R (local - tinv)
    if (sh.type == 0) {  // plane: phi = n . (Ri x + tinv) - d = (R n) . x + n . tinv - d
      double nw[3];
      qrot(wq, sh.p, nw);
      for (int k = 0; k < 3; ++k) d.bnd[k] = (float)nw[k];
      d.bnd[3] = (float)(sh.p[0] * -it[0] + sh.p[1] * -it[1] + sh.p[2] * -it[2] - sh.p[3]);
      d.bplane = 1;
    } else {
      double lc[3] = {0.0, 0.0, 0.0}, rad = 0.0;
      if (sh.type == 1) rad = sh.p[0];
      else if (sh.type == 2) rad = sqrt(sh.p[0] * sh.p[0] + sh.p[1] * sh.p[1] + sh.p[2] * sh.p[2]);
      else if (sh.type == 3) rad = sh.p[0] + sh.p[1];
      else {  // volume: box half-diagonal, phi >= vol_min + distance outside the box
        double hd2 = 0.0;
        for (int k = 0; k < 3; ++k) {
          const double ext = (sh.vol_dims[k] - 1) * sh.vol_voxel;
          lc[k] = sh.vol_origin[k] + 0.5 * ext;
          hd2 += 0.25 * ext * ext;
        }
        rad = sqrt(hd2) + fmax(0.0, -sh.vol_min);
      }
      double wc[3];
      qrot(wq, lc, wc);
      for (int k = 0; k < 3; ++k) d.bnd[k] = (float)(wc[k] + wt[k]);
      d.bnd[3] = (float)rad;
      d.bplane = 0;
    }
  }
}

// Particle leaving the domain this cycle: its penalty reaction still counts
// (the hook runs before p2g's loss detection, coupling.hpp:266-274).
template <bool DET>
__device__ MSIM_COLD void penalty_reaction_only(const SimParams& P, int env, f3 x, f3 v) {
  const int s0 = P.shape_off[env], s1 = P.shape_off[env + 1];
  const int b0 = P.body_off[env];
  for (int s = s0; s < s1; ++s) {
    const ShapeDev& sh = P.shapes[s];
    f3 f;
    float pen;
    if (!msim_dev::penalty_force(sh, P.vol_pool, x, v, P.r_c_particle, P.c_d, f, pen)) continue;
    f3 com = {sh.com[0], sh.com[1], sh.com[2]};
    f3 tq = msim_dev::cross(x - com, f3{-f.x, -f.y, -f.z});
    if constexpr (DET) {  // integer sums (deterministic mode)
      const double r6[6] = {-(double)f.x, -(double)f.y, -(double)f.z, (double)tq.x, (double)tq.y, (double)tq.z};
      unsigned long long* w = reinterpret_cast<unsigned long long*>(P.w64 + 6 * (b0 + sh.body));
      for (int k = 0; k < 6; ++k) atomicAdd(w + k, (unsigned long long)__double2ll_rn(ldexp(r6[k], kDetWrenchExp)));
      for (int k = 0; k < 3; ++k) {
        const long long rk = __double2ll_rn(ldexp(r6[k], kDetWrenchExp));
        atomicAdd(reinterpret_cast<unsigned long long*>(P.r64 + 3 * env + k), (unsigned long long)rk);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.a64 + 3 * env + k), (unsigned long long)(-rk));
      }
    } else {
      double* wr = P.wrench + 6 * (b0 + sh.body);
      atomicAdd(wr + 0, -(double)f.x);
      atomicAdd(wr + 1, -(double)f.y);
      atomicAdd(wr + 2, -(double)f.z);
      atomicAdd(wr + 3, (double)tq.x);
      atomicAdd(wr + 4, (double)tq.y);
      atomicAdd(wr + 5, (double)tq.z);
      for (int k = 0; k < 3; ++k) {
        double fk = k == 0 ? f.x : (k == 1 ? f.y : f.z);
        atomicAdd(P.applied + 3 * env + k, fk);
        atomicAdd(P.react + 3 * env + k, -fk);
      }
    }
    float_bits_max(&P.max_pen_bits[env], pen);
  }
}

}  // namespace msim_impl
