// Hot path of the B200 MLS-MPM substep (sm_100a).
//
// The reference runs each CFL cycle as clear -> penalty hook -> p2g ->
// grid hook -> grid_update -> g2p_advect (mpm.hpp:410-418). Here one
// batched launch sequence per cycle does, for every environment at once:
//
//   k_particles  persistent CTAs over buckets (1 or 2^3 node blocks of
//                kBX x kBY x kBZ base cells, by particle density). Gathers the
//                bucket's particles (perm), runs G2P of this cycle against a
//                shared-memory velocity tile (mpm.hpp:346-379), the F update
//                and the material's return map (mpm.hpp:166-181 for the
//                reference's von Mises clay), and in the same pass the P2G of
//                the next cycle: penalty hook (coupling.hpp:151-172), Kirchhoff
//                stress from the SAME strain evaluation (mpm.hpp:152-161; the
//                Hencky strain as a matrix function of F F^T, msim_device.cuh),
//                and a scatter into a shared-memory node tile: each thread adds
//                one staged particle's 27 node contributions with native int32
//                shared atomics on a per-round fixed-point scale, lanes taking
//                slots ~0.618 rn apart so a warp's stencils rarely collide.
//                The tile goes to HBM with vector REDs. Particles are written
//                back in bucket order with their next bucket key (the
//                per-cycle re-sort).
//   scans        bucket offsets + active list, node-block list
//   k_iter_end   per env: substep/cycle counters, CFL plan (mpm.hpp:400-409),
//                lost-fraction check, force-balance diagnostic; zeroes the
//                accumulators of an env whose P2G must be redone
//   redo         only when a CFL halving changed the next cycle's dt: the
//                P2G of that env is redone with the planned dt
//   k_grid       per touched node block: (p + dt f)/m + dt g, grid-mode
//                penalty (coupling.hpp:186-214), boundary bands
//                (mpm.hpp:315-342); consumes (zeroes) the accumulators
//   k_perm       the next launch's slot map (after k_grid, alongside it)
//   k_iter_begin the next cycle's rigid step (alongside k_grid)
//
// Small scenes split a bucket's rounds over several CTAs (split_r). The
// per-cycle kernels are launched with programmatic dependent launch; those
// whose inputs are complete when they are scheduled work before waiting
// (msim_internal.h launch_pdl).
//
// Because G2P(c) and P2G(c+1) share one pass, each particle-substep reads and
// writes x, F-I, mass, V0, meta, pid once; v and C stay in registers except
// at the first/last cycle of a call.
//
// Momentum channels: the default path folds the force into the momentum,
// p + dt f (4 channels: what grid_update consumes, mpm.hpp:321). The dt of
// the next cycle is known inside a substep; across substeps it is
// speculated as the current cycle's and re-done on the device if the CFL
// plan halves differently. The phase API and grid coupling keep momentum and
// force apart (7 channels) like MpmGrid.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>

#include "msim_common.cuh"

using namespace msim_dev;

namespace msim_impl {
namespace {

#ifndef MSIM_KT
#define MSIM_KT 128
#endif
#ifndef MSIM_KCAP
#define MSIM_KCAP 128
#endif
// 128 threads / 128 particles per round measured best with the dynamic bucket
// hand-out (D, 1024 envs: 2.85 vs 2.98 ms per launch at 256 particles, 4.06 at 64;
// 256 threads at 2-3 CTAs/SM +6-15 %; 64 threads / 128 at 9 CTAs/SM +12 %)
constexpr int kT = MSIM_KT;      // threads per CTA (particle kernel), ctas_per_sm() CTAs per SM
constexpr int kCap = MSIM_KCAP;  // particles staged per round
// Tile geometry of a particle bucket of F^3 node blocks (QX x QY x QZ base cells).
template <int F>
struct Geo {
  static constexpr int QX = kBX * F, QY = kBY * F, QZ = kBZ * F;
  static constexpr int GX = QX + 2, GY = QY + 2, GZ = QZ + 2, GN = GX * GY * GZ;  // G2P velocity tile
  static constexpr int PX = QX + 4, PY = QY + 4, PZ = QZ + 4;  // P2G node tile (origin o-1)
  // z-layer stride padded by 4 words: for F = 1 (64 -> 68) the 32 base cells of a
  // bucket hit 32 distinct shared-memory banks for every stencil offset
  static constexpr int TZS = PX * PY + 4;
  static constexpr int PN = PZ * TZS;
  static constexpr int CX = QX + 2, CY = QY + 2, CZ = QZ + 2;  // P2G base cells (origin o-1)
  // node blocks (kBX x kBY x kBZ nodes) a tile cell's stencil can touch, origin block o / kB - 1
  static constexpr int NBX = F + 2, NBY = F + 2, NBZ = F + 3, NBT = NBX * NBY * NBZ;
  // particles per round: one trip per thread between barriers (see MSIM_KCAP)
  static constexpr int CAP = kCap;
  // fixed point: |contribution| <= 0.75^3 * 2^SC_LOG2 < 2^22 (the fix_rn range),
  // CAP contributions per node <= 2^30
  static constexpr int SC_LOG2 = CAP == 512 ? 21 : (CAP == 256 ? 22 : 23);
};
#define MSIM_GEO_ALIASES(F)                                                                            \
  using Gm = Geo<F>;                                                                                   \
  [[maybe_unused]] constexpr int QX = Gm::QX, QY = Gm::QY, QZ = Gm::QZ, GX = Gm::GX, GY = Gm::GY,      \
                                 GZ = Gm::GZ, GN = Gm::GN, PX = Gm::PX, PY = Gm::PY, PZ = Gm::PZ,      \
                                 kTZS = Gm::TZS, PN = Gm::PN, CX = Gm::CX, CY = Gm::CY, CZ = Gm::CZ,  \
                                 CAP = Gm::CAP;
// staged P2G payload per particle: m, fx (weights recomputed in the scatter), b, A
// (+ b_f, symmetric A_f in 7-channel mode)
template <int NCH> constexpr int pay_floats() { return NCH == 4 ? 16 : 28; }
// Resident CTAs per SM (__launch_bounds__ -> register budget) and the L2
// prefetch of the next round's particle, per instantiation. Dense buckets
// (F = 1) in the 4-channel path run 8 CTAs at 64 registers without the
// prefetch: D +3.8 % against 5 CTAs at 96 with it (6 CTAs +2.5 %, 7 +0.5 %),
// batched sand B +3 %; the deterministic twin runs best at 6 (its int64 flush).
// Sparse 2^3-block buckets (E, C: 6 CTAs -7 %) and the 7-channel path keep 5
// with the prefetch (profiles/r02_experiments_D.txt).
constexpr bool dense_4ch(int NCH, int F) { return NCH == 4 && F == 1; }
#ifdef MSIM_CTAS_PER_SM  // variant builds: one setting for every instantiation
constexpr int ctas_per_sm(int, int, bool) { return MSIM_CTAS_PER_SM; }
#else
constexpr int ctas_per_sm(int NCH, int F, bool DET) { return dense_4ch(NCH, F) ? (DET ? 6 : 8) : 5; }
#endif
#ifdef MSIM_NO_L2_PREFETCH
constexpr bool l2_prefetch(int, int) { return false; }
#else
constexpr bool l2_prefetch(int NCH, int F) { return !dense_4ch(NCH, F); }
#endif
#ifdef MSIM_STATIC_ITEMS  // variant build: static round-robin bucket assignment
constexpr bool kDynamicItems = false;
#else
constexpr bool kDynamicItems = true;
#endif

// Particle state is streamed once per launch: evict-first loads / stores
// (ld/st .cs) keep L1 for the register spills and the per-bucket tiles.
#ifdef MSIM_NO_STREAM_HINTS  // variant build: plain cached accesses
template <class T> __device__ __forceinline__ T lds(const T* p) { return *p; }
template <class T> __device__ __forceinline__ void sts(T* p, T v) { *p = v; }
#else
template <class T> __device__ __forceinline__ T lds(const T* p) { return __ldcs(p); }
template <class T> __device__ __forceinline__ void sts(T* p, T v) { __stcs(p, v); }
#endif
#ifdef MSIM_NO_CULL  // variant build: no bounding test ahead of the collider SDFs
constexpr bool kNoCull = true;
#else
constexpr bool kNoCull = false;
#endif
// Loop unrolling of the 27-node stencils: the kernel is issue/latency bound
// with a large instruction footprint, and rolled scatter loops measured faster
// (ms per launch, D 256 envs: all unrolled 0.975, z rolled 0.961, z and y
// rolled 0.938).
#ifdef MSIM_SCATTER_UNROLLED
constexpr int kScatterDkUnroll = 3, kScatterDjUnroll = 3;
#else
constexpr int kScatterDkUnroll = 1, kScatterDjUnroll = 1;
#endif
#ifdef MSIM_SCATTER_ROLLED3  // variant: x-offset loop rolled as well
constexpr int kScatterDiUnroll = 1;
#else
constexpr int kScatterDiUnroll = 3;
#endif
#ifndef MSIM_TAIL_SPLIT  // parts per tail bucket (1: no tail split)
#define MSIM_TAIL_SPLIT 4
#endif
constexpr int kTailSplit = MSIM_TAIL_SPLIT;
#ifdef MSIM_G2P_ROLLED  // variant: G2P z-offset loop rolled
constexpr int kG2pDkUnroll = 1;
#else
constexpr int kG2pDkUnroll = 3;
#endif
constexpr int kWs = kMaxBodiesPerEnv * 6 + 3;

// Bucket-uniform values of k_particles, kept in shared memory and re-read at
// each use (volatile): held in registers across the per-particle phase they
// were spilled to local memory (measured 15 % of the executed instructions).
struct ItemCtx {
  int key, benv, s, e, act, ox, oy, oz, s0, s1;
  float dt, dtp;
  int lostb, do_g2p, do_p2g, penalty;
  int rstep;           // slot stride between this item's rounds (CAP x parts)
  int split;           // the bucket's rounds are spread over several CTAs: atomic (unordered) ranks
  unsigned smask;      // env shapes (bit k = shape s0 + k, k < 32) that can reach the bucket box
  float blo[3], bhi[3];  // the bucket's particles' box widened by 2 h (positions after G2P)
};

template <int NCH, int F>
struct Smem {
  float4 gtile[Geo<F>::GN];
  int itile[NCH][Geo<F>::PN];  // fixed-point node accumulators (native int shared atomics)
  float4 pay[pay_floats<NCH>() / 4][Geo<F>::CAP];  // float4 k of slot t at pay[k][t]: conflict-free
  int cellof[Geo<F>::CAP];  // local P2G cell of each staged slot, -1 if not staged
  // node blocks of the tile touched by the staged particles' 3x3x3 stencils
  // during the current bucket (the reference's active nodes, mpm.hpp:266-280, at
  // block granularity); written out and cleared once per bucket
  unsigned char bflag[Geo<F>::NBT];
  double wsum[kWs];
  unsigned penmax;
  // per-round fixed-point bounds, double-buffered by round parity: round r
  // publishes into maxb[r & 1] before its post-staging barrier while slot
  // (r + 1) & 1 is zeroed between that barrier and the post-scatter one
  unsigned maxb[2][3];
  // per warp slot of a round: ballot of the particles staying in this bucket
  // (order-preserving ranks), double-buffered by round parity like maxb
  unsigned wball[2][Geo<F>::CAP / 32];
  ItemCtx ic;              // the current bucket's uniform context (read back instead of held in registers)
  int next_item;
};


__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int gcd_c(int a, int b) { return b ? gcd_c(b, a % b) : a; }
// Scatter slot stride per round size rn: odd, coprime with rn, ~0.618 rn (see k_particles)
struct SpreadTable {
  unsigned short g[kCap + 1];
};
constexpr SpreadTable make_spread() {
  SpreadTable t{};
  for (int rn = 1; rn <= kCap; ++rn) {
    int g = ((int)(0.618034 * rn)) | 1;
    while (gcd_c(g, rn) != 1) g += 2;
    t.g[rn] = (unsigned short)g;
  }
  return t;
}
__constant__ SpreadTable kSpread = make_spread();

// Deterministic mode: integer fixed-point accumulation (commutative, so the
// result does not depend on the order CTAs / warps add in).
__device__ __forceinline__ void red_add_i64(long long* a, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ long long det_fix(double v, int e) { return __double2ll_rn(ldexp(v, e)); }

// Round-to-nearest float -> int for |x| < 2^22 with one FFMA-able add: the
// integer lands in the low mantissa bits of x + 1.5 * 2^23 (avoids F2I).
__device__ __forceinline__ int fix_rn(float x) { return __float_as_int(x + 12582912.0f) - 0x4B400000; }

// Fire-and-forget vector float add to global memory (RED, no return value).
__device__ __forceinline__ void red_add_v4(float4* a, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// Global-memory scatter of one particle (fallback when its stencil leaves the
// bucket's P2G tile, e.g. a particle faster than the CFL bound assumed).
template <int NCH, bool DET>
__device__ MSIM_COLD void scatter_global(const SimParams& P, int env, const int* b, const float* w9, float m, f3 bp,
                               const float* Ap, f3 bf, const float* Af, bool mark) {
  for (int dk = 0; dk < 3; ++dk)
    for (int dj = 0; dj < 3; ++dj)
      for (int di = 0; di < 3; ++di) {
        const float w = w9[di] * w9[3 + dj] * w9[6 + dk];
        const f3 pq = {bp.x + Ap[0] * di + Ap[1] * dj + Ap[2] * dk, bp.y + Ap[3] * di + Ap[4] * dj + Ap[5] * dk,
                       bp.z + Ap[6] * di + Ap[7] * dj + Ap[8] * dk};
        const int gx = b[0] + di, gy = b[1] + dj, gz = b[2] + dk;
        const long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
        if constexpr (DET) {
          const int sm = P.run[env].det_sm, sp = P.run[env].det_sp;
          long long* g = &P.gPMd[gi].x;
          red_add_i64(g + 0, det_fix((double)(w * pq.x), sp));
          red_add_i64(g + 1, det_fix((double)(w * pq.y), sp));
          red_add_i64(g + 2, det_fix((double)(w * pq.z), sp));
          red_add_i64(g + 3, det_fix((double)(w * m), sm));
        } else {
          red_add_v4(&P.gPM[gi], w * pq.x, w * pq.y, w * pq.z, w * m);
        }
        if (NCH == 7) {
          const f3 fq = {bf.x + Af[0] * di + Af[1] * dj + Af[2] * dk, bf.y + Af[3] * di + Af[4] * dj + Af[5] * dk,
                         bf.z + Af[6] * di + Af[7] * dj + Af[8] * dk};
          red_add_v4(&P.gF[gi], w * fq.x, w * fq.y, w * fq.z, 0.0f);
        }
        if (mark) P.nb_flag[env * P.blocks_per_env + ((gz / kBZ) * P.bdims[1] + gy / kBY) * P.bdims[0] + gx / kBX] = 1;
      }
}

// The rounds of one bucket (<= kCap particles each): per-particle phase, then
// the fixed-point scatter and flush. Bucket-uniform values come from S.ic.
template <int NCH, int F, bool AM, bool DET>
__device__ __forceinline__ void item_rounds(const SimParams& P, Smem<NCH, F>& S, bool redo) {
  MSIM_GEO_ALIASES(F)
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  volatile ItemCtx& IC = S.ic;
  {
    int stay_base = 0;  // particles of this bucket that stay in it, so far (CTA-uniform)
    for (int r0 = IC.s, rpar = 0; r0 < IC.e; r0 += IC.rstep, rpar ^= 1) {
      const int rn = min(CAP, IC.e - r0);
      const int trips = (rn + kT - 1) / kT;
      float mx_m = 0.f, mx_p = 0.f, mx_f = 0.f;
      // ---------------- per-particle phase (CTA-uniform trip count for warp collectives)
      for (int trip = 0; trip < trips; ++trip) {
        const int t = trip * kT + tid;
        const bool valid = t < rn;
        const int j = r0 + t;
        const int i = valid ? P.perm[j] : 0;
        // L2 prefetch of this thread's next particle, one round ahead
        const int i_pf = l2_prefetch(NCH, F) && j + IC.rstep < IC.e ? P.perm[j + IC.rstep] : -1;
        unsigned meta = valid ? lds(&P.cur.meta[i]) : (1u << kLostBit);
        const int penv = (meta >> 8) & kEnvMask;
        const bool was_lost = meta >> kLostBit;
        const int pact = IC.lostb ? (valid ? P.run[penv].action : kActIdle) : IC.act;
        f3 x = {0.f, 0.f, 0.f}, v = {0.f, 0.f, 0.f};
        float G[9], Cm[9];
        float m = 0.f, V0 = 0.f, jp = 1.f;
        int pid = 0;
        if (valid) {
          x = {lds(&P.cur.x[0][i]), lds(&P.cur.x[1][i]), lds(&P.cur.x[2][i])};
#pragma unroll
          for (int k = 0; k < 9; ++k) G[k] = lds(&P.cur.G[k][i]);
          m = lds(&P.cur.mass[i]);
          V0 = lds(&P.cur.vol0[i]);
          if (AM) jp = lds(&P.cur.jp[i]);
          pid = lds(&P.cur.pid[i]);
        } else {
#pragma unroll
          for (int k = 0; k < 9; ++k) G[k] = 0.f;
        }
        const bool read_vc = valid && (IC.lostb || !IC.do_g2p);
        if (read_vc) {
          v = load3(P.cur.v, i);
#pragma unroll
          for (int k = 0; k < 9; ++k) Cm[k] = P.cur.C[k][i];
        } else {
#pragma unroll
          for (int k = 0; k < 9; ++k) Cm[k] = 0.f;
        }
        bool write_vc = valid && (IC.lostb || IC.act != kActFused);
        const bool live = valid && !IC.lostb && !was_lost && IC.act != kActIdle;
        float speed = -1.0f;
        // Kirchhoff stress of the updated state for the next P2G (one strain evaluation per substep)
        Sym ts = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        // AM = false (every material of the context is the reference's von Mises
        // clay): the model dispatch and the jp field compile away (7 % of the kernel)
        MatParams mp = P.mats[meta & 0xFFu];
        if (!AM) mp.model = kModelVonMises;
        // Hencky strain for the models that use it (von Mises, Drucker-Prager)
        auto hencky_of = [&](const float* g) -> Sym {
          return (mp.model == kModelVonMises || mp.model == kModelDruckerPrager) ? hencky_strain(g)
                                                                                 : Sym{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        };

        // ---------------- G2P of this cycle (mpm.hpp:346-379)
        if (live && IC.do_g2p) {
          int b[3];
          float fx[3];
          base_of(P, x.x, x.y, x.z, b, fx);
          const int lx = b[0] - IC.ox, ly = b[1] - IC.oy, lz = b[2] - IC.oz;
          float wx[3], wy[3], wz[3];
          bspline_w(fx[0], wx);
          bspline_w(fx[1], wy);
          bspline_w(fx[2], wz);
          f3 vs = {0.f, 0.f, 0.f}, Sx = {0.f, 0.f, 0.f}, Sy = {0.f, 0.f, 0.f}, Sz = {0.f, 0.f, 0.f};
#ifdef MSIM_ABLATE_G2P  // profiling-only build: no grid gather (lx >= 0 always)
          if (lx < 0)
#endif
#pragma unroll kG2pDkUnroll
          for (int dk = 0; dk < 3; ++dk)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj) {
              const int tb = ((lz + dk) * GY + (ly + dj)) * GX + lx;
              const float4 v0 = S.gtile[tb], v1 = S.gtile[tb + 1], v2 = S.gtile[tb + 2];
              const f3 a = {wx[0] * v0.x + wx[1] * v1.x + wx[2] * v2.x, wx[0] * v0.y + wx[1] * v1.y + wx[2] * v2.y,
                            wx[0] * v0.z + wx[1] * v1.z + wx[2] * v2.z};
              const f3 ax = {wx[1] * v1.x + 2.f * wx[2] * v2.x, wx[1] * v1.y + 2.f * wx[2] * v2.y,
                             wx[1] * v1.z + 2.f * wx[2] * v2.z};
              const float wr = wy[dj] * (dk == 0 ? wz[0] : (dk == 1 ? wz[1] : wz[2]));
              vs = vs + wr * a;
              Sx = Sx + wr * ax;
              if (dj) Sy = Sy + (wr * dj) * a;
              if (dk) Sz = Sz + (wr * dk) * a;
            }
          // C = (4/h) sum w v (off - fx)^T = (4/h)(S - v fx^T)  (partition of unity)
          const float k4h = 4.0f / P.h_f;
          Cm[0] = k4h * (Sx.x - vs.x * fx[0]); Cm[1] = k4h * (Sy.x - vs.x * fx[1]); Cm[2] = k4h * (Sz.x - vs.x * fx[2]);
          Cm[3] = k4h * (Sx.y - vs.y * fx[0]); Cm[4] = k4h * (Sy.y - vs.y * fx[1]); Cm[5] = k4h * (Sz.y - vs.y * fx[2]);
          Cm[6] = k4h * (Sx.z - vs.z * fx[0]); Cm[7] = k4h * (Sy.z - vs.z * fx[1]); Cm[8] = k4h * (Sz.z - vs.z * fx[2]);
          v = vs;
          x = x + IC.dt * vs;
          if (IC.dt != 0.0f && mp.model == kModelFluid) {  // J-only: J *= 1 + dt tr(C)
            jp *= 1.0f + IC.dt * (Cm[0] + Cm[4] + Cm[8]);
            if (!(jp > 0.0f)) set_error(P, penv, kErrDetReturn, pid);
            ts = stress_of(kModelFluid, G, ts, jp, mp);
          } else if (IC.dt != 0.0f) {  // F <- (I + dt C) F, then the model's return map (mpm.hpp:367-373)
            float Gn[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int c = 0; c < 3; ++c)
                Gn[r * 3 + c] = G[r * 3 + c] + IC.dt * (Cm[r * 3 + c] + Cm[r * 3 + 0] * G[0 * 3 + c] +
                                                     Cm[r * 3 + 1] * G[1 * 3 + c] + Cm[r * 3 + 2] * G[2 * 3 + c]);
            if (!(det_I_plus(Gn) > 0.0f)) set_error(P, penv, kErrDetReturn, pid);
            Sym eps = hencky_of(Gn);
            if (mp.model == kModelVonMises) von_mises_project_strain(Gn, eps, mp);
            else if (mp.model == kModelDruckerPrager) drucker_prager_project_strain(Gn, eps, jp, mp);
#pragma unroll
            for (int k = 0; k < 9; ++k) G[k] = Gn[k];
            ts = stress_of(mp.model, G, eps, jp, mp);
          } else if (IC.do_p2g) {
            ts = stress_of(mp.model, G, hencky_of(G), jp, mp);
          }
          bool bad = false;
#pragma unroll
          for (int k = 0; k < 9; ++k) bad |= !isfinite(G[k]);
          bad |= !isfinite(x.x) || !isfinite(x.y) || !isfinite(x.z) || !isfinite(v.x) || !isfinite(v.y) ||
                 !isfinite(v.z);
          if (bad) set_error(P, penv, kErrNan, pid);
          speed = norm(v);
          if (!(speed >= 0.0f)) speed = FLT_MAX;
        } else if (live && IC.do_p2g) {
          if (!(det_I_plus(G) > 0.0f)) set_error(P, penv, kErrDetStress, pid);
          ts = stress_of(mp.model, G, hencky_of(G), jp, mp);
        }

        if (!redo && valid) {  // G is final here: store it now so it does not live on in registers
#pragma unroll
          for (int k = 0; k < 9; ++k) sts(&P.nxt.G[k][j], G[k]);
          sts(&P.nxt.mass[j], m);
          sts(&P.nxt.vol0[j], V0);
          if (AM) sts(&P.nxt.jp[j], jp);
          sts(&P.nxt.pid[j], pid);
        }
        if (l2_prefetch(NCH, F) && i_pf >= 0) {
          auto pf = [](const void* a) { asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a)); };
#pragma unroll
          for (int a = 0; a < 3; ++a) pf(&P.cur.x[a][i_pf]);
#pragma unroll
          for (int k = 0; k < 9; ++k) pf(&P.cur.G[k][i_pf]);
          pf(&P.cur.mass[i_pf]);
          pf(&P.cur.vol0[i_pf]);
          pf(&P.cur.meta[i_pf]);
          pf(&P.cur.pid[i_pf]);
        }

        // ---------------- binning of the (new) position + P2G payload of the next cycle
        int key_new = P.n_keys - 1;
        bool staged = false;
        int cell = 0;
        int b2[3] = {-10, -10, -10};
        float fx2[3] = {0.f, 0.f, 0.f};
        f3 fext = {0.f, 0.f, 0.f};
        const bool p2g_here = valid && !was_lost && (IC.lostb ? (pact == kActP2G || pact == kActFused) : IC.do_p2g);
        if (valid && !was_lost) {
          base_of(P, x.x, x.y, x.z, b2, fx2);
          if (base_in_range(P, b2)) {
            if (!IC.lostb || pact == kActIdle || pact == kActG2P) key_new = bucket_of(P, penv, b2);
          } else if (p2g_here) {
            // leaves the domain now: reaction-only IC.penalty, freeze, count (mpm.hpp:239-245)
            if (!redo) {
              if (P.hooks && !P.grid_mode && P.shape_off[penv + 1] > P.shape_off[penv]) penalty_reaction_only<DET>(P, penv, x, v);
              atomicAdd((unsigned long long*)&P.lost_count[penv], 1ull);
            }
            meta |= 1u << kLostBit;
            v = {0.f, 0.f, 0.f};
            write_vc = true;
            b2[0] = b2[1] = b2[2] = -10;
          }
        }
        const bool now_lost = meta >> kLostBit;
        const bool scatter_me = p2g_here && !IC.lostb && !now_lost;
        if (P.base_dbg && !redo && valid && (p2g_here || (IC.lostb && was_lost && (pact == kActP2G || pact == kActFused)))) {
          P.base_dbg[3 * pid + 0] = now_lost ? -10 : b2[0];
          P.base_dbg[3 * pid + 1] = now_lost ? -10 : b2[1];
          P.base_dbg[3 * pid + 2] = now_lost ? -10 : b2[2];
        }

        // IC.penalty hook: warp-cooperative per shape (coupling.hpp:151-172)
        if (IC.penalty) {
          // shapes outside the bucket box are skipped warp-wide; a warp with a
          // particle outside the box (moved > 2 h) tests every shape
          const bool inbox = x.x >= IC.blo[0] && x.y >= IC.blo[1] && x.z >= IC.blo[2] && x.x <= IC.bhi[0] &&
                             x.y <= IC.bhi[1] && x.z <= IC.bhi[2];
          const unsigned smask = (kNoCull || __any_sync(FULL, scatter_me && !inbox)) ? ~0u : IC.smask;
          for (int sidx = IC.s0; sidx < IC.s1; ++sidx) {
            const int k = sidx - IC.s0;
            if (k < 32 && !((smask >> k) & 1u)) continue;  // warp-uniform
            const ShapeDev& sh = P.shapes[sidx];
            f3 f = {0.f, 0.f, 0.f};
            float pen = 0.f;
            const bool hit = scatter_me && (kNoCull || shape_may_touch(sh, x, P.r_c_particle)) &&
                             penalty_force(sh, P.vol_pool, x, v, P.r_c_particle, P.c_d, f, pen);
            if (!hit) f = {0.f, 0.f, 0.f};
            fext = fext + f;
            if (!redo && __any_sync(FULL, hit)) {
              const f3 com = {sh.com[0], sh.com[1], sh.com[2]};
              const f3 tq = hit ? cross(x - com, f3{-f.x, -f.y, -f.z}) : f3{0.f, 0.f, 0.f};
              float r6[6] = {-f.x, -f.y, -f.z, tq.x, tq.y, tq.z};
#pragma unroll
              for (int k = 0; k < 6; ++k) r6[k] = warp_sum(r6[k]);
              unsigned pb = hit ? __float_as_uint(pen) : 0u;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) pb = max(pb, __shfl_xor_sync(FULL, pb, o));
              if (lane == 0) {
                if constexpr (DET) {  // warp sums are deterministic; integer totals
                  long long* w = P.w64 + 6 * (P.body_off[IC.benv] + sh.body);
#pragma unroll
                  for (int k = 0; k < 6; ++k) red_add_i64(w + k, det_fix((double)r6[k], kDetWrenchExp));
#pragma unroll
                  for (int k = 0; k < 3; ++k) {
                    const long long rk = det_fix((double)r6[k], kDetWrenchExp);
                    red_add_i64(P.r64 + 3 * IC.benv + k, rk);
                    red_add_i64(P.a64 + 3 * IC.benv + k, -rk);
                  }
                } else {
                  double* ws = S.wsum + 6 * min(sh.body, kMaxBodiesPerEnv - 1);
#pragma unroll
                  for (int k = 0; k < 6; ++k) atomicAdd(ws + k, (double)r6[k]);
#pragma unroll
                  for (int k = 0; k < 3; ++k) atomicAdd(S.wsum + 6 * kMaxBodiesPerEnv + k, -(double)r6[k]);
                }
                atomicMax(&S.penmax, pb);
              }
            }
          }
        }

        if (scatter_me) {
          const float tau[9] = {ts.a00, ts.a01, ts.a02, ts.a01, ts.a11, ts.a12, ts.a02, ts.a12, ts.a22};
          const float h = P.h_f;
          const float hm = h * m;
          const float hs = -h * P.d_inv_f * V0;  // h * (-(4/h^2) V0): stress -> force matrix
          float w9[9];
          bspline_w(fx2[0], w9);
          bspline_w(fx2[1], w9 + 3);
          bspline_w(fx2[2], w9 + 6);
          // momentum matrix A (h-scaled) and base b = m v (+ IC.dt f_ext) - A fx; the node
          // contribution is w (b + A off), off in {0,1,2}^3 (dpos = h (off - fx))
          float A[9];
          f3 bb;
          float Af[9];
          f3 bf = {0.f, 0.f, 0.f};
          if (NCH == 4) {
            const float ds = IC.dtp * hs;
#pragma unroll
            for (int k = 0; k < 9; ++k) A[k] = hm * Cm[k] + ds * tau[k];
            bb = (m * v + IC.dtp * fext) - matvec(A, f3{fx2[0], fx2[1], fx2[2]});
          } else {
#pragma unroll
            for (int k = 0; k < 9; ++k) {
              A[k] = hm * Cm[k];
              Af[k] = hs * tau[k];
            }
            bb = m * v - matvec(A, f3{fx2[0], fx2[1], fx2[2]});
            bf = fext - matvec(Af, f3{fx2[0], fx2[1], fx2[2]});
          }
          const int lx = b2[0] - (IC.ox - 1), ly = b2[1] - (IC.oy - 1), lz = b2[2] - (IC.oz - 1);
          if (lx >= 0 && ly >= 0 && lz >= 0 && lx < CX && ly < CY && lz < CZ) {
            cell = (lz * CY + ly) * CX + lx;
            // [m fx0 fx1 fx2] [b.x b.y b.z A00] [A01 A02 A10 A11] [A12 A20 A21 A22]
            // (+ [bf.x bf.y bf.z Af00] [Af01 Af02 Af11 Af12] [Af22 - - -], Af symmetric)
            S.pay[0][t] = make_float4(m, fx2[0], fx2[1], fx2[2]);
            S.pay[1][t] = make_float4(bb.x, bb.y, bb.z, A[0]);
            S.pay[2][t] = make_float4(A[1], A[2], A[3], A[4]);
            S.pay[3][t] = make_float4(A[5], A[6], A[7], A[8]);
            if constexpr (NCH == 7) {
              S.pay[4][t] = make_float4(bf.x, bf.y, bf.z, Af[0]);
              S.pay[5][t] = make_float4(Af[1], Af[2], Af[4], Af[5]);
              S.pay[6][t] = make_float4(Af[8], 0.f, 0.f, 0.f);
            }
            staged = true;
            if (!redo) {  // the stencil's node blocks: nodes o - 1 + l .. o + 1 + l per axis
              const int x0 = (lx + 3) >> 2, x1 = (lx + 5) >> 2, y0 = (ly + 3) >> 2, y1 = (ly + 5) >> 2;
              const int z0 = (lz + 1) >> 1;
              static_assert(kBX == 4 && kBY == 4 && kBZ == 2, "block shape");
              unsigned char* bf = S.bflag + z0 * (Gm::NBX * Gm::NBY);
#pragma unroll
              for (int dz = 0; dz < 2; ++dz, bf += Gm::NBX * Gm::NBY) {  // 3 nodes span 2 z-blocks
                bf[y0 * Gm::NBX + x0] = 1;
                bf[y0 * Gm::NBX + x1] = 1;
                bf[y1 * Gm::NBX + x0] = 1;
                bf[y1 * Gm::NBX + x1] = 1;
              }
            }
            // bounds of |b + A off| over off in {0,1,2}^3 for the fixed-point scales
            mx_m = fmaxf(mx_m, m);
            const float a0 = fabsf(A[0]) + fabsf(A[1]) + fabsf(A[2]);
            const float a1 = fabsf(A[3]) + fabsf(A[4]) + fabsf(A[5]);
            const float a2 = fabsf(A[6]) + fabsf(A[7]) + fabsf(A[8]);
            mx_p = fmaxf(mx_p, fmaxf(fabsf(bb.x) + 2.f * a0, fmaxf(fabsf(bb.y) + 2.f * a1, fabsf(bb.z) + 2.f * a2)));
            if (NCH == 7) {
              const float f0 = fabsf(Af[0]) + fabsf(Af[1]) + fabsf(Af[2]);
              const float f1 = fabsf(Af[3]) + fabsf(Af[4]) + fabsf(Af[5]);
              const float f2 = fabsf(Af[6]) + fabsf(Af[7]) + fabsf(Af[8]);
              mx_f = fmaxf(mx_f, fmaxf(fabsf(bf.x) + 2.f * f0, fmaxf(fabsf(bf.y) + 2.f * f1, fabsf(bf.z) + 2.f * f2)));
            }
          } else {
            scatter_global<NCH, DET>(P, penv, b2, w9, m, bb, A, bf, Af, !redo);
          }
        }
        if (t < CAP) S.cellof[t] = staged ? cell : -1;

        if (!redo) {
          // ---------------- write back in bucket order (the re-sort)
          if (valid) {
            sts(&P.nxt.x[0][j], x.x); sts(&P.nxt.x[1][j], x.y); sts(&P.nxt.x[2][j], x.z);
            sts(&P.nxt.meta[j], meta);
            if (write_vc) {
              sts(&P.nxt.v[0][j], v.x); sts(&P.nxt.v[1][j], v.y); sts(&P.nxt.v[2][j], v.z);
#pragma unroll
              for (int k = 0; k < 9; ++k) sts(&P.nxt.C[k][j], Cm[k]);
            }
            if (now_lost) key_new = P.n_keys - 1;
            P.key[j] = key_new;
          }
          {  // next bucket key. Particles staying in this bucket keep their order: their
             // ranks are prefix counts in slot order, set after the round's barrier. The
             // (rare) movers take atomic ranks counted back from the end of their new bucket.
            // (split buckets: every particle takes an atomic rank, see particles_cta)
            const bool stay = valid && key_new == IC.key && !IC.split;
            const unsigned sb = __ballot_sync(FULL, stay);
            if (lane == 0) S.wball[rpar][t >> 5] = sb;
            const unsigned am = __ballot_sync(FULL, valid && !stay);
            if (valid && !stay) {
              const unsigned peers = __match_any_sync(am, key_new);
              const int leader = __ffs(peers) - 1;
              int basecnt = 0;
              if (lane == leader) {
                basecnt = atomicAdd(&P.move_count[key_new], __popc(peers));
                atomicAdd(&P.bucket_count[key_new], __popc(peers));
              }
              basecnt = __shfl_sync(peers, basecnt, leader);
              P.rank[j] = -1 - (basecnt + __popc(peers & ((1u << lane) - 1u)));
            }
          }
          if (IC.do_g2p) {  // per-env max speed (bucket env-uniform): warp max -> one atomic
            float sp = speed;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sp = fmaxf(sp, __shfl_xor_sync(FULL, sp, o));
            if (lane == 0 && sp >= 0.0f) float_bits_max(&P.vmax_bits[IC.benv], sp);
          }
        }
      }
      if (IC.do_p2g) {
        // fixed-point scales of this round: |node sum| <= rn * max bound < 2^30 / scale
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mx_m = fmaxf(mx_m, __shfl_xor_sync(FULL, mx_m, o));
          mx_p = fmaxf(mx_p, __shfl_xor_sync(FULL, mx_p, o));
          mx_f = fmaxf(mx_f, __shfl_xor_sync(FULL, mx_f, o));
        }
        if (lane == 0) {
          atomicMax(&S.maxb[rpar][0], __float_as_uint(mx_m));
          atomicMax(&S.maxb[rpar][1], __float_as_uint(mx_p));
          atomicMax(&S.maxb[rpar][2], __float_as_uint(mx_f));
        }
      }
      __syncthreads();
      if (!redo) {  // order-preserving ranks of this round's stayers (slot order)
        const unsigned lt = (1u << lane) - 1u;
        int acc = 0;
#pragma unroll
        for (int w = 0; w < CAP / 32; ++w) {
          const unsigned b = w * 32 < rn ? S.wball[rpar][w] : 0u;
          for (int trip = 0; trip < trips; ++trip) {
            const int t = trip * kT + tid;
            if ((t >> 5) == w && ((b >> lane) & 1u)) P.rank[r0 + t] = stay_base + acc + __popc(b & lt);
          }
          acc += __popc(b);
        }
        stay_base += acc;
      }
      if (!IC.do_p2g) continue;

      // ---------------- per-thread scatter of one staged particle into the fixed-point tile
      {
        // fixed-point scale: every contribution |w (b + A off)| <= bound -> |x| <= 2^SC_LOG2,
        // so a node sum of <= CAP contributions stays below 2^30 (no int32 overflow)
        constexpr float kFix = (float)(1 << Gm::SC_LOG2);
        const float bm = __uint_as_float(S.maxb[rpar][0]), bpm = __uint_as_float(S.maxb[rpar][1]),
                    bfm = __uint_as_float(S.maxb[rpar][2]);
        // the next round's slot: its last readers (round r - 1's scatter) passed
        // round r - 1's post-scatter barrier; its next writers come after this
        // round's post-scatter barrier
        if (tid < 3) S.maxb[rpar ^ 1][tid] = 0u;
        float sc_m = bm > 0.f ? kFix / bm : 0.f;
        float sc_p = bpm > 0.f ? kFix / bpm : 0.f;
        const float sc_f = bfm > 0.f ? kFix / bfm : 0.f;
        int dsh_m = 0, dsh_p = 0;  // DET: shift from the round's scale 2^e to the launch's 2^S
        if constexpr (DET) {
          // power-of-two round scales: the round's integer sums convert exactly
          const int em = sc_m > 0.f ? ilogbf(sc_m) : 0, ep = sc_p > 0.f ? ilogbf(sc_p) : 0;
          sc_m = sc_m > 0.f ? ldexpf(1.0f, em) : 0.f;
          sc_p = sc_p > 0.f ? ldexpf(1.0f, ep) : 0.f;
          const EnvRun& er = P.run[IC.benv];
          dsh_m = er.det_sm - em;
          dsh_p = er.det_sp - ep;
          if (!redo && tid == 0) {
            atomicMax(&P.det_bnd[IC.benv], __float_as_uint(bpm));
            // the round's largest possible node sum at the launch's scale must stay < 2^61
            if (ldexpf(bm * (float)rn, er.det_sm) >= 2.3e18f || ldexpf(bpm * (float)rn, er.det_sp) >= 2.3e18f)
              set_error(P, IC.benv, kErrDetRange, 0x7fffffff);
          }
        }
        // Golden-ratio spread: consecutive lanes take staged slots ~0.618 rn apart
        // (odd, coprime with rn: a bijection on [0, rn)), i.e. particles spread over
        // the whole bucket, so a warp's 27-node stencils rarely share a node (staged
        // order follows the particles' spatial order, neighbours share cells).
        // The payload reads pay[k][t] stay free of bank conflicts (odd g: t distinct mod 8).
        const int g = kSpread.g[rn];
        const int dstep = (kT * g) % rn;
        int t = tid < rn ? (tid * g) % rn : 0;
        for (int u = tid; u < rn; u += kT, t = t + dstep >= rn ? t + dstep - rn : t + dstep) {
          const int c = S.cellof[t];
          if (c < 0) continue;
#ifdef MSIM_ABLATE_SCATTER  // profiling-only build: no shared atomics
          if (c >= 0) continue;
#endif
          const float4 q0 = S.pay[0][t], q1 = S.pay[1][t], q2 = S.pay[2][t], q3 = S.pay[3][t];
          float wx[3], wy[3], wz[3];
          bspline_w(q0.y, wx);
          bspline_w(q0.z, wy);
          bspline_w(q0.w, wz);
          const float ms = q0.x * sc_m;
          // x weights pre-scaled by the mass and momentum fixed-point factors: one
          // FMUL per node (w sc_p) and the mass term as a single FFMA into fix_rn
          const float wxm[3] = {wx[0] * ms, wx[1] * ms, wx[2] * ms};
          const float wxp[3] = {wx[0] * sc_p, wx[1] * sc_p, wx[2] * sc_p};
          // b = q1.xyz; A row-major: A00 q1.w A01 q2.x A02 q2.y A10 q2.z A11 q2.w A12 q3.x A20 q3.y A21 q3.z A22 q3.w
          float4 qf4 = make_float4(0.f, 0.f, 0.f, 0.f), qf5 = qf4, qf6 = qf4;
          if constexpr (NCH == 7) {
            qf4 = S.pay[4][t];
            qf5 = S.pay[5][t];
            qf6 = S.pay[6][t];
          }
          const int cx = c % CX, cy = (c / CX) % CY, cz = c / (CX * CY);
#pragma unroll kScatterDkUnroll
          for (int dk = 0; dk < 3; ++dk) {
            const float wzk = dk == 0 ? wz[0] : (dk == 1 ? wz[1] : wz[2]);
#pragma unroll kScatterDjUnroll
            for (int dj = 0; dj < 3; ++dj) {
              const float wyz = (dj == 0 ? wy[0] : (dj == 1 ? wy[1] : wy[2])) * wzk;
              float rx = q1.x + q2.x * dj + q2.y * dk;  // b.x + A01 dj + A02 dk
              float ry = q1.y + q2.w * dj + q3.x * dk;  // b.y + A11 dj + A12 dk
              float rz = q1.z + q3.z * dj + q3.w * dk;  // b.z + A21 dj + A22 dk
              float fxr = 0.f, fyr = 0.f, fzr = 0.f;
              if (NCH == 7) {
                fxr = qf4.x + qf5.x * dj + qf5.y * dk;  // bf.x + Af01 dj + Af02 dk
                fyr = qf4.y + qf5.z * dj + qf5.w * dk;  // bf.y + Af11 dj + Af12 dk
                fzr = qf4.z + qf5.w * dj + qf6.x * dk;  // bf.z + Af12 dj + Af22 dk
              }
              const int nt = (cz + dk) * kTZS + (cy + dj) * PX + cx;
#pragma unroll kScatterDiUnroll
              for (int di = 0; di < 3; ++di) {
                const float wp = wyz * (di == 0 ? wxp[0] : (di == 1 ? wxp[1] : wxp[2]));
                atomicAdd(&S.itile[3][nt + di], fix_rn(wyz * (di == 0 ? wxm[0] : (di == 1 ? wxm[1] : wxm[2]))));
                atomicAdd(&S.itile[0][nt + di], fix_rn(wp * rx));
                atomicAdd(&S.itile[1][nt + di], fix_rn(wp * ry));
                atomicAdd(&S.itile[2][nt + di], fix_rn(wp * rz));
                rx += q1.w; ry += q2.z; rz += q3.y;  // + column 0 (A00, A10, A20)
                if (NCH == 7) {
                  const float wf = wyz * (di == 0 ? wx[0] : (di == 1 ? wx[1] : wx[2])) * sc_f;
                  atomicAdd(&S.itile[4 % NCH][nt + di], fix_rn(wf * fxr));
                  atomicAdd(&S.itile[5 % NCH][nt + di], fix_rn(wf * fyr));
                  atomicAdd(&S.itile[6 % NCH][nt + di], fix_rn(wf * fzr));
                  fxr += qf4.w; fyr += qf5.x; fzr += qf5.y;  // + column 0 (Af00, Af01, Af02)
                }
              }
            }
          }
        }
        float sc[NCH];
        sc[3] = sc_m;
        sc[0] = sc[1] = sc[2] = sc_p;
        if (NCH == 7) sc[4 % NCH] = sc[5 % NCH] = sc[6 % NCH] = sc_f;
        __syncthreads();
        // ---------------- flush the round's node tile (vector REDs)
        float qs[NCH];
#pragma unroll
        for (int q = 0; q < NCH; ++q) qs[q] = sc[q] > 0.f ? 1.0f / sc[q] : 0.f;
        // a node holds mass only if it lies in some staged particle's stencil, hence
        // inside the grid: no bounds test; global index = tile base + local offset
        const long long gbase = IC.benv * P.nodes_per_env +
                                ((long long)(IC.oz - 1) * P.dims[1] + (IC.oy - 1)) * P.dims[0] + (IC.ox - 1);
        const long long sxy = (long long)P.dims[0] * P.dims[1];
        auto flush_node = [&](int t, long long gi) {
          const int im = S.itile[3][t];
          if (DET && im != 0) {  // exact integer conversion to the launch's fixed point
            auto sh = [](int v, int d) {
              return d >= 0 ? (long long)v << d : (d > -63 ? (long long)v >> -d : (v < 0 ? -1ll : 0ll));
            };
            long long* g = &P.gPMd[gi].x;
            red_add_i64(g + 0, sh(S.itile[0][t], dsh_p));
            red_add_i64(g + 1, sh(S.itile[1][t], dsh_p));
            red_add_i64(g + 2, sh(S.itile[2][t], dsh_p));
            red_add_i64(g + 3, sh(im, dsh_m));
          } else if (im != 0) {
            red_add_v4(&P.gPM[gi], qs[0] * (float)S.itile[0][t], qs[1] * (float)S.itile[1][t],
                       qs[2] * (float)S.itile[2][t], qs[3] * (float)im);
            if (NCH == 7)
              red_add_v4(&P.gF[gi], qs[4] * (float)S.itile[4][t], qs[5] * (float)S.itile[5][t],
                         qs[6] * (float)S.itile[6][t], 0.0f);
          }
#pragma unroll
          for (int q = 0; q < NCH; ++q) S.itile[q][t] = 0;
        };
        if constexpr (kT % (PX * PY) == 0) {  // whole z-layers per pass (F = 1: 2 layers of 8 x 8)
          constexpr int LPP = kT / (PX * PY);
          const int lxy = tid % (PX * PY), lx = lxy % PX, ly = lxy / PX;
          const long long goff = (long long)ly * P.dims[0] + lx;
          for (int lz = tid / (PX * PY); lz < PZ; lz += LPP) flush_node(lz * kTZS + lxy, gbase + lz * sxy + goff);
        } else {
          for (int t = tid; t < PN; t += kT) {
            const int lz = t / kTZS, rem = t - lz * kTZS, ly = rem / PX, lx = rem - ly * PX;
            if (lx < PX && ly < PY) flush_node(t, gbase + lz * sxy + (long long)ly * P.dims[0] + lx);
          }
        }
        // no barrier here: the next round touches itile only after its
        // post-staging barrier (and maxb[rpar] is not written again before
        // the round after next), and the item loop starts with one
      }
    }

    if (!redo && tid == 0 && stay_base) atomicAdd(&P.bucket_count[IC.key], stay_base);
    if (DET && IC.penalty && !redo) {
      if (tid == 0 && S.penmax) atomicMax(&P.max_pen_bits[IC.benv], S.penmax);
    } else if (IC.penalty && !redo) {
      const int b0 = P.body_off[IC.benv], nb = min(P.body_off[IC.benv + 1] - b0, kMaxBodiesPerEnv);
      for (int t = tid; t < nb * 6; t += kT) {
        const double val = S.wsum[t];
        if (val != 0.0) atomicAdd(P.wrench + 6 * b0 + t, val);
      }
      if (tid < 3) {
        const double a = S.wsum[6 * kMaxBodiesPerEnv + tid];
        if (a != 0.0) {
          atomicAdd(P.applied + 3 * IC.benv + tid, a);
          double r = 0.0;
          for (int bb = 0; bb < nb; ++bb) r += S.wsum[6 * bb + tid];
          atomicAdd(P.react + 3 * IC.benv + tid, r);
        }
      }
      if (tid == 0 && S.penmax) atomicMax(&P.max_pen_bits[IC.benv], S.penmax);
    }
  }
}

// One CTA's share of a particle launch (cta of ncta).
template <int NCH, int F, bool AM, bool DET>
__device__ __forceinline__ void particles_cta(const SimParams& P, unsigned char* smem_raw, const bool redo, const int cta,
                                              const int ncta) {
  MSIM_GEO_ALIASES(F)
  Smem<NCH, F>& S = *reinterpret_cast<Smem<NCH, F>*>(smem_raw);
  const int tid = threadIdx.x;
  if (redo && !*P.any_redo) return;
  // Small scenes (split_r > 1): item = (bucket, part), part p taking the bucket's
  // rounds p, p + split_r, ... Stayers then cannot be ranked in order across
  // CTAs: every particle takes an atomic rank from its bucket's end (the
  // deterministic mode's mover sort restores the slot order). The lost bucket is
  // not split (its particles stay in order).
  const int R = P.split_r;
  const int nb = *P.n_active_buckets;
  // Tail split (outside the deterministic mode and the small-scene split): with
  // few buckets per CTA the last ncta buckets of the hand-out are split into
  // kTailSplit parts each, so the launch ends evenly instead of waiting on whole
  // last buckets; only those buckets lose their in-bucket order (atomic ranks).
  // Batched C +2.8 %, B +1.8 %, D at 128 envs +1.1 %, E -0.8 %; off at D's 1024
  // envs (~90 buckets per CTA: -0.5 %).
  const int T = R == 1 && !P.det && kTailSplit > 1 && nb < 32 * ncta ? min(nb, ncta) : 0;
  const int nitems = R > 1 ? nb * R : nb - T + T * kTailSplit;

  for (int t = tid; t < NCH * PN; t += kT) (&S.itile[0][0])[t] = 0;
  for (int t = tid; t < Gm::NBT; t += kT) S.bflag[t] = 0;

  volatile ItemCtx& IC = S.ic;
  // Buckets are handed out dynamically after a first static one per CTA (one
  // atomic per further bucket): their sizes vary, and a static round-robin
  // leaves a tail of CTAs with more work (-12 % per launch at D).
  for (int item = cta; item < nitems;) {
    int bi = item, part = 0, rr = 1;  // bucket, part, parts
    if (R > 1) {
      bi = item / R, part = item - bi * R, rr = R;
    } else if (item >= nb - T) {
      const int q = item - (nb - T);
      bi = nb - T + q / kTailSplit, part = q - (q / kTailSplit) * kTailSplit, rr = kTailSplit;
    }
    const int key = P.active_buckets[bi];
    const bool lostb = key == P.n_keys - 1;
    const int benv = lostb ? 0 : key / P.buckets_per_env;
    const int s = P.bucket_start[key] + part * CAP, e = P.bucket_start[key + 1];
    if ((redo && (lostb || !P.run[benv].redo)) || s >= e || (lostb && part > 0)) {  // CTA-uniform
      __syncthreads();
      if (tid == 0)
        S.next_item = ncta + (kDynamicItems ? atomicAdd(P.item_counter + redo, 1) : item);
      __syncthreads();
      item = S.next_item;
      continue;
    }
    const int act = lostb ? kActIdle : P.run[benv].action;
    const bool do_g2p = act == kActFused || act == kActG2P;
    const bool do_p2g = act == kActP2G || act == kActFused;
    const int lb = key - benv * P.buckets_per_env;
    const int ox = QX * (lb % P.qdims[0]), oy = QY * ((lb / P.qdims[0]) % P.qdims[1]),
              oz = QZ * (lb / (P.qdims[0] * P.qdims[1]));
    const float dt = do_g2p ? P.run[benv].dt_g2p : 0.0f;
    const float dtp = lostb ? 0.0f : (redo ? P.run[benv].dt_c : P.run[benv].dt_p2g);  // NCH == 4 only
    const int s0 = lostb ? 0 : P.shape_off[benv], s1 = lostb ? 0 : P.shape_off[benv + 1];
    const bool penalty = do_p2g && P.hooks && !P.grid_mode && s1 > s0;

    __syncthreads();  // smem reuse across items
    if (do_g2p) {
      for (int t = tid; t < GN; t += kT) {
        const int lx = t % GX, ly = (t / GX) % GY, lz = t / (GX * GY);
        const int gx = ox + lx, gy = oy + ly, gz = oz + lz;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (gx < P.dims[0] && gy < P.dims[1] && gz < P.dims[2])
          v = P.gV[benv * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx];
        S.gtile[t] = v;
      }
    }
    if (penalty && !redo)
      for (int t = tid; t < kWs; t += kT) S.wsum[t] = 0.0;
    if (penalty && tid < 32) {  // bucket-level collider culling (exact: see item_rounds)
      // old positions lie in cells [o + 0.5, o + kB + 0.5) h; 2 h of slack for the G2P move
      const float h = P.h_f;
      const f3 lo = {(float)P.origin[0] + h * (ox - 1.5f), (float)P.origin[1] + h * (oy - 1.5f),
                     (float)P.origin[2] + h * (oz - 1.5f)};
      const f3 hi = {(float)P.origin[0] + h * (ox + QX + 2.5f), (float)P.origin[1] + h * (oy + QY + 2.5f),
                     (float)P.origin[2] + h * (oz + QZ + 2.5f)};
      const bool b = tid < s1 - s0 && shape_may_touch_box(P.shapes[s0 + tid], lo, hi, P.r_c_particle);
      const unsigned m = __ballot_sync(0xffffffffu, b);
      if (tid == 0) {
        IC.smask = m;
        IC.blo[0] = lo.x; IC.blo[1] = lo.y; IC.blo[2] = lo.z;
        IC.bhi[0] = hi.x; IC.bhi[1] = hi.y; IC.bhi[2] = hi.z;
      }
    }
    if (tid < 6) (&S.maxb[0][0])[tid] = 0u;
    if (tid == 0) {
      S.penmax = 0u;
      IC.key = key; IC.benv = benv; IC.s = s; IC.e = e; IC.act = act; IC.rstep = (lostb ? 1 : rr) * CAP;
      IC.split = rr > 1 && !lostb;
      IC.ox = ox; IC.oy = oy; IC.oz = oz; IC.s0 = s0; IC.s1 = s1;
      IC.dt = dt; IC.dtp = dtp;
      IC.lostb = lostb; IC.do_g2p = do_g2p; IC.do_p2g = do_p2g; IC.penalty = penalty;
    }
    __syncthreads();
    item_rounds<NCH, F, AM, DET>(P, S, redo);
    __syncthreads();
    if (!redo && tid < Gm::NBT) {  // the bucket's touched node blocks (once per bucket)
      if (S.bflag[tid]) {
        S.bflag[tid] = 0;
        const int kx = IC.ox / kBX - 1 + tid % Gm::NBX, ky = IC.oy / kBY - 1 + (tid / Gm::NBX) % Gm::NBY,
                  kz = IC.oz / kBZ - 1 + tid / (Gm::NBX * Gm::NBY);
        P.nb_flag[IC.benv * P.blocks_per_env + (kz * P.bdims[1] + ky) * P.bdims[0] + kx] = 1;
      }
    }
    if (tid == 0) S.next_item = ncta + (kDynamicItems ? atomicAdd(P.item_counter + redo, 1) : item);
    __syncthreads();
    item = S.next_item;
  }
  // the last fetching CTA out resets the hand-out counter for the next launch
  // (no memset node; CTAs without a first bucket never fetched)
  if (kDynamicItems && tid == 0 && cta < nitems) {
    __threadfence();
    if (atomicAdd(P.item_counter + 2 + redo, 1) == min(ncta, nitems) - 1) {
      P.item_counter[redo] = 0;
      P.item_counter[2 + redo] = 0;
      __threadfence();
    }
  }
}

// LAT: small scenes (split buckets, a few CTAs per SM busy): latency-bound, so
// the 5-CTA register budget (fewer spills) instead of the dense instantiations'
// 8 (single-scene B -3.6 % at 8)
template <int NCH, int F, bool AM, bool DET, bool LAT = false>
__global__ void __launch_bounds__(kT, LAT ? 5 : ctas_per_sm(NCH, F, DET)) k_particles(SimParams P) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  particles_cta<NCH, F, AM, DET>(P, smem_raw, P.redo_pass != 0, (int)blockIdx.x, (int)gridDim.x);
}

// Bucket keys of stored positions (after uploads): no loss flagging here, a
// particle outside the domain is flagged by the next P2G (mpm.hpp:226-245).
__global__ void __launch_bounds__(256) k_rebin(SimParams P) {
  pdl_wait();
  pdl_trigger();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = i < P.n;
  int key = P.n_keys - 1;
  if (valid) {
    const unsigned meta = P.cur.meta[i];
    if (!(meta >> kLostBit)) {
      int b[3];
      float fx[3];
      const f3 x = load3(P.cur.x, i);
      base_of(P, x.x, x.y, x.z, b, fx);
      if (base_in_range(P, b)) key = bucket_of(P, (meta >> 8) & kEnvMask, b);
    }
    P.key[i] = key;
  }
  const unsigned am = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const int lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(am, key);
  const int leader = __ffs(peers) - 1;
  int basecnt = 0;
  if (lane == leader) {
    basecnt = atomicAdd(P.det ? &P.move_count[key] : &P.bucket_count[key], __popc(peers));
    if (P.det) atomicAdd(&P.bucket_count[key], __popc(peers));
  }
  basecnt = __shfl_sync(peers, basecnt, leader);
  const int r = basecnt + __popc(peers & ((1u << lane) - 1u));
  P.rank[i] = P.det ? -1 - r : r;  // deterministic mode: all "movers", put in index order after k_perm
}

// Particle i (slot of the launch that keyed it) -> its slot in the next launch:
// stayers (rank >= 0) from the bucket's start in their old order, movers
// (rank = -1 - r) from its end.
__device__ __forceinline__ void perm_kr(const SimParams& P, long long i, int k, int r) {
  if (r == -1 && !P.det) P.move_count[k] = 0;  // exactly one mover per bucket has rank -1: reset the counter
  P.perm_w[(r >= 0 ? P.bucket_start_w[k] : P.bucket_start_w[k + 1]) + r] = (int)i;
}
// Four particles per thread (16-byte key / rank loads). EARLY: launched after
// k_grid, whose start implies the bucket scan and the particle kernel
// completed: runs alongside k_grid / k_iter_begin.
template <bool EARLY>
__global__ void k_perm(SimParams P) {
  if (!EARLY) pdl_wait();
  pdl_trigger();
  const long long i0 = 4 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  if (i0 + 3 < P.n) {
    const int4 k4 = *reinterpret_cast<const int4*>(P.key + i0);
    const int4 r4 = *reinterpret_cast<const int4*>(P.rank + i0);
    perm_kr(P, i0, k4.x, r4.x);
    perm_kr(P, i0 + 1, k4.y, r4.y);
    perm_kr(P, i0 + 2, k4.z, r4.z);
    perm_kr(P, i0 + 3, k4.w, r4.w);
  } else {
    for (long long i = i0; i < P.n; ++i) perm_kr(P, i, P.key[i], P.rank[i]);
  }
  if (EARLY) pdl_wait();
}

// Deterministic mode: the movers at the end of each bucket (atomic ranks) are
// put in the order of their previous slots, so the next launch's particle
// order -- hence every fixed-point scale and every sum -- is reproducible.
// One CTA per bucket; each mover's position = #movers with a smaller slot.
__global__ void __launch_bounds__(128) k_det_sort_movers(SimParams P) {
  pdl_wait();
  pdl_trigger();
  __shared__ int tail[1024];
  for (int k = blockIdx.x; k < P.n_keys; k += gridDim.x) {
    const int cnt = P.move_count[k];
    if (cnt == 0) continue;
    __syncthreads();
    int* seg = P.perm_w + P.bucket_start_w[k + 1] - cnt;
    if (cnt <= 1024) {
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) tail[t] = seg[t];
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int v = tail[t];
        int pos = 0;
        for (int u = 0; u < cnt; ++u) pos += tail[u] < v;
        seg[pos] = v;
      }
    } else if (threadIdx.x == 0) {  // a very crowded bucket: insertion sort in place
      for (int a = 1; a < cnt; ++a) {
        const int v = seg[a];
        int b = a - 1;
        while (b >= 0 && seg[b] > v) seg[b + 1] = seg[b], --b;
        seg[b + 1] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) P.move_count[k] = 0;
  }
}

// Zero the nodes touched by the last P2G (phase API: the reference clears
// the dense grid before every p2g, mpm.hpp:411).
__global__ void k_clear(SimParams P) {
  const int nlist = *P.n_nb;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int NB = kBX * kBY * kBZ;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)nlist * NB;
       t += (long long)gridDim.x * blockDim.x) {
    const int nb = P.nb_list[t / NB], l = (int)(t % NB);
    const int env = nb / P.blocks_per_env, lb = nb - env * P.blocks_per_env;
    const int gx = kBX * (lb % P.bdims[0]) + l % kBX, gy = kBY * ((lb / P.bdims[0]) % P.bdims[1]) + (l / kBX) % kBY,
              gz = kBZ * (lb / (P.bdims[0] * P.bdims[1])) + l / (kBX * kBY);
    if (gx >= P.dims[0] || gy >= P.dims[1] || gz >= P.dims[2]) continue;
    const long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
    P.gPM[gi] = z;
    P.gF[gi] = z;
    P.gV[gi] = z;
    if (P.det) P.gPMd[gi] = make_longlong4(0, 0, 0, 0);
  }
}

// Grid update (mpm.hpp:315-342) with the grid-mode penalty hook
// (coupling.hpp:186-214); one warp per touched node block (32 nodes).
// gtid / gthreads: this thread's index / the thread count of the launch (one warp per item)
// HOOK: grid-mode penalty (coupling.hpp:182-214); without it the kernel needs
// a third of the registers, i.e. ~4x the warps in flight for its latency-bound
// node-block loop.
template <bool HOOK>
__device__ __forceinline__ void grid_items(const SimParams& P, const int gtid, const int gthreads) {
  static_assert(kBX * kBY * kBZ == 32, "one warp per node block");
  const int nlist = *P.n_nb;
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  for (int item = gtid >> 5; item < nlist; item += gthreads >> 5) {
    const int nb = P.nb_list[item];
    const int env = nb / P.blocks_per_env, lb = nb - env * P.blocks_per_env;
    const int gx = kBX * (lb % P.bdims[0]) + lane % kBX, gy = kBY * ((lb / P.bdims[0]) % P.bdims[1]) + (lane / kBX) % kBY,
              gz = kBZ * (lb / (P.bdims[0] * P.bdims[1])) + lane / (kBX * kBY);
    const bool inside = gx < P.dims[0] && gy < P.dims[1] && gz < P.dims[2];
    const long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
    float4 pm = inside ? P.gPM[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (P.det && inside) {  // int64 fixed point of this launch (4 channels)
      const longlong4 q = P.gPMd[gi];
      const int sm = P.run[env].det_sm, sp = P.run[env].det_sp;
      pm = make_float4((float)ldexp((double)q.x, -sp), (float)ldexp((double)q.y, -sp), (float)ldexp((double)q.z, -sp),
                       (float)ldexp((double)q.w, -sm));
      if (P.clear_on_read) P.gPMd[gi] = make_longlong4(0, 0, 0, 0);
    }
    const float4 ff = (inside && P.split) ? P.gF[gi] : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool live = inside && pm.w > 0.0f;
    const float dt = P.run[env].dt_c;
    f3 vel = {0.f, 0.f, 0.f};
    f3 f = {ff.x, ff.y, ff.z};
    if (live) vel = (1.0f / pm.w) * f3{pm.x, pm.y, pm.z};  // pre-force node velocity
    if (HOOK) {
      const int s0 = P.shape_off[env], s1 = P.shape_off[env + 1];
      const int b0 = P.body_off[env];
      const f3 xi = {(float)(P.origin[0] + P.h * gx), (float)(P.origin[1] + P.h * gy), (float)(P.origin[2] + P.h * gz)};
      const float scale = P.mean_mass[env] > 0.0 ? (float)(pm.w / P.mean_mass[env]) : 1.0f;
      for (int sidx = s0; sidx < s1; ++sidx) {
        const ShapeDev& sh = P.shapes[sidx];
        f3 fp = {0.f, 0.f, 0.f};
        float pen = 0.0f;
        const bool hit = live && shape_may_touch(sh, xi, P.r_c_grid) &&
                         penalty_force(sh, P.vol_pool, xi, vel, P.r_c_grid, P.c_d, fp, pen);
        if (hit) {
          fp = scale * fp;
          f = f + fp;
        } else {
          fp = {0.f, 0.f, 0.f};
        }
        if (__any_sync(FULL, hit)) {
          const f3 com = {sh.com[0], sh.com[1], sh.com[2]};
          const f3 tq = cross(xi - com, f3{-fp.x, -fp.y, -fp.z});
          double r[6] = {-(double)fp.x, -(double)fp.y, -(double)fp.z, (double)tq.x, (double)tq.y, (double)tq.z};
#pragma unroll
          for (int k = 0; k < 6; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r[k] += __shfl_xor_sync(FULL, r[k], o);
          unsigned pb = hit ? __float_as_uint(pen) : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) pb = max(pb, __shfl_xor_sync(FULL, pb, o));
          if (lane == 0) {
            double* wr = P.wrench + 6 * (b0 + sh.body);
#pragma unroll
            for (int k = 0; k < 6; ++k) atomicAdd(wr + k, r[k]);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              atomicAdd(P.react + 3 * env + k, r[k]);
              atomicAdd(P.applied + 3 * env + k, -r[k]);
            }
            atomicMax(&P.max_pen_bits[env], pb);
          }
        }
      }
    }
    if (!inside) continue;
    if (live) {
      vel = vel + dt * (f3{P.gravity[0], P.gravity[1], P.gravity[2]} + (1.0f / pm.w) * f);
      const int idx[3] = {gx, gy, gz};
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if (idx[ax] < 2) {
          if (!((P.boundary_slip >> (2 * ax)) & 1u)) vel = {0.f, 0.f, 0.f};
          else if (comp(vel, ax) < 0.0f) vel = ax == 0 ? f3{0.f, vel.y, vel.z} : (ax == 1 ? f3{vel.x, 0.f, vel.z} : f3{vel.x, vel.y, 0.f});
        }
        if (idx[ax] >= P.dims[ax] - 2) {
          if (!((P.boundary_slip >> (2 * ax + 1)) & 1u)) vel = {0.f, 0.f, 0.f};
          else if (comp(vel, ax) > 0.0f) vel = ax == 0 ? f3{0.f, vel.y, vel.z} : (ax == 1 ? f3{vel.x, 0.f, vel.z} : f3{vel.x, vel.y, 0.f});
        }
      }
    }
    P.gV[gi] = make_float4(vel.x, vel.y, vel.z, 0.0f);
    if (P.clear_on_read) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      P.gPM[gi] = z;
      if (P.split) P.gF[gi] = z;
    } else if (P.grid_mode && live) {
      P.gF[gi] = make_float4(f.x, f.y, f.z, 0.0f);  // the grid hook adds to grid.force (phase API)
    }
  }
}

template <bool HOOK>
__global__ void __launch_bounds__(256) k_grid(SimParams P) {
  pdl_wait();
  pdl_trigger();
  grid_items<HOOK>(P, (int)(blockIdx.x * blockDim.x + threadIdx.x), (int)(gridDim.x * blockDim.x));
}

// ---------------------------------------------------------------------------
// Per-env bookkeeping.

// ---------------------------------------------------------------------------
// Per-env bookkeeping.

// Deterministic mode: this launch's grid fixed-point exponents of an env: mass
// from the env's total mass (node sums < 2^61), momentum from the largest round
// bound of the previous launch (a contribution of that size ~ 2^kDetMomentumExp).
__device__ void det_exponents(const SimParams& P, int env, EnvRun& r) {
  if (!P.det) return;
  r.det_sm = P.det_mexp[env];
  const float b = __uint_as_float(P.det_bnd[env]);
  r.det_sp = b > 0.f ? kDetMomentumExp - ilogbf(b) : kDetMomentumExp;
  P.det_bnd[env] = 0u;
}

__device__ void plan_cycles(const SimParams& P, int env, EnvRun& r) {  // mpm.hpp:399-409
  const double vmax = (double)__uint_as_float(P.vmax_bits[env]);
  int halvings = 0;
  while (halvings < P.max_halvings && vmax * P.dt_full / (1 << halvings) > P.cfl_h) ++halvings;
  if (vmax * P.dt_full / (1 << halvings) > P.cfl_h) {
    set_error(P, env, kErrCfl, 0x7fffffff);
    r.action = kActIdle;
    r.substeps_left = 0;
    return;
  }
  r.cycles = 1 << halvings;
  r.dt_c = (float)(P.dt_full / r.cycles);
  r.cyc_sum += r.cycles;
}

__global__ void k_set_action(SimParams P, int action, float dt) {
  const int env = blockIdx.x * blockDim.x + threadIdx.x;
  if (env == 0) *P.any_redo = 0;
  if (env >= P.n_env) return;
  EnvRun& r = P.run[env];
  r.action = action;
  r.dt_c = r.dt_g2p = r.dt_p2g = dt;
  r.cycle = 0;
  r.cycles = 1;
  r.substeps_left = 0;
  r.redo = 0;
  if (action == kActG2P) P.vmax_bits[env] = 0u;
}

// One warp per env (lane 0: the env's state machine; all lanes: its rigid step).
// The kernels run kRigidWarps warps per CTA; sbody: the warp's body slots.
constexpr int kRigidWarps = 4;
__device__ void call_begin_env(const SimParams& P, int env, int n_sub, int first_action, int lane, BodyDev* sbody) {
  EnvRun& r = P.run[env];
  const EnvRange g = env_range(P, env);
  int rigid = 0;
  if (lane == 0) {
    r.substeps_left = n_sub;
    r.soft_in_rigid = 0;
    r.cycle = 0;
    r.cyc_sum = 0;
    r.next_new_sub = 0;
    r.next_new_rigid = 0;
    r.redo = 0;
    r.action = n_sub > 0 ? first_action : kActIdle;
    if (P.err_code[env]) {
      r.action = kActIdle;
      r.substeps_left = 0;
    } else {
      r.rigid_idx = 0;
      rigid = n_sub > 0 && P.integrate_rigid;
    }
  }
  rigid = __shfl_sync(0xffffffffu, rigid, 0);
  if (rigid) rigid_env(P, env, 1, lane, 32, g, 0, false, sbody);  // rigid step 0: integrate + sync
  __syncwarp();
  if (lane == 0 && !P.err_code[env]) {
    if (n_sub > 0) plan_cycles(P, env, r);
    det_exponents(P, env, r);
    r.dt_g2p = 0.0f;
    r.dt_p2g = r.dt_c;  // the first P2G knows its dt exactly
    P.vmax_bits[env] = 0u;
  }
}

__global__ void __launch_bounds__(32 * kRigidWarps) k_call_begin(SimParams P, int n_sub, int first_action) {
  pdl_wait();
  pdl_trigger();
  __shared__ BodyDev sbody[kRigidWarps][kMaxBodiesPerEnv];
  const int t = blockIdx.x * blockDim.x + threadIdx.x, env = t >> 5;
  if (t == 0) *P.any_redo = 0;
  if (env < P.n_env) call_begin_env(P, env, n_sub, first_action, t & 31, sbody[threadIdx.x >> 5]);
}

// One warp per env (lane 0: the env's state machine; all lanes: its rigid step).
__device__ void iter_begin_env(const SimParams& P, int env, int lane, BodyDev* sbody) {
  EnvRun& r = P.run[env];
  const EnvRange g = env_range(P, env);  // all lanes, in the same batch as lane 0's state
  int rigid = 0, active = 0, ridx = 0;
  if (lane == 0) {  // the env's state in registers (one batch of loads), changed fields written back
    const EnvRun l = r;
    const int err = P.err_code[env];
    int action = kActIdle, nns = 0, nnr = 0;
    if (l.substeps_left > 0 && !err) {
      active = 1;
      r.dt_g2p = l.dt_c;
      r.dt_p2g = l.dt_c;  // same substep: exact; new substep: speculated (same cycle count)
      if (l.cycle == l.cycles - 1 && l.substeps_left == 1) {
        action = kActG2P;
      } else {
        action = kActFused;
        if (l.cycle + 1 >= l.cycles) {
          nns = 1;
          nnr = P.integrate_rigid && (l.soft_in_rigid + 1 == P.n_soft);
        }
        if (nnr) {
          ridx = l.rigid_idx + 1;
          r.rigid_idx = ridx;
          rigid = 1;
        }
      }
    }
    r.action = action;
    r.next_new_sub = nns;
    r.next_new_rigid = nnr;
    r.redo = 0;
  }
  rigid = __shfl_sync(0xffffffffu, rigid, 0);
  active = __shfl_sync(0xffffffffu, active, 0);
  ridx = __shfl_sync(0xffffffffu, ridx, 0);
  // end of rigid step: pending_wrenches = wrenches (coupling.hpp:288, staged by
  // the body lanes), then the next rigid step integrates with them and syncs
  // (coupling.hpp:250-259)
  if (rigid) rigid_env(P, env, 1, lane, 32, g, ridx, true, sbody);
  if (lane == 0 && active) {
    det_exponents(P, env, r);
    P.vmax_bits[env] = 0u;
  }
}
// Scheduled (programmatic launch) once k_grid has started, i.e. after k_iter_end
// and the particle kernel completed. In particle coupling mode outside the
// deterministic mode k_grid reads nothing this kernel writes (only the envs'
// dt_c and the grid), so the rigid step runs alongside k_grid and waits for it
// only before exiting; otherwise (grid-mode penalty reads the shapes, the
// deterministic grid reads the launch exponents) it waits first.
__global__ void __launch_bounds__(32 * kRigidWarps) k_iter_begin(SimParams P) {
  const bool early = !P.grid_mode && !P.det;
  if (!early) pdl_wait();
  pdl_trigger();
  __shared__ BodyDev sbody[kRigidWarps][kMaxBodiesPerEnv];
  const int t = blockIdx.x * blockDim.x + threadIdx.x, env = t >> 5;
  if (t == 0) *P.any_redo = 0;
  if (env < P.n_env) iter_begin_env(P, env, t & 31, sbody[threadIdx.x >> 5]);
  if (early) pdl_wait();
}

__device__ void iter_end_env(const SimParams& P, int env) {
  EnvRun& r = P.run[env];
  if (r.action == kActIdle) return;
  if (P.det) {  // integer sums of this cycle -> the double accumulators (exact up to 2^-36)
    const int b0 = P.body_off[env], b1 = P.body_off[env + 1];
    for (int k = 6 * b0; k < 6 * b1; ++k) P.wrench[k] = ldexp((double)P.w64[k], -kDetWrenchExp);
    for (int k = 0; k < 3; ++k) {
      P.applied[3 * env + k] = ldexp((double)P.a64[3 * env + k], -kDetWrenchExp);
      P.react[3 * env + k] = ldexp((double)P.r64[3 * env + k], -kDetWrenchExp);
      P.a64[3 * env + k] = P.r64[3 * env + k] = 0;
    }
  }
  double ex = P.applied[3 * env] + P.react[3 * env];
  double ey = P.applied[3 * env + 1] + P.react[3 * env + 1];
  double ez = P.applied[3 * env + 2] + P.react[3 * env + 2];
  const double err = sqrt(ex * ex + ey * ey + ez * ez);
  if (err > P.balance_max[env]) P.balance_max[env] = err;
  for (int k = 0; k < 3; ++k) P.applied[3 * env + k] = P.react[3 * env + k] = 0.0;
  const long long n_env_p = P.env_off[env + 1] - P.env_off[env];
  if (n_env_p > 0 && (double)P.lost_count[env] / (double)n_env_p > P.lost_threshold)
    set_error(P, env, kErrLost, 0x7fffffff);
  if (r.action == kActFused) {
    if (r.next_new_sub) {
      r.substeps_left -= 1;
      r.soft_in_rigid = (r.soft_in_rigid + 1) % P.n_soft;
      r.cycle = 0;
      plan_cycles(P, env, r);
      // the fused P2G folded dt_p2g into the momentum; a different plan needs a redo
      if (!P.split && r.substeps_left > 0 && !P.err_code[env] && r.dt_c != r.dt_p2g) {
        r.redo = 1;
        atomicExch(P.any_redo, 1);
      }
    } else {
      r.cycle += 1;
    }
  } else if (r.action == kActG2P) {
    r.substeps_left = 0;
    if (P.integrate_rigid) {
      const int b0 = P.body_off[env], b1 = P.body_off[env + 1];
      for (int k = 6 * b0; k < 6 * b1; ++k) P.pending[k] = P.wrench[k];
    }
  }
  if (P.err_code[env]) r.substeps_left = 0;
}
// One CTA per env: thread 0 runs the env's state machine; when the speculated
// dt of the fused P2G missed (redo), the CTA zeroes the env's P2G accumulators
// right away (its node blocks: a contiguous range of the ascending node-block
// list) for the redo pass.
constexpr int kIterEndThreads = 128;
// Scheduled (programmatic launch) once the node-block scan has started, i.e.
// after the particle kernel completed: the state machine only reads the
// particle kernel's outputs and runs alongside the bucket / node-block scans;
// the redo clear reads the node-block list and waits first.
__global__ void __launch_bounds__(kIterEndThreads) k_iter_end(SimParams P) {
  pdl_trigger();
  const int env = blockIdx.x, lane = threadIdx.x;
  __shared__ int redo;
  if (lane == 0) {
    iter_end_env(P, env);
    redo = P.run[env].redo;
  }
  __syncthreads();
  pdl_wait();
  if (!redo) return;
  const int nlist = *P.n_nb;
  auto lower = [&](int key) {  // first list entry >= key
    int lo = 0, hi = nlist;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (P.nb_list[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const int a = lower(env * P.blocks_per_env), b = lower((env + 1) * P.blocks_per_env);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int NB = kBX * kBY * kBZ;
  for (long long q = (long long)a * NB + lane; q < (long long)b * NB; q += kIterEndThreads) {
    const int nb = P.nb_list[q / NB], l = (int)(q % NB);
    const int lb = nb - env * P.blocks_per_env;
    const int gx = kBX * (lb % P.bdims[0]) + l % kBX, gy = kBY * ((lb / P.bdims[0]) % P.bdims[1]) + (l / kBX) % kBY,
              gz = kBZ * (lb / (P.bdims[0] * P.bdims[1])) + l / (kBX * kBY);
    if (gx >= P.dims[0] || gy >= P.dims[1] || gz >= P.dims[2]) continue;
    const long long gi = env * P.nodes_per_env + ((long long)gz * P.dims[1] + gy) * P.dims[0] + gx;
    P.gPM[gi] = z;
    if (P.det) P.gPMd[gi] = make_longlong4(0, 0, 0, 0);
  }
}

inline unsigned nblk(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct Timed {
  KernelTimer* t;
  int id;
  cudaStream_t s;
  cudaEvent_t a;
  Timed(const SimParams& P, int id_, cudaStream_t s_, int nlaunch = 1) : t(P.timer), id(id_), s(s_), a(nullptr) {
    if (t) a = t->begin(s, nlaunch);
  }
  ~Timed() {
    if (t) t->end(id, a, s);
  }
};

// persistent grid: as many CTAs as fit on the device at once (occupancy query)
template <int NCH, int F, bool AM, bool DET = false, bool LAT = false>
void launch_k_particles(const SimParams& P, cudaStream_t s) {
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_particles<NCH, F, AM, DET, LAT>, kT,
                                                  sizeof(Smem<NCH, F>));
    if (per_sm <= 0) per_sm = 1;
  }
  // the redo pass (speculated dt missed: rare) exits at once when no env redoes;
  // for small scenes one CTA per SM keeps that no-op launch cheap on the
  // per-cycle critical path (A -1 %)
  const int g = P.redo_pass && P.split_r > 1 ? sm_count() : sm_count() * per_sm;
  launch_pdl(k_particles<NCH, F, AM, DET, LAT>, g, kT, sizeof(Smem<NCH, F>), s, P);
}

template <bool AM>
void particle_kernel_m(const SimParams& P, cudaStream_t s) {
  if (P.det) {  // deterministic mode: 4 channels only (msim_gpu_set_deterministic)
    if (P.qf == 2) launch_k_particles<4, 2, AM, true>(P, s);
    else launch_k_particles<4, 1, AM, true>(P, s);
    return;
  }
  if (P.qf == 2) {
    if (P.split) launch_k_particles<7, 2, AM>(P, s);
    else launch_k_particles<4, 2, AM>(P, s);
  } else {
    if (P.split) launch_k_particles<7, 1, AM>(P, s);
    else if (P.split_r > 1) launch_k_particles<4, 1, AM, false, true>(P, s);
    else launch_k_particles<4, 1, AM>(P, s);
  }
}

void particle_kernel(const SimParams& P, cudaStream_t s) {
  if (P.any_model) particle_kernel_m<true>(P, s);
  else particle_kernel_m<false>(P, s);
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MSIM_NO_PDL");
    return !(e && *e && *e != '0');
  }();
  return on;
}

void configure_kernels() {
#define MSIM_SET_SMEM(NCH, F, AM, DET, ...)                                                                      \
  cudaFuncSetAttribute(k_particles<NCH, F, AM, DET, ##__VA_ARGS__>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)sizeof(Smem<NCH, F>))
  MSIM_SET_SMEM(4, 1, false, false); MSIM_SET_SMEM(7, 1, false, false); MSIM_SET_SMEM(4, 2, false, false);
  MSIM_SET_SMEM(7, 2, false, false); MSIM_SET_SMEM(4, 1, true, false); MSIM_SET_SMEM(7, 1, true, false);
  MSIM_SET_SMEM(4, 2, true, false); MSIM_SET_SMEM(7, 2, true, false);
  MSIM_SET_SMEM(4, 1, false, true); MSIM_SET_SMEM(4, 2, false, true); MSIM_SET_SMEM(4, 1, true, true);
  MSIM_SET_SMEM(4, 2, true, true); MSIM_SET_SMEM(4, 1, false, false, true); MSIM_SET_SMEM(4, 1, true, false, true);
#undef MSIM_SET_SMEM
}

void launch_rebin(const SimParams& P, cudaStream_t s) {
  {
    Timed tm(P, kKBin, s);
    if (P.n > 0) launch_pdl(k_rebin, nblk(P.n), 256, 0, s, P);
  }
  // keys of the stored positions describe the NEXT particle launch: write the read set
  SimParams Q = P;
  Q.perm_w = P.perm;
  Q.bucket_start_w = P.bucket_start;
  Q.active_buckets_w = P.active_buckets;
  Q.n_active_buckets_w = P.n_active_buckets;
  Timed tm(P, kKBucketScan, s, P.det ? 3 : 2);
  scan_exclusive(Q.bucket_count, Q.bucket_start_w, Q.n_keys, Q.active_buckets_w, Q.n_active_buckets_w, Q.scan_tmp, s);
  if (Q.n > 0) launch_pdl(k_perm<false>, nblk((Q.n + 3) / 4), 256, 0, s, Q);
  if (Q.det) launch_pdl(k_det_sort_movers, sm_count() * 8, 128, 0, s, Q);
}

void launch_clear(const SimParams& P, cudaStream_t s) {
  Timed tm(P, kKClear, s);
  k_clear<<<sm_count() * 4, 256, 0, s>>>(P);
}

void launch_set_action(const SimParams& P, int action, float dt, cudaStream_t s) {
  k_set_action<<<nblk(P.n_env), 256, 0, s>>>(P, action, dt);
}

void launch_call_begin(const SimParams& P, int n_sub, int first_action, cudaStream_t s) {
  Timed tm(P, kKPlan, s);
  launch_pdl(k_call_begin, nblk(32LL * P.n_env, 32 * kRigidWarps), 32 * kRigidWarps, 0, s, P, n_sub, first_action);
}

void launch_perm(const SimParams& P, cudaStream_t s, bool early) {
  Timed tm(P, kKBucketScan, s, P.det ? 2 : 1);
  if (P.n > 0) launch_pdl(early ? k_perm<true> : k_perm<false>, nblk((P.n + 3) / 4), 256, 0, s, P);
  if (P.det) launch_pdl(k_det_sort_movers, sm_count() * 8, 128, 0, s, P);
}

void launch_particles(const SimParams& P, cudaStream_t s, bool perm_now) {
  {
    Timed tm(P, kKP2G, s);
    SimParams Q = P;
    Q.redo_pass = 0;
    particle_kernel(Q, s);
  }
  // the next launch's bucket structure goes to the write set: the redo pass of this
  // launch still reads this launch's perm / bucket offsets
  {
    Timed tm(P, kKBucketScan, s, 1);
    scan_exclusive(P.bucket_count, P.bucket_start_w, P.n_keys, P.active_buckets_w, P.n_active_buckets_w, P.scan_tmp, s);
  }
  {  // node-block list: its flags are complete with the particle kernel, so it runs
     // alongside the bucket scan (own status area)
    Timed tm(P, kKBlockScan, s, 1);
    scan_exclusive(P.nb_flag, P.nb_scan, P.n_blocks, P.nb_list, P.n_nb, P.scan_tmp2, s, true);
  }
  if (perm_now) launch_perm(P, s, false);
}

void launch_grid(const SimParams& P, cudaStream_t s) {
  Timed tm(P, kKGrid, s);
  launch_pdl(P.grid_mode && P.hooks ? k_grid<true> : k_grid<false>, sm_count() * 8, 256, 0, s, P);
}

void launch_iteration_end(const SimParams& P, cudaStream_t s) {
  Timed tm(P, kKEnd, s);
  launch_pdl(k_iter_end, P.n_env, kIterEndThreads, 0, s, P);
}

void launch_iteration(const SimParams& P, bool bookkeeping, bool grid_update, cudaStream_t s) {
  if (bookkeeping) {
    Timed tm(P, kKRigid, s);
    launch_pdl(k_iter_begin, nblk(32LL * P.n_env, 32 * kRigidWarps), 32 * kRigidWarps, 0, s, P);
  }
  // the slot map of the next launch is only needed by that launch: it goes after
  // k_grid (and runs alongside it) when there is one
  launch_particles(P, s, !grid_update);
  launch_iteration_end(P, s);  // also zeroes the accumulators of envs that redo
  if (bookkeeping && !P.split) {
    // speculated-dt misses (CFL halving changed between substeps): redo those envs' P2G.
    // Exits immediately when no env needs it.
    Timed tm(P, kKRedo, s, 1);
    SimParams Q = P;
    Q.redo_pass = 1;
    particle_kernel(Q, s);
  }
  if (grid_update) {
    launch_grid(P, s);
    launch_perm(P, s, true);
  }
}

}  // namespace msim_impl
