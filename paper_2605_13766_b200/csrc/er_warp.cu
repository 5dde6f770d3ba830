// er_warp.cu -- the warp-local step kernel for batches of equal-length short rods
// (ER_WARP_MIN_N..32 elements; BASELINE configs[2]'s 1024^2 filaments of 16 elements), sm_100a, fp64.
// No tensor cores: nothing here is a dense contraction.
//
// Mapping: lane = element.  A rod of N elements sits on N consecutive lanes of one warp (wR =
// floor(32/N) rods per warp; rods never straddle warps).  Lane i holds node i (r, v), element i
// (d1, d2 -> Q, w) and Voronoi domain i (i >= 1); the rod's last lane also holds node N.  Every
// neighbour value the step needs (node i+1, element i-1, n_{i-1}, mbar_{i+1},
// beta_{i+1}) is one warp shuffle away, so a step has no shared-memory exchange and no CTA barrier
// (the tile kernel of er_kernels.cu needs three per step, because its rods straddle warps).
//
// Pipeline: persistent CTAs of 8 warps walk the tiles (8 wR rods each, the standard tile block of
// er_layout.h).  A tile streams into one of wnb shared-memory stage buffers by TMA bulk copies that
// complete an mbarrier.  Each warp waits for its tile's data, advances its rods n_steps steps in
// registers and writes its results back in place (no other warp reads them); the last warp to finish
// a tile (an acq_rel counter per buffer) bulk-stores the block to HBM, waits until the store has read
// the buffer and refills it with the tile wnb positions ahead.  Warps drift up to wnb - 1 tiles
// apart: nobody waits for anybody except for data.
//
// The physics is step_body's of er_kernels.cu line for line (same operation order, same helpers), so
// both kernels give bitwise the same trajectory (tests/test_gpu_warp.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "er_layout.h"
#include "er_math.cuh"
#include "er_tma.cuh"

namespace er {

// Per-lane role bits (registers are the scarce resource of this kernel: a struct of bools and the
// node-N state in registers pushed it into local memory; node N lives in the stage buffer instead).
enum : unsigned {
  WL_ACTIVE = 1,    // the lane holds element i of a rod
  WL_HAS_V = 2,     // Voronoi domain i exists (i >= 1)
  WL_LAST = 4,      // i == N - 1: the lane also advances node N (its r, v stay in the stage buffer)
  WL_CL_NODE = 8,   // node i clamped
  WL_CL_NODEN = 16, // node N clamped
  WL_CL_ELEM = 32,  // element i clamped
  WL_TIP_I = 64,    // the tip force acts on node i
  WL_TIP_N = 128,   // the tip force acts on node N
};
struct WLane {
  int i, N;        // element index in the rod, rod length
  int fl;          // rod flag word
  unsigned lb;     // WL_* bits
  int64_t node;    // packed node index of node i (node N = node + 1)
  int64_t elem;    // packed element index of element i
  int rod;         // packed rod id
};

constexpr unsigned kFull = 0xffffffffu;

// One position-Verlet step of one lane; see step_body in er_kernels.cu.
// One position-Verlet step of one lane: step_body of er_kernels.cu with
// warp-shuffle exchanges.
// Node N of a rod (its last lane's second node): r, v either in the stage buffer (XSmem, plane stride
// ns) or in registers (XReg).
struct XSmem {
  double *x;
  int ns;
  __device__ __forceinline__ double r(int c) const { return x[c * ns]; }
  __device__ __forceinline__ double v(int c) const { return x[(3 + c) * ns]; }
  __device__ __forceinline__ void set_r(int c, double a) { x[c * ns] = a; }
  __device__ __forceinline__ void set_v(int c, double a) { x[(3 + c) * ns] = a; }
};
struct XReg {
  double rr[3], vv[3];
  __device__ __forceinline__ double r(int c) const { return rr[c]; }
  __device__ __forceinline__ double v(int c) const { return vv[c]; }
  __device__ __forceinline__ void set_r(int c, double a) { rr[c] = a; }
  __device__ __forceinline__ void set_v(int c, double a) { vv[c] = a; }
};

// Neighbour exchange across a warp boundary.  NoCross: every rod lies in one warp.  PairCross: a rod
// of 33..64 elements lies on two warps of a pair; element 31 (warp 0, lane 31) and element 32 (warp 1,
// lane 0) swap their neighbour values through a mailbox in shared memory, one named barrier of the
// pair's 64 threads per exchange (the three mailboxes are separate, so a mailbox is rewritten only
// after both warps have passed the two later barriers of the step).
struct NoCross {
  __device__ __forceinline__ void a(const double *, const double *, const double *, double *, double *, double *) const {}
  __device__ __forceinline__ void b(double, const double *, double &, double *) const {}
  __device__ __forceinline__ void c(const double *, const double *, double *, double *) const {}
};
__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
struct PairCross {
  double *mb;  // this pair's mailboxes: [0..5] r, v of element 32's node; [6..11] d1, d2 of element 31;
               // [12..15] l, n of edge 31; [16..21] mbar, beta of Voronoi 32
  int id;      // named barrier of the pair (1..4)
  bool lo, hi; // this lane is warp 0 / lane 31, warp 1 / lane 0
  __device__ __forceinline__ void a(const double *r, const double *v, const double *Q, double *rn, double *vn,
                                    double *Qp) const {
    if (hi) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { mb[c] = r[c]; mb[3 + c] = v[c]; }
    }
    if (lo) {
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) mb[6 + c] = Q[c];
    }
    pair_sync(id);
    if (lo) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { rn[c] = mb[c]; vn[c] = mb[3 + c]; }
    }
    if (hi) {
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) Qp[c] = mb[6 + c];
    }
  }
  __device__ __forceinline__ void b(double l, const double *n, double &lp, double *np) const {
    if (lo) {
      mb[12] = l;
#pragma unroll
      for (int c = 0; c < 3; ++c) mb[13 + c] = n[c];
    }
    pair_sync(id);
    if (hi) {
      lp = mb[12];
#pragma unroll
      for (int c = 0; c < 3; ++c) np[c] = mb[13 + c];
    }
  }
  __device__ __forceinline__ void c(const double *m, const double *be, double *mbn, double *ben) const {
    if (hi) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { mb[16 + c] = m[c]; mb[19 + c] = be[c]; }
    }
    pair_sync(id);
    if (lo) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { mbn[c] = mb[16 + c]; ben[c] = mb[19 + c]; }
    }
  }
};

// Rod-record access.  RecFull: the rod's ER_REC-double record, staged in the slot.  RecUni
// (FEAT_UNI, a shared-material batch): the 17 shared constants from the kernel parameters (constant
// bank operands), tip force / actuation / flags from the rod's ER_WREC-double record in the slot.
// Both hand wstep the same values, so the trajectory is bitwise the same.
struct RecFull {
  const double *r;
  __device__ __forceinline__ double operator[](int k) const { return r[k]; }
  __device__ __forceinline__ int flags() const { return rec_flags(r); }
  __device__ __forceinline__ int canon() const { return (int)r[REC_CANON]; }
};
struct RecUni {
  const double *r;
  const ErStepParams &p;
  __device__ __forceinline__ double operator[](int k) const {
    return (k >= REC_TIPX && k <= REC_ACTF) ? r[WREC_TIPX + (k - REC_TIPX)] : k == REC_ACTIL ? p.umat[16] : p.umat[k];
  }
  __device__ __forceinline__ int flags() const { return (int)(__double_as_longlong(r[WREC_FC]) & 0xffffffffll); }
  __device__ __forceinline__ int canon() const { return (int)(__double_as_longlong(r[WREC_FC]) >> 32); }
};

template <int FEAT, class XN, class CR = NoCross, class RC = RecFull>
__device__ __forceinline__ void wstep(const ErStepParams &p, const RC &rec, const WLane &L,
                                      double r[3], double v[3], XN &xN, double Q[9], double w[3],
                                      const double k0s[3], double &t, unsigned &fbits, const CR &cr = CR(),
                                      bool final_step = false) {
  constexpr bool GEN = (FEAT & FEAT_GENERAL) != 0;
  constexpr bool EXTRA = (FEAT & FEAT_EXTRA) != 0;
  constexpr bool ACT = (FEAT & (FEAT_EXTRA | FEAT_ACT)) != 0;
  const int i = L.i;
  const double h = p.h, hh = 0.5 * p.h;
  const bool general = GEN && (L.fl & FL_GENERAL);
  const bool active = L.lb & WL_ACTIVE, last = L.lb & WL_LAST, has_v = L.lb & WL_HAS_V;
  const double t_half = t + hh;
  auto gp = [&](int plane, int64_t node) { return __ldg(p.gpar + plane * p.ng + node); };

  // ---- A1-A3 drift-1.  A clamped node / element moves by a zero step (r + 0 v = r; rot(0) Q = Q
  // exactly), so the warp takes no branch for the rods' clamped ends.
  const double hr = (L.lb & WL_CL_NODE) ? 0.0 : hh, hq = (L.lb & WL_CL_ELEM) ? 0.0 : hh;
  if (active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = fma(hr, v[c], r[c]);
    rotate_inplace(Q, hq * w[0], hq * w[1], hq * w[2]);
  }
  // ---- exchange A: node i+1 from the next lane (the rod's last lane owns node N), element i-1
  double rn[3], vn[3], Qp[9];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    rn[c] = __shfl_down_sync(kFull, r[c], 1);
    vn[c] = __shfl_down_sync(kFull, v[c], 1);
  }
#pragma unroll
  for (int c = 0; c < ER_QST; ++c) {  // a rod's first lane pairs its element with itself (kappa = 0)
    const double q = __shfl_up_sync(kFull, Q[c], 1);
    Qp[c] = has_v ? q : Q[c];
  }
  cr.a(r, v, Q, rn, vn, Qp);
  if (last) {  // node N: drift-1 (one divergent block with its use as node i+1)
    const double hN = (L.lb & WL_CL_NODEN) ? 0.0 : hh;  // (a clamped node moves by a zero step: r + 0 v = r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vn[c] = xN.v(c);
      rn[c] = fma(hN, vn[c], xN.r(c));
      xN.set_r(c, rn[c]);
    }
  }
  // ---- A4-A5 edge i: kinematics, shear/stretch strain, stress
  double Ql[3] = {0.0, 0.0, 0.0}, nb[3] = {0.0, 0.0, 0.0}, n[3] = {0.0, 0.0, 0.0};
  double l = 0.0, inv_e = 0.0, e = 1.0, edot = 0.0;
  const double lh = general ? gp(GP_LHAT, L.node) : rec[REC_LHAT];
  if (active) {
    const double ilh = general ? gp(GP_ILHAT, L.node) : rec[REC_ILHAT];
    double ell[3], dv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ell[c] = rn[c] - r[c];
      dv[c] = vn[c] - v[c];
    }
    const double l2 = dot3(ell, ell);
    const double il = rsqrt_fast(l2);
    l = l2 * il;
    e = l * ilh;
    inv_e = lh * il;
    edot = dot3(ell, dv) * il * ilh;
    if (!(e >= 1e-12)) fbits |= 2u;  // ER_F_DEGENERATE
    Ql[0] = dot3(Q, ell);
    Ql[1] = dot3(Q + 3, ell);
    Ql[2] = dot3(Q + 6, ell);
    double sg[3] = {Ql[0] * ilh, Ql[1] * ilh, fma(Ql[2], ilh, -1.0)};  // sigma = Q l/lhat - e3
    if (EXTRA && p.sigma0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) sg[c] -= __ldg(p.sigma0 + c * p.ne + L.elem);
    }
    const double S1 = general ? gp(GP_S1, L.node) : rec[REC_S1];
    const double S3 = general ? gp(GP_S3, L.node) : rec[REC_S3];
    nb[0] = S1 * sg[0] * inv_e;
    nb[1] = S1 * sg[1] * inv_e;
    nb[2] = S3 * sg[2] * inv_e;
#pragma unroll
    for (int c = 0; c < 3; ++c) n[c] = fma(Q[c], nb[0], fma(Q[3 + c], nb[1], Q[6 + c] * nb[2]));  // Q^T nbar
  }
  // ---- A6 Voronoi i: curvature via inverse Rodrigues
  // (no branch: a rod's first lane computes kappa = 0 from its own frame and masks the moment below,
  // so the curvature can be scheduled beside the edge block)
  double kap[3];
  {
    double cth, s2;
    complete_d3(Qp);  // the bits the neighbour holds in its registers
    logrot_pair(Q, Qp, kap, cth, s2);
    if (has_v && cth < 0.0 && s2 <= 1e-12 * cth * cth) fbits |= 4u;  // ER_F_ANTIPODAL: theta >= pi - 1e-6
  }
  // ---- exchange B: l_{i-1}, n_{i-1}
  double lp = __shfl_up_sync(kFull, l, 1);
  double np[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) np[c] = __shfl_up_sync(kFull, n[c], 1);
  cr.b(l, n, lp, np);

  // ---- A6 bending moment and its averaged cross term
  double mb[3] = {0.0, 0.0, 0.0}, be[3] = {0.0, 0.0, 0.0};
  {
    const double Dh = general ? gp(GP_DH, L.node) : rec[REC_LHAT];
    const double iDh = general ? 1.0 / Dh : rec[REC_ILHAT];
#pragma unroll
    for (int c = 0; c < 3; ++c) kap[c] *= iDh;
    const double D = 0.5 * (lp + l);
    const double ieps = Dh * rcp_fast(D);
    const double ieps3 = ieps * ieps * ieps;
    double k0[3] = {k0s[0], k0s[1], k0s[2]};
    if (ACT && (L.fl & FL_ACT)) {
      const double sk = general ? gp(GP_SK, L.node) : i * rec[REC_LHAT];
      const double arg = 2.0 * fma(sk, rec[REC_ACTIL], -rec[REC_ACTF] * t_half);
      const double act = rec[REC_ACTA] * sinpi(arg);
      k0[0] += p.act_comp == 0 ? act : 0.0;
      k0[1] += p.act_comp == 1 ? act : 0.0;
      k0[2] += p.act_comp == 2 ? act : 0.0;
    }
    const double B1 = general ? gp(GP_BV1, L.node) : rec[REC_B1];
    const double B2 = general ? gp(GP_BV2, L.node) : rec[REC_B2];
    const double B3 = general ? gp(GP_BV3, L.node) : rec[REC_B3];
    mb[0] = B1 * (kap[0] - k0[0]) * ieps3;
    mb[1] = B2 * (kap[1] - k0[1]) * ieps3;
    mb[2] = B3 * (kap[2] - k0[2]) * ieps3;
    be[0] = (kap[1] * mb[2] - kap[2] * mb[1]) * Dh;
    be[1] = (kap[2] * mb[0] - kap[0] * mb[2]) * Dh;
    be[2] = (kap[0] * mb[1] - kap[1] * mb[0]) * Dh;
    if (EXTRA && (L.fl & FL_MUS)) {  // muscular couple pair folded into the exchanged moment
      const double *mu = p.musc + 4 * (int64_t)L.rod;
      const double sk = general ? gp(GP_SK, L.node) : i * rec[REC_LHAT];
      const double tau = __ldg(mu) * sinpi(fma(2.0, fma(t_half, __ldg(mu + 1), -sk * __ldg(mu + 2)), __ldg(mu + 3)));
      mb[0] -= p.musc_comp == 0 ? tau : 0.0;
      mb[1] -= p.musc_comp == 1 ? tau : 0.0;
      mb[2] -= p.musc_comp == 2 ? tau : 0.0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // no Voronoi domain on a rod's first lane
      mb[c] = has_v ? mb[c] : 0.0;
      be[c] = has_v ? be[c] : 0.0;
    }
  }
  // ---- A7 + A9 node force, linear acceleration, kick: node i, and node N on the rod's last lane
  const double nu = rec[REC_NU];
  if (active) {
    double F[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) F[c] = n[c] - (i >= 1 ? np[c] : 0.0);
    if (L.lb & WL_TIP_I) {
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] += rec[REC_TIPX + c];
    }
    if (EXTRA && p.fext) {
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] += __ldg(p.fext + c * p.ng + L.node);
    }
    const double im = general ? gp(GP_IM, L.node) : rec[REC_IM] * (i == 0 ? 2.0 : 1.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double a = fma(F[c], im, fma(-nu, v[c], p.g[c]));
      v[c] = (L.lb & WL_CL_NODE) ? 0.0 : fma(h, a, v[c]);
    }
  }
  // ---- exchange C: mbar_{i+1}, beta_{i+1} (zero past the rod's last Voronoi domain)
  double mbn[3], ben[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    mbn[c] = __shfl_down_sync(kFull, mb[c], 1);
    ben[c] = __shfl_down_sync(kFull, be[c], 1);
  }
  cr.c(mb, be, mbn, ben);
  if (last) {
#pragma unroll
    for (int c = 0; c < 3; ++c) { mbn[c] = 0.0; ben[c] = 0.0; }
  }
  // ---- A8 + A9 element couple, angular acceleration, kick
  if (active) {
    double C[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) C[c] = (mbn[c] - mb[c]) + 0.5 * (ben[c] + be[c]);
    C[0] += Ql[1] * nb[2] - Ql[2] * nb[1];  // shear torque lhat (Q t) x S(sigma - sigma0) == (Q l) x nbar
    C[1] += Ql[2] * nb[0] - Ql[0] * nb[2];
    C[2] += Ql[0] * nb[1] - Ql[1] * nb[0];
    if (EXTRA && p.mag) {  // c_mag = lhat m x (Q b(t))
      double sn, cs;
      sincos(p.b_omega * t_half, &sn, &cs);
      const double b[3] = {fma(cs, p.b0[0], fma(sn, p.b1[0], p.b2[0])), fma(cs, p.b0[1], fma(sn, p.b1[1], p.b2[1])),
                           fma(cs, p.b0[2], fma(sn, p.b1[2], p.b2[2]))};
      const double Qb[3] = {dot3(Q, b), dot3(Q + 3, b), dot3(Q + 6, b)};
      double m[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) m[c] = __ldg(p.mag + c * p.ne + L.elem);
      C[0] += lh * (m[1] * Qb[2] - m[2] * Qb[1]);
      C[1] += lh * (m[2] * Qb[0] - m[0] * Qb[2]);
      C[2] += lh * (m[0] * Qb[1] - m[1] * Qb[0]);
    }
    if (EXTRA && p.cext) {
#pragma unroll
      for (int c = 0; c < 3; ++c) C[c] += __ldg(p.cext + c * p.ne + L.elem);
    }
    const double rate = edot * inv_e - nu;
    const double eu[3] = {w[1] * w[2], w[2] * w[0], w[0] * w[1]};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double iJ = general ? gp(GP_IJ1 + c, L.node) : rec[REC_IJ1 + c];
      const double kJ = general ? gp(GP_KJ1 + c, L.node) : rec[REC_KJ1 + c];
      const double al = fma(e * iJ, C[c], fma(kJ, eu[c], rate * w[c]));
      w[c] = (L.lb & WL_CL_ELEM) ? 0.0 : fma(h, al, w[c]);
    }
  }
  // ---- A10 drift-2
  t = t_half + hh;
  if (active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = fma(hr, v[c], r[c]);
    rotate_inplace(Q, hq * w[0], hq * w[1], hq * w[2], !final_step);  // (d3 of the last step is not stored)
  }
  // fault checks: non-finite state, overspeed (as step_body)
  if (active) {
    const double acc = ((r[0] + r[1]) + (r[2] + v[0])) + ((v[1] + v[2]) + (w[0] + (w[1] + w[2])));
    if (!isfinite(acc)) fbits |= 1u;
    if (dot3(v, v) > rec[REC_VMAX2]) fbits |= 8u;
  }
  if (last) {  // node N: force, kick (A7, A9), drift-2 and its fault checks in one divergent block
    double F[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) F[c] = 0.0 - n[c];  // n_N = 0 (zero-padded difference operator)
    if (L.lb & WL_TIP_N) {
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] += rec[REC_TIPX + c];
    }
    if (EXTRA && p.fext) {
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] += __ldg(p.fext + c * p.ng + L.node + 1);
    }
    const double im = general ? gp(GP_IM, L.node + 1) : rec[REC_IM] * 2.0;
    const bool cl = (L.lb & WL_CL_NODEN) != 0;
    double rN[3], vN[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double vc = xN.v(c);
      const double a = fma(F[c], im, fma(-nu, vc, p.g[c]));
      vN[c] = cl ? 0.0 : fma(h, a, vc);
      rN[c] = fma(cl ? 0.0 : hh, vN[c], xN.r(c));
      xN.set_v(c, vN[c]);
      xN.set_r(c, rN[c]);
    }
    const double acc = ((rN[0] + rN[1]) + (rN[2] + vN[0])) + (vN[1] + vN[2]);
    if (!isfinite(acc)) fbits |= 1u;
    if (dot3(vN, vN) > rec[REC_VMAX2]) fbits |= 8u;
  }
}

struct WHead {
  int64_t boff;
  int32_t r0, nr, nslots, nel, nvor;
};
__device__ __forceinline__ WHead wload_head(const ErTile *t) {
  WHead h;
  h.boff = __ldg(&t->boff);
  const int4 v = __ldg(reinterpret_cast<const int4 *>(&t->r0));
  h.r0 = v.x; h.nr = v.y; h.nslots = v.z; h.nel = v.w;
  h.nvor = h.nel - h.nr;
  return h;
}

// The tile's state block, its rod records and its descriptor into stage buffer B: three TMA bulk
// copies completing on `bar`.
__device__ __forceinline__ void issue_wtile(const ErStepParams &p, const WHead &T, const ErTile *tile_ptr, double *B,
                                            uint64_t *bar, bool kappa0) {
  const int64_t sz = 6 * (int64_t)T.nslots + ER_EPL * (int64_t)T.nel + (kappa0 ? 3 * (int64_t)T.nvor : 0);
  const uint32_t cs = (uint32_t)((sz + 1) & ~1ll);
  const uint32_t bytes = 8u * cs + (uint32_t)T.nr * ER_REC * 8u + (uint32_t)sizeof(ErTile);
  ER_CHECK(cs <= (uint32_t)p.wrec && p.wrec + T.nr * ER_REC <= p.wdesc);
  ER_CHECK(T.boff >= 0 && T.boff + cs <= p.state_doubles + 64);
  mbar_expect_tx(bar, bytes);
  bulk_g2s(B, p.state + T.boff, 8u * cs, bar);
  bulk_g2s(B + p.wrec, p.rec + (int64_t)T.r0 * ER_REC, (uint32_t)T.nr * ER_REC * 8u, bar);
  bulk_g2s(B + p.wdesc, tile_ptr, (uint32_t)sizeof(ErTile), bar);
}

constexpr int kWarpBlock = 256;  // 8 warps per CTA
constexpr int kWarps = kWarpBlock / 32;

template <int FEAT>
__global__ void __launch_bounds__(kWarpBlock, 2) warp_persistent(const ErStepParams p) {
  extern __shared__ __align__(16) double sm[];
  const int NB = p.wnb, BUFD = p.wbufd;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)NB * BUFD);
  unsigned *cnt = reinterpret_cast<unsigned *>(full + NB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool kappa0 = (FEAT & FEAT_KAPPA0) && p.has_kappa0;
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&full[b], 1);
      cnt[b] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();  // (programmatic launch) the previous kernel's results are complete and visible
  const double t0 = launch_t0(p);
  const int64_t ntc = p.n_tiles > (int64_t)blockIdx.x ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (int64_t k = 0; k < NB && k < ntc; ++k) {
      const int64_t tile = blockIdx.x + k * gridDim.x;
      issue_wtile(p, wload_head(p.tiles + tile), p.tiles + tile, sm + k * BUFD, &full[k], kappa0);
    }
  }
  // lane geometry (the same for every tile of the batch)
  const int N = p.wN, R = p.wR;
  const int g = lane / N;
  const int i = lane - g * N;
  const int q = warp * R + g;  // rod within the tile
  unsigned fbits_all = 0;
  int frod = INT_MAX;
  bool stored = false;
  for (int64_t k = 0; k < ntc; ++k) {
    const int b = (int)(k % NB);
    double *B = sm + (size_t)b * BUFD;
    if (k + 1 == ntc) griddep_launch_dependents();  // last tile: the next grid may launch
    mbar_wait(&full[b], (uint32_t)((k / NB) & 1));
    const ErTile &T = *reinterpret_cast<const ErTile *>(B + p.wdesc);
    const int ns = T.nslots, nel = T.nel;
    const int64_t boff = T.boff;
    WLane L;
    L.i = i;
    L.N = N;
    const bool active = g < R && q < T.nr;
    const RecFull rec{B + p.wrec + (active ? q : 0) * ER_REC};
    L.fl = active ? rec.flags() : 0;
    const int clamp = L.fl & FL_CLAMP_MASK;
    const bool last = active && i == N - 1;
    L.lb = (active ? WL_ACTIVE : 0u) | (active && i >= 1 ? WL_HAS_V : 0u) | (last ? WL_LAST : 0u) |
           (active && clamp == 1 && i == 0 ? WL_CL_NODE : 0u) | (last && clamp == 2 ? WL_CL_NODEN : 0u) |
           (active && ((clamp == 1 && i == 0) || (clamp == 2 && i == N - 1)) ? WL_CL_ELEM : 0u) |
           (active && (L.fl & FL_TIP) && clamp == 2 && i == 0 ? WL_TIP_I : 0u) |
           (last && (L.fl & FL_TIP) && clamp != 2 ? WL_TIP_N : 0u);
    const int slot = q * (N + 1) + i, el = q * N + i;
    L.node = T.nbase + slot;
    L.elem = T.ebase + el;
    L.rod = T.r0 + q;

    // ---- stage -> registers (node N stays in the buffer: xN)
    double r[3] = {0.0, 0.0, 0.0}, v[3] = {0.0, 0.0, 0.0};
    double Q[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, w[3] = {0.0, 0.0, 0.0}, k0s[3] = {0.0, 0.0, 0.0};
    if (active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        r[c] = B[c * ns + slot];
        v[c] = B[(3 + c) * ns + slot];
        w[c] = B[6 * ns + (ER_QST + c) * nel + el];
      }
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) Q[c] = B[6 * ns + c * nel + el];
    }
    XSmem xN{B + slot + 1, ns};
    complete_d3(Q);
    if ((FEAT & FEAT_KAPPA0) && active && i >= 1) {
      const int nvor = nel - T.nr;
#pragma unroll
      for (int c = 0; c < 3; ++c) k0s[c] = B[6 * ns + ER_EPL * nel + c * nvor + q * (N - 1) + i - 1];
    }

    // ---- the steps, in registers
    double t = t0;
    unsigned fbits = 0;
    for (int st = 0; st < p.n_steps; ++st) wstep<FEAT, XSmem, NoCross, RecFull>(p, rec, L, r, v, xN, Q, w, k0s, t, fbits);
    if (fbits) {
      fbits_all |= fbits;
      frod = min(frod, rec.canon());  // canonical rod id
    }

    // ---- registers -> stage, in place (only this lane ever touches these entries; node N is there already)
    if (active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        B[c * ns + slot] = r[c];
        B[(3 + c) * ns + slot] = v[c];
        B[6 * ns + (ER_QST + c) * nel + el] = w[c];
      }
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) B[6 * ns + c * nel + el] = Q[c];
    }
    fence_proxy_async();  // this thread's generic smem writes -> visible to the async proxy
    __syncwarp();
    if (lane == 0) {
      // the last of the CTA's warps to finish this tile stores it and refills the buffer
      const unsigned old = atom_add_acq_rel(&cnt[b], 1u);
      if (old == (unsigned)(kWarps * (k / NB) + kWarps - 1)) {
        const uint32_t tot = (uint32_t)(6 * ns + ER_EPL * nel);
        ER_CHECK(boff + tot <= p.state_doubles);
        bulk_s2g(p.state + boff, B, 8u * (tot & ~1u));
        bulk_commit();
        if (tot & 1u) p.state[boff + tot - 1] = B[tot - 1];
        stored = true;
        const int64_t kn = k + NB;
        if (kn < ntc) {
          const int64_t tile = blockIdx.x + kn * gridDim.x;
          const WHead Tn = wload_head(p.tiles + tile);
          bulk_wait_read_all();  // the store has read the buffer
          issue_wtile(p, Tn, p.tiles + tile, B, &full[b], kappa0);
        }
      }
    }
  }
  if (lane == 0 && stored) bulk_wait_all();  // stores complete before the kernel retires
  advance_tdev(p, t0);
  report_fault(p, fbits_all, frod);
}

// ------------------------------------------------------------------------------------------
// warp_stream: the same lane mapping and step, but every warp is its own pipeline.  The batch is laid
// out in warp-sized tiles (wR rods each; the standard tile block of er_layout.h, so a tile's state is
// one contiguous block of a few KB).  The warps of the grid take the tiles in turn (warp gw: tiles gw,
// gw + G, ...); a warp prefetches its next tiles into its own ring of wnb shared-memory slots with
// 16-byte cp.async copies, waits only for its own copies (cp.async.wait_group + __syncwarp), computes,
// and stores its results straight from registers with coalesced streaming stores.  No mbarrier, no
// block barrier, no warp ever waits for another.  Tile geometry comes from the uniform layout (equal
// rods, identity order: tile t holds rods t*wR .. and starts at t*wcs), so no descriptor is read.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

struct WTile {
  int64_t boff;           // the tile's block (doubles)
  int64_t r0;             // packed id of its first rod
  int32_t nr;             // rods in the tile
  int32_t ns, nel, cs;    // node / element plane strides, block size (even)
};
// NT > 0: rods of NT elements and a full tile (wR rods) -- the geometry is compile-time; NT = 0: from p
template <int NT>
__device__ __forceinline__ WTile wtile_geom(const ErStepParams &p, int64_t t, bool kappa0) {
  constexpr int RT = NT ? 32 / NT : 1;
  const int N = NT ? NT : p.wN, R = NT ? RT : p.wR;
  WTile g;
  g.r0 = t * R;
  g.nr = NT ? RT : (int)min((int64_t)R, p.wrods - g.r0);
  g.boff = t * p.wcs;
  g.ns = g.nr * (N + 1);
  g.nel = g.nr * N;
  g.cs = (6 * g.ns + ER_EPL * g.nel + (kappa0 ? 3 * (g.nel - g.nr) : 0) + 1) & ~1;
  return g;
}
// the tile's block and its rod records into slot S: 16-byte copies over contiguous ranges
template <int NT>
__device__ __forceinline__ void issue_wtile_async(const ErStepParams &p, const WTile &g, double *S, int lane) {
  const double *G = p.state + g.boff;
  if (NT) {
    constexpr int NTc = NT ? NT : 1;
    constexpr int CS = (6 * (32 / NTc) * (NTc + 1) + ER_EPL * (32 / NTc) * NTc + 1) & ~1;  // state planes
#pragma unroll
    for (int x = 2 * lane; x < CS; x += 64) cp_async16(S + x, G + x);
    for (int x = CS + 2 * lane; x < g.cs; x += 64) cp_async16(S + x, G + x);  // kappa0 planes
  } else {
    for (int x = 2 * lane; x < g.cs; x += 64) cp_async16(S + x, G + x);
  }
  const double *Rc = p.rec + g.r0 * ER_REC;
  double *SR = S + p.wcs;
  for (int x = 2 * lane; x < g.nr * ER_REC; x += 64) cp_async16(SR + x, Rc + x);
}

template <bool UNI>
__device__ __forceinline__ typename std::conditional<UNI, RecUni, RecFull>::type make_rc(const ErStepParams &p,
                                                                                     const double *r);
template <>
__device__ __forceinline__ RecFull make_rc<false>(const ErStepParams &, const double *r) { return RecFull{r}; }
template <>
__device__ __forceinline__ RecUni make_rc<true>(const ErStepParams &p, const double *r) { return RecUni{r, p}; }

// Size and source of a tile's rod records (full or shared-material form).
template <int FEAT>
__device__ __forceinline__ uint32_t rec_bytes(int nr) { return (uint32_t)nr * ((FEAT & FEAT_UNI) ? ER_WREC : ER_REC) * 8u; }
template <int FEAT>
__device__ __forceinline__ const double *rec_src(const ErStepParams &p, int64_t r0) {
  return (FEAT & FEAT_UNI) ? p.wrecu + r0 * ER_WREC : p.rec + r0 * ER_REC;
}

// One tile of one warp: stage slot -> registers, n_steps steps, results to HBM.
// TO_SMEM: the results go back into the slot, in place (a bulk store moves the block); else straight
// to HBM from registers.
// lane: the lane's position in the tile's element range (a pair's second warp: 32 + lane).
template <int FEAT, int NT, bool TO_SMEM = false, class CR = NoCross>
__device__ __forceinline__ void stream_tile(const ErStepParams &p, const WTile &g, const double *S, int lane,
                                            double t0, unsigned &fbits_all, int &frod, const CR &cr = CR()) {
  constexpr int NTc = NT ? NT : 1;
  const int N = NT ? NT : p.wN;
  const int gl = NT ? lane / NTc : lane / N;
  const int i = lane - gl * N;
  const int ns = NT ? (32 / NTc) * (NTc + 1) : g.ns, nel = NT ? (32 / NTc) * NTc : g.nel;
  WLane L;
  L.i = i;
  L.N = N;
  const bool active = NT ? true : gl < g.nr;
  constexpr bool UNI = (FEAT & FEAT_UNI) != 0;
  using RC = typename std::conditional<UNI, RecUni, RecFull>::type;
  const RC rec = make_rc<UNI>(p, S + p.wcs + (active ? gl : 0) * (UNI ? ER_WREC : ER_REC));
  L.fl = active ? rec.flags() : 0;
  const int clamp = L.fl & FL_CLAMP_MASK;
  const bool last = active && i == N - 1;
  L.lb = (active ? WL_ACTIVE : 0u) | (active && i >= 1 ? WL_HAS_V : 0u) | (last ? WL_LAST : 0u) |
         (active && clamp == 1 && i == 0 ? WL_CL_NODE : 0u) | (last && clamp == 2 ? WL_CL_NODEN : 0u) |
         (active && ((clamp == 1 && i == 0) || (clamp == 2 && i == N - 1)) ? WL_CL_ELEM : 0u) |
         (active && (L.fl & FL_TIP) && clamp == 2 && i == 0 ? WL_TIP_I : 0u) |
         (last && (L.fl & FL_TIP) && clamp != 2 ? WL_TIP_N : 0u);
  const int sl = gl * (N + 1) + i, el = gl * N + i;
  L.rod = (int)(g.r0 + gl);
  L.node = g.r0 * (N + 1) + sl;
  L.elem = g.r0 * N + el;
  double r[3] = {0.0, 0.0, 0.0}, v[3] = {0.0, 0.0, 0.0};
  double Q[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}, w[3] = {0.0, 0.0, 0.0}, k0s[3] = {0.0, 0.0, 0.0};
  if (active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = S[c * ns + sl];
      v[c] = S[(3 + c) * ns + sl];
      w[c] = S[6 * ns + (ER_QST + c) * nel + el];
    }
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) Q[c] = S[6 * ns + c * nel + el];
  }
  complete_d3(Q);
  if ((FEAT & FEAT_KAPPA0) && active && i >= 1) {
    const int nvor = nel - (NT ? 32 / NTc : g.nr);
#pragma unroll
    for (int c = 0; c < 3; ++c) k0s[c] = S[6 * ns + ER_EPL * nel + c * nvor + gl * (N - 1) + i - 1];
  }
  XSmem xN{const_cast<double *>(S) + sl + 1, ns};  // node N (last lanes), plane stride ns
  double tt = t0;
  unsigned fbits = 0;
  for (int st = 0; st < p.n_steps; ++st)
    wstep<FEAT, XSmem, CR, RC>(p, rec, L, r, v, xN, Q, w, k0s, tt, fbits, cr, st + 1 == p.n_steps);
  if (fbits) {
    fbits_all |= fbits;
    frod = min(frod, rec.canon());
  }
  if (TO_SMEM) {  // in place: only this lane touches these entries (node N is there already)
    double *O = const_cast<double *>(S);
    if (active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        O[c * ns + sl] = r[c];
        O[(3 + c) * ns + sl] = v[c];
        O[6 * ns + (ER_QST + c) * nel + el] = w[c];
      }
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) O[6 * ns + c * nel + el] = Q[c];
    }
    return;
  }
  // ---- results straight to HBM (coalesced streaming stores per plane)
  double *Gs = p.state + g.boff;
  if (active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      __stcs(Gs + c * ns + sl, r[c]);
      __stcs(Gs + (3 + c) * ns + sl, v[c]);
    }
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) __stcs(Gs + 6 * ns + c * nel + el, Q[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c) __stcs(Gs + 6 * ns + (ER_QST + c) * nel + el, w[c]);
  }
  if (last) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      __stcs(Gs + c * ns + sl + 1, xN.r(c));
      __stcs(Gs + (3 + c) * ns + sl + 1, xN.v(c));
    }
  }
}

// NT: the batch's rod length when this instantiation is specialised for it (full tiles take the
// compile-time geometry; a partial last tile the general one), else 0.
template <int FEAT, int NB, int NT>
__global__ void __launch_bounds__(kWarpBlock, 2) warp_stream(const ErStepParams p) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *ring = sm + (size_t)warp * NB * p.wch;  // this warp's NB slots
  const bool kappa0 = (FEAT & FEAT_KAPPA0) && p.has_kappa0;
  griddep_wait();  // (programmatic launch) the previous kernel's results are complete and visible
  const double t0 = launch_t0(p);
  const int64_t G = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  // tiles [0, nfull) are full (wR rods); a partial last tile takes the general path
  const int64_t nfull = p.wrods / p.wR;
  auto issue = [&](int64_t t, double *S) {
    if (NT && t < nfull) issue_wtile_async<NT>(p, wtile_geom<NT>(p, t, kappa0), S, lane);
    else issue_wtile_async<0>(p, wtile_geom<0>(p, t, kappa0), S, lane);
  };
  // prefetch the first NB - 1 tiles (one commit group each, empty past the end)
#pragma unroll
  for (int j = 0; j < NB - 1; ++j) {
    const int64_t t = gw + j * G;
    if (t < p.n_tiles) issue(t, ring + j * p.wch);
    cp_async_commit();
  }
  unsigned fbits_all = 0;
  int frod = INT_MAX;
  int slot_j = 0;  // ring slot of the current tile
  for (int64_t t = gw; t < p.n_tiles; t += G) {
    {  // prefetch tile t + (NB-1) G into the slot the previous tile used (its reads are done)
      const int64_t tn = t + (NB - 1) * G;
      const int sn = slot_j == 0 ? NB - 1 : slot_j - 1;
      if (tn < p.n_tiles) issue(tn, ring + sn * p.wch);
      cp_async_commit();
    }
    if (t + G >= p.n_tiles) griddep_launch_dependents();  // last tile of this warp
    cp_async_wait<NB - 1>();  // this lane's copies of tile t have landed
    __syncwarp();             // ... and every other lane's
    const double *S = ring + slot_j * p.wch;
    slot_j = slot_j + 1 == NB ? 0 : slot_j + 1;
    if (NT && t < nfull) stream_tile<FEAT, NT>(p, wtile_geom<NT>(p, t, kappa0), S, lane, t0, fbits_all, frod);
    else stream_tile<FEAT, 0>(p, wtile_geom<0>(p, t, kappa0), S, lane, t0, fbits_all, frod);
    __syncwarp();  // every lane's reads of this slot are done before a later prefetch reuses it
  }
  cp_async_wait<0>();
  advance_tdev(p, t0);
  report_fault(p, fbits_all, frod);
}

// warp_bulk: warp_stream's per-warp pipeline with TMA bulk copies: lane 0 loads a tile's contiguous
// block and records into a slot with two cp.async.bulk copies completing the slot's mbarrier, the warp
// computes, writes its results back into the slot, and lane 0 bulk-stores the block.  The slot of the
// previous tile is refilled (NB - 1 tiles ahead) once its store has read it.
constexpr int kBulkWarps = ER_WB_WARPS;
// threadIdx.x read once: the result of a volatile asm is not rematerialised, so the S2R and the
// lane / warp arithmetic hanging off it are not re-issued at every use under register pressure
// (warp_bulk: 16 -> 8 S2R in the loop, cfg3 0.7434 -> 0.7381 ms/step, interleaved A/B).
__device__ __forceinline__ int tid_once() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}
template <int FEAT, int NB, int NT>
__global__ void __launch_bounds__(32 * kBulkWarps, ER_WB_MINB) warp_bulk(const ErStepParams p) {
  constexpr int kWarps = kBulkWarps;
  extern __shared__ __align__(16) double sm[];
  const int tid = tid_once(), lane = tid & 31, warp = tid >> 5;
  double *ring = sm + (size_t)warp * NB * p.wch;  // this warp's NB slots
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)kWarps * NB * p.wch) + warp * NB;
  const bool kappa0 = (FEAT & FEAT_KAPPA0) && p.has_kappa0;
  if (lane == 0) {
    for (int j = 0; j < NB; ++j) mbar_init(&bars[j], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();  // (programmatic launch) the previous kernel's results are complete and visible
  const double t0 = launch_t0(p);
  const int64_t G = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nfull = p.wrods / p.wR;
  auto geom = [&](int64_t t) { return (NT && t < nfull) ? wtile_geom<NT>(p, t, kappa0) : wtile_geom<0>(p, t, kappa0); };
  auto issue = [&](int64_t t, int j) {  // lane 0
    const WTile g = geom(t);
    double *S = ring + j * p.wch;
    mbar_expect_tx(&bars[j], 8u * (uint32_t)g.cs + rec_bytes<FEAT>(g.nr));
    bulk_g2s(S, p.state + g.boff, 8u * (uint32_t)g.cs, &bars[j]);
    bulk_g2s(S + p.wcs, rec_src<FEAT>(p, g.r0), rec_bytes<FEAT>(g.nr), &bars[j]);
  };
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NB - 1; ++j)
      if (gw + j * G < p.n_tiles) issue(gw + j * G, j);
  }
  unsigned fbits_all = 0;
  int frod = INT_MAX;
  int64_t k = 0;
  // slot of tile k, its load parity, and the slot the refill goes to (k + NB - 1): counters instead of
  // 64-bit k % NB, k / NB per tile
  int j = 0, jn = NB - 1;
  uint32_t par = 0;
  for (int64_t t = gw; t < p.n_tiles; t += G, ++k) {
#if ER_TRACE  // measurement builds: per-warp timeline [global warp][64 tiles][4] (tools/warp_timeline.py)
    unsigned long long *tr = (p.trace && lane == 0 && k < ER_TRACE_ITERS) ? p.trace + (gw * ER_TRACE_ITERS + k) * 8 : nullptr;
    if (tr) tr[0] = (gtimer() & ((1ull << 48) - 1)) | ((unsigned long long)smid() << 56);
#endif
    if (t + G >= p.n_tiles) griddep_launch_dependents();  // last tile of this warp
    mbar_wait(&bars[j], par);
#if ER_TRACE
    if (tr) tr[1] = gtimer() & ((1ull << 48) - 1);
#endif
    double *S = ring + j * p.wch;
    const WTile g = geom(t);
#ifndef ER_EXP_PROBE  // (measurement builds, -DER_EXP_PROBE: the memory stream alone, tiles stored back unchanged)
    if (NT && t < nfull) stream_tile<FEAT, NT, true>(p, g, S, lane, t0, fbits_all, frod);
    else stream_tile<FEAT, 0, true>(p, g, S, lane, t0, fbits_all, frod);
#endif
#if ER_TRACE
    if (tr) tr[2] = gtimer() & ((1ull << 48) - 1);
#endif
    fence_proxy_async();  // this lane's generic smem writes -> visible to the async proxy
    __syncwarp();
#if ER_TRACE
    if (tr) tr[3] = gtimer() & ((1ull << 48) - 1);
#endif
#if !ER_TRACE  // full uniform tiles (this one and the refill): store and refill geometry are compile-time
    // (cfg3 0.7381 -> 0.7327 ms/step, interleaved A/B; the general path below serves the last tiles)
    if (NT && !(FEAT & FEAT_KAPPA0) && p.wl2pf == 0 && t + (NB - 1) * G < nfull) {
      if (lane == 0) {
        constexpr int NTc = NT ? NT : 1, RT = 32 / NTc;
        constexpr uint32_t TOT = 6u * RT * (NTc + 1) + ER_EPL * 32u, CS = (TOT + 1u) & ~1u;
        constexpr uint32_t RB = (uint32_t)RT * ((FEAT & FEAT_UNI) ? ER_WREC : ER_REC) * 8u;
        static_assert((TOT & 1u) == 0, "odd block");
        bulk_s2g(p.state + t * p.wcs, S, 8u * TOT);
        bulk_commit();
        const int64_t tn = t + (NB - 1) * G;
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        double *Sn = ring + jn * p.wch;
        mbar_expect_tx(&bars[jn], 8u * CS + RB);
        bulk_g2s(Sn, p.state + tn * p.wcs, 8u * CS, &bars[jn]);
        bulk_g2s(Sn + p.wcs, rec_src<FEAT>(p, tn * RT), RB, &bars[jn]);
      }
    } else
#endif
    if (lane == 0) {
      const uint32_t tot = (uint32_t)(6 * g.ns + ER_EPL * g.nel);
      bulk_s2g(p.state + g.boff, S, 8u * (tot & ~1u));
      bulk_commit();
      if (tot & 1u) p.state[g.boff + tot - 1] = S[tot - 1];
#if ER_TRACE
      if (tr) tr[4] = gtimer() & ((1ull << 48) - 1);
#endif
      const int64_t tn = t + (NB - 1) * G;
      if (tn < p.n_tiles) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the previous tile's store read its slot
#if ER_TRACE
        if (tr) tr[5] = gtimer() & ((1ull << 48) - 1);
#endif
        issue(tn, jn);
      }
#if ER_TRACE
      if (tr) tr[6] = gtimer() & ((1ull << 48) - 1);
#endif
      // L2 prefetch further ahead (measurement option ER_WARP_L2PF; no shared memory needed)
      if (p.wl2pf > 0) {
        const int64_t tp = tn + (int64_t)p.wl2pf * G;
        if (tp < p.n_tiles) {
          const WTile gp = geom(tp);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.state + gp.boff), "r"(8u * (uint32_t)gp.cs) : "memory");
        }
      }
    }
    __syncwarp();
    jn = j;
    if (++j == NB) {
      j = 0;
      par ^= 1u;
    }
  }
  if (lane == 0) bulk_wait_all();  // stores complete before the kernel retires
  advance_tdev(p, t0);
  report_fault(p, fbits_all, frod);
}

// pair_bulk: warp_bulk for rods of 33..64 elements (cfg4's 64): a rod is one tile and lies on the 64
// lanes of a warp pair (element i on warp i / 32, lane i % 32); the pair shares a slot ring, its
// lane 0 of warp 0 issues the TMA loads and stores, and the two warps meet at a named barrier in each
// of the three exchanges and once per tile before the store.
template <int FEAT, int NB>
__global__ void __launch_bounds__(kWarpBlock, 2) pair_bulk(const ErStepParams p) {
  constexpr int kPairs = kWarps / 2;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;  // (tid_once: more spills here, no gain)
  const int pw = warp >> 1, wp = warp & 1;
  double *ring = sm + (size_t)pw * NB * p.wch;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)kPairs * NB * p.wch) + pw * NB;
  double *mbox = reinterpret_cast<double *>(reinterpret_cast<uint64_t *>(sm + (size_t)kPairs * NB * p.wch) + kPairs * NB) + pw * 24;
  const bool kappa0 = (FEAT & FEAT_KAPPA0) && p.has_kappa0;
  const bool issuer = wp == 0 && lane == 0;
  const int barid = 1 + pw;
  if (issuer) {
    for (int j = 0; j < NB; ++j) mbar_init(&bars[j], 1);
    fence_mbar_init();
  }
  pair_sync(barid);
  griddep_wait();
  const double t0 = launch_t0(p);
  const int64_t G = (int64_t)gridDim.x * kPairs;
  const int64_t gp = (int64_t)blockIdx.x * kPairs + pw;
  // Step-graph launches alternate the direction of the walk over the tiles (tpar = launch parity):
  // a launch starts on the tiles the previous one stored last, which the L2 still holds (cfg4: 1 GB
  // of state, 12% of it fits the 126 MB L2: 0.221 -> 0.216 ms/step; no gain for cfg3's 4 GB in
  // warp_bulk).  Rods are independent, so the order changes no result.
  const bool rev = p.tdev && (p.tpar & 1);
  auto issue = [&](int64_t t, int j) {
    const WTile g = wtile_geom<0>(p, rev ? p.n_tiles - 1 - t : t, kappa0);
    double *S = ring + j * p.wch;
    mbar_expect_tx(&bars[j], 8u * (uint32_t)g.cs + rec_bytes<FEAT>(g.nr));
    bulk_g2s(S, p.state + g.boff, 8u * (uint32_t)g.cs, &bars[j]);
    bulk_g2s(S + p.wcs, rec_src<FEAT>(p, g.r0), rec_bytes<FEAT>(g.nr), &bars[j]);
  };
  if (issuer) {
#pragma unroll
    for (int j = 0; j < NB - 1; ++j)
      if (gp + j * G < p.n_tiles) issue(gp + j * G, j);
  }
  const PairCross cr{mbox, barid, wp == 0 && lane == 31, wp == 1 && lane == 0};
  unsigned fbits_all = 0;
  int frod = INT_MAX;
  int j = 0, jn = NB - 1;  // slot of this tile, slot of the refill (k + NB - 1), load parity
  uint32_t par = 0;
  for (int64_t t = gp; t < p.n_tiles; t += G) {
    if (t + G >= p.n_tiles) griddep_launch_dependents();
    mbar_wait(&bars[j], par);
    const WTile g = wtile_geom<0>(p, rev ? p.n_tiles - 1 - t : t, kappa0);
    double *S = ring + j * p.wch;
    stream_tile<FEAT, 0, true, PairCross>(p, g, S, wp * 32 + lane, t0, fbits_all, frod, cr);
    fence_proxy_async();
    pair_sync(barid);  // both warps' results are in the slot
    if (issuer) {
      const uint32_t tot = (uint32_t)(6 * g.ns + ER_EPL * g.nel);
      bulk_s2g(p.state + g.boff, S, 8u * (tot & ~1u));
      bulk_commit();
      if (tot & 1u) p.state[g.boff + tot - 1] = S[tot - 1];
      const int64_t tn = t + (NB - 1) * G;
      if (tn < p.n_tiles) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        issue(tn, jn);
      }
    }
    jn = j;
    if (++j == NB) {
      j = 0;
      par ^= 1u;
    }
  }
  if (issuer) bulk_wait_all();
  advance_tdev(p, t0);
  report_fault(p, fbits_all, frod);
}

}  // namespace er

namespace {

template <int FEAT>
cudaError_t launch_warp(const ErStepParams &p, cudaStream_t st) {
  auto k = er::warp_persistent<FEAT>;
  const size_t sm = (size_t)p.wnb * p.wbufd * 8 + (size_t)p.wnb * 12 + 16;
  // occupancy per (device, shared-memory size): the size depends on the batch's tile geometry
  static int cached_dev = -1, cached_per_sm = 0;
  static size_t cached_sm = 0, set_sm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (p.wnb < 1 || p.wnb > 8) return cudaErrorInvalidValue;
  if (dev != cached_dev || sm != cached_sm) {
    if (sm > set_sm || dev != cached_dev) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(sm, set_sm));
      if (e != cudaSuccess) return e;
      set_sm = std::max(sm, set_sm);
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, er::kWarpBlock, sm);
    if (e != cudaSuccess) return e;
    cached_dev = dev;
    cached_sm = sm;
    cached_per_sm = per_sm > 0 ? per_sm : 1;
  }
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::min<int64_t>(p.n_tiles, (int64_t)n_sm * cached_per_sm);
  static const bool pdl = std::getenv("ER_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g, 1, 1);
  cfg.blockDim = dim3(er::kWarpBlock, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int FEAT, int NB>
cudaError_t launch_stream_nb(const ErStepParams &p, cudaStream_t st) {
  // rods of 16 elements (BASELINE configs[2], 1024^2 filaments) get the specialised instantiation
  static const bool generic = std::getenv("ER_WARP_GENERIC") != nullptr;
  static const bool cpasync = std::getenv("ER_WARP_CPASYNC") != nullptr;  // A/B: per-lane cp.async + direct stores
  const bool pair = p.wN > 32;  // rods of 33..64 elements: one rod per warp pair
  void (*k)(ErStepParams);
  if constexpr ((FEAT & FEAT_UNI) != 0) {  // (er_launch_warp never combines FEAT_UNI with ER_WARP_CPASYNC)
    k = pair ? er::pair_bulk<FEAT, NB> : (p.wN == 16 && !generic) ? er::warp_bulk<FEAT, NB, 16> : er::warp_bulk<FEAT, NB, 0>;
  } else {
    k = pair ? er::pair_bulk<FEAT, NB>
        : cpasync ? ((p.wN == 16 && !generic) ? er::warp_stream<FEAT, NB, 16> : er::warp_stream<FEAT, NB, 0>)
                  : ((p.wN == 16 && !generic) ? er::warp_bulk<FEAT, NB, 16> : er::warp_bulk<FEAT, NB, 0>);
  }
  const int units = pair ? er::kWarps / 2 : er::kBulkWarps;  // pipelines per CTA
  const int block = pair ? er::kWarpBlock : 32 * er::kBulkWarps;
  const size_t sm = (size_t)units * NB * p.wch * 8 + (size_t)units * NB * 8 + (pair ? (size_t)units * 24 * 8 : 0);
  static int cached_dev = -1, cached_per_sm = 0;
  static size_t cached_sm = 0, set_sm = 0;
  static const void *cached_k = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev || sm != cached_sm || (const void *)k != cached_k) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(sm, set_sm));
    if (e != cudaSuccess) return e;
    set_sm = std::max(sm, set_sm);
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, sm);
    if (e != cudaSuccess) return e;
    cached_dev = dev;
    cached_sm = sm;
    cached_k = (const void *)k;
    cached_per_sm = per_sm > 0 ? per_sm : 1;
  }
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::min<int64_t>((p.n_tiles + units - 1) / units, (int64_t)n_sm * cached_per_sm);
  static const bool pdl = std::getenv("ER_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g, 1, 1);
  cfg.blockDim = dim3((unsigned)block, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}
template <int FEAT>
cudaError_t launch_stream(const ErStepParams &p, cudaStream_t st) {
  if (p.wnb <= 2) return launch_stream_nb<FEAT, 2>(p, st);
  if (p.wnb == 3) return launch_stream_nb<FEAT, 3>(p, st);
  return launch_stream_nb<FEAT, 4>(p, st);
}

}  // namespace

extern "C" {

// The warp kernel for the batch's feature set (GENERAL | KAPPA0 bits, plus FEAT_EXTRA or FEAT_ACT).
cudaError_t er_launch_warp(const ErStepParams *p, int feat, cudaStream_t st) {
  if (p->n_tiles <= 0) return cudaSuccess;
  const int base = feat & (FEAT_GENERAL | FEAT_KAPPA0);
  const int x = (feat & FEAT_EXTRA) ? FEAT_EXTRA : (feat & FEAT_ACT) ? FEAT_ACT : 0;
  if (p->wrt > 0) {  // per-warp streaming pipeline (default)
    static const bool cpasync = std::getenv("ER_WARP_CPASYNC") != nullptr;
    if (p->wuni && p->wrecu && !cpasync && !(base & FEAT_GENERAL) && x != FEAT_EXTRA) {  // shared material
      switch (x | base) {
        case 0: return launch_stream<FEAT_UNI>(*p, st);
        case FEAT_KAPPA0: return launch_stream<FEAT_UNI | FEAT_KAPPA0>(*p, st);
        case FEAT_ACT: return launch_stream<FEAT_UNI | FEAT_ACT>(*p, st);
        default: return launch_stream<FEAT_UNI | FEAT_ACT | FEAT_KAPPA0>(*p, st);
      }
    }
    switch (x | base) {
      case 0: return launch_stream<0>(*p, st);
      case 1: return launch_stream<1>(*p, st);
      case 2: return launch_stream<2>(*p, st);
      case 3: return launch_stream<3>(*p, st);
      case FEAT_ACT | 0: return launch_stream<FEAT_ACT | 0>(*p, st);
      case FEAT_ACT | 1: return launch_stream<FEAT_ACT | 1>(*p, st);
      case FEAT_ACT | 2: return launch_stream<FEAT_ACT | 2>(*p, st);
      case FEAT_ACT | 3: return launch_stream<FEAT_ACT | 3>(*p, st);
      case FEAT_EXTRA | 0: return launch_stream<FEAT_EXTRA | 0>(*p, st);
      case FEAT_EXTRA | 1: return launch_stream<FEAT_EXTRA | 1>(*p, st);
      case FEAT_EXTRA | 2: return launch_stream<FEAT_EXTRA | 2>(*p, st);
      default: return launch_stream<FEAT_EXTRA | 3>(*p, st);
    }
  }
  switch (x | base) {
    case 0: return launch_warp<0>(*p, st);
    case 1: return launch_warp<1>(*p, st);
    case 2: return launch_warp<2>(*p, st);
    case 3: return launch_warp<3>(*p, st);
    case FEAT_ACT | 0: return launch_warp<FEAT_ACT | 0>(*p, st);
    case FEAT_ACT | 1: return launch_warp<FEAT_ACT | 1>(*p, st);
    case FEAT_ACT | 2: return launch_warp<FEAT_ACT | 2>(*p, st);
    case FEAT_ACT | 3: return launch_warp<FEAT_ACT | 3>(*p, st);
    case FEAT_EXTRA | 0: return launch_warp<FEAT_EXTRA | 0>(*p, st);
    case FEAT_EXTRA | 1: return launch_warp<FEAT_EXTRA | 1>(*p, st);
    case FEAT_EXTRA | 2: return launch_warp<FEAT_EXTRA | 2>(*p, st);
    default: return launch_warp<FEAT_EXTRA | 3>(*p, st);
  }
}

}  // extern "C"
