// er_kernels.cu -- the hot path (L2) of the batched Cosserat rod step on sm_100a, fp64.
// No tensor cores: nothing here is a dense contraction.
//
// Mapping: a rod-aligned tile of <= BLOCK "slots" per CTA; slot s of a rod is
// node i, element i (i < N) and Voronoi domain i (1 <= i < N) of that rod, one thread per
// slot.  Neighbour data (node i+1, element i-1, n_{i-1}, mbar_{i+1}, beta_{i+1}) move through
// shared memory; rods never straddle tiles, so there are no halos in HBM and no grid-wide
// barrier -- the paper's asynchronous protocol is free here.
//
// One step of one slot, `step_body` below:
//   A1-A3  r += h/2 v; Q <- rot(h/2 w) Q; clamped entries are not moved
//   A4-A5  l = r_{i+1} - r_i, e, de/dt, sigma = Q l / lhat - e3, nbar = S (sigma - sigma0)/e, n = Q^T nbar
//   A6     kappa = logrot(Q_k Q_{k-1}^T)/Dh, mbar = Bv (kappa - kappa0(t+h/2))/eps^3, beta = (kappa x mbar) Dh
//   A7,A9  a = (n_i - n_{i-1} + F_tip)/m + g - nu v;   v += h a
//   A8,A9  C = mbar_{i+1} - mbar_i + (beta_{i+1} + beta_i)/2 + (Q l) x nbar + c_mag
//          alpha = e J^-1 C + Euler((J w) x w) / J + w de/dt / e - nu w;   w += h alpha
//   A10    r += h/2 v; Q <- rot(h/2 w) Q
// (Q l) x nbar == lhat (Q t) x S(sigma - sigma0); the two rate terms are Eq. (1b)'s
// (J w / e) x w and (J w / e^2) de/dt multiplied by e/J.
//
// Kernels:
//  fused_persistent : production.  148 x k persistent CTAs walk the tile list; while a tile is
//                     computed, the next tile's state, records and offsets stream into the
//                     other half of a double-buffered smem stage with TMA 1-D bulk copies
//                     (cp.async.bulk + mbarrier).  n_steps steps per tile (1 = the B_min
//                     design; k > 1 = temporal blocking).
//  simple_kernel    : one tile per CTA, plain loads; MODE_FUSED (ablation), MODE_DRIFT /
//                     MODE_DYN (the staged three-launch path).
//  diag_kernel      : per-tile partial sums of the energy functional, deterministic.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "er_layout.h"
#include "er_math.cuh"
#include "er_tma.cuh"

namespace er {

enum { MODE_FUSED = 0, MODE_DRIFT = 1, MODE_DYN = 2 };

// exchange planes (stride BLOCK): A = r(0-2) v(3-5) d1 d2 (6-11; the reader rebuilds d3);
// B = l(12) n(13-15); C aliases A: mbar(0-2) beta(3-5).  16 planes.
enum { XR = 0, XV = 3, XQ = 6, XL = 6 + ER_QST, XN = 7 + ER_QST, XM = 0, XB = 3, XPLANES = 10 + ER_QST };

struct SlotInfo {
  int s;            // slot (thread) index in the tile
  int i, N, q;      // node index in the rod, rod length, rod index in the tile
  int rod;          // global rod id
  int64_t node, elem, vor;  // global indices
  int fl;
  bool active, has_e, has_v, cl_node, cl_elem;
};

__device__ __forceinline__ void finish_slot(SlotInfo &si) {
  const int clamp = si.fl & FL_CLAMP_MASK;
  si.has_e = si.active && si.i < si.N;
  si.has_v = si.active && si.i >= 1 && si.i < si.N;
  si.cl_node = si.active && ((clamp == 1 && si.i == 0) || (clamp == 2 && si.i == si.N));
  si.cl_elem = si.has_e && ((clamp == 1 && si.i == 0) || (clamp == 2 && si.i == si.N - 1));
}

// Contact force on node i (NEXT-4, DESIGN §3 #27): er_contact.cu left, per element j, the force
// on its nodes j and j+1 in ErContactParams.fc (half-space forces included); node i collects
// element i's first and element i-1's second share.
__device__ __forceinline__ void contact_node_load(const ErStepParams &p, const SlotInfo &si, double f[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double lo = si.has_e ? __ldg(p.cfc + c * p.cfs + si.elem) : 0.0;
    const double hi = si.active && si.i >= 1 ? __ldg(p.cfc + (3 + c) * p.cfs + si.elem - 1) : 0.0;
    f[c] = lo + hi;
  }
}

// Contact mode, after drift-1: node r (half step) and v^n to the AoS node records the contact
// kernels read, and the Verlet-list check against the positions of the last list build (a node
// farther than skin/2 from it raises the rebuild flag).  Called by every thread of the CTA.
__device__ __forceinline__ void contact_emit(const ErStepParams &p, const SlotInfo &si, const double r[3],
                                             const double v[3], const double rb[3]) {
  bool moved = false;
  if (si.active) {
    double *o = p.cnode + 6 * si.node;
    double d2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      o[c] = r[c];
      o[3 + c] = v[c];
      const double d = r[c] - rb[c];
      d2 = fma(d, d, d2);
    }
    moved = !(d2 <= p.disp2);  // also for NaN
  }
  if (__any_sync(0xffffffffu, moved) && (threadIdx.x & 31) == 0) atomicOr(p.rebuild, 1);
}
__device__ __forceinline__ void contact_build_pos(const ErStepParams &p, const SlotInfo &si, double rb[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) rb[c] = si.active ? __ldg(p.cbuild + 3 * si.node + c) : 0.0;
}


// ------------------------------------------------------------------------------------------
// One position-Verlet step (or one stage of it) of one slot.  State in registers; X is the
// smem exchange area (XPLANES planes of stride BLOCK); rec points at the rod record (smem in
// the persistent kernel, global in the simple one).  k0s: static rest curvature of the slot's
// Voronoi domain (FEAT_KAPPA0).
// Exchange barrier of one CTA (tiles); long rods pass a cluster-wide one that also fills the halos.
struct CtaSync {
  __device__ __forceinline__ void operator()(int) const { __syncthreads(); }
};

template <int BLOCK, int FEAT, bool DRIFT1, bool DYN, bool DRIFT2, int XS = BLOCK, class XSync = CtaSync>
__device__ __forceinline__ void step_body(const ErStepParams &p, double *__restrict__ X,
                                          const double *__restrict__ rec, const SlotInfo &si,
                                          double r[3], double v[3], double Q[9], double w[3],
                                          const double k0s[3], double &t, unsigned &fbits,
                                          const double *fcon = nullptr, XSync xsync = XSync(),
                                          bool final_step = false) {
  constexpr bool GEN = (FEAT & FEAT_GENERAL) != 0;
  constexpr bool EXTRA = (FEAT & FEAT_EXTRA) != 0;
  constexpr bool ACT = (FEAT & (FEAT_EXTRA | FEAT_ACT)) != 0;
  constexpr bool CONTACT = (FEAT & FEAT_CONTACT) != 0;
  const int s = si.s, i = si.i, N = si.N;
  const double h = p.h, hh = 0.5 * p.h;
  const bool general = GEN && (si.fl & FL_GENERAL);
  const double t_half = t + hh;
  auto gp = [&](int plane) { return __ldg(p.gpar + plane * p.ng + si.node); };

  // A clamped node / element (and a slot without an element) moves by a zero step: r + 0 v = r and
  // rot(0) Q = Q exactly, so the drifts take no branch at the rods' ends.
  const double hr = si.cl_node ? 0.0 : hh, hq = (si.has_e && !si.cl_elem) ? hh : 0.0;
  if (DRIFT1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = fma(hr, v[c], r[c]);
    rotate_inplace(Q, hq * w[0], hq * w[1], hq * w[2]);
  }
  if (DYN) {
    // ---- exchange A
    if (si.active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { X[(XR + c) * XS + s] = r[c]; X[(XV + c) * XS + s] = v[c]; }
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) X[(XQ + c) * XS + s] = Q[c];  // d3 is rebuilt by the reader
    }
    xsync(0);

    // ---- A4-A5 edge i: kinematics, shear/stretch strain, stress
    double Ql[3] = {0.0, 0.0, 0.0}, nb[3] = {0.0, 0.0, 0.0}, n[3] = {0.0, 0.0, 0.0};
    double l = 0.0, inv_e = 0.0, e = 1.0, edot = 0.0;
    if (si.has_e) {
      const double lh = general ? gp(GP_LHAT) : rec[REC_LHAT];
      const double ilh = general ? gp(GP_ILHAT) : rec[REC_ILHAT];
      double ell[3], dv[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ell[c] = X[(XR + c) * XS + s + 1] - r[c];
        dv[c] = X[(XV + c) * XS + s + 1] - v[c];
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
        for (int c = 0; c < 3; ++c) sg[c] -= __ldg(p.sigma0 + c * p.ne + si.elem);
      }
      const double S1 = general ? gp(GP_S1) : rec[REC_S1];
      const double S3 = general ? gp(GP_S3) : rec[REC_S3];
      nb[0] = S1 * sg[0] * inv_e;
      nb[1] = S1 * sg[1] * inv_e;
      nb[2] = S3 * sg[2] * inv_e;
#pragma unroll
      for (int c = 0; c < 3; ++c) n[c] = fma(Q[c], nb[0], fma(Q[3 + c], nb[1], Q[6 + c] * nb[2]));  // Q^T nbar
    }
    // ---- A6 Voronoi i: curvature via inverse Rodrigues
    // (no branch: a slot without a Voronoi domain pairs its element with itself -- kappa = 0 -- and
    // its moment is masked below)
    double kap[3];
    {
      double Qp[9], cth, s2;
      const int sp = si.has_v ? s - 1 : s;  // (a long-rod segment's slot 0 reads its halo at -1)
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) {
        const double q = X[(XQ + c) * XS + sp];
        Qp[c] = si.has_v ? q : Q[c];
      }
      complete_d3(Qp);  // the bits the neighbour holds in its registers
      logrot_pair(Q, Qp, kap, cth, s2);
      if (si.has_v && cth < 0.0 && s2 <= 1e-12 * cth * cth) fbits |= 4u;  // ER_F_ANTIPODAL: theta >= pi - 1e-6
    }
    // ---- exchange B
    if (si.has_e) {
      X[XL * XS + s] = l;
#pragma unroll
      for (int c = 0; c < 3; ++c) X[(XN + c) * XS + s] = n[c];
    }
    xsync(1);

    // ---- A6 bending moment and its averaged cross term
    double mb[3] = {0.0, 0.0, 0.0}, be[3] = {0.0, 0.0, 0.0};
    {
      const double Dh = general ? gp(GP_DH) : rec[REC_LHAT];
      const double iDh = general ? 1.0 / Dh : rec[REC_ILHAT];
#pragma unroll
      for (int c = 0; c < 3; ++c) kap[c] *= iDh;
      const double D = 0.5 * (X[XL * XS + s - 1] + l);
      const double ieps = Dh * rcp_fast(D);
      const double ieps3 = ieps * ieps * ieps;
      double k0[3] = {k0s[0], k0s[1], k0s[2]};
      if (ACT && (si.fl & FL_ACT)) {
        const double sk = general ? gp(GP_SK) : i * rec[REC_LHAT];
        // A sin(2 pi (s/L - f t)) = A sinpi(2 (s/L - f t))
        const double arg = 2.0 * fma(sk, rec[REC_ACTIL], -rec[REC_ACTF] * t_half);
        const double act = rec[REC_ACTA] * sinpi(arg);
        // no dynamically indexed register array (it would live in local memory)
        k0[0] += p.act_comp == 0 ? act : 0.0;
        k0[1] += p.act_comp == 1 ? act : 0.0;
        k0[2] += p.act_comp == 2 ? act : 0.0;
      }
      const double B1 = general ? gp(GP_BV1) : rec[REC_B1];
      const double B2 = general ? gp(GP_BV2) : rec[REC_B2];
      const double B3 = general ? gp(GP_BV3) : rec[REC_B3];
      mb[0] = B1 * (kap[0] - k0[0]) * ieps3;
      mb[1] = B2 * (kap[1] - k0[1]) * ieps3;
      mb[2] = B3 * (kap[2] - k0[2]) * ieps3;
      be[0] = (kap[1] * mb[2] - kap[2] * mb[1]) * Dh;
      be[1] = (kap[2] * mb[0] - kap[0] * mb[2]) * Dh;
      be[2] = (kap[0] * mb[1] - kap[1] * mb[0]) * Dh;
      if (EXTRA && (si.fl & FL_MUS)) {
        // muscular couple pair (+tau_k on element k, -tau_k on element k-1) folded into the
        // exchanged moment: C_j += (mb - tau)_{j+1} - (mb - tau)_j; beta keeps the elastic mb
        const double *mu = p.musc + 4 * (int64_t)si.rod;
        const double sk = general ? gp(GP_SK) : i * rec[REC_LHAT];
        const double tau = __ldg(mu) * sinpi(fma(2.0, fma(t_half, __ldg(mu + 1), -sk * __ldg(mu + 2)), __ldg(mu + 3)));
        mb[0] -= p.musc_comp == 0 ? tau : 0.0;
        mb[1] -= p.musc_comp == 1 ? tau : 0.0;
        mb[2] -= p.musc_comp == 2 ? tau : 0.0;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {  // no Voronoi domain at the slot
        mb[c] = si.has_v ? mb[c] : 0.0;
        be[c] = si.has_v ? be[c] : 0.0;
      }
    }
    // ---- A7 + A9 node force, linear acceleration, kick
    if (si.active) {
      double F[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) F[c] = n[c] - (i >= 1 ? X[(XN + c) * XS + s - 1] : 0.0);
      if ((si.fl & FL_TIP) && i == ((si.fl & FL_CLAMP_MASK) == 2 ? 0 : N)) {
#pragma unroll
        for (int c = 0; c < 3; ++c) F[c] += rec[REC_TIPX + c];
      }
      if (CONTACT && fcon) {  // NEXT-4: rod-rod + half-space contact force on this node
#pragma unroll
        for (int c = 0; c < 3; ++c) F[c] += fcon[c];
      }
      if (EXTRA && p.fext) {  // user external force f of Eq. (1a)
#pragma unroll
        for (int c = 0; c < 3; ++c) F[c] += __ldg(p.fext + c * p.ng + si.node);
      }
      const double im = general ? gp(GP_IM) : rec[REC_IM] * ((i == 0 || i == N) ? 2.0 : 1.0);
      const double nu = rec[REC_NU];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double a = fma(F[c], im, fma(-nu, v[c], p.g[c]));
        v[c] = si.cl_node ? 0.0 : fma(h, a, v[c]);
      }
    }
    // ---- exchange C (aliases A; every A read happened before the B barrier)
    if (si.active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) { X[(XM + c) * XS + s] = mb[c]; X[(XB + c) * XS + s] = be[c]; }
    }
    xsync(2);

    // ---- A8 + A9 element couple, angular acceleration, kick
    if (si.has_e) {
      double C[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        C[c] = (X[(XM + c) * XS + s + 1] - mb[c]) + 0.5 * (X[(XB + c) * XS + s + 1] + be[c]);
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
        for (int c = 0; c < 3; ++c) m[c] = __ldg(p.mag + c * p.ne + si.elem);
        const double lh = general ? gp(GP_LHAT) : rec[REC_LHAT];
        C[0] += lh * (m[1] * Qb[2] - m[2] * Qb[1]);
        C[1] += lh * (m[2] * Qb[0] - m[0] * Qb[2]);
        C[2] += lh * (m[0] * Qb[1] - m[1] * Qb[0]);
      }
      if (EXTRA && p.cext) {  // user external couple c-bar of Eq. (1b)
#pragma unroll
        for (int c = 0; c < 3; ++c) C[c] += __ldg(p.cext + c * p.ne + si.elem);
      }
      const double nu = rec[REC_NU];
      const double rate = edot * inv_e - nu;
      const double eu[3] = {w[1] * w[2], w[2] * w[0], w[0] * w[1]};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double iJ = general ? gp(GP_IJ1 + c) : rec[REC_IJ1 + c];
        const double kJ = general ? gp(GP_KJ1 + c) : rec[REC_KJ1 + c];
        const double al = fma(e * iJ, C[c], fma(kJ, eu[c], rate * w[c]));
        w[c] = si.cl_elem ? 0.0 : fma(h, al, w[c]);
      }
    }
  }
  if (DRIFT2) {
    t = t_half + hh;
#pragma unroll
    for (int c = 0; c < 3; ++c) r[c] = fma(hr, v[c], r[c]);
    rotate_inplace(Q, hq * w[0], hq * w[1], hq * w[2], !final_step);  // (d3 of the last step is not stored)
  }
  if ((DRIFT1 || DRIFT2) && si.active) {
    // fault checks: non-finite state, overspeed.  r, v and w suffice: Q changes only through
    // rot(h w / 2) and enters v within the same step (sigma -> n -> F), so a non-finite Q
    // shows up in v or w before the step ends.
    const double acc = ((r[0] + r[1]) + (r[2] + v[0])) + ((v[1] + v[2]) + (w[0] + (w[1] + w[2])));
    if (!isfinite(acc)) fbits |= 1u;
    if (dot3(v, v) > rec[REC_VMAX2]) fbits |= 8u;
  }
}

// Stage geometry of the persistent kernel: per buffer the tile's state block (<= 18 or 21
// planes of <= BLOCK doubles; the exchange area of XPLANES x BLOCK reuses it), then the rod
// records (RMAX x ER_REC) and the tile's element offsets (RMAX + 4 int64).
template <int BLOCK, int FEAT, bool LONG = false>
struct Stage {
  static constexpr int NPL = 6 + ER_EPL + ((FEAT & FEAT_KAPPA0) ? 3 : 0);  // staged input planes
  static constexpr int RMAX = BLOCK / 8;
  static constexpr int XS = LONG ? BLOCK + 2 : BLOCK;  // exchange plane stride (long rods: halos)
  // the results of a tile are written at OUTOFF (clear of the exchange-C planes 0-5, which other
  // warps may still read) and bulk-stored from there
  static constexpr int OUTOFF = 6 * XS;
  static constexpr int NP0 = NPL > XPLANES ? NPL : XPLANES;
  static constexpr int PLANES = (NP0 > 6 + 6 + ER_EPL ? NP0 : 6 + 6 + ER_EPL) * XS + 8;
  static constexpr int RECOFF = PLANES;
  static constexpr int EOFF = RECOFF + RMAX * ER_REC;
  static constexpr int TOFF = EOFF + RMAX + 4;   // staged ErTile (16 doubles)
  static constexpr int BUFD = TOFF + 16;         // doubles per buffer (even)
  // two buffers and their load mbarriers
  static constexpr size_t bytes() { return (size_t)(2 * BUFD) * 8 + 2 * 8; }
};

// Thread 0 issues the bulk copies of tile `T` into stage buffer B: the tile's contiguous state
// block, its rod records and its element offsets -- three TMA 1-D bulk copies.
struct TileHead {  // the descriptor fields the issuing thread needs
  int64_t boff;
  int32_t r0, nr, nslots, nel, nvor;
};
__device__ __forceinline__ TileHead load_head(const ErTile *t) {
  TileHead h;
  h.boff = __ldg(&t->boff);
  const int4 v = __ldg(reinterpret_cast<const int4 *>(&t->r0));
  h.r0 = v.x; h.nr = v.y; h.nslots = v.z; h.nel = v.w;
  h.nvor = h.nel - (__ldg(&t->seg) == 0 ? h.nr : 0);  // see tile_nvor
  return h;
}

template <int BLOCK, int FEAT, bool LONG = false>
__device__ __forceinline__ void issue_tile(const ErStepParams &p, const TileHead &T, const ErTile *tile_ptr, double *B,
                                           uint64_t *bar) {
  using SG = Stage<BLOCK, FEAT, LONG>;
  const int64_t sz = 6 * (int64_t)T.nslots + ER_EPL * (int64_t)T.nel +
                     (((FEAT & FEAT_KAPPA0) && p.has_kappa0) ? 3 * (int64_t)T.nvor : 0);
  const uint32_t cs = (uint32_t)((sz + 1) & ~1ll);
  const int64_t ra = T.r0 & ~1ll;
  const uint32_t ceo = (uint32_t)(((T.r0 + T.nr + 2) & ~1ll) - ra);
  const uint32_t bytes = 8u * cs + (uint32_t)T.nr * ER_REC * 8u + 8u * ceo + (uint32_t)sizeof(ErTile);
  ER_CHECK(cs <= (uint32_t)SG::PLANES && T.nr <= SG::RMAX && ceo <= (uint32_t)SG::RMAX + 4);
  ER_CHECK(T.boff >= 0 && T.boff + cs <= p.state_doubles + 64);
  mbar_expect_tx(bar, bytes);
  bulk_g2s(B, p.state + T.boff, 8u * cs, bar);
  bulk_g2s(B + SG::RECOFF, p.rec + (int64_t)T.r0 * ER_REC, (uint32_t)T.nr * ER_REC * 8u, bar);
  bulk_g2s(B + SG::EOFF, p.eoff + ra, 8u * ceo, bar);
  bulk_g2s(B + SG::TOFF, tile_ptr, (uint32_t)sizeof(ErTile), bar);
}

template <int BLOCK, int MINB, int FEAT, bool DSTORE = false, bool SWEEP = false>
__global__ void __launch_bounds__(BLOCK, MINB) fused_persistent(const ErStepParams p) {
  using SG = Stage<BLOCK, FEAT>;
  extern __shared__ __align__(16) double sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 2 * SG::BUFD);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();  // (programmatic launch) the previous kernel's results are complete and visible
  const double t0 = launch_t0(p);
  uint32_t phase = 0;  // bit b = load parity of buffer b
  unsigned fbits_all = 0;
  int frod = 0x7fffffff;
  // Sweeps (p.sweeps > 1): the launch streams its tiles through the pipeline that many times, one
  // step (p.n_steps on-chip steps) per pass and the state through HBM every pass -- the work of
  // that many launches without their boundaries.  Between passes thread 0 lets this CTA's stores
  // land (and fences the odd-tail plain store against the async proxy) before reloading.
  // (a separate instantiation: the pass loop alone costs the one-pass kernel 2-5% -- DESIGN §4)
  const int sweeps = (SWEEP && !DSTORE && p.sweeps > 1) ? p.sweeps : 1;
  double t_pass = t0;
  for (int sw = 0; sw < sweeps; ++sw) {
  if (sw > 0) {
    if (tid == 0) fence_proxy_async_all();  // the pass's stores landed (wait at its end); the odd-tail plain store too
    for (int st = 0; st < p.n_steps; ++st) {  // step_body's own time arithmetic
      const double th = t_pass + 0.5 * p.h;
      t_pass = th + 0.5 * p.h;
    }
  }
  const bool last_pass = sw + 1 == sweeps;
  // every pass starts in buffer 0: every thread is past the previous pass's last epilogue barrier
  // and thread 0 has waited for its stores, so both buffers are free (mbarrier phases carry on)
  int64_t tile = blockIdx.x;
  if (tid == 0 && tile < p.n_tiles) issue_tile<BLOCK, FEAT>(p, load_head(p.tiles + tile), p.tiles + tile, sm, &bar[0]);
  // Pipeline per tile k in buffer b (the other buffer b^1 held tile k-1):
  //   wait load(k) -> stage to registers -> barrier -> [t0: once the bulk store of tile k-1 has
  //   read b^1, load tile k+1 into b^1] -> steps (exchange in b) -> barrier -> results to b ->
  //   barrier -> [t0: bulk store b -> HBM].  Loads and stores are TMA bulk copies, so no warp
  //   ever waits on HBM except for the (prefetched) load of its next tile.
  for (int k = 0; tile < p.n_tiles; tile += gridDim.x, ++k) {
    const int b = k & 1;
    double *B = sm + b * SG::BUFD;
    const int64_t tnext = tile + gridDim.x;
    TileHead Tn;
    if (tid == 0 && tnext < p.n_tiles) Tn = load_head(p.tiles + tnext);  // overlaps the wait
    if (last_pass && tnext >= p.n_tiles) griddep_launch_dependents();  // last tile: the next grid may launch
#if ER_TRACE  // measurement builds only (ER_NVCC_EXTRA=-DER_TRACE=1): the per-tile timeline
    unsigned long long *tr = (p.trace && tid == 0 && k < ER_TRACE_ITERS)
                                 ? p.trace + ((int64_t)blockIdx.x * ER_TRACE_ITERS + k) * 4 : nullptr;
#else
    constexpr unsigned long long *tr = nullptr;
#endif
    if (tr) tr[0] = (gtimer() & ((1ull << 48) - 1)) | ((unsigned long long)smid() << 56);
    mbar_wait(&bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    if (tr) tr[1] = gtimer() & ((1ull << 48) - 1);

    // ---- decode this thread's slot from the staged tile descriptor and element offsets
    const ErTile &T = *reinterpret_cast<const ErTile *>(B + SG::TOFF);
    const int64_t *eo = reinterpret_cast<const int64_t *>(B + SG::EOFF) + (T.r0 & 1);
    SlotInfo si;
    si.s = tid;
    si.active = tid < T.nslots;
    const int lo = T.pfx[tid >> 5] + __popc(T.smask[tid >> 5] & lanemask_le()) - 1;
    const int64_t e0 = eo[0];
    si.q = lo;
    si.rod = T.r0 + lo;
    const int st0 = (int)(eo[lo] - e0) + lo;
    si.i = tid - st0;
    si.N = (int)(eo[lo + 1] - eo[lo]);
    si.node = T.nbase + tid;
    si.elem = T.ebase + tid - lo;
    si.vor = si.elem - si.rod - 1;
    const double *rec = B + SG::RECOFF + lo * ER_REC;
    si.fl = si.active ? rec_flags(rec) : 0;
    finish_slot(si);

    // ---- stage -> registers (tile-local SoA planes)
    const int ns = T.nslots, nel = T.nel;
    const int le = tid - lo;
    ER_CHECK(6 * ns + (ER_EPL - 1) * nel + le < SG::BUFD && (!si.has_e || (le >= 0 && le < nel)));
    const int64_t boff = T.boff;
    double r[3], v[3], Q[9], w[3], k0s[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = B[c * ns + tid];
      v[c] = B[(3 + c) * ns + tid];
    }
    // a rod's last node owns no element: its w stays 0 (le would index past the element planes,
    // into stale stage contents that the non-finite check would otherwise see); its Q is loaded
    // unguarded (a neighbouring in-buffer value) because nothing reads it: rotations, kinematics
    // and stores are per element, and no slot reads Q from a rod's last node
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) Q[c] = B[6 * ns + c * nel + le];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = si.has_e ? B[6 * ns + (ER_QST + c) * nel + le] : 0.0;
    complete_d3(Q);
    if ((FEAT & FEAT_KAPPA0) && si.has_v) {
      const int nvor = tile_nvor(T);
#pragma unroll
      for (int c = 0; c < 3; ++c) k0s[c] = B[6 * ns + ER_EPL * nel + c * nvor + (tid - 2 * lo - 1)];
    }
    // contact mode: this node's contact force and build position, loaded now so their latency
    // hides behind the step's first phases
    double fcon[3] = {0.0, 0.0, 0.0}, rbld[3] = {0.0, 0.0, 0.0};
    if ((FEAT & FEAT_CONTACT) && p.cfc) contact_node_load(p, si, fcon);
    if ((FEAT & FEAT_CONTACT) && p.cnode) contact_build_pos(p, si, rbld);
    __syncthreads();  // stage planes consumed: they become this tile's exchange area
#ifdef ER_TRACE_FINE
    if (tr) tr[2] = gtimer() & ((1ull << 48) - 1);
#endif
    if (tid == 0 && tnext < p.n_tiles) {
      bulk_wait_read_all();  // the bulk store of tile k-1 has finished reading buffer b^1
      issue_tile<BLOCK, FEAT>(p, Tn, p.tiles + tnext, sm + (b ^ 1) * SG::BUFD, &bar[b ^ 1]);
    }
#ifdef ER_TRACE_FINE  // measurement: [2] = after the stage barrier, [3] = prefetch issued
    if (tr) tr[3] = gtimer() & ((1ull << 48) - 1);
#endif
    // ---- the steps
    double t = t_pass;
    unsigned fbits = 0;
    if (FEAT & FEAT_CONTACT) {
      // contact mode: the state arrives after drift-1 (contact forces were evaluated there);
      // kick + drift-2, then -- unless this is the call's last step -- the next step's drift-1
      // and the node records for the next contact evaluation
      step_body<BLOCK, FEAT, false, true, true>(p, B, rec, si, r, v, Q, w, k0s, t, fbits, p.cfc ? fcon : nullptr);
      if (p.cnode) {
        step_body<BLOCK, FEAT, true, false, false>(p, B, rec, si, r, v, Q, w, k0s, t, fbits);
        contact_emit(p, si, r, v, rbld);
      }
    } else {
      for (int st = 0; st < p.n_steps; ++st) {
        step_body<BLOCK, FEAT, true, true, true>(p, B, rec, si, r, v, Q, w, k0s, t, fbits, nullptr, CtaSync(),
                                                 st + 1 == p.n_steps);
        if (st + 1 < p.n_steps) __syncthreads();  // exchange C is re-used as A by the next step
      }
    }
    if (fbits) { fbits_all |= fbits; frod = min(frod, (int)rec[REC_CANON]); }  // canonical rod id
#ifndef ER_TRACE_FINE
    if (tr) tr[2] = gtimer() & ((1ull << 48) - 1);
#endif

    if (DSTORE) {  // ablation: results straight from registers to HBM (coalesced SoA planes)
      double *G = p.state + boff;
      if (si.active) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          __stcs(G + c * ns + tid, r[c]);
          __stcs(G + (3 + c) * ns + tid, v[c]);
        }
      }
      if (si.has_e) {
#pragma unroll
        for (int c = 0; c < ER_QST; ++c) __stcs(G + 6 * ns + c * nel + le, Q[c]);
#pragma unroll
        for (int c = 0; c < 3; ++c) __stcs(G + 6 * ns + (ER_QST + c) * nel + le, w[c]);
      }
#ifndef ER_TRACE_FINE
      if (tr) tr[3] = gtimer() & ((1ull << 48) - 1);
#endif
      continue;
    }
    // ---- registers -> stage (block layout at OUTOFF) -> HBM with one TMA bulk store
    double *O = B + SG::OUTOFF;
    if (si.active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        O[c * ns + tid] = r[c];
        O[(3 + c) * ns + tid] = v[c];
      }
    }
    if (si.has_e) {
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) O[6 * ns + c * nel + le] = Q[c];
#pragma unroll
      for (int c = 0; c < 3; ++c) O[6 * ns + (ER_QST + c) * nel + le] = w[c];
    }
    fence_proxy_async();  // this thread's generic smem writes -> visible to the async proxy
    __syncthreads();
    if (tid == 0) {
      // bulk copies move multiples of 16 bytes; with an odd element count the block's last
      // double (d1, d2, w planes: 9 nel doubles) goes with a plain store
      const uint32_t tot = (uint32_t)(6 * ns + ER_EPL * nel);
      ER_CHECK(boff + tot <= p.state_doubles && SG::OUTOFF + tot <= (uint32_t)SG::PLANES);
      bulk_s2g(p.state + boff, O, 8u * (tot & ~1u));
      bulk_commit();
      if (tot & 1u) p.state[boff + tot - 1] = O[tot - 1];
    }
#ifndef ER_TRACE_FINE
    if (tr) tr[3] = gtimer() & ((1ull << 48) - 1);
#endif
  }
  if (tid == 0) bulk_wait_all();  // stores complete before the kernel retires
  }  // passes
  advance_tdev(p, t0, sweeps);
  report_fault(p, fbits_all, frod);
}

// ------------------------------------------------------------------------------------------
// simple kernel: one tile per CTA, plain global loads; decode from the global tile table.
template <int BLOCK>
__device__ __forceinline__ void decode_global(const ErStepParams &p, const ErTile &T, SlotInfo &si, int *rst) {
  for (int q = threadIdx.x; q <= T.nr; q += BLOCK) rst[q] = (int)(p.eoff[T.r0 + q] - T.ebase) + q;
  __syncthreads();
  const int s = threadIdx.x;
  si.s = s;
  si.active = s < T.nslots;
  const int lo = T.pfx[s >> 5] + __popc(T.smask[s >> 5] & lanemask_le()) - 1;
  si.q = lo;
  si.rod = T.r0 + lo;
  si.i = s - rst[lo];
  si.N = rst[lo + 1] - rst[lo] - 1;
  si.node = T.nbase + s;
  si.elem = T.ebase + s - lo;
  si.vor = si.elem - si.rod - 1;
  si.fl = si.active ? rec_flags(p.rec + (int64_t)si.rod * ER_REC) : 0;
  finish_slot(si);
}

template <int BLOCK, int MINB, int MODE>
__global__ void __launch_bounds__(BLOCK, MINB) simple_kernel(const ErStepParams p) {
  constexpr int FEAT = FEAT_GENERAL | FEAT_KAPPA0 | FEAT_EXTRA | FEAT_CONTACT;
  extern __shared__ __align__(16) double sm[];
  int *rst = reinterpret_cast<int *>(sm + XPLANES * BLOCK);
  const ErTile T = p.tiles[blockIdx.x];
  SlotInfo si;
  decode_global<BLOCK>(p, T, si, rst);
  const double *rec = p.rec + (int64_t)si.rod * ER_REC;
  double r[3] = {0, 0, 0}, v[3] = {0, 0, 0}, Q[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, w[3] = {0, 0, 0};
  double k0s[3] = {0.0, 0.0, 0.0};
  double *G = p.state + T.boff;
  const int ns = T.nslots, nel = T.nel, s = threadIdx.x, le = s - si.q;
  if (si.active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = __ldcs(G + c * ns + s);
      v[c] = __ldcs(G + (3 + c) * ns + s);
    }
  }
  if (si.has_e) {
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) Q[c] = __ldcs(G + 6 * ns + c * nel + le);
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = __ldcs(G + 6 * ns + (ER_QST + c) * nel + le);
    complete_d3(Q);
  }
  if (p.has_kappa0 && si.has_v) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
      k0s[c] = __ldg(G + tile_vor_plane(T, c) + (T.nseg > 1 ? s - (T.seg == 0 ? 1 : 0) : s - 2 * si.q - 1));
  }
  double t = p.t;
  unsigned fbits = 0;
  const int nsteps = (MODE == MODE_FUSED) ? p.n_steps : 1;
  for (int st = 0; st < nsteps; ++st) {
    if (MODE == MODE_FUSED) step_body<BLOCK, FEAT, true, true, true>(p, sm, rec, si, r, v, Q, w, k0s, t, fbits);
    if (MODE == MODE_DRIFT) step_body<BLOCK, FEAT, true, false, false>(p, sm, rec, si, r, v, Q, w, k0s, t, fbits);
    if (MODE == MODE_DYN) {
      double fcon[3] = {0.0, 0.0, 0.0};
      if (p.cfc) contact_node_load(p, si, fcon);
      step_body<BLOCK, FEAT, false, true, false>(p, sm, rec, si, r, v, Q, w, k0s, t, fbits, p.cfc ? fcon : nullptr);
    }
    if (MODE == MODE_FUSED && st + 1 < nsteps) __syncthreads();
  }
  if (si.active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      __stcs(G + c * ns + s, r[c]);
      __stcs(G + (3 + c) * ns + s, v[c]);
    }
  }
  if (MODE == MODE_DRIFT && p.cnode) {
    double rb[3];
    contact_build_pos(p, si, rb);
    contact_emit(p, si, r, v, rb);
  }
  if (si.has_e) {
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) __stcs(G + 6 * ns + c * nel + le, Q[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c) __stcs(G + 6 * ns + (ER_QST + c) * nel + le, w[c]);
  }
  report_fault(p, fbits, si.active ? (int)rec[REC_CANON] : 0);  // canonical rod id
}

// ------------------------------------------------------------------------------------------
// Long rods (more than 511 elements): the rod's nseg segments of ER_LONG_SEG slots are the CTAs
// of one thread-block cluster.  The step is step_body with an exchange area that has a halo
// slot on each side; at every exchange barrier the boundary slots also write their values into
// the neighbouring segments' halos through distributed shared memory, then the whole cluster
// synchronises (barrier.cluster, release / acquire).  Plain coalesced loads / stores.
namespace cgx = cooperative_groups;

template <int BLOCK, int XS>
struct ClusterSync {
  double *X;  // this CTA's exchange area: plane c at X[c * XS + s], halos at s = -1 and s = BLOCK
  int s, nslots, seg, nseg;
  __device__ __forceinline__ void operator()(int phase) const {
    cgx::cluster_group cl = cgx::this_cluster();
    const int p0 = phase == 1 ? XL : 0, np = phase == 0 ? XL : phase == 1 ? 4 : 6;
    if (s == 0 && seg > 0) {  // my first slot -> the previous segment's right halo
      double *R = cl.map_shared_rank(X, seg - 1);
      for (int c = 0; c < np; ++c) R[(p0 + c) * XS + BLOCK] = X[(p0 + c) * XS];
    }
    if (s == nslots - 1 && seg < nseg - 1) {  // my last slot -> the next segment's left halo
      double *L = cl.map_shared_rank(X, seg + 1);
      for (int c = 0; c < np; ++c) L[(p0 + c) * XS - 1] = X[(p0 + c) * XS + s];
    }
    cl.sync();
  }
};

#ifndef ER_LONG_MINB
#define ER_LONG_MINB 2
#endif
template <int BLOCK, int FEAT>
__global__ void __launch_bounds__(BLOCK, BLOCK > 256 ? 1 : ER_LONG_MINB) long_kernel(const ErStepParams p, int64_t tile0) {
  constexpr int XS = BLOCK + 2;
  extern __shared__ __align__(16) double sm[];
  double *X = sm + 1;
  cgx::cluster_group cl = cgx::this_cluster();
  const ErTile T = p.tiles[tile0 + blockIdx.x];
  const int s = threadIdx.x;
  SlotInfo si;
  si.s = s;
  si.q = 0;
  si.rod = T.r0;
  si.N = (int)(p.eoff[T.r0 + 1] - p.eoff[T.r0]);
  si.i = T.seg * BLOCK + s;
  si.active = s < T.nslots;
  si.node = T.nbase + s;
  si.elem = T.ebase + s;
  si.vor = si.elem - si.rod - 1;
  const double *rec = p.rec + (int64_t)si.rod * ER_REC;
  si.fl = si.active ? rec_flags(rec) : 0;
  finish_slot(si);
  double r[3] = {0, 0, 0}, v[3] = {0, 0, 0}, Q[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, w[3] = {0, 0, 0};
  double k0s[3] = {0.0, 0.0, 0.0};
  double *G = p.state + T.boff;
  const int ns = T.nslots, nel = T.nel;
  if (si.active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = __ldcs(G + c * ns + s);
      v[c] = __ldcs(G + (3 + c) * ns + s);
    }
  }
  if (si.has_e) {
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) Q[c] = __ldcs(G + 6 * ns + c * nel + s);
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = __ldcs(G + 6 * ns + (ER_QST + c) * nel + s);
    complete_d3(Q);
  }
  if (p.has_kappa0 && si.has_v) {
#pragma unroll
    for (int c = 0; c < 3; ++c) k0s[c] = __ldg(G + tile_vor_plane(T, c) + (s - (T.seg == 0 ? 1 : 0)));
  }
  cl.sync();  // every segment of the cluster is resident before any distributed-smem access
  const ClusterSync<BLOCK, XS> xs{X, s, T.nslots, T.seg, T.nseg};
  const double t0 = launch_t0(p);
  double t = t0;
  unsigned fbits = 0;
  for (int st = 0; st < p.n_steps; ++st) {
    step_body<BLOCK, FEAT, true, true, true, XS, ClusterSync<BLOCK, XS>>(p, X, rec, si, r, v, Q, w, k0s, t, fbits,
                                                                        nullptr, xs);
    if (st + 1 < p.n_steps) cl.sync();  // the next step's exchange A re-uses these planes
  }
  if (si.active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      __stcs(G + c * ns + s, r[c]);
      __stcs(G + (3 + c) * ns + s, v[c]);
    }
  }
  if (si.has_e) {
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) __stcs(G + 6 * ns + c * nel + s, Q[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c) __stcs(G + 6 * ns + (ER_QST + c) * nel + s, w[c]);
  }
  report_fault(p, fbits, si.active ? (int)rec[REC_CANON] : 0);
  advance_tdev(p, t0);
  cl.sync();  // no CTA leaves while a neighbour may still access its shared memory
}

// Persistent long-rod kernel: clusters of K CTAs walk the group's rods (one segment tile per CTA)
// with the tile kernel's TMA double-buffered pipeline; a cluster barrier replaces the stage
// barrier (a neighbour's halo writes land in this CTA's stage area).
template <int BLOCK, int FEAT>
__global__ void __launch_bounds__(BLOCK, BLOCK > 256 ? 1 : 2) long_persistent(const ErStepParams p, int64_t tile0, int64_t n_rods) {
  using SG = Stage<BLOCK, FEAT, true>;
  constexpr int XS = SG::XS;
  extern __shared__ __align__(16) double sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 2 * SG::BUFD);
  cgx::cluster_group cl = cgx::this_cluster();
  const int tid = threadIdx.x;
  const int K = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int64_t ncl = gridDim.x / K;
  auto tile_of = [&](int64_t rr) { return tile0 + rr * K + rank; };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t rod = blockIdx.x / K;
  if (tid == 0 && rod < n_rods)
    issue_tile<BLOCK, FEAT, true>(p, load_head(p.tiles + tile_of(rod)), p.tiles + tile_of(rod), sm, &bar[0]);
  cl.sync();  // every CTA of the cluster resident before any distributed-smem access
  const double t0 = launch_t0(p);
  uint32_t phase = 0;
  unsigned fbits_all = 0;
  int frod = 0x7fffffff;
  for (int k = 0; rod < n_rods; rod += ncl, ++k) {
    const int b = k & 1;
    double *B = sm + b * SG::BUFD;
    const int64_t rnext = rod + ncl;
    TileHead Tn;
    if (tid == 0 && rnext < n_rods) Tn = load_head(p.tiles + tile_of(rnext));
    mbar_wait(&bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const ErTile &T = *reinterpret_cast<const ErTile *>(B + SG::TOFF);
    const int64_t *eo = reinterpret_cast<const int64_t *>(B + SG::EOFF) + (T.r0 & 1);
    const double *rec = B + SG::RECOFF;
    SlotInfo si;
    si.s = tid;
    si.q = 0;
    si.rod = T.r0;
    si.N = (int)(eo[1] - eo[0]);
    si.i = T.seg * BLOCK + tid;
    si.active = tid < T.nslots;
    si.node = T.nbase + tid;
    si.elem = T.ebase + tid;
    si.vor = si.elem - si.rod - 1;
    si.fl = si.active ? rec_flags(rec) : 0;
    finish_slot(si);
    const int ns = T.nslots, nel = T.nel, seg = T.seg, nseg = T.nseg;
    const int64_t boff = T.boff;
    double r[3], v[3], Q[9], w[3], k0s[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      r[c] = si.active ? B[c * ns + tid] : 0.0;
      v[c] = si.active ? B[(3 + c) * ns + tid] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < ER_QST; ++c) Q[c] = si.has_e ? B[6 * ns + c * nel + tid] : 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) w[c] = si.has_e ? B[6 * ns + (ER_QST + c) * nel + tid] : 0.0;
    complete_d3(Q);
    if ((FEAT & FEAT_KAPPA0) && p.has_kappa0 && si.has_v) {
      const int nvor = tile_nvor(T);
#pragma unroll
      for (int c = 0; c < 3; ++c) k0s[c] = B[6 * ns + ER_EPL * nel + c * nvor + (tid - (seg == 0 ? 1 : 0))];
    }
    double fcon[3] = {0.0, 0.0, 0.0}, rbld[3] = {0.0, 0.0, 0.0};  // contact mode, as in fused_persistent
    if ((FEAT & FEAT_CONTACT) && p.cfc) contact_node_load(p, si, fcon);
    if ((FEAT & FEAT_CONTACT) && p.cnode) contact_build_pos(p, si, rbld);
    cl.sync();  // all segments consumed their stage: exchange areas and halos are free
    if (tid == 0 && rnext < n_rods) {
      bulk_wait_read_all();  // the bulk store of the previous rod has read buffer b^1
      issue_tile<BLOCK, FEAT, true>(p, Tn, p.tiles + tile_of(rnext), sm + (b ^ 1) * SG::BUFD, &bar[b ^ 1]);
    }
    double *X = B + 1;
    const ClusterSync<BLOCK, XS> xs{X, tid, ns, seg, nseg};
    double t = t0;
    unsigned fbits = 0;
    if (FEAT & FEAT_CONTACT) {  // state after drift-1: kick + drift-2 [+ next drift-1 + node records]
      step_body<BLOCK, FEAT, false, true, true, XS, ClusterSync<BLOCK, XS>>(p, X, rec, si, r, v, Q, w, k0s, t, fbits,
                                                                           p.cfc ? fcon : nullptr, xs);
      if (p.cnode) {
        step_body<BLOCK, FEAT, true, false, false>(p, X, rec, si, r, v, Q, w, k0s, t, fbits);
        contact_emit(p, si, r, v, rbld);
      }
    } else {
      for (int st = 0; st < p.n_steps; ++st) {
        step_body<BLOCK, FEAT, true, true, true, XS, ClusterSync<BLOCK, XS>>(p, X, rec, si, r, v, Q, w, k0s, t, fbits,
                                                                            nullptr, xs);
        if (st + 1 < p.n_steps) cl.sync();
      }
    }
    if (fbits) { fbits_all |= fbits; frod = min(frod, (int)rec[REC_CANON]); }
    double *O = B + SG::OUTOFF;
    if (si.active) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        O[c * ns + tid] = r[c];
        O[(3 + c) * ns + tid] = v[c];
      }
    }
    if (si.has_e) {
#pragma unroll
      for (int c = 0; c < ER_QST; ++c) O[6 * ns + c * nel + tid] = Q[c];
#pragma unroll
      for (int c = 0; c < 3; ++c) O[6 * ns + (ER_QST + c) * nel + tid] = w[c];
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      // bulk copies move multiples of 16 bytes; with an odd element count the block's last
      // double (d1, d2, w planes: 9 nel doubles) goes with a plain store
      const uint32_t tot = (uint32_t)(6 * ns + ER_EPL * nel);
      ER_CHECK(boff + tot <= p.state_doubles && SG::OUTOFF + tot <= (uint32_t)SG::PLANES);
      bulk_s2g(p.state + boff, O, 8u * (tot & ~1u));
      bulk_commit();
      if (tot & 1u) p.state[boff + tot - 1] = O[tot - 1];
    }
  }
  if (tid == 0) bulk_wait_all();
  advance_tdev(p, t0);
  report_fault(p, fbits_all, frod);
  cl.sync();  // no CTA leaves while a neighbour may still access its shared memory
}

// --------------------------------------------------------------------------- diagnostics
// Per-tile partial sums of the energy functional at time p.t; deterministic.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) diag_kernel(const ErStepParams p) {
  extern __shared__ __align__(16) double sm[];
  double *xr = sm;
  double *xQ = xr + 3 * BLOCK;
  double *red = xQ + 9 * BLOCK;  // [16][BLOCK/32]
  int *rst = reinterpret_cast<int *>(red + 16 * (BLOCK / 32));
  double acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  // tiles tb = blockIdx.x, blockIdx.x + gridDim.x, ...: per-thread sums in a fixed order (deterministic)
  for (int64_t tb = blockIdx.x; tb < p.n_tiles; tb += gridDim.x) {
  const ErTile T = p.tiles[tb];
  SlotInfo si;
  decode_global<BLOCK>(p, T, si, rst);
  const int s = threadIdx.x;
  const int i = si.i, N = si.N;
  const bool general = (si.fl & FL_GENERAL) != 0;
  const double *rec = p.rec + (int64_t)si.rod * ER_REC;
  auto gp = [&](int plane) { return p.gpar[plane * p.ng + si.node]; };
  const double *G = p.state + T.boff;
  const int ns = T.nslots, nel = T.nel, le = s - si.q;
  double r[3] = {0, 0, 0}, v[3] = {0, 0, 0}, Q[9], w[3] = {0, 0, 0};
  for (int c = 0; c < 3; ++c) {
    if (si.active) { r[c] = G[c * ns + s]; v[c] = G[(3 + c) * ns + s]; }
    if (si.has_e) w[c] = G[6 * ns + (ER_QST + c) * nel + le];
  }
  for (int c = 0; c < ER_QST; ++c) Q[c] = si.has_e ? G[6 * ns + c * nel + le] : 0.0;
  complete_d3(Q);
  if (si.active) {
    for (int c = 0; c < 3; ++c) xr[c * BLOCK + s] = r[c];
    for (int c = 0; c < 9; ++c) xQ[c * BLOCK + s] = Q[c];
  }
  __syncthreads();
  if (si.active) {
    const double im = general ? gp(GP_IM) : rec[REC_IM] * ((i == 0 || i == N) ? 2.0 : 1.0);
    const double m = 1.0 / im;
    const double vv = dot3(v, v);
    acc[0] += 0.5 * m * vv;
    acc[4] += -m * (p.g[0] * r[0] + p.g[1] * r[1] + p.g[2] * r[2]);
    if ((si.fl & FL_TIP) && i == ((si.fl & FL_CLAMP_MASK) == 2 ? 0 : N))
      acc[5] += -(rec[REC_TIPX] * r[0] + rec[REC_TIPY] * r[1] + rec[REC_TIPZ] * r[2]);
    acc[6] += m * v[0]; acc[7] += m * v[1]; acc[8] += m * v[2];
    acc[9] = fmax(acc[9], sqrt(vv));
    acc[10] += m;
  }
  if (si.has_e) {
    const double lh = general ? gp(GP_LHAT) : rec[REC_LHAT];
    const double ilh = general ? gp(GP_ILHAT) : rec[REC_ILHAT];
    double ell[3];
    if (s + 1 == T.nslots && T.seg + 1 < T.nseg) {  // long rod: next node is slot 0 of the next segment
      const ErTile Tn = p.tiles[tb + 1];
      for (int c = 0; c < 3; ++c) ell[c] = p.state[Tn.boff + c * Tn.nslots] - r[c];
    } else {
      for (int c = 0; c < 3; ++c) ell[c] = xr[c * BLOCK + s + 1] - r[c];
    }
    const double l = sqrt(dot3(ell, ell));
    const double e = l * ilh;
    double sg[3] = {dot3(Q, ell) * ilh, dot3(Q + 3, ell) * ilh, dot3(Q + 6, ell) * ilh - 1.0};
    if (p.sigma0) for (int c = 0; c < 3; ++c) sg[c] -= p.sigma0[c * p.ne + si.elem];
    const double S1 = general ? gp(GP_S1) : rec[REC_S1];
    const double S3 = general ? gp(GP_S3) : rec[REC_S3];
    acc[2] += 0.5 * (S1 * sg[0] * sg[0] + S1 * sg[1] * sg[1] + S3 * sg[2] * sg[2]) * lh;
    for (int c = 0; c < 3; ++c) {
      const double iJ = general ? gp(GP_IJ1 + c) : rec[REC_IJ1 + c];
      acc[1] += 0.5 * w[c] * w[c] / (iJ * e);
    }
    acc[11] += 1.0;
  }
  if (si.has_v) {
    double Qp[9], kap[3], cth, s2;
    if (s == 0) {  // long rod segment: previous element is the last of the previous segment
      const ErTile Tp = p.tiles[tb - 1];
      for (int c = 0; c < ER_QST; ++c) Qp[c] = p.state[Tp.boff + 6 * Tp.nslots + c * Tp.nel + Tp.nel - 1];
      complete_d3(Qp);
    } else {
      for (int c = 0; c < 9; ++c) Qp[c] = xQ[c * BLOCK + s - 1];
    }
    logrot_pair(Q, Qp, kap, cth, s2);
    const double Dh = general ? gp(GP_DH) : rec[REC_LHAT];
    double k0[3] = {0, 0, 0};
    const int lv = T.nseg > 1 ? s - (T.seg == 0 ? 1 : 0) : s - 2 * si.q - 1;  // local Voronoi index
    if (p.has_kappa0) for (int c = 0; c < 3; ++c) k0[c] = G[tile_vor_plane(T, c) + lv];
    if (si.fl & FL_ACT) {
      const double sk = general ? gp(GP_SK) : i * rec[REC_LHAT];
      const double act = rec[REC_ACTA] * sinpi(2.0 * (sk * rec[REC_ACTIL] - rec[REC_ACTF] * p.t));
      k0[0] += p.act_comp == 0 ? act : 0.0;
      k0[1] += p.act_comp == 1 ? act : 0.0;
      k0[2] += p.act_comp == 2 ? act : 0.0;
    }
    for (int c = 0; c < 3; ++c) {
      const double Bv = general ? gp(GP_BV1 + c) : rec[REC_B1 + c];
      const double d = kap[c] / Dh - k0[c];
      acc[3] += 0.5 * Bv * d * d * Dh;
    }
  }
  __syncthreads();  // the exchange arrays and rod starts are refilled for the next tile
  }
  // deterministic block reduction: warp shuffles, then warp partials in fixed order
  const int s = threadIdx.x;
  const int lane = s & 31, wid = s >> 5;
  for (int k = 0; k < 12; ++k) {
    double x = acc[k];
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_down_sync(0xffffffffu, x, o);
      x = (k == 9) ? fmax(x, y) : x + y;
    }
    if (lane == 0) red[k * (BLOCK / 32) + wid] = x;
  }
  __syncthreads();
  if (s < 12) {
    double x = 0.0;
    for (int q = 0; q < BLOCK / 32; ++q) {
      const double y = red[s * (BLOCK / 32) + q];
      x = (s == 9) ? fmax(x, y) : x + y;
    }
    p.diag_partial[(int64_t)blockIdx.x * 16 + s] = x;
  }
}

__global__ void diag_finish_kernel(const double *partial, int64_t n_tiles, double *out) {
  // one warp per diagnostic: fixed-order strided sums, then a fixed shuffle tree
  const int k = blockIdx.x;
  double x = 0.0;
  for (int64_t q = threadIdx.x; q < n_tiles; q += 32) {
    const double y = partial[q * 16 + k];
    x = (k == 9) ? fmax(x, y) : x + y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_down_sync(0xffffffffu, x, o);
    x = (k == 9) ? fmax(x, y) : x + y;
  }
  if (threadIdx.x == 0) out[k] = x;
}

// --------------------------------------------------------------------------- layout helpers
// AoS [n][k] (canonical) <-> k SoA planes of stride `stride`
__global__ void aos_to_soa(const double *__restrict__ src, double *__restrict__ dst, int64_t n, int k,
                           int64_t stride) {
  const int64_t total = n * k;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = q / k;
    const int c = (int)(q - e * k);
    dst[c * stride + e] = src[q];
  }
}
// Canonical AoS [rows][3] -> 3 planes in packed rod order (user external loads): one warp per
// packed rod, lanes stride over the rod's contiguous canonical rows (coalesced reads).
// nodes = 1: node rows (N_r + 1 per rod, offset eoff + rod); 0: element rows.
__global__ void pack_planes(const double *__restrict__ src, double *__restrict__ dst, int64_t stride,
                            const int64_t *__restrict__ eoffp, const int32_t *__restrict__ ord,
                            const int64_t *__restrict__ eoffc, int64_t n_rods, int nodes) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pr = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; pr < n_rods; pr += nw) {
    const int64_t r = ord[pr];
    const int64_t c0 = eoffc[r] + (nodes ? r : 0), p0 = eoffp[pr] + (nodes ? pr : 0);
    const int64_t cnt = 3 * (eoffc[r + 1] - eoffc[r] + nodes);
    ER_CHECK(p0 + cnt / 3 <= stride);
    for (int64_t q = lane; q < cnt; q += 32) {
      const int64_t row = q / 3;
      dst[(q - 3 * row) * stride + p0 + row] = src[3 * c0 + q];
    }
  }
}
// Canonical AoS [rows][k] <-> tile-blocked planes, one CTA per tile, rod by rod: the rods of a tile
// are consecutive in packed order, and each rod's rows are contiguous in the canonical array (at
// its canonical offset).  canon == nullptr with to_tiles writes zeros.
//
// Directors: the canonical rows hold all 9 components; the tiles store d1, d2 (er_layout.h), so
// to_tiles drops d3 and the way back rebuilds it with complete_d3, the bits every kernel uses.
__global__ void canon_tiles(const ErStepParams p, double *canon, int field, int to_tiles) {
  // one warp per tile (warp-sized tiles of the warp kernel are small)
  const int64_t tix = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tix >= p.n_tiles) return;
  const int lane = threadIdx.x & 31;
  const ErTile T = p.tiles[tix];
  const int k = field == FIELD_DIR ? 9 : 3;
  int64_t count, off;
  int shift;  // rows per rod = N + shift
  if (field <= FIELD_VEL) {
    count = T.nslots; off = tile_node_plane(T, field == FIELD_VEL ? 3 : 0); shift = 1;
  } else if (field <= FIELD_OMEGA) {
    count = T.nel; off = tile_elem_plane(T, field == FIELD_OMEGA ? ER_QST : 0); shift = 0;
  } else {
    count = tile_nvor(T); off = tile_vor_plane(T, 0); shift = -1;
  }
  double *blk = p.state + T.boff + off;
  ER_CHECK(T.boff + off + (int64_t)(field == FIELD_DIR ? ER_QST : 3) * count <= p.state_doubles);
  for (int q = 0; q < T.nr; ++q) {
    const int64_t pr = T.r0 + q, cr = p.ord[pr];
    int64_t n = p.eoff[pr + 1] - p.eoff[pr] + shift;                           // rows of this rod
    int64_t loc = p.eoff[pr] - T.ebase + (int64_t)q * shift;                  // first row in the tile
    int64_t can = p.eoffc[cr] + cr * shift;                                    // first canonical row
    if (T.nseg > 1) {  // long rod: this segment's rows only
      const int64_t k0 = (int64_t)T.seg * ER_LONG_SEG;
      n = count;
      loc = 0;
      can += shift < 0 ? (T.seg == 0 ? 0 : k0 - 1) : k0;
    }
    if (field == FIELD_DIR) {  // consecutive threads on consecutive canonical doubles (coalesced)
      for (int64_t x = lane; x < n * 9; x += 32) {
        const int64_t u = x / 9;
        const int c = (int)(x - u * 9);
        const double *q = blk + loc + u;  // this element's stored components, plane stride count
        if (to_tiles) {
          if (c < ER_QST) blk[c * count + loc + u] = canon ? canon[can * 9 + x] : 0.0;
        } else {
          canon[can * 9 + x] = c < ER_QST ? q[c * count] : d3_component(c - ER_QST, q, count);
        }
      }
      continue;
    }
    for (int64_t x = lane; x < n * k; x += 32) {
      const int64_t u = x / k;
      const int c = (int)(x - u * k);
      if (to_tiles) blk[c * count + loc + u] = canon ? canon[can * k + x] : 0.0;
      else canon[can * k + x] = blk[c * count + loc + u];
    }
  }
}

// Validation of an uploaded canonical AoS array: out[2] += non-finite rows; for directors
// (orth) out[0] = max |Q Q^T - I|, out[1] = max |det Q - 1|.
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}
__global__ void validate_aos(const double *a, int64_t n, int k, int orth, double *out) {
  double m_orth = 0.0, m_det = 0.0, bad = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const double *x = a + q * k;
    bool fin = true;
    for (int c = 0; c < k; ++c) fin = fin && isfinite(x[c]);
    if (!fin) { bad += 1.0; continue; }
    if (orth) {
      for (int u = 0; u < 3; ++u)
        for (int w = 0; w < 3; ++w) m_orth = fmax(m_orth, fabs(dot3(x + 3 * u, x + 3 * w) - (u == w ? 1.0 : 0.0)));
      const double det = x[0] * (x[4] * x[8] - x[5] * x[7]) - x[1] * (x[3] * x[8] - x[5] * x[6]) +
                         x[2] * (x[3] * x[7] - x[4] * x[6]);
      m_det = fmax(m_det, fabs(det - 1.0));
    }
  }
  if (orth) {
    atomic_max_nonneg(out + 0, m_orth);
    atomic_max_nonneg(out + 1, m_det);
  }
  if (bad > 0.0) atomicAdd(out + 2, bad);
}

// er_set_bc / er_set_forcing: write the flag word and (forcing) damping, tip force and actuation
// fields of every rod record from the caller's per-rod arrays.
__global__ void apply_forcing(double *rec, int64_t n_rods, const int32_t *flags, const double *damping,
                              double damping_all, const double *tip, const double *actA, const double *actF,
                              const double *actL, int forcing) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rods; r += (int64_t)gridDim.x * blockDim.x) {
    double *x = rec + r * ER_REC;
    x[REC_FLAGS] = __longlong_as_double((long long)flags[r]);
    if (!forcing) continue;
    x[REC_NU] = damping ? damping[r] : damping_all;
    for (int c = 0; c < 3; ++c) x[REC_TIPX + c] = tip ? tip[3 * r + c] : 0.0;
    x[REC_ACTA] = actA ? actA[r] : 0.0;
    x[REC_ACTF] = actA ? actF[r] : 0.0;
    x[REC_ACTIL] = actA ? 1.0 / actL[r] : 0.0;
  }
}

// Shared-material records (er_layout.h ER_WREC): the compact record of every rod, and whether any
// rod's material constants (REC_LHAT..REC_VMAX2, REC_ACTIL) differ bitwise from rod 0's.
__global__ void compact_records(const double *rec, int64_t n_rods, double *wrec, int *differ) {
  bool d = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rods; r += (int64_t)gridDim.x * blockDim.x) {
    const double *x = rec + r * ER_REC;
    double *y = wrec + r * ER_WREC;
    for (int c = 0; c < 3; ++c) y[WREC_TIPX + c] = x[REC_TIPX + c];
    y[WREC_ACTA] = x[REC_ACTA];
    y[WREC_ACTF] = x[REC_ACTF];
    const long long fl = __double_as_longlong(x[REC_FLAGS]) & 0xffffffffll;
    const long long cn = (long long)x[REC_CANON];
    y[WREC_FC] = __longlong_as_double(fl | (cn << 32));
    for (int k = 0; k <= REC_VMAX2; ++k) d |= __double_as_longlong(x[k]) != __double_as_longlong(rec[k]);
    d |= __double_as_longlong(x[REC_ACTIL]) != __double_as_longlong(rec[REC_ACTIL]);
  }
  if (d) atomicOr(differ, 1);
}

}  // namespace er

// --------------------------------------------------------------------------- launch wrappers
namespace {

size_t simple_smem(int block) { return (size_t)er::XPLANES * 8 * block + sizeof(int) * (block / 8 + 4); }
size_t diag_smem(int block) { return (size_t)12 * 8 * block + 16 * 8 * (block / 32) + sizeof(int) * (block / 8 + 4); }

template <int BLOCK, int MINB, int FEAT, bool DSTORE = false, bool SWEEP = false>
cudaError_t launch_persistent(const ErStepParams &p, cudaStream_t st) {
  auto k = er::fused_persistent<BLOCK, MINB, FEAT, DSTORE, SWEEP>;
#ifdef ER_ONE_CTA_PER_SM  // measurement: request enough smem that only one CTA fits per SM
  const size_t sm = 160 * 1024;
#else
  const size_t sm = er::Stage<BLOCK, FEAT>::bytes();
#endif
  static int grid_per_sm[64] = {0};  // per device (and instantiation)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (grid_per_sm[dev] == 0) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, BLOCK, sm);
    if (e != cudaSuccess) return e;
    grid_per_sm[dev] = per_sm > 0 ? per_sm : 1;
  }
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = std::min<int64_t>(p.n_tiles, (int64_t)n_sm * grid_per_sm[dev]);
  // programmatic dependent launch: this grid's CTAs may start (and set up their stage barriers)
  // while the previous kernel on the stream drains; they read no global memory before
  // griddepcontrol.wait (which waits for the previous grids to complete and flush)
  static const bool pdl = std::getenv("ER_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g, 1, 1);
  cfg.blockDim = dim3(BLOCK, 1, 1);
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

// feat: GENERAL | KAPPA0 | CONTACT bits, plus at most one of FEAT_EXTRA / FEAT_ACT (24 kernels)
template <int BLOCK, int MINB, int X>
cudaError_t launch_persistent_base(const ErStepParams &p, int base, cudaStream_t st) {
  switch (base) {
    case 0: return p.sweeps > 1 ? launch_persistent<BLOCK, MINB, X | 0, false, true>(p, st) : launch_persistent<BLOCK, MINB, X | 0>(p, st);
    case 1: return p.sweeps > 1 ? launch_persistent<BLOCK, MINB, X | 1, false, true>(p, st) : launch_persistent<BLOCK, MINB, X | 1>(p, st);
    case 2: return p.sweeps > 1 ? launch_persistent<BLOCK, MINB, X | 2, false, true>(p, st) : launch_persistent<BLOCK, MINB, X | 2>(p, st);
    case 3: return p.sweeps > 1 ? launch_persistent<BLOCK, MINB, X | 3, false, true>(p, st) : launch_persistent<BLOCK, MINB, X | 3>(p, st);
    case 8: return launch_persistent<BLOCK, MINB, X | 8>(p, st);
    case 9: return launch_persistent<BLOCK, MINB, X | 9>(p, st);
    case 10: return launch_persistent<BLOCK, MINB, X | 10>(p, st);
    default: return launch_persistent<BLOCK, MINB, X | 11>(p, st);
  }
}
template <int BLOCK, int MINB>
cudaError_t launch_persistent_feat(const ErStepParams &p, int feat, cudaStream_t st) {
  const int base = feat & (FEAT_GENERAL | FEAT_KAPPA0 | FEAT_CONTACT);
  if (feat & FEAT_EXTRA) return launch_persistent_base<BLOCK, MINB, FEAT_EXTRA>(p, base, st);
  if (feat & FEAT_ACT) return launch_persistent_base<BLOCK, MINB, FEAT_ACT>(p, base, st);
  return launch_persistent_base<BLOCK, MINB, 0>(p, base, st);
}

template <int BLOCK, int MINB, int MODE>
cudaError_t launch_simple(const ErStepParams &p, cudaStream_t st) {
  auto k = er::simple_kernel<BLOCK, MINB, MODE>;
  const size_t sm = simple_smem(BLOCK);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)p.n_tiles, BLOCK, sm, st>>>(p);
  return cudaGetLastError();
}

template <int FEAT>
cudaError_t launch_long_persistent(const ErStepParams *p, int64_t tile0, int64_t n_rods, int nseg, cudaStream_t st) {
  constexpr int B = ER_LONG_SEG;
  auto k = er::long_persistent<B, FEAT>;
  const size_t sm = er::Stage<B, FEAT, true>::bytes();
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e == cudaSuccess && nseg > 8) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(B, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)nseg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)nseg, 1, 1);
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
  if (e != cudaSuccess) return e;
  if (std::getenv("ER_DEBUG_LONG"))
    fprintf(stderr, "[long_persistent] nseg %d: %d clusters resident (%d CTAs), %lld rods\n", nseg, ncl, ncl * nseg,
            (long long)n_rods);
  ncl = (int)std::max<int64_t>(1, std::min<int64_t>(n_rods, ncl));
  cfg.gridDim = dim3((unsigned)(ncl * nseg), 1, 1);
  e = cudaLaunchKernelEx(&cfg, k, *p, tile0, n_rods);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

extern "C" {

// kind: 0 persistent fused (production), 1 simple drift stage, 2 simple dynamics stage,
//       3 simple fused (one tile per CTA; ablation)
cudaError_t er_launch_warp(const ErStepParams *p, int feat, cudaStream_t st);  // er_warp.cu

cudaError_t er_launch_step(const ErStepParams *p, int block, int kind, int feat, cudaStream_t st) {
  if (p->n_tiles <= 0) return cudaSuccess;
  // equal-length short rods: the warp-local kernel (one pass per launch, no contact)
  if (kind == 0 && p->wN > 0 && p->sweeps <= 1 && !(feat & FEAT_CONTACT)) return er_launch_warp(p, feat, st);
  if (block == 128) {
    if (kind == 0 || kind == 5) return launch_persistent_feat<128, 4>(*p, feat, st);
    if (kind == 1) return launch_simple<128, 4, er::MODE_DRIFT>(*p, st);
    if (kind == 2) return launch_simple<128, 4, er::MODE_DYN>(*p, st);
    return launch_simple<128, 4, er::MODE_FUSED>(*p, st);
  }
  if (block == 256) {
    if (kind == 0) return launch_persistent_feat<256, 2>(*p, feat, st);
    if (kind == 5 && feat == 0) return launch_persistent<256, 2, 0, true>(*p, st);  // ablation
    if (kind == 5) return launch_persistent_feat<256, 2>(*p, feat, st);
    if (kind == 1) return launch_simple<256, 2, er::MODE_DRIFT>(*p, st);
    if (kind == 2) return launch_simple<256, 2, er::MODE_DYN>(*p, st);
    return launch_simple<256, 2, er::MODE_FUSED>(*p, st);
  }
  if (kind == 0 || kind == 5) return launch_persistent_feat<512, 1>(*p, feat, st);
  if (kind == 1) return launch_simple<512, 1, er::MODE_DRIFT>(*p, st);
  if (kind == 2) return launch_simple<512, 1, er::MODE_DYN>(*p, st);
  return launch_simple<512, 1, er::MODE_FUSED>(*p, st);
}

// Long rods: `n_rods` rods of `nseg` segments each, tiles [tile0, tile0 + n_rods * nseg), one
// cluster of nseg CTAs per rod.
cudaError_t er_launch_long(const ErStepParams *p, int64_t tile0, int64_t n_rods, int nseg, int feat, cudaStream_t st) {
  if (n_rods <= 0) return cudaSuccess;
  constexpr int ALL = FEAT_GENERAL | FEAT_KAPPA0 | FEAT_EXTRA;
  if (feat & FEAT_CONTACT)  // contact mode: always the persistent kernel
    return (feat & ~FEAT_CONTACT) == 0 ? launch_long_persistent<FEAT_CONTACT>(p, tile0, n_rods, nseg, st)
                                       : launch_long_persistent<ALL | FEAT_CONTACT>(p, tile0, n_rods, nseg, st);
  if (!std::getenv("ER_LONG_SIMPLE"))  // persistent, TMA-pipelined clusters (default)
    return feat == 0 ? launch_long_persistent<0>(p, tile0, n_rods, nseg, st)
                     : launch_long_persistent<ALL>(p, tile0, n_rods, nseg, st);
  constexpr int B = ER_LONG_SEG;
  // plain rods get the lean instantiation; any feature takes the general one
  auto k = feat == 0 ? er::long_kernel<B, 0> : er::long_kernel<B, FEAT_GENERAL | FEAT_KAPPA0 | FEAT_EXTRA>;
  const size_t sm = (size_t)er::XPLANES * (B + 2) * 8 + 16;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e == cudaSuccess && nseg > 8) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_rods * nseg), 1, 1);
  cfg.blockDim = dim3(B, 1, 1);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)nseg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, k, *p, tile0);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t er_launch_diag(const ErStepParams *p, int block, double *out, cudaStream_t st) {
  // a grid of at most 148 x 8 CTAs walks the tiles (partials per CTA, summed in a fixed order)
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p->n_tiles, 148 * 8));
  if (p->n_tiles > 0) {
    const size_t sm = diag_smem(block);
    auto go = [&](auto kern, int b) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<(unsigned)grid, b, sm, st>>>(*p);
    };
    if (block == 64) go(er::diag_kernel<64>, 64);
    else if (block == 128) go(er::diag_kernel<128>, 128);
    else if (block == 256) go(er::diag_kernel<256>, 256);
    else go(er::diag_kernel<512>, 512);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  er::diag_finish_kernel<<<12, 32, 0, st>>>(p->diag_partial, p->n_tiles > 0 ? grid : 0, out);
  return cudaGetLastError();
}

cudaError_t er_launch_aos_to_soa(const double *src, double *dst, int64_t n, int k, int64_t stride, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  er::aos_to_soa<<<148 * 8, 256, 0, st>>>(src, dst, n, k, stride);
  return cudaGetLastError();
}
cudaError_t er_launch_pack_planes(const double *src, double *dst, int64_t stride, const int64_t *eoffp,
                                  const int32_t *ord, const int64_t *eoffc, int64_t n_rods, int nodes, cudaStream_t st) {
  if (n_rods <= 0) return cudaSuccess;
  er::pack_planes<<<148 * 8, 256, 0, st>>>(src, dst, stride, eoffp, ord, eoffc, n_rods, nodes);
  return cudaGetLastError();
}
cudaError_t er_launch_canon_tiles(const ErStepParams *p, double *canon, int field, int to_tiles, cudaStream_t st) {
  if (p->n_tiles <= 0) return cudaSuccess;
  er::canon_tiles<<<(unsigned)((p->n_tiles + 7) / 8), 256, 0, st>>>(*p, canon, field, to_tiles);
  return cudaGetLastError();
}
cudaError_t er_launch_apply_forcing(double *rec, int64_t n_rods, const int32_t *flags, const double *damping,
                                    double damping_all, const double *tip, const double *actA, const double *actF,
                                    const double *actL, int forcing, cudaStream_t st) {
  if (n_rods <= 0) return cudaSuccess;
  er::apply_forcing<<<148 * 4, 256, 0, st>>>(rec, n_rods, flags, damping, damping_all, tip, actA, actF, actL, forcing);
  return cudaGetLastError();
}
cudaError_t er_launch_compact_records(const double *rec, int64_t n_rods, double *wrec, int *differ, cudaStream_t st) {
  if (n_rods <= 0) return cudaSuccess;
  er::compact_records<<<148 * 4, 256, 0, st>>>(rec, n_rods, wrec, differ);
  return cudaGetLastError();
}
cudaError_t er_launch_validate(const double *aos, int64_t n, int k, int orth, double *out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  er::validate_aos<<<148 * 4, 256, 0, st>>>(aos, n, k, orth, out);
  return cudaGetLastError();
}

}  // extern "C"
