// er_kernels.cu -- the hot path (L2): one fused single-pass Cosserat rod step per launch
// (or k steps per launch with the rod tile kept on chip), plus the staged ablation kernels,
// the diagnostics reduction and layout/validation helpers.  sm_100a, fp64, no tensor cores
// (nothing here is a dense contraction).
//
// Mapping: one CTA per rod-aligned tile of <= BLOCK "slots"; slot s of a rod is
// node i, element i (i < N) and Voronoi domain i (1 <= i < N) of that rod, one thread per slot.
// Neighbour data (node i+1, element i-1, n_{i-1}, mbar_{i+1}, beta_{i+1}) are exchanged through
// shared memory; rods never straddle tiles, so there are no halos in HBM and no grid barrier:
// the paper's asynchronous protocol is free here.
//
// One step of one slot:
//   A1-A3  r += h/2 v; Q <- rot(h/2 w) Q; clamped entries are not moved
//   A4-A5  l = r_{i+1} - r_i, e, de/dt, sigma = Q l / lhat - e3, nbar = S (sigma - sigma0)/e, n = Q^T nbar
//   A6     kappa = logrot(Q_k Q_{k-1}^T)/Dh, mbar = Bv (kappa - kappa0(t+h/2))/eps^3, beta = (kappa x mbar) Dh
//   A7,A9  a = (n_i - n_{i-1} + F_tip)/m + g - nu v;   v += h a
//   A8,A9  C = mbar_{i+1} - mbar_i + (beta_{i+1} + beta_i)/2 + (Q l) x nbar + c_mag
//          alpha = e J^-1 C + Euler((J w) x w) / J + w de/dt / e - nu w;   w += h alpha
//   A10    r += h/2 v; Q <- rot(h/2 w) Q
// (Q l) x nbar == lhat (Q t) x S(sigma - sigma0) and the two rate terms are Eq. (1b)'s
// (J w / e) x w and (J w / e^2) de/dt multiplied by e/J; see DESIGN.md §4 for the algebra.
#include <cuda_runtime.h>
#include <stdint.h>

#include "er_layout.h"
#include "er_math.cuh"

namespace er {

enum { MODE_FUSED = 0, MODE_DRIFT = 1, MODE_DYN = 2 };

// per-slot index bookkeeping shared by all kernels
struct Slot {
  int64_t node, elem, vor;
  int32_t rod, i, N, fl;
  bool active, has_e, has_v;
};

// Decode this thread's slot from the tile table.  rstart must hold BLOCK/2 + 2 ints.
template <int BLOCK>
__device__ __forceinline__ Slot decode_slot(const ErStepParams &p, int tile, int *rstart) {
  const int r0 = p.tiles[tile], r1 = p.tiles[tile + 1];
  const int nr = r1 - r0;
  const int64_t nbase = p.eoff[r0] + r0;
  for (int q = threadIdx.x; q <= nr; q += BLOCK) rstart[q] = (int)(p.eoff[r0 + q] + (r0 + q) - nbase);
  __syncthreads();
  Slot sl;
  const int s = threadIdx.x;
  const int nslots = rstart[nr];
  sl.active = s < nslots;
  int lo = 0, hi = nr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rstart[mid] <= s) lo = mid; else hi = mid - 1;
  }
  sl.rod = r0 + lo;
  sl.i = s - rstart[lo];
  sl.N = rstart[lo + 1] - rstart[lo] - 1;
  sl.node = nbase + s;
  sl.elem = sl.node - sl.rod;
  sl.vor = sl.elem - sl.rod - 1;
  sl.has_e = sl.active && sl.i < sl.N;
  sl.has_v = sl.active && sl.i >= 1 && sl.i < sl.N;
  sl.fl = sl.active ? __ldg(p.flags + sl.rod) : 0;
  return sl;
}

__device__ __forceinline__ void report_fault(const ErStepParams &p, unsigned bits, int rod) {
  const unsigned mask = __ballot_sync(0xffffffffu, bits != 0);
  if (mask == 0) return;
  if (bits) {
    atomicOr(p.fault, (unsigned long long)bits);
    atomicMin(p.fault + 1, (unsigned long long)rod);
  }
}

// The fused step.  MODE_FUSED: p.n_steps full steps per launch with the tile held in
// registers/shared memory; MODE_DRIFT: one drift(h/2) stage; MODE_DYN: one kick stage.
template <int BLOCK, int MINB, int MODE>
__global__ void __launch_bounds__(BLOCK, MINB) step_kernel(const ErStepParams p) {
  extern __shared__ double smem[];
  double *xr = smem;               // exchange A: r (3), v (3), Q (9)
  double *xv = xr + 3 * BLOCK;
  double *xQ = xv + 3 * BLOCK;
  double *xl = xQ + 9 * BLOCK;     // exchange B: l (1), n (3)
  double *xn = xl + BLOCK;
  double *xm = smem;               // exchange C (aliases A): mbar (3), beta (3)
  double *xb = smem + 3 * BLOCK;
  int *rstart = reinterpret_cast<int *>(xn + 3 * BLOCK);

  const Slot sl = decode_slot<BLOCK>(p, blockIdx.x, rstart);
  const int s = threadIdx.x;
  const int i = sl.i, N = sl.N;
  const int clamp = sl.fl & FL_CLAMP_MASK;
  const bool cl_node = sl.active && ((clamp == 1 && i == 0) || (clamp == 2 && i == N));
  const bool cl_elem = sl.has_e && ((clamp == 1 && i == 0) || (clamp == 2 && i == N - 1));
  const bool general = (sl.fl & FL_GENERAL) != 0;
  const double *rec = p.rec + (int64_t)sl.rod * ER_REC;

  // ---- load state (once per launch)
  double r[3], v[3], Q[9], w[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    r[c] = sl.active ? __ldcs(p.node + c * p.nn + sl.node) : 0.0;
    v[c] = sl.active ? __ldcs(p.node + (3 + c) * p.nn + sl.node) : 0.0;
  }
#pragma unroll
  for (int c = 0; c < 9; ++c) Q[c] = sl.has_e ? __ldcs(p.elem + c * p.ne + sl.elem) : 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) w[c] = sl.has_e ? __ldcs(p.elem + (9 + c) * p.ne + sl.elem) : 0.0;

  const double h = p.h, hh = 0.5 * p.h;
  double t = p.t;
  unsigned fbits = 0;

  const int nsteps = (MODE == MODE_FUSED) ? p.n_steps : 1;
  for (int step = 0; step < nsteps; ++step) {
    const double t_half = t + hh;
    if (MODE == MODE_FUSED || MODE == MODE_DRIFT) {
      // ---- A1-A3 drift h/2 (clamped node / element are held at their pose)
      if (!cl_node) {
#pragma unroll
        for (int c = 0; c < 3; ++c) r[c] = fma(hh, v[c], r[c]);
      }
      if (sl.has_e && !cl_elem) rotate_inplace(Q, hh * w[0], hh * w[1], hh * w[2]);
    }
    if (MODE == MODE_FUSED || MODE == MODE_DYN) {
      // ---- exchange A
      if (sl.active) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { xr[c * BLOCK + s] = r[c]; xv[c * BLOCK + s] = v[c]; }
#pragma unroll
        for (int c = 0; c < 9; ++c) xQ[c * BLOCK + s] = Q[c];
      }
      __syncthreads();

      // ---- A4-A5 edge i: kinematics, shear/stretch strain, stress
      double ell[3] = {0, 0, 0}, Ql[3] = {0, 0, 0}, nb[3] = {0, 0, 0}, n[3] = {0, 0, 0};
      double l = 0.0, inv_e = 0.0, e = 1.0, edot = 0.0;
      if (sl.has_e) {
        const double lh = general ? __ldg(p.gpar + GP_LHAT * p.ng + sl.node) : __ldg(rec + REC_LHAT);
        const double ilh = general ? __ldg(p.gpar + GP_ILHAT * p.ng + sl.node) : __ldg(rec + REC_ILHAT);
        double dv[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          ell[c] = xr[c * BLOCK + s + 1] - r[c];
          dv[c] = xv[c * BLOCK + s + 1] - v[c];
        }
        const double l2 = dot3(ell, ell);
        const double il = rsqrt(l2);
        l = l2 * il;
        e = l * ilh;
        inv_e = lh * il;
        edot = dot3(ell, dv) * il * ilh;
        if (!(e >= 1e-12)) fbits |= 2u;  // ER_F_DEGENERATE
        // sigma = e Q t - e3 = Q l / lhat - e3
        Ql[0] = dot3(Q, ell);
        Ql[1] = dot3(Q + 3, ell);
        Ql[2] = dot3(Q + 6, ell);
        double sg[3] = {Ql[0] * ilh, Ql[1] * ilh, fma(Ql[2], ilh, -1.0)};
        if (p.sigma0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) sg[c] -= __ldg(p.sigma0 + c * p.ne + sl.elem);
        }
        const double S1 = general ? __ldg(p.gpar + GP_S1 * p.ng + sl.node) : __ldg(rec + REC_S1);
        const double S3 = general ? __ldg(p.gpar + GP_S3 * p.ng + sl.node) : __ldg(rec + REC_S3);
        nb[0] = S1 * sg[0] * inv_e;
        nb[1] = S1 * sg[1] * inv_e;
        nb[2] = S3 * sg[2] * inv_e;
        // n = Q^T nbar (lab)
#pragma unroll
        for (int c = 0; c < 3; ++c) n[c] = fma(Q[c], nb[0], fma(Q[3 + c], nb[1], Q[6 + c] * nb[2]));
      }
      // ---- A6 Voronoi i: curvature via inverse Rodrigues
      double kap[3] = {0, 0, 0};
      double cth = 1.0, s2 = 0.0;
      if (sl.has_v) {
        double Qp[9];
#pragma unroll
        for (int c = 0; c < 9; ++c) Qp[c] = xQ[c * BLOCK + s - 1];
        logrot_pair(Q, Qp, kap, cth, s2);
        if (cth < 0.0 && s2 <= 1e-12 * cth * cth) fbits |= 4u;  // ER_F_ANTIPODAL: theta >= pi - 1e-6
      }
      // ---- exchange B
      if (sl.has_e) {
        xl[s] = l;
#pragma unroll
        for (int c = 0; c < 3; ++c) xn[c * BLOCK + s] = n[c];
      }
      __syncthreads();

      // ---- A6 bending moment and its cross term
      double mb[3] = {0, 0, 0}, be[3] = {0, 0, 0};
      if (sl.has_v) {
        const double Dh = general ? __ldg(p.gpar + GP_DH * p.ng + sl.node) : __ldg(rec + REC_LHAT);
        const double iDh = general ? 1.0 / Dh : __ldg(rec + REC_ILHAT);
#pragma unroll
        for (int c = 0; c < 3; ++c) kap[c] *= iDh;
        const double D = 0.5 * (xl[s - 1] + l);
        const double ieps = Dh / D;
        const double ieps3 = ieps * ieps * ieps;
        double k0[3] = {0, 0, 0};
        if (p.kappa0) {
#pragma unroll
          for (int c = 0; c < 3; ++c) k0[c] = __ldg(p.kappa0 + c * p.nv + sl.vor);
        }
        if (sl.fl & FL_ACT) {
          const double *r2 = p.rec2 + (int64_t)sl.rod * ER_REC2;
          const double sk = general ? __ldg(p.gpar + GP_SK * p.ng + sl.node) : i * __ldg(rec + REC_LHAT);
          // A sin(2 pi (s/L - f t)) = A sinpi(2 (s/L - f t))
          const double arg = 2.0 * fma(sk, __ldg(r2 + REC2_ACTIL), -__ldg(r2 + REC2_ACTF) * t_half);
          k0[p.act_comp] += __ldg(r2 + REC2_ACTA) * sinpi(arg);
        }
        const double B1 = general ? __ldg(p.gpar + GP_BV1 * p.ng + sl.node) : __ldg(rec + REC_B1);
        const double B2 = general ? __ldg(p.gpar + GP_BV2 * p.ng + sl.node) : __ldg(rec + REC_B2);
        const double B3 = general ? __ldg(p.gpar + GP_BV3 * p.ng + sl.node) : __ldg(rec + REC_B3);
        mb[0] = B1 * (kap[0] - k0[0]) * ieps3;
        mb[1] = B2 * (kap[1] - k0[1]) * ieps3;
        mb[2] = B3 * (kap[2] - k0[2]) * ieps3;
        be[0] = (kap[1] * mb[2] - kap[2] * mb[1]) * Dh;
        be[1] = (kap[2] * mb[0] - kap[0] * mb[2]) * Dh;
        be[2] = (kap[0] * mb[1] - kap[1] * mb[0]) * Dh;
      }
      // ---- A7 + A9 node force, linear acceleration, kick
      if (sl.active) {
        double F[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) F[c] = n[c] - (i >= 1 ? xn[c * BLOCK + s - 1] : 0.0);
        if ((sl.fl & FL_TIP) && i == (clamp == 2 ? 0 : N)) {
          const double *r2 = p.rec2 + (int64_t)sl.rod * ER_REC2;
#pragma unroll
          for (int c = 0; c < 3; ++c) F[c] += __ldg(r2 + REC2_TIPX + c);
        }
        const double im = general ? __ldg(p.gpar + GP_IM * p.ng + sl.node)
                                  : __ldg(rec + REC_IM) * ((i == 0 || i == N) ? 2.0 : 1.0);
        const double nu = __ldg(rec + REC_NU);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double a = fma(F[c], im, fma(-nu, v[c], p.g[c]));
          v[c] = cl_node ? 0.0 : fma(h, a, v[c]);
        }
      }
      // ---- exchange C (aliases A; all A reads happened before the B barrier)
      if (sl.active) {
#pragma unroll
        for (int c = 0; c < 3; ++c) { xm[c * BLOCK + s] = mb[c]; xb[c * BLOCK + s] = be[c]; }
      }
      __syncthreads();

      // ---- A8 + A9 element couple, angular acceleration, kick
      if (sl.has_e) {
        double C[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
          C[c] = (xm[c * BLOCK + s + 1] - mb[c]) + 0.5 * (xb[c * BLOCK + s + 1] + be[c]);
        // shear torque lhat (Q t) x S(sigma - sigma0) == (Q l) x nbar
        C[0] += Ql[1] * nb[2] - Ql[2] * nb[1];
        C[1] += Ql[2] * nb[0] - Ql[0] * nb[2];
        C[2] += Ql[0] * nb[1] - Ql[1] * nb[0];
        if (p.mag) {  // c_mag = lhat m x (Q b(t))
          double sn, cs;
          sincos(p.b_omega * t_half, &sn, &cs);
          const double b[3] = {cs * p.b0[0] - sn * p.b0[1], sn * p.b0[0] + cs * p.b0[1], p.b0[2]};
          const double Qb[3] = {dot3(Q, b), dot3(Q + 3, b), dot3(Q + 6, b)};
          double m[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) m[c] = __ldg(p.mag + c * p.ne + sl.elem);
          const double lh = general ? __ldg(p.gpar + GP_LHAT * p.ng + sl.node) : __ldg(rec + REC_LHAT);
          C[0] += lh * (m[1] * Qb[2] - m[2] * Qb[1]);
          C[1] += lh * (m[2] * Qb[0] - m[0] * Qb[2]);
          C[2] += lh * (m[0] * Qb[1] - m[1] * Qb[0]);
        }
        double iJ[3], kJ[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          iJ[c] = general ? __ldg(p.gpar + (GP_IJ1 + c) * p.ng + sl.node) : __ldg(rec + REC_IJ1 + c);
          kJ[c] = general ? __ldg(p.gpar + (GP_KJ1 + c) * p.ng + sl.node) : __ldg(rec + REC_KJ1 + c);
        }
        const double nu = __ldg(rec + REC_NU);
        const double rate = edot * inv_e;
        const double eu[3] = {w[1] * w[2], w[2] * w[0], w[0] * w[1]};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double al = fma(e * iJ[c], C[c], fma(kJ[c], eu[c], (rate - nu) * w[c]));
          w[c] = cl_elem ? 0.0 : fma(h, al, w[c]);
        }
      }
    }
    if (MODE == MODE_FUSED) {
      // ---- A10 drift h/2 with the new rates
      t = t_half + hh;
      if (!cl_node) {
#pragma unroll
        for (int c = 0; c < 3; ++c) r[c] = fma(hh, v[c], r[c]);
      }
      if (sl.has_e && !cl_elem) rotate_inplace(Q, hh * w[0], hh * w[1], hh * w[2]);
      if (step + 1 < nsteps) __syncthreads();  // exchange C buffers are re-used as A next step
    }
    // ---- fault checks: non-finite state, overspeed
    if (sl.active && MODE != MODE_DYN) {
      double acc = r[0] + r[1] + r[2] + v[0] + v[1] + v[2];
      if (sl.has_e) {
#pragma unroll
        for (int c = 0; c < 9; ++c) acc += Q[c];
        acc += w[0] + w[1] + w[2];
      }
      if (!isfinite(acc)) fbits |= 1u;
      if (dot3(v, v) > __ldg(rec + REC_VMAX2)) fbits |= 8u;
    }
  }

  // ---- store state (once per launch)
  if (sl.active) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      __stcs(p.node + c * p.nn + sl.node, r[c]);
      __stcs(p.node + (3 + c) * p.nn + sl.node, v[c]);
    }
  }
  if (sl.has_e) {
#pragma unroll
    for (int c = 0; c < 9; ++c) __stcs(p.elem + c * p.ne + sl.elem, Q[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c) __stcs(p.elem + (9 + c) * p.ne + sl.elem, w[c]);
  }
  report_fault(p, fbits, sl.rod);
}

// --------------------------------------------------------------------------- diagnostics
// Per-tile partial sums of the energy functional at time p.t; deterministic.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) diag_kernel(const ErStepParams p) {
  extern __shared__ double smem[];
  double *xr = smem;
  double *xQ = xr + 3 * BLOCK;
  double *red = xQ + 9 * BLOCK;  // [16][BLOCK/32]
  int *rstart = reinterpret_cast<int *>(red + 16 * (BLOCK / 32));
  const Slot sl = decode_slot<BLOCK>(p, blockIdx.x, rstart);
  const int s = threadIdx.x;
  const int i = sl.i, N = sl.N;
  const bool general = (sl.fl & FL_GENERAL) != 0;
  const double *rec = p.rec + (int64_t)sl.rod * ER_REC;
  double r[3] = {0, 0, 0}, v[3] = {0, 0, 0}, Q[9], w[3] = {0, 0, 0};
  for (int c = 0; c < 3; ++c) {
    if (sl.active) { r[c] = p.node[c * p.nn + sl.node]; v[c] = p.node[(3 + c) * p.nn + sl.node]; }
    if (sl.has_e) w[c] = p.elem[(9 + c) * p.ne + sl.elem];
  }
  for (int c = 0; c < 9; ++c) Q[c] = sl.has_e ? p.elem[c * p.ne + sl.elem] : 0.0;
  if (sl.active) {
    for (int c = 0; c < 3; ++c) xr[c * BLOCK + s] = r[c];
    for (int c = 0; c < 9; ++c) xQ[c * BLOCK + s] = Q[c];
  }
  __syncthreads();
  double acc[16];
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  if (sl.active) {
    const double im = general ? p.gpar[GP_IM * p.ng + sl.node] : rec[REC_IM] * ((i == 0 || i == N) ? 2.0 : 1.0);
    const double m = 1.0 / im;
    const double vv = dot3(v, v);
    acc[0] = 0.5 * m * vv;
    acc[4] = -m * dot3(p.g, r);
    const int clamp = sl.fl & FL_CLAMP_MASK;
    if ((sl.fl & FL_TIP) && i == (clamp == 2 ? 0 : N)) {
      const double *r2 = p.rec2 + (int64_t)sl.rod * ER_REC2;
      acc[5] = -(r2[0] * r[0] + r2[1] * r[1] + r2[2] * r[2]);
    }
    acc[6] = m * v[0]; acc[7] = m * v[1]; acc[8] = m * v[2];
    acc[9] = sqrt(vv);
    acc[10] = m;
  }
  if (sl.has_e) {
    const double lh = general ? p.gpar[GP_LHAT * p.ng + sl.node] : rec[REC_LHAT];
    const double ilh = general ? p.gpar[GP_ILHAT * p.ng + sl.node] : rec[REC_ILHAT];
    double ell[3];
    for (int c = 0; c < 3; ++c) ell[c] = xr[c * BLOCK + s + 1] - r[c];
    const double l = sqrt(dot3(ell, ell));
    const double e = l * ilh;
    double sg[3] = {dot3(Q, ell) * ilh, dot3(Q + 3, ell) * ilh, dot3(Q + 6, ell) * ilh - 1.0};
    if (p.sigma0) for (int c = 0; c < 3; ++c) sg[c] -= p.sigma0[c * p.ne + sl.elem];
    const double S1 = general ? p.gpar[GP_S1 * p.ng + sl.node] : rec[REC_S1];
    const double S3 = general ? p.gpar[GP_S3 * p.ng + sl.node] : rec[REC_S3];
    acc[2] = 0.5 * (S1 * sg[0] * sg[0] + S1 * sg[1] * sg[1] + S3 * sg[2] * sg[2]) * lh;
    for (int c = 0; c < 3; ++c) {
      const double iJ = general ? p.gpar[(GP_IJ1 + c) * p.ng + sl.node] : rec[REC_IJ1 + c];
      acc[1] += 0.5 * w[c] * w[c] / (iJ * e);
    }
    acc[11] = 1.0;
  }
  if (sl.has_v) {
    double Qp[9], kap[3], cth, s2;
    for (int c = 0; c < 9; ++c) Qp[c] = xQ[c * BLOCK + s - 1];
    logrot_pair(Q, Qp, kap, cth, s2);
    const double Dh = general ? p.gpar[GP_DH * p.ng + sl.node] : rec[REC_LHAT];
    double k0[3] = {0, 0, 0};
    if (p.kappa0) for (int c = 0; c < 3; ++c) k0[c] = p.kappa0[c * p.nv + sl.vor];
    if (sl.fl & FL_ACT) {
      const double *r2 = p.rec2 + (int64_t)sl.rod * ER_REC2;
      const double sk = general ? p.gpar[GP_SK * p.ng + sl.node] : i * rec[REC_LHAT];
      k0[p.act_comp] += r2[REC2_ACTA] * sinpi(2.0 * (sk * r2[REC2_ACTIL] - r2[REC2_ACTF] * p.t));
    }
    for (int c = 0; c < 3; ++c) {
      const double Bv = general ? p.gpar[(GP_BV1 + c) * p.ng + sl.node] : rec[REC_B1 + c];
      const double d = kap[c] / Dh - k0[c];
      acc[3] += 0.5 * Bv * d * d * Dh;
    }
  }
  // deterministic block reduction: warp shuffles, then warp partials in fixed order
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
  // one block of 32 threads per diagnostic, fixed-order strided sums then a fixed tree
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
__global__ void soa_to_aos(const double *__restrict__ src, double *__restrict__ dst, int64_t n, int k,
                           int64_t stride) {
  const int64_t total = n * k;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = q / k;
    const int c = (int)(q - e * k);
    dst[q] = src[c * stride + e];
  }
}
__global__ void fill_planes(double *dst, int64_t n, int k, int64_t stride, double value) {
  const int64_t total = n * k;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = q / k;
    const int c = (int)(q - e * k);
    dst[c * stride + e] = value;
  }
}

// Validation of uploaded state: [0] max |Q Q^T - I|, [1] max |det Q - 1|, [2] non-finite count.
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}
__global__ void validate_state(const double *node, int64_t nn, int64_t n_nodes, const double *elem, int64_t ne,
                               int64_t n_elems, double *out) {
  double m_orth = 0.0, m_det = 0.0, bad = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_elems; q += (int64_t)gridDim.x * blockDim.x) {
    double Q[9];
    for (int c = 0; c < 9; ++c) Q[c] = elem[c * ne + q];
    bool fin = true;
    for (int c = 0; c < 12; ++c) fin = fin && isfinite(elem[c * ne + q]);
    if (!fin) { bad += 1.0; continue; }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        const double d = dot3(Q + 3 * a, Q + 3 * b) - (a == b ? 1.0 : 0.0);
        m_orth = fmax(m_orth, fabs(d));
      }
    const double det = Q[0] * (Q[4] * Q[8] - Q[5] * Q[7]) - Q[1] * (Q[3] * Q[8] - Q[5] * Q[6]) +
                       Q[2] * (Q[3] * Q[7] - Q[4] * Q[6]);
    m_det = fmax(m_det, fabs(det - 1.0));
  }
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n_nodes; q += (int64_t)gridDim.x * blockDim.x) {
    bool fin = true;
    for (int c = 0; c < 6; ++c) fin = fin && isfinite(node[c * nn + q]);
    if (!fin) bad += 1.0;
  }
  atomic_max_nonneg(out + 0, m_orth);
  atomic_max_nonneg(out + 1, m_det);
  if (bad > 0.0) atomicAdd(out + 2, bad);
}

}  // namespace er

// --------------------------------------------------------------------------- launch wrappers
static size_t step_smem(int block) { return (size_t)(15 + 4) * 8 * block + sizeof(int) * (block / 2 + 2); }
static size_t diag_smem(int block) { return (size_t)12 * 8 * block + 16 * 8 * (block / 32) + sizeof(int) * (block / 2 + 2); }

template <int BLOCK, int MINB, int MODE>
static cudaError_t launch_step_t(const ErStepParams &p, int64_t n_tiles, cudaStream_t st) {
  auto k = er::step_kernel<BLOCK, MINB, MODE>;
  const size_t sm = step_smem(BLOCK);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k<<<(unsigned)n_tiles, BLOCK, sm, st>>>(p);
  return cudaGetLastError();
}

extern "C" {

// mode: 0 fused, 1 drift, 2 dyn
cudaError_t er_launch_step(const ErStepParams *p, int64_t n_tiles, int block, int mode, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  if (block == 256) {
    if (mode == 0) return launch_step_t<256, 2, er::MODE_FUSED>(*p, n_tiles, st);
    if (mode == 1) return launch_step_t<256, 2, er::MODE_DRIFT>(*p, n_tiles, st);
    return launch_step_t<256, 2, er::MODE_DYN>(*p, n_tiles, st);
  }
  if (mode == 0) return launch_step_t<512, 1, er::MODE_FUSED>(*p, n_tiles, st);
  if (mode == 1) return launch_step_t<512, 1, er::MODE_DRIFT>(*p, n_tiles, st);
  return launch_step_t<512, 1, er::MODE_DYN>(*p, n_tiles, st);
}

cudaError_t er_launch_diag(const ErStepParams *p, int64_t n_tiles, int block, double *out, cudaStream_t st) {
  if (n_tiles > 0) {
    const size_t sm = diag_smem(block);
    if (block == 256) {
      cudaFuncSetAttribute(er::diag_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      er::diag_kernel<256><<<(unsigned)n_tiles, 256, sm, st>>>(*p);
    } else {
      cudaFuncSetAttribute(er::diag_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      er::diag_kernel<512><<<(unsigned)n_tiles, 512, sm, st>>>(*p);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  er::diag_finish_kernel<<<12, 32, 0, st>>>(p->diag_partial, n_tiles, out);
  return cudaGetLastError();
}

cudaError_t er_launch_aos_to_soa(const double *src, double *dst, int64_t n, int k, int64_t stride, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  er::aos_to_soa<<<148 * 8, 256, 0, st>>>(src, dst, n, k, stride);
  return cudaGetLastError();
}
cudaError_t er_launch_soa_to_aos(const double *src, double *dst, int64_t n, int k, int64_t stride, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  er::soa_to_aos<<<148 * 8, 256, 0, st>>>(src, dst, n, k, stride);
  return cudaGetLastError();
}
cudaError_t er_launch_fill(double *dst, int64_t n, int k, int64_t stride, double value, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  er::fill_planes<<<148 * 8, 256, 0, st>>>(dst, n, k, stride, value);
  return cudaGetLastError();
}
cudaError_t er_launch_validate(const double *node, int64_t nn, int64_t n_nodes, const double *elem, int64_t ne,
                               int64_t n_elems, double *out, cudaStream_t st) {
  er::validate_state<<<148 * 4, 256, 0, st>>>(node, nn, n_nodes, elem, ne, n_elems, out);
  return cudaGetLastError();
}

}  // extern "C"
