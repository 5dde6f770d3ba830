// er_contact.cu -- rod-rod and rod-boundary contact with friction on sm_100a.
//
// The paper names the model but leaves its formulas to the missing supplement: "rod interactions
// via normal force and friction", a collision engine whose broad phase is a
// hierarchical hash grid (HHG, Fig. 2e) and which forces synchronous stepping
// (PAPER.md:86).  Readings: DESIGN.md §3 #27.  Contact forces are evaluated once per step, at
// the half-step configuration (after drift-1) with v^n, like every other force (reading #12).
//
// Per step, after the drift-1 kernel has written the canonical node planes (r, v):
//   hhg_keys    one thread per element: capsule AABB, HHG level (smallest cell >= the AABB's
//               largest extent), cell of the AABB centre, hashed key
//   CUB radix sort of (key, element) -- stable, so a bucket lists its elements in id order
//   hhg_cells   bucket ranges; proxies gathered into sorted (spatially coherent) order
//   hhg_narrow  one thread per sorted proxy a: the 27 cells around a at a's level and at every
//               coarser populated level; per candidate b the AABB test, the exact segment-segment
//               closest points, the penalty + friction law.  Same-level pairs are evaluated by
//               BOTH proxies (gather, no atomics) in one canonical order (lower element id first),
//               so the two sides compute bit-identical forces; a pair across levels is evaluated
//               once, by the finer proxy, which leaves a record for the coarser one.
//   hhg_finish  one thread per element: cross-level records summed in source-id order, the
//               half-space law on the element's node(s), result in fc.
// Every sum has a fixed order: results are bitwise reproducible run to run.
//
// This file is compiled with -fmad=false: the closest-point selection and the contact / friction
// branch decisions are taken on IEEE-rounded products and sums in the order written, which is
// the plain reading of the definitions (DESIGN §3 #27, §6).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "er_layout.h"

namespace erc {

constexpr unsigned long long F_CONTACT = 16ull;  // ER_F_CONTACT (include/er.h)

__device__ __forceinline__ void flag_fault(const ErContactParams &p, int rod) {
  atomicOr(p.fault, F_CONTACT);
  atomicMin(p.fault + 1, (unsigned long long)rod);
}

__device__ __forceinline__ uint32_t cell_hash(int cx, int cy, int cz, int l, int hbits) {
  const uint32_t h = ((uint32_t)cx * 73856093u) ^ ((uint32_t)cy * 19349663u) ^ ((uint32_t)cz * 83492791u) ^
                     ((uint32_t)l * 2654435761u);
  return h & ((1u << hbits) - 1u);
}

// AABB of the capsule (segment p0-p1, radius r).
__device__ __forceinline__ void capsule_aabb(const double p0[3], const double p1[3], double r, double lo[3],
                                             double hi[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = fmin(p0[c], p1[c]) - r;
    hi[c] = fmax(p0[c], p1[c]) + r;
  }
}

// HHG level and cell of a proxy: the smallest level whose cell is >= the AABB's largest extent
// (SPEC.md:339), cell of the AABB centre.  Returns false when the proxy cannot be binned
// (wider than the top level, non-finite, or a cell index beyond +-2^30).
__device__ __forceinline__ bool proxy_cell(const ErContactParams &p, const double lo[3], const double hi[3], int &l,
                                           int c[3]) {
  const double w = fmax(hi[0] - lo[0], fmax(hi[1] - lo[1], hi[2] - lo[2]));
  l = 0;
  while (l < p.nlev - 1 && w > p.cell[l]) ++l;
  bool ok = w <= p.cell[l];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = floor((0.5 * (lo[k] + hi[k])) * p.icell[l]);
    ok = ok && (x > -1073741824.0 && x < 1073741824.0);  // also false for NaN
    c[k] = ok ? (int)x : 0;
  }
  return ok;
}

__device__ __forceinline__ void load_nodes(const ErContactParams &p, int64_t n0, double p0[3], double p1[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    p0[c] = p.cnode[c * p.ns + n0];
    p1[c] = p.cnode[c * p.ns + n0 + 1];
  }
}

__global__ void hhg_keys(const ErContactParams p) {
  unsigned lmask = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n_elems; e += (int64_t)gridDim.x * blockDim.x) {
    const int rod = __ldg(p.erod + e);
    double p0[3], p1[3], lo[3], hi[3];
    load_nodes(p, e + rod, p0, p1);
    capsule_aabb(p0, p1, __ldg(p.rad + rod), lo, hi);
    int l, c[3];
    if (!proxy_cell(p, lo, hi, l, c)) flag_fault(p, rod);
    lmask |= 1u << l;
    p.key[e] = cell_hash(c[0], c[1], c[2], l, p.hbits);
    p.val[e] = (int32_t)e;
  }
  lmask = __reduce_or_sync(0xffffffffu, lmask);
  if ((threadIdx.x & 31) == 0 && lmask) atomicOr(p.ctr + 4, (unsigned long long)lmask);
}

__global__ void hhg_cells(const ErContactParams p) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < p.n_elems; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = p.key_s[q];
    if (q == 0 || p.key_s[q - 1] != k) p.cstart[k] = (int32_t)q;
    if (q == p.n_elems - 1 || p.key_s[q + 1] != k) p.cend[k] = (int32_t)(q + 1);
    const int32_t e = p.val_s[q];
    const int rod = __ldg(p.erod + e);
    const int64_t n0 = (int64_t)e + rod;
    double p0[3], p1[3], lo[3], hi[3];
    load_nodes(p, n0, p0, p1);
    capsule_aabb(p0, p1, __ldg(p.rad + rod), lo, hi);
    int l, c[3];
    proxy_cell(p, lo, hi, l, c);
    double *P = p.p01 + 6 * q, *V = p.v01 + 6 * q;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      P[d] = p0[d];
      P[3 + d] = p1[d];
      V[d] = p.cnode[(3 + d) * p.ns + n0];
      V[3 + d] = p.cnode[(3 + d) * p.ns + n0 + 1];
    }
    p.meta[q] = make_int4(e, rod, l, 0);
    p.cellc[q] = make_int4(c[0], c[1], c[2], l);
  }
}

__device__ __forceinline__ double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

// Closest points of segments P(s) = p0 + s (p1 - p0), Q(t) = q0 + t (q1 - q0), s, t in [0, 1]:
// the minimiser of |P(s) - Q(t)|^2 over the unit square.  Candidates in this order: the interior
// stationary point (when inside the square), then the edges s = 0, s = 1, t = 0, t = 1 each with
// its clamped 1-D minimiser; the first candidate of least distance wins (DESIGN §3 #27).
__device__ void segment_closest(const double p0[3], const double p1[3], const double q0[3], const double q1[3], double &s,
                                double &t, double &dist) {
  double u[3], v[3], w[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    u[c] = p1[c] - p0[c];
    v[c] = q1[c] - q0[c];
    w[c] = p0[c] - q0[c];
  }
  const double uu = dot3(u, u), vv = dot3(v, v), uv = dot3(u, v), uw = dot3(u, w), vw = dot3(v, w);
  double cs[5], ct[5];
  int n = 0;
  const double det = uu * vv - uv * uv;
  if (det > 0.0) {
    const double si = (uv * vw - uw * vv) / det, ti = (uu * vw - uv * uw) / det;
    if (si >= 0.0 && si <= 1.0 && ti >= 0.0 && ti <= 1.0) { cs[n] = si; ct[n] = ti; ++n; }
  }
  cs[n] = 0.0; ct[n] = vv > 0.0 ? clamp01(vw / vv) : 0.0; ++n;
  cs[n] = 1.0; ct[n] = vv > 0.0 ? clamp01((vw + uv) / vv) : 0.0; ++n;
  cs[n] = uu > 0.0 ? clamp01(-uw / uu) : 0.0; ct[n] = 0.0; ++n;
  cs[n] = uu > 0.0 ? clamp01((uv - uw) / uu) : 0.0; ct[n] = 1.0; ++n;
  double best = -1.0;
  s = 0.0;
  t = 0.0;
  for (int k = 0; k < n; ++k) {
    double x[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) x[c] = p0[c] + cs[k] * u[c] - q0[c] - ct[k] * v[c];
    const double d2 = dot3(x, x);
    if (best < 0.0 || d2 < best) { best = d2; s = cs[k]; t = ct[k]; }
  }
  dist = sqrt(best);
}

// Penalty normal force F_n = max(0, k (-gap) - gamma_n v_n) along n, regularised Coulomb friction
// F_t = -mu_k F_n v_t/|v_t| (|v_t| > v_stick) or -mu_s F_n v_t / v_stick: the force on the body
// whose relative velocity is vr (DESIGN §3 #27).
__device__ __forceinline__ void contact_law(const ErContactLaw &L, double k, double gap, const double n[3],
                                            const double vr[3], double F[3]) {
  const double vn = dot3(vr, n);
  double fn = k * (-gap) - L.gamma_n * vn;
  if (fn < 0.0) fn = 0.0;
  double vt[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) vt[c] = vr[c] - vn * n[c];
  const double svt = sqrt(dot3(vt, vt));
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double ft = 0.0;
    if (svt > L.v_stick) ft = -L.mu_k * fn * vt[c] / svt;
    else if (L.v_stick > 0.0) ft = -L.mu_s * fn * vt[c] / L.v_stick;
    F[c] = fn * n[c] + ft;
  }
}

// Force of the pair (x, y), x the lower element id, on x; false when not in contact.
__device__ __forceinline__ bool pair_force(const ErContactParams &p, const double *Px, const double *Py,
                                           const double *Vx, const double *Vy, double rx, double ry, double k,
                                           double F[3], double &s, double &t) {
  double d;
  segment_closest(Px, Px + 3, Py, Py + 3, s, t, d);
  const double gap = d - (rx + ry);
  if (!(gap < 0.0) || d == 0.0) return false;
  double n[3], vr[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double pa = (1.0 - s) * Px[c] + s * Px[3 + c];
    const double pb = (1.0 - t) * Py[c] + t * Py[3 + c];
    n[c] = (pa - pb) / d;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double va = (1.0 - s) * Vx[c] + s * Vx[3 + c];
    const double vb = (1.0 - t) * Vy[c] + t * Vy[3 + c];
    vr[c] = va - vb;
  }
  contact_law(p.law, k, gap, n, vr, F);
  return true;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) hhg_narrow(const ErContactParams p) {
  const int64_t q = blockIdx.x * (int64_t)BLOCK + threadIdx.x;
  unsigned long long n_cand = 0, n_cont = 0, n_cross = 0;
  if (q < p.n_elems) {
    const int4 ma = p.meta[q];
    const int ea = ma.x, roda = ma.y, la = ma.z;
    double Pa[6], Va[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) { Pa[c] = p.p01[6 * q + c]; Va[c] = p.v01[6 * q + c]; }
    const double ra = __ldg(p.rad + roda), kra = __ldg(p.kr + roda);
    double lo[3], hi[3];
    capsule_aabb(Pa, Pa + 3, ra, lo, hi);
    double f[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const unsigned lmask = (unsigned)*((volatile unsigned long long *)(p.ctr + 4));
    for (int L = la; L < p.nlev; ++L) {
      if (!((lmask >> L) & 1u)) continue;
      const double cs = p.cell[L], ics = p.icell[L], mg = 0.5 * cs * (1.0 + 1e-9);
      int c0[3], c1[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        c0[k] = (int)floor((lo[k] - mg) * ics);
        c1[k] = (int)floor((hi[k] + mg) * ics);
      }
      for (int cz = c0[2]; cz <= c1[2]; ++cz)
        for (int cy = c0[1]; cy <= c1[1]; ++cy)
          for (int cx = c0[0]; cx <= c1[0]; ++cx) {
            const uint32_t key = cell_hash(cx, cy, cz, L, p.hbits);
            const int b0 = p.cstart[key];
            if (b0 < 0) continue;
            const int b1 = p.cend[key];
            for (int b = b0; b < b1; ++b) {
              if (b == q) continue;
              const int4 cb = __ldg(p.cellc + b);
              if (cb.w != L || cb.x != cx || cb.y != cy || cb.z != cz) continue;  // another cell in the bucket
              const int4 mb = __ldg(p.meta + b);
              const int eb = mb.x, rodb = mb.y;
              if (roda == rodb && abs(ea - eb) <= p.law.exclude) continue;
              const double *Pb = p.p01 + 6 * (int64_t)b;
              const double rb = __ldg(p.rad + rodb);
              double lob[3], hib[3], Pbl[6];
#pragma unroll
              for (int c = 0; c < 6; ++c) Pbl[c] = __ldg(Pb + c);
              capsule_aabb(Pbl, Pbl + 3, rb, lob, hib);
              const bool ov = fmax(lo[0], lob[0]) <= fmin(hi[0], hib[0]) && fmax(lo[1], lob[1]) <= fmin(hi[1], hib[1]) &&
                              fmax(lo[2], lob[2]) <= fmin(hi[2], hib[2]);
              if (!ov) continue;
              const bool owner = L > la || ea < eb;  // counts each pair once
              n_cand += owner;
              double Vb[6];
#pragma unroll
              for (int c = 0; c < 6; ++c) Vb[c] = __ldg(p.v01 + 6 * (int64_t)b + c);
              const double krb = __ldg(p.kr + rodb);
              const double k = p.law.k_n > 0.0 ? p.law.k_n : fmin(kra, krb);
              const bool a_first = ea < eb;
              double F[3], s, t;
              const bool hit = a_first ? pair_force(p, Pa, Pbl, Va, Vb, ra, rb, k, F, s, t)
                                       : pair_force(p, Pbl, Pa, Vb, Va, rb, ra, k, F, s, t);
              if (!hit) continue;
              n_cont += owner;
              // F acts on the first (lower-id) element at weights (1-s, s); -F on the second at (1-t, t)
              const double wa0 = a_first ? 1.0 - s : 1.0 - t, wa1 = a_first ? s : t;
              const double sg = a_first ? 1.0 : -1.0;
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                f[c] += wa0 * (sg * F[c]);
                f[3 + c] += wa1 * (sg * F[c]);
              }
              if (L > la) {  // the coarser proxy b never sees this pair: leave it a record
                ++n_cross;
                const unsigned long long r = atomicAdd(p.ctr + 0, 1ull);
                if (r >= (unsigned long long)p.pcap) { flag_fault(p, rodb); continue; }
                const double wb0 = a_first ? 1.0 - t : 1.0 - s, wb1 = a_first ? t : s;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                  p.pf[6 * r + c] = wb0 * (-sg * F[c]);
                  p.pf[6 * r + 3 + c] = wb1 * (-sg * F[c]);
                }
                p.psrc[r] = ea;
                p.pnext[r] = atomicExch(p.head + eb, (int32_t)r);
              }
            }
          }
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) p.fc[c * p.fs + ea] = f[c];
  }
  // statistics: warp sums, one atomic per warp
  n_cand = __reduce_add_sync(0xffffffffu, (unsigned)n_cand);
  n_cont = __reduce_add_sync(0xffffffffu, (unsigned)n_cont);
  n_cross = __reduce_add_sync(0xffffffffu, (unsigned)n_cross);
  if ((threadIdx.x & 31) == 0) {
    if (n_cand) atomicAdd(p.ctr + 1, n_cand);
    if (n_cont) atomicAdd(p.ctr + 2, n_cont);
    if (n_cross) atomicAdd(p.ctr + 3, n_cross);
  }
}

constexpr int MAX_CROSS = 64;

__global__ void hhg_finish(const ErContactParams p, int cross) {
  unsigned n_plane = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n_elems; e += (int64_t)gridDim.x * blockDim.x) {
    const int rod = __ldg(p.erod + e);
    int h = cross ? p.head[e] : -1;
    const bool plane_last = p.law.plane_on && (e + 1 == p.n_elems || __ldg(p.erod + e + 1) != rod);
    if (h < 0 && !p.law.plane_on) continue;
    double f[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) f[c] = p.fc[c * p.fs + e];
    if (h >= 0) {  // cross-level records, summed in increasing source-element order
      int src[MAX_CROSS], idx[MAX_CROSS], m = 0;
      for (; h >= 0; h = p.pnext[h]) {
        if (m == MAX_CROSS) { flag_fault(p, rod); break; }
        int j = m++;
        const int sv = p.psrc[h];
        while (j > 0 && src[j - 1] > sv) { src[j] = src[j - 1]; idx[j] = idx[j - 1]; --j; }
        src[j] = sv;
        idx[j] = h;
      }
      for (int j = 0; j < m; ++j)
#pragma unroll
        for (int c = 0; c < 6; ++c) f[c] += p.pf[6 * (int64_t)idx[j] + c];
    }
    if (p.law.plane_on) {  // half-space n.x >= d on node j (and node j+1 for a rod's last element)
      const ErContactLaw &L = p.law;
      const double k = L.k_n > 0.0 ? L.k_n : __ldg(p.kr + rod);
      const double r = __ldg(p.rad + rod);
      for (int side = 0; side < (plane_last ? 2 : 1); ++side) {
        const int64_t node = e + rod + side;
        double x[3], v[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) { x[c] = p.cnode[c * p.ns + node]; v[c] = p.cnode[(3 + c) * p.ns + node]; }
        const double gap = dot3(L.pn, x) - L.pd - r;
        if (!(gap < 0.0)) continue;
        ++n_plane;
        double F[3];
        contact_law(L, k, gap, L.pn, v, F);
#pragma unroll
        for (int c = 0; c < 3; ++c) f[3 * side + c] += F[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) p.fc[c * p.fs + e] = f[c];
  }
  n_plane = __reduce_add_sync(0xffffffffu, n_plane);
  if ((threadIdx.x & 31) == 0 && n_plane) atomicAdd(p.ctr + 5, (unsigned long long)n_plane);
}

}  // namespace erc

extern "C" {

// Temporary-storage bytes of the broad-phase sort for n keys of `bits` bits.
cudaError_t er_contact_sort_bytes(int64_t n, int bits, size_t *bytes) {
  *bytes = 0;
  return cub::DeviceRadixSort::SortPairs(nullptr, *bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                         (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, bits);
}

// One contact evaluation (broad + narrow phase) at the positions/velocities in p.cnode: fills
// p.fc.  Stream-ordered; no host synchronisation.  `launches` += kernels launched.
cudaError_t er_contact_eval(const ErContactParams *pp, void *sort_tmp, size_t sort_bytes, cudaStream_t st,
                            int64_t *launches) {
  const ErContactParams &p = *pp;
  const int64_t E = p.n_elems;
  if (E <= 0) return cudaSuccess;
  const int64_t T = 1ll << p.hbits;
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.ctr, 0, 8 * sizeof(unsigned long long), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.cstart, 0xff, sizeof(int32_t) * T, st)) != cudaSuccess) return e;
  const int cross = p.nlev > 1;
  if (cross && (e = cudaMemsetAsync(p.head, 0xff, sizeof(int32_t) * E, st)) != cudaSuccess) return e;
  const unsigned g = (unsigned)std::min<int64_t>((E + 255) / 256, 148 * 16);
  erc::hhg_keys<<<g, 256, 0, st>>>(p);
  size_t bytes = sort_bytes;
  if ((e = cub::DeviceRadixSort::SortPairs(sort_tmp, bytes, p.key, p.key_s, p.val, p.val_s, (int)E, 0, p.hbits, st)) !=
      cudaSuccess)
    return e;
  erc::hhg_cells<<<g, 256, 0, st>>>(p);
  erc::hhg_narrow<128><<<(unsigned)((E + 127) / 128), 128, 0, st>>>(p);
  erc::hhg_finish<<<g, 256, 0, st>>>(p, cross);
  *launches += 5;  // keys, sort (counted once), cells, narrow, finish
  return cudaGetLastError();
}

}  // extern "C"
