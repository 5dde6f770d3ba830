// er_contact.cu -- rod-rod and rod-boundary contact with friction on sm_100a.
//
// The paper names the model but leaves its formulas to the missing supplement: "rod interactions
// via normal force and friction", a collision engine whose broad phase is a
// hierarchical hash grid (HHG, Fig. 2e) and which forces synchronous stepping
// (PAPER.md:86).  Readings: DESIGN.md §3 #27.  Contact forces are evaluated once per step, at
// the half-step configuration (after drift-1) with v^n, like every other force (reading #12).
//
// Broad phase with Verlet lists (the standard neighbour-list reuse of particle codes): proxies
// are capsule AABBs grown by skin/2, so a candidate list built now stays a superset of the
// touching pairs until some node has moved skin/2 from its build position (a pair's distance
// then dropped by less than skin).  The drift-1 kernel, which writes the node planes (r, v),
// checks that bound and raises a device flag; the build kernels below run their work only
// when it is set (no host round trip).
//
// Build (flagged steps only):
//   hhg_aabb     one thread per element: grown AABB, its HHG level (the smallest level whose
//                cell is >= the AABB's largest extent), per level and axis the
//                largest extent (warp-reduced atomicMax) -> query margins and cell boxes
//   hhg_dims     cell box of each level: per axis the largest extent of its proxies (>= 1/4 of
//                the largest axis) -- anisotropic boxes for flat packings
//   hhg_keys     cell of each AABB centre at its level, hashed bucket key; build positions
//   CUB radix sort of (key, element) -- stable, so a bucket lists its elements in id order
//   hhg_cells    sorted float AABB records and cell codes
//   hhg_table    per bucket: (range, the cell code when all its proxies share one cell, else MIXED)
//   hhg_broad    one thread per sorted proxy a: the cells around a's AABB (margin: the largest
//                half extent at that level) at a's level and every coarser populated level;
//                conservative float AABB test + same-rod exclusion -> a's candidate list
// Every step:
//   hhg_narrow   one thread per element a: exact segment-segment closest points and the
//                penalty + friction law for each candidate, gathered into a's two nodes.  Pairs
//                within a level are evaluated by BOTH elements (no atomics) in one canonical
//                order (lower element id first), so the two sides compute bit-identical forces;
//                a pair across levels is evaluated once, by the finer element, which leaves a
//                record for the coarser one.
//   hhg_finish   one thread per element: cross-level records summed in source-id order, the
//                half-space law on the element's node(s).
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
constexpr int CBITS = 20;                        // cell index bits per axis in a cell code
constexpr int CHALF = 1 << (CBITS - 1);

__device__ __forceinline__ void flag_fault(const ErContactParams &p, int rod) {  // rod: packed id
  atomicOr(p.fault, F_CONTACT);
  atomicMin(p.fault + 1, (unsigned long long)__ldg(p.ord + rod));
}

__device__ __forceinline__ uint32_t cell_hash(int cx, int cy, int cz, int l, int hbits) {
  const uint32_t h = ((uint32_t)cx * 73856093u) ^ ((uint32_t)cy * 19349663u) ^ ((uint32_t)cz * 83492791u) ^
                     ((uint32_t)l * 2654435761u);
  return h & ((1u << hbits) - 1u);
}
__device__ __forceinline__ long long cell_code(int cx, int cy, int cz, int l) {
  return ((long long)l << (3 * CBITS)) | ((long long)(cx + CHALF) << (2 * CBITS)) |
         ((long long)(cy + CHALF) << CBITS) | (long long)(cz + CHALF);
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

// HHG level of an AABB: the smallest level whose cell is >= its largest extent.  false when it
// is wider than the top level (or not finite).
__device__ __forceinline__ bool proxy_level(const ErContactParams &p, const double lo[3], const double hi[3], int &l) {
  const double w = fmax(hi[0] - lo[0], fmax(hi[1] - lo[1], hi[2] - lo[2]));
  l = 0;
  while (l < p.nlev - 1 && w > p.cell[l]) ++l;
  return w <= p.cell[l];
}

// Segment of element e: its two nodes, 96 contiguous bytes of the AoS node array.
__device__ __forceinline__ void load_seg(const ErContactParams &p, int64_t e, int &rod, double p0[3], double p1[3]) {
  rod = __ldg(p.erod + e);
  const double *x = p.cnode + 6 * (e + rod);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    p0[c] = x[c];
    p1[c] = x[6 + c];
  }
}

__device__ __forceinline__ double grown(const ErContactParams &p, int rod) { return __ldg(p.rad + rod) + 0.5 * p.skin; }

__device__ __forceinline__ void atomic_max_pos(unsigned long long *a, double x) {
  atomicMax(a, (unsigned long long)__double_as_longlong(x));  // x >= 0: bit order = value order
}

__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__global__ void hhg_aabb(const ErContactParams p) {
  if (!*p.rebuild) return;
  double ext[ER_HHG_MAXLEV][3];
#pragma unroll
  for (int l = 0; l < ER_HHG_MAXLEV; ++l) ext[l][0] = ext[l][1] = ext[l][2] = 0.0;
  unsigned lmask = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n_elems; e += (int64_t)gridDim.x * blockDim.x) {
    int rod, l;
    double p0[3], p1[3], lo[3], hi[3];
    load_seg(p, e, rod, p0, p1);
    capsule_aabb(p0, p1, grown(p, rod), lo, hi);
    if (!proxy_level(p, lo, hi, l)) { flag_fault(p, rod); continue; }
    lmask |= 1u << l;
#pragma unroll
    for (int m = 0; m < ER_HHG_MAXLEV; ++m)  // static register indexing
      if (m == l) {
#pragma unroll
        for (int c = 0; c < 3; ++c) ext[m][c] = fmax(ext[m][c], hi[c] - lo[c]);
      }
  }
  lmask = __reduce_or_sync(0xffffffffu, lmask);
  const bool lead = (threadIdx.x & 31) == 0;
#pragma unroll
  for (int m = 0; m < ER_HHG_MAXLEV; ++m) {
    if (!((lmask >> m) & 1u)) continue;  // warp-uniform
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = warp_max(ext[m][c]);
      if (lead) atomic_max_pos(p.gext + 3 * m + c, x);
    }
  }
  if (lead && lmask) atomicOr(p.bctr + 3, (unsigned long long)lmask);
}

// Cell box of each populated level: per axis the largest extent of its proxies, at least 1/4 of
// the largest axis.  Any box is correct (the query margin is the real largest half extent);
// the box only sets how many proxies a query scans.
__global__ void hhg_dims(const ErContactParams p) {
  const int l = threadIdx.x;
  if (!*p.rebuild || l >= p.nlev) return;
  double x[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) x[c] = __longlong_as_double((long long)p.gext[3 * l + c]);
  const double m = fmax(x[0], fmax(x[1], x[2]));
  const bool pop = (p.bctr[3] >> l) & 1ull;
#pragma unroll
  for (int c = 0; c < 3; ++c) p.gdim[4 * l + c] = pop ? fmax(x[c], 0.25 * m) : p.cell[l];
  p.gdim[4 * l + 3] = pop ? 1.0 : 0.0;
}

__device__ __forceinline__ bool proxy_cell(const ErContactParams &p, const double lo[3], const double hi[3], int l,
                                           int c[3]) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x = floor((0.5 * (lo[k] + hi[k])) / p.gdim[4 * l + k]);
    ok = ok && (x > -(double)CHALF + 2.0 && x < (double)CHALF - 2.0);  // also false for NaN
    c[k] = ok ? (int)x : 0;
  }
  return ok;
}

__global__ void hhg_keys(const ErContactParams p) {
  if (!*p.rebuild) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n_elems; e += (int64_t)gridDim.x * blockDim.x) {
    int rod, l, c[3];
    double p0[3], p1[3], lo[3], hi[3];
    load_seg(p, e, rod, p0, p1);
    capsule_aabb(p0, p1, grown(p, rod), lo, hi);
    const bool okl = proxy_level(p, lo, hi, l);
    if (!proxy_cell(p, lo, hi, l, c) && okl) flag_fault(p, rod);
    p.key[e] = cell_hash(c[0], c[1], c[2], l, p.hbits);
    p.val[e] = (int32_t)e;
    // build positions (node j of element j; the rod's last node with its last element)
    double *b = p.cbuild + 3 * (e + rod);
    const bool last = e + 1 == p.n_elems || __ldg(p.erod + e + 1) != rod;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      b[k] = p0[k];
      if (last) b[3 + k] = p1[k];
    }
  }
}

__global__ void hhg_cells(const ErContactParams p) {
  if (!*p.rebuild) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < p.n_elems; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = p.val_s[q];
    int rod, l, c[3];
    double p0[3], p1[3], lo[3], hi[3];
    load_seg(p, e, rod, p0, p1);
    capsule_aabb(p0, p1, grown(p, rod), lo, hi);
    proxy_level(p, lo, hi, l);
    proxy_cell(p, lo, hi, l, c);
    p.code_s[q] = cell_code(c[0], c[1], c[2], l);
    p.boxa[q] = make_float4(__double2float_rd(lo[0]), __double2float_rd(lo[1]), __double2float_rd(lo[2]), __int_as_float(e));
    p.boxb[q] = make_float4(__double2float_ru(hi[0]), __double2float_ru(hi[1]), __double2float_ru(hi[2]), __int_as_float(rod));
    p.qidx[e] = (int32_t)q;
  }
}

// Bucket table: for the first sorted proxy of each bucket, (start | end << 32, cell code of the
// bucket when all its proxies share one cell, else MIXED).  Empty buckets keep start = -1.
__global__ void hhg_table(const ErContactParams p) {
  if (!*p.rebuild) return;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < p.n_elems; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = p.key_s[q];
    if (q > 0 && p.key_s[q - 1] == k) continue;
    const long long c0 = p.code_s[q];
    long long code = c0;
    int64_t j = q + 1;
    for (; j < p.n_elems && p.key_s[j] == k; ++j)
      if (p.code_s[j] != c0) code = ER_CELL_MIXED;
    p.table[k] = make_longlong2((long long)q | ((long long)j << 32), code);
  }
}

// Broad phase of sorted proxy q: calls visit(b) for every candidate b in a fixed order -- the
// proxies of a's level and of every coarser populated level whose centre cell lies within a's
// AABB grown by that level's largest half extent, and whose float AABB overlaps a's, minus a
// itself and the same-rod stencil.
template <class F>
__device__ __forceinline__ void broad_visit(const ErContactParams &p, int64_t q, F &&visit, unsigned &scanned) {
  const float4 A = p.boxa[q], B = p.boxb[q];
  const int ea = __float_as_int(A.w), roda = __float_as_int(B.w);
  const int la = (int)(p.code_s[q] >> (3 * CBITS));
  const double lo[3] = {(double)A.x, (double)A.y, (double)A.z}, hi[3] = {(double)B.x, (double)B.y, (double)B.z};
  const unsigned lmask = (unsigned)p.bctr[3];
  for (int L = la; L < p.nlev; ++L) {
    if (!((lmask >> L) & 1u)) continue;
    int c0[3], c1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double d = p.gdim[4 * L + k];
      const double hm = 0.5 * __longlong_as_double((long long)p.gext[3 * L + k]) * (1.0 + 1e-9) + 1e-300;
      c0[k] = (int)floor((lo[k] - hm) / d);
      c1[k] = (int)floor((hi[k] + hm) / d);
    }
    for (int cz = c0[2]; cz <= c1[2]; ++cz)
      for (int cy = c0[1]; cy <= c1[1]; ++cy)
        for (int cx = c0[0]; cx <= c1[0]; ++cx) {
          const uint32_t key = cell_hash(cx, cy, cz, L, p.hbits);
          const longlong2 bk = __ldg(p.table + key);  // (start | end << 32, cell code)
          const int b0 = (int)(bk.x & 0xffffffffll);
          if (b0 < 0) continue;
          const long long want = cell_code(cx, cy, cz, L), tc = bk.y;
          if (tc != want && tc != ER_CELL_MIXED) continue;  // bucket of another cell
          const int b1 = (int)(bk.x >> 32);
          scanned += (unsigned)(b1 - b0);
          for (int b = b0; b < b1; ++b) {
            if (tc == ER_CELL_MIXED && __ldg(p.code_s + b) != want) continue;
            if (b == q) continue;
            const float4 Ab = __ldg(p.boxa + b), Bb = __ldg(p.boxb + b);
            if (fmaxf(A.x, Ab.x) > fminf(B.x, Bb.x) || fmaxf(A.y, Ab.y) > fminf(B.y, Bb.y) ||
                fmaxf(A.z, Ab.z) > fminf(B.z, Bb.z))
              continue;
            const int eb = __float_as_int(Ab.w);
            if (__float_as_int(Bb.w) == roda && abs(ea - eb) <= p.law.exclude) continue;
            visit(eb + __float_as_int(Bb.w), L > la, L > la || ea < eb);  // partner's first node
          }
        }
  }
}

// One broad pass over the sorted proxies: the first ER_CAND_K candidates of element e go to
// cand[k * E + e], cnt[e] = the full count; an element with more candidates re-runs the broad
// visit in hhg_narrow (same order).
__global__ void __launch_bounds__(128) hhg_broad(const ErContactParams p) {
  if (!*p.rebuild) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned n = 0, own = 0, scanned = 0;
  if (q < p.n_elems) {
    const int64_t E = p.n_elems;
    const int e = __float_as_int(p.boxa[q].w);
    broad_visit(p, q, [&](int nb, bool cross, bool owner) {
      if (n < ER_CAND_K) p.cand[n * E + e] = nb | (cross ? ER_CAND_CROSS : 0);
      ++n;
      own += owner;
    }, scanned);
    p.cnt[e] = (int32_t)n;
  }
  const unsigned lng = __reduce_add_sync(0xffffffffu, n > ER_CAND_K ? 1u : 0u);
  const unsigned tot = __reduce_add_sync(0xffffffffu, n);
  own = __reduce_add_sync(0xffffffffu, own);
  scanned = __reduce_add_sync(0xffffffffu, scanned);
  if ((threadIdx.x & 31) == 0) {
    if (own) atomicAdd(p.bctr + 0, (unsigned long long)own);
    if (tot) atomicAdd(p.bctr + 1, (unsigned long long)tot);
    if (scanned) atomicAdd(p.bctr + 2, (unsigned long long)scanned);
    if (lng) atomicAdd(p.bctr + 4, (unsigned long long)lng);
  }
}

// Start of a build: empty bucket table, zero build statistics (the cumulative build count stays).
__global__ void hhg_reset(const ErContactParams p, int64_t T) {
  if (!*p.rebuild) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < T; k += (int64_t)gridDim.x * blockDim.x)
    p.table[k] = make_longlong2(-1ll, 0ll);
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < 5) p.bctr[t] = 0ull;
  if (t < 3 * ER_HHG_MAXLEV) p.gext[t] = 0ull;
}

// Graph conditions: the list build runs when the device flag is set; the long-list narrow
// phase when the last build left any list longer than ER_CAND_K.
__global__ void hhg_cond_build(const ErContactParams p, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, *p.rebuild ? 1u : 0u);
}
__global__ void hhg_cond_long(const ErContactParams p, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, p.bctr[4] ? 1u : 0u);
}
__global__ void hhg_cond_cross(const ErContactParams p, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, p.ctr[2] ? 1u : 0u);
}

// End of a build: clear the flag, count the build.
__global__ void hhg_built(const ErContactParams p) {
  if (!*p.rebuild) return;
  *p.rebuild = 0;
  p.bctr[5] += 1;
}

__device__ __forceinline__ double dot3(const double a[3], const double b[3]) { return fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2])); }
__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

// Closest points of segments P(s) = p0 + s u, Q(t) = q0 + t v, s, t in [0, 1], given u, v and
// w = p0 - q0: the minimiser of |P(s) - Q(t)|^2 over the unit square.  Candidates in this order:
// the interior stationary point (when inside the square), then the edges s = 0, s = 1, t = 0,
// t = 1 each with its clamped 1-D minimiser; the first candidate of least distance wins (DESIGN
// §3 #27).  Returns s, t, x = P(s) - Q(t) and |x|^2.
__device__ __forceinline__ double segment_closest(const double u[3], const double v[3], const double w[3], double &s,
                                                  double &t, double x[3]) {
  const double uu = dot3(u, u), vv = dot3(v, v), uv = dot3(u, v), uw = dot3(u, w), vw = dot3(v, w);
  double best = -1.0;
  s = 0.0;
  t = 0.0;
  auto consider = [&](double cs, double ct) {
    double y[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) y[c] = fma(-ct, v[c], fma(cs, u[c], w[c]));
    const double d2 = dot3(y, y);
    if (best < 0.0 || d2 < best) {
      best = d2; s = cs; t = ct;
#pragma unroll
      for (int c = 0; c < 3; ++c) x[c] = y[c];
    }
  };
  const double det = fma(uu, vv, -uv * uv);
  if (det > 0.0) {
    const double idet = 1.0 / det;
    const double si = fma(uv, vw, -uw * vv) * idet, ti = fma(uu, vw, -uv * uw) * idet;
    if (si >= 0.0 && si <= 1.0 && ti >= 0.0 && ti <= 1.0) consider(si, ti);
  }
  const double ivv = vv > 0.0 ? 1.0 / vv : 0.0, iuu = uu > 0.0 ? 1.0 / uu : 0.0;
  consider(0.0, clamp01(vw * ivv));
  consider(1.0, clamp01((vw + uv) * ivv));
  consider(clamp01(-uw * iuu), 0.0);
  consider(clamp01((uv - uw) * iuu), 1.0);
  return best;
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
  const double ck = svt > L.v_stick ? -L.mu_k * fn / svt : (L.v_stick > 0.0 ? -L.mu_s * fn / L.v_stick : 0.0);
#pragma unroll
  for (int c = 0; c < 3; ++c) F[c] = fn * n[c] + ck * vt[c];
}

// Force of the pair (x, y), x the lower element id, on x; false when not in contact.  u, v: the
// segments' edge vectors, w = x's first node - y's first node; Vx, Vy: end-point velocity
// records (node stride 6), read only for touching pairs.
__device__ __forceinline__ bool pair_force(const ErContactParams &p, const double u[3], const double v[3],
                                           const double w[3], const double *Vx, const double *Vy, double rx,
                                           double ry, double k, double F[3], double &s, double &t) {
  double x[3];
  const double d = sqrt(segment_closest(u, v, w, s, t, x));
  const double gap = d - (rx + ry);
  if (!(gap < 0.0) || d == 0.0) return false;
  double n[3], vr[3];
  const double id = 1.0 / d;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    n[c] = x[c] * id;
    const double va = fma(s, __ldg(Vx + 6 + c), (1.0 - s) * __ldg(Vx + c));
    const double vb = fma(t, __ldg(Vy + 6 + c), (1.0 - t) * __ldg(Vy + c));
    vr[c] = va - vb;
  }
  contact_law(p.law, k, gap, n, vr, F);
  return true;
}

// Half-space n.x >= d on node j of element j (and node j+1 for a rod's last element), added to
// the element's node shares f[0..2] / f[3..5]; returns the nodes in contact.
__device__ __forceinline__ unsigned plane_forces(const ErContactParams &p, int64_t e, int rod, double f[6]) {
  const ErContactLaw &L = p.law;
  const double k = L.k_n > 0.0 ? L.k_n : __ldg(p.kr + rod);
  const double r = __ldg(p.rad + rod);
  const bool last = e + 1 == p.n_elems || __ldg(p.erod + e + 1) != rod;
  unsigned n = 0;
  for (int side = 0; side < (last ? 2 : 1); ++side) {
    const double *x = p.cnode + 6 * (e + rod + side);
    const double X[3] = {x[0], x[1], x[2]};
    const double gap = dot3(L.pn, X) - L.pd - r;
    if (!(gap < 0.0)) continue;
    ++n;
    const double V[3] = {x[3], x[4], x[5]};
    double F[3];
    contact_law(L, k, gap, L.pn, V, F);
#pragma unroll
    for (int c = 0; c < 3; ++c) f[3 * side + c] += F[c];
  }
  return n;
}

// LONG = false: elements with <= ER_CAND_K candidates (their stored list); LONG = true: the
// others, which re-run the broad visit of the last build (same order) -- a separate kernel so the
// common path does not carry the broad visit's registers.
template <bool LONG>
#ifndef ER_NARROW_MINB
#define ER_NARROW_MINB 6
#endif
__global__ void __launch_bounds__(128, LONG ? 4 : ER_NARROW_MINB) hhg_narrow(const ErContactParams p) {
  const int64_t ea = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned n_cont = 0, n_cross = 0, n_plane = 0;
  if (ea < p.n_elems && ((p.cnt[ea] > ER_CAND_K) == LONG)) {
    const int64_t na = ea + __ldg(p.erod + ea);        // first node of element a
    const double *Va = p.cnode + 6 * na + 3;          // velocities: read only on contact
    double A0[3], ua[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { A0[c] = Va[c - 3]; ua[c] = Va[3 + c] - A0[c]; }
    const double ra = __ldg(p.nrad + na), kra = __ldg(p.nkr + na);
    double f[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    // candidates are named by their first node: node order = element order, so the canonical
    // (lower element id first) order is the lower first node
    auto pair = [&](int nb, bool cross) {
      const double *xb = p.cnode + 6 * (int64_t)nb;
      const double *Vb = xb + 3;
      double ub[3], wab[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double b0 = __ldg(xb + c);
        ub[c] = __ldg(xb + 6 + c) - b0;
        wab[c] = A0[c] - b0;
      }
      const double rb = __ldg(p.nrad + nb);
      const double k = p.law.k_n > 0.0 ? p.law.k_n : fmin(kra, __ldg(p.nkr + nb));
      const bool a_first = na < nb;
      // one call site in canonical order (lower element id first): both elements of a pair run the
      // same instructions on the same operands (w changes sign exactly), so their forces are
      // bitwise opposite
      double u[3], v[3], w[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        u[c] = a_first ? ua[c] : ub[c];
        v[c] = a_first ? ub[c] : ua[c];
        w[c] = a_first ? wab[c] : -wab[c];
      }
      double F[3], s, t;
      const bool hit = pair_force(p, u, v, w, a_first ? Va : Vb, a_first ? Vb : Va, a_first ? ra : rb,
                                  a_first ? rb : ra, k, F, s, t);
      if (!hit) return;
      n_cont += (cross || a_first);  // each pair once
      // F acts on the first (lower-id) element at weights (1-s, s); -F on the second at (1-t, t)
      const double w0 = a_first ? 1.0 - s : 1.0 - t, w1 = a_first ? s : t;
      const double sg = a_first ? 1.0 : -1.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        f[c] += w0 * (sg * F[c]);
        f[3 + c] += w1 * (sg * F[c]);
      }
      if (cross) {  // the coarser element b never sees this pair: leave it a record
        ++n_cross;
        const unsigned long long r = atomicAdd(p.ctr + 0, 1ull);
        if (r >= (unsigned long long)p.pcap) { flag_fault(p, 0); return; }
        const double v0 = a_first ? 1.0 - t : 1.0 - s, v1 = a_first ? t : s;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          p.pf[6 * r + c] = v0 * (-sg * F[c]);
          p.pf[6 * r + 3 + c] = v1 * (-sg * F[c]);
        }
        p.psrc[r] = (int32_t)na;
        p.pnext[r] = atomicExch(p.head + nb, (int32_t)r);
      }
    };
    if (!LONG) {
      const int n = p.cnt[ea];
      for (int j = 0; j < n; ++j) {
        const int c = p.cand[j * p.n_elems + ea];
        pair(c & ~ER_CAND_CROSS, (c & ER_CAND_CROSS) != 0);
      }
    } else {
      unsigned sc = 0;
      broad_visit(p, p.qidx[ea], [&](int nb, bool cross, bool) { pair(nb, cross); }, sc);
    }
    if (p.law.plane_on) n_plane = plane_forces(p, ea, (int)(na - ea), f);
#pragma unroll
    for (int c = 0; c < 6; ++c) p.fc[c * p.fs + ea] = f[c];
  }
  n_plane = __reduce_add_sync(0xffffffffu, n_plane);
  if ((threadIdx.x & 31) == 0 && n_plane) atomicAdd(p.ctr + 3, (unsigned long long)n_plane);
  n_cont = __reduce_add_sync(0xffffffffu, n_cont);
  n_cross = __reduce_add_sync(0xffffffffu, n_cross);
  if ((threadIdx.x & 31) == 0) {
    if (n_cont) atomicAdd(p.ctr + 1, (unsigned long long)n_cont);
    if (n_cross) atomicAdd(p.ctr + 2, (unsigned long long)n_cross);
  }
}

constexpr int MAX_CROSS = 64;

// Cross-level records of each coarse element, summed in increasing source-element order.
__global__ void hhg_finish(const ErContactParams p) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.n_elems; e += (int64_t)gridDim.x * blockDim.x) {
    const int rod = __ldg(p.erod + e);
    int h = p.head[e + rod];  // records are filed under the element's first node
    if (h < 0) continue;
    double f[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) f[c] = p.fc[c * p.fs + e];
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
#pragma unroll
    for (int c = 0; c < 6; ++c) p.fc[c * p.fs + e] = f[c];
  }
}

// Ghost rods (contact across GPUs): the caller supplied their node records; a node farther than
// skin/2 from its position at the last list build raises the rebuild flag, as the drift kernel does
// for the own nodes.
__global__ void hhg_ghost_check(const ErContactParams p, int64_t n0, double disp2) {
  bool moved = false;
  for (int64_t n = n0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < p.n_nodes; n += (int64_t)gridDim.x * blockDim.x) {
    double d2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double d = p.cnode[6 * n + c] - p.cbuild[3 * n + c];
      d2 = fma(d, d, d2);
    }
    moved = moved || !(d2 <= disp2);  // also for NaN
  }
  if (__any_sync(0xffffffffu, moved) && (threadIdx.x & 31) == 0) atomicOr(p.rebuild, 1);
}

}  // namespace erc

namespace {

cudaError_t enqueue_build(const ErContactParams &p, void *tmp, size_t tmp_bytes, cudaStream_t st) {
  const int64_t E = p.n_elems, T = 1ll << p.hbits;
  const unsigned g = (unsigned)std::min<int64_t>((E + 255) / 256, 148 * 16);
  const unsigned gq = (unsigned)((E + 127) / 128);
  erc::hhg_reset<<<(unsigned)std::min<int64_t>((T + 255) / 256, 148 * 16), 256, 0, st>>>(p, T);
  erc::hhg_aabb<<<g, 256, 0, st>>>(p);
  erc::hhg_dims<<<1, 32, 0, st>>>(p);
  erc::hhg_keys<<<g, 256, 0, st>>>(p);
  size_t bytes = tmp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, bytes, p.key, p.key_s, p.val, p.val_s, (int)E, 0, p.hbits, st);
  if (e != cudaSuccess) return e;
  erc::hhg_cells<<<g, 256, 0, st>>>(p);
  erc::hhg_table<<<g, 256, 0, st>>>(p);
  erc::hhg_broad<<<gq, 128, 0, st>>>(p);
  erc::hhg_built<<<1, 1, 0, st>>>(p);
  return cudaGetLastError();
}

// Append an IF node (condition set on the device by `cond`) to the capture on `st`; its body is
// captured from `body` on the side stream `side`.
template <class Cond, class Body>
cudaError_t capture_if(cudaStream_t st, cudaStream_t side, Cond &&cond, Body &&body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  if ((e = cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
  cond(h);  // the kernel that sets h, captured on st
  if ((e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd)) != cudaSuccess) return e;
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeIf;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, g, deps, nd, &np)) != cudaSuccess) return e;
  if ((e = cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess) return e;
  cudaGraph_t bg = np.conditional.phGraph_out[0];
  if ((e = cudaStreamBeginCaptureToGraph(side, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return e;
  cudaError_t eb = body(side);
  e = cudaStreamEndCapture(side, &bg);
  return eb != cudaSuccess ? eb : e;
}

}  // namespace

extern "C" {

cudaError_t er_contact_ghost_check(const ErContactParams *pp, int64_t n0, double disp2, cudaStream_t st) {
  if (pp->n_nodes <= n0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>((pp->n_nodes - n0 + 255) / 256, 148 * 8);
  erc::hhg_ghost_check<<<g, 256, 0, st>>>(*pp, n0, disp2);
  return cudaGetLastError();
}

// Temporary-storage bytes of the broad-phase sort (n keys of `bits` bits).
cudaError_t er_contact_tmp_bytes(int64_t n, int bits, size_t *bytes) {
  *bytes = 0;
  return cub::DeviceRadixSort::SortPairs(nullptr, *bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                         (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, bits);
}


// The per-step contact evaluation as one CUDA graph: counters reset, [IF rebuild flag: list build],
// narrow phase, [IF long lists: long-list narrow phase], cross-level gather.  The build (CUB sort
// included) and the long-list pass are skipped on the device when not needed -- no host round trip.
cudaError_t er_contact_graph(const ErContactParams *pp, void *tmp, size_t tmp_bytes, cudaGraphExec_t *exec,
                             int *kernels) {
  const ErContactParams &p = *pp;
  const int64_t E = p.n_elems;
  *exec = nullptr;
  *kernels = 0;
  if (E <= 0) return cudaSuccess;
  cudaStream_t st, side;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking)) != cudaSuccess) { cudaStreamDestroy(st); return e; }
  cudaGraph_t graph = nullptr;
  const int cross = p.nlev > 1;
  const unsigned g = (unsigned)std::min<int64_t>((E + 255) / 256, 148 * 16);
  const unsigned gq = (unsigned)((E + 127) / 128);
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    cudaMemsetAsync(p.ctr, 0, 4 * sizeof(unsigned long long), st);
    if (cross) cudaMemsetAsync(p.head, 0xff, sizeof(int32_t) * p.n_nodes, st);
    e = capture_if(st, side, [&](cudaGraphConditionalHandle h) { erc::hhg_cond_build<<<1, 1, 0, st>>>(p, h); },
                   [&](cudaStream_t s2) { return enqueue_build(p, tmp, tmp_bytes, s2); });
    if (e == cudaSuccess) {
      erc::hhg_narrow<false><<<gq, 128, 0, st>>>(p);
      e = capture_if(st, side, [&](cudaGraphConditionalHandle h) { erc::hhg_cond_long<<<1, 1, 0, st>>>(p, h); },
                     [&](cudaStream_t s2) {
                       erc::hhg_narrow<true><<<gq, 128, 0, s2>>>(p);
                       return cudaGetLastError();
                     });
    }
    if (e == cudaSuccess && cross)
      e = capture_if(st, side, [&](cudaGraphConditionalHandle h) { erc::hhg_cond_cross<<<1, 1, 0, st>>>(p, h); },
                     [&](cudaStream_t s2) {
                       erc::hhg_finish<<<g, 256, 0, s2>>>(p);
                       return cudaGetLastError();
                     });
    cudaError_t e2 = cudaStreamEndCapture(st, &graph);
    if (e == cudaSuccess) e = e2;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(side);
  cudaStreamDestroy(st);
  *kernels = 3 + cross;  // kernels every step runs (narrow, conditions)
  return e;
}

// One contact evaluation at the positions/velocities in p.cnode: fills p.fc.  Stream-ordered, no
// host synchronisation.  With `exec` (er_contact_graph) one graph launch; else the same work as
// plain launches, the build kernels returning at once unless the device flag is set.
cudaError_t er_contact_eval(const ErContactParams *pp, void *tmp, size_t tmp_bytes, cudaGraphExec_t exec,
                            cudaStream_t st, int64_t *launches, int graph_kernels) {
  const ErContactParams &p = *pp;
  const int64_t E = p.n_elems;
  if (E <= 0) return cudaSuccess;
  if (exec) {
    *launches += graph_kernels;
    return cudaGraphLaunch(exec, st);
  }
  cudaError_t e;
  if ((e = cudaMemsetAsync(p.ctr, 0, 4 * sizeof(unsigned long long), st)) != cudaSuccess) return e;
  const int cross = p.nlev > 1;
  if (cross && (e = cudaMemsetAsync(p.head, 0xff, sizeof(int32_t) * p.n_nodes, st)) != cudaSuccess) return e;
  const unsigned g = (unsigned)std::min<int64_t>((E + 255) / 256, 148 * 16);
  const unsigned gq = (unsigned)((E + 127) / 128);
  if ((e = enqueue_build(p, tmp, tmp_bytes, st)) != cudaSuccess) return e;
  erc::hhg_narrow<false><<<gq, 128, 0, st>>>(p);
  erc::hhg_narrow<true><<<gq, 128, 0, st>>>(p);
  *launches += 10;
  if (cross) {
    erc::hhg_finish<<<g, 256, 0, st>>>(p);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // extern "C"
