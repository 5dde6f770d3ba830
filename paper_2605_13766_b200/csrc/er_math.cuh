// er_math.cuh -- device math (L1) of the rod step: the SO(3) exponential and log maps in
// registers.  Independent of oracle/ (no shared code); both follow PAPER.md:238-239 and the
// sign-locked readings of SURVEY §8 C.2 / DESIGN.md §3 #2.
#pragma once

namespace er {

// Series coefficients in constant memory: DFMA reads them as c[][] operands directly.
// sin(t)/t and (1 - cos t)/t^2 in x = t^2 (Taylor), asin(s)/s in x = s^2.
__constant__ double kSinc[9] = {1.0, -1.0 / 6.0, 1.0 / 120.0, -1.0 / 5040.0, 1.0 / 362880.0, -1.0 / 39916800.0,
                                1.0 / 6227020800.0, -1.0 / 1307674368000.0, 1.0 / 355687428096000.0};
__constant__ double kCosc[9] = {0.5, -1.0 / 24.0, 1.0 / 720.0, -1.0 / 40320.0, 1.0 / 3628800.0, -1.0 / 479001600.0,
                                1.0 / 87178291200.0, -1.0 / 20922789888000.0, 1.0 / 6402373705728000.0};
__constant__ double kAsinc[12] = {1.0, 1.0 / 6.0, 3.0 / 40.0, 5.0 / 112.0, 35.0 / 1152.0, 63.0 / 2816.0,
                                  231.0 / 13312.0, 143.0 / 10240.0, 6435.0 / 557056.0, 12155.0 / 1245184.0,
                                  46189.0 / 5505024.0, 88179.0 / 12058624.0};

template <int NT>
__device__ __forceinline__ double horner(const double *c, double x) {
  double p = c[NT - 1];
#pragma unroll
  for (int k = NT - 2; k >= 0; --k) p = fma(p, x, c[k]);
  return p;
}

// Truncation errors (relative, all < 2^-53 / 8):
//  sinc/cosc: x < 1e-8: 2 terms (x^2/120 < 1e-18);  x < 1e-4: 4 terms (x^4/362880 < 3e-22);
//             x < 0.25: 9 terms (x^9/19! < 3e-23).
//  asinc:     x < 1e-8: 2 terms (3x^2/40 < 1e-17);  x < 1e-4: 4 terms (35x^4/1152 < 4e-18);
//             x < 0.04: 12 terms (< 3e-18).
__device__ __forceinline__ void sinc_cosc(double x, double &a, double &b) {
  if (x < 1e-8) {
    a = horner<2>(kSinc, x);
    b = horner<2>(kCosc, x);
  } else if (x < 1e-4) {
    a = horner<4>(kSinc, x);
    b = horner<4>(kCosc, x);
  } else {
    a = horner<9>(kSinc, x);
    b = horner<9>(kCosc, x);
  }
}
__device__ __forceinline__ double asinc_x(double x) {
  if (x < 1e-8) return horner<2>(kAsinc, x);
  if (x < 1e-4) return horner<4>(kAsinc, x);
  return horner<12>(kAsinc, x);
}

// 1/x and 1/sqrt(x) for finite positive normal x without the IEEE slow paths: hardware
// approximation (MUFU.RCP64H / MUFU.RSQ64H, ~2^-20) refined by Newton steps to <= 1 ulp.
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  double e = fma(-hx * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-hx * y, y, 0.5);
  return fma(y, e, y);
}

// d3 = d1 x d2: the third director row, rebuilt from the two stored rows (er_layout.h).  Written
// with explicit fma so every kernel (and er_get_state) computes the same bits.
__device__ __forceinline__ void complete_d3(double Q[9]) {
  Q[6] = fma(Q[1], Q[5], -Q[2] * Q[4]);
  Q[7] = fma(Q[2], Q[3], -Q[0] * Q[5]);
  Q[8] = fma(Q[0], Q[4], -Q[1] * Q[3]);
}

// One component of complete_d3 from components strided by st (layout conversion); the same
// expressions, so the same bits.
__device__ __forceinline__ double d3_component(int j, const double *q, int64_t st) {
  const double q0 = q[0], q1 = q[st], q2 = q[2 * st], q3 = q[3 * st], q4 = q[4 * st], q5 = q[5 * st];
  return j == 0 ? fma(q1, q5, -q2 * q4) : j == 1 ? fma(q2, q3, -q0 * q5) : fma(q0, q4, -q1 * q3);
}

// Q <- rot(v) Q with rot(v) = exp(-[v]x) = I - a [v]x + b [v]x^2 (Rodrigues; the in-place SO(3)
// rotation of PAPER.md:30).  Rows of Q are the directors.  Rows d1, d2 are rotated, d3 is rebuilt
// as d1 x d2 (equal in exact arithmetic for a proper rotation).  v = 0 leaves Q bit-identical
// when it already holds d3 = complete_d3(d1, d2), which every kernel maintains.
// complete = false skips rebuilding d3 (the caller's last rotation before only d1, d2 are stored).
__device__ __forceinline__ void rotate_inplace(double Q[9], double vx, double vy, double vz, bool complete = true) {
  const double x = fma(vx, vx, fma(vy, vy, vz * vz));
  double a, b;
  if (x < 0.25) {
    sinc_cosc(x, a, b);
  } else {
    const double th = sqrt(x);
    double s, c;
    sincos(th, &s, &c);
    a = s / th;
    b = (1.0 - c) / x;
  }
  const double c1 = fma(-b, x, 1.0);
  const double bx = b * vx, by = b * vy, bz = b * vz;
  const double ax = a * vx, ay = a * vy, az = a * vz;
  const double s01 = bx * vy, s02 = bx * vz, s12 = by * vz;
  const double R00 = fma(bx, vx, c1), R11 = fma(by, vy, c1), R22 = fma(bz, vz, c1);
  const double R01 = s01 + az, R10 = s01 - az;
  const double R02 = s02 - ay, R20 = s02 + ay;
  const double R12 = s12 + ax, R21 = s12 - ax;
  (void)R20; (void)R21; (void)R22;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double q0 = Q[c], q1 = Q[3 + c], q2 = Q[6 + c];
    Q[c] = fma(R00, q0, fma(R01, q1, R02 * q2));
    Q[3 + c] = fma(R10, q0, fma(R11, q1, R12 * q2));
  }
  if (complete) complete_d3(Q);
}

__device__ __forceinline__ double dot3(const double *a, const double *b) {
  return fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2]));
}

// v = logrot(Q Qp^T) (inverse Rodrigues): the discrete kappa_k * Dh_k with
// Q = Q_k, Qp = Q_{k-1}.  Returns c = cos(theta) and s2 = sin^2(theta) for the antipodal check.
__device__ __forceinline__ void logrot_pair(const double Q[9], const double Qp[9], double v[3],
                                            double &c, double &s2) {
  const double tr = dot3(Q, Qp) + dot3(Q + 3, Qp + 3) + dot3(Q + 6, Qp + 6);
  const double w0 = dot3(Q + 6, Qp + 3) - dot3(Q + 3, Qp + 6);  // R21 - R12
  const double w1 = dot3(Q, Qp + 6) - dot3(Q + 6, Qp);          // R02 - R20
  const double w2 = dot3(Q + 3, Qp) - dot3(Q, Qp + 3);          // R10 - R01
  s2 = 0.25 * fma(w0, w0, fma(w1, w1, w2 * w2));
  c = 0.5 * (tr - 1.0);
  double f;
  if (c > 0.0 && s2 < 0.04) {
    f = 0.5 * asinc_x(s2);  // theta/(2 sin theta) with sin theta = s
  } else {
    const double s = sqrt(s2);
    f = atan2(s, c) / (2.0 * s);
  }
  v[0] = -f * w0;
  v[1] = -f * w1;
  v[2] = -f * w2;
}

}  // namespace er
