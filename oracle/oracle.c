/*
 * oracle.c -- CPU ORACLE for the discrete Cosserat rod step (arxiv 2605.13766).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
 * (`cpu_baseline` and `--impl reference`) may load or run it.  Shares no code,
 * header, table or constant with the CUDA path (include/er.h,
 * paper_2605_13766_b200/csrc/).
 *
 * What it computes (PAPER.md "Methods / Cosserat rod dynamics", lines 231-258):
 *   Eq. (1a)  rho A d2r/dt2 = d/ds( Q^T S sigma / e ) + f
 *   Eq. (1b)  rho I/e dw/dt = d/ds(B kappa/e^3) + kappa x B kappa / e^3 + Q t x S sigma
 *                             + (rho I w / e) x w + (rho I w / e^2) de/dt + c
 *   strains   sigma = Q(r' - d3), kappa = ax(Q dQ^T/ds), e = |r'|
 *   w         = ax(Q dQ^T/dt)
 * discretised on the staggered node / element / Voronoi scheme (SURVEY §8 C.1,
 * reading C.4 #1) and advanced by position Verlet drift(h/2)-kick(h)-drift(h/2)
 * with constraints after every stage.
 * All readings of silent/ambiguous passages are SURVEY §8 C.4 and are listed in
 * DESIGN.md §3.
 *
 * Contact: exhaustive O(E^2) pair search,
 * exact segment-segment closest points, penalty normal force + regularised Coulomb
 * friction, optional half-space -- reading DESIGN.md §3 #27 (the paper's formulas
 * are in its missing supplement).  Pinned by tests/test_oracle_contact.py.
 *
 * Deliberately plain: no blocking, no fusion, no reordering beyond the algorithm
 * as written; every intermediate of C.3 is materialised per rod.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.14159265358979323846

/* ---------------------------------------------------------------- small 3-vector helpers */
static void v_sub(const double *a, const double *b, double *o) { o[0] = a[0] - b[0]; o[1] = a[1] - b[1]; o[2] = a[2] - b[2]; }
static double v_dot(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void v_cross(const double *a, const double *b, double *o) {
  double x = a[1] * b[2] - a[2] * b[1];
  double y = a[2] * b[0] - a[0] * b[2];
  double z = a[0] * b[1] - a[1] * b[0];
  o[0] = x; o[1] = y; o[2] = z;
}
/* y = M x (M row-major 3x3) */
static void m_vec(const double *M, const double *x, double *y) {
  double a = M[0] * x[0] + M[1] * x[1] + M[2] * x[2];
  double b = M[3] * x[0] + M[4] * x[1] + M[5] * x[2];
  double c = M[6] * x[0] + M[7] * x[1] + M[8] * x[2];
  y[0] = a; y[1] = b; y[2] = c;
}
/* y = M^T x */
static void mt_vec(const double *M, const double *x, double *y) {
  double a = M[0] * x[0] + M[3] * x[1] + M[6] * x[2];
  double b = M[1] * x[0] + M[4] * x[1] + M[7] * x[2];
  double c = M[2] * x[0] + M[5] * x[1] + M[8] * x[2];
  y[0] = a; y[1] = b; y[2] = c;
}
/* C = A B */
static void m_mul(const double *A, const double *B, double *C) {
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      T[3 * i + j] = A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
  memcpy(C, T, sizeof T);
}
/* C = A B^T */
static void m_mul_t(const double *A, const double *B, double *C) {
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      T[3 * i + j] = A[3 * i + 0] * B[3 * j + 0] + A[3 * i + 1] * B[3 * j + 1] + A[3 * i + 2] * B[3 * j + 2];
  memcpy(C, T, sizeof T);
}

/* ---------------------------------------------------------------- SO(3) maps */

/* [v]x, so that [v]x u = v x u. */
void orc_skew(const double v[3], double W[9]) {
  W[0] = 0.0;   W[1] = -v[2]; W[2] = v[1];
  W[3] = v[2];  W[4] = 0.0;   W[5] = -v[0];
  W[6] = -v[1]; W[7] = v[0];  W[8] = 0.0;
}

/* ax(U)_i = eps_ijk U_kj / 2   (written out as the index sum). */
void orc_ax(const double U[9], double v[3]) {
  for (int i = 0; i < 3; ++i) {
    double s = 0.0;
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k) {
        int eps = 0;
        if (i != j && j != k && i != k) eps = ((j - i + 3) % 3 == 1) ? 1 : -1;
        if (eps) s += eps * U[3 * k + j];
      }
    v[i] = 0.5 * s;
  }
}

/* rot(v) = exp(-[v]x) = I - a [v]x + b [v]x^2, theta = |v|, a = sin(theta)/theta,
 * b = (1 - cos theta)/theta^2 = (1/2) (sin(theta/2)/(theta/2))^2.
 * Sign fixed by w = ax(Q dQ^T/dt): Q(t+h) = exp(-h[w]x) Q(t)
 * (SURVEY §8 C.2, C.4 #2).  Series for theta < 1e-4 (C.4 #19). */
void orc_rot(const double v[3], double R[9]) {
  double th2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  double th = sqrt(th2);
  double a, b;
  if (th < 1e-4) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
  } else {
    a = sin(th) / th;
    double h = 0.5 * th;
    double sh = sin(h) / h;
    b = 0.5 * sh * sh;
  }
  double K[9], K2[9];
  orc_skew(v, K);
  m_mul(K, K, K2);
  for (int i = 0; i < 9; ++i) R[i] = ((i % 4) == 0 ? 1.0 : 0.0) - a * K[i] + b * K2[i];
}

/* logrot = rot^{-1} for rotation angle < pi:
 * w = (R32-R23, R13-R31, R21-R12), s = |w|/2, c = (tr R - 1)/2, theta = atan2(s, c),
 * v = -(theta/(2 s)) w, with theta/(2s) -> (1 + s^2/6)/2 for s < 1e-8. */
int orc_logrot(const double R[9], double v[3]) {
  double w[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
  double s = 0.5 * sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  double c = 0.5 * (R[0] + R[4] + R[8] - 1.0);
  double th = atan2(s, c);
  double f;
  int fault = 0;
  if (th >= PI - 1e-6) fault = ORC_F_ANTIPODAL;          /* SPEC.md:113 reading */
  if (s < 1e-8 && c > 0.0) f = 0.5 * (1.0 + s * s / 6.0);
  else f = th / (2.0 * s);
  v[0] = -f * w[0]; v[1] = -f * w[1]; v[2] = -f * w[2];
  return fault;
}

/* ---------------------------------------------------------------- per-rod context */

typedef struct {
  int32_t N;
  int64_t e0, n0, v0;        /* element / node / Voronoi offsets of this rod */
  /* per element j */
  double *lhat, *S, *B, *J, *me;
  /* per node i */
  double *m;
  /* per Voronoi k (index k in 1..N-1, arrays sized N+1) */
  double *Dh, *Bv;
  double nu, vmax;
  int clamp, tip_node;
  /* scratch */
  double *ell, *l, *tg, *e, *edot, *sig, *nbar, *nlab, *kap, *mbar, *beta, *eps, *F, *C, *a, *al;
  double rfix[3], Qfix[9];
} rod_ctx;

static double matv(const orc_problem *P, const double *arr, int32_t rod, int64_t j) {
  return P->material_per_rod ? arr[rod] : arr[j];
}

static void ctx_alloc(rod_ctx *c, int32_t Nmax) {
  size_t n = (size_t)Nmax + 1;
  double *blk = (double *)calloc(n * 64, sizeof(double));
  double *p = blk;
#define TAKE(x, k) do { c->x = p; p += (k) * n; } while (0)
  TAKE(lhat, 1); TAKE(S, 3); TAKE(B, 3); TAKE(J, 3); TAKE(me, 1); TAKE(m, 1); TAKE(Dh, 1); TAKE(Bv, 3);
  TAKE(ell, 3); TAKE(l, 1); TAKE(tg, 3); TAKE(e, 1); TAKE(edot, 1); TAKE(sig, 3); TAKE(nbar, 3);
  TAKE(nlab, 3); TAKE(kap, 3); TAKE(mbar, 3); TAKE(beta, 3); TAKE(eps, 1); TAKE(F, 3); TAKE(C, 3);
  TAKE(a, 3); TAKE(al, 3);
#undef TAKE
}
static void ctx_free(rod_ctx *c) { free(c->lhat); }

/* Derived constants (PAPER.md:239 with the hat convention of C.4 #5):
 * S_j = diag(alpha_c G A, alpha_c G A, E A); B_j = diag(E I1, E I2, G(I1+I2));
 * J_j = rho lhat_j diag(I1, I2, I1+I2); m_i = (rho A lhat)_{i-1}/2 + (rho A lhat)_i/2 (C.4 #10);
 * Dh_k = (lhat_{k-1}+lhat_k)/2 (distance of the element centres);
 * Bv_k = 2 Dh_k / (lhat_{k-1}/B_{k-1} + lhat_k/B_k): the Voronoi domain's two half elements act in
 * series under a uniform moment, so its stiffness is the compliance mean (DESIGN §3 #9; equals B for
 * a uniform rod, i.e. in every BASELINE config). */
static void ctx_setup(const orc_problem *P, int32_t rod, int64_t e0, rod_ctx *c) {
  int32_t N = P->n_elems[rod];
  c->N = N;
  c->e0 = e0;
  c->n0 = e0 + rod;
  c->v0 = e0 - rod;
  for (int32_t j = 0; j < N; ++j) {
    int64_t g = e0 + j;
    double rho = matv(P, P->density, rod, g), A = matv(P, P->area, rod, g);
    double I1 = matv(P, P->I1, rod, g), I2 = matv(P, P->I2, rod, g);
    double E = matv(P, P->youngs, rod, g), G = matv(P, P->shear_mod, rod, g);
    double ac = matv(P, P->alpha_c, rod, g);
    double lh = P->rest_lengths[g];
    c->lhat[j] = lh;
    c->S[3 * j + 0] = ac * G * A; c->S[3 * j + 1] = ac * G * A; c->S[3 * j + 2] = E * A;
    c->B[3 * j + 0] = E * I1; c->B[3 * j + 1] = E * I2; c->B[3 * j + 2] = G * (I1 + I2);
    c->J[3 * j + 0] = rho * lh * I1; c->J[3 * j + 1] = rho * lh * I2; c->J[3 * j + 2] = rho * lh * (I1 + I2);
    c->me[j] = rho * A * lh;
  }
  for (int32_t i = 0; i <= N; ++i) {
    double m = 0.0;
    if (i > 0) m += 0.5 * c->me[i - 1];
    if (i < N) m += 0.5 * c->me[i];
    c->m[i] = m;
  }
  for (int32_t k = 1; k < N; ++k) {
    c->Dh[k] = 0.5 * (c->lhat[k - 1] + c->lhat[k]);
    for (int q = 0; q < 3; ++q)
      c->Bv[3 * k + q] = (2.0 * c->Dh[k]) / (c->lhat[k - 1] / c->B[3 * (k - 1) + q] + c->lhat[k] / c->B[3 * k + q]);
  }
  c->nu = P->damping ? P->damping[rod] : 0.0;
  {
    double E = matv(P, P->youngs, rod, e0), rho = matv(P, P->density, rod, e0);
    c->vmax = 1e6 * sqrt(E / rho);                       /* SPEC.md:213 reading */
  }
  c->clamp = P->clamp ? P->clamp[rod] : -1;
  c->tip_node = (c->clamp == 1) ? 0 : N;               /* C.4 #16 */
}

/* kappa0_k(t) = static rest curvature + A sin(2 pi (s_k/L - f t)) on one component,
 * s_k = sum_{j<k} lhat_j (C.4 #14). */
static void rest_kappa_at(const orc_problem *P, int32_t rod, const rod_ctx *c, int32_t k, double t, double *k0) {
  k0[0] = k0[1] = k0[2] = 0.0;
  if (P->rest_kappa) {
    const double *src = P->rest_kappa + 3 * (c->v0 + k - 1);
    k0[0] = src[0]; k0[1] = src[1]; k0[2] = src[2];
  }
  if (P->act_A) {
    double s = 0.0;
    for (int32_t j = 0; j < k; ++j) s += c->lhat[j];
    k0[P->act_component] += P->act_A[rod] * sin(2.0 * PI * (s / P->act_L[rod] - P->act_f[rod] * t));
  }
}

/* b(t): b(0) rotated by the angle b_omega t about the unit axis a (Rodrigues' rotation formula,
 * right-handed): b = b0 cos + (a x b0) sin + a (a . b0)(1 - cos).  a = 0 means the lab z axis. */
/* Muscular torque at interior node k ("internal (net-zero) muscular torques as a
 * traveling wave with period T and wavelength L"; reading DESIGN §3 #26):
 * tau_k(t) = A sin(2 pi (t/T - s_k/lambda) + phi0) about local axis `musc_component`,
 * s_k = sum_{j<k} lhat_j.  Applied as a couple pair: +tau_k on element k, -tau_k on element k-1. */
static double muscle_tau(const orc_problem *P, int32_t rod, const rod_ctx *c, int32_t k, double t) {
  double s = 0.0;
  for (int32_t j = 0; j < k; ++j) s += c->lhat[j];
  return P->musc_A[rod] * sin(2.0 * PI * (t / P->musc_T[rod] - s / P->musc_lambda[rod]) + P->musc_phi[rod]);
}

static void b_field_at(const orc_problem *P, double t, double *b) {
  double a[3] = {P->b_axis[0], P->b_axis[1], P->b_axis[2]};
  double na = sqrt(v_dot(a, a));
  if (na == 0.0) { a[0] = 0.0; a[1] = 0.0; a[2] = 1.0; na = 1.0; }
  for (int q = 0; q < 3; ++q) a[q] /= na;
  double ph = P->b_omega * t;
  double cs = cos(ph), sn = sin(ph);
  double axb[3];
  v_cross(a, P->b_field, axb);
  double ad = v_dot(a, P->b_field);
  for (int q = 0; q < 3; ++q) b[q] = P->b_field[q] * cs + axb[q] * sn + a[q] * ad * (1.0 - cs);
}

/* ---------------------------------------------------------------- strains (C.3 steps 2-3) */

int orc_rod_strains(int32_t N, const double *lhat, const double *pos, const double *dirs,
                    double *e, double *sigma, double *kappa) {
  int fault = 0;
  double *l = (double *)malloc(sizeof(double) * (size_t)N);
  for (int32_t j = 0; j < N; ++j) {
    double ell[3], t[3], Qt[3];
    v_sub(pos + 3 * (j + 1), pos + 3 * j, ell);
    l[j] = sqrt(v_dot(ell, ell));
    for (int q = 0; q < 3; ++q) t[q] = ell[q] / l[j];
    e[j] = l[j] / lhat[j];
    m_vec(dirs + 9 * j, t, Qt);                          /* sigma = e Q t - e3 (C.4 #3) */
    sigma[3 * j + 0] = e[j] * Qt[0];
    sigma[3 * j + 1] = e[j] * Qt[1];
    sigma[3 * j + 2] = e[j] * Qt[2] - 1.0;
  }
  for (int32_t k = 1; k < N; ++k) {
    double R[9], v[3];
    double Dh = 0.5 * (lhat[k - 1] + lhat[k]);
    m_mul_t(dirs + 9 * k, dirs + 9 * (k - 1), R);        /* kappa = logrot(Q_k Q_{k-1}^T)/Dh */
    fault |= orc_logrot(R, v);
    for (int q = 0; q < 3; ++q) kappa[3 * (k - 1) + q] = v[q] / Dh;
  }
  free(l);
  return fault;
}

/* ---------------------------------------------------------------- dynamics (C.3 steps 2-6) */

static int rod_dynamics(const orc_problem *P, int32_t rod, rod_ctx *c, const double *r, const double *v,
                        const double *Q, const double *w, double t, const double *Fext) {
  const int32_t N = c->N;
  int fault = 0;
  const double e3[3] = {0.0, 0.0, 1.0};
  /* 2. kinematics */
  for (int32_t j = 0; j < N; ++j) {
    double dv[3];
    v_sub(r + 3 * (j + 1), r + 3 * j, c->ell + 3 * j);
    c->l[j] = sqrt(v_dot(c->ell + 3 * j, c->ell + 3 * j));
    for (int q = 0; q < 3; ++q) c->tg[3 * j + q] = c->ell[3 * j + q] / c->l[j];
    c->e[j] = c->l[j] / c->lhat[j];
    if (!(c->e[j] >= 1e-12)) fault |= ORC_F_DEGENERATE;
    v_sub(v + 3 * (j + 1), v + 3 * j, dv);
    c->edot[j] = v_dot(c->tg + 3 * j, dv) / c->lhat[j];     /* de/dt */
  }
  for (int32_t k = 1; k < N; ++k) c->eps[k] = (0.5 * (c->l[k - 1] + c->l[k])) / c->Dh[k];
  /* 3. strains */
  for (int32_t j = 0; j < N; ++j) {
    double Qt[3];
    m_vec(Q + 9 * j, c->tg + 3 * j, Qt);
    for (int q = 0; q < 3; ++q) c->sig[3 * j + q] = c->e[j] * Qt[q] - e3[q];
  }
  for (int32_t k = 1; k < N; ++k) {
    double R[9], vv[3];
    m_mul_t(Q + 9 * k, Q + 9 * (k - 1), R);
    fault |= orc_logrot(R, vv);
    for (int q = 0; q < 3; ++q) c->kap[3 * k + q] = vv[q] / c->Dh[k];
  }
  /* 4. stresses */
  for (int32_t j = 0; j < N; ++j) {
    double d[3];
    for (int q = 0; q < 3; ++q) {
      double s0 = P->rest_sigma ? P->rest_sigma[3 * (c->e0 + j) + q] : 0.0;
      d[q] = c->sig[3 * j + q] - s0;
      c->nbar[3 * j + q] = c->S[3 * j + q] * d[q] / c->e[j];
    }
    mt_vec(Q + 9 * j, c->nbar + 3 * j, c->nlab + 3 * j);    /* n = Q^T nbar */
  }
  for (int32_t k = 1; k < N; ++k) {
    double k0[3];
    rest_kappa_at(P, rod, c, k, t, k0);
    double e3k = c->eps[k] * c->eps[k] * c->eps[k];
    for (int q = 0; q < 3; ++q) c->mbar[3 * k + q] = c->Bv[3 * k + q] * (c->kap[3 * k + q] - k0[q]) / e3k;
    v_cross(c->kap + 3 * k, c->mbar + 3 * k, c->beta + 3 * k);
    for (int q = 0; q < 3; ++q) c->beta[3 * k + q] *= c->Dh[k];
  }
  /* 5. forces: F_i = n_i - n_{i-1} (zero padded) + m_i g + contact + tip + f_i; a_i = F_i/m_i - nu v_i */
  for (int32_t i = 0; i <= N; ++i) {
    for (int q = 0; q < 3; ++q) {
      double f = 0.0;
      if (i < N) f += c->nlab[3 * i + q];
      if (i > 0) f -= c->nlab[3 * (i - 1) + q];
      f += c->m[i] * P->gravity[q];
      if (Fext) f += Fext[3 * i + q];                       /* contact forces (NEXT-4) */
      if (P->tip_force && i == c->tip_node) f += P->tip_force[3 * rod + q];
      if (P->ext_force) f += P->ext_force[3 * (c->n0 + i) + q];   /* f of Eq. (1a) */
      c->F[3 * i + q] = f;
      c->a[3 * i + q] = f / c->m[i] - c->nu * v[3 * i + q];
    }
  }
  /* 6. couples */
  double b[3] = {0.0, 0.0, 0.0};
  if (P->magnetization) b_field_at(P, t, b);
  for (int32_t j = 0; j < N; ++j) {
    double Cj[3], tmp[3], Qt[3], Sd[3], Jw[3];
    for (int q = 0; q < 3; ++q) {
      double mn = (j + 1 <= N - 1) ? c->mbar[3 * (j + 1) + q] : 0.0;
      double mc = (j >= 1) ? c->mbar[3 * j + q] : 0.0;
      double bn = (j + 1 <= N - 1) ? c->beta[3 * (j + 1) + q] : 0.0;
      double bc = (j >= 1) ? c->beta[3 * j + q] : 0.0;
      Cj[q] = (mn - mc) + 0.5 * (bn + bc);                 /* bend/twist difference + average */
    }
    m_vec(Q + 9 * j, c->tg + 3 * j, Qt);                   /* shear torque lhat (Q t) x S(sigma - sigma0) */
    for (int q = 0; q < 3; ++q) {
      double s0 = P->rest_sigma ? P->rest_sigma[3 * (c->e0 + j) + q] : 0.0;
      Sd[q] = c->S[3 * j + q] * (c->sig[3 * j + q] - s0);
    }
    v_cross(Qt, Sd, tmp);
    for (int q = 0; q < 3; ++q) Cj[q] += c->lhat[j] * tmp[q];
    for (int q = 0; q < 3; ++q) Jw[q] = c->J[3 * j + q] * w[3 * j + q];
    for (int q = 0; q < 3; ++q) tmp[q] = Jw[q] / c->e[j];  /* Lagrangian transport (J w / e) x w */
    v_cross(tmp, w + 3 * j, tmp);
    for (int q = 0; q < 3; ++q) Cj[q] += tmp[q];
    for (int q = 0; q < 3; ++q) Cj[q] += Jw[q] / (c->e[j] * c->e[j]) * c->edot[j];  /* unsteady dilatation */
    if (P->musc_A) {                                        /* muscular couple pair */
      if (j >= 1) Cj[P->musc_component] += muscle_tau(P, rod, c, j, t);
      if (j + 1 <= N - 1) Cj[P->musc_component] -= muscle_tau(P, rod, c, j + 1, t);
    }
    if (P->magnetization) {                                 /* c_mag = m x (Q b(t)) */
      double Qb[3], mb[3];
      m_vec(Q + 9 * j, b, Qb);
      v_cross(P->magnetization + 3 * (c->e0 + j), Qb, mb);
      for (int q = 0; q < 3; ++q) Cj[q] += c->lhat[j] * mb[q];
    }
    if (P->ext_couple)                                      /* c-bar of Eq. (1b) */
      for (int q = 0; q < 3; ++q) Cj[q] += P->ext_couple[3 * (c->e0 + j) + q];
    for (int q = 0; q < 3; ++q) {
      c->C[3 * j + q] = Cj[q];
      c->al[3 * j + q] = c->e[j] / c->J[3 * j + q] * Cj[q] - c->nu * w[3 * j + q];
    }
  }
  return fault;
}

/* ---------------------------------------------------------------- stages */

static void stage_drift(rod_ctx *c, double *r, const double *v, double *Q, const double *w, double h2) {
  for (int32_t i = 0; i <= c->N; ++i)
    for (int q = 0; q < 3; ++q) r[3 * i + q] += h2 * v[3 * i + q];
  for (int32_t j = 0; j < c->N; ++j) {
    double hv[3] = {h2 * w[3 * j + 0], h2 * w[3 * j + 1], h2 * w[3 * j + 2]};
    double R[9];
    orc_rot(hv, R);
    m_mul(R, Q + 9 * j, Q + 9 * j);                        /* Q <- rot(h w) Q (C.2) */
  }
}

static void clamp_pose(const rod_ctx *c, double *r, double *Q) {
  if (c->clamp == 0) { memcpy(r, c->rfix, sizeof c->rfix); memcpy(Q, c->Qfix, sizeof c->Qfix); }
  if (c->clamp == 1) { memcpy(r + 3 * c->N, c->rfix, sizeof c->rfix); memcpy(Q + 9 * (c->N - 1), c->Qfix, sizeof c->Qfix); }
}
static void clamp_rates(const rod_ctx *c, double *v, double *w) {
  if (c->clamp == 0) { memset(v, 0, 3 * sizeof(double)); memset(w, 0, 3 * sizeof(double)); }
  if (c->clamp == 1) { memset(v + 3 * c->N, 0, 3 * sizeof(double)); memset(w + 3 * (c->N - 1), 0, 3 * sizeof(double)); }
}

static int rod_check(const rod_ctx *c, const double *r, const double *v, const double *Q, const double *w) {
  int fault = 0;
  for (int32_t i = 0; i <= c->N; ++i) {
    for (int q = 0; q < 3; ++q)
      if (!isfinite(r[3 * i + q]) || !isfinite(v[3 * i + q])) fault |= ORC_F_NONFINITE;
    if (sqrt(v_dot(v + 3 * i, v + 3 * i)) > c->vmax) fault |= ORC_F_OVERSPEED;
  }
  for (int32_t j = 0; j < c->N; ++j) {
    for (int q = 0; q < 9; ++q) if (!isfinite(Q[9 * j + q])) fault |= ORC_F_NONFINITE;
    for (int q = 0; q < 3; ++q) if (!isfinite(w[3 * j + q])) fault |= ORC_F_NONFINITE;
  }
  return fault;
}

static int32_t max_elems(const orc_problem *P) {
  int32_t m = 1;
  for (int32_t r = 0; r < P->n_rods; ++r) if (P->n_elems[r] > m) m = P->n_elems[r];
  return m;
}

int orc_rod_loads(const orc_problem *P, int32_t rod, const double *pos, const double *vel,
                  const double *dirs, const double *omega, double t,
                  double *F, double *C, double *a, double *alpha) {
  int64_t e0 = 0;
  for (int32_t q = 0; q < rod; ++q) e0 += P->n_elems[q];
  rod_ctx c;
  ctx_alloc(&c, P->n_elems[rod]);
  ctx_setup(P, rod, e0, &c);
  int fault = rod_dynamics(P, rod, &c, pos, vel, dirs, omega, t, NULL);
  int32_t N = c.N;
  memcpy(F, c.F, sizeof(double) * 3 * (size_t)(N + 1));
  memcpy(a, c.a, sizeof(double) * 3 * (size_t)(N + 1));
  memcpy(C, c.C, sizeof(double) * 3 * (size_t)N);
  memcpy(alpha, c.al, sizeof(double) * 3 * (size_t)N);
  ctx_free(&c);
  return fault;
}

/* One rod, one stage; stage 1/3 = drift h/2 + pose constraint, stage 2 = kick + rate constraint. */
static int rod_stage(const orc_problem *P, int32_t rod, rod_ctx *c, int stage, double *pos, double *vel,
                     double *dirs, double *omega, double h, double t_half, const double *Fext) {
  double *r = pos + 3 * c->n0, *v = vel + 3 * c->n0, *Q = dirs + 9 * c->e0, *w = omega + 3 * c->e0;
  int fault = 0;
  if (stage == 1 || stage == 3) {
    stage_drift(c, r, v, Q, w, 0.5 * h);
    clamp_pose(c, r, Q);
  } else {
    fault |= rod_dynamics(P, rod, c, r, v, Q, w, t_half, Fext ? Fext + 3 * c->n0 : NULL);
    for (int32_t i = 0; i <= c->N; ++i)
      for (int q = 0; q < 3; ++q) v[3 * i + q] += h * c->a[3 * i + q];
    for (int32_t j = 0; j < c->N; ++j)
      for (int q = 0; q < 3; ++q) w[3 * j + q] += h * c->al[3 * j + q];
    clamp_rates(c, v, w);
  }
  if (stage == 3) fault |= rod_check(c, r, v, Q, w);
  return fault;
}

int orc_step(const orc_problem *P, double *pos, double *vel, double *dirs, double *omega,
             double *t, int64_t n_steps, double dt, int32_t protocol,
             int64_t *bad_rod, int32_t *fault_out) {
  if (!(dt > 0.0)) return ORC_EINVAL;
  const int32_t R = P->n_rods;
  int64_t *eoff = (int64_t *)calloc((size_t)R + 1, sizeof(int64_t));
  double *rfix = (double *)calloc((size_t)R * 3 + 3, sizeof(double));
  double *Qfix = (double *)calloc((size_t)R * 9 + 9, sizeof(double));
  rod_ctx c;
  ctx_alloc(&c, max_elems(P));
  for (int32_t r = 0; r < R; ++r) {
    eoff[r + 1] = eoff[r] + P->n_elems[r];
    int8_t cl = P->clamp ? P->clamp[r] : -1;
    int64_t n0 = eoff[r] + r, N = P->n_elems[r];
    /* fixed pose = clamped node/element state at entry */
    if (cl == 0) { memcpy(rfix + 3 * r, pos + 3 * n0, 3 * sizeof(double)); memcpy(Qfix + 9 * r, dirs + 9 * eoff[r], 9 * sizeof(double)); }
    if (cl == 1) { memcpy(rfix + 3 * r, pos + 3 * (n0 + N), 3 * sizeof(double)); memcpy(Qfix + 9 * r, dirs + 9 * (eoff[r] + N - 1), 9 * sizeof(double)); }
  }
  int64_t first_bad = -1;
  int32_t bits = 0;
  double tt = *t;
#define RUN_STAGE(r, stage)                                                              \
  do {                                                                                   \
    ctx_setup(P, (r), eoff[(r)], &c);                                                    \
    memcpy(c.rfix, rfix + 3 * (r), sizeof c.rfix);                                       \
    memcpy(c.Qfix, Qfix + 9 * (r), sizeof c.Qfix);                                       \
    int f_ = rod_stage(P, (r), &c, (stage), pos, vel, dirs, omega, dt, t_half, Fext);    \
    if (f_) { bits |= f_; if (first_bad < 0 || (r) < first_bad) first_bad = (r); }       \
  } while (0)
  const int contact = P->contact && P->contact->enable;
  double *Fext = NULL;
  if (contact) Fext = (double *)calloc((size_t)(eoff[R] + R) * 3 + 3, sizeof(double));
  for (int64_t s = 0; s < n_steps; ++s) {
    double t_half = tt + 0.5 * dt;
    if (protocol == ORC_SYNC || contact) { /* barrier after every stage; rods that
                                              interact need it */
      for (int stage = 1; stage <= 3; ++stage) {
        if (stage == 2 && contact) {       /* contact forces at the half-step configuration, v^n */
          memset(Fext, 0, sizeof(double) * 3 * (size_t)(eoff[R] + R));
          orc_contact_forces(P, pos, vel, Fext);
        }
        for (int32_t r = 0; r < R; ++r) RUN_STAGE(r, stage);
      }
    } else {                             /* barrier once per step */
      for (int32_t r = 0; r < R; ++r)
        for (int stage = 1; stage <= 3; ++stage) RUN_STAGE(r, stage);
    }
    tt = t_half + 0.5 * dt;
  }
#undef RUN_STAGE
  free(Fext);
  *t = tt;
  ctx_free(&c);
  free(eoff); free(rfix); free(Qfix);
  if (bad_rod) *bad_rod = first_bad;
  if (fault_out) *fault_out = bits;
  return first_bad >= 0 ? ORC_EUNSTABLE : ORC_OK;
}

/* ---------------------------------------------------------------- contact (NEXT-4) */

/* Closest points of two segments: minimise |p0 + s d1 - q0 - t d2|^2 over [0,1]^2.  Candidates
 * (in this order): the interior stationary point when it lies inside the square, then the four
 * edges s = 0, s = 1, t = 0, t = 1 each with its clamped 1-D minimiser; the first candidate with
 * the smallest distance wins (so ties resolve deterministically). */
static double seg_dist2(const double *p0, const double *d1, const double *q0, const double *d2, double s, double t) {
  double x[3];
  for (int q = 0; q < 3; ++q) x[q] = p0[q] + s * d1[q] - q0[q] - t * d2[q];
  return v_dot(x, x);
}
static double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

void orc_segment_closest(const double p0[3], const double p1[3], const double q0[3], const double q1[3],
                         double *s_out, double *t_out, double *dist) {
  double d1[3], d2[3], r[3];
  v_sub(p1, p0, d1);
  v_sub(q1, q0, d2);
  v_sub(p0, q0, r);
  double a = v_dot(d1, d1), e = v_dot(d2, d2), b = v_dot(d1, d2), c = v_dot(d1, r), f = v_dot(d2, r);
  double best = -1.0, bs = 0.0, bt = 0.0;
  double cs[5], ct[5];
  int n = 0;
  double den = a * e - b * b;
  if (den > 0.0) {
    double s = (b * f - c * e) / den, t = (a * f - b * c) / den;
    if (s >= 0.0 && s <= 1.0 && t >= 0.0 && t <= 1.0) { cs[n] = s; ct[n] = t; ++n; }
  }
  /* s = 0: minimise over t |r - t d2|^2 -> t = f / e;  s = 1: t = (f + b) / e */
  cs[n] = 0.0; ct[n] = e > 0.0 ? clamp01(f / e) : 0.0; ++n;
  cs[n] = 1.0; ct[n] = e > 0.0 ? clamp01((f + b) / e) : 0.0; ++n;
  /* t = 0: minimise over s |r + s d1|^2 -> s = -c / a;  t = 1: s = (b - c) / a */
  cs[n] = a > 0.0 ? clamp01(-c / a) : 0.0; ct[n] = 0.0; ++n;
  cs[n] = a > 0.0 ? clamp01((b - c) / a) : 0.0; ct[n] = 1.0; ++n;
  for (int k = 0; k < n; ++k) {
    double d = seg_dist2(p0, d1, q0, d2, cs[k], ct[k]);
    if (best < 0.0 || d < best) { best = d; bs = cs[k]; bt = ct[k]; }
  }
  *s_out = bs;
  *t_out = bt;
  *dist = sqrt(best);
}

static double contact_radius(const orc_problem *P, int32_t rod, int64_t e0) {
  if (P->contact->radius) return P->contact->radius[rod];
  return sqrt(matv(P, P->area, rod, e0) / PI);
}

/* element -> rod, element -> first node, rod radius / stiffness scale, for the whole batch */
typedef struct { int32_t *rod; int64_t *node; double *rad, *Er; } elem_map;
static void elem_map_build(const orc_problem *P, elem_map *m, int64_t *E_out) {
  int64_t E = 0;
  for (int32_t r = 0; r < P->n_rods; ++r) E += P->n_elems[r];
  m->rod = (int32_t *)malloc(sizeof(int32_t) * (size_t)(E + 1));
  m->node = (int64_t *)malloc(sizeof(int64_t) * (size_t)(E + 1));
  m->rad = (double *)malloc(sizeof(double) * (size_t)(P->n_rods + 1));
  m->Er = (double *)malloc(sizeof(double) * (size_t)(P->n_rods + 1));
  int64_t e = 0;
  for (int32_t r = 0; r < P->n_rods; ++r) {
    m->rad[r] = contact_radius(P, r, e);
    m->Er[r] = matv(P, P->youngs, r, e) * m->rad[r];
    for (int32_t j = 0; j < P->n_elems[r]; ++j, ++e) { m->rod[e] = r; m->node[e] = e + r; }
  }
  *E_out = E;
}
static void elem_map_free(elem_map *m) { free(m->rod); free(m->node); free(m->rad); free(m->Er); }

static int excluded(const orc_problem *P, const elem_map *m, int64_t a, int64_t b) {
  if (m->rod[a] != m->rod[b]) return 0;
  int64_t dj = a > b ? a - b : b - a;
  return dj <= P->contact->exclude;
}

int64_t orc_contact_pairs(const orc_problem *P, const double *pos, int64_t max_pairs, int64_t *pairs, double *gaps) {
  elem_map m;
  int64_t E, found = 0;
  elem_map_build(P, &m, &E);
  for (int64_t a = 0; a < E; ++a)
    for (int64_t b = a + 1; b < E; ++b) {
      if (excluded(P, &m, a, b)) continue;
      double s, t, d;
      orc_segment_closest(pos + 3 * m.node[a], pos + 3 * (m.node[a] + 1), pos + 3 * m.node[b], pos + 3 * (m.node[b] + 1),
                          &s, &t, &d);
      double gap = d - (m.rad[m.rod[a]] + m.rad[m.rod[b]]);
      if (gap < 0.0) {
        if (found < max_pairs) { pairs[2 * found] = a; pairs[2 * found + 1] = b; gaps[found] = gap; }
        ++found;
      }
    }
  elem_map_free(&m);
  return found;
}

/* Penalty normal force F_n = max(0, k (-gap) - gamma v_n) along n (from b to a), regularised
 * Coulomb friction F_t = -mu_k F_n v_t/|v_t| when |v_t| > v_stick, else -mu_s F_n v_t / v_stick
 * (SPEC.md:385-400 design decisions).  Returns the force on body a. */
static void contact_law(const orc_contact *C, double k, double gap, const double *n, const double *vr, double *F) {
  double vn = v_dot(vr, n);
  double fn = k * (-gap) - C->gamma_n * vn;
  if (fn < 0.0) fn = 0.0;
  double vt[3];
  for (int q = 0; q < 3; ++q) vt[q] = vr[q] - vn * n[q];
  double svt = sqrt(v_dot(vt, vt));
  for (int q = 0; q < 3; ++q) {
    double ft = 0.0;
    if (svt > C->v_stick) ft = -C->mu_k * fn * vt[q] / svt;
    else if (C->v_stick > 0.0) ft = -C->mu_s * fn * vt[q] / C->v_stick;
    F[q] = fn * n[q] + ft;
  }
}

void orc_contact_forces(const orc_problem *P, const double *pos, const double *vel, double *F) {
  const orc_contact *C = P->contact;
  elem_map m;
  int64_t E;
  elem_map_build(P, &m, &E);
  for (int64_t a = 0; a < E; ++a)
    for (int64_t b = a + 1; b < E; ++b) {
      if (excluded(P, &m, a, b)) continue;
      int64_t ja = m.node[a], jb = m.node[b];
      double s, t, d;
      orc_segment_closest(pos + 3 * ja, pos + 3 * (ja + 1), pos + 3 * jb, pos + 3 * (jb + 1), &s, &t, &d);
      int32_t ra = m.rod[a], rb = m.rod[b];
      double gap = d - (m.rad[ra] + m.rad[rb]);
      if (!(gap < 0.0) || d == 0.0) continue;
      double pa[3], pb[3], n[3], va[3], vb[3], vr[3], f[3];
      for (int q = 0; q < 3; ++q) {
        pa[q] = (1.0 - s) * pos[3 * ja + q] + s * pos[3 * (ja + 1) + q];
        pb[q] = (1.0 - t) * pos[3 * jb + q] + t * pos[3 * (jb + 1) + q];
      }
      for (int q = 0; q < 3; ++q) n[q] = (pa[q] - pb[q]) / d;
      for (int q = 0; q < 3; ++q) {
        va[q] = (1.0 - s) * vel[3 * ja + q] + s * vel[3 * (ja + 1) + q];
        vb[q] = (1.0 - t) * vel[3 * jb + q] + t * vel[3 * (jb + 1) + q];
        vr[q] = va[q] - vb[q];
      }
      double k = C->k_n > 0.0 ? C->k_n : (m.Er[ra] < m.Er[rb] ? m.Er[ra] : m.Er[rb]);
      contact_law(C, k, gap, n, vr, f);
      for (int q = 0; q < 3; ++q) {
        F[3 * ja + q] += (1.0 - s) * f[q];
        F[3 * (ja + 1) + q] += s * f[q];
        F[3 * jb + q] -= (1.0 - t) * f[q];
        F[3 * (jb + 1) + q] -= t * f[q];
      }
    }
  if (C->plane_on) {                   /* half-space n . x >= d, node-wise (capsule ends) */
    double nn = sqrt(v_dot(C->plane_n, C->plane_n)), n[3];
    for (int q = 0; q < 3; ++q) n[q] = C->plane_n[q] / nn;
    int64_t node = 0;
    for (int32_t r = 0; r < P->n_rods; ++r) {
      double k = C->k_n > 0.0 ? C->k_n : m.Er[r];
      for (int32_t i = 0; i <= P->n_elems[r]; ++i, ++node) {
        double gap = v_dot(n, pos + 3 * node) - C->plane_d - m.rad[r];
        if (!(gap < 0.0)) continue;
        double f[3];
        contact_law(C, k, gap, n, vel + 3 * node, f);
        for (int q = 0; q < 3; ++q) F[3 * node + q] += f[q];
      }
    }
  }
  elem_map_free(&m);
}

/* Diagnostics (SURVEY §8 C.3 "energy"):
 * 1/2 sum m |v|^2 + 1/2 sum w.(J/e)w + 1/2 sum (sig-sig0).S(sig-sig0) lhat
 * + 1/2 sum (kap-kap0).Bv(kap-kap0) Dh - sum m g.r - F_tip.r_tip. */
int orc_energy(const orc_problem *P, const double *pos, const double *vel, const double *dirs,
               const double *omega, double t, double *out) {
  for (int q = 0; q < ORC_NDIAG; ++q) out[q] = 0.0;
  int32_t Nmax = max_elems(P);
  rod_ctx c;
  ctx_alloc(&c, Nmax);
  int64_t e0 = 0;
  int fault = 0;
  for (int32_t rod = 0; rod < P->n_rods; ++rod) {
    ctx_setup(P, rod, e0, &c);
    const double *r = pos + 3 * c.n0, *v = vel + 3 * c.n0, *Q = dirs + 9 * c.e0, *w = omega + 3 * c.e0;
    const int32_t N = c.N;
    double *e = c.e, *sg = c.sig, *kp = c.kap;
    fault |= orc_rod_strains(N, c.lhat, r, Q, e, sg, kp);
    for (int32_t i = 0; i <= N; ++i) {
      double vv = v_dot(v + 3 * i, v + 3 * i);
      out[ORC_D_KE_T] += 0.5 * c.m[i] * vv;
      out[ORC_D_PE_GRAV] -= c.m[i] * v_dot(P->gravity, r + 3 * i);
      out[ORC_D_PX] += c.m[i] * v[3 * i + 0];
      out[ORC_D_PY] += c.m[i] * v[3 * i + 1];
      out[ORC_D_PZ] += c.m[i] * v[3 * i + 2];
      if (sqrt(vv) > out[ORC_D_VMAX]) out[ORC_D_VMAX] = sqrt(vv);
      out[ORC_D_MASS] += c.m[i];
    }
    if (P->tip_force) out[ORC_D_PE_TIP] -= v_dot(P->tip_force + 3 * rod, r + 3 * c.tip_node);
    for (int32_t j = 0; j < N; ++j) {
      for (int q = 0; q < 3; ++q) {
        double s0 = P->rest_sigma ? P->rest_sigma[3 * (c.e0 + j) + q] : 0.0;
        double d = sg[3 * j + q] - s0;
        out[ORC_D_KE_R] += 0.5 * c.J[3 * j + q] * w[3 * j + q] * w[3 * j + q] / e[j];
        out[ORC_D_PE_SHEAR] += 0.5 * c.S[3 * j + q] * d * d * c.lhat[j];
      }
    }
    for (int32_t k = 1; k < N; ++k) {
      double k0[3];
      rest_kappa_at(P, rod, &c, k, t, k0);
      for (int q = 0; q < 3; ++q) {
        double d = kp[3 * (k - 1) + q] - k0[q];
        out[ORC_D_PE_BEND] += 0.5 * c.Bv[3 * k + q] * d * d * c.Dh[k];
      }
    }
    out[ORC_D_NELEM] += N;
    e0 += N;
  }
  ctx_free(&c);
  return fault ? ORC_EUNSTABLE : ORC_OK;
}
