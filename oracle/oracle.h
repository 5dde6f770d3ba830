/*
 * oracle.h -- CPU ORACLE for the discrete Cosserat rod step (arxiv 2605.13766).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py
 * (its `cpu_baseline` leg and `--impl reference`) may load or execute anything
 * under oracle/.  The product path (include/er.h, paper_2605_13766_b200/) never
 * includes, links or calls this code, and this code includes nothing from it.
 *
 * Plain single-threaded fp64 C, AoS per rod, libm transcendentals, compiled
 * with -O2 -ffp-contract=off (no FMA contraction, no SIMD, no threads).
 * Every function cites the passage of PAPER.md (or the SURVEY.md §8 C.4
 * reading) it follows.  Array conventions are the canonical ones of
 * workloads/__init__.py.
 */
#ifndef ELASTICA_ORACLE_H
#define ELASTICA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Contact (SURVEY NEXT-4; PAPER.md:73, :80-84 name "normal force and friction" and an HHG broad
 * phase, the formulas are in the missing supplement -- readings DESIGN §3 #27). */
typedef struct {
  int32_t enable;
  double k_n;            /* penalty stiffness; <= 0: min(E_A r_A, E_B r_B) per pair            */
  double gamma_n;        /* normal damping                                                     */
  double mu_s, mu_k;     /* static / kinetic friction coefficients                              */
  double v_stick;        /* regularised Coulomb: |v_t| <= v_stick -> static branch              */
  const double *radius;  /* [R] contact radius, or NULL = sqrt(A / pi)                          */
  int32_t exclude;       /* same-rod element pairs with |j - k| <= exclude never touch            */
  int32_t plane_on;      /* half-space boundary n . x >= d                                       */
  double plane_n[3];
  double plane_d;
} orc_contact;

typedef struct {
  int32_t n_rods;
  const int32_t *n_elems;          /* [R], each >= 1                                   */
  int32_t material_per_rod;        /* 1: material arrays [R]; 0: [n_elems_total]       */
  const double *density;           /* rho, volumetric                  */
  const double *area, *I1, *I2, *youngs, *shear_mod, *alpha_c;
  const double *rest_lengths;      /* [E]                                              */
  const double *rest_sigma;        /* [E*3] local, or NULL = 0                         */
  const double *rest_kappa;        /* [V*3] local, static part, or NULL = 0            */
  const int8_t *clamp;             /* [R]: -1 free, 0 clamp s=0 end, 1 clamp s=L end    */
  double gravity[3];
  const double *damping;           /* [R] s^-1 rate form (C.4 #11), or NULL = 0         */
  const double *tip_force;         /* [R*3] lab, at the free end node, or NULL          */
  const double *act_A, *act_f, *act_L; /* [R] rest-curvature actuation, or NULL        */
  int32_t act_component;           /* 0,1,2: which local component of kappa0            */
  const double *magnetization;     /* [E*3] local m̄ per unit rest length, or NULL      */
  double b_field[3];               /* b(0) lab                                          */
  double b_omega;                  /* b(t) = R_axis(b_omega t) b(0)                      */
  double b_axis[3];                /* rotation axis of b(t) (normalised here), 0 = lab z */
  const double *musc_A, *musc_T, *musc_lambda, *musc_phi; /* [R] muscular torque wave, or NULL */
  int32_t musc_component;          /* local axis of the muscle couple (0 = d1)           */
  const orc_contact *contact;      /* NULL = rods do not interact                        */
  /* User external loads f and c-bar of Eqs. (1a)-(1b), discrete (DESIGN §3 #30):
   * a force per node [n_nodes*3] lab frame (N) and a couple per element [E*3] local frame (N m),
   * constant in time, added to F_i and C_j; NULL = none. */
  const double *ext_force;
  const double *ext_couple;
} orc_problem;

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EUNSTABLE = 2 };
enum { ORC_SYNC = 0, ORC_ASYNC = 1 };

/* fault bits (same meaning as the product's, defined independently) */
enum { ORC_F_NONFINITE = 1, ORC_F_DEGENERATE = 2, ORC_F_ANTIPODAL = 4, ORC_F_OVERSPEED = 8 };

/* diagnostics layout */
enum { ORC_D_KE_T = 0, ORC_D_KE_R, ORC_D_PE_SHEAR, ORC_D_PE_BEND, ORC_D_PE_GRAV, ORC_D_PE_TIP,
       ORC_D_PX, ORC_D_PY, ORC_D_PZ, ORC_D_VMAX, ORC_D_MASS, ORC_D_NELEM, ORC_NDIAG };

void orc_skew(const double v[3], double W[9]);
void orc_ax(const double U[9], double v[3]);
void orc_rot(const double v[3], double R[9]);
int  orc_logrot(const double R[9], double v[3]);   /* returns 0, or ORC_F_ANTIPODAL */

/* strains of one rod: e[N], sigma[N*3], kappa[(N-1)*3] */
int orc_rod_strains(int32_t N, const double *lhat, const double *pos, const double *dirs,
                    double *e, double *sigma, double *kappa);

/* accelerations of rod `rod` at the given state and time (C.3 steps 2-6):
 * internal+external nodal force F[(N+1)*3], element couple C[N*3],
 * a[(N+1)*3], alpha[N*3].  Pointers are to this rod's slices. */
int orc_rod_loads(const orc_problem *P, int32_t rod, const double *pos, const double *vel,
                  const double *dirs, const double *omega, double t,
                  double *F, double *C, double *a, double *alpha);

/* n_steps position-Verlet steps of the whole batch, in place (C.3).
 * *t is advanced.  On a fault returns ORC_EUNSTABLE, *bad_rod = first rod id,
 * *fault = fault bits of that rod. */
int orc_step(const orc_problem *P, double *pos, double *vel, double *dirs, double *omega,
             double *t, int64_t n_steps, double dt, int32_t protocol,
             int64_t *bad_rod, int32_t *fault);

/* closest points of segments p0-p1 and q0-q1: parameters s, t in [0,1] and distance */
void orc_segment_closest(const double p0[3], const double p1[3], const double q0[3], const double q1[3],
                         double *s, double *t, double *dist);

/* exhaustive contact detection at the given positions: element pairs (a < b, global element ids)
 * with gap = dist - (r_a + r_b) < 0; returns the number found (writes at most max_pairs) */
int64_t orc_contact_pairs(const orc_problem *P, const double *pos, int64_t max_pairs, int64_t *pairs, double *gaps);

/* contact forces on every node (added into F[n_nodes*3], which the caller zeroes) */
void orc_contact_forces(const orc_problem *P, const double *pos, const double *vel, double *F);

/* diagnostics at the current (integer-time) state: out[ORC_NDIAG] */
int orc_energy(const orc_problem *P, const double *pos, const double *vel, const double *dirs,
               const double *omega, double t, double *out);

#ifdef __cplusplus
}
#endif
#endif
