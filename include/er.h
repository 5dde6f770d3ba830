/*
 * er.h -- C-ABI of libelasticarod: batched discrete Cosserat rod stepping on B200 (sm_100a).
 *
 * The operation (PAPER.md "Methods / Cosserat rod dynamics", lines 231-258):
 *   Eq. (1a)  rho A d2r/dt2 = d/ds( Q^T S sigma / e ) + f
 *   Eq. (1b)  (rho I / e) dw/dt = d/ds( B kappa / e^3 ) + kappa x B kappa / e^3 + Q t x S sigma
 *                                + (rho I w / e) x w + (rho I w / e^2) de/dt + c
 *   sigma = Q(r' - d3), kappa = ax(Q dQ^T/ds), w = ax(Q dQ^T/dt), e = |r'|
 *   B = diag{E I1, E I2, G(I1+I2)}, S = diag{alpha_c G A, alpha_c G A, E A},
 *   I = diag{I1, I2, I1+I2}
 * discretised on N+1 nodes / N elements / N-1 Voronoi domains per rod and advanced by
 * position Verlet, drift(h/2) - kick(h) - drift(h/2), with kinematic constraints after
 * every stage.  The discrete readings are DESIGN.md §3 (= SURVEY.md §8 C.3-C.4).
 * Rods do not interact (every rod of a batch is advanced independently) unless contact is
 * enabled with er_set_contact.
 *
 * Conventions shared by every call
 *  - fp64 throughout.  Lab-frame vectors: positions, velocities, tip forces, gravity, b(t).
 *    Local-frame vectors (components on d1, d2, d3): omega, rest_sigma, rest_kappa,
 *    magnetization.
 *  - Rod r owns n_elems[r] >= 1 elements, n_elems[r]+1 nodes and n_elems[r]-1 Voronoi
 *    domains; rods are stored back to back in the order given ("canonical order").
 *    elem_offset(r) = sum_{q<r} n_elems[q], node_offset(r) = elem_offset(r) + r,
 *    voronoi_offset(r) = elem_offset(r) - r.
 *  - Canonical array layouts (AoS per quantity, C order):
 *      positions, velocities [n_nodes_total][3];  directors [n_elems_total][3][3], row a is
 *      the director d_{a+1} in lab coordinates (Q maps lab -> local);
 *      omega [n_elems_total][3];  rest_sigma [n_elems_total][3];  rest_kappa [n_voronoi_total][3].
 *  - Ownership: the library copies every input at create/set time; the caller keeps its
 *    arrays.  The handle owns all device memory until er_destroy.  Output pointers are
 *    caller-owned buffers of the canonical size.
 *  - Errors: every call returns er_status and never aborts.  ER_EINVAL messages list every
 *    validation error found (not only the first).  er_last_error() returns the message of the
 *    last failing call on that handle (or, for a NULL handle, of the last failed
 *    er_create_batch on the calling thread).
 *  - Threading / streams: one handle per host thread at a time.  All device work of a handle
 *    is issued on its stream (the caller's, or one the library creates); calls that return
 *    data to the caller synchronise that stream.
 */
#ifndef ELASTICAROD_ER_H
#define ELASTICAROD_ER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ER_ABI_VERSION 3

typedef struct er_batch er_batch; /* opaque handle; owns device memory */

typedef enum {
  ER_OK = 0,
  ER_EINVAL = 1,     /* invalid argument / input data (all problems listed in er_last_error) */
  ER_EUNSTABLE = 2,  /* a fault was detected while stepping (er_fault gives rod and bits)   */
  ER_EIO = 3,        /* reserved (no file I/O in the library)                               */
  ER_ENOMEM = 4,     /* device allocation failed                                            */
  ER_ECUDA = 5       /* any other CUDA error (message has the CUDA error string)            */
} er_status;

typedef enum { ER_HOST = 0, ER_DEVICE = 1 } er_mem;

/* fault bits reported by er_fault after ER_EUNSTABLE */
#define ER_F_NONFINITE 1   /* a state component became NaN/Inf                                  */
#define ER_F_DEGENERATE 2  /* dilatation e = |edge|/lhat < 1e-12                               */
#define ER_F_ANTIPODAL 4   /* adjacent-element relative rotation angle >= pi - 1e-6            */
#define ER_F_OVERSPEED 8   /* |v| > 1e6 sqrt(E/rho)                                           */
#define ER_F_CONTACT 16    /* contact broad phase could not bin an element (wider than the top
                              HHG level, non-finite or |coordinate| > 2^30 cells) or the
                              cross-level record pool / per-element record list overflowed    */

/* ------------------------------------------------------------------------- er_create_batch
 * A ragged batch of rods with per-rod element counts (north_star "er_create_batch").
 *  n_elems            HOST  [n_rods], each 1 <= n <= ER_MAX_ELEMS_PER_ROD.  Rods longer than
 *                     the tile capacity minus one run in thread-block clusters of 256-slot
 *                     segments: > ER_TILE_MAX_ELEMS with 512-slot tiles, > 255 with 256-slot
 *                     tiles (tile_slots 256, or automatically for ragged batches whose rods of
 *                     256..511 elements hold <= 2% of the elements); not with tile_slots 128.
 *  material_per_rod   1: the seven material arrays have n_rods entries (one value per rod);
 *                     0: they have n_elems_total entries (one value per element).
 *  density            HOST  rho, volumetric mass density (kg/m^3) (reading DESIGN §3 #6).
 *  area, I1, I2       HOST  cross-section area A and second moments of area I1, I2.
 *  youngs, shear_mod  HOST  E and G.   alpha_c  HOST  shear correction factor.
 *  rest_lengths       HOST  [n_elems_total] reference element lengths lhat > 0.
 *  rest_sigma         HOST  [n_elems_total*3] intrinsic shear/stretch strain, or NULL (= 0).
 *  rest_kappa         HOST  [n_voronoi_total*3] static intrinsic curvature, or NULL (= 0).
 *  positions          src_mem [n_nodes_total*3]   (required)
 *  velocities         src_mem [n_nodes_total*3]   or NULL (= 0)
 *  directors          src_mem [n_elems_total*9]   (required; orthonormal, det +1 within 1e-10)
 *  omega              src_mem [n_elems_total*3]   or NULL (= 0)
 *  t0                 initial time (rest-curvature actuation and b(t) depend on t).
 *  src_mem            memory space of positions/velocities/directors/omega.
 *  device             CUDA device ordinal.
 *  stream             cudaStream_t to use, or NULL to let the library create its own.
 *  tile_slots         rod-tile capacity (see the struct); fixes the device layout.
 * Errors: ER_EINVAL (all problems listed), ER_ENOMEM, ER_ECUDA.  *out is NULL on error.
 */
#define ER_MAX_ELEMS_PER_ROD 4095  /* rods up to 511 elements share rod tiles; longer ones are
                                      advanced by a thread-block cluster of up to 16 CTAs */
#define ER_TILE_MAX_ELEMS 511

typedef struct {
  int32_t n_rods;
  const int32_t *n_elems;
  int32_t material_per_rod;
  const double *density, *area, *I1, *I2, *youngs, *shear_mod, *alpha_c;
  const double *rest_lengths;
  const double *rest_sigma;
  const double *rest_kappa;
  const double *positions;
  const double *velocities;
  const double *directors;
  const double *omega;
  double t0;
  int32_t src_mem; /* er_mem */
  int32_t device;
  void *stream;
  int32_t tile_slots; /* 0 = auto (256; 512 when a rod has more than 255 elements, or when
                         equal-length rods keep clearly more lanes busy in 512-slot tiles);
                         128, 256 or 512 = slots (threads) per rod tile; must be >= max N + 1 */
} er_batch_desc;

er_status er_create_batch(const er_batch_desc *desc, er_batch **out);

/* ------------------------------------------------------------------------- er_set_bc
 * Kinematic boundary conditions (reading DESIGN §3 #15).
 *  clamp_end  HOST [n_rods]: -1 free-free; 0 clamp the s = 0 end (node 0 position and
 *             element 0 frame); 1 clamp the s = L end (node N and element N-1).  NULL = all free.
 * The clamped pose is the state at the time of this call; clamped node/element rates are
 * zeroed after every kick.  Default after create: all free.   Errors: ER_EINVAL.
 */
er_status er_set_bc(er_batch *b, const int8_t *clamp_end);

/* ------------------------------------------------------------------------- er_set_forcing
 * External loads and actuation (PAPER.md:252 f and c; :263-268 magnetic couple;
 * BASELINE configs[3] rest-curvature actuation).  All pointers HOST.
 *  gravity         lab acceleration g; node i receives m_i g.
 *  damping         [n_rods] linear damping rate nu (1/s): a -= nu v, alpha -= nu w
 *                  (reading DESIGN §3 #11), or NULL to use damping_all for every rod.
 *  tip_force       [n_rods*3] constant lab force on the free-end node (node N, or node 0 for
 *                  rods clamped at s = L), or NULL.
 *  act_A, act_f, act_L  [n_rods] each, or all NULL: time-varying rest curvature
 *                  kappa0_k[act_component] += A sin(2 pi (s_k/L - f t)), s_k = arc length of
 *                  interior node k, evaluated at t_n + h/2 (DESIGN §3 #13, #14).
 *  magnetization   [n_elems_total*3] local magnetic moment per unit rest length m, or NULL;
 *                  element couple c_j = lhat_j m_j x (Q_j b(t)) with b(t) = b_field rotated by
 *                  the angle b_omega t about b_axis (right-handed; b_axis = 0 means lab z):
 *                  a homogeneous field rotating in the plane normal to b_axis.
 *  musc_A, musc_T, musc_lambda, musc_phi  [n_rods] each, or all NULL: muscular torque wave
 *                  (DESIGN §3 #26) tau_k(t) = A sin(2 pi (t/T - s_k/lambda) + phi)
 *                  about the local axis musc_component at every interior node k, applied as a
 *                  couple pair (+tau_k on element k, -tau_k on element k-1: net zero per rod),
 *                  evaluated at t_n + h/2.  T, lambda > 0.
 * Replaces all previous forcing.  Default after create: none.   Errors: ER_EINVAL.
 */
typedef struct {
  double gravity[3];
  const double *damping;
  double damping_all;
  const double *tip_force;
  const double *act_A, *act_f, *act_L;
  int32_t act_component;
  const double *magnetization;
  double b_field[3];
  double b_omega;
  double b_axis[3];
  const double *musc_A, *musc_T, *musc_lambda, *musc_phi;
  int32_t musc_component;
} er_forcing;

er_status er_set_forcing(er_batch *b, const er_forcing *f);

/* ------------------------------------------------------------------------- er_set_external_loads
 * User external loads: the distributed force f of Eq. (1a) and couple c-bar of Eq. (1b)
 * (PAPER.md:252), e.g. the hydrodynamic loads an external flow solver returns every step
 * (reading DESIGN §3 #30).  Discrete and already integrated:
 *  node_force   [n_nodes_total*3] lab-frame force on each node (N), canonical node order
 *               (rod by rod, N_r + 1 nodes each), added to F_i; or NULL for none.
 *  elem_couple  [n_elems_total*3] local-frame (director basis) couple on each element (N m),
 *               added to C_j; or NULL for none.
 * src_mem says where both arrays live (ER_DEVICE: device pointers on the batch's device, read on
 * the batch's stream (er_query().stream) without host synchronisation, so a solver can update
 * them every step; the caller orders their producer before the call -- same stream or an event).  Values are
 * copied; they stay in force, constant in time, until the next call (NULL clears that array).
 * Independent of er_set_forcing.  Not validated: non-finite loads surface as ER_F_NONFINITE at the
 * next er_step.  They do no work in the diagnostics' potential energies (non-conservative).
 * Errors: ER_EINVAL (bad src_mem), ER_ECUDA.
 */
er_status er_set_external_loads(er_batch *b, int32_t src_mem, const double *node_force, const double *elem_couple);

/* ------------------------------------------------------------------------- er_step
 * Advance every rod by n_steps >= 0 position-Verlet steps of size dt > 0 (north_star
 * "er_step(n_steps, dt)").  Stream-ordered; returns after the work completed and one 16-byte
 * fault-word read.  ER_EUNSTABLE if any rod faulted during these steps (state is then
 * undefined for the faulted rods; other rods are unaffected).  Errors: ER_EINVAL, ER_ECUDA.
 */
er_status er_step(er_batch *b, int64_t n_steps, double dt);

/* ------------------------------------------------------------------------- er_get_state
 * Copy the current state out in canonical order (north_star "er_get_state"): the rod's
 * dynamic unknowns of Eqs. (1a)-(1b), i.e. the centerline r and its velocity at the nodes, the
 * frame Q (rows d1, d2, d3) and the local angular velocity w = ax(Q dQ^T/dt)
 * on the elements, at the end of the last completed step.  dst_mem says
 * where the (caller-owned) buffers live.  Any pointer may be NULL to skip that quantity.
 * *t receives the time.  Synchronises the batch's stream.  d3 is rebuilt as d1 x d2 from the
 * stored pair (DESIGN §4 "Director storage").  Errors: ER_EINVAL (bad dst_mem), ER_ECUDA.
 */
er_status er_get_state(er_batch *b, int32_t dst_mem, double *positions, double *velocities,
                       double *directors, double *omega, double *t);

/* ------------------------------------------------------------------------- er_set_state
 * Overwrite the state (resume from a snapshot taken with er_get_state, or inject a state).
 * src_mem says where the arrays live (ER_DEVICE arrays are read on the batch's stream: the caller
 * orders their producer before the call); any pointer may be NULL to keep that quantity; t may be
 * NULL to keep the time.  Deliberately NOT validated (no orthonormality / finiteness check):
 * a bad state surfaces as ER_EUNSTABLE at the next er_step.  Clamped poses are unchanged
 * (call er_set_bc again to re-pose).   Errors: ER_EINVAL (bad src_mem), ER_ECUDA.
 */
er_status er_set_state(er_batch *b, int32_t src_mem, const double *positions, const double *velocities,
                       const double *directors, const double *omega, const double *t);

/* ------------------------------------------------------------------------- er_diagnostics
 * Batch-local scalar diagnostics at the current state:
 *  out[ER_D_*] below.  Sums over this batch only (a multi-GPU caller all-reduces them:
 *  ER_D_VMAX with max, the rest with sum).  Deterministic (fixed-order reduction).
 */
enum {
  ER_D_KE_TRANS = 0, /* 1/2 sum m |v|^2                               */
  ER_D_KE_ROT,       /* 1/2 sum w . (J/e) w                           */
  ER_D_PE_SHEAR,     /* 1/2 sum (s - s0) . S (s - s0) lhat            */
  ER_D_PE_BEND,      /* 1/2 sum (k - k0(t)) . Bv (k - k0(t)) Dh       */
  ER_D_PE_GRAV,      /* - sum m g . r                                 */
  ER_D_PE_TIP,       /* - F_tip . r_tip                               */
  ER_D_PX, ER_D_PY, ER_D_PZ, /* sum m v                               */
  ER_D_VMAX,         /* max |v|                                       */
  ER_D_MASS,         /* sum m                                         */
  ER_D_NELEM,        /* number of elements                            */
  ER_NDIAG
};
er_status er_diagnostics(er_batch *b, double out[ER_NDIAG]);

/* ------------------------------------------------------------------------- er_fault
 * After ER_EUNSTABLE: lowest faulted rod id (canonical order) and the OR of fault bits.
 */
er_status er_fault(const er_batch *b, int64_t *rod, int32_t *bits);

/* ------------------------------------------------------------------------- er_set_contact
 * Rod-rod and rod-boundary contact with friction.  The paper names the
 * model -- "rod interactions via normal force and friction", a collision engine with
 * a hierarchical hash-grid (HHG) broad phase (Fig. 2e) that forces synchronous
 * stepping -- and leaves the formulas to its missing supplement; the law below is
 * reading DESIGN §3 #27.  Each element is a capsule (segment between its nodes, radius r_rod).
 * A pair of elements (a, b), not of the same rod within `exclude` elements, whose closest points
 * pa, pb (exact segment-segment minimiser) are closer than r_a + r_b (gap = |pa - pb| - r_a - r_b
 * < 0, |pa - pb| > 0) receives, with n = (pa - pb)/|pa - pb| and v_r the relative velocity of the
 * closest points (barycentric in the segment's nodes):
 *   F = max(0, k (-gap) - gamma_n v_r.n) n + F_t  on a, -F on b,
 *   F_t = -mu_k F_n v_t/|v_t| if |v_t| > v_stick, else -mu_s F_n v_t/v_stick  (v_t = v_r - (v_r.n) n),
 * each distributed to the segment's two nodes with the closest-point weights (1 - s, s).
 * k = k_n if k_n > 0, else min(E_a r_a, E_b r_b).  With plane_on, every node x with
 * gap = n.x - d - r < 0 receives the same law against the half-space n.x >= d (v_r = its velocity).
 * Contact forces are evaluated once per step at the half-step configuration (after drift-1) with
 * v^n (the synchronous protocol): while contact is enabled every er_step step is
 * one contact evaluation plus one step-kernel launch, ER_OPT_STEPS_PER_LAUNCH does not apply, and
 * ER_OPT_KERNEL = 1 selects the staged kernels (any other value the fused contact step).
 *  radius      HOST [n_rods] contact radius, or NULL = sqrt(A/pi) of the rod's first element.
 *  cell0       finest HHG cell (m); 0 = auto: 1.25 x the smallest rest capsule extent
 *              (lhat + 2r).  n_levels (1..8); 0 = auto: enough levels of doubling cells for the
 *              largest rest extent x 1.25, plus one level of headroom.
 *  pool_factor cross-level record pool = pool_factor x n_elems records (0 = auto, 4).
 *  skin        Verlet skin (m; 0 = auto: a quarter of the smallest contact radius).  The broad
 *              phase bins capsule AABBs grown by skin/2 and its candidate lists are reused until
 *              a node has moved more than skin/2 from where it was at the last build (checked on
 *              the device every step; the lists are then rebuilt in the same step).  Results do
 *              not depend on the skin beyond round-off of the summation order.
 * An element whose AABB outgrows the top level, or a full pool, faults the step with
 * ER_F_CONTACT.  c == NULL or c->enable == 0 disables contact.
 * Errors: ER_EINVAL, ER_ENOMEM.
 */
typedef struct {
  int32_t enable;
  double k_n, gamma_n, mu_s, mu_k, v_stick;
  const double *radius;
  int32_t exclude;
  int32_t plane_on;
  double plane_n[3];  /* need not be unit; normalised by the library */
  double plane_d;
  double cell0;
  int32_t n_levels;
  double pool_factor;
  double skin;
} er_contact;
er_status er_set_contact(er_batch *b, const er_contact *c);

/* ------------------------------------------------------------------------- contact across GPUs
 * Rods sharded over ranks may touch rods of another rank (NEXT-4; the paper's
 * collision engine with synchronisation after every stage).  Such rods enter this
 * batch as GHOST rods: only their contact geometry is declared here, and their node records
 * (r, v after drift-1: 6 doubles per node, lab frame) are supplied by the caller every step; this
 * batch never advances them.  The broad and narrow phases then run over own + ghost elements; only
 * the own nodes receive forces.  Pair forces are evaluated from both sides with bit-identical
 * inputs (the ghost records are copies), so the owner of either rod applies exactly the opposite
 * force of the other (momentum balance across ranks).
 *
 * er_set_contact_ghosts declares n_ghost ghost rods (HOST arrays [n_ghost]): elements per rod (>= 1),
 * contact radius (> 0), stiffness scale E r (k_n <= 0 uses min(E_a r_a, E_b r_b)), shortest and
 * longest rest element length (HHG levels).  n_ghost = 0 removes them.  If contact is enabled,
 * it is re-initialised with the same parameters (candidate lists rebuilt).  Ghost node records
 * start at zero: set them before the first step.
 *
 * With ghosts, a step is split so that the caller can exchange node records between the halves:
 *   er_step_begin(b, dt)   drift-1 of one step (every own rod), own node records ready;
 *   er_contact_records(b, ER_..., dst)           own node records [n_nodes][6] -> dst;
 *   er_set_ghost_records(b, ER_..., src)         ghost node records [n_ghost_nodes][6] <- src
 *                                                 (ghost rods in declaration order, N_g + 1 nodes each);
 *   er_step_finish(b, dt)  contact evaluation over own + ghost elements, kick, drift-2.
 * er_step_begin / er_step_finish also work without ghosts (a plain contact step in two calls; the
 * trajectory is bitwise that of er_step).  er_step itself returns ER_EINVAL while ghosts are
 * declared (their records would be stale).  Both calls are stream-ordered; er_step_finish reads
 * the fault word like er_step (ER_EUNSTABLE).  Errors: ER_EINVAL (contact off, begin/finish out of
 * order, a dt different from begin's), ER_ECUDA. */
er_status er_set_contact_ghosts(er_batch *b, int64_t n_ghost, const int32_t *n_elems, const double *radius,
                                const double *stiffness, const double *lhat_min, const double *lhat_max);
er_status er_step_begin(er_batch *b, double dt);
er_status er_step_finish(er_batch *b, double dt);
er_status er_contact_records(er_batch *b, int32_t dst_mem, double *dst);
er_status er_set_ghost_records(er_batch *b, int32_t src_mem, const double *src);

/* Contact statistics (synchronises the stream): per step = of the last step of the last er_step
 * call; per build = of the last candidate-list build. */
typedef struct {
  int64_t candidates;      /* build: element pairs whose grown AABBs overlap (each pair once) */
  int64_t contacts;        /* step:  element pairs in contact (gap < 0)                       */
  int64_t cross_level;     /* step:  of those, pairs across HHG levels                        */
  int64_t plane_contacts;  /* step:  nodes in contact with the half-space                     */
  int64_t pool_used;       /* step:  cross-level records written                              */
  int64_t list_entries;    /* build: candidate-list entries (both sides of a pair)            */
  int64_t scanned;         /* build: proxies the broad phase scanned (its work measure)       */
  int64_t long_lists;      /* build: elements with more than 16 candidates (re-visited)       */
  int64_t builds;          /* list builds so far                                              */
  int32_t n_levels;        /* HHG levels configured                                           */
  int32_t level_mask;      /* build: levels populated (bit l)                                 */
  double cell0;            /* finest cell size                                                */
  double skin;             /* Verlet skin in use                                              */
} er_contact_stats;
er_status er_get_contact_stats(er_batch *b, er_contact_stats *out);

/* ------------------------------------------------------------------------- options / info */
typedef enum {
  ER_OPT_STEPS_PER_LAUNCH = 1, /* 1 (default): every step streams the state through HBM
                                  (SURVEY §8 D.3 B_min design).  k > 1: each launch keeps a
                                  rod tile on chip for k steps (temporal blocking, SURVEY §8(f)
                                  NEXT-1); identical results. */
  ER_OPT_KERNEL = 2,           /* 0 (default): fused single-pass step, persistent CTAs with
                                  TMA bulk prefetch of the next rod tile.
                                  1: staged three-kernel path (drift / dynamics+kick / drift),
                                  state through HBM between stages (ablation, debugging).
                                  2: fused step, one tile per CTA, plain loads (ablation).
                                  All three give identical results.
                                  3: memory-pipeline probe (measurement aid): the persistent
                                  kernel moves every tile through its TMA stage and back
                                  without computing -- the state and t are left unchanged.
                                  4: as 0 but results go from registers straight to HBM
                                  (plain coalesced stores instead of the smem stage + TMA
                                  bulk store; ablation, cfg3-type batches only). */
  ER_OPT_PHASE_TIMING = 3,     /* measurement aid: 1 = er_step records a CUDA event pair (on the
                                  handle's stream) around every step-kernel launch and every
                                  contact evaluation, summed into er_get_phase_times (a launch
                                  of S sweeps counts as S launches); setting the option (0 or 1)
                                  resets the sums.  Default 0. */
  ER_OPT_SWEEPS_PER_LAUNCH = 4 /* S >= 1: without contact, one persistent launch streams all rod
                                  tiles through HBM S times (S steps, each of ER_OPT_STEPS_PER_
                                  LAUNCH on-chip steps) -- the work of S launches without their
                                  boundaries or host submissions; identical results.  1 = one
                                  launch per step (CUDA-graph replays of 32).  0 (default,
                                  ER_DEFAULT_SWEEPS): 128 for small batches (at most 4 tiles per
                                  CTA of the grid), else 1. */
} er_option;
#define ER_DEFAULT_SWEEPS 0
er_status er_set_option(er_batch *b, int32_t option, int64_t value);

/* Device time of er_step's phases since ER_OPT_PHASE_TIMING was last set (CUDA events). */
typedef struct {
  double step_kernel_ms;        /* the rod step kernel launches (all kinds)                 */
  int64_t step_kernel_launches;
  double contact_ms;            /* contact evaluations (broad + narrow phase graphs)        */
  int64_t contact_evals;
} er_phase_times;
er_status er_get_phase_times(const er_batch *b, er_phase_times *out);

/* Measurement aid: when `trace` (DEVICE memory, [grid][64][4] uint64, zeroed by the caller) is
 * non-NULL, the persistent step kernel records for thread 0 of each CTA and its first 64 tiles
 * the low 48 bits of %globaltimer at: wait start (bits 56-63 = SM id), data arrival, compute
 * end, stores issued.  NULL disables it.  Compiled in only with -DER_TRACE=1 (a measurement
 * build, ER_NVCC_EXTRA); otherwise a non-NULL trace returns ER_EINVAL. */
er_status er_set_trace(er_batch *b, void *trace);

typedef struct {
  int64_t n_rods, n_elems_total, n_nodes_total, n_voronoi_total;
  int64_t n_tiles;         /* CTAs per fused-step launch                       */
  int32_t tile_slots;      /* threads per CTA (slots per tile)                 */
  int32_t device;
  void *stream;            /* the cudaStream_t all work is issued on            */
  int64_t launches;        /* kernels launched by er_step so far               */
  int64_t device_bytes;    /* device memory owned by the handle                */
  double t;                /* current time                                     */
  double bytes_per_step;   /* algorithmic HBM bytes of one step    */
  int32_t warp_rod_elems;  /* > 0: streaming steps run the warp-local kernel  */
                           /* (equal-length rods of this many elements, one   */
                           /* rod per <= 32 lanes); 0: tile kernel */
  int32_t warp_buffers;    /* its stage buffers per CTA (0 if not used)       */
  int32_t shared_material; /* 1: every rod has the same material constants and */
                           /* the warp kernel reads them from its parameters, */
                           /* with a 48-byte record per rod       */
  int32_t reserved_;
} er_info;
er_status er_query(const er_batch *b, er_info *info);

const char *er_last_error(const er_batch *b);
int32_t er_abi_version(void);
void er_destroy(er_batch *b);

#ifdef __cplusplus
}
#endif
#endif /* ELASTICAROD_ER_H */
