// er_layout.h -- device-resident layout of a rod batch (L0) and the kernel parameter block.
//
// HBM layout:
//  - node planes  : 6 fp64 planes [rx ry rz vx vy vz][n_nodes_pad]      (compact SoA, no ghosts)
//  - elem planes  : 12 fp64 planes [Q00..Q22 wx wy wz][n_elems_pad]      (row a of Q = d_{a+1})
//  - rod records  : [n_rods][ER_REC] fp64 derived constants of uniform rods + damping + vmax^2
//  - rod extras   : [n_rods][ER_REC2] fp64 tip force, actuation (read only when flagged)
//  - rod flags    : [n_rods] int32 (clamp mode, general, tip, actuation)
//  - eoff         : [n_rods+1] int64 element offsets (node offset = eoff + rod)
//  - tiles        : [n_tiles+1] int32 first rod of each tile (rod-aligned, <= tile_slots slots)
//  - gpar         : optional [ER_GP][n_nodes_pad] per-slot parameters of "general" rods
//                   (non-uniform rest lengths or per-element material)
//  - sigma0/kappa0/mag : optional [3][n_elems_pad] / [3][n_vor_pad] / [3][n_elems_pad] planes
// Ghost nodes exist only in shared memory (never in HBM).
#pragma once
#include <stdint.h>

// ---- rod record (uniform rods): everything one slot needs, read once per rod per step
enum {
  REC_LHAT = 0,  // rest length (uniform)
  REC_ILHAT,     // 1/lhat
  REC_S1,        // alpha_c G A   (shear, d1 and d2)
  REC_S3,        // E A           (stretch)
  REC_B1,        // E I1          (Voronoi bend/twist stiffness; = B for uniform rods)
  REC_B2,        // E I2
  REC_B3,        // G (I1 + I2)
  REC_IJ1,       // 1/(rho lhat I1)
  REC_IJ2,       // 1/(rho lhat I2)
  REC_IJ3,       // 1/(rho lhat (I1+I2))
  REC_KJ1,       // (J2 - J3)/J1   Euler coefficients of (J w) x w / J
  REC_KJ2,       // (J3 - J1)/J2
  REC_KJ3,       // (J1 - J2)/J3
  REC_IM,        // 1/(rho A lhat): inverse interior node mass (end nodes: 2x)
  REC_NU,        // damping rate
  REC_VMAX2,     // (1e6 sqrt(E/rho))^2
  ER_REC
};
enum { REC2_TIPX = 0, REC2_TIPY, REC2_TIPZ, REC2_ACTA, REC2_ACTF, REC2_ACTIL, REC2_PAD0, REC2_PAD1, ER_REC2 };

// ---- per-slot general parameters (node-indexed planes), general rods only
enum {
  GP_LHAT = 0, GP_ILHAT, GP_S1, GP_S3, GP_IJ1, GP_IJ2, GP_IJ3, GP_KJ1, GP_KJ2, GP_KJ3,  // element at slot
  GP_BV1, GP_BV2, GP_BV3, GP_DH,                                                      // Voronoi at slot
  GP_IM,                                                                              // node at slot
  GP_SK,                                                                              // arc length of node
  ER_GP
};

// ---- rod flags
enum {
  FL_CLAMP_MASK = 3,   // 0 free, 1 clamp s=0 end, 2 clamp s=L end
  FL_GENERAL = 4,      // per-slot parameters from gpar
  FL_TIP = 8,          // tip force present
  FL_ACT = 16,         // rest-curvature actuation
};

struct ErStepParams {
  double *node;  // 6 planes
  double *elem;  // 12 planes
  int64_t nn;    // node plane stride (doubles)
  int64_t ne;    // element plane stride
  const double *rec;
  const double *rec2;
  const int32_t *flags;
  const int64_t *eoff;
  const int32_t *tiles;
  const double *gpar;     // may be null
  int64_t ng;             // gpar plane stride
  const double *sigma0;   // may be null, planes stride ne
  const double *kappa0;   // may be null, planes stride nv
  int64_t nv;
  const double *mag;      // may be null, planes stride ne
  double g[3];
  double b0[3];
  double b_omega;
  int32_t act_comp;
  int32_t n_steps;        // steps in this launch
  double t;               // time at the start of the launch
  double h;               // dt
  unsigned long long *fault;  // [0] = OR of bits, [1] = min rod id
  double *diag_partial;   // diagnostics: [n_tiles][16]
};
