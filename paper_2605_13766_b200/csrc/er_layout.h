// er_layout.h -- device-resident layout of a rod batch (L0) and the kernel parameter block.
//
// HBM layout:
//  - state        : tile-blocked SoA.  The rods are packed into rod-aligned tiles (<= BLOCK
//                   slots, <= BLOCK/8 rods); tile T owns one contiguous block at T.boff:
//                   6 node planes [rx ry rz vx vy vz] x nslots, then ER_EPL = 9 element planes
//                   [d1 (Q00..Q02), d2 (Q10..Q12), wx wy wz] x nel, then (static kappa0 only) 3
//                   Voronoi planes x nvor, padded to 16 bytes.  The third director is not stored:
//                   d3 = d1 x d2 is rebuilt on every load and after every rotation (complete_d3),
//                   so it is the same function of (d1, d2) everywhere (DESIGN §4 "Director
//                   storage"); 48 of the 302 bytes per element-step the 3x3 form would move.  SoA per component inside the block, so every warp
//                   access is coalesced, and one TMA bulk copy moves a whole tile.
//  - rod records  : [n_rods][ER_REC] fp64: derived constants, damping, v_max^2, tip force,
//                   actuation and the flag word -- one 192-byte record read per rod per step
//  - eoff         : [n_rods+4] int64 element offsets (node offset = eoff + rod); padded so
//                   16-byte-aligned bulk copies may over-read
//  - rod order    : rods are stored in a packed (tile) order, ord[p] = canonical id of packed rod
//                   p -- the identity unless rod lengths differ (best-fit-decreasing tiles); every
//                   per-rod / per-element / per-node device array is in packed order
//  - tiles        : [n_tiles] ErTile
//  - gpar         : optional [ER_GP][ng] per-slot parameters of "general" rods (non-uniform
//                   rest lengths or per-element material), canonical node index
//  - sigma0, mag  : optional [3][ne] element planes (packed rod order)
//  - fext / cext  : optional user external loads, [3][ng] node / [3][ne] element planes
// Ghost nodes exist only in shared memory, never in HBM.
#pragma once
#include <stdint.h>
#include <vector_types.h>

#define ER_QST 6  // stored director components per element (rows d1, d2 of Q)
#define ER_EPL 9  // stored element planes per tile: d1, d2, w

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

enum {
  REC_LHAT = 0,  // rest length (uniform rod)
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
  REC_TIPX,      // tip force (lab)
  REC_TIPY,
  REC_TIPZ,
  REC_ACTA,      // actuation amplitude A
  REC_ACTF,      // actuation frequency f
  REC_ACTIL,     // 1/L of the actuation wave
  REC_FLAGS,     // flag word (int64 bits)
  REC_CANON,     // canonical id of the rod (records are stored in packed rod order)
  ER_REC
};

// per-slot general parameters (node-indexed planes), general rods only
enum {
  GP_LHAT = 0, GP_ILHAT, GP_S1, GP_S3, GP_IJ1, GP_IJ2, GP_IJ3, GP_KJ1, GP_KJ2, GP_KJ3,  // element at slot
  GP_BV1, GP_BV2, GP_BV3, GP_DH,                                                      // Voronoi at slot
  GP_IM,                                                                              // node at slot
  GP_SK,                                                                              // arc length of node
  ER_GP
};

enum {
  FL_CLAMP_MASK = 3,  // 0 free, 1 clamp s=0 end, 2 clamp s=L end
  FL_GENERAL = 4,     // per-slot parameters from gpar
  FL_TIP = 8,         // tip force present
  FL_ACT = 16,        // rest-curvature actuation
  FL_MUS = 32,        // muscular torque wave (side array `musc`)
};

// batch-level feature bits (kernel template parameter)
enum { FEAT_GENERAL = 1, FEAT_KAPPA0 = 2,
       FEAT_EXTRA = 4   /* sigma0 / magnetization / muscle wave (and actuation) */,
       FEAT_CONTACT = 8 /* contact forces from ErStepParams.cfc; launch = kick + drift-2 [+ next drift-1] */,
       FEAT_ACT = 16    /* rest-curvature actuation only (a lighter kernel than FEAT_EXTRA) */,
       FEAT_UNI = 32    /* warp kernels: shared material constants (ErStepParams.umat), 48-byte rod records */ };

// Shared-material batches (warp kernels; DESIGN §4 "Shared material"): when every rod of a batch has
// the same REC_LHAT..REC_VMAX2 and REC_ACTIL, those 17 constants travel in the kernel parameters
// (constant bank: FP64 instructions take them as operands, no shared-memory load) and each rod keeps
// a 48-byte record of what differs per rod -- 144 fewer bytes per rod and step than ER_REC's 192.
enum { WREC_TIPX = 0, WREC_TIPY, WREC_TIPZ, WREC_ACTA, WREC_ACTF,
       WREC_FC,  // flag word (low 32 bits) | canonical rod id (high 32 bits)
       ER_WREC };
#define ER_UMAT 17  // umat[0..15] = REC_LHAT..REC_VMAX2, umat[16] = REC_ACTIL

// canonical fields (er_get_state / er_set_state order)
enum { FIELD_POS = 0, FIELD_VEL = 1, FIELD_DIR = 2, FIELD_OMEGA = 3, FIELD_KAPPA0 = 4 };

// Tile descriptor (128 bytes, 16-byte aligned so a TMA bulk copy can stage it).  smask marks
// the slots that start a rod; pfx[w] counts the rod starts in words < w, so the rod of slot s
// is pfx[s/32] + popc(smask[s/32] & lanemask_le) - 1.
struct __align__(16) ErTile {
  int32_t r0;      // first rod                       (r0..nel: one 16-byte load)
  int32_t nr;      // rods in the tile
  int32_t nslots;  // nodes (= slots) in the tile
  int32_t nel;     // elements in the tile
  int64_t nbase;   // first node of the tile (canonical index)
  int64_t ebase;   // first element of the tile (canonical index)
  int64_t boff;    // offset of the tile's state block (doubles, even)
  uint32_t smask[16];
  uint8_t pfx[16];
  int32_t seg;     // long rods (> 511 elements): segment k of the rod's nseg tiles of
  int32_t nseg;    //   ER_LONG_SEG slots each, advanced by a thread-block cluster; else 0 / 1
};
#ifndef ER_LONG_SEG
#define ER_LONG_SEG 256     // slots per segment of a long rod (one CTA of the cluster)
#endif
#define ER_LONG_MAXSEG 16   // cluster size limit (non-portable 16 on sm_100a): N + 1 <= 4096

// Contact law (DESIGN §3 #27): penalty normal force with damping, regularised
// Coulomb friction, optional half-space n.x >= d.
struct ErContactLaw {
  double k_n;             // > 0: fixed stiffness; else min(E_a r_a, E_b r_b) per pair (kr below)
  double gamma_n;
  double mu_s, mu_k, v_stick;
  double pn[3], pd;       // plane (unit normal, offset)
  int32_t plane_on;
  int32_t exclude;        // same-rod pairs with |j - k| <= exclude never touch
};

// Broad phase (hierarchical hash grid) + narrow phase buffers, all device memory.
#define ER_HHG_MAXLEV 8
#define ER_CELL_MIXED (-1ll)   // hash bucket holding proxies of more than one cell
#define ER_CAND_K 16           // candidate list slots per element (longer lists are re-visited)
#define ER_CAND_CROSS (1 << 30) // candidate flag: the partner is on a coarser level (leave it a record)
struct ErContactParams {
  ErContactLaw law;
  double cell[ER_HHG_MAXLEV];   // level l holds the proxies whose AABB's largest extent is
  double icell[ER_HHG_MAXLEV];  // <= cell[l] (= cell[0] * 2^l), the smallest such level
  int32_t nlev;
  int32_t hbits;                // hash table size 2^hbits
  double skin;                  // Verlet skin: proxies are AABBs grown by skin/2; lists are rebuilt
                                //   when a node has moved more than skin/2 since the last build
  int64_t n_elems, n_nodes, n_rods;
  const double *rad;            // [R] contact radius
  const double *kr;             // [R] E r (pair stiffness scale)
  const int32_t *erod;          // [E] rod of each element (packed ids, like every array here)
  const int32_t *ord;           // [R] packed -> canonical rod (fault reports)
  const double *nrad, *nkr;     // [n_nodes] contact radius / E r of the node's rod
  double *cnode;                // [n_nodes][6] node r, v after drift-1 (AoS: an element's two
                                //   nodes are 96 contiguous bytes)
  double *cbuild;               // [n_nodes][3] node positions at the last list build
  int32_t *rebuild;             // [1] device flag: rebuild the lists this step
  unsigned long long *gext;     // [nlev][3] max AABB extent per level and axis (double bits), at build
  double *gdim;                 // [nlev][4] cell box per level (x, y, z) and 1 if populated
  uint32_t *key, *key_s;        // [E] bucket keys, unsorted / sorted
  int32_t *val, *val_s;         // [E] element ids, unsorted / sorted
  longlong2 *table;             // [2^hbits] bucket: (start | end << 32, cell code of a pure bucket
                                //   or ER_CELL_MIXED); start = -1 (all bits set): empty
  long long *code_s;            // [E] cell code (level, cx, cy, cz) of each sorted proxy
  float4 *boxa, *boxb;          // [E] sorted proxies: float AABB (lo rounded down, hi up);
                                //     boxa.w = element id bits, boxb.w = rod id bits
  int32_t *qidx;                // [E] sorted position of each element
  int32_t *cnt;                 // [E] candidates of each element (at the last build)
  int32_t *cand;                // [ER_CAND_K][E] the first ER_CAND_K of them: the partner's first
                                //   node | ER_CAND_CROSS when the partner is on a coarser level
  double *fc;                   // [6][fs] contact force on the element's (node j, node j+1)
  int64_t fs;
  int32_t *head;                // [n_nodes] cross-level records per coarse element, filed under its
                                //   first node (-1 = none)
  int32_t *pnext, *psrc;        // [pcap] record chain / source (fine) element's first node
  double *pf;                   // [pcap][6] record force on the coarse element's two nodes
  int64_t pcap;
  unsigned long long *ctr;      // [8] per step: 0 pool used, 1 contacts, 2 cross-level contacts,
                                //      3 plane contacts
  unsigned long long *bctr;     // [8] of the last build: 0 candidate pairs, 1 list entries (both
                                //      sides), 2 proxies scanned, 3 level mask, 4 long lists;
                                //      5 builds so far (cumulative)
  unsigned long long *fault;    // shared with the step kernels
};

struct ErStepParams {
  double *state;          // tile-blocked state
  const double *rec;
  const int64_t *eoff;     // [n_rods+4] element offsets in packed rod order
  const int32_t *ord;      // [n_rods] packed -> canonical rod
  const int64_t *eoffc;    // [n_rods+1] canonical element offsets
  const ErTile *tiles;
  int64_t n_tiles;
  int64_t state_doubles;  // size of `state` (bounds checks of -DER_CHECK_BOUNDS=1 builds)
  const double *gpar;     // may be null
  int64_t ng;             // gpar plane stride
  const double *sigma0;   // may be null, planes stride ne
  const double *mag;      // may be null, planes stride ne
  const double *musc;     // may be null: [n_rods][4] = A, 1/T, 1/lambda, phi/pi
  const double *fext;     // may be null: user node forces f (lab), planes stride ng
  const double *cext;     // may be null: user element couples c-bar (local), planes stride ne
  int64_t ne;
  int32_t has_kappa0;     // static kappa0 planes present in the tile blocks
  int32_t act_comp;
  int32_t musc_comp;
  int32_t pad2_;
  double g[3];
  double b0[3];           // b(t) = b0 cos(b_omega t) + b1 sin(b_omega t) + b2
  double b1[3];
  double b2[3];
  double b_omega;
  int32_t n_steps;        // steps in this launch
  int32_t tpar;           // with tdev: the launch reads tdev[tpar], block 0 writes tdev[tpar ^ 1]
  double t;               // time at the start of the launch (when tdev is null)
  double *tdev;           // CUDA-graph step launches: [2] device time, ping-pong
  double h;               // dt
  unsigned long long *fault;  // [0] = OR of bits, [1] = min rod id
  double *diag_partial;   // diagnostics: [n_tiles][16]
  unsigned long long *trace;  // optional timeline (measurement aid): [cta][ER_TRACE_ITERS][4]
  // contact (NEXT-4): null cfc = rods do not interact
  const double *cfc;      // [6][cfs] contact force on each element's two nodes (ErContactParams.fc)
  int64_t cfs;
  double *cnode;          // drift-1 stage: [n_nodes][6] node r, v for the contact phase
  const double *cbuild;   // [n_nodes][3] positions at the last contact-list build
  double disp2;           // (skin/2)^2: a larger squared displacement since the build ...
  int32_t *rebuild;       // ... sets this flag
  int32_t sweeps;         // tile kernel: passes over all tiles in this launch (one step each), >= 1
  int32_t pad3_;
  // warp-local kernel (er_warp.cu): uniform rods of ER_WARP_MIN_N..32 elements, each rod on N lanes
  // of one warp (lane = element; the rod's last lane also owns node N), wR rods per warp, 8 warps
  // per tile; neighbour values move by warp shuffles, warps never wait for each other
  int32_t wN;             // elements per rod (0: the batch does not use the warp kernel)
  int32_t wR;             // rods per warp (floor(32 / wN))
  int32_t wnb;            // stage buffers per CTA
  int32_t wbufd;          // doubles per stage buffer (state block | rod records | tile descriptor)
  int32_t wrec;           // offset of the rod records in a buffer (doubles)
  int32_t wdesc;          // offset of the tile descriptor in a buffer (doubles)
  // per-warp streaming variant (warp_stream): uniform tiles of wrt rods, blocks of wcs doubles
  int32_t wrt;            // rods per tile (all tiles but the last are full)
  int32_t wch;            // doubles per warp stage slot (node | element | kappa0 planes | records)
  int64_t wcs;            // doubles per full tile block (tile t starts at t * wcs)
  int64_t wrods;          // rods in the tile part of the batch
  int32_t wl2pf;          // warp_bulk: L2 prefetch distance in tiles beyond the slot ring (0 = none)
  int32_t wuni;           // shared-material batch: wrecu / umat are valid (FEAT_UNI kernels)
  const double *wrecu;    // [n_rods][ER_WREC] compact rod records (packed order)
  double umat[ER_UMAT];   // the shared material constants
};
#ifndef ER_WB_WARPS
#define ER_WB_WARPS 8  // warp_bulk: warps per CTA (measurement builds may change it with ER_WB_MINB)
#endif
#ifndef ER_WB_MINB
#define ER_WB_MINB 2   // warp_bulk: CTAs per SM its register budget is compiled for
#endif
#define ER_WARP_MIN_N 4     // warp kernel: <= 8 rods per warp, <= 64 per tile (the record staging)
#define ER_TRACE_ITERS 64
#ifndef ER_TRACE
#define ER_TRACE 0  // per-tile timeline compiled in (measurement builds: -DER_TRACE=1)
#endif
#ifndef ER_CHECK_BOUNDS
#define ER_CHECK_BOUNDS 0  // debug builds (-DER_CHECK_BOUNDS=1): index checks that trap (the pool has no sanitizer)
#endif
#define ER_CHECK(cond)                                                      \
  do {                                                                      \
    if (ER_CHECK_BOUNDS && !(cond)) {                                       \
      printf("ER_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);   \
      __trap();                                                             \
    }                                                                       \
  } while (0)

// offsets inside a tile block (doubles)
__host__ __device__ inline int64_t tile_node_plane(const ErTile &T, int c) { return (int64_t)c * T.nslots; }
__host__ __device__ inline int64_t tile_elem_plane(const ErTile &T, int c) {
  return 6 * (int64_t)T.nslots + (int64_t)c * T.nel;
}
// Voronoi domains of a tile: one per element except each rod's first (a long rod's first
// element is in its segment 0)
__host__ __device__ inline int32_t tile_nvor(const ErTile &T) { return T.nel - (T.seg == 0 ? T.nr : 0); }
__host__ __device__ inline int64_t tile_vor_plane(const ErTile &T, int c) {
  return 6 * (int64_t)T.nslots + ER_EPL * (int64_t)T.nel + (int64_t)c * tile_nvor(T);
}
__host__ __device__ inline int64_t tile_block_size(const ErTile &T, int has_kappa0) {
  const int64_t sz = 6 * (int64_t)T.nslots + ER_EPL * (int64_t)T.nel + (has_kappa0 ? 3 * (int64_t)tile_nvor(T) : 0);
  return (sz + 1) & ~1ll;
}
static_assert(sizeof(ErTile) == 128, "ErTile must stay 128 bytes (bulk-copied)");
