// er_api.cu -- host implementation of the C-ABI (L3) declared in include/er.h.
//
// Validation (collect-all), the rod-layout builder (offsets, derived per-rod
// constants, rod-aligned tiles, tile-blocked SoA state), device allocation, stream-ordered
// stepping with one fault-word read per er_step, state read-back and the diagnostics
// reduction.  Nothing here does per-element physics on the host: every step of the path runs
// in er_kernels.cu.
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "er.h"
#include "er_layout.h"

extern "C" {
cudaError_t er_launch_step(const ErStepParams *p, int block, int kind, int feat, cudaStream_t st);
cudaError_t er_launch_warp(const ErStepParams *p, int feat, cudaStream_t st);
cudaError_t er_contact_ghost_check(const ErContactParams *pp, int64_t n0, double disp2, cudaStream_t st);
cudaError_t er_launch_long(const ErStepParams *p, int64_t tile0, int64_t n_rods, int nseg, int feat, cudaStream_t st);
cudaError_t er_launch_diag(const ErStepParams *p, int block, double *out, cudaStream_t st);
cudaError_t er_launch_canon_tiles(const ErStepParams *p, double *canon, int field, int to_tiles, cudaStream_t st);
cudaError_t er_launch_aos_to_soa(const double *src, double *dst, int64_t n, int k, int64_t stride, cudaStream_t st);
cudaError_t er_launch_pack_planes(const double *src, double *dst, int64_t stride, const int64_t *eoffp,
                                  const int32_t *ord, const int64_t *eoffc, int64_t n_rods, int nodes, cudaStream_t st);
cudaError_t er_launch_validate(const double *aos, int64_t n, int k, int orth, double *out, cudaStream_t st);
cudaError_t er_launch_compact_records(const double *rec, int64_t n_rods, double *wrec, int *differ, cudaStream_t st);
cudaError_t er_launch_apply_forcing(double *rec, int64_t n_rods, const int32_t *flags, const double *damping,
                                    double damping_all, const double *tip, const double *actA, const double *actF,
                                    const double *actL, int forcing, cudaStream_t st);
cudaError_t er_contact_tmp_bytes(int64_t n, int bits, size_t *bytes);
cudaError_t er_contact_eval(const ErContactParams *p, void *tmp, size_t tmp_bytes, cudaGraphExec_t exec,
                            cudaStream_t st, int64_t *launches, int graph_kernels);
cudaError_t er_contact_graph(const ErContactParams *p, void *tmp, size_t tmp_bytes, cudaGraphExec_t *exec, int *kernels);
}

#include <chrono>

#define ER_GRAPH_LAUNCHES 32  // step launches per CUDA-graph launch (even: the time ping-pong)

namespace {

// NVTX range around each public call (SURVEY §5 tracing): visible to ncu --nvtx / nsys; the calls
// cost nothing measurable when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};


thread_local std::string g_create_error;

// Optional phase timing of er_create_batch (env ER_TIMING=1), printed to stderr.
struct PhaseTimer {
  bool on = std::getenv("ER_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char *what, cudaStream_t st = nullptr) {
    if (!on) return;
    if (st) cudaStreamSynchronize(st);
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[er_create_batch] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

int64_t pad_to(int64_t n, int64_t q) { return ((n + q - 1) / q) * q + q; }

struct Errors {
  std::string msg;
  int count = 0;
  void add(const char *fmt, ...) {
    if (count < 64) {
      char buf[512];
      va_list ap;
      va_start(ap, fmt);
      vsnprintf(buf, sizeof buf, fmt, ap);
      va_end(ap);
      if (!msg.empty()) msg += "; ";
      msg += buf;
    } else if (count == 64) {
      msg += "; ...";
    }
    ++count;
  }
};

}  // namespace

struct er_batch {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t n_rods = 0, n_elems = 0, n_nodes = 0, n_vor = 0;
  int32_t max_n = 0;
  int block = 256;
  // warp kernel (er_warp.cu): equal-length rods of ER_WARP_MIN_N..32 elements; 0 = not used
  int32_t wN = 0, wR = 0, wnb = 0, wbufd = 0, wrec = 0, wdesc = 0;
  int32_t wrt = 0, wch = 0;    // per-warp streaming variant (0: the tile-pipelined warp kernel)
  // ghost rods (contact across GPUs, er_set_contact_ghosts): contact geometry only, packed after the
  // own rods in the contact arrays; node records supplied by the caller every split step
  int64_t g_rods = 0, g_elems = 0, g_nodes = 0;
  std::vector<int32_t> g_nel;
  std::vector<double> g_rad, g_kr, g_lmin, g_lmax;
  int32_t *d_cord = nullptr;   // packed -> reported rod id for own + ghost rods (contact faults)
  er_contact saved_contact{};  // the last er_set_contact parameters (ghost changes re-apply them)
  std::vector<double> saved_radius;
  bool have_saved_contact = false;
  int split_mode = 0;          // er_step internals: 0 whole steps, 1 begin (drift-1), 2 finish
  bool split_begun = false;
  double split_dt = 0.0;
  int64_t wcs = 0, wrods = 0;
  int64_t n_tiles = 0;       // all tiles (layout conversion, diagnostics)
  int64_t n_tiles_norm = 0;  // tiles of rods with <= 511 elements (the step kernels); long rods'
  struct LongGroup { int64_t tile0, n_rods; int nseg; };  // segment tiles follow, by cluster size
  std::vector<LongGroup> long_groups;
  double t = 0.0;
  int64_t steps_per_launch = 1;
  int64_t sweeps = ER_DEFAULT_SWEEPS;  // ER_OPT_SWEEPS_PER_LAUNCH
  int kernel_mode = 0;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  // device buffers
  double *d_state = nullptr;  // tile-blocked SoA state (+ static kappa0 planes)
  int64_t state_doubles = 0;
  int64_t ng = 0, ne = 0;     // canonical plane strides of gpar (nodes) and sigma0/mag (elements)
  double *d_rec = nullptr;
  double *d_wrecu = nullptr;  // shared-material warp batches: [n_rods][ER_WREC] compact records
  bool wuni = false;          // ... valid (every rod has the same material constants, umat)
  double umat[ER_UMAT] = {};
  int *d_uni_flag = nullptr;
  int64_t *d_eoff = nullptr;
  ErTile *d_tiles = nullptr;
  double *d_gpar = nullptr, *d_sigma0 = nullptr, *d_mag = nullptr, *d_musc = nullptr;
  double *d_fext = nullptr, *d_cext = nullptr;  // user external loads (er_set_external_loads)
  unsigned long long *d_fault = nullptr;
  unsigned long long *trace = nullptr;  // caller-owned, optional
  double *d_diag_partial = nullptr, *d_diag_out = nullptr, *d_valid = nullptr;
  bool has_kappa0 = false, any_general = false, has_sigma0 = false, has_act = false, has_musc = false;
  int musc_comp = 0;
  // host mirrors
  // Rods are stored in a packed order (tile order): packed rod p is canonical rod ord[p].  The
  // order is the identity unless the rod lengths differ, when a best-fit-decreasing packing fills
  // the tiles.  Per-rod and per-element device arrays are all in packed order; the
  // API converts at its boundary.
  std::vector<int32_t> ord;        // packed -> canonical rod
  bool identity = true;
  std::vector<int32_t> n_elems_h;  // packed
  std::vector<int64_t> eoff;       // packed element offsets
  std::vector<int64_t> eoffc;      // canonical element offsets
  int32_t *d_ord = nullptr;
  int64_t *d_eoffc = nullptr;
  std::unique_ptr<double[]> rec;  // host records during create (not value-initialised)
  size_t rec_n = 0;
  std::vector<int32_t> flags;
  double g[3] = {0, 0, 0};
  double b0[3] = {0, 0, 0}, b1[3] = {0, 0, 0}, b2[3] = {0, 0, 0};  // b(t) = b0 cos + b1 sin + b2
  double b_omega = 0.0;
  int act_comp = 0;
  int64_t fault_rod = -1;
  int32_t fault_bits = 0;
  std::string last_error;
  double *upload_stage = nullptr;  // during er_create_batch: device staging of the host state arrays
  double *staged[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // per field, inside upload_stage
  // contact (NEXT-4)
  bool contact_on = false;
  ErContactParams cp{};
  void *sort_tmp = nullptr;
  size_t sort_bytes = 0;
  // ER_OPT_PHASE_TIMING: event pool, this call's intervals (start, end, phase), running sums
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> iv;  // (start event, end event, phase, launches) quadruples
  double phase_ms[2] = {0.0, 0.0};
  int64_t phase_n[2] = {0, 0};
  cudaGraphExec_t cgraph = nullptr;  // per-step contact evaluation (conditional build)
  // streaming steps as a CUDA graph of ER_GRAPH_LAUNCHES step launches (no host launch per step);
  // the launch time lives in tdev (ping-pong); rebuilt when its parameters change
  cudaGraphExec_t sgraph = nullptr;
  int64_t sgraph_key = -1;
  uint64_t sgraph_h_bits = 0;   // the step size captured into sgraph (ErStepParams.h, by value)
  bool sgraph_while = false;    // sgraph repeats its 32 launches in a device-side WHILE loop
  long long *d_loop = nullptr;  // its iteration counter
  double *tdev = nullptr;
  int64_t forcing_version = 0;
  int cgraph_kernels = 0;
  std::vector<double> rod_A0, rod_E0, rod_lmin, rod_lmax;  // host, per rod (contact radius, stiffness, HHG)
};

namespace {

// Best-fit-decreasing packing of rods (n + 1 slots each) into tiles of `cap` slots and at most
// `rmax` rods: rods by decreasing length, each into the fullest tile it still fits; tiles listed
// by their lowest rod id, rods inside a tile in canonical order.  Returns packed -> canonical.
std::vector<int32_t> pack_rods(const int32_t *n, int64_t R, int cap, int rmax) {
  std::vector<int32_t> idx((size_t)R);
  for (int64_t r = 0; r < R; ++r) idx[r] = (int32_t)r;
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return n[a] > n[b]; });
  std::vector<std::vector<int32_t>> bins;
  std::vector<int> room;
  std::multimap<int, int> open;  // remaining slots -> bin
  for (int32_t r : idx) {
    const int need = n[r] + 1;
    auto it = open.lower_bound(need);
    int bin;
    if (it == open.end()) {
      bin = (int)bins.size();
      bins.emplace_back();
      room.push_back(cap);
    } else {
      bin = it->second;
      open.erase(it);
    }
    bins[bin].push_back(r);
    room[bin] -= need;
    if ((int)bins[bin].size() < rmax && room[bin] >= 2) open.emplace(room[bin], bin);
  }
  for (auto &bn : bins) std::sort(bn.begin(), bn.end());
  std::sort(bins.begin(), bins.end(), [](const std::vector<int32_t> &a, const std::vector<int32_t> &b) { return a[0] < b[0]; });
  std::vector<int32_t> ord;
  ord.reserve((size_t)R);
  for (auto &bn : bins) ord.insert(ord.end(), bn.begin(), bn.end());
  return ord;
}

// Rows of a canonical per-element (or per-rod) array in packed order (host copy), k doubles/row.
std::vector<double> pack_rows(const er_batch *b, const double *src, int k, bool per_elem) {
  std::vector<double> out;
  if (!src) return out;
  const int64_t R = b->n_rods;
  out.resize((size_t)(per_elem ? b->n_elems : R) * k);
  for (int64_t p = 0; p < R; ++p) {
    const int32_t r = b->ord[p];
    if (per_elem)
      std::memcpy(&out[(size_t)b->eoff[p] * k], src + b->eoffc[r] * k, sizeof(double) * (size_t)(b->n_elems_h[p] * k));
    else
      std::memcpy(&out[(size_t)p * k], src + (int64_t)r * k, sizeof(double) * k);
  }
  return out;
}

er_status cuda_fail(er_batch *b, cudaError_t e, const char *what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (b) b->last_error = m; else g_create_error = m;
  return e == cudaErrorMemoryAllocation ? ER_ENOMEM : ER_ECUDA;
}

#define CK(call, what)                                    \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(b, e_, what); \
  } while (0)

template <class T>
cudaError_t dalloc(er_batch *b, T **p, int64_t count) {
  *p = nullptr;
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)count);
  if (e == cudaSuccess) b->device_bytes += (int64_t)(sizeof(T) * (size_t)count);
  return e;
}

void free_contact(er_batch *b) {
  ErContactParams &c = b->cp;
  void *ptrs[] = {(void *)c.rad, (void *)c.kr, (void *)c.erod, (void *)c.nrad, (void *)c.nkr, c.cnode, c.cbuild, c.rebuild, c.gext, c.gdim, c.key,
                  c.key_s, c.val, c.val_s, c.table, c.code_s, c.boxa, c.boxb, c.qidx, c.cnt, c.cand, c.fc, c.head,
                  c.pnext, c.psrc, c.pf, c.ctr, c.bctr, b->sort_tmp};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (b->cgraph) cudaGraphExecDestroy(b->cgraph);
  b->cgraph = nullptr;
  b->cp = ErContactParams{};
  if (b->d_cord) cudaFree(b->d_cord);
  b->d_cord = nullptr;
  b->sort_tmp = nullptr;
  b->sort_bytes = 0;
  b->contact_on = false;
}

// Phase timing: mark() records an event on the stream and returns its index (-1 when off).
int mark(er_batch *b) {
  if (!b->timing) return -1;
  if (b->ev_used == b->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    b->ev_pool.push_back(e);
  }
  const int k = (int)b->ev_used++;
  cudaEventRecord(b->ev_pool[k], b->stream);
  return k;
}
void interval(er_batch *b, int e0, int e1, int phase, int launches = 1) {
  if (e0 >= 0 && e1 >= 0) { b->iv.push_back(e0); b->iv.push_back(e1); b->iv.push_back(phase); b->iv.push_back(launches); }
}
void collect_times(er_batch *b) {  // after the stream was synchronised
  for (size_t k = 0; k + 3 < b->iv.size(); k += 4) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, b->ev_pool[b->iv[k]], b->ev_pool[b->iv[k + 1]]) == cudaSuccess) {
      b->phase_ms[b->iv[k + 2]] += ms;
      b->phase_n[b->iv[k + 2]] += b->iv[k + 3];
    }
  }
  b->iv.clear();
  b->ev_used = 0;
}

// WHILE-loop control of the step graph: one more pass of its 32 launches while the counter lasts.
__global__ void er_step_loop_ctl(long long *counter, cudaGraphConditionalHandle h) {
  const long long left = --*counter;
  cudaGraphSetConditional(h, left > 0 ? 1u : 0u);
}

void free_step_graph(er_batch *b) {
  if (b->sgraph) cudaGraphExecDestroy(b->sgraph);
  b->sgraph = nullptr;
  b->sgraph_key = -1;
}

void free_all(er_batch *b) {
  free_step_graph(b);
  if (b->d_loop) cudaFree(b->d_loop);
  b->d_loop = nullptr;
  if (b->tdev) cudaFree(b->tdev);
  b->tdev = nullptr;
  if (b->upload_stage) cudaFree(b->upload_stage);
  b->upload_stage = nullptr;
  for (cudaEvent_t e : b->ev_pool) cudaEventDestroy(e);
  b->ev_pool.clear();
  void *ptrs[] = {b->d_state, b->d_rec, b->d_wrecu, b->d_uni_flag, b->d_eoff, b->d_ord, b->d_eoffc, b->d_tiles, b->d_gpar, b->d_sigma0, b->d_mag, b->d_musc,
                  b->d_fext, b->d_cext,
                  b->d_fault, b->d_diag_partial, b->d_diag_out, b->d_valid};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  free_contact(b);
  if (b->own_stream && b->stream) cudaStreamDestroy(b->stream);
}

bool pos_finite(double x) { return std::isfinite(x) && x > 0.0; }

// First index k < n with !ok(a[k]), or -1; large arrays are scanned by host threads.
template <class Ok>
int64_t first_bad(const double *a, int64_t n, Ok ok) {
  const int nthr = (int)std::max<unsigned>(1u, std::min<unsigned>(16u, std::thread::hardware_concurrency()));
  auto scan = [&](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k)
      if (!ok(a[k])) return k;
    return (int64_t)-1;
  };
  if (n < (1 << 20) || nthr == 1) return scan(0, n);
  std::vector<int64_t> res((size_t)nthr, -1);
  std::vector<std::thread> th;
  for (int q = 0; q < nthr; ++q) th.emplace_back([&, q] { res[q] = scan(n * q / nthr, n * (q + 1) / nthr); });
  for (auto &t : th) t.join();
  for (int64_t x : res)
    if (x >= 0) return x;
  return -1;
}

ErStepParams params_of(const er_batch *b) {
  ErStepParams p;
  std::memset(&p, 0, sizeof p);
  p.state = b->d_state;
  p.rec = b->d_rec; p.eoff = b->d_eoff; p.tiles = b->d_tiles; p.n_tiles = b->n_tiles;
  p.state_doubles = b->state_doubles;
  p.sweeps = 1;
  p.ord = b->d_ord; p.eoffc = b->d_eoffc;
  p.gpar = b->d_gpar; p.ng = b->ng; p.sigma0 = b->d_sigma0; p.mag = b->d_mag; p.ne = b->ne;
  p.fext = b->d_fext; p.cext = b->d_cext;
  p.musc = b->has_musc ? b->d_musc : nullptr;
  p.musc_comp = b->musc_comp;
  p.has_kappa0 = b->has_kappa0 ? 1 : 0;
  for (int c = 0; c < 3; ++c) { p.g[c] = b->g[c]; p.b0[c] = b->b0[c]; p.b1[c] = b->b1[c]; p.b2[c] = b->b2[c]; }
  p.b_omega = b->b_omega; p.act_comp = b->act_comp;
  p.fault = b->d_fault; p.diag_partial = b->d_diag_partial;
  p.trace = b->trace;
  p.wN = b->wN; p.wR = b->wR; p.wnb = b->wnb; p.wbufd = b->wbufd; p.wrec = b->wrec; p.wdesc = b->wdesc;
  p.wrt = b->wrt; p.wch = b->wch; p.wcs = b->wcs; p.wrods = b->wrods;
  p.wuni = b->wuni ? 1 : 0;
  p.wrecu = b->d_wrecu;
  for (int k = 0; k < ER_UMAT; ++k) p.umat[k] = b->umat[k];
  {
    static const int l2pf = std::getenv("ER_WARP_L2PF") ? std::atoi(std::getenv("ER_WARP_L2PF")) : 0;
    p.wl2pf = l2pf;
  }
  return p;
}

// Field sizes in canonical AoS order.
int64_t field_rows(const er_batch *b, int field) {
  return field <= FIELD_VEL ? b->n_nodes : field <= FIELD_OMEGA ? b->n_elems : b->n_vor;
}
int field_k(int field) { return field == FIELD_DIR ? 9 : 3; }

// Canonical AoS array (host or device, or NULL = zeros) -> tile-blocked planes.  With
// `validate`, non-finite counts (and, for directors, max |QQ^T - I| and |det Q - 1|)
// accumulate in d_valid.
// Device alias of a page-locked host pointer (pinned or registered memory is mapped into the
// device address space under UVA), or nullptr for pageable memory.  er_get_state's layout
// kernel then writes host memory directly over PCIe (posted writes run at the DMA rate; reads
// of host memory from a kernel do not, so uploads keep the DMA copy into a staging buffer).
double *mapped_host(const void *h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer ? static_cast<double *>(a.devicePointer) : nullptr;
}

er_status upload_field(er_batch *b, const double *src, int src_mem, int field, bool validate) {
  const int64_t n = field_rows(b, field);
  if (n <= 0) return ER_OK;
  ErStepParams p = params_of(b);
  const int k = field_k(field);
  if (src == nullptr) {
    CK(er_launch_canon_tiles(&p, nullptr, field, 1, b->stream), "zero field");
    return ER_OK;
  }
  const double *dsrc = src;
  double *stage = nullptr;
  if (src_mem == ER_HOST && b->staged[field]) {  // copied at the start of er_create_batch
    dsrc = b->staged[field];
  } else if (src_mem == ER_HOST) {  // DMA into a temporary device buffer
    CK(cudaMallocAsync((void **)&stage, sizeof(double) * (size_t)(n * k), b->stream), "cudaMallocAsync(stage)");
    CK(cudaMemcpyAsync(stage, src, sizeof(double) * (size_t)(n * k), cudaMemcpyHostToDevice, b->stream), "H2D");
    dsrc = stage;
  }
  if (validate) CK(er_launch_validate(dsrc, n, k, field == FIELD_DIR, b->d_valid, b->stream), "validate");
  CK(er_launch_canon_tiles(&p, const_cast<double *>(dsrc), field, 1, b->stream), "canon->tiles");
  if (stage) CK(cudaFreeAsync(stage, b->stream), "cudaFreeAsync");
  return ER_OK;
}

er_status download_field(er_batch *b, double *dst, int dst_mem, int field) {
  const int64_t n = field_rows(b, field);
  if (dst == nullptr || n <= 0) return ER_OK;
  ErStepParams p = params_of(b);
  const int k = field_k(field);
  if (dst_mem == ER_DEVICE) {
    CK(er_launch_canon_tiles(&p, dst, field, 0, b->stream), "tiles->canon");
    return ER_OK;
  }
  if (double *hm = mapped_host(dst)) {  // page-locked host array: written directly
    CK(er_launch_canon_tiles(&p, hm, field, 0, b->stream), "tiles->canon(host)");
    return ER_OK;
  }
  double *stage = nullptr;
  CK(cudaMallocAsync((void **)&stage, sizeof(double) * (size_t)(n * k), b->stream), "cudaMallocAsync(stage)");
  CK(er_launch_canon_tiles(&p, stage, field, 0, b->stream), "tiles->canon");
  CK(cudaMemcpyAsync(dst, stage, sizeof(double) * (size_t)(n * k), cudaMemcpyDeviceToHost, b->stream), "D2H");
  CK(cudaFreeAsync(stage, b->stream), "cudaFreeAsync");
  return ER_OK;
}

// Canonical AoS [n][3] (host) -> 3 canonical SoA planes (side arrays: sigma0, magnetization).
er_status upload_side_planes(er_batch *b, const double *src, double *planes, int64_t n, int64_t stride) {
  if (n <= 0) return ER_OK;
  double *stage = nullptr;
  CK(cudaMallocAsync((void **)&stage, sizeof(double) * (size_t)(n * 3), b->stream), "cudaMallocAsync(stage)");
  CK(cudaMemcpyAsync(stage, src, sizeof(double) * (size_t)(n * 3), cudaMemcpyHostToDevice, b->stream), "H2D");
  CK(er_launch_aos_to_soa(stage, planes, n, 3, stride, b->stream), "aos_to_soa");
  CK(cudaFreeAsync(stage, b->stream), "cudaFreeAsync");
  return ER_OK;
}

// Derived constants (DESIGN §3 #5, #9, #10): S = diag(ac G A, ac G A, E A),
// B = diag(E I1, E I2, G (I1+I2)), J = rho lhat diag(I1, I2, I1+I2), m_node = half element masses.
struct ElemMat { double rho, A, I1, I2, E, G, ac, lh; };

void fill_record(double *rec, const ElemMat &m) {
  const double J1 = m.rho * m.lh * m.I1, J2 = m.rho * m.lh * m.I2, J3 = m.rho * m.lh * (m.I1 + m.I2);
  rec[REC_LHAT] = m.lh;
  rec[REC_ILHAT] = 1.0 / m.lh;
  rec[REC_S1] = m.ac * m.G * m.A;
  rec[REC_S3] = m.E * m.A;
  rec[REC_B1] = m.E * m.I1;
  rec[REC_B2] = m.E * m.I2;
  rec[REC_B3] = m.G * (m.I1 + m.I2);
  rec[REC_IJ1] = 1.0 / J1;
  rec[REC_IJ2] = 1.0 / J2;
  rec[REC_IJ3] = 1.0 / J3;
  rec[REC_KJ1] = (J2 - J3) / J1;
  rec[REC_KJ2] = (J3 - J1) / J2;
  rec[REC_KJ3] = (J1 - J2) / J3;
  rec[REC_IM] = 1.0 / (m.rho * m.A * m.lh);
  const double vmax = 1e6 * std::sqrt(m.E / m.rho);
  rec[REC_VMAX2] = vmax * vmax;
}

// The flag word lives inside each rod record (REC_FLAGS), so one bulk copy brings it along.
void sync_flags(er_batch *b) {
  for (int64_t r = 0; r < b->n_rods; ++r) {
    const int64_t bits = (int64_t)b->flags[r];
    std::memcpy(&b->rec[(size_t)r * ER_REC + REC_FLAGS], &bits, sizeof bits);
  }
}

int feat_of(const er_batch *b) {
  int f = 0;
  if (b->any_general) f |= FEAT_GENERAL;
  if (b->has_kappa0) f |= FEAT_KAPPA0;
  if (b->has_sigma0 || b->d_mag || b->has_musc || b->d_fext || b->d_cext) f |= FEAT_EXTRA;
  else if (b->has_act) f |= FEAT_ACT;  // actuation alone: the lighter kernel
  return f;
}

er_status upload_records(er_batch *b) {
  sync_flags(b);
  if (b->n_rods > 0)
    CK(cudaMemcpyAsync(b->d_rec, b->rec.get(), sizeof(double) * b->rec_n, cudaMemcpyHostToDevice, b->stream),
       "H2D rec");
  return ER_OK;
}

// Shared-material form of the records (DESIGN §4 "Shared material"), after every record change: for a
// warp-layout batch without per-slot parameters, a kernel writes the 48-byte compact records and
// tests whether every rod has rod 0's material constants; if so the warp kernels take those from
// the kernel parameters.  Captured step graphs hold the parameters by value: they are re-captured.
er_status refresh_shared_material(er_batch *b) {
  const int64_t R = b->n_rods;
  const bool want = b->wN > 0 && b->wrt > 0 && !b->any_general && R > 0 && std::getenv("ER_NO_UNI") == nullptr;
  bool uni = false;
  if (want) {
    if (!b->d_wrecu) CK(dalloc(b, &b->d_wrecu, R * ER_WREC + 2), "cudaMalloc(wrecu)");
    if (!b->d_uni_flag) CK(cudaMalloc((void **)&b->d_uni_flag, sizeof(int)), "cudaMalloc(uni flag)");
    CK(cudaMemsetAsync(b->d_uni_flag, 0, sizeof(int), b->stream), "memset");
    CK(er_launch_compact_records(b->d_rec, R, b->d_wrecu, b->d_uni_flag, b->stream), "compact records");
    int differ = 1;
    double r0[ER_REC];
    CK(cudaMemcpyAsync(&differ, b->d_uni_flag, sizeof(int), cudaMemcpyDeviceToHost, b->stream), "D2H");
    CK(cudaMemcpyAsync(r0, b->d_rec, sizeof r0, cudaMemcpyDeviceToHost, b->stream), "D2H");
    CK(cudaStreamSynchronize(b->stream), "sync");
    uni = differ == 0;
    if (uni) {
      double u[ER_UMAT];
      for (int k = 0; k <= REC_VMAX2; ++k) u[k] = r0[k];
      u[16] = r0[REC_ACTIL];
      if (std::memcmp(u, b->umat, sizeof u) != 0) {
        std::memcpy(b->umat, u, sizeof u);
        free_step_graph(b);  // captured step graphs hold umat by value
      }
    }
  } else {
    CK(cudaStreamSynchronize(b->stream), "sync");
  }
  if (uni != b->wuni) free_step_graph(b);
  b->wuni = uni;
  return ER_OK;
}

// Upload the per-rod flags (and, with `forcing`, the caller's damping / tip / actuation arrays as
// given) and let a kernel write those record fields -- no 192-byte records cross PCIe again.
er_status apply_forcing(er_batch *b, const er_forcing *f, bool forcing) {
  const int64_t R = b->n_rods;
  if (R == 0) return ER_OK;
  size_t n = (size_t)R;  // int32 flags, packed as doubles below
  const bool damp = forcing && f->damping, tip = forcing && f->tip_force, act = forcing && f->act_A;
  size_t total = (n + 1) / 2 + (damp ? n : 0) + (tip ? 3 * n : 0) + (act ? 3 * n : 0);
  double *d = nullptr;
  CK(cudaMallocAsync((void **)&d, sizeof(double) * (total + 4), b->stream), "cudaMallocAsync(forcing)");
  double *p = d;
  int32_t *dflags = reinterpret_cast<int32_t *>(p);
  CK(cudaMemcpyAsync(dflags, b->flags.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, b->stream), "H2D flags");
  p += (n + 1) / 2;
  const double *ddamp = nullptr, *dtip = nullptr, *dA = nullptr, *dF = nullptr, *dL = nullptr;
  std::vector<std::vector<double>> keep;  // packed-order copies, alive until the final sync
  auto up = [&](const double *src, size_t cnt) -> const double * {
    double *q = p;
    p += cnt;
    if (!b->identity) {  // caller's canonical per-rod rows -> packed order
      keep.push_back(pack_rows(b, src, (int)(cnt / n), false));
      src = keep.back().data();
    }
    return cudaMemcpyAsync(q, src, sizeof(double) * cnt, cudaMemcpyHostToDevice, b->stream) == cudaSuccess ? q : nullptr;
  };
  if (damp) ddamp = up(f->damping, n);
  if (tip) dtip = up(f->tip_force, 3 * n);
  if (act) { dA = up(f->act_A, n); dF = up(f->act_f, n); dL = up(f->act_L, n); }
  CK(cudaGetLastError(), "H2D forcing");
  CK(er_launch_apply_forcing(b->d_rec, R, dflags, ddamp, forcing ? f->damping_all : 0.0, dtip, dA, dF, dL,
                             forcing ? 1 : 0, b->stream), "apply forcing");
  CK(cudaFreeAsync(d, b->stream), "cudaFreeAsync");
  return refresh_shared_material(b);
}

}  // namespace

extern "C" {

int32_t er_abi_version(void) { return ER_ABI_VERSION; }

const char *er_last_error(const er_batch *b) { return b ? b->last_error.c_str() : g_create_error.c_str(); }

er_status er_create_batch(const er_batch_desc *d, er_batch **out) {
  NvtxRange nvtx_("er_create_batch");
  g_create_error.clear();
  if (out) *out = nullptr;
  if (!d || !out) { g_create_error = "desc and out must be non-NULL"; return ER_EINVAL; }
  PhaseTimer tm;
  Errors err;
  const int64_t R = d->n_rods;
  if (R < 0) err.add("n_rods = %lld < 0", (long long)R);
  if (R > 0 && !d->n_elems) err.add("n_elems is NULL");
  if (d->src_mem != ER_HOST && d->src_mem != ER_DEVICE) err.add("src_mem = %d is not ER_HOST/ER_DEVICE", d->src_mem);
  if (err.count) { g_create_error = err.msg; return ER_EINVAL; }

  std::vector<int64_t> eoff((size_t)std::max<int64_t>(R, 0) + 1, 0);
  for (int64_t r = 0; r < R; ++r) {
    const int32_t n = d->n_elems[r];
    if (n < 1 || n > ER_MAX_ELEMS_PER_ROD) err.add("rod %lld: n_elems = %d outside [1, %d]", (long long)r, n, ER_MAX_ELEMS_PER_ROD);
    eoff[r + 1] = eoff[r] + std::max(n, 0);
  }
  // Longest rod that shares rod tiles (lmax); longer rods run as thread-block clusters.  512-slot
  // tiles (1 CTA per SM) only when rods of 256..511 elements carry a real share of the work;
  // otherwise 256-slot tiles (2 CTAs per SM overlap each other's staging) and those few rods go
  // to 2-segment clusters (DESIGN §4 "Tile size").
  int32_t lmax = ER_TILE_MAX_ELEMS;
  if (d->tile_slots == 256 || d->tile_slots == 128) lmax = d->tile_slots - 1;
  if (d->tile_slots == 0 && R > 0) {
    int64_t mid = 0;  // elements in rods of 256..511 elements
    int32_t lo = ER_MAX_ELEMS_PER_ROD, hi = 0;
    for (int64_t r = 0; r < R; ++r) {
      const int32_t n = d->n_elems[r];
      if (n >= 256 && n <= ER_TILE_MAX_ELEMS) mid += n;
      if (n <= ER_TILE_MAX_ELEMS) { lo = std::min(lo, n); hi = std::max(hi, n); }
    }
    if (mid > 0 && lo != hi && (double)mid <= 0.02 * (double)eoff[R] && !std::getenv("ER_NO_MID_CLUSTERS")) lmax = 255;
  }
  int32_t max_n = 0;       // longest tile rod (<= lmax elements)
  int64_t n_long = 0;      // rods longer than that: segments of a thread-block cluster
  for (int64_t r = 0; r < R; ++r) {
    const int32_t n = d->n_elems[r];
    if (n > lmax) ++n_long;
    else max_n = std::max(max_n, n);
  }
  const int64_t E = eoff[R];
  const int64_t NN = E + R, NV = E - R;

  // ---- the device, the batch and the host->device copies of the state come first: from
  // page-locked arrays the DMA then runs under all the host work below (validation, records,
  // tiles); the layout kernels later read the staged copies
  {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) err.add("no CUDA device available");
    else if (d->device < 0 || d->device >= ndev) err.add("device %d outside [0, %d)", d->device, ndev);
  }
  er_batch *b = nullptr;
  if (err.count == 0) {  // (with errors already found: collect the rest, then report them all)
    b = new er_batch();
    b->device = d->device;
    auto early = [&](cudaError_t e, const char *what) {
      cuda_fail(nullptr, e, what);
      free_all(b);
      delete b;
      return e == cudaErrorMemoryAllocation ? ER_ENOMEM : ER_ECUDA;
    };
#undef CK
#define CK(call, what)                              \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return early(e_, what);  \
  } while (0)
    CK(cudaSetDevice(d->device), "cudaSetDevice");
    if (d->stream) b->stream = (cudaStream_t)d->stream;
    else { CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking), "cudaStreamCreate"); b->own_stream = true; }
    // ---- start the host->device copies of the state now: from page-locked arrays the DMA runs
    // while the host builds records and tiles below (the layout kernels use the staged copies)
    {
      const struct { const double *src; int field; int64_t n; } fs[5] = {
          {d->src_mem == ER_HOST ? d->positions : nullptr, FIELD_POS, 3 * NN},
          {d->src_mem == ER_HOST ? d->velocities : nullptr, FIELD_VEL, 3 * NN},
          {d->src_mem == ER_HOST ? d->directors : nullptr, FIELD_DIR, 9 * E},
          {d->src_mem == ER_HOST ? d->omega : nullptr, FIELD_OMEGA, 3 * E},
          {NV > 0 ? d->rest_kappa : nullptr, FIELD_KAPPA0, 3 * NV}};
      int64_t total = 0;
      for (const auto &f : fs) total += f.src ? f.n : 0;
      if (total > 0) {
        CK(cudaMalloc((void **)&b->upload_stage, sizeof(double) * (size_t)total + 64), "cudaMalloc(stage)");
        int64_t o = 0;
        for (const auto &f : fs)
          if (f.src) {
            b->staged[f.field] = b->upload_stage + o;
            CK(cudaMemcpyAsync(b->staged[f.field], f.src, sizeof(double) * (size_t)f.n, cudaMemcpyHostToDevice, b->stream),
               "H2D state");
            o += f.n;
          }
      }
    }
    tm.mark("state copies issued");
  }
  const int64_t nmat = d->material_per_rod ? R : E;
  const char *mnames[7] = {"density", "area", "I1", "I2", "youngs", "shear_mod", "alpha_c"};
  const double *marr[7] = {d->density, d->area, d->I1, d->I2, d->youngs, d->shear_mod, d->alpha_c};
  if (R > 0) {
    auto fin = [](double x) { return std::isfinite(x); };
    for (int q = 0; q < 7; ++q) {
      if (!marr[q]) { err.add("%s is NULL", mnames[q]); continue; }
      const int64_t k = first_bad(marr[q], nmat, pos_finite);
      if (k >= 0) err.add("%s[%lld] = %g is not positive and finite", mnames[q], (long long)k, marr[q][k]);
    }
    if (!d->rest_lengths) err.add("rest_lengths is NULL");
    else if (const int64_t k = first_bad(d->rest_lengths, E, pos_finite); k >= 0)
      err.add("rest_lengths[%lld] = %g is not positive and finite", (long long)k, d->rest_lengths[k]);
    if (!d->positions) err.add("positions is NULL");
    if (!d->directors) err.add("directors is NULL");
    if (d->rest_sigma)
      if (const int64_t k = first_bad(d->rest_sigma, 3 * E, fin); k >= 0) err.add("rest_sigma[%lld] is not finite", (long long)k);
    if (d->rest_kappa)
      if (const int64_t k = first_bad(d->rest_kappa, 3 * NV, fin); k >= 0) err.add("rest_kappa[%lld] is not finite", (long long)k);
  }
  if (!std::isfinite(d->t0)) err.add("t0 is not finite");
  if (d->tile_slots != 0 && d->tile_slots != 128 && d->tile_slots != 256 && d->tile_slots != 512)
    err.add("tile_slots = %d not in {0, 128, 256, 512}", d->tile_slots);
  else if (d->tile_slots != 0 && max_n + 1 > d->tile_slots)
    err.add("tile_slots = %d < longest rod's %d slots", d->tile_slots, max_n + 1);
  else if (d->tile_slots == 128 && n_long > 0)
    err.add("tile_slots = 128 cannot be combined with rods longer than 127 elements");
  if (err.count) {
    g_create_error = err.msg;
    if (b) { free_all(b); delete b; }
    return ER_EINVAL;
  }

  tm.mark("host validation");
  b->n_rods = R; b->n_elems = E; b->n_nodes = NN; b->n_vor = NV; b->max_n = max_n;
  const int64_t Rn = R - n_long;  // tile rods come first in the packed order
  b->t = d->t0;
  b->block = d->tile_slots ? d->tile_slots : (max_n + 1 <= 256) ? 256 : 512;
  int32_t min_n = max_n;
  for (int64_t r = 0; r < R; ++r)
    if (d->n_elems[r] <= lmax) min_n = std::min(min_n, d->n_elems[r]);
  if (!d->tile_slots && b->block == 256 && Rn > 0 && min_n == max_n) {
    // equal-length rods fill a tile with floor(B / (N+1)) of them (<= B/8): take 512-slot tiles
    // when that keeps clearly more lanes busy (65-slot rods: 76% at 256, 89% at 512)
    auto fill = [&](int B) { return (double)std::min<int>(B / (max_n + 1), B / 8) * (max_n + 1) / B; };
    if (Rn * (int64_t)(max_n + 1) >= 4 * 512 && fill(512) > fill(256) + 0.05) b->block = 512;
  }
  // Warp kernel: every rod has the same N in [ER_WARP_MIN_N, 32] elements (no long rods); tiles then
  // hold 8 warps x floor(32/N) rods (ER_WARP_TILE_RODS overrides, measurement), and the tile kernels
  // that still run on them (staged ablations, contact mode, sweeps of small batches, diagnostics)
  // take the block size those tiles need.
  int32_t wtile_rods = 0;
  // Small batches (the tile kernel would run them as sweeps: <= 4 tiles of 256 slots per CTA of the
  // grid) stay in the tile layout: there the launch boundary, not the step, is the cost (cfg2: 11 vs
  // 21 us per step).  ER_WARP=1 forces the warp layout (tests), ER_NO_WARP=1 forbids it.
  const bool warp_size_ok = std::getenv("ER_WARP") != nullptr || R * (int64_t)(max_n + 1) > 4 * 296 * 256;
  if (!d->tile_slots && n_long == 0 && R > 0 && min_n == max_n && max_n >= ER_WARP_MIN_N && warp_size_ok &&
      max_n <= (std::getenv("ER_NO_WARP_PAIR") ? 32 : 64) && std::getenv("ER_NO_WARP") == nullptr) {
    b->wN = max_n;
    b->wR = max_n <= 32 ? 32 / max_n : 1;  // 33..64 elements: one rod per warp pair
    // default: warp-sized tiles (wR rods, one contiguous block per warp) for the per-warp streaming
    // kernel; ER_WARP_TMA=1: tiles of 8 warps for the tile-pipelined warp kernel
    wtile_rods = (std::getenv("ER_WARP_TMA") && max_n <= 32) ? 8 * b->wR : b->wR;
    if (const char *e = std::getenv("ER_WARP_TILE_RODS")) wtile_rods = std::max(1, std::min(8 * b->wR, std::atoi(e)));
    b->block = (int64_t)wtile_rods * (max_n + 1) <= 256 && wtile_rods <= 32 ? 256 : 512;
  }
  {
    // packed order: tile rods (best-fit-decreasing when their lengths differ), then long rods by
    // cluster size (so each size is one launch), canonical order within
    std::vector<int32_t> tile_rods, long_rods;
    for (int64_t r = 0; r < R; ++r) (d->n_elems[r] > lmax ? long_rods : tile_rods).push_back((int32_t)r);
    const bool pack = Rn > 1 && min_n != max_n && std::getenv("ER_NO_PACK") == nullptr;
    if (pack) {
      std::vector<int32_t> nt(tile_rods.size());
      for (size_t q = 0; q < tile_rods.size(); ++q) nt[q] = d->n_elems[tile_rods[q]];
      std::vector<int32_t> o = pack_rods(nt.data(), (int64_t)nt.size(), b->block, b->block / 8);
      for (auto &x : o) x = tile_rods[x];
      tile_rods = o;
    }
    auto nseg = [&](int32_t r) { return (d->n_elems[r] + ER_LONG_SEG) / ER_LONG_SEG; };  // ceil((N+1)/S)
    std::stable_sort(long_rods.begin(), long_rods.end(), [&](int32_t a, int32_t c) { return nseg(a) < nseg(c); });
    b->ord = tile_rods;
    b->ord.insert(b->ord.end(), long_rods.begin(), long_rods.end());
    b->identity = true;
    for (int64_t r = 0; r < R; ++r) b->identity = b->identity && b->ord[r] == r;
  }
  b->eoffc = eoff;
  b->n_elems_h.resize((size_t)R);
  b->eoff.assign((size_t)R + 1, 0);
  for (int64_t p = 0; p < R; ++p) {
    b->n_elems_h[p] = d->n_elems[b->ord[p]];
    b->eoff[p + 1] = b->eoff[p] + b->n_elems_h[p];
  }
  const std::vector<int64_t> &eoffp = b->eoff;
  auto fail = [&](er_status s) { g_create_error = b->last_error; free_all(b); delete b; return s; };
#undef CK
#define CK(call, what)                                                 \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) { cuda_fail(b, e_, what); return fail(e_ == cudaErrorMemoryAllocation ? ER_ENOMEM : ER_ECUDA); } \
  } while (0)

  // ---- rod-aligned tiles (greedy contiguous packing, <= block slots and <= block/8 rods per
  // tile); each tile's state is one contiguous SoA block: 6 node planes x nslots, ER_EPL element
  // planes x nel, [3 Voronoi planes x nvor], padded to an even number of doubles (16 B).  Built
  // on a host thread of its own while the records are built (they share no data).
  std::vector<ErTile> tiles;
  b->has_kappa0 = d->rest_kappa != nullptr && NV > 0;
  std::thread tile_thread([&]() {
    if (wtile_rods > 0) {
      // warp layout: equal rods in the identity order, every tile but the last full -- each tile's
      // descriptor is a function of its index, filled by host threads in parallel (cfg3: 524,288
      // warp-sized tiles)
      const int32_t N = max_n;
      const int64_t nt = (Rn + wtile_rods - 1) / wtile_rods;
      tiles.resize((size_t)nt);
      ErTile full;
      std::memset(&full, 0, sizeof full);
      full.nr = (int32_t)std::min<int64_t>(wtile_rods, Rn);
      full.nslots = full.nr * (N + 1);
      full.nel = full.nr * N;
      full.nseg = 1;
      for (int32_t q = 0, st = 0; q < full.nr; ++q, st += N + 1) full.smask[st >> 5] |= 1u << (st & 31);
      for (int wd = 1; wd < 16; ++wd) full.pfx[wd] = (uint8_t)(full.pfx[wd - 1] + __builtin_popcount(full.smask[wd - 1]));
      const int64_t bsz = tile_block_size(full, b->has_kappa0);
      auto fill = [&](int64_t t0, int64_t t1) {
        for (int64_t t = t0; t < t1; ++t) {
          ErTile T = full;
          const int64_t r0 = t * wtile_rods;
          T.r0 = (int32_t)r0;
          T.nbase = r0 * (N + 1);
          T.ebase = r0 * N;
          T.boff = t * bsz;
          if (t == nt - 1 && Rn - r0 < wtile_rods) {  // partial last tile
            T.nr = (int32_t)(Rn - r0);
            T.nslots = T.nr * (N + 1);
            T.nel = T.nr * N;
            std::memset(T.smask, 0, sizeof T.smask);
            std::memset(T.pfx, 0, sizeof T.pfx);
            for (int32_t q = 0, st = 0; q < T.nr; ++q, st += N + 1) T.smask[st >> 5] |= 1u << (st & 31);
            for (int wd = 1; wd < 16; ++wd) T.pfx[wd] = (uint8_t)(T.pfx[wd - 1] + __builtin_popcount(T.smask[wd - 1]));
          }
          tiles[(size_t)t] = T;
        }
      };
      const int nth = (int)std::max<unsigned>(1u, std::min<unsigned>(8u, std::thread::hardware_concurrency() / 2));
      std::vector<std::thread> th;
      for (int k = 0; k < nth; ++k) th.emplace_back(fill, nt * k / nth, nt * (k + 1) / nth);
      for (auto &x : th) x.join();
      b->n_tiles_norm = nt;
      b->state_doubles = nt ? tiles.back().boff + tile_block_size(tiles.back(), b->has_kappa0) : 0;
      return;
    }
    tiles.reserve((size_t)(Rn / std::max(1, b->block / std::max<int32_t>(max_n + 1, 1))) + (size_t)(R - Rn) * 16 + 64);
    int64_t r = 0, boff = 0;
    while (r < Rn) {
      ErTile T;
      T.r0 = (int32_t)r;
      T.nbase = eoffp[r] + r;
      T.ebase = eoffp[r];
      T.boff = boff;
      int64_t used = 0;
      int32_t nr = 0;
      const int32_t rmax = wtile_rods ? wtile_rods : b->block / 8;
      while (r < Rn && nr < rmax && used + b->n_elems_h[r] + 1 <= b->block) {
        used += b->n_elems_h[r] + 1;
        ++nr;
        ++r;
      }
      T.nr = nr;
      T.nslots = (int32_t)used;
      T.nel = (int32_t)(eoffp[r] - eoffp[T.r0]);
      std::memset(T.smask, 0, sizeof T.smask);
      std::memset(T.pfx, 0, sizeof T.pfx);
      T.seg = 0;
      T.nseg = 1;
      for (int32_t q = 0, st = 0; q < nr; ++q) {
        T.smask[st >> 5] |= 1u << (st & 31);
        st += b->n_elems_h[T.r0 + q] + 1;
      }
      for (int wd = 1; wd < 16; ++wd) T.pfx[wd] = (uint8_t)(T.pfx[wd - 1] + __builtin_popcount(T.smask[wd - 1]));
      boff += tile_block_size(T, b->has_kappa0);
      tiles.push_back(T);
    }
    b->n_tiles_norm = (int64_t)tiles.size();
    // long rods: ceil((N+1)/S) segment tiles of S slots each (the last one shorter)
    for (; r < R; ++r) {
      const int32_t N = b->n_elems_h[r], K = (N + ER_LONG_SEG) / ER_LONG_SEG;
      if (b->long_groups.empty() || b->long_groups.back().nseg != K)
        b->long_groups.push_back({(int64_t)tiles.size(), 0, K});
      b->long_groups.back().n_rods += 1;
      for (int32_t k = 0; k < K; ++k) {
        ErTile T;
        const int32_t k0 = k * ER_LONG_SEG;
        T.r0 = (int32_t)r;
        T.nr = 1;
        T.nslots = std::min(ER_LONG_SEG, N + 1 - k0);
        T.nel = std::max(0, std::min(ER_LONG_SEG, N - k0));
        T.nbase = eoffp[r] + r + k0;
        T.ebase = eoffp[r] + k0;
        T.boff = boff;
        std::memset(T.smask, 0, sizeof T.smask);
        std::memset(T.pfx, 0, sizeof T.pfx);
        T.smask[0] = 1u;  // one rod, starting at slot 0 (slot s is node k0 + s of the rod)
        for (int wd = 1; wd < 16; ++wd) T.pfx[wd] = 1;
        T.seg = k;
        T.nseg = K;
        boff += tile_block_size(T, b->has_kappa0);
        tiles.push_back(T);
      }
    }
    b->state_doubles = boff;
  });
  // ---- per-rod records; general rods get per-slot parameter planes
  b->rec_n = (size_t)std::max<int64_t>(R, 1) * ER_REC;
  b->rec.reset(new double[b->rec_n]);  // every record is fully written below (in parallel)
  if (R == 0) std::fill_n(b->rec.get(), b->rec_n, 0.0);
  b->flags.assign((size_t)std::max<int64_t>(R, 1), 0);
  auto mat_at = [&](int64_t r, int64_t j) {
    const int64_t k = d->material_per_rod ? r : j;
    ElemMat m{d->density[k], d->area[k], d->I1[k], d->I2[k], d->youngs[k], d->shear_mod[k], d->alpha_c[k], d->rest_lengths[j]};
    return m;
  };
  // per-rod records in parallel over host threads (independent rods)
  const int nthr = (int)std::max<unsigned>(1u, std::min<unsigned>(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::vector<char> gen_flag((size_t)std::max<int64_t>(R, 1), 0);
  for (auto *v : {&b->rod_A0, &b->rod_E0, &b->rod_lmin, &b->rod_lmax}) v->assign((size_t)std::max<int64_t>(R, 1), 0.0);
  auto rec_range = [&](int64_t ra, int64_t rb) {
  for (int64_t pr = ra; pr < rb; ++pr) {
    const int64_t r = b->ord[pr];  // canonical rod of packed rod pr
    const ElemMat m0 = mat_at(r, eoff[r]);
    bool uniform = true;
    if (d->material_per_rod) {  // only the rest lengths can vary along the rod
      const double *lh = d->rest_lengths;
      for (int64_t j = eoff[r] + 1; j < eoff[r + 1]; ++j) uniform &= lh[j] == m0.lh;
    } else {
      for (int64_t j = eoff[r] + 1; j < eoff[r + 1] && uniform; ++j) {
        const ElemMat m = mat_at(r, j);
        uniform = m.rho == m0.rho && m.A == m0.A && m.I1 == m0.I1 && m.I2 == m0.I2 && m.E == m0.E && m.G == m0.G &&
                  m.ac == m0.ac && m.lh == m0.lh;
      }
    }
    std::fill_n(&b->rec[(size_t)pr * ER_REC], ER_REC, 0.0);
    fill_record(&b->rec[(size_t)pr * ER_REC], m0);
    b->rec[(size_t)pr * ER_REC + REC_CANON] = (double)r;
    if (!uniform) gen_flag[pr] = 1;
    double lmin = d->rest_lengths[eoff[r]], lmax = lmin;
    for (int64_t j = eoff[r] + 1; j < eoff[r + 1]; ++j) {
      lmin = std::min(lmin, d->rest_lengths[j]);
      lmax = std::max(lmax, d->rest_lengths[j]);
    }
    b->rod_A0[pr] = m0.A;
    b->rod_E0[pr] = m0.E;
    b->rod_lmin[pr] = lmin;
    b->rod_lmax[pr] = lmax;
  }
  };
  if (R < 65536) rec_range(0, R);
  else {
    for (int q = 0; q < nthr; ++q) pool.emplace_back(rec_range, R * q / nthr, R * (q + 1) / nthr);
    for (auto &th : pool) th.join();
  }
  for (int64_t r = 0; r < R; ++r)
    if (gen_flag[r]) { b->flags[r] |= FL_GENERAL; b->any_general = true; }
  tm.mark("records");
  b->has_sigma0 = d->rest_sigma != nullptr;
  b->ng = pad_to(NN, 32);
  b->ne = pad_to(E, 32);
  std::vector<double> gpar;
  if (b->any_general) {
    gpar.assign((size_t)ER_GP * b->ng, 0.0);
    for (int64_t pr = 0; pr < R; ++pr) {
      if (!(b->flags[pr] & FL_GENERAL)) continue;
      const int64_t r = b->ord[pr];
      const int32_t N = b->n_elems_h[pr];
      const int64_t n0 = eoffp[pr] + pr;
      double sk = 0.0;
      for (int32_t i = 0; i <= N; ++i) {
        auto G = [&](int q) -> double & { return gpar[(size_t)q * b->ng + n0 + i]; };
        double mass = 0.0;
        if (i < N) {
          const ElemMat m = mat_at(r, eoff[r] + i);
          double tmp[ER_REC];
          fill_record(tmp, m);
          G(GP_LHAT) = tmp[REC_LHAT]; G(GP_ILHAT) = tmp[REC_ILHAT]; G(GP_S1) = tmp[REC_S1]; G(GP_S3) = tmp[REC_S3];
          for (int c = 0; c < 3; ++c) { G(GP_IJ1 + c) = tmp[REC_IJ1 + c]; G(GP_KJ1 + c) = tmp[REC_KJ1 + c]; }
          mass += 0.5 * m.rho * m.A * m.lh;
        }
        if (i > 0) {
          const ElemMat m = mat_at(r, eoff[r] + i - 1);
          mass += 0.5 * m.rho * m.A * m.lh;
        }
        G(GP_IM) = 1.0 / mass;
        G(GP_SK) = sk;
        if (i >= 1 && i < N) {
          const ElemMat ml = mat_at(r, eoff[r] + i - 1), mr = mat_at(r, eoff[r] + i);
          const double Dh = 0.5 * (ml.lh + mr.lh);
          const double Bl[3] = {ml.E * ml.I1, ml.E * ml.I2, ml.G * (ml.I1 + ml.I2)};
          const double Br[3] = {mr.E * mr.I1, mr.E * mr.I2, mr.G * (mr.I1 + mr.I2)};
          G(GP_DH) = Dh;
          // Voronoi stiffness = series (compliance) mean over the domain's two half elements, the
          // exact stiffness of a composite segment under a uniform moment (DESIGN §3 #9)
          for (int c = 0; c < 3; ++c) G(GP_BV1 + c) = (2.0 * Dh) / (ml.lh / Bl[c] + mr.lh / Br[c]);
        }
        if (i < N) sk += d->rest_lengths[eoff[r] + i];
      }
    }
  }

  tile_thread.join();
  if (b->wN > 0) {
    // warp-kernel stage buffer: the largest tile block | its rod records | the descriptor; as many
    // buffers (2..4) as keep two 256-thread CTAs per SM within the 228 KB of shared memory
    int64_t cs = 0, nr = 0;
    for (int64_t k = 0; k < b->n_tiles_norm; ++k) {
      cs = std::max(cs, tile_block_size(tiles[(size_t)k], b->has_kappa0));
      nr = std::max<int64_t>(nr, tiles[(size_t)k].nr);
    }
    b->wrec = (int32_t)cs;
    b->wdesc = (int32_t)(cs + nr * ER_REC);
    b->wbufd = b->wdesc + 16;
    const int64_t per_cta = 113 * 1024 - 64;
    b->wnb = (int32_t)std::max<int64_t>(2, std::min<int64_t>(4, per_cta / (8 * (int64_t)b->wbufd + 12)));
    if (const char *e = std::getenv("ER_WARP_BUFFERS")) b->wnb = std::max(1, std::min(8, std::atoi(e)));
    if ((std::getenv("ER_WARP_TMA") == nullptr || b->wN > 32) && b->n_tiles_norm > 0 && wtile_rods == b->wR) {
      // per-warp streaming (default): uniform tiles (every rod N elements, identity order), a ring
      // of 2..4 slots of one warp chunk (wR rods: node, element, kappa0 planes, records) per warp
      const int32_t Rw = b->wR, N = b->wN;
      b->wrt = wtile_rods;
      b->wcs = tile_block_size(tiles[0], b->has_kappa0);
      b->wrods = Rn;
      b->wch = (int32_t)(b->wcs + Rw * ER_REC);  // block | records (both even: 16-byte copies)
      const int64_t units = N > 32 ? 4 : ER_WB_WARPS;  // pipelines per CTA (warps, or warp pairs)
      const int64_t budget = N > 32 ? 113 * 1024 - 512 : 227 * 1024 / ER_WB_MINB - 1024;  // smem per CTA
      b->wnb = (int32_t)std::max<int64_t>(2, std::min<int64_t>(4, budget / (units * 8 * (int64_t)b->wch)));
      if (const char *e = std::getenv("ER_WARP_BUFFERS")) b->wnb = std::max(2, std::min(4, std::atoi(e)));
    }
  }
  b->n_tiles = (int64_t)tiles.size();
  tm.mark("gpar + tiles");

  // ---- device allocation and upload
  CK(dalloc(b, &b->d_state, b->state_doubles + 64), "cudaMalloc(state)");
  CK(dalloc(b, &b->d_rec, (int64_t)b->rec_n), "cudaMalloc(rec)");
  CK(dalloc(b, &b->d_eoff, R + 4), "cudaMalloc(eoff)");
  CK(dalloc(b, &b->d_tiles, std::max<int64_t>((int64_t)tiles.size(), 1)), "cudaMalloc(tiles)");
  CK(dalloc(b, &b->d_fault, 2), "cudaMalloc(fault)");
  CK(dalloc(b, &b->d_diag_partial, std::max<int64_t>(b->n_tiles, 1) * 16), "cudaMalloc(diag)");
  CK(dalloc(b, &b->d_diag_out, 16), "cudaMalloc(diag_out)");
  CK(dalloc(b, &b->d_valid, 4), "cudaMalloc(valid)");
  CK(cudaMemsetAsync(b->d_state, 0, sizeof(double) * (b->state_doubles + 64), b->stream), "memset");
  CK(dalloc(b, &b->d_ord, R + 1), "cudaMalloc(ord)");
  CK(dalloc(b, &b->d_eoffc, R + 1), "cudaMalloc(eoffc)");
  {
    std::vector<int64_t> ep(eoffp);
    ep.resize((size_t)R + 4, eoffp[R]);
    CK(cudaMemcpyAsync(b->d_eoff, ep.data(), sizeof(int64_t) * ep.size(), cudaMemcpyHostToDevice, b->stream), "H2D eoff");
    if (R > 0) CK(cudaMemcpyAsync(b->d_ord, b->ord.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, b->stream), "H2D ord");
    CK(cudaMemcpyAsync(b->d_eoffc, eoff.data(), sizeof(int64_t) * (R + 1), cudaMemcpyHostToDevice, b->stream), "H2D eoffc");
    if (!tiles.empty())
      CK(cudaMemcpyAsync(b->d_tiles, tiles.data(), sizeof(ErTile) * tiles.size(), cudaMemcpyHostToDevice, b->stream), "H2D tiles");
    if (b->any_general) {
      CK(dalloc(b, &b->d_gpar, (int64_t)gpar.size()), "cudaMalloc(gpar)");
      CK(cudaMemcpyAsync(b->d_gpar, gpar.data(), sizeof(double) * gpar.size(), cudaMemcpyHostToDevice, b->stream), "H2D gpar");
    }
    er_status st0 = upload_records(b);
    if (st0 != ER_OK) return fail(st0);
    CK(cudaStreamSynchronize(b->stream), "sync");  // host vectors above are freed at scope exit
  }
  tm.mark("alloc + small uploads", b->stream);
  er_status st;
  CK(cudaMemsetAsync(b->d_valid, 0, sizeof(double) * 4, b->stream), "memset");
  if ((st = upload_field(b, d->positions, d->src_mem, FIELD_POS, true)) != ER_OK) return fail(st);
  if ((st = upload_field(b, d->velocities, d->src_mem, FIELD_VEL, true)) != ER_OK) return fail(st);
  if ((st = upload_field(b, d->directors, d->src_mem, FIELD_DIR, true)) != ER_OK) return fail(st);
  if ((st = upload_field(b, d->omega, d->src_mem, FIELD_OMEGA, true)) != ER_OK) return fail(st);
  if (b->has_kappa0 && (st = upload_field(b, d->rest_kappa, ER_HOST, FIELD_KAPPA0, false)) != ER_OK) return fail(st);
  CK(cudaStreamSynchronize(b->stream), "sync");
  cudaFree(b->upload_stage);
  b->upload_stage = nullptr;
  for (auto &sp : b->staged) sp = nullptr;
  if (d->rest_sigma) {
    CK(dalloc(b, &b->d_sigma0, 3 * b->ne), "cudaMalloc(sigma0)");
    const std::vector<double> ps = b->identity ? std::vector<double>() : pack_rows(b, d->rest_sigma, 3, true);
    if ((st = upload_side_planes(b, b->identity ? d->rest_sigma : ps.data(), b->d_sigma0, E, b->ne)) != ER_OK) return fail(st);
  }
  tm.mark("state upload + layout", b->stream);
  // ---- validation of the uploaded state (directors orthonormal within 1e-10, all finite)
  double vres[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(vres, b->d_valid, sizeof vres, cudaMemcpyDeviceToHost, b->stream), "D2H valid");
  CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
  if (vres[2] > 0) err.add("%g state entries (positions/velocities/directors/omega) are not finite", vres[2]);
  if (vres[0] > 1e-10) err.add("directors not orthonormal: max |Q Q^T - I| = %.3g > 1e-10", vres[0]);
  if (vres[1] > 1e-10) err.add("directors not proper rotations: max |det Q - 1| = %.3g", vres[1]);
  if (err.count) { b->last_error = err.msg; return fail(ER_EINVAL); }
#undef CK
  b->rec.reset();  // the device records are authoritative from here on
  b->rec_n = 0;
  *out = b;
  return ER_OK;
}

#define CK(call, what)                                    \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(b, e_, what); \
  } while (0)

er_status er_set_bc(er_batch *b, const int8_t *clamp_end) {
  NvtxRange nvtx_("er_set_bc");
  if (!b) return ER_EINVAL;
  Errors err;
  if (clamp_end)
    for (int64_t r = 0; r < b->n_rods; ++r)
      if (clamp_end[r] < -1 || clamp_end[r] > 1) err.add("clamp_end[%lld] = %d not in {-1, 0, 1}", (long long)r, clamp_end[r]);
  if (err.count) { b->last_error = err.msg; return ER_EINVAL; }
  for (int64_t pr = 0; pr < b->n_rods; ++pr) {
    const int64_t r = b->ord[pr];
    b->flags[pr] &= ~FL_CLAMP_MASK;
    if (clamp_end && clamp_end[r] == 0) b->flags[pr] |= 1;
    if (clamp_end && clamp_end[r] == 1) b->flags[pr] |= 2;
  }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  return apply_forcing(b, nullptr, false);
}

er_status er_set_forcing(er_batch *b, const er_forcing *f) {
  NvtxRange nvtx_("er_set_forcing");
  if (!b || !f) { if (b) b->last_error = "forcing is NULL"; return ER_EINVAL; }
  b->forcing_version += 1;  // step-graph parameters (gravity, field, features) may change
  Errors err;
  const int64_t R = b->n_rods;
  for (int c = 0; c < 3; ++c) {
    if (!std::isfinite(f->gravity[c])) err.add("gravity[%d] not finite", c);
    if (!std::isfinite(f->b_field[c])) err.add("b_field[%d] not finite", c);
    if (!std::isfinite(f->b_axis[c])) err.add("b_axis[%d] not finite", c);
  }
  if (!std::isfinite(f->b_omega)) err.add("b_omega not finite");
  if (f->damping) {
    for (int64_t r = 0; r < R; ++r)
      if (!(std::isfinite(f->damping[r]) && f->damping[r] >= 0)) { err.add("damping[%lld] = %g must be finite and >= 0", (long long)r, f->damping[r]); break; }
  } else if (!(std::isfinite(f->damping_all) && f->damping_all >= 0)) err.add("damping_all = %g must be finite and >= 0", f->damping_all);
  if (f->tip_force)
    for (int64_t k = 0; k < 3 * R; ++k)
      if (!std::isfinite(f->tip_force[k])) { err.add("tip_force[%lld] not finite", (long long)k); break; }
  const bool act = f->act_A || f->act_f || f->act_L;
  if (act) {
    if (!(f->act_A && f->act_f && f->act_L)) err.add("act_A, act_f and act_L must be all set or all NULL");
    else
      for (int64_t r = 0; r < R; ++r) {
        if (!std::isfinite(f->act_A[r]) || !std::isfinite(f->act_f[r])) { err.add("act_A/act_f[%lld] not finite", (long long)r); break; }
        if (!pos_finite(f->act_L[r])) { err.add("act_L[%lld] = %g must be positive", (long long)r, f->act_L[r]); break; }
      }
    if (f->act_component < 0 || f->act_component > 2) err.add("act_component = %d not in {0,1,2}", f->act_component);
  }
  const bool musc = f->musc_A || f->musc_T || f->musc_lambda || f->musc_phi;
  if (musc) {
    if (!(f->musc_A && f->musc_T && f->musc_lambda && f->musc_phi)) err.add("musc_A, musc_T, musc_lambda and musc_phi must be all set or all NULL");
    else
      for (int64_t r = 0; r < R; ++r) {
        if (!std::isfinite(f->musc_A[r]) || !std::isfinite(f->musc_phi[r])) { err.add("musc_A/musc_phi[%lld] not finite", (long long)r); break; }
        if (!pos_finite(f->musc_T[r]) || !pos_finite(f->musc_lambda[r])) { err.add("musc_T/musc_lambda[%lld] must be positive", (long long)r); break; }
      }
    if (f->musc_component < 0 || f->musc_component > 2) err.add("musc_component = %d not in {0,1,2}", f->musc_component);
  }
  if (f->magnetization)
    for (int64_t k = 0; k < 3 * b->n_elems; ++k)
      if (!std::isfinite(f->magnetization[k])) { err.add("magnetization[%lld] not finite", (long long)k); break; }
  if (err.count) { b->last_error = err.msg; return ER_EINVAL; }

  {
    // b(t) = R_axis(w t) b_field = bp cos + (a x b_field) sin + a (a . b_field), bp = b_field - a (a . b_field)
    double ax[3] = {f->b_axis[0], f->b_axis[1], f->b_axis[2]};
    double na = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    if (na == 0.0) { ax[0] = 0.0; ax[1] = 0.0; ax[2] = 1.0; na = 1.0; }
    for (int c = 0; c < 3; ++c) ax[c] /= na;
    const double *bf = f->b_field;
    const double ad = ax[0] * bf[0] + ax[1] * bf[1] + ax[2] * bf[2];
    const double axb[3] = {ax[1] * bf[2] - ax[2] * bf[1], ax[2] * bf[0] - ax[0] * bf[2], ax[0] * bf[1] - ax[1] * bf[0]};
    for (int c = 0; c < 3; ++c) {
      b->g[c] = f->gravity[c];
      b->b2[c] = ax[c] * ad;
      b->b0[c] = bf[c] - b->b2[c];
      b->b1[c] = axb[c];
    }
  }
  b->b_omega = f->b_omega;
  b->act_comp = act ? f->act_component : 0;
  b->has_act = act;
  for (int64_t r = 0; r < R; ++r) {
    b->flags[r] &= ~(FL_TIP | FL_ACT | FL_MUS);
    if (f->tip_force) b->flags[r] |= FL_TIP;
    if (act) b->flags[r] |= FL_ACT;
    if (musc) b->flags[r] |= FL_MUS;
  }
  b->has_musc = musc;
  b->musc_comp = musc ? f->musc_component : 0;
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  er_status st = apply_forcing(b, f, true);
  if (st != ER_OK) return st;
  if (musc && R > 0) {
    std::vector<double> mh((size_t)R * 4);
    for (int64_t pr = 0; pr < R; ++pr) {
      const int64_t r = b->ord[pr];
      mh[4 * pr + 0] = f->musc_A[r];
      mh[4 * pr + 1] = 1.0 / f->musc_T[r];
      mh[4 * pr + 2] = 1.0 / f->musc_lambda[r];
      mh[4 * pr + 3] = f->musc_phi[r] / 3.14159265358979323846;
    }
    if (!b->d_musc) CK(dalloc(b, &b->d_musc, 4 * R), "cudaMalloc(musc)");
    CK(cudaMemcpyAsync(b->d_musc, mh.data(), sizeof(double) * mh.size(), cudaMemcpyHostToDevice, b->stream), "H2D musc");
    CK(cudaStreamSynchronize(b->stream), "sync");
  }
  if (f->magnetization && b->n_elems > 0) {
    if (!b->d_mag) CK(dalloc(b, &b->d_mag, 3 * b->ne), "cudaMalloc(mag)");
    const std::vector<double> pm = b->identity ? std::vector<double>() : pack_rows(b, f->magnetization, 3, true);
    if ((st = upload_side_planes(b, b->identity ? f->magnetization : pm.data(), b->d_mag, b->n_elems, b->ne)) != ER_OK)
      return st;
  } else if (b->d_mag) {
    CK(cudaStreamSynchronize(b->stream), "sync");
    cudaFree(b->d_mag);
    b->device_bytes -= (int64_t)sizeof(double) * 3 * b->ne;
    b->d_mag = nullptr;
  }
  CK(cudaStreamSynchronize(b->stream), "sync");
  return ER_OK;
}

// One external-load array: canonical AoS [rows][3] (host or device) -> planes in packed rod order.
// NULL frees the planes.  Returns whether the plane pointer changed (step graphs capture it).
static er_status set_ext_planes(er_batch *b, int32_t src_mem, const double *src, double **planes, int64_t stride,
                         int64_t rows, int nodes, bool *changed) {
  if (!src) {
    if (*planes) {
      CK(cudaStreamSynchronize(b->stream), "sync");
      cudaFree(*planes);
      b->device_bytes -= (int64_t)sizeof(double) * 3 * stride;
      *planes = nullptr;
      *changed = true;
    }
    return ER_OK;
  }
  if (!*planes) {
    CK(dalloc(b, planes, 3 * stride), "cudaMalloc(ext)");
    CK(cudaMemsetAsync(*planes, 0, sizeof(double) * 3 * (size_t)stride, b->stream), "memset(ext)");
    *changed = true;
  }
  if (rows <= 0) return ER_OK;
  const double *dsrc = src;
  double *stage = nullptr;
  if (src_mem == ER_HOST) {
    CK(cudaMallocAsync((void **)&stage, sizeof(double) * 3 * (size_t)rows, b->stream), "cudaMallocAsync(stage)");
    CK(cudaMemcpyAsync(stage, src, sizeof(double) * 3 * (size_t)rows, cudaMemcpyHostToDevice, b->stream), "H2D ext");
    dsrc = stage;
  }
  CK(er_launch_pack_planes(dsrc, *planes, stride, b->d_eoff, b->d_ord, b->d_eoffc, b->n_rods, nodes, b->stream),
     "pack_planes");
  if (stage) CK(cudaFreeAsync(stage, b->stream), "cudaFreeAsync");
  return ER_OK;
}

er_status er_set_external_loads(er_batch *b, int32_t src_mem, const double *node_force, const double *elem_couple) {
  if (!b) return ER_EINVAL;
  if (src_mem != ER_HOST && src_mem != ER_DEVICE) { b->last_error = "src_mem must be ER_HOST or ER_DEVICE"; return ER_EINVAL; }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  bool changed = false;
  er_status st = set_ext_planes(b, src_mem, node_force, &b->d_fext, b->ng, b->n_nodes, 1, &changed);
  if (st != ER_OK) return st;
  if ((st = set_ext_planes(b, src_mem, elem_couple, &b->d_cext, b->ne, b->n_elems, 0, &changed)) != ER_OK) return st;
  if (changed) b->forcing_version += 1;  // new plane pointers / kernel features: recapture step graphs
  if (src_mem == ER_HOST) CK(cudaStreamSynchronize(b->stream), "sync");  // caller may reuse its buffers
  return ER_OK;
}

er_status er_set_option(er_batch *b, int32_t option, int64_t value) {
  if (!b) return ER_EINVAL;
  if (option == ER_OPT_STEPS_PER_LAUNCH) {
    if (value < 1 || value > (1 << 30)) { b->last_error = "steps_per_launch must be in [1, 2^30]"; return ER_EINVAL; }
    b->steps_per_launch = value;
    return ER_OK;
  }
  if (option == ER_OPT_SWEEPS_PER_LAUNCH) {
    if (value < 0 || value > (1 << 20)) { b->last_error = "sweeps_per_launch must be in [0 (auto), 2^20]"; return ER_EINVAL; }
    b->sweeps = value;
    return ER_OK;
  }
  if (option == ER_OPT_PHASE_TIMING) {
    if (value != 0 && value != 1) { b->last_error = "phase timing must be 0 or 1"; return ER_EINVAL; }
    b->timing = value == 1;
    b->phase_ms[0] = b->phase_ms[1] = 0.0;
    b->phase_n[0] = b->phase_n[1] = 0;
    return ER_OK;
  }
  if (option == ER_OPT_KERNEL) {
    if (value < 0 || value > 4) { b->last_error = "kernel must be 0 (fused persistent), 1 (staged), 2 (fused, one tile per CTA), 3 (memory probe) or 4 (persistent, direct stores)"; return ER_EINVAL; }
    b->kernel_mode = (int)value;
    return ER_OK;
  }
  b->last_error = "unknown option";
  return ER_EINVAL;
}

er_status er_set_trace(er_batch *b, void *trace) {
  if (!b) return ER_EINVAL;
  if (trace && !ER_TRACE) { b->last_error = "the timeline needs a build with -DER_TRACE=1 (ER_NVCC_EXTRA)"; return ER_EINVAL; }
  b->trace = reinterpret_cast<unsigned long long *>(trace);
  b->forcing_version += 1;
  return ER_OK;
}

er_status er_step(er_batch *b, int64_t n_steps, double dt) {
  NvtxRange nvtx_("er_step");
  if (!b) return ER_EINVAL;
  Errors err;
  if (n_steps < 0) err.add("n_steps = %lld < 0", (long long)n_steps);
  if (!(std::isfinite(dt) && dt > 0.0)) err.add("dt = %g must be positive and finite", dt);
  if (b->g_rods > 0 && b->split_mode == 0)
    err.add("ghost rods are declared (er_set_contact_ghosts): step with er_step_begin / er_step_finish");
  if (err.count) { b->last_error = err.msg; return ER_EINVAL; }
  b->fault_rod = -1;
  b->fault_bits = 0;
  b->iv.clear();
  b->ev_used = 0;
  if (n_steps == 0 || b->n_rods == 0) return ER_OK;
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  const unsigned long long init[2] = {0ull, ~0ull};
  CK(cudaMemcpyAsync(b->d_fault, init, sizeof init, cudaMemcpyHostToDevice, b->stream), "H2D fault");
  ErStepParams p = params_of(b);
  p.h = dt;
  p.n_tiles = b->n_tiles_norm;  // long rods: er_launch_long below
  int64_t done = 0;
  double t = b->t;
  const int feat = feat_of(b);
  // long rods advance k steps from time t (all step kinds give the same trajectory)
  auto launch_long = [&](int64_t k, double t0, int lfeat = -1) -> cudaError_t {
    ErStepParams q = p;
    q.n_tiles = b->n_tiles;
    q.n_steps = (int32_t)k;
    q.t = t0;
    for (const auto &g : b->long_groups) {
      cudaError_t e = er_launch_long(&q, g.tile0, g.n_rods, g.nseg, lfeat < 0 ? feat : lfeat, b->stream);
      if (e != cudaSuccess) return e;
      b->launches += 1;
    }
    return cudaSuccess;
  };
  if (b->kernel_mode == 3) {  // memory-pipeline probe: n_steps passes of load + store, no physics
    p.n_steps = 0;
    p.t = t;
    for (int64_t q = 0; q < n_steps; ++q) {
      CK(er_launch_step(&p, b->block, 0, feat, b->stream), "probe kernel");
      b->launches += 1;
    }
    CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
    return ER_OK;
  }
  // contact: every step needs all rods' half-step positions, so ER_OPT_STEPS_PER_LAUNCH does not
  // apply; ER_OPT_KERNEL 1 selects the staged path, any other value the fused contact step
  if (b->contact_on && b->kernel_mode != 1) {
    // NEXT-4, fused: drift-1 of the first step (+ node records); then per step the contact
    // evaluation and one persistent launch doing kick + drift-2 + the next step's drift-1
    p.n_steps = 1;
    p.t = t;
    p.cnode = b->cp.cnode;
    p.cbuild = b->cp.cbuild;
    p.disp2 = 0.25 * b->cp.skin * b->cp.skin;
    p.rebuild = b->cp.rebuild;
    int m0 = mark(b);
    if (b->split_mode != 2) {  // (er_step_finish: the drift-1 ran in er_step_begin)
      p.n_tiles = b->n_tiles;  // the drift kernel handles long-rod segment tiles too (no exchange)
      CK(er_launch_step(&p, b->block, 1, 15, b->stream), "drift kernel");
      p.n_tiles = b->n_tiles_norm;
      b->launches += 1;
    }
    int m1 = mark(b);
    interval(b, m0, m1, 0);
    p.cfc = b->cp.fc;
    p.cfs = b->cp.fs;
    for (int64_t q = 0; q < n_steps && b->split_mode != 1; ++q) {
      if (b->g_rods > 0) {  // ghost records (just supplied): their Verlet bound
        CK(er_contact_ghost_check(&b->cp, b->n_nodes, p.disp2, b->stream), "ghost check");
        b->launches += 1;
      }
      CK(er_contact_eval(&b->cp, b->sort_tmp, b->sort_bytes, b->cgraph, b->stream, &b->launches, b->cgraph_kernels), "contact");
      const int m2 = mark(b);
      interval(b, m1, m2, 1);
      p.t = t;
      p.cnode = q + 1 < n_steps && b->split_mode == 0 ? b->cp.cnode : nullptr;
      CK(er_launch_step(&p, b->block, 0, feat | FEAT_CONTACT, b->stream), "step kernel");
      b->launches += 1;
      CK(launch_long(1, t, feat | FEAT_CONTACT), "long-rod kernel");
      m1 = mark(b);
      interval(b, m2, m1, 0);
      const double th = t + 0.5 * dt;
      t = th + 0.5 * dt;
    }
    done = n_steps;
  }
  const int64_t spl = b->steps_per_launch;
  // Sweeps: one persistent launch streams every tile through HBM S times (S steps of spl on-chip
  // steps each); long-rod clusters advance the same steps in their own launch.
  // Default (0): sweeps only for small batches -- a few tiles per CTA, where launch boundaries
  // dominate (cfg1/cfg2); large batches keep one launch per step (graph replays), which measured
  // faster there.
  const int64_t grid = 148 * (b->block <= 128 ? 4 : b->block <= 256 ? 2 : 1);
  // (the warp kernel's batches keep one launch per step: its tiles are warp-sized)
  const int64_t sweeps = b->sweeps > 0 ? b->sweeps : (b->wN == 0 && b->n_tiles_norm <= 4 * grid ? 128 : 1);
  if (!b->contact_on && b->kernel_mode == 0 && sweeps > 1) {
    while (n_steps - done >= spl) {
      const int64_t S = std::min<int64_t>(sweeps, (n_steps - done) / spl);
      p.n_steps = (int32_t)spl;
      p.sweeps = (int32_t)S;
      p.t = t;
      const int m0 = mark(b);
      CK(er_launch_step(&p, b->block, 0, feat, b->stream), "step kernel");
      b->launches += 1;
      interval(b, m0, mark(b), 0, (int)S);
      CK(launch_long(spl * S, t), "long-rod kernel");
      for (int64_t q = 0; q < spl * S; ++q) { const double th = t + 0.5 * dt; t = th + 0.5 * dt; }
      done += spl * S;
    }
    p.sweeps = 1;
  }
  // Streaming steps as CUDA-graph launches of ER_GRAPH_LAUNCHES step launches each (the time is
  // carried on the device between launches); the rest as plain launches below.
  if (!b->contact_on && b->kernel_mode == 0 && n_steps - done >= ER_GRAPH_LAUNCHES * spl &&
      !std::getenv("ER_NO_STEP_GRAPH")) {
    const int64_t key = ((b->forcing_version * 32 + feat) << 31) + spl;
    uint64_t h_bits;
    std::memcpy(&h_bits, &dt, sizeof h_bits);
    if (!b->tdev) CK(dalloc(b, &b->tdev, 2), "cudaMalloc(tdev)");
    // the graph holds ErStepParams by value, including h = dt: a call with another dt recaptures
    if (b->sgraph_key != key || b->sgraph_h_bits != h_bits) {
      free_step_graph(b);
      if (!b->d_loop) CK(dalloc(b, &b->d_loop, 1), "cudaMalloc(loop)");
      cudaStream_t cs;
      CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate");
      auto capture_launches = [&](cudaStream_t s_) -> cudaError_t {
        cudaError_t e_ = cudaSuccess;
        for (int j = 0; e_ == cudaSuccess && j < ER_GRAPH_LAUNCHES; ++j) {
          ErStepParams q = p;
          q.n_steps = (int32_t)spl;
          q.tdev = b->tdev;
          q.tpar = j & 1;
          e_ = er_launch_step(&q, b->block, 0, feat, s_);
          q.n_tiles = b->n_tiles;
          for (const auto &gr : b->long_groups)
            if (e_ == cudaSuccess) e_ = er_launch_long(&q, gr.tile0, gr.n_rods, gr.nseg, feat, s_);
        }
        return e_;
      };
      // Preferred: a WHILE node whose body is the 32 launches plus a loop-control kernel, so one
      // cudaGraphLaunch runs every full chunk of an er_step call with no host submissions in
      // between (host-side stalls -- a monitoring query holding the driver -- cannot starve the
      // GPU).  Fallback: the 32 launches as a plain graph, launched once per chunk.
      cudaGraph_t g = nullptr;
      cudaError_t e = std::getenv("ER_NO_WHILE_GRAPH") ? cudaErrorNotSupported : cudaGraphCreate(&g, 0);
      cudaGraphConditionalHandle h;
      if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams np = {};
      cudaGraphNode_t wnode;
      if (e == cudaSuccess) {
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        e = cudaGraphAddNode(&wnode, g, nullptr, 0, &np);
      }
      if (e == cudaSuccess) {
        cudaGraph_t body = np.conditional.phGraph_out[0];
        e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
          cudaError_t eb = capture_launches(cs);
          if (eb == cudaSuccess) {
            er_step_loop_ctl<<<1, 1, 0, cs>>>(b->d_loop, h);
            eb = cudaGetLastError();
          }
          e = cudaStreamEndCapture(cs, &body);
          if (eb != cudaSuccess) e = eb;
        }
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&b->sgraph, g, 0);
      if (g) cudaGraphDestroy(g);
      b->sgraph_while = e == cudaSuccess;
      if (e != cudaSuccess) {
        cudaGetLastError();  // clear a sticky-free failure of the WHILE path
        b->sgraph = nullptr;
        g = nullptr;
        e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);  // launchers query attributes
        if (e == cudaSuccess) {
          cudaError_t eb = capture_launches(cs);
          e = cudaStreamEndCapture(cs, &g);
          if (eb != cudaSuccess) e = eb;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&b->sgraph, g, 0);
        if (g) cudaGraphDestroy(g);
      }
      cudaStreamDestroy(cs);
      CK(e, "step graph");
      b->sgraph_key = key;
      b->sgraph_h_bits = h_bits;
    }
    const double t_host = t;  // pageable 8-byte copy: staged before cudaMemcpyAsync returns
    CK(cudaMemcpyAsync(b->tdev, &t_host, sizeof(double), cudaMemcpyHostToDevice, b->stream), "H2D t");
    const int64_t chunk = ER_GRAPH_LAUNCHES * spl;
    if (b->sgraph_while) {  // every full chunk in one launch: the device counts the iterations
      const long long iters = (long long)((n_steps - done) / chunk);
      CK(cudaMemcpyAsync(b->d_loop, &iters, sizeof iters, cudaMemcpyHostToDevice, b->stream), "H2D loop");
      const int m0 = mark(b);
      CK(cudaGraphLaunch(b->sgraph, b->stream), "step graph launch");
      interval(b, m0, mark(b), 0, (int)(ER_GRAPH_LAUNCHES * iters));
      b->launches += ER_GRAPH_LAUNCHES * iters * (1 + (int64_t)b->long_groups.size());
      for (int64_t q = 0; q < chunk * iters; ++q) { const double th = t + 0.5 * dt; t = th + 0.5 * dt; }
      done += chunk * iters;
    }
    while (n_steps - done >= chunk) {
      const int m0 = mark(b);
      CK(cudaGraphLaunch(b->sgraph, b->stream), "step graph launch");
      interval(b, m0, mark(b), 0, ER_GRAPH_LAUNCHES);
      b->launches += ER_GRAPH_LAUNCHES * (1 + (int64_t)b->long_groups.size());
      for (int64_t q = 0; q < chunk; ++q) { const double th = t + 0.5 * dt; t = th + 0.5 * dt; }
      done += chunk;
    }
  }
  while (done < n_steps) {
    if (b->contact_on) {  // NEXT-4 staged: drift | contact (broad + narrow phase) | dynamics + kick | drift
      p.n_steps = 1;
      p.t = t;
      p.cnode = b->cp.cnode;
      p.cbuild = b->cp.cbuild;
      p.disp2 = 0.25 * b->cp.skin * b->cp.skin;
      p.rebuild = b->cp.rebuild;
      p.n_tiles = b->n_tiles;  // drift-1 + node records for long-rod segments too
      CK(er_launch_step(&p, b->block, 1, 15, b->stream), "drift kernel");
      p.n_tiles = b->n_tiles_norm;
      p.cnode = nullptr;
      CK(er_contact_eval(&b->cp, b->sort_tmp, b->sort_bytes, b->cgraph, b->stream, &b->launches, b->cgraph_kernels), "contact");
      p.cfc = b->cp.fc;
      p.cfs = b->cp.fs;
      CK(er_launch_step(&p, b->block, 2, 7, b->stream), "dyn kernel");
      CK(launch_long(1, t, feat | FEAT_CONTACT), "long-rod kernel");  // kick + drift-2 (cnode unset)
      p.cfc = nullptr;
      CK(er_launch_step(&p, b->block, 1, 7, b->stream), "drift kernel");
      b->launches += 3;
      const double th = t + 0.5 * dt;
      t = th + 0.5 * dt;
      done += 1;
    } else if (b->kernel_mode == 0 || b->kernel_mode == 2 || b->kernel_mode == 4) {
      const int64_t k = std::min<int64_t>(b->steps_per_launch, n_steps - done);
      p.n_steps = (int32_t)k;
      p.t = t;
      const int m0 = mark(b);
      CK(er_launch_step(&p, b->block, b->kernel_mode == 0 ? 0 : b->kernel_mode == 4 ? 5 : 3, feat, b->stream),
         "step kernel");
      b->launches += 1;
      interval(b, m0, mark(b), 0);
      CK(launch_long(k, t), "long-rod kernel");
      for (int64_t q = 0; q < k; ++q) { const double th = t + 0.5 * dt; t = th + 0.5 * dt; }
      done += k;
    } else {  // staged ablation: drift | dynamics + kick | drift, state through HBM between stages
      p.n_steps = 1;
      p.t = t;
      CK(er_launch_step(&p, b->block, 1, 7, b->stream), "drift kernel");
      CK(er_launch_step(&p, b->block, 2, 7, b->stream), "dyn kernel");
      CK(er_launch_step(&p, b->block, 1, 7, b->stream), "drift kernel");
      b->launches += 3;
      CK(launch_long(1, t), "long-rod kernel");
      const double th = t + 0.5 * dt;
      t = th + 0.5 * dt;
      done += 1;
    }
  }
  b->t = t;
  unsigned long long fw[2];
  CK(cudaMemcpyAsync(fw, b->d_fault, sizeof fw, cudaMemcpyDeviceToHost, b->stream), "D2H fault");
  CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
  collect_times(b);
  if (fw[0]) {
    b->fault_bits = (int32_t)fw[0];
    b->fault_rod = (int64_t)fw[1];
    char buf[256];
    snprintf(buf, sizeof buf, "unstable: rod %lld faulted (bits 0x%x:%s%s%s%s) during er_step(%lld, %g)",
             (long long)b->fault_rod, b->fault_bits, (fw[0] & ER_F_NONFINITE) ? " nonfinite" : "",
             (fw[0] & ER_F_DEGENERATE) ? " degenerate" : "", (fw[0] & ER_F_ANTIPODAL) ? " antipodal" : "",
             (fw[0] & ER_F_OVERSPEED) ? " overspeed" : "", (long long)n_steps, dt);
    b->last_error = buf;
    return ER_EUNSTABLE;
  }
  return ER_OK;
}

// A warp-layout batch (warp-sized tiles of the warp kernel, er_warp.cu) -> the tile kernels' layout
// (rod-aligned tiles of <= 256 slots): contact mode runs the tile kernels.  Equal-length rods in the
// identity order, so only the tiles and the state blocks change; the state moves through canonical
// device arrays (d1, d2 exactly; d3 is rebuilt as everywhere).
er_status relayout_to_tiles(er_batch *b) {
  if (b->wN <= 0) return ER_OK;
  CK(cudaStreamSynchronize(b->stream), "sync");
  const int fields[5] = {FIELD_POS, FIELD_VEL, FIELD_DIR, FIELD_OMEGA, FIELD_KAPPA0};
  const int nf = b->has_kappa0 ? 5 : 4;
  double *tmp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int f = 0; f < nf; ++f) {
    const int64_t n = field_rows(b, fields[f]) * field_k(fields[f]);
    CK(cudaMalloc((void **)&tmp[f], sizeof(double) * (size_t)std::max<int64_t>(n, 1)), "cudaMalloc(relayout)");
    er_status st = download_field(b, tmp[f], ER_DEVICE, fields[f]);
    if (st != ER_OK) return st;
  }
  const int32_t N = b->wN;
  const int64_t R = b->n_rods;
  b->block = 256;
  const int32_t rmax = std::min<int32_t>(b->block / 8, b->block / (N + 1));
  std::vector<ErTile> tiles;
  tiles.reserve((size_t)(R / rmax + 1));
  int64_t boff = 0;
  for (int64_t r = 0; r < R;) {
    ErTile T;
    const int32_t nr = (int32_t)std::min<int64_t>(rmax, R - r);
    T.r0 = (int32_t)r;
    T.nr = nr;
    T.nslots = nr * (N + 1);
    T.nel = nr * N;
    T.nbase = r * (N + 1);
    T.ebase = r * N;
    T.boff = boff;
    std::memset(T.smask, 0, sizeof T.smask);
    std::memset(T.pfx, 0, sizeof T.pfx);
    T.seg = 0;
    T.nseg = 1;
    for (int32_t q = 0, st = 0; q < nr; ++q, st += N + 1) T.smask[st >> 5] |= 1u << (st & 31);
    for (int wd = 1; wd < 16; ++wd) T.pfx[wd] = (uint8_t)(T.pfx[wd - 1] + __builtin_popcount(T.smask[wd - 1]));
    boff += tile_block_size(T, b->has_kappa0);
    tiles.push_back(T);
    r += nr;
  }
  free_step_graph(b);
  cudaFree(b->d_state);
  cudaFree(b->d_tiles);
  cudaFree(b->d_diag_partial);
  b->device_bytes -= (int64_t)sizeof(double) * (b->state_doubles + 64) + (int64_t)sizeof(ErTile) * std::max<int64_t>(b->n_tiles, 1) +
                     (int64_t)sizeof(double) * std::max<int64_t>(b->n_tiles, 1) * 16;
  b->state_doubles = boff;
  b->n_tiles = b->n_tiles_norm = (int64_t)tiles.size();
  CK(dalloc(b, &b->d_state, b->state_doubles + 64), "cudaMalloc(state)");
  CK(dalloc(b, &b->d_tiles, std::max<int64_t>(b->n_tiles, 1)), "cudaMalloc(tiles)");
  CK(dalloc(b, &b->d_diag_partial, std::max<int64_t>(b->n_tiles, 1) * 16), "cudaMalloc(diag)");
  CK(cudaMemsetAsync(b->d_state, 0, sizeof(double) * (b->state_doubles + 64), b->stream), "memset");
  if (!tiles.empty())
    CK(cudaMemcpyAsync(b->d_tiles, tiles.data(), sizeof(ErTile) * tiles.size(), cudaMemcpyHostToDevice, b->stream), "H2D tiles");
  b->wN = b->wR = b->wnb = b->wbufd = b->wrec = b->wdesc = b->wrt = b->wch = 0;
  b->wuni = false;
  b->wcs = b->wrods = 0;
  for (int f = 0; f < nf; ++f) {
    er_status st = upload_field(b, tmp[f], ER_DEVICE, fields[f], false);
    if (st != ER_OK) return st;
  }
  CK(cudaStreamSynchronize(b->stream), "sync");  // the host tile vector is freed at scope exit
  for (int f = 0; f < nf; ++f) cudaFree(tmp[f]);
  b->forcing_version += 1;
  return ER_OK;
}

er_status er_set_contact(er_batch *b, const er_contact *c) {
  if (!b) return ER_EINVAL;
  if (!c || !c->enable) {
    CK(cudaSetDevice(b->device), "cudaSetDevice");
    CK(cudaStreamSynchronize(b->stream), "sync");
    free_contact(b);
    return ER_OK;
  }
  Errors err;
  const int64_t R = b->n_rods, E = b->n_elems;
  auto nonneg = [&](double x, const char *what) { if (!(std::isfinite(x) && x >= 0.0)) err.add("%s = %g must be finite and >= 0", what, x); };
  if (!std::isfinite(c->k_n)) err.add("k_n = %g not finite", c->k_n);
  nonneg(c->gamma_n, "gamma_n");
  nonneg(c->mu_s, "mu_s");
  nonneg(c->mu_k, "mu_k");
  nonneg(c->v_stick, "v_stick");
  nonneg(c->cell0, "cell0");
  nonneg(c->pool_factor, "pool_factor");
  nonneg(c->skin, "skin");
  if (c->exclude < 0) err.add("exclude = %d < 0", c->exclude);
  if (c->n_levels < 0 || c->n_levels > ER_HHG_MAXLEV) err.add("n_levels = %d not in [0, %d]", c->n_levels, ER_HHG_MAXLEV);
  double nn = 0.0;
  if (c->plane_on) {
    for (int q = 0; q < 3; ++q) if (!std::isfinite(c->plane_n[q])) err.add("plane_n[%d] not finite", q);
    nn = std::sqrt(c->plane_n[0] * c->plane_n[0] + c->plane_n[1] * c->plane_n[1] + c->plane_n[2] * c->plane_n[2]);
    if (!(nn > 0.0)) err.add("plane_n must be non-zero");
    if (!std::isfinite(c->plane_d)) err.add("plane_d not finite");
  }
  if (c->radius)
    for (int64_t r = 0; r < R; ++r)
      if (!pos_finite(c->radius[r])) { err.add("radius[%lld] = %g must be positive and finite", (long long)r, c->radius[r]); break; }
  if (E + b->g_elems >= (1ll << 30)) err.add("contact supports < 2^30 elements per batch incl. ghosts (got %lld)", (long long)(E + b->g_elems));
  if (err.count) { b->last_error = err.msg; return ER_EINVAL; }
  if (c != &b->saved_contact) {  // kept for er_set_contact_ghosts, which re-applies them
    b->saved_contact = *c;
    if (c->radius) {
      b->saved_radius.assign(c->radius, c->radius + R);
      b->saved_contact.radius = b->saved_radius.data();
    }
    b->have_saved_contact = true;
  }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  CK(cudaStreamSynchronize(b->stream), "sync");
  free_contact(b);
  if (b->wN > 0) {  // contact runs the tile kernels: warp-sized tiles -> rod-aligned 256-slot tiles
    er_status st = relayout_to_tiles(b);
    if (st != ER_OK) return st;
  }
  ErContactParams &cp = b->cp;
  ErContactLaw &L = cp.law;
  L.k_n = c->k_n; L.gamma_n = c->gamma_n; L.mu_s = c->mu_s; L.mu_k = c->mu_k; L.v_stick = c->v_stick;
  L.plane_on = c->plane_on ? 1 : 0;
  for (int q = 0; q < 3; ++q) L.pn[q] = c->plane_on ? c->plane_n[q] / nn : 0.0;
  L.pd = c->plane_d;
  L.exclude = c->exclude;
  // per-rod contact radius (default sqrt(A/pi)) and stiffness scale E r; rest capsule extents.
  // Ghost rods (er_set_contact_ghosts) follow the own rods: RT rods, ET elements, NT nodes.
  const int64_t RT = R + b->g_rods, ET = E + b->g_elems, NT = b->n_nodes + b->g_nodes;
  std::vector<double> rad((size_t)std::max<int64_t>(RT, 1)), kr((size_t)std::max<int64_t>(RT, 1));
  double xmin = 0.0, xmax = 0.0;
  for (int64_t r = 0; r < RT; ++r) {
    double lmn, lmx;
    if (r < R) {
      rad[r] = c->radius ? c->radius[b->ord[r]] : std::sqrt(b->rod_A0[r] / 3.14159265358979323846);  // r packed
      kr[r] = b->rod_E0[r] * rad[r];
      lmn = b->rod_lmin[r];
      lmx = b->rod_lmax[r];
    } else {
      rad[r] = b->g_rad[r - R];
      kr[r] = b->g_kr[r - R];
      lmn = b->g_lmin[r - R];
      lmx = b->g_lmax[r - R];
    }
    const double lo = lmn + 2.0 * rad[r], hi = lmx + 2.0 * rad[r];
    xmin = r == 0 ? lo : std::min(xmin, lo);
    xmax = r == 0 ? hi : std::max(xmax, hi);
  }
  // Verlet skin (default: a quarter of the smallest contact radius)
  double rmin = 0.0;
  for (int64_t r = 0; r < RT; ++r) rmin = r == 0 ? rad[r] : std::min(rmin, rad[r]);
  cp.skin = c->skin > 0.0 ? c->skin : 0.25 * rmin;
  xmin += cp.skin;
  xmax += cp.skin;
  // HHG levels: cell_l = cell0 2^l
  double cell0 = c->cell0 > 0.0 ? c->cell0 : 1.25 * xmin;
  int nlev = c->n_levels;
  if (nlev == 0) {
    nlev = 1;
    while (nlev < ER_HHG_MAXLEV && cell0 * std::ldexp(1.0, nlev - 1) < 1.25 * xmax) ++nlev;
    if (c->cell0 == 0.0 && cell0 * std::ldexp(1.0, nlev - 1) < 1.25 * xmax) cell0 = 1.25 * xmax / std::ldexp(1.0, nlev - 1);
    nlev = std::min(nlev + 1, ER_HHG_MAXLEV);  // one level of headroom for stretched elements
  }
  if (RT > 0 && !(cell0 > 0.0)) { b->last_error = "HHG cell size must be positive"; return ER_EINVAL; }
  cp.nlev = nlev;
  for (int l = 0; l < ER_HHG_MAXLEV; ++l) {
    cp.cell[l] = cell0 * std::ldexp(1.0, l);
    cp.icell[l] = 1.0 / cp.cell[l];
  }
  int hb = 10;
  while (hb < 29 && (1ll << hb) < 2 * ET) ++hb;
  cp.hbits = hb;
  cp.n_elems = ET; cp.n_nodes = NT; cp.n_rods = RT;
  cp.fs = pad_to(ET, 32);
  const double pf = c->pool_factor > 0.0 ? c->pool_factor : 4.0;
  cp.pcap = std::max<int64_t>(1024, (int64_t)(pf * (double)ET));

  std::vector<int32_t> erod((size_t)std::max<int64_t>(ET, 1)), cord((size_t)std::max<int64_t>(RT, 1));
  std::vector<double> nrad((size_t)std::max<int64_t>(NT, 1)), nkr((size_t)std::max<int64_t>(NT, 1));
  for (int64_t r = 0, e0 = 0; r < RT; ++r) {  // element e of rod r: nodes e + r and e + r + 1
    const int64_t ne = r < R ? b->eoff[r + 1] - b->eoff[r] : b->g_nel[r - R];
    for (int64_t j = e0; j < e0 + ne; ++j) erod[j] = (int32_t)r;
    for (int64_t n = e0 + r; n <= e0 + ne + r; ++n) { nrad[n] = rad[r]; nkr[n] = kr[r]; }
    cord[r] = r < R ? b->ord[r] : (int32_t)r;  // a ghost rod reports as n_rods + its index
    e0 += ne;
  }
  double *d_nrad = nullptr, *d_nkr = nullptr;
  double *d_rad = nullptr, *d_kr = nullptr;
  int32_t *d_erod = nullptr;
  const int64_t T = 1ll << hb;
#define CA(ptr, n) CK(dalloc(b, &(ptr), (n)), "cudaMalloc(contact)")
  CA(d_rad, RT); CA(d_kr, RT); CA(d_erod, ET);
  CA(d_nrad, NT); CA(d_nkr, NT);
  CA(b->d_cord, RT);
  cp.rad = d_rad; cp.kr = d_kr; cp.erod = d_erod; cp.nrad = d_nrad; cp.nkr = d_nkr;
  cp.ord = b->d_cord;
  CA(cp.cnode, 6 * NT); CA(cp.cbuild, 3 * NT); CA(cp.rebuild, 1);
  CA(cp.gext, 3 * ER_HHG_MAXLEV); CA(cp.gdim, 4 * ER_HHG_MAXLEV);
  CA(cp.key, ET); CA(cp.key_s, ET); CA(cp.val, ET); CA(cp.val_s, ET);
  CA(cp.table, T); CA(cp.code_s, ET);
  CA(cp.boxa, ET); CA(cp.boxb, ET); CA(cp.qidx, ET);
  CA(cp.cnt, ET); CA(cp.cand, ER_CAND_K * ET);
  CA(cp.fc, 6 * cp.fs);
  CA(cp.head, NT); CA(cp.pnext, cp.pcap); CA(cp.psrc, cp.pcap); CA(cp.pf, 6 * cp.pcap);
  CA(cp.ctr, 8); CA(cp.bctr, 8);
#undef CA
  cp.fault = b->d_fault;
  CK(er_contact_tmp_bytes(ET, hb, &b->sort_bytes), "cub temp size");
  CK(cudaMalloc(&b->sort_tmp, std::max<size_t>(b->sort_bytes, 16)), "cudaMalloc(sort)");
  b->device_bytes += (int64_t)b->sort_bytes;
  if (RT > 0) {
    CK(cudaMemcpyAsync(d_rad, rad.data(), sizeof(double) * RT, cudaMemcpyHostToDevice, b->stream), "H2D rad");
    CK(cudaMemcpyAsync(d_kr, kr.data(), sizeof(double) * RT, cudaMemcpyHostToDevice, b->stream), "H2D kr");
    CK(cudaMemcpyAsync(d_erod, erod.data(), sizeof(int32_t) * ET, cudaMemcpyHostToDevice, b->stream), "H2D erod");
    CK(cudaMemcpyAsync(d_nrad, nrad.data(), sizeof(double) * NT, cudaMemcpyHostToDevice, b->stream), "H2D nrad");
    CK(cudaMemcpyAsync(d_nkr, nkr.data(), sizeof(double) * NT, cudaMemcpyHostToDevice, b->stream), "H2D nkr");
    CK(cudaMemcpyAsync(b->d_cord, cord.data(), sizeof(int32_t) * RT, cudaMemcpyHostToDevice, b->stream), "H2D cord");
  }
  if (NT > 0) CK(cudaMemsetAsync(cp.cnode, 0, sizeof(double) * 6 * NT, b->stream), "memset");
  CK(cudaMemsetAsync(cp.ctr, 0, 8 * sizeof(unsigned long long), b->stream), "memset");
  CK(cudaMemsetAsync(cp.bctr, 0, 8 * sizeof(unsigned long long), b->stream), "memset");
  CK(cudaMemsetAsync(cp.rebuild, 1, sizeof(int32_t), b->stream), "memset");
  CK(cudaMemsetAsync(cp.fc, 0, 6 * sizeof(double) * cp.fs, b->stream), "memset");
  CK(cudaStreamSynchronize(b->stream), "sync");
  if (!std::getenv("ER_NO_GRAPH"))
    CK(er_contact_graph(&cp, b->sort_tmp, b->sort_bytes, &b->cgraph, &b->cgraph_kernels), "contact graph");
  b->contact_on = true;
  return ER_OK;
}

er_status er_set_contact_ghosts(er_batch *b, int64_t n_ghost, const int32_t *n_elems, const double *radius,
                                const double *stiffness, const double *lhat_min, const double *lhat_max) {
  if (!b) return ER_EINVAL;
  Errors err;
  if (n_ghost < 0) err.add("n_ghost = %lld < 0", (long long)n_ghost);
  if (n_ghost > 0 && !(n_elems && radius && stiffness && lhat_min && lhat_max)) err.add("ghost arrays must be non-NULL");
  if (b->split_begun) err.add("a split step is in progress (er_step_begin without er_step_finish)");
  int64_t ge = 0;
  for (int64_t g = 0; g < n_ghost && !err.count; ++g) {
    if (n_elems[g] < 1) err.add("ghost n_elems[%lld] = %d < 1", (long long)g, n_elems[g]);
    if (!pos_finite(radius[g])) err.add("ghost radius[%lld] = %g must be positive and finite", (long long)g, radius[g]);
    if (!std::isfinite(stiffness[g])) err.add("ghost stiffness[%lld] not finite", (long long)g);
    if (!(pos_finite(lhat_min[g]) && pos_finite(lhat_max[g]) && lhat_min[g] <= lhat_max[g]))
      err.add("ghost rest lengths [%lld] must satisfy 0 < lhat_min <= lhat_max", (long long)g);
    ge += n_elems[g];
  }
  if (err.count) { b->last_error = err.msg; return ER_EINVAL; }
  b->g_rods = n_ghost;
  b->g_elems = ge;
  b->g_nodes = ge + n_ghost;
  b->g_nel.assign(n_elems, n_elems + n_ghost);
  b->g_rad.assign(radius, radius + n_ghost);
  b->g_kr.assign(stiffness, stiffness + n_ghost);
  b->g_lmin.assign(lhat_min, lhat_min + n_ghost);
  b->g_lmax.assign(lhat_max, lhat_max + n_ghost);
  if (b->contact_on && b->have_saved_contact) return er_set_contact(b, &b->saved_contact);
  return ER_OK;
}

er_status er_step_begin(er_batch *b, double dt) {
  if (!b) return ER_EINVAL;
  if (!b->contact_on || b->kernel_mode == 1) { b->last_error = "er_step_begin needs contact (fused kernels)"; return ER_EINVAL; }
  if (b->split_begun) { b->last_error = "er_step_begin twice without er_step_finish"; return ER_EINVAL; }
  b->split_mode = 1;
  const er_status st = er_step(b, 1, dt);
  b->split_mode = 0;
  if (st == ER_OK) {
    b->split_begun = true;
    b->split_dt = dt;
  }
  return st;
}

er_status er_step_finish(er_batch *b, double dt) {
  if (!b) return ER_EINVAL;
  if (!b->split_begun) { b->last_error = "er_step_finish without er_step_begin"; return ER_EINVAL; }
  if (dt != b->split_dt) { b->last_error = "er_step_finish dt differs from er_step_begin's"; return ER_EINVAL; }
  b->split_mode = 2;
  const er_status st = er_step(b, 1, dt);
  b->split_mode = 0;
  b->split_begun = false;
  return st;
}

er_status er_contact_records(er_batch *b, int32_t dst_mem, double *dst) {
  if (!b || !dst) return ER_EINVAL;
  if (!b->contact_on) { b->last_error = "contact is not enabled"; return ER_EINVAL; }
  if (dst_mem != ER_HOST && dst_mem != ER_DEVICE) { b->last_error = "dst_mem must be ER_HOST or ER_DEVICE"; return ER_EINVAL; }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  const size_t bytes = sizeof(double) * 6 * (size_t)b->n_nodes;
  CK(cudaMemcpyAsync(dst, b->cp.cnode, bytes, dst_mem == ER_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                     b->stream), "node records");
  CK(cudaStreamSynchronize(b->stream), "sync");
  return ER_OK;
}

er_status er_set_ghost_records(er_batch *b, int32_t src_mem, const double *src) {
  if (!b || !src) return ER_EINVAL;
  if (!b->contact_on || b->g_rods == 0) { b->last_error = "no ghost rods (er_set_contact_ghosts) or contact off"; return ER_EINVAL; }
  if (src_mem != ER_HOST && src_mem != ER_DEVICE) { b->last_error = "src_mem must be ER_HOST or ER_DEVICE"; return ER_EINVAL; }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  const size_t bytes = sizeof(double) * 6 * (size_t)b->g_nodes;
  CK(cudaMemcpyAsync(b->cp.cnode + 6 * b->n_nodes, src, bytes,
                     src_mem == ER_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, b->stream), "ghost records");
  if (src_mem == ER_HOST) CK(cudaStreamSynchronize(b->stream), "sync");  // the caller may reuse its buffer
  return ER_OK;
}

er_status er_get_contact_stats(er_batch *b, er_contact_stats *out) {
  if (!b || !out) return ER_EINVAL;
  std::memset(out, 0, sizeof *out);
  if (!b->contact_on) return ER_OK;
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  unsigned long long c[8], bc[8];
  CK(cudaMemcpyAsync(c, b->cp.ctr, sizeof c, cudaMemcpyDeviceToHost, b->stream), "D2H contact stats");
  CK(cudaMemcpyAsync(bc, b->cp.bctr, sizeof bc, cudaMemcpyDeviceToHost, b->stream), "D2H contact stats");
  CK(cudaStreamSynchronize(b->stream), "sync");
  out->candidates = (int64_t)bc[0];
  out->list_entries = (int64_t)bc[1];
  out->scanned = (int64_t)bc[2];
  out->long_lists = (int64_t)bc[4];
  out->builds = (int64_t)bc[5];
  out->contacts = (int64_t)c[1];
  out->cross_level = (int64_t)c[2];
  out->plane_contacts = (int64_t)c[3];
  out->pool_used = (int64_t)c[0];
  out->skin = b->cp.skin;
  out->n_levels = b->cp.nlev;
  out->level_mask = (int32_t)bc[3];
  out->cell0 = b->cp.cell[0];
  return ER_OK;
}

er_status er_get_state(er_batch *b, int32_t dst_mem, double *positions, double *velocities, double *directors,
                       double *omega, double *t) {
  NvtxRange nvtx_("er_get_state");
  if (!b) return ER_EINVAL;
  if (dst_mem != ER_HOST && dst_mem != ER_DEVICE) { b->last_error = "dst_mem must be ER_HOST or ER_DEVICE"; return ER_EINVAL; }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  er_status st;
  if ((st = download_field(b, positions, dst_mem, FIELD_POS)) != ER_OK) return st;
  if ((st = download_field(b, velocities, dst_mem, FIELD_VEL)) != ER_OK) return st;
  if ((st = download_field(b, directors, dst_mem, FIELD_DIR)) != ER_OK) return st;
  if ((st = download_field(b, omega, dst_mem, FIELD_OMEGA)) != ER_OK) return st;
  CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
  if (t) *t = b->t;
  return ER_OK;
}

er_status er_set_state(er_batch *b, int32_t src_mem, const double *positions, const double *velocities,
                       const double *directors, const double *omega, const double *t) {
  NvtxRange nvtx_("er_set_state");
  if (!b) return ER_EINVAL;
  if (src_mem != ER_HOST && src_mem != ER_DEVICE) { b->last_error = "src_mem must be ER_HOST or ER_DEVICE"; return ER_EINVAL; }
  if (t && !std::isfinite(*t)) { b->last_error = "t is not finite"; return ER_EINVAL; }
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  er_status st;
  if (positions && (st = upload_field(b, positions, src_mem, FIELD_POS, false)) != ER_OK) return st;
  if (velocities && (st = upload_field(b, velocities, src_mem, FIELD_VEL, false)) != ER_OK) return st;
  if (directors && (st = upload_field(b, directors, src_mem, FIELD_DIR, false)) != ER_OK) return st;
  if (omega && (st = upload_field(b, omega, src_mem, FIELD_OMEGA, false)) != ER_OK) return st;
  if (b->contact_on && positions) CK(cudaMemsetAsync(b->cp.rebuild, 1, sizeof(int32_t), b->stream), "memset");
  CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
  if (t) b->t = *t;
  return ER_OK;
}

er_status er_diagnostics(er_batch *b, double out[ER_NDIAG]) {
  NvtxRange nvtx_("er_diagnostics");
  if (!b || !out) return ER_EINVAL;
  CK(cudaSetDevice(b->device), "cudaSetDevice");
  ErStepParams p = params_of(b);
  p.t = b->t;
  int dblock = b->block;  // slots per tile at most (warp layouts: small tiles)
  if (b->wN > 0 && b->wrt > 0) {
    const int64_t slots = (int64_t)b->wrt * (b->wN + 1);
    dblock = slots <= 64 ? 64 : slots <= 128 ? 128 : slots <= 256 ? 256 : 512;
  }
  CK(er_launch_diag(&p, dblock, b->d_diag_out, b->stream), "diag kernel");
  CK(cudaMemcpyAsync(out, b->d_diag_out, sizeof(double) * ER_NDIAG, cudaMemcpyDeviceToHost, b->stream), "D2H diag");
  CK(cudaStreamSynchronize(b->stream), "cudaStreamSynchronize");
  return ER_OK;
}

er_status er_get_phase_times(const er_batch *b, er_phase_times *out) {
  if (!b || !out) return ER_EINVAL;
  out->step_kernel_ms = b->phase_ms[0];
  out->step_kernel_launches = b->phase_n[0];
  out->contact_ms = b->phase_ms[1];
  out->contact_evals = b->phase_n[1];
  return ER_OK;
}

er_status er_fault(const er_batch *b, int64_t *rod, int32_t *bits) {
  if (!b) return ER_EINVAL;
  if (rod) *rod = b->fault_rod;
  if (bits) *bits = b->fault_bits;
  return ER_OK;
}

er_status er_query(const er_batch *b, er_info *info) {
  if (!b || !info) return ER_EINVAL;
  info->n_rods = b->n_rods;
  info->n_elems_total = b->n_elems;
  info->n_nodes_total = b->n_nodes;
  info->n_voronoi_total = b->n_vor;
  info->n_tiles = b->n_tiles;
  info->tile_slots = b->block;
  info->warp_rod_elems = b->wN;
  info->warp_buffers = b->wnb;
  info->shared_material = b->wuni ? 1 : 0;
  info->reserved_ = 0;
  info->device = b->device;
  info->stream = (void *)b->stream;
  info->launches = b->launches;
  info->device_bytes = b->device_bytes;
  info->t = b->t;
  // bytes one fused step moves: state read + written once (r, v: 6 per node; d1, d2, w: ER_EPL
  // per element), the 192-byte rod record (48 bytes in a shared-material batch) read once, static
  // kappa0 read once
  double bytes = 16.0 * (6.0 * b->n_nodes + (double)ER_EPL * b->n_elems) + 8.0 * (b->wuni ? ER_WREC : ER_REC) * b->n_rods;
  if (b->has_kappa0) bytes += 24.0 * b->n_vor;
  info->bytes_per_step = bytes;
  return ER_OK;
}

void er_destroy(er_batch *b) {
  if (!b) return;
  cudaSetDevice(b->device);
  if (b->stream) cudaStreamSynchronize(b->stream);
  free_all(b);
  delete b;
}

}  // extern "C"
