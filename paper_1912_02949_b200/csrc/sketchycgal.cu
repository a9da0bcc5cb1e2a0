// sketchycgal.cu -- host driver and C ABI (include/sketchycgal.h) of the B200-native
// SketchyCGAL MaxCut hot path.  See DESIGN.md for the method, the arithmetic
// contract, the data layout and the kernel rooflines.
//
// A context owns one or more row shards (struct Shard).  One GPU: one shard owning
// all rows.  Multi-GPU (one process per GPU): one shard per rank, peers reached
// through CUDA IPC mappings (NVLink), NCCL only for setup and the one-shot
// reconstruction reductions.  Emulated shards: P shards of one problem on one
// device in one context, peers = the sibling shards.  The
// iteration loop is the same code for all three: each step launches the kernel for
// every shard, then (P > 1) the k_pull collective for every shard.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -lineinfo
// (--fmad=false is part of the arithmetic contract: no contraction of a*b+c).
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sketchycgal.h"
#include "kernels.cuh"
#include "linalg.h"

#ifdef SCG_WITH_NCCL
#include <nccl.h>
#endif

using namespace scg;
using namespace scg_host;

namespace {

// Host vectors of the init passes without value-initialization: the first touch (and its page
// faults) happens in the parallel fill loops instead of a serial zeroing pass.
template <class T>
struct noinit_alloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = noinit_alloc<U>;
  };
  noinit_alloc() = default;
  template <class U>
  noinit_alloc(const noinit_alloc<U> &) noexcept {}
  template <class U>
  void construct(U *p) noexcept {
    ::new ((void *)p) U;
  }
  template <class U, class... A>
  void construct(U *p, A &&...a) {
    ::new ((void *)p) U(std::forward<A>(a)...);
  }
};
template <class T>
using hvec = std::vector<T, noinit_alloc<T>>;

enum KClass {
  KC_LANCZOS_A = 0, KC_LANCZOS_B, KC_TRIDIAG, KC_LANCZOS_C, KC_NORM_X, KC_COMBINE, KC_MONITOR, KC_PRIMAL,
  KC_DUAL_SKETCH, KC_SKETCH, KC_PULL, KC_OTHER, KC_PASS1, KC_GEN, KC_RESIDENT, KC_PASS1_FLOW, KC_COUNT
};
const char *kKClassName[KC_COUNT] = {"lanczos_a_spmv_dot", "lanczos_b_axpy_norm", "tridiag_mineig",
                                     "lanczos_c_spmv_regen", "norm_x", "combine_stored", "monitor_spmv",
                                     "primal_z_gpart", "dual_next_g", "sketch_flush", "pull_collective", "other",
                                     "lanczos_pass1_fused", "gen_start_side", "resident_iteration",
                                     "lanczos_pass1_in_flow"};

struct EvPair {
  cudaEvent_t a, b;
  int cls;
};

enum { SLOT_NU0 = 0, SLOT_OM, SLOT_RHO, SLOT_XX, SLOT_MON, SLOT_NZ, SLOT_INIT, SLOT_BAR, SLOT_GEN, SLOT_BALL, SLOT_COUNT };

}  // namespace

// One contiguous row block [rb, rb + nl) and all its device state.
struct Shard {
  int rank = 0;
  int64_t nl = 0, rb = 0, nlpad = 0;
  long long nnz_off = 0;
  int *rp = nullptr, *col = nullptr;
  double *val = nullptr, *wts = nullptr, *ldiag = nullptr, *cdiag = nullptr;
  double *d = nullptr, *z = nullptr, *y = nullptr, *a = nullptr, *v = nullptr;
  double *V = nullptr, *ckr = nullptr;  // deferred sketch updates: ring of kSketchB eigenvectors + coefficients
  double *G = nullptr;  // gathered region: [x | W slot 0 (= g) | W slot 1 | ...], each npad long
  double *gB = nullptr; // side-stream draws: start vector of even iterations (odd ones use W slot 0)
  double *S = nullptr, *Om = nullptr, *gpart = nullptr;
  double *U = nullptr, *tmp1 = nullptr, *tmp2 = nullptr, *dmat = nullptr, *partial = nullptr, *dlam = nullptr;
  double *dscalar = nullptr;
  DevScalars *sc = nullptr;
  XSlot *slots = nullptr;
  scg_iter_rec *dlog = nullptr;
  int *longrows = nullptr;  // rows of 33..1024 entries (warp per row), longest first
  int nlong = 0;
  int *heavyrows = nullptr;  // rows of more than 1024 entries (block per row), longest first
  int nheavy = 0;
  int *sell_col = nullptr;
  int2 *sell_meta = nullptr;
  double *sell_val = nullptr;
  double sell_m0 = 0.0, sell_slots = 0.0;
  bool sell_uniform = false;
  int nslice = 0;
  unsigned *work = nullptr;  // dynamic slice counter of k_lanczos_a (graphs with long rows)
  int *ell_col = nullptr;    // ELL-W layout (rows of <= kEllMax entries), W = ellw; 0: none
  double *ell_val = nullptr;
  int ellw = 0, padc = 0;
  int grid_ell = 1, grid_ell_mon = 1, grid_ell_c = 1, grid_dual_s = 1;
  bool dyn = false;
  // row relabeling (SELL engine): local row nu holds input row rb + origloc[nu]
  std::vector<int> origloc;
  int *orig = nullptr;            // device copy of origloc
  hvec<int> h_rp, h_col;   // host CSR (device labels) kept from build_shard to build_layout
  hvec<double> h_w;
  // sharding
  unsigned char *mask = nullptr;  // device [nl], nullptr when world == 1
  Mailbox *mb = nullptr;
  double **peerG = nullptr;       // device [world]
  Mailbox **peerMB = nullptr;     // device [world]
  std::vector<void *> ipc_opened;
  int64_t halo_rows = 0;
  // grids
  unsigned long long *gflag = nullptr;  // grid-barrier flag of the fused pass-1 kernel
  bool ws = false;  // k_lanczos_a as the warp-specialized TMA kernel (SCG_WS_SPMV)
  int grid_ws = 1;
  int grid_rows = 1, grid_primal = 1, grid_spmv = 1, grid_b = 1, grid_comb = 1, grid_dual = 1, grid_norm = 1,
      grid_mon = 1, grid_flush = 1, grid_a = 1, grid_btma = 1;
  double kb[KC_COUNT] = {0};  // algorithmic bytes of one launch of each class
};

struct scg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // one GPU: the next iteration's start vector is drawn on this lower-priority stream while the
  // current iteration's Lanczos passes run (evA: its buffer is free; evB: drawn) -- DESIGN.md section 5
  cudaStream_t side = nullptr;
  cudaEvent_t evA = nullptr, evB = nullptr;
  bool side_rng = false;
  // small graphs (L2-resident): each iteration is one launch of one thread-block cluster (k_resident)
  int res_cl = 0;  // cluster size, 0: off
  bool own_stream = false;
  int nsm = 148;
  int64_t n = 0, npad = 0;
  int R = 0;
  uint32_t flags = 0;
  double alpha_orig = 0, alpha = 0, beta0 = 1, b = 0, nrmL = 1, lnN = 0;
  uint64_t seed = 0;
  // sharding: world ranks; this context holds shards sh (all of them when emulating)
  int world = 1, mode = 0;  // mode 0: single, 1: emulated shards, 2: one rank of a multi-process job
  bool box = false;           // constraint set K = {klo <= u <= khi} (scaled units): SCG_INEQ or sketchycgal_set_box
  double klo = 0.0, khi = 0.0;
  int ball = 0;               // K = {||u - b|| <= delta}: 2 l2, 1 l1 (sketchycgal_set_ball[_l1]; box is set too)
  double delta = 0.0;         //   scaled units
  bool fused = false;        // one GPU: Lanczos pass 1 as one persistent kernel (SCG_FUSED_PASS1)
  unsigned long long gphase = 0;  // grid-barrier phases issued so far (fused pass 1)
  bool pdl = true;          // programmatic dependent launches (SCG_NO_PDL disables)
  bool btma = false;        // TMA-staged k_lanczos_b (SCG_TMA_B; measured slower: 115-166 vs 93 us on c3)
  int rank = 0;
  std::vector<int64_t> splits;
  std::vector<Shard *> sh;
  std::vector<int> gmap;  // input vertex id -> device row label (identity without relabeling)
  unsigned long long epoch = 0;
#ifdef SCG_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  bool hcomm = false;     // multi-process setup transport: the caller's host callbacks (else NCCL)
  scg_host_comm hc{};
  double *dred = nullptr;  // device scratch for host all-reduces (mode 2)
  double *dmet = nullptr;  // device scratch of the one-shot metrics (feasibility)
  int8_t *dchi = nullptr;  // device scratch of the rounded cut
  int64_t dchi_cap = 0;
  int64_t t = 0;
  int64_t launches = 0;
  int64_t log_cap = 0;
  // Lanczos vector storage: W slot 0 = start vector g; store mode: slot j-1 = w_j (j <= q);
  // regenerate mode: slots 1, 2 = ring of w_i
  int wcap = 0;
  bool store = true;
  int qfix = 0;  // > 0: fixed Lanczos bound instead of the q_t schedule (sketchycgal_set_lanczos_q)
  // deferred sketch updates (k_sketch_flush): iterations pending, their 1 - eta, last v slot
  int spend = 0, vlast = 0;
  double ome[kSketchB] = {0};
  double *vslot(const Shard *s, int j) const { return s->V + (long long)j * s->nlpad; }
  // reconstruction
  bool have_recon = false;
  std::vector<double> lam_raw, lam_orig, lam_tc, err;
  // profiling
  std::vector<EvPair> pending;
  std::vector<cudaEvent_t> evpool;
  int64_t kl[KC_COUNT] = {0};
  int64_t ks[KC_COUNT] = {0};  // launches timed (every prof_every-th launch of each class)
  int prof_every = 16;
  bool in_flow = false;  // inside a pass 1 bracketed as a whole (KC_PASS1_FLOW): no per-launch events
  double kms[KC_COUNT] = {0};
  double kbytes_sum[KC_COUNT] = {0};
  // errors
  int failed = 0;
  std::string err_msg;

  int64_t nl_total() const {
    int64_t s = 0;
    for (auto *p : sh) s += p->nl;
    return s;
  }
  double *xg(const Shard *s) const { return s->G; }
  // buffer of the start vector w_1 of iteration t
  double *gslot(const Shard *s, int64_t t) const { return (side_rng && !(t & 1)) ? s->gB : s->G + npad; }
  double *wslot(const Shard *s, int j) const { return s->G + (long long)(1 + j) * npad; }
};

namespace {

scg_status fail(scg_ctx *c, scg_status st, const std::string &msg) {
  if (c) {
    c->err_msg = msg;
    if (st == SCG_ECUDA || st == SCG_ENCCL) c->failed = 1;
  }
  return st;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, SCG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#ifdef SCG_WITH_NCCL
#define NK(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess) return fail(c, SCG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#endif

int grid_for(int64_t rows, int maxgrid) {
  int64_t g = (rows + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  return (int)std::min<int64_t>(g, maxgrid);
}

void ev_flush(scg_ctx *c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->stream);
  if (c->side) cudaStreamSynchronize(c->side);
  for (auto &p : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->kms[p.cls] += ms;
    c->evpool.push_back(p.a);
    c->evpool.push_back(p.b);
  }
  c->pending.clear();
}

cudaEvent_t ev_get(scg_ctx *c) {
  if (c->evpool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->evpool.back();
  c->evpool.pop_back();
  return e;
}

template <typename Kern, typename... Args>
void launch_on(scg_ctx *c, cudaStream_t stream, bool pdl, int cls, double bytes, Kern kern, dim3 grid, dim3 block,
               size_t smem, Args... args);
template <typename Kern, typename... Args>
void launch_smem(scg_ctx *c, int cls, double bytes, Kern kern, dim3 grid, dim3 block, size_t smem, Args... args) {
  launch_on(c, c->stream, c->pdl, cls, bytes, kern, grid, block, smem, args...);
}
template <typename Kern, typename... Args>
void launch_on(scg_ctx *c, cudaStream_t stream, bool pdl, int cls, double bytes, Kern kern, dim3 grid, dim3 block,
               size_t smem, Args... args) {
  // SCG_PROFILE: CUDA events around every prof_every-th launch of each kernel class (events
  // between kernels serialize programmatic launches; timing all of them costs ~5% on c3)
  const bool prof = (c->flags & SCG_PROFILE) != 0 && !c->in_flow && c->kl[cls] % c->prof_every == 0;
  if (prof) c->ks[cls]++;
  EvPair p{};
  if (prof) {
    if (c->pending.size() >= 8192) ev_flush(c);
    p.a = ev_get(c);
    p.b = ev_get(c);
    p.cls = cls;
    cudaEventRecord(p.a, stream);
  }
  if (pdl) {  // programmatic dependent launch (kernels.cuh pdl_entry)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
  } else {
    kern<<<grid, block, smem, stream>>>(args...);
  }
  if (prof) {
    cudaEventRecord(p.b, stream);
    c->pending.push_back(p);
  }
  c->kl[cls]++;
  c->kbytes_sum[cls] += bytes;
  c->launches++;
}

template <typename Kern, typename... Args>
void launch(scg_ctx *c, int cls, double bytes, Kern kern, dim3 grid, dim3 block, Args... args) {
  launch_smem(c, cls, bytes, kern, grid, block, 0, args...);
}

// Cooperative launch (every block co-resident: the fused pass-1 kernel's grid barriers),
// with the programmatic-serialization attribute when enabled; same profiling as launch_smem.
template <typename Kern, typename... Args>
void launch_coop(scg_ctx *c, int cls, double bytes, Kern kern, dim3 grid, dim3 block, Args... args) {
  const bool prof = (c->flags & SCG_PROFILE) != 0 && !c->in_flow && c->kl[cls] % c->prof_every == 0;
  if (prof) c->ks[cls]++;
  EvPair p{};
  if (prof) {
    if (c->pending.size() >= 8192) ev_flush(c);
    p.a = ev_get(c);
    p.b = ev_get(c);
    p.cls = cls;
    cudaEventRecord(p.a, c->stream);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeCooperative;
  attr[na].val.cooperative = 1;
  ++na;
  if (c->pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, args...);
  if (prof) {
    cudaEventRecord(p.b, c->stream);
    c->pending.push_back(p);
  }
  c->kl[cls]++;
  c->kbytes_sum[cls] += bytes;
  c->launches++;
}

// One-cluster launch (k_resident): grid = one cluster of cl CTAs, with the programmatic-serialization
// attribute when enabled; same profiling as launch_smem.
template <typename Kern, typename... Args>
void launch_cluster(scg_ctx *c, int cls, double bytes, Kern kern, int cl, dim3 block, size_t smem, Args... args) {
  const bool prof = (c->flags & SCG_PROFILE) != 0 && !c->in_flow && c->kl[cls] % c->prof_every == 0;
  if (prof) c->ks[cls]++;
  EvPair p{};
  if (prof) {
    if (c->pending.size() >= 8192) ev_flush(c);
    p.a = ev_get(c);
    p.b = ev_get(c);
    p.cls = cls;
    cudaEventRecord(p.a, c->stream);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = cl;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (c->pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, args...);
  if (prof) {
    cudaEventRecord(p.b, c->stream);
    c->pending.push_back(p);
  }
  c->kl[cls]++;
  c->kbytes_sum[cls] += bytes;
  c->launches++;
}

Rows rows_of(const Shard *s, bool dyn = false) {
  Rows r{};
  r.work = dyn ? s->work : nullptr;
  r.longrows = s->longrows;
  r.nlong = s->nlong;
  r.heavyrows = s->heavyrows;
  r.nheavy = s->nheavy;
  r.meta = s->sell_meta;
  r.scol = s->sell_col;
  r.sval = s->sell_val;
  r.m0 = s->sell_m0;
  r.nslice = s->nslice;
  r.ecol = s->ell_col;
  r.eval = s->ell_val;
  r.padc = s->padc;
  return r;
}

// Kernel instantiation for a shard's layout: uniform weights (values in the column's sign bit) or
// not, and the ELL width (0: SELL + long rows).
constexpr int kEllWidths[] = {2, 3, 4, 6, 8};
// the resident cluster kernel exists for SELL (0) and ELL-3 / ELL-4; other widths use its SELL form
#define SCG_RES_W(W) (((W) == 3 || (W) == 4 || (W) == (3 | kEllPos) || (W) == (4 | kEllPos)) ? (W) : 0)
#define SCG_PICK_RES(U, W)                                                                          \
  (SCG_RES_W(W) == 3 ? ((U) ? k_resident<true, 3> : k_resident<false, 3>)                           \
   : SCG_RES_W(W) == 4 ? ((U) ? k_resident<true, 4> : k_resident<false, 4>)                         \
   : SCG_RES_W(W) == (3 | kEllPos) ? k_resident<true, 3 | kEllPos>                                  \
   : SCG_RES_W(W) == (4 | kEllPos) ? k_resident<true, 4 | kEllPos>                                  \
                       : ((U) ? k_resident<true, 0> : k_resident<false, 0>))
// W: ELL width code (kernels.cuh kEllPos); the sign-free codes exist for uniform weights only
#define SCG_PICK(K, U, W)                                          \
  ((W) == (3 | kEllPos) ? K<true, 3 | kEllPos>                      \
   : (W) == (4 | kEllPos) ? K<true, 4 | kEllPos>                    \
   : (W) == 2   ? ((U) ? K<true, 2> : K<false, 2>)                 \
   : (W) == 3 ? ((U) ? K<true, 3> : K<false, 3>)                   \
   : (W) == 4 ? ((U) ? K<true, 4> : K<false, 4>)                   \
   : (W) == 6 ? ((U) ? K<true, 6> : K<false, 6>)                   \
   : (W) == 8 ? ((U) ? K<true, 8> : K<false, 8>)                   \
              : ((U) ? K<true, 0> : K<false, 0>))

Net net_of(const scg_ctx *c, const Shard *s, unsigned long long E) {
  Net n{};
  n.mask = c->world > 1 ? s->mask : nullptr;
  n.G = s->G;
  n.peerG = s->peerG;
  n.peerMB = s->peerMB;
  n.mb = s->mb;
  n.P = c->world;
  n.me = s->rank;
  n.nowait = c->hcomm && c->hc.sync_collectives ? 1 : 0;
  n.E = E;
  return n;
}

// P > 1: the collective half of a reduction -- every shard of this context waits
// for all ranks' contributions to epoch E and finalizes.
void pull_all(scg_ctx *c, int kind, int ns, unsigned long long E, const FinArgs &f0) {
  if (c->world <= 1) return;
  if (c->hcomm && c->hc.sync_collectives) {  // ranks sharing a GPU: meet on the host, the pull only checks
    if (cudaStreamSynchronize(c->stream) != cudaSuccess || c->hc.barrier(c->hc.ctx) != 0) {
      c->failed = 1;
      c->err_msg = "host barrier before a collective failed";
    }
  }
  for (Shard *s : c->sh) {
    FinArgs f = f0;
    if (kind == FK_NZ || kind == FK_NZZ) f.log = s->dlog;
    if (kind == FK_FROB) f.out = s->dscalar;
    launch(c, KC_PULL, 0.0, k_pull, dim3(1), dim3(32), kind, ns, net_of(c, s, E), s->sc, f);
  }
}

// Sum a small host vector over the ranks of a multi-process job (identity otherwise).
scg_status host_allreduce(scg_ctx *c, std::vector<double> &v) {
  if (c->mode != 2 || c->world <= 1 || v.empty()) return SCG_OK;
  if (c->hcomm) {
    if (c->hc.allreduce_sum(c->hc.ctx, v.data(), (int64_t)v.size()) != 0) return fail(c, SCG_ECOMM, "host allreduce");
    return SCG_OK;
  }
#ifdef SCG_WITH_NCCL
  const size_t bytes = sizeof(double) * v.size();
  if (v.size() > (size_t)kMaxR * kMaxR * 4) return fail(c, SCG_EINVAL, "host_allreduce: vector too long");
  CK(cudaMemcpyAsync(c->dred, v.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  NK(ncclAllReduce(c->dred, c->dred, v.size(), ncclDouble, ncclSum, c->comm, c->stream));
  CK(cudaMemcpyAsync(v.data(), c->dred, bytes, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return SCG_OK;
#else
  return fail(c, SCG_EUNSUPPORTED, "built without NCCL");
#endif
}

void free_shard(Shard *s) {
  void *ptrs[] = {s->rp, s->col, s->val, s->wts, s->ldiag, s->cdiag, s->d, s->z, s->y, s->a, s->v, s->G,
                  s->S, s->Om, s->gpart, s->U, s->tmp1, s->tmp2, s->dmat, s->partial, s->dlam, s->dscalar,
                  s->sc, s->slots, s->dlog, s->longrows, s->heavyrows, s->sell_col, s->sell_meta, s->sell_val,
                  s->mask, s->mb, s->peerG, s->peerMB, s->orig, s->V, s->ckr, s->work, s->gflag, s->ell_col,
                  s->ell_val, s->gB};
  for (void *p : s->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void *p : ptrs)
    if (p) cudaFree(p);
  delete s;
}

// Row relabeling of one shard (SELL engine): within windows of kSortWin consecutive rows,
// rows sorted by length, longest first (long rows lead), ties by input order.  A
// symmetric permutation of L: the SpMV slices become contiguous rows.  The CAC-3 chain
// order (ascending INPUT column) and every exact sum are unchanged, so results are
// bitwise those of the input labeling; the seeded streams and all outputs use input ids.
constexpr int64_t kSortWin = 256;
void relabel_perm(const int64_t *rp, const int32_t *colp, int64_t nl, int64_t rb, bool halo_first,
                  std::vector<int> &origloc) {
  origloc.resize((size_t)nl);
  for (int64_t r = 0; r < nl; ++r) origloc[(size_t)r] = (int)r;
  if (halo_first) {
    // sharded: the rows other ranks read (a column outside this shard; L is symmetric) first,
    // in input order, then the interior rows -- so that only the first blocks of the kernels
    // producing gathered vectors store into peer memory and need the system-scope fence
    // (commit_and_ticket's peer flag).  A symmetric permutation: results are bitwise unchanged.
    const int64_t base = rp[0];
    std::vector<unsigned char> halo((size_t)nl, 0);
#pragma omp parallel for schedule(static, 4096)
    for (int64_t r = 0; r < nl; ++r)
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
        const int64_t cc = colp[k - base];
        if (cc < rb || cc >= rb + nl) {
          halo[(size_t)r] = 1;
          break;
        }
      }
    std::stable_partition(origloc.begin(), origloc.end(), [&](int r) { return halo[(size_t)r] != 0; });
  }
#pragma omp parallel for schedule(static, 64)
  for (int64_t w = 0; w < nl; w += kSortWin) {
    const int64_t e = std::min<int64_t>(nl, w + kSortWin);
    std::stable_sort(origloc.begin() + w, origloc.begin() + e,
                     [&](int x, int y) { return rp[x + 1] - rp[x] > rp[y + 1] - rp[y]; });
  }
}

// gmap[input id] = device label, for every vertex (all ranks' permutations).
scg_status build_gmap(scg_ctx *c) {
  c->gmap.assign((size_t)c->n, 0);
  if (c->mode != 2) {
    for (Shard *s : c->sh)
#pragma omp parallel for schedule(static, 65536)
      for (int64_t nu = 0; nu < s->nl; ++nu) c->gmap[(size_t)(s->rb + s->origloc[(size_t)nu])] = (int)(s->rb + nu);
    return SCG_OK;
  }
  if (c->hcomm) {  // every rank's origloc (padded to the largest shard) through the host allgather
    int64_t mx = 0;
    for (int q = 0; q < c->world; ++q) mx = std::max<int64_t>(mx, c->splits[(size_t)q + 1] - c->splits[(size_t)q]);
    std::vector<int> mine((size_t)mx, 0), all((size_t)mx * c->world);
    std::copy(c->sh[0]->origloc.begin(), c->sh[0]->origloc.end(), mine.begin());
    if (c->hc.allgather(c->hc.ctx, mine.data(), all.data(), (int64_t)sizeof(int) * mx) != 0)
      return fail(c, SCG_ECOMM, "host allgather (row labels)");
    for (int q = 0; q < c->world; ++q) {
      const int64_t a = c->splits[(size_t)q], b = c->splits[(size_t)q + 1];
      for (int64_t nu = 0; nu < b - a; ++nu) c->gmap[(size_t)(a + all[(size_t)(q * mx + nu)])] = (int)(a + nu);
    }
    return SCG_OK;
  }
#ifdef SCG_WITH_NCCL
  // every rank's origloc, broadcast by its owner (variable sizes: grouped broadcasts)
  int *buf = nullptr;
  CK(cudaMalloc(&buf, sizeof(int) * (size_t)c->n));
  Shard *me = c->sh[0];
  CK(cudaMemcpyAsync(buf + me->rb, me->origloc.data(), sizeof(int) * me->nl, cudaMemcpyHostToDevice, c->stream));
  NK(ncclGroupStart());
  for (int q = 0; q < c->world; ++q) {
    const int64_t a = c->splits[(size_t)q], b = c->splits[(size_t)q + 1];
    NK(ncclBroadcast(buf + a, buf + a, (size_t)(b - a), ncclInt32, q, c->comm, c->stream));
  }
  NK(ncclGroupEnd());
  std::vector<int> all((size_t)c->n);
  CK(cudaMemcpyAsync(all.data(), buf, sizeof(int) * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(buf);
  for (int q = 0; q < c->world; ++q) {
    const int64_t a = c->splits[(size_t)q], b = c->splits[(size_t)q + 1];
    for (int64_t nu = 0; nu < b - a; ++nu) c->gmap[(size_t)(a + all[(size_t)(a + nu)])] = (int)(a + nu);
  }
  return SCG_OK;
#else
  return fail(c, SCG_EUNSUPPORTED, "multi-process sharding needs the NCCL build");
#endif
}

// CSR checks of one shard's rows (before any device work).
scg_status validate_rows(scg_ctx *c, const int64_t *rp, const int32_t *colp, const double *valp, int64_t nl) {
  const int64_t base = rp[0];
  int bad = 0;  // 1 monotone, 2 range, 4 order, 8 finite
#pragma omp parallel for schedule(static, 4096) reduction(| : bad)
  for (int64_t r = 0; r < nl; ++r) {
    if (rp[r + 1] < rp[r]) { bad |= 1; continue; }
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int32_t cc = colp[k - base];
      if (cc < 0 || cc >= c->n) bad |= 2;
      if (k > rp[r] && cc <= colp[k - 1 - base]) bad |= 4;
      if (!std::isfinite(valp[k - base])) bad |= 8;
    }
  }
  if (bad & 1) return fail(c, SCG_EINVAL, "row_ptr not monotone");
  if (bad & 2) return fail(c, SCG_EINVAL, "column out of range");
  if (bad & 4) return fail(c, SCG_EINVAL, "columns not strictly ascending");
  if (bad & 8) return fail(c, SCG_EINVAL, "non-finite value");
  return SCG_OK;
}

// Structural symmetry of the full CSR (every stored (r, c) has a stored (c, r)): the halo
// plan derives the reader ranks of row r from row r's own columns, which is exact only for
// a symmetric pattern (L is symmetric, eqn:comb-laplacian P:97-100).
bool csr_symmetric(const int64_t *rp, const int32_t *col, int64_t n) {
  int bad = 0;
#pragma omp parallel for schedule(static, 4096) reduction(| : bad)
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rp[r]; k < rp[r + 1] && !bad; ++k) {
      const int64_t c2 = col[k];
      const int32_t *b = col + rp[c2], *e = col + rp[c2 + 1];
      const int32_t *f = std::lower_bound(b, e, (int32_t)r);
      if (f == e || *f != r) bad = 1;
    }
  return !bad;
}

// Host part of shard construction: split this shard's rows into off-diagonal
// weights w = -L_rj and the diagonal, the long-row list, the SELL-32-sigma layout of
// the short rows and the halo mask; then allocate and upload.  rp/colp/valp point at
// this shard's rows (rp[0] may be nonzero).
template <class... A>
void dbg_log(const scg_ctx *c, const char *fmt, A... a) {  // SCG_DEBUG_LOG: layout facts on stderr
  if (c->flags & SCG_DEBUG_LOG) std::fprintf(stderr, fmt, a...);
}
void dbg_split(const scg_ctx *c, const char *what) {  // SCG_DEBUG_LOG: host init stage timings
  static auto t0 = std::chrono::steady_clock::now();
  if (!(c->flags & SCG_DEBUG_LOG)) return;
  const auto t1 = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[scg]   %-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
  t0 = t1;
}

scg_status build_shard(scg_ctx *c, Shard *s, const int64_t *rp, const int32_t *colp, const double *valp,
                       int has_diagonal) {
  dbg_split(c, "shard: start");
  const int64_t nl = s->nl, rb = s->rb;
  const int R = c->R;
  const int64_t base = rp[0];
  // device row nu is input row r = origloc[nu]; its entries stay in the input (ascending
  // input column) order -- the CAC-3 chain order -- with columns relabeled by gmap.
  // Two parallel passes: count off-diagonal entries per row, then fill.
  hvec<int> &h_rp = s->h_rp;
  h_rp.resize((size_t)nl + 1);  // entry nu + 1 written by the count pass below
  h_rp[0] = 0;
#pragma omp parallel for schedule(static, 4096)
  for (int64_t nu = 0; nu < nl; ++nu) {
    const int64_t r = s->origloc[(size_t)nu];
    int cnt = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) cnt += colp[k - base] != r + rb;
    h_rp[(size_t)nu + 1] = cnt;
  }
  dbg_split(c, "shard: count");
  int64_t cnt_off = 0;
  for (int64_t nu = 0; nu < nl; ++nu) {
    cnt_off += h_rp[(size_t)nu + 1];
    if (cnt_off >= (1ll << 31)) return fail(c, SCG_EINVAL, "too many nonzeros for int32 row pointers");
    h_rp[(size_t)nu + 1] = (int)cnt_off;
  }
  hvec<int> &h_col = s->h_col;
  hvec<double> &h_w = s->h_w;
  h_col.resize((size_t)cnt_off);
  h_w.resize((size_t)cnt_off);
  hvec<double> h_diag((size_t)nl);  // every entry is written by the fill pass
  std::vector<unsigned char> h_mask;
  if (c->world > 1) h_mask.assign((size_t)nl, 0);
  long long halo = 0;
#pragma omp parallel for schedule(static, 4096) reduction(+ : halo)
  for (int64_t nu = 0; nu < nl; ++nu) {
    const int64_t r = s->origloc[(size_t)nu];
    int64_t o = h_rp[(size_t)nu];
    double dsum = 0.0;
    bool had = false;
    unsigned m = 0;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int32_t c_in = colp[k - base];
      const double lv = valp[k - base];
      if (c_in == r + rb) { h_diag[(size_t)nu] = lv; had = true; }
      else {
        const int32_t cc = c->gmap[(size_t)c_in];
        h_col[(size_t)o] = cc;
        h_w[(size_t)o] = -lv;
        dsum += -lv;
        ++o;
        if (c->world > 1 && (cc < rb || cc >= rb + nl)) {
          const int q = (int)(std::upper_bound(c->splits.begin(), c->splits.end(), (int64_t)cc) - c->splits.begin()) - 1;
          m |= 1u << q;
        }
      }
    }
    if (!has_diagonal || !had) h_diag[(size_t)nu] = has_diagonal ? 0.0 : dsum;
    if (c->world > 1) {
      h_mask[(size_t)nu] = (unsigned char)m;
      halo += m != 0;
    }
  }
  dbg_split(c, "shard: fill");
  s->halo_rows = halo;
  s->nnz_off = cnt_off;
  std::vector<int> h_long;
  for (int64_t r = 0; r < nl; ++r)
    if (h_rp[(size_t)r + 1] - h_rp[(size_t)r] > kLongRow) h_long.push_back((int)r);
  std::stable_sort(h_long.begin(), h_long.end(), [&](int x, int y) {
    return h_rp[(size_t)x + 1] - h_rp[(size_t)x] > h_rp[(size_t)y + 1] - h_rp[(size_t)y];
  });
  // rows of more than kHeavyRow entries get a block each (256 strided chains, reading R27)
  size_t nh = 0;  // (h_long is sorted longest first)
  while (nh < h_long.size() && h_rp[(size_t)h_long[nh] + 1] - h_rp[(size_t)h_long[nh]] > kHeavyRow) ++nh;
  std::vector<int> h_heavy(h_long.begin(), h_long.begin() + (long)nh);
  h_long.erase(h_long.begin(), h_long.begin() + (long)nh);
  s->nlong = (int)h_long.size();
  s->nheavy = (int)h_heavy.size();

  auto alloc = [&](void **p, size_t bytes) -> bool { return cudaMalloc(p, bytes ? bytes : 8) == cudaSuccess; };
  s->nlpad = (nl + 4 + kWin - 1) / kWin * kWin;  // >= 16 bytes of slack for the bulk copies
  const size_t nlb = sizeof(double) * (size_t)s->nlpad;
  bool ok = alloc((void **)&s->rp, sizeof(int) * (nl + 1)) && alloc((void **)&s->col, sizeof(int) * cnt_off) &&
            alloc((void **)&s->val, sizeof(double) * cnt_off) && alloc((void **)&s->wts, sizeof(double) * cnt_off) &&
            alloc((void **)&s->ldiag, nlb) && alloc((void **)&s->cdiag, nlb) && alloc((void **)&s->d, nlb) &&
            alloc((void **)&s->z, nlb) && alloc((void **)&s->y, nlb) && alloc((void **)&s->a, nlb) &&
            alloc((void **)&s->V, nlb * kSketchB) && alloc((void **)&s->ckr, sizeof(double) * kSketchB * kMaxR) &&
            alloc((void **)&s->S, nlb * R) && alloc((void **)&s->Om, nlb * R) &&
            alloc((void **)&s->sc, sizeof(DevScalars)) && alloc((void **)&s->slots, sizeof(XSlot) * SLOT_COUNT) &&
            alloc((void **)&s->dscalar, sizeof(double) * 8) &&
            alloc((void **)&s->dlog, sizeof(scg_iter_rec) * c->log_cap) &&
            alloc((void **)&s->longrows, sizeof(int) * h_long.size()) &&
            alloc((void **)&s->heavyrows, sizeof(int) * h_heavy.size()) &&
            alloc((void **)&s->mb, sizeof(Mailbox)) && alloc((void **)&s->peerG, sizeof(double *) * kMaxRanks) &&
            alloc((void **)&s->orig, sizeof(int) * (size_t)nl) && alloc((void **)&s->work, sizeof(unsigned)) &&
            alloc((void **)&s->peerMB, sizeof(Mailbox *) * kMaxRanks) &&
            alloc((void **)&s->gflag, sizeof(unsigned long long));
  if (!ok) return fail(c, SCG_ENOMEM, "device allocation");
  if (c->world > 1 && !alloc((void **)&s->mask, (size_t)nl)) return fail(c, SCG_ENOMEM, "halo mask");
  dbg_split(c, "shard: long rows+malloc");

  // grid sizes from occupancy
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_a<true, 0>, kBlock, 0);
  s->grid_rows = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_primal<false>, kBlock, 0);
  s->grid_primal = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_b, kBlock, 0);
  s->grid_b = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_combine, kBlock, 0);
  s->grid_comb = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dual_sketch<false, true>, kBlock, 0);
  s->grid_dual = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dual_sketch<false, false>, kBlock, 0);
  s->grid_dual_s = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_norm_x, kBlock, 0);
  s->grid_norm = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaFuncSetAttribute((const void *)k_lanczos_b_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BSmem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_b_tma, kBlock, sizeof(BSmem));
  s->grid_btma = (int)std::max<int64_t>(1, std::min<int64_t>((nl + kBT - 1) / kBT, (int64_t)std::max(1, occ) * c->nsm));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sketch_flush, kBlock, 0);
  s->grid_flush = grid_for(nl, std::max(1, occ) * c->nsm);
  if (!alloc((void **)&s->gpart, sizeof(double) * (size_t)s->grid_primal * R)) return fail(c, SCG_ENOMEM, "gpart");

  cudaStream_t st = c->stream;
  CK(cudaMemcpyAsync(s->rp, h_rp.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s->col, h_col.data(), sizeof(int) * cnt_off, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s->wts, h_w.data(), sizeof(double) * cnt_off, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(s->ldiag, 0, nlb, st));
  CK(cudaMemcpyAsync(s->ldiag, h_diag.data(), sizeof(double) * nl, cudaMemcpyHostToDevice, st));
  if (!h_long.empty())
    CK(cudaMemcpyAsync(s->longrows, h_long.data(), sizeof(int) * h_long.size(), cudaMemcpyHostToDevice, st));
  if (!h_heavy.empty())
    CK(cudaMemcpyAsync(s->heavyrows, h_heavy.data(), sizeof(int) * h_heavy.size(), cudaMemcpyHostToDevice, st));
  if (c->world > 1) CK(cudaMemcpyAsync(s->mask, h_mask.data(), (size_t)nl, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(s->orig, s->origloc.data(), sizeof(int) * (size_t)nl, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(s->sc, 0, sizeof(DevScalars), st));
  CK(cudaMemsetAsync(s->gflag, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(s->work, 0, sizeof(unsigned), st));
  CK(cudaMemsetAsync(s->slots, 0, sizeof(XSlot) * SLOT_COUNT, st));
  CK(cudaMemsetAsync(s->mb, 0, sizeof(Mailbox), st));
  CK(cudaMemsetAsync(s->z, 0, nlb, st));
  CK(cudaMemsetAsync(s->y, 0, nlb, st));
  CK(cudaMemsetAsync(s->S, 0, nlb * R, st));
  CK(cudaStreamSynchronize(st));  // host vectors go out of scope (the SELL layout follows in build_sell)
  dbg_split(c, "shard: grids+H2D+memsets");
  return SCG_OK;
}

// Short-row layout of the SpMV engine (needs ||L||_F for the values), built on the host
// from the device CSR copy: SELL-32-sigma.
// Values are scaled exactly as k_scale_c forms them (one IEEE division each).
scg_status build_layout(scg_ctx *c, Shard *s) {
  const int64_t nl = s->nl;
  const bool scale = (c->flags & SCG_SCALE) != 0;
  const hvec<int> &h_rp = s->h_rp, &h_col = s->h_col;
  const hvec<double> &h_w = s->h_w;
  cudaStream_t st = c->stream;
  const long long cnt_off = s->nnz_off;
  const double w0 = cnt_off > 0 ? std::fabs(h_w[0]) : 0.0;
  int nonuni = 0;
#pragma omp parallel for schedule(static, 65536) reduction(| : nonuni)
  for (int64_t k = 0; k < cnt_off; ++k) nonuni |= std::fabs(h_w[(size_t)k]) != w0;
  const bool uni = cnt_off > 0 && !nonuni;  // all |w| equal: values are encoded in the column's sign bit
  s->sell_m0 = scale ? w0 / c->nrmL : w0;  // |C_rj| = fl(|w| / ||L||_F)
  s->sell_uniform = uni;
  auto alloc = [&](void **p, size_t bytes) -> bool { return cudaMalloc(p, bytes ? bytes : 8) == cudaSuccess; };
  auto enc = [&](int64_t e) {
    int cc = h_col[(size_t)e];
    if (uni && h_w[(size_t)e] < 0) cc = (int)((unsigned)cc | 0x80000000u);
    return cc;
  };
  auto valof = [&](int64_t e) { return scale ? h_w[(size_t)e] / c->nrmL : h_w[(size_t)e]; };
  double matbytes = 0.0;
  {
    // ELL-W: every row has <= kEllMax entries (no long rows) and the padding
    // to the widest row stays below 2x the entries -- configs[1], [3] and [4]; SCG_NO_ELL opts out.
    // The SELL layout is built only when a kernel needs it (no ELL, the fused / warp-specialized
    // pass-1 options, which run the SELL engine, or a graph small enough for the resident kernel).
    int maxlen = 0;
#pragma omp parallel for schedule(static, 4096) reduction(max : maxlen)
    for (int64_t r = 0; r < nl; ++r) maxlen = std::max(maxlen, h_rp[(size_t)r + 1] - h_rp[(size_t)r]);
    int W = 0;
    for (int w : kEllWidths)
      if (W == 0 && w >= maxlen) W = w;
    const bool ell_ok = !(c->flags & SCG_NO_ELL) && s->nlong == 0 && s->nheavy == 0 && W > 0 &&
                        (double)W * (double)nl <= 2.0 * (double)cnt_off + 64.0;
    // (small graphs keep it too: the resident cluster kernel has ELL engines for widths 3 and 4 only)
    const bool need_sell = !ell_ok || (c->flags & (SCG_FUSED_PASS1 | SCG_WS_SPMV)) || c->n <= kResMaxN;
    const int padc = (int)c->n;
    s->padc = padc;
    // rows are already sorted by length within windows of kSortWin rows (relabel_perm), so a
    // slice is 32 consecutive rows; leading long rows (warp engine) are skipped lanes
    const int64_t nsl = (nl + 31) / 32;
    s->nslice = (int)nsl;
    if (need_sell) {
    hvec<int> scol;  // every slot is written by the fill pass (padding included)
    std::vector<int2> meta;
    hvec<double> sval;
    // pass 1 (parallel): slice widths and leading long lanes; slot bases by prefix sum
    std::vector<int> swid((size_t)nsl), sskip((size_t)nsl);
    int badlong = 0;
#pragma omp parallel for schedule(static, 1024) reduction(| : badlong)
    for (int64_t q = 0; q < nsl; ++q) {
      int nskip = 0, width = 0;
      for (int l = 0; l < 32; ++l) {
        const int64_t r = q * 32 + l;
        if (r >= nl) break;
        const int len = h_rp[(size_t)r + 1] - h_rp[(size_t)r];
        if (len > kLongRow) {
          if (nskip != l) badlong = 1;
          nskip = l + 1;
        } else width = std::max(width, len);
      }
      swid[(size_t)q] = width;
      sskip[(size_t)q] = nskip;
    }
    if (badlong) return fail(c, SCG_EINVAL, "SELL: long rows must lead their slice");
    meta.resize((size_t)nsl);
    size_t slots = 0;
    for (int64_t q = 0; q < nsl; ++q) {
      meta[(size_t)q] = make_int2((int)slots, swid[(size_t)q] | (sskip[(size_t)q] << 8));
      slots += (size_t)swid[(size_t)q] * 32;
      if (slots >= (size_t)INT32_MAX) return fail(c, SCG_EINVAL, "SELL layout too large");
    }
    // padding slots (rows shorter than their slice, long-row lanes) point at the dummy column n,
    // whose gathered value is -0 in every gathered vector (set_pad_zero), with a positive
    // coefficient (+m0, or the value +0): the product is -0 and fma(., ., acc) == acc exactly for
    // every acc (also +-0), so the kernels need no per-slot padding test.
    scol.resize(slots);
    if (!uni) sval.resize(slots);
    // pass 2 (parallel): fill every slot, padding included
#pragma omp parallel for schedule(static, 1024)
    for (int64_t q = 0; q < nsl; ++q) {
      const int width = swid[(size_t)q], nskip = sskip[(size_t)q];
      const size_t b0 = (size_t)meta[(size_t)q].x;
      for (int j = 0; j < width; ++j)
        for (int l = 0; l < 32; ++l) {
          const int64_t r = q * 32 + l;
          const size_t slot = b0 + (size_t)j * 32 + l;
          const int e = (l >= nskip && r < nl) ? h_rp[(size_t)r] + j : -1;
          if (e >= 0 && e < h_rp[(size_t)r + 1]) {
            scol[slot] = enc(e);
            if (!uni) sval[slot] = valof(e);
          } else {
            scol[slot] = padc;
            if (!uni) sval[slot] = 0.0;
          }
        }
    }
    s->nslice = (int)meta.size();
    if (!alloc((void **)&s->sell_meta, sizeof(int2) * meta.size()) ||
        !alloc((void **)&s->sell_col, sizeof(int) * scol.size()) ||
        (!uni && !alloc((void **)&s->sell_val, sizeof(double) * sval.size())))
      return fail(c, SCG_ENOMEM, "SELL layout");
    if (!meta.empty()) CK(cudaMemcpyAsync(s->sell_meta, meta.data(), sizeof(int2) * meta.size(), cudaMemcpyHostToDevice, st));
    if (!scol.empty()) CK(cudaMemcpyAsync(s->sell_col, scol.data(), sizeof(int) * scol.size(), cudaMemcpyHostToDevice, st));
    if (!uni && !sval.empty())
      CK(cudaMemcpyAsync(s->sell_val, sval.data(), sizeof(double) * sval.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    s->sell_slots = (double)scol.size();
    }  // need_sell
    const int64_t nsl32 = (nl + 31) / 32;
    if (ell_ok) {
      const size_t ne = (size_t)nsl32 * 32 * W;
      hvec<int> ecol(ne);
      hvec<double> eval;
      if (!uni) eval.resize(ne);
#pragma omp parallel for schedule(static, 1024)
      for (int64_t q = 0; q < nsl32; ++q) {
        const int w = W;
        const size_t base = (size_t)q * 32 * W;
        for (int j = 0; j < w; ++j)
          for (int l = 0; l < 32; ++l) {
            const int64_t r = q * 32 + l;
            // widths 2, 4: lane-major (lane l's slots contiguous, one vector load); else slot-major
            const size_t slot = base + ((w == 2 || w == 4) ? (size_t)l * w + j : (size_t)j * 32 + l);
            const int e = r < nl ? h_rp[(size_t)r] + j : -1;
            if (e >= 0 && e < h_rp[(size_t)r + 1]) {
              ecol[slot] = enc(e);
              if (!uni) eval[slot] = valof(e);
            } else {
              ecol[slot] = padc;
              if (!uni) eval[slot] = 0.0;
            }
          }
      }
      // every slot's coefficient +m0 (uniform positive weights -- unit-weight MaxCut graphs --, padding
      // included): the kernels skip the sign handling (kEllPos)
      int allpos = uni && (W == 3 || W == 4) ? 1 : 0;
      if (allpos) {
#pragma omp parallel for schedule(static, 65536) reduction(& : allpos)
        for (size_t k = 0; k < ne; ++k) allpos &= (int)(1u - ((unsigned)ecol[k] >> 31));
      }
      if (!alloc((void **)&s->ell_col, sizeof(int) * ne) || (!uni && !alloc((void **)&s->ell_val, sizeof(double) * ne)))
        return fail(c, SCG_ENOMEM, "ELL layout");
      CK(cudaMemcpyAsync(s->ell_col, ecol.data(), sizeof(int) * ne, cudaMemcpyHostToDevice, st));
      if (!uni) CK(cudaMemcpyAsync(s->ell_val, eval.data(), sizeof(double) * ne, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
      s->ellw = allpos ? (W | kEllPos) : W;
    }
    // algorithmic matrix bytes: one column index (+ value unless uniform) per stored entry --
    // independent of the layout's padding and metadata
    matbytes = (double)cnt_off * (uni ? 4.0 : 12.0);
  }
  {  // grids of the SpMV kernels
    const bool U = s->sell_uniform;
    int oa = 1, om = 1;
    if (U) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, k_lanczos_a<true, 0>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k_monitor<true, 0>, kBlock, 0);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, k_lanczos_a<false, 0>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k_monitor<false, 0>, kBlock, 0);
    }
    const int need = (int)std::max<int64_t>(std::max<int64_t>((s->nslice + 7) / 8, (s->nlong + 7) / 8), s->nheavy);
    s->grid_spmv = std::max(1, std::min(need, std::max(1, oa) * c->nsm));
    const int needA = (int)std::max<int64_t>((s->nslice + kBlockA / 32 - 1) / (kBlockA / 32), 1);
    s->grid_a = std::max(1, std::min(needA, std::max(1, oa) * c->nsm));
    s->grid_mon = std::max(1, std::min(need, std::max(1, om) * c->nsm));
    if (s->ellw) {
      int oe = 1, oem = 1, oec = 1;
      auto kA = SCG_PICK(k_lanczos_a, U, s->ellw);
      auto kM = SCG_PICK(k_monitor, U, s->ellw);
      auto kC = SCG_PICK(k_lanczos_c, U, s->ellw);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oe, kA, kBlockA, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oem, kM, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oec, kC, kBlock, 0);
      const int needE = (int)std::max<int64_t>(((nl + 31) / 32 + 7) / 8, 1);
      s->grid_ell = std::max(1, std::min(needE, std::max(1, oe) * c->nsm));
      s->grid_ell_mon = std::max(1, std::min(needE, std::max(1, oem) * c->nsm));
      s->grid_ell_c = std::max(1, std::min(needE, std::max(1, oec) * c->nsm));
    }
    dbg_log(c, "[scg] shard %d: nl=%lld long=%d uni=%d ellw=%d occ_a=%d occ_m=%d grid_a=%d grid_ell=%d\n", s->rank,
            (long long)nl, s->nlong, (int)U, s->ellw, oa, om, s->grid_a, s->grid_ell);
  }
  // dynamic slice distribution for skewed graphs (long rows present): warps that carry hub
  // rows take fewer slices.  Off for graphs without long rows (static ranges keep L1 locality).
  s->dyn = s->nlong + s->nheavy > 0;
  // warp-specialized TMA k_lanczos_a (uniform weights, static slice ranges; SCG_WS_SPMV)
  s->ws = s->sell_uniform && !s->dyn && (c->flags & SCG_WS_SPMV);
  if (s->ws) {
    const int wsb = (int)sizeof(WsSmem);
    cudaFuncSetAttribute((const void *)k_lanczos_a_ws<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, wsb);
    const int pct = std::min(100, (kWsMinBlocks * (wsb + 4096) * 100 + 233471) / 233472);
    cudaFuncSetAttribute((const void *)k_lanczos_a_ws<true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    int ow = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ow, k_lanczos_a_ws<true>, kWsThreads, wsb);
    const int need = (int)std::max<int64_t>((s->nslice + kWsCons - 1) / kWsCons, 1);
    s->grid_ws = std::max(1, std::min(need, std::max(1, ow) * c->nsm));
    dbg_log(c, "[scg] shard %d: warp-specialized k_lanczos_a, smem %d B, %d blocks/SM, grid %d\n", s->rank, wsb, ow,
            s->grid_ws);
  }
  // algorithmic bytes per launch
  const double N = (double)c->n, NL = (double)nl;
  const double mat = matbytes;
  const double gath = c->world > 1 ? NL + (double)s->halo_rows : N;  // gathered entries read once
  s->kb[KC_LANCZOS_A] = mat + 8.0 * NL + 8.0 * gath + 8.0 * NL;
  s->kb[KC_LANCZOS_B] = 32.0 * NL;
  s->kb[KC_LANCZOS_C] = mat + 8.0 * NL + 8.0 * gath + 8.0 * NL + 8.0 * NL + 16.0 * NL;
  s->kb[KC_NORM_X] = 8.0 * NL;
  s->kb[KC_MONITOR] = mat + 16.0 * NL + 8.0 * gath + 8.0 * NL;
  s->kb[KC_PRIMAL] = 24.0 * NL + 8.0 * NL * c->R;
  s->kb[KC_DUAL_SKETCH] = 60.0 * NL;  // z, y, cdiag, orig read; y, d, g written
  hvec<int>().swap(s->h_col);  // host copies no longer needed
  hvec<double>().swap(s->h_w);
  return SCG_OK;
}

// X[n] = -0 in `count` gathered vectors `pitch` doubles apart (the SpMV padding's dummy column: its
// product with the padding coefficient +m0 / value +0 is -0, an exact no-op in every fma chain).
cudaError_t set_pad_zero(scg_ctx *c, double *p, size_t pitch, size_t count) {
  const std::vector<double> nz(count, -0.0);
  cudaError_t e = cudaMemcpy2DAsync(p, sizeof(double) * pitch, nz.data(), sizeof(double), sizeof(double), count,
                                    cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e;
}

// Allocate the gathered region with `cap` W slots (+ the x slot).  Slots are always
// written before they are read; only the x slot and W slot 0 are zeroed.
scg_status alloc_G(scg_ctx *c, Shard *s, int cap) {
  const size_t bytes = sizeof(double) * (size_t)c->npad * (size_t)(1 + cap);
  double *G = nullptr;
  CK(cudaMalloc(&G, bytes));
  CK(cudaMemsetAsync(G, 0, sizeof(double) * (size_t)c->npad * 2, c->stream));
  // slack [n, npad) of every slot reads as +0, except the padding's dummy column n: -0
  CK(cudaMemset2DAsync(G + c->n, sizeof(double) * (size_t)c->npad, 0, sizeof(double) * (size_t)(c->npad - c->n),
                       (size_t)(1 + cap), c->stream));
  CK(set_pad_zero(c, G + c->n, (size_t)c->npad, (size_t)(1 + cap)));
  if (s->G) {  // keep W slot 0 (the start vector g of the next iteration)
    CK(cudaMemcpyAsync(G + c->npad, s->G + c->npad, sizeof(double) * c->npad, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(s->G);
  }
  s->G = G;
  if (c->world == 1) {
    CK(cudaMemcpyAsync(s->peerG, &s->G, sizeof(double *), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(s->peerMB, &s->mb, sizeof(Mailbox *), cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return SCG_OK;
}

// Peer tables: every shard's view of every rank's G and mailbox.
scg_status connect_peers(scg_ctx *c, const void *uid) {
  const int P = c->world;
  std::vector<double *> hG(P, nullptr);
  std::vector<Mailbox *> hM(P, nullptr);
  if (c->mode == 1 || P == 1) {
    for (Shard *s : c->sh) { hG[s->rank] = s->G; hM[s->rank] = s->mb; }
  } else {
    Shard *s = c->sh[0];
    (void)uid;  // the communicator was created at the start of init
    cudaIpcMemHandle_t hh[2];
    CK(cudaIpcGetMemHandle(&hh[0], s->G));
    CK(cudaIpcGetMemHandle(&hh[1], s->mb));
    const size_t per = sizeof(hh);
    std::vector<cudaIpcMemHandle_t> all((size_t)2 * P);
    if (c->hcomm) {
      if (c->hc.allgather(c->hc.ctx, hh, all.data(), (int64_t)per) != 0) return fail(c, SCG_ECOMM, "host allgather (IPC)");
    } else {
#ifdef SCG_WITH_NCCL
      char *dbuf = nullptr;
      CK(cudaMalloc(&dbuf, per * P));
      CK(cudaMemcpyAsync(dbuf + per * c->rank, hh, per, cudaMemcpyHostToDevice, c->stream));
      NK(ncclAllGather(dbuf + per * c->rank, dbuf, per, ncclChar, c->comm, c->stream));
      CK(cudaMemcpyAsync(all.data(), dbuf, per * P, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cudaFree(dbuf);
#else
      return fail(c, SCG_EUNSUPPORTED, "multi-process sharding needs the NCCL build or a host transport");
#endif
    }
    for (int q = 0; q < P; ++q) {
      if (q == c->rank) { hG[q] = s->G; hM[q] = s->mb; continue; }
      void *pg = nullptr, *pm = nullptr;
      CK(cudaIpcOpenMemHandle(&pg, all[(size_t)2 * q], cudaIpcMemLazyEnablePeerAccess));
      CK(cudaIpcOpenMemHandle(&pm, all[(size_t)2 * q + 1], cudaIpcMemLazyEnablePeerAccess));
      s->ipc_opened.push_back(pg);
      s->ipc_opened.push_back(pm);
      hG[q] = (double *)pg;
      hM[q] = (Mailbox *)pm;
    }
  }
  for (Shard *s : c->sh) {
    CK(cudaMemcpyAsync(s->peerG, hG.data(), sizeof(double *) * P, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(s->peerMB, hM.data(), sizeof(Mailbox *) * P, cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  if (c->mode == 2 && P > 1) {  // every rank's tables are in place before anyone stores to a peer
    if (c->hcomm) {
      if (c->hc.barrier(c->hc.ctx) != 0) return fail(c, SCG_ECOMM, "host barrier");
    } else {
#ifdef SCG_WITH_NCCL
      NK(ncclAllReduce(c->dred, c->dred, 1, ncclDouble, ncclSum, c->comm, c->stream));
      CK(cudaStreamSynchronize(c->stream));
#endif
    }
  }
  return SCG_OK;
}

scg_status balanced_splits(const int64_t *rp, int64_t n, int world, std::vector<int64_t> &sp) {
  // smallest contiguous split whose largest part cost (rows + nnz) is minimal: binary search on the cap
  sp.assign((size_t)world + 1, 0);
  auto cost = [&](int64_t a, int64_t b) { return (b - a) + (rp[b] - rp[a]); };
  int64_t lo = 1, hi = cost(0, n);
  auto feasible = [&](int64_t cap, std::vector<int64_t> *out) {
    int64_t r = 0;
    for (int p = 0; p < world; ++p) {
      if (out) (*out)[(size_t)p] = r;
      // advance r as far as the cap allows (binary search on the prefix)
      int64_t a = r, b = n;
      while (a < b) {
        const int64_t mid = a + (b - a + 1) / 2;
        if (cost(r, mid) <= cap) a = mid;
        else b = mid - 1;
      }
      r = a;
    }
    if (out) (*out)[(size_t)world] = n;
    return r >= n;
  };
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (feasible(mid, nullptr)) hi = mid;
    else lo = mid + 1;
  }
  feasible(lo, &sp);
  // no empty shard: every rank owns at least one row when n >= world
  for (int p = 1; p <= world; ++p)
    if (sp[(size_t)p] <= sp[(size_t)p - 1]) sp[(size_t)p] = std::min<int64_t>(n, sp[(size_t)p - 1] + 1);
  for (int p = world - 1; p >= 1; --p)
    if (sp[(size_t)p] >= sp[(size_t)p + 1]) sp[(size_t)p] = sp[(size_t)p + 1] - 1;
  return SCG_OK;
}

// Apply the pending rank-one sketch updates (k_sketch_flush) on every shard.
void sketch_flush(scg_ctx *c) {
  if (c->spend == 0) return;
  FlushArgs F{};
  F.nb = c->spend;
  for (int j = 0; j < c->spend; ++j) F.ome[j] = c->ome[j];
  for (Shard *s : c->sh)
    launch(c, KC_SKETCH, 8.0 * F.nb * (double)s->nl + 16.0 * c->R * (double)s->nl, k_sketch_flush,
           dim3(s->grid_flush), dim3(kBlock), s->S, (const double *)s->V, (long long)s->nlpad,
           (const double *)s->ckr, F, (int)s->nl, c->R);
  c->spend = 0;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char *sketchycgal_last_error(const scg_ctx *c) { return c ? c->err_msg.c_str() : "null context"; }

scg_status sketchycgal_selftest_division(int32_t device, int64_t n, uint64_t seed, int64_t *mismatches) {
  if (!mismatches || n < 0) return SCG_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SCG_ECUDA;
  unsigned long long *d = nullptr;
  if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return SCG_ECUDA;
  cudaMemset(d, 0, sizeof(unsigned long long));
  k_selftest_div<<<1184, 256>>>((long long)n, seed, d);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return SCG_ECUDA;
  *mismatches = (int64_t)h;
  return SCG_OK;
}

scg_status sketchycgal_selftest_xsum(int32_t device, const double *values, int64_t n, int32_t grid, int32_t block,
                                     double *sum, int32_t *range_error) {
  if (!sum || !range_error || n < 0 || (n > 0 && !values) || grid < 1 || block < 32 || block > 1024 || (block & 31))
    return SCG_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SCG_ECUDA;
  double *dv = nullptr, *dout = nullptr;
  XSlot *slot = nullptr;
  DevScalars *sc = nullptr;
  scg_status st = SCG_OK;
  if (cudaMalloc(&dv, sizeof(double) * (size_t)std::max<int64_t>(n, 1)) != cudaSuccess ||
      cudaMalloc(&dout, sizeof(double)) != cudaSuccess || cudaMalloc(&slot, sizeof(XSlot)) != cudaSuccess ||
      cudaMalloc(&sc, sizeof(DevScalars)) != cudaSuccess)
    st = SCG_ENOMEM;
  if (!st && ((n > 0 && cudaMemcpy(dv, values, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice) != cudaSuccess) ||
              cudaMemset(slot, 0, sizeof(XSlot)) != cudaSuccess || cudaMemset(sc, 0, sizeof(DevScalars)) != cudaSuccess))
    st = SCG_ECUDA;
  if (!st) {
    k_selftest_xsum<<<grid, block>>>(dv, (long long)n, slot, sc, dout);
    int e = 0;
    if (cudaMemcpy(sum, dout, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&e, &sc->err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
      st = SCG_ECUDA;
    *range_error = e & 1;
  }
  cudaFree(dv);
  cudaFree(dout);
  cudaFree(slot);
  cudaFree(sc);
  return st;
}

int64_t sketchycgal_iterations(const scg_ctx *c) { return c ? c->t : -1; }

int64_t sketchycgal_launch_count(const scg_ctx *c) { return c ? c->launches : -1; }

scg_status sketchycgal_nccl_unique_id(void *out128) {
#ifdef SCG_WITH_NCCL
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SCG_ENCCL;
  std::memcpy(out128, &id, sizeof(id));
  return SCG_OK;
#else
  (void)out128;
  return SCG_EUNSUPPORTED;
#endif
}

scg_status sketchycgal_row_splits(const int64_t *row_ptr, int64_t n, int32_t world, int64_t *splits) {
  if (!row_ptr || !splits || n < 1 || world < 1 || world > kMaxRanks || world > n) return SCG_EINVAL;
  std::vector<int64_t> sp;
  balanced_splits(row_ptr, n, world, sp);
  std::memcpy(splits, sp.data(), sizeof(int64_t) * sp.size());
  return SCG_OK;
}

int64_t sketchycgal_halo_plan(const int64_t *row_ptr, const int32_t *col_idx, int64_t row_begin, int64_t row_end,
                              const int64_t *splits, int32_t world, uint8_t *mask) {
  if (!row_ptr || !col_idx || !splits || !mask || world < 1 || world > kMaxRanks || row_end < row_begin) return -1;
  const int64_t base = row_ptr[0];
  int64_t halo = 0;
  for (int64_t r = 0; r < row_end - row_begin; ++r) {
    unsigned m = 0;
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
      const int64_t cc = col_idx[k - base];
      if (cc >= row_begin && cc < row_end) continue;
      const int q = (int)(std::upper_bound(splits, splits + world + 1, cc) - splits) - 1;
      if (q < 0 || q >= world) return -1;
      m |= 1u << q;
    }
    mask[r] = (uint8_t)m;
    halo += m != 0;
  }
  return halo;
}

void sketchycgal_destroy(scg_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (Shard *s : c->sh) free_shard(s);
  c->sh.clear();
#ifdef SCG_WITH_NCCL
  if (c->comm) ncclCommDestroy(c->comm);
#endif
  if (c->dred) cudaFree(c->dred);
  if (c->dmet) cudaFree(c->dmet);
  if (c->dchi) cudaFree(c->dchi);
  for (auto &p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  if (c->evA) cudaEventDestroy(c->evA);
  if (c->evB) cudaEventDestroy(c->evB);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

scg_status sketchycgal_maxcut_init(scg_ctx **out, const scg_csr *L, int32_t R, double alpha, double beta0,
                                   uint64_t seed, uint32_t flags, const scg_dist *dist, int32_t device,
                                   void *cuda_stream) {
  if (!out) return SCG_EINVAL;
  *out = nullptr;
  scg_ctx *c = new scg_ctx();
  auto bad = [&](scg_status st) {
    sketchycgal_destroy(c);
    return st;
  };
  if (!L || !L->row_ptr || !L->col_idx || !L->val) return bad(SCG_EINVAL);
  const bool dbg = (flags & SCG_DEBUG_LOG) != 0;
  auto t_0 = std::chrono::steady_clock::now();
  auto tick = [&](const char *what) {
    if (!dbg) return;
    const auto t_1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[scg] init %-14s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t_1 - t_0).count());
    t_0 = t_1;
  };
  const int64_t n = L->n_global;
  if (n < 2 || R < 1 || R > n || R > kMaxR || !(alpha > 0) || !(beta0 > 0) || !std::isfinite(alpha) ||
      !std::isfinite(beta0))
    return bad(SCG_EINVAL);
  if (n >= (1ll << 31)) return bad(SCG_EINVAL);
  c->n = n;
  c->R = R;
  c->flags = flags;
  c->alpha_orig = alpha;
  c->beta0 = beta0;
  c->seed = seed;
  c->device = device;
  const bool scale = (flags & SCG_SCALE) != 0;
  c->alpha = scale ? alpha / (double)n : alpha;  // X~ = X / n (= 1 for the MaxCut trace n)
  c->b = scale ? 1.0 / (double)n : 1.0;
  if (flags & SCG_INEQ) {  // K = {u <= b} (reading R32)
    c->box = true;
    c->klo = -INFINITY;
    c->khi = c->b;
  }
  c->lnN = std::log((double)n);
  c->log_cap = 1024;
  {
    // Programmatic dependent launches (triggered at the block commit), measured without
    // profiling events against no PDL: c0 +8%, c1 +23%, c2 +0%, c3 +0.5% (triggered at kernel
    // entry instead they cost c3 17%: profiles/r01/pdl_policy.txt).  SCG_NO_PDL disables.
    c->pdl = (flags & SCG_NO_PDL) == 0;
    c->fused = (flags & SCG_FUSED_PASS1) != 0;
    c->btma = (flags & SCG_TMA_B) != 0;
  }
  c->npad = (n + 4 + kWin - 1) / kWin * kWin;  // >= 16 bytes of slack for the bulk copies

  // ---- sharding mode and row splits
  int world = 1, emulate = 0, rank = 0;
  if (dist && dist->world > 1) {
    world = dist->world;
    emulate = dist->emulate;
    rank = dist->rank;
    if (world > kMaxRanks || world > n || rank < 0 || rank >= world) return bad(SCG_EINVAL);
    if (!emulate && (!dist->row_splits || (!dist->nccl_unique_id && !dist->host_comm))) return bad(SCG_EINVAL);
    if (!emulate && dist->host_comm) {
      const scg_host_comm *h = dist->host_comm;
      if (!h->allgather || !h->allreduce_sum || !h->barrier) return bad(SCG_EINVAL);
      c->hcomm = true;
      c->hc = *h;
    }
  }
  c->world = world;
  c->mode = world == 1 ? 0 : (emulate ? 1 : 2);
  c->rank = emulate ? 0 : rank;
  if (world > 1 && dist->row_splits) c->splits.assign(dist->row_splits, dist->row_splits + world + 1);
  else if (world > 1) {
    if (L->row_begin != 0 || L->row_end != n) return bad(SCG_EINVAL);
    balanced_splits(L->row_ptr, n, world, c->splits);
  } else c->splits = {0, n};
  if (c->splits.front() != 0 || c->splits.back() != n) return bad(SCG_EINVAL);
  for (int p = 0; p < world; ++p)
    if (c->splits[(size_t)p + 1] <= c->splits[(size_t)p]) return bad(SCG_EINVAL);
  if (c->mode == 2) {
    if (L->row_begin != c->splits[(size_t)rank] || L->row_end != c->splits[(size_t)rank + 1]) return bad(SCG_EINVAL);
  } else if (L->row_begin != 0 || L->row_end != n) {
    return bad(SCG_EINVAL);
  }
  if (L->row_ptr[0] != 0) return bad(SCG_EINVAL);
  {
    const int64_t nrows = L->row_end - L->row_begin;
    if (validate_rows(c, L->row_ptr, L->col_idx, L->val, nrows)) return bad(SCG_EINVAL);
    // sharded runs need a symmetric pattern (halo plan); checkable here when all rows are given
    if (c->mode == 1 && !csr_symmetric(L->row_ptr, L->col_idx, n)) return bad(SCG_EINVAL);
  }

  // ---- device setup
  if (cudaSetDevice(device) != cudaSuccess) return bad(SCG_ECUDA);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) c->stream = (cudaStream_t)cuda_stream;
  else {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // (lo = least urgent, hi = most urgent)
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi) != cudaSuccess) return bad(SCG_ECUDA);
    c->own_stream = true;
  }
  scg_status st;
  const int nshard = c->mode == 1 ? world : 1;
#ifdef SCG_WITH_NCCL
  if (c->mode == 2 && !c->hcomm) {
    ncclUniqueId id;
    std::memcpy(&id, dist->nccl_unique_id, sizeof(id));
    if (ncclCommInitRank(&c->comm, world, id, c->rank) != ncclSuccess) return bad(SCG_ENCCL);
    if (cudaMalloc(&c->dred, sizeof(double) * kMaxR * kMaxR * 4) != cudaSuccess) return bad(SCG_ENOMEM);
  }
#else
  if (c->mode == 2 && !c->hcomm) return bad(SCG_EUNSUPPORTED);
#endif
  // row relabeling within sorting windows (SELL engine), then the global id map
  for (int p = 0; p < nshard; ++p) {
    Shard *s = new Shard();
    c->sh.push_back(s);
    s->rank = c->mode == 1 ? p : c->rank;
    s->rb = c->splits[(size_t)s->rank];
    s->nl = c->splits[(size_t)s->rank + 1] - s->rb;
    const int64_t off = c->mode == 2 ? 0 : s->rb;  // index of this shard's first row in L->row_ptr
    relabel_perm(L->row_ptr + off, L->col_idx + L->row_ptr[off], s->nl, s->rb,
                 world > 1,
                 s->origloc);
  }
  tick("device+relabel");
  if ((st = build_gmap(c))) return bad(st);
  tick("gmap");
  for (Shard *s : c->sh) {
    const int64_t off = c->mode == 2 ? 0 : s->rb;
    if ((st = build_shard(c, s, L->row_ptr + off, L->col_idx + L->row_ptr[off], L->val + L->row_ptr[off],
                          L->has_diagonal)))
      return bad(st);
  }
  tick("shards");
  // Lanczos vector storage.  One rank: grown on demand.  Sharded: fixed at init (peers map it),
  // sized for q_t up to t = 1000 (+16); a later q_t above it switches every rank to the two-pass
  // form (bitwise the same iterates) in sketchycgal_step.
  c->store = (flags & SCG_REGENERATE) == 0;
  int cap = 3;
  int64_t q1000 = (int64_t)std::ceil(std::sqrt(std::sqrt(1000.0)) * c->lnN);
  q1000 = std::min<int64_t>(std::min<int64_t>(q1000, n - 1), kMaxQ - 1);
  if (world == 1 && c->store) {  // pre-size the store for q_t up to t = 1000 when it fits comfortably
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = sizeof(double) * (size_t)c->npad * (size_t)(q1000 + 2);
    if (2 * need < fr) cap = (int)std::max<int64_t>(3, q1000 + 1);
  }
  if (world > 1 && c->store) {
    const int64_t want = std::max<int64_t>(3, std::min<int64_t>(q1000 + 16, kMaxQ - 1));
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = sizeof(double) * (size_t)c->npad * (size_t)(want + 1) * nshard;
    if (need + (size_t)(2ull << 30) < fr) cap = (int)want;
    else c->store = false;  // (multi-process: every rank must decide alike, checked after connect_peers)
  }
  c->wcap = cap;
  for (Shard *s : c->sh)
    if ((st = alloc_G(c, s, cap))) return bad(st);
  if ((st = connect_peers(c, dist ? dist->nccl_unique_id : nullptr))) return bad(st);
  if (c->mode == 2) {  // agree on the storage mode (all ranks store, or none)
    std::vector<double> v{c->store ? 0.0 : 1.0};
    if ((st = host_allreduce(c, v))) return bad(st);
    if (v[0] != 0.0) c->store = false;  // some rank cannot store: all ranks run the two-pass form
  }

  // ||L||_F (exact sum over all stored entries of all ranks) and C = -L / ||L||_F
  const unsigned long long E0 = ++c->epoch;
  for (Shard *s : c->sh) {
    const int gnnz = (int)std::min<long long>(std::max<long long>(1, (s->nnz_off + kBlock - 1) / kBlock), 8 * c->nsm);
    launch(c, KC_OTHER, 0.0, k_frob, dim3(gnnz), dim3(kBlock), (const double *)s->wts, (long long)s->nnz_off,
           (const double *)s->ldiag, (int)s->nl, s->slots + SLOT_INIT, s->sc, s->dscalar, net_of(c, s, E0));
  }
  pull_all(c, FK_FROB, 1, E0, FinArgs{});
  if (cudaMemcpyAsync(&c->nrmL, c->sh[0]->dscalar, sizeof(double), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return bad(SCG_ECUDA);
  {
    int err = 0;
    cudaMemcpy(&err, &c->sh[0]->sc->err, sizeof(int), cudaMemcpyDeviceToHost);
    if (err & 2) return bad(fail(c, SCG_ECUDA, "collective timeout at init"));
  }
  c->nrmL = std::sqrt(c->nrmL);
  if (!(c->nrmL > 0) || !std::isfinite(c->nrmL)) return bad(SCG_EINVAL);
  tick("G+peers+frob");
  for (Shard *s : c->sh) {
    if ((st = build_layout(c, s))) return bad(st);
    if (cudaMemcpyAsync(s->dscalar, &c->nrmL, sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
      return bad(SCG_ECUDA);
    const int gnnz = (int)std::min<long long>(std::max<long long>(1, (s->nnz_off + kBlock - 1) / kBlock), 8 * c->nsm);
    launch(c, KC_OTHER, 0.0, k_scale_c, dim3(gnnz), dim3(kBlock), (const double *)s->wts, (long long)s->nnz_off,
           (const double *)s->ldiag, (int)s->nl, (const double *)s->dscalar, scale ? 1 : 0, s->val, s->cdiag);
    launch(c, KC_OTHER, 0.0, k_omega, dim3(8 * c->nsm), dim3(kBlock), s->Om, (int)s->nl, (long long)s->rb, (int)R, seed,
           (const int *)s->orig);
    const double beta1 = beta0 * std::sqrt(2.0);
    launch(c, KC_OTHER, 0.0, k_init_d, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z, (const double *)s->y,
           (const double *)s->cdiag, s->d, (int)s->nl, c->b, beta1, c->box ? 1 : 0, c->klo, c->khi);
  }
  // one GPU: draw each next start vector on a lower-priority side stream during the Lanczos passes
  // (SCG_FUSED_RNG keeps the draw inside k_dual_sketch, as sharded runs always do)
  // small graphs on one GPU: one cluster launch per iteration (k_resident), largest cluster that fits
  if (world == 1 && c->store && n <= kResMaxN && !(flags & SCG_NO_RESIDENT)) {
    Shard *s = c->sh[0];
    auto kR = SCG_PICK_RES(s->sell_uniform, s->ellw);
    const int smem = (int)sizeof(ResShared);
    cudaFuncSetAttribute((const void *)kR, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute((const void *)kR, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cl : {16, 8}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cl);
      cfg.blockDim = dim3(kResThreads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at{};
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = cl;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)kR, &cfg) == cudaSuccess && ncl >= 1) {
        c->res_cl = cl;
        break;
      }
    }
    cudaGetLastError();  // (a refused query leaves the multi-kernel path)
    dbg_log(c, "[scg] resident cluster kernel: %d CTAs, %d B shared memory\n", c->res_cl, smem);
  }
  c->side_rng = world == 1 && !(flags & SCG_FUSED_RNG) && c->res_cl == 0;
  if (c->side_rng) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    Shard *s = c->sh[0];
    if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->evA, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->evB, cudaEventDisableTiming) != cudaSuccess ||
        cudaMalloc(&s->gB, sizeof(double) * (size_t)c->npad) != cudaSuccess ||
        cudaMemsetAsync(s->gB, 0, sizeof(double) * (size_t)c->npad, c->stream) != cudaSuccess ||
        set_pad_zero(c, s->gB + n, (size_t)c->npad, 1) != cudaSuccess)
      return bad(fail(c, SCG_ECUDA, "side stream"));
  }
  const unsigned long long E1 = ++c->epoch;
  for (Shard *s : c->sh)
    launch(c, KC_OTHER, 0.0, k_gen_start, dim3(s->grid_rows), dim3(kBlock), c->gslot(s, 1), (int)s->nl,
           (long long)s->rb, seed, (long long)1, s->slots + SLOT_NU0, s->sc, net_of(c, s, E1), (const int *)s->orig,
           (int)FK_RHO0);
  pull_all(c, FK_RHO0, 1, E1, FinArgs{});
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) return bad(SCG_ECUDA);
  tick("layout+omega");
  for (int k = 0; k < KC_COUNT; ++k) { c->kl[k] = 0; c->ks[k] = 0; c->kms[k] = 0; c->kbytes_sum[k] = 0; }
  c->launches = 0;
  *out = c;
  return SCG_OK;
}

// Ball projection j of the points z + y / beta over all ranks: l2 (reading R34) N = ||p - b|| -> scale and
// inside flag; l1 (reading R35) the inside test and the 63-step exact bisection for the threshold.
static void ball_norm(scg_ctx *c, double beta, const IterArgs &A, int j) {
  if (c->ball == 1) {
    for (int pass = -1; pass < 63; ++pass) {
      const unsigned long long E = ++c->epoch;
      for (Shard *s : c->sh)
        launch(c, KC_OTHER, 0.0, k_l1_pass, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z,
               (const double *)s->y, beta, (int)s->nl, A, j, pass, s->slots + SLOT_BALL, s->sc, net_of(c, s, E));
      FinArgs f{};
      f.i = j;
      f.A = A;
      pull_all(c, pass < 0 ? FK_L1S : FK_L1B, 2, E, f);
    }
    return;
  }
  const unsigned long long E = ++c->epoch;
  for (Shard *s : c->sh)
    launch(c, KC_OTHER, 0.0, k_ball_sum, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z, (const double *)s->y,
           beta, (int)s->nl, A, j, s->slots + SLOT_BALL, s->sc, net_of(c, s, E));
  FinArgs f{};
  f.i = j;
  f.A = A;
  pull_all(c, FK_BALLS, 1, E, f);
}

// l2 ball: w = proj_K(z + y / beta) of the current state, d = beta (z - w) + y + cdiag, and the
// general-template gap / bound sums <y,z>, <z-w,z>, <y,w>, <z-w,z+w> (reading R33).
static void ball_state(scg_ctx *c, double beta, const IterArgs &A) {
  ball_norm(c, beta, A, 1);
  const unsigned long long E = ++c->epoch;
  for (Shard *s : c->sh)
    launch(c, KC_OTHER, 0.0, c->ball == 1 ? k_ball_d<3> : k_ball_d<2>, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z, (const double *)s->y,
           (const double *)s->cdiag, s->d, (int)s->nl, beta, A, s->slots + SLOT_BALL, s->sc, net_of(c, s, E));
  pull_all(c, FK_MY4, 4, E, FinArgs{});
}

scg_status sketchycgal_step(scg_ctx *c, int64_t T) {
  if (!c) return SCG_EINVAL;
  if (c->failed) return SCG_ESTATE;
  if (T < 0) return SCG_EINVAL;
  CK(cudaSetDevice(c->device));
  if (c->t + T > c->log_cap) {  // grow the device iteration logs
    int64_t cap = std::max<int64_t>(c->log_cap * 2, c->t + T);
    for (Shard *s : c->sh) {
      scg_iter_rec *nlg = nullptr;
      CK(cudaMalloc(&nlg, sizeof(scg_iter_rec) * cap));
      CK(cudaMemcpyAsync(nlg, s->dlog, sizeof(scg_iter_rec) * c->t, cudaMemcpyDeviceToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      cudaFree(s->dlog);
      s->dlog = nlg;
    }
    c->log_cap = cap;
  }
  const bool P1 = c->world == 1;
  for (int64_t it = 0; it < T; ++it) {
    const int64_t t = c->t + 1;
    // Alg. 4 line 5 and the q_t schedule (CAC-6), evaluated on the host
    IterArgs A;
    A.t = t;
    A.sq = std::sqrt((double)(t + 1));
    A.eta = 2.0 / (double)(t + 1);
    A.one_m_eta = 1.0 - A.eta;
    A.alpha = c->alpha;
    A.b = c->b;
    A.beta0 = c->beta0;
    A.beta_next = c->beta0 * std::sqrt((double)(t + 2));
    A.nbb = ((double)c->n * c->b) * c->b;
    A.trace_le = (c->flags & SCG_TRACE_LE) ? 1 : 0;
    A.ineq = c->box ? 1 : 0;
    A.lo = c->klo;
    A.hi = c->khi;
    A.delta = c->delta;
    int64_t q = (int64_t)std::ceil(std::sqrt(std::sqrt((double)t)) * c->lnN);
    if (q < 2) q = 2;
    if (q > c->n - 1) q = c->n - 1;
    if (c->qfix > 0) q = c->qfix;  // sketchycgal_set_lanczos_q: fixed bound (Alg. 2 input q)
    if (q > kMaxQ - 1)  // the device arrays hold kMaxQ - 1 Lanczos steps: never truncate silently
      return fail(c, SCG_EUNSUPPORTED, "Lanczos bound q_t = " + std::to_string(q) + " exceeds the device bound " +
                                           std::to_string(kMaxQ - 1) + " at t = " + std::to_string(t));
    A.q = (int)q;
    if (!P1 && c->store && c->wcap < q) c->store = false;  // sharded store (peer-mapped) too small: two-pass
    if (P1 && c->store && c->wcap < q) {  // grow the Lanczos-vector store (slot 0 = g is kept)
      const int cap = (int)std::min<int64_t>(q + 16, kMaxQ - 1);
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      const size_t need = sizeof(double) * (size_t)c->npad * (cap + 1);
      if (need + (size_t)(1ull << 30) < fr) {
        scg_status st = alloc_G(c, c->sh[0], cap);
        if (st) return st;
        c->wcap = cap;
      } else {
        c->store = false;  // does not fit: storage-optimal two-pass mode
      }
    }
    auto slot = [&](const Shard *s, int j) -> double * {  // buffer holding w_j (j >= 1; w_1 = g)
      if (j == 1) return c->gslot(s, t);
      if (c->store) return c->wslot(s, j - 1);
      return c->wslot(s, 1 + (j & 1));
    };
    if (c->res_cl && !c->box && c->store && !c->fused) {  // ---- the whole iteration in one cluster launch
      Shard *s = c->sh[0];
      const int js = c->spend;
      ResArgs P{};
      P.G = s->G;
      P.npad = c->npad;
      P.a = s->a;
      P.d = s->d;
      P.z = s->z;
      P.y = s->y;
      P.cdiag = s->cdiag;
      P.Om = s->Om;
      P.V = s->V;
      P.ldv = s->nlpad;
      P.js = js;
      P.ckr = s->ckr;
      P.sc = s->sc;
      P.log = s->dlog;
      P.A = A;
      P.R = c->R;
      P.nl = (int)s->nl;
      P.seed = c->seed;
      P.orig = s->orig;
      const double nb = (double)s->nl;
      launch_cluster(c, KC_RESIDENT, q * s->kb[KC_LANCZOS_A] + (q - 1) * s->kb[KC_LANCZOS_B] + 8.0 * nb * q +
                                         s->kb[KC_MONITOR] + s->kb[KC_PRIMAL] + s->kb[KC_DUAL_SKETCH],
                     SCG_PICK_RES(s->sell_uniform, s->ellw), c->res_cl, dim3(kResThreads), sizeof(ResShared),
                     Csr{s->rp, s->col, s->val}, rows_of(s), P);
      c->ome[js] = A.one_m_eta;
      c->vlast = js;
      if (++c->spend == kSketchB) sketch_flush(c);
      c->t = t;
      continue;
    }
    if (c->side_rng) {  // draw g_{t+1} into the buffer iteration t-1 used, once its readers are done
      Shard *s = c->sh[0];
      // SCG_SERIAL_RNG: the same draw on the main stream, between iterations (no overlap with pass 1)
      const bool ser = (c->flags & SCG_SERIAL_RNG) != 0;
      if (!ser) {
        cudaEventRecord(c->evA, c->stream);
        cudaStreamWaitEvent(c->side, c->evA, 0);
      }
      launch_on(c, ser ? c->stream : c->side, false, KC_GEN, 8.0 * (double)s->nl, k_gen_start, dim3(grid_for(s->nl, 64 * c->nsm)),
                dim3(kBlock), 0, c->gslot(s, t + 1), (int)s->nl, (long long)s->rb, c->seed, (long long)(t + 1),
                s->slots + SLOT_GEN, s->sc, net_of(c, s, 0), (const int *)s->orig, (int)FK_GEN);
      if (!ser) cudaEventRecord(c->evB, c->side);
    }
    // ---- Lanczos pass 1 (Alg. 2 lines 1-9)
    if (c->fused && c->world == 1) {  // all q steps in one persistent launch
      Shard *s = c->sh[0];
      Csr C{s->rp, s->col, s->val};
      Rows TT = rows_of(s, s->dyn);
      auto kP = s->sell_uniform ? k_lanczos_pass1<true> : k_lanczos_pass1<false>;
      const unsigned long long E = ++c->epoch;
      const unsigned long long eb = c->gphase;
      c->gphase += 2ull * (unsigned long long)q;
      launch_coop(c, KC_PASS1, q * s->kb[KC_LANCZOS_A] + (q - 1) * s->kb[KC_LANCZOS_B], kP, dim3(s->grid_a),
                  dim3(kBlockA), C, TT, (const double *)s->d, s->G, slot(s, 1), (long long)c->npad, c->store ? 1 : 0, q,
                  (int)s->nl, s->a, s->slots + SLOT_OM, s->slots + SLOT_RHO, s->sc, net_of(c, s, E), s->gflag, eb);
    } else
    {
    // SCG_INLINE_PULL (P > 1): the per-step collectives are pulled in the prologue of the kernel that
    // consumes them (omega_i in k_lanczos_b, rho_{i-1} in k_lanczos_a) instead of by k_pull launches;
    // the last omega still goes through k_pull for the tridiagonal solve
    bool inl = c->world > 1 && (c->flags & SCG_INLINE_PULL) && !c->btma && !c->hcomm;
    for (Shard *s : c->sh) inl = inl && !s->ws;
    unsigned long long Erho = 0;
    // SCG_PROFILE, one GPU: every 8th iteration the whole pass 1 (q k_lanczos_a + (q - 1) k_lanczos_b
    // launches) sits between ONE pair of events and its launches carry none, so the programmatic
    // launches overlap as they do unprofiled: the Lanczos step's time in flow (KC_PASS1_FLOW)
    EvPair pf{};
    if ((c->flags & SCG_PROFILE) != 0 && c->world == 1 && c->sh.size() == 1 && t % 8 == 0) {
      if (c->pending.size() >= 8192) ev_flush(c);
      pf.a = ev_get(c);
      pf.b = ev_get(c);
      pf.cls = KC_PASS1_FLOW;
      cudaEventRecord(pf.a, c->stream);
      c->in_flow = true;
    }
    for (int i = 1; i <= q; ++i) {
      unsigned long long E = ++c->epoch;
      const unsigned long long pa = (inl && i >= 2) ? Erho : 0ull;
      for (Shard *s : c->sh) {
        Csr C{s->rp, s->col, s->val};
        Rows TT = rows_of(s, s->dyn);
        auto kA = SCG_PICK(k_lanczos_a, s->sell_uniform, s->ellw);
        if (s->ws)
          launch_smem(c, KC_LANCZOS_A, s->kb[KC_LANCZOS_A], k_lanczos_a_ws<true>, dim3(s->grid_ws), dim3(kWsThreads),
                      sizeof(WsSmem), C, TT, (const double *)s->d, (const double *)slot(s, i), (int)s->nl,
                      (long long)s->rb, i, s->a, s->slots + SLOT_OM, s->sc, net_of(c, s, E));
        else
          launch_smem(c, KC_LANCZOS_A, s->kb[KC_LANCZOS_A], kA, dim3(s->ellw ? s->grid_ell : s->grid_a), dim3(kBlockA), 0, C, TT,
                      (const double *)s->d, (const double *)slot(s, i), (int)s->nl, (long long)s->rb, i, s->a,
                      s->slots + SLOT_OM, s->sc, net_of(c, s, E), pa);
      }
      FinArgs f{};
      f.i = i;
      if (!inl || i == q) pull_all(c, FK_OM, 1, E, f);
      if (i < q) {
        const unsigned long long Eom = E;
        E = ++c->epoch;
        for (Shard *s : c->sh) {
          const double *Xim1 = (i == 1) ? nullptr : slot(s, i - 1);
          if (c->btma)
            launch_smem(c, KC_LANCZOS_B, s->kb[KC_LANCZOS_B], k_lanczos_b_tma, dim3(s->grid_btma), dim3(kBlock),
                        sizeof(BSmem), (const double *)s->a, (const double *)slot(s, i), Xim1, slot(s, i + 1),
                        (int)s->nl, (long long)s->rb, i, s->slots + SLOT_RHO, s->sc, net_of(c, s, E));
          else
            launch(c, KC_LANCZOS_B, s->kb[KC_LANCZOS_B], k_lanczos_b, dim3(s->grid_b), dim3(kBlock),
                   (const double *)s->a, (const double *)slot(s, i), Xim1, slot(s, i + 1), (int)s->nl, (long long)s->rb,
                   i, s->slots + SLOT_RHO, s->sc, net_of(c, s, E), inl ? Eom : 0ull);
        }
        if (inl) Erho = E;
        else pull_all(c, FK_RHO, 1, E, f);
      }
    }
    if (c->in_flow) {
      Shard *s = c->sh[0];
      cudaEventRecord(pf.b, c->stream);
      c->pending.push_back(pf);
      c->in_flow = false;
      c->kl[KC_PASS1_FLOW]++;
      c->ks[KC_PASS1_FLOW]++;
      c->kbytes_sum[KC_PASS1_FLOW] += q * s->kb[KC_LANCZOS_A] + (q - 1) * s->kb[KC_LANCZOS_B];
    }
    }
    // ---- tridiagonal eigenpair (lines 11-12), replicated on every rank
    for (Shard *s : c->sh) launch(c, KC_TRIDIAG, 0.0, k_tridiag, dim3(1), dim3(32), s->sc, (int)q);
    if (c->store) {  // ---- line 13 from the stored vectors (Remark)
      const unsigned long long E = ++c->epoch;
      for (Shard *s : c->sh)
        launch(c, KC_COMBINE, 8.0 * (double)s->nl * (double)q + 8.0 * (double)s->nl, k_combine, dim3(s->grid_comb),
               dim3(kBlock), (const double *)slot(s, 1), (const double *)c->wslot(s, 0), (long long)c->npad, c->xg(s), (int)s->nl,
               (long long)s->rb, s->slots + SLOT_XX, s->sc, net_of(c, s, E));
      pull_all(c, FK_NUX, 1, E, FinArgs{});
    } else {  // ---- pass 2 (line 13): regenerate v_2..v_k
      for (int j = 1; j < q; ++j) {
        const unsigned long long E = ++c->epoch;
        for (Shard *s : c->sh) {
          Csr C{s->rp, s->col, s->val};
          Rows TT = rows_of(s);
          auto kC = SCG_PICK(k_lanczos_c, s->sell_uniform, s->ellw);
          const double *Xjm1 = (j == 1) ? nullptr : slot(s, j - 1);
          launch_smem(c, KC_LANCZOS_C, s->kb[KC_LANCZOS_C], kC, dim3(s->ellw ? s->grid_ell_c : s->grid_spmv), dim3(kBlock), 0, C, TT,
                 (const double *)s->d, (const double *)slot(s, j), Xjm1, slot(s, j + 1), c->xg(s), (int)s->nl,
                 (long long)s->rb, j, s->sc, s->slots + SLOT_BAR, net_of(c, s, E));
        }
        FinArgs f{};
        f.i = j;
        pull_all(c, FK_BAR, 0, E, f);
      }
      const unsigned long long E = ++c->epoch;
      for (Shard *s : c->sh)
        launch(c, KC_NORM_X, s->kb[KC_NORM_X], k_norm_x, dim3(s->grid_norm), dim3(kBlock),
               (const double *)slot(s, 1), c->xg(s), (int)s->nl, (long long)s->rb, s->slots + SLOT_XX, s->sc,
               net_of(c, s, E));
      pull_all(c, FK_NUX, 1, E, FinArgs{});
    }
    // ---- monitors, primal, dual, sketch (Alg. 4 lines 8-10)
    const int js = c->spend;  // ring slot of this iteration's v
    unsigned long long E = ++c->epoch;
    for (Shard *s : c->sh) {
      Csr C{s->rp, s->col, s->val};
      Rows TT = rows_of(s, s->dyn);
      auto kM = SCG_PICK(k_monitor, s->sell_uniform, s->ellw);
      launch_smem(c, KC_MONITOR, s->kb[KC_MONITOR], kM, dim3(s->ellw ? s->grid_ell_mon : s->grid_mon), dim3(kBlock), 0, C, TT, (const double *)s->d,
             (const double *)s->cdiag, (const double *)c->xg(s), c->vslot(s, js), (int)s->nl, (long long)s->rb,
             s->slots + SLOT_MON, s->sc, net_of(c, s, E));
    }
    pull_all(c, FK_MON, 3, E, FinArgs{});
    E = ++c->epoch;
    const int ks = c->ball == 2 ? 2 : c->ball == 1 ? 3 : (c->box ? 1 : 0);  // A X = b, box, l2, l1 ball
    for (Shard *s : c->sh)
      launch(c, KC_PRIMAL, s->kb[KC_PRIMAL], ks >= 2 ? k_primal<2> : (ks ? k_primal<1> : k_primal<0>),
             dim3(s->grid_primal), dim3(kBlock), (const double *)c->vslot(s, js), s->z,
             (const double *)s->y, (const double *)s->Om, (int)s->nl, c->R, A, s->gpart, s->slots + SLOT_NZ, s->sc, s->dlog, net_of(c, s, E));
    {
      FinArgs f{};
      f.R = c->R;
      f.A = A;
      pull_all(c, ks >= 2 ? FK_GK : (ks == 0 ? FK_NZZ : FK_NZ), ks == 0 ? 3 : 1, E, f);
    }
    if (ks >= 2) {  // balls (readings R34, R35): wbar_t needs the projection pass over z_{t+1} + y_t / beta_{t+1}
      ball_norm(c, A.beta_next, A, 0);
      E = ++c->epoch;
      for (Shard *s : c->sh)
        launch(c, KC_OTHER, 0.0, ks == 3 ? k_ball_nz<3> : k_ball_nz<2>, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z,
               (const double *)s->y, (int)s->nl, A, s->slots + SLOT_BALL, s->sc, s->dlog, net_of(c, s, E));
      FinArgs f{};
      f.R = 0;  // g finalized by FK_GK
      f.A = A;
      pull_all(c, FK_NZ, 1, E, f);
    }
    E = ++c->epoch;
    if (c->side_rng && !(c->flags & SCG_SERIAL_RNG)) cudaStreamWaitEvent(c->stream, c->evB, 0);  // g_{t+1} drawn
    for (Shard *s : c->sh) {
      auto kD = c->side_rng ? (ks == 1 ? k_dual_sketch<1, false> : k_dual_sketch<0, false>)
                            : (ks == 3 ? k_dual_sketch<3, true> : ks == 2 ? k_dual_sketch<2, true>
                                         : (ks ? k_dual_sketch<1, true> : k_dual_sketch<0, true>));
      launch(c, KC_DUAL_SKETCH, c->side_rng ? 40.0 * (double)s->nl : s->kb[KC_DUAL_SKETCH], kD,
             dim3(c->side_rng ? s->grid_dual_s : s->grid_dual), dim3(kBlock),
             (const double *)s->z, s->y, s->d, (const double *)s->cdiag, s->ckr, js, c->wslot(s, 0),
             (int)s->nl, (long long)s->rb, c->R, A, c->seed, s->slots + SLOT_NU0, s->sc, net_of(c, s, E),
             (const int *)s->orig);
    }
    if (ks >= 2) {
      pull_all(c, FK_RHO0, 1, E, FinArgs{});
      ball_state(c, A.beta_next, A);  // w_{t+1}, D_{t+1}'s diagonal and the gap / bound sums
    } else {
      if (ks == 0) pull_all(c, FK_RHO0Y, 3, E, FinArgs{});
      else pull_all(c, FK_RHO0M, 5, E, FinArgs{});
    }
    c->ome[js] = A.one_m_eta;
    c->vlast = js;
    if (++c->spend == kSketchB) sketch_flush(c);
    c->t = t;
  }
  if (c->failed) return SCG_ECOMM;  // a host barrier of the transport failed (pull_all)
  CK(cudaGetLastError());
  c->have_recon = false;
  return SCG_OK;
}

// Stopping rule on the iteration records: iteration t meets it when
//   bound_t / (1 + |p_t|) <= eps  and  ||z_t - b|| / (1 + ||b||) <= eps,
// p_t and z_t being the state BEFORE iteration t's update (record t-1; p_1 = 0, z_1 = 0).
// Evaluated in ORIGINAL units (reading R28): objective values scale by
// ||L||_F alpha/alpha~ and z by alpha/alpha~ when SCG_SCALE is set; b = 1, ||b|| = sqrt(n).
static bool meets_stop(const scg_ctx *c, const scg_iter_rec &r, const scg_iter_rec *prev, double eps) {
  const bool scale = (c->flags & SCG_SCALE) != 0;
  const double uz = c->alpha_orig / c->alpha, uo = scale ? c->nrmL * uz : 1.0;
  const double pt = prev ? prev->p * uo : 0.0;
  const double nb = std::sqrt((double)c->n);
  const double zres = prev ? prev->znorm * uz : nb;
  return (r.bound * uo) / (1.0 + std::fabs(pt)) <= eps && zres / (1.0 + nb) <= eps;
}

scg_status sketchycgal_run(scg_ctx *c, int64_t T_max, double eps, int64_t check_every, int64_t *t_stop) {
  if (!c || !t_stop || T_max < 0 || !(eps > 0) || check_every < 1) return SCG_EINVAL;
  *t_stop = -1;
  scg_iter_rec prev{};
  bool have_prev = false;
  if (c->t > 0) {
    scg_status st = sketchycgal_iter_log(c, c->t, 1, &prev);
    if (st) return st;
    have_prev = true;
  }
  std::vector<scg_iter_rec> rec;
  int64_t done = 0;
  while (done < T_max) {
    const int64_t k = std::min(check_every, T_max - done);
    const int64_t t0 = c->t + 1;
    scg_status st = sketchycgal_step(c, k);
    if (st) return st;
    rec.resize((size_t)k);
    if ((st = sketchycgal_iter_log(c, t0, k, rec.data()))) return st;
    for (int64_t j = 0; j < k; ++j) {
      if (meets_stop(c, rec[(size_t)j], have_prev ? &prev : nullptr, eps)) {
        *t_stop = rec[(size_t)j].t;
        return SCG_OK;
      }
      prev = rec[(size_t)j];
      have_prev = true;
    }
    done += k;
  }
  return SCG_OK;
}

scg_status sketchycgal_synchronize(scg_ctx *c) {
  if (!c) return SCG_EINVAL;
  if (c->failed) return SCG_ESTATE;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  for (Shard *s : c->sh) {
    int err = 0;
    CK(cudaMemcpy(&err, &s->sc->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err & 2) return fail(c, SCG_ECUDA, "collective timeout (a rank's contribution never arrived)");
    if (err) return fail(c, SCG_ERANGE, "exact-sum summand out of range (non-finite or >= 2^100)");
  }
  return SCG_OK;
}

scg_status sketchycgal_iter_log(scg_ctx *c, int64_t t0, int64_t count, scg_iter_rec *out) {
  if (!c || !out || t0 < 1 || count < 0 || t0 + count - 1 > c->t) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  CK(cudaMemcpy(out, c->sh[0]->dlog + (t0 - 1), sizeof(scg_iter_rec) * count, cudaMemcpyDeviceToHost));
  return SCG_OK;
}

// Copy a device row vector (device labels) of shard s into out[off + input row] (host).
// (un-permuted on the device into the shard's scratch vector a, then one copy)
static scg_status fetch_rows(scg_ctx *c, const Shard *s, const double *dsrc, double *out, int64_t off) {
  launch(c, KC_OTHER, 0.0, k_unperm, dim3(grid_for(s->nl, 8 * c->nsm)), dim3(kBlock), s->a, dsrc,
         (const int *)s->orig, (int)s->nl);
  CK(cudaMemcpyAsync(out + off, s->a, sizeof(double) * (size_t)s->nl, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return SCG_OK;
}

scg_status sketchycgal_get_state(scg_ctx *c, int32_t which, double *out) {
  if (!c || !out) return SCG_EINVAL;
  if (c->failed) return SCG_ESTATE;
  if (which == 2) sketch_flush(c);
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  const int64_t NL = c->nl_total();
  int64_t off = 0;
  for (Shard *s : c->sh) {
    const double *src = nullptr;
    bool mat = false;
    switch (which) {
      case 0: src = s->z; break;
      case 1: src = s->y; break;
      case 2: src = s->S; mat = true; break;
      case 3: src = s->Om; mat = true; break;
      case 4: src = c->vslot(s, c->vlast); break;
      case 5: src = s->d; break;
      case 6: src = s->cdiag; break;
      default: return SCG_EINVAL;
    }
    // column-major with leading dimension NL (all rows of this context), input row order
    for (int k = 0; k < (mat ? c->R : 1); ++k)
      if ((st = fetch_rows(c, s, src + (size_t)k * s->nl, out + (size_t)k * NL, off))) return st;
    off += s->nl;
  }
  return SCG_OK;
}

scg_status sketchycgal_apply_D(scg_ctx *c, const double *xh, double *yh) {
  if (!c || !xh || !yh) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  double *dx = nullptr, *dy = nullptr;
  CK(cudaMalloc(&dx, sizeof(double) * c->npad));
  CK(cudaMemset(dx, 0, sizeof(double) * c->npad));
  CK(set_pad_zero(c, dx + c->n, (size_t)c->npad, 1));
  {  // x in input order -> device labels
    std::vector<double> xr((size_t)c->n);
    for (int64_t g = 0; g < c->n; ++g) xr[(size_t)c->gmap[(size_t)g]] = xh[g];
    CK(cudaMemcpy(dx, xr.data(), sizeof(double) * c->n, cudaMemcpyHostToDevice));
  }
  int64_t off = 0;
  for (Shard *s : c->sh) {
    CK(cudaMalloc(&dy, sizeof(double) * std::max<int64_t>(1, s->nl)));
    Csr C{s->rp, s->col, s->val};
    Rows TT = rows_of(s);
    launch_smem(c, KC_OTHER, 0.0, SCG_PICK(k_apply_d, s->sell_uniform, s->ellw),
                dim3(s->ellw ? s->grid_ell : s->grid_spmv), dim3(kBlock), 0,
           C, TT, (const double *)s->d, (const double *)dx, (int)s->nl, (long long)s->rb, dy);
    CK(cudaStreamSynchronize(c->stream));
    if ((st = fetch_rows(c, s, dy, yh, off))) return st;
    cudaFree(dy);
    off += s->nl;
  }
  cudaFree(dx);
  return SCG_OK;
}

// ---------------------------------------------------------------- reconstruction (Alg. 3 / SM3)
// G = sum over all rows (all shards, all ranks) of A[:,i] B[:,j].
static scg_status gram(scg_ctx *c, double *Shard::*A, double *Shard::*B, std::vector<double> &G) {
  const int R = c->R;
  G.assign((size_t)R * R, 0.0);
  for (Shard *s : c->sh) {
    const int gx = std::max(1, std::min(grid_for(s->nl, 4 * c->nsm), 64));
    const size_t need = (size_t)R * R * gx;
    launch(c, KC_OTHER, 0.0, k_colpair, dim3(gx, R * R), dim3(kBlock), (const double *)(s->*A),
           (const double *)(s->*B), (int)s->nl, R, s->partial);
    std::vector<double> h(need);
    CK(cudaMemcpyAsync(h.data(), s->partial, sizeof(double) * need, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int p = 0; p < R * R; ++p) {
      double sum = 0.0;
      for (int b = 0; b < gx; ++b) sum += h[(size_t)p * gx + b];
      G[(size_t)p] += sum;
    }
  }
  return host_allreduce(c, G);
}

static scg_status rowmat(scg_ctx *c, double *Shard::*out, double *Shard::*A, double *Shard::*B, double beta,
                         const std::vector<double> &M) {
  for (Shard *s : c->sh) {
    CK(cudaMemcpyAsync(s->dmat, M.data(), sizeof(double) * M.size(), cudaMemcpyHostToDevice, c->stream));
    launch(c, KC_OTHER, 0.0, k_rowmat, dim3(grid_for(s->nl, 4 * c->nsm)), dim3(kBlock), s->*out,
           (const double *)(s->*A), B ? (const double *)(s->*B) : (const double *)nullptr, beta,
           (const double *)s->dmat, (int)s->nl, c->R);
  }
  return SCG_OK;
}

scg_status sketchycgal_reconstruct(scg_ctx *c, double *Uh, double *Lambda, double *errh) {
  if (!c || !Lambda) return SCG_EINVAL;
  if (c->t < 1) return fail(c, SCG_ESTATE, "reconstruct before any iteration");
  if (c->failed) return SCG_ESTATE;
  sketch_flush(c);
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  const int R = c->R;
  for (Shard *s : c->sh)
    if (!s->U) {
      const size_t nlbR = sizeof(double) * (size_t)std::max<int64_t>(1, s->nl) * R;
      CK(cudaMalloc(&s->U, nlbR));
      CK(cudaMalloc(&s->tmp1, nlbR));
      CK(cudaMalloc(&s->tmp2, nlbR));
      CK(cudaMalloc(&s->dmat, sizeof(double) * kMaxR * kMaxR));
      CK(cudaMalloc(&s->dlam, sizeof(double) * kMaxR));
      CK(cudaMalloc(&s->partial, sizeof(double) * (size_t)kMaxR * kMaxR * 64));
    }
  std::vector<double> Gss, Gos, Goo;
  if ((st = gram(c, &Shard::S, &Shard::S, Gss)) || (st = gram(c, &Shard::Om, &Shard::S, Gos)) ||
      (st = gram(c, &Shard::Om, &Shard::Om, Goo)))
    return st;
  std::vector<double> ev = sym_eigvals(Gss, R);
  double lmax = 0.0;
  for (double e : ev) lmax = std::max(lmax, e);
  const double nrmS = std::sqrt(std::max(0.0, lmax));
  double sigma = std::sqrt((double)c->n) * matlab_eps(nrmS);  // Alg. 3 line 12
  std::vector<double> Rc;
  bool ok = false;
  for (int tr = 0; tr < 40 && !ok; ++tr) {
    std::vector<double> B((size_t)R * R);
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        // B = Omega^T (S + sigma Omega), symmetrized
        const double bij = Gos[(size_t)i * R + j] + sigma * Goo[(size_t)i * R + j];
        const double bji = Gos[(size_t)j * R + i] + sigma * Goo[(size_t)j * R + i];
        B[(size_t)i * R + j] = 0.5 * (bij + bji);
      }
    ok = chol_upper(B, R, Rc);  // line 14
    if (!ok) sigma *= 2.0;
  }
  if (!ok) return fail(c, SCG_ECHOL, "Cholesky failed after 40 shift doublings");
  // Y = S_sigma Rc^{-1}   (line 15: S/L)
  if ((st = rowmat(c, &Shard::tmp1, &Shard::S, &Shard::Om, sigma, inv_upper(Rc, R)))) return st;
  // CholeskyQR2 of Y: Y = Q Rf
  std::vector<double> G1, R1, G2, R2;
  if ((st = gram(c, &Shard::tmp1, &Shard::tmp1, G1))) return st;
  if (!chol_upper(G1, R, R1)) {
    // shifted CholeskyQR: add a tiny diagonal shift
    double tr = 0;
    for (int i = 0; i < R; ++i) tr += G1[(size_t)i * R + i];
    for (int i = 0; i < R; ++i) G1[(size_t)i * R + i] += 1e-15 * tr;
    if (!chol_upper(G1, R, R1)) return fail(c, SCG_ECHOL, "CholeskyQR failed");
  }
  if ((st = rowmat(c, &Shard::tmp2, &Shard::tmp1, nullptr, 0.0, inv_upper(R1, R)))) return st;
  if ((st = gram(c, &Shard::tmp2, &Shard::tmp2, G2))) return st;
  if (!chol_upper(G2, R, R2)) return fail(c, SCG_ECHOL, "CholeskyQR2 failed");
  if ((st = rowmat(c, &Shard::tmp1, &Shard::tmp2, nullptr, 0.0, inv_upper(R2, R)))) return st;  // Q in tmp1
  std::vector<double> Rf = matmul(R2, R1, R);
  std::vector<double> Ur, sv;
  svd_jacobi(Rf, R, Ur, sv);
  if ((st = rowmat(c, &Shard::U, &Shard::tmp1, nullptr, 0.0, Ur))) return st;  // U = Q Ur
  // Lambda = max(0, Sigma^2 - sigma) (line 16); err (SM3 line 6); trace correction (Alg. 4 line 13)
  double tau = 0.0;
  CK(cudaMemcpy(&tau, &c->sh[0]->sc->tau, sizeof(double), cudaMemcpyDeviceToHost));
  const double unit = c->alpha_orig / c->alpha;
  c->lam_raw.assign(R, 0.0);
  c->lam_orig.assign(R, 0.0);
  c->lam_tc.assign(R, 0.0);
  c->err.assign(R, 0.0);
  double cum = 0.0, tot = 0.0;
  for (int k = 0; k < R; ++k) {
    c->lam_raw[k] = std::max(0.0, sv[k] * sv[k] - sigma);
    tot += c->lam_raw[k];
  }
  for (int k = 0; k < R; ++k) {
    cum += c->lam_raw[k];
    c->err[k] = (tau - cum) * unit;
    c->lam_orig[k] = c->lam_raw[k] * unit;
    // trace correction (Alg. 4 line 13) to the known trace: alpha, or tau when tr X <= alpha (R29)
    const double trace = (c->flags & SCG_TRACE_LE) ? tau : c->alpha;
    c->lam_tc[k] = (c->lam_raw[k] + (trace - tot) / R) * unit;
  }
  const std::vector<double> &lam_out = (c->flags & SCG_TRACE_CORRECT) ? c->lam_tc : c->lam_orig;
  for (int k = 0; k < R; ++k) Lambda[k] = lam_out[k];
  if (errh)
    for (int k = 0; k < R; ++k) errh[k] = c->err[k];
  CK(cudaStreamSynchronize(c->stream));
  if (Uh) {
    const int64_t NL = c->nl_total();
    int64_t off = 0;
    for (Shard *s : c->sh) {
      for (int k = 0; k < R; ++k)
        if ((st = fetch_rows(c, s, s->U + (size_t)k * s->nl, Uh + (size_t)k * NL, off))) return st;
      off += s->nl;
    }
  }
  c->have_recon = true;
  return SCG_OK;
}

// Per-column statistics of the reconstruction summed over all rows of all ranks
// (which: 0 u_k^T L u_k, 1 cut weight of sgn(U[:,k]), 2 sum (diag X^ - 1)^2).
static scg_status colstats(scg_ctx *c, int which, const double *lam_host, std::vector<double> &outk) {
  const int R = c->R;
  const int ny = which == 2 ? 1 : R;
  outk.assign(ny, 0.0);
  auto run = [&](Shard *s, const double *Ug, long long ldg, int k0, int cols) -> scg_status {
    const int gx = std::max(1, std::min(grid_for(s->nl, 4 * c->nsm), 64));
    launch(c, KC_OTHER, 0.0, k_colstats, dim3(gx, cols), dim3(kBlock), (const int *)s->rp, (const int *)s->col,
           (const double *)s->wts, (const double *)s->ldiag, (const double *)s->U, Ug, ldg, k0,
           (const double *)s->dlam, (int)s->nl, (long long)s->rb, R, which, s->partial);
    std::vector<double> h((size_t)cols * gx);
    CK(cudaMemcpyAsync(h.data(), s->partial, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int y = 0; y < cols; ++y)
      for (int b = 0; b < gx; ++b) outk[(size_t)(which == 2 ? 0 : k0 + y)] += h[(size_t)y * gx + b];
    return SCG_OK;
  };
  scg_status st;
  for (Shard *s : c->sh)
    if (lam_host) CK(cudaMemcpyAsync(s->dlam, lam_host, sizeof(double) * R, cudaMemcpyHostToDevice, c->stream));
  if (which == 2 || c->world == 1) {
    for (Shard *s : c->sh)
      if ((st = run(s, s->U, (long long)s->nl, 0, ny))) return st;
  } else {
    // sharded: gather one column at a time (halo stores + barrier) into alternating buffers --
    // the x slot for even k, W slot 1 for odd k (both free between iterations; every iteration
    // writes them before reading).  A rank may push column k+1 into a peer's buffer while that
    // peer still reads column k; it pushes column k+2 into the same buffer only after its pull of
    // collective k+1, which waits for the peer's push of k+1, enqueued after the peer's column-k
    // statistics.
    auto gbuf = [&](const Shard *s, int k) { return (k & 1) ? c->wslot(s, 1) : c->xg(s); };
    for (int k = 0; k < R; ++k) {
      const unsigned long long E = ++c->epoch;
      for (Shard *s : c->sh)
        launch(c, KC_OTHER, 0.0, k_push_col, dim3(grid_for(s->nl, 4 * c->nsm)), dim3(kBlock),
               (const double *)(s->U + (long long)k * s->nl), gbuf(s, k), (int)s->nl, (long long)s->rb,
               s->slots + SLOT_BAR, s->sc, net_of(c, s, E));
      FinArgs f{};
      f.i = -1;
      pull_all(c, FK_BAR, 0, E, f);
      for (Shard *s : c->sh)
        if ((st = run(s, gbuf(s, k), 0, k, 1))) return st;
    }
  }
  return host_allreduce(c, outk);
}

scg_status sketchycgal_maxcut_alpha_doubling(scg_ctx **out, const scg_csr *L, int32_t R, double alpha0,
                                             double beta0, uint64_t seed, uint32_t flags, int32_t device,
                                             void *cuda_stream, int64_t T, double rtol, int32_t max_rounds,
                                             double *alphas, double *objs, int32_t *rounds, int32_t *converged) {
  if (!out || !L || !(alpha0 > 0) || T < 1 || !(rtol >= 0) || max_rounds < 1 || !alphas || !objs || !rounds ||
      !converged)
    return SCG_EINVAL;
  *out = nullptr;
  *rounds = 0;
  *converged = 0;
  double alpha = alpha0;
  scg_ctx *prev = nullptr;
  for (int32_t i = 0; i < max_rounds; ++i) {
    scg_ctx *c = nullptr;
    scg_status st = sketchycgal_maxcut_init(&c, L, R, alpha, beta0, seed, flags | SCG_TRACE_LE, nullptr, device,
                                            cuda_stream);
    double ob[2] = {0.0, 0.0};
    if (!st) st = sketchycgal_step(c, T);
    if (!st) st = sketchycgal_objective(c, ob);
    if (st) {
      if (c) sketchycgal_destroy(c);
      if (prev) sketchycgal_destroy(prev);
      return st;
    }
    alphas[i] = alpha;
    objs[i] = ob[0];
    *rounds = i + 1;
    if (prev) sketchycgal_destroy(prev);
    prev = c;
    if (i > 0 && std::fabs(objs[i] - objs[i - 1]) <= rtol * std::fabs(objs[i])) {  // step 3 (reading R31)
      *converged = 1;
      break;
    }
    alpha = 2.0 * alpha;  // step 4
  }
  *out = prev;
  return SCG_OK;
}

scg_status sketchycgal_set_lanczos_q(scg_ctx *c, int32_t q) {
  if (!c || q < 0 || q > kMaxQ - 1 || q > c->n) return SCG_EINVAL;
  c->qfix = q;
  return SCG_OK;
}

scg_status sketchycgal_set_box(scg_ctx *c, double lo, double hi) {
  if (!c || c->t != 0 || std::isnan(lo) || std::isnan(hi) || !(lo <= hi) || !(hi > -INFINITY)) return SCG_EINVAL;
  const bool scale = (c->flags & SCG_SCALE) != 0;
  c->box = true;
  c->klo = scale ? lo / (double)c->n : lo;  // scaled units like b = 1/n
  c->khi = scale ? hi / (double)c->n : hi;
  const double beta1 = c->beta0 * std::sqrt(2.0);
  // D_1's diagonal with the slack w_1 = proj_K(z_1 + y_1 / beta_1), and the general-template gap /
  // bound sums over the initial state (reading R33)
  const unsigned long long E = ++c->epoch;
  for (Shard *s : c->sh)
    launch(c, KC_OTHER, 0.0, k_init_box, dim3(s->grid_rows), dim3(kBlock), (const double *)s->z, (const double *)s->y,
           (const double *)s->cdiag, s->d, (int)s->nl, beta1, c->klo, c->khi, s->slots + SLOT_INIT, s->sc,
           net_of(c, s, E));
  pull_all(c, FK_MY4, 4, E, FinArgs{});
  return sketchycgal_synchronize(c);
}

static scg_status set_ball(scg_ctx *c, double delta, int kind) {
  if (!c || c->t != 0 || !(delta >= 0.0) || !std::isfinite(delta)) return SCG_EINVAL;
  const bool scale = (c->flags & SCG_SCALE) != 0;
  c->box = true;  // general template (gap / bound with the slack, reading R33)
  c->ball = kind;
  c->delta = scale ? delta / (double)c->n : delta;  // scaled units like b = 1/n
  if (c->side_rng) {  // the ball's dual step keeps the draw of g_{t+1} in k_dual_sketch
    cudaStreamSynchronize(c->side);
    c->side_rng = false;
  }
  IterArgs A{};
  A.b = c->b;
  A.delta = c->delta;
  ball_state(c, c->beta0 * std::sqrt(2.0), A);  // D_1 with w_1 = proj_K(z_1 + y_1 / beta_1)
  return sketchycgal_synchronize(c);
}

scg_status sketchycgal_set_ball(scg_ctx *c, double delta) { return set_ball(c, delta, 2); }

scg_status sketchycgal_set_ball_l1(scg_ctx *c, double delta) { return set_ball(c, delta, 1); }

scg_status sketchycgal_objective(scg_ctx *c, double out[2]) {
  if (!c || !out) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  double p = 0.0;
  CK(cudaMemcpy(&p, &c->sh[0]->sc->p, sizeof(double), cudaMemcpyDeviceToHost));
  const bool scale = (c->flags & SCG_SCALE) != 0;
  out[0] = scale ? -p * c->nrmL * c->alpha_orig / c->alpha : -p;
  out[1] = NAN;
  if (c->have_recon) {
    const std::vector<double> &lam = (c->flags & SCG_TRACE_CORRECT) ? c->lam_tc : c->lam_orig;
    std::vector<double> q;
    if ((st = colstats(c, 0, nullptr, q))) return st;
    double s = 0.0;
    for (int k = 0; k < c->R; ++k) s += lam[k] * q[k];
    out[1] = s;
  }
  return SCG_OK;
}

scg_status sketchycgal_feasibility(scg_ctx *c, double out[3]) {
  if (!c || !out) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  // implicit: || n z~ - 1 || / (1 + sqrt n) in original units (scaled: z_orig = z * alpha_orig)
  const double unit = c->alpha_orig / c->alpha;
  std::vector<double> ssum{0.0};
  for (Shard *s : c->sh) {  // device reduction (k_sqdist + k_sum_partials), one double back per shard
    if (!c->dmet && cudaMalloc(&c->dmet, sizeof(double) * (4096 + 1)) != cudaSuccess)
      return fail(c, SCG_ENOMEM, "feasibility scratch");
    const int g = std::min(4096, std::max(1, (int)((s->nl + kBlock - 1) / kBlock)));
    k_sqdist<<<g, kBlock, 0, c->stream>>>(s->z, (int)s->nl, c->b, unit, c->dmet + 1);
    k_sum_partials<<<1, kBlock, 0, c->stream>>>(c->dmet + 1, g, c->dmet);
    double part = 0.0;
    CK(cudaMemcpyAsync(&part, c->dmet, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    ssum[0] += part;
  }
  if ((st = host_allreduce(c, ssum))) return st;
  const double nb = std::sqrt((double)c->n);
  out[0] = std::sqrt(ssum[0]) / (1.0 + nb);
  out[1] = out[2] = NAN;
  if (c->have_recon) {
    const std::vector<double> &lam = (c->flags & SCG_TRACE_CORRECT) ? c->lam_tc : c->lam_orig;
    std::vector<double> q;
    if ((st = colstats(c, 2, lam.data(), q))) return st;
    const double r = std::sqrt(q[0]);
    out[1] = r / nb;
    out[2] = r / (1.0 + nb);
  }
  return SCG_OK;
}

scg_status sketchycgal_round(scg_ctx *c, int8_t *chi, double *cut_weight) {
  if (!c || !chi || !cut_weight) return SCG_EINVAL;
  if (!c->have_recon) return fail(c, SCG_ESTATE, "round before reconstruct");
  std::vector<double> w;
  scg_status st = colstats(c, 1, nullptr, w);
  if (st) return st;
  int best = 0;
  for (int k = 1; k < c->R; ++k)
    if (w[k] > w[best]) best = k;
  // chi_0 = +1: the sign of U[0, best] lives on the rank owning global row 0
  std::vector<double> u0{0.0};
  for (Shard *s : c->sh)
    if (s->rb == 0)
      CK(cudaMemcpy(&u0[0], s->U + (size_t)best * s->nl + c->gmap[0], sizeof(double), cudaMemcpyDeviceToHost));
  if ((st = host_allreduce(c, u0))) return st;
  const int flip = u0[0] >= 0.0 ? 1 : -1;
  int64_t off = 0;
  for (Shard *s : c->sh) {  // signs on the device in input order (k_round_signs), n bytes back
    if (c->dchi_cap < s->nl) {
      if (c->dchi) cudaFree(c->dchi);
      c->dchi = nullptr;
      if (cudaMalloc(&c->dchi, (size_t)s->nl) != cudaSuccess) return fail(c, SCG_ENOMEM, "round scratch");
      c->dchi_cap = s->nl;
    }
    k_round_signs<<<grid_for(s->nl, 8 * c->nsm), kBlock, 0, c->stream>>>(s->U + (size_t)best * s->nl, s->orig,
                                                                          (int)s->nl, flip, c->dchi);
    CK(cudaMemcpyAsync(chi + off, c->dchi, (size_t)s->nl, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    off += s->nl;
  }
  *cut_weight = w[best];
  return SCG_OK;
}

int32_t sketchycgal_kernel_stats(scg_ctx *c, scg_kstat *out, int32_t max) {
  if (!c || !out) return -1;
  ev_flush(c);
  int cnt = 0;
  for (int k = 0; k < KC_COUNT && cnt < max; ++k) {
    std::memset(&out[cnt], 0, sizeof(scg_kstat));
    std::snprintf(out[cnt].name, sizeof(out[cnt].name), "%s", kKClassName[k]);
    out[cnt].launches = c->kl[k];
    out[cnt].total_ms = c->ks[k] ? c->kms[k] * (double)c->kl[k] / (double)c->ks[k] : 0.0;  // extrapolated
    out[cnt].bytes_per_launch = c->kl[k] ? c->kbytes_sum[k] / (double)c->kl[k] : 0.0;
    ++cnt;
  }
  return cnt;
}

void sketchycgal_reset_stats(scg_ctx *c) {
  if (!c) return;
  ev_flush(c);
  for (int k = 0; k < KC_COUNT; ++k) { c->kl[k] = 0; c->ks[k] = 0; c->kms[k] = 0; c->kbytes_sum[k] = 0; }
  c->launches = 0;
}

}  // extern "C"
