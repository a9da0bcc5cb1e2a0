// sketchycgal.cu -- host driver and C ABI (include/sketchycgal.h) of the B200-native
// SketchyCGAL MaxCut hot path.  See DESIGN.md for the method, the arithmetic
// contract, the data layout and the kernel rooflines.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -lineinfo
// (--fmad=false is part of the arithmetic contract: no contraction of a*b+c).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sketchycgal.h"
#include "kernels.cuh"

#ifdef SCG_WITH_NCCL
#include <nccl.h>
#endif

using namespace scg;

namespace {

enum KClass {
  KC_LANCZOS_A = 0, KC_LANCZOS_B, KC_TRIDIAG, KC_LANCZOS_C, KC_NORM_X, KC_COMBINE, KC_MONITOR, KC_PRIMAL,
  KC_DUAL_SKETCH, KC_OTHER, KC_COUNT
};
const char *kKClassName[KC_COUNT] = {"lanczos_a_spmv_dot", "lanczos_b_axpy_norm", "tridiag_mineig",
                                     "lanczos_c_spmv_regen", "norm_x", "combine_stored", "monitor_spmv",
                                     "primal_z_gpart", "dual_sketch_next_g", "other"};

struct EvPair {
  cudaEvent_t a, b;
  int cls;
};

}  // namespace

struct scg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nsm = 148;
  int64_t n = 0, nl = 0, rb = 0, npad = 0;
  long long nnz_off = 0;
  int R = 0;
  uint32_t flags = 0;
  double alpha_orig = 0, alpha = 0, beta0 = 1, b = 0, nrmL = 1, lnN = 0;
  uint64_t seed = 0;
  int rank = 0, world = 1;
  // device arrays
  int *rp = nullptr, *col = nullptr;
  double *val = nullptr, *wts = nullptr, *ldiag = nullptr, *cdiag = nullptr;
  double *d = nullptr, *z = nullptr, *y = nullptr, *a = nullptr, *v = nullptr;
  double *g = nullptr, *W0 = nullptr, *W1 = nullptr, *x = nullptr;
  double *S = nullptr, *Om = nullptr, *gpart = nullptr;
  double *U = nullptr, *tmp1 = nullptr, *tmp2 = nullptr, *dmat = nullptr, *partial = nullptr, *dlam = nullptr;
  double *dscalar = nullptr;
  DevScalars *sc = nullptr;
  XSlot *slots = nullptr;
  scg_iter_rec *dlog = nullptr;
  int64_t log_cap = 0;
  int grid_rows = 1, grid_primal = 1, grid_tiles = 1, grid_b = 1, grid_comb = 1, grid_dual = 1, grid_norm = 1;
  int *longrows = nullptr;
  int *sell_perm = nullptr, *sell_col = nullptr;
  int2 *sell_meta = nullptr;
  double *sell_val = nullptr;
  double sell_m0 = 0.0;
  int nslice = 0;
  int *sell_wstart = nullptr;
  int nwin = 0;
  size_t smem1 = 0, smem2 = 0;
  int grid_mon = 1;
  double sell_slots = 0.0;
  bool sell_uniform = false;
  int nlong = 0;
  int64_t t = 0;
  int64_t launches = 0;
  // reconstruction
  bool have_recon = false;
  std::vector<double> lam_raw, lam_orig, lam_tc, err;
  // profiling
  std::vector<EvPair> pending;
  std::vector<cudaEvent_t> evpool;
  int64_t kl[KC_COUNT] = {0};
  double kms[KC_COUNT] = {0};
  double kbytes[KC_COUNT] = {0};     // algorithmic bytes of one launch (fixed-size classes)
  double kbytes_sum[KC_COUNT] = {0}; // accumulated algorithmic bytes
  // Lanczos vector storage: slot 0 = start vector g; store mode: slot j-1 = w_j (j <= q);
  // regenerate mode: slots 1, 2 = ring of w_i
  double *Wst = nullptr;
  int wcap = 0;
  bool store = true;
  // errors
  int failed = 0;
  std::string err_msg;
};

namespace {

enum { SLOT_NU0 = 0, SLOT_OM, SLOT_RHO, SLOT_XX, SLOT_MON, SLOT_NZ, SLOT_INIT, SLOT_COUNT };

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

int grid_for(int64_t rows, int maxgrid) {
  int64_t g = (rows + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  return (int)std::min<int64_t>(g, maxgrid);
}

void ev_flush(scg_ctx *c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->stream);
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
void launch_smem(scg_ctx *c, int cls, Kern kern, dim3 grid, dim3 block, size_t smem, Args... args);

template <typename Kern, typename... Args>
void launch(scg_ctx *c, int cls, Kern kern, dim3 grid, dim3 block, Args... args) {
  launch_smem(c, cls, kern, grid, block, 0, args...);
}

template <typename Kern, typename... Args>
void launch_smem(scg_ctx *c, int cls, Kern kern, dim3 grid, dim3 block, size_t smem, Args... args) {
  const bool prof = (c->flags & SCG_PROFILE) != 0;
  EvPair p{};
  if (prof) {
    if (c->pending.size() >= 8192) ev_flush(c);
    p.a = ev_get(c);
    p.b = ev_get(c);
    p.cls = cls;
    cudaEventRecord(p.a, c->stream);
  }
  kern<<<grid, block, smem, c->stream>>>(args...);
  if (prof) {
    cudaEventRecord(p.b, c->stream);
    c->pending.push_back(p);
  }
  c->kl[cls]++;
  c->kbytes_sum[cls] += c->kbytes[cls];
  c->launches++;
}

// ---------------------------------------------------------------- small dense fp64 linear algebra (host)
// R x R matrices, row-major.
bool chol_upper(const std::vector<double> &B, int R, std::vector<double> &Rc) {  // B = Rc^T Rc
  Rc.assign((size_t)R * R, 0.0);
  for (int j = 0; j < R; ++j) {
    double s = B[(size_t)j * R + j];
    for (int k = 0; k < j; ++k) s -= Rc[(size_t)k * R + j] * Rc[(size_t)k * R + j];
    if (!(s > 0.0) || !std::isfinite(s)) return false;
    const double rjj = std::sqrt(s);
    Rc[(size_t)j * R + j] = rjj;
    for (int i = j + 1; i < R; ++i) {
      double t = B[(size_t)j * R + i];
      for (int k = 0; k < j; ++k) t -= Rc[(size_t)k * R + j] * Rc[(size_t)k * R + i];
      Rc[(size_t)j * R + i] = t / rjj;
    }
  }
  return true;
}

std::vector<double> inv_upper(const std::vector<double> &U, int R) {
  std::vector<double> X((size_t)R * R, 0.0);
  for (int j = 0; j < R; ++j) {  // solve U x = e_j
    for (int i = j; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) s -= U[(size_t)i * R + k] * X[(size_t)k * R + j];
      X[(size_t)i * R + j] = s / U[(size_t)i * R + i];
    }
  }
  return X;
}

std::vector<double> matmul(const std::vector<double> &A, const std::vector<double> &B, int R) {
  std::vector<double> C((size_t)R * R, 0.0);
  for (int i = 0; i < R; ++i)
    for (int k = 0; k < R; ++k)
      for (int j = 0; j < R; ++j) C[(size_t)i * R + j] += A[(size_t)i * R + k] * B[(size_t)k * R + j];
  return C;
}

// cyclic Jacobi eigenvalues of a symmetric matrix (values only)
std::vector<double> sym_eigvals(std::vector<double> A, int R) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = i + 1; j < R; ++j) off += A[(size_t)i * R + j] * A[(size_t)i * R + j];
    if (off == 0.0) break;
    for (int p = 0; p < R; ++p)
      for (int q = p + 1; q < R; ++q) {
        const double apq = A[(size_t)p * R + q];
        if (apq == 0.0) continue;
        const double app = A[(size_t)p * R + p], aqq = A[(size_t)q * R + q];
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = t * cs;
        for (int k = 0; k < R; ++k) {
          const double akp = A[(size_t)k * R + p], akq = A[(size_t)k * R + q];
          A[(size_t)k * R + p] = cs * akp - sn * akq;
          A[(size_t)k * R + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < R; ++k) {
          const double apk = A[(size_t)p * R + k], aqk = A[(size_t)q * R + k];
          A[(size_t)p * R + k] = cs * apk - sn * aqk;
          A[(size_t)q * R + k] = sn * apk + cs * aqk;
        }
      }
  }
  std::vector<double> ev(R);
  for (int i = 0; i < R; ++i) ev[i] = A[(size_t)i * R + i];
  return ev;
}

// One-sided Jacobi SVD of a square R x R matrix F = U diag(sv) V^T; U returned row-major.
void svd_jacobi(std::vector<double> F, int R, std::vector<double> &U, std::vector<double> &sv) {
  // work on columns of F
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < R; ++p)
      for (int q = p + 1; q < R; ++q) {
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < R; ++i) {
          const double fp = F[(size_t)i * R + p], fq = F[(size_t)i * R + q];
          alpha += fp * fp;
          beta += fq * fq;
          gamma += fp * fq;
        }
        if (gamma == 0.0 || std::fabs(gamma) <= 1e-300 + 2.2e-16 * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (int i = 0; i < R; ++i) {
          const double fp = F[(size_t)i * R + p], fq = F[(size_t)i * R + q];
          F[(size_t)i * R + p] = cs * fp - sn * fq;
          F[(size_t)i * R + q] = sn * fp + cs * fq;
        }
      }
    if (!rotated) break;
  }
  std::vector<int> idx(R);
  std::vector<double> nrm(R);
  for (int j = 0; j < R; ++j) {
    double s = 0;
    for (int i = 0; i < R; ++i) s += F[(size_t)i * R + j] * F[(size_t)i * R + j];
    nrm[j] = std::sqrt(s);
    idx[j] = j;
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
  U.assign((size_t)R * R, 0.0);
  sv.assign(R, 0.0);
  for (int jj = 0; jj < R; ++jj) {
    const int j = idx[jj];
    sv[jj] = nrm[j];
    for (int i = 0; i < R; ++i) U[(size_t)i * R + jj] = nrm[j] > 0 ? F[(size_t)i * R + j] / nrm[j] : (i == jj ? 1.0 : 0.0);
  }
}

double matlab_eps(double x) {
  if (x == 0.0) return std::ldexp(1.0, -1074);
  int e;
  std::frexp(std::fabs(x), &e);  // x = m 2^e, m in [0.5, 1)
  return std::ldexp(1.0, e - 1 - 52);
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

void sketchycgal_destroy(scg_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  void *ptrs[] = {c->rp, c->col, c->val, c->wts, c->ldiag, c->cdiag, c->d, c->z, c->y, c->a, c->v, c->Wst,
                  c->x, c->S, c->Om, c->gpart, c->U, c->tmp1, c->tmp2, c->dmat, c->partial,
                  c->dlam, c->dscalar, c->sc, c->slots, c->dlog, c->longrows,
                  c->sell_perm, c->sell_col, c->sell_meta, c->sell_val,
                  c->sell_wstart};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  for (auto &p : c->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto e : c->evpool) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

scg_status sketchycgal_maxcut_init(scg_ctx **out, const scg_csr *L, int32_t R, double alpha, double beta0,
                                   uint64_t seed, uint32_t flags, const scg_dist *dist, int32_t device,
                                   void *cuda_stream) {
  if (!out) return SCG_EINVAL;
  *out = nullptr;
  scg_ctx *c = new scg_ctx();
  auto bad = [&](scg_status st, const char *msg) {
    std::string m = msg;
    sketchycgal_destroy(c);
    (void)m;
    return st;
  };
  if (!L || !L->row_ptr || !L->col_idx || !L->val) return bad(SCG_EINVAL, "null CSR");
  const int64_t n = L->n_global;
  if (n < 2 || R < 1 || R > n || R > kMaxR || !(alpha > 0) || !(beta0 > 0) || !std::isfinite(alpha) ||
      !std::isfinite(beta0))
    return bad(SCG_EINVAL, "bad scalar argument");
  if (dist && dist->world > 1) return bad(SCG_EUNSUPPORTED, "multi-GPU: use the dist build");
  if (L->row_begin != 0 || L->row_end != n) return bad(SCG_EINVAL, "single GPU owns all rows");
  if (n >= (1ll << 31)) return bad(SCG_EINVAL, "n too large for int32 column ids");
  c->n = n;
  c->nl = L->row_end - L->row_begin;
  c->rb = L->row_begin;
  c->R = R;
  c->flags = flags;
  c->alpha_orig = alpha;
  c->beta0 = beta0;
  c->seed = seed;
  c->device = device;
  const bool scale = (flags & SCG_SCALE) != 0;
  c->alpha = scale ? 1.0 : alpha;
  c->b = scale ? 1.0 / (double)n : 1.0;
  c->lnN = std::log((double)n);

  // ---- host: validate, split L into off-diagonal weights w = -L_rj and the diagonal
  const int64_t nl = c->nl;
  const int64_t *rp = L->row_ptr;
  if (rp[0] != 0) return bad(SCG_EINVAL, "row_ptr[0] != 0");
  std::vector<int> h_rp((size_t)nl + 1);
  std::vector<int> h_col;
  std::vector<double> h_w, h_diag((size_t)nl, 0.0);
  int64_t cnt_off = 0;
  for (int64_t r = 0; r < nl; ++r) {
    if (rp[r + 1] < rp[r]) return bad(SCG_EINVAL, "row_ptr not monotone");
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int32_t cc = L->col_idx[k];
      if (cc < 0 || cc >= n) return bad(SCG_EINVAL, "column out of range");
      if (k > rp[r] && cc <= L->col_idx[k - 1]) return bad(SCG_EINVAL, "columns not strictly ascending");
      if (!std::isfinite(L->val[k])) return bad(SCG_EINVAL, "non-finite value");
      if (cc != r + c->rb) cnt_off++;
    }
  }
  if (cnt_off >= (1ll << 31)) return bad(SCG_EINVAL, "too many nonzeros for int32 row pointers");
  h_col.resize((size_t)cnt_off);
  h_w.resize((size_t)cnt_off);
  int64_t o = 0;
  for (int64_t r = 0; r < nl; ++r) {
    h_rp[(size_t)r] = (int)o;
    double dsum = 0.0;
    bool had = false;
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int32_t cc = L->col_idx[k];
      if (cc == r + c->rb) { h_diag[(size_t)r] = L->val[k]; had = true; }
      else {
        h_col[(size_t)o] = cc;
        h_w[(size_t)o] = -L->val[k];
        dsum += -L->val[k];
        ++o;
      }
    }
    if (!L->has_diagonal || !had) h_diag[(size_t)r] = L->has_diagonal ? 0.0 : dsum;
  }
  h_rp[(size_t)nl] = (int)o;
  c->nnz_off = cnt_off;
  // long rows (kernels.cuh row engine), longest first so they start early
  std::vector<int> h_long;
  for (int64_t r = 0; r < nl; ++r)
    if (h_rp[(size_t)r + 1] - h_rp[(size_t)r] > kLongRow) h_long.push_back((int)r);
  std::stable_sort(h_long.begin(), h_long.end(), [&](int x, int y) {
    return h_rp[(size_t)x + 1] - h_rp[(size_t)x] > h_rp[(size_t)y + 1] - h_rp[(size_t)y];
  });

  // ---- device setup
  cudaError_t e0 = cudaSetDevice(device);
  if (e0 != cudaSuccess) return bad(SCG_ECUDA, "cudaSetDevice");
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) c->stream = (cudaStream_t)cuda_stream;
  else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bad(SCG_ECUDA, "stream");
    c->own_stream = true;
  }
  auto alloc = [&](void **p, size_t bytes) -> bool { return cudaMalloc(p, bytes ? bytes : 8) == cudaSuccess; };
  // vectors are padded to whole kWin-row windows (the TMA engine copies whole windows)
  c->npad = (n + kWin - 1) / kWin * kWin;
  const int64_t nlpad = (nl + kWin - 1) / kWin * kWin;
  const size_t nb = sizeof(double) * (size_t)c->npad, nlb = sizeof(double) * (size_t)nlpad;
  bool ok = alloc((void **)&c->rp, sizeof(int) * (nl + 1)) && alloc((void **)&c->col, sizeof(int) * cnt_off) &&
            alloc((void **)&c->val, sizeof(double) * cnt_off) && alloc((void **)&c->wts, sizeof(double) * cnt_off) &&
            alloc((void **)&c->ldiag, nlb) && alloc((void **)&c->cdiag, nlb) && alloc((void **)&c->d, nlb) &&
            alloc((void **)&c->z, nlb) && alloc((void **)&c->y, nlb) && alloc((void **)&c->a, nlb) &&
            alloc((void **)&c->v, nlb) && alloc((void **)&c->Wst, nb * 3) && alloc((void **)&c->x, nb) &&
            alloc((void **)&c->S, nlb * R) && alloc((void **)&c->Om, nlb * R) &&
            alloc((void **)&c->sc, sizeof(DevScalars)) && alloc((void **)&c->slots, sizeof(XSlot) * SLOT_COUNT) &&
            alloc((void **)&c->dscalar, sizeof(double) * 8);
  if (!ok) return bad(SCG_ENOMEM, "device allocation");
  c->log_cap = 1024;
  if (!alloc((void **)&c->dlog, sizeof(scg_iter_rec) * c->log_cap)) return bad(SCG_ENOMEM, "log");
  c->nlong = (int)h_long.size();
  if (!alloc((void **)&c->longrows, sizeof(int) * h_long.size())) return bad(SCG_ENOMEM, "long rows");

  // grid sizes from occupancy
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_a<true>, kBlock, 0);
  c->grid_rows = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_c<true>, kBlock, 0);
  c->grid_tiles = grid_for(std::max<int64_t>(nl, (int64_t)c->nlong * 32), std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_primal, kBlock, 0);
  c->grid_primal = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lanczos_b, kBlock, 0);
  c->grid_b = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_combine, kBlock, 0);
  c->grid_comb = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dual_sketch, kBlock, 0);
  c->grid_dual = grid_for(nl, std::max(1, occ) * c->nsm);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_norm_x, kBlock, 0);
  c->grid_norm = grid_for(nl, std::max(1, occ) * c->nsm);
  c->wcap = 3;
  c->g = c->Wst;
  c->store = (flags & SCG_REGENERATE) == 0;
  if (!alloc((void **)&c->gpart, sizeof(double) * (size_t)c->grid_primal * R)) return bad(SCG_ENOMEM, "gpart");

  cudaStream_t s = c->stream;
#define CKI(call)                                                           \
  do {                                                                      \
    if ((call) != cudaSuccess) return bad(SCG_ECUDA, #call);                \
  } while (0)
  CKI(cudaMemcpyAsync(c->rp, h_rp.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, s));
  CKI(cudaMemcpyAsync(c->col, h_col.data(), sizeof(int) * cnt_off, cudaMemcpyHostToDevice, s));
  CKI(cudaMemcpyAsync(c->wts, h_w.data(), sizeof(double) * cnt_off, cudaMemcpyHostToDevice, s));
  CKI(cudaMemcpyAsync(c->ldiag, h_diag.data(), nlb, cudaMemcpyHostToDevice, s));
  if (!h_long.empty())
    CKI(cudaMemcpyAsync(c->longrows, h_long.data(), sizeof(int) * h_long.size(), cudaMemcpyHostToDevice, s));
  CKI(cudaMemsetAsync(c->sc, 0, sizeof(DevScalars), s));
  CKI(cudaMemsetAsync(c->slots, 0, sizeof(XSlot) * SLOT_COUNT, s));
  CKI(cudaMemsetAsync(c->z, 0, nlb, s));
  CKI(cudaMemsetAsync(c->y, 0, nlb, s));
  CKI(cudaMemsetAsync(c->S, 0, nlb * R, s));
  CKI(cudaMemsetAsync(c->x, 0, nb, s));
  CKI(cudaMemsetAsync(c->Wst, 0, nb * 3, s));
  // ||L||_F (exact sum over all stored entries) and C = -L / ||L||_F
  const int gnnz = (int)std::min<long long>(std::max<long long>(1, (cnt_off + kBlock - 1) / kBlock), 8 * c->nsm);
  launch(c, KC_OTHER, k_frob, dim3(gnnz), dim3(kBlock), (const double *)c->wts, (long long)cnt_off,
         (const double *)c->ldiag, (int)nl, c->slots + SLOT_INIT, c->sc, c->dscalar);
  CKI(cudaMemcpyAsync(&c->nrmL, c->dscalar, sizeof(double), cudaMemcpyDeviceToHost, s));
  CKI(cudaStreamSynchronize(s));
  c->nrmL = std::sqrt(c->nrmL);
  if (!(c->nrmL > 0) || !std::isfinite(c->nrmL)) return bad(SCG_EINVAL, "||L||_F must be positive and finite");
  CKI(cudaMemcpyAsync(c->dscalar, &c->nrmL, sizeof(double), cudaMemcpyHostToDevice, s));
  {  // SELL-32-sigma layout of the short rows (kernels.cuh row engine)
    const int kSigma = SCG_TMA ? kWin : 256;  // sorting window of SELL-32-sigma (= TMA staging window)
    std::vector<int> wstart;
    bool uni = cnt_off > 0;
    const double w0 = cnt_off > 0 ? std::fabs(h_w[0]) : 0.0;
    for (int64_t k = 0; k < cnt_off && uni; ++k) uni = std::fabs(h_w[(size_t)k]) == w0;
    c->sell_m0 = scale ? w0 / c->nrmL : w0;  // |C_rj| = fl(|w| / ||L||_F)
    std::vector<int> perm, scol, win;
    std::vector<int2> meta;
    std::vector<double> sval;
    for (int64_t w = 0; w < nl; w += kSigma) {
      wstart.push_back((int)meta.size());
      win.clear();
      for (int64_t r = w; r < std::min<int64_t>(nl, w + kSigma); ++r)
        if (h_rp[(size_t)r + 1] - h_rp[(size_t)r] <= kLongRow) win.push_back((int)r);
      std::stable_sort(win.begin(), win.end(), [&](int x, int y) {
        return h_rp[(size_t)x + 1] - h_rp[(size_t)x] > h_rp[(size_t)y + 1] - h_rp[(size_t)y];
      });
      for (size_t s0 = 0; s0 < win.size(); s0 += 32) {
        const int cnt = (int)std::min<size_t>(32, win.size() - s0);
        const int width = h_rp[(size_t)win[s0] + 1] - h_rp[(size_t)win[s0]];
        meta.push_back(make_int2((int)scol.size(), width));
        for (int j = 0; j < width; ++j)
          for (int l = 0; l < 32; ++l) {
            int cc = -1;
            double vv = 0.0;
            if (l < cnt) {
              const int r = win[s0 + l];
              const int e = h_rp[(size_t)r] + j;
              if (e < h_rp[(size_t)r + 1]) {
                cc = h_col[(size_t)e];
                const double wv = h_w[(size_t)e];
                if (uni && wv < 0) cc = (int)((unsigned)cc | 0x80000000u);
                vv = scale ? wv / c->nrmL : wv;  // = C_rj exactly as k_scale_c forms it
              }
            }
            scol.push_back(cc);
            if (!uni) sval.push_back(vv);
          }
        for (int l = 0; l < 32; ++l) perm.push_back(l < cnt ? win[s0 + l] : -1);
      }
      if (scol.size() >= (size_t)INT32_MAX) return bad(SCG_EINVAL, "SELL layout too large");
    }
    c->nslice = (int)meta.size();
    wstart.push_back((int)meta.size());
    c->nwin = (int)wstart.size() - 1;
    if (!alloc((void **)&c->sell_wstart, sizeof(int) * wstart.size())) return bad(SCG_ENOMEM, "SELL windows");
    CKI(cudaMemcpyAsync(c->sell_wstart, wstart.data(), sizeof(int) * wstart.size(), cudaMemcpyHostToDevice, s));
    if (!alloc((void **)&c->sell_perm, sizeof(int) * perm.size()) ||
        !alloc((void **)&c->sell_meta, sizeof(int2) * meta.size()) ||
        !alloc((void **)&c->sell_col, sizeof(int) * scol.size()) ||
        (!uni && !alloc((void **)&c->sell_val, sizeof(double) * sval.size())))
      return bad(SCG_ENOMEM, "SELL layout");
    CKI(cudaMemcpyAsync(c->sell_perm, perm.data(), sizeof(int) * perm.size(), cudaMemcpyHostToDevice, s));
    CKI(cudaMemcpyAsync(c->sell_meta, meta.data(), sizeof(int2) * meta.size(), cudaMemcpyHostToDevice, s));
    CKI(cudaMemcpyAsync(c->sell_col, scol.data(), sizeof(int) * scol.size(), cudaMemcpyHostToDevice, s));
    if (!uni) CKI(cudaMemcpyAsync(c->sell_val, sval.data(), sizeof(double) * sval.size(), cudaMemcpyHostToDevice, s));
    CKI(cudaStreamSynchronize(s));  // host vectors go out of scope
    c->sell_slots = (double)scol.size();
    c->sell_uniform = uni;
  }
  {  // dynamic shared memory and grids of the TMA-staged SpMV kernels
    const bool U = c->sell_uniform;
    c->smem1 = !SCG_TMA ? 0 : (U ? sizeof(TmaSmem<1, true>) : sizeof(TmaSmem<1, false>));
    c->smem2 = !SCG_TMA ? 0 : (U ? sizeof(TmaSmem<2, true>) : sizeof(TmaSmem<2, false>));
    auto setsm = [&](const void *k, size_t b) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b); };
    if (U) {
      setsm((const void *)k_lanczos_a<true>, c->smem1);
      setsm((const void *)k_lanczos_c<true>, c->smem1);
      setsm((const void *)k_apply_d<true>, c->smem1);
      setsm((const void *)k_monitor<true>, c->smem2);
    } else {
      setsm((const void *)k_lanczos_a<false>, c->smem1);
      setsm((const void *)k_lanczos_c<false>, c->smem1);
      setsm((const void *)k_apply_d<false>, c->smem1);
      setsm((const void *)k_monitor<false>, c->smem2);
    }
    int oa = 1, om = 1;
    if (U) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, k_lanczos_a<true>, kBlock, c->smem1);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k_monitor<true>, kBlock, c->smem2);
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, k_lanczos_a<false>, kBlock, c->smem1);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k_monitor<false>, kBlock, c->smem2);
    }
    const int need = SCG_TMA ? std::max(c->nwin, (c->nlong + 7) / 8)
                             : (int)std::max<int64_t>((c->nslice + 7) / 8, (c->nlong + 7) / 8);
    c->grid_tiles = std::max(1, std::min(need, std::max(1, oa) * c->nsm));
    c->grid_mon = std::max(1, std::min(need, std::max(1, om) * c->nsm));
  }
  launch(c, KC_OTHER, k_scale_c, dim3(gnnz), dim3(kBlock), (const double *)c->wts, (long long)cnt_off,
         (const double *)c->ldiag, (int)nl, (const double *)c->dscalar, scale ? 1 : 0, c->val, c->cdiag);
  launch(c, KC_OTHER, k_omega, dim3(8 * c->nsm), dim3(kBlock), c->Om, (int)nl, (long long)c->rb, (int)R, seed);
  const double beta1 = beta0 * std::sqrt(2.0);
  launch(c, KC_OTHER, k_init_d, dim3(c->grid_rows), dim3(kBlock), (const double *)c->z, (const double *)c->y,
         (const double *)c->cdiag, c->d, (int)nl, c->b, beta1);
  launch(c, KC_OTHER, k_gen_start, dim3(c->grid_rows), dim3(kBlock), c->g, (int)nl, (long long)c->rb, seed,
         (long long)1, c->slots + SLOT_NU0, c->sc, 1);
  CKI(cudaGetLastError());
  CKI(cudaStreamSynchronize(s));
#undef CKI
  // algorithmic bytes per launch
  const double N = (double)n, NL = (double)nl, NNZ = (double)cnt_off;
  // SpMV matrix stream: SELL slots (4 B col [+ 8 B val]) + perm 4 B/row + slice meta + long-row CSR
  const double mat = c->sell_slots * (c->sell_uniform ? 4.0 : 12.0) + 4.0 * NL + 8.0 * c->nslice;
  c->kbytes[KC_LANCZOS_A] = mat + 8.0 * NL + 8.0 * N + 8.0 * NL;
  c->kbytes[KC_LANCZOS_B] = 32.0 * NL;
  c->kbytes[KC_TRIDIAG] = 0.0;
  c->kbytes[KC_LANCZOS_C] = mat + 8.0 * NL + 8.0 * N + 8.0 * NL + 8.0 * NL + 16.0 * NL;
  c->kbytes[KC_NORM_X] = 8.0 * NL;
  c->kbytes[KC_COMBINE] = 0.0;  // 8 nl k + 8 nl per launch, accumulated in step()
  c->kbytes[KC_MONITOR] = mat + 16.0 * NL + 8.0 * N + 8.0 * NL;
  c->kbytes[KC_PRIMAL] = 24.0 * NL + 8.0 * NL * R;
  c->kbytes[KC_DUAL_SKETCH] = 56.0 * NL + 16.0 * NL * R;
  for (int k = 0; k < KC_COUNT; ++k) { c->kl[k] = 0; c->kms[k] = 0; c->kbytes_sum[k] = 0; }
  c->launches = 0;
  *out = c;
  return SCG_OK;
}

scg_status sketchycgal_step(scg_ctx *c, int64_t T) {
  if (!c) return SCG_EINVAL;
  if (c->failed) return SCG_ESTATE;
  if (T < 0) return SCG_EINVAL;
  CK(cudaSetDevice(c->device));
  if (c->t + T > c->log_cap) {  // grow the device iteration log
    int64_t cap = std::max<int64_t>(c->log_cap * 2, c->t + T);
    scg_iter_rec *nl = nullptr;
    CK(cudaMalloc(&nl, sizeof(scg_iter_rec) * cap));
    CK(cudaMemcpyAsync(nl, c->dlog, sizeof(scg_iter_rec) * c->t, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(c->dlog);
    c->dlog = nl;
    c->log_cap = cap;
  }

  const int nl = (int)c->nl;
  const long long rb = c->rb;
  Csr C{c->rp, c->col, c->val};
  Rows TT{c->longrows, c->nlong, c->sell_perm, c->sell_meta, c->sell_col, c->sell_val, c->sell_m0, c->nslice,
          c->sell_wstart, c->nwin};
  const int GT = c->grid_tiles;
  const long long ldw = (long long)c->npad;
  const bool U = c->sell_uniform;
  auto kA = U ? k_lanczos_a<true> : k_lanczos_a<false>;
  auto kC = U ? k_lanczos_c<true> : k_lanczos_c<false>;
  auto kM = U ? k_monitor<true> : k_monitor<false>;
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
    int64_t q = (int64_t)std::ceil(std::sqrt(std::sqrt((double)t)) * c->lnN);
    if (q < 2) q = 2;
    if (q > c->n - 1) q = c->n - 1;
    if (q > kMaxQ - 1) q = kMaxQ - 1;
    A.q = (int)q;
    if (c->store && c->wcap < q) {  // grow the Lanczos-vector store (slot 0 = g is kept)
      const int cap = (int)std::min<int64_t>(q + 16, kMaxQ);
      double *nw = nullptr;
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      const size_t need = sizeof(double) * (size_t)c->npad * cap;
      if (need + (size_t)(1ull << 30) < fr && cudaMalloc(&nw, need) == cudaSuccess) {
        CK(cudaMemcpyAsync(nw, c->Wst, sizeof(double) * c->npad, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        cudaFree(c->Wst);
        c->Wst = nw;
        c->g = nw;
        c->wcap = cap;
      } else {
        c->store = false;  // does not fit: storage-optimal two-pass mode
      }
    }
    auto slot = [&](int j) -> double * {  // buffer holding w_j (j >= 1; w_1 = g)
      if (c->store) return c->Wst + (long long)(j - 1) * ldw;
      return j == 1 ? c->Wst : c->Wst + (long long)(1 + (j & 1)) * ldw;
    };
    // ---- Lanczos pass 1 (Alg. 2 lines 1-9)
    for (int i = 1; i <= q; ++i) {
      const double *Xi = slot(i);
      launch_smem(c, KC_LANCZOS_A, kA, dim3(GT), dim3(kBlock), c->smem1, C, TT, (const double *)c->d, Xi, nl, rb, i, c->a,
             c->slots + SLOT_OM, c->sc, 1);
      if (i < q) {
        const double *Xim1 = (i == 1) ? nullptr : slot(i - 1);
        launch(c, KC_LANCZOS_B, k_lanczos_b, dim3(c->grid_b), dim3(kBlock), (const double *)c->a, Xi, Xim1, slot(i + 1),
               nl, rb, i, c->slots + SLOT_RHO, c->sc, 1);
      }
    }
    // ---- tridiagonal eigenpair (lines 11-12)
    launch(c, KC_TRIDIAG, k_tridiag, dim3(1), dim3(32), c->sc, (int)q);
    if (c->store) {  // ---- line 13 from the stored vectors (Remark)
      c->kbytes[KC_COMBINE] = 8.0 * (double)c->nl * (double)q + 8.0 * (double)c->nl;
      launch(c, KC_COMBINE, k_combine, dim3(c->grid_comb), dim3(kBlock), (const double *)c->Wst, ldw, c->x, nl, rb,
             c->slots + SLOT_XX, c->sc, 1);
    } else {  // ---- pass 2 (line 13): regenerate v_2..v_k
      for (int j = 1; j < q; ++j) {
        const double *Xj = slot(j);
        const double *Xjm1 = (j == 1) ? nullptr : slot(j - 1);
        launch_smem(c, KC_LANCZOS_C, kC, dim3(GT), dim3(kBlock), c->smem1, C, TT, (const double *)c->d, Xj, Xjm1,
               slot(j + 1), c->x, nl, rb, j, (const DevScalars *)c->sc);
      }
      launch(c, KC_NORM_X, k_norm_x, dim3(c->grid_norm), dim3(kBlock), (const double *)c->g, c->x, nl, rb,
             c->slots + SLOT_XX, c->sc, 1);
    }
    // ---- monitors, primal, dual, sketch (Alg. 4 lines 8-10)
    launch_smem(c, KC_MONITOR, kM, dim3(c->grid_mon), dim3(kBlock), c->smem2, C, TT, (const double *)c->d, (const double *)c->cdiag,
           (const double *)c->x, c->v, nl, rb, c->slots + SLOT_MON, c->sc, 1);
    launch(c, KC_PRIMAL, k_primal, dim3(c->grid_primal), dim3(kBlock), (const double *)c->v, c->z,
           (const double *)c->Om, nl, c->R, A, c->gpart, c->slots + SLOT_NZ, c->sc, c->dlog, 1);
    launch(c, KC_DUAL_SKETCH, k_dual_sketch, dim3(c->grid_dual), dim3(kBlock), (const double *)c->z, c->y, c->d,
           (const double *)c->cdiag, (const double *)c->v, c->S, c->g, nl, rb, c->R, A, c->seed,
           c->slots + SLOT_NU0, c->sc, 1);
    c->t = t;
  }
  CK(cudaGetLastError());
  c->have_recon = false;
  return SCG_OK;
}

scg_status sketchycgal_synchronize(scg_ctx *c) {
  if (!c) return SCG_EINVAL;
  if (c->failed) return SCG_ESTATE;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  int err = 0;
  CK(cudaMemcpy(&err, &c->sc->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) return fail(c, SCG_ERANGE, "exact-sum summand out of range (non-finite or >= 2^100)");
  return SCG_OK;
}

scg_status sketchycgal_iter_log(scg_ctx *c, int64_t t0, int64_t count, scg_iter_rec *out) {
  if (!c || !out || t0 < 1 || count < 0 || t0 + count - 1 > c->t) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  CK(cudaMemcpy(out, c->dlog + (t0 - 1), sizeof(scg_iter_rec) * count, cudaMemcpyDeviceToHost));
  return SCG_OK;
}

scg_status sketchycgal_get_state(scg_ctx *c, int32_t which, double *out) {
  if (!c || !out) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  const size_t nlb = sizeof(double) * (size_t)c->nl;
  const double *src = nullptr;
  size_t bytes = nlb;
  switch (which) {
    case 0: src = c->z; break;
    case 1: src = c->y; break;
    case 2: src = c->S; bytes = nlb * c->R; break;
    case 3: src = c->Om; bytes = nlb * c->R; break;
    case 4: src = c->v; break;
    case 5: src = c->d; break;
    case 6: src = c->cdiag; break;
    default: return SCG_EINVAL;
  }
  CK(cudaMemcpy(out, src, bytes, cudaMemcpyDeviceToHost));
  return SCG_OK;
}

scg_status sketchycgal_apply_D(scg_ctx *c, const double *xh, double *yh) {
  if (!c || !xh || !yh) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  // use tmp buffers: x into c->x is not allowed (state); allocate scratch
  double *dx = nullptr, *dy = nullptr;
  CK(cudaMalloc(&dx, sizeof(double) * c->npad));
  CK(cudaMalloc(&dy, sizeof(double) * c->nl));
  CK(cudaMemcpy(dx, xh, sizeof(double) * c->n, cudaMemcpyHostToDevice));
  Csr C{c->rp, c->col, c->val};
  Rows TT{c->longrows, c->nlong, c->sell_perm, c->sell_meta, c->sell_col, c->sell_val, c->sell_m0, c->nslice,
          c->sell_wstart, c->nwin};
  launch_smem(c, KC_OTHER, c->sell_uniform ? k_apply_d<true> : k_apply_d<false>, dim3(c->grid_tiles), dim3(kBlock),
              c->smem1, C, TT, (const double *)c->d, (const double *)dx,
         (int)c->nl, (long long)c->rb, dy);
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(yh, dy, sizeof(double) * c->nl, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dy);
  return SCG_OK;
}

// ---------------------------------------------------------------- reconstruction (Alg. 3 / SM3)
static scg_status gram(scg_ctx *c, const double *A, const double *B, std::vector<double> &G) {
  const int R = c->R;
  const int gx = std::max(1, std::min(grid_for(c->nl, 4 * c->nsm), 64));
  const size_t need = (size_t)R * R * gx;
  if (!c->partial) CK(cudaMalloc(&c->partial, sizeof(double) * (size_t)kMaxR * kMaxR * 64));
  launch(c, KC_OTHER, k_colpair, dim3(gx, R * R), dim3(kBlock), A, B, (int)c->nl, R, c->partial);
  std::vector<double> h(need);
  CK(cudaMemcpyAsync(h.data(), c->partial, sizeof(double) * need, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  G.assign((size_t)R * R, 0.0);
  for (int p = 0; p < R * R; ++p) {
    double s = 0.0;
    for (int b = 0; b < gx; ++b) s += h[(size_t)p * gx + b];
    G[(size_t)p] = s;
  }
  return SCG_OK;
}

static scg_status rowmat(scg_ctx *c, double *out, const double *A, const double *B, double beta,
                         const std::vector<double> &M) {
  CK(cudaMemcpyAsync(c->dmat, M.data(), sizeof(double) * M.size(), cudaMemcpyHostToDevice, c->stream));
  launch(c, KC_OTHER, k_rowmat, dim3(grid_for(c->nl, 4 * c->nsm)), dim3(kBlock), out, A, B, beta,
         (const double *)c->dmat, (int)c->nl, c->R);
  return SCG_OK;
}

scg_status sketchycgal_reconstruct(scg_ctx *c, double *Uh, double *Lambda, double *errh) {
  if (!c || !Lambda) return SCG_EINVAL;
  if (c->t < 1) return fail(c, SCG_ESTATE, "reconstruct before any iteration");
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  const int R = c->R;
  const size_t nlbR = sizeof(double) * (size_t)c->nl * R;
  if (!c->U) {
    CK(cudaMalloc(&c->U, nlbR));
    CK(cudaMalloc(&c->tmp1, nlbR));
    CK(cudaMalloc(&c->tmp2, nlbR));
    CK(cudaMalloc(&c->dmat, sizeof(double) * kMaxR * kMaxR));
    CK(cudaMalloc(&c->dlam, sizeof(double) * kMaxR));
  }
  std::vector<double> Gss, Gos, Goo;
  if ((st = gram(c, c->S, c->S, Gss)) || (st = gram(c, c->Om, c->S, Gos)) || (st = gram(c, c->Om, c->Om, Goo)))
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
  if ((st = rowmat(c, c->tmp1, c->S, c->Om, sigma, inv_upper(Rc, R)))) return st;
  // CholeskyQR2 of Y: Y = Q Rf
  std::vector<double> G1, R1, G2, R2;
  if ((st = gram(c, c->tmp1, c->tmp1, G1))) return st;
  if (!chol_upper(G1, R, R1)) {
    // shifted CholeskyQR: add a tiny diagonal shift
    double tr = 0;
    for (int i = 0; i < R; ++i) tr += G1[(size_t)i * R + i];
    for (int i = 0; i < R; ++i) G1[(size_t)i * R + i] += 1e-15 * tr;
    if (!chol_upper(G1, R, R1)) return fail(c, SCG_ECHOL, "CholeskyQR failed");
  }
  if ((st = rowmat(c, c->tmp2, c->tmp1, nullptr, 0.0, inv_upper(R1, R)))) return st;
  if ((st = gram(c, c->tmp2, c->tmp2, G2))) return st;
  if (!chol_upper(G2, R, R2)) return fail(c, SCG_ECHOL, "CholeskyQR2 failed");
  if ((st = rowmat(c, c->tmp1, c->tmp2, nullptr, 0.0, inv_upper(R2, R)))) return st;  // Q in tmp1
  std::vector<double> Rf = matmul(R2, R1, R);
  std::vector<double> Ur, sv;
  svd_jacobi(Rf, R, Ur, sv);
  if ((st = rowmat(c, c->U, c->tmp1, nullptr, 0.0, Ur))) return st;  // U = Q Ur
  // Lambda = max(0, Sigma^2 - sigma) (line 16); err (SM3 line 6); trace correction (Alg. 4 line 13)
  double tau = 0.0;
  CK(cudaMemcpy(&tau, &c->sc->tau, sizeof(double), cudaMemcpyDeviceToHost));
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
    c->lam_tc[k] = (c->lam_raw[k] + (c->alpha - tot) / R) * unit;
  }
  const std::vector<double> &lam_out = (c->flags & SCG_TRACE_CORRECT) ? c->lam_tc : c->lam_orig;
  for (int k = 0; k < R; ++k) Lambda[k] = lam_out[k];
  if (errh)
    for (int k = 0; k < R; ++k) errh[k] = c->err[k];
  CK(cudaStreamSynchronize(c->stream));
  if (Uh) CK(cudaMemcpy(Uh, c->U, nlbR, cudaMemcpyDeviceToHost));
  c->have_recon = true;
  return SCG_OK;
}

static scg_status colstats(scg_ctx *c, int which, const double *lam_host, std::vector<double> &outk) {
  const int R = c->R;
  const int gx = std::max(1, std::min(grid_for(c->nl, 4 * c->nsm), 64));
  if (lam_host) CK(cudaMemcpyAsync(c->dlam, lam_host, sizeof(double) * R, cudaMemcpyHostToDevice, c->stream));
  const int ny = which == 2 ? 1 : R;
  launch(c, KC_OTHER, k_colstats, dim3(gx, ny), dim3(kBlock), (const int *)c->rp, (const int *)c->col,
         (const double *)c->wts, (const double *)c->ldiag, (const double *)c->U, (const double *)c->U,
         (const double *)c->dlam, (int)c->nl, (long long)c->rb, (long long)c->n, R, which, c->partial);
  std::vector<double> h((size_t)ny * gx);
  CK(cudaMemcpyAsync(h.data(), c->partial, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  outk.assign(ny, 0.0);
  for (int k = 0; k < ny; ++k)
    for (int b = 0; b < gx; ++b) outk[k] += h[(size_t)k * gx + b];
  return SCG_OK;
}

scg_status sketchycgal_objective(scg_ctx *c, double out[2]) {
  if (!c || !out) return SCG_EINVAL;
  scg_status st = sketchycgal_synchronize(c);
  if (st) return st;
  double p = 0.0;
  CK(cudaMemcpy(&p, &c->sc->p, sizeof(double), cudaMemcpyDeviceToHost));
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
  std::vector<double> z((size_t)c->nl);
  CK(cudaMemcpy(z.data(), c->z, sizeof(double) * c->nl, cudaMemcpyDeviceToHost));
  const double unit = c->alpha_orig / c->alpha;
  double s = 0.0;
  for (int64_t r = 0; r < c->nl; ++r) {
    const double e = (z[(size_t)r] - c->b) * unit;
    s += e * e;
  }
  const double nb = std::sqrt((double)c->n);
  out[0] = std::sqrt(s) / (1.0 + nb);
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
  std::vector<double> u((size_t)c->nl);
  CK(cudaMemcpy(u.data(), c->U + (size_t)best * c->nl, sizeof(double) * c->nl, cudaMemcpyDeviceToHost));
  const int flip = u[0] >= 0.0 ? 1 : -1;  // normalize chi_0 = +1 (global row 0 is local on one GPU)
  for (int64_t r = 0; r < c->nl; ++r) chi[r] = (int8_t)((u[(size_t)r] >= 0.0 ? 1 : -1) * flip);
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
    out[cnt].total_ms = c->kms[k];
    out[cnt].bytes_per_launch = c->kl[k] ? c->kbytes_sum[k] / (double)c->kl[k] : c->kbytes[k];
    ++cnt;
  }
  return cnt;
}

void sketchycgal_reset_stats(scg_ctx *c) {
  if (!c) return;
  ev_flush(c);
  for (int k = 0; k < KC_COUNT; ++k) { c->kl[k] = 0; c->kms[k] = 0; c->kbytes_sum[k] = 0; }
  c->launches = 0;
}

}  // extern "C"
