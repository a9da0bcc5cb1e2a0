// kernels.cuh -- the per-iteration hot path of SketchyCGAL for MaxCut on sm_100a.
//
// Every kernel is HBM-bandwidth bound fp64 work (sparse matvec, axpys, rank-one
// sketch update); none is a dense contraction, so no tensor cores are used
// (DESIGN.md section 5).  Arithmetic follows the Canonical Arithmetic Contract
// (DESIGN.md section 3): one IEEE operation per written op, fma only where written
// (the library is compiled with --fmad=false), exact global sums (xsum.cuh).
//
// Data layout, one GPU owning rows [rb, rb + nl):
//   CSR of the off-diagonal part of C = -L/||L||_F: rp[nl+1] int32, col int32
//   (global ids, ascending), val fp64; cdiag[nl] = C_rr; d[nl] = diagonal of D_t.
//   Gathered vectors (Lanczos w_i, g, x) are full length n (global index); own
//   rows live at [rb, rb + nl).  Local vectors (a, z, y, v) are length nl.
//   Omega, S: nl x R column-major, leading dimension nl.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "xsum.cuh"
#include "../../scg_inputs/include/scg_rng.h"

namespace scg {

constexpr int kMaxQ = 256;   // device arrays hold q <= kMaxQ - 1 = 255 Lanczos steps (q_t of configs[0..4]
                             // is <= 94; a larger q_t is an SCG_EUNSUPPORTED error, never truncated)
constexpr int kMaxR = 64;    // sketch rank cap (BASELINE: R <= 50)
constexpr int kBlock = 256;
constexpr int kBlockA = 256;  // threads per block of k_lanczos_a (the SpMV of pass 1)

// Device-resident scalars of the current iteration.
struct DevScalars {
  double om[kMaxQ];        // omega_i, i = 1..k  (om[i-1])
  double rho[kMaxQ + 1];   // rho[0] = ||g|| (start-vector norm), rho[i] = rho_i  (Alg. 2 line 7)
  double s[kMaxQ];         // eigenvector of the tridiagonal (CAC-5)
  double gk[kMaxR];        // g = v^T Omega
  double theta, nu_x, xi, c, vv, nz, gamma, p, tau;
  double my[4];            // sums over the state (y_t, z_t) of the NEXT iteration: y, y.z, z.z, z (k_dual_sketch)
  double g2n[2];           // ||g||^2 of the start vector drawn ahead on the side stream, by parity of its t
  double bs[2];            // ball projections [0] wbar_t, [1] w_{t+1}: l2 scale fl(delta / N) (reading R34),
                           //   l1 threshold theta (reading R35)
  int bin[2];              //   and whether the point is already inside the ball (the projection is then the point)
  unsigned long long bk[2];  // l1 threshold search: keys (bit patterns) lo, hi of the bracket (reading R35)
  double mz[2];            // A X = b: sum z_{t+1}, z_{t+1}.z_{t+1} from k_primal (FK_NZZ), taken into my by the dual
  int bdone, bpad;
  int k, brk, err, pad;
};

// Exact-sum slot: up to 3 accumulators + a block ticket counter.
constexpr int kMaxSums = 5;  // exact sums one kernel can produce
struct XSlot {
  long long limbs[kMaxSums][kLimbs];
  unsigned int counter;
  unsigned int pad;
};

struct Csr {
  const int *rp;
  const int *col;
  const double *val;
};

// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialization and waits at entry until the previous grid has completed and flushed
// (griddepcontrol.wait).  Kernels with exact sums let the next grid be scheduled when a
// block reaches its commit (pdl_trigger: the main work is done), the others at exit, so the
// next launch overlaps the tail (ticket, finalize) without the dependent grid's blocks
// holding SM slots during the main work.  All data dependences are honored by the wait.
// (No-ops when launched without the attribute.)
// (Triggering right after the wait instead was measured 17% slower on configs[3]: the dependent
// grid's blocks then hold SM slots during the whole main loop.)
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Host-computed scalars of iteration t (CAC-6).
struct IterArgs {
  long long t;
  int q;
  int trace_le;  // SCG_TRACE_LE: H = 0 when xi_t >= 0
  int ineq;      // general template A X in K (box or ball): gap / bound with the slack (reading R33)
  double lo, hi; // box K = {lo <= u <= hi} (SCG_INEQ: lo = -inf, hi = b): w = min(max(z + y/beta, lo), hi) (R32)
  double delta;  // l2 ball K = {||u - b|| <= delta} (sketchycgal_set_ball, reading R34)
  double eta, one_m_eta, alpha, b, beta0, sq, beta_next, nbb;  // nbb = fl(fl(n b) b) = ||b||^2
};

// ---------------------------------------------------------------- row-sharded execution
// P ranks own contiguous row blocks.  Each rank keeps the gathered vectors (the
// Lanczos vectors w_i, the start vector g, x) at GLOBAL indices in its "gathered
// region" G; own rows are written locally and, for rows some other rank reads
// (halo rows: a column of that rank's rows -- by symmetry of L, exactly the rows r
// with a column owned by that rank), also stored straight into that rank's G over
// NVLink peer memory by the producing kernel (mask[r] = bitmask of reader ranks).
// Global exact sums (CAC-2) are combined through per-rank mailboxes: the last block
// of a producer stores its rank's integer limbs into every rank's mailbox and then
// raises a per-(epoch, source) flag with release semantics (system scope); a
// one-warp "pull" kernel on each rank waits for all P flags, adds the P limb sets
// (exact integers: bitwise independent of P) and runs the same finalize code the
// single-GPU last block runs.  The flag is raised after every block of the
// producer fenced its peer stores, so a completed pull also means every halo entry
// of that producer has landed.  The same code runs P shards inside one process on
// one device ("emulated shards": peers are the other shards' buffers), which is how
// the sharded kernels are checked bitwise against the oracle on a single GPU.
constexpr int kMaxRanks = 8;

struct Mailbox {
  long long limbs[4][kMaxRanks][kMaxSums][kLimbs];  // [epoch & 3][source rank][sum][limb]
  double fv[4][kMaxRanks][kMaxR];            // fp64 payload (g = v^T Omega partials)
  unsigned long long flag[4][kMaxRanks];     // epoch published by the source rank
};

struct Net {
  const unsigned char *mask;  // [nl] reader-rank bitmask of each own row; nullptr when P == 1
  double *G;                  // this rank's gathered region
  double *const *peerG;       // [P] every rank's gathered region (device pointers, peer-mapped)
  Mailbox *const *peerMB;     // [P] every rank's mailbox
  Mailbox *mb;                // own mailbox
  int P, me;
  int nowait;                 // the host synchronized the ranks before this pull: check the flags once
  unsigned long long E;       // epoch of the collective this launch takes part in
};

// Store v at dst (this rank's gathered region) and into the reader ranks' copies given the
// row's reader mask m (loaded by the caller together with the row's data).
__device__ __forceinline__ void gstore_m(const Net &net, double *dst, unsigned m, double v) {
  *dst = v;
  if (m) {
    const long long off = dst - net.G;
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
      net.peerG[q][off] = v;
    }
  }
}
// Mask byte of own row r (0 when P == 1).
__device__ __forceinline__ unsigned gmask(const Net &net, int r) { return net.mask ? (unsigned)net.mask[r] : 0u; }

// Store v at dst (this rank's gathered region, own row r) and into every reader rank's copy.
__device__ __forceinline__ void gstore(const Net &net, double *dst, int r, double v) {
  *dst = v;
  if (net.mask) {
    unsigned m = net.mask[r];
    if (m) {
      const long long off = dst - net.G;
      while (m) {
        const int q = __ffs(m) - 1;
        m &= m - 1;
        net.peerG[q][off] = v;
      }
    }
  }
}

enum FinKind { FK_FROB = 0, FK_RHO0, FK_OM, FK_RHO, FK_NUX, FK_MON, FK_NZ, FK_BAR, FK_RHO0M, FK_GEN, FK_RHO0S, FK_MY4,
               FK_NZZ, FK_RHO0Y, FK_RHO0SY,
               FK_GK, FK_BALLS, FK_L1S, FK_L1B };

struct FinArgs {
  int i;                 // Lanczos step (FK_OM, FK_RHO, FK_BAR)
  int R;                 // sketch rank (FK_NZ)
  IterArgs A;            // FK_NZ
  scg_iter_rec *log;     // FK_NZ
  double *out;           // FK_FROB
};

// ---------------------------------------------------------------- division
// (Diagnostics only since the contract evaluates v / rho as v * fl(1/rho), R26.)
// a / b, correctly rounded (IEEE), for a divisor b shared by many quotients:
// rb = RN(1/b) is computed once; two Markstein corrections with exact fma
// residuals r = a - q b give RN(a / b) for normal-range operands (tested
// bitwise against the hardware division in tests/test_gpu_parity.py).  Used
// for the normalization v = w / rho of Alg. 2 line 9.
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
  const double q0 = a * rb;
  const double q1 = fma(fma(-q0, b, a), rb, q0);
  const double q2 = fma(fma(-q1, b, a), rb, q1);
  return a == 0.0 ? q0 : q2;
}

// ---------------------------------------------------------------- row engine
// Rows with at most kLongRow off-diagonal entries are "short": they live in a SELL-32-sigma
// layout (slices of 32 consecutive relabeled rows, one lane per row) walked by a
// three-stage register pipeline (spmv_rows).  Longer rows are "long": a warp loads 32
// entries per round (coalesced) and the lanes run the strided partial chains of reading
// R27; long rows are listed at init (longest first) and taken by the first warps of the
// grid so they start early.
constexpr int kMinBlocksUni = 3;  // min blocks per SM of the uniform-weight SELL SpMV kernels (80-register cap)
// min blocks per SM of the ELL SpMV kernels: 64-register cap up to W = 4, wider rows need more stage registers
// (a deeper pipeline -- gathers two slices ahead, 78 registers, 3 blocks/SM -- measured 171 us against
// 140 us on configs[3]: the fourth block per SM is worth more than the extra slack; on configs[4]'s
// valued ELL-3, 80 registers, 911 us either way: that launch moves 5.07 GB of DRAM reads for 2.01 GB
// algorithmic, so it is bound by the random gathers' DRAM traffic, not by latency -- gpurun_out/ed)
constexpr int ell_min_blocks(int W, bool uni) { return (W & 15) <= 4 ? 4 : (uni ? 3 : 2); }
// ELL width code: W & 15 = slots per row; kEllPos set = every coefficient is +m0 (uniform positive
// weights -- C~ = -L / ||L|| has the positive off-diagonals w / ||L|| -- padding included): the layout
// then carries no sign bits and the SpMV no sign handling
constexpr int kEllPos = 32;
constexpr int kLongRow = 32;
constexpr int kHeavyRow = 1024;  // rows with more entries are "heavy": a block each (256 strided chains)

struct Rows {
  const int *longrows;  // local ids of long rows (33..1024 entries), longest first
  int nlong;
  const int *heavyrows; // local ids of heavy rows (> 1024 entries), longest first
  int nheavy;
  // SELL-32-sigma layout of the short rows.  Rows are relabeled at init so that each
  // window of kSortWin rows is sorted by length (long rows first): slice s covers the 32
  // consecutive rows 32 s .. 32 s + 31; slot j of lane l is at meta[s].x + 32 j + l;
  // meta[s].y = width | (number of leading long-row lanes, skipped) << 8.
  const int2 *meta;
  const int *scol;      // column | 0x80000000 for a negative uniform value; padding = dummy column n
  const double *sval;   // per-slot values, or nullptr when all |C_rj| equal m0
  double m0;
  int nslice;
  unsigned *work;       // non-null: dynamic slice distribution (chunks of kDynCh slices from this
                        // counter; zeroed again by the kernel's last block) -- skewed graphs
  // ELL-W layout (graphs whose rows all have <= kEllMax entries: no long rows, no slice metadata):
  // slice s = rows 32 s .. 32 s + 31, slot j of lane l at ecol[(32 s) W + 32 j + l] (W = 2, 4:
  // at ecol[(32 s) W + W l + j], one vector load per lane); rows shorter
  // than W are padded with the dummy column n (gathered value -0, coefficient +m0 or value +0: the
  // product is -0 and fma(., ., acc) == acc for every acc, -0 included)
  const int *ecol;      // column | 0x80000000 for a negative uniform value (no sign bits: kEllPos)
  const double *eval;   // per-slot values, or nullptr when all |C_rj| equal m0
  int padc;             // the padding code
};
constexpr int kEllMax = 8;  // widest ELL layout (rows of at most 8 off-diagonal entries)
constexpr int kDynCh = 8;

constexpr int kWin = 1024;  // vector padding granularity (rows)

template <int NC>
struct RowOut {
  int r;        // local row
  double xr;    // x_r (own entry of the gathered vector, divided by den)
  double s[NC]; // chain results
};

// One long row (> kLongRow entries) by a warp; result valid in lane 0.  CAC-3 for long
// rows (reading R27): lane l runs the partial chain over the row's entries l, l+32, ...
// (ascending column order) by fma from 0 -- exactly the coalesced round structure --;
// the partials combine by halving (L[l] += L[l+off], off = 16..1) and the row is
// fl(fl(d_r x_r) + L[0]).  Rounds k+1 .. k+kLR-1 are loaded while round k is chained.
template <int NC>
__device__ __forceinline__ void long_row_chain(const Csr &C, int r, const double *__restrict__ X, double den,
                                               const double *__restrict__ diag0, const double *__restrict__ diag1,
                                               long long rb, RowOut<NC> &o) {
  const int lane = threadIdx.x & 31;
  const int e0 = __ldg(&C.rp[r]), e1 = __ldg(&C.rp[r + 1]);
  const double rden = 1.0 / den;
  // columns (and values) are loaded kLC rounds ahead, the gathers x[col] kLR rounds ahead,
  // so a round never waits on a load chain issued in the same round
  constexpr int kLR = 4, kLC = 8;
  int cq[kLC];
  double mq[kLC], xq[kLR];
#pragma unroll
  for (int u = 0; u < kLC; ++u) {
    const int e = e0 + 32 * u + lane;
    cq[u] = e < e1 ? __ldg(&C.col[e]) : -1;
    mq[u] = e < e1 ? __ldg(&C.val[e]) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kLR; ++u) xq[u] = cq[u] >= 0 ? __ldg(&X[cq[u]]) : 0.0;
  double part[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) part[c] = 0.0;
  for (int base = e0; base < e1; base += 32) {
    const bool have = base + lane < e1;
    const double m = mq[0], x = (xq[0]) * rden;  // v = w * fl(1/rho) (Alg. 2 line 9, reading R26)
    // gather of round k + kLR (its column arrived kLC - kLR rounds ago)
    const double xn = cq[kLR] >= 0 ? __ldg(&X[cq[kLR]]) : 0.0;
#pragma unroll
    for (int u = 0; u + 1 < kLR; ++u) xq[u] = xq[u + 1];
    xq[kLR - 1] = xn;
#pragma unroll
    for (int u = 0; u + 1 < kLC; ++u) { cq[u] = cq[u + 1]; mq[u] = mq[u + 1]; }
    {
      const int e = base + 32 * kLC + lane;
      cq[kLC - 1] = e < e1 ? __ldg(&C.col[e]) : -1;
      mq[kLC - 1] = e < e1 ? __ldg(&C.val[e]) : 0.0;
    }
    if (have)
#pragma unroll
      for (int c = 0; c < NC; ++c) part[c] = fma(m, x, part[c]);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double t = __shfl_down_sync(0xffffffffu, part[c], off);
      if (lane < off) part[c] = part[c] + t;
    }
  o.r = r;
  o.xr = (X[rb + r]) * rden;
  o.s[0] = diag0[r] * o.xr + part[0];
  if (NC > 1) o.s[NC - 1] = diag1[r] * o.xr + part[NC - 1];
}


// ---------------------------------------------------------------- TMA / mbarrier / cp.async helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// One heavy row (> kHeavyRow entries) by a block; result valid in thread 0.  CAC-3 for heavy rows
// (reading R27, SURVEY CAC-2's W = 256 bin): thread l (l < 256) runs the partial chain over the row's
// entries l, l+256, ... (ascending column order) by fma from 0; the partials combine by halving in
// shared memory (L[l] = L[l] + L[l+off], off = 128..1) and the row is fl(fl(d_r x_r) + L[0]).  Every
// thread of the block calls this (threads >= 256 only take part in the barriers).
template <int NC>
__device__ __forceinline__ void heavy_row_chain(const Csr &C, int r, const double *__restrict__ X, double den,
                                                const double *__restrict__ diag0, const double *__restrict__ diag1,
                                                long long rb, RowOut<NC> &o) {
  __shared__ double hv[NC][256];
  const int tid = threadIdx.x;
  const int e0 = __ldg(&C.rp[r]), e1 = __ldg(&C.rp[r + 1]);
  const double rden = 1.0 / den;
  double part[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) part[c] = 0.0;
  if (tid < 256) {
    int e = e0 + tid;
    // four entries of the thread's chain in flight at a time
    for (; e + 3 * 256 < e1; e += 4 * 256) {
      double m[4], x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m[u] = __ldg(&C.val[e + u * 256]);
        x[u] = __ldg(&X[__ldg(&C.col[e + u * 256])]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c) part[c] = fma(m[u], x[u] * rden, part[c]);  // v = w * fl(1/rho) (R26)
    }
    for (; e < e1; e += 256) {
      const double m = __ldg(&C.val[e]), x = __ldg(&X[__ldg(&C.col[e])]) * rden;
#pragma unroll
      for (int c = 0; c < NC; ++c) part[c] = fma(m, x, part[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) hv[c][tid] = part[c];
  }
  __syncthreads();
#pragma unroll
  for (int off = 128; off >= 1; off >>= 1) {
    if (tid < off)
#pragma unroll
      for (int c = 0; c < NC; ++c) hv[c][tid] = hv[c][tid] + hv[c][tid + off];
    __syncthreads();
  }
  o.r = r;
  o.xr = X[rb + r] * rden;
  o.s[0] = diag0[r] * o.xr + hv[0][0];
  if (NC > 1) o.s[NC - 1] = diag1[r] * o.xr + hv[NC - 1][0];
  __syncthreads();  // hv is reused by the block's next heavy row
}

// Visit every row of this rank once: epi(RowOut) is called by the owning thread
// (short rows), lane 0 of the owning warp (long rows) or thread 0 of the owning block (heavy rows).
template <int NC, bool UNI, class Epi>
__device__ __forceinline__ void spmv_rows(const Csr &C, const Rows &RL, const double *__restrict__ X, double den,
                                          const double *__restrict__ diag0, const double *__restrict__ diag1,
                                          long long rb, int nl, Epi &epi) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int h = blockIdx.x; h < RL.nheavy; h += gridDim.x) {  // block-uniform loop
    RowOut<NC> o;
    heavy_row_chain<NC>(C, RL.heavyrows[h], X, den, diag0, diag1, rb, o);
    if (threadIdx.x == 0) epi(o);
  }
  for (int w = gw; w < RL.nlong; w += nw) {
    RowOut<NC> o;
    long_row_chain<NC>(C, RL.longrows[w], X, den, diag0, diag1, rb, o);
    if (lane == 0) epi(o);
  }
  const double rden = 1.0 / den;
  {
  // Width-specialized three-stage pipeline: while slice i is computed, the gathers and
  // own entries of slice i+1, the columns of slice i+2 and the meta of slice i+3 are in
  // flight; every stage runs only the slots of its slice's width (warp-uniform switch).
  // static: each block owns a contiguous slice range, its warps interleave (L1 locality);
  // dynamic (RL.work): warps take chunks of kDynCh consecutive slices from a counter
  const int per = (RL.nslice + gridDim.x - 1) / gridDim.x;
  int ns = min(RL.nslice, (int)(blockIdx.x + 1) * per);
  int wstep = blockDim.x >> 5;
  int sl = blockIdx.x * per + (threadIdx.x >> 5);
  auto grab = [&]() {
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(RL.work, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    sl = (int)c * kDynCh;
    ns = min(RL.nslice, sl + kDynCh);
    wstep = 1;
  };
  if (RL.work) grab();
  while (sl < ns) {
  auto mload = [&](int q) -> int2 { return q < ns ? __ldg(&RL.meta[q]) : make_int2(0, 0); };
  auto cload = [&](int2 m, int (&cv)[4], double (&vv)[4]) {
    const int w = m.y & 0xff;
    const int *cp = RL.scol + m.x + lane;
    cv[0] = w > 0 ? __ldg(cp) : -1;
    cv[1] = w > 1 ? __ldg(cp + 32) : -1;
    cv[2] = w > 2 ? __ldg(cp + 64) : -1;
    cv[3] = w > 3 ? __ldg(cp + 96) : -1;
    if (!UNI) {  // values travel with their columns
      const double *vp = RL.sval + m.x + lane;
#pragma unroll
      for (int u = 0; u < 4; ++u) vv[u] = w > u ? __ldg(vp + 32 * u) : 0.0;
    }
  };
  // padding slots hold the dummy column n (gathered value -0, positive coefficient): no test
  auto gload = [&](int2 m, const int (&cv)[4], double (&gv)[4]) {
    switch (m.y & 0xff) {
      case 0: break;
      case 1: gv[0] = __ldg(&X[cv[0] & 0x7fffffff]); break;
      case 2:
        gv[0] = __ldg(&X[cv[0] & 0x7fffffff]);
        gv[1] = __ldg(&X[cv[1] & 0x7fffffff]);
        break;
      case 3:
        gv[0] = __ldg(&X[cv[0] & 0x7fffffff]);
        gv[1] = __ldg(&X[cv[1] & 0x7fffffff]);
        gv[2] = __ldg(&X[cv[2] & 0x7fffffff]);
        break;
      default:
        gv[0] = __ldg(&X[cv[0] & 0x7fffffff]);
        gv[1] = __ldg(&X[cv[1] & 0x7fffffff]);
        gv[2] = __ldg(&X[cv[2] & 0x7fffffff]);
        gv[3] = __ldg(&X[cv[3] & 0x7fffffff]);
        break;
    }
  };
  auto oload = [&](int q, int2 m, double &xo, double &dd, double &dd1) {
    const int p = q * 32 + lane;
    xo = 0.0;
    dd = 0.0;
    dd1 = 0.0;
    if (q < ns && p < nl && lane >= (m.y >> 8)) {
      xo = X[rb + p];
      dd = diag0[p];
      if (NC > 1) dd1 = diag1[p];
    }
  };
  int2 m0 = mload(sl), m1 = mload(sl + wstep), m2 = mload(sl + 2 * wstep);
  int c0[4], c1[4];
  double v0[4], v1[4];
  cload(m0, c0, v0);
  cload(m1, c1, v1);
  double g0[4] = {0.0, 0.0, 0.0, 0.0};
  double xo0, d00, d10;
  gload(m0, c0, g0);
  oload(sl, m0, xo0, d00, d10);
  for (; sl < ns; sl += wstep) {
    const int2 m3 = mload(sl + 3 * wstep);
    int c2[4];
    double v2[4];
    cload(m2, c2, v2);
    double g1[4] = {0.0, 0.0, 0.0, 0.0};
    double xo1, d01, d11;
    gload(m1, c1, g1);
    oload(sl + wstep, m1, xo1, d01, d11);
    // compute slice i
    const int p = sl * 32 + lane;
    const bool ok = p < nl && lane >= (m0.y >> 8);
    RowOut<NC> o;
    o.r = p;
    o.xr = xo0 * rden;
    o.s[0] = d00 * o.xr;
    if (NC > 1) o.s[NC - 1] = d10 * o.xr;
    auto step = [&](int c, double g) {  // c is a real entry or the dummy padding entry
      const double mm = UNI ? (c < 0 ? -RL.m0 : RL.m0) : 0.0;
      const double x = g * rden;  // v = w * fl(1/rho) (Alg. 2 line 9, reading R26)
#pragma unroll
      for (int t = 0; t < NC; ++t) o.s[t] = fma(mm, x, o.s[t]);
    };
    auto stepv = [&](int c, double g, double vv) {
      (void)c;
      const double x = g * rden;
#pragma unroll
      for (int t = 0; t < NC; ++t) o.s[t] = fma(vv, x, o.s[t]);
    };
    const int w = m0.y & 0xff;
    if (UNI) {
      switch (w) {
        case 0: break;
        case 1: step(c0[0], g0[0]); break;
        case 2: step(c0[0], g0[0]); step(c0[1], g0[1]); break;
        case 3: step(c0[0], g0[0]); step(c0[1], g0[1]); step(c0[2], g0[2]); break;
        default: step(c0[0], g0[0]); step(c0[1], g0[1]); step(c0[2], g0[2]); step(c0[3], g0[3]); break;
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < w) stepv(c0[u], g0[u], v0[u]);
    }
    if (w > 4) {  // rows longer than four slots: the next chunk's columns load while this chunk runs
      int cn[4];
      double vn[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cn[u] = 4 + u < w ? __ldg(&RL.scol[m0.x + (4 + u) * 32 + lane]) : -1;
        vn[u] = (!UNI && cn[u] != -1) ? __ldg(&RL.sval[m0.x + (4 + u) * 32 + lane]) : 0.0;
      }
      for (int j0 = 4; j0 < w; j0 += 4) {
        int cx[4];
        double gx[4], vx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { cx[u] = cn[u]; vx[u] = vn[u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) gx[u] = cx[u] != -1 ? __ldg(&X[cx[u] & 0x7fffffff]) : 0.0;
        const int j1 = j0 + 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cn[u] = j1 + u < w ? __ldg(&RL.scol[m0.x + (j1 + u) * 32 + lane]) : -1;
          vn[u] = (!UNI && cn[u] != -1) ? __ldg(&RL.sval[m0.x + (j1 + u) * 32 + lane]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (cx[u] != -1) {  // slots beyond the slice width are not loaded
            if (UNI) step(cx[u], gx[u]);
            else stepv(cx[u], gx[u], vx[u]);
          }
      }
    }
    if (ok) epi(o);
    // rotate
    m0 = m1; m1 = m2; m2 = m3;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c0[u] = c1[u]; c1[u] = c2[u]; g0[u] = g1[u];
      if (!UNI) { v0[u] = v1[u]; v1[u] = v2[u]; }
    }
    xo0 = xo1; d00 = d01; d10 = d11;
  }
  if (!RL.work) break;
  grab();
  }  // while (chunks)
  return;
  }
  (void)nl;
}



// Elements [i0, i1) of a global array (element size ES) are copied as the 16-byte
// aligned byte range around them; sdst then holds the array from the aligned element
// at or below i0 (seg_shift elements before i0).  Arrays carry >= 16 bytes of slack.
template <int ES>
__device__ __forceinline__ uint32_t seg_bytes(long long i0, long long i1) {
  if (i1 <= i0) return 0u;
  return (uint32_t)((((i1 * ES) + 15) & ~15ll) - ((i0 * ES) & ~15ll));
}
template <int ES>
__device__ __forceinline__ void bulk_seg(void *sdst, const void *gbase, long long i0, long long i1,
                                         unsigned long long *bar) {
  if (i1 <= i0) return;
  bulk_g2s(sdst, (const char *)gbase + ((i0 * ES) & ~15ll), seg_bytes<ES>(i0, i1), bar);
}
template <int ES>
__device__ __forceinline__ int seg_shift(long long i0) { return (int)(((i0 * ES) & 15ll) / ES); }

// ---------------------------------------------------------------- ELL-W engine
// Every row has at most W off-diagonal entries (W a compile-time constant): slices of 32 rows
// with exactly W slots each, so a slice's column block sits at a computed offset -- no slice
// metadata, no dependent meta load, no width switch.  Each warp walks its block's slices with a
// register pipeline: while slice i is computed, the gathers of slice i+1, the own entries (x_r,
// d_r) of slice i+2 and the columns of slice i+3 are in flight -- the column stream gets two
// steps of slack before its gathers are issued (one step left the DRAM latency exposed: ncu put
// half of the stall samples on the first use of the columns).  Once a slice's gathers are issued
// its columns are dead; only their sign bits (uniform weights) travel on, packed in one word.
// Per row the arithmetic is the CAC-3 single chain (every row has <= 32 entries, reading R27);
// padding slots add fma(-m, +0, acc) == acc.
template <bool MASK>
__device__ __forceinline__ const double *gaddr(const double *X, int c) {
  // X + c (sign bit masked off) as one 32x32->64 multiply-add (a shift pair in SASS; the compiler
  // otherwise builds the 64-bit offset with six integer instructions)
  const double *p;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(p) : "r"(MASK ? (unsigned)c & 0x7fffffffu : (unsigned)c), "l"(X));
  return p;
}

// One warp-pipelined pass of the fixed-width engine over the slice positions [q0, q1) of this block:
// slice q has its W slots at ec0 + q 32 W (lane-major for W = 2, 4, else slot-major) and its rows at
// 32 q + lane.  (Tried and reverted on configs[3], where ELL-4 pads 40 % of the slots: slices
// grouped in equal-width classes, each class through its own fixed-width run -- 30 % fewer column
// bytes but the gathers lost their locality: DRAM read 566 -> 698 MB, 126 -> 174 us, gpurun_out/r3j;
// a per-slice width inside one run: more instructions than bytes saved, 126 -> 145 us, r3i; 16-bit
// column codes relative to the row with escaped far rows: DRAM read 566 -> 428 MB but a longer
// decode -> address -> gather chain, 126 -> 157 us, r3m.)
template <int NC, bool UNI, bool POS, int W, class Epi>
__device__ __forceinline__ void ell_run(const double *__restrict__ X, double rden, const double *__restrict__ diag0,
                                        const double *__restrict__ diag1, long long rb, int nl,
                                        const int *__restrict__ ec0, const double *__restrict__ ev0, int q0,
                                        int q1, int padc, double m0, Epi &epi) {
  constexpr bool SGN = UNI && !POS;  // uniform magnitude, sign in bit 31 of the column
  constexpr bool VEC = W == 2 || W == 4;
  const int lane = threadIdx.x & 31;
  const int wstep = blockDim.x >> 5;
  int sl = q0 + (int)(threadIdx.x >> 5);
  const int *__restrict__ ec = ec0 + (VEC ? W * lane : lane);
  const double *__restrict__ ev = ev0 + (VEC ? W * lane : lane);
  auto cload = [&](int q, int (&c)[W]) {
    if (q < q1) {
      const int *cp = ec + (long long)q * (32 * W);
      if constexpr (W == 4) {
        const int4 v = __ldg(reinterpret_cast<const int4 *>(cp));
        c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
      } else if constexpr (W == 2) {
        const int2 v = __ldg(reinterpret_cast<const int2 *>(cp));
        c[0] = v.x; c[1] = v.y;
      } else {
#pragma unroll
        for (int u = 0; u < W; ++u) c[u] = __ldg(cp + 32 * u);
      }
    } else {
#pragma unroll
      for (int u = 0; u < W; ++u) c[u] = padc;
    }
  };
  // gathers of slice q from its columns; values (non-uniform weights) travel with the gathers;
  // returns the packed sign bits of the uniform coefficients (bit u = slot u negative)
  auto gload = [&](int q, const int (&c)[W], double (&g)[W], double (&v)[W]) -> unsigned {
    unsigned sg = 0u;
#pragma unroll
    for (int u = 0; u < W; ++u) {
      g[u] = __ldg(gaddr<SGN>(X, c[u]));
      if (SGN) sg |= ((unsigned)c[u] >> 31) << u;
    }
    if (!UNI) {
      const double *vp = ev + (long long)q * (32 * W);
      if constexpr (VEC) {
#pragma unroll
        for (int u = 0; u < W; u += 2) {
          double2 t = make_double2(0.0, 0.0);
          if (q < q1) t = __ldg(reinterpret_cast<const double2 *>(vp + u));
          v[u] = t.x;
          v[u + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < W; ++u) v[u] = q < q1 ? __ldg(vp + 32 * u) : 0.0;
      }
    }
    return sg;
  };
  auto oload = [&](int q, double &xo, double &dd0, double &dd1) {
    const int p = q * 32 + lane;
    xo = 0.0;
    dd0 = 0.0;
    dd1 = 0.0;
    if (q < q1 && p < nl) {
      xo = X[rb + p];
      dd0 = diag0[p];
      if (NC > 1) dd1 = diag1[p];
    }
  };
  int cb[W], cc[W];
  double g0[W], v0[W];
  double xo0, d00, d10, xo1, d01, d11;
  unsigned s0;
  {
    int ca[W];
    cload(sl, ca);
    oload(sl, xo0, d00, d10);
    s0 = gload(sl, ca, g0, v0);
  }
  cload(sl + wstep, cb);
  oload(sl + wstep, xo1, d01, d11);
  cload(sl + 2 * wstep, cc);
  // not unrolled: unrolling by 2 / 3 / 6 kept most register moves and measured 7-19 % slower on
  // configs[3] (gpurun_out/r3a)
#pragma unroll 1
  for (; sl < q1; sl += wstep) {
    double g1[W], v1[W];
    const unsigned s1 = gload(sl + wstep, cb, g1, v1);  // gathers of slice i+1
    int cd[W];
    cload(sl + 3 * wstep, cd);                         // columns of slice i+3
    double xo2, d02, d12;
    oload(sl + 2 * wstep, xo2, d02, d12);              // own entries of slice i+2
    // compute slice i
    const int p = sl * 32 + lane;
    RowOut<NC> o;
    o.r = p;
    o.xr = xo0 * rden;  // v = w * fl(1/rho) (Alg. 2 line 9, reading R26)
    o.s[0] = d00 * o.xr;
    if (NC > 1) o.s[NC - 1] = d10 * o.xr;
#pragma unroll
    for (int u = 0; u < W; ++u) {
      double x = g0[u] * rden;
      if (UNI) {
        // fma(-m0, x, acc) == fma(m0, -x, acc) exactly: the coefficient's sign is moved onto x
        // with one XOR of its high word (POS: no negative coefficient)
        if (SGN) x = __hiloint2double(__double2hiint(x) ^ (int)(((s0 >> u) & 1u) << 31), __double2loint(x));
#pragma unroll
        for (int t = 0; t < NC; ++t) o.s[t] = fma(m0, x, o.s[t]);
      } else {
#pragma unroll
        for (int t = 0; t < NC; ++t) o.s[t] = fma(v0[u], x, o.s[t]);
      }
    }
    if (p < nl) epi(o);
#pragma unroll
    for (int u = 0; u < W; ++u) {
      cb[u] = cc[u];
      cc[u] = cd[u];
      g0[u] = g1[u];
      if (!UNI) v0[u] = v1[u];
    }
    s0 = s1;
    xo0 = xo1; d00 = d01; d10 = d11;
    xo1 = xo2; d01 = d02; d11 = d12;
  }
}

// ELL SpMV (width code W): the block's share of the slices in row order through the fixed-width engine.
template <int NC, bool UNI, int WC, class Epi>
__device__ __forceinline__ void spmv_ell(const Rows &RL, const double *__restrict__ X, double den,
                                         const double *__restrict__ diag0, const double *__restrict__ diag1,
                                         long long rb, int nl, Epi &epi) {
  constexpr int W = WC & 15;
  constexpr bool POS = UNI && (WC & kEllPos) != 0;  // every coefficient +m0, no sign bits
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int nsl = (nl + 31) >> 5;
  const int per = (nsl + G - 1) / G;
  ell_run<NC, UNI, POS, W>(X, 1.0 / den, diag0, diag1, rb, nl, RL.ecol, RL.eval, b * per, min(nsl, (b + 1) * per),
                           RL.padc, RL.m0, epi);
}

// SpMV dispatch: ELL-W when the layout has one (W > 0), else SELL + long rows.
template <int NC, bool UNI, int W, class Epi>
__device__ __forceinline__ void spmv_any(const Csr &C, const Rows &RL, const double *__restrict__ X, double den,
                                         const double *__restrict__ diag0, const double *__restrict__ diag1,
                                         long long rb, int nl, Epi &epi) {
  if constexpr (W > 0) spmv_ell<NC, UNI, W>(RL, X, den, diag0, diag1, rb, nl, epi);  // W: width code
  else spmv_rows<NC, UNI>(C, RL, X, den, diag0, diag1, rb, nl, epi);
}

// ---------------------------------------------------------------- block reduction
// Block-level exact accumulators (shared memory) for NS sums.
template <int NS>
struct XBlk {
  long long l[NS][kLimbs];
};

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

template <int NS>
__device__ __forceinline__ void xblk_init(XBlk<NS> &b) {
  for (int i = threadIdx.x; i < NS * kLimbs; i += blockDim.x) (&b.l[0][0])[i] = 0;
  __syncthreads();
}

// Flush every thread's window into the block accumulator, add the block total to
// the global slot (exact integer atomics), and take a ticket: returns true in the
// last block to finish (which then finalizes the slot).
// Thread 0 fences after the block barrier (fences are cumulative): at system scope when
// P > 1 and the block stored into peer memory, so the mailbox flag the last block raises
// afterwards orders the block's halo stores for the readers.  An acq_rel fence is enough
// for this release pattern.
// peer: nonzero in a thread that stored into a peer rank's memory; only blocks with such a
// thread need the system-scope fence (the others' stores are read on this GPU only).
template <int NS>
__device__ __forceinline__ bool commit_and_ticket(XWin (&acc)[NS], XBlk<NS> &blk, XSlot *slot, int err,
                                                  DevScalars *sc, int P = 1, unsigned peer = 1u) {
  __shared__ int s_last;
  pdl_trigger();  // the block's main work is done: the next grid may start launching
#pragma unroll
  for (int s = 0; s < NS; ++s) xwin_flush(acc[s], blk.l[s]);
  if (__syncthreads_or(err) && threadIdx.x == 0) atomicOr(&sc->err, 1);
  if ((int)threadIdx.x < NS * kLimbs) {
    const int s = threadIdx.x / kLimbs, i = threadIdx.x % kLimbs;
    const long long v = blk.l[s][i];
    if (v != 0) atomicAdd(reinterpret_cast<unsigned long long *>(&slot->limbs[s][i]), (unsigned long long)v);
  }
  // the block's stores (incl. peer halo stores) precede thread 0's fence (cumulative)
  int sys = 0;
  if (P > 1) sys = __syncthreads_or(peer != 0u);
  else __syncthreads();
  if (threadIdx.x == 0) {
    if (sys) fence_acq_rel_sys();
    else fence_acq_rel_gpu();
    const bool last = atomicAdd(&slot->counter, 1u) == gridDim.x - 1;
    // acquire side: every other block's partials (limb atomics and plain stores such as
    // k_primal's gpart) precede the ticket it took; this fence, then the block barrier,
    // orders them before the last block's reads
    if (last) fence_acq_rel_gpu();
    s_last = last;
  }
  __syncthreads();
  return s_last != 0;
}

// Ticket only (kernels without sums that still take part in a collective: the
// pass-2 barrier of the regenerate mode).
__device__ __forceinline__ bool ticket_only(XSlot *slot) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();
    const bool last = atomicAdd(&slot->counter, 1u) == gridDim.x - 1;
    if (last) fence_acq_rel_gpu();
    s_last = last;
  }
  __syncthreads();
  return s_last != 0;
}

// Called by thread 0 of the last block: read + reset slot accumulator s.
__device__ __noinline__ double slot_take(XSlot *slot, int s) {
  long long l[kLimbs];
  for (int i = 0; i < kLimbs; ++i) {
    l[i] = (long long)atomicExch(reinterpret_cast<unsigned long long *>(&slot->limbs[s][i]), 0ull);
  }
  return xacc_round(l);
}

// ---------------------------------------------------------------- finalize (shared by both paths)
__device__ __forceinline__ double gamma_rule(const IterArgs &A, double nz) {
  // eqn:sketchy-cgal-dual-step with ||A||^2 = 1 (CAC-6)
  if (nz == 0.0) return A.beta0;
  double num = 4.0 * A.alpha;
  num = num * A.alpha;
  num = num * A.beta0;
  const double den = ((double)(A.t + 1) * A.sq) * nz;
  const double g = num / den;
  return g < A.beta0 ? g : A.beta0;
}

__device__ __forceinline__ void fin_rho(DevScalars *sc, int i, double rho2) {
  const double rho = sqrt(rho2);
  sc->rho[i] = rho;
  const double rp = i >= 2 ? sc->rho[i - 1] : 0.0;
  if (rho <= 0x1p-45 * (fabs(sc->om[i - 1]) + rp)) {  // Alg. 2 line 8 (reading A3)
    sc->k = i;
    sc->brk = 1;
  }
}

// Turn the rounded global sums of one collective into the device scalars.  Runs in
// the last block of the producer (P == 1) or in k_pull (P > 1): same code, same bits.
__device__ __noinline__ void finalize(int kind, DevScalars *sc, const long long (*L)[kLimbs], const double *gk,
                                      const FinArgs &f) {
  switch (kind) {
    case FK_FROB: *f.out = xacc_round(L[0]); break;
    case FK_RHO0:
    case FK_RHO0M:
      sc->rho[0] = sqrt(xacc_round(L[0]));
      sc->brk = 0;
      sc->k = 0;
      if (kind == FK_RHO0M)
        for (int j = 0; j < 4; ++j) sc->my[j] = xacc_round(L[1 + j]);
      break;
    case FK_GEN: sc->g2n[f.i & 1] = xacc_round(L[0]); break;  // start vector of iteration f.i, drawn ahead
    case FK_MY4:  // gap / bound sums over the state (box sets k_init_box, l2 ball k_ball_d)
      for (int j = 0; j < 4; ++j) sc->my[j] = xacc_round(L[j]);
      break;
    case FK_GK:  // g = v^T Omega (l2 ball: the dual step needs another pass first)
      for (int k = 0; k < f.R; ++k) sc->gk[k] = gk[k];
      break;
    case FK_BALLS: {  // N = ||p - b|| of the points to project onto the l2 ball (reading R34)
      const double N = sqrt(xacc_round(L[0]));
      const int j = f.i;
      sc->bin[j] = !(N > f.A.delta);
      sc->bs[j] = sc->bin[j] ? 1.0 : f.A.delta / N;
      break;
    }
    case FK_L1S: {  // l1 ball: ||p - b||_1 - delta <= 0 (exact sign): p is inside (reading R35)
      XAcc g;
      for (int i = 0; i < kLimbs; ++i) g.d[i] = L[0][i];
      int e = 0;
      xacc_add(g, -f.A.delta, e);
      const int j = f.i;
      sc->bin[j] = !(xacc_round(g.d) > 0.0);
      sc->bdone = sc->bin[j];
      if (!sc->bin[j] && f.A.delta == 0.0) {  // K = {b}: theta = inf gives w = b
        sc->bs[j] = INFINITY;
        sc->bdone = 1;
      }
      sc->bk[0] = 0ull;                    // G(0) > 0
      sc->bk[1] = 0x7fefffffffffffffull;   // G(DBL_MAX) = -delta < 0
      break;
    }
    case FK_L1B: {  // one bisection step on the key of v: G(v) = S(v) - c(v) v - delta < 0 ?
      if (sc->bdone) break;
      const unsigned long long lo = sc->bk[0], hi = sc->bk[1], mid = lo + ((hi - lo) >> 1);
      const double v = __longlong_as_double((long long)mid);
      const double c = xacc_round(L[1]);
      XAcc g;
      for (int i = 0; i < kLimbs; ++i) g.d[i] = L[0][i];
      XAcc sd = g;
      int e = 0;
      const double ph = c * v, pl = fma(c, v, -ph);  // exact product c v
      xacc_add(g, -ph, e);
      xacc_add(g, -pl, e);
      xacc_add(g, -f.A.delta, e);
      xacc_add(sd, -f.A.delta, e);
      if (xacc_round(g.d) < 0.0) {
        sc->bk[1] = mid;
        sc->bs[f.i] = xacc_round(sd.d) / c;  // theta = fl(fl(S - delta) / c) of the new bracket top
      } else {
        sc->bk[0] = mid;
      }
      if (sc->bk[1] - sc->bk[0] <= 1ull) sc->bdone = 1;
      break;
    }
    case FK_RHO0Y:   // A X = b: [||g||^2,] sum y, y.z from k_dual_sketch; z.z, sum z from k_primal (FK_NZZ)
    case FK_RHO0SY: {
      const int o = kind == FK_RHO0Y ? 1 : 0;
      sc->rho[0] = o ? sqrt(xacc_round(L[0])) : sqrt(sc->g2n[f.i & 1]);
      sc->brk = 0;
      sc->k = 0;
      sc->my[0] = xacc_round(L[o]);
      sc->my[1] = xacc_round(L[o + 1]);
      sc->my[2] = sc->mz[1];
      sc->my[3] = sc->mz[0];
      break;
    }
    case FK_RHO0S:  // k_dual_sketch without the draw: the next start vector's norm comes from FK_GEN
      sc->rho[0] = sqrt(sc->g2n[f.i & 1]);
      sc->brk = 0;
      sc->k = 0;
      for (int j = 0; j < 4; ++j) sc->my[j] = xacc_round(L[j]);
      break;
    case FK_OM: sc->om[f.i - 1] = xacc_round(L[0]); break;
    case FK_RHO: fin_rho(sc, f.i, xacc_round(L[0])); break;
    case FK_NUX: sc->nu_x = sqrt(xacc_round(L[0])); break;
    case FK_MON:
      sc->xi = xacc_round(L[0]);
      sc->c = xacc_round(L[1]);
      sc->vv = xacc_round(L[2]);
      break;
    case FK_NZ:
    case FK_NZZ: {
      for (int k = 0; k < f.R; ++k) sc->gk[k] = gk[k];
      const IterArgs &A = f.A;
      const double nz = xacc_round(L[0]);
      // surrogate duality gap (eqn:cgal-gap) and posterior suboptimality
      // bound (eqn:scgal-posterior-error-bd; = the stopping numerator
      // P:4044-4048) of the implicit iterate X_t, with lambda_min(D_t) ~ xi_t and
      // the sums my = (sum y_t, y_t.z_t, z_t.z_t, sum z_t) -- DESIGN.md CAC-6
      double gapv, boundv;
      {
        const double beta = A.beta0 * A.sq;
        // min over the constraint set of <D_t, H>: alpha xi_t (tr X = alpha), alpha min(xi_t, 0) (tr X <= alpha)
        const double pt = sc->p, ax = A.alpha * ((A.trace_le && sc->xi > 0.0) ? 0.0 : sc->xi);
        if (A.ineq) {  // general template (reading R33): my = (<y,z>, <z-w,z>, <y,w>, <z-w,z+w>)
          double g = pt + sc->my[0];
          g = g + beta * sc->my[1];
          gapv = g - ax;
          double u = pt + sc->my[2];
          u = u + (0.5 * beta) * sc->my[3];
          boundv = u - ax;
        } else {       // my = (sum y, <y,z>, <z,z>, sum z)
          const double zmb_z = sc->my[2] - A.b * sc->my[3];
          double g = pt + sc->my[1];
          g = g + beta * zmb_z;
          gapv = g - ax;
          const double zpb = sc->my[2] - A.nbb;
          double u = pt + A.b * sc->my[0];
          u = u + (0.5 * beta) * zpb;
          boundv = u - ax;
        }
      }
      sc->nz = nz;
      if (kind == FK_NZZ) {  // sums over z_{t+1} for the next gap (my is read above, before this)
        sc->mz[0] = xacc_round(L[1]);
        sc->mz[1] = xacc_round(L[2]);
      }
      sc->gamma = gamma_rule(A, nz);
      const double ea2 = A.eta * A.alpha;
      if (A.trace_le && !(sc->xi < 0.0)) {  // H = 0: X <- (1 - eta) X
        sc->tau = A.one_m_eta * sc->tau;
        sc->p = A.one_m_eta * sc->p;
      } else {
        sc->tau = fma(ea2, sc->vv, A.one_m_eta * sc->tau);
        sc->p = fma(ea2, sc->c, A.one_m_eta * sc->p);
      }
      scg_iter_rec rec;
      rec.t = A.t;
      rec.q = A.q;
      rec.k = sc->k;
      rec.theta = sc->theta;
      rec.xi = sc->xi;
      rec.c = sc->c;
      rec.p = sc->p;
      rec.znorm = sqrt(nz);
      rec.gamma = sc->gamma;
      rec.tau = sc->tau;
      rec.gap = gapv;
      rec.bound = boundv;
      if (f.log) f.log[A.t - 1] = rec;
      break;
    }
    default: break;
  }
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// A strong relaxed store: after a fence.sc.sys it completes a release pattern without the
// per-store membar st.release.sys carries (one fence for all P flags instead of P + 1).
__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Last block, thread 0: take this rank's limbs (resetting the slot) and either
// finalize (P == 1) or publish them to every rank's mailbox (P > 1).
template <int NS>
__device__ __forceinline__ void emit(XSlot *slot, DevScalars *sc, const Net &net, int kind, const FinArgs &f,
                                     const double *gk) {
  // acquire side of the block ticket: every block's limb atomics (performed in L2) precede
  // these L2 loads; the slot is idle until the next launch, so plain stores reset it
  fence_acq_rel_gpu();
  long long L[kMaxSums][kLimbs];
#pragma unroll
  for (int s = 0; s < kMaxSums; ++s)
#pragma unroll
    for (int i = 0; i < kLimbs; ++i) L[s][i] = s < NS ? __ldcg(&slot->limbs[s][i]) : 0ll;
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int i = 0; i < kLimbs; ++i) slot->limbs[s][i] = 0;
  slot->counter = 0;
  if (net.P <= 1) {
    finalize(kind, sc, L, gk, f);
    return;
  }
  const int e = (int)(net.E & 3ull);
  const int nf = (kind == FK_NZ || kind == FK_NZZ || kind == FK_GK) ? f.R : 0;
  for (int q = 0; q < net.P; ++q) {
    Mailbox *m = net.peerMB[q];
    for (int s = 0; s < NS; ++s)
      for (int i = 0; i < kLimbs; ++i) m->limbs[e][net.me][s][i] = L[s][i];
    for (int k = 0; k < nf; ++k) m->fv[e][net.me][k] = gk[k];
  }
  __threadfence_system();  // releases the limbs above (and, cumulatively, the halo stores) ...
  for (int q = 0; q < net.P; ++q) st_relaxed_sys(&net.peerMB[q]->flag[e][net.me], net.E);  // ... with these flags
}

// P > 1: wait for every rank's contribution to collective net.E, add, finalize.
// A lost flag (a bug or a dead peer) ends the wait after ~2^34 cycles with sc->err = 2
// instead of hanging the GPU.
__global__ void k_pull(int kind, int ns, Net net, DevScalars *sc, FinArgs f) {
  pdl_entry();
  // one warp: lane p waits for rank p's flag, the limb sums are spread over the lanes (exact
  // integer adds in any order), lane 0 gathers them and finalizes
  const int lane = threadIdx.x;
  if (sc->err & 2) return;  // an earlier collective timed out: fail fast (reported by synchronize)
  if ((kind == FK_OM || kind == FK_RHO) && sc->brk) return;  // producer skipped (Lanczos break)
  if (kind == FK_BAR && f.i >= sc->k) return;
  const int e = (int)(net.E & 3ull);
  Mailbox *m = net.mb;
  int ok = 1;
  if (lane < net.P) {
    const long long t0 = clock64();
    while (ld_acquire_sys(&m->flag[e][lane]) != net.E) {
      if (net.nowait || clock64() - t0 > (1ll << 34)) {  // (nowait: every producer has completed)
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
  }
  if (!__all_sync(0xffffffffu, ok)) {
    if (lane == 0) atomicOr(&sc->err, 2);
    return;
  }
  __syncwarp();  // every flag acquired by some lane precedes lane 0's reads below
  long long part[2] = {0, 0};  // entries lane and lane + 32 of the ns x kLimbs sums
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int idx = lane + 32 * h;
    if (idx < ns * kLimbs)
      for (int p = 0; p < net.P; ++p) part[h] += __ldcv(&m->limbs[e][p][idx / kLimbs][idx % kLimbs]);
  }
  double gpart[2] = {0.0, 0.0};  // g_k = sum over ranks in rank order, k = lane, lane + 32
  if (kind == FK_NZ || kind == FK_NZZ || kind == FK_GK)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = lane + 32 * h;
      if (k < f.R)
        for (int p = 0; p < net.P; ++p) gpart[h] += __ldcv(&m->fv[e][p][k]);
    }
  long long L[kMaxSums][kLimbs];
  double gk[kMaxR];
  // only the ns sums and the R entries of g this kind carries cross the warp (uniform trip counts)
  for (int idx = 0; idx < ns * kLimbs; ++idx) {
    const long long v = __shfl_sync(0xffffffffu, part[idx >> 5], idx & 31);
    if (lane == 0) L[idx / kLimbs][idx % kLimbs] = v;
  }
  if (lane == 0)
    for (int idx = ns * kLimbs; idx < kMaxSums * kLimbs; ++idx) L[idx / kLimbs][idx % kLimbs] = 0ll;
  if (kind == FK_NZ || kind == FK_NZZ || kind == FK_GK)
    for (int k = 0; k < f.R && k < 64; ++k) {
      const double v = __shfl_sync(0xffffffffu, gpart[k >> 5], k & 31);
      if (lane == 0) gk[k] = v;
    }
  if (lane == 0) finalize(kind, sc, L, gk, f);
}

// Consumer-side pull (SCG_INLINE_PULL, P > 1), warp 0 of a block: wait for every rank's flag of
// collective E, add the P limb sets of its first sum (exact integers, any order), round in lane 0 (*out).
// The same flags, limbs and rounding as k_pull; returns 0 (sc->err |= 2) when a flag is lost.
__device__ __forceinline__ int pull_one(const Net &net, unsigned long long E, DevScalars *sc, double *out) {
  const int lane = threadIdx.x & 31;
  const int e = (int)(E & 3ull);
  Mailbox *m = net.mb;
  int ok = 1;
  if (lane < net.P) {
    const long long t0 = clock64();
    while (ld_acquire_sys(&m->flag[e][lane]) != E) {
      if (net.nowait || clock64() - t0 > (1ll << 34)) {
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
  }
  if (!__all_sync(0xffffffffu, ok)) {
    if (lane == 0) atomicOr(&sc->err, 2);
    return 0;
  }
  __syncwarp();
  long long part = 0;
  if (lane < kLimbs)
    for (int p = 0; p < net.P; ++p) part += __ldcv(&m->limbs[e][p][0][lane]);
  long long L[kLimbs];
#pragma unroll
  for (int i = 0; i < kLimbs; ++i) L[i] = __shfl_sync(0xffffffffu, part, i);
  if (lane == 0) *out = xacc_round(L);
  return 1;
}

// ---------------------------------------------------------------- init kernels
// ||L||_F^2 over all stored entries: off-diagonal weights (each stored once per
// direction) and the diagonal (scaling).
__global__ void k_frob(const double *__restrict__ w, long long nnz, const double *__restrict__ diag, int nl,
                       XSlot *slot, DevScalars *sc, double *out, Net net) {
  pdl_entry();
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += st) xwin_add_nn(acc[0], w[k] * w[k], err, xb.l[0]);
  for (long long r = tid; r < nl; r += st) xwin_add_nn(acc[0], diag[r] * diag[r], err, xb.l[0]);
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P) && threadIdx.x == 0) {
    FinArgs f{};
    f.out = out;
    emit<1>(slot, sc, net, FK_FROB, f, nullptr);
  }
}

// C = -L (scaled by 1/nrm when scale): val = fl(w / nrm), cdiag = fl(-L_rr / nrm).
__global__ void k_scale_c(const double *__restrict__ w, long long nnz, const double *__restrict__ ldiag, int nl,
                          const double *__restrict__ nrm_ptr, int scale, double *__restrict__ val,
                          double *__restrict__ cdiag) {
  pdl_entry();
  const double nrm = *nrm_ptr;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += st) val[k] = scale ? w[k] / nrm : w[k];
  for (long long r = tid; r < nl; r += st) cdiag[r] = scale ? (-ldiag[r]) / nrm : -ldiag[r];
}

// Omega[i, k] ~ N(0,1) from the seeded stream (Alg. 3 line 2).
// orig[r]: original (input) index of local row r minus rb -- rows are relabeled at init
// (DESIGN.md section 5); the seeded streams are indexed by the ORIGINAL vertex id.
__global__ void k_omega(double *__restrict__ Om, int nl, long long rb, int R, uint64_t seed,
                        const int *__restrict__ orig) {
  pdl_entry();
  const long long tot = (long long)nl * R;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e / nl);
    const long long r = e - (long long)k * nl;
    Om[e] = scg_omega(seed, rb + orig[r], k);
  }
}

// d = fl(fma(beta, fl(z - b), y) + C_rr) (primitive 2 with y + beta (z - b)).
__global__ void k_init_d(const double *__restrict__ z, const double *__restrict__ y, const double *__restrict__ cdiag,
                         double *__restrict__ d, int nl, double b, double beta, int ineq, double lo, double hi) {
  pdl_entry();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double w = ineq ? fmin(fmax(z[r] + y[r] / beta, lo), hi) : b;  // slack w_1 = proj_K(z + y / beta)
    d[r] = fma(beta, z[r] - w, y[r]) + cdiag[r];
  }
}

// Box sets (sketchycgal_set_box, before the first step): d for t = 1 with w_1 = proj_K(z_1 + y_1 / beta_1)
// and the general-template gap / bound sums over the initial state (reading R33).
__global__ void k_init_box(const double *__restrict__ z, const double *__restrict__ y, const double *__restrict__ cdiag,
                           double *__restrict__ d, int nl, double beta, double lo, double hi, XSlot *slot,
                           DevScalars *sc, Net net) {
  pdl_entry();
  __shared__ XBlk<4> xb;
  xblk_init<4>(xb);
  XWin acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xwin_init(acc[q]);
  int err = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double zr = z[r], yr = y[r];
    const double w = fmin(fmax(zr + yr / beta, lo), hi);  // slack w_1 = proj_K(z_1 + y_1 / beta_1)
    const double e = zr - w;
    d[r] = fma(beta, e, yr) + cdiag[r];
    xwin_add(acc[0], yr * zr, err, xb.l[0]);
    xwin_add(acc[1], e * zr, err, xb.l[1]);
    xwin_add(acc[2], yr * w, err, xb.l[2]);
    xwin_add(acc[3], e * (zr + w), err, xb.l[3]);
  }
  if (commit_and_ticket<4>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0)
    emit<4>(slot, sc, net, FK_MY4, FinArgs{}, nullptr);
}

// Lanczos start vector g = randn (Alg. 2 line 1) for iteration t and ||g||^2 (exact).
// kind FK_RHO0: the start vector of the iteration about to run (init); FK_GEN: drawn one iteration
// ahead on the side stream, its norm parked in sc->g2n[t & 1].
__global__ void __launch_bounds__(kBlock) k_gen_start(double *__restrict__ g, int nl, long long rb, uint64_t seed,
                                                      long long t, XSlot *slot, DevScalars *sc, Net net,
                                                      const int *__restrict__ orig, int kind) {
  pdl_entry();
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double v = scg_lanczos_start(seed, t, rb + orig[r]);
    gstore(net, g + rb + r, r, v);
    xwin_add_nn(acc[0], v * v, err, xb.l[0]);
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = (int)(t & 1);
    emit<1>(slot, sc, net, kind, f, nullptr);
  }
}

// ---------------------------------------------------------------- Lanczos pass 1
// Step i, part A (Alg. 2 lines 4-5): a = D v_i with v_i = X_i / rho[i-1] formed on the
// fly (Alg. 2 line 9 division), omega_i = v_i . a (exact).
//   (D x)_r = fl(d_r x_r) then fma(C_rj, x_j, acc) over j ascending (CAC-3).
struct EpiA {
  double *a;
  long long *blk;
  XWin acc[1];
  int err;
  __device__ __forceinline__ void operator()(const RowOut<1> &o) {
    a[o.r] = o.s[0];
    xwin_add(acc[0], o.xr * o.s[0], err, blk);
  }
};

template <bool UNI, int W>  // W > 0: ELL-W layout (spmv_ell), 0: SELL + long rows
__global__ void __launch_bounds__(kBlockA, W > 0 ? ell_min_blocks(W, UNI) : (UNI ? kMinBlocksUni : 2)) k_lanczos_a(Csr C, Rows RL, const double *__restrict__ d,
                                                         const double *__restrict__ X, int nl, long long rb, int i,
                                                         double *__restrict__ a, XSlot *slot, DevScalars *sc,
                                                         Net net, unsigned long long pE) {
  pdl_entry();
  if (sc->brk) return;
  double den;
  if (pE) {  // SCG_INLINE_PULL: rho_{i-1} of collective pE (k_lanczos_b of step i - 1), fin_rho's arithmetic
    __shared__ double s_den;
    __shared__ int s_go;
    if (threadIdx.x < 32) {
      double r2 = 0.0;
      const int ok = pull_one(net, pE, sc, &r2);
      if (threadIdx.x == 0) {
        const int j = i - 1;
        const double rho = sqrt(r2);
        const double rp = j >= 2 ? sc->rho[j - 1] : 0.0;
        const bool brk = rho <= 0x1p-45 * (fabs(sc->om[j - 1]) + rp);  // fin_rho's test (Alg. 2 line 8)
        if (ok && blockIdx.x == 0) fin_rho(sc, j, r2);  // the device scalars for later kernels
        s_den = rho;
        s_go = ok && !brk;
      }
    }
    __syncthreads();
    if (!s_go) return;
    den = s_den;
  } else {
    den = sc->rho[i - 1];
  }
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  EpiA epi;
  epi.a = a;
  epi.blk = xb.l[0];
  xwin_init(epi.acc[0]);
  epi.err = 0;
  spmv_any<1, UNI, W>(C, RL, X, den, d, nullptr, rb, nl, epi);
  int err = epi.err;
  XWin (&acc)[1] = epi.acc;
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    if (RL.work) *RL.work = 0u;  // every warp has stopped taking chunks
    FinArgs f{};
    f.i = i;
    emit<1>(slot, sc, net, FK_OM, f, nullptr);
  }
}

// ---------------------------------------------------------------- warp-specialized TMA SpMV
// k_lanczos_a for uniform weights and static slice ranges with one producer warp and
// kWsCons consumer warps per block.  The producer streams each stage -- the metas, the
// columns, the own entries and the diagonal of kWsCons consecutive slices, all contiguous in
// HBM -- into a kWsD-deep shared ring with cp.async.bulk (one thread, completion counted on
// the stage's "full" mbarrier); consumer warp w takes slice w of every stage, copies what
// it needs into registers, releases the stage ("empty" mbarrier, one arrival per warp) and
// issues its gathers one slice ahead.  Every DRAM stream is in flight kWsD stages ahead
// without holding registers; only the gathers (L1/L2) use the register pipeline.  The
// per-row arithmetic is spmv_rows' (CAC-3) exactly.
constexpr int kWsCons = 8;
constexpr int kWsThreads = 32 * (kWsCons + 1);
constexpr int kWsD = 4;
constexpr int kWsCap = 2048;  // column slots per stage (larger stages read columns from HBM)
struct __align__(16) WsStage {
  int cols[kWsCap];
  double x[kWsCons * 32 + 2];  // own entries from a 16-byte aligned start (xsh = 0 or 1)
  double d[kWsCons * 32];
  int2 meta[kWsCons];
  int cbase, ovf, xsh, pad;
};
struct __align__(16) WsSmem {
  WsStage st[kWsD];
  unsigned long long full[kWsD], empty[kWsD];
};
constexpr int kWsMinBlocks = 3;  // 72 registers, 3 blocks/SM (measured: 2 blocks/SM 190 us, 3: 165 us on c3)

template <bool UNI>
__global__ void __launch_bounds__(kWsThreads, kWsMinBlocks) k_lanczos_a_ws(Csr C, Rows RL, const double *__restrict__ d,
                                                                       const double *__restrict__ X, int nl,
                                                                       long long rb, int i, double *__restrict__ a,
                                                                       XSlot *slot, DevScalars *sc, Net net) {
  pdl_entry();
  if (sc->brk) return;
  const double den = sc->rho[i - 1];
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  extern __shared__ __align__(128) unsigned char smraw[];
  WsSmem &sm = *reinterpret_cast<WsSmem *>(smraw);
  EpiA epi;
  epi.a = a;
  epi.blk = xb.l[0];
  xwin_init(epi.acc[0]);
  epi.err = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < kWsCons) {  // long rows (> 32 entries, reading R27): consumer warps, grid-wide
    const int nw = gridDim.x * kWsCons;
    for (int w = blockIdx.x * kWsCons + warp; w < RL.nlong; w += nw) {
      RowOut<1> o;
      long_row_chain<1>(C, RL.longrows[w], X, den, d, nullptr, rb, o);
      if (lane == 0) epi(o);
    }
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < kWsD; ++k) {
      mbar_init(&sm.full[k], 1);
      mbar_init(&sm.empty[k], kWsCons);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int per = (RL.nslice + gridDim.x * kWsCons - 1) / (gridDim.x * kWsCons) * kWsCons;
  const int s_beg = min(RL.nslice, (int)blockIdx.x * per), s_end = min(RL.nslice, s_beg + per);
  const int nst = (s_end - s_beg + kWsCons - 1) / kWsCons;
  const double rden = 1.0 / den, m0v = RL.m0;
  if (warp == kWsCons) {
    // ---- producer: metas come 32 slices (4 stages) per coalesced load, one batch ahead
    auto mbatch = [&](int b) -> int2 {
      const int q = s_beg + 32 * b + lane;
      return q < s_end ? __ldg(&RL.meta[q]) : make_int2(0, 0);
    };
    int2 mcur = mbatch(0), mnext = mbatch(1);
    for (int j = 0; j < nst; ++j) {
      const int sl = j % kWsD;
      if (j > 0 && (j & 3) == 0) {
        mcur = mnext;
        mnext = mbatch((j >> 2) + 1);
      }
      if (j >= kWsD) mbar_wait(&sm.empty[sl], (uint32_t)(((j / kWsD) - 1) & 1));
      WsStage &st = sm.st[sl];
      const int s0 = s_beg + kWsCons * j;
      const int nsl = min(kWsCons, s_end - s0);
      const int src = kWsCons * (j & 3);
      const int2 mv = make_int2(__shfl_sync(0xffffffffu, mcur.x, src + (lane & 7)),
                                __shfl_sync(0xffffffffu, mcur.y, src + (lane & 7)));
      const int first = __shfl_sync(0xffffffffu, mcur.x, src);
      const int lx = __shfl_sync(0xffffffffu, mcur.x, src + nsl - 1);
      const int ly = __shfl_sync(0xffffffffu, mcur.y, src + nsl - 1);
      const int cints = lx + 32 * (ly & 0xff) - first;
      const int ovf = cints > kWsCap ? 1 : 0;
      const long long r0 = (long long)s0 * 32;
      const int nr = (int)min((long long)kWsCons * 32, (long long)nl - r0);
      const double *xs = X + rb + r0;
      const int xsh = (int)(((unsigned long long)(size_t)xs >> 3) & 1ull);
      const uint32_t xbytes = (uint32_t)(((nr + xsh) * 8 + 15) & ~15);
      const uint32_t dbytes = (uint32_t)((nr * 8 + 15) & ~15);
      if (lane < kWsCons) st.meta[lane] = lane < nsl ? mv : make_int2(0, 0);
      if (lane == 0) {
        st.cbase = first;
        st.ovf = ovf;
        st.xsh = xsh;
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t cb = ovf ? 0u : (uint32_t)cints * 4u;
        mbar_arrive_tx(&sm.full[sl], cb + xbytes + dbytes);
        if (cb) bulk_g2s(st.cols, RL.scol + first, cb, &sm.full[sl]);
        bulk_g2s(st.x, xs - xsh, xbytes, &sm.full[sl]);
        bulk_g2s(st.d, d + r0, dbytes, &sm.full[sl]);
      }
    }
  } else {
    // ---- consumer warp: slice "warp" of every stage
    auto take = [&](int j, int2 &m, int (&c)[4], double (&g)[4], double &xo, double &dd) {
      const int sl = j % kWsD;
      mbar_wait(&sm.full[sl], (uint32_t)((j / kWsD) & 1));
      const WsStage &st = sm.st[sl];
      m = st.meta[warp];
      const int w = m.y & 0xff;
      if (!st.ovf) {
        const int *cp = st.cols + (m.x - st.cbase) + lane;
        c[0] = w > 0 ? cp[0] : 0;
        c[1] = w > 1 ? cp[32] : 0;
        c[2] = w > 2 ? cp[64] : 0;
        c[3] = w > 3 ? cp[96] : 0;
      } else {
        const int *cp = RL.scol + m.x + lane;
        c[0] = w > 0 ? __ldg(cp) : 0;
        c[1] = w > 1 ? __ldg(cp + 32) : 0;
        c[2] = w > 2 ? __ldg(cp + 64) : 0;
        c[3] = w > 3 ? __ldg(cp + 96) : 0;
      }
      xo = st.x[st.xsh + warp * 32 + lane];
      dd = st.d[warp * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[sl]);  // the stage's data is in registers now
      switch (w) {
        case 0: break;
        case 1: g[0] = __ldg(&X[c[0] & 0x7fffffff]); break;
        case 2:
          g[0] = __ldg(&X[c[0] & 0x7fffffff]);
          g[1] = __ldg(&X[c[1] & 0x7fffffff]);
          break;
        case 3:
          g[0] = __ldg(&X[c[0] & 0x7fffffff]);
          g[1] = __ldg(&X[c[1] & 0x7fffffff]);
          g[2] = __ldg(&X[c[2] & 0x7fffffff]);
          break;
        default:
          g[0] = __ldg(&X[c[0] & 0x7fffffff]);
          g[1] = __ldg(&X[c[1] & 0x7fffffff]);
          g[2] = __ldg(&X[c[2] & 0x7fffffff]);
          g[3] = __ldg(&X[c[3] & 0x7fffffff]);
          break;
      }
    };
    int2 m0 = make_int2(0, 0);
    int c0[4] = {0, 0, 0, 0};
    double g0[4] = {0.0, 0.0, 0.0, 0.0}, x0 = 0.0, d0 = 0.0;
    if (nst > 0) take(0, m0, c0, g0, x0, d0);
    for (int j = 0; j < nst; ++j) {
      int2 m1 = make_int2(0, 0);
      int c1[4] = {0, 0, 0, 0};
      double g1[4] = {0.0, 0.0, 0.0, 0.0}, x1 = 0.0, d1 = 0.0;
      if (j + 1 < nst) take(j + 1, m1, c1, g1, x1, d1);  // gathers of the next slice in flight
      const int q = s_beg + kWsCons * j + warp;
      const int p = q * 32 + lane;
      const bool ok = q < s_end && p < nl && lane >= (m0.y >> 8);
      RowOut<1> o;
      o.r = p;
      o.xr = x0 * rden;
      o.s[0] = d0 * o.xr;
      auto step = [&](int cc, double gv) {
        const double mm = cc < 0 ? -m0v : m0v;
        o.s[0] = fma(mm, gv * rden, o.s[0]);  // v = w * fl(1/rho) (Alg. 2 line 9, reading R26)
      };
      const int w = m0.y & 0xff;
      switch (w) {
        case 0: break;
        case 1: step(c0[0], g0[0]); break;
        case 2: step(c0[0], g0[0]); step(c0[1], g0[1]); break;
        case 3: step(c0[0], g0[0]); step(c0[1], g0[1]); step(c0[2], g0[2]); break;
        default: step(c0[0], g0[0]); step(c0[1], g0[1]); step(c0[2], g0[2]); step(c0[3], g0[3]); break;
      }
      if (w > 4) {  // rows longer than four slots: remaining chunks from HBM
        for (int j0 = 4; j0 < w; j0 += 4) {
          int cx[4];
          double gx[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) cx[u] = j0 + u < w ? __ldg(&RL.scol[m0.x + (j0 + u) * 32 + lane]) : -1;
#pragma unroll
          for (int u = 0; u < 4; ++u) gx[u] = cx[u] != -1 ? __ldg(&X[cx[u] & 0x7fffffff]) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cx[u] != -1) step(cx[u], gx[u]);
        }
      }
      if (ok) epi(o);
      m0 = m1;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c0[u] = c1[u];
        g0[u] = g1[u];
      }
      x0 = x1;
      d0 = d1;
    }
  }
  int err = epi.err;
  XWin (&acc)[1] = epi.acc;
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = i;
    emit<1>(slot, sc, net, FK_OM, f, nullptr);
  }
}

// Step i, part B (Alg. 2 lines 6-7): w_{i+1} = fma(-rho_{i-1}, v_{i-1}, fma(-omega_i, v_i, a)),
// rho_i = ||w_{i+1}|| (exact); breakdown test.  Writes the un-normalized w_{i+1}.
constexpr int kMinBlocksB = 4;
constexpr int kBU = 2;  // row pairs in flight per thread
__global__ void __launch_bounds__(kBlock, kMinBlocksB) k_lanczos_b(const double *__restrict__ a, const double *Xi,
                                                      const double *Xim1, double *Xip1, int nl, long long rb,
                                                      int i, XSlot *slot, DevScalars *sc, Net net,
                                                      unsigned long long pE) {
  pdl_entry();
  if (sc->brk) return;
  double om;
  if (pE) {  // SCG_INLINE_PULL: omega_i of collective pE (k_lanczos_a of this step)
    __shared__ double s_om;
    __shared__ int s_go;
    if (threadIdx.x < 32) {
      double v = 0.0;
      const int ok = pull_one(net, pE, sc, &v);
      if (threadIdx.x == 0) {
        if (ok && blockIdx.x == 0) sc->om[i - 1] = v;  // FK_OM's finalize, for the tridiagonal solve
        s_om = v;
        s_go = ok;
      }
    }
    __syncthreads();
    if (!s_go) return;
    om = s_om;
  } else {
    om = sc->om[i - 1];
  }
  const double den = sc->rho[i - 1];
  const double denm = i >= 2 ? sc->rho[i - 2] : 1.0;
  const double rden = 1.0 / den, rdenm = 1.0 / denm;
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  const int stride = gridDim.x * blockDim.x;
  unsigned peer = 0u;
  auto row = [&](int r, double av, double xi, double xm, unsigned mk) {
    const double vi = (xi) * rden;
    double w = fma(-om, vi, av);
    if (i >= 2) w = fma(-den, (xm) * rdenm, w);  // rho_{i-1} = rho[i-1] = den
    gstore_m(net, Xip1 + rb + r, mk, w);
    peer |= mk;
    xwin_add_nn(acc[0], w * w, err, xb.l[0]);
  };
  if ((rb & 1) == 0) {
    // 16-byte vectors: thread handles row pairs (2p, 2p+1), two pairs in flight
    const int np = nl >> 1;
    const double2 *a2 = reinterpret_cast<const double2 *>(a);
    const double2 *xi2 = reinterpret_cast<const double2 *>(Xi + rb);
    const double2 *xm2 = reinterpret_cast<const double2 *>(Xim1 ? Xim1 + rb : Xi + rb);
    for (int p0 = blockIdx.x * blockDim.x + threadIdx.x; p0 < np; p0 += kBU * stride) {
      double2 av[kBU], xi[kBU], xm[kBU];
      unsigned mk[kBU];
#pragma unroll
      for (int u = 0; u < kBU; ++u) {
        const int p = p0 + u * stride;
        if (p < np) {
          av[u] = __ldcs(&a2[p]);  // a is dead after this step: evict first
          xi[u] = xi2[p];
          xm[u] = i >= 2 ? xm2[p] : make_double2(0.0, 0.0);
          mk[u] = net.mask ? (unsigned)reinterpret_cast<const unsigned short *>(net.mask)[p] : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < kBU; ++u) {
        const int p = p0 + u * stride;
        if (p < np) {
          row(2 * p, av[u].x, xi[u].x, xm[u].x, mk[u] & 0xffu);
          row(2 * p + 1, av[u].y, xi[u].y, xm[u].y, mk[u] >> 8);
        }
      }
    }
    if ((nl & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const int r = nl - 1;
      row(r, a[r], Xi[rb + r], i >= 2 ? Xim1[rb + r] : 0.0, gmask(net, r));
    }
  } else {
    for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < nl; r0 += 4 * stride) {
      double av[4], xi[4], xm[4];
      unsigned mk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * stride;
        if (r < nl) {
          av[u] = a[r];
          xi[u] = Xi[rb + r];
          xm[u] = i >= 2 ? Xim1[rb + r] : 0.0;
          mk[u] = gmask(net, r);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + u * stride;
        if (r < nl) row(r, av[u], xi[u], xm[u], mk[u]);
      }
    }
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, peer) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = i;
    emit<1>(slot, sc, net, FK_RHO, f, nullptr);
  }
}

// ---------------------------------------------------------------- fused Lanczos pass 1
// Alg. 2 lines 1-9, all q steps in ONE persistent launch (one GPU): step i is phase A
// (a = D_t v_i, omega_i = <v_i, a>: the k_lanczos_a work) and phase B (w_{i+1} =
// a - omega_i v_i - rho_{i-1} v_{i-1}, rho_i = ||w_{i+1}||: the k_lanczos_b work), each closed
// by a grid barrier built on the exact-sum ticket: the last block to commit finalizes the sum
// (emit, the same code and bits as the two-kernel path) and releases a monotonic flag that the
// other blocks' thread 0 waits for (acquire; the fence also invalidates this SM's L1, so the
// next phase's loads see the other blocks' stores).  The grid is co-resident (cooperative
// launch).  A barrier that does not open within ~2^34 cycles sets sc->err |= 4 and ends the
// kernel instead of hanging.  Per-row arithmetic and every exact sum are those of
// k_lanczos_a / k_lanczos_b: bitwise the same iterates.
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool UNI>
__global__ void __launch_bounds__(kBlockA, UNI ? kMinBlocksUni : 2)
    k_lanczos_pass1(Csr C, Rows RL, const double *__restrict__ d, double *G, double *W1, long long npad, int store, int q,
                    int nl, double *a, XSlot *slot_om, XSlot *slot_rho, DevScalars *sc, Net net,
                    unsigned long long *gflag, unsigned long long ebase) {
  pdl_entry();
  __shared__ XBlk<1> xb;
  __shared__ int s_go;
  auto vslot = [&](int j) -> double * {  // buffer of w_j (the host's slot(s, j)); w_1 = W1
    if (j == 1) return W1;
    if (store) return G + (long long)j * npad;
    return G + (long long)(2 + (j & 1)) * npad;
  };
  unsigned long long ph = ebase;
  // close a phase: the last block finalizes (fin) and opens the barrier, the others wait
  auto barrier = [&](bool last, auto fin) -> bool {
    ++ph;
    if (last) {
      if (threadIdx.x == 0) {
        fin();
        st_release_gpu(gflag, ph);
      }
      __syncthreads();
      return true;
    }
    if (threadIdx.x == 0) {
      int ok = 1;
      const long long t0 = clock64();
      while (ld_acquire_gpu(gflag) < ph) {
        if (clock64() - t0 > (1ll << 34)) {
          atomicOr(&sc->err, 4);
          ok = 0;
          break;
        }
        __nanosleep(64);
      }
      s_go = ok;
    }
    __syncthreads();
    return s_go != 0;
  };
  for (int i = 1; i <= q; ++i) {
    if (sc->brk) break;  // Alg. 2 line 8 break (read after the barrier: the same on every block)
    // ---- phase A (k_lanczos_a)
    {
      const double den = sc->rho[i - 1];
      xblk_init<1>(xb);
      EpiA epi;
      epi.a = a;
      epi.blk = xb.l[0];
      xwin_init(epi.acc[0]);
      epi.err = 0;
      spmv_rows<1, UNI>(C, RL, vslot(i), den, d, nullptr, 0, nl, epi);
      int err = epi.err;
      XWin (&acc)[1] = epi.acc;
      const bool last = commit_and_ticket<1>(acc, xb, slot_om, err, sc, 1, 0u);
      if (!barrier(last, [&]() {
            if (RL.work) *RL.work = 0u;
            FinArgs f{};
            f.i = i;
            emit<1>(slot_om, sc, net, FK_OM, f, nullptr);
          }))
        return;
    }
    if (i == q) break;
    // ---- phase B (k_lanczos_b, vector path: one GPU, rb = 0)
    {
      const double om = sc->om[i - 1];
      const double den = sc->rho[i - 1];
      const double denm = i >= 2 ? sc->rho[i - 2] : 1.0;
      const double rden = 1.0 / den, rdenm = 1.0 / denm;
      const double *Xi = vslot(i);
      const double *Xim1 = i >= 2 ? vslot(i - 1) : nullptr;
      double *Xip1 = vslot(i + 1);
      xblk_init<1>(xb);
      XWin acc[1];
      xwin_init(acc[0]);
      int err = 0;
      const int stride = gridDim.x * blockDim.x;
      auto row = [&](int r, double av, double xi, double xm) {
        const double vi = (xi) * rden;
        double w = fma(-om, vi, av);
        if (i >= 2) w = fma(-den, (xm) * rdenm, w);  // rho_{i-1} = rho[i-1] = den
        Xip1[r] = w;
        xwin_add_nn(acc[0], w * w, err, xb.l[0]);
      };
      const double2 *a2 = reinterpret_cast<const double2 *>(a);
      const double2 *xi2 = reinterpret_cast<const double2 *>(Xi);
      const double2 *xm2 = reinterpret_cast<const double2 *>(Xim1 ? Xim1 : Xi);
      // this block's phase-A rows (static slice ranges), walked backwards: the a / v_i entries
      // phase A touched last are still in L2, and the next phase A meets w_{i+1}'s last-written
      // rows first (any order: the rho sum is exact)
      const int per = (RL.nslice + gridDim.x - 1) / gridDim.x;
      const int pb = (int)min((long long)nl, (long long)blockIdx.x * per * 32) >> 1;
      const int pe = (int)min((long long)nl, (long long)(blockIdx.x + 1) * per * 32) >> 1;
      if (RL.work == nullptr) {
#pragma unroll 2
        for (int p = pe - 1 - (int)threadIdx.x; p >= pb; p -= blockDim.x) {
          const double2 av = __ldcs(&a2[p]);
          const double2 xv = xi2[p];
          const double2 xm = i >= 2 ? xm2[p] : make_double2(0.0, 0.0);
          row(2 * p, av.x, xv.x, xm.x);
          row(2 * p + 1, av.y, xv.y, xm.y);
        }
      } else {  // dynamic slice distribution in phase A: plain grid-stride pairs
        const int np = nl >> 1;
        for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += stride) {
          const double2 av = __ldcs(&a2[p]);
          const double2 xv = xi2[p];
          const double2 xm = i >= 2 ? xm2[p] : make_double2(0.0, 0.0);
          row(2 * p, av.x, xv.x, xm.x);
          row(2 * p + 1, av.y, xv.y, xm.y);
        }
      }
      if ((nl & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int r = nl - 1;
        row(r, a[r], Xi[r], i >= 2 ? Xim1[r] : 0.0);
      }
      const bool last = commit_and_ticket<1>(acc, xb, slot_rho, err, sc, 1, 0u);
      if (!barrier(last, [&]() {
            FinArgs f{};
            f.i = i;
            emit<1>(slot_rho, sc, net, FK_RHO, f, nullptr);
          }))
        return;
    }
  }
}

// TMA-staged variant of k_lanczos_b (the same arithmetic, row by row): tiles of kBT rows of
// a, X_i and X_{i-1} are bulk-copied (cp.async.bulk, mbarrier completion) into shared
// memory, kBS stages deep, by one thread; the block computes the tile from shared memory.
// The bytes in flight live in shared memory, not registers, so the exact-sum window keeps
// its registers without limiting the memory-level parallelism.
constexpr int kBT = 2048;  // rows per tile
constexpr int kBS = 3;     // stages
struct __align__(16) BStage {
  double a[kBT + 2], xi[kBT + 4], xm[kBT + 4];
};
struct __align__(16) BSmem {
  BStage st[kBS];
  unsigned long long bar[kBS];
};

__global__ void __launch_bounds__(kBlock, 2) k_lanczos_b_tma(const double *__restrict__ a, const double *Xi,
                                                            const double *Xim1, double *Xip1, int nl, long long rb,
                                                            int i, XSlot *slot, DevScalars *sc, Net net) {
  pdl_entry();
  if (sc->brk) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  BSmem &sm = *reinterpret_cast<BSmem *>(smraw);
  const double om = sc->om[i - 1];
  const double den = sc->rho[i - 1];
  const double denm = i >= 2 ? sc->rho[i - 2] : 1.0;
  const double rden = 1.0 / den, rdenm = 1.0 / denm;
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  const int ntile = (nl + kBT - 1) / kBT;
  const int J = ntile > (int)blockIdx.x ? (ntile - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto tile = [&](int j) { return (int)blockIdx.x + j * (int)gridDim.x; };
  auto issue = [&](int j, int q) {
    const long long r0 = (long long)tile(j) * kBT, r1 = min((long long)nl, r0 + kBT);
    uint32_t bytes = seg_bytes<8>(r0, r1) + seg_bytes<8>(rb + r0, rb + r1);
    if (i >= 2) bytes += seg_bytes<8>(rb + r0, rb + r1);
    mbar_arrive_tx(&sm.bar[q], bytes);
    bulk_seg<8>(sm.st[q].a, a, r0, r1, &sm.bar[q]);
    bulk_seg<8>(sm.st[q].xi, Xi, rb + r0, rb + r1, &sm.bar[q]);
    if (i >= 2) bulk_seg<8>(sm.st[q].xm, Xim1, rb + r0, rb + r1, &sm.bar[q]);
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < kBS; ++q) mbar_init(&sm.bar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < kBS && q < J; ++q) issue(q, q);
  for (int j = 0; j < J; ++j) {
    const int q = j % kBS;
    mbar_wait(&sm.bar[q], (uint32_t)((j / kBS) & 1));
    const long long r0 = (long long)tile(j) * kBT;
    const int nr = (int)min((long long)kBT, (long long)nl - r0);
    const double *ap = sm.st[q].a + seg_shift<8>(r0);
    const double *xp = sm.st[q].xi + seg_shift<8>(rb + r0);
    const double *mp = sm.st[q].xm + seg_shift<8>(rb + r0);
    for (int u = threadIdx.x; u < nr; u += blockDim.x) {
      const int r = (int)r0 + u;
      const double vi = (xp[u]) * rden;
      double w = fma(-om, vi, ap[u]);
      if (i >= 2) w = fma(-den, (mp[u]) * rdenm, w);  // rho_{i-1} = rho[i-1] = den
      gstore(net, Xip1 + rb + r, r, w);
      xwin_add_nn(acc[0], w * w, err, xb.l[0]);
    }
    __syncthreads();  // stage q consumed
    if (threadIdx.x == 0 && j + kBS < J) issue(j + kBS, q);
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = i;
    emit<1>(slot, sc, net, FK_RHO, f, nullptr);
  }
}

// ---------------------------------------------------------------- tridiagonal (CAC-5)
__device__ int sturm_count(const double *om, const double *rho2, int k, double x) {
  double pprev = 1.0, p = om[0] - x;
  int sprev = 1;
  int s = p > 0.0 ? 1 : (p < 0.0 ? -1 : -sprev);
  int cnt = (s != sprev);
  for (int j = 1; j < k; ++j) {
    const double pn = fma(om[j] - x, p, -(rho2[j - 1] * pprev));
    const int sn = pn > 0.0 ? 1 : (pn < 0.0 ? -1 : -s);
    cnt += (sn != s);
    pprev = p;
    p = pn;
    s = sn;
    // rescale by 2^-500 / 2^500 when the sequence leaves [2^-500, 2^500]: branch-free (every lane has
    // its own x, a branch would diverge); a multiplication by 1.0 is exact, so the bits are those of
    // the branching form
    const double ap = fabs(p), aq = fabs(pprev);
    const double f = ap > 0x1p500 ? 0x1p-500 : ((ap < 0x1p-500 && aq < 0x1p-500) ? 0x1p500 : 1.0);
    p *= f;
    pprev *= f;
  }
  return cnt;
}

// One warp: multisection (32 Sturm counts per round, one per lane) for theta, then
// inverse iteration (lane 0, partial pivoting) for s (Alg. 2 lines 11-12).
struct TriScratch {  // shared-memory working arrays of one tridiagonal solve
  double om[kMaxQ], rho[kMaxQ], rho2[kMaxQ], u0[kMaxQ], u1[kMaxQ], u2[kMaxQ], mul[kMaxQ], xv[kMaxQ], s[kMaxQ],
      ru0[kMaxQ];
  int swp[kMaxQ];
  unsigned char uok[kMaxQ];  // u0[i] inside the range where the shared-divisor division is exact
};

// Warp reductions that return, on every lane, exactly what a left-to-right scan over j = 0..k-1
// returns: the first (lowest j) extreme value; v, j hold the lane's own scan result (j = -1: none).
__device__ __forceinline__ void warp_first_min(double &v, int &j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (oj >= 0 && (j < 0 || ov < v || (ov == v && oj < j))) { v = ov; j = oj; }
  }
}
__device__ __forceinline__ void warp_first_max(double &v, int &j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (oj >= 0 && (j < 0 || ov > v || (ov == v && oj < j))) { v = ov; j = oj; }
  }
}

// CAC-5 on one full warp (lanes 0..31 of the calling warp); sc may live in shared memory.  The
// arithmetic is the sequential algorithm's, operation for operation: the independent parts (the
// Gershgorin bounds, the 32 Sturm counts of a multisection round, 1/u0, the initial vector, the
// max-norm rescaling, the sign fix) are spread over the lanes -- exact min / max scans keep the
// first extreme, like the sequential scan -- and the three dependent recurrences (the pivoted LU,
// forward elimination and back substitution) run on lane 0 with their running values in registers.
__device__ __noinline__ void tridiag_warp(DevScalars *sc, int q, TriScratch &T) {
  double *om = T.om, *rho = T.rho, *rho2 = T.rho2;
  const int lane = threadIdx.x & 31;
  const int k = sc->brk ? sc->k : q;
  for (int j = lane; j < k; j += 32) om[j] = sc->om[j];
  for (int j = lane; j < k - 1; j += 32) { rho[j] = sc->rho[j + 1]; rho2[j] = rho[j] * rho[j]; }
  __syncwarp();
  if (k == 1) {
    if (lane == 0) { sc->theta = om[0]; sc->s[0] = 1.0; sc->k = 1; }
    return;
  }
  // Gershgorin interval: lo = min_j (om_j - r_j), hi = max_j (om_j + r_j), exact
  double lo = 0.0, hi = 0.0;
  int jl = -1, jh = -1;
  for (int j = lane; j < k; j += 32) {
    const double rl = j > 0 ? rho[j - 1] : 0.0;
    const double rr = j < k - 1 ? rho[j] : 0.0;
    const double rj = rl + rr;
    const double a = om[j] - rj, b = om[j] + rj;
    if (jl < 0 || a < lo) { lo = a; jl = j; }
    if (jh < 0 || b > hi) { hi = b; jh = j; }
  }
  warp_first_min(lo, jl);
  warp_first_max(hi, jh);
  const double NT = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
  if (NT == 0.0) {
    for (int j = lane; j < k; j += 32) sc->s[j] = j == 0 ? 1.0 : 0.0;
    if (lane == 0) { sc->theta = 0.0; sc->k = k; }
    return;
  }
  const double pad = NT * 0x1p-20;
  lo = lo - pad;
  hi = hi + pad;
  for (int round = 0; round < 12; ++round) {
    const double h = (hi - lo) / 33.0;
    const double x = fma((double)(lane + 1), h, lo);
    const int c = sturm_count(om, rho2, k, x);
    const unsigned mask = __ballot_sync(0xffffffffu, c >= 1);
    const double xm1 = __shfl_up_sync(0xffffffffu, x, 1);
    if (mask) {
      const int f = __ffs(mask) - 1;  // first lane (lowest point) with count >= 1
      const double nhi = __shfl_sync(0xffffffffu, x, f);
      const double prevx = __shfl_sync(0xffffffffu, xm1, f);
      const double nlo = f == 0 ? lo : prevx;
      lo = nlo;
      hi = nhi;
    } else {
      lo = __shfl_sync(0xffffffffu, x, 31);
    }
  }
  const double th = (lo + hi) * 0.5;
  double *u0 = T.u0, *u1 = T.u1, *u2 = T.u2, *mul = T.mul, *xv = T.xv, *s = T.s, *ru0 = T.ru0;
  int *swp = T.swp;
  const double tiny = NT * 0x1p-60;
  if (lane == 0) {  // Gaussian elimination with partial pivoting of T - theta I (three upper diagonals)
    sc->theta = th;
    double c0 = om[0] - th, c1 = rho[0], c2 = 0.0;
#pragma unroll 4
    for (int i = 0; i < k - 1; ++i) {
      const double nb = rho[i], na = om[i + 1] - th, nc = (i + 1 < k - 1) ? rho[i + 1] : 0.0;
      if (fabs(c0) >= fabs(nb)) {
        const double m = c0 != 0.0 ? nb / c0 : 0.0;
        u0[i] = c0; u1[i] = c1; u2[i] = c2; swp[i] = 0; mul[i] = m;
        c0 = na - m * c1;
        c1 = nc - m * c2;
        c2 = 0.0;
      } else {
        const double m = c0 / nb;
        u0[i] = nb; u1[i] = na; u2[i] = nc; swp[i] = 1; mul[i] = m;
        const double t0 = c1 - m * na, t1 = c2 - m * nc;
        c0 = t0;
        c1 = t1;
        c2 = 0.0;
      }
    }
    u0[k - 1] = c0; u1[k - 1] = 0.0; u2[k - 1] = 0.0;
  }
  __syncwarp();
  // pivot clamp; the three back substitutions divide by the same pivots: RN(1/u0) once, then the
  // shared-divisor IEEE division div_rn (bitwise RN(t/u0) for normal-range operands, self-tested;
  // hardware division outside that range)
  for (int i = lane; i < k; i += 32) {
    double u = u0[i];
    if (fabs(u) < tiny) u = u < 0.0 ? -tiny : tiny;
    u0[i] = u;
    ru0[i] = 1.0 / u;
    const double au = fabs(u);
    T.uok[i] = au > 0x1p-400 && au < 0x1p400;
  }
  for (int j = lane; j < k; j += 32) s[j] = (double)(j % 5 + 1) * 0.25;
  __syncwarp();
  for (int it = 0; it < 3; ++it) {
    for (int j = lane; j < k; j += 32) xv[j] = s[j];
    __syncwarp();
    if (lane == 0) {
      // forward elimination: a = the running entry i, b = entry i+1
      double a = xv[0];
#pragma unroll 4
      for (int i = 0; i < k - 1; ++i) {
        double b = xv[i + 1];
        if (swp[i]) { const double t = a; a = b; b = t; }
        xv[i] = a;
        a = fma(-mul[i], a, b);
      }
      xv[k - 1] = a;
      // back substitution: x1, x2 = the new entries i+1, i+2
      double x1 = 0.0, x2 = 0.0;
#pragma unroll 4
      for (int i = k - 1; i >= 0; --i) {
        double t = xv[i];
        if (i + 1 < k) t = fma(-u1[i], x1, t);
        if (i + 2 < k) t = fma(-u2[i], x2, t);
        const double at = fabs(t);
        double r = div_rn(t, u0[i], ru0[i]);
        if (!(at > 0x1p-400 && at < 0x1p400 && T.uok[i])) r = t / u0[i];  // (rare: outside the exact range)
        xv[i] = r;
        x2 = x1;
        x1 = r;
      }
    }
    __syncwarp();
    double mx = 0.0;
    for (int j = lane; j < k; j += 32) mx = fabs(xv[j]) > mx ? fabs(xv[j]) : mx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double om2 = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = om2 > mx ? om2 : mx;
    }
    const double p2 = __longlong_as_double(__double_as_longlong(mx) & 0x7ff0000000000000ll);
    const double sc2 = 1.0 / p2;
    for (int j = lane; j < k; j += 32) s[j] = xv[j] * sc2;
    __syncwarp();
  }
  // sign: the largest |s_j| (first on ties) positive
  double am = -1.0;
  int jm = -1;
  for (int j = lane; j < k; j += 32)
    if (jm < 0 || fabs(s[j]) > am) { am = fabs(s[j]); jm = j; }
  warp_first_max(am, jm);
  const bool neg = s[jm] < 0.0;
  for (int j = lane; j < k; j += 32) sc->s[j] = neg ? -s[j] : s[j];
  if (lane == 0) sc->k = k;
}

__global__ void k_tridiag(DevScalars *sc, int q) {
  pdl_entry();
  __shared__ TriScratch T;
  tridiag_warp(sc, q, T);
}

// ---------------------------------------------------------------- Lanczos pass 2
// Step j (Alg. 2 line 13 "regenerate v_2..v_i and form sum"): regenerate w_{j+1}
// bitwise as in pass 1, v_{j+1} = w_{j+1} / rho_j, x += s_{j+1} v_{j+1}.
struct EpiC {
  const double *Xjm1;
  double *Xjp1, *x;
  long long rb;
  const Net *net;
  int j;
  double om, den, denm, rhoj, s1, sj1, rrhoj, rdenm;
  __device__ __forceinline__ void operator()(const RowOut<1> &o) {
    const double vj = o.xr;
    double w = fma(-om, vj, o.s[0]);
    if (j >= 2) w = fma(-den, Xjm1[rb + o.r] * rdenm, w);
    gstore(*net, Xjp1 + rb + o.r, o.r, w);
    const double vn = (w) * rrhoj;
    const double xr = j == 1 ? s1 * vj : x[rb + o.r];
    x[rb + o.r] = fma(sj1, vn, xr);
  }
};

template <bool UNI, int W>
__global__ void __launch_bounds__(kBlock, W > 0 ? ell_min_blocks(W, UNI) : (UNI ? kMinBlocksUni : 2)) k_lanczos_c(Csr C, Rows RL, const double *__restrict__ d,
                                                         const double *__restrict__ Xj, const double *Xjm1,
                                                         double *Xjp1, double *__restrict__ x, int nl, long long rb,
                                                         int j, DevScalars *sc, XSlot *slot, Net net) {
  pdl_entry();
  if (j >= sc->k) return;  // sc->k holds the effective k after k_tridiag
  EpiC epi{Xjm1, Xjp1, x, rb, &net, j, sc->om[j - 1], sc->rho[j - 1], j >= 2 ? sc->rho[j - 2] : 1.0, sc->rho[j],
           sc->s[0], sc->s[j], 1.0 / sc->rho[j], 1.0 / (j >= 2 ? sc->rho[j - 2] : 1.0)};
  spmv_any<1, UNI, W>(C, RL, Xj, epi.den, d, nullptr, rb, nl, epi);
  // P > 1: the next step gathers w_{j+1} -- a barrier collective (no sums)
  if (net.P > 1 && ticket_only(slot) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = j;
    emit<0>(slot, sc, net, FK_BAR, f, nullptr);
  }
}

// Stored-vector mode (Remark "Time-storage tradeoff"): the
// Lanczos vectors w_j kept by pass 1 (slot j-1 of Wst, leading dimension ldw)
// replace the pass-2 regeneration: x = s_1 v_1 + sum_j fma(s_j, v_j, .), v_j = w_j / rho_{j-1},
// bitwise equal to the two-pass result; then ||x||^2 (exact).
__global__ void __launch_bounds__(kBlock, 4) k_combine(const double *__restrict__ W1, const double *__restrict__ Wst,
                                                       long long ldw,
                                                       double *__restrict__ x, int nl, long long rb, XSlot *slot,
                                                       DevScalars *sc, Net net) {
  pdl_entry();
  __shared__ double s_s[kMaxQ], s_rr[kMaxQ];
  const int k = sc->k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    s_s[j] = sc->s[j];
    s_rr[j] = 1.0 / sc->rho[j];
  }
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  unsigned peer = 0u;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const unsigned mk = gmask(net, r);  // issued with the row's loads
    const double *w = Wst + rb + r;  // w_{j+1} at slot j (j >= 1); w_1 = the start vector in W1
    double xr = s_s[0] * (__ldg(W1 + rb + r) * s_rr[0]);
    int j = 1;
    for (; j + 4 <= k; j += 4) {
      double wv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) wv[u] = __ldg(w + (long long)(j + u) * ldw);
#pragma unroll
      for (int u = 0; u < 4; ++u) xr = fma(s_s[j + u], (wv[u]) * s_rr[j + u], xr);
    }
    for (; j < k; ++j) xr = fma(s_s[j], __ldg(w + (long long)j * ldw) * s_rr[j], xr);
    gstore_m(net, x + rb + r, mk, xr);
    peer |= mk;
    xwin_add_nn(acc[0], xr * xr, err, xb.l[0]);
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, peer) && threadIdx.x == 0)
    emit<1>(slot, sc, net, FK_NUX, FinArgs{}, nullptr);
}

// ||x||^2 (exact); k == 1 case: x = s_1 v_1.
__global__ void __launch_bounds__(kBlock) k_norm_x(const double *__restrict__ g, double *__restrict__ x, int nl,
                                                   long long rb, XSlot *slot, DevScalars *sc, Net net) {
  pdl_entry();
  const bool k1 = sc->k == 1;
  const double s1 = sc->s[0], rden = 1.0 / sc->rho[0];
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  const int stride = gridDim.x * blockDim.x;
  for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < nl; r0 += 4 * stride) {
    double xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = r0 + u * stride;
      if (r < nl) xv[u] = k1 ? g[rb + r] : x[rb + r];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = r0 + u * stride;
      if (r < nl) {
        double xr = xv[u];
        if (k1) xr = s1 * (xr * rden);
        if (k1 || net.P > 1) gstore(net, x + rb + r, r, xr);  // P > 1: publish x's halo for the monitor
        xwin_add_nn(acc[0], xr * xr, err, xb.l[0]);
      }
    }
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P) && threadIdx.x == 0)
    emit<1>(slot, sc, net, FK_NUX, FinArgs{}, nullptr);
}

// Monitor matvec: v = x / ||x|| (written), xi = v.(D v), c = v.(C v), ||v||^2 (exact).
// (eqn 5.1 PAPER.md:1382; objective tracker PAPER.md:1553; tau PAPER.md:3224.)
struct EpiM {
  double *v;
  long long (*blk)[kLimbs];
  XWin acc[3];
  int err;
  __device__ __forceinline__ void operator()(const RowOut<2> &o) {
    v[o.r] = o.xr;
    xwin_add(acc[0], o.xr * o.s[0], err, blk[0]);
    xwin_add(acc[1], o.xr * o.s[1], err, blk[1]);
    xwin_add_nn(acc[2], o.xr * o.xr, err, blk[2]);
  }
};

template <bool UNI, int W>
__global__ void __launch_bounds__(kBlock, 2) k_monitor(Csr C, Rows RL, const double *__restrict__ d,
                                                       const double *__restrict__ cdiag, const double *__restrict__ x,
                                                       double *__restrict__ v, int nl, long long rb, XSlot *slot,
                                                       DevScalars *sc, Net net) {
  pdl_entry();
  const double nu = sc->nu_x;
  __shared__ XBlk<3> xb;
  xblk_init<3>(xb);
  EpiM epi;
  epi.v = v;
  epi.blk = xb.l;
  xwin_init(epi.acc[0]);
  xwin_init(epi.acc[1]);
  xwin_init(epi.acc[2]);
  epi.err = 0;
  spmv_any<2, UNI, W>(C, RL, x, nu, d, cdiag, rb, nl, epi);
  int err = epi.err;
  XWin (&acc)[3] = epi.acc;
  if (commit_and_ticket<3>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    if (RL.work) *RL.work = 0u;  // every warp has stopped taking chunks
    emit<3>(slot, sc, net, FK_MON, FinArgs{}, nullptr);
  }
}

// ---------------------------------------------------------------- primal / dual / sketch
// z <- (1-eta) z + eta alpha (v o v) (Alg. 4 line 8, primitive 3), ||z - b||^2 (exact),
// per-block partials of g = v^T Omega (fp64, fixed tree; off the feedback path).
// The projection onto the constraint set K of the point p = fl(z + fl(y / beta)): KS = 1 box
// (min / max, reading R32), KS = 2 l2 ball with the scale s and the inside flag of the exact-sum
// norm pass (k_ball_sum, reading R34), KS = 3 l1 ball with the threshold s of the exact bisection
// (k_l1_pass, reading R35).
template <int KS>
__device__ __forceinline__ double proj_k(double zr, double yr, double beta, const IterArgs &A, double s, int inside) {
  const double p = zr + yr / beta;
  if (KS == 1) return fmin(fmax(p, A.lo), A.hi);
  if (inside) return p;
  const double e = p - A.b;
  if (KS == 3) return A.b + copysign(fmax(fabs(e) - s, 0.0), e);  // l1: soft threshold s = theta (R35)
  return A.b + s * e;
}

template <int KS>  // constraint set: 0 A X = b, 1 box (A.ineq), 2/3 l2/l1 ball (nz in k_ball_nz)
__global__ void __launch_bounds__(kBlock, 2) k_primal(const double *__restrict__ v, double *__restrict__ z,
                                                   const double *__restrict__ y,
                                                   const double *__restrict__ Om, int nl, int R, IterArgs A,
                                                   double *__restrict__ gpart, XSlot *slot, DevScalars *sc,
                                                   scg_iter_rec *log, Net net) {
  pdl_entry();
  const bool hoff = A.trace_le && !(sc->xi < 0.0);
  __shared__ double red[kBlock / 32][kMaxR];
  // exact sums: ||z_{t+1} - b||^2 (or - wbar_t); A X = b: also sum z_{t+1}, z_{t+1}.z_{t+1} (the next
  // iteration's gap / bound, FK_NZZ; summed here, where z_{t+1} is formed, instead of in the dual step)
  constexpr int NS = KS == 0 ? 3 : 1;
  __shared__ XBlk<NS> xb;
  xblk_init<NS>(xb);
  XWin acc[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) xwin_init(acc[q]);
  int err = 0;
  // thread-per-row; per-thread partial g_k for 16 columns at a time
  constexpr int kPR = 1;
  const int stride = gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int kc = 0; kc < R; kc += 16) {
    double gp[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) gp[u] = 0.0;
    for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < nl; r0 += kPR * stride) {
      double vr[kPR], zv[kPR], om[kPR][16];
#pragma unroll
      for (int h = 0; h < kPR; ++h) {
        const int r = r0 + h * stride;
        vr[h] = r < nl ? v[r] : 0.0;
        zv[h] = (kc == 0 && r < nl) ? z[r] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) om[h][u] = (r < nl && kc + u < R) ? __ldg(&Om[(long long)(kc + u) * nl + r]) : 0.0;
      }
#pragma unroll
      for (int h = 0; h < kPR; ++h) {
        const int r = r0 + h * stride;
        if (r < nl) {
          if (kc == 0) {
            const double hv = A.alpha * (vr[h] * vr[h]);
            // trace-bounded LMO with xi_t >= 0: H = 0
            const double zr = hoff ? A.one_m_eta * zv[h] : fma(A.eta, hv, A.one_m_eta * zv[h]);
            z[r] = zr;
            // z_{t+1} - b, or z_{t+1} - wbar_t, wbar_t = proj_K(z_{t+1} + y_t / beta_{t+1})
            if (KS < 2) {
              const double e = zr - (KS == 1 ? proj_k<1>(zr, y[r], A.beta_next, A, 0.0, 0) : A.b);
              xwin_add_nn(acc[0], e * e, err, xb.l[0]);
            }
            if (KS == 0) {
              xwin_add_nn(acc[NS - 2], zr, err, xb.l[NS - 2]);  // z >= 0 (convex combination of alpha v o v)
              xwin_add_nn(acc[NS - 1], zr * zr, err, xb.l[NS - 1]);
            }
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) gp[u] = fma(vr[h], om[h][u], gp[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      double t = gp[u];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
      if (lane == 0 && kc + u < R) red[warp][kc + u] = t;
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < R) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t += red[w][threadIdx.x];
    gpart[(long long)blockIdx.x * R + threadIdx.x] = t;
  }
  __syncthreads();
  if (commit_and_ticket<NS>(acc, xb, slot, err, sc, net.P, 0u)) {
    __shared__ double gsum[kMaxR];
    // sum block partials in a fixed order: thread k sums column k over blocks
    if (threadIdx.x < R) {
      double t = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(&gpart[(long long)b * R + threadIdx.x]);
      gsum[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      FinArgs f{};
      f.R = R;
      f.A = A;
      f.log = log;
      emit<NS>(slot, sc, net, KS >= 2 ? FK_GK : (KS == 0 ? FK_NZZ : FK_NZ), f, gsum);
    }
  }
}

// y <- y + gamma (z - b) (Alg. 4 line 9); d for t+1; GEN: also the next start vector g_{t+1} and
// ||g_{t+1}||^2 (exact) -- otherwise g_{t+1} was drawn ahead on the side stream (k_gen_start, FK_GEN)
// and only its norm is taken over.  The sketch update of Alg. 4 line 10 is deferred (k_sketch_flush):
// this kernel records its coefficients ck = fl(eta alpha) g_k in the ring slot js.
template <int KS, bool GEN>  // constraint set: 0 A X = b, 1 box, 2/3 l2/l1 ball (d and gap sums in k_ball_d)
__global__ void __launch_bounds__(kBlock, GEN ? 2 : 4) k_dual_sketch(const double *__restrict__ z, double *__restrict__ y,
                                                        double *__restrict__ d, const double *__restrict__ cdiag,
                                                        double *__restrict__ ckr, int js,
                                                        double *__restrict__ g, int nl, long long rb, int R,
                                                        IterArgs A, uint64_t seed, XSlot *slot, DevScalars *sc,
                                                        Net net, const int *__restrict__ orig) {
  pdl_entry();
  const double gam = sc->gamma;
  const double bs0 = KS >= 2 ? sc->bs[0] : 0.0;  // balls: projection of wbar_t (j = 0)
  const int bin0 = KS >= 2 ? sc->bin[0] : 0;
  if (blockIdx.x == 0 && (int)threadIdx.x < R)  // H = 0 (trace-bounded, xi_t >= 0): no rank-one term
    ckr[js * kMaxR + threadIdx.x] = (A.trace_le && !(sc->xi < 0.0)) ? 0.0 : (A.eta * A.alpha) * sc->gk[threadIdx.x];
  // exact sums: [GEN: ||g_{t+1}||^2,] and over the next iteration's state (y_{t+1}, z_{t+1}) for the
  // surrogate gap / stopping rule (finalize FK_NZ): A X = b sum y, y.z (z.z, sum z: k_primal); box
  // the four general-template dots
  constexpr int NS = (GEN ? 1 : 0) + (KS >= 2 ? 0 : (KS == 1 ? 4 : 2)), o = GEN ? 1 : 0;
  __shared__ XBlk<NS> xb;
  xblk_init<NS>(xb);
  XWin acc[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) xwin_init(acc[q]);
  int err = 0;
  unsigned peer = 0u;
  const int stride = gridDim.x * blockDim.x;
  for (int r0 = blockIdx.x * blockDim.x + threadIdx.x; r0 < nl; r0 += 2 * stride) {
    double zr[2], yv[2], cd[2];
    int og[2];
    unsigned mk[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = r0 + u * stride;
      if (r < nl) {
        zr[u] = z[r];
        yv[u] = y[r];
        cd[u] = cdiag[r];
        if (GEN) { og[u] = orig[r]; mk[u] = gmask(net, r); }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = r0 + u * stride;
      if (r < nl) {
        // dual update with wbar_t (b when A X = b) and the next diagonal with w_{t+1}
        const double e = zr[u] - (KS ? proj_k<KS>(zr[u], yv[u], A.beta_next, A, bs0, bin0) : A.b);
        const double yr = fma(gam, e, yv[u]);
        y[r] = yr;
        const double e1 = KS == 1 ? zr[u] - proj_k<1>(zr[u], yr, A.beta_next, A, 0.0, 0) : e;
        if (KS < 2) d[r] = fma(A.beta_next, e1, yr) + cd[u];
        if (GEN) {
          const double gv = scg_lanczos_start(seed, A.t + 1, rb + og[u]);
          gstore_m(net, g + rb + r, mk[u], gv);
          peer |= mk[u];
          xwin_add_nn(acc[0], gv * gv, err, xb.l[0]);
        }
        if (KS >= 2) {
          // balls: d and the gap sums follow the projection passes over the new points (k_ball_d)
        } else if (KS == 1) {  // general template (reading R33): <y,z>, <z-w,z>, <y,w>, <z-w,z+w>, w = w_{t+1}
          const double wk = proj_k<1>(zr[u], yr, A.beta_next, A, 0.0, 0);  // (the w of e1 above)
          xwin_add(acc[o + 0], yr * zr[u], err, xb.l[o + 0]);
          xwin_add(acc[o + 1], e1 * zr[u], err, xb.l[o + 1]);
          xwin_add(acc[o + 2], yr * wk, err, xb.l[o + 2]);
          xwin_add(acc[o + 3], e1 * (zr[u] + wk), err, xb.l[o + 3]);
        } else {  // sum y, y.z (sum z and z.z come from k_primal)
          xwin_add(acc[o + 0], yr, err, xb.l[o + 0]);
          xwin_add(acc[o + 1], yr * zr[u], err, xb.l[o + 1]);
        }
      }
    }
  }
  if (commit_and_ticket<NS>(acc, xb, slot, err, sc, net.P, peer) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = (int)((A.t + 1) & 1);
    emit<NS>(slot, sc, net,
             KS >= 2 ? FK_RHO0 : (KS == 1 ? (GEN ? FK_RHO0M : FK_RHO0S) : (GEN ? FK_RHO0Y : FK_RHO0SY)), f, nullptr);
  }
}

// l2 ball (reading R34): N^2 = ||p - b||^2 (exact) of the points p = fl(z + fl(y / beta)), finalized into
// the scale / inside flag of projection j (0: wbar_t of the dual step, 1: w_{t+1} of D_{t+1}).
__global__ void __launch_bounds__(kBlock) k_ball_sum(const double *__restrict__ z, const double *__restrict__ y,
                                                     double beta, int nl, IterArgs A, int j, XSlot *slot,
                                                     DevScalars *sc, Net net) {
  pdl_entry();
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double e = (z[r] + y[r] / beta) - A.b;
    xwin_add_nn(acc[0], e * e, err, xb.l[0]);
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = j;
    f.A = A;
    emit<1>(slot, sc, net, FK_BALLS, f, nullptr);
  }
}

// l1 ball (reading R35): one pass of the exact threshold search for projection j of the points
// p = fl(z + fl(y / beta)), a = |fl(p - b)|.  Pass -1: sum a (inside test, FK_L1S).  Pass >= 0: with v
// the value of the bracket's middle key, sum a and count over a >= v (FK_L1B: G(v) < 0 moves the top).
// 63 passes close the bracket [0, DBL_MAX] to the least key with G < 0: the active set a >= v* is the
// sorted top-rho set of the oracle (G decreasing in v).
__global__ void __launch_bounds__(kBlock) k_l1_pass(const double *__restrict__ z, const double *__restrict__ y,
                                                    double beta, int nl, IterArgs A, int j, int pass, XSlot *slot,
                                                    DevScalars *sc, Net net) {
  pdl_entry();
  __shared__ XBlk<2> xb;
  xblk_init<2>(xb);
  XWin acc[2];
  xwin_init(acc[0]);
  xwin_init(acc[1]);
  int err = 0;
  const bool run = pass < 0 || !sc->bdone;
  const unsigned long long mid = sc->bk[0] + ((sc->bk[1] - sc->bk[0]) >> 1);
  if (run)
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
      const double a = fabs((z[r] + y[r] / beta) - A.b);
      if (pass < 0 || (unsigned long long)__double_as_longlong(a) >= mid) {
        xwin_add_nn(acc[0], a, err, xb.l[0]);
        xwin_add_nn(acc[1], 1.0, err, xb.l[1]);
      }
    }
  if (commit_and_ticket<2>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = j;
    f.A = A;
    emit<2>(slot, sc, net, pass < 0 ? FK_L1S : FK_L1B, f, nullptr);
  }
}

// l2 ball: ||z_{t+1} - wbar_t||^2 (exact) -> the dual step, objective tracker and record (FK_NZ; g was
// finalized by k_primal's FK_GK, so no g payload here).
template <int KS>
__global__ void __launch_bounds__(kBlock) k_ball_nz(const double *__restrict__ z, const double *__restrict__ y, int nl,
                                                    IterArgs A, XSlot *slot, DevScalars *sc, scg_iter_rec *log,
                                                    Net net) {
  pdl_entry();
  const double s = sc->bs[0];
  const int inside = sc->bin[0];
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double e = z[r] - proj_k<KS>(z[r], y[r], A.beta_next, A, s, inside);
    xwin_add_nn(acc[0], e * e, err, xb.l[0]);
  }
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0) {
    FinArgs f{};
    f.R = 0;  // g already in sc->gk
    f.A = A;
    f.log = log;
    emit<1>(slot, sc, net, FK_NZ, f, sc->gk);
  }
}

// l2 ball: d for D_{t+1} with w_{t+1} = proj_K(z_{t+1} + y_{t+1} / beta_{t+1}) and the general-template
// gap / bound sums over the state (y_{t+1}, z_{t+1}, w_{t+1}) (reading R33); also the t = 1 setup.
template <int KS>
__global__ void __launch_bounds__(kBlock) k_ball_d(const double *__restrict__ z, const double *__restrict__ y,
                                                   const double *__restrict__ cdiag, double *__restrict__ d, int nl,
                                                   double beta, IterArgs A, XSlot *slot, DevScalars *sc, Net net) {
  pdl_entry();
  const double s = sc->bs[1];
  const int inside = sc->bin[1];
  __shared__ XBlk<4> xb;
  xblk_init<4>(xb);
  XWin acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xwin_init(acc[q]);
  int err = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double zr = z[r], yr = y[r];
    const double w = proj_k<KS>(zr, yr, beta, A, s, inside);
    const double e = zr - w;
    d[r] = fma(beta, e, yr) + cdiag[r];
    xwin_add(acc[0], yr * zr, err, xb.l[0]);
    xwin_add(acc[1], e * zr, err, xb.l[1]);
    xwin_add(acc[2], yr * w, err, xb.l[2]);
    xwin_add(acc[3], e * (zr + w), err, xb.l[3]);
  }
  if (commit_and_ticket<4>(acc, xb, slot, err, sc, net.P, 0u) && threadIdx.x == 0)
    emit<4>(slot, sc, net, FK_MY4, FinArgs{}, nullptr);
}

// Deferred sketch updates (Alg. 4 line 10, eqn:sketch-update PAPER.md:1162-1169): S is
// write-only between reconstructions, so the last nb rank-one updates
//   S <- (1 - eta_j) S + (eta_j alpha) v_j g_j^T,   j = 0 .. nb-1 in iteration order,
// are applied in one pass over S, element by element in registers with exactly the
// per-iteration operations fma(ck_j[k], v_j[r], fl((1 - eta_j) S[r, k])): bitwise the
// S of one update per iteration, with one read and one write of S per nb iterations.
constexpr int kSketchB = 16;
struct FlushArgs {
  int nb;
  double ome[kSketchB];  // 1 - eta_j
};
__global__ void __launch_bounds__(kBlock) k_sketch_flush(double *__restrict__ S, const double *__restrict__ V,
                                                         long long ldv, const double *__restrict__ ckr, FlushArgs F,
                                                         int nl, int R) {
  pdl_entry();
  __shared__ double ck[kSketchB][kMaxR];
  for (int e = threadIdx.x; e < F.nb * kMaxR; e += blockDim.x) ck[e / kMaxR][e % kMaxR] = ckr[e];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    double vj[kSketchB];
#pragma unroll
    for (int j = 0; j < kSketchB; ++j) vj[j] = j < F.nb ? __ldcs(&V[(long long)j * ldv + r]) : 0.0;
    for (int k0 = 0; k0 < R; k0 += 4) {
      double sv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k0 + k < R) sv[k] = S[(long long)(k0 + k) * nl + r];
#pragma unroll
      for (int j = 0; j < kSketchB; ++j)
        if (j < F.nb) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k0 + k < R) sv[k] = fma(ck[j][k0 + k], vj[j], F.ome[j] * sv[k]);
        }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k0 + k < R) S[(long long)(k0 + k) * nl + r] = sv[k];
    }
  }
}

// ---------------------------------------------------------------- one-shot kernels
// out = (A + beta B) M   (n x R times R x R), row-wise; M in shared memory.
__global__ void k_rowmat(double *__restrict__ out, const double *__restrict__ A, const double *__restrict__ B,
                         double beta, const double *__restrict__ M, int nl, int R) {
  pdl_entry();
  __shared__ double Ms[kMaxR * kMaxR];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Ms[e] = M[e];
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    double row[kMaxR];
    for (int i = 0; i < R; ++i) {
      double a = A[(long long)i * nl + r];
      if (B) a = fma(beta, B[(long long)i * nl + r], a);
      row[i] = a;
    }
    for (int j = 0; j < R; ++j) {
      double s = 0.0;
      for (int i = 0; i < R; ++i) s = fma(row[i], Ms[i * R + j], s);  // M row-major [i][j]
      out[(long long)j * nl + r] = s;
    }
  }
}

// partial[pair][block] of column dot products A[:,i]^T B[:,j]  (pair = i*R + j).
__global__ void k_colpair(const double *__restrict__ A, const double *__restrict__ B, int nl, int R,
                          double *__restrict__ partial) {
  pdl_entry();
  __shared__ double red[kBlock / 32];
  const int pair = blockIdx.y;
  const int i = pair / R, j = pair % R;
  const double *a = A + (long long)i * nl, *b = B + (long long)j * nl;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) s = fma(a[r], b[r], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    partial[(long long)pair * gridDim.x + blockIdx.x] = t;
  }
}

// Per-column quantities of the reconstruction, partial sums per block, for the
// columns k = k0 + blockIdx.y (Ug + blockIdx.y * ldg = column k at GLOBAL indices:
// U itself on one GPU, the gathered copy of one column when sharded):
//   which 0: u_k^T L u_k  (objective)          partial[y][block]
//   which 1: cut weight of sgn(U[:,k])          partial[y][block]
//   which 2: sum_r (diag(X^)_r - 1)^2 with Lam  partial[0][block]
__global__ void k_colstats(const int *__restrict__ rp, const int *__restrict__ col, const double *__restrict__ w,
                           const double *__restrict__ ldiag, const double *__restrict__ U, const double *__restrict__ Ug,
                           long long ldg, int k0, const double *__restrict__ lam, int nl, long long rb, int R,
                           int which, double *__restrict__ partial) {
  pdl_entry();
  __shared__ double red[kBlock / 32];
  const int kcol = k0 + (int)blockIdx.y;
  const double *Ufull = Ug + (long long)blockIdx.y * ldg;
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    if (which == 0) {
      const double ur = U[(long long)kcol * nl + r];
      double lu = ldiag[r] * ur;
      for (int e = rp[r]; e < rp[r + 1]; ++e) lu = fma(-w[e], Ufull[col[e]], lu);
      s = fma(ur, lu, s);
    } else if (which == 1) {
      const bool sr = U[(long long)kcol * nl + r] >= 0.0;
      const long long gr = rb + r;
      for (int e = rp[r]; e < rp[r + 1]; ++e) {
        const int c = col[e];
        if (c > gr) {
          const bool sc_ = Ufull[c] >= 0.0;
          if (sr != sc_) s += w[e];
        } else if (c < rb || c >= rb + nl) {
          // edge to a lower row owned by another rank: counted by that rank
        }
      }
    } else {
      double dx = 0.0;
      for (int k = 0; k < R; ++k) {
        const double u = U[(long long)k * nl + r];
        dx = fma(lam[k], u * u, dx);
      }
      const double e = dx - 1.0;
      s = fma(e, e, s);
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) t += red[ww];
    partial[(long long)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// Sharded reconstruction: gather column k of U (own rows -> this rank's and the
// reader ranks' gathered region at global indices), then a barrier collective.
__global__ void k_push_col(const double *__restrict__ Ucol, double *__restrict__ xg, int nl, long long rb,
                           XSlot *slot, DevScalars *sc, Net net) {
  pdl_entry();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x)
    gstore(net, xg + rb + r, r, Ucol[r]);
  if (ticket_only(slot) && threadIdx.x == 0) {
    FinArgs f{};
    f.i = -1;
    emit<0>(slot, sc, net, FK_BAR, f, nullptr);
  }
}

// y = D x for the current d (diagnostics; same chain order as the Lanczos kernels)
struct EpiY {
  double *y;
  __device__ __forceinline__ void operator()(const RowOut<1> &o) { y[o.r] = o.s[0]; }
};

template <bool UNI, int W>  // W > 0: ELL-W layout, 0: SELL + long rows (the engines of k_lanczos_a)
__global__ void __launch_bounds__(kBlock) k_apply_d(Csr C, Rows RL, const double *__restrict__ d,
                                                    const double *__restrict__ X, int nl, long long rb,
                                                    double *__restrict__ y) {
  pdl_entry();
  EpiY epi{y};
  spmv_any<1, UNI, W>(C, RL, X, 1.0, d, nullptr, rb, nl, epi);
}

// out[orig[r]] = in[r]: device rows back to input order (outputs).
__global__ void k_unperm(double *__restrict__ out, const double *__restrict__ in, const int *__restrict__ orig, int nl) {
  pdl_entry();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) out[orig[r]] = in[r];
}

// Sign rounding of one reconstructed column: chi[orig[r]] = sgn(u[r]) * flip (sgn(0) = +1),
// in input order.
__global__ void k_round_signs(const double *__restrict__ u, const int *__restrict__ orig, int nl, int flip,
                              int8_t *__restrict__ chi) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x)
    chi[orig[r]] = (int8_t)((u[r] >= 0.0 ? 1 : -1) * flip);
}

// One-shot metric (implicit infeasibility, not on the feedback path): per-block partial sums of
// ((z_r - b) unit)^2 in a fixed order; k_sum_partials adds the partials in block order (one block).
__global__ void __launch_bounds__(kBlock) k_sqdist(const double *__restrict__ z, int nl, double b, double unit,
                                                   double *__restrict__ part) {
  __shared__ double red[kBlock / 32];
  double s = 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nl; r += gridDim.x * blockDim.x) {
    const double e = (z[r] - b) * unit;
    s += e * e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void __launch_bounds__(kBlock) k_sum_partials(const double *__restrict__ part, int np, double *out) {
  __shared__ double red[kBlock];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) t += red[i];
    *out = t;
  }
}

// Self-test: div_rn against the hardware IEEE division on pseudo-random operands
// (mantissas drawn uniformly, including the extremes 1 and 2 - ulp), exponents in +-60.
// Exact-sum self-test (sketchycgal_selftest_xsum): the n values through the kernels' per-thread
// accumulators (xwin_add, spills, flush, block and grid commits) and the final rounding.
__global__ void k_selftest_xsum(const double *__restrict__ v, long long n, XSlot *slot, DevScalars *sc,
                                double *out) {
  __shared__ XBlk<1> xb;
  xblk_init<1>(xb);
  XWin acc[1];
  xwin_init(acc[0]);
  int err = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
    xwin_add(acc[0], v[k], err, xb.l[0]);
  if (commit_and_ticket<1>(acc, xb, slot, err, sc, 1, 0u) && threadIdx.x == 0) {
    long long L[kLimbs];
    for (int i = 0; i < kLimbs; ++i) L[i] = __ldcg(&slot->limbs[0][i]);
    *out = xacc_round(L);
  }
}

__global__ void k_selftest_div(long long n, uint64_t seed, unsigned long long *mismatch) {
  pdl_entry();
  unsigned long long bad = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    scg_philox_out o = scg_draw(seed, 77u, 0u, (uint64_t)i);
    unsigned long long ma = ((unsigned long long)o.w[0] << 32 | o.w[1]) & 0x000fffffffffffffull;
    unsigned long long mb = ((unsigned long long)o.w[2] << 32 | o.w[3]) & 0x000fffffffffffffull;
    if ((i & 7) == 1) mb = 0x000fffffffffffffull;  // b = 2 - ulp
    if ((i & 7) == 2) mb = 0;                      // b = power of two
    if ((i & 7) == 3) ma = 0x000fffffffffffffull;
    const int ea = 1023 + (int)(o.w[0] % 121) - 60, eb = 1023 + (int)(o.w[2] % 121) - 60;
    double a = __longlong_as_double((long long)(((unsigned long long)ea << 52) | ma));
    const double b = __longlong_as_double((long long)(((unsigned long long)eb << 52) | mb));
    if (o.w[1] & 1) a = -a;
    if ((i & 1023) == 5) a = 0.0;
    const double q = div_rn(a, b, 1.0 / b);
    const double ref = a / b;
    bad += (__double_as_longlong(q) != __double_as_longlong(ref));
  }
  atomicAdd(mismatch, bad);
}


// ---------------------------------------------------------------- resident cluster kernel (small graphs)
// One whole iteration of Alg. 4 (Lanczos pass 1, tridiagonal eigenpair, stored-vector combine,
// monitor, primal, dual) in ONE launch of ONE thread-block cluster (up to 16 CTAs on 16 SMs), for
// graphs that live in L2 (configs[0], [1]).  The multi-kernel path pays a launch and a grid-wide
// exact-sum tail (block flush, global limb atomics, ticket, last-block finalize) per reduction -- two
// per Lanczos step, about 60 launches per iteration; here a reduction is a block flush into shared
// memory, one cluster barrier, and a read of the other CTAs' limbs through distributed shared memory.
// Every CTA adds the limbs of all CTAs (exact integers: the same bits in every CTA) and finalizes
// into its own shared-memory copy of the scalar state, so all CTAs proceed with identical scalars and
// no second barrier is needed.  Vectors stay in global memory (L2); the cluster barrier (release /
// acquire at cluster scope) orders one phase's stores before the next phase's gathers.  Per-row
// arithmetic is that of the multi-kernel path's kernels: the same iterates, bit for bit.
namespace cg = cooperative_groups;
constexpr int kResThreads = 512;
constexpr int kResMaxN = 1 << 16;  // rows up to which an iteration runs as one cluster launch

struct ResShared {
  DevScalars sc;                              // replicated scalar state (identical in every CTA)
  long long xb[2][kMaxSums][kLimbs];          // this CTA's block partials, double-buffered by reduction
  double gk[2][kMaxR];                        // this CTA's partials of g = v^T Omega
  double red[kResThreads / 32][kMaxR];        // warp partials of g
  double sv[kMaxQ], srr[kMaxQ];               // s_j and fl(1/rho_j) of the combine
  TriScratch tri;
  long long Lsum[kMaxSums][kLimbs];           // the cluster totals of the current reduction
  double gsum[kMaxR];
};

// Cluster-wide exact reduction of NS sums (and, with R > 0, of the CTAs' g partials in CTA order),
// then finalize(kind) in every CTA into its own copy of the scalars.  par: this reduction's buffer.
template <int NS>
__device__ __forceinline__ void res_reduce(XWin (&acc)[NS], int err, ResShared &sm, int &par, int kind,
                                           const FinArgs &f, int R) {
  cg::cluster_group cl = cg::this_cluster();
#pragma unroll
  for (int s = 0; s < NS; ++s) xwin_flush(acc[s], sm.xb[par][s]);
  if (__syncthreads_or(err) && threadIdx.x == 0) sm.sc.err |= 1;
  cl.sync();  // every CTA's partials are complete (and every store of the phase is visible)
  const int ncta = (int)cl.num_blocks();
  if (threadIdx.x < 32) {
    // lanes add the CTAs' limbs (exact integers) and g partials (fp64, CTA order) straight into
    // shared memory; lane 0 finalizes from there (no shuffles, no local-memory arrays)
    const int lane = threadIdx.x;
    for (int idx = lane; idx < kMaxSums * kLimbs; idx += 32) {
      long long t = 0;
      if (idx < NS * kLimbs)
        for (int c = 0; c < ncta; ++c) t += *cl.map_shared_rank(&sm.xb[par][0][0] + idx, c);
      (&sm.Lsum[0][0])[idx] = t;
    }
    for (int k = lane; k < R; k += 32) {
      double t = 0.0;
      for (int c = 0; c < ncta; ++c) t += *cl.map_shared_rank(&sm.gk[par][k], c);
      sm.gsum[k] = t;
    }
    __syncwarp();
    if (lane == 0) finalize(kind, &sm.sc, sm.Lsum, sm.gsum, f);
  }
  // the other buffer is free: its readers (the previous reduction) are past this barrier
  for (int i = threadIdx.x; i < kMaxSums * kLimbs; i += blockDim.x) (&sm.xb[par ^ 1][0][0])[i] = 0;
  par ^= 1;
  __syncthreads();
}

struct ResArgs {
  double *G;            // gathered region: [x | w_1 | w_2 | ...] (store mode), npad apart
  long long npad;
  double *a, *d, *z, *y;
  const double *cdiag, *Om;
  double *V;            // v ring (deferred sketch): slot js
  long long ldv;
  int js;
  double *ckr;          // deferred sketch coefficients
  DevScalars *sc;       // global scalar state (loaded at entry, stored back by CTA 0 at exit)
  scg_iter_rec *log;
  IterArgs A;
  int R, nl;
  uint64_t seed;
  const int *orig;
};

template <bool UNI, int W>
__global__ void __launch_bounds__(kResThreads, 1) k_resident(Csr C, Rows RL, ResArgs P) {
  pdl_entry();
  extern __shared__ __align__(16) unsigned char res_raw[];
  ResShared &sm = *reinterpret_cast<ResShared *>(res_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int gtid = (int)blockIdx.x * blockDim.x + tid, gstride = (int)gridDim.x * blockDim.x;
  const IterArgs &A = P.A;
  const int nl = P.nl, q = A.q;
  const Net net{};  // one GPU: no peers (mask == nullptr)
  for (int i = tid; i < (int)(sizeof(DevScalars) / sizeof(int)); i += blockDim.x)
    reinterpret_cast<int *>(&sm.sc)[i] = __ldcg(reinterpret_cast<const int *>(P.sc) + i);
  for (int i = tid; i < 2 * kMaxSums * kLimbs; i += blockDim.x) (&sm.xb[0][0][0])[i] = 0;
  int par = 0;
  cl.sync();
  auto slot = [&](int j) -> double * { return P.G + (long long)j * P.npad; };  // w_j (j >= 1); x = slot(0)
  // ---- Lanczos pass 1 (Alg. 2 lines 1-9): k_lanczos_a + k_lanczos_b per step
  for (int i = 1; i <= q && !sm.sc.brk; ++i) {
    {
      EpiA epi;
      epi.a = P.a;
      epi.blk = sm.xb[par][0];
      xwin_init(epi.acc[0]);
      epi.err = 0;
      spmv_any<1, UNI, W>(C, RL, slot(i), sm.sc.rho[i - 1], P.d, nullptr, 0, nl, epi);
      FinArgs f{};
      f.i = i;
      res_reduce<1>(epi.acc, epi.err, sm, par, FK_OM, f, 0);
    }
    if (i == q) break;
    {
      const double om = sm.sc.om[i - 1], den = sm.sc.rho[i - 1];
      const double denm = i >= 2 ? sm.sc.rho[i - 2] : 1.0;
      const double rden = 1.0 / den, rdenm = 1.0 / denm;
      const double *Xi = slot(i), *Xim1 = slot(i > 1 ? i - 1 : 1);
      double *Xip1 = slot(i + 1);
      XWin acc[1];
      xwin_init(acc[0]);
      int err = 0;
      for (int r = gtid; r < nl; r += gstride) {
        double w = fma(-om, Xi[r] * rden, P.a[r]);
        if (i >= 2) w = fma(-den, Xim1[r] * rdenm, w);  // rho_{i-1} = rho[i-1] = den
        Xip1[r] = w;
        xwin_add_nn(acc[0], w * w, err, sm.xb[par][0]);
      }
      FinArgs f{};
      f.i = i;
      res_reduce<1>(acc, err, sm, par, FK_RHO, f, 0);
    }
  }
  // ---- tridiagonal eigenpair (lines 11-12), replicated in every CTA
  if (tid < 32) tridiag_warp(&sm.sc, q, sm.tri);
  __syncthreads();
  // ---- line 13 from the stored vectors (k_combine), ||x||^2
  {
    const int k = sm.sc.k;
    for (int j = tid; j < k; j += blockDim.x) {
      sm.sv[j] = sm.sc.s[j];
      sm.srr[j] = 1.0 / sm.sc.rho[j];
    }
    __syncthreads();
    XWin acc[1];
    xwin_init(acc[0]);
    int err = 0;
    double *x = slot(0);
    for (int r = gtid; r < nl; r += gstride) {
      double xr = sm.sv[0] * (__ldcg(slot(1) + r) * sm.srr[0]);
      for (int j = 1; j < k; ++j) xr = fma(sm.sv[j], __ldcg(slot(j + 1) + r) * sm.srr[j], xr);
      x[r] = xr;
      xwin_add_nn(acc[0], xr * xr, err, sm.xb[par][0]);
    }
    res_reduce<1>(acc, err, sm, par, FK_NUX, FinArgs{}, 0);
  }
  // ---- monitor: v = x / ||x||, xi, v^T C v, ||v||^2 (k_monitor)
  double *v = P.V + (long long)P.js * P.ldv;
  {
    EpiM epi;
    epi.v = v;
    epi.blk = sm.xb[par];
    xwin_init(epi.acc[0]);
    xwin_init(epi.acc[1]);
    xwin_init(epi.acc[2]);
    epi.err = 0;
    spmv_any<2, UNI, W>(C, RL, slot(0), sm.sc.nu_x, P.d, P.cdiag, 0, nl, epi);
    res_reduce<3>(epi.acc, epi.err, sm, par, FK_MON, FinArgs{}, 0);
  }
  // ---- primal: z <- (1 - eta) z + eta alpha (v o v), ||z - b||^2, g = v^T Omega (k_primal)
  {
    const bool hoff = A.trace_le && !(sm.sc.xi < 0.0);
    XWin acc[1];
    xwin_init(acc[0]);
    int err = 0;
    const int lane = tid & 31, warp = tid >> 5;
    for (int kc = 0; kc < P.R; kc += 16) {
      double gp[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) gp[u] = 0.0;
      for (int r = gtid; r < nl; r += gstride) {
        const double vr = v[r];
        if (kc == 0) {
          const double hv = A.alpha * (vr * vr);
          const double zr = hoff ? A.one_m_eta * P.z[r] : fma(A.eta, hv, A.one_m_eta * P.z[r]);
          P.z[r] = zr;
          const double e = zr - A.b;
          xwin_add_nn(acc[0], e * e, err, sm.xb[par][0]);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (kc + u < P.R) gp[u] = fma(vr, __ldg(&P.Om[(long long)(kc + u) * nl + r]), gp[u]);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        double t = gp[u];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (lane == 0 && kc + u < P.R) sm.red[warp][kc + u] = t;
      }
    }
    __syncthreads();
    if (tid < P.R) {
      double t = 0.0;
      for (int w = 0; w < kResThreads / 32; ++w) t += sm.red[w][tid];
      sm.gk[par][tid] = t;
    }
    FinArgs f{};
    f.R = P.R;
    f.A = A;
    f.log = blockIdx.x == 0 ? P.log : nullptr;
    res_reduce<1>(acc, err, sm, par, FK_NZ, f, P.R);
  }
  // ---- dual: y <- y + gamma (z - b), d for t+1, next start vector and ||g||^2, gap sums (k_dual_sketch)
  {
    const double gam = sm.sc.gamma;
    if (blockIdx.x == 0 && tid < P.R)
      P.ckr[P.js * kMaxR + tid] = (A.trace_le && !(sm.sc.xi < 0.0)) ? 0.0 : (A.eta * A.alpha) * sm.sc.gk[tid];
    XWin acc[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) xwin_init(acc[s]);
    int err = 0;
    double *g = slot(1);
    for (int r = gtid; r < nl; r += gstride) {
      const double zr = P.z[r], yv = P.y[r];
      const double e = zr - A.b;
      const double yr = fma(gam, e, yv);
      P.y[r] = yr;
      P.d[r] = fma(A.beta_next, e, yr) + P.cdiag[r];
      const double gv = scg_lanczos_start(P.seed, A.t + 1, P.orig[r]);
      g[r] = gv;
      xwin_add_nn(acc[0], gv * gv, err, sm.xb[par][0]);
      xwin_add(acc[1], yr, err, sm.xb[par][1]);
      xwin_add(acc[2], yr * zr, err, sm.xb[par][2]);
      xwin_add_nn(acc[3], zr * zr, err, sm.xb[par][3]);
      xwin_add_nn(acc[4], zr, err, sm.xb[par][4]);
    }
    res_reduce<5>(acc, err, sm, par, FK_RHO0M, FinArgs{}, 0);
  }
  (void)net;
  if (blockIdx.x == 0) {
    for (int i = tid; i < (int)(sizeof(DevScalars) / sizeof(int)); i += blockDim.x)
      reinterpret_cast<int *>(P.sc)[i] = reinterpret_cast<const int *>(&sm.sc)[i];
  }
  cl.sync();  // range errors seen by any CTA (its own summands) reach the global flag
  if (blockIdx.x != 0 && tid == 0 && sm.sc.err) atomicOr(&P.sc->err, sm.sc.err);
}

}  // namespace scg
