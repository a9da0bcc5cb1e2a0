// phase.cu -- B200-native SketchyCGAL for the abstract phase retrieval SDP.
//
// C ABI: include/scg_phase.h.  Method: Alg. 4 with the trace-bounded LMO
// on the scaled phase retrieval SDP; randomized Lanczos
// (Alg. 2) over C^n; complex Nystrom sketch (Alg. 3).
// section 11 has the data layout, the readings R36-R38 and the rooflines.
//
// The matrix-vector product D x = x / sqrt(n) + sum_j kappa_j M_j^* (w_j o M_j x),
// M_j = W_n diag(conj psi_j), is a four-step FFT (n = n1 n2, m = m1 + n1 m2, l = k2 + n2 k1):
//   k_pr_f1  per m1 tile, per j: modulate by conj(psi_j), length-n2 FFT over m2 -> Y_j[k2][m1]
//   k_pr_b   per k2 tile, per j: twiddle w_n^{m1 k2}, length-n1 FFT over m1 (-> (M_j x)_l), times
//            the weight kappa_j w_j[l], inverse length-n1 FFT over k1, twiddle w_n^{-m1 k2}, in place
//   k_pr_c   per m1 tile: for every j the inverse length-n2 FFT over k2, demodulate by psi_j and
//            accumulate over j in registers; + x / sqrt(n); write D x and the Lanczos dot v^* D x.
// The dual vectors z, y, b~, w live in the FFT's natural output order p = k2 n1 + k1 ("p-order"),
// so the weights are read contiguously; psi is stored as one byte per entry into a codebook.
// Each sub-FFT runs in shared memory as a mixed-radix Stockham transform (radices 2, 3, 4, 5, 8;
// stage 0 loads straight from global memory, the last stage stays in registers).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "../../include/scg_phase.h"
#include "../../include/sketchycgal.h"
#include "../../scg_inputs/include/scg_rng.h"

namespace {

constexpr int kQMax = 256;
constexpr int kRMax = 16;
constexpr int kLMax = 32;
constexpr int kMaxStages = 12;
constexpr int kSubMax = 4096;
constexpr int kXR = 10;  // largest radix (10: compile-time plans of powers of ten)

typedef std::complex<double> cplx;

struct Plan {
  int N, ns;
  int R[kMaxStages];
  int Ns[kMaxStages];
};

struct PrScal {
  double omega[kQMax];
  double rho[kQMax];
  double scale[kQMax + 1];  // v_i = scale[i-1] * U[i-1]
  double svec[kQMax];
  double theta, vnrm, vv, cval, xi, gamma, tau, p, nz;
  double g[2 * kRMax];  // v^* Omega
  int kbreak, k;
  unsigned ticket[8];
};

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// ------------------------------------------------------------------ small DFTs (sign -1 forward)
template <bool INV>
__device__ __forceinline__ void dft2(double2 &a, double2 &b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
template <bool INV>
__device__ __forceinline__ void dft4(double2 &x0, double2 &x1, double2 &x2, double2 &x3) {
  double2 s02 = cadd(x0, x2), d02 = csub(x0, x2), s13 = cadd(x1, x3), d13 = mul_mi<INV>(csub(x1, x3));
  x0 = cadd(s02, s13);
  x2 = csub(s02, s13);
  x1 = cadd(d02, d13);
  x3 = csub(d02, d13);
}
template <bool INV>
__device__ __forceinline__ void dft3(double2 &x0, double2 &x1, double2 &x2) {
  const double h = 0.86602540378443864676;  // sqrt(3)/2
  double2 t = cadd(x1, x2);
  double2 m = make_double2(x0.x - 0.5 * t.x, x0.y - 0.5 * t.y);
  double2 d = mul_mi<INV>(cscale(csub(x1, x2), h));
  x0 = cadd(x0, t);
  x1 = cadd(m, d);
  x2 = csub(m, d);
}
template <bool INV>
__device__ __forceinline__ void dft5(double2 &x0, double2 &x1, double2 &x2, double2 &x3, double2 &x4) {
  const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;  // cos(2pi/5), cos(4pi/5)
  const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;   // sin(2pi/5), sin(4pi/5)
  double2 t1 = cadd(x1, x4), t2 = cadd(x2, x3), t3 = csub(x1, x4), t4 = csub(x2, x3);
  double2 a1 = make_double2(x0.x + c1 * t1.x + c2 * t2.x, x0.y + c1 * t1.y + c2 * t2.y);
  double2 a2 = make_double2(x0.x + c2 * t1.x + c1 * t2.x, x0.y + c2 * t1.y + c1 * t2.y);
  double2 b1 = mul_mi<INV>(make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y));
  double2 b2 = mul_mi<INV>(make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y));
  x0 = cadd(x0, cadd(t1, t2));
  x1 = cadd(a1, b1);
  x4 = csub(a1, b1);
  x2 = cadd(a2, b2);
  x3 = csub(a2, b2);
}
template <bool INV>
__device__ __forceinline__ void dft8(double2 (&x)[kXR]) {
  const double r = 0.70710678118654752440;
  dft4<INV>(x[0], x[2], x[4], x[6]);
  dft4<INV>(x[1], x[3], x[5], x[7]);
  // twiddles w8^k on the odd half: w8 = e^{-i pi/4} (forward)
  double2 o1 = x[3], o2 = x[5], o3 = x[7];
  // x[1]*1, x[3]*w8, x[5]*w8^2, x[7]*w8^3 (the dft4 outputs are in positions 1,3,5,7 for k=0..3)
  o1 = INV ? make_double2(r * (o1.x - o1.y), r * (o1.x + o1.y)) : make_double2(r * (o1.x + o1.y), r * (o1.y - o1.x));
  o2 = mul_mi<INV>(o2);
  o3 = INV ? make_double2(-r * (o3.x + o3.y), r * (o3.x - o3.y)) : make_double2(r * (o3.y - o3.x), -r * (o3.x + o3.y));
  double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  x[0] = cadd(e0, x[1]);
  x[4] = csub(e0, x[1]);
  x[1] = cadd(e1, o1);
  x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2);
  x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3);
  x[7] = csub(e3, o3);
}

// DFT10 = 5 DFT2 (n = n2 + 5 n1), twiddles w10^{n2} on the odd half, 2 DFT5 (outputs k = k1 + 2 k2)
template <bool INV>
__device__ __forceinline__ void dft10(double2 (&x)[kXR]) {
  const double c1 = 0.80901699437494742410, s1 = 0.58778525229247312917;  // w10 = e^{-2 pi i / 10}
  const double c2 = 0.30901699437494742410, s2 = 0.95105651629515357212;  // w10^2
  double2 u0[5], u1[5];
#pragma unroll
  for (int m = 0; m < 5; ++m) {
    u0[m] = cadd(x[m], x[m + 5]);
    u1[m] = csub(x[m], x[m + 5]);
  }
  // w10^{m} (forward: cos - i sin), m = 1..4: w^3 = -conj(w^2), w^4 = -conj(w^1)
  const double2 w1 = make_double2(c1, INV ? s1 : -s1), w2 = make_double2(c2, INV ? s2 : -s2);
  const double2 w3 = make_double2(-c2, INV ? s2 : -s2), w4 = make_double2(-c1, INV ? s1 : -s1);
  u1[1] = cmul(u1[1], w1);
  u1[2] = cmul(u1[2], w2);
  u1[3] = cmul(u1[3], w3);
  u1[4] = cmul(u1[4], w4);
  dft5<INV>(u0[0], u0[1], u0[2], u0[3], u0[4]);
  dft5<INV>(u1[0], u1[1], u1[2], u1[3], u1[4]);
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    x[2 * k] = u0[k];
    x[2 * k + 1] = u1[k];
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2 (&x)[kXR]) {
  if constexpr (R == 2) dft2<INV>(x[0], x[1]);
  if constexpr (R == 3) dft3<INV>(x[0], x[1], x[2]);
  if constexpr (R == 4) dft4<INV>(x[0], x[1], x[2], x[3]);
  if constexpr (R == 5) dft5<INV>(x[0], x[1], x[2], x[3], x[4]);
  if constexpr (R == 8) dft8<INV>(x);
  if constexpr (R == 10) dft10<INV>(x);
}

// Radix plan of a sub-transform length N (host and device, constexpr): the power-of-two part in
// 8s and 4s (never a lone 2 unless N has a single factor 2), then 5s, then 3s.  ns = 0: unsupported.
struct CPlan {
  int ns, rmin;
  int R[kMaxStages];
  int Ns[kMaxStages];
};
__host__ __device__ constexpr CPlan make_cplan(int N, bool allow10 = false) {
  CPlan c{0, 8, {0}, {0}};
  if (N < 2 || N > kSubMax) return c;
  if (allow10 && N == 1000) {  // radix-10 stages: 3 instead of 4 (measured faster at 1000, slower at 100)
    int m = N, k = 0;
    while (m % 10 == 0) { m /= 10; ++k; }
    if (m == 1) {
      c.ns = k;
      c.rmin = 10;
      int acc = 1;
      for (int s = 0; s < k; ++s) {
        c.R[s] = 10;
        c.Ns[s] = acc;
        acc *= 10;
      }
      return c;
    }
  }
  int m = N, a = 0;
  while (m % 2 == 0) { m /= 2; ++a; }
  int R[kMaxStages] = {0};
  int ns = 0;
  while (a > 0) {
    int r = a >= 3 && a != 4 ? 8 : (a >= 2 ? 4 : 2);
    R[ns++] = r;
    a -= r == 8 ? 3 : (r == 4 ? 2 : 1);
  }
  while (m % 5 == 0) { R[ns++] = 5; m /= 5; }
  while (m % 3 == 0) { R[ns++] = 3; m /= 3; }
  if (m != 1 || ns > kMaxStages) return c;
  c.ns = ns;
  int acc = 1, rmin = 8;
  for (int s = 0; s < ns; ++s) {
    c.R[s] = R[s];
    c.Ns[s] = acc;
    acc *= R[s];
    rmin = R[s] < rmin ? R[s] : rmin;
  }
  c.rmin = rmin;
  return c;
}

// ---- runtime plan (any supported length): one Stockham stage for a compile-time radix.
// sm layout: element i of transform t at sm[i * TM + t]; tw = w_N^e table (shared memory).
template <int R, bool INV>
__device__ __forceinline__ void stage_body(double2 (&x)[kXR], double2 *sm, int s, const Plan &P, const double2 *tw,
                                           int TM, int t, int jb) {
  const int N = P.N, Ns = P.Ns[s], NR = N / R;
  const bool act = jb < NR;
  if (s > 0) {
    if (act) {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = sm[(jb + r * NR) * TM + t];
    }
    __syncthreads();
  }
  if (act) {
    if (Ns > 1) {
      const int k = jb % Ns, step = N / (Ns * R);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 w = tw[(k * r) * step];
        x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
      }
    }
    dft<R, INV>(x);
  }
  if (s < P.ns - 1) {
    if (act) {
      const int k = jb % Ns, idxD = (jb / Ns) * Ns * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm[(idxD + r * Ns) * TM + t] = x[r];
    }
    __syncthreads();
  }
}

template <bool INV>
__device__ __forceinline__ void fft_stages(double2 (&x)[kXR], double2 *sm, const Plan &P, const double2 *tw, int TM,
                                           int t, int jb) {
  for (int s = 0; s < P.ns; ++s) {
    switch (P.R[s]) {
      case 2: stage_body<2, INV>(x, sm, s, P, tw, TM, t, jb); break;
      case 3: stage_body<3, INV>(x, sm, s, P, tw, TM, t, jb); break;
      case 4: stage_body<4, INV>(x, sm, s, P, tw, TM, t, jb); break;
      case 5: stage_body<5, INV>(x, sm, s, P, tw, TM, t, jb); break;
      default: stage_body<8, INV>(x, sm, s, P, tw, TM, t, jb); break;
    }
  }
}

// Shared-memory swizzle of the compile-time plans (element e = i * TM + t): chosen by a bank-conflict
// simulation of every stage's 128-bit accesses (8 lanes per wavefront): the radix-8 first stage stores
// with a stride of 8 TM elements.  (1000, 2): XOR of the 8-element group index into the low bits (no
// padding, conflict-free); TM = 4: two pad elements per 8 (conflict-free for 400).  Radix-10 plans
// (1000): XOR swizzles (5 % / 20 % excess wavefronts left for TM = 4 / 2).
template <int N, int TM>
__host__ __device__ constexpr int swz(int e) {
  if constexpr (N == 1000 && TM == 4) return (e & ~7) | ((e ^ (e >> 3)) & 7);  // radix 10
  else if constexpr (N == 1000 && TM == 2) return (e & ~7) | ((e ^ (e >> 5)) & 7);
  else if constexpr (TM == 4) return e + ((e >> 3) << 1);
  else return e;
}
// transform buffer (double2 elements) of TM transforms of length N, room for the padded swizzle
__host__ __device__ constexpr size_t fft_buf(int TM, int N) {
  return (size_t)TM * N + (((size_t)TM * N) >> 3) * 2 + 8;
}

// ---- compile-time plan (the hot lengths): every index is a constant expression.
template <int N, int S, bool INV, int TM>
__device__ __forceinline__ void ct_stage(double2 (&x)[kXR], double2 *sm, const double2 *tw, int t, int jb) {
  constexpr CPlan c = make_cplan(N, true);
  constexpr int R = c.R[S], Ns = c.Ns[S], NR = N / R;
  const bool act = jb < NR;
  if constexpr (S > 0) {
    if (act) {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = sm[swz<N, TM>((jb + r * NR) * TM + t)];
    }
    __syncthreads();
  }
  if (act) {
    if constexpr (Ns > 1) {
      constexpr int step = N / (Ns * R);
      const int k = jb % Ns;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 w = tw[(k * r) * step];
        x[r] = INV ? cmulc(x[r], w) : cmul(x[r], w);
      }
    }
    dft<R, INV>(x);
  }
  if constexpr (S < c.ns - 1) {
    if (act) {
      const int k = jb % Ns, idxD = (jb / Ns) * Ns * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm[swz<N, TM>((idxD + r * Ns) * TM + t)] = x[r];
    }
    __syncthreads();
    ct_stage<N, S + 1, INV, TM>(x, sm, tw, t, jb);
  }
}

// Sub-transform engine: NC > 0 compile-time length / TMC transforms per block, NC = 0 runtime plan.
template <int NC, int TMC>
struct Sub {
  static constexpr bool CT = NC > 0;
  const Plan &P;
  int TM, t, jb;
  __device__ __forceinline__ Sub(const Plan &P_, int TMr) : P(P_) {
    TM = CT ? TMC : TMr;
    t = threadIdx.x % TM;
    jb = threadIdx.x / TM;
  }
  __device__ __forceinline__ int N() const { return CT ? NC : P.N; }
  __device__ __forceinline__ int R0() const {
    if constexpr (CT) { constexpr CPlan c = make_cplan(NC, true); return c.R[0]; } else { return P.R[0]; }
  }
  __device__ __forceinline__ int RL() const {
    if constexpr (CT) { constexpr CPlan c = make_cplan(NC, true); return c.R[c.ns - 1]; } else { return P.R[P.ns - 1]; }
  }
  __device__ __forceinline__ int NR0() const { return N() / R0(); }
  __device__ __forceinline__ int NRL() const { return N() / RL(); }
  __device__ __forceinline__ int in_pos(int r) const { return jb + r * NR0(); }
  // shared-memory slot of element i of this thread's transform
  __device__ __forceinline__ int slot(int i) const {
    if constexpr (CT) return swz<NC, TMC>(i * TMC + t);
    else return i * TM + t;
  }
  __device__ __forceinline__ size_t buf() const { return fft_buf(TM, N()); }
  // the last stage leaves element out_pos(r) = jb + r N / R_last in x[r], which is exactly the first
  // stage's input in_pos(r) = jb + r N / R_0 when R_0 = R_last (radix-10 plans): a forward transform can
  // feed an inverse one from registers
  __host__ __device__ static constexpr bool sym() {
    if constexpr (CT) {
      constexpr CPlan c = make_cplan(NC, true);
      return c.R[0] == c.R[c.ns - 1] && c.Ns[c.ns - 1] == NC / c.R[0];
    } else {
      return false;
    }
  }
  __device__ __forceinline__ int out_stride() const {
    if constexpr (CT) { constexpr CPlan c = make_cplan(NC, true); return c.Ns[c.ns - 1]; } else { return P.Ns[P.ns - 1]; }
  }
  __device__ __forceinline__ int out_pos(int r) const {
    if constexpr (CT) {
      constexpr CPlan c = make_cplan(NC, true);
      constexpr int R = c.R[c.ns - 1], Ns = c.Ns[c.ns - 1];
      return (jb / Ns) * Ns * R + (jb % Ns) + r * Ns;
    } else {
      const int R = P.R[P.ns - 1], Ns = P.Ns[P.ns - 1];
      return (jb / Ns) * Ns * R + (jb % Ns) + r * Ns;
    }
  }
  template <bool INV>
  __device__ __forceinline__ void run(double2 (&x)[kXR], double2 *sm, const double2 *tw) const {
    if constexpr (CT) ct_stage<NC, 0, INV, TMC>(x, sm, tw, t, jb);
    else fft_stages<INV>(x, sm, P, tw, TM, t, jb);
  }
};

// w_n^e = hi[e >> 11] * lo[e & 2047]
__device__ __forceinline__ double2 twn(const double2 *__restrict__ lo, const double2 *__restrict__ hi, long long e) {
  return cmul(__ldg(hi + (e >> 11)), __ldg(lo + (e & 2047)));
}

// ------------------------------------------------------------------ reductions
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double *red /* >= 32 * NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w * NV + i];
      v[i] = s;
    }
  }
}

// Block partials -> the last block (ticket) sums them in a fixed order (deterministic).  Returns true in
// the last block (all threads); v[i] then holds the totals in thread 0.
template <int NV>
__device__ __forceinline__ bool grid_sum(double (&v)[NV], double *partials, unsigned *ticket, double *red) {
  __shared__ bool s_last;
  block_sum<NV>(v, red);
  const unsigned nb = gridDim.x * gridDim.y;
  const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) partials[(size_t)bid * NV + i] = v[i];
    __threadfence();
    unsigned prev = atomicAdd(ticket, 1u);
    s_last = (prev == nb - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  // all threads of the last block: strided loads in block order, then the fixed-order block sum
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) s += __ldcg(partials + (size_t)b * NV + i);
    v[i] = s;
  }
  block_sum<NV>(v, red);
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

__device__ __forceinline__ bool skip_step(const PrScal *sc, int step) { return step > 0 && step > sc->kbreak; }

// ------------------------------------------------------------------ kernels
// Lanczos start vector of iteration t (Alg. 2 line 1): u0 = g, scale[0] = 1 / ||g||.
__global__ void k_pr_start(double2 *__restrict__ u0, int64_t n, uint64_t seed, int64_t t, PrScal *sc,
                           double *partials) {
  __shared__ double red[32];
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double re = scg_normal(seed, SCG_STREAM_LANCZOS, (uint32_t)t, (uint64_t)(2 * i));
    double im = scg_normal(seed, SCG_STREAM_LANCZOS, (uint32_t)t, (uint64_t)(2 * i + 1));
    u0[i] = make_double2(re, im);
    v[0] += re * re + im * im;
  }
  if (grid_sum<1>(v, partials, &sc->ticket[0], red) && threadIdx.x == 0) {
    sc->scale[0] = 1.0 / sqrt(v[0]);
    sc->kbreak = kQMax + 1;
  }
}

// Shared memory of the FFT kernels: [TM * N transform buffer][N twiddles w_N^e][256 codebook].
__device__ __forceinline__ void load_tables(double2 *twsm, const double2 *__restrict__ tw, int N, double2 *cbsm,
                                            const double2 *__restrict__ book) {
  for (int i = threadIdx.x; i < N; i += blockDim.x) twsm[i] = __ldg(tw + i);
  if (cbsm)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cbsm[i] = __ldg(book + i);
}

// Forward step A: per (m1 tile, j): x = conj(psi_j) o (s u), length-n2 FFT over m2 -> Y[j][k2][m1].
// Persistent: each block walks tiles (j, m1 tile) with the next tile's inputs loaded into registers
// while the current one is transformed.
template <int NC, int TMC, bool PF>
__global__ void __launch_bounds__(512) k_pr_f1(const double2 *__restrict__ u, const double *__restrict__ scale_p,
                                               int step, const PrScal *__restrict__ sc,
                                               const uint8_t *__restrict__ codes, const double2 *__restrict__ book,
                                               double2 *__restrict__ Y, Plan P, const double2 *__restrict__ tw,
                                               int n1, int n2, int TMr, int L) {
  if (skip_step(sc, step)) return;
  const Sub<NC, TMC> F(P, TMr);
  extern __shared__ double2 sm[];
  double2 *twsm = sm + F.buf();
  double2 *cb = twsm + F.N();
  load_tables(twsm, tw, F.N(), cb, book);
  __syncthreads();
  const int64_t n = (int64_t)n1 * F.N();
  const int tiles_per_j = n1 / F.TM, ntiles = tiles_per_j * L;
  const double s = scale_p ? *scale_p : 1.0;
  const bool ld = F.jb < F.NR0();
  double2 un[kXR];
  uint8_t cn[kXR];
  auto fetch = [&](int tile) {
    const int j = tile / tiles_per_j, m1_0 = (tile - j * tiles_per_j) * F.TM;
    const uint8_t *cj = codes + (size_t)j * n;
#pragma unroll
    for (int r = 0; r < kXR; ++r)
      if (r < F.R0()) {
        const int64_t m = m1_0 + F.t + (int64_t)n1 * F.in_pos(r);
        un[r] = __ldg(u + m);
        cn[r] = __ldg(cj + m);
      }
  };
  int tile = blockIdx.x;
  if (ld && tile < ntiles) fetch(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    double2 x[kXR];
    if (ld) {
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.R0()) x[r] = cmulc(cscale(un[r], s), cb[cn[r]]);
      if (PF && tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);
    }
    F.template run<false>(x, sm, twsm);
    if (!PF && ld && tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);
    if (F.jb < F.NRL()) {
      const int j = tile / tiles_per_j, m1_0 = (tile - j * tiles_per_j) * F.TM;
      double2 *Yj = Y + (size_t)j * n + m1_0 + F.t;
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) Yj[(size_t)F.out_pos(r) * n1] = x[r];
    }
  }
}

// Middle step: per (k2 tile, j): twiddle, length-n1 FFT over m1, [h = |.|^2], times w, inverse FFT,
// twiddle back, in place.  mode 0: matvec, 1: matvec + h (monitor), 2: h only (measure).  Persistent with
// the next tile's row loaded during the current tile's transforms.
template <int NC, int TMC, bool PF>
__global__ void __launch_bounds__(512) k_pr_b(double2 *__restrict__ Y, const double *__restrict__ wk,
                                              double *__restrict__ h, int mode, int step,
                                              const PrScal *__restrict__ sc, Plan P, const double2 *__restrict__ tw,
                                              const double2 *__restrict__ twlo, const double2 *__restrict__ twhi,
                                              int n1, int n2, int TMr, int L) {
  if (skip_step(sc, step)) return;
  const Sub<NC, TMC> F(P, TMr);
  extern __shared__ double2 sm[];
  double2 *twsm = sm + F.buf();
  load_tables(twsm, tw, F.N(), nullptr, nullptr);
  __syncthreads();
  const int n1c = F.N();
  const int64_t n = (int64_t)n1c * n2;
  const int tiles_per_j = n2 / F.TM, ntiles = tiles_per_j * L;
  const bool ld = F.jb < F.NR0();
  double2 yn[kXR];
  auto fetch = [&](int tile) {
    const int j = tile / tiles_per_j, k2 = (tile - j * tiles_per_j) * F.TM + F.t;
    const double2 *row = Y + (size_t)j * n + (size_t)k2 * n1c;
#pragma unroll
    for (int r = 0; r < kXR; ++r)
      if (r < F.R0()) yn[r] = row[F.in_pos(r)];
  };
  int tile = blockIdx.x;
  if (ld && tile < ntiles) fetch(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const int j = tile / tiles_per_j, k2 = (tile - j * tiles_per_j) * F.TM + F.t;
    const size_t base = (size_t)j * n + (size_t)k2 * n1c;
    double2 x[kXR];
    double wv[kXR];
    if (mode <= 1 && F.jb < F.NRL()) {
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) wv[r] = __ldg(wk + base + F.out_pos(r));
    }
    if (ld) {
      // w_n^{m1 k2} for m1 = jb + r NR0: base w_n^{jb k2} times powers of w_n^{NR0 k2}
      const double2 w1 = twn(twlo, twhi, (long long)F.NR0() * k2);
      double2 w = twn(twlo, twhi, (long long)F.jb * k2);
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.R0()) {
          x[r] = cmul(yn[r], w);
          w = cmul(w, w1);
        }
      if (PF && tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);
    }
    F.template run<false>(x, sm, twsm);
    if (F.jb < F.NRL()) {
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) {
          if (mode >= 1) h[base + F.out_pos(r)] = x[r].x * x[r].x + x[r].y * x[r].y;
          if (mode <= 1) x[r] = cscale(x[r], wv[r]);
        }
    }
    if (mode == 2) continue;
    // re-enter shared memory for the inverse transform over k1 (not needed when the plan is symmetric:
    // the forward's last-stage reads are complete at its barrier, the inverse's stage 0 starts from x)
    if constexpr (!Sub<NC, TMC>::sym()) {
      if (F.jb < F.NRL()) {
#pragma unroll
        for (int r = 0; r < kXR; ++r)
          if (r < F.RL()) sm[F.slot(F.out_pos(r))] = x[r];
      }
      __syncthreads();
      if (ld) {
#pragma unroll
        for (int r = 0; r < kXR; ++r)
          if (r < F.R0()) x[r] = sm[F.slot(F.in_pos(r))];
      }
      __syncthreads();
    }
    if (!PF && ld && tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);
    F.template run<true>(x, sm, twsm);
    if (F.jb < F.NRL()) {
      double2 *row = Y + base;
      // w_n^{-m1 k2} for m1 = out_pos(0) + r Ns_last: base times powers
      const double2 v1 = twn(twlo, twhi, (long long)F.out_stride() * k2);
      double2 v = twn(twlo, twhi, (long long)F.out_pos(0) * k2);
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) {
          row[F.out_pos(r)] = cmulc(x[r], v);
          v = cmul(v, v1);
        }
    }
  }
}

// Inverse step A' + demodulation + sum over j + C~ x + Lanczos dot:
//   a = s u / sqrt(n) + sum_j psi_j o (inverse length-n2 FFT over k2 of Y[j][.][m1]).
// mode 0: write a, omega[step-1] = Re((s u)^* a);  mode 1 (monitor): xi = Re(v^* a), a not written;
// mode 2 (apply_D hook): write a only.  The sum over j accumulates in shared memory (each position is
// owned by one thread); Y of modulation j + 1 is loaded while j is transformed.
template <int NC, int TMC, bool PF>
__global__ void __launch_bounds__(512) k_pr_c(const double2 *__restrict__ Y, const double2 *__restrict__ u,
                                              const double *__restrict__ scale_p, double2 *__restrict__ a,
                                              const uint8_t *__restrict__ codes, const double2 *__restrict__ book,
                                              Plan P, const double2 *__restrict__ tw, int n1, int n2, int TMr, int L,
                                              double rsn, int mode, int step, PrScal *sc, double *partials) {
  if (skip_step(sc, step)) return;
  const Sub<NC, TMC> F(P, TMr);
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  double2 *twsm = sm + F.buf();
  double2 *cb = twsm + F.N();
  double2 *acc = cb + 256;
  load_tables(twsm, tw, F.N(), cb, book);
  const int64_t n = (int64_t)n1 * F.N();
  const double s = scale_p ? *scale_p : 1.0;
  const bool ld = F.jb < F.NR0(), st = F.jb < F.NRL();
  double v[1] = {0.0};
  for (int tile = blockIdx.x; tile < n1 / F.TM; tile += gridDim.x) {
    const int m1_0 = tile * F.TM;
    double2 yn[kXR];
    auto fetch = [&](int j) {
      const double2 *Yj = Y + (size_t)j * n + m1_0 + F.t;
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.R0()) yn[r] = Yj[(size_t)F.in_pos(r) * n1];
    };
    if (ld) fetch(0);
    if (st) {
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) acc[F.out_pos(r) * F.TM + F.t] = make_double2(0.0, 0.0);
    }
    for (int j = 0; j < L; ++j) {
      double2 x[kXR];
#pragma unroll
      for (int r = 0; r < kXR; ++r) x[r] = yn[r];
      if (PF && ld && j + 1 < L) fetch(j + 1);
      __syncthreads();  // the tables are in (first pass); previous shared-memory reads are done
      F.template run<true>(x, sm, twsm);
      if (!PF && ld && j + 1 < L) fetch(j + 1);
      if (st) {
        const uint8_t *cj = codes + (size_t)j * n + m1_0 + F.t;
#pragma unroll
        for (int r = 0; r < kXR; ++r)
          if (r < F.RL()) {
            const int pos = F.out_pos(r);
            acc[pos * F.TM + F.t] = cadd(acc[pos * F.TM + F.t], cmul(cb[__ldg(cj + (int64_t)n1 * pos)], x[r]));
          }
      }
    }
    if (st) {
#pragma unroll
      for (int r = 0; r < kXR; ++r)
        if (r < F.RL()) {
          const int pos = F.out_pos(r);
          const int64_t m = m1_0 + F.t + (int64_t)n1 * pos;
          const double2 uv = cscale(__ldg(u + m), s);
          const double2 am = cadd(cscale(uv, rsn), acc[pos * F.TM + F.t]);
          if (mode != 1) a[m] = am;
          v[0] += uv.x * am.x + uv.y * am.y;
        }
    }
  }
  if (mode == 2) return;
  if (grid_sum<1>(v, partials, &sc->ticket[1], red) && threadIdx.x == 0) {
    if (mode == 0) sc->omega[step - 1] = v[0];
    else sc->xi = v[0];
  }
}

// Kernel variants: compile-time plans for the sub-lengths of the paper's n = 10^4..10^6
// (100, 250, 400, 1000) with TM = 2 or 4 transforms per block; any other length runs the runtime plan.
typedef void (*F1Fn)(const double2 *, const double *, int, const PrScal *, const uint8_t *, const double2 *, double2 *,
                     Plan, const double2 *, int, int, int, int);
typedef void (*BFn)(double2 *, const double *, double *, int, int, const PrScal *, Plan, const double2 *,
                    const double2 *, const double2 *, int, int, int, int);
typedef void (*CFn)(const double2 *, const double2 *, const double *, double2 *, const uint8_t *, const double2 *, Plan,
                    const double2 *, int, int, int, int, double, int, int, PrScal *, double *);
struct Variant {
  int N, TM;
  F1Fn f1, f1n;  // with / without the register prefetch of the next tile
  BFn b, bn;
  CFn c, cn;
};
#define SCG_PR_VARIANT(N, TM)                                                                      \
  {N, TM, k_pr_f1<N, TM, true>, k_pr_f1<N, TM, false>, k_pr_b<N, TM, true>, k_pr_b<N, TM, false>, \
   k_pr_c<N, TM, true>, k_pr_c<N, TM, false>}
const Variant kVariants[] = {SCG_PR_VARIANT(100, 4),  SCG_PR_VARIANT(250, 4), SCG_PR_VARIANT(400, 4),
                             SCG_PR_VARIANT(1000, 4), SCG_PR_VARIANT(1000, 2), SCG_PR_VARIANT(100, 2),
                             SCG_PR_VARIANT(250, 2),  SCG_PR_VARIANT(400, 2)};
const Variant kGeneric = SCG_PR_VARIANT(0, 0);
const Variant *find_variant(int N, int TM) {
  for (const Variant &v : kVariants)
    if (v.N == N && v.TM == TM) return &v;
  return nullptr;
}

// Three-term recurrence (Alg. 2 lines 6-9): U[i] = a - omega_i v_i - rho_{i-1} v_{i-1}; rho_i = ||U[i]||,
// scale[i] = 1 / rho_i; break (kbreak = i) when rho_i <= 2^-45 (|omega_i| + rho_{i-1}) (reading A3).
__global__ void k_pr_recur(const double2 *__restrict__ a, double2 *__restrict__ U, int64_t n, int step,
                           PrScal *sc, double *partials) {
  if (skip_step(sc, step)) return;
  __shared__ double red[32];
  const int i = step;
  const double om = sc->omega[i - 1], si = sc->scale[i - 1];
  const double rp = i >= 2 ? sc->rho[i - 2] : 0.0, sp = i >= 2 ? sc->scale[i - 2] : 0.0;
  const double2 *ui = U + (size_t)(i - 1) * n;
  const double2 *up = U + (size_t)(i >= 2 ? i - 2 : 0) * n;
  double2 *un = U + (size_t)i * n;
  double v[1] = {0.0};
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    double2 w = csub(__ldg(a + m), cscale(cscale(__ldg(ui + m), si), om));
    if (i >= 2) w = csub(w, cscale(cscale(__ldg(up + m), sp), rp));
    un[m] = w;
    v[0] += w.x * w.x + w.y * w.y;
  }
  if (grid_sum<1>(v, partials, &sc->ticket[2], red) && threadIdx.x == 0) {
    const double rho = sqrt(v[0]);
    sc->rho[i - 1] = rho;
    if (rho <= 0x1p-45 * (fabs(om) + rp)) sc->kbreak = i;
    else sc->scale[i] = 1.0 / rho;
  }
}

// Minimum eigenpair of tridiag(rho, omega, rho) (Alg. 2 lines 11-12) on one warp: 32-way multisection
// with Sturm counts for theta, then inverse iteration (3 sweeps, lane 0) for the eigenvector.
__global__ void k_pr_tridiag(PrScal *sc, int q) {
  __shared__ double s_lo, s_hi;
  __shared__ double om[kQMax], rh[kQMax];
  const int lane = threadIdx.x;
  const int k = min(q, sc->kbreak);
  for (int i = lane; i < k; i += 32) {
    om[i] = sc->omega[i];
    rh[i] = i < k - 1 ? sc->rho[i] : 0.0;
  }
  __syncwarp();
  if (lane == 0) {
    double lo = INFINITY, hi = -INFINITY, rmax = 0.0;
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(rh[i - 1]) : 0.0) + (i < k - 1 ? fabs(rh[i]) : 0.0);
      lo = fmin(lo, om[i] - r);
      hi = fmax(hi, om[i] + r);
      rmax = fmax(rmax, fabs(rh[i]));
    }
    const double pad = 1e-14 * fmax(fabs(lo), fabs(hi)) + 1e-300;
    s_lo = lo - pad;
    s_hi = hi + pad;
    sc->k = k;
  }
  __syncwarp();
  double lo = s_lo, hi = s_hi;
  const double pivmin = 1e-300;
  for (int it = 0; it < 64; ++it) {
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < k; ++i) {
      const double r2 = i > 0 ? rh[i - 1] * rh[i - 1] : 0.0;
      d = (om[i] - x) - (i > 0 ? r2 / d : 0.0);
      if (fabs(d) < pivmin) d = -pivmin;
      cnt += d < 0.0;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, cnt >= 1);
    const int first = ball ? __ffs(ball) - 1 : 32;
    const double nlo = first == 0 ? lo : lo + (hi - lo) * (double)first / 33.0;
    const double nhi = first == 32 ? hi : lo + (hi - lo) * (double)(first + 1) / 33.0;
    if (nhi - nlo >= hi - lo || !(nhi > nlo)) break;
    lo = nlo;
    hi = nhi;
    if (hi - lo <= 2e-16 * fmax(fabs(lo), fabs(hi))) break;
  }
  if (lane == 0) {
    const double th = 0.5 * (lo + hi);
    sc->theta = th;
    // inverse iteration: (T - th I) x = b, LU without pivoting (Thomas) with a pivot guard
    double xv[kQMax], dd[kQMax];
    for (int i = 0; i < k; ++i) xv[i] = 1.0;
    const double guard = 1e-15 * fmax(fabs(hi), 1e-300);
    for (int sweep = 0; sweep < 3; ++sweep) {
      // forward elimination
      double dprev = 0.0;
      for (int i = 0; i < k; ++i) {
        double di = om[i] - th;
        if (i > 0) {
          const double l = rh[i - 1] / dprev;
          di -= l * rh[i - 1];
          xv[i] -= l * xv[i - 1];
        }
        if (fabs(di) < guard) di = di < 0.0 ? -guard : guard;
        dd[i] = di;
        dprev = di;
      }
      // back substitution
      xv[k - 1] /= dd[k - 1];
      for (int i = k - 2; i >= 0; --i) xv[i] = (xv[i] - rh[i] * xv[i + 1]) / dd[i];
      double nrm = 0.0;
      for (int i = 0; i < k; ++i) nrm += xv[i] * xv[i];
      nrm = 1.0 / sqrt(nrm);
      for (int i = 0; i < k; ++i) xv[i] *= nrm;
    }
    for (int i = 0; i < k; ++i) sc->svec[i] = xv[i];
  }
}

// v = sum_i s_i v_i (Alg. 2 line 13), ||v||.
__global__ void k_pr_combine(const double2 *__restrict__ U, double2 *__restrict__ v, int64_t n, PrScal *sc,
                             double *partials) {
  __shared__ double red[32];
  __shared__ double coef[kQMax];
  const int k = sc->k;
  for (int i = threadIdx.x; i < k; i += blockDim.x) coef[i] = sc->svec[i] * sc->scale[i];
  __syncthreads();
  double s[1] = {0.0};
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) acc = cadd(acc, cscale(__ldg(U + (size_t)i * n + m), coef[i]));
    v[m] = acc;
    s[0] += acc.x * acc.x + acc.y * acc.y;
  }
  if (grid_sum<1>(s, partials, &sc->ticket[3], red) && threadIdx.x == 0) sc->vnrm = sqrt(s[0]);
}

// v <- v / ||v||; vv = ||v||^2, c = v^* C~ v, g = v^* Omega (R complex).
template <int RC>  // the sketch rank as a compile-time constant: 1 + 2 RC sums, no dead accumulators
__global__ void k_pr_vnorm(double2 *__restrict__ v, const double2 *__restrict__ Om, int64_t n, int R, double rsn,
                           PrScal *sc, double *partials) {
  constexpr int NV = 1 + 2 * RC;
  __shared__ double red[32 * NV];
  const double inv = 1.0 / sc->vnrm;
  double s[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) s[i] = 0.0;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = cscale(v[m], inv);
    v[m] = x;
    s[0] += x.x * x.x + x.y * x.y;
#pragma unroll
    for (int kk = 0; kk < RC; ++kk) {
      const double2 o = __ldg(Om + (size_t)kk * n + m);
      s[1 + 2 * kk] += x.x * o.x + x.y * o.y;  // conj(x) o
      s[2 + 2 * kk] += x.x * o.y - x.y * o.x;
    }
  }
  if (grid_sum<NV>(s, partials, &sc->ticket[4], red) && threadIdx.x == 0) {
    sc->vv = s[0];
    sc->cval = s[0] * rsn;
    for (int i = 0; i < 2 * RC; ++i) sc->g[i] = s[1 + i];
  }
}
typedef void (*VnFn)(double2 *, const double2 *, int64_t, int, double, PrScal *, double *);
const VnFn kVnorm[kRMax] = {k_pr_vnorm<1>,  k_pr_vnorm<2>,  k_pr_vnorm<3>,  k_pr_vnorm<4>,
                            k_pr_vnorm<5>,  k_pr_vnorm<6>,  k_pr_vnorm<7>,  k_pr_vnorm<8>,
                            k_pr_vnorm<9>,  k_pr_vnorm<10>, k_pr_vnorm<11>, k_pr_vnorm<12>,
                            k_pr_vnorm<13>, k_pr_vnorm<14>, k_pr_vnorm<15>, k_pr_vnorm<16>};

__device__ __forceinline__ double dual_gamma(int64_t t, double beta0, double nz) {
  if (nz == 0.0) return beta0;
  const double sq = sqrt((double)(t + 1));
  const double g = (4.0 * beta0) / (((double)(t + 1) * sq) * nz);
  return g < beta0 ? g : beta0;
}

// Primal update (Alg. 4 line 8) with the trace-bounded LMO: z <- (1 - eta) z + eta [xi < 0] kappa_j h;
// gap / bound sums of the state before the update; ||z - b~||^2 after; gamma; tau, p; the log record.
__global__ void k_pr_primal(double *__restrict__ z, const double *__restrict__ y, const double *__restrict__ bt,
                            const double *__restrict__ h, const double *__restrict__ kappa, int64_t n, int L,
                            int64_t t, int q, double eta, double beta, double beta0, PrScal *sc, scg_pr_rec *log,
                            double *partials) {
  __shared__ double red[32 * 5];
  const bool on = sc->xi < 0.0;
  const double ome = 1.0 - eta;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t d = n * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = z[i], yi = __ldg(y + i), bi = __ldg(bt + i);
    const double e = zi - bi;
    s[0] += yi * zi;
    s[1] += e * zi;
    s[2] += yi * bi;
    s[3] += e * (zi + bi);
    const double zn = on ? ome * zi + eta * (__ldg(kappa + i / n) * __ldg(h + i)) : ome * zi;
    z[i] = zn;
    const double e1 = zn - bi;
    s[4] += e1 * e1;
  }
  if (grid_sum<5>(s, partials, &sc->ticket[5], red) && threadIdx.x == 0) {
    const double nz = s[4];
    const double gam = dual_gamma(t, beta0, nz);
    const double p_t = sc->p;
    const double ax = fmin(sc->xi, 0.0);
    scg_pr_rec r;
    r.t = t;
    r.q = q;
    r.k = sc->k;
    r.theta = sc->theta;
    r.xi = sc->xi;
    r.c = sc->cval;
    r.gap = (p_t + s[0]) + beta * s[1] - ax;
    r.bound = (p_t + s[2]) + 0.5 * beta * s[3] - ax;
    sc->tau = on ? ome * sc->tau + eta * sc->vv : ome * sc->tau;
    sc->p = on ? ome * sc->p + eta * sc->cval : ome * sc->p;
    r.p = sc->p;
    r.tau = sc->tau;
    r.znorm = sqrt(nz);
    r.gamma = gam;
    sc->gamma = gam;
    sc->nz = nz;
    log[t - 1] = r;
  }
}

// Dual update (Alg. 4 line 9) and the weights of iteration t+1: y <- y + gamma (z - b~),
// wk = kappa_j (y + beta_{t+1} (z - b~)).  (gamma < 0 is the init / hook form: y untouched.)
__global__ void k_pr_dual(const double *__restrict__ z, double *__restrict__ y, const double *__restrict__ bt,
                          double *__restrict__ wk, const double *__restrict__ kappa, int64_t n, int L, double beta1,
                          const PrScal *__restrict__ sc, int update_y) {
  const double gam = update_y ? sc->gamma : 0.0;
  const int64_t d = n * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    const double e = z[i] - bt[i];
    double yi = y[i];
    if (update_y) {
      yi = yi + gam * e;
      y[i] = yi;
    }
    wk[i] = __ldg(kappa + i / n) * (yi + beta1 * e);
  }
}

// Sketch (Alg. 4 line 10): S_k <- (1 - eta) S_k + eta [xi < 0] v g_k.
__global__ void k_pr_sketch(double2 *__restrict__ S, const double2 *__restrict__ v, int64_t n, int R, double eta,
                            const PrScal *__restrict__ sc) {
  const bool on = sc->xi < 0.0;
  const double ome = 1.0 - eta;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    const double2 vm = v[m];
    for (int kk = 0; kk < R; ++kk) {
      double2 sk = S[(size_t)kk * n + m];
      sk = cscale(sk, ome);
      if (on) sk = cadd(sk, cscale(cmul(vm, make_double2(sc->g[2 * kk], sc->g[2 * kk + 1])), eta));
      S[(size_t)kk * n + m] = sk;
    }
  }
}

__global__ void k_pr_omega(double2 *__restrict__ Om, int64_t n, int R, uint64_t seed) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x)
    for (int kk = 0; kk < R; ++kk)
      Om[(size_t)kk * n + m] = make_double2(scg_normal(seed, SCG_STREAM_OMEGA, (uint32_t)kk, (uint64_t)(2 * m)),
                                            scg_normal(seed, SCG_STREAM_OMEGA, (uint32_t)kk, (uint64_t)(2 * m + 1)));
}

// Column statistics of psi for the scaling (reading R38): per j, N_j = ||psi_j||^2 and
// M_jk = <|psi_j|^2, |psi_k|^2>; grid (blocks, L), partials [block][j][L + 1].
__global__ void k_pr_psistats(const uint8_t *__restrict__ codes, const double2 *__restrict__ book, int64_t n, int L,
                              double *__restrict__ part) {
  __shared__ double mag[256];
  __shared__ double red[32];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) mag[i] = book[i].x * book[i].x + book[i].y * book[i].y;
  __syncthreads();
  const int j = blockIdx.y;
  for (int k = 0; k <= L; ++k) {
    double s[1] = {0.0};
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
      const double aj = mag[codes[(size_t)j * n + m]];
      s[0] += k == L ? aj : aj * mag[codes[(size_t)k * n + m]];
    }
    block_sum<1>(s, red);
    if (threadIdx.x == 0) part[((size_t)blockIdx.x * L + j) * (L + 1) + k] = s[0];
    __syncthreads();
  }
}

// natural [L][n] (l = k2 + n2 k1) <-> p-order [L][n] (p = k2 n1 + k1); optional per-j scale.
__global__ void k_pr_perm(const double *__restrict__ src, double *__restrict__ dst, int n1, int n2, int L,
                          const double *__restrict__ jscale, double mul, int to_p) {
  const int64_t n = (int64_t)n1 * n2, d = n * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / n, p = i - j * n;
    const int64_t k2 = p / n1, k1 = p - k2 * n1;
    const int64_t l = k2 + (int64_t)n2 * k1;
    const double sj = jscale ? jscale[j] * mul : mul;
    if (to_p) dst[i] = src[j * n + l] * sj;
    else dst[j * n + l] = src[i] * sj;
  }
}

// G = A^* B for column-major n x R complex A, B (R <= 16): per block partials, fixed-order total.
__global__ void k_pr_gram(const double2 *__restrict__ A, const double2 *__restrict__ B, int64_t n, int R,
                          double *__restrict__ part, double *__restrict__ G, unsigned *ticket) {
  constexpr int CH = 32;
  __shared__ double2 sa[CH][kRMax], sb[CH][kRMax];
  __shared__ bool s_last;
  const int pr = threadIdx.x / R, pc = threadIdx.x % R;  // pair (pr, pc) for threadIdx.x < R*R
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t base = (int64_t)blockIdx.x * CH; base < n; base += (int64_t)gridDim.x * CH) {
    for (int e = threadIdx.x; e < CH * R; e += blockDim.x) {
      const int rr = e / R, cc = e % R;
      const int64_t m = base + rr;
      sa[rr][cc] = m < n ? A[(size_t)cc * n + m] : make_double2(0.0, 0.0);
      sb[rr][cc] = m < n ? B[(size_t)cc * n + m] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (threadIdx.x < R * R)
      for (int rr = 0; rr < CH; ++rr) acc = cadd(acc, cmulc(sb[rr][pc], sa[rr][pr]));  // conj(A) B
    __syncthreads();
  }
  if (threadIdx.x < R * R) {
    part[((size_t)blockIdx.x * R * R + threadIdx.x) * 2] = acc.x;
    part[((size_t)blockIdx.x * R * R + threadIdx.x) * 2 + 1] = acc.y;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < R * R) {
    double re = 0.0, im = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      re += __ldcg(part + ((size_t)b * R * R + threadIdx.x) * 2);
      im += __ldcg(part + ((size_t)b * R * R + threadIdx.x) * 2 + 1);
    }
    G[threadIdx.x * 2] = re;
    G[threadIdx.x * 2 + 1] = im;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// Y = (A + nu B) M for column-major n x R complex A, B and an R x R complex M (row-major [r][c]).
__global__ void k_pr_rmul(const double2 *__restrict__ A, const double2 *__restrict__ B, double nu,
                          const double2 *__restrict__ Mx, int64_t n, int R, double2 *__restrict__ Yo) {
  __shared__ double2 sM[kRMax * kRMax];
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) sM[i] = Mx[i];
  __syncthreads();
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    double2 row[kRMax];
    for (int c = 0; c < R; ++c) {
      double2 x = A[(size_t)c * n + m];
      if (B) x = cadd(x, cscale(B[(size_t)c * n + m], nu));
      row[c] = x;
    }
    for (int c = 0; c < R; ++c) {
      double2 s = make_double2(0.0, 0.0);
      for (int r = 0; r < R; ++r) s = cadd(s, cmul(row[r], sM[r * R + c]));
      Yo[(size_t)c * n + m] = s;
    }
  }
}

__global__ void k_pr_scalecol(const double2 *__restrict__ U, double s, int64_t n, double2 *__restrict__ out) {
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x)
    out[m] = cscale(U[m], s);
}

// ------------------------------------------------------------------ host helpers
bool factor_plan(int N, Plan *P) {
  const CPlan c = make_cplan(N);
  if (c.ns == 0) return false;
  P->N = N;
  P->ns = c.ns;
  for (int s = 0; s < c.ns; ++s) {
    P->R[s] = c.R[s];
    P->Ns[s] = c.Ns[s];
  }
  return true;
}
int plan_rmin(const Plan &P) { return make_cplan(P.N).rmin; }
// Transforms per block: a compile-time variant with TM = 4 (then 2) when it divides the other dimension and
// fits 512 threads; else the runtime plan with the largest TM | other, TM * N / rmin <= 512, TM * N * 16 B <= 64 KB.
// prefer2: try two transforms per block first (k_pr_b at length 1000: 214 vs 249 us with four).
int choose_tm(const Plan &P, int other, bool force2, bool generic, bool prefer2) {
  const int per = P.N / plan_rmin(P);
  const int per_ct = P.N / make_cplan(P.N, true).rmin;  // compile-time plans may use radix 10
  for (int tm : {prefer2 ? 2 : 4, prefer2 ? 4 : 2})
    if (!generic && !(force2 && tm == 4) && other % tm == 0 && tm * per_ct <= 512 && find_variant(P.N, tm))
      return tm;
  int best = 1;
  for (int tm = 1; tm <= 64 && tm <= other; ++tm) {
    if (other % tm) continue;
    if (tm * per > 512 || (size_t)tm * P.N * 16 > 65536) break;
    best = tm;
  }
  return best;
}

std::vector<double2> twiddles(int64_t N, int64_t count, int64_t stride) {
  std::vector<double2> t((size_t)count);
  for (int64_t e = 0; e < count; ++e) {
    const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)((e * stride) % N) /
                            (long double)N;
    t[(size_t)e] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  return t;
}

// Hermitian Jacobi eigensolver (cyclic), ascending eigenvalues; A is row-major R x R.
void herm_eig(std::vector<cplx> A, int R, std::vector<double> &w, std::vector<cplx> &V) {
  V.assign((size_t)R * R, cplx(0.0, 0.0));
  for (int i = 0; i < R; ++i) V[(size_t)i * R + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        tot += std::norm(A[(size_t)i * R + j]);
        if (i != j) off += std::norm(A[(size_t)i * R + j]);
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < R; ++p)
      for (int q = p + 1; q < R; ++q) {
        const cplx apq = A[(size_t)p * R + q];
        const double mag = std::abs(apq);
        if (mag == 0.0) continue;
        const double app = A[(size_t)p * R + p].real(), aqq = A[(size_t)q * R + q].real();
        const cplx ph = apq / mag;  // a_pq = |a_pq| e^{i phi}
        const double theta = 0.5 * (aqq - app) / mag;
        const double tt = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(tt * tt + 1.0), s = tt * c;
        // rotation J: columns p, q: [c, s e^{i phi}; -s e^{-i phi}, c] applied as A <- J^* A J
        for (int k = 0; k < R; ++k) {  // A <- A J
          const cplx akp = A[(size_t)k * R + p], akq = A[(size_t)k * R + q];
          A[(size_t)k * R + p] = c * akp - s * std::conj(ph) * akq;
          A[(size_t)k * R + q] = s * ph * akp + c * akq;
        }
        for (int k = 0; k < R; ++k) {  // A <- J^* A
          const cplx apk = A[(size_t)p * R + k], aqk = A[(size_t)q * R + k];
          A[(size_t)p * R + k] = c * apk - s * ph * aqk;
          A[(size_t)q * R + k] = s * std::conj(ph) * apk + c * aqk;
        }
        for (int k = 0; k < R; ++k) {
          const cplx vkp = V[(size_t)k * R + p], vkq = V[(size_t)k * R + q];
          V[(size_t)k * R + p] = c * vkp - s * std::conj(ph) * vkq;
          V[(size_t)k * R + q] = s * ph * vkp + c * vkq;
        }
      }
  }
  std::vector<int> idx(R);
  for (int i = 0; i < R; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(),
            [&](int a, int b) { return A[(size_t)a * R + a].real() < A[(size_t)b * R + b].real(); });
  std::vector<cplx> V2((size_t)R * R);
  w.resize(R);
  for (int c = 0; c < R; ++c) {
    w[c] = A[(size_t)idx[c] * R + idx[c]].real();
    for (int r = 0; r < R; ++r) V2[(size_t)r * R + c] = V[(size_t)r * R + idx[c]];
  }
  V = V2;
}

// B = C^* C with C upper triangular (row-major); false if not positive definite.
bool chol_upper(const std::vector<cplx> &B, int R, std::vector<cplx> &C) {
  C.assign((size_t)R * R, cplx(0.0, 0.0));
  for (int j = 0; j < R; ++j) {
    double d = B[(size_t)j * R + j].real();
    for (int k = 0; k < j; ++k) d -= std::norm(C[(size_t)k * R + j]);
    if (!(d > 0.0)) return false;
    const double cjj = std::sqrt(d);
    C[(size_t)j * R + j] = cjj;
    for (int i = j + 1; i < R; ++i) {
      cplx s = B[(size_t)j * R + i];
      for (int k = 0; k < j; ++k) s -= std::conj(C[(size_t)k * R + j]) * C[(size_t)k * R + i];
      C[(size_t)j * R + i] = s / cjj;
    }
  }
  return true;
}
std::vector<cplx> inv_upper(const std::vector<cplx> &C, int R) {
  std::vector<cplx> X((size_t)R * R, cplx(0.0, 0.0));
  for (int c = 0; c < R; ++c) {
    for (int r = c; r >= 0; --r) {
      cplx s = (r == c) ? cplx(1.0, 0.0) : cplx(0.0, 0.0);
      for (int k = r + 1; k <= c; ++k) s -= C[(size_t)r * R + k] * X[(size_t)k * R + c];
      X[(size_t)r * R + c] = s / C[(size_t)r * R + r];
    }
  }
  return X;
}
double matlab_eps(double x) {
  if (x == 0.0) return std::ldexp(1.0, -1074);
  int e;
  std::frexp(std::fabs(x), &e);
  return std::ldexp(1.0, e - 1 - 52);
}

}  // namespace

// ------------------------------------------------------------------ context
enum { KS_START, KS_F1, KS_B, KS_C, KS_RECUR, KS_TRI, KS_COMB, KS_VNORM, KS_F1M, KS_BM, KS_CM, KS_PRIMAL, KS_DUAL,
       KS_SKETCH, KS_COUNT };
static const char *kKsNames[KS_COUNT] = {"k_pr_start", "k_pr_f1", "k_pr_b", "k_pr_c", "k_pr_recur",
                                         "k_pr_tridiag", "k_pr_combine", "k_pr_vnorm", "k_pr_f1(monitor)",
                                         "k_pr_b(monitor)", "k_pr_c(monitor)", "k_pr_primal", "k_pr_dual",
                                         "k_pr_sketch"};

struct scg_pr_ctx {
  int64_t n;
  int L, R, n1, n2, tm1, tm2, nthr1, nthr2;
  size_t smem1, smem2, smemc;
  int gf1, gb, gc;  // persistent grids of the FFT kernels
  Plan P1, P2;  // P1: length n1 (k_pr_b), P2: length n2 (k_pr_f1 / k_pr_c)
  const Variant *v1, *v2;  // v1: k_pr_f1 / k_pr_c (length n2, tm1), v2: k_pr_b (length n1, tm2)
  F1Fn kf1;
  BFn kb;
  CFn kc;
  double alpha, beta0, opnorm, rsn;
  uint64_t seed;
  uint32_t flags;
  int64_t t;
  int failed;
  bool have_rec;
  cudaStream_t st;
  // device
  uint8_t *codes;
  double2 *book, *tw1, *tw2, *twlo, *twhi;
  double *kappa, *bt, *z, *y, *wk, *h;
  double2 *Y, *a, *v, *Om, *S, *U, *tmpA, *tmpB;
  int64_t ucap;  // Lanczos vectors allocated
  double *partials;
  PrScal *sc;
  scg_pr_rec *log;
  int64_t logcap;
  double *G;
  double2 *Mx;
  unsigned *gticket;
  std::vector<double> h_kappa;
  std::vector<double> lam;
  std::vector<double2> Uhost;
  // profiling
  cudaEvent_t ev[2 * 4096];
  int nev;
  int evk[4096];
  int64_t ks_launch[KS_COUNT];
  double ks_ms[KS_COUNT];
  double ks_bytes[KS_COUNT];
};

#define PR_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "scg_phase: %s failed: %s (%s:%d)\n", #x, cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                                   \
      c->failed = 1;                                                                       \
      return SCG_ECUDA;                                                                    \
    }                                                                                      \
  } while (0)

static int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}

static void prof_begin(scg_pr_ctx *c, int k) {
  if (!(c->flags & SCG_PR_PROFILE) || c->nev >= 4096) return;
  c->evk[c->nev] = k;
  cudaEventRecord(c->ev[2 * c->nev], c->st);
}
static void prof_end(scg_pr_ctx *c) {
  if (!(c->flags & SCG_PR_PROFILE) || c->nev >= 4096) return;
  cudaEventRecord(c->ev[2 * c->nev + 1], c->st);
  c->nev++;
}
static void prof_collect(scg_pr_ctx *c) {
  if (!(c->flags & SCG_PR_PROFILE)) return;
  cudaStreamSynchronize(c->st);
  for (int i = 0; i < c->nev; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]);
    c->ks_ms[c->evk[i]] += ms;
    c->ks_launch[c->evk[i]]++;
  }
  c->nev = 0;
}

// Algorithmic bytes per launch.
static void set_bytes(scg_pr_ctx *c) {
  const double n = (double)c->n, L = c->L, R = c->R;
  c->ks_bytes[KS_START] = 16 * n;
  c->ks_bytes[KS_F1] = c->ks_bytes[KS_F1M] = 16 * n + L * n + 16 * L * n;  // x, codes, Y
  c->ks_bytes[KS_B] = 32 * L * n + 8 * L * n;                               // Y in/out, w
  c->ks_bytes[KS_BM] = 32 * L * n + 16 * L * n;                             // + h
  c->ks_bytes[KS_C] = 16 * L * n + L * n + 16 * n + 16 * n;                 // Y, codes, x, a
  c->ks_bytes[KS_CM] = 16 * L * n + L * n + 16 * n;
  c->ks_bytes[KS_RECUR] = 64 * n;
  c->ks_bytes[KS_TRI] = 0;
  c->ks_bytes[KS_COMB] = 0;  // depends on k (reported per launch by the bench)
  c->ks_bytes[KS_VNORM] = 32 * n + 16 * R * n;
  c->ks_bytes[KS_PRIMAL] = 5 * 8 * L * n + 8 * L * n;  // z, y, b, h in; z out
  c->ks_bytes[KS_DUAL] = 3 * 8 * L * n + 2 * 8 * L * n;
  c->ks_bytes[KS_SKETCH] = 16 * n + 32 * R * n;
}

static int launch_matvec(scg_pr_ctx *c, const double2 *x, const double *scale_p, double2 *out, int step,
                         int mode /* 0 lanczos, 1 monitor, 2 hook */) {
  prof_begin(c, mode == 1 ? KS_F1M : KS_F1);
  c->kf1<<<c->gf1, c->nthr1, c->smem1, c->st>>>(x, scale_p, step, c->sc, c->codes, c->book, c->Y, c->P2, c->tw2,
                                                   c->n1, c->n2, c->tm1, c->L);
  prof_end(c);
  prof_begin(c, mode == 1 ? KS_BM : KS_B);
  c->kb<<<c->gb, c->nthr2, c->smem2, c->st>>>(c->Y, c->wk, c->h, mode == 1 ? 1 : 0, step, c->sc, c->P1, c->tw1,
                                                 c->twlo, c->twhi, c->n1, c->n2, c->tm2, c->L);
  prof_end(c);
  prof_begin(c, mode == 1 ? KS_CM : KS_C);
  c->kc<<<c->gc, c->nthr1, c->smemc, c->st>>>(c->Y, x, scale_p, out, c->codes, c->book, c->P2, c->tw2, c->n1,
                                                 c->n2, c->tm1, c->L, c->rsn, mode, step, c->sc, c->partials);
  prof_end(c);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "scg_phase: matvec launch failed: %s\n", cudaGetErrorString(e));
    c->failed = 1;
    return SCG_ECUDA;
  }
  return SCG_OK;
}

static int ensure_ucap(scg_pr_ctx *c, int q) {
  if (q + 1 <= c->ucap) return SCG_OK;
  double2 *nu = nullptr;
  const int64_t cap = std::max<int64_t>(q + 1, c->ucap * 3 / 2);
  PR_CUDA(cudaStreamSynchronize(c->st));
  PR_CUDA(cudaMalloc(&nu, sizeof(double2) * (size_t)cap * c->n));
  if (c->U) cudaFree(c->U);
  c->U = nu;
  c->ucap = cap;
  return SCG_OK;
}

static int q_of(int64_t t, int64_t n) {
  const double x = std::sqrt(std::sqrt((double)t)) * std::log((double)n);
  int64_t q = (int64_t)std::ceil(x);
  if (q < 2) q = 2;
  if (q > n - 1) q = n - 1;
  return (int)q;
}

static int pr_init_device(scg_pr_ctx *c, const std::vector<uint8_t> &codes, const std::vector<double2> &book,
                          const double *b);

extern "C" {

int scg_pr_init(int64_t n, int32_t L, const double *psi, const double *b, int32_t R, double alpha, double beta0,
                uint64_t seed, uint32_t flags, scg_pr_ctx **out) {
  if (!out || !psi || !b) return SCG_EINVAL;
  *out = nullptr;
  if (n < 4 || L < 1 || L > kLMax || R < 1 || R > kRMax || R > n || !(alpha > 0.0) || !(beta0 > 0.0))
    return SCG_EINVAL;
  if ((int64_t)L * n >= (int64_t)1 << 31) return SCG_EUNSUPPORTED;
  // n = n1 n2, both {2,3,5}-smooth in [2, 4096], n1 <= n2 closest to sqrt(n)
  int n1 = 0, n2 = 0;
  Plan P1{}, P2{};
  for (int64_t d = (int64_t)std::floor(std::sqrt((double)n)); d >= 2; --d) {
    if (n % d) continue;
    Plan a{}, bb{};
    if (factor_plan((int)d, &a) && n / d <= kSubMax && factor_plan((int)(n / d), &bb)) {
      n1 = (int)d;
      n2 = (int)(n / d);
      P1 = a;
      P2 = bb;
      break;
    }
  }
  if (!n1) return SCG_EUNSUPPORTED;
  // codebook of psi values: open addressing on the bit patterns (1024 slots for at most 256 values)
  std::vector<double2> book(256, make_double2(0.0, 0.0));
  std::vector<uint8_t> codes((size_t)L * n);
  {
    std::vector<uint64_t> kre(1024), kim(1024);
    std::vector<int> kc(1024, -1);
    int ncode = 0;
    for (int64_t i = 0; i < (int64_t)L * n; ++i) {
      uint64_t re, im;
      memcpy(&re, psi + 2 * i, 8);
      memcpy(&im, psi + 2 * i + 1, 8);
      int slot = (int)(((re * 0x9E3779B97F4A7C15ull) ^ (im * 0xC2B2AE3D27D4EB4Full)) >> 54);
      while (kc[slot] >= 0 && (kre[slot] != re || kim[slot] != im)) slot = (slot + 1) & 1023;
      if (kc[slot] < 0) {
        if (ncode >= 256) return SCG_EUNSUPPORTED;
        kre[slot] = re;
        kim[slot] = im;
        kc[slot] = ncode;
        book[ncode++] = make_double2(psi[2 * i], psi[2 * i + 1]);
      }
      codes[(size_t)i] = (uint8_t)kc[slot];
    }
  }
  scg_pr_ctx *c = static_cast<scg_pr_ctx *>(::operator new(sizeof(scg_pr_ctx)));
  memset((void *)c, 0, sizeof(*c));
  new (&c->h_kappa) std::vector<double>();
  new (&c->lam) std::vector<double>();
  new (&c->Uhost) std::vector<double2>();
  c->n = n;
  c->L = L;
  c->R = R;
  c->n1 = n1;
  c->n2 = n2;
  c->P1 = P1;
  c->P2 = P2;
  c->alpha = alpha;
  c->beta0 = beta0;
  c->seed = seed;
  c->flags = flags;
  c->rsn = 1.0 / std::sqrt((double)n);
  c->tm1 = choose_tm(P2, n1, flags & SCG_PR_TM2, flags & SCG_PR_GENERIC, false);
  c->tm2 = choose_tm(P1, n2, flags & SCG_PR_TM2, flags & SCG_PR_GENERIC, n1 == 1000);
  c->v1 = find_variant(n2, c->tm1);
  c->v2 = find_variant(n1, c->tm2);
  if (!c->v1 || (flags & SCG_PR_GENERIC)) c->v1 = &kGeneric;
  if (!c->v2 || (flags & SCG_PR_GENERIC)) c->v2 = &kGeneric;
  c->kf1 = (flags & SCG_PR_NOPF_F1) ? c->v1->f1n : c->v1->f1;
  c->kb = (flags & SCG_PR_NOPF_B) ? c->v2->bn : c->v2->b;
  c->kc = (flags & SCG_PR_NOPF_C) ? c->v1->cn : c->v1->c;
  c->nthr1 = c->tm1 * (n2 / (c->v1 != &kGeneric ? make_cplan(n2, true).rmin : plan_rmin(P2)));
  c->nthr2 = c->tm2 * (n1 / (c->v2 != &kGeneric ? make_cplan(n1, true).rmin : plan_rmin(P1)));
  c->smem1 = sizeof(double2) * (fft_buf(c->tm1, n2) + n2 + 256);
  c->smem2 = sizeof(double2) * (fft_buf(c->tm2, n1) + n1);
  c->smemc = c->smem1 + sizeof(double2) * (size_t)c->tm1 * n2;
  const int rc = pr_init_device(c, codes, book, b);
  if (rc != SCG_OK) {
    scg_pr_destroy(c);
    return rc;
  }
  *out = c;
  return SCG_OK;
}

}  // extern "C"

static int pr_init_device(scg_pr_ctx *c, const std::vector<uint8_t> &codes, const std::vector<double2> &book,
                          const double *b) {
  const int64_t n = c->n;
  const int L = c->L, R = c->R, n1 = c->n1, n2 = c->n2;
  const double alpha = c->alpha, beta0 = c->beta0;
  const uint64_t seed = c->seed;
  const uint32_t flags = c->flags;
  PR_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  PR_CUDA(cudaFuncSetAttribute(c->kf1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem1));
  PR_CUDA(cudaFuncSetAttribute(c->kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smemc));
  PR_CUDA(cudaFuncSetAttribute(c->kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem2));
  {  // persistent grids: resident blocks per SM x SMs, capped at the tile counts
    int dev = 0, sms = 148, o1 = 1, o2 = 1, o3 = 1;
    PR_CUDA(cudaGetDevice(&dev));
    PR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, c->kf1, c->nthr1, c->smem1));
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, c->kb, c->nthr2, c->smem2));
    PR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, c->kc, c->nthr1, c->smemc));
    c->gf1 = (int)std::min<int64_t>((int64_t)std::max(o1, 1) * sms, (int64_t)(n1 / c->tm1) * L);
    c->gb = (int)std::min<int64_t>((int64_t)std::max(o2, 1) * sms, (int64_t)(n2 / c->tm2) * L);
    c->gc = (int)std::min<int64_t>((int64_t)std::max(o3, 1) * sms, (int64_t)(n1 / c->tm1));
  }
  const size_t dn = (size_t)L * n;
  PR_CUDA(cudaMalloc(&c->codes, dn));
  PR_CUDA(cudaMalloc(&c->book, sizeof(double2) * 256));
  PR_CUDA(cudaMalloc(&c->tw1, sizeof(double2) * n1));
  PR_CUDA(cudaMalloc(&c->tw2, sizeof(double2) * n2));
  const int64_t nhi = (n + 2047) / 2048;
  PR_CUDA(cudaMalloc(&c->twlo, sizeof(double2) * 2048));
  PR_CUDA(cudaMalloc(&c->twhi, sizeof(double2) * nhi));
  PR_CUDA(cudaMalloc(&c->kappa, sizeof(double) * L));
  for (double **p : {&c->bt, &c->z, &c->y, &c->wk, &c->h}) PR_CUDA(cudaMalloc(p, sizeof(double) * dn));
  PR_CUDA(cudaMalloc(&c->Y, sizeof(double2) * dn));
  for (double2 **p : {&c->a, &c->v}) PR_CUDA(cudaMalloc(p, sizeof(double2) * n));
  for (double2 **p : {&c->Om, &c->S, &c->tmpA, &c->tmpB}) PR_CUDA(cudaMalloc(p, sizeof(double2) * (size_t)R * n));
  const size_t npart = (size_t)4096 * (1 + 2 * kRMax) + (size_t)2048 * kLMax * (kLMax + 1);
  PR_CUDA(cudaMalloc(&c->partials, sizeof(double) * npart));
  PR_CUDA(cudaMalloc(&c->sc, sizeof(PrScal)));
  PR_CUDA(cudaMalloc(&c->G, sizeof(double) * 2 * kRMax * kRMax));
  PR_CUDA(cudaMalloc(&c->gticket, sizeof(unsigned)));
  PR_CUDA(cudaMalloc(&c->Mx, sizeof(double2) * kRMax * kRMax));
  PR_CUDA(cudaMemsetAsync(c->sc, 0, sizeof(PrScal), c->st));
  PR_CUDA(cudaMemsetAsync(c->gticket, 0, sizeof(unsigned), c->st));
  for (double *p : {c->z, c->y, c->h}) PR_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * dn, c->st));
  PR_CUDA(cudaMemsetAsync(c->S, 0, sizeof(double2) * (size_t)R * n, c->st));
  PR_CUDA(cudaMemcpyAsync(c->codes, codes.data(), dn, cudaMemcpyHostToDevice, c->st));
  PR_CUDA(cudaMemcpyAsync(c->book, book.data(), sizeof(double2) * 256, cudaMemcpyHostToDevice, c->st));
  std::vector<double2> t1 = twiddles(n1, n1, 1), t2 = twiddles(n2, n2, 1), tlo = twiddles(n, 2048, 1),
                       thi = twiddles(n, nhi, 2048);
  PR_CUDA(cudaMemcpyAsync(c->tw1, t1.data(), sizeof(double2) * n1, cudaMemcpyHostToDevice, c->st));
  PR_CUDA(cudaMemcpyAsync(c->tw2, t2.data(), sizeof(double2) * n2, cudaMemcpyHostToDevice, c->st));
  PR_CUDA(cudaMemcpyAsync(c->twlo, tlo.data(), sizeof(double2) * 2048, cudaMemcpyHostToDevice, c->st));
  PR_CUDA(cudaMemcpyAsync(c->twhi, thi.data(), sizeof(double2) * nhi, cudaMemcpyHostToDevice, c->st));
  // scaling (reading R38): N_j, M_jk on the device; the L x L eigenvalue on the host
  const int sb = (int)std::min<int64_t>(2048, (n + 255) / 256);
  k_pr_psistats<<<dim3(sb, L), 256, 0, c->st>>>(c->codes, c->book, n, L, c->partials);
  std::vector<double> part((size_t)sb * L * (L + 1));
  PR_CUDA(cudaMemcpyAsync(part.data(), c->partials, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  std::vector<double> tot((size_t)L * (L + 1), 0.0);
  for (int bb = 0; bb < sb; ++bb)
    for (size_t i = 0; i < tot.size(); ++i) tot[i] += part[(size_t)bb * L * (L + 1) + i];
  std::vector<double> cj(L);
  for (int j = 0; j < L; ++j) {
    const double Nj = tot[(size_t)j * (L + 1) + L];
    if (!(Nj > 0.0)) return SCG_EINVAL;
    cj[j] = 1.0 / Nj;
  }
  std::vector<cplx> Gm((size_t)L * L);
  for (int j = 0; j < L; ++j)
    for (int k = 0; k < L; ++k) Gm[(size_t)j * L + k] = cj[j] * cj[k] * tot[(size_t)j * (L + 1) + k];
  std::vector<double> ev;
  std::vector<cplx> EV;
  herm_eig(Gm, L, ev, EV);
  c->opnorm = std::sqrt((double)n * ev[L - 1]);
  c->h_kappa.resize(L);
  for (int j = 0; j < L; ++j) c->h_kappa[j] = cj[j] / c->opnorm;
  PR_CUDA(cudaMemcpyAsync(c->kappa, c->h_kappa.data(), sizeof(double) * L, cudaMemcpyHostToDevice, c->st));
  // b~ = kappa b / alpha in p-order; initial weights wk = kappa (y + beta_1 (z - b~))
  double *bnat = c->wk;
  PR_CUDA(cudaMemcpyAsync(bnat, b, sizeof(double) * dn, cudaMemcpyHostToDevice, c->st));
  k_pr_perm<<<grid_for((int64_t)dn, 256), 256, 0, c->st>>>(bnat, c->bt, n1, n2, L, c->kappa, 1.0 / alpha, 1);
  k_pr_dual<<<grid_for((int64_t)dn, 256), 256, 0, c->st>>>(c->z, c->y, c->bt, c->wk, c->kappa, n, L,
                                                           beta0 * std::sqrt(2.0), c->sc, 0);
  k_pr_omega<<<grid_for(n, 256), 256, 0, c->st>>>(c->Om, n, R, seed);
  PR_CUDA(cudaGetLastError());
  if (flags & SCG_PR_PROFILE)
    for (int i = 0; i < 2 * 4096; ++i) PR_CUDA(cudaEventCreate(&c->ev[i]));
  set_bytes(c);
  c->logcap = 0;
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

extern "C" {

int scg_pr_step(scg_pr_ctx *c, int64_t T) {
  if (!c || c->failed) return SCG_ESTATE;
  if (T < 0) return SCG_EINVAL;
  if (T == 0) return SCG_OK;
  const int64_t n = c->n;
  const int qmax = q_of(c->t + T, n);
  if (qmax > kQMax) return SCG_EUNSUPPORTED;
  int rc = ensure_ucap(c, qmax);
  if (rc) return rc;
  if (c->t + T > c->logcap) {
    const int64_t cap = std::max<int64_t>(c->t + T, c->logcap * 2 + 64);
    scg_pr_rec *nl = nullptr;
    PR_CUDA(cudaStreamSynchronize(c->st));
    PR_CUDA(cudaMalloc(&nl, sizeof(scg_pr_rec) * (size_t)cap));
    if (c->log) {
      PR_CUDA(cudaMemcpy(nl, c->log, sizeof(scg_pr_rec) * (size_t)c->t, cudaMemcpyDeviceToDevice));
      cudaFree(c->log);
    }
    c->log = nl;
    c->logcap = cap;
  }
  const int gb = grid_for(n, 256);
  const int64_t dn = n * c->L;
  const int gd = grid_for(dn, 256);
  const double *scale = reinterpret_cast<const double *>(reinterpret_cast<const char *>(c->sc) +
                                                         offsetof(PrScal, scale));
  for (int64_t it = 0; it < T; ++it) {
    const int64_t t = c->t + 1;
    const double beta = c->beta0 * std::sqrt((double)(t + 1));
    const double beta1 = c->beta0 * std::sqrt((double)(t + 2));
    const double eta = 2.0 / (double)(t + 1);
    const int q = q_of(t, n);
    prof_begin(c, KS_START);
    k_pr_start<<<gb, 256, 0, c->st>>>(c->U, n, c->seed, t, c->sc, c->partials);
    prof_end(c);
    for (int i = 1; i <= q; ++i) {
      rc = launch_matvec(c, c->U + (size_t)(i - 1) * n, scale + (i - 1), c->a, i, 0);
      if (rc) return rc;
      if (i < q) {
        prof_begin(c, KS_RECUR);
        k_pr_recur<<<gb, 256, 0, c->st>>>(c->a, c->U, n, i, c->sc, c->partials);
        prof_end(c);
      }
    }
    prof_begin(c, KS_TRI);
    k_pr_tridiag<<<1, 32, 0, c->st>>>(c->sc, q);
    prof_end(c);
    prof_begin(c, KS_COMB);
    k_pr_combine<<<gb, 256, 0, c->st>>>(c->U, c->v, n, c->sc, c->partials);
    prof_end(c);
    prof_begin(c, KS_VNORM);
    kVnorm[c->R - 1]<<<gb, 256, 0, c->st>>>(c->v, c->Om, n, c->R, c->rsn, c->sc, c->partials);
    prof_end(c);
    rc = launch_matvec(c, c->v, nullptr, c->a, 0, 1);
    if (rc) return rc;
    prof_begin(c, KS_PRIMAL);
    k_pr_primal<<<gd, 256, 0, c->st>>>(c->z, c->y, c->bt, c->h, c->kappa, n, c->L, t, q, eta, beta, c->beta0, c->sc,
                                       c->log, c->partials);
    prof_end(c);
    prof_begin(c, KS_DUAL);
    k_pr_dual<<<gd, 256, 0, c->st>>>(c->z, c->y, c->bt, c->wk, c->kappa, n, c->L, beta1, c->sc, 1);
    prof_end(c);
    prof_begin(c, KS_SKETCH);
    k_pr_sketch<<<gb, 256, 0, c->st>>>(c->S, c->v, n, c->R, eta, c->sc);
    prof_end(c);
    PR_CUDA(cudaGetLastError());
    c->t = t;
    if ((c->flags & SCG_PR_PROFILE) && c->nev > 4000) prof_collect(c);
  }
  c->have_rec = false;
  PR_CUDA(cudaStreamSynchronize(c->st));
  prof_collect(c);
  return SCG_OK;
}

int scg_pr_iter_log(scg_pr_ctx *c, scg_pr_rec *out, int64_t cap, int64_t *count) {
  if (!c || c->failed) return SCG_ESTATE;
  const int64_t m = std::min<int64_t>(cap, c->t);
  if (m > 0) PR_CUDA(cudaMemcpy(out, c->log, sizeof(scg_pr_rec) * (size_t)m, cudaMemcpyDeviceToHost));
  if (count) *count = m;
  return SCG_OK;
}

int scg_pr_get_state(scg_pr_ctx *c, int32_t which, double *out) {
  if (!c || c->failed) return SCG_ESTATE;
  const int64_t n = c->n, dn = n * c->L;
  PR_CUDA(cudaStreamSynchronize(c->st));
  switch (which) {
    case 0:
    case 1:
    case 5: {
      const double *src = which == 0 ? c->z : which == 1 ? c->y : c->bt;
      double *tmp = reinterpret_cast<double *>(c->Y);
      k_pr_perm<<<grid_for(dn, 256), 256, 0, c->st>>>(src, tmp, c->n1, c->n2, c->L, nullptr, 1.0, 0);
      PR_CUDA(cudaMemcpyAsync(out, tmp, sizeof(double) * dn, cudaMemcpyDeviceToHost, c->st));
      break;
    }
    case 2: PR_CUDA(cudaMemcpyAsync(out, c->v, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->st)); break;
    case 3: PR_CUDA(cudaMemcpyAsync(out, c->S, sizeof(double2) * n * c->R, cudaMemcpyDeviceToHost, c->st)); break;
    case 4: PR_CUDA(cudaMemcpyAsync(out, c->Om, sizeof(double2) * n * c->R, cudaMemcpyDeviceToHost, c->st)); break;
    case 6: memcpy(out, c->h_kappa.data(), sizeof(double) * c->L); break;
    case 7: {
      PrScal h;
      PR_CUDA(cudaMemcpyAsync(&h, c->sc, sizeof(PrScal), cudaMemcpyDeviceToHost, c->st));
      PR_CUDA(cudaStreamSynchronize(c->st));
      double v[8] = {(double)c->t, h.tau, h.p, c->opnorm, (double)c->n1, (double)c->n2, c->alpha, c->beta0};
      memcpy(out, v, sizeof(v));
      break;
    }
    default: return SCG_EINVAL;
  }
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

static int gram(scg_pr_ctx *c, const double2 *A, const double2 *B, std::vector<cplx> &G) {
  const int R = c->R;
  const int blocks = (int)std::min<int64_t>(1024, (c->n + 31) / 32);
  k_pr_gram<<<blocks, std::max(32, ((R * R + 31) / 32) * 32), 0, c->st>>>(A, B, c->n, R, c->partials, c->G,
                                                                          c->gticket);
  std::vector<double> h((size_t)2 * R * R);
  PR_CUDA(cudaMemcpyAsync(h.data(), c->G, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  G.resize((size_t)R * R);
  for (int i = 0; i < R * R; ++i) G[i] = cplx(h[2 * i], h[2 * i + 1]);
  return SCG_OK;
}

int scg_pr_reconstruct(scg_pr_ctx *c, double *Uout, double *Lam) {
  if (!c || c->failed) return SCG_ESTATE;
  const int R = c->R;
  const int64_t n = c->n;
  std::vector<cplx> G, C, E;
  std::vector<double> w;
  int rc = gram(c, c->S, c->S, G);
  if (rc) return rc;
  herm_eig(G, R, w, E);
  const double nrm = std::sqrt(std::max(w[R - 1], 0.0));
  std::vector<double2> Mh((size_t)R * R);
  // S = 0 (no iteration took H = v v^*): X^ = 0 -- Lam = 0 with an orthonormal basis of range(Omega)
  const bool zero = nrm == 0.0;
  double nu = zero ? 0.0 : std::sqrt((double)n) * matlab_eps(nrm);  // Alg. 3 line 1
  double2 *dM = c->Mx;
  auto upload = [&](const std::vector<cplx> &M) {
    for (int i = 0; i < R * R; ++i) Mh[i] = make_double2(M[i].real(), M[i].imag());
    return cudaMemcpyAsync(dM, Mh.data(), sizeof(double2) * R * R, cudaMemcpyHostToDevice, c->st);
  };
  if (zero) {
    PR_CUDA(cudaMemcpyAsync(c->tmpB, c->Om, sizeof(double2) * (size_t)R * n, cudaMemcpyDeviceToDevice, c->st));
  } else {
    bool ok = false;
    for (int attempt = 0; attempt < 40; ++attempt) {
      // B = Omega^* (S + nu Omega)  (line 2-3)
      std::vector<double2> I((size_t)R * R, make_double2(0.0, 0.0));
      for (int i = 0; i < R; ++i) I[(size_t)i * R + i] = make_double2(1.0, 0.0);
      PR_CUDA(cudaMemcpyAsync(dM, I.data(), sizeof(double2) * R * R, cudaMemcpyHostToDevice, c->st));
      k_pr_rmul<<<grid_for(n, 256), 256, 0, c->st>>>(c->S, c->Om, nu, dM, n, R, c->tmpA);  // S_nu
      rc = gram(c, c->Om, c->tmpA, G);
      if (rc) return rc;
      std::vector<cplx> B((size_t)R * R);
      for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) B[(size_t)i * R + j] = 0.5 * (G[(size_t)i * R + j] + std::conj(G[(size_t)j * R + i]));
      if (chol_upper(B, R, C)) {
        ok = true;
        break;
      }
      nu *= 2.0;
    }
    if (!ok) return SCG_ECHOL;
    // Y = S_nu C^{-1} (line 4), then CholQR: Q = Y R1^{-1}, and the SVD of the R x R factor
    std::vector<cplx> Ci = inv_upper(C, R);
    PR_CUDA(upload(Ci));
    k_pr_rmul<<<grid_for(n, 256), 256, 0, c->st>>>(c->tmpA, nullptr, 0.0, dM, n, R, c->tmpB);  // Y
  }
  // two CholQR rounds: Y = Q Rt
  std::vector<cplx> Rt((size_t)R * R, cplx(0.0, 0.0));
  for (int i = 0; i < R; ++i) Rt[(size_t)i * R + i] = 1.0;
  double2 *src = c->tmpB, *dst = c->tmpA;
  for (int round = 0; round < 2; ++round) {
    rc = gram(c, src, src, G);
    if (rc) return rc;
    std::vector<cplx> R1;
    if (!chol_upper(G, R, R1)) return SCG_ECHOL;
    PR_CUDA(upload(inv_upper(R1, R)));
    k_pr_rmul<<<grid_for(n, 256), 256, 0, c->st>>>(src, nullptr, 0.0, dM, n, R, dst);
    std::vector<cplx> Rn((size_t)R * R, cplx(0.0, 0.0));  // Rt <- R1 Rt
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j)
        for (int k = 0; k < R; ++k) Rn[(size_t)i * R + j] += R1[(size_t)i * R + k] * Rt[(size_t)k * R + j];
    Rt = Rn;
    std::swap(src, dst);
  }
  // Y = Q Rt;  Rt Rt^* = W diag(sigma^2) W^*  ->  U = Q W, Lam = max(sigma^2 - nu, 0)  (line 5)
  std::vector<cplx> RR((size_t)R * R, cplx(0.0, 0.0));
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j)
      for (int k = 0; k < R; ++k) RR[(size_t)i * R + j] += Rt[(size_t)i * R + k] * std::conj(Rt[(size_t)j * R + k]);
  herm_eig(RR, R, w, E);
  std::vector<cplx> Wd((size_t)R * R);  // descending order
  c->lam.assign(R, 0.0);
  for (int col = 0; col < R; ++col) {
    const int s = R - 1 - col;
    c->lam[col] = zero ? 0.0 : std::max(w[s] - nu, 0.0);
    for (int r = 0; r < R; ++r) Wd[(size_t)r * R + col] = E[(size_t)r * R + s];
  }
  PR_CUDA(upload(Wd));
  k_pr_rmul<<<grid_for(n, 256), 256, 0, c->st>>>(src, nullptr, 0.0, dM, n, R, dst);
  c->Uhost.resize((size_t)R * n);
  PR_CUDA(cudaMemcpyAsync(c->Uhost.data(), dst, sizeof(double2) * (size_t)R * n, cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  // keep U on the device for scg_pr_signal
  if (dst != c->tmpA) PR_CUDA(cudaMemcpyAsync(c->tmpA, dst, sizeof(double2) * (size_t)R * n,
                                              cudaMemcpyDeviceToDevice, c->st));
  if (Uout) memcpy(Uout, c->Uhost.data(), sizeof(double2) * (size_t)R * n);
  if (Lam) memcpy(Lam, c->lam.data(), sizeof(double) * R);
  c->have_rec = true;
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

int scg_pr_signal(scg_pr_ctx *c, double *chi) {
  if (!c || c->failed || !c->have_rec) return SCG_ESTATE;
  const double s = std::sqrt(c->alpha * c->lam[0]);
  k_pr_scalecol<<<grid_for(c->n, 256), 256, 0, c->st>>>(c->tmpA, s, c->n, c->a);
  PR_CUDA(cudaMemcpyAsync(chi, c->a, sizeof(double2) * c->n, cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

int scg_pr_apply_D(scg_pr_ctx *c, const double *w, const double *x, double *yout) {
  if (!c || c->failed) return SCG_ESTATE;
  const int64_t n = c->n, dn = n * c->L;
  PR_CUDA(cudaStreamSynchronize(c->st));
  // save the iteration's weights, install kappa w (p-order), run the product, restore
  double *saved = c->h;
  PR_CUDA(cudaMemcpyAsync(saved, c->wk, sizeof(double) * dn, cudaMemcpyDeviceToDevice, c->st));
  double *tmp = reinterpret_cast<double *>(c->Y);
  PR_CUDA(cudaMemcpyAsync(tmp, w, sizeof(double) * dn, cudaMemcpyHostToDevice, c->st));
  k_pr_perm<<<grid_for(dn, 256), 256, 0, c->st>>>(tmp, c->wk, c->n1, c->n2, c->L, c->kappa, 1.0, 1);
  // x in a scratch buffer (tmpB: n complex at least; the reconstruction's U stays in tmpA), not in v
  PR_CUDA(cudaMemcpyAsync(c->tmpB, x, sizeof(double2) * n, cudaMemcpyHostToDevice, c->st));
  int rc = launch_matvec(c, c->tmpB, nullptr, c->a, 0, 2);
  if (rc) return rc;
  PR_CUDA(cudaMemcpyAsync(yout, c->a, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaMemcpyAsync(c->wk, saved, sizeof(double) * dn, cudaMemcpyDeviceToDevice, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

int scg_pr_measure(scg_pr_ctx *c, const double *x, double *hout) {
  if (!c || c->failed) return SCG_ESTATE;
  const int64_t n = c->n, dn = n * c->L;
  PR_CUDA(cudaStreamSynchronize(c->st));
  double2 *xd = c->a;
  PR_CUDA(cudaMemcpyAsync(xd, x, sizeof(double2) * n, cudaMemcpyHostToDevice, c->st));
  c->kf1<<<c->gf1, c->nthr1, c->smem1, c->st>>>(xd, nullptr, 0, c->sc, c->codes, c->book, c->Y, c->P2, c->tw2,
                                                   c->n1, c->n2, c->tm1, c->L);
  c->kb<<<c->gb, c->nthr2, c->smem2, c->st>>>(c->Y, c->wk, c->h, 2, 0, c->sc, c->P1, c->tw1, c->twlo, c->twhi,
                                                 c->n1, c->n2, c->tm2, c->L);
  double *tmp = reinterpret_cast<double *>(c->Y);
  k_pr_perm<<<grid_for(dn, 256), 256, 0, c->st>>>(c->h, tmp, c->n1, c->n2, c->L, c->kappa, 1.0, 0);
  PR_CUDA(cudaGetLastError());
  PR_CUDA(cudaMemcpyAsync(hout, tmp, sizeof(double) * dn, cudaMemcpyDeviceToHost, c->st));
  PR_CUDA(cudaStreamSynchronize(c->st));
  return SCG_OK;
}

int scg_pr_kernel_stats(scg_pr_ctx *c, scg_pr_kstat *out, int32_t cap, int32_t *count) {
  if (!c) return SCG_ESTATE;
  int m = 0;
  for (int k = 0; k < KS_COUNT && m < cap; ++k) {
    strncpy(out[m].name, kKsNames[k], 31);
    out[m].name[31] = 0;
    out[m].launches = c->ks_launch[k];
    out[m].total_ms = c->ks_ms[k];
    out[m].bytes_per_launch = c->ks_bytes[k];
    ++m;
  }
  if (count) *count = m;
  return SCG_OK;
}

int scg_pr_reset_stats(scg_pr_ctx *c) {
  if (!c) return SCG_ESTATE;
  for (int k = 0; k < KS_COUNT; ++k) {
    c->ks_launch[k] = 0;
    c->ks_ms[k] = 0.0;
  }
  return SCG_OK;
}

void *scg_pr_stream(scg_pr_ctx *c) { return c ? (void *)c->st : nullptr; }

int scg_pr_destroy(scg_pr_ctx *c) {
  if (!c) return SCG_OK;
  if (c->st) cudaStreamSynchronize(c->st);
  void *ptrs[] = {c->codes, c->book, c->tw1, c->tw2, c->twlo, c->twhi, c->kappa, c->bt, c->z, c->y, c->wk, c->h,
                  c->Y, c->a, c->v, c->Om, c->S, c->U, c->tmpA, c->tmpB, c->partials, c->sc, c->log, c->G,
                  c->Mx, c->gticket};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (c->flags & SCG_PR_PROFILE)
    for (int i = 0; i < 2 * 4096; ++i)
      if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->st) cudaStreamDestroy(c->st);
  c->h_kappa.~vector();
  c->lam.~vector();
  c->Uhost.~vector();
  ::operator delete(c);
  return SCG_OK;
}

}  // extern "C"
