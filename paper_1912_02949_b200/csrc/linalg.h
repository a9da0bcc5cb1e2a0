// linalg.h -- small dense fp64 R x R linear algebra on the host for the one-shot
// Nystrom reconstruction (Alg. 3 lines 12-16): Cholesky,
// triangular inverse, cyclic Jacobi eigenvalues and one-sided Jacobi SVD.
// Negligible in size (R <= 64); off the iteration feedback path.
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

namespace scg_host {

inline bool chol_upper(const std::vector<double> &B, int R, std::vector<double> &Rc) {  // B = Rc^T Rc
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

inline std::vector<double> inv_upper(const std::vector<double> &U, int R) {
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

inline std::vector<double> matmul(const std::vector<double> &A, const std::vector<double> &B, int R) {
  std::vector<double> C((size_t)R * R, 0.0);
  for (int i = 0; i < R; ++i)
    for (int k = 0; k < R; ++k)
      for (int j = 0; j < R; ++j) C[(size_t)i * R + j] += A[(size_t)i * R + k] * B[(size_t)k * R + j];
  return C;
}

// cyclic Jacobi eigenvalues of a symmetric matrix (values only)
inline std::vector<double> sym_eigvals(std::vector<double> A, int R) {
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
inline void svd_jacobi(std::vector<double> F, int R, std::vector<double> &U, std::vector<double> &sv) {
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

inline double matlab_eps(double x) {
  if (x == 0.0) return std::ldexp(1.0, -1074);
  int e;
  std::frexp(std::fabs(x), &e);  // x = m 2^e, m in [0.5, 1)
  return std::ldexp(1.0, e - 1 - 52);
}


}  // namespace scg_host
