// pde.cu — Experiment 2 of the paper: the uniform 1-D
// ODE  -(a(x,y) u')' = g,  a(x,y) = 2 + Σ_j y_j j^{-3/2} sin(2π j x)
// (PAPER.md:839-882).  The stiffness matrices B(y_n) = A_0 + Σ_j y_{n,j} A_j
// are tridiagonal; their perturbations Σ_j y_{n,j} A_j for
// all N QMC points are X = Y·A computed by the fast path (qmc_matmul, row n of
// the row-major X = sample n's K diagonal then K-1 off-diagonal entries).
// This file solves the N tridiagonal systems B(y_n) û^(n) = ĝ in place in X
// (Thomas algorithm, one thread per sample) and averages the coefficients,
// ū = (1/N) Σ_n û^(n).
#include <cuda_runtime.h>
#include <stdint.h>

#include "qmc_internal.cuh"

namespace qmc {

// Forward sweep (c'_k over the off-diagonal slot k, g'_k over the diagonal
// slot k), then back substitution (û_k over the diagonal slot k).  B is
// symmetric: sub- and super-diagonal entry k are both e0 + X[n, K + k].
__global__ void k_thomas(int64_t N, int64_t K, double d0, double e0, const double* __restrict__ rhs,
                         double* __restrict__ X, int64_t ldx) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double* d = X + n * ldx;   // diagonal slots 0..K-1
  double* e = d + K;         // off-diagonal slots 0..K-2
  double cprev = 0.0, gprev = 0.0, eprev = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    const double g = rhs ? __ldg(&rhs[k]) : 1.0;
    const double den = (d0 + d[k]) - eprev * cprev;
    const double inv = 1.0 / den;
    const double gk = (g - eprev * gprev) * inv;
    double ck = 0.0;
    if (k + 1 < K) {
      const double ek = e0 + e[k];
      ck = ek * inv;
      e[k] = ck;
      eprev = ek;
    }
    d[k] = gk;
    cprev = ck;
    gprev = gk;
  }
  double u = d[K - 1];
  for (int64_t k = K - 2; k >= 0; --k) {
    u = d[k] - e[k] * u;
    d[k] = u;
  }
}

// ū_k = (1/N) Σ_n û_k^(n), n in increasing order (deterministic), thread per k
__global__ void k_col_mean(int64_t N, int64_t K, const double* __restrict__ X, int64_t ldx,
                           double* __restrict__ out) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double s = 0.0;
  for (int64_t n = 0; n < N; ++n) s += X[n * ldx + k];
  out[k] = s / double(N);
}

}  // namespace qmc

using namespace qmc;

extern "C" int qmc_tridiag_solve_mean(int64_t N, int64_t K, double d0, double e0, const double* rhs, double* X,
                                      int64_t ldx, double* mean_out, void* stream) {
  if (!X || !mean_out) return QMC_ENULL;
  if (N < 1 || K < 1 || ldx < 2 * K - 1) return QMC_EINVAL_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  k_thomas<<<unsigned((N + 127) / 128), 128, 0, st>>>(N, K, d0, e0, rhs, X, ldx);
  QMC_LAUNCHED();
  k_col_mean<<<unsigned((K + 255) / 256), 256, 0, st>>>(N, K, X, ldx, mean_out);
  QMC_LAUNCHED();
  return QMC_OK;
}
