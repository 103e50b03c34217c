// pde.cu — Experiment 2 of the paper: the uniform 1-D
// ODE  -(a(x,y) u')' = g,  a(x,y) = 2 + Σ_j y_j j^{-3/2} sin(2π j x)
// (PAPER.md:839-882).  The stiffness matrices B(y_n) = A_0 + Σ_j y_{n,j} A_j
// are tridiagonal; their perturbations Σ_j y_{n,j} A_j for
// all N QMC points are X = Y·A computed by the fast path (qmc_matmul, row n of
// the row-major X = sample n's K diagonal then K-1 off-diagonal entries).
// This file solves the N tridiagonal systems B(y_n) û^(n) = ĝ in place in X
// (Thomas algorithm, one thread per sample, rows streamed through shared
// memory) and averages the coefficients,
// ū = (1/N) Σ_n û^(n).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qmc_internal.cuh"

namespace qmc {

// Tiled Thomas: a CTA of one warp owns 32 samples (lane = sample).  The rows
// of X are streamed through shared memory in tiles of kTT unknowns by
// cp.async (coalesced: 32 rows × kTT consecutive doubles, double buffered);
// each lane runs the recurrence of its own sample over the tile from shared
// memory and the updated tile is written back coalesced.  Forward sweep over
// tiles in increasing k, back substitution in decreasing k.
constexpr int kTT = 32;              // unknowns per tile (one per lane)
constexpr int kTP = kTT + 1;         // padded pitch (doubles): lane rows in distinct banks

__device__ __forceinline__ void cpa8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

// stage tile [k0, k0+kTT) of the diagonal and off-diagonal slots of the
// warp's 32 rows (rows >= N and k >= K are skipped)
__device__ __forceinline__ void thomas_stage(const double* X, int64_t ldx, int64_t N, int64_t K, int64_t n0, int64_t k0,
                                             double* sd, double* se) {
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) {
    const int64_t n = n0 + r;
    if (n >= N) break;
    const double* row = X + n * ldx;
    for (int c = lane; c < kTT; c += 32) {
      const int64_t k = k0 + c;
      if (k < K) cpa8(&sd[r * kTP + c], row + k);
      if (k + 1 < K) cpa8(&se[r * kTP + c], row + K + k);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void thomas_store(double* X, int64_t ldx, int64_t N, int64_t K, int64_t n0, int64_t k0,
                                             const double* sd, const double* se, bool off) {
  const int lane = threadIdx.x;
  for (int r = 0; r < 32; ++r) {
    const int64_t n = n0 + r;
    if (n >= N) break;
    double* row = X + n * ldx;
    for (int c = lane; c < kTT; c += 32) {
      const int64_t k = k0 + c;
      if (k < K) row[k] = sd[r * kTP + c];
      if (off && k + 1 < K) row[K + k] = se[r * kTP + c];
    }
  }
}

__global__ void __launch_bounds__(32) k_thomas_tiled(int64_t N, int64_t K, double d0, double e0,
                                                      const double* __restrict__ rhs, double* __restrict__ X,
                                                      int64_t ldx) {
  __shared__ double sd[2][32 * kTP], se[2][32 * kTP];
  const int lane = threadIdx.x;
  const int64_t n0 = int64_t(blockIdx.x) * 32;
  const int64_t ntile = (K + kTT - 1) / kTT;
  // forward sweep: slots become g'_k (diagonal) and c'_k (off-diagonal)
  double cprev = 0.0, gprev = 0.0, eprev = 0.0;
  thomas_stage(X, ldx, N, K, n0, 0, sd[0], se[0]);
  for (int64_t tI = 0; tI < ntile; ++tI) {
    const int b = int(tI & 1);
    if (tI + 1 < ntile) {
      thomas_stage(X, ldx, N, K, n0, (tI + 1) * kTT, sd[b ^ 1], se[b ^ 1]);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int64_t k0 = tI * kTT;
    double* d = &sd[b][lane * kTP];
    double* e = &se[b][lane * kTP];
    const int cnt = int(K - k0 < kTT ? K - k0 : kTT);
    for (int c = 0; c < cnt; ++c) {
      const int64_t k = k0 + c;
      const double g = rhs ? __ldg(&rhs[k]) : 1.0;
      const double inv = 1.0 / ((d0 + d[c]) - eprev * cprev);
      const double gk = (g - eprev * gprev) * inv;
      double ck = 0.0;
      if (k + 1 < K) {
        const double ek = e0 + e[c];
        ck = ek * inv;
        e[c] = ck;
        eprev = ek;
      }
      d[c] = gk;
      cprev = ck;
      gprev = gk;
    }
    __syncwarp();
    thomas_store(X, ldx, N, K, n0, k0, sd[b], se[b], true);
    __syncwarp();
  }
  // back substitution, tiles in decreasing k: u_k = g'_k - c'_k u_{k+1}
  double u = 0.0;
  thomas_stage(X, ldx, N, K, n0, (ntile - 1) * kTT, sd[0], se[0]);
  for (int64_t tI = ntile - 1, it = 0; tI >= 0; --tI, ++it) {
    const int b = int(it & 1);
    if (tI > 0) {
      thomas_stage(X, ldx, N, K, n0, (tI - 1) * kTT, sd[b ^ 1], se[b ^ 1]);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int64_t k0 = tI * kTT;
    double* d = &sd[b][lane * kTP];
    const double* e = &se[b][lane * kTP];
    const int cnt = int(K - k0 < kTT ? K - k0 : kTT);
    for (int c = cnt - 1; c >= 0; --c) {
      const int64_t k = k0 + c;
      u = (k + 1 < K) ? d[c] - e[c] * u : d[c];
      d[c] = u;
    }
    __syncwarp();
    thomas_store(X, ldx, N, K, n0, k0, sd[b], se[b], false);
    __syncwarp();
  }
}

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
  if (getenv("QMC_THOMAS_SIMPLE")) {
    k_thomas<<<unsigned((N + 127) / 128), 128, 0, st>>>(N, K, d0, e0, rhs, X, ldx);
  } else {
    k_thomas_tiled<<<unsigned((N + 31) / 32), 32, 0, st>>>(N, K, d0, e0, rhs, X, ldx);
  }
  QMC_LAUNCHED();
  k_col_mean<<<unsigned((K + 255) / 256), 256, 0, st>>>(N, K, X, ldx, mean_out);
  QMC_LAUNCHED();
  return QMC_OK;
}
