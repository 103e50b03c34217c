// cbc.cu — component-by-component (CBC) construction of a rank-1 lattice
// generating vector (the paper cites the fast CBC of
// Nuyens–Cools without restating it).  The
// criterion is the shift-averaged worst-case error in the weighted Korobov
// space with product weights γ_j and smoothness 1:
//   e²(z_1..z_d) = -1 + (1/N) Σ_n Π_{j<=d} (1 + γ_j 2π² B_2({n z_j / N})),
// B_2(u) = u² - u + 1/6.  Step d keeps p_n = Π_{j<d}(1 + γ_j 2π² B_2(·)) and
// picks z_d minimising Σ_n B_2({n z/N}) p_n over the candidates — a product of
// the point matrix of the "all generators" lattice (rows z, columns n) with
// p, i.e. exactly the fast Y·A of this library (one plan with generating
// vector (1, ..., N-1) and φ = B_2; qmc_matmul with A = p_1..p_{N-1}).  This
// file holds the selection and the update of p.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "qmc_internal.cuh"

namespace qmc {

constexpr int kCbcThreads = 1024;

__global__ void __launch_bounds__(kCbcThreads)
    k_cbc_step(int64_t N, const double* __restrict__ crit, int64_t zmax, double gamma, double* __restrict__ p,
               int64_t* __restrict__ zout, int64_t d) {
  __shared__ double bv[kCbcThreads];
  __shared__ int64_t bz[kCbcThreads];
  const int tid = threadIdx.x;
  // argmin over z in [1, zmax]: smallest value, then smallest z (deterministic)
  double v = INFINITY;
  int64_t zb = zmax + 1;
  for (int64_t z = 1 + tid; z <= zmax; z += kCbcThreads) {
    const double c = crit[z];
    if (c < v) {
      v = c;
      zb = z;
    }
  }
  bv[tid] = v;
  bz[tid] = zb;
  __syncthreads();
  for (int o = kCbcThreads / 2; o > 0; o >>= 1) {
    if (tid < o) {
      const double v2 = bv[tid + o];
      const int64_t z2 = bz[tid + o];
      if (v2 < bv[tid] || (v2 == bv[tid] && z2 < bz[tid])) {
        bv[tid] = v2;
        bz[tid] = z2;
      }
    }
    __syncthreads();
  }
  const int64_t zs = bz[0];
  if (tid == 0) zout[d] = zs;
  // p_n *= 1 + γ 2π² B_2({n z_d / N})
  const double g2 = gamma * 2.0 * M_PI * M_PI;
  for (int64_t n = tid; n < N; n += kCbcThreads) {
    const double u = double((n * zs) % N) / double(N);
    p[n] *= 1.0 + g2 * (u * u - u + 1.0 / 6.0);
  }
}

}  // namespace qmc

using namespace qmc;

extern "C" int qmc_cbc_step(int64_t N, const double* crit, int64_t zmax, double gamma, double* p, int64_t* z_out,
                            int64_t d, void* stream) {
  if (!crit || !p || !z_out) return QMC_ENULL;
  if (N < 3 || zmax < 1 || zmax >= N || d < 0) return QMC_EINVAL_DIM;
  k_cbc_step<<<1, kCbcThreads, 0, (cudaStream_t)stream>>>(N, crit, zmax, gamma, p, z_out, d);
  QMC_LAUNCHED();
  return QMC_OK;
}
