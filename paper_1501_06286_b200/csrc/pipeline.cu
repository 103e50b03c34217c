// pipeline.cu — the hot path of libqmc: X = Y·A by the fast QMC matrix
// method, fused with the row-0 term, the un-permutation
// to conventional order and the optional QMC-mean epilogue.
//
// Per column pair (k1, k2) packed as a = A[:,k1] + i·A[:,k2] (ζ is real, so
// one complex correlation serves two real columns), with the plan's split
// L = L1·L2 (e = L2·e1 + e2, f = f1 + L1·f2):
//
//   K0 k_pack      a in bucket order (e2-major) + column sums Σ_j a_j
//   K1 k_rows      T[f1,e2] = Σ_{j: e_j ≡ e2} a_j ω_L^{e_j f1}   (scatter a' = P a
//                  fused with the first FFT dimension)
//                  → FFT_L2 → ·W → IFFT_L2 → ·ω_L^{-e2 f1}            (smem)
//   K2 k_cols      IFFT_L1 over f1 → B'[e] in natural order           (skipped if L1 = 1)
//   K3 k_gather_*  X[0,k] = φ(0) Σ_j A[j,k],
//                  X[n,k] = B'_k[R[n]], R[n] = (m - L[n]) mod m, n >= 1,
//                  + optional f / row sums / per-column partial means
//   K4 k_colmean_reduce   fixed-order reduction of the partial means
//
// B'[i] = Σ_j a_j ζ[(e_j - i) mod m] = (Z P a)_i is a cyclic correlation,
// computed as IDFT(DFT(a') · DFT(K)), K[d] = ζ[(-d) mod m] (zero-padded to
// L >= 2m-1 when m does not split into supported radices).  Scratch for a
// batch of column pairs is sized (plan->batch_pairs) to stay in L2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "fft.cuh"
#include "qmc_internal.cuh"

namespace qmc {

constexpr int kPackThreads = 256;
constexpr int kGatherThreads = 256;
constexpr int kColMeanRows = 2048;  // rows per CTA in the column-mean epilogue

enum GatherMode { GM_X = 0, GM_ROWSUM = 1 };

// deterministic block sum (fixed shuffle tree, then warp 0 over warps)
template <int NT>
__device__ __forceinline__ double2 block_sum2(double2 v, double2* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < NT / 32 ? red[l] : make_double2(0.0, 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_down_sync(0xffffffffu, v.x, o);
      v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
  }
  return v;  // valid in thread 0
}

// ---------------------------------------------------------------- K0
__global__ void __launch_bounds__(kPackThreads)
    k_pack(const double* __restrict__ A, int64_t lda, int64_t t, int64_t pair0, int64_t s,
           const int32_t* __restrict__ bidx, double2* __restrict__ Ab, double* __restrict__ colsum) {
  __shared__ double2 red[kPackThreads / 32];
  const int64_t p = blockIdx.x;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const bool has2 = k2 < t;
  const double* a1 = A + k1 * lda;
  const double* a2 = A + (has2 ? k2 : k1) * lda;
  double2* out = Ab + p * s;
  double2 cs = make_double2(0.0, 0.0);
  for (int64_t i = threadIdx.x; i < s; i += kPackThreads) {
    const int j = bidx[i];
    out[i] = make_double2(__ldg(a1 + j), has2 ? __ldg(a2 + j) : 0.0);
    cs.x += __ldg(a1 + i);
    if (has2) cs.y += __ldg(a2 + i);
  }
  cs = block_sum2<kPackThreads>(cs, red);
  if (threadIdx.x == 0) {
    colsum[k1] = cs.x;
    if (has2) colsum[k2] = cs.y;
  }
}

// ---------------------------------------------------------------- K1
template <int L2>
__global__ void __launch_bounds__(RowThreads<L2>::value, 1)
    k_rows(const double2* __restrict__ Ab, int64_t s, const int32_t* __restrict__ bstart,
           const int32_t* __restrict__ be1, const double2* __restrict__ tw1,
           const double2* __restrict__ twL, const double2* __restrict__ tw2,
           const double2* __restrict__ W, double2* __restrict__ U, int64_t L, int L1) {
  extern __shared__ double2 smem[];
  constexpr int NT = RowThreads<L2>::value;
  constexpr int EPT = L2 / NT;
  double2* S = smem;
  double2* rowtw = smem + L2;  // ω_{L1}^{e1·f1}, e1 < L1
  const int f1 = blockIdx.x;
  const int64_t p = blockIdx.y;
  for (int e1 = threadIdx.x; e1 < L1; e1 += NT) rowtw[e1] = __ldg(&tw1[(e1 * f1) % L1]);
  __syncthreads();
  const double2* ab = Ab + p * s;
#pragma unroll 1
  for (int i = 0; i < EPT; ++i) {
    const int e2 = threadIdx.x + i * NT;
    const int b0 = __ldg(&bstart[e2]), b1 = __ldg(&bstart[e2 + 1]);
    double2 acc = make_double2(0.0, 0.0);
    for (int b = b0; b < b1; ++b) {
      const double2 a = __ldg(&ab[b]);
      const double2 w = rowtw[__ldg(&be1[b])];
      acc = cadd(acc, cmul(a, w));
    }
    const int x = e2 * f1;  // < L, ω_L^x = ω_{L1}^{x/L2} · ω_L^{x mod L2}
    const double2 w = cmul(__ldg(&tw1[x / L2]), __ldg(&twL[x % L2]));
    S[swz(e2)] = cmul(acc, w);
  }
  __syncthreads();
  row_fft<L2, -1>(S, tw2);
  const double2* Wr = W + int64_t(f1) * L2;
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int f2 = threadIdx.x + i * NT;
    S[swz(f2)] = cmul(S[swz(f2)], __ldg(&Wr[f2]));
  }
  __syncthreads();
  row_fft<L2, +1>(S, tw2);
  double2* Ur = U + p * L + int64_t(f1) * L2;
#pragma unroll 2
  for (int i = 0; i < EPT; ++i) {
    const int e2 = threadIdx.x + i * NT;
    const int x = e2 * f1;
    const double2 w = cmul(__ldg(&tw1[x / L2]), __ldg(&twL[x % L2]));
    Ur[e2] = cmulc(S[swz(e2)], w);
  }
}

// ---------------------------------------------------------------- K2
// One inverse Stockham stage of radix R over CB interleaved columns
// (element (i, c) at buf[i·CB + c]); ping-pong in -> out.
template <int R>
__device__ __forceinline__ void col_stage(const double2* in, double2* out, int L1, int CB, int Ns,
                                          const double2* __restrict__ tw1) {
  const int NB = L1 / R, nbf = NB * CB, step = L1 / (Ns * R);
  for (int q = threadIdx.x; q < nbf; q += blockDim.x) {
    const int j = q / CB, c = q - j * CB;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[(j + r * NB) * CB + c];
    const int k = j % Ns;
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twid<+1>(__ldg(&tw1[k * r * step])));
    }
    Dft<R, +1>::run(v);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) out[(base + r * Ns) * CB + c] = v[r];
  }
}

// In-place inverse DFT of length L1 along f1 for CB adjacent columns e2 of
// U[p] (layout [f1][e2]); result y[e1][e2] = B'[L2·e1 + e2].
__global__ void __launch_bounds__(256)
    k_cols(double2* __restrict__ U, int64_t L, int L1, int L2, int CB,
           const int32_t* __restrict__ rad, int nrad, const double2* __restrict__ tw1) {
  extern __shared__ double2 smem[];
  double2* in = smem;
  double2* out = smem + L1 * CB;
  const int64_t p = blockIdx.y;
  const int c0 = blockIdx.x * CB;
  double2* Up = U + p * L + c0;
  const int tot = L1 * CB;
  for (int q = threadIdx.x; q < tot; q += blockDim.x) {
    const int f1 = q / CB, c = q - f1 * CB;
    in[q] = Up[int64_t(f1) * L2 + c];
  }
  __syncthreads();
  int Ns = 1;
  for (int st = 0; st < nrad; ++st) {
    const int R = __ldg(&rad[st]);
    switch (R) {
      case 2: col_stage<2>(in, out, L1, CB, Ns, tw1); break;
      case 3: col_stage<3>(in, out, L1, CB, Ns, tw1); break;
      case 4: col_stage<4>(in, out, L1, CB, Ns, tw1); break;
      case 5: col_stage<5>(in, out, L1, CB, Ns, tw1); break;
      default: col_stage<8>(in, out, L1, CB, Ns, tw1); break;
    }
    __syncthreads();
    double2* tmp = in;
    in = out;
    out = tmp;
    Ns *= R;
  }
  for (int q = threadIdx.x; q < tot; q += blockDim.x) {
    const int e1 = q / CB, c = q - e1 * CB;
    Up[int64_t(e1) * L2 + c] = in[q];
  }
}

// ---------------------------------------------------------------- K3
// One thread per conventional row n, looping over the pairs of the batch.
template <int MODE>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather(const double2* __restrict__ U, int64_t L, int npairs, int64_t pair0, int64_t t,
             const int32_t* __restrict__ R, const double* __restrict__ colsum,
             const double* __restrict__ scal, int64_t N, double* __restrict__ X, int64_t ldx,
             double* __restrict__ rowsum, int first) {
  const int64_t n = int64_t(blockIdx.x) * kGatherThreads + threadIdx.x;
  if (n >= N) return;
  const double phi0 = __ldg(scal);
  const int r = n > 0 ? __ldg(&R[n]) : 0;
  double rs = 0.0;
  for (int p = 0; p < npairs; ++p) {
    const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
    const bool has2 = k2 < t;
    double2 v;
    if (n == 0) v = make_double2(phi0 * colsum[k1], has2 ? phi0 * colsum[k2] : 0.0);
    else v = __ldg(&U[int64_t(p) * L + r]);
    if (X) {
      X[n + k1 * ldx] = v.x;
      if (has2) X[n + k2 * ldx] = v.y;
    }
    if (MODE == GM_ROWSUM) {
      rs += v.x;
      if (has2) rs += v.y;
    }
  }
  if (MODE == GM_ROWSUM) rowsum[n] = (first ? 0.0 : rowsum[n]) + rs;
}

// Per (row block, pair): writes X (c + X for AFFINE) and Σ_rows f(X) per
// column into partial[nb·t + k].
template <int F>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather_colmean(const double2* __restrict__ U, int64_t L, int64_t pair0, int64_t t,
                     const int32_t* __restrict__ R, const double* __restrict__ colsum,
                     const double* __restrict__ scal, int64_t N, double fparam,
                     double* __restrict__ X, int64_t ldx, double* __restrict__ partial) {
  __shared__ double2 red[kGatherThreads / 32];
  const int64_t nb = blockIdx.x;
  const int p = blockIdx.y;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const bool has2 = k2 < t;
  const double phi0 = __ldg(scal);
  const double2* Up = U + int64_t(p) * L;
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int i = 0; i < kColMeanRows / kGatherThreads; ++i) {
    const int64_t n = nb * kColMeanRows + i * kGatherThreads + threadIdx.x;
    if (n < N) {
      double2 v;
      if (n == 0) v = make_double2(phi0 * colsum[k1], has2 ? phi0 * colsum[k2] : 0.0);
      else v = __ldg(&Up[__ldg(&R[n])]);
      if (F == QMC_F_AFFINE) {
        v.x += fparam;
        v.y += fparam;
      }
      if (X) {
        X[n + k1 * ldx] = v.x;
        if (has2) X[n + k2 * ldx] = v.y;
      }
      if (F == QMC_F_EXP) {
        acc.x += exp(v.x);
        acc.y += exp(v.y);
      } else {
        acc.x += v.x;
        acc.y += v.y;
      }
    }
  }
  acc = block_sum2<kGatherThreads>(acc, red);
  if (threadIdx.x == 0) {
    partial[nb * t + k1] = acc.x;
    if (has2) partial[nb * t + k2] = acc.y;
  }
}

// ---------------------------------------------------------------- K4 / finalize
__global__ void k_colmean_reduce(const double* __restrict__ partial, int64_t nblocks, int64_t t,
                                 int64_t N, double* __restrict__ out) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= t) return;
  double s = 0.0;
  for (int64_t b = 0; b < nblocks; ++b) s += partial[b * t + k];
  out[k] = s / double(N);
}

__global__ void __launch_bounds__(1024)
    k_rowmean_relu_finalize(const double* reduced, int64_t N, int64_t t_total, double* out) {
  __shared__ double2 red[32];
  const double inv_t = 1.0 / double(t_total);
  double s = 0.0;
  for (int64_t n = threadIdx.x; n < N; n += 1024) s += fmax(0.0, reduced[n] * inv_t);
  double2 v = block_sum2<1024>(make_double2(s, 0.0), red);
  __syncthreads();  // every read of `reduced` precedes the write below (out may alias)
  if (threadIdx.x == 0) out[0] = v.x / double(N);
}

__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && a != b) b[i] = a[i];
}

// ---------------------------------------------------------------- host side
struct CallLayout {
  size_t off_Ab, off_U, off_colsum, off_partial, total;
};

static CallLayout call_layout(const qmc_plan* pl, int64_t t, int f) {
  CallLayout c;
  const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(pl->batch_pairs, (t + 1) / 2));
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o = align_up(o + b);
    return r;
  };
  c.off_Ab = take(size_t(pairs) * pl->s * 16);
  c.off_U = take(size_t(pairs) * pl->sp.L * 16);
  c.off_colsum = take(size_t(std::max<int64_t>(t, 1)) * 8);
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  const int64_t nblocks = (pl->N + kColMeanRows - 1) / kColMeanRows;
  c.off_partial = take(colmean ? size_t(nblocks) * std::max<int64_t>(t, 1) * 8 : 0);
  c.total = o;
  return c;
}

template <int L2>
static int launch_rows(const qmc_plan* pl, const double2* Ab, double2* U, int npairs, cudaStream_t st) {
  const size_t smem = size_t(L2 + pl->sp.L1) * sizeof(double2);
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    cudaFuncSetAttribute(k_rows<L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_done = true;
  }
  dim3 grid((unsigned)pl->sp.L1, (unsigned)npairs);
  k_rows<L2><<<grid, RowThreads<L2>::value, smem, st>>>(Ab, pl->s, pl->d_bstart, pl->d_be1, pl->d_tw1,
                                                        pl->d_twL, pl->d_tw2, pl->d_W, U, pl->sp.L,
                                                        int(pl->sp.L1));
  QMC_LAUNCHED();
  return QMC_OK;
}

static int rows_dispatch(const qmc_plan* pl, const double2* Ab, double2* U, int npairs, cudaStream_t st) {
  switch (pl->sp.L2) {
    case 16: return launch_rows<16>(pl, Ab, U, npairs, st);
    case 32: return launch_rows<32>(pl, Ab, U, npairs, st);
    case 64: return launch_rows<64>(pl, Ab, U, npairs, st);
    case 128: return launch_rows<128>(pl, Ab, U, npairs, st);
    case 256: return launch_rows<256>(pl, Ab, U, npairs, st);
    case 512: return launch_rows<512>(pl, Ab, U, npairs, st);
    case 1024: return launch_rows<1024>(pl, Ab, U, npairs, st);
    case 2048: return launch_rows<2048>(pl, Ab, U, npairs, st);
    case 4096: return launch_rows<4096>(pl, Ab, U, npairs, st);
    case 8192: return launch_rows<8192>(pl, Ab, U, npairs, st);
  }
  return QMC_EINVAL_N;
}

static unsigned nblk(int64_t n, int b) { return unsigned((n + b - 1) / b); }

// core: all batches; mode: -1 = X only, else f
static int run(const qmc_plan* pl, const double* A, int64_t lda, int64_t t, int f, double fparam,
               double* out, double* X, int64_t ldx, void* call_ws, size_t call_ws_bytes, cudaStream_t st) {
  if (!pl) return QMC_ENULL;
  if (t < 0 || lda < pl->s) return QMC_EINVAL_DIM;
  if (X && ldx < pl->N) return QMC_EINVAL_DIM;
  if (t == 0) return QMC_OK;
  if (!A || !call_ws) return QMC_ENULL;
  if (f >= 0 && !out) return QMC_ENULL;
  if (f < 0 && !X) return QMC_ENULL;
  const CallLayout cl = call_layout(pl, t, f);
  if (call_ws_bytes < cl.total || (uintptr_t(call_ws) % kAlign)) return QMC_EWORKSPACE;
  char* ws = (char*)call_ws;
  double2* Ab = (double2*)(ws + cl.off_Ab);
  double2* U = (double2*)(ws + cl.off_U);
  double* colsum = (double*)(ws + cl.off_colsum);
  double* partial = (double*)(ws + cl.off_partial);
  const int64_t npairs_total = (t + 1) / 2;
  const int64_t nb3 = (pl->N + kColMeanRows - 1) / kColMeanRows;
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  static bool cols_attr = false;
  if (!cols_attr) {
    cudaFuncSetAttribute(k_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cols_attr = true;
  }
  for (int64_t pair0 = 0; pair0 < npairs_total; pair0 += pl->batch_pairs) {
    const int np = int(std::min<int64_t>(pl->batch_pairs, npairs_total - pair0));
    prof_begin(KC_PACK, st);
    k_pack<<<np, kPackThreads, 0, st>>>(A, lda, t, pair0, pl->s, pl->d_bidx, Ab, colsum);
    QMC_LAUNCHED();
    prof_end(KC_PACK, st);
    prof_begin(KC_ROWS, st);
    int rc = rows_dispatch(pl, Ab, U, np, st);
    if (rc) return rc;
    prof_end(KC_ROWS, st);
    if (pl->sp.L1 > 1) {
      dim3 g((unsigned)(pl->sp.L2 / pl->col_cb), (unsigned)np);
      const size_t smem = size_t(2) * pl->sp.L1 * pl->col_cb * sizeof(double2);
      prof_begin(KC_COLS, st);
      k_cols<<<g, 256, smem, st>>>(U, pl->sp.L, int(pl->sp.L1), int(pl->sp.L2), pl->col_cb, pl->d_rad1,
                                   pl->nrad1, pl->d_tw1);
      QMC_LAUNCHED();
      prof_end(KC_COLS, st);
    }
    prof_begin(KC_GATHER, st);
    if (colmean) {
      dim3 g((unsigned)nb3, (unsigned)np);
      switch (f) {
        case QMC_F_IDENTITY:
          k_gather_colmean<QMC_F_IDENTITY><<<g, kGatherThreads, 0, st>>>(U, pl->sp.L, pair0, t, pl->d_R, colsum,
                                                                        pl->d_scal, pl->N, fparam, X, ldx, partial);
          break;
        case QMC_F_AFFINE:
          k_gather_colmean<QMC_F_AFFINE><<<g, kGatherThreads, 0, st>>>(U, pl->sp.L, pair0, t, pl->d_R, colsum,
                                                                      pl->d_scal, pl->N, fparam, X, ldx, partial);
          break;
        default:
          k_gather_colmean<QMC_F_EXP><<<g, kGatherThreads, 0, st>>>(U, pl->sp.L, pair0, t, pl->d_R, colsum,
                                                                   pl->d_scal, pl->N, fparam, X, ldx, partial);
      }
      QMC_LAUNCHED();
    } else if (f == QMC_F_ROWMEAN_RELU) {
      k_gather<GM_ROWSUM><<<nblk(pl->N, kGatherThreads), kGatherThreads, 0, st>>>(
          U, pl->sp.L, np, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, X, ldx, out, pair0 == 0);
      QMC_LAUNCHED();
    } else {
      k_gather<GM_X><<<nblk(pl->N, kGatherThreads), kGatherThreads, 0, st>>>(
          U, pl->sp.L, np, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, X, ldx, nullptr, 0);
      QMC_LAUNCHED();
    }
    prof_end(KC_GATHER, st);
  }
  if (colmean) {
    prof_begin(KC_REDUCE, st);
    k_colmean_reduce<<<nblk(t, 256), 256, 0, st>>>(partial, nb3, t, pl->N, out);
    QMC_LAUNCHED();
    prof_end(KC_REDUCE, st);
  }
  return QMC_OK;
}

}  // namespace qmc

using namespace qmc;

extern "C" {

int qmc_call_workspace_size(qmc_plan_t pl, int64_t t, int f, size_t* call_bytes) {
  if (!pl || !call_bytes) return QMC_ENULL;
  if (t < 0) return QMC_EINVAL_DIM;
  if (f < -1 || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  *call_bytes = call_layout(pl, t, f).total;
  return QMC_OK;
}

int qmc_matmul(qmc_plan_t pl, const double* A, int64_t lda, int64_t t, double* X, int64_t ldx,
               void* call_ws, size_t call_ws_bytes, void* stream) {
  return run(pl, A, lda, t, -1, 0.0, nullptr, X, ldx, call_ws, call_ws_bytes, (cudaStream_t)stream);
}

int qmc_mean(qmc_plan_t pl, const double* A, int64_t lda, int64_t t, int f, double f_param,
             double* out, double* X_or_null, int64_t ldx, void* call_ws, size_t call_ws_bytes,
             void* stream) {
  if (f < QMC_F_IDENTITY || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  return run(pl, A, lda, t, f, f_param, out, X_or_null, ldx, call_ws, call_ws_bytes, (cudaStream_t)stream);
}

int qmc_mean_finalize(qmc_plan_t pl, int f, const double* reduced, int64_t t_total, double* out,
                      void* stream) {
  if (!pl || !reduced || !out) return QMC_ENULL;
  if (f < QMC_F_IDENTITY || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  if (t_total < 1) return QMC_EINVAL_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  prof_begin(KC_FINALIZE, st);
  if (f == QMC_F_ROWMEAN_RELU) {
    k_rowmean_relu_finalize<<<1, 1024, 0, st>>>(reduced, pl->N, t_total, out);
  } else {
    k_copy<<<nblk(t_total, 256), 256, 0, st>>>(reduced, out, t_total);
  }
  QMC_LAUNCHED();
  prof_end(KC_FINALIZE, st);
  return QMC_OK;
}

int qmc_mean_host(qmc_plan_t pl, const double* A_host, int64_t lda, int64_t t, int f, double f_param,
                  double* out_host, double* A_dev, double* X_dev, int64_t ldx, double* out_dev,
                  void* call_ws, size_t call_ws_bytes, void* stream) {
  if (!pl || !A_host || !out_host || !A_dev || !out_dev) return QMC_ENULL;
  if (f < QMC_F_IDENTITY || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  if (t < 1 || lda < pl->s) return QMC_EINVAL_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpy2DAsync(A_dev, size_t(pl->s) * 8, A_host, size_t(lda) * 8, size_t(pl->s) * 8, size_t(t),
                        cudaMemcpyHostToDevice, st) != cudaSuccess)
    return QMC_ECUDA;
  int rc = run(pl, A_dev, pl->s, t, f, f_param, out_dev, X_dev, ldx, call_ws, call_ws_bytes, st);
  if (rc) return rc;
  rc = qmc_mean_finalize(pl, f, out_dev, t, out_dev, stream);
  if (rc) return rc;
  const size_t nout = f == QMC_F_ROWMEAN_RELU ? 1 : size_t(t);
  if (cudaMemcpyAsync(out_host, out_dev, nout * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) return QMC_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return QMC_ECUDA;
  return QMC_OK;
}

}  // extern "C"
