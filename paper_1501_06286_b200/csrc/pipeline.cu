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

#include <stdlib.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "fft.cuh"
#include "qmc_internal.cuh"
#include "rowcfg.cuh"

namespace qmc {

constexpr int kGatherThreads = 256;
constexpr int kColMeanRows = 1024;  // rows per CTA in the column-mean epilogue

enum GatherMode { GM_X = 0, GM_ROWSUM = 1 };

// column-block width of K1's output U (== K2's register-path CB)
constexpr int kUB = 4;

// cache policy of the epilogue: Y is dead after the gather and X is only
// written, so both use evict-first (streaming) accesses unless disabled
#ifndef QMC_NO_STREAMING
#define QMC_LD2(p, a, b) ldcs2_256(p, a, b)
#define QMC_LD1(p) ldcs(p)
#define QMC_ST(p, v) stcs(p, v)
#else
#define QMC_LD2(p, a, b) ldg2_256(p, a, b)
#define QMC_LD1(p) __ldg(p)
#define QMC_ST(p, v) (*(p) = (v))
#endif

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

// ---------------------------------------------------------------- K1
// One CTA per (row f1, pair p): L2/16 threads, 16 points per thread.
//   T[f1,e2] = Σ_{j in bucket(e2)} a_j ω_L^{e_j f1}     (a_j = A[j,k1] + i A[j,k2])
//   forward FFT_L2 → ·W[f1,:] → inverse FFT_L2 → U[p][f1][e2]
// The twiddle conj(ω_L^{e2 f1}) of the second FFT dimension is applied by K2.
// CTA f1 = 0 also writes the row-0 sums Σ_j a_j = DC term of the spectrum.
#ifdef QMC_PHASE_TIMING
__device__ long long g_phase[4096][8];
#define QMC_TS(i)                                                                                      \
  do {                                                                                               \
    __syncthreads();                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x + gridDim.x * blockIdx.y < 4096)                              \
      g_phase[blockIdx.x + gridDim.x * blockIdx.y][i] = clock64();                                   \
  } while (0)
extern "C" int qmc_debug_phases(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(long long) * 8 * n) == cudaSuccess ? 0 : -7;
}
#else
#define QMC_TS(i) \
  do {            \
  } while (0)
#endif
// L1C = 0: write U[p][f1][e2] (the column pass runs in K2).
// L1C = L1 > 0: the grid's x-dimension (f1) is one thread-block cluster of
// L1 CTAs; after the row transforms every CTA keeps its row in shared memory
// and computes, for its share of the columns e2, the twiddle
// conj(ω_L^{e2 f1}) and the inverse DFT over f1 from the L1 rows read
// through distributed shared memory, writing B'[p][L2·e1 + e2] (natural).
template <int L2, int L1C>
__global__ void __launch_bounds__(L2 / QMC_ROW_E, (L2 / QMC_ROW_E >= 512 ? 1 : QMC_ROWS_MINB))
    k_rows16(const double* __restrict__ A, int64_t lda, int64_t t, int64_t pair0,
             const int32_t* __restrict__ e, const int32_t* __restrict__ bnext, int64_t s,
             const double2* __restrict__ twj, const double2* __restrict__ tws,
             const double2* __restrict__ W, double2* __restrict__ U, int64_t L, double* __restrict__ colsum,
             const double2* __restrict__ twL, const double2* __restrict__ tw1) {
  extern __shared__ double2 smem[];
  constexpr int E = QMC_ROW_E;
  constexpr int NT = L2 / E;
  double2* S = smem;
  const int tid = threadIdx.x;
  const int f1 = blockIdx.x;
  const int64_t p = blockIdx.y;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const bool has2 = k2 < t;
  const double* a1 = A + k1 * lda;
  const double* a2 = A + (has2 ? k2 : k1) * lda;
  QMC_TS(0);
  // scatter a' = P a fused with the first DFT dimension:
  //   T[f1, e2] = Σ_{j: e_j ≡ e2 (mod L2)} a_j ω_L^{(e_j·f1) mod L}
  // Entries in natural j order (coalesced, independent loads, issued before
  // the shared row is cleared); the smallest j of each bucket sums the bucket
  // along its collision chain in increasing j -> deterministic.
  constexpr int UE = 4;
  const double2* twr = twj + int64_t(f1) * s;
  for (int j0 = 0; j0 < s; j0 += NT * UE) {
    int ej[UE], nx[UE];
    double2 a[UE], w[UE];
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      const int j = j0 + tid + u * NT;
      nx[u] = -2;
      if (j < s) {
        ej[u] = __ldg(&e[j]);
        nx[u] = __ldg(&bnext[j]);
        a[u] = make_double2(__ldg(a1 + j), has2 ? __ldg(a2 + j) : 0.0);
        w[u] = __ldg(&twr[j]);
      }
    }
    if (j0 == 0) {
#pragma unroll
      for (int q = 0; q < E; ++q) S[padE<E>(tid + q * NT)] = make_double2(0.0, 0.0);
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < UE; ++u) {
      if (nx[u] >= -1) {
        double2 acc = cmul(a[u], w[u]);
        for (int jj = nx[u]; jj >= 0;) {  // collisions (rare)
          acc = cadd(acc, cmul(make_double2(__ldg(a1 + jj), has2 ? __ldg(a2 + jj) : 0.0), __ldg(&twr[jj])));
          const int v = __ldg(&bnext[jj]);
          jj = v <= -3 ? -3 - v : -1;
        }
        S[padE<E>(ej[u] & (L2 - 1))] = acc;
      }
    }
  }
  __syncthreads();
  QMC_TS(1);
  double2 v[E];
  load_strided<L2, E>(v, S);
  fftE<L2, E, -1>(v, S, tws, tid);
  QMC_TS(2);
  if (f1 == 0 && tid == 0) {
    colsum[k1] = v[0].x;
    if (has2) colsum[k2] = v[0].y;
  }
  const double2* Wr = W + int64_t(f1) * L2;
#pragma unroll
  for (int q = 0; q < E; ++q) v[q] = cmul(v[q], ldg_ordered(&Wr[tid + q * NT]));
  QMC_TS(3);
  fftE<L2, E, +1>(v, S, tws, tid);
  QMC_TS(4);
  if constexpr (L1C == 0) {
    // U[p] in column blocks of kUB: [e2 / kUB][f1][e2 % kUB], so that K2 reads
    // (and discards) whole contiguous lines
    double2* Up = U + p * L + int64_t(f1) * kUB;
    const int L1 = int(L / L2);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int e2 = tid + q * NT;
      Up[int64_t(e2 / kUB) * (L1 * kUB) + (e2 % kUB)] = v[q];
    }
  } else {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __syncthreads();  // every thread has finished reading S in the last stage
    store_strided<L2, E>(v, S);
    cluster.sync();
    const double2* Sr[L1C];
#pragma unroll
    for (int r = 0; r < L1C; ++r) Sr[r] = cluster.map_shared_rank(S, r);
    double2* Bp = U + p * L;
    for (int c = f1 * NT + tid; c < L2; c += L1C * NT) {
      double2 u[L1C], pw[L1C];
      pw[0] = make_double2(1.0, 0.0);
      if (L1C > 1) pw[1] = __ldg(&twL[c]);  // ω_L^{c}
#pragma unroll
      for (int r = 2; r < L1C; ++r) pw[r] = cmul(pw[r / 2], pw[r - r / 2]);
#pragma unroll
      for (int r = 0; r < L1C; ++r) u[r] = Sr[r][padE<E>(c)];
#pragma unroll
      for (int r = 1; r < L1C; ++r) u[r] = cmulc(u[r], pw[r]);
      reg_dft<L1C, +1>(u, tw1);
#pragma unroll
      for (int r = 0; r < L1C; ++r) Bp[int64_t(r) * L2 + c] = u[r];
    }
    cluster.sync();  // keep this CTA's row alive until every reader is done
  }
  QMC_TS(5);
}

// ---------------------------------------------------------------- K2
// Inverse DFT of length L1 along f1 for CB adjacent columns e2 of every pair
// of the batch, after the twiddle conj(ω_L^{e2 f1}); writes the batch
// pair-interleaved: Y[(L2·e1 + e2)·np + p] = B'_p[L2·e1 + e2].
// Register path (L1 = R·M, R, M direct radices): one thread per column.
constexpr int kColCB = kUB;  // columns e2 per CTA in the register path
// Grid (L2/CB column blocks, pair groups of kColPG): the shared tile does not
// grow with the batch.
constexpr int kColPG = 16;
template <int L1>
__global__ void __launch_bounds__(256)
    k_cols_reg(const double2* __restrict__ U, int64_t L, int L2, int lg2L2, int npb, int NPP,
               const double2* __restrict__ tw1, const double2* __restrict__ twL, double2* __restrict__ Yb) {
  constexpr int CB = kColCB, SA = L1 + 2;  // SA ≡ 2 (mod 8) for even L1: phase A conflict-free
  extern __shared__ double2 sm[];
  const int pg0 = blockIdx.y * kColPG;
  const int np = min(kColPG, npb - pg0);   // pairs of this CTA
  U += int64_t(pg0) * L;
  double2* Y = Yb + pg0;                   // Y[e·npb + pg0 + p]
  double2* tcta = sm;                      // [L1][CB] ω_L^{e2·f1}
  double2* tileA = sm + L1 * CB;           // [p·CB + c][SA]
  double2* tileC = tileA + kColPG * CB * SA;  // [e1·CB + c][NPP], NPP ≡ 2 (mod 8)
  const int e2_0 = blockIdx.x * CB;
  for (int i = threadIdx.x; i < L1 * CB; i += blockDim.x) {
    const int f1 = i / CB, c = i % CB;
    const int x = (e2_0 + c) * f1;
    tcta[i] = cmul(__ldg(&tw1[x >> lg2L2]), __ldg(&twL[x & (L2 - 1)]));
  }
  __syncthreads();
  const int tot = np * L1 * CB;
  constexpr int UA = 8;  // loads in flight per thread
  for (int i0 = 0; i0 < tot; i0 += 256 * UA) {
    double2 u[UA];
#pragma unroll
    for (int k = 0; k < UA; ++k) {
      const int idx = i0 + k * 256 + threadIdx.x;
      if (idx < tot) {
        const int c = idx % CB, r = idx / CB;
        const int f1 = r % L1, p = r / L1;
        u[k] = __ldg(&U[int64_t(p) * L + int64_t(blockIdx.x) * (L1 * CB) + f1 * CB + c]);
      }
    }
#pragma unroll
    for (int k = 0; k < UA; ++k) {
      const int idx = i0 + k * 256 + threadIdx.x;
      if (idx < tot) {
        const int c = idx % CB, r = idx / CB;
        const int f1 = r % L1, p = r / L1;
        tileA[(p * CB + c) * SA + f1] = cmulc(u[k], tcta[f1 * CB + c]);
      }
    }
  }
  __syncthreads();
  // this CTA's block of U (L1·CB complex per pair, contiguous) is dead now
  {
    constexpr int LPB = (L1 * CB * 16) / 128;  // whole lines per pair block
    for (int i = threadIdx.x; i < np * LPB; i += blockDim.x) {
      const int p = i / LPB, l = i % LPB;
      discard_l2(reinterpret_cast<const char*>(U + int64_t(p) * L + int64_t(blockIdx.x) * (L1 * CB)) + 128 * l);
    }
  }
  for (int col = threadIdx.x; col < np * CB; col += blockDim.x) {
    double2 v[L1];
#pragma unroll
    for (int f1 = 0; f1 < L1; ++f1) v[f1] = tileA[col * SA + f1];
    reg_dft<L1, +1>(v, tw1);
    const int p = col / CB, c = col % CB;
#pragma unroll
    for (int e1 = 0; e1 < L1; ++e1) tileC[(e1 * CB + c) * NPP + p] = v[e1];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {  // p fastest: coalesced rows of Y
    const int p = idx % np, rc = idx / np;
    const int e1 = rc / CB, c = rc % CB;
    Y[(int64_t(e1) * L2 + e2_0 + c) * npb + p] = tileC[rc * NPP + p];
  }
}

// Persistent, software-pipelined register path.  A tile is (column block of
// kUB columns, kPipePG pairs): kPipePG contiguous blocks of L1·kUB complex
// (K1's blocked layout), copied into shared memory with cp.async while the
// previous tile is transformed and stored.  One thread per column (p, c).
constexpr int kPipePG = 16;
constexpr int kPipeThreads = kPipePG * kUB;  // 64

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int L1>
__global__ void __launch_bounds__(kPipeThreads)
    k_cols_pipe(const double2* __restrict__ U, int64_t L, int L2, int lg2L2, int npb, int NPP,
                const double2* __restrict__ tw1, const double2* __restrict__ twL, double2* __restrict__ Y) {
  constexpr int CB = kUB, BLK = L1 * CB, BLKP = BLK + 4;  // pair stride padded: conflict-free reads
  extern __shared__ double2 sm[];
  double2* buf[2] = {sm, sm + kPipePG * BLKP};
  double2* tileC = sm + 2 * kPipePG * BLKP;  // [e1·CB + c][NPP]
  const int nblk = L2 / CB, ngrp = (npb + kPipePG - 1) / kPipePG;
  const int ntiles = nblk * ngrp;
  const int tid = threadIdx.x;
  auto issue = [&](int tile, double2* dst) {
    const int b = tile % nblk, g = tile / nblk;
    const int np = min(kPipePG, npb - g * kPipePG);
    for (int i = tid; i < np * BLK; i += kPipeThreads) {
      const int p = i / BLK, o = i % BLK;
      cp_async16(dst + p * BLKP + o, U + int64_t(g * kPipePG + p) * L + int64_t(b) * BLK + o);
    }
  };
  int tile = blockIdx.x;
  if (tile < ntiles) issue(tile, buf[0]);
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int nxt = tile + gridDim.x;
    if (nxt < ntiles) issue(nxt, buf[(it + 1) & 1]);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double2* cur = buf[it & 1];
    const int b = tile % nblk, g = tile / nblk;
    const int np = min(kPipePG, npb - g * kPipePG);
    const int p = tid / CB, c = tid % CB;
    if (p < np) {
      const int e2 = b * CB + c;
      // twiddles conj(ω_L^{e2·f1}) = conj(w^f1), w = ω_L^{e2}: product tree
      double2 pw[L1], v[L1];
      pw[0] = make_double2(1.0, 0.0);
      if (L1 > 1) pw[1] = __ldg(&twL[e2]);
#pragma unroll
      for (int r = 2; r < L1; ++r) pw[r] = cmul(pw[r / 2], pw[r - r / 2]);
#pragma unroll
      for (int f1 = 0; f1 < L1; ++f1) v[f1] = cmulc(cur[p * BLKP + f1 * CB + c], pw[f1]);
      reg_dft<L1, +1>(v, tw1);
#pragma unroll
      for (int e1 = 0; e1 < L1; ++e1) tileC[(e1 * CB + c) * NPP + p] = v[e1];
    }
    __syncthreads();
    // the U block of this tile is dead: drop it from L2 without write-back
    for (int i = tid; i < np * (BLK * 16 / 128); i += kPipeThreads) {
      const int pp = i / (BLK * 16 / 128), l = i % (BLK * 16 / 128);
      discard_l2(reinterpret_cast<const char*>(U + int64_t(g * kPipePG + pp) * L + int64_t(b) * BLK) + 128 * l);
    }
    double2* Yg = Y + g * kPipePG;
    for (int i = tid; i < BLK * np; i += kPipeThreads) {  // p fastest: coalesced rows of Y
      const int pp = i % np, rc = i / np;
      const int e1 = rc / CB, cc = rc % CB;
      Yg[(int64_t(e1) * L2 + b * CB + cc) * npb + pp] = tileC[rc * NPP + pp];
    }
    __syncthreads();  // tileC and buf[it & 1] are reused
  }
  cp_async_wait<0>();
}

// Generic path (any smooth L1 <= 1024): one CTA per (CB columns, pair),
// Stockham stages over shared memory with runtime radices.
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

__global__ void __launch_bounds__(256)
    k_cols_smem(const double2* __restrict__ U, int64_t L, int L1, int L2, int CB, int np,
                const int32_t* __restrict__ rad, int nrad, const double2* __restrict__ tw1,
                const double2* __restrict__ twL, double2* __restrict__ Y) {
  extern __shared__ double2 smem[];
  double2* in = smem;
  double2* out = smem + L1 * CB;
  const int p = blockIdx.y;
  const int c0 = blockIdx.x * CB;
  const double2* Up = U + int64_t(p) * L;
  const int tot = L1 * CB;
  for (int q = threadIdx.x; q < tot; q += blockDim.x) {
    const int f1 = q / CB, c = q - f1 * CB;
    const int e2 = c0 + c;
    const int x = e2 * f1;
    const double2 w = cmul(__ldg(&tw1[x / L2]), __ldg(&twL[x % L2]));
    in[q] = cmulc(Up[int64_t(e2 / kUB) * (L1 * kUB) + f1 * kUB + (e2 % kUB)], w);
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
    Y[(int64_t(e1) * L2 + c0 + c) * np + p] = in[q];
  }
}

// ---------------------------------------------------------------- K3
// Grid (row blocks, pair groups): thread = conventional row n, looping over
// the pairs [g·ppg, (g+1)·ppg) of the batch; B' of all pairs of the batch at
// reordered index R[n] is contiguous in Y.  ROWSUM mode accumulates
// Σ_k X[n,k] into rowsum[g·N + n] (reduced over g at the end of the call).
template <int MODE>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather(const double2* __restrict__ Y, int64_t sE, int64_t sP, int np, int ppg, int64_t pair0, int64_t t,
             const int32_t* __restrict__ R, const double* __restrict__ colsum,
             const double* __restrict__ scal, int64_t N, double* __restrict__ X, int64_t ldx,
             double* __restrict__ rowsum, int first) {
  const int64_t n = int64_t(blockIdx.x) * kGatherThreads + threadIdx.x;
  if (n >= N) return;
  const int g = blockIdx.y;
  const int pb = g * ppg, pe = min(np, pb + ppg);
  double rs = 0.0;
  if (n == 0) {
    const double phi0 = __ldg(scal);
    for (int p = pb; p < pe; ++p) {
      const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
      const bool has2 = k2 < t;
      const double2 v = make_double2(phi0 * colsum[k1], has2 ? phi0 * colsum[k2] : 0.0);
      if (X) {
        X[k1 * ldx] = v.x;
        if (has2) X[k2 * ldx] = v.y;
      }
      rs += v.x;
      if (has2) rs += v.y;
    }
  } else {
    const double2* yp = Y + int64_t(__ldg(&R[n])) * sE;
    double* Xn = X ? X + n + 2 * pair0 * ldx : nullptr;
    int p = pb;
    constexpr int U8 = 8;
    const bool al32 = sP == 1 && ((np | pb) & 1) == 0;  // interleaved and yp + p 32-byte aligned
    for (; p + U8 <= pe && 2 * (pair0 + p + U8 - 1) + 1 < t; p += U8) {
      double2 v[U8];
      if (al32) {
#pragma unroll
        for (int i = 0; i < U8; i += 2) QMC_LD2(&yp[p + i], v[i], v[i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < U8; ++i) v[i] = QMC_LD1(&yp[(p + i) * sP]);
      }
#pragma unroll
      for (int i = 0; i < U8; ++i) {
        if (Xn) {
          QMC_ST(&Xn[(2 * (p + i)) * ldx], v[i].x);
          QMC_ST(&Xn[(2 * (p + i) + 1) * ldx], v[i].y);
        }
        rs += v[i].x;
        rs += v[i].y;
      }
    }
    for (; p < pe; ++p) {
      const int64_t k2 = 2 * (pair0 + p) + 1;
      const bool has2 = k2 < t;
      const double2 v = __ldg(&yp[p * sP]);
      if (Xn) {
        Xn[(2 * p) * ldx] = v.x;
        if (has2) Xn[(2 * p + 1) * ldx] = v.y;
      }
      rs += v.x;
      if (has2) rs += v.y;
    }
    // interleaved layout: whole lines inside [pb, pe) were read only by this
    // thread and are dead now
    if (sP == 1) {
      const uintptr_t b0 = (reinterpret_cast<uintptr_t>(yp + pb) + 127) & ~uintptr_t(127);
      const uintptr_t b1 = reinterpret_cast<uintptr_t>(yp + pe) & ~uintptr_t(127);
      for (uintptr_t b = b0; b < b1; b += 128) discard_l2(reinterpret_cast<const void*>(b));
    }
  }
  if (MODE == GM_ROWSUM) {
    double* rsg = rowsum + int64_t(g) * N;
    rsg[n] = (first ? 0.0 : rsg[n]) + rs;
  }
}

__global__ void k_rowsum_reduce(const double* __restrict__ parts, int ng, int ngstride, int nsets, int64_t N,
                                double* __restrict__ out) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int k = 0; k < nsets; ++k)
    for (int g = 0; g < ng; ++g) s += parts[(int64_t(k) * ngstride + g) * N + n];
  out[n] = s;
}

// Grid (row blocks of kColMeanRows, pair groups): writes X (c + X for
// AFFINE) and the per-column block sums of f(X) into partial[nb·t + k]
// (warp shuffles, then a fixed-order sum over warps).
template <int F>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather_colmean(const double2* __restrict__ Y, int64_t sE, int64_t sP, int np, int ppg, int64_t pair0, int64_t t,
                     const int32_t* __restrict__ R, const double* __restrict__ colsum,
                     const double* __restrict__ scal, int64_t N, double fparam,
                     double* __restrict__ X, int64_t ldx, double* __restrict__ partial) {
  extern __shared__ double2 red[];  // [kGatherThreads/32][ppg]
  constexpr int RPT = kColMeanRows / kGatherThreads;
  const int64_t nb = blockIdx.x;
  const int g = blockIdx.y;
  const int pb = g * ppg, pe = min(np, pb + ppg);
  const double phi0 = __ldg(scal);
  int64_t rows[RPT];
  int rr[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    rows[i] = nb * kColMeanRows + i * kGatherThreads + threadIdx.x;
    rr[i] = (rows[i] > 0 && rows[i] < N) ? __ldg(&R[rows[i]]) : 0;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int p = pb; p < pe; ++p) {
    const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
    const bool has2 = k2 < t;
    double2 vv[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      vv[i] = rows[i] == 0 ? make_double2(phi0 * colsum[k1], has2 ? phi0 * colsum[k2] : 0.0)
              : rows[i] < N ? __ldg(&Y[int64_t(rr[i]) * sE + p * sP]) : make_double2(0.0, 0.0);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t n = rows[i];
      if (n < N) {
        double2 v = vv[i];
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
          if (has2) acc.y += exp(v.y);
        } else {
          acc.x += v.x;
          if (has2) acc.y += v.y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
    }
    if (l == 0) red[w * ppg + (p - pb)] = acc;
  }
  __syncthreads();
  for (int p = pb + threadIdx.x; p < pe; p += kGatherThreads) {
    double2 sacc = make_double2(0.0, 0.0);
    for (int ww = 0; ww < kGatherThreads / 32; ++ww) sacc = cadd(sacc, red[ww * ppg + (p - pb)]);
    const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
    partial[nb * t + k1] = sacc.x;
    if (k2 < t) partial[nb * t + k2] = sacc.y;
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
  size_t off_U, off_Y, off_colsum, off_partial, off_rowsum, total;
  int ngroups, ppg, nsets;
};

// pair groups of the gather: enough rows × groups for ~2 waves of threads
static void gather_groups(const qmc_plan* pl, int64_t pairs, int* ngroups, int* ppg) {
  int64_t g = std::max<int64_t>(1, (int64_t(148) * 2048 * 2) / std::max<int64_t>(pl->N, 1));
  g = std::min<int64_t>(g, pairs);
  const int64_t per = (pairs + g - 1) / g;
  *ppg = int(per);
  *ngroups = int((pairs + per - 1) / per);
}

static CallLayout call_layout(const qmc_plan* pl, int64_t t, int f) {
  CallLayout c;
  const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(pl->batch_pairs, (t + 1) / 2));
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o = align_up(o + b);
    return r;
  };
  // one scratch set (U, Y, row-sum parts) per internal stream in use
  const int64_t nbatch = ((t + 1) / 2 + pl->batch_pairs - 1) / pl->batch_pairs;
  c.nsets = (pl->nstreams == 2 && nbatch > 1) ? 2 : 1;
  c.off_U = take(size_t(c.nsets) * pairs * pl->sp.L * 16);
  c.off_Y = take(pl->cluster || pl->sp.L1 == 1 ? 0 : size_t(c.nsets) * pairs * pl->sp.L * 16);
  c.off_colsum = take(size_t(std::max<int64_t>(t, 1)) * 8);
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  const int64_t nblocks = (pl->N + kColMeanRows - 1) / kColMeanRows;
  c.off_partial = take(colmean ? size_t(nblocks) * std::max<int64_t>(t, 1) * 8 : 0);
  gather_groups(pl, pairs, &c.ngroups, &c.ppg);
  c.off_rowsum = take(f == QMC_F_ROWMEAN_RELU ? size_t(c.nsets) * c.ngroups * pl->N * 8 : 0);
  c.total = o;
  return c;
}

template <typename K>
static void set_smem_attr(K kernel) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

template <int L2, int L1C>
static int launch_rows(const qmc_plan* pl, const double* A, int64_t lda, int64_t t, int64_t pair0,
                       double2* U, int npairs, double* colsum, cudaStream_t st) {
  const size_t smem = size_t(PadE<L2, QMC_ROW_E>::size) * sizeof(double2);
  auto kern = k_rows16<L2, L1C>;
  set_smem_attr(kern);
  dim3 grid((unsigned)pl->sp.L1, (unsigned)npairs);
  if constexpr (L1C == 0) {
    kern<<<grid, L2 / QMC_ROW_E, smem, st>>>(A, lda, t, pair0, pl->d_e, pl->d_bnext, pl->s, pl->d_twj, pl->d_tws,
                                             pl->d_W, U, pl->sp.L, colsum, pl->d_twL, pl->d_tw1);
  } else {
    if (L1C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(L2 / QMC_ROW_E, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L1C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, A, lda, t, pair0, (const int32_t*)pl->d_e, (const int32_t*)pl->d_bnext,
                           pl->s, (const double2*)pl->d_twj, (const double2*)pl->d_tws, (const double2*)pl->d_W, U,
                           pl->sp.L, colsum, (const double2*)pl->d_twL, (const double2*)pl->d_tw1) != cudaSuccess) {
      cudaGetLastError();
      return QMC_ECUDA;
    }
  }
  QMC_LAUNCHED();
  return QMC_OK;
}

// (L2, L1) pairs with a cluster instantiation of K1
#define QMC_CLUSTER_PAIRS(X)                                                                               \
  X(1024, 2) X(1024, 4) X(1024, 5) X(1024, 8) X(1024, 10) X(1024, 16) X(2048, 2) X(2048, 4) X(2048, 5)    \
  X(2048, 8) X(2048, 10) X(2048, 16) X(4096, 2) X(4096, 4) X(4096, 5) X(4096, 8) X(4096, 10) X(4096, 16)  \
  X(8192, 2) X(8192, 4) X(8192, 5) X(8192, 8) X(8192, 10) X(8192, 16)

static int rows_dispatch(const qmc_plan* pl, const double* A, int64_t lda, int64_t t, int64_t pair0, double2* U,
                         int np, double* colsum, cudaStream_t st) {
  if (pl->cluster) {
#define QMC_CL_CASE(A2, A1) \
  if (pl->sp.L2 == A2 && pl->sp.L1 == A1) return launch_rows<A2, A1>(pl, A, lda, t, pair0, U, np, colsum, st);
    QMC_CLUSTER_PAIRS(QMC_CL_CASE)
#undef QMC_CL_CASE
    return QMC_EINVAL_N;
  }
  switch (pl->sp.L2) {
#define QMC_ROWS_CASE(NN) \
  case NN: return launch_rows<NN, 0>(pl, A, lda, t, pair0, U, np, colsum, st);
    QMC_ROWS_CASE(16) QMC_ROWS_CASE(32) QMC_ROWS_CASE(64) QMC_ROWS_CASE(128) QMC_ROWS_CASE(256)
    QMC_ROWS_CASE(512) QMC_ROWS_CASE(1024) QMC_ROWS_CASE(2048) QMC_ROWS_CASE(4096) QMC_ROWS_CASE(8192)
#undef QMC_ROWS_CASE
  }
  return QMC_EINVAL_N;
}

// Can K1 run with the fused cluster column pass for this plan?  (an
// instantiation exists and at least one cluster fits on the device)
int rows_cluster_supported(const qmc_plan* pl) {
#define QMC_CL_OCC(A2, A1)                                                                           \
  if (pl->sp.L2 == A2 && pl->sp.L1 == A1) {                                                        \
    auto kern = k_rows16<A2, A1>;                                                                  \
    set_smem_attr(kern);                                                                           \
    if (A1 > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);     \
    cudaLaunchConfig_t cfg = {};                                                                   \
    cfg.gridDim = dim3(A1, 1, 1);                                                                  \
    cfg.blockDim = dim3(A2 / QMC_ROW_E, 1, 1);                                                     \
    cfg.dynamicSmemBytes = size_t(PadE<A2, QMC_ROW_E>::size) * sizeof(double2);                    \
    cudaLaunchAttribute attr[1];                                                                   \
    attr[0].id = cudaLaunchAttributeClusterDimension;                                              \
    attr[0].val.clusterDim.x = A1;                                                                 \
    attr[0].val.clusterDim.y = 1;                                                                  \
    attr[0].val.clusterDim.z = 1;                                                                  \
    cfg.attrs = attr;                                                                              \
    cfg.numAttrs = 1;                                                                              \
    int nclusters = 0;                                                                             \
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess) {                   \
      cudaGetLastError();                                                                          \
      return 0;                                                                                    \
    }                                                                                              \
    return nclusters > 0;                                                                          \
  }
  QMC_CLUSTER_PAIRS(QMC_CL_OCC)
#undef QMC_CL_OCC
  return 0;
}

static int ilog2(int64_t x) {
  int r = 0;
  while ((int64_t(1) << r) < x) ++r;
  return r;
}

size_t cols_reg_smem(int64_t L1, int64_t /*np*/) {
  const int64_t np = kColPG, npp = np + ((2 - np % 8) + 8) % 8;  // ≡ 2 (mod 8)
  return size_t(L1 * kColCB + np * kColCB * (L1 + 2) + L1 * kColCB * npp) * 16;
}

template <int L1>
static int launch_cols_reg(const qmc_plan* pl, const double2* U, double2* Y, int np, cudaStream_t st) {
  if (getenv("QMC_COLS_OLD")) {
    const size_t smem = cols_reg_smem(L1, np);
    const int npp = kColPG + ((2 - kColPG % 8) + 8) % 8;
    set_smem_attr(k_cols_reg<L1>);
    dim3 g((unsigned)(pl->sp.L2 / kColCB), (unsigned)((np + kColPG - 1) / kColPG));
    k_cols_reg<L1><<<g, 256, smem, st>>>(U, pl->sp.L, int(pl->sp.L2), ilog2(pl->sp.L2), np, npp, pl->d_tw1,
                                         pl->d_twL, Y);
    QMC_LAUNCHED();
    return QMC_OK;
  }
  constexpr int BLKP = L1 * kUB + 4;
  const int npp = kPipePG + ((2 - kPipePG % 8) + 8) % 8;
  const size_t smem = size_t(2 * kPipePG * BLKP + L1 * kUB * npp) * sizeof(double2);
  set_smem_attr(k_cols_pipe<L1>);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cols_pipe<L1>, kPipeThreads, smem);
  const int64_t ntiles = (pl->sp.L2 / kUB) * ((np + kPipePG - 1) / kPipePG);
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(nsm) * std::max(per_sm, 1))));
  k_cols_pipe<L1><<<grid, kPipeThreads, smem, st>>>(U, pl->sp.L, int(pl->sp.L2), ilog2(pl->sp.L2), np, npp,
                                                    pl->d_tw1, pl->d_twL, Y);
  QMC_LAUNCHED();
  return QMC_OK;
}

static int cols_dispatch(const qmc_plan* pl, const double2* U, double2* Y, int np, cudaStream_t st) {
  if (pl->col_reg) {
    switch (pl->sp.L1) {
#define QMC_COLS_CASE(NN) \
  case NN: return launch_cols_reg<NN>(pl, U, Y, np, st);
      QMC_COLS_CASE(2) QMC_COLS_CASE(3) QMC_COLS_CASE(4) QMC_COLS_CASE(5) QMC_COLS_CASE(6) QMC_COLS_CASE(8)
      QMC_COLS_CASE(9) QMC_COLS_CASE(10) QMC_COLS_CASE(12) QMC_COLS_CASE(15) QMC_COLS_CASE(16) QMC_COLS_CASE(20)
      QMC_COLS_CASE(24) QMC_COLS_CASE(25) QMC_COLS_CASE(32)
#undef QMC_COLS_CASE
    }
  }
  const int CB = pl->col_cb_smem;
  const size_t smem = size_t(2) * pl->sp.L1 * CB * sizeof(double2);
  set_smem_attr(k_cols_smem);
  dim3 g((unsigned)(pl->sp.L2 / CB), (unsigned)np);
  k_cols_smem<<<g, 256, smem, st>>>(U, pl->sp.L, int(pl->sp.L1), int(pl->sp.L2), CB, np, pl->d_rad1, pl->nrad1,
                                    pl->d_tw1, pl->d_twL, Y);
  QMC_LAUNCHED();
  return QMC_OK;
}

static unsigned nblk(int64_t n, int b) { return unsigned((n + b - 1) / b); }

// all batches of column pairs; f = -1: X only
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
  const int64_t pairs_b = std::max<int64_t>(1, std::min<int64_t>(pl->batch_pairs, (t + 1) / 2));
  double* colsum = (double*)(ws + cl.off_colsum);
  double* partial = (double*)(ws + cl.off_partial);
  const int64_t npairs_total = (t + 1) / 2;
  const int64_t nb3 = (pl->N + kColMeanRows - 1) / kColMeanRows;
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  const int nsets = cl.nsets;
  std::unique_lock<std::mutex> lock;
  if (nsets == 2) {  // fork: both internal streams start after the caller's prior work
    lock = std::unique_lock<std::mutex>(*pl->mu);
    if (cudaEventRecord(pl->ev_fork, st) != cudaSuccess ||
        cudaStreamWaitEvent(pl->ist[0], pl->ev_fork, 0) != cudaSuccess ||
        cudaStreamWaitEvent(pl->ist[1], pl->ev_fork, 0) != cudaSuccess) {
      cudaGetLastError();
      return QMC_ECUDA;
    }
  }
  int64_t bidx = 0;
  for (int64_t pair0 = 0; pair0 < npairs_total; pair0 += pl->batch_pairs, ++bidx) {
    const int np = int(std::min<int64_t>(pl->batch_pairs, npairs_total - pair0));
    const int set = nsets == 2 ? int(bidx & 1) : 0;
    const cudaStream_t bs = nsets == 2 ? pl->ist[set] : st;
    double2* U = (double2*)(ws + cl.off_U) + size_t(set) * pairs_b * pl->sp.L;
    double2* Y = (double2*)(ws + cl.off_Y) + size_t(set) * pairs_b * pl->sp.L;
    double* rowparts = (double*)(ws + cl.off_rowsum) + size_t(set) * cl.ngroups * pl->N;
    const int first = bidx < nsets;  // first batch of this scratch set
    {
      const cudaStream_t st = bs;
      prof_begin(KC_ROWS, st);
      int rc = rows_dispatch(pl, A, lda, t, pair0, U, np, colsum, st);
      if (rc) return rc;
      prof_end(KC_ROWS, st);
      // B' of the batch: natural [p][e] (cluster K1, or L1 = 1) or pair-interleaved [e][p] (K2)
      const double2* Yb = U;
      int64_t sE = 1, sP = pl->sp.L;
      if (!pl->cluster && pl->sp.L1 > 1) {
        prof_begin(KC_COLS, st);
        rc = cols_dispatch(pl, U, Y, np, st);
        if (rc) return rc;
        prof_end(KC_COLS, st);
        Yb = Y;
        sE = np;
        sP = 1;
      }
      prof_begin(KC_GATHER, st);
      const int ppg = cl.ppg;
      const unsigned ng = unsigned((np + ppg - 1) / ppg);
      if (colmean) {
        const size_t smem = size_t(kGatherThreads / 32) * ppg * sizeof(double2);
        dim3 g((unsigned)nb3, ng);
        switch (f) {
          case QMC_F_IDENTITY:
            k_gather_colmean<QMC_F_IDENTITY><<<g, kGatherThreads, smem, st>>>(
                Yb, sE, sP, np, ppg, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, fparam, X, ldx, partial);
            break;
          case QMC_F_AFFINE:
            k_gather_colmean<QMC_F_AFFINE><<<g, kGatherThreads, smem, st>>>(
                Yb, sE, sP, np, ppg, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, fparam, X, ldx, partial);
            break;
          default:
            k_gather_colmean<QMC_F_EXP><<<g, kGatherThreads, smem, st>>>(
                Yb, sE, sP, np, ppg, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, fparam, X, ldx, partial);
        }
        QMC_LAUNCHED();
      } else if (f == QMC_F_ROWMEAN_RELU) {
        // groups absent from a short last batch keep their sums (first = 0)
        dim3 g(nblk(pl->N, kGatherThreads), ng);
        k_gather<GM_ROWSUM><<<g, kGatherThreads, 0, st>>>(Yb, sE, sP, np, ppg, pair0, t, pl->d_R, colsum, pl->d_scal,
                                                          pl->N, X, ldx, rowparts, first);
        QMC_LAUNCHED();
      } else {
        dim3 g(nblk(pl->N, kGatherThreads), ng);
        k_gather<GM_X><<<g, kGatherThreads, 0, st>>>(Yb, sE, sP, np, ppg, pair0, t, pl->d_R, colsum, pl->d_scal, pl->N, X,
                                                     ldx, nullptr, 0);
        QMC_LAUNCHED();
      }
      prof_end(KC_GATHER, st);
    }
  }
  if (nsets == 2) {  // join
    if (cudaEventRecord(pl->ev_join[0], pl->ist[0]) != cudaSuccess ||
        cudaEventRecord(pl->ev_join[1], pl->ist[1]) != cudaSuccess ||
        cudaStreamWaitEvent(st, pl->ev_join[0], 0) != cudaSuccess ||
        cudaStreamWaitEvent(st, pl->ev_join[1], 0) != cudaSuccess) {
      cudaGetLastError();
      return QMC_ECUDA;
    }
  }
  if (f == QMC_F_ROWMEAN_RELU) {
    prof_begin(KC_REDUCE, st);
    // parts [set][group][N]; every written group of every set, fixed order
    const int ngr = int(std::min<int64_t>(cl.ngroups, (npairs_total + cl.ppg - 1) / cl.ppg));
    const int nsets_used = int(std::min<int64_t>(nsets, (npairs_total + pl->batch_pairs - 1) / pl->batch_pairs));
    k_rowsum_reduce<<<nblk(pl->N, 256), 256, 0, st>>>((double*)(ws + cl.off_rowsum), ngr, cl.ngroups,
                                                      nsets_used, pl->N, out);
    QMC_LAUNCHED();
    prof_end(KC_REDUCE, st);
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
