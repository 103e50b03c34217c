// pipeline.cu — the hot path of libqmc: X = Y·A by the fast QMC matrix
// method, fused with the row-0 term, the un-permutation
// to conventional order and the optional QMC-mean epilogue.
//
// Per column pair (k1, k2) packed as a = A[:,k1] + i·A[:,k2] (ζ is real, so
// one complex correlation serves two real columns), with the plan's split
// L = L1·L2 (e = L2·e1 + e2, f = f1 + L1·f2, NT = L2/16 row threads, e2 =
// t + NT q):
//
//   K0 k_pack*     a of the batch in the K1 slot order (or the dense a', then
//                  the first DFT dimension by k_dense_cols*)
//   K1 k_rows16    T'[f1,e2] = ω_L^{e2 f1} Σ_{j: e_j ≡ e2} a_j ω_{L1}^{e1_j f1}
//                  (scatter a' = P a fused with the first FFT dimension,
//                  PAPER.md:355-357; e1_j = e_j div L2; the bucket's common
//                  four-step twiddle ω_L^{e2 f1} applied to the summed row:
//                  ω_{16 L1}^{q f1} per register, ω_L^{t f1} in the row FFT's
//                  first stage)
//                  → FFT_L2 → ·W → IFFT_L2 → ·conj(ω_L^{e2 f1}) → U[p][f1][e2]
//                  (fft.cuh dif_fwd / dif_inv, registers + shared memory)
//   K2 k_cols_*    IFFT_L1 over f1 → B'[L2 e1 + e2]; the reordered row
//                  i = L2 e1 + e2 is conventional row n = β^{-i} =
//                  P[(m - i) mod m], so K2 writes the row
//                  chunk X[n, 2p..2p+1 of the pair group] directly (X
//                  row-major); X[0,k] = φ(0) Σ_j A[j,k];
//                  fused f, per-column or per-row partial sums
//   K3 k_colpart_reduce / k_rowsum_reduce   fixed-order reductions
//   one-row plans (L1 = 1): k_small, the whole call in one kernel;
//   Korobov p-sets: k_pset, all blocks of one plan in one launch
//
// B'[i] = Σ_j a_j ζ[(e_j - i) mod m] = (Z P a)_i is a cyclic correlation,
// computed as IDFT(DFT(a') · DFT(K)), K[d] = ζ[(-d) mod m] (zero-padded to
// L >= 2m-1 when m does not split into supported radices).  U of a batch of
// column pairs (plan->batch_pairs) round-trips through DRAM between K1 and
// K2; the batch is sized for launch efficiency.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "fft.cuh"
#include "qmc_internal.cuh"
#include "rowcfg.cuh"

namespace qmc {

constexpr int kColThreads = 256;  // K2 CTA size

// X is written once and never read back by the library: evict-first stores
// keep it from pushing the batch's U out of L2 (QMC_X_PLAIN_STORES: plain)
#ifndef QMC_X_PLAIN_STORES
#define QMC_XST2(p, v) stcs2(p, v)
#define QMC_XST(p, v) stcs(p, v)
#else
#define QMC_XST2(p, v) (*reinterpret_cast<double2*>(p) = (v))
#define QMC_XST(p, v) (*(p) = (v))
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

// ---------------------------------------------------------------- K0
// a of the batch in the K1 order: asort[p·S1 + q] = (A[j_q, k1], A[j_q, k2]),
// j_q = jq[q] (plan.cu k1_balanced_order; bucket order as fallback), zero for
// padding slots (j_q = -1)
__global__ void k_pack(const double* __restrict__ A, int64_t lda, int64_t t, int64_t pair0, int np,
                       const int32_t* __restrict__ jq, int64_t S1, double2* __restrict__ asort) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (q >= S1 || p >= np) return;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const int64_t j = __ldg(&jq[q]);
  asort[int64_t(p) * S1 + q] = j < 0 ? make_double2(0.0, 0.0)
                                     : make_double2(__ldg(&A[k1 * lda + j]), k2 < t ? __ldg(&A[k2 * lda + j]) : 0.0);
}

// Same output, for s up to kPackSmemMax: the CTA first reads the pair's two
// columns of A into shared memory (coalesced), then gathers from there, so
// the scattered reads hit shared memory instead of L2 sectors.  blockIdx.x =
// pair, blockIdx.y = slice of the S1 slots.  (Measured on B200: config 3,
// s = 4096, 27.0 vs 28.1 ms/step; config 5, s = 8192 with 128 KB per CTA,
// slower than the direct gather — hence the limit.)
constexpr int kPackSmemMax = 4096;
__global__ void __launch_bounds__(256) k_pack_smem(const double* __restrict__ A, int64_t lda, int64_t t,
                                                   int64_t pair0, const int32_t* __restrict__ jq, int64_t s,
                                                   int64_t S1, double2* __restrict__ asort) {
  extern __shared__ double colAB[];  // [2][s]
  const int p = blockIdx.x;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const double* a1 = A + k1 * lda;
  const double* a2 = A + k2 * lda;
  for (int64_t j = threadIdx.x; j < s; j += blockDim.x) {
    colAB[j] = __ldg(&a1[j]);
    colAB[s + j] = k2 < t ? __ldg(&a2[j]) : 0.0;
  }
  __syncthreads();
  const int64_t per = (S1 + gridDim.y - 1) / gridDim.y;
  const int64_t q0 = int64_t(blockIdx.y) * per, q1 = q0 + per < S1 ? q0 + per : S1;
  double2* dst = asort + int64_t(p) * S1;
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const int j = __ldg(&jq[q]);
    dst[q] = j < 0 ? make_double2(0.0, 0.0) : make_double2(colAB[j], colAB[s + j]);
  }
}

// Dense input (plan->k1_dense: every e holds at most one entry and s is too
// large for the sparse first pass, e.g. the CBC all-generators plan):
//   k_pack_dense  a'[p][e] = Σ_{j: e_j = e} (A[j, k1], A[j, k2]) in j order
//                 (jlist / estart: the entries sorted by e, plan.cu)
//   k_dense_cols  T[p][f1][e2] = ω_L^{e2 f1} Σ_{e1} a'[p][L2 e1 + e2] ω_{L1}^{e1 f1}
//                 (the first DFT dimension, an L1-point DFT per column e2)
// K1 then loads its row T[p][f1][:] instead of scattering.
__global__ void k_pack_dense(const double* __restrict__ A, int64_t lda, int64_t t, int64_t pair0,
                             const int32_t* __restrict__ jlist, const int32_t* __restrict__ estart, int64_t L,
                             double2* __restrict__ ad) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (e >= L) return;
  const int64_t k1 = 2 * (pair0 + p), k2 = k1 + 1;
  const double* a1 = A + k1 * lda;
  const double* a2 = A + k2 * lda;
  double2 acc = make_double2(0.0, 0.0);
  for (int q = __ldg(&estart[e]), q1 = __ldg(&estart[e + 1]); q < q1; ++q) {
    const int j = __ldg(&jlist[q]);
    acc.x += __ldg(&a1[j]);
    if (k2 < t) acc.y += __ldg(&a2[j]);
  }
  ad[int64_t(p) * L + e] = acc;
}

template <int L1>
__global__ void __launch_bounds__(256) k_dense_cols(const double2* __restrict__ ad, int64_t L, int L2,
                                                    const double2* __restrict__ tw1,
                                                    const double2* __restrict__ twL, double2* __restrict__ T,
                                                    int64_t ldT) {
  const int e2 = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (e2 >= L2) return;
  const double2* src = ad + int64_t(p) * L + e2;
  double2 v[L1];
#pragma unroll
  for (int e1 = 0; e1 < L1; ++e1) v[e1] = src[int64_t(e1) * L2];
  reg_dft<L1, -1>(v, tw1);
  // × ω_L^{(e2 - e2 mod NT) f1} = w^f1, w = ω_L^{e2 - e2 mod NT}: the four-step
  // twiddle ω_L^{e2 f1} without its row-thread part ω_L^{(e2 mod NT) f1},
  // which K1 folds into its first stage (NT = L2/16): running products
  const int NT = L2 / 16;
  const double2 w = __ldg(&twL[e2 - e2 % NT]);
  double2 tw = w;
  double2* dst = T + int64_t(p) * ldT + e2;
  dst[0] = v[0];
#pragma unroll
  for (int f1 = 1; f1 < L1; ++f1) {
    dst[int64_t(f1) * L2] = cmul(v[f1], tw);
    tw = cmul(tw, w);
  }
}

// L1 = R·M > 16: two register stages through shared memory.  CTA = (pair,
// 32 columns e2); e1 = r + R·mm, f1 = k2 + M·k1:
//   stage A, item (c, r): y[k2] = ω_{L1}^{r k2} Σ_mm a'[L2 (r + R mm) + e2] ω_M^{mm k2}
//   stage B, item (c, k2): T[f1 = k2 + M k1] = ω_L^{e2 f1} Σ_r y_r[k2] ω_R^{r k1}
// columns per CTA of k_dense_cols2 (static shared memory ≤ 48 KB)
__host__ __device__ constexpr int dense2_cb(int L1) { return L1 > 128 ? 8 : (L1 > 64 ? 16 : 32); }

template <int R, int M>
__global__ void __launch_bounds__(256) k_dense_cols2(const double2* __restrict__ ad, int64_t L, int L2,
                                                     const double2* __restrict__ tw1,
                                                     const double2* __restrict__ twL, double2* __restrict__ T,
                                                     int64_t ldT) {
  constexpr int L1 = R * M, CB = dense2_cb(L1), LP = L1 | 1;
  __shared__ double2 Y[CB * LP];  // [c][r·M + k2]
  const int p = blockIdx.y, e20 = blockIdx.x * CB;
  const double2* src = ad + int64_t(p) * L;
  for (int it = threadIdx.x; it < CB * R; it += blockDim.x) {
    const int c = it % CB, r = it / CB;
    const int e2 = e20 + c;
    double2 x[M];
#pragma unroll
    for (int mm = 0; mm < M; ++mm)
      x[mm] = e2 < L2 ? src[int64_t(r + R * mm) * L2 + e2] : make_double2(0.0, 0.0);
    reg_dft<M, -1>(x, tw1, L1 / M);
#pragma unroll
    for (int k2 = 1; k2 < M; ++k2)
      if (r) x[k2] = cmul(x[k2], __ldg(&tw1[r * k2]));
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) Y[c * LP + r * M + k2] = x[k2];
  }
  __syncthreads();
  double2* dst = T + int64_t(p) * ldT;
  for (int it = threadIdx.x; it < CB * M; it += blockDim.x) {
    const int c = it % CB, k2 = it / CB;
    const int e2 = e20 + c;
    if (e2 >= L2) continue;
    double2 z[R];
#pragma unroll
    for (int r = 0; r < R; ++r) z[r] = Y[c * LP + r * M + k2];
    reg_dft<R, -1>(z, tw1, L1 / R);
    // × ω_L^{e2' f1}, e2' = e2 - e2 mod (L2/16) (K1 folds the rest),
    // f1 = k2 + M k1: ω_L^{e2' k2} · (ω_L^{e2' M})^{k1}
    const double2 w = __ldg(&twL[e2 - e2 % (L2 / 16)]);
    double2 b = make_double2(1.0, 0.0);
    for (int q = 0; q < k2; ++q) b = cmul(b, w);
    double2 wM = make_double2(1.0, 0.0);
#pragma unroll
    for (int q = 0; q < M; ++q) wM = cmul(wM, w);
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) {
      dst[int64_t(k2 + M * k1) * L2 + e2] = cmul(z[k1], b);
      b = cmul(b, wM);
    }
  }
}

// ---------------------------------------------------------------- K1
// Persistent: CTA b takes the items (f1, p) = b, b + gridDim.x, ... (f1
// fastest) of the batch; L2/16 threads, 16 points per thread.  Per item:
//   T[f1,e2] = Σ_{j in bucket(e2)} a_j ω_L^{e_j f1}     (a_j = A[j,k1] + i A[j,k2])
//   forward FFT_L2 → ·W[f1,:] → inverse FFT_L2 → U[p][f1][e2]
// The scatter input of an item — (a, twiddle, e2) for the s entries in bucket
// order — is staged in shared memory by cp.async in chunks of CH entries; the
// next item's first chunk is in flight while this item's FFTs run.  A bucket
// is summed in j order by the thread of its first entry in the chunk
// (deterministic).  The twiddle conj(ω_L^{e2 f1}) of the second FFT dimension
// is applied by K2.  Item f1 = 0 also writes the row-0 sums Σ_j a_j = DC term
// of the spectrum.
#ifdef QMC_PHASE_TIMING
__device__ long long g_phase[4096][8];
#define QMC_TS(i)                                                          \
  do {                                                                     \
    __syncthreads();                                                       \
    if (threadIdx.x == 0 && item < 4096) g_phase[item][i] = clock64();     \
  } while (0)
extern "C" int qmc_debug_phases(long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(long long) * 8 * n) == cudaSuccess ? 0 : -7;
}
#else
#define QMC_TS(i) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// U is read exactly once by the column pass: with QMC_U_EF its cp.async
// loads carry an L2 evict-first policy (diagnostic build flag)
__device__ __forceinline__ void cp_async16_u(void* smem, const void* gmem) {
#ifdef QMC_U_EF
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "l"(pol)
               : "memory");
#else
  cp_async16(smem, gmem);
#endif
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// slots of the direct scatter in flight per thread (loop unroll)
#ifndef QMC_K1_PF
#define QMC_K1_PF 0
#endif
#ifndef QMC_W_PF
#define QMC_W_PF 0
#endif
#ifndef QMC_K1_UNROLL
#define QMC_K1_UNROLL 4
#endif
#ifndef QMC_K1_UNROLL_BIG  // rows of 8192 (one CTA per SM): 8 measured best (c5 K1 48.6 -> 47.7 ms, c4 2.39 -> 2.33 ms/step)
#define QMC_K1_UNROLL_BIG 8
#endif
#define QMC_PRAGMA_(x) _Pragma(#x)
#define QMC_UNROLL_(n) QMC_PRAGMA_(unroll n)
#define QMC_UNROLL(n) QMC_UNROLL_(n)

// shared memory of K1 (16-byte slots): the padded row with its padding and
// overflow slots (k1_row_slots); then kK1Aux slots — two buffers of the
// item's 16 register twiddles T16[q] = ω_{16 L1}^{q f1}, the constant
// Tlo[k] = ω_{16 L1}^k (k < 16) — and the constant T1s[k] = ω_{L1}^k (L1
// slots); then, for staged plans, the staging of CH slots (a, twiddle, code:
// 36 B each, CH a multiple of 4) and its mbarrier, for the others the item's
// scatter twiddles ω_{L1}^{e1 f1} in kTwRep replicas (k1_item), followed,
// when the plan stages the first SRn slots (k1_srn), by their a (16 B) and
// codes (4 B) and an mbarrier
constexpr int kTwRep = kK1TwRep;
template <int L2>
__host__ __device__ constexpr int k1_aux_base() { return int(k1_row_slots(L2, QMC_ROW_E)); }
template <int L2>
__host__ __device__ constexpr size_t rows_smem(int CH, int L1, int SRn) {
  return size_t(k1_aux_base<L2>() + kK1Aux + L1) * 16 +
         (CH > 0 ? size_t(CH) * (16 + 16 + 4) + 16
                 : size_t(L1) * kTwRep * 16 + (SRn > 0 ? size_t(SRn) * 20 + 16 : 0));
}

struct K1Args {
  const double2* __restrict__ asort;   // [np][S1] a in the K1 order (K0)
  const int32_t* __restrict__ e2q;     // [S1] bucket codes
  const uint32_t* __restrict__ occ;    // nonempty buckets
  int64_t S1;
  const int32_t* __restrict__ k1c;     // [nch+1] chunk starts, [nch] regular-round slots
  int nch, bal;
  int CH;                              // > 0: staged (one chunk of CH slots, prefetched)
  int SRn;                             // CH = 0, one chunk: its first SRn slots (whole rounds) staged
  int dense;                           // asort holds T[p][f1][e2] (k_dense_cols): no scatter
  const double2* __restrict__ twj;     // [L1][S1]
  const double2* __restrict__ tw2;     // [L2] ω_{L2}^i (row-FFT stage twiddles)
  const double2* __restrict__ tw1;     // [L1] ω_{L1}^i
  const double2* __restrict__ twL;     // [L2] ω_L^i, i < L2
  const double2* __restrict__ tw16;    // [16 L1] ω_{16 L1}^i
  int lg2L2;
  const double2* __restrict__ W;       // [L1][L2] spectrum, row f1 in the K1 register order (dif_freq)
  double2* __restrict__ U;             // [np][L] blocked
  int64_t L;
  int L1, np;
  int64_t pair0, t;
  double* __restrict__ colsum;
};

// Staged mode (plans whose balanced order is one chunk of at most CH slots):
// the scatter input of the NEXT item is copied into shared memory by three
// bulk async copies (one thread, completing on an mbarrier) while this item's
// FFTs run, so its L2 latency is hidden.
template <int L2>
struct K1Stage {
  double2* stA;   // staging: a
  double2* stW;   // staging: twiddles
  int32_t* stE;   // staging: codes
  uint64_t* bar;  // staging complete (one phase per item)
  __device__ K1Stage(double2* base, int CH, int L1)
      : stA(base + k1_aux_base<L2>() + kK1Aux + L1),
        stW(stA + CH),
        stE(reinterpret_cast<int32_t*>(stW + CH)),
        bar(reinterpret_cast<uint64_t*>(stE + CH)) {}
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Direct mode with staged first rounds (SRn > 0): the a and codes of the
// NEXT item's first SRn slots are copied into shared memory by two bulk async
// copies (one thread, an mbarrier) while this item's FFTs run; the item's
// later slots are read from global memory as before.
template <int L2>
struct K1Hyb {
  double2* stA;   // [SRn] a of the pair
  int32_t* stE;   // [SRn] codes
  uint64_t* bar;  // one phase per item
  __device__ K1Hyb(double2* base, int L1, int SRn)
      : stA(base + k1_aux_base<L2>() + kK1Aux + L1 + L1 * kTwRep),
        stE(reinterpret_cast<int32_t*>(stA + SRn)),
        bar(reinterpret_cast<uint64_t*>(stE + SRn)) {}
};
template <int L2>
__device__ __forceinline__ void k1_issue_hyb(const K1Args& a, const K1Hyb<L2>& hb, int it) {
  const int p = it / a.L1;
  const unsigned n = unsigned(a.SRn);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging reads before the async writes
  mbar_expect_tx(hb.bar, n * 20u);
  bulk_g2s(hb.stA, a.asort + int64_t(p) * a.S1, n * 16u, hb.bar);
  bulk_g2s(hb.stE, a.e2q, n * 4u, hb.bar);
}

// stage the single chunk of item it (a of the pair, twiddles of f1, codes);
// the staging buffers must be free.  The code copy is rounded up to 16 bytes
// (the table has 16 bytes of slack).
template <int L2>
__device__ __forceinline__ void k1_issue(const K1Args& a, const K1Stage<L2>& sg, int it) {
  const int f1 = it % a.L1, p = it / a.L1;
  const int n = __ldg(&a.k1c[1]);
  const unsigned b16 = unsigned(n) * 16u, b4 = unsigned((n + 3) & ~3) * 4u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging reads before the async writes
  mbar_expect_tx(sg.bar, 2 * b16 + b4);
  bulk_g2s(sg.stA, a.asort + int64_t(p) * a.S1, b16, sg.bar);
  bulk_g2s(sg.stW, a.twj + int64_t(f1) * a.S1, b16, sg.bar);
  bulk_g2s(sg.stE, a.e2q, b4, sg.bar);
}

// One K1 item (f1, pair).  The scatter input of the item — per slot of the
// plan's order: a_j of the pair (asort, K0), the twiddle of row f1 (twj),
// the code (e2q) — is read straight from global memory (L2-resident: asort
// per batch, twj and e2q per plan) into registers, several slots in flight
// per thread, so no staging buffer, copy or extra barrier is needed.
template <int L2>
__device__ __forceinline__ void k1_item(const K1Args& a, double2* S, int item, int next, unsigned& phase,
                                        unsigned occm) {
  constexpr int E = QMC_ROW_E;
  constexpr int NT = L2 / E;
  const int tid = threadIdx.x;
  const int L1 = a.L1;
  const int f1 = item % L1, p = item / L1;
#ifndef QMC_DIAG_NO_SCATTER
  const int nch = a.CH > 0 ? 0 : a.nch;
#else  // diagnostic: no scatter (the row holds stale data; timing bound of the rest)
  const int nch = 0;
#endif
  const double2* ap = a.asort + int64_t(p) * a.S1;
  const double2* tp = a.twj + int64_t(f1) * a.S1;
  QMC_TS(0);
  if (a.CH > 0) {  // staged mode: this item's chunk was copied during the previous item
    const K1Stage<L2> sg(S, a.CH, a.L1);
    mbar_wait(sg.bar, phase);
    phase ^= 1u;
    __syncthreads();  // every use of S by the previous item is done
    const int n = __ldg(&a.k1c[1]), nreg = __ldg(&a.k1c[2]);
    double2 acc = make_double2(0.0, 0.0);
    for (int i = tid; i < nreg; i += NT) {
      const int cd = sg.stE[i];
      const double2 pr = cmul(sg.stA[i], sg.stW[i]);
      acc = (cd & kK1First) ? pr : cadd(acc, pr);
      QMC_CHECK_IDX(i, a.CH);
      QMC_CHECK_IDX(padE<E>(cd & 0x3fff), k1_row_slots(L2, E));
      S[padE<E>(cd & 0x3fff)] = acc;
    }
    if (n > nreg) {  // fix-up: later pieces of split buckets, in order
      __syncthreads();
      for (int r = nreg + tid; r < n; r += NT) {
        const int rc = sg.stE[r];
        QMC_CHECK_IDX(padE<E>(L2 + 1 + ((rc >> 14) & 63) + (rc >> 20)), k1_row_slots(L2, E) + 1);
        const int e2 = rc & 0x3fff, o0 = (rc >> 14) & 63, cnt = rc >> 20;
        double2 t = S[padE<E>(e2)];
        for (int k = 0; k < cnt; ++k) t = cadd(t, S[padE<E>(L2 + 1 + o0 + k)]);
        S[padE<E>(e2)] = t;
      }
    }
    __syncthreads();  // staging consumed
    if (tid == 0 && next >= 0) k1_issue<L2>(a, sg, next);  // overlaps this item's FFTs
  }
  // the item's scatter twiddles TWs[e1·kTwRep + r] = ω_{L1}^{(e1 f1) mod L1},
  // replica r read by the lanes l ≡ r (mod 8): a quarter-warp's 16-byte loads
  // fall in distinct bank groups whatever the e1 (the previous item's reads
  // ended at its row barrier)
  // (from the constant tables: shared memory only, no global latency before
  // the scatter's barrier)
  const double2* T1s = S + k1_aux_base<L2>() + kK1Aux;
  double2* TWs = const_cast<double2*>(T1s) + L1;
  if (nch > 0 && a.bal)
    for (int i = tid; i < L1 * kTwRep; i += NT) TWs[i] = T1s[((i / kTwRep) * f1) % L1];
  // the item's register twiddles T16[q] = ω_{16 L1}^{x} = Tlo[x mod 16]·
  // ω_{L1}^{x div 16}, x = (q f1) mod 16 L1, read as broadcasts after the row
  // barrier; two buffers by item parity (the previous item may still read
  // its own; the one before ended at the previous row barrier)
  const double2* T16 = S + k1_aux_base<L2>() + 16 * ((item / int(gridDim.x)) & 1);
  for (int q = tid; q < 16; q += NT) {  // NT >= 2
    const int x = (q * f1) % (16 * L1);
    const_cast<double2*>(T16)[q] = cmul(S[k1_aux_base<L2>() + 32 + (x & 15)], T1s[x >> 4]);
  }
  for (int c = 0; c < nch; ++c) {
    const int q0 = __ldg(&a.k1c[c]), n = __ldg(&a.k1c[c + 1]) - q0;
    // every use of S by the previous item (or the previous chunk's fix-ups)
    // is done before this chunk's stores
    __syncthreads();
    // scatter a' = P a fused with the first DFT dimension:
    //   T'[f1, e2] = Σ_{j: e_j ≡ e2 (mod L2)} a_j ω_{L1}^{(e1_j·f1) mod L1}
    // (the bucket's common factor ω_L^{e2 f1} is applied to the row below)
    // (S holds the previous item's data elsewhere: only nonempty buckets are
    // read back, by the occupancy mask)
    if (a.bal) {
      // balanced order: the thread's slots tid, tid + NT, ... hold its
      // bucket pieces one after the other, in j order; the running sum is
      // stored after every entry (the last store of a piece is its total)
      const int nreg = __ldg(&a.k1c[nch + 1 + c]);
      double2 acc = make_double2(0.0, 0.0);
      const double2* tws = TWs + (tid & (kTwRep - 1));
      int i0 = q0 + tid;
      // Slots go in groups of U rounds: every load of a group (codes, a, then
      // the twiddles the codes select) is issued before the group's first
      // store to S — the compiler cannot reorder the shared-memory loads
      // across those stores itself (same base pointer), which serialised the
      // slots' latency chains
      constexpr int U = L2 >= 8192 ? QMC_K1_UNROLL_BIG : QMC_K1_UNROLL;
      if (a.SRn > 0) {  // the first SRn slots (one chunk: q0 = 0) were staged during the previous item
        const K1Hyb<L2> hb(S, L1, a.SRn);
        mbar_wait(hb.bar, phase);
        phase ^= 1u;
        int i = tid;
        for (; i + (U - 1) * NT < a.SRn; i += U * NT) {
          int cd[U];
          double2 av[U], tw[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            cd[u] = hb.stE[i + u * NT];
            av[u] = hb.stA[i + u * NT];
          }
#pragma unroll
          for (int u = 0; u < U; ++u) tw[u] = tws[((cd[u] >> kK1E1Shift) & 511) * kTwRep];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double2 pr = cmul(av[u], tw[u]);
            acc = (cd[u] & kK1First) ? pr : cadd(acc, pr);
            QMC_CHECK_IDX(padE<E>(cd[u] & 0x3fff), k1_row_slots(L2, E));
            S[padE<E>(cd[u] & 0x3fff)] = acc;
          }
        }
        for (; i < a.SRn; i += NT) {
          const int cd = hb.stE[i];
          const double2 pr = cmul(hb.stA[i], tws[((cd >> kK1E1Shift) & 511) * kTwRep]);
          acc = (cd & kK1First) ? pr : cadd(acc, pr);
          QMC_CHECK_IDX(padE<E>(cd & 0x3fff), k1_row_slots(L2, E));
          S[padE<E>(cd & 0x3fff)] = acc;
        }
        i0 = a.SRn + tid;
      }
      {
        int i = i0;
        for (; i + (U - 1) * NT < q0 + nreg; i += U * NT) {
          int cd[U];
          double2 av[U], tw[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            cd[u] = __ldg(&a.e2q[i + u * NT]);
            av[u] = __ldg(&ap[i + u * NT]);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) tw[u] = tws[((cd[u] >> kK1E1Shift) & 511) * kTwRep];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double2 pr = cmul(av[u], tw[u]);
            acc = (cd[u] & kK1First) ? pr : cadd(acc, pr);
            QMC_CHECK_IDX(i + u * NT, a.S1);
            QMC_CHECK_IDX(padE<E>(cd[u] & 0x3fff), k1_row_slots(L2, E));
            S[padE<E>(cd[u] & 0x3fff)] = acc;
          }
        }
        i0 = i;
      }
      for (int i = i0; i < q0 + nreg; i += NT) {
#if QMC_K1_PF > 0
        // the slot QMC_K1_PF rounds ahead into L1 (no register held)
        if (i + QMC_K1_PF * NT < q0 + nreg) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(ap + i + QMC_K1_PF * NT));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.e2q + i + QMC_K1_PF * NT));
        }
#endif
        const int cd = __ldg(&a.e2q[i]);
        const double2 pr = cmul(__ldg(&ap[i]), tws[((cd >> kK1E1Shift) & 511) * kTwRep]);
        acc = (cd & kK1First) ? pr : cadd(acc, pr);
        QMC_CHECK_IDX(i, a.S1);
        QMC_CHECK_IDX(padE<E>(cd & 0x3fff), k1_row_slots(L2, E));
        S[padE<E>(cd & 0x3fff)] = acc;
      }
      if (n > nreg) {  // fix-up: later pieces of split buckets, in order
        __syncthreads();
        for (int r = q0 + nreg + tid; r < q0 + n; r += NT) {
          const int rc = __ldg(&a.e2q[r]);
          QMC_CHECK_IDX(padE<E>(L2 + 1 + ((rc >> 14) & 63) + (rc >> 20)), k1_row_slots(L2, E) + 1);
          const int e2 = rc & 0x3fff, o0 = (rc >> 14) & 63, cnt = rc >> 20;
          double2 t = S[padE<E>(e2)];
          for (int k = 0; k < cnt; ++k) t = cadd(t, S[padE<E>(L2 + 1 + o0 + k)]);
          S[padE<E>(e2)] = t;
        }
      }
    } else {
      // bucket order (one chunk): the first entry of a bucket (nonzero size
      // field e2q >> 13) sums it in j order — up to the next head — and
      // stores T
      for (int i = tid; i < n; i += NT) {
        const int pk = __ldg(&a.e2q[q0 + i]);
        if ((pk >> 13) > 0) {
          double2 acc = cmul(__ldg(&ap[q0 + i]), __ldg(&tp[q0 + i]));
          for (int k = i + 1; k < n && (__ldg(&a.e2q[q0 + k]) >> 13) == 0; ++k)
            acc = cadd(acc, cmul(__ldg(&ap[q0 + k]), __ldg(&tp[q0 + k])));
          S[padE<E>(pk & 8191)] = acc;
        }
      }
    }
  }
  __syncthreads();  // the row T' is complete
  if (a.SRn > 0 && tid == 0 && next >= 0) k1_issue_hyb<L2>(a, K1Hyb<L2>(S, L1, a.SRn), next);  // overlaps the FFTs
  QMC_TS(1);
  double2 v[E];
  if (a.dense) {  // the first DFT dimension was done by k_dense_cols: load the row
    const double2* Tr = a.asort + int64_t(p) * a.S1 + int64_t(f1) * L2 + tid_fresh();
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = Tr[q * NT];
  } else {
    // nonempty buckets only (the rest of S is stale): bit q of occm says
    // whether bucket t + NT q has an entry (k_rows16 reads the bitmap once)
    const int t0 = tid_fresh();
#pragma unroll
    for (int q = 0; q < E; ++q)
      v[q] = (occm >> q) & 1u ? S[padE<E>(t0 + q * NT)] : make_double2(0.0, 0.0);
#if QMC_W_PF
    // the item's spectrum row into L1 ahead of dif_fwd's product (no register held)
#pragma unroll
    for (int q = 0; q < E; ++q)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(a.W + int64_t(f1) * L2 + t0 + q * NT));
#endif
    // the bucket's common factor ω_L^{e2 f1}, e2 = t + NT q: the register
    // part ω_L^{NT q f1} = ω_{16 L1}^{q f1} here, the thread part below
#pragma unroll
    for (int q = 1; q < E; ++q) v[q] = cmul(v[q], T16[q]);
  }
  // b = ω_L^{t·f1}: the thread's part of the four-step twiddle ω_L^{e2·f1}
  // (e2 = t + NT q), folded into the first row-FFT stage (k_dense_cols*
  // applied the rest to dense rows, the loop above to scattered ones)
  const int t0 = tid_fresh();
  double2 b;
  {
    const int x = t0 * f1;  // < NT·L1 = L/16
    b = cmul(__ldg(&a.tw1[x >> a.lg2L2]), __ldg(&a.twL[x & (L2 - 1)]));
  }
  // forward row FFT, then × the spectrum row (stored in this register order:
  // W[f1][r·NT + t]), half of it loaded during the last exchange
  double2 dc;
  dif_fwd<L2>(v, S, a.tw2, b, a.W + int64_t(f1) * L2 + tid_fresh(), &dc);
  QMC_TS(2);
  if (f1 == 0 && tid == 0) {  // DC term (register 0 of thread 0) = Σ_j a_j, the row-0 sums
    const int64_t k1 = 2 * (a.pair0 + p);
    a.colsum[k1] = dc.x;
    if (k1 + 1 < a.t) a.colsum[k1 + 1] = dc.y;
  }
  QMC_TS(3);
  dif_inv<L2>(v, S, a.tw2, b);
  // the rest of conj(ω_L^{e2 f1}) (the column pass's twiddle): conj(ω_{16 L1}^{q f1})
  {
    static_assert(E == 16, "K1's row FFT holds 16 points per thread");
#pragma unroll
    for (int q = 1; q < E; ++q) v[q] = cmulc(v[q], T16[q]);
  }
  QMC_TS(4);
  // U[p] in column blocks of kUB: [e2 / kUB][f1][e2 % kUB], so that K2 reads
  // whole sectors of kUB·16 bytes per f1; evict-first stores (U exceeds L2
  // on the large configs: the plan's tables and the batch's a stay resident)
  double2* Up = a.U + int64_t(p) * a.L + int64_t(f1) * kUB;
  QMC_CHECK_IDX(p, a.np);
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int e2 = tid + q * NT;
    QMC_CHECK_IDX(int64_t(e2 / kUB) * (L1 * kUB) + (e2 % kUB) + int64_t(f1) * kUB, a.L);
#ifndef QMC_U_PLAIN_STORES
    stcs2(reinterpret_cast<double*>(Up + int64_t(e2 / kUB) * (L1 * kUB) + (e2 % kUB)), v[q]);
#else
    Up[int64_t(e2 / kUB) * (L1 * kUB) + (e2 % kUB)] = v[q];
#endif
  }
  QMC_TS(5);
}

template <int L2>
__global__ void __launch_bounds__(L2 / QMC_ROW_E, (L2 / QMC_ROW_E >= 512 ? QMC_ROWS_MINB512 : QMC_ROWS_MINB))
    k_rows16(K1Args a) {
  extern __shared__ double2 smem[];
  const int nitems = a.L1 * a.np;
  unsigned phase = 0;
  if (a.CH > 0) {
    const K1Stage<L2> sg(smem, a.CH, a.L1);
    if (threadIdx.x == 0) mbar_init(sg.bar, 1);
    __syncthreads();
    if (threadIdx.x == 0 && int(blockIdx.x) < nitems) k1_issue<L2>(a, sg, blockIdx.x);
  } else if (a.SRn > 0) {
    const K1Hyb<L2> hb(smem, a.L1, a.SRn);
    if (threadIdx.x == 0) mbar_init(hb.bar, 1);
    __syncthreads();
    if (threadIdx.x == 0 && int(blockIdx.x) < nitems) k1_issue_hyb<L2>(a, hb, blockIdx.x);
  }
  // the constant twiddle tables after the row (rows_smem): Tlo, T1s
  {
    double2* aux = smem + k1_aux_base<L2>();
    for (int i = threadIdx.x; i < 16 + a.L1; i += blockDim.x)
      aux[32 + i] = i < 16 ? __ldg(&a.tw16[i]) : __ldg(&a.tw1[i - 16]);
    __syncthreads();
  }
  // the thread's nonempty buckets e2 = t + NT q (a plan constant): bit q
  unsigned occm = 0;
  if (!a.dense) {
    constexpr int NT = L2 / QMC_ROW_E;
#pragma unroll
    for (int q = 0; q < QMC_ROW_E; ++q) {
      const int e2 = int(threadIdx.x) + q * NT;
      occm |= ((__ldg(&a.occ[e2 >> 5]) >> (e2 & 31)) & 1u) << q;
    }
  }
  for (int item = blockIdx.x; item < nitems; item += gridDim.x)
    k1_item<L2>(a, smem, item, item + int(gridDim.x) < nitems ? item + int(gridDim.x) : -1, phase, occm);
}

// ---------------------------------------------------------------- one-row plans
// L1 = 1 (L = L2 <= 8192, e.g. config 1): the whole path of one column pair
// in one CTA, one launch per call — the pair's two columns of A into shared
// memory, per bucket e2 = t + NT q the sum of its a_j (f1 = 0: no twiddles),
// forward row FFT, ×W, inverse row FFT, then reordered row i = e2 written to
// conventional row n = P[(m - i) mod m] and row 0 =
// φ(0) Σ_j a_j, with the column's fused mean (the CTA
// owns the whole column pair: no cross-CTA reduction).
constexpr int kSmallMaxS = 2048;  // A's two columns, the bucket lists in shared memory
// the row, the pair's two columns of A, the columns in bucket order, the bucket starts
inline size_t small_smem(int64_t L2, int64_t s) {
  return size_t(k1_row_slots(L2, 16)) * 16 + size_t(s) * 20 + size_t(L2 + 4) * 4 + 32 +
         (L2 == 256 ? size_t(L2) * 20 : 0);  // rows of 256: the spectrum row and the row map too
}

// epilogue kinds (compile time) of the column passes: LIN writes c + X (c = 0
// unless AFFINE) and sums it per column; EXP writes X and sums exp(X) per
// column; ROWSUM writes X and row sums; NONE (one-row kernel) writes X only
enum { EPK_NONE = -1, EPK_LIN = 0, EPK_EXP = 1, EPK_ROWSUM = 2 };

struct SmallArgs {
  const double* __restrict__ A;
  int64_t lda, t;
  const int32_t* __restrict__ bstart;  // [L2+1]
  const int4* __restrict__ bent;       // [s] bucket order {j, e_j, e2, ...}
  int64_t s, m, N;
  const double2* __restrict__ tw2;
  const double2* __restrict__ W;
  const int32_t* __restrict__ P;
  const double* __restrict__ scal;     // [0] = φ(0)
  double* __restrict__ X;
  int64_t ldx;
  double fparam;
  double* __restrict__ out;
};

// threads of the one-row kernel: rows of 256 (NT = 16) take 128 threads for
// the loads and bucket sums (the row FFT of that length synchronises only
// within its half-warp, so the other threads may leave after the sums)
template <int L2>
__host__ __device__ constexpr int small_threads() { return L2 == 256 ? 128 : L2 / 16; }

template <int L2, int EP>
__global__ void __launch_bounds__(small_threads<L2>()) k_small(SmallArgs a) {
  constexpr int NT = L2 / 16, BT = small_threads<L2>();
  extern __shared__ double2 smem[];
  double2* S = smem;
  double* colA = reinterpret_cast<double*>(smem + k1_row_slots(L2, 16));  // [2][s]
  int* js = reinterpret_cast<int*>(colA + 2 * a.s);                        // [s] columns, bucket order
  int* bs = js + a.s;                                                       // [L2 + 1] bucket starts
  const int p = blockIdx.x, t = threadIdx.x;
  const int64_t k1 = 2 * int64_t(p), k2 = k1 + 1;
  const bool has2 = k2 < a.t;
  const double* a1 = a.A + k1 * a.lda;
  const double* a2 = a.A + (has2 ? k2 : k1) * a.lda;
#pragma unroll 8
  for (int j = t; j < int(a.s); j += BT) {  // independent loads, many in flight
    colA[j] = __ldg(&a1[j]);
    colA[a.s + j] = has2 ? __ldg(&a2[j]) : 0.0;
    js[j] = __ldg(&a.bent[j]).x;
  }
#pragma unroll 8
  for (int i = t; i <= L2; i += BT) bs[i] = __ldg(&a.bstart[i]);
  // rows of 256: the spare threads also bring the spectrum row and the row map
  double2* Ws = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(bs + L2 + 1) + 15) & ~uintptr_t(15));  // [L2]
  int* Ps = reinterpret_cast<int*>(Ws + L2);                        // [L2]: P[(m - i) mod m]
  if constexpr (BT > NT) {
    for (int i = t; i < L2; i += BT) {
      Ws[i] = __ldg(&a.W[i]);
      Ps[i] = i < a.m ? __ldg(&a.P[i == 0 ? 0 : a.m - i]) : -1;
    }
  }
  __syncthreads();
  for (int e2 = t; e2 < L2; e2 += BT) {  // bucket e2's entries in j order -> row slot
    double2 acc = make_double2(0.0, 0.0);
    for (int i = bs[e2], i1 = bs[e2 + 1]; i < i1; ++i) {
      const int j = js[i];
      QMC_CHECK_IDX(j, a.s);
      acc.x += colA[j];
      acc.y += colA[a.s + j];
    }
    S[padE<16>(e2)] = acc;
  }
  __syncthreads();
  if (BT > NT && t >= NT) return;  // (rows of 256: no CTA-wide barrier follows)
  double2 v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = S[padE<16>(t + NT * q)];
  const double2 one = make_double2(1.0, 0.0);
  dif_fwd<L2>(v, S, a.tw2, one);
  const double2 dc = v[0];  // thread 0: Σ_j a_j (the row-0 sums)
  if constexpr (BT > NT) {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = cmul(v[q], Ws[t + q * NT]);
  } else {
    const double2* Wr = a.W + t;
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = cmul(v[q], __ldg(&Wr[q * NT]));
  }
  dif_inv<L2>(v, S, a.tw2, one);
  double2 acc = make_double2(0.0, 0.0);
  double* xk = a.X ? a.X + k1 : nullptr;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int64_t i = t + int64_t(NT) * q;  // reordered row (i >= m: zero padding)
    if (i < a.m) {
      const int64_t n = BT > NT ? int64_t(Ps[i]) : int64_t(__ldg(&a.P[i == 0 ? 0 : a.m - i]));
      QMC_CHECK_IDX(n, a.N);
      double2 x = v[q];
      if (EP == EPK_LIN) {
        x.x += a.fparam;
        x.y += a.fparam;
      }
      if (xk) {
        xk[n * a.ldx] = x.x;
        if (has2) xk[n * a.ldx + 1] = x.y;
      }
      if (EP == EPK_LIN) {
        acc.x += x.x;
        acc.y += x.y;
      } else if (EP == EPK_EXP) {
        acc.x += exp(x.x);
        acc.y += exp(x.y);
      }
    }
  }
  if (t == 0) {  // row 0: X[0, k] = φ(0) Σ_j A[j, k]
    const double phi0 = __ldg(a.scal);
    double2 x = make_double2(phi0 * dc.x, phi0 * dc.y);
    if (EP == EPK_LIN) {
      x.x += a.fparam;
      x.y += a.fparam;
    }
    if (xk) {
      xk[0] = x.x;
      if (has2) xk[1] = x.y;
    }
    if (EP == EPK_LIN) {
      acc.x += x.x;
      acc.y += x.y;
    } else if (EP == EPK_EXP) {
      acc.x += exp(x.x);
      acc.y += exp(x.y);
    }
  }
  if (EP >= 0 && a.out) {  // the column means, a fixed-order reduction over the row's threads
    if constexpr (BT > NT) __syncwarp(0xffffu); else __syncthreads();
    double2* red = S;
    red[t] = acc;
    if constexpr (BT > NT) __syncwarp(0xffffu); else __syncthreads();
    if (t == 0) {
      double2 sum = red[0];
      for (int u = 1; u < NT; ++u) sum = cadd(sum, red[u]);
      a.out[k1] = sum.x / double(a.N);
      if (has2) a.out[k2] = sum.y / double(a.N);
    }
  }
}

// ---------------------------------------------------------------- Korobov p-set
// The union of all Korobov lattices: block g = 1..K-1 is
// the rank-1 lattice with z_j = g^j mod K (j = 0..s-1) without its row 0.
// In the reordered indexing every block is Z·P_g with the SAME circulant Z
// (one plan: one ζ, one spectrum W, one P/L), only the column map changes:
// e_{g,j} = L[g^j] = j·ℓ_g mod m, ℓ_g = L[g] (the paper's c_{g,j} - 1 =
// (j-1)(g-1) mod (K-1) with 1-based j and g = β^{g-1}).  One CTA per (pair,
// block); bucket e receives the j with j·ℓ ≡ e (mod m): with d = gcd(ℓ, m)
// and u = (ℓ/d)^{-1} mod m/d these are j ≡ (e/d)·u (mod m/d), summed in
// increasing j (deterministic).  Conventional row n of block g is p-set row
// (g-1)(K-1) + n-1 (reading R24).  One-row plans only (L1 = 1).
__device__ __forceinline__ int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t r = a % b;
    a = b;
    b = r;
  }
  return a;
}
// x^{-1} mod mm for gcd(x, mm) = 1, mm >= 1 (extended Euclid)
__device__ __forceinline__ int64_t modinv64(int64_t x, int64_t mm) {
  if (mm == 1) return 0;
  int64_t r0 = mm, r1 = x % mm, s0 = 0, s1 = 1;
  while (r1) {
    const int64_t qq = r0 / r1;
    int64_t tmp = r0 - qq * r1;
    r0 = r1;
    r1 = tmp;
    tmp = s0 - qq * s1;
    s0 = s1;
    s1 = tmp;
  }
  return ((s0 % mm) + mm) % mm;
}

template <int L2>
__global__ void __launch_bounds__(L2 / 16) k_pset(SmallArgs a, const int32_t* __restrict__ Ltab) {
  constexpr int NT = L2 / 16;
  extern __shared__ double2 smem[];
  double2* S = smem;
  double* colA = reinterpret_cast<double*>(smem + k1_row_slots(L2, 16));  // [2][s]
  const int p = blockIdx.x, g = blockIdx.y + 1, t = threadIdx.x;
  const int64_t m = a.m;
  const int64_t k1 = 2 * int64_t(p), k2 = k1 + 1;
  const bool has2 = k2 < a.t;
  const double* a1 = a.A + k1 * a.lda;
  const double* a2 = a.A + (has2 ? k2 : k1) * a.lda;
#pragma unroll 8
  for (int j = t; j < int(a.s); j += NT) {
    colA[j] = __ldg(&a1[j]);
    colA[a.s + j] = has2 ? __ldg(&a2[j]) : 0.0;
  }
  const int64_t ell = __ldg(&Ltab[g]);      // ℓ_g = L[g]
  const int64_t d = ell ? gcd64(ell, m) : m;
  const int64_t mm = m / d;
  const int64_t u = modinv64(ell / d, mm);
  __syncthreads();
  double2 v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int64_t e2 = t + int64_t(NT) * q;
    double2 acc = make_double2(0.0, 0.0);
    if (e2 < m && e2 % d == 0) {
      for (int64_t j = ((e2 / d) * u) % mm; j < a.s; j += mm) {
        acc.x += colA[j];
        acc.y += colA[a.s + j];
      }
    }
    v[q] = acc;
  }
  const double2 one = make_double2(1.0, 0.0);
  dif_fwd<L2>(v, S, a.tw2, one);
  {
    const double2* Wr = a.W + t;
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = cmul(v[q], __ldg(&Wr[q * NT]));
  }
  dif_inv<L2>(v, S, a.tw2, one);
  double* xk = a.X + k1 + int64_t(g - 1) * m * a.ldx;  // block g: rows (g-1)(K-1) + n-1
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int64_t i = t + int64_t(NT) * q;
    if (i < m) {
      const int64_t n = __ldg(&a.P[i == 0 ? 0 : m - i]);  // conventional row n in 1..K-1
      QMC_CHECK_IDX(n - 1, m);
      xk[(n - 1) * a.ldx] = v[q].x;
      if (has2) xk[(n - 1) * a.ldx + 1] = v[q].y;
    }
  }
}

template <int L2>
static int launch_pset(const qmc_plan* pl, const SmallArgs& sa, int64_t npairs, cudaStream_t st) {
  const size_t smem = size_t(k1_row_slots(L2, 16)) * 16 + size_t(2 * sa.s) * 8;
  auto kern = k_pset<L2>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(size_t(k1_row_slots(L2, 16)) * 16 + size_t(2 * kSmallMaxS) * 8));
    attr = true;
  }
  kern<<<dim3(unsigned(npairs), unsigned(pl->m)), L2 / 16, smem, st>>>(sa, pl->d_L);
  QMC_LAUNCHED();
  return QMC_OK;
}

// ---------------------------------------------------------------- K2
// Column pass, un-permutation and epilogue; X is row-major (X[n·ldx + k]).
//
// Tile: CB columns e2 (blockIdx.x) × PG pairs (blockIdx.y) of the batch,
// lane = pair within the group fastest, so the PG pairs of one output row
// (2·PG consecutive doubles of X) are written by PG adjacent lanes.
// L1 = R·M:
//   R = 1 — one item (p, c) per thread: the L1 values u[f1] = U[p][f1][e2]
//           times conj(ω_L^{e2 f1}), the L1-point inverse DFT in registers;
//   R > 1 — stage A, item (p, c, r): M-point inverse DFT over f1 = r + R·mm,
//           times ω_{L1}^{r k2} → shared memory; stage B, item (p, c, k2):
//           R-point inverse DFT over r → outputs e1 = k2 + M·k1.
// Output i = L2·e1 + e2 < m is reordered row i, conventional row
// n = P[(m - i) mod m] (i = 0 → n = 1).
//
// Epilogue EP (compile time): LIN writes c + X (c = 0 unless AFFINE) and
// sums it per column; EXP writes X and sums exp(X) per column; ROWSUM writes
// X and the row sums over the pair group (warp transpose through shared
// memory, then a fixed-order sum).

struct EpiArgs {
  double fparam;     // c of AFFINE (0 otherwise)
  double* X;         // may be NULL (means only)
  int64_t ldx;
  int xvec;          // X + n·ldx + k 16-byte aligned for even k
  int64_t t;
  double* rowpart;   // ROWSUM: partial row sums [pair group of the call][N]
  int64_t N;
};

// one output value v of columns (k, k + 1), row n (ok: a real row and pair)
template <int EP>
__device__ __forceinline__ void emit(const EpiArgs& E, double2 v, int64_t n, bool ok, bool has2, double* xk,
                                     double2& acc, double& rsum) {
  if (EP == EPK_LIN) {
    v.x += E.fparam;
    v.y += E.fparam;
  }
  if (!has2) v.y = 0.0;
  if (ok && xk) {
    QMC_CHECK_IDX(n, E.N);
    double* xp = xk + n * E.ldx;
    if (E.xvec && has2) {
      QMC_XST2(xp, v);
    } else {
      QMC_XST(xp, v.x);
      if (has2) QMC_XST(xp + 1, v.y);
    }
  }
  if (EP == EPK_LIN) {
    if (ok) {
      acc.x += v.x;
      acc.y += v.y;
    }
  } else if (EP == EPK_EXP) {
    if (ok) {
      acc.x += exp(v.x);
      if (has2) acc.y += exp(v.y);
    }
  } else {
    rsum = ok ? v.x + v.y : 0.0;
  }
}

// Fast path (every pair of the tile present, t even, X 16-byte aligned with
// even ldx, every output row real): no predicates
template <int EP>
__device__ __forceinline__ void emit_fast(const EpiArgs& E, double2 v, int n, double* xk, double2& acc,
                                          double& rsum) {
  if (EP == EPK_LIN) {
    v.x += E.fparam;
    v.y += E.fparam;
  }
  QMC_CHECK_IDX(n, E.N);
  if (xk) QMC_XST2(xk + int64_t(n) * E.ldx, v);
  if (EP == EPK_LIN) {
    acc.x += v.x;
    acc.y += v.y;
  } else if (EP == EPK_EXP) {
    acc.x += exp(v.x);
    acc.y += exp(v.y);
  } else {
    rsum = v.x + v.y;
  }
}

// ROWSUM, 16 rows × 16 lanes (PG = 16): butterfly reduce-scatter over the
// half-warp (xor 8, 4, 2, 1; fixed order) — on return r[0] of lane l is the
// sum over the 16 lanes of row (l & 15).
__device__ __forceinline__ double rowsum_butterfly16(double (&r)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 8; h > 0; h >>= 1) {
    const bool up = lane & h;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double send = up ? r[k] : r[k + h];
      const double keep = up ? r[k + h] : r[k];
      r[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return r[0];
}

// ROWSUM: the NR row values of every lane of the warp → per (lane group of
// PG pairs, row slot) sums over the group's lanes in lane order → rowpart[n].
// Tw: this warp's NR·33 doubles of shared memory, Tn: NR·8 ints.
template <int NR>
__device__ __forceinline__ void rowsum_flush(const double (&r)[NR], const int (&nrow)[NR], int PG, double* Tw,
                                             int* Tn, double* rowpart) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    Tw[k * 33 + lane] = r[k];
    if (lane % PG == 0) Tn[k * 8 + lane / PG] = nrow[k];
  }
  __syncwarp();
  const int G = 32 / PG;
  for (int rr = lane; rr < G * NR; rr += 32) {
    const int q = rr / NR, k = rr - q * NR;
    const double* src = Tw + k * 33 + q * PG;
    double sum = 0.0;
    for (int p = 0; p < PG; ++p) sum += src[p];
    const int n = Tn[k * 8 + q];
    if (n >= 0) rowpart[n] = sum;
  }
  __syncwarp();
}

// ω_L^x for 0 <= x < L from ω_{L1} (tw1) and ω_L^k, k < L2 (twL)
__device__ __forceinline__ double2 omegaL(int64_t x, int lg2L2, int L2, const double2* __restrict__ tw1,
                                          const double2* __restrict__ twL) {
  return cmul(__ldg(&tw1[x >> lg2L2]), __ldg(&twL[x & (L2 - 1)]));
}

template <int R, int M, int EP, bool FAST>
__global__ void __launch_bounds__(kColThreads, 2)
    k_cols_x(const double2* __restrict__ U, int64_t L, int L2, int lg2L2, int64_t m, int np, int PG,
             const int32_t* __restrict__ P, const double* __restrict__ colsum, const double* __restrict__ scal,
             const double2* __restrict__ tw1, const double2* __restrict__ twL, int64_t pair0, EpiArgs E,
             double* __restrict__ part, int part_stride) {
  constexpr int L1 = R * M;
  constexpr int LP = L1 | 1;  // odd pitch (in 16-B units): conflict-free stage exchange
  constexpr int NR = R == 1 ? L1 : R;  // output rows per item
  extern __shared__ double2 sm[];
  __shared__ double rsT[EP == EPK_ROWSUM ? kColThreads / 32 : 1][EP == EPK_ROWSUM ? NR * 33 : 1];
  __shared__ int rsN[EP == EPK_ROWSUM ? kColThreads / 32 : 1][EP == EPK_ROWSUM ? NR * 8 : 1];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int CB = (R == 1 ? kColThreads : 32) / PG;
  const int pg0 = blockIdx.y * PG;
  const int p = tid % PG;
  const int pair = pg0 + p;
  const bool okp = pair < np;
  const double2* Up = U + int64_t(okp ? pair : 0) * L;
  const int64_t k = 2 * (pair0 + pair);  // this lane's columns k, k + 1
  const bool has2 = k + 1 < E.t;
  double* xk = E.X ? E.X + k : nullptr;
  double* rowpart = EP == EPK_ROWSUM ? E.rowpart + (pair0 / PG + blockIdx.y) * E.N : nullptr;
  double2 acc = make_double2(0.0, 0.0);
  // column groups bx = blockIdx.x, + gridDim.x, ... (the CTA's column sums
  // accumulate over all of them: one partial slot per CTA)
  const int nbxT = (L2 + CB - 1) / CB;
  for (int bx = blockIdx.x; bx < nbxT; bx += gridDim.x) {
  // row 0: X[0, k] = φ(0) Σ_j A[j, k]
  if (bx == 0 && warp == 0) {
    const bool okrow = tid < PG;
    double2 v0 = make_double2(0.0, 0.0);
    if (okp && okrow) {
      const double phi0 = __ldg(scal);
      v0.x = phi0 * colsum[k];
      v0.y = has2 ? phi0 * colsum[k + 1] : 0.0;
    }
    double r0[1];
    int n0[1] = {okrow ? 0 : -1};
    emit<EP>(E, v0, 0, okp && okrow, has2, xk, acc, r0[0]);
    if (EP == EPK_ROWSUM) rowsum_flush<1>(r0, n0, PG, &rsT[0][0], &rsN[0][0], rowpart);
  }
  if constexpr (R == 1) {
    const int c = tid / PG;
    const int e2 = bx * CB + c;
    const bool okc = e2 < L2;
    // rows first: every load of the tile is issued before the first store
    int nrow[L1];
#pragma unroll
    for (int e1 = 0; e1 < L1; ++e1) {
      const int64_t i = int64_t(L2) * e1 + e2;
      nrow[e1] = (okc && i < m) ? __ldg(&P[i == 0 ? 0 : m - i]) : -1;
    }
    double2 v[L1];
    const double2* ub = Up + int64_t(e2 >> 2) * (L1 * kUB) + (e2 & 3);
    if (okp && okc) {
#pragma unroll
      for (int f1 = 0; f1 < L1; ++f1) v[f1] = __ldg(&ub[f1 * kUB]);
    } else {
#pragma unroll
      for (int f1 = 0; f1 < L1; ++f1) v[f1] = make_double2(0.0, 0.0);
    }
    // (the twiddle conj(ω_L^{e2 f1}) was applied by K1)
    // this CTA's U blocks (PG pairs × CB/kUB column blocks of L1·kUB complex,
    // read only here) are dead: drop them from L2 without write-back
    if (CB % kUB == 0) {
      __syncthreads();
      const int lines = L1 * kUB * 16 / 128;  // per block (L1·kUB·16 bytes)
      const int nb = CB / kUB;
      for (int i = tid; i < PG * nb * lines; i += kColThreads) {
        const int pp = i / (nb * lines), rest = i % (nb * lines);
        const int b = rest / lines, l = rest % lines;
        if (pg0 + pp < np && (bx * CB) / kUB + b < L2 / kUB && (L1 * kUB * 16) % 128 == 0)
          discard_l2(reinterpret_cast<const char*>(U + int64_t(pg0 + pp) * L +
                                                   int64_t((bx * CB) / kUB + b) * (L1 * kUB)) + 128 * l);
      }
    }
    reg_dft<L1, +1>(v, tw1);
    double r[L1];
    if constexpr (FAST) {
#pragma unroll
      for (int e1 = 0; e1 < L1; ++e1) emit_fast<EP>(E, v[e1], nrow[e1], xk, acc, r[e1]);
      if constexpr (EP == EPK_ROWSUM && L1 == 16) {
        if (PG == 16) {
          const double sum = rowsum_butterfly16(r);
          const int e1 = tid & 15;
          const int64_t i = int64_t(L2) * e1 + e2;
          rowpart[__ldg(&P[i == 0 ? 0 : m - i])] = sum;
        } else {
          rowsum_flush<L1>(r, nrow, PG, &rsT[warp][0], &rsN[warp][0], rowpart);
        }
      } else if constexpr (EP == EPK_ROWSUM) {
        rowsum_flush<L1>(r, nrow, PG, &rsT[warp][0], &rsN[warp][0], rowpart);
      }
    } else {
#pragma unroll
      for (int e1 = 0; e1 < L1; ++e1) emit<EP>(E, v[e1], nrow[e1], okp && nrow[e1] >= 0, has2, xk, acc, r[e1]);
      if (EP == EPK_ROWSUM) rowsum_flush<L1>(r, nrow, PG, &rsT[warp][0], &rsN[warp][0], rowpart);
    }
  } else {
    double2* T = sm;  // [(p + PG·c)·LP + r·M + k2]
    const int nA = 32 * R;  // = PG·CB·R items
    for (int it = tid; it < nA; it += kColThreads) {
      const int rest = it / PG;
      const int r = rest % R, c = rest / R;
      const int e2 = bx * CB + c;
      const bool ok = okp && e2 < L2;
      double2 x[M];
      if (ok) {
        const double2* ub = Up + int64_t(e2 >> 2) * (L1 * kUB) + (e2 & 3);
#pragma unroll
        for (int mm = 0; mm < M; ++mm) x[mm] = __ldg(&ub[(r + R * mm) * kUB]);
      } else {
#pragma unroll
        for (int mm = 0; mm < M; ++mm) x[mm] = make_double2(0.0, 0.0);
      }
      reg_dft<M, +1>(x, tw1, L1 / M);
#pragma unroll
      for (int k2 = 1; k2 < M; ++k2)
        if (r) x[k2] = cmul(x[k2], twid<+1>(__ldg(&tw1[r * k2])));
      double2* Tp = T + (p + PG * c) * LP + r * M;
#pragma unroll
      for (int k2 = 0; k2 < M; ++k2) Tp[k2] = x[k2];
    }
    __syncthreads();
    const int nB = 32 * M;  // = PG·CB·M items (a multiple of 32: warp-uniform loop)
    for (int it = tid; it < nB; it += kColThreads) {
      const int rest = it / PG;
      const int k2 = rest % M, c = rest / M;
      const int e2 = bx * CB + c;
      const bool okc = e2 < L2;
      int nrow[R];
#pragma unroll
      for (int k1 = 0; k1 < R; ++k1) {
        const int64_t i = int64_t(L2) * (k2 + M * k1) + e2;
        nrow[k1] = (okc && i < m) ? __ldg(&P[i == 0 ? 0 : m - i]) : -1;
      }
      double2 z[R];
      const double2* Tp = T + (p + PG * c) * LP + k2;
#pragma unroll
      for (int r = 0; r < R; ++r) z[r] = Tp[r * M];
      reg_dft<R, +1>(z, tw1, L1 / R);
      double rr[R];
#pragma unroll
      for (int k1 = 0; k1 < R; ++k1) emit<EP>(E, z[k1], nrow[k1], okp && nrow[k1] >= 0, has2, xk, acc, rr[k1]);
      if (EP == EPK_ROWSUM) rowsum_flush<R>(rr, nrow, PG, &rsT[warp][0], &rsN[warp][0], rowpart);
    }
  }
  __syncthreads();  // shared tiles are reused by the next column group
  }
  // per-column partial sums of this CTA: lanes with equal p, then warps in order
  if (EP != EPK_ROWSUM) {
    for (int o = PG; o < 32; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    __shared__ double2 red[kColThreads / 32][16];
    const int l = tid & 31;
    if (l < PG) red[warp][l] = acc;
    __syncthreads();
    if (tid < PG && okp && part) {
      double2 sacc = red[0][tid];
      for (int ww = 1; ww < kColThreads / 32; ++ww) sacc = cadd(sacc, red[ww][tid]);
      double* dst = part + int64_t(blockIdx.x) * part_stride + 2 * pair;
      dst[0] = sacc.x;
      dst[1] = sacc.y;
    }
  }
}

// Persistent, software-pipelined K2 for the fast path (R = 1, PG = 16): tile =
// (16 columns e2, 16 pairs), its U blocks (16 pairs × 4 blocks × L1·kUB
// complex, contiguous per pair) and its output row indices staged in shared
// memory by cp.async one tile ahead, so the DRAM/L2 reads of the next tile
// overlap the DFTs and X stores of this one.  Same arithmetic and output as
// k_cols_x<1, L1, EP, true>.
#ifndef QMC_K2_STAGES
#define QMC_K2_STAGES 2
#endif
constexpr int kPipeStages = QMC_K2_STAGES;
#ifndef QMC_K2_CB
#define QMC_K2_CB 8
#endif
#ifndef QMC_K2_MINB
#define QMC_K2_MINB 1
#endif
template <int L1, int CB>
__host__ __device__ constexpr int pipe_pair_stride() { return (CB / kUB) * L1 * kUB + 1; }
template <int L1, int CB>
__host__ __device__ constexpr size_t cols_pipe_smem() {
  return size_t(kPipeStages) * 16 * pipe_pair_stride<L1, CB>() * 16 + size_t(kPipeStages) * L1 * CB * 4;
}

struct K2Args {
  const double2* __restrict__ U;
  int64_t L;
  int L2;
  int64_t m;
  int ntx, ngroups;                    // tiles: ntx column groups × ngroups pair groups
  const int32_t* __restrict__ P;
  const double* __restrict__ colsum;
  const double* __restrict__ scal;
  const double2* __restrict__ tw1;
  const double2* __restrict__ twL;
  int64_t pair0;
  EpiArgs E;
  double* __restrict__ part;
  int part_stride;
  const int32_t* __restrict__ k2n;     // plan.cu k_k2rows: output rows in U column-block order
};

// stage tile (16 pairs × CB columns = CB/kUB U column blocks) by bulk async
// copies, one thread: per pair one contiguous run of the tile's U blocks into
// dst (pair pitch PSTR), and the tile's run of the plan's row table k2n into
// nd ([block][e1][c], k2_nidx), completing on bar
template <int L1, int CB>
__device__ __forceinline__ void k2_issue(const K2Args& a, int tile, double2* dst, int* nd, uint64_t* bar) {
  constexpr int PG = 16, NB = CB / kUB, BLK = L1 * kUB;
  constexpr int PSTR = pipe_pair_stride<L1, CB>();
  constexpr unsigned UB = NB * BLK * 16, NB4 = L1 * CB * 4;
  const int bx = tile % a.ntx, g = tile / a.ntx;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer's reads before the async writes
  mbar_expect_tx(bar, PG * UB + NB4);
#pragma unroll
  for (int pp = 0; pp < PG; ++pp)
    bulk_g2s(dst + pp * PSTR, a.U + int64_t(g * PG + pp) * a.L + int64_t(bx) * (NB * BLK), UB, bar);
  bulk_g2s(nd, a.k2n + int64_t(bx) * (L1 * CB), NB4, bar);
}
// index of the output row of (e1, column c of the tile) in the staged k2n run
template <int L1>
__device__ __forceinline__ int k2_nidx(int e1, int c) {
  return (c / kUB) * (L1 * kUB) + e1 * kUB + (c % kUB);
}

// column pass + epilogue of one staged tile (16·CB threads, one column each)
template <int L1, int EP, int CB>
__device__ __forceinline__ void k2_tile(const K2Args& a, int tile, const double2* tileS, const int* nS,
                                        double2 (*red)[16]) {
  constexpr int PG = 16, NT = PG * CB, BLK = L1 * kUB;
  constexpr int PSTR = pipe_pair_stride<L1, CB>();  // odd (16-B units): conflict-free column reads
  const EpiArgs& E = a.E;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int p = tid % PG, c = tid / PG;
  const int bx = tile % a.ntx, g = tile / a.ntx;
  const int pair = g * PG + p;
  const int64_t k = 2 * (a.pair0 + pair);
  double* xk = E.X ? E.X + k : nullptr;
  double* rowpart = EP == EPK_ROWSUM ? E.rowpart + (a.pair0 / PG + g) * E.N : nullptr;
  double2 acc = make_double2(0.0, 0.0);
  if (bx == 0 && warp == 0) {  // row 0: X[0, k] = φ(0) Σ_j A[j, k]
    const bool okrow = tid < PG;
    const double phi0 = __ldg(a.scal);
    const double2 v0 = make_double2(phi0 * a.colsum[k], phi0 * a.colsum[k + 1]);
    double r0 = 0.0;
    emit<EP>(E, v0, 0, okrow, true, xk, acc, r0);
    if (EP == EPK_ROWSUM) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) r0 += __shfl_xor_sync(0xffffffffu, r0, o);
      if (tid == 0) rowpart[0] = r0;
    }
  }
  const double2* src = tileS + p * PSTR + (c / kUB) * BLK + (c % kUB);
  double2 v[L1];
#pragma unroll
  for (int f1 = 0; f1 < L1; ++f1) v[f1] = src[f1 * kUB];
  reg_dft<L1, +1>(v, a.tw1);  // (the twiddle conj(ω_L^{e2 f1}) was applied by K1)
  double r[L1];
#pragma unroll
  for (int e1 = 0; e1 < L1; ++e1) {
    const int n = nS[k2_nidx<L1>(e1, c)];  // -1: padding row (uniform over the 16 lanes of the row)
    if (n >= 0) {
      emit_fast<EP>(E, v[e1], n, xk, acc, r[e1]);
    } else {
      r[e1] = 0.0;
    }
  }
  if constexpr (EP == EPK_ROWSUM) {
    static_assert(EP != EPK_ROWSUM || L1 == 16, "row sums of the pipelined K2 need L1 = 16");
    const double sum = rowsum_butterfly16(r);
    const int n = nS[k2_nidx<L1>(tid & 15, c)];
    if (n >= 0) rowpart[n] = sum;
  } else {
    if (a.part) {  // per-column partial sums of this tile (lanes with equal p, then warps)
#pragma unroll
      for (int o = PG; o < 32; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if ((tid & 31) < PG) red[warp][tid & 31] = acc;
      __syncthreads();
      if (tid < PG) {
        double2 sacc = red[0][tid];
        for (int ww = 1; ww < NT / 32; ++ww) sacc = cadd(sacc, red[ww][tid]);
        double* dst = a.part + int64_t(bx) * a.part_stride + 2 * pair;
        dst[0] = sacc.x;
        dst[1] = sacc.y;
      }
    }
  }
}

template <int L1, int EP, int CB>
__global__ void __launch_bounds__(16 * CB, QMC_K2_MINB) k_cols_pipe(K2Args a) {
  constexpr int NT = 16 * CB;
  constexpr int STAGE = 16 * pipe_pair_stride<L1, CB>();
  extern __shared__ double2 sm[];
  int* nS = reinterpret_cast<int*>(sm + kPipeStages * STAGE);  // [stage][e1][c]
  __shared__ double2 red[NT / 32][16];
  __shared__ uint64_t bars[kPipeStages];  // stage complete (phase per use)
  const int ntiles = a.ntx * a.ngroups;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s0 = 0; s0 < kPipeStages; ++s0) mbar_init(&bars[s0], 1);
#pragma unroll
    for (int s0 = 0; s0 < kPipeStages - 1; ++s0) {
      const int tl = blockIdx.x + s0 * gridDim.x;
      if (tl < ntiles) k2_issue<L1, CB>(a, tl, sm + s0 * STAGE, nS + s0 * (L1 * CB), &bars[s0]);
    }
  }
  __syncthreads();  // the barriers are initialised before anyone waits on them
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kPipeStages;
    const int ahead = tile + (kPipeStages - 1) * gridDim.x;
    if (threadIdx.x == 0 && ahead < ntiles) {  // its buffer was freed by the previous tile's last barrier
      const int sa = (it + kPipeStages - 1) % kPipeStages;
      k2_issue<L1, CB>(a, ahead, sm + sa * STAGE, nS + sa * (L1 * CB), &bars[sa]);
    }
    mbar_wait(&bars[st], unsigned(it / kPipeStages) & 1u);
    __syncthreads();
    k2_tile<L1, EP, CB>(a, tile, sm + st * STAGE, nS + st * (L1 * CB), red);
    __syncthreads();  // stage st and red are reused
  }
}

// Persistent, software-pipelined two-stage K2 (L1 = R·M, R > 1; config 5:
// 96 = 6·16): tile = (PG pairs, one U column block of kUB = 4 columns e2),
// i.e. PG contiguous runs of L1·kUB complex, staged one tile ahead with its
// output row indices (the plan's k2n run) by bulk async copies (one thread,
// an mbarrier per stage).  Stage A, item (p, c, r): the M values
// f1 = r + R·mm times conj(ω_L^{e2 f1}), M-point inverse DFT, times
// ω_{L1}^{r k2}, written back in place (position r + R·k2).  Stage B, item
// (p, c, k2): R-point inverse DFT over r → rows e1 = k2 + M·k1, stored as
// PG-pair row chunks (16·PG bytes) of X.  Same arithmetic as k_cols_x<R, M>.
// Pairs per tile: 16 (512 threads, 256-byte row chunks of X, one CTA per SM)
// where L1 >= 80 and two stages of 16 pairs fit in shared memory — config 5's
// L1 = 96: K2 20.95 -> 19.41 ms against 8-pair tiles at two CTAs per SM —
// else 8 (256 threads).  QMC_P2PG forces one value (diagnostic).
template <int L1>
__host__ __device__ constexpr int p2pg() {
#ifdef QMC_P2PG
  return QMC_P2PG;
#else
  return (L1 >= 80 && 2 * (size_t(16) * (L1 * kUB + 1) * 16 + size_t(L1) * kUB * 4) <= 232448) ? 16 : 8;
#endif
}
template <int L1>
__host__ __device__ constexpr int p2thr() {
#ifdef QMC_P2THR
  return QMC_P2THR;  // diagnostic (a multiple of 32)
#else
  return 32 * p2pg<L1>();
#endif
}
template <int L1>
__host__ __device__ constexpr int pipe2_pair_stride() { return L1 * kUB + 1; }  // odd, 16-B units
template <int L1>
__host__ __device__ constexpr size_t cols_pipe2_smem() {
  return size_t(kPipeStages) * (size_t(p2pg<L1>()) * pipe2_pair_stride<L1>() * 16 + size_t(L1) * kUB * 4);
}

// stage tile `tile` into dst (pair pitch PSTR) and its output rows into nd
// by bulk async copies, one thread: PG contiguous U runs of L1·kUB complex
// and the tile's run of the plan's row table (k2n), completing on bar
template <int L1>
__device__ __forceinline__ void k2p2_issue(const K2Args& a, int tile, double2* dst, int* nd, uint64_t* bar) {
  constexpr int BLK = L1 * kUB, PSTR = pipe2_pair_stride<L1>();
  constexpr unsigned UB = BLK * 16, NB4 = L1 * kUB * 4;
  const int bx = tile % a.ntx, g = tile / a.ntx;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer's reads before the async writes
  constexpr int PG = p2pg<L1>();
  mbar_expect_tx(bar, PG * UB + NB4);
#pragma unroll
  for (int pp = 0; pp < PG; ++pp)
    bulk_g2s(dst + pp * PSTR, a.U + int64_t(g * PG + pp) * a.L + int64_t(bx) * BLK, UB, bar);
  bulk_g2s(nd, a.k2n + int64_t(bx) * (L1 * kUB), NB4, bar);
}

template <int R, int M, int EP, bool PAD>
__device__ __forceinline__ void k2p2_tile(const K2Args& a, int tile, double2* T, const int* nS, double2& acc,
                                          const double2* tw1) {
  constexpr int L1 = R * M, PSTR = pipe2_pair_stride<L1>(), PG = p2pg<L1>(), kP2Thr = p2thr<L1>();
  const EpiArgs& E = a.E;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int p = tid % PG;
  const int bx = tile % a.ntx, g = tile / a.ntx;
  const int pair = g * PG + p;
  const int64_t k = 2 * (a.pair0 + pair);
  double* xk = E.X ? E.X + k : nullptr;
  if (bx == 0 && warp == 0) {  // row 0: X[0, k] = φ(0) Σ_j A[j, k]
    const bool okrow = tid < PG;
    const double phi0 = __ldg(a.scal);
    const double2 v0 = make_double2(phi0 * a.colsum[k], phi0 * a.colsum[k + 1]);
    double r0 = 0.0;
    emit<EP>(E, v0, 0, okrow, true, xk, acc, r0);
  }
  // stage A: items (p, c, r), it = p + PG·(c + kUB·r)
  for (int it = tid; it < PG * kUB * R; it += kP2Thr) {
    const int c = (it / PG) % kUB, r = it / (PG * kUB);
    double2* Tp = T + p * PSTR + c;
    double2 x[M];
#pragma unroll
    for (int mm = 0; mm < M; ++mm) x[mm] = Tp[(r + R * mm) * kUB];
    reg_dft<M, +1>(x, tw1, L1 / M);  // (conj(ω_L^{e2 f1}) was applied by K1)
#pragma unroll
    for (int k2 = 1; k2 < M; ++k2)
      if (r) x[k2] = cmul(x[k2], twid<+1>(tw1[r * k2]));
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) Tp[(r + R * k2) * kUB] = x[k2];
  }
  __syncthreads();
  // stage B: items (p, c, k2), it = p + PG·(c + kUB·k2); a warp = PG pairs ×
  // 32/PG columns of one k2, so each output row gets one 16·PG-byte chunk
  for (int it = tid; it < PG * kUB * M; it += kP2Thr) {
    const int c = (it / PG) % kUB, k2 = it / (PG * kUB);
    const double2* Tp = T + p * PSTR + c;
    double2 z[R];
#pragma unroll
    for (int r = 0; r < R; ++r) z[r] = Tp[(r + R * k2) * kUB];
    reg_dft<R, +1>(z, tw1, L1 / R);
    double rr;
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) {
      const int n = nS[(k2 + M * k1) * kUB + c];  // -1: padding row (uniform over the 8 lanes of the row)
      if (!PAD || n >= 0) emit_fast<EP>(E, z[k1], n, xk, acc, rr);  // PAD: zero-padded length
    }
  }
}

// per-column partial sums of a CTA's run of tiles in pair group g (lanes with
// equal pair, then warps in order) -> part[blockIdx.x][pairs of g]; a CTA
// visits each pair group in one run of consecutive tiles (tile = blockIdx.x
// + k·gridDim.x, g = tile / ntx nondecreasing), so the slot row of every
// group it visits is written once and the rest stays zero
template <int PG, int kP2Thr>
__device__ __forceinline__ void k2p2_flush(const K2Args& a, int g, double2& acc, double2 (*red)[16]) {
  const int tid = threadIdx.x, warp = tid >> 5;
#pragma unroll
  for (int o = PG; o < 32; o <<= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if ((tid & 31) < PG) red[warp][tid & 31] = acc;
  __syncthreads();
  if (tid < PG) {
    double2 sacc = red[0][tid];
    for (int ww = 1; ww < kP2Thr / 32; ++ww) sacc = cadd(sacc, red[ww][tid]);
    double* dst = a.part + int64_t(blockIdx.x) * a.part_stride + 2 * (g * PG + tid);
    dst[0] = sacc.x;
    dst[1] = sacc.y;
  }
  __syncthreads();  // red is reused
  acc = make_double2(0.0, 0.0);
}

template <int R, int M, int EP, bool PAD>
__global__ void __launch_bounds__(p2thr<R * M>(), p2thr<R * M>() > 256 ? 1 : 2) k_cols_pipe2(K2Args a, int lg2L2) {
  constexpr int L1 = R * M, kP2PG = p2pg<L1>(), kP2Thr = p2thr<L1>();
  constexpr int STAGE = kP2PG * pipe2_pair_stride<L1>();
  extern __shared__ double2 sm[];
  int* nS = reinterpret_cast<int*>(sm + kPipeStages * STAGE);  // [stage][e1][c]
  __shared__ double2 red[kP2Thr / 32][16];
  __shared__ double2 tw1s[L1];  // ω_{L1}^k: the stage twiddles, read from shared memory
  for (int i = threadIdx.x; i < L1; i += kP2Thr) tw1s[i] = __ldg(&a.tw1[i]);
  if (a.part)  // this CTA's slot row of column partials starts at zero
    for (int i = threadIdx.x; i < a.part_stride; i += kP2Thr) a.part[int64_t(blockIdx.x) * a.part_stride + i] = 0.0;
  __shared__ uint64_t bars[kPipeStages];  // stage st complete (phase per use)
  const int ntiles = a.ntx * a.ngroups;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0 && int(blockIdx.x) < ntiles) k2p2_issue<L1>(a, blockIdx.x, sm, nS, &bars[0]);
  double2 acc = make_double2(0.0, 0.0);
  int gcur = int(blockIdx.x) / a.ntx;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    // this tile's data has landed, and every thread is done with the
    // previous tile: its buffer takes the next tile (one barrier per tile)
    mbar_wait(&bars[st], unsigned(it >> 1) & 1u);
    __syncthreads();
    const int g = tile / a.ntx;
    if (a.part && g != gcur) {
      k2p2_flush<kP2PG, kP2Thr>(a, gcur, acc, red);
      gcur = g;
    }
    const int ahead = tile + gridDim.x;
    if (threadIdx.x == 0 && ahead < ntiles)
      k2p2_issue<L1>(a, ahead, sm + (st ^ 1) * STAGE, nS + (st ^ 1) * (L1 * kUB), &bars[st ^ 1]);
    k2p2_tile<R, M, EP, PAD>(a, tile, sm + st * STAGE, nS + st * (L1 * kUB), acc, tw1s);
  }
  if (a.part && int(blockIdx.x) < ntiles) k2p2_flush<kP2PG, kP2Thr>(a, gcur, acc, red);
}

// out[k] = (1/N) Σ_bx part[bx][kk], k = 2·pair0 + kk: one warp per column,
// lane-strided partial sums, then a fixed shuffle tree (deterministic)
__global__ void k_colpart_reduce(const double* __restrict__ part, int nbx, int part_stride, int ncols, int64_t k0,
                                 int64_t t, int64_t N, double* __restrict__ out) {
  const int kk = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int l = threadIdx.x & 31;
  if (kk >= ncols || k0 + kk >= t) return;  // warp-uniform
  double s = 0.0;
  for (int b = l; b < nbx; b += 32) s += __ldg(&part[int64_t(b) * part_stride + kk]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (l == 0) out[k0 + kk] = s / double(N);
}

__global__ void k_rowsum_reduce(const double* __restrict__ parts, int ng, int64_t N, double* __restrict__ out) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int g = 0; g < ng; ++g) s += __ldg(&parts[int64_t(g) * N + n]);
  out[n] = s;
}

// ---------------------------------------------------------------- finalize
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
static int pair_group(int64_t pairs_b) { return pairs_b >= 16 ? 16 : pairs_b >= 8 ? 8 : 4; }

// K2 tile width (columns e2 per CTA) and grid x for the plan's split
static int cols_cb(const qmc_plan* pl, int PG) { return (k2_split_R(pl->sp.L1) == 1 ? kColThreads : 32) / PG; }

struct CallLayout {
  size_t off_U, off_asort, off_colsum, off_part, off_rowsum, total;
  int PG, ngroups, ngroups_all, nbx, nsets, part_stride;
};

// Whether a call may run its batches on the two internal streams: where they
// overlap something — the per-batch host copies of qmc_mean_host (host), or
// the column pass of plans with L1 <= 16 (measured on B200: c2 0.61 vs 0.68
// ms, c3 24.2 vs 26.7, c4 2.37 vs 2.47; c5 (L1 = 96) 78.8 vs 79.0 ms —
// equal, so its device calls run on the caller's stream, where each kernel's
// event time is its own); green mode: K0/K1 on one SM partition, K2 on the
// other
static bool two_stream_mode(const qmc_plan* pl, bool host) {
#ifdef QMC_DIAG_TWO_ALWAYS
  return pl->nstreams == 2;
#else
  return pl->green || (pl->nstreams == 2 && (host || pl->sp.L1 <= 16));
#endif
}

// pairs per batch of a call on t columns: the plan's batch (the large
// single-stream batch for device calls that stay on the caller's stream),
// capped at half the call's pairs (rounded up to the pair group) so that two
// batches overlap
static int64_t call_batch(const qmc_plan* pl, int64_t t, bool host) {
  const int64_t npairs = std::max<int64_t>(1, (t + 1) / 2);
  const bool one = !two_stream_mode(pl, host);
  int64_t b = one ? pl->batch_pairs_1s : pl->batch_pairs;
  if (npairs >= 128 && !pl->batch_fixed && !one) {  // small calls: one batch (launch-bound)
    const int64_t half = ((npairs + 1) / 2 + 15) / 16 * 16;
    b = std::min(b, half);
  }
  b = std::max<int64_t>(1, b);
  // every batch but the last starts on a K2 pair-group boundary (the row-sum
  // slot of a pair group is pair0 / PG + group)
  const int64_t pg = pair_group(b);
  b = (b + pg - 1) / pg * pg;
  return std::min(b, npairs);
}

static CallLayout call_layout(const qmc_plan* pl, int64_t t, int f, bool host) {
  CallLayout c;
  const int64_t pairs = call_batch(pl, t, host);
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o = align_up(o + b);
    return r;
  };
  // one scratch set (U, partial sums) per internal stream in use
  const int64_t nbatch = ((t + 1) / 2 + pairs - 1) / pairs;
  c.nsets = (two_stream_mode(pl, host) && nbatch > 1) ? 2 : 1;
  c.PG = pair_group(pairs);
  c.ngroups = int((pairs + c.PG - 1) / c.PG);
  // column-partial slots: the larger of the two K2 tilings (k_cols_x: CB
  // columns per CTA; k_cols_pipe: QMC_K2_CB columns per tile)
  const int CB = std::min(cols_cb(pl, c.PG), int(QMC_K2_CB));
  c.nbx = int((pl->sp.L2 + CB - 1) / CB);
  c.part_stride = int(2 * c.ngroups * c.PG);
  c.off_U = take(size_t(c.nsets) * pairs * pl->sp.L * 16);
  c.off_asort = take(size_t(c.nsets) * pairs * pl->S1 * 16);
  c.off_colsum = take(size_t(std::max<int64_t>(t, 1)) * 8);
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  c.off_part = take(colmean ? size_t(c.nsets) * c.nbx * c.part_stride * 8 : 0);
  // row sums: one N-vector per pair group of the whole call (no read-modify-write)
  c.ngroups_all = int(((t + 1) / 2 + c.PG - 1) / c.PG);
  c.off_rowsum = take(f == QMC_F_ROWMEAN_RELU ? size_t(c.ngroups_all) * pl->N * 8 : 0);
  c.total = o;
  return c;
}

template <typename K>
static void set_smem_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

static int ilog2(int64_t x) {
  int r = 0;
  while ((int64_t(1) << r) < x) ++r;
  return r;
}

static K1Args k1_args(const qmc_plan* pl, const double2* asort, int64_t t, int64_t pair0, double2* U, int np,
                      double* colsum) {
  K1Args a;
  a.asort = asort;
  a.e2q = pl->d_e2q;
  a.occ = pl->d_occ;
  a.S1 = pl->S1;
  a.CH = pl->k1_stage;
  a.SRn = (pl->k1_stage == 0 && pl->k1_nch == 1 && pl->k1_bal && !pl->k1_dense) ? pl->k1_srn : 0;
#ifdef QMC_DIAG_NO_SCATTER
  a.SRn = 0;
#endif
  a.k1c = pl->d_k1c;
  a.nch = pl->k1_nch;
  a.bal = pl->k1_bal;
  a.dense = pl->k1_dense;
  a.twj = pl->d_twj;
  a.tw2 = pl->d_tw2;
  a.tw1 = pl->d_tw1;
  a.twL = pl->d_twL;
  a.tw16 = pl->d_tw16;
  a.lg2L2 = ilog2(pl->sp.L2);
  a.W = pl->d_W;
  a.U = U;
  a.L = pl->sp.L;
  a.L1 = int(pl->sp.L1);
  a.np = np;
  a.pair0 = pair0;
  a.t = t;
  a.colsum = colsum;
  return a;
}

static int stream_sms(const qmc_plan* pl, cudaStream_t st);

template <int L2>
static int launch_rows(const qmc_plan* pl, const double2* asort, int64_t t, int64_t pair0, double2* U, int np,
                       double* colsum, cudaStream_t st) {
  const size_t smem = rows_smem<L2>(pl->k1_stage, int(pl->sp.L1),
                                     (pl->k1_stage == 0 && pl->k1_nch == 1 && pl->k1_bal && !pl->k1_dense) ? pl->k1_srn : 0);
  auto kern = k_rows16<L2>;
  static int nsm = 0;
  static size_t last_smem = 0;  // attribute and occupancy of the last shared-memory size (per instantiation)
  static int last_per_sm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  if (smem != last_smem) {
    set_smem_attr(kern, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&last_per_sm, kern, L2 / QMC_ROW_E, smem);
    last_smem = smem;
  }
  int per_sm = last_per_sm;
  if (pl->k1_per_sm > 0) per_sm = std::min(per_sm, pl->k1_per_sm);
  const int64_t items = pl->sp.L1 * int64_t(np);
  int64_t cap = int64_t(pl->green ? stream_sms(pl, st) : nsm) * std::max(per_sm, 1);
  if (pl->k1_grid_cap > 0) cap = std::min<int64_t>(cap, pl->k1_grid_cap);
  const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>(items, cap)));
  kern<<<grid, L2 / QMC_ROW_E, smem, st>>>(k1_args(pl, asort, t, pair0, U, np, colsum));
  QMC_LAUNCHED();
  return QMC_OK;
}

static int rows_dispatch(const qmc_plan* pl, const double2* asort, int64_t t, int64_t pair0, double2* U, int np,
                         double* colsum, cudaStream_t st) {
  switch (pl->sp.L2) {
#define QMC_ROWS_CASE(NN) \
  case NN: return launch_rows<NN>(pl, asort, t, pair0, U, np, colsum, st);
    QMC_ROWS_CASE(16) QMC_ROWS_CASE(32) QMC_ROWS_CASE(64) QMC_ROWS_CASE(128) QMC_ROWS_CASE(256)
    QMC_ROWS_CASE(512) QMC_ROWS_CASE(1024) QMC_ROWS_CASE(2048) QMC_ROWS_CASE(4096) QMC_ROWS_CASE(8192)
#undef QMC_ROWS_CASE
  }
  return QMC_EINVAL_N;
}

static int sm_count_cols() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

// SMs a launch on stream st may use: the plan's green-context partition for
// its internal streams in green mode, else the whole device
static int stream_sms(const qmc_plan* pl, cudaStream_t st) {
  if (pl->green) {
    if (st == pl->ist[0]) return pl->gsm[0];
    if (st == pl->ist[1]) return pl->gsm[1];
  }
  return sm_count_cols();
}

static K2Args k2_args(const qmc_plan* pl, const CallLayout& cl, const double2* U, int ntx, int ng, int64_t pair0,
                      const EpiArgs& E, double* part, double* colsum) {
  K2Args a;
  a.U = U;
  a.L = pl->sp.L;
  a.L2 = int(pl->sp.L2);
  a.m = pl->m;
  a.ntx = ntx;
  a.ngroups = ng;
  a.P = pl->d_P;
  a.colsum = colsum;
  a.scal = pl->d_scal;
  a.tw1 = pl->d_tw1;
  a.twL = pl->d_twL;
  a.pair0 = pair0;
  a.E = E;
  a.part = part;
  a.part_stride = cl.part_stride;
  a.k2n = pl->d_k2n;
  return a;
}

template <int R, int M, int EP>
static int launch_cols_ep(const qmc_plan* pl, const CallLayout& cl, const double2* U, int np, int64_t pair0,
                          const EpiArgs& E, double* part, double* colsum, cudaStream_t st, int* nbx_used) {
  constexpr int L1 = R * M;
  const size_t smem = R == 1 ? 0 : size_t(32) * (L1 | 1) * sizeof(double2);
  // fast path: whole pair groups, whole pairs, vector X stores, no padded rows
  const bool fast = R == 1 && np % cl.PG == 0 && E.t % 2 == 0 && (!E.X || E.xvec) && pl->sp.L == pl->m &&
                    (pl->sp.L2 % ((R == 1 ? kColThreads : 32) / cl.PG)) == 0;
  // the pipelined kernel also takes zero-padded lengths (rows i >= m skipped)
  const bool fastp = R == 1 && np % cl.PG == 0 && E.t % 2 == 0 && (!E.X || E.xvec) &&
                     (pl->sp.L2 % ((R == 1 ? kColThreads : 32) / cl.PG)) == 0;
  if constexpr (R == 1 && (EP != EPK_ROWSUM || L1 == 16)) {
    if (fastp && cl.PG == 16 && !pl->k2_nopipe) {
      constexpr int CBP = QMC_K2_CB;
      constexpr size_t psm = cols_pipe_smem<L1, CBP>();
      auto pk = k_cols_pipe<L1, EP, CBP>;
      static int nsm = 0, per_sm0 = -1;  // per instantiation: constant shared memory
      if (per_sm0 < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        set_smem_attr(pk, psm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm0, pk, 16 * CBP, psm);
      }
      int per_sm = per_sm0;
      if (pl->k2_per_sm > 0) per_sm = std::min(per_sm, pl->k2_per_sm);
      const int ntx = int(pl->sp.L2 / CBP), ng = (np + 15) / 16;
      const int64_t ntiles = int64_t(ntx) * ng;
      const unsigned grid = unsigned(
          std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(pl->green ? stream_sms(pl, st) : nsm) * std::max(per_sm, 1))));
      pk<<<grid, 16 * CBP, psm, st>>>(k2_args(pl, cl, U, ntx, ng, pair0, E, part, colsum));
      QMC_LAUNCHED();
      *nbx_used = ntx;
      return QMC_OK;
    }
  }
  if constexpr (R > 1 && EP != EPK_ROWSUM && cols_pipe2_smem<R * M>() <= 232448) {
    // two-stage column pass, pipelined: whole PG-pair groups, whole pairs,
    // vector X stores, whole U column blocks
    constexpr int kP2PG = p2pg<L1>(), kP2Thr = p2thr<L1>();
    if (np % kP2PG == 0 && E.t % 2 == 0 && (!E.X || E.xvec) && pl->sp.L2 % kUB == 0 && !pl->k2_nopipe) {
      constexpr size_t psm = cols_pipe2_smem<L1>();
      // zero-padded lengths (L > m) skip the rows i >= m; exact lengths need no test
      auto pk = pl->sp.L != pl->m ? k_cols_pipe2<R, M, EP, true> : k_cols_pipe2<R, M, EP, false>;
      static int per_sm0 = -1;  // per instantiation (both variants): constant shared memory
      if (per_sm0 < 0) {
        set_smem_attr(k_cols_pipe2<R, M, EP, true>, psm);
        set_smem_attr(k_cols_pipe2<R, M, EP, false>, psm);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm0, pk, kP2Thr, psm);
      }
      int per_sm = per_sm0;
      if (pl->k2_per_sm > 0) per_sm = std::min(per_sm, pl->k2_per_sm);
      const int ntx = int(pl->sp.L2 / kUB), ng = np / kP2PG;
      const int64_t ntiles = int64_t(ntx) * ng;
      const unsigned grid =
          unsigned(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(stream_sms(pl, st)) * std::max(per_sm, 1))));
      pk<<<grid, kP2Thr, psm, st>>>(k2_args(pl, cl, U, ntx, ng, pair0, E, part, colsum), ilog2(pl->sp.L2));
      QMC_LAUNCHED();
      *nbx_used = int(grid);  // one partial slot row per CTA (k2p2_flush)
      return QMC_OK;
    }
  }
  auto kern = fast ? k_cols_x<R, M, EP, (R == 1)> : k_cols_x<R, M, EP, false>;
  set_smem_attr(kern, smem);
  const int CBx = cols_cb(pl, cl.PG);
  const int nbxT = int((pl->sp.L2 + CBx - 1) / CBx), ngr = (np + cl.PG - 1) / cl.PG;
  // enough CTAs for ~8 per SM; each loops over several column groups, so the
  // column means need only gridDim.x partial slots per pair
  const int gx = std::max(1, std::min(nbxT, (stream_sms(pl, st) * 8 + ngr - 1) / ngr));
  dim3 g((unsigned)gx, (unsigned)ngr);
  *nbx_used = gx;
  kern<<<g, kColThreads, smem, st>>>(U, pl->sp.L, int(pl->sp.L2), ilog2(pl->sp.L2), pl->m, np, cl.PG, pl->d_P,
                                     colsum, pl->d_scal, pl->d_tw1, pl->d_twL, pair0, E, part, cl.part_stride);
  QMC_LAUNCHED();
  return QMC_OK;
}

template <int R, int M>
static int launch_cols(const qmc_plan* pl, const CallLayout& cl, const double2* U, int np, int64_t pair0, int ep,
                       const EpiArgs& E, double* part, double* colsum, cudaStream_t st, int* nbx_used) {
  switch (ep) {
    case EPK_EXP: return launch_cols_ep<R, M, EPK_EXP>(pl, cl, U, np, pair0, E, part, colsum, st, nbx_used);
    case EPK_ROWSUM: return launch_cols_ep<R, M, EPK_ROWSUM>(pl, cl, U, np, pair0, E, part, colsum, st, nbx_used);
    default: return launch_cols_ep<R, M, EPK_LIN>(pl, cl, U, np, pair0, E, part, colsum, st, nbx_used);
  }
}

// launches K2 for the batch; *nbx_used = column-partial slots it wrote
static int cols_dispatch(const qmc_plan* pl, const CallLayout& cl, const double2* U, int np, int64_t pair0, int ep,
                         const EpiArgs& E, double* part, double* colsum, cudaStream_t st, int* nbx_used) {
  const int R = k2_split_R(pl->sp.L1), M = int(pl->sp.L1) / std::max(R, 1);
#define QMC_COLS_CASE(RR, MM) \
  if (R == RR && M == MM) return launch_cols<RR, MM>(pl, cl, U, np, pair0, ep, E, part, colsum, st, nbx_used);
  QMC_K2_SPLITS(QMC_COLS_CASE)
#undef QMC_COLS_CASE
  return QMC_EINVAL_N;
}

static unsigned nblk(int64_t n, int b) { return unsigned((n + b - 1) / b); }

static int dense_cols_dispatch(const qmc_plan* pl, const double2* ad, int np, double2* T, cudaStream_t st) {
  const dim3 g(nblk(pl->sp.L2, 256), unsigned(np));
  switch (pl->sp.L1) {
#define QMC_DENSE_CASE(NN)                                                                                      \
  case NN:                                                                                                      \
    k_dense_cols<NN><<<g, 256, 0, st>>>(ad, pl->sp.L, int(pl->sp.L2), pl->d_tw1, pl->d_twL, T, pl->S1);          \
    QMC_LAUNCHED();                                                                                             \
    return QMC_OK;
    QMC_DENSE_CASE(1) QMC_DENSE_CASE(2) QMC_DENSE_CASE(3) QMC_DENSE_CASE(4) QMC_DENSE_CASE(5) QMC_DENSE_CASE(6)
    QMC_DENSE_CASE(8) QMC_DENSE_CASE(9) QMC_DENSE_CASE(10) QMC_DENSE_CASE(12) QMC_DENSE_CASE(15) QMC_DENSE_CASE(16)
#undef QMC_DENSE_CASE
  }
  const int R = k2_split_R(pl->sp.L1), M = int(pl->sp.L1) / std::max(R, 1);
  const dim3 g2(nblk(pl->sp.L2, dense2_cb(int(pl->sp.L1))), unsigned(np));
#define QMC_DENSE2_CASE(RR, MM)                                                                                   \
  if (RR > 1 && R == RR && M == MM) {                                                                             \
    k_dense_cols2<RR, MM><<<g2, 256, 0, st>>>(ad, pl->sp.L, int(pl->sp.L2), pl->d_tw1, pl->d_twL, T, pl->S1);     \
    QMC_LAUNCHED();                                                                                               \
    return QMC_OK;                                                                                                \
  }
  QMC_K2_SPLITS(QMC_DENSE2_CASE)
#undef QMC_DENSE2_CASE
  return QMC_EINVAL_N;
}

template <int L2, int EP>
static int launch_small(const SmallArgs& sa, int64_t npairs, cudaStream_t st) {
  const size_t smem = small_smem(L2, sa.s);
  auto kern = k_small<L2, EP>;
  static bool attr = false;  // per instantiation: the largest smem this process may request
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(small_smem(L2, kSmallMaxS)));
    attr = true;
  }
  kern<<<unsigned(npairs), small_threads<L2>(), smem, st>>>(sa);
  QMC_LAUNCHED();
  return QMC_OK;
}

template <int L2>
static int launch_small_f(const SmallArgs& sa, int f, int64_t npairs, cudaStream_t st) {
  if (f < 0) return launch_small<L2, EPK_NONE>(sa, npairs, st);
  if (f == QMC_F_EXP) return launch_small<L2, EPK_EXP>(sa, npairs, st);
  return launch_small<L2, EPK_LIN>(sa, npairs, st);
}

static int small_dispatch(const qmc_plan* pl, const SmallArgs& sa, int f, int64_t npairs, cudaStream_t st) {
  switch (pl->sp.L2) {
#define QMC_SMALL_CASE(NN) \
  case NN: return launch_small_f<NN>(sa, f, npairs, st);
    QMC_SMALL_CASE(16) QMC_SMALL_CASE(32) QMC_SMALL_CASE(64) QMC_SMALL_CASE(128) QMC_SMALL_CASE(256)
    QMC_SMALL_CASE(512) QMC_SMALL_CASE(1024) QMC_SMALL_CASE(2048) QMC_SMALL_CASE(4096) QMC_SMALL_CASE(8192)
#undef QMC_SMALL_CASE
  }
  return QMC_EINVAL_N;
}

// one batch of column pairs [pair0, pair0 + np) on stream bs (scratch set
// bidx & 1 when two sets are in use): K0, K1, K2 and the column-mean reduce
static int run_batch(const qmc_plan* pl, const CallLayout& cl, const double* A, int64_t lda, int64_t t, int f,
                     double* out, EpiArgs E, char* ws, int64_t pairs_b, int64_t pair0, int64_t bidx, cudaStream_t bs,
                     cudaStream_t bs2, const double* A_host, int64_t lda_host) {
  const int64_t npairs_total = (t + 1) / 2;
  const bool colmean = f == QMC_F_IDENTITY || f == QMC_F_AFFINE || f == QMC_F_EXP;
  const int nsets = cl.nsets;
  const int ep = f == QMC_F_ROWMEAN_RELU ? EPK_ROWSUM : f == QMC_F_EXP ? EPK_EXP : EPK_LIN;
  double* colsum = (double*)(ws + cl.off_colsum);
  const int np = int(std::min<int64_t>(pairs_b, npairs_total - pair0));
  const int set = nsets == 2 ? int(bidx & 1) : 0;
  double2* U = (double2*)(ws + cl.off_U) + size_t(set) * pairs_b * pl->sp.L;
  double* part = (double*)(ws + cl.off_part) + size_t(set) * cl.nbx * cl.part_stride;
  E.rowpart = (double*)(ws + cl.off_rowsum);
  double2* asort = (double2*)(ws + cl.off_asort) + size_t(set) * pairs_b * pl->S1;
  // green mode (bs2 != bs): K0/K1 on bs, K2 and the reduce on bs2 once the
  // set's U is written; batch bidx reuses the set after batch bidx - 2's K2
  // and reduce have read it
  const bool split = bs2 != bs;
  if (split && bidx >= nsets && cudaStreamWaitEvent(bs, pl->ev_free[set], 0) != cudaSuccess) return QMC_ECUDA;
  if (A_host) {
    const int64_t c0 = 2 * pair0, nc = std::min<int64_t>(2 * int64_t(np), t - c0);
    if (cudaMemcpy2DAsync(const_cast<double*>(A) + c0 * lda, size_t(lda) * 8, A_host + c0 * lda_host,
                          size_t(lda_host) * 8, size_t(pl->s) * 8, size_t(nc), cudaMemcpyHostToDevice,
                          bs) != cudaSuccess)
      return QMC_ECUDA;
  }
  prof_begin(KC_PACK, bs);
  if (pl->k1_dense) {
    // a' into this set's U (K1 overwrites it afterwards), T into asort
    k_pack_dense<<<dim3(nblk(pl->sp.L, 256), unsigned(np)), 256, 0, bs>>>(A, lda, t, pair0, pl->d_jq,
                                                                        pl->d_e2q, pl->sp.L, U);
    QMC_LAUNCHED();
    int rc0 = dense_cols_dispatch(pl, U, np, asort, bs);
    if (rc0) return rc0;
  } else if (pl->s <= kPackSmemMax && !pl->pack_gather) {
    const size_t psm = size_t(pl->s) * 16;
    set_smem_attr(k_pack_smem, psm);
    // slices of the slots: ~2 CTAs of work per SM in total
    const int ny = int(std::max<int64_t>(1, std::min<int64_t>((2 * stream_sms(pl, bs) + np - 1) / np,
                                                              (pl->S1 + 1023) / 1024)));
    k_pack_smem<<<dim3(unsigned(np), unsigned(ny)), 256, psm, bs>>>(A, lda, t, pair0, pl->d_jq, pl->s, pl->S1,
                                                                    asort);
  } else {
    k_pack<<<dim3(nblk(pl->S1, 256), unsigned(np)), 256, 0, bs>>>(A, lda, t, pair0, np, pl->d_jq, pl->S1, asort);
  }
  QMC_LAUNCHED();
  prof_end(KC_PACK, bs);
  prof_begin(KC_ROWS, bs);
  int rc = rows_dispatch(pl, asort, t, pair0, U, np, colsum, bs);
  if (rc) return rc;
  prof_end(KC_ROWS, bs);
  if (split && (cudaEventRecord(pl->ev_ready[set], bs) != cudaSuccess ||
                cudaStreamWaitEvent(bs2, pl->ev_ready[set], 0) != cudaSuccess))
    return QMC_ECUDA;
  prof_begin(KC_COLS, bs2);
  int nbx_used = cl.nbx;
  rc = cols_dispatch(pl, cl, U, np, pair0, ep, E, colmean ? part : nullptr, colsum, bs2, &nbx_used);
  if (rc) return rc;
  prof_end(KC_COLS, bs2);
  if (colmean) {
    prof_begin(KC_REDUCE, bs2);
    k_colpart_reduce<<<nblk(2 * np, 8), 256, 0, bs2>>>(part, nbx_used, cl.part_stride, 2 * np, 2 * pair0, t,
                                                        pl->N, out);
    QMC_LAUNCHED();
    prof_end(KC_REDUCE, bs2);
  }
  if (split && cudaEventRecord(pl->ev_free[set], bs2) != cudaSuccess) return QMC_ECUDA;
  return QMC_OK;
}

// all batches of column pairs; f = -1: X only.  A_host != NULL: each batch
// first copies its own columns of A from the host (A_host, leading dimension
// lda_host) into A on the batch's stream, so that the copy of one batch
// overlaps the kernels of the other.
static int run(const qmc_plan* pl, const double* A, int64_t lda, int64_t t, int f, double fparam,
               double* out, double* X, int64_t ldx, void* call_ws, size_t call_ws_bytes, cudaStream_t st,
               const double* A_host = nullptr, int64_t lda_host = 0) {
  if (!pl) return QMC_ENULL;
  if (t < 0 || lda < pl->s) return QMC_EINVAL_DIM;
  if (X && ldx < t) return QMC_EINVAL_DIM;
  if (f >= 0 && !out) return QMC_ENULL;
  if (t == 0) {
    // an empty slab (e.g. a rank with no columns): the row functional's
    // partial row sums are all zero, so a later all-reduce stays exact; the
    // per-column means have no entries
    if (f == QMC_F_ROWMEAN_RELU && cudaMemsetAsync(out, 0, size_t(pl->N) * 8, st) != cudaSuccess) return QMC_ECUDA;
    return QMC_OK;
  }
  if (!A || !call_ws) return QMC_ENULL;
  if (f < 0 && !X) return QMC_ENULL;
  if (pl->sp.L1 == 1 && pl->s <= kSmallMaxS && f != QMC_F_ROWMEAN_RELU) {
    // one-row plan: one fused launch per call
    if (A_host && cudaMemcpy2DAsync(const_cast<double*>(A), size_t(lda) * 8, A_host, size_t(lda_host) * 8,
                                    size_t(pl->s) * 8, size_t(t), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return QMC_ECUDA;
    SmallArgs sa;
    sa.A = A;
    sa.lda = lda;
    sa.t = t;
    sa.bstart = pl->d_bstart;
    sa.bent = pl->d_bent;
    sa.s = pl->s;
    sa.m = pl->m;
    sa.N = pl->N;
    sa.tw2 = pl->d_tw2;
    sa.W = pl->d_W;
    sa.P = pl->d_P;
    sa.scal = pl->d_scal;
    sa.X = X;
    sa.ldx = ldx;
    sa.fparam = f == QMC_F_AFFINE ? fparam : 0.0;
    sa.out = f >= 0 ? out : nullptr;
    prof_begin(KC_ROWS, st);
    const int rc = small_dispatch(pl, sa, f, (t + 1) / 2, st);
    if (rc) return rc;
    prof_end(KC_ROWS, st);
    return QMC_OK;
  }
  const CallLayout cl = call_layout(pl, t, f, A_host != nullptr);
  if (call_ws_bytes < cl.total || (uintptr_t(call_ws) % kAlign)) return QMC_EWORKSPACE;
  char* ws = (char*)call_ws;
  const int64_t pairs_b = call_batch(pl, t, A_host != nullptr);
  const int64_t npairs_total = (t + 1) / 2;
  EpiArgs E;
  E.fparam = f == QMC_F_AFFINE ? fparam : 0.0;
  E.X = X;
  E.ldx = ldx;
  E.xvec = X && (ldx % 2 == 0) && (uintptr_t(X) % 16 == 0);
  E.t = t;
  E.N = pl->N;
  E.rowpart = (double*)(ws + cl.off_rowsum);
  std::unique_lock<std::mutex> lock;
  // two internal streams where they overlap something (two_stream_mode; the
  // layout holds two scratch sets exactly then); green mode: K0/K1 of every
  // batch on one SM partition, K2 on the other
  const bool green = cl.nsets == 2 && pl->green;
  const bool two = cl.nsets == 2;
  if (two) {  // fork: both internal streams start after the caller's prior work
    lock = std::unique_lock<std::mutex>(*pl->mu);
    if (cudaEventRecord(pl->ev_fork, st) != cudaSuccess ||
        cudaStreamWaitEvent(pl->ist[0], pl->ev_fork, 0) != cudaSuccess ||
        cudaStreamWaitEvent(pl->ist[1], pl->ev_fork, 0) != cudaSuccess) {
      cudaGetLastError();
      return QMC_ECUDA;
    }
  }
  int64_t bidx = 0;
  int rc = QMC_OK;
  for (int64_t pair0 = 0; pair0 < npairs_total && rc == QMC_OK; pair0 += pairs_b, ++bidx) {
    const cudaStream_t bs = green ? pl->ist[0] : two ? pl->ist[bidx & 1] : st;
    rc = run_batch(pl, cl, A, lda, t, f, out, E, ws, pairs_b, pair0, bidx, bs, green ? pl->ist[1] : bs, A_host,
                   lda_host);
  }
  if (two) {  // join (also after an error: the caller's stream must not run ahead of queued batches)
    const bool ok = cudaEventRecord(pl->ev_join[0], pl->ist[0]) == cudaSuccess &&
                    cudaEventRecord(pl->ev_join[1], pl->ist[1]) == cudaSuccess &&
                    cudaStreamWaitEvent(st, pl->ev_join[0], 0) == cudaSuccess &&
                    cudaStreamWaitEvent(st, pl->ev_join[1], 0) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      if (rc == QMC_OK) rc = QMC_ECUDA;
    }
  }
  if (rc) return rc;
  if (f == QMC_F_ROWMEAN_RELU) {
    prof_begin(KC_REDUCE, st);
    // parts [group][N], every pair group of the call, fixed order
    k_rowsum_reduce<<<nblk(pl->N, 256), 256, 0, st>>>((double*)(ws + cl.off_rowsum), cl.ngroups_all, pl->N, out);
    QMC_LAUNCHED();
    prof_end(KC_REDUCE, st);
  }
  return QMC_OK;
}
static int pset_dispatch(const qmc_plan* pl, const SmallArgs& sa, int64_t npairs, cudaStream_t st) {
  switch (pl->sp.L2) {
#define QMC_PSET_CASE(NN) \
  case NN: return launch_pset<NN>(pl, sa, npairs, st);
    QMC_PSET_CASE(16) QMC_PSET_CASE(32) QMC_PSET_CASE(64) QMC_PSET_CASE(128) QMC_PSET_CASE(256)
    QMC_PSET_CASE(512) QMC_PSET_CASE(1024) QMC_PSET_CASE(2048) QMC_PSET_CASE(4096) QMC_PSET_CASE(8192)
#undef QMC_PSET_CASE
  }
  return QMC_EINVAL_N;
}

}  // namespace qmc

using namespace qmc;

// randomised-QMC estimate over R replicates (qmc_replicate_mean; reading
// R28): one thread per column k, replicates summed in the fixed order r = 0..R-1
__global__ void k_replicate_mean(const double* __restrict__ means, int64_t R, int64_t t, int64_t ld,
                                 double* __restrict__ mean_out, double* __restrict__ stderr_out) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= t) return;
  double sum = 0.0;
  for (int64_t r = 0; r < R; ++r) sum += means[r * ld + k];
  const double mu = sum / double(R);
  mean_out[k] = mu;
  if (stderr_out) {
    double ss = 0.0;
    for (int64_t r = 0; r < R; ++r) {
      const double d = means[r * ld + k] - mu;
      ss = fma(d, d, ss);
    }
    stderr_out[k] = R > 1 ? sqrt(ss / (double(R) * double(R - 1))) : __longlong_as_double(0x7ff8000000000000LL);
  }
}

extern "C" {

int qmc_call_workspace_size(qmc_plan_t pl, int64_t t, int f, size_t* call_bytes) {
  if (!pl || !call_bytes) return QMC_ENULL;
  if (t < 0) return QMC_EINVAL_DIM;
  if (f < -1 || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  // the larger of the device-call and host-entry layouts (their batches differ)
  *call_bytes = std::max(call_layout(pl, t, f, false).total, call_layout(pl, t, f, true).total);
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

int qmc_pset_matmul(qmc_plan_t pl, const double* A, int64_t lda, int64_t t, double* X, int64_t ldx,
                    void* stream) {
  if (!pl) return QMC_ENULL;
  if (pl->family != QMC_FAMILY_LATTICE || pl->delta != 0.0) return QMC_EINVAL_N;
  if (pl->sp.L1 != 1 || pl->s > kSmallMaxS) return QMC_EUNSUPPORTED;
  if (t < 0 || lda < pl->s || ldx < t) return QMC_EINVAL_DIM;
  if (t == 0) return QMC_OK;
  if (!A || !X) return QMC_ENULL;
  SmallArgs sa;
  sa.A = A;
  sa.lda = lda;
  sa.t = t;
  sa.bstart = nullptr;
  sa.bent = nullptr;
  sa.s = pl->s;
  sa.m = pl->m;
  sa.N = pl->N;
  sa.tw2 = pl->d_tw2;
  sa.W = pl->d_W;
  sa.P = pl->d_P;
  sa.scal = pl->d_scal;
  sa.X = X;
  sa.ldx = ldx;
  sa.fparam = 0.0;
  sa.out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  prof_begin(KC_ROWS, st);
  const int rc = pset_dispatch(pl, sa, (t + 1) / 2, st);
  if (rc) return rc;
  prof_end(KC_ROWS, st);
  return QMC_OK;
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

int qmc_replicate_mean(const double* means, int64_t R, int64_t t, int64_t ld, double* mean_out,
                       double* stderr_out, void* stream) {
  if (R < 1 || t < 0 || ld < t) return QMC_EINVAL_DIM;
  if (t == 0) return QMC_OK;
  if (!means || !mean_out) return QMC_ENULL;
  k_replicate_mean<<<nblk(t, 128), 128, 0, (cudaStream_t)stream>>>(means, R, t, ld, mean_out, stderr_out);
  QMC_LAUNCHED();
  return QMC_OK;
}

int qmc_mean_host(qmc_plan_t pl, const double* A_host, int64_t lda, int64_t t, int f, double f_param,
                  double* out_host, double* A_dev, double* X_dev, int64_t ldx, double* out_dev,
                  void* call_ws, size_t call_ws_bytes, void* stream) {
  if (!pl || !A_host || !out_host || !A_dev || !out_dev) return QMC_ENULL;
  if (f < QMC_F_IDENTITY || f > QMC_F_ROWMEAN_RELU) return QMC_EINVAL_F;
  if (t < 1 || lda < pl->s) return QMC_EINVAL_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  // the H2D copy of A goes batch by batch inside run (overlapping the kernels)
  int rc = run(pl, A_dev, pl->s, t, f, f_param, out_dev, X_dev, ldx, call_ws, call_ws_bytes, st, A_host, lda);
  if (rc) return rc;
  rc = qmc_mean_finalize(pl, f, out_dev, t, out_dev, stream);
  if (rc) return rc;
  const size_t nout = f == QMC_F_ROWMEAN_RELU ? 1 : size_t(t);
  if (cudaMemcpyAsync(out_host, out_dev, nout * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess) return QMC_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return QMC_ECUDA;
  return QMC_OK;
}

}  // extern "C"
