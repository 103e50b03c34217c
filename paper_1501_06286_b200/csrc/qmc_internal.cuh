// qmc_internal.cuh — plan object and shared helpers of libqmc (not part of
// the ABI).  See include/qmc.h for the contract and DESIGN.md for the data
// layout in HBM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "../../include/qmc.h"

namespace qmc {

constexpr size_t kAlign = 256;

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// Bounds checks of the checked build (-DQMC_CHECK, tools/check_build.sh):
// every shared-memory row slot, staged slot, U and X index the kernels
// compute is tested against its buffer; a violation prints and traps.
// compute-sanitizer is closed on this GPU pool, so this build (run on the
// GPU parity suite) and the guard-zone tests (tests/test_guards_gpu.py)
// stand in for memcheck.  Compiles to nothing otherwise.
#ifdef QMC_CHECK
#include <stdio.h>
#define QMC_CHECK_IDX(i, n)                                                                          \
  do {                                                                                               \
    const long long _i = (long long)(i), _n = (long long)(n);                                        \
    if (_i < 0 || _i >= _n) {                                                                        \
      printf("QMC_CHECK %s:%d: index %lld outside [0, %lld)\n", __FILE__, __LINE__, _i, _n);         \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define QMC_CHECK_IDX(i, n) \
  do {                      \
  } while (0)
#endif

// number of kernels launched by the library (qmc_launch_count)
extern std::atomic<int64_t> g_launches;

// Optional per-kernel-class CUDA-event timing (qmc_profile_*): events are
// recorded on the launching stream around every hot-path launch.
enum KernelClass { KC_PACK = 0, KC_ROWS, KC_COLS, KC_GATHER, KC_REDUCE, KC_FINALIZE, KC_COUNT };
void prof_begin(int kc, cudaStream_t st);
void prof_end(int kc, cudaStream_t st);

inline int cuda_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QMC_OK : QMC_ECUDA;
}

#define QMC_LAUNCHED()                                    \
  do {                                                    \
    ::qmc::g_launches.fetch_add(1, std::memory_order_relaxed); \
    if (cudaPeekAtLastError() != cudaSuccess) {           \
      cudaGetLastError();                                 \
      return QMC_ECUDA;                                   \
    }                                                     \
  } while (0)

// FFT length selection (host): L = L1·L2, L2 a power of two in [16, 8192]
// (row FFT, shared memory), L1 ∈ {1} ∪ 2^a 3^b 5^c ≤ 1024 (column FFT).
// L = m when m splits that way, otherwise the smallest such L ≥ 2m-1
// (zero-padded cyclic correlation; exact).
struct Split {
  int64_t L, L1, L2;
  bool padded;
};
bool choose_split(int64_t m, int64_t s, Split* out);

// Plan-workspace carve-up (device pointers), identical for the size query
// and the create call.
struct PlanLayout {
  size_t off_scal, off_P, off_L, off_R, off_e, off_bstart, off_bent, off_e2q, off_occ, off_cursor, off_zeta, off_W,
      off_tw1, off_tw2, off_twL, off_tw16, off_twj, off_jq, off_k1c, off_k2n, off_tmp, total;
};
// K1 scatter-input order (plan.cu k1_balanced_order): tried when the
// buckets are small enough to balance (s <= 8·L2), at most k1_s1max slots;
// otherwise the bucket order (s slots) or, when every e_j is distinct, the
// dense input of L slots (pipeline.cu k_dense_cols)
inline bool k1_try_balanced(int64_t s, int64_t L2) { return s <= 8 * L2; }
inline int64_t k1_s1max(int64_t s, int64_t L2, int64_t L) {
  return k1_try_balanced(s, L2) ? 2 * s + L2 + 64 : (s > L ? s : L);
}
// K1 balanced order (plan.cu k1_balanced_order): slot codes hold the row
// index v of the running sum in bits 0..13 — a bucket e2 < L2, the padding
// slot v = L2, or overflow slot v = L2 + 1 + o (o < kK1Ovf) of a bucket's
// second and later pieces — and kK1First on the first entry of a piece;
// fix-up records (after a chunk's slots) are e2 | o0 << 14 | count << 20
// (S[e2] += S[L2+1+o0] + ... in order).
// column-block width of K1's output U: U[p] is [e2 / kUB][f1][e2 % kUB]
constexpr int kUB = 4;
constexpr int kK1First = 1 << 14;
// regular slot codes also carry e1 = e_j div L2 (< 512) from bit 15: the
// index of the scatter twiddle ω_{L1}^{e1 f1}
constexpr int kK1E1Shift = 15;
constexpr int kK1Ovf = 64;
// K1 shared memory after the row: two buffers of the item's 16 register
// twiddles and 16 constant ones, before the L1 constant column twiddles
// (pipeline.cu rows_smem)
constexpr int kK1Aux = 48;
// replicas of the item's scatter-twiddle table in K1's shared memory (direct mode)
constexpr int kK1TwRep = 8;
// shared-memory row slots of K1: padE(v) for every v <= L2 + kK1Ovf
__host__ __device__ inline constexpr int64_t k1_row_slots(int64_t L2, int E) {
  return L2 + kK1Ovf + 1 + (L2 + kK1Ovf) / E + 1;
}
PlanLayout plan_layout(int64_t N, int64_t m, int64_t s, const Split& sp);

// K2 column-pass splits L1 = R·M (pipeline.cu k_cols_x): R = 1 is one thread
// per column with L1 values in registers; R > 1 is two register stages
// through shared memory.  X(R, M) for every supported L1.
// (QMC_K2_R96: R of config 5's L1 = 96 — 6·16 by default; 8·12 and 12·8
// are build knobs for the stage balance of k_cols_pipe2)
#ifndef QMC_K2_R96
#define QMC_K2_R96 6
#endif
#define QMC_K2_SPLITS(X)                                                                       \
  X(1, 1) X(1, 2) X(1, 3) X(1, 4) X(1, 5) X(1, 6) X(1, 8) X(1, 9) X(1, 10) X(1, 12) X(1, 15)   \
  X(1, 16) X(2, 10) X(2, 12) X(5, 5) X(2, 16) X(4, 10) X(3, 16) X(4, 16) X(5, 16)               \
  X(QMC_K2_R96, (96 / QMC_K2_R96)) X(8, 16) X(10, 16) X(12, 16) X(16, 16)
// R of the K2 split of L1 (0: L1 not supported)
inline int k2_split_R(int64_t L1) {
#define QMC_K2_R(RR, MM) \
  if (L1 == RR * MM) return RR;
  QMC_K2_SPLITS(QMC_K2_R)
#undef QMC_K2_R
  return 0;
}

}  // namespace qmc

struct qmc_plan {
  int family;
  int phi;
  double delta;         // equal shift Δ of the rule (0: unshifted)
  int64_t N, m, s;
  int D;
  uint64_t p;
  int64_t gen;
  qmc::Split sp;
  int64_t batch_pairs;  // column pairs per batch of two-stream calls (one U set <= ~768 MB)
  int64_t batch_pairs_1s;  // column pairs per batch of single-stream device calls (L1 > 16)
  int k1_per_sm;        // persistent K1 CTAs per SM (0: as many as fit)
  int k2_per_sm;        // persistent K2 CTAs per SM (0: as many as fit)
  int k1_grid_cap;      // QMC_K1_GRID: cap on K1's persistent grid (0: none; leaves SMs to the other stream)
  // tuning knobs, read from the environment once at plan creation
  int batch_fixed;      // QMC_BATCH_PAIRS set: no per-call halving of the batch
  int k2_nopipe;        // QMC_K2_NOPIPE: non-persistent column pass
  int pack_gather;      // QMC_PACK_GATHER: K0 gathers A straight from global memory
  // K1 scatter input (plan.cu k1_balanced_order): S1 staged slots per pair / per f1
  // in k1_nch chunks of at most k1_ch slots; k1_bal = 1: balanced
  // thread-major order of bucket pieces (codes: kK1First), 0: bucket order
  int64_t S1;
  int k1_bal, k1_nch, k1_ch;
  int k1_stage;  // > 0: the balanced order is one chunk of k1_stage slots, staged in shared memory
  int k1_srn;    // direct mode: the first k1_srn slots (whole rounds; a and code, 20 B each) staged
  int k1_dense;  // 1: dense first pass (k_pack_dense + k_dense_cols), S1 = L, no chunks
  cudaStream_t stream;
  // batches alternate over nstreams internal streams (fork/join from the
  // caller's stream) so one batch's K1 overlaps the previous batch's K2/K3
  int nstreams;
  cudaStream_t ist[2];
  cudaEvent_t ev_fork, ev_join[2];
  // green mode (QMC_GREEN, plan_streams): ist[0] runs on one green-context
  // SM partition (K0, K1: gsm[0] SMs), ist[1] on the other (K2: gsm[1] SMs);
  // ev_ready[set] = the set's U is written, ev_free[set] = it was read
  int green;
  int gsm[2];
  cudaEvent_t ev_ready[2], ev_free[2];
  std::mutex* mu;
  // device pointers into plan_ws
  char* ws;
  size_t ws_bytes;
  double* d_scal;    // [0] = φ(0), [1] = generator (as double), [2] = status flags
  int32_t* d_P;      // [m]
  int32_t* d_L;      // [N]
  int32_t* d_R;      // [N]  R[n] = (m - L[n]) mod m, n >= 1 (tables / tests)
  int32_t* d_e;      // [s]
  int32_t* d_bstart; // [L2+1]
  int32_t* d_e2q;    // [S1]  bucket codes of the K1 order: heads — e2 = e_j mod L2, |
                     //       (bucket size << 13) on the first entry of each bucket;
                     //       balanced — see kK1First
  uint32_t* d_occ;   // [L2/32+1] bitmap of the nonempty buckets e2
  int4* d_bent;      // [s]   bucket order (e2 = e_j mod L2, then j): {j, e_j, e2,
                     //       end of this bucket if the entry is its first, else -1}
  double* d_zeta;    // [m]
  double2* d_W;      // [L]   W[f1*L2 + r*L2/16 + t] = DFT_L(K)[f1 + L1 f2] / L, f2 = dif_freq(t, r)
  double2* d_tw1;    // [L1]  ω_{L1}^k
  double2* d_tw2;    // [L2]  ω_{L2}^k
  double2* d_twL;    // [L2]  ω_L^k, k < L2
  double2* d_tw16;   // [16 L1] ω_{16 L1}^k (K1: the column-register part of ω_L^{e2 f1})
  int32_t* d_k2n;    // [L] conventional row n of reordered row i = L2 e1 + 4 bx + c at [bx][e1][c] (-1: i >= m), K2's tiles
  double2* d_twj;    // [L1·S1] twj[f1·S1 + q] = ω_{L1}^{(e1_j·f1) mod L1}, e1 = e div L2, j = jq[q] (K1 scatter
                     //        twiddles in the K1 order; 0 for padding slots)
  int32_t* d_jq;     // [S1]  column j of slot q of the K1 order (-1: padding)
  int32_t* d_k1c;    // [k1_nch+1] chunk starts, then [k1_nch] regular-round slots per chunk
};
