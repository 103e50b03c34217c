/*
 * qmc.h — C ABI of the B200-native fast QMC matrix product
 *         X = Y·A  (Dick, Kuo, Le Gia, Schwab, "Fast QMC matrix-vector
 *         multiplication", arXiv 1501.06286; text in PAPER.md).
 *
 * What is computed (§1): for QMC points y_0..y_{N-1}
 * (rows of Y, N×s) and a dense fp64 matrix A (s×t), the product
 *     X = Y·A,   X[n,k] = Σ_j Y[n,j]·A[j,k],
 * with Y[n,j] = φ(x_{n,j}) the same univariate φ on every coordinate
 * (PAPER.md:288-302), where x_n is either
 *   - the rank-1 lattice point ({n z_1/N}, …, {n z_s/N}), N prime
 *     (PAPER.md:243-253), or
 *   - the polynomial-lattice point over F_2 with modulus p(x) primitive of
 *     degree D, N = 2^D: x_{n,j} = v_D(n(x) q_j(x) mod p(x) / p(x))
 *     (reading R3).
 * Rows are returned in the CONVENTIONAL order n = 0..N-1 (reading R4).
 *
 * How (§2.1): with β a primitive element (the smallest,
 * reading R1) and z_j = β^{c_j-1}, rows 1..N-1 in the reordered order
 * factor as Y' = Z·P (Eq. ZPa), Z circulant of length
 * m = N-1 (m = 2^D-1 for F_2).  Per column a of A the library scatter-adds
 * a into m bins (a' = P a), computes Z a' by FFT
 * (PAPER.md:358-362), fuses the un-permutation to conventional order and
 * the row-0 term y_0·a = φ(0) Σ_j a_j, and optionally
 * a downstream f and its QMC mean (1/N) Σ_n f(b_n) (PAPER.md:60-62,
 * 154-157).  Every step runs in this library's CUDA kernels (sm_100a).
 *
 * Conventions for every entry point
 *   - Return value: QMC_OK (0) or a negative QMC_E* code; qmc_strerror()
 *     names it.  No exception crosses the ABI.  Invalid arguments are
 *     detected on the host before anything is launched.
 *   - Asynchrony: compute calls enqueue work on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream) and return; device
 *     faults surface at the caller's next synchronisation.  qmc_plan_create*
 *     and qmc_plan_tables synchronise `stream` before returning.
 *   - Memory: "device" pointers are CUDA device memory on the current
 *     device, owned by the caller; the library never allocates device
 *     memory.  The plan handle is a small host object owned by the caller
 *     (free with qmc_plan_destroy); it references plan_ws, which must
 *     outlive it.  A plan is immutable after creation; concurrent calls on
 *     one plan are safe if each uses its own call workspace.
 *   - Layouts: A is column-major s×t with leading dimension lda >= s
 *     (column k at A + k*lda); X is ROW-major N×t with ldx >= t (row n, the
 *     t outputs of QMC point n, at X + n*ldx).  A column shard of either is
 *     a pointer offset (A + k0*lda, X + k0) with the same leading dimension.
 *     Row-major X lets the column pass write each reordered output row i
 *     straight to its conventional row n as one contiguous chunk (DESIGN.md
 *     §5).  Fastest with ldx even and X 16-byte aligned.
 */
#ifndef QMC_H
#define QMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qmc_plan* qmc_plan_t;

/* point-set family */
enum { QMC_FAMILY_LATTICE = 0, QMC_FAMILY_POLY = 1 };

/* φ: the univariate transform applied to every coordinate.
 * IDENTITY φ(u)=u; SHIFT_HALF φ(u)=u-1/2; TENT φ(u)=1-|2u-1|;
 * INVNORM_MID φ(u)=Φ^{-1}(u + 1/(2N)) — the paper's Φ^{-1} with the equal
 * shift Δ=1/(2N) it allows, finite at u=0 (reading R6).
 * Plain Φ^{-1} is not offered: Φ^{-1}(0) = -inf at row 0. */
enum { QMC_PHI_IDENTITY = 0, QMC_PHI_SHIFT_HALF = 1, QMC_PHI_TENT = 2, QMC_PHI_INVNORM_MID = 3,
       QMC_PHI_BERNOULLI2 = 4 /* B_2(u) = u^2 - u + 1/6: the kernel of the shift-averaged
                                 worst-case error used by the CBC search (qmc_cbc_step) */ };

/* fused downstream functional for qmc_mean (PAPER.md:60-62 eq_qmc) */
enum {
  QMC_F_IDENTITY = 0,      /* out[k] = (1/N) Σ_n X[n,k]                       */
  QMC_F_AFFINE = 1,        /* out[k] = (1/N) Σ_n (c + X[n,k]); X receives c+X  */
  QMC_F_EXP = 2,           /* out[k] = (1/N) Σ_n exp(X[n,k]); X receives X     */
  QMC_F_ROWMEAN_RELU = 3   /* out[n] = Σ_k X[n,k] over the local columns (N
                              partial row sums); qmc_mean_finalize then gives
                              Q = (1/N) Σ_n max(0, r_n / t_total) (reading R10) */
};

/* status codes */
enum {
  QMC_OK = 0,
  QMC_EINVAL_N = -1,      /* N not prime / out of range / unsupported length  */
  QMC_EINVAL_Z = -2,      /* z_j not in [1, N-1] (q_j not in [1, 2^D-1])      */
  QMC_EINVAL_POLY = -3,   /* p not of degree D, or not primitive              */
  QMC_EINVAL_DIM = -4,    /* s < 1, t < 0, lda < s, ldx < t                   */
  QMC_EINVAL_PHI = -5,    /* unknown φ                                        */
  QMC_ENULL = -6,         /* required pointer is NULL                         */
  QMC_ECUDA = -7,         /* CUDA launch / runtime error                      */
  QMC_EWORKSPACE = -8,    /* workspace too small or misaligned (256 B)        */
  QMC_EINVAL_F = -9,      /* unknown f                                        */
  QMC_EUNSUPPORTED = -10  /* valid request this entry point does not cover    */
};

/* Bytes of device memory the plan needs (plan_ws).  family/N_or_D/s as in
 * qmc_plan_create / qmc_plan_create_poly.  Validates N (or D) and s. */
int qmc_plan_workspace_size(int family, int64_t N_or_D, int64_t s, size_t* plan_bytes);

/* Bytes of device scratch one qmc_matmul / qmc_mean / qmc_mean_host call
 * on t columns needs (call_ws).  Independent of A and X.  Dominated by U, the
 * batch's row-FFT output: two sets of up to ~768 MB for calls on the two
 * internal streams (host entry, plans with L1 <= 16), one set of up to
 * ~16 GB for device calls of plans with L1 > 16, which run on the caller's
 * stream in large batches; the larger of the two; for ROWMEAN_RELU add one
 * N-vector of partial row sums per group of 16 column pairs
 * (8·N·ceil(t/32) bytes). */
int qmc_call_workspace_size(qmc_plan_t plan, int64_t t, int f, size_t* call_bytes);

/* Rank-1 lattice plan.  N prime, 3 <= N < 2^31;
 * z_host: s host int64 values, each in [1, N-1] (repeats allowed,
 * reading R18).  Builds on the device, in plan_ws (256-B aligned, at least
 * qmc_plan_workspace_size bytes): β (smallest primitive root, R1), the power
 * table P[k] = β^k mod N, the log table L (L[P[k]] = k, L[0] = -1), e_j =
 * c_j - 1 = L[z_j], the circulant base ζ_k = φ(P[k]/N)
 * and the spectrum of Z.  Synchronises `stream`.  On error *out is NULL. */
int qmc_plan_create(qmc_plan_t* out, int64_t N, int64_t s, const int64_t* z_host, int phi,
                    void* plan_ws, size_t plan_ws_bytes, void* stream);

/* Randomly shifted rank-1 lattice (the paper's equal shift, PAPER.md:466-468;
 * SURVEY §8(f) NEXT #4): as qmc_plan_create with every point shifted by the
 * same Δ in [0, 1) in every coordinate, x_{n,j} = frac(n z_j / N + Δ); for
 * INVNORM_MID the midpoint shift 1/(2N) is composed with Δ:
 * φ = Φ^{-1}(frac(n z_j/N + 1/(2N) + Δ)).  Only ζ (the circulant base) and
 * φ(x_0) change, so independent shifts Δ_r give cheap randomised replicates
 * and error bars.  Δ outside [0, 1) -> QMC_EINVAL_PHI.  With INVNORM_MID a Δ
 * that puts a point exactly on 0 (Δ ≡ -(2i+1)/(2N) mod 1) makes that φ
 * infinite; such Δ have measure zero and are not rejected. */
int qmc_plan_create_shifted(qmc_plan_t* out, int64_t N, int64_t s, const int64_t* z_host, int phi,
                            double delta, void* plan_ws, size_t plan_ws_bytes, void* stream);

/* Shifted replicate of a lattice plan (with an equal shift
 * only the circulant base ζ — so φ(x_0) and the spectrum of Z — depends on
 * Δ).  *out shares every table of `base` (P, L, e, the K1 scatter order and
 * twiddles: they live in base's plan_ws, which must outlive *out) and owns
 * only ζ, φ(x_0) and W, built in shift_ws (device, 256-B aligned, at least
 * qmc_shift_workspace_size(base) bytes ≈ 8m + 16L; caller-owned, must
 * outlive *out).  The result computes the same as qmc_plan_create_shifted
 * (N, z, phi, Δ) and is used like any plan (qmc_matmul / qmc_mean / ...);
 * free it with qmc_plan_destroy (base's tables are not touched).  base must
 * be a lattice plan (else QMC_EUNSUPPORTED); its own Δ is ignored.
 * Δ outside [0, 1) -> QMC_EINVAL_PHI.  Synchronises `stream`. */
int qmc_shift_workspace_size(qmc_plan_t base, size_t* shift_bytes);
int qmc_plan_shift(qmc_plan_t* out, qmc_plan_t base, double delta, void* shift_ws, size_t shift_ws_bytes,
                   void* stream);

/* Randomised-QMC estimate from R replicates (the R shifted rules above;
 * reading R28): means[r*ld + k], r < R, k < t (device) ->
 * mean_out[k] = (1/R) Σ_r means[r,k], summed in the fixed order r = 0..R-1
 * (bit-reproducible), and, if stderr_out is not NULL,
 * stderr_out[k] = sqrt(Σ_r (means[r,k] - mean_out[k])^2 / (R (R-1)))
 * (NaN for R = 1).  R >= 1, t >= 0, ld >= t, else QMC_EINVAL_DIM. */
int qmc_replicate_mean(const double* means, int64_t R, int64_t t, int64_t ld, double* mean_out,
                       double* stderr_out, void* stream);

/* Polynomial lattice over F_2 (PAPER.md:456-459 Remark; reading R2/R3):
 * p has bit D set, 2 <= D <= 24, and must be primitive (checked on the
 * device: x has order 2^D-1); q_host: s values in [1, 2^D-1] (integer
 * encoding, bit i = coefficient of x^i).  N = 2^D points, m = 2^D-1. */
int qmc_plan_create_poly(qmc_plan_t* out, int D, uint64_t p, int64_t s, const int64_t* q_host,
                         int phi, void* plan_ws, size_t plan_ws_bytes, void* stream);

/* X = Y·A (device pointers; X row-major, ldx >= t).  t >= 0 columns;
 * t = 0 is a no-op. */
int qmc_matmul(qmc_plan_t plan, const double* A, int64_t lda, int64_t t, double* X, int64_t ldx,
               void* call_ws, size_t call_ws_bytes, void* stream);

/* X = Y·A fused with f and the QMC mean.  out (device): t doubles for
 * IDENTITY/AFFINE/EXP (complete means of the local columns), N doubles for
 * ROWMEAN_RELU (partial row sums over the local columns).  X_or_null: if not
 * NULL, X (or c + X for AFFINE) is written as in qmc_matmul. */
int qmc_mean(qmc_plan_t plan, const double* A, int64_t lda, int64_t t, int f, double f_param,
             double* out, double* X_or_null, int64_t ldx, void* call_ws, size_t call_ws_bytes,
             void* stream);

/* After the (optional, caller-side) allreduce of qmc_mean's out over column
 * shards.  ROWMEAN_RELU: out[0] = (1/N) Σ_n max(0, reduced[n]/t_total), a
 * fixed-order device reduction.  Other f: copies the t_total means
 * (reduced → out, may alias).  Device pointers. */
int qmc_mean_finalize(qmc_plan_t plan, int f, const double* reduced, int64_t t_total, double* out,
                      void* stream);

/* The union of all Korobov lattice point sets (SURVEY
 * §8(f) NEXT #1): N_pset = (K-1)^2 points x_{n,g} = ({n g^j / K})_{j<s},
 * n, g = 1..K-1, K prime, in the conventional order row = (g-1)(K-1) + (n-1)
 * (reading R24).  X = Y_pset · A for a lattice plan with N = K and the p-set's
 * dimension s (its generating vector is not used): every block g is Z·P_g
 * with the plan's one circulant Z (Eq. Y_pset), so the
 * plan's spectrum, power and log tables serve all K-1 blocks, and the block
 * index is a grid dimension of one launch (column map e_{g,j} = j·L[g] mod
 * (K-1), computed on the device).  A: device, column-major s×t (lda >= s);
 * X: device, row-major (K-1)^2 × t (ldx >= t).  One-row plans only
 * (L1 = 1, i.e. K <= 4097, and s <= 2048): QMC_EUNSUPPORTED otherwise (the
 * caller then runs one lattice plan per block).  Asynchronous on `stream`. */
int qmc_pset_matmul(qmc_plan_t plan, const double* A, int64_t lda, int64_t t, double* X, int64_t ldx,
                    void* stream);

/* End-to-end entry with HOST buffers: copies A_host (pinned or pageable,
 * column-major s×t, lda) into A_dev (device, s*t doubles, ld = s) — batch by
 * batch of column pairs, each copy on the stream that then runs that batch,
 * so copies overlap kernels — runs qmc_mean (+ finalize), and copies the
 * result to out_host (1 double for
 * ROWMEAN_RELU, else t doubles); X_dev (device, ldx) receives X.  out_dev
 * (device) must hold max(N, t) doubles.  X_dev is row-major with ldx >= t.
 * Synchronises `stream`. */
int qmc_mean_host(qmc_plan_t plan, const double* A_host, int64_t lda, int64_t t, int f,
                  double f_param, double* out_host, double* A_dev, double* X_dev, int64_t ldx,
                  double* out_dev, void* call_ws, size_t call_ws_bytes, void* stream);

/* Experiment 2 of the paper: the
 * uniform 1-D ODE -(a u')' = g with a(x,y) = 2 + Σ_j y_j j^{-3/2} sin(2πjx),
 * K = M-1 hat functions.  Its stiffness matrices B(y_n) = A_0 + Σ_j y_{n,j}A_j
 * are tridiagonal; X (device, row-major N × ldx, ldx >=
 * 2K-1) holds, per QMC point n, the perturbations Σ_j y_{n,j} A_j as computed
 * by qmc_matmul: K diagonal entries then the K-1 entries (k, k+1) (B is
 * symmetric).  d0, e0: the diagonal and off-diagonal entries of A_0.
 * Solves B(y_n) û^(n) = ĝ for every n IN PLACE (X row n: û^(n) in its first
 * K slots afterwards; the other slots are scratch) by the Thomas algorithm
 * (one warp per 32 samples, lane = sample, 32-unknown tiles of the rows
 * staged through shared memory), and writes mean_out[k] = (1/N) Σ_n û_k^(n)
 * (PAPER.md:665-668), summed in increasing n.  rhs: device ĝ (K doubles) or
 * NULL for ĝ = (1, ..., 1).  B must be positive definite
 * (true for this ODE: a >= 2 - ζ(3/2)/2 > 0).  Asynchronous on `stream`. */
int qmc_tridiag_solve_mean(int64_t N, int64_t K, double d0, double e0, const double* rhs, double* X,
                           int64_t ldx, double* mean_out, void* stream);

/* Experiment 3 of the paper (SURVEY §8(f) NEXT
 * #3): the log-normal 1-D ODE, a(x,y) = exp(ψ_0 + Σ_j y_j ψ_j(x)), M hat
 * elements, equal-weight quadrature at the M element midpoints (reading
 * R25).  X (device, row-major N × ldx, ldx >= 2M-2) holds in its first M
 * slots θ_{n,i} = Σ_j y_{n,j} ψ_j(x_i) as computed by qmc_matmul (Θ = Y·Ψ,
 * Eq. fastB).  Forms B̂(y_n) on the fly — a_i = exp(ψ_0 + θ_i), diagonal
 * M (a_{k-1} + a_k), off-diagonal -M a_k (Eq. def:b nkl) — and solves
 * B̂ û = ĝ in place (û^(n) in the first M-1 slots of row n afterwards; slots
 * up to 2M-3 are scratch), one warp per 32 samples; mean_out[k] =
 * (1/N) Σ_n û_k^(n), summed in increasing n.  rhs: device ĝ (M-1 doubles) or
 * NULL for ĝ = 1.  Asynchronous on `stream`. */
int qmc_fe1d_lognormal_solve_mean(int64_t N, int64_t M, double psi0, const double* rhs, double* X,
                                  int64_t ldx, double* mean_out, void* stream);

/* One step of the component-by-component construction of z (SURVEY §8(f)
 * NEXT #4; fast CBC, cited but not restated by the paper):
 * criterion e² = -1 + (1/N) Σ_n Π_j (1 + γ_j 2π² B_2({n z_j/N})) (weighted
 * Korobov space, product weights, shift-averaged worst case).  crit (device,
 * N doubles): crit[z] = Σ_{n>=1} B_2({n z/N}) p_n, i.e. X of qmc_matmul for
 * the plan with generating vector (1, 2, ..., N-1), φ = QMC_PHI_BERNOULLI2 and
 * A = p_1..p_{N-1} (the fast product of this library; the n = 0 term is the
 * same for every z).  Picks z_d = argmin_{1 <= z <= zmax} crit[z] (smallest z
 * among equal values), stores it to z_out[d] (device int64) and updates p
 * (device, N doubles) to p_n (1 + γ 2π² B_2({n z_d/N})).  Start with p = 1;
 * zmax = 1 fixes z_1 = 1; zmax = (N-1)/2 uses the symmetry crit[z] =
 * crit[N-z].  Asynchronous on `stream`. */
int qmc_cbc_step(int64_t N, const double* crit, int64_t zmax, double gamma, double* p, int64_t* z_out,
                 int64_t d, void* stream);

/* Plan facts: info[0..11] = family, N, m, s, phi, generator (β or the
 * encoding of x = 2), L (FFT length; L = m or padded L >= 2m-1), L1, L2,
 * pairs per batch, D, p, then the row kernel's scatter-input layout:
 * bucket order (0), balanced (1) or dense (2), staged slots per pair,
 * chunks, slots per chunk; info[16] = slots of the direct scatter's first
 * rounds staged in shared memory (0: none), info[17] = SMs of the column
 * pass's green-context partition (0: green mode off, QMC_GREEN).  Host
 * pointer, >= 18 int64. */
int qmc_plan_info(qmc_plan_t plan, int64_t* info);

/* D2H copies of the plan tables for bit-exact tests (host buffers; any may
 * be NULL): gen[1]; P[m] (β^k mod N or x^k mod p); L[N] (L[0] = -1);
 * e[s] (e_j = c_j - 1); zeta[m] (ζ_k).  Synchronises the plan's stream. */
int qmc_plan_tables(qmc_plan_t plan, int64_t* gen, int32_t* P, int32_t* L, int32_t* e,
                    double* zeta);

/* Kernels this library has launched since it was loaded (all entry points). */
int64_t qmc_launch_count(void);

/* Build flags of this library: bit 0 = the checked build (-DQMC_CHECK:
 * device-side bounds checks of the computed indices, tools/check_build.sh),
 * bit 1 = phase timing (-DQMC_PHASE_TIMING).  0 for the product build. */
int qmc_build_flags(void);

/* Per-kernel-class timing for roofline reporting.  qmc_profile_enable(1)
 * makes every later hot-path call record CUDA events on its stream around
 * each launch class (k_pack, k_rows, k_cols, k_gather, k_reduce,
 * k_finalize — qmc_profile_class_name(i) for i = 0..5; k_pack and k_gather
 * are retired classes and stay empty).  qmc_profile_read
 * waits for those events and returns, per class i < n, the number of
 * timed launches (one "launch" of k_rows = the launch for one batch) and
 * their summed device time in ms (host arrays of n entries); it then clears
 * the record.  Not thread-safe; for benchmarking only. */
int qmc_profile_enable(int on);
int qmc_profile_read(int64_t* launches, double* ms, int n);
const char* qmc_profile_class_name(int i);

void qmc_plan_destroy(qmc_plan_t plan);
const char* qmc_strerror(int code);

#ifdef __cplusplus
}
#endif

#endif /* QMC_H */
