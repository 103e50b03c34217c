// plan.cu — plan construction of libqmc: host validation and the integer /
// spectral plan kernels (sm_100a).
//
//   a0  validate N prime (or p of degree D), factor m            host
//   a0  β = smallest primitive root (R1)      k_find_generator
//       or check x generates F_2[x]/p (p primitive, R2)          k_check_poly
//   a1  P[k] = β^k mod N  /  x^k mod p      k_pow_table
//   a2  L[P[k]] = k, L[0] = -1      k_log_table
//   a3  e_j = L[z_j] = c_j - 1; buckets by e_j mod L2           k_colmap, k_bucket_*
//       R[n] = (m - L[n]) mod m  (conventional row n is reordered row R[n])
//   a4  ζ_k = φ(u(P[k])); W = DFT_L(K)/L     k_zeta, k_spectrum_rows
//
// The plan is excluded from the paper's timings and from
// bench.py's timed region.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <queue>
#include <vector>

#include "fft.cuh"
#include "qmc_internal.cuh"
#include "rowcfg.cuh"

namespace qmc {

std::atomic<int64_t> g_launches{0};

// ------------------------------------------------------------------ profiling
namespace {
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[KC_COUNT];
  cudaEvent_t open[KC_COUNT] = {};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
Prof g_prof;
}  // namespace

void prof_begin(int kc, cudaStream_t st) {
  if (!g_prof.on) return;
  cudaEvent_t e = g_prof.get();
  cudaEventRecord(e, st);
  g_prof.open[kc] = e;
}

void prof_end(int kc, cudaStream_t st) {
  if (!g_prof.on || !g_prof.open[kc]) return;
  cudaEvent_t e = g_prof.get();
  cudaEventRecord(e, st);
  g_prof.ev[kc].push_back({g_prof.open[kc], e});
  g_prof.open[kc] = nullptr;
}

// ------------------------------------------------------------------ host
static bool host_is_prime(int64_t n) {
  if (n < 2) return false;
  if (n % 2 == 0) return n == 2;
  for (int64_t d = 3; d * d <= n; d += 2)
    if (n % d == 0) return false;
  return true;
}

static std::vector<int64_t> host_prime_factors(int64_t m) {
  std::vector<int64_t> q;
  for (int64_t d = 2; d * d <= m; ++d)
    if (m % d == 0) {
      q.push_back(d);
      while (m % d == 0) m /= d;
    }
  if (m > 1) q.push_back(m);
  return q;
}

static bool smooth235(int64_t x) {
  for (int q : {2, 3, 5})
    while (x % q == 0) x /= q;
  return x == 1;
}

bool choose_split(int64_t m, int64_t s, Split* out) {
  int64_t cap_env = 0;
  if (const char* ev = getenv("QMC_L2_CAP")) cap_env = strtol(ev, nullptr, 10);  // tuning override
  auto try_len = [&](int64_t len) -> bool {
    // rows of 4096 unless the columns would then exceed 16 (one register
    // stage in K2) or s > 4096 (keep buckets small): then rows of 8192
    int64_t cap = s > 4096 ? 8192 : 4096;
    if (cap == 4096 && len % 8192 == 0 && len / 4096 > 16) cap = 8192;
    if (cap_env >= 16) cap = cap_env;
    int64_t l2 = 1;
    while (len % (l2 * 2) == 0 && l2 * 2 <= cap) l2 *= 2;
    if (l2 < 16 || (l2 < 256 && l2 != len)) return false;  // rows of >= 256, or one short row
    int64_t l1 = len / l2;
    if (!k2_split_R(l1)) return false;  // a column length K2 instantiates
    out->L = len;
    out->L1 = l1;
    out->L2 = l2;
    return true;
  };
  if (m >= 64 && try_len(m)) {
    out->padded = false;
    return true;
  }
  for (int64_t len = 2 * m - 1; len <= (int64_t(1) << 26); ++len)
    if (smooth235(len) && try_len(len)) {
      out->padded = true;
      return true;
    }
  return false;
}

// the dense first pass is taken whatever the bucket sizes: the balanced
// order is not tried (s > 8·L2), a' is at least half full and the K2 split
// exists (create_common decides k1_dense the same way)
static bool k1_dense_certain(int64_t s, const Split& sp) {
  return !k1_try_balanced(s, sp.L2) && 2 * s >= sp.L && k2_split_R(sp.L1) > 0 && !getenv("QMC_K1_HEADS") &&
         !getenv("QMC_NO_DENSE");
}

PlanLayout plan_layout(int64_t N, int64_t m, int64_t s, const Split& sp) {
  PlanLayout l;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  l.off_scal = take(16 * 8);
  l.off_P = take(size_t(m) * 4);
  l.off_L = take(size_t(N) * 4);
  l.off_R = take(size_t(N) * 4);
  l.off_e = take(size_t(s) * 4);
  l.off_bstart = take(size_t(sp.L2 + 1) * 4);
  l.off_bent = take(size_t(s) * 16);
  const int64_t s1 = k1_s1max(s, sp.L2, sp.L);
  l.off_e2q = take(size_t(s1) * 4 + 16);
  l.off_occ = take(size_t(sp.L2 / 32 + 1) * 4);
  l.off_cursor = take(size_t(sp.L2) * 4);
  l.off_zeta = take(size_t(m) * 8);
  l.off_W = take(size_t(sp.L) * 16);
  l.off_tw1 = take(size_t(sp.L1) * 16);
  l.off_tw2 = take(size_t(sp.L2) * 16);
  l.off_twL = take(size_t(sp.L2) * 16);
  l.off_tw16 = take(size_t(16 * sp.L1) * 16);
  // per-entry twiddles of the sparse first pass; none when the plan is
  // certain to take the dense first pass (create_common: k1_dense)
  l.off_twj = take(k1_dense_certain(s, sp) ? 0 : size_t(sp.L1) * size_t(s1) * 16);
  l.off_jq = take(size_t(s1) * 4);
  l.off_k1c = take(size_t(2 * s1 + 4) * 4);
  l.off_k2n = take(size_t(sp.L) * 4);
  l.off_tmp = take(size_t(s + 64 + 2) * 8);  // plan-time scratch: z, factors of m, flag
  l.total = o;
  return l;
}

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t n) { return (a * b) % n; }

__device__ uint64_t powmod(uint64_t b, uint64_t e, uint64_t n) {
  uint64_t r = 1 % n;
  b %= n;
  while (e) {
    if (e & 1) r = mulmod(r, b, n);
    b = mulmod(b, b, n);
    e >>= 1;
  }
  return r;
}

// a·b mod p in F_2[x], deg a, deg b < D (Horner, keeps the partial < 2^D)
__device__ __forceinline__ uint64_t gf2_mulmod(uint64_t a, uint64_t b, uint64_t p, int D) {
  uint64_t r = 0;
  for (int i = D - 1; i >= 0; --i) {
    r <<= 1;
    if ((r >> D) & 1) r ^= p;
    if ((b >> i) & 1) r ^= a;
  }
  return r;
}

__device__ uint64_t gf2_powmod(uint64_t b, uint64_t e, uint64_t p, int D) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = gf2_mulmod(r, b, p, D);
    b = gf2_mulmod(b, b, p, D);
    e >>= 1;
  }
  return r;
}

// 2^D · v_D(r/p): digits of r(x)/p(x) by long division (reading R3)
__device__ __forceinline__ int64_t gf2_vd_index(uint64_t r, uint64_t p, int D) {
  uint64_t idx = 0;
  for (int i = 0; i < D; ++i) {
    uint64_t t = (r >> (D - 1)) & 1;
    r = (r << 1) ^ (t ? p : 0);
    idx = (idx << 1) | t;
  }
  return int64_t(idx);
}

// φ(i/N) (INVNORM_MID per reading R6)
// φ at the grid point i/N, shifted by the equal shift Δ (
// Δ = 0: the unshifted rule).  INVNORM_MID composes its own midpoint shift
// 1/(2N) with Δ: Φ^{-1}(frac(i/N + 1/(2N) + Δ)).
__device__ __forceinline__ double phi_eval(int phi, int64_t i, int64_t N, double delta) {
  if (delta == 0.0) {
    const double u = double(i) / double(N);
    switch (phi) {
      case QMC_PHI_IDENTITY: return u;
      case QMC_PHI_SHIFT_HALF: return u - 0.5;
      case QMC_PHI_TENT: return 1.0 - fabs(2.0 * u - 1.0);
      case QMC_PHI_BERNOULLI2: return u * u - u + 1.0 / 6.0;
      default: return normcdfinv(double(2 * i + 1) / double(2 * N));
    }
  }
  double u = double(i) / double(N) + (phi == QMC_PHI_INVNORM_MID ? 0.5 / double(N) : 0.0) + delta;
  u -= floor(u);
  switch (phi) {
    case QMC_PHI_IDENTITY: return u;
    case QMC_PHI_SHIFT_HALF: return u - 0.5;
    case QMC_PHI_TENT: return 1.0 - fabs(2.0 * u - 1.0);
    case QMC_PHI_BERNOULLI2: return u * u - u + 1.0 / 6.0;
    default: return normcdfinv(u);
  }
}

// ------------------------------------------------------------------ plan kernels
__global__ void k_find_generator(int64_t N, int64_t base, const int64_t* __restrict__ qf, int nq,
                                 unsigned long long* best) {
  const int64_t beta = base + blockIdx.x * blockDim.x + threadIdx.x;
  if (beta >= N) return;
  const uint64_t m = uint64_t(N - 1);
  for (int i = 0; i < nq; ++i)
    if (powmod(uint64_t(beta), m / uint64_t(qf[i]), uint64_t(N)) == 1) return;
  atomicMin(best, (unsigned long long)beta);
}

// flags bit0: x^m != 1; bit1: some x^{m/q} == 1  (p primitive iff flags == 0)
__global__ void k_check_poly(uint64_t p, int D, const int64_t* __restrict__ qf, int nq,
                             unsigned long long* flags) {
  const int i = threadIdx.x;
  const uint64_t m = (uint64_t(1) << D) - 1;
  if (i == 0) {
    if (gf2_powmod(2, m, p, D) != 1) atomicOr(flags, 1ull);
  } else if (i <= nq) {
    if (gf2_powmod(2, m / uint64_t(qf[i - 1]), p, D) == 1) atomicOr(flags, 2ull);
  }
}

__global__ void k_pow_table(int family, int64_t N, uint64_t p, int D, int64_t gen, int64_t m,
                            int32_t* __restrict__ P) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  P[k] = family == QMC_FAMILY_LATTICE ? int32_t(powmod(uint64_t(gen), uint64_t(k), uint64_t(N)))
                                      : int32_t(gf2_powmod(2, uint64_t(k), p, D));
}

__global__ void k_fill_i32(int32_t* __restrict__ a, int64_t n, int32_t v) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void k_log_scatter(const int32_t* __restrict__ P, int64_t m, int32_t* __restrict__ L) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) L[P[k]] = int32_t(k);
}

__global__ void k_colmap(const int64_t* __restrict__ z, int64_t s, const int32_t* __restrict__ L,
                         int32_t* __restrict__ e) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < s) e[j] = L[z[j]];
}

// Stable counting sort of j by e2 = e_j mod L2 (one CTA; plan time only):
// bent[q] = {j, e_j, e2, end of the bucket if q is its first entry else -1};
// e2q[q] = e2 | (bucket size << 13) if q is the first entry of its bucket,
// else e2 (K1 stages e2q; L2 <= 8192); occ = bitmap of the nonempty buckets.
// Buckets of the column map by e2 = e_j mod L2, entries of a bucket in
// increasing j (a stable counting sort, in parallel):
//   count -> inclusive scan (bstart) -> placement by atomic cursors (any order
//   within a bucket) -> per bucket, sort its j's (insertion sort) and write
//   bent / e2q / occ.  The result does not depend on the atomic order.
__global__ void k_bucket_count(const int32_t* __restrict__ e, int64_t s, int L2, int32_t* __restrict__ bstart) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < s) atomicAdd(&bstart[(e[j] & (L2 - 1)) + 1], 1);
}

// bstart[0..L2] (bstart[0] = 0) -> inclusive prefix sums; cursor[i] = bstart[i]
__global__ void __launch_bounds__(1024) k_bucket_scan(int32_t* __restrict__ bstart, int L2,
                                                      int32_t* __restrict__ cursor) {
  __shared__ int32_t part[1024];
  const int n = L2 + 1, per = (n + 1023) / 1024;
  const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
  int32_t run = 0;
  for (int i = i0; i < i1; ++i) {
    run += bstart[i];
    bstart[i] = run;
  }
  part[threadIdx.x] = run;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int w = 0; w < 1024; ++w) {
      const int32_t v = part[w];
      part[w] = acc;
      acc += v;
    }
  }
  __syncthreads();
  const int32_t off = part[threadIdx.x];
  for (int i = i0; i < i1; ++i) {
    bstart[i] += off;
    if (i < L2) cursor[i] = bstart[i];
  }
}

__global__ void k_bucket_place(const int32_t* __restrict__ e, int64_t s, int L2, int32_t* __restrict__ cursor,
                               int32_t* __restrict__ slot_j) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < s) slot_j[atomicAdd(&cursor[e[j] & (L2 - 1)], 1)] = int32_t(j);
}

// one thread per bucket b: e2q[lo, hi) holds its j's on entry, its codes on exit
__global__ void k_bucket_finish(const int32_t* __restrict__ e, int L2, const int32_t* __restrict__ bstart,
                                int32_t* __restrict__ e2q, int4* __restrict__ bent, uint32_t* __restrict__ occ) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= L2) return;
  const int lo = bstart[b], hi = bstart[b + 1];
  for (int i = lo + 1; i < hi; ++i) {  // insertion sort by j
    const int32_t v = e2q[i];
    int k = i - 1;
    while (k >= lo && e2q[k] > v) {
      e2q[k + 1] = e2q[k];
      --k;
    }
    e2q[k + 1] = v;
  }
  for (int pos = lo; pos < hi; ++pos) {
    const int j = e2q[pos];
    bent[pos] = make_int4(j, e[j], b, pos == lo ? hi : -1);
  }
  // the size field only bounds the head's sum inside its chunk (at most 2048
  // entries), so capping it at 2^18 - 1 keeps the code exact for any bucket
  const int len = min(hi - lo, (1 << 18) - 1);
  for (int pos = lo; pos < hi; ++pos) e2q[pos] = pos == lo ? b | (len << 13) : b;
  if (hi > lo) atomicOr(&occ[b >> 5], 1u << (b & 31));
}

__global__ void k_rtable(const int32_t* __restrict__ L, int64_t N, int64_t m, int32_t* __restrict__ R) {
  const int64_t n = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n >= N) return;
  R[n] = n == 0 ? -1 : int32_t((m - L[n]) % m);
}

__global__ void k_zeta(int family, int phi, double delta, int64_t N, uint64_t p, int D, int64_t m,
                       const int32_t* __restrict__ P, double* __restrict__ zeta, double* __restrict__ scal) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k == 0) scal[0] = phi_eval(phi, 0, N, delta);
  if (k >= m) return;
  const int64_t r = P[k];
  const int64_t idx = family == QMC_FAMILY_LATTICE ? r : gf2_vd_index(uint64_t(r), p, D);
  zeta[k] = phi_eval(phi, idx, N, delta);
}

// tw[k] = ω_n^k = exp(-2πi k/n), k < count
__global__ void k_twiddles(double2* __restrict__ tw, int64_t n, int64_t count) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= count) return;
  double sv, cv;
  sincospi(2.0 * double(k) / double(n), &sv, &cv);
  tw[k] = make_double2(cv, -sv);
}

// k2n[(bx·L1 + e1)·kUB + c] = conventional row n = P[(m - i) mod m] of the
// reordered row i = L2·e1 + kUB·bx + c, -1 when i >= m
// (zero-padded length): the output rows of a K2 tile (one U column block of
// kUB columns e2) in the order of its U block, one contiguous run per tile
__global__ void k_k2rows(const int32_t* __restrict__ P, int64_t m, int64_t L, int L1, int L2,
                         int32_t* __restrict__ k2n) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= L) return;
  const int64_t bx = idx / (int64_t(L1) * kUB), rem = idx % (int64_t(L1) * kUB);
  const int64_t e1 = rem / kUB, c2 = kUB * bx + rem % kUB;
  const int64_t i = int64_t(L2) * e1 + c2;
  k2n[idx] = (c2 < L2 && i < m) ? P[i == 0 ? 0 : m - i] : -1;
}

// twj[f1·S1 + q] = ω_{L1}^{(e1_j·f1) mod L1}, e1_j = e_j div L2, for the
// column j = jq[q] of slot q of the K1 order (0 for padding slots)
__global__ void k_twj(const int32_t* __restrict__ jq, const int32_t* __restrict__ e, int64_t S1, int64_t L, int L1,
                      int NT, double2* __restrict__ twj) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= S1 * L1) return;
  const int64_t f1 = i / S1, q = i % S1;
  const int j = jq[q];
  if (j < 0) {
    twj[i] = make_double2(0.0, 0.0);
    return;
  }
  // ω_L^{L2 e1 f1} = ω_{L1}^{(e1 f1) mod L1}, e1 = e_j div L2: the part of
  // ω_L^{e_j f1} that differs between the entries of a bucket; the bucket's
  // common factor ω_L^{e2 f1} is applied by K1 to the summed row
  // (ω_{16 L1}^{q f1} per register, ω_L^{t f1} in the first row-FFT stage)
  const int64_t L2 = L / L1;
  const int64_t x = ((e[j] / L2) * f1) % L1;
  (void)NT;
  double sv, cv;
  sincospi(2.0 * double(x) / double(L1), &sv, &cv);
  twj[i] = make_double2(cv, -sv);
}

// Slots of one K1 chunk: K1 reads its scatter input straight from global
// memory, so a chunk is bounded only by the balanced order's overflow slots
// (kK1Ovf per chunk, 16 pieces per bucket); one chunk normally suffices.
static int k1_slot_budget(int64_t /*L2*/) { return 1 << 24; }

// K1 "balanced" order of the scatter input (pipeline.cu k1_item).  Buckets
// e2 are cut into chunks of whole buckets.  In a chunk of n entries, with
// M = ⌈n / NT⌉ (NT threads of the row CTA), every bucket is cut into pieces
// of at most M entries (j order kept); pieces go, largest first, to the
// least-loaded thread, whose entries sit at slots base + i·NT + tid.  The
// scatter of a chunk is then one pass without divergence, each thread
// keeping a running sum per piece.  A bucket's first piece sums into its own
// row entry, later pieces into overflow slots, added after a barrier by
// fix-up records, in piece order.  Padding slots have no column.  Returns
// false when no chunking fits the staging budget (K1 then uses the
// bucket-order heads scatter).
static bool k1_balanced_order(const std::vector<int32_t>& hb, const std::vector<int4>& hbent, int64_t L2, int NT,
                              int budget, int64_t s1max, std::vector<int32_t>& jq, std::vector<int32_t>& code,
                              std::vector<int32_t>& cs, std::vector<int32_t>& cr, int& chmax) {
  struct Piece {
    int q0, len, v;
  };
  using Load = std::pair<int, int>;  // (entries, thread)
  for (size_t q = 0; q < hbent.size(); ++q)  // e1 must fit the code field (L1 <= 512)
    if (hbent[q].y / L2 >= 512) return false;
  for (int64_t target = budget; target >= NT; target = target * 3 / 4) {
    jq.clear();
    code.clear();
    cs.assign(1, 0);
    cr.clear();
    chmax = 0;
    bool ok = true;
    for (int64_t b = 0; b < L2 && ok;) {
      int64_t e = b + 1;
      while (e < L2 && hb[e + 1] - hb[b] <= target) ++e;
      const int64_t n = hb[e] - hb[b];
      const int M = int(std::max<int64_t>(1, (n + NT - 1) / NT));
      std::vector<Piece> pc;
      std::vector<int32_t> rec;
      int ovf = 0;
      for (int64_t x = b; x < e && ok; ++x) {
        const int sz = hb[x + 1] - hb[x];
        const int np = (sz + M - 1) / M;
        for (int k = 0; k < np; ++k)
          pc.push_back({hb[x] + k * M, std::min(M, sz - k * M), k == 0 ? int(x) : int(L2) + 1 + ovf + k - 1});
        if (np > 1) {
          if (ovf + np - 1 > kK1Ovf || np - 1 > 15) ok = false;
          rec.push_back(int(x) | (ovf << 14) | ((np - 1) << 20));
          ovf += np - 1;
        }
      }
      if (!ok) break;
      std::stable_sort(pc.begin(), pc.end(), [](const Piece& u, const Piece& v) { return u.len > v.len; });
      std::vector<std::vector<Piece>> own(NT);
      std::priority_queue<Load, std::vector<Load>, std::greater<Load>> h;
      for (int t = 0; t < NT; ++t) h.push({0, t});
      int mr = 0;
      for (const Piece& p : pc) {
        const Load l = h.top();
        h.pop();
        own[l.second].push_back(p);
        h.push({l.first + p.len, l.second});
        mr = std::max(mr, l.first + p.len);
      }
      const int64_t nreg = (int64_t(mr) * NT + 3) / 4 * 4;  // chunk starts stay 16-byte aligned
      const int64_t slots = nreg + (int64_t(rec.size()) + 3) / 4 * 4;
      if (slots > budget || int64_t(jq.size()) + slots > s1max) {
        ok = false;
        break;
      }
      const size_t base = jq.size();
      jq.resize(base + slots, -1);
      code.resize(base + nreg, int(L2) | kK1First);
      code.insert(code.end(), rec.begin(), rec.end());
      code.resize(base + slots, int(L2));  // no-op records
      for (int t = 0; t < NT; ++t) {
        int i = 0;
        for (const Piece& p : own[t])
          for (int k = 0; k < p.len; ++k, ++i) {
            const size_t slot = base + size_t(i) * NT + t;
            jq[slot] = hbent[p.q0 + k].x;
            // e1 = e_j div L2 selects the scatter twiddle ω_{L1}^{e1 f1} (K1)
            code[slot] = p.v | (k == 0 ? kK1First : 0) | int((hbent[p.q0 + k].y / L2) << kK1E1Shift);
          }
      }
      cr.push_back(int(nreg));
      cs.push_back(int(jq.size()));
      chmax = std::max<int>(chmax, int(slots));
      b = e;
    }
    if (ok) return true;
  }
  return false;
}

// W[f1*L2 + f2] = DFT_L(K)[f1 + L1·f2] / L with the correlation kernel
// K[d] = ζ[(-d) mod m] for d < m, K[L-d'] = ζ[d'] for 0 < d' < m (padded),
// 0 otherwise.  Four-step: T[f1,e2] = Σ_{e1} K[L2 e1 + e2] ω_L^{(L2 e1+e2) f1}
// evaluated directly, then the length-L2 row FFT over e2.
template <int L2>
__global__ void __launch_bounds__(RowThreads<L2>::value)
    k_spectrum_rows(const double* __restrict__ zeta, int64_t m, int64_t L, int L1,
                    const double2* __restrict__ tw1, const double2* __restrict__ twL,
                    const double2* __restrict__ tw2, double2* __restrict__ W) {
  extern __shared__ double2 S[];
  constexpr int NT = RowThreads<L2>::value;
  const int f1 = blockIdx.x;
  for (int e2 = threadIdx.x; e2 < L2; e2 += NT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int e1 = 0; e1 < L1; ++e1) {
      const int64_t d = int64_t(L2) * e1 + e2;
      double kv = 0.0;
      if (d < m) kv = zeta[(m - d) % m];
      else if (d > L - m) kv = zeta[L - d];
      if (kv != 0.0) {
        const int64_t x = (d * f1) % L;
        const double2 w = cmul(tw1[x / L2], twL[x % L2]);
        acc.x = fma(kv, w.x, acc.x);
        acc.y = fma(kv, w.y, acc.y);
      }
    }
    S[swz(e2)] = acc;
  }
  __syncthreads();
  row_fft<L2, -1>(S, tw2);
  // stored in K1's register order: slot r·NTk + t holds frequency f2 =
  // dif_freq(t, r) (NTk = L2/16 threads of the row kernel)
  const double inv = 1.0 / double(L);
  constexpr int NTk = L2 / 16;
  for (int i = threadIdx.x; i < L2; i += NT) {
    const double2 v = S[swz(dif_freq<L2>(i % NTk, i / NTk))];
    W[int64_t(f1) * L2 + i] = make_double2(v.x * inv, v.y * inv);
  }
}

template <int L2>
static int launch_spectrum(const qmc_plan* pl) {
  const size_t smem = size_t(L2) * sizeof(double2);
  cudaFuncSetAttribute(k_spectrum_rows<L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_spectrum_rows<L2><<<unsigned(pl->sp.L1), RowThreads<L2>::value, smem, pl->stream>>>(
      pl->d_zeta, pl->m, pl->sp.L, int(pl->sp.L1), pl->d_tw1, pl->d_twL, pl->d_tw2, pl->d_W);
  QMC_LAUNCHED();
  return QMC_OK;
}

static int spectrum_dispatch(const qmc_plan* pl) {
  switch (pl->sp.L2) {
    case 16: return launch_spectrum<16>(pl);
    case 32: return launch_spectrum<32>(pl);
    case 64: return launch_spectrum<64>(pl);
    case 128: return launch_spectrum<128>(pl);
    case 256: return launch_spectrum<256>(pl);
    case 512: return launch_spectrum<512>(pl);
    case 1024: return launch_spectrum<1024>(pl);
    case 2048: return launch_spectrum<2048>(pl);
    case 4096: return launch_spectrum<4096>(pl);
    case 8192: return launch_spectrum<8192>(pl);
  }
  return QMC_EINVAL_N;
}

static unsigned blocks(int64_t n, int b) { return unsigned((n + b - 1) / b); }

// ------------------------------------------------------------------ create
static int validate_family(int family, int64_t N_or_D, int64_t s, int64_t* N, int64_t* m) {
  if (s < 1 || s > (int64_t(1) << 30)) return QMC_EINVAL_DIM;
  if (family == QMC_FAMILY_LATTICE) {
    if (N_or_D < 3 || N_or_D >= (int64_t(1) << 31) || !host_is_prime(N_or_D)) return QMC_EINVAL_N;
    *N = N_or_D;
    *m = N_or_D - 1;
  } else if (family == QMC_FAMILY_POLY) {
    if (N_or_D < 2 || N_or_D > 24) return QMC_EINVAL_POLY;
    *N = int64_t(1) << N_or_D;
    *m = *N - 1;
  } else {
    return QMC_EINVAL_N;
  }
  return QMC_OK;
}

// the plan's internal streams: two overlap consecutive batches when the
// column pass is a persistent pipelined kernel (k_cols_pipe, k_cols_pipe2:
// L1 <= 192); with the non-persistent k_cols_x (L1 = 256) the overlap
// measured slower, so such plans use the caller's stream (run() further
// restricts the two streams to calls where they overlap something)
// Green-context SM partitions (driver API through cudaGetDriverEntryPoint, so
// libqmc.so links no libcuda): the device's SMs split into groups of 8; the
// last ceil(G/8) groups form partition 1, the rest (and the remainder)
// partition 0.  Created once per (device, G) and kept for the process.
struct GreenParts {
  int dev = -1, G = 0, ok = 0;
  CUgreenCtx g[2] = {nullptr, nullptr};
  int nsm[2] = {0, 0};
};
typedef CUresult (*PFN_getRes)(CUdevice, CUdevResource*, CUdevResourceType);
typedef CUresult (*PFN_split)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
typedef CUresult (*PFN_desc)(CUdevResourceDesc*, CUdevResource*, unsigned);
typedef CUresult (*PFN_gctx)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
typedef CUresult (*PFN_gstream)(CUstream*, CUgreenCtx, unsigned, int);
template <typename F>
static bool drv_fn(const char* name, F* f) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    return false;
  *f = reinterpret_cast<F>(p);
  return true;
}
static std::mutex g_green_mu;
static GreenParts g_green[8];
static const GreenParts* green_parts(int G) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 8) return nullptr;
  std::lock_guard<std::mutex> lk(g_green_mu);
  GreenParts& gp = g_green[dev];
  if (gp.dev == dev && gp.G == G) return gp.ok ? &gp : nullptr;
  if (gp.dev == dev) return nullptr;  // one partitioning per device and process
  gp.dev = dev;
  gp.G = G;
  PFN_getRes getRes;
  PFN_split split;
  PFN_desc desc;
  PFN_gctx gctx;
  if (!drv_fn("cuDeviceGetDevResource", &getRes) || !drv_fn("cuDevSmResourceSplitByCount", &split) ||
      !drv_fn("cuDevResourceGenerateDesc", &desc) || !drv_fn("cuGreenCtxCreate", &gctx))
    return nullptr;
  CUdevResource all, rem;
  unsigned ng = 0;
  if (getRes(CUdevice(dev), &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(nullptr, &ng, &all, nullptr, 0, 8) != CUDA_SUCCESS || ng < 2)
    return nullptr;
  std::vector<CUdevResource> grp(ng);
  memset(&rem, 0, sizeof(rem));
  if (split(grp.data(), &ng, &all, &rem, 0, 8) != CUDA_SUCCESS) return nullptr;
  const unsigned n1 = unsigned(std::min<int>((G + 7) / 8, int(ng) - 1));
  std::vector<CUdevResource> r0(grp.begin(), grp.end() - n1), r1(grp.end() - n1, grp.end());
  if (rem.sm.smCount > 0) r0.push_back(rem);
  CUdevResourceDesc d0, d1;
  if (desc(&d0, r0.data(), unsigned(r0.size())) != CUDA_SUCCESS ||
      desc(&d1, r1.data(), unsigned(r1.size())) != CUDA_SUCCESS ||
      gctx(&gp.g[0], d0, CUdevice(dev), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      gctx(&gp.g[1], d1, CUdevice(dev), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return nullptr;
  for (const CUdevResource& r : r0) gp.nsm[0] += int(r.sm.smCount);
  for (const CUdevResource& r : r1) gp.nsm[1] += int(r.sm.smCount);
  gp.ok = 1;
  return &gp;
}

// green mode: the two internal streams on the two SM partitions, and the
// per-set hand-off events
static bool plan_green_streams(qmc_plan* pl, int G) {
  const GreenParts* gp = green_parts(G);
  PFN_gstream gstream;
  if (!gp || !drv_fn("cuGreenCtxStreamCreate", &gstream)) return false;
  CUstream s0 = nullptr, s1 = nullptr;
  if (gstream(&s0, gp->g[0], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) return false;
  if (gstream(&s1, gp->g[1], CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    cudaStreamDestroy(cudaStream_t(s0));
    return false;
  }
  pl->ist[0] = cudaStream_t(s0);
  pl->ist[1] = cudaStream_t(s1);
  bool ok = cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&pl->ev_join[0], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&pl->ev_join[1], cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; i < 2 && ok; ++i)
    ok = cudaEventCreateWithFlags(&pl->ev_ready[i], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&pl->ev_free[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) return false;  // (a plan without its events is not created: create_common fails on nstreams)
  pl->gsm[0] = gp->nsm[0];
  pl->gsm[1] = gp->nsm[1];
  pl->green = 1;
  return true;
}

static void plan_streams(qmc_plan* pl) {
  pl->nstreams = 1;
  pl->green = 0;
  pl->mu = new (std::nothrow) std::mutex();
  if (const char* gv = getenv("QMC_GREEN")) {  // K2 partition of G SMs (multiple of 8)
    const int G = int(strtol(gv, nullptr, 10));
    if (G > 0 && pl->mu && plan_green_streams(pl, G)) {
      pl->nstreams = 2;
      cudaGetLastError();
      return;
    }
    cudaGetLastError();
  }
  const char* one = getenv("QMC_ONE_STREAM");
  const bool want2 = one ? one[0] != '1' : pl->sp.L1 <= 192;
  if (want2 && pl->mu &&
      cudaStreamCreateWithFlags(&pl->ist[0], cudaStreamNonBlocking) == cudaSuccess &&
      cudaStreamCreateWithFlags(&pl->ist[1], cudaStreamNonBlocking) == cudaSuccess &&
      cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
      cudaEventCreateWithFlags(&pl->ev_join[0], cudaEventDisableTiming) == cudaSuccess &&
      cudaEventCreateWithFlags(&pl->ev_join[1], cudaEventDisableTiming) == cudaSuccess)
    pl->nstreams = 2;
  cudaGetLastError();
}

static int create_common(qmc_plan_t* out, int family, int64_t N_or_D, uint64_t p, double delta, int64_t s,
                         const int64_t* z_host, int phi, void* plan_ws, size_t plan_ws_bytes,
                         void* stream) {
  if (!out) return QMC_ENULL;
  *out = nullptr;
  if (!z_host || !plan_ws) return QMC_ENULL;
  if (phi < QMC_PHI_IDENTITY || phi > QMC_PHI_BERNOULLI2) return QMC_EINVAL_PHI;
  int64_t N, m;
  int rc = validate_family(family, N_or_D, s, &N, &m);
  if (rc) return rc;
  if (family == QMC_FAMILY_POLY) {
    const int D = int(N_or_D);
    if ((p >> D) != 1 || !(p & 1)) return QMC_EINVAL_POLY;
  }
  for (int64_t j = 0; j < s; ++j)
    if (z_host[j] < 1 || z_host[j] > m) return QMC_EINVAL_Z;
  Split sp;
  if (!choose_split(m, s, &sp)) return QMC_EINVAL_N;
  const PlanLayout lay = plan_layout(N, m, s, sp);
  if (plan_ws_bytes < lay.total || (uintptr_t(plan_ws) % kAlign)) return QMC_EWORKSPACE;

  qmc_plan* pl = new (std::nothrow) qmc_plan();
  if (!pl) return QMC_ECUDA;
  pl->family = family;
  pl->phi = phi;
  pl->delta = delta;
  pl->N = N;
  pl->m = m;
  pl->s = s;
  pl->D = family == QMC_FAMILY_POLY ? int(N_or_D) : 0;
  pl->p = p;
  pl->sp = sp;
  pl->stream = (cudaStream_t)stream;
  pl->ws = (char*)plan_ws;
  pl->ws_bytes = plan_ws_bytes;
  {
    // Batch of column pairs (measured on B200): enough K1 items
    // (L1 per pair) for ~16384 per launch — persistent CTAs then keep several
    // items each and the long launches amortise their tails — with U (16·L
    // bytes per pair) at least ~128 MB and at most ~768 MB per scratch set;
    // a multiple of the K2 pair group (16, 8 or 4 pairs).  Per call the
    // batch is further capped at half the call's pairs (run() / call_layout),
    // so that two batches can overlap on the two internal streams.
    const int64_t per_pair = 16 * sp.L;
    int64_t bp = std::max<int64_t>((int64_t(128) << 20) / per_pair, (16384 + sp.L1 - 1) / sp.L1);
    bp = std::max<int64_t>(1, std::min<int64_t>(bp, (int64_t(768) << 20) / per_pair));
    bp = std::min<int64_t>(bp, 4096);
    bp = bp >= 16 ? bp / 16 * 16 : bp >= 8 ? 8 : bp >= 4 ? 4 : bp;
    pl->batch_pairs = bp;
    // Device calls of plans with L1 > 16 run on the caller's stream (one
    // scratch set, nothing to overlap): the batch only sets how many K1/K2
    // launches — each with a persistent grid's tail, its column-partial
    // reduce and K0 — the call takes, so it is large: ~98304 K1 items per
    // launch (~664 per SM), U at most ~16 GB (measured on B200, config 5:
    // 64 pairs 72.0 ms, 1024 pairs 68.0 ms, 2048 pairs 67.8 ms per step)
    {
      int64_t b1 = std::max<int64_t>(bp, (98304 + sp.L1 - 1) / sp.L1);
      b1 = std::max<int64_t>(1, std::min<int64_t>(b1, (int64_t(16) << 30) / per_pair));
      b1 = std::min<int64_t>(b1, 4096);
      pl->batch_pairs_1s = b1 >= 16 ? b1 / 16 * 16 : bp;
    }
    if (const char* ev = getenv("QMC_K1_PER_SM")) pl->k1_per_sm = int(strtol(ev, nullptr, 10));  // tuning
    if (const char* ev = getenv("QMC_K2_PER_SM")) pl->k2_per_sm = int(strtol(ev, nullptr, 10));  // tuning
    if (const char* ev = getenv("QMC_K1_GRID")) pl->k1_grid_cap = int(strtol(ev, nullptr, 10));     // tuning
    if (const char* ev = getenv("QMC_BATCH_PAIRS")) {  // tuning override
      const long v = strtol(ev, nullptr, 10);
      if (v > 0) {
        pl->batch_pairs = v;
        pl->batch_pairs_1s = v;
        pl->batch_fixed = 1;
      }
    }
    pl->k2_nopipe = getenv("QMC_K2_NOPIPE") != nullptr;
    pl->pack_gather = getenv("QMC_PACK_GATHER") != nullptr;
  }
  char* b = pl->ws;
  pl->d_scal = (double*)(b + lay.off_scal);
  pl->d_P = (int32_t*)(b + lay.off_P);
  pl->d_L = (int32_t*)(b + lay.off_L);
  pl->d_R = (int32_t*)(b + lay.off_R);
  pl->d_e = (int32_t*)(b + lay.off_e);
  pl->d_bstart = (int32_t*)(b + lay.off_bstart);
  pl->d_bent = (int4*)(b + lay.off_bent);
  pl->d_e2q = (int32_t*)(b + lay.off_e2q);
  pl->d_occ = (uint32_t*)(b + lay.off_occ);
  pl->d_zeta = (double*)(b + lay.off_zeta);
  pl->d_W = (double2*)(b + lay.off_W);
  pl->d_tw1 = (double2*)(b + lay.off_tw1);
  pl->d_tw2 = (double2*)(b + lay.off_tw2);
  pl->d_twL = (double2*)(b + lay.off_twL);
  pl->d_tw16 = (double2*)(b + lay.off_tw16);
  pl->d_twj = (double2*)(b + lay.off_twj);
  pl->d_jq = (int32_t*)(b + lay.off_jq);
  pl->d_k2n = (int32_t*)(b + lay.off_k2n);
  pl->d_k1c = (int32_t*)(b + lay.off_k1c);
  cudaStream_t st = pl->stream;

  auto fail = [&](int code) {
    delete pl;
    return code;
  };

  // plan-time scratch inside plan_ws: z, the prime factors of m, one flag
  std::vector<int64_t> qf = host_prime_factors(m);
  int64_t* d_z = (int64_t*)(b + lay.off_tmp);
  int64_t* d_qf = d_z + s;
  int32_t* d_cursor = (int32_t*)(b + lay.off_cursor);  // plan-time bucket cursors
  unsigned long long* d_flag = (unsigned long long*)(d_qf + 64);
  auto cleanup = [&]() { cudaStreamSynchronize(st); };
#define QMC_PLAN_CHECK(expr)              \
  do {                                    \
    int _rc = (expr);                     \
    if (_rc) {                            \
      cleanup();                          \
      return fail(_rc);                   \
    }                                     \
  } while (0)
#define QMC_PLAN_LAUNCHED() QMC_PLAN_CHECK(cudaPeekAtLastError() == cudaSuccess ? (g_launches++, 0) : (cudaGetLastError(), QMC_ECUDA))

  QMC_PLAN_CHECK(cudaMemcpyAsync(d_z, z_host, sizeof(int64_t) * s, cudaMemcpyHostToDevice, st) ? QMC_ECUDA : 0);
  if (!qf.empty())
    QMC_PLAN_CHECK(cudaMemcpyAsync(d_qf, qf.data(), sizeof(int64_t) * qf.size(), cudaMemcpyHostToDevice, st) ? QMC_ECUDA : 0);

  // a0: generator
  if (family == QMC_FAMILY_LATTICE) {
    unsigned long long best = ~0ull;
    for (int64_t base = 2; base < N && best == ~0ull; base += 4096) {
      unsigned long long init = ~0ull;
      QMC_PLAN_CHECK(cudaMemcpyAsync(d_flag, &init, 8, cudaMemcpyHostToDevice, st) ? QMC_ECUDA : 0);
      k_find_generator<<<16, 256, 0, st>>>(N, base, d_qf, int(qf.size()), d_flag);
      QMC_PLAN_LAUNCHED();
      QMC_PLAN_CHECK(cudaMemcpyAsync(&best, d_flag, 8, cudaMemcpyDeviceToHost, st) ? QMC_ECUDA : 0);
      QMC_PLAN_CHECK(cudaStreamSynchronize(st) ? QMC_ECUDA : 0);
    }
    if (best == ~0ull) { cleanup(); return fail(QMC_EINVAL_N); }
    pl->gen = int64_t(best);
  } else {
    unsigned long long flags = 0;
    QMC_PLAN_CHECK(cudaMemcpyAsync(d_flag, &flags, 8, cudaMemcpyHostToDevice, st) ? QMC_ECUDA : 0);
    k_check_poly<<<1, 64, 0, st>>>(p, pl->D, d_qf, int(qf.size()), d_flag);
    QMC_PLAN_LAUNCHED();
    QMC_PLAN_CHECK(cudaMemcpyAsync(&flags, d_flag, 8, cudaMemcpyDeviceToHost, st) ? QMC_ECUDA : 0);
    QMC_PLAN_CHECK(cudaStreamSynchronize(st) ? QMC_ECUDA : 0);
    if (flags) { cleanup(); return fail(QMC_EINVAL_POLY); }
    pl->gen = 2;  // the polynomial x
  }

  // a1..a3
  k_pow_table<<<blocks(m, 256), 256, 0, st>>>(family, N, p, pl->D, pl->gen, m, pl->d_P);
  QMC_PLAN_LAUNCHED();
  k_fill_i32<<<blocks(N, 256), 256, 0, st>>>(pl->d_L, N, -1);
  QMC_PLAN_LAUNCHED();
  k_log_scatter<<<blocks(m, 256), 256, 0, st>>>(pl->d_P, m, pl->d_L);
  QMC_PLAN_LAUNCHED();
  if (pl->d_k2n) {
    k_k2rows<<<blocks(sp.L, 256), 256, 0, st>>>(pl->d_P, m, sp.L, int(sp.L1), int(sp.L2), pl->d_k2n);
    QMC_PLAN_LAUNCHED();
  }
  k_colmap<<<blocks(s, 256), 256, 0, st>>>(d_z, s, pl->d_L, pl->d_e);
  QMC_PLAN_LAUNCHED();
  QMC_PLAN_CHECK(cudaMemsetAsync(pl->d_bstart, 0, size_t(sp.L2 + 1) * 4, st) ? QMC_ECUDA : 0);
  QMC_PLAN_CHECK(cudaMemsetAsync(pl->d_occ, 0, size_t(sp.L2 / 32 + 1) * 4, st) ? QMC_ECUDA : 0);
  k_bucket_count<<<blocks(s, 256), 256, 0, st>>>(pl->d_e, s, int(sp.L2), pl->d_bstart);
  QMC_PLAN_LAUNCHED();
  k_bucket_scan<<<1, 1024, 0, st>>>(pl->d_bstart, int(sp.L2), d_cursor);
  QMC_PLAN_LAUNCHED();
  k_bucket_place<<<blocks(s, 256), 256, 0, st>>>(pl->d_e, s, int(sp.L2), d_cursor, pl->d_e2q);
  QMC_PLAN_LAUNCHED();
  k_bucket_finish<<<blocks(sp.L2, 128), 128, 0, st>>>(pl->d_e, int(sp.L2), pl->d_bstart, pl->d_e2q, pl->d_bent,
                                                       pl->d_occ);
  QMC_PLAN_LAUNCHED();
  k_rtable<<<blocks(N, 256), 256, 0, st>>>(pl->d_L, N, m, pl->d_R);
  QMC_PLAN_LAUNCHED();
  // a4
  k_zeta<<<blocks(m, 256), 256, 0, st>>>(family, phi, delta, N, p, pl->D, m, pl->d_P, pl->d_zeta, pl->d_scal);
  QMC_PLAN_LAUNCHED();
  k_twiddles<<<blocks(sp.L1, 256), 256, 0, st>>>(pl->d_tw1, sp.L1, sp.L1);
  QMC_PLAN_LAUNCHED();
  k_twiddles<<<blocks(sp.L2, 256), 256, 0, st>>>(pl->d_tw2, sp.L2, sp.L2);
  QMC_PLAN_LAUNCHED();
  k_twiddles<<<blocks(sp.L2, 256), 256, 0, st>>>(pl->d_twL, sp.L, sp.L2);
  QMC_PLAN_LAUNCHED();
  k_twiddles<<<blocks(16 * sp.L1, 256), 256, 0, st>>>(pl->d_tw16, 16 * sp.L1, 16 * sp.L1);
  QMC_PLAN_LAUNCHED();
  {
    // K1 order of the scatter input (k1_balanced_order, else bucket order)
    QMC_PLAN_CHECK(cudaStreamSynchronize(st) ? QMC_ECUDA : 0);
    std::vector<int32_t> hb(size_t(sp.L2) + 1);
    std::vector<int4> hbent(static_cast<size_t>(s));
    QMC_PLAN_CHECK(cudaMemcpy(hb.data(), pl->d_bstart, 4 * hb.size(), cudaMemcpyDeviceToHost) ? QMC_ECUDA : 0);
    QMC_PLAN_CHECK(cudaMemcpy(hbent.data(), pl->d_bent, 16 * hbent.size(), cudaMemcpyDeviceToHost) ? QMC_ECUDA : 0);
    const int NT = int(sp.L2 / QMC_ROW_E);
    std::vector<int32_t> jq, code, cs, cr;
    int chmax = 0;
    // a' at least half full with more than 2 entries per bucket: the dense
    // first pass (below) is cheaper than any scatter
    const bool want_dense = 2 * s >= sp.L && s > 2 * sp.L2 && k2_split_R(sp.L1) > 0 && !getenv("QMC_K1_HEADS") &&
                            !getenv("QMC_NO_DENSE");
    pl->k1_bal = !want_dense && !getenv("QMC_K1_HEADS") && k1_try_balanced(s, sp.L2) &&
                 k1_balanced_order(hb, hbent, sp.L2, NT, k1_slot_budget(sp.L2), k1_s1max(s, sp.L2, sp.L), jq, code, cs, cr,
                                   chmax);
    // dense input: the balanced order does not apply and a' is at least half
    // full (e.g. the CBC all-generators plan, a permutation); entries sorted
    // by e (then j) with per-e starts, so k_pack_dense sums collisions in j
    // order.  jlist (s) fits jq and estart (L+1) fits e2q: both hold
    // k1_s1max >= L slots when 2s >= L
    pl->k1_dense = want_dense || (!pl->k1_bal && 2 * s >= sp.L && k2_split_R(sp.L1) > 0 &&
                                  !getenv("QMC_K1_HEADS") && !getenv("QMC_NO_DENSE"));
    if (pl->k1_dense) {
      std::vector<int32_t> estart(size_t(sp.L) + 1, 0), jlist(static_cast<size_t>(s));
      for (int64_t q = 0; q < s; ++q) ++estart[size_t(hbent[q].y) + 1];
      for (int64_t e = 0; e < sp.L; ++e) estart[e + 1] += estart[e];
      std::vector<int32_t> cur(estart.begin(), estart.end() - 1);
      std::vector<int32_t> eofj(static_cast<size_t>(s));
      for (int64_t q = 0; q < s; ++q) eofj[hbent[q].x] = hbent[q].y;
      for (int64_t j = 0; j < s; ++j) jlist[cur[eofj[j]]++] = int32_t(j);  // j order within each e
      jq.swap(jlist);
      QMC_PLAN_CHECK(cudaMemcpy(pl->d_e2q, estart.data(), 4 * estart.size(), cudaMemcpyHostToDevice) ? QMC_ECUDA : 0);
      cs.assign(1, 0);
      cr.clear();
      pl->S1 = sp.L;
      pl->k1_ch = 4;
    } else if (pl->k1_bal) {
      pl->S1 = int64_t(jq.size());
      pl->k1_ch = chmax;
      // one chunk that fits the staging next to the row (36 B per slot, at
      // the row kernel's residency): staged and prefetched during the
      // previous item's FFTs; otherwise K1 reads its input from global memory
      const int64_t limit = sp.L2 >= 8192 ? 232448 : 115712;
      const int64_t room = (limit - (k1_row_slots(sp.L2, QMC_ROW_E) + kK1Aux + sp.L1) * 16 - 16 - 64) / 36 / 4 * 4;
      if (cr.size() == 1 && chmax <= room) pl->k1_stage = int((chmax + 3) / 4 * 4);
      // otherwise (one chunk, read from global memory): its first whole
      // rounds of (a, code) — 20 B per slot, the twiddle comes from the
      // item's shared table — fill the rest of the shared memory, copied
      // during the previous item's FFTs; the later rounds stay direct
      const int64_t room20 = (limit - (k1_row_slots(sp.L2, QMC_ROW_E) + kK1Aux + sp.L1) * 16 -
                              sp.L1 * kK1TwRep * 16 - 16 - 64) / 20;
      int64_t sr_cap = room20 / NT;  // QMC_K1_SR: cap on the staged rounds (tuning)
      if (const char* ev = getenv("QMC_K1_SR")) sr_cap = std::min<int64_t>(sr_cap, strtol(ev, nullptr, 10));
      if (!pl->k1_stage && cr.size() == 1 && !getenv("QMC_K1_NOHYB"))
        pl->k1_srn = int(std::min<int64_t>(sr_cap, cr[0] / NT) * NT);
      QMC_PLAN_CHECK(cudaMemcpy(pl->d_e2q, code.data(), 4 * code.size(), cudaMemcpyHostToDevice) ? QMC_ECUDA : 0);
    } else {
      // bucket order, one chunk
      jq.clear();
      pl->S1 = s;
      pl->k1_ch = int(s);
      jq.resize(size_t(s));
      for (int64_t q = 0; q < s; ++q) jq[q] = hbent[q].x;
      cs.assign({0, int(s)});
      cr.assign({int(s)});
    }
    pl->k1_nch = int(cr.size());
    cs.insert(cs.end(), cr.begin(), cr.end());
    QMC_PLAN_CHECK(cudaMemcpy(pl->d_jq, jq.data(), 4 * jq.size(), cudaMemcpyHostToDevice) ? QMC_ECUDA : 0);
    QMC_PLAN_CHECK(cudaMemcpy(pl->d_k1c, cs.data(), 4 * cs.size(), cudaMemcpyHostToDevice) ? QMC_ECUDA : 0);
  }
  if (!pl->k1_dense) {  // the dense first pass needs no per-entry twiddles
    k_twj<<<blocks(sp.L1 * pl->S1, 256), 256, 0, st>>>(pl->d_jq, pl->d_e, pl->S1, sp.L, int(sp.L1),
                                                        int(sp.L2 / QMC_ROW_E), pl->d_twj);
    QMC_PLAN_LAUNCHED();
  }
  QMC_PLAN_CHECK(spectrum_dispatch(pl));
  QMC_PLAN_CHECK(cudaStreamSynchronize(st) ? QMC_ECUDA : 0);
#undef QMC_PLAN_CHECK
#undef QMC_PLAN_LAUNCHED
  plan_streams(pl);
  *out = pl;
  return QMC_OK;
}

}  // namespace qmc

using namespace qmc;

extern "C" {

int qmc_plan_workspace_size(int family, int64_t N_or_D, int64_t s, size_t* plan_bytes) {
  if (!plan_bytes) return QMC_ENULL;
  int64_t N, m;
  int rc = validate_family(family, N_or_D, s, &N, &m);
  if (rc) return rc;
  Split sp;
  if (!choose_split(m, s, &sp)) return QMC_EINVAL_N;
  *plan_bytes = plan_layout(N, m, s, sp).total;
  return QMC_OK;
}

int qmc_plan_create(qmc_plan_t* out, int64_t N, int64_t s, const int64_t* z_host, int phi,
                    void* plan_ws, size_t plan_ws_bytes, void* stream) {
  return create_common(out, QMC_FAMILY_LATTICE, N, 0, 0.0, s, z_host, phi, plan_ws, plan_ws_bytes, stream);
}

int qmc_plan_create_shifted(qmc_plan_t* out, int64_t N, int64_t s, const int64_t* z_host, int phi, double delta,
                            void* plan_ws, size_t plan_ws_bytes, void* stream) {
  if (!(delta >= 0.0 && delta < 1.0)) return QMC_EINVAL_PHI;
  return create_common(out, QMC_FAMILY_LATTICE, N, 0, delta, s, z_host, phi, plan_ws, plan_ws_bytes, stream);
}

// a replicate plan of an equally shifted rule shares every table of its base
// lattice plan except ζ, φ(x_0) and the spectrum W (only the
// circulant base changes with Δ)
static size_t shift_ws_layout(const qmc_plan* base, size_t* off_zeta, size_t* off_W) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  take(16 * 8);  // scal
  *off_zeta = take(size_t(base->m) * 8);
  *off_W = take(size_t(base->sp.L) * 16);
  return o;
}

int qmc_shift_workspace_size(qmc_plan_t base, size_t* bytes) {
  if (!base || !bytes) return QMC_ENULL;
  size_t a, b;
  *bytes = shift_ws_layout(base, &a, &b);
  return QMC_OK;
}

int qmc_plan_shift(qmc_plan_t* out, qmc_plan_t base, double delta, void* shift_ws, size_t shift_ws_bytes,
                   void* stream) {
  if (!out) return QMC_ENULL;
  *out = nullptr;
  if (!base || !shift_ws) return QMC_ENULL;
  if (base->family != QMC_FAMILY_LATTICE) return QMC_EUNSUPPORTED;
  if (!(delta >= 0.0 && delta < 1.0)) return QMC_EINVAL_PHI;
  size_t off_zeta, off_W;
  const size_t need = shift_ws_layout(base, &off_zeta, &off_W);
  if (shift_ws_bytes < need || (uintptr_t(shift_ws) % kAlign)) return QMC_EWORKSPACE;
  qmc_plan* pl = new (std::nothrow) qmc_plan(*base);  // the shared tables: same device pointers
  if (!pl) return QMC_ECUDA;
  pl->delta = delta;
  pl->stream = (cudaStream_t)stream;
  char* b = (char*)shift_ws;
  pl->d_scal = (double*)b;
  pl->d_zeta = (double*)(b + off_zeta);
  pl->d_W = (double2*)(b + off_W);
  pl->nstreams = 1;
  pl->mu = nullptr;
  const cudaStream_t st = pl->stream;
  k_zeta<<<blocks(pl->m, 256), 256, 0, st>>>(pl->family, pl->phi, delta, pl->N, pl->p, pl->D, pl->m, pl->d_P,
                                             pl->d_zeta, pl->d_scal);
  const bool zeta_ok = cudaPeekAtLastError() == cudaSuccess;
  if (zeta_ok) g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!zeta_ok || spectrum_dispatch(pl) != QMC_OK || cudaStreamSynchronize(st) != cudaSuccess) {
    cudaGetLastError();
    delete pl;
    return QMC_ECUDA;
  }
  plan_streams(pl);
  *out = pl;
  return QMC_OK;
}

int qmc_plan_create_poly(qmc_plan_t* out, int D, uint64_t p, int64_t s, const int64_t* q_host,
                         int phi, void* plan_ws, size_t plan_ws_bytes, void* stream) {
  return create_common(out, QMC_FAMILY_POLY, D, p, 0.0, s, q_host, phi, plan_ws, plan_ws_bytes, stream);
}

int qmc_plan_info(qmc_plan_t pl, int64_t* info) {
  if (!pl || !info) return QMC_ENULL;
  info[0] = pl->family;
  info[1] = pl->N;
  info[2] = pl->m;
  info[3] = pl->s;
  info[4] = pl->phi;
  info[5] = pl->gen;
  info[6] = pl->sp.L;
  info[7] = pl->sp.L1;
  info[8] = pl->sp.L2;
  info[9] = (pl->sp.L1 > 16 && !pl->green) ? pl->batch_pairs_1s : pl->batch_pairs;  // device calls' batch
  info[10] = pl->D;
  info[11] = int64_t(pl->p);
  info[12] = pl->k1_dense ? 2 : pl->k1_bal;
  info[13] = pl->S1;
  info[14] = pl->k1_nch;
  info[15] = pl->k1_ch;
  info[16] = pl->k1_srn;
  info[17] = pl->green ? pl->gsm[1] : 0;
  return QMC_OK;
}

int qmc_plan_tables(qmc_plan_t pl, int64_t* gen, int32_t* P, int32_t* L, int32_t* e, double* zeta) {
  if (!pl) return QMC_ENULL;
  if (cudaStreamSynchronize(pl->stream) != cudaSuccess) return QMC_ECUDA;
  if (gen) *gen = pl->gen;
  if (P && cudaMemcpy(P, pl->d_P, 4 * pl->m, cudaMemcpyDeviceToHost) != cudaSuccess) return QMC_ECUDA;
  if (L && cudaMemcpy(L, pl->d_L, 4 * pl->N, cudaMemcpyDeviceToHost) != cudaSuccess) return QMC_ECUDA;
  if (e && cudaMemcpy(e, pl->d_e, 4 * pl->s, cudaMemcpyDeviceToHost) != cudaSuccess) return QMC_ECUDA;
  if (zeta && cudaMemcpy(zeta, pl->d_zeta, 8 * pl->m, cudaMemcpyDeviceToHost) != cudaSuccess) return QMC_ECUDA;
  return QMC_OK;
}

int64_t qmc_launch_count(void) { return g_launches.load(); }

int qmc_build_flags(void) {
  int f = 0;
#ifdef QMC_CHECK
  f |= 1;
#endif
#ifdef QMC_PHASE_TIMING
  f |= 2;
#endif
  return f;
}

int qmc_profile_enable(int on) {
  g_prof.on = on != 0;
  return QMC_OK;
}

int qmc_profile_read(int64_t* launches, double* ms, int n) {
  if (!launches || !ms) return QMC_ENULL;
  for (int k = 0; k < KC_COUNT; ++k) {
    double tot = 0.0;
    for (auto& pr : g_prof.ev[k]) {
      if (cudaEventSynchronize(pr.second) != cudaSuccess) return QMC_ECUDA;
      float x = 0.f;
      cudaEventElapsedTime(&x, pr.first, pr.second);
      tot += x;
      g_prof.pool.push_back(pr.first);
      g_prof.pool.push_back(pr.second);
    }
    if (k < n) {
      launches[k] = int64_t(g_prof.ev[k].size());
      ms[k] = tot;
    }
    g_prof.ev[k].clear();
  }
  return QMC_OK;
}

const char* qmc_profile_class_name(int k) {
  static const char* names[KC_COUNT] = {"k_pack", "k_rows", "k_cols", "k_gather", "k_reduce",
                                        "k_finalize"};
  return (k >= 0 && k < KC_COUNT) ? names[k] : "";
}

void qmc_plan_destroy(qmc_plan_t pl) {
  if (!pl) return;
  if (pl->green) {
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(pl->ev_ready[i]);
      cudaEventDestroy(pl->ev_free[i]);
    }
  }
  if (pl->nstreams == 2) {
    cudaStreamDestroy(pl->ist[0]);
    cudaStreamDestroy(pl->ist[1]);
    cudaEventDestroy(pl->ev_fork);
    cudaEventDestroy(pl->ev_join[0]);
    cudaEventDestroy(pl->ev_join[1]);
  }
  delete pl->mu;
  delete pl;
}

const char* qmc_strerror(int code) {
  switch (code) {
    case QMC_OK: return "ok";
    case QMC_EINVAL_N: return "N not prime, out of range, or circulant length unsupported";
    case QMC_EINVAL_Z: return "generating vector entry outside [1, m]";
    case QMC_EINVAL_POLY: return "modulus not of degree D or not primitive over F_2";
    case QMC_EINVAL_DIM: return "invalid dimension (s < 1, t < 0, lda < s, ldx < N)";
    case QMC_EINVAL_PHI: return "unknown phi";
    case QMC_ENULL: return "required pointer is NULL";
    case QMC_ECUDA: return "CUDA error";
    case QMC_EWORKSPACE: return "workspace too small or not 256-byte aligned";
    case QMC_EUNSUPPORTED: return "request not covered by this entry point";
    case QMC_EINVAL_F: return "unknown f";
  }
  return "unknown status";
}

}  // extern "C"
