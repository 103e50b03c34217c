// fft.cuh — fp64 complex FFT building blocks for sm_100a (shared memory,
// register butterflies).  The circulant product Z·a' of PAPER.md:355-362
// ("can be computed in O(N log N) operations using FFT") is evaluated as
// a cyclic convolution through these transforms.
//
// Conventions: forward DFT X[f] = Σ_e x[e] ω^{ef}, ω = exp(-2πi/n)
// (DIR = -1); inverse uses ω^{-1} (DIR = +1) and is unnormalised (1/L is
// folded into the spectrum W at plan time).
//
// Transform shape: Stockham auto-sort, natural order in and out, radix
// R ∈ {2,3,4,5,8}.  Stage with span Ns (product of the radices already
// applied): butterfly j ∈ [0, n/R) reads x[j + r·n/R], multiplies by
// ω_{Ns·R}^{(j mod Ns)·r}, runs DFT_R and writes
// y[(j/Ns)·Ns·R + (j mod Ns) + r·Ns].
#pragma once
#include <cuda_runtime.h>

namespace qmc {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a · conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// multiply by DIR·i  (forward: -i, inverse: +i)
template <int DIR>
__device__ __forceinline__ double2 rot(double2 a) {
  return DIR < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
template <int DIR>
__device__ __forceinline__ double2 twid(double2 w) {  // forward table → direction
  return DIR < 0 ? w : make_double2(w.x, -w.y);
}
// 32-byte read-only load of two adjacent complex values (LDG.E.256 on
// sm_100a); p must be 32-byte aligned.
__device__ __forceinline__ void ldg2_256(const double2* p, double2& a, double2& b) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
      : "l"(p));
}
// streaming (evict-first) variants for data read or written exactly once
__device__ __forceinline__ void ldcs2_256(const double2* p, double2& a, double2& b) {
  asm("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
      : "l"(p));
}
__device__ __forceinline__ double2 ldcs(const double2* p) {
  double2 r;
  asm("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void stcs(double* p, double v) { asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }
__device__ __forceinline__ void stcs2(double* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// Drop a dead 128-byte line from L2 without writing it back (scratch data
// that is never read again); p must be 128-byte aligned.
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
// Read-only 16-byte load kept in program order (volatile): stops the compiler
// from hoisting every stage's twiddles to the kernel start, which costs more
// registers than the latency it hides.
__device__ __forceinline__ double2 ldg_ordered(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// ----------------------------------------------------------------- DFT_R
template <int R, int DIR> struct Dft;

template <int DIR> struct Dft<2, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR> struct Dft<4, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    double2 t2 = cadd(v[1], v[3]), t3 = rot<DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

template <int DIR> struct Dft<8, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    const double c = 0.70710678118654752440084436210485;
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR>::run(e);
    Dft<4, DIR>::run(o);
    // o[k] *= ω8^k, ω8 = (c, DIR·c)
    double2 o1 = make_double2(c * (o[1].x - DIR * o[1].y), c * (o[1].y + DIR * o[1].x));
    double2 o2 = rot<DIR>(o[2]);
    double2 o3 = make_double2(c * (-o[3].x - DIR * o[3].y), c * (-o[3].y + DIR * o[3].x));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
};

template <int DIR> struct Dft<3, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    const double s3 = 0.86602540378443864676372317075294;  // sin(2π/3)
    double2 t1 = cadd(v[1], v[2]);
    double2 d = csub(v[1], v[2]);
    double2 m = make_double2(fma(-0.5, t1.x, v[0].x), fma(-0.5, t1.y, v[0].y));
    // DIR·i·s3·d
    double2 q = rot<DIR>(make_double2(s3 * d.x, s3 * d.y));
    v[0] = cadd(v[0], t1);
    v[1] = cadd(m, q);
    v[2] = csub(m, q);
  }
};

template <int DIR> struct Dft<5, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    const double c1 = 0.30901699437494742410229341718282;   // cos(2π/5)
    const double c2 = -0.80901699437494742410229341718282;  // cos(4π/5)
    const double s1 = 0.95105651629515357211643933337938;   // sin(2π/5)
    const double s2 = 0.58778525229247312916870595463907;   // sin(4π/5)
    double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    double2 a1 = make_double2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    double2 a2 = make_double2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    double2 b1 = rot<DIR>(make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y));
    double2 b2 = rot<DIR>(make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y));
    v[0] = cadd(v[0], cadd(t1, t2));
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
  }
};

// DFT16 = 4 x 4 with internal twiddles ω16^{n2·k1} (constants)
template <int DIR>
__device__ __forceinline__ double2 cmul_k(double2 a, double c, double s) {  // a · (c + DIR·i·s)
  return make_double2(fma(a.x, c, -DIR * a.y * s), fma(a.y, c, DIR * a.x * s));
}

template <int DIR> struct Dft<16, DIR> {
  static __device__ __forceinline__ void run(double2* v) {
    const double c1 = 0.92387953251128675612818318939679;  // cos(π/8)
    const double s1 = 0.38268343236508977172845998403040;  // sin(π/8)
    const double h = 0.70710678118654752440084436210485;
    double2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      double2 a[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      Dft<4, DIR>::run(a);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = a[k1];
    }
    // y[n2][k1] *= ω16^{n2 k1}, ω16^q = (cos(qπ/8), DIR·sin(qπ/8))
    y[1][1] = cmul_k<DIR>(y[1][1], c1, s1);
    y[1][2] = cmul_k<DIR>(y[1][2], h, h);
    y[1][3] = cmul_k<DIR>(y[1][3], s1, c1);
    y[2][1] = cmul_k<DIR>(y[2][1], h, h);
    y[2][2] = rot<DIR>(y[2][2]);
    y[2][3] = cmul_k<DIR>(y[2][3], -h, h);
    y[3][1] = cmul_k<DIR>(y[3][1], s1, c1);
    y[3][2] = cmul_k<DIR>(y[3][2], -h, h);
    y[3][3] = cmul_k<DIR>(y[3][3], -c1, -s1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 b[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
      Dft<4, DIR>::run(b);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = b[k2];
    }
  }
};

template <int DIR> struct Dft<1, DIR> {
  static __device__ __forceinline__ void run(double2*) {}
};

template <int DIR>
__device__ __forceinline__ void dft_runtime(int R, double2* v) {
  switch (R) {
    case 2: Dft<2, DIR>::run(v); break;
    case 3: Dft<3, DIR>::run(v); break;
    case 4: Dft<4, DIR>::run(v); break;
    case 5: Dft<5, DIR>::run(v); break;
    default: Dft<8, DIR>::run(v); break;
  }
}

// ----------------------------------------------------------------- row FFT
// Shared-memory swizzle for 16-byte elements: XOR the low 3 index bits with
// bits 3..5 so that every 8-thread phase of the Stockham loads and stores
// touches 8 distinct 16-B bank groups.
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 3) & 7); }

template <int N> struct RowRadices;
#define QMC_RADICES(NN, ...)                                                   \
  template <> struct RowRadices<NN> {                                          \
    static constexpr int r[] = {__VA_ARGS__};                                  \
    static constexpr int count = sizeof(r) / sizeof(int);                      \
    static __host__ __device__ constexpr int get(int i) { return r[i]; }       \
  };
QMC_RADICES(16, 4, 4)
QMC_RADICES(32, 8, 4)
QMC_RADICES(64, 8, 8)
QMC_RADICES(128, 8, 4, 4)
QMC_RADICES(256, 8, 8, 4)
QMC_RADICES(512, 8, 8, 8)
QMC_RADICES(1024, 8, 8, 4, 4)
QMC_RADICES(2048, 8, 8, 8, 4)
QMC_RADICES(4096, 8, 8, 8, 8)
QMC_RADICES(8192, 8, 8, 8, 4, 4)
#undef QMC_RADICES

// threads per CTA for a row FFT of length N (16 complex values per thread
// once N >= 512)
template <int N> struct RowThreads {
  static constexpr int value = (N / 8) > 1024 ? 1024 : (N / 8);
};

// One Stockham stage over a length-N row held in shared memory S (swizzled),
// NT threads; tw = ω_N^k table (k < N, forward sign) in global memory.
template <int R, int N, int NT, int DIR, int NS>
__device__ __forceinline__ void row_stage(double2* S, const double2* __restrict__ tw, int tid) {
  constexpr int NB = N / R;
  constexpr int BPT = (NB + NT - 1) / NT;
  double2 v[BPT][R];
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = tid + b * NT;
    if (NB % NT == 0 || j < NB) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][r] = S[swz(j + r * NB)];
    }
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = tid + b * NT;
    if (NB % NT == 0 || j < NB) {
      const int k = j % NS;
      if (NS > 1) {
        constexpr int STEP = N / (NS * R);
#pragma unroll
        for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], twid<DIR>(__ldg(&tw[k * r * STEP])));
      }
      Dft<R, DIR>::run(v[b]);
      const int base = (j / NS) * NS * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) S[swz(base + r * NS)] = v[b][r];
    }
  }
  __syncthreads();
}

template <int N, int NT, int DIR, int NS, int I>
__device__ __forceinline__ void row_fft_rec(double2* S, const double2* __restrict__ tw, int tid) {
  if constexpr (I < RowRadices<N>::count) {
    constexpr int R = RowRadices<N>::get(I);
    row_stage<R, N, NT, DIR, NS>(S, tw, tid);
    row_fft_rec<N, NT, DIR, NS * R, I + 1>(S, tw, tid);
  }
}

// Full length-N FFT of the swizzled shared row S (natural order in and out).
// Caller must __syncthreads() after writing S; returns after a barrier.
template <int N, int DIR>
__device__ __forceinline__ void row_fft(double2* S, const double2* __restrict__ tw) {
  row_fft_rec<N, RowThreads<N>::value, DIR, 1, 0>(S, tw, threadIdx.x);
}

}  // namespace qmc


namespace qmc {

// ----------------------------------------------------------------- register row FFT helpers
// %tid.x read through volatile asm: addresses derived from it cannot be
// hoisted above the point of use, so each stage holds only its own
// shared-memory / twiddle addresses live (instead of all stages' at once).
__device__ __forceinline__ int tid_fresh() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

template <int E> struct Lg;
template <> struct Lg<8> { static constexpr int v = 3; };
template <> struct Lg<16> { static constexpr int v = 4; };

// padded shared-memory index (one pad slot per E elements)
template <int E>
__device__ __forceinline__ int padE(int i) { return i + (i >> Lg<E>::v); }

// ----------------------------------------------------------------- DIF / DIT register row FFT (K1)
// Length-L2 row held by NT = L2/16 threads, 16 points each; on entry and on
// exit of the round trip thread t holds v[q] = x[t + NT·q] (natural order).
// L2 = RHO·SUB with SUB = 16^K ∈ {16, 256, 4096} and RHO ∈ {1, 2, 4, 8}.
//
// Forward (decimation in frequency): an in-register radix-RHO stage over
// the stride-L2/RHO pairs a thread already holds (RHO > 1), then per
// sub-transform of SUB points (G = SUB/16 threads) radix-16 stages whose
// exchanges shrink from the whole sub (G threads) to one half-warp (16
// threads), each stage's 16 outputs twiddled by ω_n^{j·k}.  The spectrum
// ends in digit-reversed order (dif_freq gives the frequency of register r
// of thread t); the pointwise product uses a spectrum stored in that order,
// and the inverse (decimation in time) mirrors every step, so no reordering
// pass exists.  Every exchange writes exactly the shared-memory slots the
// same thread read in the previous exchange, so one barrier per exchange
// suffices, at the exchange's own scope: the CTA (RHO-stage, or SUB = L2),
// half the CTA (named barrier, L2 = 8192), or the half-warp (__syncwarp).
// Region of sub c: c·REG + lay(r, j) with lay = 272 r + j + (j >> 4)
// (SUB = 4096), 17 r + j (SUB = 256), r (SUB = 16); padE<16>(t + NT q) is the
// same slot, so the scatter's row and the region layouts coincide.
template <int L2>
struct Dif {
  static constexpr int NT = L2 / 16;
  static constexpr int SUB = L2 >= 4096 ? 4096 : (L2 >= 256 ? 256 : 16);
  static constexpr int RHO = L2 / SUB;
  static constexpr int G = SUB / 16;
  static constexpr int REG = SUB / 16 * 17;
  static_assert(RHO == 1 || RHO == 2 || RHO == 4 || RHO == 8, "unsupported row length");
};

// frequency index (natural order) of register r of thread t after dif_fwd
template <int L2>
__host__ __device__ inline int dif_freq(int t, int r) {
  constexpr int G = Dif<L2>::G, RHO = Dif<L2>::RHO;
  int o = 0, sg = 1, j = t;
  if (RHO > 1) {
    o = t / G;
    j = t % G;
    sg = RHO;
  }
  for (int g = G; g > 1; g /= 16) {
    const int gp = g / 16;
    o += sg * (j / gp);
    j %= gp;
    sg *= 16;
  }
  return o + sg * r;
}

// cos / sin of 2πk/16
__host__ __device__ constexpr double c16(int k) {
  constexpr double c[16] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                            0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                            -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
                            0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};
  return c[k & 15];
}
__host__ __device__ constexpr double s16(int k) { return c16(k - 4); }  // sin(2πk/16) = cos(2π(k-4)/16)

// a · ω_16^k (forward sign: ω = exp(-2πi/16)), k a compile-time constant
template <int K>
__device__ __forceinline__ double2 mul_w16(double2 a) {
  constexpr int k = K & 15;
  if constexpr (k == 0) return a;
  else if constexpr (k == 4) return make_double2(a.y, -a.x);
  else if constexpr (k == 8) return make_double2(-a.x, -a.y);
  else if constexpr (k == 12) return make_double2(-a.y, a.x);
  else {
    constexpr double c = c16(k), s = s16(k);  // ω^k = c - i s
    return make_double2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));
  }
}

// v[k] *= w^k (k = 1..15), conjugated for DIR = +1; w forward-sign
template <int DIR>
__device__ __forceinline__ void twiddle16(double2 (&v)[16], double2 w) {
  double2 pw[16];
  pw[1] = twid<DIR>(w);
#pragma unroll
  for (int r = 2; r < 16; ++r) pw[r] = cmul(pw[r / 2], pw[r - r / 2]);
#pragma unroll
  for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], pw[r]);
}

// v[k] *= b·w^k (k = 0..15), conjugated for DIR = +1
template <int DIR>
__device__ __forceinline__ void twiddle16_fold(double2 (&v)[16], double2 w, double2 b) {
  double2 wp[9], T[16];
  wp[1] = twid<DIR>(w);
#pragma unroll
  for (int r = 2; r <= 8; ++r) wp[r] = cmul(wp[r / 2], wp[r - r / 2]);
  T[0] = twid<DIR>(b);
#pragma unroll
  for (int k = 1; k < 16; ++k) T[k] = cmul(T[k / 2], wp[k - k / 2]);
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = cmul(v[k], T[k]);
}

template <int DIR>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
  Dft<16, DIR>::run(v);
}

// barrier over the G threads of one sub-transform (SUB = 4096 level)
template <int L2>
__device__ __forceinline__ void dif_bar_sub(int c) {
  if constexpr (Dif<L2>::RHO == 1) {
    __syncthreads();
  } else {
    if (c == 0)
      asm volatile("bar.sync 1, %0;" ::"n"(Dif<L2>::G) : "memory");
    else
      asm volatile("bar.sync 2, %0;" ::"n"(Dif<L2>::G) : "memory");
  }
}

// RHO-stage twiddle of (q0, c'): b · ω_{L2}^{(t + NT q0) c'} = b·w^{c'}·ω_16^{q0 c'}
template <int RHO, int Q0, int CP, int DIR>
__device__ __forceinline__ double2 rho_apply(double2 a, const double2 (&bw)[8]) {
  const double2 t = mul_w16<Q0 * CP>(bw[CP]);
  return cmul(a, twid<DIR>(t));
}

template <int RHO, int DIR, int Q0>
__device__ __forceinline__ void rho_stage_fwd(double2 (&v)[16], const double2 (&bw)[8]) {
  if constexpr (Q0 < 16 / RHO) {
    constexpr int ST = 16 / RHO;
    double2 u[RHO];
#pragma unroll
    for (int c = 0; c < RHO; ++c) u[c] = v[Q0 + ST * c];
    Dft<RHO, -1>::run(u);
    v[Q0] = cmul(u[0], bw[0]);
    if constexpr (RHO > 1) v[Q0 + ST * 1] = rho_apply<RHO, Q0, 1, -1>(u[1], bw);
    if constexpr (RHO > 2) v[Q0 + ST * 2] = rho_apply<RHO, Q0, 2, -1>(u[2], bw);
    if constexpr (RHO > 3) v[Q0 + ST * 3] = rho_apply<RHO, Q0, 3, -1>(u[3], bw);
    if constexpr (RHO > 4) {
      v[Q0 + ST * 4] = rho_apply<RHO, Q0, 4, -1>(u[4], bw);
      v[Q0 + ST * 5] = rho_apply<RHO, Q0, 5, -1>(u[5], bw);
      v[Q0 + ST * 6] = rho_apply<RHO, Q0, 6, -1>(u[6], bw);
      v[Q0 + ST * 7] = rho_apply<RHO, Q0, 7, -1>(u[7], bw);
    }
    rho_stage_fwd<RHO, DIR, Q0 + 1>(v, bw);
  }
}

template <int RHO, int Q0>
__device__ __forceinline__ void rho_stage_inv(double2 (&v)[16], const double2 (&bw)[8]) {
  if constexpr (Q0 < 16 / RHO) {
    constexpr int ST = 16 / RHO;
    double2 u[RHO];
    u[0] = cmulc(v[Q0], bw[0]);
    if constexpr (RHO > 1) u[1] = rho_apply<RHO, Q0, 1, +1>(v[Q0 + ST * 1], bw);
    if constexpr (RHO > 2) u[2] = rho_apply<RHO, Q0, 2, +1>(v[Q0 + ST * 2], bw);
    if constexpr (RHO > 3) u[3] = rho_apply<RHO, Q0, 3, +1>(v[Q0 + ST * 3], bw);
    if constexpr (RHO > 4) {
      u[4] = rho_apply<RHO, Q0, 4, +1>(v[Q0 + ST * 4], bw);
      u[5] = rho_apply<RHO, Q0, 5, +1>(v[Q0 + ST * 5], bw);
      u[6] = rho_apply<RHO, Q0, 6, +1>(v[Q0 + ST * 6], bw);
      u[7] = rho_apply<RHO, Q0, 7, +1>(v[Q0 + ST * 7], bw);
    }
    Dft<RHO, +1>::run(u);
#pragma unroll
    for (int c = 0; c < RHO; ++c) v[Q0 + ST * c] = u[c];
    rho_stage_inv<RHO, Q0 + 1>(v, bw);
  }
}

// bw[c'] = b·w^{c'} (c' < RHO), w = ω_{L2}^t
template <int RHO>
__device__ __forceinline__ void rho_bases(double2 (&bw)[8], double2 w, double2 b) {
  bw[0] = b;
#pragma unroll
  for (int c = 1; c < RHO; ++c) bw[c] = cmul(bw[c - 1], w);
}

// Forward DIF of the row (see Dif).  On entry v[q] = x[t + NT q] and the
// caller has made S safe to write (the thread's own padE slots); tw2 =
// ω_{L2}^i (i < L2), b = ω_L^{t f1}: the four-step twiddle of the thread's
// column is folded into the first stage (all 16 inputs share it).
// Wr != nullptr: the spectrum row in this register order (Wr[q·NT] for
// v[q] of the calling thread, Wr already offset by the thread): v leaves
// multiplied by it, dc receives v[0] before the product.
template <int L2>
__device__ __forceinline__ void dif_fwd(double2 (&v)[16], double2* S, const double2* __restrict__ tw2, double2 b,
                                        const double2* __restrict__ Wr = nullptr, double2* dcp = nullptr) {
  double2 dc_unused;
  double2& dc = dcp ? *dcp : dc_unused;
  using D = Dif<L2>;
  constexpr int NT = D::NT, RHO = D::RHO, G = D::G, SUB = D::SUB;
  const int t = tid_fresh();
  int c = 0, j = t;
  if constexpr (RHO > 1) {
    double2 bw[8];
    rho_bases<RHO>(bw, ldg_ordered(&tw2[t]), b);
    rho_stage_fwd<RHO, -1, 0>(v, bw);
    if constexpr (NT % 16 == 0) {
      double2* St = S + padE<16>(t);
#pragma unroll
      for (int q = 0; q < 16; ++q) St[q * (NT + NT / 16)] = v[q];  // padE(t + NT q)
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) S[padE<16>(t + NT * q)] = v[q];
    }
    __syncthreads();
    c = t / G;
    j = t % G;
    const double2* Sr = S + c * D::REG;
    if constexpr (SUB == 4096) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = Sr[272 * r + j + (j >> 4)];
    } else if constexpr (SUB == 256) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = Sr[17 * r + j];
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = Sr[r];
    }
  }
  double2* B = S + c * D::REG;
  if constexpr (SUB == 4096) {
    dft16<-1>(v);
    const double2 w = ldg_ordered(&tw2[j * (L2 / 4096)]);
    if constexpr (RHO == 1) twiddle16_fold<-1>(v, w, b);
    else twiddle16<-1>(v, w);
    double2* Bw = B + j + (j >> 4);
#pragma unroll
    for (int k = 0; k < 16; ++k) Bw[272 * k] = v[k];
    dif_bar_sub<L2>(c);
    const int k = j >> 4;
    j &= 15;
    B += 272 * k;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = B[j + 17 * r];
  }
#ifndef QMC_W_AHEAD
#define QMC_W_AHEAD 0
#endif
  constexpr int WA = QMC_W_AHEAD;  // spectrum values loaded during the last exchange
  double2 wv[WA > 0 ? WA : 1];
  if constexpr (SUB >= 256) {
    dft16<-1>(v);
    const double2 w = ldg_ordered(&tw2[j * (L2 / 256)]);
    if constexpr (SUB == 256 && RHO == 1) twiddle16_fold<-1>(v, w, b);
    else twiddle16<-1>(v, w);
#ifndef QMC_DIAG_NO_XW
#pragma unroll
    for (int k = 0; k < 16; ++k) B[j + 17 * k] = v[k];
#endif
    // v is dead until the exchange's reads: the first half of the spectrum
    // row goes in flight now (its latency overlaps the exchange and the last
    // butterflies)
    if (Wr) {
#pragma unroll
      for (int q = 0; q < WA; ++q) wv[q] = ldg_ordered(&Wr[q * NT]);
    }
    __syncwarp(NT >= 32 ? 0xffffffffu : 0xffffu);  // the half-warp group (rows of 256: 16 lanes exist)
#ifndef QMC_DIAG_NO_XW  // diagnostic: the half-warp exchange skipped (wrong results; timing bound)
#pragma unroll
    for (int p = 0; p < 16; ++p) v[p] = B[17 * j + p];
#endif
  } else if (Wr) {
#pragma unroll
    for (int q = 0; q < WA; ++q) wv[q] = ldg_ordered(&Wr[q * NT]);
  }
  dft16<-1>(v);
  if (Wr) {  // × the spectrum row (this register order), v[0] of thread 0 = DC term first
    dc = v[0];
#pragma unroll
    for (int q = 0; q < WA; ++q) v[q] = cmul(v[q], wv[q]);
#pragma unroll
    for (int q = WA; q < 16; ++q) v[q] = cmul(v[q], ldg_ordered(&Wr[q * NT]));
  }
}

// Inverse DIT, the mirror of dif_fwd (same b): on entry the spectrum in
// dif_fwd's output order, on exit v[q] = x[t + NT q] (unnormalised).
template <int L2>
__device__ __forceinline__ void dif_inv(double2 (&v)[16], double2* S, const double2* __restrict__ tw2, double2 b) {
  using D = Dif<L2>;
  constexpr int NT = D::NT, RHO = D::RHO, G = D::G, SUB = D::SUB;
  const int t = tid_fresh();
  const int c = RHO > 1 ? t / G : 0;
  const int j0 = RHO > 1 ? t % G : t;
  double2* B = S + c * D::REG;
  dft16<+1>(v);
  if constexpr (SUB >= 256) {
    const int k = SUB == 4096 ? (j0 >> 4) : 0, j = j0 & 15;
    double2* B2 = B + 272 * k;
#ifndef QMC_DIAG_NO_XW
#pragma unroll
    for (int p = 0; p < 16; ++p) B2[17 * j + p] = v[p];
#endif
    __syncwarp(NT >= 32 ? 0xffffffffu : 0xffffu);  // the half-warp group (rows of 256: 16 lanes exist)
#ifndef QMC_DIAG_NO_XW
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = B2[j + 17 * r];
#endif
    const double2 w = ldg_ordered(&tw2[j * (L2 / 256)]);
    if constexpr (SUB == 256 && RHO == 1) twiddle16_fold<+1>(v, w, b);
    else twiddle16<+1>(v, w);
    dft16<+1>(v);
    if constexpr (SUB == 4096) {
#pragma unroll
      for (int r = 0; r < 16; ++r) B2[j + 17 * r] = v[r];
      dif_bar_sub<L2>(c);
      const double2* Br = B + j0 + (j0 >> 4);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) v[kk] = Br[272 * kk];
      const double2 w4 = ldg_ordered(&tw2[j0 * (L2 / 4096)]);
      if constexpr (RHO == 1) twiddle16_fold<+1>(v, w4, b);
      else twiddle16<+1>(v, w4);
      dft16<+1>(v);
    }
  }
  if constexpr (RHO > 1) {
    double2* Bw = B;
    if constexpr (SUB == 4096) {
#pragma unroll
      for (int r = 0; r < 16; ++r) Bw[272 * r + j0 + (j0 >> 4)] = v[r];
    } else if constexpr (SUB == 256) {
#pragma unroll
      for (int r = 0; r < 16; ++r) Bw[17 * r + j0] = v[r];
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r) Bw[r] = v[r];
    }
    __syncthreads();
    if constexpr (NT % 16 == 0) {
      const double2* St = S + padE<16>(t);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = St[q * (NT + NT / 16)];
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = S[padE<16>(t + NT * q)];
    }
    double2 bw[8];
    rho_bases<RHO>(bw, ldg_ordered(&tw2[t]), b);
    rho_stage_inv<RHO, 0>(v, bw);
  }
}

// ----------------------------------------------------------------- register column DFT
// Length-N DFT entirely in one thread's registers, N = R·M with R, M in
// {1,2,3,4,5,8,16}: M-point DFTs over stride-R subsequences, twiddles
// ω_N^{r·k2} from the table twN (ω_N^k, forward sign), R-point DFTs.
// Natural order in and out.
__host__ __device__ constexpr bool direct_radix(int n) {
  return n == 1 || n == 2 || n == 3 || n == 4 || n == 5 || n == 8 || n == 16;
}
__host__ __device__ constexpr int reg_split(int n) {  // R with n = R·M, both direct; 0 if none
  for (int r = 2; r <= 16; ++r)
    if (n % r == 0 && direct_radix(r) && direct_radix(n / r)) return r;
  return direct_radix(n) ? 1 : 0;
}

// twN[k·ts] = ω_N^k (a table of a multiple of N read with stride ts; global
// or shared memory).
template <int N, int DIR>
__device__ __forceinline__ void reg_dft(double2* v, const double2* __restrict__ twN, int ts = 1) {
  if constexpr (direct_radix(N)) {
    Dft<N, DIR>::run(v);
  } else {
    constexpr int R = reg_split(N), M = N / R;
    static_assert(R > 1, "unsupported register DFT length");
    double2 y[N];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double2 sv[M];
#pragma unroll
      for (int m = 0; m < M; ++m) sv[m] = v[m * R + r];
      Dft<M, DIR>::run(sv);
#pragma unroll
      for (int k2 = 0; k2 < M; ++k2)
        y[r * M + k2] = (r * k2 == 0) ? sv[k2] : cmul(sv[k2], twid<DIR>(twN[r * k2 * ts]));
    }
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) {
      double2 sv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) sv[r] = y[r * M + k2];
      Dft<R, DIR>::run(sv);
#pragma unroll
      for (int k1 = 0; k1 < R; ++k1) v[k2 + M * k1] = sv[k1];
    }
  }
}

}  // namespace qmc
