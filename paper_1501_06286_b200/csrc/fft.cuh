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

#ifndef QMC_TW_RECUR
#define QMC_TW_RECUR 1
#endif

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

// ----------------------------------------------------------------- register row FFT
// Length-N FFT with E points per thread (E = 8 or 16, NT = N/E threads):
// thread `tid` holds element tid + NT·q in v[q] before and after the
// transform (natural order, strided).  Stages are radix E (plus one smaller
// radix stage when N is not a power of E); between stages the row is
// exchanged through shared memory S (padding of one slot per E elements),
// two barriers per exchange.  A forward transform, a pointwise product and
// an inverse transform therefore never round-trip through shared memory
// between them.

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

// padded shared-memory index: all 8-thread phases of the stage loads and
// stores hit distinct bank groups; every address of a stage is a per-thread
// base plus a compile-time offset
template <int E>
__device__ __forceinline__ int padE(int i) { return i + (i >> Lg<E>::v); }
template <int N, int E> struct PadE { static constexpr int size = N + N / E; };
__device__ __forceinline__ int swz16(int i) { return padE<16>(i); }
template <int N> struct Pad16 { static constexpr int size = PadE<N, 16>::size; };

// radix plan: log_E(N) radix-E stages, then the remainder
template <int N, int E> struct RPlan {
  static constexpr int count = (N >= E) ? 1 + RPlan<(N >= E ? N / E : 1), E>::count : (N > 1 ? 1 : 0);
  static __host__ __device__ constexpr int get(int i) {
    return i == 0 ? (N >= E ? E : N) : RPlan<(N >= E ? N / E : 1), E>::get(i - 1);
  }
};
template <int E> struct RPlan<1, E> {
  static constexpr int count = 0;
  static __host__ __device__ constexpr int get(int) { return 1; }
};

// One radix-R stage on registers.  twS = this stage's twiddle table,
// stage-major: twS[(r-1)·NS + k] = ω_{NS·R}^{k·r} (forward sign), so the
// loads of consecutive threads (consecutive k) are contiguous.
template <int R, int N, int E, int NS, int DIR>
__device__ __forceinline__ void reg_stage(double2 (&v)[E], const double2* __restrict__ twS, int tid) {
  constexpr int NT = N / E, BPT = E / R;
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + r * BPT];
    if (NS > 1) {
      const double2* twk = twS + (tid_fresh() + b * NT) % NS;
#if QMC_TW_RECUR
      // one load; w^r by a product tree of depth <= 4 (w^r = w^{r/2} w^{r-r/2})
      double2 pw[R];
      pw[1] = twid<DIR>(ldg_ordered(twk));
#pragma unroll
      for (int r = 2; r < R; ++r) pw[r] = cmul(pw[r / 2], pw[r - r / 2]);
#pragma unroll
      for (int r = 1; r < R; ++r) u[r] = cmul(u[r], pw[r]);
#else
#pragma unroll
      for (int r = 1; r < R; ++r) u[r] = cmul(u[r], twid<DIR>(ldg_ordered(twk + (r - 1) * NS)));
#endif
    }
    Dft<R, DIR>::run(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + r * BPT] = u[r];
  }
}

// padE(x + r·stride) = padE(x) + r·pad_step(stride) for every r of a stage
// when stride is a multiple of E, or stride = 1 with x a multiple of R and
// R dividing E (the run x .. x + R - 1 stays inside one E-block): then all
// accesses of a stage are one base address plus immediate offsets.
template <int E, int R, int STRIDE>
struct PadStep {
  static constexpr bool lin = STRIDE % E == 0 || (STRIDE == 1 && E % R == 0);
  static constexpr int step = STRIDE + STRIDE / E;
};

// After reg_stage<R,N,E,NS>: v[b + r·BPT] holds output index base_b + r·NS.
template <int R, int N, int E, int NS>
__device__ __forceinline__ void store_stage(const double2 (&v)[E], double2* S) {
  constexpr int NT = N / E, BPT = E / R;
  const int tid = tid_fresh();
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = tid + b * NT;
    const int base = (j / NS) * NS * R + (j % NS);
    if constexpr (PadStep<E, R, NS>::lin) {
      double2* Sb = S + padE<E>(base);
#pragma unroll
      for (int r = 0; r < R; ++r) Sb[r * PadStep<E, R, NS>::step] = v[b + r * BPT];
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) S[padE<E>(base + r * NS)] = v[b + r * BPT];
    }
  }
}

template <int N, int E>
__device__ __forceinline__ void load_strided(double2 (&v)[E], const double2* S) {
  constexpr int NT = N / E;
  const int tid = tid_fresh();
  if constexpr (NT % E == 0) {
    const double2* Sb = S + padE<E>(tid);
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = Sb[q * (NT + NT / E)];
  } else {
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = S[padE<E>(tid + q * NT)];
  }
}

template <int N, int E>
__device__ __forceinline__ void store_strided(const double2 (&v)[E], double2* S) {
  constexpr int NT = N / E;
  const int tid = tid_fresh();
  if constexpr (NT % E == 0) {
    double2* Sb = S + padE<E>(tid);
#pragma unroll
    for (int q = 0; q < E; ++q) Sb[q * (NT + NT / E)] = v[q];
  } else {
#pragma unroll
    for (int q = 0; q < E; ++q) S[padE<E>(tid + q * NT)] = v[q];
  }
}

// tws: all stages' twiddle tables back to back (stage I >= 1 at offset OFF,
// NS·(R-1) entries each; see qmc_plan.d_tws).
template <int N, int E, int DIR, int NS, int I, int OFF>
__device__ __forceinline__ void fftE_rec(double2 (&v)[E], double2* S, const double2* __restrict__ tws, int tid) {
  if constexpr (I < RPlan<N, E>::count) {
    constexpr int R = RPlan<N, E>::get(I);
    if constexpr (I > 0) {
      constexpr int RP = RPlan<N, E>::get(I - 1);
      __syncthreads();
      store_stage<RP, N, E, NS / RP>(v, S);
      __syncthreads();
      load_strided<N, E>(v, S);
    }
    reg_stage<R, N, E, NS, DIR>(v, tws + OFF, tid);
    fftE_rec<N, E, DIR, NS * R, I + 1, (I > 0 ? OFF + NS * (R - 1) : OFF)>(v, S, tws, tid);
  }
}

template <int N, int E, int DIR>
__device__ __forceinline__ void fftE(double2 (&v)[E], double2* S, const double2* __restrict__ tws, int tid) {
  fftE_rec<N, E, DIR, 1, 0, 0>(v, S, tws, tid);
}

// Forward FFT fused with the pointwise product by the spectrum row Wr
// (natural order, Wr[tid + q·NT] for v[q]): the first E/2 spectrum values are
// loaded while the last exchange is in flight, the rest after the last
// butterflies; dc receives the unmultiplied v[0] (the DC term for tid 0).
template <int N, int E, int NS, int I, int OFF>
__device__ __forceinline__ void fftE_fwd_w_rec(double2 (&v)[E], double2* S, const double2* __restrict__ tws, int tid,
                                               const double2* __restrict__ Wr, double2& dc) {
  if constexpr (I < RPlan<N, E>::count) {
    constexpr int R = RPlan<N, E>::get(I);
    constexpr bool LAST = I + 1 == RPlan<N, E>::count;
    constexpr int NT = N / E, H = E / 2;
    double2 wv[LAST ? H : 1];
    if constexpr (I > 0) {
      constexpr int RP = RPlan<N, E>::get(I - 1);
      __syncthreads();
      store_stage<RP, N, E, NS / RP>(v, S);
      if constexpr (LAST) {
        const double2* Wt = Wr + tid_fresh();
#pragma unroll
        for (int q = 0; q < H; ++q) wv[q] = ldg_ordered(&Wt[q * NT]);
      }
      __syncthreads();
      load_strided<N, E>(v, S);
    } else if constexpr (LAST) {
      const double2* Wt = Wr + tid_fresh();
#pragma unroll
      for (int q = 0; q < H; ++q) wv[q] = ldg_ordered(&Wt[q * NT]);
    }
    reg_stage<R, N, E, NS, -1>(v, tws + OFF, tid);
    if constexpr (LAST) {
      dc = v[0];
#pragma unroll
      for (int q = 0; q < H; ++q) v[q] = cmul(v[q], wv[q]);
      const double2* Wt = Wr + tid_fresh();
#pragma unroll
      for (int q = H; q < E; ++q) v[q] = cmul(v[q], ldg_ordered(&Wt[q * NT]));
    }
    fftE_fwd_w_rec<N, E, NS * R, I + 1, (I > 0 ? OFF + NS * (R - 1) : OFF)>(v, S, tws, tid, Wr, dc);
  }
}

template <int N, int E>
__device__ __forceinline__ void fftE_fwd_w(double2 (&v)[E], double2* S, const double2* __restrict__ tws, int tid,
                                           const double2* __restrict__ Wr, double2& dc) {
  fftE_fwd_w_rec<N, E, 1, 0, 0>(v, S, tws, tid, Wr, dc);
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

// twN[k·ts] = ω_N^k (a table of a multiple of N read with stride ts).
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
        y[r * M + k2] = (r * k2 == 0) ? sv[k2] : cmul(sv[k2], twid<DIR>(__ldg(&twN[r * k2 * ts])));
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
