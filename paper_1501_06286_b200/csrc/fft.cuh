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
