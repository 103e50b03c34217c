// fp64_peak.cu — measured fp64 CUDA-core peak of the B200 in this pool (the
// roofline denominator of K1).  Every SM runs CTAs of
// independent DFMA / DMUL / DADD chains (8 chains per thread, 32 warps per
// SM) for a fixed number of iterations; the rate is instructions per second
// from CUDA events, best of R repetitions, with the SM clock sampled by the
// caller (tools/fp64_peak.sh).  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int kChains = 8;

template <int OP>
__global__ void __launch_bounds__(256) k_fp64(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if (OP == 0) x[c] = fma(x[c], a, b);  // DFMA
        if (OP == 1) x[c] = x[c] * a;         // DMUL
        if (OP == 2) x[c] = x[c] + b;         // DADD
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

template <int OP>
static double run(int nsm, int iters, int reps, double* d) {
  const int blocks = nsm * 8, threads = 256;  // 8 CTAs x 8 warps = 64 warps per SM
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64<OP><<<blocks, threads>>>(d, iters / 10, 0.999999, 1e-9);  // warm-up
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    k_fp64<OP><<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = double(blocks) * threads * iters * 16.0 * kChains;
    const double rate = inst / (ms * 1e-3);  // thread instructions per second
    if (rate > best) best = rate;
  }
  return best;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz (max)
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  double* d;
  cudaMalloc(&d, 64);
  const int iters = 40000, reps = 5;
  const double dfma = run<0>(nsm, iters, reps, d);
  const double dmul = run<1>(nsm, iters, reps, d);
  const double dadd = run<2>(nsm, iters, reps, d);
  const cudaError_t err = cudaGetLastError();
  // per SM per clock at the maximum SM clock
  const double per_clk = dfma / (double(nsm) * clk * 1e3);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_max_mhz\": %.0f, "
         "\"dfma_inst_per_s\": %.6e, \"dmul_inst_per_s\": %.6e, \"dadd_inst_per_s\": %.6e, "
         "\"fp64_tflops_fma\": %.4f, \"dfma_per_sm_per_clk_at_max\": %.2f, \"cuda_error\": \"%s\", "
         "\"how\": \"%d CTAs x 256 threads, %d independent chains per thread, %d x 16 unrolled ops; best of %d; "
         "TFLOP/s = 2 x DFMA rate\"}\n",
         prop.name, nsm, clk / 1e3, dfma, dmul, dadd, 2.0 * dfma / 1e12, per_clk, cudaGetErrorString(err),
         nsm * 8, kChains, iters, reps);
  return err == cudaSuccess ? 0 : 1;
}
