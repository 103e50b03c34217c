// Feasibility probe: green-context SM partitions driven through runtime-API
// launches on memory allocated in the primary context.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__global__ void k_smid(int* out, double* buf, long n) {
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) out[blockIdx.x] = int(sm);
  for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) buf[i] += 1.0;
}
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
int main() {
  cudaFree(0);
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("SMs %u\n", all.sm.smCount);
  unsigned ng = 0; CUdevResource rem;
  CK(cuDevSmResourceSplitByCount(nullptr, &ng, &all, nullptr, 0, 8));
  std::vector<CUdevResource> g(ng);
  CK(cuDevSmResourceSplitByCount(g.data(), &ng, &all, &rem, 0, 8));
  printf("groups %u of %u, remainder %u\n", ng, g[0].sm.smCount, rem.sm.smCount);
  const int nk2 = 3;  // groups for the second partition
  std::vector<CUdevResource> a(g.begin(), g.end() - nk2), b(g.end() - nk2, g.end());
  if (rem.sm.smCount) a.push_back(rem);
  CUdevResourceDesc da, db; CK(cuDevResourceGenerateDesc(&da, a.data(), a.size())); CK(cuDevResourceGenerateDesc(&db, b.data(), b.size()));
  CUgreenCtx ga, gb; CK(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM)); CK(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb; CK(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0)); CK(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  const long n = 1 << 24; double* buf; cudaMalloc(&buf, n * 8); cudaMemset(buf, 0, n * 8);
  int* sm; cudaMalloc(&sm, 4096 * 4);
  cudaDeviceSynchronize();
  for (int w = 0; w < 2; ++w) {
    cudaStream_t s = (cudaStream_t)(w ? sb : sa);
    cudaMemset(sm, 0xff, 4096 * 4);
    k_smid<<<2048, 256, 0, s>>>(sm, buf, n);
    printf("launch %d: %s\n", w, cudaGetErrorString(cudaGetLastError()));
    printf("sync: %s\n", cudaGetErrorString(cudaStreamSynchronize(s)));
    std::vector<int> h(2048); cudaMemcpy(h.data(), sm, 2048 * 4, cudaMemcpyDeviceToHost);
    std::vector<int> used(256, 0); int cnt = 0;
    for (int x : h) if (x >= 0 && x < 256 && !used[x]++) ++cnt;
    printf("partition %d: distinct SMs %d\n", w, cnt);
  }
  std::vector<double> hb(4); cudaMemcpy(hb.data(), buf, 32, cudaMemcpyDeviceToHost);
  printf("buf[0] = %g (expect 2)\n", hb[0]);
  // concurrency: a long kernel on each partition at once, events timing
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, (cudaStream_t)sa);
  for (int r = 0; r < 20; ++r) { k_smid<<<2048, 256, 0, (cudaStream_t)sa>>>(sm, buf, n); k_smid<<<2048, 256, 0, (cudaStream_t)sb>>>(sm + 2048, buf, n); }
  cudaEventRecord(e1, (cudaStream_t)sa);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("both partitions: %s, %.3f ms\n", cudaGetErrorString(cudaGetLastError()), ms);
  return 0;
}
