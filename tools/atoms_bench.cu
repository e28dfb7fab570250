// Microbenchmark: shared-memory atomic throughput on B200 (int RED, float CAS loop, conflict-free lanes).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int* out, int iters, float val) {
  __shared__ int si[4096];
  __shared__ float sf[4096];
  for (int t = threadIdx.x; t < 4096; t += blockDim.x) { si[t] = 0; sf[t] = 0.f; }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int a = ((w * 8 + k) * 32 + lane + it) & 4095;  // distinct banks per instruction
      if (MODE == 0) atomicAdd(&si[a], it + k + lane);
      else if (MODE == 1) atomicAdd(&sf[a], val);
      else if (MODE == 2) { si[a] += 1; }
      else { atomicAdd(&si[a], __float2int_rn(val * (float)(a + it))); }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = si[0] + (int)sf[1] + acc;
}
int main() {
  int* d; cudaMalloc(&d, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[4] = {"int atomicAdd (RED.shared)", "float atomicAdd (CAS loop)", "plain ld/add/st", "F2I + int atomicAdd"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int threads : {128, 256}) {
      int blocks = sms * (2048 / threads) / 2;
      int iters = 2000;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<blocks, threads>>>(d, iters, 1.f);
        if (mode == 1) k<1><<<blocks, threads>>>(d, iters, 1.f);
        if (mode == 2) k<2><<<blocks, threads>>>(d, iters, 1.f);
        if (mode == 3) k<3><<<blocks, threads>>>(d, iters, 1.f);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * threads * iters * 8;
      printf("%-28s threads %d: %.3f ms, %.1f lane-ops/clk/SM (at 1.95 GHz)\n", names[mode], threads, ms,
             ops / (ms * 1e-3) / sms / 1.95e9);
    }
  }
  return 0;
}
