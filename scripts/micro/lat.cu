// Latency / throughput microbenchmark for FP64 ops on the B200 (dependent chains, one warp and many warps).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_dadd(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __dadd_rn(x, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void chain_dmul(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __dmul_rn(x, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void chain_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __fma_rn(x, b, a);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// 8 independent chains per thread: throughput
__global__ void indep_dadd(double* out, long long* cyc, double a, double b, int n) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __dadd_rn(x[j], b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void chain_lds(double* out, long long* cyc, int n) {
  __shared__ int sidx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sidx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) p = sidx[p];
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = p;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  long long h[1024];
  const int n = 1000;
  auto run = [&](const char* name, auto kern, int blocks, int threads, double ops_per_thread) {
    kern<<<blocks, threads>>>(out, cyc, 1.0000001, 1e-9, n);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, cyc, 1.0000001, 1e-9, n);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, cyc, sizeof(long long) * 1, cudaMemcpyDeviceToHost);
    double tot = ops_per_thread * blocks * threads;
    printf("%-12s blocks %4d thr %4d: %.2f cyc/op (thread 0 chain), %.2f Gop/s (%.1f%% of 64/clk/SM @1.965GHz)\n", name, blocks,
           threads, (double)h[0] / ops_per_thread, tot / ms / 1e6, 100.0 * tot / (ms * 1e-3) / (148 * 64 * 1.965e9));
  };
  for (int th : {32, 128, 256, 512}) run("dadd-chain", chain_dadd, 1, th, 16.0 * n);
  run("dmul-chain", chain_dmul, 1, 32, 16.0 * n);
  run("dfma-chain", chain_dfma, 1, 32, 16.0 * n);
  for (int th : {32, 64, 128, 256}) run("dadd-indep8", indep_dadd, 148, th, 128.0 * n);
  run("dadd-chain", chain_dadd, 148 * 4, 512, 16.0 * n);
  chain_lds<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  printf("lds-chain: %.2f cyc/op\n", (double)h[0] / (16.0 * n));
  return 0;
}
