// Does SHFL share the shared-memory data pipe with LDS?  Throughput of LDS.64 alone,
// SHFL alone, and both interleaved (independent streams), 4 CTAs x 256 threads per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int n) {
  __shared__ double buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = i * 0.5;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int lane = threadIdx.x & 31;
  int base = (threadIdx.x >> 5) * 64 + lane;
  double v = lane * 1.0, w = lane * 2.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0 || MODE == 2) {
        acc0 += buf[(base + k * 32 + i) & 2047];
        acc1 += buf[(base + k * 32 + 256 + i) & 2047];
      }
      if (MODE == 1 || MODE == 2) {
        v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31);
        w = __shfl_sync(0xffffffffu, w, (lane + 31) & 31);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3 + v + w;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  const int n = 2000, blocks = 148 * 4;
  auto run = [&](const char* name, void (*kern)(double*, int), double lds, double shfl) {
    kern<<<blocks, 256>>>(out, n); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kern<<<blocks, 256>>>(out, n); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warps = blocks * 8.0, cyc = ms * 1e-3 * 1.965e9;
    printf("%-10s %.3f ms  LDS.64/SM/cyc %.3f  SHFL.32/SM/cyc %.3f\n", name, ms, warps * n * 8 * lds / 148 / cyc,
           warps * n * 8 * shfl / 148 / cyc);
  };
  run("lds", k<0>, 2, 0);
  run("shfl", k<1>, 0, 4);
  run("both", k<2>, 2, 4);
  return 0;
}
