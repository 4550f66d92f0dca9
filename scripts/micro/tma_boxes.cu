// Micro-benchmark: stage the 160 volumes a 3D p=4 update reads (interior + 6 face slabs) of
// each 6^3 haloed AoS patch with three strided TMA tensor boxes, against one bulk copy of the
// whole 8,640-byte patch.  Checks the boxes' contents, then times a persistent read-only
// sweep over 1M patches (ring of NST stages per CTA, 8 CTAs/SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_boxes.cu -lcuda -o tma_boxes
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void load4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
               ::"r"(su32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(n), "r"(su32(b)) : "memory");
}

constexpr int BX = 22;                        // x = 4 .. 25 doubles of a haloed row (16-byte aligned start)
constexpr int A_D = 96 * 5, B_D = BX * 2 * 4, C_D = BX * 4 * 2, PD = A_D + B_D + C_D;   // doubles per staged patch
constexpr int NST = 3;

__global__ void check_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                             const __grid_constant__ CUtensorMap mc, double* out, int pid, int mask, int x0) {
  __shared__ __align__(128) double s[PD];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    expect_tx(&bar, ((mask & 1) * A_D + (mask >> 1 & 1) * B_D + (mask >> 2 & 1) * C_D) * 8);
    if (mask & 1) load4(s, &ma, 0, 1, 1, pid, &bar);
    if (mask & 2) load4(s + A_D, &mb, x0, 0, 1, pid, &bar);
    if (mask & 4) load4(s + A_D + B_D, &mc, x0, 1, 0, pid, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < PD; i += blockDim.x) out[i] = s[i];
}

template <bool BOXES>
__global__ void __launch_bounds__(64) sweep(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                           const __grid_constant__ CUtensorMap mc, const double* q, int n, double* sink) {
  constexpr int STG = BOXES ? PD : 216 * 5;
  extern __shared__ __align__(128) double s[];
  __shared__ uint64_t bars[NST];
  if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&bars[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const int my = n > (int)blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto issue = [&](int g) {
    const int pid = blockIdx.x + g * gridDim.x, st = g % NST;
    double* d = s + st * STG;
    if (BOXES) {
      expect_tx(&bars[st], PD * 8);
      load4(d, &ma, 0, 1, 1, pid, &bars[st]);
      load4(d + A_D, &mb, 4, 0, 1, pid, &bars[st]);
      load4(d + A_D + B_D, &mc, 4, 1, 0, pid, &bars[st]);
    } else {
      expect_tx(&bars[st], 216 * 5 * 8);
      bulk(d, q + (size_t)pid * 216 * 5, 216 * 5 * 8, &bars[st]);
    }
  };
  if (threadIdx.x == 0) for (int g = 0; g < NST && g < my; ++g) issue(g);
  double acc = 0.0;
  for (int g = 0; g < my; ++g) {
    mbar_wait(&bars[g % NST], (g / NST) & 1);
    acc += s[(g % NST) * STG + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && g + NST < my) issue(g + NST);
  }
  if (acc == 12345.678) sink[0] = acc;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int mask = argc > 1 ? atoi(argv[1]) : 7, x0 = argc > 2 ? atoi(argv[2]) : 4, bstride = argc > 3 ? atoi(argv[3]) : 5;
  const int n = 1 << 20;
  const size_t nd = (size_t)n * 216 * 5;
  double* q;
  CK(cudaMalloc(&q, nd * 8));
  std::vector<double> h(216 * 5 * 4);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  CK(cudaMemcpy(q, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr));
  Enc enc = (Enc)fp;
  CUtensorMap ma, mb, mc;
  const cuuint64_t dims[4] = {30, 6, 6, (cuuint64_t)n};
  const cuuint64_t str[3] = {240, 1440, 8640};
  const cuuint32_t ba[4] = {30, 4, 4, 1}, bb[4] = {BX, 6, 4, 1}, bc[4] = {BX, 4, 6, 1};
  const cuuint32_t e1[4] = {1, 1, 1, 1}, eb[4] = {1, (cuuint32_t)bstride, 1, 1}, ec[4] = {1, 1, (cuuint32_t)bstride, 1};
  int r1 = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, q, dims, str, ba, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int r2 = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, q, dims, str, bb, eb, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int r3 = enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, q, dims, str, bc, ec, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d %d %d\n", r1, r2, r3);
  if (r1 || r2 || r3) return 1;
  double* out;
  CK(cudaMalloc(&out, PD * 8));
  check_kernel<<<1, 64>>>(ma, mb, mc, out, 2, mask, x0);
  CK(cudaDeviceSynchronize());
  printf("mask %d x0 %d stride %d: ok\n", mask, x0, bstride);
  if (mask != 7 || x0 != 4 || bstride != 5) return 0;
  std::vector<double> o(PD);
  CK(cudaMemcpy(o.data(), out, PD * 8, cudaMemcpyDeviceToHost));
  // expected: box A [z 1..4][y 1..4][x 0..5], B [z 1..4][y 0,5][x 1..4], C [z 0,5][y 1..4][x 1..4]
  int bad = 0, k = 0;
  auto vol = [&](int z, int y, int x, int u) { return (double)(((2 * 6 + z) * 6 + y) * 6 * 5 + x * 5 + u); };
  for (int z = 1; z <= 4; ++z) for (int y = 1; y <= 4; ++y) for (int x = 0; x < 6; ++x) for (int u = 0; u < 5; ++u) bad += o[k++] != vol(z, y, x, u);
  auto row = [&](int z, int y, int j) { return (double)(((2 * 6 + z) * 6 + y) * 30 + j); };
  for (int z = 1; z <= 4; ++z) for (int y = 0; y <= 5; y += 5) for (int j = 4; j < 4 + BX; ++j) bad += o[k++] != row(z, y, j);
  for (int z = 0; z <= 5; z += 5) for (int y = 1; y <= 4; ++y) for (int j = 4; j < 4 + BX; ++j) bad += o[k++] != row(z, y, j);
  printf("box contents: %d mismatches of %d\n", bad, PD);
  if (bad) { for (int i = 0; i < 12; ++i) printf(" %g", o[A_D + i]); printf("\n"); }
  double* sink;
  CK(cudaMalloc(&sink, 8));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep)
    for (int boxes = 0; boxes < 2; ++boxes) {
      const int smem = NST * (boxes ? PD : 1080) * 8;
      if (boxes) CK(cudaFuncSetAttribute(sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      else CK(cudaFuncSetAttribute(sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      for (int per = 8; per <= 16; per += 8) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        const int grid = sms * per;
        for (int it = 0; it < 2; ++it) {
          cudaEventRecord(a);
          if (boxes) sweep<true><<<grid, 64, smem>>>(ma, mb, mc, q, n, sink);
          else sweep<false><<<grid, 64, smem>>>(ma, mb, mc, q, n, sink);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)n * (boxes ? PD : 1080) * 8;
        printf("%s CTAs/SM %2d: %.3f ms, %.0f GB/s of staged bytes, %.1f Mpatch/s\n", boxes ? "3 boxes (160 vol)" : "1 bulk (216 vol) ",
               per, ms, bytes / ms / 1e6, n / ms / 1e3);
      }
    }
  return 0;
}
