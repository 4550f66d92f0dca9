// fvb_halo_tma.cu -- halo_project (mesh.py:261-310) for AoS batches with the
// tensor-memory-access engine doing the bulk of the copy.
//
// Work item: one destination haloed z-plane (hz) of one patch (2D: the patch).
// The plane's interior block (hy = 1..p, hx = 1..p: p rows of p*s doubles) is
// one box of one source plane of one source patch, and each y-halo row
// (hy = 0, p+1; hx = 1..p) one row of a y-neighbour: three TMA loads into a
// shared-memory stage, three TMA stores into QIn at inner coordinate s (the
// tensor map does the s-double row offset and the row pitch e*s).  The x-halo
// columns (hx = 0, p+1, every hy: 2*e*s doubles) are s-double pieces in
// other patches' rows, so warps copy them directly while the TMA traffic is
// in flight.  TMA needs 16-byte aligned global addresses, so this path serves
// s = 4 (2D); 3D's 40-byte volumes keep the thread-copy kernels
// (fvb_generic.cu).  Bytes written are disjoint, so the two paths
// need no ordering.  Pure data movement: bit-exact by construction.
//
// CTA = 1 + XW warps over items blockIdx.x + k * gridDim.x.  Lane 0 of warp 0 runs
// an NST-stage ring (mbarrier complete_tx for the loads, one bulk group per
// item for the stores, a stage is refilled once its stores have finished
// reading it); warps 1..XW copy the x-halo columns of every XW-th item.
#include <cuda_runtime.h>

#include "fvb_kernels.h"
#include "fvb_tma.cuh"

namespace fvb {
namespace hx {

using namespace f16;

constexpr int NST = 4;

constexpr int XW = 3;      // x-halo warps per CTA (warp 0 drives the TMA ring)
constexpr int XB = 8;      // x-halo doubles per lane per batch (all loads before the stores)

struct Geo {
  int d, p, e, s, nz, gx, gy, gz, periodic;
  int ps, es;                 // interior / haloed row length in doubles
  int plane_b, row_b, stage_b;  // stage layout (bytes, 128-aligned)
  int64_t n, I, V;
};

struct Src {
  int c, i;
};
__device__ __forceinline__ Src src_of(int c, int h, int p, int ext, int periodic) {
  if (h == 0) {
    if (c > 0) return {c - 1, p - 1};
    return periodic ? Src{ext - 1, p - 1} : Src{0, 0};
  }
  if (h == p + 1) {
    if (c < ext - 1) return {c + 1, 0};
    return periodic ? Src{0, 0} : Src{ext - 1, p - 1};
  }
  return {c, h - 1};
}

__global__ void __launch_bounds__(32 * (1 + XW))
halo_tma_kernel(const double* __restrict__ qout, double* __restrict__ qin, Geo G,
                const __grid_constant__ CUtensorMap ld_plane, const __grid_constant__ CUtensorMap ld_row,
                const __grid_constant__ CUtensorMap st_plane, const __grid_constant__ CUtensorMap st_row) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[NST];
  unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);   // TMA boxes: 128-B aligned
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // items blockIdx.x, +gridDim.x, ...: the CTAs in flight cover a window of
  // consecutive items, so neighbour rows read by one were just read by another (L2)
  const int64_t items = G.n * G.nz;
  if ((int64_t)blockIdx.x >= items) return;
  const int count = (int)((items - 1 - blockIdx.x) / gridDim.x + 1);
  auto item_of = [&](int j) { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };
  const bool d3 = G.d == 3;

  struct Cur {   // item -> (patch, hz, cx, cy, cz)
    int64_t patch;
    int hz, cx, cy, cz;
  };
  auto decompose = [&](int64_t item) {
    Cur c;
    c.patch = item / G.nz;
    c.hz = (int)(item - c.patch * G.nz);
    c.cx = (int)(c.patch % G.gx);
    const int64_t r = c.patch / G.gx;
    c.cy = (int)(r % G.gy);
    c.cz = (int)(r / G.gy);
    return c;
  };
  auto src_patch = [&](int x, int y, int z) -> int64_t { return ((int64_t)z * G.gy + y) * G.gx + x; };

  if (warp > 0) {
    // ---- x-halo columns (hx = 0 and p+1 of every hy) of items warp-1, warp-1+XW, ...
    const int xn = 2 * G.es;
    for (int j = warp - 1; j < count; j += XW) {
      const Cur c = decompose(item_of(j));
      const Src zs = d3 ? src_of(c.cz, c.hz, G.p, G.gz, G.periodic) : Src{0, 0};
      const Src xl = src_of(c.cx, 0, G.p, G.gx, G.periodic), xr = src_of(c.cx, G.p + 1, G.p, G.gx, G.periodic);
      double* dplane = qin + (c.patch * G.V + (int64_t)c.hz * G.e * G.e) * G.s;
      for (int t0 = 0; t0 < xn; t0 += 32 * XB) {
        double v[XB];
        int64_t dof[XB];
#pragma unroll
        for (int k = 0; k < XB; ++k) {
          const int t = t0 + lane + 32 * k;
          dof[k] = -1;
          if (t < xn) {
            const int side = t >= G.es;
            const int rem = t - side * G.es;
            const int hy = rem / G.s, u = rem - hy * G.s;
            const Src ys = src_of(c.cy, hy, G.p, G.gy, G.periodic);
            const Src xs = side ? xr : xl;
            const int64_t sp = src_patch(xs.c, ys.c, zs.c);
            v[k] = __ldg(qout + (sp * G.I + ((int64_t)zs.i * G.p + ys.i) * G.p + xs.i) * G.s + u);
            dof[k] = ((int64_t)hy * G.e + (side ? G.e - 1 : 0)) * G.s + u;
          }
        }
#pragma unroll
        for (int k = 0; k < XB; ++k)
          if (dof[k] >= 0) __stcs(dplane + dof[k], v[k]);
      }
    }
    return;
  }
  if (lane != 0) return;

  // ---- lane 0 of warp 0: interior block + y-halo rows through the TMA ring
  auto issue_loads = [&](const Cur& c, int stg) {
    unsigned char* b = smem + stg * G.stage_b;
    const Src zs = d3 ? src_of(c.cz, c.hz, G.p, G.gz, G.periodic) : Src{0, 0};
    const Src lo = src_of(c.cy, 0, G.p, G.gy, G.periodic), hi = src_of(c.cy, G.p + 1, G.p, G.gy, G.periodic);
    mbar_expect_tx(&full[stg], (uint32_t)((G.p + 2) * G.ps * 8));
    tma_load_4d(b, &ld_plane, 0, 0, zs.i, (int)src_patch(c.cx, c.cy, zs.c), &full[stg]);
    tma_load_4d(b + G.plane_b, &ld_row, 0, lo.i, zs.i, (int)src_patch(c.cx, lo.c, zs.c), &full[stg]);
    tma_load_4d(b + G.plane_b + G.row_b, &ld_row, 0, hi.i, zs.i, (int)src_patch(c.cx, hi.c, zs.c), &full[stg]);
  };
  for (int k = 0; k < NST; ++k) mbar_init(&full[k], 1);
  fence_mbar_init();
  for (int k = 0; k < NST && k < count; ++k) issue_loads(decompose(item_of(k)), k);
  for (int j = 0; j < count; ++j) {
    const Cur cur = decompose(item_of(j));
    const int stg = j % NST;
    mbar_wait(&full[stg], (uint32_t)((j / NST) & 1));
    const unsigned char* b = smem + stg * G.stage_b;
    const int pz = (int)cur.patch;
    tma_store_4d(&st_plane, G.s, 1, cur.hz, pz, b);
    tma_store_4d(&st_row, G.s, 0, cur.hz, pz, b + G.plane_b);
    tma_store_4d(&st_row, G.s, G.e - 1, cur.hz, pz, b + G.plane_b + G.row_b);
    bulk_commit();
    // the stores of item j-1 have finished reading their stage: refill it with item j-1+NST
    if (j >= 1 && j - 1 + NST < count) {
      bulk_wait_read<1>();
      issue_loads(decompose(item_of(j - 1 + NST)), (j - 1) % NST);
    }
  }
  bulk_wait_all0();
}

cudaError_t make_map(CUtensorMap* tm, const double* base, const cuuint64_t (&dims)[4], const cuuint64_t (&strides)[3],
                     const cuuint32_t (&box)[4]) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace hx
}  // namespace fvb

using namespace fvb;

bool fvb_halo_tma_supported(int dim, int p) {
  const int s = dim + 2, e = p + 2;
  // TMA global addresses must be 16-byte aligned: row pitches and the store's inner
  // coordinate s (2D: 32 B; 3D's 40 B is not, so 3D keeps the thread-copy kernels),
  // and the interior row is one box of <= 256 elements
  return (dim == 2 || dim == 3) && p >= 1 && s % 2 == 0 && (p * s) % 2 == 0 && (e * s) % 2 == 0 && p * s <= 256 &&
         hx::encode_tiled() != nullptr;
}

cudaError_t fvb_launch_halo_tma(int dim, int p, int64_t n, const double* qout, double* qin, const int* grid,
                                int periodic, cudaStream_t st) {
  using namespace hx;
  Geo G;
  G.d = dim;
  G.p = p;
  G.e = p + 2;
  G.s = dim + 2;
  G.nz = dim == 3 ? G.e : 1;
  G.gx = grid[0];
  G.gy = grid[1];
  G.gz = dim == 3 ? grid[2] : 1;
  G.periodic = periodic;
  G.ps = p * G.s;
  G.es = G.e * G.s;
  G.plane_b = (p * G.ps * 8 + 127) / 128 * 128;
  G.row_b = (G.ps * 8 + 127) / 128 * 128;
  G.stage_b = G.plane_b + 2 * G.row_b;
  G.n = n;
  G.I = dim == 3 ? (int64_t)p * p * p : (int64_t)p * p;
  G.V = dim == 3 ? (int64_t)G.e * G.e * G.e : (int64_t)G.e * G.e;
  const int pz = dim == 3 ? p : 1;
  CUtensorMap ld_plane, ld_row, st_plane, st_row;
  const cuuint64_t odims[4] = {(cuuint64_t)G.ps, (cuuint64_t)p, (cuuint64_t)pz, (cuuint64_t)n};
  const cuuint64_t ostr[3] = {(cuuint64_t)G.ps * 8, (cuuint64_t)G.ps * p * 8, (cuuint64_t)G.I * G.s * 8};
  const cuuint64_t idims[4] = {(cuuint64_t)G.es, (cuuint64_t)G.e, (cuuint64_t)G.nz, (cuuint64_t)n};
  const cuuint64_t istr[3] = {(cuuint64_t)G.es * 8, (cuuint64_t)G.es * G.e * 8, (cuuint64_t)G.V * G.s * 8};
  const cuuint32_t bplane[4] = {(cuuint32_t)G.ps, (cuuint32_t)p, 1u, 1u};
  const cuuint32_t brow[4] = {(cuuint32_t)G.ps, 1u, 1u, 1u};
  cudaError_t e = make_map(&ld_plane, qout, odims, ostr, bplane);
  if (e == cudaSuccess) e = make_map(&ld_row, qout, odims, ostr, brow);
  if (e == cudaSuccess) e = make_map(&st_plane, qin, idims, istr, bplane);
  if (e == cudaSuccess) e = make_map(&st_row, qin, idims, istr, brow);
  if (e != cudaSuccess) return e;
  const size_t bytes = (size_t)NST * G.stage_b + 128;
  e = cudaFuncSetAttribute(halo_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, halo_tma_kernel, 32 * (1 + XW), bytes);
  if (per_sm < 1) per_sm = 1;
  const int64_t items = n * G.nz;
  int64_t ctas = (int64_t)sms * per_sm;
  if (ctas > items) ctas = items;
  halo_tma_kernel<<<(unsigned)ctas, 32 * (1 + XW), bytes, st>>>(qout, qin, G, ld_plane, ld_row, st_plane, st_row);
  return cudaGetLastError();
}
