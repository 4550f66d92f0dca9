// fvb_fused2d.cu -- fused 2D Rusanov patch update for p = 16 patches.
//
// One persistent CTA (8 "interior" warps + 1 "halo" warp, 2 CTAs per SM)
// streams whole haloed patches (18x18x4 doubles = 10,368 B) through a ring
// of TMA bulk-copy stages (cp.async.bulk + mbarrier complete_tx), one patch
// per iteration:
//
//   A  interior lanes (lane -> x, two rows per warp) evaluate the Euler
//      closure of their volume once (9 quotients sharing one reciprocal
//      refinement, fvb_exact.cuh) and publish x- and y-side data; the halo
//      warp evaluates the 64 face-halo volumes.                  -- barrier
//   B  each lane accumulates its cell's four face terms in the reference
//      order (vectorized.py:161-200) from the published side data and
//      writes the patch's interior to a staging buffer that one thread
//      stores with a TMA bulk store; the per-patch max wave speed
//      (vectorized.py:226-231) is reduced with warp shuffles.
//
// Quotients that need CUDA's division slow path (zero / tiny numerators,
// huge densities) are not evaluated here: the patch is queued on the redo
// list in the status buffer and re-evaluated exactly by fvb_redo_kernel.
#include <cuda_runtime.h>

#include <cstdlib>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tail.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace f2 {

using namespace f16;

constexpr int P = 16, E = 18, S = 4;
constexpr int PLANE = E * E;
constexpr int STAGE = PLANE * S;       // one haloed patch
constexpr int NST = 4;
constexpr int64_t VOL = (int64_t)E * E;
constexpr int64_t IVOL = (int64_t)P * P;
constexpr int SIDE = S * E * P;        // side buffer: 4 comps (lam, f[0..2]) x 18 x 16
constexpr int OUTN = P * P * S;
constexpr int OFF_RING = 0;
constexpr int OFF_YS = OFF_RING + NST * STAGE;
constexpr int OFF_XS = OFF_YS + 2 * SIDE;
constexpr int OFF_OUT = OFF_XS + 2 * SIDE;
constexpr int OFF_WMAX = OFF_OUT + 2 * OUTN;
constexpr int OFF_INV = OFF_WMAX + 16;      // (inv, half_inv) per patch parity
constexpr int OFF_FLAG = OFF_INV + 4;
constexpr int OFF_BAR = OFF_FLAG + 2;   // 3 flag words (4 B) fit in 2 doubles
constexpr int TOTAL = OFF_BAR + NST;
constexpr size_t BYTES = (size_t)TOTAL * 8;

template <int L>
__device__ __forceinline__ double qs(const double* st, int hy, int hx, int u) {
  return L == kAoS ? st[(hy * E + hx) * S + u] : st[(u * E + hy) * E + hx];
}
template <int L>
__device__ __forceinline__ void load_q(const double* st, int hy, int hx, double (&q)[S]) {
#pragma unroll
  for (int u = 0; u < S; ++u) q[u] = qs<L>(st, hy, hx, u);
}
__device__ __forceinline__ int ys_at(int c, int hy, int x) { return (c * E + hy) * P + x; }
__device__ __forceinline__ int xs_at(int c, int y, int hx) { return (c * P + y) * E + hx; }

__device__ __forceinline__ void put_ys(double* b, int hy, int x, const Side<2>& s) {
  b[ys_at(0, hy, x)] = s.lam;
#pragma unroll
  for (int k = 0; k < 3; ++k) b[ys_at(k + 1, hy, x)] = s.f[k];
}
__device__ __forceinline__ void put_xs(double* b, int y, int hx, const Side<2>& s) {
  b[xs_at(0, y, hx)] = s.lam;
#pragma unroll
  for (int k = 0; k < 3; ++k) b[xs_at(k + 1, y, hx)] = s.f[k];
}

template <int L, int MINB>
__global__ void __launch_bounds__(288, MINB)
fused2d_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
               const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
               int64_t n, Closure cl, CflTail tail) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + OFF_RING;
  double* ysb = sm + OFF_YS;
  double* xsb = sm + OFF_XS;
  double* outb = sm + OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + OFF_WMAX);
  double* invs = sm + OFF_INV;
  unsigned* slowflag = reinterpret_cast<unsigned*>(sm + OFF_FLAG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);

  const int tid = threadIdx.x;
  const bool interior = tid < 256;
  const int warp = tid >> 5, lane = tid & 31;
  const int x = lane & 15;
  const int y = ((warp & 7) << 1) | (lane >> 4);
  const bool producer = tid == 256;

  const int G = (n > (int64_t)blockIdx.x) ? (int)((n - 1 - (int64_t)blockIdx.x) / gridDim.x + 1) : 0;
  auto patch_of = [&](int g) -> int64_t { return (int64_t)blockIdx.x + (int64_t)g * gridDim.x; };

  auto issue = [&](int g) {
    const int64_t pidx = patch_of(g);
    double* st = ring + (g % NST) * STAGE;
    uint64_t* bar = bars + (g % NST);
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)(STAGE * 8));
    if (L == kAoS) {
      tma_load_1d(st, qin + pidx * VOL * S, (uint32_t)(STAGE * 8), bar);
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_load_1d(st + u * PLANE, qin + ((int64_t)u * n + pidx) * VOL, (uint32_t)(PLANE * 8), bar);
    }
  };
  auto store_out = [&](int g) {
    const int64_t pidx = patch_of(g);
    const double* src = outb + (g & 1) * OUTN;
    if (L == kAoS) {
      tma_store_1d(qout + pidx * IVOL * S, src, (uint32_t)(OUTN * 8));
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_store_1d(qout + ((int64_t)u * n + pidx) * IVOL, src + u * P * P, (uint32_t)(P * P * 8));
    }
    bulk_commit();
  };
  auto finish_patch = [&](int g) {
    unsigned long long m = wmax[(g & 1) * 8];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const unsigned long long v = wmax[(g & 1) * 8 + w];
      m = v > m ? v : m;
    }
    const int64_t pidx = patch_of(g);
    max_eig[pidx] = __longlong_as_double((long long)m);
    if (slowflag[g % 3]) {   // queue for the exact re-evaluation
      const unsigned k = atomicAdd(&status[1], 1u);
      status[2 + k] = (unsigned)pidx;
      slowflag[g % 3] = 0;   // slot reused by patch g+3, set only after the next barrier
    }
  };

  if (producer) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    slowflag[0] = slowflag[1] = slowflag[2] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  // dt / dx of a patch, computed once by the producer (vectorized.py:169-170)
  auto put_inv = [&](int g) {
    const int64_t pi = patch_of(g);
    const double dx = __ddiv_rn(cell_size[pi * 2], (double)P);
    const double inv = __ddiv_rn(dtv[pi], dx);
    invs[(g & 1) * 2] = inv;
    invs[(g & 1) * 2 + 1] = dmul(0.5, inv);   // `0.5 * inv * a` evaluates 0.5*inv first
    // the flux rewrite needs 0.5*inv exact: 0 or |inv| >= 2^-1021, finite
    const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
    if (!(inv == 0.0 || (e >= 2u && e < 0x7ffu))) atomicOr(&slowflag[g % 3], 1u);
  };
  if (producer)
    for (int g = 0; g < NST - 1 && g < G; ++g) issue(g);

  unsigned long long cmax = 0;            // this lane's wave speed of the patch in flight
  unsigned stg = 0, par = 0, slot3 = 0;   // ring stage / mbarrier parity / g % 3 of patch g
  // Software pipeline, ONE CTA barrier per patch: iteration g evaluates the
  // closures of patch g (A) and updates patch g-1 (B) from the side data
  // published in iteration g-1.  A(g) and B(g) touch different parities.
  for (int g = 0; g <= G; ++g) {
    const unsigned pstg = stg == 0 ? NST - 1 : stg - 1;   // stage of patch g-1
    const double* st = ring + stg * STAGE;
    double* ys_w = ysb + (g & 1) * SIDE;
    double* xs_w = xsb + (g & 1) * SIDE;
    unsigned long long cnew = 0;
    bool slow = false;
    // ---------------- A: closure of this lane's volume of patch g ----------------
    auto closure_int = [&]() {
      double q[S];
      load_q<L>(st, y + 1, x + 1, q);
      Side<2> sd[2];
      bool ok;
      closure_all_ranged<2>(q, cl, sd, ok);
      slow = slow | !ok;
      const unsigned long long a = (unsigned long long)__double_as_longlong(sd[0].lam);
      const unsigned long long b = (unsigned long long)__double_as_longlong(sd[1].lam);
      cnew = a > b ? a : b;
      put_xs(xs_w, y, x + 1, sd[0]);
      put_ys(ys_w, y + 1, x, sd[1]);
    };
    // ---------------- B: update of this lane's cell of patch g-1 ----------------
    const int gp = g - 1;
    const double* stp = ring + pstg * STAGE;
    const double* ys_r = ysb + (gp & 1) * SIDE;
    const double* xs_r = xsb + (gp & 1) * SIDE;
    auto update_int = [&]() {
      const double half_inv = invs[(gp & 1) * 2 + 1];
      double qc[S], qn[S], val[S];
      load_q<L>(stp, y + 1, x + 1, qc);
#pragma unroll
      for (int u = 0; u < S; ++u) val[u] = qc[u];                       // _pass_copy
      const double lx = xs_r[xs_at(0, y, x + 1)];
      load_q<L>(stp, y + 1, x, qn);
      const double jl = qn[1];
      dissipate<2>(val, half_inv, lx, qc, xs_r[xs_at(0, y, x)], qn);
      load_q<L>(stp, y + 1, x + 2, qn);
      const double jr = qn[1];
      dissipate<2>(val, half_inv, lx, qc, xs_r[xs_at(0, y, x + 2)], qn);
      const double ly = ys_r[ys_at(0, y + 1, x)];
      load_q<L>(stp, y, x + 1, qn);
      const double jd = qn[2];
      dissipate<2>(val, half_inv, ly, qc, ys_r[ys_at(0, y, x)], qn);
      load_q<L>(stp, y + 2, x + 1, qn);
      const double ju = qn[2];
      dissipate<2>(val, half_inv, ly, qc, ys_r[ys_at(0, y + 2, x)], qn);
      // flux differences (vectorized.py:193-200) as RN(half_inv * RN(a - b)), a/b the
      // unscaled face sums: bit-identical to RN(inv * RN(RN(0.5a) - RN(0.5b))) inside
      // the range gate (no subnormals; see fvb_fused3d.cu add_flux).
#pragma unroll
      for (int u = 0; u < S; ++u) {   // x flux difference
        const double fm = u == 0 ? jl : xs_r[xs_at(u, y, x)];
        const double fc = u == 0 ? qc[1] : xs_r[xs_at(u, y, x + 1)];
        const double fp = u == 0 ? jr : xs_r[xs_at(u, y, x + 2)];
        val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
      }
#pragma unroll
      for (int u = 0; u < S; ++u) {   // y flux difference
        const double fm = u == 0 ? jd : ys_r[ys_at(u, y, x)];
        const double fc = u == 0 ? qc[2] : ys_r[ys_at(u, y + 1, x)];
        const double fp = u == 0 ? ju : ys_r[ys_at(u, y + 2, x)];
        val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
      }
      double* ob = outb + (gp & 1) * OUTN;
#pragma unroll
      for (int u = 0; u < S; ++u) {
        if (L == kAoS) ob[(y * P + x) * S + u] = val[u];
        else ob[u * P * P + y * P + x] = val[u];
      }
      fence_proxy_async();
    };

    if (interior) {
      if (g < G) mbar_wait(&bars[stg], par);
      if (g >= 1 && g < G) {   // steady state: one basic block the scheduler can interleave
        closure_int();
        update_int();
      } else if (g < G) {
        closure_int();
      } else {
        update_int();
      }
      if (g >= 1) {
        // per-patch max wave speed: 64-bit max as (high word, then low word) warp reductions
        const unsigned hi = (unsigned)(cmax >> 32), lo = (unsigned)cmax;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        if (lane == 0) wmax[(gp & 1) * 8 + warp] = ((unsigned long long)mhi << 32) | mlo;
      }
    } else if (g < G) {
      mbar_wait(&bars[stg], par);
      {   // y-face halo rows (haloed y = 0, 17)
        const int hy = lane < 16 ? 0 : E - 1;
        double q[S];
        load_q<L>(st, hy, x + 1, q);
        Side<2> sh;
        bool ok;
        closure_one_ranged<2>(q, cl, 1, sh, ok);
        slow = slow | !ok;
        put_ys(ys_w, hy, x, sh);
      }
      {   // x-face halo columns (haloed x = 0, 17)
        const int hx = lane < 16 ? 0 : E - 1;
        double q[S];
        load_q<L>(st, x + 1, hx, q);
        Side<2> sh;
        bool ok;
        closure_one_ranged<2>(q, cl, 0, sh, ok);
        slow = slow | !ok;
        put_xs(xs_w, x, hx, sh);
      }
      if (producer) put_inv(g);   // read by B(g+1), behind this iteration's barrier
    }
    if (__any_sync(0xffffffffu, slow) && lane == 0) atomicOr(&slowflag[slot3], 1u);
    cmax = cnew;
    if (producer) bulk_wait_read0();   // output buffer of patch g-1's parity is rewritten by B(g+1)
    __syncthreads();
    if (producer) {
      if (g + NST - 1 < G) issue(g + NST - 1);   // into the stage of patch g-1, retired just now
      if (g >= 1) {
        store_out(g - 1);
        finish_patch(g - 1);
      }
    }
    stg = stg == NST - 1 ? 0 : stg + 1;
    par ^= (stg == 0);
    slot3 = slot3 == 2 ? 0 : slot3 + 1;
  }

  if (tail.gmax) {   // fvb_update_cfl: fold the CTA's max_eig into the step's max (fvb_tail.cuh)
    __syncthreads();   // the producer wrote them
    unsigned long long m = 0;
    for (int g = tid; g < G; g += 288) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(max_eig[patch_of(g)]);
      m = v > m ? v : m;
    }
    fused_warp_tail(tail, status, n, m, gridDim.x * 9);
  }
  if (producer) bulk_wait_all0();
}

template <int L>
cudaError_t launch(const FvbArgs& a, cudaStream_t st) {
  auto kfn = fused2d_kernel<L, 2>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 288, BYTES);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.n) grid = a.n;
  const Closure cl{a.gamma, a.gamma - 1.0};
  const CflTail tail{a.gmax, a.cfl, a.dx, a.dt_scalar, a.dt_patches, a.tail_dt};
  kfn<<<(unsigned)grid, 288, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl, tail);
  return cudaGetLastError();
}

}  // namespace f2
}  // namespace fvb

// Shapes with a fused kernel: 3D p=16 (AoS/SoA), 3D p=4 (AoS), 2D p=16 (AoS/SoA)
// and 2D p=2..32 (AoS, the warp kernel); everything else runs the generic kernel.
bool fvb_fused16_supported(int dim, int p, int layout) {
  if (dim == 2 && layout == fvb::kAoS && fvb_fused2d_warp_supported(p)) return true;
  return (p == 16 && (dim == 2 || dim == 3) && (layout == fvb::kAoS || layout == fvb::kSoA)) ||
         fvb_small3d_supported(dim, p, layout);
}

cudaError_t fvb_launch_fused16(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb;
  if (a.n <= 0) return cudaSuccess;
  if (a.dim == 3 && a.p != 16) return fvb_launch_small3d(a, st);   // includes its redo pass
  cudaError_t e;
  if (a.dim == 3) {
    e = fvb_launch_fused3d16_half(a, st);
  } else if (a.layout == kAoS) {
    e = fvb_launch_fused2d16_warp(a, st);   // AoS: warp-autonomous kernel (any p = 2..32)
  } else {
    e = f2::launch<kSoA>(a, st);            // SoA (packed layout): the block kernel above
  }
  if (e != cudaSuccess) return e;
  return fvb_launch_redo(a, st);   // exact re-evaluation of queued patches (usually none)
}
