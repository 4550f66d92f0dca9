// fvb_fused3d.cu -- fused 3D Rusanov patch update for p = 16 (the headline shape).
//
// One persistent CTA (8 "interior" warps + 1 "halo" warp, 2 CTAs per SM)
// marches each patch plane by plane in z:
//
//   ring    3 TMA bulk-copy stages of one haloed z-plane (18x18x5 doubles,
//           12,960 B), mbarrier complete_tx; plane g+2 is issued as soon as
//           plane g-1 retires.
//   xs, ys  x- and y-side data (lam, f[1..4]) of every volume of the plane,
//           including the face-halo columns / rows (written by the halo
//           warp), double-buffered by plane parity.
//   ostage  two output planes (16x16x5) stored back with TMA bulk stores.
//
// Iteration g (haloed plane zh), ONE CTA barrier:
//   A  interior lanes evaluate the Euler closure of their volume of plane zh
//      once (14 quotients sharing one reciprocal refinement, fvb_exact.cuh)
//      and publish its x/y-side data; the halo warp publishes the x/y face
//      halo volumes of plane zh.
//   B  interior lanes update their cell of plane zh-1 from the side data
//      published in the previous iteration (x and y faces evaluated from both
//      sides, exactly as the reference's per-volume passes) and the z faces
//      marching in registers: the face (zh-1 | zh) is evaluated once and
//      re-used, negated, as the minus face of the next plane.  -- barrier
//   A(g) and B(g) touch disjoint buffers, so they need no barrier between
//   them; the barrier after B(g) orders A(g) before B(g+1) and B(g) before
//   A(g+2)'s reuse of the same parity.
//
// The re-used z face is the only place the arithmetic is not literally the
// reference's: -RN(c*(a-b)) equals RN(c*(b-a)) except for the sign of an
// exact zero, which could only surface as a -0.0 result whose lower neighbour
// holds -0.0 in that unknown (where the reference has +0.0).  Inside the range
// gate no unknown of an evaluated volume is -0.0, and a sum that starts from
// +0.0 or a nonzero value can only reach zero as +0.0 (a sum is -0.0 only when
// both addends are): a -0.0 result is impossible on the fused path.
// Patches holding -0.0 leave the gate and are re-evaluated by fvb_redo_kernel,
// which evaluates every face from both sides exactly as the reference does.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace f3 {

using namespace f16;

constexpr int P = 16, E = 18, S = 5;
constexpr int PLANE = E * E;              // haloed volumes per plane
constexpr int STAGE = PLANE * S;          // doubles per ring stage
constexpr int NST = 3;                    // ring stages: planes g-1 and g are read in iteration g, g+1 in flight
constexpr int NPL = E;                    // planes per patch
constexpr int64_t VOL = (int64_t)E * E * E;
constexpr int64_t IVOL = (int64_t)P * P * P;
constexpr int SIDE = S * E * P;           // one x- or y-side buffer: 5 comps x 18 x 16
constexpr int OUTN = P * P * S;
constexpr int OFF_RING = 0;
constexpr int OFF_YS = OFF_RING + NST * STAGE;
constexpr int OFF_XS = OFF_YS + 2 * SIDE;
constexpr int OFF_OUT = OFF_XS + 2 * SIDE;
constexpr int OFF_WMAX = OFF_OUT + 2 * OUTN;   // output planes double-buffered
constexpr int OFF_FLAG = OFF_WMAX + 16;
constexpr int OFF_BAR = OFF_FLAG + 1;
constexpr int TOTAL = OFF_BAR + NST;
constexpr int NTHREADS = 288;             // 8 interior warps (one column each) + the halo / producer warp
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
// ys: [c][haloed row hy][interior col x];  xs: [c][interior row y][haloed col hx]
__device__ __forceinline__ int ys_at(int c, int hy, int x) { return (c * E + hy) * P + x; }
__device__ __forceinline__ int xs_at(int c, int y, int hx) { return (c * P + y) * E + hx; }

__device__ __forceinline__ void put_ys(double* b, int hy, int x, const Side<3>& s) {
  b[ys_at(0, hy, x)] = s.lam;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[ys_at(k + 1, hy, x)] = s.f[k];
}
__device__ __forceinline__ void put_xs(double* b, int y, int hx, const Side<3>& s) {
  b[xs_at(0, y, hx)] = s.lam;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[xs_at(k + 1, y, hx)] = s.f[k];
}

// vectorized.py:193-200 for one direction: RN(inv * RN(RN(0.5*a) - RN(0.5*b)))
// with a = RN(f_m+f_c), b = RN(f_c+f_p), evaluated as RN(half_inv * RN(a - b)).
// Scaling by 0.5 is exact and commutes with rounding whenever nothing is
// subnormal: inside the range gate every flux is 0 or has magnitude >= 2^-601,
// so a, b and a-b are 0 or >= 2^-705, and half_inv = 0.5*inv exactly (the
// kernels route patches with 0 < |inv| < 2^-1021 to the exact redo path).
// Hence the two forms are bit-identical there, at 2 DMUL less per term.
template <class FM, class FC, class FP>
__device__ __forceinline__ void add_flux(double (&val)[S], double half_inv, FM fm, FC fc, FP fp) {
#pragma unroll
  for (int u = 0; u < S; ++u) {
    const double c = fc(u);
    val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm(u), c), dadd(c, fp(u)))));
  }
}

// 0 or |inv| >= 2^-1021 (0.5*inv exact), finite: the flux rewrite above applies.
__device__ __forceinline__ bool inv_ok(double inv) {
  const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
  return inv == 0.0 || (e >= 2u && e < 0x7ffu);
}


// Plane kinds of the z march (haloed plane index zh = 0 .. 17).
enum PlaneKind { kZLo = 0, kFirst = 1, kSteady = 2, kZHi = 3 };
template <int K>
using Kind = std::integral_constant<int, K>;

template <int L, int MINB>
__global__ void __launch_bounds__(NTHREADS, MINB)
fused3d_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
               const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
               int64_t n, Closure cl) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + OFF_RING;
  double* ysb = sm + OFF_YS;
  double* xsb = sm + OFF_XS;
  double* outb = sm + OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + OFF_WMAX);
  unsigned* slowflag = reinterpret_cast<unsigned*>(sm + OFF_FLAG);   // 2 words, by patch parity
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);

  const int tid = threadIdx.x;
  const bool interior = tid < 256;
  const int warp = tid >> 5, lane = tid & 31;
  const int x = lane & 15;
  const int y = ((warp & 7) << 1) | (lane >> 4);
  const bool producer = tid == 256;   // TMA issue / output store / patch max

  const int my_patches = (n > (int64_t)blockIdx.x) ? (int)((n - 1 - (int64_t)blockIdx.x) / gridDim.x + 1) : 0;
  auto patch_index = [&](int j) -> int64_t { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };

  // plane zh of this CTA's j-th patch into ring stage s
  auto issue = [&](int j, int zh, unsigned s) {
    const int64_t pidx = patch_index(j);
    double* st = ring + s * STAGE;
    uint64_t* bar = bars + s;
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)(STAGE * 8));
    if (L == kAoS) {
      tma_load_1d(st, qin + (pidx * VOL + (int64_t)zh * PLANE) * S, (uint32_t)(STAGE * 8), bar);
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_load_1d(st + u * PLANE, qin + ((int64_t)u * n + pidx) * VOL + (int64_t)zh * PLANE,
                    (uint32_t)(PLANE * 8), bar);
    }
  };
  auto store_out = [&](int64_t pidx, int z) {   // interior plane z from output buffer z & 1
    const double* src = outb + (z & 1) * OUTN;
    if (L == kAoS) {
      tma_store_1d(qout + (pidx * IVOL + (int64_t)z * P * P) * S, src, (uint32_t)(OUTN * 8));
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_store_1d(qout + ((int64_t)u * n + pidx) * IVOL + (int64_t)z * P * P, src + u * P * P,
                     (uint32_t)(P * P * 8));
    }
    bulk_commit();
  };
  auto finish_patch_max = [&](int j, int64_t pidx) {
    unsigned long long m = wmax[(j & 1) * 8];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const unsigned long long v = wmax[(j & 1) * 8 + w];
      m = v > m ? v : m;
    }
    max_eig[pidx] = __longlong_as_double((long long)m);
    if (slowflag[j & 1]) {   // queue the patch for the exact re-evaluation (fvb_redo_kernel)
      const unsigned k = atomicAdd(&status[1], 1u);
      status[2 + k] = (unsigned)pidx;
      slowflag[j & 1] = 0;
    }
  };

  if (producer) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    slowflag[0] = slowflag[1] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (producer && my_patches > 0) {
    issue(0, 0, 0);
    issue(0, 1, 1);
  }

  bool slow = false;           // some quotient of this thread's volumes left the range gate (this patch)
  unsigned long long cm = 0;   // running max wave speed (bit pattern) of this column
  // z-march carries: z-side data of the previous plane, and the previous z face
  // (its dissipation term seen from the lower cell, tp, and the unscaled flux
  // sum f_{z-1} + f_z, favg_zm)
  Side<3> zprev;
  double tp[S], favg_zm[S];
  zprev.lam = 0.0;
#pragma unroll
  for (int u = 0; u < S; ++u) { tp[u] = 0.0; favg_zm[u] = 0.0; }
#pragma unroll
  for (int k = 0; k < 4; ++k) zprev.f[k] = 0.0;

  unsigned stg = 0, par = 0;   // ring stage of the current plane and its mbarrier phase parity

  for (int jp = 0; jp < my_patches; ++jp) {
    const int64_t pidx = patch_index(jp);
    const double dx = __ddiv_rn(cell_size[pidx * 3], (double)P);   // vectorized.py:169
    const double inv = __ddiv_rn(dtv[pidx], dx);                    // vectorized.py:170
    const double half_inv = dmul(0.5, inv);                         // `0.5 * inv * a`
    if (tid == 0 && !inv_ok(inv)) slow = true;

    // One plane of the march.  18 planes per patch and NST = 3 keep the ring
    // stage / parity and the side-buffer parity (zh & 1) patch-periodic.
    auto plane = [&](int zh, auto kind) {
      constexpr int K = decltype(kind)::value;
      const double* st = ring + stg * STAGE;                                // plane zh
      const double* stc = ring + (stg == 0 ? NST - 1 : stg - 1) * STAGE;   // plane zh-1
      double* ys_w = ysb + (zh & 1) * SIDE;
      double* xs_w = xsb + (zh & 1) * SIDE;
      const double* ys_r = ysb + ((zh - 1) & 1) * SIDE;
      const double* xs_r = xsb + ((zh - 1) & 1) * SIDE;
      mbar_wait(&bars[stg], par);

      if (interior) {
        Side<3> zcur;
        double q[S];
        load_q<L>(st, y + 1, x + 1, q);
        // ---- A: closure of this column's volume of plane zh ----
        if (K == kFirst || K == kSteady) {
          Side<3> sd[3];
          bool ok;
          closure_all_ranged<3>(q, cl, sd, ok);
          slow = slow | !ok;
          unsigned long long m = (unsigned long long)__double_as_longlong(sd[0].lam);
          unsigned long long v = (unsigned long long)__double_as_longlong(sd[1].lam);
          m = v > m ? v : m;
          v = (unsigned long long)__double_as_longlong(sd[2].lam);
          m = v > m ? v : m;
          cm = m > cm ? m : cm;
          put_xs(xs_w, y, x + 1, sd[0]);
          put_ys(ys_w, y + 1, x, sd[1]);
          zcur = sd[2];
        } else {   // z-halo planes: only their z-side data
          bool ok;
          closure_one_ranged<3>(q, cl, 2, zcur, ok);
          slow = slow | !ok;
        }
        if (K == kFirst) {
          // only the face (0 | 1) -- the minus face of the first interior plane
          double qc[S];
          load_q<L>(stc, y + 1, x + 1, qc);
          const double cz = dmul(half_inv, speed_max(zcur.lam, zprev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) {
            tp[u] = dmul(cz, dsub(q[u], qc[u]));
            const double c = u == 0 ? qc[3] : zprev.f[u - 1];
            favg_zm[u] = dadd(c, u == 0 ? q[3] : zcur.f[u - 1]);
          }
        }
        // ---- B: update of this column's cell of plane zh-1 ----
        // Plane zh-1's side data were published in the previous iteration
        // (behind the barrier that ended it); this column's plane-zh z data are
        // zcur.  No barrier between A and B: the steady state is one basic
        // block the scheduler interleaves.
        if (K == kSteady || K == kZHi) {
          double qc[S], val[S], qn[S];
          load_q<L>(stc, y + 1, x + 1, qc);
          const double lx = xs_r[xs_at(0, y, x + 1)];
          const double ly = ys_r[ys_at(0, y + 1, x)];
          // z face (zh-1 | zh) seen from the lower cell: coeff*(Q_zh - Q_zh-1)
          const double cz = dmul(half_inv, speed_max(zcur.lam, zprev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = qc[u];                       // _pass_copy
          // dissipation x-, x+, y-, y+ (vectorized.py:173-180)
          load_q<L>(stc, y + 1, x, qn);
          dissipate<3>(val, half_inv, lx, qc, xs_r[xs_at(0, y, x)], qn);
          load_q<L>(stc, y + 1, x + 2, qn);
          dissipate<3>(val, half_inv, lx, qc, xs_r[xs_at(0, y, x + 2)], qn);
          load_q<L>(stc, y, x + 1, qn);
          dissipate<3>(val, half_inv, ly, qc, ys_r[ys_at(0, y, x)], qn);
          load_q<L>(stc, y + 2, x + 1, qn);
          dissipate<3>(val, half_inv, ly, qc, ys_r[ys_at(0, y + 2, x)], qn);
          // z-: the previous face's term, negated; z+: this face's term
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = dsub(val[u], tp[u]);
#pragma unroll
          for (int u = 0; u < S; ++u) {
            tp[u] = dmul(cz, dsub(q[u], qc[u]));
            val[u] = dadd(val[u], tp[u]);
          }
          // flux differences x, y, z (vectorized.py:193-200)
          {
            double fo[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) fo[k] = xs_r[xs_at(k + 1, y, x + 1)];
            add_flux(val, half_inv,
                     [&](int u) { return u == 0 ? qs<L>(stc, y + 1, x, 1) : xs_r[xs_at(u, y, x)]; },
                     [&](int u) { return u == 0 ? qc[1] : fo[u - 1]; },
                     [&](int u) { return u == 0 ? qs<L>(stc, y + 1, x + 2, 1) : xs_r[xs_at(u, y, x + 2)]; });
          }
          {
            double fo[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) fo[k] = ys_r[ys_at(k + 1, y + 1, x)];
            add_flux(val, half_inv,
                     [&](int u) { return u == 0 ? qs<L>(stc, y, x + 1, 2) : ys_r[ys_at(u, y, x)]; },
                     [&](int u) { return u == 0 ? qc[2] : fo[u - 1]; },
                     [&](int u) { return u == 0 ? qs<L>(stc, y + 2, x + 1, 2) : ys_r[ys_at(u, y + 2, x)]; });
          }
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const double c = u == 0 ? qc[3] : zprev.f[u - 1];
            const double sum_p = dadd(c, u == 0 ? q[3] : zcur.f[u - 1]);
            val[u] = dadd(val[u], dmul(half_inv, dsub(favg_zm[u], sum_p)));
            favg_zm[u] = sum_p;
          }
          double* ob = outb + (zh & 1) * OUTN;   // output buffer of interior plane zh-2 (parity (zh-2)&1)
#pragma unroll
          for (int u = 0; u < S; ++u) {
            if (L == kAoS) ob[(y * P + x) * S + u] = val[u];
            else ob[u * P * P + y * P + x] = val[u];
          }
          fence_proxy_async();
        }
        zprev = zcur;
      } else if (K == kFirst || K == kSteady) {
        // the halo warp: face-halo volumes of plane zh, only their face-normal side data
        {   // y-face halo rows (haloed y = 0, 17), interior columns
          const int hy = lane < 16 ? 0 : E - 1;
          double qh[S];
          load_q<L>(st, hy, x + 1, qh);
          Side<3> sh;
          bool ok;
          closure_one_ranged<3>(qh, cl, 1, sh, ok);
          slow = slow | !ok;
          put_ys(ys_w, hy, x, sh);
        }
        {   // x-face halo columns (haloed x = 0, 17), interior rows
          const int hx = lane < 16 ? 0 : E - 1;
          double qh[S];
          load_q<L>(st, x + 1, hx, qh);
          Side<3> sh;
          bool ok;
          closure_one_ranged<3>(qh, cl, 0, sh, ok);
          slow = slow | !ok;
          put_xs(xs_w, x, hx, sh);
        }
      }
      if (K == kZHi) {   // patch complete
        if (__any_sync(0xffffffffu, slow) && lane == 0) atomicOr(&slowflag[jp & 1], 1u);
        slow = false;
        if (interior) {   // per-warp max of the wave speeds
          unsigned long long m = cm;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
            m = v > m ? v : m;
          }
          if (lane == 0) wmax[(jp & 1) * 8 + warp] = m;
          cm = 0;
        }
      }
      // One barrier per plane: publishes this plane's side data and output, and
      // retires plane zh-1's ring stage and side buffers for reuse.
      if (producer) bulk_wait_read0();   // output buffer (zh+1)&1, written next iteration, is free
      __syncthreads();
      if (producer) {
        // plane zh+2 (of this or the next patch) into the stage of plane zh-1, retired just now
        const int zn = zh + 2 < NPL ? zh + 2 : zh + 2 - NPL;
        const int jn = zh + 2 < NPL ? jp : jp + 1;
        if (jn < my_patches) issue(jn, zn, stg == 0 ? NST - 1 : stg - 1);
        if (K == kSteady || K == kZHi) store_out(pidx, zh - 2);
        if (K == kZHi) finish_patch_max(jp, pidx);
      }
      stg = stg == NST - 1 ? 0 : stg + 1;
      par ^= (stg == 0);
    };

    plane(0, Kind<kZLo>{});
    plane(1, Kind<kFirst>{});
#pragma unroll 1
    for (int zh = 2; zh <= P; ++zh) plane(zh, Kind<kSteady>{});
    plane(NPL - 1, Kind<kZHi>{});
  }

  if (producer) bulk_wait_all0();
}

static int min_blocks_choice() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FVB_FUSED_MINB");
    v = (e && e[0] == '1') ? 1 : 2;
  }
  return v;
}

template <int L, int MINB>
cudaError_t launch_impl(const FvbArgs& a, cudaStream_t st) {
  auto kfn = fused3d_kernel<L, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NTHREADS, BYTES);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.n) grid = a.n;
  const Closure cl{a.gamma, a.gamma - 1.0};
  kfn<<<(unsigned)grid, NTHREADS, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl);
  return cudaGetLastError();
}

}  // namespace f3
}  // namespace fvb

cudaError_t fvb_launch_fused3d16(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb;
  if (a.n <= 0) return cudaSuccess;
  const bool one = f3::min_blocks_choice() == 1;
  if (a.layout == kAoS) return one ? f3::launch_impl<kAoS, 1>(a, st) : f3::launch_impl<kAoS, 2>(a, st);
  return one ? f3::launch_impl<kSoA, 1>(a, st) : f3::launch_impl<kSoA, 2>(a, st);
}
