// fvb_fused3d_pair.cu -- fused 3D Rusanov patch update for p = 16: half-patch CTAs,
// TWO cells per thread.
//
// Same z march, ring, ghost row and bit-exact arithmetic as fvb_fused3d_half.cu,
// but every interior thread owns a y pair of columns (local rows 2k and 2k+1)
// of its half patch: 64 interior threads (2 warps) + the halo/producer warp.
// The face between the two cells of a pair never goes through shared memory:
// each cell's own data, loaded once, is also its partner's y neighbour.  That
// removes 10 of the 55 LDS.64 per cell of the update (the shared-memory data
// pipe is the binding resource of the one-cell kernel), halves the per-plane
// control overhead per cell, and gives each thread two independent cells to
// interleave.  Registers: two sets of z-march carries (~60).
#include <cuda_runtime.h>

#include <type_traits>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace f3p {

using namespace f16;

constexpr int P = 16, E = 18, S = 5;
#ifndef FVB3D_PAIR_ROWS
#define FVB3D_PAIR_ROWS 8
#endif
constexpr int R = FVB3D_PAIR_ROWS;        // interior rows per CTA work item (8: half patches, 16: whole patches)
constexpr int IPP = P / R;                // work items per patch
constexpr int SR = R + 2;                 // stage rows (halo/ghost above and below)
constexpr int PLANE = E * E;
constexpr int SVOL = SR * E;
constexpr int STAGE = SVOL * S;           // 7,200 B
constexpr int NST = 3;
constexpr int NPL = E;
constexpr int64_t VOL = (int64_t)E * E * E;
constexpr int64_t IVOL = (int64_t)P * P * P;
constexpr int YS = S * SR * P;            // ys: [c][stage row 0..9][x 0..15]
constexpr int XS = S * R * E;             // xs: [c][local row 0..7][hx 0..17]
constexpr int OUTN = R * P * S;
#ifndef FVB3D_PAIR_CELLS
#define FVB3D_PAIR_CELLS 2
#endif
constexpr int KC = FVB3D_PAIR_CELLS;      // cells per thread along y (2 or 4)
constexpr int NIW = R / (2 * KC);         // interior warps (a warp covers 2 row groups of KC rows)
constexpr int NTHREADS = 32 * (NIW + 1);
constexpr int OFF_RING = 0;
constexpr int OFF_YS = OFF_RING + NST * STAGE;
constexpr int OFF_XS = OFF_YS + 2 * YS;
constexpr int OFF_OUT = OFF_XS + 2 * XS;
constexpr int OFF_WMAX = OFF_OUT + 2 * OUTN;
constexpr int OFF_FLAG = OFF_WMAX + 2 * NIW;
constexpr int OFF_BAR = OFF_FLAG + 1;
constexpr int TOTAL = OFF_BAR + NST;
constexpr size_t BYTES = (size_t)TOTAL * 8;

template <int L>
__device__ __forceinline__ double qs(const double* st, int r, int hx, int u) {
  return L == kAoS ? st[(r * E + hx) * S + u] : st[(u * SR + r) * E + hx];
}
template <int L>
__device__ __forceinline__ void load_q(const double* st, int r, int hx, double (&q)[S]) {
#pragma unroll
  for (int u = 0; u < S; ++u) q[u] = qs<L>(st, r, hx, u);
}
__device__ __forceinline__ int ys_at(int c, int r, int x) { return (c * SR + r) * P + x; }
__device__ __forceinline__ int xs_at(int c, int ly, int hx) { return (c * R + ly) * E + hx; }

__device__ __forceinline__ void put_ys(double* b, int r, int x, const Side<3>& s) {
  b[ys_at(0, r, x)] = s.lam;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[ys_at(k + 1, r, x)] = s.f[k];
}
__device__ __forceinline__ void put_xs(double* b, int ly, int hx, const Side<3>& s) {
  b[xs_at(0, ly, hx)] = s.lam;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[xs_at(k + 1, ly, hx)] = s.f[k];
}

__device__ __forceinline__ bool inv_ok(double inv) {
  const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
  return inv == 0.0 || (e >= 2u && e < 0x7ffu);
}

// A y neighbour as the update needs it: state, y wave speed, y fluxes.
struct YNb {
  double q[S];
  double lam;
  double f[4];
};

// z-march carries of one column
struct ZCarry {
  Side<3> prev;        // z-side data of plane zh-1
  double tp[S];        // dissipation term of the face (zh-2 | zh-1) seen from below
  double favg[S];      // unscaled flux sum of that face
};

enum PlaneKind { kZLo = 0, kFirst = 1, kSteady = 2, kZHi = 3 };
template <int K>
using Kind = std::integral_constant<int, K>;

template <int L>
__global__ void __launch_bounds__(NTHREADS, (R == 8 && KC == 2) ? 4 : (R == 8 ? 4 : 2))
fused3d_pair_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
                    const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
                    int64_t n, Closure cl) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + OFF_RING;
  double* ysb = sm + OFF_YS;
  double* xsb = sm + OFF_XS;
  double* outb = sm + OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + OFF_WMAX);
  unsigned* slowflag = reinterpret_cast<unsigned*>(sm + OFF_FLAG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);

  const int tid = threadIdx.x;
  const bool interior = tid < 32 * NIW;
  const int warp = tid >> 5, lane = tid & 31;
  const int x = lane & 15;
  const int lya = ((warp << 1) | (lane >> 4)) * KC;   // local rows lya .. lya + KC - 1 (interior warps)
  const bool producer = tid == 32 * NIW;

  const int64_t items = IPP * n;
  const int my_items = (items > (int64_t)blockIdx.x) ? (int)((items - 1 - (int64_t)blockIdx.x) / gridDim.x + 1) : 0;
  auto item_index = [&](int j) -> int64_t { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };

  auto issue = [&](int j, int zh, unsigned s) {
    const int64_t it = item_index(j);
    const int64_t pidx = it / IPP;
    const int y0 = (int)(it % IPP) * R;
    double* st = ring + s * STAGE;
    uint64_t* bar = bars + s;
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)(STAGE * 8));
    if (L == kAoS) {
      tma_load_1d(st, qin + (pidx * VOL + (int64_t)zh * PLANE + (int64_t)y0 * E) * S, (uint32_t)(STAGE * 8), bar);
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_load_1d(st + u * SVOL, qin + ((int64_t)u * n + pidx) * VOL + (int64_t)zh * PLANE + (int64_t)y0 * E,
                    (uint32_t)(SVOL * 8), bar);
    }
  };
  auto store_out = [&](int64_t pidx, int y0, int z) {
    const double* src = outb + (z & 1) * OUTN;
    if (L == kAoS) {
      tma_store_1d(qout + (pidx * IVOL + (int64_t)z * P * P + (int64_t)y0 * P) * S, src, (uint32_t)(OUTN * 8));
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_store_1d(qout + ((int64_t)u * n + pidx) * IVOL + (int64_t)z * P * P + (int64_t)y0 * P, src + u * R * P,
                     (uint32_t)(R * P * 8));
    }
    bulk_commit();
  };
  auto finish_item = [&](int j, int64_t pidx) {
    unsigned long long m = wmax[(j & 1) * NIW];
#pragma unroll
    for (int w = 1; w < NIW; ++w) {
      const unsigned long long v = wmax[(j & 1) * NIW + w];
      m = v > m ? v : m;
    }
    atomicMax(reinterpret_cast<unsigned long long*>(max_eig) + pidx, m);
    if (slowflag[j & 1]) {
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
  if (producer && my_items > 0) {
    issue(0, 0, 0);
    issue(0, 1, 1);
  }

  bool slow = false;
  unsigned long long cm = 0;
  ZCarry zk[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
#pragma unroll
    for (int u = 0; u < S; ++u) { zk[c].tp[u] = 0.0; zk[c].favg[u] = 0.0; }
    zk[c].prev.lam = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) zk[c].prev.f[k] = 0.0;
  }

  unsigned stg = 0, par = 0;

  for (int jp = 0; jp < my_items; ++jp) {
    const int64_t it = item_index(jp);
    const int64_t pidx = it / IPP;
    const int y0 = (int)(it % IPP) * R;
    const double dx = __ddiv_rn(cell_size[pidx * 3], (double)P);   // vectorized.py:169
    const double inv = __ddiv_rn(dtv[pidx], dx);                    // vectorized.py:170
    const double half_inv = dmul(0.5, inv);
    if (tid == 0 && !inv_ok(inv)) slow = true;

    auto plane = [&](int zh, auto kind) {
      constexpr int K = decltype(kind)::value;
      const double* st = ring + stg * STAGE;
      const double* stc = ring + (stg == 0 ? NST - 1 : stg - 1) * STAGE;
      double* ys_w = ysb + (zh & 1) * YS;
      double* xs_w = xsb + (zh & 1) * XS;
      const double* ys_r = ysb + ((zh - 1) & 1) * YS;
      const double* xs_r = xsb + ((zh - 1) & 1) * XS;
      mbar_wait(&bars[stg], par);

      if (interior) {
        auto closure = [&](const double (&q)[S], int ly, Side<3>& zc) {
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
            put_xs(xs_w, ly, x + 1, sd[0]);
            put_ys(ys_w, ly + 1, x, sd[1]);
            zc = sd[2];
          } else {
            bool ok;
            closure_one_ranged<3>(q, cl, 2, zc, ok);
            slow = slow | !ok;
          }
        };
        auto first_face = [&](const double (&q)[S], int ly, const Side<3>& zc, ZCarry& zz) {
          double qc[S];
          load_q<L>(stc, ly + 1, x + 1, qc);
          const double cz = dmul(half_inv, speed_max(zc.lam, zz.prev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) {
            zz.tp[u] = dmul(cz, dsub(q[u], qc[u]));
            const double c = u == 0 ? qc[3] : zz.prev.f[u - 1];
            zz.favg[u] = dadd(c, u == 0 ? q[3] : zc.f[u - 1]);
          }
        };
        // y neighbour record (state, y wave speed, y fluxes) of stage row r, plane zh-1
        auto load_ynb = [&](int r, YNb& o) {
          load_q<L>(stc, r, x + 1, o.q);
          o.lam = ys_r[ys_at(0, r, x)];
#pragma unroll
          for (int k = 0; k < 4; ++k) o.f[k] = ys_r[ys_at(k + 1, r, x)];
        };
        // update of the cell at local row ly of plane zh-1 (vectorized.py:161-200)
        auto update = [&](const YNb& own, const YNb& ym, const YNb& yp, int ly, const double (&q)[S],
                          const Side<3>& zc, ZCarry& zz) {
          double val[S], qn[S];
          const double lx = xs_r[xs_at(0, ly, x + 1)];
          const double cz = dmul(half_inv, speed_max(zc.lam, zz.prev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = own.q[u];                      // _pass_copy
          // dissipation x-, x+, y-, y+ (vectorized.py:173-180)
          load_q<L>(stc, ly + 1, x, qn);
          const double jl = qn[1];
          dissipate<3>(val, half_inv, lx, own.q, xs_r[xs_at(0, ly, x)], qn);
          load_q<L>(stc, ly + 1, x + 2, qn);
          const double jr = qn[1];
          dissipate<3>(val, half_inv, lx, own.q, xs_r[xs_at(0, ly, x + 2)], qn);
          dissipate<3>(val, half_inv, own.lam, own.q, ym.lam, ym.q);
          dissipate<3>(val, half_inv, own.lam, own.q, yp.lam, yp.q);
          // z-: the previous face's term, negated; z+: this face's term
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = dsub(val[u], zz.tp[u]);
#pragma unroll
          for (int u = 0; u < S; ++u) {
            zz.tp[u] = dmul(cz, dsub(q[u], own.q[u]));
            val[u] = dadd(val[u], zz.tp[u]);
          }
          // flux differences x, y, z (vectorized.py:193-200), see fvb_fused3d.cu add_flux
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const double fm = u == 0 ? jl : xs_r[xs_at(u, ly, x)];
            const double fc = u == 0 ? own.q[1] : xs_r[xs_at(u, ly, x + 1)];
            const double fp = u == 0 ? jr : xs_r[xs_at(u, ly, x + 2)];
            val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
          }
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const double fm = u == 0 ? ym.q[2] : ym.f[u - 1];
            const double fc = u == 0 ? own.q[2] : own.f[u - 1];
            const double fp = u == 0 ? yp.q[2] : yp.f[u - 1];
            val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
          }
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const double c = u == 0 ? own.q[3] : zz.prev.f[u - 1];
            const double sum_p = dadd(c, u == 0 ? q[3] : zc.f[u - 1]);
            val[u] = dadd(val[u], dmul(half_inv, dsub(zz.favg[u], sum_p)));
            zz.favg[u] = sum_p;
          }
          double* ob_ = outb + (zh & 1) * OUTN;
#pragma unroll
          for (int u = 0; u < S; ++u) {
            if (L == kAoS) ob_[(ly * P + x) * S + u] = val[u];
            else ob_[(u * R + ly) * P + x] = val[u];
          }
        };
        // Cell by cell along y: closure of the cell's volume of plane zh, then its
        // update of plane zh-1 through a sliding window of three y-neighbour
        // records (the cells of a group are each other's y neighbours).
        YNb wm, wc, wp;
        if (K == kSteady || K == kZHi) {
          load_ynb(lya, wm);       // y- neighbour of the first cell (shared memory)
          load_ynb(lya + 1, wc);   // the first cell itself
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const int ly = lya + c;
          double q[S];
          Side<3> zc;
          load_q<L>(st, ly + 1, x + 1, q);
          closure(q, ly, zc);
          if (K == kFirst) first_face(q, ly, zc, zk[c]);
          if (K == kSteady || K == kZHi) {
            load_ynb(ly + 2, wp);   // next cell of the group, or the y+ neighbour after the last
            update(wc, wm, wp, ly, q, zc, zk[c]);
            wm = wc;
            wc = wp;
          }
          zk[c].prev = zc;
        }
        if (K == kSteady || K == kZHi) fence_proxy_async();
      } else if (K == kFirst || K == kSteady) {
        // the halo warp: stage rows 0 and 9 (y-face halo row and ghost row: y-side data);
        // the x-face halo columns of the 8 interior rows (x-side data)
        {
          const int r = lane < 16 ? 0 : SR - 1;
          double qh[S];
          load_q<L>(st, r, x + 1, qh);
          Side<3> sh;
          bool ok;
          closure_one_ranged<3>(qh, cl, 1, sh, ok);
          slow = slow | !ok;
          put_ys(ys_w, r, x, sh);
        }
        if (lane < 2 * R) {
          const int lr = lane % R;
          const int hx = lane < R ? 0 : E - 1;
          double qh[S];
          load_q<L>(st, lr + 1, hx, qh);
          Side<3> sh;
          bool ok;
          closure_one_ranged<3>(qh, cl, 0, sh, ok);
          slow = slow | !ok;
          put_xs(xs_w, lr, hx, sh);
        }
      }
      if (K == kZHi) {
        if (__any_sync(0xffffffffu, slow) && lane == 0) atomicOr(&slowflag[jp & 1], 1u);
        slow = false;
        if (interior) {
          unsigned long long m = cm;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
            m = v > m ? v : m;
          }
          if (lane == 0) wmax[(jp & 1) * NIW + warp] = m;
          cm = 0;
        }
      }
      if (producer) bulk_wait_read0();
      __syncthreads();
      if (producer) {
        const int zn = zh + 2 < NPL ? zh + 2 : zh + 2 - NPL;
        const int jn = zh + 2 < NPL ? jp : jp + 1;
        if (jn < my_items) issue(jn, zn, stg == 0 ? NST - 1 : stg - 1);
        if (K == kSteady || K == kZHi) store_out(pidx, y0, zh - 2);
        if (K == kZHi) finish_item(jp, pidx);
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

template <int L>
cudaError_t launch_impl(const FvbArgs& a, cudaStream_t st) {
  auto kfn = fused3d_pair_kernel<L>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BYTES);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.max_eig, 0, sizeof(double) * (size_t)a.n, st);   // atomicMax of the two halves
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NTHREADS, BYTES);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > IPP * a.n) grid = IPP * a.n;
  const Closure cl{a.gamma, a.gamma - 1.0};
  kfn<<<(unsigned)grid, NTHREADS, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl);
  return cudaGetLastError();
}

}  // namespace f3p
}  // namespace fvb

cudaError_t fvb_launch_fused3d16_pair(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb;
  if (a.n <= 0) return cudaSuccess;
  return a.layout == kAoS ? f3p::launch_impl<kAoS>(a, st) : f3p::launch_impl<kSoA>(a, st);
}
