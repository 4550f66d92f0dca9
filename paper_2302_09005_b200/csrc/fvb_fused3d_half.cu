// fvb_fused3d_half.cu -- fused 3D Rusanov patch update for p = 16, half-patch CTAs.
//
// Same z march and bit-exact arithmetic as fvb_fused3d.cu, but each CTA owns
// HALF a patch: interior rows y0 .. y0+7 (y0 = 0 or 8) of every plane.  The CTA
// is 4 interior warps (one column each) + 1 halo/producer warp, 160 threads,
// about 56 KB of shared memory, so FOUR independent CTAs share an SM instead of
// two full-patch CTAs: the per-plane CTA barrier then spans 5 warps, and four
// barrier domains drift against each other, which keeps the FP64 pipe fed
// while one CTA waits (the full-patch kernel spends ~13 % of its warp cycles at
// the barrier with every warp of a CTA in the same phase).
//
// The price is one "ghost" row per plane: the row just outside the half (y0-1
// or y0+8, an interior row of the other half) whose y-side data the boundary
// cells need.  The halo warp evaluates it, together with the y-face halo row
// and the x-face halo columns, so 48 face-normal closures per 128 cells
// (vs 64 per 256 for the full patch).
//
// Ring stage = haloed rows y0 .. y0+9 of one plane: 10 x 18 x 5 doubles,
// contiguous in the AoS input (7,200 B, one TMA bulk copy).  Stage row r is
// haloed row y0 + r; interior local row ly (0..7) is stage row ly + 1.
//
// Per-patch outputs: each half writes its 8 x 16 cells of every interior plane
// with a TMA bulk store.  A CTA processes both halves of its patches back to
// back, so it writes the patch's max_eigenvalue (the max of the two halves'
// maxima on the bit patterns) and, when a volume of either half left the range
// gate, queues the patch once for the exact redo pass.
#include <cuda_runtime.h>

#include <type_traits>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tail.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace f3h {

using namespace f16;

constexpr int P = 16, E = 18, S = 5;
#ifndef FVB3D_HALF_ROWS
#define FVB3D_HALF_ROWS 8
#endif
constexpr int R = FVB3D_HALF_ROWS;        // interior rows per CTA work item (8: half patches, 4: quarters)
constexpr int IPP = P / R;                // work items per patch
constexpr int NIW = R / 2;                // interior warps (a warp covers two rows)
constexpr int SR = R + 2;                 // stage rows (halo/ghost above and below)
constexpr int PLANE = E * E;              // haloed volumes per plane (global layout)
constexpr int SVOL = SR * E;              // volumes per stage
constexpr int STAGE = SVOL * S;           // doubles per ring stage (7,200 B)
constexpr int NST = 3;
constexpr int NPL = E;
constexpr int64_t VOL = (int64_t)E * E * E;
constexpr int64_t IVOL = (int64_t)P * P * P;
constexpr int YS = S * SR * P;            // ys: [c][stage row 0..9][x 0..15]
constexpr int XS = S * R * E;             // xs: [c][local row 0..7][hx 0..17]
constexpr int OUTN = R * P * S;           // one output half-plane
constexpr int NTHREADS = 32 * (NIW + 1);   // interior warps + the halo / producer warp
constexpr int OFF_RING = 0;
constexpr int OFF_YS = OFF_RING + NST * STAGE;
constexpr int OFF_XS = OFF_YS + 2 * YS;
constexpr int OFF_OUT = OFF_XS + 2 * XS;
constexpr int OFF_WMAX = OFF_OUT + 2 * OUTN;
constexpr int OFF_FLAG = OFF_WMAX + 8;
constexpr int OFF_BAR = OFF_FLAG + 1;
constexpr int TOTAL = OFF_BAR + NST;
constexpr size_t BYTES = (size_t)TOTAL * 8;
// (Measured and removed: per-warp mbarriers instead of the
// CTA barrier, 554 vs 465 us; the own volume's data carried through TMEM,
// 1,062 us.)

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

// RN(half_inv * RN(RN(fm+fc) - RN(fc+fp))): see fvb_fused3d.cu add_flux.
template <class FM, class FC, class FP>
__device__ __forceinline__ void add_flux(double (&val)[S], double half_inv, FM fm, FC fc, FP fp) {
#pragma unroll
  for (int u = 0; u < S; ++u) {
    const double c = fc(u);
    val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm(u), c), dadd(c, fp(u)))));
  }
}

__device__ __forceinline__ bool inv_ok(double inv) {
  const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
  return inv == 0.0 || (e >= 2u && e < 0x7ffu);
}


#ifndef FVB3D_STEADY_UNROLL
#define FVB3D_STEADY_UNROLL 1
#endif
constexpr int STEADY_UNROLL = FVB3D_STEADY_UNROLL;   // unroll of the steady plane loop
enum PlaneKind { kZLo = 0, kFirst = 1, kSteady = 2, kZHi = 3 };
template <int K>
using Kind = std::integral_constant<int, K>;

template <int L>
#ifndef FVB3D_HALF_MINB
#define FVB3D_HALF_MINB (R == 8 ? 4 : 7)
#endif
__global__ void __launch_bounds__(NTHREADS, FVB3D_HALF_MINB)
fused3d_half_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
                    const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
                    int64_t n, Closure cl, CflTail tail) {
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + OFF_RING;
  double* ysb = sm + OFF_YS;
  double* xsb = sm + OFF_XS;
  double* outb = sm + OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + OFF_WMAX);
  unsigned* slowflag = reinterpret_cast<unsigned*>(sm + OFF_FLAG);   // 2 words, by item parity
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);

  const int tid = threadIdx.x;
  const bool interior = tid < 32 * NIW;
  const int warp = tid >> 5, lane = tid & 31;
  const int x = lane & 15;
  const int ly = (warp << 1) | (lane >> 4);   // local interior row 0..R-1 (interior warps)
  const bool producer = tid == 32 * NIW;

  // Work items: the CTA's patches blockIdx.x + i * gridDim.x, each as its IPP row blocks
  // back to back (item j = patch j / IPP, rows (j % IPP) * R ..), so one CTA sees every
  // row block of its patches and writes max_eigenvalue / the redo entry itself -- no
  // zero-initialised max_eig (atomicMax) and no duplicate redo entries.
  const int my_patches = (n > (int64_t)blockIdx.x) ? (int)((n - 1 - (int64_t)blockIdx.x) / gridDim.x + 1) : 0;
  const int my_items = IPP * my_patches;
  auto item_patch = [&](int j) -> int64_t { return (int64_t)blockIdx.x + (int64_t)(j / IPP) * gridDim.x; };

  auto issue = [&](int j, int zh, unsigned s) {
    const int64_t pidx = item_patch(j);
    const int y0 = (j % IPP) * R;
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
  auto store_out = [&](int64_t pidx, int y0, int z) {   // interior plane z (rows y0..y0+7) from buffer z & 1
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
  __shared__ unsigned long long tail_m;   // max of the max_eig the producer wrote (fused_kernel_tail)
  auto finish_patch = [&](int j, int64_t pidx) {   // after the patch's last row block, item j
    static_assert(IPP <= 2, "wmax / slowflag hold two items");
    unsigned long long m = 0;
    unsigned slow_any = 0;
#pragma unroll
    for (int i = 0; i < IPP; ++i) {
      const int par = (j - i) & 1;
#pragma unroll
      for (int w = 0; w < NIW; ++w) {
        const unsigned long long v = wmax[par * NIW + w];
        m = v > m ? v : m;
      }
      slow_any |= slowflag[par];
      slowflag[par] = 0;
    }
    reinterpret_cast<unsigned long long*>(max_eig)[pidx] = m;
    tail_m = m > tail_m ? m : tail_m;   // (the producer alone)
    if (slow_any) {   // queue the patch for the exact re-evaluation (fvb_redo_kernel)
      const unsigned k = atomicAdd(&status[1], 1u);
      status[2 + k] = (unsigned)pidx;
    }
  };

  if (producer) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    tail_m = 0;
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
  Side<3> zprev;
  double tp[S], favg_zm[S];
  zprev.lam = 0.0;
#pragma unroll
  for (int u = 0; u < S; ++u) { tp[u] = 0.0; favg_zm[u] = 0.0; }
#pragma unroll
  for (int k = 0; k < 4; ++k) zprev.f[k] = 0.0;

  // 18 planes per item and NST = 3: the ring stage of plane zh is zh % 3 and its
  // mbarrier phase parity (zh / 3) & 1 for every item (each item uses six full
  // ring cycles), so both follow from zh alone.
  static_assert(NPL % (2 * NST) == 0, "stage / parity must be item-periodic");

  for (int jp = 0; jp < my_items; ++jp) {
    const int64_t pidx = item_patch(jp);
    const int y0 = (jp % IPP) * R;
    const double dx = __ddiv_rn(cell_size[pidx * 3], (double)P);   // vectorized.py:169
    const double inv = __ddiv_rn(dtv[pidx], dx);                    // vectorized.py:170
    const double half_inv = dmul(0.5, inv);
    if (tid == 0 && !inv_ok(inv)) slow = true;

    auto plane = [&](int zh, auto kind) {
      constexpr int K = decltype(kind)::value;
      const unsigned stg = (unsigned)(zh % NST), par = (unsigned)((zh / NST) & 1);
      const unsigned stp = stg == 0 ? NST - 1 : stg - 1;   // stage of plane zh-1
      const double* st = ring + stg * STAGE;
      const double* stc = ring + stp * STAGE;
      double* ys_w = ysb + (zh & 1) * YS;
      double* xs_w = xsb + (zh & 1) * XS;
      const double* ys_r = ysb + ((zh - 1) & 1) * YS;
      const double* xs_r = xsb + ((zh - 1) & 1) * XS;
      mbar_wait(&bars[stg], par);

      if (interior) {
        Side<3> zcur;
        double q[S];
        load_q<L>(st, ly + 1, x + 1, q);
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
          zcur = sd[2];
        } else {
          bool ok;
          closure_one_ranged<3>(q, cl, 2, zcur, ok);
          slow = slow | !ok;
        }
        if (K == kFirst) {
          double qc[S];
          load_q<L>(stc, ly + 1, x + 1, qc);
          const double cz = dmul(half_inv, speed_max(zcur.lam, zprev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) {
            tp[u] = dmul(cz, dsub(q[u], qc[u]));
            const double c = u == 0 ? qc[3] : zprev.f[u - 1];
            favg_zm[u] = dadd(c, u == 0 ? q[3] : zcur.f[u - 1]);
          }
        }
        if (K == kSteady || K == kZHi) {
          double qc[S], val[S], qn[S], rb[8];
          load_q<L>(stc, ly + 1, x + 1, qc);
          const double lx = xs_r[xs_at(0, ly, x + 1)];
          const double lyv = ys_r[ys_at(0, ly + 1, x)];
#pragma unroll
          for (int k = 0; k < 4; ++k) { rb[k] = xs_r[xs_at(k + 1, ly, x + 1)]; rb[4 + k] = ys_r[ys_at(k + 1, ly + 1, x)]; }
          const double cz = dmul(half_inv, speed_max(zcur.lam, zprev.lam));
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = qc[u];                       // _pass_copy
          // neighbours' normal momenta (flux component 0) kept from the dissipation loads
          double jxm, jxp, jym, jyp;
          load_q<L>(stc, ly + 1, x, qn);
          jxm = qn[1];
          dissipate<3>(val, half_inv, lx, qc, xs_r[xs_at(0, ly, x)], qn);
          load_q<L>(stc, ly + 1, x + 2, qn);
          jxp = qn[1];
          dissipate<3>(val, half_inv, lx, qc, xs_r[xs_at(0, ly, x + 2)], qn);
          load_q<L>(stc, ly, x + 1, qn);
          jym = qn[2];
          dissipate<3>(val, half_inv, lyv, qc, ys_r[ys_at(0, ly, x)], qn);
          load_q<L>(stc, ly + 2, x + 1, qn);
          jyp = qn[2];
          dissipate<3>(val, half_inv, lyv, qc, ys_r[ys_at(0, ly + 2, x)], qn);
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = dsub(val[u], tp[u]);
#pragma unroll
          for (int u = 0; u < S; ++u) {
            tp[u] = dmul(cz, dsub(q[u], qc[u]));
            val[u] = dadd(val[u], tp[u]);
          }
          add_flux(val, half_inv, [&](int u) { return u == 0 ? jxm : xs_r[xs_at(u, ly, x)]; },
                   [&](int u) { return u == 0 ? qc[1] : rb[u - 1]; },
                   [&](int u) { return u == 0 ? jxp : xs_r[xs_at(u, ly, x + 2)]; });
          add_flux(val, half_inv, [&](int u) { return u == 0 ? jym : ys_r[ys_at(u, ly, x)]; },
                   [&](int u) { return u == 0 ? qc[2] : rb[3 + u]; },
                   [&](int u) { return u == 0 ? jyp : ys_r[ys_at(u, ly + 2, x)]; });
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const double c = u == 0 ? qc[3] : zprev.f[u - 1];
            const double sum_p = dadd(c, u == 0 ? q[3] : zcur.f[u - 1]);
            val[u] = dadd(val[u], dmul(half_inv, dsub(favg_zm[u], sum_p)));
            favg_zm[u] = sum_p;
          }
          double* ob = outb + (zh & 1) * OUTN;
#pragma unroll
          for (int u = 0; u < S; ++u) {
            if (L == kAoS) ob[(ly * P + x) * S + u] = val[u];
            else ob[(u * R + ly) * P + x] = val[u];
          }
          fence_proxy_async();
        }
        zprev = zcur;
      } else if (K == kFirst || K == kSteady) {
        // the halo warp: stage rows 0 and 9 (y-face halo row and the ghost row
        // of the other half) need y-side data; interior rows need the x-face
        // halo columns' x-side data
        {
          const int r = lane < 16 ? 0 : SR - 1;
          double qh[S];
          load_q<L>(st, r, x + 1, qh);
          Side<3> sh;
          bool ok;
          closure_one_ranged<3>(qh, cl, 1, sh, ok);
          // (the ghost row is also checked by the half that owns it; flagging
          // it twice is harmless)
          slow = slow | !ok;
          put_ys(ys_w, r, x, sh);
        }
        if (lane < 2 * R) {   // x-face halo columns (hx = 0, 17) of the R interior rows
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
        if (jn < my_items) issue(jn, zn, stp);
        if (K == kSteady || K == kZHi) store_out(pidx, y0, zh - 2);
        if (K == kZHi && jp % IPP == IPP - 1) finish_patch(jp, pidx);
      }
    };

    plane(0, Kind<kZLo>{});
    plane(1, Kind<kFirst>{});
#pragma unroll STEADY_UNROLL
    for (int zh = 2; zh <= P; ++zh) plane(zh, Kind<kSteady>{});
    plane(NPL - 1, Kind<kZHi>{});
  }

  if (producer) bulk_wait_all0();
  fused_kernel_tail(tail, status, n, producer ? tail_m : 0ull);   // fvb_update_cfl: the step's max / dt
}

template <int L>
cudaError_t launch_impl(const FvbArgs& a, cudaStream_t st) {
  auto kfn = fused3d_half_kernel<L>;
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
  const CflTail tail{a.gmax, a.cfl, a.dx, a.dt_scalar, a.dt_patches, a.tail_dt};
  kfn<<<(unsigned)grid, NTHREADS, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl, tail);
  return cudaGetLastError();
}

}  // namespace f3h
}  // namespace fvb

cudaError_t fvb_launch_fused3d16_half(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb;
  if (a.n <= 0) return cudaSuccess;
  return a.layout == kAoS ? f3h::launch_impl<kAoS>(a, st) : f3h::launch_impl<kSoA>(a, st);
}
