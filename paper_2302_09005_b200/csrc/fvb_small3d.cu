// fvb_small3d.cu -- fused 3D Rusanov update for small patches, even p = 2 .. 8 (p = 4:
// BASELINE config 4, 1M patches, with a tuned face-halo split).
//
// A persistent CTA of 64 threads processes PPC = 1 patch per iteration (one
// thread per interior cell; 6 CTAs per SM).  The haloed patch(es) of an
// iteration are contiguous in HBM (AoS) and arrive with ONE TMA bulk copy into
// a 2-stage ring.  Per iteration:
//   A  every thread evaluates the closure of its interior volume (all three
//      directions); the one-direction closures of the 96 face-halo volumes
//      are balanced over the warps (1.5 passes each); side data (lam,
//      f[1..4]) goes to per-direction shared arrays.            -- barrier
//   B  every cell accumulates its six face terms from the side arrays in the
//      reference order (vectorized.py:161-200) and writes the interior to a
//      staging buffer stored with one TMA bulk store per iteration. -- barrier
// Closures use the range-gated exact arithmetic of fvb_exact.cuh; patches
// leaving the gate go to the exact redo list (fvb_redo_kernel).
#include <cuda_runtime.h>

#include "fvb_exact.cuh"
#include "fvb_fast.cuh"
#include <cstring>

#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tail.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace fs {

using namespace f16;

template <int P, bool FAST = false>
struct Cfg {
  static constexpr int S = 5;
  static constexpr int E = P + 2;
  static constexpr int VOL = E * E * E;             // haloed volumes per patch
  static constexpr int IVOL = P * P * P;            // interior cells per patch
#ifndef FVB_SMALL3D_NOB
#define FVB_SMALL3D_NOB 2
#endif
#ifndef FVB_SMALL3D_PPC
#define FVB_SMALL3D_PPC 1
#endif
  // patches per CTA iteration: 1 (64 threads, ~34 KB, 6 CTAs/SM) measured 11 % faster than
  // 2 (128 threads, 3 CTAs/SM) -- barriers over two warps, twice the independent CTAs
  static constexpr int PPC = FVB_SMALL3D_PPC;
  static constexpr int THREADS = (PPC * IVOL + 31) / 32 * 32;   // whole warps; threads past the cells idle
  static constexpr int NHALO = 6 * P * P;           // face-halo volumes per patch
  static constexpr int LINE = E * P * P;            // records of one direction: (E along n) x P x P
  // BOXED (fast p = 4): a patch is staged as two TMA tensor boxes -- the 4 interior z planes
  // whole (6 x 6 volumes, incl. the x / y face halos) and the 4 x 4 face-halo rows of the two
  // z-halo planes (22 doubles from byte 32 of each row: the box start must be 16-byte aligned,
  // so the last unknown of volume 0 and the first of volume 5 come along) -- 7,168 of the
  // patch's 8,640 bytes: the z-halo planes' edge / corner volumes are never read
#ifndef FVB_SMALL3D_BOXES
#define FVB_SMALL3D_BOXES 1
#endif
  static constexpr bool BOXED = FAST && P == 4 && FVB_SMALL3D_BOXES && PPC == 1;
  static constexpr int BOXA = P * E * E * S;          // interior z planes, whole
  static constexpr int ZROW = P * S + 2;              // a z-halo row's face volumes + 2 boundary doubles
  static constexpr int BOXC = 2 * P * ZROW;
  static constexpr int PSTAGE = BOXED ? BOXA + BOXC : VOL * S;   // doubles per staged patch
  static constexpr int STAGE = PPC * PSTAGE;        // doubles per ring stage
#ifndef FVB_SMALL3D_NST8
#define FVB_SMALL3D_NST8 3
#endif
  static constexpr int NST = FAST && P >= 8 ? FVB_SMALL3D_NST8 : 2;   // fast p = 8: a third stage, 754.8 vs 768 us (x3p8)
  // exact: side data of one patch, 3 directions; FAST: (r, p, c) of every haloed volume
  static constexpr int SIDE = FAST ? VOL * 3 : 3 * S * LINE;
  static constexpr int OUTN = (PPC * IVOL * S + 15) / 16 * 16;   // staging buffers 128-byte aligned (TMA)
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_SIDE = OFF_RING + NST * STAGE;
  static constexpr int OFF_OUT = (OFF_SIDE + PPC * SIDE + 15) / 16 * 16;
  // output staging: NOB buffers (1: the store of iteration g-1 must have read it
  // before phase B of iteration g writes; checked before the mid-iteration barrier)
  static constexpr int NOB = FAST ? 1 : FVB_SMALL3D_NOB;   // FAST: one buffer measured 1.5 % faster (C4)
  static constexpr int OFF_WMAX = OFF_OUT + NOB * OUTN;
  static constexpr int OFF_FLAG = OFF_WMAX + 2 * (THREADS / 32);   // wmax double-buffered
  static constexpr int OFF_BAR = OFF_FLAG + 1;   // two 32-bit flag words
  static constexpr int TOTAL = OFF_BAR + NST;
  static constexpr size_t BYTES = (size_t)TOTAL * 8;
};

// Record (direction n, component c) of the volume whose haloed coordinate along
// n is hn and whose interior coordinates across n are (a, b) -- a, b the
// lower / higher remaining axes (x: (y, z), y: (x, z), z: (x, y)).  The layouts
// are chosen for the thread mapping below (a half-warp = the 16 cells of one y
// row pair (x, z) at fixed y), so every LDS.64 / STS.64 of a half-warp hits 16
// distinct bank pairs:
//   x records [a=y][hn=hx][b=z]   lanes vary (hx, z): hn*P + b
//   y records [hn=hy][b=z][a=x]   lanes vary (z, x) at fixed hy: b*P + a
//   z records [b=y][hn=hz][a=x]   lanes vary (hz, x): hn*P + a
template <int P>
__device__ __forceinline__ int side_at(int n, int c, int hn, int a, int b) {
  using C = Cfg<P>;
  constexpr int E = C::E;
  const int base = (n * C::S + c) * C::LINE;
  if (n == 0) return base + (a * E + hn) * P + b;
  if (n == 1) return base + (hn * P + b) * P + a;
  return base + (b * E + hn) * P + a;
}

template <int P>
__device__ __forceinline__ void put_rec(double* side, int n, int hn, int a, int b, const Side<3>& s) {
  side[side_at<P>(n, 0, hn, a, b)] = s.lam;
#pragma unroll
  for (int k = 0; k < 4; ++k) side[side_at<P>(n, k + 1, hn, a, b)] = s.f[k];
}

// Output staging order.  The thread mapping puts (x, z) in a half-warp, for which
// the AoS interior order (x, y, z) makes the z step a multiple of 16 doubles: the
// five STS.64 per cell would be 4-way bank-conflicted (ncu: 4x the ideal
// wavefronts at p = 4).  The staging is therefore (x, z, y) -- word offsets
// 5x + 4z mod 16 distinct at p = 4 -- and one tiled TMA store whose tensor map
// walks QOut as {x*S, z, y, patch} writes it back in AoS order.
#ifndef FVB_SMALL3D_TOUT
#define FVB_SMALL3D_TOUT 1
#endif
constexpr bool TOUT = FVB_SMALL3D_TOUT != 0;
// Trimmed staging (three bulk copies per patch, the z-halo planes' edge rows
// skipped): p = 8 1,047 -> 1,034 us; p = 4 2.74 -> 2.84 ms (the extra TMA ops
// cost more than the 8 % of bytes), so only for p >= 6.
#ifndef FVB_SMALL3D_TRIM
#define FVB_SMALL3D_TRIM (P >= 6 && !(P & 1))
#endif
#ifndef FVB_SMALL3D_REMAP
#define FVB_SMALL3D_REMAP 1
#endif

// FAST (mode "fast", fvb_fast.cuh): the same staging and side-data records, filled from one
// FMA closure per volume; phase B forms each of the cell's six faces as the shared flux G
// (the neighbour forms the same G bit for bit), QOut within ~1e-16 relative.
template <int P, bool FAST = false>
__global__ void __launch_bounds__(Cfg<P, FAST>::THREADS, P == 4 ? (FAST ? 8 : 6) / Cfg<P, FAST>::PPC : 1)
small3d_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
               const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
               int64_t n_patches, Closure cl, const __grid_constant__ CUtensorMap omap, CflTail tail,
               const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap cmap) {
  using C = Cfg<P, FAST>;
  constexpr int S = C::S, E = C::E;
  // Odd P: a patch is an odd multiple of 8 bytes, so neither the bulk copies nor the
  // tensor store (16-byte granularity) can address it.  The CTA stages it with 8-byte
  // cp.async copies into the same ring (the mbarrier counts every thread's arrive),
  // and writes the output back with coalesced 8-byte stores.
  constexpr bool ODD = (P & 1) != 0;
  constexpr bool TOUT_P = TOUT && !ODD;
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + C::OFF_RING;
  double* sideb = sm + C::OFF_SIDE;
  double* outb = sm + C::OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + C::OFF_WMAX);
  unsigned* slowflag = reinterpret_cast<unsigned*>(sm + C::OFF_FLAG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);

  const int tid = threadIdx.x;
  const int lp = tid / C::IVOL;              // patch slot within the iteration
  const int cell = tid % C::IVOL;
  // cell -> (x, z, y) with x fastest, then z: a half-warp covers one y row pair
  // (x, z) at fixed y, for which the 40-byte AoS volume stride is conflict-free
  // (word offsets 4*hz + 5*hx mod 16 are distinct).
  const int cx = cell % P, cz = (cell / P) % P, cy = cell / (P * P);
  const int warp = tid >> 5, lane = tid & 31;
  // stage offset (doubles) of haloed volume (hx, hy, hz) of a staged patch
  auto soff = [&](int hx, int hy, int hz) -> int {
    if constexpr (C::BOXED) {
      return (hz >= 1 && hz <= P) ? ((hz - 1) * E + hy) * E * S + hx * S
                                  : C::BOXA + ((hz > P ? P : 0) + hy - 1) * C::ZROW + (hx - 1) * S + 1;
    } else {
      return ((hz * E + hy) * E + hx) * S;
    }
  };
  constexpr int WPP = C::THREADS / 32 / C::PPC;   // warps per patch (PPC > 1 needs IVOL % 32 == 0)
  static_assert(C::PPC == 1 || C::IVOL % 32 == 0, "patch slots must own whole warps");
  const int64_t ngroups = (n_patches + C::PPC - 1) / C::PPC;
  const int G = ngroups > (int64_t)blockIdx.x ? (int)((ngroups - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto group_of = [&](int g) -> int64_t { return (int64_t)blockIdx.x + (int64_t)g * gridDim.x; };
  auto patches_in = [&](int64_t grp) -> int {
    const int64_t left = n_patches - grp * C::PPC;
    return left < C::PPC ? (int)left : C::PPC;
  };

  auto issue = [&](int g) {
    const int64_t grp = group_of(g);
    const int np = patches_in(grp);
    double* st = ring + (g % C::NST) * C::STAGE;
    uint64_t* bar = bars + (g % C::NST);
    fence_proxy_async();
    if (FVB_SMALL3D_TRIM) {
      // per patch: rows 1..P of the two z-halo planes and the P interior planes whole --
      // the z-halo planes' y-halo rows are edges / corners the update never reads
      // (8 % of a p = 4 patch's bytes); every piece is 16-byte aligned for even P
      constexpr uint32_t ZROWS = (uint32_t)(P * E * S * 8), MID = (uint32_t)(P * E * E * S * 8);
      mbar_expect_tx(bar, (uint32_t)np * (2 * ZROWS + MID));
      for (int k = 0; k < np; ++k) {
        const double* src = qin + (grp * C::PPC + k) * (int64_t)C::VOL * S;
        double* dst = st + k * C::VOL * S;
        tma_load_1d(dst + E * S, src + E * S, ZROWS, bar);
        tma_load_1d(dst + E * E * S, src + E * E * S, MID, bar);
        tma_load_1d(dst + ((E - 1) * E * E + E) * S, src + ((E - 1) * E * E + E) * S, ZROWS, bar);
      }
    } else if (C::BOXED) {   // {x*S, y, z, patch} boxes: z = 1..P whole, z = 0 / P+1 face rows
      mbar_expect_tx(bar, (uint32_t)(C::PSTAGE * 8));
      tma_load_4d(st, &amap, 0, 0, 1, (int)grp, bar);
      tma_load_4d(st + C::BOXA, &cmap, S - 1, 1, 0, (int)grp, bar);
    } else {
      mbar_expect_tx(bar, (uint32_t)(np * C::VOL * S * 8));
      tma_load_1d(st, qin + grp * C::PPC * (int64_t)C::VOL * S, (uint32_t)(np * C::VOL * S * 8), bar);
    }
  };

  auto issue_coop = [&](int g) {   // odd P: every thread copies its share, then arrives
    const int64_t grp = group_of(g);
    const int np = patches_in(grp);
    double* st = ring + (g % C::NST) * C::STAGE;
    const double* src = qin + grp * C::PPC * (int64_t)C::VOL * S;
    for (int i = tid; i < np * C::VOL * S; i += C::THREADS) cp_async8(st + i, src + i);
    cp_async_mbar_arrive_noinc(bars + (g % C::NST));
  };

  if (tid == 0) {
    for (int s = 0; s < C::NST; ++s) mbar_init(&bars[s], ODD ? C::THREADS : 1);
    slowflag[0] = slowflag[1] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (ODD) {
    for (int g = 0; g < C::NST && g < G; ++g) issue_coop(g);
  } else if (tid == 0) {
    for (int g = 0; g < C::NST && g < G; ++g) issue(g);
  }

  unsigned stg = 0, par = 0;
  // per-patch scalars, loaded one iteration ahead (their latency used to stall the closures)
  auto scalars = [&](int g, double& cs, double& dtp) {
    cs = 1.0;
    dtp = 0.0;
    if (g < G) {
      const int64_t grp = group_of(g);
      if (lp < patches_in(grp)) {
        const int64_t pi = grp * C::PPC + lp;
        cs = __ldg(cell_size + pi * 3);
        dtp = __ldg(dtv + pi);
      }
    }
  };
  double cs_next, dt_next;
  scalars(0, cs_next, dt_next);
  for (int g = 0; g < G; ++g) {
    const int64_t grp = group_of(g);
    const int np = patches_in(grp);
    const bool active = lp < np;
    const int64_t pidx = grp * C::PPC + lp;
    const double cs_cur = cs_next, dt_cur = dt_next;
    scalars(g + 1, cs_next, dt_next);
    const double* st = ring + stg * C::STAGE + lp * C::PSTAGE;
    double* side = sideb + lp * C::SIDE;
    mbar_wait(&bars[stg], par);
    auto qat = [&](int hx, int hy, int hz, int u) { return st[soff(hx, hy, hz) + u]; };
    auto load = [&](int hx, int hy, int hz, double (&q)[S]) {
#pragma unroll
      for (int u = 0; u < S; ++u) q[u] = qat(hx, hy, hz, u);
    };

    bool slow = false;
    unsigned long long cmax = 0;
    double inv = 0.0, half_inv = 0.0;
    if (active) {
      const double dx = __ddiv_rn(cs_cur, (double)P);   // vectorized.py:169
      inv = __ddiv_rn(dt_cur, dx);                       // vectorized.py:170
      half_inv = dmul(0.5, inv);
      const unsigned ie = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
      slow = !(inv == 0.0 || (ie >= 2u && ie < 0x7ffu));
      // ---- A1: closure of this thread's interior volume ----
      double q[S];
      load(cx + 1, cy + 1, cz + 1, q);
      Side<3> sd[3];
      bool ok = true;
      if constexpr (FAST) {
        // (r, p, c) of the volume; the faces reconstruct from it in phase B.  Wave speeds:
        // max_d |j_d r| + c = (max_d |j_d r|) + c (RN is monotonic)
        const fast::Rpc w = fast::closure<3>(q, cl, ok);
        double* rp = side + (((cz + 1) * E + (cy + 1)) * E + (cx + 1)) * 3;
        rp[0] = w.r;
        rp[1] = w.p;
        rp[2] = w.c;
        const double u0 = fabs(__dmul_rn(q[1], w.r)), u1 = fabs(__dmul_rn(q[2], w.r)), u2 = fabs(__dmul_rn(q[3], w.r));
        const double um = speed_max(speed_max(u0, u1), u2);
        sd[0].lam = sd[1].lam = sd[2].lam = __dadd_rn(um, w.c);
      } else {
        closure_all_ranged<3>(q, cl, sd, ok);
      }
      slow = slow | !ok;
      unsigned long long m = (unsigned long long)__double_as_longlong(sd[0].lam);
      unsigned long long v = (unsigned long long)__double_as_longlong(sd[1].lam);
      m = v > m ? v : m;
      v = (unsigned long long)__double_as_longlong(sd[2].lam);
      cmax = v > m ? v : m;
      if constexpr (!FAST) {
        put_rec<P>(side, 0, cx + 1, cy, cz, sd[0]);
        put_rec<P>(side, 1, cy + 1, cx, cz, sd[1]);
        put_rec<P>(side, 2, cz + 1, cx, cy, sd[2]);
      }
    }
    // ---- A2: face-halo volumes, one direction each, balanced over the CTA's warps ----
    // The PPC x 96 tasks form 3*PPC chunks of 32 (one patch slot, one face pair -> a
    // warp-uniform direction).  Warp w evaluates chunk w whole and half of chunk
    // 2*PPC + w/2, so every warp does 1.5 passes (a per-patch split would leave one
    // warp of each patch with two passes and stall the barrier).
    auto halo_eval = [&](int lpt, int nd, int hn, int a, int b) {
      const int hx = nd == 0 ? hn : a + 1;
      const int hy = nd == 1 ? hn : (nd == 0 ? a + 1 : b + 1);
      const int hz = nd == 2 ? hn : b + 1;
      const double* stt = ring + stg * C::STAGE + lpt * C::PSTAGE;
      double qh[S];
#pragma unroll
      for (int u = 0; u < S; ++u) qh[u] = stt[soff(hx, hy, hz) + u];
      Side<3> sh;
      bool okh = true;
      if constexpr (FAST) {
        const fast::Rpc w = fast::closure<3>(qh, cl, okh);
        double* rp = sideb + lpt * C::SIDE + ((hz * E + hy) * E + hx) * 3;
        rp[0] = w.r;
        rp[1] = w.p;
        rp[2] = w.c;
        if (!okh) atomicOr(&slowflag[g & 1], 1u << lpt);
        return;
      } else if (nd == 0) {
        closure_one_ranged<3>(qh, cl, 0, sh, okh);
      } else if (nd == 1) {
        closure_one_ranged<3>(qh, cl, 1, sh, okh);
      } else {
        closure_one_ranged<3>(qh, cl, 2, sh, okh);
      }
      if (!okh) atomicOr(&slowflag[g & 1], 1u << lpt);   // rare: queue that patch for the exact pass
      put_rec<P>(sideb + lpt * C::SIDE, nd, hn, a, b, sh);
    };
    if (P == 4 && C::THREADS == 64 * C::PPC) {
      // task idx -> (face side h, a, b), chosen per direction so that a half-warp's
      // stage loads and record stores hit distinct bank pairs where possible:
      //   x faces: a in {0,1} / {2,3} per half-warp, h, b      (loads and stores)
      //   y faces: a, b, h per half-warp                        (loads and stores)
      //   z faces: a, h, b in {0,1} / {2,3} per half-warp       (stores; loads 2 pairs 2-way)
      auto halo_task = [&](int chunk, int idx) {
        const int lpt = chunk / 3, nd = chunk % 3;
        if (lpt >= np) return;
        int h, a, b;
        if (!FVB_SMALL3D_REMAP) {
          a = idx & 3;
          b = (idx >> 2) & 3;
          h = idx >> 4;
        } else if (nd == 0) {
          a = (idx & 1) | ((idx >> 4) << 1);
          h = (idx >> 1) & 1;
          b = (idx >> 2) & 3;
        } else if (nd == 1) {
          a = idx & 3;
          b = (idx >> 2) & 3;
          h = idx >> 4;
        } else {
          a = idx & 3;
          h = (idx >> 2) & 1;
          b = ((idx >> 3) & 1) | ((idx >> 4) << 1);
        }
        halo_eval(lpt, nd, h ? E - 1 : 0, a, b);
      };
      halo_task(warp, lane);   // chunks 0 .. 2*PPC-1 whole, chunks 2*PPC .. 3*PPC-1 in halves
      if ((lane >> 4) == (warp & 1)) halo_task(2 * C::PPC + (warp >> 1), lane);
    } else {
      // other p: tasks (patch slot, face, a, b) strided over the CTA
      for (int h = tid; h < C::PPC * C::NHALO; h += C::THREADS) {
        const int lpt = h / C::NHALO, r = h - lpt * C::NHALO;
        if (lpt >= np) break;
        const int face = r / (P * P), ab = r - face * P * P;
        halo_eval(lpt, face >> 1, (face & 1) ? E - 1 : 0, ab % P, ab / P);
      }
    }
    if (__any_sync(0xffffffffu, slow) && lane == 0) atomicOr(&slowflag[g & 1], 1u << (lp & 31));
    if (C::NOB == 1 && tid == 0) bulk_wait_read0();   // the single staging buffer, stored last iteration, is free
    __syncthreads();

    // ---- B: face terms and update of this thread's cell ----
    if (FAST && active) {
      double qc[S], qn[S], val[S], slo[S], shi[S];
      load(cx + 1, cy + 1, cz + 1, qc);
      const int hcc[3] = {cx + 1, cy + 1, cz + 1};
      auto rpc_at = [&](int hx, int hy, int hz) -> fast::Rpc {
        const double* rp = side + ((hz * E + hy) * E + hx) * 3;
        return fast::Rpc{rp[0], rp[1], rp[2]};
      };
      const fast::Rpc wc = rpc_at(hcc[0], hcc[1], hcc[2]);
#pragma unroll
      for (int nd = 0; nd < 3; ++nd) {
        double fc[4], fn[4], G[S];
        const double lc = fast::recon<3>(qc, wc, nd, fc);
#pragma unroll
        for (int sh = -1; sh <= 1; sh += 2) {
          int hq[3] = {hcc[0], hcc[1], hcc[2]};
          hq[nd] += sh;
          load(hq[0], hq[1], hq[2], qn);
          const double ln = fast::recon<3>(qn, rpc_at(hq[0], hq[1], hq[2]), nd, fn);
          if (sh < 0) fast::face<3>(G, nd, qn, ln, fn, qc, lc, fc);   // lower face: neighbour below
          else fast::face<3>(G, nd, qc, lc, fc, qn, ln, fn);          // upper face: neighbour above
#pragma unroll
          for (int u = 0; u < S; ++u) {
            if (sh < 0) slo[u] = nd == 0 ? G[u] : dadd(slo[u], G[u]);
            else shi[u] = nd == 0 ? G[u] : dadd(shi[u], G[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < S; ++u) val[u] = __fma_rn(half_inv, dsub(slo[u], shi[u]), qc[u]);
      const int lin = TOUT_P ? (cy * P + cz) * P + cx : (cz * P + cy) * P + cx;
#pragma unroll
      for (int u = 0; u < S; ++u) outb[(g % C::NOB) * C::OUTN + (lp * C::IVOL + lin) * S + u] = val[u];
      if (!ODD) fence_proxy_async();
    } else if (active) {
      double qc[S], qn[S], val[S];
      load(cx + 1, cy + 1, cz + 1, qc);
#pragma unroll
      for (int u = 0; u < S; ++u) val[u] = qc[u];                       // _pass_copy
      const int hcc[3] = {cx + 1, cy + 1, cz + 1};
      const int ab[3][2] = {{cy, cz}, {cx, cz}, {cx, cy}};
      // dissipation: x-, x+, y-, y+, z-, z+ (vectorized.py:173-180)
#pragma unroll
      for (int nd = 0; nd < 3; ++nd) {
        const double lc = side[side_at<P>(nd, 0, hcc[nd], ab[nd][0], ab[nd][1])];
#pragma unroll
        for (int sh = -1; sh <= 1; sh += 2) {
          int hq[3] = {hcc[0], hcc[1], hcc[2]};
          hq[nd] += sh;
          load(hq[0], hq[1], hq[2], qn);
          dissipate<3>(val, half_inv, lc, qc, side[side_at<P>(nd, 0, hcc[nd] + sh, ab[nd][0], ab[nd][1])], qn);
        }
      }
      // flux differences x, y, z (vectorized.py:193-200), exact half_inv form (fvb_fused3d.cu)
#pragma unroll
      for (int nd = 0; nd < 3; ++nd) {
        int hm[3] = {hcc[0], hcc[1], hcc[2]}, hp[3] = {hcc[0], hcc[1], hcc[2]};
        hm[nd] -= 1;
        hp[nd] += 1;
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const double fm = u == 0 ? qat(hm[0], hm[1], hm[2], 1 + nd)
                                   : side[side_at<P>(nd, u, hcc[nd] - 1, ab[nd][0], ab[nd][1])];
          const double fc = u == 0 ? qc[1 + nd] : side[side_at<P>(nd, u, hcc[nd], ab[nd][0], ab[nd][1])];
          const double fp = u == 0 ? qat(hp[0], hp[1], hp[2], 1 + nd)
                                   : side[side_at<P>(nd, u, hcc[nd] + 1, ab[nd][0], ab[nd][1])];
          val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
        }
      }
      const int lin = TOUT_P ? (cy * P + cz) * P + cx    // staging order (x, z, y), see TOUT
                             : (cz * P + cy) * P + cx;   // AoS interior order (x fastest)
#pragma unroll
      for (int u = 0; u < S; ++u) outb[(g % C::NOB) * C::OUTN + (lp * C::IVOL + lin) * S + u] = val[u];
      if (!ODD) fence_proxy_async();
    }
    // per-patch max wave speed: 64-bit max as (high word, low word) warp reductions
    {
      const unsigned hi = (unsigned)(cmax >> 32), lo = (unsigned)cmax;
      const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
      const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      if (lane == 0) wmax[(g & 1) * (C::THREADS / 32) + warp] = ((unsigned long long)mhi << 32) | mlo;
    }
    if (C::NOB == 2 && tid == 0) bulk_wait_read0();   // staging buffer (g & 1) was stored two iterations ago
    __syncthreads();
    if (tid == 0) {
      // output of this group, per-patch maxima, redo list; then refill the freed stage
      if (TOUT_P)
        tma_store_4d(&omap, 0, 0, 0, (int)(grp * C::PPC), outb + (g % C::NOB) * C::OUTN);
      else if (!ODD)
        tma_store_1d(qout + grp * C::PPC * (int64_t)C::IVOL * S, outb + (g % C::NOB) * C::OUTN,
                     (uint32_t)(np * C::IVOL * S * 8));
      if (!ODD) bulk_commit();
      const unsigned flags = slowflag[g & 1];
      for (int k = 0; k < np; ++k) {
        unsigned long long m = 0;
        for (int w = 0; w < WPP; ++w) {
          const unsigned long long v = wmax[(g & 1) * (C::THREADS / 32) + k * WPP + w];
          m = v > m ? v : m;
        }
        max_eig[grp * C::PPC + k] = __longlong_as_double((long long)m);
        if (flags & (1u << k)) {
          const unsigned r = atomicAdd(&status[1], 1u);
          status[2 + r] = (unsigned)(grp * C::PPC + k);
        }
      }
      slowflag[g & 1] = 0;   // next set in iteration g+2, after the next barrier
      if (!ODD && g + C::NST < G) issue(g + C::NST);   // stage of this group, fully consumed
    }
    if (ODD) {   // coalesced write-back of the staged output, then refill the consumed stage
      const double* ob = outb + (g % C::NOB) * C::OUTN;
      double* dst = qout + grp * C::PPC * (int64_t)C::IVOL * S;
      for (int i = tid; i < np * C::IVOL * S; i += C::THREADS) dst[i] = ob[i];
      if (g + C::NST < G) issue_coop(g + C::NST);
    }
    stg = stg == C::NST - 1 ? 0 : stg + 1;
    par ^= (stg == 0);
  }
  if (tail.gmax) {   // fvb_update_cfl: fold the CTA's max_eig into the step's max (fvb_tail.cuh)
    __syncthreads();   // thread 0 wrote them
    unsigned long long m = 0;
    for (int i = tid; i < G * C::PPC; i += C::THREADS) {
      const int64_t pidx = group_of(i / C::PPC) * C::PPC + i % C::PPC;
      if (pidx < n_patches) {
        const unsigned long long v = (unsigned long long)__double_as_longlong(max_eig[pidx]);
        m = v > m ? v : m;
      }
    }
    fused_warp_tail(tail, status, n_patches, m, gridDim.x * (C::THREADS / 32));
  }
  if (tid == 0) bulk_wait_all0();
}

template <int P, bool FAST = false>
cudaError_t launch(const FvbArgs& a, cudaStream_t st) {
  using C = Cfg<P, FAST>;
  auto kfn = small3d_kernel<P, FAST>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, C::THREADS, C::BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t groups = (a.n + C::PPC - 1) / C::PPC;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > groups) grid = groups;
  const Closure cl{a.gamma, a.gamma - 1.0};
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  if (TOUT && !(P & 1)) {   // QOut as {x*S, z, y, patch}: the staging's (x, z, y) order, AoS in memory
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[4] = {(cuuint64_t)P * C::S, (cuuint64_t)P, (cuuint64_t)P, (cuuint64_t)a.n};
    const cuuint64_t strides[3] = {(cuuint64_t)P * P * C::S * 8, (cuuint64_t)P * C::S * 8,
                                   (cuuint64_t)C::IVOL * C::S * 8};
    const cuuint32_t box[4] = {(cuuint32_t)(P * C::S), (cuuint32_t)P, (cuuint32_t)P, (cuuint32_t)C::PPC};
    const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    if (enc(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a.qout, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const CflTail tail{a.gmax, a.cfl, a.dx, a.dt_scalar, a.dt_patches, a.tail_dt};
  CUtensorMap amap, cmap;   // BOXED: QIn as {x*S, y, z, patch}
  memset(&amap, 0, sizeof(amap));
  memset(&cmap, 0, sizeof(cmap));
  if (C::BOXED) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return cudaErrorNotSupported;
    constexpr int E = C::E, S = C::S;
    const cuuint64_t dims[4] = {(cuuint64_t)E * S, (cuuint64_t)E, (cuuint64_t)E, (cuuint64_t)a.n};
    const cuuint64_t strides[3] = {(cuuint64_t)E * S * 8, (cuuint64_t)E * E * S * 8, (cuuint64_t)C::VOL * S * 8};
    const cuuint32_t boxa[4] = {(cuuint32_t)(E * S), (cuuint32_t)E, (cuuint32_t)P, 1u};
    const cuuint32_t boxc[4] = {(cuuint32_t)C::ZROW, (cuuint32_t)P, (cuuint32_t)E, 1u};
    const cuuint32_t esa[4] = {1u, 1u, 1u, 1u}, esc[4] = {1u, 1u, (cuuint32_t)(E - 1), 1u};   // z = 0, E-1
    if (enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.qin), dims, strides, boxa, esa,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.qin), dims, strides, boxc, esc,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  kfn<<<(unsigned)grid, C::THREADS, C::BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n,
                                                    cl, omap, tail, amap, cmap);
  return cudaGetLastError();
}

}  // namespace fs
}  // namespace fvb

// 3D AoS patches of p = 2, 4 .. 8 (one patch per CTA; p = 4 has the tuned halo split).
// Odd p makes the haloed / interior patch sizes odd multiples of 8 bytes, which the
// TMA bulk copies (16-byte granularity) cannot address per patch: those stage with
// 8-byte cp.async copies and write back with plain stores (ODD in the kernel).
bool fvb_small3d_supported(int dim, int p, int layout) {
  // p = 3 stays on the generic kernel: 27 cells fill one warp poorly (measured 9.2 vs 9.8 Gcell/s)
  return dim == 3 && p >= 2 && p <= 8 && p != 3 && layout == fvb::kAoS;
}

cudaError_t fvb_launch_small3d(const FvbArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  cudaError_t e;
  switch (a.p) {
    case 2: e = fvb::fs::launch<2>(a, st); break;
    case 4: e = fvb::fs::launch<4>(a, st); break;
    case 5: e = fvb::fs::launch<5>(a, st); break;
    case 7: e = fvb::fs::launch<7>(a, st); break;
    case 6: e = fvb::fs::launch<6>(a, st); break;
    case 8: e = fvb::fs::launch<8>(a, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return fvb_launch_redo(a, st);
}

// mode "fast" (fvb_fast.cuh): every shape the small-patch kernel takes (3D AoS p = 2, 4 .. 8)
bool fvb_fast_small3d_supported(int dim, int p, int layout) { return fvb_small3d_supported(dim, p, layout); }

cudaError_t fvb_launch_fast_small3d(const FvbArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  cudaError_t e;
  switch (a.p) {
    case 2: e = fvb::fs::launch<2, true>(a, st); break;
    case 4: e = fvb::fs::launch<4, true>(a, st); break;
    case 5: e = fvb::fs::launch<5, true>(a, st); break;
    case 6: e = fvb::fs::launch<6, true>(a, st); break;
    case 7: e = fvb::fs::launch<7, true>(a, st); break;
    case 8: e = fvb::fs::launch<8, true>(a, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return fvb_launch_redo(a, st);
}
