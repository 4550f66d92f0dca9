// fvb_fused2d_warp.cu -- fused 2D Rusanov patch update for p = 16, warp-autonomous y march.
//
// Each warp owns TWO patches at a time (lane l -> patch slot l & 1, column
// x = l >> 1) and marches them row by row in y, exactly like the 3D kernels
// march planes in z:
//
//   * the y faces are evaluated once and re-used (negated) by the upper cell,
//     the y-side data and the face carries live in registers;
//   * x neighbours are exchanged through a per-warp shared-memory row buffer,
//     so the only synchronisation is __syncwarp -- no CTA barrier at all;
//   * haloed rows stream through a per-warp ring of TMA bulk-copy stages
//     (one 576 B row of each patch per stage, mbarrier complete_tx), issued
//     by lane 0 as soon as a row retires;
//   * the x-face halo columns (hx = 0, 17) are evaluated two rows at a time by
//     eight lanes;
//   * output rows are staged in shared memory and written back with TMA bulk
//     stores (one 512 B row per patch).
//
// Shared-memory layout per warp is bank-conflict free for the 32-byte AoS
// volumes: the two patches' rows are offset by 16 B modulo 128 B, so a
// quarter-warp's eight 16-byte LDS.128 accesses hit eight distinct bank
// quads.  (The block kernel in fvb_fused2d.cu reads 32-byte-strided LDS.64
// with 4-way conflicts.)
//
// Arithmetic: the reference's operation order, bit for bit (fvb_exact.cuh);
// the re-used y face differs from the reference only in the sign of an exact
// zero, which cannot occur inside the range gate (see fvb_fused3d.cu).  AoS only (the
// packed SoA layout uses the block kernel).
#include <cuda_runtime.h>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tma.cuh"

namespace fvb {
namespace f2w {

using namespace f16;

constexpr int P = 16, E = 18, S = 4;
constexpr int64_t VOL = (int64_t)E * E;
constexpr int64_t IVOL = (int64_t)P * P;
constexpr int ROWD = E * S;               // doubles per haloed patch row (576 B)
constexpr int OFFB = 82;                  // patch-B row offset in a stage: 656 B = 16 mod 128
constexpr int STGD = 154;                 // stage: two rows + padding (1,232 B)
constexpr int NS = 7;                     // ring stages per warp
constexpr int HB = 4;                     // halo-column rows per batch (16 lanes)
constexpr int XSD = 4 * 32;               // x-side row: [c][lane]
constexpr int HXR = 8;                    // halo x-side ring rows
constexpr int HXC = HXR * 4;              // halo x-side doubles per component: [row slot][side][patch slot]
constexpr int HXS = 4 * HXC;              // [c][row slot][side][patch slot]
constexpr int OUTR = P * S;               // one output row of one patch (512 B)
constexpr int OFFO = 130;                 // patch-B output offset: 1,040 B = 16 mod 128
constexpr int OUTD = OFFO + 2 * OUTR;     // output staging: two rows of each patch, stored together
constexpr int WPC = 4;                    // warps per CTA
#ifndef FVB2D_HY_UNROLL
#define FVB2D_HY_UNROLL 2
#endif
constexpr int HY_UNROLL = FVB2D_HY_UNROLL;
constexpr int W_RING = 0;
constexpr int W_XS = W_RING + NS * STGD;
constexpr int W_HX = W_XS + 2 * XSD;
constexpr int W_OUT = W_HX + HXS;
constexpr int W_BAR = W_OUT + OUTD;
constexpr int WARPD = (W_BAR + NS + 1) & ~1;   // doubles per warp (16 B multiple)
constexpr size_t BYTES = (size_t)WPC * WARPD * 8;

__device__ __forceinline__ void lds_q(const double* p, double (&q)[S]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
}
__device__ __forceinline__ void sts_q(double* p, const double (&q)[S]) {
  *reinterpret_cast<double2*>(p) = make_double2(q[0], q[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(q[2], q[3]);
}
__device__ __forceinline__ bool inv_ok(double inv) {
  const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
  return inv == 0.0 || (e >= 2u && e < 0x7ffu);
}

__global__ void __launch_bounds__(WPC * 32, 4)
fused2d_warp_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
                    const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
                    int64_t n, Closure cl) {
  extern __shared__ __align__(128) double sm[];
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
  double* wb = sm + warp * WARPD;
  double* ring = wb + W_RING;
  double* xsb = wb + W_XS;
  double* hxs = wb + W_HX;
  double* outb = wb + W_OUT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + W_BAR);

  const int ps = l & 1;          // patch slot
  const int x = l >> 1;          // interior column 0..15
  const int64_t items = (n + 1) >> 1;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;
  const int64_t tw = (int64_t)gridDim.x * WPC;
  const int my_items = items > gw ? (int)((items - 1 - gw) / tw + 1) : 0;
  const int rows_total = my_items * E;

  // Lane 0's issue cursor: the next haloed row to load (item ij, row ihy) and
  // its ring stage / patch pair, advanced incrementally (no divisions).
  int ij = 0, ihy = 0, is = 0, iissued = 0;
  int64_t ipa = 2 * gw;
  auto issue_next = [&]() {
    const bool vb = ipa + 1 < n;
    double* st = ring + is * STGD;
    uint64_t* bar = bars + is;
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)((vb ? 2 : 1) * ROWD * 8));
    tma_load_1d(st, qin + (ipa * VOL + ihy * E) * S, (uint32_t)(ROWD * 8), bar);
    if (vb) tma_load_1d(st + OFFB, qin + ((ipa + 1) * VOL + ihy * E) * S, (uint32_t)(ROWD * 8), bar);
    ++iissued;
    is = is == NS - 1 ? 0 : is + 1;
    if (++ihy == E) {
      ihy = 0;
      ++ij;
      ipa += 2 * tw;
    }
  };

  if (l == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) mbar_init(&bars[k], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (l == 0)
    while (iissued < NS && iissued < rows_total) issue_next();   // the whole ring; row r+NS refills r

  // per-lane constant offsets
  const int own = ps * OFFB + (x + 1) * S;          // this lane's volume in a stage
  const int left = ps * OFFB + x * S;               // x-1 neighbour
  const int right = ps * OFFB + (x + 2) * S;        // x+1 neighbour
  const bool lh = x == 0, rh = x == P - 1;          // neighbour is a face-halo column
  const int lcs = lh ? HXC : 32, rcs = rh ? HXC : 32;   // component strides of the neighbours' x-side data

  int s = 0;          // ring stage of the current row
  unsigned par = 0;   // its mbarrier phase parity
  int done = 0;       // rows consumed (refill trigger)
  // per-patch scalars of item j (an invalid slot mirrors patch A; its results are discarded),
  // loaded one item ahead so their latency never stalls the march
  auto scalars = [&](int j, double& cs, double& dtp) {
    cs = 1.0;
    dtp = 0.0;
    if (j < my_items) {
      const int64_t pa = 2 * (gw + (int64_t)j * tw);
      const int64_t pi = pa + ps < n ? pa + ps : pa;
      cs = __ldg(cell_size + pi * 2);
      dtp = __ldg(dtv + pi);
    }
  };
  double cs_next, dt_next;
  scalars(0, cs_next, dt_next);
  for (int j = 0; j < my_items; ++j) {
    const int64_t pa = 2 * (gw + (int64_t)j * tw);
    const int64_t pidx = pa + ps;
    const bool valid = pidx < n;
    const int64_t pl = valid ? pidx : pa;
    const double cs_cur = cs_next, dt_cur = dt_next;
    scalars(j + 1, cs_next, dt_next);
    const double dx = __ddiv_rn(cs_cur, (double)P);   // vectorized.py:169
    const double inv = __ddiv_rn(dt_cur, dx);          // vectorized.py:170
    const double half_inv = dmul(0.5, inv);
    bool slow = !inv_ok(inv);
    unsigned long long cm = 0;

    // y-march carries (row hy-1): own state and x-side data, y-side data,
    // the previous y face's dissipation term tp and unscaled flux sum favg
    double oq[S], olx = 0.0, ofx[3] = {0.0, 0.0, 0.0};
    Side<2> yprev;
    double tp[S], favg[S];
#pragma unroll
    for (int u = 0; u < S; ++u) { oq[u] = 0.0; tp[u] = 0.0; favg[u] = 0.0; }
    yprev.lam = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) yprev.f[k] = 0.0;

#pragma unroll HY_UNROLL
    for (int hy = 0; hy < E; ++hy) {
      const double* st = ring + s * STGD;                         // row hy
      const double* stp = ring + (s == 0 ? NS - 1 : s - 1) * STGD;   // row hy-1
      mbar_wait(&bars[s], par);

      // ---- halo columns hx = 0, 17 of rows hy .. hy+3 (x-side data only) ----
      if ((hy & 3) == 1 && hy < E - 1) {
#pragma unroll
        for (int d = 1; d < HB; ++d) {
          const int sd = s + d;
          mbar_wait(&bars[sd >= NS ? sd - NS : sd], par ^ (sd >= NS ? 1u : 0u));
        }
        if (l < 16) {
          const int hps = l & 1, side = (l >> 1) & 1, dr = l >> 2;
          const int sd = s + dr;
          const double* hst = ring + (sd >= NS ? sd - NS : sd) * STGD + hps * OFFB;
          double qh[S];
          lds_q(hst + (side ? E - 1 : 0) * S, qh);
          Side<2> sh;
          bool ok;
          closure_one_ranged<2>(qh, cl, 0, sh, ok);
          const int idx = (((hy + dr - 1) & (HXR - 1)) * 2 + side) * 2 + hps;
          hxs[0 * HXC + idx] = sh.lam;
#pragma unroll
          for (int k = 0; k < 3; ++k) hxs[(k + 1) * HXC + idx] = sh.f[k];
          // a halo volume outside the range gate invalidates its patch: a lane
          // with the same slot carries it into the per-patch vote
          const unsigned m = __ballot_sync(0xffffu, !ok);
          slow = slow | ((m & (ps ? 0xaaaau : 0x5555u)) != 0u);
        }
      }

      // ---- closure of this lane's volume of row hy ----
      Side<2> ycur;
      double q[S];
      lds_q(st + own, q);
      double nlx = 0.0, nfx[3] = {0.0, 0.0, 0.0};
      if (hy >= 1 && hy <= P) {
        Side<2> sd2[2];
        bool ok;
        closure_all_ranged<2>(q, cl, sd2, ok);
        slow = slow | !ok;
        const unsigned long long a = (unsigned long long)__double_as_longlong(sd2[0].lam);
        const unsigned long long b = (unsigned long long)__double_as_longlong(sd2[1].lam);
        const unsigned long long m = a > b ? a : b;
        cm = m > cm ? m : cm;
        double* xw = xsb + (hy & 1) * XSD + l;
        xw[0 * 32] = sd2[0].lam;
#pragma unroll
        for (int k = 0; k < 3; ++k) xw[(k + 1) * 32] = sd2[0].f[k];
        nlx = sd2[0].lam;
#pragma unroll
        for (int k = 0; k < 3; ++k) nfx[k] = sd2[0].f[k];
        ycur = sd2[1];
      } else {   // y-face halo rows: only their y-side data
        bool ok;
        closure_one_ranged<2>(q, cl, 1, ycur, ok);
        slow = slow | !ok;
      }
      // No __syncwarp here: the update below reads only data published in earlier
      // steps (x-side row hy-1, halo rows <= hy-1), so the closure of row hy and the
      // update of row hy-1 form one block the scheduler interleaves; the syncwarp at
      // the end of the step publishes row hy's x-side data and this step's halo batch.

      if (hy == 1) {
        // the face (0 | 1): minus face of the first interior row
        const double cy = dmul(half_inv, speed_max(ycur.lam, yprev.lam));
#pragma unroll
        for (int u = 0; u < S; ++u) {
          tp[u] = dmul(cy, dsub(q[u], oq[u]));
          const double c = u == 0 ? oq[2] : yprev.f[u - 1];
          favg[u] = dadd(c, u == 0 ? q[2] : ycur.f[u - 1]);
        }
      } else if (hy >= 2) {
        // ---- update of this lane's cell of row hy-1 (interior row hy-2) ----
        const double* xr = xsb + ((hy - 1) & 1) * XSD;
        const double* hr = hxs + ((hy - 2) & (HXR - 1)) * 4 + ps;   // halo x-side of row hy-1, side 0
        const double* ml = lh ? hr : xr + (l - 2);
        const double* mr = rh ? hr + 2 : xr + (l + 2);
        double val[S], qn[S];
#pragma unroll
        for (int u = 0; u < S; ++u) val[u] = oq[u];                        // _pass_copy
        // x- face, x+ face (vectorized.py:173-180)
        lds_q(stp + left, qn);
        const double jl = qn[1];
        dissipate<2>(val, half_inv, olx, oq, ml[0], qn);
        lds_q(stp + right, qn);
        const double jr = qn[1];
        dissipate<2>(val, half_inv, olx, oq, mr[0], qn);
        // y-: the previous face's term, negated; y+: this face's term
        const double cy = dmul(half_inv, speed_max(ycur.lam, yprev.lam));
#pragma unroll
        for (int u = 0; u < S; ++u) val[u] = dsub(val[u], tp[u]);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          tp[u] = dmul(cy, dsub(q[u], oq[u]));
          val[u] = dadd(val[u], tp[u]);
        }
        // flux differences x, y (vectorized.py:193-200), see fvb_fused3d.cu add_flux
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const double fm = u == 0 ? jl : ml[u * lcs];
          const double fc = u == 0 ? oq[1] : ofx[u - 1];
          const double fp = u == 0 ? jr : mr[u * rcs];
          val[u] = dadd(val[u], dmul(half_inv, dsub(dadd(fm, fc), dadd(fc, fp))));
        }
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const double c = u == 0 ? oq[2] : yprev.f[u - 1];
          const double sum_p = dadd(c, u == 0 ? q[2] : ycur.f[u - 1]);
          val[u] = dadd(val[u], dmul(half_inv, dsub(favg[u], sum_p)));
          favg[u] = sum_p;
        }
        // stage the output row; rows are stored in pairs (one 1 KB bulk store per patch), so
        // before the first row of a pair the previous pair's store must have read the buffer
        const int z = hy - 2;
        if (!(z & 1)) {
          if (l == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        sts_q(outb + ps * OFFO + (z & 1) * OUTR + x * S, val);
        if (z & 1) {
          fence_proxy_async();
          __syncwarp();
          if (l == 0) {
            tma_store_1d(qout + (pa * IVOL + (z - 1) * P) * S, outb, (uint32_t)(2 * OUTR * 8));
            if (pa + 1 < n)
              tma_store_1d(qout + ((pa + 1) * IVOL + (z - 1) * P) * S, outb + OFFO, (uint32_t)(2 * OUTR * 8));
            bulk_commit();
          }
        }
      }
      if (done >= 1) {
        __syncwarp();   // the previous row (this item's row hy-1, or the last item's row 17) is consumed
        if (l == 0 && iissued < rows_total) issue_next();   // refills its stage
      }
      ++done;
      s = s == NS - 1 ? 0 : s + 1;
      par ^= (s == 0);
#pragma unroll
      for (int u = 0; u < S; ++u) oq[u] = q[u];
      olx = nlx;
#pragma unroll
      for (int k = 0; k < 3; ++k) ofx[k] = nfx[k];
      yprev = ycur;
    }

    // ---- per-patch results: max wave speed (vectorized.py:226-231), redo queue ----
#pragma unroll
    for (int o = 2; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, cm, o);
      cm = v > cm ? v : cm;
    }
    const unsigned sm_ = __ballot_sync(0xffffffffu, slow);
    if (l < 2 && valid) {
      max_eig[pidx] = __longlong_as_double((long long)cm);
      if (sm_ & (ps ? 0xaaaaaaaau : 0x55555555u)) {
        const unsigned k = atomicAdd(&status[1], 1u);
        status[2 + k] = (unsigned)pidx;
      }
    }
  }
  if (l == 0) bulk_wait_all0();
}

}  // namespace f2w
}  // namespace fvb

cudaError_t fvb_launch_fused2d16_warp(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb::f2w;
  if (a.n <= 0) return cudaSuccess;
  auto kfn = fused2d_warp_kernel;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, WPC * 32, BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t items = (a.n + 1) / 2;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (items + WPC - 1) / WPC;
  if (grid > need) grid = need;
  const fvb::Closure cl{a.gamma, a.gamma - 1.0};
  kfn<<<(unsigned)grid, WPC * 32, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl);
  return cudaGetLastError();
}
