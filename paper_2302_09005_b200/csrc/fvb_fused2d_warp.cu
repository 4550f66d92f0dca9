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
#include "fvb_fast.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"
#include "fvb_tail.cuh"
#include "fvb_tma.cuh"

#include <cuda.h>

namespace fvb {
namespace f2w {

using namespace f16;

// Per-P configuration.  P <= 16: two patches per warp (lane l -> slot l & 1,
// column l >> 1); 16 < P <= 32: one patch per warp (lane = column).  Lanes
// whose column is >= P idle through the march (their results are discarded).
template <int P_>
struct W2 {
  static constexpr int P = P_, E = P + 2, S = 4;
  static constexpr int PPW = P <= 16 ? 2 : 1;                    // patches per warp
  static constexpr int64_t VOL = (int64_t)E * E;
  static constexpr int64_t IVOL = (int64_t)P * P;
  static constexpr int ROWD = E * S;                             // doubles per haloed patch row
  // A stage is one TMA tensor box of [PPW patches][1 row][BOXW doubles]: the row
  // padded by two zero-filled (out-of-bounds) doubles, so patch B's row starts
  // 8*(ROWD+2) = 16 mod 32 bytes after patch A's (ROWD is a multiple of 4):
  // conflict-free LDS.128 for the lane map.  One TMA op loads both patches' rows.
  static constexpr int BOXW = ROWD + 2;
  static constexpr int OFFB = BOXW;                              // patch-B row offset in a stage
  static constexpr int STGD = (PPW * BOXW + 15) / 16 * 16;      // stage (tensor TMA needs 128 B alignment)
  static constexpr int NS = 7;                                   // ring stages per warp
  static constexpr int HB = 4;                                   // halo-column rows per batch
  static constexpr int XSD = 4 * 32;                             // x-side row: [c][lane]
  static constexpr int HXR = 8;                                  // halo x-side ring rows
  static constexpr int HXC = HXR * 4;                            // per component: [row slot][side][patch slot]
  static constexpr int HXS = 4 * HXC;
  static constexpr int OUTR = P * S;                             // one output row of one patch
  // output staging: one TMA tensor box [PPW patches][2 rows][OUTR] (dense), stored
  // with one op every two rows; rows / patches past the tensor are not written
  static constexpr int OFFO = 2 * OUTR;                          // patch-B offset in the staging box
  static constexpr int OUTD = (PPW * 2 * OUTR + 15) / 16 * 16;
  static constexpr int W_RING = 0;
  static constexpr int W_XS = W_RING + NS * STGD;
  static constexpr int W_HX = W_XS + 2 * XSD;
  static constexpr int W_OUT = (W_HX + HXS + 15) / 16 * 16;      // tensor TMA source: 128 B aligned
  static constexpr int W_BAR = W_OUT + OUTD;
  static constexpr int WARPD = (W_BAR + NS + 15) / 16 * 16;      // doubles per warp (128 B multiple)
};
constexpr int S = 4;
constexpr int WPC = 4;                    // warps per CTA
#ifndef FVB2D_HY_UNROLL
#define FVB2D_HY_UNROLL 2
#endif
constexpr int HY_UNROLL = FVB2D_HY_UNROLL;
template <int P>
constexpr size_t bytes_of() { return (size_t)WPC * W2<P>::WARPD * 8; }

__device__ __forceinline__ void lds_q(const double* p, double (&q)[S]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
}
__device__ __forceinline__ void sts_q(double* p, const double (&q)[S]) {
  *reinterpret_cast<double2*>(p) = make_double2(q[0], q[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(q[2], q[3]);
}
#ifndef FVB2D_HALO_LANES
#define FVB2D_HALO_LANES 1
#endif
__device__ __forceinline__ bool inv_ok(double inv) {
  const unsigned e = ((unsigned)__double2hiint(inv) >> 20) & 0x7ffu;
  return inv == 0.0 || (e >= 2u && e < 0x7ffu);
}

// FAST (mode "fast", fvb_fast.cuh): one closure per volume with FMA contraction, face
// fluxes shared by the two cells of a face (the y face is carried down the march, both x
// faces are formed by the lane from its own and its neighbours' reconstructions), QOut
// within ~1e-16 relative of the reference instead of bit-exact.
template <int P, bool FAST = false>
__global__ void __launch_bounds__(WPC * 32, 4)
fused2d_warp_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
                    const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
                    int64_t n, Closure cl, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ CUtensorMap omap, int out_haloed, CflTail tail) {
  using C = W2<P>;
  constexpr int E = C::E, PPW = C::PPW, ROWD = C::ROWD, OFFB = C::OFFB, STGD = C::STGD, NS = C::NS, HB = C::HB;
  constexpr int XSD = C::XSD, HXR = C::HXR, HXC = C::HXC, OUTR = C::OUTR, OFFO = C::OFFO;
  constexpr int64_t VOL = C::VOL, IVOL = C::IVOL;
  constexpr int WARPD = C::WARPD, W_RING = C::W_RING, W_XS = C::W_XS, W_HX = C::W_HX, W_OUT = C::W_OUT,
                W_BAR = C::W_BAR;
  extern __shared__ __align__(128) double sm[];
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
  double* wb = sm + warp * WARPD;
  double* ring = wb + W_RING;
  double* xsb = wb + W_XS;
  double* hxs = wb + W_HX;
  double* outb = wb + W_OUT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wb + W_BAR);

  // HL (one patch per warp, P + 2 <= 32): lane l owns haloed column l, so the two
  // x-face halo columns are evaluated by lanes 0 and P+1 in the same pass as the
  // interior (no separate halo batches) and every lane finds its x neighbours'
  // data in the same row buffer.
  constexpr bool HL = PPW == 1 && P + 2 <= 32 && FVB2D_HALO_LANES;
  const int ps = PPW == 2 ? (l & 1) : 0;          // patch slot
  const int xl = HL ? l - 1 : (PPW == 2 ? (l >> 1) : l);   // interior column of this lane
  constexpr bool FULL = !HL && (PPW == 2 ? P == 16 : P == 32);   // every lane owns a column
  const bool act = FULL || (xl >= 0 && xl < P);   // lanes past the last column idle
  // (addressing only) HL: lane l addresses haloed column min(l, P+1), i.e. interior column -1 .. P
  const int x = HL ? (l < E ? l : E - 1) - 1 : (act ? xl : P - 1);
  const bool hlane = HL && (l == 0 || l == E - 1);        // HL: an x-face halo column
  constexpr int LST = PPW;                        // lane step between x neighbours
  const int64_t items = (n + PPW - 1) / PPW;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;
  const int64_t tw = (int64_t)gridDim.x * WPC;
  const int my_items = items > gw ? (int)((items - 1 - gw) / tw + 1) : 0;
  const int rows_total = my_items * E;

  // Lane 0's issue cursor: the next haloed row to load (item ij, row ihy) and
  // its ring stage / patch pair, advanced incrementally (no divisions).
  int ij = 0, ihy = 0, is = 0, iissued = 0;
  int64_t ipa = PPW * gw;
  auto issue_next = [&]() {
    double* st = ring + is * STGD;
    uint64_t* bar = bars + is;
    fence_proxy_async();
    // the whole box always lands (out-of-bounds elements, e.g. a missing patch B, read as zeros)
    mbar_expect_tx(bar, (uint32_t)(PPW * C::BOXW * 8));
    tma_load_3d(st, &tmap, 0, ihy, (int)ipa, bar);
    ++iissued;
    is = is == NS - 1 ? 0 : is + 1;
    if (++ihy == E) {
      ihy = 0;
      ++ij;
      ipa += PPW * tw;
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
  const int left = ps * OFFB + (x < 1 ? 0 : x) * S;              // x-1 neighbour (clamped for halo lanes)
  const int right = ps * OFFB + (x + 2 > E - 1 ? E - 1 : x + 2) * S;   // x+1 neighbour
  const bool lh = !HL && x == 0, rh = !HL && x == P - 1;   // neighbour is a face-halo column (halo ring)
  const int lcs = lh ? HXC : 32, rcs = rh ? HXC : 32;   // component strides of the neighbours' x-side data
  (void)lcs;
  (void)rcs;

  int s = 0;          // ring stage of the current row
  unsigned par = 0;   // its mbarrier phase parity
  int done = 0;       // rows consumed (refill trigger)
  // per-patch scalars of item j (an invalid slot mirrors patch A; its results are discarded),
  // loaded one item ahead so their latency never stalls the march
  auto scalars = [&](int j, double& cs, double& dtp) {
    cs = 1.0;
    dtp = 0.0;
    if (j < my_items) {
      const int64_t pa = PPW * (gw + (int64_t)j * tw);
      const int64_t pi = pa + ps < n ? pa + ps : pa;
      cs = __ldg(cell_size + pi * 2);
      dtp = __ldg(dtv + pi);
    }
  };
  double cs_next, dt_next;
  scalars(0, cs_next, dt_next);
  for (int j = 0; j < my_items; ++j) {
    const int64_t pa = PPW * (gw + (int64_t)j * tw);
    const int64_t pidx = pa + ps;
    const bool valid = pidx < n && act;
    const int64_t pl = valid ? pidx : pa;
    const double cs_cur = cs_next, dt_cur = dt_next;
    scalars(j + 1, cs_next, dt_next);
    const double dx = __ddiv_rn(cs_cur, (double)P);   // vectorized.py:169
    const double inv = __ddiv_rn(dt_cur, dx);          // vectorized.py:170
    const double half_inv = dmul(0.5, inv);
    bool slow = !inv_ok(inv);
    bool hslow = false;   // halo-batch gate failures, for patch slot l % PPW
    unsigned long long cm = 0;

    // y-march carries (row hy-1): own state and x-side data, y-side data,
    // the previous y face's dissipation term tp and unscaled flux sum favg
    double oq[S], olx = 0.0, ofx[3] = {0.0, 0.0, 0.0};
    Side<2> yprev;
    double tp[S], favg[S];
    double gyl[S];   // FAST: the lower y face of row hy-1
#pragma unroll
    for (int u = 0; u < S; ++u) { oq[u] = 0.0; tp[u] = 0.0; favg[u] = 0.0; gyl[u] = 0.0; }
    yprev.lam = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) yprev.f[k] = 0.0;

#pragma unroll HY_UNROLL
    for (int hy = 0; hy < E; ++hy) {
      const double* st = ring + s * STGD;                         // row hy
      const double* stp = ring + (s == 0 ? NS - 1 : s - 1) * STGD;   // row hy-1
      mbar_wait(&bars[s], par);

      // ---- halo columns hx = 0, P+1 of rows hy .. min(hy+3, P) (x-side data only) ----
      if (!HL && (hy & 3) == 1 && hy <= P) {
#pragma unroll
        for (int d = 1; d < HB; ++d) {
          const int sd = s + d;
          if ((P % HB == 0) || hy + d <= P) mbar_wait(&bars[sd >= NS ? sd - NS : sd], par ^ (sd >= NS ? 1u : 0u));
        }
        const int hps = l % PPW, side = (l / PPW) & 1, dr = l / (2 * PPW);
        if (l < 2 * PPW * HB && ((P % HB == 0) || hy + dr <= P)) {
          const int sd = s + dr;
          const double* hst = ring + (sd >= NS ? sd - NS : sd) * STGD + hps * OFFB;
          double qh[S];
          lds_q(hst + (side ? E - 1 : 0) * S, qh);
          Side<2> sh;
          bool ok = true;
          if constexpr (FAST) {
            const fast::Rpc w = fast::closure<2>(qh, cl, ok);
            sh.lam = fast::recon<2>(qh, w, 0, sh.f);
          } else {
            closure_one_ranged<2>(qh, cl, 0, sh, ok);
          }
          const int idx = (((hy + dr - 1) & (HXR - 1)) * 2 + side) * 2 + hps;
          hxs[0 * HXC + idx] = sh.lam;
#pragma unroll
          for (int k = 0; k < 3; ++k) hxs[(k + 1) * HXC + idx] = sh.f[k];
          // a halo volume outside the range gate invalidates its patch: a lane
          // with the same slot carries it into the per-patch vote
          hslow = hslow | !ok;   // a halo volume outside the gate invalidates patch slot hps
        }
      }

      // ---- closure of this lane's volume of row hy ----
      Side<2> ycur;
      double q[S];
      lds_q(st + own, q);
      double nlx = 0.0, nfx[3] = {0.0, 0.0, 0.0};
      if (hy >= 1 && hy <= P) {
        Side<2> sd2[2];
        bool ok = true;
        if constexpr (FAST) {
          const fast::Rpc w = fast::closure<2>(q, cl, ok);
          sd2[0].lam = fast::recon<2>(q, w, 0, sd2[0].f);
          sd2[1].lam = fast::recon<2>(q, w, 1, sd2[1].f);
        } else {
          closure_all_ranged<2>(q, cl, sd2, ok);
        }
        if (HL && hlane) hslow = hslow | !ok;   // x-face halo volume: gated like the reference's face box
        else slow = slow | !ok;
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
        bool ok = true;
        if constexpr (FAST) {
          const fast::Rpc w = fast::closure<2>(q, cl, ok);
          ycur.lam = fast::recon<2>(q, w, 1, ycur.f);
        } else {
          closure_one_ranged<2>(q, cl, 1, ycur, ok);
        }
        slow = slow | !ok;
      }
      // No __syncwarp here: the update below reads only data published in earlier
      // steps (x-side row hy-1, halo rows <= hy-1), so the closure of row hy and the
      // update of row hy-1 form one block the scheduler interleaves; the syncwarp at
      // the end of the step publishes row hy's x-side data and this step's halo batch.

      if (FAST && hy == 1) {
        fast::face<2>(gyl, 1, oq, yprev.lam, yprev.f, q, ycur.lam, ycur.f);   // face (0 | 1)
      } else if (FAST && hy >= 2) {
        // ---- fast update of this lane's cell of row hy-1: both x faces from the lane's and
        // its neighbours' reconstructions, the y faces carried / formed here ----
        const double* xr = xsb + ((hy - 1) & 1) * XSD;
        const double* hr = hxs + ((hy - 2) & (HXR - 1)) * 4 + ps;
        const double* ml = lh ? hr : xr + (HL && l == 0 ? 0 : l - LST);
        const double* mr = rh ? hr + 2 : xr + (HL && l == 31 ? 31 : l + LST);
        double qn[S], fn[3], gx_lo[S], gx_hi[S], gy_hi[S], val[S];
        lds_q(stp + left, qn);
#pragma unroll
        for (int k = 0; k < 3; ++k) fn[k] = ml[(k + 1) * lcs];
        fast::face<2>(gx_lo, 0, qn, ml[0], fn, oq, olx, ofx);
        lds_q(stp + right, qn);
#pragma unroll
        for (int k = 0; k < 3; ++k) fn[k] = mr[(k + 1) * rcs];
        fast::face<2>(gx_hi, 0, oq, olx, ofx, qn, mr[0], fn);
        fast::face<2>(gy_hi, 1, oq, yprev.lam, yprev.f, q, ycur.lam, ycur.f);
#pragma unroll
        for (int u = 0; u < S; ++u) {
          val[u] = __fma_rn(half_inv, dsub(dadd(gx_lo[u], gyl[u]), dadd(gx_hi[u], gy_hi[u])), oq[u]);
          gyl[u] = gy_hi[u];
        }
        const int z = hy - 2;
        if (!(z & 1)) {
          if (l == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        if (act) sts_q(outb + ps * OFFO + (z & 1) * OUTR + x * S, val);
        if ((z & 1) || ((P & 1) && z == P - 1)) {
          const int z0 = z & ~1;
          fence_proxy_async();
          __syncwarp();
          if (l == 0) {
            tma_store_3d(&omap, out_haloed ? S : 0, z0 + out_haloed, (int)pa, outb);
            bulk_commit();
          }
        }
      } else if (hy == 1) {
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
        const double* ml = lh ? hr : xr + (HL && l == 0 ? 0 : l - LST);
        const double* mr = rh ? hr + 2 : xr + (HL && l == 31 ? 31 : l + LST);
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
        if (act) sts_q(outb + ps * OFFO + (z & 1) * OUTR + x * S, val);
        if ((z & 1) || ((P & 1) && z == P - 1)) {   // a full pair, or the last row of an odd P
          const int z0 = z & ~1;   // (for odd P the box's second row is past the tensor: not written)
          fence_proxy_async();
          __syncwarp();
          if (l == 0) {
            // out_haloed: the rows land in the interior of a haloed batch (row z0+1, inner
            // offset S doubles = 32 B); for odd P the box's second row hits the upper halo
            // row, which the shell fill (fvb_halo_shell) rewrites afterwards
            tma_store_3d(&omap, out_haloed ? S : 0, z0 + out_haloed, (int)pa, outb);
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
    if (!act) cm = 0;
#pragma unroll
    for (int o = PPW; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, cm, o);
      cm = v > cm ? v : cm;
    }
    // slot of lane l: l % PPW, both for the own volumes (slow) and the halo tasks (hslow)
    const unsigned sm_ = __ballot_sync(0xffffffffu, (slow && act) || hslow);
    const unsigned slot_mask = PPW == 2 ? (ps ? 0xaaaaaaaau : 0x55555555u) : 0xffffffffu;
    if (l < PPW && pidx < n) {
      max_eig[pidx] = __longlong_as_double((long long)cm);
      if (sm_ & slot_mask) {
        const unsigned k = atomicAdd(&status[1], 1u);
        status[2 + k] = (unsigned)pidx;
      }
    }
  }
  if (tail.gmax) {   // fvb_update_cfl: fold the warp's max_eig into the step's max (fvb_tail.cuh)
    __syncwarp();
    unsigned long long m = 0;
    for (int i = l; i < my_items * PPW; i += 32) {
      const int j = i / PPW;
      const int64_t pidx = PPW * (gw + (int64_t)j * tw) + (i - j * PPW);
      if (pidx < n) {
        const unsigned long long v = (unsigned long long)__double_as_longlong(max_eig[pidx]);
        m = v > m ? v : m;
      }
    }
    fused_warp_tail(tail, status, n, m, gridDim.x * WPC);
  }
  if (l == 0) bulk_wait_all0();
}

}  // namespace f2w
}  // namespace fvb

namespace fvb {
namespace f2w {

// QIn as a 3D tensor {row doubles, rows, patches}; box {row + 2 zero-filled, 1, PPW}
template <int P>
cudaError_t make_qin_map(const FvbArgs& a, CUtensorMap* tm) {
  using C = W2<P>;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {(cuuint64_t)C::ROWD, (cuuint64_t)C::E, (cuuint64_t)a.n};
  const cuuint64_t strides[2] = {(cuuint64_t)C::ROWD * 8, (cuuint64_t)C::ROWD * C::E * 8};
  const cuuint32_t box[3] = {(cuuint32_t)C::BOXW, 1u, (cuuint32_t)C::PPW};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.qin), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// QOut as a 3D tensor {row doubles, rows, patches}; box {row, 2 rows, PPW}
template <int P>
cudaError_t make_qout_map(const FvbArgs& a, CUtensorMap* tm) {
  using C = W2<P>;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  // out_haloed: the output tensor is the haloed batch {row of E volumes, E rows, patches}
  const cuuint64_t dims[3] = {(cuuint64_t)(a.out_haloed ? C::ROWD : C::OUTR), (cuuint64_t)(a.out_haloed ? C::E : P),
                              (cuuint64_t)a.n};
  const cuuint64_t strides[2] = {(cuuint64_t)(a.out_haloed ? C::ROWD : C::OUTR) * 8,
                                 (cuuint64_t)(a.out_haloed ? C::ROWD * C::E : C::OUTR * P) * 8};
  const cuuint32_t box[3] = {(cuuint32_t)C::OUTR, 2u, (cuuint32_t)C::PPW};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.qout, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int P, bool FAST = false>
cudaError_t launch(const FvbArgs& a, cudaStream_t st) {
  auto kfn = fused2d_warp_kernel<P, FAST>;
  constexpr size_t BYTES = bytes_of<P>();
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, WPC * 32, BYTES);
  if (per_sm < 1) per_sm = 1;
  const int64_t items = (a.n + W2<P>::PPW - 1) / W2<P>::PPW;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (items + WPC - 1) / WPC;
  if (grid > need) grid = need;
  const Closure cl{a.gamma, a.gamma - 1.0};
  CUtensorMap tm, om;
  e = make_qin_map<P>(a, &tm);
  if (e == cudaSuccess) e = make_qout_map<P>(a, &om);
  if (e != cudaSuccess) return e;
  const CflTail tail{a.gmax, a.cfl, a.dx, a.dt_scalar, a.dt_patches, a.tail_dt};
  kfn<<<(unsigned)grid, WPC * 32, BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl, tm,
                                               om, a.out_haloed, tail);
  return cudaGetLastError();
}
}  // namespace f2w
}  // namespace fvb

// 2D patches of P = 2 .. 32 volumes per axis (AoS)
bool fvb_fused2d_warp_supported(int p) { return p >= 2 && p <= 32; }

cudaError_t fvb_launch_fused2d16_warp(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb::f2w;
  if (a.n <= 0) return cudaSuccess;
  switch (a.p) {
#define FVB_P(k) \
  case k:        \
    return launch<k>(a, st);
    FVB_P(2) FVB_P(3) FVB_P(4) FVB_P(5) FVB_P(6) FVB_P(7) FVB_P(8) FVB_P(9) FVB_P(10) FVB_P(11) FVB_P(12)
    FVB_P(13) FVB_P(14) FVB_P(15) FVB_P(16) FVB_P(17) FVB_P(18) FVB_P(19) FVB_P(20) FVB_P(21) FVB_P(22)
    FVB_P(23) FVB_P(24) FVB_P(25) FVB_P(26) FVB_P(27) FVB_P(28) FVB_P(29) FVB_P(30) FVB_P(31) FVB_P(32)
#undef FVB_P
    default:
      return cudaErrorInvalidValue;
  }
}

// mode "fast" (fvb_fast.cuh): every 2D AoS shape the warp kernel takes (p = 2 .. 32)
bool fvb_fast2d_supported(int dim, int p, int layout) {
  return dim == 2 && layout == fvb::kAoS && fvb_fused2d_warp_supported(p);
}

cudaError_t fvb_launch_fast2d16(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb::f2w;
  if (a.n <= 0) return cudaSuccess;
  switch (a.p) {
#define FVB_P(k) \
  case k:        \
    return launch<k, true>(a, st);
    FVB_P(2) FVB_P(3) FVB_P(4) FVB_P(5) FVB_P(6) FVB_P(7) FVB_P(8) FVB_P(9) FVB_P(10) FVB_P(11) FVB_P(12)
    FVB_P(13) FVB_P(14) FVB_P(15) FVB_P(16) FVB_P(17) FVB_P(18) FVB_P(19) FVB_P(20) FVB_P(21) FVB_P(22)
    FVB_P(23) FVB_P(24) FVB_P(25) FVB_P(26) FVB_P(27) FVB_P(28) FVB_P(29) FVB_P(30) FVB_P(31) FVB_P(32)
#undef FVB_P
    default:
      return cudaErrorInvalidValue;
  }
}
