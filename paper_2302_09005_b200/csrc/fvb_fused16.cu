// fvb_fused16.cu -- fused Rusanov patch update for p = 16 patches (2D and 3D).
//
// One persistent CTA streams whole patches through shared memory:
//
//   * TMA bulk copies (cp.async.bulk + mbarrier complete_tx) bring one haloed
//     z-plane (3D: 18x18 volumes x 5 unknowns = 12,960 B) or one whole haloed
//     patch (2D: 18x18 x 4 = 10,368 B) per stage into a ring of NST stages,
//     prefetched NST-LAG planes ahead.  AoS planes are one contiguous copy;
//     SoA planes one copy per unknown.
//   * 8 "interior" warps own the 16x16 cells of a plane (lane -> x, two rows
//     per warp) and march in z (3D).  They evaluate the Euler closure of
//     their volume ONCE (pressure, sound speed, 14 quotients sharing one
//     reciprocal refinement, see fvb_exact.cuh) and publish the y-side data
//     to shared memory; x-neighbour side data moves by warp shuffles; z-side
//     data is carried in registers from plane to plane.
//   * A 9th "halo" warp evaluates the x- and y-face halo volumes of the
//     plane (1-direction closures) while the interior warps work.
//   * Every cell then accumulates its 2d face terms in the reference order
//     (vectorized.py:161-200) and writes the interior plane to a staging
//     buffer that one thread stores back with a TMA bulk store.
//   * The per-patch maximum wave speed (vectorized.py:226-231) is reduced
//     with warp shuffles and written once per patch.
//
// Faces are evaluated from both sides (each cell forms its own 2d face
// terms from the neighbours' side data), which keeps every operation
// exactly the reference's and needs no sign-of-zero special cases.
#include <cuda_runtime.h>

#include <cstdlib>

#include "fvb_exact.cuh"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"

namespace fvb {
namespace f16 {

constexpr int P = 16, E = 18;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int D, int L>
struct Cfg {
  static constexpr int S = D + 2;
  static constexpr int NPL = D == 3 ? E : 1;        // stages (planes) per patch
  static constexpr int PLANE = E * E;               // volumes per stage
  static constexpr int STAGE = PLANE * S;           // doubles per stage
  static constexpr int NST = D == 3 ? 5 : 4;        // ring depth
  static constexpr int LAG = D == 3 ? 3 : 1;        // stages still read while a new one lands
  static constexpr int OUTN = P * P * S;            // doubles per output plane / patch
  static constexpr int64_t VOL = D == 3 ? (int64_t)E * E * E : (int64_t)E * E;
  static constexpr int64_t IVOL = D == 3 ? (int64_t)P * P * P : (int64_t)P * P;
  static constexpr int YS = S * E * P;              // y-side buffer: [S][E rows][P x]
  static constexpr int XS = 2 * S * P;              // x-side buffer: [lo/hi][S][P rows]
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_YS = OFF_RING + NST * STAGE;
  static constexpr int OFF_XS = OFF_YS + 2 * YS;
  static constexpr int OFF_OUT = OFF_XS + 2 * XS;
  static constexpr int OFF_WMAX = OFF_OUT + 2 * OUTN;
  static constexpr int OFF_BAR = OFF_WMAX + 16;
  static constexpr int TOTAL = OFF_BAR + NST;
  static constexpr size_t BYTES = (size_t)TOTAL * 8;
};

template <int D, int L>
__device__ __forceinline__ double qs(const double* st, int hy, int hx, int u) {
  constexpr int S = D + 2;
  return L == kAoS ? st[(hy * E + hx) * S + u] : st[(u * E + hy) * E + hx];
}

template <int D, int L>
__device__ __forceinline__ void load_state(const double* st, int hy, int hx, double (&q)[D + 2]) {
#pragma unroll
  for (int u = 0; u < D + 2; ++u) q[u] = qs<D, L>(st, hy, hx, u);
}

// y-side buffer [S][E][P]: component c of the side data of haloed row hy, interior column x
__device__ __forceinline__ int ys_idx(int c, int hy, int x) { return (c * E + hy) * P + x; }
// x-side buffer [2][S][P]: lo/hi halo column, component c, interior row y
__device__ __forceinline__ int xs_idx(int hi, int c, int y, int S) { return (hi * S + c) * P + y; }

template <int D>
__device__ __forceinline__ void store_side(double* buf, int idx_c0, int cstride, const Side<D>& s) {
  buf[idx_c0] = s.lam;
#pragma unroll
  for (int k = 0; k <= D; ++k) buf[idx_c0 + (k + 1) * cstride] = s.f[k];
}

template <int D>
__device__ __forceinline__ Side<D> load_side(const double* buf, int idx_c0, int cstride) {
  Side<D> s;
  s.lam = buf[idx_c0];
#pragma unroll
  for (int k = 0; k <= D; ++k) s.f[k] = buf[idx_c0 + (k + 1) * cstride];
  return s;
}

template <int D>
__device__ __forceinline__ Side<D> shfl_side_up(const Side<D>& s) {
  Side<D> r;
  r.lam = __shfl_up_sync(0xffffffffu, s.lam, 1, 16);
#pragma unroll
  for (int k = 0; k <= D; ++k) r.f[k] = __shfl_up_sync(0xffffffffu, s.f[k], 1, 16);
  return r;
}

template <int D>
__device__ __forceinline__ Side<D> shfl_side_down(const Side<D>& s) {
  Side<D> r;
  r.lam = __shfl_down_sync(0xffffffffu, s.lam, 1, 16);
#pragma unroll
  for (int k = 0; k <= D; ++k) r.f[k] = __shfl_down_sync(0xffffffffu, s.f[k], 1, 16);
  return r;
}

// Flux-difference term of one direction: inv*(0.5*(f_m + f_c) - 0.5*(f_c + f_p)),
// vectorized.py:193-200.  fm/fc/fp[0] are the normal momenta j_n.
template <int D>
__device__ __forceinline__ void flux_term(double (&F)[D + 2], double inv, double jm, const Side<D>& sm, double jc,
                                          const Side<D>& sc, double jp, const Side<D>& sp) {
  {
    const double favg_m = dmul(0.5, dadd(jm, jc));
    const double favg_p = dmul(0.5, dadd(jc, jp));
    F[0] = dmul(inv, dsub(favg_m, favg_p));
  }
#pragma unroll
  for (int u = 1; u < D + 2; ++u) {
    const double favg_m = dmul(0.5, dadd(sm.f[u - 1], sc.f[u - 1]));
    const double favg_p = dmul(0.5, dadd(sc.f[u - 1], sp.f[u - 1]));
    F[u] = dmul(inv, dsub(favg_m, favg_p));
  }
}

template <int D, int L, int MINB>
__global__ void __launch_bounds__(288, MINB)
fused16_kernel(const double* __restrict__ qin, double* __restrict__ qout, const double* __restrict__ cell_size,
               const double* __restrict__ dtv, double* __restrict__ max_eig, unsigned* __restrict__ status,
               int64_t n, Closure cl) {
  using C = Cfg<D, L>;
  constexpr int S = C::S;
  extern __shared__ __align__(128) double sm[];
  double* ring = sm + C::OFF_RING;
  double* ysb = sm + C::OFF_YS;
  double* xsb = sm + C::OFF_XS;
  double* outb = sm + C::OFF_OUT;
  unsigned long long* wmax = reinterpret_cast<unsigned long long*>(sm + C::OFF_WMAX);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);

  const int tid = threadIdx.x;
  const bool interior = tid < 256;
  const int warp = tid >> 5, lane = tid & 31;
  const int x = lane & 15;
  const int y = ((warp & 7) << 1) | (lane >> 4);
  const bool producer = tid == 256;

  const int64_t my_patches = (n > (int64_t)blockIdx.x) ? (n - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t G = my_patches * C::NPL;

  auto patch_of = [&](int64_t g) -> int64_t { return (int64_t)blockIdx.x + (g / C::NPL) * (int64_t)gridDim.x; };

  auto issue = [&](int64_t g) {
    const int64_t pidx = patch_of(g);
    const int zh = (int)(g % C::NPL);
    double* st = ring + (g % C::NST) * C::STAGE;
    uint64_t* bar = bars + (g % C::NST);
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)(C::STAGE * 8));
    if (L == kAoS) {
      tma_load_1d(st, qin + (pidx * C::VOL + (int64_t)zh * C::PLANE) * S, (uint32_t)(C::STAGE * 8), bar);
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_load_1d(st + u * C::PLANE, qin + ((int64_t)u * n + pidx) * C::VOL + (int64_t)zh * C::PLANE,
                    (uint32_t)(C::PLANE * 8), bar);
    }
  };

  auto has_output = [&](int64_t g) -> bool { return D == 2 || (g % C::NPL) >= 2; };

  auto store_out = [&](int64_t g) {
    const int64_t pidx = patch_of(g);
    const int z = D == 3 ? (int)(g % C::NPL) - 2 : 0;
    const double* src = outb + (g & 1) * C::OUTN;
    if (L == kAoS) {
      tma_store_1d(qout + (pidx * C::IVOL + (int64_t)z * P * P) * S, src, (uint32_t)(C::OUTN * 8));
    } else {
#pragma unroll
      for (int u = 0; u < S; ++u)
        tma_store_1d(qout + ((int64_t)u * n + pidx) * C::IVOL + (int64_t)z * P * P, src + u * P * P,
                     (uint32_t)(P * P * 8));
    }
    bulk_commit();
  };

  auto finish_patch_max = [&](int64_t j) {
    unsigned long long m = wmax[(j & 1) * 8];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const unsigned long long v = wmax[(j & 1) * 8 + w];
      m = v > m ? v : m;
    }
    max_eig[(int64_t)blockIdx.x + j * (int64_t)gridDim.x] = __longlong_as_double((long long)m);
  };

  if (producer) {
#pragma unroll
    for (int s = 0; s < C::NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (producer)
    for (int64_t g = 0; g <= C::NST - C::LAG && g < G; ++g) issue(g);

  bool bad = false;
  unsigned long long cm = 0;  // running max wave speed (bit pattern) of this thread's cells
  double inv = 0.0, half_inv = 0.0;
  // z-marching carries (3D): side data of planes zc-1 (z dir) and zc (x and z dirs), state of zc
  Side<D> prev2_z, prev_z, prev_x;
  double prev_q[S];
#pragma unroll
  for (int u = 0; u < S; ++u) prev_q[u] = 0.0;
  prev2_z.lam = prev_z.lam = prev_x.lam = 0.0;
#pragma unroll
  for (int k = 0; k <= D; ++k) prev2_z.f[k] = prev_z.f[k] = prev_x.f[k] = 0.0;

  for (int64_t g = 0; g < G; ++g) {
    const int zh = (int)(g % C::NPL);
    const int64_t pidx = patch_of(g);
    if (zh == 0) {
      const double dx = __ddiv_rn(cell_size[pidx * D], (double)P);   // vectorized.py:169
      inv = __ddiv_rn(dtv[pidx], dx);                                  // vectorized.py:170
      half_inv = dmul(0.5, inv);                                       // `0.5 * inv * a`, left to right
    }
    const double* st = ring + (g % C::NST) * C::STAGE;
    mbar_wait(&bars[g % C::NST], (uint32_t)((g / C::NST) & 1));
    const bool full_plane = D == 2 || (zh >= 1 && zh <= P);
    double* ys_w = ysb + (g & 1) * C::YS;
    double* xs_w = xsb + (g & 1) * C::XS;

    // ---------------- phase A: closures of this plane ----------------
    Side<D> cur_x = prev_x, cur_z = prev_z;
    double qcur[S];
    if (interior) {
      load_state<D, L>(st, y + 1, x + 1, qcur);
      const Thermo<D> T = thermo<D>(qcur, cl);
      bad = bad || T.bad;
      if (full_plane) {
        Side<D> sd[D];
        side_all<D>(qcur, T, sd);
        unsigned long long m = (unsigned long long)__double_as_longlong(sd[0].lam);
#pragma unroll
        for (int k = 1; k < D; ++k) {
          const unsigned long long v = (unsigned long long)__double_as_longlong(sd[k].lam);
          m = v > m ? v : m;
        }
        cm = m > cm ? m : cm;
        store_side<D>(ys_w, ys_idx(0, y + 1, x), E * P, sd[1]);
        cur_x = sd[0];
        if (D == 3) cur_z = sd[D - 1];
      } else {
        cur_z = side_one<D>(qcur, T, D - 1);
      }
    } else if (full_plane) {
      // y-face halo rows (haloed y = 0 and E-1) for interior x
      {
        const int hy = lane < 16 ? 0 : E - 1;
        double q[S];
        load_state<D, L>(st, hy, x + 1, q);
        const Thermo<D> T = thermo<D>(q, cl);
        bad = bad || T.bad;
        store_side<D>(ys_w, ys_idx(0, hy, x), E * P, side_one<D>(q, T, 1));
      }
      // x-face halo columns (haloed x = 0 and E-1) for interior rows
      {
        const int hi = lane >> 4;
        const int hx = hi ? E - 1 : 0;
        double q[S];
        load_state<D, L>(st, x + 1, hx, q);
        const Thermo<D> T = thermo<D>(q, cl);
        bad = bad || T.bad;
        store_side<D>(xs_w, xs_idx(hi, 0, x, S), P, side_one<D>(q, T, 0));
      }
    }
    if (producer) bulk_wait_read0();   // output buffer (g & 1) is free again
    __syncthreads();
    if (producer) {
      if (g >= 1 && g + C::NST - C::LAG < G) issue(g + C::NST - C::LAG);
      if (g >= 1 && has_output(g - 1)) store_out(g - 1);
      if (g >= 1 && (g - 1) % C::NPL == C::NPL - 1) finish_patch_max((g - 1) / C::NPL);
    }

    // ---------------- phase B: face terms and update ----------------
    if (interior) {
      const bool process = D == 2 || zh >= 2;
      if (process) {
        // centre volume: D == 2 -> this patch; D == 3 -> plane zc = zh - 1
        const double* stc = D == 2 ? st : ring + ((g - 1) % C::NST) * C::STAGE;
        const double* ys_r = D == 2 ? ys_w : ysb + ((g - 1) & 1) * C::YS;
        const double* xs_r = D == 2 ? xs_w : xsb + ((g - 1) & 1) * C::XS;
        const Side<D>& cx = D == 2 ? cur_x : prev_x;
        double qc[S];
#pragma unroll
        for (int u = 0; u < S; ++u) qc[u] = D == 2 ? qcur[u] : prev_q[u];
        double val[S];
#pragma unroll
        for (int u = 0; u < S; ++u) val[u] = qc[u];                        // _pass_copy

        // x faces: neighbour side data by shuffle, halo columns from smem
        double Fx[S], Fy[S];
        {
          Side<D> sl = shfl_side_up<D>(cx);
          Side<D> sr = shfl_side_down<D>(cx);
          if (x == 0) sl = load_side<D>(xs_r, xs_idx(0, 0, y, S), P);
          if (x == P - 1) sr = load_side<D>(xs_r, xs_idx(1, 0, y, S), P);
          double ql[S], qr[S];
          load_state<D, L>(stc, y + 1, x, ql);
          load_state<D, L>(stc, y + 1, x + 2, qr);
          dissipate<D>(val, half_inv, cx.lam, qc, sl.lam, ql);
          dissipate<D>(val, half_inv, cx.lam, qc, sr.lam, qr);
          flux_term<D>(Fx, inv, ql[1], sl, qc[1], cx, qr[1], sr);
        }
        // y faces: side data of rows y-1, y, y+1 from smem
        {
          const Side<D> sd = load_side<D>(ys_r, ys_idx(0, y, x), E * P);
          const Side<D> sc = load_side<D>(ys_r, ys_idx(0, y + 1, x), E * P);
          const Side<D> su = load_side<D>(ys_r, ys_idx(0, y + 2, x), E * P);
          double qd[S], qu[S];
          load_state<D, L>(stc, y, x + 1, qd);
          load_state<D, L>(stc, y + 2, x + 1, qu);
          dissipate<D>(val, half_inv, sc.lam, qc, sd.lam, qd);
          dissipate<D>(val, half_inv, sc.lam, qc, su.lam, qu);
          flux_term<D>(Fy, inv, qd[2], sd, qc[2], sc, qu[2], su);
        }
        if (D == 3) {
          double Fz[S];
          const double* stm = ring + ((g - 2) % C::NST) * C::STAGE;
          double qm[S];
          load_state<D, L>(stm, y + 1, x + 1, qm);
          dissipate<D>(val, half_inv, prev_z.lam, qc, prev2_z.lam, qm);
          dissipate<D>(val, half_inv, prev_z.lam, qc, cur_z.lam, qcur);
          flux_term<D>(Fz, inv, qm[D], prev2_z, qc[D], prev_z, qcur[D], cur_z);
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = dadd(dadd(dadd(val[u], Fx[u]), Fy[u]), Fz[u]);
        } else {
#pragma unroll
          for (int u = 0; u < S; ++u) val[u] = dadd(dadd(val[u], Fx[u]), Fy[u]);
        }
        double* ob = outb + (g & 1) * C::OUTN;
#pragma unroll
        for (int u = 0; u < S; ++u) {
          if (L == kAoS) ob[(y * P + x) * S + u] = val[u];
          else ob[u * P * P + y * P + x] = val[u];
        }
        fence_proxy_async();
      }
      if (D == 3) {
        prev2_z = prev_z;
        prev_z = cur_z;
        prev_x = cur_x;
#pragma unroll
        for (int u = 0; u < S; ++u) prev_q[u] = qcur[u];
      }
      if (zh == C::NPL - 1) {   // patch complete: per-warp max of the wave speeds
        unsigned long long m = cm;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
          m = v > m ? v : m;
        }
        if (lane == 0) wmax[((g / C::NPL) & 1) * 8 + warp] = m;
        cm = 0;
      }
    }
    // 3D: phase A of the next plane overwrites the y/x-side buffers (parity of
    // plane zh-1) that phase B just read, so every warp must be past phase B.
    if (D == 3) __syncthreads();
  }

  const int any_bad = __syncthreads_or(bad ? 1 : 0);
  if (producer) {
    if (G >= 1 && has_output(G - 1)) store_out(G - 1);
    if (G >= 1) finish_patch_max((G - 1) / C::NPL);
    bulk_wait_all0();
  }
  if (tid == 0 && any_bad) atomicOr(status, 1u);
}

// FVB_FUSED_MINB=1 selects the 1-CTA/SM build (no register cap); default 2 CTAs/SM.
static int min_blocks_choice() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FVB_FUSED_MINB");
    v = (e && e[0] == '1') ? 1 : 2;
  }
  return v;
}

template <int D, int L, int MINB>
cudaError_t launch_impl(const FvbArgs& a, cudaStream_t st) {
  using C = Cfg<D, L>;
  auto kfn = fused16_kernel<D, L, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 288, C::BYTES);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.n) grid = a.n;
  const Closure cl{a.gamma, a.gamma - 1.0};
  kfn<<<(unsigned)grid, 288, C::BYTES, st>>>(a.qin, a.qout, a.cell_size, a.dt, a.max_eig, a.status, a.n, cl);
  return cudaGetLastError();
}

template <int D, int L>
cudaError_t launch(const FvbArgs& a, cudaStream_t st) {
  return min_blocks_choice() == 1 ? launch_impl<D, L, 1>(a, st) : launch_impl<D, L, 2>(a, st);
}

}  // namespace f16
}  // namespace fvb

bool fvb_fused16_supported(int dim, int p, int layout) {
  return p == 16 && (dim == 2 || dim == 3) && (layout == fvb::kAoS || layout == fvb::kSoA);
}

cudaError_t fvb_launch_fused16(const FvbArgs& a, cudaStream_t st) {
  using namespace fvb;
  if (a.n <= 0) return cudaSuccess;
  if (a.dim == 2) return a.layout == kAoS ? f16::launch<2, kAoS>(a, st) : f16::launch<2, kSoA>(a, st);
  return a.layout == kAoS ? f16::launch<3, kAoS>(a, st) : f16::launch<3, kSoA>(a, st);
}
