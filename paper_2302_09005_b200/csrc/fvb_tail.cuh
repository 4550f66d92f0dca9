// fvb_tail.cuh -- the CFL step control that rides on the update's own launches
// (fvb_update_cfl): gmax = max over the batch's max_eig (NaN wins, as
// numpy's max), dt = (cfl*dx)/gmax into dt_scalar and every dt[patch].
//
// Status words (fvb_status_words = 2n + 8): [0] flag, [1] redo count, [2 .. 2n+1] redo
// list, [2n+2] redo-pass CTA counter, [2n+3] fused-kernel CTA counter, [2n+4..2n+5]
// unused, [2n+6..2n+7] the running max (u64 bit pattern, 8-byte aligned).
// Every fused kernel's CTAs fold the max_eig they wrote into the running max (one atomic
// per CTA); the last CTA takes it (resetting it for the next step) and, when the redo list
// is empty (the usual case), writes gmax and dt_scalar.  The redo pass that follows then
// broadcasts dt over the patches with all its CTAs (count 0), or -- after an exact
// re-evaluation -- its last CTA reduces max_eig afresh and writes gmax and dt itself.
#pragma once

#include <cstdint>

#include "fvb_exact.cuh"

namespace fvb {

struct CflTail {
  double* gmax;          // nullptr: no tail (plain fvb_update)
  double cfl, dx;
  double* dt_scalar;
  double* dt_patches;
  int do_dt;
};

__device__ __forceinline__ unsigned* redo_done_word(unsigned* status, int64_t n) { return status + 2 + 2 * n; }
__device__ __forceinline__ unsigned* fused_done_word(unsigned* status, int64_t n) { return status + 3 + 2 * n; }
__device__ __forceinline__ unsigned long long* tail_acc_word(unsigned* status, int64_t n) {
  return reinterpret_cast<unsigned long long*>(status + 6 + 2 * n);
}

__device__ __forceinline__ double cfl_dt(double cfl, double dx, double gmax) {
  return __ddiv_rn(dmul(cfl, dx), gmax);   // as set_dt_kernel / block_reduce_dt
}

// One CTA (blockDim a multiple of 32, <= 1024): the reduction and the dt broadcast.
__device__ __forceinline__ void block_reduce_dt(const double* __restrict__ max_eig, int64_t n,
                                                double* __restrict__ gmax, double cfl, double dx,
                                                double* __restrict__ dt_scalar, double* __restrict__ dt_patches,
                                                int do_dt) {
  __shared__ unsigned long long w[32];
  unsigned long long m = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(max_eig[i]);
    m = v > m ? v : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? w[threadIdx.x] : 0ull;
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
      m = v > m ? v : m;
    }
    if (threadIdx.x == 0) {
      *gmax = __longlong_as_double((long long)m);
      w[0] = m;
    }
  }
  __syncthreads();
  if (do_dt) {
    const double dt = cfl_dt(cfl, dx, __longlong_as_double((long long)w[0]));
    if (threadIdx.x == 0 && dt_scalar) *dt_scalar = dt;
    if (dt_patches)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dt_patches[i] = dt;
  }
}

// End of a persistent fused kernel, called by every thread: `m` is the max_eig bit pattern
// of the patches the thread wrote (0 for threads that wrote none).  Each CTA folds its max
// into the running max; the last CTA to arrive takes it and, if the redo list is empty,
// writes gmax and dt_scalar (the redo pass broadcasts dt).
__device__ __forceinline__ void fused_kernel_tail(const CflTail& tail, unsigned* status, int64_t n,
                                                  unsigned long long m) {
  if (!tail.gmax) return;
  __shared__ unsigned long long tw[32];
  __shared__ int last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) == 0) tw[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = tw[w] > m ? tw[w] : m;
    if (m) atomicMax(tail_acc_word(status, n), m);
    __threadfence();
    unsigned* done = fused_done_word(status, n);
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) {
      *done = 0;
      __threadfence();
      const unsigned long long g = atomicExch(tail_acc_word(status, n), 0ull);
      if (*((volatile unsigned*)status + 1) == 0) {   // else the redo pass reduces max_eig afresh
        const double gm = __longlong_as_double((long long)g);
        *tail.gmax = gm;
        if (tail.do_dt && tail.dt_scalar) *tail.dt_scalar = cfl_dt(tail.cfl, tail.dx, gm);
      }
    }
  }
}

// The same for kernels without CTA-wide barriers (warp-autonomous) or without shared
// memory to spare: every warp folds its lanes' `m` into the running max and counts itself
// in (total_warps = gridDim.x * warps per CTA); the last warp runs the step's gmax / dt_scalar.
__device__ __forceinline__ void fused_warp_tail(const CflTail& tail, unsigned* status, int64_t n,
                                                unsigned long long m, unsigned total_warps) {
  if (!tail.gmax) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
    m = v > m ? v : m;
  }
  if ((threadIdx.x & 31) != 0) return;
  if (m) atomicMax(tail_acc_word(status, n), m);
  __threadfence();
  unsigned* done = fused_done_word(status, n);
  if (atomicAdd(done, 1u) != total_warps - 1) return;
  *done = 0;
  __threadfence();
  const unsigned long long g = atomicExch(tail_acc_word(status, n), 0ull);
  if (*((volatile unsigned*)status + 1) == 0) {
    const double gm = __longlong_as_double((long long)g);
    *tail.gmax = gm;
    if (tail.do_dt && tail.dt_scalar) *tail.dt_scalar = cfl_dt(tail.cfl, tail.dx, gm);
  }
}

}  // namespace fvb
