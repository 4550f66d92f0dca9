// fvb_tail.cuh -- the CFL step control that rides on the update's last CTA
// (fvb_update_cfl): gmax = max over the batch's max_eig (NaN wins, as
// numpy's max), dt = (cfl*dx)/gmax into dt_scalar and every dt[patch].
//
// Status words (fvb_status_words = 2n + 5): [0] flag, [1] redo count, [2 .. 2n+1] redo
// list, [2n+2] redo-pass CTA counter, [2n+3] fused-kernel CTA counter, [2n+4] "tail done".
// The fused kernel's last CTA runs the tail when its redo list is empty (the usual
// case) and marks it done; the redo pass then only clears the mark.  With a non-empty
// list the redo pass's last CTA runs it after the exact re-evaluation.
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
__device__ __forceinline__ unsigned* tail_mark_word(unsigned* status, int64_t n) { return status + 4 + 2 * n; }

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
    const double dt = __ddiv_rn(dmul(cfl, dx), __longlong_as_double((long long)w[0]));   // as set_dt_kernel
    if (threadIdx.x == 0 && dt_scalar) *dt_scalar = dt;
    if (dt_patches)
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dt_patches[i] = dt;
  }
}

// End of a persistent fused kernel: the CTA's max_eig / redo-list writes were made by
// `writer` before the __syncthreads that precedes this call.  The last CTA to arrive
// runs the tail if the redo list is empty and marks it done for the redo pass.
__device__ __forceinline__ void fused_kernel_tail(const CflTail& tail, const double* max_eig, unsigned* status,
                                                  int64_t n, bool writer) {
  if (!tail.gmax) return;
  __shared__ int last;
  __syncthreads();
  if (writer) {
    __threadfence();
    unsigned* done = fused_done_word(status, n);
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) *done = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (*((volatile unsigned*)status + 1) != 0) return;   // the redo pass will run the tail
  block_reduce_dt(max_eig, n, tail.gmax, tail.cfl, tail.dx, tail.dt_scalar, tail.dt_patches, tail.do_dt);
  if (threadIdx.x == 0) *tail_mark_word(status, n) = 1u;
}

}  // namespace fvb
