// fvb_kernels.h -- internal launcher interface between the C ABI and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

struct BoxInfo {
  int64_t trig_rho, trig_p, first_nonpos, first_badpl;
};

constexpr int kTotalsBlocks = 592;   // partial-sum blocks of fvb_totals (scratch = blocks x unknowns doubles)
constexpr int kScratchBlocks = 2048;  // scratch partials available (fvb_totals_scratch_bytes): also the halo CTAs

struct FvbArgs {
  int dim, p, layout;
  int64_t n;
  double gamma;
  const double* qin;
  double* qout;
  const double* cell_size;
  const double* dt;
  double* max_eig;
  unsigned* status;
  int out_haloed = 0;   // 1: qout is a haloed AoS batch (N*V*S); the update fills its interior
  // CFL tail (fvb_update_cfl, fvb_tail.cuh): the fused kernel's last CTA / warp writes
  // *gmax (and dt_scalar) from the running max, the redo pass broadcasts dt = (cfl*dx)/gmax
  double* gmax = nullptr;
  double cfl = 0.0, dx = 0.0;
  double* dt_scalar = nullptr;
  double* dt_patches = nullptr;
  int tail_dt = 0;
};


cudaError_t fvb_launch_generic(const FvbArgs& a, cudaStream_t st);
cudaError_t fvb_launch_step_record(int64_t* step, const double* dt_scalar, const unsigned* status,
                                   const double* totals, int s, const double* gmax, double* dt_hist, int* flag_hist,
                                   double* totals_hist, double* gmax_hist, cudaStream_t st);
cudaError_t fvb_launch_fused16(const FvbArgs& a, cudaStream_t st);
cudaError_t fvb_launch_fused3d16_half(const FvbArgs& a, cudaStream_t st);
cudaError_t fvb_launch_fused2d16_warp(const FvbArgs& a, cudaStream_t st);
bool fvb_fused2d_warp_supported(int p);
bool fvb_fast3d_supported(int dim, int p, int layout);
cudaError_t fvb_launch_fast3d16(const FvbArgs& a, cudaStream_t st);
bool fvb_fast2d_supported(int dim, int p, int layout);
// measurement hook (fvb_time_next_update): record the pending start / stop event of this
// thread's next update around its main kernel (the redo pass calls the stop mark first)
void fvb_timing_mark_start(cudaStream_t st);
void fvb_timing_mark_stop(cudaStream_t st);
bool fvb_fast_small3d_supported(int dim, int p, int layout);
cudaError_t fvb_launch_fast_small3d(const FvbArgs& a, cudaStream_t st);   // includes its redo pass
cudaError_t fvb_launch_fast2d16(const FvbArgs& a, cudaStream_t st);
cudaError_t fvb_launch_redo(const FvbArgs& a, cudaStream_t st);
bool fvb_fused16_supported(int dim, int p, int layout);
bool fvb_small3d_supported(int dim, int p, int layout);
cudaError_t fvb_launch_small3d(const FvbArgs& a, cudaStream_t st);
cudaError_t fvb_launch_locate(int dim, int p, int64_t n, double gamma, int layout, const double* qin,
                              BoxInfo* info, cudaStream_t st);
cudaError_t fvb_launch_pack(const double* src, double* dst, int64_t n, int64_t vols, int s, int to_soa,
                            cudaStream_t st);
cudaError_t fvb_launch_reduce_dt(const double* max_eig, int64_t n, double cfl, double dx, double* gmax,
                                 double* dt_scalar, double* dt_patches, int do_dt, cudaStream_t st);
cudaError_t fvb_launch_set_dt(const double* gmax, double cfl, double dx, double* dt_scalar, double* dt_patches,
                              int64_t n, cudaStream_t st);
cudaError_t fvb_launch_patch_max_eig(int dim, int p, int64_t n, double gamma, int layout, const double* qin,
                                     double* max_eig, unsigned* status, cudaStream_t st);
cudaError_t fvb_launch_selftest_div(const double* a, const double* b, double* out_shared, double* out_ieee,
                                    int64_t n, cudaStream_t st);
cudaError_t fvb_launch_probe(int dim, double gamma, const double* states, int64_t n, double* lam, double* flux,
                             double* pressure, uint8_t* bad, cudaStream_t st);
bool fvb_halo_tma_supported(int dim, int p);
cudaError_t fvb_launch_halo_tma(int dim, int p, int64_t n, const double* qout, double* qin, const int* grid,
                                int periodic, cudaStream_t st);
cudaError_t fvb_launch_halo_project_any_s(int dim, int p, int s, int64_t n, int layout, const double* qout,
                                          double* qin, const int* grid, int periodic, cudaStream_t st);
cudaError_t fvb_launch_halo_project(int dim, int p, int64_t n, int layout, const double* qout, double* qin,
                                    const int* grid, int periodic, cudaStream_t st);
cudaError_t fvb_launch_halo_project_totals(int dim, int p, int64_t n, int layout, const double* qout, double* qin,
                                           const int* grid, int periodic, double* scratch, double* totals,
                                           cudaStream_t st);
bool fvb_halo_window_supported(int dim, int p);
cudaError_t fvb_launch_halo_window(int dim, int p, int64_t n, const double* ghost_lo, const double* qout,
                                   const double* ghost_hi, double* qin, const int* window_grid, int nlo, int pmask,
                                   double* scratch, double* totals, cudaStream_t st);
cudaError_t fvb_launch_halo_shell2d(int p, int64_t n, double* q, const int* grid, int periodic, cudaStream_t st);
cudaError_t fvb_launch_totals_haloed(int dim, int p, int64_t n, const double* q, double* scratch, double* totals,
                                     cudaStream_t st);
cudaError_t fvb_launch_totals(int dim, int p, int64_t n, int layout, const double* qout, double* scratch,
                              double* totals, cudaStream_t st);
