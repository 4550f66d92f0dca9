// fvb_capi.cu -- the extern "C" boundary of libfvb200.so (declared in include/fvb200.h).
//
// Thin, allocation-free argument checking and dispatch on top of the kernel
// launchers, plus the host-buffer pipeline of fvb_update_host (chunked H2D ->
// update -> D2H overlapped across three streams).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/fvb200.h"
#include "fvb_kernels.h"
#include "fvb_layout.cuh"


namespace {

thread_local char g_last_error[256] = "";

int set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
  return FVB_ERR_CUDA;
}

int set_contract(const char* msg) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
  return FVB_ERR_CONTRACT;
}

int check_spec(const fvb_spec* s) {
  if (!s) return set_contract("null spec");
  if (s->dim != 2 && s->dim != 3) return set_contract("dimensions must be 2 or 3");
  if (s->p < 1) return set_contract("volumes_per_axis must be >= 1");
  if (s->unknowns != s->dim + 2) return set_contract("Euler needs dim + 2 unknowns");
  if (s->layout != 0 && s->layout != 1) return set_contract("layout must be 0 (AoS) or 1 (SoA)");
  if (s->n_patches < 0) return set_contract("negative patch count");
  if (!(s->gamma > 1.0)) return set_contract("gamma must exceed 1");
  return FVB_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int resolve_kernel(const fvb_spec* s, int kernel) {
  if (kernel == FVB_KERNEL_AUTO)
    return fvb_fused16_supported(s->dim, s->p, s->layout) ? FVB_KERNEL_FUSED : FVB_KERNEL_GENERIC;
  return kernel;
}

}  // namespace

extern "C" {

int fvb_version(void) { return 1; }

const char* fvb_strerror(int code) {
  if (code == FVB_OK) return "ok";
  if (g_last_error[0]) return g_last_error;
  switch (code) {
    case FVB_ERR_CONTRACT: return "contract violation";
    case FVB_ERR_NONPHYSICAL: return "non-physical state";
    case FVB_ERR_CUDA: return "CUDA error";
    default: return "unknown error";
  }
}

int fvb_select_kernel(const fvb_spec* spec) {
  int rc = check_spec(spec);
  if (rc) return -rc;
  return resolve_kernel(spec, FVB_KERNEL_AUTO);
}

}  // extern "C"

// ---- measurement hook: fvb_time_next_update ----
static thread_local cudaEvent_t t_ev_start = nullptr, t_ev_stop = nullptr;
void fvb_timing_mark_start(cudaStream_t st) {
  if (t_ev_start) cudaEventRecord(t_ev_start, st);
  t_ev_start = nullptr;
}
void fvb_timing_mark_stop(cudaStream_t st) {
  if (t_ev_stop) cudaEventRecord(t_ev_stop, st);
  t_ev_stop = nullptr;
}
// the hook is one-shot per update call: whatever the call did (or an early contract
// error), nothing stays armed for a later call
struct TimingHookScope {
  ~TimingHookScope() { t_ev_start = t_ev_stop = nullptr; }
};
extern "C" int fvb_step_record(int64_t* step, const double* dt_scalar, const uint32_t* status, const double* totals,
                               int unknowns, const double* gmax, double* dt_hist, int32_t* flag_hist,
                               double* totals_hist, double* gmax_hist, void* stream) {
  if (!step || !dt_scalar || !status || !totals || !gmax || !dt_hist || !flag_hist || !totals_hist || !gmax_hist ||
      unknowns < 1)
    return set_contract("step_record: null buffer or unknowns < 1");
  const cudaError_t e = fvb_launch_step_record(step, dt_scalar, status, totals, unknowns, gmax, dt_hist, flag_hist,
                                               totals_hist, gmax_hist, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_step_record");
}
extern "C" int fvb_time_next_update(void* start, void* stop) {
  t_ev_start = static_cast<cudaEvent_t>(start);
  t_ev_stop = static_cast<cudaEvent_t>(stop);
  return FVB_OK;
}

namespace {
// fvb_update / fvb_update_cfl.  With tail != nullptr (fvb_update_cfl) the step also reduces
// max_eig to *tail->gmax and optionally sets dt: inside the redo pass when the fused path
// runs one and the batch is small enough for one CTA, else with the reduce kernels.
int update_impl(const fvb_spec* spec, const double* qin, double* qout, const double* cell_size, double* dt,
                double* max_eig, uint32_t* status, int kernel, int zero_status, const FvbArgs* tail, void* stream) {
  const TimingHookScope hook_scope;
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->n_patches == 0) return FVB_OK;   // kernel/__init__.py:123-124
  if (!qin || !qout || !cell_size || !dt || !max_eig || !status) return set_contract("null buffer");
  const bool fast = (kernel & FVB_MODE_FAST) != 0;
  kernel &= ~FVB_MODE_FAST;
  const int k = resolve_kernel(spec, kernel);
  if (k == FVB_KERNEL_FUSED && !fvb_fused16_supported(spec->dim, spec->p, spec->layout))
    return set_contract("no fused kernel for this shape (2D/3D p=16, 3D even p=2..8 AoS, 2D p=2..32 AoS)");
  if (k != FVB_KERNEL_FUSED && k != FVB_KERNEL_GENERIC) return set_contract("unknown kernel selector");
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  if (zero_status) {
    e = cudaMemsetAsync(status, 0, 2 * sizeof(uint32_t), st);   // flag + redo count
    if (e != cudaSuccess) return set_cuda_error(e, "memset status");
  }
  FvbArgs a;
  a.dim = spec->dim;
  a.p = spec->p;
  a.layout = spec->layout;
  a.n = spec->n_patches;
  a.gamma = spec->gamma;
  a.qin = qin;
  a.qout = qout;
  a.cell_size = cell_size;
  a.dt = dt;
  a.max_eig = max_eig;
  a.status = status;
  const bool tail_in_redo = tail && k == FVB_KERNEL_FUSED;   // every fused kernel carries the CFL tail
  if (tail_in_redo) {
    a.gmax = tail->gmax;
    a.cfl = tail->cfl;
    a.dx = tail->dx;
    a.dt_scalar = tail->dt_scalar;
    a.dt_patches = tail->tail_dt ? dt : nullptr;
    a.tail_dt = tail->tail_dt;
  }
  fvb_timing_mark_start(st);   // (measurement hook: the main kernel starts here)
  if (k == FVB_KERNEL_GENERIC) {
    // per-patch maxima are combined with atomicMax on the bit patterns
    e = cudaMemsetAsync(max_eig, 0, sizeof(double) * (size_t)spec->n_patches, st);
    if (e != cudaSuccess) return set_cuda_error(e, "memset max_eig");
    e = fvb_launch_generic(a, st);
  } else if (fast && fvb_fast3d_supported(spec->dim, spec->p, spec->layout)) {
    e = fvb_launch_fast3d16(a, st);
    if (e == cudaSuccess) e = fvb_launch_redo(a, st);   // exact re-evaluation of queued patches
  } else if (fast && fvb_fast_small3d_supported(spec->dim, spec->p, spec->layout)) {
    e = fvb_launch_fast_small3d(a, st);
  } else if (fast && fvb_fast2d_supported(spec->dim, spec->p, spec->layout)) {
    e = fvb_launch_fast2d16(a, st);
    if (e == cudaSuccess) e = fvb_launch_redo(a, st);
  } else {
    e = fvb_launch_fused16(a, st);
  }
  fvb_timing_mark_stop(st);   // no redo pass (generic kernel): the stop mark is still pending
  if (e == cudaSuccess && tail && !tail_in_redo)
    e = fvb_launch_reduce_dt(max_eig, spec->n_patches, tail->cfl, tail->dx, tail->gmax, tail->dt_scalar,
                             tail->tail_dt ? dt : nullptr, tail->tail_dt, st);
  if (e != cudaSuccess) return set_cuda_error(e, "fvb_update launch");
  return FVB_OK;
}
}  // namespace

extern "C" {

int fvb_update(const fvb_spec* spec, const double* qin, double* qout, const double* cell_size, const double* dt,
               double* max_eig, uint32_t* status, int kernel, int zero_status, void* stream) {
  return update_impl(spec, qin, qout, cell_size, const_cast<double*>(dt), max_eig, status, kernel, zero_status,
                     nullptr, stream);
}

int fvb_update_cfl(const fvb_spec* spec, const double* qin, double* qout, const double* cell_size, double* dt,
                   double* max_eig, uint32_t* status, int kernel, double cfl, double dx, double* gmax,
                   double* dt_scalar, int set_dt, void* stream) {
  if (!gmax) return set_contract("null gmax");
  FvbArgs tail;
  tail.gmax = gmax;
  tail.cfl = cfl;
  tail.dx = dx;
  tail.dt_scalar = set_dt ? dt_scalar : nullptr;
  tail.tail_dt = set_dt ? 1 : 0;
  return update_impl(spec, qin, qout, cell_size, dt, max_eig, status, kernel, 0, &tail, stream);
}

static size_t status_bytes(int64_t chunk) { return ((size_t)(2 * chunk + 8) * 4 + 255) / 256 * 256; }
static size_t align256(size_t b) { return (b + 255) / 256 * 256; }
// One buffer set of the host pipeline: qin, qout, cell_size, dt, max_eig, each
// 256-byte aligned (the fused kernels move patches with TMA bulk copies, which
// need 16-byte aligned global addresses whatever the chunk length).
static size_t host_set_bytes(const fvb_spec* spec, int64_t chunk) {
  const fvb::Geom g = fvb::make_geom(spec->dim, spec->p, chunk);
  return align256((size_t)chunk * g.V * g.s * 8) + align256((size_t)chunk * g.I * g.s * 8) +
         align256((size_t)chunk * spec->dim * 8) + 2 * align256((size_t)chunk * 8);
}

size_t fvb_status_words(int64_t n_patches) { return (size_t)(2 * n_patches + 8); }

size_t fvb_update_host_workspace(const fvb_spec* spec, int64_t chunk) {
  if (check_spec(spec) || chunk < 1) return 0;
  return 2 * host_set_bytes(spec, chunk) + 2 * status_bytes(chunk);
}

int fvb_update_host(const fvb_spec* spec, const double* qin_h, double* qout_h, const double* cell_size_h,
                    const double* dt_h, double* max_eig_h, void* workspace, size_t workspace_bytes,
                    int64_t chunk, int kernel, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->layout != 0) return set_contract("host buffers are AoS (PatchBatch layout)");
  const int64_t n = spec->n_patches;
  if (n == 0) return FVB_OK;
  if (chunk < 1 || chunk > n) chunk = n;
  if (workspace_bytes < fvb_update_host_workspace(spec, chunk)) return set_contract("workspace too small");
  const fvb::Geom g = fvb::make_geom(spec->dim, spec->p, chunk);
  const int d = spec->dim, s = g.s;
  // carve the two buffer sets
  char* base = static_cast<char*>(workspace);
  // two status buffers (flag, redo count, redo list), one per buffer set
  uint32_t* status_b[2] = {reinterpret_cast<uint32_t*>(base),
                           reinterpret_cast<uint32_t*>(base + status_bytes(chunk))};
  char* bufs = base + 2 * status_bytes(chunk);
  const size_t per = host_set_bytes(spec, chunk);
  double *qin_d[2], *qout_d[2], *cs_d[2], *dt_d[2], *me_d[2];
  for (int b = 0; b < 2; ++b) {
    char* p = bufs + b * per;
    qin_d[b] = reinterpret_cast<double*>(p); p += align256((size_t)chunk * g.V * s * 8);
    qout_d[b] = reinterpret_cast<double*>(p); p += align256((size_t)chunk * g.I * s * 8);
    cs_d[b] = reinterpret_cast<double*>(p); p += align256((size_t)chunk * d * 8);
    dt_d[b] = reinterpret_cast<double*>(p); p += align256((size_t)chunk * 8);
    me_d[b] = reinterpret_cast<double*>(p);
  }
  cudaStream_t comp = as_stream(stream);
  // copy streams and events: created once per thread and device, reused by every call
  // (creating them per call cost ~0.1 ms, most of a small batch's latency)
  struct Pipe {
    int dev = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr;
    uint32_t* flags = nullptr;   // pinned readback of the two status flags
  };
  static thread_local Pipe pipes[8];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
  Pipe& pp = pipes[dev & 7];
  if (pp.dev != dev) {
    pp = Pipe();
    e = cudaStreamCreateWithFlags(&pp.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.d2h, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      e = cudaEventCreateWithFlags(&pp.ev_in[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_k[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_out[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_start, cudaEventDisableTiming);
    if (e != cudaSuccess) return set_cuda_error(e, "fvb_update_host streams");
    pp.dev = dev;
  }
  cudaStream_t h2d = pp.h2d, d2h = pp.d2h;
  cudaEvent_t* ev_in = pp.ev_in;
  cudaEvent_t* ev_k = pp.ev_k;
  cudaEvent_t* ev_out = pp.ev_out;
  // flag words of both status buffers accumulate over the chunks; redo counts are reset per chunk
  // both status buffers whole (flag, list, the redo kernel's CTA counter): the workspace
  // is caller memory of unknown content
  if (e == cudaSuccess) e = cudaMemsetAsync(status_b[0], 0, 2 * status_bytes(chunk), comp);
  // the copy streams must not run ahead of the status reset / earlier work on `comp`
  cudaEvent_t ev_start = pp.ev_start;
  if (e == cudaSuccess) e = cudaEventRecord(ev_start, comp);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h2d, ev_start, 0);
  int nch = (int)((n + chunk - 1) / chunk);
  int krc = FVB_OK;
  for (int c = 0; c < nch && e == cudaSuccess && krc == FVB_OK; ++c) {
    const int b = c & 1;
    const int64_t p0 = (int64_t)c * chunk;
    const int64_t np = (p0 + chunk <= n) ? chunk : n - p0;
    if (c >= 2) e = cudaStreamWaitEvent(h2d, ev_out[b], 0);   // buffer set b drained
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(qin_d[b], qin_h + p0 * g.V * s, (size_t)np * g.V * s * 8, cudaMemcpyHostToDevice, h2d);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(cs_d[b], cell_size_h + p0 * d, (size_t)np * d * 8, cudaMemcpyHostToDevice, h2d);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dt_d[b], dt_h + p0, (size_t)np * 8, cudaMemcpyHostToDevice, h2d);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[b], h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, ev_in[b], 0);
    if (e != cudaSuccess) break;
    fvb_spec sub = *spec;
    sub.n_patches = np;
    krc = fvb_update(&sub, qin_d[b], qout_d[b], cs_d[b], dt_d[b], me_d[b], status_b[b], kernel, 0, stream);
    if (krc != FVB_OK) break;
    e = cudaEventRecord(ev_k[b], comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, ev_k[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(qout_h + p0 * g.I * s, qout_d[b], (size_t)np * g.I * s * 8, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess) e = cudaMemcpyAsync(max_eig_h + p0, me_d[b], (size_t)np * 8, cudaMemcpyDeviceToHost, d2h);
    if (e == cudaSuccess) e = cudaEventRecord(ev_out[b], d2h);
  }
  // the two flag words come back with the last D2H (pinned, per thread) instead of two
  // synchronous copies after the drain
  if (!pp.flags && e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&pp.flags), 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, ev_k[(nch - 1) & 1], 0);   // every kernel done (comp order)
  if (e == cudaSuccess) e = cudaMemcpyAsync(&pp.flags[0], status_b[0], 4, cudaMemcpyDeviceToHost, d2h);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&pp.flags[1], status_b[1], 4, cudaMemcpyDeviceToHost, d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(comp);
  uint32_t st_h[2] = {0, 0};
  if (e == cudaSuccess) {
    st_h[0] = pp.flags[0];
    st_h[1] = pp.flags[1];
  }
  if (krc != FVB_OK) {   // an aborted pipeline may leave copies queued: drain before the buffers are reused
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(d2h);
    return krc;
  }
  if (e != cudaSuccess) return set_cuda_error(e, "fvb_update_host");
  return (st_h[0] | st_h[1]) ? FVB_ERR_NONPHYSICAL : FVB_OK;
}

int fvb_update_to_haloed(const fvb_spec* spec, const double* qin, double* qin_next, const double* cell_size,
                         const double* dt, double* max_eig, uint32_t* status, int flags, void* stream) {
  const TimingHookScope hook_scope;
  const int zero_status = flags & 1;
  const bool fast = (flags & FVB_MODE_FAST) != 0;
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->n_patches == 0) return FVB_OK;
  if (spec->dim != 2 || spec->layout != 0 || !fvb_fused2d_warp_supported(spec->p))
    return set_contract("update_to_haloed: 2D AoS batches with 2 <= p <= 32");
  if (!qin || !qin_next || !cell_size || !dt || !max_eig || !status || qin == qin_next)
    return set_contract("update_to_haloed: null or aliased buffer");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaSuccess;
  if (zero_status) e = cudaMemsetAsync(status, 0, 2 * sizeof(uint32_t), st);
  if (e != cudaSuccess) return set_cuda_error(e, "memset status");
  FvbArgs a;
  a.dim = 2;
  a.p = spec->p;
  a.layout = 0;
  a.n = spec->n_patches;
  a.gamma = spec->gamma;
  a.qin = qin;
  a.qout = qin_next;
  a.cell_size = cell_size;
  a.dt = dt;
  a.max_eig = max_eig;
  a.status = status;
  a.out_haloed = 1;
  fvb_timing_mark_start(st);
  e = fast && fvb_fast2d_supported(2, spec->p, 0) ? fvb_launch_fast2d16(a, st) : fvb_launch_fused2d16_warp(a, st);
  if (e == cudaSuccess) e = fvb_launch_redo(a, st);
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_update_to_haloed");
}

int fvb_halo_shell(const fvb_spec* spec, double* qin, const int32_t* grid_shape, int periodic, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->dim != 2 || spec->layout != 0) return set_contract("halo_shell: 2D AoS batches");
  if (!grid_shape || grid_shape[0] < 1 || grid_shape[1] < 1 ||
      (int64_t)grid_shape[0] * grid_shape[1] != spec->n_patches)
    return set_contract("grid shape does not match the patch count");
  if (spec->n_patches == 0) return FVB_OK;
  const int g[2] = {grid_shape[0], grid_shape[1]};
  cudaError_t e = fvb_launch_halo_shell2d(spec->p, spec->n_patches, qin, g, periodic, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_halo_shell");
}

int fvb_totals_haloed(const fvb_spec* spec, const double* qin, double* scratch, double* totals, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->layout != 0) return set_contract("totals_haloed: AoS batches");
  if (spec->n_patches == 0) return set_contract("totals over an empty batch");
  cudaError_t e = fvb_launch_totals_haloed(spec->dim, spec->p, spec->n_patches, qin, scratch, totals,
                                           as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_totals_haloed");
}

int fvb_host_pin(const void* p, size_t bytes) {
  if (!p || bytes == 0) return set_contract("null host range");
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost) return 1;   // already
  cudaGetLastError();
  const cudaError_t e = cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();   // leave no stale error for the next launch check
    return set_cuda_error(e, "cudaHostRegister");
  }
  return FVB_OK;
}

int fvb_host_unpin(const void* p) {
  const cudaError_t e = cudaHostUnregister(const_cast<void*>(p));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_cuda_error(e, "cudaHostUnregister");
  }
  return FVB_OK;
}

int fvb_locate(const fvb_spec* spec, const double* qin, fvb_boxinfo* info, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->n_patches == 0) return FVB_OK;
  static_assert(sizeof(fvb_boxinfo) == sizeof(BoxInfo), "boxinfo layout");
  cudaError_t e = fvb_launch_locate(spec->dim, spec->p, spec->n_patches, spec->gamma, spec->layout, qin,
                                    reinterpret_cast<BoxInfo*>(info), as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_locate");
}

int fvb_pack(const fvb_spec* spec, const double* aos, double* soa, int interior, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  const fvb::Geom g = fvb::make_geom(spec->dim, spec->p, spec->n_patches);
  if (g.n == 0) return FVB_OK;
  cudaError_t e = fvb_launch_pack(aos, soa, g.n, interior ? g.I : g.V, g.s, 1, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_pack");
}

int fvb_unpack(const fvb_spec* spec, const double* soa, double* aos, int interior, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  const fvb::Geom g = fvb::make_geom(spec->dim, spec->p, spec->n_patches);
  if (g.n == 0) return FVB_OK;
  cudaError_t e = fvb_launch_pack(soa, aos, g.n, interior ? g.I : g.V, g.s, 0, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_unpack");
}

int fvb_reduce_dt(const double* max_eig, int64_t n, double cfl, double dx, double* gmax, double* dt_scalar,
                  double* dt_patches, int do_dt, void* stream) {
  if (n < 1 || !max_eig || !gmax) return set_contract("reduce over an empty batch");
  cudaError_t e = fvb_launch_reduce_dt(max_eig, n, cfl, dx, gmax, dt_scalar, dt_patches, do_dt, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_reduce_dt");
}

int fvb_set_dt(const double* gmax, double cfl, double dx, double* dt_scalar, double* dt_patches, int64_t n,
               void* stream) {
  if (!gmax) return set_contract("null gmax");
  cudaError_t e = fvb_launch_set_dt(gmax, cfl, dx, dt_scalar, dt_patches, n, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_set_dt");
}

int fvb_patch_max_eig(const fvb_spec* spec, const double* qin, double* max_eig, uint32_t* status, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->n_patches == 0) return FVB_OK;
  cudaError_t e = fvb_launch_patch_max_eig(spec->dim, spec->p, spec->n_patches, spec->gamma, spec->layout, qin,
                                           max_eig, status, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_patch_max_eig");
}

int fvb_probe(int dim, double gamma, const double* states, int64_t n, double* lam, double* flux,
              double* pressure, uint8_t* bad, void* stream) {
  if (dim != 2 && dim != 3) return set_contract("dimensions must be 2 or 3");
  if (n == 0) return FVB_OK;
  cudaError_t e = fvb_launch_probe(dim, gamma, states, n, lam, flux, pressure, bad, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_probe");
}

int fvb_selftest_div(const double* a, const double* b, double* out_shared, double* out_ieee, int64_t n,
                     void* stream) {
  if (n == 0) return FVB_OK;
  cudaError_t e = fvb_launch_selftest_div(a, b, out_shared, out_ieee, n, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_selftest_div");
}

int fvb_halo_project(const fvb_spec* spec, const double* qout, double* qin, const int32_t* grid_shape,
                     int periodic, void* stream) {
  // Pure data movement: any unknown count s >= 1 (the reference's halo_project
  // works for every PatchSpec); only the Euler shape s = d + 2 has the fast kernels.
  if (spec && spec->unknowns >= 1 && spec->unknowns != spec->dim + 2) {
    fvb_spec euler = *spec;
    euler.unknowns = spec->dim + 2;
    int rc0 = check_spec(&euler);
    if (rc0) return rc0;
  } else {
    int rc = check_spec(spec);
    if (rc) return rc;
  }
  if (!grid_shape) return set_contract("null grid shape");
  int64_t cells = 1;
  for (int a = 0; a < spec->dim; ++a) {
    if (grid_shape[a] < 1) return set_contract("grid extents must be >= 1");
    cells *= grid_shape[a];
  }
  if (cells != spec->n_patches) return set_contract("grid shape does not match the patch count");
  if (spec->n_patches == 0) return FVB_OK;
  cudaError_t e = spec->unknowns == spec->dim + 2
                      ? fvb_launch_halo_project(spec->dim, spec->p, spec->n_patches, spec->layout, qout, qin,
                                                grid_shape, periodic, as_stream(stream))
                      : fvb_launch_halo_project_any_s(spec->dim, spec->p, spec->unknowns, spec->n_patches,
                                                      spec->layout, qout, qin, grid_shape, periodic,
                                                      as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_halo_project");
}

int fvb_halo_project_totals(const fvb_spec* spec, const double* qout, double* qin, const int32_t* grid_shape,
                            int periodic, double* scratch, double* totals, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (!grid_shape) return set_contract("null grid shape");
  int64_t cells = 1;
  for (int a = 0; a < spec->dim; ++a) {
    if (grid_shape[a] < 1) return set_contract("grid extents must be >= 1");
    cells *= grid_shape[a];
  }
  if (cells != spec->n_patches) return set_contract("grid shape does not match the patch count");
  if (spec->n_patches == 0) return set_contract("totals over an empty batch");
  cudaError_t e = fvb_launch_halo_project_totals(spec->dim, spec->p, spec->n_patches, spec->layout, qout, qin,
                                                 grid_shape, periodic, scratch, totals, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_halo_project_totals");
}

int fvb_halo_project_window(const fvb_spec* spec, const double* ghost_lo, const double* qout,
                            const double* ghost_hi, double* qin, const int32_t* window_grid, int32_t lo_layers,
                            int periodic_mask, double* scratch, double* totals, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (!window_grid) return set_contract("null window grid");
  if (spec->layout != 0) return set_contract("halo window: AoS batches only");
  if (!fvb_halo_window_supported(spec->dim, spec->p)) return set_contract("halo window: patch size must be 2..32");
  int64_t cells = 1, layer = 1;
  for (int a = 0; a < spec->dim; ++a) {
    if (window_grid[a] < 1) return set_contract("grid extents must be >= 1");
    cells *= window_grid[a];
    if (a < spec->dim - 1) layer *= window_grid[a];
  }
  if (lo_layers < 0 || spec->n_patches % layer != 0 || lo_layers * layer + spec->n_patches > cells)
    return set_contract("own patches must be whole layers of the window");
  if ((lo_layers > 0 && !ghost_lo) || (lo_layers * layer + spec->n_patches < cells && !ghost_hi))
    return set_contract("missing ghost layer buffer");
  if ((int64_t)window_grid[0] * (int64_t)spec->p * spec->p * (spec->dim == 3 ? spec->p : 1) * spec->unknowns >=
      (1ll << 31))
    return set_contract("halo window: x extent too large");
  if (totals && !scratch) return set_contract("totals need the scratch buffer");
  if (spec->n_patches == 0) return FVB_OK;
  int g[3] = {window_grid[0], window_grid[1], spec->dim == 3 ? window_grid[2] : 1};
  cudaError_t e = fvb_launch_halo_window(spec->dim, spec->p, spec->n_patches, ghost_lo, qout, ghost_hi, qin, g,
                                         lo_layers, periodic_mask & 7, scratch, totals, as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_halo_project_window");
}

size_t fvb_totals_scratch_bytes(const fvb_spec* spec) {
  if (check_spec(spec)) return 0;
  return (size_t)kScratchBlocks * spec->unknowns * sizeof(double);
}

int fvb_totals(const fvb_spec* spec, const double* qout, double* scratch, double* totals, void* stream) {
  int rc = check_spec(spec);
  if (rc) return rc;
  if (spec->n_patches == 0) return set_contract("totals over an empty batch");
  cudaError_t e = fvb_launch_totals(spec->dim, spec->p, spec->n_patches, spec->layout, qout, scratch, totals,
                                    as_stream(stream));
  return e == cudaSuccess ? FVB_OK : set_cuda_error(e, "fvb_totals");
}

}  // extern "C"
