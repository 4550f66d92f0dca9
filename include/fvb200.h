/*
 * fvb200.h -- C ABI of libfvb200.so, the B200 (sm_100a) batched Rusanov
 * finite-volume patch update.
 *
 * Drop-in boundary for the reference package `fvbatch` (arXiv 2302.09005
 * clean-room re-implementation, /root/reference/pkg).  Each entry point names
 * the reference interface it replaces.  Plain C types only: device pointers
 * are raw `double*` / `uint32_t*`, streams are `cudaStream_t` passed as
 * `void*` (NULL = legacy default stream).  The library allocates no device
 * memory per call; callers own every buffer.
 *
 * Array layouts (mesh.py:6-7, :119-134):
 *   AoS (layout 0): qin[(patch*V + vol)*S + u], qout[(patch*I + vol)*S + u]
 *   SoA (layout 1): qin[(u*N + patch)*V + vol], qout[(u*N + patch)*I + vol]
 *   V = (p+2)^d haloed volumes, I = p^d interior volumes, S = d+2 unknowns,
 *   volumes linearised x fastest, [z][y][x].
 *
 * Return codes map to the reference's exceptions (errors.py):
 *   FVB_OK 0, FVB_ERR_CONTRACT 1 -> ContractViolationError,
 *   FVB_ERR_NONPHYSICAL 2 -> NonPhysicalStateError (locate with fvb_locate),
 *   FVB_ERR_CUDA 3 -> device failure (fvb_strerror / cudaGetLastError text).
 */
#ifndef FVB200_H
#define FVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVB_OK 0
#define FVB_ERR_CONTRACT 1
#define FVB_ERR_NONPHYSICAL 2
#define FVB_ERR_CUDA 3
#define FVB_ERR_IO 4          /* file open / read / write failure (FVB1 I/O) */

/* kernel selector for fvb_update / fvb_update_host */
#define FVB_KERNEL_AUTO 0     /* the shape's fused kernel when it has one, else generic */
#define FVB_KERNEL_GENERIC 1  /* any d, p */
#define FVB_KERNEL_FUSED 2    /* 2D/3D p == 16 (AoS or SoA), 3D p == 2, 4..8 (AoS), 2D p == 2..32 (AoS) */
/* OR'ed into the kernel selector: "fast" mode (AoS: 3D p = 16, 3D p = 2, 4..8, 2D p = 2..32).  QOut and
 * max_eig within 1e-12 relative per unknown of the reference (the north star's
 * parity bar; measured ~1e-16 / a few ulp).  Shapes without a fast kernel run the
 * exact one (trivially within the bar).  Without the flag every result is
 * bit-exact. */
#define FVB_MODE_FAST 0x100

typedef struct fvb_spec {
  int32_t dim;       /* PatchSpec.dimensions (mesh.py:29), 2 or 3 */
  int32_t p;         /* PatchSpec.volumes_per_axis (mesh.py:30) */
  int32_t unknowns;  /* PatchSpec.unknowns; must be dim + 2 (Euler, pde.py:121) */
  int32_t layout;    /* 0 = AoS (PatchBatch), 1 = SoA (LayoutEnumerator SOA) */
  int64_t n_patches; /* PatchBatch.n_patches */
  double gamma;      /* EulerParameters.gamma (pde.py:19-30) */
} fvb_spec;

/* Per-(patch, box) diagnostics of the face-box volumes (see fvb_locate). */
typedef struct fvb_boxinfo {
  int64_t trig_rho;     /* any rho <= 0           (pde.py:36-38) */
  int64_t trig_p;       /* any p < 0              (pde.py:66-68) */
  int64_t first_nonpos; /* first box index with !(rho > 0), -1 if none   (vectorized.py:86) */
  int64_t first_badpl;  /* first box index with !(E - |j|^2/(2 rho) >= 0), -1 if none (vectorized.py:88-90) */
} fvb_boxinfo;

int fvb_version(void);
const char* fvb_strerror(int code);

/* Which kernel FVB_KERNEL_AUTO resolves to for this spec (1 generic, 2 fused). */
int fvb_select_kernel(const fvb_spec* spec);

/* One forward-Euler Rusanov step for every patch, device-resident.
 * Replaces fvbatch.kernel.update_patch_batch (kernel/__init__.py:114-140) and
 * the engine it dispatches to (vectorized.run, vectorized.py:246-288).
 *   qin        [N*V*S]  haloed input, read only
 *   qout       [N*I*S]  interior output (written)
 *   cell_size  [N*dim]  only cell_size[patch*dim + 0] is read (vectorized.py:169)
 *   dt         [N]      per-patch time step, must be >= 0 (checked by the host)
 *   max_eig    [N]      per-patch max directional wave speed (written, vectorized.py:226-231)
 *   status     [2N+8]   device words (fvb_status_words), zero-initialised once by the caller:
 *                       status[0] is ORed with 1 when a face-box volume has rho <= 0 or
 *                       p < 0 (sticky: clear it with zero_status = 1 or a memset);
 *                       status[1] / status[2..2N+1] are the redo list the fused kernels use
 *                       for patches whose quotients need CUDA's division slow path
 *                       (re-evaluated exactly before returning); status[2N+2 .. 2N+7] are
 *                       CTA counters and the CFL tail's running max (csrc/fvb_tail.cuh).  The
 *                       kernels leave all of them at zero, so a step loop needs no memset
 *                       (zero_status = 0).
 * Asynchronous on `stream`.  Returns FVB_OK or FVB_ERR_CONTRACT / FVB_ERR_CUDA. */
int fvb_update(const fvb_spec* spec, const double* qin, double* qout, const double* cell_size,
               const double* dt, double* max_eig, uint32_t* status, int kernel, int zero_status,
               void* stream);

/* fvb_update (zero_status = 0) followed by the CFL step control of the multi-step
 * driver (no reference code): *gmax = max over the batch's max_eig
 * (NaN wins, as numpy's max), and with set_dt, dt = (cfl*dx)/gmax into *dt_scalar and
 * every dt[patch].  On the fused paths the reduction rides on the update itself (each CTA
 * folds its patches' max_eig into a running max, the last one writes gmax and dt_scalar)
 * and the redo pass broadcasts dt, so a step is two launches and no memset; the generic
 * kernel is followed by the reduce kernels.  Asynchronous on `stream`. */
int fvb_update_cfl(const fvb_spec* spec, const double* qin, double* qout, const double* cell_size,
                   double* dt, double* max_eig, uint32_t* status, int kernel, double cfl, double dx,
                   double* gmax, double* dt_scalar, int set_dt, void* stream);

/* run_simulation's per-step history record, one single-thread launch on `stream`: with
 * k = *step (a device int64), flag_hist[k] = status[0] (the sticky non-physical flag),
 * dt_hist[k+1] = *dt_scalar (the next step's dt), gmax_hist[k+1] = *gmax,
 * totals_hist[(k+1)*unknowns + u] = totals[u], then *step = k + 1.  All device pointers. */
int fvb_step_record(int64_t* step, const double* dt_scalar, const uint32_t* status, const double* totals,
                    int unknowns, const double* gmax, double* dt_hist, int32_t* flag_hist, double* totals_hist,
                    double* gmax_hist, void* stream);

/* Measurement hook (bench.py's per-launch roofline timing): the NEXT fvb_update /
 * fvb_update_cfl / fvb_update_to_haloed call made by this host thread records the CUDA
 * event `start` (a cudaEvent_t) on its stream right before its main kernel and `stop`
 * right after it -- the exact redo pass and the reduce kernels excluded (the CFL tail
 * that runs at the end of the main kernel is included).  One-shot;
 * either pointer may be NULL. */
int fvb_time_next_update(void* start, void* stop);

/* Number of uint32 status words fvb_update needs for n patches (2n + 8: flag,
 * redo count, redo list -- sized 2n for kernels that may queue a patch twice --
 * two CTA counters, two spare words and the CFL tail's 64-bit running max). */
size_t fvb_status_words(int64_t n_patches);

/* Same step from HOST arrays (the reference's calling convention, numpy
 * buffers): chunked, double-buffered H2D copy -> update -> D2H copy, with
 * copies and kernels overlapped on the given stream plus one internal copy
 * stream per direction.  `workspace` is device memory of at least
 * fvb_update_host_workspace(spec, chunk_patches) bytes.  Synchronous; returns
 * FVB_ERR_NONPHYSICAL when the status word was raised (then call fvb_locate). */
size_t fvb_update_host_workspace(const fvb_spec* spec, int64_t chunk_patches);
int fvb_update_host(const fvb_spec* spec, const double* qin_host, double* qout_host,
                    const double* cell_size_host, const double* dt_host, double* max_eig_host,
                    void* workspace, size_t workspace_bytes, int64_t chunk_patches, int kernel,
                    void* stream);

/* Error path: per-(patch, box) diagnostics for the 2*dim+1 boxes of
 * vectorized._plan (vectorized.py:42-53), box-linear index in C order over the
 * box's (z, y, x) extents.  info has N*(2*dim+1) entries (device). */
int fvb_locate(const fvb_spec* spec, const double* qin, fvb_boxinfo* info, void* stream);

/* AoS <-> SoA batch packer (LayoutEnumerator AOS/SOA maps, mesh.py:127-130).
 * interior = 0 packs haloed QIn-shaped arrays, 1 interior QOut-shaped arrays. */
int fvb_pack(const fvb_spec* spec, const double* aos, double* soa, int interior, void* stream);
int fvb_unpack(const fvb_spec* spec, const double* soa, double* aos, int interior, void* stream);

/* Global wave speed and CFL step: gmax = max over patches
 * of max_eig (NaN propagates), then dt = (cfl*dx)/gmax written to dt_scalar
 * and broadcast to dt_patches[N] (either may be NULL).  For multi-GPU runs
 * call with do_dt = 0, all-reduce gmax (MAX) across ranks, then fvb_set_dt. */
int fvb_reduce_dt(const double* max_eig, int64_t n, double cfl, double dx, double* gmax,
                  double* dt_scalar, double* dt_patches, int do_dt, void* stream);
int fvb_set_dt(const double* gmax, double cfl, double dx, double* dt_scalar, double* dt_patches,
               int64_t n, void* stream);

/* First-step wave-speed pre-pass: per-patch max over interior
 * volumes and directions of |u_n| + c, no update. max_eig must be zeroed. */
int fvb_patch_max_eig(const fvb_spec* spec, const double* qin, double* max_eig, uint32_t* status,
                      void* stream);

/* Closure probe: wave speeds lam[i*dim + k], fluxes flux[(i*dim + k)*S + u],
 * pressure[i] and bad[i] (0 ok, 1 rho <= 0, 2 p < 0) of n AoS states -- the
 * device twin of the Euler callbacks (euler_pressure / euler_flux /
 * euler_max_eigenvalue, pde.py:33-70, bound by make_euler_pde, :115-119).
 * pressure and bad may be NULL. */
int fvb_probe(int dim, double gamma, const double* states, int64_t n, double* lam, double* flux,
              double* pressure, uint8_t* bad, void* stream);

/* Between steps: rebuild QIn (haloed) from QOut (interior) over a logical
 * uniform patch grid, grid_shape[0..dim) = patch counts along x, y[, z]
 * (patch index x-fastest), periodic wrap or zero-gradient edge.  Replaces
 * mesh.halo_project (mesh.py:261-310) bit for bit, corners included. */
int fvb_halo_project(const fvb_spec* spec, const double* qout, double* qin, const int32_t* grid_shape,
                     int periodic, void* stream);

/* Conserved totals: totals[u] = sum over all interior volumes of unknown u
 * (deterministic order) -- the per-step diagnostics of run_simulation
 * (SPEC.md:446-455, :473).  scratch: fvb_totals_scratch_bytes(spec) bytes. */
size_t fvb_totals_scratch_bytes(const fvb_spec* spec);
int fvb_totals(const fvb_spec* spec, const double* qout, double* scratch, double* totals, void* stream);

/* fvb_halo_project followed by fvb_totals of the same QOut, in one pass over
 * QOut where the batch shape allows (3D AoS, p <= 32 listed in
 * fvb_generic.cu: the row-copy kernel sums the interior runs it moves);
 * otherwise the two calls back to back.  The per-step loop of run_simulation
 * (SPEC.md:446-455, :473).  The totals' summation order is deterministic for a
 * given device but differs from fvb_totals' (both are fixed-order fp64 sums). */
int fvb_halo_project_totals(const fvb_spec* spec, const double* qout, double* qin, const int32_t* grid_shape,
                            int periodic, double* scratch, double* totals, void* stream);

/* Halo projection of one shard of a sharded grid (multi-GPU run_simulation).
 * The shard owns whole layers of the patch grid along its slowest axis (z in
 * 3D, y in 2D); its window is [lo_layers ghost layers from the lower
 * neighbour | its own layers | the ghost layers from the upper neighbour],
 * window_grid[0..dim) the window's patch counts.  qout (the shard's own QOut,
 * spec->n_patches patches) and the ghost buffers ghost_lo / ghost_hi (interior
 * QOut of the ghost patches, NULL when that side has none) are read; the own
 * patches' QIn is written.  periodic_mask: bit a = wrap along axis a (x = 0);
 * along the slowest axis a window without a ghost layer on a side clamps
 * (zero-gradient), so a shard sets that bit only when it is the whole periodic
 * grid.  If totals is not NULL it receives the shard's conserved totals (as
 * fvb_halo_project_totals).  AoS, 2 <= p <= 32.  Bit-exact with
 * fvb_halo_project of the whole grid (row f1 / §8(e)). */
int fvb_halo_project_window(const fvb_spec* spec, const double* ghost_lo, const double* qout,
                            const double* ghost_hi, double* qin, const int32_t* window_grid, int32_t lo_layers,
                            int periodic_mask, double* scratch, double* totals, void* stream);

/* 2D multi-step fast path (run_simulation): the update writes the new state straight
 * into the interior of the next step's haloed batch qin_next (the warp kernel's TMA
 * store addresses a haloed row at a 32-byte offset), fvb_halo_shell then fills only
 * that batch's halo shell from the neighbours' interiors (21 % of the bytes of a full
 * halo projection), and fvb_totals_haloed sums the interiors for the step's totals.
 * Bit-identical to fvb_update + fvb_halo_project.  2D AoS, 2 <= p <= 32. */
/* flags: bit 0 = zero the status words first; FVB_MODE_FAST = fast mode (2D p = 16, as fvb_update). */
int fvb_update_to_haloed(const fvb_spec* spec, const double* qin, double* qin_next, const double* cell_size,
                         const double* dt, double* max_eig, uint32_t* status, int flags, void* stream);
int fvb_halo_shell(const fvb_spec* spec, double* qin, const int32_t* grid_shape, int periodic, void* stream);
int fvb_totals_haloed(const fvb_spec* spec, const double* qin, double* scratch, double* totals, void* stream);

/* Page-lock a caller's host range for the H2D / D2H of fvb_update_host (pageable
 * copies are driver-staged and synchronous: ~6.7x slower for C3).  Returns FVB_OK when
 * registered, 1 when the range is already page-locked (nothing to undo), FVB_ERR_CUDA
 * when it cannot be (the call then still works on pageable memory).  fvb_host_unpin
 * releases a range fvb_host_pin registered. */
int fvb_host_pin(const void* p, size_t bytes);
int fvb_host_unpin(const void* p);

/* Multi-GPU: the step's single exchange, a MAX all-reduce of the global wave
 * speed (one fp64) over NCCL on NVLink / NVSwitch (the
 * ncclAllReduce of the north star), for hosts that do not use torch.distributed.
 * NCCL is dlopen'ed ("libnccl.so.2") on first use.
 *   One process, ndev GPUs:   fvb_mgpu_init(ndev, devs) (ncclCommInitAll), then per
 *     step fvb_mgpu_allreduce_max_all(bufs, streams) (one NCCL group over all
 *     ranks) or fvb_mgpu_allreduce_max(rank, buf, stream) from one thread per GPU.
 *   One process per GPU:      rank 0 calls fvb_mgpu_unique_id(id) and the caller
 *     broadcasts the FVB_MGPU_ID_BYTES bytes; every rank then calls
 *     fvb_mgpu_init_rank(nranks, rank, id) with its device current, and
 *     fvb_mgpu_allreduce_max(rank, buf, stream) per step.
 * buf is a device pointer to one double; asynchronous on stream.
 * fvb_mgpu_finalize destroys the communicators. */
#define FVB_MGPU_ID_BYTES 128
int fvb_mgpu_unique_id(uint8_t* id_out /* [FVB_MGPU_ID_BYTES] */);
int fvb_mgpu_init_rank(int nranks, int rank, const uint8_t* id /* [FVB_MGPU_ID_BYTES] */);
int fvb_mgpu_init(int ndev, const int* devs);
int fvb_mgpu_allreduce_max(int rank, double* buf, void* stream);
int fvb_mgpu_allreduce_max_all(double* const* bufs, void* const* streams);
int fvb_mgpu_finalize(void);

/* FVB1 batch files (host memory, no device work), byte
 * compatible with the reference's fixture dumps save_batch / load_batch
 * (mesh.py:313-353): "FVB1", int64 (d, p, s, N), then QIn, QOut,
 * cell_centre, cell_size, t, dt, max_eigenvalue as little-endian float64.
 * fvb_fvb1_header reads the header; fvb_fvb1_read fills caller-sized arrays
 * (header must equal the file's; a NULL array is skipped);
 * fvb_fvb1_write writes a dump.  FVB_ERR_CONTRACT on a bad magic / header /
 * size mismatch, FVB_ERR_IO on file errors. */
int fvb_fvb1_header(const char* path, int64_t* header /* [4] */);
int fvb_fvb1_read(const char* path, const int64_t* header, double* qin, double* qout, double* cell_centre,
                  double* cell_size, double* t, double* dt, double* max_eig);
int fvb_fvb1_write(const char* path, const int64_t* header, const double* qin, const double* qout,
                   const double* cell_centre, const double* cell_size, const double* t, const double* dt,
                   const double* max_eig);

/* Self-test: shared-reciprocal division vs IEEE division for n operand pairs. */
int fvb_selftest_div(const double* a, const double* b, double* out_shared, double* out_ieee,
                     int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FVB200_H */
