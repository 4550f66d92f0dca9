/*
 * fvb_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's batched Rusanov patch update
 * (fvbatch.kernel.vectorized, /root/reference/pkg/src/fvbatch/kernel/vectorized.py)
 * used as the parity checker by tests/, by __graft_entry__.smoke() and as the
 * cpu_baseline / `--impl reference` leg of bench.py.  Nothing in the product
 * package (paper_2302_09005_b200/) links or calls this code.
 *
 * Parity of this restatement is pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py, run in the build container
 * where /root/reference is importable).
 */
#ifndef FVB_ORACLE_H
#define FVB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Per-(patch, box) diagnostic record, mirroring what
 * vectorized._pass_fill_eigenvalues (vectorized.py:123-139) and
 * vectorized._locate_bad_state (vectorized.py:82-99) observe for one box:
 *   trig_rho     any rho <= 0              (pde.py:36-38 raise condition)
 *   trig_p       any p < 0                 (pde.py:66-68 raise condition)
 *   first_nonpos first box-linear index with !(rho > 0)       (vectorized.py:86), -1 if none
 *   first_badpl  first box-linear index with !(E-|j|^2/(2rho) >= 0) (vectorized.py:88-90), -1 if none
 * Box order follows vectorized._plan (vectorized.py:42-53): interior, then
 * (low, high) face slab per direction x, y[, z]. Box-linear index is C order
 * over the box's (z,) y, x extents. */
typedef struct {
  int64_t trig_rho, trig_p, first_nonpos, first_badpl;
} fvb_oracle_boxinfo;

/* One forward-Euler Rusanov step for n patches, AoS layout
 * (mesh.py:174-177, [patch][z][y][x][unknown]).  Returns 0, or 2 if any
 * face-box volume is non-physical (outputs then unspecified, as in the
 * reference).  nthreads <= 0 means "all available". */
int fvb_oracle_update(int dim, int p, int64_t n, double gamma,
                      const double* qin, double* qout,
                      const double* cell_size, const double* dt,
                      double* max_eig, int nthreads);

/* Fill info[n * (2*dim+1)] with the per-(patch, box) diagnostics. */
int fvb_oracle_locate(int dim, int p, int64_t n, double gamma,
                      const double* qin, fvb_oracle_boxinfo* info, int nthreads);

/* Compose the first error the vectorized engine raises, given the per-box
 * diagnostics.  ordering: 0 = patchwise, 1 = batched.  nchunks: number of
 * contiguous patch chunks (vectorized._patch_chunks, vectorized.py:234-243;
 * 1 for sequential).  Outputs: patch index, box, box-linear index and kind
 * (1 = density message, 2 = pressure message).  Returns 1 if an error is
 * raised, 0 otherwise. */
int fvb_oracle_first_error(int dim, int p, int64_t n,
                           const fvb_oracle_boxinfo* info, int ordering,
                           int64_t nchunks, int64_t* patch, int* box,
                           int64_t* lin, int* kind);

#ifdef __cplusplus
}
#endif
#endif
