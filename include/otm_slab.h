/*
 * otm_slab.h - slab-decomposed pieces of the homogenization solve (multi-GPU,
 * "z-slabs" of the reference's (nx, ny, nz) arrays are cut along
 * axis 0, the slowest C-order axis).
 *
 * A slab of a multigrid level owns nxl consecutive x planes.  Every field passed
 * here is stored with ONE ghost plane on each side: (nxl + 2) * ny * nz values,
 * 3-case fields case-major (case c starts at c * (nxl + 2) * ny * nz).  The caller
 * refreshes ghost planes from the neighbouring ranks (NCCL send/recv) before a
 * call that reads them; kernels write interior planes only.  Element factors use
 * the element = lower-corner-vertex convention (element e spans vertices e..e+1),
 * so operator calls read the LEFT factor ghost only.  y and z are periodic inside
 * the slab.  Scalar results are this slab's partial sums in a fixed order; the
 * caller all-reduces them across ranks.  All pointers are device pointers except
 * scale/beta/alpha/mean/fmean and the scalar outputs (host).
 *
 * Reference interfaces restated (paths relative to /root/reference/pkg/src/opentm/):
 *   otm_slab_stencil     solver.py:111 (apply_K), 131 (relax; damped Jacobi here)
 *   otm_slab_restrict    solver.py:167-180 (full weighting, R = P^T / 8)
 *   otm_slab_prolong     solver.py:194-200 (trilinear)
 *   otm_slab_coarsen     solver.py:233-245 (child mean)
 *   otm_slab_dinv        solver.py:119-128 (diagonal)
 *   otm_slab_res64       solver.py:386-401 (macro loads, mean projection, residual)
 *   otm_slab_tensor_sums homogenize.py:103-122 (kappa_H sums)
 */
#ifndef OTM_SLAB_H
#define OTM_SLAB_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct otm_slab_ws otm_slab_ws;

/* Workspace for the reductions (max_items >= 3 * nxl * ny * nz of the largest level). */
otm_slab_ws* otm_slab_create(long long max_items);
int otm_slab_destroy(otm_slab_ws* w);
int otm_slab_set_stream(otm_slab_ws* w, void* stream);
const char* otm_slab_last_error(otm_slab_ws* w);

/* op 0: o1 = w D^-1 f (z0), o2 = f - K o1 (residual)            [a unused]
 * op 1: o1 = a + w D^-1 (f - K a) (Jacobi); dots3 = sum f * o1     [per case]
 * op 2: o1 = K a;                          dots3 = sum a * o1
 * scale: the level's axis scales (GridLevel.axis_scale); dots3 may be NULL. */
int otm_slab_stencil(otm_slab_ws* w, int op, int nxl, int ny, int nz, const double scale[3], const float* kap,
                     const float* a, const float* f, const float* dinv, double omega, float* o1, float* o2,
                     double* dots3);
/* fine slab (nxl_f even, starting at an even global plane) -> coarse slab interior */
int otm_slab_restrict(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* res_f, float* f_c);
/* z_f (interior) += P z_c; z_c needs its right ghost plane */
int otm_slab_prolong(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* z_c, float* z_f);
int otm_slab_coarsen(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* k_f, float* k_c);
int otm_slab_dinv(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const float* kap, float* dinv);
/* p = z + beta p;  d += alpha p, r -= alpha q, rr3 = sum r^2 (interior, per case) */
int otm_slab_pupd(otm_slab_ws* w, int nxl, int ny, int nz, const float* z, float* p, const double beta3[3]);
int otm_slab_upd(otm_slab_ws* w, int nxl, int ny, int nz, float* d, float* r, const float* p, const float* q,
                 const double alpha3[3], double* rr3);
/* fp64: sums of the three macro loads (their global mean is subtracted, solver.py:386-387) */
int otm_slab_load_sums(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* kap64,
                       double* sums3);
/* fp64 defect r32 = (f - fmean) - K T; sums9 = [sum r^2 (3), sum f^2 (3), sum T (3)] */
int otm_slab_res64(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* kap64,
                   const double* T, const double fmean3[3], float* r32, double* sums9);
/* T = T + d - mean (interior; d is the fp32 correction, may be NULL) */
int otm_slab_tupd(otm_slab_ws* w, int nxl, int ny, int nz, double* T, const float* d, const double mean3[3]);
/* sums6 = sum_e kappa_e E_pq[e] over the slab's elements (T needs its right ghost) */
int otm_slab_tensor_sums(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* T,
                         const double* kap64, double* sums6);

#ifdef __cplusplus
}
#endif

#endif
