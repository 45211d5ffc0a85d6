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
 *   otm_slab_filter      field.py:230-236 (cone filter, forward / adjoint) + element.py:91-94
 *   otm_slab_sensitivity homogenize.py:143-160
 *   otm_slab_oc_sums/apply optimize.py:114-160 (candidate means / update)
 */
#ifndef OTM_SLAB_H
#define OTM_SLAB_H

#include "otm.h"

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
/* otm_slab_stencil on the output planes [x_lo, x_hi) of the ghost-padded slab only
 * (1 <= x_lo < x_hi <= nxl + 1; dots3 sums over those planes).  Planes 2 .. nxl-1 do
 * not read the ghost planes, so they can run while the halo exchange is in flight;
 * planes 1 and nxl follow it (slab.py SlabSolver._overlapped). */
int otm_slab_stencil_range(otm_slab_ws* w, int op, int nxl, int ny, int nz, const double scale[3], const float* kap,
                           const float* a, const float* f, const float* dinv, double omega, float* o1, float* o2,
                           int x_lo, int x_hi, double* dots3);
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

/* Density filter on a slab (field.py:230-236, radius <= 2: one ghost plane), bit-identical
 * taps.  mode 2: forward + SIMP (element.py:91-94): out = rho_f, kap64 = kappa(rho_f), sums3 =
 * [sum rho, sum rho^p, sum rho_f]; mode 1: adjoint (kap64, sums3 unused).  in needs both ghosts. */
int otm_slab_filter(otm_slab_ws* w, int mode, int nxl, int ny, int nz, double radius, double kappa0,
                    double kappa_min, double penalty, const double* in, double* out, double* kap64,
                    double* sums3);
/* sens_f = kappa'(rho_f) (dG . E) / n_total (homogenize.py:143-160); T needs its right ghost. */
int otm_slab_sensitivity(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, double kappa0, double kappa_min,
                         double penalty, const double* T, const double* rho_f, const double dG6[6], double* sens_f);
/* OC candidate sums for nlam <= 32 multipliers (optimize.py:114-160; lam 0 = free step). */
int otm_slab_oc_sums(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, const otm_oc_params* pp,
                     const double* rho, const double* sens, int nlam, const double* lams, double* sums32);
/* rho_out = candidate of lam (reference expression); changed = number of vertices that moved. */
int otm_slab_oc_apply(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, const otm_oc_params* pp,
                      const double* rho, const double* sens, double lam, double* rho_out, double* changed);

/* Device scalars (round 2): with mode 1 the PCG calls take and return their scalars
 * in DEVICE memory and never synchronise the stream -- otm_slab_stencil's dots3,
 * otm_slab_pupd's beta3, otm_slab_upd's alpha3 / rr3 (and the other sums3/6/9
 * outputs) -- so a slab PCG iteration runs without host round trips; the caller
 * all-reduces the partial sums in device memory (NCCL) and advances the scalars
 * with otm_slab_pcg_step.  Mode 0 (default): host scalars, as documented above. */
int otm_slab_set_scalar_mode(otm_slab_ws* w, int device);
/* The PCG scalar recurrences on a device array S of 28 doubles:
 *   S[0..2] r.z (all-reduced)   S[3..5] previous r.z   S[6..8] beta    S[9..11] p.q (all-reduced)
 *   S[12..14] alpha            S[15..17] r.r (all-reduced)   S[18..20] target^2
 *   S[21..23] active (1/0)     S[24] first (1 before the first iteration)   S[25..27] V-cycles per case
 * stage 0: beta = first ? 0 : r.z / previous (0 if previous is 0); previous = r.z
 * stage 1: alpha = active && p.q > 0 ? r.z / p.q : 0
 * stage 2: cycles += active; active &= r.r > target^2 */
int otm_slab_pcg_step(otm_slab_ws* w, int stage, double* S_dev);

/* Ghost planes of a slab field from its neighbours' interiors, in one launch on
 * `stream`: for every case c < ncases, dst plane 0 <- left plane nxl_left and dst
 * plane nxl + 1 <- right plane 1 (planes of pl elements of elem_size 4 or 8 bytes;
 * a field holds ncases blocks of (its nxl + 2) planes).  In-process slabs
 * (LocalComm) and the single-rank case of DistComm; left == right == dst for one
 * slab.  Replaces 2 strided copies per case and side. */
int otm_slab_halo_local(void* stream, int elem_size, int ncases, long long pl, void* dst, int nxl,
                        const void* left, int nxl_left, const void* right, int nxl_right);

#ifdef __cplusplus
}
#endif

#endif
