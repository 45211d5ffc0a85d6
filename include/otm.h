/*
 * otm.h - C ABI of libotm, the B200 (sm_100a) implementation of the OpenTM
 * homogenization + Optimality-Criteria hot path (arXiv 2405.19991).
 *
 * Every entry point takes plain pointers and sizes.  Array arguments named
 * *_dev are DEVICE pointers (the caller owns them; PyTorch allocates them in
 * the Python host layer); arrays without the suffix are host memory.  All
 * fields are C-order (nx, ny, nz) float64, contiguous along z, exactly the
 * numpy layout of the reference.  Work is ordered on the context's stream.
 *
 * Return codes:
 *   OTM_OK            0
 *   OTM_EINVAL        1  -> ValueError           in the Python layer
 *   OTM_ENOCONV       2  -> ConvergenceError(residual) / OptimizationAborted
 *   OTM_ECUDA         3  -> RuntimeError (CUDA failure)
 *   OTM_ESTATE        4  -> RuntimeError (e.g. hierarchy not built)
 * otm_last_error() returns the message of the most recent failure.
 *
 * Which reference interface each call replaces is cited per function
 * (paths relative to /root/reference/pkg/src/opentm/).
 */
#ifndef OTM_H
#define OTM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTM_OK 0
#define OTM_EINVAL 1
#define OTM_ENOCONV 2
#define OTM_ECUDA 3
#define OTM_ESTATE 4

typedef struct otm_ctx otm_ctx;

/* Material + filter + solver knobs.  Mirrors MaterialParams (element.py:42-56),
 * FilterSpec (field.py:69-93) and the GridHierarchy defaults (solver.py:211). */
typedef struct otm_params {
    double kappa0;         /* 1.0   */
    double kappa_min;      /* 1e-4  */
    double penalty;        /* 3.0   */
    double filter_radius;  /* 1.5 (cone kernel, <= 27 taps: radius <= sqrt(3)+1) */
    int coarse_target;     /* 64    (solver.py:211) */
    int direct_limit;      /* 40000 (solver.py:212) */
    /* B200 solver knobs (no reference counterpart) */
    double jacobi_omega;   /* level-0 Jacobi weight of the V-cycle smoother, 0.95 (coarse levels: 1.25) */
    double inner_reduction;/* fp32 inner PCG relative reduction floor per refinement step, 1e-5 */
    int max_inner;         /* cap on inner PCG iterations per refinement step, 40 */
    int device;            /* CUDA ordinal */
} otm_params;

typedef struct otm_oc_params {   /* OCParams, optimize.py:89-111 */
    double min_density;   /* 0.001 */
    double step_limit;    /* 0.02  */
    double damp;          /* 0.5   */
    double bisection_tol; /* 1e-5  */
} otm_oc_params;

typedef struct otm_governor {    /* GovernorState, optimize.py:38-54 */
    double vstar, df, gap;
    int count;
    double bound;
    int iter;
    double g_prev;
    int reduced;
} otm_governor;

/* One design-loop record: IterationRecord, optimize.py:222-230 */
typedef struct otm_iter_record {
    int iter;
    double g;
    double volfrac;
    double volfrac_filtered;
    double vstar;
    int vcycles;
    double ms;
    double kappa[6];
    double solve_residual[3];
} otm_iter_record;

/* RunConfig subset that drives the loop (optimize.py:171-219); model "oc" or "fixed". */
typedef struct otm_run_config {
    double target[6];       /* packed k11,k22,k33,k12,k23,k13 ; NaN = unconstrained */
    int objective;          /* 0 mse, 1 rel, 2 l1 (objective.py:18-25) */
    int model;              /* 0 adaptive OC, 2 fixed-volume OC */
    double volume_bound;    /* fixed model only */
    otm_oc_params oc;
    int max_iter;
    double conv_threshold;  /* 1e-4 */
    int symmetry;           /* 0 none, 1 central */
    double solver_tol;      /* 1e-6 */
    int max_vcycles;        /* 200 */
    double governor_bound;  /* 1e-4 */
} otm_run_config;

typedef struct otm_run_state {
    otm_governor gov;
    int iter;
    int plateau;
    int have_g_last;
    double g_last;
    int converged;
    int finished;
    int warm;               /* T fields hold the previous iteration's solution */
    double g;               /* objective of the last evaluation */
    double mean_rho;        /* mean(rho), mean(rho^p) of the last evaluated density */
    double mean_rho_p;
} otm_run_state;

/* ---- lifetime ------------------------------------------------------------ */
void otm_default_params(otm_params* p);
void otm_default_oc_params(otm_oc_params* p);
void otm_default_run_config(otm_run_config* c);
void otm_default_governor(otm_governor* g);
/* GridHierarchy(dims) (solver.py:203-247): validates dims, builds the level chain,
 * allocates every device workspace.  OTM_EINVAL for bad / uncoarsenable dims. */
int otm_create(otm_ctx** out, int nx, int ny, int nz, const otm_params* p);
int otm_destroy(otm_ctx* ctx);
int otm_set_stream(otm_ctx* ctx, void* cuda_stream);
const char* otm_last_error(const otm_ctx* ctx);
const char* otm_version(void);
int otm_num_levels(const otm_ctx* ctx);
int otm_level_info(const otm_ctx* ctx, int level, int dims[3], double axis_scale[3]);
size_t otm_device_bytes(const otm_ctx* ctx);

/* Change the SIMP material of an existing context (element.py:42-56). */
int otm_set_material(otm_ctx* ctx, double kappa0, double kappa_min, double penalty);

/* ---- L1 field (field.py) -------------------------------------------------- */
/* filter_forward / filter_backward (field.py:222-243): out = F in, or F^T in. */
int otm_filter(otm_ctx* ctx, const double* in_dev, double* out_dev, int adjoint);
/* project_central_symmetry (field.py:246-255), in place. */
int otm_symmetrize(otm_ctx* ctx, double* a_dev);

/* ---- L2/L3 solver + homogenization (solver.py, homogenize.py) ------------- */
/* simp_conductivity + GridHierarchy.build (element.py:91-94, solver.py:269-305). */
int otm_build(otm_ctx* ctx, const double* rho_filtered_dev);
/* GridHierarchy.build with explicit element factors (solver.py:269). */
int otm_build_kappa(otm_ctx* ctx, const double* kappa_dev);
/* One V-cycle of the built hierarchy (the MG preconditioner, solver.py:206-215, with
 * the damped-Jacobi smoother) on 3 fp32 fields: z3 = V(f3), both 3*n floats on the
 * device.  Used by the slab solver for the agglomerated coarse levels. */
int otm_vcycle(otm_ctx* ctx, const float* f3_dev, float* z3_dev);
/* apply_K on level 0 in fp64 (solver.py:111-119). */
int otm_apply_K(otm_ctx* ctx, const double* T_dev, double* out_dev);
/* assemble_macro_load (solver.py:347-363) for case 0..2. */
int otm_macro_load(otm_ctx* ctx, int which, double* f_dev);
/* Warm start (solver.py:388-391): T_dev holds 3 fields (3*n doubles) or NULL to zero.
 * Loaded fields also become the fields otm_tensor / otm_sensitivity contract. */
int otm_set_warm(otm_ctx* ctx, const double* T_dev);
/* solve_cases / solve_equation (homogenize.py:71-91, solver.py:366-406): solves the
 * three load cases batched.  f_dev = NULL uses the macro loads of the built factors;
 * otherwise 3*n doubles (a zero field is the reference's zero-load short circuit).
 * residual_out[c] = ||f_c - K T_c|| / ||f_c|| (fp64).  OTM_ENOCONV if any case
 * misses tol within max_cycles preconditioner applications. */
int otm_solve(otm_ctx* ctx, const double* f_dev, double tol, int max_cycles,
              int* cycles_out, double residual_out[3]);
/* The mean-free corrective fields (3*n doubles). */
int otm_get_T(otm_ctx* ctx, double* T_dev);
/* GridHierarchy.residual_history (solver.py:247, 395-401) of the last otm_solve: one
 * relative residual per preconditioner application (the worst over the cases it
 * served; the last entry of every fp64 refinement step is the true fp64 residual).
 * Copies min(count, cap) values to out (host) and returns count. */
int otm_residual_history(const otm_ctx* ctx, double* out, int cap);

/* ---- API-level multigrid pieces (solver.py:85-338), fp64, any level ----------
 * The reference exposes its V-cycle parts as functions over mutable level arrays
 * (GridLevel.T/f/r).  These run them on caller-owned fp64 device fields of level
 * `level` (n_l doubles).  They use the reference's own smoother (8-colour GS);
 * the design loop does not call them (it runs the batched MG-PCG above). */
/* GridLevel.kappa: the level's child-mean element factors (solver.py:257-267). */
int otm_level_kappa(otm_ctx* ctx, int level, double* kappa_dev);
/* apply_K on any level (solver.py:111-119); f_dev != NULL gives f - K T (solver.py:334). */
int otm_level_apply(otm_ctx* ctx, int level, const double* T_dev, const double* f_dev, double* out_dev);
/* relax_gs8 (solver.py:131-164): colour-ordered Gauss-Seidel on T_dev in place.
 * OTM_EINVAL for odd axes > 1, as the reference's ValueError. */
int otm_relax_gs8(otm_ctx* ctx, int level, double* T_dev, const double* f_dev, int sweeps);
/* restrict (solver.py:167-177): fc_dev (level_f + 1) = full-weighting R r_dev. */
int otm_restrict(otm_ctx* ctx, int level_f, const double* r_dev, double* fc_dev);
/* prolong_correct (solver.py:194-200): Tf_dev += P Tc_dev (Tc on level_f + 1). */
int otm_prolong_correct(otm_ctx* ctx, int level_f, double* Tf_dev, const double* Tc_dev);
/* coarse_solve (solver.py:307-324): T_dev = pinned direct solve of the coarsest level
 * with the load mean projected out, mean-free result. */
int otm_coarse_solve(otm_ctx* ctx, const double* f_dev, double* T_dev);
/* effective_tensor (homogenize.py:103-130): packed [k11,k22,k33,k12,k23,k13]. */
int otm_tensor(otm_ctx* ctx, double kappa_out[6]);
/* pair_energy cache (6*n doubles, homogenize.py:116-120), for API compatibility. */
int otm_pair_energy(otm_ctx* ctx, double* E_dev);

/* HomogenizationResult.elem_diff (homogenize.py:94-100): for one load case's field T
 * (device, level-0 layout, n doubles) the per-element corner differences
 * w[e*8 + a] = c_a[load_case] - T[e + c_a] as float32 (n*8 floats, device). */
int otm_elem_diff(otm_ctx* ctx, const double* T_dev, int load_case, float* w_dev);
/* tensor_sensitivity (homogenize.py:143-160): sens_f = kappa'(rho_f) dG.E / M. */
int otm_sensitivity(otm_ctx* ctx, const double dG[6], double* sens_f_dev);

/* ---- L4/L5 objective + optimizer (objective.py, optimize.py) -------------- */
int otm_objective(int kind, const double target[6], const double kappa[6],
                  double* g_out, double dG_out[6]);
/* mean(rho) and mean(rho^penalty), fp64 fixed-order sums. */
int otm_means(otm_ctx* ctx, const double* rho_dev, double penalty, double out[2]);
/* oc_update (optimize.py:114-160).  rho_out_dev may alias rho_dev. */
int otm_oc_update(otm_ctx* ctx, const double* rho_dev, const double* sens_dev,
                  double vol_bound, const otm_oc_params* p, double* rho_out_dev,
                  double* lam_out, int* active_out, int* changed_out);
/* governor_update (optimize.py:57-86): pure host scalar logic. */
double otm_governor_update(otm_governor* st, double g, double mean_rho, double mean_rho_p);

/* ---- the design loop (optimize.py:257-379) -------------------------------- */
void otm_run_init(otm_run_state* st, const otm_run_config* cfg);
/* Evaluation half of one loop iteration (optimize.py:288-345) on the device density
 * rho_dev: filter, SIMP, solve, tensor, objective, sensitivities, log record and the
 * convergence test (st->finished set when the loop breaks).  rho_f_dev / sens_dev
 * (n doubles each, may be NULL) receive the filtered density and the sensitivity. */
int otm_run_step(otm_ctx* ctx, const otm_run_config* cfg, otm_run_state* st,
                 double* rho_dev, double* rho_f_dev, double* sens_dev, otm_iter_record* rec);
/* Update half (optimize.py:347-379): governor, move-limited OC step (with the
 * frozen-state retry) and the optional symmetry projection, rho_dev in place. */
int otm_run_update(otm_ctx* ctx, const otm_run_config* cfg, otm_run_state* st, double* rho_dev);

/* Up to max_iters iterations of the design loop (optimize.py:288-379), each ONE
 * launch of a captured graph that keeps every decision on the device: the solve's
 * stopping rule and per-case budgets, the objective, the log record, the convergence
 * rule, the volume governor and the OC search (nested conditional WHILE / IF nodes;
 * otm_loop.cu).  The host synchronises once per `batch` iterations to collect the
 * records; iterations launched after the run finished are no-ops.  st is read at
 * entry and written back at exit (the same state otm_run_step / otm_run_update
 * advance, bit-identical results).  records receive *n_out entries.  Returns
 * OTM_ENOCONV when a solve fails (the records hold the iterations before it) and
 * OTM_ESTATE when the graph path is unavailable (profiling, no cooperative launch):
 * the caller then drives the same loop with otm_run_step / otm_run_update. */
int otm_run_batch(otm_ctx* ctx, const otm_run_config* cfg, otm_run_state* st, double* rho_dev,
                  int max_iters, int batch, otm_iter_record* records, int* n_out);

/* ---- instrumentation (bench.py) ------------------------------------------- */
/* Per-kernel-class device time accumulated with CUDA events on the context stream
 * while enabled.  Classes: 0 level-0 stencil (K.p / smoother / residual), 1 V-cycle
 * (all levels), 2 fp64 residual, 3 tensor+sens, 4 filter, 5 OC. */
int otm_profile_enable(otm_ctx* ctx, int on);
int otm_profile_read(otm_ctx* ctx, int cls, double* ms_total, long long* launches,
                     double* bytes);
int otm_profile_reset(otm_ctx* ctx);
long long otm_launch_count(const otm_ctx* ctx);
/* Solver / OC counters since creation or the last reset: solves, fp64 refinement
 * steps, inner PCG iterations (one V-cycle per active case each), OC updates, OC
 * multiplier passes, frozen-state retries. */
int otm_stats(const otm_ctx* ctx, long long out[6]);
int otm_stats_reset(otm_ctx* ctx);

/* Device time of the phases of the graph-path design iterations since the last
 * otm_stats_reset (%globaltimer stamps written by the loop-control kernels), ms:
 * [0] filter + hierarchy build + solve, [1] tensor + objective / governor,
 * [2] sensitivities + adjoint filter + OC step, [3] gaps between iterations. */
int otm_loop_phases(const otm_ctx* ctx, double ms[4]);

#ifdef __cplusplus
}
#endif
#endif /* OTM_H */
