// Design-loop control shared by the host-driven path (otm_run_step / otm_run_update)
// and the device-resident iteration graph (otm_run_batch): objective, volume
// governor, convergence rule, solve control.  The same __host__ __device__ code
// runs on both sides, so the two paths produce bit-identical trajectories.
#pragma once

#include <math.h>

#include "otm_internal.h"

namespace otm {

__host__ __device__ inline bool loop_isnan(double x) { return x != x; }

// round-to-nearest products and sums without FMA contraction on either side: the
// reference's numpy evaluates every product and sum separately, and host (gcc) and
// device (nvcc contracts a*b+c by default) must agree bit for bit
__host__ __device__ inline double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ inline double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ inline double sub_rn(double a, double b) { return add_rn(a, -b); }

// objective.py:48-72 (mse / rel / l1 with NaN-masked components); false if invalid
__host__ __device__ inline bool objective_eval(int kind, const double* t, const double* k, double* g_out,
                                               double* dG) {
    double g = 0.0;
    int any = 0;
    for (int c = 0; c < 6; ++c) {
        if (loop_isnan(k[c]) || fabs(k[c]) > 1.7976931348623157e308) return false;
        if (!loop_isnan(t[c])) any = 1;
    }
    if (!any) return false;
    for (int c = 0; c < 6; ++c) {
        const bool m = !loop_isnan(t[c]);
        if (kind == 0) {
            const double d = m ? sub_rn(k[c], t[c]) : 0.0;
            g = add_rn(g, mul_rn(d, d));
            dG[c] = mul_rn(2.0, d);
        } else if (kind == 1) {
            const double tt = m ? t[c] : 1.0;
            const double d = m ? sub_rn(k[c] / tt, 1.0) : 0.0;
            g = add_rn(g, mul_rn(d, d));
            dG[c] = m ? mul_rn(2.0, d) / tt : 0.0;
        } else {
            const double d = m ? sub_rn(k[c], t[c]) : 0.0;
            g = add_rn(g, fabs(d));
            dG[c] = (d > 0) - (d < 0);
        }
    }
    *g_out = g;
    return true;
}

// GovernorState (optimize.py:38-54)
struct GovCtl {
    double vstar, df, gap;
    int count;
    double bound;
    int iter;
    double g_prev;
    int reduced;
};

// governor_update, Algorithm 1 (optimize.py:57-86); returns V*
__host__ __device__ inline double governor_step(GovCtl* st, double g, double mean_rho, double mean_rho_p) {
    if (g <= st->bound) {
        st->gap = sub_rn(st->vstar, mean_rho_p);
        st->vstar = sub_rn(st->vstar, mul_rn(st->gap, st->df));
        st->df = mul_rn(0.8, st->df);
        st->reduced = 1;
    }
    const bool little = fabs(sub_rn(st->g_prev, g)) < fmax(mul_rn(0.1, g), 1e-7);
    const bool too_big = g > st->bound;
    const bool near = mean_rho > sub_rn(st->vstar, 0.01);
    if (little && too_big && near) st->count += 1;
    else st->count = 0;
    if (st->count >= 5) {
        st->vstar = add_rn(st->vstar, mul_rn(mul_rn(0.3, st->gap), st->df));
        st->count = 0;
    }
    st->g_prev = g;
    st->iter += 1;
    return st->vstar;
}

// volume bounds of the OC step (optimize.py:347-362): the governor's V* capped at half
// a move above the current volume, and the frozen-state retry bound
__host__ __device__ inline void oc_bounds(double vstar, double mean_rho, double step, double* V, double* V_retry) {
    *V = fmin(vstar, add_rn(mean_rho, mul_rn(0.5, step)));
    *V_retry = sub_rn(mean_rho, mul_rn(0.25, step));
}

// RunConfig subset on the device (mirrors otm_run_config)
struct LoopCfg {
    double target[6];
    int objective, model;
    double volume_bound;
    double oc_min_density, oc_step, oc_damp, oc_bis_tol;
    int max_iter;
    double conv_threshold;
    int symmetry;
    double solver_tol;
    int max_vcycles;
    double governor_bound;
    double inner_reduction, tolf;     // solver knobs of the inner MG-PCG (otm_solve)
    int max_inner;
};

struct LoopRecord {       // IterationRecord (optimize.py:222-230) + tensor and solve residuals
    int iter;
    int vcycles;
    int status;           // 0 ok, 2 solver failure (no convergence)
    int finished;
    double g, volfrac, volfrac_filtered, vstar, ms;
    double kappa[6];
    double resid[3];
};

constexpr int kLoopRing = 64;

// run state (optimize.py:277-286) + the solve control of the current iteration
struct LoopState {
    GovCtl gov;
    int iter, plateau, have_g_last, converged, finished, warm, status;
    double g_last, g, mean_rho, mean_rho_p;
    // solve control (otm_solve)
    double fnorm[3], rnorm[3], rel[3];
    int done[3], zero_load[3], ccyc[3];
    int cycles, outer;
    int batch_left;               // iterations the current graph launch may still run (otm_run_batch)
    unsigned long long t0;        // %globaltimer at the start of the iteration
    unsigned long long t_solve, t_eval, t_oc;   // ... at the end of the solve, of the evaluation, of the OC step
    double ph_ms[4];              // accumulated: filter+build+solve, tensor+objective, sens+OC, gap to next
    unsigned long long t_mark;    // OTM_STAMPS: last k_stamp
    double mark_ms[20];           // OTM_STAMPS: device time before each k_stamp since the previous one
    long long n_solves, n_outer, n_inner, n_oc, n_oc_passes, n_oc_retries;   // otm_stats counters
    Dg dG;
    LoopRecord rec[kLoopRing];
};

// convergence rule (optimize.py:327-345); updates plateau / g_last, returns converged
__host__ __device__ inline bool convergence_step(int model, double conv_threshold, const GovCtl& gov, double g,
                                                 int* plateau, int* have_g_last, double* g_last) {
    if (*have_g_last && fabs(sub_rn(g, *g_last)) < conv_threshold) *plateau += 1;
    else *plateau = 0;
    *g_last = g;
    *have_g_last = 1;
    if (g <= 1e-12) return true;
    if (*plateau >= 3) {
        if (model == 0) {
            const double cd = gov.reduced ? mul_rn(gov.gap, gov.df) : INFINITY;
            return cd < 1e-4 && g <= gov.bound;
        }
        return true;
    }
    return false;
}

// launchers (otm_loop.cu)
void launch_iter_begin(cudaStream_t s, LoopState* S, unsigned long long h_body, unsigned long long h_loop);
void launch_T_cold(cudaStream_t s, const LoopState* S, long long n3, double* T, unsigned long long h_out);
void launch_solve_ctl(cudaStream_t s, LoopState* S, const LoopCfg& C, const double* res9, PcgScalars* sc,
                      unsigned long long h_out, unsigned long long h_in);
void launch_solve_fin(cudaStream_t s, LoopState* S, long long n, double* T);
void launch_design_eval(cudaStream_t s, LoopState* S, const LoopCfg& C, const double* kap6, const double* sums3,
                        long long n, OcCtl* ocl, unsigned long long h_upd);
void launch_oc_account(cudaStream_t s, LoopState* S, const OcCtl* ocl);
void launch_stamp(cudaStream_t s, LoopState* S, int idx);

}  // namespace otm
