// Device-resident design iteration (optimize.py:288-379): the control kernels of
// the iteration graph that otm_run_batch (otm_api.cu) captures once per context.
//
// One graph launch = one design iteration with NO host round trip:
//   k_iter_begin -> IF(not finished) {
//     filter + SIMP | hierarchy build (side branch)  ; load means ; cold-start T
//     fp64 defect ; WHILE(not converged) { k_solve_ctl ; WHILE(PCG) { V-cycle, K p, updates } ; T += d ; defect }
//     k_solve_fin ; tensor sums ; k_design_eval (objective, record, convergence,
//     governor, OC bounds) ; sensitivities ; adjoint filter ;
//     IF(not finished) { cooperative OC search + update ; k_oc_account } }
// The decisions the host used to take between launches (solve stopping rule and
// per-case budgets, objective, convergence rule, volume governor, OC bounds) are
// the same __host__ __device__ functions (otm_loopctl.cuh), so the graph path and
// the host-driven path give bit-identical designs.
#include "otm_loopctl.cuh"

namespace otm {

namespace {

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// one design iteration of the batch loop: run it unless the run finished or the
// batch is used up; the WHILE around the batch ends with the first no-run
__global__ void k_iter_begin(LoopState* S, cudaGraphConditionalHandle h, cudaGraphConditionalHandle h_loop) {
    const bool run = !S->finished && S->batch_left > 0;
    cudaGraphSetConditional(h_loop, run ? 1u : 0u);
    if (run) {
        S->batch_left -= 1;
        S->t0 = global_ns();
        if (S->t_oc) S->ph_ms[3] += (double)(S->t0 - S->t_oc) * 1e-6;
        S->outer = 0;
        S->cycles = 0;
        for (int c = 0; c < 3; ++c) S->ccyc[c] = 0;
    }
    cudaGraphSetConditional(h, run ? 1u : 0u);
}

// cold start (solver.py:388-391 with x0 = None): T = 0 before the first solve
// also re-arms the solve's outer WHILE: a conditional's default value is applied per
// graph launch, and one launch now runs a whole batch of design iterations
__global__ void k_T_cold(const LoopState* __restrict__ S, long long n3, double* __restrict__ T,
                         cudaGraphConditionalHandle h_out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h_out, 1u);
    if (S->warm) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += (long long)gridDim.x * blockDim.x)
        T[i] = 0.0;
}

// otm_solve's outer step (solver.py:396-406 stopping rule, per-case V-cycle budgets):
// reads the fp64 defect sums, decides whether to run another inner MG-PCG loop and
// initialises its scalars
__global__ void k_solve_ctl(LoopState* S, LoopCfg C, const double* __restrict__ res9, PcgScalars* sc,
                            cudaGraphConditionalHandle h_out, cudaGraphConditionalHandle h_in) {
    bool done[3];
    for (int c = 0; c < 3; ++c) {
        const double fn = sqrt(res9[3 + c]), rn = sqrt(res9[c]);
        S->fnorm[c] = fn;
        S->rnorm[c] = rn;
        S->rel[c] = fn > 0.0 ? rn / fn : 0.0;
        done[c] = fn == 0.0 || S->rel[c] <= C.solver_tol;
        if (S->outer == 0) S->zero_load[c] = fn == 0.0;
    }
    if (S->outer > 0) {                         // an inner loop ran since the last decision
        S->cycles = sc->cycles;
        for (int c = 0; c < 3; ++c) S->ccyc[c] = sc->ccyc[c];
        S->n_inner += sc->it;
        S->n_outer += 1;
    } else {
        S->n_solves += 1;
    }
    bool all = true, over = false;
    for (int c = 0; c < 3; ++c) {
        all = all && done[c];
        over = over || (!done[c] && S->ccyc[c] >= C.max_vcycles);
    }
    S->outer += 1;
    for (int c = 0; c < 3; ++c) S->done[c] = done[c];
    if (all || over) {
        S->t_solve = global_ns();
        if (!all) S->status = 2;               // ConvergenceError (solver.py:404-406)
        sc->skip = 1;
        cudaGraphSetConditional(h_out, 0u);
        cudaGraphSetConditional(h_in, 0u);
        return;
    }
    for (int k = 0; k < 16; ++k) sc->red[k] = 0.0;
    for (int c = 0; c < 3; ++c) {
        const double tgt = fmax(C.inner_reduction * S->rnorm[c], C.tolf * C.solver_tol * S->fnorm[c]);
        sc->rz[c] = sc->beta[c] = sc->pq[c] = sc->alpha[c] = sc->rr[c] = sc->sumT[c] = sc->rr_min[c] = 0.0;
        sc->target2[c] = tgt * tgt;
        sc->active[c] = done[c] ? 0.0 : 1.0;
        sc->ccyc[c] = S->ccyc[c];
    }
    for (int k = 0; k < 8; ++k) sc->flags[k] = 0.0;
    sc->first = 1;
    sc->it = 0;
    sc->max_it = C.max_inner;
    sc->cycles = S->cycles;
    sc->max_cycles = C.max_vcycles;
    sc->nact = (int)!done[0] + (int)!done[1] + (int)!done[2];
    sc->hist = nullptr;
    sc->hcount = sc->hcap = 0;
    sc->skip = 0;
    cudaGraphSetConditional(h_out, 1u);
    cudaGraphSetConditional(h_in, 1u);
}

// zero loads short-circuit to T = 0 (solver.py:382-385)
__global__ void k_solve_fin(const LoopState* __restrict__ S, long long n, double* __restrict__ T) {
    if (!(S->zero_load[0] || S->zero_load[1] || S->zero_load[2])) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * n; i += (long long)gridDim.x * blockDim.x)
        if (S->zero_load[i / n]) T[i] = 0.0;
}

// evaluation tail of the iteration: objective, the log record, convergence rule
// (optimize.py:300-345), then the governor and the OC bounds (optimize.py:347-362)
__global__ void k_design_eval(LoopState* S, LoopCfg C, const double* __restrict__ kap6,
                              const double* __restrict__ sums3, long long n, OcCtl* ocl,
                              cudaGraphConditionalHandle h_upd) {
    const int it = S->iter + 1;
    LoopRecord* rec = &S->rec[(it - 1) % kLoopRing];
    S->t_eval = global_ns();
    S->ph_ms[0] += (double)(S->t_solve - S->t0) * 1e-6;
    S->ph_ms[1] += (double)(S->t_eval - S->t_solve) * 1e-6;
    S->t_oc = 0;
    const double mean_rho = sums3[0] / (double)n, mean_rho_p = sums3[1] / (double)n, mean_rf = sums3[2] / (double)n;
    rec->iter = it;
    rec->vcycles = S->cycles;
    for (int c = 0; c < 6; ++c) rec->kappa[c] = kap6[c];
    for (int c = 0; c < 3; ++c) rec->resid[c] = S->rel[c];
    rec->volfrac = mean_rho;
    rec->volfrac_filtered = mean_rf;
    rec->vstar = C.model == 0 ? S->gov.vstar : (C.model == 2 ? C.volume_bound : NAN);
    double g = NAN;
    bool ok = S->status == 0;
    if (ok) ok = objective_eval(C.objective, C.target, kap6, &g, S->dG.v);
    if (ok) S->warm = 1;
    else if (S->status == 0) S->status = 1;
    rec->g = g;
    rec->status = S->status;
    bool finished = !ok;
    if (ok) {
        S->iter = it;
        const bool conv = convergence_step(C.model, C.conv_threshold, S->gov, g, &S->plateau, &S->have_g_last,
                                           &S->g_last);
        S->converged = conv ? 1 : 0;
        S->g = g;
        S->mean_rho = mean_rho;
        S->mean_rho_p = mean_rho_p;
        finished = conv || it == C.max_iter;
    }
    S->finished = finished ? 1 : 0;
    rec->finished = S->finished;
    rec->ms = (double)(global_ns() - S->t0) * 1e-6;
    if (!finished) {
        double V, V_retry;
        if (C.model == 0) {
            oc_bounds(governor_step(&S->gov, g, mean_rho, mean_rho_p), mean_rho, C.oc_step, &V, &V_retry);
        } else {
            V = C.volume_bound;
            V_retry = NAN;
        }
        OcCtl z = {};
        z.V = V;
        z.V_retry = V_retry;
        z.bis_tol = C.oc_bis_tol;
        z.first_update = it == 1;                // the OC search predicts from the previous update
        *ocl = z;
    }
    cudaGraphSetConditional(h_upd, finished ? 0u : 1u);
}

// diagnostic time stamps inside the iteration graph (OTM_STAMPS=1): idx 0 restarts
__global__ void k_stamp(LoopState* S, int idx) {
    const unsigned long long t = global_ns();
    if (idx > 0 && S->t_mark) S->mark_ms[idx] += (double)(t - S->t_mark) * 1e-6;
    S->t_mark = t;
}

__global__ void k_oc_account(LoopState* S, const OcCtl* ocl) {
    S->t_oc = global_ns();
    S->ph_ms[2] += (double)(S->t_oc - S->t_eval) * 1e-6;
    S->n_oc += 1;
    S->n_oc_passes += ocl->passes;
    S->n_oc_retries += ocl->retried;
}

}  // namespace

void launch_oc_account(cudaStream_t s, LoopState* S, const OcCtl* ocl) { k_oc_account<<<1, 1, 0, s>>>(S, ocl); }
void launch_iter_begin(cudaStream_t s, LoopState* S, unsigned long long h, unsigned long long h_loop) {
    k_iter_begin<<<1, 1, 0, s>>>(S, (cudaGraphConditionalHandle)h, (cudaGraphConditionalHandle)h_loop);
}
void launch_T_cold(cudaStream_t s, const LoopState* S, long long n3, double* T, unsigned long long h_out) {
    k_T_cold<<<592, 256, 0, s>>>(S, n3, T, (cudaGraphConditionalHandle)h_out);
}
void launch_solve_ctl(cudaStream_t s, LoopState* S, const LoopCfg& C, const double* res9, PcgScalars* sc,
                      unsigned long long h_out, unsigned long long h_in) {
    k_solve_ctl<<<1, 1, 0, s>>>(S, C, res9, sc, (cudaGraphConditionalHandle)h_out, (cudaGraphConditionalHandle)h_in);
}
void launch_solve_fin(cudaStream_t s, LoopState* S, long long n, double* T) {
    k_solve_fin<<<592, 256, 0, s>>>(S, n, T);
}
void launch_stamp(cudaStream_t s, LoopState* S, int idx) { k_stamp<<<1, 1, 0, s>>>(S, idx); }
void launch_design_eval(cudaStream_t s, LoopState* S, const LoopCfg& C, const double* kap6, const double* sums3,
                        long long n, OcCtl* ocl, unsigned long long h_upd) {
    k_design_eval<<<1, 1, 0, s>>>(S, C, kap6, sums3, n, ocl, (cudaGraphConditionalHandle)h_upd);
}

}  // namespace otm
