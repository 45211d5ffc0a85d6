// Internal declarations shared by the kernel and host translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "otm_common.cuh"
#include "otm_vbottom.cuh"

namespace otm {

constexpr int kOcLam = 32;   // multipliers evaluated per OC bisection pass

struct SimpParams {          // element.py:42-56, 91-100
    double k0, kmin, p;
};

// Level template: K[a][b] = kt[a ^ b]; equal axis scales use the compact form
// with s12 = scale / 12.  f0[a*3+i] = (K @ corners)[a][i] (element.py:86).
struct LevelTemplate {
    int equal;
    double s12;
    double kt[8];
    double f0[24];
};

struct CoarseTemplate {
    double kt[8];
};

struct Dg {
    double v[6];
};

struct LamSet {
    double v[kOcLam];    // lam^-damp per candidate multiplier; 0 encodes the free step
};

struct OcArgs {
    double step, rmin, damp, floor_ratio;   // floor_ratio = (1e-10)^damp
    int sqrt_damp;
};

// Device-resident state of the cooperative OC search (k_oc_coop).
struct OcCtl {
    double V;            // volume bound of the current search
    double V_retry;      // bound of the frozen-state retry (NaN: none)
    double bis_tol;
    double l1, l2;
    int phase;           // 0 first pass, 1 bracket, 2 bisection tree, 3 apply
    int bracket_it;
    int nlam;
    int active;
    int changed;
    int retried;
    int passes;
    double lam;
    double lams[kOcLam];
    double lam_pow[kOcLam];
    double means[kOcLam];
    int first_update;               // 1: no previous update of this run (no predicted multiplier)
    int nbr;                        // bracket values in the first pass (slots 1 .. nbr)
    int plan;                       // 1: the next bisection subtree is to be planned (oc_plan_node)
    double lam_prev;                // the previous update's multiplier (0: none)
    double ka, kb;                  // multipliers whose mean is known to be > V + tol (ka) / < V - tol (kb)
};

// Device-resident scalars of the batched PCG (3 load cases).
struct PcgScalars {
    double red[16];
    double rz[3], beta[3], pq[3], alpha[3], rr[3], target2[3], active[3];
    double sumT[3];
    double rr_min[3];    // smallest r.r of the current inner loop per case (0: none yet)
    double flags[8];     // active[3], rr[3]: copied to the host after the inner loop
    int first;
    int it;              // device-side inner loop control (conditional graph node)
    int max_it;
    int cycles;          // preconditioner applications summed over active cases
    int max_cycles;      // budget PER CASE (homogenize.py:85-90 gives every case its own)
    int nact;            // cases active at the start of the current iteration
    int ccyc[3];         // preconditioner applications of each case
    int hcount, hcap;    // residual history of the current inner loop: hist[3 * it + c] = r.r
    double* hist;        // (-1 for a case that was not active in that iteration)
    int skip;            // set by the device-side solve control once the solve is over:
                         // the T update and the trailing fp64 defect pass become no-ops
};

// Output x-plane range of a level kernel and the divisor of its sums: the whole
// periodic grid ([0, nx), n), or a slab's interior planes [1, nxl + 1) of a ghosted
// array of nxl + 2 planes (the slab path, otm_slab.cu), whose neighbour planes are
// the ghosts -- no index wraps -- and whose sums are partials of the global ones.
struct XRange {
    int xa, xb;
    double norm;
};

// Deterministic two-stage reduction workspace.
struct Red {
    double* partials;    // >= max blocks * 32 doubles
    unsigned* counter;   // zero-initialised
};

struct FilterSetup {
    int window;          // 1: reach <= 1, register-window kernel
    int ntaps;
    double w27[27];
    int* offs_dev;       // generic path
    double* wts_dev;
};

int stencil_chunks(const Geo& g, int* xb);
void launch_vbottom(cudaStream_t s, int N, const VBotArgs& a);   // N = 16 or 8

void launch_filter(cudaStream_t s, const Geo& g, const FilterSetup& fs, int adjoint, const double* in,
                   double* out, Red& red);
void launch_filter_simp(cudaStream_t s, const Geo& g, const FilterSetup& fs, const SimpParams& sp,
                        const double* rho, double* rho_f, double* k64, float* k32, Red& red, double* out4);
// the z-pair filter kernel on the planes [xr.xa, xr.xb) (mode 2: + SIMP into k64 and the
// sums of rho, rho^p, rho_f into out3; mode 1: adjoint); false if the shape has no pair kernel
bool launch_filter_range(cudaStream_t s, const Geo& g, const FilterSetup& fs, int mode, const SimpParams& sp,
                         const double* in, double* out, double* k64, Red& red, double* out3, const XRange& xr);
void launch_simp(cudaStream_t s, long long n, const double* rf, double* k64, float* k32, const SimpParams& sp);
void launch_set_kappa(cudaStream_t s, long long n, const double* kin, double* k64, float* k32);
void launch_means(cudaStream_t s, long long n, const double* rho, double p, Red& red, double* out2);
void launch_symmetrize(cudaStream_t s, const Geo& g, double* a);
void launch_coarsen(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* kf, float* kc);
void launch_dinv(cudaStream_t s, const Geo& g, const float* k, float kdiag, float* dinv);
void launch_coarsen_dinv(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* kf, float* kc,
                         float kdiag_f, float* dinv_f);
int launch_coarse_setup(cudaStream_t s, const Geo& g, const float* k, const CoarseTemplate& ct, double* work,
                         float* G);
void launch_coarse_solve(cudaStream_t s, int n, const float* G, const float* f, float* z);
void launch_res64(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                  const double* fext, const double* fmean, float* r32, Red& red, double* out9,
                  const int* skip = nullptr);   // *skip != 0: no-op (device-side solve control)
// k_res64p on the output planes [xr.xa, xr.xb); false if the shape has no k_res64p
bool launch_res64_range(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                        const double* fmean, float* r32, Red& red, double* out9, const XRange& xr);
void launch_apply64(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                    double* out, int load_case);
void launch_load_means(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, Red& red,
                       double* out3, const XRange* xr = nullptr);
void launch_sum3(cudaStream_t s, long long n, const double* f, Red& red, double* out3);
void launch_smooth_res(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* f,
                       const float* dinv, float omega, float* z, float* res);
void launch_jacobi(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* z,
                   const float* f, const float* dinv, float omega, float* zout, bool dot, Red& red,
                   PcgScalars* sc);
bool k10_level(const Geo& g, const LevelTemplate& lt);
bool launch_k10_range(cudaStream_t s, int op, const Geo& g, const LevelTemplate& lt, int xa, int xb,
                      const float* kap, const float* a, const float* f, const float* dinv, float omega, float* o1,
                      float* o2, bool dot, Red& red, PcgScalars* sc);
void launch_spmv(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* p,
                 float* q, Red& red, PcgScalars* sc);
void launch_pupd(cudaStream_t s, long long n, const float* z, float* p, float* d, const PcgScalars* sc);
// loop != 0: the conditional-WHILE handle of the inner-loop graph (the kernel's last
// block also runs the loop control)
void launch_upd(cudaStream_t s, long long n, float* r, const float* q, Red& red, PcgScalars* sc,
                unsigned long long loop = 0);
void launch_restrict(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* res, float* fc);
void launch_prolong(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* zc, float* zf);
void launch_Tupd(cudaStream_t s, long long n, double* T, const float* d, const float* p, const PcgScalars* sc);
void launch_submean_means(cudaStream_t s, long long n, double* T, const double* means);
void launch_submean(cudaStream_t s, long long n, double* T, const double* sumT);
void launch_tensor(cudaStream_t s, const Geo& g, const double* T, const double* kap, Red& red, double* out6,
                   const XRange* xr = nullptr);
void launch_pair_energy(cudaStream_t s, const Geo& g, const double* T, double* E);
void launch_elem_diff(cudaStream_t s, const Geo& g, const double* T, int ci, float* w);
void launch_sens(cudaStream_t s, const Geo& g, const double* T, const double* rf, const SimpParams& sp,
                 const Dg& dG, double* sens, const Dg* dG_dev = nullptr,   // dG_dev != NULL overrides dG
                 const XRange* xr = nullptr);
void launch_oc_eval(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a, int nlam,
                    const LamSet& lam_pow, Red& red, double* out);
int launch_oc_coop(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a,
                   double* rho_out, OcCtl* ctl, double* partials, double* qbuf, double* lam_mem);
void launch_oc_apply(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a,
                     double lam, double* rho_out, int* changed);

// API-level multigrid operations in fp64 (otm_levelops.cu; solver.py:85-338)
void launch_lv_apply(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                     const double* f, double* out);   // f != NULL: out = f - K T
void launch_lv_gs8(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* f, double* T,
                   int sweeps);
void launch_lv_coarsen(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* kf, double* kc);
void launch_lv_restrict(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* r, double* fc);
void launch_lv_prolong(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* Tc, double* Tf);
void launch_lv_coarse_factor(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, double* M);
void launch_lv_coarse_solve(cudaStream_t s, int n, const double* Minv, const double* f, double* T);

}  // namespace otm
