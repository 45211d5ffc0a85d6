// libotm kernels (sm_100a).  See DESIGN.md for the roofline and byte counts of
// each kernel; reference symbols are cited per kernel
// (paths relative to /root/reference/pkg/src/opentm/).
#include "otm_common.cuh"
#include "otm_internal.h"
#include "otm_res64p.cuh"
#include "otm_res64w.cuh"
#include "otm_stencil10.cuh"

#ifndef OTM_MINB
#define OTM_MINB 2   // min resident blocks of the fp32 fast-path stencils (register cap 128)
#endif

#include <math.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <utility>
#include <cstdlib>
#include <cstdio>

namespace otm {

// ===========================================================================
// Field kernels: filter (+SIMP), adjoint filter, symmetry, means
// ===========================================================================

// Taps of the cone filter on the 3x3x3 window (reach 1, radius <= 2): weight of
// offset o = (dx,dy,dz) at w27[(dx+1)*9 + (dy+1)*3 + (dz+1)] (0 = excluded).
// Taps are visited in the reference's order (field.py:222-227): lexicographic in
// o; the adjoint reads slot(-o) in the order of o, so the fp64 mul-then-add
// sequence equals numpy's bit for bit.
struct FilterTaps {
    double w27[27];
};

// One thread per (y, z) column, walking x; window of rho in registers.
// mode 0: plain forward filter; 1: plain adjoint; 2: forward + SIMP + kappa32 + means.
template <int MODE>
__global__ void __launch_bounds__(128) k_filter(Geo g, int xb, FilterTaps taps, const double* __restrict__ in,
                                                double* __restrict__ out, double* __restrict__ kappa64,
                                                float* __restrict__ kappa32, SimpParams sp,
                                                double* partials, unsigned* counter, double* red_out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc_r = 0.0, acc_rp = 0.0, acc_rf = 0.0;
    if (t < g.pl) {
        const int y = t / g.nz, z = t - (t / g.nz) * g.nz;
        Nbr nb;
        nbr_init(nb, g, y, z);
        const int x0 = blockIdx.y * xb, x1 = min(g.nx, x0 + xb);
        double w[3][9];
        auto load = [&](double (&dst)[9], int x) {
            const long long po = plane_off(g, x);
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int k = 0; k < 3; ++k) dst[j * 3 + k] = __ldg(in + po + nb.ro[j] + nb.co[k]);
        };
        if (x0 < x1) {
            load(w[0], x0 - 1);
            load(w[1], x0);
        }
        for (int x = x0; x < x1; ++x) {
            load(w[2], x + 1);
            // taps in the reference's order: slot(o) ascending; the adjoint reads slot(-o)
            double s = 0.0;
#pragma unroll
            for (int slot = 0; slot < 27; ++slot) {
                const double wt = taps.w27[slot];
                if (wt != 0.0) {
                    const int src = MODE == 1 ? 26 - slot : slot;
                    s = __dadd_rn(s, __dmul_rn(wt, w[src / 9][src % 9]));
                }
            }
            const long long v = (long long)x * g.pl + t;
            out[v] = s;
            if (MODE == 2) {
                const double kap = sp.kmin + simp_pow(s, sp.p) * (sp.k0 - sp.kmin);
                kappa64[v] = kap;
                kappa32[v] = (float)kap;
                const double r = w[1][4];
                acc_r += r;
                acc_rp += simp_pow(r, sp.p);
                acc_rf += s;
            }
#pragma unroll
            for (int i = 0; i < 9; ++i) { w[0][i] = w[1][i]; w[1][i] = w[2][i]; }
        }
    }
    if (MODE == 2) {
        double v3[3] = {acc_r, acc_rp, acc_rf};
        reduce_finalize<3>(v3, partials, counter, red_out);
    }
}

// High-parallelism filter (reach 1): one thread per z pair, 27 window loads up front,
// taps in the reference's order (bit-exact, see k_filter).  nz even.  MASK = the
// nonzero taps (bit slot) when known at compile time (radius 1.5: no corners; radius
// >= sqrt 3: all 27), so zero taps cost neither a compare nor their window loads;
// MASK = 0 tests every weight at run time.
constexpr unsigned kTapsAll = (1u << 27) - 1;
constexpr unsigned taps_no_corners() {
    unsigned m = 0;
    for (int s = 0; s < 27; ++s)
        if (s / 9 == 1 || (s / 3) % 3 == 1 || s % 3 == 1) m |= 1u << s;
    return m;
}
constexpr unsigned kTapsNoCorners = taps_no_corners();

template <int MODE, unsigned MASK = 0, bool GS = false>
__global__ void __launch_bounds__(256) k_filter_b(Geo g, long long p0, long long p1, FilterTaps taps,
                                                  const double* __restrict__ in, double* __restrict__ out,
                                                  double* __restrict__ kappa64, float* __restrict__ kappa32,
                                                  SimpParams sp, double* partials, unsigned* counter,
                                                  double* red_out) {
    // z pairs [p0, p1): the whole grid, or a slab's interior planes (XRange); GS: a
    // capped grid walks them (gs_cap)
    double acc3[3] = {0.0, 0.0, 0.0};
    for (long long i = p0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p1;
         i += GS ? (long long)gridDim.x * blockDim.x : p1) {
        const long long vp = i * 2;
        // 32-bit index arithmetic (fields < 2^31 vertices; see element_energies)
        const unsigned uv = (unsigned)vp, upl = (unsigned)g.pl;
        const int x = (int)(uv / upl), rem = (int)(uv - (unsigned)x * upl);
        const int y = rem / g.nz, z = rem - y * g.nz;
        const unsigned xo[3] = {(unsigned)wrap_m(x, g.nx) * upl, (unsigned)x * upl, (unsigned)wrap_p(x, g.nx) * upl};
        const int yo[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
        const int zm = z == 0 ? g.nz - 1 : z - 1, zp2 = z + 2 == g.nz ? 0 : z + 2;
        double t[3][3][4];
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double* row = in + (xo[p] + (unsigned)yo[j]);
                t[p][j][0] = __ldg(row + zm);
                const double2 m = __ldg(reinterpret_cast<const double2*>(row + z));
                t[p][j][1] = m.x;
                t[p][j][2] = m.y;
                t[p][j][3] = __ldg(row + zp2);
            }
        double res[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double s = 0.0;
#pragma unroll
            for (int slot = 0; slot < 27; ++slot) {
                const double wt = taps.w27[slot];
                if (MASK ? ((MASK >> slot) & 1u) != 0u : wt != 0.0) {
                    const int src = MODE == 1 ? 26 - slot : slot;
                    const int p = src / 9, j = (src / 3) % 3, m = src % 3;
                    s = __dadd_rn(s, __dmul_rn(wt, t[p][j][h + m]));
                }
            }
            res[h] = s;
        }
        *reinterpret_cast<double2*>(out + vp) = make_double2(res[0], res[1]);
        if (MODE == 2) {
            double k0 = sp.kmin + simp_pow(res[0], sp.p) * (sp.k0 - sp.kmin);
            double k1 = sp.kmin + simp_pow(res[1], sp.p) * (sp.k0 - sp.kmin);
            *reinterpret_cast<double2*>(kappa64 + vp) = make_double2(k0, k1);
            if (kappa32) *reinterpret_cast<float2*>(kappa32 + vp) = make_float2((float)k0, (float)k1);
            const double r0 = t[1][1][1], r1 = t[1][1][2];
            if (GS) {
                acc3[0] += r0 + r1;
                acc3[1] += simp_pow(r0, sp.p) + simp_pow(r1, sp.p);
                acc3[2] += res[0] + res[1];
            } else {
                acc3[0] = r0 + r1;
                acc3[1] = simp_pow(r0, sp.p) + simp_pow(r1, sp.p);
                acc3[2] = res[0] + res[1];
            }
        }
    }
    if (MODE == 2) reduce_finalize<3>(acc3, partials, counter, red_out);
}

// Generic-reach filter (radius > 2): one vertex per thread, taps from global memory.
__global__ void k_filter_generic(Geo g, int ntaps, const int* __restrict__ offs,
                                 const double* __restrict__ wts, int adjoint,
                                 const double* __restrict__ in, double* __restrict__ out) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.n) return;
    const int x = (int)(v / g.pl), rem = (int)(v - (long long)x * g.pl);
    const int y = rem / g.nz, z = rem - y * g.nz;
    const int sgn = adjoint ? -1 : 1;
    double s = 0.0;
    for (int i = 0; i < ntaps; ++i) {
        int xx = (x + sgn * offs[3 * i]) % g.nx; if (xx < 0) xx += g.nx;
        int yy = (y + sgn * offs[3 * i + 1]) % g.ny; if (yy < 0) yy += g.ny;
        int zz = (z + sgn * offs[3 * i + 2]) % g.nz; if (zz < 0) zz += g.nz;
        s = __dadd_rn(s, __dmul_rn(wts[i], in[((long long)xx * g.ny + yy) * g.nz + zz]));
    }
    out[v] = s;
}

__global__ void k_simp(long long n, const double* __restrict__ rf, double* __restrict__ k64,
                       float* __restrict__ k32, SimpParams sp) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double kap = sp.kmin + simp_pow(rf[v], sp.p) * (sp.k0 - sp.kmin);
    k64[v] = kap;
    k32[v] = (float)kap;
}

__global__ void k_set_kappa(long long n, const double* __restrict__ kin, double* __restrict__ k64,
                            float* __restrict__ k32) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    k64[v] = kin[v];
    k32[v] = (float)kin[v];
}

// sum(rho), sum(rho^p) (optimize.py:67, :352)
__global__ void k_means(long long n, const double* __restrict__ rho, double p, double* partials,
                        unsigned* counter, double* out) {
    double v2[2] = {0.0, 0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double r = rho[i];
        v2[0] += r;
        v2[1] += simp_pow(r, p);
    }
    reduce_finalize<2>(v2, partials, counter, out);
}

// 0.5 (a + a[rev]) in place (field.py:246-255); each pair handled by its lower index.
__global__ void k_symmetrize(Geo g, double* a) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.n) return;
    const long long w = g.n - 1 - v;   // (nx-1-i, ny-1-j, nz-1-k) in C order
    if (w < v) return;
    const double m = 0.5 * (a[v] + a[w]);
    a[v] = m;
    a[w] = m;
}

// ===========================================================================
// Multigrid setup: child-mean coarsening, Jacobi diagonal, coarse pseudo-inverse
// ===========================================================================

// kappa_{l+1} = mean of children (solver.py:257-267)
__global__ void k_coarsen(Geo f, Geo c, int cx, int cy, int cz, const float* __restrict__ kf,
                          float* __restrict__ kc) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= c.n) return;
    const int X = (int)(v / c.pl), rem = (int)(v - (long long)X * c.pl);
    const int Y = rem / c.nz, Z = rem - Y * c.nz;
    float s = 0.f;
    int cnt = 0;
    for (int a = 0; a <= cx; ++a)
        for (int b = 0; b <= cy; ++b)
            for (int d = 0; d <= cz; ++d) {
                const int x = (cx ? 2 * X : X) + a, y = (cy ? 2 * Y : Y) + b, z = (cz ? 2 * Z : Z) + d;
                s += kf[((long long)x * f.ny + y) * f.nz + z];
                ++cnt;
            }
    kc[v] = s / (float)cnt;
}

// dinv[v] = 1 / (K[a][a] * sum of the 8 incident element factors)
__global__ void k_dinv(Geo g, const float* __restrict__ k, float kdiag, float* __restrict__ dinv) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.n) return;
    const int x = (int)(v / g.pl), rem = (int)(v - (long long)x * g.pl);
    const int y = rem / g.nz, z = rem - y * g.nz;
    const int xm = wrap_m(x, g.nx), ym = wrap_m(y, g.ny), zm = wrap_m(z, g.nz);
    float s = 0.f;
    const int xs[2] = {xm, x}, ys[2] = {ym, y}, zs[2] = {zm, z};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d) s += k[((long long)xs[a] * g.ny + ys[b]) * g.nz + zs[d]];
    dinv[v] = 1.0f / (kdiag * s);
}

// One step of the hierarchy build chain: child means of level l (from level l-1)
// and D^-1 of level l-1 (whose factors the previous step produced) in one launch.
__global__ void k_coarsen_dinv(Geo f, Geo c, int cx, int cy, int cz, const float* __restrict__ kf,
                               float* __restrict__ kc, float kdiag_f, float* __restrict__ dinv_f) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < c.n) {
        const int X = (int)(v / c.pl), rem = (int)(v - (long long)X * c.pl);
        const int Y = rem / c.nz, Z = rem - Y * c.nz;
        float s = 0.f;
        int cnt = 0;
        for (int a = 0; a <= cx; ++a)
            for (int b = 0; b <= cy; ++b)
                for (int d = 0; d <= cz; ++d) {
                    const int x = (cx ? 2 * X : X) + a, y = (cy ? 2 * Y : Y) + b, z = (cz ? 2 * Z : Z) + d;
                    s += kf[((long long)x * f.ny + y) * f.nz + z];
                    ++cnt;
                }
        kc[v] = s / (float)cnt;
    }
    if (v < f.n) {
        const int x = (int)(v / f.pl), rem = (int)(v - (long long)x * f.pl);
        const int y = rem / f.nz, z = rem - y * f.nz;
        const int xs[2] = {wrap_m(x, f.nx), x}, ys[2] = {wrap_m(y, f.ny), y}, zs[2] = {wrap_m(z, f.nz), z};
        float s = 0.f;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int d = 0; d < 2; ++d) s += kf[((long long)xs[a] * f.ny + ys[b]) * f.nz + zs[d]];
        dinv_f[v] = 1.0f / (kdiag_f * s);
    }
}

// Coarsest level: assemble the dense periodic matrix (solver.py:278-296), invert
// the vertex-0-pinned block (solver.py:298-305), and fold the mean projections of
// coarse_solve (solver.py:307-324) into one symmetric matrix G = P Z P so the
// per-cycle coarse solve is a dense mat-vec.  One block; A and Z live in shared
// memory when they fit (n <= 64, the default chain) and in `work` otherwise.
__global__ void __launch_bounds__(1024) k_coarse_setup(Geo g, const float* __restrict__ k, CoarseTemplate ct,
                                                       double* __restrict__ work, float* __restrict__ G,
                                                       int use_smem) {
    extern __shared__ double sm[];
    const int n = (int)g.n;
    double* A = use_smem ? sm : work;
    double* Z = A + (size_t)n * n;
    for (int i = threadIdx.x; i < 2 * n * n; i += blockDim.x) A[i] = 0.0;
    __syncthreads();
    // row-wise assembly: row r couples through its 8 incident elements (no races)
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        const int x = r / g.pl, rem = r - x * g.pl, y = rem / g.nz, z = rem - y * g.nz;
        for (int a = 0; a < 8; ++a) {
            const int ex = (x - (a & 1) + g.nx) % g.nx, ey = (y - ((a >> 1) & 1) + g.ny) % g.ny,
                      ez = (z - ((a >> 2) & 1) + g.nz) % g.nz;
            const double ke = (double)k[(ex * g.ny + ey) * g.nz + ez];
            for (int b = 0; b < 8; ++b) {
                const int cx = (ex + (b & 1)) % g.nx, cy = (ey + ((b >> 1) & 1)) % g.ny,
                          cz = (ez + ((b >> 2) & 1)) % g.nz;
                A[(size_t)r * n + (cx * g.ny + cy) * g.nz + cz] += ke * ct.kt[a ^ b];
            }
        }
    }
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
        const int r = i / n, c = i - (i / n) * n;
        Z[i] = (r == c && r > 0) ? 1.0 : 0.0;
    }
    __syncthreads();
    // Gauss-Jordan on the SPD block A[1:,1:] (no pivoting needed), fully parallel per
    // pivot: column p of A is copied aside, row p is normalised, then every thread
    // updates a fixed column (t % 2n) of A|Z on rows t / 2n, t / 2n + rstep, ...
    // (all loads of a thread issued before its stores).
    const int m = n - 1;
    double* colp = Z + (size_t)n * n;          // n doubles after Z (smem or work)
    const int ncols = 2 * n;
    const int rstep = blockDim.x / ncols > 0 ? blockDim.x / ncols : 1;
    for (int p = 1; p <= m; ++p) {
        const double piv = A[(size_t)p * n + p];
        for (int r = threadIdx.x; r < n; r += blockDim.x) colp[r] = (r >= 1 && r != p) ? A[(size_t)r * n + p] : 0.0;
        __syncthreads();                       // pivot and column p read by everyone
        for (int t = threadIdx.x; t < ncols; t += blockDim.x) {
            double* M = t < n ? A : Z;
            const int cidx = t < n ? t : t - n;
            if (cidx >= 1) M[(size_t)p * n + cidx] /= piv;
        }
        __syncthreads();                       // row p normalised
        for (int w = threadIdx.x; w < rstep * ncols; w += blockDim.x) {
            const int t = w % ncols;
            double* M = t < n ? A : Z;
            const int cidx = t < n ? t : t - n;
            if (cidx >= 1) {
                const double rowp = M[(size_t)p * n + cidx];
                for (int r0 = 1 + w / ncols; r0 <= m; r0 += 4 * rstep) {
                    double v[4], c[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int r = r0 + u * rstep;
                        const bool ok = r <= m;
                        v[u] = ok ? M[(size_t)r * n + cidx] : 0.0;
                        c[u] = ok ? colp[r] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int r = r0 + u * rstep;
                        if (r <= m && r != p) M[(size_t)r * n + cidx] = v[u] - c[u] * rowp;
                    }
                }
            }
        }
        __syncthreads();
    }
    // G = P Z P with P = I - 11^T/n
    double* rmean = A;
    double* cmean = A + n;
    __shared__ double gmean;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
        double s = 0.0, t = 0.0;
        for (int c = 0; c < n; ++c) { s += Z[(size_t)r * n + c]; t += Z[(size_t)c * n + r]; }
        rmean[r] = s / n;
        cmean[r] = t / n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += rmean[r];
        gmean = s / n;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
        const int r = i / n, c = i - (i / n) * n;
        G[i] = (float)(Z[i] - rmean[r] - cmean[c] + gmean);
    }
}

// Coarse pseudo-inverse for the common 4^3 coarsest level (n = 64): in-place
// Gauss-Jordan inversion of the SPD block A[1:,1:] in shared memory (64 x 64
// doubles; row/column 0 = the pinned vertex), 256 threads, two barriers per pivot,
// a branch-free rank-1 update per pivot (~260 -> ~50 -> see DESIGN.md 4 for the
// measured history of this kernel).
__global__ void __launch_bounds__(256) k_coarse_setup64(Geo g, const float* __restrict__ k, CoarseTemplate ct,
                                                         float* __restrict__ G) {
    constexpr int N = 64;
    extern __shared__ double sm[];
    double* A = sm;                      // N x N
    double* colp = sm + N * N;           // N: column p;  N..2N-1: row p;  2N: 1 / pivot
    double* rowp = colp + N;
    const int tid = threadIdx.x;
    for (int i = tid; i < N * N; i += blockDim.x) A[i] = 0.0;
    __syncthreads();
    if (tid < N) {                       // row-wise assembly (row r touches only its own row)
        const int r = tid;
        const int x = r / g.pl, rem = r - x * g.pl, y = rem / g.nz, z = rem - y * g.nz;
        for (int a = 0; a < 8; ++a) {
            const int ex = (x - (a & 1) + g.nx) % g.nx, ey = (y - ((a >> 1) & 1) + g.ny) % g.ny,
                      ez = (z - ((a >> 2) & 1) + g.nz) % g.nz;
            const double ke = (double)k[(ex * g.ny + ey) * g.nz + ez];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int cx = (ex + (b & 1)) % g.nx, cy = (ey + ((b >> 1) & 1)) % g.ny,
                          cz = (ez + ((b >> 2) & 1)) % g.nz;
                A[r * N + (cx * g.ny + cy) * g.nz + cz] += ke * ct.kt[a ^ b];
            }
        }
    }
    __syncthreads();
    // pinned vertex: zero row and column 0, so the uniform update below leaves them zero
    if (tid < N) { A[tid] = 0.0; A[tid * N] = 0.0; }
    __syncthreads();
    // In-place Gauss-Jordan, branch-free: with E = A whose column p is e_p,
    // u = d * row p (u[p] = d) and v = column p (v[p] = a_pp - 1), d = 1/a_pp,
    // the step is A <- E - v u^T.  Thread: column c = tid % 64, rows tid/64 + 4k.
    const int c = tid % N, g4 = tid / N;
    double* u = rowp;
    double* v = colp;
    for (int p = 1; p < N; ++p) {
        if (tid < N) {
            const double a = A[tid * N + p];
            v[tid] = tid == p ? a - 1.0 : a;
        } else if (tid < 2 * N) {
            const int cc = tid - N;
            const double a = A[p * N + p];
            double d = (double)__frcp_rn((float)a);      // fp32 seed + two Newton steps
            d = d * (2.0 - a * d);
            d = d * (2.0 - a * d);
            u[cc] = cc == p ? d : A[p * N + cc] * d;
        }
        __syncthreads();
        const double uc = u[c];
        const bool colp_ = c == p;
#pragma unroll
        for (int q = 0; q < N / 4; ++q) {
            const int r = g4 + 4 * q;
            const double e = colp_ ? (r == p ? 1.0 : 0.0) : A[r * N + c];
            A[r * N + c] = fma(-v[r], uc, e);
        }
        __syncthreads();
    }
    // Z = inverse on [1:,1:], zero on the pinned row/column;  G = P Z P, P = I - 11^T/N
    __shared__ double rmean[N], cmean[N], gmean;
    if (tid < N) {
        double sr = 0.0;
        for (int q = 1; q < N; ++q) sr += tid ? A[tid * N + q] : 0.0;
        rmean[tid] = sr / N;
    } else if (tid < 2 * N) {
        const int cc = tid - N;
        double t = 0.0;
        for (int q = 1; q < N; ++q) t += cc ? A[q * N + cc] : 0.0;
        cmean[cc] = t / N;
    }
    __syncthreads();
    if (tid == 0) {
        double sg = 0.0;
        for (int q = 0; q < N; ++q) sg += rmean[q];
        gmean = sg / N;
    }
    __syncthreads();
    for (int i = tid; i < N * N; i += blockDim.x) {
        const int r = i / N, cc = i % N;
        const double zv = (r == 0 || cc == 0) ? 0.0 : A[i];
        G[i] = (float)(zv - rmean[r] - cmean[cc] + gmean);
    }
}

// Coarse pseudo-inverse for large coarsest levels (odd-sized chains such as the
// 25 x 25 x 1 bottom of a 100 x 100 x 1 grid, up to the 2048-vertex limit): the
// same in-place Gauss-Jordan as k_coarse_setup64, spread over the whole GPU --
// per pivot one tiny launch copies row/column p aside and one launch applies the
// rank-1 update to every entry (2 (n - 1) launches in the captured build graph,
// against O(n^3 / 1024) serial steps of the single-CTA kernel).
__global__ void k_cs_assemble(Geo g, const float* __restrict__ k, CoarseTemplate ct, double* __restrict__ A) {
    const int n = (int)g.n;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    double* row = A + (size_t)r * n;
    for (int c = 0; c < n; ++c) row[c] = 0.0;
    if (r == 0) return;                          // pinned vertex: zero row and column 0
    const int x = r / g.pl, rem = r - x * g.pl, y = rem / g.nz, z = rem - y * g.nz;
    for (int a = 0; a < 8; ++a) {
        const int ex = (x - (a & 1) + g.nx) % g.nx, ey = (y - ((a >> 1) & 1) + g.ny) % g.ny,
                  ez = (z - ((a >> 2) & 1) + g.nz) % g.nz;
        const double ke = (double)k[(ex * g.ny + ey) * g.nz + ez];
        for (int b = 0; b < 8; ++b) {
            const int cx = (ex + (b & 1)) % g.nx, cy = (ey + ((b >> 1) & 1)) % g.ny,
                      cz = (ez + ((b >> 2) & 1)) % g.nz;
            const int c = (cx * g.ny + cy) * g.nz + cz;
            if (c > 0) row[c] += ke * ct.kt[a ^ b];
        }
    }
}
// u = d * row p (u[p] = d), v = column p (v[p] = a_pp - 1), d = 1 / a_pp
__global__ void k_cs_pivot(const double* __restrict__ A, int n, int p, double* __restrict__ uv) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const double a = A[(size_t)p * n + p];
    if (t < n) uv[n + t] = t == p ? a - 1.0 : A[(size_t)t * n + p];
    else if (t < 2 * n) {
        const int c = t - n;
        uv[c] = c == p ? 1.0 / a : A[(size_t)p * n + c] / a;
    }
}
// A <- E - v u^T, E = A with column p replaced by e_p
__global__ void k_cs_update(double* __restrict__ A, int n, int p, const double* __restrict__ uv) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y * blockDim.y + threadIdx.y;
    if (r >= n || c >= n) return;
    const double e = c == p ? (r == p ? 1.0 : 0.0) : A[(size_t)r * n + c];
    A[(size_t)r * n + c] = fma(-uv[n + r], uv[c], e);
}
// row / column means of Z (the inverse, zero on the pinned row/column), then G = P Z P
__global__ void k_cs_means(const double* __restrict__ A, int n, double* __restrict__ means) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double sr = 0.0, sc = 0.0;
    for (int q = 1; q < n; ++q) {
        sr += t ? A[(size_t)t * n + q] : 0.0;
        sc += t ? A[(size_t)q * n + t] : 0.0;
    }
    means[t] = sr / n;
    means[n + t] = sc / n;
}
__global__ void k_cs_write(const double* __restrict__ A, int n, const double* __restrict__ means,
                           float* __restrict__ G) {
    __shared__ double gmean;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        double s = 0.0;
        for (int q = 0; q < n; ++q) s += means[q];
        gmean = s / n;
    }
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y * blockDim.y + threadIdx.y;
    if (r >= n || c >= n) return;
    const double z = (r == 0 || c == 0) ? 0.0 : A[(size_t)r * n + c];
    G[(size_t)r * n + c] = (float)(z - means[r] - means[n + c] + gmean);
}

// z = G f per case (coarse_solve, solver.py:307-324); one block.
__global__ void k_coarse_solve(int n, const float* __restrict__ G, const float* __restrict__ f,
                               float* __restrict__ z) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int i = w0; i < 3 * n; i += nw) {                      // one warp per row, G rows coalesced
        const int c = i / n, r = i - (i / n) * n;
        const float* fr = f + (size_t)c * n;
        float s = 0.f;
        for (int j = lane; j < n; j += 32) s += G[(size_t)r * n + j] * fr[j];
        s = warp_sum(s);
        if (lane == 0) z[i] = s;
    }
}

// ===========================================================================
// fp64 defect: r = f - K T on level 0 (solver.py:398-401) for the 3 cases.
// f comes from the macro loads of kappa (solver.py:347-363; f0 table in ct) or
// from an explicit field minus its mean.  Emits r as fp32 for the inner solve and
// the fixed-order sums ||r||^2, ||f||^2, sum(T) per case.
// ===========================================================================
template <bool EXPLICIT_F>
__global__ void __launch_bounds__(128) k_res64(Geo g, int xb, LevelTemplate lt, const double* __restrict__ kap,
                                               const double* __restrict__ T, const double* __restrict__ fext,
                                               const double* __restrict__ fmean, float* __restrict__ r32,
                                               double* partials, unsigned* counter, double* red_out,
                                               const int* __restrict__ skip) {
    if (skip && *skip) return;      // device-side solve control: the solve is already over
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = 0.0;
    if (t < g.pl) {
        const int y = t / g.nz, z = t - (t / g.nz) * g.nz;
        Nbr nb;
        nbr_init(nb, g, y, z);
        const int x0 = blockIdx.y * xb, x1 = min(g.nx, x0 + xb);
        for (int c = 0; c < 3; ++c) {
            const double* Tc = T + (size_t)c * g.n;
            double w[3][9], k[2][4];
            auto loadT = [&](double (&dst)[9], int x) {
                const long long po = plane_off(g, x);
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk) dst[j * 3 + kk] = __ldg(Tc + po + nb.ro[j] + nb.co[kk]);
            };
            auto loadK = [&](double (&dst)[4], int x) {
                const long long po = plane_off(g, x);
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) dst[j * 2 + kk] = __ldg(kap + po + nb.ro[j] + nb.co[kk]);
            };
            if (x0 < x1) {
                loadT(w[0], x0 - 1);
                loadT(w[1], x0);
                loadK(k[0], x0 - 1);
            }
            for (int x = x0; x < x1; ++x) {
                loadT(w[2], x + 1);
                loadK(k[1], x);
                double kt;
                if (lt.equal) {
                    const KSum<double> s = ksum<double>(k);
                    kt = apply_compact<double>(w, k, s, lt.s12);
                } else {
                    kt = apply_generic<double>(w, k, lt.kt);
                }
                const long long v = (long long)x * g.pl + t;
                double f;
                if (EXPLICIT_F) {
                    f = fext[(size_t)c * g.n + v];
                } else {
                    // reference order: sum over corners a = 0..7 of f0[a,c] * kappa[v - c_a]
                    f = 0.0;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        const int q = 1 - (a & 1), jj = 1 - ((a >> 1) & 1), kk = 1 - ((a >> 2) & 1);
                        f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + c], k[q][jj * 2 + kk]));
                    }
                }
                const double r = (f - fmean[c]) - kt;   // ||f|| before projection (solver.py:381)
                r32[(size_t)c * g.n + v] = (float)r;
                acc[c] += r * r;
                acc[3 + c] += f * f;
                acc[6 + c] += w[1][4];
#pragma unroll
                for (int i = 0; i < 9; ++i) { w[0][i] = w[1][i]; w[1][i] = w[2][i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i) k[0][i] = k[1][i];
            }
        }
    }
    reduce_finalize<9>(acc, partials, counter, red_out);
}

// Single-case fp64 K T (apply_K, solver.py:111-119) and macro load (solver.py:347-363).
__global__ void __launch_bounds__(128) k_apply64(Geo g, int xb, LevelTemplate lt, const double* __restrict__ kap,
                                                 const double* __restrict__ T, double* __restrict__ out,
                                                 int load_case) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.pl) return;
    const int y = t / g.nz, z = t - (t / g.nz) * g.nz;
    Nbr nb;
    nbr_init(nb, g, y, z);
    const int x0 = blockIdx.y * xb, x1 = min(g.nx, x0 + xb);
    double w[3][9], k[2][4];
    auto loadT = [&](double (&dst)[9], int x) {
        const long long po = plane_off(g, x);
        for (int j = 0; j < 3; ++j)
            for (int kk = 0; kk < 3; ++kk)
                dst[j * 3 + kk] = load_case < 0 ? __ldg(T + po + nb.ro[j] + nb.co[kk]) : 0.0;
    };
    auto loadK = [&](double (&dst)[4], int x) {
        const long long po = plane_off(g, x);
        for (int j = 0; j < 2; ++j)
            for (int kk = 0; kk < 2; ++kk) dst[j * 2 + kk] = __ldg(kap + po + nb.ro[j] + nb.co[kk]);
    };
    if (x0 < x1) {
        loadT(w[0], x0 - 1);
        loadT(w[1], x0);
        loadK(k[0], x0 - 1);
    }
    for (int x = x0; x < x1; ++x) {
        loadT(w[2], x + 1);
        loadK(k[1], x);
        const long long v = (long long)x * g.pl + t;
        if (load_case >= 0) {
            double f = 0.0;
            for (int a = 0; a < 8; ++a) {
                const int q = 1 - (a & 1), jj = 1 - ((a >> 1) & 1), kk = 1 - ((a >> 2) & 1);
                f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + load_case], k[q][jj * 2 + kk]));
            }
            out[v] = f;
        } else if (lt.equal) {
            const KSum<double> s = ksum<double>(k);
            out[v] = apply_compact<double>(w, k, s, lt.s12);
        } else {
            out[v] = apply_generic<double>(w, k, lt.kt);
        }
        for (int i = 0; i < 9; ++i) { w[0][i] = w[1][i]; w[1][i] = w[2][i]; }
        for (int i = 0; i < 4; ++i) k[0][i] = k[1][i];
    }
}

// Means of the three macro loads (solver.py:386-387 projects them out; they are
// round-off, but for a uniform medium round-off is all the load there is).
// One (y, z) column per thread marching x: the element factors of plane x - 1
// carry over (4 loads per vertex instead of 8, no per-vertex index division); each
// vertex's load is the fixed-order sum of its 8 element terms.
__global__ void __launch_bounds__(256) k_load_means_x(Geo g, int chunks, XRange xr, LevelTemplate lt,
                                                      const double* __restrict__ kap, double* partials,
                                                      unsigned* counter, double* out) {
    double v3[3] = {0.0, 0.0, 0.0};
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned cols = (unsigned)g.pl;
    if (t < cols * (unsigned)chunks) {
        const unsigned c = t / cols, r = t - c * cols;
        const unsigned y = r / (unsigned)g.nz, z = r - y * (unsigned)g.nz;
        const unsigned ym = y == 0 ? (unsigned)g.ny - 1 : y - 1, zm = z == 0 ? (unsigned)g.nz - 1 : z - 1;
        // slot (dy, dz) = element (y - dy, z - dz)
        const unsigned o[4] = {y * g.nz + z, y * g.nz + zm, ym * g.nz + z, ym * g.nz + zm};
        const int per = (xr.xb - xr.xa + chunks - 1) / chunks;
        const int x0 = xr.xa + (int)c * per, x1 = min(xr.xb, x0 + per);
        if (x0 < x1) {
            double P[4], Q[4];
            const unsigned pm = (unsigned)(x0 == 0 ? g.nx - 1 : x0 - 1) * cols;
#pragma unroll
            for (int k = 0; k < 4; ++k) P[k] = __ldg(kap + pm + o[k]);
            for (int x = x0; x < x1; ++x) {
                const unsigned po = (unsigned)x * cols;
#pragma unroll
                for (int k = 0; k < 4; ++k) Q[k] = __ldg(kap + po + o[k]);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    double f = 0.0;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {   // element v - c_a
                        const int slot = ((a >> 1) & 1) * 2 + ((a >> 2) & 1);
                        f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + cc], (a & 1) ? P[slot] : Q[slot]));
                    }
                    v3[cc] += f;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) P[k] = Q[k];
            }
        }
    }
    if (reduce_finalize<3>(v3, partials, counter, out)) {
        for (int c = 0; c < 3; ++c) out[c] /= xr.norm;
    }
}

// sum of each of 3 fields (mean projection of an explicit load, solver.py:386-387)
__global__ void k_sum3(long long n, const double* __restrict__ f, double* partials, unsigned* counter,
                       double* out) {
    double v3[3] = {0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        v3[0] += f[i];
        v3[1] += f[n + i];
        v3[2] += f[2 * n + i];
    }
    if (reduce_finalize<3>(v3, partials, counter, out)) {
        for (int c = 0; c < 3; ++c) out[c] /= (double)n;
    }
}

// ===========================================================================
// fp32 MG-PCG inner solver, 3 load cases per launch.
// ===========================================================================

// Operand sources for the stencil window.
struct SrcPlain {      // value = a[c*n + v]
    const float* a;
    long long n;
    __device__ __forceinline__ float operator()(int c, long long v) const { return __ldg(a + c * n + v); }
};
struct SrcJacobi0 {    // value = omega * dinv[v] * f[c*n + v]  (Jacobi sweep from zero)
    const float* f;
    const float* dinv;
    float omega;
    long long n;
    __device__ __forceinline__ float operator()(int c, long long v) const {
        return omega * __ldg(dinv + v) * __ldg(f + c * n + v);
    }
};

template <class Src, class Sink>
__device__ __forceinline__ void march3(const Geo& g, int xb, const LevelTemplate& lt, const float* __restrict__ kap,
                                       const Src& src, Sink& sink) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.pl) return;
    const int y = t / g.nz, z = t - (t / g.nz) * g.nz;
    Nbr nb;
    nbr_init(nb, g, y, z);
    const int x0 = blockIdx.y * xb, x1 = min(g.nx, x0 + xb);
    if (x0 >= x1) return;
    float w[3][3][9], k[2][4];
    auto loadT = [&](int slot, int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) w[c][slot][j * 3 + kk] = src(c, po + nb.ro[j] + nb.co[kk]);
    };
    auto loadK = [&](float (&dst)[4], int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) dst[j * 2 + kk] = __ldg(kap + po + nb.ro[j] + nb.co[kk]);
    };
    loadT(0, x0 - 1);
    loadT(1, x0);
    loadK(k[0], x0 - 1);
    for (int x = x0; x < x1; ++x) {
        loadT(2, x + 1);
        loadK(k[1], x);
        float kt[3], ctr[3];
        if (lt.equal) {
            const KSum<float> s = ksum<float>(k);
#pragma unroll
            for (int c = 0; c < 3; ++c) kt[c] = apply_compact<float>(w[c], k, s, (float)lt.s12);
        } else {
            float ktab[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) ktab[i] = (float)lt.kt[i];
#pragma unroll
            for (int c = 0; c < 3; ++c) kt[c] = apply_generic<float>(w[c], k, ktab);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) ctr[c] = w[c][1][4];
        sink((long long)x * g.pl + t, kt, ctr);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int i = 0; i < 9; ++i) { w[c][0][i] = w[c][1][i]; w[c][1][i] = w[c][2][i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i) k[0][i] = k[1][i];
    }
}

// Down-sweep smoother from zero + residual: z = w D^-1 f ; res = f - K z.
struct SinkSmoothRes {
    const float* f; float* z; float* res; long long n;
    __device__ __forceinline__ void operator()(long long v, const float (&kz)[3], const float (&zc)[3]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            z[c * n + v] = zc[c];
            res[c * n + v] = __ldg(f + c * n + v) - kz[c];
        }
    }
};
__global__ void __launch_bounds__(128) k_smooth_res(Geo g, int xb, LevelTemplate lt, const float* __restrict__ kap,
                                                    const float* __restrict__ f, const float* __restrict__ dinv,
                                                    float omega, float* __restrict__ z, float* __restrict__ res) {
    SrcJacobi0 src{f, dinv, omega, g.n};
    SinkSmoothRes sink{f, z, res, g.n};
    march3(g, xb, lt, kap, src, sink);
}

// Post-sweep: zout = z + w D^-1 (f - K z); optional fused r.zout partial sums (level 0).
template <bool DOT>
struct SinkJacobi {
    const float* f; const float* dinv; float* zout; float omega; long long n; double acc[3];
    __device__ __forceinline__ void operator()(long long v, const float (&kz)[3], const float (&zc)[3]) {
        const float di = __ldg(dinv + v);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float fv = __ldg(f + c * n + v);
            const float zn = zc[c] + omega * di * (fv - kz[c]);
            zout[c * n + v] = zn;
            if (DOT) acc[c] += (double)fv * (double)zn;
        }
    }
};
template <bool DOT>
__global__ void __launch_bounds__(128) k_jacobi(Geo g, int xb, LevelTemplate lt, const float* __restrict__ kap,
                                                const float* __restrict__ z, const float* __restrict__ f,
                                                const float* __restrict__ dinv, float omega, float* __restrict__ zout,
                                                double* partials, unsigned* counter, PcgScalars* sc) {
    SrcPlain src{z, g.n};
    SinkJacobi<DOT> sink{f, dinv, zout, omega, g.n, {0.0, 0.0, 0.0}};
    march3(g, xb, lt, kap, src, sink);
    if (DOT) {
        if (reduce_finalize<3>(sink.acc, partials, counter, sc->red)) {
            // beta = rz / rz_old (0 on the first inner iteration)
            for (int c = 0; c < 3; ++c) {
                const double rz = sc->red[c];
                sc->beta[c] = (sc->first || sc->rz[c] == 0.0) ? 0.0 : rz / sc->rz[c];
                sc->rz[c] = rz;
            }
            sc->first = 0;
        }
    }
}

// q = K p with fused p.q partial sums; alpha = rz / pq for active cases.
struct SinkSpmv {
    float* q; long long n; double acc[3];
    __device__ __forceinline__ void operator()(long long v, const float (&kp)[3], const float (&pc)[3]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            q[c * n + v] = kp[c];
            acc[c] += (double)pc[c] * (double)kp[c];
        }
    }
};
__global__ void __launch_bounds__(128) k_spmv(Geo g, int xb, LevelTemplate lt, const float* __restrict__ kap,
                                              const float* __restrict__ p, float* __restrict__ q, double* partials,
                                              unsigned* counter, PcgScalars* sc) {
    SrcPlain src{p, g.n};
    SinkSpmv sink{q, g.n, {0.0, 0.0, 0.0}};
    march3(g, xb, lt, kap, src, sink);
    if (reduce_finalize<3>(sink.acc, partials, counter, sc->red + 3)) {
        for (int c = 0; c < 3; ++c) {
            const double pq = sc->red[3 + c];
            sc->pq[c] = pq;
            sc->alpha[c] = (sc->active[c] != 0.0 && pq > 0.0) ? sc->rz[c] / pq : 0.0;
        }
    }
}

// p = z + beta p   (float4: n is a multiple of 4 on every level >= 4^3; scalar tail otherwise)
// p = z + beta p, with the previous iteration's d += alpha p folded in (k_upd no
// longer touches d: one read-modify-write pass less per PCG iteration; the last
// iteration's alpha p goes into T in k_Tupd)
__global__ void k_pupd(long long n, const float* __restrict__ z, float* __restrict__ p, float* __restrict__ d,
                       const PcgScalars* sc) {
    pdl_wait();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n4 = n >> 2;
    const float b[3] = {(float)sc->beta[0], (float)sc->beta[1], (float)sc->beta[2]};
    const float al[3] = {(float)sc->alpha[0], (float)sc->alpha[1], (float)sc->alpha[2]};
    if (sc->it == 0) {
        // first iteration of an inner solve: d = 0, p = z (the buffers hold the previous
        // solve's vectors, or nothing yet; this replaces two memsets per outer step)
        if (i < n4) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                reinterpret_cast<float4*>(p + c * n)[i] = __ldg(reinterpret_cast<const float4*>(z + c * n) + i);
                reinterpret_cast<float4*>(d + c * n)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const long long t = (n4 << 2) + i;
        if (i < (n & 3))
            for (int c = 0; c < 3; ++c) {
                p[c * n + t] = z[c * n + t];
                d[c * n + t] = 0.f;
            }
        return;
    }
    if (i < n4) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float4 zv = __ldg(reinterpret_cast<const float4*>(z + c * n) + i);
            float4* pp = reinterpret_cast<float4*>(p + c * n) + i;
            float4* dp = reinterpret_cast<float4*>(d + c * n) + i;
            const float4 pv = *pp;
            float4 dv = *dp;
            dv.x += al[c] * pv.x; dv.y += al[c] * pv.y; dv.z += al[c] * pv.z; dv.w += al[c] * pv.w;
            *dp = dv;
            *pp = make_float4(zv.x + b[c] * pv.x, zv.y + b[c] * pv.y, zv.z + b[c] * pv.z, zv.w + b[c] * pv.w);
        }
    }
    const long long t = (n4 << 2) + i;     // scalar tail
    if (i < (n & 3)) {
        for (int c = 0; c < 3; ++c) {
            d[c * n + t] += al[c] * p[c * n + t];
            p[c * n + t] = z[c * n + t] + b[c] * p[c * n + t];
        }
    }
}

// r -= alpha q ; r.r partial sums -> convergence flags (d is updated by the next k_pupd)
// GS: grid-stride over a capped grid (large fields: the per-block fence + atomic of
// the reduction epilogue, once per 256 float4, was a third of the kernel at 512^3)
template <bool GS>
__global__ void __launch_bounds__(256) k_upd(long long n, float* __restrict__ r, const float* __restrict__ q,
                                             double* partials, unsigned* counter, PcgScalars* sc,
                                             unsigned long long loop) {
    pdl_wait();
    double acc[3] = {0.0, 0.0, 0.0};
    const float al[3] = {(float)sc->alpha[0], (float)sc->alpha[1], (float)sc->alpha[2]};
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n4 = n >> 2;
    auto body = [&](long long j) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float4 qv = __ldg(reinterpret_cast<const float4*>(q + c * n) + j);
            float4* rp = reinterpret_cast<float4*>(r + c * n) + j;
            float4 rv = *rp;
            rv.x -= al[c] * qv.x; rv.y -= al[c] * qv.y; rv.z -= al[c] * qv.z; rv.w -= al[c] * qv.w;
            *rp = rv;
            acc[c] += ((double)rv.x * rv.x + (double)rv.y * rv.y) + ((double)rv.z * rv.z + (double)rv.w * rv.w);
        }
    };
    if constexpr (GS) {
        for (long long j = i; j < n4; j += (long long)gridDim.x * blockDim.x) body(j);
    } else {
        if (i < n4) body(i);
    }
    if (i < (n & 3)) {
        const long long t = (n4 << 2) + i;
        for (int c = 0; c < 3; ++c) {
            const float rn = r[c * n + t] - al[c] * q[c * n + t];
            r[c * n + t] = rn;
            acc[c] += (double)rn * rn;
        }
    }
    if (reduce_finalize<3>(acc, partials, counter, sc->red + 6)) {
        bool was[3];
        for (int c = 0; c < 3; ++c) {
            was[c] = sc->active[c] != 0.0;
            sc->rr[c] = sc->red[6 + c];
            if (was[c] && sc->rr[c] <= sc->target2[c]) sc->active[c] = 0.0;
            // fp32 breakdown guard: a recursive residual 10x above its minimum in this
            // loop means the fp32 recurrences have lost the preconditioned operator's
            // positivity (seen on thin, high-contrast 2-D designs at tol 1e-8); the case
            // stops and the outer fp64 step restarts it from the true residual
            else if (was[c] && sc->rr_min[c] > 0.0 && sc->rr[c] > 100.0 * sc->rr_min[c]) sc->active[c] = 0.0;
            if (was[c]) sc->rr_min[c] = sc->rr_min[c] > 0.0 ? fmin(sc->rr_min[c], sc->rr[c]) : sc->rr[c];
            sc->flags[c] = sc->active[c];
        }
        sc->flags[3] = sc->rr[0];
        sc->flags[4] = sc->rr[1];
        sc->flags[5] = sc->rr[2];
        if (sc->hist && sc->hcount < sc->hcap) {
            for (int c = 0; c < 3; ++c) sc->hist[3 * sc->hcount + c] = was[c] ? sc->rr[c] : -1.0;
            sc->hcount += 1;
        }
        // the inner-loop control: count the preconditioner applications (in total and
        // per case), decide whether the WHILE node runs again; every case has its own
        // budget of max_cycles V-cycles (homogenize.py:85-90)
        int nact = 0, worst = 0;
        for (int c = 0; c < 3; ++c) {
            sc->ccyc[c] += was[c];
            if (sc->active[c] != 0.0) {
                ++nact;
                worst = max(worst, sc->ccyc[c]);
            }
        }
        sc->cycles += sc->nact;
        sc->nact = nact;
        sc->it += 1;
        if (loop) {
            const bool more = nact > 0 && sc->it < sc->max_it && worst < sc->max_cycles;
            cudaGraphSetConditional((cudaGraphConditionalHandle)loop, more ? 1u : 0u);
        }
    }
}

// Prolongation, every axis coarsened, one thread per coarse vertex (X,Y,Z) and case:
// it owns the fine block (2X..2X+1, 2Y..2Y+1, 2Z..2Z+1), whose trilinear values
// only involve the coarse corners X..X+1 x Y..Y+1 x Z..Z+1 (8 loads per 8 fine
// vertices), and updates it with 4 float2 read-modify-writes.
// loads of data written earlier in the same (cooperative) kernel must bypass L1
template <bool CG>
__device__ __forceinline__ float ldf(const float* p) { return CG ? __ldcg(p) : __ldg(p); }

// (case, vertex) of a flat 3-case item index: 32-bit division when 3 n fits
__device__ __forceinline__ void split_case(long long i, long long n, int& c, int& v) {
    if (3 * n < (1LL << 31)) {
        const unsigned ui = (unsigned)i, un = (unsigned)n;
        c = (int)(ui / un);
        v = (int)(ui - (unsigned)c * un);
    } else {
        c = (int)(i / n);
        v = (int)(i - (long long)c * n);
    }
}

template <bool CG, bool ASSIGN = false>
__device__ __forceinline__ void prolong3b_at(const Geo& f, const Geo& c, const float* __restrict__ zc,
                                             float* __restrict__ zf, int cc, int X, int Y, int Z);

template <bool CG, bool ASSIGN = false>
__device__ __forceinline__ void prolong3b_body(const Geo& f, const Geo& c, const float* __restrict__ zc,
                                               float* __restrict__ zf, long long i) {
    int cc, v;
    split_case(i, c.n, cc, v);
    const int X = v / c.pl, rem = v - X * c.pl, Y = rem / c.nz, Z = rem - Y * c.nz;
    prolong3b_at<CG, ASSIGN>(f, c, zc, zf, cc, X, Y, Z);
}

// the 2x2x2 fine block of coarse vertex (X, Y, Z) of case cc
template <bool CG, bool ASSIGN>
__device__ __forceinline__ void prolong3b_at(const Geo& f, const Geo& c, const float* __restrict__ zc,
                                             float* __restrict__ zf, int cc, int X, int Y, int Z) {
    const int X1 = X + 1 == c.nx ? 0 : X + 1, Y1 = Y + 1 == c.ny ? 0 : Y + 1, Z1 = Z + 1 == c.nz ? 0 : Z + 1;
    const float* a = zc + (size_t)cc * c.n;
    float q[2][2][2];
    const int xs[2] = {X, X1}, ys[2] = {Y, Y1}, zs[2] = {Z, Z1};
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) q[p][j][k] = ldf<CG>(a + (long long)xs[p] * c.pl + ys[j] * c.nz + zs[k]);
    // interpolate along z: even fine z -> q0, odd -> (q0 + q1)/2
    float qz[2][2][2];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 2; ++j) { qz[p][j][0] = q[p][j][0]; qz[p][j][1] = 0.5f * (q[p][j][0] + q[p][j][1]); }
    float* out = zf + (size_t)cc * f.n;
#pragma unroll
    for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
            float2 add;
            // along y then x
            float vz0, vz1;
            {
                const float y00 = b2 ? 0.5f * (qz[0][0][0] + qz[0][1][0]) : qz[0][0][0];
                const float y01 = b2 ? 0.5f * (qz[0][0][1] + qz[0][1][1]) : qz[0][0][1];
                const float y10 = b2 ? 0.5f * (qz[1][0][0] + qz[1][1][0]) : qz[1][0][0];
                const float y11 = b2 ? 0.5f * (qz[1][0][1] + qz[1][1][1]) : qz[1][0][1];
                vz0 = a2 ? 0.5f * (y00 + y10) : y00;
                vz1 = a2 ? 0.5f * (y01 + y11) : y01;
            }
            add = make_float2(vz0, vz1);
            float2* dst = reinterpret_cast<float2*>(out + (long long)(2 * X + a2) * f.pl + (2 * Y + b2) * f.nz + 2 * Z);
            if (ASSIGN) {
                *dst = add;                       // z = P zc (the k10 legs recompute z0 on the fly)
            } else {
                float2 cur = CG ? __ldcg(dst) : *dst;
                cur.x += add.x;
                cur.y += add.y;
                *dst = cur;
            }
        }
}

template <bool ASSIGN>
__global__ void __launch_bounds__(256) k_prolong3b(Geo f, Geo c, const float* __restrict__ zc,
                                                   float* __restrict__ zf) {
    pdl_wait();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * c.n) return;
    prolong3b_body<false, ASSIGN>(f, c, zc, zf, i);
}

// the same on a (Y, Z) x (case, X) grid: 32-bit index arithmetic, no division by n
template <bool ASSIGN>
__global__ void __launch_bounds__(256) k_prolong3c(Geo f, Geo c, const float* __restrict__ zc,
                                                   float* __restrict__ zf) {
    pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= c.pl) return;
    const int cc = blockIdx.y / c.nx, X = blockIdx.y - cc * c.nx;
    const int Y = t / c.nz, Z = t - Y * c.nz;
    prolong3b_at<false, ASSIGN>(f, c, zc, zf, cc, X, Y, Z);
}

// ---- small levels: one thread per (case, vertex), every load issued up front ----
// one (case, vertex) item of the small-level smoother (OP 0: smooth_res, OP 1: jacobi)
template <int OP, bool DOT, bool CG>
__device__ __forceinline__ void small_item(const Geo& g, const LevelTemplate& lt, const float* __restrict__ kap,
                                           const float* __restrict__ a, const float* __restrict__ f,
                                           const float* __restrict__ dinv, float omega, float* __restrict__ o1,
                                           float* __restrict__ o2, long long i, double (&dot3)[3]) {
    int c, v;
    split_case(i, g.n, c, v);
    const int x = v / g.pl, rem = v - x * g.pl, y = rem / g.nz, z = rem - y * g.nz;
    const int xs[3] = {wrap_m(x, g.nx), x, wrap_p(x, g.nx)};
    const int ys[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
    const int zs[3] = {wrap_m(z, g.nz), z, wrap_p(z, g.nz)};
    const float* src = (OP == 0 ? f : a) + (size_t)c * g.n;
    float t[3][9], k[2][4];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int idx = xs[p] * g.pl + ys[j] + zs[q];
                float val = ldf<CG>(src + idx);
                if (OP == 0) val *= omega * ldf<CG>(dinv + idx);
                t[p][j * 3 + q] = val;
            }
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) k[p][j * 2 + q] = ldf<CG>(kap + xs[p] * g.pl + ys[j] + zs[q]);
    float kt;
    if (lt.equal) {
        const KSum<float> s = ksum<float>(k);
        kt = apply_compact<float>(t, k, s, (float)lt.s12);
    } else {
        float ktab[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) ktab[q] = (float)lt.kt[q];
        kt = apply_generic<float>(t, k, ktab);
    }
    const float fv = ldf<CG>(f + (size_t)c * g.n + v);
    if (OP == 0) {
        o1[(size_t)c * g.n + v] = t[1][4];
        o2[(size_t)c * g.n + v] = fv - kt;
    } else {
        const float zn = t[1][4] + omega * ldf<CG>(dinv + v) * (fv - kt);
        o1[(size_t)c * g.n + v] = zn;
        if (DOT) dot3[c] = (double)fv * (double)zn;
    }
}

template <int OP, bool DOT>
__global__ void __launch_bounds__(256) k_small(Geo g, LevelTemplate lt, const float* __restrict__ kap,
                                               const float* __restrict__ a, const float* __restrict__ f,
                                               const float* __restrict__ dinv, float omega, float* __restrict__ o1,
                                               float* __restrict__ o2, double* partials, unsigned* counter,
                                               PcgScalars* sc) {
    pdl_wait();
    // OP 0: smooth_res  (operand w D^-1 f; o1 = z0, o2 = f - K z0)
    // OP 1: jacobi      (operand a = z;    o1 = z + w D^-1 (f - K z); DOT: r.z -> beta)
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double dot3[3] = {0.0, 0.0, 0.0};
    if (i < 3 * g.n) small_item<OP, DOT, false>(g, lt, kap, a, f, dinv, omega, o1, o2, i, dot3);
    if (DOT) {
        if (reduce_finalize<3>(dot3, partials, counter, sc->red)) {
            for (int cc = 0; cc < 3; ++cc) {
                const double rz = sc->red[cc];
                sc->beta[cc] = (sc->first || sc->rz[cc] == 0.0) ? 0.0 : rz / sc->rz[cc];
                sc->rz[cc] = rz;
            }
            sc->first = 0;
        }
    }
}

// restriction with every axis coarsened (3-D levels): unrolled 27-point gather
template <bool CG>
__device__ __forceinline__ void restrict3_body(const Geo& f, const Geo& c, const float* __restrict__ res,
                                               float* __restrict__ fc, long long i) {
    int cc, v;
    split_case(i, c.n, cc, v);
    const int X = v / c.pl, rem = v - X * c.pl, Y = rem / c.nz, Z = rem - Y * c.nz;
    const int xs[3] = {wrap_m(2 * X, f.nx), 2 * X, wrap_p(2 * X, f.nx)};
    const int ys[3] = {wrap_m(2 * Y, f.ny) * f.nz, 2 * Y * f.nz, wrap_p(2 * Y, f.ny) * f.nz};
    const int zs[3] = {wrap_m(2 * Z, f.nz), 2 * Z, wrap_p(2 * Z, f.nz)};
    const float w[3] = {0.25f, 0.5f, 0.25f};
    const float* r = res + (size_t)cc * f.n;
    float vals[27];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int d = 0; d < 3; ++d) vals[(a * 3 + b) * 3 + d] = ldf<CG>(r + (long long)xs[a] * f.pl + ys[b] + zs[d]);
    float s = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float sb = 0.f;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const float sz = w[0] * vals[(a * 3 + b) * 3] + w[1] * vals[(a * 3 + b) * 3 + 1] + w[2] * vals[(a * 3 + b) * 3 + 2];
            sb += w[b] * sz;
        }
        s += w[a] * sb;
    }
    fc[i] = s;
}

__global__ void __launch_bounds__(256) k_restrict3(Geo f, Geo c, const float* __restrict__ res,
                                                   float* __restrict__ fc) {
    pdl_wait();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * c.n) return;
    restrict3_body<false>(f, c, res, fc, i);
}

// Restriction for coarse levels with c.nz % 32 == 0: a warp covers 32 consecutive
// coarse z, so each fine row (2Z, 2Z+1) is one coalesced float2 load per lane and
// the 2Z-1 neighbour comes from the lane below by a shuffle (lane 0 loads it).
// Same weights and summation order as k_restrict3.
__global__ void __launch_bounds__(256) k_restrict3w(Geo f, Geo c, const float* __restrict__ res,
                                                    float* __restrict__ fc) {
    pdl_wait();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * c.n) return;                      // c.n % 32 == 0: whole warps only
    const int lane = threadIdx.x & 31;
    int cc, v;
    split_case(i, c.n, cc, v);
    const int X = v / c.pl, rem = v - X * c.pl, Y = rem / c.nz, Z = rem - Y * c.nz;
    const int xs[3] = {wrap_m(2 * X, f.nx), 2 * X, wrap_p(2 * X, f.nx)};
    const int ys[3] = {wrap_m(2 * Y, f.ny) * f.nz, 2 * Y * f.nz, wrap_p(2 * Y, f.ny) * f.nz};
    const int zm = wrap_m(2 * Z, f.nz);
    const float w[3] = {0.25f, 0.5f, 0.25f};
    const float* r = res + (size_t)cc * f.n;
    float s = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float sb = 0.f;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const float* row = r + (long long)xs[a] * f.pl + ys[b];
            const float2 m = __ldg(reinterpret_cast<const float2*>(row + 2 * Z));
            float left = __shfl_up_sync(0xffffffffu, m.y, 1);
            if (lane == 0) left = __ldg(row + zm);
            const float sz = w[0] * left + w[1] * m.x + w[2] * m.y;
            sb += w[b] * sz;
        }
        s += w[a] * sb;
    }
    fc[i] = s;
}

// Restriction for coarse rows with c.nz % 64 == 0: a thread makes two
// consecutive coarse z (one float4 of fine z per row, the 4Z-1 neighbour from the lane
// below), grid (Y, Z pair) x (case, X): no 64-bit index division, half the load
// instructions per output.  Same weights and summation order as k_restrict3w.
__global__ void __launch_bounds__(256) k_restrict3v(Geo f, Geo c, const float* __restrict__ res,
                                                    float* __restrict__ fc) {
    pdl_wait();
    const int hz = c.nz >> 1;                       // coarse z pairs per row
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= c.ny * hz) return;                     // hz % 32 == 0: whole warps only
    const int lane = threadIdx.x & 31;
    const int cc = blockIdx.y / c.nx, X = blockIdx.y - cc * c.nx;
    const int Y = t / hz, Zp = t - Y * hz;
    const int xs[3] = {wrap_m(2 * X, f.nx), 2 * X, wrap_p(2 * X, f.nx)};
    const int ys[3] = {wrap_m(2 * Y, f.ny) * f.nz, 2 * Y * f.nz, wrap_p(2 * Y, f.ny) * f.nz};
    const int z4 = 4 * Zp;
    const int zm = z4 == 0 ? f.nz - 1 : z4 - 1;
    const float w[3] = {0.25f, 0.5f, 0.25f};
    const float* r = res + (size_t)cc * f.n;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float sb0 = 0.f, sb1 = 0.f;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const float* row = r + (size_t)xs[a] * f.pl + ys[b];
            const float4 m = __ldg(reinterpret_cast<const float4*>(row + z4));
            float left = __shfl_up_sync(0xffffffffu, m.w, 1);
            if (lane == 0) left = __ldg(row + zm);
            const float sz0 = w[0] * left + w[1] * m.x + w[2] * m.y;
            const float sz1 = w[0] * m.y + w[1] * m.z + w[2] * m.w;
            sb0 += w[b] * sz0;
            sb1 += w[b] * sz1;
        }
        s0 += w[a] * sb0;
        s1 += w[a] * sb1;
    }
    *reinterpret_cast<float2*>(fc + (size_t)cc * c.n + (size_t)X * c.pl + Y * c.nz + 2 * Zp) = make_float2(s0, s1);
}

// full-weighting restriction (solver.py:167-177): coarse J <- sum_d w(d) res[2J+d]
__global__ void k_restrict(Geo f, Geo c, int cx, int cy, int cz, const float* __restrict__ res,
                           float* __restrict__ fc) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= c.n) return;
    const int X = (int)(v / c.pl), rem = (int)(v - (long long)X * c.pl);
    const int Y = rem / c.nz, Z = rem - Y * c.nz;
    int xs[3], ys[3], zs[3];
    float wx[3], wy[3], wz[3];
    int nxs = 1, nys = 1, nzs = 1;
    if (cx) { xs[0] = wrap_m(2 * X, f.nx); xs[1] = 2 * X; xs[2] = wrap_p(2 * X, f.nx); wx[0] = .25f; wx[1] = .5f; wx[2] = .25f; nxs = 3; }
    else { xs[0] = X; wx[0] = 1.f; }
    if (cy) { ys[0] = wrap_m(2 * Y, f.ny); ys[1] = 2 * Y; ys[2] = wrap_p(2 * Y, f.ny); wy[0] = .25f; wy[1] = .5f; wy[2] = .25f; nys = 3; }
    else { ys[0] = Y; wy[0] = 1.f; }
    if (cz) { zs[0] = wrap_m(2 * Z, f.nz); zs[1] = 2 * Z; zs[2] = wrap_p(2 * Z, f.nz); wz[0] = .25f; wz[1] = .5f; wz[2] = .25f; nzs = 3; }
    else { zs[0] = Z; wz[0] = 1.f; }
    for (int cc = 0; cc < 3; ++cc) {
        const float* r = res + (size_t)cc * f.n;
        float s = 0.f;
        for (int a = 0; a < nxs; ++a)
            for (int b = 0; b < nys; ++b) {
                const long long row = ((long long)xs[a] * f.ny + ys[b]) * f.nz;
                float sz = 0.f;
                for (int d = 0; d < nzs; ++d) sz += wz[d] * r[row + zs[d]];
                s += wx[a] * wy[b] * sz;
            }
        fc[(size_t)cc * c.n + v] = s;
    }
}

// trilinear prolongation + correction (solver.py:180-200): z_f += P z_c
__global__ void k_prolong(Geo f, Geo c, int cx, int cy, int cz, const float* __restrict__ zc,
                          float* __restrict__ zf) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= f.n) return;
    const int x = (int)(v / f.pl), rem = (int)(v - (long long)x * f.pl);
    const int y = rem / f.nz, z = rem - y * f.nz;
    int xs[2], ys[2], zs[2];
    float wx[2], wy[2], wz[2];
    int nxs, nys, nzs;
    auto axis = [](int i, int coars, int nc, int* idx, float* w, int& cnt) {
        if (!coars) { idx[0] = i; w[0] = 1.f; cnt = 1; return; }
        const int J = i >> 1;
        if (i & 1) { idx[0] = J; idx[1] = J + 1 == nc ? 0 : J + 1; w[0] = .5f; w[1] = .5f; cnt = 2; }
        else { idx[0] = J; w[0] = 1.f; cnt = 1; }
    };
    axis(x, cx, c.nx, xs, wx, nxs);
    axis(y, cy, c.ny, ys, wy, nys);
    axis(z, cz, c.nz, zs, wz, nzs);
    for (int cc = 0; cc < 3; ++cc) {
        const float* a = zc + (size_t)cc * c.n;
        float s = 0.f;
        for (int i = 0; i < nxs; ++i)
            for (int j = 0; j < nys; ++j)
                for (int k = 0; k < nzs; ++k)
                    s += wx[i] * wy[j] * wz[k] * a[((long long)xs[i] * c.ny + ys[j]) * c.nz + zs[k]];
        zf[(size_t)cc * f.n + v] += s;
    }
}

// Warm-start extrapolation across design iterations: T <- T + theta (T - T_prev), T_prev <- T.
__global__ void k_Tupd(long long n, double* __restrict__ T, const float* __restrict__ d, const float* __restrict__ p,
                       const PcgScalars* __restrict__ sc) {
    if (sc->skip) return;           // device-side solve control: no inner loop ran
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const int c = (int)(i / n);
    T[i] += (double)(d[i] + (float)sc->alpha[c] * p[i]);
}

// T -= mean per case, means given
__global__ void k_submean_means(long long n, double* __restrict__ T, const double* __restrict__ means) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    T[i] -= means[i / n];
}

// T -= mean(T) per case (solver.py:398)
__global__ void k_submean(long long n, double* __restrict__ T, const double* __restrict__ sumT) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const int c = (int)(i / n);
    T[i] -= sumT[c] / (double)n;
}

// ===========================================================================
// Homogenized tensor + sensitivities (homogenize.py:94-160)
// ===========================================================================

// Per element e: w_i[a] = c_a[i] - T_i[e + c_a]; E_c = w_i . K0 w_j for the packed
// pairs (00,11,22,01,12,02).  K0 w = (5 w + N1 w - sum w) / 12.
__device__ __forceinline__ void element_energies(const Geo& g, long long e, const double* __restrict__ T,
                                                 double (&E)[6]) {
    // 32-bit index arithmetic (every field here has < 2^31 vertices): the 64-bit
    // divisions and per-corner 64-bit products were a third of the kernel's instructions
    const unsigned ue = (unsigned)e, upl = (unsigned)g.pl, unz = (unsigned)g.nz;
    const unsigned x = ue / upl, rem = ue - x * upl;
    const unsigned y = rem / unz, z = rem - y * unz;
    const unsigned xp = x + 1 == (unsigned)g.nx ? 0u : x + 1, yp = y + 1 == (unsigned)g.ny ? 0u : y + 1,
                   zp = z + 1 == unz ? 0u : z + 1;
    const unsigned ox[2] = {x * upl, xp * upl}, oy[2] = {y * unz, yp * unz}, oz[2] = {z, zp};
    unsigned vid[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) vid[a] = ox[a & 1] + oy[(a >> 1) & 1] + oz[(a >> 2) & 1];
    double w[3][8], kw[3][8];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double* Ti = T + (size_t)i * g.n;
        double sum = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            w[i][a] = (double)((a >> i) & 1) - __ldg(Ti + vid[a]);
            sum += w[i][a];
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
            kw[i][a] = (5.0 * w[i][a] + w[i][a ^ 1] + w[i][a ^ 2] + w[i][a ^ 4] - sum) * (1.0 / 12.0);
    }
    const int pi[6] = {0, 1, 2, 0, 1, 0}, pj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int c = 0; c < 6; ++c) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) s += w[pi[c]][a] * kw[pj[c]][a];
        E[c] = s;
    }
}

__global__ void k_pair_energy(Geo g, const double* __restrict__ T, double* __restrict__ Eout) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.n) return;
    double E[6];
    element_energies(g, e, T, E);
    for (int c = 0; c < 6; ++c) Eout[(size_t)c * g.n + e] = E[c];
}


// ---- x-marching form (the design-loop path) ---------------------------------
// In the Walsh-Hadamard basis of the 8 corners (chi_s(a) = (-1)^popcount(s & a))
// the element matrix is diagonal: K0 = (5 I + N1 - J) / 12 has eigenvalue 0 on
// s = 0 and 1/2, 1/3, 1/6 on popcount(s) = 1, 2, 3.  So with what_i = H w_i,
//   E_ij = w_i . K0 w_j = (1/8) sum_s mu_s what_i[s] what_j[s]:
// a 24-add butterfly per case and 7 products per pair instead of the 8 x 8 form.
// w_i = c_i - T_i, and H c_i is 4 on s = 0 and -4 on s = 2^i (zero elsewhere).
// A thread owns one (y, z) column and marches a chunk of x planes, carrying the
// 4 corners of plane x (3 cases) from the previous step: 12 loads per element
// instead of 24, and no per-element index division.
struct MarchCol {
    unsigned o00, o01, o10, o11;     // in-plane offsets of (y,z), (y,z+1), (y+1,z), (y+1,z+1)
};

__device__ __forceinline__ void load_plane(const double* __restrict__ T, long long n, unsigned po, const MarchCol& q,
                                           double (&P)[3][4]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double* Ti = T + (size_t)i * n + po;
        P[i][0] = __ldg(Ti + q.o00);
        P[i][1] = __ldg(Ti + q.o01);
        P[i][2] = __ldg(Ti + q.o10);
        P[i][3] = __ldg(Ti + q.o11);
    }
}

// energies of the element between planes A (x) and B (x + 1); corner a = (a&1: x,
// a&2: y, a&4: z) -> plane (a & 1), in-plane slot ((a >> 1) & 1) * 2 + ((a >> 2) & 1)
__device__ __forceinline__ void energies_wht(const double (&A)[3][4], const double (&B)[3][4], double (&E)[6]) {
    double u[3][8];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double v[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int slot = ((a >> 1) & 1) * 2 + ((a >> 2) & 1);
            v[a] = -((a & 1) ? B[i][slot] : A[i][slot]);      // -T (c_i added in the spectrum)
        }
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
            for (int a = 0; a < 8; ++a)
                if (!(a & h)) {
                    const double p = v[a], q = v[a | h];
                    v[a] = p + q;
                    v[a | h] = p - q;
                }
        v[1 << i] -= 4.0;                                      // + H c_i (the s = 0 term drops)
        // scale by sqrt(mu_s / 8): mu = 1/2, 1/3, 1/6 for popcount 1, 2, 3
        const double r1 = 0.25, r2 = 0.2041241452319315, r3 = 0.14433756729740643;
        u[i][1] = v[1] * r1; u[i][2] = v[2] * r1; u[i][4] = v[4] * r1;
        u[i][3] = v[3] * r2; u[i][5] = v[5] * r2; u[i][6] = v[6] * r2;
        u[i][7] = v[7] * r3;
    }
    const int pi[6] = {0, 1, 2, 0, 1, 0}, pj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int c = 0; c < 6; ++c) {
        double s = 0.0;
#pragma unroll
        for (int t = 1; t < 8; ++t) s = fma(u[pi[c]][t], u[pj[c]][t], s);
        E[c] = s;
    }
}

// one (y, z) column and a chunk [x0, x1) of planes per thread
__device__ __forceinline__ bool march_setup(const Geo& g, int chunks, int xa, int xb, MarchCol& q, int& x0,
                                            int& x1) {
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned cols = (unsigned)g.pl;
    if (t >= cols * (unsigned)chunks) return false;
    const unsigned c = t / cols, r = t - c * cols;
    const unsigned y = r / (unsigned)g.nz, z = r - y * (unsigned)g.nz;
    const unsigned yp = y + 1 == (unsigned)g.ny ? 0u : y + 1, zp = z + 1 == (unsigned)g.nz ? 0u : z + 1;
    q.o00 = y * g.nz + z;
    q.o01 = y * g.nz + zp;
    q.o10 = yp * g.nz + z;
    q.o11 = yp * g.nz + zp;
    const int per = (xb - xa + chunks - 1) / chunks;
    x0 = xa + (int)c * per;
    x1 = min(xb, x0 + per);
    return x0 < x1;
}

__global__ void __launch_bounds__(256) k_tensor_x(Geo g, int chunks, XRange xr, const double* __restrict__ T,
                                                  const double* __restrict__ kap, double* partials, unsigned* counter,
                                                  double* out) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    MarchCol q;
    int x0, x1;
    if (march_setup(g, chunks, xr.xa, xr.xb, q, x0, x1)) {
        // planes x and x + 1 in registers, plane x + 2 prefetched while x is consumed
        double A[3][4], B[3][4], Cn[3][4];
        load_plane(T, g.n, (unsigned)x0 * (unsigned)g.pl, q, A);
        load_plane(T, g.n, (unsigned)(x0 + 1 == g.nx ? 0 : x0 + 1) * (unsigned)g.pl, q, B);
        for (int x = x0; x < x1; ++x) {
            if (x + 1 < x1) {
                const int xn = x + 2 >= g.nx ? x + 2 - g.nx : x + 2;
                load_plane(T, g.n, (unsigned)xn * (unsigned)g.pl, q, Cn);
            }
            const double k = __ldg(kap + (unsigned)x * (unsigned)g.pl + q.o00);
            double E[6];
            energies_wht(A, B, E);
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[c] = fma(k, E[c], acc[c]);
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    A[i][s] = B[i][s];
                    B[i][s] = Cn[i][s];
                }
        }
    }
    if (reduce_finalize<6>(acc, partials, counter, out)) {
        for (int c = 0; c < 6; ++c) out[c] /= xr.norm;
    }
}

__global__ void __launch_bounds__(256) k_sens_x(Geo g, int chunks, XRange xr, const double* __restrict__ T,
                                                const double* __restrict__ rf, SimpParams sp, Dg dG,
                                                const Dg* __restrict__ dG_dev, double* __restrict__ sens) {
    MarchCol q;
    int x0, x1;
    if (!march_setup(g, chunks, xr.xa, xr.xb, q, x0, x1)) return;
    if (dG_dev) dG = *dG_dev;               // objective weights computed on the device (otm_loop.cu)
    double A[3][4], B[3][4], Cn[3][4];
    load_plane(T, g.n, (unsigned)x0 * (unsigned)g.pl, q, A);
    load_plane(T, g.n, (unsigned)(x0 + 1 == g.nx ? 0 : x0 + 1) * (unsigned)g.pl, q, B);
    const double scale = (sp.k0 - sp.kmin) * sp.p / xr.norm;
    for (int x = x0; x < x1; ++x) {
        if (x + 1 < x1) {
            const int xn = x + 2 >= g.nx ? x + 2 - g.nx : x + 2;
            load_plane(T, g.n, (unsigned)xn * (unsigned)g.pl, q, Cn);
        }
        const unsigned e = (unsigned)x * (unsigned)g.pl + q.o00;
        const double rfe = __ldg(rf + e);
        double E[6];
        energies_wht(A, B, E);
        double con = 0.0;
#pragma unroll
        for (int c = 0; c < 6; ++c) con = fma(dG.v[c], E[c], con);
        sens[e] = simp_pow(rfe, sp.p - 1.0) * scale * con;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                A[i][s] = B[i][s];
                B[i][s] = Cn[i][s];
            }
    }
}

// ===========================================================================
// OC update (optimize.py:114-160)
// ===========================================================================
// Bisection passes: mean of the candidate field for up to kOcLam multipliers per
// launch.  The candidate clip(rho * max(desc/lam, 1e-10)^damp, lo, hi) is evaluated
// as clip(max(c_e * lam^-damp, rho * 1e-10^damp), lo, hi) with c_e = rho * desc^damp:
// a few ulps from the reference's expression, which only matters for the means the
// host compares against the bound; the final density is written by k_oc_apply with
// the reference's exact expression.  lams[k] == 0 encodes the lam -> 0 "free" step.
__global__ void __launch_bounds__(256, 2) k_oc_eval(long long n, const double* __restrict__ rho,
                                                    const double* __restrict__ sens, const OcArgs a, int nlam,
                                                    const LamSet lam_pow, double* partials, unsigned* counter,
                                                    double* out) {
    static_assert(kOcLam == 32, "reduce_finalize32 assumes 32 multipliers per pass");
    double acc[kOcLam];
#pragma unroll
    for (int k = 0; k < kOcLam; ++k) acc[k] = 0.0;
    const double M = (double)n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double r = __ldg(rho + i);
        const double desc = M * (-__ldg(sens + i));
        const double lo = fmax(r - a.step, a.rmin), hi = fmin(r + a.step, 1.0);
        const double lof = fmax(lo, r * a.floor_ratio);      // clip(max(x, floor), lo, hi) = min(max(x, lof), hi)
        const double ce = desc > 0.0 ? r * (a.sqrt_damp ? sqrt(desc) : pow(desc, a.damp)) : 0.0;
        const double freev = desc > 0.0 ? hi : (desc < 0.0 ? lo : r);
#pragma unroll
        for (int k = 0; k < kOcLam; ++k) {
            const double lp = lam_pow.v[k];   // lam^-damp, or 0 for the free step
            const double cand = lp == 0.0 ? freev : fmin(fmax(ce * lp, lof), hi);
            acc[k] += k < nlam ? cand : 0.0;
        }
    }
    if (reduce_finalize32(acc, partials, counter, out)) {
        for (int k = 0; k < kOcLam; ++k) out[k] /= M;
    }
}

// The whole oc_update (optimize.py:114-160) in one cooperative launch.  Every
// pass evaluates the candidate means of up to 32 multipliers (as k_oc_eval);
// between passes, thread 0 of block 0 replays the reference's sequential search
// (free step, bracket l2 *= 4, bisection of [1e-30, l2] with its two stopping
// rules) over the evaluated means, exactly as the host version did, and picks the
// next multipliers.  Then the density is written with the exact expression and,
// if nothing changed and a retry bound is set (optimize.py:355-362), the search
// reruns once with that bound.
__device__ double oc_lam_pow(const OcArgs& a, double lam) {
    return a.sqrt_damp ? 1.0 / sqrt(lam) : pow(lam, -a.damp);
}

// First pass: the free step and bracket values 4^0, 4^1, ... (optimize.py:141-150);
// with a predicted multiplier (the previous update's), 15 bracket values and 16
// multipliers spaced by 3.5 % around the prediction: their means bound the
// crossing tightly, and every bisection midpoint outside those bounds is decided
// without being evaluated (oc_learn / oc_skip), usually saving a whole pass.
constexpr int kOcBracket = 15;
constexpr double kOcSpread = 1.035;
__device__ void oc_plan_first(OcCtl* C, const OcArgs& a) {
    C->phase = 0;
    C->lams[0] = 0.0;
    const bool pred = C->lam_prev > 0.0;
    const int nb = pred ? kOcBracket : kOcLam - 1;
    double l2 = 1.0;
    for (int k = 1; k <= nb; ++k) { C->lams[k] = l2; l2 *= 4.0; }
    if (pred) {
        double v = C->lam_prev;
        for (int i = 0; i < (kOcLam - 1 - nb) / 2; ++i) v /= kOcSpread;
        for (int k = nb + 1; k < kOcLam; ++k) { C->lams[k] = v; v *= kOcSpread; }
    }
    C->nbr = nb;
    C->nlam = kOcLam;
    C->ka = 0.0;
    C->kb = INFINITY;
    C->plan = 0;
}

// The candidate mean is monotone non-increasing in the multiplier (every element's
// candidate is, and the fixed-order sum of monotone terms is).  A bisection midpoint
// at or below a multiplier whose mean exceeded V by more than the tolerance sends
// the search right without stopping it (optimize.py:153-158), one at or above a
// multiplier whose mean was below V by more than the tolerance sends it left: such
// midpoints are decided without evaluating them.  The margin covers the rounding
// difference between passes (their settled / mixed splits differ).
constexpr double kOcMargin = 1e-12;
__device__ void oc_learn(OcCtl* C, double lam, double mean) {
    if (mean - C->V > C->bis_tol + kOcMargin) C->ka = fmax(C->ka, lam);
    else if (C->V - mean > C->bis_tol + kOcMargin) C->kb = fmin(C->kb, lam);
}
// advance (l1, l2) through the midpoints the known bounds decide; false: the
// bisection's own stopping rule ends the search inside (l1, l2)
__device__ bool oc_skip(const OcCtl* C, double& l1, double& l2) {
    while (true) {
        if (!((l2 - l1) / (l1 + l2) > 1e-13)) return false;
        const double m = 0.5 * (l1 + l2);
        if (m <= C->ka) l1 = m;
        else if (m >= C->kb) l2 = m;
        else return true;
    }
}
__device__ void oc_finish(OcCtl* C, double l1, double l2) {
    C->lam = 0.5 * (l1 + l2);
    C->active = 1;
    C->phase = 3;
}

// Next pass of the bisection (optimize.py:151-158): the depth-5 subtree of undecided
// midpoints below (l1, l2), node i's children 2i+1 (lo, mid) and 2i+2 (mid, hi), the
// decided midpoints between them stepped over exactly as oc_walk does.  Requested by
// thread 0 (oc_plan_tree), planned by threads 0..30 in parallel (oc_plan_node).
__device__ void oc_plan_tree(OcCtl* C) {
    double l1 = C->l1, l2 = C->l2;
    if (!oc_skip(C, l1, l2)) { oc_finish(C, l1, l2); return; }   // decided without another pass
    C->phase = 2;
    C->nlam = kOcLam - 1;
    C->plan = 1;
}
__device__ void oc_plan_node(OcCtl* C, int t) {
    const int d = 31 - __clz(t + 1);             // depth of node t; path = the low d bits of t + 1
    double l1 = C->l1, l2 = C->l2;
    bool live = oc_skip(C, l1, l2);
    for (int b = d - 1; b >= 0 && live; --b) {
        const double m = 0.5 * (l1 + l2);
        if (((t + 1) >> b) & 1) l1 = m;
        else l2 = m;
        live = oc_skip(C, l1, l2);
    }
    C->lams[t] = live ? 0.5 * (l1 + l2) : 0.0;   // 0: no node (the walk ends above it)
}

// consume C->means of the pass just evaluated; plan the next pass or finish
__device__ void oc_walk(OcCtl* C) {
    const double V = C->V;
    C->passes += 1;
    if (C->phase <= 1) {
        for (int k = C->phase == 0 ? 1 : 0; k < C->nlam; ++k) oc_learn(C, C->lams[k], C->means[k]);
    }
    if (C->phase == 0) {
        if (C->means[0] <= V) { C->lam = 0.0; C->active = 0; C->phase = 3; return; }
        C->l2 = 1.0;
        C->bracket_it = 0;
        for (int k = 1; k <= C->nbr; ++k) {
            if (C->means[k] <= V) { C->l1 = 1e-30; oc_plan_tree(C); return; }
            C->l2 *= 4.0;
            if (++C->bracket_it >= 200) { C->l1 = 1e-30; oc_plan_tree(C); return; }
        }
        // bracket continues from l2
        double v = C->l2;
        int k = 0;
        for (; k < kOcLam && C->bracket_it + k < 200; ++k) { C->lams[k] = v; v *= 4.0; }
        C->nlam = k;
        C->phase = 1;
        return;
    }
    if (C->phase == 1) {
        for (int k = 0; k < C->nlam; ++k) {
            if (C->means[k] <= V) { C->l1 = 1e-30; oc_plan_tree(C); return; }
            C->l2 *= 4.0;
            if (++C->bracket_it >= 200) { C->l1 = 1e-30; oc_plan_tree(C); return; }
        }
        double v = C->l2;
        int k = 0;
        for (; k < kOcLam && C->bracket_it + k < 200; ++k) { C->lams[k] = v; v *= 4.0; }
        C->nlam = k;
        return;
    }
    // phase 2: walk the evaluated subtree (decided midpoints stepped over as planned)
    int node = 0;
    const int nodes = kOcLam - 1;
    double l1 = C->l1, l2 = C->l2;
    while (true) {
        if (!oc_skip(C, l1, l2)) { oc_finish(C, l1, l2); return; }
        if (node >= nodes) break;                // below the evaluated subtree: next pass
        const double m = 0.5 * (l1 + l2);
        const double cur = C->means[node];
        if (cur > V) { l1 = m; node = 2 * node + 2; }
        else { l2 = m; node = 2 * node + 1; }
        if (fabs(cur - V) <= C->bis_tol) { oc_finish(C, l1, l2); return; }
    }
    for (int k = 0; k < C->nlam; ++k)
        if (C->lams[k] != 0.0) oc_learn(C, C->lams[k], C->means[k]);
    C->l1 = l1;
    C->l2 = l2;
    oc_plan_tree(C);
}

// SMACC: the 32 per-lane candidate accumulators in shared memory instead of 64
// registers (3 CTAs per SM instead of 2; chosen beyond L2, launch_oc_coop)
template <bool SMACC>
__global__ void __launch_bounds__(256, SMACC ? 3 : 2) k_oc_coop(long long n, const double* __restrict__ rho,
                                                    const double* __restrict__ sens, const OcArgs a,
                                                    double* rho_out, OcCtl* C, double* partials,
                                                    double* __restrict__ qbuf, double* lam_mem) {
    // Every block keeps its own copy of the search state in shared memory and replays
    // the same walk on the same fixed-order sums, so all blocks agree on the next
    // multipliers with ONE grid barrier per pass.  Partial sums are double-buffered by
    // pass parity (a block may start writing pass t+1 while another still reads pass t).
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double sm[32][33];
    __shared__ double s_lp[kOcLam];
    __shared__ double s_lpr[2];
    __shared__ OcCtl sC;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned nb = gridDim.x;
    const double M = (double)n;
    double* flags = partials + 2 * (size_t)nb * 32;
    auto set_pows = [&]() {                       // all threads; sC.lams/nlam final
        if (threadIdx.x < kOcLam) {
            const int k = threadIdx.x;
            sC.lam_pow[k] = k < sC.nlam && sC.lams[k] != 0.0 ? oc_lam_pow(a, sC.lams[k]) : 0.0;
        }
    };
    if (threadIdx.x == 0) {
        sC.V = C->V;
        sC.V_retry = C->V_retry;
        sC.bis_tol = C->bis_tol;
        sC.passes = 0;
        sC.retried = 0;
        sC.changed = 0;
        sC.active = 0;
        sC.lam = 0.0;
        sC.first_update = C->first_update;
        sC.lam_prev = (C->first_update || !lam_mem) ? 0.0 : *lam_mem;
        oc_plan_first(&sC, a);
    }
    __syncthreads();
    set_pows();
    int parity = 0;
    int epass = 0;                                 // evaluation passes done in this launch
    while (true) {
        __syncthreads();
        if (threadIdx.x < kOcLam) s_lp[threadIdx.x] = sC.lam_pow[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {                          // range of the pass's nonzero lam^-damp
            double lo = INFINITY, hi = 0.0;
            for (int k = 0; k < sC.nlam; ++k)
                if (s_lp[k] != 0.0) { lo = fmin(lo, s_lp[k]); hi = fmax(hi, s_lp[k]); }
            if (hi == 0.0) lo = 0.0;
            s_lpr[0] = lo;
            s_lpr[1] = hi;
        }
        __syncthreads();
        if (sC.phase == 3) {
            // exact candidate of the chosen multiplier (reference expression)
            const double lam = sC.lam;
            int ch = 0;
#pragma unroll 4
            for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
                 i += (long long)gridDim.x * blockDim.x) {
                const double r = rho[i];
                const double desc = M * (-sens[i]);
                const double lo = fmax(r - a.step, a.rmin), hi = fmin(r + a.step, 1.0);
                double out;
                if (lam == 0.0) {
                    out = desc > 0.0 ? hi : (desc < 0.0 ? lo : r);
                } else {
                    const double q = fmax(desc / lam, 1e-10);
                    const double ratio = a.sqrt_damp ? sqrt(q) : pow(q, a.damp);
                    out = fmin(fmax(r * ratio, lo), hi);
                }
                ch |= out != r;
                rho_out[i] = out;
            }
            ch = __syncthreads_or(ch);
            if (threadIdx.x == 0) flags[(size_t)parity * nb + blockIdx.x] = ch ? 1.0 : 0.0;
            grid.sync();
            int any = 0;
            for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) any |= __ldcg(flags + (size_t)parity * nb + b) != 0.0;
            any = __syncthreads_or(any);
            parity ^= 1;
            if (threadIdx.x == 0) {
                sC.changed = any;
                if (!any && !sC.retried && !isnan(sC.V_retry)) {
                    sC.retried = 1;
                    sC.V = sC.V_retry;
                    oc_plan_first(&sC, a);
                } else {
                    sC.phase = 4;
                }
            }
            __syncthreads();
            if (sC.phase == 4) break;
            set_pows();
            continue;
        }
        // ---- one evaluation pass ----
        // Vertices whose candidate is clamped to the same bound, or lies inside its
        // bounds, for every multiplier of the pass ("settled") add to three per-thread
        // sums (bound value, c_e for the linear part, free-step value); only the others
        // ("mixed") evaluate the candidates: per lane when many lanes of a warp are
        // mixed, else transposed (lane k = multiplier k, the vertex broadcast by shuffles).
        // The clamp decisions are exact (fp64 products are monotone in lam^-damp).
        const int nlam = sC.nlam;
        const double lpk = lane < nlam ? s_lp[lane] : 0.0;
        const bool free0 = s_lp[0] == 0.0;
        const double lpmin = s_lpr[0], lpmax = s_lpr[1];
        extern __shared__ double oc_acc_dyn[];          // SMACC: [kOcLam][256]
        double* A = oc_acc_dyn + threadIdx.x;
        double acc[SMACC ? 1 : kOcLam];
        if constexpr (SMACC) {
#pragma unroll
            for (int k = 0; k < kOcLam; ++k) A[k * 256] = 0.0;
        } else {
#pragma unroll
            for (int k = 0; k < kOcLam; ++k) acc[k] = 0.0;
        }
        double acck = 0.0, sCn = 0.0, sL = 0.0, sF = 0.0;
        const long long wstride = (long long)gridDim.x * nw * 32;
        // the next element's (rho, sens) are loaded before this one is processed: the
        // loop is otherwise one L2 round trip per element (long-scoreboard bound)
        // The pass-invariant c_e = rho * desc^damp (a square root per element) is formed
        // in the first pass and kept in qbuf with the sign of desc encoded
        // (q >= 0: c_e, desc > 0;  -1: desc < 0;  -2: desc == 0); later passes read q
        // instead of the sensitivity.  Each thread revisits its own elements only.
        const bool first = epass == 0 || !qbuf;
        const double* src = first ? sens : qbuf;
        long long base = ((long long)blockIdx.x * nw + wid) * 32;
        double r_nx = 0.0, s_nx = 0.0;
        if (base + lane < n) {
            r_nx = __ldg(rho + base + lane);
            s_nx = src[base + lane];
        }
        for (; base < n; base += wstride) {
            const long long i = base + lane;
            const double r_cur = r_nx, s_cur = s_nx;
            if (i + wstride < n) {
                r_nx = __ldg(rho + i + wstride);
                s_nx = src[i + wstride];
            }
            bool mixed = false;
            double ce = 0.0, lof = 0.0, hi = 0.0, freev = 0.0;
            if (i < n) {
                const double r = r_cur;
                double q;
                if (first) {
                    const double desc = M * (-s_cur);
                    q = desc > 0.0 ? r * (a.sqrt_damp ? sqrt(desc) : pow(desc, a.damp)) : (desc < 0.0 ? -1.0 : -2.0);
                    if (qbuf) qbuf[i] = q;
                } else {
                    q = s_cur;
                }
                const double lo = fmax(r - a.step, a.rmin);
                hi = fmin(r + a.step, 1.0);
                lof = fmax(lo, r * a.floor_ratio);
                ce = fmax(q, 0.0);
                freev = q >= 0.0 ? hi : (q == -1.0 ? lo : r);
                const double tlo = ce * lpmin, thi = ce * lpmax;
                // branch-free classification: all multipliers of the pass clamp to lof,
                // all to hi, all stay inside (linear), or mixed
                const bool c_lo = thi <= lof, c_hi = !c_lo && tlo >= hi;
                const bool c_lin = !c_lo && !c_hi && tlo >= lof && thi <= hi;
                mixed = !(c_lo || c_hi || c_lin);
                sCn += c_lo ? lof : (c_hi ? hi : 0.0);
                sL += c_lin ? ce : 0.0;
                sF += mixed ? 0.0 : freev;
            }
            unsigned m = __ballot_sync(0xffffffffu, mixed);
            if (!m) continue;
            if (__popc(m) > 10) {
                if (mixed) {
                    // only slot 0 can be the free step (lam = 0); slots >= nlam (lam^-damp 0)
                    // accumulate values nobody reads
                    if constexpr (SMACC) {
                        A[0] += free0 ? freev : fmin(fmax(ce * s_lp[0], lof), hi);
#pragma unroll
                        for (int k = 1; k < kOcLam; ++k) A[k * 256] += fmin(fmax(ce * s_lp[k], lof), hi);
                    } else {
                        acc[0] += free0 ? freev : fmin(fmax(ce * s_lp[0], lof), hi);
#pragma unroll
                        for (int k = 1; k < kOcLam; ++k) acc[k] += fmin(fmax(ce * s_lp[k], lof), hi);
                    }
                }
            } else {
                while (m) {
                    const int j = __ffs(m) - 1;
                    m &= m - 1;
                    const double cej = __shfl_sync(0xffffffffu, ce, j);
                    const double lofj = __shfl_sync(0xffffffffu, lof, j);
                    const double hij = __shfl_sync(0xffffffffu, hi, j);
                    const double fj = __shfl_sync(0xffffffffu, freev, j);
                    const double cand = lpk == 0.0 ? fj : fmin(fmax(cej * lpk, lofj), hij);
                    acck += lane < nlam ? cand : 0.0;
                }
            }
        }
        double mine;
        if constexpr (SMACC) {
            double t[kOcLam];
#pragma unroll
            for (int k = 0; k < kOcLam; ++k) t[k] = A[k * 256];
            mine = acck + warp_reduce_scatter32(t);
        } else {
            mine = acck + warp_reduce_scatter32(acc);
        }
        {
            // warp_sum leaves the total in lane 0
            const double Cs = __shfl_sync(0xffffffffu, warp_sum(sCn), 0);
            const double L = __shfl_sync(0xffffffffu, warp_sum(sL), 0);
            const double F = __shfl_sync(0xffffffffu, warp_sum(sF), 0);
            mine += lane < nlam ? (lpk == 0.0 ? F : Cs + lpk * L) : 0.0;
        }
        sm[wid][lane] = mine;
        __syncthreads();
        double* part = partials + (size_t)parity * nb * 32;
        if (threadIdx.x < 32) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += sm[w][threadIdx.x];
            part[(size_t)blockIdx.x * 32 + threadIdx.x] = t;
        }
        grid.sync();
        // every block: the same fixed-order sum of all blocks' partials
        {
            // 16 loads in flight per thread (the sum is a chain of L2 round trips otherwise)
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            for (unsigned b = wid; b < nb; b += 16 * nw) {
                double v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const unsigned bb = b + j * nw;
                    v[j] = bb < nb ? __ldcg(part + (size_t)bb * 32 + lane) : 0.0;
                }
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    t0 += v[j];
                    t1 += v[j + 1];
                    t2 += v[j + 2];
                    t3 += v[j + 3];
                }
            }
            sm[wid][lane] = (t0 + t1) + (t2 + t3);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            double u = 0.0;
            for (int w = 0; w < nw; ++w) u += sm[w][threadIdx.x];
            sC.means[threadIdx.x] = u / M;
        }
        parity ^= 1;
        ++epass;
        __syncthreads();
        if (threadIdx.x == 0) oc_walk(&sC);
        __syncthreads();
        if (sC.plan) {
            if (threadIdx.x < kOcLam - 1) oc_plan_node(&sC, threadIdx.x);
            __syncthreads();
            if (threadIdx.x == 0) sC.plan = 0;
            __syncthreads();
        }
        set_pows();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (lam_mem) *lam_mem = sC.active ? sC.lam : 0.0;   // the next update's prediction
        C->passes = sC.passes;
        C->retried = sC.retried;
        C->changed = sC.changed;
        C->active = sC.active;
        C->lam = sC.lam;
        C->V = sC.V;
        C->phase = sC.phase;
    }
}

// Exact candidate for the chosen multiplier (lam == 0: free step), written to
// rho_out; flags[0] |= any(rho_out != rho).
__global__ void k_oc_apply(long long n, const double* __restrict__ rho, const double* __restrict__ sens,
                           OcArgs a, double lam, double* __restrict__ rho_out, int* changed) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int ch = 0;
    if (i < n) {
        const double r = rho[i];
        const double desc = (double)n * (-sens[i]);
        const double lo = fmax(r - a.step, a.rmin), hi = fmin(r + a.step, 1.0);
        double out;
        if (lam == 0.0) {
            out = desc > 0.0 ? hi : (desc < 0.0 ? lo : r);
        } else {
            const double q = fmax(desc / lam, 1e-10);
            const double ratio = a.sqrt_damp ? sqrt(q) : pow(q, a.damp);
            out = fmin(fmax(r * ratio, lo), hi);
        }
        ch = out != r;
        rho_out[i] = out;
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(changed, 1);
}

// ===========================================================================
// Level stencils
// ===========================================================================
// ---- k10: push x-march, operand consumed once per plane (otm_stencil10.cuh) ----
// CPS = CTAs per SM the ring is sized for (TY rows x NZ/2 threads per CTA)
template <int NZ, int TY, int CPS, bool WZ>
__global__ void __launch_bounds__(NZ / 2 * TY, CPS) k10_smooth_res(Geo g, float s12, const __grid_constant__ K10Maps maps,
                                                                  float omega, float* z, float* res) {
    K10Op<K10_SMOOTH, NZ, TY, false, CPS, WZ> op;
    op.omega = omega; op.out0 = z; op.out1 = res; op.n = g.n;
    march10(g, s12, maps, op);
}

template <bool DOT, int NZ, int TY, int CPS>
__global__ void __launch_bounds__(NZ / 2 * TY, CPS) k10_jacobi(Geo g, float s12, const __grid_constant__ K10Maps maps,
                                                              float omega, float* zout, double* partials,
                                                              unsigned* counter, PcgScalars* sc) {
    K10Op<K10_JACOBI, NZ, TY, DOT, CPS> op;
    op.omega = omega; op.out0 = zout; op.out1 = nullptr; op.n = g.n;
    op.acc[0] = op.acc[1] = op.acc[2] = 0.0;
    march10(g, s12, maps, op);
    if (DOT) {
        double v3[3] = {op.acc[0], op.acc[1], op.acc[2]};
        if (reduce_finalize<3>(v3, partials, counter, sc->red)) {
            for (int cc = 0; cc < 3; ++cc) {
                const double rz = sc->red[cc];
                sc->beta[cc] = (sc->first || sc->rz[cc] == 0.0) ? 0.0 : rz / sc->rz[cc];
                sc->rz[cc] = rz;
            }
            sc->first = 0;
        }
    }
}

template <int NZ, int TY, int CPS>
__global__ void __launch_bounds__(NZ / 2 * TY, CPS) k10_spmv(Geo g, float s12, const __grid_constant__ K10Maps maps,
                                                            float* q, double* partials, unsigned* counter,
                                                            PcgScalars* sc) {
    K10Op<K10_SPMV, NZ, TY, true, CPS> op;
    op.omega = 0.f; op.out0 = q; op.out1 = nullptr; op.n = g.n;
    op.acc[0] = op.acc[1] = op.acc[2] = 0.0;
    march10(g, s12, maps, op);
    double v3[3] = {op.acc[0], op.acc[1], op.acc[2]};
    if (reduce_finalize<3>(v3, partials, counter, sc->red + 3)) {
        for (int cc = 0; cc < 3; ++cc) {
            const double pq = sc->red[3 + cc];
            sc->pq[cc] = pq;
            sc->alpha[cc] = (sc->active[cc] != 0.0 && pq > 0.0) ? sc->rz[cc] / pq : 0.0;
        }
    }
}

// host: tensor maps through the driver entry point (no libcuda link needed)
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled_t)p;
    }
    return fn;
}
// a failed tensor-map encode silently demotes the level stencils to the generic
// kernels: say so once on stderr
static bool tma_check(CUresult r, const char* what) {
    static bool warned = false;
    if (r != CUDA_SUCCESS && !warned) {
        warned = true;
        fprintf(stderr, "[otm] cuTensorMapEncodeTiled (%s) failed with CUresult %d: TMA stencils disabled\n", what,
                (int)r);
    }
    return r == CUDA_SUCCESS;
}
static bool encode_map(CUtensorMap* m, const float* base, int nz, int ny, long long planes, int box_rows) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return tma_check(CUDA_ERROR_NOT_FOUND, "entry point");
    const cuuint64_t dims[3] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)nz * 4, (cuuint64_t)nz * ny * 4};
    const cuuint32_t box[3] = {(cuuint32_t)nz, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return tma_check(fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE), "3-d");
}
static bool encode_map64(CUtensorMap* m, const double* base, int nz, int ny, long long planes, int box_rows) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    if (nz > 256) {                       // z split into (256, nz / 256): box dims hold <= 256 elements
        const cuuint64_t d4[4] = {256, (cuuint64_t)(nz / 256), (cuuint64_t)ny, (cuuint64_t)planes};
        const cuuint64_t s4[3] = {256 * 8, (cuuint64_t)nz * 8, (cuuint64_t)nz * ny * 8};
        const cuuint32_t b4[4] = {256, (cuuint32_t)(nz / 256), (cuuint32_t)box_rows, 1};
        const cuuint32_t e4[4] = {1, 1, 1, 1};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const cuuint64_t dims[3] = {(cuuint64_t)nz, (cuuint64_t)ny, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)nz * 8, (cuuint64_t)nz * ny * 8};
    const cuuint32_t box[3] = {(cuuint32_t)nz, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// ===========================================================================
// Host launchers
// ===========================================================================

static inline unsigned nblk(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

// Grid cap for the one-item-per-thread kernels that end in a cross-block reduction
// (k_upd, the forward filter's sums) on fields above 4M vertices: 8 blocks per SM
// walking the field, instead of one fence + atomic per 256 items.  0: no cap (the
// 128^3 headline keeps its one-pass grids; OTM_GS_CAP=0 turns the cap off).
static unsigned gs_cap(long long n) {
    static const bool on = !(getenv("OTM_GS_CAP") && atoi(getenv("OTM_GS_CAP")) == 0);
    if (!on || n <= (1LL << 22)) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)(8 * sms);
}

// Inner-loop kernels go through launch_pdl: programmatic stream serialisation lets
// the next kernel's CTAs be scheduled while the previous grid drains (each such
// kernel starts with pdl_wait()).  OTM_PDL=0 turns it off.
static bool pdl_enabled() {
    static const bool on = !(getenv("OTM_PDL") && atoi(getenv("OTM_PDL")) == 0);
    return on;
}
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// opt a kernel into more than 48 KB of dynamic shared memory (once per kernel)
template <class K>
static void smem_attr(K kernel, size_t bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int stencil_chunks(const Geo& g, int* xb) {
    const long long blocks_plane = (g.pl + 127) / 128;
    long long chunks = (4LL * 148 + blocks_plane - 1) / blocks_plane;
    if (chunks < 1) chunks = 1;
    if (chunks > g.nx) chunks = g.nx;
    int b = (int)((g.nx + chunks - 1) / chunks);
    if (b < 1) b = 1;
    *xb = b;
    return (int)((g.nx + b - 1) / b);
}

static inline dim3 stencil_grid(const Geo& g, int* xb) {
    const int ch = stencil_chunks(g, xb);
    return dim3((unsigned)((g.pl + 127) / 128), (unsigned)ch, 1);
}

// k_filter_b for the tap pattern of fs (compile-time mask when it is a common one)
template <int MODE>
static void launch_filter_b(cudaStream_t s, const Geo& g, const FilterSetup& fs, const double* in, double* out,
                            double* k64, float* k32, const SimpParams& sp, double* partials, unsigned* counter,
                            double* out3, const XRange* xr = nullptr) {
    FilterTaps taps;
    unsigned mask = 0;
    for (int i = 0; i < 27; ++i) {
        taps.w27[i] = fs.w27[i];
        if (fs.w27[i] != 0.0) mask |= 1u << i;
    }
    const long long p0 = xr ? (long long)xr->xa * g.pl / 2 : 0, p1 = xr ? (long long)xr->xb * g.pl / 2 : g.n >> 1;
    unsigned blocks = nblk(p1 - p0, 256);
    const unsigned cap = MODE == 2 ? gs_cap(2 * (p1 - p0)) : 0;
    if (cap && blocks > cap) {                     // the forward filter's sums over a capped grid
        blocks = cap;
        if (mask == kTapsNoCorners)
            k_filter_b<MODE, kTapsNoCorners, true><<<blocks, 256, 0, s>>>(g, p0, p1, taps, in, out, k64, k32, sp,
                                                                          partials, counter, out3);
        else
            k_filter_b<MODE, 0, true><<<blocks, 256, 0, s>>>(g, p0, p1, taps, in, out, k64, k32, sp, partials,
                                                             counter, out3);
        return;
    }
    if (mask == kTapsNoCorners)
        k_filter_b<MODE, kTapsNoCorners><<<blocks, 256, 0, s>>>(g, p0, p1, taps, in, out, k64, k32, sp, partials,
                                                                counter, out3);
    else if (mask == kTapsAll)
        k_filter_b<MODE, kTapsAll><<<blocks, 256, 0, s>>>(g, p0, p1, taps, in, out, k64, k32, sp, partials, counter,
                                                          out3);
    else
        k_filter_b<MODE, 0><<<blocks, 256, 0, s>>>(g, p0, p1, taps, in, out, k64, k32, sp, partials, counter, out3);
}

bool launch_filter_range(cudaStream_t s, const Geo& g, const FilterSetup& fs, int mode, const SimpParams& sp,
                         const double* in, double* out, double* k64, Red& red, double* out3, const XRange& xr) {
    if (!fs.window || g.nz % 2 != 0) return false;
    if (mode == 2) launch_filter_b<2>(s, g, fs, in, out, k64, nullptr, sp, red.partials, red.counter, out3, &xr);
    else launch_filter_b<1>(s, g, fs, in, out, nullptr, nullptr, sp, nullptr, nullptr, nullptr, &xr);
    return true;
}

void launch_filter(cudaStream_t s, const Geo& g, const FilterSetup& fs, int adjoint, const double* in,
                   double* out, Red& red) {
    if (fs.window && g.nz % 2 == 0) {
        SimpParams sp{};
        if (adjoint) launch_filter_b<1>(s, g, fs, in, out, nullptr, nullptr, sp, nullptr, nullptr, nullptr);
        else launch_filter_b<0>(s, g, fs, in, out, nullptr, nullptr, sp, nullptr, nullptr, nullptr);
        return;
    }
    if (fs.window) {
        int xb;
        const dim3 grid = stencil_grid(g, &xb);
        FilterTaps taps;
        for (int i = 0; i < 27; ++i) taps.w27[i] = fs.w27[i];
        SimpParams sp{};
        if (adjoint)
            k_filter<1><<<grid, 128, 0, s>>>(g, xb, taps, in, out, nullptr, nullptr, sp, nullptr, nullptr, nullptr);
        else
            k_filter<0><<<grid, 128, 0, s>>>(g, xb, taps, in, out, nullptr, nullptr, sp, nullptr, nullptr, nullptr);
    } else {
        k_filter_generic<<<nblk(g.n, 256), 256, 0, s>>>(g, fs.ntaps, fs.offs_dev, fs.wts_dev, adjoint, in, out);
    }
}

void launch_filter_simp(cudaStream_t s, const Geo& g, const FilterSetup& fs, const SimpParams& sp,
                        const double* rho, double* rho_f, double* k64, float* k32, Red& red, double* out3) {
    if (fs.window && g.nz % 2 == 0) {
        launch_filter_b<2>(s, g, fs, rho, rho_f, k64, k32, sp, red.partials, red.counter, out3);
        return;
    }
    if (fs.window) {
        int xb;
        const dim3 grid = stencil_grid(g, &xb);
        FilterTaps taps;
        for (int i = 0; i < 27; ++i) taps.w27[i] = fs.w27[i];
        k_filter<2><<<grid, 128, 0, s>>>(g, xb, taps, rho, rho_f, k64, k32, sp, red.partials, red.counter, out3);
    } else {
        k_filter_generic<<<nblk(g.n, 256), 256, 0, s>>>(g, fs.ntaps, fs.offs_dev, fs.wts_dev, 0, rho, rho_f);
        k_simp<<<nblk(g.n, 256), 256, 0, s>>>(g.n, rho_f, k64, k32, sp);
        launch_means(s, g.n, rho, sp.p, red, out3);   // sums of rho, rho^p
        // sum of rho_f: k_means on rho_f with p = 1 into out3[2] (out3[3] scratch)
        k_means<<<592, 256, 0, s>>>(g.n, rho_f, 1.0, red.partials, red.counter, out3 + 2);
    }
}

void launch_simp(cudaStream_t s, long long n, const double* rf, double* k64, float* k32, const SimpParams& sp) {
    k_simp<<<nblk(n, 256), 256, 0, s>>>(n, rf, k64, k32, sp);
}
void launch_set_kappa(cudaStream_t s, long long n, const double* kin, double* k64, float* k32) {
    k_set_kappa<<<nblk(n, 256), 256, 0, s>>>(n, kin, k64, k32);
}
void launch_means(cudaStream_t s, long long n, const double* rho, double p, Red& red, double* out2) {
    k_means<<<592, 256, 0, s>>>(n, rho, p, red.partials, red.counter, out2);
}
void launch_symmetrize(cudaStream_t s, const Geo& g, double* a) {
    k_symmetrize<<<nblk(g.n, 256), 256, 0, s>>>(g, a);
}
void launch_coarsen(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* kf, float* kc) {
    k_coarsen<<<nblk(c.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], kf, kc);
}
void launch_coarsen_dinv(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* kf, float* kc,
                         float kdiag_f, float* dinv_f) {
    k_coarsen_dinv<<<nblk(std::max(f.n, c.n), 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], kf, kc, kdiag_f, dinv_f);
}
void launch_dinv(cudaStream_t s, const Geo& g, const float* k, float kdiag, float* dinv) {
    k_dinv<<<nblk(g.n, 256), 256, 0, s>>>(g, k, kdiag, dinv);
}
int launch_coarse_setup(cudaStream_t s, const Geo& g, const float* k, const CoarseTemplate& ct, double* work,
                        float* G) {
    if (g.n == 64 && !getenv("OTM_GENERIC_COARSE")) {
        const size_t b64 = (64 * 64 + 2 * 64 + 1) * sizeof(double);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_coarse_setup64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b64);
            attr = true;
        }
        k_coarse_setup64<<<1, 256, b64, s>>>(g, k, ct, G);
        return 1;
    }
    if (g.n > 256) {
        const int n = (int)g.n;
        double* A = work;
        double* uv = work + (size_t)n * n;       // 2n doubles (work holds 2 n^2 + n + 2)
        k_cs_assemble<<<nblk(n, 128), 128, 0, s>>>(g, k, ct, A);
        const dim3 blk(32, 8), grd((unsigned)((n + 31) / 32), (unsigned)((n + 7) / 8));
        for (int p = 1; p < n; ++p) {
            k_cs_pivot<<<nblk(2 * n, 256), 256, 0, s>>>(A, n, p, uv);
            k_cs_update<<<grd, blk, 0, s>>>(A, n, p, uv);
        }
        k_cs_means<<<nblk(n, 128), 128, 0, s>>>(A, n, uv);
        k_cs_write<<<grd, blk, 0, s>>>(A, n, uv, G);
        return 2 * (n - 1) + 3;
    }
    const size_t bytes = (2 * (size_t)g.n * g.n + g.n) * sizeof(double);
    const int use_smem = bytes <= 96 * 1024;
    if (use_smem) {
        cudaFuncSetAttribute(k_coarse_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    }
    k_coarse_setup<<<1, 1024, use_smem ? bytes : 0, s>>>(g, k, ct, work, G, use_smem);
    return 1;
}
void launch_coarse_solve(cudaStream_t s, int n, const float* G, const float* f, float* z) {
    const int rows = 3 * n;
    const int blocks = rows <= 32 ? 1 : (rows + 31) / 32 > 148 ? 148 : (rows + 31) / 32;
    launch_pdl(k_coarse_solve, blocks, 1024, 0, s, n, G, f, z);
}
// 4-D (z, case, y, x) fp64 map of the three stacked cases (k_res64p), box rows x 3 cases x nz
static bool encode_map64c(CUtensorMap* m, const double* base, const Geo& g, int box_rows) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    if (g.nz > 256) {                     // z split into (256, nz / 256) (box dims hold <= 256 elements)
        const cuuint64_t d5[5] = {256, (cuuint64_t)(g.nz / 256), 3, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
        const cuuint64_t s5[4] = {256 * 8, (cuuint64_t)g.n * 8, (cuuint64_t)g.nz * 8, (cuuint64_t)g.pl * 8};
        const cuuint32_t b5[5] = {256, (cuuint32_t)(g.nz / 256), 3, (cuuint32_t)box_rows, 1};
        const cuuint32_t e5[5] = {1, 1, 1, 1, 1};
        return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, d5, s5, b5, e5, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)g.nz, 3, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
    const cuuint64_t strides[3] = {(cuuint64_t)g.n * 8, (cuuint64_t)g.nz * 8, (cuuint64_t)g.pl * 8};
    const cuuint32_t box[4] = {(cuuint32_t)g.nz, 3, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)base, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NZ>
static void l_res64p(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const R64PMaps& M0, const double* fmean,
                     float* r32, Red& red, double* out9, const int* skip) {
    using P = R64P<NZ>;
    smem_attr(k_res64p<NZ>, P::SMEM);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_res64p<NZ>, P::THREADS, P::SMEM);
    if (per_sm < 1) per_sm = 1;
    const int nxr = M0.xb - M0.xa;
    const long long nty = g.ny / P::TY, units = nty * nxr, slots = (long long)per_sm * sms;
    R64PMaps M = M0;
    M.lock = 0;
    long long blocks = std::min(slots, units);
    // lockstep row-tile order where the three fp64 cases (24 B per vertex) exceed half the L2
    static const bool lock_on = !(getenv("OTM_K10_LOCK") && atoi(getenv("OTM_K10_LOCK")) == 0);
    if (lock_on && (long long)nxr * g.pl * 24 > (64LL << 20)) {
        const long long k = std::max<long long>(1, std::min<long long>(slots / nty, nxr / 8));
        M.lock = (int)k;
        blocks = nty * k;
    }
    k_res64p<NZ><<<(unsigned)blocks, dim3(NZ, P::TY), P::SMEM, s>>>(g, lt, M, fmean, r32, red.partials, red.counter,
                                                                    out9, skip);
}

// z extents with a k_res64p instantiation (OTM_RES64P_512=0: nz = 512 on k_res64w<512>)
static bool res64p_nz(int nz) {
    static const bool p512 = !(getenv("OTM_RES64P_512") && atoi(getenv("OTM_RES64P_512")) == 0);
    return nz == 64 || nz == 128 || nz == 256 || (nz == 512 && p512);
}
static void l_res64p_nz(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const R64PMaps& M, const double* fmean,
                        float* r32, Red& red, double* out9, const int* skip) {
    if (g.nz == 64) l_res64p<64>(s, g, lt, M, fmean, r32, red, out9, skip);
    else if (g.nz == 128) l_res64p<128>(s, g, lt, M, fmean, r32, red, out9, skip);
    else if (g.nz == 256) l_res64p<256>(s, g, lt, M, fmean, r32, red, out9, skip);
    else l_res64p<512>(s, g, lt, M, fmean, r32, red, out9, skip);
}

bool launch_res64_range(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                        const double* fmean, float* r32, Red& red, double* out9, const XRange& xr) {
    if (!lt.equal || !res64p_nz(g.nz) || xr.xa < 1 || xr.xb > g.nx - 1 || xr.xb <= xr.xa)
        return false;
    const int ty = g.nz >= 256 ? 1 : 256 / g.nz;
    if (g.ny % ty != 0 || g.ny < 2 * ty) return false;
    R64PMaps M;
    if (!(encode_map64c(&M.t_full, T, g, ty + 2) && encode_map64c(&M.t_main, T, g, ty) &&
          encode_map64c(&M.t_halo, T, g, 1) && encode_map64(&M.k_full, kap, g.nz, g.ny, g.nx, ty + 1) &&
          encode_map64(&M.k_main, kap, g.nz, g.ny, g.nx, ty) && encode_map64(&M.k_halo, kap, g.nz, g.ny, g.nx, 1)))
        return false;
    M.xa = xr.xa;
    M.xb = xr.xb;
    l_res64p_nz(s, g, lt, M, fmean, r32, red, out9, nullptr);
    return true;
}

void launch_res64(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                  const double* fext, const double* fmean, float* r32, Red& red, double* out9, const int* skip) {
    // all three cases in one push march (k_res64p; OTM_RES64P=0: the per-case k_res64w)
    static const bool use_p = !(getenv("OTM_RES64P") && atoi(getenv("OTM_RES64P")) == 0);
    if (use_p && !fext && lt.equal && res64p_nz(g.nz) && g.nx >= 2) {
        const int ty = g.nz >= 256 ? 1 : 256 / g.nz;
        if (g.ny % ty == 0 && g.ny >= 2 * ty) {
            // per host thread: structures designed concurrently from several threads
            // (one stream each) must not share the tensor-map cache
            static thread_local R64PMaps M;
            static thread_local const double *lastT = nullptr, *lastK = nullptr;
            static thread_local int lastdims[3] = {0, 0, 0};
            static thread_local bool lastok = false;
            if (T != lastT || kap != lastK || g.nx != lastdims[0] || g.ny != lastdims[1] || g.nz != lastdims[2]) {
                lastok = encode_map64c(&M.t_full, T, g, ty + 2) && encode_map64c(&M.t_main, T, g, ty) &&
                         encode_map64c(&M.t_halo, T, g, 1) && encode_map64(&M.k_full, kap, g.nz, g.ny, g.nx, ty + 1) &&
                         encode_map64(&M.k_main, kap, g.nz, g.ny, g.nx, ty) &&
                         encode_map64(&M.k_halo, kap, g.nz, g.ny, g.nx, 1);
                lastT = T;
                lastK = kap;
                lastdims[0] = g.nx;
                lastdims[1] = g.ny;
                lastdims[2] = g.nz;
            }
            if (lastok) {
                M.xa = 0;
                M.xb = g.nx;
                l_res64p_nz(s, g, lt, M, fmean, r32, red, out9, skip);
                return;
            }
        }
    }
    static const bool r512 = !(getenv("OTM_RES64_512") && atoi(getenv("OTM_RES64_512")) == 0);
    const bool w512 = r512 && lt.equal && g.nz == 512 && g.nx >= 2;
    if (!fext && (tma_tiling(g, lt) || w512)) {
        const int tyd = g.nz >= 256 ? 1 : 256 / g.nz;
        // tensor maps of the last (T, kappa, grid) are reused: encoding costs a few us of
        // host time per map, on the critical path between two host waits
        static thread_local R64Maps M;
        static thread_local const double *lastT = nullptr, *lastK = nullptr;
        static thread_local int lastdims[3] = {0, 0, 0};
        static thread_local bool lastok = false;
        if (T != lastT || kap != lastK || g.nx != lastdims[0] || g.ny != lastdims[1] || g.nz != lastdims[2]) {
            lastok = encode_map64(&M.Tm, T, g.nz, g.ny, 3LL * g.nx, tyd) &&
                     encode_map64(&M.Th, T, g.nz, g.ny, 3LL * g.nx, 1) &&
                     encode_map64(&M.Km, kap, g.nz, g.ny, g.nx, tyd) && encode_map64(&M.Kh, kap, g.nz, g.ny, g.nx, 1);
            lastT = T;
            lastK = kap;
            lastdims[0] = g.nx;
            lastdims[1] = g.ny;
            lastdims[2] = g.nz;
        }
        if (lastok) {
            const size_t sm = r64_smem_bytes(g.nz);
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const long long units = 3LL * (g.ny / tyd) * g.nx;
            static const int bps = getenv("OTM_R64_BPS") ? atoi(getenv("OTM_R64_BPS")) : 2;
            const long long slots = (long long)sms * (g.nz > 256 ? 1 : bps);
            unsigned blocks = (unsigned)std::min<long long>(slots, units);
            // lockstep row order beyond L2 (T, one 8-byte case per vertex, > 64 MB)
            static const bool lock_on = !(getenv("OTM_K10_LOCK") && atoi(getenv("OTM_K10_LOCK")) == 0);
            M.lock = 0;
            if (lock_on && g.n * 8 > (64LL << 20)) {
                const long long rows = 3LL * (g.ny / tyd);
                const long long k = std::max<long long>(1, std::min<long long>((4 * slots + rows / 2) / rows, g.nx / 8));
                M.lock = (int)k;
                blocks = (unsigned)(rows * k);
            }
            const dim3 blk((unsigned)g.nz, (unsigned)tyd);
            switch (g.nz) {
            case 512:
                smem_attr(k_res64w<512>, sm);
                k_res64w<512><<<blocks, blk, sm, s>>>(g, lt, M, fmean, r32, red.partials, red.counter, out9, skip);
                break;
            case 64:
                smem_attr(k_res64w<64>, sm);
                k_res64w<64><<<blocks, blk, sm, s>>>(g, lt, M, fmean, r32, red.partials, red.counter, out9, skip);
                break;
            case 128:
                smem_attr(k_res64w<128>, sm);
                k_res64w<128><<<blocks, blk, sm, s>>>(g, lt, M, fmean, r32, red.partials, red.counter, out9, skip);
                break;
            default:
                smem_attr(k_res64w<256>, sm);
                k_res64w<256><<<blocks, blk, sm, s>>>(g, lt, M, fmean, r32, red.partials, red.counter, out9, skip);
                break;
            }
            return;
        }
    }
    int xb;
    const dim3 grid = stencil_grid(g, &xb);
    if (fext)
        k_res64<true><<<grid, 128, 0, s>>>(g, xb, lt, kap, T, fext, fmean, r32, red.partials, red.counter, out9, skip);
    else
        k_res64<false><<<grid, 128, 0, s>>>(g, xb, lt, kap, T, nullptr, fmean, r32, red.partials, red.counter,
                                            out9, skip);
}
void launch_apply64(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                    double* out, int load_case) {
    int xb;
    const dim3 grid = stencil_grid(g, &xb);
    k_apply64<<<grid, 128, 0, s>>>(g, xb, lt, kap, T, out, load_case);
}
template <class K>
static int march_chunks(K kernel, const Geo& g, int planes) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
    const long long want = 2LL * sms * std::max(per_sm, 1) * 256;
    long long c = (want + g.pl - 1) / g.pl;
    c = std::min<long long>(c, std::max(1, planes / 4));
    return (int)std::max<long long>(1, c);
}
static XRange whole(const Geo& g, const XRange* xr) { return xr ? *xr : XRange{0, g.nx, (double)g.n}; }
// x chunks per (y, z) column of a marching kernel, cached per (plane size, plane count)
template <class K>
static int chunks_for(K kernel, const Geo& g, int planes, int& ch, int& for_pl, int& for_np) {
    if (for_pl != g.pl || for_np != planes) {
        ch = march_chunks(kernel, g, planes);
        for_pl = g.pl;
        for_np = planes;
    }
    return ch;
}
void launch_load_means(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, Red& red,
                       double* out3, const XRange* xr) {
    static thread_local int ch = 0, for_pl = -1, for_np = -1;
    const XRange r = whole(g, xr);
    chunks_for(k_load_means_x, g, r.xb - r.xa, ch, for_pl, for_np);
    k_load_means_x<<<nblk((long long)g.pl * ch, 256), 256, 0, s>>>(g, ch, r, lt, kap, red.partials, red.counter,
                                                                   out3);
}
void launch_sum3(cudaStream_t s, long long n, const double* f, Red& red, double* out3) {
    k_sum3<<<592, 256, 0, s>>>(n, f, red.partials, red.counter, out3);
}
static inline bool small_level(const Geo& g) { return g.n <= 65536; }


static bool encode_map4_split(CUtensorMap* m, const float* base, const Geo& g, int box_rows, bool cases) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return tma_check(CUDA_ERROR_NOT_FOUND, "entry point");
    const cuuint32_t h = (cuuint32_t)(g.nz / 256);
    const cuuint64_t dims5[5] = {256, h, 3, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
    const cuuint64_t strides5[4] = {256 * 4, (cuuint64_t)g.n * 4, (cuuint64_t)g.nz * 4, (cuuint64_t)g.pl * 4};
    const cuuint32_t box5[5] = {256, h, 3, (cuuint32_t)box_rows, 1};
    const cuuint64_t dims4[4] = {256, h, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
    const cuuint64_t strides4[3] = {256 * 4, (cuuint64_t)g.nz * 4, (cuuint64_t)g.pl * 4};
    const cuuint32_t box4[4] = {256, h, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return tma_check(fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cases ? 5 : 4, (void*)base, cases ? dims5 : dims4,
                        cases ? strides5 : strides4, cases ? box5 : box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE), cases ? "5-d split" : "4-d split");
}
// single-field (z, y, x) map of the k10 march (split along z for nz > 256)
static bool encode_map1(CUtensorMap* m, const float* base, const Geo& g, int box_rows) {
    if (g.nz > 256) return encode_map4_split(m, base, g, box_rows, false);
    return encode_map(m, base, g.nz, g.ny, g.nx, box_rows);
}
static bool encode_map4(CUtensorMap* m, const float* base, const Geo& g, int box_rows) {
    if (g.nz > 256) return encode_map4_split(m, base, g, box_rows, true);
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return tma_check(CUDA_ERROR_NOT_FOUND, "entry point");
    const cuuint64_t dims[4] = {(cuuint64_t)g.nz, 3, (cuuint64_t)g.ny, (cuuint64_t)g.nx};
    const cuuint64_t strides[3] = {(cuuint64_t)g.n * 4, (cuuint64_t)g.nz * 4, (cuuint64_t)g.pl * 4};
    const cuuint32_t box[4] = {(cuuint32_t)g.nz, 3, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return tma_check(fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE), "4-d");
}
static int k10_ty(int nz) { return nz == 512 ? 2 : 512 / nz; }   // rows per CTA tile
static long long k10_min_n() {           // smallest level on the k10 path (OTM_K10_MINN, tuning)
    static const long long v = getenv("OTM_K10_MINN") ? atoll(getenv("OTM_K10_MINN")) : 32768;
    return v;
}
static bool k10_512() {                 // nz = 512 on k10 (z-split TMA maps); OTM_K10_512=0 disables
    static const bool v = !(getenv("OTM_K10_512") && atoi(getenv("OTM_K10_512")) == 0);
    return v;
}
static bool k10_ok(const Geo& g, const LevelTemplate& lt) {
    return lt.equal && (g.nz == 64 || g.nz == 128 || g.nz == 256 || (g.nz == 512 && k10_512())) && g.ny % k10_ty(g.nz) == 0 &&
           g.ny >= 2 * k10_ty(g.nz) && g.nx >= 2 && g.n >= k10_min_n();
}
// op3: 3-case operand (halo), d: D^-1 (smooth_res: halo, jacobi: centre), f3: jacobi right-hand side
static bool k10_maps(K10Maps& M, const Geo& g, const float* op3, const float* d, const float* f3, const float* kap) {
    const int TY = k10_ty(g.nz);
    M.xa = 0;
    M.xb = g.nx;
    bool ok = encode_map4(&M.op_full, op3, g, TY + 2) && encode_map4(&M.op_main, op3, g, TY) &&
              encode_map4(&M.op_halo, op3, g, 1) && encode_map1(&M.k_full, kap, g, TY + 1) &&
              encode_map1(&M.k_main, kap, g, TY) && encode_map1(&M.k_halo, kap, g, 1);
    if (d)
        ok = ok && encode_map1(&M.d_full, d, g, TY + 2) && encode_map1(&M.d_main, d, g, TY) &&
             encode_map1(&M.d_halo, d, g, 1);
    else
        M.d_full = M.d_main = M.d_halo = M.k_main;
    if (f3)
        ok = ok && encode_map4(&M.f_main, f3, g, TY);
    else
        M.f_main = M.op_main;
    return ok;
}
static thread_local int g_k10_nxr = 0;            // output plane count of the launch being issued (0: all nx)
// Lockstep tile order: CTA b takes row tile b % nty and x chunk b / nty, so the CTAs
// resident together cover contiguous bands of row tiles marching the same x planes
// and a tile's y-halo rows -- its neighbours' main rows -- are read from L2, not HBM
// (ncu at 256^3 / 512^3 with contiguous x ranges: 1.38x / 1.40x the algorithmic DRAM
// bytes).  One CTA per (tile, chunk); chunks of >= 8 planes.  OTM_K10_LOCK=0: the
// contiguous per-CTA ranges of round 1.
static thread_local int g_k10_lock = 0;
template <class K>
static dim3 k10_grid(K kernel, size_t smem, const Geo& g, int TY) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, g.nz / 2 * TY, smem);
    if (per_sm < 1) per_sm = 1;
    const int nxr = g_k10_nxr > 0 ? g_k10_nxr : g.nx;
    const long long nty = g.ny / TY;
    const long long units = nty * nxr;
    const long long slots = (long long)per_sm * sms;
    static const bool lock_on = !(getenv("OTM_K10_LOCK") && atoi(getenv("OTM_K10_LOCK")) == 0);
    g_k10_lock = 0;
    // only where a 3-case field (12 B per vertex) no longer fits half of the 126 MB L2:
    // below that the halo rows are L2 hits in any order and the contiguous ranges keep
    // every SM busy
    if (lock_on && (long long)g.nz * g.ny * nxr * 12 > (64LL << 20)) {
        long long k = std::max<long long>(1, slots / nty);
        k = std::min<long long>(k, std::max(1, nxr / 8));
        g_k10_lock = (int)k;
        return dim3((unsigned)(nty * k), 1, 1);
    }
    long long b = slots;
    if (b > units) b = units;
    return dim3((unsigned)b, 1, 1);
}
template <int NZ, int TY, int CPS, bool WZ = true>
static void l10_smooth_res(cudaStream_t s, const Geo& g, float s12, const K10Maps& M, float omega, float* z,
                           float* res) {
    const size_t sm = K10Geo<K10_SMOOTH, NZ, TY, CPS>::SMEM;
    smem_attr(k10_smooth_res<NZ, TY, CPS, WZ>, sm);
    const dim3 grid = k10_grid(k10_smooth_res<NZ, TY, CPS, WZ>, sm, g, TY);
    K10Maps Ml = M;
    Ml.lock = g_k10_lock;
    launch_pdl(k10_smooth_res<NZ, TY, CPS, WZ>, grid, dim3(NZ / 2, TY), sm, s, g, s12, Ml, omega, z, res);
}
template <bool DOT, int NZ, int TY, int CPS>
static void l10_jacobi(cudaStream_t s, const Geo& g, float s12, const K10Maps& M, float omega, float* zout,
                       double* partials, unsigned* counter, PcgScalars* sc) {
    const size_t sm = K10Geo<K10_JACOBI, NZ, TY, CPS>::SMEM;
    smem_attr(k10_jacobi<DOT, NZ, TY, CPS>, sm);
    const dim3 grid = k10_grid(k10_jacobi<DOT, NZ, TY, CPS>, sm, g, TY);
    K10Maps Ml = M;
    Ml.lock = g_k10_lock;
    launch_pdl(k10_jacobi<DOT, NZ, TY, CPS>, grid, dim3(NZ / 2, TY), sm, s, g, s12, Ml, omega, zout, partials,
               counter, sc);
}
template <int NZ, int TY, int CPS>
static void l10_spmv(cudaStream_t s, const Geo& g, float s12, const K10Maps& M, float* q, Red& red,
                     PcgScalars* sc) {
    const size_t sm = K10Geo<K10_SPMV, NZ, TY, CPS>::SMEM;
    smem_attr(k10_spmv<NZ, TY, CPS>, sm);
    const dim3 grid = k10_grid(k10_spmv<NZ, TY, CPS>, sm, g, TY);
    K10Maps Ml = M;
    Ml.lock = g_k10_lock;
    launch_pdl(k10_spmv<NZ, TY, CPS>, grid, dim3(NZ / 2, TY), sm, s, g, s12, Ml, q, red.partials, red.counter, sc);
}
// tile rows per CTA (OTM_K10_TY: 2/4/8 at nz = 128, tuning) and CTAs per SM
#define OTM_K10_SWITCH(CALL)                                                   \
    do {                                                                       \
        switch (g.nz) {                                                        \
        case 64: CALL(64, 8, 2); break;                                        \
        case 128: CALL(128, 4, 2); break;                                      \
        case 512: CALL(512, 2, 1); break;                                      \
        default: CALL(256, 2, 2); break;                                       \
        }                                                                      \
    } while (0)

bool k10_level(const Geo& g, const LevelTemplate& lt) { return k10_ok(g, lt); }
bool launch_k10_range(cudaStream_t s, int op, const Geo& g, const LevelTemplate& lt, int xa, int xb,
                      const float* kap, const float* a, const float* f, const float* dinv, float omega, float* o1,
                      float* o2, bool dot, Red& red, PcgScalars* sc) {
    if (!k10_ok(g, lt) || xa < 1 || xb > g.nx - 1 || xb <= xa) return false;
    K10Maps M;
    const float* op3 = op == 0 ? f : a;
    if (!k10_maps(M, g, op3, dinv, op == 1 ? f : nullptr, kap)) return false;
    M.xa = xa;
    M.xb = xb;
    g_k10_nxr = xb - xa;
    const float s12 = (float)lt.s12;
    if (op == 0) {
#define C_(NZ, TY, CPS) l10_smooth_res<NZ, TY, CPS>(s, g, s12, M, omega, o1, o2)
        OTM_K10_SWITCH(C_);
#undef C_
    } else if (op == 1) {
        if (dot) {
#define C_(NZ, TY, CPS) l10_jacobi<true, NZ, TY, CPS>(s, g, s12, M, omega, o1, red.partials, red.counter, sc)
            OTM_K10_SWITCH(C_);
#undef C_
        } else {
#define C_(NZ, TY, CPS) l10_jacobi<false, NZ, TY, CPS>(s, g, s12, M, omega, o1, nullptr, nullptr, sc)
            OTM_K10_SWITCH(C_);
#undef C_
        }
    } else {
#define C_(NZ, TY, CPS) l10_spmv<NZ, TY, CPS>(s, g, s12, M, o1, red, sc)
        OTM_K10_SWITCH(C_);
#undef C_
    }
    g_k10_nxr = 0;
    return true;
}
void launch_smooth_res(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* f,
                       const float* dinv, float omega, float* z, float* res) {
    if (k10_ok(g, lt)) {
        K10Maps M;
        if (k10_maps(M, g, f, dinv, nullptr, kap)) {
#define C_(NZ, TY, CPS) l10_smooth_res<NZ, TY, CPS>(s, g, (float)lt.s12, M, omega, z, res)
            OTM_K10_SWITCH(C_);
#undef C_
            return;
        }
    }
    if (small_level(g)) {
        launch_pdl(k_small<0, false>, nblk(3 * g.n, 256), 256, 0, s, g, lt, kap, nullptr, f, dinv, omega, z, res, nullptr,
                   nullptr, nullptr);
        return;
    }
    int xb;
    const dim3 grid = stencil_grid(g, &xb);
    k_smooth_res<<<grid, 128, 0, s>>>(g, xb, lt, kap, f, dinv, omega, z, res);
}
void launch_jacobi(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* z,
                   const float* f, const float* dinv, float omega, float* zout, bool dot, Red& red,
                   PcgScalars* sc) {
    if (k10_ok(g, lt)) {
        K10Maps M;
        if (k10_maps(M, g, z, dinv, f, kap)) {
            if (dot) {
#define C_(NZ, TY, CPS) l10_jacobi<true, NZ, TY, CPS>(s, g, (float)lt.s12, M, omega, zout, red.partials, red.counter, sc)
                OTM_K10_SWITCH(C_);
#undef C_
            } else {
#define C_(NZ, TY, CPS) l10_jacobi<false, NZ, TY, CPS>(s, g, (float)lt.s12, M, omega, zout, nullptr, nullptr, sc)
                OTM_K10_SWITCH(C_);
#undef C_
            }
            return;
        }
    }
    if (small_level(g)) {
        if (dot)
            launch_pdl(k_small<1, true>, nblk(3 * g.n, 256), 256, 0, s, g, lt, kap, z, f, dinv, omega, zout, nullptr,
                       red.partials, red.counter, sc);
        else
            launch_pdl(k_small<1, false>, nblk(3 * g.n, 256), 256, 0, s, g, lt, kap, z, f, dinv, omega, zout, nullptr,
                       nullptr, nullptr, sc);
        return;
    }
    int xb;
    const dim3 grid = stencil_grid(g, &xb);
    if (dot)
        k_jacobi<true><<<grid, 128, 0, s>>>(g, xb, lt, kap, z, f, dinv, omega, zout, red.partials, red.counter, sc);
    else
        k_jacobi<false><<<grid, 128, 0, s>>>(g, xb, lt, kap, z, f, dinv, omega, zout, nullptr, nullptr, sc);
}
void launch_spmv(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const float* kap, const float* p,
                 float* q, Red& red, PcgScalars* sc) {
    if (k10_ok(g, lt)) {
        K10Maps M;
        if (k10_maps(M, g, p, nullptr, nullptr, kap)) {
#define C_(NZ, TY, CPS) l10_spmv<NZ, TY, CPS>(s, g, (float)lt.s12, M, q, red, sc)
            OTM_K10_SWITCH(C_);
#undef C_
            return;
        }
    }
    int xb;
    const dim3 grid = stencil_grid(g, &xb);
    k_spmv<<<grid, 128, 0, s>>>(g, xb, lt, kap, p, q, red.partials, red.counter, sc);
}
void launch_pupd(cudaStream_t s, long long n, const float* z, float* p, float* d, const PcgScalars* sc) {
    const long long th = std::max<long long>(n >> 2, n & 3);
    launch_pdl(k_pupd, nblk(th, 256), 256, 0, s, n, z, p, d, sc);
}
void launch_upd(cudaStream_t s, long long n, float* r, const float* q, Red& red, PcgScalars* sc,
                unsigned long long loop) {
    const long long th = std::max<long long>(n >> 2, n & 3);
    const unsigned cap = gs_cap(n);
    if (cap && nblk(th, 256) > cap)
        launch_pdl(k_upd<true>, cap, 256, 0, s, n, r, q, red.partials, red.counter, sc, loop);
    else
        launch_pdl(k_upd<false>, nblk(th, 256), 256, 0, s, n, r, q, red.partials, red.counter, sc, loop);
}
void launch_restrict(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* res, float* fc) {
    if (cf[0] && cf[1] && cf[2]) {
        // two coarse z per thread where the coarse rows allow it (OTM_RESTRICT_V=0: off)
        static const bool rv = !(getenv("OTM_RESTRICT_V") && atoi(getenv("OTM_RESTRICT_V")) == 0);
        if (rv && c.nz % 64 == 0 && 3LL * c.nx <= 65535)
            launch_pdl(k_restrict3v, dim3(nblk((long long)c.ny * (c.nz / 2), 256), 3 * c.nx), 256, 0, s, f, c, res,
                       fc);
        else if (c.nz % 32 == 0)
            launch_pdl(k_restrict3w, nblk(3 * c.n, 256), 256, 0, s, f, c, res, fc);
        else
            launch_pdl(k_restrict3, nblk(3 * c.n, 256), 256, 0, s, f, c, res, fc);
        return;
    }
    k_restrict<<<nblk(c.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], res, fc);
}
void launch_prolong(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const float* zc, float* zf) {
    if (cf[0] && cf[1] && cf[2]) {
        static const bool pc = !(getenv("OTM_PROLONG_C") && atoi(getenv("OTM_PROLONG_C")) == 0);
        if (pc && 3LL * c.nx <= 65535)
            launch_pdl(k_prolong3c<false>, dim3(nblk(c.pl, 256), 3 * c.nx), 256, 0, s, f, c, zc, zf);
        else
            launch_pdl(k_prolong3b<false>, nblk(3 * c.n, 256), 256, 0, s, f, c, zc, zf);
        return;
    }
    k_prolong<<<nblk(f.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], zc, zf);
}
void launch_vbottom(cudaStream_t s, int N, const VBotArgs& a) {
    if (N == 16) {
        const size_t sm = (size_t)vbot_smem_floats(16) * 4;
        smem_attr(k_vbottom<16>, sm);
        launch_pdl(k_vbottom<16>, dim3(1), dim3(1024), sm, s, a);
    } else {
        const size_t sm = (size_t)vbot_smem_floats(8) * 4;
        smem_attr(k_vbottom<8>, sm);
        launch_pdl(k_vbottom<8>, dim3(1), dim3(1024), sm, s, a);
    }
}
void launch_Tupd(cudaStream_t s, long long n, double* T, const float* d, const float* p, const PcgScalars* sc) {
    k_Tupd<<<nblk(3 * n, 256), 256, 0, s>>>(n, T, d, p, sc);
}
void launch_submean_means(cudaStream_t s, long long n, double* T, const double* means) {
    k_submean_means<<<nblk(3 * n, 256), 256, 0, s>>>(n, T, means);
}
void launch_submean(cudaStream_t s, long long n, double* T, const double* sumT) {
    k_submean<<<nblk(3 * n, 256), 256, 0, s>>>(n, T, sumT);
}
// x chunks per (y, z) column: about 2 waves of the kernel's resident threads,
// >= 4 planes each (a chunk reloads its first plane)
void launch_tensor(cudaStream_t s, const Geo& g, const double* T, const double* kap, Red& red, double* out6,
                   const XRange* xr) {
    static thread_local int ch = 0, for_pl = -1, for_np = -1;
    const XRange r = whole(g, xr);
    chunks_for(k_tensor_x, g, r.xb - r.xa, ch, for_pl, for_np);
    const long long th = (long long)g.pl * ch;
    k_tensor_x<<<nblk(th, 256), 256, 0, s>>>(g, ch, r, T, kap, red.partials, red.counter, out6);
}
// HomogenizationResult.elem_diff (homogenize.py:94-100): w[e, a] = c_a[i] - T_i[e + c_a]
// as float32, element e = its lower corner, corners periodic
__global__ void k_elem_diff(Geo g, const double* __restrict__ T, int ci, float* __restrict__ w) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.n) return;
    const int x = (int)(e / g.pl), rem = (int)(e - (long long)x * g.pl);
    const int y = rem / g.nz, z = rem - y * g.nz;
    const int xs[2] = {x, wrap_p(x, g.nx)}, ys[2] = {y, wrap_p(y, g.ny)}, zs[2] = {z, wrap_p(z, g.nz)};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const int bx = a & 1, by = (a >> 1) & 1, bz = (a >> 2) & 1;
        const double c = (double)((a >> ci) & 1);
        w[e * 8 + a] = (float)(c - T[((long long)xs[bx] * g.ny + ys[by]) * g.nz + zs[bz]]);
    }
}
void launch_elem_diff(cudaStream_t s, const Geo& g, const double* T, int ci, float* w) {
    k_elem_diff<<<nblk(g.n, 256), 256, 0, s>>>(g, T, ci, w);
}
void launch_pair_energy(cudaStream_t s, const Geo& g, const double* T, double* E) {
    k_pair_energy<<<nblk(g.n, 256), 256, 0, s>>>(g, T, E);
}
void launch_sens(cudaStream_t s, const Geo& g, const double* T, const double* rf, const SimpParams& sp,
                 const Dg& dG, double* sens, const Dg* dG_dev, const XRange* xr) {
    static thread_local int ch = 0, for_pl = -1, for_np = -1;
    const XRange r = whole(g, xr);
    chunks_for(k_sens_x, g, r.xb - r.xa, ch, for_pl, for_np);
    const long long th = (long long)g.pl * ch;
    k_sens_x<<<nblk(th, 256), 256, 0, s>>>(g, ch, r, T, rf, sp, dG, dG_dev, sens);
}
void launch_oc_eval(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a, int nlam,
                    const LamSet& lam_pow, Red& red, double* out) {
    long long want = (n + 255) / 256;
    unsigned blocks = (unsigned)(want < 592 ? want : 592);
    k_oc_eval<<<blocks, 256, 0, s>>>(n, rho, sens, a, nlam, lam_pow, red.partials, red.counter, out);
}
int launch_oc_coop(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a,
                   double* rho_out, OcCtl* ctl, double* partials, double* qbuf, double* lam_mem) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // beyond L2 (rho and c_e > 64 MB) the search is bound by loads in flight: the
    // shared-memory accumulators' third CTA per SM pays (512^3: 11.2 -> 8.3 ms per
    // single-pass update); at 128^3 the register version is faster (21.5 vs 23.8 ms
    // per 200 updates).  OTM_OC_SMACC=0/1 forces either.
    static const int smacc_env = getenv("OTM_OC_SMACC") ? atoi(getenv("OTM_OC_SMACC")) : -1;
    const bool smacc = smacc_env >= 0 ? smacc_env == 1 : n * 16 > (64LL << 20);
    const size_t dyn = smacc ? (size_t)kOcLam * 256 * sizeof(double) : 0;
    void* kern = smacc ? (void*)k_oc_coop<true> : (void*)k_oc_coop<false>;
    if (smacc) smem_attr(k_oc_coop<true>, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, dyn);
    if (per_sm < 1) return 1;
    long long want = (n + 255) / 256;
    long long blocks = (long long)per_sm * sms;
    if (blocks > want) blocks = want;
    if (blocks < 1) blocks = 1;
    void* args[] = {(void*)&n,       (void*)&rho, (void*)&sens,     (void*)&a,        (void*)&rho_out,
                    (void*)&ctl,     (void*)&partials, (void*)&qbuf, (void*)&lam_mem};
    return cudaLaunchCooperativeKernel(kern, dim3((unsigned)blocks), dim3(256), args, dyn, s) == cudaSuccess
               ? 0 : 1;
}
void launch_oc_apply(cudaStream_t s, long long n, const double* rho, const double* sens, const OcArgs& a,
                     double lam, double* rho_out, int* changed) {
    k_oc_apply<<<nblk(n, 256), 256, 0, s>>>(n, rho, sens, a, lam, rho_out, changed);
}

}  // namespace otm
