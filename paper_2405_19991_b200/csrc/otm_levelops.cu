// API-level multigrid operations in fp64 (solver.py:85-338).
//
// The reference exposes its multigrid pieces as functions over mutable level
// arrays: relax_gs8 (8-colour Gauss-Seidel), restrict, prolong_correct,
// coarse_solve, GridHierarchy.vcycle, and apply_K on any level.  The design loop
// never calls them -- it runs the batched fp32 MG-PCG with a damped-Jacobi
// V-cycle (otm_kernels.cu) -- so these kernels are written for exactness, not
// bandwidth: fp64 throughout, the matrix-free element operator evaluated per
// vertex from the level's child-mean factors (no 27 stored coefficient arrays),
// any level shape including flat (n = 1) and two-vertex (n = 2) axes.
//
// Operator of level l (solver.py:85-119): (K T)[v] = sum over the 8 elements e
// around v (e = v - c_a) of kappa_e sum_b K_l[a][b] T[e + c_b], periodic, with
// K_l[a][b] = kt[a ^ b] (box element: the entry depends only on which axes
// differ).  Couplings that wrap back onto v itself (flat axes) are part of the
// diagonal, exactly as _fold merges them into W[(0,0,0)] (solver.py:56-63, 97-105).
#include "otm_common.cuh"
#include "otm_internal.h"

namespace otm {

namespace {

__device__ __forceinline__ int wrapi(int i, int n) {
    i %= n;
    return i < 0 ? i + n : i;
}
__device__ __forceinline__ long long vid(const Geo& g, int x, int y, int z) {
    return ((long long)x * g.ny + y) * g.nz + z;
}
__device__ __forceinline__ void vxyz(const Geo& g, long long v, int& x, int& y, int& z) {
    x = (int)(v / g.pl);
    const long long r = v - (long long)x * g.pl;
    y = (int)(r / g.nz);
    z = (int)(r - (long long)y * g.nz);
}

// diagonal (self couplings) and off-diagonal sum sum_{u != v} K[v][u] T[u] of row v
__device__ void row_terms(const Geo& g, const LevelTemplate& lt, const double* __restrict__ kap,
                          const double* __restrict__ T, int x, int y, int z, double& diag, double& off) {
    diag = 0.0;
    off = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int ex = wrapi(x - (a & 1), g.nx), ey = wrapi(y - ((a >> 1) & 1), g.ny),
                  ez = wrapi(z - ((a >> 2) & 1), g.nz);
        const double ke = kap[vid(g, ex, ey, ez)];
        for (int b = 0; b < 8; ++b) {
            const int ux = wrapi(ex + (b & 1), g.nx), uy = wrapi(ey + ((b >> 1) & 1), g.ny),
                      uz = wrapi(ez + ((b >> 2) & 1), g.nz);
            const double coef = lt.kt[a ^ b] * ke;
            if (ux == x && uy == y && uz == z) diag += coef;
            else off += coef * T[vid(g, ux, uy, uz)];
        }
    }
}

__global__ void k_lv_apply(Geo g, LevelTemplate lt, const double* __restrict__ kap, const double* __restrict__ T,
                           const double* __restrict__ f, double* __restrict__ out) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.n) return;
    int x, y, z;
    vxyz(g, v, x, y, z);
    double diag, off;
    row_terms(g, lt, kap, T, x, y, z, diag, off);
    const double kt = diag * T[v] + off;
    out[v] = f ? f[v] - kt : kt;          // residual f - K T (solver.py:334) or K T
}

// one colour (cx, cy, cz) of relax_gs8 (solver.py:131-164): no two vertices of a
// colour share an element, so the colour updates at once from the other colours
__global__ void k_lv_gs_color(Geo g, LevelTemplate lt, const double* __restrict__ kap, const double* __restrict__ f,
                              double* T, int cx, int cy, int cz) {
    const int hx = g.nx > 1 ? g.nx / 2 : 1, hy = g.ny > 1 ? g.ny / 2 : 1, hz = g.nz > 1 ? g.nz / 2 : 1;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)hx * hy * hz) return;
    const int X = (int)(i / ((long long)hy * hz));
    const int rem = (int)(i - (long long)X * hy * hz);
    const int Y = rem / hz, Z = rem - Y * hz;
    const int x = g.nx > 1 ? 2 * X + cx : 0, y = g.ny > 1 ? 2 * Y + cy : 0, z = g.nz > 1 ? 2 * Z + cz : 0;
    double diag, off;
    row_terms(g, lt, kap, T, x, y, z, diag, off);
    T[vid(g, x, y, z)] = (f[vid(g, x, y, z)] - off) / diag;
}

// child-mean factors (solver.py:257-267): pairs along x, then y, then z, each a
// two-element mean -- numpy's reshape(...).mean order
__global__ void k_lv_coarsen(Geo f, Geo c, int cx, int cy, int cz, const double* __restrict__ kf,
                             double* __restrict__ kc) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= c.n) return;
    int X, Y, Z;
    vxyz(c, v, X, Y, Z);
    double q[2][2];
    for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k) {
            const int y = cy ? 2 * Y + j : Y, z = cz ? 2 * Z + k : Z;
            q[j][k] = cx ? (kf[vid(f, 2 * X, y, z)] + kf[vid(f, 2 * X + 1, y, z)]) / 2.0 : kf[vid(f, X, y, z)];
        }
    double r[2];
    for (int k = 0; k < 2; ++k) r[k] = cy ? (q[0][k] + q[1][k]) / 2.0 : q[0][k];
    kc[v] = cz ? (r[0] + r[1]) / 2.0 : r[0];
}

// full-weighting restriction (solver.py:167-177): [1/4, 1/2, 1/4] on every coarsened
// axis, then the even subsample
__global__ void k_lv_restrict(Geo f, Geo c, int cx, int cy, int cz, const double* __restrict__ r,
                              double* __restrict__ fc) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= c.n) return;
    int X, Y, Z;
    vxyz(c, v, X, Y, Z);
    const int cf[3] = {cx, cy, cz};
    double acc = 0.0;
    for (int ox = -cf[0]; ox <= cf[0]; ++ox) {
        const double wx = cf[0] ? (ox == 0 ? 0.5 : 0.25) : 1.0;
        const int x = wrapi(cf[0] ? 2 * X + ox : X, f.nx);
        for (int oy = -cf[1]; oy <= cf[1]; ++oy) {
            const double wy = cf[1] ? (oy == 0 ? 0.5 : 0.25) : 1.0;
            const int y = wrapi(cf[1] ? 2 * Y + oy : Y, f.ny);
            for (int oz = -cf[2]; oz <= cf[2]; ++oz) {
                const double wz = cf[2] ? (oz == 0 ? 0.5 : 0.25) : 1.0;
                const int z = wrapi(cf[2] ? 2 * Z + oz : Z, f.nz);
                acc += wx * wy * wz * r[vid(f, x, y, z)];
            }
        }
    }
    fc[v] = acc;
}

// trilinear prolongation + correction (solver.py:180-200): even fine index = coarse
// value, odd = mean of the two coarse neighbours (periodic)
__global__ void k_lv_prolong(Geo f, Geo c, int cx, int cy, int cz, const double* __restrict__ Tc,
                             double* __restrict__ Tf) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= f.n) return;
    int x, y, z;
    vxyz(f, v, x, y, z);
    int ix[2], iy[2], iz[2];
    double wx[2], wy[2], wz[2];
    auto axis = [](int i, int cfa, int nc, int (&idx)[2], double (&w)[2]) {
        if (!cfa) { idx[0] = idx[1] = i; w[0] = 1.0; w[1] = 0.0; return; }
        idx[0] = i >> 1;
        if (i & 1) { idx[1] = wrapi((i >> 1) + 1, nc); w[0] = w[1] = 0.5; }
        else { idx[1] = idx[0]; w[0] = 1.0; w[1] = 0.0; }
    };
    axis(x, cx, c.nx, ix, wx);
    axis(y, cy, c.ny, iy, wy);
    axis(z, cz, c.nz, iz, wz);
    double acc = 0.0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d) {
                const double w = wx[a] * wy[b] * wz[d];
                if (w != 0.0) acc += w * Tc[vid(c, ix[a], iy[b], iz[d])];
            }
    Tf[v] += acc;
}

// dense coarsest-level matrix with vertex 0 pinned (solver.py:278-305): M = A[1:, 1:]
__global__ void k_lv_assemble(Geo g, LevelTemplate lt, const double* __restrict__ kap, double* __restrict__ M) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= g.n || v == 0) return;
    const long long m = g.n - 1;
    int x, y, z;
    vxyz(g, v, x, y, z);
    double* row = M + (v - 1) * m;
    for (long long j = 0; j < m; ++j) row[j] = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int ex = wrapi(x - (a & 1), g.nx), ey = wrapi(y - ((a >> 1) & 1), g.ny),
                  ez = wrapi(z - ((a >> 2) & 1), g.nz);
        const double ke = kap[vid(g, ex, ey, ez)];
        for (int b = 0; b < 8; ++b) {
            const long long u = vid(g, wrapi(ex + (b & 1), g.nx), wrapi(ey + ((b >> 1) & 1), g.ny),
                                    wrapi(ez + ((b >> 2) & 1), g.nz));
            if (u > 0) row[u - 1] += lt.kt[a ^ b] * ke;
        }
    }
}

// in-place Gauss-Jordan inversion of the SPD pinned matrix, pivot k: the Schur
// update of every entry off row/column k, then the pivot row/column (separate
// launches: the update reads row and column k)
__global__ void k_lv_gj_update(double* M, int m, int k) {
    const int i = blockIdx.y * blockDim.y + threadIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || j >= m || i == k || j == k) return;
    const double p = 1.0 / M[(long long)k * m + k];
    M[(long long)i * m + j] -= M[(long long)i * m + k] * M[(long long)k * m + j] * p;
}
__global__ void k_lv_gj_pivot(double* M, int m, int k) {     // one CTA
    const double p = 1.0 / M[(long long)k * m + k];
    for (int t = threadIdx.x; t < m; t += blockDim.x)
        if (t != k) {
            M[(long long)k * m + t] *= p;
            M[(long long)t * m + k] *= -p;
        }
    __syncthreads();
    if (threadIdx.x == 0) M[(long long)k * m + k] = p;
}

// coarse_solve (solver.py:307-324): project the mean out of f, x[1:] = M^-1 f[1:],
// x[0] = 0, subtract the mean of x.  One CTA (the coarsest level has <= 2048
// vertices); fixed-order sums.
__global__ void __launch_bounds__(1024) k_lv_coarse_solve(int n, const double* __restrict__ Minv,
                                                          const double* __restrict__ f, double* __restrict__ T) {
    __shared__ double red[32];
    __shared__ double sh_mean;
    extern __shared__ double fx[];       // n doubles: the projected load, then x
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += f[i];
    double v[1] = {s};
    block_sum<1>(v, red);
    if (threadIdx.x == 0) sh_mean = v[0] / n;
    __syncthreads();
    const double fmean = sh_mean;
    for (int i = threadIdx.x; i < n; i += blockDim.x) fx[i] = f[i] - fmean;
    __syncthreads();
    const int m = n - 1;
    double xs = 0.0;
    double xv[2] = {0.0, 0.0};
    const int per = (n + blockDim.x - 1) / blockDim.x;    // <= 2 rows per thread
    for (int k = 0; k < per; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i == 0 || i >= n) continue;
        double acc = 0.0;
        const double* row = Minv + (long long)(i - 1) * m;
        for (int j = 0; j < m; ++j) acc += row[j] * fx[j + 1];
        xv[k] = acc;
        xs += acc;
    }
    double w[1] = {xs};
    __syncthreads();
    block_sum<1>(w, red);
    if (threadIdx.x == 0) sh_mean = w[0] / n;
    __syncthreads();
    const double xmean = sh_mean;
    for (int k = 0; k < per; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= n) continue;
        T[i] = (i == 0 ? 0.0 : xv[k]) - xmean;
    }
}

inline unsigned nb(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

void launch_lv_apply(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* T,
                     const double* f, double* out) {
    k_lv_apply<<<nb(g.n, 256), 256, 0, s>>>(g, lt, kap, T, f, out);
}

void launch_lv_gs8(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, const double* f, double* T,
                   int sweeps) {
    const int hx = g.nx > 1 ? g.nx / 2 : 1, hy = g.ny > 1 ? g.ny / 2 : 1, hz = g.nz > 1 ? g.nz / 2 : 1;
    const long long per = (long long)hx * hy * hz;
    // colour order of _colors (solver.py:122-128): cx outermost, cz innermost
    for (int sw = 0; sw < sweeps; ++sw)
        for (int cx = 0; cx < (g.nx > 1 ? 2 : 1); ++cx)
            for (int cy = 0; cy < (g.ny > 1 ? 2 : 1); ++cy)
                for (int cz = 0; cz < (g.nz > 1 ? 2 : 1); ++cz)
                    k_lv_gs_color<<<nb(per, 256), 256, 0, s>>>(g, lt, kap, f, T, cx, cy, cz);
}

void launch_lv_coarsen(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* kf, double* kc) {
    k_lv_coarsen<<<nb(c.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], kf, kc);
}

void launch_lv_restrict(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* r, double* fc) {
    k_lv_restrict<<<nb(c.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], r, fc);
}

void launch_lv_prolong(cudaStream_t s, const Geo& f, const Geo& c, const int cf[3], const double* Tc, double* Tf) {
    k_lv_prolong<<<nb(f.n, 256), 256, 0, s>>>(f, c, cf[0], cf[1], cf[2], Tc, Tf);
}

void launch_lv_coarse_factor(cudaStream_t s, const Geo& g, const LevelTemplate& lt, const double* kap, double* M) {
    const int m = (int)g.n - 1;
    if (m < 1) return;
    k_lv_assemble<<<nb(g.n, 128), 128, 0, s>>>(g, lt, kap, M);
    const dim3 blk(32, 8), grd(nb(m, 32), nb(m, 8));
    for (int k = 0; k < m; ++k) {
        k_lv_gj_update<<<grd, blk, 0, s>>>(M, m, k);
        k_lv_gj_pivot<<<1, 1024, 0, s>>>(M, m, k);
    }
}

void launch_lv_coarse_solve(cudaStream_t s, int n, const double* Minv, const double* f, double* T) {
    k_lv_coarse_solve<<<1, 1024, (size_t)n * sizeof(double), s>>>(n, Minv, f, T);
}

}  // namespace otm
