// libotm slab kernels: the level-0 .. agglomeration-level pieces of the homogenization
// solve on an x-slab of the periodic grid.
//
// A slab owns nxl consecutive x planes of a level; every field is stored with one
// ghost plane on each side, (nxl + 2) planes of ny * nz values (3 load cases
// case-major: case c at c * (nxl + 2) * ny * nz).  Ghost planes are refreshed by
// the caller (NCCL send/recv between neighbouring ranks) before any kernel that
// reads them; kernels write interior planes only.  y and z stay periodic inside the
// slab.  Element factors use the element = lower-corner vertex convention, so a
// vertex needs the factor ghost on the left only.  Scalars (dot products, norms,
// tensor sums) are per-slab fixed-order partial sums; the caller all-reduces them.
#include "otm_common.cuh"
#include "otm_internal.h"
#include "../../include/otm.h"
#include "../../include/otm_slab.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>

void level_template(const double scale[3], otm::LevelTemplate& lt);   // otm_api.cu
void filter_weights(double radius, std::vector<int>& offs, std::vector<double>& w);   // otm_api.cu

namespace otm {
namespace {

struct W27 {
    double w[27];
};

struct SGeo {
    int nxl, ny, nz;
    int pl;             // ny * nz
    long long ni;       // items per case: nxl * pl (a plane range: its planes * pl)
    long long na;       // allocated values per case: (nxl + 2) * pl
    int x0;             // first item plane (1: the whole interior)
};

SGeo make_sgeo(int nxl, int ny, int nz) {
    SGeo g;
    g.nxl = nxl; g.ny = ny; g.nz = nz;
    g.pl = ny * nz;
    g.ni = (long long)nxl * g.pl;
    g.na = (long long)(nxl + 2) * g.pl;
    g.x0 = 1;
    return g;
}

// item i (0 .. ni-1) -> local plane (x0 .. ; 1 .. nxl for the interior), y, z
__device__ __forceinline__ void s_decode(const SGeo& g, long long i, int& x, int& y, int& z) {
    x = (int)(i / g.pl);
    const int rem = (int)(i - (long long)x * g.pl);
    y = rem / g.nz;
    z = rem - y * g.nz;
    x += g.x0;
}

// 27 operand values around (x, y, z): x from the ghosted planes, y/z periodic
template <int OP>
__device__ __forceinline__ void s_gather(const SGeo& g, const float* __restrict__ a, const float* __restrict__ dinv,
                                         float omega, int x, int y, int z, float (&t)[3][9]) {
    const int ys[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
    const int zs[3] = {wrap_m(z, g.nz), z, wrap_p(z, g.nz)};
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const long long idx = (long long)(x - 1 + p) * g.pl + ys[j] + zs[q];
                float v = __ldg(a + idx);
                if (OP == 0) v *= omega * __ldg(dinv + idx);
                t[p][j * 3 + q] = v;
            }
}

// factors of the 8 elements around the vertex: planes x-1, x; rows y-1, y; cols z-1, z
__device__ __forceinline__ void s_kappa(const SGeo& g, const float* __restrict__ k, int x, int y, int z,
                                        float (&kk)[2][4]) {
    const int ys[2] = {wrap_m(y, g.ny) * g.nz, y * g.nz};
    const int zs[2] = {wrap_m(z, g.nz), z};
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) kk[p][j * 2 + q] = __ldg(k + (long long)(x - 1 + p) * g.pl + ys[j] + zs[q]);
}

__device__ __forceinline__ float s_apply(const LevelTemplate& lt, const float (&t)[3][9], const float (&k)[2][4]) {
    if (lt.equal) {
        const KSum<float> s = ksum<float>(k);
        return apply_compact<float>(t, k, s, (float)lt.s12);
    }
    float ktab[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) ktab[q] = (float)lt.kt[q];
    return apply_generic<float>(t, k, ktab);
}

// OP 0 smooth_res: z = w D^-1 f, res = f - K z          (o1 = z, o2 = res)
// OP 1 jacobi:     zout = z + w D^-1 (f - K z); dot f.zout (o1 = zout)
// OP 2 spmv:       q = K p; dot p.q                       (o1 = q)
template <int OP>
__global__ void __launch_bounds__(256) ks_stencil(SGeo g, LevelTemplate lt, const float* __restrict__ kap,
                                                  const float* __restrict__ a, const float* __restrict__ f,
                                                  const float* __restrict__ dinv, float omega, float* __restrict__ o1,
                                                  float* __restrict__ o2, int dot, double* partials,
                                                  unsigned* counter, double* out3) {
    double d3[3] = {0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * g.ni; i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i / g.ni);
        const long long v = i - (long long)c * g.ni;
        int x, y, z;
        s_decode(g, v, x, y, z);
        const long long off = (long long)c * g.na;
        const long long idx = (long long)x * g.pl + y * g.nz + z;
        float t[3][9], k[2][4];
        s_gather<OP>(g, (OP == 0 ? f : a) + off, dinv, omega, x, y, z, t);
        s_kappa(g, kap, x, y, z, k);
        const float kt = s_apply(lt, t, k);
        if (OP == 0) {
            o1[off + idx] = t[1][4];
            o2[off + idx] = __ldg(f + off + idx) - kt;
        } else if (OP == 1) {
            const float fv = __ldg(f + off + idx);
            const float zn = t[1][4] + omega * __ldg(dinv + idx) * (fv - kt);
            o1[off + idx] = zn;
            d3[c] += (double)fv * (double)zn;
        } else {
            o1[off + idx] = kt;
            d3[c] += (double)t[1][4] * (double)kt;
        }
    }
    if (dot && reduce_finalize<3>(d3, partials, counter, out3)) {}
}

// full-weighting restriction: coarse interior J <- fine local 2J-2 .. 2J (x), periodic y/z
__global__ void ks_restrict(SGeo f, SGeo c, const float* __restrict__ res, float* __restrict__ fc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * c.ni) return;
    const int cc = (int)(i / c.ni);
    int X, Y, Z;
    s_decode(c, i - (long long)cc * c.ni, X, Y, Z);
    const int xs[3] = {2 * X - 2, 2 * X - 1, 2 * X};
    const int ys[3] = {wrap_m(2 * Y, f.ny) * f.nz, 2 * Y * f.nz, wrap_p(2 * Y, f.ny) * f.nz};
    const int zs[3] = {wrap_m(2 * Z, f.nz), 2 * Z, wrap_p(2 * Z, f.nz)};
    const float w[3] = {0.25f, 0.5f, 0.25f};
    const float* r = res + (long long)cc * f.na;
    float s = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float sb = 0.f;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const float* row = r + (long long)xs[a] * f.pl + ys[b];
            const float sz = w[0] * __ldg(row + zs[0]) + w[1] * __ldg(row + zs[1]) + w[2] * __ldg(row + zs[2]);
            sb += w[b] * sz;
        }
        s += w[a] * sb;
    }
    fc[(long long)cc * c.na + (long long)X * c.pl + Y * c.nz + Z] = s;
}

// trilinear prolongation + correction: fine interior i <- coarse local (i+1)/2 (+1 for odd offsets)
__global__ void ks_prolong(SGeo f, SGeo c, const float* __restrict__ zc, float* __restrict__ zf) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * f.ni) return;
    const int cc = (int)(i / f.ni);
    int x, y, z;
    s_decode(f, i - (long long)cc * f.ni, x, y, z);
    // fine local x (1..nxl) is global 2*X0 + x - 1: even offsets (x odd) sit on coarse local (x+1)/2
    const int J0 = (x + 1) >> 1;
    const int J1 = (x & 1) ? J0 : J0 + 1;
    const float wx1 = (x & 1) ? 0.f : 0.5f, wx0 = 1.f - wx1;
    const int Y0 = y >> 1, Z0 = z >> 1;
    const int Y1 = Y0 + 1 == c.ny ? 0 : Y0 + 1, Z1 = Z0 + 1 == c.nz ? 0 : Z0 + 1;
    const float wy1 = (y & 1) ? 0.5f : 0.f, wz1 = (z & 1) ? 0.5f : 0.f;
    const float wy0 = 1.f - wy1, wz0 = 1.f - wz1;
    const float* a = zc + (long long)cc * c.na;
    auto at = [&](int X, int Y, int Z) { return __ldg(a + (long long)X * c.pl + Y * c.nz + Z); };
    const float s = wx0 * (wy0 * (wz0 * at(J0, Y0, Z0) + wz1 * at(J0, Y0, Z1)) +
                           wy1 * (wz0 * at(J0, Y1, Z0) + wz1 * at(J0, Y1, Z1))) +
                    wx1 * (wy0 * (wz0 * at(J1, Y0, Z0) + wz1 * at(J1, Y0, Z1)) +
                           wy1 * (wz0 * at(J1, Y1, Z0) + wz1 * at(J1, Y1, Z1)));
    zf[(long long)cc * f.na + (long long)x * f.pl + y * f.nz + z] += s;
}

// prolongation + correction, one thread per coarse interior vertex (case, X, Y, Z):
// the fine block x = 2X-1 (on coarse X), 2X (between X and X+1, the right ghost),
// y = 2Y, 2Y+1, z pair (2Z, 2Z+1) as float2 read-modify-writes (as k_prolong3b)
__global__ void ks_prolong_b(SGeo f, SGeo c, const float* __restrict__ zc, float* __restrict__ zf) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * c.ni) return;
    const int cc = (int)(i / c.ni);
    int X, Y, Z;
    s_decode(c, i - (long long)cc * c.ni, X, Y, Z);
    const int Y1 = Y + 1 == c.ny ? 0 : Y + 1, Z1 = Z + 1 == c.nz ? 0 : Z + 1;
    const float* a = zc + (long long)cc * c.na;
    float q[2][2][2];
    const int xs[2] = {X, X + 1}, ys[2] = {Y, Y1}, zs[2] = {Z, Z1};
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int k = 0; k < 2; ++k) q[p][j][k] = __ldg(a + (long long)xs[p] * c.pl + ys[j] * c.nz + zs[k]);
    float* out = zf + (long long)cc * f.na;
#pragma unroll
    for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
            float v[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {                  // fine z = 2Z + h
                float qy[2];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float z0 = q[p][0][0] * (h ? 0.5f : 1.f) + (h ? 0.5f * q[p][0][1] : 0.f);
                    const float z1 = q[p][1][0] * (h ? 0.5f : 1.f) + (h ? 0.5f * q[p][1][1] : 0.f);
                    qy[p] = b2 ? 0.5f * (z0 + z1) : z0;
                }
                v[h] = a2 ? 0.5f * (qy[0] + qy[1]) : qy[0];
            }
            float2* dst = reinterpret_cast<float2*>(out + (long long)(2 * X - 1 + a2) * f.pl + (2 * Y + b2) * f.nz + 2 * Z);
            float2 cur = *dst;
            cur.x += v[0];
            cur.y += v[1];
            *dst = cur;
        }
}

// p = z + beta p on the interior, float4, blockIdx.y = case (pl % 4 == 0)
__global__ void ks_pupd4(SGeo g, const float* __restrict__ z, float* __restrict__ p, double b0, double b1, double b2,
                         const double* __restrict__ bdev) {
    const int c = blockIdx.y;
    const float b = (float)(bdev ? bdev[c] : (c == 0 ? b0 : (c == 1 ? b1 : b2)));
    const long long base = (long long)c * g.na + g.pl;
    const float4* zz = reinterpret_cast<const float4*>(z + base);
    float4* pp = reinterpret_cast<float4*>(p + base);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni / 4; i += (long long)gridDim.x * blockDim.x) {
        const float4 zv = __ldg(zz + i);
        const float4 pv = pp[i];
        pp[i] = make_float4(zv.x + b * pv.x, zv.y + b * pv.y, zv.z + b * pv.z, zv.w + b * pv.w);
    }
}

// d += alpha p, r -= alpha q, partial r.r; float4, blockIdx.y = case (pl % 4 == 0)
__global__ void __launch_bounds__(256) ks_upd4(SGeo g, float* __restrict__ d, float* __restrict__ r,
                                               const float* __restrict__ p, const float* __restrict__ q, double a0,
                                               double a1, double a2, double* partials, unsigned* counter,
                                               double* out3, const double* __restrict__ adev) {
    const int c = blockIdx.y;
    const float al = (float)(adev ? adev[c] : (c == 0 ? a0 : (c == 1 ? a1 : a2)));
    const long long base = (long long)c * g.na + g.pl;
    float4* dd = reinterpret_cast<float4*>(d + base);
    float4* rr = reinterpret_cast<float4*>(r + base);
    const float4* pp = reinterpret_cast<const float4*>(p + base);
    const float4* qq = reinterpret_cast<const float4*>(q + base);
    double d3[3] = {0.0, 0.0, 0.0};
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni / 4; i += (long long)gridDim.x * blockDim.x) {
        const float4 pv = __ldg(pp + i), qv = __ldg(qq + i);
        float4 dv = dd[i], rv = rr[i];
        dv.x += al * pv.x; dv.y += al * pv.y; dv.z += al * pv.z; dv.w += al * pv.w;
        rv.x -= al * qv.x; rv.y -= al * qv.y; rv.z -= al * qv.z; rv.w -= al * qv.w;
        dd[i] = dv;
        rr[i] = rv;
        acc += ((double)rv.x * rv.x + (double)rv.y * rv.y) + ((double)rv.z * rv.z + (double)rv.w * rv.w);
    }
    d3[c] = acc;
    reduce_finalize<3>(d3, partials, counter, out3);
}

// child-mean factors: coarse element J <- fine elements 2J-1, 2J (local x), 2x2 in y/z
__global__ void ks_coarsen(SGeo f, SGeo c, const float* __restrict__ kf, float* __restrict__ kc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.ni) return;
    int X, Y, Z;
    s_decode(c, i, X, Y, Z);
    float s = 0.f;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d) s += kf[(long long)(2 * X - 1 + a) * f.pl + (2 * Y + b) * f.nz + 2 * Z + d];
    kc[(long long)X * c.pl + Y * c.nz + Z] = s / 8.f;
}

__global__ void ks_dinv(SGeo g, const float* __restrict__ k, float kdiag, float* __restrict__ dinv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.ni) return;
    int x, y, z;
    s_decode(g, i, x, y, z);
    const int ys[2] = {wrap_m(y, g.ny), y}, zs[2] = {wrap_m(z, g.nz), z};
    float s = 0.f;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int d = 0; d < 2; ++d) s += k[(long long)(x - 1 + a) * g.pl + ys[b] * g.nz + zs[d]];
    dinv[(long long)x * g.pl + y * g.nz + z] = 1.0f / (kdiag * s);
}

// p = z + beta p (interior)
__global__ void ks_pupd(SGeo g, const float* __restrict__ z, float* __restrict__ p, double b0, double b1,
                        double b2, const double* __restrict__ bdev) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * g.ni) return;
    const int c = (int)(i / g.ni);
    const long long idx = (long long)c * g.na + g.pl + (i - (long long)c * g.ni);
    const float b = (float)(bdev ? bdev[c] : (c == 0 ? b0 : (c == 1 ? b1 : b2)));
    p[idx] = z[idx] + b * p[idx];
}

// d += alpha p, r -= alpha q, partial r.r (interior)
__global__ void __launch_bounds__(256) ks_upd(SGeo g, float* __restrict__ d, float* __restrict__ r,
                                              const float* __restrict__ p, const float* __restrict__ q, double a0,
                                              double a1, double a2, double* partials, unsigned* counter,
                                              double* out3, const double* __restrict__ adev) {
    double d3[3] = {0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * g.ni; i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i / g.ni);
        const long long idx = (long long)c * g.na + g.pl + (i - (long long)c * g.ni);
        const float al = (float)(adev ? adev[c] : (c == 0 ? a0 : (c == 1 ? a1 : a2)));
        d[idx] += al * p[idx];
        const float rn = r[idx] - al * q[idx];
        r[idx] = rn;
        d3[c] += (double)rn * (double)rn;
    }
    reduce_finalize<3>(d3, partials, counter, out3);
}

// fp64 defect r = (f(kappa) - fmean) - K T (solver.py:398-401) and the loads'
// partial sums: mode 0 -> sums of f per case (for the global mean); mode 1 -> r
// (fp32, interior) and partial sums r^2, f^2, T per case.
template <int MODE>
__global__ void __launch_bounds__(128) ks_res64(SGeo g, LevelTemplate lt, const double* __restrict__ kap,
                                                const double* __restrict__ T, const double* __restrict__ fmean,
                                                float* __restrict__ r32, double* partials, unsigned* counter,
                                                double* out9) {
    double acc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni; i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        s_decode(g, i, x, y, z);
        const int ys[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
        const int zs[3] = {wrap_m(z, g.nz), z, wrap_p(z, g.nz)};
        double k[2][4];
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int q = 0; q < 2; ++q) k[p][j * 2 + q] = __ldg(kap + (long long)(x - 1 + p) * g.pl + ys[j] + zs[q]);
        const long long idx = (long long)x * g.pl + y * g.nz + z;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // loads: element (q, jj, kk) has v as corner a = (1-q) | (1-jj)<<1 | (1-kk)<<2 (k2_res64 order)
            double f = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int q = 1 - (a & 1), jj = 1 - ((a >> 1) & 1), kk = 1 - ((a >> 2) & 1);
                f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + c], k[q][jj * 2 + kk]));
            }
            if (MODE == 0) {
                acc[c] += f;
                continue;
            }
            const double* Tc = T + (long long)c * g.na;
            double t[3][9];
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int q = 0; q < 3; ++q) t[p][j * 3 + q] = __ldg(Tc + (long long)(x - 1 + p) * g.pl + ys[j] + zs[q]);
            double kt;
            if (lt.equal) {
                const KSum<double> s = ksum<double>(k);
                kt = apply_compact<double>(t, k, s, lt.s12);
            } else {
                kt = apply_generic<double>(t, k, lt.kt);
            }
            const double r = (f - fmean[c]) - kt;
            r32[(long long)c * g.na + idx] = (float)r;
            acc[c] += r * r;
            acc[3 + c] += f * f;
            acc[6 + c] += t[1][4];
        }
    }
    reduce_finalize<9>(acc, partials, counter, out9);
}

// T += d (interior), optional subtraction of per-case means
__global__ void ks_tupd(SGeo g, double* __restrict__ T, const float* __restrict__ d, double m0, double m1,
                        double m2, int with_d) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * g.ni) return;
    const int c = (int)(i / g.ni);
    const long long idx = (long long)c * g.na + g.pl + (i - (long long)c * g.ni);
    const double m = c == 0 ? m0 : (c == 1 ? m1 : m2);
    T[idx] = (T[idx] + (with_d ? (double)d[idx] : 0.0)) - m;
}

// partial sums kappa_e * E_c[e] (homogenize.py:103-122), element e = vertex e, corners e + c_a
__global__ void __launch_bounds__(256) ks_tensor(SGeo g, const double* __restrict__ T, const double* __restrict__ kap,
                                                 const double* __restrict__ kt, double* partials, unsigned* counter,
                                                 double* out6) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni; i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        s_decode(g, i, x, y, z);
        const int ys[2] = {y, wrap_p(y, g.ny)}, zs[2] = {z, wrap_p(z, g.nz)};
        // chi_i = e_i - T_i at the 8 corners (homogenize.py:103-110): corner a at (x + a&1, y + a>>1&1, z + a>>2&1)
        double chi[3][8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const long long idx = (long long)(x + (a & 1)) * g.pl + ys[(a >> 1) & 1] * g.nz + zs[(a >> 2) & 1];
#pragma unroll
            for (int c = 0; c < 3; ++c) chi[c][a] = (double)((a >> c) & 1) - __ldg(T + (long long)c * g.na + idx);
        }
        const double ke = __ldg(kap + (long long)x * g.pl + y * g.nz + z);
        const int pr[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {1, 2}, {0, 2}};
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            double e = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                double ka = 0.0;
#pragma unroll
                for (int b = 0; b < 8; ++b) ka += kt[a ^ b] * chi[pr[q][1]][b];
                e += chi[pr[q][0]][a] * ka;
            }
            acc[q] += ke * e;
        }
    }
    reduce_finalize<6>(acc, partials, counter, out6);
}


// density filter on a slab (field.py:230-236; reach <= 1, 27-slot weights in the
// single-GPU tap order, so results are bit-identical).  MODE 2: forward + SIMP
// (element.py:91-94) + partial sums of rho, rho^p, rho_f; MODE 1: adjoint.
template <int MODE>
__global__ void __launch_bounds__(256) ks_filter(SGeo g, W27 taps, const double* __restrict__ in,
                                                 double* __restrict__ out, double* __restrict__ kap64,
                                                 SimpParams sp, double* partials, unsigned* counter,
                                                 double* out3) {
    double acc3[3] = {0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni; i += (long long)gridDim.x * blockDim.x) {
        int x, y, z;
        s_decode(g, i, x, y, z);
        const int ys[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
        const int zs[3] = {wrap_m(z, g.nz), z, wrap_p(z, g.nz)};
        double sacc = 0.0;
#pragma unroll
        for (int slot = 0; slot < 27; ++slot) {
            const double wt = taps.w[slot];
            if (wt != 0.0) {
                const int src = MODE == 1 ? 26 - slot : slot;
                const int p = src / 9, j = (src / 3) % 3, m = src % 3;
                sacc = __dadd_rn(sacc, __dmul_rn(wt, __ldg(in + (long long)(x - 1 + p) * g.pl + ys[j] + zs[m])));
            }
        }
        const long long idx = (long long)x * g.pl + y * g.nz + z;
        out[idx] = sacc;
        if (MODE == 2) {
            kap64[idx] = sp.kmin + simp_pow(sacc, sp.p) * (sp.k0 - sp.kmin);
            const double r = __ldg(in + idx);
            acc3[0] += r;
            acc3[1] += simp_pow(r, sp.p);
            acc3[2] += sacc;
        }
    }
    if (MODE == 2) reduce_finalize<3>(acc3, partials, counter, out3);
}

// sens_f = kappa'(rho_f) (dG . E) / M (homogenize.py:143-160); element e = vertex e
__global__ void __launch_bounds__(256) ks_sens(SGeo g, const double* __restrict__ T, const double* __restrict__ rf,
                                               const double* __restrict__ kt, SimpParams sp, Dg dG, double M,
                                               double* __restrict__ sens) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.ni) return;
    int x, y, z;
    s_decode(g, i, x, y, z);
    const int ys[2] = {y, wrap_p(y, g.ny)}, zs[2] = {z, wrap_p(z, g.nz)};
    double chi[3][8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const long long idx = (long long)(x + (a & 1)) * g.pl + ys[(a >> 1) & 1] * g.nz + zs[(a >> 2) & 1];
#pragma unroll
        for (int c = 0; c < 3; ++c) chi[c][a] = (double)((a >> c) & 1) - __ldg(T + (long long)c * g.na + idx);
    }
    const int pr[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {1, 2}, {0, 2}};
    double con = 0.0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        double e = 0.0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            double ka = 0.0;
#pragma unroll
            for (int b = 0; b < 8; ++b) ka += kt[a ^ b] * chi[pr[q][1]][b];
            e += chi[pr[q][0]][a] * ka;
        }
        con += dG.v[q] * e;
    }
    const long long idx = (long long)x * g.pl + y * g.nz + z;
    const double dk = sp.p * simp_pow(rf[idx], sp.p - 1.0) * (sp.k0 - sp.kmin);
    sens[idx] = dk * con / M;
}

// OC candidate sums for up to 32 multipliers (optimize.py:114-160) over the slab's
// interior (contiguous: planes 1 .. nxl).  The candidate clip(rho * max(desc/lam,
// 1e-10)^damp, lo, hi) is evaluated as clip(max(c_e lam^-damp, rho 1e-10^damp), lo,
// hi) with c_e = rho desc^damp formed once per element (the single-GPU search's form,
// k_oc_coop); lam_pow[k] = lam^-damp, 0 for the free step (lam = 0).
__global__ void __launch_bounds__(256) ks_oc_sums(SGeo g, const double* __restrict__ rho,
                                                  const double* __restrict__ sens, OcArgs a, double M, LamSet lam_pow,
                                                  double* partials, unsigned* counter, double* out32) {
    double acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni; i += (long long)gridDim.x * blockDim.x) {
        const long long idx = g.pl + i;
        const double r = __ldg(rho + idx);
        const double desc = M * (-__ldg(sens + idx));
        const double lo = fmax(r - a.step, a.rmin), hi = fmin(r + a.step, 1.0);
        const double lof = fmax(lo, r * a.floor_ratio);
        const double ce = desc > 0.0 ? r * (a.sqrt_damp ? sqrt(desc) : pow(desc, a.damp)) : 0.0;
        const double freev = desc > 0.0 ? hi : (desc < 0.0 ? lo : r);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double lp = lam_pow.v[k];
            acc[k] += lp == 0.0 ? freev : fmin(fmax(ce * lp, lof), hi);
        }
    }
    reduce_finalize32(acc, partials, counter, out32);
}

// the update with the chosen multiplier, the reference's exact expression
// (optimize.py:131-138, bit-identical to k_oc_apply); out[0] = changed elements
__global__ void __launch_bounds__(256) ks_oc_apply(SGeo g, const double* rho,          // may alias rho_out
                                                   const double* __restrict__ sens, OcArgs a, double M, double lam,
                                                   double* rho_out, double* partials, unsigned* counter,
                                                   double* out) {
    double acc[1] = {0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < g.ni; i += (long long)gridDim.x * blockDim.x) {
        const long long idx = g.pl + i;
        const double r = rho[idx];
        const double desc = M * (-sens[idx]);
        const double lo = fmax(r - a.step, a.rmin), hi = fmin(r + a.step, 1.0);
        double o;
        if (lam == 0.0) {
            o = desc > 0.0 ? hi : (desc < 0.0 ? lo : r);
        } else {
            const double q = fmax(desc / lam, 1e-10);
            const double ratio = a.sqrt_damp ? sqrt(q) : pow(q, a.damp);
            o = fmin(fmax(r * ratio, lo), hi);
        }
        rho_out[idx] = o;
        acc[0] += o != r ? 1.0 : 0.0;
    }
    reduce_finalize<1>(acc, partials, counter, out);
}

// ghost planes from the neighbours (otm_slab_halo_local); T = float or double, one thread
// per (case, side, element of the plane)
template <class T>
__global__ void ks_halo_local(int ncases, long long pl, T* __restrict__ dst, int nxl, const T* __restrict__ left,
                              int nxl_left, const T* __restrict__ right, int nxl_right) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long per = 2 * pl;
    if (i >= ncases * per) return;
    const int c = (int)(i / per);
    const long long r = i - (long long)c * per;
    const int side = (int)(r / pl);
    const long long e = r - (long long)side * pl;
    const long long nd = (long long)(nxl + 2) * pl;
    if (side == 0) dst[c * nd + e] = left[c * (long long)(nxl_left + 2) * pl + (long long)nxl_left * pl + e];
    else dst[c * nd + (long long)(nxl + 1) * pl + e] = right[c * (long long)(nxl_right + 2) * pl + pl + e];
}

inline unsigned nb(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }
// reducing kernels are grid-stride with a bounded grid: one partial per block and one
// ticket atomic per block (an unbounded one-item-per-thread grid serialised ~10^5
// atomics on the ticket counter)
inline unsigned nbr(long long n, int bs) { const unsigned b = nb(n, bs); return b < 1184u ? b : 1184u; }

// Device-side PCG scalars of the slab solve (layout in otm_slab.h: otm_slab_pcg_step);
// stage 0 after the r.z all-reduce, 1 after p.q, 2 after r.r -- the host loop of
// round 1 (slab.py) moved to the device, same expressions.
__global__ void ks_pcg_step(int stage, double* S) {
    double* rz = S;
    double* rz_old = S + 3;
    double* beta = S + 6;
    double* pq = S + 9;
    double* alpha = S + 12;
    double* rr = S + 15;
    double* target2 = S + 18;
    double* active = S + 21;
    double* cyc = S + 25;
    for (int c = 0; c < 3; ++c) {
        if (stage == 0) {
            beta[c] = S[24] != 0.0 ? 0.0 : (rz_old[c] != 0.0 ? rz[c] / rz_old[c] : 0.0);
            rz_old[c] = rz[c];
        } else if (stage == 1) {
            alpha[c] = (active[c] != 0.0 && pq[c] > 0.0) ? rz[c] / pq[c] : 0.0;
        } else {
            cyc[c] += active[c];
            if (!(rr[c] > target2[c])) active[c] = 0.0;
        }
    }
    if (stage == 0) S[24] = 0.0;
}

}  // namespace
}  // namespace otm

using namespace otm;

struct otm_slab_ws {
    cudaStream_t stream = nullptr;
    double* partials = nullptr;
    unsigned* counter = nullptr;
    double* out = nullptr;       // device scalars
    double* h = nullptr;         // pinned host copy
    double* out32 = nullptr;     // 32 OC candidate sums (device) and their host copy
    double* h32 = nullptr;
    PcgScalars* sc = nullptr;    // scratch scalars of the k10 level kernels (their dot sums land in red[])
    int dev = 0;                 // 1: scalar arguments / results of the PCG calls are device pointers
    size_t max_blocks = 0;
    char err[256] = {0};
};

static int sfail(otm_slab_ws* w, const char* m) {
    if (w) std::snprintf(w->err, sizeof w->err, "%s", m);
    return OTM_ECUDA;
}
#define SCK(x)                                                   \
    do {                                                         \
        cudaError_t e_ = (x);                                    \
        if (e_ != cudaSuccess) return sfail(w, cudaGetErrorString(e_)); \
    } while (0)

static int scheck(otm_slab_ws* w) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? OTM_OK : sfail(w, cudaGetErrorString(e));
}
static int sfetch(otm_slab_ws* w, int nq, double* out) {
    if (w->dev) {       // device scalars: stream-ordered copy, no host round trip
        SCK(cudaMemcpyAsync(out, w->out, nq * sizeof(double), cudaMemcpyDeviceToDevice, w->stream));
        return OTM_OK;
    }
    SCK(cudaMemcpyAsync(w->h, w->out, nq * sizeof(double), cudaMemcpyDeviceToHost, w->stream));
    SCK(cudaStreamSynchronize(w->stream));
    std::memcpy(out, w->h, nq * sizeof(double));
    return OTM_OK;
}
// OTM_SLAB_GENERIC=1: the slab's own per-element kernels instead of the single-GPU
// marching / TMA kernels restricted to the interior planes (A/B and fallback)
static bool fast_off() {
    static const bool v = getenv("OTM_SLAB_GENERIC") && atoi(getenv("OTM_SLAB_GENERIC")) != 0;
    return v;
}
static LevelTemplate tmpl(const double scale[3]) {
    LevelTemplate lt;
    ::level_template(scale, lt);
    return lt;
}
static bool blocks_ok(otm_slab_ws* w, long long items, int bs) {
    return (size_t)nb(items, bs) <= w->max_blocks;
}

extern "C" {

otm_slab_ws* otm_slab_create(long long max_items) {
    otm_slab_ws* w = new otm_slab_ws();
    w->max_blocks = (size_t)((max_items + 127) / 128) + 64;
    if (cudaMalloc(&w->partials, w->max_blocks * 32 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->counter, 4 * sizeof(unsigned)) != cudaSuccess ||
        cudaMalloc(&w->out, 16 * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&w->h, 16 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->out32, 32 * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&w->h32, 32 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&w->sc, sizeof(PcgScalars)) != cudaSuccess) {
        delete w;
        return nullptr;
    }
    cudaMemset(w->counter, 0, 4 * sizeof(unsigned));
    cudaMemset(w->sc, 0, sizeof(PcgScalars));
    return w;
}

int otm_slab_destroy(otm_slab_ws* w) {
    if (!w) return OTM_OK;
    cudaFree(w->partials);
    cudaFree(w->counter);
    cudaFree(w->out);
    cudaFreeHost(w->h);
    cudaFree(w->out32);
    cudaFreeHost(w->h32);
    cudaFree(w->sc);
    delete w;
    return OTM_OK;
}

int otm_slab_set_stream(otm_slab_ws* w, void* stream) {
    if (!w) return OTM_EINVAL;
    w->stream = (cudaStream_t)stream;
    return OTM_OK;
}

const char* otm_slab_last_error(otm_slab_ws* w) { return w ? w->err : "null workspace"; }

int otm_slab_stencil(otm_slab_ws* w, int op, int nxl, int ny, int nz, const double scale[3], const float* kap,
                     const float* a, const float* f, const float* dinv, double omega, float* o1, float* o2,
                     double* dots3) {
    return otm_slab_stencil_range(w, op, nxl, ny, nz, scale, kap, a, f, dinv, omega, o1, o2, 1, nxl + 1, dots3);
}

int otm_slab_stencil_range(otm_slab_ws* w, int op, int nxl, int ny, int nz, const double scale[3], const float* kap,
                           const float* a, const float* f, const float* dinv, double omega, float* o1, float* o2,
                           int x_lo, int x_hi, double* dots3) {
    if (!w || nxl < 1 || ny < 1 || nz < 1 || op < 0 || op > 2) return OTM_EINVAL;
    if (x_lo < 1 || x_hi > nxl + 1 || x_hi <= x_lo) return OTM_EINVAL;
    SGeo g = make_sgeo(nxl, ny, nz);
    g.x0 = x_lo;
    g.ni = (long long)(x_hi - x_lo) * g.pl;
    const LevelTemplate lt = tmpl(scale);
    const long long items = 3 * g.ni;
    if (!blocks_ok(w, items, 256)) return OTM_EINVAL;
    const int dot = dots3 != nullptr && op > 0;
    {
        // fast path: the single-GPU k10 march on the output planes [x_lo, x_hi) of the
        // ghost-padded slab (the x neighbours are the ghost planes; y, z periodic)
        const Geo gg = make_geo(nxl + 2, ny, nz);
        Red red{w->partials, w->counter};
        if (launch_k10_range(w->stream, op, gg, lt, x_lo, x_hi, kap, a, f, dinv, (float)omega, o1, o2, dot != 0,
                             red, w->sc)) {
            int rc = scheck(w);
            if (rc || !dot) return rc;
            if (w->dev) {
                SCK(cudaMemcpyAsync(dots3, reinterpret_cast<const double*>(w->sc) + (op == 1 ? 0 : 3),
                                    3 * sizeof(double), cudaMemcpyDeviceToDevice, w->stream));
                return OTM_OK;
            }
            SCK(cudaMemcpyAsync(w->h, reinterpret_cast<const double*>(w->sc) + (op == 1 ? 0 : 3), 3 * sizeof(double),
                                cudaMemcpyDeviceToHost, w->stream));
            SCK(cudaStreamSynchronize(w->stream));
            std::memcpy(dots3, w->h, 3 * sizeof(double));
            return OTM_OK;
        }
    }
    if (op == 0)
        ks_stencil<0><<<nbr(items, 256), 256, 0, w->stream>>>(g, lt, kap, nullptr, f, dinv, (float)omega, o1, o2, 0,
                                                              w->partials, w->counter, w->out);
    else if (op == 1)
        ks_stencil<1><<<nbr(items, 256), 256, 0, w->stream>>>(g, lt, kap, a, f, dinv, (float)omega, o1, nullptr, dot,
                                                              w->partials, w->counter, w->out);
    else
        ks_stencil<2><<<nbr(items, 256), 256, 0, w->stream>>>(g, lt, kap, a, nullptr, nullptr, 0.f, o1, nullptr, dot,
                                                              w->partials, w->counter, w->out);
    int rc = scheck(w);
    if (rc || !dot) return rc;
    return sfetch(w, 3, dots3);
}

int otm_slab_restrict(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* res_f, float* f_c) {
    if (!w || nxl_f < 2 || (nxl_f & 1) || (ny_f & 1) || (nz_f & 1)) return OTM_EINVAL;
    const SGeo f = make_sgeo(nxl_f, ny_f, nz_f), c = make_sgeo(nxl_f / 2, ny_f / 2, nz_f / 2);
    ks_restrict<<<nb(3 * c.ni, 256), 256, 0, w->stream>>>(f, c, res_f, f_c);
    return scheck(w);
}

int otm_slab_prolong(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* z_c, float* z_f) {
    if (!w || nxl_f < 2 || (nxl_f & 1) || (ny_f & 1) || (nz_f & 1)) return OTM_EINVAL;
    const SGeo f = make_sgeo(nxl_f, ny_f, nz_f), c = make_sgeo(nxl_f / 2, ny_f / 2, nz_f / 2);
    if (nz_f % 2 == 0 && ny_f % 2 == 0)
        ks_prolong_b<<<nb(3 * c.ni, 256), 256, 0, w->stream>>>(f, c, z_c, z_f);
    else
        ks_prolong<<<nb(3 * f.ni, 256), 256, 0, w->stream>>>(f, c, z_c, z_f);
    return scheck(w);
}

int otm_slab_coarsen(otm_slab_ws* w, int nxl_f, int ny_f, int nz_f, const float* k_f, float* k_c) {
    if (!w || nxl_f < 2 || (nxl_f & 1) || (ny_f & 1) || (nz_f & 1)) return OTM_EINVAL;
    const SGeo f = make_sgeo(nxl_f, ny_f, nz_f), c = make_sgeo(nxl_f / 2, ny_f / 2, nz_f / 2);
    ks_coarsen<<<nb(c.ni, 256), 256, 0, w->stream>>>(f, c, k_f, k_c);
    return scheck(w);
}

int otm_slab_dinv(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const float* kap, float* dinv) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    const LevelTemplate lt = tmpl(scale);
    ks_dinv<<<nb(g.ni, 256), 256, 0, w->stream>>>(g, kap, (float)lt.kt[0], dinv);
    return scheck(w);
}

int otm_slab_pupd(otm_slab_ws* w, int nxl, int ny, int nz, const float* z, float* p, const double beta3[3]) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (g.pl % 4 == 0)
        ks_pupd4<<<dim3(std::min<unsigned>(nb(g.ni / 4, 256), 592u), 3), 256, 0, w->stream>>>(
            g, z, p, w->dev ? 0.0 : beta3[0], w->dev ? 0.0 : beta3[1], w->dev ? 0.0 : beta3[2], w->dev ? beta3 : nullptr);
    else
        ks_pupd<<<nb(3 * g.ni, 256), 256, 0, w->stream>>>(g, z, p, w->dev ? 0.0 : beta3[0], w->dev ? 0.0 : beta3[1],
                                                          w->dev ? 0.0 : beta3[2], w->dev ? beta3 : nullptr);
    return scheck(w);
}

int otm_slab_upd(otm_slab_ws* w, int nxl, int ny, int nz, float* d, float* r, const float* p, const float* q,
                 const double alpha3[3], double* rr3) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (!blocks_ok(w, 3 * g.ni, 256)) return OTM_EINVAL;
    if (g.pl % 4 == 0)
        ks_upd4<<<dim3(std::min<unsigned>(nb(g.ni / 4, 256), 394u), 3), 256, 0, w->stream>>>(
            g, d, r, p, q, w->dev ? 0.0 : alpha3[0], w->dev ? 0.0 : alpha3[1], w->dev ? 0.0 : alpha3[2], w->partials,
            w->counter, w->out, w->dev ? alpha3 : nullptr);
    else
        ks_upd<<<nbr(3 * g.ni, 256), 256, 0, w->stream>>>(g, d, r, p, q, w->dev ? 0.0 : alpha3[0],
                                                          w->dev ? 0.0 : alpha3[1], w->dev ? 0.0 : alpha3[2],
                                                          w->partials, w->counter, w->out, w->dev ? alpha3 : nullptr);
    int rc = scheck(w);
    if (rc) return rc;
    return sfetch(w, 3, rr3);
}

int otm_slab_load_sums(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* kap64,
                       double* sums3) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (!blocks_ok(w, g.ni, 128)) return OTM_EINVAL;
    const LevelTemplate lt = tmpl(scale);
    if (!fast_off()) {
        Red red{w->partials, w->counter};
        const XRange xr{1, nxl + 1, 1.0};
        launch_load_means(w->stream, make_geo(nxl + 2, ny, nz), lt, kap64, red, w->out, &xr);
    } else {
        ks_res64<0><<<nbr(g.ni, 128), 128, 0, w->stream>>>(g, lt, kap64, nullptr, nullptr, nullptr, w->partials,
                                                           w->counter, w->out);
    }
    int rc = scheck(w);
    if (rc) return rc;
    double o[9];
    rc = sfetch(w, 9, o);
    if (rc) return rc;
    for (int c = 0; c < 3; ++c) sums3[c] = o[c];
    return OTM_OK;
}

int otm_slab_res64(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* kap64,
                   const double* T, const double fmean3[3], float* r32, double* sums9) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (!blocks_ok(w, g.ni, 128)) return OTM_EINVAL;
    const LevelTemplate lt = tmpl(scale);
    SCK(cudaMemcpyAsync(w->out + 9, fmean3, 3 * sizeof(double), cudaMemcpyHostToDevice, w->stream));
    // the single-GPU push march (k_res64p) on the interior planes of the ghosted slab
    Red red{w->partials, w->counter};
    const XRange xr{1, nxl + 1, 1.0};
    if (!fast_off() && launch_res64_range(w->stream, make_geo(nxl + 2, ny, nz), lt, kap64, T, w->out + 9, r32, red,
                                          w->out, xr)) {
        int rc = scheck(w);
        if (rc) return rc;
        return sfetch(w, 9, sums9);
    }
    ks_res64<1><<<nbr(g.ni, 128), 128, 0, w->stream>>>(g, lt, kap64, T, w->out + 9, r32, w->partials, w->counter,
                                                       w->out);
    int rc = scheck(w);
    if (rc) return rc;
    return sfetch(w, 9, sums9);
}

int otm_slab_tupd(otm_slab_ws* w, int nxl, int ny, int nz, double* T, const float* d, const double mean3[3]) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    ks_tupd<<<nb(3 * g.ni, 256), 256, 0, w->stream>>>(g, T, d, mean3[0], mean3[1], mean3[2], d != nullptr);
    return scheck(w);
}

int otm_slab_tensor_sums(otm_slab_ws* w, int nxl, int ny, int nz, const double scale[3], const double* T,
                         const double* kap64, double* sums6) {
    if (!w || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (!blocks_ok(w, g.ni, 256)) return OTM_EINVAL;
    const LevelTemplate lt = tmpl(scale);
    if (!fast_off() && scale[0] == 1.0 && scale[1] == 1.0 && scale[2] == 1.0) {
        // k_tensor_x (energies in the Walsh-Hadamard basis of the unit element) on the interior
        Red red{w->partials, w->counter};
        const XRange xr{1, nxl + 1, 1.0};
        launch_tensor(w->stream, make_geo(nxl + 2, ny, nz), T, kap64, red, w->out, &xr);
    } else {
        SCK(cudaMemcpyAsync(w->out + 8, lt.kt, 8 * sizeof(double), cudaMemcpyHostToDevice, w->stream));
        ks_tensor<<<nbr(g.ni, 256), 256, 0, w->stream>>>(g, T, kap64, w->out + 8, w->partials, w->counter, w->out);
    }
    int rc = scheck(w);
    if (rc) return rc;
    return sfetch(w, 6, sums6);
}

int otm_slab_filter(otm_slab_ws* w, int mode, int nxl, int ny, int nz, double radius, double kappa0,
                    double kappa_min, double penalty, const double* in, double* out, double* kap64,
                    double* sums3) {
    if (!w || nxl < 1 || (mode != 1 && mode != 2) || !(radius >= 1.0) || radius > 2.0 ||
        (mode == 2 && (!kap64 || !sums3)))
        return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if (!blocks_ok(w, g.ni, 256)) return OTM_EINVAL;
    std::vector<int> offs;
    std::vector<double> wt;
    filter_weights(radius, offs, wt);
    W27 taps;
    for (int i = 0; i < 27; ++i) taps.w[i] = 0.0;
    for (size_t i = 0; i < wt.size(); ++i) {
        const int slot = (offs[3 * i] + 1) * 9 + (offs[3 * i + 1] + 1) * 3 + (offs[3 * i + 2] + 1);
        taps.w[slot] = wt[i];
    }
    SimpParams sp;
    sp.k0 = kappa0;
    sp.kmin = kappa_min;
    sp.p = penalty;
    FilterSetup fs{};
    fs.window = 1;
    for (int i = 0; i < 27; ++i) fs.w27[i] = taps.w[i];
    Red red{w->partials, w->counter};
    const XRange xr{1, nxl + 1, 1.0};
    if (!fast_off() &&
        launch_filter_range(w->stream, make_geo(nxl + 2, ny, nz), fs, mode, sp, in, out, kap64, red, w->out, xr)) {
        int rc = scheck(w);
        if (rc || mode == 1) return rc;
        return sfetch(w, 3, sums3);
    }
    if (mode == 2)
        ks_filter<2><<<nbr(g.ni, 256), 256, 0, w->stream>>>(g, taps, in, out, kap64, sp, w->partials, w->counter,
                                                            w->out);
    else
        ks_filter<1><<<nb(g.ni, 256), 256, 0, w->stream>>>(g, taps, in, out, nullptr, sp, w->partials, w->counter,
                                                            w->out);
    int rc = scheck(w);
    if (rc || mode == 1) return rc;
    return sfetch(w, 3, sums3);
}

int otm_slab_sensitivity(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, double kappa0, double kappa_min,
                         double penalty, const double* T, const double* rho_f, const double dG6[6], double* sens_f) {
    if (!w || nxl < 1 || !(n_total > 0)) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    const double unit[3] = {1.0, 1.0, 1.0};
    const LevelTemplate lt = tmpl(unit);
    SCK(cudaMemcpyAsync(w->out + 8, lt.kt, 8 * sizeof(double), cudaMemcpyHostToDevice, w->stream));
    SimpParams sp;
    sp.k0 = kappa0;
    sp.kmin = kappa_min;
    sp.p = penalty;
    Dg dg;
    for (int q = 0; q < 6; ++q) dg.v[q] = dG6[q];
    if (!fast_off()) {
        const XRange xr{1, nxl + 1, n_total};
        launch_sens(w->stream, make_geo(nxl + 2, ny, nz), T, rho_f, sp, dg, sens_f, nullptr, &xr);
        return scheck(w);
    }
    ks_sens<<<nb(g.ni, 256), 256, 0, w->stream>>>(g, T, rho_f, w->out + 8, sp, dg, n_total, sens_f);
    return scheck(w);
}

int otm_slab_oc_sums(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, const otm_oc_params* pp,
                     const double* rho, const double* sens, int nlam, const double* lams, double* sums32) {
    if (!w || !pp || nxl < 1 || nlam < 1 || nlam > 32) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if ((size_t)nb(g.ni, 256) * 32 > w->max_blocks * 9) return OTM_EINVAL;
    OcArgs a;
    a.step = pp->step_limit;
    a.rmin = pp->min_density;
    a.damp = pp->damp;
    a.floor_ratio = std::pow(1e-10, pp->damp);
    a.sqrt_damp = pp->damp == 0.5;
    LamSet ls;
    for (int k = 0; k < 32; ++k) {
        const double lam = k < nlam ? lams[k] : 0.0;
        ls.v[k] = lam == 0.0 ? 0.0 : (a.sqrt_damp ? 1.0 / std::sqrt(lam) : std::pow(lam, -a.damp));
    }
    ks_oc_sums<<<nbr(g.ni, 256), 256, 0, w->stream>>>(g, rho, sens, a, n_total, ls, w->partials, w->counter,
                                                      w->out32);
    int rc = scheck(w);
    if (rc) return rc;
    SCK(cudaMemcpyAsync(w->h32, w->out32, 32 * sizeof(double), cudaMemcpyDeviceToHost, w->stream));
    SCK(cudaStreamSynchronize(w->stream));
    std::memcpy(sums32, w->h32, nlam * sizeof(double));
    return OTM_OK;
}

int otm_slab_oc_apply(otm_slab_ws* w, int nxl, int ny, int nz, double n_total, const otm_oc_params* pp,
                      const double* rho, const double* sens, double lam, double* rho_out, double* changed) {
    if (!w || !pp || nxl < 1) return OTM_EINVAL;
    const SGeo g = make_sgeo(nxl, ny, nz);
    if ((size_t)nb(g.ni, 256) * 32 > w->max_blocks * 9) return OTM_EINVAL;
    OcArgs a;
    a.step = pp->step_limit;
    a.rmin = pp->min_density;
    a.damp = pp->damp;
    a.floor_ratio = std::pow(1e-10, pp->damp);
    a.sqrt_damp = pp->damp == 0.5;
    ks_oc_apply<<<nbr(g.ni, 256), 256, 0, w->stream>>>(g, rho, sens, a, n_total, lam, rho_out, w->partials,
                                                       w->counter, w->out32);
    int rc = scheck(w);
    if (rc) return rc;
    SCK(cudaMemcpyAsync(w->h32, w->out32, sizeof(double), cudaMemcpyDeviceToHost, w->stream));
    SCK(cudaStreamSynchronize(w->stream));
    *changed = w->h32[0];
    return OTM_OK;
}

int otm_slab_set_scalar_mode(otm_slab_ws* w, int device) {
    if (!w) return OTM_EINVAL;
    w->dev = device != 0;
    return OTM_OK;
}

int otm_slab_halo_local(void* stream, int elem_size, int ncases, long long pl, void* dst, int nxl,
                        const void* left, int nxl_left, const void* right, int nxl_right) {
    if (!dst || !left || !right || ncases < 1 || pl < 1 || nxl < 1 || nxl_left < 1 || nxl_right < 1 ||
        (elem_size != 4 && elem_size != 8))
        return OTM_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned blocks = nb(2 * pl * ncases, 256);
    if (elem_size == 4)
        ks_halo_local<float><<<blocks, 256, 0, s>>>(ncases, pl, (float*)dst, nxl, (const float*)left, nxl_left,
                                                    (const float*)right, nxl_right);
    else
        ks_halo_local<double><<<blocks, 256, 0, s>>>(ncases, pl, (double*)dst, nxl, (const double*)left, nxl_left,
                                                     (const double*)right, nxl_right);
    return cudaGetLastError() == cudaSuccess ? OTM_OK : OTM_ECUDA;
}

int otm_slab_pcg_step(otm_slab_ws* w, int stage, double* S) {
    if (!w || !S || stage < 0 || stage > 2) return OTM_EINVAL;
    ks_pcg_step<<<1, 1, 0, w->stream>>>(stage, S);
    return scheck(w);
}
}  // extern "C"
