// Vectorised register-window stencil engine (fast path of the level stencils).
//
// Thread = one load case x two consecutive z vertices (z even) of one y row;
// block = 32 (z pairs) x 8 (rows); grid = (nz/64, ny/8, cases x x-chunks).  Each
// thread walks its x chunk holding planes x-1, x, x+1 of the operand at columns
// z-1..z+2 of rows y-1..y+1 (36 values) and the element factors of element planes
// x-1, x at columns z-1..z+1 of rows y-1, y (12 values).  Per plane a thread
// issues 3 vector + 6 scalar operand loads and 2 vector + 2 scalar factor loads
// for two outputs; the z+-1 / y+-1 neighbours are L1 hits of the adjacent lanes /
// rows of the same block.
#pragma once

#include "otm_common.cuh"
#include "otm_internal.h"

namespace otm {

template <typename R> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

constexpr int kTileZ = 64;   // 32 threads x 2 vertices
constexpr int kTileY = 8;

__host__ __device__ inline bool fast_tiling(const Geo& g) {
    return g.nz % kTileZ == 0 && g.ny % kTileY == 0 && g.nx >= 2;
}

// Per-vertex operator on sub-windows; ksub is the element-factor window of that vertex.
template <typename R>
__device__ __forceinline__ R apply_sub(const R (&t)[3][3][4], const R (&k)[2][2][3], int i,
                                       const LevelTemplate& lt, R (&ksub)[2][4]) {
    R w[3][9];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) w[p][j * 3 + kk] = t[p][j][i + kk];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) ksub[q][jj * 2 + kk] = k[q][jj][i + kk];
    if (lt.equal) {
        const KSum<R> s = ksum<R>(ksub);
        return apply_compact<R>(w, ksub, s, (R)lt.s12);
    }
    R kt[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) kt[a] = (R)lt.kt[a];
    return apply_generic<R>(w, ksub, kt);
}

// Op contract:
//   R t1(int c, long long v) const;              operand at vertex v, case c
//   V2 t2(int c, long long v) const;             operand at v, v+1
//   R k1(long long v) const; V2 k2(long long v) const;   element factors
//   void sink(int c, long long v, const R (&kt)[2], const R (&ctr)[2], const R (&ks)[2][2][4]);
template <typename R, class Op>
__device__ __forceinline__ void march2(const Geo& g, int xb, int nch, const LevelTemplate& lt, Op& op) {
    using V2 = typename Vec2<R>::T;
    const int c = blockIdx.z / nch;
    const int ch = blockIdx.z - c * nch;
    const int z = (blockIdx.x * 32 + threadIdx.x) * 2;
    const int y = blockIdx.y * kTileY + threadIdx.y;
    const int zm = z == 0 ? g.nz - 1 : z - 1;
    const int zp2 = z + 2 == g.nz ? 0 : z + 2;
    const int ro[3] = {wrap_m(y, g.ny) * g.nz, y * g.nz, wrap_p(y, g.ny) * g.nz};
    const int x0 = ch * xb, x1 = min(g.nx, x0 + xb);
    if (x0 >= x1) return;
    R t[3][3][4];
    R k[2][2][3];
    auto loadT = [&](int slot, int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const long long b = po + ro[j];
            t[slot][j][0] = op.t1(c, b + zm);
            const V2 v = op.t2(c, b + z);
            t[slot][j][1] = v.x;
            t[slot][j][2] = v.y;
            t[slot][j][3] = op.t1(c, b + zp2);
        }
    };
    auto loadK = [&](int slot, int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const long long b = po + ro[jj];
            k[slot][jj][0] = op.k1(b + zm);
            const V2 v = op.k2(b + z);
            k[slot][jj][1] = v.x;
            k[slot][jj][2] = v.y;
        }
    };
    loadT(0, x0 - 1);
    loadT(1, x0);
    loadK(0, x0 - 1);
    for (int x = x0; x < x1; ++x) {
        loadT(2, x + 1);
        loadK(1, x);
        R kt[2], ctr[2], ks[2][2][4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            kt[i] = apply_sub<R>(t, k, i, lt, ks[i]);
            ctr[i] = t[1][1][1 + i];
        }
        op.sink(c, (long long)x * g.pl + (long long)y * g.nz + z, kt, ctr, ks);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) { t[0][j][q] = t[1][j][q]; t[1][j][q] = t[2][j][q]; }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int q = 0; q < 3; ++q) k[0][jj][q] = k[1][jj][q];
    }
}

}  // namespace otm
