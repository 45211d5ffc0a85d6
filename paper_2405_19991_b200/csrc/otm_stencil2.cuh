// Vectorised register-window stencil engine (fast path of the level stencils).
//
// Thread = one load case x two consecutive z vertices (z even) of one y row;
// block = 32 (z pairs) x 8 (rows); grid = (nz/64, ny/8, cases x x-chunks).  Each
// thread walks its x chunk.  Per plane it loads the operand at rows y-1..y+1,
// columns z-1..z+2 (3 vector + 6 scalar loads) and the element factors of rows
// y-1, y, columns z-1..z+1 (2 vector + 2 scalar loads), one plane AHEAD of the
// arithmetic so the loads of plane x+2 are in flight while plane x is computed.
//
// Arithmetic (equal axis scales only; other levels use the generic kernels),
// K = s K0, K0 = (5 I + N1 - J)/12:
//   (K T)_v = s/12 ( 5 K_v T_v + sum_6 E_vu T_u - sum_{e ni v} k_e S_e )
// is evaluated separably.  For the element plane between operand planes x and x+1
// the corner sums S_e come from plane-pair sums -> z-pair sums -> y-pair sums,
// Q_e = k_e S_e, and the vertex sum of Q over the two element planes is again a
// z-pair + y-pair sum.  The element plane x of step x is the plane x-1 of step
// x+1, so its Q and its factor box sum (E_{+x}, which becomes E_{-x}) are reused:
// ~40 flops per vertex and case instead of ~100 for the direct 8-element form.
#pragma once

#include "otm_common.cuh"
#include "otm_internal.h"

namespace otm {

template <typename R> struct Vec2;
template <> struct Vec2<float> { using T = float2; };
template <> struct Vec2<double> { using T = double2; };

constexpr int kTileZ = 64;   // 32 threads x 2 vertices
constexpr int kTileY = 8;

// fast path: exact (64 x 8) tiling of the (z, y) plane and equal axis scales
__host__ __device__ inline bool fast_tiling(const Geo& g, const LevelTemplate& lt) {
    return lt.equal && g.nz % kTileZ == 0 && g.ny % kTileY == 0 && g.nx >= 2;
}

// Element plane between operand planes Pa (x) and Pb (x+1) with factors kp:
//   Q[jj][m] = k[jj][m] * S[jj][m]  (element row y-1+jj, column z-1+m)
//   Ex[i]    = sum of the 4 factors around vertex z+i (its E_{+x} / E_{-x})
template <typename R>
__device__ __forceinline__ void element_plane(const R (&Pa)[3][4], const R (&Pb)[3][4], const R (&kp)[2][3],
                                              R (&Q)[2][3], R (&Ex)[2]) {
    R bz[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        R a[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) a[m] = Pa[j][m] + Pb[j][m];
#pragma unroll
        for (int m = 0; m < 3; ++m) bz[j][m] = a[m] + a[m + 1];
    }
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int m = 0; m < 3; ++m) Q[jj][m] = kp[jj][m] * (bz[jj][m] + bz[jj + 1][m]);
#pragma unroll
    for (int i = 0; i < 2; ++i) Ex[i] = (kp[0][i] + kp[0][i + 1]) + (kp[1][i] + kp[1][i + 1]);
}

// Op contract:
//   R t1(int c, long long v) const;  V2 t2(int c, long long v) const;   operand
//   R k1(long long v) const;         V2 k2(long long v) const;          element factors
//   void sink(int c, long long v, const R (&kt)[2], const R (&ctr)[2],
//             const R (&K0)[2][3], const R (&K1)[2][3]);
// K0 / K1: factors of element planes x-1 / x, rows y-1, y, columns z-1..z+1.
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
    auto loadT = [&](R (&P)[3][4], int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const long long b = po + ro[j];
            P[j][0] = op.t1(c, b + zm);
            const V2 v = op.t2(c, b + z);
            P[j][1] = v.x;
            P[j][2] = v.y;
            P[j][3] = op.t1(c, b + zp2);
        }
    };
    auto loadK = [&](R (&K)[2][3], int x) {
        const long long po = plane_off(g, x);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const long long b = po + ro[jj];
            K[jj][0] = op.k1(b + zm);
            const V2 v = op.k2(b + z);
            K[jj][1] = v.x;
            K[jj][2] = v.y;
        }
    };
    const R s12 = (R)lt.s12;
    R P1[3][4], P2[3][4], K0[2][3], K1[2][3];
    R Qlo[2][3], Exlo[2], P0c[2];
    {
        R P0[3][4];
        loadT(P0, x0 - 1);
        loadT(P1, x0);
        loadK(K0, x0 - 1);
        element_plane<R>(P0, P1, K0, Qlo, Exlo);
        P0c[0] = P0[1][1];
        P0c[1] = P0[1][2];
    }
    loadT(P2, x0 + 1);
    loadK(K1, x0);
    for (int x = x0; x < x1; ++x) {
        // prefetch plane x+2 / element plane x+1 (consumed next step)
        R Pn[3][4], Kn[2][3];
        const bool more = x + 1 < x1;
        if (more) {
            loadT(Pn, x + 2);
            loadK(Kn, x + 1);
        }
        R kt[2], ctr[2];
        {
            R Qhi[2][3], Exhi[2];
            element_plane<R>(P1, P2, K1, Qhi, Exhi);
            R KX[2][3];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int m = 0; m < 3; ++m) KX[jj][m] = K0[jj][m] + K1[jj][m];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const R qx = ((Qlo[0][i] + Qhi[0][i]) + (Qlo[0][i + 1] + Qhi[0][i + 1])) +
                             ((Qlo[1][i] + Qhi[1][i]) + (Qlo[1][i + 1] + Qhi[1][i + 1]));
                const R eym = KX[0][i] + KX[0][i + 1], eyp = KX[1][i] + KX[1][i + 1];
                const R ezm = KX[0][i] + KX[1][i], ezp = KX[0][i + 1] + KX[1][i + 1];
                const R kv = Exlo[i] + Exhi[i];
                R acc = R(5) * kv * P1[1][1 + i];
                acc += Exhi[i] * P2[1][1 + i] + Exlo[i] * P0c[i];
                acc += eyp * P1[2][1 + i] + eym * P1[0][1 + i];
                acc += ezp * P1[1][2 + i] + ezm * P1[1][i];
                kt[i] = s12 * (acc - qx);
            }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int m = 0; m < 3; ++m) Qlo[jj][m] = Qhi[jj][m];
            Exlo[0] = Exhi[0];
            Exlo[1] = Exhi[1];
        }
        ctr[0] = P1[1][1];
        ctr[1] = P1[1][2];
        op.sink(c, (long long)x * g.pl + (long long)y * g.nz + z, kt, ctr, K0, K1);
        P0c[0] = P1[1][1];
        P0c[1] = P1[1][2];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m) P1[j][m] = P2[j][m];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 3; ++m) K0[jj][m] = K1[jj][m];
        if (more) {
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int m = 0; m < 4; ++m) P2[j][m] = Pn[j][m];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int m = 0; m < 3; ++m) K1[jj][m] = Kn[jj][m];
        }
    }
}

}  // namespace otm
