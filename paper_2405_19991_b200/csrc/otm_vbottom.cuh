// Bottom of the V-cycle in ONE single-CTA launch: the levels N^3 (N = 16 or 8)
// halving down to the 4^3 direct solve (solver.py:326-338 restricted to those
// levels; damped-Jacobi smoother, full-weighting restriction R = P^T/8,
// trilinear prolongation, pinned pseudo-inverse G on 4^3).  Every level lives in
// shared memory (16^3: ~200 KB), so the 4 + 4 + 1 per-level launches of the
// latency-bound tail (each a full dependent launch of a few microseconds) become
// one launch whose phases are separated by CTA barriers.  Same arithmetic as the
// per-level kernels (apply_compact, restrict3_body / prolong3b_body weights).
#pragma once

#include "otm_common.cuh"

namespace otm {

constexpr int kVBotMaxLev = 3;         // 16^3, 8^3, 4^3

struct VBotArgs {
    int nlev;                          // levels in the bottom (last one = 4^3, direct)
    float omega;
    float s12[kVBotMaxLev];
    const float* kap[kVBotMaxLev];
    const float* dinv[kVBotMaxLev];
    const float* f0;                   // right-hand side of the first bottom level (3 cases)
    float* out0;                       // its V-cycle result (3 cases)
    const float* G;                    // 64 x 64 coarse pseudo-inverse
};

template <int N>
struct VBotLev {
    static constexpr int n = N * N * N;
    static constexpr int F = 0, Z = 3 * n, R = 6 * n, K = 9 * n, D = 10 * n, FLOATS = 11 * n;
};

__host__ __device__ constexpr int vbot_floats(int N) {
    return N == 4 ? 6 * 64 : 11 * N * N * N + vbot_floats(N / 2);
}
// the coarse pseudo-inverse is staged behind the level data (loaded before the
// programmatic-dependency wait: it does not depend on the predecessor)
__host__ __device__ constexpr int vbot_smem_floats(int N) { return vbot_floats(N) + 64 * 64; }

template <int N>
__device__ __forceinline__ int vb_idx(int x, int y, int z) {
    return ((x & (N - 1)) * N + (y & (N - 1))) * N + (z & (N - 1));
}

// MODE 0: r = f - K z  (z = omega D^-1 f already in place);  MODE 1: r = z + omega D^-1 (f - K z)
template <int N, int MODE>
__device__ __forceinline__ void vb_stencil(float* L, float s12, float omega) {
    using V = VBotLev<N>;
    for (int v = threadIdx.x; v < V::n; v += blockDim.x) {
        const int x = v / (N * N), y = (v / N) % N, z = v % N;
        float k[2][4];
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int q = 0; q < 2; ++q) k[p][j * 2 + q] = L[V::K + vb_idx<N>(x - 1 + p, y - 1 + j, z - 1 + q)];
        const KSum<float> s = ksum<float>(k);
        const float dw = omega * L[V::D + v];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float t[3][9];
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        t[p][j * 3 + q] = L[V::Z + c * V::n + vb_idx<N>(x - 1 + p, y - 1 + j, z - 1 + q)];
            const float kt = apply_compact<float>(t, k, s, s12);
            const float f = L[V::F + c * V::n + v];
            L[V::R + c * V::n + v] = MODE == 0 ? f - kt : t[1][4] + dw * (f - kt);
        }
    }
}

// fine r (level N) -> coarse f (level N/2), weights (1/4, 1/2, 1/4) per axis
template <int N>
__device__ __forceinline__ void vb_restrict(const float* Lf, float* Lc_f) {
    using V = VBotLev<N>;
    constexpr int M = N / 2, m = M * M * M;
    const float w[3] = {0.25f, 0.5f, 0.25f};
    for (int i = threadIdx.x; i < 3 * m; i += blockDim.x) {
        const int c = i / m, v = i % m;
        const int X = v / (M * M), Y = (v / M) % M, Zc = v % M;
        const float* r = Lf + V::R + c * V::n;
        float s = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float sb = 0.f;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const float sz = w[0] * r[vb_idx<N>(2 * X - 1 + a, 2 * Y - 1 + b, 2 * Zc - 1)] +
                                 w[1] * r[vb_idx<N>(2 * X - 1 + a, 2 * Y - 1 + b, 2 * Zc)] +
                                 w[2] * r[vb_idx<N>(2 * X - 1 + a, 2 * Y - 1 + b, 2 * Zc + 1)];
                sb += w[b] * sz;
            }
            s += w[a] * sb;
        }
        Lc_f[i] = s;
    }
}

// fine z (level N) += P coarse r (level N/2)
template <int N>
__device__ __forceinline__ void vb_prolong(float* Lf, const float* rc) {
    using V = VBotLev<N>;
    constexpr int M = N / 2, m = M * M * M;
    for (int i = threadIdx.x; i < 3 * V::n; i += blockDim.x) {
        const int c = i / V::n, v = i % V::n;
        const int x = v / (N * N), y = (v / N) % N, z = v % N;
        const float* a = rc + c * m;
        const int X = x >> 1, Y = y >> 1, Zc = z >> 1;
        const int X1 = (X + 1) & (M - 1), Y1 = (Y + 1) & (M - 1), Z1 = (Zc + 1) & (M - 1);
        auto at = [&](int p, int q, int r) { return a[(p * M + q) * M + r]; };
        // z, then y, then x (prolong3b_body order)
        float qz[2][2];
        const int xs[2] = {X, X1}, ys[2] = {Y, Y1};
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int j = 0; j < 2; ++j)
                qz[p][j] = (z & 1) ? 0.5f * (at(xs[p], ys[j], Zc) + at(xs[p], ys[j], Z1)) : at(xs[p], ys[j], Zc);
        const float y0 = (y & 1) ? 0.5f * (qz[0][0] + qz[0][1]) : qz[0][0];
        const float y1 = (y & 1) ? 0.5f * (qz[1][0] + qz[1][1]) : qz[1][0];
        const float add = (x & 1) ? 0.5f * (y0 + y1) : y0;
        Lf[V::Z + i] += add;
    }
}

template <int N>
__device__ __forceinline__ void vb_load(float* L, const float* kap, const float* dinv) {
    using V = VBotLev<N>;
    for (int i = threadIdx.x; i < V::n; i += blockDim.x) {
        L[V::K + i] = kap[i];
        L[V::D + i] = dinv[i];
    }
}

// down from level N (f in place) to the direct solve, back up; result in r of level N
template <int N>
__device__ void vb_cycle(float* L, const VBotArgs& A, const float* G, int lev) {
    using V = VBotLev<N>;
    if constexpr (N == 4) {
        // r = G f per case (one warp per row)
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int i = w; i < 3 * 64; i += nw) {
            const int c = i >> 6, r = i & 63;
            float s = G[r * 64 + lane] * L[c * 64 + lane] + G[r * 64 + 32 + lane] * L[c * 64 + 32 + lane];
            s = (float)warp_sum((double)s);
            if (lane == 0) L[3 * 64 + i] = s;
        }
        __syncthreads();
    } else {
        const float om = A.omega;
        for (int i = threadIdx.x; i < 3 * V::n; i += blockDim.x) L[V::Z + i] = L[V::F + i] * (om * L[V::D + i % V::n]);
        __syncthreads();
        vb_stencil<N, 0>(L, A.s12[lev], om);
        __syncthreads();
        float* Lc = L + V::FLOATS;
        vb_restrict<N>(L, Lc);                         // coarse f at offset 0 of the coarse level
        __syncthreads();
        vb_cycle<N / 2>(Lc, A, G, lev + 1);
        const float* rc = Lc + (N / 2 == 4 ? 3 * 64 : VBotLev<N / 2>::R);
        vb_prolong<N>(L, rc);
        __syncthreads();
        vb_stencil<N, 1>(L, A.s12[lev], om);
        __syncthreads();
    }
}

template <int N>
__global__ void __launch_bounds__(1024, 1) k_vbottom(VBotArgs A) {
    extern __shared__ __align__(16) float vb_smem[];
    using V = VBotLev<N>;
    // factors and D^-1 of every bottom level do not depend on the predecessor: load
    // them before the programmatic-dependency wait
    vb_load<N>(vb_smem, A.kap[0], A.dinv[0]);
    if constexpr (N >= 16) vb_load<N / 2>(vb_smem + V::FLOATS, A.kap[1], A.dinv[1]);
    float* G = vb_smem + vbot_floats(N);
    for (int i = threadIdx.x; i < 64 * 64 / 4; i += blockDim.x)
        reinterpret_cast<float4*>(G)[i] = __ldg(reinterpret_cast<const float4*>(A.G) + i);
    pdl_wait();
    for (int i = threadIdx.x; i < 3 * V::n; i += blockDim.x) vb_smem[V::F + i] = A.f0[i];
    __syncthreads();
    vb_cycle<N>(vb_smem, A, G, 0);
    for (int i = threadIdx.x; i < 3 * V::n; i += blockDim.x) A.out0[i] = vb_smem[V::R + i];
}

}  // namespace otm
