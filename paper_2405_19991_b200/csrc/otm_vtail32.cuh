// The V-cycle tail from 32^3 down (32^3 -> 16^3 -> 8^3 -> 4^3 direct solve and back,
// solver.py:326-338) in ONE launch of a 16-CTA thread-block cluster.  Every level
// below 64^3 is latency-bound: as separate launches each costs ~3 us of dependency
// latency (9 launches, ~28 us per V-cycle).  Here the levels live in the cluster's
// shared memory -- CTA c owns x-planes [c P, c P + P) of the 32^3 (P = 2) and 16^3
// (P = 1) levels -- and the phases are separated by cluster barriers; halo planes
// and transfer stencils read the neighbour CTA's planes through distributed shared
// memory.  The 8^3 + 4^3 bottom runs in CTA 0 (the k_vbottom phases).  Same
// arithmetic as the per-level kernels (apply_compact, restriction / prolongation
// weights (1/4, 1/2, 1/4) and (1/2, 1, 1/2)).
#pragma once

#include <cooperative_groups.h>

#include "otm_vbottom.cuh"

namespace otm {

constexpr int kVtCtas = 16;

struct VTailArgs {
    float omega;
    float s12[4];                       // 32^3, 16^3, 8^3, 4^3
    const float* kap[3];                // 32^3, 16^3, 8^3
    const float* dinv[3];
    const float* f32;                   // right-hand side of the 32^3 level (3 cases)
    float* out32;                       // its V-cycle result (3 cases)
    const float* G;                     // 64 x 64 coarse pseudo-inverse
};

// shared-memory layout (floats) of one CTA
struct VtLay {
    // 32^3: own planes x0, x0+1 (P = 2), 1024 vertices per plane
    static constexpr int PL32 = 1024;
    static constexpr int F32 = 0;                       // [c][p<2][v]      f (own)
    static constexpr int D32 = F32 + 3 * 2 * PL32;      // [p<4][v]         D^-1, planes x0-1 .. x0+2
    static constexpr int K32 = D32 + 4 * PL32;          // [p<3][v]         factors, element planes x0-1 .. x0+1
    static constexpr int Z32 = K32 + 3 * PL32;          // [c][p<4][v]      operand, planes x0-1 .. x0+2
    static constexpr int R32 = Z32 + 3 * 4 * PL32;      // [c][p<2][v]      residual / result (own)
    // 16^3: own plane X (P = 1), 256 vertices per plane
    static constexpr int PL16 = 256;
    static constexpr int F16 = R32 + 3 * 2 * PL32;      // [c][v]
    static constexpr int D16 = F16 + 3 * PL16;          // [p<3][v]  planes X-1 .. X+1
    static constexpr int K16 = D16 + 3 * PL16;          // [p<2][v]  element planes X-1, X
    static constexpr int Z16 = K16 + 2 * PL16;          // [c][p<3][v]
    static constexpr int R16 = Z16 + 3 * 3 * PL16;      // [c][v]
    // 8^3 + 4^3 bottom (CTA 0; VBotLev<8> layout) and the pseudo-inverse
    static constexpr int B8 = R16 + 3 * PL16;
    static constexpr int G = B8 + vbot_floats(8);
    static constexpr int FLOATS = G + 64 * 64;
};

__device__ __forceinline__ int vt_w(int i, int n) { return i & (n - 1); }

// one level stencil on own planes: t from Z (planes own-1 .. own+P), k from K (element
// planes own-1 .. own+P-1); MODE 0: R = F - K Z ; MODE 1: R = Z + w D (F - K Z)
template <int N, int P, int MODE>
__device__ __forceinline__ void vt_stencil(const float* Z, const float* K, const float* F, const float* D, float* R,
                                           float s12, float omega, int tid, int nt) {
    constexpr int PL = N * N;
    for (int i = tid; i < P * PL; i += nt) {
        const int p = i / PL, v = i - p * PL, y = v / N, z = v - y * N;
        float k[2][4];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    k[q][j * 2 + r] = K[(p + q) * PL + vt_w(y - 1 + j, N) * N + vt_w(z - 1 + r, N)];
        const KSum<float> s = ksum<float>(k);
        const float dw = omega * D[(p + 1) * PL + v];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float* Zc = Z + c * (P + 2) * PL;
            float t[3][9];
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                    for (int r = 0; r < 3; ++r)
                        t[q][j * 3 + r] = Zc[(p + q) * PL + vt_w(y - 1 + j, N) * N + vt_w(z - 1 + r, N)];
            const float kt = apply_compact<float>(t, k, s, s12);
            const float f = F[(c * P + p) * PL + v];
            R[(c * P + p) * PL + v] = MODE == 0 ? f - kt : t[1][4] + dw * (f - kt);
        }
    }
}

// restriction of one fine plane triple (planes a = 2X-1, b = 2X, c = 2X+1, each [case][N*N]
// with case stride cs) to the coarse plane X (N/2 x N/2, case stride N*N/4)
template <int N>
__device__ __forceinline__ void vt_restrict_plane(const float* a, const float* b, const float* cpl, int cs,
                                                  float* out, int tid, int nt) {
    constexpr int M = N / 2;
    const float w[3] = {0.25f, 0.5f, 0.25f};
    for (int i = tid; i < 3 * M * M; i += nt) {
        const int cc = i / (M * M), v = i - cc * M * M, Y = v / M, Zc = v - Y * M;
        const float* pl[3] = {a + cc * cs, b + cc * cs, cpl + cc * cs};
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            float sb = 0.f;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const float* row = pl[q] + vt_w(2 * Y - 1 + j, N) * N;
                const float sz = w[0] * row[vt_w(2 * Zc - 1, N)] + w[1] * row[2 * Zc] + w[2] * row[vt_w(2 * Zc + 1, N)];
                sb += w[j] * sz;
            }
            s += w[q] * sb;
        }
        out[cc * M * M + v] = s;
    }
}

// value of the trilinear prolongation at fine (y, z) of a fine plane that interpolates
// the coarse planes ca (and cb when odd, else nullptr), coarse M x M
template <int M>
__device__ __forceinline__ float vt_prolong_at(const float* ca, const float* cb, int y, int z) {
    const int Y = y >> 1, Zc = z >> 1, Y1 = vt_w(Y + 1, M), Z1 = vt_w(Zc + 1, M);
    auto pz = [&](const float* pl, int yy) {
        return (z & 1) ? 0.5f * (pl[yy * M + Zc] + pl[yy * M + Z1]) : pl[yy * M + Zc];
    };
    auto py = [&](const float* pl) { return (y & 1) ? 0.5f * (pz(pl, Y) + pz(pl, Y1)) : pz(pl, Y); };
    return cb ? 0.5f * (py(ca) + py(cb)) : py(ca);
}

template <int CTAS = kVtCtas>   // (a template: the header is seen by several translation units)
__global__ void __launch_bounds__(512, 1) k_vtail32(VTailArgs A) {   // launched as ONE 16-CTA cluster
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) float vt_smem[];
    float* S = vt_smem;
    using L = VtLay;
    const int c = (int)cl.block_rank();                  // == blockIdx.x for a 1-D grid of one cluster
    const int tid = threadIdx.x, nt = blockDim.x;
    const float om = A.omega;
    auto peer = [&](int rank) { return cl.map_shared_rank(S, vt_w(rank, kVtCtas)); };
    // ---- static data (factors, D^-1, G): before the programmatic-dependency wait ----
    {
        const int x0 = 2 * c;
        for (int i = tid; i < 4 * L::PL32; i += nt) {            // D^-1 planes x0-1 .. x0+2
            const int p = i / L::PL32, v = i - p * L::PL32;
            S[L::D32 + i] = __ldg(A.dinv[0] + vt_w(x0 - 1 + p, 32) * L::PL32 + v);
        }
        for (int i = tid; i < 3 * L::PL32; i += nt) {            // factors, element planes x0-1 .. x0+1
            const int p = i / L::PL32, v = i - p * L::PL32;
            S[L::K32 + i] = __ldg(A.kap[0] + vt_w(x0 - 1 + p, 32) * L::PL32 + v);
        }
        for (int i = tid; i < 3 * L::PL16; i += nt) {
            const int p = i / L::PL16, v = i - p * L::PL16;
            S[L::D16 + i] = __ldg(A.dinv[1] + vt_w(c - 1 + p, 16) * L::PL16 + v);
        }
        for (int i = tid; i < 2 * L::PL16; i += nt) {
            const int p = i / L::PL16, v = i - p * L::PL16;
            S[L::K16 + i] = __ldg(A.kap[1] + vt_w(c - 1 + p, 16) * L::PL16 + v);
        }
        if (c == 0) {
            using V8 = VBotLev<8>;
            for (int i = tid; i < V8::n; i += nt) {
                S[L::B8 + V8::K + i] = __ldg(A.kap[2] + i);
                S[L::B8 + V8::D + i] = __ldg(A.dinv[2] + i);
            }
            for (int i = tid; i < 64 * 64 / 4; i += nt)
                reinterpret_cast<float4*>(S + L::G)[i] = __ldg(reinterpret_cast<const float4*>(A.G) + i);
        }
    }
    pdl_wait();
    // ---- 32^3 down: f own, z0 = w D^-1 f on planes x0-1 .. x0+2, res own ----
    {
        const int x0 = 2 * c;
        for (int i = tid; i < 3 * 4 * L::PL32; i += nt) {
            const int cc = i / (4 * L::PL32), r = i - cc * 4 * L::PL32, p = r / L::PL32, v = r - p * L::PL32;
            const float f = __ldg(A.f32 + (size_t)cc * 32768 + vt_w(x0 - 1 + p, 32) * L::PL32 + v);
            S[L::Z32 + i] = f * (om * S[L::D32 + p * L::PL32 + v]);
            if (p == 1 || p == 2) S[L::F32 + (cc * 2 + p - 1) * L::PL32 + v] = f;
        }
        __syncthreads();
        vt_stencil<32, 2, 0>(S + L::Z32, S + L::K32, S + L::F32, S + L::D32, S + L::R32, A.s12[0], om, tid, nt);
    }
    cl.sync();                                                     // S1: every res32 plane
    // ---- restrict 32 -> 16: coarse plane c from fine planes 2c-1 (CTA c-1), 2c, 2c+1 ----
    {
        const float* prev = peer(c - 1) + L::R32 + L::PL32;        // its local plane 1
        vt_restrict_plane<32>(prev, S + L::R32, S + L::R32 + L::PL32, 2 * L::PL32, S + L::F16, tid, nt);
    }
    cl.sync();                                                     // S2: every f16 plane
    // ---- 16^3 down: z0 on planes c-1 .. c+1 (neighbour f through DSMEM), res own ----
    {
        const float* fm = peer(c - 1) + L::F16;
        const float* fp = peer(c + 1) + L::F16;
        for (int i = tid; i < 3 * 3 * L::PL16; i += nt) {
            const int cc = i / (3 * L::PL16), r = i - cc * 3 * L::PL16, p = r / L::PL16, v = r - p * L::PL16;
            const float* src = p == 0 ? fm : (p == 1 ? S + L::F16 : fp);
            S[L::Z16 + i] = src[cc * L::PL16 + v] * (om * S[L::D16 + p * L::PL16 + v]);
        }
        __syncthreads();
        vt_stencil<16, 1, 0>(S + L::Z16, S + L::K16, S + L::F16, S + L::D16, S + L::R16, A.s12[1], om, tid, nt);
    }
    cl.sync();                                                     // S3: every res16 plane
    // ---- CTA 0: restrict 16 -> 8 (all 8 planes) and the 8^3 + 4^3 bottom ----
    if (c == 0) {
        using V8 = VBotLev<8>;
        float* B = S + L::B8;
        for (int X = 0; X < 8; ++X) {
            const float* a = peer(2 * X - 1) + L::R16;
            const float* b = peer(2 * X) + L::R16;
            const float* d = peer(2 * X + 1) + L::R16;
            // coarse plane X of all three cases into the 8^3 f (case stride 512)
            constexpr int M = 8;
            const float w[3] = {0.25f, 0.5f, 0.25f};
            for (int i = tid; i < 3 * M * M; i += nt) {
                const int cc = i / (M * M), v = i - cc * M * M, Y = v / M, Zc = v - Y * M;
                const float* pl[3] = {a + cc * L::PL16, b + cc * L::PL16, d + cc * L::PL16};
                float s = 0.f;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    float sb = 0.f;
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const float* row = pl[q] + vt_w(2 * Y - 1 + j, 16) * 16;
                        const float sz = w[0] * row[vt_w(2 * Zc - 1, 16)] + w[1] * row[2 * Zc] +
                                         w[2] * row[vt_w(2 * Zc + 1, 16)];
                        sb += w[j] * sz;
                    }
                    s += w[q] * sb;
                }
                B[V8::F + cc * V8::n + X * 64 + v] = s;
            }
        }
        __syncthreads();
        VBotArgs vb{};
        vb.omega = om;
        vb.s12[0] = A.s12[2];
        vb.s12[1] = A.s12[3];
        vb_cycle<8>(B, vb, S + L::G, 0);                          // result in B + V8::R
    }
    cl.sync();                                                     // S4: e8 in CTA 0
    // ---- 16^3 up: z = z0 + P e8 on the own plane, halo exchange, Jacobi ----
    {
        using V8 = VBotLev<8>;
        const float* e8 = peer(0) + L::B8 + V8::R;
        const int X = c >> 1;
        const float* ca_base = e8 + X * 64;
        const float* cb_base = (c & 1) ? e8 + vt_w(X + 1, 8) * 64 : nullptr;
        for (int i = tid; i < 3 * L::PL16; i += nt) {
            const int cc = i / L::PL16, v = i - cc * L::PL16, y = v >> 4, z = v & 15;
            const float add = vt_prolong_at<8>(ca_base + cc * 512, cb_base ? cb_base + cc * 512 : nullptr, y, z);
            S[L::Z16 + (cc * 3 + 1) * L::PL16 + v] += add;
        }
    }
    cl.sync();                                                     // S5: every z16 own plane
    {
        const float* zm = peer(c - 1) + L::Z16;
        const float* zp = peer(c + 1) + L::Z16;
        for (int i = tid; i < 3 * L::PL16; i += nt) {
            const int cc = i / L::PL16, v = i - cc * L::PL16;
            S[L::Z16 + (cc * 3 + 0) * L::PL16 + v] = zm[(cc * 3 + 1) * L::PL16 + v];
            S[L::Z16 + (cc * 3 + 2) * L::PL16 + v] = zp[(cc * 3 + 1) * L::PL16 + v];
        }
    }
    __syncthreads();                                               // halos in place (peers only read plane 1)
    vt_stencil<16, 1, 1>(S + L::Z16, S + L::K16, S + L::F16, S + L::D16, S + L::R16, A.s12[1], om, tid, nt);
    cl.sync();                                                     // S6: every e16 plane
    // ---- 32^3 up: z = z0 + P e16 on own planes 2c (plane c) and 2c+1 (planes c, c+1) ----
    {
        const float* ec = S + L::R16;
        const float* en = peer(c + 1) + L::R16;
        for (int i = tid; i < 3 * 2 * L::PL32; i += nt) {
            const int cc = i / (2 * L::PL32), r = i - cc * 2 * L::PL32, p = r / L::PL32, v = r - p * L::PL32;
            const int y = v >> 5, z = v & 31;
            const float add = vt_prolong_at<16>(ec + cc * L::PL16, p ? en + cc * L::PL16 : nullptr, y, z);
            S[L::Z32 + (cc * 4 + 1 + p) * L::PL32 + v] += add;
        }
    }
    cl.sync();                                                     // S7: every z32 own plane
    {
        const float* zm = peer(c - 1) + L::Z32;
        const float* zp = peer(c + 1) + L::Z32;
        for (int i = tid; i < 3 * L::PL32; i += nt) {
            const int cc = i / L::PL32, v = i - cc * L::PL32;
            S[L::Z32 + (cc * 4 + 0) * L::PL32 + v] = zm[(cc * 4 + 2) * L::PL32 + v];   // its plane x0+1
            S[L::Z32 + (cc * 4 + 3) * L::PL32 + v] = zp[(cc * 4 + 1) * L::PL32 + v];   // its plane x0
        }
    }
    cl.sync();                                                     // S8: halos read; no DSMEM access after this
    vt_stencil<32, 2, 1>(S + L::Z32, S + L::K32, S + L::F32, S + L::D32, S + L::R32, A.s12[0], om, tid, nt);
    __syncthreads();
    {
        const int x0 = 2 * c;
        for (int i = tid; i < 3 * 2 * L::PL32; i += nt) {
            const int cc = i / (2 * L::PL32), r = i - cc * 2 * L::PL32;
            A.out32[(size_t)cc * 32768 + x0 * L::PL32 + r] = S[L::R32 + i];
        }
    }
}

}  // namespace otm
