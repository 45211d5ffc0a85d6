// k6: TMA-staged level stencils (three load cases per thread, 21-point weights,
// paired fp32) -- the Blackwell-native form of k4.
//
// Every x-plane of the staged arrays arrives in shared memory through the Tensor
// Memory Accelerator: one elected thread issues cp.async.bulk.tensor boxes that
// complete on a per-slot mbarrier (expect_tx bytes), so address generation and the
// global->shared transfer bypass the LSU/L1 pipe that the stencil's shared-memory
// reads need (the measured limit of the cp.async ring in k3/k4/k5).
//
// Tile = the full z extent (nz in {64, 128, 256}: one TMA box row) x TY = 512/nz
// rows, so periodic z neighbours are resolved inside shared memory; the wrapped y
// halo rows are extra one-row boxes (a second tensor map with box height 1).  The
// three load-case arrays are one tensor of 3 nx planes (case-major).
#pragma once

#include <cuda.h>

#include "otm_stencil4.cuh"

namespace otm {

constexpr int kAhead6 = 3;
constexpr int kStages6 = kAhead6 + 3;    // iteration s reads planes s-2..s; plane s+kAhead6 reuses the slot of s-3

__host__ __device__ inline int k6_ty(int nz) { return 512 / nz; }
__host__ __device__ inline bool k6_ok(const Geo& g, const LevelTemplate& lt) {
    return lt.equal && (g.nz == 64 || g.nz == 128 || g.nz == 256) && g.ny % k6_ty(g.nz) == 0 && g.nx >= 2;
}
// floats per slot: NT operand tiles of (TY+2) rows + the factor tile of (TY+1) rows
__host__ __device__ inline int k6_slot_floats(int NT, int nz) { return (NT * (k6_ty(nz) + 2) + k6_ty(nz) + 1) * nz; }
__host__ __device__ inline size_t k6_smem_bytes(int NT, int nz) {
    return (size_t)kStages6 * k6_slot_floats(NT, nz) * 4 + kStages6 * 8;
}

// main (TY rows) and halo (1 row) box maps: [0] the 3-case array, [1] D^-1, [2] factors
struct K6Maps {
    CUtensorMap main[3];
    CUtensorMap halo[3];
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
// bounded wait: a transaction-count mismatch traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    for (unsigned spin = 0;; ++spin) {
        unsigned done;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done) : "r"(a), "r"(phase) : "memory");
        if (done) return;
        if (spin > (1u << 22)) __trap();
    }
}
__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int z, int y, int x, uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(d), "l"(map), "r"(z), "r"(y), "r"(x), "r"(b)
        : "memory");
}

// Op contract (k6):
//   static constexpr int NT;           staged tiles: 0..2 the three cases of the operand array, 3 = D^-1 (optional)
//   float  op1(const float* S, int c, int r, int z) const    operand of case c at tile row r, column z
//   float2 op2(const float* S, int c, int r, int z) const    operand at (r, z), (r, z+1); z even
//   void prefetch(int x, long long vrow)
//   void sink(const float* S0, int c, long long v, int r, int z, float2 kt, float2 ctr)
// Ops see the tile geometry through `tile` (floats per operand tile) and `nz`.
template <class Op>
__device__ __forceinline__ void march6(const Geo& g, const LevelTemplate& lt, const K6Maps& maps, Op& op) {
    extern __shared__ __align__(128) float4 k6_smem4[];
    float* smem = reinterpret_cast<float*>(k6_smem4);
    constexpr int NT = Op::NT;
    constexpr int NZ = Op::NZ;
    constexpr int TY = 512 / NZ;
    constexpr int ROWS = TY + 2;
    constexpr int SLOT = (NT * (TY + 2) + TY + 1) * NZ;
    constexpr int TILE = ROWS * NZ;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages6 * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < kStages6; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    pdl_wait();                                            // predecessor outputs visible from here
    unsigned phase_bits = 0;                               // bit k: parity of slot k's next completion
    const unsigned plane_bytes = (unsigned)((NT * ROWS + TY + 1) * NZ * 4);
    const int tz = threadIdx.x * 2;
    const int zl = tz == 0 ? NZ - 1 : tz - 1;
    const int zr = tz + 2 == NZ ? 0 : tz + 2;
    const int tr = threadIdx.y + 1;
    const float2 s12 = f2((float)lt.s12, (float)lt.s12);
    const int nty = g.ny / TY;
    const long long W = (long long)nty * g.nx;
    const long long B = gridDim.x;
    long long u = W * blockIdx.x / B;
    const long long u1 = W * (blockIdx.x + 1) / B;
    int seq = 0;                                           // ring position of the segment's plane 0
    while (u < u1) {
        const int yt = (int)(u / g.nx);
        const int x0 = (int)(u - (long long)yt * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int y0 = yt * TY;
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TY == g.ny ? 0 : y0 + TY;
        const int nplanes = (x1 - x0) + 2;
        auto issue = [&](int s) {
            const int k = (seq + s) % kStages6;
            float* S = smem + k * SLOT;
            int x = x0 - 1 + s;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(bars + k, plane_bytes);
#pragma unroll
            for (int a = 0; a < NT; ++a) {
                float* T = S + a * TILE;
                const int mi = a < 3 ? 0 : 1;
                const int xc = a < 3 ? a * g.nx + x : x;
                tma_load_3d(T + NZ, &maps.main[mi], 0, y0, xc, bars + k);
                tma_load_3d(T, &maps.halo[mi], 0, ym, xc, bars + k);
                tma_load_3d(T + (TY + 1) * NZ, &maps.halo[mi], 0, yp, xc, bars + k);
            }
            float* K = S + NT * TILE;
            tma_load_3d(K + NZ, &maps.main[2], 0, y0, x, bars + k);
            tma_load_3d(K, &maps.halo[2], 0, ym, x, bars + k);
        };
        if (tid == 0)
            for (int s = 0; s < kAhead6 && s < nplanes; ++s) issue(s);
        const long long vrow = (long long)(y0 + threadIdx.y) * NZ + tz;
        op.prefetch(x0, vrow);
        for (int s = 0; s < nplanes; ++s) {
            const int k = (seq + s) % kStages6;
            mbar_wait(bars + k, (phase_bits >> k) & 1u);
            phase_bits ^= 1u << k;
            __syncthreads();             // all reads of iteration s-1 retired: the slot of plane s-3 is free
            if (tid == 0 && s + kAhead6 < nplanes) issue(s + kAhead6);
            if (s < 2) continue;
            const float* Sm = smem + ((seq + s - 2) % kStages6) * SLOT;
            const float* S0 = smem + ((seq + s - 1) % kStages6) * SLOT;
            const float* Sp = smem + k * SLOT;
            const int x = x0 + s - 2;
            W21 w;
            {
                float Ka[2][3], Kb[2][3];
                const float* ka = Sm + NT * TILE;
                const float* kb = S0 + NT * TILE;
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int o = (tr - 1 + jj) * NZ;
                    Ka[jj][0] = ka[o + zl];
                    const float2 va = *reinterpret_cast<const float2*>(ka + o + tz);
                    Ka[jj][1] = va.x; Ka[jj][2] = va.y;
                    Kb[jj][0] = kb[o + zl];
                    const float2 vb = *reinterpret_cast<const float2*>(kb + o + tz);
                    Kb[jj][1] = vb.x; Kb[jj][2] = vb.y;
                }
                w21_build(Ka, Kb, w);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                auto row = [&](const float* S, int j, float2& L, float2& C, float2& R) {
                    const float a0 = op.op1(S, c, tr + j, zl);
                    const float2 m = op.op2(S, c, tr + j, tz);
                    const float a3 = op.op1(S, c, tr + j, zr);
                    L = f2(a0, m.x);
                    C = m;
                    R = f2(m.y, a3);
                };
                float2 L0, C0, R0, l, cc, r;
                row(S0, 0, L0, C0, R0);
                float2 acc = fmul2(w.kv4, C0);
                float2 acc2 = f2(0.f, 0.f);
                row(S0, -1, l, cc, r);
                acc2 = ffma2(w.e[8], l, acc2);
                acc = ffma2(w.e[9], r, acc);
                row(S0, +1, l, cc, r);
                acc2 = ffma2(w.e[10], l, acc2);
                acc = ffma2(w.e[11], r, acc);
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const float* S = q == 0 ? Sm : Sp;
                    row(S, 0, l, cc, r);
                    acc2 = ffma2(w.e[4 + q * 2], l, acc2);
                    acc = ffma2(w.e[5 + q * 2], r, acc);
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        row(S, jj == 0 ? -1 : 1, l, cc, r);
                        acc2 = ffma2(w.e[q * 2 + jj], cc, acc2);
                        acc = ffma2(w.k[q | (jj << 1)], l, acc);
                        acc2 = ffma2(w.k[q | (jj << 1) | 4], r, acc2);
                    }
                }
                op.sink(S0, c, vrow + (long long)x * g.pl, tr, tz, fmul2(s12, fadd2(acc, acc2)), C0);
            }
            if (x + 1 < x1) op.prefetch(x + 1, vrow);
        }
        seq = (seq + nplanes) % kStages6;
        __syncthreads();
        u += x1 - x0;
    }
}

}  // namespace otm

namespace otm {

// ---------------------------------------------------------------------------
// k7: TMA staging (as k6) + one load case per thread with the operand window kept
// in registers across x (only the newly landed plane is read from shared memory)
// + z neighbours by warp shuffles (one LDS.64 per row; the two warp-edge lanes
// read their outer neighbour from shared memory) + 21-weight FFMA2 arithmetic.
// Work units: (case, row tile, x plane), persistent contiguous ranges per block.
// Staged tiles per plane: NT operand-side tiles of the block's case (T, or f and
// D^-1) with TY+2 rows, then the factor tile with TY+1 rows.
// ---------------------------------------------------------------------------
template <class Op>
__device__ __forceinline__ void march7(const Geo& g, const LevelTemplate& lt, const K6Maps& maps, Op& op,
                                       int& last_case) {
    extern __shared__ __align__(128) float4 k6_smem4[];
    float* smem = reinterpret_cast<float*>(k6_smem4);
    constexpr int NT = Op::NT;
    const int TY = k6_ty(g.nz);
    const int ROWS = TY + 2;
    const int SLOT = k6_slot_floats(NT, g.nz);
    const int TILE = ROWS * g.nz;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages6 * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < kStages6; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    unsigned phase_bits = 0;
    const unsigned plane_bytes = (unsigned)((NT * ROWS + TY + 1) * g.nz * 4);
    const int tz = threadIdx.x * 2;
    const int zl = tz == 0 ? g.nz - 1 : tz - 1;
    const int zr = tz + 2 == g.nz ? 0 : tz + 2;
    const int tr = threadIdx.y + 1;
    const float2 s12 = f2((float)lt.s12, (float)lt.s12);
    const int nty = g.ny / TY;
    const long long W = 3LL * nty * g.nx;
    const long long B = gridDim.x;
    long long u = W * blockIdx.x / B;
    const long long u1 = W * (blockIdx.x + 1) / B;
    int seq = 0;
    last_case = -1;
    // operand row of the new plane: value pairs at (z-1, z), (z, z+1), (z+1, z+2) from one LDS.64 + shuffles
    auto read_row = [&](const float* S, int r, float (&out)[4]) {
        const float2 m = op.op2(S, r, tz);
        float left = __shfl_up_sync(0xffffffffu, m.y, 1);
        float right = __shfl_down_sync(0xffffffffu, m.x, 1);
        if (lane == 0) left = op.op1(S, r, zl);
        if (lane == 31) right = op.op1(S, r, zr);
        out[0] = left; out[1] = m.x; out[2] = m.y; out[3] = right;
    };
    auto read_k = [&](const float* S, int r, float (&out)[3]) {
        const float* K = S + NT * TILE + r * g.nz;
        const float2 m = *reinterpret_cast<const float2*>(K + tz);
        float left = __shfl_up_sync(0xffffffffu, m.y, 1);
        if (lane == 0) left = K[zl];
        out[0] = left; out[1] = m.x; out[2] = m.y;
    };
    while (u < u1) {
        const long long colu = u / g.nx;
        const int x0 = (int)(u - colu * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int c = (int)(colu / nty);
        const int y0 = (int)(colu - (long long)c * nty) * TY;
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TY == g.ny ? 0 : y0 + TY;
        const int nplanes = (x1 - x0) + 2;
        op.begin_case(c, last_case);
        auto issue = [&](int s) {
            const int k = (seq + s) % kStages6;
            float* S = smem + k * SLOT;
            int x = x0 - 1 + s;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(bars + k, plane_bytes);
#pragma unroll
            for (int a = 0; a < NT; ++a) {
                float* T = S + a * TILE;
                const int mi = a == 0 ? 0 : 1;                 // tile 0: the case array; tile 1: D^-1
                const int xc = a == 0 ? c * g.nx + x : x;
                tma_load_3d(T + g.nz, &maps.main[mi], 0, y0, xc, bars + k);
                tma_load_3d(T, &maps.halo[mi], 0, ym, xc, bars + k);
                tma_load_3d(T + (TY + 1) * g.nz, &maps.halo[mi], 0, yp, xc, bars + k);
            }
            float* K = S + NT * TILE;
            tma_load_3d(K + g.nz, &maps.main[2], 0, y0, x, bars + k);
            tma_load_3d(K, &maps.halo[2], 0, ym, x, bars + k);
        };
        if (tid == 0)
            for (int s = 0; s < kAhead6 && s < nplanes; ++s) issue(s);
        const long long vrow = (long long)(y0 + threadIdx.y) * g.nz + tz;
        op.prefetch(c, x0, vrow);
        float Pm[3][4], P0[3][4], Pp[3][4], Ka[2][3], Kb[2][3];
        for (int s = 0; s < nplanes; ++s) {
            const int k = (seq + s) % kStages6;
            mbar_wait(bars + k, (phase_bits >> k) & 1u);
            phase_bits ^= 1u << k;
            __syncthreads();
            if (tid == 0 && s + kAhead6 < nplanes) issue(s + kAhead6);
            const float* Sk = smem + k * SLOT;
            if (s == 0) {
#pragma unroll
                for (int j = 0; j < 3; ++j) read_row(Sk, tr - 1 + j, Pm[j]);
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) read_k(Sk, tr - 1 + jj, Ka[jj]);
                continue;
            }
            if (s == 1) {
#pragma unroll
                for (int j = 0; j < 3; ++j) read_row(Sk, tr - 1 + j, P0[j]);
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) read_k(Sk, tr - 1 + jj, Kb[jj]);
                continue;
            }
            // operand plane x+1 lands in Pp; factor planes x-1 (Ka) and x (Kb) are held
#pragma unroll
            for (int j = 0; j < 3; ++j) read_row(Sk, tr - 1 + j, Pp[j]);
            W21 w;
            w21_build(Ka, Kb, w);
            const float2 kt = fmul2(s12, apply21(w, Pm, P0, Pp));
            const int x = x0 + s - 2;
            const float* S0 = smem + ((seq + s - 1) % kStages6) * SLOT;
            op.sink(S0, c, vrow + (long long)x * g.pl, tr, tz, kt, f2(P0[1][1], P0[1][2]));
            if (x + 1 < x1) op.prefetch(c, x + 1, vrow);
            // slide: factor plane x+1 comes from the slot just landed
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
                for (int m = 0; m < 4; ++m) { Pm[j][m] = P0[j][m]; P0[j][m] = Pp[j][m]; }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
#pragma unroll
                for (int m = 0; m < 3; ++m) Ka[jj][m] = Kb[jj][m];
            }
            if (s + 1 < nplanes) {
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) read_k(Sk, tr - 1 + jj, Kb[jj]);
            }
        }
        last_case = c;
        seq = (seq + nplanes) % kStages6;
        __syncthreads();
        u += x1 - x0;
    }
}

}  // namespace otm
