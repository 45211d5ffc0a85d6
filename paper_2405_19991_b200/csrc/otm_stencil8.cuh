// k8: level-0 stencil marcher = k6's TMA + mbarrier staging (full-z row tiles of
// TY rows + halos, one slot per x plane) + a register window along x for all
// three load cases.  Each thread owns the vertex pair (z, z+1) of one row and
// keeps the 3 rows x (z-1, z, z+1, z+2) operand values of the previous and the
// current plane in registers, so each newly landed plane is read from shared
// memory ONCE (3 rows per case) instead of three times (9 rows per case in k6):
// ~2.9x fewer shared-memory wavefronts per output.  ~190 registers per thread
// -> one 256-thread CTA per SM; the deeper TMA ring (kAhead8 planes in flight)
// keeps the HBM pipe full with fewer resident warps.
#pragma once

#include "otm_stencil6.cuh"

namespace otm {

constexpr int kStages8 = 9;
constexpr int kAhead8 = 7;          // kStages8 >= kAhead8 + 2: the slot refilled at step s held plane s-2
static_assert(kStages8 >= kAhead8 + 2, "k8 ring too shallow");

__host__ __device__ inline size_t k8_smem_bytes(int NT, int nz) {
    return (size_t)kStages8 * k6_slot_floats(NT, nz) * 4 + kStages8 * 8;
}

struct K8Row {
    float a0, mx, my, a3;           // operand at z-1, z, z+1, z+2 of the thread's pair
};

__device__ __forceinline__ float2 k8L(const K8Row& r) { return f2(r.a0, r.mx); }
__device__ __forceinline__ float2 k8C(const K8Row& r) { return f2(r.mx, r.my); }
__device__ __forceinline__ float2 k8R(const K8Row& r) { return f2(r.my, r.a3); }

// rows tr-1, tr, tr+1 of the three cases from one staged plane
template <class Op>
__device__ __forceinline__ void k8_load(const Op& op, const float* S, int tr, int tz, int zl, int zr,
                                        K8Row (&N)[3][3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int r = tr - 1 + j;
            N[c][j].a0 = op.op1(S, c, r, zl);
            const float2 m = op.op2(S, c, r, tz);
            N[c][j].mx = m.x;
            N[c][j].my = m.y;
            N[c][j].a3 = op.op1(S, c, r, zr);
        }
}

// factor rows tr-1, tr of one staged element plane (columns z-1, z, z+1)
__device__ __forceinline__ void k8_kappa(const float* kb, int nz, int tr, int tz, int zl, float (&K)[2][3]) {
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
        const int o = (tr - 1 + jj) * nz;
        K[jj][0] = kb[o + zl];
        const float2 v = *reinterpret_cast<const float2*>(kb + o + tz);
        K[jj][1] = v.x;
        K[jj][2] = v.y;
    }
}

// (K T) at the pair for the three cases from planes P (x-1), Q (x), N (x+1); same
// term order as march6
template <class Op>
__device__ __forceinline__ void k8_out(Op& op, const W21& w, const K8Row (&P)[3][3], const K8Row (&Q)[3][3],
                                       const K8Row (&N)[3][3], const float* S0, long long v, int tr, int tz,
                                       float2 s12) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float2 C0 = k8C(Q[c][1]);
        float2 acc = fmul2(w.kv4, C0);
        float2 acc2 = f2(0.f, 0.f);
        acc2 = ffma2(w.e[8], k8L(Q[c][0]), acc2);
        acc = ffma2(w.e[9], k8R(Q[c][0]), acc);
        acc2 = ffma2(w.e[10], k8L(Q[c][2]), acc2);
        acc = ffma2(w.e[11], k8R(Q[c][2]), acc);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const K8Row(&S)[3][3] = q == 0 ? P : N;
            acc2 = ffma2(w.e[4 + q * 2], k8L(S[c][1]), acc2);
            acc = ffma2(w.e[5 + q * 2], k8R(S[c][1]), acc);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const K8Row& row = S[c][jj == 0 ? 0 : 2];
                acc2 = ffma2(w.e[q * 2 + jj], k8C(row), acc2);
                acc = ffma2(w.k[q | (jj << 1)], k8L(row), acc);
                acc2 = ffma2(w.k[q | (jj << 1) | 4], k8R(row), acc2);
            }
        }
        op.sink(S0, c, v, tr, tz, fmul2(s12, fadd2(acc, acc2)), C0);
    }
}

template <class Op>
__device__ __forceinline__ void march8(const Geo& g, const LevelTemplate& lt, const K6Maps& maps, Op& op) {
    extern __shared__ __align__(128) float4 k8_smem4[];
    float* smem = reinterpret_cast<float*>(k8_smem4);
    constexpr int NT = Op::NT;
    constexpr int NZ = Op::NZ;
    constexpr int TY = 512 / NZ;
    constexpr int ROWS = TY + 2;
    constexpr int SLOT = (NT * (TY + 2) + TY + 1) * NZ;
    constexpr int TILE = ROWS * NZ;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages8 * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    if (tid == 0) {
        for (int k = 0; k < kStages8; ++k) mbar_init(bars + k, 1);
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
            const int k = (seq + s) % kStages8;
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
        // wait for plane s, retire step s-1 everywhere, refill the slot of plane s-2
        auto arrive = [&](int s) -> const float* {
            const int k = (seq + s) % kStages8;
            mbar_wait(bars + k, (phase_bits >> k) & 1u);
            phase_bits ^= 1u << k;
            __syncthreads();
            if (tid == 0 && s + kAhead8 < nplanes) issue(s + kAhead8);
            return smem + k * SLOT;
        };
        if (tid == 0)
            for (int s = 0; s < kAhead8 && s < nplanes; ++s) issue(s);
        const long long vrow = (long long)(y0 + threadIdx.y) * NZ + tz;
        op.prefetch(x0, vrow);
        K8Row A[3][3], Bq[3][3], Cq[3][3];
        float Ka[2][3];
        {
            const float* S = arrive(0);
            k8_load(op, S, tr, tz, zl, zr, A);
            k8_kappa(S + NT * TILE, NZ, tr, tz, zl, Ka);
            S = arrive(1);
            k8_load(op, S, tr, tz, zl, zr, Bq);
        }
        // one output plane: P = x-1, Q = x (slot S0, still resident), N = x+1 (just landed)
        auto step = [&](int s, const K8Row(&P)[3][3], const K8Row(&Q)[3][3], K8Row(&N)[3][3]) {
            const float* S = arrive(s);
            const float* S0 = smem + ((seq + s - 1) % kStages8) * SLOT;
            k8_load(op, S, tr, tz, zl, zr, N);
            float Kb[2][3];
            k8_kappa(S0 + NT * TILE, NZ, tr, tz, zl, Kb);
            W21 w;
            w21_build(Ka, Kb, w);
            const int x = x0 + s - 2;
            k8_out(op, w, P, Q, N, S0, vrow + (long long)x * g.pl, tr, tz, s12);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int q = 0; q < 3; ++q) Ka[jj][q] = Kb[jj][q];
            if (x + 1 < x1) op.prefetch(x + 1, vrow);
        };
        for (int s = 2; s < nplanes; s += 3) {
            step(s, A, Bq, Cq);
            if (s + 1 < nplanes) step(s + 1, Bq, Cq, A);
            if (s + 2 < nplanes) step(s + 2, Cq, A, Bq);
        }
        seq = (seq + nplanes) % kStages8;
        __syncthreads();
        u += x1 - x0;
    }
}

}  // namespace otm

namespace otm {

// ---------------------------------------------------------------------------
// k9: k8's register window without the per-plane CTA barrier.  Slots carry a
// "full" mbarrier (TMA transaction count) and an "empty" mbarrier that each of the
// 8 warps arrives on once it no longer reads the slot; thread 0 refills a slot
// only after its empty barrier completes, so warps drift freely and no warp waits
// for the TMA issue of another.  Slot lifetime: plane s is loaded at step s and
// read again (factors, sink) at step s+1, so it is released after step s+1 (plane
// 0 after the prologue, the segment's last plane after its own step).
// ---------------------------------------------------------------------------
constexpr int kStages9 = 9;          // all slots in flight: plane s + 7 is issued at step s

__host__ __device__ inline size_t k9_smem_bytes(int NT, int nz) {
    return (size_t)kStages9 * k6_slot_floats(NT, nz) * 4 + 2 * kStages9 * 8;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}

template <class Op>
__device__ __forceinline__ void march9(const Geo& g, const LevelTemplate& lt, const K6Maps& maps, Op& op) {
    extern __shared__ __align__(128) float4 k9_smem4[];
    float* smem = reinterpret_cast<float*>(k9_smem4);
    constexpr int NT = Op::NT;
    constexpr int NZ = Op::NZ;
    constexpr int TY = 512 / NZ;
    constexpr int ROWS = TY + 2;
    constexpr int SLOT = (NT * (TY + 2) + TY + 1) * NZ;
    constexpr int TILE = ROWS * NZ;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages9 * SLOT);
    uint64_t* empty = full + kStages9;
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    const int nwarps = (blockDim.x * blockDim.y) >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int k = 0; k < kStages9; ++k) {
            mbar_init(full + k, 1);
            mbar_init(empty + k, nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    pdl_wait();                                            // predecessor outputs visible from here
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
    long long pc = 0;                                      // global plane index of the segment's plane 0
    while (u < u1) {
        const int yt = (int)(u / g.nx);
        const int x0 = (int)(u - (long long)yt * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int y0 = yt * TY;
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TY == g.ny ? 0 : y0 + TY;
        const int nplanes = (x1 - x0) + 2;
        auto slot = [&](int s) { return (int)((pc + s) % kStages9); };
        auto issue = [&](int s) {                          // thread 0 only
            const int k = slot(s);
            const long long use = (pc + s) / kStages9;
            if (use > 0) mbar_wait(empty + k, (unsigned)((use - 1) & 1));
            float* S = smem + k * SLOT;
            int x = x0 - 1 + s;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(full + k, plane_bytes);
#pragma unroll
            for (int a = 0; a < NT; ++a) {
                float* T = S + a * TILE;
                const int mi = a < 3 ? 0 : 1;
                const int xc = a < 3 ? a * g.nx + x : x;
                tma_load_3d(T + NZ, &maps.main[mi], 0, y0, xc, full + k);
                tma_load_3d(T, &maps.halo[mi], 0, ym, xc, full + k);
                tma_load_3d(T + (TY + 1) * NZ, &maps.halo[mi], 0, yp, xc, full + k);
            }
            float* K = S + NT * TILE;
            tma_load_3d(K + NZ, &maps.main[2], 0, y0, x, full + k);
            tma_load_3d(K, &maps.halo[2], 0, ym, x, full + k);
        };
        auto arrive = [&](int s) -> const float* {
            const int k = slot(s);
            mbar_wait(full + k, (unsigned)(((pc + s) / kStages9) & 1));
            return smem + k * SLOT;
        };
        auto release = [&](int s) {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + slot(s));
        };
        if (tid == 0)
            for (int s = 0; s < kStages9 && s < nplanes; ++s) issue(s);      // fill the ring
        const long long vrow = (long long)(y0 + threadIdx.y) * NZ + tz;
        op.prefetch(x0, vrow);
        K8Row A[3][3], Bq[3][3], Cq[3][3];
        float Ka[2][3];
        {
            const float* S = arrive(0);
            k8_load(op, S, tr, tz, zl, zr, A);
            k8_kappa(S + NT * TILE, NZ, tr, tz, zl, Ka);
            release(0);
            S = arrive(1);
            k8_load(op, S, tr, tz, zl, zr, Bq);
        }
        auto step = [&](int s, const K8Row(&P)[3][3], const K8Row(&Q)[3][3], K8Row(&N)[3][3]) {
            const float* S = arrive(s);
            const float* S0 = smem + slot(s - 1) * SLOT;
            k8_load(op, S, tr, tz, zl, zr, N);
            float Kb[2][3];
            k8_kappa(S0 + NT * TILE, NZ, tr, tz, zl, Kb);
            W21 w;
            w21_build(Ka, Kb, w);
            const int x = x0 + s - 2;
            k8_out(op, w, P, Q, N, S0, vrow + (long long)x * g.pl, tr, tz, s12);
            release(s - 1);
            if (s == nplanes - 1) release(s);
            if (tid == 0 && s + kStages9 - 2 < nplanes) issue(s + kStages9 - 2);   // slot of plane s-2
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int q = 0; q < 3; ++q) Ka[jj][q] = Kb[jj][q];
            if (x + 1 < x1) op.prefetch(x + 1, vrow);
        };
        for (int s = 2; s < nplanes; s += 3) {
            step(s, A, Bq, Cq);
            if (s + 1 < nplanes) step(s + 1, Bq, Cq, A);
            if (s + 2 < nplanes) step(s + 2, Cq, A, Bq);
        }
        pc += nplanes;
        u += x1 - x0;
    }
}

}  // namespace otm
