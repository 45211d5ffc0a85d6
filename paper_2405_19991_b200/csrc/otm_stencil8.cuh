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
constexpr int kChunk8 = 16;         // planes per dynamically scheduled chunk
constexpr int kAhead8 = 7;          // kStages8 >= kAhead8 + 2: the slot refilled at step s held plane s-2
static_assert(kStages8 >= kAhead8 + 2, "k8 ring too shallow");

__host__ __device__ inline size_t k8_smem_bytes(int NT, int nz, int ty = 0) {
    if (ty == 0) ty = 512 / nz;
    return (size_t)kStages8 * ((NT * (ty + 2) + ty + 1) * nz) * 4 + kStages8 * 8;
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
__device__ __forceinline__ void march8(const Geo& g, const LevelTemplate& lt, const K6Maps& maps, Op& op,
                                       unsigned* work = nullptr) {
    extern __shared__ __align__(128) float4 k8_smem4[];
    float* smem = reinterpret_cast<float*>(k8_smem4);
    constexpr int NT = Op::NT;
    constexpr int NZ = Op::NZ;
    constexpr int TY = Op::TY;
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
    // work distribution: static contiguous ranges, or (work != nullptr) chunks of
    // kChunk8 planes of one row tile grabbed from a global counter, which balances
    // CTAs that stream from the far HBM stacks more slowly
    const int nct = (g.nx + kChunk8 - 1) / kChunk8;
    const int nchunks = nty * nct;
    __shared__ int s_chunk;
    while (true) {
        int yt, x0, x1;
        if (work) {
            if (tid == 0) s_chunk = (int)atomicAdd(work, 1u);
            __syncthreads();
            const int ch = s_chunk;
            if (ch >= nchunks) break;
            yt = ch / nct;
            x0 = (ch - yt * nct) * kChunk8;
            x1 = min(g.nx, x0 + kChunk8);
        } else {
            if (u >= u1) break;
            yt = (int)(u / g.nx);
            x0 = (int)(u - (long long)yt * g.nx);
            x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        }
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
    if (work && tid == 0) {                                // last CTA out resets the counter
        __threadfence();
        if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {
            atomicExch(work, 0u);
            atomicExch(work + 1, 0u);
        }
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

namespace otm {

// ---------------------------------------------------------------------------
// fp64 defect r = (f(kappa) - fmean) - K T on level 0 (solver.py:398-401) with the
// k8 structure in double precision: TMA + mbarrier ring of (row tile, x plane)
// slots holding T of ONE case (TYD + 2 rows) and kappa (TYD + 1 rows); each thread
// owns one vertex and keeps the 3 x 3 (y, z) neighbourhood of the previous, current
// and next plane in registers (27 doubles), so a plane is read from shared memory
// once.  Work units = (case, row tile, x plane); a CTA walks a contiguous range.
// The 21-point form of the element operator (face weights 0) in fp64; the loads f
// use the same fixed-order sum as k2_res64.  Per case and CTA: sum r^2, sum f^2,
// sum T, finished by the last CTA (fixed order).
// ---------------------------------------------------------------------------
constexpr int kStagesR = 10;
constexpr int kAheadR = 8;
static_assert(kStagesR >= kAheadR + 2, "res64 ring too shallow");

template <int NZ>
struct R64Geo {
    static constexpr int TYD = NZ >= 256 ? 1 : 256 / NZ;   // rows per tile (one vertex per thread)
    static constexpr int THREADS = NZ * TYD;
    static constexpr int MINB = THREADS > 256 ? 1 : 2;     // CTAs per SM
    static constexpr int TROWS = TYD + 2;
    static constexpr int KROWS = TYD + 1;
    static constexpr int SLOT = (TROWS + KROWS) * NZ;     // doubles
};

__host__ __device__ inline size_t r64_smem_bytes(int nz) {
    const int tyd = nz >= 256 ? 1 : 256 / nz;
    return (size_t)kStagesR * (2 * tyd + 3) * nz * 8 + kStagesR * 8;
}

struct R64Maps {
    CUtensorMap Tm, Th;      // T (3 cases stacked along x): main (TYD rows) / halo (1 row)
    CUtensorMap Km, Kh;      // kappa (fp64)
};

// nz = 512: 512 threads, 1 CTA per SM, and z-split (256, 2) maps (a TMA box
// dimension holds at most 256 elements; the box still lands as [row][nz])
__device__ __forceinline__ void r64_tma4(void* dst, const CUtensorMap* map, int z, int h, int y, int x, uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
        ::"r"(d), "l"(map), "r"(z), "r"(h), "r"(y), "r"(x), "r"(b)
        : "memory");
}
template <int NZ>
__device__ __forceinline__ void r64_ld(double* dst, const CUtensorMap* map, int y, int x, uint64_t* bar) {
    if constexpr (NZ > 256) r64_tma4(dst, map, 0, 0, y, x, bar);
    else tma_load_3d(reinterpret_cast<float*>(dst), map, 0, y, x, bar);
}

template <int NZ>
__global__ void __launch_bounds__(R64Geo<NZ>::THREADS, R64Geo<NZ>::MINB) k_res64w(Geo g, LevelTemplate lt, const __grid_constant__ R64Maps maps,
                                                   const double* __restrict__ fmean, float* __restrict__ r32,
                                                   double* partials, unsigned* counter, double* out9) {
    using RG = R64Geo<NZ>;
    constexpr int TYD = RG::TYD, TROWS = RG::TROWS, SLOT = RG::SLOT;
    extern __shared__ __align__(128) double r64_smem[];
    double* smem = r64_smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStagesR * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    if (tid == 0) {
        for (int k = 0; k < kStagesR; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    unsigned phase_bits = 0;
    const unsigned plane_bytes = (unsigned)(SLOT * 8);
    const int tz = threadIdx.x;
    const int zl = tz == 0 ? NZ - 1 : tz - 1;
    const int zr = tz + 1 == NZ ? 0 : tz + 1;
    const int ty = threadIdx.y;
    const double s12 = lt.s12;
    const int nty = g.ny / TYD;
    const long long W = 3LL * nty * g.nx;
    const long long B = gridDim.x;
    long long u = W * blockIdx.x / B;
    const long long u1 = W * (blockIdx.x + 1) / B;
    double acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = 0.0;
    int seq = 0;
    while (u < u1) {
        const long long per_case = (long long)nty * g.nx;
        const int c = (int)(u / per_case);
        const long long uc = u - (long long)c * per_case;
        const int yt = (int)(uc / g.nx);
        const int x0 = (int)(uc - (long long)yt * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int y0 = yt * TYD;
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TYD == g.ny ? 0 : y0 + TYD;
        const int nplanes = (x1 - x0) + 2;
        auto issue = [&](int s) {
            const int k = (seq + s) % kStagesR;
            double* S = smem + k * SLOT;
            int x = x0 - 1 + s;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(bars + k, plane_bytes);
            const int xc = c * g.nx + x;
            r64_ld<NZ>(S + NZ, &maps.Tm, y0, xc, bars + k);
            r64_ld<NZ>(S, &maps.Th, ym, xc, bars + k);
            r64_ld<NZ>(S + (TYD + 1) * NZ, &maps.Th, yp, xc, bars + k);
            double* K = S + TROWS * NZ;
            r64_ld<NZ>(K + NZ, &maps.Km, y0, x, bars + k);
            r64_ld<NZ>(K, &maps.Kh, ym, x, bars + k);
        };
        auto arrive = [&](int s) -> const double* {
            const int k = (seq + s) % kStagesR;
            mbar_wait(bars + k, (phase_bits >> k) & 1u);
            phase_bits ^= 1u << k;
            __syncthreads();
            if (tid == 0 && s + kAheadR < nplanes) issue(s + kAheadR);
            return smem + k * SLOT;
        };
        if (tid == 0)
            for (int s = 0; s < kAheadR && s < nplanes; ++s) issue(s);
        // window: [plane][y row j = y-1, y, y+1][z col = z-1, z, z+1]
        auto load = [&](const double* S, double (&P)[3][3]) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double* row = S + (ty + j) * NZ;
                P[j][0] = row[zl];
                P[j][1] = row[tz];
                P[j][2] = row[zr];
            }
        };
        // element factors of one element plane: rows y-1, y; columns z-1, z
        auto kload = [&](const double* S, double (&K)[2][2]) {
            const double* kt = S + TROWS * NZ;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                K[jj][0] = kt[(ty + jj) * NZ + zl];
                K[jj][1] = kt[(ty + jj) * NZ + tz];
            }
        };
        double A[3][3], Bw[3][3], Cw[3][3], Ka[2][2];
        {
            const double* S = arrive(0);
            load(S, A);
            kload(S, Ka);
            S = arrive(1);
            load(S, Bw);
        }
        const long long vrow = (long long)(y0 + ty) * NZ + tz;
        auto step = [&](int s, const double (&P)[3][3], const double (&Q)[3][3], double (&N)[3][3]) {
            const double* S = arrive(s);
            const double* S0 = smem + ((seq + s - 1) % kStagesR) * SLOT;
            load(S, N);
            double Kb[2][2];
            kload(S0, Kb);
            // K[q][jj][kk]: element (x-1+q, y-1+jj, z-1+kk)
            const double K000 = Ka[0][0], K001 = Ka[0][1], K010 = Ka[1][0], K011 = Ka[1][1];
            const double K100 = Kb[0][0], K101 = Kb[0][1], K110 = Kb[1][0], K111 = Kb[1][1];
            const double Kv = ((K000 + K001) + (K010 + K011)) + ((K100 + K101) + (K110 + K111));
            // neighbours: plane q' (0 = x-1 (P), 1 = x (Q), 2 = x+1 (N)), row j, col k
            double t = 4.0 * Kv * Q[1][1];
            // edges (dx, dy, 0)
            t -= (K000 + K001) * P[0][1] + (K010 + K011) * P[2][1] + (K100 + K101) * N[0][1] + (K110 + K111) * N[2][1];
            // edges (dx, 0, dz)
            t -= (K000 + K010) * P[1][0] + (K001 + K011) * P[1][2] + (K100 + K110) * N[1][0] + (K101 + K111) * N[1][2];
            // edges (0, dy, dz)
            t -= (K000 + K100) * Q[0][0] + (K001 + K101) * Q[0][2] + (K010 + K110) * Q[2][0] + (K011 + K111) * Q[2][2];
            // corners (dx, dy, dz): element spanned by v and v + d
            t -= K000 * P[0][0] + K001 * P[0][2] + K010 * P[2][0] + K011 * P[2][2];
            t -= K100 * N[0][0] + K101 * N[0][2] + K110 * N[2][0] + K111 * N[2][2];
            const double kt = s12 * t;
            // loads: f = sum_a f0[a][c] * kappa of the element whose corner a is v (k2_res64 order)
            const double Kq[2][2][2] = {{{K000, K001}, {K010, K011}}, {{K100, K101}, {K110, K111}}};
            double f = 0.0;
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int q = 1 - (a & 1), jj = 1 - ((a >> 1) & 1), kk = 1 - ((a >> 2) & 1);
                f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + c], Kq[q][jj][kk]));
            }
            const double r = (f - fmean[c]) - kt;
            const int x = x0 + s - 2;
            r32[(long long)c * g.n + (long long)x * g.pl + vrow] = (float)r;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                if (cc == c) {
                    acc[cc] += r * r;
                    acc[3 + cc] += f * f;
                    acc[6 + cc] += Q[1][1];
                }
            }
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) Ka[jj][kk] = Kb[jj][kk];
        };
        for (int s = 2; s < nplanes; s += 3) {
            step(s, A, Bw, Cw);
            if (s + 1 < nplanes) step(s + 1, Bw, Cw, A);
            if (s + 2 < nplanes) step(s + 2, Cw, A, Bw);
        }
        seq = (seq + nplanes) % kStagesR;
        __syncthreads();
        u += x1 - x0;
    }
    reduce_finalize<9>(acc, partials, counter, out9);
}

}  // namespace otm
