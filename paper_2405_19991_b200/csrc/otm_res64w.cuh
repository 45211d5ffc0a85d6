// fp64 defect kernel k_res64w (level 0, TMA ring, one case per work unit).
#pragma once

#include "otm_tma.cuh"

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
    int lock;                // > 0: CTA b owns (case, row tile) b % (3 nty) and x chunk b / (3 nty) of
                             // `lock`: row-tile neighbours march the same planes together, so the halo
                             // rows hit L2 (contiguous ranges re-read them from HBM: 3.0x the
                             // algorithmic bytes at 512^3 with one-row tiles)
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
                                                   double* partials, unsigned* counter, double* out9,
                                                   const int* __restrict__ skip) {
    if (skip && *skip) return;      // device-side solve control: the solve is already over
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
    long long u, u1;
    if (maps.lock > 0) {
        const unsigned rows = 3u * (unsigned)nty;
        const long long p = blockIdx.x % rows, ch = blockIdx.x / rows;
        u = p * g.nx + (long long)g.nx * ch / maps.lock;
        u1 = p * g.nx + (long long)g.nx * (ch + 1) / maps.lock;
    } else {
        u = W * blockIdx.x / B;
        u1 = W * (blockIdx.x + 1) / B;
    }
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

