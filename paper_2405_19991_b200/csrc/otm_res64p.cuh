// fp64 defect kernel k_res64p: r = (f(kappa) - fmean) - K T on level 0 for all three
// load cases in one push x-march (solver.py:398-401, the loads of solver.py:347-363).
//
// The structure of the k10 level stencils (otm_stencil10.cuh) in double precision:
// one TMA box per landed x plane holds T of the three cases ([row][case][z], TY + 2
// rows) and one the element factors (TY + 1 rows); every landed plane is read from
// shared memory once and pushed into the three output planes it touches:
//   out(s-1) += X(kappa s-1; s)  -> finished: r = (f - fmean) - s12 (4 K_v T_v - sum)
//   out(s)   += Q(s)             (in-plane edges), centre T_v, load f_v
//   out(s+1)  = X(kappa s; s)    (started)
// One vertex per thread (NZ x TY = 256 threads), so the per-vertex weights (K_v, the
// 12 edge sums, 8 corners) and the load's element factors are formed once for the
// three cases, and one barrier per plane serves three cases (k_res64w: one case per
// work unit, weights rebuilt per case, one barrier per case-plane).  Per case and
// CTA: sum r^2, sum f^2, sum T, finished by the last CTA (fixed order).
#pragma once

#include "otm_stencil10.cuh"

namespace otm {

template <int NZ>
struct R64P {
    static constexpr int TY = NZ >= 256 ? 1 : 256 / NZ;     // rows per tile
    static constexpr int THREADS = NZ * TY;                  // one vertex per thread
    static constexpr int T = 0;                              // (TY + 2) x 3 x NZ doubles
    static constexpr int K = (TY + 2) * 3 * NZ;              // (TY + 1) x NZ doubles
    static constexpr int SLOT = K + (TY + 1) * NZ;
    static constexpr int SLOT_BYTES = SLOT * 8;
    static constexpr int CPS = NZ > 256 ? 1 : 2;             // CTAs per SM the ring is sized for
    static constexpr int BUDGET = (224 * 1024) / CPS - 2048;
    static constexpr int ST0 = BUDGET / (SLOT_BYTES + 8);
    static constexpr int STAGES = ST0 > 8 ? 8 : ST0;
    static constexpr int AHEAD = STAGES - 1;                 // a step reads only its own slot
    static constexpr size_t SMEM = (size_t)STAGES * SLOT_BYTES + STAGES * 8;
    static_assert(STAGES >= 3, "res64p ring too shallow");
};

// Box loads: a TMA box dimension holds at most 256 elements, so for NZ > 256 the
// host splits z into (256, NZ / 256) map dimensions (as k10_ld_c3); the box lands as
// [row][case][NZ] / [row][NZ], the same layout.
template <int NZ>
__device__ __forceinline__ void r64_ld_t(void* dst, const CUtensorMap* map, int y, int x, uint64_t* bar) {
    if constexpr (NZ > 256) tma_load_5d(reinterpret_cast<float*>(dst), map, 0, 0, 0, y, x, bar);
    else tma_load_4d(reinterpret_cast<float*>(dst), map, 0, 0, y, x, bar);
}
template <int NZ>
__device__ __forceinline__ void r64_ld_k(void* dst, const CUtensorMap* map, int y, int x, uint64_t* bar) {
    if constexpr (NZ > 256) tma_load_4d(reinterpret_cast<float*>(dst), map, 0, 0, y, x, bar);
    else tma_load_3d(reinterpret_cast<float*>(dst), map, 0, y, x, bar);
}

struct R64PMaps {
    CUtensorMap t_full, t_main, t_halo;      // 4-D (z, case, y, x) fp64: TY + 2 / TY / 1 rows
    CUtensorMap k_full, k_main, k_halo;      // 3-D (z, y, x) fp64: TY + 1 / TY / 1 rows
    int lock;                                // as K10Maps::lock (lockstep row-tile order beyond L2)
    int xa, xb;                              // output x planes [xa, xb) (as K10Maps)
};

// element factors of one element plane around the vertex: corners c[jj][kk] =
// element (., y-1+jj, z-1+kk), y-edges ey[jj], z-edges ez[kk], kvh = their sum
struct R64PW {
    double c[2][2], ey[2], ez[2], kvh;
};

struct R64PState {
    double Sc[3], Sn[3], C0[3], F[3];    // partial sums of out(p), out(p+1); centre T and load of out(p)
    double kv4s;                          // 4 s12 K_v of out(p)
    R64PW w;                              // factors of element plane p - 1
};

template <int NZ>
__global__ void __launch_bounds__(R64P<NZ>::THREADS, R64P<NZ>::CPS)
    k_res64p(Geo g, LevelTemplate lt, const __grid_constant__ R64PMaps maps, const double* __restrict__ fmean,
             float* __restrict__ r32, double* partials, unsigned* counter, double* out9,
             const int* __restrict__ skip) {
    if (skip && *skip) return;      // device-side solve control: the solve is already over
    using P = R64P<NZ>;
    constexpr int TY = P::TY, STAGES = P::STAGES, AHEAD = P::AHEAD, SLOT = P::SLOT;
    extern __shared__ __align__(128) double r64p_smem[];
    double* smem = r64p_smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    if (tid == 0) {
        for (int k = 0; k < STAGES; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    unsigned phase_bits = 0;
    const int tz = threadIdx.x;
    const int zl = tz == 0 ? NZ - 1 : tz - 1;
    const int zr = tz + 1 == NZ ? 0 : tz + 1;
    const int ty = threadIdx.y;
    const double s12 = lt.s12, s48 = 4.0 * lt.s12;
    const double fm[3] = {fmean[0], fmean[1], fmean[2]};
    const unsigned n = (unsigned)g.n, pl = (unsigned)g.pl;
    const int nty = g.ny / TY;
    const int nxr = maps.xb - maps.xa;
    const long long W = (long long)nty * nxr;
    long long u, u1;
    if (maps.lock > 0) {
        const int yt = (int)(blockIdx.x % (unsigned)nty), c = (int)(blockIdx.x / (unsigned)nty);
        u = (long long)yt * nxr + (long long)nxr * c / maps.lock;
        u1 = (long long)yt * nxr + (long long)nxr * (c + 1) / maps.lock;
    } else {
        u = W * blockIdx.x / gridDim.x;
        u1 = W * (blockIdx.x + 1) / gridDim.x;
    }
    double acc[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = 0.0;
    int kc = 0, ki = 0;
    auto weights = [&](const double* S, R64PW& w) {
        const double* K = S + P::K;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            w.c[jj][0] = K[(ty + jj) * NZ + zl];
            w.c[jj][1] = K[(ty + jj) * NZ + tz];
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) w.ey[jj] = w.c[jj][0] + w.c[jj][1];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) w.ez[kk] = w.c[0][kk] + w.c[1][kk];
        w.kvh = w.ey[0] + w.ey[1];
    };
    // rows y-1, y, y+1 x columns z-1, z, z+1 of case c
    auto rows = [&](const double* S, int c, double (&R)[3][3]) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double* row = S + P::T + ((ty + j) * 3 + c) * NZ;
            R[j][0] = row[zl];
            R[j][1] = row[tz];
            R[j][2] = row[zr];
        }
    };
    // X(w; neighbour plane rows R): 4 corners, 2 y-edges, 2 z-edges (face weight 0)
    auto xsum = [](const R64PW& w, const double (&R)[3][3], double a) -> double {
        double b = w.ey[0] * R[0][1];
        a = fma(w.c[0][0], R[0][0], a);
        b = fma(w.c[0][1], R[0][2], b);
        a = fma(w.c[1][0], R[2][0], a);
        b = fma(w.c[1][1], R[2][2], b);
        a = fma(w.ey[1], R[2][1], a);
        b = fma(w.ez[0], R[1][0], b);
        a = fma(w.ez[1], R[1][2], a);
        return a + b;
    };
    while (u < u1) {
        const int yt = (int)(u / nxr);
        const int x0 = maps.xa + (int)(u - (long long)yt * nxr);
        const int x1 = (int)min((long long)maps.xb, x0 + (u1 - u));
        const int y0 = yt * TY;
        const bool seam = (y0 == 0) || (y0 + TY == g.ny);
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TY == g.ny ? 0 : y0 + TY;
        const int nplanes = (x1 - x0) + 2;
        int sissue = 0;
        auto issue_next = [&]() {               // thread 0 only
            const int k = ki;
            double* S = smem + k * SLOT;
            int x = x0 - 1 + sissue;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(bars + k, (unsigned)P::SLOT_BYTES);
            if (!seam) {
                r64_ld_t<NZ>(S + P::T, &maps.t_full, y0 - 1, x, bars + k);
                r64_ld_k<NZ>(S + P::K, &maps.k_full, y0 - 1, x, bars + k);
            } else {
                r64_ld_t<NZ>(S + P::T, &maps.t_halo, ym, x, bars + k);
                r64_ld_t<NZ>(S + P::T + 3 * NZ, &maps.t_main, y0, x, bars + k);
                r64_ld_t<NZ>(S + P::T + (TY + 1) * 3 * NZ, &maps.t_halo, yp, x, bars + k);
                r64_ld_k<NZ>(S + P::K, &maps.k_halo, ym, x, bars + k);
                r64_ld_k<NZ>(S + P::K + NZ, &maps.k_main, y0, x, bars + k);
            }
            ++sissue;
            ki = ki + 1 == STAGES ? 0 : ki + 1;
        };
        auto arrive = [&]() -> const double* {
            const int k = kc;
            mbar_wait(bars + k, (phase_bits >> k) & 1u);
            phase_bits ^= 1u << k;
            __syncthreads();
            if (tid == 0 && sissue < nplanes) issue_next();
            kc = kc + 1 == STAGES ? 0 : kc + 1;
            return smem + k * SLOT;
        };
        if (tid == 0)
            while (sissue < AHEAD && sissue < nplanes) issue_next();
        const unsigned vrow = (unsigned)((y0 + ty) * NZ + tz);
        auto step = [&](int s, const R64PState& I, R64PState& O, bool doN, bool doQ, bool doP) {
            const double* S = arrive();
            weights(S, O.w);
            double q[2][2];
            O.kv4s = I.kv4s;
            if (doQ) {
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) q[jj][kk] = I.w.c[jj][kk] + O.w.c[jj][kk];
                O.kv4s = (I.w.kvh + O.w.kvh) * s48;
            }
            const unsigned vp = (unsigned)(x0 + s - 2) * pl + vrow;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double R[3][3];
                rows(S, c, R);
                if (doN) {
                    const double tot = xsum(I.w, R, I.Sc[c]);
                    const double kt = fma(I.kv4s, I.C0[c], -s12 * tot);
                    const double r = (I.F[c] - fm[c]) - kt;
                    r32[(unsigned)c * n + vp] = (float)r;
                    acc[c] += r * r;
                    acc[3 + c] += I.F[c] * I.F[c];
                    acc[6 + c] += I.C0[c];
                }
                double nc = I.Sn[c];
                if (doQ) {
                    double a = fma(q[0][0], R[0][0], nc);
                    double b = q[0][1] * R[0][2];
                    a = fma(q[1][0], R[2][0], a);
                    b = fma(q[1][1], R[2][2], b);
                    nc = a + b;
                    O.C0[c] = R[1][1];
                    // load: f = sum_a f0[a][c] * kappa of the element whose corner a is v
                    // (element v - c_a: x bit from plane p-1 = I.w, y/z bits pick the corner)
                    double f = 0.0;
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        const R64PW& w = (a & 1) ? I.w : O.w;
                        f = __dadd_rn(f, __dmul_rn(lt.f0[a * 3 + c], w.c[1 - ((a >> 1) & 1)][1 - ((a >> 2) & 1)]));
                    }
                    O.F[c] = f;
                } else {
                    O.C0[c] = I.C0[c];
                    O.F[c] = I.F[c];
                }
                O.Sc[c] = nc;
                O.Sn[c] = doP ? xsum(O.w, R, 0.0) : 0.0;
            }
        };
        R64PState A, B;
        {   // prologue: plane x0-1 only starts out(x0)
            const double* S = arrive();
            weights(S, A.w);
            A.kv4s = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double R[3][3];
                rows(S, c, R);
                A.Sn[c] = xsum(A.w, R, 0.0);
                A.Sc[c] = A.C0[c] = A.F[c] = 0.0;
            }
        }
        step(1, A, B, false, true, nplanes > 3);
        int s = 2;
        for (; s + 1 < nplanes - 2; s += 2) {
            step(s, B, A, true, true, true);
            step(s + 1, A, B, true, true, true);
        }
        if (s < nplanes - 2) {
            step(s, B, A, true, true, true);
            step(s + 1, A, B, true, true, false);
            step(s + 2, B, A, true, false, false);
        } else if (s == nplanes - 2) {
            step(s, B, A, true, true, false);
            step(s + 1, A, B, true, false, false);
        } else {
            step(s, B, A, true, false, false);
        }
        __syncthreads();
        u += x1 - x0;
    }
    reduce_finalize<9>(acc, partials, counter, out9);
}

}  // namespace otm
