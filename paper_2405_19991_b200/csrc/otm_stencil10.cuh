// k10: level stencils as a "push" x-march.  Same TMA + mbarrier plane ring as
// k8, but each landed x plane is consumed ONCE and pushed into the three output
// planes it touches, so no operand window is kept in registers:
//
//   out(x) = 4 K_v T(x) - [ X(kappa plane x-1; plane x-1) + Q(x) + X(kappa plane x; plane x+1) ]
//
// X(k; P) is the 8-term contribution of one neighbour plane through one element
// plane (4 corners + 2 y-edges + 2 z-edges, the face neighbour has weight 0 in the
// 21-point form), Q(x) the 4 in-plane (dy, dz) edges.  When plane s lands:
//   out(s-1) += X(kappa s-1; s)   -> finished, written
//   out(s)   += Q(s)  (edges kappa s-1 + kappa s)
//   out(s+1)  = X(kappa s; s)      (started)
// Live state per thread: two partial sums and one centre value per case plus the
// x-weights of the previous element plane (~40 floats instead of k8's 108-float
// window), so two 256-thread CTAs fit per SM and each hides the other's
// per-plane barrier.
//
// Shared-memory slot of one x plane, [row][case][z] so ONE 4-D TMA box moves the
// three load cases of a tile (interior tiles: one box of TY+2 rows; tiles at the
// periodic y seam: main box + two wrapped one-row boxes):
//   OP  (TY+2) x 3 x NZ   operand array (3 cases, y halo)
//   D   (TY+2) x NZ       D^-1 with halo            (smooth_res: operand = w D^-1 f)
//   K   (TY+1) x NZ       element factors, rows y0-1 .. y0+TY-1
//   F   TY x 3 x NZ       right-hand side, centre rows (jacobi)
//   DC  TY x NZ           D^-1, centre rows          (jacobi)
#pragma once

#include "otm_tma.cuh"

namespace otm {

struct K10Maps {
    CUtensorMap op_full, op_main, op_halo;   // 4-D (z, case, y, x): TY+2 / TY / 1 rows
    CUtensorMap d_full, d_main, d_halo;      // 3-D (z, y, x) D^-1: TY+2 / TY / 1 rows
    CUtensorMap f_main;                      // 4-D right-hand side, centre rows (jacobi)
    CUtensorMap k_full, k_main, k_halo;      // 3-D factors: TY+1 / TY / 1 rows
    int lock;                                // > 0: CTA b owns row tile b % nty, x chunk b / nty of `lock`
                                             // chunks (row-tile neighbours march the same planes at the
                                             // same time, so y-halo rows hit L2); 0: contiguous ranges
    int xa, xb;                              // output x planes [xa, xb): [0, nx) periodic, or a slab's
                                             // interior [1, nxl + 1) between its ghost planes
};

enum { K10_SMOOTH = 0, K10_JACOBI = 1, K10_SPMV = 2 };

template <int MODE, int NZ, int TY, int CPS = 2>
struct K10Geo {
    static constexpr bool HAS_D = MODE == K10_SMOOTH;
    static constexpr bool HAS_C = MODE == K10_JACOBI;
    static constexpr int OP = 0;
    static constexpr int D = OP + (TY + 2) * 3 * NZ;
    static constexpr int K = D + (HAS_D ? (TY + 2) * NZ : 0);
    static constexpr int F = K + (TY + 1) * NZ;
    static constexpr int DC = F + (HAS_C ? TY * 3 * NZ : 0);
    static constexpr int SLOT = DC + (HAS_C ? TY * NZ : 0);          // floats
    static constexpr int SLOT_BYTES = SLOT * 4;
    static constexpr int BUDGET = (224 * 1024) / CPS - 2048;          // CPS CTAs per SM
    static constexpr int STAGES0 = BUDGET / (SLOT_BYTES + 8);
    static constexpr int STAGES = STAGES0 > 10 ? 10 : STAGES0;
    static constexpr int AHEAD = STAGES - 2;                          // slot refilled at step s held plane s-2
    static constexpr size_t SMEM = (size_t)STAGES * SLOT_BYTES + STAGES * 8;
    static_assert(STAGES >= 3, "k10 ring too shallow");
};

__device__ __forceinline__ void tma_load_4d(float* dst, const CUtensorMap* map, int z, int c, int y, int x,
                                            uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
        ::"r"(d), "l"(map), "r"(z), "r"(c), "r"(y), "r"(x), "r"(b)
        : "memory");
}

__device__ __forceinline__ void tma_load_5d(float* dst, const CUtensorMap* map, int z, int h, int c, int y, int x,
                                            uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
        ::"r"(d), "l"(map), "r"(z), "r"(h), "r"(c), "r"(y), "r"(x), "r"(b)
        : "memory");
}

// Row loads of the march.  A TMA box dimension holds at most 256 elements, so for
// NZ > 256 the host splits z into (256, NZ / 256) map dimensions (strides 1 and 256
// elements): the box still lands as [row][case][NZ] contiguous, the same layout.
template <int NZ>
__device__ __forceinline__ void k10_ld_c3(float* dst, const CUtensorMap* map, int y, int x, uint64_t* bar) {
    if constexpr (NZ > 256) tma_load_5d(dst, map, 0, 0, 0, y, x, bar);
    else tma_load_4d(dst, map, 0, 0, y, x, bar);
}
template <int NZ>
__device__ __forceinline__ void k10_ld_1(float* dst, const CUtensorMap* map, int y, int x, uint64_t* bar) {
    if constexpr (NZ > 256) tma_load_4d(dst, map, 0, 0, y, x, bar);
    else tma_load_3d(dst, map, 0, y, x, bar);
}

// Thread mapping: thread tx of a row owns the vertex pair (z, z + H), H = NZ/2,
// so every paired-fp32 (FFMA2) operand -- the pair's left, centre and right
// neighbours -- is two independent 32-bit shared-memory loads straight into the
// two halves of a register pair (no repacking MOVs, conflict-free rows).  Only
// z - 1 of lane 0 and z + H + 1 of the last thread wrap around the periodic seam.
struct K10Cols {
    int tx;                // z
    int zm;                // z - 1 (periodic)
    int zp2;               // z + H + 1 (periodic)
};

// one staged row around the pair: L = (z-1, z+H-1), C = (z, z+H), R = (z+1, z+H+1)
struct K10Row {
    float2 L, C, R;
};

template <int NZ>
__device__ __forceinline__ K10Row k10_row(const float* b, const K10Cols& q) {
    constexpr int H = NZ / 2;
    K10Row r;
    r.L.x = b[q.zm];
    r.L.y = b[q.tx + H - 1];
    r.C.x = b[q.tx];
    r.C.y = b[q.tx + H];
    r.R.x = b[q.tx + 1];
    r.R.y = b[q.zp2];
    return r;
}

// x-weights of one element plane for the pair: corners c[jj][kk] (element
// (., y-1+jj, z-1+kk), column z+H-1+kk for the second vertex), y-edges
// ey[jj] = c[jj][0] + c[jj][1], z-edges ez[kk] = c[0][kk] + c[1][kk], kvh = sum
// of the four factors.  The factor row pattern is the operand row's L and C.
struct K10W {
    float2 c[2][2];
    float2 ey[2], ez[2];
    float2 kvh;
};

template <int NZ>
__device__ __forceinline__ void k10_weights(const float* K, int ty, const K10Cols& q, K10W& w) {
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
        const K10Row r = k10_row<NZ>(K + (ty + jj) * NZ, q);
        w.c[jj][0] = r.L;
        w.c[jj][1] = r.C;
    }
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) w.ey[jj] = fadd2(w.c[jj][0], w.c[jj][1]);
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) w.ez[kk] = fadd2(w.c[0][kk], w.c[1][kk]);
    w.kvh = fadd2(w.ey[0], w.ey[1]);
}

// X(w; rows R0 = y-1, R1 = y, R2 = y+1 of one neighbour plane) added to a
__device__ __forceinline__ float2 k10_x(const K10W& w, const K10Row (&R)[3], float2 a) {
    float2 b = fmul2(w.ey[0], R[0].C);
    a = ffma2(w.c[0][0], R[0].L, a);
    b = ffma2(w.c[0][1], R[0].R, b);
    a = ffma2(w.c[1][0], R[2].L, a);
    b = ffma2(w.c[1][1], R[2].R, b);
    a = ffma2(w.ey[1], R[2].C, a);
    b = ffma2(w.ez[0], R[1].L, b);
    a = ffma2(w.ez[1], R[1].R, a);
    return fadd2(a, b);
}

template <int MODE_, int NZ_, int TY_, bool DOT = true, int CPS = 2, bool WZ = true>
struct K10Op {
    static constexpr int MODE = MODE_, NZ = NZ_, TY = TY_, H = NZ_ / 2;
    using G = K10Geo<MODE, NZ, TY, CPS>;
    float omega;
    float* out0;          // smooth_res: z0 ; jacobi: z_out ; spmv: q
    float* out1;          // smooth_res: res
    long long n;
    double acc[3];
    K10Row dw[3];         // smooth_res: omega D^-1 around the pair, rows y-1, y, y+1 (per plane)

    __device__ __forceinline__ void plane(const float* S, int ty, const K10Cols& q) {
        if (MODE == K10_SMOOTH) {
            const float2 om = f2(omega, omega);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const K10Row d = k10_row<NZ>(S + G::D + (ty + j) * NZ, q);
                dw[j].L = fmul2(om, d.L);
                dw[j].C = fmul2(om, d.C);
                dw[j].R = fmul2(om, d.R);
            }
        }
    }
    // rows y-1, y, y+1 of case c's operand from a landed slot
    __device__ __forceinline__ void rows(const float* S, int c, int ty, const K10Cols& q, K10Row (&R)[3]) const {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            R[j] = k10_row<NZ>(S + G::OP + ((ty + j) * 3 + c) * NZ, q);
            if (MODE == K10_SMOOTH) {                     // operand = omega D^-1 f
                R[j].L = fmul2(R[j].L, dw[j].L);
                R[j].C = fmul2(R[j].C, dw[j].C);
                R[j].R = fmul2(R[j].R, dw[j].R);
            }
        }
    }
    __device__ __forceinline__ float2 pair(const float* b, int tx) const { return f2(b[tx], b[tx + H]); }
    __device__ __forceinline__ void put(float* o, float2 v) const {
        o[0] = v.x;
        o[H] = v.y;
    }
    // finished (K p) of case c at the pair, ctr = operand at the pair; Sp = slot of that plane
    __device__ __forceinline__ void sink(const float* Sp, int c, int v, int ty, int tx, float2 kt, float2 ctr) {
        if (MODE == K10_SPMV) {
            put(out0 + c * n + v, kt);
            if (DOT) acc[c] += (double)ctr.x * (double)kt.x + (double)ctr.y * (double)kt.y;
        } else if (MODE == K10_SMOOTH) {
            const float2 f = pair(Sp + G::OP + ((ty + 1) * 3 + c) * NZ, tx);
            if (WZ) put(out0 + c * n + v, ctr);
            put(out1 + c * n + v, f2(f.x - kt.x, f.y - kt.y));
        } else {
            const float2 f = pair(Sp + G::F + (ty * 3 + c) * NZ, tx);
            const float2 d = pair(Sp + G::DC + ty * NZ, tx);
            const float z0 = ctr.x + omega * d.x * (f.x - kt.x);
            const float z1 = ctr.y + omega * d.y * (f.y - kt.y);
            put(out0 + c * n + v, f2(z0, z1));
            if (DOT) acc[c] += (double)f.x * (double)z0 + (double)f.y * (double)z1;
        }
    }
};

// Rotating per-thread state of the march: partial sums of out(p) and out(p+1),
// the centre operand and 4 s12 K_v of out(p), the x-weights of element plane p-1.
// Two instances alternate roles every plane (A -> B -> A), so the hot loop has no
// register copies.
struct K10State {
    float2 Sc[3], Sn[3], C0[3];
    float2 kv4s;
    K10W w;
};

template <class Op>
__device__ __forceinline__ void march10(const Geo& g, float s12f, const K10Maps& maps, Op& op) {
    constexpr int NZ = Op::NZ, TY = Op::TY;
    using G = typename Op::G;
    constexpr int STAGES = G::STAGES, AHEAD = G::AHEAD, SLOT = G::SLOT;
    extern __shared__ __align__(128) float4 k10_smem4[];
    float* smem = reinterpret_cast<float*>(k10_smem4);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * SLOT);
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    if (tid == 0) {
        for (int k = 0; k < STAGES; ++k) mbar_init(bars + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    pdl_wait();
    unsigned phase_bits = 0;
    K10Cols cols;
    cols.tx = threadIdx.x;
    cols.zm = cols.tx == 0 ? NZ - 1 : cols.tx - 1;
    cols.zp2 = cols.tx + NZ / 2 + 1 == NZ ? 0 : cols.tx + NZ / 2 + 1;
    const int ty = threadIdx.y;
    const float2 ns12 = f2(-s12f, -s12f);
    const float2 s48 = f2(4.f * s12f, 4.f * s12f);
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
    int kc = 0;                                  // ring slot of the next plane to land
    int ki = 0;                                  // ring slot of the next plane to issue
    while (u < u1) {
        const int yt = (int)(u / nxr);
        const int x0 = maps.xa + (int)(u - (long long)yt * nxr);
        const int x1 = (int)min((long long)maps.xb, x0 + (u1 - u));
        const int y0 = yt * TY;
        const bool seam = (y0 == 0) || (y0 + TY == g.ny);
        const int ym = y0 == 0 ? g.ny - 1 : y0 - 1;
        const int yp = y0 + TY == g.ny ? 0 : y0 + TY;
        const int nplanes = (x1 - x0) + 2;
        int sissue = 0;                          // next segment plane to issue
        auto issue_next = [&]() {                // thread 0 only
            const int k = ki;
            float* S = smem + k * SLOT;
            int x = x0 - 1 + sissue;
            x = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx(bars + k, (unsigned)G::SLOT_BYTES);
            if (!seam) {
                k10_ld_c3<NZ>(S + G::OP, &maps.op_full, y0 - 1, x, bars + k);
                if (G::HAS_D) k10_ld_1<NZ>(S + G::D, &maps.d_full, y0 - 1, x, bars + k);
                k10_ld_1<NZ>(S + G::K, &maps.k_full, y0 - 1, x, bars + k);
            } else {
                k10_ld_c3<NZ>(S + G::OP, &maps.op_halo, ym, x, bars + k);
                k10_ld_c3<NZ>(S + G::OP + 3 * NZ, &maps.op_main, y0, x, bars + k);
                k10_ld_c3<NZ>(S + G::OP + (TY + 1) * 3 * NZ, &maps.op_halo, yp, x, bars + k);
                if (G::HAS_D) {
                    k10_ld_1<NZ>(S + G::D, &maps.d_halo, ym, x, bars + k);
                    k10_ld_1<NZ>(S + G::D + NZ, &maps.d_main, y0, x, bars + k);
                    k10_ld_1<NZ>(S + G::D + (TY + 1) * NZ, &maps.d_halo, yp, x, bars + k);
                }
                k10_ld_1<NZ>(S + G::K, &maps.k_halo, ym, x, bars + k);
                k10_ld_1<NZ>(S + G::K + NZ, &maps.k_main, y0, x, bars + k);
            }
            if (G::HAS_C) {
                k10_ld_c3<NZ>(S + G::F, &maps.f_main, y0, x, bars + k);
                k10_ld_1<NZ>(S + G::DC, &maps.d_main, y0, x, bars + k);
            }
            ++sissue;
            ki = ki + 1 == STAGES ? 0 : ki + 1;
        };
        // wait for the next plane, retire the previous step everywhere, refill the
        // slot of plane s-2; returns the landed slot, *prev = the slot before it
        const float* Sprev = nullptr;
        auto arrive = [&]() -> const float* {
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
        // output offsets of the thread's pair (32-bit: fields < 2^31 floats)
        const int vrow = (y0 + ty) * NZ + cols.tx;
        // one landed plane (segment step s, plane x0-1+s) moving state I -> O
        auto step = [&](int s, const K10State& I, K10State& O, bool doN, bool doQ, bool doP) {
            const float* S = arrive();
            k10_weights<NZ>(S + G::K, ty, cols, O.w);
            op.plane(S, ty, cols);
            float2 q[2][2];
            O.kv4s = I.kv4s;
            if (doQ) {
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) q[jj][kk] = fadd2(I.w.c[jj][kk], O.w.c[jj][kk]);
                O.kv4s = fmul2(fadd2(I.w.kvh, O.w.kvh), s48);
            }
            const int vp = vrow + (x0 + s - 2) * g.pl;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                K10Row R[3];
                op.rows(S, c, ty, cols, R);
                if (doN) {
                    const float2 tot = k10_x(I.w, R, I.Sc[c]);
                    op.sink(Sprev, c, vp, ty, cols.tx, ffma2(I.kv4s, I.C0[c], fmul2(ns12, tot)), I.C0[c]);
                }
                float2 nc = I.Sn[c];
                if (doQ) {
                    float2 a = ffma2(q[0][0], R[0].L, nc);
                    float2 b = fmul2(q[0][1], R[0].R);
                    a = ffma2(q[1][0], R[2].L, a);
                    b = ffma2(q[1][1], R[2].R, b);
                    nc = fadd2(a, b);
                    O.C0[c] = R[1].C;
                } else {
                    O.C0[c] = I.C0[c];
                }
                O.Sc[c] = nc;
                O.Sn[c] = doP ? k10_x(O.w, R, f2(0.f, 0.f)) : f2(0.f, 0.f);
            }
            Sprev = S;
        };
        K10State A, B;
        // prologue: plane x0-1 only starts out(x0)
        {
            const float* S = arrive();
            k10_weights<NZ>(S + G::K, ty, cols, A.w);
            op.plane(S, ty, cols);
            A.kv4s = f2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                K10Row R[3];
                op.rows(S, c, ty, cols, R);
                A.Sn[c] = k10_x(A.w, R, f2(0.f, 0.f));
                A.Sc[c] = f2(0.f, 0.f);
                A.C0[c] = f2(0.f, 0.f);
            }
            Sprev = S;
        }
        // step 1: out(x0) gets its centre plane
        step(1, A, B, false, true, nplanes > 3);
        // steady state, two planes per trip: finish out(p-1), centre of out(p), start out(p+1)
        int s = 2;
        for (; s + 1 < nplanes - 2; s += 2) {
            step(s, B, A, true, true, true);
            step(s + 1, A, B, true, true, true);
        }
        // tail: at most one more steady plane, then plane nplanes-2 (no start) and the last plane
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
}

}  // namespace otm
