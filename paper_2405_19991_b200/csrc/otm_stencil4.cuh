// k4: three load cases per thread, 21-point weights, paired fp32 (FFMA2).
//
// With equal axis scales the element matrix is s K0, K0 = (5 I + N1 - J)/12, so
// per element e with vertex v at corner a the row of v is (4 T_v - sum of the
// three face-diagonal corners - the opposite corner) / 12.  Summed over the 8
// elements around v:
//   (K T)_v = s/12 ( 4 K_v T_v - sum_{12 d, two nonzero} c_d T_{v+d}
//                              - sum_{8 d, three nonzero} k_{e(d)} T_{v+d} )
// with K_v the sum of the 8 factors, c_d the sum of the 2 factors of the elements
// containing v and v+d, k_{e(d)} the factor of the element spanned by v and v+d.
// Face neighbours have weight 0.  The 21 weights depend only on the factors, so a
// thread computes them once and applies them to all three load cases.  A thread
// owns the vertex pair (z, z+1): every weight and operand is a float2 and the
// products run as paired fp32 FMAs (__ffma2_rn, sm_100).
//
// Operands come from the same cp.async shared-memory ring as k3 (otm_stencil3.cuh):
// the operand tiles of the 3 cases (plus D^-1 when the operand is D^-1 f) and the
// factor tile of every x-plane, kAhead4 planes ahead of use.
#pragma once

#include "otm_stencil3.cuh"

namespace otm {

constexpr int kAhead4 = 2;
constexpr int kStages4 = 5;        // reads slots s-2..s while plane s+2 lands: kAhead4 + 3
constexpr int kMaxTasks4 = 4;

template <int NT>   // tiles per slot (operand-related) + 1 factor tile
__host__ __device__ constexpr size_t s4_smem_bytes() { return (size_t)kStages4 * (NT + 1) * kS3Tile * 4; }

struct S4Setup {
    const float* arr[4];   // staged halo tiles: up to 4 arrays (already offset by case)
    int narr;
    const float* kap;
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// copy tasks of one plane for this thread (task ids tid + 256 k): NT halo tiles
// (18 tasks per row, 10 rows) then the factor tile (17 per row, 9 rows)
template <int NT>
__device__ __forceinline__ void s4_tasks(const Geo& g, const S4Setup& su, int y0, int z0,
                                         S3Task (&mine)[kMaxTasks4]) {
    const int tid = threadIdx.x + 32 * threadIdx.y;
    const int zl = z0 == 0 ? g.nz - 1 : z0 - 1;
    const int zr = z0 + 64 == g.nz ? 0 : z0 + 64;
#pragma unroll
    for (int k = 0; k < kMaxTasks4; ++k) {
        const int t = tid + 256 * k;
        mine[k].g = nullptr;
        mine[k].soff = 0;
        mine[k].bytes = 16;
        if (t < NT * 180) {
            const int a = t / 180, u = t - a * 180;
            const int r = u / 18, j = u - r * 18;
            const int y = (y0 - 1 + r + g.ny) % g.ny;
            const float* base = su.arr[a] + (long long)y * g.nz;
            const int srow = a * kS3Tile + r * kS3Pitch;
            if (j < 16) { mine[k].g = base + z0 + 4 * j; mine[k].soff = srow + 4 + 4 * j; }
            else if (j == 16) { mine[k].g = base + zl; mine[k].soff = srow + 3; mine[k].bytes = 4; }
            else { mine[k].g = base + zr; mine[k].soff = srow + 68; mine[k].bytes = 4; }
        } else if (t < NT * 180 + 153) {
            const int u = t - NT * 180;
            const int r = u / 17, j = u - r * 17;
            const int y = (y0 - 1 + r + g.ny) % g.ny;
            const float* base = su.kap + (long long)y * g.nz;
            const int srow = NT * kS3Tile + r * kS3Pitch;
            if (j < 16) { mine[k].g = base + z0 + 4 * j; mine[k].soff = srow + 4 + 4 * j; }
            else { mine[k].g = base + zl; mine[k].soff = srow + 3; mine[k].bytes = 4; }
        }
    }
}

__device__ __forceinline__ void s4_issue(const Geo& g, int x, float* slot, const S3Task (&mine)[kMaxTasks4]) {
    const int xx = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
    const long long po = (long long)xx * g.pl;
#pragma unroll
    for (int k = 0; k < kMaxTasks4; ++k) {
        if (mine[k].g == nullptr) continue;
        if (mine[k].bytes == 16) cp_async16(slot + mine[k].soff, mine[k].g + po);
        else cp_async4(slot + mine[k].soff, mine[k].g + po);
    }
}

// The 21 weights of the vertex pair, from the factor planes Ka (elements x-1) and
// Kb (elements x); Kq[jj][m]: element row y-1+jj, column z-1+m.
struct W21 {
    float2 kv4;          // 4 K_v
    float2 e[12];        // NEGATED edge weights -c_d: (dx,dy) 4 combos with dz=0, (dx,dz) 4 with dy=0, (dy,dz) 4 with dx=0
    float2 k[8];         // NEGATED corner factors, index q | jj<<1 | kk<<2 (element x-1+q, y-1+jj, z-1+kk of vertex z)
};

__device__ __forceinline__ void w21_build(const float (&Ka)[2][3], const float (&Kb)[2][3], W21& w) {
    // factor pairs: element (q, jj, kk) of vertex z is column kk, of vertex z+1 column kk+1
    float2 K[2][2][2];
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            K[0][jj][kk] = f2(-Ka[jj][kk], -Ka[jj][kk + 1]);
            K[1][jj][kk] = f2(-Kb[jj][kk], -Kb[jj][kk + 1]);
        }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) w.k[q | (jj << 1) | (kk << 2)] = K[q][jj][kk];
    // (dx, dy) with dz = 0: elements (q, jj, *) ; q = (dx+1)/2, jj = (dy+1)/2
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) w.e[q * 2 + jj] = fadd2(K[q][jj][0], K[q][jj][1]);
    // (dx, dz) with dy = 0: elements (q, *, kk)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) w.e[4 + q * 2 + kk] = fadd2(K[q][0][kk], K[q][1][kk]);
    // (dy, dz) with dx = 0: elements (*, jj, kk)
#pragma unroll
    for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) w.e[8 + jj * 2 + kk] = fadd2(K[0][jj][kk], K[1][jj][kk]);
    const float2 nkv = fadd2(fadd2(w.e[0], w.e[1]), fadd2(w.e[2], w.e[3]));   // -K_v
    w.kv4 = fmul2(nkv, f2(-4.f, -4.f));
}

// Op contract (k4):
//   static constexpr int NT;                                   staged operand tiles
//   float  op1(const float* slot, int c, int r, int col) const  operand of case c at smem (r, col)
//   float2 op2(const float* slot, int c, int r, int col) const  operand at (r, col), (r, col+1)
//   void prefetch(int x, long long vrow)                        pointwise inputs of output plane x
//   void sink(const float* S0, int c, long long v, int r, int col, float2 kt, float2 ctr)
//                                                                result of case c at vertices v, v+1
template <class Op>
__device__ __forceinline__ void march4_segment(const Geo& g, const LevelTemplate& lt, const S4Setup& su, Op& op,
                                               int y0, int z0, int x0, int x1) {
    extern __shared__ float4 s4_smem4[];
    float* smem = reinterpret_cast<float*>(s4_smem4);
    constexpr int NT = Op::NT;
    constexpr int SLOT = (NT + 1) * kS3Tile;
    S3Task mine[kMaxTasks4];
    s4_tasks<NT>(g, su, y0, z0, mine);
    const int nplanes = (x1 - x0) + 2;          // operand / factor planes x0-1 .. x1
#pragma unroll
    for (int s = 0; s < kAhead4; ++s) {
        if (s < nplanes) s4_issue(g, x0 - 1 + s, smem + s * SLOT, mine);
        cp_commit();
    }
    const int tr = threadIdx.y + 1;
    const int col = 4 + 2 * threadIdx.x;
    const float2 s12 = f2((float)lt.s12, (float)lt.s12);
    const long long vrow = (long long)(y0 + threadIdx.y) * g.nz + z0 + 2 * threadIdx.x;
    op.prefetch(x0, vrow);
    for (int s = 0; s < nplanes; ++s) {
        cp_wait<kAhead4 - 1>();
        __syncthreads();
        if (s + kAhead4 < nplanes) s4_issue(g, x0 - 1 + s + kAhead4, smem + ((s + kAhead4) % kStages4) * SLOT, mine);
        cp_commit();
        if (s < 2) continue;
        // output plane x = x0 + s - 2 from operand planes x-1, x, x+1 (slots s-2, s-1, s)
        const float* Sm = smem + ((s - 2) % kStages4) * SLOT;
        const float* S0 = smem + ((s - 1) % kStages4) * SLOT;
        const float* Sp = smem + (s % kStages4) * SLOT;
        const int x = x0 + s - 2;
        W21 w;
        {
            float Ka[2][3], Kb[2][3];
            const float* ka = Sm + NT * kS3Tile;
            const float* kb = S0 + NT * kS3Tile;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int o = (tr - 1 + jj) * kS3Pitch + col;
                Ka[jj][0] = ka[o - 1];
                const float2 va = *reinterpret_cast<const float2*>(ka + o);
                Ka[jj][1] = va.x; Ka[jj][2] = va.y;
                Kb[jj][0] = kb[o - 1];
                const float2 vb = *reinterpret_cast<const float2*>(kb + o);
                Kb[jj][1] = vb.x; Kb[jj][2] = vb.y;
            }
            w21_build(Ka, Kb, w);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // operand pairs T(d) for the vertex pair, by plane P in {m, 0, p}, row j, dz
            auto row = [&](const float* S, int j, float2& L, float2& C, float2& R) {
                const float a0 = op.op1(S, c, tr + j, col - 1);
                const float2 m = op.op2(S, c, tr + j, col);
                const float a3 = op.op1(S, c, tr + j, col + 2);
                L = f2(a0, m.x);
                C = m;
                R = f2(m.y, a3);
            };
            float2 acc;
            float2 L0, C0, R0;
            // plane x (center plane): center and the 4 (dy, dz) edges
            row(S0, 0, L0, C0, R0);
            acc = fmul2(w.kv4, C0);
            {
                float2 l, cc, r;
                row(S0, -1, l, cc, r);   // dy = -1: (dy,dz) = (-1,-1) -> e[8], (-1,+1) -> e[9]
                acc = ffma2(w.e[8], l, acc);
                acc = ffma2(w.e[9], r, acc);
                row(S0, +1, l, cc, r);   // dy = +1: e[10], e[11]
                acc = ffma2(w.e[10], l, acc);
                acc = ffma2(w.e[11], r, acc);
            }
            // planes x-1 (q = 0) and x+1 (q = 1)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const float* S = q == 0 ? Sm : Sp;
                float2 l, cc, r;
                // row y (dy = 0): (dx, dz) edges e[4 + q*2 + kk]: dz = -1 -> kk = 0 (l), dz = +1 -> kk = 1 (r)
                row(S, 0, l, cc, r);
                acc = ffma2(w.e[4 + q * 2], l, acc);
                acc = ffma2(w.e[5 + q * 2], r, acc);
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    row(S, jj == 0 ? -1 : 1, l, cc, r);
                    // (dx, dy) edge e[q*2 + jj] at dz = 0 (center column)
                    acc = ffma2(w.e[q * 2 + jj], cc, acc);
                    // corners k[q | jj<<1 | kk<<2]: dz = -1 (l), dz = +1 (r)
                    acc = ffma2(w.k[q | (jj << 1)], l, acc);
                    acc = ffma2(w.k[q | (jj << 1) | 4], r, acc);
                }
            }
            op.sink(S0, c, vrow + (long long)x * g.pl, tr, col, fmul2(s12, acc), C0);
        }
        if (s + 1 < nplanes && x + 1 < x1) op.prefetch(x + 1, vrow);
    }
    cp_wait<0>();
    __syncthreads();
}

// persistent schedule over (tile column, x plane) units, all three cases per unit
template <class Op>
__device__ __forceinline__ void march4(const Geo& g, const LevelTemplate& lt, const S4Setup& su, Op& op) {
    const int tz = g.nz / kTileZ, ty = g.ny / kTileY;
    const long long cols = (long long)tz * ty;
    const long long W = cols * g.nx;
    const long long B = gridDim.x;
    long long u = W * blockIdx.x / B;
    const long long u1 = W * (blockIdx.x + 1) / B;
    while (u < u1) {
        const long long cl = u / g.nx;
        const int x0 = (int)(u - cl * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int y0 = (int)(cl / tz) * kTileY, z0 = (int)(cl - (cl / tz) * tz) * kTileZ;
        march4_segment(g, lt, su, op, y0, z0, x0, x1);
        u += x1 - x0;
    }
}

}  // namespace otm

namespace otm {

// ---------------------------------------------------------------------------
// k5: one load case per thread (the k3 ring and register window: only the newly
// arrived plane is read from shared memory) with the 21-weight paired-fp32
// arithmetic of k4.  Window: operand planes x-1, x, x+1 (3 rows x 4 columns each)
// and factor planes x-1, x in registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 apply21(const W21& w, const float (&Pm)[3][4], const float (&P0)[3][4],
                                          const float (&Pp)[3][4]) {
    auto L = [](const float (&P)[3][4], int j) { return f2(P[j][0], P[j][1]); };
    auto C = [](const float (&P)[3][4], int j) { return f2(P[j][1], P[j][2]); };
    auto R = [](const float (&P)[3][4], int j) { return f2(P[j][2], P[j][3]); };
    float2 acc = fmul2(w.kv4, C(P0, 1));
    float2 acc2 = ffma2(w.e[8], L(P0, 0), f2(0.f, 0.f));
    acc = ffma2(w.e[9], R(P0, 0), acc);
    acc2 = ffma2(w.e[10], L(P0, 2), acc2);
    acc = ffma2(w.e[11], R(P0, 2), acc);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const float (&P)[3][4] = q == 0 ? Pm : Pp;
        acc2 = ffma2(w.e[4 + q * 2], L(P, 1), acc2);
        acc = ffma2(w.e[5 + q * 2], R(P, 1), acc);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = jj == 0 ? 0 : 2;
            acc2 = ffma2(w.e[q * 2 + jj], C(P, j), acc2);
            acc = ffma2(w.k[q | (jj << 1)], L(P, j), acc);
            acc2 = ffma2(w.k[q | (jj << 1) | 4], R(P, j), acc2);
        }
    }
    return fadd2(acc, acc2);
}

template <int NARR, class Op>
__device__ __forceinline__ void march5_segment(const Geo& g, const LevelTemplate& lt, const S3Setup<NARR>& su,
                                               Op& op, int c, int y0, int z0, int x0, int x1) {
    extern __shared__ float4 s3_smem4[];
    float* smem = reinterpret_cast<float*>(s3_smem4);
    constexpr int SLOT = s3_slot_floats<NARR>();
    S3Task mine[kMaxTasks];
    s3_tasks<NARR>(g, su, c, y0, z0, mine);
    const int nplanes = (x1 - x0) + 2;
#pragma unroll
    for (int s = 0; s < kAhead; ++s) {
        if (s < nplanes) s3_issue<NARR>(g, su, c, x0 - 1 + s, smem + s * SLOT, mine);
        cp_commit();
    }
    const int tr = threadIdx.y + 1;
    const int col = 4 + 2 * threadIdx.x;
    const long long vrow = (long long)(y0 + threadIdx.y) * g.nz + z0 + 2 * threadIdx.x;
    const float2 s12 = f2((float)lt.s12, (float)lt.s12);
    float Pm[3][4], P0[3][4], Pp[3][4], Ka[2][3], Kb[2][3];
    auto readT = [&](const float* slot, float (&P)[3][4]) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            P[j][0] = op.operand(slot, tr - 1 + j, col - 1);
            const float2 m = op.operand2(slot, tr - 1 + j, col);
            P[j][1] = m.x;
            P[j][2] = m.y;
            P[j][3] = op.operand(slot, tr - 1 + j, col + 2);
        }
    };
    auto readK = [&](const float* slot, float (&K)[2][3]) {
        const float* kt = slot + NARR * kS3Tile;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int o = (tr - 1 + jj) * kS3Pitch + col;
            K[jj][0] = kt[o - 1];
            const float2 v = *reinterpret_cast<const float2*>(kt + o);
            K[jj][1] = v.x;
            K[jj][2] = v.y;
        }
    };
    auto advance = [&](int s) {
        cp_wait<kAhead - 1>();
        __syncthreads();
        if (s + kAhead < nplanes)
            s3_issue<NARR>(g, su, c, x0 - 1 + s + kAhead, smem + ((s + kAhead) % kStages) * SLOT, mine);
        cp_commit();
    };
    advance(0);
    readT(smem, Pm);
    readK(smem, Ka);
    advance(1);
    readT(smem + SLOT, P0);
    for (int s = 2; s < nplanes; ++s) {
        advance(s);
        const float* slot = smem + (s % kStages) * SLOT;
        const float* xslot = smem + ((s - 1) % kStages) * SLOT;
        readT(slot, Pp);
        readK(xslot, Kb);
        W21 w;
        w21_build(Ka, Kb, w);
        const float2 kt = fmul2(s12, apply21(w, Pm, P0, Pp));
        const int x = x0 + s - 2;
        const float kt2[2] = {kt.x, kt.y};
        const float ctr[2] = {P0[1][1], P0[1][2]};
        op.sink(xslot, c, vrow + (long long)x * g.pl, tr, col, kt2, ctr);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m) { Pm[j][m] = P0[j][m]; P0[j][m] = Pp[j][m]; }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 3; ++m) Ka[jj][m] = Kb[jj][m];
    }
    cp_wait<0>();
    __syncthreads();
}

template <int NARR, class Op>
__device__ __forceinline__ void march5(const Geo& g, const LevelTemplate& lt, const S3Setup<NARR>& su, Op& op,
                                       int& last_case) {
    const int tz = g.nz / kTileZ, ty = g.ny / kTileY;
    const long long cols = 3LL * tz * ty;
    const long long W = cols * g.nx;
    const long long B = gridDim.x;
    long long u = W * blockIdx.x / B;
    const long long u1 = W * (blockIdx.x + 1) / B;
    last_case = -1;
    while (u < u1) {
        const long long col = u / g.nx;
        const int x0 = (int)(u - col * g.nx);
        const int x1 = (int)min((long long)g.nx, x0 + (u1 - u));
        const int c = (int)(col / ((long long)tz * ty));
        const int rest = (int)(col - (long long)c * tz * ty);
        const int y0 = (rest / tz) * kTileY, z0 = (rest - (rest / tz) * tz) * kTileZ;
        op.begin_case(c, last_case);
        march5_segment<NARR>(g, lt, su, op, c, y0, z0, x0, x1);
        last_case = c;
        u += x1 - x0;
    }
}

}  // namespace otm
