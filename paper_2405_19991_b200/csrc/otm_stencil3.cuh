// Shared-memory-ring stencil engine for the fp32 level stencils (fast path).
//
// Block = 256 threads = 32 (z pairs) x 8 (rows) -> a 64 x 8 (z, y) output tile of
// ONE load case; the block walks an x chunk.  Every x-plane of every staged array
// is copied global -> shared with cp.async (16-byte chunks for the 64-wide tile
// rows, 4-byte copies for the periodic halo columns) into a ring of kStages
// slots, kAhead planes before the arithmetic needs it, so many planes of loads
// are in flight per SM without spending registers on them.  The copy work of a
// plane is a fixed list of <= kMaxTasks descriptors per thread computed once.
//
// Arithmetic: the separable form of otm_stencil2.cuh (equal axis scales), fed
// from shared memory; only the newly arrived plane is read each step.
#pragma once

#include <cuda_pipeline_primitives.h>

#include "otm_common.cuh"
#include "otm_internal.h"
#include "otm_stencil2.cuh"

namespace otm {

constexpr int kS3Rows = 10;       // tile rows y0-1 .. y0+8
constexpr int kS3Pitch = 72;      // floats per smem row: [3] = z0-1, [4..67] = z0..z0+63, [68] = z0+64
constexpr int kS3Tile = kS3Rows * kS3Pitch;
constexpr int kStages = 5;        // ring slots (kAhead + 2: the plane in use and its predecessor)
constexpr int kAhead = 3;         // planes in flight ahead of the plane being consumed
constexpr int kMaxTasks = 3;

// staged array kinds
enum S3Kind { S3Halo = 0, S3Center = 1 };

struct S3Array {
    const float* p;   // base pointer (case offset applied in-kernel when per_case)
    int per_case;     // 1: field[c*n + v]; 0: shared by all cases (D^-1)
    int kind;         // S3Halo (rows y0-1..y0+8, cols z0-1..z0+64) or S3Center (rows y0..y0+7, cols z0..z0+63)
};

template <int NARR>
struct S3Setup {
    S3Array arr[NARR];
    const float* kap;
};

// smem layout per slot: NARR tiles then the factor tile (rows y0-1..y0+7 in tile rows 0..8)
template <int NARR>
__host__ __device__ constexpr int s3_slot_floats() { return (NARR + 1) * kS3Tile; }

template <int NARR>
__host__ __device__ constexpr size_t s3_smem_bytes() { return (size_t)kStages * s3_slot_floats<NARR>() * 4; }

struct S3Task {
    const float* g;   // source at plane 0 (case offset and in-plane offset applied); null = none
    int soff;         // float offset inside the slot
    int bytes;        // 16 or 4
};

__device__ __forceinline__ void cp_async16(float* s, const float* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_async4(float* s, const float* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// This thread's copy tasks of one plane: task ids tid, tid+256, tid+512 of the
// plane's task list [array 0 tasks | array 1 tasks | ... | factor tasks], decoded
// arithmetically (halo array row: 16 chunks + left + right halo; centre array
// row: 16 chunks; factor row: 16 chunks + left halo).
template <int NARR>
__device__ __forceinline__ void s3_tasks(const Geo& g, const S3Setup<NARR>& su, int c, int y0, int z0,
                                         S3Task (&mine)[kMaxTasks]) {
    const int tid = threadIdx.x + 32 * threadIdx.y;
    const int zl = z0 == 0 ? g.nz - 1 : z0 - 1;
    const int zr = z0 + 64 == g.nz ? 0 : z0 + 64;
#pragma unroll
    for (int k = 0; k < kMaxTasks; ++k) {
        int t = tid + 256 * k;
        mine[k].g = nullptr;
        mine[k].soff = 0;
        mine[k].bytes = 16;
        bool done = false;
#pragma unroll
        for (int a = 0; a < NARR; ++a) {
            if (done) break;
            const bool halo = su.arr[a].kind == S3Halo;
            const int per_row = halo ? 18 : 16, nrows = halo ? kS3Rows : kS3Rows - 2;
            const int cnt = per_row * nrows;
            if (t < cnt) {
                const int r = t / per_row + (halo ? 0 : 1), j = t - (t / per_row) * per_row;
                const int y = (y0 - 1 + r + g.ny) % g.ny;
                const float* base = su.arr[a].p + (su.arr[a].per_case ? (long long)c * g.n : 0LL) + (long long)y * g.nz;
                const int srow = a * kS3Tile + r * kS3Pitch;
                if (j < 16) { mine[k].g = base + z0 + 4 * j; mine[k].soff = srow + 4 + 4 * j; }
                else if (j == 16) { mine[k].g = base + zl; mine[k].soff = srow + 3; mine[k].bytes = 4; }
                else { mine[k].g = base + zr; mine[k].soff = srow + 68; mine[k].bytes = 4; }
                done = true;
            } else {
                t -= cnt;
            }
        }
        if (!done && t < 17 * (kS3Rows - 1)) {
            const int r = t / 17, j = t - (t / 17) * 17;
            const int y = (y0 - 1 + r + g.ny) % g.ny;
            const float* base = su.kap + (long long)y * g.nz;
            const int srow = NARR * kS3Tile + r * kS3Pitch;
            if (j < 16) { mine[k].g = base + z0 + 4 * j; mine[k].soff = srow + 4 + 4 * j; }
            else { mine[k].g = base + zl; mine[k].soff = srow + 3; mine[k].bytes = 4; }
        }
    }
}

template <int NARR>
__device__ __forceinline__ void s3_issue(const Geo& g, const S3Setup<NARR>& su, int c, int x, float* slot,
                                         const S3Task (&mine)[kMaxTasks]) {
    const int xx = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
    const long long po = (long long)xx * g.pl;
#pragma unroll
    for (int k = 0; k < kMaxTasks; ++k) {
        const S3Task& tk = mine[k];
        if (tk.g == nullptr) continue;
        if (tk.bytes == 16) cp_async16(slot + tk.soff, tk.g + po);
        else cp_async4(slot + tk.soff, tk.g + po);
    }
}

// Op contract (fp32):
//   float operand(const float* slot, int r, int col) const  -> operand at tile row r, smem column col
//   void sink(const float* slot, int c, long long v, int r, int col, const float (&kt)[2], const float (&ctr)[2])
//     slot = ring slot of the output plane x (for center-only arrays), r = tile row of the thread (1..8),
//     col = smem column of vertex z (z+1 is col+1)
template <int NARR, class Op>
__device__ __forceinline__ void march3_segment(const Geo& g, const LevelTemplate& lt, const S3Setup<NARR>& su,
                                               Op& op, int c, int y0, int z0, int x0, int x1) {
    extern __shared__ float4 s3_smem4[];
    float* smem = reinterpret_cast<float*>(s3_smem4);
    constexpr int SLOT = s3_slot_floats<NARR>();
    S3Task mine[kMaxTasks];
    s3_tasks<NARR>(g, su, c, y0, z0, mine);
    const int nplanes = (x1 - x0) + 2;          // operand planes x0-1 .. x1 (factors x0-1 .. x1-1 suffice)
    // prologue: planes 0 .. kAhead-1
#pragma unroll
    for (int s = 0; s < kAhead; ++s) {
        if (s < nplanes) s3_issue<NARR>(g, su, c, x0 - 1 + s, smem + s * SLOT, mine);
        cp_commit();
    }
    const int tr = threadIdx.y + 1;             // tile row of this thread's output row
    const long long vrow = (long long)(y0 + threadIdx.y) * g.nz + z0 + 2 * threadIdx.x;
    const int col = 4 + 2 * threadIdx.x;        // smem column of vertex z
    const float s12 = (float)lt.s12;
    float P1[3][4], P2[3][4], K0[2][3], K1[2][3], Qlo[2][3], Exlo[2], P0c[2];
    auto readT = [&](const float* slot, float (&P)[3][4]) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m) P[j][m] = op.operand(slot, tr - 1 + j, col - 1 + m);
    };
    auto readK = [&](const float* slot, float (&K)[2][3]) {
        const float* kt = slot + NARR * kS3Tile;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 3; ++m) K[jj][m] = kt[(tr - 1 + jj) * kS3Pitch + col - 1 + m];
    };
    // stage s holds operand plane x0-1+s and factor plane x0-1+s; stage s -> slot s % kStages
    auto advance = [&](int s) {
        // plane s has landed once at most kAhead-1 newer groups are pending; the barrier
        // publishes every thread's copies and retires all reads of iteration s-1
        cp_wait<kAhead - 1>();
        __syncthreads();
        // plane s + kAhead goes to the slot of plane s - 2 (kStages = kAhead + 2),
        // whose last reader was iteration s - 1
        if (s + kAhead < nplanes)
            s3_issue<NARR>(g, su, c, x0 - 1 + s + kAhead, smem + ((s + kAhead) % kStages) * SLOT, mine);
        cp_commit();
    };
    {
        advance(0);
        float P0[3][4];
        readT(smem, P0);
        readK(smem, K0);
        P0c[0] = P0[1][1];
        P0c[1] = P0[1][2];
        advance(1);
        readT(smem + SLOT, P1);
        element_plane<float>(P0, P1, K0, Qlo, Exlo);
    }
    for (int s = 2; s < nplanes; ++s) {
        advance(s);
        // operand plane x+1 (x = x0 + s - 2) and factor plane x arrive; emit output plane x
        const float* slot = smem + (s % kStages) * SLOT;
        const float* xslot = smem + ((s - 1) % kStages) * SLOT;   // plane x: factors + pointwise arrays
        readT(slot, P2);
        readK(xslot, K1);
        float Qhi[2][3], Exhi[2];
        element_plane<float>(P1, P2, K1, Qhi, Exhi);
        float KX[2][3];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 3; ++m) KX[jj][m] = K0[jj][m] + K1[jj][m];
        float kt[2], ctr[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float qx = ((Qlo[0][i] + Qhi[0][i]) + (Qlo[0][i + 1] + Qhi[0][i + 1])) +
                             ((Qlo[1][i] + Qhi[1][i]) + (Qlo[1][i + 1] + Qhi[1][i + 1]));
            const float eym = KX[0][i] + KX[0][i + 1], eyp = KX[1][i] + KX[1][i + 1];
            const float ezm = KX[0][i] + KX[1][i], ezp = KX[0][i + 1] + KX[1][i + 1];
            const float kv = Exlo[i] + Exhi[i];
            float acc = 5.f * kv * P1[1][1 + i];
            acc += Exhi[i] * P2[1][1 + i] + Exlo[i] * P0c[i];
            acc += eyp * P1[2][1 + i] + eym * P1[0][1 + i];
            acc += ezp * P1[1][2 + i] + ezm * P1[1][i];
            kt[i] = s12 * (acc - qx);
            ctr[i] = P1[1][1 + i];
        }
        const int x = x0 + s - 2;
        op.sink(xslot, c, vrow + (long long)x * g.pl, tr, col, kt, ctr);
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int m = 0; m < 3; ++m) { Qlo[jj][m] = Qhi[jj][m]; K0[jj][m] = K1[jj][m]; }
        Exlo[0] = Exhi[0];
        Exlo[1] = Exhi[1];
        P0c[0] = P1[1][1];
        P0c[1] = P1[1][2];
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m) P1[j][m] = P2[j][m];
    }
    cp_wait<0>();
    __syncthreads();   // the next segment reuses the ring
}

// Persistent schedule: the work is the list of (case, tile column, x plane) units,
// column-major in x; block b takes the contiguous range [b W / B, (b+1) W / B) and
// walks it as one segment per tile column it touches.  B = resident blocks, so every
// SM gets the same number of planes whatever the grid shape.
template <int NARR, class Op>
__device__ __forceinline__ void march3(const Geo& g, const LevelTemplate& lt, const S3Setup<NARR>& su, Op& op,
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
        march3_segment<NARR>(g, lt, su, op, c, y0, z0, x0, x1);
        last_case = c;
        u += x1 - x0;
    }
}

}  // namespace otm
