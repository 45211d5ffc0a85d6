// Shared device helpers for libotm (sm_100a).
//
// Layout: every field is C-order (nx, ny, nz), z fastest, exactly the numpy
// layout of the reference (solver.py / field.py).  Batched load-case fields are
// case-major SoA: field[c * n + v].
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace otm {

constexpr int kCases = 3;

struct Geo {
    int nx, ny, nz;
    int pl;          // ny * nz
    long long n;     // nx * ny * nz
};

__host__ __device__ inline Geo make_geo(int nx, int ny, int nz) {
    Geo g;
    g.nx = nx; g.ny = ny; g.nz = nz;
    g.pl = ny * nz;
    g.n = (long long)nx * ny * nz;
    return g;
}

// x^p of the SIMP law (element.py:91-100): the integral penalties by multiplication
// (one or two roundings, within an ulp of numpy's pow; fp64 pow is a ~100-instruction
// log/exp sequence that made the filter+SIMP and sensitivity kernels issue-bound)
__device__ __forceinline__ double simp_pow(double x, double p) {
    if (p == 3.0) return x * x * x;
    if (p == 2.0) return x * x;
    if (p == 1.0) return x;
    if (p == 4.0) {
        const double x2 = x * x;
        return x2 * x2;
    }
    return pow(x, p);
}

__device__ __forceinline__ int wrap_m(int i, int n) { return i == 0 ? n - 1 : i - 1; }
__device__ __forceinline__ int wrap_p(int i, int n) { return i + 1 == n ? 0 : i + 1; }

// ---------------------------------------------------------------------------
// Deterministic reductions.  Every reduction is a fixed-order tree: warp
// shuffles, then warps in index order, then blocks in index order inside the
// last block to finish (ticketed by an integer atomic; the atomic only decides
// WHO sums, never the order).  No floating-point atomics anywhere, so reruns
// are bit-identical ("Determinism is a tested contract").
// ---------------------------------------------------------------------------

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialisation may start while its predecessor drains; it must not touch the
// predecessor's outputs before this wait (a no-op for ordinary launches).
// Right after the wait the kernel also triggers its own dependents, so the next
// kernel's launch and CTA rasterisation overlap this kernel's execution (without a
// trigger the dependent grid only launches once every block here has exited).  The
// dependent still waits for this grid's completion before touching its outputs.
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
#ifndef OTM_NO_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sums of NQ values; result valid in (linear) thread 0.  smem: >= 32*NQ doubles.
__device__ __forceinline__ int block_tid() {
    return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
}
__device__ __forceinline__ int block_threads() { return blockDim.x * blockDim.y * blockDim.z; }

// (works for 1-, 2- and 3-D blocks: threads are linearised x-fastest, so warps
// are consecutive linear indices)
template <int NQ>
__device__ __forceinline__ void block_sum(double (&v)[NQ], double* smem) {
    const int tid = block_tid();
    const int lane = tid & 31, wid = tid >> 5;
    const int nw = (block_threads() + 31) >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double s = warp_sum(v[q]);
        if (lane == 0) smem[q * 32 + wid] = s;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double s = lane < nw ? smem[q * 32 + lane] : 0.0;
            v[q] = warp_sum(s);
        }
    }
    __syncthreads();
}

// Writes this block's NQ partial sums, and lets the last block to finish reduce
// all partials (in block order) into out[NQ].  Returns true in thread 0 of the
// last block, after out[] is written.  nblocks = gridDim.x * gridDim.y.
template <int NQ>
__device__ bool reduce_finalize(double (&v)[NQ], double* partials, unsigned* counter,
                                double* out) {
    __shared__ double smem[32 * NQ];
    __shared__ bool is_last;
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int tid = block_tid();
    block_sum<NQ>(v, smem);
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) partials[(size_t)bid * NQ + q] = v[q];
        __threadfence();
        unsigned t = atomicAdd(counter, 1u);
        is_last = (t == nb - 1);
    }
    __syncthreads();
    if (!is_last) return false;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    for (unsigned b = tid; b < nb; b += block_threads()) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] += __ldcg(partials + (size_t)b * NQ + q);
    }
    block_sum<NQ>(acc, smem);
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) out[q] = acc[q];
        *counter = 0u;
        return true;
    }
    return false;
}

// Wide variant for 32 quantities: a butterfly reduce-scatter leaves the warp sum
// of quantity `lane` in lane `lane` (31 shuffles per lane instead of 160), then
// warps and blocks are summed in index order as above.
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const double keep = up ? v[i + o] : v[i];
            const double send = up ? v[i] : v[i + o];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// 1-D blocks only.  Returns true in thread 0 of the last block, out[0..31] written.
__device__ inline bool reduce_finalize32(double (&v)[32], double* partials, unsigned* counter, double* out) {
    __shared__ double sm[32][33];
    __shared__ bool is_last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned nb = gridDim.x;
    const double mine = warp_reduce_scatter32(v);
    sm[wid][lane] = mine;
    __syncthreads();
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += sm[w][threadIdx.x];
        partials[(size_t)blockIdx.x * 32 + threadIdx.x] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == nb - 1;
    __syncthreads();
    if (!is_last) return false;
    // last block: thread t sums quantity (t & 31) over blocks b = (t >> 5), (t >> 5) + nw, ...
    double s = 0.0;
    for (unsigned b = wid; b < nb; b += nw) s += __ldcg(partials + (size_t)b * 32 + lane);
    sm[wid][lane] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += sm[w][threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0u;
    return threadIdx.x == 0;
}

// ---------------------------------------------------------------------------
// Register-window stencil core.
//
// The periodic trilinear conduction operator (solver.py:85-119) is evaluated
// matrix-free from element factors.  A thread owns one (y, z) column and walks
// x; it keeps the 3x3 (y, z) neighbourhood of planes x-1, x, x+1 of the operand
// and the 2x2 element factors of element planes x-1, x in registers, so every
// operand value is loaded once per plane instead of 27 times per vertex.
//
// With equal axis scales s (every level of a 3-D cube) the element matrix is
// s * K0 with K0 = (5 I + N1 - J) / 12 (N1: 1-bit corner adjacency, J: all
// ones), so with S_e = sum of e's 8 corner values
//   (K T)_v = s/12 * ( 5 K_v T_v + sum_{6 axis nbrs u} E_vu T_u - sum_{e ni v} k_e S_e )
// where K_v sums the 8 incident k_e and E_vu the 4 elements sharing edge (v,u).
// ---------------------------------------------------------------------------

struct Nbr {
    long long xo[3];   // plane offsets of x-1, x, x+1 (wrapped)
    int ro[3];         // row offsets (times nz) of y-1, y, y+1
    int co[3];         // z-1, z, z+1
};

__device__ __forceinline__ void nbr_init(Nbr& nb, const Geo& g, int y, int z) {
    nb.ro[0] = wrap_m(y, g.ny) * g.nz; nb.ro[1] = y * g.nz; nb.ro[2] = wrap_p(y, g.ny) * g.nz;
    nb.co[0] = wrap_m(z, g.nz); nb.co[1] = z; nb.co[2] = wrap_p(z, g.nz);
}

__device__ __forceinline__ long long plane_off(const Geo& g, int x) {
    int xx = x < 0 ? x + g.nx : (x >= g.nx ? x - g.nx : x);
    return (long long)xx * g.pl;
}

template <typename R>
struct KSum {      // element-factor sums around a vertex
    R kv, exp_, exm, eyp, eym, ezp, ezm;
};

// k[q][jj*2+kk]: element at plane x-1+q, row y-1+jj, col z-1+kk
template <typename R>
__device__ __forceinline__ KSum<R> ksum(const R (&k)[2][4]) {
    KSum<R> s;
    s.exm = (k[0][0] + k[0][1]) + (k[0][2] + k[0][3]);
    s.exp_ = (k[1][0] + k[1][1]) + (k[1][2] + k[1][3]);
    s.eym = (k[0][0] + k[0][1]) + (k[1][0] + k[1][1]);
    s.eyp = (k[0][2] + k[0][3]) + (k[1][2] + k[1][3]);
    s.ezm = (k[0][0] + k[0][2]) + (k[1][0] + k[1][2]);
    s.ezp = (k[0][1] + k[0][3]) + (k[1][1] + k[1][3]);
    s.kv = s.exm + s.exp_;
    return s;
}

// t[p][j*3+kk]: operand at plane x-1+p, row y-1+j, col z-1+kk
template <typename R>
__device__ __forceinline__ R apply_compact(const R (&t)[3][9], const R (&k)[2][4], const KSum<R>& s,
                                           R s12) {
    // plane-pair sums A_q[j][kk] = t[q][.] + t[q+1][.]
    R ks = R(0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        R a[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) a[i] = t[q][i] + t[q + 1][i];
        R b[3][2];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            b[j][0] = a[j * 3 + 0] + a[j * 3 + 1];
            b[j][1] = a[j * 3 + 1] + a[j * 3 + 2];
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) ks += k[q][jj * 2 + kk] * (b[jj][kk] + b[jj + 1][kk]);
    }
    R acc = R(5) * s.kv * t[1][4];
    acc += s.exp_ * t[2][4] + s.exm * t[0][4];
    acc += s.eyp * t[1][7] + s.eym * t[1][1];
    acc += s.ezp * t[1][5] + s.ezm * t[1][3];
    return s12 * (acc - ks);
}

// General axis scales: K[a][b] = kt[a ^ b] (the 8x8 template depends only on the
// corner XOR pattern).  Vertex v is corner a = (1-q) | (1-jj)<<1 | (1-kk)<<2 of
// element (q, jj, kk).
template <typename R>
__device__ __forceinline__ R apply_generic(const R (&t)[3][9], const R (&k)[2][4], const R* kt) {
    R acc = R(0);
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                const int a = (1 - q) | ((1 - jj) << 1) | ((1 - kk) << 2);
                R e = R(0);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    const int bx = b & 1, by = (b >> 1) & 1, bz = (b >> 2) & 1;
                    e += kt[a ^ b] * t[q + bx][(jj + by) * 3 + (kk + bz)];
                }
                acc += k[q][jj * 2 + kk] * e;
            }
    return acc;
}

}  // namespace otm
