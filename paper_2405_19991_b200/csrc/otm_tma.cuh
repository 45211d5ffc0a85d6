// TMA + mbarrier plumbing shared by the level stencils (otm_stencil10.cuh) and the
// fp64 defect kernel (otm_res64w.cuh): one elected thread issues
// cp.async.bulk.tensor boxes that complete on a per-slot mbarrier (expect_tx
// bytes), so the global->shared transfer bypasses the LSU/L1 pipe that the
// stencils' shared-memory reads need; paired-fp32 (FFMA2) helpers.
#pragma once

#include <cuda.h>

#include "otm_common.cuh"
#include "otm_internal.h"

namespace otm {

// full-z row tiles of TY = 512 / nz rows (fp64 defect kernel geometry)
__host__ __device__ inline int tile_rows(int nz) { return 512 / nz; }
__host__ __device__ inline bool tma_tiling(const Geo& g, const LevelTemplate& lt) {
    return lt.equal && (g.nz == 64 || g.nz == 128 || g.nz == 256) && g.ny % tile_rows(g.nz) == 0 && g.nx >= 2;
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

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

}  // namespace otm
