// Level-stencil microbenchmark + correctness check against a host fp64 element
// assembly of K (K0 = template of element.py:59-88, kt[a ^ b]).  Links libotm.so;
// Usage: l0bench [n=128] [reps=50]
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2405_19991_b200/csrc \
//        tools/l0bench.cu -L paper_2405_19991_b200 -lotm -Xlinker -rpath,'$ORIGIN/../paper_2405_19991_b200' -o tools/l0bench
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "otm_internal.h"

using namespace otm;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

static const double KT[8] = {1.0 / 3, 0, 0, -1.0 / 12, 0, -1.0 / 12, -1.0 / 12, -1.0 / 12};

static void host_K(int n, const std::vector<float>& kap, const float* x, std::vector<double>& y) {
    const long long N = (long long)n * n * n;
    y.assign(N, 0.0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) {
                const long long e = ((long long)i * n + j) * n + k;
                long long v[8];
                double xv[8];
                for (int a = 0; a < 8; ++a) {
                    const int ii = (i + (a & 1)) % n, jj = (j + ((a >> 1) & 1)) % n, kk = (k + ((a >> 2) & 1)) % n;
                    v[a] = ((long long)ii * n + jj) * n + kk;
                    xv[a] = x[v[a]];
                }
                for (int a = 0; a < 8; ++a) {
                    double s = 0;
                    for (int b = 0; b < 8; ++b) s += KT[a ^ b] * xv[b];
                    y[v[a]] += kap[e] * s;
                }
            }
}

static double relerr(const std::vector<float>& got, const std::vector<double>& ref) {
    double m = 0, r = 0;
    for (size_t i = 0; i < ref.size(); ++i) {
        m = std::max(m, std::fabs(got[i] - ref[i]));
        r = std::max(r, std::fabs(ref[i]));
    }
    return m / r;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 128;
    const int reps = argc > 2 ? atoi(argv[2]) : 50;
    const bool check = !(argc > 3 && atoi(argv[3]) == 0);
    const long long N = (long long)n * n * n;
    const Geo g = make_geo(n, n, n);
    LevelTemplate lt{};
    lt.equal = 1;
    lt.s12 = 1.0 / 12.0;
    for (int a = 0; a < 8; ++a) lt.kt[a] = KT[a];
    std::mt19937 rng(1);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    std::vector<float> kap(N), dinv(N), p(3 * N), f(3 * N), z(3 * N);
    for (auto& v : kap) v = 0.05f + 0.95f * U(rng);
    for (auto& v : dinv) v = 0.5f + U(rng);
    for (auto& v : p) v = 2.f * U(rng) - 1.f;
    for (auto& v : f) v = 2.f * U(rng) - 1.f;
    for (auto& v : z) v = 2.f * U(rng) - 1.f;
    const float omega = 0.8f;
    float *dk, *dd, *dp, *df, *dz, *o0, *o1;
    CK(cudaMalloc(&dk, N * 4));
    CK(cudaMalloc(&dd, N * 4));
    CK(cudaMalloc(&dp, 3 * N * 4));
    CK(cudaMalloc(&df, 3 * N * 4));
    CK(cudaMalloc(&dz, 3 * N * 4));
    CK(cudaMalloc(&o0, 3 * N * 4));
    CK(cudaMalloc(&o1, 3 * N * 4));
    CK(cudaMemcpy(dk, kap.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dd, dinv.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, p.data(), 3 * N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(df, f.data(), 3 * N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dz, z.data(), 3 * N * 4, cudaMemcpyHostToDevice));
    Red red;
    CK(cudaMalloc(&red.partials, 8192 * 32 * 8));
    CK(cudaMalloc(&red.counter, 64));
    CK(cudaMemset(red.counter, 0, 64));
    PcgScalars* sc;
    CK(cudaMalloc(&sc, sizeof(PcgScalars)));
    CK(cudaMemset(sc, 0, sizeof(PcgScalars)));
    PcgScalars hs{};
    hs.first = 1;
    for (int c = 0; c < 3; ++c) hs.active[c] = 1.0, hs.rz[c] = 1.0;
    CK(cudaMemcpy(sc, &hs, sizeof(hs), cudaMemcpyHostToDevice));
    char* flush;
    const size_t flush_bytes = 256ull << 20;
    CK(cudaMalloc(&flush, flush_bytes));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

    const Geo gc = make_geo(n / 2, n / 2, n / 2);
    const int cf[3] = {1, 1, 1};
    auto run = [&](int which) {
        if (which == 0) launch_smooth_res(s, g, lt, dk, df, dd, omega, o0, o1);
        else if (which == 1) launch_jacobi(s, g, lt, dk, dz, df, dd, omega, o0, true, red, sc);
        else if (which == 2) launch_spmv(s, g, lt, dk, dp, o0, red, sc);
        else if (which == 3) launch_restrict(s, g, gc, cf, dp, o1);
        else launch_prolong(s, g, gc, cf, df, o0);
    };
    const char* names[5] = {"smooth_res", "jacobi", "spmv", "restrict", "prolong"};
    const double bpv[5] = {44, 44, 28, 13.5, 25.5};
    const int nkern = getenv("L0_TRANSFER") ? 5 : 3;
    for (int which = 0; which < nkern; ++which) {
        run(which);
        CK(cudaStreamSynchronize(s));
        CK(cudaGetLastError());
        if (check && which < 3) {
            std::vector<float> g0(3 * N), g1(3 * N);
            CK(cudaMemcpy(g0.data(), o0, 3 * N * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(g1.data(), o1, 3 * N * 4, cudaMemcpyDeviceToHost));
            double e0 = 0, e1 = 0, edot = 0;
            for (int c = 0; c < 3; ++c) {
                std::vector<double> Kx;
                std::vector<float> gc(g0.begin() + c * N, g0.begin() + (c + 1) * N);
                if (which == 2) {
                    host_K(n, kap, p.data() + c * N, Kx);
                    e0 = std::max(e0, relerr(gc, Kx));
                    double dot = 0;
                    for (long long v = 0; v < N; ++v) dot += (double)p[c * N + v] * Kx[v];
                    PcgScalars r;
                    CK(cudaMemcpy(&r, sc, sizeof(r), cudaMemcpyDeviceToHost));
                    edot = std::max(edot, std::fabs(r.pq[c] - dot) / std::fabs(dot));
                } else if (which == 1) {
                    host_K(n, kap, z.data() + c * N, Kx);
                    std::vector<double> ref(N);
                    for (long long v = 0; v < N; ++v)
                        ref[v] = z[c * N + v] + omega * dinv[v] * (f[c * N + v] - Kx[v]);
                    e0 = std::max(e0, relerr(gc, ref));
                } else {
                    std::vector<float> z0(N);
                    std::vector<double> z0d(N);
                    for (long long v = 0; v < N; ++v) z0[v] = omega * dinv[v] * f[c * N + v], z0d[v] = z0[v];
                    host_K(n, kap, z0.data(), Kx);
                    std::vector<double> ref(N);
                    for (long long v = 0; v < N; ++v) ref[v] = f[c * N + v] - Kx[v];
                    e0 = std::max(e0, relerr(gc, z0d));
                    std::vector<float> g1c(g1.begin() + c * N, g1.begin() + (c + 1) * N);
                    e1 = std::max(e1, relerr(g1c, ref));
                }
            }
            printf("%-10s check: out0 rel %.2e  out1 rel %.2e  dot rel %.2e\n", names[which], e0, e1, edot);
        }
        // cold: L2 flushed before each launch, event pair around the launch only
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        double cold = 0;
        for (int r = 0; r < reps; ++r) {
            cudaMemsetAsync(flush, r & 0xff, flush_bytes, s);
            cudaEventRecord(a, s);
            run(which);
            cudaEventRecord(b, s);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            cold += ms;
        }
        cold /= reps;
        // warm: back to back
        cudaEventRecord(a, s);
        for (int r = 0; r < reps; ++r) run(which);
        cudaEventRecord(b, s);
        CK(cudaEventSynchronize(b));
        float wms;
        cudaEventElapsedTime(&wms, a, b);
        const double warm = wms / reps;
        const double bytes = bpv[which] * N;
        printf("%-10s n=%d  cold %.2f us (%.0f GB/s)  back-to-back %.2f us (%.0f GB/s)\n", names[which], n,
               cold * 1e3, bytes / (cold * 1e-3) / 1e9, warm * 1e3, bytes / (warm * 1e-3) / 1e9);
        CK(cudaGetLastError());
    }
    return 0;
}
