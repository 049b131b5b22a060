// Development micro-benchmark for the vector transforms K5 (R2C) / K9 (C2R):
// times the compile-time-N kernels on C channels with CUDA events and checks
// the round trip C2R(R2C(x)) == x. Not part of the product library.
//   btg_fft_bench [N_t=1024] [channels=524288] [reps=10]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "btg_fft_fast.cuh"

using namespace btg;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

static double2 root(long long num, long long den) {
    num %= den;
    if (num < 0) num += den;
    const long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)num / (long double)den;
    return make_double2((double)cosl(a), (double)(-sinl(a)));
}

#ifndef BENCH_CPB
#define BENCH_CPB 0
#endif
template <int N>
struct Run {
    static void go(int C, int reps) {
        using P = fast::FastPlan<N>;
        constexpr int CPBR = BENCH_CPB ? BENCH_CPB : P::CPB_R2C;
        constexpr int CPBC = BENCH_CPB ? BENCH_CPB : P::CPB_C2R;
#ifdef BENCH_PF
        constexpr bool pf_r = BENCH_PF & 1, pf_c = BENCH_PF & 2;
#else
        constexpr bool pf_r = P::PF_R2C, pf_c = P::PF_C2R;
#endif

        const int hi = fast::tw_hi_count<N>();
        std::vector<double2> t(32 + hi + 32 + hi + 1);
        for (int i = 0; i < 32; ++i) t[i] = root(i, N);
        for (int h = 0; h < hi; ++h) t[32 + h] = root(32LL * h, N);
        for (int i = 0; i < 32; ++i) t[32 + hi + i] = root(i, 2LL * N);
        for (int h = 0; h <= hi; ++h) t[64 + hi + h] = root(32LL * h, 2LL * N);
        double2* dt;
        CK(cudaMalloc(&dt, t.size() * sizeof(double2)));
        CK(cudaMemcpy(dt, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice));
        std::vector<double2> wt(N + N + 1);
        for (int k = 0; k < N; ++k) wt[k] = root(k, N);
        for (int k = 0; k <= N; ++k) wt[N + k] = root(k, 2LL * N);
        double2* dw;
        CK(cudaMalloc(&dw, wt.size() * sizeof(double2)));
        CK(cudaMemcpy(dw, wt.data(), wt.size() * sizeof(double2), cudaMemcpyHostToDevice));
        FastTables tabs{dt, dt + 32, dt + 32 + hi, dt + 64 + hi, dw, dw + N};

        const size_t nx = (size_t)C * N, nf = (size_t)(N + 1) * C;
        double *x, *y;
        double2* X;
        CK(cudaMalloc(&x, nx * 8));
        CK(cudaMalloc(&y, nx * 8));
        CK(cudaMalloc(&X, nf * 16));
        std::vector<double> hx(nx);
        srand(7);
        for (size_t i = 0; i < nx; ++i) hx[i] = (double)rand() / RAND_MAX - 0.5;
        CK(cudaMemcpy(x, hx.data(), nx * 8, cudaMemcpyHostToDevice));

#ifdef BENCH_NO_TMA
        constexpr bool tma_r = false;
#elif defined(BENCH_FORCE_TMA)
        constexpr bool tma_r = true;
#else
        constexpr bool tma_r = fast::UseTmaR2C<N>::value;
#endif
        auto r2c = tma_r ? fast::k_r2c_tma<N, CPBR> : pf_r ? fast::k_r2c_pf<N, CPBR> : fast::k_r2c_fast<N, CPBR>;
        constexpr size_t smem_r = tma_r ? fast::smem_bytes_tma<N, CPBR>() : fast::smem_dir<N, CPBR, true>();
#ifdef BENCH_BLOCKED
        // the multi-RHS pipeline's channel-blocked spectrum: TMA R2C -> k_c2r_tma
        static_assert(fast::c2r_tma_ok<N, CPBC>(), "blocked C2R needs the TMA plan");
        constexpr bool c2r_persist = true;
        const long long fs = kBlockedFs;
#ifdef BENCH_LIGHT
        constexpr bool light = true;
#else
        constexpr bool light = false;
#endif
        auto c2r = fast::k_c2r_tma<N, CPBC, light>;
        constexpr size_t smem_c = fast::smem_bytes_c2r_tma<N, CPBC, light>();
#else
        constexpr bool c2r_persist = pf_c;
        const long long fs = C;
#ifdef BENCH_LIGHT
        auto c2r = pf_c ? fast::k_c2r_pf<N, CPBC, true> : fast::k_c2r_fast<N, CPBC, false, true>;
#else
        auto c2r = pf_c ? fast::k_c2r_pf<N, CPBC> : fast::k_c2r_fast<N, CPBC>;
#endif
        constexpr size_t smem_c = fast::smem_dir<N, CPBC, false>();
#endif
        CK(cudaFuncSetAttribute(r2c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r));
        CK(cudaFuncSetAttribute(c2r, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
        int occ_r = 1, occ_c = 1, sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_r, r2c, P::TPC * CPBR, smem_r);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, c2r, P::TPC * CPBC, smem_c);
        const int groups_r = (C + CPBR - 1) / CPBR, groups_c = (C + CPBC - 1) / CPBC;
        const int grid_r = (pf_r || tma_r) ? std::min(groups_r, occ_r * sms) : groups_r;
        const int grid_c = c2r_persist ? std::min(groups_c, occ_c * sms) : groups_c;
        C2REpilogue epi{};
        cudaEvent_t e0, e1, e2;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        float tr = 0, tc = 0;
        for (int r = -2; r < reps; ++r) {
            cudaEventRecord(e0);
            r2c<<<grid_r, P::TPC * CPBR, smem_r>>>(x, N, X, fs, C, tabs, R2CBlockMax{});
            cudaEventRecord(e1);
            c2r<<<grid_c, P::TPC * CPBC, smem_c>>>(X, fs, y, N, C, tabs, epi);
            cudaEventRecord(e2);
            CK(cudaEventSynchronize(e2));
            float a, b;
            cudaEventElapsedTime(&a, e0, e1);
            cudaEventElapsedTime(&b, e1, e2);
            if (r >= 0) {
                tr += a;
                tc += b;
            }
        }
        CK(cudaGetLastError());
        std::vector<double> hy(nx);
        CK(cudaMemcpy(hy.data(), y, nx * 8, cudaMemcpyDeviceToHost));
        double num = 0, den = 0;
        for (size_t i = 0; i < nx; ++i) {
            num += (hy[i] - hx[i]) * (hy[i] - hx[i]);
            den += hx[i] * hx[i];
        }
        tr /= reps;
        tc /= reps;
        const double bytes = 8.0 * nx + 16.0 * nf;
        std::printf(
            "{\"N_t\": %d, \"channels\": %d, \"cpb\": %d, \"r2c_ms\": %.4f, \"r2c_tbs\": %.3f, \"c2r_ms\": %.4f, "
            "\"c2r_tbs\": %.3f, \"roundtrip_rel_l2\": %.3e, \"occ\": [%d, %d], \"blocked\": %d}\n",
            N, C, CPBR * 100 + CPBC, tr, bytes / tr / 1e9, tc, bytes / tc / 1e9, std::sqrt(num / den), occ_r, occ_c, (int)(fs < 0));
        cudaFree(x);
        cudaFree(y);
        cudaFree(X);
        cudaFree(dt);
    }
};

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
    const int C = argc > 2 ? std::atoi(argv[2]) : 524288;
    const int reps = argc > 3 ? std::atoi(argv[3]) : 10;
#ifdef BENCH_BLOCKED
    if (n != 1024) {
        std::printf("{\"error\": \"blocked mode: N_t = 1024 only\"}\n");
        return 1;
    }
    Run<1024>::go(C, reps);
#else
    switch (n) {
        case 64: Run<64>::go(C, reps); break;
        case 128: Run<128>::go(C, reps); break;
        case 256: Run<256>::go(C, reps); break;
        case 500: Run<500>::go(C, reps); break;
        case 512: Run<512>::go(C, reps); break;
        case 1000: Run<1000>::go(C, reps); break;
        case 1024: Run<1024>::go(C, reps); break;
        case 2000: Run<2000>::go(C, reps); break;
        case 2048: Run<2048>::go(C, reps); break;
        case 4096: Run<4096>::go(C, reps); break;
        default: std::printf("{\"error\": \"unsupported N_t %d\"}\n", n); return 1;
    }
#endif
    return 0;
}
