// Measurement yardstick only (not product code): cuFFT batched D2Z/Z2D of length 2N_t,
// channel-major, timed with CUDA events — the library reference point quoted in
// profiles/r01s2_fft_sweep.md. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a cufft_yardstick.cu -lcufft
#include <cufft.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
    int N = argc > 1 ? atoi(argv[1]) : 1024, C = argc > 2 ? atoi(argv[2]) : 524288;
    int L = 2 * N;
    double* x; cufftDoubleComplex* X;
    cudaMalloc(&x, (size_t)C * L * 8); cudaMalloc(&X, (size_t)C * (N + 1) * 16);
    cudaMemset(x, 0, (size_t)C * L * 8);
    cufftHandle pf, pi;
    int n[1] = {L};
    cufftPlanMany(&pf, 1, n, nullptr, 1, L, nullptr, 1, N + 1, CUFFT_D2Z, C);
    cufftPlanMany(&pi, 1, n, nullptr, 1, N + 1, nullptr, 1, L, CUFFT_Z2D, C);
    cudaEvent_t a, b, c; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
    float tf = 0, ti = 0;
    for (int r = -2; r < 10; ++r) {
        cudaEventRecord(a); cufftExecD2Z(pf, x, X); cudaEventRecord(b); cufftExecZ2D(pi, X, x); cudaEventRecord(c);
        cudaEventSynchronize(c); float p, q; cudaEventElapsedTime(&p, a, b); cudaEventElapsedTime(&q, b, c);
        if (r >= 0) { tf += p; ti += q; }
    }
    tf /= 10; ti /= 10;
    double by = 8.0 * C * L + 16.0 * C * (N + 1);
    printf("{\"cufft\": 1, \"N_t\": %d, \"channels\": %d, \"d2z_ms\": %.4f, \"d2z_tbs\": %.3f, \"z2d_ms\": %.4f, \"z2d_tbs\": %.3f, \"our_bytes_equiv_d2z_ms_at_same_tbs\": %.4f}\n",
           N, C, tf, by / tf / 1e9, ti, by / ti / 1e9, (8.0 * C * N + 16.0 * C * (N + 1)) / (by / tf / 1e9) / 1e9 * 1e3);
    return 0;
}
