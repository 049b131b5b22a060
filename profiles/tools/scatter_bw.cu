// Dev micro-benchmark: HBM bandwidth of the frequency-major vector layout
// out[k * C + c] when each CTA writes (or reads) G adjacent channels per k-row
// (G x 16-byte segments), as the vector FFTs do with G = channels per CTA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scatter_bw.cu -o scatter_bw
#include <cstdio>
#include <cuda_runtime.h>

template <int G>
__global__ void __launch_bounds__(256) k_write(double2* out, int K, int C) {
    // CTA: G channels x (256/G) k-lanes
    const int b = threadIdx.x % G, kl = threadIdx.x / G;
    const int c = blockIdx.x * G + b;
    const double2 v = make_double2(c, 1.0);
    for (int k = kl; k < K; k += 256 / G) out[(size_t)k * C + c] = v;
}
template <int G>
__global__ void __launch_bounds__(256) k_read(const double2* in, double* sink, int K, int C) {
    const int b = threadIdx.x % G, kl = threadIdx.x / G;
    const int c = blockIdx.x * G + b;
    double acc = 0.0;
    for (int k = kl; k < K; k += 256 / G) {
        const double2 v = __ldg(in + (size_t)k * C + c);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) sink[c] = acc;
}

template <int G>
void run(double2* buf, double* sink, int K, int C) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tw = 0, tr = 0;
    for (int r = -1; r < 5; ++r) {
        cudaEventRecord(a);
        k_write<G><<<C / G, 256>>>(buf, K, C);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 0) tw += ms;
        cudaEventRecord(a);
        k_read<G><<<C / G, 256>>>(buf, sink, K, C);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 0) tr += ms;
    }
    const double bytes = 16.0 * K * C;
    printf("{\"G\": %d, \"segment_bytes\": %d, \"write_GBs\": %.0f, \"read_GBs\": %.0f}\n", G, 16 * G,
           bytes / (tw / 5 * 1e-3) / 1e9, bytes / (tr / 5 * 1e-3) / 1e9);
}

int main() {
    const int K = 1025, C = 524288;
    double2* buf;
    double* sink;
    cudaMalloc(&buf, (size_t)K * C * 16);
    cudaMalloc(&sink, (size_t)C * 8);
    run<1>(buf, sink, K, C);
    run<2>(buf, sink, K, C);
    run<4>(buf, sink, K, C);
    run<8>(buf, sink, K, C);
    run<16>(buf, sink, K, C);
    run<32>(buf, sink, K, C);
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
