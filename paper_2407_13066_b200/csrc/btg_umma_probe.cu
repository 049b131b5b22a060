// Hardware check of the tcgen05 kind::i8 conventions in btg_umma.cuh:
//  (1) A K-major x B K-major, (2) A MN-major x B K-major, both from core-matrix
//  tiles (8 x 16 B); D (int32, TMEM) compared with a host reference; (3) the
//  MMA issue rate for M=128, N=64, K=32 on every SM. Prints one JSON line.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "btg_umma.cuh"

using namespace btg::umma;

constexpr int M = 128, N = 64, K = 64;

// A_g: core matrices of 8 (i) x 16 (j) bytes. For the K-major test the MMA sees
// (row i, k = j); for the MN-major test (row j, k = i) from the same bytes.
__global__ void k_probe(const int8_t* __restrict__ Ag, const int8_t* __restrict__ Bg, int32_t* __restrict__ D,
                        int a_mn_major) {
    __shared__ __align__(1024) int8_t As[M * K];
    __shared__ __align__(1024) int8_t Bs[N * K];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int u = tid; u < M * K / 16; u += blockDim.x)
        reinterpret_cast<int4*>(As)[u] = reinterpret_cast<const int4*>(Ag)[u];
    for (int u = tid; u < N * K / 16; u += blockDim.x)
        reinterpret_cast<int4*>(Bs)[u] = reinterpret_cast<const int4*>(Bg)[u];
    fence_async_smem();
    if (warp == 0) tmem_alloc<64>(&tslot);
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t idesc = idesc_s8(M, N, a_mn_major != 0, false);
        for (int ks = 0; ks < K / 32; ++ks) {
            uint64_t ad, bd;
            if (!a_mn_major) {
                // A stored [ig = M/8][jg = K/16][8][16]: K-adjacent core matrices 128 B apart, M-adjacent 512 B
                ad = make_desc(smem_u32(As) + ks * 256, 128, (K / 16) * 128);
            } else {
                // A (row j, k = i) from [ig = K/8][jg = M/16][8][16]: M-adjacent 128 B, K-adjacent (M/16)*128 B
                ad = make_desc(smem_u32(As) + ks * 4 * (M / 16) * 128, (M / 16) * 128, 128);
            }
            // B stored [ng = N/8][kg = K/16][8][16]
            bd = make_desc(smem_u32(Bs) + ks * 256, 128, (K / 16) * 128);
            mma_s8(tmem, ad, bd, idesc, ks > 0);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after_sync();
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
        ld_wait();
        for (int q = 0; q < 16; ++q) D[row * N + c + q] = (int32_t)r[q];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_free<64>(tmem);
}

// Issue-rate probe: `iters` x (K/32) MMAs back to back on smem-resident tiles.
__global__ void k_rate(int iters, int32_t* out) {
    __shared__ __align__(1024) int8_t As[M * K];
    __shared__ __align__(1024) int8_t Bs[N * K];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int u = tid; u < M * K; u += blockDim.x) As[u] = (int8_t)(u * 7);
    for (int u = tid; u < N * K; u += blockDim.x) Bs[u] = (int8_t)(u * 3);
    fence_async_smem();
    if (warp == 0) tmem_alloc<64>(&tslot);
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        const uint32_t idesc = idesc_s8(M, N, false, false);
        for (int it = 0; it < iters; ++it)
            for (int ks = 0; ks < K / 32; ++ks)
                mma_s8(tmem, make_desc(smem_u32(As) + ks * 256, 128, 512), make_desc(smem_u32(Bs) + ks * 256, 128, 512),
                       idesc, (it | ks) > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after_sync();
    if (tid < 32) {
        uint32_t r[16];
        ld_32x32b_x16(tmem, r);
        ld_wait();
        if (tid == 0) out[blockIdx.x] = (int32_t)r[0];
    }
    fence_before_sync();
    __syncthreads();
    if (warp == 0) tmem_free<64>(tmem);
}

int main() {
    std::vector<int8_t> A(M * K), B(N * K);
    std::vector<int> a(M * K), b(N * K);  // logical a[m][k], b[n][k]
    srand(1);
    for (auto& v : a) v = rand() % 255 - 127;
    for (auto& v : b) v = rand() % 255 - 127;
    // B K-major core matrices [n/8][k/16][n%8][k%16]
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) B[((n / 8) * (K / 16) + k / 16) * 128 + (n % 8) * 16 + k % 16] = (int8_t)b[n * K + k];
    int8_t *dA, *dB;
    int32_t* dD;
    cudaMalloc(&dA, M * K);
    cudaMalloc(&dB, N * K);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
    long long err[2] = {0, 0};
    for (int mn = 0; mn < 2; ++mn) {
        for (int m = 0; m < M; ++m)
            for (int k = 0; k < K; ++k) {
                size_t off;
                if (!mn)  // rows i = m, cols j = k: [m/8][k/16][m%8][k%16]
                    off = ((size_t)(m / 8) * (K / 16) + k / 16) * 128 + (m % 8) * 16 + k % 16;
                else  // logical (row m = j, k = i): core matrix 8 i x 16 j, [k/8][m/16][k%8][m%16]
                    off = ((size_t)(k / 8) * (M / 16) + m / 16) * 128 + (k % 8) * 16 + m % 16;
                A[off] = (int8_t)a[m * K + k];
            }
        cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
        cudaMemset(dD, 0, M * N * 4);
        k_probe<<<1, 128>>>(dA, dB, dD, mn);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
            return 1;
        }
        std::vector<int32_t> D(M * N);
        cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                long long s = 0;
                for (int k = 0; k < K; ++k) s += (long long)a[m * K + k] * b[n * K + k];
                const long long d = llabs(s - D[m * N + n]);
                if (d > err[mn]) err[mn] = d;
            }
        if (err[mn]) {
            printf("mn=%d D[0][0..3]=%d %d %d %d\n", mn, D[0], D[1], D[2], D[3]);
        }
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    int32_t* dout;
    cudaMalloc(&dout, sms * 4);
    const int iters = 20000;
    k_rate<<<sms, 128>>>(100, dout);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate<<<sms, 128>>>(iters, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = (double)sms * iters * (K / 32) * M * N * 32;
    printf("{\"kmajor_maxerr\": %lld, \"mnmajor_maxerr\": %lld, \"i8_tops\": %.1f, \"cycles_per_mma_at_boost\": %.2f, "
           "\"status\": \"%s\"}\n",
           err[0], err[1], 2 * macs / (ms * 1e-3) / 1e12,
           (ms * 1e-3) * (clk_khz * 1e3) / ((double)iters * (K / 32)), cudaGetErrorString(cudaGetLastError()));
    return 0;
}
