// EWP backend (the reference's Appendix A formulation, block_operator.cpp:345-421):
// the Fourier-space step as element-wise products over a CHANNEL-major spectrum
// S[(i*N_m + j)*NF + f] (the reference's SpectralP2O::channel_spectra,
// block_operator.hpp:45, truncated to the NF = N_t+1 stored frequencies), with
// channel-major transformed vectors x[j*NF + f]:
//     forward  y[i][f] = sum_j S[i][j][f] x[j][f]          (j ascending)
//     adjoint  m[j][f] = sum_i conj(S[i][j][f]) d[i][f]     (i ascending)
// Threads run along f (coalesced 16-byte streams of S and the vector); a CTA
// owns kRows output channels so each vector row it reads is reused kRows times.
#include <cuda_runtime.h>

#include "btg_kernels.cuh"

namespace btg {
namespace {

constexpr int kRows = 8;
constexpr int kThreads = 256;

__device__ __forceinline__ double2 load_c(const double2* p) { return __ldg(p); }
__device__ __forceinline__ double2 load_c(const float2* p) {
    const float2 v = __ldg(p);
    return make_double2(v.x, v.y);
}

// [f][c] -> [c][f] in 32 x 32 tiles (F-hat frequency-major -> channel layout).
template <typename T>
__global__ void k_transpose_fc(const T* __restrict__ F, T* __restrict__ S, long long nf, long long nc) {
    __shared__ T tile[32][33];
    const long long c0 = (long long)blockIdx.x * 32, f0 = (long long)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const long long f = f0 + r, c = c0 + threadIdx.x;
        if (f < nf && c < nc) tile[r][threadIdx.x] = F[f * nc + c];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const long long c = c0 + r, f = f0 + threadIdx.x;
        if (c < nc && f < nf) S[c * nf + f] = tile[threadIdx.x][r];
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_ewp_fwd(const T* __restrict__ S, const double2* __restrict__ x,
                                                       double2* __restrict__ y, int nf, int nd, int nm) {
    const int f = blockIdx.x * kThreads + threadIdx.x;
    const int i0 = blockIdx.y * kRows;
    if (f >= nf) return;
    const int nr = min(kRows, nd - i0);
    double2 acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = make_double2(0.0, 0.0);
    for (int j = 0; j < nm; ++j) {
        const double2 v = __ldg(x + (size_t)j * nf + f);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            if (r < nr) {
                const double2 s = load_c(S + ((size_t)(i0 + r) * nm + j) * nf + f);
                acc[r].x += s.x * v.x - s.y * v.y;
                acc[r].y += s.x * v.y + s.y * v.x;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r)
        if (r < nr) y[(size_t)(i0 + r) * nf + f] = acc[r];
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_ewp_adj(const T* __restrict__ S, const double2* __restrict__ d,
                                                       double2* __restrict__ m, int nf, int nd, int nm) {
    const int f = blockIdx.x * kThreads + threadIdx.x;
    const int j0 = blockIdx.y * kRows;
    if (f >= nf) return;
    const int nr = min(kRows, nm - j0);
    double2 acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = make_double2(0.0, 0.0);
    for (int i = 0; i < nd; ++i) {
        const double2 v = __ldg(d + (size_t)i * nf + f);
#pragma unroll
        for (int r = 0; r < kRows; ++r) {
            if (r < nr) {
                const double2 s = load_c(S + ((size_t)i * nm + j0 + r) * nf + f);
                acc[r].x += s.x * v.x + s.y * v.y;  // conj(s) * v
                acc[r].y += s.x * v.y - s.y * v.x;
            }
        }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r)
        if (r < nr) m[(size_t)(j0 + r) * nf + f] = acc[r];
}

}  // namespace

template <typename T>
cudaError_t launch_channel_layout(const T* F, T* S, int nf, long long channels, cudaStream_t stream) {
    const dim3 grid((unsigned)((channels + 31) / 32), (unsigned)((nf + 31) / 32));
    k_transpose_fc<T><<<grid, dim3(32, 8), 0, stream>>>(F, S, nf, channels);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_ewp(bool adjoint, const T* S, const double2* in, double2* out, int nf, int nd, int nm,
                       cudaStream_t stream) {
    const dim3 grid((unsigned)((nf + kThreads - 1) / kThreads),
                    (unsigned)(((adjoint ? nm : nd) + kRows - 1) / kRows));
    if (adjoint)
        k_ewp_adj<T><<<grid, kThreads, 0, stream>>>(S, in, out, nf, nd, nm);
    else
        k_ewp_fwd<T><<<grid, kThreads, 0, stream>>>(S, in, out, nf, nd, nm);
    return cudaGetLastError();
}

template cudaError_t launch_channel_layout<double2>(const double2*, double2*, int, long long, cudaStream_t);
template cudaError_t launch_channel_layout<float2>(const float2*, float2*, int, long long, cudaStream_t);
template cudaError_t launch_ewp<double2>(bool, const double2*, const double2*, double2*, int, int, int,
                                         cudaStream_t);
template cudaError_t launch_ewp<float2>(bool, const float2*, const double2*, double2*, int, int, int,
                                        cudaStream_t);

}  // namespace btg
