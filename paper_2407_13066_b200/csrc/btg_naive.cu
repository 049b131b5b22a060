// Naive backend (naive_apply_forward / naive_apply_adjoint,
// block_operator.cpp:423-482): the direct triangular block-Toeplitz sum on the
// compact operator, O(N_t^2 N_d N_m / 2), in the reference's loop order
// (forward: per output step, input steps ascending, each block row a j-ascending
// dot product added to the output; adjoint: output steps ascending, sensors
// ascending) — a device cross-check of the FFT path on small problems. Vectors
// are SOTI; blocks TOSI [k][i][j].
#include <cuda_runtime.h>

#include "btg_kernels.cuh"

namespace btg {
namespace {

__global__ void k_naive_fwd(const double* __restrict__ B, const double* __restrict__ m, double* __restrict__ d,
                            int nd, int nm, int nt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (t >= nt) return;
    double out = 0.0;
    for (int ti = 0; ti <= t; ++ti) {
        const double* row = B + ((size_t)(t - ti) * nd + i) * nm;
        double acc = 0.0;
        for (int j = 0; j < nm; ++j) acc = fma(__ldg(row + j), __ldg(m + (size_t)j * nt + ti), acc);
        out += acc;
    }
    d[(size_t)i * nt + t] = out;
}

__global__ void k_naive_adj(const double* __restrict__ B, const double* __restrict__ d, double* __restrict__ m,
                            int nd, int nm, int nt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (s >= nt) return;
    double out = 0.0;
    for (int to = s; to < nt; ++to) {
        const double* blk = B + (size_t)(to - s) * nd * nm + j;
        for (int i = 0; i < nd; ++i) out = fma(__ldg(blk + (size_t)i * nm), __ldg(d + (size_t)i * nt + to), out);
    }
    m[(size_t)j * nt + s] = out;
}

}  // namespace

cudaError_t launch_naive(bool adjoint, const double* blocks, const double* in, double* out, int nd, int nm, int nt,
                         cudaStream_t stream) {
    const dim3 grid((unsigned)((nt + 127) / 128), (unsigned)(adjoint ? nm : nd));
    if (adjoint)
        k_naive_adj<<<grid, 128, 0, stream>>>(blocks, in, out, nd, nm, nt);
    else
        k_naive_fwd<<<grid, 128, 0, stream>>>(blocks, in, out, nd, nm, nt);
    return cudaGetLastError();
}

}  // namespace btg
