// Vector kernels of the device-resident CG solver (btg_cg_solve): the caller
// of the Hessian action (reference inverse.cpp:105-156).
//
// Every reduction is two-level with a FIXED grid (kRedBlocks x 256 threads,
// grid-stride ownership, tree within the block, one block summing the
// partials in index order): dot products are bit-identical run to run.
#include <cuda_runtime.h>

#include <cstdint>

#include "btg_kernels.cuh"

namespace btg {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < kThreads / 32; ++w) s += sh[w];
    }
    __syncthreads();
    return s;  // valid in thread 0
}

__global__ void __launch_bounds__(kThreads) k_dot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                          size_t n, double* __restrict__ partial) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads)
        acc = fma(a[i], b[i], acc);
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_sum_partials(const double* __restrict__ partial, int count,
                                                           double* __restrict__ out) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += kThreads) acc += partial[i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) *out = s;
}

// x += s p ; r -= s hp ; partial ||r||^2   (inverse.cpp:132-136 fused with norm(residual))
__global__ void __launch_bounds__(kThreads) k_cg_update(double* __restrict__ x, double* __restrict__ r,
                                                        const double* __restrict__ p, const double* __restrict__ hp,
                                                        double s, size_t n, double* __restrict__ partial) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0;
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads) {
        x[i] += s * p[i];
        const double ri = r[i] - s * hp[i];
        r[i] = ri;
        acc = fma(ri, ri, acc);
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// p = z + beta p   (inverse.cpp:152-153)
__global__ void __launch_bounds__(kThreads) k_xpby(double* __restrict__ p, const double* __restrict__ z, double beta,
                                                   size_t n) {
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads)
        p[i] = z[i] + beta * p[i];
}

// y = a - b (residual of the objective)
__global__ void __launch_bounds__(kThreads) k_sub(double* __restrict__ y, const double* __restrict__ a,
                                                  const double* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads)
        y[i] = a[i] - b[i];
}

// R v for the temporal Laplacian per source row (inverse.cpp:32-49), or copy.
__global__ void __launch_bounds__(kThreads) k_reg_apply(double* __restrict__ y, const double* __restrict__ v,
                                                        size_t rows, int nt, int kind) {
    const size_t n = rows * (size_t)nt;
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads) {
        if (kind == 0) {
            y[i] = v[i];
            continue;
        }
        const int t = (int)(i % nt);
        double acc = 2.0 * v[i];
        if (t > 0) acc -= v[i - 1];
        if (t + 1 < nt) acc -= v[i + 1];
        y[i] = acc;
    }
}

// R^{-1} v: Thomas solve of the (-1, 2, -1) system per source row, with the
// row-independent pivots precomputed in the reference's order
// (inverse.cpp:51-72): x[0] = b[0]/p0; x[t] = (b[t] + x[t-1]) / p_t;
// x[t] -= c_{t+1} x[t+1] backwards. One thread per row.
__global__ void __launch_bounds__(kThreads) k_reg_apply_inverse(double* __restrict__ x, const double* __restrict__ b,
                                                                const double* __restrict__ pivot,
                                                                const double* __restrict__ scratch, size_t rows,
                                                                int nt) {
    const size_t row = blockIdx.x * (size_t)kThreads + threadIdx.x;
    if (row >= rows) return;
    const double* br = b + row * nt;
    double* xr = x + row * nt;
    double prev = br[0] / pivot[0];
    xr[0] = prev;
    for (int t = 1; t < nt; ++t) {
        prev = (br[t] + prev) / pivot[t];
        xr[t] = prev;
    }
    double next = xr[nt - 1];
    for (int t = nt - 1; t-- > 0;) {
        next = xr[t] - scratch[t + 1] * next;
        xr[t] = next;
    }
}

// ---- device-resident CG control (btg_cg_solve's graph loop) -----------------
// The scalars of inverse.cpp:105-156 live in device memory (CgState) so that a
// whole iteration — Hessian, curvature, update, convergence test, beta, new
// direction — runs without a host round trip, inside the body of a CUDA graph
// WHILE node whose condition the check kernel clears. The arithmetic is the
// host loop's, operation for operation (same divisions, same fixed-grid
// reductions), so both loops produce the same bits.

// x += (rho / pHp) p ; r -= (rho / pHp) hp ; partial ||r||^2. A non-positive
// curvature leaves x and r untouched (the reference throws before updating).
__global__ void __launch_bounds__(kThreads) k_cg_update_dev(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ hp,
                                                            const double* __restrict__ st, size_t n,
                                                            double* __restrict__ partial) {
    __shared__ double sh[kThreads / 32];
    const double curv = st[kCgCurvature];
    double acc = 0.0;
    if (curv > 0.0) {
        const double s = st[kCgRho] / curv;
        for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads) {
            x[i] += s * p[i];
            const double ri = r[i] - s * hp[i];
            r[i] = ri;
            acc = fma(ri, ri, acc);
        }
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// ||r||^2 from the partials, then the loop control of inverse.cpp:137-150:
// curvature test, iteration count, relative residual, tolerance, iteration
// cap; unpreconditioned CG also takes beta = rn2 / rho here.
__global__ void __launch_bounds__(kThreads) k_cg_check(const double* __restrict__ partial, int count,
                                                       double* __restrict__ st, cudaGraphConditionalHandle cond,
                                                       int precond) {
    __shared__ double sh[kThreads / 32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += kThreads) acc += partial[i];
    const double rn2 = block_sum(acc, sh);
    if (threadIdx.x != 0) return;
    if (!(st[kCgCurvature] > 0.0)) {
        st[kCgStatus] = kCgBadCurvature;
        cudaGraphSetConditional(cond, 0);
        return;
    }
    const double it = st[kCgIterations] + 1.0;
    st[kCgIterations] = it;
    st[kCgRn2] = rn2;
    const double rel = sqrt(rn2) / st[kCgRhsNorm];
    st[kCgRelRes] = rel;
    if (rel <= st[kCgTol]) {
        st[kCgStatus] = kCgConverged;
        cudaGraphSetConditional(cond, 0);
        return;
    }
    if (it >= st[kCgMaxIt]) {
        st[kCgStatus] = kCgMaxIterations;
        cudaGraphSetConditional(cond, 0);
        return;
    }
    if (!precond) {
        st[kCgBeta] = rn2 / st[kCgRho];
        st[kCgRho] = rn2;
    }
}

// beta = (r . z) / rho ; rho = r . z  (preconditioned CG, inverse.cpp:146-151)
__global__ void k_cg_beta(double* __restrict__ st) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && st[kCgStatus] == kCgRunning) {
        const double rho_next = st[kCgRhoNext];
        st[kCgBeta] = rho_next / st[kCgRho];
        st[kCgRho] = rho_next;
    }
}

// p = z + beta p with beta from the state (inverse.cpp:152-153)
__global__ void __launch_bounds__(kThreads) k_xpby_dev(double* __restrict__ p, const double* __restrict__ z,
                                                       const double* __restrict__ st, size_t n) {
    if (st[kCgStatus] != kCgRunning) return;
    const double beta = st[kCgBeta];
    for (size_t i = blockIdx.x * (size_t)kThreads + threadIdx.x; i < n; i += (size_t)gridDim.x * kThreads)
        p[i] = z[i] + beta * p[i];
}

int grid_for(size_t n) {
    const size_t want = (n + kThreads - 1) / kThreads;
    return (int)(want < (size_t)kRedBlocks ? (want ? want : 1) : kRedBlocks);
}

}  // namespace

cudaError_t launch_dot(const double* a, const double* b, size_t n, double* partial, double* out,
                       cudaStream_t stream) {
    k_dot_partial<<<kRedBlocks, kThreads, 0, stream>>>(a, b, n, partial);
    k_sum_partials<<<1, kThreads, 0, stream>>>(partial, kRedBlocks, out);
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double* partial, int count, double* out, cudaStream_t stream) {
    k_sum_partials<<<1, kThreads, 0, stream>>>(partial, count, out);
    return cudaGetLastError();
}

cudaError_t launch_cg_update(double* x, double* r, const double* p, const double* hp, double s, size_t n,
                             double* partial, double* rnorm2, cudaStream_t stream) {
    k_cg_update<<<kRedBlocks, kThreads, 0, stream>>>(x, r, p, hp, s, n, partial);
    k_sum_partials<<<1, kThreads, 0, stream>>>(partial, kRedBlocks, rnorm2);
    return cudaGetLastError();
}

cudaError_t launch_xpby(double* p, const double* z, double beta, size_t n, cudaStream_t stream) {
    k_xpby<<<grid_for(n), kThreads, 0, stream>>>(p, z, beta, n);
    return cudaGetLastError();
}

cudaError_t launch_cg_update_dev(double* x, double* r, const double* p, const double* hp, const double* st, size_t n,
                                 double* partial, cudaStream_t stream) {
    k_cg_update_dev<<<kRedBlocks, kThreads, 0, stream>>>(x, r, p, hp, st, n, partial);
    return cudaGetLastError();
}

cudaError_t launch_cg_check(const double* partial, double* st, cudaGraphConditionalHandle cond, int precond,
                            cudaStream_t stream) {
    k_cg_check<<<1, kThreads, 0, stream>>>(partial, kRedBlocks, st, cond, precond);
    return cudaGetLastError();
}

cudaError_t launch_cg_beta(double* st, cudaStream_t stream) {
    k_cg_beta<<<1, 32, 0, stream>>>(st);
    return cudaGetLastError();
}

cudaError_t launch_xpby_dev(double* p, const double* z, const double* st, size_t n, cudaStream_t stream) {
    k_xpby_dev<<<grid_for(n), kThreads, 0, stream>>>(p, z, st, n);
    return cudaGetLastError();
}

cudaError_t launch_sub(double* y, const double* a, const double* b, size_t n, cudaStream_t stream) {
    k_sub<<<grid_for(n), kThreads, 0, stream>>>(y, a, b, n);
    return cudaGetLastError();
}

cudaError_t launch_reg_apply(double* y, const double* v, size_t rows, int nt, int kind, cudaStream_t stream) {
    k_reg_apply<<<grid_for(rows * (size_t)nt), kThreads, 0, stream>>>(y, v, rows, nt, kind);
    return cudaGetLastError();
}

cudaError_t launch_reg_apply_inverse(double* x, const double* b, const double* pivot, const double* scratch,
                                     size_t rows, int nt, cudaStream_t stream) {
    const int grid = (int)((rows + kThreads - 1) / kThreads);
    k_reg_apply_inverse<<<grid, kThreads, 0, stream>>>(x, b, pivot, scratch, rows, nt);
    return cudaGetLastError();
}

}  // namespace btg
