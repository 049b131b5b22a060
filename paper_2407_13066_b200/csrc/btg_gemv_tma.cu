// TMA-staged, persistent Fourier-space step (K7) for FP64 F-hat.
//
// The single-RHS product is a pure HBM stream over F-hat (0.5 flop/B). The
// register-load kernels in btg_kernels.cu issue a burst of 16-byte loads and
// then wait for all of them before the next burst, so each thread's memory
// pipeline drains once per iteration and every CTA pays a fill/drain at its
// start and end. Here a persistent CTA (one per SM) keeps a ring of STAGES
// shared-memory stages continuously in flight with 1-D bulk TMA copies
// (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first so the re-read
// vector slices stay resident), across work-item boundaries, while all warps
// consume the previous stages. Full/empty mbarriers implement the ring; one
// elected thread is the producer.
//
//  k_gemv_adj_tma: item = (f, block of JB columns); one stage = one row
//      segment F[f][i][j0:j0+JB] (16 KB); thread t owns columns t + 256 q and
//      accumulates conj(F) * d_f[i] over i ascending (the reference's order,
//      block_operator.cpp:306-310) — no reduction.
//  k_gemv_fwd_tma: item = (f, block of ROWS rows); one stage = ROWS row
//      segments of JC columns + the matching m-hat_f chunk; thread t owns
//      column t of each chunk, accumulates ROWS complex partial dots, and the
//      item ends with a fixed-order block reduction (bit-identical repeats).
#include <cuda_runtime.h>

#include <cstdint>

#include "btg_kernels.cuh"

namespace btg {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "BTG_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra BTG_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 1-D bulk copy global -> shared; completion counted in bytes on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_load(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Work-item cursor: items blockIdx.x, blockIdx.x + gridDim.x, ...; `sub` steps per item.
struct Cursor {
    long long item;
    int sub;
};
__device__ __forceinline__ void advance(Cursor& c, int per_item) {
    if (++c.sub == per_item) {
        c.sub = 0;
        c.item += gridDim.x;
    }
}

// ---------------------------------------------------------------------------
// adjoint
// ---------------------------------------------------------------------------
template <int JB, int STAGES>
__global__ void __launch_bounds__(kThreads, 2)
    k_gemv_adj_tma(const double2* __restrict__ F, const double2* __restrict__ x, double2* __restrict__ y, int nf,
                   int nd, int nm) {
    static_assert(JB % kThreads == 0, "JB must be a multiple of the block size");
    constexpr int Q = JB / kThreads;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* stage_buf = reinterpret_cast<double2*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)STAGES * JB * sizeof(double2));
    uint64_t* empty = full + STAGES;

    const int njb = (nm + JB - 1) / JB;
    const long long items = (long long)nf * njb;
    const long long my_items = blockIdx.x < items ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long steps = my_items * nd;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();

    // producer state (thread 0 only)
    const uint64_t pol = l2_policy_evict_first();
    Cursor pc{blockIdx.x, 0};
    long long ps = 0;
    auto issue_next = [&]() {
        const int st = (int)(ps % STAGES);
        if (ps >= STAGES) mbar_wait(&empty[st], (unsigned)(((ps / STAGES) - 1) & 1));
        const int f = (int)(pc.item / njb);
        const int j0 = (int)(pc.item - (long long)f * njb) * JB;
        const unsigned bytes = (unsigned)min(JB, nm - j0) * sizeof(double2);
        mbar_expect_tx(&full[st], bytes);
        tma_load(stage_buf + (size_t)st * JB, F + ((size_t)f * nd + pc.sub) * nm + j0, bytes, &full[st], pol);
        ++ps;
        advance(pc, nd);
    };
    if (threadIdx.x == 0)
        while (ps < STAGES - 1 && ps < steps) issue_next();

    double ar[Q], ai[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) ar[q] = ai[q] = 0.0;
    const int lane = threadIdx.x & 31;
    Cursor cc{blockIdx.x, 0};
    int f = 0, j0 = 0, cols = 0;

    for (long long s = 0; s < steps; ++s) {
        if (threadIdx.x == 0 && ps < steps) issue_next();
        if (cc.sub == 0) {
            f = (int)(cc.item / njb);
            j0 = (int)(cc.item - (long long)f * njb) * JB;
            cols = min(JB, nm - j0);
        }
        const double2 w = __ldg(x + (size_t)f * nd + cc.sub);
        const int st = (int)(s % STAGES);
        mbar_wait(&full[st], (unsigned)((s / STAGES) & 1));
        const double2* row = stage_buf + (size_t)st * JB;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int jj = threadIdx.x + q * kThreads;
            if (jj < cols) {
                const double2 a = row[jj];
                ar[q] = fma(a.x, w.x, ar[q]);
                ar[q] = fma(a.y, w.y, ar[q]);
                ai[q] = fma(a.x, w.y, ai[q]);
                ai[q] = fma(-a.y, w.x, ai[q]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (cc.sub == nd - 1) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int jj = threadIdx.x + q * kThreads;
                if (jj < cols) y[(size_t)f * nm + j0 + jj] = make_double2(ar[q], ai[q]);
                ar[q] = ai[q] = 0.0;
            }
        }
        advance(cc, nd);
    }
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <int ROWS, int JC, int STAGES>
__global__ void __launch_bounds__(kThreads, 2)
    k_gemv_fwd_tma(const double2* __restrict__ F, const double2* __restrict__ x, double2* __restrict__ y, int nf,
                   int nd, int nm) {
    static_assert(JC == kThreads, "one column per thread per chunk");
    constexpr int STAGE_ELEMS = (ROWS + 1) * JC;  // ROWS F-hat row segments + the m-hat chunk
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2* stage_buf = reinterpret_cast<double2*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)STAGES * STAGE_ELEMS * sizeof(double2));
    uint64_t* empty = full + STAGES;
    double* red = reinterpret_cast<double*>(empty + STAGES);  // [kWarps][ROWS][2]

    const int nrb = (nd + ROWS - 1) / ROWS;
    const int nch = (nm + JC - 1) / JC;
    const long long items = (long long)nf * nrb;
    const long long my_items = blockIdx.x < items ? (items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long steps = my_items * nch;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();

    const uint64_t pol_f = l2_policy_evict_first();
    const uint64_t pol_x = l2_policy_evict_last();
    Cursor pc{blockIdx.x, 0};
    long long ps = 0;
    auto issue_next = [&]() {
        const int st = (int)(ps % STAGES);
        if (ps >= STAGES) mbar_wait(&empty[st], (unsigned)(((ps / STAGES) - 1) & 1));
        const int f = (int)(pc.item / nrb);
        const int i0 = (int)(pc.item - (long long)f * nrb) * ROWS;
        const int nr = min(ROWS, nd - i0);
        const int j0 = pc.sub * JC;
        const unsigned seg = (unsigned)min(JC, nm - j0) * sizeof(double2);
        mbar_expect_tx(&full[st], seg * (nr + 1));
        double2* dst = stage_buf + (size_t)st * STAGE_ELEMS;
        tma_load(dst + ROWS * JC, x + (size_t)f * nm + j0, seg, &full[st], pol_x);
        for (int r = 0; r < nr; ++r)
            tma_load(dst + r * JC, F + ((size_t)f * nd + i0 + r) * nm + j0, seg, &full[st], pol_f);
        ++ps;
        advance(pc, nch);
    };
    if (threadIdx.x == 0)
        while (ps < STAGES - 1 && ps < steps) issue_next();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    double ar[ROWS], ai[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) ar[r] = ai[r] = 0.0;
    Cursor cc{blockIdx.x, 0};
    int f = 0, i0 = 0, nr = 0;

    for (long long s = 0; s < steps; ++s) {
        if (threadIdx.x == 0 && ps < steps) issue_next();
        if (cc.sub == 0) {
            f = (int)(cc.item / nrb);
            i0 = (int)(cc.item - (long long)f * nrb) * ROWS;
            nr = min(ROWS, nd - i0);
        }
        const int cols = min(JC, nm - cc.sub * JC);
        const int st = (int)(s % STAGES);
        mbar_wait(&full[st], (unsigned)((s / STAGES) & 1));
        const double2* src = stage_buf + (size_t)st * STAGE_ELEMS;
        if (threadIdx.x < cols) {
            const double2 xv = src[ROWS * JC + threadIdx.x];
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                if (r < nr) {
                    const double2 a = src[r * JC + threadIdx.x];
                    ar[r] = fma(a.x, xv.x, ar[r]);
                    ar[r] = fma(-a.y, xv.y, ar[r]);
                    ai[r] = fma(a.x, xv.y, ai[r]);
                    ai[r] = fma(a.y, xv.x, ai[r]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (cc.sub == nch - 1) {
            // fixed-order block reduction of the ROWS partial dots
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
                    ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
                }
                if (lane == 0) {
                    red[(warp * ROWS + r) * 2 + 0] = ar[r];
                    red[(warp * ROWS + r) * 2 + 1] = ai[r];
                }
                ar[r] = ai[r] = 0.0;
            }
            __syncthreads();
            if (threadIdx.x < nr) {
                double sr = 0.0, si = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {
                    sr += red[(w * ROWS + threadIdx.x) * 2 + 0];
                    si += red[(w * ROWS + threadIdx.x) * 2 + 1];
                }
                y[(size_t)f * nd + i0 + threadIdx.x] = make_double2(sr, si);
            }
            __syncthreads();
        }
        advance(cc, nch);
    }
}

int sm_count_tma() {
    static int count = [] {
        int dev = 0, c = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
        return c;
    }();
    return count;
}

}  // namespace

cudaError_t launch_gemv_adj_tma(const double2* F, const double2* x, double2* y, int nf, int nd, int nm,
                                cudaStream_t stream) {
    constexpr int JB = 1024, STAGES = 6;
    const size_t smem = (size_t)STAGES * JB * sizeof(double2) + 2 * STAGES * sizeof(uint64_t);
    auto kern = k_gemv_adj_tma<JB, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long items = (long long)nf * ((nm + JB - 1) / JB);
    const int grid = (int)(items < 2 * sm_count_tma() ? items : 2 * sm_count_tma());
    kern<<<grid, kThreads, smem, stream>>>(F, x, y, nf, nd, nm);
    return cudaGetLastError();
}

cudaError_t launch_gemv_fwd_tma(const double2* F, const double2* x, double2* y, int nf, int nd, int nm,
                                cudaStream_t stream) {
    constexpr int ROWS = 8, JC = kThreads, STAGES = 3;
    const size_t smem = (size_t)STAGES * (ROWS + 1) * JC * sizeof(double2) + 2 * STAGES * sizeof(uint64_t) +
                        (size_t)kWarps * ROWS * 2 * sizeof(double);
    auto kern = k_gemv_fwd_tma<ROWS, JC, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long items = (long long)nf * ((nd + ROWS - 1) / ROWS);
    const int grid = (int)(items < 2 * sm_count_tma() ? items : 2 * sm_count_tma());
    kern<<<grid, kThreads, smem, stream>>>(F, x, y, nf, nd, nm);
    return cudaGetLastError();
}

}  // namespace btg
