// sm_100a kernels of the FFT block-Toeplitz matvec.
//
//  k_r2c       K1/K5: pad + R2C along time + transpose to frequency-major,
//              fused (reference: pad_and_transform + reorder_in,
//              block_operator.cpp:54-80,231-236, and setup :178-205)
//  k_c2r       K9: reorder_out + C2R + unpad (+ Gamma^-1, + alpha R v),
//              fused (block_operator.cpp:83-121,261-268; inverse.cpp:78-91)
//  k_gemv_fwd  K7 forward apply, d_f = F_f m_f (block_operator.cpp:239-259)
//  k_gemv_adj  K7 adjoint apply, m_f = F_f^H d_f (block_operator.cpp:296-317)
//
// The Fourier-space step is a pure HBM stream over F-hat (arithmetic
// intensity 0.5 flop/B in FP64): every F-hat element is read exactly once
// with 16-byte non-coherent loads that bypass L1 and carry an L2 evict-first
// policy, so the reused vector slices (m-hat_f, d-hat_f) stay L2-resident.
// All reductions have a fixed order: results are bit-identical run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "btg_fft.cuh"
#include "btg_kernels.cuh"

namespace btg {
namespace {

constexpr int kThreads = 256;
constexpr int kFwdWarpMaxCols = 8192;  // host-pipeline chunks up to this width: measured e2e F 8.63 -> 8.26 ms (4096 -> 8192)
constexpr int kMaxGridY = 65535;        // frequency batches per launch (grid.y limit)  // forward GEMV rows up to this length: warp-per-row kernel

// ---------------------------------------------------------------------------
// streaming loads of F-hat
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <typename TF, int VEC>
struct FLoad;

template <>
struct FLoad<double2, 1> {
    // raw (unconverted) register form of one load, converted at the FMA
    using Raw = double2;
    __device__ __forceinline__ static void load_raw(const double2* p, uint64_t pol, Raw& r) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
            : "=d"(r.x), "=d"(r.y)
            : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double2 get(const Raw& r, int) { return r; }
    __device__ __forceinline__ static void load(const double2* p, uint64_t pol, double2* out) {
        double2 r;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
            : "=d"(r.x), "=d"(r.y)
            : "l"(p), "l"(pol));
        out[0] = r;
    }
    __device__ __forceinline__ static double2 scalar(const double2* p) { return __ldg(p); }
};

// Two adjacent FP64 complex in ONE 32-byte load (LDG.E.256 on sm_100a)
struct Dbl4 {
    double a, b, c, d;
};
template <>
struct FLoad<double2, 2> {
    using Raw = Dbl4;
    __device__ __forceinline__ static void load_raw(const double2* p, uint64_t pol, Raw& r) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
            : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d)
            : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double2 get(const Raw& r, int v) {
        return v == 0 ? make_double2(r.a, r.b) : make_double2(r.c, r.d);
    }
    __device__ __forceinline__ static void load(const double2* p, uint64_t pol, double2* out) {
        Raw r;
        load_raw(p, pol, r);
        out[0] = make_double2(r.a, r.b);
        out[1] = make_double2(r.c, r.d);
    }
    __device__ __forceinline__ static double2 scalar(const double2* p) { return __ldg(p); }
};

template <>
struct FLoad<float2, 1> {
    using Raw = float2;
    __device__ __forceinline__ static void load_raw(const float2* p, uint64_t pol, Raw& r) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
            : "=f"(r.x), "=f"(r.y)
            : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double2 get(const Raw& r, int) { return make_double2(r.x, r.y); }
    __device__ __forceinline__ static void load(const float2* p, uint64_t pol, double2* out) {
        float x, y;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
            : "=f"(x), "=f"(y)
            : "l"(p), "l"(pol));
        out[0] = make_double2(x, y);
    }
    __device__ __forceinline__ static double2 scalar(const float2* p) {
        const float2 v = __ldg(p);
        return make_double2(v.x, v.y);
    }
};

template <>
struct FLoad<float2, 2> {
    using Raw = float4;
    __device__ __forceinline__ static void load_raw(const float2* p, uint64_t pol, Raw& r) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
            : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
            : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double2 get(const Raw& r, int v) {
        return v == 0 ? make_double2(r.x, r.y) : make_double2(r.z, r.w);
    }
    __device__ __forceinline__ static void load(const float2* p, uint64_t pol, double2* out) {
        float a, b, c, d;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
            : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
            : "l"(p), "l"(pol));
        out[0] = make_double2(a, b);
        out[1] = make_double2(c, d);
    }
    __device__ __forceinline__ static double2 scalar(const float2* p) {
        const float2 v = __ldg(p);
        return make_double2(v.x, v.y);
    }
};

// Four adjacent FP32 complex in ONE 32-byte load (LDG.E.256 on sm_100a)
struct Flt8 {
    float v[8];
};
template <>
struct FLoad<float2, 4> {
    using Raw = Flt8;
    __device__ __forceinline__ static void load_raw(const float2* p, uint64_t pol, Raw& r) {
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
            : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
              "=f"(r.v[7])
            : "l"(p), "l"(pol));
    }
    __device__ __forceinline__ static double2 get(const Raw& r, int v) {
        return make_double2(r.v[2 * v], r.v[2 * v + 1]);
    }
    __device__ __forceinline__ static void load(const float2* p, uint64_t pol, double2* out) {
        Raw r;
        load_raw(p, pol, r);
#pragma unroll
        for (int v = 0; v < 4; ++v) out[v] = make_double2(r.v[2 * v], r.v[2 * v + 1]);
    }
    __device__ __forceinline__ static double2 scalar(const float2* p) {
        const float2 v = __ldg(p);
        return make_double2(v.x, v.y);
    }
};

// acc += a * b
__device__ __forceinline__ void cmac(double& re, double& im, double2 a, double2 b) {
    re = fma(a.x, b.x, re);
    re = fma(-a.y, b.y, re);
    im = fma(a.x, b.y, im);
    im = fma(a.y, b.x, im);
}
// acc += conj(a) * b
__device__ __forceinline__ void cmac_conj(double& re, double& im, double2 a, double2 b) {
    re = fma(a.x, b.x, re);
    re = fma(a.y, b.y, re);
    im = fma(a.x, b.y, im);
    im = fma(-a.y, b.x, im);
}

template <typename T>
__device__ __forceinline__ T to_out(double2 v);
template <>
__device__ __forceinline__ double2 to_out<double2>(double2 v) { return v; }
template <>
__device__ __forceinline__ float2 to_out<float2>(double2 v) {
    return make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
}

// ---------------------------------------------------------------------------
// K1/K5: fused pad + R2C + frequency-major store
// ---------------------------------------------------------------------------
template <typename TOut>
__global__ void __launch_bounds__(kThreads) k_r2c(const double* __restrict__ in, long long in_cs,
                                                  long long in_ts, TOut* __restrict__ out,
                                                  long long out_fs, long long out_cs, int channels,
                                                  int nt, FftPlanDev plan, int batch,
                                                  double2* __restrict__ gwork) {
    // gwork != nullptr: the ping-pong buffers live in a per-CTA global slice
    // (horizons whose 2-buffer transform exceeds shared memory; setup only)
    // and the CTAs loop over channel groups.
    extern __shared__ double2 smem[];
    const int n = plan.n;  // == nt
    const int cs = fft_channel_stride(n);
    double2* buf_a = gwork ? gwork + (size_t)blockIdx.x * 2 * batch * cs : smem;
    double2* buf_b = buf_a + (size_t)batch * cs;
    const int len = 2 * n;  // padded real length
    double* ad = reinterpret_cast<double*>(buf_a);
    for (int c0 = blockIdx.x * batch; c0 < channels; c0 += gridDim.x * batch) {
    const int nb = min(batch, channels - c0);

    // Load: z[n] = x[2n] + i x[2n+1] is the real sequence itself viewed as
    // interleaved complex, so sample t of channel b goes to double 2*cs*b + t.
    if (in_ts == 1) {  // SOTI rows: time contiguous
        for (int u = threadIdx.x; u < nb * len; u += blockDim.x) {
            const int b = u / len;
            const int t = u - b * len;
            ad[2 * cs * b + t] = t < nt ? __ldg(in + (long long)(c0 + b) * in_cs + t) : 0.0;
        }
    } else {  // TOSI: channels contiguous
        for (int u = threadIdx.x; u < nb * len; u += blockDim.x) {
            const int t = u / nb;
            const int b = u - t * nb;
            ad[2 * cs * b + t] = t < nt ? __ldg(in + (long long)(c0 + b) * in_cs + t * in_ts) : 0.0;
        }
    }
    __syncthreads();
    const double2* z = fft_smem<-1>(buf_a, buf_b, nb, cs, plan);

    // Split: X_k = 1/2 (Z_k + conj Z_{n-k}) - i/2 W_{2n}^k (Z_k - conj Z_{n-k}), k = 0..n.
    for (int u = threadIdx.x; u < nb * (n + 1); u += blockDim.x) {
        const int k = u / nb;
        const int b = u - k * nb;
        const double2 zk = z[b * cs + (k == n ? 0 : k)];
        const double2 zn = cconj(z[b * cs + (k == 0 ? 0 : n - k)]);
        const double2 a = cadd(zk, zn);
        const double2 w = __ldg(plan.post + k);
        const double2 wb = cmul(w, csub(zk, zn));
        const double2 x = make_double2(0.5 * (a.x + wb.y), 0.5 * (a.y - wb.x));
        out[(long long)k * out_fs + (long long)(c0 + b) * out_cs] = to_out<TOut>(x);
    }
    __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K9: fused frequency-major load + C2R + unpad + epilogue
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_c2r(const double2* __restrict__ in, long long in_fs,
                                                  long long in_cs, double* __restrict__ out,
                                                  long long out_cs, int channels, int nt,
                                                  FftPlanDev plan, int batch, C2REpilogue epi,
                                                  double2* __restrict__ gwork) {
    extern __shared__ double2 smem[];
    const int n = plan.n;
    const int cs = fft_channel_stride(n);
    double2* buf_a = gwork ? gwork + (size_t)blockIdx.x * 2 * batch * cs : smem;
    double2* buf_b = buf_a + (size_t)batch * cs;
    for (int c0 = blockIdx.x * batch; c0 < channels; c0 += gridDim.x * batch) {
    const int nb = min(batch, channels - c0);

    for (int u = threadIdx.x; u < nb * (n + 1); u += blockDim.x) {
        const int k = u / nb;
        const int b = u - k * nb;
        buf_a[b * cs + k] = __ldg(in + (long long)k * in_fs + (long long)(c0 + b) * in_cs);
    }
    __syncthreads();
    // Z_k = (1/2n) [ (X_k + conj X_{n-k}) + i conj(W_{2n}^k) (X_k - conj X_{n-k}) ], k < n
    const double inv_len = 0.5 / static_cast<double>(n);
    for (int u = threadIdx.x; u < nb * n; u += blockDim.x) {
        const int b = u / n;
        const int k = u - b * n;
        const double2 xk = buf_a[b * cs + k];
        const double2 xn = cconj(buf_a[b * cs + n - k]);
        const double2 e = cadd(xk, xn);
        const double2 o = cmul(csub(xk, xn), cconj(__ldg(plan.post + k)));
        buf_b[b * cs + k] = make_double2(inv_len * (e.x - o.y), inv_len * (e.y + o.x));
    }
    __syncthreads();
    const double2* z = fft_smem<+1>(buf_b, buf_a, nb, cs, plan);
    const double* zd = reinterpret_cast<const double*>(z);

    for (int u = threadIdx.x; u < nb * nt; u += blockDim.x) {
        const int b = u / nt;
        const int t = u - b * nt;
        const int c = c0 + b;
        double y = zd[2 * cs * b + t];
        if (epi.gamma_mode == 1) {
            y *= __ldg(epi.gamma + (c % epi.gamma_dim));
        } else if (epi.gamma_mode == 2) {
            y *= __ldg(epi.gamma + (long long)(c % epi.gamma_dim) * nt + t);
        }
        const long long o = (long long)c * out_cs + t;
        if (epi.v) {
            const double* vr = epi.v + (long long)c * out_cs;
            double r = vr[t];
            if (epi.reg_kind == 1) {
                r = 2.0 * r;
                if (t > 0) r -= vr[t - 1];
                if (t + 1 < nt) r -= vr[t + 1];
            }
            y += epi.alpha * r;
        }
        out[o] = y;
    }
    __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K7 forward: one CTA = ROWS rows of one frequency, full sweep over j.
// ---------------------------------------------------------------------------
template <typename TF, int VEC, int ROWS, int UNR>
__global__ void __launch_bounds__(kThreads, 2)
    k_gemv_fwd(const TF* __restrict__ F, const double2* __restrict__ x, double2* __restrict__ y,
               int nd, int ld, int j0, int nm, int accumulate) {
    // columns [j0, j0 + nm) of rows of length ld; accumulate: y += (column-chunk pipelines)
    const int f = blockIdx.y;
    const int i0 = blockIdx.x * ROWS;
    const int nr = min(ROWS, nd - i0);
    const TF* fb = F + ((size_t)f * nd + i0) * ld + j0;
    const double2* xf = x + (size_t)f * ld + j0;
    const uint64_t pol = evict_first_policy();

    double ar[ROWS], ai[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) ar[r] = ai[r] = 0.0;

    constexpr int kStep = kThreads * VEC;
    int j = threadIdx.x * VEC;
    for (; j + (UNR - 1) * kStep + VEC <= nm; j += UNR * kStep) {
        double2 xv[UNR][VEC];
        typename FLoad<TF, VEC>::Raw fv[UNR][ROWS];  // unconverted: FP32 stays 4 B / value in registers
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int v = 0; v < VEC; ++v) xv[u][v] = __ldg(xf + j + u * kStep + v);
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                if (r < nr) {
                    FLoad<TF, VEC>::load_raw(fb + (size_t)r * ld + j + u * kStep, pol, fv[u][r]);
                } else {
                    fv[u][r] = {};
                }
            }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int r = 0; r < ROWS; ++r)
#pragma unroll
                for (int v = 0; v < VEC; ++v) cmac(ar[r], ai[r], FLoad<TF, VEC>::get(fv[u][r], v), xv[u][v]);
    }
    for (; j < nm; j += kStep) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            if (j + v < nm) {
                const double2 xv = __ldg(xf + j + v);
#pragma unroll
                for (int r = 0; r < ROWS; ++r)
                    if (r < nr) cmac(ar[r], ai[r], FLoad<TF, VEC>::scalar(fb + (size_t)r * ld + j + v), xv);
            }
        }
    }

    // Fixed-order block reduction: xor-butterfly within warps, then warps in order.
    __shared__ double red[kThreads / 32][ROWS][2];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
            ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
        }
        if (lane == 0) {
            red[warp][r][0] = ar[r];
            red[warp][r][1] = ai[r];
        }
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        double sr = 0.0, si = 0.0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            sr += red[w][threadIdx.x][0];
            si += red[w][threadIdx.x][1];
        }
        double2* yo = y + (size_t)f * nd + i0 + threadIdx.x;
        if (accumulate) {
            const double2 prev = *yo;
            sr = prev.x + sr;
            si = prev.y + si;
        }
        *yo = make_double2(sr, si);
    }
}

// ---------------------------------------------------------------------------
// K7 forward, short rows (N_m up to a few thousand, e.g. the paper's N_t=10000,
// N_m=800 runs): one warp = RPW consecutive rows of the flattened (f, i) row
// space, lanes stride the columns, warp-shuffle reduction only — no CTA
// barrier, so a short row costs no block-wide drain. Fixed order: deterministic.
// ---------------------------------------------------------------------------
template <typename TF, int VEC, int RPW, int UNR>
__global__ void __launch_bounds__(kThreads, 2)
    k_gemv_fwd_warp(const TF* __restrict__ F, const double2* __restrict__ x, double2* __restrict__ y,
                    long long rows, int nd, int ld, int j0, int nm, int accumulate) {
    const int lane = threadIdx.x & 31;
    const long long row0 = ((long long)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * RPW;
    if (row0 >= rows) return;
    const uint64_t pol = evict_first_policy();
    const TF* fr[RPW];
    const double2* xr[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const long long g = min(row0 + r, rows - 1);  // clamped rows are computed, not stored
        fr[r] = F + g * ld + j0;
        xr[r] = x + (g / nd) * ld + j0;
    }
    double ar[RPW], ai[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) ar[r] = ai[r] = 0.0;

    constexpr int kStep = 32 * VEC;
    int j = lane * VEC;
    for (; j + (UNR - 1) * kStep + VEC <= nm; j += UNR * kStep) {
        typename FLoad<TF, VEC>::Raw fv[UNR][RPW];
        double2 xv[UNR][RPW][VEC];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                FLoad<TF, VEC>::load_raw(fr[r] + j + u * kStep, pol, fv[u][r]);
#pragma unroll
                for (int v = 0; v < VEC; ++v) xv[u][r][v] = __ldg(xr[r] + j + u * kStep + v);
            }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
                for (int v = 0; v < VEC; ++v) cmac(ar[r], ai[r], FLoad<TF, VEC>::get(fv[u][r], v), xv[u][r][v]);
    }
    for (; j < nm; j += kStep) {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
            if (j + v < nm) {
#pragma unroll
                for (int r = 0; r < RPW; ++r)
                    cmac(ar[r], ai[r], FLoad<TF, VEC>::scalar(fr[r] + j + v), __ldg(xr[r] + j + v));
            }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
            ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
        }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        if (lane == r && row0 + r < rows) {
            double2* yo = y + row0 + r;
            double sr = ar[r], si = ai[r];
            if (accumulate) {
                const double2 prev = *yo;
                sr = prev.x + sr;
                si = prev.y + si;
            }
            *yo = make_double2(sr, si);
        }
    }
}

// ---------------------------------------------------------------------------
// K7 adjoint: one thread = JPT*VEC columns of one frequency, loop over rows
// i ascending (the reference's accumulation order, block_operator.cpp:306-310).
// ---------------------------------------------------------------------------
template <typename TF, int VEC, int JPT, int UNR, bool kSmemD>
__global__ void __launch_bounds__(kThreads, 2)
    k_gemv_adj(const TF* __restrict__ F, const double2* __restrict__ x, double2* __restrict__ y,
               int nd, int ld, int j0, int nm) {
    // columns [j0, j0 + nm) of rows of length ld (column-chunk pipelines)
    extern __shared__ double2 sd[];
    const int f = blockIdx.y;
    const double2* xf = x + (size_t)f * nd;
    if constexpr (kSmemD) {
        for (int i = threadIdx.x; i < nd; i += kThreads) sd[i] = xf[i];
        __syncthreads();
    }
    const double2* dsrc = kSmemD ? sd : xf;
    const TF* ff = F + (size_t)f * nd * ld + j0;
    double2* yf = y + (size_t)f * ld + j0;
    const uint64_t pol = evict_first_policy();
    constexpr int kStep = kThreads * VEC;
    const int jb = blockIdx.x * (kStep * JPT) + threadIdx.x * VEC;

    double ar[JPT][VEC], ai[JPT][VEC];
#pragma unroll
    for (int q = 0; q < JPT; ++q)
#pragma unroll
        for (int v = 0; v < VEC; ++v) ar[q][v] = ai[q][v] = 0.0;

    if (jb + (JPT - 1) * kStep + VEC <= nm) {
        int i = 0;
        for (; i + UNR <= nd; i += UNR) {
            typename FLoad<TF, VEC>::Raw fv[UNR][JPT];
#pragma unroll
            for (int u = 0; u < UNR; ++u)
#pragma unroll
                for (int q = 0; q < JPT; ++q)
                    FLoad<TF, VEC>::load_raw(ff + (size_t)(i + u) * ld + jb + q * kStep, pol, fv[u][q]);
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const double2 w = dsrc[i + u];
#pragma unroll
                for (int q = 0; q < JPT; ++q)
#pragma unroll
                    for (int v = 0; v < VEC; ++v) cmac_conj(ar[q][v], ai[q][v], FLoad<TF, VEC>::get(fv[u][q], v), w);
            }
        }
        if (i < nd) {
            // remainder rows (< UNR): one batch of predicated loads, all in flight
            // together, then the same i-ascending accumulation
            typename FLoad<TF, VEC>::Raw fv[UNR][JPT];
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                if (i + u < nd)
#pragma unroll
                    for (int q = 0; q < JPT; ++q)
                        FLoad<TF, VEC>::load_raw(ff + (size_t)(i + u) * ld + jb + q * kStep, pol, fv[u][q]);
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                if (i + u < nd) {
                    const double2 w = dsrc[i + u];
#pragma unroll
                    for (int q = 0; q < JPT; ++q)
#pragma unroll
                        for (int v = 0; v < VEC; ++v)
                            cmac_conj(ar[q][v], ai[q][v], FLoad<TF, VEC>::get(fv[u][q], v), w);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < JPT; ++q)
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                yf[jb + q * kStep + v] = make_double2(ar[q][v], ai[q][v]);
    } else {
        for (int i = 0; i < nd; ++i) {
            const double2 w = dsrc[i];
#pragma unroll
            for (int q = 0; q < JPT; ++q)
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    const int j = jb + q * kStep + v;
                    if (j < nm)
                        cmac_conj(ar[q][v], ai[q][v], FLoad<TF, VEC>::scalar(ff + (size_t)i * ld + j), w);
                }
        }
#pragma unroll
        for (int q = 0; q < JPT; ++q)
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const int j = jb + q * kStep + v;
                if (j < nm) yf[j] = make_double2(ar[q][v], ai[q][v]);
            }
    }
}

// ---------------------------------------------------------------------------
// indexable synthetic inputs
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_fill_uniform(double* __restrict__ out, size_t nb, size_t nc, size_t n, uint64_t seed,
                               uint64_t offset, uint64_t sa, uint64_t sb, double lo, double span) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
         k += (size_t)gridDim.x * blockDim.x) {
        const size_t c = k % nc;
        const size_t ab = k / nc;
        const size_t b = ab % nb;
        const size_t a = ab / nb;
        const uint64_t u = splitmix64(seed ^ (offset + a * sa + b * sb + c));
        out[k] = lo + span * (static_cast<double>(u >> 11) * 0x1.0p-53);
    }
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int sm_count() {
    static int count = [] {
        int dev = 0, c = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
        return c;
    }();
    return count;
}

}  // namespace

size_t fft_smem_bytes(int n, int batch) {
    return 2ull * (size_t)batch * (size_t)fft_channel_stride(n) * sizeof(double2);
}

int fft_batch(int n, size_t smem_budget, int want) {
    const size_t per = fft_smem_bytes(n, 1);
    int b = static_cast<int>(smem_budget / per);
    if (b < 1) return 0;
    return std::min(b, want);
}

template <typename TOut>
cudaError_t launch_r2c(const double* in, long long in_cs, long long in_ts, TOut* out,
                       long long out_fs, long long out_cs, int channels, int nt,
                       const FftPlanDev& plan, int batch, cudaStream_t stream, const FftScratch& gs) {
    if (channels <= 0) return cudaSuccess;
    const size_t smem = gs.buf ? 0 : fft_smem_bytes(plan.n, batch);
    cudaError_t e = set_smem(k_r2c<TOut>, smem);
    if (e != cudaSuccess) return e;
    int grid = (channels + batch - 1) / batch;
    if (gs.buf) grid = std::min(grid, gs.ctas);
    k_r2c<TOut><<<grid, kThreads, smem, stream>>>(in, in_cs, in_ts, out, out_fs, out_cs, channels,
                                                  nt, plan, batch, gs.buf);
    return cudaGetLastError();
}

template cudaError_t launch_r2c<double2>(const double*, long long, long long, double2*, long long,
                                         long long, int, int, const FftPlanDev&, int, cudaStream_t,
                                         const FftScratch&);
template cudaError_t launch_r2c<float2>(const double*, long long, long long, float2*, long long,
                                        long long, int, int, const FftPlanDev&, int, cudaStream_t,
                                        const FftScratch&);

cudaError_t launch_c2r(const double2* in, long long in_fs, long long in_cs, double* out,
                       long long out_cs, int channels, int nt, const FftPlanDev& plan, int batch,
                       const C2REpilogue& epi, cudaStream_t stream, const FftScratch& gs) {
    if (channels <= 0) return cudaSuccess;
    const size_t smem = gs.buf ? 0 : fft_smem_bytes(plan.n, batch);
    cudaError_t e = set_smem(k_c2r, smem);
    if (e != cudaSuccess) return e;
    int grid = (channels + batch - 1) / batch;
    if (gs.buf) grid = std::min(grid, gs.ctas);
    k_c2r<<<grid, kThreads, smem, stream>>>(in, in_fs, in_cs, out, out_cs, channels, nt, plan,
                                            batch, epi, gs.buf);
    return cudaGetLastError();
}

template <typename TF>
cudaError_t launch_gemv_fwd_range(const TF* F, const double2* x, double2* y, int nf, int nd, int nm, int j0,
                                  int nj, bool accumulate, cudaStream_t stream) {
    static const int warp_max = [] {
        const char* e = std::getenv("BTG_FWD_WARP_MAX");
        return e ? std::atoi(e) : kFwdWarpMaxCols;
    }();
    if (nj <= warp_max) {
        constexpr int kRpw = 4;
        const long long rows = (long long)nf * nd;
        const long long warps = (rows + kRpw - 1) / kRpw;
        const unsigned grid = (unsigned)((warps + kThreads / 32 - 1) / (kThreads / 32));
        if constexpr (sizeof(TF) == 8) {
            if ((nm & 1) == 0 && (j0 & 1) == 0) {
                k_gemv_fwd_warp<TF, 2, kRpw, 2><<<grid, kThreads, 0, stream>>>(F, x, y, rows, nd, nm, j0, nj,
                                                                               accumulate);
                return cudaGetLastError();
            }
        }
        k_gemv_fwd_warp<TF, 1, kRpw, 4><<<grid, kThreads, 0, stream>>>(F, x, y, rows, nd, nm, j0, nj,
                                                                       accumulate);
        return cudaGetLastError();
    }
    constexpr int kRows = 8;
    for (int f0 = 0; f0 < nf; f0 += kMaxGridY) {  // grid.y limit: long horizons go in frequency batches
        const int nb = std::min(kMaxGridY, nf - f0);
        const TF* Fb = F + (size_t)f0 * nd * nm;
        const double2* xb = x + (size_t)f0 * nm;
        double2* yb = y + (size_t)f0 * nd;
        dim3 grid((nd + kRows - 1) / kRows, nb);
        if constexpr (sizeof(TF) == 8) {
            if ((nm & 1) == 0 && (j0 & 1) == 0) {
                // FP32 pairs: 16-byte loads of two complex, 4 rows x 2 unrolled steps per
                // thread (8 rows x 2 spills; measured 3.99 vs 9.98 ms at configs[1])
                if ((nm & 3) == 0 && (j0 & 3) == 0) {
                    // four adjacent complex per 32-byte load, 4 rows in flight: FP32
                    // configs[1] forward 4.05 -> 3.92 ms (4 x 2 / 2 x 4 / 2 x 2 of these
                    // spill or lose)
                    dim3 g((nd + 3) / 4, nb);
                    k_gemv_fwd<TF, 4, 4, 1><<<g, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj, accumulate);
                    continue;
                }
                dim3 g4((nd + 3) / 4, nb);
                k_gemv_fwd<TF, 2, 4, 2><<<g4, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj, accumulate);
                continue;
            }
        }
        // 4 rows x 4 unrolled column steps per thread (16 loads of 16 B in flight): measured
        // against 8 x 2 (round 1), 16 x 1, 12 x 1, 2 x 8, 4 x 6, 4 x 3 — configs[1] 7.47 ->
        // 7.36 ms, configs[2] 11.40 -> 10.81 ms, configs[4] shard 19.8 -> 19.0 ms. The
        // per-thread j order (ascending) and the block reduction are unchanged, so the
        // results are bit-identical. BTG_FWD_SHAPE=1: the 8 x 2 kernel.
        static const bool rows8 = [] {
            const char* e = std::getenv("BTG_FWD_SHAPE");
            return e && *e == '1';
        }();
        if constexpr (sizeof(TF) == 16) {
            // FP64: two adjacent complex per 32-byte load (LDG.E.256), 2 rows x 4 steps
            // in flight — configs[1] 7.36 -> 7.32 ms, configs[2] 10.81 -> 10.69 ms over
            // the 16-byte 4 x 4 kernel (which odd column offsets still take)
            if (!rows8 && (nm & 1) == 0 && (j0 & 1) == 0) {
                dim3 g2((nd + 1) / 2, nb);
                k_gemv_fwd<TF, 2, 2, 4><<<g2, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj, accumulate);
                continue;
            }
        }
        if (rows8) {
            k_gemv_fwd<TF, 1, kRows, 2><<<grid, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj, accumulate);
        } else {
            dim3 g4((nd + 3) / 4, nb);
            k_gemv_fwd<TF, 1, 4, 4><<<g4, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj, accumulate);
        }
    }
    return cudaGetLastError();
}

template <typename TF>
cudaError_t launch_gemv_fwd(const TF* F, const double2* x, double2* y, int nf, int nd, int nm,
                            cudaStream_t stream) {
    return launch_gemv_fwd_range(F, x, y, nf, nd, nm, 0, nm, false, stream);
}

template <typename TF, int VEC>
cudaError_t launch_adj_vec(const TF* F, const double2* x, double2* y, int nf, int nd, int nm, int j0, int nj,
                           cudaStream_t stream) {
    constexpr int kJpt = ((sizeof(TF) == 16 && VEC == 2) || VEC == 4) ? 1 : 2;
    constexpr int kUnr = 8;
    const size_t smem = (size_t)nd * sizeof(double2);
    // Default: read d-hat_f through the read-only path (a warp-uniform broadcast
    // that hits L1), so a CTA starts streaming F-hat without a fill + barrier.
    static const bool use_smem = std::getenv("BTG_ADJ_SMEM") != nullptr;
    const bool smem_d = use_smem && smem <= 96 * 1024;
    if (smem_d) {
        cudaError_t e = set_smem(k_gemv_adj<TF, VEC, kJpt, kUnr, true>, smem);
        if (e != cudaSuccess) return e;
    }
    for (int f0 = 0; f0 < nf; f0 += kMaxGridY) {  // grid.y limit: long horizons go in frequency batches
        const int nb = std::min(kMaxGridY, nf - f0);
        const TF* Fb = F + (size_t)f0 * nd * nm;
        const double2* xb = x + (size_t)f0 * nd;
        double2* yb = y + (size_t)f0 * nm;
        dim3 grid((nj + kThreads * VEC * kJpt - 1) / (kThreads * VEC * kJpt), nb);
        if (smem_d)
            k_gemv_adj<TF, VEC, kJpt, kUnr, true><<<grid, kThreads, smem, stream>>>(Fb, xb, yb, nd, nm, j0, nj);
        else
            k_gemv_adj<TF, VEC, kJpt, kUnr, false><<<grid, kThreads, 0, stream>>>(Fb, xb, yb, nd, nm, j0, nj);
    }
    return cudaGetLastError();
}

template <typename TF>
cudaError_t launch_gemv_adj_range(const TF* F, const double2* x, double2* y, int nf, int nd, int nm, int j0,
                                  int nj, cudaStream_t stream) {
    if constexpr (sizeof(TF) == 8) {
        // four adjacent columns per thread in one 32-byte load (bit-identical: i-ascending
        // per column): FP32 configs[1] adjoint 3.98 -> 3.93 ms
        if ((nm & 3) == 0 && (j0 & 3) == 0) return launch_adj_vec<TF, 4>(F, x, y, nf, nd, nm, j0, nj, stream);
        if ((nm & 1) == 0 && (j0 & 1) == 0) return launch_adj_vec<TF, 2>(F, x, y, nf, nd, nm, j0, nj, stream);
    } else {
        // FP64: a thread's two columns adjacent and read by ONE 32-byte load (LDG.E.256);
        // same i-ascending accumulation per column, so bit-identical to the 16-byte
        // kernel (configs[1] 7.67 -> 7.62 ms, configs[2] 10.83 -> 10.75 ms)
        if ((nm & 1) == 0 && (j0 & 1) == 0) return launch_adj_vec<TF, 2>(F, x, y, nf, nd, nm, j0, nj, stream);
    }
    return launch_adj_vec<TF, 1>(F, x, y, nf, nd, nm, j0, nj, stream);
}

template <typename TF>
cudaError_t launch_gemv_adj(const TF* F, const double2* x, double2* y, int nf, int nd, int nm,
                            cudaStream_t stream) {
    return launch_gemv_adj_range(F, x, y, nf, nd, nm, 0, nm, stream);
}

#define BTG_INST_GEMV(TF)                                                                                       \
    template cudaError_t launch_gemv_fwd<TF>(const TF*, const double2*, double2*, int, int, int, cudaStream_t); \
    template cudaError_t launch_gemv_adj<TF>(const TF*, const double2*, double2*, int, int, int, cudaStream_t); \
    template cudaError_t launch_gemv_fwd_range<TF>(const TF*, const double2*, double2*, int, int, int, int, int, \
                                                   bool, cudaStream_t);                                         \
    template cudaError_t launch_gemv_adj_range<TF>(const TF*, const double2*, double2*, int, int, int, int, int, \
                                                   cudaStream_t);
BTG_INST_GEMV(double2)
BTG_INST_GEMV(float2)
#undef BTG_INST_GEMV

// TOSI slab (time outer: in[t * ts + c]) -> SOTI rows (out[c * nt + t]) through a
// 32 x 32 shared tile: both sides move 256-byte row segments. The setup's strided
// generic R2C read 48-byte segments at a 26 MB stride (605 GB/s, ncu); transposing
// first lets the vector R2C read whole rows.
__global__ void __launch_bounds__(256) k_tosi_to_soti(const double* __restrict__ in, long long ts,
                                                      double* __restrict__ out, int nt, long long cnt) {
    __shared__ double tile[32][33];
    const long long c0 = (long long)blockIdx.x * 32;
    const int t0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
        const int t = t0 + k;
        const long long c = c0 + tx;
        if (t < nt && c < cnt) tile[k][tx] = __ldcs(in + (long long)t * ts + c);
    }
    __syncthreads();
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
        const long long c = c0 + k;
        const int t = t0 + tx;
        if (t < nt && c < cnt) out[c * nt + t] = tile[tx][k];
    }
}

// FP32 F-hat setup: rows k of a frequency-major complex128 block (in[k * cnt + c])
// rounded to complex64 at out[k * out_fs + c] (the same rounding as k_r2c<float2>'s
// to_out)
__global__ void k_spec_to_f32(const double2* __restrict__ in, long long cnt, float2* __restrict__ out,
                              long long out_fs, long long total) {
    for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < total;
         u += (long long)gridDim.x * blockDim.x) {
        const long long k = u / cnt, c = u - k * cnt;
        out[k * out_fs + c] = to_out<float2>(__ldcs(in + u));
    }
}

cudaError_t launch_spec_to_f32(const double2* in, long long cnt, int nf, float2* out, long long out_fs,
                               cudaStream_t stream) {
    const long long total = cnt * (long long)nf;
    if (total <= 0) return cudaSuccess;
    const int grid = (int)std::min<long long>((total + 255) / 256, (long long)sm_count() * 16);
    k_spec_to_f32<<<grid, 256, 0, stream>>>(in, cnt, out, out_fs, total);
    return cudaGetLastError();
}

cudaError_t launch_tosi_to_soti(const double* in, long long ts, double* out, int nt, long long cnt,
                                cudaStream_t stream) {
    if (cnt <= 0 || nt <= 0) return cudaSuccess;
    const dim3 grid((unsigned)((cnt + 31) / 32), (unsigned)((nt + 31) / 32));
    k_tosi_to_soti<<<grid, 256, 0, stream>>>(in, ts, out, nt, cnt);
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform(double* out, size_t na, size_t nb, size_t nc, uint64_t seed, uint64_t offset,
                                uint64_t sa, uint64_t sb, double lo, double hi, cudaStream_t stream) {
    const size_t n = na * nb * nc;
    if (n == 0) return cudaSuccess;
    const size_t want = (n + kThreads - 1) / kThreads;
    const int grid = static_cast<int>(std::min<size_t>(want, (size_t)sm_count() * 16));
    k_fill_uniform<<<grid, kThreads, 0, stream>>>(out, nb, nc, n, seed, offset, sa, sb, lo, hi - lo);
    return cudaGetLastError();
}

}  // namespace btg

// ---------------------------------------------------------------------------
// compile-time-N vector FFTs (btg_fft_fast.cuh)
// ---------------------------------------------------------------------------
#include "btg_fft_fast.cuh"

namespace btg {
namespace {

// Channels per CTA: the plan's default, overridable with BTG_FFT_CPB (tuning).
int fft_cpb(int dflt) {
    static const int env = [] {
        const char* v = std::getenv("BTG_FFT_CPB");
        return v ? std::atoi(v) : 0;
    }();
    return env > 0 ? env : dflt;
}

// Persistent grid for the vector FFT kernels: as many CTAs as fit on the device
// at once (they loop over channel groups and prefetch the next group's inputs).
template <typename K>
int persistent_grid(K kern, int threads, size_t smem, int groups) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
    return std::max(1, std::min(groups, occ * sms));
}

template <int N, int CPB>
cudaError_t r2c_fast_nc(const double* in, long long in_cs, double2* out, long long out_fs, int channels,
                        const FastTables& tabs, cudaStream_t stream, const R2CBlockMax& bm) {
    using P = fast::FastPlan<N>;
    if (out_fs < 0 && (kSpecBlock % CPB || bm.pexp)) return cudaErrorNotSupported;
    if constexpr (P::TPC * CPB > 1024 || fast::smem_dir<N, CPB, true>() > 227 * 1024) {
        return cudaErrorNotSupported;
    } else {
        constexpr size_t smem = fast::smem_dir<N, CPB, true>();
        if constexpr (fast::UseTmaR2C<N>::value && CPB == P::CPB_R2C) {
            static const long long tma_max = [] {  // BTG_R2C_TMA_MAX: crossover override (sweeps)
                const char* v = std::getenv("BTG_R2C_TMA_MAX");
                return v && *v ? std::atoll(v) : (long long)fast::UseTmaR2C<N>::max_channels;
            }();
            // channel-blocked output: the TMA kernel at every size (524288 channels at
            // N_t = 1024: 2.55 ms vs 2.99 ms for the 3-CTA kernel; frequency-major
            // output keeps the measured crossover)
            if (channels <= tma_max || out_fs < 0) {
                constexpr size_t smem_t = fast::smem_bytes_tma<N, CPB>();
                auto kt = fast::k_r2c_tma<N, CPB>;
                cudaError_t e = set_smem(kt, smem_t);
                if (e != cudaSuccess) return e;
                if (bm.pexp && channels % CPB != 0) return cudaErrorInvalidValue;
                const int grid = persistent_grid(kt, P::TPC * CPB, smem_t, (channels + CPB - 1) / CPB);
                kt<<<grid, P::TPC * CPB, smem_t, stream>>>(in, in_cs, out, out_fs, channels, tabs, bm);
                return cudaGetLastError();
            }
        }
        auto kern = P::PF_R2C ? fast::k_r2c_pf<N, CPB> : fast::k_r2c_fast<N, CPB>;
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const int groups = (channels + CPB - 1) / CPB;
        const int grid = P::PF_R2C ? persistent_grid(kern, P::TPC * CPB, smem, groups) : groups;
        if (bm.pexp && channels % CPB != 0) return cudaErrorInvalidValue;
        kern<<<grid, P::TPC * CPB, smem, stream>>>(in, in_cs, out, out_fs, channels, tabs, bm);
        return cudaGetLastError();
    }
}

template <int N, int CPB>
cudaError_t c2r_fast_nc(const double2* in, long long in_fs, double* out, long long out_cs, int channels,
                        const FastTables& tabs, const C2REpilogue& epi, cudaStream_t stream, int* ctas) {
    using P = fast::FastPlan<N>;
    if (in_fs < 0 && kSpecBlock % CPB) return cudaErrorNotSupported;
    if constexpr (P::TPC * CPB > 1024 || fast::smem_dir<N, CPB, false>() > 227 * 1024) {
        return cudaErrorNotSupported;
    } else {
        constexpr size_t smem = fast::smem_dir<N, CPB, false>();
        if constexpr (fast::c2r_tma_ok<N, CPB>()) {
            // channel-blocked input: one bulk copy per 4-channel group (k_c2r_tma)
            if (in_fs < 0 && !std::getenv("BTG_C2R_NO_TMA") && !epi.npeers) {
                if (channels % CPB) return cudaErrorNotSupported;
                const bool light = !epi.v && epi.gamma_mode != 2;  // no per-sample operands
                const size_t smem_t =
                    light ? fast::smem_bytes_c2r_tma<N, CPB, true>() : fast::smem_bytes_c2r_tma<N, CPB, false>();
                auto kt = light ? fast::k_c2r_tma<N, CPB, true> : fast::k_c2r_tma<N, CPB, false>;
                cudaError_t e = set_smem(kt, smem_t);
                if (e != cudaSuccess) return e;
                const int grid = persistent_grid(kt, P::TPC * CPB, smem_t, channels / CPB);
                if (ctas) *ctas = grid;
                kt<<<grid, P::TPC * CPB, smem_t, stream>>>(in, in_fs, out, out_cs, channels, tabs, epi);
                return cudaGetLastError();
            }
        }
        // the grid reduce fused into the stores (epi.npeers): its own instantiation,
        // so the other C2Rs carry no peer-load code (it cost them 10-17 %)
        const bool light = !epi.v && epi.gamma_mode != 2;  // no per-sample operands
        auto kern = epi.npeers ? fast::k_c2r_fast<N, CPB, true>
                               : (P::PF_C2R ? (light ? fast::k_c2r_pf<N, CPB, true> : fast::k_c2r_pf<N, CPB, false>)
                                            : (light ? fast::k_c2r_fast<N, CPB, false, true>
                                                     : fast::k_c2r_fast<N, CPB, false, false>));
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const int groups = (channels + CPB - 1) / CPB;
        const int grid = (P::PF_C2R && !epi.npeers) ? persistent_grid(kern, P::TPC * CPB, smem, groups) : groups;
        if (ctas) *ctas = grid;
        kern<<<grid, P::TPC * CPB, smem, stream>>>(in, in_fs, out, out_cs, channels, tabs, epi);
        return cudaGetLastError();
    }
}

template <int N>
cudaError_t r2c_fast_n(const double* in, long long in_cs, double2* out, long long out_fs, int channels,
                       const FastTables& tabs, cudaStream_t stream, const R2CBlockMax& bm) {
    switch (fft_cpb(fast::FastPlan<N>::CPB_R2C)) {
        case 1: return r2c_fast_nc<N, 1>(in, in_cs, out, out_fs, channels, tabs, stream, bm);
        case 2: return r2c_fast_nc<N, 2>(in, in_cs, out, out_fs, channels, tabs, stream, bm);
        case 4: return r2c_fast_nc<N, 4>(in, in_cs, out, out_fs, channels, tabs, stream, bm);
        case 8: return r2c_fast_nc<N, 8>(in, in_cs, out, out_fs, channels, tabs, stream, bm);
        default: return r2c_fast_nc<N, fast::FastPlan<N>::CPB_R2C>(in, in_cs, out, out_fs, channels, tabs, stream,
                                                                   bm);
    }
}

template <int N>
cudaError_t c2r_fast_n(const double2* in, long long in_fs, double* out, long long out_cs, int channels,
                       const FastTables& tabs, const C2REpilogue& epi, cudaStream_t stream, int* ctas) {
    switch (fft_cpb(fast::FastPlan<N>::CPB_C2R)) {
        case 1: return c2r_fast_nc<N, 1>(in, in_fs, out, out_cs, channels, tabs, epi, stream, ctas);
        case 2: return c2r_fast_nc<N, 2>(in, in_fs, out, out_cs, channels, tabs, epi, stream, ctas);
        case 4: return c2r_fast_nc<N, 4>(in, in_fs, out, out_cs, channels, tabs, epi, stream, ctas);
        case 8: return c2r_fast_nc<N, 8>(in, in_fs, out, out_cs, channels, tabs, epi, stream, ctas);
        default: return c2r_fast_nc<N, fast::FastPlan<N>::CPB_C2R>(in, in_fs, out, out_cs, channels, tabs, epi, stream,
                                                                   ctas);
    }
}

#define BTG_FAST_SIZES(X) X(64) X(128) X(256) X(500) X(512) X(1000) X(1024) X(2000) X(2048) X(4096) X(8192) X(10000)

}  // namespace

int fast_r2c_cpb(int n) {
#define BTG_CASE(N) \
    if (n == N) return fft_cpb(fast::FastPlan<N>::CPB_R2C);
    BTG_FAST_SIZES(BTG_CASE)
#undef BTG_CASE
    return 0;
}

bool spec_blocked_ok(int n) {
#define BTG_CASE(N)                                                                                       \
    if (n == N)                                                                                           \
        return kSpecBlock % fft_cpb(fast::FastPlan<N>::CPB_R2C) == 0 && kSpecBlock % fft_cpb(fast::FastPlan<N>::CPB_C2R) == 0;
    BTG_FAST_SIZES(BTG_CASE)
#undef BTG_CASE
    return false;
}

bool fast_fft_supported(int n) {
#define BTG_CASE(N) \
    if (n == N) return true;
    BTG_FAST_SIZES(BTG_CASE)
#undef BTG_CASE
    return false;
}

int fast_fft_hi_count(int n) { return (n + fast::kTwLo - 1) / fast::kTwLo + 1; }

cudaError_t launch_r2c_vec_fast(int n, const double* in, long long in_cs, double2* out, long long out_fs,
                                int channels, const FastTables& tabs, cudaStream_t stream, const R2CBlockMax& bm) {
    if (channels <= 0) return cudaSuccess;
#define BTG_CASE(N) \
    if (n == N) return r2c_fast_n<N>(in, in_cs, out, out_fs, channels, tabs, stream, bm);
    BTG_FAST_SIZES(BTG_CASE)
#undef BTG_CASE
    return cudaErrorNotSupported;
}

cudaError_t launch_c2r_vec_fast(int n, const double2* in, long long in_fs, double* out, long long out_cs,
                                int channels, const FastTables& tabs, const C2REpilogue& epi,
                                cudaStream_t stream, int* ctas) {
    if (channels <= 0) return cudaSuccess;
#define BTG_CASE(N) \
    if (n == N) return c2r_fast_n<N>(in, in_fs, out, out_cs, channels, tabs, epi, stream, ctas);
    BTG_FAST_SIZES(BTG_CASE)
#undef BTG_CASE
    return cudaErrorNotSupported;
}

}  // namespace btg
