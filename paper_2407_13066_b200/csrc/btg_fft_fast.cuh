// Register-resident Stockham FFT for the vector transforms (K5 / K9), with the
// transform length N = N_t fixed at compile time.
//
// Per channel, TPC threads hold the data in registers; each radix-R pass loads
// its R inputs, applies the inter-pass twiddles, runs the R-point DFT in
// registers and scatters the R outputs autosorted. Passes exchange data through
// ONE in-place shared-memory buffer per channel (loads of a pass complete at a
// barrier before any thread overwrites), so a length-1024 transform costs two
// shared-memory round trips (16 x 16 x 4) instead of a read+write per pass.
//
//  r2c: pass 1 reads z[n] = (x[2n], x[2n+1]) straight from the SOTI row with
//       16-byte loads (only n < N/2 is non-zero: the zero padding prunes half
//       the first-pass inputs), the split X_k = f(Z_k, Z_{N-k}) runs on pairs
//       (k, N-k) and stores frequency-major with CPB consecutive channels per
//       frequency.
//  c2r: the pre-split builds Z from pairs (X_k, X_{N-k}) loaded
//       frequency-major; the last pass stores x[2p], x[2p+1] straight into the
//       SOTI row (only p < N/2 survives the unpad) through the epilogue.
//
// Shared-memory index p is padded to p + p/16 so the stride-R scatter of the
// first pass is bank-conflict free. Twiddles W_N^e = lo[e % 32] * hi[e / 32]
// come from two small shared tables.
#pragma once

#include <cuda_runtime.h>

#include "btg_fft.cuh"
#include "btg_kernels.cuh"

namespace btg {
namespace fast {

template <int... Rs>
struct Radices {};

// Plans: (TPC threads per channel, CPB channels per CTA, radices in pass order).
template <int N>
struct FastPlan;
template <> struct FastPlan<64>   { static constexpr int TPC = 8,   CPB = 32; using R = Radices<8, 8>; };
template <> struct FastPlan<128>  { static constexpr int TPC = 16,  CPB = 16; using R = Radices<8, 16>; };
template <> struct FastPlan<256>  { static constexpr int TPC = 16,  CPB = 16; using R = Radices<16, 16>; };
template <> struct FastPlan<500>  { static constexpr int TPC = 64,  CPB = 4;  using R = Radices<4, 5, 5, 5>; };
template <> struct FastPlan<512>  { static constexpr int TPC = 64,  CPB = 4;  using R = Radices<8, 8, 8>; };
template <> struct FastPlan<1000> { static constexpr int TPC = 128, CPB = 2;  using R = Radices<8, 5, 5, 5>; };
template <> struct FastPlan<1024> { static constexpr int TPC = 64,  CPB = 4;  using R = Radices<16, 16, 4>; };
template <> struct FastPlan<2000> { static constexpr int TPC = 128, CPB = 2;  using R = Radices<16, 5, 5, 5>; };
template <> struct FastPlan<2048> { static constexpr int TPC = 128, CPB = 2;  using R = Radices<16, 16, 8>; };
template <> struct FastPlan<4096> { static constexpr int TPC = 256, CPB = 1;  using R = Radices<16, 16, 16>; };

// Register budget: aim for 768 resident threads per SM (<= 85 registers).
template <int N, int CPB>
constexpr int kMinBlocks = (768 / (FastPlan<N>::TPC * CPB)) > 0 ? (768 / (FastPlan<N>::TPC * CPB)) : 1;

__host__ __device__ constexpr int pad_idx(int p) { return p + (p >> 4); }
__host__ __device__ constexpr int chan_stride(int n) { return pad_idx(n) + 2; }  // room for X_N in c2r
constexpr int kTwLo = 32;

template <int N>
__host__ __device__ constexpr int tw_hi_count() { return (N + kTwLo - 1) / kTwLo + 1; }

template <int N, int CPB>
__host__ __device__ constexpr size_t smem_bytes() {
    return sizeof(double2) * ((size_t)CPB * chan_stride(N) + 2 * kTwLo + 2 * tw_hi_count<N>() + 2);
}

// W^e for W = exp(SIGN * 2 pi i / n_tw) from the split table (lo[e % 32] * hi[e / 32]).
template <int SIGN>
__device__ __forceinline__ double2 tw_lookup(const double2* lo, const double2* hi, int e) {
    double2 w = cmul(lo[e & (kTwLo - 1)], hi[e >> 5]);
    if (SIGN > 0) w.y = -w.y;
    return w;
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(double2* v) {
    if constexpr (R == 2) dft2<SIGN>(v);
    else if constexpr (R == 3) dft3<SIGN>(v);
    else if constexpr (R == 4) dft4<SIGN>(v);
    else if constexpr (R == 5) dft5<SIGN>(v);
    else if constexpr (R == 8) dft8<SIGN>(v);
    else if constexpr (R == 16) {
        // 16 = 4 x 4: columns, twiddle W_16^{q r}, rows, transpose.
        double2 a[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int q = 0; q < 4; ++q) a[r][q] = v[r + 4 * q];
            dft4<SIGN>(a[r]);
        }
        constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
        constexpr double c2 = 0.70710678118654752440;
        // a[r][k] *= W_16^{r k}, W_16 = exp(SIGN 2 pi i / 16)
#pragma unroll
        for (int r = 1; r < 4; ++r)
#pragma unroll
            for (int k = 1; k < 4; ++k) {
                const int e = r * k;  // 1..9
                double2 w;
                switch (e) {
                    case 1: w = make_double2(c1, SIGN * s1); break;
                    case 2: w = make_double2(c2, SIGN * c2); break;
                    case 3: w = make_double2(s1, SIGN * c1); break;
                    case 4: w = make_double2(0.0, SIGN * 1.0); break;
                    case 6: w = make_double2(-c2, SIGN * c2); break;
                    case 9: w = make_double2(-c1, -SIGN * s1); break;
                    default: w = make_double2(1.0, 0.0); break;
                }
                a[r][k] = cmul(a[r][k], w);
            }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            double2 b[4] = {a[0][k], a[1][k], a[2][k], a[3][k]};
            dft4<SIGN>(b);
#pragma unroll
            for (int r = 0; r < 4; ++r) v[k + 4 * r] = b[r];
        }
    }
}

// Inputs of butterfly j of a radix-R pass, already twiddled: v[q] = s[j + q N/R] * W^{k q N/(NS R)}.
template <int N, int R, int NS, int SIGN>
__device__ __forceinline__ void twiddle_inputs(double2* v, int j, const double2* lo, const double2* hi) {
    if constexpr (NS > 1) {
        // One table lookup per butterfly; the powers W^{k q step}, q = 2..R-1, are
        // products of lower powers (depth log2 R, error a few ulp) instead of
        // 2 (R-1) shared-memory loads.
        const int k = j % NS;
        constexpr int step = N / (NS * R);
        double2 w[R];
        w[1] = tw_lookup<SIGN>(lo, hi, k * step);
#pragma unroll
        for (int q = 2; q < R; ++q) w[q] = cmul(w[q / 2], w[q - q / 2]);
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
    }
}

// One in-place radix-R pass over the channel buffer `s` (smem, padded).
template <int N, int TPC, int R, int NS, int SIGN>
__device__ __forceinline__ void pass_smem(double2* s, int tc, const double2* lo, const double2* hi) {
    constexpr int NB = N / R;                 // butterflies
    constexpr int BF = (NB + TPC - 1) / TPC;  // per thread
    double2 v[BF][R];
#pragma unroll
    for (int b = 0; b < BF; ++b) {
        const int j = tc + b * TPC;
        if (NB % TPC == 0 || j < NB) {
#pragma unroll
            for (int q = 0; q < R; ++q) v[b][q] = s[pad_idx(j + q * NB)];
            twiddle_inputs<N, R, NS, SIGN>(v[b], j, lo, hi);
            dft<R, SIGN>(v[b]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < BF; ++b) {
        const int j = tc + b * TPC;
        if (NB % TPC == 0 || j < NB) {
            const int k = j % NS;
            const int base = (j - k) * R + k;
#pragma unroll
            for (int q = 0; q < R; ++q) s[pad_idx(base + q * NS)] = v[b][q];
        }
    }
    __syncthreads();
}

// Remaining passes after the first (forward direction: all in smem).
template <int N, int TPC, int NS, int SIGN>
__device__ __forceinline__ void passes_rest(double2*, int, const double2*, const double2*, Radices<>) {}

template <int N, int TPC, int NS, int SIGN, int R, int... Rest>
__device__ __forceinline__ void passes_rest(double2* s, int tc, const double2* lo, const double2* hi,
                                            Radices<R, Rest...>) {
    pass_smem<N, TPC, R, NS, SIGN>(s, tc, lo, hi);
    passes_rest<N, TPC, NS * R, SIGN>(s, tc, lo, hi, Radices<Rest...>{});
}

template <int R, int... Rest>
__device__ constexpr int first_radix(Radices<R, Rest...>) { return R; }
template <int R, int... Rest>
__device__ constexpr Radices<Rest...> tail(Radices<R, Rest...>) { return {}; }

// All passes but the last (inverse direction; the last pass stores to global).
template <int N, int TPC, int NS, int SIGN, int R>
__device__ constexpr int last_ns(Radices<R>) { return NS; }

template <int... Rs>
struct Count { static constexpr int value = sizeof...(Rs); };

template <int N, int TPC, int NS, int SIGN, int R>
__device__ __forceinline__ void passes_but_last(double2*, int, const double2*, const double2*, Radices<R>) {}

template <int N, int TPC, int NS, int SIGN, int R, int R2, int... Rest>
__device__ __forceinline__ void passes_but_last(double2* s, int tc, const double2* lo, const double2* hi,
                                                Radices<R, R2, Rest...>) {
    pass_smem<N, TPC, R, NS, SIGN>(s, tc, lo, hi);
    passes_but_last<N, TPC, NS * R, SIGN>(s, tc, lo, hi, Radices<R2, Rest...>{});
}

template <int NS, int R>
__device__ constexpr int ns_before_last(Radices<R>) { return NS; }
template <int NS, int R, int R2, int... Rest>
__device__ constexpr int ns_before_last(Radices<R, R2, Rest...>) {
    return ns_before_last<NS * R>(Radices<R2, Rest...>{});
}
template <int R>
__device__ constexpr int last_radix(Radices<R>) { return R; }
template <int R, int R2, int... Rest>
__device__ constexpr int last_radix(Radices<R, R2, Rest...>) { return last_radix(Radices<R2, Rest...>{}); }

// Shared twiddle tables for W_n (lo: W^0..31, hi: W^{32 h}) loaded once per CTA.
__device__ __forceinline__ void load_tables(double2* lo, double2* hi, int hi_count, const double2* g_lo,
                                            const double2* g_hi) {
    for (int i = threadIdx.x; i < kTwLo; i += blockDim.x) lo[i] = g_lo[i];
    for (int i = threadIdx.x; i < hi_count; i += blockDim.x) hi[i] = g_hi[i];
}

// ---------------------------------------------------------------------------
// r2c: SOTI rows (time contiguous) -> frequency-major out[k*out_fs + c]
// ---------------------------------------------------------------------------
template <int N, int CPB>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, kMinBlocks<N, CPB>)
    k_r2c_fast(const double* __restrict__ in, long long in_cs, double2* __restrict__ out, long long out_fs,
               int channels, FastTables tabs) {
    using P = FastPlan<N>;
    constexpr int TPC = P::TPC, CS = chan_stride(N);
    constexpr int HI = tw_hi_count<N>();
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;   // post twiddles W_{2N}
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    const int b = threadIdx.x / TPC;
    const int tc = threadIdx.x - b * TPC;
    const int c = blockIdx.x * CPB + b;
    const bool live = c < channels;
    double2* s = sm + b * CS;
    __syncthreads();

    // ---- first pass straight from global: z[n] = (x[2n], x[2n+1]); z[n] = 0 for n >= N/2
    {
        constexpr int R = first_radix(typename P::R{});
        constexpr int NB = N / R;
        constexpr int BF = (NB + TPC - 1) / TPC;
        const double2* row = reinterpret_cast<const double2*>(in + (long long)c * in_cs);
        double2 v[BF][R];
#pragma unroll
        for (int bf = 0; bf < BF; ++bf) {
            const int j = tc + bf * TPC;
            if (NB % TPC == 0 || j < NB) {
                // n = j + q NB < N/2 iff q < R/2: the zero-padded half is never loaded
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int n = j + q * NB;
                    v[bf][q] = (q < R / 2 && live) ? __ldg(row + n) : make_double2(0.0, 0.0);
                }
                dft<R, -1>(v[bf]);
            }
        }
#pragma unroll
        for (int bf = 0; bf < BF; ++bf) {
            const int j = tc + bf * TPC;
            if (NB % TPC == 0 || j < NB) {
#pragma unroll
                for (int q = 0; q < R; ++q) s[pad_idx(j * R + q)] = v[bf][q];
            }
        }
        __syncthreads();
        passes_rest<N, TPC, R, -1>(s, tc, lo, hi, tail(typename P::R{}));
    }

    // ---- split: X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 W_{2N}^k (Z_k - conj Z_{N-k}), pairs (k, N-k)
    constexpr int NPAIR = N / 2 + 1;  // k = 0..N/2
    for (int u = threadIdx.x; u < NPAIR * CPB; u += blockDim.x) {
        const int k = u / CPB;
        const int bb = u - k * CPB;
        const int cc = blockIdx.x * CPB + bb;
        if (cc >= channels) continue;
        const double2* z = sm + bb * CS;
        const double2 zk = z[pad_idx(k == 0 ? 0 : k)];
        const double2 zn = z[pad_idx(k == 0 ? 0 : N - k)];
        // X_k  (one table lookup per pair: W_{2N}^{N-k} = -conj(W_{2N}^k))
        const double2 w = tw_lookup<-1>(plo, phi, k);
        {
            const double2 a = cadd(zk, cconj(zn));
            const double2 wb = cmul(w, csub(zk, cconj(zn)));
            out[(long long)k * out_fs + cc] = make_double2(0.5 * (a.x + wb.y), 0.5 * (a.y - wb.x));
        }
        // X_{N-k} (k=0 gives X_N; k = N/2 is its own partner)
        if (k < N / 2) {
            const int kk = N - k;
            const double2 a = cadd(zn, cconj(zk));
            const double2 wn = make_double2(-w.x, w.y);
            const double2 wb = cmul(wn, csub(zn, cconj(zk)));
            out[(long long)kk * out_fs + cc] = make_double2(0.5 * (a.x + wb.y), 0.5 * (a.y - wb.x));
        }
    }
}

// ---------------------------------------------------------------------------
// c2r: frequency-major in[k*in_fs + c] -> SOTI rows out[c*out_cs + t], t < N
// ---------------------------------------------------------------------------
template <int N, int CPB>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, kMinBlocks<N, CPB>)
    k_c2r_fast(const double2* __restrict__ in, long long in_fs, double* __restrict__ out, long long out_cs,
               int channels, FastTables tabs, C2REpilogue epi) {
    using P = FastPlan<N>;
    constexpr int TPC = P::TPC, CS = chan_stride(N);
    constexpr int HI = tw_hi_count<N>();
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    __syncthreads();

    // ---- pre-split: Z_k = (1/2N)[(X_k + conj X_{N-k}) + i conj(W_{2N}^k)(X_k - conj X_{N-k})]
    constexpr int NPAIR = N / 2 + 1;
    constexpr double inv_len = 0.5 / N;
    for (int u = threadIdx.x; u < NPAIR * CPB; u += blockDim.x) {
        const int k = u / CPB;
        const int bb = u - k * CPB;
        const int cc = blockIdx.x * CPB + bb;
        double2* z = sm + bb * CS;
        double2 xk = make_double2(0.0, 0.0), xn = xk;
        if (cc < channels) {
            xk = __ldg(in + (long long)k * in_fs + cc);
            xn = __ldg(in + (long long)(N - k) * in_fs + cc);
        }
        const double2 w = tw_lookup<-1>(plo, phi, k);  // W_{2N}^{N-k} = -conj(W_{2N}^k)
        {
            const double2 e = cadd(xk, cconj(xn));
            const double2 o = cmul(csub(xk, cconj(xn)), cconj(w));
            z[pad_idx(k == 0 ? 0 : k)] = make_double2(inv_len * (e.x - o.y), inv_len * (e.y + o.x));
        }
        if (k > 0 && k < N / 2) {
            const int kk = N - k;
            const double2 e = cadd(xn, cconj(xk));
            const double2 o = cmul(csub(xn, cconj(xk)), make_double2(-w.x, -w.y));
            z[pad_idx(kk)] = make_double2(inv_len * (e.x - o.y), inv_len * (e.y + o.x));
        }
    }
    __syncthreads();

    const int b = threadIdx.x / TPC;
    const int tc = threadIdx.x - b * TPC;
    const int c = blockIdx.x * CPB + b;
    double2* s = sm + b * CS;
    passes_but_last<N, TPC, 1, +1>(s, tc, lo, hi, typename P::R{});

    // ---- last pass: outputs p = j + q N/R; keep p < N/2 (t = 2p, 2p+1 < N)
    constexpr int R = last_radix(typename P::R{});
    constexpr int NS = ns_before_last<1>(typename P::R{});
    constexpr int NB = N / R;
    constexpr int BF = (NB + TPC - 1) / TPC;
    if (c >= channels) return;
    double* orow = out + (long long)c * out_cs;
    const double* vrow = epi.v ? epi.v + (long long)c * out_cs : nullptr;
#pragma unroll
    for (int bf = 0; bf < BF; ++bf) {
        const int j = tc + bf * TPC;
        if (NB % TPC == 0 || j < NB) {
            double2 v[R];
#pragma unroll
            for (int q = 0; q < R; ++q) v[q] = s[pad_idx(j + q * NB)];
            twiddle_inputs<N, R, NS, +1>(v, j, lo, hi);
            dft<R, +1>(v);
#pragma unroll
            for (int q = 0; q < (R + 1) / 2; ++q) {  // keep p = j + q*NB < N/2 (unpad)
                const int p = j + q * NB;
                if ((R % 2 == 1) && q == R / 2 && p >= N / 2) break;
                double y0 = v[q].x, y1 = v[q].y;
                const int t0 = 2 * p;
                if (epi.gamma_mode == 1) {
                    const double g = __ldg(epi.gamma + (c % epi.gamma_dim));
                    y0 *= g;
                    y1 *= g;
                } else if (epi.gamma_mode == 2) {
                    const double* gr = epi.gamma + (long long)(c % epi.gamma_dim) * N;
                    y0 *= __ldg(gr + t0);
                    y1 *= __ldg(gr + t0 + 1);
                }
                if (vrow) {
                    double r0 = __ldg(vrow + t0), r1 = __ldg(vrow + t0 + 1);
                    if (epi.reg_kind == 1) {
                        const double l = t0 > 0 ? __ldg(vrow + t0 - 1) : 0.0;
                        const double h = t0 + 2 < N ? __ldg(vrow + t0 + 2) : 0.0;
                        const double a0 = 2.0 * r0 - l - r1;  // reference order: 2x - x[t-1] - x[t+1]
                        const double a1 = 2.0 * r1 - r0 - h;
                        r0 = a0;
                        r1 = a1;
                    }
                    y0 += epi.alpha * r0;
                    y1 += epi.alpha * r1;
                }
                reinterpret_cast<double2*>(orow)[p] = make_double2(y0, y1);
            }
        }
    }
}

}  // namespace fast
}  // namespace btg
