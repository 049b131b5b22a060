// Shared-memory mixed-radix Stockham FFT building blocks (sm_100a, FP64).
//
// The reference transforms each zero-padded length-2N_t channel with a full
// complex FFTW plan (fft.cpp:17-34, block_operator.cpp:54-80). Here a real
// length-L=2N_t series is transformed as a complex length-N=N_t series
// z[n] = x[2n] + i x[2n+1] plus an O(N) split (R2C), and back (C2R); only the
// N_t+1 non-redundant frequencies exist. The complex length-N transform is an
// autosort Stockham pass sequence in shared memory: each pass reads R strided
// values, twiddles, runs an R-point DFT in registers and writes autosorted, so
// no bit reversal is ever needed and every length factorizable into
// 2,3,4,5,7,8 (and any other small prime via the generic pass) works.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace btg {

constexpr int kMaxFactors = 40;

// Device-side FFT plan for complex length n (= N_t). Twiddle tables live in
// global memory (read-only path); factors are passed by value.
struct FftPlanDev {
    int n;
    int nfac;
    int fac[kMaxFactors];
    const double2* tw;    // tw[k]   = exp(-2*pi*i*k/n),      k < n
    const double2* post;  // post[k] = exp(-2*pi*i*k/(2n)),   k <= n
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by SIGN * i
template <int SIGN>
__device__ __forceinline__ double2 mul_si(double2 a) {
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}
template <int SIGN>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tw, int idx) {
    double2 w = __ldg(tw + idx);
    if (SIGN > 0) w.y = -w.y;
    return w;
}

// ---- R-point DFT kernels on registers: X_q = sum_s v_s exp(SIGN*2*pi*i*q*s/R)
template <int SIGN>
__device__ __forceinline__ void dft2(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2* v) {
    const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    const double2 b0 = cadd(v[1], v[3]), b1 = mul_si<SIGN>(csub(v[1], v[3]));
    v[0] = cadd(a0, b0);
    v[1] = cadd(a1, b1);
    v[2] = csub(a0, b0);
    v[3] = csub(a1, b1);
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* v) {
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    dft4<SIGN>(e);
    dft4<SIGN>(o);
    constexpr double r = 0.70710678118654752440;
    // w8^1 = (r, SIGN r), w8^2 = SIGN i, w8^3 = (-r, SIGN r)
    const double2 o1 = make_double2(r * (o[1].x - SIGN * o[1].y), r * (o[1].y + SIGN * o[1].x));
    const double2 o2 = mul_si<SIGN>(o[2]);
    const double2 o3 = make_double2(-r * (o[3].x + SIGN * o[3].y), r * (SIGN * o[3].x - o[3].y));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
}

template <int SIGN>
__device__ __forceinline__ void dft3(double2* v) {
    constexpr double c = -0.5;
    constexpr double s = SIGN * 0.86602540378443864676;
    const double2 t1 = cadd(v[1], v[2]);
    const double2 t2 = csub(v[1], v[2]);
    const double2 m = make_double2(fma(c, t1.x, v[0].x), fma(c, t1.y, v[0].y));
    const double2 ist2 = make_double2(-s * t2.y, s * t2.x);
    v[0] = cadd(v[0], t1);
    v[1] = cadd(m, ist2);
    v[2] = csub(m, ist2);
}

template <int SIGN>
__device__ __forceinline__ void dft5(double2* v) {
    constexpr double c1 = 0.30901699437494742410;   // cos(2pi/5)
    constexpr double c2 = -0.80901699437494742410;  // cos(4pi/5)
    constexpr double s1 = SIGN * 0.95105651629515357212;
    constexpr double s2 = SIGN * 0.58778525229247312917;
    const double2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    const double2 t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const double2 a1 = make_double2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    const double2 a2 = make_double2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    // b = i * (p) with p = s1 t3 + s2 t4 (q=1) and s2 t3 - s1 t4 (q=2)
    const double2 p1 = make_double2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
    const double2 p2 = make_double2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
    const double2 b1 = make_double2(-p1.y, p1.x), b2 = make_double2(-p2.y, p2.x);
    v[0] = make_double2(v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y);
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
}

// One radix-R Stockham pass over `nb` channels (channel stride `cs` complex
// elements in shared memory). ns = product of the radices already applied.
template <int R, int SIGN>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                              int n, int ns, int nb, int cs,
                                              const double2* __restrict__ tw) {
    const int nbf = n / R;
    const int tw_step = n / (ns * R);
    const int total = nb * nbf;
    for (int u = threadIdx.x; u < total; u += blockDim.x) {
        const int b = u / nbf;
        const int j = u - b * nbf;
        const int k = j % ns;
        const double2* s = src + b * cs;
        double2* d = dst + b * cs;
        double2 v[R];
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = s[j + q * nbf];
        if (k) {
#pragma unroll
            for (int q = 1; q < R; ++q) v[q] = cmul(v[q], twiddle<SIGN>(tw, k * q * tw_step));
        }
        if constexpr (R == 2) dft2<SIGN>(v);
        if constexpr (R == 3) dft3<SIGN>(v);
        if constexpr (R == 4) dft4<SIGN>(v);
        if constexpr (R == 5) dft5<SIGN>(v);
        if constexpr (R == 8) dft8<SIGN>(v);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int q = 0; q < R; ++q) d[base + q * ns] = v[q];
    }
}

// Generic odd-radix pass (any prime r; O(r^2) per butterfly) with combined
// twiddles: out_q = sum_s src_s * W_n^{k s tw_step + q s n/r}.
template <int SIGN>
__device__ __forceinline__ void stockham_pass_generic(const double2* __restrict__ src,
                                                      double2* __restrict__ dst, int n, int r,
                                                      int ns, int nb, int cs,
                                                      const double2* __restrict__ tw) {
    const int nbf = n / r;
    const int tw_step = n / (ns * r);
    const int total = nb * nbf;
    for (int u = threadIdx.x; u < total; u += blockDim.x) {
        const int b = u / nbf;
        const int j = u - b * nbf;
        const int k = j % ns;
        const double2* s = src + b * cs;
        double2* d = dst + b * cs;
        const int base = (j - k) * r + k;
        for (int q = 0; q < r; ++q) {
            double2 acc = s[j];
            for (int t = 1; t < r; ++t) {
                const long long e = (long long)k * t * tw_step + (long long)((q * t) % r) * nbf;
                acc = cadd(acc, cmul(s[j + t * nbf], twiddle<SIGN>(tw, (int)(e % n))));
            }
            d[base + q * ns] = acc;
        }
    }
}

// Full complex FFT of `nb` channels held at buf_a (stride cs); buf_b is the
// ping-pong partner. Returns the buffer holding the result. Callers must
// __syncthreads() before (input written) — this routine syncs after each pass.
template <int SIGN>
__device__ double2* fft_smem(double2* buf_a, double2* buf_b, int nb, int cs, const FftPlanDev& p) {
    double2* src = buf_a;
    double2* dst = buf_b;
    int ns = 1;
    for (int s = 0; s < p.nfac; ++s) {
        const int r = p.fac[s];
        switch (r) {
            case 2: stockham_pass<2, SIGN>(src, dst, p.n, ns, nb, cs, p.tw); break;
            case 3: stockham_pass<3, SIGN>(src, dst, p.n, ns, nb, cs, p.tw); break;
            case 4: stockham_pass<4, SIGN>(src, dst, p.n, ns, nb, cs, p.tw); break;
            case 5: stockham_pass<5, SIGN>(src, dst, p.n, ns, nb, cs, p.tw); break;
            case 8: stockham_pass<8, SIGN>(src, dst, p.n, ns, nb, cs, p.tw); break;
            default: stockham_pass_generic<SIGN>(src, dst, p.n, r, ns, nb, cs, p.tw); break;
        }
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
        ns *= r;
    }
    return src;
}

}  // namespace btg
