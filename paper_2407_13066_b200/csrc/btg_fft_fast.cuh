// Register-resident Stockham FFT for the vector transforms (K5 / K9), with the
// transform length N = N_t fixed at compile time.
//
// A real length-2N series is transformed as the complex length-N series
// z[n] = x[2n] + i x[2n+1] plus an O(N) split; only the N+1 non-redundant
// frequencies exist. Per channel, TPC threads hold the data in registers: each
// radix-R pass loads its R inputs, applies the inter-pass twiddles, runs the
// R-point DFT in registers and scatters the outputs autosorted through ONE
// in-place shared-memory buffer per channel (all loads of a pass complete at a
// barrier before any thread overwrites).
//
// The split between the complex transform and the real spectrum pairs
// frequency k with N-k. Both live in the SAME thread when butterflies j and
// NB-j of the last (R2C) / first (C2R) pass are processed together (butterfly
// j holds positions j + q NB, whose partners N - j - q NB are positions of
// butterfly NB - j). So:
//  r2c: pass 1 reads z straight from the SOTI row with 16-byte loads (the
//       zero-padded half, q >= R/2, is never loaded); the last pass runs on
//       butterfly pairs and computes X_k, X_{N-k} in registers, storing
//       frequency-major — no shared-memory split pass.
//  c2r: the first pass loads X_k, X_{N-k} pairs frequency-major, forms
//       Z_k, Z_{N-k} in registers and runs the pair of butterflies; the last
//       pass stores x[2p], x[2p+1] straight into the SOTI row (only p < N/2
//       survives the unpad) through the Gamma^-1 / alpha R v epilogue.
// A length-1024 transform is three passes (16,16,4 / 4,16,16) and two
// shared-memory round trips. Threads are interleaved over channels
// (channel = tid % CPB) so every global access is CPB contiguous complex
// values per frequency / 8 consecutive 16-byte words per row. Shared index p
// is padded to p + p/16 (conflict-free stride-R scatter); twiddles
// W^e = lo[e % 32] * hi[e / 32] come from two small shared tables, higher
// powers by multiplication.
#pragma once

#include <cuda_runtime.h>

#include "btg_fft.cuh"
#include "btg_kernels.cuh"
#include "btg_umma.cuh"

namespace btg {
namespace fast {

// Plans: TPC threads per channel, channels per CTA for each direction, pass radices
// for R2C (small radix last: it runs on butterfly pairs) and C2R (small first),
// and the resident threads per SM each direction is compiled for (register
// budget = 64K / RES) and whether the kernel runs persistent with the next
// channel group's first-pass loads prefetched into registers (PF): measured on
// B200 (profiles/r01s2_fft_sweep.md) — the longer transforms prefer fewer,
// fatter threads, most of all the C2R; the prefetch pays where its registers
// do not cost occupancy (short transforms, the N_t = 1024 C2R).
template <int... Rs>
struct Radices {};
template <int N>
struct FastPlan;
#define BTG_PLAN(N, tpc, cpb_r2c, cpb_c2r, res_r2c, res_c2r, pf_r2c, pf_c2r, R2CL, C2RL)      \
    template <>                                                                                  \
    struct FastPlan<N> {                                                                         \
        static constexpr int TPC = tpc, CPB_R2C = cpb_r2c, CPB_C2R = cpb_c2r;                    \
        static constexpr int RES_R2C = res_r2c, RES_C2R = res_c2r;                               \
        static constexpr bool PF_R2C = pf_r2c, PF_C2R = pf_c2r;                                  \
        using R2C = R2CL;                                                                        \
        using C2R = C2RL;                                                                        \
    };
#define BTG_R(...) Radices<__VA_ARGS__>
//       N      TPC  channels/CTA  RES r2c/c2r  prefetch r2c/c2r
BTG_PLAN(64,    8,   32, 32,  512,  512,  true,  true,  BTG_R(16, 4),           BTG_R(4, 16))
BTG_PLAN(128,   16,  16, 16,  1024, 1024, false, false, BTG_R(8, 4, 4),         BTG_R(4, 4, 8))
BTG_PLAN(256,   16,  16, 16,  512,  256,  true,  true,  BTG_R(16, 4, 4),        BTG_R(4, 4, 16))
BTG_PLAN(500,   64,  4,  4,   1024, 768,  false, false, BTG_R(4, 5, 5, 5),      BTG_R(5, 5, 5, 4))
BTG_PLAN(512,   64,  4,  4,   256,  768,  false, false, BTG_R(16, 8, 4),        BTG_R(4, 8, 16))
// N_t = 1000: 10 x 10 x 10 (radix-10 = 2 x 5 in registers), 50 threads per channel
// — three passes, no idle butterfly slots (the 8.5.5.5 plan at 128 threads left 22 %
// of its radix-5 slots idle); measured at configs[2] (8192 / 600 channels):
// R2C 0.100 -> 0.085 ms, C2R 0.127 -> 0.102 ms (profiles/r02s2_fft1000.md)
BTG_PLAN(1000,  50,  2,  2,   400,  400,  false, false, BTG_R(10, 10, 10),      BTG_R(10, 10, 10))
// (BTG_P1024_* override the N_t = 1024 plan in plan sweeps)
#ifndef BTG_P1024_TPC
#define BTG_P1024_TPC 64
#define BTG_P1024_CPBR 4
#define BTG_P1024_CPBC 4
#define BTG_P1024_RESR 768
#define BTG_P1024_RESC 256
#define BTG_P1024_PFR false
#define BTG_P1024_PFC true
#endif
BTG_PLAN(1024,  BTG_P1024_TPC, BTG_P1024_CPBR, BTG_P1024_CPBC, BTG_P1024_RESR, BTG_P1024_RESC, BTG_P1024_PFR,
         BTG_P1024_PFC, BTG_R(16, 16, 4), BTG_R(4, 16, 16))
BTG_PLAN(2000,  128, 2,  2,   512,  384,  false, false, BTG_R(16, 5, 5, 5),     BTG_R(5, 5, 5, 16))
BTG_PLAN(2048,  128, 2,  2,   512,  256,  false, false, BTG_R(16, 8, 4, 4),     BTG_R(4, 4, 8, 16))
BTG_PLAN(4096,  256, 2,  1,   512,  256,  true,  false, BTG_R(16, 16, 4, 4),    BTG_R(4, 4, 16, 16))
// long horizons: the paper's N_t = 10000 runs and 2^13
BTG_PLAN(8192,  512, 1,  1,   768,  768,  false, false, BTG_R(16, 16, 8, 4),    BTG_R(4, 8, 16, 16))
BTG_PLAN(10000, 625, 1,  1,   768,  768,  false, false, BTG_R(16, 5, 5, 5, 5),  BTG_R(5, 5, 5, 5, 16))
#undef BTG_R
#undef BTG_PLAN

// Minimum CTAs per SM for __launch_bounds__ from a resident-thread target.
// BTG_FFT_RESIDENT_THREADS (sweeps) overrides every plan.
constexpr int min_blocks(int res, int cta_threads) {
    return res / cta_threads < 1 ? 1 : (res / cta_threads > 16 ? 16 : res / cta_threads);
}
#ifdef BTG_FFT_RESIDENT_THREADS
template <int N, int CPB>
constexpr int kMinBlocksR2C = min_blocks(BTG_FFT_RESIDENT_THREADS, FastPlan<N>::TPC * CPB);
template <int N, int CPB>
constexpr int kMinBlocksC2R = min_blocks(BTG_FFT_RESIDENT_THREADS, FastPlan<N>::TPC * CPB);
#else
template <int N, int CPB>
constexpr int kMinBlocksR2C = min_blocks(FastPlan<N>::RES_R2C, FastPlan<N>::TPC * CPB);
template <int N, int CPB>
constexpr int kMinBlocksC2R = min_blocks(FastPlan<N>::RES_C2R, FastPlan<N>::TPC * CPB);
#endif

__host__ __device__ constexpr int pad_idx(int p) { return p + (p >> 4); }
// Channel-buffer stride (double2): the CPB channel buffers a quarter-warp touches
// start in distinct bank groups — stride = 8 / CPB (mod 8) for CPB <= 8, 1 for
// wider groups (8 channels of one butterfly per quarter-warp). N_t = 1000 at 2
// channels per CTA had both channels on the same banks (1064 = 0 mod 8).
template <int CPB>
__host__ __device__ constexpr int chan_stride(int n) {
    const int base = pad_idx(n) + 2;
    const int want = CPB >= 8 ? 1 : (8 / CPB) % 8;
    return CPB == 1 ? base : base + ((want - base) % 8 + 8) % 8;
}
static_assert(chan_stride<4>(1024) == 1090, "the N_t = 1024 layout is unchanged");
constexpr int kTwLo = 32;

template <int N>
__host__ __device__ constexpr int tw_hi_count() { return (N + kTwLo - 1) / kTwLo + 1; }

template <int N, int CPB>
__host__ __device__ constexpr size_t smem_bytes() {
    return sizeof(double2) * ((size_t)CPB * chan_stride<CPB>(N) + 2 * kTwLo + 2 * tw_hi_count<N>() + 2);
}

// W^e for W = exp(SIGN * 2 pi i / n_tw) from the split table (lo[e % 32] * hi[e / 32]).
template <int SIGN>
__device__ __forceinline__ double2 tw_lookup(const double2* lo, const double2* hi, int e) {
    double2 w = cmul(lo[e & (kTwLo - 1)], hi[e >> 5]);
    if (SIGN > 0) w.y = -w.y;
    return w;
}

// dft4 of (a, b, 0, 0): the zero-padded half of an R2C first pass
template <int SIGN>
__device__ __forceinline__ void dft4_half(double2* v) {
    const double2 a = v[0], b = v[1], c = mul_si<SIGN>(v[1]);
    v[0] = cadd(a, b);
    v[1] = cadd(a, c);
    v[2] = csub(a, b);
    v[3] = csub(a, c);
}

// HALF: inputs v[q], q >= R/2, are zero and never read (the R2C zero pad);
// the first butterfly stage then skips the additions of zeros — IEEE x + 0
// cannot be folded by the compiler, so these were real DADDs before.
template <int R, int SIGN, bool HALF = false>
__device__ __forceinline__ void dft(double2* v) {
    if constexpr (HALF && R == 4) dft4_half<SIGN>(v);
    else if constexpr (HALF && R == 8) {
        double2 e[4] = {v[0], v[2], {}, {}};
        double2 o[4] = {v[1], v[3], {}, {}};
        dft4_half<SIGN>(e);
        dft4_half<SIGN>(o);
        constexpr double r = 0.70710678118654752440;
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
    } else if constexpr (HALF && R != 16) {
#pragma unroll
        for (int q = R / 2; q < R; ++q) v[q] = make_double2(0.0, 0.0);
        dft<R, SIGN>(v);
    } else if constexpr (R == 2) dft2<SIGN>(v);
    else if constexpr (R == 3) dft3<SIGN>(v);
    else if constexpr (R == 4) dft4<SIGN>(v);
    else if constexpr (R == 5) dft5<SIGN>(v);
    else if constexpr (R == 10) {
        // 10 = 2 x 5: dft5 over s of a[r][s] = v[r + 2s], twiddle W_10^{r k}, dft2 over r;
        // output k + 5 m
        double2 a[2][5];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int q = 0; q < 5; ++q) a[r][q] = v[r + 2 * q];
            dft5<SIGN>(a[r]);
        }
        constexpr double c1 = 0.80901699437494742410, s1 = 0.58778525229247312917;  // W_10^1
        constexpr double c2 = 0.30901699437494742410, s2 = 0.95105651629515357212;  // W_10^2
        a[1][1] = cmul(a[1][1], make_double2(c1, SIGN * s1));
        a[1][2] = cmul(a[1][2], make_double2(c2, SIGN * s2));
        a[1][3] = cmul(a[1][3], make_double2(-c2, SIGN * s2));  // W_10^3
        a[1][4] = cmul(a[1][4], make_double2(-c1, SIGN * s1));  // W_10^4
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            v[k] = cadd(a[0][k], a[1][k]);
            v[k + 5] = csub(a[0][k], a[1][k]);
        }
    }
    else if constexpr (R == 8) dft8<SIGN>(v);
    else if constexpr (R == 16) {
        // 16 = 4 x 4: columns, twiddle W_16^{r k}, rows, transpose.
        double2 a[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int q = 0; q < (HALF ? 2 : 4); ++q) a[r][q] = v[r + 4 * q];
            if constexpr (HALF) dft4_half<SIGN>(a[r]);
            else dft4<SIGN>(a[r]);
        }
        constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
        constexpr double c2 = 0.70710678118654752440;
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

// ---- direct twiddle tables ---------------------------------------------------
// (a) W_2N^e for e in [0, N/4] (`w2q`, one octant of the 2N circle; the rest by
//     the symmetries W^{Q-r} = -i conj W^r and W^{qQ+r} = (-i)^q W^r, Q = N/2:
//     integer selects, no FP64 work). Serves the R2C split / C2R pre-split
//     twiddles and the first power of every generated pass twiddle.
// (b) Per-pass tables [k][q] = W_N^{k q N/(NS R)} (row stride R+1: the 8
//     distinct k of a warp hit 8 distinct bank groups) for the passes whose
//     table fits the plan's budget (TabPlan): their R-1 twiddles become R-1
//     shared loads (broadcast over the CPB channel lanes) instead of one lookup
//     product and R-2 power products.
// Largest per-pass table (entries) each direction may keep in shared memory,
// and whether the plan uses the octant table.
// Measured on B200 (N_t = 1024, 32768 / 524288 channels): the vector FFTs are
// latency-bound, not FP64-bound — removing the generation products moved the
// R2C by <= 1 % (and its extra shared memory costs the non-TMA R2C a CTA per
// SM), the C2R gained 5 % at 32768 channels from the octant table alone; the
// pass tables were neutral or slower. Defaults: octant table for the C2R only.
#ifndef BTG_TAB_R2C
#define BTG_TAB_R2C 0
#define BTG_TAB_C2R 0
#define BTG_TAB_W2Q_R2C 0
#define BTG_TAB_W2Q_C2R 1
#endif
template <int N>
struct TabPlan {
    static constexpr int R2C = BTG_TAB_R2C, C2R = BTG_TAB_C2R;
    static constexpr bool W2Q_R2C = BTG_TAB_W2Q_R2C, W2Q_C2R = BTG_TAB_W2Q_C2R;
};
template <int N, bool C2R>
constexpr bool kUseW2Q = (C2R ? TabPlan<N>::W2Q_C2R : TabPlan<N>::W2Q_R2C) && (N % 4 == 0) && N <= 4096;
template <int N, bool C2R>
__host__ __device__ constexpr int w2q_entries() { return kUseW2Q<N, C2R> ? N / 4 + 1 : 0; }
template <int R, int NS, int LIM>
__host__ __device__ constexpr bool pass_tab() { return NS > 1 && NS * (R + 1) <= LIM; }
template <int NS, int LIM, int R>
__host__ __device__ constexpr int tab_entries(Radices<R>) { return pass_tab<R, NS, LIM>() ? NS * (R + 1) : 0; }
template <int NS, int LIM, int R, int R2, int... Rest>
__host__ __device__ constexpr int tab_entries(Radices<R, R2, Rest...>) {
    return (pass_tab<R, NS, LIM>() ? NS * (R + 1) : 0) + tab_entries<NS * R, LIM>(Radices<R2, Rest...>{});
}
template <int N, bool R2C>
__host__ __device__ constexpr int ptab_entries() {
    if constexpr (R2C) return tab_entries<1, TabPlan<N>::R2C>(typename FastPlan<N>::R2C{});
    else return tab_entries<1, TabPlan<N>::C2R>(typename FastPlan<N>::C2R{});
}
// entries of the tables of all passes but the last (offset of the last pass's table)
template <int NS, int LIM, int R>
__host__ __device__ constexpr int tab_entries_but_last(Radices<R>) { return 0; }
template <int NS, int LIM, int R, int R2, int... Rest>
__host__ __device__ constexpr int tab_entries_but_last(Radices<R, R2, Rest...>) {
    return (pass_tab<R, NS, LIM>() ? NS * (R + 1) : 0) + tab_entries_but_last<NS * R, LIM>(Radices<R2, Rest...>{});
}
// Shared-memory bytes of a direction's kernel: channel buffers + split tables
// (smem_bytes) + the octant table + the pass tables.
template <int N, int CPB, bool R2C>
__host__ __device__ constexpr size_t smem_dir() {
    return smem_bytes<N, CPB>() + sizeof(double2) * (w2q_entries<N, !R2C>() + ptab_entries<N, R2C>());
}

template <int N, int NS, int LIM, int R>
__device__ __forceinline__ void fill_one_tab(double2* t, const double2* wn) {
    if constexpr (pass_tab<R, NS, LIM>()) {
        constexpr int step = N / (NS * R);
        for (int i = threadIdx.x; i < NS * (R + 1); i += blockDim.x) {
            const int k = i / (R + 1), q = i % (R + 1);
            t[i] = wn[(k * q * step) % N];
        }
    }
}
template <int N, int NS, int LIM, int R>
__device__ __forceinline__ void fill_pass_tabs(double2* t, const double2* wn, Radices<R>) {
    fill_one_tab<N, NS, LIM, R>(t, wn);
}
template <int N, int NS, int LIM, int R, int R2, int... Rest>
__device__ __forceinline__ void fill_pass_tabs(double2* t, const double2* wn, Radices<R, R2, Rest...>) {
    fill_one_tab<N, NS, LIM, R>(t, wn);
    fill_pass_tabs<N, NS * R, LIM>(t + (pass_tab<R, NS, LIM>() ? NS * (R + 1) : 0), wn, Radices<R2, Rest...>{});
}

// W_2N^e, e in [0, 2N): octant table when the plan has one, else the split tables.
template <int N, bool C2R>
__device__ __forceinline__ double2 w2n_lookup(const double2* w2q, const double2* plo, const double2* phi, int e) {
    if constexpr (kUseW2Q<N, C2R>) {
        constexpr int Q = N / 2, O = N / 4;
        const int qd = e / Q;
        const int r = e - qd * Q;
        const bool fold = r > O;
        const double2 t = w2q[fold ? Q - r : r];
        double2 w = fold ? make_double2(-t.y, -t.x) : t;  // -i conj(t)
        if (qd & 1) w = make_double2(w.y, -w.x);        // * (-i)
        if (qd & 2) w = make_double2(-w.x, -w.y);       // * (-1)
        return w;
    } else {
        return tw_lookup<-1>(plo, phi, e);
    }
}

// Fill the octant table and the pass tables (from the global W_N / W_2N tables).
template <int N, int LIM, typename RL, bool C2R>
__device__ __forceinline__ void load_direct_tables(double2* w2q, double2* ptab, const FastTables& tabs) {
    for (int i = threadIdx.x; i < w2q_entries<N, C2R>(); i += blockDim.x) w2q[i] = tabs.w2n[i];
    fill_pass_tabs<N, 1, LIM>(ptab, tabs.wn, RL{});
}

// Butterfly j of a radix-R pass: v[q] = s[j + q N/R] * W^{k q N/(NS R)}, k = j % NS.
// One table lookup; the powers q = 2..R-1 are products of lower powers.
template <int N, int R, int NS, int SIGN>
__device__ __forceinline__ void twiddle_inputs(double2* v, int j, const double2* lo, const double2* hi,
                                               const double2* w2q = nullptr) {
    if constexpr (NS > 1) {
        const int k = j % NS;
        constexpr int step = N / (NS * R);
        double2 w[R];
        if constexpr (kUseW2Q<N, (SIGN > 0)>) {
            w[1] = w2n_lookup<N, (SIGN > 0)>(w2q, lo, hi, 2 * k * step);  // W_N^e = W_2N^{2e}
            if (SIGN > 0) w[1].y = -w[1].y;
        } else {
            w[1] = tw_lookup<SIGN>(lo, hi, k * step);
        }
#pragma unroll
        for (int q = 2; q < R; ++q) w[q] = cmul(w[q / 2], w[q - q / 2]);
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
    }
}

// Pass twiddles from the pass's table when it has one (LIM), else generated.
template <int N, int R, int NS, int SIGN, int LIM>
__device__ __forceinline__ void twiddle_pass(double2* v, int j, const double2* lo, const double2* hi,
                                             const double2* w2q, const double2* ptab) {
    if constexpr (pass_tab<R, NS, LIM>()) {
        const double2* row = ptab + (j % NS) * (R + 1);
#pragma unroll
        for (int q = 1; q < R; ++q) {
            double2 w = row[q];
            if (SIGN > 0) w.y = -w.y;
            v[q] = cmul(v[q], w);
        }
    } else {
        twiddle_inputs<N, R, NS, SIGN>(v, j, lo, hi, w2q);
    }
}

// One in-place radix-R pass over the channel buffer `s` (smem, padded).
template <int N, int TPC, int R, int NS, int SIGN, int LIM>
__device__ __forceinline__ void pass_smem(double2* s, int tc, const double2* lo, const double2* hi,
                                          const double2* w2q, const double2* ptab) {
    constexpr int NB = N / R;
    constexpr int BF = (NB + TPC - 1) / TPC;
    double2 v[BF][R];
#pragma unroll
    for (int b = 0; b < BF; ++b) {
        const int j = tc + b * TPC;
        if (NB % TPC == 0 || j < NB) {
#pragma unroll
            for (int q = 0; q < R; ++q) v[b][q] = s[pad_idx(j + q * NB)];
            twiddle_pass<N, R, NS, SIGN, LIM>(v[b], j, lo, hi, w2q, ptab);
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

// ---- compile-time radix-list helpers -----------------------------------------
template <int R, int... Rest>
__host__ __device__ constexpr int first_radix(Radices<R, Rest...>) { return R; }
template <int R, int... Rest>
__host__ __device__ constexpr Radices<Rest...> tail(Radices<R, Rest...>) { return {}; }
template <int R>
__host__ __device__ constexpr int last_radix(Radices<R>) { return R; }
template <int R, int R2, int... Rest>
__host__ __device__ constexpr int last_radix(Radices<R, R2, Rest...>) { return last_radix(Radices<R2, Rest...>{}); }
// product of all radices but the last (the NS of the last pass)
template <int R>
__host__ __device__ constexpr int ns_of_last(Radices<R>) { return 1; }
template <int R, int R2, int... Rest>
__host__ __device__ constexpr int ns_of_last(Radices<R, R2, Rest...>) { return R * ns_of_last(Radices<R2, Rest...>{}); }

// Apply every pass of the list but the last, starting at NS.
// ptab: this pass's table (tables are laid out in pass order, see tab_entries).
template <int N, int TPC, int NS, int SIGN, int LIM, int R>
__device__ __forceinline__ void passes_but_last(double2*, int, const double2*, const double2*, const double2*,
                                                const double2*, Radices<R>) {}
template <int N, int TPC, int NS, int SIGN, int LIM, int R, int R2, int... Rest>
__device__ __forceinline__ void passes_but_last(double2* s, int tc, const double2* lo, const double2* hi,
                                                const double2* w2q, const double2* ptab, Radices<R, R2, Rest...>) {
    pass_smem<N, TPC, R, NS, SIGN, LIM>(s, tc, lo, hi, w2q, ptab);
    passes_but_last<N, TPC, NS * R, SIGN, LIM>(s, tc, lo, hi, w2q,
                                               ptab + (pass_tab<R, NS, LIM>() ? NS * (R + 1) : 0),
                                               Radices<R2, Rest...>{});
}

__device__ __forceinline__ void load_tables(double2* lo, double2* hi, int hi_count, const double2* g_lo,
                                            const double2* g_hi) {
    for (int i = threadIdx.x; i < kTwLo; i += blockDim.x) lo[i] = g_lo[i];
    for (int i = threadIdx.x; i < hi_count; i += blockDim.x) hi[i] = g_hi[i];
}

// X_k from Z_k and Z_{N-k}, w = W_{2N}^k:
//   X_k = 1/2 (Z_k + conj Z_{N-k}) - i/2 w (Z_k - conj Z_{N-k})
__device__ __forceinline__ double2 split_x(double2 zk, double2 zn, double2 w) {
    const double2 a = cadd(zk, cconj(zn));
    const double2 wb = cmul(w, csub(zk, cconj(zn)));
    return make_double2(0.5 * (a.x + wb.y), 0.5 * (a.y - wb.x));
}
// Z_k from X_k and X_{N-k}, w = W_{2N}^k:
//   Z_k = (1/2N) [ (X_k + conj X_{N-k}) + i conj(w) (X_k - conj X_{N-k}) ]
__device__ __forceinline__ double2 presplit_z(double2 xk, double2 xn, double2 w, double inv_len) {
    const double2 e = cadd(xk, cconj(xn));
    const double2 o = cmul(csub(xk, cconj(xn)), cconj(w));
    return make_double2(inv_len * (e.x - o.y), inv_len * (e.y + o.x));
}
// W_{2N}^{N-k} = -conj(W_{2N}^k)
__device__ __forceinline__ double2 partner_w(double2 w) { return make_double2(-w.x, w.y); }

// Both members of a split pair with ONE complex product (bit-identical to
// split_x(zk, zn, w) and split_x(zn, zk, partner_w(w))): with A = Z_k + conj Z_{N-k},
// B = Z_k - conj Z_{N-k}:  X_k = (A - i wB)/2,  X_{N-k} = conj((A + i wB)/2).
__device__ __forceinline__ void split_pair(double2 zk, double2 zn, double2 w, double2& xk, double2& xn) {
    const double ax = zk.x + zn.x, ay = zk.y - zn.y;
    const double2 wb = cmul(w, make_double2(zk.x - zn.x, zk.y + zn.y));
    xk = make_double2(0.5 * (ax + wb.y), 0.5 * (ay - wb.x));
    xn = make_double2(0.5 * (ax - wb.y), 0.5 * (-ay - wb.x));
}
// Inverse pair (bit-identical to presplit_z(xk, xn, w, s), presplit_z(xn, xk, partner_w(w), s)):
// with c = conj(w) B:  Z_k = s (A + i c),  Z_{N-k} = s conj(A - i c).
__device__ __forceinline__ void presplit_pair(double2 xk, double2 xn, double2 w, double inv_len, double2& zk,
                                              double2& zn) {
    const double ax = xk.x + xn.x, ay = xk.y - xn.y;
    const double2 c = cmul(make_double2(xk.x - xn.x, xk.y + xn.y), cconj(w));
    zk = make_double2(inv_len * (ax - c.y), inv_len * (ay + c.x));
    zn = make_double2(inv_len * (ax + c.y), inv_len * (-ay + c.x));
}

// Optional R2C epilogue for the tcgen05 int8 multi-RHS engine (R2CBlockMax,
// btg_kernels.cuh): the CPB lanes of a channel group reduce max |re|, |im| of X_k
// by shuffles and one lane stores its block exponent — so the engine's separate
// block-max pass over x-hat reduces to a max over 256 int16 per block.
template <int CPB>
__device__ __forceinline__ void block_max(const R2CBlockMax& bm, int c0, int b, int k, double2 x) {
    // block exponent e + 1 of m = max |re|, |im| with m < 2^e (btg_ozaki.cu scale_exp):
    // for normal m that is the biased exponent field - 1021; zero -> INT16_MIN
    const double m = fmax(fabs(x.x), fabs(x.y));
    const int E = (int)((unsigned long long)__double_as_longlong(m) >> 52);
    int e = E - 1021;
    if (E == 0) {
        e = -32768;
        if (m > 0.0) {  // subnormal
            frexp(m, &e);
            e += 1;
        }
    }
    static_assert(CPB <= 32, "channel group wider than a warp");
    if constexpr (CPB > 1) {
        const int lane = threadIdx.x & 31;
        const unsigned mask = (CPB == 32 ? 0xffffffffu : ((1u << CPB) - 1u)) << (lane & ~(CPB - 1) & 31);
#pragma unroll
        for (int o = 1; o < CPB; o <<= 1) e = max(e, __shfl_xor_sync(mask, e, o));
    }
    if (b == 0) bm.pexp[(size_t)(c0 / CPB) * bm.nf + k] = (int16_t)e;
}

// Spectral-vector addressing. fs > 0: frequency-major, element k of channel c at
// [c + k fs]. fs < 0 (kBlockedFs): channel-blocked, [c / G][k][c % G] with
// N + 1 frequencies, G = kSpecBlock: the R2C writes (C2R reads) of a CTA's CPB
// channels hit G x 16-byte rows (shared with the neighbouring CTAs of the same
// block, which run at the same time) instead of CPB x 16 bytes per frequency
// row spread over the whole vector — 64-byte segments cap HBM at ~3 TB/s at
// 524288 channels, 128-byte ones at 5.4-6.1 TB/s (profiles/r02s2_scatter_bw.md).
template <int N, int CPB>
__device__ __forceinline__ long long spec_base(int c, long long fs) {
    static_assert(kSpecBlock % CPB == 0 || CPB > kSpecBlock, "channel groups tile the spectral blocks");
    return fs < 0 ? (long long)(c / kSpecBlock) * (N + 1) * kSpecBlock + c % kSpecBlock : (long long)c;
}
template <int CPB>
__device__ __forceinline__ long long spec_stride(long long fs) {
    return fs < 0 ? kSpecBlock : fs;
}

// tree_reduce (distributed.cpp:36-47) of {(y0, y1), peer values at element
// `off`} in member order, level by level: v[a] += v[a + step].
__device__ __forceinline__ void peer_tree_reduce(const C2REpilogue& epi, long long off, double& y0, double& y1) {
    double a0[kMaxFusedPeers + 1], a1[kMaxFusedPeers + 1];
    a0[0] = y0;
    a1[0] = y1;
    const int m = epi.npeers + 1;
#pragma unroll
    for (int k = 1; k <= kMaxFusedPeers; ++k) {
        if (k < m) {
            const double2 pv = __ldg(reinterpret_cast<const double2*>(epi.peers[k - 1] + off));
            a0[k] = pv.x;
            a1[k] = pv.y;
        } else {
            a0[k] = a1[k] = 0.0;
        }
    }
#pragma unroll
    for (int step = 1; step <= kMaxFusedPeers; step *= 2)
#pragma unroll
        for (int a = 0; a + step <= kMaxFusedPeers; a += 2 * step)
            if (a + step < m) {
                a0[a] += a0[a + step];
                a1[a] += a1[a + step];
            }
    y0 = a0[0];
    y1 = a1[0];
}

// CTA sum of the folded dot product (C2REpilogue::dot_out), one value per CTA.
__device__ __forceinline__ void cta_dot_store(double acc, double* out) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        out[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------------------
// r2c: SOTI rows (time contiguous) -> frequency-major out[k*out_fs + c]
// ---------------------------------------------------------------------------
template <int N, int CPB>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, kMinBlocksR2C<N, CPB>)
    k_r2c_fast(const double* __restrict__ in, long long in_cs, double2* __restrict__ out, long long out_fs,
               int channels, FastTables tabs, R2CBlockMax bm) {
    using P = FastPlan<N>;
    using RL = typename P::R2C;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;  // W_{2N} tables
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, false>();
    constexpr int LIM = TabPlan<N>::R2C;
    load_direct_tables<N, LIM, RL, false>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    const int b = threadIdx.x % CPB;
    const long long ofs = spec_stride<CPB>(out_fs);
    const int tc = threadIdx.x / CPB;
    const int c = blockIdx.x * CPB + b;
    const bool live = c < channels;
    double2* s = sm + b * CS;
    __syncthreads();

    // ---- pass 1 from global: z[n] = (x[2n], x[2n+1]); n = j + q NB < N/2 iff q < R/2
    {
        constexpr int R = first_radix(RL{});
        constexpr int NB = N / R;
        constexpr int BF = (NB + TPC - 1) / TPC;
        const double2* row = reinterpret_cast<const double2*>(in + (long long)c * in_cs);
        double2 v[BF][R];
#pragma unroll
        for (int bf = 0; bf < BF; ++bf) {
            const int j = tc + bf * TPC;
            if (NB % TPC == 0 || j < NB) {
#pragma unroll
                for (int q = 0; q < R; ++q)
                    v[bf][q] = (q < R / 2 && live) ? __ldg(row + j + q * NB) : make_double2(0.0, 0.0);
                dft<R, -1, true>(v[bf]);
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
    }
    // ---- middle passes
    passes_but_last<N, TPC, first_radix(RL{}), -1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

    // ---- last pass on butterfly pairs (j, NB-j) + split in registers
    constexpr int R = last_radix(RL{});
    constexpr int NS = ns_of_last(RL{});
    constexpr int NB = N / R;  // == NS
    constexpr int NU = NB / 2;
    constexpr int UF = (NU + TPC - 1) / TPC;
    if (!live) return;  // no barrier follows
    double2* orow = out + spec_base<N, CPB>(c, out_fs);
#pragma unroll
    for (int uf = 0; uf < UF; ++uf) {
        const int u = tc + uf * TPC;
        if (NU % TPC != 0 && u >= NU) break;
        const int ja = u == 0 ? 0 : u;
        const int jb = u == 0 ? NB / 2 : NB - u;
        double2 va[R], vb[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            va[q] = s[pad_idx(ja + q * NB)];
            vb[q] = s[pad_idx(jb + q * NB)];
        }
        twiddle_pass<N, R, NS, -1, LIM>(va, ja, lo, hi, w2q, ptab_last);
        twiddle_pass<N, R, NS, -1, LIM>(vb, jb, lo, hi, w2q, ptab_last);
        dft<R, -1>(va);
        dft<R, -1>(vb);
        if (u != 0) {
            // position ja + q NB pairs with jb + (R-1-q) NB
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int k = ja + q * NB;
                const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                double2 xk, xn;
                split_pair(va[q], vb[R - 1 - q], w, xk, xn);
                orow[(long long)k * ofs] = xk;
                orow[(long long)(N - k) * ofs] = xn;
                if (bm.pexp) {
                    block_max<CPB>(bm, c - b, b, k, xk);
                    block_max<CPB>(bm, c - b, b, N - k, xn);
                }
            }
        } else {
            // butterfly 0: positions q NB pair with ((R - q) % R) NB; q = 0 gives X_0 and X_N
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int qp = (R - q) % R;
                if (q > qp && q != 0) continue;
                const int k = q * NB;
                const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                double2 xk, xn;
                split_pair(va[q], va[qp], w, xk, xn);
                orow[(long long)k * ofs] = xk;
                if (q != qp || q == 0) orow[(long long)(N - k) * ofs] = xn;
                if (bm.pexp) {
                    block_max<CPB>(bm, c - b, b, k, xk);
                    if (q != qp || q == 0) block_max<CPB>(bm, c - b, b, N - k, xn);
                }
            }
            // butterfly NB/2: positions NB/2 + q NB pair with index R-1-q
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int qp = R - 1 - q;
                if (q > qp) continue;
                const int k = NB / 2 + q * NB;
                const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                double2 xk, xn;
                split_pair(vb[q], vb[qp], w, xk, xn);
                orow[(long long)k * ofs] = xk;
                if (q != qp) orow[(long long)(N - k) * ofs] = xn;
                if (bm.pexp) {
                    block_max<CPB>(bm, c - b, b, k, xk);
                    if (q != qp) block_max<CPB>(bm, c - b, b, N - k, xn);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// c2r: frequency-major in[k*in_fs + c] -> SOTI rows out[c*out_cs + t], t < N
// ---------------------------------------------------------------------------
template <int N, int CPB, bool PEERS = false, bool LIGHT = false>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, kMinBlocksC2R<N, CPB>)
    k_c2r_fast(const double2* __restrict__ in, long long in_fs, double* __restrict__ out, long long out_cs,
               int channels, FastTables tabs, C2REpilogue epi) {
    using P = FastPlan<N>;
    using RL = typename P::C2R;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, true>();
    constexpr int LIM = TabPlan<N>::C2R;
    load_direct_tables<N, LIM, RL, true>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    const int b = threadIdx.x % CPB;
    const long long ifs = spec_stride<CPB>(in_fs);
    const int tc = threadIdx.x / CPB;
    const int c = blockIdx.x * CPB + b;
    const bool live = c < channels;
    double2* s = sm + b * CS;
    __syncthreads();

    // ---- pass 1 on butterfly pairs: Z from (X_k, X_{N-k}) loaded frequency-major
    {
        constexpr int R = first_radix(RL{});
        constexpr int NB = N / R;
        constexpr int NU = NB / 2;
        constexpr int UF = (NU + TPC - 1) / TPC;
        constexpr double inv_len = 0.5 / N;
        const double2* col = in + spec_base<N, CPB>(c, in_fs);
        auto X = [&](int k) { return live ? __ldg(col + (long long)k * ifs) : make_double2(0.0, 0.0); };
        double2 va[UF][R], vb[UF][R];
#pragma unroll
        for (int uf = 0; uf < UF; ++uf) {
            const int u = tc + uf * TPC;
            if (NU % TPC != 0 && u >= NU) continue;
            const int ja = u == 0 ? 0 : u;
            if (u != 0) {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int k = ja + q * NB;  // partner N - k = jb + (R-1-q) NB
                    const double2 xk = X(k), xn = X(N - k);
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    presplit_pair(xk, xn, w, inv_len, va[uf][q], vb[uf][R - 1 - q]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int qp = (R - q) % R;
                    if (q > qp && q != 0) continue;
                    const int k = q * NB;
                    const double2 xk = X(k), xn = X(N - k);  // q = 0: X_0 and X_N
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    double2 zk, zn;
                    presplit_pair(xk, xn, w, inv_len, zk, zn);
                    va[uf][q] = zk;
                    if (q != qp) va[uf][qp] = zn;
                }
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int qp = R - 1 - q;
                    if (q > qp) continue;
                    const int k = NB / 2 + q * NB;
                    const double2 xk = X(k), xn = X(N - k);
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    double2 zk, zn;
                    presplit_pair(xk, xn, w, inv_len, zk, zn);
                    vb[uf][q] = zk;
                    if (q != qp) vb[uf][qp] = zn;
                }
            }
            dft<R, +1>(va[uf]);
            dft<R, +1>(vb[uf]);
        }
#pragma unroll
        for (int uf = 0; uf < UF; ++uf) {
            const int u = tc + uf * TPC;
            if (NU % TPC != 0 && u >= NU) continue;
            const int ja = u == 0 ? 0 : u;
            const int jb = u == 0 ? NB / 2 : NB - u;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                s[pad_idx(ja * R + q)] = va[uf][q];
                s[pad_idx(jb * R + q)] = vb[uf][q];
            }
        }
        __syncthreads();
    }
    // ---- middle passes
    passes_but_last<N, TPC, first_radix(RL{}), +1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

    // ---- last pass: outputs p = j + q NB; keep p < N/2 (t = 2p, 2p+1 < N)
    constexpr int R = last_radix(RL{});
    constexpr int NS = ns_of_last(RL{});
    constexpr int NB = N / R;
    constexpr int BF = (NB + TPC - 1) / TPC;
    double dacc = 0.0;  // folded dot (epi.dot_out)
    if (live) {
    double* orow = out + (long long)c * out_cs;
    const double* vrow = (!LIGHT && epi.v) ? epi.v + (long long)c * out_cs : nullptr;
    const double* drow = epi.dot_out ? epi.dot_v + (long long)c * out_cs : nullptr;
#pragma unroll
    for (int bf = 0; bf < BF; ++bf) {
        const int j = tc + bf * TPC;
        if (NB % TPC == 0 || j < NB) {
            // epilogue operands first (16-byte loads), so their latency overlaps the pass
            constexpr int NQ = (R + 1) / 2;
            double2 er[NQ], eg[NQ];
            double el[NQ], eh[NQ];
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int p = j + q * NB;
                const bool ok = p < N / 2;
                const int t0 = 2 * p;
                er[q] = (vrow && ok) ? __ldg(reinterpret_cast<const double2*>(vrow) + p) : make_double2(0.0, 0.0);
                el[q] = (vrow && ok && epi.reg_kind == 1 && t0 > 0) ? __ldg(vrow + t0 - 1) : 0.0;
                eh[q] = (vrow && ok && epi.reg_kind == 1 && t0 + 2 < N) ? __ldg(vrow + t0 + 2) : 0.0;
                eg[q] = (!LIGHT && epi.gamma_mode == 2 && ok)
                            ? __ldg(reinterpret_cast<const double2*>(epi.gamma + (long long)(c % epi.gamma_dim) * N) + p)
                            : make_double2(1.0, 1.0);
            }
            double2 v[R];
            #pragma unroll
            for (int q = 0; q < R; ++q) v[q] = s[pad_idx(j + q * NB)];
            twiddle_pass<N, R, NS, +1, LIM>(v, j, lo, hi, w2q, ptab_last);
            dft<R, +1>(v);
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {  // keep p = j + q*NB < N/2 (unpad)
                const int p = j + q * NB;
                if ((R % 2 == 1) && q == R / 2 && p >= N / 2) break;
                double y0 = v[q].x, y1 = v[q].y;
                if (epi.gamma_mode == 1) {
                    const double g = __ldg(epi.gamma + (c % epi.gamma_dim));
                    y0 *= g;
                    y1 *= g;
                } else if (!LIGHT && epi.gamma_mode == 2) {
                    y0 *= eg[q].x;
                    y1 *= eg[q].y;
                }
                if (vrow) {
                    double r0 = er[q].x, r1 = er[q].y;
                    if (epi.reg_kind == 1) {
                        const double a0 = 2.0 * r0 - el[q] - r1;  // reference order: 2x - x[t-1] - x[t+1]
                        const double a1 = 2.0 * r1 - r0 - eh[q];
                        r0 = a0;
                        r1 = a1;
                    }
                    y0 += epi.alpha * r0;
                    y1 += epi.alpha * r1;
                }
                if constexpr (PEERS) peer_tree_reduce(epi, (long long)c * out_cs + 2 * p, y0, y1);
                reinterpret_cast<double2*>(orow)[p] = make_double2(y0, y1);
                if (drow) {
                    const double2 dv = __ldg(reinterpret_cast<const double2*>(drow) + p);
                    dacc = fma(dv.x, y0, fma(dv.y, y1, dacc));
                }
            }
        }
    }
    }
    if (epi.dot_out) cta_dot_store(dacc, epi.dot_out);
}

// ---------------------------------------------------------------------------
// c2r from the channel-blocked layout (kBlockedFs) with TMA: persistent CTAs,
// two per SM (<= 128 registers); the CTA's whole input — one contiguous
// (N+1) x CPB block — arrives by ONE bulk copy into the channel buffers, the
// first pass reads its (X_k, X_{N-k}) pairs from there, and the next group's
// block is requested as soon as the last pass has read the buffers, so it lands
// under the Gamma^-1 / alpha R v epilogue and the stores.
// ---------------------------------------------------------------------------
#ifndef BTG_C2R_TMA_MINB
#define BTG_C2R_TMA_MINB 1
#endif
template <int N, int CPB>
__host__ __device__ constexpr bool c2r_tma_ok() {
    return CPB == kSpecBlock &&
           (N / last_radix(typename FastPlan<N>::C2R{}) + FastPlan<N>::TPC - 1) / FastPlan<N>::TPC == 1 &&
           (size_t)(N + 1) * CPB <= (size_t)CPB * chan_stride<CPB>(N);
}
#ifndef BTG_C2R_TMA_STAGE
#define BTG_C2R_TMA_STAGE 1
#endif
constexpr bool kC2RTmaStage = BTG_C2R_TMA_STAGE;
// The LIGHT instantiation (no prefetched per-sample epilogue operands: <= 128
// registers) runs two CTAs per SM with the block landing in the channel buffers
// (the copy overlaps the other CTA's passes); the full-epilogue one (176
// registers, one CTA per SM) keeps the separate staging block. Measured at
// 524288 channels (profiles/r02s4_fft_c2r_light.md): 3.03 ms (full, staged) ->
// 2.79 (light, staged, one CTA) -> 2.73 (light, aliased, two CTAs).
template <bool LIGHT>
constexpr bool c2r_tma_stage() { return LIGHT ? false : kC2RTmaStage; }
template <int N, int CPB, bool LIGHT = false>
__host__ __device__ constexpr size_t smem_bytes_c2r_tma() {
    return smem_dir<N, CPB, false>() + 16 + (c2r_tma_stage<LIGHT>() ? sizeof(double2) * (N + 1) * CPB : 0);
}
// LIGHT: no per-sample epilogue operands (epi.v == nullptr, gamma_mode != 2) —
// the instantiation without the prefetched operand registers.
template <int N, int CPB, bool LIGHT = false>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, LIGHT ? 2 : BTG_C2R_TMA_MINB)
    k_c2r_tma(const double2* __restrict__ in, long long in_fs, double* __restrict__ out, long long out_cs,
               int channels, FastTables tabs, C2REpilogue epi) {
    (void)in_fs;  // always channel-blocked
    constexpr bool kStage = c2r_tma_stage<LIGHT>();
    using P = FastPlan<N>;
    using RL = typename P::C2R;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, true>();
    constexpr int LIM = TabPlan<N>::C2R;
    load_direct_tables<N, LIM, RL, true>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    const int b = threadIdx.x % CPB;
    const int tc = threadIdx.x / CPB;
    double2* s = sm + b * CS;
    // the group's channel-blocked input block lands where the channel buffers are
    // kStage: a separate staging block (the next group's copy overlaps all
    // passes) or the channel buffers themselves (copy overlaps the epilogue only)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + smem_dir<N, CPB, false>() / sizeof(double2));
    double2* stage_buf = kStage ? reinterpret_cast<double2*>(bar + 2) : sm;
    const double2* stage = stage_buf;
    const int groups = channels / CPB;
    constexpr uint32_t kBlockBytes = (uint32_t)((N + 1) * CPB * sizeof(double2));
    auto issue = [&](int g) {
        umma::mbar_expect_tx(bar, kBlockBytes);
        umma::bulk_load(stage_buf, in + (long long)g * (N + 1) * CPB, kBlockBytes, bar, umma::policy_evict_first());
    };
    if (threadIdx.x == 0) {
        umma::mbar_init(bar, 1);
        umma::mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < groups) issue(blockIdx.x);
    double dacc = 0.0;  // folded dot (epi.dot_out), over every group of this CTA
    uint32_t phase = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, phase ^= 1u) {
    const int c = g * CPB + b;
    const bool live = true;
    umma::mbar_wait(bar, phase);

    // ---- pass 1 on butterfly pairs: Z from (X_k, X_{N-k}) loaded frequency-major
    {
        constexpr int R = first_radix(RL{});
        constexpr int NB = N / R;
        constexpr int NU = NB / 2;
        constexpr int UF = (NU + TPC - 1) / TPC;
        constexpr double inv_len = 0.5 / N;
        auto X = [&](int k) { return stage[k * CPB + b]; };
        double2 va[UF][R], vb[UF][R];
#pragma unroll
        for (int uf = 0; uf < UF; ++uf) {
            const int u = tc + uf * TPC;
            if (NU % TPC != 0 && u >= NU) continue;
            const int ja = u == 0 ? 0 : u;
            if (u != 0) {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int k = ja + q * NB;  // partner N - k = jb + (R-1-q) NB
                    const double2 xk = X(k), xn = X(N - k);
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    presplit_pair(xk, xn, w, inv_len, va[uf][q], vb[uf][R - 1 - q]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int qp = (R - q) % R;
                    if (q > qp && q != 0) continue;
                    const int k = q * NB;
                    const double2 xk = X(k), xn = X(N - k);  // q = 0: X_0 and X_N
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    double2 zk, zn;
                    presplit_pair(xk, xn, w, inv_len, zk, zn);
                    va[uf][q] = zk;
                    if (q != qp) va[uf][qp] = zn;
                }
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int qp = R - 1 - q;
                    if (q > qp) continue;
                    const int k = NB / 2 + q * NB;
                    const double2 xk = X(k), xn = X(N - k);
                    const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                    double2 zk, zn;
                    presplit_pair(xk, xn, w, inv_len, zk, zn);
                    vb[uf][q] = zk;
                    if (q != qp) vb[uf][qp] = zn;
                }
            }
            dft<R, +1>(va[uf]);
            dft<R, +1>(vb[uf]);
        }
        // every pair read from the staged block before any buffer write (aliased
        // stage) / before the next block is requested (separate stage)
        __syncthreads();
        if (kStage && threadIdx.x == 0 && g + (int)gridDim.x < groups) issue(g + gridDim.x);
#pragma unroll
        for (int uf = 0; uf < UF; ++uf) {
            const int u = tc + uf * TPC;
            if (NU % TPC != 0 && u >= NU) continue;
            const int ja = u == 0 ? 0 : u;
            const int jb = u == 0 ? NB / 2 : NB - u;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                s[pad_idx(ja * R + q)] = va[uf][q];
                s[pad_idx(jb * R + q)] = vb[uf][q];
            }
        }
        __syncthreads();
    }
    // ---- middle passes
    passes_but_last<N, TPC, first_radix(RL{}), +1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

    // ---- last pass: outputs p = j + q NB; keep p < N/2 (t = 2p, 2p+1 < N)
    constexpr int R = last_radix(RL{});
    constexpr int NS = ns_of_last(RL{});
    constexpr int NB = N / R;
    constexpr int BF = (NB + TPC - 1) / TPC;
    {
    double* orow = out + (long long)c * out_cs;
    const double* vrow = (!LIGHT && epi.v) ? epi.v + (long long)c * out_cs : nullptr;
    const double* drow = epi.dot_out ? epi.dot_v + (long long)c * out_cs : nullptr;
#pragma unroll
    for (int bf = 0; bf < BF; ++bf) {
        const int j = tc + bf * TPC;
        if (NB % TPC == 0 || j < NB) {
            // epilogue operands first (16-byte loads), so their latency overlaps the pass
            constexpr int NQ = (R + 1) / 2;
            double2 er[NQ], eg[NQ];
            double el[NQ], eh[NQ];
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int p = j + q * NB;
                const bool ok = p < N / 2;
                const int t0 = 2 * p;
                er[q] = (vrow && ok) ? __ldg(reinterpret_cast<const double2*>(vrow) + p) : make_double2(0.0, 0.0);
                el[q] = (vrow && ok && epi.reg_kind == 1 && t0 > 0) ? __ldg(vrow + t0 - 1) : 0.0;
                eh[q] = (vrow && ok && epi.reg_kind == 1 && t0 + 2 < N) ? __ldg(vrow + t0 + 2) : 0.0;
                eg[q] = (!LIGHT && epi.gamma_mode == 2 && ok)
                            ? __ldg(reinterpret_cast<const double2*>(epi.gamma + (long long)(c % epi.gamma_dim) * N) + p)
                            : make_double2(1.0, 1.0);
            }
            double2 v[R];
            #pragma unroll
            for (int q = 0; q < R; ++q) v[q] = s[pad_idx(j + q * NB)];
            static_assert(BF == 1, "one last-pass butterfly per thread: the refill follows its reads");
            if (!kStage) {
                __syncthreads();  // every channel buffer read: the next block may land
                if (threadIdx.x == 0 && g + (int)gridDim.x < groups) issue(g + gridDim.x);
            }
            twiddle_pass<N, R, NS, +1, LIM>(v, j, lo, hi, w2q, ptab_last);
            dft<R, +1>(v);
            #pragma unroll
            for (int q = 0; q < NQ; ++q) {  // keep p = j + q*NB < N/2 (unpad)
                const int p = j + q * NB;
                if ((R % 2 == 1) && q == R / 2 && p >= N / 2) break;
                double y0 = v[q].x, y1 = v[q].y;
                if (epi.gamma_mode == 1) {
                    const double g = __ldg(epi.gamma + (c % epi.gamma_dim));
                    y0 *= g;
                    y1 *= g;
                } else if (!LIGHT && epi.gamma_mode == 2) {
                    y0 *= eg[q].x;
                    y1 *= eg[q].y;
                }
                if (vrow) {
                    double r0 = er[q].x, r1 = er[q].y;
                    if (epi.reg_kind == 1) {
                        const double a0 = 2.0 * r0 - el[q] - r1;  // reference order: 2x - x[t-1] - x[t+1]
                        const double a1 = 2.0 * r1 - r0 - eh[q];
                        r0 = a0;
                        r1 = a1;
                    }
                    y0 += epi.alpha * r0;
                    y1 += epi.alpha * r1;
                }
                reinterpret_cast<double2*>(orow)[p] = make_double2(y0, y1);
                if (drow) {
                    const double2 dv = __ldg(reinterpret_cast<const double2*>(drow) + p);
                    dacc = fma(dv.x, y0, fma(dv.y, y1, dacc));
                }
            }
        }
    }
    }
    }
    if (epi.dot_out) cta_dot_store(dacc, epi.dot_out);
}

// ---------------------------------------------------------------------------
// Persistent variants (plans with PF_R2C / PF_C2R): the same passes, looping
// over channel groups (group g = blockIdx.x + i gridDim.x); the first pass's
// global loads for the NEXT group are issued into registers right after this
// group's first pass consumed them, so they are in flight during the
// shared-memory passes and the stores.
// ---------------------------------------------------------------------------
template <int N, int CPB>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, kMinBlocksR2C<N, CPB>)
    k_r2c_pf(const double* __restrict__ in, long long in_cs, double2* __restrict__ out, long long out_fs,
               int channels, FastTables tabs, R2CBlockMax bm) {
    using P = FastPlan<N>;
    using RL = typename P::R2C;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    constexpr int R1 = first_radix(RL{});
    constexpr int NB1 = N / R1;
    constexpr int BF1 = (NB1 + TPC - 1) / TPC;
    constexpr int QH = R1 / 2;  // z[n], n = j + q NB1 < N/2 iff q < R1/2: the rest is zero pad
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;  // W_{2N} tables
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, false>();
    constexpr int LIM = TabPlan<N>::R2C;
    load_direct_tables<N, LIM, RL, false>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    const int b = threadIdx.x % CPB;
    const long long ofs = spec_stride<CPB>(out_fs);
    const int tc = threadIdx.x / CPB;
    double2* s = sm + b * CS;
    const int groups = (channels + CPB - 1) / CPB;

    double2 pre[BF1][QH];
    auto prefetch = [&](int g) {
        const int c = g * CPB + b;
        const bool ok = g < groups && c < channels;
        const double2* row = reinterpret_cast<const double2*>(in + (long long)(ok ? c : 0) * in_cs);
#pragma unroll
        for (int bf = 0; bf < BF1; ++bf) {
            const int j = tc + bf * TPC;
            const bool jl = ok && (NB1 % TPC == 0 || j < NB1);
#pragma unroll
            for (int q = 0; q < QH; ++q) pre[bf][q] = jl ? __ldg(row + j + q * NB1) : make_double2(0.0, 0.0);
        }
    };
    prefetch(blockIdx.x);
    __syncthreads();

    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        const int c = g * CPB + b;
        const bool live = c < channels;
        // ---- pass 1 from the prefetched registers: z[n] = (x[2n], x[2n+1])
        {
            double2 v[BF1][R1];
#pragma unroll
            for (int bf = 0; bf < BF1; ++bf) {
#pragma unroll
                for (int q = 0; q < R1; ++q) v[bf][q] = q < QH ? pre[bf][q] : make_double2(0.0, 0.0);
                dft<R1, -1, true>(v[bf]);
            }
            prefetch(g + gridDim.x);
#pragma unroll
            for (int bf = 0; bf < BF1; ++bf) {
                const int j = tc + bf * TPC;
                if (NB1 % TPC == 0 || j < NB1) {
#pragma unroll
                    for (int q = 0; q < R1; ++q) s[pad_idx(j * R1 + q)] = v[bf][q];
                }
            }
            __syncthreads();
        }
        // ---- middle passes
        passes_but_last<N, TPC, R1, -1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

        // ---- last pass on butterfly pairs (j, NB-j) + split in registers
        constexpr int R = last_radix(RL{});
        constexpr int NS = ns_of_last(RL{});
        constexpr int NB = N / R;  // == NS
        constexpr int NU = NB / 2;
        constexpr int UF = (NU + TPC - 1) / TPC;
        if (live) {
            double2* orow = out + spec_base<N, CPB>(c, out_fs);
#pragma unroll
            for (int uf = 0; uf < UF; ++uf) {
                const int u = tc + uf * TPC;
                if (NU % TPC != 0 && u >= NU) break;
                const int ja = u == 0 ? 0 : u;
                const int jb = u == 0 ? NB / 2 : NB - u;
                double2 va[R], vb[R];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    va[q] = s[pad_idx(ja + q * NB)];
                    vb[q] = s[pad_idx(jb + q * NB)];
                }
                twiddle_pass<N, R, NS, -1, LIM>(va, ja, lo, hi, w2q, ptab_last);
                twiddle_pass<N, R, NS, -1, LIM>(vb, jb, lo, hi, w2q, ptab_last);
                dft<R, -1>(va);
                dft<R, -1>(vb);
                if (u != 0) {
                    // position ja + q NB pairs with jb + (R-1-q) NB
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int k = ja + q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(va[q], vb[R - 1 - q], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
                } else {
                    // butterfly 0: positions q NB pair with ((R - q) % R) NB; q = 0 gives X_0 and X_N
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int qp = (R - q) % R;
                        if (q > qp && q != 0) continue;
                        const int k = q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(va[q], va[qp], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        if (q != qp || q == 0) orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            if (q != qp || q == 0) block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
                    // butterfly NB/2: positions NB/2 + q NB pair with index R-1-q
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int qp = R - 1 - q;
                        if (q > qp) continue;
                        const int k = NB / 2 + q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(vb[q], vb[qp], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        if (q != qp) orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            if (q != qp) block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
                }
            }
        }
        __syncthreads();  // the next group's first pass overwrites s
    }
}

// c2r, persistent: the (X_k, X_{N-k}) pairs of the next group's first pass are
// loaded into registers while this group finishes.
// LIGHT as k_c2r_tma: no prefetched per-sample epilogue operands. N_t = 1024 at
// 32768 channels (profiles/r02s4_fft_c2r_light.md): 255 -> 220 registers, C2R
// 0.247 -> 0.222 ms at one CTA per SM; forcing two CTAs (128 registers) spills
// and is slower (0.282 ms), three (80) much slower (0.588).
#ifndef BTG_C2R_PF_LIGHT_MINB
#define BTG_C2R_PF_LIGHT_MINB 1
#endif
template <int N, int CPB, bool LIGHT>
constexpr int kMinBlocksC2RPf =
    (LIGHT && kMinBlocksC2R<N, CPB> < BTG_C2R_PF_LIGHT_MINB) ? BTG_C2R_PF_LIGHT_MINB : kMinBlocksC2R<N, CPB>;
template <int N, int CPB, bool LIGHT = false>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, (kMinBlocksC2RPf<N, CPB, LIGHT>))
    k_c2r_pf(const double2* __restrict__ in, long long in_fs, double* __restrict__ out, long long out_cs,
               int channels, FastTables tabs, C2REpilogue epi) {
    using P = FastPlan<N>;
    using RL = typename P::C2R;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    constexpr int R1 = first_radix(RL{});
    constexpr int NB1 = N / R1;
    constexpr int NU1 = NB1 / 2;
    constexpr int UF1 = (NU1 + TPC - 1) / TPC;
    constexpr double inv_len = 0.5 / N;
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;
    double2* phi = plo + kTwLo;
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, true>();
    constexpr int LIM = TabPlan<N>::C2R;
    load_direct_tables<N, LIM, RL, true>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    const int b = threadIdx.x % CPB;
    const long long ifs = spec_stride<CPB>(in_fs);
    const int tc = threadIdx.x / CPB;
    double2* s = sm + b * CS;
    const int groups = (channels + CPB - 1) / CPB;

    // xa/xb[uf][q] = X(k), X(N-k) for k = ja + q NB1; xc/xd[q] = X(k), X(N-k) for
    // k = NB1/2 + q NB1 (butterfly NB1/2, only on the thread that owns u = 0)
    double2 xa[UF1][R1], xb[UF1][R1], xc[R1], xd[R1];
    auto prefetch = [&](int g) {
        const int c = g * CPB + b;
        const bool ok = g < groups && c < channels;
        const double2* col = in + spec_base<N, CPB>(ok ? c : 0, in_fs);
        auto X = [&](int k, bool use) {
            return (ok && use) ? __ldg(col + (long long)k * ifs) : make_double2(0.0, 0.0);
        };
#pragma unroll
        for (int uf = 0; uf < UF1; ++uf) {
            const int u = tc + uf * TPC;
            const bool ul = NU1 % TPC == 0 || u < NU1;
#pragma unroll
            for (int q = 0; q < R1; ++q) {
                const int k = u + q * NB1;
                xa[uf][q] = X(k, ul);
                xb[uf][q] = X(N - k, ul);
            }
        }
        const bool owner = tc == 0;
#pragma unroll
        for (int q = 0; q < R1; ++q) {
            const int k = NB1 / 2 + q * NB1;
            xc[q] = X(k, owner && q <= R1 - 1 - q);
            xd[q] = X(N - k, owner && q <= R1 - 1 - q);
        }
    };
    prefetch(blockIdx.x);
    __syncthreads();

    double dacc = 0.0;  // folded dot (epi.dot_out), over every group of this CTA
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        const int c = g * CPB + b;
        const bool live = c < channels;
        // ---- pass 1 on butterfly pairs: Z from (X_k, X_{N-k})
        {
            double2 va[UF1][R1], vb[UF1][R1];
#pragma unroll
            for (int uf = 0; uf < UF1; ++uf) {
                const int u = tc + uf * TPC;
                if (NU1 % TPC != 0 && u >= NU1) continue;
                const int ja = u;
                if (u != 0) {
#pragma unroll
                    for (int q = 0; q < R1; ++q) {
                        const int k = ja + q * NB1;  // partner N - k = jb + (R-1-q) NB
                        const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                        presplit_pair(xa[uf][q], xb[uf][q], w, inv_len, va[uf][q], vb[uf][R1 - 1 - q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < R1; ++q) {
                        const int qp = (R1 - q) % R1;
                        if (q > qp && q != 0) continue;
                        const int k = q * NB1;  // q = 0: X_0 and X_N
                        const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                        double2 zk, zn;
                        presplit_pair(xa[uf][q], xb[uf][q], w, inv_len, zk, zn);
                        va[uf][q] = zk;
                        if (q != qp) va[uf][qp] = zn;
                    }
#pragma unroll
                    for (int q = 0; q < R1; ++q) {
                        const int qp = R1 - 1 - q;
                        if (q > qp) continue;
                        const int k = NB1 / 2 + q * NB1;
                        const double2 w = w2n_lookup<N, true>(w2q, plo, phi, k);
                        double2 zk, zn;
                        presplit_pair(xc[q], xd[q], w, inv_len, zk, zn);
                        vb[uf][q] = zk;
                        if (q != qp) vb[uf][qp] = zn;
                    }
                }
                dft<R1, +1>(va[uf]);
                dft<R1, +1>(vb[uf]);
            }
            prefetch(g + gridDim.x);
#pragma unroll
            for (int uf = 0; uf < UF1; ++uf) {
                const int u = tc + uf * TPC;
                if (NU1 % TPC != 0 && u >= NU1) continue;
                const int ja = u == 0 ? 0 : u;
                const int jb = u == 0 ? NB1 / 2 : NB1 - u;
#pragma unroll
                for (int q = 0; q < R1; ++q) {
                    s[pad_idx(ja * R1 + q)] = va[uf][q];
                    s[pad_idx(jb * R1 + q)] = vb[uf][q];
                }
            }
            __syncthreads();
        }
        // ---- middle passes
        passes_but_last<N, TPC, R1, +1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

        // ---- last pass: outputs p = j + q NB; keep p < N/2 (t = 2p, 2p+1 < N)
        constexpr int R = last_radix(RL{});
        constexpr int NS = ns_of_last(RL{});
        constexpr int NB = N / R;
        constexpr int BF = (NB + TPC - 1) / TPC;
        if (live) {
            double* orow = out + (long long)c * out_cs;
            const double* vrow = (!LIGHT && epi.v) ? epi.v + (long long)c * out_cs : nullptr;
            const double* drow = epi.dot_out ? epi.dot_v + (long long)c * out_cs : nullptr;
#pragma unroll
            for (int bf = 0; bf < BF; ++bf) {
                const int j = tc + bf * TPC;
                if (NB % TPC == 0 || j < NB) {
                    // epilogue operands first (16-byte loads), so their latency overlaps the pass
                    constexpr int NQ = (R + 1) / 2;
                    double2 er[NQ], eg[NQ];
                    double el[NQ], eh[NQ];
                    #pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int p = j + q * NB;
                        const bool ok = p < N / 2;
                        const int t0 = 2 * p;
                        er[q] = (vrow && ok) ? __ldg(reinterpret_cast<const double2*>(vrow) + p) : make_double2(0.0, 0.0);
                        el[q] = (vrow && ok && epi.reg_kind == 1 && t0 > 0) ? __ldg(vrow + t0 - 1) : 0.0;
                        eh[q] = (vrow && ok && epi.reg_kind == 1 && t0 + 2 < N) ? __ldg(vrow + t0 + 2) : 0.0;
                        eg[q] = (!LIGHT && epi.gamma_mode == 2 && ok)
                                    ? __ldg(reinterpret_cast<const double2*>(epi.gamma + (long long)(c % epi.gamma_dim) * N) + p)
                                    : make_double2(1.0, 1.0);
                    }
                    double2 v[R];
                    #pragma unroll
                    for (int q = 0; q < R; ++q) v[q] = s[pad_idx(j + q * NB)];
                    twiddle_pass<N, R, NS, +1, LIM>(v, j, lo, hi, w2q, ptab_last);
                    dft<R, +1>(v);
                    #pragma unroll
                    for (int q = 0; q < NQ; ++q) {  // keep p = j + q*NB < N/2 (unpad)
                        const int p = j + q * NB;
                        if ((R % 2 == 1) && q == R / 2 && p >= N / 2) break;
                        double y0 = v[q].x, y1 = v[q].y;
                        if (epi.gamma_mode == 1) {
                            const double g = __ldg(epi.gamma + (c % epi.gamma_dim));
                            y0 *= g;
                            y1 *= g;
                        } else if (!LIGHT && epi.gamma_mode == 2) {
                            y0 *= eg[q].x;
                            y1 *= eg[q].y;
                        }
                        if (vrow) {
                            double r0 = er[q].x, r1 = er[q].y;
                            if (epi.reg_kind == 1) {
                                const double a0 = 2.0 * r0 - el[q] - r1;  // reference order: 2x - x[t-1] - x[t+1]
                                const double a1 = 2.0 * r1 - r0 - eh[q];
                                r0 = a0;
                                r1 = a1;
                            }
                            y0 += epi.alpha * r0;
                            y1 += epi.alpha * r1;
                        }
                        reinterpret_cast<double2*>(orow)[p] = make_double2(y0, y1);
                        if (drow) {
                            const double2 dv = __ldg(reinterpret_cast<const double2*>(drow) + p);
                            dacc = fma(dv.x, y0, fma(dv.y, y1, dacc));
                        }
                    }
                }
            }
        }
        __syncthreads();  // the next group's first pass overwrites s
    }
    if (epi.dot_out) cta_dot_store(dacc, epi.dot_out);
}

// ---------------------------------------------------------------------------
// r2c with TMA-staged input (plans with TMA_R2C): persistent CTAs; the CPB SOTI
// rows of the NEXT channel group are bulk-copied (cp.async.bulk, one 8·N_t-byte
// copy per row, mbarrier completion) into a shared staging area as soon as the
// first pass has read the current ones, so the loads overlap the shared-memory
// passes and the stores without costing registers. Staging rows are padded by
// 32 bytes so the CPB channels of a warp hit different banks.
// ---------------------------------------------------------------------------
template <int N>
__host__ __device__ constexpr int stage_stride() { return N + 4; }  // doubles per staged row: +32 B, so the
// CPB channel lanes of a quarter-warp hit 8 distinct 16-byte bank groups
template <int N, int CPB>
__host__ __device__ constexpr size_t smem_bytes_tma() {
    return smem_dir<N, CPB, true>() + sizeof(double) * CPB * stage_stride<N>() + 16;
}
// Plans that have the TMA-staged R2C, and the largest channel count it is used for:
// measured on B200 at N_t = 1024 it wins up to ~2e5 channels (32768: 0.194 vs 0.220 ms;
// 196608: 1.276 vs 1.309 ms) and loses beyond (262144: 1.82 vs 1.77; 524288: 3.8 vs
// 3.5 ms — 16 resident warps per SM instead of 24).
template <int N>
struct UseTmaR2C {
    static constexpr bool value = false;
    static constexpr int max_channels = 0;
};
template <>
struct UseTmaR2C<1024> {
    static constexpr bool value = true;
    static constexpr int max_channels = 196608;
};
// also measured ahead (up to the channel counts tested): 256 x 262144 0.39 vs 0.47 ms,
// 512 x 131072 0.43 vs 0.53, 2048 x 32768 0.62 vs 0.65; behind for 64, 1000, 4096
template <>
struct UseTmaR2C<256> {
    static constexpr bool value = true;
    static constexpr int max_channels = 262144;
};
template <>
struct UseTmaR2C<512> {
    static constexpr bool value = true;
    static constexpr int max_channels = 131072;
};
template <>
struct UseTmaR2C<2048> {
    static constexpr bool value = true;
    static constexpr int max_channels = 32768;
};

template <int N, int CPB>
__global__ void __launch_bounds__(FastPlan<N>::TPC * CPB, 2)
    k_r2c_tma(const double* __restrict__ in, long long in_cs, double2* __restrict__ out, long long out_fs,
              int channels, FastTables tabs, R2CBlockMax bm) {
    using P = FastPlan<N>;
    using RL = typename P::R2C;
    constexpr int TPC = P::TPC, CS = chan_stride<CPB>(N);
    constexpr int HI = tw_hi_count<N>();
    constexpr int R1 = first_radix(RL{});
    constexpr int NB1 = N / R1;
    constexpr int BF1 = (NB1 + TPC - 1) / TPC;
    constexpr int QH = R1 / 2;
    extern __shared__ double2 sm[];
    double2* lo = sm + CPB * CS;
    double2* hi = lo + kTwLo;
    double2* plo = hi + HI;
    double2* phi = plo + kTwLo;
    double* stage = reinterpret_cast<double*>(sm) + 2 * (smem_dir<N, CPB, true>() / sizeof(double2));
    uint64_t* bar = reinterpret_cast<uint64_t*>(stage + CPB * stage_stride<N>());
    const int b = threadIdx.x % CPB;
    const long long ofs = spec_stride<CPB>(out_fs);
    const int tc = threadIdx.x / CPB;
    double2* s = sm + b * CS;
    const int groups = (channels + CPB - 1) / CPB;

    auto issue = [&](int g) {  // one thread: the group's rows into the staging area
        const int c0 = g * CPB, nch = min(CPB, channels - c0);
        umma::mbar_expect_tx(bar, (uint32_t)(nch * N * sizeof(double)));
        const uint64_t pol = umma::policy_evict_first();
        for (int k = 0; k < nch; ++k)
            umma::bulk_load(stage + k * stage_stride<N>(), in + (long long)(c0 + k) * in_cs,
                            (uint32_t)(N * sizeof(double)), bar, pol);
    };
    if (threadIdx.x == 0) {
        umma::mbar_init(bar, 1);
        umma::mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < groups) issue(blockIdx.x);
    load_tables(lo, hi, HI, tabs.lo, tabs.hi);
    load_tables(plo, phi, HI + 1, tabs.post_lo, tabs.post_hi);
    double2* w2q = plo + kTwLo + HI + 2;  // == sm + CPB*CS + 2*kTwLo + 2*HI + 2
    double2* ptab = w2q + w2q_entries<N, false>();
    constexpr int LIM = TabPlan<N>::R2C;
    load_direct_tables<N, LIM, RL, false>(w2q, ptab, tabs);
    const double2* ptab_last = ptab + tab_entries_but_last<1, LIM>(RL{});
    __syncthreads();

    uint32_t phase = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, phase ^= 1u) {
        const int c = g * CPB + b;
        const bool live = c < channels;
        umma::mbar_wait(bar, phase);
        {
            const double2* row = reinterpret_cast<const double2*>(stage + b * stage_stride<N>());
            double2 v[BF1][R1];
#pragma unroll
            for (int bf = 0; bf < BF1; ++bf) {
                const int j = tc + bf * TPC;
#pragma unroll
                for (int q = 0; q < R1; ++q)
                    v[bf][q] = (q < QH && live && (NB1 % TPC == 0 || j < NB1)) ? row[j + q * NB1]
                                                                                : make_double2(0.0, 0.0);
                dft<R1, -1, true>(v[bf]);
            }
            __syncthreads();  // every staged row consumed: refill with the next group
            if (threadIdx.x == 0 && g + (int)gridDim.x < groups) issue(g + gridDim.x);
#pragma unroll
            for (int bf = 0; bf < BF1; ++bf) {
                const int j = tc + bf * TPC;
                if (NB1 % TPC == 0 || j < NB1) {
#pragma unroll
                    for (int q = 0; q < R1; ++q) s[pad_idx(j * R1 + q)] = v[bf][q];
                }
            }
            __syncthreads();
        }
        passes_but_last<N, TPC, R1, -1, LIM>(s, tc, lo, hi, w2q, ptab, tail(RL{}));

        constexpr int R = last_radix(RL{});
        constexpr int NS = ns_of_last(RL{});
        constexpr int NB = N / R;
        constexpr int NU = NB / 2;
        constexpr int UF = (NU + TPC - 1) / TPC;
        if (live) {
            double2* orow = out + spec_base<N, CPB>(c, out_fs);
#pragma unroll
            for (int uf = 0; uf < UF; ++uf) {
                const int u = tc + uf * TPC;
                if (NU % TPC != 0 && u >= NU) break;
                const int ja = u == 0 ? 0 : u;
                const int jb = u == 0 ? NB / 2 : NB - u;
                double2 va[R], vb[R];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    va[q] = s[pad_idx(ja + q * NB)];
                    vb[q] = s[pad_idx(jb + q * NB)];
                }
                twiddle_pass<N, R, NS, -1, LIM>(va, ja, lo, hi, w2q, ptab_last);
                twiddle_pass<N, R, NS, -1, LIM>(vb, jb, lo, hi, w2q, ptab_last);
                dft<R, -1>(va);
                dft<R, -1>(vb);
                if (u != 0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int k = ja + q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(va[q], vb[R - 1 - q], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int qp = (R - q) % R;
                        if (q > qp && q != 0) continue;
                        const int k = q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(va[q], va[qp], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        if (q != qp || q == 0) orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            if (q != qp || q == 0) block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int qp = R - 1 - q;
                        if (q > qp) continue;
                        const int k = NB / 2 + q * NB;
                        const double2 w = w2n_lookup<N, false>(w2q, plo, phi, k);
                        double2 xk, xn;
                        split_pair(vb[q], vb[qp], w, xk, xn);
                        orow[(long long)k * ofs] = xk;
                        if (q != qp) orow[(long long)(N - k) * ofs] = xn;
                        if (bm.pexp) {
                            block_max<CPB>(bm, c - b, b, k, xk);
                            if (q != qp) block_max<CPB>(bm, c - b, b, N - k, xn);
                        }
                    }
                }
            }
        }
        __syncthreads();  // the next group's first pass overwrites s
    }
}

}  // namespace fast
}  // namespace btg
