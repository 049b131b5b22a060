// Multi-RHS Fourier-space step on the 5th-generation tensor cores (tcgen05).
//
// tcgen05 has no FP64 kind, so the FP64 complex product Y_f = F_f X_f (and
// the adjoint F_f^H D_f) is computed exactly-in-integers with the Ozaki
// splitting: every real number v of a block that shares the power-of-two scale
// 2^e (max |v| < 2^e) is written as
//
//     v = 2^e * sum_{s=1..S} q_s 2^{-7 s} + r,   q_s in [-64, 64] (int8),  |r| <= 2^{e-7S-1}
//
// (max |v| < 2^{e-1}; every digit is a round-to-nearest of a value in
// [-64, 64], taken with the 1.5*2^52 magic-number add, so slicing is pure
// full-rate FP64 adds/multiplies with no conversion instructions)
//
// and  sum_k a_k b_k = 2^{eA+eB} sum_{L} 2^{-7L} C_L,  C_L = sum_{s+t=L} sum_k qa_s qb_t
// where every C_L is an exact int32 sum computed by kind::i8 MMAs into its
// own TMEM accumulator (levels L = 2..S+1; pairs with s+t > S+1 are below the
// FP64 rounding of the result). With S = 7 the per-entry truncation is 2^-49
// of the block maximum; results agree with the FP64 reference to ~1e-14 on the
// parity tests.
//
// Layouts (int8, "core matrix" = 8 rows x 16 bytes, 128 B):
//   F-hat slices  Aq[f][ig][jg][s][c][8 i][16 j]   ig = i/8, jg = j/16, c = re/im plane
//   The same bytes are the K-major A operand of the forward (rows i, K = j) and
//   the MN-major A operand of the adjoint (rows j, K = i).
//   Block scales  mA[f][jb] (max |F| over all i and the 1024-column block jb)
//   Vector scales mB[f][r][kb] (max over a 1024-entry block of x-hat_f[r] / d-hat_f[r]);
//   for the forward they come from the R2C epilogue (per-group exponents,
//   k_exponents), else from k_scale_vec
//   Adjoint B tiles Bq[f][ks][tile]: d-hat_f sliced once per frequency (k_slice_vec)
//   and TMA-fed, since every row tile of f multiplies the same d-hat_f
// The complex product uses plane-separated K: K' = (c, k); the B operand rows
// n' = 2r+q carry (xr, xi) against the real plane and (-xi, xr) against the
// imaginary plane (adjoint: (dr, di) and (di, -dr)), so one real GEMM yields
// [Re Y, Im Y] interleaved.
//
// Kernel roles (192 threads, one CTA per SM, persistent over (f, row-tile)):
//   warp 0     TMA producer of the F-hat slice tiles (cp.async.bulk ring, 2-3 stages)
//   warp 1     TMEM owner + single-thread MMA issuer. B is stored slice after
//              slice with a uniform 8-row stride, so A slice s meets the B
//              slices t = 0..S-1-s in ONE descriptor window (N = NP (S-s), split
//              at 256) whose products land in the consecutive level accumulators
//              s + t: 20 MMAs per 32-wide K step at N = 64 (instead of 56 small ones).
//   warp 0 lane 1 (adjoint) TMA producer of the pre-sliced B tiles
//   warps 2-5  prefetch the FP64 vector block of step it+2 (cp.async into a
//              thread-private ring), slice step it into the B tile (shared
//              memory), and drain the TMEM level accumulators into FP64
//              registers at the end of every 1024-wide K chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "btg_kernels.cuh"
#include "btg_umma.cuh"

namespace btg {
namespace oz {

constexpr int kS = 7;                       // slices per operand
constexpr int kLevels = kS;                 // L = 2 .. S+1
constexpr int kCM = 128;                    // bytes per core matrix
constexpr int kPos = kS * 2 * kCM;          // bytes per core-matrix position (all slices, both planes)
constexpr int kChunk = 1024;                // K entries per int32 accumulation chunk / scale block
constexpr int kStepsPerChunk = kChunk / 32;
constexpr int kTileM = 128;
constexpr int kBStages = 2;                 // sliced-vector ring (B producers)
constexpr size_t kSmemMax = 232448;
constexpr int kThreads = 192;
constexpr int kAStage = 16 * 2 * kPos;      // forward: 16 ig x 2 jg; adjoint: 4 ig x 8 jg (same size)
constexpr int kBStageMax = 2 * 8 * kPos;    // 2 K-groups x up to 8 n'-groups
constexpr int kVAhead = 2;                  // vector prefetch distance (steps)
constexpr int kVSlots = kVAhead + 1;
// Per-step vector staging: (kg, rr, quad) items, 4 complex + 1 exponent each, per B-producer thread.
template <int NG>
__host__ __device__ constexpr int VItems() { return (64 * NG + 127) / 128; }
template <int NG>
__host__ __device__ constexpr int VSlotBytes() { return VItems<NG>() * 128 * (4 * 16 + 4); }
constexpr size_t kBarBytes = 16 * 8;
template <int NG>
__host__ __device__ constexpr size_t RingBytes(int a_stages) {
    return (size_t)a_stages * kAStage + (size_t)kBStages * 2 * (16 * NG / 8) * kPos;
}
// F-hat slice ring depth (TMA): 3 stages when they fit beside the vector
// prefetch ring, else 2 (the vector prefetch matters more: ncu shows the B
// producers stalled on vector loads without it).
template <int NG, bool BPRE>
__host__ __device__ constexpr size_t VRingBytes() {
    return BPRE ? 0 : (size_t)kVSlots * VSlotBytes<NG>();
}
template <int NG, bool BPRE>
__host__ __device__ constexpr int AStages() {
    return RingBytes<NG>(3) + VRingBytes<NG, BPRE>() + kBarBytes <= kSmemMax ? 3 : 2;
}
template <int NG, bool BPRE>
__host__ __device__ constexpr size_t GemmSmemBytes() {
    return RingBytes<NG>(AStages<NG, BPRE>()) + VRingBytes<NG, BPRE>() + kBarBytes;
}
// Pre-sliced B (the adjoint: every row tile of a frequency reuses the same
// d-hat_f, so it is sliced once per frequency instead of once per tile):
// Bq[f][ks][B tile] in exactly the shared-memory tile layout.
template <int NG>
__host__ __device__ constexpr size_t BTileBytes() {
    return (size_t)2 * (16 * NG / 8) * kPos;
}

// Block exponent e with max < 2^{e-1} (so every scaled entry lies in (-1/2, 1/2)).
__device__ __forceinline__ int scale_exp(uint64_t maxbits) {
    const double m = __longlong_as_double((long long)maxbits);
    if (!(m > 0.0)) return 0;
    int e;
    frexp(m, &e);  // m = f 2^e, f in [0.5, 1): m < 2^e
    return e + 1;
}

__device__ __forceinline__ double pow2(int e) {  // exact 2^e for normal range
    return __longlong_as_double((long long)(e + 1023) << 52);
}

constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: w + kMagic rounds w to an integer

// Next signed digit of u in [-1/2, 1/2]: q = rint(128 u) in [-64, 64], u <- 128 u - q (exact).
__device__ __forceinline__ int digit(double& u) {
    const double w = u * 128.0;
    const double t = w + kMagic;
    u = w - (t - kMagic);
    return __double2loint(t);
}

__device__ __forceinline__ void digits(double u, int (&q)[kS]) {
#pragma unroll
    for (int s = 0; s < kS; ++s) q[s] = digit(u);
}

// The same 7 balanced digits with two FP64 roundings and integer shifts (the
// vector slicing is on the critical path of the forward GEMM): H = rint(2^21 u)
// carries digits 1-3, L = rint(2^28 (2^21 u - H)) digits 4-7; every digit is a
// rounding shift, in [-64, 64], and the truncation is the same 2^-50.
__device__ __forceinline__ int lo_int(double t) { return __double2loint(t); }
__device__ __forceinline__ void digits_fast(double u, int (&q)[kS]) {
    const double w = u * 2097152.0;  // 2^21 u, |w| <= 2^20
    const double t = w + kMagic;
    int h = lo_int(t);
    int l = lo_int((w - (t - kMagic)) * 268435456.0 + kMagic);  // 2^28 remainder, |l| <= 2^27
    q[0] = (h + (1 << 13)) >> 14;
    h -= q[0] << 14;
    q[1] = (h + (1 << 6)) >> 7;
    q[2] = h - (q[1] << 7);
    q[3] = (l + (1 << 20)) >> 21;
    l -= q[3] << 21;
    q[4] = (l + (1 << 13)) >> 14;
    l -= q[4] << 14;
    q[5] = (l + (1 << 6)) >> 7;
    q[6] = l - (q[5] << 7);
}

// Exact int32 -> FP64 on the FP64 pipe (one DADD instead of an I2F.F64): the
// bit pattern 0x43300000:(x ^ 2^31) is 2^52 + 2^31 + x.
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
    return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
    return (uint32_t)(a & 0xFF) | ((uint32_t)(b & 0xFF) << 8) | ((uint32_t)(c & 0xFF) << 16) |
           ((uint32_t)(d & 0xFF) << 24);
}

// ---------------------------------------------------------------------------
// Operator quantisation (once per operator, lazily)
// ---------------------------------------------------------------------------
// mA[f][jb] = max over i < nd, j in block jb, re/im of |F[f][i][j]| (as FP64 bits)
__global__ void k_scale_op(const double2* __restrict__ F, unsigned long long* __restrict__ mA, int nf, int nd,
                           int nm, int nkb) {
    const int rows_per = 8;
    const long long items = (long long)nf * nkb * ((nd + rows_per - 1) / rows_per);
    __shared__ double red[8];
    for (long long it = blockIdx.x; it < items; it += gridDim.x) {
        const int ib = (int)(it % ((nd + rows_per - 1) / rows_per));
        const long long fj = it / ((nd + rows_per - 1) / rows_per);
        const int jb = (int)(fj % nkb);
        const int f = (int)(fj / nkb);
        double m = 0.0;
        const int j0 = jb * kChunk, j1 = min(nm, j0 + kChunk);
        for (int r = 0; r < rows_per; ++r) {
            const int i = ib * rows_per + r;
            if (i >= nd) break;
            const double2* row = F + ((size_t)f * nd + i) * nm;
            for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
                const double2 v = __ldg(row + j);
                m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
            }
        }
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
            atomicMax(mA + (size_t)f * nkb + jb, (unsigned long long)__double_as_longlong(m));
        }
        __syncthreads();
    }
}

// One warp per core-matrix position (f, ig, jg): lane = (row r = lane/4, quad = lane%4),
// 4 consecutive complex j per lane -> 14 words (7 slices x 2 planes) of 4 int8.
__global__ void k_slice_op(const double2* __restrict__ F, const unsigned long long* __restrict__ mA,
                           int8_t* __restrict__ Aq, int nf, int nd, int nm, int IG, int JG, int nkb) {
    const int lane = threadIdx.x & 31;
    const long long npos = (long long)nf * IG * JG;
    const int warps = (int)(blockDim.x >> 5);
    for (long long p = (long long)blockIdx.x * warps + (threadIdx.x >> 5); p < npos; p += (long long)gridDim.x * warps) {
        const int jg = (int)(p % JG);
        const long long fi = p / JG;
        const int ig = (int)(fi % IG);
        const int f = (int)(fi / IG);
        const int i = ig * 8 + (lane >> 2);
        const int jq = jg * 16 + (lane & 3) * 4;
        const int e = scale_exp(mA[(size_t)f * nkb + (jg * 16) / kChunk]);
        const double inv = pow2(-e);
        int qr[4][kS], qi[4][kS];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double2 v = make_double2(0.0, 0.0);
            if (i < nd && jq + u < nm) v = __ldg(F + ((size_t)f * nd + i) * nm + jq + u);
            digits(v.x * inv, qr[u]);
            digits(v.y * inv, qi[u]);
        }
        uint32_t* out = reinterpret_cast<uint32_t*>(Aq + (size_t)p * kPos) + (lane >> 2) * 4 + (lane & 3);
#pragma unroll
        for (int s = 0; s < kS; ++s) {
            out[(s * 2 + 0) * (kCM / 4)] = pack4(qr[0][s], qr[1][s], qr[2][s], qr[3][s]);
            out[(s * 2 + 1) * (kCM / 4)] = pack4(qi[0][s], qi[1][s], qi[2][s], qi[3][s]);
        }
    }
}

// eB[(f*nr + r)*nkb + kb] = block exponent of max |re|,|im| over V[f][r0+r][kb*1024 ...] (one warp per item)
__global__ void k_scale_vec(const double2* __restrict__ V, int* __restrict__ mB, int nf, int ldr,
                            int r0, int nr, int K, int nkb) {
    const int lane = threadIdx.x & 31;
    const long long items = (long long)nf * nr * nkb;
    const int warps = (int)(blockDim.x >> 5);
    for (long long it = (long long)blockIdx.x * warps + (threadIdx.x >> 5); it < items;
         it += (long long)gridDim.x * warps) {
        const int kb = (int)(it % nkb);
        const long long fr = it / nkb;
        const int r = (int)(fr % nr);
        const int f = (int)(fr / nr);
        const double2* v = V + ((size_t)f * ldr + r0 + r) * K;
        double m = 0.0;
        const int k1 = min(K, (kb + 1) * kChunk);
        for (int k = kb * kChunk + lane; k < k1; k += 32) {
            const double2 x = __ldg(v + k);
            m = fmax(m, fmax(fabs(x.x), fabs(x.y)));
        }
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) mB[it] = scale_exp((uint64_t)__double_as_longlong(m));
    }
}

// Digits of item (kg, rr, quad) of a 32-wide K step into a B tile
// [c][t][n-group][kg][8 rows][16 B]: 4 complex values x (S slices, 2 planes).
template <bool ADJ, int NGRP>
__device__ __forceinline__ void slice_item(uint8_t* bst, int kg, int rr, int quad, const double2 (&xv)[4],
                                           double inv) {
    int qr[4][kS], qi[4][kS];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        digits_fast(xv[u].x * inv, qr[u]);
        digits_fast(xv[u].y * inv, qi[u]);
    }
    uint8_t* cm = bst + (rr >> 2) * 256 + kg * 128 + ((2 * rr) & 7) * 16 + quad * 4;
#pragma unroll
    for (int s = 0; s < kS; ++s) {
        const int a0 = qr[0][s], a1 = qr[1][s], a2 = qr[2][s], a3 = qr[3][s];
        const int b0 = qi[0][s], b1 = qi[1][s], b2 = qi[2][s], b3 = qi[3][s];
        const uint32_t re = pack4(a0, a1, a2, a3), im = pack4(b0, b1, b2, b3);
        uint32_t* p0 = reinterpret_cast<uint32_t*>(cm + (0 * kS + s) * NGRP * 256);
        uint32_t* p1 = reinterpret_cast<uint32_t*>(cm + (1 * kS + s) * NGRP * 256);
        p0[0] = re;  // real plane row 2rr
        p0[4] = im;  // real plane row 2rr+1
        if (!ADJ) {  // imaginary plane: (-xi, xr)
            p1[0] = pack4(-b0, -b1, -b2, -b3);
            p1[4] = re;
        } else {  // imaginary plane: (di, -dr)
            p1[0] = im;
            p1[4] = pack4(-a0, -a1, -a2, -a3);
        }
    }
}

// Pre-slice V[f][r0 .. r0+nr)[0 .. K) into Bq[f][ks][tile], one thread per item.
template <bool ADJ, int NG>
__global__ void k_slice_vec(const double2* __restrict__ V, const int* __restrict__ mB, uint8_t* __restrict__ Bq,
                            int nf, int ldr, int r0, int nr, int K) {
    constexpr int NP = 16 * NG, NGRP = NP / 8, kTot = 64 * NG;
    const int nks = (K + 31) / 32, nkb = (K + kChunk - 1) / kChunk;
    const long long total = (long long)nf * nks * kTot;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int item = (int)(idx % kTot);
        const long long fk = idx / kTot;
        const int ks = (int)(fk % nks);
        const int f = (int)(fk / nks);
        const int quad = item & 3;
        const int rr = (item >> 2) % (NP / 2);
        const int kg = (item >> 2) / (NP / 2);
        const int k = ks * 32 + kg * 16 + quad * 4;
        const bool live = rr < nr;
        const double inv = live ? pow2(-mB[((size_t)f * nr + rr) * nkb + ks / kStepsPerChunk]) : 0.0;
        const double2* src = V + ((size_t)f * ldr + r0 + (live ? rr : 0)) * K;
        double2 xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = (live && k + u < K) ? __ldg(src + k + u) : make_double2(0.0, 0.0);
        slice_item<ADJ, NGRP>(Bq + ((size_t)f * nks + ks) * BTileBytes<NG>(), kg, rr, quad, xv, inv);
    }
}

// ---------------------------------------------------------------------------
// The GEMM
// ---------------------------------------------------------------------------
struct GemmArgs {
    const int8_t* Aq;
    const unsigned long long* mA;
    const double2* V;   // x-hat (forward) / d-hat (adjoint): [f][ldr][K]
    const int* mB;      // block exponents of V
    double2* Y;         // [f][ldr][rows]
    int nf, nd, nm;
    int ldr, r0, nr;    // rhs stride, first rhs of this pass, rhs in this pass (<= 8 NG)
    int IG, JG, nkbA;
    const uint8_t* Bq;  // pre-sliced B tiles (BPRE)
};

template <bool ADJ, int NG, bool BPRE>
__global__ void __launch_bounds__(kThreads, 1) k_oz_gemm(GemmArgs g) {
    constexpr int NP = 16 * NG;  // MMA N (columns n' = 2r+q)
    constexpr int NGRP = NP / 8;
    constexpr int kBStage = 2 * NGRP * kPos;
    constexpr uint32_t kTmemCols = kLevels * NP <= 128 ? 128 : kLevels * NP <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr bool kVRing = !BPRE;
    constexpr int kAStages = AStages<NG, BPRE>();
    static_assert(BTileBytes<NG>() == (size_t)kBStage, "B tile");
    uint8_t* As = smem;                                 // [kAStages][kAStage]
    uint8_t* Bs = smem + kAStages * kAStage;             // [kBStages][kBStage]
    uint8_t* Vs = Bs + kBStages * kBStage;               // [kVSlots][VSlotBytes] (kVRing)
    uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + GemmSmemBytes<NG, BPRE>() - kBarBytes);
    uint64_t* emptyA = fullA + kAStages;
    uint64_t* fullB = emptyA + kAStages;
    uint64_t* emptyB = fullB + kBStages;
    uint64_t* acc_full = emptyB + kBStages;
    uint64_t* acc_empty = acc_full + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = ADJ ? g.nm : g.nd;
    const int K = ADJ ? g.nd : g.nm;
    const int mtiles = (rows + kTileM - 1) / kTileM;
    const int nks = (K + 31) / 32;
    const int nkb = (K + kChunk - 1) / kChunk;
    const long long ntiles = (long long)g.nf * mtiles;

    if (warp == 1) umma::tmem_alloc<kTmemCols>(tslot);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAStages; ++s) {
            umma::mbar_init(fullA + s, 1);
            umma::mbar_init(emptyA + s, 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            umma::mbar_init(fullB + s, BPRE ? 1 : 128);
            umma::mbar_init(emptyB + s, 1);
        }
        umma::mbar_init(acc_full, 1);
        umma::mbar_init(acc_empty, 128);
        umma::mbar_fence_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        // ===== TMA producer: F-hat slice tiles =====
        if (lane == 0) {
            const uint64_t pol = umma::policy_evict_first();
            long long it = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int f = (int)(tile / mtiles), mt = (int)(tile % mtiles);
                for (int ks = 0; ks < nks; ++ks, ++it) {
                    const int st = (int)(it % kAStages);
                    if (it >= kAStages) umma::mbar_wait(emptyA + st, (uint32_t)(((it / kAStages) - 1) & 1));
                    uint8_t* dst = As + st * kAStage;
                    const int8_t* base = g.Aq + (size_t)f * g.IG * g.JG * kPos;
                    if (!ADJ) {
                        const int ig0 = mt * 16, ig1 = min(g.IG, ig0 + 16);
                        const int njg = min(2, g.JG - 2 * ks);
                        const uint32_t bytes = (uint32_t)(njg * kPos);
                        umma::mbar_expect_tx(fullA + st, bytes * (uint32_t)(ig1 - ig0));
                        for (int ig = ig0; ig < ig1; ++ig)
                            umma::bulk_load(dst + (ig - ig0) * 2 * kPos, base + ((size_t)ig * g.JG + 2 * ks) * kPos,
                                            bytes, fullA + st, pol);
                    } else {
                        const int ig0 = 4 * ks, ig1 = min(g.IG, ig0 + 4);
                        const int jg0 = mt * 8, njg = min(8, g.JG - jg0);
                        const uint32_t bytes = (uint32_t)(njg * kPos);
                        umma::mbar_expect_tx(fullA + st, bytes * (uint32_t)(ig1 - ig0));
                        for (int ig = ig0; ig < ig1; ++ig)
                            umma::bulk_load(dst + (ig - ig0) * 8 * kPos, base + ((size_t)ig * g.JG + jg0) * kPos,
                                            bytes, fullA + st, pol);
                    }
                }
            }
        }
        if constexpr (BPRE) {
            if (lane == 1) {
                // pre-sliced B tiles on their own thread, so a full B ring never
                // holds back the A prefetch
                const uint64_t pol_b = umma::policy_evict_last();  // reused by every row tile of f
                long long it = 0;
                for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                    const int f = (int)(tile / mtiles);
                    for (int ks = 0; ks < nks; ++ks, ++it) {
                        const int sb = (int)(it % kBStages);
                        if (it >= kBStages) umma::mbar_wait(emptyB + sb, (uint32_t)(((it / kBStages) - 1) & 1));
                        umma::mbar_expect_tx(fullB + sb, (uint32_t)kBStage);
                        umma::bulk_load(Bs + sb * kBStage, g.Bq + ((size_t)f * nks + ks) * kBStage,
                                        (uint32_t)kBStage, fullB + sb, pol_b);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: the whole warp runs the loop (warp-uniform
        // descriptors), one elected lane issues the MMAs and commits =====
        {
            constexpr int kPiece = 256 / NP;  // B slices per MMA (N <= 256)
            const bool leader = umma::elect_one();
            long long it = 0, chunks = 0;
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int ck = 0; ck < nkb; ++ck, ++chunks) {
                    if (chunks > 0) umma::mbar_wait(acc_empty, (uint32_t)((chunks - 1) & 1));
                    umma::fence_after_sync();
                    const int ks1 = min(nks, (ck + 1) * kStepsPerChunk);
                    for (int ks = ck * kStepsPerChunk; ks < ks1; ++ks, ++it) {
                        const int sa = (int)(it % kAStages), sb = (int)(it % kBStages);
                        umma::mbar_wait(fullA + sa, (uint32_t)((it / kAStages) & 1));
                        umma::mbar_wait(fullB + sb, (uint32_t)((it / kBStages) & 1));
                        umma::fence_after_sync();
                        const uint32_t a0 = umma::smem_u32(As + sa * kAStage);
                        const uint32_t b0 = umma::smem_u32(Bs + sb * kBStage);
                        const bool first_step = ks == ck * kStepsPerChunk;
                        if (leader) {
#pragma unroll
                            for (int c = 0; c < 2; ++c)
#pragma unroll
                                for (int s = 0; s < kS; ++s) {
                                    const uint64_t ad =
                                        ADJ ? umma::make_desc(a0 + (s * 2 + c) * kCM, 8 * kPos, kPos)
                                            : umma::make_desc(a0 + (s * 2 + c) * kCM, kPos, 2 * kPos);
                                    // A slice s against the B slices t = 0 .. S-1-s at once: the
                                    // B planes are stored slice after slice with a uniform 8-row
                                    // stride, so one descriptor spans several slices and the
                                    // products land in consecutive level accumulators (s + t).
#pragma unroll
                                    for (int t0 = 0; t0 < kS - s; t0 += kPiece) {
                                        const int ns = (kS - s - t0) < kPiece ? (kS - s - t0) : kPiece;
                                        const uint64_t bd =
                                            umma::make_desc(b0 + (c * kS + t0) * NGRP * 256, 128, 256);
                                        const uint32_t acc = (first_step && c == 0 && s == 0) ? 0u : 1u;
                                        umma::mma_s8(tmem + (uint32_t)((s + t0) * NP), ad, bd,
                                                     umma::idesc_s8(kTileM, ns * NP, ADJ, false), acc);
                                    }
                                }
                            umma::commit(emptyA + sa);
                            umma::commit(emptyB + sb);
                        }
                        __syncwarp();
                    }
                    if (leader) umma::commit(acc_full);
                    __syncwarp();
                }
            }
        }
    } else {
        // ===== B producers + epilogue (warps 2..5, 128 threads) =====
        const int et = threadIdx.x - 64;     // 0..127
        const int quarter = warp & 3;        // TMEM lane quarter this warp may access
        const int trow = quarter * 32 + lane;
        double acc[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) acc[q] = 0.0;

        constexpr int kTotItems = 2 * (NP / 2) * 4;              // (kg, rr, quad) items per K step
        constexpr int kItems = VItems<NG>();                      // per thread
        static_assert(kItems == (kTotItems + 127) / 128, "item count");
        // chunk bookkeeping for interleaving drains with production
        long long drained = 0;  // chunks drained so far (global count)
        long long tile_of_drain = blockIdx.x;
        int ck_of_drain = 0;
        auto drain = [&]() {
            const int f = (int)(tile_of_drain / mtiles), mt = (int)(tile_of_drain % mtiles);
            const int ck = ck_of_drain;
            // the block exponents are global loads: issue them before the wait
            const int ebA = ADJ ? scale_exp(g.mA[(size_t)f * g.nkbA + (mt * kTileM) / kChunk])
                                : scale_exp(g.mA[(size_t)f * g.nkbA + ck]);
            int ebB[NP / 2];
#pragma unroll
            for (int rr = 0; rr < NP / 2; ++rr)
                ebB[rr] = rr < g.nr ? g.mB[((size_t)f * g.nr + rr) * nkb + ck] : 0;
            umma::mbar_wait(acc_full, (uint32_t)(drained & 1));
            umma::fence_after_sync();
            // 8 columns at a time: all 7 level loads in flight before one wait
#pragma unroll
            for (int cg = 0; cg < NP / 8; ++cg) {
                uint32_t r[kLevels][8];
#pragma unroll
                for (int L = 0; L < kLevels; ++L)
                    umma::ld_32x32b_x8(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(L * NP + cg * 8), r[L]);
                umma::ld_wait();
                double v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = 0.0;
#pragma unroll
                for (int L = 0; L < kLevels; ++L) {
                    const double w = pow2(-7 * (L + 2));
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = fma(i32_to_f64(r[L][q]), w, v[q]);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int col = cg * 8 + q, rr = col >> 1;
                    if (rr < g.nr) acc[col] = fma(v[q], pow2(ebA + ebB[rr]), acc[col]);
                }
            }
            umma::fence_before_sync();
            umma::mbar_arrive(acc_empty);
            ++drained;
            if (++ck_of_drain == nkb) {
                // tile complete: store rows, reset
                const int row = mt * kTileM + trow;
                if (row < rows) {
#pragma unroll
                    for (int q = 0; q < NP; q += 2) {
                        const int rr = q >> 1;
                        if (rr < g.nr)
                            g.Y[((size_t)f * g.ldr + g.r0 + rr) * rows + row] = make_double2(acc[q], acc[q + 1]);
                    }
                }
#pragma unroll
                for (int q = 0; q < NP; ++q) acc[q] = 0.0;
                ck_of_drain = 0;
                tile_of_drain += gridDim.x;
            }
        };

        // With kVRing, the vector data of step `itp` is fetched kVAhead steps early
        // with per-thread cp.async into a ring of thread-private shared slots: each
        // thread later reads back exactly the 16-byte words it copied (no
        // cross-thread sync). Otherwise the loads go to registers right before the
        // ring-slot wait.
        auto item_pos = [&](int ii, int k0, int& rr, int& k, bool& live) {
            const int item = et + ii * 128;
            const int quad = item & 3;
            rr = (item >> 2) % (NP / 2);
            const int kg = (item >> 2) / (NP / 2);
            k = k0 + kg * 16 + quad * 4;
            live = rr < g.nr && item < kTotItems;
        };
        auto prefetch = [&](long long itp) {
            const long long tl = (long long)blockIdx.x + (itp / nks) * gridDim.x;
            if (tl < ntiles) {
                const int f = (int)(tl / mtiles), ks = (int)(itp % nks);
                const int ck = ks / kStepsPerChunk;
                uint8_t* slot = Vs + (int)(itp % kVSlots) * VSlotBytes<NG>();
#pragma unroll
                for (int ii = 0; ii < kItems; ++ii) {
                    int rr, k;
                    bool live;
                    item_pos(ii, ks * 32, rr, k, live);
                    if (!live) continue;
                    umma::cp_async4(slot + kItems * 4 * 16 * 128 + (ii * 128 + et) * 4,
                                    g.mB + ((size_t)f * g.nr + rr) * nkb + ck);
                    const double2* src = g.V + ((size_t)f * g.ldr + g.r0 + rr) * K + k;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (k + u < K) umma::cp_async16(slot + ((ii * 4 + u) * 128 + et) * 16, src + u);
                }
            }
            umma::cp_async_commit();  // one group per step, empty past the end
        };

        // Step `it` may only wait for the MMAs of step it-kBStages after every
        // chunk before that step's chunk has been drained (the MMA warp waits for it).
        long long it = 0, chunk_idx = 0;  // chunk_idx: global index of the tile's first chunk
        long long step_chunk[kBStages] = {};
        if constexpr (BPRE) {  // B arrives by TMA: these warps only drain
            for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) chunk_idx += nkb;
            while (drained < chunk_idx) drain();
        } else {
        if constexpr (kVRing) {
#pragma unroll
            for (int a = 0; a < kVAhead; ++a) prefetch(a);
        }
        for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int f = (int)(tile / mtiles);
            for (int ks = 0; ks < nks; ++ks, ++it) {
                const int sb = (int)(it % kBStages);
                if (it >= kBStages)
                    while (drained < step_chunk[sb]) drain();
                const int k0 = ks * 32;
                double2 xv[kItems][4];
                double inv[kItems];
                if constexpr (kVRing) {
                    prefetch(it + kVAhead);
                } else {
                    const int ck = ks / kStepsPerChunk;
#pragma unroll
                    for (int ii = 0; ii < kItems; ++ii) {
                        int rr, k;
                        bool live;
                        item_pos(ii, k0, rr, k, live);
                        inv[ii] = live ? pow2(-g.mB[((size_t)f * g.nr + rr) * nkb + ck]) : 0.0;
                        const double2* src = g.V + ((size_t)f * g.ldr + g.r0 + (live ? rr : 0)) * K;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            xv[ii][u] = (live && k + u < K) ? __ldg(src + k + u) : make_double2(0.0, 0.0);
                    }
                }
                if (it >= kBStages) umma::mbar_wait(emptyB + sb, (uint32_t)(((it / kBStages) - 1) & 1));
                step_chunk[sb] = chunk_idx + ks / kStepsPerChunk;
                if constexpr (kVRing) {
                    umma::cp_async_wait<kVAhead>();  // this step's group has landed
                    const uint8_t* slot = Vs + (int)(it % kVSlots) * VSlotBytes<NG>();
#pragma unroll
                    for (int ii = 0; ii < kItems; ++ii) {
                        int rr, k;
                        bool live;
                        item_pos(ii, k0, rr, k, live);
                        inv[ii] = live ? pow2(-*reinterpret_cast<const int*>(slot + kItems * 4 * 16 * 128 +
                                                                             (ii * 128 + et) * 4))
                                       : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            xv[ii][u] = (live && k + u < K) ? *reinterpret_cast<const double2*>(
                                                                  slot + ((ii * 4 + u) * 128 + et) * 16)
                                                            : make_double2(0.0, 0.0);
                    }
                }
                // slice V[f][r][k0 .. k0+32) into the B tile
                uint8_t* bst = Bs + sb * kBStage;
#pragma unroll
                for (int ii = 0; ii < kItems; ++ii) {
                    const int item = et + ii * 128;  // (kg, rr, quad), quad fastest
                    if (item >= kTotItems) break;
                    slice_item<ADJ, NGRP>(bst, (item >> 2) / (NP / 2), (item >> 2) % (NP / 2), item & 3, xv[ii],
                                          inv[ii]);
                }
                umma::fence_async_smem();
                umma::mbar_arrive(fullB + sb);
            }
            chunk_idx += nkb;
        }
        while (drained < chunk_idx) drain();
        }
    }

    umma::fence_before_sync();
    __syncthreads();
    if (warp == 1) umma::tmem_free<kTmemCols>(tmem);
}

template <bool ADJ, int NG>
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t stream) {
    constexpr bool BPRE = ADJ;  // the adjoint's B (d-hat slices) is shared by all row tiles of f
    constexpr size_t smem = GemmSmemBytes<NG, BPRE>();
    static_assert(smem <= 232448, "shared memory");
    auto kern = k_oz_gemm<ADJ, NG, BPRE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if constexpr (BPRE) {
        if (!a.Bq) return cudaErrorInvalidValue;
        k_slice_vec<ADJ, NG><<<sms * 8, 256, 0, stream>>>(a.V, a.mB, const_cast<uint8_t*>(a.Bq), a.nf, a.ldr,
                                                          a.r0, a.nr, ADJ ? a.nd : a.nm);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const int rows = ADJ ? a.nm : a.nd;
    const long long tiles = (long long)a.nf * ((rows + kTileM - 1) / kTileM);
    const int grid = (int)std::min<long long>(tiles, sms);
    kern<<<grid, kThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace oz

size_t oz_operator_bytes(int nf, int nd, int nm) {
    return (size_t)nf * ((nd + 7) / 8) * ((nm + 15) / 16) * oz::kPos;
}
size_t oz_operator_scales(int nf, int nm) { return (size_t)nf * ((nm + oz::kChunk - 1) / oz::kChunk); }
size_t oz_vector_scales(int nf, int nrhs, int kdim) {  // ints
    return (size_t)nf * nrhs * ((kdim + oz::kChunk - 1) / oz::kChunk);
}

cudaError_t oz_quantize_operator(const double2* F, int nf, int nd, int nm, int8_t* Aq, unsigned long long* mA,
                                 cudaStream_t stream) {
    const int nkb = (nm + oz::kChunk - 1) / oz::kChunk;
    cudaError_t e = cudaMemsetAsync(mA, 0, oz_operator_scales(nf, nm) * sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    oz::k_scale_op<<<sms * 8, 256, 0, stream>>>(F, mA, nf, nd, nm, nkb);
    const int IG = (nd + 7) / 8, JG = (nm + 15) / 16;
    oz::k_slice_op<<<sms * 8, 256, 0, stream>>>(F, mA, Aq, nf, nd, nm, IG, JG, nkb);
    return cudaGetLastError();
}

namespace oz {
// Block exponents from the R2C's per-group exponents (R2CBlockMax): the max over
// the channel groups of each 1024-channel block; thread per (f, r, kb), f fastest
// along the (coalesced) pexp rows. The R2C-fused alternative to k_scale_vec.
__global__ void k_exponents(const int16_t* __restrict__ pexp, int* __restrict__ mB, int nf, int nrhs, int nm,
                            int cpb) {
    const int nkb = (nm + kChunk - 1) / kChunk;
    const long long n = (long long)nf * nrhs * nkb;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i % nf);
        const long long rk = i / nf;
        const int kb = (int)(rk % nkb), r = (int)(rk / nkb);
        const long long g0 = ((long long)r * nm + (long long)kb * kChunk) / cpb;
        const long long g1 = ((long long)r * nm + min(nm, (kb + 1) * kChunk) + cpb - 1) / cpb;
        int e = -32768;
        for (long long g = g0; g < g1; ++g) e = max(e, (int)pexp[g * nf + f]);
        mB[((size_t)f * nrhs + r) * nkb + kb] = e == -32768 ? 0 : e;
    }
}
}  // namespace oz

size_t oz_presliced_bytes(int nf, int nd) {  // adjoint B tiles, up to 32 RHS per pass
    return (size_t)nf * ((nd + 31) / 32) * oz::BTileBytes<4>();
}

cudaError_t oz_apply(bool adjoint, const int8_t* Aq, const unsigned long long* mA, const double2* V, double2* Y,
                     int nf, int nd, int nm, int nrhs, int* mB, uint8_t* Bq, cudaStream_t stream,
                     const int16_t* vexp, int vexp_cpb) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int K = adjoint ? nd : nm;
    const int nkb = (K + oz::kChunk - 1) / oz::kChunk;
    oz::GemmArgs a{};
    a.Aq = Aq;
    a.mA = mA;
    a.V = V;
    a.mB = mB;
    a.Y = Y;
    a.nf = nf;
    a.nd = nd;
    a.nm = nm;
    a.ldr = nrhs;
    a.IG = (nd + 7) / 8;
    a.JG = (nm + 15) / 16;
    a.nkbA = (nm + oz::kChunk - 1) / oz::kChunk;
    a.Bq = Bq;
    for (int r0 = 0; r0 < nrhs; r0 += 32) {
        const int nr = std::min(32, nrhs - r0);
        a.r0 = r0;
        a.nr = nr;
        if (vexp && nrhs <= 32 && !adjoint)  // block exponents folded into the R2C (R2CBlockMax)
            oz::k_exponents<<<sms * 8, 256, 0, stream>>>(vexp, mB, nf, nrhs, nm, vexp_cpb);
        else
            oz::k_scale_vec<<<sms * 8, 256, 0, stream>>>(V, mB, nf, nrhs, r0, nr, K, nkb);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const int ng = (nr + 7) / 8;  // N' = 16 ng columns
        switch (ng * 2 + (adjoint ? 1 : 0)) {
            case 2: e = oz::launch_gemm<false, 1>(a, stream); break;
            case 3: e = oz::launch_gemm<true, 1>(a, stream); break;
            case 4: e = oz::launch_gemm<false, 2>(a, stream); break;
            case 5: e = oz::launch_gemm<true, 2>(a, stream); break;
            case 6: e = oz::launch_gemm<false, 3>(a, stream); break;
            case 7: e = oz::launch_gemm<true, 3>(a, stream); break;
            case 8: e = oz::launch_gemm<false, 4>(a, stream); break;
            default: e = oz::launch_gemm<true, 4>(a, stream); break;
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace btg
