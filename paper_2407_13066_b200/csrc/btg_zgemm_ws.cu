// Warp-specialised, persistent 3M ZGEMM for the multi-RHS Fourier-space step
// (north star K7m; block_operator.cpp:239-259 / 296-317 applied to R vectors):
//   forward  D_f (N_d x R) = F_f (N_d x N_m) M_f (N_m x R)
//   adjoint  G_f (N_m x R) = F_f^H (N_m x N_d) D_f (N_d x R)
// Same arithmetic as k_zgemm3m_fwd/adj (btg_zgemm.cu: three real DMMA products
// per complex product, K in a fixed order per output tile) with a different
// pipeline:
//  * one persistent CTA per SM walks a static tile list (tile = blockIdx.x +
//    i * gridDim.x), so the next tile's first K stages stream in while the
//    current tile finishes and stores — no per-CTA prologue / epilogue bubble;
//  * a PRODUCER warp moves every K stage into padded shared rows (conflict-free
//    fragment loads, the strides of btg_zgemm.cu): the adjoint with 1-D bulk
//    copies (TMA engine, cp.async.bulk + mbarrier complete_tx; one 2 KB copy
//    per F-hat row segment), the forward — whose row segments are 256 B — with
//    16-byte cp.async chunks completing onto the same kind of mbarrier;
//  * 16 MMA warps (16 x 16-complex warp tiles) wait only on the stage's FULL barrier and release it on its
//    EMPTY barrier: no CTA-wide barrier in the K loop, a KST-deep ring.
// Ragged edges: rows / columns beyond the matrix are copied short (their
// outputs are never stored); the K tail is zeroed in the fragments.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "btg_kernels.cuh"
#include "btg_umma.cuh"

namespace btg {
namespace {

#ifndef BTG_ZWS_WARPS
#define BTG_ZWS_WARPS 8
#endif
constexpr int kMmaWarps = BTG_ZWS_WARPS;            // MMA warps per CTA (8 or 16)
constexpr int kWsThreads = (kMmaWarps + 1) * 32;  // + producer warp
constexpr int kTM = 128;                         // output rows per tile (i fwd, j adj)
constexpr int kTR = 32;                          // complex right-hand sides per tile
constexpr int kKC = 16;                          // complex K per stage
constexpr int kMT = kMmaWarps == 16 ? 1 : 2;      // m16 tiles per MMA warp (x 2 n8 tiles of rhs)
constexpr int kWarpsM = kTM / (16 * kMT);         // MMA warps along the tile rows
static_assert(kMmaWarps == kWarpsM * 2, "warps = rows x 2 rhs halves of 16");

// forward stage: A [128 i][2*16 + 8 doubles], B [32 r][16 + 4 complex]
constexpr int kFA = 2 * kKC + 8;
constexpr int kBS = kKC + 4;
constexpr size_t kFwdA = (size_t)kTM * kFA * sizeof(double);
constexpr size_t kFwdStage = kFwdA + (size_t)kTR * kBS * sizeof(double2);
// adjoint stage: A [16 i][128 j + 2 complex], B [32 r][16 + 4 complex]
constexpr int kAA = kTM + 2;
constexpr size_t kAdjA = (size_t)kKC * kAA * sizeof(double2);
constexpr size_t kAdjStage = kAdjA + (size_t)kTR * kBS * sizeof(double2);

constexpr int kFwdStages = 4;  // 4 x 51.2 KB
constexpr int kAdjStages = 5;  // 5 x 43.5 KB

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
        "{%0, %1, %2, %3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

// P1 = Ar Br, P2 = Ai Bi, P3 = (Ar +- Ai)(Br + Bi) for the warp's 2 x 2 m16n8 tiles
template <bool kAdj>
__device__ __forceinline__ void mma3(double (&p1)[kMT][2][4], double (&p2)[kMT][2][4], double (&p3)[kMT][2][4],
                                     const double2 (&a)[kMT][2], const double2 (&b)[2]) {
    double as[kMT][2];
#pragma unroll
    for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) as[mt][h] = kAdj ? a[mt][h].x - a[mt][h].y : a[mt][h].x + a[mt][h].y;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const double bs = b[nt].x + b[nt].y;
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt) {
            dmma(p1[mt][nt], a[mt][0].x, a[mt][1].x, b[nt].x);
            dmma(p2[mt][nt], a[mt][0].y, a[mt][1].y, b[nt].y);
            dmma(p3[mt][nt], as[mt][0], as[mt][1], bs);
        }
    }
}

__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(umma::smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
// arrive on `bar` once this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}

struct TileF {  // forward tile: frequency, first output row, first rhs
    int f, m0, r0;
};
__device__ __forceinline__ TileF fwd_tile(int t, int mt, int rt) {
    // rhs tiles innermost, then row tiles: CTAs running together share X_f / F_f rows in L2
    TileF d;
    d.r0 = (t % rt) * kTR;
    t /= rt;
    d.m0 = (t % mt) * kTM;
    d.f = t / mt;
    return d;
}

__global__ void __launch_bounds__(kWsThreads, 1)
    k_zgemm3m_fwd_ws(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nf,
                     int nd, int nm, int nrhs, int j0, int nj, bool accumulate) {
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + kFwdStages * kFwdStage);
    uint64_t* empty = full + kFwdStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mtiles = (nd + kTM - 1) / kTM, rtiles = (nrhs + kTR - 1) / kTR;
    const int ntiles = nf * mtiles * rtiles;
    const int nk = (nj + kKC - 1) / kKC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kFwdStages; ++s) {
            umma::mbar_init(full + s, 32);
            umma::mbar_init(empty + s, kMmaWarps);
        }
        umma::mbar_fence_init();
    }
    __syncthreads();

    if (warp == kMmaWarps) {
        // ---------------- producer ----------------
        // 16-byte cp.async chunks (a warp instruction = 2 rows x 256 B): the
        // forward's rows are only 256 B per stage, too short for one bulk copy
        // each (measured: 160 bulk copies per stage starve the MMA warps, 2.6x
        // slower). Each lane's copies complete onto FULL (count 32, .noinc);
        // chunks past the matrix are zero-filled.
        // lane -> (row half, complex column) of every 2-row chunk group; the
        // per-stage source advances by kc only
        const int lr = lane / kKC, lc = lane % kKC;
        uint32_t it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const TileF d = fwd_tile(t, mtiles, rtiles);
            const double2* Fa = F + ((size_t)d.f * nd + d.m0 + lr) * nm + j0 + lc;
            const double2* Xa = X + ((size_t)d.f * nrhs + d.r0 + lr) * nm + j0 + lc;
            const bool full_rows = d.m0 + kTM <= nd && d.r0 + kTR <= nrhs;
            for (int kt = 0; kt < nk; ++kt, ++it) {
                const int s = it % kFwdStages;
                umma::mbar_wait(empty + s, ((it / kFwdStages) & 1u) ^ 1u);
                const int kc = kt * kKC;
                unsigned char* st = smraw + (size_t)s * kFwdStage;
                double* As = reinterpret_cast<double*>(st) + lr * kFA + 2 * lc;
                double2* Bs = reinterpret_cast<double2*>(st + kFwdA) + lr * kBS + lc;
                if (full_rows && kc + kKC <= nj) {
                    const double2* fa = Fa + kc;
                    const double2* xa = Xa + kc;
#pragma unroll
                    for (int q = 0; q < kTM / 2; ++q) cp_async16z(As + 2 * q * kFA, fa + (size_t)2 * q * nm, true);
#pragma unroll
                    for (int q = 0; q < kTR / 2; ++q) cp_async16z(Bs + 2 * q * kBS, xa + (size_t)2 * q * nm, true);
                } else {
                    const bool kok = kc + lc < nj;
#pragma unroll 4
                    for (int q = 0; q < kTM / 2; ++q) {
                        const bool ok = kok && d.m0 + lr + 2 * q < nd;
                        cp_async16z(As + 2 * q * kFA, ok ? Fa + kc + (size_t)2 * q * nm : F, ok);
                    }
#pragma unroll 4
                    for (int q = 0; q < kTR / 2; ++q) {
                        const bool ok = kok && d.r0 + lr + 2 * q < nrhs;
                        cp_async16z(Bs + 2 * q * kBS, ok ? Xa + kc + (size_t)2 * q * nm : X, ok);
                    }
                }
                cp_async_arrive(full + s);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ---------------- MMA warps ----------------
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileF d = fwd_tile(t, mtiles, rtiles);
        double p1[kMT][2][4], p2[kMT][2][4], p3[kMT][2][4];
#pragma unroll
        for (int a = 0; a < kMT; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;
        for (int kt = 0; kt < nk; ++kt, ++it) {
            const int s = it % kFwdStages;
            umma::mbar_wait(full + s, (it / kFwdStages) & 1u);
            const unsigned char* st = smraw + (size_t)s * kFwdStage;
            const double* As = reinterpret_cast<const double*>(st);
            const double2* Bs = reinterpret_cast<const double2*>(st + kFwdA);
            const int kw = min(kKC, nj - kt * kKC);
#pragma unroll
            for (int ks = 0; ks < kKC / 4; ++ks) {
                const int kk = ks * 4 + tig;
                double2 a[kMT][2], b[2];
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        a[mt][h] = *reinterpret_cast<const double2*>(As + (wm * (16 * kMT) + mt * 16 + h * 8 + g) * kFA +
                                                                     2 * kk);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[(wn * 16 + nt * 8 + g) * kBS + kk];
                if (kw < kKC && kk >= kw) {  // K tail: the stage holds stale data past kw
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) a[mt][0] = a[mt][1] = make_double2(0.0, 0.0);
                    b[0] = b[1] = make_double2(0.0, 0.0);
                }
                mma3<false>(p1, p2, p3, a, b);
            }
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(empty + s);
        }
        // epilogue: lane holds C[g (+8)][2 tig + q] of each m16n8 tile
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int r = d.r0 + wn * 16 + nt * 8 + 2 * tig + q;
                    if (r >= nrhs) continue;
                    double2* yr = Y + ((size_t)d.f * nrhs + r) * nd;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int row = d.m0 + wm * (16 * kMT) + mt * 16 + h * 8 + g;
                        const int c = 2 * h + q;
                        if (row < nd) {
                            double2 v = make_double2(p1[mt][nt][c] - p2[mt][nt][c],
                                                     p3[mt][nt][c] - p1[mt][nt][c] - p2[mt][nt][c]);
                            if (accumulate) {
                                const double2 o = yr[row];
                                v.x += o.x;
                                v.y += o.y;
                            }
                            yr[row] = v;
                        }
                    }
                }
    }
}

// ---------------------------------------------------------------------------
// Forward with TMA tensor copies: per stage FOUR cp.async.bulk.tensor.3d (the
// two 8-complex K halves of the 128-row F-hat tile and of the 32-row X tile),
// 128-byte swizzled rows (16-byte chunk c of row r at c ^ (r & 7)). The MMA
// warps map lane quad tig of K step ks to complex k = 8 (ks / 2) + 2 tig +
// (ks & 1), so the 2 rows x 4 chunks of every quarter-warp fragment load land
// in 8 distinct bank groups. Rows / right-hand sides past the matrix and
// columns past N_m are zero-filled by the TMA unit; a column range's K tail is
// masked in the fragments.
// ---------------------------------------------------------------------------
constexpr int kTmaStages = 5;
constexpr bool kXBlockSwizzle = kSpecBlock == 8;  // blocked X tile swizzled (128-byte inner box)
static_assert(kSpecBlock == 4 || kSpecBlock == 8, "one or two spectral blocks per 8-complex K half");
constexpr uint32_t kTmaA = kTM * 256;  // 2 halves x 128 rows x 128 B
constexpr uint32_t kTmaB = kTR * 256;
constexpr uint32_t kTmaStage = kTmaA + kTmaB;  // 40 KB, 1024-byte aligned

__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, int x, int y, int z,
                                          uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(umma::smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tma_load4(uint32_t dst, const CUtensorMap* map, int x, int y, int z, int w,
                                          uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(w), "r"(umma::smem_u32(bar)), "l"(policy)
        : "memory");
}

__global__ void __launch_bounds__(kWsThreads, 1)
    k_zgemm3m_fwd_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      double2* __restrict__ Y, int nf, int nd, int nm, int nrhs, int j0, int nj, bool accumulate,
                      bool xblocked) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    const uint32_t base_u = (umma::smem_u32(smraw) + 1023u) & ~1023u;
    unsigned char* base = smraw + (base_u - umma::smem_u32(smraw));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kTmaStages * kTmaStage);
    uint64_t* empty = full + kTmaStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mtiles = (nd + kTM - 1) / kTM, rtiles = (nrhs + kTR - 1) / kTR;
    const int ntiles = nf * mtiles * rtiles;
    const int nk = (nj + kKC - 1) / kKC;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kTmaStages; ++st) {
            umma::mbar_init(full + st, 1);
            umma::mbar_init(empty + st, kMmaWarps);
        }
        umma::mbar_fence_init();
    }
    __syncthreads();

    if (warp == kMmaWarps) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            const uint64_t pol_a = umma::policy_evict_first();
            const uint64_t pol_b = umma::policy_evict_last();
            uint32_t it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const TileF d = fwd_tile(t, mtiles, rtiles);
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int st = it % kTmaStages;
                    umma::mbar_wait(empty + st, ((it / kTmaStages) & 1u) ^ 1u);
                    umma::mbar_expect_tx(full + st, kTmaStage);
                    const uint32_t sa = base_u + st * kTmaStage;
                    const int x = 2 * (j0 + kt * kKC);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        tma_load3(sa + h * (kTmaA / 2), &tmA, x + 16 * h, d.m0, d.f, full + st, pol_a);
                        if (xblocked)  // X channel-blocked: (G complex, f, j / G, r), 8 / G j blocks per half
                            tma_load4(sa + kTmaA + h * (kTmaB / 2), &tmB, 0, d.f,
                                      (j0 + kt * kKC) / kSpecBlock + (8 / kSpecBlock) * h, d.r0, full + st, pol_b);
                        else
                            tma_load3(sa + kTmaA + h * (kTmaB / 2), &tmB, x + 16 * h, d.r0, d.f, full + st, pol_b);
                    }
                }
            }
        }
        return;
    }

    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileF d = fwd_tile(t, mtiles, rtiles);
        double p1[kMT][2][4], p2[kMT][2][4], p3[kMT][2][4];
#pragma unroll
        for (int a = 0; a < kMT; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;
        for (int kt = 0; kt < nk; ++kt, ++it) {
            const int st = it % kTmaStages;
            umma::mbar_wait(full + st, (it / kTmaStages) & 1u);
            const unsigned char* sa = base + st * kTmaStage;
            const int kw = min(kKC, nj - kt * kKC);
            // (one K step of fragments at a time: with 9 warps the register cap is
            // 168 per thread — 3 warps share an SMSP's 16K registers — and the
            // double-buffered variant spilled, 12.4 -> 12.8 ms)
#pragma unroll
            for (int ks = 0; ks < kKC / 4; ++ks) {
                const int half = ks >> 1, c = 2 * tig + (ks & 1);
                const int kk = 8 * half + c;
                const int sw = (c ^ g) << 4;  // every fragment row here is = g (mod 8)
                const unsigned char* Ah = sa + half * (kTmaA / 2) + sw;
                // blocked X arrives unswizzled (a 64-byte inner box cannot take the
                // 128-byte swizzle): 2-way conflicts on the two B loads only
                const unsigned char* Bh = sa + kTmaA + half * (kTmaB / 2) + (xblocked && !kXBlockSwizzle ? c << 4 : sw);
                double2 a[kMT][2], b[2];
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        a[mt][h] = *reinterpret_cast<const double2*>(Ah + (wm * (16 * kMT) + mt * 16 + h * 8 + g) * 128);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
                    b[nt] = *reinterpret_cast<const double2*>(Bh + (wn * 16 + nt * 8 + g) * 128);
                if (kw < kKC && kk >= kw) {
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) a[mt][0] = a[mt][1] = make_double2(0.0, 0.0);
                    b[0] = b[1] = make_double2(0.0, 0.0);
                }
                mma3<false>(p1, p2, p3, a, b);
            }
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(empty + st);
        }
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int r = d.r0 + wn * 16 + nt * 8 + 2 * tig + q;
                    if (r >= nrhs) continue;
                    double2* yr = Y + ((size_t)d.f * nrhs + r) * nd;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int row = d.m0 + wm * (16 * kMT) + mt * 16 + h * 8 + g;
                        const int cc = 2 * h + q;
                        if (row < nd) {
                            double2 v = make_double2(p1[mt][nt][cc] - p2[mt][nt][cc],
                                                     p3[mt][nt][cc] - p1[mt][nt][cc] - p2[mt][nt][cc]);
                            if (accumulate) {
                                const double2 o = yr[row];
                                v.x += o.x;
                                v.y += o.y;
                            }
                            yr[row] = v;
                        }
                    }
                }
    }
}

struct TileA {  // adjoint tile: frequency, first output column j, first rhs
    int f, j0, r0;
};
// (f, j tile, r tile) of tile t = blockIdx.x + i gridDim.x, rhs tiles fastest:
// one division at the start, then carries (the stride's own decomposition is
// smaller than each radix, so each digit wraps at most once per step)
struct TileWalk {
    int r, j, f, sr, sj, sf, jt, rt;
    __device__ TileWalk(int t, int stride, int jt_, int rt_) : jt(jt_), rt(rt_) {
        r = t % rt;
        t /= rt;
        j = t % jt;
        f = t / jt;
        sr = stride % rt;
        stride /= rt;
        sj = stride % jt;
        sf = stride / jt;
    }
    __device__ __forceinline__ void next() {
        r += sr;
        int c = 0;
        if (r >= rt) {
            r -= rt;
            c = 1;
        }
        j += sj + c;
        c = 0;
        if (j >= jt) {
            j -= jt;
            c = 1;
        }
        f += sf + c;
    }
};

__device__ __forceinline__ TileA adj_tile(int t, int jt, int rt, int jbase) {
    TileA d;
    d.r0 = (t % rt) * kTR;
    t /= rt;
    d.j0 = jbase + (t % jt) * kTM;
    d.f = t / jt;
    return d;
}

__global__ void __launch_bounds__(kWsThreads, 1)
    k_zgemm3m_adj_ws(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nf,
                     int nd, int nm, int nrhs, int jbase, int jend) {
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + kAdjStages * kAdjStage);
    uint64_t* empty = full + kAdjStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jtiles = (jend - jbase + kTM - 1) / kTM, rtiles = (nrhs + kTR - 1) / kTR;
    const int ntiles = nf * jtiles * rtiles;
    const int nk = (nd + kKC - 1) / kKC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAdjStages; ++s) {
            umma::mbar_init(full + s, 1);
            umma::mbar_init(empty + s, kMmaWarps);
        }
        umma::mbar_fence_init();
    }
    __syncthreads();

    if (warp == kMmaWarps) {
        const uint64_t pol_a = umma::policy_evict_first();
        const uint64_t pol_b = umma::policy_evict_last();  // D_f: shared by the N_m / 128 column tiles
        uint32_t it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const TileA d = adj_tile(t, jtiles, rtiles, jbase);
            const double2* Ff = F + (size_t)d.f * nd * nm + d.j0;
            const double2* Xf = X + (size_t)d.f * nrhs * nd;
            const uint32_t ab = (uint32_t)min(kTM, jend - d.j0) * sizeof(double2);
            const int brows = min(kTR, nrhs - d.r0);
            for (int kt = 0; kt < nk; ++kt, ++it) {
                const int s = it % kAdjStages;
                umma::mbar_wait(empty + s, ((it / kAdjStages) & 1u) ^ 1u);
                const int kc = kt * kKC, kw = min(kKC, nd - kc);
                const uint32_t bb = (uint32_t)kw * sizeof(double2);
                unsigned char* st = smraw + (size_t)s * kAdjStage;
                if (lane == 0) umma::mbar_expect_tx(full + s, ab * (uint32_t)kw + bb * (uint32_t)brows);
                __syncwarp();
                if (lane < kw)
                    umma::bulk_load(st + (size_t)lane * kAA * sizeof(double2), Ff + (size_t)(kc + lane) * nm, ab,
                                    full + s, pol_a);
                if (lane < brows)
                    umma::bulk_load(st + kAdjA + (size_t)lane * kBS * sizeof(double2),
                                    Xf + (size_t)(d.r0 + lane) * nd + kc, bb, full + s, pol_b);
            }
        }
        return;
    }

    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;
    uint32_t it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileA d = adj_tile(t, jtiles, rtiles, jbase);
        double p1[kMT][2][4], p2[kMT][2][4], p3[kMT][2][4];
#pragma unroll
        for (int a = 0; a < kMT; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;
        for (int kt = 0; kt < nk; ++kt, ++it) {
            const int s = it % kAdjStages;
            umma::mbar_wait(full + s, (it / kAdjStages) & 1u);
            const unsigned char* st = smraw + (size_t)s * kAdjStage;
            const double2* As = reinterpret_cast<const double2*>(st);
            const double2* Bs = reinterpret_cast<const double2*>(st + kAdjA);
            const int kw = min(kKC, nd - kt * kKC);
#pragma unroll
            for (int ks = 0; ks < kKC / 4; ++ks) {
                const int kk = ks * 4 + tig;
                double2 a[kMT][2], b[2];
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) a[mt][h] = As[kk * kAA + wm * (16 * kMT) + mt * 16 + h * 8 + g];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[(wn * 16 + nt * 8 + g) * kBS + kk];
                if (kw < kKC && kk >= kw) {
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) a[mt][0] = a[mt][1] = make_double2(0.0, 0.0);
                    b[0] = b[1] = make_double2(0.0, 0.0);
                }
                mma3<true>(p1, p2, p3, a, b);
            }
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(empty + s);
        }
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int r = d.r0 + wn * 16 + nt * 8 + 2 * tig + q;
                    if (r >= nrhs) continue;
                    double2* yr = Y + ((size_t)d.f * nrhs + r) * nm;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int jj = d.j0 + wm * (16 * kMT) + mt * 16 + h * 8 + g;
                        const int c = 2 * h + q;
                        if (jj < jend)
                            yr[jj] = make_double2(p1[mt][nt][c] + p2[mt][nt][c],
                                                  p3[mt][nt][c] - p1[mt][nt][c] + p2[mt][nt][c]);
                    }
                }
    }
}

// Adjoint with TMA tensor copies: per stage 16 boxes of 16 F-hat rows (i) x 8
// complex columns (j) — each its own 2 KB swizzled block, chunk (j % 8) ^ (i & 7)
// — and the two K halves of the 32-row D_f tile. Lane quad tig of K step ks
// takes i = 8 (ks / 2) + 2 tig + (ks & 1) (conflict-free, as the forward).
// Everything past N_d / N_m / nrhs is zero-filled by the TMA unit.
__global__ void __launch_bounds__(kWsThreads, 1)
    k_zgemm3m_adj_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      double2* __restrict__ Y, int nf, int nd, int nm, int nrhs, int jbase, int jend,
                      bool yblocked, bool chunked) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    const uint32_t base_u = (umma::smem_u32(smraw) + 1023u) & ~1023u;
    unsigned char* base = smraw + (base_u - umma::smem_u32(smraw));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + kTmaStages * kTmaStage);
    uint64_t* empty = full + kTmaStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jtiles = (jend - jbase + kTM - 1) / kTM, rtiles = (nrhs + kTR - 1) / kTR;
    const int ntiles = nf * jtiles * rtiles;
    const int nk = (nd + kKC - 1) / kKC;
    if (threadIdx.x == 0) {
        for (int st = 0; st < kTmaStages; ++st) {
            umma::mbar_init(full + st, 1);
            umma::mbar_init(empty + st, kMmaWarps);
        }
        umma::mbar_fence_init();
    }
    __syncthreads();

    if (warp == kMmaWarps) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            const uint64_t pol_a = umma::policy_evict_first();
            const uint64_t pol_b = umma::policy_evict_last();  // D_f: shared by the column tiles
            uint32_t it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const TileA d = adj_tile(t, jtiles, rtiles, jbase);
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int st = it % kTmaStages;
                    umma::mbar_wait(empty + st, ((it / kTmaStages) & 1u) ^ 1u);
                    umma::mbar_expect_tx(full + st, kTmaStage);
                    const uint32_t sa = base_u + st * kTmaStage;
                    const int kc = kt * kKC;
                    if (chunked) {
                        // one box each: A = 16 chunks of 8 complex x 16 rows, B = 2 chunks x 32 rows
                        tma_load4(sa, &tmA, 0, kc, d.j0 / 8, d.f, full + st, pol_a);
                        tma_load4(sa + kTmaA, &tmB, 0, d.r0, kc / 8, d.f, full + st, pol_b);
                        continue;
                    }
#pragma unroll
                    for (int b = 0; b < kTM / 8; ++b)
                        tma_load3(sa + b * 2048, &tmA, 2 * (d.j0 + 8 * b), kc, d.f, full + st, pol_a);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_load3(sa + kTmaA + h * (kTmaB / 2), &tmB, 2 * kc + 16 * h, d.r0, d.f, full + st, pol_b);
                }
            }
        }
        return;
    }

    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp % kWarpsM, wn = warp / kWarpsM;
    uint32_t it = 0;
    // tiles walked incrementally (no integer division per tile: the epilogue and
    // tile setup were ~9 % of the MMA warps' samples)
    TileWalk tw(blockIdx.x, gridDim.x, jtiles, rtiles);
    const size_t rstride = yblocked ? (size_t)nm * nf : (size_t)nm;  // Y offset per right-hand side
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, tw.next()) {
        TileA d;
        d.r0 = tw.r * kTR;
        d.j0 = jbase + tw.j * kTM;
        d.f = tw.f;
        double p1[kMT][2][4], p2[kMT][2][4], p3[kMT][2][4];
#pragma unroll
        for (int a = 0; a < kMT; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;
        for (int kt = 0; kt < nk; ++kt, ++it) {
            const int st = it % kTmaStages;
            umma::mbar_wait(full + st, (it / kTmaStages) & 1u);
            const unsigned char* sa = base + st * kTmaStage;
            auto load = [&](int ks, double2 (&a)[kMT][2], double2 (&b)[2]) {
                const int half = ks >> 1, c = 2 * tig + (ks & 1);
                const int i = 8 * half + c;  // K row of this lane (i & 7 == c)
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int jb = (wm * (16 * kMT) + mt * 16 + h * 8) / 8;  // j block; j % 8 == g
                        a[mt][h] = *reinterpret_cast<const double2*>(sa + jb * 2048 + i * 128 + ((g ^ c) << 4));
                    }
                const unsigned char* Bh = sa + kTmaA + half * (kTmaB / 2) + ((c ^ g) << 4);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
                    b[nt] = *reinterpret_cast<const double2*>(Bh + (wn * 16 + nt * 8 + g) * 128);
            };
            double2 a0[kMT][2], b0[2], a1[kMT][2], b1[2];
            load(0, a0, b0);
            load(1, a1, b1);
            mma3<true>(p1, p2, p3, a0, b0);
            load(2, a0, b0);
            mma3<true>(p1, p2, p3, a1, b1);
            load(3, a1, b1);
            mma3<true>(p1, p2, p3, a0, b0);
            mma3<true>(p1, p2, p3, a1, b1);
            __syncwarp();
            if (lane == 0) umma::mbar_arrive(empty + st);
        }
        // per-lane output offsets: Y[f][r][j] (or channel-blocked [c/4][f][c%4],
        // c = r N_m + j, N_m and j0 multiples of 4): base + r * rstride + col(j)
        const size_t ftile = yblocked ? (size_t)kSpecBlock * d.f : (size_t)d.f * nrhs * nm;
        if (d.r0 + kTR <= nrhs && d.j0 + kTM <= jend) {
            // full tile: one base address per lane, every store at a constant
            // offset from it — (mt, h) steps 8 columns (two spectral blocks when
            // blocked), (nt, q) steps right-hand sides; no per-store index math
            // or bounds branches (they were ~400 instructions per tile per lane)
            const int jj0 = d.j0 + wm * (16 * kMT) + g;
            const size_t col0 = yblocked ? (size_t)(jj0 / kSpecBlock) * kSpecBlock * nf + (jj0 % kSpecBlock)
                                         : (size_t)jj0;
            const size_t j8 = yblocked ? (size_t)(8 / kSpecBlock) * kSpecBlock * nf : (size_t)8;
            double2* yb = Y + ftile + col0 + (size_t)(d.r0 + wn * 16 + 2 * tig) * rstride;
#pragma unroll
            for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double2* yc = yb + (size_t)(2 * mt + h) * j8;
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int cc = 2 * h + q;
                            yc[(size_t)(8 * nt + q) * rstride] =
                                make_double2(p1[mt][nt][cc] + p2[mt][nt][cc], p3[mt][nt][cc] - p1[mt][nt][cc] + p2[mt][nt][cc]);
                        }
                }
            continue;
        }
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jj = d.j0 + wm * (16 * kMT) + mt * 16 + h * 8 + g;
                if (jj >= jend) continue;
                const size_t col = yblocked ? (size_t)(jj / kSpecBlock) * kSpecBlock * nf + (jj % kSpecBlock)
                                            : (size_t)jj;
                double2* yc = Y + ftile + col;
                const int cc0 = 2 * h;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int r = d.r0 + wn * 16 + nt * 8 + 2 * tig + q;
                        if (r >= nrhs) continue;
                        const int cc = cc0 + q;
                        yc[(size_t)r * rstride] = make_double2(p1[mt][nt][cc] + p2[mt][nt][cc],
                                                               p3[mt][nt][cc] - p1[mt][nt][cc] + p2[mt][nt][cc]);
                    }
            }
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

// [planes][rows][2 * cols] doubles, box 16 doubles x box_rows x 1, 128-byte swizzle
bool encode_rows(CUtensorMap* m, const void* ptr, int cols, int rows, int planes, int box_rows) {
    const EncodeTiled fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)2 * cols, (cuuint64_t)rows, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)cols * 16, (cuuint64_t)cols * 16 * rows};
    const cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [planes][rows][cols complex] as (16 doubles, rows, cols / 8 chunks, planes): ONE
// box of box_rows rows x box_chunks 8-complex chunks lands chunk-major,
// [chunk][row][128 B], 128-byte swizzled — the layout of box_chunks separate
// encode_rows boxes side by side (the adjoint's A stage in one copy, not 16)
bool encode_chunks(CUtensorMap* m, const void* ptr, int cols, int rows, int planes, int box_rows,
                   int box_chunks) {
    const EncodeTiled fn = encode_fn();
    if (!fn || cols % 8) return false;
    const cuuint64_t dims[4] = {16, (cuuint64_t)rows, (cuuint64_t)cols / 8, (cuuint64_t)planes};
    const cuuint64_t strides[3] = {(cuuint64_t)cols * 16, 128, (cuuint64_t)cols * 16 * rows};
    const cuuint32_t box[4] = {16, (cuuint32_t)box_rows, (cuuint32_t)box_chunks, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// X channel-blocked ([r nm + j] / 4, f, (r nm + j) % 4): dims (8 doubles, nf, nm / 4, nrhs), box (8, 1, 2, 32)
bool encode_blocked(CUtensorMap* m, const void* ptr, int nm, int nrhs, int nf) {
    const EncodeTiled fn = encode_fn();
    if (!fn || nm % kSpecBlock) return false;
    const cuuint64_t blk = (cuuint64_t)kSpecBlock * 16;  // bytes per (block, f)
    const cuuint64_t dims[4] = {(cuuint64_t)2 * kSpecBlock, (cuuint64_t)nf, (cuuint64_t)nm / kSpecBlock,
                                (cuuint64_t)nrhs};
    const cuuint64_t strides[3] = {blk, blk * nf, blk * nf * (nm / kSpecBlock)};
    const cuuint32_t box[4] = {2 * kSpecBlock, 1, 8 / kSpecBlock, (cuuint32_t)kTR};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    // 8-channel blocks: 128-byte inner box, swizzled like the frequency-major tile.
    // (4-channel blocks take no swizzle: with a 64-byte inner box the 128-byte
    // swizzle pads every row to 128 bytes — measured: the box overran its slot.)
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(ptr), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, kXBlockSwizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace

// Host launchers (declared in btg_kernels.cuh): one persistent CTA per SM.
bool zgemm_tma_ok(int nm) { return encode_fn() != nullptr && nm % kSpecBlock == 0; }

cudaError_t launch_zgemm3m_fwd_ws(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                                  int j0, int nj, bool accumulate, cudaStream_t stream, bool xblocked) {
    const char* cp = std::getenv("BTG_ZGEMM_FWD_CPASYNC");  // A/B: the cp.async producer
    CUtensorMap ta, tb;
    if (xblocked && (j0 % kSpecBlock || !zgemm_tma_ok(nm))) return cudaErrorNotSupported;
    if (xblocked || (!(cp && *cp && *cp != '0') && encode_rows(&tb, X, nm, nrhs, nf, kTR))) {
        if (!encode_rows(&ta, F, nm, nd, nf, kTM)) return cudaErrorNotSupported;
        if (xblocked && !encode_blocked(&tb, X, nm, nrhs, nf)) return cudaErrorNotSupported;
        const size_t smem = kTmaStages * kTmaStage + 1024 + 2 * kTmaStages * sizeof(uint64_t);
        cudaError_t e =
            cudaFuncSetAttribute(k_zgemm3m_fwd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const long long tiles = (long long)nf * ((nd + kTM - 1) / kTM) * ((nrhs + kTR - 1) / kTR);
        const int grid = (int)std::min<long long>(tiles, sm_count());
        k_zgemm3m_fwd_tma<<<grid, kWsThreads, smem, stream>>>(ta, tb, Y, nf, nd, nm, nrhs, j0, nj, accumulate,
                                                              xblocked);
        return cudaGetLastError();
    }
    const size_t smem = kFwdStages * kFwdStage + 2 * kFwdStages * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(k_zgemm3m_fwd_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (long long)nf * ((nd + kTM - 1) / kTM) * ((nrhs + kTR - 1) / kTR);
    const int grid = (int)std::min<long long>(tiles, sm_count());
    k_zgemm3m_fwd_ws<<<grid, kWsThreads, smem, stream>>>(F, X, Y, nf, nd, nm, nrhs, j0, nj, accumulate);
    return cudaGetLastError();
}

cudaError_t launch_zgemm3m_adj_ws(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                                  int j0, int nj, cudaStream_t stream, bool yblocked) {
    const char* bk = std::getenv("BTG_ZGEMM_ADJ_BULK");  // A/B: the 1-D bulk-copy producer
    CUtensorMap ta, tb;
    if (yblocked && (j0 % kSpecBlock || !zgemm_tma_ok(nm))) return cudaErrorNotSupported;
    // one TMA box per operand and stage when N_m, N_d and the column origin allow it
    const char* sb = std::getenv("BTG_ZGEMM_ADJ_BOXES");  // A/B: 16 + 2 boxes per stage
    const bool chunked = !(sb && *sb && *sb != '0') && nm % 8 == 0 && nd % 8 == 0 && j0 % 8 == 0 &&
                         encode_chunks(&ta, F, nm, nd, nf, kKC, kTM / 8) && encode_chunks(&tb, X, nd, nrhs, nf, kTR, 2);
    if ((yblocked || !(bk && *bk && *bk != '0')) &&
        (chunked || (encode_rows(&ta, F, nm, nd, nf, kKC) && encode_rows(&tb, X, nd, nrhs, nf, kTR)))) {
        const size_t smem = kTmaStages * kTmaStage + 1024 + 2 * kTmaStages * sizeof(uint64_t);
        cudaError_t e =
            cudaFuncSetAttribute(k_zgemm3m_adj_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const long long tiles = (long long)nf * ((nj + kTM - 1) / kTM) * ((nrhs + kTR - 1) / kTR);
        const int grid = (int)std::min<long long>(tiles, sm_count());
        k_zgemm3m_adj_tma<<<grid, kWsThreads, smem, stream>>>(ta, tb, Y, nf, nd, nm, nrhs, j0, j0 + nj, yblocked,
                                                              chunked);
        return cudaGetLastError();
    }
    const size_t smem = kAdjStages * kAdjStage + 2 * kAdjStages * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(k_zgemm3m_adj_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long tiles = (long long)nf * ((nj + kTM - 1) / kTM) * ((nrhs + kTR - 1) / kTR);
    const int grid = (int)std::min<long long>(tiles, sm_count());
    k_zgemm3m_adj_ws<<<grid, kWsThreads, smem, stream>>>(F, X, Y, nf, nd, nm, nrhs, j0, j0 + nj);
    return cudaGetLastError();
}

}  // namespace btg
