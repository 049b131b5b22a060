// Multi-right-hand-side Fourier-space step on the FP64 tensor cores (DMMA).
//
// With R right-hand sides the per-frequency product is a ZGEMM
// (block_operator.cpp:239-259 / 296-317 applied to R vectors at once):
//   forward  D_f (N_d x R) = F_f (N_d x N_m) M_f (N_m x R)
//   adjoint  G_f (N_m x R) = F_f^H (N_m x N_d) D_f (N_d x R)
// tcgen05 has no f64 kind on sm_100a, so FP64 tensor-core math is the warp-level
// mma.sync.m16n8k4.f64 (DMMA). Complex products use the real embedding that
// reads F-hat in its native interleaved (re, im) layout as a real matrix with
// K' = 2K:   A'[i][2k+s] = (re, im)_s of F[i][k]   and
//   forward  B'[2k][2r] = Br, B'[2k+1][2r] = -Bi, B'[2k][2r+1] = Bi, B'[2k+1][2r+1] = Br
//   adjoint  B'[2k][2r] = Br, B'[2k+1][2r] = +Bi, B'[2k][2r+1] = Bi, B'[2k+1][2r+1] = -Br
// so C'[i][2r], C'[i][2r+1] are the real and imaginary parts of the complex
// result (8 real flops per complex MAC, the 4M count), and the conjugation of
// the adjoint folds into B' signs. Each CTA computes a 128 x 32-complex output
// tile of one frequency with 8 warps (4 x 2), each warp 2 x 4 m16n8k4 tiles,
// the K loop fed by a 4-stage cp.async pipeline. K is reduced in a fixed order
// inside one CTA: results are deterministic.
#include <algorithm>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "btg_kernels.cuh"

namespace btg {
namespace {

constexpr int kThreads = 256;
constexpr int kTileM = 128;   // output rows per CTA (N_d rows fwd, N_m columns adj)
constexpr int kTileR = 32;    // complex right-hand sides per CTA (64 real columns)
constexpr int kStages = 4;

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
        "{%0, %1, %2, %3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = valid ? 16 : 0;  // zero-fill out-of-range chunks
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// B' element for real (k', n') inside the embedding from complex b = B[k][r].
template <bool kAdjoint>
__device__ __forceinline__ double embed_b(double2 b, int s, int t) {
    if (!kAdjoint) return s == 0 ? (t == 0 ? b.x : b.y) : (t == 0 ? -b.y : b.x);
    return s == 0 ? (t == 0 ? b.x : b.y) : (t == 0 ? b.y : -b.x);
}

// ---------------------------------------------------------------------------
// forward: per f, D_f[r][i] = sum_j F[f][i][j] X[f][r][j]
// ---------------------------------------------------------------------------
constexpr int kFwdKc = 16;                  // complex j per stage
constexpr int kFwdAStride = 2 * kFwdKc + 2;  // doubles per A row (padded)
constexpr int kFwdBStride = kFwdKc + 2;      // complex per B row (padded: the 4 r x 2 k fragment words hit 8 distinct banks)
constexpr size_t kFwdStageDoubles = (size_t)kTileM * kFwdAStride + 2 * (size_t)kTileR * kFwdBStride;

__global__ void __launch_bounds__(kThreads, 1)
    k_zgemm_fwd(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nd,
                int nm, int nrhs) {
    extern __shared__ __align__(16) double sm[];
    const int f = blockIdx.y;
    const int m0 = blockIdx.x * kTileM;
    const int r0 = blockIdx.z * kTileR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const double2* Ff = F + (size_t)f * nd * nm;
    const double2* Xf = X + (size_t)f * nrhs * nm;

    auto stage_a = [&](int st) { return sm + (size_t)st * kFwdStageDoubles; };
    auto stage_b = [&](int st) {
        return reinterpret_cast<double2*>(sm + (size_t)st * kFwdStageDoubles + (size_t)kTileM * kFwdAStride);
    };
    auto load_stage = [&](int st, int kc) {
        double* As = stage_a(st);
        double2* Bs = stage_b(st);
        // A: 128 rows x 16 complex = 2048 16-byte chunks
#pragma unroll
        for (int q = 0; q < (kTileM * kFwdKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int row = idx / kFwdKc, col = idx % kFwdKc;
            const int gi = m0 + row, gj = kc + col;
            const bool ok = gi < nd && gj < nm;
            cp_async16(As + row * kFwdAStride + 2 * col, Ff + (size_t)(ok ? gi : 0) * nm + (ok ? gj : 0), ok);
        }
        // B: 32 rhs x 16 complex = 512 chunks
#pragma unroll
        for (int q = 0; q < (kTileR * kFwdKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int r = idx / kFwdKc, col = idx % kFwdKc;
            const int gr = r0 + r, gj = kc + col;
            const bool ok = gr < nrhs && gj < nm;
            cp_async16(Bs + r * kFwdBStride + col, Xf + (size_t)(ok ? gr : 0) * nm + (ok ? gj : 0), ok);
        }
    };

    double acc[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

    const int nk = (nm + kFwdKc - 1) / kFwdKc;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load_stage(s, s * kFwdKc);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nxt = kt + kStages - 1;
            if (nxt < nk) load_stage(nxt % kStages, nxt * kFwdKc);
            cp_async_commit();
        }
        const double* As = stage_a(kt % kStages);
        const double2* Bs = stage_b(kt % kStages);
#pragma unroll
        for (int ks = 0; ks < (2 * kFwdKc) / 4; ++ks) {
            const int kp = ks * 4 + tig;  // real k' of this lane's A column / B row
            double a0[2], a1[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int row = wm * 32 + mt * 16 + g;
                a0[mt] = As[row * kFwdAStride + kp];
                a1[mt] = As[(row + 8) * kFwdAStride + kp];
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int n = wn * 32 + nt * 8 + g;  // real output column
                const double2 b = Bs[(n >> 1) * kFwdBStride + (kp >> 1)];
                const double bv = embed_b<false>(b, kp & 1, n & 1);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) dmma(acc[mt][nt], a0[mt], a1[mt], bv);
            }
        }
    }
    cp_async_wait<0>();

    // epilogue: lane holds C'[row][2c], C'[row][2c+1] = complex D[r][row]
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int r = r0 + ((wn * 32 + nt * 8) >> 1) + tig;
            const int row = m0 + wm * 32 + mt * 16 + g;
            if (r < nrhs) {
                double2* yr = Y + ((size_t)f * nrhs + r) * nd;
                if (row < nd) yr[row] = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
                if (row + 8 < nd) yr[row + 8] = make_double2(acc[mt][nt][2], acc[mt][nt][3]);
            }
        }
}

// ---------------------------------------------------------------------------
// adjoint: per f, G_f[r][j] = sum_i conj(F[f][i][j]) D[f][r][i]
// ---------------------------------------------------------------------------
constexpr int kAdjKc = 16;                      // complex i per stage
constexpr int kAdjAStride = kTileM + 4;         // complex per A row (i), padded
constexpr int kAdjBStride = kAdjKc + 2;         // complex per B row (r)
constexpr size_t kAdjStageDoubles = 2 * ((size_t)kAdjKc * kAdjAStride + (size_t)kTileR * kAdjBStride);

__global__ void __launch_bounds__(kThreads, 1)
    k_zgemm_adj(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nd,
                int nm, int nrhs) {
    extern __shared__ __align__(16) double sm[];
    const int f = blockIdx.y;
    const int j0 = blockIdx.x * kTileM;
    const int r0 = blockIdx.z * kTileR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const double2* Ff = F + (size_t)f * nd * nm;
    const double2* Xf = X + (size_t)f * nrhs * nd;

    auto stage_a = [&](int st) { return reinterpret_cast<double2*>(sm + (size_t)st * kAdjStageDoubles); };
    auto stage_b = [&](int st) {
        return reinterpret_cast<double2*>(sm + (size_t)st * kAdjStageDoubles + 2 * (size_t)kAdjKc * kAdjAStride);
    };
    auto load_stage = [&](int st, int kc) {
        double2* As = stage_a(st);
        double2* Bs = stage_b(st);
        // A: 16 rows (i) x 128 complex (j) = 2048 chunks
#pragma unroll
        for (int q = 0; q < (kAdjKc * kTileM) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int ii = idx / kTileM, jj = idx % kTileM;
            const int gi = kc + ii, gj = j0 + jj;
            const bool ok = gi < nd && gj < nm;
            cp_async16(As + ii * kAdjAStride + jj, Ff + (size_t)(ok ? gi : 0) * nm + (ok ? gj : 0), ok);
        }
        // B: 32 rhs x 16 complex (i)
#pragma unroll
        for (int q = 0; q < (kTileR * kAdjKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int r = idx / kAdjKc, ii = idx % kAdjKc;
            const int gr = r0 + r, gi = kc + ii;
            const bool ok = gr < nrhs && gi < nd;
            cp_async16(Bs + r * kAdjBStride + ii, Xf + (size_t)(ok ? gr : 0) * nd + (ok ? gi : 0), ok);
        }
    };

    double acc[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

    const int nk = (nd + kAdjKc - 1) / kAdjKc;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load_stage(s, s * kAdjKc);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nxt = kt + kStages - 1;
            if (nxt < nk) load_stage(nxt % kStages, nxt * kAdjKc);
            cp_async_commit();
        }
        const double* As = reinterpret_cast<const double*>(stage_a(kt % kStages));
        const double2* Bs = stage_b(kt % kStages);
#pragma unroll
        for (int ks = 0; ks < (2 * kAdjKc) / 4; ++ks) {
            const int kp = ks * 4 + tig;  // real k' = 2 i + s
            const int ii = kp >> 1, sp = kp & 1;
            double a0[2], a1[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int jj = wm * 32 + mt * 16 + g;
                a0[mt] = As[2 * (ii * kAdjAStride + jj) + sp];
                a1[mt] = As[2 * (ii * kAdjAStride + jj + 8) + sp];
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int n = wn * 32 + nt * 8 + g;
                const double2 b = Bs[(n >> 1) * kAdjBStride + ii];
                const double bv = embed_b<true>(b, sp, n & 1);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) dmma(acc[mt][nt], a0[mt], a1[mt], bv);
            }
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int r = r0 + ((wn * 32 + nt * 8) >> 1) + tig;
            const int jj = j0 + wm * 32 + mt * 16 + g;
            if (r < nrhs) {
                double2* yr = Y + ((size_t)f * nrhs + r) * nm;
                if (jj < nm) yr[jj] = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
                if (jj + 8 < nm) yr[jj + 8] = make_double2(acc[mt][nt][2], acc[mt][nt][3]);
            }
        }
}

// ---------------------------------------------------------------------------
// 3M variants (default): three real products per complex product instead of the
// four the embedding above performs, so each DMMA carries 4/3 as many complex
// MACs (6 real flops per complex MAC instead of 8):
//   forward  P1 = Fr Xr, P2 = Fi Xi, P3 = (Fr + Fi)(Xr + Xi);  D = (P1 - P2, P3 - P1 - P2)
//   adjoint  P1 = Fr Dr, P2 = Fi Di, P3 = (Fr - Fi)(Dr + Di);  G = (P1 + P2, P3 - P1 + P2)
// K runs over complex indices; one 16-byte shared load yields both parts of an
// operand, and the operand sums are formed in registers. The same 128 x 32-complex
// CTA tile; each warp owns 32 rows x 16 complex RHS (2 x 2 m16n8k4 tiles per
// product). Padded strides keep every fragment load conflict-free (16-byte
// slots: row stride = 16 banks mod 32 for the forward A / both B, 8 for the
// adjoint A). Normwise the 3M error bound is a small constant times the 4M one
// (the parity bar is relative L2 over the output); the fixed K order keeps results
// deterministic.
// ---------------------------------------------------------------------------
constexpr int kF3AStride = 2 * kFwdKc + 8;  // doubles per A row
constexpr int kM3BStride = kFwdKc + 4;      // complex per B row (both directions)
constexpr size_t kF3StageDoubles = (size_t)kTileM * kF3AStride + 2 * (size_t)kTileR * kM3BStride;
constexpr int kA3AStride = kTileM + 2;      // complex per adjoint A row (i)
constexpr size_t kA3StageDoubles = 2 * ((size_t)kAdjKc * kA3AStride + (size_t)kTileR * kM3BStride);

template <bool kAdj>
__device__ __forceinline__ void mma3(double (&p1)[2][2][4], double (&p2)[2][2][4], double (&p3)[2][2][4],
                                     const double2 (&a)[2][2], const double2 (&b)[2]) {
    double as[2][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) as[mt][h] = kAdj ? a[mt][h].x - a[mt][h].y : a[mt][h].x + a[mt][h].y;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const double bs = b[nt].x + b[nt].y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            dmma(p1[mt][nt], a[mt][0].x, a[mt][1].x, b[nt].x);
            dmma(p2[mt][nt], a[mt][0].y, a[mt][1].y, b[nt].y);
            dmma(p3[mt][nt], as[mt][0], as[mt][1], bs);
        }
    }
}

template <int ST, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_zgemm3m_fwd(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nd,
                  int nm, int nrhs, int j0, int nj, bool accumulate) {
    extern __shared__ __align__(16) double sm[];
    const int f = blockIdx.y;
    const int m0 = blockIdx.x * kTileM;
    const int r0 = blockIdx.z * kTileR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const double2* Ff = F + (size_t)f * nd * nm;
    const double2* Xf = X + (size_t)f * nrhs * nm;

    auto stage_a = [&](int st) { return sm + (size_t)st * kF3StageDoubles; };
    auto stage_b = [&](int st) {
        return reinterpret_cast<double2*>(sm + (size_t)st * kF3StageDoubles + (size_t)kTileM * kF3AStride);
    };
    auto load_stage = [&](int st, int kc) {
        double* As = stage_a(st);
        double2* Bs = stage_b(st);
#pragma unroll
        for (int q = 0; q < (kTileM * kFwdKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int row = idx / kFwdKc, col = idx % kFwdKc;
            const int gi = m0 + row, gj = j0 + kc + col;
            const bool ok = gi < nd && kc + col < nj;
            cp_async16(As + row * kF3AStride + 2 * col, Ff + (size_t)(ok ? gi : 0) * nm + (ok ? gj : 0), ok);
        }
#pragma unroll
        for (int q = 0; q < (kTileR * kFwdKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int r = idx / kFwdKc, col = idx % kFwdKc;
            const int gr = r0 + r, gj = j0 + kc + col;
            const bool ok = gr < nrhs && kc + col < nj;
            cp_async16(Bs + r * kM3BStride + col, Xf + (size_t)(ok ? gr : 0) * nm + (ok ? gj : 0), ok);
        }
    };

    double p1[2][2][4], p2[2][2][4], p3[2][2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;

    const int nk = (nj + kFwdKc - 1) / kFwdKc;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) load_stage(s, s * kFwdKc);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nxt = kt + ST - 1;
            if (nxt < nk) load_stage(nxt % ST, nxt * kFwdKc);
            cp_async_commit();
        }
        const double* As = stage_a(kt % ST);
        const double2* Bs = stage_b(kt % ST);
#pragma unroll
        for (int ks = 0; ks < kFwdKc / 4; ++ks) {
            const int kk = ks * 4 + tig;  // complex k of this lane's A column / B row
            double2 a[2][2], b[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    a[mt][h] = *reinterpret_cast<const double2*>(As + (wm * 32 + mt * 16 + h * 8 + g) * kF3AStride +
                                                                 2 * kk);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[(wn * 16 + nt * 8 + g) * kM3BStride + kk];
            mma3<false>(p1, p2, p3, a, b);
        }
    }
    cp_async_wait<0>();

    // lane holds C[g (+8)][2 tig + q]: rows (i) x complex RHS
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int r = r0 + wn * 16 + nt * 8 + 2 * tig + q;
                if (r >= nrhs) continue;
                double2* yr = Y + ((size_t)f * nrhs + r) * nd;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int row = m0 + wm * 32 + mt * 16 + h * 8 + g;
                    const int c = 2 * h + q;
                    if (row < nd) {
                        double2 v = make_double2(p1[mt][nt][c] - p2[mt][nt][c],
                                                 p3[mt][nt][c] - p1[mt][nt][c] - p2[mt][nt][c]);
                        if (accumulate) {  // column-chunk partial sums, added in chunk order
                            const double2 o = yr[row];
                            v.x += o.x;
                            v.y += o.y;
                        }
                        yr[row] = v;
                    }
                }
            }
}

template <int ST, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_zgemm3m_adj(const double2* __restrict__ F, const double2* __restrict__ X, double2* __restrict__ Y, int nd,
                  int nm, int nrhs, int jbase, int jend) {
    extern __shared__ __align__(16) double sm[];
    const int f = blockIdx.y;
    const int j0 = jbase + blockIdx.x * kTileM;
    const int r0 = blockIdx.z * kTileR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const double2* Ff = F + (size_t)f * nd * nm;
    const double2* Xf = X + (size_t)f * nrhs * nd;

    auto stage_a = [&](int st) { return reinterpret_cast<double2*>(sm + (size_t)st * kA3StageDoubles); };
    auto stage_b = [&](int st) {
        return reinterpret_cast<double2*>(sm + (size_t)st * kA3StageDoubles + 2 * (size_t)kAdjKc * kA3AStride);
    };
    auto load_stage = [&](int st, int kc) {
        double2* As = stage_a(st);
        double2* Bs = stage_b(st);
#pragma unroll
        for (int q = 0; q < (kAdjKc * kTileM) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int ii = idx / kTileM, jj = idx % kTileM;
            const int gi = kc + ii, gj = j0 + jj;
            const bool ok = gi < nd && gj < jend;
            cp_async16(As + ii * kA3AStride + jj, Ff + (size_t)(ok ? gi : 0) * nm + (ok ? gj : 0), ok);
        }
#pragma unroll
        for (int q = 0; q < (kTileR * kAdjKc) / kThreads; ++q) {
            const int idx = threadIdx.x + q * kThreads;
            const int r = idx / kAdjKc, ii = idx % kAdjKc;
            const int gr = r0 + r, gi = kc + ii;
            const bool ok = gr < nrhs && gi < nd;
            cp_async16(Bs + r * kM3BStride + ii, Xf + (size_t)(ok ? gr : 0) * nd + (ok ? gi : 0), ok);
        }
    };

    double p1[2][2][4], p2[2][2][4], p3[2][2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < 4; ++c) p1[a][b][c] = p2[a][b][c] = p3[a][b][c] = 0.0;

    const int nk = (nd + kAdjKc - 1) / kAdjKc;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) load_stage(s, s * kAdjKc);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nxt = kt + ST - 1;
            if (nxt < nk) load_stage(nxt % ST, nxt * kAdjKc);
            cp_async_commit();
        }
        const double2* As = stage_a(kt % ST);
        const double2* Bs = stage_b(kt % ST);
#pragma unroll
        for (int ks = 0; ks < kAdjKc / 4; ++ks) {
            const int kk = ks * 4 + tig;  // complex i of this lane's A column / B row
            double2 a[2][2], b[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) a[mt][h] = As[kk * kA3AStride + wm * 32 + mt * 16 + h * 8 + g];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[(wn * 16 + nt * 8 + g) * kM3BStride + kk];
            mma3<true>(p1, p2, p3, a, b);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int r = r0 + wn * 16 + nt * 8 + 2 * tig + q;
                if (r >= nrhs) continue;
                double2* yr = Y + ((size_t)f * nrhs + r) * nm;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int jj = j0 + wm * 32 + mt * 16 + h * 8 + g;
                    const int c = 2 * h + q;
                    if (jj < jend)
                        yr[jj] = make_double2(p1[mt][nt][c] + p2[mt][nt][c],
                                              p3[mt][nt][c] - p1[mt][nt][c] + p2[mt][nt][c]);
                }
            }
}

bool use_4m() {
    static const bool v = std::getenv("BTG_ZGEMM_4M") != nullptr;
    return v;
}
// BTG_ZGEMM_LEGACY=1: the two-CTAs-per-SM cp.async kernels below instead of the
// warp-specialised ones (btg_zgemm_ws.cu). Read per call (A/B measurements).
bool use_legacy() {
    const char* v = std::getenv("BTG_ZGEMM_LEGACY");
    return v && *v && *v != '0';
}

constexpr int kMaxGridY = 65535;

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

bool zgemm_3m() { return !use_4m(); }
bool zgemm_ws_active() { return !use_4m() && !use_legacy(); }

cudaError_t launch_zgemm_fwd_range(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm,
                                   int nrhs, int j0, int nj, bool accumulate, cudaStream_t stream) {
    if (use_4m() && (j0 != 0 || nj != nm || accumulate)) return cudaErrorNotSupported;
    const bool m4 = use_4m();
    if (!m4 && !use_legacy()) return launch_zgemm3m_fwd_ws(F, X, Y, nf, nd, nm, nrhs, j0, nj, accumulate, stream);
    // 2 CTAs per SM (<= 128 registers, 2 stages), as the adjoint: 15.0 -> 13.7 ms at
    // configs[3] (1 CTA x 4 stages), despite 3.5 instead of 6.9 waves.
    const auto k3 = k_zgemm3m_fwd<2, 2>;
    const size_t smem = (m4 ? kStages * kFwdStageDoubles : 2 * kF3StageDoubles) * sizeof(double);
    cudaError_t e = m4 ? set_smem(k_zgemm_fwd, smem) : set_smem(k3, smem);
    if (e != cudaSuccess) return e;
    for (int f0 = 0; f0 < nf; f0 += kMaxGridY) {  // grid.y limit: long horizons go in frequency batches
        const int nb = std::min(kMaxGridY, nf - f0);
        dim3 grid((nd + kTileM - 1) / kTileM, nb, (nrhs + kTileR - 1) / kTileR);
        const double2* Fb = F + (size_t)f0 * nd * nm;
        const double2* Xb = X + (size_t)f0 * nrhs * nm;
        double2* Yb = Y + (size_t)f0 * nrhs * nd;
        if (m4)
            k_zgemm_fwd<<<grid, kThreads, smem, stream>>>(Fb, Xb, Yb, nd, nm, nrhs);
        else
            k3<<<grid, kThreads, smem, stream>>>(Fb, Xb, Yb, nd, nm, nrhs, j0, nj, accumulate);
    }
    return cudaGetLastError();
}

cudaError_t launch_zgemm_fwd(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                             cudaStream_t stream) {
    return launch_zgemm_fwd_range(F, X, Y, nf, nd, nm, nrhs, 0, nm, false, stream);
}

cudaError_t launch_zgemm_adj_range(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm,
                                   int nrhs, int j0, int nj, cudaStream_t stream) {
    if (use_4m() && (j0 != 0 || nj != nm)) return cudaErrorNotSupported;
    const bool m4 = use_4m();
    if (!m4 && !use_legacy()) return launch_zgemm3m_adj_ws(F, X, Y, nf, nd, nm, nrhs, j0, nj, stream);
    // 2 CTAs per SM (<= 128 registers, 2 stages): one CTA's prologue / epilogue
    // overlaps the other's MMAs; K = N_d is short (configs[3]: 8 stages per tile).
    // Measured 16.3 -> 14.1 ms at configs[3] (1 CTA x 4 stages before).
    const auto k3 = k_zgemm3m_adj<2, 2>;
    const size_t smem = (m4 ? kStages * kAdjStageDoubles : 2 * kA3StageDoubles) * sizeof(double);
    cudaError_t e = m4 ? set_smem(k_zgemm_adj, smem) : set_smem(k3, smem);
    if (e != cudaSuccess) return e;
    for (int f0 = 0; f0 < nf; f0 += kMaxGridY) {
        const int nb = std::min(kMaxGridY, nf - f0);
        dim3 grid((nj + kTileM - 1) / kTileM, nb, (nrhs + kTileR - 1) / kTileR);
        const double2* Fb = F + (size_t)f0 * nd * nm;
        const double2* Xb = X + (size_t)f0 * nrhs * nd;
        double2* Yb = Y + (size_t)f0 * nrhs * nm;
        if (m4)
            k_zgemm_adj<<<grid, kThreads, smem, stream>>>(Fb, Xb, Yb, nd, nm, nrhs);
        else
            k3<<<grid, kThreads, smem, stream>>>(Fb, Xb, Yb, nd, nm, nrhs, j0, j0 + nj);
    }
    return cudaGetLastError();
}

cudaError_t launch_zgemm_adj(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                             cudaStream_t stream) {
    return launch_zgemm_adj_range(F, X, Y, nf, nd, nm, nrhs, 0, nm, stream);
}

}  // namespace btg
