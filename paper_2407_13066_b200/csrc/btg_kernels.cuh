// Launch interface of the sm_100a kernels behind the C ABI (btg_capi.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "btg_fft.cuh"

namespace btg {

// Epilogue of the C2R kernel: y = x * gamma (optional) + alpha * R(v) (optional).
struct C2REpilogue {
    const double* gamma = nullptr;  // per channel (mode 1) or per (channel, t) (mode 2)
    int gamma_mode = 0;
    int gamma_dim = 1;              // channels per right-hand side (gamma index = c % gamma_dim)
    const double* v = nullptr;      // SOTI vector sharing the output layout
    double alpha = 0.0;
    int reg_kind = 0;               // 0 identity, 1 temporal Laplacian (inverse.cpp:32-49)
    // Optional dot product folded into the stores (CG's p^T H p): each CTA writes
    // sum_t dot_v[c][t] * y[c][t] over its channels to dot_out[blockIdx.x] (fast
    // kernels only; the launcher reports the CTA count).
    const double* dot_v = nullptr;  // SOTI vector sharing the output layout
    double* dot_out = nullptr;
    // Grid reduce fused into the stores (btg_grid_engine.cu, P2P transport): the
    // partials of the other npeers members of this cell's row / column group,
    // same layout as the output, possibly on other GPUs (NVLink peer loads);
    // device array of pointers. The stored value is the reference's tree_reduce
    // (distributed.cpp:36-47) of {own, peers[0], ..} in member order.
    const double* const* peers = nullptr;
    int npeers = 0;
};
constexpr int kMaxFusedPeers = 7;  // groups of up to 8 members

// Split twiddle tables of the compile-time-N vector FFTs (btg_fft_fast.cuh):
// lo[i] = W_N^i (i < 32), hi[h] = W_N^{32h}; post_* the same for W_{2N}.
// R2C epilogue of the int8 multi-RHS engine (btg_fft_fast.cuh block_max): per
// channel group (the CTA's CPB channels) and frequency, the block exponent of
// max |re|, |im| (scale_exp, INT16_MIN for zero) — pexp[group][k], plain stores;
// oz_exponents_from_groups() takes the max over each 1024-channel block. The
// exponent is monotonic in the value, so this is the exponent of the exact max.
struct R2CBlockMax {
    int16_t* pexp = nullptr;
    int nf = 0;  // frequencies (row length of pexp)
};

struct FastTables {
    const double2* lo = nullptr;
    const double2* hi = nullptr;
    const double2* post_lo = nullptr;
    const double2* post_hi = nullptr;
    const double2* wn = nullptr;   // W_N^k, k < N (direct pass tables)
    const double2* w2n = nullptr;  // W_2N^k, k <= N (octant table)
};

// Lengths N = N_t with a register-resident compile-time plan.
bool fast_fft_supported(int n);
// Channels per CTA of the fast R2C for length n (0 if no fast plan).
int fast_r2c_cpb(int n);
int fast_fft_hi_count(int n);  // entries of hi (post_hi has one more)

// Channel-blocked spectral layout (out_fs / in_fs = kBlockedFs): [c / kSpecBlock]
// [k][c % kSpecBlock], N_t + 1 frequencies (btg_fft_fast.cuh spec_base). Only
// lengths whose fast R2C and C2R channels per CTA divide kSpecBlock take it
// (spec_blocked_ok); the multi-RHS ZGEMM (TMA kernels) reads / writes it.
constexpr long long kBlockedFs = -1;
#ifndef BTG_SPEC_BLOCK
#define BTG_SPEC_BLOCK 4
#endif
constexpr int kSpecBlock = BTG_SPEC_BLOCK;
bool spec_blocked_ok(int n);
// SOTI rows (16-byte aligned) -> frequency-major; returns cudaErrorNotSupported
// when N has no compile-time plan.
cudaError_t launch_r2c_vec_fast(int n, const double* in, long long in_cs, double2* out, long long out_fs,
                                int channels, const FastTables& tabs, cudaStream_t stream,
                                const R2CBlockMax& bm = R2CBlockMax{});
cudaError_t launch_c2r_vec_fast(int n, const double2* in, long long in_fs, double* out, long long out_cs,
                                int channels, const FastTables& tabs, const C2REpilogue& epi,
                                cudaStream_t stream, int* ctas = nullptr);

// Per-channel shared-memory footprint (complex elements) of an FFT of length n.
__host__ __device__ inline int fft_channel_stride(int n) { return n + 1; }

// Channels per CTA for the FFT kernels given the smem budget.
int fft_batch(int n, size_t smem_budget, int want);
size_t fft_smem_bytes(int n, int batch);

// Global-memory ping-pong buffers for horizons whose two-buffer transform does
// not fit shared memory (generic path; setup and lengths without a fast plan):
// `ctas` persistent CTAs, each owning 2 * batch * fft_channel_stride(n) elements.
struct FftScratch {
    double2* buf = nullptr;
    int ctas = 0;
};

// Real-to-complex along time of C channels: channel c sample t at
// in[c*in_cs + t*in_ts] (t < nt, zero-padded to 2nt); frequency k <= nt lands
// at out[k*out_fs + c*out_cs]. TOut = double2 (FP64) or float2 (FP32 F-hat).
template <typename TOut>
cudaError_t launch_r2c(const double* in, long long in_cs, long long in_ts, TOut* out,
                       long long out_fs, long long out_cs, int channels, int nt,
                       const FftPlanDev& plan, int batch, cudaStream_t stream,
                       const FftScratch& gs = FftScratch{});

// Complex-to-real: frequency k <= nt of channel c at in[k*in_fs + c*in_cs];
// output time t < nt (1/(2nt) normalised, real part) at out[c*out_cs + t],
// through the epilogue.
cudaError_t launch_c2r(const double2* in, long long in_fs, long long in_cs, double* out,
                       long long out_cs, int channels, int nt, const FftPlanDev& plan,
                       int batch, const C2REpilogue& epi, cudaStream_t stream,
                       const FftScratch& gs = FftScratch{});

// Fourier-space step, one right-hand side: y[f][i] = sum_j F[f][i][j] x[f][j].
template <typename TF>
cudaError_t launch_gemv_fwd(const TF* F, const double2* x, double2* y, int nf, int nd, int nm,
                            cudaStream_t stream);

// Column-chunk variants for host<->device pipelines: columns [j0, j0 + nj)
// only; the forward one adds into y when `accumulate` (chunks in a fixed order).
template <typename TF>
cudaError_t launch_gemv_fwd_range(const TF* F, const double2* x, double2* y, int nf, int nd, int nm, int j0,
                                  int nj, bool accumulate, cudaStream_t stream);
template <typename TF>
cudaError_t launch_gemv_adj_range(const TF* F, const double2* x, double2* y, int nf, int nd, int nm, int j0,
                                  int nj, cudaStream_t stream);

// Adjoint: y[f][j] = sum_i conj(F[f][i][j]) x[f][i].
template <typename TF>
cudaError_t launch_gemv_adj(const TF* F, const double2* x, double2* y, int nf, int nd, int nm,
                            cudaStream_t stream);

// TMA-staged persistent single-RHS Fourier-space step, FP64 F-hat (btg_gemv_tma.cu).
cudaError_t launch_gemv_fwd_tma(const double2* F, const double2* x, double2* y, int nf, int nd, int nm,
                                cudaStream_t stream);
cudaError_t launch_gemv_adj_tma(const double2* F, const double2* x, double2* y, int nf, int nd, int nm,
                                cudaStream_t stream);

// Multi-RHS Fourier-space step on FP64 tensor cores (btg_zgemm.cu). X/Y are
// [f][r][dim] (dim = N_m or N_d), FP64 F-hat only.
// Multi-RHS step on the tcgen05 int8 tensor cores (Ozaki splitting, btg_ozaki.cu).
size_t oz_operator_bytes(int nf, int nd, int nm);
size_t oz_operator_scales(int nf, int nm);
size_t oz_vector_scales(int nf, int nrhs, int kdim);
cudaError_t oz_quantize_operator(const double2* F, int nf, int nd, int nm, int8_t* Aq, unsigned long long* mA,
                                 cudaStream_t stream);
// EWP backend (btg_ewp.cu): channel layout S[c][f] of F-hat, element-wise products.
template <typename T>
cudaError_t launch_channel_layout(const T* F, T* S, int nf, long long channels, cudaStream_t stream);
template <typename T>
cudaError_t launch_ewp(bool adjoint, const T* S, const double2* in, double2* out, int nf, int nd, int nm,
                       cudaStream_t stream);

// Naive backend (btg_naive.cu): direct triangular sum on the compact operator.
cudaError_t launch_naive(bool adjoint, const double* blocks, const double* in, double* out, int nd, int nm, int nt,
                         cudaStream_t stream);

// Bq: workspace of oz_presliced_bytes(nf, nd) for the adjoint's pre-sliced d-hat tiles.
size_t oz_presliced_bytes(int nf, int nd);
// vexp: optional per-group exponents of V from the R2C epilogue (R2CBlockMax,
// forward, nrhs <= 32; groups of vexp_cpb channels).
cudaError_t oz_apply(bool adjoint, const int8_t* Aq, const unsigned long long* mA, const double2* V, double2* Y,
                     int nf, int nd, int nm, int nrhs, int* mB, uint8_t* Bq, cudaStream_t stream,
                     const int16_t* vexp = nullptr, int vexp_cpb = 1);

// Warp-specialised persistent 3M kernels (btg_zgemm_ws.cu; the default unless
// BTG_ZGEMM_LEGACY / BTG_ZGEMM_4M): one CTA per SM, producer warp on bulk copies.
// xblocked / yblocked: the N_m-side spectrum in the channel-blocked layout
// (kBlockedFs; TMA kernels only — cudaErrorNotSupported otherwise).
cudaError_t launch_zgemm3m_fwd_ws(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                                  int j0, int nj, bool accumulate, cudaStream_t stream, bool xblocked = false);
cudaError_t launch_zgemm3m_adj_ws(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                                  int j0, int nj, cudaStream_t stream, bool yblocked = false);
// the TMA ZGEMM (and with it the blocked layout) is available for this N_m
bool zgemm_tma_ok(int nm);
// the warp-specialised 3M kernels are selected (not BTG_ZGEMM_LEGACY / BTG_ZGEMM_4M)
bool zgemm_ws_active();
// 3M kernels active (BTG_ZGEMM_4M unset): column ranges [j0, j0 + nj) supported.
bool zgemm_3m();
cudaError_t launch_zgemm_fwd_range(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm,
                                   int nrhs, int j0, int nj, bool accumulate, cudaStream_t stream);
cudaError_t launch_zgemm_adj_range(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm,
                                   int nrhs, int j0, int nj, cudaStream_t stream);
cudaError_t launch_zgemm_fwd(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                             cudaStream_t stream);
cudaError_t launch_zgemm_adj(const double2* F, const double2* X, double2* Y, int nf, int nd, int nm, int nrhs,
                             cudaStream_t stream);

// CG vector kernels (btg_blas.cu). Reductions use a fixed grid of kRedBlocks
// blocks; `partial` holds kRedBlocks doubles; scalar results land in device memory.
constexpr int kRedBlocks = 592;
cudaError_t launch_dot(const double* a, const double* b, size_t n, double* partial, double* out,
                       cudaStream_t stream);
cudaError_t launch_cg_update(double* x, double* r, const double* p, const double* hp, double s, size_t n,
                             double* partial, double* rnorm2, cudaStream_t stream);
cudaError_t launch_xpby(double* p, const double* z, double beta, size_t n, cudaStream_t stream);
// out = sum of partial[0..count) in index order (one block; deterministic)
cudaError_t launch_sum_partials(const double* partial, int count, double* out, cudaStream_t stream);
// Device-side CG loop (btg_cg_solve's CUDA graph WHILE body): scalars in a
// CgState array of kCgStateLen doubles.
enum CgStateIdx {
    kCgRho = 0, kCgCurvature, kCgRn2, kCgRhoNext, kCgRhsNorm, kCgTol, kCgRelRes, kCgIterations, kCgMaxIt,
    kCgStatus, kCgBeta, kCgStateLen
};
constexpr double kCgRunning = 0.0, kCgConverged = 1.0, kCgBadCurvature = 2.0, kCgMaxIterations = 3.0;
cudaError_t launch_cg_update_dev(double* x, double* r, const double* p, const double* hp, const double* st, size_t n,
                                 double* partial, cudaStream_t stream);
cudaError_t launch_cg_check(const double* partial, double* st, cudaGraphConditionalHandle cond, int precond,
                            cudaStream_t stream);
cudaError_t launch_cg_beta(double* st, cudaStream_t stream);
cudaError_t launch_xpby_dev(double* p, const double* z, const double* st, size_t n, cudaStream_t stream);
cudaError_t launch_sub(double* y, const double* a, const double* b, size_t n, cudaStream_t stream);
cudaError_t launch_reg_apply(double* y, const double* v, size_t rows, int nt, int kind, cudaStream_t stream);
cudaError_t launch_reg_apply_inverse(double* x, const double* b, const double* pivot, const double* scratch,
                                     size_t rows, int nt, cudaStream_t stream);

// SOTI rows out[c * nt + t] from a TOSI slab in[t * ts + c], c < cnt, t < nt
cudaError_t launch_tosi_to_soti(const double* in, long long ts, double* out, int nt, long long cnt,
                                cudaStream_t stream);

// out[k * out_fs + c] = (complex64) in[k * cnt + c], k < nf, c < cnt
cudaError_t launch_spec_to_f32(const double2* in, long long cnt, int nf, float2* out, long long out_fs,
                               cudaStream_t stream);

// out[(a*nb + b)*nc + c] = uniform(seed ^ (offset + a*sa + b*sb + c))
cudaError_t launch_fill_uniform(double* out, size_t na, size_t nb, size_t nc, uint64_t seed, uint64_t offset,
                                uint64_t sa, uint64_t sb, double lo, double hi, cudaStream_t stream);

}  // namespace btg
