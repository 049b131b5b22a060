// C ABI (include/btg.h) over the sm_100a kernels: the device-resident
// frequency-domain operator handle, its workspace, streams, counters and
// host<->device staging. Host logic mirrors the reference's operator API:
//   setup                block_operator.cpp:178-205
//   apply_forward        block_operator.cpp:218-273  (check_apply_input :123-133)
//   apply_adjoint        block_operator.cpp:275-331
//   HessianOperator::apply  inverse.cpp:78-91 (+ Gamma^-1, north star)
// There is no CPU compute path: every arithmetic step is a CUDA kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/btg.h"
#include "btg_fft.cuh"
#include "btg_kernels.cuh"

namespace {

thread_local std::string g_err;

btg_status fail(btg_status s, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define BTG_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? BTG_ENOMEM : BTG_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                   \
    } while (0)

#define BTG_TRY(call)                       \
    do {                                    \
        btg_status s_ = (call);             \
        if (s_ != BTG_OK) return s_;        \
    } while (0)

// exp(-2*pi*i*num/den) with exact integer argument reduction.
double2 root(long long num, long long den) {
    num %= den;
    if (num < 0) num += den;
    const long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)num / (long double)den;
    return make_double2((double)cosl(a), (double)(-sinl(a)));
}

std::vector<int> factorize(int n) {
    std::vector<int> f;
    while (n % 8 == 0) { f.push_back(8); n /= 8; }
    while (n % 4 == 0) { f.push_back(4); n /= 4; }
    while (n % 2 == 0) { f.push_back(2); n /= 2; }
    while (n % 5 == 0) { f.push_back(5); n /= 5; }
    while (n % 3 == 0) { f.push_back(3); n /= 3; }
    for (int p = 7; (long long)p * p <= n; p += 2)
        while (n % p == 0) { f.push_back(p); n /= p; }
    if (n > 1) f.push_back(n);
    return f;
}

constexpr size_t kFftSmemBudget = 200 * 1024;      // per CTA
constexpr size_t kFftSmemTarget = 100 * 1024;      // aim for 2 CTAs / SM
constexpr size_t kHostStageBytes = 512ull << 20;   // host->device setup staging
constexpr size_t kScratchCapBytes = 1ull << 30;    // global FFT scratch bound
constexpr size_t kSetupSotiBytes = 1ull << 30;     // setup: transposed (SOTI) slab buffer

}  // namespace

struct HessKey {
    const double* v;
    double* hv;
    size_t nrhs;
    const double* gamma;
    int gamma_mode;
    double alpha;
    int reg_kind;
    const void *wa, *wb, *wt, *F;
    bool i8, no_dmma, legacy;
    bool operator==(const HessKey& o) const {
        return v == o.v && hv == o.hv && nrhs == o.nrhs && gamma == o.gamma && gamma_mode == o.gamma_mode &&
               alpha == o.alpha && reg_kind == o.reg_kind && wa == o.wa && wb == o.wb && wt == o.wt && F == o.F &&
               i8 == o.i8 && no_dmma == o.no_dmma && legacy == o.legacy;
    }
};
struct HessGraph {
    HessKey key{};
    cudaGraphExec_t exec = nullptr;
    btg_counters delta{};
};

struct btg_op_s {
    int device = 0;
    int precision = BTG_F64;
    size_t nd = 0, nm = 0, nt = 0, nf = 0;
    void* F = nullptr;  // [nf][nd][nm] double2 or float2
    size_t F_elem = 16;

    btg::FftPlanDev plan{};
    double2* d_tw = nullptr;
    double2* d_post = nullptr;
    double2* d_fast = nullptr;  // split twiddle tables of the compile-time-N FFTs
    btg::FftScratch gscratch;   // global ping-pong buffers when N_t exceeds shared memory
    btg::FastTables fast{};
    bool fast_ok = false;
    bool no_dmma = false;      // BTG_DISABLE_DMMA: per-RHS GEMV streams instead of the ZGEMM
    bool tensor_i8 = false;    // BTG_TENSOR_I8=1: multi-RHS step on tcgen05 int8 (Ozaki splitting)
    int8_t* oz_A = nullptr;    // int8 slices of F-hat (built lazily, invalidated by setup)
    unsigned long long* oz_mA = nullptr;
    int* oz_mB = nullptr;
    size_t oz_mB_cap = 0;
    uint8_t* oz_B = nullptr;  // adjoint: d-hat slices pre-sliced once per frequency
    int16_t* oz_vexp = nullptr;  // forward: x-hat block exponents per channel group, from the R2C
    size_t oz_vexp_cap = 0;
    size_t oz_B_cap = 0;
    bool oz_valid = false;
    bool keep_channel = false;  // EWP backend: SetupOptions::keep_channel_layout
    void* S = nullptr;          // channel-major copy of F-hat [c][f] (built on first EWP use)
    bool S_valid = false;
    bool legacy_gemv = true;   // register-load GEMV; BTG_GEMV_TMA=1 selects the TMA ring
    int fft_batch = 1;        // channels per CTA for vector transforms
    int fft_batch_setup = 1;  // channels per CTA for the TOSI setup transform

    cudaStream_t own_stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host<->device chunks of host-pointer calls
    cudaStream_t capture_stream = nullptr;  // CUDA-graph capture (CG iteration, Hessian replay)
    cudaEvent_t ev[17] = {};              // kHostChunks + 1 chunk / ordering events
    cudaStream_t fft_stream = nullptr;   // chunk R2Cs of host-pointer forward calls
    double* pinned_scalar = nullptr;     // page-locked landing slot for solver scalars
    double* pinned_state = nullptr;      // page-locked copy of the device CG state
    double* solver_ws[11] = {};           // CG / objective vectors, kept across calls
    size_t solver_cap[11] = {};
    cudaEvent_t ev_h2d[17] = {};          // chunk H2D done (copy stream -> fft stream)
    cudaStream_t stream = nullptr;

    // workspace (grown on demand)
    double2* wa = nullptr;
    double2* wb = nullptr;
    size_t wcap = 0;  // complex elements each
    double* wt = nullptr;
    size_t wtcap = 0;  // doubles: time-domain Hessian intermediate
    double* hin = nullptr;
    double* hout = nullptr;
    size_t hcap = 0;  // doubles each: staging for host-pointer calls
    double* gam = nullptr;
    size_t gcap = 0;
    double* vcopy = nullptr;
    size_t vcap = 0;

    HessGraph hess_graph;  // last device-pointer Hessian chain, replayed while its key matches
    std::vector<char> rows_ready;
    size_t rows_ready_count = 0;

    bool timing = false;
    btg_counters counters{};
    std::mutex mu;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
btg_status grow(T*& ptr, size_t& cap, size_t need) {
    if (need <= cap) return BTG_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&ptr), need * sizeof(T));
    if (e != cudaSuccess) {
        ptr = nullptr;
        return fail(BTG_ENOMEM, "device allocation of %zu bytes failed: %s", need * sizeof(T),
                    cudaGetErrorString(e));
    }
    cap = need;
    return BTG_OK;
}

// Stage timing: one event pair per stage when timing is enabled.
struct StageClock {
    btg_op op;
    btg_stage_counters* st;
    cudaEvent_t a = nullptr, b = nullptr;
    StageClock(btg_op o, btg_stage_counters* s) : op(o), st(s) {
        if (op->timing) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, op->stream);
        }
    }
    void stop() {
        if (op->timing && a) {
            cudaEventRecord(b, op->stream);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            st->seconds += ms * 1e-3;
            cudaEventDestroy(a);
            cudaEventDestroy(b);
            a = b = nullptr;
        }
    }
    ~StageClock() { stop(); }
};

double fft_ops(size_t channels, size_t nt) {
    const double len = 2.0 * (double)nt;
    return (double)channels * len * std::log2(len);
}

btg_status check_ready(btg_op op) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (op->rows_ready_count != op->nd)
        return fail(BTG_EARG, "operator setup incomplete: %zu of %zu sensor rows transformed",
                    op->rows_ready_count, op->nd);
    return BTG_OK;
}

// The two spectral buffers share one capacity counter; grow both together.
btg_status ensure_spectral(btg_op op, size_t nrhs) {
    const size_t need = op->nf * nrhs * std::max(op->nm, op->nd);
    if (need <= op->wcap && op->wa && op->wb) return BTG_OK;
    if (op->wa) cudaFree(op->wa);
    if (op->wb) cudaFree(op->wb);
    op->wa = op->wb = nullptr;
    op->wcap = 0;
    cudaError_t e = cudaMalloc(&op->wa, need * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc(&op->wb, need * sizeof(double2));
    if (e != cudaSuccess) {
        if (op->wa) cudaFree(op->wa);
        op->wa = nullptr;
        return fail(BTG_ENOMEM, "workspace allocation (2 x %zu bytes) failed: %s",
                    need * sizeof(double2), cudaGetErrorString(e));
    }
    op->wcap = need;
    return BTG_OK;
}

btg_status host_buffers(btg_op op, size_t nin, size_t nout) {
    const size_t need = std::max(nin, nout);
    if (need <= op->hcap && op->hin && op->hout) return BTG_OK;
    if (op->hin) cudaFree(op->hin);
    if (op->hout) cudaFree(op->hout);
    op->hin = op->hout = nullptr;
    op->hcap = 0;
    cudaError_t e = cudaMalloc(&op->hin, need * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&op->hout, need * sizeof(double));
    if (e != cudaSuccess) return fail(BTG_ENOMEM, "staging allocation failed: %s", cudaGetErrorString(e));
    op->hcap = need;
    return BTG_OK;
}

// ---- pipeline pieces --------------------------------------------------------
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// R2C of `channels` SOTI rows into a frequency-major array whose frequency
// stride is `fs` (default: channels; a column chunk of a wider array otherwise).
// blocked: write the channel-blocked layout (btg::kBlockedFs; the caller checked
// mrhs_blocked, which implies the fast plan runs kSpecBlock channels per CTA).
btg_status run_r2c_vec(btg_op op, const double* v, size_t channels, double2* out, size_t fs = 0,
                       const btg::R2CBlockMax* bm = nullptr, bool blocked = false) {
    StageClock clk(op, &op->counters.forward_fft);
    if (!fs) fs = channels;
    if (blocked)
        BTG_CUDA(btg::launch_r2c_vec_fast((int)op->nt, v, (long long)op->nt, out, btg::kBlockedFs, (int)channels,
                                          op->fast, op->stream));
    else if (op->fast_ok && aligned16(v) && aligned16(out))
        BTG_CUDA(btg::launch_r2c_vec_fast((int)op->nt, v, (long long)op->nt, out, (long long)fs,
                                          (int)channels, op->fast, op->stream, bm ? *bm : btg::R2CBlockMax{}));
    else if (bm)
        return fail(BTG_EARG, "internal: block maxima need the fast R2C");
    else
        BTG_CUDA(btg::launch_r2c<double2>(v, (long long)op->nt, 1, out, (long long)fs, 1,
                                          (int)channels, (int)op->nt, op->plan, op->fft_batch, op->stream,
                                          op->gscratch));
    op->counters.launches++;
    op->counters.forward_fft.ops += fft_ops(channels, op->nt);
    op->counters.forward_fft.bytes += 8.0 * channels * op->nt + 16.0 * op->nf * channels;
    // the zero-pad is fused into the R2C loads: the reference's op model
    // (block_operator.cpp:67-68), no separate bytes moved
    op->counters.pad.ops += 2.0 * channels * op->nt;
    return BTG_OK;
}

btg_status run_c2r_vec(btg_op op, const double2* in, size_t channels, double* out,
                       const btg::C2REpilogue& epi, size_t fs = 0, int* dot_ctas = nullptr, bool blocked = false) {
    StageClock clk(op, &op->counters.inverse_fft);
    if (!fs) fs = channels;
    // the fast epilogue reads alpha R v and per-sample Gamma^-1 as 16-byte pairs
    const bool epi_aligned = (!epi.v || aligned16(epi.v)) && (epi.gamma_mode != 2 || aligned16(epi.gamma));
    const bool dot_aligned = !epi.dot_out || aligned16(epi.dot_v);
    if (dot_ctas) *dot_ctas = 0;
    if (blocked) {
        if (!(aligned16(out) && epi_aligned && dot_aligned))
            return fail(BTG_EARG, "internal: blocked C2R needs 16-byte aligned vectors");
        BTG_CUDA(btg::launch_c2r_vec_fast((int)op->nt, in, btg::kBlockedFs, out, (long long)op->nt, (int)channels,
                                          op->fast, epi, op->stream, dot_ctas));
    } else if (op->fast_ok && aligned16(in) && aligned16(out) && epi_aligned && dot_aligned) {
        BTG_CUDA(btg::launch_c2r_vec_fast((int)op->nt, in, (long long)fs, out, (long long)op->nt,
                                          (int)channels, op->fast, epi, op->stream, dot_ctas));
    } else {
        // the generic kernels have no folded dot: the caller falls back (dot_ctas = 0)
        if (epi.npeers) return fail(BTG_EARG, "internal: fused grid reduce needs the fast C2R");
        btg::C2REpilogue e = epi;
        e.dot_v = nullptr;
        e.dot_out = nullptr;
        BTG_CUDA(btg::launch_c2r(in, (long long)fs, 1, out, (long long)op->nt, (int)channels,
                                 (int)op->nt, op->plan, op->fft_batch, e, op->stream, op->gscratch));
    }
    op->counters.launches++;
    op->counters.inverse_fft.ops += fft_ops(channels, op->nt);
    op->counters.inverse_fft.bytes += 16.0 * op->nf * channels + 8.0 * channels * op->nt;
    // unpad fused into the C2R stores (block_operator.cpp:105-106 op model)
    op->counters.unpad.ops += 2.0 * channels * op->nt;
    return BTG_OK;
}

// int8 slices of F-hat for the tensor-core multi-RHS path, built on first use.
btg_status ensure_oz(btg_op op, size_t nrhs) {
    const int nf = (int)op->nf, nd = (int)op->nd, nm = (int)op->nm;
    if (!op->oz_A) {
        const size_t bytes = btg::oz_operator_bytes(nf, nd, nm);
        cudaError_t e = cudaMalloc(&op->oz_A, bytes);
        if (e == cudaSuccess) e = cudaMalloc(&op->oz_mA, btg::oz_operator_scales(nf, nm) * sizeof(unsigned long long));
        if (e != cudaSuccess) return fail(BTG_ENOMEM, "int8 F-hat slices (%zu bytes): %s", bytes, cudaGetErrorString(e));
        op->oz_valid = false;
    }
    if (!op->oz_valid) {
        BTG_CUDA(btg::oz_quantize_operator(static_cast<const double2*>(op->F), nf, nd, nm, op->oz_A, op->oz_mA,
                                           op->stream));
        op->oz_valid = true;
    }
    const size_t need = btg::oz_vector_scales(nf, (int)std::min<size_t>(nrhs, 32), (int)std::max(op->nd, op->nm));
    if (need > op->oz_mB_cap) {
        cudaFree(op->oz_mB);
        op->oz_mB = nullptr;
        BTG_CUDA(cudaMalloc(&op->oz_mB, need * sizeof(int)));
        op->oz_mB_cap = need;
    }
    const size_t bneed = btg::oz_presliced_bytes((int)op->nf, (int)op->nd);
    if (bneed > op->oz_B_cap) {
        cudaFree(op->oz_B);
        op->oz_B = nullptr;
        cudaError_t e = cudaMalloc(&op->oz_B, bneed);
        if (e != cudaSuccess) return fail(BTG_ENOMEM, "int8 d-hat tiles (%zu bytes): %s", bneed, cudaGetErrorString(e));
        op->oz_B_cap = bneed;
    }
    return BTG_OK;
}

btg_status run_apply(btg_op op, bool adjoint, const double2* in, double2* out, size_t nrhs,
                     const int16_t* vexp = nullptr, int vexp_cpb = 1, bool blocked = false) {
    StageClock clk(op, &op->counters.apply);
    const size_t nin = adjoint ? op->nd : op->nm;
    const size_t nout = adjoint ? op->nm : op->nd;
    const int nf = (int)op->nf, nd = (int)op->nd, nm = (int)op->nm;
    cudaError_t e;
    if (nrhs > 1 && op->tensor_i8) {
        // tcgen05 int8 tensor cores, exact-integer Ozaki splitting (btg_ozaki.cu)
        if (op->precision != BTG_F64) return fail(BTG_EARG, "internal: batched apply needs FP64 F-hat");
        BTG_TRY(ensure_oz(op, nrhs));
        e = btg::oz_apply(adjoint, op->oz_A, op->oz_mA, in, out, nf, nd, nm, (int)nrhs, op->oz_mB, op->oz_B,
                          op->stream, vexp, vexp_cpb);
    } else if (nrhs > 1) {
        // ZGEMM on the FP64 tensor cores (btg_zgemm.cu); FP64 F-hat only.
        if (op->precision != BTG_F64) return fail(BTG_EARG, "internal: batched apply needs FP64 F-hat");
        const double2* F = static_cast<const double2*>(op->F);
        if (blocked)  // the N_m side (X forward, G adjoint) channel-blocked
            e = adjoint ? btg::launch_zgemm3m_adj_ws(F, in, out, nf, nd, nm, (int)nrhs, 0, nm, op->stream, true)
                        : btg::launch_zgemm3m_fwd_ws(F, in, out, nf, nd, nm, (int)nrhs, 0, nm, false, op->stream,
                                                     true);
        else
            e = adjoint ? btg::launch_zgemm_adj(F, in, out, nf, nd, nm, (int)nrhs, op->stream)
                        : btg::launch_zgemm_fwd(F, in, out, nf, nd, nm, (int)nrhs, op->stream);
    } else if (op->precision == BTG_F64 && !op->legacy_gemv) {
        // persistent TMA-staged stream (btg_gemv_tma.cu)
        const double2* F = static_cast<const double2*>(op->F);
        e = adjoint ? btg::launch_gemv_adj_tma(F, in, out, nf, nd, nm, op->stream)
                    : btg::launch_gemv_fwd_tma(F, in, out, nf, nd, nm, op->stream);
    } else if (op->precision == BTG_F64) {
        const double2* F = static_cast<const double2*>(op->F);
        e = adjoint ? btg::launch_gemv_adj(F, in, out, nf, nd, nm, op->stream)
                    : btg::launch_gemv_fwd(F, in, out, nf, nd, nm, op->stream);
    } else {
        const float2* F = static_cast<const float2*>(op->F);
        e = adjoint ? btg::launch_gemv_adj(F, in, out, nf, nd, nm, op->stream)
                    : btg::launch_gemv_fwd(F, in, out, nf, nd, nm, op->stream);
    }
    BTG_CUDA(e);
    op->counters.launches++;
    op->counters.apply.ops += 8.0 * op->nd * op->nm * op->nf * nrhs;
    op->counters.apply.bytes +=
        (double)op->F_elem * op->nf * op->nd * op->nm + 16.0 * op->nf * (nin + nout) * nrhs;
    return BTG_OK;
}

// Multi-RHS device pipeline with the N_m-side spectrum channel-blocked
// (btg::kBlockedFs): FP64 3M ZGEMM on its TMA kernels, a fast plan with
// kSpecBlock channels per CTA in both directions, aligned vectors.
// BTG_SPEC_BLOCKED=0 keeps the frequency-major layout (A/B).
bool mrhs_blocked(btg_op op, const double* in, const double* out, const btg::C2REpilogue& epi) {
    const char* v = std::getenv("BTG_SPEC_BLOCKED");
    if (v && *v == '0') return false;
    return op->precision == BTG_F64 && !op->no_dmma && !op->tensor_i8 && op->fast_ok &&
           btg::spec_blocked_ok((int)op->nt) && btg::zgemm_ws_active() && btg::zgemm_tma_ok((int)op->nm) &&
           aligned16(in) && aligned16(out) && aligned16(op->wa) && aligned16(op->wb) &&
           (!epi.v || aligned16(epi.v)) && (epi.gamma_mode != 2 || aligned16(epi.gamma));
}

// One direction (forward or adjoint) for nrhs right-hand sides, device pointers.
// FP64: all right-hand sides go through one R2C, one ZGEMM (DMMA) and one C2R;
// FP32 F-hat: one GEMV stream per right-hand side.
btg_status pipeline(btg_op op, bool adjoint, const double* in, double* out, size_t nrhs,
                    const btg::C2REpilogue& epi, int* dot_ctas = nullptr) {
    const size_t cin = adjoint ? op->nd : op->nm;
    const size_t cout = adjoint ? op->nm : op->nd;
    if (nrhs > 1 && op->precision == BTG_F64 && !op->no_dmma) {
        BTG_TRY(ensure_spectral(op, nrhs));
        // int8 engine, forward: the x-hat block maxima come out of the R2C
        const int cpb = btg::fast_r2c_cpb((int)op->nt);
        if (op->tensor_i8 && !adjoint && nrhs <= 32 && op->fast_ok && cpb > 0 && cin % cpb == 0 &&
            aligned16(in) && aligned16(op->wa) && !std::getenv("BTG_OZ_SCALE_PASS")) {
            btg::R2CBlockMax bm;
            bm.nf = (int)op->nf;
            const size_t n = (nrhs * cin / cpb) * op->nf;
            BTG_TRY(grow(op->oz_vexp, op->oz_vexp_cap, n));
            bm.pexp = op->oz_vexp;
            BTG_TRY(run_r2c_vec(op, in, nrhs * cin, op->wa, 0, &bm));
            BTG_TRY(run_apply(op, adjoint, op->wa, op->wb, nrhs, op->oz_vexp, cpb));
            BTG_TRY(run_c2r_vec(op, op->wb, nrhs * cout, out, epi));
            return BTG_OK;
        }
        // The N_m-side spectrum (x-hat forward, g-hat adjoint) in the channel-blocked
        // layout: the big R2C writes / C2R reads stream contiguous blocks
        const bool blk = mrhs_blocked(op, in, out, epi);
        BTG_TRY(run_r2c_vec(op, in, nrhs * cin, op->wa, 0, nullptr, blk && !adjoint));
        BTG_TRY(run_apply(op, adjoint, op->wa, op->wb, nrhs, nullptr, 1, blk));
        BTG_TRY(run_c2r_vec(op, op->wb, nrhs * cout, out, epi, 0, nullptr, blk && adjoint));
        return BTG_OK;
    }
    BTG_TRY(ensure_spectral(op, 1));
    for (size_t r = 0; r < nrhs; ++r) {
        BTG_TRY(run_r2c_vec(op, in + r * cin * op->nt, cin, op->wa));
        BTG_TRY(run_apply(op, adjoint, op->wa, op->wb, 1));
        btg::C2REpilogue e = epi;
        if (e.v) e.v = epi.v + r * cout * op->nt;
        BTG_TRY(run_c2r_vec(op, op->wb, cout, out + r * cout * op->nt, e, 0, nrhs == 1 ? dot_ctas : nullptr));
    }
    return BTG_OK;
}

btg_status check_len(const char* what, size_t got, size_t want_dim, size_t nt, size_t nrhs,
                     size_t op_dim) {
    if (got != want_dim * nt * nrhs)
        return fail(BTG_EDIM, "%s: input has %zu values but operator expects %zu x %zu (x %zu rhs)",
                    what, got, op_dim, nt, nrhs);
    return BTG_OK;
}

btg_status finish_host(btg_op op, double* out_host, const double* out_dev, size_t n, unsigned flags) {
    if (!(flags & BTG_DEVICE_PTRS)) {
        BTG_CUDA(cudaMemcpyAsync(out_host, out_dev, n * sizeof(double), cudaMemcpyDeviceToHost, op->stream));
        BTG_CUDA(cudaStreamSynchronize(op->stream));
    } else {
        BTG_CUDA(cudaGetLastError());
    }
    return BTG_OK;
}

// Device-side copy of a host epilogue operand (gamma or reg_v).
btg_status stage_small(btg_op op, const double* src, size_t n, double*& buf, size_t& cap, const double** dev) {
    BTG_TRY(grow(buf, cap, n));
    BTG_CUDA(cudaMemcpyAsync(buf, src, n * sizeof(double), cudaMemcpyHostToDevice, op->stream));
    *dev = buf;
    return BTG_OK;
}

// ---------------------------------------------------------------------------
// Host-pointer calls: overlap the PCIe transfers of the long (N_m x N_t)
// vector with the HBM-bound Fourier-space step. The N_m channels are cut into
// column chunks; chunk c's H2D copy (copy stream) overlaps chunk c-1's R2C +
// forward GEMV partial (compute stream), and on the way out chunk c's D2H
// overlaps chunk c+1's adjoint GEMV + C2R. Forward partial products are added
// chunk by chunk in a fixed order (deterministic).
// ---------------------------------------------------------------------------
constexpr size_t kHostChunks = 16;

bool host_pipelined(btg_op op, size_t nrhs) {
    static const bool off = std::getenv("BTG_NO_HOST_PIPELINE") != nullptr;
    return !off && nrhs == 1 && op->legacy_gemv && op->nm >= 4096;
}

// Column chunks (multiples of 256 columns): a geometric ramp x1.5 per chunk from
// ~512 columns, scaled so the series ends exactly at N_m (no small leftover
// chunk: a GEMV over a few thousand columns runs at ~6 TB/s, not ~7.2). The first
// H2D (last D2H) is the only transfer left exposed; x1.5 keeps each next chunk's
// PCIe copy (8 N_t B per column at ~55 GB/s) shorter than the current chunk's
// GEMV (16 N_d (N_t+1) B per column at ~7 TB/s), so the GEMVs never wait — a x2
// ramp did (CUPTI timeline, profiles/tools/host_timeline.py; 33.5 -> 33.2 ms per
// configs[1] e2e step). At most kHostChunks chunks (wider N_m: the ramp, then
// equal chunks). BTG_HOST_RAMP (percent) is a tuning knob.
//
// When the copies are not the faster side (FP32 F-hat, small N_d: a chunk GEMV
// costs about what its copy does or less) the copy stream is the critical path
// and a ramp only adds small, inefficient GEMVs: equal chunks instead (FP32
// configs[1]: a mirrored ramp measured F 6.43 ms, the x2 ramp 5.85).
std::vector<std::pair<size_t, size_t>> mrhs_chunks(size_t nm);

std::vector<std::pair<size_t, size_t>> chunk_plan(btg_op op, bool ramp_first) {
    static const double growth = [] {
        const char* s = std::getenv("BTG_HOST_RAMP");
        return s ? std::max(1.1, std::strtod(s, nullptr) / 100.0) : 1.5;
    }();
    // chunk GEMV ~6.5 TB/s (FP32 measured ~6 TB/s), PCIe ~55 GB/s
    const double gemv_col = (double)op->F_elem * op->nd * op->nf / 6.5e12;
    const double pcie_col = 8.0 * op->nt / 55.0e9;
    if (gemv_col < 1.2 * pcie_col) return mrhs_chunks(op->nm);
    const size_t nm = op->nm;
    std::vector<double> geo;
    double sum = 0.0;
    for (double w = 512.0; sum < (double)nm && geo.size() < kHostChunks; w *= growth) {
        geo.push_back(w);
        sum += w;
    }
    std::vector<size_t> sizes;
    size_t used = 0;
    if (sum >= (double)nm) {
        const double scale = (double)nm / sum;
        for (size_t k = 0; k + 1 < geo.size(); ++k) {
            const size_t w = std::max<size_t>(256, (size_t)std::llround(geo[k] * scale / 256.0) * 256);
            if (used + w >= nm) break;
            sizes.push_back(w);
            used += w;
        }
        sizes.push_back(nm - used);
    } else {  // the ramp's widest chunk, repeated; the remainder folds into the last
        for (size_t k = 0; k + 1 < kHostChunks / 2 && used < nm; ++k) {
            sizes.push_back(std::min<size_t>((size_t)geo[k] / 256 * 256, nm - used));
            used += sizes.back();
        }
        const size_t n_eq = kHostChunks - sizes.size();
        const size_t w = ((nm - used) / n_eq + 255) / 256 * 256;
        while (used < nm) {
            sizes.push_back(std::min(w, nm - used));
            used += sizes.back();
        }
    }
    if (!ramp_first) std::reverse(sizes.begin(), sizes.end());
    std::vector<std::pair<size_t, size_t>> plan;
    size_t j0 = 0;
    for (size_t w : sizes) {
        plan.emplace_back(j0, w);
        j0 += w;
    }
    return plan;
}

btg_status ensure_copy_stream(btg_op op) {
    if (!op->copy_stream) BTG_CUDA(cudaStreamCreateWithFlags(&op->copy_stream, cudaStreamNonBlocking));
    if (!op->fft_stream) BTG_CUDA(cudaStreamCreateWithFlags(&op->fft_stream, cudaStreamNonBlocking));
    for (size_t c = 0; c <= kHostChunks; ++c) {
        if (!op->ev[c]) BTG_CUDA(cudaEventCreateWithFlags(&op->ev[c], cudaEventDisableTiming));
        if (!op->ev_h2d[c]) BTG_CUDA(cudaEventCreateWithFlags(&op->ev_h2d[c], cudaEventDisableTiming));
    }
    return BTG_OK;
}

btg_status gemv_range(btg_op op, bool adjoint, const double2* in, double2* out, size_t j0, size_t nc, bool acc) {
    const int nf = (int)op->nf, nd = (int)op->nd, nm = (int)op->nm;
    cudaError_t e;
    if (op->precision == BTG_F64) {
        const double2* F = static_cast<const double2*>(op->F);
        e = adjoint ? btg::launch_gemv_adj_range(F, in, out, nf, nd, nm, (int)j0, (int)nc, op->stream)
                    : btg::launch_gemv_fwd_range(F, in, out, nf, nd, nm, (int)j0, (int)nc, acc, op->stream);
    } else {
        const float2* F = static_cast<const float2*>(op->F);
        e = adjoint ? btg::launch_gemv_adj_range(F, in, out, nf, nd, nm, (int)j0, (int)nc, op->stream)
                    : btg::launch_gemv_fwd_range(F, in, out, nf, nd, nm, (int)j0, (int)nc, acc, op->stream);
    }
    BTG_CUDA(e);
    op->counters.launches++;
    return BTG_OK;
}

void count_apply(btg_op op) {
    op->counters.apply.ops += 8.0 * op->nd * op->nm * op->nf;
    op->counters.apply.bytes += (double)op->F_elem * op->nf * op->nd * op->nm + 16.0 * op->nf * (op->nm + op->nd);
}

// m (host, N_m x N_t) -> d-hat in op->wb; the device copy of m stays in op->hin.
btg_status host_forward_stage(btg_op op, const double* m_host) {
    BTG_TRY(ensure_spectral(op, 1));
    BTG_TRY(ensure_copy_stream(op));
    const size_t nt = op->nt;
    const auto plan = chunk_plan(op, true);
    BTG_CUDA(cudaEventRecord(op->ev[kHostChunks], op->stream));  // hin free of earlier readers
    BTG_CUDA(cudaStreamWaitEvent(op->copy_stream, op->ev[kHostChunks], 0));
    StageClock clk(op, &op->counters.apply);
    for (size_t c = 0; c < plan.size(); ++c) {
        const auto [j0, nc] = plan[c];
        BTG_CUDA(cudaMemcpyAsync(op->hin + j0 * nt, m_host + j0 * nt, nc * nt * sizeof(double),
                                 cudaMemcpyHostToDevice, op->copy_stream));
        BTG_CUDA(cudaEventRecord(op->ev_h2d[c], op->copy_stream));
        // the chunk's R2C runs on its own stream behind its H2D, so it overlaps the
        // previous chunk's GEMV instead of sitting between GEMVs on the compute
        // stream, and never holds up the next H2D while it waits for SMs
        BTG_CUDA(cudaStreamWaitEvent(op->fft_stream, op->ev_h2d[c], 0));
        {
            cudaStream_t main = op->stream;
            op->stream = op->fft_stream;
            const btg_status st = run_r2c_vec(op, op->hin + j0 * nt, nc, op->wa + j0, op->nm);
            op->stream = main;
            BTG_TRY(st);
        }
        BTG_CUDA(cudaEventRecord(op->ev[c], op->fft_stream));
        BTG_CUDA(cudaStreamWaitEvent(op->stream, op->ev[c], 0));
        BTG_TRY(gemv_range(op, false, op->wa, op->wb, j0, nc, c > 0));
    }
    count_apply(op);
    return BTG_OK;
}

// The C2R epilogue of a column chunk [j0, j0 + nc): its channel index restarts at 0,
// so the per-channel operands (Gamma^-1, the alpha R v vector) are offset to j0.
btg::C2REpilogue chunk_epilogue(const btg::C2REpilogue& epi, size_t j0, size_t nt, size_t v_off) {
    btg::C2REpilogue e = epi;
    if (e.v) e.v = epi.v + v_off;
    if (e.gamma) e.gamma = epi.gamma + (e.gamma_mode == BTG_GAMMA_PER_SENSOR ? j0 : j0 * nt);
    return e;
}

// d-hat spectrum in op->wa -> m (host) through chunked adjoint GEMV + C2R + D2H.
btg_status host_adjoint_stage(btg_op op, double* m_host, const btg::C2REpilogue& epi) {
    BTG_TRY(ensure_copy_stream(op));
    const size_t nt = op->nt;
    const auto plan = chunk_plan(op, false);
    {
        StageClock clk(op, &op->counters.apply);
        for (size_t c = 0; c < plan.size(); ++c) {
            const auto [j0, nc] = plan[c];
            BTG_TRY(gemv_range(op, true, op->wa, op->wb, j0, nc, false));
            BTG_TRY(run_c2r_vec(op, op->wb + j0, nc, op->hout + j0 * nt, chunk_epilogue(epi, j0, nt, j0 * nt),
                                op->nm));
            BTG_CUDA(cudaEventRecord(op->ev[c], op->stream));
        }
    }
    count_apply(op);
    for (size_t c = 0; c < plan.size(); ++c) {
        const auto [j0, nc] = plan[c];
        BTG_CUDA(cudaStreamWaitEvent(op->copy_stream, op->ev[c], 0));
        BTG_CUDA(cudaMemcpyAsync(m_host + j0 * nt, op->hout + j0 * nt, nc * nt * sizeof(double),
                                 cudaMemcpyDeviceToHost, op->copy_stream));
    }
    BTG_CUDA(cudaStreamSynchronize(op->copy_stream));
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    return BTG_OK;
}

// ---------------------------------------------------------------------------
// Multi-RHS host calls (FP64 F-hat, 3M ZGEMM engine). These are PCIe-bound: a
// column moves nrhs x 8 N_t bytes over PCIe (~4.7 us at 32 RHS, N_t=1024) but
// costs ~1 us of ZGEMM, so the ZGEMM (column chunks; the forward's K = j
// partials accumulate in chunk order, deterministic) hides under the copies and
// only the last (first) chunk's compute stays exposed: equal chunks, kHostChunks
// of them. Each chunk moves as one 2-D copy (nrhs rows of nc x N_t values).
// ---------------------------------------------------------------------------
bool host_pipelined_mrhs(btg_op op, size_t nrhs) {
    static const bool off = std::getenv("BTG_NO_HOST_PIPELINE") != nullptr;
    return !off && nrhs > 1 && op->precision == BTG_F64 && !op->no_dmma && !op->tensor_i8 && btg::zgemm_3m() &&
           op->nm >= 4096;
}

std::vector<std::pair<size_t, size_t>> mrhs_chunks(size_t nm) {
    const size_t w = std::max<size_t>(256, (nm / kHostChunks + 255) / 256 * 256);
    std::vector<std::pair<size_t, size_t>> plan;
    for (size_t j0 = 0; j0 < nm; j0 += w) plan.emplace_back(j0, std::min(w, nm - j0));
    return plan;
}

btg_status zgemm_range(btg_op op, bool adjoint, size_t nrhs, size_t j0, size_t nc, bool acc) {
    const double2* F = static_cast<const double2*>(op->F);
    const int nf = (int)op->nf, nd = (int)op->nd, nm = (int)op->nm;
    BTG_CUDA(adjoint ? btg::launch_zgemm_adj_range(F, op->wa, op->wb, nf, nd, nm, (int)nrhs, (int)j0, (int)nc,
                                                   op->stream)
                     : btg::launch_zgemm_fwd_range(F, op->wa, op->wb, nf, nd, nm, (int)nrhs, (int)j0, (int)nc, acc,
                                                   op->stream));
    op->counters.launches++;
    return BTG_OK;
}

void count_apply_mrhs(btg_op op, size_t nrhs) {
    op->counters.apply.ops += 8.0 * op->nd * op->nm * op->nf * nrhs;
    op->counters.apply.bytes += (double)op->F_elem * op->nf * op->nd * op->nm + 16.0 * op->nf * (op->nm + op->nd) * nrhs;
}

// m (host, nrhs x N_m x N_t) -> d-hat (nrhs stacked) in op->wb.
btg_status host_forward_stage_mrhs(btg_op op, const double* m_host, size_t nrhs) {
    BTG_TRY(ensure_spectral(op, nrhs));
    BTG_TRY(ensure_copy_stream(op));
    const size_t nt = op->nt, nm = op->nm, pitch = nm * nt * sizeof(double);
    BTG_CUDA(cudaEventRecord(op->ev[kHostChunks], op->stream));  // hin free of earlier readers
    BTG_CUDA(cudaStreamWaitEvent(op->copy_stream, op->ev[kHostChunks], 0));
    const auto plan = mrhs_chunks(nm);
    StageClock clk(op, &op->counters.apply);
    for (size_t c = 0; c < plan.size(); ++c) {
        const auto [j0, nc] = plan[c];
        BTG_CUDA(cudaMemcpy2DAsync(op->hin + j0 * nt, pitch, m_host + j0 * nt, pitch, nc * nt * sizeof(double), nrhs,
                                   cudaMemcpyHostToDevice, op->copy_stream));
        BTG_CUDA(cudaEventRecord(op->ev_h2d[c], op->copy_stream));
        BTG_CUDA(cudaStreamWaitEvent(op->fft_stream, op->ev_h2d[c], 0));
        cudaStream_t main = op->stream;
        op->stream = op->fft_stream;
        btg_status st = BTG_OK;
        for (size_t r = 0; r < nrhs && st == BTG_OK; ++r)
            st = run_r2c_vec(op, op->hin + (r * nm + j0) * nt, nc, op->wa + r * nm + j0, nrhs * nm);
        op->stream = main;
        BTG_TRY(st);
        BTG_CUDA(cudaEventRecord(op->ev[c], op->fft_stream));
        BTG_CUDA(cudaStreamWaitEvent(op->stream, op->ev[c], 0));
        BTG_TRY(zgemm_range(op, false, nrhs, j0, nc, c > 0));
    }
    count_apply_mrhs(op, nrhs);
    return BTG_OK;
}

// d-hat spectra (nrhs stacked) in op->wa -> m (host) through chunked adjoint
// ZGEMM + C2R + 2-D D2H.
btg_status host_adjoint_stage_mrhs(btg_op op, double* m_host, size_t nrhs, const btg::C2REpilogue& epi) {
    BTG_TRY(ensure_copy_stream(op));
    const size_t nt = op->nt, nm = op->nm, pitch = nm * nt * sizeof(double);
    const auto plan = mrhs_chunks(nm);
    {
        StageClock clk(op, &op->counters.apply);
        for (size_t c = 0; c < plan.size(); ++c) {
            const auto [j0, nc] = plan[c];
            BTG_TRY(zgemm_range(op, true, nrhs, j0, nc, false));
            for (size_t r = 0; r < nrhs; ++r)
                BTG_TRY(run_c2r_vec(op, op->wb + r * nm + j0, nc, op->hout + (r * nm + j0) * nt,
                                    chunk_epilogue(epi, j0, nt, (r * nm + j0) * nt), nrhs * nm));
            BTG_CUDA(cudaEventRecord(op->ev[c], op->stream));
        }
    }
    count_apply_mrhs(op, nrhs);
    for (size_t c = 0; c < plan.size(); ++c) {
        const auto [j0, nc] = plan[c];
        BTG_CUDA(cudaStreamWaitEvent(op->copy_stream, op->ev[c], 0));
        BTG_CUDA(cudaMemcpy2DAsync(m_host + j0 * nt, pitch, op->hout + j0 * nt, pitch, nc * nt * sizeof(double), nrhs,
                                   cudaMemcpyDeviceToHost, op->copy_stream));
    }
    BTG_CUDA(cudaStreamSynchronize(op->copy_stream));
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    return BTG_OK;
}

btg_status apply_dir(btg_op op, bool adjoint, const double* in, size_t in_len, double* out,
                     size_t out_len, size_t nrhs, const btg_epilogue* ex, unsigned flags,
                     const double* const* peers = nullptr, int npeers = 0) {
    BTG_TRY(check_ready(op));
    if (nrhs == 0) return fail(BTG_EARG, "nrhs must be >= 1");
    if (!in || !out) return fail(BTG_EARG, "null vector pointer");
    const char* what = adjoint ? "apply_adjoint" : "apply_forward";
    const size_t din = adjoint ? op->nd : op->nm;
    const size_t dout = adjoint ? op->nm : op->nd;
    BTG_TRY(check_len(what, in_len, din, op->nt, nrhs, din));
    BTG_TRY(check_len(what, out_len, dout, op->nt, nrhs, dout));
    btg::C2REpilogue epi{};
    if (ex) {
        if (ex->gamma_kind < BTG_GAMMA_NONE || ex->gamma_kind > BTG_GAMMA_PER_SAMPLE)
            return fail(BTG_EARG, "unknown gamma kind %d", ex->gamma_kind);
        if (ex->gamma_kind != BTG_GAMMA_NONE && !ex->gamma_inv) return fail(BTG_EARG, "gamma_inv is null");
        if (ex->reg_kind != BTG_REG_IDENTITY && ex->reg_kind != BTG_REG_TEMPORAL_LAPLACIAN)
            return fail(BTG_EARG, "unknown regularization kind %d", ex->reg_kind);
        if (ex->alpha != 0.0 && !ex->reg_v) return fail(BTG_EARG, "reg_v is null with alpha != 0");
    }
    DeviceGuard g(op->device);
    const double* din_p = in;
    double* dout_p = out;
    const bool host = !(flags & BTG_DEVICE_PTRS);
    const bool chunked = host && host_pipelined(op, nrhs);
    const bool mchunked = host && host_pipelined_mrhs(op, nrhs);
    if (host) {
        BTG_TRY(host_buffers(op, in_len, out_len));
        if (!((chunked || mchunked) && !adjoint))  // the chunked forward streams its input itself
            BTG_CUDA(cudaMemcpyAsync(op->hin, in, in_len * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        din_p = op->hin;
        dout_p = op->hout;
    }
    if (ex && ex->gamma_kind != BTG_GAMMA_NONE) {
        epi.gamma_mode = ex->gamma_kind;
        epi.gamma_dim = (int)dout;
        epi.gamma = ex->gamma_inv;
        if (!(flags & BTG_DEVICE_PTRS)) {
            const size_t glen = ex->gamma_kind == BTG_GAMMA_PER_SENSOR ? dout : dout * op->nt;
            BTG_TRY(stage_small(op, ex->gamma_inv, glen, op->gam, op->gcap, &epi.gamma));
        }
    }
    if (ex && ex->alpha != 0.0) {
        epi.alpha = ex->alpha;
        epi.reg_kind = ex->reg_kind;
        epi.v = ex->reg_v;
        if (!(flags & BTG_DEVICE_PTRS)) {
            BTG_TRY(stage_small(op, ex->reg_v, out_len, op->vcopy, op->vcap, &epi.v));
        } else if (epi.v == out) {
            BTG_TRY(grow(op->vcopy, op->vcap, out_len));
            BTG_CUDA(cudaMemcpyAsync(op->vcopy, epi.v, out_len * sizeof(double), cudaMemcpyDeviceToDevice,
                                     op->stream));
            epi.v = op->vcopy;
        }
    }
    if (chunked && !adjoint) {
        BTG_TRY(host_forward_stage(op, in));
        BTG_TRY(run_c2r_vec(op, op->wb, op->nd, dout_p, epi));
        return finish_host(op, out, dout_p, out_len, flags);
    }
    if (chunked && adjoint) {
        BTG_TRY(ensure_spectral(op, 1));
        BTG_TRY(run_r2c_vec(op, din_p, op->nd, op->wa));
        return host_adjoint_stage(op, out, epi);
    }
    if (mchunked && !adjoint) {
        BTG_TRY(host_forward_stage_mrhs(op, in, nrhs));
        BTG_TRY(run_c2r_vec(op, op->wb, nrhs * op->nd, dout_p, epi));
        return finish_host(op, out, dout_p, out_len, flags);
    }
    if (mchunked && adjoint) {
        BTG_TRY(ensure_spectral(op, nrhs));
        BTG_TRY(run_r2c_vec(op, din_p, nrhs * op->nd, op->wa));
        return host_adjoint_stage_mrhs(op, out, nrhs, epi);
    }
    epi.peers = peers;
    epi.npeers = npeers;
    BTG_TRY(pipeline(op, adjoint, din_p, dout_p, nrhs, epi));
    return finish_host(op, out, dout_p, out_len, flags);
}

// Device-pointer Hessian calls replay a captured graph of the whole
// F -> C2R(Gamma^-1) -> R2C -> F* -> C2R(alpha R v) chain (6+ launches, one
// graph launch) when the pointers, epilogues and engine match the previous
// call; anything else re-captures. The workspace is grown before the capture,
// so a replay never sees a reallocated buffer (the key holds those pointers).
void add_counters(btg_counters& dst, const btg_counters& d) {
    auto add = [](btg_stage_counters& a, const btg_stage_counters& b) {
        a.ops += b.ops;
        a.bytes += b.bytes;
    };
    add(dst.pad, d.pad);
    add(dst.forward_fft, d.forward_fft);
    add(dst.reorder_in, d.reorder_in);
    add(dst.apply, d.apply);
    add(dst.reorder_out, d.reorder_out);
    add(dst.inverse_fft, d.inverse_fft);
    add(dst.unpad, d.unpad);
    dst.launches += d.launches;
}

btg_status hessian_graph(btg_op op, const double* vd, double* hvd, size_t nrhs, const btg::C2REpilogue& e1,
                         const btg::C2REpilogue& e2) {
    // grow everything the chain touches before keying / capturing
    BTG_TRY(grow(op->wt, op->wtcap, op->nd * op->nt * nrhs));
    BTG_TRY(ensure_spectral(op, (nrhs > 1 && op->precision == BTG_F64 && !op->no_dmma) ? nrhs : 1));
    if (op->tensor_i8 && nrhs > 1) {
        // the int8 engine allocates lazily on first use: run it eagerly once
        BTG_TRY(pipeline(op, false, vd, op->wt, nrhs, e1));
        return pipeline(op, true, op->wt, hvd, nrhs, e2);
    }
    const HessKey key{vd, hvd, nrhs, e1.gamma, e1.gamma_mode, e2.alpha, e2.reg_kind, op->wa, op->wb, op->wt,
                      op->F, op->tensor_i8, op->no_dmma, op->legacy_gemv};
    HessGraph& hg = op->hess_graph;
    if (!hg.exec || !(hg.key == key)) {
        if (hg.exec) cudaGraphExecDestroy(hg.exec);
        hg.exec = nullptr;
        if (!op->capture_stream) BTG_CUDA(cudaStreamCreateWithFlags(&op->capture_stream, cudaStreamNonBlocking));
        const cudaStream_t run_stream = op->stream;
        const btg_counters c0 = op->counters;
        op->counters = btg_counters{};
        BTG_CUDA(cudaStreamBeginCapture(op->capture_stream, cudaStreamCaptureModeRelaxed));
        op->stream = op->capture_stream;
        btg_status s = pipeline(op, false, vd, op->wt, nrhs, e1);
        if (s == BTG_OK) s = pipeline(op, true, op->wt, hvd, nrhs, e2);
        op->stream = run_stream;
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(op->capture_stream, &g);
        hg.delta = op->counters;
        op->counters = c0;
        if (s != BTG_OK) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return s;
        }
        BTG_CUDA(ec);
        const cudaError_t ei = cudaGraphInstantiate(&hg.exec, g, 0);
        cudaGraphDestroy(g);
        BTG_CUDA(ei);
        hg.key = key;
    }
    BTG_CUDA(cudaGraphLaunch(hg.exec, op->stream));
    add_counters(op->counters, hg.delta);
    return BTG_OK;
}

}  // namespace

extern "C" {

const char* btg_last_error(void) { return g_err.c_str(); }
int btg_abi_version(void) { return BTG_ABI_VERSION; }

btg_status btg_create(size_t nd, size_t nm, size_t nt, int precision, int device, btg_op* out) {
    if (!out) return fail(BTG_EARG, "null output handle");
    *out = nullptr;
    if (nd == 0 || nm == 0 || nt == 0)
        return fail(BTG_EDIM, "compact operator: all dimensions must be positive");
    if (precision != BTG_F64 && precision != BTG_F32)
        return fail(BTG_EARG, "precision must be 64 or 32 (got %d)", precision);
    if (nt > (1u << 30) || nd > (1u << 30) || nm > (1u << 30))
        return fail(BTG_EDIM, "dimension exceeds 2^30");
    int ndev = 0;
    BTG_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(BTG_EARG, "device %d not present (%d devices)", device, ndev);

    const std::vector<int> fac = factorize((int)nt);
    if ((int)fac.size() > btg::kMaxFactors) return fail(BTG_EARG, "N_t=%zu has too many factors", nt);
    const int batch_vec = btg::fft_batch((int)nt, kFftSmemTarget, 4);
    // Horizons beyond the shared-memory two-buffer transform (N_t > ~6400) run
    // the generic kernels on a bounded global scratch; lengths with a
    // compile-time plan (8192, 10000) still take the register path for vectors.
    const bool smem_fits = btg::fft_batch((int)nt, kFftSmemBudget, 1) >= 1;

    DeviceGuard g(device);
    btg_op op = new (std::nothrow) btg_op_s();
    if (!op) return fail(BTG_ENOMEM, "host allocation failed");
    op->device = device;
    op->precision = precision;
    op->nd = nd;
    op->nm = nm;
    op->nt = nt;
    op->nf = nt + 1;
    op->F_elem = precision == BTG_F64 ? sizeof(double2) : sizeof(float2);
    op->fft_batch = std::max(1, batch_vec);
    op->fft_batch_setup = std::max(1, std::min(btg::fft_batch((int)nt, kFftSmemBudget, 8), 8));

    auto cleanup_fail = [&](btg_status s) {
        btg_destroy(op);
        return s;
    };
    cudaError_t e = cudaStreamCreateWithFlags(&op->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cleanup_fail(fail(BTG_ECUDA, "stream: %s", cudaGetErrorString(e)));
    op->stream = op->own_stream;

    // twiddle tables
    std::vector<double2> tw(nt), post(nt + 1);
    for (size_t k = 0; k < nt; ++k) tw[k] = root((long long)k, (long long)nt);
    for (size_t k = 0; k <= nt; ++k) post[k] = root((long long)k, 2 * (long long)nt);
    e = cudaMalloc(&op->d_tw, nt * sizeof(double2));
    if (e == cudaSuccess) e = cudaMalloc(&op->d_post, (nt + 1) * sizeof(double2));
    if (e == cudaSuccess) e = cudaMemcpy(op->d_tw, tw.data(), nt * sizeof(double2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(op->d_post, post.data(), (nt + 1) * sizeof(double2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cleanup_fail(fail(BTG_ECUDA, "twiddles: %s", cudaGetErrorString(e)));
    if (btg::fast_fft_supported((int)nt) && !std::getenv("BTG_DISABLE_FAST_FFT")) {
        const int hi = btg::fast_fft_hi_count((int)nt);
        std::vector<double2> t(32 + hi + 32 + hi + 1);
        for (int i = 0; i < 32; ++i) t[i] = root(i, (long long)nt);
        for (int h = 0; h < hi; ++h) t[32 + h] = root(32LL * h, (long long)nt);
        for (int i = 0; i < 32; ++i) t[32 + hi + i] = root(i, 2 * (long long)nt);
        for (int h = 0; h <= hi; ++h) t[64 + hi + h] = root(32LL * h, 2 * (long long)nt);
        e = cudaMalloc(&op->d_fast, t.size() * sizeof(double2));
        if (e == cudaSuccess)
            e = cudaMemcpy(op->d_fast, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cleanup_fail(fail(BTG_ECUDA, "fast twiddles: %s", cudaGetErrorString(e)));
        op->fast.lo = op->d_fast;
        op->fast.hi = op->d_fast + 32;
        op->fast.post_lo = op->d_fast + 32 + hi;
        op->fast.post_hi = op->d_fast + 64 + hi;
        op->fast.wn = op->d_tw;
        op->fast.w2n = op->d_post;
        op->fast_ok = true;
    }
    op->no_dmma = std::getenv("BTG_DISABLE_DMMA") != nullptr;
    op->tensor_i8 = std::getenv("BTG_TENSOR_I8") != nullptr;
    // Default: the register-load GEMV (7.4 TB/s at configs[1]); the TMA ring is
    // opt-in (BTG_GEMV_TMA=1): faster on a 6.7 GB operator, slower at 54 GB.
    op->legacy_gemv = std::getenv("BTG_GEMV_TMA") == nullptr;
    if (!smem_fits) {
        const size_t per_cta = btg::fft_smem_bytes((int)nt, 1);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const size_t cap = kScratchCapBytes / per_cta;
        op->gscratch.ctas = (int)std::max<size_t>(1, std::min<size_t>(2 * (size_t)sms, cap));
        e = cudaMalloc(&op->gscratch.buf, per_cta * op->gscratch.ctas);
        if (e != cudaSuccess)
            return cleanup_fail(fail(BTG_ENOMEM, "FFT scratch (%zu bytes): %s", per_cta * op->gscratch.ctas,
                                     cudaGetErrorString(e)));
        op->fft_batch = op->fft_batch_setup = 1;
    }
    op->plan.n = (int)nt;
    op->plan.nfac = (int)fac.size();
    for (size_t i = 0; i < fac.size(); ++i) op->plan.fac[i] = fac[i];
    op->plan.tw = op->d_tw;
    op->plan.post = op->d_post;

    const size_t fbytes = op->nf * nd * nm * op->F_elem;
    e = cudaMalloc(&op->F, fbytes);
    if (e != cudaSuccess)
        return cleanup_fail(fail(BTG_ENOMEM, "F-hat allocation of %zu bytes failed: %s", fbytes,
                                 cudaGetErrorString(e)));
    op->rows_ready.assign(nd, 0);
    *out = op;
    return BTG_OK;
}

btg_status btg_setup_rows(btg_op op, const double* blocks, size_t i0, size_t i1, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (!blocks) return fail(BTG_EARG, "null blocks pointer");
    if (i0 >= i1 || i1 > op->nd)
        return fail(BTG_EDIM, "setup rows [%zu, %zu) outside [0, %zu)", i0, i1, op->nd);
    std::lock_guard<std::mutex> lock(op->mu);
    DeviceGuard g(op->device);
    op->oz_valid = false;  // F-hat changes: int8 slices and the channel layout are stale
    op->S_valid = false;
    const size_t rows = i1 - i0;
    const size_t slab_channels = rows * op->nm;
    const long long out_fs = (long long)(op->nd * op->nm);
    // FP64 with a compile-time FFT plan: transpose the TOSI slab to SOTI rows in a
    // bounded device buffer, then the vector R2C (frequency-major stores into F-hat);
    // otherwise (FP32 F-hat, lengths without a plan, BTG_SETUP_GENERIC, or no room
    // for the buffer) the generic strided R2C. Each channel's transform is the
    // vector R2C's, wherever the channel lands.
    // FP32 F-hat: the vector R2C writes a complex128 block (frequency-major, stride
    // = the chunk's channels) after the SOTI rows, rounded into F-hat by
    // k_spec_to_f32 — the same per-element rounding as the strided kernel.
    double* soti = nullptr;
    double2* spec64 = nullptr;
    size_t soti_channels = 0;
    if (op->fast_ok && !std::getenv("BTG_SETUP_GENERIC")) {
        soti_channels = std::min(slab_channels, std::max<size_t>(1, kSetupSotiBytes / (op->nt * sizeof(double))));
        const size_t spec_bytes = op->precision == BTG_F64 ? 0 : soti_channels * op->nf * sizeof(double2);
        if (cudaMalloc(&soti, soti_channels * op->nt * sizeof(double) + spec_bytes) != cudaSuccess) {
            (void)cudaGetLastError();
            soti = nullptr;
        } else if (spec_bytes) {
            spec64 = reinterpret_cast<double2*>(soti + soti_channels * op->nt);
        }
    }
    struct SotiFree {
        double* p;
        ~SotiFree() {
            if (p) cudaFree(p);
        }
    } soti_free{soti};
    auto launch = [&](const double* src, long long in_ts, size_t c_begin, size_t count) -> btg_status {
        StageClock clk(op, &op->counters.forward_fft);
        cudaError_t e;
        const size_t off = i0 * op->nm + c_begin;
        if (soti) {
            for (size_t c = 0; c < count; c += soti_channels) {
                const size_t cnt = std::min(soti_channels, count - c);
                BTG_CUDA(btg::launch_tosi_to_soti(src + c, in_ts, soti, (int)op->nt, (long long)cnt, op->stream));
                if (spec64) {
                    BTG_CUDA(btg::launch_r2c_vec_fast((int)op->nt, soti, (long long)op->nt, spec64, (long long)cnt,
                                                      (int)cnt, op->fast, op->stream));
                    BTG_CUDA(btg::launch_spec_to_f32(spec64, (long long)cnt, (int)op->nf,
                                                     static_cast<float2*>(op->F) + off + c, out_fs, op->stream));
                    op->counters.launches += 3;
                } else {
                    BTG_CUDA(btg::launch_r2c_vec_fast((int)op->nt, soti, (long long)op->nt,
                                                      static_cast<double2*>(op->F) + off + c, out_fs, (int)cnt,
                                                      op->fast, op->stream));
                    op->counters.launches += 2;
                }
            }
            return BTG_OK;
        }
        if (op->precision == BTG_F64)
            e = btg::launch_r2c<double2>(src, 1, in_ts, static_cast<double2*>(op->F) + off, out_fs, 1,
                                         (int)count, (int)op->nt, op->plan, op->fft_batch_setup, op->stream,
                                         op->gscratch);
        else
            e = btg::launch_r2c<float2>(src, 1, in_ts, static_cast<float2*>(op->F) + off, out_fs, 1,
                                        (int)count, (int)op->nt, op->plan, op->fft_batch_setup, op->stream,
                                         op->gscratch);
        BTG_CUDA(e);
        op->counters.launches++;
        return BTG_OK;
    };
    if (flags & BTG_DEVICE_PTRS) {
        // Channel counts must fit an int grid; split very large slabs.
        const size_t max_chunk = (size_t)1 << 30;
        for (size_t c = 0; c < slab_channels; c += max_chunk) {
            const size_t cnt = std::min(max_chunk, slab_channels - c);
            BTG_TRY(launch(blocks + c, (long long)slab_channels, c, cnt));
        }
    } else {
        // Host input: stream channel ranges through a bounded device staging buffer.
        size_t chunk = std::max<size_t>(1, kHostStageBytes / (op->nt * sizeof(double)));
        chunk = std::min(chunk, slab_channels);
        BTG_TRY(host_buffers(op, chunk * op->nt, 0));
        for (size_t c = 0; c < slab_channels; c += chunk) {
            const size_t cnt = std::min(chunk, slab_channels - c);
            BTG_CUDA(cudaMemcpy2DAsync(op->hin, cnt * sizeof(double), blocks + c,
                                       slab_channels * sizeof(double), cnt * sizeof(double), op->nt,
                                       cudaMemcpyHostToDevice, op->stream));
            BTG_TRY(launch(op->hin, (long long)cnt, c, cnt));
        }
        BTG_CUDA(cudaStreamSynchronize(op->stream));
    }
    for (size_t i = i0; i < i1; ++i)
        if (!op->rows_ready[i]) {
            op->rows_ready[i] = 1;
            op->rows_ready_count++;
        }
    return BTG_OK;
}

btg_status btg_setup(const double* blocks, size_t nd, size_t nm, size_t nt, int precision,
                     int device, unsigned flags, btg_op* out) {
    BTG_TRY(btg_create(nd, nm, nt, precision, device, out));
    if (flags & BTG_KEEP_CHANNEL_LAYOUT) (*out)->keep_channel = true;
    btg_status s = btg_setup_rows(*out, blocks, 0, nd, flags & ~BTG_KEEP_CHANNEL_LAYOUT);
    if (s != BTG_OK) {
        const std::string msg = g_err;
        btg_destroy(*out);
        *out = nullptr;
        g_err = msg;
    }
    return s;
}

// ---- EWP backend (block_operator.cpp:345-421) ---------------------------------
btg_status btg_set_channel_layout(btg_op op, int keep) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    DeviceGuard g(op->device);
    op->keep_channel = keep != 0;
    if (!op->keep_channel && op->S) {
        BTG_CUDA(cudaStreamSynchronize(op->stream));
        cudaFree(op->S);
        op->S = nullptr;
        op->S_valid = false;
    }
    return BTG_OK;
}

btg_status btg_has_channel_layout(btg_op op, int* out) {
    if (!op || !out) return fail(BTG_EARG, "null argument");
    *out = op->keep_channel ? 1 : 0;
    return BTG_OK;
}

namespace {
btg_status ewp_dir(btg_op op, bool adjoint, const double* in, size_t in_len, double* out, size_t out_len,
                   unsigned flags) {
    BTG_TRY(check_ready(op));
    const char* what = adjoint ? "apply_adjoint_ewp" : "apply_forward_ewp";
    if (!in || !out) return fail(BTG_EARG, "null vector pointer");
    const size_t din = adjoint ? op->nd : op->nm;
    const size_t dout = adjoint ? op->nm : op->nd;
    BTG_TRY(check_len(what, in_len, din, op->nt, 1, din));
    BTG_TRY(check_len(what, out_len, dout, op->nt, 1, dout));
    if (!op->keep_channel)  // require_channel_layout (block_operator.cpp:335-341)
        return fail(BTG_EARG,
                    "%s: spectral operator was built without the channel layout (setup with keep_channel_layout)",
                    what);
    DeviceGuard g(op->device);
    const double* din_p = in;
    double* dout_p = out;
    if (!(flags & BTG_DEVICE_PTRS)) {
        BTG_TRY(host_buffers(op, in_len, out_len));
        BTG_CUDA(cudaMemcpyAsync(op->hin, in, in_len * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        din_p = op->hin;
        dout_p = op->hout;
    }
    BTG_TRY(ensure_spectral(op, 1));
    const size_t channels = op->nd * op->nm;
    if (!op->S) {
        const size_t bytes = op->nf * channels * op->F_elem;
        cudaError_t e = cudaMalloc(&op->S, bytes);
        if (e != cudaSuccess) {
            op->S = nullptr;
            return fail(BTG_ENOMEM, "channel layout (%zu bytes): %s", bytes, cudaGetErrorString(e));
        }
        op->S_valid = false;
    }
    if (!op->S_valid) {
        BTG_CUDA(op->precision == BTG_F64
                     ? btg::launch_channel_layout(static_cast<const double2*>(op->F), static_cast<double2*>(op->S),
                                                  (int)op->nf, (long long)channels, op->stream)
                     : btg::launch_channel_layout(static_cast<const float2*>(op->F), static_cast<float2*>(op->S),
                                                  (int)op->nf, (long long)channels, op->stream));
        op->counters.launches++;
        op->S_valid = true;
    }
    const long long nf = (long long)op->nf;
    {
        StageClock clk(op, &op->counters.forward_fft);
        BTG_CUDA(btg::launch_r2c<double2>(din_p, (long long)op->nt, 1, op->wa, 1, nf, (int)din, (int)op->nt,
                                          op->plan, op->fft_batch, op->stream, op->gscratch));
    }
    {
        StageClock clk(op, &op->counters.apply);
        BTG_CUDA(op->precision == BTG_F64
                     ? btg::launch_ewp(adjoint, static_cast<const double2*>(op->S), op->wa, op->wb, (int)op->nf,
                                       (int)op->nd, (int)op->nm, op->stream)
                     : btg::launch_ewp(adjoint, static_cast<const float2*>(op->S), op->wa, op->wb, (int)op->nf,
                                       (int)op->nd, (int)op->nm, op->stream));
    }
    {
        StageClock clk(op, &op->counters.inverse_fft);
        BTG_CUDA(btg::launch_c2r(op->wb, 1, nf, dout_p, (long long)op->nt, (int)dout, (int)op->nt, op->plan,
                                 op->fft_batch, btg::C2REpilogue{}, op->stream, op->gscratch));
    }
    op->counters.launches += 3;
    op->counters.pad.ops += 2.0 * din * op->nt;
    op->counters.forward_fft.ops += fft_ops(din, op->nt);
    op->counters.forward_fft.bytes += 8.0 * din * op->nt + 16.0 * op->nf * din;
    // the reference's EWP op / byte model (block_operator.cpp:371-376) with NF frequencies
    op->counters.apply.ops += 8.0 * channels * op->nf;
    op->counters.apply.bytes += 16.0 * op->nf * (3.0 * channels + 2.0 * (op->nd + op->nm));
    op->counters.inverse_fft.ops += fft_ops(dout, op->nt);
    op->counters.inverse_fft.bytes += 16.0 * op->nf * dout + 8.0 * dout * op->nt;
    op->counters.unpad.ops += 2.0 * dout * op->nt;
    return finish_host(op, out, dout_p, out_len, flags);
}
}  // namespace

namespace {
btg_status naive_dir(bool adjoint, const double* blocks, size_t nd, size_t nm, size_t nt, const double* in,
                     double* out, int device, unsigned flags) {
    if (!blocks || !in || !out) return fail(BTG_EARG, "null pointer");
    if (nd == 0 || nm == 0 || nt == 0) return fail(BTG_EDIM, "compact operator: all dimensions must be positive");
    if (nd > INT32_MAX || nm > INT32_MAX || nt > INT32_MAX) return fail(BTG_EDIM, "naive backend: dimension too large");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count)
        return fail(BTG_ECUDA, "no CUDA device %d", device);
    DeviceGuard g(device);
    const size_t nb = nt * nd * nm, nin = (adjoint ? nd : nm) * nt, nout = (adjoint ? nm : nd) * nt;
    const double *b_d = blocks, *in_d = in;
    double* out_d = out;
    double* tmp = nullptr;
    const bool host = !(flags & BTG_DEVICE_PTRS);
    if (host) {
        BTG_CUDA(cudaMalloc(&tmp, (nb + nin + nout) * sizeof(double)));
        cudaError_t e = cudaMemcpy(tmp, blocks, nb * sizeof(double), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(tmp + nb, in, nin * sizeof(double), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(tmp);
            return fail(BTG_ECUDA, "naive backend upload: %s", cudaGetErrorString(e));
        }
        b_d = tmp;
        in_d = tmp + nb;
        out_d = tmp + nb + nin;
    }
    cudaError_t e = btg::launch_naive(adjoint, b_d, in_d, out_d, (int)nd, (int)nm, (int)nt, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess && host) e = cudaMemcpy(out, out_d, nout * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(BTG_ECUDA, "naive backend: %s", cudaGetErrorString(e));
    return BTG_OK;
}
}  // namespace

btg_status btg_naive_forward(const double* blocks, size_t nd, size_t nm, size_t nt, const double* m, double* d,
                             int device, unsigned flags) {
    return naive_dir(false, blocks, nd, nm, nt, m, d, device, flags);
}

btg_status btg_naive_adjoint(const double* blocks, size_t nd, size_t nm, size_t nt, const double* d, double* m,
                             int device, unsigned flags) {
    return naive_dir(true, blocks, nd, nm, nt, d, m, device, flags);
}

btg_status btg_forward_ewp(btg_op op, const double* m, size_t m_len, double* d, size_t d_len, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return ewp_dir(op, false, m, m_len, d, d_len, flags);
}

btg_status btg_adjoint_ewp(btg_op op, const double* d, size_t d_len, double* m, size_t m_len, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return ewp_dir(op, true, d, d_len, m, m_len, flags);
}

btg_status btg_forward(btg_op op, const double* m, size_t m_len, double* d, size_t d_len,
                       size_t nrhs, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return apply_dir(op, false, m, m_len, d, d_len, nrhs, nullptr, flags);
}

btg_status btg_forward_ex(btg_op op, const double* m, size_t m_len, double* d, size_t d_len,
                          size_t nrhs, const btg_epilogue* epi, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return apply_dir(op, false, m, m_len, d, d_len, nrhs, epi, flags);
}

btg_status btg_adjoint_ex(btg_op op, const double* d, size_t d_len, double* m, size_t m_len,
                          size_t nrhs, const btg_epilogue* epi, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return apply_dir(op, true, d, d_len, m, m_len, nrhs, epi, flags);
}

btg_status btg_adjoint(btg_op op, const double* d, size_t d_len, double* m, size_t m_len,
                       size_t nrhs, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    return apply_dir(op, true, d, d_len, m, m_len, nrhs, nullptr, flags);
}

btg_status btg_hessian(btg_op op, const double* v, size_t v_len, double* hv, size_t hv_len,
                       size_t nrhs, const double* gamma_inv, int gamma_kind, double alpha,
                       int reg_kind, unsigned flags) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    BTG_TRY(check_ready(op));
    if (nrhs == 0) return fail(BTG_EARG, "nrhs must be >= 1");
    if (!v || !hv) return fail(BTG_EARG, "null vector pointer");
    if (reg_kind != BTG_REG_IDENTITY && reg_kind != BTG_REG_TEMPORAL_LAPLACIAN)
        return fail(BTG_EARG, "unknown regularization kind %d", reg_kind);
    if (gamma_kind < BTG_GAMMA_NONE || gamma_kind > BTG_GAMMA_PER_SAMPLE)
        return fail(BTG_EARG, "unknown gamma kind %d", gamma_kind);
    if (gamma_kind != BTG_GAMMA_NONE && !gamma_inv) return fail(BTG_EARG, "gamma_inv is null");
    BTG_TRY(check_len("hessian", v_len, op->nm, op->nt, nrhs, op->nm));
    BTG_TRY(check_len("hessian", hv_len, op->nm, op->nt, nrhs, op->nm));
    DeviceGuard g(op->device);

    const double* vd = v;
    double* hvd = hv;
    const bool chunked = !(flags & BTG_DEVICE_PTRS) && host_pipelined(op, nrhs);
    const bool mchunked = !(flags & BTG_DEVICE_PTRS) && host_pipelined_mrhs(op, nrhs);
    if (!(flags & BTG_DEVICE_PTRS)) {
        BTG_TRY(host_buffers(op, v_len, hv_len));
        if (!chunked && !mchunked)
            BTG_CUDA(cudaMemcpyAsync(op->hin, v, v_len * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        vd = op->hin;
        hvd = op->hout;
    } else if (vd == hvd && alpha != 0.0) {
        // in-place call: the final epilogue reads v while writing hv
        BTG_TRY(grow(op->vcopy, op->vcap, v_len));
        BTG_CUDA(cudaMemcpyAsync(op->vcopy, v, v_len * sizeof(double), cudaMemcpyDeviceToDevice, op->stream));
        vd = op->vcopy;
    }
    const double* gd = nullptr;
    if (gamma_kind != BTG_GAMMA_NONE) {
        const size_t glen = gamma_kind == BTG_GAMMA_PER_SENSOR ? op->nd : op->nd * op->nt;
        if (flags & BTG_DEVICE_PTRS) {
            gd = gamma_inv;
        } else {
            BTG_TRY(grow(op->gam, op->gcap, glen));
            BTG_CUDA(cudaMemcpyAsync(op->gam, gamma_inv, glen * sizeof(double), cudaMemcpyHostToDevice,
                                     op->stream));
            gd = op->gam;
        }
    }
    BTG_TRY(grow(op->wt, op->wtcap, op->nd * op->nt * nrhs));

    btg::C2REpilogue e1{};
    e1.gamma = gd;
    e1.gamma_mode = gamma_kind;
    e1.gamma_dim = (int)op->nd;
    btg::C2REpilogue e2{};
    if (alpha != 0.0) {
        e2.v = vd;
        e2.alpha = alpha;
        e2.reg_kind = reg_kind;
    }
    if (chunked) {
        // H2D of v overlapped with the forward GEMV, D2H of Hv with the adjoint GEMV
        BTG_TRY(host_forward_stage(op, v));
        BTG_TRY(run_c2r_vec(op, op->wb, op->nd, op->wt, e1));
        BTG_TRY(run_r2c_vec(op, op->wt, op->nd, op->wa));
        return host_adjoint_stage(op, hv, e2);
    }
    if (mchunked) {
        BTG_TRY(host_forward_stage_mrhs(op, v, nrhs));
        BTG_TRY(run_c2r_vec(op, op->wb, nrhs * op->nd, op->wt, e1));
        BTG_TRY(run_r2c_vec(op, op->wt, nrhs * op->nd, op->wa));
        return host_adjoint_stage_mrhs(op, hv, nrhs, e2);
    }
    if ((flags & BTG_DEVICE_PTRS) && !op->timing && !std::getenv("BTG_NO_GRAPH")) {
        BTG_TRY(hessian_graph(op, vd, hvd, nrhs, e1, e2));
        return BTG_OK;
    }
    BTG_TRY(pipeline(op, false, vd, op->wt, nrhs, e1));
    BTG_TRY(pipeline(op, true, op->wt, hvd, nrhs, e2));
    return finish_host(op, hv, hvd, hv_len, flags);
}

// partition_operator(const SpectralP2O&) (distributed.cpp:198-218) on the
// device: the shard's rectangle of every stored frequency block is copied
// HBM->HBM (or peer-to-peer over NVLink when `device` differs) with one 3-D
// copy — no re-setup, no host round trip. Entries are bit-identical.
btg_status btg_slice_operator(btg_op src, size_t i0, size_t i1, size_t j0, size_t j1, int device,
                              btg_op* out) {
    if (!src) return fail(BTG_EARG, "null operator handle");
    if (!out) return fail(BTG_EARG, "null output handle");
    *out = nullptr;
    if (i0 >= i1 || i1 > src->nd || j0 >= j1 || j1 > src->nm)
        return fail(BTG_EGRID, "slice [%zu,%zu) x [%zu,%zu) outside the %zu x %zu operator (or empty)", i0, i1,
                    j0, j1, src->nd, src->nm);
    {
        std::lock_guard<std::mutex> lock(src->mu);
        for (size_t i = i0; i < i1; ++i)
            if (!src->rows_ready[i]) return fail(BTG_EARG, "slice: sensor row %zu of the source is not set up", i);
    }
    btg_op dst = nullptr;
    BTG_TRY(btg_create(i1 - i0, j1 - j0, src->nt, src->precision, device, &dst));
    cudaMemcpy3DPeerParms p = {};
    p.srcPtr = make_cudaPitchedPtr(static_cast<char*>(src->F) + (i0 * src->nm + j0) * src->F_elem,
                                   src->nm * src->F_elem, (j1 - j0) * src->F_elem, src->nd);
    p.srcDevice = src->device;
    p.dstPtr = make_cudaPitchedPtr(dst->F, dst->nm * dst->F_elem, dst->nm * dst->F_elem, dst->nd);
    p.dstDevice = dst->device;
    p.extent = make_cudaExtent((j1 - j0) * src->F_elem, i1 - i0, src->nf);
    cudaError_t e;
    {
        DeviceGuard g(src->device);
        std::lock_guard<std::mutex> lock(src->mu);
        e = cudaMemcpy3DPeerAsync(&p, src->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(src->stream);
    }
    if (e != cudaSuccess) {
        btg_destroy(dst);
        return fail(BTG_ECUDA, "slice copy: %s", cudaGetErrorString(e));
    }
    std::fill(dst->rows_ready.begin(), dst->rows_ready.end(), 1);
    dst->rows_ready_count = dst->nd;
    *out = dst;
    return BTG_OK;
}

// Internal hooks for btg_io.cu (C++ linkage, not part of the C ABI).
btg_status btg_internal_fail(btg_status s, const char* msg) { return fail(s, "%s", msg); }

// Grid engine (btg_grid_engine.cu, P2P transport): one device-pointer, single-RHS
// F / F* whose final C2R also tree-reduces the partials of `npeers` other group
// members into its stores (C2REpilogue::peers). btg_internal_fused_ok says
// whether this handle's C2R takes that path (fast plan, FP64 or FP32, 1 RHS).
int btg_internal_fused_ok(btg_op op, int adjoint) {
    if (!op || !op->fast_ok) return 0;
    (void)adjoint;
    return 1;
}
btg_status btg_internal_apply_fused(btg_op op, int adjoint, const double* in, size_t in_len, double* out,
                                    size_t out_len, const btg_epilogue* ex, const double* const* peers, int npeers) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (npeers < 1 || npeers > btg::kMaxFusedPeers) return fail(BTG_EARG, "fused reduce: %d peers", npeers);
    if (!btg_internal_fused_ok(op, adjoint)) return fail(BTG_EARG, "fused reduce: no fast C2R for this horizon");
    if (!aligned16(out) || (ex && ex->reg_v && !aligned16(ex->reg_v)))
        return fail(BTG_EARG, "fused reduce: 16-byte aligned vectors required");
    std::lock_guard<std::mutex> lock(op->mu);
    return apply_dir(op, adjoint != 0, in, in_len, out, out_len, 1, ex, BTG_DEVICE_PTRS, peers, npeers);
}

btg_status btg_internal_upload_spectrum_block(btg_op op, size_t f, const double* block) {
    if (!op || !block || f > op->nt) return fail(BTG_EARG, "bad spectrum block upload");
    std::lock_guard<std::mutex> lock(op->mu);
    op->oz_valid = false;
    op->S_valid = false;
    DeviceGuard g(op->device);
    const size_t blk = op->nd * op->nm;
    if (op->precision == BTG_F64) {
        BTG_CUDA(cudaMemcpy(static_cast<double2*>(op->F) + f * blk, block, blk * sizeof(double2),
                            cudaMemcpyHostToDevice));
    } else {
        std::vector<float2> tmp(blk);
        for (size_t k = 0; k < blk; ++k)
            tmp[k] = make_float2(static_cast<float>(block[2 * k]), static_cast<float>(block[2 * k + 1]));
        BTG_CUDA(cudaMemcpy(static_cast<float2*>(op->F) + f * blk, tmp.data(), blk * sizeof(float2),
                            cudaMemcpyHostToDevice));
    }
    return BTG_OK;
}

btg_status btg_internal_mark_ready(btg_op op) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    std::fill(op->rows_ready.begin(), op->rows_ready.end(), 1);
    op->rows_ready_count = op->nd;
    return BTG_OK;
}

// ---------------------------------------------------------------------------
// Device-resident CG (inverse.cpp:105-156) and objective (inverse.cpp:93-103)
// ---------------------------------------------------------------------------
namespace {

// Solver / objective vectors live in per-handle slots grown on demand and kept
// across calls: a cudaMalloc + cudaFree of several N_m x N_t vectors per solve
// cost tens to hundreds of milliseconds at configs[1] (measured: 20-iteration
// solves at 17 to 57 ms per iteration with per-call allocation, the Hessian
// itself 16 ms).
enum CgSlot { kSlotX, kSlotR, kSlotZ, kSlotP, kSlotHp, kSlotPartial, kSlotScal, kSlotPivot, kSlotScratch,
              kSlotRhs, kSlotGam };
struct CgBuffers {
    double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *hp = nullptr, *partial = nullptr,
           *scal = nullptr, *pivot = nullptr, *scratch = nullptr, *rhs = nullptr, *gam = nullptr;
    size_t partial_cap = 0;  // doubles: reduction partials / folded-dot CTA partials
};

// The slots outlive the call: every exit (errors included) drains the handle's
// stream, so a later call on another stream never races work still in flight.
struct DrainOnExit {
    btg_op op;
    ~DrainOnExit() { cudaStreamSynchronize(op->stream); }
};

btg_status slot(btg_op op, CgSlot k, double** p, size_t n) {
    BTG_TRY(grow(op->solver_ws[k], op->solver_cap[k], std::max<size_t>(n, 1)));
    *p = op->solver_ws[k];
    return BTG_OK;
}

// Solver scalars land in page-locked memory (a direct DMA instead of the
// driver's pageable staging path).
btg_status read_scalar(btg_op op, const double* dev, double* host) {
    if (!op->pinned_scalar) BTG_CUDA(cudaMallocHost(&op->pinned_scalar, sizeof(double)));
    BTG_CUDA(cudaMemcpyAsync(op->pinned_scalar, dev, sizeof(double), cudaMemcpyDeviceToHost, op->stream));
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    *host = *op->pinned_scalar;
    return BTG_OK;
}

// H v on device pointers (the body of btg_hessian without staging). With
// `curv`, also v^T H v into *curv (device): folded into the final C2R's stores
// (per-CTA partials in `part`, capacity `part_cap`, summed in index order), or a
// separate dot when the generic C2R ran.
btg_status hessian_dev(btg_op op, const double* vd, double* hvd, const double* gd, int gamma_kind, double alpha,
                       int reg_kind, double* part = nullptr, size_t part_cap = 0, double* curv = nullptr) {
    BTG_TRY(grow(op->wt, op->wtcap, op->nd * op->nt));
    btg::C2REpilogue e1{};
    e1.gamma = gd;
    e1.gamma_mode = gamma_kind;
    e1.gamma_dim = (int)op->nd;
    BTG_TRY(pipeline(op, false, vd, op->wt, 1, e1));
    btg::C2REpilogue e2{};
    if (alpha != 0.0) {
        e2.v = vd;
        e2.alpha = alpha;
        e2.reg_kind = reg_kind;
    }
    if (!curv) return pipeline(op, true, op->wt, hvd, 1, e2);
    e2.dot_v = vd;
    e2.dot_out = part;
    int ctas = 0;
    BTG_TRY(pipeline(op, true, op->wt, hvd, 1, e2, &ctas));
    const size_t n = op->nm * op->nt;
    if (ctas > 0 && (size_t)ctas <= part_cap) {
        BTG_CUDA(btg::launch_sum_partials(part, ctas, curv, op->stream));
        op->counters.launches++;
    } else {
        if (ctas > 0) return fail(BTG_EARG, "internal: %d folded-dot partials exceed %zu", ctas, part_cap);
        BTG_CUDA(btg::launch_dot(vd, hvd, n, part, curv, op->stream));
        op->counters.launches += 2;
    }
    return BTG_OK;
}

// CG building blocks shared by the host-driven and the graph loop.
btg_status cg_precondition(btg_op op, const CgBuffers& b, bool lap, size_t n, double* zout, const double* rin) {
    if (lap) {
        BTG_CUDA(btg::launch_reg_apply_inverse(zout, rin, b.pivot, b.scratch, op->nm, (int)op->nt, op->stream));
    } else {
        BTG_CUDA(cudaMemcpyAsync(zout, rin, n * sizeof(double), cudaMemcpyDeviceToDevice, op->stream));
    }
    op->counters.launches++;
    return BTG_OK;
}

btg_status cg_dot(btg_op op, const CgBuffers& b, size_t n, const double* a, const double* c, double* host) {
    BTG_CUDA(btg::launch_dot(a, c, n, b.partial, b.scal, op->stream));
    op->counters.launches += 2;
    return read_scalar(op, b.scal, host);
}

btg_status cg_bad_curvature(double curvature) {
    return fail(BTG_ESOLVER, "cg: direction of non-positive curvature, p^T H p = %g; the Hessian is "
                             "not positive definite", curvature);
}

// inverse.cpp:118-153 driven from the host: two scalar read-backs per
// iteration (BTG_CG_HOST_LOOP=1; the graph loop below is the default and
// produces the same bits).
btg_status cg_host_loop(btg_op op, const CgBuffers& b, double* x, const double* gd, int gamma_kind, double alpha,
                        int reg_kind, bool precond, bool lap, double tol, size_t max_iterations, double rho,
                        double rhs_norm, size_t n, btg_cg_result* result) {
    for (size_t it = 1; it <= max_iterations; ++it) {
        BTG_TRY(hessian_dev(op, b.p, b.hp, gd, gamma_kind, alpha, reg_kind, b.partial, b.partial_cap, b.scal));
        double curvature = 0.0;
        BTG_TRY(read_scalar(op, b.scal, &curvature));
        if (!(curvature > 0.0)) return cg_bad_curvature(curvature);
        const double step = rho / curvature;
        double rn2 = 0.0;
        BTG_CUDA(btg::launch_cg_update(x, b.r, b.p, b.hp, step, n, b.partial, b.scal, op->stream));
        op->counters.launches += 2;
        BTG_TRY(read_scalar(op, b.scal, &rn2));
        result->iterations = it;
        result->relative_residual = std::sqrt(rn2) / rhs_norm;
        if (result->relative_residual <= tol) {
            result->converged = 1;
            break;
        }
        double rho_next = rn2;
        if (precond) {
            BTG_TRY(cg_precondition(op, b, lap, n, b.z, b.r));
            BTG_TRY(cg_dot(op, b, n, b.r, b.z, &rho_next));
        }
        const double beta = rho_next / rho;
        rho = rho_next;
        BTG_CUDA(btg::launch_xpby(b.p, precond ? b.z : b.r, beta, n, op->stream));
        op->counters.launches++;
    }
    return BTG_OK;
}

// The whole iteration loop as ONE graph launch: a WHILE conditional node whose
// body (captured once from the same stream code) is Hessian -> p.Hp ->
// update + ||r||^2 -> loop control (k_cg_check clears the condition on
// convergence, the iteration cap or a non-positive curvature) -> [M^-1 r,
// r.z, beta] -> p = z + beta p. No host round trip until the loop ends; the
// scalars never leave the device.
struct GraphGuard {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t e = nullptr;
    cudaStream_t capturing = nullptr;
    ~GraphGuard() {
        if (capturing) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(capturing, &junk);
            if (junk) cudaGraphDestroy(junk);
            cudaGetLastError();
        }
        if (e) cudaGraphExecDestroy(e);
        if (g) cudaGraphDestroy(g);
    }
};

btg_status cg_graph_loop(btg_op op, const CgBuffers& b, double* x, const double* gd, int gamma_kind, double alpha,
                         int reg_kind, bool precond, bool lap, double tol, size_t max_iterations, double rho,
                         double rhs_norm, size_t n, btg_cg_result* result) {
    using namespace btg;
    double st0[kCgStateLen] = {};
    st0[kCgRho] = rho;
    st0[kCgRhsNorm] = rhs_norm;
    st0[kCgTol] = tol;
    st0[kCgRelRes] = 1.0;
    st0[kCgMaxIt] = (double)max_iterations;
    st0[kCgStatus] = kCgRunning;
    double* st = b.scal;
    BTG_CUDA(cudaMemcpyAsync(st, st0, sizeof(st0), cudaMemcpyHostToDevice, op->stream));
    // everything the body touches is allocated before the capture
    BTG_TRY(grow(op->wt, op->wtcap, op->nd * op->nt));
    BTG_TRY(ensure_spectral(op, 1));
    BTG_CUDA(cudaStreamSynchronize(op->stream));  // st0 is a stack array

    GraphGuard gg;
    BTG_CUDA(cudaGraphCreate(&gg.g, 0));
    cudaGraphConditionalHandle cond;
    BTG_CUDA(cudaGraphConditionalHandleCreate(&cond, gg.g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    BTG_CUDA(cudaGraphAddNode(&node, gg.g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];

    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot capture); the graph then runs on the caller's
    if (!op->capture_stream) BTG_CUDA(cudaStreamCreateWithFlags(&op->capture_stream, cudaStreamNonBlocking));
    const cudaStream_t run_stream = op->stream;
    const bool timing = op->timing;
    op->timing = false;  // no event sync inside a capture
    const btg_counters c0 = op->counters;
    BTG_CUDA(cudaStreamBeginCaptureToGraph(op->capture_stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    op->stream = op->capture_stream;
    gg.capturing = op->capture_stream;
    btg_status s = hessian_dev(op, b.p, b.hp, gd, gamma_kind, alpha, reg_kind, b.partial, b.partial_cap,
                               st + kCgCurvature);
    cudaError_t e = cudaSuccess;
    if (s == BTG_OK) {
        e = launch_cg_update_dev(x, b.r, b.p, b.hp, st, n, b.partial, op->stream);
        if (e == cudaSuccess) e = launch_cg_check(b.partial, st, cond, precond ? 1 : 0, op->stream);
        op->counters.launches += 2;
    }
    if (s == BTG_OK && e == cudaSuccess && precond) {
        s = cg_precondition(op, b, lap, n, b.z, b.r);
        if (s == BTG_OK) e = launch_dot(b.r, b.z, n, b.partial, st + kCgRhoNext, op->stream);
        if (e == cudaSuccess) e = launch_cg_beta(st, op->stream);
        op->counters.launches += 3;
    }
    if (s == BTG_OK && e == cudaSuccess) {
        e = launch_xpby_dev(b.p, precond ? b.z : b.r, st, n, op->stream);
        op->counters.launches++;
    }
    op->timing = timing;
    op->stream = run_stream;
    gg.capturing = nullptr;
    cudaGraph_t captured = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(op->capture_stream, &captured);
    if (s != BTG_OK) return s;
    BTG_CUDA(e);
    BTG_CUDA(ec);
    // per-iteration counters from the capture, scaled by the iterations run below
    btg_counters delta = op->counters;
    op->counters = c0;

    BTG_CUDA(cudaGraphInstantiate(&gg.e, gg.g, 0));
    BTG_CUDA(cudaGraphLaunch(gg.e, op->stream));
    if (!op->pinned_state) BTG_CUDA(cudaMallocHost(&op->pinned_state, kCgStateLen * sizeof(double)));
    BTG_CUDA(cudaMemcpyAsync(op->pinned_state, st, kCgStateLen * sizeof(double), cudaMemcpyDeviceToHost, op->stream));
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    const double* fin = op->pinned_state;
    const double bodies = fin[kCgIterations] + (fin[kCgStatus] == kCgBadCurvature ? 1.0 : 0.0);
    auto scale = [&](btg_stage_counters& dst, const btg_stage_counters& d0, const btg_stage_counters& d1) {
        dst.ops += bodies * (d1.ops - d0.ops);
        dst.bytes += bodies * (d1.bytes - d0.bytes);
    };
    scale(op->counters.pad, c0.pad, delta.pad);
    scale(op->counters.forward_fft, c0.forward_fft, delta.forward_fft);
    scale(op->counters.reorder_in, c0.reorder_in, delta.reorder_in);
    scale(op->counters.apply, c0.apply, delta.apply);
    scale(op->counters.reorder_out, c0.reorder_out, delta.reorder_out);
    scale(op->counters.inverse_fft, c0.inverse_fft, delta.inverse_fft);
    scale(op->counters.unpad, c0.unpad, delta.unpad);
    op->counters.launches += (uint64_t)bodies * (delta.launches - c0.launches);

    result->iterations = (size_t)fin[kCgIterations];
    if (fin[kCgIterations] > 0) result->relative_residual = fin[kCgRelRes];
    if (fin[kCgStatus] == kCgConverged) result->converged = 1;
    if (fin[kCgStatus] == kCgBadCurvature) return cg_bad_curvature(fin[kCgCurvature]);
    return BTG_OK;
}

}  // namespace

btg_status btg_cg_solve(btg_op op, const double* rhs, size_t rhs_len, double* x_out, size_t x_len,
                        const double* gamma_inv, int gamma_kind, double alpha, int reg_kind, double tol,
                        size_t max_iterations, int use_reg_preconditioner, unsigned flags, btg_cg_result* result) {
    if (!op || !result) return fail(BTG_EARG, "null argument");
    std::lock_guard<std::mutex> lock(op->mu);
    BTG_TRY(check_ready(op));
    if (!rhs || !x_out) return fail(BTG_EARG, "null vector pointer");
    if (reg_kind != BTG_REG_IDENTITY && reg_kind != BTG_REG_TEMPORAL_LAPLACIAN)
        return fail(BTG_EARG, "unknown regularization kind %d", reg_kind);
    if (gamma_kind < BTG_GAMMA_NONE || gamma_kind > BTG_GAMMA_PER_SAMPLE)
        return fail(BTG_EARG, "unknown gamma kind %d", gamma_kind);
    if (gamma_kind != BTG_GAMMA_NONE && !gamma_inv) return fail(BTG_EARG, "gamma_inv is null");
    BTG_TRY(check_len("cg_solve", rhs_len, op->nm, op->nt, 1, op->nm));
    BTG_TRY(check_len("cg_solve", x_len, op->nm, op->nt, 1, op->nm));
    DeviceGuard g(op->device);
    const size_t n = rhs_len;
    if (max_iterations == 0)
        max_iterations = 10 * static_cast<size_t>(std::ceil(std::sqrt(static_cast<double>(n)))) + 1;
    *result = btg_cg_result{};
    struct Events {  // destroyed on every exit, early errors included
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        ~Events() {
            if (t0) cudaEventDestroy(t0);
            if (t1) cudaEventDestroy(t1);
        }
    } evs;
    BTG_CUDA(cudaEventCreate(&evs.t0));
    BTG_CUDA(cudaEventCreate(&evs.t1));
    const cudaEvent_t t0 = evs.t0, t1 = evs.t1;
    cudaEventRecord(t0, op->stream);

    CgBuffers b;
    DrainOnExit drain{op};
    const bool dev = flags & BTG_DEVICE_PTRS;
    BTG_TRY(slot(op, kSlotR, &b.r, n));
    BTG_TRY(slot(op, kSlotP, &b.p, n));
    BTG_TRY(slot(op, kSlotHp, &b.hp, n));
    // the folded p^T H p writes one partial per C2R CTA (<= one per source channel)
    b.partial_cap = std::max<size_t>(btg::kRedBlocks, op->nm);
    BTG_TRY(slot(op, kSlotPartial, &b.partial, b.partial_cap));
    BTG_TRY(slot(op, kSlotScal, &b.scal, btg::kCgStateLen));
    const bool precond = use_reg_preconditioner != 0;
    if (precond) BTG_TRY(slot(op, kSlotZ, &b.z, n));
    double* x = dev ? x_out : nullptr;
    if (!dev) {
        BTG_TRY(slot(op, kSlotX, &b.x, n));
        x = b.x;
    }
    const double* rhs_d = rhs;
    if (!dev) {
        BTG_TRY(slot(op, kSlotRhs, &b.rhs, n));
        BTG_CUDA(cudaMemcpyAsync(b.rhs, rhs, n * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        rhs_d = b.rhs;
    }
    const double* gd = nullptr;
    if (gamma_kind != BTG_GAMMA_NONE) {
        const size_t glen = gamma_kind == BTG_GAMMA_PER_SENSOR ? op->nd : op->nd * op->nt;
        gd = gamma_inv;
        if (!dev) {
            BTG_TRY(slot(op, kSlotGam, &b.gam, glen));
            BTG_CUDA(cudaMemcpyAsync(b.gam, gamma_inv, glen * sizeof(double), cudaMemcpyHostToDevice, op->stream));
            gd = b.gam;
        }
    }
    const bool lap = reg_kind == BTG_REG_TEMPORAL_LAPLACIAN;
    if (precond && lap) {
        // Thomas pivots of the (-1, 2, -1) system, in the reference's order (inverse.cpp:57-63)
        std::vector<double> piv(op->nt), scr(op->nt, 0.0);
        double pivot = 2.0;
        piv[0] = pivot;
        for (size_t t = 1; t < op->nt; ++t) {
            scr[t] = -1.0 / pivot;
            pivot = 2.0 + scr[t];
            piv[t] = pivot;
        }
        BTG_TRY(slot(op, kSlotPivot, &b.pivot, op->nt));
        BTG_TRY(slot(op, kSlotScratch, &b.scratch, op->nt));
        BTG_CUDA(cudaMemcpyAsync(b.pivot, piv.data(), op->nt * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        BTG_CUDA(cudaMemcpyAsync(b.scratch, scr.data(), op->nt * sizeof(double), cudaMemcpyHostToDevice,
                                 op->stream));
    }
    BTG_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), op->stream));
    double rhs_n2 = 0.0;
    BTG_TRY(cg_dot(op, b, n, rhs_d, rhs_d, &rhs_n2));
    const double rhs_norm = std::sqrt(rhs_n2);
    btg_status status = BTG_OK;
    if (rhs_norm == 0.0) {
        result->converged = 1;
    } else {
        BTG_CUDA(cudaMemcpyAsync(b.r, rhs_d, n * sizeof(double), cudaMemcpyDeviceToDevice, op->stream));
        const double* zp = b.r;
        if (precond) {
            BTG_TRY(cg_precondition(op, b, lap, n, b.z, b.r));
            zp = b.z;
        }
        BTG_CUDA(cudaMemcpyAsync(b.p, zp, n * sizeof(double), cudaMemcpyDeviceToDevice, op->stream));
        double rho = 0.0;
        BTG_TRY(cg_dot(op, b, n, b.r, zp, &rho));
        if (rho <= 0.0 && precond)
            return fail(BTG_ESOLVER, "cg: preconditioned residual product r^T z = %g <= 0; regularization is not "
                                     "positive definite", rho);
        result->relative_residual = 1.0;
        if (std::getenv("BTG_CG_HOST_LOOP")) {
            status = cg_host_loop(op, b, x, gd, gamma_kind, alpha, reg_kind, precond, lap, tol, max_iterations, rho,
                                  rhs_norm, n, result);
        } else {
            status = cg_graph_loop(op, b, x, gd, gamma_kind, alpha, reg_kind, precond, lap, tol, max_iterations, rho,
                                   rhs_norm, n, result);
        }
    }
    if (status != BTG_OK) return status;
    if (!dev) BTG_CUDA(cudaMemcpyAsync(x_out, x, n * sizeof(double), cudaMemcpyDeviceToHost, op->stream));
    cudaEventRecord(t1, op->stream);
    BTG_CUDA(cudaEventSynchronize(t1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    result->seconds = ms * 1e-3;
    return BTG_OK;
}

btg_status btg_objective(btg_op op, const double* m, size_t m_len, const double* d_obs, size_t d_len, double alpha,
                         int reg_kind, unsigned flags, double* value) {
    if (!op || !value) return fail(BTG_EARG, "null argument");
    std::lock_guard<std::mutex> lock(op->mu);
    BTG_TRY(check_ready(op));
    if (!m || !d_obs) return fail(BTG_EARG, "null vector pointer");
    if (reg_kind != BTG_REG_IDENTITY && reg_kind != BTG_REG_TEMPORAL_LAPLACIAN)
        return fail(BTG_EARG, "unknown regularization kind %d", reg_kind);
    if (d_len != op->nd * op->nt)
        return fail(BTG_EDIM, "objective: observations do not match the operator");
    BTG_TRY(check_len("objective", m_len, op->nm, op->nt, 1, op->nm));
    DeviceGuard g(op->device);
    CgBuffers b;
    DrainOnExit drain{op};
    const bool dev = flags & BTG_DEVICE_PTRS;
    const double* md = m;
    const double* dd = d_obs;
    if (!dev) {
        BTG_TRY(slot(op, kSlotX, &b.x, m_len));
        BTG_TRY(slot(op, kSlotRhs, &b.rhs, d_len));
        BTG_CUDA(cudaMemcpyAsync(b.x, m, m_len * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        BTG_CUDA(cudaMemcpyAsync(b.rhs, d_obs, d_len * sizeof(double), cudaMemcpyHostToDevice, op->stream));
        md = b.x;
        dd = b.rhs;
    }
    BTG_TRY(slot(op, kSlotR, &b.r, d_len));
    BTG_TRY(slot(op, kSlotP, &b.p, m_len));
    // the folded p^T H p writes one partial per C2R CTA (<= one per source channel)
    b.partial_cap = std::max<size_t>(btg::kRedBlocks, op->nm);
    BTG_TRY(slot(op, kSlotPartial, &b.partial, b.partial_cap));
    BTG_TRY(slot(op, kSlotScal, &b.scal, 1));
    BTG_TRY(pipeline(op, false, md, b.r, 1, btg::C2REpilogue{}));
    BTG_CUDA(btg::launch_sub(b.r, b.r, dd, d_len, op->stream));
    double misfit = 0.0, reg = 0.0;
    BTG_CUDA(btg::launch_dot(b.r, b.r, d_len, b.partial, b.scal, op->stream));
    BTG_TRY(read_scalar(op, b.scal, &misfit));
    BTG_CUDA(btg::launch_reg_apply(b.p, md, op->nm, (int)op->nt, reg_kind, op->stream));
    BTG_CUDA(btg::launch_dot(md, b.p, m_len, b.partial, b.scal, op->stream));
    BTG_TRY(read_scalar(op, b.scal, &reg));
    op->counters.launches += 6;
    *value = 0.5 * misfit + 0.5 * alpha * reg;
    return BTG_OK;
}

btg_status btg_set_stream(btg_op op, void* stream) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    std::lock_guard<std::mutex> lock(op->mu);
    op->stream = stream ? static_cast<cudaStream_t>(stream) : op->own_stream;
    return BTG_OK;
}

btg_status btg_synchronize(btg_op op) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    DeviceGuard g(op->device);
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    return BTG_OK;
}

btg_status btg_set_timing(btg_op op, int enabled) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    op->timing = enabled != 0;
    return BTG_OK;
}

btg_status btg_set_multi_rhs_engine(btg_op op, int engine) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (engine != BTG_MRHS_DMMA && engine != BTG_MRHS_TENSOR_I8)
        return fail(BTG_EARG, "unknown multi-RHS engine %d", engine);
    std::lock_guard<std::mutex> lock(op->mu);
    op->tensor_i8 = engine == BTG_MRHS_TENSOR_I8;
    return BTG_OK;
}

btg_status btg_get_counters(btg_op op, btg_counters* out) {
    if (!op || !out) return fail(BTG_EARG, "null argument");
    *out = op->counters;
    return BTG_OK;
}

btg_status btg_reset_counters(btg_op op) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    op->counters = btg_counters{};
    return BTG_OK;
}

btg_status btg_get_dims(btg_op op, size_t* nd, size_t* nm, size_t* nt, int* precision) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (nd) *nd = op->nd;
    if (nm) *nm = op->nm;
    if (nt) *nt = op->nt;
    if (precision) *precision = op->precision;
    return BTG_OK;
}

btg_status btg_export_spectrum(btg_op op, double* out, int full) {
    if (!op || !out) return fail(BTG_EARG, "null argument");
    std::lock_guard<std::mutex> lock(op->mu);
    BTG_TRY(check_ready(op));
    DeviceGuard g(op->device);
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    const size_t blk = op->nd * op->nm;
    const size_t count = op->nf * blk;
    std::vector<std::complex<double>> half(count);
    if (op->precision == BTG_F64) {
        BTG_CUDA(cudaMemcpy(half.data(), op->F, count * sizeof(double2), cudaMemcpyDeviceToHost));
    } else {
        std::vector<std::complex<float>> tmp(count);
        BTG_CUDA(cudaMemcpy(tmp.data(), op->F, count * sizeof(float2), cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < count; ++k) half[k] = std::complex<double>(tmp[k].real(), tmp[k].imag());
    }
    auto* dst = reinterpret_cast<std::complex<double>*>(out);
    if (!full) {
        std::memcpy(dst, half.data(), count * sizeof(std::complex<double>));
        return BTG_OK;
    }
    const size_t len = 2 * op->nt;
    for (size_t f = 0; f < len; ++f) {
        if (f <= op->nt) {
            std::memcpy(dst + f * blk, half.data() + f * blk, blk * sizeof(std::complex<double>));
        } else {
            const std::complex<double>* src = half.data() + (len - f) * blk;
            for (size_t c = 0; c < blk; ++c) dst[f * blk + c] = std::conj(src[c]);
        }
    }
    return BTG_OK;
}

btg_status btg_export_spectrum_block(btg_op op, size_t f, double* out) {
    if (!op || !out) return fail(BTG_EARG, "null argument");
    std::lock_guard<std::mutex> lock(op->mu);
    BTG_TRY(check_ready(op));
    if (f > op->nt) return fail(BTG_EDIM, "frequency %zu outside the stored 0..%zu", f, op->nt);
    DeviceGuard g(op->device);
    BTG_CUDA(cudaStreamSynchronize(op->stream));
    const size_t blk = op->nd * op->nm;
    if (op->precision == BTG_F64) {
        BTG_CUDA(cudaMemcpy(out, static_cast<double2*>(op->F) + f * blk, blk * sizeof(double2),
                            cudaMemcpyDeviceToHost));
    } else {
        std::vector<float2> tmp(blk);
        BTG_CUDA(cudaMemcpy(tmp.data(), static_cast<float2*>(op->F) + f * blk, blk * sizeof(float2),
                            cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < blk; ++k) {
            out[2 * k] = tmp[k].x;
            out[2 * k + 1] = tmp[k].y;
        }
    }
    return BTG_OK;
}

btg_status btg_spectrum_device(btg_op op, void** ptr, size_t* elem_bytes) {
    if (!op) return fail(BTG_EARG, "null operator handle");
    if (ptr) *ptr = op->F;
    if (elem_bytes) *elem_bytes = op->F_elem;
    return BTG_OK;
}

void btg_destroy(btg_op op) {
    if (!op) return;
    {
        DeviceGuard g(op->device);
        if (op->own_stream) cudaStreamSynchronize(op->own_stream);
        if (op->stream && op->stream != op->own_stream) cudaStreamSynchronize(op->stream);
        cudaFree(op->F);
        cudaFree(op->oz_A);
        cudaFree(op->oz_mA);
        cudaFree(op->oz_B);
        cudaFree(op->S);
        cudaFree(op->oz_vexp);
        cudaFree(op->oz_mB);
        cudaFree(op->d_tw);
        cudaFree(op->d_post);
        cudaFree(op->d_fast);
        cudaFree(op->gscratch.buf);
        cudaFree(op->wa);
        cudaFree(op->wb);
        cudaFree(op->wt);
        cudaFree(op->hin);
        cudaFree(op->hout);
        cudaFree(op->gam);
        cudaFree(op->vcopy);
        if (op->own_stream) cudaStreamDestroy(op->own_stream);
        if (op->hess_graph.exec) cudaGraphExecDestroy(op->hess_graph.exec);
        if (op->capture_stream) cudaStreamDestroy(op->capture_stream);
        if (op->copy_stream) {
            cudaStreamSynchronize(op->copy_stream);
            cudaStreamDestroy(op->copy_stream);
        }
        if (op->fft_stream) {
            cudaStreamSynchronize(op->fft_stream);
            cudaStreamDestroy(op->fft_stream);
        }
        if (op->pinned_scalar) cudaFreeHost(op->pinned_scalar);
        if (op->pinned_state) cudaFreeHost(op->pinned_state);
        for (double* q : op->solver_ws) cudaFree(q);
        for (cudaEvent_t e : op->ev)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : op->ev_h2d)
            if (e) cudaEventDestroy(e);
    }
    delete op;
}

btg_status btg_fill_uniform(double* out, size_t n, uint64_t seed, uint64_t offset, double lo, double hi,
                            void* stream) {
    return btg_fill_uniform_3d(out, 1, 1, n, seed, offset, 0, 0, lo, hi, stream);
}

btg_status btg_fill_uniform_3d(double* out, size_t na, size_t nb, size_t nc, uint64_t seed, uint64_t offset,
                               uint64_t stride_a, uint64_t stride_b, double lo, double hi, void* stream) {
    if (!out && na * nb * nc != 0) return fail(BTG_EARG, "null output pointer");
    BTG_CUDA(btg::launch_fill_uniform(out, na, nb, nc, seed, offset, stride_a, stride_b, lo, hi,
                                      static_cast<cudaStream_t>(stream)));
    return BTG_OK;
}

}  // extern "C"
