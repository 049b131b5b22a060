// TEST INFRASTRUCTURE ONLY — the checker, never the thing measured or shipped.
//
// A flat C ABI over the UNMODIFIED reference sources under
// /root/reference/proj/src (compiled by oracle/Makefile into
// oracle/_ref/libbtoep_ref.so together with oracle/ref_fft_shim.cpp). It lets
// the pytest suite, the golden-fixture generator and bench.py's CPU arm call
// the reference's own C++ operator API through ctypes:
//
//   setup            block_operator.hpp:64   (block_operator.cpp:178-205)
//   apply_forward    block_operator.hpp:71   (block_operator.cpp:218-273)
//   apply_adjoint    block_operator.hpp:76   (block_operator.cpp:275-331)
//   naive_apply_*    block_operator.hpp:88   (block_operator.cpp:423-482)
//   HessianOperator  inverse.hpp:32-39       (inverse.cpp:78-91)
//   partition + distributed_forward/adjoint  distributed.hpp:57-121
//   Rng              rng.hpp:12-32  (the seeded inputs of tests/oracles.cpp:87-98)
//   run_verification verify.hpp:13
//   select_grid / weak_scaling_shape / modified_cost / comm_cost  grid_planner.hpp:43-65
//
// Every entry point returns 0 on success, 1 on a btoep::Error (message in
// ref_last_error()), 2 on any other exception.
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "btoep/block_operator.hpp"
#include "btoep/distributed.hpp"
#include "btoep/errors.hpp"
#include "btoep/grid_planner.hpp"
#include "btoep/inverse.hpp"
#include "btoep/io.hpp"
#include "btoep/rng.hpp"
#include "btoep/verify.hpp"

using namespace btoep;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

CompactP2O make_compact(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt) {
    CompactP2O op = CompactP2O::zeros(nd, nm, nt);
    std::memcpy(op.blocks.data(), blocks, sizeof(double) * op.blocks.size());
    return op;
}

SpaceTimeVector make_soti(const double* v, std::size_t dim, std::size_t nt) {
    SpaceTimeVector out = SpaceTimeVector::zeros(dim, nt, Ordering::SOTI);
    std::memcpy(out.values.data(), v, sizeof(double) * out.values.size());
    return out;
}

void copy_out(const SpaceTimeVector& v, double* out) {
    const SpaceTimeVector soti = with_ordering(v, Ordering::SOTI);
    std::memcpy(out, soti.values.data(), sizeof(double) * soti.values.size());
}

struct PartitionHandle {
    Partition partition;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- seeded inputs (tests/oracles.cpp:87-98 draws: blocks, then m, then d) ----
int ref_rng_uniform(std::uint64_t seed, std::size_t n, double lo, double hi, double* out) {
    return guarded([&] {
        Rng rng(seed);
        for (std::size_t i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
    });
}

int ref_rng_raw(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    return guarded([&] {
        std::mt19937_64 gen(seed);
        for (std::size_t i = 0; i < n; ++i) out[i] = gen();
    });
}

// ---- spectral operator handle ------------------------------------------------
void* ref_setup(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt) {
    SpectralP2O* op = nullptr;
    const int rc = guarded([&] { op = new SpectralP2O(setup(make_compact(blocks, nd, nm, nt))); });
    return rc == 0 ? op : nullptr;
}

// setup with SetupOptions::keep_channel_layout (block_operator.hpp:58-60): the
// channel-major copy the EWP backend (block_operator.cpp:345-421) streams.
void* ref_setup_channel_layout(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt) {
    SpectralP2O* op = nullptr;
    const int rc = guarded([&] {
        SetupOptions o;
        o.keep_channel_layout = true;
        op = new SpectralP2O(setup(make_compact(blocks, nd, nm, nt), o));
    });
    return rc == 0 ? op : nullptr;
}

void ref_destroy(void* h) { delete static_cast<SpectralP2O*>(h); }

int ref_forward_ewp(void* h, const double* m, double* d) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        copy_out(apply_forward_ewp(op, make_soti(m, op.num_sources, op.num_steps)), d);
    });
}

int ref_adjoint_ewp(void* h, const double* d, double* m) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        copy_out(apply_adjoint_ewp(op, make_soti(d, op.num_sensors, op.num_steps)), m);
    });
}

// Full reference spectrum, freq-major (2*nt, nd, nm) complex128 interleaved.
int ref_spectrum(void* h, double* out_c128) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        std::memcpy(out_c128, op.freq_blocks.data(),
                    sizeof(std::complex<double>) * op.freq_blocks.size());
    });
}

// stage_seconds (7 doubles: pad, fwd_fft, reorder_in, apply, reorder_out,
// inv_fft, unpad) is filled when non-null (PipelineCounters::time_stages).
static void stages_out(const PipelineCounters& c, double* s) {
    if (!s) return;
    s[0] = c.pad.seconds;
    s[1] = c.forward_fft.seconds;
    s[2] = c.reorder_in.seconds;
    s[3] = c.apply.seconds;
    s[4] = c.reorder_out.seconds;
    s[5] = c.inverse_fft.seconds;
    s[6] = c.unpad.seconds;
}

int ref_forward(void* h, const double* m, double* d, double* stage_seconds) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        PipelineCounters c;
        c.time_stages = stage_seconds != nullptr;
        copy_out(apply_forward(op, make_soti(m, op.num_sources, op.num_steps), &c), d);
        stages_out(c, stage_seconds);
    });
}

int ref_adjoint(void* h, const double* d, double* m, double* stage_seconds) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        PipelineCounters c;
        c.time_stages = stage_seconds != nullptr;
        copy_out(apply_adjoint(op, make_soti(d, op.num_sensors, op.num_steps), &c), m);
        stages_out(c, stage_seconds);
    });
}

// reg_kind: 0 = ScaledIdentity, 1 = TemporalLaplacian (inverse.hpp:16).
int ref_hessian(void* h, const double* v, double* hv, double alpha, int reg_kind) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        HessianOperator hess;
        hess.op = &op;
        hess.reg.kind = reg_kind ? RegKind::TemporalLaplacian : RegKind::ScaledIdentity;
        hess.reg.alpha = alpha;
        copy_out(hess.apply(make_soti(v, op.num_sources, op.num_steps)), hv);
    });
}

// cg_solve (inverse.cpp:105-156) on HessianOperator{op, reg}; out[0..2] =
// iterations, relative_residual, converged.
int ref_cg_solve(void* h, const double* rhs, double* x, double alpha, int reg_kind, double tol,
                 std::size_t max_iterations, int precondition, double* out) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        HessianOperator hess;
        hess.op = &op;
        hess.reg.kind = reg_kind ? RegKind::TemporalLaplacian : RegKind::ScaledIdentity;
        hess.reg.alpha = alpha;
        const CGResult r = cg_solve(hess, make_soti(rhs, op.num_sources, op.num_steps), tol, max_iterations,
                                    precondition != 0);
        copy_out(r.solution, x);
        out[0] = static_cast<double>(r.iterations);
        out[1] = r.relative_residual;
        out[2] = r.converged ? 1.0 : 0.0;
    });
}

int ref_objective(void* h, const double* m, const double* d_obs, double alpha, int reg_kind, double* value) {
    return guarded([&] {
        const SpectralP2O& op = *static_cast<SpectralP2O*>(h);
        Regularization reg;
        reg.kind = reg_kind ? RegKind::TemporalLaplacian : RegKind::ScaledIdentity;
        reg.alpha = alpha;
        *value = objective_eval(op, make_soti(m, op.num_sources, op.num_steps),
                                make_soti(d_obs, op.num_sensors, op.num_steps), reg);
    });
}

// ---- file formats (io.cpp) -----------------------------------------------------
int ref_write_compact(const char* path, const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt) {
    return guarded([&] { io::write_operator(path, make_compact(blocks, nd, nm, nt)); });
}

int ref_save_spectral(void* h, const char* path) {
    return guarded([&] { io::write_operator(path, *static_cast<SpectralP2O*>(h)); });
}

void* ref_load_spectral(const char* path) {
    SpectralP2O* op = nullptr;
    const int rc = guarded([&] { op = new SpectralP2O(io::read_spectral_operator(path)); });
    return rc == 0 ? op : nullptr;
}

int ref_write_vector(const char* path, const double* v, std::size_t dim, std::size_t nt) {
    return guarded([&] { io::write_vector(path, make_soti(v, dim, nt)); });
}

int ref_read_vector(const char* path, double* out, std::size_t capacity) {
    return guarded([&] {
        const SpaceTimeVector v = with_ordering(io::read_vector(path), Ordering::SOTI);
        if (v.values.size() > capacity) throw DimensionError("capacity");
        std::memcpy(out, v.values.data(), v.values.size() * sizeof(double));
    });
}

// ---- naive (time-domain) backend: SOTI in, SOTI out ---------------------------
int ref_naive_forward(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt,
                      const double* m, double* d) {
    return guarded([&] {
        const CompactP2O op = make_compact(blocks, nd, nm, nt);
        copy_out(naive_apply_forward(op, soti_to_tosi(make_soti(m, nm, nt))), d);
    });
}

int ref_naive_adjoint(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt,
                      const double* d, double* m) {
    return guarded([&] {
        const CompactP2O op = make_compact(blocks, nd, nm, nt);
        copy_out(naive_apply_adjoint(op, soti_to_tosi(make_soti(d, nd, nt))), m);
    });
}

// ---- distributed engine (distributed.hpp:57-121) ------------------------------
void* ref_partition(const double* blocks, std::size_t nd, std::size_t nm, std::size_t nt,
                    std::size_t rows, std::size_t cols) {
    PartitionHandle* p = nullptr;
    const int rc = guarded([&] {
        p = new PartitionHandle{
            partition_operator(make_compact(blocks, nd, nm, nt), GridShape{rows, cols})};
    });
    return rc == 0 ? p : nullptr;
}

void ref_partition_destroy(void* h) { delete static_cast<PartitionHandle*>(h); }

// Shard bounds: out[4*w + {0,1,2,3}] = sensor_begin, sensor_end, source_begin, source_end.
int ref_partition_bounds(void* h, std::size_t* out) {
    return guarded([&] {
        const Partition& part = static_cast<PartitionHandle*>(h)->partition;
        for (std::size_t w = 0; w < part.shards.size(); ++w) {
            out[4 * w + 0] = part.shards[w].sensor_begin;
            out[4 * w + 1] = part.shards[w].sensor_end;
            out[4 * w + 2] = part.shards[w].source_begin;
            out[4 * w + 3] = part.shards[w].source_end;
        }
    });
}

int ref_distributed_forward(void* h, const double* m, double* d, int parallel) {
    return guarded([&] {
        const Partition& part = static_cast<PartitionHandle*>(h)->partition;
        EngineOptions eo;
        eo.policy = parallel ? ExecutionPolicy::Parallel : ExecutionPolicy::Serial;
        copy_out(distributed_forward(part, make_soti(m, part.num_sources, part.num_steps), eo), d);
    });
}

int ref_distributed_adjoint(void* h, const double* d, double* m, int parallel) {
    return guarded([&] {
        const Partition& part = static_cast<PartitionHandle*>(h)->partition;
        EngineOptions eo;
        eo.policy = parallel ? ExecutionPolicy::Parallel : ExecutionPolicy::Serial;
        copy_out(distributed_adjoint(part, make_soti(d, part.num_sensors, part.num_steps), eo), m);
    });
}

// HessianOperator::apply's partition branch (inverse.cpp:80-85) plus the
// penalty add (:87-89); the operator pointer only has to be non-null there.
int ref_distributed_hessian(void* h, const double* v, double* hv, double alpha, int reg_kind,
                            int parallel) {
    return guarded([&] {
        const Partition& part = static_cast<PartitionHandle*>(h)->partition;
        SpectralP2O placeholder;
        HessianOperator hess;
        hess.op = &placeholder;
        hess.partition = &part;
        hess.engine.policy = parallel ? ExecutionPolicy::Parallel : ExecutionPolicy::Serial;
        hess.reg.kind = reg_kind ? RegKind::TemporalLaplacian : RegKind::ScaledIdentity;
        hess.reg.alpha = alpha;
        copy_out(hess.apply(make_soti(v, part.num_sources, part.num_steps)), hv);
    });
}

// ---- the reference's own invariant suite (verify.cpp:72-250) ------------------
int ref_verify(std::uint64_t seed, char* report, std::size_t report_len, int* passed) {
    return guarded([&] {
        std::ostringstream os;
        *passed = run_verification(os, seed) ? 1 : 0;
        const std::string s = os.str();
        if (report && report_len) {
            std::strncpy(report, s.c_str(), report_len - 1);
            report[report_len - 1] = '\0';
        }
    });
}

// ---- grid planner (grid_planner.cpp:105-207) ------------------------------------
int ref_select_grid(std::size_t workers, double log_dim_ratio, unsigned gpus_per_node, std::size_t* rc) {
    return guarded([&] {
        const GridShape g = select_grid(workers, log_dim_ratio, gpus_per_node);
        rc[0] = g.rows;
        rc[1] = g.cols;
    });
}

int ref_weak_scaling_shape(double local_ratio, std::size_t workers, std::size_t* out3) {
    return guarded([&] {
        const WeakScalingChoice c = weak_scaling_shape(local_ratio, workers);
        out3[0] = c.indifferent ? 1 : 0;
        out3[1] = c.shape.rows;
        out3[2] = c.shape.cols;
    });
}

int ref_modified_cost(double rows, std::size_t workers, double log_dim_ratio, double* out) {
    return guarded([&] { *out = modified_cost(rows, workers, log_dim_ratio); });
}

int ref_comm_cost(std::size_t rows, std::size_t cols, std::size_t nsrc, std::size_t nsens, std::size_t nt,
                  double latency, double bandwidth, double* out) {
    return guarded([&] {
        CostParams p;
        p.latency = latency;
        p.bandwidth = bandwidth;
        ProblemDims d;
        d.num_sources = nsrc;
        d.num_sensors = nsens;
        d.num_steps = nt;
        *out = comm_cost(GridShape{rows, cols}, d, p);
    });
}

// ---- partition of an operator already in frequency form (distributed.cpp:198-218)
void* ref_partition_spectral(void* h, std::size_t rows, std::size_t cols) {
    PartitionHandle* p = nullptr;
    const int rc = guarded([&] {
        p = new PartitionHandle{partition_operator(*static_cast<SpectralP2O*>(h), GridShape{rows, cols})};
    });
    return rc == 0 ? p : nullptr;
}

// Shard (r, c)'s frequency blocks in the reference's full 2N_t layout.
int ref_partition_shard_spectrum(void* h, std::size_t r, std::size_t c, double* out_c128) {
    return guarded([&] {
        const Partition& part = static_cast<PartitionHandle*>(h)->partition;
        const SpectralP2O& s = part.shard(r, c).spectral;
        std::memcpy(out_c128, s.freq_blocks.data(), sizeof(std::complex<double>) * s.freq_blocks.size());
    });
}

}  // extern "C"
