// A reference-style C++ caller compiled against include/btoep_gpu.hpp and
// linked with libbtg.so (instead of the reference's btoep_core + FFTW). The
// statements mirror the reference's own tests (test_block_operator.cpp:88-115,
// test_inverse.cpp:81-98): identity and shift operators, typed errors, the
// Hessian of the zero operator, and CG.
#include <cmath>
#include <cstdio>

#include "btoep_gpu.hpp"

using namespace btoep;

static int failures = 0;
#define CHECK(cond)                                              \
    do {                                                         \
        if (!(cond)) {                                           \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                          \
        }                                                        \
    } while (0)

int main() {
    // identity-block operator acts as the identity
    CompactP2O eye = CompactP2O::zeros(3, 3, 8);
    for (std::size_t i = 0; i < 3; ++i) eye.entry(0, i, i) = 1.0;
    SpectralP2O op = setup(eye);
    SpaceTimeVector m = SpaceTimeVector::zeros(3, 8, Ordering::SOTI);
    for (std::size_t k = 0; k < m.values.size(); ++k) m.values[k] = std::sin(0.3 * k);
    PipelineCounters counters;
    counters.time_stages = true;
    SpaceTimeVector d = apply_forward(op, m, &counters);
    for (std::size_t k = 0; k < m.values.size(); ++k) CHECK(std::abs(d.values[k] - m.values[k]) < 1e-12);
    CHECK(counters.apply.ops > 0.0 && counters.apply.seconds > 0.0);
    SpaceTimeVector a = apply_adjoint(op, m);
    for (std::size_t k = 0; k < m.values.size(); ++k) CHECK(std::abs(a.values[k] - m.values[k]) < 1e-12);
    CHECK(op.num_freq() == 16);
    CHECK(op.freq_blocks().size() == 16 * 9);

    // shift delays the input
    CompactP2O sh = CompactP2O::zeros(2, 2, 6);
    for (std::size_t i = 0; i < 2; ++i) sh.entry(1, i, i) = 1.0;
    SpectralP2O sop = setup(sh);
    SpaceTimeVector v = SpaceTimeVector::zeros(2, 6, Ordering::SOTI);
    for (std::size_t k = 0; k < v.values.size(); ++k) v.values[k] = 1.0 + k;
    SpaceTimeVector dv = apply_forward(sop, v);
    for (std::size_t s = 0; s < 2; ++s) {
        CHECK(std::abs(dv.at(s, 0)) < 1e-12);
        for (std::size_t t = 1; t < 6; ++t) CHECK(std::abs(dv.at(s, t) - v.at(s, t - 1)) < 1e-12);
    }

    // EWP backend: needs keep_channel_layout, then agrees with the FFT backend
    bool threw = false;
    CHECK(!sop.has_channel_layout());
    try {
        apply_forward_ewp(sop, v);
    } catch (const Error&) {
        threw = true;
    }
    CHECK(threw);
    SetupOptions keep;
    keep.keep_channel_layout = true;
    SpectralP2O eop = setup(sh, keep);
    CHECK(eop.has_channel_layout());
    SpaceTimeVector de = apply_forward_ewp(eop, v);
    for (std::size_t k = 0; k < de.values.size(); ++k) CHECK(std::abs(de.values[k] - dv.values[k]) < 1e-12);
    SpaceTimeVector ae = apply_adjoint_ewp(eop, dv);
    SpaceTimeVector af = apply_adjoint(sop, dv);
    for (std::size_t k = 0; k < ae.values.size(); ++k) CHECK(std::abs(ae.values[k] - af.values[k]) < 1e-12);

    // typed errors
    threw = false;
    try {
        apply_forward(op, SpaceTimeVector::zeros(4, 8, Ordering::SOTI));
    } catch (const DimensionError&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        apply_forward(op, SpaceTimeVector::zeros(3, 8, Ordering::TOSI));
    } catch (const OrderingError&) {
        threw = true;
    }
    CHECK(threw);

    // zero operator with identity regularization scales by alpha (test_inverse.cpp:88-97)
    SpectralP2O zop = setup(CompactP2O::zeros(2, 3, 4));
    HessianOperator h{&zop, {RegKind::ScaledIdentity, 0.25}};
    SpaceTimeVector w = SpaceTimeVector::zeros(3, 4, Ordering::SOTI);
    for (std::size_t k = 0; k < w.values.size(); ++k) w.values[k] = 0.1 * k - 0.3;
    SpaceTimeVector hw = h.apply(w);
    for (std::size_t k = 0; k < w.values.size(); ++k) CHECK(std::abs(hw.values[k] - 0.25 * w.values[k]) < 1e-14);

    // CG on the identity operator: (I + alpha I) x = b
    HessianOperator hi{&op, {RegKind::ScaledIdentity, 1.0}};
    CGResult r = cg_solve(hi, m, 1e-12, 50, false);
    CHECK(r.converged);
    for (std::size_t k = 0; k < m.values.size(); ++k) CHECK(std::abs(r.solution.values[k] - 0.5 * m.values[k]) < 1e-12);

    // grid planner (test_grid_planner.cpp:93-99) and a spectral shard (distributed.cpp:198-218)
    CHECK((select_grid(80, -2.0, 4) == GridShape{4, 20}));
    CHECK((select_grid(48, -3.0, 1) == GridShape{1, 48}));
    CHECK(weak_scaling_shape(1.0, 4).indifferent);
    SpectralP2O part = slice(op, 1, 3, 0, 2);
    CHECK(part.num_sensors == 2 && part.num_sources == 2 && part.num_steps == 8);
    SpaceTimeVector m2 = SpaceTimeVector::zeros(2, 8, Ordering::SOTI);
    for (std::size_t k = 0; k < m2.values.size(); ++k) m2.values[k] = std::cos(0.7 * k);
    SpaceTimeVector d2 = apply_forward(part, m2);  // identity rows 1,2 x cols 0,1: d2[0] = m2[1], d2[1] = 0
    for (std::size_t t = 0; t < 8; ++t) {
        CHECK(std::abs(d2.at(0, t) - m2.at(1, t)) < 1e-12);
        CHECK(std::abs(d2.at(1, t)) < 1e-12);
    }

    // single-process partition (distributed.hpp): 2 x 1 grid of the shift operator
    {
        GridShape g2;
        g2.rows = 2;
        Partition pp = partition_operator(sh, g2);
        SpaceTimeVector dp = distributed_forward(pp, v);
        for (std::size_t k = 0; k < dp.values.size(); ++k) CHECK(std::abs(dp.values[k] - dv.values[k]) < 1e-12);
        EngineOptions par;
        par.policy = ExecutionPolicy::Parallel;
        SpaceTimeVector ap = distributed_adjoint(pp, dv, par);
        SpaceTimeVector af2 = apply_adjoint(sop, dv);
        for (std::size_t k = 0; k < ap.values.size(); ++k) CHECK(std::abs(ap.values[k] - af2.values[k]) < 1e-12);
        CHECK(pp.shard_bounds(1, 0)[0] == 1);
        // HessianOperator on the partition (inverse.cpp:80-85) equals the fused device Hessian
        HessianOperator hp{&sop, {RegKind::TemporalLaplacian, 0.3}};
        HessianOperator hd = hp;
        hp.partition = &pp;
        SpaceTimeVector x1 = hp.apply(v), x2 = hd.apply(v);
        for (std::size_t k = 0; k < x1.values.size(); ++k) CHECK(std::abs(x1.values[k] - x2.values[k]) < 1e-12);
    }
    // CommLog byte model (test_distributed.cpp:139-186)
    {
        const std::size_t steps = 16;
        auto rnd_op = [&](std::size_t nd_, std::size_t nm_) {
            CompactP2O c = CompactP2O::zeros(nd_, nm_, steps);
            for (std::size_t k = 0; k < c.blocks.size(); ++k) c.blocks[k] = std::sin(0.7 * k);
            return c;
        };
        CommLog l1;
        Partition p11 = partition_operator(rnd_op(3, 4), GridShape{1, 1});
        distributed_forward(p11, SpaceTimeVector::zeros(4, steps, Ordering::SOTI), {}, &l1);
        CHECK(l1.total_bytes() == 0 && l1.total_messages() == 0);
        CommLog l2;
        Partition p14 = partition_operator(rnd_op(3, 8), GridShape{1, 4});
        distributed_forward(p14, SpaceTimeVector::zeros(8, steps, Ordering::SOTI), {}, &l2);
        std::uint64_t rb = 0;
        std::size_t rm = 0;
        for (const CommEvent& e : l2.events) {
            if (e.phase == "broadcast") CHECK(e.total_bytes == 0);
            if (e.phase != "reduce") continue;
            CHECK(e.link_bytes == 8 * steps * 3);
            rb += e.total_bytes;
            rm += e.messages;
        }
        CHECK(rm == 3 && rb == 3 * 8 * steps * 3);
        CommLog l3;
        Partition p22 = partition_operator(rnd_op(4, 6), GridShape{2, 2});
        distributed_forward(p22, SpaceTimeVector::zeros(6, steps, Ordering::SOTI), {}, &l3);
        CHECK(l3.total_bytes() == 2 * 1 * 8 * steps * 3 + 2 * 1 * 8 * steps * 2);
    }

    // multi-process NCCL grid (btg_grid_*): world size 1 here (one GPU per
    // box); every rank of a real job runs the same lines with its own rank and rectangle
    {
        const std::size_t nd = 3, nm = 5, nt = 12;
        CompactP2O c = CompactP2O::zeros(nd, nm, nt);
        for (std::size_t k = 0; k < c.blocks.size(); ++k) c.blocks[k] = std::cos(0.37 * k);
        SpectralP2O full = setup(c);
        const Grid::Id id = Grid::nccl_id();
        Grid grid(GridShape{1, 1}, 0, id, 0, nd, nm, nt);
        grid.setup(c);
        SpaceTimeVector mv = SpaceTimeVector::zeros(nm, nt, Ordering::SOTI);
        SpaceTimeVector dvv = SpaceTimeVector::zeros(nd, nt, Ordering::SOTI);
        for (std::size_t k = 0; k < mv.values.size(); ++k) mv.values[k] = std::sin(0.11 * k);
        for (std::size_t k = 0; k < dvv.values.size(); ++k) dvv.values[k] = std::cos(0.23 * k);
        auto gf = grid.forward(&mv);
        auto ga = grid.adjoint(&dvv);
        std::vector<double> gam(nd, 1.5);
        auto gh = grid.hessian(&mv, Regularization{RegKind::TemporalLaplacian, 0.2}, gam);
        CHECK(gf && ga && gh);
        SpaceTimeVector wf = apply_forward(full, mv), wa = apply_adjoint(full, dvv);
        HessianOperator hw{&full, {RegKind::TemporalLaplacian, 0.2}};
        hw.gamma_inv = gam;
        SpaceTimeVector wh = hw.apply(mv);
        for (std::size_t k = 0; k < wf.values.size(); ++k) CHECK(std::abs(gf->values[k] - wf.values[k]) < 1e-12);
        for (std::size_t k = 0; k < wa.values.size(); ++k) CHECK(std::abs(ga->values[k] - wa.values[k]) < 1e-12);
        for (std::size_t k = 0; k < wh.values.size(); ++k) CHECK(std::abs(gh->values[k] - wh.values[k]) < 1e-11);
        bool threw = false;
        try {
            grid.forward(nullptr);  // rank 0 owns the parameter slice
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
    }

    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
