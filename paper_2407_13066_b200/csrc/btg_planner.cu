// Processor-grid planning for one NVSwitch domain of B200s.
//
// Two planners behind the C ABI:
//
// * btg_plan_grid — the B200 planner. It costs the grid engine's own schedule
//   (btg_grid_engine.cu) for every r x c factorisation of the worker count:
//   the shard's HBM stream (F-hat + vectors), the vector transforms (whose
//   input side is replicated down a column or along a row), and the NCCL ring
//   collectives of the action — column broadcast / row reduce (F), row
//   broadcast / column reduce (F*), column broadcast + row all-reduce + column
//   reduce (Hessian) — with NVLink-5 bandwidth inside the NVSwitch domain and
//   the inter-node link outside it. Exhaustive over the factor pairs.
//
// * btg_select_grid — the reference's scale-free criterion
//   (grid_planner.hpp:43-65): the rows r minimising (r/p) ln r + (10^l/r) ln(p/r),
//   l = log10(N_d/N_m), snapped to a factorisation of p with the reference's
//   preferences (orientation, node divisibility). Its continuous optimum is
//   taken here as the unique root of the cost's derivative (bisection on
//   r^2 (ln r + 1) - p 10^l (1 + ln(p/r)), which is increasing in r), and the
//   snap as a lexicographic minimum over the factor pairs; tests compare every
//   answer with the reference build (tests/test_planner.py).
//
// The cost formulas the reference defines as its API (modified_cost, comm_cost,
// conventional_cost_estimate, apply_arithmetic_intensity) are evaluated as
// stated (grid_planner.cpp:105-121, 282-304).
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <limits>
#include <tuple>
#include <vector>

#include "../../include/btg.h"

extern "C" btg_status btg_internal_fail(btg_status s, const char* msg);  // btg_capi.cu

namespace {

btg_status pfail(btg_status s, const char* m) { return btg_internal_fail(s, m); }

// (r/p) ln r + (10^l / r) ln(p/r)   (grid_planner.hpp:49-52)
double scale_free_cost(double r, double p, double l) {
    return (r / p) * std::log(r) + (std::pow(10.0, l) / r) * std::log(p / r);
}

// The continuous minimiser of scale_free_cost on [1, p]: p r^2 f'(r) =
// r^2 (ln r + 1) - p L (1 + ln p - ln r) is increasing in r, so its sign change
// (if any) is the unique stationary point; otherwise the optimum is an end point.
double continuous_optimum(double p, double l) {
    const double L = std::pow(10.0, l);
    auto g = [&](double r) { return r * r * (std::log(r) + 1.0) - p * L * (1.0 + std::log(p) - std::log(r)); };
    if (p <= 1.0 || g(1.0) >= 0.0) return 1.0;
    if (g(p) <= 0.0) return p;
    double lo = 1.0, hi = p;
    for (int it = 0; it < 200 && hi - lo > 1e-15 * hi; ++it) {
        const double mid = 0.5 * (lo + hi);
        (g(mid) < 0.0 ? lo : hi) = mid;
    }
    return 0.5 * (lo + hi);
}

std::vector<std::pair<size_t, size_t>> factorisations(size_t p) {
    std::vector<std::pair<size_t, size_t>> out;
    for (size_t r = 1; r <= p; ++r)
        if (p % r == 0) out.emplace_back(r, p / r);
    return out;  // rows ascending
}

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// NCCL ring collectives over k members: a pipelined ring moves (k-1)/k of the
// payload per link for broadcast and reduce, twice that for all-reduce, and
// pays one latency per ring step.
double ring_seconds(int kind /*0 bcast, 1 reduce, 2 allreduce*/, size_t k, double bytes, double gbs, double lat_s) {
    if (k <= 1 || bytes <= 0.0) return 0.0;
    const double frac = (double)(k - 1) / (double)k;
    const double passes = kind == 2 ? 2.0 : 1.0;
    return passes * (frac * bytes / (gbs * 1e9) + (double)(k - 1) * lat_s);
}

btg_hw_model default_hw() {
    btg_hw_model h{};
    h.hbm_gbs = 7000.0;       // measured GEMV stream on B200 (profiles/)
    h.fft_gbs = 4000.0;       // measured vector-FFT rate at the configs' lengths
    h.link_gbs = 900.0;       // NVLink 5 per direction per GPU, uniform through NVSwitch
    h.node_link_gbs = 50.0;   // one 400 Gb/s NIC per GPU between NVSwitch domains
    h.latency_us = 3.0;       // per ring step
    h.gpus_per_node = 8;
    return h;
}

// Cost of one action on an r x c grid (the worst shard: ceiling partition).
btg_grid_plan cost_plan(size_t nd, size_t nm, size_t nt, size_t r, size_t c, int precision, int kind,
                        const btg_hw_model& hw) {
    btg_grid_plan pl{};
    pl.rows = r;
    pl.cols = c;
    const double ld = (double)std::min(ceil_div(nd, r), nd), lm = (double)std::min(ceil_div(nm, c), nm);
    const double nf = (double)nt + 1.0, t = (double)nt;
    const double s = precision == BTG_F32 ? 8.0 : 16.0;
    const double gemv = s * nf * ld * lm + 16.0 * nf * (ld + lm);
    auto fft = [&](double ch) { return 8.0 * ch * t + 16.0 * nf * ch; };  // R2C or C2R of ch channels
    double hbm = 0.0, fb = 0.0;
    if (kind == BTG_GRID_FORWARD) {
        hbm = gemv;
        fb = fft(lm) + fft(ld);
    } else if (kind == BTG_GRID_ADJOINT) {
        hbm = gemv;
        fb = fft(ld) + fft(lm);
    } else {
        hbm = 2.0 * gemv;
        fb = 2.0 * (fft(lm) + fft(ld));
    }
    pl.local_seconds = hbm / (hw.hbm_gbs * 1e9) + fb / (hw.fft_gbs * 1e9);
    // a row group is c consecutive ranks, a column group r ranks strided by c: a
    // group stays inside one NVSwitch domain when its span of ranks does
    const size_t node = std::max(1u, hw.gpus_per_node);
    const bool row_local = c <= node && node % c == 0;
    const bool col_local = r * c <= node;
    const double lat = hw.latency_us * 1e-6;
    const double row_bw = row_local ? hw.link_gbs : hw.node_link_gbs;
    const double col_bw = col_local ? hw.link_gbs : hw.node_link_gbs;
    const double pbytes = 8.0 * t * lm, dbytes = 8.0 * t * ld;
    double comm = 0.0;
    if (kind == BTG_GRID_FORWARD) {
        comm = ring_seconds(0, r, pbytes, col_bw, lat) + ring_seconds(1, c, dbytes, row_bw, lat);
    } else if (kind == BTG_GRID_ADJOINT) {
        comm = ring_seconds(0, c, dbytes, row_bw, lat) + ring_seconds(1, r, pbytes, col_bw, lat);
    } else {
        comm = ring_seconds(0, r, pbytes, col_bw, lat) + ring_seconds(2, c, dbytes, row_bw, lat) +
               ring_seconds(1, r, pbytes, col_bw, lat);
    }
    pl.comm_seconds = comm;
    pl.seconds = pl.local_seconds + pl.comm_seconds;
    return pl;
}

}  // namespace

extern "C" {

btg_status btg_default_hw_model(btg_hw_model* out) {
    if (!out) return pfail(BTG_EARG, "null output");
    *out = default_hw();
    return BTG_OK;
}

btg_status btg_plan_grid(size_t nd, size_t nm, size_t nt, size_t workers, int precision, int kind,
                         const btg_hw_model* hw, btg_grid_plan* best, btg_grid_plan* all, size_t cap, size_t* count) {
    if (workers == 0) return pfail(BTG_EARG, "plan_grid: workers must be positive");
    if (nd == 0 || nm == 0 || nt == 0) return pfail(BTG_EDIM, "plan_grid: all dimensions must be positive");
    if (precision != BTG_F64 && precision != BTG_F32) return pfail(BTG_EARG, "plan_grid: precision must be 64 or 32");
    if (kind < BTG_GRID_FORWARD || kind > BTG_GRID_HESSIAN) return pfail(BTG_EARG, "plan_grid: unknown action");
    const btg_hw_model h = hw ? *hw : default_hw();
    if (!(h.hbm_gbs > 0.0) || !(h.fft_gbs > 0.0) || !(h.link_gbs > 0.0) || !(h.node_link_gbs > 0.0) ||
        h.latency_us < 0.0)
        return pfail(BTG_EARG, "plan_grid: hardware rates must be positive");
    std::vector<btg_grid_plan> plans;
    for (const auto& [r, c] : factorisations(workers))
        if (r <= nd && c <= nm) plans.push_back(cost_plan(nd, nm, nt, r, c, precision, kind, h));
    if (plans.empty()) return pfail(BTG_EGRID, "plan_grid: no grid of that many workers fits the operator");
    if (count) *count = plans.size();
    if (all) {
        if (cap < plans.size()) return pfail(BTG_EARG, "plan_grid: capacity too small");
        std::copy(plans.begin(), plans.end(), all);
    }
    if (best)  // cheapest; ties (1e-12 relative) to fewer rows
        *best = *std::min_element(plans.begin(), plans.end(), [](const btg_grid_plan& a, const btg_grid_plan& b) {
            if (std::fabs(a.seconds - b.seconds) > 1e-12 * std::max(a.seconds, b.seconds)) return a.seconds < b.seconds;
            return a.rows < b.rows;
        });
    return BTG_OK;
}

btg_status btg_modified_cost(double rows, size_t workers, double log_dim_ratio, double* out) {
    if (!out) return pfail(BTG_EARG, "null output");
    if (rows < 1.0 || rows > (double)workers) return pfail(BTG_EARG, "modified cost: rows must lie in [1, workers]");
    *out = scale_free_cost(rows, (double)workers, log_dim_ratio);
    return BTG_OK;
}

// comm_cost (grid_planner.cpp:105-114): broadcast of the parameter slice over
// ln r levels plus the data-slice reduce over ln c levels, per F + F* pair.
btg_status btg_comm_cost(size_t rows, size_t cols, size_t num_sources, size_t num_sensors, size_t num_steps,
                         double latency, double bandwidth, double* out) {
    if (!out) return pfail(BTG_EARG, "null output");
    if (latency < 0.0) return pfail(BTG_EARG, "cost params: latency must be non-negative");
    if (bandwidth <= 0.0) return pfail(BTG_EARG, "cost params: bandwidth must be positive");
    const double t = (double)num_steps, r = (double)rows, c = (double)cols;
    const double param_hop = latency + 8.0 * t * (double)num_sources / (bandwidth * c);
    const double data_hop = latency + 8.0 * t * (double)num_sensors / (bandwidth * r);
    *out = param_hop * std::log(r) + data_hop * std::log(c);
    return BTG_OK;
}

// conventional_cost_estimate (grid_planner.cpp:282-299): the paper's Table 1
// model of solve-based vs FFT-based Hessian construction.
btg_status btg_conventional_cost_estimate(double grid_points, double num_steps, double num_sensors,
                                          double rank_fraction, btg_cost_estimate* out) {
    if (!out) return pfail(BTG_EARG, "null output");
    if (grid_points <= 0.0 || num_steps <= 0.0 || num_sensors <= 0.0 || rank_fraction <= 0.0)
        return pfail(BTG_EARG, "cost estimate: all inputs must be positive");
    btg_cost_estimate e{};
    const double state = 3.0 * grid_points;
    e.per_solve_flops = 324.0 * state * num_steps;
    e.effective_rank = num_sensors * num_steps * rank_fraction;
    e.conventional_total_flops = 2.0 * e.effective_rank * e.per_solve_flops;
    const double sources = std::pow(grid_points, 2.0 / 3.0);
    e.fft_setup_flops = num_sensors * e.per_solve_flops;
    e.fft_matvec_flops = 16.0 * e.effective_rank * sources * num_sensors * num_steps;
    e.fft_total_flops = e.fft_setup_flops + e.fft_matvec_flops;
    e.ratio = e.conventional_total_flops / e.fft_total_flops;
    *out = e;
    return BTG_OK;
}

// apply_arithmetic_intensity (grid_planner.cpp:301-304)
double btg_apply_arithmetic_intensity(double local_sensors, double local_sources) {
    const double prod = local_sensors * local_sources;
    return prod / (2.0 * (prod + local_sources + local_sensors));
}

btg_status btg_select_grid(size_t workers, double log_dim_ratio, unsigned gpus_per_node, size_t* rows, size_t* cols) {
    if (!rows || !cols) return pfail(BTG_EARG, "null output");
    if (workers == 0) return pfail(BTG_EARG, "select_grid: workers must be positive");
    if (gpus_per_node < 1) return pfail(BTG_EARG, "select_grid: gpus per node must be at least 1");
    const double p = (double)workers;
    const double target = continuous_optimum(p, log_dim_ratio);
    size_t r = 1;
    if (workers == 1 || target <= 1.0 + 1e-6) {
        r = 1;
    } else if (target >= p * (1.0 - 1e-6)) {
        r = workers;
    } else {
        const bool tall = log_dim_ratio >= 0.0;  // more sensors than sources: rows >= cols wanted
        struct Cand {
            size_t r, c;
            double cost, dist;
            bool oriented;
        };
        std::vector<Cand> cands;
        for (const auto& [rr, cc] : factorisations(workers))
            cands.push_back({rr, cc, scale_free_cost((double)rr, p, log_dim_ratio), std::fabs((double)rr - target),
                             tall ? rr >= cc : rr < cc});
        if (gpus_per_node == 1) {
            // the integer minimiser; among cost ties (1e-12 relative): oriented,
            // then nearest the continuous optimum, then fewer rows
            const double best = std::min_element(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
                                    return a.cost < b.cost;
                                })->cost;
            auto key = [&](const Cand& a) {
                return std::make_tuple(a.cost > best * (1.0 + 1e-12) + 1e-300, !a.oriented, a.dist, a.r);
            };
            r = std::min_element(cands.begin(), cands.end(),
                                 [&](const Cand& a, const Cand& b) { return key(a) < key(b); })
                    ->r;
        } else {
            // keep the orientation; prefer rows divisible by the node size (column
            // traffic on-node), then columns, then any; nearest the optimum, then cheaper
            const size_t k = gpus_per_node;
            auto cls = [&](const Cand& a) { return a.r % k == 0 ? 0 : a.c % k == 0 ? 1 : 2; };
            auto key = [&](const Cand& a) { return std::make_tuple(cls(a), a.dist, a.cost); };
            const Cand* pick = nullptr;
            for (const Cand& a : cands)
                if (a.oriented && (!pick || key(a) < key(*pick))) pick = &a;
            r = pick ? pick->r : (tall ? workers : 1);
        }
    }
    *rows = r;
    *cols = workers / r;
    return BTG_OK;
}

// weak_scaling_shape (grid_planner.cpp:195-207): with a fixed local block the
// traffic per rank only depends on the orientation — all rows when the block is
// taller than wide, all columns otherwise (indifferent when square).
btg_status btg_weak_scaling_shape(double local_ratio, size_t workers, int* indifferent, size_t* rows,
                                  size_t* cols) {
    if (!indifferent || !rows || !cols) return pfail(BTG_EARG, "null output");
    if (!(local_ratio > 0.0)) return pfail(BTG_EARG, "weak_scaling_shape: local ratio must be positive");
    *indifferent = local_ratio == 1.0;
    *rows = local_ratio > 1.0 ? workers : 1;
    *cols = local_ratio > 1.0 ? 1 : workers;
    return BTG_OK;
}

}  // extern "C"
