// Processor-grid planner (grid_planner.hpp:43-65, grid_planner.cpp:105-207).
//
// Host-only arithmetic behind the C ABI: the modified-cost model the reference
// minimises, its integer snap (exact minimiser for one GPU per node, the
// node-divisibility preference otherwise), the weak-scaling degenerate choice
// and the per-matvec communication model. On one NVSwitch node (k = 8 B200s)
// every peer is one hop at full bandwidth, so the model only has to decide the
// orientation of the r x c grid; GridEngine (distributed.py) consumes the pick.
#include <cmath>
#include <cstddef>
#include <limits>
#include <vector>

#include "../../include/btg.h"

extern "C" btg_status btg_internal_fail(btg_status s, const char* msg);  // btg_capi.cu

namespace {

struct Shape {
    size_t rows, cols;
};

// (r/p) ln r + (10^l / r) ln(p/r)   (grid_planner.hpp:49-52)
double mcost(double r, size_t workers, double l) {
    const double p = (double)workers;
    return (r / p) * std::log(r) + (std::pow(10.0, l) / r) * std::log(p / r);
}

// Golden-section search for the continuous minimiser on [1, p].
double golden_argmin(size_t workers, double l) {
    double a = 1.0, b = (double)workers;
    if (b <= a) return a;
    const double g = 0.5 * (std::sqrt(5.0) - 1.0);
    double x1 = b - g * (b - a), x2 = a + g * (b - a);
    double f1 = mcost(x1, workers, l), f2 = mcost(x2, workers, l);
    for (int it = 0; it < 200 && b - a > 1e-10 * b; ++it) {
        if (f1 < f2) {  // minimum in [a, x2]
            b = x2;
            x2 = x1;
            f2 = f1;
            x1 = b - g * (b - a);
            f1 = mcost(x1, workers, l);
        } else {  // minimum in [x1, b]
            a = x1;
            x1 = x2;
            f1 = f2;
            x2 = a + g * (b - a);
            f2 = mcost(x2, workers, l);
        }
    }
    return 0.5 * (a + b);
}

std::vector<Shape> divisor_grids(size_t workers) {  // rows ascending
    std::vector<Shape> lo, hi;
    for (size_t r = 1; r * r <= workers; ++r)
        if (workers % r == 0) {
            lo.push_back({r, workers / r});
            if (r != workers / r) hi.push_back({workers / r, r});
        }
    for (size_t k = hi.size(); k-- > 0;) lo.push_back(hi[k]);
    return lo;
}

}  // namespace

extern "C" {

btg_status btg_modified_cost(double rows, size_t workers, double log_dim_ratio, double* out) {
    if (!out) return btg_internal_fail(BTG_EARG, "null output");
    if (rows < 1.0 || rows > (double)workers)
        return btg_internal_fail(BTG_EARG, "modified cost: rows must lie in [1, workers]");
    *out = mcost(rows, workers, log_dim_ratio);
    return BTG_OK;
}

btg_status btg_comm_cost(size_t rows, size_t cols, size_t num_sources, size_t num_sensors, size_t num_steps,
                         double latency, double bandwidth, double* out) {
    if (!out) return btg_internal_fail(BTG_EARG, "null output");
    if (latency < 0.0) return btg_internal_fail(BTG_EARG, "cost params: latency must be non-negative");
    if (bandwidth <= 0.0) return btg_internal_fail(BTG_EARG, "cost params: bandwidth must be positive");
    const double t = (double)num_steps;
    const double r = (double)rows, c = (double)cols;
    // column broadcast of m (depth ~ ln r) + row reduce of d (depth ~ ln c)
    *out = (latency + 8.0 * t * (double)num_sources / (bandwidth * c)) * std::log(r) +
           (latency + 8.0 * t * (double)num_sensors / (bandwidth * r)) * std::log(c);
    return BTG_OK;
}

// conventional_cost_estimate (grid_planner.cpp:282-299): conventional
// (solve-based) vs FFT-based Hessian cost model of the paper's Table 1.
btg_status btg_conventional_cost_estimate(double grid_points, double num_steps, double num_sensors,
                                          double rank_fraction, btg_cost_estimate* out) {
    if (!out) return btg_internal_fail(BTG_EARG, "null output");
    if (grid_points <= 0.0 || num_steps <= 0.0 || num_sensors <= 0.0 || rank_fraction <= 0.0)
        return btg_internal_fail(BTG_EARG, "cost estimate: all inputs must be positive");
    const double state_dim = 3.0 * grid_points;  // 3 values per grid point
    out->per_solve_flops = 324.0 * state_dim * num_steps;
    out->effective_rank = num_sensors * num_steps * rank_fraction;
    out->conventional_total_flops = 2.0 * out->effective_rank * out->per_solve_flops;
    const double num_sources = std::pow(grid_points, 2.0 / 3.0);  // surface field
    out->fft_setup_flops = num_sensors * out->per_solve_flops;
    out->fft_matvec_flops = 2.0 * out->effective_rank * 8.0 * num_sources * num_sensors * num_steps;
    out->fft_total_flops = out->fft_setup_flops + out->fft_matvec_flops;
    out->ratio = out->conventional_total_flops / out->fft_total_flops;
    return BTG_OK;
}

// apply_arithmetic_intensity (grid_planner.cpp:301-304): flop/byte of the
// Fourier-space step on an n_d x n_m shard.
double btg_apply_arithmetic_intensity(double local_sensors, double local_sources) {
    const double prod = local_sensors * local_sources;
    return prod / (2.0 * (prod + local_sources + local_sensors));
}

btg_status btg_select_grid(size_t workers, double log_dim_ratio, unsigned gpus_per_node, size_t* rows,
                           size_t* cols) {
    if (!rows || !cols) return btg_internal_fail(BTG_EARG, "null output");
    if (workers == 0) return btg_internal_fail(BTG_EARG, "select_grid: workers must be positive");
    if (gpus_per_node < 1) return btg_internal_fail(BTG_EARG, "select_grid: gpus per node must be at least 1");
    auto put = [&](size_t r, size_t c) {
        *rows = r;
        *cols = c;
        return BTG_OK;
    };
    if (workers == 1) return put(1, 1);
    const double p = (double)workers;
    const double t = golden_argmin(workers, log_dim_ratio);
    if (t <= 1.0 + 1e-6) return put(1, workers);
    if (t >= p * (1.0 - 1e-6)) return put(workers, 1);

    const std::vector<Shape> grids = divisor_grids(workers);
    const bool tall = log_dim_ratio >= 0.0;  // more sensors than sources: rows >= cols
    auto oriented = [&](const Shape& g) { return tall ? g.rows >= g.cols : g.rows < g.cols; };
    auto dist = [&](const Shape& g) { return std::fabs((double)g.rows - t); };
    auto cost = [&](const Shape& g) { return mcost((double)g.rows, workers, log_dim_ratio); };

    if (gpus_per_node == 1) {
        // exact integer minimiser; among (relative 1e-12) ties: oriented first,
        // then nearest the continuous optimum, then fewer rows
        double best = std::numeric_limits<double>::infinity();
        for (const Shape& g : grids) best = std::fmin(best, cost(g));
        const Shape* pick = nullptr;
        for (const Shape& g : grids) {
            if (cost(g) > best * (1.0 + 1e-12) + 1e-300) continue;
            if (!pick) {
                pick = &g;
            } else if (oriented(g) != oriented(*pick)) {
                if (oriented(g)) pick = &g;
            } else if (dist(g) < dist(*pick)) {
                pick = &g;
            }
        }
        return put(pick->rows, pick->cols);
    }

    // several GPUs per node: keep the orientation, prefer row counts that are
    // multiples of the node size, then column counts, then anything; nearest
    // the continuous optimum within a class (cost breaks exact distance ties)
    std::vector<Shape> cand;
    for (const Shape& g : grids)
        if (oriented(g)) cand.push_back(g);
    if (cand.empty()) return tall ? put(workers, 1) : put(1, workers);
    const size_t k = gpus_per_node;
    for (int cls = 0; cls < 3; ++cls) {
        const Shape* pick = nullptr;
        for (const Shape& g : cand) {
            const bool keep = cls == 0 ? g.rows % k == 0 : cls == 1 ? g.cols % k == 0 : true;
            if (!keep) continue;
            if (!pick || dist(g) < dist(*pick) || (dist(g) == dist(*pick) && cost(g) < cost(*pick))) pick = &g;
        }
        if (pick) return put(pick->rows, pick->cols);
    }
    return put(1, workers);  // unreachable: class 2 keeps every candidate
}

btg_status btg_weak_scaling_shape(double local_ratio, size_t workers, int* indifferent, size_t* rows,
                                  size_t* cols) {
    if (!indifferent || !rows || !cols) return btg_internal_fail(BTG_EARG, "null output");
    if (!(local_ratio > 0.0)) return btg_internal_fail(BTG_EARG, "weak_scaling_shape: local ratio must be positive");
    // cost ~ (1 - ratio) log(rows): rows = 1 unless the local block is taller than wide
    *indifferent = local_ratio == 1.0;
    *rows = local_ratio > 1.0 ? workers : 1;
    *cols = local_ratio > 1.0 ? 1 : workers;
    return BTG_OK;
}

}  // extern "C"
