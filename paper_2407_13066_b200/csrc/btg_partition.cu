// Single-process partition over the visible GPUs: the C-ABI form of the
// reference's Partition / distributed_forward / distributed_adjoint
// (distributed.hpp:43-121, distributed.cpp:145-392). One device handle per
// non-empty grid cell, placed round-robin on the caller's device list; the
// partial data (F) / parameter (F*) slices come back to the host and are summed
// with the reference's fixed binary tree (tree_reduce, distributed.cpp:36-47),
// so serial and parallel execution give bit-identical results. (The
// multi-process NCCL engine is paper_2407_13066_b200/distributed.py.)
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/btg.h"

extern "C" btg_status btg_internal_fail(btg_status s, const char* msg);

struct btg_partition_s {
    size_t nd = 0, nm = 0, nt = 0, rows = 0, cols = 0;
    struct Shard {
        size_t i0 = 0, i1 = 0, j0 = 0, j1 = 0;
        btg_op op = nullptr;
        std::vector<double> blocks;  // compact shard (naive backend; partitions of compact operators only)
        bool empty() const { return i1 == i0 || j1 == j0; }
    };
    std::vector<Shard> shards;  // row-major
    bool has_compact = false;
    bool channel_layout = false;
    std::vector<int> devices;
};

namespace {

btg_status pfail(btg_status s, const std::string& m) { return btg_internal_fail(s, m.c_str()); }

// partition_skeleton (distributed.cpp:145-175): ceiling cuts, trailing shards may be empty.
btg_status skeleton(btg_partition p, size_t rows, size_t cols) {
    if (rows == 0 || cols == 0) return pfail(BTG_EGRID, "partition: grid must be positive");
    if (rows > p->nd || cols > p->nm)
        return pfail(BTG_EGRID, "partition: grid " + std::to_string(rows) + "x" + std::to_string(cols) +
                                    " leaves workers without any of " + std::to_string(p->nd) + " sensors x " +
                                    std::to_string(p->nm) + " sources");
    p->rows = rows;
    p->cols = cols;
    const size_t sc = (p->nd + rows - 1) / rows, mc = (p->nm + cols - 1) / cols;
    p->shards.resize(rows * cols);
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) {
            auto& s = p->shards[i * cols + j];
            s.i0 = std::min(i * sc, p->nd);
            s.i1 = std::min((i + 1) * sc, p->nd);
            s.j0 = std::min(j * mc, p->nm);
            s.j1 = std::min((j + 1) * mc, p->nm);
        }
    return BTG_OK;
}

void tree_reduce(std::vector<std::vector<double>>& parts) {
    const size_t count = parts.size();
    for (size_t step = 1; step < count; step *= 2)
        for (size_t i = 0; i + step < count; i += 2 * step) {
            auto& dst = parts[i];
            const auto& src = parts[i + step];
            for (size_t k = 0; k < dst.size(); ++k) dst[k] += src[k];
        }
}

// Run `work(idx)` for every shard index in `ids`, one thread per shard when parallel.
template <typename F>
btg_status for_shards(const std::vector<size_t>& ids, bool parallel, F work) {
    std::vector<btg_status> st(ids.size(), BTG_OK);
    if (!parallel || ids.size() < 2) {
        for (size_t k = 0; k < ids.size(); ++k)
            if ((st[k] = work(ids[k])) != BTG_OK) return st[k];
        return BTG_OK;
    }
    std::vector<std::thread> th;
    th.reserve(ids.size());
    for (size_t k = 0; k < ids.size(); ++k) th.emplace_back([&, k] { st[k] = work(ids[k]); });
    for (auto& t : th) t.join();
    for (btg_status s : st)
        if (s != BTG_OK) return s;
    return BTG_OK;
}

// One shard's local apply (backend 0 fft, 1 ewp, 2 naive), host vectors.
btg_status local_apply(btg_partition p, const btg_partition_s::Shard& s, bool adjoint, int backend, const double* in,
                       double* out, int device) {
    const size_t ld = s.i1 - s.i0, lm = s.j1 - s.j0, nt = p->nt;
    const size_t nin = (adjoint ? ld : lm) * nt, nout = (adjoint ? lm : ld) * nt;
    switch (backend) {
        case 0:
            return adjoint ? btg_adjoint(s.op, in, nin, out, nout, 1, 0u) : btg_forward(s.op, in, nin, out, nout, 1, 0u);
        case 1:
            return adjoint ? btg_adjoint_ewp(s.op, in, nin, out, nout, 0u) : btg_forward_ewp(s.op, in, nin, out, nout, 0u);
        default:
            return adjoint ? btg_naive_adjoint(s.blocks.data(), ld, lm, nt, in, out, device, 0u)
                           : btg_naive_forward(s.blocks.data(), ld, lm, nt, in, out, device, 0u);
    }
}

btg_status check_backend(btg_partition p, int backend) {
    if (backend < 0 || backend > 2) return pfail(BTG_EARG, "unknown backend " + std::to_string(backend));
    if (backend == 1 && !p->channel_layout)
        return pfail(BTG_EARG, "distributed apply: ewp backend needs a partition set up with keep_channel_layout");
    if (backend == 2 && !p->has_compact)
        return pfail(BTG_EARG, "distributed apply: naive backend needs time-domain blocks (partition of a "
                               "compact operator)");
    return BTG_OK;
}

btg_status apply(btg_partition p, bool adjoint, const double* in, size_t in_len, double* out, size_t out_len,
                 int backend, int parallel) {
    if (!p) return pfail(BTG_EARG, "null partition");
    if (!in || !out) return pfail(BTG_EARG, "null vector pointer");
    const size_t din = adjoint ? p->nd : p->nm, dout = adjoint ? p->nm : p->nd;
    const char* what = adjoint ? "distributed_adjoint" : "distributed_forward";
    if (in_len != din * p->nt || out_len != dout * p->nt)
        return pfail(BTG_EDIM, std::string(what) + ": vector does not match the partition");
    btg_status s = check_backend(p, backend);
    if (s != BTG_OK) return s;
    const size_t groups = adjoint ? p->cols : p->rows, members = adjoint ? p->rows : p->cols;
    // partials[g][k]: member k of output group g (F: row g, members j; F*: column g, members i)
    std::vector<std::vector<std::vector<double>>> partials(groups, std::vector<std::vector<double>>(members));
    std::vector<size_t> ids(p->shards.size());
    for (size_t k = 0; k < ids.size(); ++k) ids[k] = k;
    s = for_shards(ids, parallel != 0, [&](size_t idx) -> btg_status {
        const auto& sh = p->shards[idx];
        const size_t i = idx / p->cols, j = idx % p->cols;
        const size_t g = adjoint ? j : i, k = adjoint ? i : j;
        const size_t lout = (adjoint ? sh.j1 - sh.j0 : sh.i1 - sh.i0) * p->nt;
        auto& part = partials[g][k];
        part.assign(lout, 0.0);
        if (sh.empty()) return BTG_OK;
        const double* xin = in + (adjoint ? sh.i0 : sh.j0) * p->nt;  // SOTI slice (scatter_param / scatter_data)
        return local_apply(p, sh, adjoint, backend, xin, part.data(), p->devices[idx % p->devices.size()]);
    });
    if (s != BTG_OK) return s;
    for (size_t g = 0; g < groups; ++g) {
        tree_reduce(partials[g]);
        const auto& sh = p->shards[adjoint ? g : g * p->cols];
        const size_t off = (adjoint ? sh.j0 : sh.i0) * p->nt;
        if (!partials[g][0].empty()) std::memcpy(out + off, partials[g][0].data(), partials[g][0].size() * 8);
    }
    return BTG_OK;
}

btg_status init_devices(btg_partition p, const int* devices, size_t num_devices) {
    if (devices && num_devices) {
        p->devices.assign(devices, devices + num_devices);
    } else {
        p->devices = {0};
    }
    return BTG_OK;
}

}  // namespace

extern "C" {

btg_status btg_partition_create(const double* blocks, size_t nd, size_t nm, size_t nt, size_t rows, size_t cols,
                                const int* devices, size_t num_devices, int precision, unsigned flags,
                                btg_partition* out) {
    if (!out) return pfail(BTG_EARG, "null output handle");
    *out = nullptr;
    if (!blocks) return pfail(BTG_EARG, "null blocks");
    if (nd == 0 || nm == 0 || nt == 0) return pfail(BTG_EDIM, "compact operator: all dimensions must be positive");
    auto* p = new btg_partition_s;
    p->nd = nd;
    p->nm = nm;
    p->nt = nt;
    p->has_compact = true;
    p->channel_layout = (flags & BTG_KEEP_CHANNEL_LAYOUT) != 0;
    init_devices(p, devices, num_devices);
    btg_status s = skeleton(p, rows, cols);
    for (size_t idx = 0; s == BTG_OK && idx < p->shards.size(); ++idx) {
        auto& sh = p->shards[idx];
        if (sh.empty()) continue;
        const size_t ld = sh.i1 - sh.i0, lm = sh.j1 - sh.j0;
        sh.blocks.resize(nt * ld * lm);
        for (size_t k = 0; k < nt; ++k)
            for (size_t i = 0; i < ld; ++i)
                std::memcpy(sh.blocks.data() + (k * ld + i) * lm, blocks + (k * nd + sh.i0 + i) * nm + sh.j0, lm * 8);
        s = btg_setup(sh.blocks.data(), ld, lm, nt, precision, p->devices[idx % p->devices.size()],
                      flags & BTG_KEEP_CHANNEL_LAYOUT, &sh.op);
    }
    if (s != BTG_OK) {
        btg_partition_destroy(p);
        return s;
    }
    *out = p;
    return BTG_OK;
}

btg_status btg_partition_from_operator(btg_op op, size_t rows, size_t cols, const int* devices, size_t num_devices,
                                       btg_partition* out) {
    if (!out) return pfail(BTG_EARG, "null output handle");
    *out = nullptr;
    size_t nd = 0, nm = 0, nt = 0;
    int prec = 0;
    btg_status s = btg_get_dims(op, &nd, &nm, &nt, &prec);
    if (s != BTG_OK) return s;
    auto* p = new btg_partition_s;
    p->nd = nd;
    p->nm = nm;
    p->nt = nt;
    int layout = 0;
    btg_has_channel_layout(op, &layout);
    p->channel_layout = layout != 0;
    init_devices(p, devices, num_devices);
    s = skeleton(p, rows, cols);
    for (size_t idx = 0; s == BTG_OK && idx < p->shards.size(); ++idx) {
        auto& sh = p->shards[idx];
        if (sh.empty()) continue;
        s = btg_slice_operator(op, sh.i0, sh.i1, sh.j0, sh.j1, p->devices[idx % p->devices.size()], &sh.op);
        if (s == BTG_OK && p->channel_layout) s = btg_set_channel_layout(sh.op, 1);
    }
    if (s != BTG_OK) {
        btg_partition_destroy(p);
        return s;
    }
    *out = p;
    return BTG_OK;
}

btg_status btg_partition_shard(btg_partition p, size_t row, size_t col, size_t* bounds, btg_op* op) {
    if (!p) return pfail(BTG_EARG, "null partition");
    if (row >= p->rows || col >= p->cols) return pfail(BTG_EGRID, "shard index outside the grid");
    const auto& sh = p->shards[row * p->cols + col];
    if (bounds) {
        bounds[0] = sh.i0;
        bounds[1] = sh.i1;
        bounds[2] = sh.j0;
        bounds[3] = sh.j1;
    }
    if (op) *op = sh.op;
    return BTG_OK;
}

btg_status btg_partition_forward(btg_partition p, const double* m, size_t m_len, double* d, size_t d_len,
                                 int backend, int parallel) {
    return apply(p, false, m, m_len, d, d_len, backend, parallel);
}

btg_status btg_partition_adjoint(btg_partition p, const double* d, size_t d_len, double* m, size_t m_len,
                                 int backend, int parallel) {
    return apply(p, true, d, d_len, m, m_len, backend, parallel);
}

void btg_partition_destroy(btg_partition p) {
    if (!p) return;
    for (auto& sh : p->shards)
        if (sh.op) btg_destroy(sh.op);
    delete p;
}

}  // extern "C"
