// Processor-grid engine: the reference's distributed F / F* (distributed.cpp:
// 145-392) and the Hessian over a partition (inverse.cpp:78-91), as one
// per-rank schedule executed over three transports (include/btg.h):
//   NCCL      one process per GPU (ncclCommInitRank + ncclCommSplit into row /
//             column communicators), or every cell in one process on distinct
//             devices (ncclCommInitAll); collectives on the cell's stream, so the
//             local pipeline and the exchange are ordered without host syncs;
//   P2P       the reference's single-process Partition on any placement:
//             device copies plus a sum kernel in the reference's fixed tree
//             order (tree_reduce, distributed.cpp:36-47);
//   external  host callbacks (tests run several ranks on one GPU over gloo).
// The local step is the single-GPU pipeline of the cell's handle (btg_capi.cu)
// on device pointers, with Gamma^-1 and alpha R v fused into its C2R epilogue.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/btg.h"
#include "btg_kernels.cuh"

extern "C" btg_status btg_internal_fail(btg_status s, const char* msg);
extern "C" int btg_internal_fused_ok(btg_op op, int adjoint);
extern "C" btg_status btg_internal_apply_fused(btg_op op, int adjoint, const double* in, size_t in_len, double* out,
                                               size_t out_len, const btg_epilogue* ex, const double* const* peers,
                                               int npeers);

namespace {

btg_status gfail(btg_status s, const std::string& m) { return btg_internal_fail(s, m.c_str()); }

#define G_CUDA(call)                                                                                  \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            return gfail(e_ == cudaErrorMemoryAllocation ? BTG_ENOMEM : BTG_ECUDA,                    \
                         std::string(#call) + ": " + cudaGetErrorString(e_));                         \
    } while (0)

#define G_NCCL(call)                                                                                  \
    do {                                                                                              \
        ncclResult_t r_ = (call);                                                                     \
        if (r_ != ncclSuccess)                                                                        \
            return gfail(BTG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));             \
    } while (0)

#define G_TRY(call)                  \
    do {                             \
        btg_status s_ = (call);      \
        if (s_ != BTG_OK) return s_; \
    } while (0)

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// ---- small kernels of the grid data plane ------------------------------------
// dst[k] += src[k]: one edge of the reference's binary reduction tree. The tree
// itself (which partial is added into which, level by level) is walked on the
// host in tree_reduce's order, so every element sees exactly the reference's
// additions.
__global__ void k_add_inplace(double* __restrict__ dst, const double* __restrict__ src, size_t n) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        dst[k] += src[k];
}

// y *= Gamma^-1 rows (backends without the fused epilogue)
__global__ void k_scale_rows(double* __restrict__ y, const double* __restrict__ g, int per_sample, size_t rows,
                             size_t nt) {
    const size_t n = rows * nt;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
        y[k] *= per_sample ? g[k] : g[k / nt];
}

// y += alpha R v (Regularization::apply, inverse.cpp:32-49), backends without the epilogue
__global__ void k_add_reg(double* __restrict__ y, const double* __restrict__ v, double alpha, int lap, size_t rows,
                          size_t nt) {
    const size_t n = rows * nt;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        const size_t t = k % nt;
        double r = v[k];
        if (lap) r = 2.0 * v[k] - (t > 0 ? v[k - 1] : 0.0) - (t + 1 < nt ? v[k + 1] : 0.0);
        y[k] += alpha * r;
    }
}

int grid_blocks(size_t n) { return (int)std::max<size_t>(1, std::min<size_t>(ceil_div(n, 256), 148 * 8)); }

// NCCL determinism: a fixed algorithm and protocol give run-to-run identical
// bits for a fixed grid. Read by NCCL at communicator creation.
void pin_nccl_env() {
    if (std::getenv("BTG_NCCL_UNPINNED")) return;
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
}

}  // namespace

struct btg_grid_s {
    size_t rows = 0, cols = 0;
    int transport = BTG_TRANSPORT_P2P;
    bool local = false;        // every cell in this process
    size_t my_rank = SIZE_MAX;  // one-rank grids
    size_t nd = 0, nm = 0, nt = 0;
    bool dims_set = false;
    int backend = 0;
    bool parallel = false;
    btg_grid_callbacks cb{};
    std::mutex mu;

    struct Bounds {
        size_t i0 = 0, i1 = 0, j0 = 0, j1 = 0;
    };
    std::vector<Bounds> bounds;  // every cell, row-major

    struct Cell {
        size_t rank = 0, i = 0, j = 0;
        int device = 0;
        btg_op op = nullptr;
        bool own_op = false;
        cudaStream_t own_stream = nullptr;
        cudaStream_t stream = nullptr;
        cudaEvent_t ev = nullptr;
        double* buf[4] = {};  // X, Y, Z, W (P2P receive scratch)
        size_t cap = 0;       // doubles per buffer
        double* gam = nullptr;      // Gamma^-1 rows of this call (borrowed or gam_buf)
        double* gam_buf = nullptr;
        size_t gcap = 0;
        double* host_stage = nullptr;  // external transport
        std::vector<double> blocks;    // compact rectangle (naive backend)
        double* d_blocks = nullptr;
        ncclComm_t world = nullptr, row = nullptr, col = nullptr;
        const double** peer_ptrs = nullptr;  // fused reduce: device array of the group's partials
    };
    std::vector<Cell> cells;  // local cells (all for local grids, one otherwise)
    std::vector<std::vector<char>> peer_ok;  // local grids: device a can load device b's memory
    std::vector<btg_comm_event> log;
};

namespace {

using Grid = btg_grid_s;
using Cell = btg_grid_s::Cell;

size_t cell_ld(const Grid* g, const Cell& c) { return g->bounds[c.rank].i1 - g->bounds[c.rank].i0; }
size_t cell_lm(const Grid* g, const Cell& c) { return g->bounds[c.rank].j1 - g->bounds[c.rank].j0; }
bool cell_empty(const Grid* g, const Cell& c) { return cell_ld(g, c) == 0 || cell_lm(g, c) == 0; }

// partition_skeleton (distributed.cpp:145-175)
btg_status skeleton(Grid* g) {
    if (g->rows > g->nd || g->cols > g->nm)
        return gfail(BTG_EGRID, "partition: grid " + std::to_string(g->rows) + "x" + std::to_string(g->cols) +
                                    " leaves workers without any of " + std::to_string(g->nd) + " sensors x " +
                                    std::to_string(g->nm) + " sources");
    const size_t sc = ceil_div(g->nd, g->rows), mc = ceil_div(g->nm, g->cols);
    g->bounds.assign(g->rows * g->cols, {});
    for (size_t i = 0; i < g->rows; ++i)
        for (size_t j = 0; j < g->cols; ++j) {
            auto& b = g->bounds[i * g->cols + j];
            b.i0 = std::min(i * sc, g->nd);
            b.i1 = std::min((i + 1) * sc, g->nd);
            b.j0 = std::min(j * mc, g->nm);
            b.j1 = std::min((j + 1) * mc, g->nm);
        }
    return BTG_OK;
}

// Per-cell device buffers sized for the cell's slices.
btg_status cell_buffers(Grid* g, Cell& c) {
    const size_t need = std::max<size_t>(1, std::max(cell_ld(g, c), cell_lm(g, c)) * g->nt);
    if (c.cap >= need) return BTG_OK;
    DevGuard dg(c.device);
    for (double*& b : c.buf) {
        if (b) cudaFree(b);
        b = nullptr;
    }
    c.cap = 0;
    for (double*& b : c.buf) G_CUDA(cudaMalloc(&b, need * sizeof(double)));
    c.cap = need;
    return BTG_OK;
}

btg_status create_cells(Grid* g, const std::vector<std::pair<size_t, int>>& rank_dev) {
    for (const auto& [rank, dev] : rank_dev) {
        Cell c;
        c.rank = rank;
        c.i = rank / g->cols;
        c.j = rank % g->cols;
        c.device = dev;
        DevGuard dg(dev);
        G_CUDA(cudaStreamCreateWithFlags(&c.own_stream, cudaStreamNonBlocking));
        c.stream = c.own_stream;
        G_CUDA(cudaEventCreateWithFlags(&c.ev, cudaEventDisableTiming));
        g->cells.push_back(c);
    }
    return BTG_OK;
}

Cell* find_cell(Grid* g, size_t rank) {
    for (auto& c : g->cells)
        if (c.rank == rank) return &c;
    return nullptr;
}

btg_status check_grid(size_t rows, size_t cols) {
    if (rows == 0 || cols == 0) return gfail(BTG_EGRID, "partition: grid must be positive");
    if (rows > (1u << 20) || cols > (1u << 20)) return gfail(BTG_EGRID, "grid too large");
    return BTG_OK;
}

// ---- the schedule ------------------------------------------------------------
btg_status make_schedule(size_t nd, size_t nm, size_t nt, size_t rows, size_t cols, size_t rank, int kind,
                         bool with_gamma, bool with_reg, std::vector<btg_grid_step>& out) {
    out.clear();
    if (rows == 0 || cols == 0 || rank >= rows * cols) return gfail(BTG_EGRID, "schedule: rank outside the grid");
    if (kind < BTG_GRID_FORWARD || kind > BTG_GRID_HESSIAN) return gfail(BTG_EARG, "schedule: unknown kind");
    const size_t sc = ceil_div(nd, rows), mc = ceil_div(nm, cols);
    const size_t i = rank / cols, j = rank % cols;
    const size_t ld = std::min((i + 1) * sc, nd) - std::min(i * sc, nd);
    const size_t lm = std::min((j + 1) * mc, nm) - std::min(j * mc, nm);
    auto step = [&](int op, int group, int src, int dst, size_t count) {
        btg_grid_step s{};
        s.op = op;
        s.group = group;
        s.root = 0;
        s.src = src;
        s.dst = dst;
        s.count = count;
        s.active = 1;
        out.push_back(s);
        return &out.back();
    };
    if (kind == BTG_GRID_FORWARD) {  // distributed.cpp:312-351
        step(BTG_STEP_INPUT, 0, -1, 0, lm * nt)->active = i == 0;
        if (rows > 1) step(BTG_STEP_BROADCAST, BTG_GROUP_COL, 0, 0, lm * nt);
        step(BTG_STEP_FORWARD, 0, 0, 1, ld * nt)->gamma = with_gamma;
        if (cols > 1) step(BTG_STEP_REDUCE, BTG_GROUP_ROW, 1, 1, ld * nt);
        step(BTG_STEP_OUTPUT, 0, 1, -1, ld * nt)->active = j == 0;
    } else if (kind == BTG_GRID_ADJOINT) {  // distributed.cpp:353-392
        step(BTG_STEP_INPUT, 0, -1, 0, ld * nt)->active = j == 0;
        if (cols > 1) step(BTG_STEP_BROADCAST, BTG_GROUP_ROW, 0, 0, ld * nt);
        step(BTG_STEP_ADJOINT, 0, 0, 1, lm * nt)->reg = with_reg && i == 0;
        if (rows > 1) step(BTG_STEP_REDUCE, BTG_GROUP_COL, 1, 1, lm * nt);
        step(BTG_STEP_OUTPUT, 0, 1, -1, lm * nt)->active = i == 0;
    } else {  // inverse.cpp:78-91 through a partition, reduce + broadcast merged
        step(BTG_STEP_INPUT, 0, -1, 0, lm * nt)->active = i == 0;
        if (rows > 1) step(BTG_STEP_BROADCAST, BTG_GROUP_COL, 0, 0, lm * nt);
        step(BTG_STEP_FORWARD, 0, 0, 1, ld * nt)->gamma = with_gamma;
        if (cols > 1) step(BTG_STEP_ALLREDUCE, BTG_GROUP_ROW, 1, 1, ld * nt);
        step(BTG_STEP_ADJOINT, 0, 1, 2, lm * nt)->reg = with_reg && i == 0;
        if (rows > 1) step(BTG_STEP_REDUCE, BTG_GROUP_COL, 2, 2, lm * nt);
        step(BTG_STEP_OUTPUT, 0, 2, -1, lm * nt)->active = i == 0;
    }
    return BTG_OK;
}

size_t tree_depth(size_t participants) {
    size_t depth = 0, reach = 1;
    while (reach < participants) {
        reach *= 2;
        ++depth;
    }
    return depth;
}

// record_collective (distributed.cpp:23-34) for every group of one direction
void comm_model(size_t nd, size_t nm, size_t nt, size_t rows, size_t cols, int kind,
                std::vector<btg_comm_event>& out) {
    const size_t sc = ceil_div(nd, rows), mc = ceil_div(nm, cols);
    auto ev = [&](int phase, size_t participants, size_t dim) {
        btg_comm_event e{};
        e.phase = phase;
        e.participants = participants;
        e.messages = participants ? participants - 1 : 0;
        e.link_bytes = 8ull * nt * dim;
        e.total_bytes = e.messages * e.link_bytes;
        e.tree_depth = tree_depth(participants);
        out.push_back(e);
    };
    auto pdim = [&](size_t j) { return std::min((j + 1) * mc, nm) - std::min(j * mc, nm); };
    auto ddim = [&](size_t i) { return std::min((i + 1) * sc, nd) - std::min(i * sc, nd); };
    if (kind == BTG_GRID_FORWARD) {
        for (size_t j = 0; j < cols; ++j) ev(0, rows, pdim(j));
        for (size_t i = 0; i < rows; ++i) ev(1, cols, ddim(i));
    } else {
        for (size_t i = 0; i < rows; ++i) ev(0, cols, ddim(i));
        for (size_t j = 0; j < cols; ++j) ev(1, rows, pdim(j));
    }
}

// ---- transports -----------------------------------------------------------------
size_t group_id(const Cell& c, int group) { return group == BTG_GROUP_ROW ? c.i : c.j; }
size_t member_idx(const Cell& c, int group) { return group == BTG_GROUP_ROW ? c.j : c.i; }

// One NCCL group call over the local cells (a single cell for one-rank grids).
// Row groups move data slices (local N_d x N_t), column groups parameter slices
// (local N_m x N_t); the count is the same on every member of a group.
btg_status nccl_collective(Grid* g, const btg_grid_step& s) {
    G_NCCL(ncclGroupStart());
    for (auto& c : g->cells) {
        const size_t n = (s.group == BTG_GROUP_ROW ? cell_ld(g, c) : cell_lm(g, c)) * g->nt;
        if (n == 0) continue;
        ncclComm_t comm = s.group == BTG_GROUP_ROW ? c.row : c.col;
        double* b = c.buf[s.src];
        ncclResult_t r;
        if (s.op == BTG_STEP_BROADCAST)
            r = ncclBroadcast(b, b, n, ncclDouble, s.root, comm, c.stream);
        else if (s.op == BTG_STEP_REDUCE)
            r = ncclReduce(b, b, n, ncclDouble, ncclSum, s.root, comm, c.stream);
        else
            r = ncclAllReduce(b, b, n, ncclDouble, ncclSum, comm, c.stream);
        if (r != ncclSuccess) {
            ncclGroupEnd();
            return gfail(BTG_ENCCL, std::string("nccl collective: ") + ncclGetErrorString(r));
        }
    }
    G_NCCL(ncclGroupEnd());
    return BTG_OK;
}

// P2P: every member of every group is a local cell.
btg_status p2p_collective(Grid* g, const btg_grid_step& s) {
    const size_t ngroups = s.group == BTG_GROUP_ROW ? g->rows : g->cols;
    const size_t members = s.group == BTG_GROUP_ROW ? g->cols : g->rows;
    for (size_t grp = 0; grp < ngroups; ++grp) {
        std::vector<Cell*> mem(members, nullptr);
        for (auto& c : g->cells)
            if (group_id(c, s.group) == grp) mem[member_idx(c, s.group)] = &c;
        for (Cell* c : mem)
            if (!c) return gfail(BTG_EARG, "p2p transport: a group member is not local");
        const size_t n = (s.group == BTG_GROUP_ROW ? cell_ld(g, *mem[0]) : cell_lm(g, *mem[0])) * g->nt;
        if (n == 0) continue;
        auto bcast = [&](size_t root) -> btg_status {
            Cell* r = mem[root];
            {
                DevGuard dg(r->device);
                G_CUDA(cudaEventRecord(r->ev, r->stream));
            }
            for (size_t k = 0; k < members; ++k) {
                if (k == root) continue;
                Cell* c = mem[k];
                DevGuard dg(c->device);
                G_CUDA(cudaStreamWaitEvent(c->stream, r->ev, 0));
                G_CUDA(cudaMemcpyAsync(c->buf[s.src], r->buf[s.src], n * sizeof(double), cudaMemcpyDefault,
                                       c->stream));
            }
            // the root's buffer is not overwritten before every copy of it has run
            for (size_t k = 0; k < members; ++k) {
                if (k == root) continue;
                Cell* c = mem[k];
                DevGuard dg(c->device);
                G_CUDA(cudaEventRecord(c->ev, c->stream));
                DevGuard dr(r->device);
                G_CUDA(cudaStreamWaitEvent(r->stream, c->ev, 0));
            }
            return BTG_OK;
        };
        if (s.op == BTG_STEP_BROADCAST) {
            G_TRY(bcast((size_t)s.root));
            continue;
        }
        if (s.root != 0 && s.op == BTG_STEP_REDUCE) return gfail(BTG_EARG, "p2p transport: reduce root must be 0");
        // tree_reduce (distributed.cpp:36-47): level by level, partial i += partial i+step
        for (size_t step = 1; step < members; step *= 2)
            for (size_t a = 0; a + step < members; a += 2 * step) {
                Cell* dst = mem[a];
                Cell* src = mem[a + step];
                {
                    DevGuard dg(src->device);
                    G_CUDA(cudaEventRecord(src->ev, src->stream));
                }
                DevGuard dg(dst->device);
                G_CUDA(cudaStreamWaitEvent(dst->stream, src->ev, 0));
                const double* from = src->buf[s.src];
                if (src->device != dst->device) {
                    G_CUDA(cudaMemcpyAsync(dst->buf[3], from, n * sizeof(double), cudaMemcpyDefault, dst->stream));
                    from = dst->buf[3];
                }
                k_add_inplace<<<grid_blocks(n), 256, 0, dst->stream>>>(dst->buf[s.src], from, n);
                G_CUDA(cudaGetLastError());
                // src's partial may be overwritten only after this edge read it
                G_CUDA(cudaEventRecord(dst->ev, dst->stream));
                DevGuard ds(src->device);
                G_CUDA(cudaStreamWaitEvent(src->stream, dst->ev, 0));
            }
        if (s.op == BTG_STEP_ALLREDUCE) G_TRY(bcast(0));
    }
    return BTG_OK;
}

btg_status external_collective(Grid* g, const btg_grid_step& s) {
    Cell& c = g->cells[0];
    const size_t n = (s.group == BTG_GROUP_ROW ? cell_ld(g, c) : cell_lm(g, c)) * g->nt;
    if (n == 0) return BTG_OK;
    DevGuard dg(c.device);
    if (!c.host_stage) G_CUDA(cudaMallocHost(&c.host_stage, c.cap * sizeof(double)));
    G_CUDA(cudaMemcpyAsync(c.host_stage, c.buf[s.src], n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    G_CUDA(cudaStreamSynchronize(c.stream));
    int rc = 0;
    if (s.op == BTG_STEP_BROADCAST)
        rc = g->cb.broadcast(g->cb.user, s.group, c.host_stage, n, s.root);
    else if (s.op == BTG_STEP_REDUCE)
        rc = g->cb.reduce(g->cb.user, s.group, c.host_stage, n, s.root);
    else
        rc = g->cb.allreduce(g->cb.user, s.group, c.host_stage, n);
    if (rc != 0) return gfail(BTG_ENCCL, "external transport callback failed (" + std::to_string(rc) + ")");
    G_CUDA(cudaMemcpyAsync(c.buf[s.src], c.host_stage, n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
    return BTG_OK;
}

btg_status collective(Grid* g, const btg_grid_step& s) {
    switch (g->transport) {
        case BTG_TRANSPORT_NCCL:
            return nccl_collective(g, s);
        case BTG_TRANSPORT_P2P:
            return p2p_collective(g, s);
        default:
            return external_collective(g, s);
    }
}

// ---- the local step ----------------------------------------------------------------
struct CallArgs {
    const double* in = nullptr;
    size_t in_len = 0;
    double* out = nullptr;
    size_t out_len = 0;
    const double* gamma = nullptr;
    int gamma_kind = BTG_GAMMA_NONE;
    double alpha = 0.0;
    int reg_kind = BTG_REG_IDENTITY;
    unsigned flags = 0;
};

btg_status local_step(Grid* g, Cell& c, const btg_grid_step& s, const CallArgs& a) {
    DevGuard dg(c.device);
    const size_t ld = cell_ld(g, c), lm = cell_lm(g, c), nt = g->nt;
    const bool adjoint = s.op == BTG_STEP_ADJOINT;
    double* src = c.buf[s.src];
    double* dst = c.buf[s.dst];
    const size_t nin = (adjoint ? ld : lm) * nt, nout = (adjoint ? lm : ld) * nt;
    if (nout == 0) return BTG_OK;
    if (cell_empty(g, c) || !c.op) {
        if (!cell_empty(g, c)) return gfail(BTG_EARG, "grid cell " + std::to_string(c.rank) + " has no operator");
        G_CUDA(cudaMemsetAsync(dst, 0, nout * sizeof(double), c.stream));
        if (s.reg && a.alpha != 0.0) {  // row-0 cell with sources but no sensors: alpha R v alone
            k_add_reg<<<grid_blocks(nout), 256, 0, c.stream>>>(dst, c.buf[0], a.alpha,
                                                               a.reg_kind == BTG_REG_TEMPORAL_LAPLACIAN, lm, nt);
            G_CUDA(cudaGetLastError());
        }
        return BTG_OK;
    }
    const bool gamma = s.gamma && a.gamma_kind != BTG_GAMMA_NONE;
    const bool reg = s.reg && a.alpha != 0.0;
    G_TRY(btg_set_stream(c.op, c.stream));  // the handle may have been used on another stream
    if (g->backend == 0) {
        btg_epilogue epi{};
        if (gamma) {
            epi.gamma_inv = c.gam;
            epi.gamma_kind = a.gamma_kind;
        }
        if (reg) {
            epi.reg_v = c.buf[0];
            epi.alpha = a.alpha;
            epi.reg_kind = a.reg_kind;
        }
        const btg_epilogue* ep = (gamma || reg) ? &epi : nullptr;
        return adjoint ? btg_adjoint_ex(c.op, src, nin, dst, nout, 1, ep, BTG_DEVICE_PTRS)
                       : btg_forward_ex(c.op, src, nin, dst, nout, 1, ep, BTG_DEVICE_PTRS);
    }
    if (g->backend == 1) {
        G_TRY(adjoint ? btg_adjoint_ewp(c.op, src, nin, dst, nout, BTG_DEVICE_PTRS)
                      : btg_forward_ewp(c.op, src, nin, dst, nout, BTG_DEVICE_PTRS));
    } else {
        if (c.blocks.empty() && !c.d_blocks)
            return gfail(BTG_EARG, "distributed apply: naive backend needs time-domain blocks (partition of a "
                                   "compact operator)");
        if (!c.d_blocks) {
            G_CUDA(cudaMalloc(&c.d_blocks, c.blocks.size() * sizeof(double)));
            G_CUDA(cudaMemcpy(c.d_blocks, c.blocks.data(), c.blocks.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        G_CUDA(cudaStreamSynchronize(c.stream));  // the naive kernels run on the legacy stream
        G_TRY(adjoint ? btg_naive_adjoint(c.d_blocks, ld, lm, nt, src, dst, c.device, BTG_DEVICE_PTRS)
                      : btg_naive_forward(c.d_blocks, ld, lm, nt, src, dst, c.device, BTG_DEVICE_PTRS));
    }
    if (gamma) {
        k_scale_rows<<<grid_blocks(nout), 256, 0, c.stream>>>(dst, c.gam, a.gamma_kind == BTG_GAMMA_PER_SAMPLE, ld,
                                                              nt);
        G_CUDA(cudaGetLastError());
    }
    if (reg) {
        k_add_reg<<<grid_blocks(nout), 256, 0, c.stream>>>(dst, c.buf[0], a.alpha,
                                                           a.reg_kind == BTG_REG_TEMPORAL_LAPLACIAN, lm, nt);
        G_CUDA(cudaGetLastError());
    }
    return BTG_OK;
}

// ---- reduce fused into the final C2R (P2P transport) -------------------------
// A local F (F*) followed by a row (column) reduce / all-reduce onto member 0:
// the other members compute their partials first, then member 0's C2R loads
// them over NVLink (peer access) and stores the reference's tree_reduce of all
// members (C2REpilogue::peers) — no receive copies, no separate add kernels.
// Bit-identical to the unfused P2P path (same tree, same additions).
bool fused_enabled() {
    const char* v = std::getenv("BTG_GRID_FUSED");
    return !(v && *v == '0');
}

std::vector<Cell*> group_members(Grid* g, int group, size_t grp) {
    const size_t members = group == BTG_GROUP_ROW ? g->cols : g->rows;
    std::vector<Cell*> mem(members, nullptr);
    for (auto& c : g->cells)
        if (group_id(c, group) == grp) mem[member_idx(c, group)] = &c;
    return mem;
}

bool fusable(Grid* g, const btg_grid_step& local, const btg_grid_step& red) {
    if (!fused_enabled() || g->transport != BTG_TRANSPORT_P2P || !g->local || g->backend != 0) return false;
    if ((red.op != BTG_STEP_REDUCE && red.op != BTG_STEP_ALLREDUCE) || red.root != 0 || red.src != local.dst)
        return false;
    const bool adjoint = local.op == BTG_STEP_ADJOINT;
    const size_t ngroups = red.group == BTG_GROUP_ROW ? g->rows : g->cols;
    for (size_t grp = 0; grp < ngroups; ++grp) {
        auto mem = group_members(g, red.group, grp);
        if (mem.size() > (size_t)btg::kMaxFusedPeers + 1) return false;
        if (mem.size() < 2) continue;
        for (Cell* c : mem)
            if (!c) return false;
        Cell* root = mem[0];
        if (cell_empty(g, *root) || !root->op || !btg_internal_fused_ok(root->op, adjoint ? 1 : 0)) return false;
        for (Cell* c : mem)
            if (root->device >= (int)g->peer_ok.size() || c->device >= (int)g->peer_ok.size() ||
                !g->peer_ok[root->device][c->device])
                return false;
    }
    return true;
}

btg_status fused_local_reduce(Grid* g, const std::vector<std::vector<btg_grid_step>>& sch, size_t st,
                              const CallArgs& a) {
    const btg_grid_step& red = sch[0][st + 1];
    const bool adjoint = sch[0][st].op == BTG_STEP_ADJOINT;
    const size_t ngroups = red.group == BTG_GROUP_ROW ? g->rows : g->cols;
    for (size_t grp = 0; grp < ngroups; ++grp) {
        auto mem = group_members(g, red.group, grp);
        Cell* root = mem[0];
        const btg_grid_step& rs = sch[root->rank][st];
        if (mem.size() < 2) {
            G_TRY(local_step(g, *root, rs, a));
            continue;
        }
        // the other members' partials
        std::vector<const double*> ptrs;
        for (size_t k = 1; k < mem.size(); ++k) {
            Cell* c = mem[k];
            G_TRY(local_step(g, *c, sch[c->rank][st], a));
            DevGuard dg(c->device);
            G_CUDA(cudaEventRecord(c->ev, c->stream));
            DevGuard dr(root->device);
            G_CUDA(cudaStreamWaitEvent(root->stream, c->ev, 0));
            ptrs.push_back(c->buf[sch[c->rank][st].dst]);
        }
        // member 0: its own F / F* with the tree reduce in the C2R stores
        DevGuard dg(root->device);
        if (!root->peer_ptrs) G_CUDA(cudaMalloc(&root->peer_ptrs, btg::kMaxFusedPeers * sizeof(double*)));
        G_CUDA(cudaMemcpyAsync(root->peer_ptrs, ptrs.data(), ptrs.size() * sizeof(double*), cudaMemcpyHostToDevice,
                               root->stream));
        const size_t ld = cell_ld(g, *root), lm = cell_lm(g, *root), nt = g->nt;
        const size_t nin = (adjoint ? ld : lm) * nt, nout = (adjoint ? lm : ld) * nt;
        btg_epilogue epi{};
        const bool gamma = rs.gamma && a.gamma_kind != BTG_GAMMA_NONE;
        const bool reg = rs.reg && a.alpha != 0.0;
        if (gamma) {
            epi.gamma_inv = root->gam;
            epi.gamma_kind = a.gamma_kind;
        }
        if (reg) {
            epi.reg_v = root->buf[0];
            epi.alpha = a.alpha;
            epi.reg_kind = a.reg_kind;
        }
        G_TRY(btg_set_stream(root->op, root->stream));
        G_TRY(btg_internal_apply_fused(root->op, adjoint ? 1 : 0, root->buf[rs.src], nin, root->buf[rs.dst], nout,
                                       (gamma || reg) ? &epi : nullptr, root->peer_ptrs, (int)ptrs.size()));
        // the partials are read: their buffers may be reused
        G_CUDA(cudaEventRecord(root->ev, root->stream));
        for (size_t k = 1; k < mem.size(); ++k) {
            DevGuard dm(mem[k]->device);
            G_CUDA(cudaStreamWaitEvent(mem[k]->stream, root->ev, 0));
        }
    }
    if (red.op == BTG_STEP_ALLREDUCE) {  // member 0 holds the sum: broadcast it over the group
        btg_grid_step b = red;
        b.op = BTG_STEP_BROADCAST;
        b.root = 0;
        G_TRY(p2p_collective(g, b));
    }
    return BTG_OK;
}


// Gamma^-1 rows of the cell on its device (the C2R epilogue reads them there):
// a one-rank grid with a 16-byte aligned device pointer borrows them in place.
btg_status stage_gamma(Grid* g, Cell& c, const CallArgs& a) {
    c.gam = nullptr;
    if (a.gamma_kind == BTG_GAMMA_NONE) return BTG_OK;
    const auto& b = g->bounds[c.rank];
    const size_t per = a.gamma_kind == BTG_GAMMA_PER_SENSOR ? 1 : g->nt;
    const size_t n = (b.i1 - b.i0) * per;
    if (n == 0) return BTG_OK;
    const double* src = a.gamma + b.i0 * per;
    if ((a.flags & BTG_DEVICE_PTRS) && !g->local && ((uintptr_t)src & 15u) == 0) {
        c.gam = const_cast<double*>(src);
        return BTG_OK;
    }
    DevGuard dg(c.device);
    if (c.gcap < n) {
        cudaFree(c.gam_buf);
        c.gam_buf = nullptr;
        c.gcap = 0;
        G_CUDA(cudaMalloc(&c.gam_buf, n * sizeof(double)));
        c.gcap = n;
    }
    G_CUDA(cudaMemcpyAsync(c.gam_buf, src, n * sizeof(double), cudaMemcpyDefault, c.stream));
    c.gam = c.gam_buf;
    return BTG_OK;
}

// Offset of cell c's slice in the global vector of an INPUT / OUTPUT step.
size_t slice_offset(const Grid* g, const Cell& c, int kind, bool input) {
    const auto& b = g->bounds[c.rank];
    const bool param = kind == BTG_GRID_HESSIAN || (kind == BTG_GRID_FORWARD) == input;
    return (param ? b.j0 : b.i0) * g->nt;
}

btg_status run(Grid* g, int kind, const CallArgs& a) {
    if (!g) return gfail(BTG_EARG, "null grid");
    std::lock_guard<std::mutex> lock(g->mu);
    if (!g->dims_set) return gfail(BTG_EARG, "grid: operator dims not set (setup / attach first)");
    for (auto& c : g->cells)
        if (!cell_empty(g, c) && !c.op)
            return gfail(BTG_EARG, "grid cell " + std::to_string(c.rank) + " has no operator attached");
    const char* what = kind == BTG_GRID_FORWARD ? "distributed_forward"
                       : kind == BTG_GRID_ADJOINT ? "distributed_adjoint"
                                                  : "hessian";
    const size_t din = kind == BTG_GRID_ADJOINT ? g->nd : g->nm;
    const size_t dout = kind == BTG_GRID_FORWARD ? g->nd : g->nm;
    if (a.gamma_kind < BTG_GAMMA_NONE || a.gamma_kind > BTG_GAMMA_PER_SAMPLE)
        return gfail(BTG_EARG, "unknown gamma kind " + std::to_string(a.gamma_kind));
    if (a.gamma_kind != BTG_GAMMA_NONE && !a.gamma) return gfail(BTG_EARG, "gamma_inv is null");
    if (a.reg_kind != BTG_REG_IDENTITY && a.reg_kind != BTG_REG_TEMPORAL_LAPLACIAN)
        return gfail(BTG_EARG, "unknown regularization kind " + std::to_string(a.reg_kind));
    // schedules of the local cells (identical step ops on every rank)
    std::vector<std::vector<btg_grid_step>> sch(g->cells.size());
    for (size_t k = 0; k < g->cells.size(); ++k)
        G_TRY(make_schedule(g->nd, g->nm, g->nt, g->rows, g->cols, g->cells[k].rank, kind,
                            a.gamma_kind != BTG_GAMMA_NONE, a.alpha != 0.0, sch[k]));
    if (g->local) {
        if (!a.in || !a.out) return gfail(BTG_EARG, "null vector pointer");
        if (a.in_len != din * g->nt || a.out_len != dout * g->nt)
            return gfail(BTG_EDIM, std::string(what) + ": vector does not match the partition");
    } else {
        const auto& s0 = sch[0];
        const btg_grid_step& in = s0.front();
        const btg_grid_step& out = s0.back();
        if (in.active && (!a.in || a.in_len != in.count))
            return gfail(a.in ? BTG_EDIM : BTG_EARG,
                         std::string(what) + ": this rank owns an input slice of " + std::to_string(in.count) +
                             " values (got " + std::to_string(a.in_len) + ")");
        if (out.active && (!a.out || a.out_len != out.count))
            return gfail(a.out ? BTG_EDIM : BTG_EARG,
                         std::string(what) + ": this rank receives an output slice of " +
                             std::to_string(out.count) + " values (got " + std::to_string(a.out_len) + ")");
    }
    for (auto& c : g->cells) {
        G_TRY(cell_buffers(g, c));
        G_TRY(stage_gamma(g, c, a));
    }
    const size_t nsteps = sch[0].size();
    for (size_t st = 0; st < nsteps; ++st) {
        const btg_grid_step& s = sch[0][st];
        switch (s.op) {
            case BTG_STEP_INPUT:
            case BTG_STEP_OUTPUT: {
                const bool input = s.op == BTG_STEP_INPUT;
                for (size_t k = 0; k < g->cells.size(); ++k) {
                    Cell& c = g->cells[k];
                    const btg_grid_step& cs = sch[k][st];
                    if (!cs.active || cs.count == 0) continue;
                    const size_t off = g->local ? slice_offset(g, c, kind, input) : 0;
                    DevGuard dg(c.device);
                    if (input)
                        G_CUDA(cudaMemcpyAsync(c.buf[cs.dst], a.in + off, cs.count * sizeof(double),
                                               cudaMemcpyDefault, c.stream));
                    else
                        G_CUDA(cudaMemcpyAsync(a.out + off, c.buf[cs.src], cs.count * sizeof(double),
                                               cudaMemcpyDefault, c.stream));
                }
                break;
            }
            case BTG_STEP_FORWARD:
            case BTG_STEP_ADJOINT: {
                if (st + 1 < nsteps && fusable(g, s, sch[0][st + 1])) {
                    G_TRY(fused_local_reduce(g, sch, st, a));
                    ++st;  // the reduce ran inside member 0's C2R
                    break;
                }
                // BTG_GRID_FUSED_REQUIRE=1 (tests): a P2P reduce that could not be fused is an error
                if (st + 1 < nsteps && g->transport == BTG_TRANSPORT_P2P && fused_enabled() &&
                    (sch[0][st + 1].op == BTG_STEP_REDUCE || sch[0][st + 1].op == BTG_STEP_ALLREDUCE) &&
                    std::getenv("BTG_GRID_FUSED_REQUIRE"))
                    return gfail(BTG_EARG, "fused reduce required but not applicable");
                if (g->parallel && g->cells.size() > 1) {
                    std::vector<btg_status> rs(g->cells.size(), BTG_OK);
                    std::vector<std::string> msg(g->cells.size());
                    std::vector<std::thread> th;
                    for (size_t k = 0; k < g->cells.size(); ++k)
                        th.emplace_back([&, k] {
                            rs[k] = local_step(g, g->cells[k], sch[k][st], a);
                            if (rs[k] != BTG_OK) msg[k] = btg_last_error();
                        });
                    for (auto& t : th) t.join();
                    for (size_t k = 0; k < rs.size(); ++k)
                        if (rs[k] != BTG_OK) return gfail(rs[k], msg[k]);  // re-issued on this thread
                } else {
                    for (size_t k = 0; k < g->cells.size(); ++k) G_TRY(local_step(g, g->cells[k], sch[k][st], a));
                }
                break;
            }
            default:
                G_TRY(collective(g, s));
        }
    }
    if (!(a.flags & BTG_DEVICE_PTRS) || g->local)
        for (auto& c : g->cells) {
            DevGuard dg(c.device);
            G_CUDA(cudaStreamSynchronize(c.stream));
        }
    if (kind != BTG_GRID_HESSIAN) comm_model(g->nd, g->nm, g->nt, g->rows, g->cols, kind, g->log);
    return BTG_OK;
}

void destroy_cell(Cell& c) {
    DevGuard dg(c.device);
    if (c.stream) cudaStreamSynchronize(c.stream);
    if (c.op && c.own_op) btg_destroy(c.op);
    for (double* b : c.buf) cudaFree(b);
    cudaFree(c.gam_buf);
    cudaFree(c.d_blocks);
    if (c.host_stage) cudaFreeHost(c.host_stage);
    if (c.row) ncclCommDestroy(c.row);
    if (c.col) ncclCommDestroy(c.col);
    if (c.world) ncclCommDestroy(c.world);
    if (c.ev) cudaEventDestroy(c.ev);
    if (c.own_stream) cudaStreamDestroy(c.own_stream);
    cudaFree(c.peer_ptrs);
}

btg_status bind_op(Cell& c, btg_op op, bool own) {
    if (c.op && c.own_op && c.op != op) btg_destroy(c.op);
    c.op = op;
    c.own_op = own;
    if (op) G_TRY(btg_set_stream(op, c.stream));
    return BTG_OK;
}

btg_status new_grid(size_t rows, size_t cols, int transport, Grid** out) {
    if (!out) return gfail(BTG_EARG, "null output handle");
    *out = nullptr;
    G_TRY(check_grid(rows, cols));
    auto* g = new Grid;
    g->rows = rows;
    g->cols = cols;
    g->transport = transport;
    *out = g;
    return BTG_OK;
}

// NCCL row / column communicators of the local cells. Every rank of the parent
// takes part in each split; the two splits run one after the other (each a
// group call over the local cells, so a single thread can drive all the cells
// of a local grid). A split is skipped when its groups would have one member.
btg_status split_comms(Grid* g) {
    for (int round = 0; round < 2; ++round) {
        const bool rows_split = round == 0;
        if (rows_split ? g->cols == 1 : g->rows == 1) continue;
        G_NCCL(ncclGroupStart());
        for (auto& c : g->cells) {
            DevGuard dg(c.device);
            const ncclResult_t r = rows_split ? ncclCommSplit(c.world, (int)c.i, (int)c.j, &c.row, nullptr)
                                              : ncclCommSplit(c.world, (int)c.j, (int)c.i, &c.col, nullptr);
            if (r != ncclSuccess) {
                ncclGroupEnd();
                return gfail(BTG_ENCCL, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
            }
        }
        G_NCCL(ncclGroupEnd());
    }
    return BTG_OK;
}

}  // namespace

extern "C" {

btg_status btg_grid_schedule(size_t nd, size_t nm, size_t nt, size_t rows, size_t cols, size_t rank, int kind,
                             int with_gamma, int with_reg, btg_grid_step* steps, size_t cap, size_t* count) {
    std::vector<btg_grid_step> s;
    G_TRY(make_schedule(nd, nm, nt, rows, cols, rank, kind, with_gamma != 0, with_reg != 0, s));
    if (count) *count = s.size();
    if (steps) {
        if (cap < s.size()) return gfail(BTG_EARG, "schedule: capacity too small");
        std::copy(s.begin(), s.end(), steps);
    }
    return BTG_OK;
}

btg_status btg_comm_events(size_t nd, size_t nm, size_t nt, size_t rows, size_t cols, int kind, btg_comm_event* out,
                           size_t cap, size_t* count) {
    if (rows == 0 || cols == 0) return gfail(BTG_EGRID, "partition: grid must be positive");
    if (kind != BTG_GRID_FORWARD && kind != BTG_GRID_ADJOINT) return gfail(BTG_EARG, "comm events: F or F* only");
    std::vector<btg_comm_event> ev;
    comm_model(nd, nm, nt, rows, cols, kind, ev);
    if (count) *count = ev.size();
    if (out) {
        if (cap < ev.size()) return gfail(BTG_EARG, "comm events: capacity too small");
        std::copy(ev.begin(), ev.end(), out);
    }
    return BTG_OK;
}

btg_status btg_grid_nccl_id(void* id_out) {
    if (!id_out) return gfail(BTG_EARG, "null id buffer");
    static_assert(sizeof(ncclUniqueId) == BTG_NCCL_ID_BYTES, "NCCL unique id size");
    pin_nccl_env();
    ncclUniqueId id;
    G_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof id);
    return BTG_OK;
}

btg_status btg_grid_create(size_t rows, size_t cols, size_t rank, const void* nccl_id, int device, btg_grid* out) {
    Grid* g = nullptr;
    G_TRY(new_grid(rows, cols, BTG_TRANSPORT_NCCL, &g));
    auto bail = [&](btg_status s) {
        btg_grid_destroy(g);
        *out = nullptr;
        return s;
    };
    if (!nccl_id) return bail(gfail(BTG_EARG, "null NCCL id"));
    if (rank >= rows * cols) return bail(gfail(BTG_EGRID, "rank outside the grid"));
    g->my_rank = rank;
    btg_status s = create_cells(g, {{rank, device}});
    if (s != BTG_OK) return bail(s);
    pin_nccl_env();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    {
        DevGuard dg(device);
        ncclResult_t r = ncclCommInitRank(&g->cells[0].world, (int)(rows * cols), id, (int)rank);
        if (r != ncclSuccess) return bail(gfail(BTG_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
    }
    s = split_comms(g);
    if (s != BTG_OK) return bail(s);
    *out = g;
    return BTG_OK;
}

btg_status btg_grid_create_local(size_t rows, size_t cols, const int* devices, size_t num_devices, int transport,
                                 btg_grid* out) {
    if (transport != BTG_TRANSPORT_NCCL && transport != BTG_TRANSPORT_P2P)
        return gfail(BTG_EARG, "local grid: transport must be NCCL or P2P");
    Grid* g = nullptr;
    G_TRY(new_grid(rows, cols, transport, &g));
    g->local = true;
    auto bail = [&](btg_status s) {
        btg_grid_destroy(g);
        *out = nullptr;
        return s;
    };
    std::vector<int> devs = (devices && num_devices) ? std::vector<int>(devices, devices + num_devices)
                                                     : std::vector<int>{0};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
    for (int d : devs)
        if (d < 0 || d >= ndev) return bail(gfail(BTG_EARG, "device " + std::to_string(d) + " not present"));
    const size_t n = rows * cols;
    std::vector<std::pair<size_t, int>> rd;
    for (size_t k = 0; k < n; ++k) rd.emplace_back(k, devs[k % devs.size()]);
    btg_status s = create_cells(g, rd);
    if (s != BTG_OK) return bail(s);
    // P2P: direct loads between the grid's devices (NVLink) where the hardware allows
    g->peer_ok.assign(ndev, std::vector<char>(ndev, 0));
    for (int a : devs)
        for (int b : devs) {
            if (a == b) {
                g->peer_ok[a][b] = 1;
                continue;
            }
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
                DevGuard dg(a);
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) g->peer_ok[a][b] = 1;
                cudaGetLastError();
            }
        }
    if (transport == BTG_TRANSPORT_NCCL) {
        std::vector<int> list;
        for (auto& c : g->cells) list.push_back(c.device);
        std::vector<int> sorted = list;
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end() || devs.size() < n)
            return bail(gfail(BTG_EARG, "NCCL local grid needs rows*cols distinct devices (use P2P)"));
        pin_nccl_env();
        std::vector<ncclComm_t> comms(n);
        ncclResult_t r = ncclCommInitAll(comms.data(), (int)n, list.data());
        if (r != ncclSuccess) return bail(gfail(BTG_ENCCL, std::string("ncclCommInitAll: ") + ncclGetErrorString(r)));
        for (size_t k = 0; k < n; ++k) g->cells[k].world = comms[k];
        s = split_comms(g);
        if (s != BTG_OK) return bail(s);
    }
    *out = g;
    return BTG_OK;
}

btg_status btg_grid_create_external(size_t rows, size_t cols, size_t rank, int device, const btg_grid_callbacks* cb,
                                    btg_grid* out) {
    if (!cb || !cb->broadcast || !cb->reduce || !cb->allreduce) return gfail(BTG_EARG, "missing transport callbacks");
    Grid* g = nullptr;
    G_TRY(new_grid(rows, cols, BTG_TRANSPORT_EXTERNAL, &g));
    g->cb = *cb;
    if (rank >= rows * cols) {
        btg_grid_destroy(g);
        return gfail(BTG_EGRID, "rank outside the grid");
    }
    g->my_rank = rank;
    btg_status s = create_cells(g, {{rank, device}});
    if (s != BTG_OK) {
        btg_grid_destroy(g);
        return s;
    }
    *out = g;
    return BTG_OK;
}

btg_status btg_grid_set_dims(btg_grid g, size_t nd, size_t nm, size_t nt) {
    if (!g) return gfail(BTG_EARG, "null grid");
    std::lock_guard<std::mutex> lock(g->mu);
    if (nd == 0 || nm == 0 || nt == 0) return gfail(BTG_EDIM, "compact operator: all dimensions must be positive");
    if (g->dims_set) {
        if (g->nd != nd || g->nm != nm || g->nt != nt) return gfail(BTG_EDIM, "grid: dims already set differently");
        return BTG_OK;
    }
    g->nd = nd;
    g->nm = nm;
    g->nt = nt;
    G_TRY(skeleton(g));
    g->dims_set = true;
    return BTG_OK;
}

btg_status btg_grid_setup(btg_grid g, const double* blocks, size_t nd, size_t nm, size_t nt, int precision,
                          unsigned flags) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (!blocks) return gfail(BTG_EARG, "null blocks");
    G_TRY(btg_grid_set_dims(g, nd, nm, nt));
    const bool dev = flags & BTG_DEVICE_PTRS;
    for (auto& c : g->cells) {
        const auto& b = g->bounds[c.rank];
        const size_t ld = b.i1 - b.i0, lm = b.j1 - b.j0;
        if (ld == 0 || lm == 0) continue;
        btg_op op = nullptr;
        if (!g->local) {
            G_TRY(btg_setup(blocks, ld, lm, nt, precision, c.device, flags, &op));
        } else if (dev) {
            // device-resident global blocks: transform the rectangle row by row
            G_TRY(btg_create(ld, lm, nt, precision, c.device, &op));
            double* rect = nullptr;
            {
                DevGuard dg(c.device);
                G_CUDA(cudaMalloc(&rect, nt * ld * lm * sizeof(double)));
                G_CUDA(cudaMemcpy3D([&] {
                    cudaMemcpy3DParms p{};
                    p.srcPtr = make_cudaPitchedPtr(const_cast<double*>(blocks) + b.i0 * nm + b.j0, nm * sizeof(double),
                                                   lm * sizeof(double), nd);
                    p.dstPtr = make_cudaPitchedPtr(rect, lm * sizeof(double), lm * sizeof(double), ld);
                    p.extent = make_cudaExtent(lm * sizeof(double), ld, nt);
                    p.kind = cudaMemcpyDefault;
                    return &p;
                }()));
            }
            btg_status s = btg_setup_rows(op, rect, 0, ld, BTG_DEVICE_PTRS);
            if (s == BTG_OK) s = btg_synchronize(op);
            cudaFree(rect);
            if (s != BTG_OK) {
                btg_destroy(op);
                return s;
            }
        } else {
            c.blocks.resize(nt * ld * lm);
            for (size_t k = 0; k < nt; ++k)
                for (size_t i = 0; i < ld; ++i)
                    std::memcpy(c.blocks.data() + (k * ld + i) * lm, blocks + (k * nd + b.i0 + i) * nm + b.j0,
                                lm * sizeof(double));
            G_TRY(btg_setup(c.blocks.data(), ld, lm, nt, precision, c.device, flags & BTG_KEEP_CHANNEL_LAYOUT, &op));
        }
        G_TRY(bind_op(c, op, true));
    }
    return BTG_OK;
}

btg_status btg_grid_from_operator(btg_grid g, btg_op global) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (!g->local) return gfail(BTG_EARG, "from_operator: local grids only (one-rank grids attach their shard)");
    size_t nd = 0, nm = 0, nt = 0;
    int prec = 0;
    G_TRY(btg_get_dims(global, &nd, &nm, &nt, &prec));
    G_TRY(btg_grid_set_dims(g, nd, nm, nt));
    int layout = 0;
    btg_has_channel_layout(global, &layout);
    for (auto& c : g->cells) {
        const auto& b = g->bounds[c.rank];
        if (b.i1 == b.i0 || b.j1 == b.j0) continue;
        btg_op op = nullptr;
        G_TRY(btg_slice_operator(global, b.i0, b.i1, b.j0, b.j1, c.device, &op));
        if (layout) btg_set_channel_layout(op, 1);
        G_TRY(bind_op(c, op, true));
    }
    return BTG_OK;
}

btg_status btg_grid_attach(btg_grid g, size_t rank, btg_op shard, int take_ownership) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (!g->dims_set) return gfail(BTG_EARG, "attach: set the grid's operator dims first");
    Cell* c = find_cell(g, rank);
    if (!c) return gfail(BTG_EGRID, "attach: cell " + std::to_string(rank) + " is not local to this process");
    const auto& b = g->bounds[rank];
    if (shard) {
        size_t nd = 0, nm = 0, nt = 0;
        G_TRY(btg_get_dims(shard, &nd, &nm, &nt, nullptr));
        if (nd != b.i1 - b.i0 || nm != b.j1 - b.j0 || nt != g->nt)
            return gfail(BTG_EDIM, "attach: shard is " + std::to_string(nd) + "x" + std::to_string(nm) + "x" +
                                       std::to_string(nt) + ", cell " + std::to_string(rank) + " needs " +
                                       std::to_string(b.i1 - b.i0) + "x" + std::to_string(b.j1 - b.j0) + "x" +
                                       std::to_string(g->nt));
    } else if (b.i1 > b.i0 && b.j1 > b.j0) {
        return gfail(BTG_EARG, "attach: cell " + std::to_string(rank) + " is not empty and needs an operator");
    }
    std::lock_guard<std::mutex> lock(g->mu);
    return bind_op(*c, shard, take_ownership != 0);
}

btg_status btg_grid_shard(btg_grid g, size_t rank, size_t* bounds, btg_op* op) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (!g->dims_set) return gfail(BTG_EARG, "grid: operator dims not set");
    if (rank >= g->rows * g->cols) return gfail(BTG_EGRID, "shard index outside the grid");
    const auto& b = g->bounds[rank];
    if (bounds) {
        bounds[0] = b.i0;
        bounds[1] = b.i1;
        bounds[2] = b.j0;
        bounds[3] = b.j1;
    }
    if (op) {
        Cell* c = find_cell(g, rank);
        *op = c ? c->op : nullptr;
    }
    return BTG_OK;
}

btg_status btg_grid_info(btg_grid g, size_t* rows, size_t* cols, size_t* rank, int* transport) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (rows) *rows = g->rows;
    if (cols) *cols = g->cols;
    if (rank) *rank = g->my_rank;
    if (transport) *transport = g->transport;
    return BTG_OK;
}

btg_status btg_grid_forward(btg_grid g, const double* m, size_t m_len, double* d, size_t d_len, unsigned flags) {
    CallArgs a;
    a.in = m;
    a.in_len = m_len;
    a.out = d;
    a.out_len = d_len;
    a.flags = flags;
    return run(g, BTG_GRID_FORWARD, a);
}

btg_status btg_grid_adjoint(btg_grid g, const double* d, size_t d_len, double* m, size_t m_len, unsigned flags) {
    CallArgs a;
    a.in = d;
    a.in_len = d_len;
    a.out = m;
    a.out_len = m_len;
    a.flags = flags;
    return run(g, BTG_GRID_ADJOINT, a);
}

btg_status btg_grid_hessian(btg_grid g, const double* v, size_t v_len, double* hv, size_t hv_len,
                            const double* gamma_inv, int gamma_kind, double alpha, int reg_kind, unsigned flags) {
    CallArgs a;
    a.in = v;
    a.in_len = v_len;
    a.out = hv;
    a.out_len = hv_len;
    a.gamma = gamma_inv;
    a.gamma_kind = gamma_kind;
    a.alpha = alpha;
    a.reg_kind = reg_kind;
    a.flags = flags;
    return run(g, BTG_GRID_HESSIAN, a);
}

btg_status btg_grid_set_backend(btg_grid g, int backend, int parallel) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (backend < 0 || backend > 2) return gfail(BTG_EARG, "unknown backend " + std::to_string(backend));
    std::lock_guard<std::mutex> lock(g->mu);
    if (backend == 1)
        for (auto& c : g->cells) {
            int keep = 0;
            if (c.op && (btg_has_channel_layout(c.op, &keep) != BTG_OK || !keep))
                return gfail(BTG_EARG, "distributed apply: ewp backend needs a partition set up with "
                                       "keep_channel_layout");
        }
    if (backend == 2)
        for (auto& c : g->cells)
            if (c.op && c.blocks.empty() && !c.d_blocks)
                return gfail(BTG_EARG, "distributed apply: naive backend needs time-domain blocks (partition of a "
                                       "compact operator)");
    g->backend = backend;
    g->parallel = parallel != 0;
    return BTG_OK;
}

btg_status btg_grid_set_stream(btg_grid g, void* stream) {
    if (!g) return gfail(BTG_EARG, "null grid");
    if (g->local) return gfail(BTG_EARG, "set_stream: one-rank grids only");
    std::lock_guard<std::mutex> lock(g->mu);
    Cell& c = g->cells[0];
    c.stream = stream ? static_cast<cudaStream_t>(stream) : c.own_stream;
    if (c.op) G_TRY(btg_set_stream(c.op, c.stream));
    return BTG_OK;
}

btg_status btg_grid_synchronize(btg_grid g) {
    if (!g) return gfail(BTG_EARG, "null grid");
    for (auto& c : g->cells) {
        DevGuard dg(c.device);
        G_CUDA(cudaStreamSynchronize(c.stream));
    }
    return BTG_OK;
}

btg_status btg_grid_comm_log(btg_grid g, btg_comm_event* out, size_t cap, size_t* count) {
    if (!g) return gfail(BTG_EARG, "null grid");
    std::lock_guard<std::mutex> lock(g->mu);
    if (count) *count = g->log.size();
    if (out) {
        if (cap < g->log.size()) return gfail(BTG_EARG, "comm log: capacity too small");
        std::copy(g->log.begin(), g->log.end(), out);
    }
    return BTG_OK;
}

btg_status btg_grid_reset_comm_log(btg_grid g) {
    if (!g) return gfail(BTG_EARG, "null grid");
    std::lock_guard<std::mutex> lock(g->mu);
    g->log.clear();
    return BTG_OK;
}

void btg_grid_destroy(btg_grid g) {
    if (!g) return;
    for (auto& c : g->cells) destroy_cell(c);
    delete g;
}

// ---- the reference's single-process Partition over a local P2P grid ------------
btg_status btg_partition_create(const double* blocks, size_t nd, size_t nm, size_t nt, size_t rows, size_t cols,
                                const int* devices, size_t num_devices, int precision, unsigned flags,
                                btg_partition* out) {
    if (!out) return gfail(BTG_EARG, "null output handle");
    *out = nullptr;
    if (!blocks) return gfail(BTG_EARG, "null blocks");
    if (nd == 0 || nm == 0 || nt == 0) return gfail(BTG_EDIM, "compact operator: all dimensions must be positive");
    btg_grid g = nullptr;
    G_TRY(check_grid(rows, cols));
    G_TRY(btg_grid_create_local(rows, cols, devices, num_devices, BTG_TRANSPORT_P2P, &g));
    btg_status s = btg_grid_setup(g, blocks, nd, nm, nt, precision, flags & BTG_KEEP_CHANNEL_LAYOUT);
    if (s != BTG_OK) {
        const std::string msg = btg_last_error();
        btg_grid_destroy(g);
        return gfail(s, msg);
    }
    *out = g;
    return BTG_OK;
}

btg_status btg_partition_from_operator(btg_op op, size_t rows, size_t cols, const int* devices, size_t num_devices,
                                       btg_partition* out) {
    if (!out) return gfail(BTG_EARG, "null output handle");
    *out = nullptr;
    if (!op) return gfail(BTG_EARG, "null operator handle");
    btg_grid g = nullptr;
    G_TRY(btg_grid_create_local(rows, cols, devices, num_devices, BTG_TRANSPORT_P2P, &g));
    btg_status s = btg_grid_from_operator(g, op);
    if (s != BTG_OK) {
        const std::string msg = btg_last_error();
        btg_grid_destroy(g);
        return gfail(s, msg);
    }
    *out = g;
    return BTG_OK;
}

btg_status btg_partition_shard(btg_partition p, size_t row, size_t col, size_t* bounds, btg_op* op) {
    if (!p) return gfail(BTG_EARG, "null partition");
    if (row >= p->rows || col >= p->cols) return gfail(BTG_EGRID, "shard index outside the grid");
    return btg_grid_shard(p, row * p->cols + col, bounds, op);
}

btg_status btg_partition_forward(btg_partition p, const double* m, size_t m_len, double* d, size_t d_len,
                                 int backend, int parallel) {
    G_TRY(btg_grid_set_backend(p, backend, parallel));
    return btg_grid_forward(p, m, m_len, d, d_len, 0u);
}

btg_status btg_partition_adjoint(btg_partition p, const double* d, size_t d_len, double* m, size_t m_len,
                                 int backend, int parallel) {
    G_TRY(btg_grid_set_backend(p, backend, parallel));
    return btg_grid_adjoint(p, d, d_len, m, m_len, 0u);
}

btg_status btg_partition_hessian(btg_partition p, const double* v, size_t v_len, double* hv, size_t hv_len,
                                 const double* gamma_inv, int gamma_kind, double alpha, int reg_kind, int backend,
                                 int parallel) {
    G_TRY(btg_grid_set_backend(p, backend, parallel));
    return btg_grid_hessian(p, v, v_len, hv, hv_len, gamma_inv, gamma_kind, alpha, reg_kind, 0u);
}

void btg_partition_destroy(btg_partition p) { btg_grid_destroy(p); }

}  // extern "C"
