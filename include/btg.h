/*
 * btg.h — C ABI of the B200-native FFT block-Toeplitz matvec (libbtg.so).
 *
 * Drop-in boundary for the reference's operator API (paths are relative to
 * /root/reference/proj). The reference is C++ with value semantics; this ABI
 * is what its FFI for the hot path binds: plain pointers and sizes, an opaque
 * handle that owns the device-resident frequency-domain operator, status codes
 * instead of exceptions. include/btoep_gpu.hpp re-exposes the reference's C++
 * signatures on top of it; INTEGRATION.md shows the bindings.
 *
 * Layouts (identical to the reference's, so no caller-side reordering):
 *   blocks  TOSI first block column  blocks[(k*N_d + i)*N_m + j], k < N_t
 *           (CompactP2O::entry, block_operator.cpp:147-153)
 *   m, d    SOTI space-time vectors  v[s*N_t + t]   (space_time.hpp:10-11)
 *           nrhs > 1 stacks right-hand sides: v[(r*dim + s)*N_t + t]
 *   F-hat   device-resident, frequency-major [f][i][j] for f <= N_t
 *           (the reference's freq_blocks, block_operator.cpp:164-167,199-202,
 *           truncated to the N_t+1 non-redundant frequencies of a real signal).
 *
 * Pointer arguments are host pointers unless BTG_DEVICE_PTRS is set in
 * `flags`, in which case they are device pointers on the handle's device and
 * no host<->device copies happen. All calls on one handle are serialized
 * (internal mutex); distinct handles may be used concurrently.
 */
#ifndef BTG_H_
#define BTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BTG_ABI_VERSION 1

typedef enum {
    BTG_OK = 0,
    BTG_EDIM = 1,    /* shape/length mismatch  -> btoep::DimensionError (block_operator.cpp:123-133) */
    BTG_EORDER = 2,  /* wrong ordering tag     -> btoep::OrderingError (space_time.cpp:39-44)      */
    BTG_EARG = 3,    /* invalid argument / state -> btoep::Error                                   */
    BTG_ECUDA = 4,   /* CUDA runtime failure                                                       */
    BTG_ENOMEM = 5,  /* device allocation failed                                                   */
    BTG_EGRID = 6,   /* unserviceable processor grid -> btoep::GridError (distributed.cpp:147-152) */
    BTG_ESOLVER = 7, /* CG lost positive definiteness -> btoep::SolverError (inverse.cpp:124-136) */
    BTG_EFORMAT = 8, /* malformed / inconsistent file -> btoep::FormatError (io.cpp)              */
    BTG_ENCCL = 9    /* NCCL / grid transport failure                                             */
} btg_status;

typedef enum { BTG_F64 = 64, BTG_F32 = 32 } btg_precision;

/* flags */
#define BTG_DEVICE_PTRS 0x1u  /* data pointers are device pointers */
#define BTG_KEEP_CHANNEL_LAYOUT 0x2u  /* btg_setup: SetupOptions::keep_channel_layout (EWP backend) */

/* Hessian options (inverse.hpp:16; Gamma^-1 is the north star's noise weighting) */
typedef enum { BTG_REG_IDENTITY = 0, BTG_REG_TEMPORAL_LAPLACIAN = 1 } btg_reg_kind;
typedef enum {
    BTG_GAMMA_NONE = 0,        /* Gamma^-1 = I                     */
    BTG_GAMMA_PER_SENSOR = 1,  /* gamma_inv[i], length N_d         */
    BTG_GAMMA_PER_SAMPLE = 2   /* gamma_inv[i*N_t + t], N_d x N_t  */
} btg_gamma_kind;

/* Mirrors btoep::StageCounters / PipelineCounters (counters.hpp:12-45). On the
 * GPU pad+forward_fft+reorder_in run as ONE fused kernel (reported under
 * forward_fft) and reorder_out+inverse_fft+unpad as one (inverse_fft). Bytes
 * follow the algorithmic model with N_t+1 frequencies; seconds are CUDA-event
 * times, filled only while btg_set_timing(op, 1) is active. */
typedef struct { double ops, bytes, seconds; } btg_stage_counters;
typedef struct {
    btg_stage_counters pad, forward_fft, reorder_in, apply, reorder_out, inverse_fft, unpad;
    uint64_t launches; /* kernels this handle launched */
} btg_counters;

typedef struct btg_op_s* btg_op;

/* Thread-local message of the last failing call on this thread. */
const char* btg_last_error(void);
int btg_abi_version(void);

/* Allocate the device operator (F-hat uninitialised). Replaces the allocation
 * half of btoep::setup (block_operator.hpp:64, block_operator.cpp:178-205). */
btg_status btg_create(size_t num_sensors, size_t num_sources, size_t num_steps,
                      int precision, int device, btg_op* out);

/* Setup (Alg. 1) for the sensor rows [sensor_begin, sensor_end): `blocks` is
 * the TOSI first block column RESTRICTED to those rows, shape
 * (N_t, sensor_end-sensor_begin, N_m). Zero-pad to 2N_t, R2C along time,
 * write F-hat frequency-major. Lets a caller stream an operator too large to
 * hold twice in HBM. block_operator.cpp:178-205. */
btg_status btg_setup_rows(btg_op op, const double* blocks, size_t sensor_begin,
                          size_t sensor_end, unsigned flags);

/* create + setup_rows(0, N_d): the drop-in for btoep::setup. */
btg_status btg_setup(const double* blocks, size_t num_sensors, size_t num_sources,
                     size_t num_steps, int precision, int device, unsigned flags,
                     btg_op* out);

/* d = F m (Alg. 2). m: nrhs x N_m x N_t SOTI (m_len elements), d: nrhs x N_d x N_t.
 * btoep::apply_forward, block_operator.hpp:71 / block_operator.cpp:218-273. */
btg_status btg_forward(btg_op op, const double* m, size_t m_len, double* d, size_t d_len,
                       size_t nrhs, unsigned flags);

/* m = F* d (Alg. 3), same operator, conjugate-transpose indexing.
 * btoep::apply_adjoint, block_operator.hpp:76 / block_operator.cpp:275-331. */
btg_status btg_adjoint(btg_op op, const double* d, size_t d_len, double* m, size_t m_len,
                       size_t nrhs, unsigned flags);

/* hv = F* Gamma^-1 F v + alpha R v. With gamma_kind = BTG_GAMMA_NONE this is
 * btoep::HessianOperator::apply (inverse.hpp:32-39, inverse.cpp:78-91). */
btg_status btg_hessian(btg_op op, const double* v, size_t v_len, double* hv, size_t hv_len,
                       size_t nrhs, const double* gamma_inv, int gamma_kind, double alpha,
                       int reg_kind, unsigned flags);

/* Device-resident conjugate gradients on (F* Gamma^-1 F + alpha R) x = rhs,
 * optionally preconditioned with R^-1 (Thomas solve per source): the caller
 * of the Hessian action, btoep::cg_solve (inverse.hpp:51-53, inverse.cpp:105-156),
 * same stopping rule (relative residual <= tol; max_iterations = 0 selects
 * 10 ceil(sqrt(N_m N_t)) + 1) and the same SolverError conditions
 * (BTG_ESOLVER). x starts at zero. Vectors stay in HBM; only the scalars of
 * each iteration cross to the host. */
typedef struct {
    size_t iterations;
    double relative_residual;
    int converged;
    double seconds;  /* device time of the solve */
} btg_cg_result;

btg_status btg_cg_solve(btg_op op, const double* rhs, size_t rhs_len, double* x, size_t x_len,
                        const double* gamma_inv, int gamma_kind, double alpha, int reg_kind,
                        double tol, size_t max_iterations, int use_reg_preconditioner,
                        unsigned flags, btg_cg_result* result);

/* 1/2 |F m - d_obs|^2 + alpha/2 m^T R m  (btoep::objective_eval, inverse.cpp:93-103). */
btg_status btg_objective(btg_op op, const double* m, size_t m_len, const double* d_obs, size_t d_len,
                         double alpha, int reg_kind, unsigned flags, double* value);

/* Fused output epilogue of one direction (the C2R store, K9): y = Gamma^-1 x
 * (gamma_kind != NONE; per output channel or per (channel, t)) + alpha R reg_v
 * (alpha != 0; reg_v has the output's layout). Used to compose the
 * Gauss-Newton action across a processor grid without extra passes. */
typedef struct {
    const double* gamma_inv;
    int gamma_kind;
    const double* reg_v;
    double alpha;
    int reg_kind;
} btg_epilogue;

btg_status btg_forward_ex(btg_op op, const double* m, size_t m_len, double* d, size_t d_len,
                          size_t nrhs, const btg_epilogue* epi, unsigned flags);
btg_status btg_adjoint_ex(btg_op op, const double* d, size_t d_len, double* m, size_t m_len,
                          size_t nrhs, const btg_epilogue* epi, unsigned flags);

/* Run subsequent work on `stream` (a cudaStream_t). NULL selects the handle's
 * own non-blocking stream; pass cudaStreamLegacy ((void*)0x1) for the legacy
 * default stream. Device-pointer calls are asynchronous on that stream. */
btg_status btg_set_stream(btg_op op, void* stream);
btg_status btg_synchronize(btg_op op);
btg_status btg_set_timing(btg_op op, int enabled);

/* Engine of the multi-right-hand-side Fourier step (nrhs > 1, FP64 F-hat):
 * BTG_MRHS_DMMA (default) = ZGEMM on the FP64 tensor cores (mma.sync f64);
 * BTG_MRHS_TENSOR_I8 = exact-integer Ozaki splitting on the tcgen05 int8 tensor
 * cores (7 signed 7-bit digits per 1024-wide block scale; int8 slices of F-hat
 * are built on first use, 14 B per complex entry). The environment variable
 * BTG_TENSOR_I8 selects the latter at creation. */
typedef enum { BTG_MRHS_DMMA = 0, BTG_MRHS_TENSOR_I8 = 1 } btg_mrhs_engine;

/* EWP backend (the paper's Appendix A; block_operator.cpp:345-421): the
 * Fourier-space step as element-wise products over the channel-major spectrum
 * (SpectralP2O::channel_spectra, block_operator.hpp:45). The layout is kept when
 * the operator is set up with BTG_KEEP_CHANNEL_LAYOUT (or after
 * btg_set_channel_layout(op, 1)) and built on the device on first use; without
 * it the EWP calls fail with BTG_EARG like require_channel_layout
 * (block_operator.cpp:335-341). One right-hand side, SOTI vectors. */
btg_status btg_set_channel_layout(btg_op op, int keep);

/* Naive backend (naive_apply_forward / naive_apply_adjoint,
 * block_operator.cpp:423-482): the direct O(N_t^2 N_d N_m) triangular sum on the
 * compact TOSI blocks (N_t x N_d x N_m) with SOTI vectors, in the reference's
 * summation order; stateless (no handle). */
btg_status btg_naive_forward(const double* blocks, size_t num_sensors, size_t num_sources, size_t num_steps,
                             const double* m, double* d, int device, unsigned flags);
btg_status btg_naive_adjoint(const double* blocks, size_t num_sensors, size_t num_sources, size_t num_steps,
                             const double* d, double* m, int device, unsigned flags);
btg_status btg_has_channel_layout(btg_op op, int* out);
btg_status btg_forward_ewp(btg_op op, const double* m, size_t m_len, double* d, size_t d_len, unsigned flags);
btg_status btg_adjoint_ewp(btg_op op, const double* d, size_t d_len, double* m, size_t m_len, unsigned flags);
btg_status btg_set_multi_rhs_engine(btg_op op, int engine);
btg_status btg_get_counters(btg_op op, btg_counters* out);
btg_status btg_reset_counters(btg_op op);
btg_status btg_get_dims(btg_op op, size_t* num_sensors, size_t* num_sources,
                        size_t* num_steps, int* precision);

/* Copy F-hat to host complex128 (interleaved re,im). full = 1: the reference's
 * 2*N_t-frequency layout (freq_blocks, block_operator.hpp:40) with the upper
 * half rebuilt by conjugate symmetry; full = 0: the N_t+1 stored frequencies. */
btg_status btg_export_spectrum(btg_op op, double* out, int full);

/* One stored frequency block f <= N_t (N_d x N_m complex128) to host memory. */
btg_status btg_export_spectrum_block(btg_op op, size_t f, double* out);

/* ---- reference file formats (proj/include/btoep/io.hpp, src/io.cpp) ---------
 * "BTOP" operator files (64-byte header; time domain: N_t real64 TOSI blocks;
 * frequency domain: 2 N_t complex128 blocks) and "BTVC" vector files. */
typedef struct {
    int ordering;        /* 0 TOSI, 1 SOTI */
    int domain;          /* 0 time, 1 frequency */
    uint64_t num_sensors, num_sources, num_steps;
    int complex_scalar;
} btg_file_header;

btg_status btg_peek_operator(const char* path, btg_file_header* out);       /* io::peek_operator */
/* Build the device operator from a file (streamed; never whole in host memory):
 * time domain -> setup (Alg. 1); frequency domain -> the N_t+1 stored blocks. */
btg_status btg_load_operator(const char* path, int precision, int device, btg_op* out);
/* The shard of one grid cell: sensors [i0, i1) x sources [j0, j1) of a file.
 * Time domain -> setup of the rectangle (partition_operator(CompactP2O),
 * distributed.cpp:179-196); frequency domain -> the rectangle of every stored
 * block, no re-setup (partition_operator(SpectralP2O), distributed.cpp:198-218). */
btg_status btg_load_operator_rect(const char* path, size_t i0, size_t i1, size_t j0, size_t j1,
                                  int precision, int device, btg_op* out);
/* io::write_operator(CompactP2O) / io::read_compact_operator (io.cpp:97-111,159-180):
 * time-domain TOSI files of the first block column (N_t x N_d x N_m). read:
 * blocks == NULL queries the dimensions only. */
btg_status btg_write_compact(const char* path, const double* blocks, size_t num_sensors, size_t num_sources,
                             size_t num_steps);
btg_status btg_read_compact(const char* path, double* blocks, size_t capacity, size_t* num_sensors,
                            size_t* num_sources, size_t* num_steps);
/* io::write_operator(SpectralP2O): the reference's 2 N_t frequency-domain file. */
btg_status btg_save_operator(btg_op op, const char* path);
btg_status btg_write_vector(const char* path, const double* values, size_t spatial_dim,
                            size_t num_steps, int ordering);                 /* io::write_vector */
/* io::read_vector; values == NULL queries the dimensions only. */
btg_status btg_read_vector(const char* path, double* values, size_t capacity, size_t* spatial_dim,
                           size_t* num_steps, int* ordering);

/* partition_operator(const SpectralP2O&) (distributed.hpp:61-66,
 * distributed.cpp:198-218) without a host round trip: a new handle on `device`
 * holding sensors [i0, i1) x sources [j0, j1) of every stored frequency block
 * of `src`, copied HBM->HBM (peer-to-peer over NVLink when the devices differ).
 * Entries are bit-identical to the source's. Empty/out-of-range -> BTG_EGRID. */
btg_status btg_slice_operator(btg_op src, size_t i0, size_t i1, size_t j0, size_t j1, int device,
                              btg_op* out);

/* Grid planner, reference criterion (grid_planner.hpp:43-65): the scale-free cost
 * (r/p) ln r + (10^l/r) ln(p/r), l = log10(N_d/N_m), its minimiser snapped to an
 * r x c factorisation of `workers` with the reference's preferences
 * (select_grid, grid_planner.cpp:123-193), the weak-scaling choice (:195-207)
 * and the broadcast+reduce model (:105-114). */
btg_status btg_select_grid(size_t workers, double log_dim_ratio, unsigned gpus_per_node, size_t* rows,
                           size_t* cols);
btg_status btg_weak_scaling_shape(double local_ratio, size_t workers, int* indifferent, size_t* rows,
                                  size_t* cols);
btg_status btg_modified_cost(double rows, size_t workers, double log_dim_ratio, double* out);
btg_status btg_comm_cost(size_t rows, size_t cols, size_t num_sources, size_t num_sensors, size_t num_steps,
                         double latency, double bandwidth, double* out);
/* CostEstimate / conventional_cost_estimate (grid_planner.hpp:84-97) and
 * apply_arithmetic_intensity (grid_planner.hpp:100). */
typedef struct {
    double per_solve_flops, effective_rank, conventional_total_flops, fft_setup_flops, fft_matvec_flops,
        fft_total_flops, ratio;
} btg_cost_estimate;
btg_status btg_conventional_cost_estimate(double grid_points, double num_steps, double num_sensors,
                                          double rank_fraction, btg_cost_estimate* out);
double btg_apply_arithmetic_intensity(double local_sensors, double local_sources);

/* B200 / NVSwitch planner: the modelled time of one action
 * (btg_grid_kind) of the grid engine's schedule on every r x c factorisation of
 * `workers` — the worst shard's HBM stream and vector transforms plus the NCCL
 * ring collectives at NVLink-5 rates inside the NVSwitch domain (the node link
 * outside it). `best` = the cheapest (ties to fewer rows); `all` (optional,
 * `cap` entries) = every feasible factorisation, rows ascending. hw NULL =
 * btg_default_hw_model (measured B200 rates). */
typedef struct {
    double hbm_gbs;        /* local F-hat stream, GB/s            */
    double fft_gbs;        /* vector transforms, GB/s             */
    double link_gbs;       /* NVLink per direction per GPU, GB/s  */
    double node_link_gbs;  /* between NVSwitch domains, GB/s      */
    double latency_us;     /* per ring step                       */
    unsigned gpus_per_node;
} btg_hw_model;
typedef struct {
    size_t rows, cols;
    double seconds, local_seconds, comm_seconds;
} btg_grid_plan;
btg_status btg_default_hw_model(btg_hw_model* out);
btg_status btg_plan_grid(size_t num_sensors, size_t num_sources, size_t num_steps, size_t workers, int precision,
                         int kind, const btg_hw_model* hw, btg_grid_plan* best, btg_grid_plan* all, size_t cap,
                         size_t* count);

/* ---- processor grid engine (distributed.hpp:43-121, distributed.cpp:145-392) ----
 * An r x c grid over N_d x N_m: grid cell (i, j) = rank i*c + j owns sensors
 * [i*ceil(N_d/r), ...) x sources [j*ceil(N_m/c), ...) of every stored frequency
 * block (the reference's ceiling partition, distributed.cpp:145-175; trailing
 * shards may be empty; grids wider than the operator -> BTG_EGRID). One
 * schedule (btg_grid_schedule) drives every transport:
 *   F  (distributed.cpp:312-351): column broadcast of the parameter slice from
 *      row 0, local F, row reduce (sum) onto column 0;
 *   F* (distributed.cpp:353-392): row broadcast of the data slice from column 0,
 *      local F*, column reduce onto row 0;
 *   H  (inverse.cpp:78-91 on a partition, + Gamma^-1): column broadcast, local F
 *      with Gamma^-1 in its C2R epilogue, ONE row all-reduce (the F reduce and
 *      the F* broadcast merged), local F* with alpha R v added on row 0, column
 *      reduce onto row 0.
 * Transports:
 *   NCCL  (btg_grid_create: one process per GPU, ncclCommInitRank + ncclCommSplit
 *          into row / column communicators; btg_grid_create_local with
 *          BTG_TRANSPORT_NCCL: every cell in this process on distinct devices,
 *          ncclCommInitAll). NCCL_ALGO=Ring / NCCL_PROTO=Simple are pinned at
 *          creation (unless already set in the environment) so a fixed grid
 *          gives run-to-run identical bits.
 *   P2P   (btg_grid_create_local with BTG_TRANSPORT_P2P: the reference's
 *          single-process Partition; any device placement, several cells per
 *          device allowed): device-to-device copies and a sum kernel that adds
 *          the partials in the reference's fixed binary tree order
 *          (tree_reduce, distributed.cpp:36-47), so results are bit-identical
 *          to tree-summing the same partials and serial == parallel.
 *   external (btg_grid_create_external): host callbacks; used by the tests to
 *          run several ranks on ONE GPU over torch.distributed/gloo (NCCL
 *          refuses two ranks on one device). Not a compute path. */
typedef struct btg_grid_s* btg_grid;

typedef enum { BTG_GRID_FORWARD = 0, BTG_GRID_ADJOINT = 1, BTG_GRID_HESSIAN = 2 } btg_grid_kind;
typedef enum {
    BTG_STEP_INPUT = 0,     /* caller's slice -> buffer dst (active ranks own the input)        */
    BTG_STEP_BROADCAST = 1, /* buffer src from the group's member `root` to the whole group      */
    BTG_STEP_FORWARD = 2,   /* local F: src -> dst (gamma: Gamma^-1 rows of this shard)          */
    BTG_STEP_ADJOINT = 3,   /* local F*: src -> dst (reg: + alpha R (buffer 0) in the epilogue) */
    BTG_STEP_REDUCE = 4,    /* sum of buffer src over the group onto member `root`               */
    BTG_STEP_ALLREDUCE = 5, /* sum of buffer src over the group, on every member                */
    BTG_STEP_OUTPUT = 6     /* buffer src -> caller (active ranks return the output slice)       */
} btg_step_op;
typedef enum { BTG_GROUP_ROW = 0, BTG_GROUP_COL = 1 } btg_group_kind;
typedef struct {
    int op;        /* btg_step_op */
    int group;     /* collectives: btg_group_kind (row i: members j = 0..c-1; column j: members i) */
    int root;      /* collectives: member index of the root within the group */
    int src, dst;  /* buffer ids 0, 1, 2 */
    int active;    /* INPUT / OUTPUT: this rank takes part */
    int gamma;     /* FORWARD: apply Gamma^-1 */
    int reg;       /* ADJOINT: add alpha R (buffer 0) */
    size_t count;  /* doubles in the buffer this step touches on this rank */
} btg_grid_step;

/* The per-rank schedule (host logic only; the executor and the tests run it).
 * Every rank of a grid gets the same sequence of step ops; `active`, `gamma`,
 * `reg` and `count` are rank-specific. Steps over groups of one member are
 * omitted. */
btg_status btg_grid_schedule(size_t num_sensors, size_t num_sources, size_t num_steps, size_t rows, size_t cols,
                             size_t rank, int kind, int with_gamma, int with_reg, btg_grid_step* steps, size_t cap,
                             size_t* count);

/* CommLog events of the reference's byte model (record_collective,
 * distributed.cpp:23-34) for one F (kind 0) or F* (kind 1) over the grid. */
typedef struct {
    int phase;  /* 0 "broadcast", 1 "reduce" */
    size_t participants, messages;
    uint64_t link_bytes, total_bytes;
    size_t tree_depth;
} btg_comm_event;
btg_status btg_comm_events(size_t num_sensors, size_t num_sources, size_t num_steps, size_t rows, size_t cols,
                           int kind, btg_comm_event* out, size_t cap, size_t* count);

typedef enum { BTG_TRANSPORT_NCCL = 0, BTG_TRANSPORT_P2P = 1, BTG_TRANSPORT_EXTERNAL = 2 } btg_transport;
#define BTG_NCCL_ID_BYTES 128

/* ncclGetUniqueId: rank 0 creates it and ships the bytes to the other ranks. */
btg_status btg_grid_nccl_id(void* id_out /* BTG_NCCL_ID_BYTES */);
/* Multi-process grid: this process is grid cell `rank` on `device` (NCCL). */
btg_status btg_grid_create(size_t rows, size_t cols, size_t rank, const void* nccl_id, int device, btg_grid* out);
/* Single-process grid: every cell in this process, cell k on devices[k % num_devices]
 * (NULL: device 0). transport: BTG_TRANSPORT_P2P or BTG_TRANSPORT_NCCL (needs
 * rows*cols distinct devices). */
btg_status btg_grid_create_local(size_t rows, size_t cols, const int* devices, size_t num_devices, int transport,
                                 btg_grid* out);
/* Host-callback transport for one rank (tests). Buffers are page-locked host
 * copies of `n` doubles; return 0 on success. */
typedef struct {
    void* user;
    int (*broadcast)(void* user, int group, double* buf, size_t n, int root);
    int (*reduce)(void* user, int group, double* buf, size_t n, int root);
    int (*allreduce)(void* user, int group, double* buf, size_t n);
} btg_grid_callbacks;
btg_status btg_grid_create_external(size_t rows, size_t cols, size_t rank, int device, const btg_grid_callbacks* cb,
                                    btg_grid* out);

/* Global operator dims (fixes the partition). Implied by setup / from_operator. */
btg_status btg_grid_set_dims(btg_grid g, size_t num_sensors, size_t num_sources, size_t num_steps);
/* Setup (partition_operator(CompactP2O), distributed.cpp:179-196). Local grids:
 * `blocks` is the global TOSI first block column (N_t x N_d x N_m) and every
 * cell transforms its rectangle; one-rank grids: `blocks` is this rank's
 * rectangle (N_t x local N_d x local N_m). Host pointer unless BTG_DEVICE_PTRS. */
btg_status btg_grid_setup(btg_grid g, const double* blocks, size_t num_sensors, size_t num_sources, size_t num_steps,
                          int precision, unsigned flags);
/* partition_operator(const SpectralP2O&) (distributed.cpp:198-218) for a local
 * grid: every cell slices its rectangle of `global` HBM->HBM (btg_slice_operator). */
btg_status btg_grid_from_operator(btg_grid g, btg_op global);
/* Adopt `shard` (dims = the cell's rectangle; NULL for an empty cell) as the
 * operator of cell `rank` (must be local). take_ownership: destroyed with the grid. */
btg_status btg_grid_attach(btg_grid g, size_t rank, btg_op shard, int take_ownership);
/* bounds[4] = sensor_begin, sensor_end, source_begin, source_end of cell `rank`;
 * *op = its operator when local (else NULL). */
btg_status btg_grid_shard(btg_grid g, size_t rank, size_t* bounds, btg_op* op);
/* rows, cols; rank = this process's cell (SIZE_MAX for a local grid); transport */
btg_status btg_grid_info(btg_grid g, size_t* rows, size_t* cols, size_t* rank, int* transport);

/* Local grids: global SOTI vectors (N_m x N_t, N_d x N_t). One-rank grids: this
 * rank's slices — inputs on the ranks whose INPUT step is active (F, H: row 0;
 * F*: column 0), outputs on the OUTPUT-active ranks (F: column 0; F*, H: row 0);
 * pass NULL / 0 elsewhere. Host pointers unless BTG_DEVICE_PTRS (then the call
 * is asynchronous on the grid stream). distributed_forward / distributed_adjoint
 * (distributed.cpp:312-392); btg_grid_hessian: F* Gamma^-1 F v + alpha R v with a
 * GLOBAL gamma_inv (N_d or N_d x N_t; each cell uses its rows). */
btg_status btg_grid_forward(btg_grid g, const double* m, size_t m_len, double* d, size_t d_len, unsigned flags);
btg_status btg_grid_adjoint(btg_grid g, const double* d, size_t d_len, double* m, size_t m_len, unsigned flags);
btg_status btg_grid_hessian(btg_grid g, const double* v, size_t v_len, double* hv, size_t hv_len,
                            const double* gamma_inv, int gamma_kind, double alpha, int reg_kind, unsigned flags);
/* backend of the local step: 0 fft, 1 ewp (needs BTG_KEEP_CHANNEL_LAYOUT), 2 naive
 * (grids set up from time-domain blocks); parallel: one host thread per local cell
 * for the local step (ExecutionPolicy::Parallel). */
btg_status btg_grid_set_backend(btg_grid g, int backend, int parallel);
/* One-rank grids: run on `stream` (NULL = the grid's own stream). */
btg_status btg_grid_set_stream(btg_grid g, void* stream);
btg_status btg_grid_synchronize(btg_grid g);
/* The CommLog of the F / F* calls since creation (or the last reset). */
btg_status btg_grid_comm_log(btg_grid g, btg_comm_event* out, size_t cap, size_t* count);
btg_status btg_grid_reset_comm_log(btg_grid g);
void btg_grid_destroy(btg_grid g);

/* ---- single-process partition (distributed.hpp:43-121) ------------------------
 * partition_operator / distributed_forward / distributed_adjoint with global
 * host SOTI vectors: a local grid on the P2P transport (see above) — one device
 * handle per non-empty cell, placed round-robin on `devices` (NULL: device 0),
 * partial slices summed on the device in the reference's fixed tree order, so
 * `parallel` (one host thread per cell, the reference's ExecutionPolicy::Parallel)
 * gives bit-identical results. backend: 0 fft, 1 ewp (needs
 * BTG_KEEP_CHANNEL_LAYOUT), 2 naive (partitions of compact operators only, as in
 * the reference). */
typedef struct btg_grid_s* btg_partition;
btg_status btg_partition_create(const double* blocks, size_t num_sensors, size_t num_sources, size_t num_steps,
                                size_t rows, size_t cols, const int* devices, size_t num_devices, int precision,
                                unsigned flags, btg_partition* out);      /* partition_operator(CompactP2O) */
btg_status btg_partition_from_operator(btg_op op, size_t rows, size_t cols, const int* devices,
                                       size_t num_devices, btg_partition* out);  /* partition_operator(SpectralP2O) */
/* bounds[4] = sensor_begin, sensor_end, source_begin, source_end; *op NULL for an empty cell */
btg_status btg_partition_shard(btg_partition p, size_t row, size_t col, size_t* bounds, btg_op* op);
btg_status btg_partition_forward(btg_partition p, const double* m, size_t m_len, double* d, size_t d_len,
                                 int backend, int parallel);
btg_status btg_partition_adjoint(btg_partition p, const double* d, size_t d_len, double* m, size_t m_len,
                                 int backend, int parallel);
/* HessianOperator::apply with a partition (inverse.cpp:78-91, + Gamma^-1): the grid
 * Hessian schedule, host vectors, global gamma_inv. */
btg_status btg_partition_hessian(btg_partition p, const double* v, size_t v_len, double* hv, size_t hv_len,
                                 const double* gamma_inv, int gamma_kind, double alpha, int reg_kind, int backend,
                                 int parallel);
void btg_partition_destroy(btg_partition p);

/* Device pointer of F-hat and bytes per element (16 f64 / 8 f32). */
btg_status btg_spectrum_device(btg_op op, void** ptr, size_t* elem_bytes);

void btg_destroy(btg_op op);

/* Synthetic-input generator (bench / large-config parity): out[k] =
 * lo + (hi-lo) * ((splitmix64(seed ^ (offset + k)) >> 11) * 2^-53), the same
 * 53-bit mapping as btoep::Rng::uniform (rng.hpp:16-18) but indexable so any
 * slice is reproducible on the host. `out` is a device pointer. */
btg_status btg_fill_uniform(double* out, size_t n, uint64_t seed, uint64_t offset, double lo,
                            double hi, void* stream);

/* 3-D strided variant: out[(a*nb + b)*nc + c] = the same stream at global
 * index offset + a*stride_a + b*stride_b + c (a TOSI slab of a larger operator). */
btg_status btg_fill_uniform_3d(double* out, size_t na, size_t nb, size_t nc, uint64_t seed,
                               uint64_t offset, uint64_t stride_a, uint64_t stride_b, double lo,
                               double hi, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BTG_H_ */
