/* rimdp_b200.h — C ABI of the B200 robust value-iteration engine.
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/include/rimdp/ headers, umbrella rimdp.hpp:6-19).  The
 * reference has no C ABI of its own: its hot path is the header-only
 * template chain
 *
 *   value_iteration / control_synthesis   solver.hpp:149-198
 *   verify_policy                         solver.hpp:204-251
 *   detail::iterate                       solver.hpp:85-137
 *   bellman_step / bellman_step_impl      bellman.hpp:75-133
 *   robust_expectation / omax_expectation omax.hpp:164-199
 *
 * and the drop-in headers in include/rimdp/ route every Value = double|float
 * instantiation of those functions through the entry points below.  Plain
 * pointers and sizes only; all buffers passed in or out are HOST memory
 * unless a name says otherwise.  Every function returns an rimdp_status; on
 * failure rimdp_last_error() describes the error of the calling thread.
 */
#ifndef RIMDP_B200_H
#define RIMDP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RIMDP_B200_ABI_VERSION 4

/* Scalar type of a model: NumericTraits<double|float> (numeric.hpp:53-81).
 * The exact Rational instantiation (numeric.hpp:83-101) has no device path. */
typedef enum rimdp_dtype { RIMDP_F64 = 0, RIMDP_F32 = 1 } rimdp_dtype;

/* Status codes.  The C++ wrappers rethrow the reference's exception types
 * (errors.hpp:11-140) from these. */
typedef enum rimdp_status {
    RIMDP_OK = 0,
    RIMDP_ERR_INVALID_ARGUMENT = 1,
    RIMDP_ERR_INFEASIBLE_COLUMN = 2, /* ModelError{InfeasibleColumn}, omax.hpp:72-80 */
    RIMDP_ERR_NON_CONVERGENCE = 3,   /* NonConvergence(k, residual), solver.hpp:131-133 */
    RIMDP_ERR_CUDA = 4,
    RIMDP_ERR_OUT_OF_MEMORY = 5,
    RIMDP_ERR_NO_DEVICE = 6,
    RIMDP_ERR_INTERNAL = 7,
    RIMDP_ERR_MISSING_FILE = 8,      /* io::MissingFile (errors.hpp), native model containers */
    RIMDP_ERR_SCHEMA = 9,            /* io::SchemaViolation (errors.hpp:92-95), native.hpp:459-461 */
    RIMDP_ERR_INVALID_MODEL = 10     /* ModelError from the upload checks: StructuralError (csc.hpp:89-104),
                                        EntryOutOfRange / BoundOrderViolation (interval.hpp:148-164) */
} rimdp_status;

typedef struct rimdp_model rimdp_model; /* opaque, owns the device CSC store */

/* Details of the last failure on the calling thread. */
typedef struct rimdp_error_info {
    int32_t status;          /* rimdp_status */
    int64_t iterations;      /* NON_CONVERGENCE: iterations run */
    double residual;         /* NON_CONVERGENCE: max residual as double */
    int64_t column;          /* INFEASIBLE_COLUMN: offending column */
    int32_t infeasible_kind; /* 1: lower bounds sum > 1 + tol, 2: upper bounds sum < 1 - tol */
    double infeasible_sum;   /* the sum quoted by the reference message */
    int32_t violation_kind;  /* INVALID_MODEL: rimdp::ViolationKind value (errors.hpp:18-27) */
    int64_t row;             /* INVALID_MODEL: destination row of the offending entry */
} rimdp_error_info;

const char* rimdp_last_error(void);
int rimdp_last_error_info(rimdp_error_info* out);
int rimdp_abi_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int rimdp_device_count(int* count);

/* ---- device transition store ------------------------------------------
 * Replaces IntervalMDP<V> (imdp.hpp:26-181) + IntervalProbabilities<V>
 * (interval.hpp:34-304) + CscMatrix (csc.hpp:22-109) on the device.  The
 * caller passes the model's aligned CSC pattern exactly as
 * IntervalProbabilities stores it (one pattern, lower/upper value arrays,
 * rows strictly increasing per column), widened to int64 colptr so models
 * with more than 2^31-1 transitions are representable. */
typedef struct rimdp_model_desc {
    rimdp_dtype dtype;
    int32_t device;          /* CUDA ordinal */
    int32_t num_states;      /* n */
    int32_t num_cols;        /* state-action columns */
    int64_t nnz;
    const int32_t* stateptr; /* [n+1]; state s owns columns [stateptr[s], stateptr[s+1]) (imdp.hpp:22-23) */
    const int64_t* colptr;   /* [num_cols+1] */
    const int32_t* rowval;   /* [nnz] destination state per entry */
    const void* lower;       /* [nnz] dtype */
    const void* upper;       /* [nnz] dtype */
} rimdp_model_desc;

/* Checks at upload, on the device, in the reference's report order
 * (IntervalProbabilities::validate, interval.hpp:132-179, first violation as
 * check_or_throw :254-258): rows in range and strictly increasing per column,
 * bounds finite in [0,1], lower <= upper -> RIMDP_ERR_INVALID_MODEL with the
 * reference's ModelError text and the kind / column / row in
 * rimdp_error_info.  Column sums are not rejected here: an infeasible column
 * is reported when a step evaluates it (RIMDP_ERR_INFEASIBLE_COLUMN), as the
 * reference's step does for unchecked models (omax.hpp:72-80). */
int rimdp_model_create(const rimdp_model_desc* desc, rimdp_model** out);
/* One shard of a model for state-sharded multi-GPU solves: `desc` holds the
 * local states [state_begin, state_begin + desc->num_states) only (stateptr
 * and colptr local, rows global destinations in [0, num_global_states)).
 * The value vector stays global: V is replicated on every shard. */
int rimdp_model_create_shard(const rimdp_model_desc* desc, int32_t state_begin, int32_t num_global_states,
                             rimdp_model** out);
/* Capacity (entries) of the solve's value buffers, >= the global state
 * count: the sharded driver pads V to world_size equal slices so one
 * in-place all-gather per iteration can exchange it. */
int rimdp_model_set_value_capacity(rimdp_model* model, int64_t entries);
int rimdp_model_destroy(rimdp_model* model);

/* Synthetic transition stores generated directly in HBM by a counter-based
 * generator (no host copy): the configs that the reference's random_imdp
 * (random_model.hpp:42-101) cannot express.  See DESIGN.md "Workloads". */
typedef struct rimdp_gen_config {
    rimdp_dtype dtype;
    int32_t device;
    int32_t num_states;
    int32_t actions;         /* columns per state */
    int32_t law;             /* 0: fixed support `support`; 1: power law k^-alpha on [1, kmax] */
    int32_t support;         /* law 0 */
    double alpha;            /* law 1 */
    int32_t kmax;            /* law 1 */
    double lower_scale;      /* lower = u * lower_scale / k (law 1) or u * lower_scale (law 0) */
    double upper_scale;      /* law 1: upper = min(lower + v * upper_scale / k, 1) */
    uint64_t seed;
    int32_t state_begin;     /* shard: generate only states [state_begin, state_end) (columns */
    int32_t state_end;       /*  of other states are absent); 0,0 = all */
} rimdp_gen_config;

int rimdp_model_generate(const rimdp_gen_config* cfg, rimdp_model** out);
/* The same generator on the host (bit-identical columns), for sampled and
 * scaled-down parity checks against the CPU reference.  Two-phase: with
 * null arrays only the sizes are returned.  stateptr has (state_end -
 * state_begin) + 1 entries, colptr num_cols + 1. */
int rimdp_generate_host(const rimdp_gen_config* cfg, int32_t* num_cols, int64_t* nnz, int32_t* stateptr,
                        int64_t* colptr, int32_t* rowval, void* lower, void* upper);
/* Host copies of columns [col_begin, col_end) of a device store, as stored:
 * rows, lower bounds and gaps (upper - lower, rounded in dtype; the store
 * keeps gaps).  colptr_out (col_end - col_begin
 * + 1 entries) is relative to col_begin's first entry. */
int rimdp_model_read_columns(rimdp_model* model, int32_t col_begin, int32_t col_end, int64_t* colptr_out,
                             int32_t* rowval_out, void* lower_out, void* gap_out);

typedef struct rimdp_model_info {
    rimdp_dtype dtype;
    int32_t device;
    int32_t num_states;
    int32_t num_cols;
    int64_t nnz;
    int32_t state_begin, state_end; /* shard range (whole model: 0, n) */
    int32_t max_column_length;
    int32_t num_infeasible_columns;
    int64_t device_bytes;
    int32_t short_columns, mid_columns, long_columns; /* scheduler classes */
} rimdp_model_info;

int rimdp_model_info_get(rimdp_model* model, rimdp_model_info* out);
/* The CUDA stream (cudaStream_t) every kernel of this model is launched on. */
int rimdp_model_stream(rimdp_model* model, void** stream_out);

/* ---- native IMDPCSC1 containers --------------------
 * Replaces io::read_native_model (io/native.hpp:457-561) for the engine:
 * the container's named CSC arrays (native.hpp:15-41) are read, checked
 * (attributes, CscMatrix structure csc.hpp:75-107, the pattern merge of
 * IntervalProbabilities::align interval.hpp:218-252, [0,0] removal :261-279,
 * IntervalMDP structure imdp.hpp:129-168) and returned in the exact layout
 * rimdp_model_desc takes (colptr widened to int64).  Entry/column-sum checks
 * (interval.hpp:132-179) happen at upload.  Failures are RIMDP_ERR_MISSING_FILE
 * or RIMDP_ERR_SCHEMA with the reference's "<path>: <reason>" message.
 * Two-phase: read returns sizes and an opaque host handle, take copies the
 * arrays into caller buffers (any may be NULL), free releases the handle. */
typedef struct rimdp_native_sizes {
    int32_t num_states;
    int32_t num_cols;
    int64_t nnz;            /* after alignment and [0,0] removal */
    int32_t imdp;           /* 1: model = imdp, 0: imc (one action "0" per state) */
    int64_t label_bytes;    /* action labels, each NUL-terminated, concatenated */
} rimdp_native_sizes;

int rimdp_native_read(const char* path, int32_t dtype, rimdp_native_sizes* sizes, void** handle);
int rimdp_native_take(void* handle, int32_t* stateptr, int64_t* colptr, int32_t* rowval, void* lower, void* upper,
                      char* labels);
void rimdp_native_free(void* handle);
/* The engine's CSC arrays (rimdp_model_desc layout) as a container, like
 * write_native_model (native.hpp:424-455).  index64 = 0: int32 column
 * pointers when they fit (then the file is byte-identical to the
 * reference's), int64 (variable dtype 6, an engine extension the reference's
 * reader does not know) beyond 2^31-1 transitions; index64 = 1: always int64.
 * labels: num_cols NUL-terminated action labels, or NULL for "0", "1", ...
 * within each state. */
int rimdp_native_write(const char* path, int32_t dtype, int32_t num_states, int32_t num_cols, const int32_t* stateptr,
                       const int64_t* colptr, const int32_t* rowval, const void* lower, const void* upper,
                       const char* labels, int32_t index64);

/* ---- value iteration ---------------------------------------------------
 * One POD plan per solve, the marshalled form of detail::IterationPlan
 * (solver.hpp:27-80) + OptimizationMode (omax.hpp:21-24) + SolverOptions
 * (solver.hpp:19-23). */
typedef struct rimdp_plan {
    int32_t pessimistic;      /* SatisfactionMode: adversary direction (sort order) */
    int32_t maximize;         /* StrategyMode: action reduction */
    int32_t finite;           /* 1: run exactly `horizon` iterations */
    int64_t horizon;
    double eps;               /* infinite: stop at first k with max residual <= eps (converted to dtype) */
    int64_t max_iterations;   /* infinite: NonConvergence past this */
    const void* initial;      /* [n] V_0 (dtype) */
    const uint8_t* frozen;    /* [n] or NULL: value carried over, chosen = -1 */
    const void* rewards;      /* [n] or NULL: V_k = r + discount * T(V_{k-1}) */
    double discount;          /* converted to dtype */
    const int32_t* forced;    /* NULL, [n] (stationary) or [horizon][n] (row t = horizon - k) */
    int32_t forced_time_dependent;
    int32_t external_stop;    /* sharded solves: the device stop test waits for rimdp_solve_stop_test */
} rimdp_plan;

/* Called after iteration k with V_k on the host (on_iteration_f64,
 * solver.hpp:119-125).  Forces one device->host copy per iteration. */
typedef void (*rimdp_iteration_cb)(int64_t k, const void* values, void* user);

typedef struct rimdp_outputs {
    void* values;             /* [n] V at stop (dtype), may be NULL */
    void* residual;           /* [n] |V_k - V_{k-1}| (dtype), may be NULL */
    int64_t* iterations;      /* may be NULL */
    int32_t* chosen;          /* NULL, [n] (last step) or [horizon][n] (record_all_steps) */
    int32_t record_all_steps; /* finite horizon: per-step chosen columns, row t = horizon - k */
    rimdp_iteration_cb on_iteration;
    void* user;
} rimdp_outputs;

int rimdp_solve(rimdp_model* model, const rimdp_plan* plan, const rimdp_outputs* out);

/* Split form of rimdp_solve for callers that keep everything resident
 * (benchmarks, sharded drivers).  begin uploads the plan and resets the
 * device loop state; advance enqueues up to `iterations` more Bellman
 * iterations on the model stream without synchronising; poll synchronises
 * and reports progress; finish downloads the outputs. */
int rimdp_solve_begin(rimdp_model* model, const rimdp_plan* plan);
int rimdp_solve_advance(rimdp_model* model, int64_t iterations);
int rimdp_solve_poll(rimdp_model* model, int64_t* iterations_done, int32_t* finished, double* max_residual);
int rimdp_solve_finish(rimdp_model* model, const rimdp_outputs* out);

/* Kernel timing: when enabled, every enqueued iteration records CUDA events
 * on the model stream around its three phases: the fused short-state kernel,
 * the per-column kernels of the remaining states, and their action kernel.
 * profile_read synchronises, returns the summed milliseconds of each phase
 * and the iteration count since the last read, and resets the accumulators;
 * kernels_per_iteration is the number of kernels the last enqueued iteration
 * launched (every class kernel, fallback pass, range pass and stop test). */
int rimdp_profile_enable(rimdp_model* model, int32_t on);
int rimdp_profile_read(rimdp_model* model, double* fused_ms, double* columns_ms, double* action_ms,
                       int64_t* iterations, int32_t* kernels_per_iteration);

/* Device pointers of the solve's double-buffered value vector, for
 * collective exchange in the sharded driver: V_k lives in buffer k & 1. */
int rimdp_solve_value_buffers(rimdp_model* model, void** buf0, void** buf1);
/* Device pointer to the two per-iteration residual slots (uint64 bit patterns
 * of the non-negative max residual; iteration k uses slot k & 1). */
int rimdp_solve_residual_slots(rimdp_model* model, void** slots);
/* Enqueues the stop test of the last enqueued iteration k on the model stream
 * (solver.hpp:127-134).  With external_stop, call it after the value buffer
 * of iteration k holds every shard's slice (the all-gather): the residual
 * max |V_k - V_{k-1}| is then taken over the whole value vector on the
 * device, so no collective is needed for it. */
int rimdp_solve_stop_test(rimdp_model* model);

/* ---- multi-GPU: peer exchange of a state-sharded solve -----
 * New: the reference has no multi-device path (its only parallelism is the
 * per-state fork/join of parallel.hpp:56-64 inside bellman.hpp:88-115).
 * Every shard owns an exchange window in its HBM (the double-buffered value
 * vector, per-rank residual slots and iteration flags).  Each iteration the
 * action kernel stores every new value of the shard's states into every
 * peer's window over NVLink (CUDA IPC or peer access) as it computes them, and
 * publishes its residual and a flag with system-scope release; a one-warp
 * kernel then waits for all ranks' flags and runs the stop test on the
 * maximum published residual (identical on every rank).  No collective
 * library call, no host synchronisation per iteration.
 *
 * Multi-process (one process per GPU): call rimdp_model_set_value_capacity
 * (same value on every rank, >= the global state count), export the window's
 * 64-byte CUDA IPC handle, exchange the handles (e.g. torch.distributed
 * all_gather_object), connect.  Then per solve: rimdp_solve_begin with
 * external_stop = 1 on every rank, a barrier across ranks (the windows are
 * reset by begin), then rimdp_solve_advance / _poll / _finish as usual. */
#define RIMDP_MAX_WORLD 8
int rimdp_exchange_export(rimdp_model* model, void* ipc_handle_out /* 64 bytes, may be NULL */);
int rimdp_exchange_connect(rimdp_model* model, int32_t rank, int32_t world,
                           const void* ipc_handles /* world x 64 bytes, rank order */);
/* Single process, several shards (devices may repeat: shards sharing a GPU). */
int rimdp_exchange_connect_local(rimdp_model* const* shards, int32_t world);

/* Single process, several devices: the model cut into `world` contiguous
 * state ranges of equal transition counts (one shard per entry of `devices`,
 * NULL = 0 .. world-1; a device may repeat), connected as above.  solve has
 * rimdp_solve's contract on the whole model: global column indices in
 * plan.forced and out.chosen, V and residual of all states; results are
 * bit-identical to a one-device solve (sharding changes no per-state
 * arithmetic). */
typedef struct rimdp_multi rimdp_multi;
int rimdp_multi_create(const rimdp_model_desc* desc, int32_t world, const int32_t* devices, rimdp_multi** out);
int rimdp_multi_solve(rimdp_multi* multi, const rimdp_plan* plan, const rimdp_outputs* out);
/* world, state_begin[world + 1] (the cut), devices[world]; any may be NULL. */
int rimdp_multi_info(rimdp_multi* multi, int32_t* world, int32_t* state_begin, int32_t* devices);
int rimdp_multi_destroy(rimdp_multi* multi);

/* One Bellman step from `v_in` (bellman.hpp:127-133, with the optional
 * forced column per state of bellman_step_impl, :96-101). */
int rimdp_bellman_step(rimdp_model* model, const void* v_in, int32_t pessimistic, int32_t maximize,
                       const uint8_t* frozen, const int32_t* forced, void* v_out, int32_t* chosen_out);

/* The robust expectation of every column for value vector `v_in`
 * (detail::column_value, bellman.hpp:60-70 == robust_expectation,
 * omax.hpp:182-189).  q_out has num_cols entries. */
int rimdp_column_values(rimdp_model* model, const void* v_in, int32_t pessimistic, void* q_out);

#ifdef __cplusplus
}
#endif
#endif /* RIMDP_B200_H */
