/*
 * gensor-b200 C-ABI: operator description -> construct -> execute, B200-native.
 *
 * Drop-in boundary for the reference's construct/execute path (arXiv 2502.11407 "Gensor",
 * /root/reference/proj). Every entry point below names the reference interface it replaces.
 * Conventions:
 *   - every function returns int: GENSOR_OK (0) or a status code; the first 18 codes are the
 *     reference's ErrorCode enum (include/gensor/error.hpp:8-27) as ordinal + 1;
 *   - gensor_last_error() returns a thread-local "<CodeName>: detail" message, the reference's
 *     what() text (error.hpp:33-34);
 *   - op / hw / schedule handles are opaque and immutable after creation, safe to share across
 *     threads; a kernel handle's plan is immutable too: gensor_execute may be called on one
 *     handle from several threads and streams at once (each stream gets its own device
 *     workspace; gensor_execute_ws takes a caller-owned one). gensor_execute_host and the timing
 *     instrumentation take a non-const handle and run one call at a time;
 *   - lifetimes: an op must outlive every schedule and kernel made from it (the reference's
 *     ETIRState keeps a non-owning op pointer, etir.hpp:75); a hw must outlive schedules;
 *   - JSON outputs use caller buffers: on cap < need the call returns GENSOR_ETRUNCATED and
 *     sets *need (bytes including the terminating NUL);
 *   - no torch types, no CUDA types in signatures: streams are passed as void* (cudaStream_t),
 *     device buffers as plain pointers owned by the caller.
 */
#ifndef GENSOR_B200_H
#define GENSOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------------------- */
enum gensor_status {
  GENSOR_OK = 0,
  GENSOR_EUNKNOWN_KIND = 1,          /* ErrorCode::UnknownKind */
  GENSOR_EMISSING_PARAM = 2,         /* ErrorCode::MissingParam */
  GENSOR_ENONPOSITIVE_EXTENT = 3,    /* ErrorCode::NonPositiveExtent */
  GENSOR_EAXIS_NOT_FOUND = 4,        /* ErrorCode::AxisNotFound */
  GENSOR_EILLEGAL_ACTION = 5,        /* ErrorCode::IllegalAction */
  GENSOR_ELEVEL_OUT_OF_RANGE = 6,    /* ErrorCode::LevelOutOfRange */
  GENSOR_EMONOTONICITY = 7,          /* ErrorCode::MonotonicityViolation */
  GENSOR_EMISSING_LEVEL = 8,         /* ErrorCode::MissingLevel */
  GENSOR_EINCOMPLETE_STATE = 9,      /* ErrorCode::IncompleteState */
  GENSOR_ETOO_LARGE_TO_ENUMERATE = 10,
  GENSOR_ENO_LEGAL_ACTION = 11,
  GENSOR_EEMPTY_CANDIDATES = 12,
  GENSOR_ESPACE_TOO_LARGE = 13,
  GENSOR_ENOT_ERGODIC = 14,
  GENSOR_ENO_CONVERGENCE = 15,
  GENSOR_ESHAPE_MISMATCH = 16,       /* ErrorCode::ShapeMismatch (execute: wrong input count) */
  GENSOR_EREPLAY_MISMATCH = 17,
  GENSOR_ECONFIG = 18,               /* ErrorCode::ConfigError (bad JSON / config fields) */
  GENSOR_ECUDA = 19,                 /* new: CUDA runtime/driver failure */
  GENSOR_EUNSUPPORTED = 20,          /* new: schedule/variant the kernel family cannot run */
  GENSOR_EINVALID = 21,              /* new: null handle / bad argument */
  GENSOR_ETRUNCATED = 22             /* new: output buffer too small, see *need */
};

/* Kernel variants instantiated from a constructed schedule. */
enum gensor_variant {
  GENSOR_VARIANT_AUTO = -1,        /* fastest family legal for the op and dtype */
  GENSOR_VARIANT_SIMT_PARITY = 0,  /* state-driven SIMT kernel, fp64 accumulation in the
                                      interpreter's loop order: bit-exact to the oracle */
  GENSOR_VARIANT_SIMT_F32 = 1,     /* state-driven SIMT kernel, fp32 FFMA accumulation */
  GENSOR_VARIANT_TC_TF32 = 2,      /* tcgen05 kind::tf32, TMEM accumulator (gemm, conv2d) */
  GENSOR_VARIANT_TC_BF16 = 3,      /* tcgen05 kind::f16 bf16 operands (gemm, conv2d) */
  GENSOR_VARIANT_STREAM = 4,       /* HBM-streaming families: gemv/row-sum, softmax, pooling,
                                      depthwise conv (128-bit loads, warp shuffles) */
  GENSOR_VARIANT_TC_3XTF32 = 5     /* fp32-grade tcgen05 GEMM: each fp32 operand split into
                                      tf32 hi + lo in shared memory, 3 MMAs per k-step (~fp32
                                      accuracy, the SPEC's 1e-6 single-precision bar) */
};

enum gensor_mode {
  GENSOR_MODE_REFERENCE_COMPAT = 0, /* bit-identical to the reference engine */
  GENSOR_MODE_B200 = 1              /* B200 legality gates + wave/occupancy cost */
};

typedef struct gensor_op gensor_op;
typedef struct gensor_hw gensor_hw;
typedef struct gensor_schedule gensor_schedule;
typedef struct gensor_kernel gensor_kernel;

/* EngineConfig field for field (include/gensor/engine.hpp:14-24) + mode/threads. */
typedef struct gensor_engine_cfg {
  double t0;                 /* 2^20 */
  double threshold;          /* 1 */
  int32_t restarts;          /* 8 */
  int32_t top_k;             /* 10 */
  uint64_t seed;             /* 0 */
  int64_t vthread_options[8];
  int32_t n_vthread_options; /* 4: {1,2,4,8} */
  int32_t mode;              /* gensor_mode */
  int64_t max_tile_factor;   /* 2 */
  int32_t threads;           /* restart worker threads; 0 = min(restarts, cores) */
  int32_t reserved;
} gensor_engine_cfg;

const char* gensor_last_error(void);
const char* gensor_version(void);

/* Defaults of EngineConfig (engine.hpp:14-24). */
void gensor_engine_cfg_init(gensor_engine_cfg* cfg);

/* ---- operator description: replaces TensorOpSpec::parse_text (op_spec.hpp:51) ----------- */
int gensor_op_parse(const char* json, gensor_op** out);
void gensor_op_free(gensor_op* op);
/* Axes, tensors (true dims, affine layout coefficients), FLOPs and compulsory bytes. */
int gensor_op_info(const gensor_op* op, char* buf, size_t cap, size_t* need);

/* ---- hardware model: replaces HardwareSpec::load_text (hardware.hpp:31) ------------------ */
int gensor_hw_load(const char* json, gensor_hw** out);
/* B200 model from the live device query + measured peaks (JSON text of MEASURED_PEAKS.json or
 * NULL for the built-in defaults); device < 0 uses the nominal B200 limits without a device
 * query (construction on a host without a GPU). New: the reference has no device model. */
int gensor_hw_b200(int device, const char* measured_peaks_json, gensor_hw** out);
void gensor_hw_free(gensor_hw* hw);
int gensor_hw_json(const gensor_hw* hw, char* buf, size_t cap, size_t* need);

/* ---- construct: replaces optimize / construct / construct_tree (engine.hpp:83-99,
 *      tree_baseline.hpp:26) ---------------------------------------------------------------- */
int gensor_optimize(const gensor_op* op, const gensor_hw* hw, const gensor_engine_cfg* cfg,
                    gensor_schedule** out, int* n_out);
/* One annealed walk with cfg->seed as the rng seed: raw snapshots (uncompleted, no cost). */
int gensor_construct(const gensor_op* op, const gensor_hw* hw, const gensor_engine_cfg* cfg,
                     gensor_schedule** out, int* n_out);
int gensor_construct_tree(const gensor_op* op, const gensor_hw* hw, int beam_width, int mode,
                          gensor_schedule** out, int* n_out);
/* Replays a trace (JSON [[kind,axis,factor],...], kinds 0=Tile 1=InvTile 2=SetVThread 3=Cache)
 * from the unscheduled state; costs it when complete. Replaces the SPEC's trace replay. */
int gensor_schedule_from_trace(const gensor_op* op, const gensor_hw* hw, const char* trace_json,
                               int mode, gensor_schedule** out);
/* {state:{level,tiles,vthreads,repr}, trace, cost, seed, iterations}; index -1 = all results. */
int gensor_schedule_json(const gensor_schedule* s, int index, char* buf, size_t cap, size_t* need);
/* Explicit construction-chain analysis (the reference's markov-verify module, markov.hpp:1-70,
 * SPEC.md:380-457): enumerates the schedule space reachable under the candidate policy frozen at
 * an annealing iteration and reports per-level SCCs / irreducibility / stationary entropy,
 * aperiodicity, the value iteration of Eqs. 5-6 and its greedy policy path as JSON.
 * caps_json (optional) keys: max_states (50000), fixed_iteration (10), enable_inv_tile (true),
 * vthread_options ([1,2,4,8]), max_tile_factor (2), mode ("reference"|"b200"), detail (false:
 * every state, edge, value and stationary vector). GENSOR_ESPACE_TOO_LARGE past max_states. */
int gensor_analyze(const gensor_op* op, const gensor_hw* hw, const char* caps_json, char* buf, size_t cap,
                   size_t* need);
/* Portable C source of result `index`'s tiled loop nest (the SPEC's emit_source, SPEC.md:488-496;
 * absent from the reference): deterministic text, guards iff padding, double accumulation.
 * GENSOR_EINCOMPLETE_STATE for an incomplete state (e.g. gensor_construct snapshots). */
int gensor_emit_source(const gensor_schedule* s, int index, char* buf, size_t cap, size_t* need);
int gensor_schedule_count(const gensor_schedule* s);
void gensor_schedule_free(gensor_schedule* s);

/* ---- cost model: memory_traffic / tile_footprint / capacity_check / estimate_cost /
 *      enumerate_candidates (cost_model.hpp:32-71, hardware.hpp:58-62, engine.hpp:54-57) ----- */
int gensor_state_eval(const gensor_op* op, const gensor_hw* hw, const char* trace_json, int mode,
                      char* buf, size_t cap, size_t* need);
int gensor_candidates(const gensor_op* op, const gensor_hw* hw, const char* trace_json,
                      const gensor_engine_cfg* cfg, int iteration, char* buf, size_t cap, size_t* need);
double gensor_caching_benefit(double lat_low, double bw_low, double lat_high, double bw_high, double s_bytes);
double gensor_vthread_conflict_ratio(int64_t x, int64_t bank_width, int64_t v);
double gensor_anneal_cache_multiplier(int iteration);
double gensor_record_probability(double temperature);
uint64_t gensor_derive_seed(uint64_t seed, int restart);

/* ---- execute: replaces the SPEC's lower(state) + interpret(prog, inputs)
 *      (lowering.cpp is absent from the reference snapshot) ---------------- */
/* Instantiates a kernel for result `index` of a schedule. Device work (workspace allocation,
 * attribute setup) happens on the current CUDA device. */
int gensor_kernel_prepare(const gensor_op* op, const gensor_schedule* s, int index, int variant,
                          gensor_kernel** out);
/* Grid, block, smem, variant, per-launch algorithmic FLOPs/bytes, launch count per execute. */
int gensor_kernel_info(const gensor_kernel* k, char* buf, size_t cap, size_t* need);
/* Asynchronous on `stream` (a cudaStream_t). Inputs in the op's tensor order (gemm: A,B;
 * gemv: A,x; conv2d: I,K; avgpool2d: I; dwconv2d: I,K; softmax: X), row-major true-domain
 * layouts (op_spec.cpp:251-262). fp32 tensors for dtype_bytes 4, bf16 for dtype_bytes 2. */
int gensor_execute(const gensor_kernel* k, const void* const* d_inputs, int n_inputs, void* d_output,
                   void* stream);
/* Device workspace one execute needs (bytes; 0 for families without a pre-pass). */
int gensor_kernel_workspace_size(const gensor_kernel* k, size_t* bytes);
/* gensor_execute with a caller-owned device workspace of at least gensor_kernel_workspace_size
 * bytes (the cuDNN/cuBLASLt convention): concurrent calls on one handle with distinct workspaces
 * never touch shared device state. gensor_execute uses a per-stream workspace owned by the handle
 * (allocated on the stream's first execute). */
int gensor_execute_ws(const gensor_kernel* k, const void* const* d_inputs, int n_inputs, void* d_output,
                      void* d_workspace, size_t workspace_bytes, void* stream);
/* Host-buffer execute, the interpreter's calling convention: copies the inputs host->device,
 * runs, copies the output back and synchronises. Device staging buffers are owned by the
 * kernel handle (one call at a time per handle). */
int gensor_execute_host(gensor_kernel* k, const void* const* h_inputs, int n_inputs, void* h_output,
                        void* stream);
void gensor_kernel_free(gensor_kernel* k);

/* On-device re-ranking of the constructed top-k (the paper profiles its top
 * candidates on hardware, the reference ranks by the analytical estimate_cost only, engine.cpp:
 * 179-190): instantiates every complete result of `s` with `variant`, times `iters` executes on
 * the caller's device buffers and writes {"ms":[...],"order":[...],"best":i,"plans":[...]} (order:
 * fastest first; plans: the kernel plan each result instantiates). */
int gensor_rerank(const gensor_op* op, const gensor_schedule* s, int variant, const void* const* d_inputs,
                  int n_inputs, void* d_output, void* stream, int iters, char* buf, size_t cap, size_t* need);

/* Per-launch device timing (CUDA events recorded on the execute stream around every internal
 * launch). While enabled, gensor_kernel_timings() returns the durations of the LAST execute's
 * launches in ms (synchronising on its events) and their names as a JSON array in `names`. */
int gensor_kernel_set_timing(gensor_kernel* k, int enable);
int gensor_kernel_timings(gensor_kernel* k, float* ms, int cap, int* n, char* names, size_t names_cap);

/* Number of kernels this library launched since load (process-wide counter). */
uint64_t gensor_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* GENSOR_B200_H */
