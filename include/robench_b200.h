/*
 * robench_b200 — C ABI of the B200-native batched test-function evaluator.
 *
 * Drop-in boundary for the reference's evaluation path:
 *   reference (Python rendition)            this ABI
 *   engine.initialize      engine.py:225-228  rb_initialize
 *   Engine.evaluate        engine.py:174-214  rb_func_evaluate   (device ptrs, fp64)
 *   Engine.evaluate(...,"single")  :216-217   rb_func_evaluatef  (device ptrs, fp32)
 *   (host-memory wrappers)                    rb_h_func_evaluate / rb_h_func_evaluatef
 *   Engine.dispose         engine.py:219-222  rb_dispose
 * The C names are the paper's own host API (initialize,
 * func_evaluate, func_evaluatef, h_func_evaluate, h_func_evaluatef, dispose),
 * prefixed rb_.  Values include the suite bias of +100 (engine.py:209).
 *
 * Plain C types only: pointers, sizes, status codes.  The instance pack is
 * built on the host (paper_1407_7737_b200/pack.py) and copied to the device
 * once in rb_initialize; the engine never retains caller pointers.
 */
#ifndef ROBENCH_B200_H
#define ROBENCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes; 1:1 with the reference's exceptions (errors.py:4-52) */
typedef int32_t rb_status;
#define RB_OK                    0
#define RB_E_UNKNOWN_FUNCTION    1  /* UnknownFunction   (catalog.py:224-229) */
#define RB_E_DISABLED_FUNCTION   2  /* DisabledFunction  (engine.py:186-189)  */
#define RB_E_BATCH_TOO_LARGE     3  /* BatchTooLarge     (engine.py:190-193)  */
#define RB_E_DIMENSION_MISMATCH  4  /* DimensionMismatch (engine.py:194-195)  */
#define RB_E_NON_FINITE_INPUT    5  /* NonFiniteInput    (engine.py:202-203, kernels.py:45-49) */
#define RB_E_USE_AFTER_DISPOSE   6  /* UseAfterDispose   (engine.py:180-181)  */
#define RB_E_INVALID_ARGUMENT    7  /* ValueError / malformed pack            */
#define RB_E_UNSUPPORTED         8  /* configuration outside the built kernels */
#define RB_E_CUDA                9  /* CUDA runtime failure                    */

/* ---- instance pack ---------------------------------------------------- */
/* Categories (catalog.py:25-29); RB_DISABLED marks ids switched off at
 * dim < 10 (engine.py:148-154). */
#define RB_DISABLED    (-1)
#define RB_BASIC        0
#define RB_HYBRID       1
#define RB_COMPOSITION  2

/* One diagonal block of a rotation: the block-diagonal-in-permuted-basis R
 * of transforms.py:110-128 (3 groups), or a whole hybrid chunk rotation
 * (transforms.py:137-140, 1 group).  Columns are stored in "q-order": sorted
 * by the NumPy pairwise-sum accumulator slot they fall in (slot = column % 8
 * below the last multiple of 8, then the ordered tail), ascending inside a
 * slot, so exact-order single precision can replay NumPy's rounding
 * (SURVEY.md Appendix A).  Segments longer than 128 are NumPy's recursive
 * split: columns sorted by (leaf, slot, index), see `leaf`; up to 968 (4 pending sums). */
typedef struct rb_group {
  int32_t m;        /* block size */
  int32_t qb[10];   /* slot s spans q in [qb[s], qb[s+1]) for s < 8; tail [qb[8], qb[9]); qb[9] == m */
  int32_t col;      /* index[col + q]: input position (into the segment vector v) of the q-th column */
  int32_t row;      /* index[row + r]: output position (into z) of block row r */
  int32_t mat;      /* values[mat + q*m4 + r] = block[r][column of q], m4 = m rounded up to 4
                       (rows zero-padded; float32 exact-order rotate, 16-byte aligned) */
  int32_t frag;     /* values_f64[frag + ((nt*nks + ks)*32 + lane)] = scale * block[8nt + lane/4][c(4ks + lane%4)]
                       (zero outside m x m), c(q) the q-th column in col64 order: the
                       mma.m16n8k4 B fragments of the segment's scaled block, nt < ceil(m/8),
                       ks < ceil(m/4) (float64 DMMA rotate) */
  int32_t cz;       /* values_f64[cz + r] = -pre * sum_q mat[q][r] - post: the float64 rotate
                       computes z_r = sum_q (scale B)[q][r] (x[src_q] - o[src_q]) - cz[r] */
  int32_t col64;    /* index[col64 + q]: input position of the q-th float64 column (an order
                       whose 4-column k-steps read shared memory without bank conflicts) */
  int32_t leaf;     /* -1: one pairwise leaf (qb above).  -2: tree deeper than the device stack
                       (float32 unsupported).  Else index[leaf ...] = [n_leaf, then per leaf
                       its qb (10 ints, absolute q) and the number of (left + right) additions
                       that follow it]: float32 rows longer than 128 replay NumPy's recursive
                       pairwise tree as a post-order program (pack.py pairwise_program) */
} rb_group;

/* One kernel application: v = scale*((x - o)[src..]) + pre; z = R v + post;
 * value = K(z)  (engine.py:96-104, hybrid.py:108-114, composition.py:147-154). */
typedef struct rb_segment {
  int32_t kernel;    /* 0..20 in catalog.KERNEL_NAMES order */
  int32_t d;         /* kernel length: dim, or the hybrid chunk size */
  int32_t src;       /* offset of this chunk inside the member's split permutation (0 for basic) */
  int32_t n_groups;  /* 0 = not rotated (ids 10, 15) */
  int32_t group0;    /* first rb_group */
  int32_t ctab;      /* values[ctab ...]: per-(kernel, d) constants computed by NumPy in the pack dtype */
  double scale, pre, post;
} rb_segment;

/* A basic function, a hybrid, or one composition member (composition.py:25-40). */
typedef struct rb_member {
  int32_t n_segments;
  int32_t segment0;
  int32_t shift;     /* values[shift + j]: optimum o (dim) */
  int32_t perm;      /* index[perm + t]: hybrid split permutation (dim), or -1 */
  double sigma, height, bias;  /* composition blend (composition.py:114-166); unused otherwise */
} rb_member;

typedef struct rb_function {
  int32_t category;  /* RB_DISABLED / RB_BASIC / RB_HYBRID / RB_COMPOSITION */
  int32_t n_members;
  int32_t member0;
  int32_t reserved;  /* ignored (set 0): the library's device copy uses it internally */
} rb_function;

typedef struct rb_pack {
  int32_t dim;
  int32_t n_functions;                 /* 37 */
  const rb_function* functions;
  int32_t n_members;   const rb_member*  members;
  int32_t n_segments;  const rb_segment* segments;
  int32_t n_groups;    const rb_group*   groups;
  int64_t n_index;     const int32_t*    index;
  int64_t n_values;                    /* length of both value tables */
  const double* values_f64;            /* shifts, rotations, constants in float64 */
  const float*  values_f32;            /* the same, cast / recomputed in float32 */
} rb_pack;

typedef struct rb_engine rb_engine;

/* ---- lifecycle -------------------------------------------------------- */
rb_status rb_initialize(const rb_pack* pack, int64_t max_concurrency, int32_t device,
                        rb_engine** out);
rb_status rb_dispose(rb_engine** engine);          /* idempotent; *engine = NULL */

/* ---- evaluation: f[i] = F_fn(x[i, :]) + 100 ---------------------------- */
/* Device pointers, stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 * default).  x is row-major n x dim.  Synchronises on `stream` only to read
 * the non-finite flag; on RB_E_NON_FINITE_INPUT the contents of f are
 * unspecified (the reference returns no values). */
rb_status rb_func_evaluate (rb_engine* e, int32_t fn_id, const double* x, int64_t n,
                            double* f, void* stream);
rb_status rb_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n,
                            float* f, void* stream);
/* Host-memory wrappers (paper: h_func_evaluate / h_func_evaluatef). */
rb_status rb_h_func_evaluate (rb_engine* e, int32_t fn_id, const double* x, int64_t n,
                              double* f);
rb_status rb_h_func_evaluatef(rb_engine* e, int32_t fn_id, const float* x, int64_t n,
                              float* f);

/* precision: RB_DOUBLE (double) or RB_SINGLE (float). */
#define RB_DOUBLE 0
#define RB_SINGLE 1
/* Host float64 rows evaluated in `precision`: RB_SINGLE rounds each x to
 * float32 first, as the reference's Engine.evaluate(..., "single") casts its
 * float64 batch (engine.py:201), inside the transfer pipeline (no separate
 * host cast pass); f is double* or float*.  The host wrappers pipeline rows
 * through pinned chunks: host staging, H2D, evaluation and D2H overlap. */
rb_status rb_h_func_evaluate_x64(rb_engine* e, int32_t fn_id, int32_t precision, const double* x,
                                 int64_t n, void* f);

/* Many (fn_ids[i], precisions[i]) evaluations of ONE host population of
 * float64 rows, synchronous: the rows cross PCIe once (per ~32 MB chunk) for
 * all calls instead of once per call; single-precision calls evaluate
 * float32(x) (engine.py:201).  f[i]: n values (double* or float*).  Every
 * call is validated (the reference's order) before any work; a non-finite x
 * returns RB_E_NON_FINITE_INPUT (f unspecified).  At most 1024 calls. */
rb_status rb_h_func_evaluate_many(rb_engine* e, int32_t n_calls, const int32_t* fn_ids,
                                  const int32_t* precisions, const double* x, int64_t n,
                                  void* const* f);

/* ---- stream-ordered calls with a deferred status ------------------------ */
/* Enqueue the evaluation on `stream` and return at once: argument errors
 * (the reference's validation order) come back now; the input's finiteness
 * (NonFiniteInput) is read later with rb_ticket_status, after the caller has
 * synchronised `stream` (or an event recorded after this call).  At most
 * 4096 calls per engine may be outstanding.  Lets a caller queue many
 * functions, and overlap them with copies or collectives, without a host
 * synchronisation per call (the blocking rb_func_evaluate[f] wait on the
 * stream to read the status). */
rb_status rb_func_evaluate_async(rb_engine* e, int32_t fn_id, int32_t precision, const void* x,
                                 int64_t n, void* f, void* stream, int64_t* ticket);
/* RB_OK or RB_E_NON_FINITE_INPUT for a completed call; RB_E_INVALID_ARGUMENT
 * once the ticket's slot was reused (4096 later calls). */
rb_status rb_ticket_status(rb_engine* e, int64_t ticket);
/* n_calls stream-ordered evaluations in one call (e.g. every function of the
 * suite on one population): call i is rb_func_evaluate_async(e, fn_ids[i],
 * precisions[i], x[i], n[i], f[i], stream, &tickets[i]).  Stops at the first
 * argument error (its status is returned; later tickets are not written).
 * When every f[i] is disjoint from the other outputs and from every input,
 * and each call is at most RB_FORK_WAVES (default 128) waves of the grid,
 * the calls alternate between `stream` and an engine stream forked from it
 * and joined back before returning: work queued on `stream` afterwards
 * still sees every value. */
rb_status rb_func_evaluate_many(rb_engine* e, int32_t n_calls, const int32_t* fn_ids,
                                const int32_t* precisions, const void* const* x, const int64_t* n,
                                void* const* f, void* stream, int64_t* tickets);

/* ---- one process, several GPUs ---------------------------
 * A replica of the instance pack on each device; rows are sharded
 * contiguously, device g owning rows [start_g, start_g + count_g) with
 * count_g = n/G (+1 for the first n%G devices).  x_shards[g]: device g's rows
 * (row-major count_g x dim, on devices[g]); f_full[g]: a length-n_total buffer
 * on devices[g].  Each device evaluates its rows into f_full[g] + start_g and
 * stores that slice into every peer's f_full (P2P stores over NVLink /
 * NVSwitch; copy-engine peer copies where peer access is unavailable), so on
 * completion every f_full[g] holds all n_total values -- the fitness
 * all-gather.  streams: per-device cudaStream_t, a NULL entry being that
 * device's legacy default stream; a NULL array: the engine's own streams.  tickets == NULL: synchronous, errors as rb_func_evaluate;
 * else tickets[g] receives device g's ticket (-1: no rows) and the call
 * returns once everything is queued (rb_sharded_ticket_status). */
typedef struct rb_sharded rb_sharded;
rb_status rb_initialize_sharded(const rb_pack* pack, int64_t max_concurrency_per_device,
                                const int32_t* devices, int32_t n_devices, rb_sharded** out);
rb_status rb_func_evaluate_sharded(rb_sharded* s, int32_t fn_id, int32_t precision,
                                   const void* const* x_shards, int64_t n_total, void* const* f_full,
                                   void* const* streams, int64_t* tickets);
rb_status rb_sharded_ticket_status(rb_sharded* s, int32_t device_index, int64_t ticket);
rb_status rb_dispose_sharded(rb_sharded** s);      /* idempotent; *s = NULL */

/* ---- CUDA graphs -------------------------------------------------------- */
/* One evaluation captured as a CUDA graph and replayed (no reference
 * counterpart: the reference has no device; this is the launch-bound
 * small-batch case of Engine.evaluate, engine.py:174-214, called in a loop
 * on the same buffers).  rb_graph_capture validates like rb_func_evaluate
 * and records: reset of the graph's own status words, the evaluation
 * kernel, and (float64 HappyCat / HGBat functions) the exact-order fixup
 * pass.  Each rb_graph_launch evaluates the CURRENT contents of d_x into d_f
 * on `stream`; after the stream has synchronised, rb_graph_status returns
 * RB_E_NON_FINITE_INPUT if that replay saw a non-finite input.  Replays of
 * one graph must not overlap (they share the status words).  A graph reads
 * its engine's device tables: destroy it before rb_dispose of the engine
 * (Engine.dispose closes its captures). */
typedef struct rb_graph rb_graph;
rb_status rb_graph_capture(rb_engine* e, int32_t fn_id, int32_t precision, const void* d_x,
                           int64_t n, void* d_f, rb_graph** out);
rb_status rb_graph_launch(rb_graph* g, void* stream);
rb_status rb_graph_status(rb_graph* g);
rb_status rb_graph_destroy(rb_graph** g);          /* idempotent; *g = NULL */

/* ---- introspection ---------------------------------------------------- */
const char* rb_last_error(void);                   /* thread-local message */
int32_t rb_abi_version(void);
/* sizeof of rb_group, rb_segment, rb_member, rb_function, rb_pack (host
 * layout check for FFI bindings). */
void rb_struct_sizes(int64_t out[5]);
/* Number of kernel launches issued by this process so far (bench evidence). */
int64_t rb_launch_count(void);
/* Diagnostic: out[i] = x[i] ** y[i] with NumPy's float32 array-power
 * semantics (bit-exact SVML powf restatement, csrc/rb_svml_powf.cuh), on
 * device pointers; synchronous on `stream`. */
rb_status rb_np_powf(const float* x, const float* y, float* out, int64_t n, void* stream);
/* On-device population source: elements
 * [first_element, first_element + n_elements) of the stream that
 * numpy.random.Generator(numpy.random.Philox(key)).uniform(low, high) draws
 * (Philox4x64-10, key = SeedSequence(...).generate_state(2, uint64)), bit
 * for bit, into out64 and/or out32 (float32 = the float64 value rounded);
 * asynchronous on `stream`. */
rb_status rb_uniform_population(uint64_t key0, uint64_t key1, uint64_t first_element,
                                int64_t n_elements, double low, double high, double* out64,
                                float* out32, void* stream);
/* Diagnostic: clock64() sums of the evaluation kernels of one precision
 * (0 = float64, 1 = float32) over CTAs: [0] tile load, [1] z staging
 * (rotate), [2] kernel values, [3] whole tiles, [4] tiles; zeros unless the
 * library is built with -DRB_PHASE_TIMING.  reset != 0 clears them. */
void rb_debug_phases(int32_t precision, uint64_t out[8], int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* ROBENCH_B200_H */
