/*
 * libopevo -- C ABI of the B200 trial evaluator for OpEvo.
 *
 * This library replaces the reference tuner's evaluation seam: the objective
 * callable `Callable[[tuple], float]` consumed by `evaluate_batch` / `run`
 * (reference pkg/src/topotune/engine.py:264-310), whose CPU implementation is
 * the synthetic cost model `synthetic_cost` (benchmarks.py:278-291), and the
 * subprocess protocol `ExternalEvaluator` (external.py:29-75).  A trial is:
 * canonical kernel knobs -> JIT-compiled sm_100a kernel (NVRTC, cubin cache)
 * -> verified against an independent reference on the same synthetic inputs
 * -> timed with CUDA events -> fitness in TFLOP/s.
 *
 * Conventions (mirroring the reference's error semantics, engine.py:276-285):
 *   status  0          ok
 *   status  > 0        this configuration is invalid -> fitness 0
 *                      (infeasible knobs, compile error, launch failure,
 *                       result mismatch)
 *   status  < 0        fatal for the worker (no device / driver / NVRTC, a
 *                      sticky CUDA context error) -> FatalEvaluationError or
 *                      worker respawn
 * Error text is written to the caller's `err` buffer (may be NULL).  No C++
 * exception crosses this boundary.  All pointers are plain; no torch types.
 * Threading: one opevo_ctx per device, used by one thread at a time;
 * opevo_compile() is thread-safe and needs no device (host NVRTC pool).
 */
#ifndef OPEVO_H
#define OPEVO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPEVO_ABI_VERSION 8   /* 8: opevo_ctx_flush_l2_async; 7: opevo_kernels_time_rotating; 6: 14-slot knobs (conv padded lines), conv stride / narrow Cin, conv CTA pairs; 5: timing policy, native search core */

enum opevo_status {
    OPEVO_OK = 0,
    OPEVO_INVALID_CONFIG = 1,   /* knobs infeasible for this operator */
    OPEVO_COMPILE_ERROR = 2,    /* NVRTC rejected the instance        */
    OPEVO_LAUNCH_ERROR = 3,     /* launch refused (non-sticky)        */
    OPEVO_VERIFY_FAILED = 4,    /* output differs from the reference  */
    OPEVO_ERR_NO_DEVICE = -1,   /* libcuda / device unavailable       */
    OPEVO_ERR_NO_NVRTC = -2,    /* libnvrtc unavailable               */
    OPEVO_ERR_STICKY = -3,      /* context poisoned: restart worker   */
    OPEVO_ERR_ARG = -4,         /* caller error                       */
    OPEVO_ERR_CUDA = -5         /* other driver error                 */
};

/* operator kinds (reference benchmarks.py:36-107) */
enum opevo_op_kind { OPEVO_MATMUL = 0, OPEVO_BATCHMATMUL = 1, OPEVO_CONV2D = 2 };
/* OPEVO_F32: fp32 in/out on the CUDA cores (the paper's SIMT schedule, knob
 * slots 0..7 = n2 n3 n4 m2 m3 m4 k2 k3).  OPEVO_F32_TF32X3: fp32 in/out on
 * the tensor cores as three kind::tf32 MMAs per K step (hi*hi + hi*lo +
 * lo*hi), the tcgen05 knob layout with BK in fp32 elements (a multiple of 8;
 * 8, 16 or a multiple of 32 up to 128). */
enum opevo_dtype { OPEVO_BF16 = 0, OPEVO_F32 = 1, OPEVO_F32_TF32X3 = 2 };

/*
 * Operator descriptor.  MatMul / BatchMatMul use GEMM naming:
 *   rows = reference `n`, cols = reference `m`, depth = reference `k`,
 *   batch = reference `b` (1 for MatMul).
 * Conv2d uses conv[] = {batch, cin, h, w, cout, kh, kw, stride, pad}
 * (reference Conv2dSpec field order, benchmarks.py:69-81).
 */
typedef struct opevo_op_desc {
    int32_t kind;
    int32_t dtype;
    int64_t batch, rows, cols, depth;
    int32_t conv[9];
    uint64_t seed;            /* synthetic-input seed */
} opevo_op_desc;

/* Deepest split-K (knob OPEVO_KNOB_SPLIT): the fp32 partial workspace is
 * allocated for this many slices when the operator is prepared. */
#define OPEVO_MAX_SPLIT 16

/* Kernel knob vector: fixed order, OPEVO_NUM_KNOBS entries. */
enum opevo_knob {
    OPEVO_KNOB_BM = 0,        /* CTA tile rows (UMMA M / atoms)          */
    OPEVO_KNOB_BN = 1,        /* CTA tile cols (UMMA N)                  */
    OPEVO_KNOB_BK = 2,        /* K per pipeline stage                    */
    OPEVO_KNOB_STAGES = 3,    /* smem ring depth                          */
    OPEVO_KNOB_SPLIT = 4,     /* split-K factor (runtime)                 */
    OPEVO_KNOB_CLUSTER = 5,   /* CTAs per cluster sharing A (multicast)   */
    OPEVO_KNOB_TILE_H = 6,    /* conv: output rows per CTA tile           */
    OPEVO_KNOB_TILE_W = 7,    /* conv: output cols per CTA tile; 17 - KW
                                 (a width not dividing BM) selects "halo
                                 lines": 16-row lines, one TMA box per
                                 filter row serving its KW taps           */
    OPEVO_KNOB_ACC = 8,       /* K-interleaved TMEM accumulators (1,2,4)  */
    OPEVO_KNOB_CTA_GROUP = 9, /* 2: CTA-pair MMA (cta_group::2), BM=256;
                                 BM=512 (256 rows per CTA, two M=256
                                 atoms) for halo-line conv tiles          */
    OPEVO_KNOB_GRID = 10,     /* 0: persistent when work > residency
                                 1: one CTA (cluster) per tile
                                 2: persistent, partial last wave split
                                    along K (stream-K style tail)         */
    OPEVO_KNOB_B_RES = 11,    /* conv: 1 = the whole weight panel (BN = Cout
                                 x K) is loaded once into shared memory and
                                 stays resident across the CTA's tiles     */
    OPEVO_KNOB_BPU = 12,      /* BatchMatMul: consecutive batches per CTA
                                 work unit (1, 2, 4), loaded by one TMA box
                                 per operand and stage                    */
    OPEVO_KNOB_LINE = 13,     /* conv: 16 / 32 = "padded lines": lines of
                                 TILE_W <= LINE output pixels padded to
                                 LINE tile rows, one TMA box per filter tap
                                 (any stride; widths no power of two
                                 divides); 0 = dense tile or halo lines   */
    OPEVO_NUM_KNOBS = 14
};

/* Result of one trial (opevo_trial). */
typedef struct opevo_trial_result {
    double tflops;            /* fitness: algorithmic FLOPs / device time */
    double ms;                /* device ms per launch                     */
    double rel_err;           /* max|C-R| / max|R| vs the reference       */
    double compile_ms;        /* NVRTC (0 on cache hit)                   */
    double load_ms;           /* module load + launch setup               */
    int32_t cache_hit;        /* 1: memory, 2: disk, 0: compiled          */
    int32_t grid_ctas;
    int32_t smem_bytes;
    int32_t launches;         /* tuned-kernel launches this trial made    */
    int32_t verify_cached;    /* 1: instance verified on these operands by an
                                 earlier trial of the batch API; re-timed,
                                 not re-checked (rel_err is that check's)  */
} opevo_trial_result;

typedef struct opevo_ctx opevo_ctx;
typedef struct opevo_op opevo_op;
typedef struct opevo_kernel opevo_kernel;

int opevo_abi_version(void);

/* NVRTC compile of one instance into the on-disk cubin cache; no device
 * needed.  family: 0 = GEMM, 1 = implicit-GEMM conv, 2 = fp32 SIMT,
 * 3 = fp32 3xTF32 GEMM (out_f32 = 1).  Thread-safe. */
int opevo_compile(int family, const int32_t* knobs, int nknobs, int batched, int out_f32,
                  const char* cache_dir, double* compile_ms, char* err, size_t errlen);

/* Canonical cache key of an instance (writes a NUL-terminated string). */
int opevo_kernel_key(int family, const int32_t* knobs, int nknobs, int batched, int out_f32,
                     char* key, size_t keylen);

int opevo_ctx_create(int device, const char* cache_dir, opevo_ctx** out, char* err, size_t errlen);
void opevo_ctx_destroy(opevo_ctx* ctx);
int opevo_ctx_info(opevo_ctx* ctx, int* sm_count, int* max_smem_optin, int* cc_major, int* cc_minor);

/* Allocate operands, fill them from desc->seed, compute the fp32 reference. */
int opevo_op_prepare(opevo_ctx* ctx, const opevo_op_desc* desc, opevo_op** out,
                     char* err, size_t errlen);
void opevo_op_destroy(opevo_op* op);
/* Operand sizes in bytes (A, B in the kernel layout, C output). */
int opevo_op_sizes(const opevo_op* op, size_t* a_bytes, size_t* b_bytes, size_t* c_bytes);
/* Host <-> device copies for the end-to-end path (inputs in kernel layout:
 * MatMul/BMM A [batch][rows][depth], B [batch][cols][depth]; Conv2d X NHWC,
 * W [Cout][Kh][Kw][Cin]).  Uploading marks the reference stale: the next
 * check recomputes it from the new operands (for Conv2d after converting
 * them back to the paper's NCHW / OIHW layouts), and every instance is
 * verified again. */
int opevo_op_upload(opevo_op* op, const void* a_host, const void* b_host, char* err, size_t errlen);
int opevo_op_download(opevo_op* op, void* c_host, size_t bytes, char* err, size_t errlen);
/* Device operands (kernel layout) to host, e.g. to stage them in pinned memory. */
int opevo_op_read_inputs(opevo_op* op, void* a_host, void* b_host, char* err, size_t errlen);
/* Reference output (fp32, kernel output layout) to host. */
int opevo_op_reference(opevo_op* op, float* host, size_t count, char* err, size_t errlen);
/* Recompute the reference now (opevo_op_upload otherwise defers it to the next check). */
int opevo_op_refresh_reference(opevo_op* op, char* err, size_t errlen);

/* Bind knobs to an operator: validate, fetch/compile the module, build the
 * TMA descriptors and launch plan. */
int opevo_kernel_get(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs,
                     opevo_kernel** out, opevo_trial_result* info, char* err, size_t errlen);
void opevo_kernel_release(opevo_kernel* k);
int opevo_kernel_run(opevo_kernel* k, char* err, size_t errlen);
/* Output vs reference; *rel_err = max|C-R|/max|R| (inf if non-finite). */
int opevo_kernel_check(opevo_kernel* k, double tol, double* rel_err, char* err, size_t errlen);
/* flush_l2 = 0: `reps` back-to-back launches in one CUDA graph (PDL edges,
 *               L2 warm; captured while the warm-up runs) -- the fitness;
 * flush_l2 = 1: an L2-sized write before every launch, each launch timed;
 * flush_l2 = 2: `reps` back-to-back stream launches released together from a
 *               device-side gate (no graph, no host gaps).
 * Exactly `reps` timed launches: the per-trial device budget
 * (OPEVO_TIME_BUDGET_MS) that caps repetitions of slow candidates applies to
 * opevo_trial / opevo_trial_batch only. */
int opevo_kernel_time(opevo_kernel* k, int warmup, int reps, int flush_l2, double* ms_per_launch,
                      char* err, size_t errlen);

/* HBM-fed back-to-back timing for operators below the ridge: `reps` launches
 * cycling through `n` kernels of the same instance bound to n distinct
 * operand copies (one opevo_op each, prepared alike) in one CUDA graph, PDL
 * between launches as in every other mode.  With n copies spanning more than
 * twice the L2, each launch's operands were evicted since their last use, so
 * the kernel streams them from HBM while its prologue still overlaps the
 * previous launch -- the steady state of a tuned kernel in a pipeline whose
 * working set does not fit in L2.  All kernels must belong to one context. */
int opevo_kernels_time_rotating(opevo_kernel* const* ks, int n, int warmup, int reps,
                                double* ms_per_launch, char* err, size_t errlen);

/* One complete trial: get + check (tol) + time, with one host synchronisation
 * before the timed launches.  Fitness in res->tflops. */
int opevo_trial(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, int warmup,
                int reps, int flush_l2, double tol, opevo_trial_result* res, char* err,
                size_t errlen);

/* Up to OPEVO_MAX_BATCH trials (knobs: count x nknobs, row-major) with two
 * host synchronisations in total: every instance's check, warm-up and
 * estimate are enqueued together (their timed graphs are built meanwhile),
 * then all timed launches run back to back.  status[i] / res[i] / the
 * NUL-terminated message at msgs + i * msg_stride are per trial, as
 * opevo_trial would return them.  The return value is OPEVO_OK unless a
 * fatal (< 0) error aborted the batch; unfinished trials then carry it. */
#define OPEVO_MAX_BATCH 64
int opevo_trial_batch(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs, int count,
                      int warmup, int reps, int flush_l2, double tol, opevo_trial_result* res,
                      int32_t* status, char* msgs, size_t msg_stride, char* err, size_t errlen);

/* Compile-or-read and load the module of one instance into the context's
 * module cache (no launch).  Thread-safe with respect to other preloads and
 * to the trial thread, so a host pool can stage the next batch's modules.
 * Status as for opevo_kernel_get's structural checks. */
int opevo_op_preload(opevo_ctx* ctx, opevo_op* op, const int32_t* knobs, int nknobs,
                     double* compile_ms, int* cache_hit, char* err, size_t errlen);

/* Debug: launches of an instance compiled with OPEVO_EXTRA_FLAGS=-DOPEVO_TRACE=1;
 * copies 16 uint64 per CTA (smid, %globaltimer phase stamps) to `host`.  When
 * `count` holds L > 1 launches' worth (L <= 8), L launches run back to back
 * (as in timing) and launch i's stamps follow launch i-1's. */
int opevo_kernel_trace(opevo_kernel* k, uint64_t* host, size_t count, char* err, size_t errlen);

/* Trial timing policy of opevo_trial / opevo_trial_batch on this context.
 * budget_ms (default OPEVO_TIME_BUDGET_MS or 0.3; <= 0 disables): a
 * candidate whose verified launch alone exceeds it is timed by that launch;
 * otherwise the repetitions are capped at budget_ms / (one-launch time),
 * min 5.  loser_ratio (default 0 = off): a verified candidate whose
 * one-launch time exceeds loser_ratio x the fastest one verified on the same
 * operator so far gets loser_reps timed launches and no extra warm-up. */
int opevo_ctx_set_timing(opevo_ctx* ctx, double budget_ms, double loser_ratio, int loser_reps);

/* Read a 256 MB buffer (2x L2) on the context's stream so the next work
 * starts with a cold L2 holding only clean lines (no write-backs land on the
 * next work); returns after the flush completes. */
int opevo_ctx_flush_l2(opevo_ctx* ctx, char* err, size_t errlen);

/* The same read pass, enqueued without waiting: the context's later work
 * (same stream) still starts after it, while the host goes on (e.g. with the
 * next generation's ask) -- bench.py's per-step flush. */
int opevo_ctx_flush_l2_async(opevo_ctx* ctx, char* err, size_t errlen);

/* Pinned host memory for honest end-to-end copies. */
void* opevo_host_alloc(size_t bytes);
void opevo_host_free(void* p);

/* ------------------------------------------------------------------------
 * Native OpEvo proposal core (host only, no device).  Replaces the Python
 * ask path of the reference -- OpEvo._initial_batch / _offspring_batch,
 * recombine, mutate / sample_walk, the four neighbour relations and unrank,
 * the archive ranking (pkg/src/topotune/engine.py:73-261, walk.py:41-59,
 * spaces.py:71-84, 189-221, 266-289, 334-342, 385-387) -- drawing from
 * numpy's Generator(PCG64) stream exactly as the reference does, so its
 * proposals are the reference's bit for bit under the same told fitness.
 * A configuration crosses the ABI as int64 "slots": a factorization value
 * is its factor tuple, a permutation value its item indices, a discrete /
 * categorical value its index in the declared list.
 * ---------------------------------------------------------------------- */
enum opevo_param_kind {
    OPEVO_PARAM_FACTORIZATION = 0,   /* a = product, arity = tuple length   */
    OPEVO_PARAM_DISCRETE = 1,        /* a = number of values (a path graph)  */
    OPEVO_PARAM_CATEGORICAL = 2,     /* a = number of labels (complete graph) */
    OPEVO_PARAM_PERMUTATION = 3      /* a = number of items (<= 20)          */
};
#define OPEVO_SEARCH_WALK_LIMIT (-10)   /* a q-walk did not stop within 1e6 steps */

typedef struct opevo_search opevo_search;

int opevo_search_create(int nparams, const int32_t* kinds, const int64_t* a, const int32_t* arity,
                        int parents, int offspring, double q, int retry_cap, opevo_search** out);
void opevo_search_destroy(opevo_search* s);
/* int64 slots per configuration (sum of the parameters' arities) */
int opevo_search_slots(const opevo_search* s);
/* numpy PCG64 state: st = {state hi, state lo, inc hi, inc lo}, plus the
 * buffered upper 32-bit half (has_uint32, uinteger) */
int opevo_search_set_rng(opevo_search* s, const uint64_t st[4], int has_uint32, uint32_t uinteger);
int opevo_search_get_rng(const opevo_search* s, uint64_t st[4], int* has_uint32, uint32_t* uinteger);
/* Up to `want` proposals of the pending batch into out[want][slots]:
 * initial = 1 for the first batch (uniform draws, deduplicated in-batch),
 * else offspring of the archive's top `parents` (deduplicated against the
 * archive and the batch); first = 1 starts a new batch.  Returns how many
 * were made; *need_fallback = 1 when the next one exhausted the retry cap:
 * the caller draws it with sample_unvisited from this RNG state (get_rng /
 * set_rng around it), records it with opevo_search_add_pending and calls
 * again for the rest. */
int opevo_search_propose(opevo_search* s, int initial, int first, int want, int64_t* out,
                         int* need_fallback);
int opevo_search_add_pending(opevo_search* s, const int64_t* slots);
/* Insert evaluated configurations in ask order (ranked by fitness, ties by
 * insertion); ends the pending batch. */
int opevo_search_tell(opevo_search* s, int n, const int64_t* slots, const double* fitness);
/* RNG primitives (tests of the stream contract) */
int opevo_search_uniform_int(opevo_search* s, uint64_t n, uint64_t* out);
int opevo_search_random(opevo_search* s, double* out);
double opevo_search_np_sum(const double* a, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* OPEVO_H */
