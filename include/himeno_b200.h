/*
 * himeno_b200.h -- C ABI of libhimeno_b200.so, the B200 fitness-evaluation engine.
 *
 * The reference evaluates one genome by emitting OpenACC C, compiling it and
 * timing the process (acctuner/evaluators.py:178-222, ExternalEvaluator.measure
 * -> _compile_and_run).  This library replaces that compile+run step: the
 * Python evaluator lowers (genome, directive kinds, loop tree, TransferPlan)
 * into an hp_schedule and one hp_run() call executes the Himeno program under
 * that pattern -- gene=1 loops as sm_100a kernels, gene=0 loops as C++ host
 * loops, plan entries as pinned host<->device transfers -- and reports the
 * wall time the reference would have measured around the process
 * (evaluators.py:207-214).
 *
 * Reference interface each entry point replaces:
 *   hp_run          ExternalEvaluator.measure / _compile_and_run   evaluators.py:178-181, 190-222
 *   hp_result.gosa  + samples: the program's stdout that
 *                   ExternalEvaluator.run_for_output returns      evaluators.py:183-188
 *   status codes    MeasuredTime.ok / timeout / failed             evaluators.py:28-46
 *   hp_last_error   diagnostic text of MeasuredTime.failed / EvaluatorUnavailable
 *                                                                   evaluators.py:204-205, 219-222
 *   hp_create/hp_destroy  one device context per evaluator worker; the reference's
 *                   max_concurrency thread pool (ga.py:222-230) leases one each.
 *
 * Conventions: plain C types only; all pointers are caller-owned and only
 * read during the call; a context is NOT re-entrant, distinct contexts may be
 * used concurrently from different threads (ctypes releases the GIL).
 * Return codes: 0 ok; >0 pattern-level failure (maps to MeasuredTime.failed /
 * timeout, the GA continues); <0 environment failure (maps to
 * EvaluatorUnavailable, the run aborts).
 */
#ifndef HIMENO_B200_H
#define HIMENO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_ABI_VERSION 2

/* ---- status codes ------------------------------------------------------ */
enum hp_status {
  HP_OK = 0,
  HP_FAIL_PATTERN = 1,   /* invalid pattern, e.g. nested compute construct      */
  HP_FAIL_LAUNCH = 2,    /* kernel launch / execution error                      */
  HP_TIMEOUT = 3,        /* watchdog (hp_schedule.timeout_s) expired             */
  HP_FAIL_PRESENT = 4,   /* present assertion failed (data not on device)        */
  HP_ERR_DEVICE = -1,    /* no device / CUDA context failure                     */
  HP_ERR_ARG = -2,       /* bad argument (null pointer, wrong sizes)             */
  HP_ERR_OOM = -3        /* device or pinned host allocation failed              */
};

/* ---- program description (Himeno, apps/himeno.py) ---------------------- */
#define HP_NLOOPS 13     /* loop ids 0..12 in document order                    */
#define HP_NFIELDS 14    /* fp32 arrays                                          */

enum hp_field {          /* device/host fp32 arrays, each I*J*K               */
  HP_F_P = 0, HP_F_BND, HP_F_WRK1, HP_F_WRK2,
  HP_F_A0, HP_F_A1, HP_F_A2, HP_F_A3,
  HP_F_B0, HP_F_B1, HP_F_B2,
  HP_F_C0, HP_F_C1, HP_F_C2
};

enum hp_var {            /* plannable variables of the program (VarRefTable keys) */
  HP_V_P = 0,            /* p                      -> HP_F_P                   */
  HP_V_BND,              /* bnd                                                */
  HP_V_WRK1,             /* wrk1                                               */
  HP_V_WRK2,             /* wrk2                                               */
  HP_V_A,                /* a[4]                   -> HP_F_A0..A3              */
  HP_V_B,                /* b[3]                                               */
  HP_V_C,                /* c[3]                                               */
  HP_V_IMAX, HP_V_JMAX, HP_V_KMAX, HP_V_OMEGA,   /* global scalars             */
  HP_V_NN,               /* jacobi:nn                                          */
  HP_V_GOSA,             /* jacobi:gosa (carried in fp64)       */
  HP_V_S0, HP_V_SS,      /* jacobi:s0, jacobi:ss (private in kernels)          */
  HP_V_MAIN_GOSA,        /* main:gosa (never on device)                        */
  HP_NVARS
};

enum hp_kind {           /* per-loop execution: gene 0 = host, else directive kind */
  HP_K_HOST = 0,
  HP_K_KERNELS = 1,      /* collapse the tight nest below the loop into one launch */
  HP_K_PARALLEL_LOOP = 2,/* one gang per iteration of this loop, vector inside     */
  HP_K_PLV = 3,          /* parallel loop vector: one gang, vector lanes only      */
  HP_K_COVERED = 4       /* inside a device anchor (executed by the anchor)        */
};

enum hp_event_op {       /* data-manager events lowered from TransferPlan entries */
  HP_EV_UPDATE_DEVICE = 1,  /* temp_region && into_device   : before each open  */
  HP_EV_UPDATE_SELF = 2,    /* temp_region && out_of_device : after each close  */
  HP_EV_DATA_ENTER = 3,     /* structured region enter, arg = copyin            */
  HP_EV_DATA_EXIT = 4,      /* structured region exit,  arg = copyout           */
  HP_EV_DECLARE = 5,        /* declare create (program lifetime), loop_id = -1  */
  HP_EV_PRESENT = 6         /* present assertion at a covered anchor            */
};

enum hp_when { HP_BEFORE = 0, HP_AFTER = 1 };

typedef struct hp_grid {
  int32_t I, J, K;       /* static extents, k contiguous (RIKEN MIMAX/MJMAX/MKMAX) */
} hp_grid;

typedef struct hp_event {
  int32_t loop_id;       /* statement the event is attached to (-1: program start) */
  int32_t when;          /* hp_when                                                */
  int32_t op;            /* hp_event_op                                            */
  int32_t var;           /* hp_var                                                 */
  int32_t arg;           /* copy flag for DATA_ENTER / DATA_EXIT                   */
  int32_t entry;         /* index of the PlanEntry it came from (diagnostics)      */
} hp_event;

enum hp_flags {
  HP_FLAG_COHERENCE_GUARD = 1,  /* skip transfers from a stale copy    */
  HP_FLAG_FRESH_PROCESS = 2,    /* reset host arrays to static-zero before the run  */
  HP_FLAG_POISON_DEVICE = 4,    /* fill device mirrors with NaN before the run      */
  HP_FLAG_KERNEL_TIMING = 8,    /* CUDA events around every launch (slower)         */
  HP_FLAG_GRAPH_TIME_LOOP = 16, /* reserved, no effect: the time loop's passes are
                                   enqueued back to back with programmatic dependent
                                   launch, or as one flow launch (a captured graph
                                   would replay a flow launch's completion tags)     */
  HP_FLAG_FUSED_TIME_LOOP = 32, /* time loop: fused stencil with p/wrk2 rotation    */
  HP_FLAG_HOST_REFERENCE = 128, /* genes = 0: the reference-faithful host build
                                   (the program's loops, gcc -O2) instead of the
                                   tuned one (-O3 -march=x86-64-v3); same values     */
  HP_FLAG_LITERAL_GOSA = 64     /* verification: when the last iteration's stencil
                                   runs on the device, its ss*ss terms are also
                                   written out (side kernel on the same device
                                   state) and summed in program order on the host
                                   after the timed run -> gosa_f32 literal          */
};

typedef struct hp_schedule {
  int32_t n_loops;                 /* must be HP_NLOOPS                            */
  int32_t loop_kind[HP_NLOOPS];    /* hp_kind per loop id                          */
  int32_t n_events;
  const hp_event* events;          /* program order within one (loop, when) slot   */
  int32_t nn;                      /* jacobi(nn) iteration count                   */
  int32_t flags;                   /* hp_flags                                     */
  double timeout_s;                /* watchdog; <= 0 disables                      */
} hp_schedule;

#define HP_MAX_SAMPLES 8

typedef struct hp_result {
  double wall_s;          /* host wall clock around the program run (the fitness time) */
  double kernel_s;        /* sum of kernel durations (HP_FLAG_KERNEL_TIMING only)       */
  double host_s;          /* time in host (gene=0) loop nests                           */
  double xfer_s;          /* host time blocked in transfers                             */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t n_h2d, n_d2h;            /* issued transfers                                 */
  uint64_t n_skipped_stale;         /* plan transfers skipped by the coherence guard    */
  uint64_t n_implicit;              /* implicit present_or_copy transfers               */
  uint64_t n_launch;                /* kernels launched                                 */
  uint64_t n_stale_reads;           /* compute read a copy older than the other side    */
  double gosa;            /* jacobi's gosa, terms summed in fp64 (host copy at return) */
  float samples[HP_MAX_SAMPLES];    /* main's printed p samples (host copy)         */
  int32_t n_samples;
  float gosa_f32;         /* main's printed float gosa: the program's literal fp32
                             sequential sum when every ss*ss term of the last
                             iteration was summed on the host, or with
                             HP_FLAG_LITERAL_GOSA (gosa_f32_literal = 1); else
                             (float)gosa -- a parallel device reduction has no
                             sequential order to reproduce (B.5)      */
  int32_t gosa_f32_literal;
  int32_t status;         /* hp_status                                              */
  char diag[256];
} hp_result;

/* ---- library ------------------------------------------------------------ */
int hp_abi_version(void);
int hp_device_count(void);
const char* hp_last_error(void);   /* thread-local message of the last failure */

/* ---- context: one per device/worker --------------------------------------- */
typedef struct hp_ctx hp_ctx;
int hp_create(int device, const hp_grid* grid, int flags, hp_ctx** out);
void hp_destroy(hp_ctx* ctx);
void* hp_stream(hp_ctx* ctx);      /* the cudaStream_t every launch/copy uses */

/* Set the p-sample points main prints (i,j,k triples); default: none. */
int hp_set_samples(hp_ctx* ctx, int n, const int32_t* ijk);

/* ---- fitness evaluation: run the program under one pattern ---------------- */
int hp_run(hp_ctx* ctx, const hp_schedule* sched, hp_result* res);

/* ---- field access (parity / e2e) ------------------------------------------ */
/* side 0 = host copy (the program's static array), 1 = device mirror.
 * dst/src hold I*J*K floats in the program's [i][j][k] layout. */
int hp_read_field(hp_ctx* ctx, int field, int side, float* dst, size_t n);
int hp_write_field(hp_ctx* ctx, int field, int side, const float* src, size_t n);
int hp_read_gosa(hp_ctx* ctx, int side, double* out);

/* ---- device-resident Jacobi (bench value / e2e) ----------------------------
 * hp_jacobi_device: nn iterations of jacobi's loop body on the device mirrors,
 * enqueued on hp_stream(ctx) without host synchronisation.  variant: 0 = one
 * stencil + one copy launch per iteration (the unfused loop body), 1 = fused
 * time loop (p/wrk2 rotation, copy nest elided; two iterations per stencil
 * pass while temporal blocking is on).
 * hp_jacobi_host: end-to-end offload of jacobi(nn) from host buffers: H2D of
 * the 13 input fields (fields[HP_F_*], wrk2 ignored), the device loop, D2H of
 * p into p_out and gosa into *gosa_out; synchronous.  Host buffers may be
 * pageable or pinned (pinned is faster). */
int hp_jacobi_device(hp_ctx* ctx, int nn, int variant);
int hp_jacobi_host(hp_ctx* ctx, const float* const* fields, int nn, int variant,
                   float* p_out, double* gosa_out);
/* hp_jacobi_host_async: hp_jacobi_host without the final synchronisation: the
 * copies and launches are enqueued on hp_stream(ctx) and the call returns;
 * p_out and *gosa_out are valid after hp_sync(ctx).  With pinned host buffers
 * the copies are asynchronous, so two contexts on one device pipeline
 * consecutive jobs (one job's H2D overlaps the other's loop and D2H).  One
 * outstanding call per context (HP_ERR_ARG otherwise).
 * hp_sync: wait for everything enqueued on the context; deliver gosa. */
int hp_jacobi_host_async(hp_ctx* ctx, const float* const* fields, int nn, int variant,
                         float* p_out, double* gosa_out);
int hp_sync(hp_ctx* ctx);
/* Initialise the device mirrors to the program's post-initmt state on device. */
int hp_init_device(hp_ctx* ctx);

/* ---- device timing (bench.py) ----------------------------------------------
 * hp_time_steps: CUDA events on hp_stream(ctx) around `steps` back-to-back
 * hp_jacobi_device(nn, variant) calls; synchronous; *ms_out = elapsed ms.
 * hp_time_jacobi: one jacobi(nn) call with events around every launch; reports
 * the mean duration of the stencil launches and of the other launches. */
typedef struct hp_kernel_times {
  double total_ms;        /* first to last event of the call                 */
  double stencil_ms;      /* mean duration of one stencil launch (pass)       */
  double other_ms;        /* mean duration of the other launches (copies)     */
  double stencil_iters;   /* mean Jacobi iterations per stencil launch: 1, 2 (two-step
                             pass) or all pairs of a flow launch (stencil_flow_ok) */
  int32_t n_stencil, n_other;
} hp_kernel_times;
int hp_time_steps(hp_ctx* ctx, int steps, int nn, int variant, double* ms_out);
int hp_time_jacobi(hp_ctx* ctx, int nn, int variant, hp_kernel_times* out);
uint64_t hp_launch_count(hp_ctx* ctx);   /* kernels launched by this context so far */
/* Tuning sweeps: select the tuned-stencil configuration (vector width x CTAs
 * per SM, process-wide); returns the number of configurations, <0 if invalid. */
int hp_set_stencil_config(int cfg);
/* Two Jacobi iterations per stencil pass in the device time loop (temporal
 * blocking; default on); on < 0 queries; returns the previous setting. */
int hp_set_temporal_blocking(int on);

/* ---- slab decomposition over several GPUs -----------------
 * The interior planes [1, I-2) of the slowest dimension are split into
 * contiguous slabs (hp_slab_range); a slab context holds global planes
 * [i_begin-1, i_end+1) (its interior + one halo plane each side) and supports
 * hp_init_device / hp_read_field (local planes) / hp_read_gosa.
 * hp_group_jacobi: one thread drives n slab contexts (in-process; halo planes by
 * cudaMemcpyPeerAsync, also usable with several slabs on one GPU); *gosa_out =
 * global gosa.  hp_dd_*: one process per GPU over NCCL (dlopen'ed libnccl.so.2):
 * rank 0 makes the id with hp_nccl_unique_id, every rank passes it to
 * hp_dd_init; hp_dd_jacobi enqueues nn iterations with halo send/recv after each
 * and one fp64 all-reduce of gosa (read it with hp_read_gosa(ctx, 1, ...)). */
int hp_slab_range(int I, int nranks, int rank, int32_t* i_begin, int32_t* i_end);
int hp_create_slab(int device, const hp_grid* global, int i_begin, int i_end, hp_ctx** out);
int hp_group_jacobi(hp_ctx** ctxs, int n, int nn, double* gosa_out);
int hp_nccl_unique_id(unsigned char* out, size_t n);
int hp_dd_init(hp_ctx* ctx, int nranks, int rank, const unsigned char* id, size_t n);
int hp_dd_jacobi(hp_ctx* ctx, int nn);
int hp_dd_time_steps(hp_ctx* ctx, int steps, int nn, double* ms_out);

/* Diagnostics: the dynamic shared-memory limit (bytes) the large-shared-memory
 * kernel `id` has in `device`'s context (0..2 single-step stencil with 2..4
 * stages, 3..6 two-step shapes, 7 two-step with the tensor-memory stash, 8 the
 * two-step tile-exchange kernel, 9 kernel 7 with evict_first coefficient loads, used
 * by flow launches, 10 kernel 7 with the cross-warp stash, 11 kernel 10 for flow launches
 * (evict_first, coefficients-first order), 12 kernel 10 with the coefficients-first order
 * -- 10 / 11 / 12 are the defaults).  The library raises it per device before the
 * first launch there. */
int hp_smem_optin(int id, int device, int* bytes);
/* Diagnostics: the kernel the most recent two-step launch (any context) used:
 * 0 none yet, 1 k_stencil_tb2 (halo-recomputing tiles, one pass), 2 k_stencil_tx
 * (tiles exchanging their p1 boundary through L2), 3 k_stencil_tb2 running several
 * passes in one flow launch (the device time loop's default for nn >= 4). */
int hp_last_two_step_kernel(void);
/* Diagnostics: 1 if an exchange-kernel launch of this context ever timed out
 * waiting for a neighbour tile (its results are invalid and gosa was set to NaN),
 * 0 if not, <0 on error.  Synchronous. */
int hp_tx_status(hp_ctx* ctx);

/* Pinned host buffers for callers without their own allocator (e2e inputs). */
void* hp_host_alloc(size_t bytes);
void hp_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* HIMENO_B200_H */
