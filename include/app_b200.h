/* C ABI of a generated B200 executor (codegen.py): one shared library per
 * application text, libapp_<app>.so, exporting the same entry points.
 *
 * It replaces, for any program the reference's parser accepts, what
 * ExternalEvaluator.measure does per genome (pkg/src/acctuner/evaluators.py:
 * 178-222: emit the OpenACC variant, compile it, run and time it): the
 * program is compiled once with every loop's host and device versions, and a
 * genome selects per loop which one runs; the reference's TransferPlan
 * (transfer.py:413-418) arrives as loop-anchored events, as for the Himeno
 * library (include/himeno_b200.h, whose event / kind / status codes these
 * reuse).  Return codes: 0 ok, > 0 pattern failure (MeasuredTime.failed /
 * timeout), < 0 environment failure (EvaluatorUnavailable).
 */
#ifndef APP_B200_H
#define APP_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpg_ctx hpg_ctx;

typedef struct {
  int32_t loop_id; /* -1: program start */
  int32_t when;    /* 0 before the loop statement, 1 after */
  int32_t op;      /* 1 update device, 2 update self, 3 data enter, 4 data exit,
                      5 declare create, 6 present */
  int32_t var;     /* index into hpg_var_name() */
  int32_t arg;     /* enter: copy in?  exit: copy out? */
  int32_t entry;   /* plan entry index (diagnostics) */
} hpg_event;

typedef struct {
  int32_t n_loops;
  const int32_t* loop_kind; /* per loop: 0 host, 1 kernels, 2 parallel loop,
                               3 parallel loop vector, 4 covered by an outer one */
  int32_t n_events;
  const hpg_event* events;
  int32_t flags;            /* 1 coherence guard, 2 fresh process */
  double timeout_s;
} hpg_schedule;

typedef struct {
  double wall_s;            /* host wall clock around the program run */
  double xfer_s;
  uint64_t h2d_bytes, d2h_bytes, n_h2d, n_d2h, n_skipped_stale, n_implicit, n_launch;
  uint64_t n_guard_init;     /* device copies initialised from the host before a partial write */
  int32_t status;
  char diag[256];
} hpg_result;

/* device < 0: host-only context (every loop must run on the host) */
int hpg_create(int device, hpg_ctx** out);
void hpg_destroy(hpg_ctx* c);
int hpg_run(hpg_ctx* c, const hpg_schedule* s, hpg_result* r);
/* the program's stdout of the last run (printf), NUL-terminated; returns its length */
size_t hpg_output(hpg_ctx* c, char* dst, size_t cap);
int hpg_n_loops(void);
int hpg_n_vars(void);
const char* hpg_var_name(int var);
/* per loop: the directive kind it was generated for (0 = host only) and a note
   on the device mapping ("grid/3", "block/1", "seq/1 loop-carried scalar x") */
int hpg_loop_kind(int loop);
const char* hpg_loop_note(int loop);
const char* hpg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
