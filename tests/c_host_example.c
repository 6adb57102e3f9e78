/* C host of libhimeno_b200.so (the INTEGRATION.md example, complete).
 * Evaluates Himeno XS under pattern 0000001000000 (loop 6 = device time loop)
 * with the batched plan's events; prints wall time and gosa.
 * Exit: 0 ok, 1 pattern failure, 2 environment failure (no device). */
#include <stdio.h>

#include "himeno_b200.h"

int main(void) {
  hp_grid g = {33, 33, 65};
  hp_ctx* ctx = NULL;
  if (hp_create(0, &g, 0, &ctx) != HP_OK) {
    printf("environment: %s\n", hp_last_error());
    return 2;
  }
  /* Planner.plan(0000001000000): globals declared + update device/self at loop 6,
   * locals (nn, gosa, s0, ss) as structured data regions around loop 6. */
  const int arrays[] = {HP_V_P, HP_V_BND, HP_V_WRK1, HP_V_WRK2, HP_V_A, HP_V_B, HP_V_C,
                        HP_V_IMAX, HP_V_JMAX, HP_V_KMAX, HP_V_OMEGA};
  hp_event ev[64];
  int n = 0;
  for (unsigned v = 0; v < sizeof arrays / sizeof arrays[0]; ++v) {
    hp_event d = {-1, HP_BEFORE, HP_EV_DECLARE, arrays[v], 0, (int)v};
    hp_event u = {6, HP_BEFORE, HP_EV_UPDATE_DEVICE, arrays[v], 0, (int)v};
    ev[n++] = d;
    ev[n++] = u;
  }
  hp_event out = {6, HP_AFTER, HP_EV_UPDATE_SELF, HP_V_P, 0, 0};
  ev[n++] = out;
  const int locals[] = {HP_V_NN, HP_V_GOSA, HP_V_S0, HP_V_SS};
  const int copyout[] = {0, 1, 0, 0};
  for (int v = 0; v < 4; ++v) {
    hp_event in = {6, HP_BEFORE, HP_EV_DATA_ENTER, locals[v], 1, 11 + v};
    hp_event ex = {6, HP_AFTER, HP_EV_DATA_EXIT, locals[v], copyout[v], 11 + v};
    ev[n++] = in;
    ev[n++] = ex;
  }
  hp_schedule s = {HP_NLOOPS, {0, 0, 0, 0, 0, 0, HP_K_PARALLEL_LOOP, 4, 4, 4, 4, 4, 4},
                   n, ev, /*nn=*/3,
                   HP_FLAG_COHERENCE_GUARD | HP_FLAG_FRESH_PROCESS | HP_FLAG_FUSED_TIME_LOOP,
                   /*timeout_s=*/180.0};
  hp_result r;
  const int rc = hp_run(ctx, &s, &r);
  if (rc != HP_OK) {
    printf("run failed (%d): %s\n", rc, hp_last_error());
    hp_destroy(ctx);
    return rc > 0 ? 1 : 2;
  }
  printf("wall_s %.6f launches %llu gosa %.17g\n", r.wall_s, (unsigned long long)r.n_launch,
         r.gosa);
  hp_destroy(ctx);
  return 0;
}
