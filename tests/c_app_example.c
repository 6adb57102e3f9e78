/* A plain C host of a generated executor (include/app_b200.h): runs the all-CPU
 * pattern of NAS FT class S on a host-only context (device -1) or, with argv[1]
 * = "gpu", its twiddle loop (loop 0) on device 0, and prints the program's stdout.
 * Exit codes: 0 ok, 1 pattern failure, 2 environment failure. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "app_b200.h"

int main(int argc, char** argv) {
  const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
  hpg_ctx* ctx = NULL;
  int rc = hpg_create(gpu ? 0 : -1, &ctx);
  if (rc != 0) {
    printf("environment: %s\n", hpg_last_error());
    return 2;
  }
  const int n = hpg_n_loops();
  int32_t* kinds = calloc((size_t)n, sizeof(int32_t));
  if (gpu) kinds[0] = hpg_loop_kind(0);   /* the loop's directive kind */
  hpg_schedule s = {n, kinds, 0, NULL, 1 | 2, 60.0};
  hpg_result r;
  rc = hpg_run(ctx, &s, &r);
  if (rc != 0) {
    printf("%s: %s\n", rc < 0 ? "environment" : "pattern", hpg_last_error());
    hpg_destroy(ctx);
    free(kinds);
    return rc < 0 ? 2 : 1;
  }
  char out[4096];
  hpg_output(ctx, out, sizeof out);
  fputs(out, stdout);
  fprintf(stderr, "wall %.3f ms, %llu launches\n", r.wall_s * 1e3, (unsigned long long)r.n_launch);
  hpg_destroy(ctx);
  free(kinds);
  return 0;
}
