/*
 * himeno_oracle.c -- CPU ORACLE for the Himeno hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this; the product path (libhimeno_b200.so) never
 * calls it.
 *
 * What it restates: the application the reference tunes, i.e. the Himeno
 * C-subset program emitted by paper_2002_12115_b200/apps/himeno.py (RIKEN
 * himenoBMTxps.c static version [third party, not in /root/reference],
 * restated per SURVEY.md Appendix A), executed as the reference's
 * ExternalEvaluator would run it: compiled by gcc with the pragmas ignored
 * (acctuner/evaluators.py:190-222).  Loop bodies:
 *   loops 0-2  initmt zero nest          (himeno.py _TEMPLATE, "for(i=0;i<I;i++)")
 *   loops 3-5  initmt coefficient nest
 *   loop  6    jacobi time loop, gosa = 0 per iteration
 *   loops 7-9  19-point stencil, gosa += ss*ss, wrk2 = p + omega*ss
 *   loops 10-12 p = wrk2
 *
 * Pinning: tests/test_oracle.py checks oracle_run()'s fp32-sequential gosa and
 * p samples against the tests/golden .stdout files, the stdout of the reference's own
 * ExternalEvaluator.run_for_output on the same program text
 * (oracle/pin_reference.py).  gosa is reported two ways: the literal fp32
 * sequential sum (what the C program prints) and an fp64 sum of the same fp32
 * terms ss*ss (what the B200 path computes).
 *
 * Build (oracle/Makefile): gcc -O2 -ffp-contract=off -fPIC -shared [-fopenmp]
 * -- no FMA contraction, so every product/sum rounds like the C program.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NF 14
enum { F_P, F_BND, F_WRK1, F_WRK2, F_A0, F_A1, F_A2, F_A3, F_B0, F_B1, F_B2, F_C0, F_C1, F_C2 };

typedef struct {
  float* f[NF];
  int I, J, K;
} fields_t;

static size_t at(const fields_t* F, int i, int j, int k) {
  return ((size_t)i * F->J + j) * (size_t)F->K + k;
}

/* loops 0-5 (initmt) */
static void initmt(fields_t* F) {
  const int I = F->I, J = F->J, K = F->K;
  const int imax = I - 1, jmax = J - 1, kmax = K - 1;
  for (int i = 0; i < I; i++)
    for (int j = 0; j < J; j++)
      for (int k = 0; k < K; k++) {
        size_t c = at(F, i, j, k);
        for (int f = 0; f < NF; f++)
          if (f != F_WRK2) F->f[f][c] = 0.0f;
      }
  for (int i = 0; i < imax; i++)
    for (int j = 0; j < jmax; j++)
      for (int k = 0; k < kmax; k++) {
        size_t c = at(F, i, j, k);
        F->f[F_A0][c] = 1.0f;
        F->f[F_A1][c] = 1.0f;
        F->f[F_A2][c] = 1.0f;
        F->f[F_A3][c] = (float)(1.0 / 6.0);
        F->f[F_B0][c] = 0.0f;
        F->f[F_B1][c] = 0.0f;
        F->f[F_B2][c] = 0.0f;
        F->f[F_C0][c] = 1.0f;
        F->f[F_C1][c] = 1.0f;
        F->f[F_C2][c] = 1.0f;
        F->f[F_P][c] = (float)(i * i) / (float)((imax - 1) * (imax - 1));
        F->f[F_WRK1][c] = 0.0f;
        F->f[F_BND][c] = 1.0f;
      }
}

/* one (i) plane of loops 7-9; returns the fp64 sum, updates the fp32 sum in order */
static double stencil_plane(fields_t* F, int i, int jmax, int kmax, float omega, float* gosa32) {
  const size_t R = (size_t)F->K, L = (size_t)F->J * F->K;
  const float* p = F->f[F_P];
  double acc = 0.0;
  float g = gosa32 ? *gosa32 : 0.0f;
  for (int j = 1; j < jmax - 1; j++)
    for (int k = 1; k < kmax - 1; k++) {
      const size_t c = at(F, i, j, k);
      float s0 = F->f[F_A0][c] * p[c + L] + F->f[F_A1][c] * p[c + R] + F->f[F_A2][c] * p[c + 1] +
                 F->f[F_B0][c] * (p[c + L + R] - p[c + L - R] - p[c - L + R] + p[c - L - R]) +
                 F->f[F_B1][c] * (p[c + R + 1] - p[c - R + 1] - p[c + R - 1] + p[c - R - 1]) +
                 F->f[F_B2][c] * (p[c + L + 1] - p[c - L + 1] - p[c + L - 1] + p[c - L - 1]) +
                 F->f[F_C0][c] * p[c - L] + F->f[F_C1][c] * p[c - R] + F->f[F_C2][c] * p[c - 1] +
                 F->f[F_WRK1][c];
      float ss = (s0 * F->f[F_A3][c] - p[c]) * F->f[F_BND][c];
      float t = ss * ss;
      g = g + t;
      acc += (double)t;
      F->f[F_WRK2][c] = p[c] + omega * ss;
    }
  if (gosa32) *gosa32 = g;
  return acc;
}

static void copy_plane(fields_t* F, int i, int jmax, int kmax) {
  for (int j = 1; j < jmax - 1; j++) {
    size_t c = at(F, i, j, 1);
    if (kmax - 2 > 0) memcpy(F->f[F_P] + c, F->f[F_WRK2] + c, (size_t)(kmax - 2) * sizeof(float));
  }
}

/* loop 6: nn iterations; gosa of the last iteration, both accumulations */
static void jacobi(fields_t* F, int nn, double* gosa64, float* gosa32, int threads) {
  const int imax = F->I - 1, jmax = F->J - 1, kmax = F->K - 1;
  const float omega = 0.8f;
  double g64 = 0.0;
  float g32 = 0.0f;
  for (int n = 0; n < nn; ++n) {
    g64 = 0.0;
    g32 = 0.0f;
    if (threads <= 1) {
      for (int i = 1; i < imax - 1; i++) g64 += stencil_plane(F, i, jmax, kmax, omega, &g32);
      for (int i = 1; i < imax - 1; i++) copy_plane(F, i, jmax, kmax);
    } else {
#ifdef _OPENMP
      double acc = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : acc) num_threads(threads)
      for (int i = 1; i < imax - 1; i++) acc += stencil_plane(F, i, jmax, kmax, omega, NULL);
#pragma omp parallel for schedule(static) num_threads(threads)
      for (int i = 1; i < imax - 1; i++) copy_plane(F, i, jmax, kmax);
      g64 = acc;
      g32 = (float)acc; /* no literal sequential fp32 sum in the threaded variant */
#endif
    }
  }
  if (gosa64) *gosa64 = g64;
  if (gosa32) *gosa32 = g32;
}

/* ---------------------------------------------------------------- C API */

int oracle_abi(void) { return 1; }

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Whole program (initmt + jacobi(nn)) on caller-provided arrays.
 * fields: NF pointers to I*J*K floats (the program's static arrays; wrk2 is
 * used as is -- zero for a fresh program).  Results are left in the arrays. */
int oracle_run(int I, int J, int K, int nn, float* const* fields, double* gosa64, float* gosa32) {
  if (I < 4 || J < 4 || K < 4 || nn < 0 || !fields) return -1;
  fields_t F;
  F.I = I; F.J = J; F.K = K;
  for (int f = 0; f < NF; f++) {
    if (!fields[f]) return -1;
    F.f[f] = fields[f];
  }
  initmt(&F);
  jacobi(&F, nn, gosa64, gosa32, 1);
  return 0;
}

/* initmt only (loops 0-5). */
int oracle_initmt(int I, int J, int K, float* const* fields) {
  if (I < 4 || J < 4 || K < 4 || !fields) return -1;
  fields_t F;
  F.I = I; F.J = J; F.K = K;
  for (int f = 0; f < NF; f++) F.f[f] = fields[f];
  initmt(&F);
  return 0;
}

/* initmt with the planes first touched by the OpenMP threads that compute them
 * in oracle_jacobi (same static schedule over i): the arrays' pages land on the
 * NUMA node of their thread (for the multi-threaded CPU baseline).  Same values
 * as initmt. */
int oracle_initmt_par(int I, int J, int K, float* const* fields, int threads) {
  if (I < 4 || J < 4 || K < 4 || !fields) return -1;
  fields_t F;
  F.I = I; F.J = J; F.K = K;
  for (int f = 0; f < NF; f++) F.f[f] = fields[f];
  if (threads <= 1) {
    initmt(&F);
    return 0;
  }
#ifdef _OPENMP
  const int imax = I - 1, jmax = J - 1, kmax = K - 1;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int i = 0; i < I; i++) {
    for (int j = 0; j < J; j++)
      for (int k = 0; k < K; k++) {
        size_t c = at(&F, i, j, k);
        for (int f = 0; f < NF; f++) F.f[f][c] = 0.0f;   /* wrk2 too: first touch */
      }
    if (i < imax)
      for (int j = 0; j < jmax; j++)
        for (int k = 0; k < kmax; k++) {
          size_t c = at(&F, i, j, k);
          F.f[F_A0][c] = 1.0f;
          F.f[F_A1][c] = 1.0f;
          F.f[F_A2][c] = 1.0f;
          F.f[F_A3][c] = (float)(1.0 / 6.0);
          F.f[F_C0][c] = 1.0f;
          F.f[F_C1][c] = 1.0f;
          F.f[F_C2][c] = 1.0f;
          F.f[F_P][c] = (float)(i * i) / (float)((imax - 1) * (imax - 1));
          F.f[F_BND][c] = 1.0f;
        }
  }
#else
  initmt(&F);
#endif
  return 0;
}

/* jacobi(nn) only, on the given state; threads > 1 uses OpenMP over i planes
 * (fp64 gosa only; p/wrk2 identical to the sequential run). */
int oracle_jacobi(int I, int J, int K, int nn, float* const* fields, int threads,
                  double* gosa64, float* gosa32) {
  if (I < 4 || J < 4 || K < 4 || nn < 0 || !fields) return -1;
  fields_t F;
  F.I = I; F.J = J; F.K = K;
  for (int f = 0; f < NF; f++) F.f[f] = fields[f];
  jacobi(&F, nn, gosa64, gosa32, threads);
  return 0;
}
