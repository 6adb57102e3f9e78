// Host loop bodies, reference-faithful build: the program's loops as written
// (triple loops, one statement per array element, gosa summed
// inside the k loop), compiled like the reference's compile template (`gcc -O2 -w`,
// evaluators.py:154-165; build.py gives this file -O2 and no -march).  Selected per run
// by HP_FLAG_HOST_REFERENCE, so host-heavy patterns cost what the reference's binary
// would make them cost.  Same values as host_loops_tuned.cpp, bit for bit.
#include "host_loops.h"

namespace hp {
namespace host_ref {

void init0(const HostFields& H, const Box& b) {
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j)
      for (int k = b.k0; k < b.k1; ++k) {
        const size_t c = H.at(i, j, k);
        H.f[HP_F_A0][c] = 0.0f;
        H.f[HP_F_A1][c] = 0.0f;
        H.f[HP_F_A2][c] = 0.0f;
        H.f[HP_F_A3][c] = 0.0f;
        H.f[HP_F_B0][c] = 0.0f;
        H.f[HP_F_B1][c] = 0.0f;
        H.f[HP_F_B2][c] = 0.0f;
        H.f[HP_F_C0][c] = 0.0f;
        H.f[HP_F_C1][c] = 0.0f;
        H.f[HP_F_C2][c] = 0.0f;
        H.f[HP_F_P][c] = 0.0f;
        H.f[HP_F_WRK1][c] = 0.0f;
        H.f[HP_F_BND][c] = 0.0f;
      }
}

void init1(const HostFields& H, const Box& b, int imax) {
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j)
      for (int k = b.k0; k < b.k1; ++k) {
        const size_t c = H.at(i, j, k);
        H.f[HP_F_A0][c] = 1.0f;
        H.f[HP_F_A1][c] = 1.0f;
        H.f[HP_F_A2][c] = 1.0f;
        H.f[HP_F_A3][c] = (float)(1.0 / 6.0);
        H.f[HP_F_B0][c] = 0.0f;
        H.f[HP_F_B1][c] = 0.0f;
        H.f[HP_F_B2][c] = 0.0f;
        H.f[HP_F_C0][c] = 1.0f;
        H.f[HP_F_C1][c] = 1.0f;
        H.f[HP_F_C2][c] = 1.0f;
        H.f[HP_F_P][c] = (float)(i * i) / (float)((imax - 1) * (imax - 1));
        H.f[HP_F_WRK1][c] = 0.0f;
        H.f[HP_F_BND][c] = 1.0f;
      }
}

double stencil(const HostFields& H, const Box& b, float omega, float* lit32) {
  const float* p = H.f[HP_F_P];
  const float *a0 = H.f[HP_F_A0], *a1 = H.f[HP_F_A1], *a2 = H.f[HP_F_A2], *a3 = H.f[HP_F_A3];
  const float *b0 = H.f[HP_F_B0], *b1 = H.f[HP_F_B1], *b2 = H.f[HP_F_B2];
  const float *c0 = H.f[HP_F_C0], *c1 = H.f[HP_F_C1], *c2 = H.f[HP_F_C2];
  const float *wrk1 = H.f[HP_F_WRK1], *bnd = H.f[HP_F_BND];
  float* wrk2 = H.f[HP_F_WRK2];
  const size_t R = (size_t)H.K, L = (size_t)H.J * H.K;
  float g32 = *lit32;
  double acc = 0.0;
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j)
      for (int k = b.k0; k < b.k1; ++k) {
        const size_t c = H.at(i, j, k);
        const float s0 = a0[c] * p[c + L] + a1[c] * p[c + R] + a2[c] * p[c + 1] +
                         b0[c] * (p[c + L + R] - p[c + L - R] - p[c - L + R] + p[c - L - R]) +
                         b1[c] * (p[c + R + 1] - p[c - R + 1] - p[c + R - 1] + p[c - R - 1]) +
                         b2[c] * (p[c + L + 1] - p[c - L + 1] - p[c + L - 1] + p[c - L - 1]) +
                         c0[c] * p[c - L] + c1[c] * p[c - R] + c2[c] * p[c - 1] + wrk1[c];
        const float ss = (s0 * a3[c] - p[c]) * bnd[c];
        const float t = ss * ss;
        g32 += t;                // gosa += ss*ss;  (the program's float gosa)
        acc += (double)t;        // the fp64 sum every other path reports
        wrk2[c] = p[c] + omega * ss;
      }
  *lit32 = g32;
  return acc;
}

void copy(const HostFields& H, const Box& b) {
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j)
      for (int k = b.k0; k < b.k1; ++k) {
        const size_t c = H.at(i, j, k);
        H.f[HP_F_P][c] = H.f[HP_F_WRK2][c];
      }
}

}  // namespace host_ref
}  // namespace hp
