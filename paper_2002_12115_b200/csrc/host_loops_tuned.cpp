// Host loop bodies, tuned build (g++ -O3 -march=x86-64-v3 -ffp-contract=off, like the
// rest of the library): row-wise with restrict-qualified pointers so the k loops
// vectorise; every product and sum rounds separately (no FMA contraction), so values
// equal the kernels' and the oracle's bit for bit.  HP_FLAG_HOST_REFERENCE runs the
// reference-faithful build instead (host_loops_ref.cpp).
#include <cstring>
#include <vector>

#include "host_loops.h"

namespace hp {
namespace host_tuned {
// Same expression order as the C program; built with -ffp-contract=off so
// every product and sum rounds separately, exactly like the kernels.

// Row-wise: per (i, j) row each field is filled / computed over the k range with
// restrict-qualified pointers, so the inner loops vectorise; values and their
// order of rounding are those of the program's statements.
void init0(const HostFields& H, const Box& b) {
  if (b.k1 <= b.k0) return;
  const size_t n = (size_t)(b.k1 - b.k0) * sizeof(float);
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j) {
      const size_t c = H.at(i, j, b.k0);
      for (int f = 0; f < HP_NFIELDS; ++f)
        if (f != HP_F_WRK2) memset(H.f[f] + c, 0, n);
    }
}

static inline void fill_row(float* __restrict__ d, int n, float v) {
  for (int k = 0; k < n; ++k) d[k] = v;
}

void init1(const HostFields& H, const Box& b, int imax) {
  const float a3 = (float)(1.0 / 6.0);
  const int n = b.k1 - b.k0;
  if (n <= 0) return;
  for (int i = b.i0; i < b.i1; ++i) {
    const float pv = (float)(i * i) / (float)((imax - 1) * (imax - 1));
    for (int j = b.j0; j < b.j1; ++j) {
      const size_t c = H.at(i, j, b.k0);
      fill_row(H.f[HP_F_A0] + c, n, 1.0f);
      fill_row(H.f[HP_F_A1] + c, n, 1.0f);
      fill_row(H.f[HP_F_A2] + c, n, 1.0f);
      fill_row(H.f[HP_F_A3] + c, n, a3);
      fill_row(H.f[HP_F_B0] + c, n, 0.0f);
      fill_row(H.f[HP_F_B1] + c, n, 0.0f);
      fill_row(H.f[HP_F_B2] + c, n, 0.0f);
      fill_row(H.f[HP_F_C0] + c, n, 1.0f);
      fill_row(H.f[HP_F_C1] + c, n, 1.0f);
      fill_row(H.f[HP_F_C2] + c, n, 1.0f);
      fill_row(H.f[HP_F_P] + c, n, pv);
      fill_row(H.f[HP_F_WRK1] + c, n, 0.0f);
      fill_row(H.f[HP_F_BND] + c, n, 1.0f);
    }
  }
}

// One k row of the stencil: wrk2 and the ss*ss terms (vectorised: no
// reduction in the loop); the caller sums the terms in k order.
static void stencil_row(const float* __restrict__ p, const float* __restrict__ a0,
                             const float* __restrict__ a1, const float* __restrict__ a2,
                             const float* __restrict__ a3, const float* __restrict__ b0,
                             const float* __restrict__ b1, const float* __restrict__ b2,
                             const float* __restrict__ c0, const float* __restrict__ c1,
                             const float* __restrict__ c2, const float* __restrict__ wrk1,
                             const float* __restrict__ bnd, float* __restrict__ wrk2,
                             float* __restrict__ t, int n, size_t R, size_t L, float omega) {
  for (int k = 0; k < n; ++k) {
    const float s0 = a0[k] * p[k + L] + a1[k] * p[k + R] + a2[k] * p[k + 1] +
                     b0[k] * (p[k + L + R] - p[k + L - R] - p[k - L + R] + p[k - L - R]) +
                     b1[k] * (p[k + R + 1] - p[k - R + 1] - p[k + R - 1] + p[k - R - 1]) +
                     b2[k] * (p[k + L + 1] - p[k - L + 1] - p[k + L - 1] + p[k - L - 1]) +
                     c0[k] * p[k - L] + c1[k] * p[k - R] + c2[k] * p[k - 1] + wrk1[k];
    const float ss = (s0 * a3[k] - p[k]) * bnd[k];
    t[k] = ss * ss;
    wrk2[k] = p[k] + omega * ss;
  }
}

// Returns the fp64 sum of the box's ss*ss terms; *lit32 continues the program's
// literal fp32 sequential sum (`gosa += ss*ss` with float gosa) over the same terms.
double stencil(const HostFields& H, const Box& b, float omega, float* lit32) {
  const int n = b.k1 - b.k0;
  if (n <= 0) return 0.0;
  float g32 = *lit32;
  const size_t R = (size_t)H.K, L = (size_t)H.J * H.K;
  std::vector<float> t((size_t)n);
  double acc = 0.0;
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j) {
      const size_t c = H.at(i, j, b.k0);
      // p is read through indices k - L .. k + L + R + 1 of the row base: pass the
      // row base itself (negative offsets stay inside the array for interior rows)
      stencil_row(H.f[HP_F_P] + c, H.f[HP_F_A0] + c, H.f[HP_F_A1] + c, H.f[HP_F_A2] + c,
                       H.f[HP_F_A3] + c, H.f[HP_F_B0] + c, H.f[HP_F_B1] + c, H.f[HP_F_B2] + c,
                       H.f[HP_F_C0] + c, H.f[HP_F_C1] + c, H.f[HP_F_C2] + c,
                       H.f[HP_F_WRK1] + c, H.f[HP_F_BND] + c, H.f[HP_F_WRK2] + c, t.data(), n,
                       R, L, omega);
      for (int k = 0; k < n; ++k) {   // k order, as the program
        acc += (double)t[k];
        g32 += t[k];
      }
    }
  *lit32 = g32;
  return acc;
}

void copy(const HostFields& H, const Box& b) {
  for (int i = b.i0; i < b.i1; ++i)
    for (int j = b.j0; j < b.j1; ++j) {
      const size_t c = H.at(i, j, b.k0);
      if (b.k1 > b.k0)
        memcpy(H.f[HP_F_P] + c, H.f[HP_F_WRK2] + c, (size_t)(b.k1 - b.k0) * sizeof(float));
    }
}

}  // namespace host_tuned
}  // namespace hp
