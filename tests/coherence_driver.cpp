// CPU unit driver for csrc/coherence.h (compiled by tests/test_coherence.py).
#include <cstdio>
#include <cstdlib>

#include "coherence.h"

using hp::Box;
using hp::Coherence;

static long long vol(const std::vector<Box>& v) {
  long long n = 0;
  for (const Box& b : v) n += b.count();
  return n;
}
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                               \
    }                                                         \
  } while (0)

int main() {
  const Box full{0, 10, 0, 10, 0, 20}, init{0, 9, 0, 9, 0, 19}, in{1, 8, 1, 8, 1, 18};
  // subtraction: pieces are disjoint and cover a \ b
  {
    std::vector<Box> out;
    hp::box_subtract(full, in, out);
    CHECK(vol(out) == full.count() - in.count());
    for (size_t i = 0; i < out.size(); ++i)
      for (size_t j = i + 1; j < out.size(); ++j) CHECK(!hp::box_meets(out[i], out[j]));
    out.clear();
    hp::box_subtract(in, full, out);
    CHECK(out.empty());
  }
  // fresh program: host owns everything, device stale everywhere
  Coherence c;
  c.reset(full);
  CHECK(vol(c.region(hp::OWN_HOST)) == full.count());
  CHECK(c.region(hp::OWN_DEV).empty());
  CHECK(c.newer_in(hp::OWN_HOST, in));
  // 0010000000001: init0 rows on device, init1 on host, copy interior on device
  c.write(full, hp::OWN_DEV);            // device zeroes everything
  CHECK(c.log.size() == 1);              // host entry pruned
  c.mark_synced(hp::OWN_DEV);            // update self after loop 0
  c.write(init, hp::OWN_HOST);           // host coefficients / p
  c.write(in, hp::OWN_DEV);              // device copy nest writes the interior
  const std::vector<Box> dev = c.region(hp::OWN_DEV);
  CHECK(vol(dev) == in.count());         // only the interior is device-newer
  // a guarded update self copies everything but the host-newer shell init \ interior
  CHECK(vol(c.region_excluding(hp::OWN_HOST, full)) == full.count() - (init.count() - in.count()));
  const std::vector<Box> host = c.region(hp::OWN_HOST);
  CHECK(vol(host) == init.count() - in.count());   // shell init \ interior is host-newer
  CHECK(c.newer_in(hp::OWN_HOST, hp::grow(in, 1)));  // stencil on device would read stale p
  CHECK(!c.newer_in(hp::OWN_HOST, Box{3, 4, 3, 4, 3, 4}));
  c.mark_synced(hp::OWN_DEV);
  CHECK(c.region(hp::OWN_DEV).empty());
  // after a deallocation the device is undefined: an update device copies everything
  c.reset(full);
  CHECK(vol(c.region_excluding(hp::OWN_DEV, full)) == full.count());
  CHECK(c.region_excluding(hp::OWN_HOST, full).empty());   // nothing defined to copy back
  // a full host write prunes everything
  c.write(full, hp::OWN_HOST);
  CHECK(c.log.size() == 1 && vol(c.region(hp::OWN_HOST)) == full.count());
  c.all_synced(full);
  CHECK(c.region(hp::OWN_HOST).empty() && c.region(hp::OWN_DEV).empty());
  // row-by-row writes (row kernels under host loops) coalesce into one slab
  {
    Coherence r;
    r.reset(full);
    for (int i = in.i0; i < in.i1; ++i)
      for (int j = in.j0; j < in.j1; ++j) {
        r.write(Box{i, i + 1, j, j + 1, in.k0, in.k1}, hp::OWN_DEV);
        CHECK(r.log.size() <= 3);
      }
    CHECK(vol(r.region(hp::OWN_DEV)) == in.count());
    CHECK(vol(r.region(hp::OWN_HOST)) == full.count() - in.count());
  }
  // randomized: newer_in agrees with the explicit region (point test over the box)
  {
    unsigned seed = 12345;
    auto rnd = [&](int n) { seed = seed * 1103515245u + 12345u; return (int)((seed >> 8) % (unsigned)n); };
    const Box g{0, 6, 0, 5, 0, 7};
    for (int trial = 0; trial < 300; ++trial) {
      Coherence r;
      r.reset(g);
      const int nw = 1 + rnd(6);
      for (int w = 0; w < nw; ++w) {
        const int i0 = rnd(6), j0 = rnd(5), k0 = rnd(7);
        const Box b{i0, i0 + 1 + rnd(6 - i0), j0, j0 + 1 + rnd(5 - j0), k0, k0 + 1 + rnd(7 - k0)};
        r.write(b, rnd(3));
        if (rnd(4) == 0) r.mark_synced(rnd(2));
      }
      for (int q = 0; q < 10; ++q) {
        const int i0 = rnd(6), j0 = rnd(5), k0 = rnd(7);
        const Box b{i0, i0 + 1 + rnd(6 - i0), j0, j0 + 1 + rnd(5 - j0), k0, k0 + 1 + rnd(7 - k0)};
        for (int owner = 0; owner < 3; ++owner) {
          bool want = false;
          for (const Box& x : r.region(owner)) want = want || hp::box_meets(x, b);
          CHECK(r.newer_in(owner, b) == want);
        }
      }
    }
  }
  std::printf("OK\n");
  return 0;
}
