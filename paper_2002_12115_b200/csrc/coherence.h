#pragma once
#include <algorithm>
#include <vector>

#include "hp_internal.h"

namespace hp {
// Coherence bookkeeping of the device data manager (pure host C++).
//
// A chronological log of write boxes, each tagged with the side that holds the
// latest data there: HOST (host newer), DEV (device newer), BOTH (in sync).
// Entries fully covered by a later write are pruned, so for Himeno's nested
// write boxes (full >= [0,max)^3 >= interior) the log never exceeds a few
// entries.  A guarded transfer copies everything except the region where the
// destination holds newer data (a list of disjoint boxes), then marks the
// source's newer region in sync.  Device memory that was never defined (or was
// deallocated at a data-region exit) is modelled as HOST-owned.
enum Owner { OWN_HOST = 0, OWN_DEV = 1, OWN_BOTH = 2 };

inline bool box_empty(const Box& b) { return b.count() <= 0; }
inline bool box_contains(const Box& o, const Box& in) {
  if (box_empty(in)) return true;
  return o.i0 <= in.i0 && in.i1 <= o.i1 && o.j0 <= in.j0 && in.j1 <= o.j1 && o.k0 <= in.k0 &&
         in.k1 <= o.k1;
}
inline Box box_clip(const Box& a, const Box& b) {
  return Box{std::max(a.i0, b.i0), std::min(a.i1, b.i1), std::max(a.j0, b.j0),
             std::min(a.j1, b.j1), std::max(a.k0, b.k0), std::min(a.k1, b.k1)};
}
inline bool box_meets(const Box& a, const Box& b) { return !box_empty(box_clip(a, b)); }
inline Box grow(const Box& b, int h) { return Box{b.i0 - h, b.i1 + h, b.j0 - h, b.j1 + h, b.k0 - h, b.k1 + h}; }

// a minus b as up to 6 disjoint boxes
inline void box_subtract(const Box& a, const Box& b, std::vector<Box>& out) {
  const Box x = box_clip(a, b);
  if (box_empty(x)) {
    if (!box_empty(a)) out.push_back(a);
    return;
  }
  auto put = [&](const Box& q) { if (!box_empty(q)) out.push_back(q); };
  put(Box{a.i0, x.i0, a.j0, a.j1, a.k0, a.k1});
  put(Box{x.i1, a.i1, a.j0, a.j1, a.k0, a.k1});
  put(Box{x.i0, x.i1, a.j0, x.j0, a.k0, a.k1});
  put(Box{x.i0, x.i1, x.j1, a.j1, a.k0, a.k1});
  put(Box{x.i0, x.i1, x.j0, x.j1, a.k0, x.k0});
  put(Box{x.i0, x.i1, x.j0, x.j1, x.k1, a.k1});
}

// a and b form exactly one box together (one contains the other, or they agree
// on two dimensions and overlap / touch on the third)
inline bool box_union_is_box(const Box& a, const Box& b) {
  if (box_contains(a, b) || box_contains(b, a)) return true;
  const bool si = a.i0 == b.i0 && a.i1 == b.i1, sj = a.j0 == b.j0 && a.j1 == b.j1,
             sk = a.k0 == b.k0 && a.k1 == b.k1;
  if (si && sj) return a.k1 >= b.k0 && b.k1 >= a.k0;
  if (si && sk) return a.j1 >= b.j0 && b.j1 >= a.j0;
  if (sj && sk) return a.i1 >= b.i0 && b.i1 >= a.i0;
  return false;
}
inline Box box_hull(const Box& a, const Box& b) {
  return Box{std::min(a.i0, b.i0), std::max(a.i1, b.i1), std::min(a.j0, b.j0),
             std::max(a.j1, b.j1), std::min(a.k0, b.k0), std::max(a.k1, b.k1)};
}

struct Coherence {
  struct Span { Box box; int owner; };
  std::vector<Span> log;

  void reset(const Box& full) { log.assign(1, Span{full, OWN_HOST}); }
  // Record a write.  Consecutive writes of the same side coalesce while their
  // union is a box (row launches -> planes -> slabs), and entries the write
  // covers are dropped, so the log stays a handful of boxes.
  void write(const Box& b, int owner) {
    if (box_empty(b)) return;
    Box nb = b;
    while (!log.empty() && log.back().owner == owner && box_union_is_box(log.back().box, nb)) {
      nb = box_hull(log.back().box, nb);
      log.pop_back();
    }
    // in place (no allocation: row launches write once per launch)
    log.erase(std::remove_if(log.begin(), log.end(),
                             [&](const Span& e) { return box_contains(nb, e.box); }),
              log.end());
    log.push_back(Span{nb, owner});
  }
  // disjoint boxes whose latest writer is `owner`
  std::vector<Box> region(int owner) const {
    std::vector<Box> out;
    for (size_t n = 0; n < log.size(); ++n) {
      if (log[n].owner != owner) continue;
      std::vector<Box> pieces{log[n].box};
      for (size_t m = n + 1; m < log.size() && !pieces.empty(); ++m) {
        std::vector<Box> next;
        for (const Box& q : pieces) box_subtract(q, log[m].box, next);
        pieces.swap(next);
      }
      out.insert(out.end(), pieces.begin(), pieces.end());
    }
    return out;
  }
  // does any point of b have `owner` as its latest writer?  Checks b's overlap with
  // each `owner` entry minus the later entries, with reused scratch (called for every
  // array at every launch)
  bool newer_in(int owner, const Box& b) const {
    static thread_local std::vector<Box> pieces, next;
    for (size_t n = 0; n < log.size(); ++n) {
      if (log[n].owner != owner) continue;
      const Box x = box_clip(log[n].box, b);
      if (box_empty(x)) continue;
      pieces.assign(1, x);
      for (size_t m = n + 1; m < log.size() && !pieces.empty(); ++m) {
        next.clear();
        for (const Box& q : pieces) box_subtract(q, log[m].box, next);
        pieces.swap(next);
      }
      if (!pieces.empty()) return true;
    }
    return false;
  }
  // points whose latest writer is NOT `owner` (the region a guarded transfer
  // from the other side may copy without clobbering newer data)
  std::vector<Box> region_excluding(int owner, const Box& full) const {
    std::vector<Box> keep{full};
    for (const Box& q : region(owner)) {
      std::vector<Box> next;
      for (const Box& k : keep) box_subtract(k, q, next);
      keep.swap(next);
    }
    return keep;
  }
  void mark_synced(int owner) {
    for (Span& e : log)
      if (e.owner == owner) e.owner = OWN_BOTH;
  }
  void all_synced(const Box& full) { log.assign(1, Span{full, OWN_BOTH}); }
};


}  // namespace hp
