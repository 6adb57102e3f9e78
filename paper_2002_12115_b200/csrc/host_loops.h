// Host versions of the Himeno loop nests (genes = 0), two builds of the same
// arithmetic: host_tuned (host_loops_tuned.cpp, the library's flags) and host_ref
// (host_loops_ref.cpp, the reference's compile template `gcc -O2`, the program's
// literal loops).  Both round every product and sum separately and sum the stencil's
// ss*ss terms in program order: identical values, different speed.
#pragma once
#include "hp_internal.h"

namespace hp {
namespace host_tuned {
void init0(const HostFields& H, const Box& b);
void init1(const HostFields& H, const Box& b, int imax);
// returns the fp64 sum of the box's ss*ss terms; *lit32 continues the program's
// literal fp32 sequential sum over the same terms
double stencil(const HostFields& H, const Box& b, float omega, float* lit32);
void copy(const HostFields& H, const Box& b);
}  // namespace host_tuned
namespace host_ref {
void init0(const HostFields& H, const Box& b);
void init1(const HostFields& H, const Box& b, int imax);
double stencil(const HostFields& H, const Box& b, float omega, float* lit32);
void copy(const HostFields& H, const Box& b);
}  // namespace host_ref
}  // namespace hp
