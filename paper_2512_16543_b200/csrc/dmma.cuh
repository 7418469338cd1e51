// FP64 tensor-pipe helpers (DMMA, mma.sync m8n8k4 f64).  Fragment layout
// (PTX ISA): lane L = 4 g + t holds A[g][t], B[t][g] (one double each) and
// C[g][2t], C[g][2t + 1].  A complex MAC block is four real DMMAs on the
// (re, im) halves of the same fragments.
#pragma once

#include "common.cuh"

namespace lrz {

LRZ_DEV void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

LRZ_DEV c128 ldg_c(const c128 *p) {
  const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
  return mk<double>(v.x, v.y);
}
LRZ_DEV c128 ldg_c(const c64 *p) {  // complex64 widened to complex128 on load
  const float2 v = __ldg(reinterpret_cast<const float2 *>(p));
  return mk<double>(double(v.x), double(v.y));
}

}  // namespace lrz
