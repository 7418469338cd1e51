// Shared device helpers for the leorzf_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/leorzf_b200.h"
#include "prof.cuh"

#define LRZ_DEV __device__ __forceinline__

namespace lrz {

constexpr double EPS64 = 2.220446049250313e-16;  // np.finfo(float).eps

// Interleaved complex with 2*sizeof(T) alignment so loads are one LDG.64/128.
template <typename T>
struct __align__(2 * sizeof(T)) cplx {
  T re, im;
};
using c64 = cplx<float>;
using c128 = cplx<double>;

template <typename T>
LRZ_DEV cplx<T> mk(T re, T im) {
  cplx<T> z;
  z.re = re;
  z.im = im;
  return z;
}
template <typename T>
LRZ_DEV cplx<T> czero() {
  return mk<T>(T(0), T(0));
}
template <typename To, typename Ti>
LRZ_DEV cplx<To> ccast(cplx<Ti> a) {
  return mk<To>(To(a.re), To(a.im));
}
template <typename T>
LRZ_DEV cplx<T> cadd(cplx<T> a, cplx<T> b) {
  return mk<T>(a.re + b.re, a.im + b.im);
}
template <typename T>
LRZ_DEV cplx<T> csub(cplx<T> a, cplx<T> b) {
  return mk<T>(a.re - b.re, a.im - b.im);
}
template <typename T>
LRZ_DEV cplx<T> cconj(cplx<T> a) {
  return mk<T>(a.re, -a.im);
}
template <typename T>
LRZ_DEV cplx<T> cscale(cplx<T> a, T s) {
  return mk<T>(a.re * s, a.im * s);
}
template <typename T>
LRZ_DEV cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return mk<T>(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
// acc += a * b
template <typename T>
LRZ_DEV void cfma(cplx<T> &acc, cplx<T> a, cplx<T> b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
}
// acc += a * conj(b)
template <typename T>
LRZ_DEV void cfma_cb(cplx<T> &acc, cplx<T> a, cplx<T> b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(a.im, b.im, acc.re);
  acc.im = fma(a.im, b.re, acc.im);
  acc.im = fma(-a.re, b.im, acc.im);
}
// acc += conj(a) * b
template <typename T>
LRZ_DEV void cfma_ca(cplx<T> &acc, cplx<T> a, cplx<T> b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(-a.im, b.re, acc.im);
}
template <typename T>
LRZ_DEV T cabs2(cplx<T> a) {
  return a.re * a.re + a.im * a.im;
}
LRZ_DEV c128 cdiv(c128 a, c128 b) {
  // Smith's algorithm
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, den = b.re + b.im * r;
    return mk<double>((a.re + a.im * r) / den, (a.im - a.re * r) / den);
  } else {
    double r = b.re / b.im, den = b.re * r + b.im;
    return mk<double>((a.re * r + a.im) / den, (a.im * r - a.re) / den);
  }
}
LRZ_DEV c128 cinv(c128 b) { return cdiv(mk<double>(1.0, 0.0), b); }

template <typename T>
LRZ_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
LRZ_DEV T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block sum: fixed warp partial order.  `red` must hold
// blockDim.x/32 doubles.  All threads get the result.  Contains 2 barriers.
LRZ_DEV double block_sum(double v, double *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

LRZ_DEV bool finite(double x) { return isfinite(x); }

}  // namespace lrz

// host-side error helper (defined in capi.cu)
void lrz_set_error(const char *fmt, ...);
int lrz_launch_status(const char *what);
