// glibc-compatible log1p, shared by the device RNG (rng.cu) and the host
// check that compiles this same file with gcc (tests/test_host.py).
#pragma once
#ifdef __CUDACC__
#include <math_constants.h>
#define LRZ_L1P_FN __device__ __forceinline__
#define L1P_MUL __dmul_rn
#define L1P_ADD __dadd_rn
#define L1P_SUB __dsub_rn
#define L1P_DIV __ddiv_rn
#define L1P_FMA __fma_rn
#define L1P_HI(v) __double2hiint(v)
#define L1P_SETHI(v, h) __hiloint2double((h), __double2loint(v))
#define L1P_INF CUDART_INF
#define L1P_NAN CUDART_NAN
#else  // host twin: compile with -ffp-contract=off
#include <math.h>
#include <stdint.h>
#include <string.h>
#define LRZ_L1P_FN static inline
static inline double L1P_MUL(double a, double b) { return a * b; }
static inline double L1P_ADD(double a, double b) { return a + b; }
static inline double L1P_SUB(double a, double b) { return a - b; }
static inline double L1P_DIV(double a, double b) { return a / b; }
static inline double L1P_FMA(double a, double b, double c) { return fma(a, b, c); }
static inline int L1P_HI(double v) { uint64_t b; memcpy(&b, &v, 8); return (int)(b >> 32); }
static inline double L1P_SETHI(double v, int h) {
  uint64_t b; memcpy(&b, &v, 8);
  b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
  memcpy(&v, &b, 8); return v;
}
#define L1P_INF INFINITY
#define L1P_NAN NAN
#endif

// log1p bit-identical to the one numpy's ziggurat tail calls (npy_log1p ->
// libm log1p; distributions.c random_standard_normal).  That is glibc's
// fdlibm-derived s_log1p (Estrin-grouped polynomial) in its x86_64 FMA ifunc
// variant, so the fused multiply-adds below are exactly the ones that build
// contracts and every other operation is a separately rounded IEEE op
// (explicit _rn intrinsics: nvcc must not contract them).  Checked against
// the host libm on 5e7 arguments in every branch (0 mismatches,
// tests/test_host.py::test_device_log1p_restatement_matches_libm runs the C
// twin of this function).  Only x in (-1, 0] reaches it here.
LRZ_L1P_FN double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int hx = (int)L1P_HI(x), ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -L1P_INF : L1P_NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return L1P_FMA(-L1P_MUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) { k = 0; f = x; hu = 1; }
  } else if (hx >= 0x7ff00000) {
    return L1P_ADD(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = L1P_ADD(1.0, x);
      hu = L1P_HI(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? L1P_SUB(1.0, L1P_SUB(u, x)) : L1P_SUB(x, L1P_SUB(u, 1.0));
      c = L1P_DIV(c, u);
    } else {
      u = x;
      hu = L1P_HI(u);
      k = (hu >> 20) - 1023;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = L1P_SETHI(u, hu | 0x3ff00000);
    } else {
      ++k;
      u = L1P_SETHI(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = L1P_SUB(u, 1.0);
  }
  const double hfsq = L1P_MUL(L1P_MUL(0.5, f), f), dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : L1P_FMA(dk, ln2_hi, L1P_FMA(dk, ln2_lo, c));
    const double R = L1P_MUL(L1P_FMA(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return L1P_SUB(f, R);
    return L1P_FMA(dk, ln2_hi, -L1P_SUB(L1P_SUB(R, L1P_FMA(dk, ln2_lo, c)), f));
  }
  const double s = L1P_DIV(f, L1P_ADD(2.0, f)), z = L1P_MUL(s, s);
  const double R2 = L1P_FMA(z, Lp3, Lp2), R3 = L1P_FMA(z, Lp5, Lp4), R4 = L1P_FMA(z, Lp7, Lp6);
  const double z2 = L1P_MUL(z, z), z4 = L1P_MUL(z2, z2), z6 = L1P_MUL(z4, z2);
  const double R = L1P_FMA(z6, R4, L1P_FMA(z4, R3, L1P_FMA(z, Lp1, L1P_MUL(R2, z2))));
  const double q = L1P_MUL(L1P_ADD(hfsq, R), s);
  if (k == 0) return L1P_SUB(f, L1P_SUB(hfsq, q));
  return L1P_FMA(dk, ln2_hi,
                  -L1P_SUB(L1P_SUB(hfsq, L1P_ADD(L1P_FMA(dk, ln2_lo, c), q)), f));
}

