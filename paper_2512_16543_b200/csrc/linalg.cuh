// CTA-cooperative small dense linear algebra in complex128 (K <= 256):
// Gauss-Jordan inversion (HPD without pivoting, general with partial row
// pivoting), 2-norm estimation by power iteration, the Hermitian inverse
// with the reference's condition guard, and the rank-r Woodbury update.
// All reductions use fixed orders (deterministic).
#pragma once

#include "common.cuh"

namespace lrz {

// In-place Gauss-Jordan inverse of the K x K matrix M (leading dim ld,
// shared or global memory).  Returns 0 ok, 1 non-positive pivot (only in
// the unpivoted HPD mode), 2 zero / non-finite pivot.  colbuf/rowbuf: K
// entries of scratch (shared), perm: K ints (shared), red: >= 2*NW doubles,
// ired: >= NW ints.  The return value is block-uniform.
LRZ_DEV int cta_gauss_jordan(c128 *M, int K, int ld, bool pivot, c128 *colbuf, c128 *rowbuf,
                             int *perm, double *red, int *ired) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, w = tid >> 5, nw = NT >> 5;
  for (int k = 0; k < K; ++k) {
    if (pivot) {
      double best = -1.0;
      int bi = K;
      for (int i = k + tid; i < K; i += NT) {
        const double v = cabs2(M[int64_t(i) * ld + k]);
        if (v > best) {  // strict: keeps the smallest index on ties
          best = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      __syncthreads();
      if (lane == 0) {
        red[w] = best;
        ired[w] = bi;
      }
      __syncthreads();
      best = -1.0;
      bi = K;
      for (int i = 0; i < nw; ++i)
        if (red[i] > best || (red[i] == best && ired[i] < bi)) {
          best = red[i];
          bi = ired[i];
        }
      if (!(best > 0.0) || bi >= K) return 2;
      if (bi != k) {
        for (int j = tid; j < K; j += NT) {
          const c128 t = M[int64_t(k) * ld + j];
          M[int64_t(k) * ld + j] = M[int64_t(bi) * ld + j];
          M[int64_t(bi) * ld + j] = t;
        }
      }
      if (tid == 0) perm[k] = bi;
      __syncthreads();
    }
    const c128 piv = M[int64_t(k) * ld + k];
    if (!pivot && !(piv.re > 0.0)) return 1;
    if (!(isfinite(piv.re) && isfinite(piv.im)) || (piv.re == 0.0 && piv.im == 0.0)) return 2;
    const c128 pinv = cinv(piv);
    for (int i = tid; i < K; i += NT) {
      colbuf[i] = M[int64_t(i) * ld + k];
      rowbuf[i] = cmul(M[int64_t(k) * ld + i], pinv);
    }
    __syncthreads();
    // thread -> column j (tpc threads per column, interleaved rows): the
    // pivot-row factor stays in a register, column factors are broadcasts
    const int tpc = max(1, NT / K);
    for (int jt = tid; jt < K * tpc; jt += NT) {
      const int j = jt % K, i0 = jt / K;
      const c128 r = rowbuf[j];
      for (int i = i0; i < K; i += tpc) {
        c128 &m = M[int64_t(i) * ld + j];
        if (i == k) {
          m = (j == k) ? pinv : r;
        } else if (j == k) {
          m = cmul(mk<double>(-colbuf[i].re, -colbuf[i].im), pinv);
        } else {
          const c128 c = colbuf[i];
          m.re = fma(-c.re, r.re, m.re);
          m.re = fma(c.im, r.im, m.re);
          m.im = fma(-c.re, r.im, m.im);
          m.im = fma(-c.im, r.re, m.im);
        }
      }
    }
    __syncthreads();
  }
  if (pivot) {
    for (int k = K - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k) {
        for (int i = tid; i < K; i += NT) {
          const c128 t = M[int64_t(i) * ld + k];
          M[int64_t(i) * ld + k] = M[int64_t(i) * ld + p];
          M[int64_t(i) * ld + p] = t;
        }
      }
      __syncthreads();
    }
  }
  return 0;
}

LRZ_DEV double cta_fro2(const c128 *M, int K, int ld, double *red) {
  double s = 0.0;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, j = e - i * K;
    s += cabs2(M[int64_t(i) * ld + j]);
  }
  return block_sum(s, red);
}

// sigma_max(X) by power iteration on X^H X from a fixed start vector.
// v, w: K entries of scratch.
LRZ_DEV double cta_sigma_max(const c128 *X, int K, int ld, c128 *v, c128 *w, double *red,
                             int iters) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int i = tid; i < K; i += NT) v[i] = mk<double>(1.0 + 0.01 * i, 0.001 * i);
  __syncthreads();
  double lam = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (int i = tid; i < K; i += NT) {
      c128 a = czero<double>();
      for (int j = 0; j < K; ++j) cfma(a, X[int64_t(i) * ld + j], v[j]);
      w[i] = a;
    }
    __syncthreads();
    double loc = 0.0;
    for (int j = tid; j < K; j += NT) {
      c128 a = czero<double>();
      for (int i = 0; i < K; ++i) cfma_ca(a, X[int64_t(i) * ld + j], w[i]);
      v[j] = a;
      loc += cabs2(a);
    }
    const double n2 = block_sum(loc, red);  // ||X^H X v||^2 with ||v|| = 1 before
    const double nrm = sqrt(n2);
    if (!(nrm > 0.0) || !isfinite(nrm)) return nrm;
    lam = nrm;
    for (int j = tid; j < K; j += NT) v[j] = cscale(v[j], 1.0 / nrm);
    __syncthreads();
  }
  return sqrt(lam);
}

// Condition guard shared by direct_inverse (1e14) and the Woodbury aux (1e12):
// ||X||_F ||X^-1||_F bounds cond_2 from above; only when that bound exceeds
// the limit is cond_2 estimated by power iteration (lowrank.py:135,212).
LRZ_DEV bool cta_cond_ok(const c128 *X, const c128 *Xinv, int K, int ldx, int ldi, double fx,
                         double fi, double limit, c128 *v, c128 *w, double *red) {
  const double fb = sqrt(fx) * sqrt(fi);
  if (fb <= limit) return true;
  if (!isfinite(fx) || !isfinite(fi)) return false;
  const double s1 = cta_sigma_max(X, K, ldx, v, w, red, 60);
  const double s2 = cta_sigma_max(Xinv, K, ldi, v, w, red, 60);
  const double c = s1 * s2;
  return c <= limit;
}

// Shared-memory scratch for the inverse (beyond the matrix itself).
struct InvScratch {
  c128 *colbuf, *rowbuf, *v, *w;
  int *perm, *ired;
  double *red;
};

// Hermitian inverse with the reference's guard (lowrank.py:127-144):
// Ain (global, K x K, row-major) -> Aout (global).  If M is non-null it is
// a K*K shared buffer used for the factorisation (K <= 64), otherwise the
// factorisation runs in place in Aout.  Returns LRZ_INFO_*.
LRZ_DEV int cta_herm_inverse(const c128 *Ain, c128 *Aout, int K, c128 *M, double limit,
                             const InvScratch &sc) {
  const int tid = threadIdx.x, NT = blockDim.x;
  c128 *W = M ? M : Aout;
  double loc = 0.0;
  for (int e = tid; e < K * K; e += NT) {
    const c128 a = Ain[e];
    W[e] = a;
    loc += cabs2(a);
  }
  const double fa = block_sum(loc, sc.red);  // also a barrier
  int st = cta_gauss_jordan(W, K, K, false, sc.colbuf, sc.rowbuf, sc.perm, sc.red, sc.ired);
  bool indefinite = false;
  if (st == 1) {  // Hermitian but not PD: pivoted path (scipy solve assume_a='her')
    indefinite = true;
    for (int e = tid; e < K * K; e += NT) W[e] = Ain[e];
    __syncthreads();
    st = cta_gauss_jordan(W, K, K, true, sc.colbuf, sc.rowbuf, sc.perm, sc.red, sc.ired);
  }
  int info = LRZ_INFO_OK;
  if (st != 0) {
    info = LRZ_INFO_SINGULAR;
  } else {
    const double fi = cta_fro2(W, K, K, sc.red);
    if (!cta_cond_ok(Ain, W, K, K, K, fa, fi, limit, sc.v, sc.w, sc.red))
      info = LRZ_INFO_SINGULAR;
    else if (indefinite)
      info = LRZ_INFO_INDEFINITE;
  }
  if (M) {
    __syncthreads();
    for (int e = tid; e < K * K; e += NT) Aout[e] = M[e];
  }
  __syncthreads();
  return info;
}

// Woodbury scratch: aux/auxinv r x r in shared memory; AiU, T (K x r col-major)
// and VhAi (r x K row-major) in global workspace.
struct WbScratch {
  c128 *aux, *auxinv;          // shared, r_max^2 each
  c128 *AiU, *T, *VhAi;        // global, K * r_max each
  InvScratch inv;              // colbuf/rowbuf/perm sized r_max, v/w sized r_max
};

// One Woodbury step (lowrank.py:208-220).  Ainv_in, Ainv_out, A_in, A_out
// row-major K x K (Ainv_out != Ainv_in; A_out may alias A_in);
// U, V column-major [j][K]; S descending.  Returns LRZ_INFO_OK or
// LRZ_INFO_SINGULAR_AUX (nothing written).  `ld` is the row stride of
// A^-1 and the column stride of U, V and the K-long scratch columns (K in
// global memory; K + 1 when they sit in shared memory, which spreads the
// K-strided accesses over the banks); A itself is K-strided.
LRZ_DEV int cta_woodbury(int K, int r, const c128 *__restrict__ Ainv_in, c128 *Ainv_out,
                         const c128 *A_in, c128 *A_out, const c128 *__restrict__ U,
                         const c128 *__restrict__ V, const double *__restrict__ S,
                         const WbScratch &sc, int ld = 0) {
  if (ld == 0) ld = K;
  const int tid = threadIdx.x, NT = blockDim.x;
  // 1. AiU = A^-1 U (K x r) and VhAi = V^H A^-1 (r x K)
  for (int e = tid; e < K * r; e += NT) {
    const int j = e / K, k = e - j * K;
    c128 a = czero<double>();
    const c128 *arow = Ainv_in + int64_t(k) * ld;
    const c128 *uc = U + int64_t(j) * ld;
    for (int m = 0; m < K; ++m) cfma(a, arow[m], uc[m]);
    sc.AiU[int64_t(j) * ld + k] = a;
  }
  for (int e = tid; e < K * r; e += NT) {
    const int j = e / K, m = e - j * K;
    c128 a = czero<double>();
    const c128 *vc = V + int64_t(j) * ld;
    for (int k = 0; k < K; ++k) cfma_ca(a, vc[k], Ainv_in[int64_t(k) * ld + m]);
    sc.VhAi[int64_t(j) * ld + m] = a;
  }
  __syncthreads();
  // 2. aux = diag(1/S) + V^H AiU
  double loc = 0.0;
  for (int e = tid; e < r * r; e += NT) {
    const int i = e / r, j = e - i * r;
    c128 a = czero<double>();
    const c128 *vc = V + int64_t(i) * ld;
    const c128 *au = sc.AiU + int64_t(j) * ld;
    for (int k = 0; k < K; ++k) cfma_ca(a, vc[k], au[k]);
    if (i == j) a.re = 1.0 / S[i] + a.re;
    sc.aux[e] = a;
    sc.auxinv[e] = a;
    loc += cabs2(a);
  }
  const double fa = block_sum(loc, sc.inv.red);
  // 3. aux^-1 with the 1e12 condition guard (lowrank.py:212-217)
  int st = cta_gauss_jordan(sc.auxinv, r, r, true, sc.inv.colbuf, sc.inv.rowbuf, sc.inv.perm,
                            sc.inv.red, sc.inv.ired);
  if (st != 0) return LRZ_INFO_SINGULAR_AUX;
  const double fi = cta_fro2(sc.auxinv, r, r, sc.inv.red);
  if (!cta_cond_ok(sc.aux, sc.auxinv, r, r, r, fa, fi, 1e12, sc.inv.v, sc.inv.w, sc.inv.red))
    return LRZ_INFO_SINGULAR_AUX;
  // 4. T = AiU aux^-1 (K x r)
  for (int e = tid; e < K * r; e += NT) {
    const int j = e / K, k = e - j * K;
    c128 a = czero<double>();
    for (int i = 0; i < r; ++i) cfma(a, sc.AiU[int64_t(i) * ld + k], sc.auxinv[i * r + j]);
    sc.T[int64_t(j) * ld + k] = a;
  }
  __syncthreads();
  // 5. A^-1 - T VhAi ;  A + (U S) V^H
  for (int e = tid; e < K * K; e += NT) {
    const int k = e / K, m = e - k * K;
    c128 a = czero<double>();
    for (int j = 0; j < r; ++j) cfma(a, sc.T[int64_t(j) * ld + k], sc.VhAi[int64_t(j) * ld + m]);
    const c128 o = Ainv_in[int64_t(k) * ld + m];
    Ainv_out[int64_t(k) * ld + m] = mk<double>(o.re - a.re, o.im - a.im);
    if (A_out) {
      c128 b = czero<double>();
      for (int j = 0; j < r; ++j)
        cfma_cb(b, cscale(U[int64_t(j) * ld + k], S[j]), V[int64_t(j) * ld + m]);
      const c128 x = A_in[e];
      A_out[e] = mk<double>(x.re + b.re, x.im + b.im);
    }
  }
  __syncthreads();
  return LRZ_INFO_OK;
}

}  // namespace lrz
