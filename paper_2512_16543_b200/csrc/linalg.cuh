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
// Pivoted Gauss-Jordan for K <= 64 with two CTA barriers per pivot: warp 0 finds
// the pivot (each lane its rows' largest |m|^2, then two integer redux steps on
// the ordered bit pattern and one on the row index -- smallest row on ties, like
// the generic path), swaps the rows, forms the pivot's reciprocal and snapshots
// column k and the scaled row k; the whole CTA then applies the rank-1 update.
// The generic path below spends five barriers and a shared-memory reduction per
// pivot on the search alone (ncu, Woodbury chain: 20 % of the instructions).
LRZ_DEV int cta_gj_pivot_small(c128 *M, int K, int ld, c128 *colbuf, c128 *rowbuf, int *perm,
                               int *ired) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  const int KK = K * K;
  const float inv_k = 1.0f / float(K);
  for (int k = 0; k < K; ++k) {
    if (tid < 32) {
      double mag = 0.0;
      int bi = K;
      for (int i = k + lane; i < K; i += 32) {
        const double v = cabs2(M[int64_t(i) * ld + k]);
        if (v > mag || !(v == v)) {  // strict: keeps the smallest of my rows on ties
          mag = v;
          bi = i;
        }
      }
      const unsigned long long bits =
          (mag == mag) ? (unsigned long long)__double_as_longlong(mag) : 0xFFFFFFFFFFFFFFFFull;
      const unsigned hi = unsigned(bits >> 32), lo = unsigned(bits);
      const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
      const bool cand = bi < K && hi == mh && lo == ml;
      const unsigned row = __reduce_min_sync(0xffffffffu, cand ? unsigned(bi) : 0xFFFFFFFFu);
      int st = 0;
      if (row >= unsigned(K) || (mh == 0u && ml == 0u) || mh >= 0x7FF00000u) st = 2;
      if (st == 0) {
        const int p = int(row);
        if (p != k)
          for (int j = lane; j < K; j += 32) {
            const c128 x = M[int64_t(k) * ld + j];
            M[int64_t(k) * ld + j] = M[int64_t(p) * ld + j];
            M[int64_t(p) * ld + j] = x;
          }
        if (lane == 0) perm[k] = p;
        __syncwarp();
        const c128 piv = M[int64_t(k) * ld + k];
        const double id = 1.0 / cabs2(piv);
        const c128 pinv = mk<double>(piv.re * id, -piv.im * id);
        if (!(isfinite(pinv.re) && isfinite(pinv.im))) st = 2;
        for (int i = lane; i < K; i += 32) {
          colbuf[i] = M[int64_t(i) * ld + k];
          rowbuf[i] = (i == k) ? pinv : cmul(M[int64_t(k) * ld + i], pinv);
        }
      }
      if (lane == 0) ired[0] = st;
    }
    __syncthreads();
    if (ired[0] != 0) return 2;
    const c128 pinv = rowbuf[k];
    for (int e = tid; e < KK; e += NT) {
      const int i = int((float(e) + 0.5f) * inv_k), j = e - i * K;  // exact: e < 4096
      const c128 rj = rowbuf[j];
      c128 m;
      if (i == k) {
        m = rj;
      } else {
        const c128 c = colbuf[i];
        if (j == k) {
          m = cmul(mk<double>(-c.re, -c.im), pinv);
        } else {
          m = M[int64_t(i) * ld + j];
          m.re = fma(-c.re, rj.re, m.re);
          m.re = fma(c.im, rj.im, m.re);
          m.im = fma(-c.re, rj.im, m.im);
          m.im = fma(-c.im, rj.re, m.im);
        }
      }
      M[int64_t(i) * ld + j] = m;
    }
    __syncthreads();
  }
  // undo the column permutation: thread i owns row i
  for (int i = tid; i < K; i += NT)
    for (int k = K - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k) {
        const c128 x = M[int64_t(i) * ld + k];
        M[int64_t(i) * ld + k] = M[int64_t(i) * ld + p];
        M[int64_t(i) * ld + p] = x;
      }
    }
  __syncthreads();
  return 0;
}

LRZ_DEV int cta_gauss_jordan(c128 *M, int K, int ld, bool pivot, c128 *colbuf, c128 *rowbuf,
                             int *perm, double *red, int *ired) {
  if (pivot && K <= 64 && blockDim.x >= 32) return cta_gj_pivot_small(M, K, ld, colbuf, rowbuf, perm, ired);
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

// Exact 2-norm condition number of the n x n matrix X (row stride ld) by
// one-sided Jacobi (Hestenes) on its columns, in place (X is destroyed):
// sigma_max / sigma_min of the converged column norms, the quantity
// np.linalg.cond computes (lowrank.py:135,212).  Block-cooperative; one warp
// per column pair, round-robin ordering.  inf when sigma_min == 0.
LRZ_DEV double cta_jacobi_cond(c128 *X, int n, int ld, double *red, int *flag) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const int dp = n + (n & 1), npairs = dp / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < dp - 1; ++rnd) {
      for (int pi = wid; pi < npairs; pi += NW) {
        int a, b;
        if (pi == 0) {
          a = rnd;
          b = dp - 1;
        } else {
          a = (rnd + pi) % (dp - 1);
          b = (rnd - pi + dp - 1) % (dp - 1);
        }
        if (a > b) {
          const int t_ = a;
          a = b;
          b = t_;
        }
        if (b >= n) continue;  // warp-uniform
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (int k = lane; k < n; k += 32) {
          const c128 x = X[int64_t(k) * ld + a], y = X[int64_t(k) * ld + b];
          al += cabs2(x);
          be += cabs2(y);
          gr += x.re * y.re + x.im * y.im;  // (x^H y)
          gi += x.re * y.im - x.im * y.re;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        gr = warp_sum(gr);
        gi = warp_sum(gi);
        const double g = hypot(gr, gi);
        if (!(g > 1e-15 * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        const c128 ph = mk<double>(gr / g, -gi / g);  // e^{-i phi}
        for (int k = lane; k < n; k += 32) {
          c128 &x = X[int64_t(k) * ld + a];
          c128 &y = X[int64_t(k) * ld + b];
          const c128 xv = x, yv = cmul(y, ph);
          x = mk<double>(c * xv.re - sn * yv.re, c * xv.im - sn * yv.im);
          y = mk<double>(sn * xv.re + c * yv.re, sn * xv.im + c * yv.im);
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    const int rot = *flag;
    __syncthreads();
    if (!rot) break;
  }
  // column norms -> sigma_max, sigma_min
  double smax = 0.0, smin = 1e308;
  for (int j = wid; j < n; j += NW) {
    double s2 = 0.0;
    for (int k = lane; k < n; k += 32) s2 += cabs2(X[int64_t(k) * ld + j]);
    s2 = warp_sum(s2);
    smax = fmax(smax, s2);
    smin = fmin(smin, s2);
  }
  // block max / min of the per-warp values (lane-uniform)
  __syncthreads();
  if (lane == 0) {
    red[wid] = smax;
    red[NW + wid] = smin;
  }
  __syncthreads();
  double M = 0.0, m = 1e308;
  for (int i = 0; i < NW; ++i) {
    M = fmax(M, red[i]);
    m = fmin(m, red[NW + i]);
  }
  __syncthreads();
  return m > 0.0 ? sqrt(M) / sqrt(m) : INFINITY;
}

// Condition guard shared by direct_inverse (1e14) and the Woodbury aux (1e12),
// deciding exactly like np.linalg.cond(X) > limit (lowrank.py:135,212):
// ||X||_F ||X^-1||_F >= cond_2(X), so a bound at or below the limit accepts;
// otherwise cond_2 is computed exactly by one-sided Jacobi on the writable
// copy `work` (n x n, row stride ldw, destroyed; `red` needs 2 * warps doubles).
LRZ_DEV bool cta_cond_ok(double fx, double fi, double limit, c128 *work, int n, int ldw,
                         double *red, int *flag) {
  const double fb = sqrt(fx) * sqrt(fi);
  if (fb <= limit) return true;
  if (!isfinite(fx) || !isfinite(fi)) return false;
  const double c = cta_jacobi_cond(work, n, ldw, red, flag);
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
    const double fb = sqrt(fa) * sqrt(fi);
    bool ok = fb <= limit;
    if (!ok && isfinite(fb)) {
      // exact cond_2 of A (one-sided Jacobi on a copy in the output buffer, the
      // accuracy class of np.linalg.cond), then invert again
      for (int e = tid; e < K * K; e += NT) W[e] = Ain[e];
      __syncthreads();
      ok = cta_jacobi_cond(W, K, K, sc.red, sc.ired) <= limit;
      for (int e = tid; e < K * K; e += NT) W[e] = Ain[e];
      __syncthreads();
      cta_gauss_jordan(W, K, K, indefinite, sc.colbuf, sc.rowbuf, sc.perm, sc.red, sc.ired);
    }
    if (!ok)
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
  // (sc.aux is not needed after this point: the exact path rotates it in place)
  if (!cta_cond_ok(fa, fi, 1e12, sc.aux, r, r, sc.inv.red, sc.inv.ired))
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
