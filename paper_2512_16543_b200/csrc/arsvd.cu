// K2 + K3: adaptive randomised SVD of a K x K Gram correction
// (reference lowrank.py:243-316, Alg. 1), one CTA per item.
//
// Per sketch iteration of width d:
//   Y = dA Omega                  (Omega from the caller's normal stream)
//   Q = orth(Y)                   Householder QR + explicit Q, columns rotated so
//                                 diag(R) > 0: the unique basis the reference's
//                                 phase-fixed zgeqrf gives (lowrank.py:230-240)
//                                 for full-rank Y; orthonormal to working
//                                 precision even when Y is rank deficient
//   M = dA^H Q  (= B^H)           B = Q^H dA (lowrank.py:289)
//   one-sided Jacobi on M         M J = V S  ->  B = J S V^H
//   sort, energy test             cumsum(s^2) >= eta ||dA||_F^2
//   U = Q J                       (lowrank.py:291)
// All in complex128 / fp64 (the reference promotes c64 input here, D8).

#include "common.cuh"

namespace lrz {

constexpr int ARSVD_THREADS = 256;
constexpr int ARSVD_DMAX = 256;
constexpr double JACOBI_TOL = 1e-15;
constexpr int JACOBI_MAX_SWEEPS = 40;

struct ArsvdArgs {
  int K;
  const c128 *dA;
  int64_t as;
  const double *omega;
  int64_t os;
  const int32_t *orow;
  const int64_t *cursor;
  double eta;
  int k_init, p, i_max, D;
  c128 *U, *V;
  double *S;
  int32_t *k_est, *iters, *fallback;
  int64_t *consumed;
  const uint8_t *mask;
  c128 *ws;
};

// circle-method round robin: pair pi of round rnd among dp (even) players
LRZ_DEV void rr_pair(int rnd, int pi, int dp, int &a, int &b) {
  const int n1 = dp - 1;
  if (pi == 0) {
    a = rnd;
    b = n1;
  } else {
    a = (rnd + pi) % n1;
    b = (rnd - pi + n1) % n1;
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

__global__ void __launch_bounds__(ARSVD_THREADS) arsvd_kernel(ArsvdArgs g) {
  const int64_t item = blockIdx.x;
  if (g.mask && !g.mask[item]) return;
  const int K = g.K, D = g.D;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;

  __shared__ double red[ARSVD_THREADS / 32];
  __shared__ double sval[ARSVD_DMAX];
  __shared__ int perm[ARSVD_DMAX];
  __shared__ c128 rbuf[ARSVD_DMAX];
  __shared__ double s_tau[ARSVD_DMAX];
  __shared__ c128 s_ph[ARSVD_DMAX];
  __shared__ int s_rot[2];
  __shared__ int s_r;

  const c128 *dA = g.dA + item * g.as;
  const double *om = g.omega + (g.orow ? int64_t(g.orow[item]) : item) * g.os;
  int64_t cur = g.cursor ? g.cursor[item] : 0;
  const int64_t cur0 = cur;
  c128 *Q = g.ws + item * (int64_t(2) * D * K + int64_t(D) * D);  // [D][K]
  c128 *M = Q + int64_t(D) * K;                                    // [D][K]
  c128 *J = M + int64_t(D) * K;                                    // [D][D] col-major
  c128 *U = g.U + item * int64_t(D) * K;
  c128 *V = g.V + item * int64_t(D) * K;
  double *S = g.S + item * D;

  // ||dA||_F^2 (lowrank.py:274)
  double loc = 0.0;
  for (int e = tid; e < K * K; e += NT) loc += cabs2(dA[e]);
  const double energy = block_sum(loc, red);
  if (energy == 0.0) {  // empty factor (lowrank.py:275-276)
    if (tid == 0) {
      g.k_est[item] = 0;
      g.iters[item] = 0;
      g.fallback[item] = 0;
      g.consumed[item] = 0;
    }
    return;
  }
  const double target = g.eta * energy;
  const double SQH = 0.7071067811865476;  // np.sqrt(0.5)
  int k0 = g.k_init, d = 0, it = 0, r = -1;

  for (it = 0; it < g.i_max; ++it) {
    d = min(k0 + g.p, K);
    const double *zre = om + cur;
    const double *zim = zre + int64_t(K) * d;
    cur += int64_t(2) * K * d;
    // ---- Y = dA Omega  (threads: k slow, j fast -> Omega row contiguous)
    for (int e = tid; e < K * d; e += NT) {
      const int k = e / d, j = e - k * d;
      c128 a = czero<double>();
      const c128 *row = dA + int64_t(k) * K;
      for (int m = 0; m < K; ++m) {
        const c128 w = mk<double>(SQH * zre[m * d + j], SQH * zim[m * d + j]);
        cfma(a, row[m], w);
      }
      Q[int64_t(j) * K + k] = a;
    }
    __syncthreads();
    // ---- Householder QR of Y (in Q), explicit Q formed in M, then swap.
    //      Columns are rotated so diag(R) is real positive (lowrank.py:230-240).
    for (int j = 0; j < d; ++j) {
      c128 *wj = Q + int64_t(j) * K;
      if (wid == 0) {
        double sig2 = 0.0;
        for (int k = j + 1 + lane; k < K; k += 32) sig2 += cabs2(wj[k]);
        sig2 = warp_sum(sig2);
        if (lane == 0) {
          const c128 x0 = wj[j];
          const double ax = sqrt(cabs2(x0));
          const double nrm = sqrt(ax * ax + sig2);
          if (nrm == 0.0) {
            s_tau[j] = 0.0;
            s_ph[j] = mk<double>(1.0, 0.0);
          } else {
            const c128 e = ax > 0.0 ? mk<double>(x0.re / ax, x0.im / ax) : mk<double>(1.0, 0.0);
            const c128 v0 = mk<double>(e.re * (ax + nrm), e.im * (ax + nrm));
            s_tau[j] = 2.0 / (cabs2(v0) + sig2);
            s_ph[j] = mk<double>(-e.re, -e.im);  // alpha / |alpha|
            wj[j] = v0;
          }
        }
      }
      __syncthreads();
      const double tau = s_tau[j];
      if (tau != 0.0) {
        for (int c = j + 1 + wid; c < d; c += NW) {
          const c128 *wc = Q + int64_t(c) * K;
          double re = 0.0, im = 0.0;
          for (int k = j + lane; k < K; k += 32) {
            const c128 a = wj[k], b = wc[k];
            re = fma(a.re, b.re, fma(a.im, b.im, re));
            im = fma(a.re, b.im, fma(-a.im, b.re, im));
          }
          re = warp_sum(re);
          im = warp_sum(im);
          if (lane == 0) rbuf[c] = mk<double>(tau * re, tau * im);
        }
        __syncthreads();
        const int rows = K - j, ncol = d - j - 1;
        for (int e = tid; e < rows * ncol; e += NT) {
          const int c = j + 1 + e / rows, k = j + e % rows;
          const c128 v = wj[k], w = rbuf[c];
          c128 &x = Q[int64_t(c) * K + k];
          x.re -= v.re * w.re - v.im * w.im;
          x.im -= v.re * w.im + v.im * w.re;
        }
        __syncthreads();
      }
    }
    for (int e = tid; e < K * d; e += NT) {
      const int c = e / K, k = e - c * K;
      M[e] = mk<double>(k == c ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    for (int j = d - 1; j >= 0; --j) {
      const double tau = s_tau[j];
      if (tau == 0.0) continue;  // block-uniform
      const c128 *vj = Q + int64_t(j) * K;
      for (int c = j + wid; c < d; c += NW) {
        const c128 *qc = M + int64_t(c) * K;
        double re = 0.0, im = 0.0;
        for (int k = j + lane; k < K; k += 32) {
          const c128 a = vj[k], b = qc[k];
          re = fma(a.re, b.re, fma(a.im, b.im, re));
          im = fma(a.re, b.im, fma(-a.im, b.re, im));
        }
        re = warp_sum(re);
        im = warp_sum(im);
        if (lane == 0) rbuf[c] = mk<double>(tau * re, tau * im);
      }
      __syncthreads();
      const int rows = K - j, ncol = d - j;
      for (int e = tid; e < rows * ncol; e += NT) {
        const int c = j + e / rows, k = j + e % rows;
        const c128 v = vj[k], w = rbuf[c];
        c128 &x = M[int64_t(c) * K + k];
        x.re -= v.re * w.re - v.im * w.im;
        x.im -= v.re * w.im + v.im * w.re;
      }
      __syncthreads();
    }
    for (int e = tid; e < K * d; e += NT) {
      const int c = e / K;
      M[e] = cmul(M[e], s_ph[c]);
    }
    {
      c128 *t = Q;
      Q = M;
      M = t;
    }
    __syncthreads();
    // ---- M = dA^H Q  (B^H; threads: j slow, k fast -> dA row contiguous)
    for (int e = tid; e < K * d; e += NT) {
      const int j = e / K, k = e - j * K;
      c128 a = czero<double>();
      const c128 *qj = Q + int64_t(j) * K;
      for (int m = 0; m < K; ++m) cfma_ca(a, dA[int64_t(m) * K + k], qj[m]);
      M[int64_t(j) * K + k] = a;
    }
    for (int e = tid; e < d * d; e += NT) J[e] = mk<double>((e % (d + 1)) == 0 ? 1.0 : 0.0, 0.0);
    if (tid == 0) s_rot[0] = s_rot[1] = 0;
    __syncthreads();
    // ---- one-sided Jacobi (Hestenes), parallel round-robin ordering
    const int dp = d + (d & 1), npairs = dp / 2;
    for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
      for (int rnd = 0; rnd < dp - 1; ++rnd) {
        for (int pi = wid; pi < npairs; pi += NW) {
          int a, b;
          rr_pair(rnd, pi, dp, a, b);
          if (b >= d) continue;
          c128 *ma = M + int64_t(a) * K, *mb = M + int64_t(b) * K;
          double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
          for (int k = lane; k < K; k += 32) {
            const c128 x = ma[k], y = mb[k];
            al += cabs2(x);
            be += cabs2(y);
            gr = fma(x.re, y.re, fma(x.im, y.im, gr));
            gi = fma(x.re, y.im, fma(-x.im, y.re, gi));
          }
          al = warp_sum(al);
          be = warp_sum(be);
          gr = warp_sum(gr);
          gi = warp_sum(gi);
          const double gabs = hypot(gr, gi);
          if (!(gabs > JACOBI_TOL * sqrt(al) * sqrt(be)) || gabs == 0.0) continue;
          const double zeta = (be - al) / (2.0 * gabs);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          const c128 ph = mk<double>(gr / gabs, -gi / gabs);  // e^{-i phi}
          for (int k = lane; k < K; k += 32) {
            const c128 x = ma[k], y = cmul(mb[k], ph);
            ma[k] = mk<double>(c * x.re - s * y.re, c * x.im - s * y.im);
            mb[k] = mk<double>(s * x.re + c * y.re, s * x.im + c * y.im);
          }
          c128 *ja = J + int64_t(a) * d, *jb = J + int64_t(b) * d;
          for (int k = lane; k < d; k += 32) {
            const c128 x = ja[k], y = cmul(jb[k], ph);
            ja[k] = mk<double>(c * x.re - s * y.re, c * x.im - s * y.im);
            jb[k] = mk<double>(s * x.re + c * y.re, s * x.im + c * y.im);
          }
          if (lane == 0) s_rot[sweep & 1] = 1;
        }
        __syncthreads();
        // the next sweep's flag was last read before this sweep's first barrier
        if (rnd == 0 && tid == 0) s_rot[(sweep + 1) & 1] = 0;
      }
      if (dp - 1 == 0) __syncthreads();
      const int rotated = s_rot[sweep & 1];
      if (!rotated) break;
    }
    // ---- singular values, descending order, energy test (lowrank.py:290-301)
    for (int j = wid; j < d; j += NW) {
      const c128 *mj = M + int64_t(j) * K;
      double s2 = 0.0;
      for (int k = lane; k < K; k += 32) s2 += cabs2(mj[k]);
      s2 = warp_sum(s2);
      if (lane == 0) sval[j] = sqrt(s2);
    }
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < d; ++j) perm[j] = j;
      for (int j = 1; j < d; ++j) {  // stable insertion sort, descending
        const int pj = perm[j];
        int i = j - 1;
        while (i >= 0 && sval[perm[i]] < sval[pj]) {
          perm[i + 1] = perm[i];
          --i;
        }
        perm[i + 1] = pj;
      }
      double cum = 0.0;
      int hit = -1;
      for (int j = 0; j < d; ++j) {
        const double sj = sval[perm[j]];
        cum += sj * sj;
        if (cum >= target) {
          hit = j + 1;
          break;
        }
      }
      s_r = hit;
    }
    __syncthreads();
    r = s_r;
    __syncthreads();
    if (r > 0) break;
    k0 *= 2;
  }
  bool fb = false;
  if (r <= 0) {  // iteration cap: full rank-d factor minus numerical zeros (lowrank.py:304-316)
    fb = true;
    it = g.i_max - 1;
    const double floor = sval[perm[0]] * K * EPS64;
    int cnt = 0;
    for (int j = 0; j < d; ++j) cnt += sval[perm[j]] > floor ? 1 : 0;
    r = cnt > 1 ? cnt : 1;
  }
  // ---- outputs: S, V = M_perm / s, U = Q J_perm (all d columns, sorted)
  for (int e = tid; e < K * d; e += NT) {
    const int j = e / K, k = e - j * K;
    const int pj = perm[j];
    const double sj = sval[pj];
    const c128 m = M[int64_t(pj) * K + k];
    V[int64_t(j) * K + k] = sj > 0.0 ? cscale(m, 1.0 / sj) : czero<double>();
    c128 a = czero<double>();
    const c128 *jc = J + int64_t(pj) * d;
    for (int i = 0; i < d; ++i) cfma(a, Q[int64_t(i) * K + k], jc[i]);
    U[int64_t(j) * K + k] = a;
  }
  for (int j = tid; j < d; j += NT) S[j] = sval[perm[j]];
  if (tid == 0) {
    g.k_est[item] = r;
    g.iters[item] = it + 1;
    g.fallback[item] = fb ? 1 : 0;
    g.consumed[item] = cur - cur0;
  }
}

}  // namespace lrz

using namespace lrz;

size_t lrz_arsvd_ws(int64_t B, int K, int D) {
  return size_t(B) * (size_t(2) * D * K + size_t(D) * D) * sizeof(c128);
}

extern "C" int lrz_arsvd(int64_t B, int K, const void *dA, int64_t a_stride,
                         const double *omega, int64_t omega_stride, const int32_t *omega_row,
                         const int64_t *cursor, const lrz_arsvd_cfg *cfg, void *U, void *V,
                         double *S, int32_t *k_est, int32_t *iters, int32_t *fallback,
                         int64_t *consumed, const uint8_t *item_mask, void *workspace,
                         void *stream) {
  if (B < 0 || K < 1 || !dA || !omega || !cfg || !U || !V || !S || !k_est || !iters ||
      !fallback || !consumed || !workspace) {
    lrz_set_error("lrz_arsvd: bad arguments");
    return LRZ_EINVAL;
  }
  if (!(cfg->eta > 0.0 && cfg->eta <= 1.0) || cfg->k_init < 1 || cfg->p < 0 || cfg->i_max < 1) {
    lrz_set_error("lrz_arsvd: bad ArSvdConfig");
    return LRZ_EINVAL;
  }
  int dneed = 0;
  long long k0 = cfg->k_init;
  for (int i = 0; i < cfg->i_max; ++i) {
    dneed = (int)std::min<long long>(k0 + cfg->p, K);
    k0 *= 2;
  }
  if (cfg->d_max < dneed || cfg->d_max > ARSVD_DMAX) {
    lrz_set_error("lrz_arsvd: d_max %d must be in [%d, %d]", cfg->d_max, dneed, ARSVD_DMAX);
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  ArsvdArgs g;
  g.K = K;
  g.dA = (const c128 *)dA;
  g.as = a_stride;
  g.omega = omega;
  g.os = omega_stride;
  g.orow = omega_row;
  g.cursor = cursor;
  g.eta = cfg->eta;
  g.k_init = cfg->k_init;
  g.p = cfg->p;
  g.i_max = cfg->i_max;
  g.D = cfg->d_max;
  g.U = (c128 *)U;
  g.V = (c128 *)V;
  g.S = S;
  g.k_est = k_est;
  g.iters = iters;
  g.fallback = fallback;
  g.consumed = consumed;
  g.mask = item_mask;
  g.ws = (c128 *)workspace;
  arsvd_kernel<<<unsigned(B), ARSVD_THREADS, 0, (cudaStream_t)stream>>>(g);
  return lrz_launch_status("lrz_arsvd");
}
