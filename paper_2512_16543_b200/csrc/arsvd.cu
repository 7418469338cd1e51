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

#include "dmma.cuh"

int lrz_sketch_gemm(int64_t B, int K, int Dtot, const void *dA, int64_t a_stride,
                    const double *omega, int64_t omega_stride, const int32_t *omega_row,
                    int64_t orow_div, const int64_t *cursor, int k_init, int p,
                    const uint8_t *mask, void *Y, void *W, void *stream);

int lrz_use_dmma();
int lrz_arsvd_tail_M(int64_t B, int K, int D, const void *dA, int64_t a_stride, const void *Q,
                     void *M, int64_t wst, const uint8_t *tail, cudaStream_t s);
int lrz_arsvd_tail_U(int64_t B, int K, int D, const void *Jp, const void *Q, int64_t wst,
                     void *U, const uint8_t *tail, cudaStream_t s);
int lrz_sketch_dmma_large(int64_t B, int K, int Dtot, const void *dA, int64_t a_stride,
                          const double *omega, int64_t omega_stride, const int32_t *omega_row,
                          int64_t orow_div, const int64_t *cursor, int k_init, int p,
                          const uint8_t *mask, void *Om, void *Y, void *W, cudaStream_t s);

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
  int64_t orow_div;  // orow == NULL: omega row of item = item / orow_div
  const int64_t *cursor;
  double eta;
  const double *eta_row;  // nullable: energy fraction per omega row (overrides eta)
  int64_t omega_len;      // > 0: normals available per omega row (guard)
  int k_init, p, i_max, D;
  int want;  // 1: always produce U/S/V; 0: only when 2 k_est <= K (Woodbury candidate)
  const int32_t *start_it;  // nullable: iteration to resume at (warp front end), < 0 = skip
  const c128 *ya;           // nullable: the front end's Y_all [item][K][ydtot]; a resumed
  int ydtot;                //   iteration takes its sketch Y from there
  // K > 32 tail pipeline for items the front end resumed at the last iteration:
  // phase 1 forms Q (Householder) and stops; M = dA^H Q runs as a batched DMMA
  // GEMM; phase 2 takes M and finishes (SVD, rank, V); U = Q J_perm is a second
  // GEMM.  tail[item]: 1 = in the pipeline, 2 = U wanted from the GEMM.
  int phase;
  int smem_ws;  // 1: per-item Q / M / J live in dynamic shared memory (no tail pipeline)
  int smem_j;   // 1: J and the preconditioned Jacobi's R live in dynamic shared memory
  uint8_t *tail;
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
  } else {  // rnd < n1, 0 < pi <= n1 / 2: one conditional wrap instead of a modulo
    a = rnd + pi;
    if (a >= n1) a -= n1;
    b = rnd - pi;
    if (b < 0) b += n1;
  }
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
}

// One-sided Jacobi (Hestenes) on the d columns of M (length K), rotations
// accumulated in J (d x d, column-major); parallel round-robin ordering, one
// 8-lane group per column pair (a warp carries four pairs, so the per-pair
// scalar chain -- hypot, sqrt, divisions -- is issued once for four pairs and
// the dot products reduce in three shuffle rounds).  On exit sval[j] = ||M_j||
// and perm sorts them descending (stable).  Block-cooperative; contains barriers.
constexpr int JG = 8;  // lanes per column pair

LRZ_DEV double grp_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

LRZ_DEV void jacobi_sv(c128 *M, c128 *J, int K, int d, double *sval, int *perm, int *s_rot) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;
  const int gl = lane & (JG - 1), grp = tid / JG, NG = NT / JG;
  for (int e = tid; e < d * d; e += NT) J[e] = mk<double>((e % (d + 1)) == 0 ? 1.0 : 0.0, 0.0);
  if (tid == 0) s_rot[0] = s_rot[1] = 0;
  __syncthreads();
  const int dp = d + (d & 1), npairs = dp / 2;
  for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
    for (int rnd = 0; rnd < dp - 1; ++rnd) {
      // warp-uniform trip count: every lane reaches the group shuffles
      for (int base = 0; base < npairs; base += NG) {
        const int pi = base + grp;
        int a = 0, b = 0;
        if (pi < npairs) rr_pair(rnd, pi, dp, a, b);
        const bool act = pi < npairs && b < d;
        const c128 *ma = M + int64_t(a) * K, *mb = M + int64_t(b) * K;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        if (act) {
          for (int k = gl; k < K; k += JG) {
            const c128 x = ma[k], y = mb[k];
            al += cabs2(x);
            be += cabs2(y);
            gr = fma(x.re, y.re, fma(x.im, y.im, gr));
            gi = fma(x.re, y.im, fma(-x.im, y.re, gi));
          }
        }
        al = grp_sum(al);
        be = grp_sum(be);
        gr = grp_sum(gr);
        gi = grp_sum(gi);
        if (!act) continue;
        // |g|^2 against (tol ||a|| ||b||)^2: no square roots on the skip path; 1 / |g|
        // by rsqrt, the tangent's quotient by a reciprocal (the rotation only has to
        // be unitary to rounding, which c and s from one rsqrt are)
        const double g2 = fma(gr, gr, gi * gi);
        if (!(g2 > (JACOBI_TOL * JACOBI_TOL) * al * be) || !(g2 > 0.0)) continue;
        const double ig = rsqrt(g2);
        const double zeta = (be - al) * (0.5 * ig);
        const double z1 = fma(zeta, zeta, 1.0);
        const double t = copysign(__drcp_rn(fabs(zeta) + z1 * rsqrt(z1)), zeta);
        const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
        const c128 ph = mk<double>(gr * ig, -gi * ig);  // e^{-i phi}
        c128 *wa = M + int64_t(a) * K, *wb = M + int64_t(b) * K;
        for (int k = gl; k < K; k += JG) {
          const c128 x = wa[k], y = cmul(wb[k], ph);
          wa[k] = mk<double>(c * x.re - s * y.re, c * x.im - s * y.im);
          wb[k] = mk<double>(s * x.re + c * y.re, s * x.im + c * y.im);
        }
        c128 *ja = J + int64_t(a) * d, *jb = J + int64_t(b) * d;
        for (int k = gl; k < d; k += JG) {
          const c128 x = ja[k], y = cmul(jb[k], ph);
          ja[k] = mk<double>(c * x.re - s * y.re, c * x.im - s * y.im);
          jb[k] = mk<double>(s * x.re + c * y.re, s * x.im + c * y.im);
        }
        // another sweep only if some pair of this one was coupled above 1e-8: pairs
        // below that are rotated here and leave second-order (~1e-16) couplings, so
        // the sweep that would merely confirm convergence is not run
        if (gl == 0 && g2 > 1e-16 * al * be) s_rot[sweep & 1] = 1;
      }
      __syncthreads();
      // the next sweep's flag was last read before this sweep's first barrier
      if (rnd == 0 && tid == 0) s_rot[(sweep + 1) & 1] = 0;
    }
    const int rotated = s_rot[sweep & 1];
    if (!rotated) break;
  }
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
  }
  __syncthreads();
}

// Certificate that every singular value of B (d of them; B^H = M) is far
// above the fallback floor s_max K eps: C = M^H M = L L^H (Cholesky) and
// lambda_min(C) >= 1 / ||L^-1||_F^2 >= 1e-9 tr(C).  C lives in Cw (d x d),
// L^-1 columns in Xw (d x d).  Returns a block-uniform bool.
LRZ_DEV bool gram_certificate(const c128 *M, int K, int d, double trC, c128 *Cw, c128 *Xw,
                              double *red) {
  const int tid = threadIdx.x, NT = blockDim.x;
  for (int e = tid; e < d * d; e += NT) {
    const int i = e / d, j = e - i * d;
    if (i < j) continue;
    const c128 *mi = M + int64_t(i) * K, *mj = M + int64_t(j) * K;
    c128 a = czero<double>();
    for (int k = 0; k < K; ++k) cfma_ca(a, mi[k], mj[k]);  // C_ij = m_i^H m_j
    Cw[e] = a;
  }
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    const double piv = Cw[j * d + j].re;
    if (!(piv > 0.0)) return false;
    const double l = sqrt(piv), il = 1.0 / l;
    __syncthreads();
    for (int i = j + 1 + tid; i < d; i += NT) Cw[i * d + j] = cscale(Cw[i * d + j], il);
    if (tid == 0) Cw[j * d + j] = mk<double>(l, 0.0);
    __syncthreads();
    const int n = d - j - 1;
    for (int e = tid; e < n * n; e += NT) {
      const int i = j + 1 + e / n, k = j + 1 + e % n;
      if (k > i) continue;
      const c128 a = Cw[i * d + j], b = Cw[k * d + j];
      c128 &x = Cw[i * d + k];
      x.re -= a.re * b.re + a.im * b.im;
      x.im -= a.im * b.re - a.re * b.im;
    }
    __syncthreads();
  }
  double loc = 0.0;
  for (int t = tid; t < d; t += NT) {
    c128 *x = Xw + int64_t(t) * d;
    for (int i = t; i < d; ++i) {
      c128 acc = mk<double>(i == t ? 1.0 : 0.0, 0.0);
      for (int k = t; k < i; ++k) {
        const c128 lk = Cw[i * d + k], xk = x[k];
        acc.re -= lk.re * xk.re - lk.im * xk.im;
        acc.im -= lk.re * xk.im + lk.im * xk.re;
      }
      x[i] = cscale(acc, 1.0 / Cw[i * d + i].re);
      loc += cabs2(x[i]);
    }
  }
  const double F = block_sum(loc, red);
  return isfinite(F) && F * trC <= 1e9;
}

// In-place Householder QR of the d columns (length K, column-major [d][K]) of
// X: reflector j = (v0 at X[j][j], X[j][j+1..K-1]) with tau[j]; the strictly
// upper part of R stays in X[c][r], r < c; R's diagonal goes to rdiag.
// Block-cooperative (barriers inside).
LRZ_DEV void hh_qr(c128 *X, int K, int d, double *tau, c128 *rdiag, c128 *rbuf) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;
  for (int j = 0; j < d; ++j) {
    c128 *wj = X + int64_t(j) * K;
    if (wid == 0) {
      double sig2 = 0.0;
      for (int k = j + 1 + lane; k < K; k += 32) sig2 += cabs2(wj[k]);
      sig2 = warp_sum(sig2);
      if (lane == 0) {
        const c128 x0 = wj[j];
        const double ax = sqrt(cabs2(x0));
        const double nrm = sqrt(ax * ax + sig2);
        if (nrm == 0.0) {
          tau[j] = 0.0;
          rdiag[j] = czero<double>();
        } else {
          const c128 e = ax > 0.0 ? mk<double>(x0.re / ax, x0.im / ax) : mk<double>(1.0, 0.0);
          const c128 v0 = mk<double>(e.re * (ax + nrm), e.im * (ax + nrm));
          tau[j] = 2.0 / (cabs2(v0) + sig2);
          rdiag[j] = mk<double>(-e.re * nrm, -e.im * nrm);
          wj[j] = v0;
        }
      }
    }
    __syncthreads();
    const double tj = tau[j];
    if (tj != 0.0) {
      for (int c = j + 1 + wid; c < d; c += NW) {
        const c128 *wc = X + int64_t(c) * K;
        double re = 0.0, im = 0.0;
        for (int k = j + lane; k < K; k += 32) {
          const c128 a = wj[k], b = wc[k];
          re = fma(a.re, b.re, fma(a.im, b.im, re));
          im = fma(a.re, b.im, fma(-a.im, b.re, im));
        }
        re = warp_sum(re);
        im = warp_sum(im);
        if (lane == 0) rbuf[c] = mk<double>(tj * re, tj * im);
      }
      __syncthreads();
      const int rows = K - j, ncol = d - j - 1;
      for (int e = tid; e < rows * ncol; e += NT) {
        const int c = j + 1 + e / rows, k = j + e % rows;
        const c128 v = wj[k], w = rbuf[c];
        c128 &x = X[int64_t(c) * K + k];
        x.re -= v.re * w.re - v.im * w.im;
        x.im -= v.re * w.im + v.im * w.re;
      }
      __syncthreads();
    }
  }
}

// C <- Q C for the Q of hh_qr (reflectors in X, tau), C: nc columns of length K
// (column-major [nc][K]).  Block-cooperative.
LRZ_DEV void hh_apply(const c128 *X, int K, int d, const double *tau, c128 *C, int nc,
                      c128 *rbuf) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;
  for (int j = d - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj == 0.0) continue;  // block-uniform
    const c128 *vj = X + int64_t(j) * K;
    for (int c = wid; c < nc; c += NW) {
      const c128 *qc = C + int64_t(c) * K;
      double re = 0.0, im = 0.0;
      for (int k = j + lane; k < K; k += 32) {
        const c128 a = vj[k], b = qc[k];
        re = fma(a.re, b.re, fma(a.im, b.im, re));
        im = fma(a.re, b.im, fma(-a.im, b.re, im));
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == 0) rbuf[c] = mk<double>(tj * re, tj * im);
    }
    __syncthreads();
    const int rows = K - j;
    for (int e = tid; e < rows * nc; e += NT) {
      const int c = e / rows, k = j + e % rows;
      const c128 v = vj[k], w = rbuf[c];
      c128 &x = C[int64_t(c) * K + k];
      x.re -= v.re * w.re - v.im * w.im;
      x.im -= v.re * w.im + v.im * w.re;
    }
    __syncthreads();
  }
}

// One arsvd call (item) by the whole CTA, sketch stream read from `cur`,
// resuming at iteration it0.  Returns the normals consumed (block-uniform).
// DM: bound on the sketch width d (sizes the per-item shared scratch: the small
// kernel's items leave the SM's shared memory to the kernels they overlap with).
template <int DM = ARSVD_DMAX>
LRZ_DEV int64_t arsvd_item(const ArsvdArgs &g, const int64_t item, int64_t cur, const int it0) {
  const int K = g.K, D = g.D;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, wid = tid >> 5, NW = NT >> 5;

  __shared__ double red[ARSVD_THREADS / 32];
  __shared__ double sval[DM];
  __shared__ int perm[DM];
  __shared__ c128 rbuf[DM];
  __shared__ double s_tau[DM];
  __shared__ c128 s_ph[DM];
  __shared__ int s_rot[2];
  __shared__ int s_r;

  const bool tail = g.phase != 0 && g.ya && it0 == g.i_max - 1;
  if (g.phase == 2 && !tail) return 0;
  const c128 *dA = g.dA + item * g.as;
  const int64_t orw = g.orow ? int64_t(g.orow[item]) : item / g.orow_div;
  const double *om = g.omega + orw * g.os;
  const int64_t cur0 = cur;
  // small problems keep Q / M / J in shared memory (g.smem_ws: the launch reserved
  // (2 D K + D^2) complex of dynamic shared memory), the rest in the global workspace
  extern __shared__ __align__(16) char arsvd_dyn_smem[];
  c128 *Q = g.smem_ws ? (c128 *)arsvd_dyn_smem
                      : g.ws + item * (int64_t(2) * D * K + int64_t(D) * D);  // [D][K]
  c128 *M = Q + int64_t(D) * K;                                    // [D][K]
  c128 *J = M + int64_t(D) * K;                                    // [D][D] col-major
  // K >= 64: the QR-preconditioned Jacobi's d x d operands (rotation matrix J and
  // the triangular factor) in dynamic shared memory (g.smem_j: 2 D^2 complex) --
  // every round re-reads the columns the last one wrote, which from global memory
  // is an L2 round trip per round
  c128 *Rsm = nullptr;
  if (g.smem_j) {
    J = (c128 *)arsvd_dyn_smem;
    Rsm = J + int64_t(D) * D;
  }
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
    return 0;
  }
  const double target = (g.eta_row ? g.eta_row[orw] : g.eta) * energy;
  const double SQH = 0.7071067811865476;  // np.sqrt(0.5)
  int k0 = g.k_init, d = 0, it = 0, r = -1;
  bool have_sv = false, hit_found = false;
  int yo = 0;                      // column offset of iteration it0 in Y_all
  for (int i = 0; i < it0; ++i) {  // resume: skip iterations the front end already ran
    cur += int64_t(2) * K * min(k0 + g.p, K);
    yo += min(k0 + g.p, K);
    k0 *= 2;
  }

  for (it = it0; it < g.i_max; ++it) {
    d = min(k0 + g.p, K);
    if (g.omega_len > 0 && cur + int64_t(2) * K * d > g.omega_len) {
      // sketch window too short for this call: report, never read past it
      if (tid == 0) {
        g.k_est[item] = 0;
        g.iters[item] = -1;
        g.fallback[item] = 0;
        g.consumed[item] = 0;
      }
      return 0;
    }
    const double *zre = om + cur;
    const double *zim = zre + int64_t(K) * d;
    cur += int64_t(2) * K * d;
    const bool p2 = g.phase == 2 && it == it0;  // Q and M come from phase 1 + the GEMM
    if (p2) {
      Q = g.ws + item * (int64_t(2) * D * K + int64_t(D) * D) + int64_t(D) * K;
      M = Q - int64_t(D) * K;
    } else {
    // ---- Y = dA Omega  (threads: k slow, j fast -> Omega row contiguous); a
    //      resumed iteration takes the front end's Y block (same Omega, DMMA product)
    if (g.ya && it == it0) {
      const c128 *ys = g.ya + item * int64_t(K) * g.ydtot + yo;
      for (int e = tid; e < K * d; e += NT) {
        const int k = e / d, j = e - k * d;
        Q[int64_t(j) * K + k] = ys[int64_t(k) * g.ydtot + j];
      }
    } else
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
    if (g.phase == 1 && tail) {  // Q formed: M = dA^H Q runs as a batched GEMM
      if (tid == 0) g.tail[item] = 1;
      return 0;
    }
    }  // !p2
    // ---- M = dA^H Q  (B^H; threads: j slow, k fast -> dA row contiguous)
    double loc2 = 0.0;
    if (p2) {
      for (int e = tid; e < K * d; e += NT) loc2 += cabs2(M[e]);
    } else
    for (int e = tid; e < K * d; e += NT) {
      const int j = e / K, k = e - j * K;
      c128 a = czero<double>();
      const c128 *qj = Q + int64_t(j) * K;
      for (int m = 0; m < K; ++m) cfma_ca(a, dA[int64_t(m) * K + k], qj[m]);
      M[int64_t(j) * K + k] = a;
      loc2 += cabs2(a);
    }
    // ||B||_F^2 = sum of all d squared singular values = cumsum(s^2)[-1]
    const double mf = block_sum(loc2, red);
    const bool last = (it == g.i_max - 1);
    const bool below = mf < target * (1.0 - 1e-12);  // no prefix can reach the target
    if (below && !last) {
      k0 *= 2;
      continue;
    }
    if (below && g.want == 0 && 2 * d > K) {
      // iteration-cap tail with r > K/2 (full branch, no factor needed): the
      // count of s > s_max K eps is d whenever sigma_min is certified far above
      // that floor (lowrank.py:307-309); otherwise fall through to the SVD.
      if (gram_certificate(M, K, d, mf, J, V, red)) {  // V: scratch for L^-1
        r = d;
        have_sv = false;
        break;
      }
    }
    if (K >= 64 && K >= 2 * d) {
      // QR-preconditioned one-sided Jacobi: M = Q2 R2 (Householder), rotate the
      // d x d R2 (columns of length d instead of K), then M J = Q2 (R2 J).  The
      // rotations and singular values are those of M (M^H M = R2^H R2).
      c128 *Rb = Rsm ? Rsm : V, *Ub = U;   // the item's factor outputs as scratch (written below)
      hh_qr(M, K, d, s_tau, s_ph, rbuf);
      for (int e = tid; e < d * d; e += NT) {
        const int c = e / d, r = e - c * d;
        Rb[e] = r < c ? M[int64_t(c) * K + r] : (r == c ? s_ph[c] : czero<double>());
      }
      __syncthreads();
      jacobi_sv(Rb, J, d, d, sval, perm, s_rot);
      for (int e = tid; e < K * d; e += NT) {
        const int c = e / K, k = e - c * K;
        Ub[e] = k < d ? Rb[int64_t(c) * d + k] : czero<double>();
      }
      __syncthreads();
      hh_apply(M, K, d, s_tau, Ub, d, rbuf);
      for (int e = tid; e < K * d; e += NT) M[e] = Ub[e];
      __syncthreads();
    } else {
      jacobi_sv(M, J, K, d, sval, perm, s_rot);
    }
    have_sv = true;
    // ---- energy test on the exact singular values (lowrank.py:290-301)
    if (tid == 0) {
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
    if (r > 0) {
      hit_found = true;
      break;
    }
    k0 *= 2;
  }
  bool fb = false;
  if (!hit_found) {  // iteration cap (lowrank.py:304-316)
    fb = true;
    it = g.i_max - 1;
    if (have_sv) {  // full rank-d factor minus numerical zeros
      const double floor = sval[perm[0]] * K * EPS64;
      int cnt = 0;
      for (int j = 0; j < d; ++j) cnt += sval[perm[j]] > floor ? 1 : 0;
      r = cnt > 1 ? cnt : 1;
    }
  }
  // ---- outputs: S, V = M_perm / s, U = Q J_perm (all d columns, sorted)
  if (tail && have_sv && (g.want == 1 || 2 * r <= K)) {
    // phase 2: V here; J_perm (column-major d x d) into M's buffer once M is
    // consumed, U = Q J_perm by the batched GEMM that follows
    for (int e = tid; e < K * d; e += NT) {
      const int j = e / K, k = e - j * K;
      const int pj = perm[j];
      const double sj = sval[pj];
      const c128 m = M[int64_t(pj) * K + k];
      V[int64_t(j) * K + k] = sj > 0.0 ? cscale(m, 1.0 / sj) : czero<double>();
    }
    __syncthreads();
    for (int e = tid; e < d * d; e += NT) {
      const int j = e / d, i = e - j * d;
      M[e] = J[int64_t(perm[j]) * d + i];
    }
    if (tid == 0) g.tail[item] = 2;
  } else if (have_sv && (g.want == 1 || 2 * r <= K)) {
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
  }
  if (have_sv)
    for (int j = tid; j < d; j += NT) S[j] = sval[perm[j]];
  if (tid == 0) {
    g.k_est[item] = r;
    g.iters[item] = it + 1;
    g.fallback[item] = fb ? 1 : 0;
    g.consumed[item] = cur - cur0;
  }
  return cur - cur0;
}

__global__ void __launch_bounds__(ARSVD_THREADS) arsvd_kernel(ArsvdArgs g) {
  const int64_t item = blockIdx.x;
  if (g.mask && !g.mask[item]) return;
  const int it0 = g.start_it ? g.start_it[item] : 0;
  if (it0 < 0) return;
  arsvd_item(g, item, g.cursor ? g.cursor[item] : 0, it0);
}

// The same item code for small problems (K <= 32): 128 threads per item and a
// register budget that keeps ARSVD_SMALL_CTAS items resident per SM -- the item is
// latency bound (one barrier and one scalar chain per reflector / Jacobi round),
// so throughput comes from the number of items in flight.
template <int CTAS>
__global__ void __launch_bounds__(128, CTAS) arsvd_small_kernel(ArsvdArgs g) {
  const int64_t item = blockIdx.x;
  if (g.mask && !g.mask[item]) return;
  const int it0 = g.start_it ? g.start_it[item] : 0;
  if (it0 < 0) return;
  arsvd_item<32>(g, item, g.cursor ? g.cursor[item] : 0, it0);
}

// In-order resolution of the unverified suffix of every trial: one CTA per
// trial walks its sketch steps t >= first[b] and feeds each call the cursor
// the previous one ended at -- the reference's sequential use of one
// Generator per (method, trial) (harness.py:211,236-237), with no speculation.
__global__ void __launch_bounds__(ARSVD_THREADS)
arsvd_seq_kernel(ArsvdArgs g, int T, const uint8_t *__restrict__ is_sketch,
                 const int32_t *__restrict__ first, int64_t *__restrict__ cursor,
                 int32_t *__restrict__ iters_pred) {
  const int64_t b = blockIdx.x;
  int t = first[b];
  if (t >= T) return;
  int64_t cur = cursor[b * T + t];
  for (; t < T; ++t) {
    const int64_t bt = b * T + t;
    if (threadIdx.x == 0) cursor[bt] = cur;
    if (!is_sketch[bt]) continue;
    cur += arsvd_item(g, bt, cur, 0);
    if (threadIdx.x == 0) iters_pred[bt] = g.iters[bt];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Batched screening front end (hermitian dA, factor not requested, D <= 32).
//
// Every sketch iteration i of one arsvd call reads its Omega block at a cursor
// that does not depend on the outcome of earlier iterations (cursor +
// sum_{i'<i} 2 K d_i', lowrank.py:284-286), so all i_max sketches are formed
// at once:   Y_all = dA [Omega_0 ... Omega_{i_max-1}],  W_all = dA Y_all
// (two batched GEMMs over all items; dA^H = dA).  A warp per item then screens
// the iterations in order with CholeskyQR: G_i = Y_i^H Y_i = L L^H,
// X_i = W_i L^-H (= dA^H Q_i for the CholeskyQR basis Q_i = Y_i L^-H), and
// ||X_i||_F^2 = ||Q_i^H dA||_F^2 = sum of all squared singular values of B_i
// (basis independent).  If that total is below the energy target
// by more than the CholeskyQR error bound, no prefix can reach it and the
// iteration is decided without an SVD.  The iteration-cap tail is decided
// here too when its rank d > K/2 is certified (lambda_min(X^H X) far above
// the s_max K eps floor).  Everything else is handed to arsvd_kernel, which
// redoes that iteration with Householder QR + one-sided Jacobi.
// ---------------------------------------------------------------------------
constexpr int SCR_DMAX = 40;

// Lower triangle of P^H P (d x d, d <= 32) for the K x d block P (row stride
// ld) on the FP64 tensor pipe, one warp: lane (g, t) loads P[k0 + t][8a + g],
// which is at once the (conjugated) A fragment of row block a and the B
// fragment of column block a, so NB (NB + 1) / 2 lower 8 x 8 tiles need no
// shared memory; written to L (row stride LD).  Replaces K-long per-entry dot
// products that were ~45 % of the screen's stall samples.
template <int NB, int IB0, int IB1>
LRZ_DEV void warp_gram_dmma_nb(const c128 *P, int64_t ld, int K, int d, c128 *L, int LD) {
  // row blocks IB0 <= ib < IB1 (all jb <= ib); plain loads: P may have been
  // written earlier in this kernel by other lanes (the tail's X)
  constexpr int NT = (IB1 * (IB1 + 1) - IB0 * (IB0 + 1)) / 2;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double cr[NT][2], ci[NT][2];
#pragma unroll
  for (int x = 0; x < NT; ++x) cr[x][0] = cr[x][1] = ci[x][0] = ci[x][1] = 0.0;
  for (int k0 = 0; k0 < K; k0 += 4) {
    const int k = k0 + t;
    double xr[IB1], xi[IB1];
#pragma unroll
    for (int a = 0; a < IB1; ++a) {
      const int col = 8 * a + g;
      const c128 v = (k < K && col < d) ? P[int64_t(k) * ld + col] : czero<double>();
      xr[a] = v.re;
      xi[a] = v.im;
    }
#pragma unroll
    for (int ib = IB0; ib < IB1; ++ib)
#pragma unroll
      for (int jb = 0; jb <= ib; ++jb) {
        const int x = (ib * (ib + 1) - IB0 * (IB0 + 1)) / 2 + jb;
        // conj(p_i) p_j = (pr_i pr_j + pi_i pi_j) + i (pr_i pi_j - pi_i pr_j)
        dmma(cr[x], xr[ib], xr[jb]);
        dmma(cr[x], xi[ib], xi[jb]);
        dmma(ci[x], xr[ib], xi[jb]);
        dmma(ci[x], -xi[ib], xr[jb]);
      }
  }
#pragma unroll
  for (int ib = IB0; ib < IB1; ++ib)
#pragma unroll
    for (int jb = 0; jb <= ib; ++jb) {
      const int x = (ib * (ib + 1) - IB0 * (IB0 + 1)) / 2 + jb;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * ib + g, col = 8 * jb + 2 * t + e;
        if (row < d && col <= row) L[row * LD + col] = mk<double>(cr[x][e], ci[x][e]);
      }
    }
}

LRZ_DEV void warp_gram_dmma(const c128 *P, int64_t ld, int K, int d, c128 *L, int LD) {
  switch ((d + 7) / 8) {
    case 1: warp_gram_dmma_nb<1, 0, 1>(P, ld, K, d, L, LD); break;
    case 2: warp_gram_dmma_nb<2, 0, 2>(P, ld, K, d, L, LD); break;
    case 3: warp_gram_dmma_nb<3, 0, 3>(P, ld, K, d, L, LD); break;
    case 4:  // 10 tiles in two passes (register budget of the 4-CTA/SM screen)
      warp_gram_dmma_nb<4, 0, 3>(P, ld, K, d, L, LD);
      warp_gram_dmma_nb<4, 3, 4>(P, ld, K, d, L, LD);
      break;
    default:  // d <= 40 (large K, cap 32 + p): 15 tiles in three passes
      warp_gram_dmma_nb<5, 0, 3>(P, ld, K, d, L, LD);
      warp_gram_dmma_nb<5, 3, 4>(P, ld, K, d, L, LD);
      warp_gram_dmma_nb<5, 4, 5>(P, ld, K, d, L, LD);
      break;
  }
}



// X row k = W row k L^-H (forward substitution, d = DD columns in registers);
// returns ||x||^2 and stores the row (stride 1) to xo.
template <int DD>
LRZ_DEV double scr_xrow(const c128 *__restrict__ wr, const c128 *L, int LD, c128 *xo) {
  c128 x[DD];
  double loc = 0.0;
#pragma unroll
  for (int j = 0; j < DD; ++j) {
    c128 acc = wr[j];
#pragma unroll
    for (int m = 0; m < j; ++m) {
      const c128 lj = L[j * LD + m];  // x_j -= x_m conj(L_jm)
      acc.re -= x[m].re * lj.re + x[m].im * lj.im;
      acc.im -= x[m].im * lj.re - x[m].re * lj.im;
    }
    x[j] = cscale(acc, 1.0 / L[j * LD + j].re);
    loc += cabs2(x[j]);
    if (xo) xo[j] = x[j];
  }
  return loc;
}

// ||column t of L^-1||^2 for a DD x DD lower-triangular L.
template <int DD>
LRZ_DEV double scr_linv_col(const c128 *L, int LD, int t) {
  c128 x[DD];
  double f = 0.0;
#pragma unroll
  for (int i = 0; i < DD; ++i) {
    if (i < t) {
      x[i] = czero<double>();
      continue;
    }
    c128 acc = mk<double>(i == t ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const c128 lk = L[i * LD + k];
      acc.re -= lk.re * x[k].re - lk.im * x[k].im;
      acc.im -= lk.re * x[k].im + lk.im * x[k].re;
    }
    x[i] = cscale(acc, 1.0 / L[i * LD + i].re);
    f += cabs2(x[i]);
  }
  return f;
}

// widths up to 24 are unrolled with x in registers; wider sketches take the
// generic loop below (x through the row's scratch), which keeps the kernel's
// register budget -- and so its occupancy -- set by the common widths
#define SCR_CASES(F)                                                                  \
  F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14) F(15) F(16) \
  F(17) F(18) F(19) F(20) F(21) F(22) F(23) F(24)

LRZ_DEV double scr_xrow_generic(int d, const c128 *wr, const c128 *L, int LD, c128 *xo) {
  double loc = 0.0;
  for (int j = 0; j < d; ++j) {
    c128 acc = wr[j];
    for (int m = 0; m < j; ++m) {
      const c128 x = xo[m], lj = L[j * LD + m];
      acc.re -= x.re * lj.re + x.im * lj.im;
      acc.im -= x.im * lj.re - x.re * lj.im;
    }
    const c128 xj = cscale(acc, 1.0 / L[j * LD + j].re);
    xo[j] = xj;
    loc += cabs2(xj);
  }
  return loc;
}

LRZ_DEV double scr_linv_col_generic(int d, const c128 *L, int LD, int t, c128 *x) {
  double f = 0.0;
  for (int i = t; i < d; ++i) {
    c128 acc = mk<double>(i == t ? 1.0 : 0.0, 0.0);
    for (int k = t; k < i; ++k) {
      const c128 lk = L[i * LD + k];
      acc.re -= lk.re * x[k].re - lk.im * x[k].im;
      acc.im -= lk.re * x[k].im + lk.im * x[k].re;
    }
    x[i] = cscale(acc, 1.0 / L[i * LD + i].re);
    f += cabs2(x[i]);
  }
  return f;
}

LRZ_DEV double scr_xrow_d(int d, const c128 *wr, const c128 *L, int LD, c128 *xo) {
  switch (d) {
#define SCR_X(n) \
  case n:        \
    return scr_xrow<n>(wr, L, LD, xo);
    SCR_CASES(SCR_X)
#undef SCR_X
  }
  return scr_xrow_generic(d, wr, L, LD, xo);
}

LRZ_DEV double scr_linv_col_d(int d, const c128 *L, int LD, int t, c128 *scratch) {
  switch (d) {
#define SCR_L(n) \
  case n:        \
    return scr_linv_col<n>(L, LD, t);
    SCR_CASES(SCR_L)
#undef SCR_L
  }
  return scr_linv_col_generic(d, L, LD, t, scratch);
}

__global__ void __launch_bounds__(128, 4) arsvd_screen_kernel(ArsvdArgs g, int64_t B, int Dtot,
                                                           const c128 *__restrict__ Yall,
                                                           const c128 *__restrict__ Wall,
                                                           c128 *__restrict__ Xs,
                                                           int32_t *__restrict__ resume) {
  extern __shared__ __align__(16) char scr_smem[];
  // (row, col) of the e-th entry of a lower triangle in row order, for the
  // Cholesky trailing updates (replaces a sqrt + correction loops per entry)
  __shared__ uint16_t s_tri[SCR_DMAX * (SCR_DMAX + 1) / 2];
  for (int e = threadIdx.x; e < SCR_DMAX * (SCR_DMAX + 1) / 2; e += blockDim.x) {
    int a = int((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    while (a * (a + 1) / 2 > e) --a;
    s_tri[e] = uint16_t((a << 8) | (e - a * (a + 1) / 2));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t item = blockIdx.x * int64_t(blockDim.x >> 5) + wib;
  if (item >= B) return;
  if (g.mask && !g.mask[item]) return;
  const int K = g.K, LD = g.D + 1;
  c128 *L = (c128 *)scr_smem + wib * g.D * LD;
  const c128 *dA = g.dA + item * g.as;
  const c128 *Y = Yall + item * int64_t(K) * Dtot;
  const c128 *W = Wall + item * int64_t(K) * Dtot;
  c128 *X = Xs + item * int64_t(K) * SCR_DMAX;
  double e2 = 0.0;
  for (int i = lane; i < K * K; i += 32) e2 += cabs2(dA[i]);
  const double energy = warp_sum(e2);
  if (energy == 0.0) {
    if (lane == 0) {
      g.k_est[item] = 0;
      g.iters[item] = 0;
      g.fallback[item] = 0;
      g.consumed[item] = 0;
      resume[item] = -1;
    }
    return;
  }
  const int64_t orw = g.orow ? int64_t(g.orow[item]) : item / g.orow_div;
  const double target = (g.eta_row ? g.eta_row[orw] : g.eta) * energy;
  int k0 = g.k_init, o = 0;
  int64_t used = 0;
  for (int it = 0; it < g.i_max; ++it) {
    const int d = min(k0 + g.p, K);
    used += int64_t(2) * K * d;
    const bool last = (it == g.i_max - 1);
    // G = Y_i^H Y_i (lower triangle), DMMA
    warp_gram_dmma(Y + o, Dtot, K, d, L, LD);
    __syncwarp();
    // Cholesky G = L L^H, warp-synchronous
    bool ok = true;
    double lmin = 1e300, lmax = 0.0;
    for (int jj = 0; jj < d; ++jj) {
      const double piv = L[jj * LD + jj].re;
      if (!(piv > 0.0)) {
        ok = false;
        break;
      }
      const double il = rsqrt(piv), l = piv * il;  // one MUFU + Newton, no divide
      lmin = fmin(lmin, l);
      lmax = fmax(lmax, l);
      __syncwarp();
      for (int a = jj + 1 + lane; a < d; a += 32) L[a * LD + jj] = cscale(L[a * LD + jj], il);
      if (lane == 0) L[jj * LD + jj] = mk<double>(l, 0.0);
      __syncwarp();
      const int n = d - jj - 1, nt = n * (n + 1) / 2;
      for (int e = lane; e < nt; e += 32) {
        const int a = s_tri[e] >> 8, b = s_tri[e] & 0xff;
        const int ra = jj + 1 + a, rb = jj + 1 + b;  // rb <= ra
        const c128 x = L[ra * LD + jj], y = L[rb * LD + jj];
        c128 &t = L[ra * LD + rb];
        t.re -= x.re * y.re + x.im * y.im;
        t.im -= x.im * y.re - x.re * y.im;
      }
      __syncwarp();
    }
    const double kap2 = ok ? (lmax / lmin) * (lmax / lmin) : 1e300;
    // CholeskyQR error bound on the captured energy (relative)
    // (kap2 comes from diag(L), a lower bound on cond(Y)^2: one more factor d covers
    // the usual gap between the diagonal ratio and cond(L))
    const double tol = 64.0 * d * d * EPS64 * kap2 + 1e-12;
    if (!ok || kap2 > 1e8) {
      if (lane == 0) {
        resume[item] = it;
        if (g.want == 2) {  // estimate only: the exact pass decides
          g.iters[item] = it + 1;
          g.consumed[item] = used;
        }
      }
      return;
    }
    // X = W_i L^-H row by row (lane = row), ||X||_F^2
    double loc = 0.0;
    for (int k = lane; k < K; k += 32)
      // X itself is only needed by the iteration-cap tail's certificate
      loc += scr_xrow_d(d, W + int64_t(k) * Dtot + o, L, LD,
                        (last || d > 24) ? X + int64_t(k) * SCR_DMAX : nullptr);
    const double mf = warp_sum(loc);
    __syncwarp();
    if (g.want == 2) {
      // cursor-resolution rounds: iteration count from the screened energy alone
      // (best estimate inside the error band; the exact pass verifies it later)
      if (mf < target && !last) {
        k0 *= 2;
        o += d;
        continue;
      }
      if (lane == 0) {
        g.iters[item] = it + 1;
        g.consumed[item] = used;
        resume[item] = it;
      }
      return;
    }
    if (mf < target * (1.0 - tol)) {  // no prefix of the spectrum reaches the target
      if (!last) {
        k0 *= 2;
        o += d;
        continue;
      }
      if (g.want == 0 && 2 * d > K && kap2 < 1e4) {
        // tail: certify sigma_min(B)^2 = lambda_min(X^H X) >= 1e-6 tr(X^H X)
        __syncwarp();  // X rows were written by other lanes
        warp_gram_dmma(X, SCR_DMAX, K, d, L, LD);
        __syncwarp();
        bool ok2 = true;
        for (int jj = 0; jj < d; ++jj) {
          const double piv = L[jj * LD + jj].re;
          if (!(piv > 0.0)) {
            ok2 = false;
            break;
          }
          const double il = rsqrt(piv), l = piv * il;  // one MUFU + Newton, no divide
          __syncwarp();
          for (int a = jj + 1 + lane; a < d; a += 32) L[a * LD + jj] = cscale(L[a * LD + jj], il);
          if (lane == 0) L[jj * LD + jj] = mk<double>(l, 0.0);
          __syncwarp();
          const int n = d - jj - 1, nt = n * (n + 1) / 2;
          for (int e = lane; e < nt; e += 32) {
            const int a = s_tri[e] >> 8, b = s_tri[e] & 0xff;
            const int ra = jj + 1 + a, rb = jj + 1 + b;
            const c128 x = L[ra * LD + jj], y = L[rb * LD + jj];
            c128 &t = L[ra * LD + rb];
            t.re -= x.re * y.re + x.im * y.im;
            t.im -= x.im * y.re - x.re * y.im;
          }
          __syncwarp();
        }
        if (ok2) {
          // ||L^-1||_F^2, column t per lane (forward substitution, kept in X's rows 0..d-1
          // is not possible: use registers)
          double f = 0.0;
          // (X is consumed by the Gram above: its rows serve as the generic path's scratch)
          for (int t = lane; t < d; t += 32)
            f += scr_linv_col_d(d, L, LD, t, X + int64_t(t) * SCR_DMAX);
          const double F = warp_sum(f);
          if (isfinite(F) && F * mf <= 1e6) {
            if (lane == 0) {
              g.k_est[item] = d;
              g.iters[item] = g.i_max;
              g.fallback[item] = 1;
              g.consumed[item] = used;
              resume[item] = -1;
            }
            return;
          }
        }
      }
      if (lane == 0) resume[item] = it;
      return;
    }
    if (lane == 0) resume[item] = it;  // a hit is possible: exact SVD on this iteration
    return;
  }
}


// ---------------------------------------------------------------------------
// Cursor walk (K <= 32, sketch widths <= 24).  In the reference the sketch
// stream is consumed sequentially across steps, and a step's consumption is
// fixed by its iteration count alone: iteration i hits iff cumsum(s^2) reaches
// eta ||dA||^2 for some prefix, i.e. iff the total ||B_i||_F^2 = ||Q_i^H dA||_F^2
// does (lowrank.py:289-300).  That total is what the CholeskyQR screen
// computes, so one warp per trial can walk its steps in order with only the
// sketch GEMMs (DMMA), the sketch Gram (DMMA), a warp Cholesky and the X rows
// -- no QR / SVD -- and fix every step's cursor and iteration count.  The
// exact factors are then computed for all steps in one batched speculative
// pass at the now-known cursors.  A step whose total is within the CholeskyQR
// error bound of the target (or ill-conditioned, or past the window) stops the
// walk there; the verifier then finds the first misprediction and the in-order
// exact path takes over from it.
// ---------------------------------------------------------------------------
constexpr int WK_LD = 33;   // row stride (complex) of the K x K / K x d shared tiles
constexpr int WK_DMAX = 24;

// C (K x NB*8) = A (K x K) B (K x NB*8), all complex128 in shared memory
// (row strides WK_LD), K <= 32 (zero padded to 32), one warp on DMMA.
template <int NB>
LRZ_DEV void warp_zgemm_dmma(const c128 *A, const c128 *Bm, c128 *C) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double cr[4][NB][2], ci[4][NB][2];
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < NB; ++cb) cr[rb][cb][0] = cr[rb][cb][1] = ci[rb][cb][0] = ci[rb][cb][1] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double br[NB], bi[NB];
#pragma unroll
    for (int cb = 0; cb < NB; ++cb) {
      const c128 v = Bm[(4 * c + t) * WK_LD + 8 * cb + g];
      br[cb] = v.re;
      bi[cb] = v.im;
    }
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) {
      const c128 a = A[(8 * rb + g) * WK_LD + 4 * c + t];
      const double nai = -a.im;
#pragma unroll
      for (int cb = 0; cb < NB; ++cb) {
        dmma(cr[rb][cb], a.re, br[cb]);  // (ar + i ai)(br + i bi)
        dmma(cr[rb][cb], nai, bi[cb]);
        dmma(ci[rb][cb], a.re, bi[cb]);
        dmma(ci[rb][cb], a.im, br[cb]);
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int cb = 0; cb < NB; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        C[(8 * rb + g) * WK_LD + 8 * cb + 2 * t + e] = mk<double>(cr[rb][cb][e], ci[rb][cb][e]);
  __syncwarp();
}

LRZ_DEV void warp_zgemm(const c128 *A, const c128 *Bm, c128 *C, int d) {
  switch ((d + 7) / 8) {
    case 1: warp_zgemm_dmma<1>(A, Bm, C); break;
    case 2: warp_zgemm_dmma<2>(A, Bm, C); break;
    default: warp_zgemm_dmma<3>(A, Bm, C); break;
  }
}

// Warp Cholesky of the lower triangle of L (d x d, row stride LD) in place;
// (lmin, lmax) of the diagonal of the factor.  False on a non-positive pivot.
LRZ_DEV bool warp_chol_tri(c128 *L, int d, int LD, const uint16_t *tri, double &lmin,
                           double &lmax) {
  const int lane = threadIdx.x & 31;
  lmin = 1e300;
  lmax = 0.0;
  for (int jj = 0; jj < d; ++jj) {
    const double piv = L[jj * LD + jj].re;
    if (!(piv > 0.0)) return false;
    const double il = rsqrt(piv), l = piv * il;  // one MUFU + Newton, no divide
    lmin = fmin(lmin, l);
    lmax = fmax(lmax, l);
    __syncwarp();
    for (int a = jj + 1 + lane; a < d; a += 32) L[a * LD + jj] = cscale(L[a * LD + jj], il);
    if (lane == 0) L[jj * LD + jj] = mk<double>(l, 0.0);
    __syncwarp();
    const int n = d - jj - 1, nt = n * (n + 1) / 2;
    for (int e = lane; e < nt; e += 32) {
      const int a = tri[e] >> 8, b = tri[e] & 0xff;
      const int ra = jj + 1 + a, rb = jj + 1 + b;
      const c128 x = L[ra * LD + jj], y = L[rb * LD + jj];
      c128 &t = L[ra * LD + rb];
      t.re -= x.re * y.re + x.im * y.im;
      t.im -= x.im * y.re - x.re * y.im;
    }
    __syncwarp();
  }
  return true;
}

LRZ_DEV void wk_cp16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
LRZ_DEV void wk_cp8(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
LRZ_DEV void wk_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
LRZ_DEV void wk_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// dA of step bt into a zero-padded [32][WK_LD] tile (one cp.async group)
LRZ_DEV void wk_prefetch_dA(const ArsvdArgs &g, int64_t bt, c128 *dst) {
  const int lane = threadIdx.x & 31, K = g.K;
  const c128 *src = g.dA + bt * int64_t(K) * K;
  for (int e = lane; e < K * K; e += 32) {
    const int r = e / K, c = e - r * K;
    wk_cp16(dst + r * WK_LD + c, src + e);
  }
  wk_commit();
}

__global__ void __launch_bounds__(32)
    arsvd_walk_kernel(ArsvdArgs g, int T, const uint8_t *__restrict__ is_sketch,
                      const int32_t *__restrict__ first, int64_t *__restrict__ cursor,
                      int32_t *__restrict__ iters_pred) {
  extern __shared__ __align__(16) char wk_smem[];
  c128 *Abuf = (c128 *)wk_smem;          // dA, two steps [2][32][WK_LD] (next step prefetched)
  c128 *Os = Abuf + 2 * 32 * WK_LD;      // Omega_i     [32][WK_LD]
  c128 *Ys = Os + 32 * WK_LD;            // Y = dA Omega
  c128 *Ws = Ys + 32 * WK_LD;            // W = dA Y
  c128 *L = Ws + 32 * WK_LD;             // [WK_DMAX][WK_DMAX + 1]
  __shared__ uint16_t tri[WK_DMAX * (WK_DMAX + 1) / 2];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < WK_DMAX * (WK_DMAX + 1) / 2; e += 32) {
    int a = int((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    while (a * (a + 1) / 2 > e) --a;
    tri[e] = uint16_t((a << 8) | (e - a * (a + 1) / 2));
  }
  __syncwarp();
  const int64_t b = blockIdx.x;
  const int K = g.K, LDL = WK_DMAX + 1;
  const double SQH = 0.7071067811865476;
  const double *om = g.omega + b * g.os;
  const double eta = g.eta_row ? g.eta_row[b] : g.eta;
  int t = first[b];
  if (t >= T) return;
  int64_t cur = cursor[b * T + t];
  // the padding of both dA tiles stays zero; the valid K x K block of step t + 1
  // is fetched with cp.async while step t runs (the walk is latency bound)
  for (int e = lane; e < 3 * 32 * WK_LD; e += 32) Abuf[e] = czero<double>();  // dA x 2, Omega
  __syncwarp();
  int cb = 0;
  wk_prefetch_dA(g, b * T + t, Abuf);
  for (; t < T; ++t, cb ^= 1) {
    const int64_t bt = b * T + t;
    cursor[bt] = cur;
    if (t + 1 < T) wk_prefetch_dA(g, bt + 1, Abuf + (cb ^ 1) * 32 * WK_LD);
    else wk_commit();
    // this step's tile has landed (the next one may be in flight); waited for
    // on skipped steps too, so no two copies into one tile are ever in flight
    wk_wait<1>();
    __syncwarp();
    if (!is_sketch[bt]) continue;
    const c128 *As = Abuf + cb * 32 * WK_LD;
    double e2 = 0.0;
    for (int e = lane; e < 32 * 32; e += 32) e2 += cabs2(As[(e >> 5) * WK_LD + (e & 31)]);
    const double energy = warp_sum(e2);
    if (energy == 0.0) {  // empty factor: no sketch drawn (lowrank.py:275-276)
      if (lane == 0) iters_pred[bt] = 0;
      continue;
    }
    const double target = eta * energy;
    int k0 = g.k_init, iters = -1;
    int64_t used = 0;
    bool undecided = false;
    for (int it = 0; it < g.i_max; ++it) {
      const int d = min(k0 + g.p, K);
      if (g.omega_len > 0 && cur + used + int64_t(2) * K * d > g.omega_len) {
        undecided = true;  // the exact path reports the short window
        break;
      }
      const double *zre = om + cur + used, *zim = zre + int64_t(K) * d;
      // Omega_i lands straight in its tile (re / im halves by 8-byte cp.async,
      // every copy in flight at once), then each lane scales the entries it
      // copied by sqrt(1/2) and clears the pad columns d .. 8 ceil(d / 8)
      const int nz = K * d;
      const float inv_d = 1.0f / float(d);
      for (int e = lane; e < nz; e += 32) {
        const int r = int((float(e) + 0.5f) * inv_d), c = e - r * d;  // exact: e < 1024
        c128 *o = Os + r * WK_LD + c;
        wk_cp8(&o->re, zre + e);
        wk_cp8(&o->im, zim + e);
      }
      wk_commit();
      const int dpad = 8 * ((d + 7) / 8);
      for (int e = lane; e < 32 * (dpad - d); e += 32) {
        const int r = e / (dpad - d), c = d + e - r * (dpad - d);
        Os[r * WK_LD + c] = czero<double>();
      }
      wk_wait<0>();
      for (int e = lane; e < nz; e += 32) {
        const int r = int((float(e) + 0.5f) * inv_d), c = e - r * d;
        c128 &o = Os[r * WK_LD + c];
        o = mk<double>(SQH * o.re, SQH * o.im);
      }
      __syncwarp();
      warp_zgemm(As, Os, Ys, d);   // Y = dA Omega (lowrank.py:288)
      warp_zgemm(As, Ys, Ws, d);   // W = dA Y = (Q^H dA)^H L^H-scaled
      warp_gram_dmma(Ys, WK_LD, K, d, L, LDL);
      __syncwarp();
      double lmin, lmax;
      const bool ok = warp_chol_tri(L, d, LDL, tri, lmin, lmax);
      const double kap2 = ok ? (lmax / lmin) * (lmax / lmin) : 1e300;
      if (!ok || kap2 > 1e8) {
        undecided = true;
        break;
      }
      double loc = 0.0;
      for (int k = lane; k < K; k += 32) loc += scr_xrow_d(d, Ws + k * WK_LD, L, LDL, nullptr);
      const double mf = warp_sum(loc);
      const double tol = 64.0 * d * d * EPS64 * kap2 + 1e-12;
      used += int64_t(2) * K * d;
      if (mf < target * (1.0 - tol)) {  // certainly no hit: next, wider sketch
        k0 *= 2;
        continue;
      }
      if (mf > target * (1.0 + tol)) {  // certainly a hit at this iteration
        iters = it + 1;
        break;
      }
      undecided = true;  // within the rounding bound of the target
      break;
    }
    if (undecided) {  // later predictions stay; the verifier finds the first miss
      wk_wait<0>();
      return;
    }
    if (iters < 0) iters = g.i_max;  // iteration cap: all sketches drawn
    if (lane == 0) iters_pred[bt] = iters;
    cur += used;
    __syncwarp();  // every lane is done with this tile before it is refilled
  }
  wk_wait<0>();
}

}  // namespace lrz

using namespace lrz;

extern "C" int lrz_cgemm(int dtype, int64_t batch, int M, int N, int Kd, int opA, const void *A,
                         int64_t lda, int64_t sA, int opB, const void *Bm, int64_t ldb,
                         int64_t sB, void *C, int64_t ldc, int64_t sC, void *stream);

// Threads per item of the exact kernel: small problems are latency bound (barrier
// and scalar chains per reflector / Jacobi round), so K <= 32 runs narrow CTAs
// and many items per SM instead of one wide CTA per item.
static int arsvd_threads(int K) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("LRZ_ARSVD_THREADS");
    env = e ? atoi(e) : 0;
  }
  if (env >= 32 && env <= ARSVD_THREADS && env % 32 == 0) return env;
  return K <= 32 ? 96 : ARSVD_THREADS;
}

size_t lrz_arsvd_ws(int64_t B, int K, int D) {
  return size_t(B) * (size_t(2) * D * K + size_t(D) * D) * sizeof(c128);
}
// plus the screening front end: resume index, three [B][K][max(Dtot, SCR_DMAX)] blocks and
// the tail-pipeline flags
size_t lrz_arsvd_ws_total(int64_t B, int K, int D) {
  const size_t dt = size_t(std::max(4 * D, SCR_DMAX));  // >= max(Dtot, SCR_DMAX) (Dtot <= 4 D)
  return lrz_arsvd_ws(B, K, D) + ((size_t(B) * sizeof(int32_t) + 255) & ~size_t(255)) +
         3 * size_t(B) * K * dt * sizeof(c128) + ((size_t(B) + 255) & ~size_t(255));
}

extern "C" int lrz_arsvd(int64_t B, int K, const void *dA, int64_t a_stride,
                         const double *omega, int64_t omega_stride, const int32_t *omega_row,
                         const int64_t *cursor, const lrz_arsvd_cfg *cfg, void *U, void *V,
                         double *S, int32_t *k_est, int32_t *iters, int32_t *fallback,
                         int64_t *consumed, const uint8_t *item_mask, int want_factor,
                         int hermitian, void *workspace, void *stream) {
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
  g.orow_div = 1;
  g.cursor = cursor;
  g.eta = cfg->eta;
  g.eta_row = cfg->eta_row;
  g.omega_len = cfg->omega_len;
  g.k_init = cfg->k_init;
  g.p = cfg->p;
  g.i_max = cfg->i_max;
  g.D = cfg->d_max;
  g.want = want_factor;
  g.start_it = nullptr;
  g.ya = nullptr;
  g.ydtot = 0;
  g.phase = 0;
  g.smem_ws = 0;
  g.smem_j = 0;
  g.tail = nullptr;
  g.U = (c128 *)U;
  g.V = (c128 *)V;
  g.S = S;
  g.k_est = k_est;
  g.iters = iters;
  g.fallback = fallback;
  g.consumed = consumed;
  g.mask = item_mask;
  g.ws = (c128 *)workspace;
  cudaStream_t st = (cudaStream_t)stream;
  int Dtot = 0;
  {
    long long kk = cfg->k_init;
    for (int i = 0; i < cfg->i_max; ++i) {
      Dtot += (int)std::min<long long>(kk + cfg->p, K);
      kk *= 2;
    }
  }
  // the front end reads every iteration's block: only when the window holds them
  const bool whole = cfg->omega_len <= 0 ||
                     [&] {
                       long long kk = cfg->k_init, need = 0;
                       for (int i = 0; i < cfg->i_max; ++i) {
                         need += 2LL * K * std::min<long long>(kk + cfg->p, K);
                         kk *= 2;
                       }
                       return need <= cfg->omega_len;
                     }();
  const bool front_ok = hermitian && g.D <= SCR_DMAX && Dtot <= 4 * g.D && whole;
  if (want_factor == 2 && !front_ok) {
    lrz_set_error("lrz_arsvd: screen-only mode needs the screening front end (hermitian dA, "
                  "d_max <= %d, the whole sketch window)", (int)SCR_DMAX);
    return LRZ_EINVAL;
  }
  if (front_ok && want_factor != 1) {
    // screening front end (see arsvd_screen_kernel); workspace layout after the
    // CTA kernel's part: resume[B] int32 | Om/X [B][K][Dtot] | Y [B][K][Dtot] | W
    char *wp = (char *)workspace + lrz_arsvd_ws(B, K, cfg->d_max);
    int32_t *resume = (int32_t *)wp;
    wp += (size_t(B) * sizeof(int32_t) + 255) & ~size_t(255);
    const size_t blk = size_t(B) * K * std::max(Dtot, (int)SCR_DMAX) * sizeof(c128);
    c128 *Om = (c128 *)wp;
    c128 *Ya = (c128 *)(wp + blk);
    c128 *Wa = (c128 *)(wp + 2 * blk);
    // Y = dA Omega_all; for K <= 32 the same kernel also forms W = dA Y per tile;
    // K > 32: Omega gathered, both products on the FP64 tensor pipe (dmma_tiled.cu)
    const bool large_dmma = K > 32 && lrz_use_dmma();
    int rc = large_dmma
                 ? lrz_sketch_dmma_large(B, K, Dtot, dA, a_stride, omega, omega_stride,
                                         omega_row, 1, cursor, cfg->k_init, cfg->p, item_mask,
                                         Om, Ya, Wa, st)
                 : lrz_sketch_gemm(B, K, Dtot, dA, a_stride, omega, omega_stride, omega_row, 1,
                                   cursor, cfg->k_init, cfg->p, item_mask, Ya,
                                   K <= 32 ? Wa : nullptr, stream);
    if (rc) return rc;
    if (K > 32 && !large_dmma) {
      rc = lrz_cgemm(LRZ_C128, B, K, Dtot, K, 0, dA, K, a_stride, 0, Ya, Dtot, int64_t(K) * Dtot,
                     Wa, Dtot, int64_t(K) * Dtot, stream);
      if (rc) return rc;
    }
    const size_t sm = 4 * size_t(g.D) * (g.D + 1) * sizeof(c128);
    if (cudaFuncSetAttribute(arsvd_screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sm)) != cudaSuccess) {
      lrz_set_error("lrz_arsvd: cannot reserve %zu bytes of shared memory", sm);
      return LRZ_ELAUNCH;
    }
    {
      LrzProf prof("arsvd_screen_kernel", st);
      arsvd_screen_kernel<<<unsigned((B + 3) / 4), 128, sm, st>>>(g, B, Dtot, Ya, Wa, Om,
                                                                  resume);
    }
    if (want_factor == 2) return lrz_launch_status("lrz_arsvd (screen only)");
    g.start_it = resume;
    g.ya = Ya;
    g.ydtot = Dtot;
    if (large_dmma && g.D == dneed) {
      // tail pipeline: the two K^2 d products of the resumed last iteration as
      // batched DMMA GEMMs (dmma_tiled.cu) between the two halves of the item
      g.tail = (uint8_t *)(wp + 3 * blk);
      g.phase = 1;
      cudaMemsetAsync(g.tail, 0, size_t(B), st);
      {
        LrzProf prof("arsvd_kernel", st);
        static int p1_small = -1;
        if (p1_small < 0) {
          const char *e = getenv("LRZ_ARSVD_P1_SMALL");
          p1_small = e ? atoi(e) : 128;  // d <= 32: C3 2.80 -> 2.45 ms, C4 7.98 -> 7.47 ms
        }
        if (p1_small && g.D <= 32)
          arsvd_small_kernel<6><<<unsigned(B), p1_small, 0, st>>>(g);
        else
          arsvd_kernel<<<unsigned(B), ARSVD_THREADS, 0, st>>>(g);
      }
      if (int rc2 = lrz_launch_status("arsvd_kernel (phase 1)")) return rc2;
      const int64_t wst = int64_t(2) * g.D * K + int64_t(g.D) * g.D;
      c128 *w0 = (c128 *)workspace;
      if (int rc2 = lrz_arsvd_tail_M(B, K, g.D, dA, a_stride, w0 + int64_t(g.D) * K, w0, wst,
                                     g.tail, st))
        return rc2;
      g.phase = 2;
      {
        const size_t dj = size_t(2) * g.D * g.D * sizeof(c128);
        const bool sj = K >= 64 && dj <= 96 * 1024;
        if (sj) {
          g.smem_j = 1;
          cudaFuncSetAttribute(arsvd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(dj));
        }
        LrzProf prof("arsvd_kernel:tail", st);
        static int tail_small = -1;
        if (tail_small < 0) {
          const char *e = getenv("LRZ_ARSVD_TAIL_SMALL");
          tail_small = e ? atoi(e) : 96;
        }
        if (tail_small && g.D <= 32) {
          // narrow items, more of them per SM (the d x d Jacobi is latency bound):
          // C3 (K 64, d 21) 8.5 -> 6.5 ms per 12,800 items at 96 threads
          if (sj)
            cudaFuncSetAttribute(arsvd_small_kernel<6>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(dj));
          arsvd_small_kernel<6><<<unsigned(B), tail_small, sj ? dj : 0, st>>>(g);
        } else {  // (d = 37 at C5: 1280 items, 128-192 thread items measured no faster)
          arsvd_kernel<<<unsigned(B), ARSVD_THREADS, sj ? dj : 0, st>>>(g);
        }
        g.smem_j = 0;
      }
      if (int rc2 = lrz_launch_status("arsvd_kernel (phase 2)")) return rc2;
      return lrz_arsvd_tail_U(B, K, g.D, w0, w0 + int64_t(g.D) * K, wst, U, g.tail, st);
    }
  }
  size_t dyn = 0;
  {
    const size_t need = (size_t(2) * g.D * K + size_t(g.D) * g.D) * sizeof(c128);
    static int use_smem = -1;
    if (use_smem < 0) {
      const char *e = getenv("LRZ_ARSVD_SMEM");
      use_smem = e ? atoi(e) : 1;
    }
    if (use_smem && need <= 48 * 1024) {
      g.smem_ws = 1;
      dyn = need;
    }
  }
  LrzProf prof("arsvd_kernel", st);
  if (arsvd_threads(K) <= 128 && g.D <= 32 && K <= 32) {
    static int ctas = -1;
    if (ctas < 0) {
      const char *e = getenv("LRZ_ARSVD_CTAS");
      ctas = e ? atoi(e) : 6;
    }
    auto launch = [&](auto kern) {
      if (dyn) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
      kern<<<unsigned(B), arsvd_threads(K), dyn, st>>>(g);
    };
    if (ctas >= 8) launch(arsvd_small_kernel<8>);
    else if (ctas >= 6) launch(arsvd_small_kernel<6>);
    else launch(arsvd_small_kernel<4>);
  } else {
    if (dyn) cudaFuncSetAttribute(arsvd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(dyn));
    arsvd_kernel<<<unsigned(B), arsvd_threads(K), dyn, st>>>(g);
  }
  return lrz_launch_status("lrz_arsvd");
}

extern "C" int lrz_arsvd_seq(int64_t B, int T, int K, const void *dA, const double *omega,
                             int64_t omega_stride, const lrz_arsvd_cfg *cfg,
                             const uint8_t *is_sketch, const int32_t *first_unverified,
                             int64_t *cursor, int32_t *iters_pred, void *U, void *V, double *S,
                             int32_t *k_est, int32_t *iters, int32_t *fallback, int64_t *consumed,
                             int want_factor, void *workspace, void *stream) {
  if (B < 0 || T < 1 || K < 1 || !dA || !omega || !cfg || !is_sketch || !first_unverified ||
      !cursor || !iters_pred || !U || !V || !S || !k_est || !iters || !fallback || !consumed ||
      !workspace) {
    lrz_set_error("lrz_arsvd_seq: bad arguments");
    return LRZ_EINVAL;
  }
  if (!(cfg->eta > 0.0 && cfg->eta <= 1.0) || cfg->k_init < 1 || cfg->p < 0 || cfg->i_max < 1 ||
      cfg->d_max < 1 || cfg->d_max > ARSVD_DMAX) {
    lrz_set_error("lrz_arsvd_seq: bad ArSvdConfig");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  ArsvdArgs g;
  g.K = K;
  g.dA = (const c128 *)dA;
  g.as = int64_t(K) * K;
  g.omega = omega;
  g.os = omega_stride;
  g.orow = nullptr;
  g.orow_div = T;
  g.cursor = nullptr;
  g.eta = cfg->eta;
  g.eta_row = cfg->eta_row;
  g.omega_len = cfg->omega_len;
  g.k_init = cfg->k_init;
  g.p = cfg->p;
  g.i_max = cfg->i_max;
  g.D = cfg->d_max;
  g.want = want_factor;
  g.start_it = nullptr;
  g.ya = nullptr;
  g.ydtot = 0;
  g.phase = 0;
  g.smem_ws = 0;
  g.smem_j = 0;
  g.tail = nullptr;
  g.U = (c128 *)U;
  g.V = (c128 *)V;
  g.S = S;
  g.k_est = k_est;
  g.iters = iters;
  g.fallback = fallback;
  g.consumed = consumed;
  g.mask = nullptr;
  g.ws = (c128 *)workspace;
  LrzProf prof("arsvd_seq_kernel", (cudaStream_t)stream);
  arsvd_seq_kernel<<<unsigned(B), ARSVD_THREADS, 0, (cudaStream_t)stream>>>(
      g, T, is_sketch, first_unverified, cursor, iters_pred);
  return lrz_launch_status("lrz_arsvd_seq");
}

extern "C" int lrz_arsvd_walk(int64_t B, int T, int K, const void *dA, const double *omega,
                              int64_t omega_stride, const lrz_arsvd_cfg *cfg,
                              const uint8_t *is_sketch, const int32_t *first_unverified,
                              int64_t *cursor, int32_t *iters_pred, void *stream) {
  if (B < 0 || T < 1 || K < 1 || K > 32 || !dA || !omega || !cfg || !is_sketch ||
      !first_unverified || !cursor || !iters_pred) {
    lrz_set_error("lrz_arsvd_walk: bad arguments (K <= 32)");
    return LRZ_EINVAL;
  }
  long long kk = cfg->k_init;
  for (int i = 0; i < cfg->i_max; ++i) {
    if (std::min<long long>(kk + cfg->p, K) > WK_DMAX) {
      lrz_set_error("lrz_arsvd_walk: sketch widths must be <= %d", WK_DMAX);
      return LRZ_EINVAL;
    }
    kk *= 2;
  }
  if (B == 0) return LRZ_OK;
  ArsvdArgs g{};
  g.K = K;
  g.dA = (const c128 *)dA;
  g.as = int64_t(K) * K;
  g.omega = omega;
  g.os = omega_stride;
  g.orow = nullptr;
  g.orow_div = T;
  g.eta = cfg->eta;
  g.eta_row = cfg->eta_row;
  g.omega_len = cfg->omega_len;
  g.k_init = cfg->k_init;
  g.p = cfg->p;
  g.i_max = cfg->i_max;
  g.D = cfg->d_max;
  const size_t sm = (5 * 32 * WK_LD + WK_DMAX * (WK_DMAX + 1)) * sizeof(c128);
  if (cudaFuncSetAttribute(arsvd_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(sm)) != cudaSuccess) {
    lrz_set_error("lrz_arsvd_walk: cannot reserve %zu bytes of shared memory", sm);
    return LRZ_ELAUNCH;
  }
  LrzProf prof("arsvd_walk_kernel", (cudaStream_t)stream);
  arsvd_walk_kernel<<<unsigned(B), 32, sm, (cudaStream_t)stream>>>(g, T, is_sketch,
                                                                   first_unverified, cursor,
                                                                   iters_pred);
  return lrz_launch_status("lrz_arsvd_walk");
}
