// Hybrid LEO pass on the device (SURVEY.md 8(f) "next" #3 and #4):
//
//   leo_snapshot_kernel   one CTA per (trial, step): pass geometry, manifold
//                         rows, DFT beam powers, greedy beam choice, and the
//                         two K x N_RF products the precoder and the rate need
//                         (reference channel.py:236-289, 128-137, 176-233,
//                         352-392; harness.py:221-226)
//   hybrid_rate_kernel    one CTA per (trial, step): RZF with analog beams,
//                         ||F_RF F_raw||_F power normalisation, coupling
//                         matrix and sum-rate (precoding.py:37-80)
//   campaign_reduce       one warp per trial: cost / rank / decision totals
//                         with the harness's accounting (harness.py:227-251)
//
// Neither the K x N channel nor F_RF ever reaches HBM: the snapshot kernel
// keeps one user row at a time in shared memory, F_RF is regenerated from the
// two DFT factors (kron, channel.py:176-190) and only the K x N_RF products
// H~ F_RF and H F_RF are written -- 2 K N_RF complex128 per step.

#include <climits>

#include "common.cuh"

namespace lrz {

constexpr int LEO_THREADS = 256;
constexpr int LEO_NMAX = 2048;      // elements per array (smem: 3 rows of N complex128)

struct Geo {
  double kx, ky, kz;   // wave vector in the array frame (channel.py:132-135)
  double gain;         // LOS amplitude gain (channel.py:366-368)
  bool below;
};

// channel.py:242-289 for one UT at pass time ts, every product/sum rounded
// separately in numpy's order.
LRZ_DEV Geo ut_geometry(const lrz_leo_cfg &c, const double *u, double ts) {
  const double R = c.orbit_radius;
  const double ang = __dmul_rn(c.orbit_rate, __dsub_rn(ts, __ddiv_rn(c.pass_s, 2.0)));
  double sa, ca;
  sincos(ang, &sa, &ca);
  const double sat0 = __dmul_rn(R, ca), sat1 = __dmul_rn(R, sa), sat2 = 0.0;
  const double xb0 = -sa, xb1 = ca, xb2 = 0.0;
  const double zb0 = __ddiv_rn(-sat0, R), zb1 = __ddiv_rn(-sat1, R), zb2 = __ddiv_rn(-sat2, R);
  // y_b = z_b x x_b
  const double yb0 = __dsub_rn(__dmul_rn(zb1, xb2), __dmul_rn(zb2, xb1));
  const double yb1 = __dsub_rn(__dmul_rn(zb2, xb0), __dmul_rn(zb0, xb2));
  const double yb2 = __dsub_rn(__dmul_rn(zb0, xb1), __dmul_rn(zb1, xb0));
  const double d0 = __dsub_rn(u[0], sat0), d1 = __dsub_rn(u[1], sat1), d2 = __dsub_rn(u[2], sat2);
  const double sl = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
  const double h0 = __ddiv_rn(d0, sl), h1 = __ddiv_rn(d1, sl), h2 = __ddiv_rn(d2, sl);
  auto dot3 = [](double a0, double a1, double a2, double b0, double b1, double b2) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
  };
  const double ux = dot3(h0, h1, h2, xb0, xb1, xb2);
  const double uy = dot3(h0, h1, h2, yb0, yb1, yb2);
  const double uz = dot3(h0, h1, h2, zb0, zb1, zb2);
  const double theta = acos(fmin(fmax(uz, -1.0), 1.0));
  const double phi = atan2(uy, ux);
  const double pn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(u[0], u[0]), __dmul_rn(u[1], u[1])),
                                   __dmul_rn(u[2], u[2])));
  const double se = __ddiv_rn(dot3(__ddiv_rn(u[0], pn), __ddiv_rn(u[1], pn), __ddiv_rn(u[2], pn),
                                   -d0, -d1, -d2), sl);
  const double el = asin(fmin(fmax(se, -1.0), 1.0));
  const double fs = __dmul_rn(20.0, log10(__ddiv_rn(__dmul_rn(4.0 * 3.141592653589793, sl),
                                                    c.wavelength)));
  Geo g;
  g.gain = pow(10.0, __ddiv_rn(__dsub_rn(__dsub_rn(u[3], fs), c.atm_loss_dB), 20.0));
  const double kap = __ddiv_rn(2.0 * 3.141592653589793, c.wavelength);
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double st = sin(theta);
  g.kx = __dmul_rn(kap, __dmul_rn(st, cp));
  g.ky = __dmul_rn(kap, __dmul_rn(st, sp));
  g.kz = __dmul_rn(kap, cos(theta));
  g.below = el < c.min_elev_rad;
  return g;
}

// conjugated unit-gain manifold entry m (channel.py:128-137)
LRZ_DEV c128 manifold_entry(const lrz_leo_cfg &c, const Geo &g, int m, double rsqrtN_div) {
  const int ix = m / c.n_y, iy = m % c.n_y;
  const double x = __dmul_rn(double(ix) - (c.n_x - 1) / 2.0, c.spacing_m);
  const double y = __dmul_rn(double(iy) - (c.n_y - 1) / 2.0, c.spacing_m);
  const double ph = __dadd_rn(__dadd_rn(__dmul_rn(g.kx, x), __dmul_rn(g.ky, y)), __dmul_rn(g.kz, 0.0));
  double s, co;
  sincos(ph, &s, &co);
  return mk<double>(__ddiv_rn(co, rsqrtN_div), __ddiv_rn(-s, rsqrtN_div));
}

// numpy complex product (ar br - ai bi, ar bi + ai br), no contraction
LRZ_DEV c128 cmul_np(c128 a, c128 b) {
  return mk<double>(__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
                    __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re)));
}

// (value, index) argmax with ties to the lower index -- np.argsort(-p, kind="stable")[0]
LRZ_DEV void arg_better(double &v, int &i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}
LRZ_DEV int block_argmax(double v, int i, double *rv, int *ri) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    arg_better(v, i, v2, i2);
  }
  __syncthreads();
  if (lane == 0) {
    rv[w] = v;
    ri[w] = i;
  }
  __syncthreads();
  double bv = rv[0];
  int bi = ri[0];
  for (int k = 1; k < nw; ++k) arg_better(bv, bi, rv[k], ri[k]);
  return bi;
}

__global__ void __launch_bounds__(LEO_THREADS)
leo_snapshot_kernel(lrz_leo_cfg c, int64_t B, int t0, int T, const double *__restrict__ ut,
                    const c128 *__restrict__ dft, const double *__restrict__ nlos,
                    int64_t nlos_stride, c128 *__restrict__ H_eff, c128 *__restrict__ H_rf,
                    int32_t *__restrict__ cols_out, int32_t *__restrict__ info,
                    c128 *__restrict__ H_full, c128 *__restrict__ H_tl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = c.K, nx = c.n_x, ny = c.n_y, N = nx * ny, R = c.N_RF;
  const int64_t item = blockIdx.x;
  const int64_t b = item / T;
  const int t = t0 + int(item % T);
  c128 *Dx = (c128 *)smem_raw;            // nx*nx
  c128 *Dy = Dx + nx * nx;                // ny*ny
  c128 *row = Dy + ny * ny;               // N: H~ row
  c128 *tmp = row + N;                    // N: DFT stage / H row
  double *pw = (double *)(tmp + N);       // N: best-over-UTs power (fill)
  unsigned char *used = (unsigned char *)(pw + N);      // N
  __shared__ Geo geo_sel[64], geo_now[64];
  __shared__ int cols[256];
  __shared__ double rv[LEO_THREADS / 32];
  __shared__ int ri[LEO_THREADS / 32];
  __shared__ int below;

  const double *U = ut + b * K * 5;
  const int tsel = t - t % c.beam_hold;
  const double sqrtN = sqrt(double(N));
  for (int i = threadIdx.x; i < nx * nx; i += blockDim.x) Dx[i] = dft[i];
  for (int i = threadIdx.x; i < ny * ny; i += blockDim.x) Dy[i] = dft[nx * nx + i];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    used[i] = 0;
    pw[i] = -INFINITY;
  }
  if (threadIdx.x == 0) below = 0;
  __syncthreads();
  for (int n = threadIdx.x; n < K; n += blockDim.x) {
    geo_now[n] = ut_geometry(c, U + n * 5, __dmul_rn(double(t), c.dt));
    geo_sel[n] = tsel == t ? geo_now[n] : ut_geometry(c, U + n * 5, __dmul_rn(double(tsel), c.dt));
    if (geo_now[n].below) atomicOr(&below, 1);
  }
  __syncthreads();

  // 1. greedy beam choice on the powers at step tsel (channel.py:202-233)
  for (int n = 0; n < K; ++n) {
    for (int m = threadIdx.x; m < N; m += blockDim.x) row[m] = manifold_entry(c, geo_sel[n], m, sqrtN);
    __syncthreads();
    for (int e = threadIdx.x; e < N; e += blockDim.x) {      // along y: tmp[ix][jy]
      const int ix = e / ny, jy = e % ny;
      c128 a = czero<double>();
      for (int iy = 0; iy < ny; ++iy) cfma(a, row[ix * ny + iy], Dy[iy * ny + jy]);
      tmp[e] = a;
    }
    __syncthreads();
    double bv = -INFINITY;
    int bi = INT_MAX;
    for (int e = threadIdx.x; e < N; e += blockDim.x) {      // along x, power, argmax
      const int jx = e / ny, jy = e % ny;
      c128 a = czero<double>();
      for (int ix = 0; ix < nx; ++ix) cfma(a, Dx[ix * nx + jx], tmp[ix * ny + jy]);
      const double h = hypot(a.re, a.im);
      const double p = h * h;
      pw[e] = fmax(pw[e], p);
      if (!used[e]) arg_better(bv, bi, p, e);
    }
    int j = block_argmax(bv, bi, rv, ri);
    if (threadIdx.x == 0) {
      if (j == INT_MAX)
        for (j = 0; used[j]; ++j) {
        }
      used[j] = 1;
      cols[n] = j;
    }
    __syncthreads();
  }
  for (int f = K; f < R; ++f) {   // leftover RF chains: best-over-UTs power
    double bv = -INFINITY;
    int bi = INT_MAX;
    for (int e = threadIdx.x; e < N; e += blockDim.x)
      if (!used[e]) arg_better(bv, bi, pw[e], e);
    int j = block_argmax(bv, bi, rv, ri);
    if (threadIdx.x == 0) {
      if (j == INT_MAX)
        for (j = 0; used[j]; ++j) {
        }
      used[j] = 1;
      cols[f] = j;
    }
    __syncthreads();
  }

  // 2. H_eff = H~ F_RF and H_rf = H F_RF at step t, one user row at a time
  const int blk0 = t0 / c.nlos_block;
  const double *S = nlos + b * nlos_stride + int64_t(t / c.nlos_block - blk0) * 2 * K * N;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int n = 0; n < K; ++n) {
    const Geo g = geo_now[n];
    const double kl = U[n * 5 + 4];
    const double wl = sqrt(__ddiv_rn(kl, __dadd_rn(kl, 1.0)));
    const double wn = sqrt(__ddiv_rn(1.0, __dadd_rn(kl, 1.0)));
    const double gn = __ddiv_rn(g.gain, sqrtN);
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      const c128 h = manifold_entry(c, g, m, sqrtN);
      row[m] = h;
      const double sr = __dmul_rn(0.7071067811865476, S[int64_t(n) * N + m]);
      const double si = __dmul_rn(0.7071067811865476, S[int64_t(K) * N + int64_t(n) * N + m]);
      const c128 v = mk<double>(
          __dadd_rn(__dmul_rn(wl, __dmul_rn(g.gain, h.re)), __dmul_rn(wn, __dmul_rn(gn, sr))),
          __dadd_rn(__dmul_rn(wl, __dmul_rn(g.gain, h.im)), __dmul_rn(wn, __dmul_rn(gn, si))));
      tmp[m] = v;
      if (H_full) H_full[(item * K + n) * N + m] = v;
      if (H_tl) H_tl[(item * K + n) * N + m] = h;
    }
    __syncthreads();
    for (int cc = w; cc < R; cc += nw) {
      const int j = cols[cc], jx = j / ny, jy = j % ny;
      c128 ae = czero<double>(), ar = czero<double>();
      for (int m = lane; m < N; m += 32) {
        const c128 f = cmul_np(Dx[(m / ny) * nx + jx], Dy[(m % ny) * ny + jy]);
        cfma(ae, row[m], f);
        cfma(ar, tmp[m], f);
      }
      ae.re = warp_sum(ae.re);
      ae.im = warp_sum(ae.im);
      ar.re = warp_sum(ar.re);
      ar.im = warp_sum(ar.im);
      if (lane == 0) {
        H_eff[(item * K + n) * R + cc] = ae;
        H_rf[(item * K + n) * R + cc] = ar;
      }
    }
    __syncthreads();
  }
  for (int cc = threadIdx.x; cc < R; cc += blockDim.x) cols_out[item * R + cc] = cols[cc];
  if (threadIdx.x == 0 && info) info[item] = below ? LRZ_INFO_BELOW_MASK : LRZ_INFO_OK;
}

// ---- hybrid precoder + rate ------------------------------------------------------

constexpr int HR_KMAX = 64;

__global__ void __launch_bounds__(LEO_THREADS)
hybrid_rate_kernel(int64_t B, int K, int R, int nx, int ny, const c128 *__restrict__ H_eff,
                   const c128 *__restrict__ A_inv, const c128 *__restrict__ H_rf,
                   const int32_t *__restrict__ cols, const c128 *__restrict__ dft, double P_t,
                   const double *__restrict__ noise, int64_t noise_div, c128 *__restrict__ F_BB,
                   double *__restrict__ scale_out, double *__restrict__ rates,
                   double *__restrict__ sum_rate, int32_t *__restrict__ info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t item = blockIdx.x;
  const int N = nx * ny;
  c128 *Dx = (c128 *)smem_raw;
  c128 *Dy = Dx + nx * nx;
  c128 *Fr = Dy + ny * ny;           // R x K
  double *pwr = (double *)(Fr + R * K);   // K x K
  __shared__ double red[LEO_THREADS / 32];
  __shared__ int jx_s[HR_KMAX * 4], jy_s[HR_KMAX * 4];
  for (int i = threadIdx.x; i < nx * nx; i += blockDim.x) Dx[i] = dft[i];
  for (int i = threadIdx.x; i < ny * ny; i += blockDim.x) Dy[i] = dft[nx * nx + i];
  for (int cc = threadIdx.x; cc < R; cc += blockDim.x) {
    const int j = cols[item * R + cc];
    jx_s[cc] = j / ny;
    jy_s[cc] = j % ny;
  }
  const c128 *He = H_eff + item * K * R;
  const c128 *Ai = A_inv + item * K * K;
  // F_raw = H_eff^H A^-1  (R x K)
  for (int e = threadIdx.x; e < R * K; e += blockDim.x) {
    const int cc = e / K, k = e % K;
    c128 a = czero<double>();
    for (int j = 0; j < K; ++j) cfma_ca(a, He[j * R + cc], Ai[j * K + k]);
    Fr[e] = a;
  }
  __syncthreads();
  // ||F_RF F_raw||_F^2, F_RF[m][c] = Dx[ix][jx_c] Dy[iy][jy_c]
  double part = 0.0;
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const int ix = m / ny, iy = m % ny;
    for (int k0 = 0; k0 < K; k0 += 16) {
      c128 acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = czero<double>();
      for (int cc = 0; cc < R; ++cc) {
        const c128 f = cmul_np(Dx[ix * nx + jx_s[cc]], Dy[iy * ny + jy_s[cc]]);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (k0 + q < K) cfma(acc[q], f, Fr[cc * K + k0 + q]);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) part += cabs2(acc[q]);
    }
  }
  const double fro2 = block_sum(part, red);
  const double nrm = sqrt(fro2);
  const double scale = nrm == 0.0 ? 0.0 : sqrt(P_t) / nrm;
  // G = H_rf (scale F_raw), powers
  const c128 *Hr = H_rf + item * K * R;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    c128 a = czero<double>();
    for (int cc = 0; cc < R; ++cc) cfma(a, Hr[n * R + cc], cscale(Fr[cc * K + k], scale));
    const double h = hypot(a.re, a.im);
    pwr[e] = h * h;
  }
  if (F_BB)
    for (int e = threadIdx.x; e < R * K; e += blockDim.x) F_BB[item * R * K + e] = cscale(Fr[e], scale);
  __syncthreads();
  const double *nz = noise + (item / noise_div) * K;
  for (int n = threadIdx.x; n < K; n += blockDim.x) {
    double tot = 0.0;
    for (int k = 0; k < K; ++k) tot += pwr[n * K + k];
    const double sig = pwr[n * K + n];
    const double sinr = sig / (tot - sig + nz[n]);
    const double rate = log2(1.0 + sinr);
    rates[item * K + n] = rate;
  }
  __syncthreads();
  // deterministic sum over users in index order
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int n = 0; n < K; ++n) s += rates[item * K + n];
    sum_rate[item] = s;
    scale_out[item] = scale;
    if (info) info[item] = nrm == 0.0 ? LRZ_INFO_ZERO_PRECODER : LRZ_INFO_OK;
  }
}

// ---- campaign aggregates ----------------------------------------------------------

__global__ void campaign_reduce_kernel(int64_t B, int T, int t_base, int K, int n_reset,
                                       int conventional, const uint8_t *__restrict__ method,
                                       const int32_t *__restrict__ k_est,
                                       double *__restrict__ stats) {
  const int64_t b = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const double Kf = K, full = Kf * Kf * Kf;
  double cost = 0, ks = 0, kc = 0, nf = 0, nw = 0, nn = 0;
  for (int t = lane; t < T; t += 32) {
    const int tg = t_base + t;
    const bool reset = conventional || tg == 0 || (n_reset > 0 && tg % n_reset == 0);
    const int m = method[b * T + t];
    const double k = k_est[b * T + t];
    if (reset) {
      cost += full;
    } else {
      ks += k;
      kc += 1;
      if (m == LRZ_METHOD_FULL)
        cost += full + (Kf * Kf * k + k * k * Kf);
      else if (m == LRZ_METHOD_WOODBURY)
        cost += Kf * Kf + Kf * Kf * k + k * k * k + k * k * Kf;
      else
        cost += Kf * Kf;
    }
    nf += (reset || m == LRZ_METHOD_FULL);
    nw += (!reset && m == LRZ_METHOD_WOODBURY);
    nn += (!reset && m == LRZ_METHOD_NONE);
  }
  cost = warp_sum(cost);
  ks = warp_sum(ks);
  kc = warp_sum(kc);
  nf = warp_sum(nf);
  nw = warp_sum(nw);
  nn = warp_sum(nn);
  if (lane == 0) {
    double *s = stats + b * 6;
    s[0] += cost;
    s[1] += ks;
    s[2] += kc;
    s[3] += nf;
    s[4] += nw;
    s[5] += nn;
  }
}

// Campaign summary on the device (harness.py:336-367): per method m of M
// (rates [M][B][T], stats [M][B][6] from campaign_reduce): per-trial mean
// rates, the pooled mean rate, mean cost units per trial, the pooled mean
// rank (k_sum / k_count) and the decision counts; fixed summation orders.
// summary[m] = (mean_rate, mean_cost, mean_k, n_full, n_woodbury, n_none).
__global__ void campaign_summary_kernel(int64_t B, int T, const double *__restrict__ rates,
                                        const double *__restrict__ stats,
                                        double *__restrict__ trial_mean,
                                        double *__restrict__ summary) {
  __shared__ double red[8];
  const int m = blockIdx.x;
  const double *r = rates + int64_t(m) * B * T;
  double tot = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    double loc = 0.0;
    for (int t = threadIdx.x; t < T; t += blockDim.x) loc += r[b * T + t];
    const double sb = block_sum(loc, red);
    if (threadIdx.x == 0) trial_mean[int64_t(m) * B + b] = sb / T;
    tot += sb;
  }
  if (threadIdx.x == 0) {
    const double *st = stats + int64_t(m) * B * 6;
    double cost = 0, ks = 0, kc = 0, nf = 0, nw = 0, nn = 0;
    for (int64_t b = 0; b < B; ++b) {
      cost += st[b * 6 + 0];
      ks += st[b * 6 + 1];
      kc += st[b * 6 + 2];
      nf += st[b * 6 + 3];
      nw += st[b * 6 + 4];
      nn += st[b * 6 + 5];
    }
    double *o = summary + m * 6;
    o[0] = tot / (double(B) * T);
    o[1] = cost / double(B);
    o[2] = kc > 0 ? ks / kc : 0.0;
    o[3] = nf;
    o[4] = nw;
    o[5] = nn;
  }
}

// the comparison table (harness.py:357-367): method 0 is the conventional
// baseline; row m = (savings %, degradation %) = 100 (1 - cost_m / cost_0),
// 100 (1 - rate_m / rate_0)
__global__ void campaign_table_kernel(int M, const double *__restrict__ summary,
                                      double *__restrict__ table) {
  const int m = threadIdx.x;
  if (m >= M) return;
  const double c0 = summary[1], r0 = summary[0];
  table[m * 2 + 0] = m == 0 ? 0.0 : 100.0 * (1.0 - summary[m * 6 + 1] / c0);
  table[m * 2 + 1] = m == 0 ? 0.0 : 100.0 * (1.0 - summary[m * 6 + 0] / r0);
}

}  // namespace lrz

using namespace lrz;

extern "C" int lrz_campaign_summary(int M, int64_t B, int T, const double *rates,
                                    const double *stats, double *trial_mean, double *summary,
                                    double *table, void *stream) {
  if (M < 1 || M > 1024 || B < 1 || T < 1 || !rates || !stats || !trial_mean || !summary ||
      !table) {
    lrz_set_error("lrz_campaign_summary: bad arguments");
    return LRZ_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  campaign_summary_kernel<<<unsigned(M), 256, 0, s>>>(B, T, rates, stats, trial_mean, summary);
  campaign_table_kernel<<<1, 1024, 0, s>>>(M, summary, table);
  return lrz_launch_status("lrz_campaign_summary");
}

static size_t leo_smem(int nx, int ny) {
  const int N = nx * ny;
  return size_t(nx * nx + ny * ny + 2 * N) * sizeof(c128) + size_t(N) * sizeof(double) + N;
}

extern "C" int lrz_leo_snapshot(const lrz_leo_cfg *cfg, int64_t B, int t0, int T, const double *ut,
                                const void *dft, const double *nlos, int64_t nlos_stride,
                                void *H_eff, void *H_rf, int32_t *cols, int32_t *info,
                                void *H_full, void *H_tilde, void *stream) {
  if (!cfg || B < 0 || T < 1 || t0 < 0 || !ut || !dft || !nlos || !H_eff || !H_rf || !cols) {
    lrz_set_error("lrz_leo_snapshot: bad arguments");
    return LRZ_EINVAL;
  }
  const lrz_leo_cfg c = *cfg;
  const int N = c.n_x * c.n_y;
  if (c.K < 1 || c.K > 64 || c.n_x < 1 || c.n_y < 1 || N > LEO_NMAX || c.N_RF < c.K ||
      c.N_RF > N || c.N_RF > 256 || c.beam_hold < 1 || c.nlos_block < 1) {
    lrz_set_error("lrz_leo_snapshot: need 1 <= K <= 64, K <= N_RF <= min(N, 256), N <= %d, "
                  "beam_hold/nlos_block >= 1 (K=%d N=%d N_RF=%d)", LEO_NMAX, c.K, N, c.N_RF);
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const size_t smem = leo_smem(c.n_x, c.n_y);
  cudaFuncSetAttribute(leo_snapshot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  leo_snapshot_kernel<<<unsigned(B * T), LEO_THREADS, smem, (cudaStream_t)stream>>>(
      c, B, t0, T, ut, (const c128 *)dft, nlos, nlos_stride, (c128 *)H_eff, (c128 *)H_rf, cols,
      info, (c128 *)H_full, (c128 *)H_tilde);
  return lrz_launch_status("leo_snapshot_kernel");
}

extern "C" int lrz_hybrid_precode_rate(int64_t B, int K, int N_RF, int n_x, int n_y,
                                       const void *H_eff, const void *A_inv, const void *H_rf,
                                       const int32_t *cols, const void *dft, double P_t,
                                       const double *noise, int64_t noise_div, void *F_BB,
                                       double *scale, double *rates, double *sum_rate,
                                       int32_t *info, void *stream) {
  if (B < 0 || K < 1 || K > HR_KMAX || N_RF < 1 || N_RF > 4 * HR_KMAX || n_x < 1 || n_y < 1 ||
      !H_eff || !A_inv || !H_rf || !cols || !dft || !noise || noise_div < 1 || !scale ||
      !rates || !sum_rate) {
    lrz_set_error("lrz_hybrid_precode_rate: bad arguments (K <= %d, N_RF <= %d)", HR_KMAX,
                  4 * HR_KMAX);
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const size_t smem = size_t(n_x * n_x + n_y * n_y + N_RF * K) * sizeof(c128) +
                      size_t(K) * K * sizeof(double);
  if (smem > 200 * 1024) {
    lrz_set_error("lrz_hybrid_precode_rate: shared memory %zu too large", smem);
    return LRZ_EINVAL;
  }
  cudaFuncSetAttribute(hybrid_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  hybrid_rate_kernel<<<unsigned(B), LEO_THREADS, smem, (cudaStream_t)stream>>>(
      B, K, N_RF, n_x, n_y, (const c128 *)H_eff, (const c128 *)A_inv, (const c128 *)H_rf, cols,
      (const c128 *)dft, P_t, noise, noise_div, (c128 *)F_BB, scale, rates, sum_rate, info);
  return lrz_launch_status("hybrid_rate_kernel");
}

extern "C" int lrz_campaign_reduce(int64_t B, int T, int t_base, int K, int n_reset,
                                   int conventional, const uint8_t *method, const int32_t *k_est,
                                   double *stats, void *stream) {
  if (B < 0 || T < 0 || K < 1 || !method || !k_est || !stats) {
    lrz_set_error("lrz_campaign_reduce: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0 || T == 0) return LRZ_OK;
  const unsigned nb = unsigned((B * 32 + 255) / 256);
  campaign_reduce_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(B, T, t_base, K, n_reset,
                                                               conventional, method, k_est, stats);
  return lrz_launch_status("campaign_reduce_kernel");
}
