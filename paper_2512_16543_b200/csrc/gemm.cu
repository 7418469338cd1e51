// N-sized batched complex products: Gram (K1), Gram correction (K1'),
// precoder / coupling GEMMs (K6) and a generic batched CGEMM.
//
// These are the HBM/FP-heavy kernels of the step (8K^2 N-class work).  Round-1
// design: SIMT tiles of 32x32 outputs per CTA, operands staged through shared
// memory in BK-wide slabs along the N (antenna) axis, fp32 FMA for complex64
// inputs and fp64 FMA for complex128 inputs; one CTA per (item, tile) so a
// B*T batch of small matrices fills all 148 SMs.

#include <stdlib.h>

#include "dmma.cuh"


namespace lrz {

constexpr int TM = 32;        // output tile edge
constexpr int GEMM_THREADS = 128;

// map a lower-triangle tile index to (I, J), I >= J
LRZ_DEV void tri_tile(int t, int &I, int &J) {
  int i = int((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

template <typename T>
LRZ_DEV void cp_async16(void *smem, const void *gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (sizeof(cplx<T>) == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(pred ? 16 : 0));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(pred ? 8 : 0));
  }
}
template <typename T>
LRZ_DEV void cp_async_el(void *smem, const void *gmem, bool pred) {
  cp_async16<T>(smem, gmem, pred);
}
LRZ_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
LRZ_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// K1: A = H H^H (Hermitian, lower tiles computed, mirrored) + alpha I
// ---------------------------------------------------------------------------
template <typename T, int BK>
__global__ void __launch_bounds__(GEMM_THREADS)
    gram_kernel(int K, int N, const cplx<T> *__restrict__ H, int64_t hs, double alpha,
                c128 *__restrict__ A, int64_t as, int ntl) {
  __shared__ cplx<T> As[BK][TM + 1];
  __shared__ cplx<T> Bs[BK][TM + 1];
  const int64_t item = blockIdx.x / ntl;
  int I, J;
  tri_tile(int(blockIdx.x % ntl), I, J);
  const bool diag = (I == J);
  const cplx<T> *h = H + item * hs;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  cplx<T> acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = czero<T>();

  for (int n0 = 0; n0 < N; n0 += BK) {
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      const int r = e / BK, k = e % BK, gk = n0 + k;
      const int ri = I * TM + r, rj = J * TM + r;
      As[k][r] = (ri < K && gk < N) ? h[int64_t(ri) * N + gk] : czero<T>();
      if (!diag) Bs[k][r] = (rj < K && gk < N) ? h[int64_t(rj) * N + gk] : czero<T>();
    }
    __syncthreads();
    const cplx<T>(*Bp)[TM + 1] = diag ? As : Bs;
#pragma unroll 4
    for (int k = 0; k < BK; ++k) {
      cplx<T> a0 = As[k][ty], a1 = As[k][ty + 16];
      cplx<T> b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bp[k][tx + 8 * j];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cfma_cb(acc[0][j], a0, b[j]);
        cfma_cb(acc[1][j], a1, b[j]);
      }
    }
    __syncthreads();
  }
  c128 *a = A + item * as;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = I * TM + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = J * TM + tx + 8 * j;
      if (row < K && col < K && row >= col) {
        c128 v = ccast<double>(acc[i][j]);
        if (row == col) {
          v.im = 0.0;  // 0.5 (A + A^H) has an exactly real diagonal (lowrank.py:161)
          v.re += alpha;
          a[int64_t(row) * K + col] = v;
        } else {
          a[int64_t(row) * K + col] = v;
          a[int64_t(col) * K + row] = cconj(v);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 for K <= 32: only the lower triangle is formed.  The 32 x 32 output is
// cut into 4 x 4 register tiles; the 36 lower tiles of an item go to 36
// threads, G32_IPB items share a CTA (288 threads), and the items' H rows
// stream through shared memory in G32_BK-wide slabs with cp.async double
// buffering.  Per k a thread does 8 shared loads for 16 complex FMAs.
// ---------------------------------------------------------------------------
constexpr int G32_IPB = 8;
constexpr int G32_BK = 8;
constexpr int G32_THREADS = 36 * G32_IPB;


template <typename T>
__global__ void __launch_bounds__(G32_THREADS, 2)
    gram32_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                  double alpha, c128 *__restrict__ A, int64_t as) {
  extern __shared__ __align__(16) char g32_smem[];
  cplx<T> *S = (cplx<T> *)g32_smem;   // [3][G32_IPB][G32_BK][32]
  const int tid = threadIdx.x;
  const int li = tid / 36, tile = tid % 36;
  int I, J;
  tri_tile(tile, I, J);
  const int64_t item0 = int64_t(blockIdx.x) * G32_IPB;
  const int nslab = (N + G32_BK - 1) / G32_BK;
  auto issue = [&](int slab, int buf) {
    // G32_IPB items x 32 rows x G32_BK columns; consecutive threads walk n
    for (int e = tid; e < G32_IPB * 32 * G32_BK; e += G32_THREADS) {
      const int kk = e % G32_BK, r = (e / G32_BK) & 31, it = e / (G32_BK * 32);
      const int n = slab * G32_BK + kk;
      const int64_t item = item0 + it;
      const bool ok = item < B && r < K && n < N;
      // row r = 4 I + i lives at column i * 8 + I: a warp's 4-row tile loads hit
      // 8 consecutive elements (one shared-memory wavefront per item)
      cp_async_el<T>(S + ((buf * G32_IPB + it) * G32_BK + kk) * 32 + (r & 3) * 8 + (r >> 2),
                     H + (ok ? item * hs + int64_t(r) * N + n : 0), ok);
    }
    cp_async_commit();
  };
  cplx<T> acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = czero<T>();
  // 3-stage ring, one barrier per slab: after the barrier of slab sl every
  // thread is done with slab sl-1, whose buffer then receives slab sl+2
  issue(0, 0);
  if (nslab > 1) issue(1, 1); else cp_async_commit();
  for (int sl = 0; sl < nslab; ++sl) {
    cp_async_wait<1>();
    __syncthreads();
    if (sl + 2 < nslab) issue(sl + 2, (sl + 2) % 3); else cp_async_commit();
    const cplx<T> *sb = S + ((sl % 3) * G32_IPB + li) * G32_BK * 32;
#pragma unroll
    for (int kk = 0; kk < G32_BK; ++kk) {
      cplx<T> a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = sb[kk * 32 + i * 8 + I];
        b[i] = sb[kk * 32 + i * 8 + J];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma_cb(acc[i][j], a[i], b[j]);
    }
  }
  const int64_t item = item0 + li;
  if (item >= B) return;
  c128 *a = A + item * as;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = 4 * I + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = 4 * J + j;
      if (row < K && col < K && row >= col) {
        c128 v = ccast<double>(acc[i][j]);
        if (row == col) {
          v.im = 0.0;  // 0.5 (A + A^H) has an exactly real diagonal (lowrank.py:161)
          v.re += alpha;
          a[int64_t(row) * K + col] = v;
        } else {
          a[int64_t(row) * K + col] = v;
          a[int64_t(col) * K + row] = cconj(v);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1': dA = C + C^H, C = X dH^H, X = H + dH/2  (== H dH^H + dH H^H + dH dH^H)
// ---------------------------------------------------------------------------
template <typename T>
LRZ_DEV void load_xd(const cplx<T> *P, const cplx<T> *Q, int mode, int64_t off, cplx<T> &x,
                     cplx<T> &d) {
  const cplx<T> p = P[off], q = Q[off];
  if (mode == 0) {
    d = q;
  } else {
    d = csub(q, p);  // dH = H_t - H_{t-1}, bit-identical to harness.py:235
  }
  x = mk<T>(p.re + T(0.5) * d.re, p.im + T(0.5) * d.im);
}

template <typename T, int BK>
__global__ void __launch_bounds__(GEMM_THREADS)
    gram_delta_kernel(int K, int N, const cplx<T> *__restrict__ P, int64_t ps,
                      const cplx<T> *__restrict__ Q, int64_t qs, int mode,
                      c128 *__restrict__ dA, int64_t as, int ntl) {
  __shared__ cplx<T> XI[BK][TM + 1], DI[BK][TM + 1], XJ[BK][TM + 1], DJ[BK][TM + 1];
  const int64_t item = blockIdx.x / ntl;
  int I, J;
  tri_tile(int(blockIdx.x % ntl), I, J);
  const bool diag = (I == J);
  const cplx<T> *p = P + item * ps;
  const cplx<T> *q = Q + item * qs;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  cplx<T> c1[2][4], c2[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c1[i][j] = c2[i][j] = czero<T>();

  for (int n0 = 0; n0 < N; n0 += BK) {
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      const int r = e / BK, k = e % BK, gk = n0 + k;
      const int ri = I * TM + r, rj = J * TM + r;
      cplx<T> x = czero<T>(), d = czero<T>();
      if (ri < K && gk < N) load_xd(p, q, mode, int64_t(ri) * N + gk, x, d);
      XI[k][r] = x;
      DI[k][r] = d;
      if (!diag) {
        x = czero<T>();
        d = czero<T>();
        if (rj < K && gk < N) load_xd(p, q, mode, int64_t(rj) * N + gk, x, d);
        XJ[k][r] = x;
        DJ[k][r] = d;
      }
    }
    __syncthreads();
    const cplx<T>(*xj)[TM + 1] = diag ? XI : XJ;
    const cplx<T>(*dj)[TM + 1] = diag ? DI : DJ;
#pragma unroll 2
    for (int k = 0; k < BK; ++k) {
      cplx<T> xi[2] = {XI[k][ty], XI[k][ty + 16]};
      cplx<T> di[2] = {DI[k][ty], DI[k][ty + 16]};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const cplx<T> xjj = xj[k][tx + 8 * j], djj = dj[k][tx + 8 * j];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          cfma_cb(c1[i][j], xi[i], djj);   // X_i dH_j^*
          cfma_cb(c2[i][j], xjj, di[i]);   // X_j dH_i^*
        }
      }
    }
    __syncthreads();
  }
  c128 *a = dA + item * as;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = I * TM + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = J * TM + tx + 8 * j;
      if (row < K && col < K && row >= col) {
        const c128 u = ccast<double>(c1[i][j]), w = ccast<double>(c2[i][j]);
        c128 v = mk<double>(u.re + w.re, u.im - w.im);
        if (row == col) {
          v.im = 0.0;
          a[int64_t(row) * K + col] = v;
        } else {
          a[int64_t(row) * K + col] = v;
          a[int64_t(col) * K + row] = cconj(v);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Generic batched complex GEMM  C = op(A) op(B), element types TA/TB converted
// to the accumulation type T on load; optional ||C||_F^2 partial per tile.
// ---------------------------------------------------------------------------
template <typename T, typename TA, typename TB, int BK>
__global__ void __launch_bounds__(GEMM_THREADS)
    cgemm_kernel(int M, int N, int Kd, int opA, const cplx<TA> *__restrict__ A, int64_t lda,
                 int64_t sA, int opB, const cplx<TB> *__restrict__ Bm, int64_t ldb, int64_t sB,
                 cplx<T> *__restrict__ C, int64_t ldc, int64_t sC, double *__restrict__ norm_part,
                 int tiles_m, int tiles_n) {
  __shared__ cplx<T> As[BK][TM + 1];
  __shared__ cplx<T> Bs[BK][TM + 1];
  __shared__ double red[GEMM_THREADS / 32];
  const int ntile = tiles_m * tiles_n;
  const int64_t item = blockIdx.x / ntile;
  const int tile = int(blockIdx.x % ntile);
  const int I = tile / tiles_n, J = tile % tiles_n;
  const cplx<TA> *a = A + item * sA;
  const cplx<TB> *b = Bm + item * sB;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  cplx<T> acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = czero<T>();

  for (int k0 = 0; k0 < Kd; k0 += BK) {
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      // A_eff[m][k]: op 0 -> A[m][k] (k contiguous); op 1/2 -> A[k][m] (m contiguous)
      int m, k;
      if (opA == 0 || opA == 3) {  // 3: conj(A[m][k]) (internal)
        m = e / BK;
        k = e % BK;
      } else {
        k = e / TM;
        m = e % TM;
      }
      const int gm = I * TM + m, gk = k0 + k;
      cplx<T> v = czero<T>();
      if (gm < M && gk < Kd) {
        cplx<TA> x = (opA == 0 || opA == 3) ? a[int64_t(gm) * lda + gk]
                                            : a[int64_t(gk) * lda + gm];
        v = ccast<T>(x);
        if (opA >= 2) v.im = -v.im;
      }
      As[k][m] = v;
    }
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      // B_eff[k][n]: op 0 -> B[k][n] (n contiguous); op 1/2 -> B[n][k] (k contiguous)
      int n, k;
      if (opB == 0) {
        k = e / TM;
        n = e % TM;
      } else {
        n = e / BK;
        k = e % BK;
      }
      const int gn = J * TM + n, gk = k0 + k;
      cplx<T> v = czero<T>();
      if (gn < N && gk < Kd) {
        cplx<TB> x = (opB == 0) ? b[int64_t(gk) * ldb + gn] : b[int64_t(gn) * ldb + gk];
        v = ccast<T>(x);
        if (opB == 2) v.im = -v.im;
      }
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < BK; ++k) {
      const cplx<T> a0 = As[k][ty], a1 = As[k][ty + 16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const cplx<T> bj = Bs[k][tx + 8 * j];
        cfma(acc[0][j], a0, bj);
        cfma(acc[1][j], a1, bj);
      }
    }
    __syncthreads();
  }
  cplx<T> *c = C + item * sC;
  double nrm = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = I * TM + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = J * TM + tx + 8 * j;
      if (row < M && col < N) {
        c[int64_t(row) * ldc + col] = acc[i][j];
        nrm += double(acc[i][j].re) * double(acc[i][j].re) +
               double(acc[i][j].im) * double(acc[i][j].im);
      }
    }
  }
  if (norm_part) {
    const double s = block_sum(nrm, red);
    if (tid == 0) norm_part[item * ntile + tile] = s;
  }
}

// ---------------------------------------------------------------------------
// SINR / rate epilogue (precoding.py:74-80) from a K x K coupling matrix.
// scale: explicit per-item (scale_in) or derived from norm partials
// (sqrt(P_t)/sqrt(sum of partials), precoding.py:47-51).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
    sinr_kernel(int K, const cplx<T> *__restrict__ G, int64_t sG, const double *scale_in,
                const double *__restrict__ norm_part, int nparts, double P_t,
                double *scale_out, const double *__restrict__ noise, int64_t noise_div,
                double *rates, double *sinr, double *sum_rate, int32_t *info,
                const c128 *__restrict__ corr = nullptr, int64_t scorr = 0, double alpha = 0.0) {
  __shared__ double red[8];
  const int64_t item = blockIdx.x;
  double s = 1.0;
  int bad = 0;
  if (scale_in) {
    s = scale_in[item];
  } else if (norm_part) {
    double n2 = 0.0;
    for (int i = 0; i < nparts; ++i) n2 += norm_part[item * nparts + i];
    const double nrm = sqrt(n2);
    if (!(nrm > 0.0)) {
      bad = 1;
      s = 0.0;
    } else {
      s = sqrt(P_t) / nrm;
    }
    if (threadIdx.x == 0) {
      if (scale_out) scale_out[item] = s;
      if (info) info[item] = bad ? LRZ_INFO_ZERO_PRECODER : LRZ_INFO_OK;
    }
  }
  const cplx<T> *g = G + item * sG;
  const c128 *cr = corr ? corr + item * scorr : nullptr;
  const double *nz = noise + (item / noise_div) * K;
  double my = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    double tot = 0.0, sig = 0.0;
    for (int j = 0; j < K; ++j) {
      c128 gv = ccast<double>(g[int64_t(i) * K + j]);
      if (cr) {  // H W = (G_true - alpha I) A^-1 = G_true A^-1 - alpha A^-1
        const c128 a = cr[int64_t(i) * K + j];
        gv.re -= alpha * a.re;
        gv.im -= alpha * a.im;
      }
      const c128 v = cscale(gv, s);
      const double p = cabs2(v);
      tot += p;
      if (j == i) sig = p;
    }
    const double q = sig / ((tot - sig) + nz[i]);
    const double r = log2(1.0 + q);
    if (rates) rates[item * K + i] = r;
    if (sinr) sinr[item * K + i] = q;
    my += r;
  }
  const double total = block_sum(my, red);
  if (threadIdx.x == 0 && sum_rate) sum_rate[item] = total;
}

template <typename T>
__global__ void fro2_kernel(int64_t n, const cplx<T> *__restrict__ X, int64_t sX, double *out) {
  __shared__ double red[8];
  const cplx<T> *x = X + blockIdx.x * sX;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += double(cabs2(x[i]));
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

template <typename T>
__global__ void axpby_kernel(int64_t n, double a, const cplx<T> *__restrict__ X, double b,
                             const cplx<T> *__restrict__ Y, cplx<T> *__restrict__ Z) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const cplx<T> x = X[i];
    cplx<T> z = mk<T>(T(a) * x.re, T(a) * x.im);
    if (Y) {
      const cplx<T> y = Y[i];
      z = (a == 1.0 && b == 1.0) ? mk<T>(x.re + y.re, x.im + y.im)
                                 : mk<T>(z.re + T(b) * y.re, z.im + T(b) * y.im);
    }
    Z[i] = z;
  }
}


// ---------------------------------------------------------------------------
// K6 precoder W = H^H A^-1 for one item per CTA (K <= 64): A^-1 staged in
// shared memory (converted to the input precision), one antenna row n per
// thread with KB register accumulators, H rows read coalesced along n;
// ||W||_F^2 reduced in the epilogue (precoding.py:47-48).
// ---------------------------------------------------------------------------
template <typename T, int KB>
__global__ void __launch_bounds__(256)
    precoder_w_kernel(int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                      const c128 *__restrict__ Ainv, int64_t ais, cplx<T> *__restrict__ W,
                      int64_t wst, double *__restrict__ norm2) {
  extern __shared__ __align__(16) char pw_smem[];
  cplx<T> *As = (cplx<T> *)pw_smem;
  __shared__ double red[8];
  const int64_t item = blockIdx.x;
  const c128 *ai = Ainv + item * ais;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) As[e] = ccast<T>(ai[e]);
  __syncthreads();
  const cplx<T> *h = H + item * hs;
  cplx<T> *w = W + item * wst;
  double nrm = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    for (int jb = 0; jb < K; jb += KB) {
      cplx<T> acc[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) acc[j] = czero<T>();
#pragma unroll 8
      for (int k = 0; k < K; ++k) {
        const cplx<T> hv = h[int64_t(k) * N + n];
        const cplx<T> *ar = As + k * K + jb;
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (jb + j < K) cfma_ca(acc[j], hv, ar[j]);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j)
        if (jb + j < K) {
          w[int64_t(n) * K + jb + j] = acc[j];
          nrm += double(acc[j].re) * double(acc[j].re) + double(acc[j].im) * double(acc[j].im);
        }
    }
  }
  nrm = block_sum(nrm, red);
  if (threadIdx.x == 0) norm2[item] = nrm;
}


// ---------------------------------------------------------------------------
// Y = dA [Omega_0 ... Omega_{i_max-1}] for the arSVD front end, with the
// sketch operand read straight from the normal window (block i: real K x d_i
// then imaginary K x d_i at cursor + sum_{i'<i} 2 K d_i', scaled by sqrt(1/2),
// lowrank.py:284-286) -- no materialised complex Omega.  Same tiling as
// cgemm_kernel (32 x 32 output tiles, A row-major).
// ---------------------------------------------------------------------------
struct SketchOperand {
  const double *omega;
  int64_t os;
  const int32_t *orow;
  int64_t orow_div;
  const int64_t *cursor;
  int k_init, p;
};

__global__ void __launch_bounds__(GEMM_THREADS)
    sketch_cgemm_kernel(int K, int Dtot, const c128 *__restrict__ A, int64_t sA, SketchOperand so,
                        const uint8_t *__restrict__ mask, c128 *__restrict__ C, int tiles_n,
                        c128 *__restrict__ W) {
  // W != nullptr (K <= 32): also W = dA Y for this tile's columns, with dA and
  // the Y tile kept in shared memory (dynamic: [32][33] each)
  extern __shared__ __align__(16) char sk_smem[];
  constexpr int BK = 16;
  __shared__ c128 As[BK][TM + 1];
  __shared__ c128 Bs[BK][TM + 1];
  __shared__ int s_off[TM], s_d[TM], s_j[TM];
  const int tiles_m = (K + TM - 1) / TM, ntile = tiles_m * tiles_n;
  const int64_t item = blockIdx.x / ntile;
  if (mask && !mask[item]) return;
  const int tile = int(blockIdx.x % ntile);
  const int I = tile / tiles_n, J = tile % tiles_n;
  const c128 *a = A + item * sA;
  const int64_t row = so.orow ? int64_t(so.orow[item]) : item / so.orow_div;
  const double *z = so.omega + row * so.os + (so.cursor ? so.cursor[item] : 0);
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  // column -> (block offset in the stream, block width d, column j in block)
  for (int n = tid; n < TM; n += GEMM_THREADS) {
    const int gn = J * TM + n;
    int o = 0, k0 = so.k_init, d = min(k0 + so.p, K);
    int off = 0;
    while (gn >= o + d && gn < Dtot) {
      o += d;
      off += 2 * K * d;
      k0 *= 2;
      d = min(k0 + so.p, K);
    }
    s_off[n] = off;
    s_d[n] = d;
    s_j[n] = gn - o;
  }
  __syncthreads();
  const double SQH = 0.7071067811865476;
  c128 acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = czero<double>();
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      const int m = e / BK, k = e % BK, gm = I * TM + m, gk = k0 + k;
      As[k][m] = (gm < K && gk < K) ? a[int64_t(gm) * K + gk] : czero<double>();
    }
    for (int e = tid; e < TM * BK; e += GEMM_THREADS) {
      const int k = e / TM, n = e % TM, gn = J * TM + n, gk = k0 + k;
      c128 v = czero<double>();
      if (gn < Dtot && gk < K) {
        const int d = s_d[n];
        const double *zb = z + s_off[n] + int64_t(gk) * d + s_j[n];
        v = mk<double>(SQH * zb[0], SQH * zb[int64_t(K) * d]);
      }
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < BK; ++k) {
      const c128 a0 = As[k][ty], a1 = As[k][ty + 16];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const c128 bj = Bs[k][tx + 8 * j];
        cfma(acc[0][j], a0, bj);
        cfma(acc[1][j], a1, bj);
      }
    }
    __syncthreads();
  }
  c128 *c = C + item * int64_t(K) * Dtot;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = I * TM + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = J * TM + tx + 8 * j;
      if (r < K && col < Dtot) c[int64_t(r) * Dtot + col] = acc[i][j];
    }
  }
  if (W == nullptr) return;
  c128(*Af)[TM + 1] = (c128(*)[TM + 1])sk_smem;                 // dA, [32][33]
  c128(*Ys)[TM + 1] = (c128(*)[TM + 1])(sk_smem + TM * (TM + 1) * sizeof(c128));
  for (int e = tid; e < TM * TM; e += GEMM_THREADS) {
    const int r = e / TM, m = e % TM;
    Af[r][m] = (r < K && m < K) ? a[int64_t(r) * K + m] : czero<double>();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Ys[ty + 16 * i][tx + 8 * j] = acc[i][j];
  __syncthreads();
  c128 wv[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) wv[i][j] = czero<double>();
  for (int m = 0; m < K; ++m) {
    const c128 a0 = Af[ty][m], a1 = Af[ty + 16][m];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const c128 y = Ys[m][tx + 8 * j];
      cfma(wv[0][j], a0, y);
      cfma(wv[1][j], a1, y);
    }
  }
  c128 *w = W + item * int64_t(K) * Dtot;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = J * TM + tx + 8 * j;
      if (r < K && col < Dtot) w[int64_t(r) * Dtot + col] = wv[i][j];
    }
  }
}


// Y = dA Omega_all and W = dA Y for K <= 32 on the FP64 tensor pipe: one CTA
// (4 warps) per (item, 32-column tile); the Omega tile is staged from the
// normal window (same addressing as sketch_cgemm_kernel) into re / im planes
// with a row stride of 36 doubles (conflict-free B fragments); warp w owns rows
// 8w..8w+7 with its dA A fragments in registers; the Y tile goes to global
// memory and to shared memory as the B operand of W = dA Y.
constexpr int SD_LD = 36;

__global__ void __launch_bounds__(128)
    sketch_dmma_kernel(int K, int Dtot, const c128 *__restrict__ A, int64_t sA, SketchOperand so,
                       const uint8_t *__restrict__ mask, c128 *__restrict__ C, int tiles_n,
                       c128 *__restrict__ W) {
  __shared__ __align__(16) double Pr[32 * SD_LD], Pi[32 * SD_LD];
  __shared__ int s_off[32], s_d[32], s_j[32];
  const int64_t item = blockIdx.x / tiles_n;
  if (mask && !mask[item]) return;
  const int J = int(blockIdx.x % tiles_n);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const c128 *a = A + item * sA;
  const int64_t row = so.orow ? int64_t(so.orow[item]) : item / so.orow_div;
  const double *z = so.omega + row * so.os + (so.cursor ? so.cursor[item] : 0);
  if (tid < 32) {
    const int gn = J * 32 + tid;
    int o = 0, k0 = so.k_init, d = min(k0 + so.p, K), off = 0;
    while (gn >= o + d && gn < Dtot) {
      o += d;
      off += 2 * K * d;
      k0 *= 2;
      d = min(k0 + so.p, K);
    }
    s_off[tid] = off;
    s_d[tid] = d;
    s_j[tid] = gn - o;
  }
  // dA fragments of this warp's rows (A[8w + g][4c + t])
  double ar[8], ai[8];
  {
    const int r = 8 * w + g;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int k = 4 * c + t;
      const c128 v = (r < K && k < K) ? ldg_c(a + int64_t(r) * K + k) : czero<double>();
      ar[c] = v.re;
      ai[c] = v.im;
    }
  }
  __syncthreads();
  // Omega tile straight from the window into the planes with cp.async (all
  // 16 loads per thread in flight at once; zero fill outside the tile); the
  // sqrt(1/2) of lowrank.py:284-286 is applied to dA in the first pass instead
  const double SQH = 0.7071067811865476;
  for (int e = tid; e < 32 * 32; e += 128) {
    const int k = e >> 5, n = e & 31, gn = J * 32 + n;
    const bool ok = gn < Dtot && k < K;
    const double *zb = z;
    int64_t im_off = 0;
    if (ok) {
      const int d = s_d[n];
      zb = z + s_off[n] + int64_t(k) * d + s_j[n];
      im_off = int64_t(K) * d;
    }
    cp_async_el<float>(Pr + k * SD_LD + n, zb, ok);           // 8-byte copies
    cp_async_el<float>(Pi + k * SD_LD + n, zb + im_off, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int pass = 0; pass < (W ? 2 : 1); ++pass) {
    double cr[4][2], ci[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[j][0] = cr[j][1] = ci[j][0] = ci[j][1] = 0.0;
    const double sc = pass == 0 ? SQH : 1.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double xr = sc * ar[c], xi = sc * ai[c], nxi = -xi;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double br = Pr[(4 * c + t) * SD_LD + 8 * j + g];
        const double bi = Pi[(4 * c + t) * SD_LD + 8 * j + g];
        dmma(cr[j], xr, br);  // (xr + i xi)(br + i bi)
        dmma(cr[j], nxi, bi);
        dmma(ci[j], xr, bi);
        dmma(ci[j], xi, br);
      }
    }
    __syncthreads();  // every warp is done reading the B planes
    c128 *out = (pass == 0 ? C : W) + item * int64_t(K) * Dtot;
    const int r = 8 * w + g;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cl = 8 * j + 2 * t + e, col = J * 32 + cl;
        if (r < K && col < Dtot) out[int64_t(r) * Dtot + col] = mk<double>(cr[j][e], ci[j][e]);
        if (pass == 0) {  // Y tile -> B planes for W = dA Y (rows >= K are zero)
          Pr[r * SD_LD + cl] = cr[j][e];
          Pi[r * SD_LD + cl] = ci[j][e];
        }
      }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K6 precoder W = H^H A^-1, one item per CTA, K <= 32, 256 threads (2 CTAs/SM).
// Thread (rg, cg): rows {rg, rg + 64} of each 128-row block, columns
// {cg + 4 c : c < 8}; H streamed through shared memory in 8-row k-slabs
// with cp.async double buffering, A^-1 staged once.  2 x 8 complex
// accumulators per thread keep the kernel FP-pipe bound (10 shared-memory
// wavefronts per 64 warp-FMAs).  ||W||_F^2 reduced in the epilogue.
// ---------------------------------------------------------------------------
constexpr int PW_KC = 8;      // k rows per slab
constexpr int PW_ROWS = 128;  // antenna rows per block pass
constexpr int PW_THREADS = 128;


template <typename T>
__global__ void __launch_bounds__(PW_THREADS, 3)
    precoder_w32_kernel(int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                        const c128 *__restrict__ Ainv, int64_t ais, cplx<T> *__restrict__ W,
                        int64_t wst, double *__restrict__ norm2) {
  extern __shared__ __align__(16) char pw2_smem[];
  cplx<T> *As = (cplx<T> *)pw2_smem;               // [32][32]
  cplx<T> *Hs = As + 32 * 32;                      // [2][PW_KC][PW_ROWS]
  __shared__ double red[16];
  const int tid = threadIdx.x, cg = tid & 3, rg = tid >> 2;   // rows rg + 32 r, r < 4
  const int64_t item = blockIdx.x;
  const c128 *ai = Ainv + item * ais;
  for (int e = tid; e < 32 * 32; e += PW_THREADS) {
    const int k = e >> 5, j = e & 31;
    As[e] = (k < K && j < K) ? ccast<T>(ai[k * K + j]) : czero<T>();
  }
  const cplx<T> *h = H + item * hs;
  cplx<T> *w = W + item * wst;
  double nrm = 0.0;
  const int nslab = (K + PW_KC - 1) / PW_KC;
  for (int n0 = 0; n0 < N; n0 += PW_ROWS) {
    cplx<T> acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = czero<T>();
    auto issue = [&](int slab, int buf) {
      // PW_KC x PW_ROWS elements, 4 per thread (coalesced along n)
#pragma unroll
      for (int q = 0; q < (PW_KC * PW_ROWS) / PW_THREADS; ++q) {
        const int e = tid + q * PW_THREADS, kk = e / PW_ROWS, nn = e % PW_ROWS;
        const int k = slab * PW_KC + kk, n = n0 + nn;
        const bool ok = (k < K) && (n < N);
        cp_async16<T>(Hs + (buf * PW_KC + kk) * PW_ROWS + nn,
                      h + (ok ? int64_t(k) * N + n : 0), ok);
      }
      cp_async_commit();
    };
    issue(0, 0);
    for (int sl = 0; sl < nslab; ++sl) {
      if (sl + 1 < nslab) {
        issue(sl + 1, (sl + 1) & 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const cplx<T> *hb = Hs + (sl & 1) * PW_KC * PW_ROWS;
#pragma unroll
      for (int kk = 0; kk < PW_KC; ++kk) {
        const int k = sl * PW_KC + kk;
        cplx<T> a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = hb[kk * PW_ROWS + rg + 32 * r];
        const cplx<T> *br = As + k * 32 + cg;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const cplx<T> b = br[4 * c];
#pragma unroll
          for (int r = 0; r < 4; ++r) cfma_ca(acc[r][c], a[r], b);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int n = n0 + rg + 32 * r;
      if (n < N) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = cg + 4 * c;
          if (j < K) {
            w[int64_t(n) * K + j] = acc[r][c];
            nrm += double(acc[r][c].re) * double(acc[r][c].re) +
                   double(acc[r][c].im) * double(acc[r][c].im);
          }
        }
      }
    }
  }
  nrm = block_sum(nrm, red);
  if (tid == 0) norm2[item] = nrm;
}

}  // namespace lrz

using namespace lrz;

extern "C" int lrz_axpby(int dtype, int64_t n, double a, const void *X, double b, const void *Y,
                         void *Z, void *stream) {
  if (n < 0 || !X || !Z) {
    lrz_set_error("lrz_axpby: bad arguments");
    return LRZ_EINVAL;
  }
  if (n == 0) return LRZ_OK;
  const unsigned nb = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 32));
  cudaStream_t s = (cudaStream_t)stream;
  LrzProf prof("axpby_kernel", s);
  if (dtype == LRZ_C64)
    axpby_kernel<float><<<nb, 256, 0, s>>>(n, a, (const c64 *)X, b, (const c64 *)Y, (c64 *)Z);
  else
    axpby_kernel<double><<<nb, 256, 0, s>>>(n, a, (const c128 *)X, b, (const c128 *)Y,
                                            (c128 *)Z);
  return lrz_launch_status("lrz_axpby");
}

static int ntiles(int K) { return (K + TM - 1) / TM; }

// DMMA kernels for K <= 32 (dmma.cu, both dtypes); LRZ_SIMT_FP64=1 selects the
// SIMT kernels instead (A/B measurements)
int lrz_gram_dmma(int dtype, int64_t B, int K, int N, const void *H, int64_t hs, double alpha,
                  void *A, int64_t as, cudaStream_t s);
int lrz_dmma_hn_tiles(int NN, int J);
int lrz_dmma_hn(int dtype, int64_t B, int NN, int J, int Kd, const void *X, int64_t xs, int ldx,
                const void *Y, int64_t ys, void *out, int64_t os, double *parts,
                cudaStream_t s, const uint8_t *mask = nullptr,
                const char *what = "dmma_hn_kernel");
int lrz_tc_w_ok(int K, int N, int64_t h_stride);
int lrz_tc_w_tiles(int N, int K);
size_t lrz_tc_w_ws(int64_t B, int K);
int lrz_tc_precoder_w(int64_t B, int K, int N, const void *H, const void *A_inv, int64_t ais,
                      void *W, double *parts, void *ws, cudaStream_t s);
// complex64 K > 32 precoder on tcgen05 (3xTF32, tc_tf32.cu) unless LRZ_TC=0 (A/B runs)
static bool use_tc() {
  static const int v = [] {
    const char *e = getenv("LRZ_TC");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}
// items per tcgen05 precoder launch group: the pre-split A^-1 operand of a
// group (8 (2K)^2 bytes per item) stays within 1 GB of workspace
static int64_t tc_group(int K) {
  const int64_t per = int64_t(8) * (2 * K) * (2 * K);
  return std::max<int64_t>(1, (int64_t(1) << 30) / per);
}
int lrz_precode_dmma32(int dtype, int64_t B, int K, int N, const void *H, int64_t hs, const void *A_inv,
                       int64_t ais, const void *G_true, double alpha, double P_t,
                       const double *noise, int64_t noise_div, void *W, int64_t wst,
                       double *scale, double *rates, double *sinr, double *sum_rate,
                       int32_t *info, cudaStream_t s);
int lrz_use_dmma();
static bool use_dmma() { return lrz_use_dmma() != 0; }
int lrz_use_dmma() {
  static const int v = [] {
    const char *e = getenv("LRZ_SIMT_FP64");
    return (e && e[0] == '1') ? 0 : 1;
  }();
  return v != 0;
}

extern "C" int lrz_gram(int dtype, int64_t B, int K, int N, const void *H, int64_t h_stride,
                        double alpha, void *A, int64_t a_stride, void *stream) {
  if (B < 0 || K < 1 || N < 1 || !H || !A) {
    lrz_set_error("lrz_gram: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (use_dmma()) return lrz_gram_dmma(dtype, B, K, N, H, h_stride, alpha, A, a_stride, s);
  if (K <= 32) {
    const unsigned nb = unsigned((B + G32_IPB - 1) / G32_IPB);
    if (dtype == LRZ_C64) {
      const size_t sm = size_t(3) * G32_IPB * G32_BK * 32 * sizeof(c64);
      cudaFuncSetAttribute(gram32_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(sm));
      gram32_kernel<float><<<nb, G32_THREADS, sm, s>>>(B, K, N, (const c64 *)H, h_stride, alpha,
                                                       (c128 *)A, a_stride);
    } else {
      const size_t sm = size_t(3) * G32_IPB * G32_BK * 32 * sizeof(c128);
      cudaFuncSetAttribute(gram32_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(sm));
      gram32_kernel<double><<<nb, G32_THREADS, sm, s>>>(B, K, N, (const c128 *)H, h_stride,
                                                        alpha, (c128 *)A, a_stride);
    }
    return lrz_launch_status("lrz_gram");
  }
  const int nt = ntiles(K), ntl = nt * (nt + 1) / 2;
  const dim3 grid(unsigned(B * ntl));
  if (dtype == LRZ_C64)
    gram_kernel<float, 32><<<grid, GEMM_THREADS, 0, s>>>(K, N, (const c64 *)H, h_stride, alpha,
                                                         (c128 *)A, a_stride, ntl);
  else
    gram_kernel<double, 32><<<grid, GEMM_THREADS, 0, s>>>(K, N, (const c128 *)H, h_stride,
                                                          alpha, (c128 *)A, a_stride, ntl);
  return lrz_launch_status("lrz_gram");
}

extern "C" int lrz_gram_delta(int dtype, int64_t B, int K, int N, const void *P,
                              int64_t p_stride, const void *Q, int64_t q_stride, int mode,
                              void *dA, int64_t a_stride, void *stream) {
  if (B < 0 || K < 1 || N < 1 || !P || !Q || !dA || (mode != 0 && mode != 1)) {
    lrz_set_error("lrz_gram_delta: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const int nt = ntiles(K), ntl = nt * (nt + 1) / 2;
  const dim3 grid(unsigned(B * ntl));
  cudaStream_t s = (cudaStream_t)stream;
  LrzProf prof("gram_delta_kernel", s);
  if (dtype == LRZ_C64)
    gram_delta_kernel<float, 16><<<grid, GEMM_THREADS, 0, s>>>(
        K, N, (const c64 *)P, p_stride, (const c64 *)Q, q_stride, mode, (c128 *)dA, a_stride,
        ntl);
  else
    gram_delta_kernel<double, 16><<<grid, GEMM_THREADS, 0, s>>>(
        K, N, (const c128 *)P, p_stride, (const c128 *)Q, q_stride, mode, (c128 *)dA,
        a_stride, ntl);
  return lrz_launch_status("lrz_gram_delta");
}

// Y = dA Omega_all with Omega read from the normal window (lrz_arsvd's front end)
int lrz_sketch_gemm(int64_t B, int K, int Dtot, const void *dA, int64_t a_stride,
                    const double *omega, int64_t omega_stride, const int32_t *omega_row,
                    int64_t orow_div, const int64_t *cursor, int k_init, int p,
                    const uint8_t *mask, void *Y, void *W, void *stream) {
  const int tn = (Dtot + TM - 1) / TM, tm = (K + TM - 1) / TM;
  SketchOperand so{omega, omega_stride, omega_row, orow_div, cursor, k_init, p};
  const bool fuse = W != nullptr && K <= TM;
  if (fuse && use_dmma()) {
    LrzProf prof("sketch_dmma_kernel", (cudaStream_t)stream);
    sketch_dmma_kernel<<<unsigned(B * tn), 128, 0, (cudaStream_t)stream>>>(
        K, Dtot, (const c128 *)dA, a_stride, so, mask, (c128 *)Y, tn, (c128 *)W);
    return lrz_launch_status("sketch_dmma_kernel");
  }
  const size_t sm = fuse ? 2 * size_t(TM) * (TM + 1) * sizeof(c128) : 0;
  if (fuse)
    cudaFuncSetAttribute(sketch_cgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  LrzProf prof("sketch_cgemm_kernel", (cudaStream_t)stream);
  sketch_cgemm_kernel<<<unsigned(B * tm * tn), GEMM_THREADS, sm, (cudaStream_t)stream>>>(
      K, Dtot, (const c128 *)dA, a_stride, so, mask, (c128 *)Y, tn,
      fuse ? (c128 *)W : nullptr);
  return lrz_launch_status("sketch_cgemm_kernel");
}

// complex128 batched GEMM without argument checks (opA 3 = conj, no transpose);
// used by the step-parallel Woodbury chain (chain.cu)
int lrz_zgemm_internal(int64_t batch, int M, int N, int Kd, int opA, const void *A, int64_t lda,
                       int64_t sA, int opB, const void *Bm, int64_t ldb, int64_t sB, void *C,
                       int64_t ldc, int64_t sC, cudaStream_t s) {
  if (batch == 0) return LRZ_OK;
  const int tm = ntiles(M), tn = ntiles(N);
  cgemm_kernel<double, double, double, 16><<<unsigned(batch * tm * tn), GEMM_THREADS, 0, s>>>(
      M, N, Kd, opA, (const c128 *)A, lda, sA, opB, (const c128 *)Bm, ldb, sB, (c128 *)C, ldc,
      sC, nullptr, tm, tn);
  return lrz_launch_status("cgemm_kernel (chain)");
}

extern "C" int lrz_cgemm(int dtype, int64_t batch, int M, int N, int Kd, int opA,
                         const void *A, int64_t lda, int64_t sA, int opB, const void *Bm,
                         int64_t ldb, int64_t sB, void *C, int64_t ldc, int64_t sC,
                         void *stream) {
  if (batch < 0 || M < 1 || N < 1 || Kd < 1 || !A || !Bm || !C || opA < 0 || opA > 2 ||
      opB < 0 || opB > 2) {
    lrz_set_error("lrz_cgemm: bad arguments");
    return LRZ_EINVAL;
  }
  if (batch == 0) return LRZ_OK;
  const int tm = ntiles(M), tn = ntiles(N);
  const dim3 grid(unsigned(batch * tm * tn));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == LRZ_C64)
    cgemm_kernel<float, float, float, 16><<<grid, GEMM_THREADS, 0, s>>>(
        M, N, Kd, opA, (const c64 *)A, lda, sA, opB, (const c64 *)Bm, ldb, sB, (c64 *)C, ldc,
        sC, nullptr, tm, tn);
  else
    cgemm_kernel<double, double, double, 16><<<grid, GEMM_THREADS, 0, s>>>(
        M, N, Kd, opA, (const c128 *)A, lda, sA, opB, (const c128 *)Bm, ldb, sB, (c128 *)C,
        ldc, sC, nullptr, tm, tn);
  return lrz_launch_status("lrz_cgemm");
}

extern "C" int lrz_fro2(int dtype, int64_t batch, int64_t n, const void *X, int64_t sX,
                        double *out, void *stream) {
  if (batch < 0 || n < 0 || !X || !out) {
    lrz_set_error("lrz_fro2: bad arguments");
    return LRZ_EINVAL;
  }
  if (batch == 0) return LRZ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == LRZ_C64)
    fro2_kernel<float><<<unsigned(batch), 256, 0, s>>>(n, (const c64 *)X, sX, out);
  else
    fro2_kernel<double><<<unsigned(batch), 256, 0, s>>>(n, (const c128 *)X, sX, out);
  return lrz_launch_status("lrz_fro2");
}

extern "C" int lrz_sinr_rate(int dtype, int64_t batch, int K, const void *G, int64_t sG,
                             const double *scale, const double *noise, int64_t noise_div,
                             double *rates, double *sinr, double *sum_rate, void *stream) {
  if (batch < 0 || K < 1 || !G || !noise || noise_div < 1) {
    lrz_set_error("lrz_sinr_rate: bad arguments");
    return LRZ_EINVAL;
  }
  if (batch == 0) return LRZ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  static const double one = 1.0;
  (void)one;
  if (dtype == LRZ_C64)
    sinr_kernel<float><<<unsigned(batch), 256, 0, s>>>(K, (const c64 *)G, sG, scale, nullptr, 0,
                                                       1.0, nullptr, noise, noise_div, rates,
                                                       sinr, sum_rate, nullptr);
  else
    sinr_kernel<double><<<unsigned(batch), 256, 0, s>>>(K, (const c128 *)G, sG, scale, nullptr,
                                                        0, 1.0, nullptr, noise, noise_div,
                                                        rates, sinr, sum_rate, nullptr);
  return lrz_launch_status("lrz_sinr_rate");
}

// K6: fully digital precoder + rate for B items.  Workspace layout:
//   [coupling B*K*K of dtype][norm partials B*tiles doubles][W if W==NULL]
size_t lrz_precode_ws(int dtype, int64_t B, int K, int N) {
  const size_t es = 16;  // coupling buffer sized for complex128 (Gram shortcut)
  const size_t tiles = size_t(ntiles(N)) * ntiles(K);
  size_t bytes = size_t(B) * K * K * es;
  bytes = (bytes + 255) & ~size_t(255);
  bytes += size_t(B) * tiles * sizeof(double);
  bytes = (bytes + 255) & ~size_t(255);
  bytes += size_t(B) * N * K * (dtype == LRZ_C64 ? 8 : 16);  // W (input precision)
  bytes = (bytes + 1023) & ~size_t(1023);
  if (dtype == LRZ_C64 && K > 32 && K <= 256)  // tcgen05 precoder: pre-split A^-1 operand
    bytes += lrz_tc_w_ws(std::min<int64_t>(B, tc_group(K)), K);
  return bytes;
}

int lrz_w_dmma_direct(int dtype, int64_t B, int K, int N, const void *H, int64_t hs,
                      const void *A_inv, int64_t ais, void *W, int64_t wstr, double *parts,
                      cudaStream_t s, const char *what = "w_dmma_direct_kernel");
// (used for K >= 256: with a short reduction the 32 x 32 register tile's prologue and
// epilogue dominate -- the coupling at K = 128 measured 11.5 -> 14 ms per 20,480 items)
static int w_kmin() {  // smallest K of the direct / 3M kernels (LRZ_W_KMIN)
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LRZ_W_KMIN");
    v = e ? atoi(e) : 33;  // the 3M tiled kernel measured faster from K = 64 (dmma.cu)
  }
  return v;
}
static int w_direct() {  // LRZ_W_DIRECT=0: the shared-memory tiled kernel (dmma_tiled.cu)
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LRZ_W_DIRECT");
    v = e ? atoi(e) : 1;
  }
  return v;
}

extern "C" int lrz_precode_rate(int dtype, int64_t B, int K, int N, const void *H,
                                int64_t h_stride, const void *A_inv, int64_t ai_stride,
                                double P_t, const double *noise, int64_t noise_div, void *W,
                                int64_t w_stride, const void *G_true, double alpha,
                                double *scale, double *rates, double *sinr, double *sum_rate,
                                int32_t *info, void *workspace, void *stream) {
  if (B < 0 || K < 1 || N < 1 || !H || !A_inv || !noise || !workspace || noise_div < 1) {
    lrz_set_error("lrz_precode_rate: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  char *ws = (char *)workspace;
  void *Gc = ws;
  size_t off = (size_t(B) * K * K * 16 + 255) & ~size_t(255);
  double *parts = (double *)(ws + off);
  const int tm = ntiles(N), tn = ntiles(K);
  off += size_t(B) * tm * tn * sizeof(double);
  off = (off + 255) & ~size_t(255);
  size_t off_w = off;
  if (!W) {
    W = ws + off;
    w_stride = int64_t(N) * K;
  }
  void *tc_ws = ws + ((off_w + size_t(B) * N * K * (dtype == LRZ_C64 ? 8 : 16) + 1023) &
                      ~size_t(1023));
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 g1(unsigned(B * tm * tn)), g2(unsigned(B * tn * tn));
  if (G_true) {
    // W = H^H A^-1 (norm partials in the epilogue), coupling from the Gram:
    // H W = (G - alpha I) A^-1, K^3 instead of K^2 N work (F_RF = I)
    if (K <= 32 && use_dmma())
      return lrz_precode_dmma32(dtype, B, K, N, H, h_stride, A_inv, ai_stride, G_true, alpha, P_t,
                                noise, noise_div, W, w_stride, scale, rates, sinr, sum_rate,
                                info, s);
    int nparts = tm * tn;
    if (K > 32 && use_dmma()) {
      int np_w = lrz_dmma_hn_tiles(N, K);
      if (dtype == LRZ_C64 && use_tc() && lrz_tc_w_ok(K, N, h_stride) &&
          w_stride == int64_t(N) * K) {
        // complex64: W = H^H A^-1 on tcgen05 (3xTF32, TMA tiles, TMEM accumulator)
        np_w = lrz_tc_w_tiles(N, K);
        const int64_t G = tc_group(K);
        for (int64_t b0 = 0; b0 < B; b0 += G) {
          const int64_t g = std::min<int64_t>(G, B - b0);
          if (int rc = lrz_tc_precoder_w(g, K, N, (const c64 *)H + b0 * h_stride,
                                         (const c128 *)A_inv + b0 * ai_stride, ai_stride,
                                         (c64 *)W + b0 * w_stride, parts + b0 * np_w, tc_ws, s))
            return rc;
        }
      } else if (w_direct() && K >= w_kmin() && w_stride == int64_t(N) * K) {
        // one warp per 32 x 32 block of W, fragments straight from global memory
        np_w = ((N + 31) / 32) * ((K + 31) / 32);
        if (int rc = lrz_w_dmma_direct(dtype, B, K, N, H, h_stride, A_inv, ai_stride, W, w_stride,
                                       parts, s))
          return rc;
      } else if (int rc = lrz_dmma_hn(dtype, B, N, K, K, H, h_stride, N, A_inv, ai_stride, W,
                                      w_stride, parts, s, nullptr, "dmma_hn_kernel:W")) {
        // FP64 tensor pipe, 64 x 64 output tiles, k streamed (dmma_tiled.cu):
        // W = H^H A^-1 with per-CTA norm partials, then the coupling G A^-1
        return rc;
      }
      // the coupling G A^-1 = conj(G)^T A^-1 (G Hermitian): the same product with N = K
      if (w_direct() && K >= w_kmin()) {
        if (int rc = lrz_w_dmma_direct(LRZ_C128, B, K, K, G_true, int64_t(K) * K, A_inv,
                                       ai_stride, Gc, int64_t(K) * K, nullptr, s, "coupling_dmma_direct"))
          return rc;
      } else if (int rc = lrz_dmma_hn(LRZ_C128, B, K, K, K, G_true, int64_t(K) * K, K, A_inv,
                                      ai_stride, Gc, int64_t(K) * K, nullptr, s, nullptr,
                                      "dmma_hn_kernel:coupling"))
        return rc;
      LrzProf prof("sinr_kernel", s);
      sinr_kernel<double><<<unsigned(B), 256, 0, s>>>(
          K, (const c128 *)Gc, int64_t(K) * K, nullptr, parts, np_w, P_t,
          scale, noise, noise_div, rates, sinr, sum_rate, info, (const c128 *)A_inv, ai_stride,
          alpha);
      return lrz_launch_status("lrz_precode_rate");
    }
    if (K <= 32) {
      const size_t es = dtype == LRZ_C64 ? 8 : 16;
      const size_t sm = (32 * 32 + 2 * PW_KC * PW_ROWS) * es;
      nparts = 1;
      if (dtype == LRZ_C64) {
        cudaFuncSetAttribute(precoder_w32_kernel<float>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        precoder_w32_kernel<float><<<unsigned(B), PW_THREADS, sm, s>>>(
            K, N, (const c64 *)H, h_stride, (const c128 *)A_inv, ai_stride, (c64 *)W, w_stride,
            parts);
        if (int rc = lrz_launch_status("precoder_w32_kernel<float>")) return rc;
      } else {
        cudaFuncSetAttribute(precoder_w32_kernel<double>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        precoder_w32_kernel<double><<<unsigned(B), PW_THREADS, sm, s>>>(
            K, N, (const c128 *)H, h_stride, (const c128 *)A_inv, ai_stride, (c128 *)W,
            w_stride, parts);
        if (int rc = lrz_launch_status("precoder_w32_kernel<double>")) return rc;
      }
    } else if (K <= 64) {
      const size_t sm = size_t(K) * K * (dtype == LRZ_C64 ? 8 : 16);
      nparts = 1;
      if (dtype == LRZ_C64) {
        cudaFuncSetAttribute(precoder_w_kernel<float, 16>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        precoder_w_kernel<float, 16><<<unsigned(B), 256, sm, s>>>(
            K, N, (const c64 *)H, h_stride, (const c128 *)A_inv, ai_stride, (c64 *)W, w_stride,
            parts);
      } else {
        cudaFuncSetAttribute(precoder_w_kernel<double, 16>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        precoder_w_kernel<double, 16><<<unsigned(B), 256, sm, s>>>(
            K, N, (const c128 *)H, h_stride, (const c128 *)A_inv, ai_stride, (c128 *)W,
            w_stride, parts);
      }
    } else if (dtype == LRZ_C64)
      cgemm_kernel<float, float, double, 16><<<g1, GEMM_THREADS, 0, s>>>(
          N, K, K, 2, (const c64 *)H, N, h_stride, 0, (const c128 *)A_inv, K, ai_stride,
          (c64 *)W, K, w_stride, parts, tm, tn);
    else
      cgemm_kernel<double, double, double, 16><<<g1, GEMM_THREADS, 0, s>>>(
          N, K, K, 2, (const c128 *)H, N, h_stride, 0, (const c128 *)A_inv, K, ai_stride,
          (c128 *)W, K, w_stride, parts, tm, tn);
    cgemm_kernel<double, double, double, 16><<<g2, GEMM_THREADS, 0, s>>>(
        K, K, K, 0, (const c128 *)G_true, K, int64_t(K) * K, 0, (const c128 *)A_inv, K,
        ai_stride, (c128 *)Gc, K, int64_t(K) * K, nullptr, tn, tn);
    if (int rc = lrz_launch_status("coupling cgemm")) return rc;
    sinr_kernel<double><<<unsigned(B), 256, 0, s>>>(
        K, (const c128 *)Gc, int64_t(K) * K, nullptr, parts, nparts, P_t, scale, noise,
        noise_div, rates, sinr, sum_rate, info, (const c128 *)A_inv, ai_stride, alpha);
    return lrz_launch_status("lrz_precode_rate");
  }
  if (dtype == LRZ_C64) {
    // W[n][j] = sum_k conj(H[k][n]) A_inv[k][j]     (precoding.py:47)
    cgemm_kernel<float, float, double, 16><<<g1, GEMM_THREADS, 0, s>>>(
        N, K, K, 2, (const c64 *)H, N, h_stride, 0, (const c128 *)A_inv, K, ai_stride,
        (c64 *)W, K, w_stride, parts, tm, tn);
    // G = H W                                           (precoding.py:74)
    cgemm_kernel<float, float, float, 16><<<g2, GEMM_THREADS, 0, s>>>(
        K, K, N, 0, (const c64 *)H, N, h_stride, 0, (const c64 *)W, K, w_stride, (c64 *)Gc, K,
        int64_t(K) * K, nullptr, tn, tn);
    sinr_kernel<float><<<unsigned(B), 256, 0, s>>>(K, (const c64 *)Gc, int64_t(K) * K, nullptr,
                                                   parts, tm * tn, P_t, scale, noise, noise_div,
                                                   rates, sinr, sum_rate, info);
  } else {
    cgemm_kernel<double, double, double, 16><<<g1, GEMM_THREADS, 0, s>>>(
        N, K, K, 2, (const c128 *)H, N, h_stride, 0, (const c128 *)A_inv, K, ai_stride,
        (c128 *)W, K, w_stride, parts, tm, tn);
    cgemm_kernel<double, double, double, 16><<<g2, GEMM_THREADS, 0, s>>>(
        K, K, N, 0, (const c128 *)H, N, h_stride, 0, (const c128 *)W, K, w_stride, (c128 *)Gc,
        K, int64_t(K) * K, nullptr, tn, tn);
    sinr_kernel<double><<<unsigned(B), 256, 0, s>>>(K, (const c128 *)Gc, int64_t(K) * K,
                                                    nullptr, parts, tm * tn, P_t, scale, noise,
                                                    noise_div, rates, sinr, sum_rate, info);
  }
  return lrz_launch_status("lrz_precode_rate");
}
