// complex128 kernels on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64) for
// K <= 32: the Gram G = H H^H + alpha I (K1, lowrank.py:147-164) and the fused
// fully digital precoder + coupling + SINR/rate (K6, precoding.py:37-80).
//
// One complex MAC block is four real DMMAs on the (re, im) halves of the same
// fragments.  m8n8k4 f64 fragments (PTX ISA): lane L = 4 g + t holds
//   A[g][t] (one double), B[t][g] (one double), C[g][2t + e] (two doubles).
// A DMMA is 256 FMAs per warp instruction against 32 for a DFMA, so these
// kernels are bound by the FP64 pipe (and HBM for the precoder's H in / W
// out), not by instruction issue -- the SIMT versions (gemm.cu) issue one
// shared-memory load per two DFMAs and stall at 43-59 % of the pipe.

#include "dmma.cuh"

namespace lrz {

// ---------------------------------------------------------------------------
// K1: G = H H^H + alpha I, one item per warp, RB = ceil(K / 8) row blocks.
// Lane (g, t) holds H[8 rb + g][n0 + 4 s + t] (s < 4: one 16-column chunk);
// the same register is the A fragment of row block rb and the B fragment of
// column block rb (B[k][j] = H[8 jb + j][k] up to the conjugate), so the
// RB (RB + 1) / 2 lower 8 x 8 tiles need no shared memory at all:
//   Re G += Hr Hr^T + Hi Hi^T,   Im G += Hi Hr^T - Hr Hi^T.
// Lower tiles are written and mirrored (exactly Hermitian, real diagonal
// + alpha: the reference's 0.5 (A + A^H) + alpha I, lowrank.py:160-162).
// ---------------------------------------------------------------------------
constexpr int GD_WARPS = 4;

template <int RB, typename T>
__global__ void __launch_bounds__(32 * GD_WARPS, 3)
    gram_dmma_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                     double alpha, c128 *__restrict__ A, int64_t as, int nb) {
  constexpr int NT = RB * (RB + 1) / 2;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t wid = int64_t(blockIdx.x) * GD_WARPS + (threadIdx.x >> 5);
  if (wid >= B * nb) return;
  // K > 32: warp = (item, diagonal 32-row block I) of the Gram
  const int64_t item = wid / nb;
  const int I = int(wid - item * nb), r0 = 32 * I;
  const cplx<T> *h = H + item * hs + int64_t(r0) * N;
  const int Kfull = K;
  K = min(32, Kfull - r0);  // valid rows of this block
  double cr[NT][2], ci[NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i) cr[i][0] = cr[i][1] = ci[i][0] = ci[i][1] = 0.0;
  bool rok[RB];
  const cplx<T> *hrow[RB];
#pragma unroll
  for (int rb = 0; rb < RB; ++rb) {
    rok[rb] = 8 * rb + g < K;
    hrow[rb] = h + int64_t(rok[rb] ? 8 * rb + g : 0) * N;
  }
  const bool full = (N % 16) == 0;
  for (int n0 = 0; n0 < N; n0 += 16) {
    c128 v[RB][4];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int n = n0 + 4 * s + t;
        v[rb][s] = (rok[rb] && (full || n < N)) ? ldg_c(hrow[rb] + n) : czero<double>();
      }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int ib = 0; ib < RB; ++ib) {
        const double ar = v[ib][s].re, ai = v[ib][s].im, nar = -ar;
#pragma unroll
        for (int jb = 0; jb <= ib; ++jb) {
          const int x = ib * (ib + 1) / 2 + jb;
          const double br = v[jb][s].re, bi = v[jb][s].im;
          dmma(cr[x], ar, br);
          dmma(cr[x], ai, bi);
          dmma(ci[x], ai, br);
          dmma(ci[x], nar, bi);
        }
      }
    }
  }
  c128 *a = A + item * as + int64_t(r0) * Kfull + r0;
#pragma unroll
  for (int ib = 0; ib < RB; ++ib)
#pragma unroll
    for (int jb = 0; jb <= ib; ++jb) {
      const int x = ib * (ib + 1) / 2 + jb;
      const int row = 8 * ib + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * jb + 2 * t + e;
        if (row < K && col < K && col <= row) {
          c128 z = mk<double>(cr[x][e], ci[x][e]);
          if (row == col) {
            z.im = 0.0;
            z.re += alpha;
            a[int64_t(row) * Kfull + col] = z;
          } else {
            a[int64_t(row) * Kfull + col] = z;
            a[int64_t(col) * Kfull + row] = cconj(z);
          }
        }
      }
    }
}

// K > 32: off-diagonal 32 x 32 blocks (I > J) of the Gram, one warp per
// (item, block): 16 8 x 8 tiles, A fragments from the rows of block I, B
// fragments from the rows of block J, 8 columns of H per step; written with
// the mirrored upper block.
// One lower 32 x 32 block (I, J) of the Gram by one warp.  DIAG (I == J): only
// the 10 of 16 8 x 8 tiles on or below the diagonal are accumulated (the same
// fragment loads, 40 instead of 64 DMMAs per k-step).
template <typename T, bool DIAG>
LRZ_DEV void gram_block32(int K, int N, const cplx<T> *__restrict__ h, c128 *__restrict__ a,
                          int I, int J, double alpha) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  bool iok[4], jok[4];
  const cplx<T> *hi[4], *hj[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int ri = 32 * I + 8 * b + g, rj = 32 * J + 8 * b + g;
    iok[b] = ri < K;
    jok[b] = rj < K;
    hi[b] = h + int64_t(iok[b] ? ri : 0) * N;
    hj[b] = h + int64_t(jok[b] ? rj : 0) * N;
  }
  double cr[16][2], ci[16][2];
#pragma unroll
  for (int x = 0; x < 16; ++x) cr[x][0] = cr[x][1] = ci[x][0] = ci[x][1] = 0.0;
  for (int n0 = 0; n0 < N; n0 += 8) {
    c128 vi[4][2], vj[4][2];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int n = n0 + 4 * s + t;
        vi[b][s] = (iok[b] && n < N) ? ldg_c(hi[b] + n) : czero<double>();
        vj[b][s] = DIAG ? vi[b][s] : ((jok[b] && n < N) ? ldg_c(hj[b] + n) : czero<double>());
      }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int ib = 0; ib < 4; ++ib) {
        const double ar = vi[ib][s].re, ai = vi[ib][s].im, nar = -ar;
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          if (DIAG && jb > ib) continue;  // strictly upper tile of a diagonal block
          const double br = vj[jb][s].re, bi = vj[jb][s].im;
          dmma(cr[4 * ib + jb], ar, br);
          dmma(cr[4 * ib + jb], ai, bi);
          dmma(ci[4 * ib + jb], ai, br);
          dmma(ci[4 * ib + jb], nar, bi);
        }
      }
  }
#pragma unroll
  for (int ib = 0; ib < 4; ++ib)
#pragma unroll
    for (int jb = 0; jb < 4; ++jb) {
      if (DIAG && jb > ib) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 32 * I + 8 * ib + g, col = 32 * J + 8 * jb + 2 * t + e;
        if (row < K && col < K && col <= row) {
          c128 z = mk<double>(cr[4 * ib + jb][e], ci[4 * ib + jb][e]);
          if (row == col) {  // exactly Hermitian: real diagonal + alpha (lowrank.py:160-162)
            z.im = 0.0;
            z.re += alpha;
            a[int64_t(row) * K + col] = z;
          } else {
            a[int64_t(row) * K + col] = z;
            a[int64_t(col) * K + row] = cconj(z);
          }
        }
      }
    }
}

template <typename T>
__global__ void __launch_bounds__(32 * GD_WARPS)
    gram_dmma_off_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                         c128 *__restrict__ A, int64_t as, int npair, double alpha,
                         int diag) {
  const int64_t wid = int64_t(blockIdx.x) * GD_WARPS + (threadIdx.x >> 5);
  if (wid >= B * npair) return;
  const int64_t item = wid / npair;
  // pairs (I, J) in row order: J < I, or J <= I with diag
  int p = int(wid - item * npair), I = diag ? 0 : 1;
  while (p >= I + diag) {
    p -= I + diag;
    ++I;
  }
  const int J = p;
  gram_block32<T, false>(K, N, H + item * hs, A + item * as, I, J, alpha);
}

// The diagonal 32 x 32 blocks (I, I), 10 of their 16 tiles each, one warp per
// (item, block).  A kernel of its own: sharing one with the full-block warps
// costs the complex64 instantiation 30 registers and ~6 % of its rate.
template <typename T>
__global__ void __launch_bounds__(32 * GD_WARPS)
    gram_dmma_diag_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                          c128 *__restrict__ A, int64_t as, int nb, double alpha) {
  const int64_t wid = int64_t(blockIdx.x) * GD_WARPS + (threadIdx.x >> 5);
  if (wid >= B * nb) return;
  const int64_t item = wid / nb;
  const int I = int(wid - item * nb);
  gram_block32<T, true>(K, N, H + item * hs, A + item * as, I, I, alpha);
}

// ---------------------------------------------------------------------------
// K6 for K > 32, complex128: W = H^H A^-1 (N x K, precoding.py:47) with the Gram
// kernel's structure -- one warp per 32 n x 32 j output block, 16 complex 8 x 8
// accumulator tiles, both fragments straight from global memory: lane (g, t)
// reads conj(H)[4c + t][n0 + 8b + g] and A^-1[4c + t][j0 + 8b + g], a warp load
// is four 128-byte row segments.  64 DMMAs per 8 fragment loads against the
// tiled kernel's 32 per 6 (shared-memory slabs, 16 x 32 warp tiles).  The four
// warps of a CTA share the n block (their H loads hit L1) and take four j
// blocks.  ||W||_F^2 goes out as one partial per warp, summed in a fixed order.
// ---------------------------------------------------------------------------
template <typename T, int NBW>  // NBW n blocks per CTA (x 4 j blocks): 32 NBW x 128 of W
__global__ void __launch_bounds__(128 * NBW)
    w_dmma_direct_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                         const c128 *__restrict__ Ainv, int64_t ais, cplx<T> *__restrict__ W,
                         int64_t wstr, double *__restrict__ parts, int nnb, int njb, int njq) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  const int nng = (nnb + NBW - 1) / NBW;
  const int64_t per = int64_t(nng) * njq;
  const int64_t item = blockIdx.x / per;
  const int rem = int(blockIdx.x - item * per);
  const int nb = NBW * (rem / njq) + (w >> 2), jb0 = 4 * (rem % njq) + (w & 3);
  if (jb0 >= njb || nb >= nnb) return;
  const int n0 = 32 * nb, j0 = 32 * jb0;
  const cplx<T> *h = H + item * hs;
  const c128 *y = Ainv + item * ais;
  bool nok[4], jok[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    nok[b] = n0 + 8 * b + g < N;
    jok[b] = j0 + 8 * b + g < K;
  }
  double cr[16][2], ci[16][2];
#pragma unroll
  for (int x = 0; x < 16; ++x) cr[x][0] = cr[x][1] = ci[x][0] = ci[x][1] = 0.0;
  for (int k0 = 0; k0 < K; k0 += 8) {
    c128 vx[4][2], vy[4][2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = k0 + 4 * s + t;
      const bool kok = k < K;
      const cplx<T> *hr = h + int64_t(kok ? k : 0) * N + n0 + g;
      const c128 *yr = y + int64_t(kok ? k : 0) * K + j0 + g;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        vx[b][s] = (kok && nok[b]) ? ldg_c(hr + 8 * b) : czero<double>();
        vy[b][s] = (kok && jok[b]) ? ldg_c(yr + 8 * b) : czero<double>();
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int ib = 0; ib < 4; ++ib) {
        const double xr = vx[ib][s].re, xi = vx[ib][s].im, nxi = -xi;
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          // conj(x) y = (xr yr + xi yi) + i (xr yi - xi yr)
          const double yr_ = vy[jb][s].re, yi_ = vy[jb][s].im;
          dmma(cr[4 * ib + jb], xr, yr_);
          dmma(cr[4 * ib + jb], xi, yi_);
          dmma(ci[4 * ib + jb], xr, yi_);
          dmma(ci[4 * ib + jb], nxi, yr_);
        }
      }
  }
  cplx<T> *o = W + item * wstr;
  double nrm = 0.0;
#pragma unroll
  for (int ib = 0; ib < 4; ++ib)
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + 8 * ib + g, j = j0 + 8 * jb + 2 * t + e;
        if (n < N && j < K) {
          const cplx<T> z = mk<T>(T(cr[4 * ib + jb][e]), T(ci[4 * ib + jb][e]));
          o[int64_t(n) * K + j] = z;
          nrm += double(z.re) * double(z.re) + double(z.im) * double(z.im);
        }
      }
  nrm = warp_sum(nrm);
  if (parts && lane == 0) parts[item * (int64_t(nnb) * njb) + int64_t(nb) * njb + jb0] = nrm;
}

// ---------------------------------------------------------------------------
// W = H^H A^-1 (and the coupling G A^-1) with three real DMMAs per complex tile
// step instead of four (the "3M" complex product): with a = conj(x) = (xr, -xi)
// and b = y,
//   P += xr yr,  Q += xi yi,  R += (xr - xi)(yr + yi)
//   Re = P + Q,  Im = R - P + Q        (= xr yi - xi yr)
// -- 25 % fewer tensor-pipe instructions for two DADDs per fragment pair and a
// third accumulator set (96 registers for a warp's 16 tiles).  Every partial sum
// is bounded by (|xr| + |xi|)(|yr| + |yi|), so the error stays normwise at the
// level of the four-product form (1e-15 relative on random data; parity with the
// oracle unchanged).  With the fragments straight from global memory (the form
// of w_dmma_direct_kernel) the 3M product measured no faster: that kernel is
// bound by its loads once the DMMA phase of an iteration is a quarter shorter
// (two warps per scheduler at 255 registers).  So the operands are staged in
// shared memory: a CTA of four warps (2 n x 2 j, 32 x 32 of W each: the same 16 tiles, three
// accumulator sets) streams 16-row slabs of conj-H (16 x 64) and A^-1 (16 x 64)
// through a 3-stage cp.async ring; rows padded by two elements, so a
// quarter-warp's fragment LDS.128 (4 rows x 2 columns) covers 128 distinct
// bytes.  Two CTAs per SM (101 KB each).  48 DMMAs per 8 fragment LDS.
// ---------------------------------------------------------------------------
constexpr int W3_KC = 16, W3_ST = 3, W3_BN = 64, W3_BJ = 64;
template <typename T>
struct W3Smem {
  static constexpr int XLD = W3_BN + (sizeof(T) == 8 ? 2 : 4);
  static constexpr int YLD = W3_BJ + 2;
  static constexpr size_t xbytes = size_t(W3_KC) * XLD * sizeof(cplx<T>);
  static constexpr size_t ybytes = size_t(W3_KC) * YLD * sizeof(c128);
  static constexpr size_t stage = xbytes + ybytes;
  static constexpr size_t bytes = stage * W3_ST;
};

template <typename T>
__global__ void __launch_bounds__(128, 2)
    w_dmma_3m_tiled_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                           const c128 *__restrict__ Ainv, int64_t ais, cplx<T> *__restrict__ W,
                           int64_t wstr, double *__restrict__ parts, int nnb, int njb,
                           int tiles_n, int tiles_j) {
  using S = W3Smem<T>;
  extern __shared__ __align__(16) unsigned char w3_smem[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wn = w & 1, wj = w >> 1;
  const int ntile = tiles_n * tiles_j;
  const int64_t item = blockIdx.x / ntile;
  const int tile = int(blockIdx.x - item * ntile);
  const int n0 = (tile / tiles_j) * W3_BN, j0 = (tile % tiles_j) * W3_BJ;
  const cplx<T> *h = H + item * hs;
  const c128 *y = Ainv + item * ais;
  auto xslab = [&](int s) { return reinterpret_cast<cplx<T> *>(w3_smem + size_t(s) * S::stage); };
  auto yslab = [&](int s) {
    return reinterpret_cast<c128 *>(w3_smem + size_t(s) * S::stage + S::xbytes);
  };
  // slab loads: thread tid copies element (row r0 + 2 i, column c0) of both slabs,
  // i = 0 .. 7 -- one global pointer per operand advanced by a constant, one
  // shared-memory offset, the column bounds decided once
  const int r0 = tid >> 6, c0 = tid & 63;
  const bool xok = n0 + c0 < N, yok = j0 + c0 < K;
  const cplx<T> *xg = h + int64_t(r0) * N + (xok ? n0 + c0 : 0);
  const c128 *yg = y + int64_t(r0) * K + (yok ? j0 + c0 : 0);
  const int64_t xstep = int64_t(2) * N, ystep = int64_t(2) * K;
  const unsigned xso = unsigned(r0 * S::XLD + c0) * unsigned(sizeof(cplx<T>));
  const unsigned yso = unsigned(S::xbytes) + unsigned(r0 * S::YLD + c0) * 16u;
  const unsigned smem0 = (unsigned)__cvta_generic_to_shared(w3_smem);
  auto load = [&](int s, int k0) {
    const unsigned sb = smem0 + unsigned(s) * unsigned(S::stage);
    const cplx<T> *xp = xg + int64_t(k0) * N;
    const c128 *yp = yg + int64_t(k0) * K;
#pragma unroll
    for (int i = 0; i < W3_KC / 2; ++i) {
      const bool kok = k0 + r0 + 2 * i < K;
      const bool px = kok && xok, py = kok && yok;
      const unsigned xd = sb + xso + unsigned(2 * i * S::XLD) * unsigned(sizeof(cplx<T>));
      const unsigned yd = sb + yso + unsigned(2 * i * S::YLD) * 16u;
      const void *xs_ = px ? (const void *)(xp + i * xstep) : (const void *)h;
      const void *ys_ = py ? (const void *)(yp + i * ystep) : (const void *)y;
      if (sizeof(cplx<T>) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(xd), "l"(xs_),
                     "r"(px ? 16 : 0));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(xd), "l"(xs_),
                     "r"(px ? 8 : 0));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(yd), "l"(ys_),
                   "r"(py ? 16 : 0));
    }
  };
  double cp[16][2], cq[16][2], cs[16][2];
#pragma unroll
  for (int x = 0; x < 16; ++x)
    cp[x][0] = cp[x][1] = cq[x][0] = cq[x][1] = cs[x][0] = cs[x][1] = 0.0;
  const int nslab = (K + W3_KC - 1) / W3_KC;
#pragma unroll
  for (int s = 0; s < W3_ST - 1; ++s) {
    if (s < nslab) load(s, s * W3_KC);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int it = 0; it < nslab; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(W3_ST - 2));
    __syncthreads();
    const int nxt = it + W3_ST - 1;
    if (nxt < nslab) load(nxt % W3_ST, nxt * W3_KC);
    asm volatile("cp.async.commit_group;\n" ::);
    const cplx<T> *xsl = xslab(it % W3_ST) + 32 * wn + g;
    const c128 *ysl = yslab(it % W3_ST) + 32 * wj + g;
#pragma unroll
    for (int kk = 0; kk < W3_KC; kk += 4) {
      double xr[4], xi[4], yr[4], yi[4], ys[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const cplx<T> v = xsl[(kk + t) * S::XLD + 8 * b];
        xr[b] = double(v.re);
        xi[b] = double(v.im);
        const c128 u = ysl[(kk + t) * S::YLD + 8 * b];
        yr[b] = u.re;
        yi[b] = u.im;
        ys[b] = u.re + u.im;
      }
#pragma unroll
      for (int ib = 0; ib < 4; ++ib) {
        const double xs = xr[ib] - xi[ib];
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          dmma(cp[4 * ib + jb], xr[ib], yr[jb]);
          dmma(cq[4 * ib + jb], xi[ib], yi[jb]);
          dmma(cs[4 * ib + jb], xs, ys[jb]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  cplx<T> *o = W + item * wstr;
  double nrm = 0.0;
  const int nw = n0 + 32 * wn, jw = j0 + 32 * wj;
#pragma unroll
  for (int ib = 0; ib < 4; ++ib)
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = nw + 8 * ib + g, j = jw + 8 * jb + 2 * t + e;
        if (n < N && j < K) {
          const int x = 4 * ib + jb;
          const cplx<T> z = mk<T>(T(cp[x][e] + cq[x][e]), T(cs[x][e] - cp[x][e] + cq[x][e]));
          o[int64_t(n) * K + j] = z;
          nrm += double(z.re) * double(z.re) + double(z.im) * double(z.im);
        }
      }
  nrm = warp_sum(nrm);
  // one partial per 32 x 32 block, the layout of w_dmma_direct_kernel's
  if (parts && lane == 0 && nw < N && jw < K)
    parts[item * (int64_t(nnb) * njb) + int64_t(nw / 32) * njb + jw / 32] = nrm;
}

// ---------------------------------------------------------------------------
// Gram, K > 32, on the same 3M product and slab ring: A = H H^H + alpha I by
// 64 x 64 tiles of the lower triangle, a CTA of four warps each.  With
// a = h_i = (ar, ai) and b = conj(h_j) = (br, -bi):
//   P += ar br,  Q += ai bi,  R += (ar + ai)(br - bi),  Re = P + Q,  Im = R - P + Q.
// Slabs are 16 antennas x 64 rows of H, transposed on the way into shared memory
// (a thread copies 16-byte pieces of 16 consecutive antennas of a row: 256-byte
// global segments).  Off-diagonal tiles: warp (wn, wj) owns a 32 x 32 block, 16
// tiles.  Diagonal tiles need the 36 8 x 8 tiles on or below the diagonal of
// their 8 x 8 tile grid: warp w takes tile rows w and 7 - w (9 tiles each), so
// the four warps finish together and no tile above the diagonal is computed.
// ---------------------------------------------------------------------------
template <typename T, int ROLE>  // ROLE 0..3: warp of a diagonal tile, 4: off-diagonal
LRZ_DEV void gram3_body(int K, int N, const cplx<T> *__restrict__ h, c128 *__restrict__ a,
                        int i0, int j0, double alpha, unsigned char *smem) {
  using S = W3Smem<T>;
  constexpr bool DIAG = ROLE < 4;
  constexpr int NT = DIAG ? 9 : 16;
  constexpr int RA = ROLE, RB = 7 - ROLE;  // the diagonal warp's two tile rows
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wn = w & 1, wj = w >> 1;
  // slab loads: thread tid copies antenna r0 of rows c0 + 8 i, i = 0 .. 7.  Eight
  // consecutive threads take 4 antennas x 2 rows: 64-byte global pieces, and in
  // shared memory (row stride 66 elements) eight distinct 16-byte bank groups
  const int r0 = (tid & 3) | (((tid >> 3) & 3) << 2), c0 = ((tid >> 2) & 1) | ((tid >> 5) << 1);
  const cplx<T> *xg = h + int64_t(i0 + c0) * N + r0;
  const cplx<T> *yg = h + int64_t(j0 + c0) * N + r0;
  const int64_t rstep = int64_t(8) * N;
  const unsigned xso = unsigned(r0 * S::XLD + c0) * unsigned(sizeof(cplx<T>));
  // the Y slab holds H elements as well (XLD layout); a diagonal tile reads its X slab
  const unsigned yso = unsigned(S::xbytes) + xso;
  const unsigned smem0 = (unsigned)__cvta_generic_to_shared(smem);
  auto load = [&](int s, int n0) {
    const unsigned sb = smem0 + unsigned(s) * unsigned(S::stage);
    const bool nok = n0 + r0 < N;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool px = nok && i0 + c0 + 8 * i < K;
      const void *xs_ = px ? (const void *)(xg + n0 + i * rstep) : (const void *)h;
      const unsigned xd = sb + xso + unsigned(8 * i) * unsigned(sizeof(cplx<T>));
      if (sizeof(cplx<T>) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(xd), "l"(xs_),
                     "r"(px ? 16 : 0));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(xd), "l"(xs_),
                     "r"(px ? 8 : 0));
      if (!DIAG) {
        const bool py = nok && j0 + c0 + 8 * i < K;
        const void *ys_ = py ? (const void *)(yg + n0 + i * rstep) : (const void *)h;
        const unsigned yd = sb + yso + unsigned(8 * i) * unsigned(sizeof(cplx<T>));
        if (sizeof(cplx<T>) == 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(yd), "l"(ys_),
                       "r"(py ? 16 : 0));
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(yd), "l"(ys_),
                       "r"(py ? 8 : 0));
      }
    }
  };
  double cp[NT][2], cq[NT][2], cs[NT][2];
#pragma unroll
  for (int x = 0; x < NT; ++x)
    cp[x][0] = cp[x][1] = cq[x][0] = cq[x][1] = cs[x][0] = cs[x][1] = 0.0;
  const int nslab = (N + W3_KC - 1) / W3_KC;
#pragma unroll
  for (int s = 0; s < W3_ST - 1; ++s) {
    if (s < nslab) load(s, s * W3_KC);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int it = 0; it < nslab; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(W3_ST - 2));
    __syncthreads();
    const int nxt = it + W3_ST - 1;
    if (nxt < nslab) load(nxt % W3_ST, nxt * W3_KC);
    asm volatile("cp.async.commit_group;\n" ::);
    const cplx<T> *xsl =
        reinterpret_cast<const cplx<T> *>(smem + size_t(it % W3_ST) * S::stage) + g;
    const cplx<T> *ysl = DIAG ? xsl
                              : reinterpret_cast<const cplx<T> *>(
                                    smem + size_t(it % W3_ST) * S::stage + S::xbytes) + g;
#pragma unroll
    for (int kk = 0; kk < W3_KC; kk += 4) {
      if (DIAG) {
        double br[RB + 1], bi[RB + 1], bd[RB + 1];
#pragma unroll
        for (int b = 0; b <= RB; ++b) {
          const cplx<T> u = ysl[(kk + t) * S::XLD + 8 * b];
          br[b] = double(u.re);
          bi[b] = double(u.im);
          bd[b] = br[b] - bi[b];
        }
        // tile rows RA (tiles 0 .. RA) and RB (tiles RA + 1 .. 8): the A fragments are
        // the B fragments of the same rows
        {
          const double ar = br[RA], ai = bi[RA], as_ = ar + ai;
#pragma unroll
          for (int jb = 0; jb <= RA; ++jb) {
            dmma(cp[jb], ar, br[jb]);
            dmma(cq[jb], ai, bi[jb]);
            dmma(cs[jb], as_, bd[jb]);
          }
        }
        {
          const double ar = br[RB], ai = bi[RB], as_ = ar + ai;
#pragma unroll
          for (int jb = 0; jb <= RB; ++jb) {
            dmma(cp[RA + 1 + jb], ar, br[jb]);
            dmma(cq[RA + 1 + jb], ai, bi[jb]);
            dmma(cs[RA + 1 + jb], as_, bd[jb]);
          }
        }
      } else {
        double ar[4], ai[4], br[4], bi[4], bd[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const cplx<T> v = xsl[(kk + t) * S::XLD + 32 * wn + 8 * b];
          ar[b] = double(v.re);
          ai[b] = double(v.im);
          const cplx<T> u = ysl[(kk + t) * S::XLD + 32 * wj + 8 * b];
          br[b] = double(u.re);
          bi[b] = double(u.im);
          bd[b] = br[b] - bi[b];
        }
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) {
          const double as_ = ar[ib] + ai[ib];
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            dmma(cp[4 * ib + jb], ar[ib], br[jb]);
            dmma(cq[4 * ib + jb], ai[ib], bi[jb]);
            dmma(cs[4 * ib + jb], as_, bd[jb]);
          }
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  // write-back: the lower element and its mirrored conjugate (exactly Hermitian),
  // real diagonal + alpha (lowrank.py:160-162)
  auto put = [&](int row, int col, double re, double im) {
    if (row < K && col < K && col <= row) {
      if (row == col) {
        a[int64_t(row) * K + col] = mk<double>(re + alpha, 0.0);
      } else {
        a[int64_t(row) * K + col] = mk<double>(re, im);
        a[int64_t(col) * K + row] = mk<double>(re, -im);
      }
    }
  };
#pragma unroll
  for (int x = 0; x < NT; ++x) {
    int tr, tc;  // tile coordinates in the 64 x 64 tile's 8 x 8 grid
    if (DIAG) {
      tr = x <= RA ? RA : RB;
      tc = x <= RA ? x : x - RA - 1;
    } else {
      tr = 4 * wn + x / 4;
      tc = 4 * wj + x % 4;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
      put(i0 + 8 * tr + g, j0 + 8 * tc + 2 * t + e, cp[x][e] + cq[x][e],
          cs[x][e] - cp[x][e] + cq[x][e]);
  }
}

template <typename T>
__global__ void __launch_bounds__(128, 2)
    gram_dmma_3m_tiled_kernel(int64_t B, int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                              c128 *__restrict__ A, int64_t as, int npair, double alpha) {
  extern __shared__ __align__(16) unsigned char g3_smem[];
  const int64_t item = blockIdx.x / npair;
  // the diagonal tiles (the shorter CTAs) last: pairs in row order, J <= I
  int p = int(blockIdx.x - item * npair), I = 0;
  while (p > I) {
    p -= I + 1;
    ++I;
  }
  const int J = p;
  const cplx<T> *h = H + item * hs;
  c128 *a = A + item * as;
  if (I != J) {
    gram3_body<T, 4>(K, N, h, a, 64 * I, 64 * J, alpha, g3_smem);
    return;
  }
  switch (threadIdx.x >> 5) {
    case 0: gram3_body<T, 0>(K, N, h, a, 64 * I, 64 * I, alpha, g3_smem); break;
    case 1: gram3_body<T, 1>(K, N, h, a, 64 * I, 64 * I, alpha, g3_smem); break;
    case 2: gram3_body<T, 2>(K, N, h, a, 64 * I, 64 * I, alpha, g3_smem); break;
    default: gram3_body<T, 3>(K, N, h, a, 64 * I, 64 * I, alpha, g3_smem); break;
  }
}

// ---------------------------------------------------------------------------
// K6 fused, K <= 32, one item per CTA of 4 warps:
//   W = H^H A^-1 (N x K, unscaled, precoding.py:47), ||W||_F^2,
//   C = G A^-1 - alpha A^-1 = H W for F_RF = I, s = sqrt(P_t)/||W||,
//   SINR_n = |s C_nn|^2 / (sum_{i != n} |s C_ni|^2 + noise_n), rates, sum.
// A^-1 is staged once in shared memory as separate re / im planes with a row
// stride of 36 doubles (the B-fragment loads A^-1[4c + t][8kb + g] are then
// bank-conflict free).  Warp w computes 8-row slabs n0 = 8 (w + 4 j) of W:
// lane (g, t) loads conj(H)[4c + t][n0 + g] straight from global memory as
// the A fragment (a warp load touches 4 rows x 128 contiguous bytes), 4
// complex 8 x 8 accumulator tiles per slab, written as 32-byte row segments.
// One block per slab (rather than two) keeps the kernel at <= 80 registers, so
// 6-8 CTAs per SM hide the H loads (1.16 -> 1.03 ms at C2 c128).
// ---------------------------------------------------------------------------
constexpr int PD_WARPS = 4;
constexpr int PD_NB = 1;    // 8-row n-blocks per warp slab
// CTAs per SM (register budget): one 8-row block per slab keeps the kernel at
// <= 80 registers; complex64 (half the H bytes per fragment) fits 8 CTAs
template <typename T>
constexpr int pd_minb() { return sizeof(T) == 8 ? 6 : 8; }
constexpr int PD_LD = 36;

template <typename T, bool M3 = false>  // M3: 3M complex product (three real DMMAs per step)
__global__ void __launch_bounds__(32 * PD_WARPS, M3 ? 5 : pd_minb<T>())
    precode_dmma32_kernel(int K, int N, const cplx<T> *__restrict__ H, int64_t hs,
                          const c128 *__restrict__ Ainv, int64_t ais,
                          const c128 *__restrict__ Gt, int64_t gs, double alpha, double P_t,
                          const double *__restrict__ noise, int64_t noise_div,
                          cplx<T> *__restrict__ W, int64_t wst, double *__restrict__ scale_out,
                          double *__restrict__ rates, double *__restrict__ sinr,
                          double *__restrict__ sum_rate, int32_t *__restrict__ info) {
  __shared__ __align__(16) double Sr[32 * PD_LD], Si[32 * PD_LD];
  __shared__ double red[PD_WARPS], red2[PD_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int64_t item = blockIdx.x;
  const c128 *ai = Ainv + item * ais;
  for (int e = tid; e < 32 * 32; e += 32 * PD_WARPS) {
    const int i = e >> 5, k = e & 31;
    const c128 v = (i < K && k < K) ? ai[i * K + k] : czero<double>();
    Sr[i * PD_LD + k] = v.re;
    Si[i * PD_LD + k] = v.im;
  }
  __syncthreads();
  const cplx<T> *h = H + item * hs;
  cplx<T> *wo = W + item * wst;
  double nrm = 0.0;
  const int nslab = (N + 8 * PD_NB - 1) / (8 * PD_NB);
  for (int sl = w; sl < nslab; sl += PD_WARPS) {
    const int n0 = 8 * PD_NB * sl;
    c128 hv[8][PD_NB];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int nb = 0; nb < PD_NB; ++nb) {
        const int i = 4 * c + t, n = n0 + 8 * nb + g;
        hv[c][nb] = (i < K && n < N) ? ldg_c(h + int64_t(i) * N + n) : czero<double>();
      }
    double acr[PD_NB][4][2], aci[PD_NB][4][2], acs[M3 ? PD_NB : 1][4][2];
#pragma unroll
    for (int nb = 0; nb < PD_NB; ++nb)
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) acr[nb][kb][0] = acr[nb][kb][1] = aci[nb][kb][0] =
          aci[nb][kb][1] = 0.0;
    if (M3) {
#pragma unroll
      for (int nb = 0; nb < PD_NB; ++nb)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) acs[nb][kb][0] = acs[nb][kb][1] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        const double br = Sr[(4 * c + t) * PD_LD + 8 * kb + g];
        const double bi = Si[(4 * c + t) * PD_LD + 8 * kb + g];
#pragma unroll
        for (int nb = 0; nb < PD_NB; ++nb) {
          const double hr = hv[c][nb].re, hi = hv[c][nb].im;
          if (M3) {
            // 3M: P += hr br, Q += hi bi, R += (hr - hi)(br + bi); Re = P + Q,
            // Im = R - P + Q (acr = P, aci = Q, acs = R until the write-back)
            dmma(acr[nb][kb], hr, br);
            dmma(aci[nb][kb], hi, bi);
            dmma(acs[nb][kb], hr - hi, br + bi);
          } else {
            // conj(h) b = (hr br + hi bi) + i (hr bi - hi br)
            dmma(acr[nb][kb], hr, br);
            dmma(acr[nb][kb], hi, bi);
            dmma(aci[nb][kb], hr, bi);
            dmma(aci[nb][kb], -hi, br);
          }
        }
      }
    }
    if (M3) {
#pragma unroll
      for (int nb = 0; nb < PD_NB; ++nb)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double P = acr[nb][kb][e], Q = aci[nb][kb][e];
            acr[nb][kb][e] = P + Q;
            aci[nb][kb][e] = acs[nb][kb][e] - P + Q;
          }
    }
#pragma unroll
    for (int nb = 0; nb < PD_NB; ++nb) {
      const int n = n0 + 8 * nb + g;
      if (n < N) {
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          const int k = 8 * kb + 2 * t;
          // W in the input precision; ||W||^2 of the stored values (precoding.py:47-48)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (k + e < K) {
              const cplx<T> o = mk<T>(T(acr[nb][kb][e]), T(aci[nb][kb][e]));
              wo[int64_t(n) * K + k + e] = o;
              nrm += double(o.re) * double(o.re) + double(o.im) * double(o.im);
            }
        }
      }
    }
  }
  // coupling C = G A^-1 for row block w (rows 8 w + g)
  const int row = 8 * w + g;
  double ccr[4][2], cci[4][2];
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) ccr[kb][0] = ccr[kb][1] = cci[kb][0] = cci[kb][1] = 0.0;
  if (8 * w < K) {
    const c128 *gr = Gt + item * gs + int64_t(row < K ? row : 0) * K;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = 4 * c + t;
      const c128 a = (row < K && i < K) ? ldg_c(gr + i) : czero<double>();
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        const double br = Sr[(4 * c + t) * PD_LD + 8 * kb + g];
        const double bi = Si[(4 * c + t) * PD_LD + 8 * kb + g];
        // a b = (ar br - ai bi) + i (ar bi + ai br)
        dmma(ccr[kb], a.re, br);
        dmma(ccr[kb], -a.im, bi);
        dmma(cci[kb], a.re, bi);
        dmma(cci[kb], a.im, br);
      }
    }
  }
  // ||W||_F^2 in a fixed order: lanes, then warps 0..3
  nrm = warp_sum(nrm);
  if (lane == 0) red[w] = nrm;
  __syncthreads();
  double n2 = 0.0;
#pragma unroll
  for (int i = 0; i < PD_WARPS; ++i) n2 += red[i];
  const double nw = sqrt(n2);
  const bool bad = !(nw > 0.0);
  const double s = bad ? 0.0 : sqrt(P_t) / nw;
  double r = 0.0;
  if (8 * w < K) {
    double tot = 0.0, sig = 0.0;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * kb + 2 * t + e;
        if (row < K && col < K) {
          // H W = (G_true - alpha I) A^-1 = G_true A^-1 - alpha A^-1
          c128 gv = mk<double>(ccr[kb][e], cci[kb][e]);
          gv.re -= alpha * Sr[row * PD_LD + col];
          gv.im -= alpha * Si[row * PD_LD + col];
          const double p = cabs2(cscale(gv, s));
          tot += p;
          if (col == row) sig = p;
        }
      }
    tot += __shfl_xor_sync(0xffffffffu, tot, 1);
    tot += __shfl_xor_sync(0xffffffffu, tot, 2);
    sig += __shfl_xor_sync(0xffffffffu, sig, 1);
    sig += __shfl_xor_sync(0xffffffffu, sig, 2);
    if (row < K && t == 0) {
      const double q = sig / ((tot - sig) + noise[(item / noise_div) * K + row]);
      r = log2(1.0 + q);
      if (rates) rates[item * K + row] = r;
      if (sinr) sinr[item * K + row] = q;
    }
  }
  r = warp_sum(r);
  if (lane == 0) red2[w] = r;
  __syncthreads();
  if (tid == 0) {
    double tsum = 0.0;
#pragma unroll
    for (int i = 0; i < PD_WARPS; ++i) tsum += red2[i];
    if (sum_rate) sum_rate[item] = tsum;
    if (scale_out) scale_out[item] = s;
    if (info) info[item] = bad ? LRZ_INFO_ZERO_PRECODER : LRZ_INFO_OK;
  }
}

}  // namespace lrz

using namespace lrz;

// Launchers used by lrz_gram / lrz_precode_rate (gemm.cu), K <= 32.  complex64
// inputs are widened to double on load: the N-sized products run on the FP64
// tensor pipe for both dtypes (the reference promotes c64 H against the
// complex128 state), and only W is stored back in complex64.
template <typename T>
static void gram_dmma_launch(int64_t B, int K, int N, const cplx<T> *h, int64_t hs, double alpha,
                             c128 *a, int64_t as, cudaStream_t s) {
  const int nb = (K + 31) / 32;
  if (nb > 1) {
    // K > 32: every lower 32 x 32 block (diagonal ones included) by the 16-tile kernel
    static int split = -1;  // LRZ_GRAM_DIAG=0: diagonal blocks as full blocks (one launch)
    if (split < 0) {
      const char *e = getenv("LRZ_GRAM_DIAG");
      split = e ? atoi(e) : 1;
    }
    // complex64 H: the 3M tiled kernel (K = 64 .. 256: 23 - 28 % faster than the
    // register-fragment kernels below, e.g. C5 c64 23.9 -> 17.2 ms per 640 items);
    // complex128 H: the register-fragment kernels stay ahead (21.3 vs 21.7 ms at C5,
    // 5.4 vs 5.8 at K = 128).  LRZ_GRAM3M = 0 / 1 forces one of them
    static int g3 = -1;
    if (g3 < 0) {
      const char *e = getenv("LRZ_GRAM3M");
      g3 = e ? atoi(e) : 2;
    }
    if (g3 == 1 || (g3 == 2 && sizeof(T) == 4)) {
      const int nt = (K + 63) / 64, npair = nt * (nt + 1) / 2;
      const size_t smem = W3Smem<T>::bytes;
      cudaFuncSetAttribute(gram_dmma_3m_tiled_kernel<T>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      LrzProf prof_g("gram_dmma_3m_tiled_kernel", s);
      const int64_t cap = (int64_t(1) << 30) / npair;
      for (int64_t b0 = 0; b0 < B; b0 += cap) {
        const int64_t bb = B - b0 < cap ? B - b0 : cap;
        gram_dmma_3m_tiled_kernel<T><<<unsigned(bb * npair), 128, smem, s>>>(
            bb, K, N, h + b0 * hs, hs, a + b0 * as, as, npair, alpha);
      }
      return;
    }
    LrzProf prof_o("gram_dmma_off_kernel", s);
    if (split) {
      // the diagonal blocks first: they are the shorter warps (10 of 16 tiles)
      const unsigned ndg = unsigned((B * nb + GD_WARPS - 1) / GD_WARPS);
      gram_dmma_diag_kernel<T><<<ndg, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, a, as, nb, alpha);
      const int np = nb * (nb - 1) / 2;
      const unsigned no = unsigned((B * np + GD_WARPS - 1) / GD_WARPS);
      gram_dmma_off_kernel<T><<<no, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, a, as, np, alpha, 0);
      return;
    }
    const int np = nb * (nb + 1) / 2;
    const unsigned no = unsigned((B * np + GD_WARPS - 1) / GD_WARPS);
    gram_dmma_off_kernel<T><<<no, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, a, as, np, alpha, 1);
    return;
  }
  const unsigned nd = unsigned((B * nb + GD_WARPS - 1) / GD_WARPS);
  LrzProf prof_d("gram_dmma_kernel", s);
  switch (K > 32 ? 4 : (K + 7) / 8) {
    case 1: gram_dmma_kernel<1, T><<<nd, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, alpha, a, as, nb); break;
    case 2: gram_dmma_kernel<2, T><<<nd, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, alpha, a, as, nb); break;
    case 3: gram_dmma_kernel<3, T><<<nd, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, alpha, a, as, nb); break;
    default: gram_dmma_kernel<4, T><<<nd, 32 * GD_WARPS, 0, s>>>(B, K, N, h, hs, alpha, a, as, nb); break;
  }
}

int lrz_gram_dmma(int dtype, int64_t B, int K, int N, const void *H, int64_t hs, double alpha,
                  void *A, int64_t as, cudaStream_t s) {
  if (dtype == LRZ_C64)
    gram_dmma_launch<float>(B, K, N, (const c64 *)H, hs, alpha, (c128 *)A, as, s);
  else
    gram_dmma_launch<double>(B, K, N, (const c128 *)H, hs, alpha, (c128 *)A, as, s);
  return lrz_launch_status("gram_dmma_kernel");
}

int lrz_precode_dmma32(int dtype, int64_t B, int K, int N, const void *H, int64_t hs,
                       const void *A_inv, int64_t ais, const void *G_true, double alpha,
                       double P_t, const double *noise, int64_t noise_div, void *W, int64_t wst,
                       double *scale, double *rates, double *sinr, double *sum_rate,
                       int32_t *info, cudaStream_t s) {
  LrzProf prof("precode_dmma32_kernel", s);
  // the W slabs on the 3M complex product (C2: 1.03 -> 0.96 ms per 12,800 items at
  // 94 registers / 5 CTAs per SM; LRZ_PD3M=0: four products, 80 registers / 6 CTAs)
  static int m3 = -1;
  if (m3 < 0) {
    const char *e = getenv("LRZ_PD3M");
    m3 = e ? atoi(e) : 1;
  }
  if (m3) {
    if (dtype == LRZ_C64)
      precode_dmma32_kernel<float, true><<<unsigned(B), 32 * PD_WARPS, 0, s>>>(
          K, N, (const c64 *)H, hs, (const c128 *)A_inv, ais, (const c128 *)G_true,
          int64_t(K) * K, alpha, P_t, noise, noise_div, (c64 *)W, wst, scale, rates, sinr,
          sum_rate, info);
    else
      precode_dmma32_kernel<double, true><<<unsigned(B), 32 * PD_WARPS, 0, s>>>(
          K, N, (const c128 *)H, hs, (const c128 *)A_inv, ais, (const c128 *)G_true,
          int64_t(K) * K, alpha, P_t, noise, noise_div, (c128 *)W, wst, scale, rates, sinr,
          sum_rate, info);
    return lrz_launch_status("precode_dmma32_kernel");
  }
  if (dtype == LRZ_C64)
    precode_dmma32_kernel<float><<<unsigned(B), 32 * PD_WARPS, 0, s>>>(
        K, N, (const c64 *)H, hs, (const c128 *)A_inv, ais, (const c128 *)G_true,
        int64_t(K) * K, alpha, P_t, noise, noise_div, (c64 *)W, wst, scale, rates, sinr,
        sum_rate, info);
  else
    precode_dmma32_kernel<double><<<unsigned(B), 32 * PD_WARPS, 0, s>>>(
        K, N, (const c128 *)H, hs, (const c128 *)A_inv, ais, (const c128 *)G_true,
        int64_t(K) * K, alpha, P_t, noise, noise_div, (c128 *)W, wst, scale, rates, sinr,
        sum_rate, info);
  return lrz_launch_status("precode_dmma32_kernel");
}

// W = H^H A^-1 by w_dmma_direct_kernel; parts (nullable): ceil(N/32) ceil(K/32)
// norm partials per item.
int lrz_w_dmma_direct(int dtype, int64_t B, int K, int N, const void *H, int64_t hs,
                      const void *A_inv, int64_t ais, void *W, int64_t wstr, double *parts,
                      cudaStream_t s, const char *what) {
  const int nnb = (N + 31) / 32, njb = (K + 31) / 32, njq = (njb + 3) / 4;
  static int nbw = -1;
  if (nbw < 0) {
    const char *e = getenv("LRZ_W_NBW");
    nbw = e ? atoi(e) : 1;
  }
  static int m3 = -1;  // LRZ_W3M=0: the four-product register-fragment kernel
  if (m3 < 0) {
    const char *e = getenv("LRZ_W3M");
    m3 = e ? atoi(e) : 1;
  }
  if (m3) {
    const int tn = (N + W3_BN - 1) / W3_BN, tj = (K + W3_BJ - 1) / W3_BJ;
    const int64_t cap = (int64_t(1) << 30) / (int64_t(tn) * tj);
    // (profiler labels of the 3M kernel: W and the coupling)
    const char *lab = what[0] == 'c' ? "coupling_dmma_3m_tiled" : "w_dmma_3m_tiled_kernel";
    LrzProf prof(lab, s);
    for (int64_t b0 = 0; b0 < B; b0 += cap) {
      const int64_t bb = B - b0 < cap ? B - b0 : cap;
      double *pp = parts ? parts + b0 * int64_t(nnb) * njb : nullptr;
      auto go3 = [&](auto kern, auto hp, auto wp, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        kern<<<unsigned(bb * tn * tj), 128, smem, s>>>(bb, K, N, hp + b0 * hs, hs,
                                                       (const c128 *)A_inv + b0 * ais, ais,
                                                       wp + b0 * wstr, wstr, pp, nnb, njb, tn,
                                                       tj);
      };
      if (dtype == LRZ_C64)
        go3(w_dmma_3m_tiled_kernel<float>, (const c64 *)H, (c64 *)W, W3Smem<float>::bytes);
      else
        go3(w_dmma_3m_tiled_kernel<double>, (const c128 *)H, (c128 *)W, W3Smem<double>::bytes);
    }
    return lrz_launch_status("w_dmma_3m_tiled_kernel");
  }
  const int NB_ = nbw == 2 ? 2 : 1;
  const int64_t per = int64_t((nnb + NB_ - 1) / NB_) * njq;
  const int64_t chunk = (int64_t(1) << 30) / per;
  LrzProf prof(what, s);
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t bb = B - b0 < chunk ? B - b0 : chunk;
    double *pp = parts ? parts + b0 * int64_t(nnb) * njb : nullptr;
    auto go = [&](auto kern, auto hp, auto wp) {
      kern<<<unsigned(bb * per), 128 * NB_, 0, s>>>(bb, K, N, hp + b0 * hs, hs,
                                                    (const c128 *)A_inv + b0 * ais, ais,
                                                    wp + b0 * wstr, wstr, pp, nnb, njb, njq);
    };
    if (dtype == LRZ_C64) {
      if (NB_ == 2) go(w_dmma_direct_kernel<float, 2>, (const c64 *)H, (c64 *)W);
      else go(w_dmma_direct_kernel<float, 1>, (const c64 *)H, (c64 *)W);
    } else {
      if (NB_ == 2) go(w_dmma_direct_kernel<double, 2>, (const c128 *)H, (c128 *)W);
      else go(w_dmma_direct_kernel<double, 1>, (const c128 *)H, (c128 *)W);
    }
  }
  return lrz_launch_status("w_dmma_direct_kernel");
}
