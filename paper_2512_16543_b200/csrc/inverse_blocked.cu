// K5 for 64 < K <= 256: blocked Gauss-Jordan inversion of the Hermitian
// positive-definite Gram (lowrank.py:127-144, 361-367) with the rank-b updates
// on the FP64 tensor pipe.  For block column j (b = 32 rows / columns):
//   P = A[j, j], C = A[:, j], R = A[j, :]
//   Pinv = P^-1 (per item, shared memory, no pivoting: PD)
//   Cp = C Pinv,  Rp = Pinv R                                   (K b^2 each)
//   A' = A - Cp R   (K x K x b, zgemm_dmma, out of place)
//   A'[j, :] = Rp,  A'[:, j] = -Cp,  A'[j, j] = Pinv            (fix-up)
// K / b steps, 8 K^3 real flops in all.  Items whose pivots are not positive
// or whose ||A||_F ||A^-1||_F bound exceeds the guard are flagged for the exact
// CTA kernel (pivoted path, exact cond_2) exactly like the cluster / warp fast
// paths.

#include <algorithm>

#include "common.cuh"

int lrz_gj_panels_dmma(int64_t B, int K, int b, int j0, const void *Acur, int64_t cst,
                       const void *Pinv, void *Cp, void *Rp, const uint8_t *mask, cudaStream_t s);
int lrz_gj_update_dmma(int64_t B, int K, int b, int j0, const void *Cp, const void *Acur,
                       int64_t cst, void *Anext, int64_t nst, const uint8_t *mask, cudaStream_t s);

namespace lrz {

constexpr int GJB = 32;        // block size
constexpr int GJ_THREADS = 256;

// One CTA per active item: Pinv, Cp, Rp for block j0 of A (K x K, item stride kk).
__global__ void __launch_bounds__(GJ_THREADS)
    gj_pivot_kernel(int K, int j0, const c128 *__restrict__ A, int64_t kk,
                    c128 *__restrict__ Pinv, c128 *__restrict__ Cp, c128 *__restrict__ Rp,
                    uint8_t *__restrict__ bad, const uint8_t *__restrict__ mask) {
  __shared__ c128 P[GJB][GJB + 1];
  __shared__ c128 piv_row[GJB], piv_col[GJB];
  __shared__ int s_bad;
  const int64_t item = blockIdx.x;
  if (mask && !mask[item]) return;
  const int tid = threadIdx.x;
  const c128 *a = A + item * kk;
  if (tid == 0) s_bad = 0;
  for (int e = tid; e < GJB * GJB; e += GJ_THREADS) {
    const int r = e / GJB, c = e % GJB;
    P[r][c] = a[int64_t(j0 + r) * K + j0 + c];
  }
  __syncthreads();
  // in-place Gauss-Jordan of the b x b block (Hermitian PD: real positive pivots)
  for (int k = 0; k < GJB; ++k) {
    const double d = P[k][k].re;
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) s_bad = 1;
      break;  // block-uniform (every thread reads the same P[k][k])
    }
    const double id = 1.0 / d;
    if (tid < GJB) piv_row[tid] = tid == k ? mk<double>(id, 0.0) : cscale(P[k][tid], id);
    if (tid >= 32 && tid < 32 + GJB) piv_col[tid - 32] = P[tid - 32][k];
    __syncthreads();
    for (int e = tid; e < GJB * GJB; e += GJ_THREADS) {
      const int r = e / GJB, c = e % GJB;
      if (r == k) continue;
      const c128 f = piv_col[r];
      const c128 pr = piv_row[c];
      if (c == k) {
        P[r][c] = mk<double>(-(f.re * id), -(f.im * id));
      } else {
        P[r][c].re -= f.re * pr.re - f.im * pr.im;
        P[r][c].im -= f.re * pr.im + f.im * pr.re;
      }
    }
    __syncthreads();
    if (tid < GJB) P[k][tid] = piv_row[tid];
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) bad[item] = 1;
    return;
  }
  c128 *pi = Pinv + item * (GJB * GJB);
  for (int e = tid; e < GJB * GJB; e += GJ_THREADS) pi[e] = P[e / GJB][e % GJB];
  (void)Cp;
  (void)Rp;  // Cp = C Pinv and Rp = Pinv R follow as batched DMMA GEMMs
}

// A'[j, :] = Rp, A'[:, j] = -Cp, A'[j, j] = Pinv
__global__ void gj_fixup_kernel(int64_t B, int K, int j0, const c128 *__restrict__ Pinv,
                                const c128 *__restrict__ Cp, const c128 *__restrict__ Rp,
                                c128 *__restrict__ An, int64_t kk, const uint8_t *__restrict__ bad,
                                const uint8_t *__restrict__ mask) {
  const int64_t per = 2 * int64_t(K) * GJB;
  const int64_t n = B * per;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t item = e / per;
    if ((mask && !mask[item]) || bad[item]) continue;
    const int64_t w = e - item * per;
    c128 *o = An + item * kk;
    if (w < int64_t(K) * GJB) {  // row block j: Rp (Pinv on the diagonal block)
      const int r = int(w / K), k = int(w % K);
      const bool diag = k >= j0 && k < j0 + GJB;
      o[int64_t(j0 + r) * K + k] = diag ? Pinv[item * GJB * GJB + r * GJB + (k - j0)]
                                        : Rp[item * int64_t(K) * GJB + w];
    } else {                     // column block j: -Cp
      const int64_t v = w - int64_t(K) * GJB;
      const int i = int(v / GJB), c = int(v % GJB);
      if (i >= j0 && i < j0 + GJB) continue;
      const c128 x = Cp[item * int64_t(K) * GJB + v];
      o[int64_t(i) * K + j0 + c] = mk<double>(-x.re, -x.im);
    }
  }
}

// guard: flag (redo) items whose pivots failed or whose ||A||_F ||A^-1||_F
// bound exceeds the limit; the CTA kernel then decides them exactly
__global__ void gj_guard_kernel(int64_t B, int K, const c128 *__restrict__ A, int64_t as,
                                const c128 *__restrict__ Ai, int64_t ais, double limit,
                                const uint8_t *__restrict__ bad, const uint8_t *__restrict__ mask,
                                uint8_t *__restrict__ redo, int32_t *__restrict__ info) {
  __shared__ double red[8];
  const int64_t item = blockIdx.x;
  if (mask && !mask[item]) {
    if (threadIdx.x == 0) redo[item] = 0;
    return;
  }
  double fa = 0.0, fi = 0.0;
  const int64_t KK = int64_t(K) * K;
  for (int64_t e = threadIdx.x; e < KK; e += blockDim.x) {
    fa += cabs2(A[item * as + e]);
    fi += cabs2(Ai[item * ais + e]);
  }
  fa = block_sum(fa, red);
  fi = block_sum(fi, red);
  if (threadIdx.x == 0) {
    const double fb = sqrt(fa) * sqrt(fi);
    const bool ok = !bad[item] && isfinite(fb) && fb <= limit;
    redo[item] = ok ? 0 : 1;
    if (ok && info) info[item] = LRZ_INFO_OK;
  }
}

}  // namespace lrz

using namespace lrz;

size_t lrz_inverse_blocked_ws(int64_t B, int K) {
  const size_t KK = size_t(K) * K;
  size_t b = size_t(B) * KK * 16;                      // ping-pong buffer
  b += size_t(B) * 2 * K * GJB * 16;                   // Cp, Rp
  b += size_t(B) * GJB * GJB * 16;                     // Pinv
  b += size_t(B);                                      // bad flags
  return (b + 255) & ~size_t(255);
}

// Blocked GJ inverse of B items (masked); writes A_inv for the items it
// accepts and redo[] = 1 for the ones the exact CTA kernel must decide.
int lrz_inverse_blocked(int64_t B, int K, const void *A, int64_t a_stride, void *A_inv,
                        int64_t ai_stride, int32_t *info, double limit, const uint8_t *mask,
                        uint8_t *redo, void *ws, cudaStream_t s) {
  LrzProf prof("herm_inverse_blocked_gj (all kernels)", s);
  const int64_t KK = int64_t(K) * K;
  char *w = (char *)ws;
  c128 *X = (c128 *)w;
  w += size_t(B) * KK * 16;
  c128 *Cp = (c128 *)w;
  w += size_t(B) * K * GJB * 16;
  c128 *Rp = (c128 *)w;
  w += size_t(B) * K * GJB * 16;
  c128 *Pinv = (c128 *)w;
  w += size_t(B) * GJB * GJB * 16;
  uint8_t *bad = (uint8_t *)w;
  cudaMemsetAsync(bad, 0, size_t(B), s);
  const int nsteps = K / GJB;
  // ping-pong so that the last step lands in A_inv (item stride ai_stride)
  const c128 *cur = (const c128 *)A;
  int64_t cst = a_stride;
  for (int st = 0; st < nsteps; ++st) {
    const bool to_out = ((nsteps - 1 - st) % 2) == 0;
    c128 *nxt = to_out ? (c128 *)A_inv : X;
    const int64_t nst = to_out ? ai_stride : KK;
    const int j0 = st * GJB;
    gj_pivot_kernel<<<unsigned(B), GJ_THREADS, 0, s>>>(K, j0, cur, cst, Pinv, Cp, Rp, bad, mask);
    if (int rc = lrz_launch_status("gj_pivot_kernel")) return rc;
    if (int rc = lrz_gj_panels_dmma(B, K, GJB, j0, cur, cst, Pinv, Cp, Rp, mask, s)) return rc;
    if (int rc = lrz_gj_update_dmma(B, K, GJB, j0, Cp, cur, cst, nxt, nst, mask, s)) return rc;
    gj_fixup_kernel<<<unsigned(std::min<int64_t>((B * 2 * K * GJB + 255) / 256, 148 * 32)), 256,
                      0, s>>>(B, K, j0, Pinv, Cp, Rp, nxt, nst, bad, mask);
    if (int rc = lrz_launch_status("gj_fixup_kernel")) return rc;
    cur = nxt;
    cst = nst;
  }
  gj_guard_kernel<<<unsigned(B), 256, 0, s>>>(B, K, (const c128 *)A, a_stride, (const c128 *)A_inv,
                                              ai_stride, limit, bad, mask, redo, info);
  return lrz_launch_status("gj_guard_kernel");
}
