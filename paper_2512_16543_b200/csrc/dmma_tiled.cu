// K6 for K > 32 on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64):
//   out[n][j] = sum_k conj(X[k][n]) Y[k][j]
// with X = H (K x N, the precoder W = H^H A^-1, precoding.py:47) or X = G_true
// (K x K, the coupling H W = (G - alpha I) A^-1 for F_RF = I, SURVEY A.6;
// G Hermitian so conj(G)^T = G), Y = A^-1 (K x K complex128).
//
// Tiling: one CTA (8 warps) per (item, 64 n x 64 j output tile); the k axis is
// streamed in 16-row slabs through a 3-stage cp.async ring in shared memory
// (X slab 16 x 64, Y slab 16 x 64, rows padded so the fragment loads are bank
// conflict free).  Warp (wn, wj) owns 16 n x 32 j = 2 x 4 complex 8 x 8 tiles:
// per k-step of 4 it loads 2 X and 4 Y fragments (one LDS.128 / LDS.64 each)
// for 32 DMMAs (4 real DMMAs per complex block).  complex64 X is widened to
// fp64 on the fragment load, accumulation is fp64, W is rounded to the input
// precision on store and ||W||_F^2 of the stored values goes out as one
// partial per CTA (summed in a fixed order by the SINR kernel).
//
// L2 traffic per item: X is read K/64 times, Y N/64 times (C5: 4 x 16 MB +
// 64 x 1 MB), against DMMA time ~60 us per C5 item -- far below L2 bandwidth.

#include "dmma.cuh"

namespace lrz {

constexpr int DT_BN = 64, DT_BJ = 64, DT_KC = 16, DT_ST = 3, DT_THREADS = 256;

template <typename T>
struct DtPad {
  static constexpr int X = sizeof(T) == 8 ? 2 : 4;  // row pad (elements) of the X slab
};

template <typename T>
struct DtSmem {
  static constexpr int XLD = DT_BN + DtPad<T>::X;
  static constexpr int YLD = DT_BJ + 2;
  static constexpr size_t xbytes = size_t(DT_KC) * XLD * sizeof(cplx<T>);
  static constexpr size_t ybytes = size_t(DT_KC) * YLD * sizeof(c128);
  static constexpr size_t stage = xbytes + ybytes;
  static constexpr size_t bytes = stage * DT_ST + 16 * sizeof(double);
};

LRZ_DEV void cpa(void *smem, const void *gmem, int bytes, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(pred ? 16 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(pred ? 8 : 0));
}

template <typename T>
__global__ void __launch_bounds__(DT_THREADS, 2)
    dmma_hn_kernel(int NN, int J, int Kd, const cplx<T> *__restrict__ X, int64_t xs, int ldx,
                   const c128 *__restrict__ Y, int64_t ys, cplx<T> *__restrict__ out,
                   int64_t os, double *__restrict__ parts, int tiles_n, int tiles_j,
                   const uint8_t *__restrict__ mask) {
  using S = DtSmem<T>;
  extern __shared__ __align__(16) unsigned char dt_smem[];
  const int ntile = tiles_n * tiles_j;
  const int64_t item = blockIdx.x / ntile;
  if (mask && !mask[item]) return;
  const int tile = int(blockIdx.x - item * ntile);
  const int n0 = (tile / tiles_j) * DT_BN, j0 = (tile % tiles_j) * DT_BJ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wn = w & 3, wj = w >> 2;
  const cplx<T> *x = X + item * xs;
  const c128 *y = Y + item * ys;

  auto xslab = [&](int s) {
    return reinterpret_cast<cplx<T> *>(dt_smem + size_t(s) * S::stage);
  };
  auto yslab = [&](int s) {
    return reinterpret_cast<c128 *>(dt_smem + size_t(s) * S::stage + S::xbytes);
  };
  auto load = [&](int s, int k0) {
    cplx<T> *xsl = xslab(s);
    c128 *ysl = yslab(s);
#pragma unroll
    for (int i = 0; i < (DT_KC * DT_BN) / DT_THREADS; ++i) {
      const int e = tid + i * DT_THREADS, r = e / DT_BN, c = e % DT_BN;
      const int k = k0 + r, n = n0 + c;
      const bool ok = k < Kd && n < NN;
      cpa(xsl + r * S::XLD + c, x + (ok ? int64_t(k) * ldx + n : 0), sizeof(cplx<T>), ok);
    }
#pragma unroll
    for (int i = 0; i < (DT_KC * DT_BJ) / DT_THREADS; ++i) {
      const int e = tid + i * DT_THREADS, r = e / DT_BJ, c = e % DT_BJ;
      const int k = k0 + r, j = j0 + c;
      const bool ok = k < Kd && j < J;
      cpa(ysl + r * S::YLD + c, y + (ok ? int64_t(k) * J + j : 0), 16, ok);
    }
  };

  double acr[2][4][2], aci[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acr[a][b][0] = acr[a][b][1] = aci[a][b][0] = aci[a][b][1] = 0.0;

  const int nslab = (Kd + DT_KC - 1) / DT_KC;
#pragma unroll
  for (int s = 0; s < DT_ST - 1; ++s) {
    if (s < nslab) load(s, s * DT_KC);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int it = 0; it < nslab; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(DT_ST - 2));
    __syncthreads();
    const int nxt = it + DT_ST - 1;
    if (nxt < nslab) load(nxt % DT_ST, nxt * DT_KC);
    asm volatile("cp.async.commit_group;\n" ::);
    const cplx<T> *xsl = xslab(it % DT_ST);
    const c128 *ysl = yslab(it % DT_ST);
#pragma unroll
    for (int kk = 0; kk < DT_KC; kk += 4) {
      double hr[2], hi[2], br[4], bi[4];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const cplx<T> v = xsl[(kk + t) * S::XLD + 16 * wn + 8 * nb + g];
        hr[nb] = double(v.re);
        hi[nb] = double(v.im);
      }
#pragma unroll
      for (int jb = 0; jb < 4; ++jb) {
        const c128 v = ysl[(kk + t) * S::YLD + 32 * wj + 8 * jb + g];
        br[jb] = v.re;
        bi[jb] = v.im;
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const double nhi = -hi[nb];
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          // conj(x) y = (xr yr + xi yi) + i (xr yi - xi yr)
          dmma(acr[nb][jb], hr[nb], br[jb]);
          dmma(acr[nb][jb], hi[nb], bi[jb]);
          dmma(aci[nb][jb], hr[nb], bi[jb]);
          dmma(aci[nb][jb], nhi, br[jb]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);

  cplx<T> *o = out + item * os;
  double nrm = 0.0;
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    const int n = n0 + 16 * wn + 8 * nb + g;
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + 32 * wj + 8 * jb + 2 * t + e;
        if (n < NN && j < J) {
          const cplx<T> z = mk<T>(T(acr[nb][jb][e]), T(aci[nb][jb][e]));
          o[int64_t(n) * J + j] = z;
          nrm += double(z.re) * double(z.re) + double(z.im) * double(z.im);
        }
      }
  }
  if (parts) {
    double *red = reinterpret_cast<double *>(dt_smem + S::stage * DT_ST);
    const double s = block_sum(nrm, red);
    if (tid == 0) parts[item * ntile + tile] = s;
  }
}

template <typename T>
static int dmma_hn_launch(int64_t B, int NN, int J, int Kd, const cplx<T> *X, int64_t xs, int ldx,
                          const c128 *Y, int64_t ys, cplx<T> *out, int64_t os, double *parts,
                          const uint8_t *mask, cudaStream_t s, const char *what) {
  LrzProf prof(what, s);
  const int tn = (NN + DT_BN - 1) / DT_BN, tj = (J + DT_BJ - 1) / DT_BJ;
  const size_t sm = DtSmem<T>::bytes;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(dmma_hn_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sm)) != cudaSuccess) {
      lrz_set_error("dmma_hn_kernel: cannot reserve %zu bytes of shared memory", sm);
      return LRZ_ELAUNCH;
    }
    attr = true;
  }
  const int64_t nb = B * tn * tj;
  // grid.x limit is 2^31 - 1; chunk the batch if it would overflow
  const int64_t per = (int64_t(1) << 30) / (int64_t(tn) * tj);
  for (int64_t b0 = 0; b0 < B; b0 += per) {
    const int64_t bb = B - b0 < per ? B - b0 : per;
    dmma_hn_kernel<T><<<unsigned(bb * tn * tj), DT_THREADS, sm, s>>>(
        NN, J, Kd, X + b0 * xs, xs, ldx, Y + b0 * ys, ys, out + b0 * os, os,
        parts ? parts + b0 * tn * tj : nullptr, tn, tj, mask ? mask + b0 : nullptr);
  }
  (void)nb;
  return lrz_launch_status("dmma_hn_kernel");
}

}  // namespace lrz

using namespace lrz;

// number of norm partials per item written by lrz_dmma_hn (precoder W)
int lrz_dmma_hn_tiles(int NN, int J) {
  return ((NN + DT_BN - 1) / DT_BN) * ((J + DT_BJ - 1) / DT_BJ);
}

// out[n][j] = sum_k conj(X[k][n]) Y[k][j]; X of dtype (c64 widened), Y c128,
// out in dtype with row length J; parts (nullable): per-CTA ||out||^2.
int lrz_dmma_hn(int dtype, int64_t B, int NN, int J, int Kd, const void *X, int64_t xs, int ldx,
                const void *Y, int64_t ys, void *out, int64_t os, double *parts,
                cudaStream_t s, const uint8_t *mask, const char *what) {
  if (dtype == LRZ_C64)
    return dmma_hn_launch<float>(B, NN, J, Kd, (const c64 *)X, xs, ldx, (const c128 *)Y, ys,
                                 (c64 *)out, os, parts, mask, s, what);
  return dmma_hn_launch<double>(B, NN, J, Kd, (const c128 *)X, xs, ldx, (const c128 *)Y, ys,
                                (c128 *)out, os, parts, mask, s, what);
}

// Omega_all [B][K][Dtot] (complex128) gathered from the normal window: column c
// of block i (offset o_i, width d_i) is sqrt(1/2) (zre[k d_i + j] + i zim[k d_i + j])
// at the item's cursor, blocks back to back in the stream (lowrank.py:284-286).
__global__ void omega_gather_kernel(int K, int Dtot, const double *__restrict__ omega,
                                    int64_t os, const int32_t *__restrict__ orow,
                                    int64_t orow_div, const int64_t *__restrict__ cursor,
                                    int k_init, int p, const uint8_t *__restrict__ mask,
                                    c128 *__restrict__ Om) {
  const int64_t item = blockIdx.x;
  if (mask && !mask[item]) return;
  __shared__ int s_off[256], s_d[256], s_j[256];
  for (int c = threadIdx.x; c < Dtot; c += blockDim.x) {
    int o = 0, k0 = k_init, d = min(k0 + p, K), off = 0;
    while (c >= o + d) {
      o += d;
      off += 2 * K * d;
      k0 *= 2;
      d = min(k0 + p, K);
    }
    s_off[c] = off;
    s_d[c] = d;
    s_j[c] = c - o;
  }
  __syncthreads();
  const int64_t row = orow ? int64_t(orow[item]) : item / orow_div;
  const double *z = omega + row * os + (cursor ? cursor[item] : 0);
  const double SQH = 0.7071067811865476;
  c128 *o = Om + item * int64_t(K) * Dtot;
  for (int e = threadIdx.x; e < K * Dtot; e += blockDim.x) {
    const int k = e / Dtot, c = e - k * Dtot, d = s_d[c];
    const double *zb = z + s_off[c] + int64_t(k) * d + s_j[c];
    o[e] = mk<double>(SQH * zb[0], SQH * zb[int64_t(K) * d]);
  }
}

// lrz_arsvd's front end for K > 32 on the FP64 tensor pipe: Omega_all gathered,
// Y = dA Omega_all and W = dA Y as two dmma_hn passes (dA is Hermitian, so
// conj(dA)^T = dA).  Om, Y, W: [B][K][Dtot] complex128.
int lrz_sketch_dmma_large(int64_t B, int K, int Dtot, const void *dA, int64_t a_stride,
                          const double *omega, int64_t omega_stride, const int32_t *omega_row,
                          int64_t orow_div, const int64_t *cursor, int k_init, int p,
                          const uint8_t *mask, void *Om, void *Y, void *W, cudaStream_t s) {
  if (Dtot > 256) {
    lrz_set_error("lrz_sketch_dmma_large: Dtot %d > 256", Dtot);
    return LRZ_EINVAL;
  }
  {
    LrzProf prof("omega_gather_kernel", s);
    omega_gather_kernel<<<unsigned(B), 256, 0, s>>>(K, Dtot, omega, omega_stride, omega_row,
                                                    orow_div, cursor, k_init, p, mask,
                                                    (c128 *)Om);
  }
  if (int rc = lrz_launch_status("omega_gather_kernel")) return rc;
  const int64_t st = int64_t(K) * Dtot;
  if (int rc = dmma_hn_launch<double>(B, K, Dtot, K, (const c128 *)dA, a_stride, K,
                                      (const c128 *)Om, st, (c128 *)Y, st, nullptr, mask, s,
                                      "dmma_hn_kernel:sketch_Y"))
    return rc;
  return dmma_hn_launch<double>(B, K, Dtot, K, (const c128 *)dA, a_stride, K, (const c128 *)Y,
                                st, (c128 *)W, st, nullptr, mask, s, "dmma_hn_kernel:sketch_W");
}
