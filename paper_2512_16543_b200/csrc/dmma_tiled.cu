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

// WNS warps along n (x 8 / WNS along j): 4 = the 64 n x 64 j tile, 2 = 32 n x 128 j
// for products with few output rows (the chain's D x K products, the arSVD tail's
// M = dA^H Q with NN = d <= 32: a 64-row tile would be one third full).
template <typename T, int WNS = 4>
struct DtSmem {
  static constexpr int BN = 16 * WNS, BJ = 32 * (8 / WNS);
  static constexpr int XLD = BN + DtPad<T>::X;
  static constexpr int YLD = BJ + 2;
  static constexpr size_t xbytes = size_t(DT_KC) * XLD * sizeof(cplx<T>);
  static constexpr size_t ybytes = size_t(DT_KC) * YLD * sizeof(c128);
  static constexpr size_t stage = xbytes + ybytes;
  // the 32 x 128 tile's Y slab is twice as wide: two stages keep two CTAs per SM
  static constexpr int ST = WNS == 4 ? DT_ST : 2;
  static constexpr size_t bytes = stage * ST + 16 * sizeof(double);
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

// Generalised form used by the Woodbury chain as well:
//   out[n][j] (MODE 0 =, 1 = base -, 2 +=) sum_k opX(k, n) opY(k, j)
// with X(k, n) at XT ? n ldx + k : k ldx + n, opX = conj when XC (the
// precoder's H^H), likewise Y / YT / YC; optional per-k real scale of Y
// (kscale, the Woodbury S) and per-item reduction length (kd_item).
struct ZgArgs {
  int NN, J, Kd;
  const void *X;
  int64_t xs;
  int ldx;
  const c128 *Y;
  int64_t ys;
  int ldy;
  void *out;
  int64_t os;
  int ldo;
  const c128 *base;  // MODE 1
  int64_t bs;
  double *parts;
  const uint8_t *mask;  // item active iff mask[item * mstride] == mval
  int64_t mstride;
  int mval;
  const int32_t *kd_item;  // nullable: reduction length of item = min(Kd, kd_item[item * kstride])
  int64_t kstride;
  const double *kscale;  // nullable: Y row k scaled by kscale[item * kss + k]
  int64_t kss;
  int tiles_n, tiles_j;
};

template <typename T, bool XT, bool XC, bool YT, bool YC, int MODE, int WNS = 4>
__global__ void __launch_bounds__(DT_THREADS, 2) zgemm_dmma_kernel(ZgArgs a) {
  using S = DtSmem<T, WNS>;
  constexpr int BN = S::BN, BJ = S::BJ, ST = S::ST;
  extern __shared__ __align__(16) unsigned char dt_smem[];
  __shared__ double s_ks[DT_ST][DT_KC];
  const int ntile = a.tiles_n * a.tiles_j;
  const int64_t item = blockIdx.x / ntile;
  if (a.mask && a.mask[item * a.mstride] != a.mval) return;
  const int tile = int(blockIdx.x - item * ntile);
  const int n0 = (tile / a.tiles_j) * BN, j0 = (tile % a.tiles_j) * BJ;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
  const int wn = w % WNS, wj = w / WNS;
  const int NN = a.NN, J = a.J;
  const int Kd = a.kd_item ? min(a.Kd, int(a.kd_item[item * a.kstride])) : a.Kd;
  const cplx<T> *x = reinterpret_cast<const cplx<T> *>(a.X) + item * a.xs;
  const c128 *y = a.Y + item * a.ys;
  const double *ksc = a.kscale ? a.kscale + item * a.kss : nullptr;

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
    for (int i = 0; i < (DT_KC * BN) / DT_THREADS; ++i) {
      const int e = tid + i * DT_THREADS;
      const int r = XT ? e % DT_KC : e / BN, c = XT ? e / DT_KC : e % BN;
      const int k = k0 + r, n = n0 + c;
      const bool ok = k < Kd && n < NN;
      const int64_t off = XT ? int64_t(n) * a.ldx + k : int64_t(k) * a.ldx + n;
      cpa(xsl + r * S::XLD + c, x + (ok ? off : 0), sizeof(cplx<T>), ok);
    }
#pragma unroll
    for (int i = 0; i < (DT_KC * BJ) / DT_THREADS; ++i) {
      const int e = tid + i * DT_THREADS;
      const int r = YT ? e % DT_KC : e / BJ, c = YT ? e / DT_KC : e % BJ;
      const int k = k0 + r, j = j0 + c;
      const bool ok = k < Kd && j < J;
      const int64_t off = YT ? int64_t(j) * a.ldy + k : int64_t(k) * a.ldy + j;
      cpa(ysl + r * S::YLD + c, y + (ok ? off : 0), 16, ok);
    }
    if (ksc && tid < DT_KC) s_ks[s][tid] = (k0 + tid < Kd) ? ksc[k0 + tid] : 0.0;
  };

  double acr[2][4][2], aci[2][4][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int b = 0; b < 4; ++b) acr[q][b][0] = acr[q][b][1] = aci[q][b][0] = aci[q][b][1] = 0.0;

  const int nslab = (Kd + DT_KC - 1) / DT_KC;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nslab) load(s, s * DT_KC);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int it = 0; it < nslab; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
    __syncthreads();
    const int nxt = it + ST - 1;
    if (nxt < nslab) load(nxt % ST, nxt * DT_KC);
    asm volatile("cp.async.commit_group;\n" ::);
    const cplx<T> *xsl = xslab(it % ST);
    const c128 *ysl = yslab(it % ST);
#pragma unroll
    for (int kk = 0; kk < DT_KC; kk += 4) {
      double hr[2], hi[2], br[4], bi[4];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const cplx<T> v = xsl[(kk + t) * S::XLD + 16 * wn + 8 * nb + g];
        hr[nb] = double(v.re);
        hi[nb] = XC ? double(v.im) : -double(v.im);  // the product below conjugates x
      }
      const double ks = ksc ? s_ks[it % ST][kk + t] : 1.0;
#pragma unroll
      for (int jb = 0; jb < 4; ++jb) {
        const c128 v = ysl[(kk + t) * S::YLD + 32 * wj + 8 * jb + g];
        br[jb] = ksc ? ks * v.re : v.re;
        bi[jb] = ksc ? ks * (YC ? -v.im : v.im) : (YC ? -v.im : v.im);
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

  cplx<T> *o = reinterpret_cast<cplx<T> *>(a.out) + item * a.os;
  const c128 *bse = MODE == 1 ? a.base + item * a.bs : nullptr;
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
          const int64_t idx = int64_t(n) * a.ldo + j;
          double zr = acr[nb][jb][e], zi = aci[nb][jb][e];
          if (MODE == 1) {
            const c128 b = bse[idx];
            zr = b.re - zr;
            zi = b.im - zi;
          } else if (MODE == 2) {
            const cplx<T> b = o[idx];
            zr = double(b.re) + zr;
            zi = double(b.im) + zi;
          }
          const cplx<T> z = mk<T>(T(zr), T(zi));
          o[idx] = z;
          nrm += double(z.re) * double(z.re) + double(z.im) * double(z.im);
        }
      }
  }
  if (a.parts) {
    double *red = reinterpret_cast<double *>(dt_smem + S::stage * ST);
    const double s = block_sum(nrm, red);
    if (tid == 0) a.parts[item * ntile + tile] = s;
  }
}

template <typename T, bool XT, bool XC, bool YT, bool YC, int MODE, int WNS>
static int zgemm_dmma_launch_w(int64_t B, ZgArgs a, cudaStream_t s, const char *what) {
  LrzProf prof(what, s);
  using S = DtSmem<T, WNS>;
  a.tiles_n = (a.NN + S::BN - 1) / S::BN;
  a.tiles_j = (a.J + S::BJ - 1) / S::BJ;
  const size_t sm = S::bytes;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(zgemm_dmma_kernel<T, XT, XC, YT, YC, MODE, WNS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)) != cudaSuccess) {
      lrz_set_error("zgemm_dmma_kernel: cannot reserve %zu bytes of shared memory", sm);
      return LRZ_ELAUNCH;
    }
    attr = true;
  }
  const int64_t nt = int64_t(a.tiles_n) * a.tiles_j;
  const int64_t per = (int64_t(1) << 30) / nt;
  for (int64_t b0 = 0; b0 < B; b0 += per) {
    const int64_t bb = B - b0 < per ? B - b0 : per;
    ZgArgs c = a;
    c.X = reinterpret_cast<const cplx<T> *>(a.X) + b0 * a.xs;
    c.Y = a.Y + b0 * a.ys;
    c.out = reinterpret_cast<cplx<T> *>(a.out) + b0 * a.os;
    if (a.base) c.base = a.base + b0 * a.bs;
    if (a.parts) c.parts = a.parts + b0 * nt;
    if (a.mask) c.mask = a.mask + b0 * a.mstride;
    if (a.kd_item) c.kd_item = a.kd_item + b0 * a.kstride;
    if (a.kscale) c.kscale = a.kscale + b0 * a.kss;
    zgemm_dmma_kernel<T, XT, XC, YT, YC, MODE, WNS><<<unsigned(bb * nt), DT_THREADS, sm, s>>>(c);
  }
  return lrz_launch_status(what);
}

// few output rows (NN <= 32) and no norm partials: the 32 n x 128 j tile
template <typename T, bool XT, bool XC, bool YT, bool YC, int MODE>
static int zgemm_dmma_launch(int64_t B, ZgArgs a, cudaStream_t s, const char *what) {
  static int narrow = -1;
  if (narrow < 0) {
    const char *e = getenv("LRZ_ZGEMM_NARROW");
    narrow = e ? atoi(e) : 1;
  }
  if (narrow && a.NN <= 32 && !a.parts)
    return zgemm_dmma_launch_w<T, XT, XC, YT, YC, MODE, 2>(B, a, s, what);
  return zgemm_dmma_launch_w<T, XT, XC, YT, YC, MODE, 4>(B, a, s, what);
}

template <typename T>
static int dmma_hn_launch(int64_t B, int NN, int J, int Kd, const cplx<T> *X, int64_t xs, int ldx,
                          const c128 *Y, int64_t ys, cplx<T> *out, int64_t os, double *parts,
                          const uint8_t *mask, cudaStream_t s, const char *what) {
  ZgArgs a{};
  a.NN = NN;
  a.J = J;
  a.Kd = Kd;
  a.X = X;
  a.xs = xs;
  a.ldx = ldx;
  a.Y = Y;
  a.ys = ys;
  a.ldy = J;
  a.out = out;
  a.os = os;
  a.ldo = J;
  a.parts = parts;
  a.mask = mask;
  a.mstride = 1;
  a.mval = 1;
  return zgemm_dmma_launch<T, false, true, false, false, 0>(B, a, s, what);
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

// Woodbury chain products for one time step t of the step-parallel chain
// (chain.cu), all trials at once on the FP64 tensor pipe.  U, V: [B][T][D][K]
// (factor column f of item (b, t) contiguous); prev: A^-1_{t-1} per trial.
//   AiUt[f][k] = (A^-1 U)[k][f] = sum_m U[m][f] A^-1[k][m]        (lowrank.py:209)
//   VhAi[f][j] = (V^H A^-1)[f][j] = sum_k conj(V[k][f]) A^-1[k][j]  (lowrank.py:219)
int lrz_chain_gemms_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *plan,
                         const void *U, const void *V, const void *prev, int64_t pst,
                         void *AiUt, void *VhAi, void *aux, int64_t ws_stride, cudaStream_t s) {
  ZgArgs a{};
  a.NN = D;
  a.J = K;
  a.Kd = K;
  a.X = (const c128 *)U + int64_t(t) * D * K;
  a.xs = int64_t(T) * D * K;
  a.ldx = K;
  a.Y = (const c128 *)prev;
  a.ys = pst;
  a.ldy = K;
  a.out = AiUt;
  a.os = ws_stride;
  a.ldo = K;
  a.mask = plan + t;
  a.mstride = T;
  a.mval = 1;
  if (int rc = zgemm_dmma_launch<double, true, false, true, false, 0>(B, a, s, "chain:AiU_dmma"))
    return rc;
  a.X = (const c128 *)V + int64_t(t) * D * K;
  a.out = VhAi;
  if (int rc = zgemm_dmma_launch<double, true, true, false, false, 0>(B, a, s,
                                                                        "chain:VhAi_dmma"))
    return rc;
  // aux' = V^H AiU (D x D; lowrank.py:210 before the 1/S diagonal):
  //   aux'[i][j] = sum_k conj(V[k][i]) AiU[k][j],  AiU[k][j] = AiUt[j][k]
  ZgArgs c = a;
  c.NN = D;
  c.J = D;
  c.Y = (const c128 *)AiUt;
  c.ys = ws_stride;
  c.ldy = K;
  c.out = aux;
  c.os = ws_stride;
  c.ldo = D;
  return zgemm_dmma_launch<double, true, true, true, false, 0>(B, c, s, "chain:aux_dmma");
}

// T = AiU aux^-1 (stored [D][K]: T[j][k] = sum_{i < r} aux^-1[i][j] AiU[k][i])
int lrz_chain_T_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *act,
                     const int32_t *r, const void *auxinv, const void *AiUt, void *Tm,
                     int64_t ws_stride, cudaStream_t s) {
  ZgArgs a{};
  a.NN = D;
  a.J = K;
  a.Kd = D;
  a.X = auxinv;
  a.xs = ws_stride;
  a.ldx = D;
  a.Y = (const c128 *)AiUt;
  a.ys = ws_stride;
  a.ldy = K;
  a.out = Tm;
  a.os = ws_stride;
  a.ldo = K;
  a.mask = act;
  a.mstride = 1;
  a.mval = 1;
  a.kd_item = r + t;
  a.kstride = T;
  return zgemm_dmma_launch<double, false, false, false, false, 0>(B, a, s, "chain:T_dmma");
}

// A^-1_t = prev - T VhAi and A_t = A_{t-1} + (U S) V^H for the trials whose
// Woodbury step went through (act[b] == 1); T, VhAi: [D][K] per trial.
int lrz_chain_apply_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *act,
                         const void *Tm, const void *VhAi, int64_t ws_stride, const void *prev,
                         int64_t pst, void *Ainv_seq, void *A_state, const void *U,
                         const void *V, const double *S, const int32_t *r, cudaStream_t s) {
  const int64_t KK = int64_t(K) * K;
  ZgArgs a{};
  a.NN = K;
  a.J = K;
  a.Kd = D;
  a.X = Tm;
  a.xs = ws_stride;
  a.ldx = K;
  a.Y = (const c128 *)VhAi;
  a.ys = ws_stride;
  a.ldy = K;
  a.out = (c128 *)Ainv_seq + int64_t(t) * KK;
  a.os = int64_t(T) * KK;
  a.ldo = K;
  a.base = (const c128 *)prev;
  a.bs = pst;
  a.mask = act;
  a.mstride = 1;
  a.mval = 1;
  a.kd_item = r + t;  // T / VhAi rows beyond the rank are not read
  a.kstride = T;
  if (int rc = zgemm_dmma_launch<double, false, false, false, false, 1>(B, a, s,
                                                                          "chain:apply_dmma"))
    return rc;
  if (!A_state) return LRZ_OK;
  ZgArgs b{};
  b.NN = K;
  b.J = K;
  b.Kd = D;
  b.X = (const c128 *)U + int64_t(t) * D * K;
  b.xs = int64_t(T) * D * K;
  b.ldx = K;
  b.Y = (const c128 *)V + int64_t(t) * D * K;
  b.ys = int64_t(T) * D * K;
  b.ldy = K;
  b.out = A_state;
  b.os = KK;
  b.ldo = K;
  b.mask = act;
  b.mstride = 1;
  b.mval = 1;
  b.kd_item = r + t;
  b.kstride = T;
  b.kscale = S + int64_t(t) * D;
  b.kss = int64_t(T) * D;
  return zgemm_dmma_launch<double, false, false, false, true, 2>(B, b, s, "chain:Aupdate_dmma");
}

// arSVD tail pipeline (arsvd.cu): M[j][k] = sum_m Q[j][m] conj(dA[m][k]) = (dA^H Q)
// for the items phase 1 marked (tail == 1); Q, M: [D][K] column blocks inside
// each item's workspace (stride wst elements).
int lrz_arsvd_tail_M(int64_t B, int K, int D, const void *dA, int64_t a_stride, const void *Q,
                     void *M, int64_t wst, const uint8_t *tail, cudaStream_t s) {
  ZgArgs a{};
  a.NN = D;
  a.J = K;
  a.Kd = K;
  a.X = Q;
  a.xs = wst;
  a.ldx = K;
  a.Y = (const c128 *)dA;
  a.ys = a_stride;
  a.ldy = K;
  a.out = M;
  a.os = wst;
  a.ldo = K;
  a.mask = tail;
  a.mstride = 1;
  a.mval = 1;
  return zgemm_dmma_launch<double, true, false, false, true, 0>(B, a, s, "arsvd_tail:M_dmma");
}

// U[j][k] = sum_i Q[i][k] J_perm[i][j] for the items phase 2 marked (tail == 2);
// J_perm column-major d x d (d = D) at the start of the item's M block.
int lrz_arsvd_tail_U(int64_t B, int K, int D, const void *Jp, const void *Q, int64_t wst,
                     void *U, const uint8_t *tail, cudaStream_t s) {
  ZgArgs a{};
  a.NN = D;
  a.J = K;
  a.Kd = D;
  a.X = Jp;
  a.xs = wst;
  a.ldx = D;
  a.Y = (const c128 *)Q;
  a.ys = wst;
  a.ldy = K;
  a.out = U;
  a.os = int64_t(D) * K;
  a.ldo = K;
  a.mask = tail;
  a.mstride = 1;
  a.mval = 2;
  return zgemm_dmma_launch<double, true, false, false, false, 0>(B, a, s, "arsvd_tail:U_dmma");
}

// Blocked Gauss-Jordan rank-b update (inverse_blocked.cu):
//   next[i][k] = cur[i][k] - sum_r Cp[i][r] cur[j0 + r][k]
int lrz_gj_update_dmma(int64_t B, int K, int b, int j0, const void *Cp, const void *Acur,
                       int64_t cst, void *Anext, int64_t nst, const uint8_t *mask,
                       cudaStream_t s) {
  ZgArgs a{};
  a.NN = K;
  a.J = K;
  a.Kd = b;
  a.X = Cp;
  a.xs = int64_t(K) * b;
  a.ldx = b;
  a.Y = (const c128 *)Acur + int64_t(j0) * K;
  a.ys = cst;
  a.ldy = K;
  a.out = Anext;
  a.os = nst;
  a.ldo = K;
  a.base = (const c128 *)Acur;
  a.bs = cst;
  a.mask = mask;
  a.mstride = 1;
  a.mval = 1;
  return zgemm_dmma_launch<double, true, false, false, false, 1>(B, a, s, "gj_update_dmma");
}

// Blocked Gauss-Jordan panels: Cp = A[:, j] Pinv (K x b), Rp = Pinv A[j, :] (b x K)
int lrz_gj_panels_dmma(int64_t B, int K, int b, int j0, const void *Acur, int64_t cst,
                       const void *Pinv, void *Cp, void *Rp, const uint8_t *mask,
                       cudaStream_t s) {
  ZgArgs a{};
  a.NN = K;  // Cp[i][c] = sum_r A[i][j0 + r] Pinv[r][c]
  a.J = b;
  a.Kd = b;
  a.X = (const c128 *)Acur + j0;
  a.xs = cst;
  a.ldx = K;
  a.Y = (const c128 *)Pinv;
  a.ys = int64_t(b) * b;
  a.ldy = b;
  a.out = Cp;
  a.os = int64_t(K) * b;
  a.ldo = b;
  a.mask = mask;
  a.mstride = 1;
  a.mval = 1;
  if (int rc = zgemm_dmma_launch<double, true, false, false, false, 0>(B, a, s, "gj_panel_dmma"))
    return rc;
  ZgArgs c{};
  c.NN = b;  // Rp[r][k] = sum_c Pinv[r][c] A[j0 + c][k]
  c.J = K;
  c.Kd = b;
  c.X = Pinv;
  c.xs = int64_t(b) * b;
  c.ldx = b;
  c.Y = (const c128 *)Acur + int64_t(j0) * K;
  c.ys = cst;
  c.ldy = K;
  c.out = Rp;
  c.os = int64_t(K) * b;
  c.ldo = K;
  c.mask = mask;
  c.mstride = 1;
  c.mval = 1;
  return zgemm_dmma_launch<double, true, false, false, false, 0>(B, c, s, "gj_panel_dmma");
}
