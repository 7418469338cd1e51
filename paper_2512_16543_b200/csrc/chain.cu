// K5 batched Hermitian inverse, K4 Woodbury update, the per-trial chain of
// the batched runner, and the speculative sketch-cursor verifier.

#include <stdlib.h>

#include <cooperative_groups.h>

#include "dmma.cuh"
#include "linalg.cuh"

int lrz_use_dmma();

namespace lrz {

constexpr int INV_THREADS = 256;
constexpr int INV_SMEM_KMAX = 64;   // K <= 64: factorise in shared memory

struct InvSmem {
  // layout inside dynamic shared memory
  __host__ __device__ static size_t bytes(int K, int rmax, bool matrix) {
    const int n = K > rmax ? K : rmax;
    size_t b = 4 * size_t(n) * sizeof(c128) + size_t(n) * sizeof(int) +
               (INV_THREADS / 32) * (sizeof(double) * 2 + sizeof(int));
    b = (b + 15) & ~size_t(15);
    if (matrix) b += size_t(K) * K * sizeof(c128);
    return b;
  }
};

LRZ_DEV InvScratch carve_inv(char *sm, int n, c128 **matrix, int K, bool want_matrix) {
  InvScratch s;
  s.colbuf = (c128 *)sm;
  s.rowbuf = s.colbuf + n;
  s.v = s.rowbuf + n;
  s.w = s.v + n;
  s.red = (double *)(s.w + n);
  s.ired = (int *)(s.red + 2 * (INV_THREADS / 32));
  s.perm = s.ired + (INV_THREADS / 32);
  size_t off = size_t((char *)(s.perm + n) - sm);
  off = (off + 15) & ~size_t(15);
  *matrix = want_matrix ? (c128 *)(sm + off) : nullptr;
  return s;
}

constexpr int WB_SMEM_DMAX = 40;  // aux / aux^-1 in shared memory up to this rank

__host__ __device__ inline int64_t wb_ws_elems(int K, int D) {
  // AiU, T, VhAi (K x D each) [+ aux, aux^-1 when they do not fit shared memory]
  // + the DMMA chain's aux and aux^-1 in global memory (D x D each)
  return 3 * int64_t(K) * D + (D > WB_SMEM_DMAX ? 2 * int64_t(D) * (D + 1) : 0) +
         2 * int64_t(D) * D;
}
// offset of the DMMA chain's global aux (then aux^-1) inside a trial's workspace
__host__ __device__ inline int64_t wb_ws_aux_off(int K, int D) {
  return 3 * int64_t(K) * D + (D > WB_SMEM_DMAX ? 2 * int64_t(D) * (D + 1) : 0);
}
__host__ __device__ inline size_t wb_aux_smem(int D) {
  // D x (D + 1) each: the resident chain keeps aux / aux^-1 at an odd row stride
  return D > WB_SMEM_DMAX ? 0 : 2 * size_t(D) * (D + 1) * sizeof(c128);
}
LRZ_DEV void carve_wb(WbScratch &sc, char *aux_smem, c128 *w, int K, int D) {
  sc.AiU = w;
  sc.T = w + int64_t(K) * D;
  sc.VhAi = w + 2 * int64_t(K) * D;
  sc.aux = D > WB_SMEM_DMAX ? w + 3 * int64_t(K) * D : (c128 *)aux_smem;
  sc.auxinv = sc.aux + D * (D + 1);
}

__global__ void __launch_bounds__(INV_THREADS)
    herm_inverse_kernel(int K, const c128 *A, int64_t as, c128 *Ainv, int64_t ais,
                        int32_t *info, double limit, const uint8_t *mask) {
  extern __shared__ __align__(16) char smem[];
  const int64_t item = blockIdx.x;
  if (mask && !mask[item]) return;
  c128 *M;
  const InvScratch sc = carve_inv(smem, K, &M, K, K <= INV_SMEM_KMAX);
  const int st = cta_herm_inverse(A + item * as, Ainv + item * ais, K, M, limit, sc);
  if (threadIdx.x == 0 && info) info[item] = st;
}

// ---------------------------------------------------------------------------
// K5 for 64 < K <= 256: the K x K complex128 matrix (256 KB at K = 128, 1 MB at
// K = 256) does not fit one SM's shared memory, so a thread-block cluster of
// CS CTAs holds it in distributed shared memory, R = ceil(K / CS) rows each.
// In-place Gauss-Jordan without pivoting (the HPD fast path of
// cta_gauss_jordan): at step k the owner of row k scales it and writes it into
// every cluster member's row buffer over DSMEM; one cluster barrier per step
// (row buffers are double-buffered).  Items that are not positive definite or
// whose ||A||_F ||A^-1||_F bound exceeds the limit are flagged in `redo` for
// the single-CTA kernel (pivoted path / power-iteration condition estimate).
// ---------------------------------------------------------------------------
constexpr int CINV_THREADS = 512;
constexpr int CINV_BMAX = 16;

// In-place inverse of the bb x bb HPD block D (row stride ld) by one warp:
// Gauss-Jordan without pivoting, lane i owns row i.  False on a non-positive
// or non-finite pivot.
LRZ_DEV bool warp_small_gj(c128 *D, int bb, int ld) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < bb; ++k) {
    const c128 piv = D[k * ld + k];
    if (!(piv.re > 0.0 && isfinite(piv.re) && isfinite(piv.im))) return false;
    const c128 pinv = cinv(piv);
    c128 c = czero<double>();
    if (lane < bb) c = D[lane * ld + k];
    __syncwarp();
    if (lane < bb) {
      for (int j = 0; j < bb; ++j) {
        const c128 r = (j == k) ? mk<double>(1.0, 0.0) : D[k * ld + j];
        const c128 rs = cmul(r, pinv);       // scaled pivot-row entry (row k of the result)
        c128 &m = D[lane * ld + j];
        if (lane == k) {
          m = (j == k) ? pinv : rs;
        } else if (j == k) {
          m = cmul(mk<double>(-c.re, -c.im), pinv);
        } else {
          m.re = fma(-c.re, rs.re, m.re);
          m.re = fma(c.im, rs.im, m.re);
          m.im = fma(-c.re, rs.im, m.im);
          m.im = fma(-c.im, rs.re, m.im);
        }
      }
    }
    __syncwarp();
  }
  return true;
}

// Blocked in-place Gauss-Jordan over the cluster: for each pivot block p of
// bb rows (owned by one CTA) the owner inverts D = M_pp, forms the new pivot
// block rows P = [D^-1 M_pq | D^-1] and pushes them to every member over
// DSMEM; after one cluster barrier every CTA applies the rank-bb update
// M_iq -= M_ip P_q, M_ip = -M_ip D^-1 to its own rows.  K / bb barriers.
__global__ void __launch_bounds__(CINV_THREADS)
    herm_inverse_cluster_kernel(int K, int CS, int bsz, const c128 *__restrict__ A, int64_t as,
                                c128 *__restrict__ Ainv, int64_t ais, int32_t *__restrict__ info,
                                double limit, const uint8_t *__restrict__ mask,
                                uint8_t *__restrict__ redo) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) char cs_smem[];
  const int R = (K + CS - 1) / CS;
  c128 *Mloc = (c128 *)cs_smem;             // [R][K] this CTA's rows
  c128 *Pbuf = Mloc + R * K;                // [2][bsz][K] pivot block rows (written remotely)
  c128 *Cs = Pbuf + 2 * bsz * K;            // [R][bsz] saved M_ip of own rows
  c128 *Dm = Cs + R * bsz;                  // [bsz][bsz + 1] owner's pivot block
  __shared__ double red[CINV_THREADS / 32];
  __shared__ double s_fa[8], s_fi[8];
  __shared__ int s_bad;
  const int rank = int(cl.block_rank());
  const int64_t item = blockIdx.x / CS;
  const bool active = !(mask && !mask[item]);
  const int tid = threadIdx.x, NT = blockDim.x;
  const int r0 = rank * R, nr = max(0, min(R, K - r0));
  const int nblk = (K + bsz - 1) / bsz;
  const c128 *a = A + item * as;
  double loc = 0.0;
  if (active)
    for (int e = tid; e < nr * K; e += NT) {
      const c128 v = a[int64_t(r0) * K + e];
      Mloc[e] = v;
      loc += cabs2(v);
    }
  const double fa_part = block_sum(loc, red);
  if (tid == 0) s_bad = 0;
  cl.sync();
  if (!active) {   // every member must still take part in the cluster barriers
    for (int n = 0; n < nblk; ++n) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    }
    cl.sync();
    if (rank == 0 && tid == 0) redo[item] = 0;
    return;
  }
  const int LDD = bsz + 1;
  for (int n = 0; n < nblk; ++n) {
    const int k0 = n * bsz, bb = min(bsz, K - k0);
    const int owner = k0 / R, lk0 = k0 - owner * R;
    c128 *P = Pbuf + (n & 1) * bsz * K;
    if (rank == owner) {
      // D = M_pp, inverted by warp 0
      for (int e = tid; e < bb * bb; e += NT) Dm[(e / bb) * LDD + e % bb] = Mloc[(lk0 + e / bb) * K + k0 + e % bb];
      __syncthreads();
      if (tid < 32) {
        const bool ok = warp_small_gj(Dm, bb, LDD);
        if (tid == 0 && !ok)
          for (int q = 0; q < CS; ++q) *cl.map_shared_rank(&s_bad, q) = 1;
      }
      __syncthreads();
      // P[t][j] = (D^-1 M_p)[t][j] for j outside the block, D^-1[t][j - k0] inside
      for (int e = tid; e < bb * K; e += NT) {
        const int t = e / K, j = e - t * K;
        c128 v;
        if (j >= k0 && j < k0 + bb) {
          v = Dm[t * LDD + (j - k0)];
        } else {
          v = czero<double>();
          for (int u = 0; u < bb; ++u) cfma(v, Dm[t * LDD + u], Mloc[(lk0 + u) * K + j]);
        }
        for (int q = 0; q < CS; ++q) *cl.map_shared_rank(P + e, q) = v;
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
    }
    // own rows' M_ip, saved before the update overwrites them
    for (int e = tid; e < nr * bb; e += NT) Cs[(e / bb) * bsz + e % bb] = Mloc[(e / bb) * K + k0 + e % bb];
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (s_bad) continue;   // uniform across the cluster (set before the barrier)
    // rank-bb update: thread -> column j (tpc threads per column), P_j in registers
    const int tpc = max(1, NT / K);
    if (tid < tpc * K) {
      const int j = tid % K, i0 = tid / K;
      const bool inblk = (j >= k0 && j < k0 + bb);
      c128 pc[CINV_BMAX];
#pragma unroll
      for (int t = 0; t < CINV_BMAX; ++t) pc[t] = (t < bb) ? P[t * K + j] : czero<double>();
      for (int i = i0; i < nr; i += tpc) {
        c128 &m = Mloc[i * K + j];
        if (rank == owner && i >= lk0 && i < lk0 + bb) {
          m = pc[i - lk0];   // pivot block rows: P itself
          continue;
        }
        c128 acc = inblk ? czero<double>() : m;
        const c128 *ci = Cs + i * bsz;
#pragma unroll
        for (int t = 0; t < CINV_BMAX; ++t) {
          if (t < bb) {
            const c128 c = ci[t];
            acc.re = fma(-c.re, pc[t].re, acc.re);
            acc.re = fma(c.im, pc[t].im, acc.re);
            acc.im = fma(-c.re, pc[t].im, acc.im);
            acc.im = fma(-c.im, pc[t].re, acc.im);
          }
        }
        m = acc;
      }
    }
    __syncthreads();
  }
  // ||A||_F^2 and ||A^-1||_F^2 summed over the cluster
  double li = 0.0;
  for (int e = tid; e < nr * K; e += NT) li += cabs2(Mloc[e]);
  const double fi_part = block_sum(li, red);
  // gather the partial sums at rank 0 through DSMEM
  if (tid == 0) {
    *cl.map_shared_rank(&s_fa[rank], 0) = fa_part;
    *cl.map_shared_rank(&s_fi[rank], 0) = fi_part;
  }
  cl.sync();
  bool flag = s_bad != 0;
  if (rank == 0 && tid == 0) {
    double fa = 0.0, fi = 0.0;
    for (int q = 0; q < CS; ++q) {
      fa += s_fa[q];
      fi += s_fi[q];
    }
    const double fb = sqrt(fa) * sqrt(fi);
    const bool good = !flag && isfinite(fb) && fb <= limit;
    redo[item] = good ? 0 : 1;
    if (good && info) info[item] = LRZ_INFO_OK;
  }
  if (!flag) {
    c128 *o = Ainv + item * ais;
    for (int e = tid; e < nr * K; e += NT) o[int64_t(r0) * K + e] = Mloc[e];
  }
}

// Batched Woodbury (single step per item).
__global__ void __launch_bounds__(INV_THREADS)
    woodbury_kernel(int K, int D, const c128 *A, const c128 *Ainv, int64_t as, const c128 *U,
                    const c128 *V, const double *S, const int32_t *r, c128 *A_out,
                    c128 *Ainv_out, int32_t *info, c128 *ws) {
  extern __shared__ __align__(16) char smem[];
  const int64_t item = blockIdx.x;
  const int rr = r[item];
  WbScratch sc;
  c128 *unused;
  sc.inv = carve_inv(smem, D, &unused, D, false);
  c128 *w = ws + item * wb_ws_elems(K, D);
  carve_wb(sc, smem + InvSmem::bytes(D, D, false), w, K, D);
  if (rr < 1 || rr > D) {
    if (threadIdx.x == 0) info[item] = LRZ_INFO_SINGULAR_AUX;
    return;
  }
  const int st = cta_woodbury(K, rr, Ainv + item * as, Ainv_out + item * as,
                              A ? A + item * as : nullptr, A_out ? A_out + item * as : nullptr,
                              U + item * int64_t(D) * K, V + item * int64_t(D) * K,
                              S + item * D, sc);
  if (threadIdx.x == 0) info[item] = st;
}

// ---------------------------------------------------------------------------
// Resident Woodbury step on the FP64 tensor pipe (K <= 32, r <= 32; every
// operand in shared memory).  The step of cta_woodbury (lowrank.py:208-220)
// with each product cut into 8 x 8 complex output blocks that the CTA's warps
// take round robin (mma.sync m8n8k4 f64, four real DMMAs per complex k-step,
// fragments straight from the resident tiles), and the r x r auxiliary inverse
// -- pivoted Gauss-Jordan, as cta_gauss_jordan -- done by one warp on
// __syncwarp while the other warps apply A += (U S) V^H.  One CTA issued ~1
// instruction per cycle on the SIMT version (ncu: pivot search over CTA
// barriers 20 %, LDS-bound cfma loops); this one is bound by the DMMA pipe.
// ---------------------------------------------------------------------------
template <class FA, class FB>
LRZ_DEV void blk_zmma(int ksteps, FA a, FB b, double (&cr)[2], double (&ci)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int c = 0; c < ksteps; ++c) {
    const c128 av = a(g, 4 * c + t), bv = b(4 * c + t, g);
    dmma(cr, av.re, bv.re);
    dmma(cr, -av.im, bv.im);
    dmma(ci, av.re, bv.im);
    dmma(ci, av.im, bv.re);
  }
}

// In-place inverse of the r x r matrix M (r <= 16, row stride ldm, shared memory)
// by one warp with the matrix in registers: lane l holds row l / 2, columns
// 8 (l & 1) .. + 7.  Gauss-Jordan with implicit row pivoting (no swaps: the pivot
// of column k is the largest |m|^2 among the rows not used yet, smallest row on
// ties; the row and column permutations are applied when the result is written
// back), the pivot loop fully unrolled so every register index is static, one
// warp-wide exchange per pivot (the scaled pivot row through rowbuf, the
// reciprocal and the column-k entries by shuffles).  ~170 instructions per
// pivot against ~390 of a shared-memory warp version -- the warp is bound by
// instruction count x latency.  Returns 0, or 2 on a zero / non-finite pivot;
// fro2 = ||M^-1||_F^2.  Warp-uniform; all 32 lanes must call.
LRZ_DEV int warp_gj_reg16(c128 *M, int r, int ldm, c128 *rowbuf, double &fro2) {
  const int lane = threadIdx.x & 31, row = lane >> 1, half = lane & 1, c0 = 8 * half;
  c128 m[8];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj)
    m[jj] = (row < r && c0 + jj < r) ? M[row * ldm + c0 + jj] : czero<double>();
  bool used = false;
  int logical = 0;          // pivot step at which my row was used = its row in (P A)^-1
  int pcol_of[16];          // pivot row of step k (warp-uniform)
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k >= r) break;
    const int kh = k >> 3, kk = k & 7;
    const bool holder = half == kh && row < r && !used;
    const double mag = holder ? cabs2(m[kk]) : 0.0;
    const unsigned long long bits = (mag == mag) ? (unsigned long long)__double_as_longlong(mag)
                                                 : 0xFFFFFFFFFFFFFFFFull;
    const unsigned hi = unsigned(bits >> 32), lo = unsigned(bits);
    const unsigned mh = __reduce_max_sync(0xffffffffu, holder ? hi : 0u);
    const unsigned ml = __reduce_max_sync(0xffffffffu, (holder && hi == mh) ? lo : 0u);
    const unsigned bal = __ballot_sync(0xffffffffu, holder && hi == mh && lo == ml);
    if (bal == 0u || (mh == 0u && ml == 0u) || mh >= 0x7FF00000u) return 2;
    const int pl = __ffs(bal) - 1, prow = pl >> 1;
    pcol_of[k] = prow;
    // reciprocal of the pivot (on its holder), then to every lane
    const c128 pv = m[kk];
    const double id = 1.0 / cabs2(pv);
    c128 pinv = mk<double>(pv.re * id, -pv.im * id);
    pinv.re = __shfl_sync(0xffffffffu, pinv.re, pl);
    pinv.im = __shfl_sync(0xffffffffu, pinv.im, pl);
    if (!(isfinite(pinv.re) && isfinite(pinv.im))) return 2;
    // my row's column-k entry (held by the lane of my row with half == kh)
    const int src = (lane & ~1) | kh;
    c128 c;
    c.re = __shfl_sync(0xffffffffu, m[kk].re, src);
    c.im = __shfl_sync(0xffffffffu, m[kk].im, src);
    const bool mine = row == prow;
    if (mine) {
      used = true;
      logical = k;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        rowbuf[c0 + jj] = (c0 + jj == k) ? pinv : cmul(m[jj], pinv);
    }
    __syncwarp();
    const c128 nc = cmul(mk<double>(-c.re, -c.im), pinv);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const c128 rj = rowbuf[c0 + jj];
      c128 x = m[jj];
      x.re = fma(-c.re, rj.re, x.re);
      x.re = fma(c.im, rj.im, x.re);
      x.im = fma(-c.re, rj.im, x.im);
      x.im = fma(-c.im, rj.re, x.im);
      m[jj] = mine ? rj : ((c0 + jj == k) ? nc : x);
    }
    __syncwarp();
  }
  // register slot l of the lane whose row was used at step i is (A^-1)[i][pivot row of l]
  double loc = 0.0;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int l = c0 + jj;
    int pr = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q == l) pr = pcol_of[q];   // static after unrolling
    if (row < r && l < r) {
      M[logical * ldm + pr] = m[jj];
      loc += cabs2(m[jj]);
    }
  }
  __syncwarp();
  fro2 = warp_sum(loc);
  return 0;
}

// Ainv_in / Ainv_out: K x K at row stride ld; U, V, sc.AiU, sc.T: column j at
// j * ld; sc.VhAi: row j at j * ld; A (nullable, in place): K x K at stride K.
// Returns LRZ_INFO_OK or LRZ_INFO_SINGULAR_AUX (then Ainv_out is untouched and
// A is garbage: the caller's full branch overwrites both).
LRZ_DEV int cta_woodbury_dmma(int K, int r, const c128 *__restrict__ Ai, c128 *Ainv_out, c128 *A,
                              const c128 *__restrict__ U, const c128 *__restrict__ V,
                              const double *__restrict__ S, const WbScratch &sc, int ld) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NW = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int KB = (K + 7) >> 3, RB = (r + 7) >> 3, ksK = (K + 3) >> 2, ksr = (r + 3) >> 2;
  const int lda = r | 1;  // odd row stride of aux / aux^-1 (bank spread for lane = row)
  const c128 Z = czero<double>();
  __shared__ double s_fi;
  __shared__ int s_st;
  // 1. AiU = A^-1 U (K x r), VhAi = V^H A^-1 (r x K)
  for (int blk = wid; blk < 2 * KB * RB; blk += NW) {
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
    if (blk < KB * RB) {
      const int k0 = 8 * (blk / RB), j0 = 8 * (blk % RB);
      blk_zmma(
          ksK,
          [&](int i, int m) { return (k0 + i < K && m < K) ? Ai[(k0 + i) * ld + m] : Z; },
          [&](int m, int j) { return (m < K && j0 + j < r) ? U[(j0 + j) * ld + m] : Z; }, cr, ci);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = k0 + g, j = j0 + 2 * t + e;
        if (k < K && j < r) sc.AiU[j * ld + k] = mk<double>(cr[e], ci[e]);
      }
    } else {
      const int b2 = blk - KB * RB, j0 = 8 * (b2 / KB), m0 = 8 * (b2 % KB);
      blk_zmma(
          ksK,
          [&](int i, int k) { return (j0 + i < r && k < K) ? cconj(V[(j0 + i) * ld + k]) : Z; },
          [&](int k, int m) { return (k < K && m0 + m < K) ? Ai[k * ld + m0 + m] : Z; }, cr, ci);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = j0 + g, m = m0 + 2 * t + e;
        if (j < r && m < K) sc.VhAi[j * ld + m] = mk<double>(cr[e], ci[e]);
      }
    }
  }
  __syncthreads();
  // 2. aux = diag(1/S) + V^H AiU  (r x r, both copies at stride lda)
  double loc = 0.0;
  for (int blk = wid; blk < RB * RB; blk += NW) {
    const int i0 = 8 * (blk / RB), j0 = 8 * (blk % RB);
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
    blk_zmma(
        ksK, [&](int i, int k) { return (i0 + i < r && k < K) ? cconj(V[(i0 + i) * ld + k]) : Z; },
        [&](int k, int j) { return (k < K && j0 + j < r) ? sc.AiU[(j0 + j) * ld + k] : Z; }, cr, ci);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = i0 + g, j = j0 + 2 * t + e;
      if (i < r && j < r) {
        c128 a = mk<double>(cr[e], ci[e]);
        if (i == j) a.re = 1.0 / S[i] + a.re;
        sc.aux[i * lda + j] = a;
        sc.auxinv[i * lda + j] = a;
        loc += cabs2(a);
      }
    }
  }
  const double fa = block_sum(loc, sc.inv.red);
  __syncthreads();
  // 3. warp 0: aux^-1; the other warps: A += (U S) V^H (overwritten by the
  //    caller's full branch if the step turns out singular)
  // r <= 16: warp 0 inverts in registers while the other warps update A; wider
  // aux matrices take the whole CTA (cta_gj_pivot_small: two barriers per pivot,
  // the rank-1 update spread over all threads), so every warp updates A first
  const bool wide = r > 16;
  if (!wide && wid == 0) {
    double fi = 0.0;
    const int st = warp_gj_reg16(sc.auxinv, r, lda, sc.inv.rowbuf, fi);
    if (lane == 0) {
      s_st = st;
      s_fi = fi;
    }
  } else if (A) {
    for (int blk = wide ? wid : wid - 1; blk < KB * KB; blk += wide ? NW : NW - 1) {
      const int k0 = 8 * (blk / KB), m0 = 8 * (blk % KB);
      double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
      // A's entries first: for K > 32 they come from global memory, and the load
      // then overlaps the block's DMMAs instead of stalling the write-back
      c128 x[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = k0 + g, m = m0 + 2 * t + e;
        x[e] = (k < K && m < K) ? A[k * K + m] : Z;
      }
      blk_zmma(
          ksr,
          [&](int i, int j) {
            return (k0 + i < K && j < r) ? cscale(U[j * ld + k0 + i], S[j]) : Z;
          },
          [&](int j, int m) { return (j < r && m0 + m < K) ? cconj(V[j * ld + m0 + m]) : Z; }, cr,
          ci);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = k0 + g, m = m0 + 2 * t + e;
        if (k < K && m < K) A[k * K + m] = mk<double>(x[e].re + cr[e], x[e].im + ci[e]);
      }
    }
  }
  __syncthreads();
  double fi_all;
  if (wide) {
    if (cta_gauss_jordan(sc.auxinv, r, lda, true, sc.inv.colbuf, sc.inv.rowbuf, sc.inv.perm,
                         sc.inv.red, sc.inv.ired) != 0)
      return LRZ_INFO_SINGULAR_AUX;
    fi_all = cta_fro2(sc.auxinv, r, lda, sc.inv.red);
  } else {
    if (s_st != 0) return LRZ_INFO_SINGULAR_AUX;
    fi_all = s_fi;
  }
  // the 1e12 condition guard (lowrank.py:212-217); sc.aux is free after this
  if (!cta_cond_ok(fa, fi_all, 1e12, sc.aux, r, lda, sc.inv.red, sc.inv.ired))
    return LRZ_INFO_SINGULAR_AUX;
  // 4. T = AiU aux^-1 (K x r)
  for (int blk = wid; blk < KB * RB; blk += NW) {
    const int k0 = 8 * (blk / RB), j0 = 8 * (blk % RB);
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
    blk_zmma(
        ksr, [&](int kk, int i) { return (k0 + kk < K && i < r) ? sc.AiU[i * ld + k0 + kk] : Z; },
        [&](int i, int j) { return (i < r && j0 + j < r) ? sc.auxinv[i * lda + j0 + j] : Z; }, cr,
        ci);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = k0 + g, j = j0 + 2 * t + e;
      if (k < K && j < r) sc.T[j * ld + k] = mk<double>(cr[e], ci[e]);
    }
  }
  __syncthreads();
  // 5. A^-1 - T VhAi
  for (int blk = wid; blk < KB * KB; blk += NW) {
    const int k0 = 8 * (blk / KB), m0 = 8 * (blk % KB);
    double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
    blk_zmma(
        ksr, [&](int kk, int j) { return (k0 + kk < K && j < r) ? sc.T[j * ld + k0 + kk] : Z; },
        [&](int j, int m) { return (j < r && m0 + m < K) ? sc.VhAi[j * ld + m0 + m] : Z; }, cr, ci);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = k0 + g, m = m0 + 2 * t + e;
      if (k < K && m < K) {
        const c128 o = Ai[k * ld + m];
        Ainv_out[k * ld + m] = mk<double>(o.re - cr[e], o.im - ci[e]);
      }
    }
  }
  __syncthreads();
  return LRZ_INFO_OK;
}

// Per-trial chain over T steps (harness.py:228-241 semantics):
//   plan 0 (full):     A_inv_seq[t] already holds inv(G_t); A_state = G_t
//   plan 1 (Woodbury): A_inv_seq[t] = woodbury(A_inv_seq[t-1]); on SingularAux
//                      fall back to inv(G_t) (lowrank.py:353-367)
//   plan 2 (none):     A_inv_seq[t] = A_inv_seq[t-1] (lowrank.py:345-351)
// K <= 32: the trial's A^-1 (double buffered), A, the step's U / V and the
// Woodbury intermediates (A^-1 U, T, V^H A^-1) stay in shared memory, so the
// serial chain pays one global-load latency per step (U / V by cp.async)
// instead of one per dependent product; the arithmetic and its order are the
// global-memory path's, so the results are bit-identical.
constexpr int CH_PLAN_BLK = 1024;  // plan entries staged per block of steps
// Resident layouts.  K <= 32: A^-1 double buffered, A resident, (U, V) double
// buffered.  32 < K <= 64 (DMMA step only): one A^-1 buffer updated in place,
// A stays in global memory (its update is off the critical path), the fallback
// inverse factorises in place in global memory, (U, V) double buffered when
// that still fits the SM's shared memory.
struct ChainPlan {
  int aibufs, uvbufs;
  bool a_res, matrix, ok;
  size_t base, bytes;
};
constexpr size_t CHAIN_SMEM_MAX = 227 * 1024;
__host__ __device__ inline ChainPlan chain_plan(int K, int D) {
  ChainPlan p{};
  p.ok = K <= 64 && D <= 32;
  if (!p.ok) return p;
  const bool small = K <= 32;
  p.aibufs = small ? 2 : 1;
  p.a_res = small;
  p.matrix = small;
  p.base = (InvSmem::bytes(K, D, p.matrix) + wb_aux_smem(D) + 15) & ~size_t(15);
  const size_t ld = size_t(K) + 1;
  auto total = [&](int uv) {
    return p.base + (p.aibufs * size_t(K) * ld + (p.a_res ? size_t(K) * K : 0) +
                     (2 * uv + 3) * ld * D) * sizeof(c128);
  };
  p.uvbufs = total(2) <= CHAIN_SMEM_MAX ? 2 : 1;
  p.bytes = total(p.uvbufs);
  p.ok = p.bytes <= CHAIN_SMEM_MAX;
  return p;
}
__host__ __device__ inline bool chain_resident(int K, int D) { return chain_plan(K, D).ok; }

LRZ_DEV void chain_cp16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// Per-trial chain over T steps (harness.py:228-241 semantics):
//   plan 0 (full):     A_inv_seq[t] already holds inv(G_t); A_state = G_t
//   plan 1 (Woodbury): A_inv_seq[t] = woodbury(A_inv_seq[t-1]); on SingularAux
//                      fall back to inv(G_t) (lowrank.py:353-367)
//   plan 2 (none):     A_inv_seq[t] = A_inv_seq[t-1] (lowrank.py:345-351)
__global__ void __launch_bounds__(INV_THREADS)
    chain_kernel(int T, int K, int D, const uint8_t *plan, const c128 *G, const c128 *Ainv_prev,
                 c128 *Ainv_seq, c128 *A_state, const c128 *U, const c128 *V, const double *S,
                 const int32_t *r, uint8_t *method, int32_t *info, c128 *ws, int resident) {
  extern __shared__ __align__(16) char smem[];
  const int64_t b = blockIdx.x;
  const int64_t KK = int64_t(K) * K;
  const int n = K > D ? K : D;
  const int tid = threadIdx.x, NT = blockDim.x;
  c128 *M;
  WbScratch sc;
  const bool res = resident != 0;
  const bool dmma_step = resident == 2;  // the step's products on the FP64 tensor pipe
  const ChainPlan cp = res ? chain_plan(K, D) : ChainPlan{};
  const bool want_m = res ? cp.matrix : K <= INV_SMEM_KMAX;
  sc.inv = carve_inv(smem, n, &M, K, want_m);
  c128 *sAi = nullptr, *sA = nullptr, *sU = nullptr, *sV = nullptr;
  const int ld = K + 1;                   // resident stride (bank spread)
  // one resident A^-1 buffer; 0 when the single buffer is updated in place
  const int64_t KL = (res && cp.aibufs == 2) ? int64_t(K) * ld : 0;
  if (res) {
    sAi = (c128 *)(smem + cp.base);                // [aibufs][K][ld]
    sA = sAi + cp.aibufs * int64_t(K) * ld;        // [K][K] when A is resident
    sU = sA + (cp.a_res ? KK : 0);                 // [uvbufs][U | V][D][ld]
    sV = sU + int64_t(ld) * D;
    carve_wb(sc, smem + InvSmem::bytes(K, D, want_m), sU + 2 * cp.uvbufs * int64_t(ld) * D, ld,
             D);
  } else {
    carve_wb(sc, smem + InvSmem::bytes(K, D, K <= INV_SMEM_KMAX), ws + b * wb_ws_elems(K, D),
             K, D);
  }
  c128 *Ast = A_state ? A_state + b * KK : nullptr;
  int cb = 0;  // resident: sAi + cb KL holds A^-1 of the previous step
  int ub = 0;            // resident: the (U, V) buffer pair of the current Woodbury step
  bool uv_ready = false; // its factors were requested by the previous step
  // resident tiles are filled lazily (a chunk of full inversions never reads them)
  bool have_ai = false, have_a = false;
  // where the A state lives (resident only for K <= 32)
  const bool a_res = res && cp.a_res;
  c128 *Acur = a_res ? (Ast ? sA : nullptr) : Ast;
  // the trial's plan row is staged in shared memory block by block (with one
  // entry of lookahead): a chunk of full inversions then costs no dependent
  // global load per step
  __shared__ uint8_t s_plan[CH_PLAN_BLK + 1];
  for (int t = 0; t < T; ++t) {
    const int64_t bt = b * T + t;
    if (t % CH_PLAN_BLK == 0) {
      __syncthreads();
      for (int i = tid; i <= CH_PLAN_BLK && t + i < T; i += NT) s_plan[i] = plan[bt + i];
      __syncthreads();
    }
    const int pl = s_plan[t % CH_PLAN_BLK];
    c128 *out = Ainv_seq + bt * KK;
    const c128 *prev = (t == 0) ? Ainv_prev + b * KK : out - KK;
    int m = LRZ_METHOD_FULL, st = LRZ_INFO_OK;
    bool reload = false;  // resident: A^-1 of this step is in `out` (global)
    if (res && pl != 0 && !have_ai) {  // A^-1 of the previous step, from global
      for (int64_t e = tid; e < KK; e += NT) sAi[cb * KL + (e / K) * ld + e % K] = prev[e];
      if (a_res && Ast && !have_a)
        for (int64_t e = tid; e < KK; e += NT) sA[e] = Ast[e];
      have_ai = true;
      have_a = true;
      __syncthreads();
    }
    if (pl == 1) {
      const c128 *Ub = U + bt * int64_t(D) * K, *Vb = V + bt * int64_t(D) * K;
      if (res) {
        // this step's factors (unless the previous step prefetched them), then the
        // next Woodbury step's into the other buffer pair: its load latency
        // overlaps this step's arithmetic
        const int64_t UV2 = cp.uvbufs == 2 ? 2 * int64_t(ld) * D : 0;
        auto fetch = [&](int64_t bt2, int buf) {
          const int rk = r[bt2] * K;
          const c128 *Ug = U + bt2 * int64_t(D) * K, *Vg = V + bt2 * int64_t(D) * K;
          c128 *du = sU + buf * UV2, *dv = sV + buf * UV2;
          for (int e = tid; e < rk; e += NT) {
            const int o = (e / K) * ld + e % K;
            chain_cp16(du + o, Ug + e);
            chain_cp16(dv + o, Vg + e);
          }
          asm volatile("cp.async.commit_group;\n" ::);
        };
        if (!uv_ready) fetch(bt, ub);
        const bool nxt = cp.uvbufs == 2 && t + 1 < T && s_plan[t % CH_PLAN_BLK + 1] == 1;
        if (nxt) {
          fetch(bt + 1, ub ^ 1);
          asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const c128 *cU = sU + ub * UV2, *cV = sV + ub * UV2;
        st = dmma_step ? cta_woodbury_dmma(K, r[bt], sAi + cb * KL, sAi + (cb ^ 1) * KL, Acur, cU,
                                           cV, S + bt * D, sc, ld)
                       : cta_woodbury(K, r[bt], sAi + cb * KL, sAi + (cb ^ 1) * KL, Acur, Acur, cU,
                                      cV, S + bt * D, sc, ld);
        uv_ready = nxt;
        if (nxt) ub ^= 1;
        if (st == LRZ_INFO_OK) {
          cb ^= 1;
          for (int64_t e = tid; e < KK; e += NT) out[e] = sAi[cb * KL + (e / K) * ld + e % K];
        }
      } else {
        st = cta_woodbury(K, r[bt], prev, out, Ast, Ast, Ub, Vb, S + bt * D, sc);
      }
      if (st == LRZ_INFO_OK) {
        m = LRZ_METHOD_WOODBURY;
      } else {
        // full branch: invert the true Gram of the new channel
        st = cta_herm_inverse(G + bt * KK, out, K, M, 1e14, sc.inv);
        if (Acur)
          for (int64_t e = tid; e < KK; e += NT) Acur[e] = G[bt * KK + e];
        m = LRZ_METHOD_FULL;
        reload = true;
        have_a = true;
      }
    } else if (pl == 2) {
      for (int64_t e = tid; e < KK; e += NT)
        out[e] = res ? sAi[cb * KL + (e / K) * ld + e % K] : prev[e];
      m = LRZ_METHOD_NONE;
    } else {
      // A = G_t; dead if the next step is another full inversion (it overwrites
      // A); needed before a Woodbury or 'none' step and at the chunk end
      const bool needed = (t == T - 1) || s_plan[t % CH_PLAN_BLK + 1] != 0;
      if (Acur && needed)
        for (int64_t e = tid; e < KK; e += NT) Acur[e] = G[bt * KK + e];
      // info[bt] was written by the batched inverse and stays as it is
      reload = needed && t + 1 < T;
      if (needed) have_a = true;
    }
    __syncthreads();
    if (res && reload) {  // out was written by this CTA (fallback) or the batched inverse
      for (int64_t e = tid; e < KK; e += NT) sAi[cb * KL + (e / K) * ld + e % K] = out[e];
      have_ai = true;
      __syncthreads();
    }
    if (tid == 0) {
      method[bt] = uint8_t(m);
      if (info && pl != 0) info[bt] = st;
    }
  }
  if (a_res && Ast && have_a) {
    for (int64_t e = tid; e < KK; e += NT) Ast[e] = sA[e];
  }
}


// ---------------------------------------------------------------------------
// Step-parallel Woodbury chain (K > 32).  chain_kernel walks each trial's
// steps in one CTA, which leaves most of the GPU idle when B is small and
// the K x K products are large (C5: 64 trials x K = 256).  Here the trials
// advance together, one time step per group of launches, and every product is
// batched over the trials (reference lowrank.py:182-227 per trial):
//   1. AiU^T = U^T A^-1^T, VhAi = V^H A^-1        (two batched GEMMs, lrz_chain)
//   2. wb_core_kernel  (CTA per trial): aux = diag(1/S) + V^H AiU, aux^-1 with
//      the 1e12 condition guard, T = AiU aux^-1 (SingularAuxiliary -> fb flag)
//   3. wb_apply_kernel (32 x 32 tiles): A^-1_t = A^-1_{t-1} - T VhAi,
//      A += U S V^H, 'none' copies, A = G_t where the reference re-forms it
//   4. wb_fallback_kernel (CTA per flagged trial): A^-1_t = inv(G_t)
// Same per-step semantics as chain_kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(INV_THREADS)
    wb_core_kernel(int T, int t, int K, int D, const uint8_t *__restrict__ plan,
                   const c128 *__restrict__ V, const double *__restrict__ S,
                   const int32_t *__restrict__ r, c128 *__restrict__ ws, uint8_t *__restrict__ fb,
                   uint8_t *__restrict__ method, int32_t *__restrict__ info, int dmma) {
  extern __shared__ __align__(16) char wbc_smem[];
  const int64_t b = blockIdx.x, bt = b * T + t;
  const int64_t nB = gridDim.x;
  if (plan[bt] != 1) {
    if (threadIdx.x == 0) fb[nB + b] = 0;  // act: no Woodbury apply for this trial
    return;
  }
  const int tid = threadIdx.x, NT = blockDim.x;
  const int rr = r[bt];
  WbScratch sc;
  c128 *unused;
  sc.inv = carve_inv(wbc_smem, D, &unused, D, false);
  carve_wb(sc, wbc_smem + InvSmem::bytes(D, D, false), ws + b * wb_ws_elems(K, D), K, D);
  const c128 *Vb = V + bt * int64_t(D) * K;
  const double *Sb = S + bt * D;
  bool ok = rr >= 1 && rr <= D;
  c128 *aux_g = ws + b * wb_ws_elems(K, D) + wb_ws_aux_off(K, D);  // DMMA path: V^H AiU in
  if (ok) {
    // aux = diag(1/S) + V^H AiU (lowrank.py:208-211)
    double loc = 0.0;
    for (int e = tid; e < rr * rr; e += NT) {
      const int i = e / rr, j = e - i * rr;
      c128 a = czero<double>();
      if (dmma) {
        a = aux_g[i * D + j];
      } else {
        const c128 *vc = Vb + int64_t(i) * K;
        const c128 *au = sc.AiU + int64_t(j) * K;
        for (int k = 0; k < K; ++k) cfma_ca(a, vc[k], au[k]);
      }
      if (i == j) a.re = 1.0 / Sb[i] + a.re;
      sc.aux[e] = a;
      sc.auxinv[e] = a;
      loc += cabs2(a);
    }
    const double fa = block_sum(loc, sc.inv.red);
    // aux^-1 with the 1e12 condition guard (lowrank.py:212-217)
    int st = cta_gauss_jordan(sc.auxinv, rr, rr, true, sc.inv.colbuf, sc.inv.rowbuf,
                              sc.inv.perm, sc.inv.red, sc.inv.ired);
    if (st != 0) {
      ok = false;
    } else {
      const double fi = cta_fro2(sc.auxinv, rr, rr, sc.inv.red);
      ok = cta_cond_ok(fa, fi, 1e12, sc.aux, rr, rr, sc.inv.red, sc.inv.ired);
    }
  }
  if (ok && dmma) {
    // aux^-1 to global memory (D x D, zero beyond r) for the T = AiU aux^-1 GEMM
    __syncthreads();
    c128 *ai_g = aux_g + int64_t(D) * D;
    for (int e = tid; e < D * D; e += NT) {
      const int i = e / D, j = e - i * D;
      ai_g[e] = (i < rr && j < rr) ? sc.auxinv[i * rr + j] : czero<double>();
    }
  } else if (ok) {
    // T = AiU aux^-1 (K x r), zero beyond r; VhAi rows beyond r zeroed too, so the
    // apply stage can run its inner loop over all D columns
    for (int e = tid; e < K * D; e += NT) {
      const int j = e / K, k = e - j * K;
      c128 a = czero<double>();
      if (j < rr)
        for (int i = 0; i < rr; ++i) cfma(a, sc.AiU[int64_t(i) * K + k], sc.auxinv[i * rr + j]);
      sc.T[int64_t(j) * K + k] = a;
      if (j >= rr) sc.VhAi[int64_t(j) * K + k] = czero<double>();
    }
  }
  if (tid == 0) {
    fb[b] = ok ? 0 : 1;
    fb[nB + b] = ok ? 1 : 0;  // act[b]: the Woodbury products apply (DMMA path)
    if (ok) {
      method[bt] = uint8_t(LRZ_METHOD_WOODBURY);
      info[bt] = LRZ_INFO_OK;
    }
  }
}

constexpr int WBA_TILE = 32;

__global__ void __launch_bounds__(256)
    wb_apply_kernel(int T, int t, int K, int D, const uint8_t *__restrict__ plan,
                    const c128 *__restrict__ G, const c128 *__restrict__ prev_base,
                    int64_t prev_stride, c128 *__restrict__ Ainv_seq, c128 *__restrict__ A_state,
                    const c128 *__restrict__ U, const c128 *__restrict__ V,
                    const double *__restrict__ S, const int32_t *__restrict__ r,
                    const c128 *__restrict__ ws, const uint8_t *__restrict__ fb,
                    uint8_t *__restrict__ method, int skip_wb) {
  __shared__ c128 Ts[8][WBA_TILE + 1], Ws[8][WBA_TILE + 1];
  const int nt = (K + WBA_TILE - 1) / WBA_TILE, ntile = nt * nt;
  const int64_t b = blockIdx.x / ntile;
  const int tile = int(blockIdx.x % ntile), I = tile / nt, J = tile % nt;
  const int64_t bt = b * T + t, KK = int64_t(K) * K;
  const int pl = plan[bt];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;  // 8 rows x 32 cols per pass
  const c128 *prev = prev_base + b * prev_stride;
  c128 *out = Ainv_seq + bt * KK;
  c128 *Ast = A_state ? A_state + b * KK : nullptr;
  const c128 *Gt = G + bt * KK;
  const int col = J * WBA_TILE + tx;
  if (pl == 2) {  // 'none': A^-1 aliases the previous one (lowrank.py:345-351)
    for (int i = ty; i < WBA_TILE; i += 8) {
      const int row = I * WBA_TILE + i;
      if (row < K && col < K) out[int64_t(row) * K + col] = prev[int64_t(row) * K + col];
    }
    if (tile == 0 && tid == 0) method[bt] = uint8_t(LRZ_METHOD_NONE);
    return;
  }
  const bool wb = pl == 1 && !fb[b];
  if (!wb) {
    // full step (plan 0, or the SingularAuxiliary fallback): A = G_t where it is
    // still needed -- before a Woodbury / 'none' step and at the chunk end
    const bool needed = (pl == 1) || (t == T - 1) || plan[bt + 1] != 0;
    if (Ast && needed)
      for (int i = ty; i < WBA_TILE; i += 8) {
        const int row = I * WBA_TILE + i;
        if (row < K && col < K) Ast[int64_t(row) * K + col] = Gt[int64_t(row) * K + col];
      }
    if (pl == 0 && tile == 0 && tid == 0) method[bt] = uint8_t(LRZ_METHOD_FULL);
    return;
  }
  if (skip_wb) return;  // the Woodbury products run on DMMA (lrz_chain_apply_dmma)
  const c128 *w = ws + b * wb_ws_elems(K, D);
  const c128 *Tm = w + int64_t(K) * D, *VhAi = w + 2 * int64_t(K) * D;
  const c128 *Ub = U + bt * int64_t(D) * K, *Vb = V + bt * int64_t(D) * K;
  const double *Sb = S + bt * D;
  const int rr = r[bt];  // factor columns beyond the rank do not enter A (lowrank.py:220)
  // rows I*32 + ty + 8 q of the tile, column col: acc over the D factor columns
  c128 acc[4], accA[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = accA[q] = czero<double>();
  for (int j0 = 0; j0 < D; j0 += 8) {
    // stage T[j][rows] and VhAi[j][cols] for 8 factor columns
    __syncthreads();
    {
      const int j = j0 + ty;
      const int row = I * WBA_TILE + tx;
      Ts[ty][tx] = (j < D && row < K) ? Tm[int64_t(j) * K + row] : czero<double>();
      Ws[ty][tx] = (j < D && col < K) ? VhAi[int64_t(j) * K + col] : czero<double>();
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const c128 wv = Ws[jj][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) cfma(acc[q], Ts[jj][ty + 8 * q], wv);
    }
    if (Ast) {
      __syncthreads();
      {
        const int j = j0 + ty;
        const int row = I * WBA_TILE + tx;
        // U S (rows) and V (cols): A += (U S) V^H (lowrank.py:220)
        Ts[ty][tx] = (j < rr && row < K) ? cscale(Ub[int64_t(j) * K + row], Sb[j])
                                        : czero<double>();
        // rows j >= rr of V were never written by arsvd: 0 * NaN must not reach A
        Ws[ty][tx] = (j < rr && col < K) ? Vb[int64_t(j) * K + col] : czero<double>();
      }
      __syncthreads();
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const c128 vv = Ws[jj][tx];
#pragma unroll
        for (int q = 0; q < 4; ++q) cfma_cb(accA[q], Ts[jj][ty + 8 * q], vv);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = I * WBA_TILE + ty + 8 * q;
    if (row < K && col < K) {
      const int64_t e = int64_t(row) * K + col;
      const c128 o = prev[e];
      out[e] = mk<double>(o.re - acc[q].re, o.im - acc[q].im);
      if (Ast) {
        const c128 x = Ast[e];
        Ast[e] = mk<double>(x.re + accA[q].re, x.im + accA[q].im);
      }
    }
  }
}

__global__ void __launch_bounds__(INV_THREADS)
    wb_fallback_kernel(int T, int t, int K, const uint8_t *__restrict__ plan,
                       const c128 *__restrict__ G, c128 *__restrict__ Ainv_seq,
                       const uint8_t *__restrict__ fb, uint8_t *__restrict__ method,
                       int32_t *__restrict__ info) {
  extern __shared__ __align__(16) char wbf_smem[];
  const int64_t b = blockIdx.x, bt = b * T + t, KK = int64_t(K) * K;
  if (plan[bt] != 1 || !fb[b]) return;
  c128 *M;
  const InvScratch sc = carve_inv(wbf_smem, K, &M, K, K <= INV_SMEM_KMAX);
  // full branch: invert the true Gram of the new channel (lowrank.py:353-367)
  const int st = cta_herm_inverse(G + bt * KK, Ainv_seq + bt * KK, K, M, 1e14, sc);
  if (threadIdx.x == 0) {
    method[bt] = uint8_t(LRZ_METHOD_FULL);
    info[bt] = st;
  }
}

// Speculative cursor verification: one thread per trial.
//   is_sketch[b][t]: step runs arsvd.  iters_pred: iterations assumed when the
//   cursor of every later step was computed; iters_act: what the last pass saw.
struct ConsumedTab {
  int64_t v[33];
};
constexpr int SPEC_VOTE_W = LRZ_SPEC_VOTE_W;  // tally slots per step (iteration counts 0 .. 15)

__global__ void spec_verify_kernel(int64_t B, int T, int K, ConsumedTab consumed_tab,
                                   const uint8_t *is_sketch, int32_t *iters_pred,
                                   const int32_t *iters_act, int64_t *cursor,
                                   const int64_t *cursor0, int32_t *first_unverified,
                                   uint8_t *active, int32_t *pending,
                                   uint8_t *__restrict__ votes) {
  // one warp per trial: ballots find the first mispredicted step, a warp scan
  // rebuilds the cursors (32 steps per iteration instead of one)
  const int lane = threadIdx.x & 31;
  const int64_t b = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const int64_t base = b * T;
  int t = first_unverified[b];
  if (votes) {
    // per-step tally of the iteration counts seen so far (every sketch step >= t
    // was evaluated by the last pass, each time with another sketch): the suffix
    // is re-predicted by majority, the first prediction counting as one vote
    for (int s = t + lane; s < T; s += 32) {
      uint8_t *v = votes + (base + s) * SPEC_VOTE_W;
      if (!iters_act) {
        for (int i = 0; i < SPEC_VOTE_W; ++i) v[i] = 0;
        if (is_sketch[base + s]) v[min(iters_pred[base + s], SPEC_VOTE_W - 1)] = 1;
      } else if (is_sketch[base + s]) {
        uint8_t &c = v[min(max(iters_act[base + s], 0), SPEC_VOTE_W - 1)];
        if (c < 255) ++c;
      }
    }
    __syncwarp();
  }
  if (iters_act) {
    // accept the verified prefix: the first sketch step s >= t whose observed
    // iteration count differs from the prediction is corrected and ends it
    int hit = T;
    for (int s0 = t; s0 < T && hit == T; s0 += 32) {
      const int s = s0 + lane;
      bool bad = false;
      if (s < T && is_sketch[base + s]) {
        const int pa = max(iters_act[base + s], 0);  // -1 = window overflow (host)
        bad = pa != iters_pred[base + s];
      }
      const unsigned m = __ballot_sync(0xffffffffu, bad);
      if (m) hit = s0 + __ffs(m) - 1;
    }
    if (hit < T) {
      if (lane == 0) iters_pred[base + hit] = max(iters_act[base + hit], 0);
      t = hit + 1;
    } else {
      t = T;
    }
    __syncwarp();
  }
  // skip trailing non-sketch steps
  for (int s0 = t; s0 < T; s0 += 32) {
    const int s = s0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, s < T && is_sketch[base + s]);
    if (m) {
      t = s0 + __ffs(m) - 1;
      break;
    }
    t = min(s0 + 32, T);
  }
  if (lane == 0) first_unverified[b] = t;
  // re-predict the unverified suffix from the last observation and recompute cursors
  int64_t carry = cursor0[b];
  for (int s0 = 0; s0 < T; s0 += 32) {
    const int s = s0 + lane;
    int64_t inc = 0;
    if (s < T) {
      const int64_t bt = base + s;
      const bool sk = is_sketch[bt];
      if (iters_act && s >= t && sk) {
        int pred = max(iters_act[bt], 0);
        if (votes) {  // majority; ties keep the standing prediction, else the latest count
          const uint8_t *v = votes + bt * SPEC_VOTE_W;
          const int cur_p = min(iters_pred[bt], SPEC_VOTE_W - 1);
          int best = min(pred, SPEC_VOTE_W - 1);
          if (v[cur_p] >= v[best]) best = cur_p;
          for (int i = 0; i < SPEC_VOTE_W; ++i)
            if (v[i] > v[best]) best = i;
          pred = best;
        }
        iters_pred[bt] = pred;
      }
      active[bt] = (s >= t && sk) ? 1 : 0;
      if (sk) inc = consumed_tab.v[iters_pred[bt]];
    }
    // exclusive scan of inc over the lanes
    int64_t x = inc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (s < T) cursor[base + s] = carry + x - inc;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0 && t < T) atomicAdd(pending, 1);
}

// Dispatcher decision per step (lowrank.py:345-359): 2 = none (k_est == 0),
// 1 = Woodbury candidate (k_est / K <= 0.5), 0 = full; non-sketch steps are
// full (step 0 / n_reset, harness.py:229-233).
__global__ void plan_kernel(int64_t n, int K, const uint8_t *is_sketch, const int32_t *k_est,
                            uint8_t *plan) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  uint8_t pl = 0;
  if (is_sketch[i]) {
    const int k = k_est[i];
    pl = (k == 0) ? 2 : ((double(k) / double(K) <= 0.5) ? 1 : 0);
  }
  plan[i] = pl;
}


// K5 fast path for K <= 32: one warp per matrix, lane i holds row i in
// registers (KP = 16 or 32 columns; rows >= K are identity rows), Gauss-Jordan
// without pivoting.  The register row is rotated by one slot per pivot step
// (slot s holds column (s + k) mod KP at step k), so the pivot column is
// always slot 0 and every register index is static inside a rolled loop
// (no per-element selects, a small instruction footprint).  Hermitian
// structure gives the pivot row for free: after pivots 0..k-1 the working
// matrix is [[A_SS^-1, A_SS^-1 A_SU], [-A_US A_SS^-1, Schur]], so
// M[k][j] = conj(M[j][k]) for j > k and -conj(M[j][k]) for j < k -- every lane
// publishes its own entry of the pivot row (one shared store per lane).
// The matrix is read column-wise (conj(A[j][i]): coalesced, the Hermitian
// matrix of the lower triangle) and A^-1 is written the same way.  Items that
// are not positive definite or whose ||A||_F ||A^-1||_F bound exceeds the
// limit are flagged in `redo` for the CTA kernel (pivoted path /
// power-iteration condition estimate).
template <int KP>
__global__ void __launch_bounds__(128, KP > 16 ? 3 : 4)
    herm_inverse_warp_kernel(int64_t B, int K, const c128 *__restrict__ A, int64_t as,
                             c128 *__restrict__ Ainv, int64_t ais, int32_t *__restrict__ info,
                             double limit, const uint8_t *__restrict__ mask,
                             uint8_t *__restrict__ redo) {
  const int lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= B) return;
  if (mask && !mask[item]) {
    // masked out: nothing for the CTA kernel to redo either (the redo array
    // lives in a reused workspace and must not carry a stale flag)
    if (lane == 0) redo[item] = 0;
    return;
  }
  const c128 *a = A + item * as;
  c128 m[KP];
  double fa = 0.0;
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    if (lane < K && j < K) {
      c128 v = cconj(a[j * K + lane]);
      if (j == lane) v.im = 0.0;
      m[j] = v;
      fa += cabs2(v);
    } else {
      m[j] = mk<double>(lane == j ? 1.0 : 0.0, 0.0);
    }
  }
  fa = warp_sum(fa);
  // the scaled pivot row is stored twice (slots lane and lane + KP), so the
  // rotated read of slot (j + 1 + k) mod KP is a constant offset from pr_s + k + 1
  __shared__ c128 prow[4][2 * KP];
  c128 *pr_s = prow[threadIdx.x >> 5];
  bool ok = true;
#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    const c128 ck = m[0];  // M[lane][k]
    const double pr = __shfl_sync(0xffffffffu, ck.re, k);
    const double pi = __shfl_sync(0xffffffffu, ck.im, k);
    if (!(pr > 0.0) || !isfinite(pr) || !isfinite(pi)) {  // warp-uniform
      ok = false;
      break;
    }
    const c128 pinv = cinv(mk<double>(pr, pi));
    // this lane's entry of the scaled pivot row, M[k][lane] / p
    const c128 mk_l = (lane == k) ? mk<double>(pr, pi)
                                  : (lane > k ? cconj(ck) : mk<double>(-ck.re, ck.im));
    if (lane < KP) {
      const c128 v = cmul(mk_l, pinv);
      pr_s[lane] = v;
      pr_s[lane + KP] = v;
    }
    __syncwarp();
    const c128 *prk = pr_s + k + 1;
    // row_i -= c_i r with c_k = p - 1 (so row k becomes r); column k is then
    // -c_i / p (i != k) and 1 / p (i = k), stored in the last slot
    const c128 c = (lane == k) ? mk<double>(ck.re - 1.0, ck.im) : ck;
    const c128 colv = (lane == k) ? pinv : cmul(mk<double>(-ck.re, -ck.im), pinv);
#pragma unroll
    for (int j = 0; j < KP - 1; ++j) {
      const c128 r = prk[j];
      c128 u = m[j + 1];
      u.re = fma(-c.re, r.re, u.re);
      u.re = fma(c.im, r.im, u.re);
      u.im = fma(-c.re, r.im, u.im);
      u.im = fma(-c.im, r.re, u.im);
      m[j] = u;
    }
    m[KP - 1] = colv;
    __syncwarp();
  }
  double fi = 0.0;
#pragma unroll
  for (int j = 0; j < KP; ++j) fi += cabs2(m[j]);
  if (lane >= K) fi = 0.0;
  // padded columns of real rows are exactly zero, identity rows are excluded
  fi = warp_sum(fi);
  const bool good = ok && isfinite(fi) && sqrt(fa) * sqrt(fi) <= limit;
  if (!good) {
    if (lane == 0) redo[item] = 1;
    return;
  }
  // slot j holds column (j + K) mod KP; A^-1[c][lane] = conj(M[lane][c])
  c128 *o = Ainv + item * ais;
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    const int col = (j + K) & (KP - 1);
    if (lane < K && col < K) o[col * K + lane] = cconj(m[j]);
  }
  if (lane == 0) {
    redo[item] = 0;
    if (info) info[item] = LRZ_INFO_OK;
  }
}

}  // namespace lrz

using namespace lrz;

extern "C" int lrz_plan(int64_t n, int K, const uint8_t *is_sketch, const int32_t *k_est,
                        uint8_t *plan, void *stream) {
  if (n < 0 || K < 1 || !is_sketch || !k_est || !plan) {
    lrz_set_error("lrz_plan: bad arguments");
    return LRZ_EINVAL;
  }
  if (n == 0) return LRZ_OK;
  plan_kernel<<<unsigned((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, K, is_sketch,
                                                                          k_est, plan);
  return lrz_launch_status("lrz_plan");
}

size_t lrz_inverse_smem(int K) { return InvSmem::bytes(K, K, K <= INV_SMEM_KMAX); }
size_t lrz_woodbury_smem(int D) { return InvSmem::bytes(D, D, false) + wb_aux_smem(D); }
size_t lrz_chain_smem(int K, int D) {
  return chain_resident(K, D) ? chain_plan(K, D).bytes
                              : InvSmem::bytes(K, D, K <= INV_SMEM_KMAX) + wb_aux_smem(D);
}
size_t lrz_wb_ws(int64_t B, int K, int D) {
  // + per-trial SingularAuxiliary flags of the step-parallel chain
  return size_t(B) * wb_ws_elems(K, D) * sizeof(c128) + 2 * size_t(B);  // + fb[B], act[B]
}
int lrz_zgemm_internal(int64_t batch, int M, int N, int Kd, int opA, const void *A, int64_t lda,
                       int64_t sA, int opB, const void *Bm, int64_t ldb, int64_t sB, void *C,
                       int64_t ldc, int64_t sC, cudaStream_t s);

static int set_smem(const void *fn, size_t bytes) {
  if (bytes > 32 * 1024) {  // static shared memory counts against the 48 KB default too
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) !=
        cudaSuccess) {
      lrz_set_error("cudaFuncSetAttribute(%zu bytes) failed", bytes);
      return LRZ_ELAUNCH;
    }
  }
  return LRZ_OK;
}

int lrz_use_dmma();
size_t lrz_inverse_blocked_ws(int64_t B, int K);
int lrz_inverse_blocked(int64_t B, int K, const void *A, int64_t a_stride, void *A_inv,
                        int64_t ai_stride, int32_t *info, double limit, const uint8_t *mask,
                        uint8_t *redo, void *ws, cudaStream_t s);

// smallest K the blocked DMMA Gauss-Jordan takes (LRZ_INV_BLOCKED_MIN overrides)
static int inv_blocked_min() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LRZ_INV_BLOCKED_MIN");
    v = e ? atoi(e) : INV_SMEM_KMAX;  // K = 64: 7.9 -> 5.9 ms per 12,800 items (C3)
  }
  return v;
}

extern "C" int lrz_herm_inverse(int64_t B, int K, const void *A, int64_t a_stride,
                                void *A_inv, int64_t ai_stride, int32_t *info, double cond_limit,
                                const uint8_t *item_mask, void *workspace, void *stream) {
  if (B < 0 || K < 1 || K > 1024 || !A || !A_inv) {
    lrz_set_error("lrz_herm_inverse: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const size_t sm = lrz_inverse_smem(K);
  if (set_smem((const void *)herm_inverse_kernel, sm)) return LRZ_ELAUNCH;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t *mask = item_mask;
  if (K <= 32 && workspace) {
    // warp-per-matrix fast path; the CTA kernel re-does only flagged items
    uint8_t *redo = (uint8_t *)workspace;
    LrzProf prof("herm_inverse_warp_kernel", st);
    if (K <= 16)
      herm_inverse_warp_kernel<16><<<unsigned((B + 3) / 4), 128, 0, st>>>(
          B, K, (const c128 *)A, a_stride, (c128 *)A_inv, ai_stride, info, cond_limit,
          item_mask, redo);
    else
      herm_inverse_warp_kernel<32><<<unsigned((B + 3) / 4), 128, 0, st>>>(
          B, K, (const c128 *)A, a_stride, (c128 *)A_inv, ai_stride, info, cond_limit,
          item_mask, redo);
    mask = redo;
  } else if (K >= inv_blocked_min() && K <= 256 && K % 32 == 0 && workspace && lrz_use_dmma()) {
    // blocked Gauss-Jordan with the rank-32 updates on DMMA (inverse_blocked.cu);
    // flagged items (non-PD pivots, guard bound exceeded) go to the CTA kernel
    uint8_t *redo = (uint8_t *)workspace;
    void *bws = (char *)workspace + ((size_t(B) + 255) & ~size_t(255));
    if (int rc = lrz_inverse_blocked(B, K, A, a_stride, A_inv, ai_stride, info, cond_limit,
                                     item_mask, redo, bws, st))
      return rc;
    mask = redo;
  } else if (K > INV_SMEM_KMAX && K <= 256 && workspace) {
    // cluster path: the matrix spread over CS CTAs' shared memory
    uint8_t *redo = (uint8_t *)workspace;
    const int CS = K <= 128 ? 2 : 8;
    const int R = (K + CS - 1) / CS;
    // pivot blocks must not straddle two members' rows: bsz divides R
    int bsz = K <= 128 ? 16 : 8;
    while (R % bsz) bsz >>= 1;
    const size_t csm = (size_t(R) * K + 2 * size_t(bsz) * K + size_t(R) * bsz +
                        size_t(bsz) * (bsz + 1)) * sizeof(c128);
    if (cudaFuncSetAttribute(herm_inverse_cluster_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(csm)) != cudaSuccess) {
      lrz_set_error("lrz_herm_inverse: cannot reserve %zu bytes of shared memory", csm);
      return LRZ_ELAUNCH;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(unsigned(B * CS));
    lc.blockDim = dim3(CINV_THREADS);
    lc.dynamicSmemBytes = csm;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    LrzProf prof("herm_inverse_cluster_kernel", st);
    if (cudaLaunchKernelEx(&lc, herm_inverse_cluster_kernel, K, CS, bsz, (const c128 *)A, a_stride,
                           (c128 *)A_inv, ai_stride, info, cond_limit, item_mask, redo) !=
        cudaSuccess)
      return lrz_launch_status("herm_inverse_cluster_kernel");
    mask = redo;
  }
  LrzProf prof("herm_inverse_kernel", st);
  herm_inverse_kernel<<<unsigned(B), INV_THREADS, sm, st>>>(
      K, (const c128 *)A, a_stride, (c128 *)A_inv, ai_stride, info, cond_limit, mask);
  return lrz_launch_status("lrz_herm_inverse");
}

extern "C" int lrz_woodbury(int64_t B, int K, int d_max, const void *A, const void *A_inv,
                            int64_t a_stride, const void *U, const void *V, const double *S,
                            const int32_t *r, void *A_out, void *A_inv_out, int32_t *info,
                            void *workspace, void *stream) {
  if (B < 0 || K < 1 || d_max < 1 || d_max > 256 || !A_inv || !U || !V || !S || !r ||
      !A_inv_out || !info || !workspace || ((A == nullptr) != (A_out == nullptr))) {
    lrz_set_error("lrz_woodbury: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const size_t sm = lrz_woodbury_smem(d_max);
  if (set_smem((const void *)woodbury_kernel, sm)) return LRZ_ELAUNCH;
  woodbury_kernel<<<unsigned(B), INV_THREADS, sm, (cudaStream_t)stream>>>(
      K, d_max, (const c128 *)A, (const c128 *)A_inv, a_stride, (const c128 *)U,
      (const c128 *)V, S, r, (c128 *)A_out, (c128 *)A_inv_out, info, (c128 *)workspace);
  return lrz_launch_status("lrz_woodbury");
}

extern "C" int lrz_chain(int64_t B, int T, int K, int d_max, const uint8_t *plan, const void *G,
                         const void *A_inv_prev, void *A_inv_seq, void *A_state, const void *U,
                         const void *V, const double *S, const int32_t *r, uint8_t *method,
                         int32_t *info, void *workspace, void *stream) {
  if (B < 0 || T < 1 || K < 1 || d_max < 1 || d_max > 256 || !plan || !G || !A_inv_prev ||
      !A_inv_seq || !U || !V || !S || !r || !method || !workspace) {
    lrz_set_error("lrz_chain: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  static int mode = -1;  // LRZ_CHAIN_RESIDENT=0: global-memory chain (A/B switch)
  if (mode < 0) {
    const char *e = getenv("LRZ_CHAIN_RESIDENT");
    mode = (e && e[0] == '0') ? 0 : 1;
    const char *c = getenv("LRZ_CHAIN_CARVEOUT");
    if (c) cudaFuncSetAttribute((const void *)chain_kernel,
                                cudaFuncAttributePreferredSharedMemoryCarveout, atoi(c));
  }
  // resident: 2 = the DMMA step (LRZ_CHAIN_RESIDENT=1 selects the SIMT resident step)
  static int simt = -1;
  if (simt < 0) {
    const char *e = getenv("LRZ_CHAIN_RESIDENT");
    simt = (e && e[0] == '1') ? 1 : 0;
  }
  // (K > 32 is resident only with the DMMA step, which updates A^-1 in place)
  const bool dm = !simt && lrz_use_dmma();
  const int resident =
      (mode && chain_resident(K, d_max) && (K <= 32 || dm)) ? (dm ? 2 : 1) : 0;
  const size_t sm = resident ? lrz_chain_smem(K, d_max)
                             : InvSmem::bytes(K, d_max, K <= INV_SMEM_KMAX) + wb_aux_smem(d_max);
  if (set_smem((const void *)chain_kernel, sm)) return LRZ_ELAUNCH;
  LrzProf prof("chain_kernel", (cudaStream_t)stream);
  chain_kernel<<<unsigned(B), INV_THREADS, sm, (cudaStream_t)stream>>>(
      T, K, d_max, plan, (const c128 *)G, (const c128 *)A_inv_prev, (c128 *)A_inv_seq,
      (c128 *)A_state, (const c128 *)U, (const c128 *)V, S, r, method, info,
      (c128 *)workspace, resident);
  return lrz_launch_status("lrz_chain");
}


int lrz_use_dmma();
int lrz_chain_gemms_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *plan,
                         const void *U, const void *V, const void *prev, int64_t pst,
                         void *AiUt, void *VhAi, void *aux, int64_t ws_stride, cudaStream_t s);
int lrz_chain_T_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *act,
                     const int32_t *r, const void *auxinv, const void *AiUt, void *Tm,
                     int64_t ws_stride, cudaStream_t s);
int lrz_chain_apply_dmma(int64_t B, int T, int t, int K, int D, const uint8_t *act,
                         const void *Tm, const void *VhAi, int64_t ws_stride, const void *prev,
                         int64_t pst, void *Ainv_seq, void *A_state, const void *U,
                         const void *V, const double *S, const int32_t *r, cudaStream_t s);

extern "C" int lrz_chain_steps(int64_t B, int T, int K, int d_max, const uint8_t *plan,
                               const void *G, const void *A_inv_prev, void *A_inv_seq,
                               void *A_state, const void *U, const void *V, const double *S,
                               const int32_t *r, uint8_t *method, int32_t *info, void *workspace,
                               void *stream) {
  if (B < 0 || T < 1 || K < 1 || d_max < 1 || d_max > 256 || !plan || !G || !A_inv_prev ||
      !A_inv_seq || !U || !V || !S || !r || !method || !info || !workspace) {
    lrz_set_error("lrz_chain_steps: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  cudaStream_t st = (cudaStream_t)stream;
  LrzProf prof("chain_steps (all kernels)", st);
  {
    // step-parallel chain: the trials advance together, products batched over them
    c128 *ws = (c128 *)workspace;
    uint8_t *fb = (uint8_t *)(ws + B * wb_ws_elems(K, d_max));
    const int64_t KK = int64_t(K) * K, E = wb_ws_elems(K, d_max);
    const size_t smc = lrz_woodbury_smem(d_max), smf = lrz_inverse_smem(K);
    if (set_smem((const void *)wb_core_kernel, smc) ||
        set_smem((const void *)wb_fallback_kernel, smf))
      return LRZ_ELAUNCH;
    const int nt = (K + WBA_TILE - 1) / WBA_TILE;
    const bool dmma = lrz_use_dmma() != 0;
    for (int t = 0; t < T; ++t) {
      const c128 *prev = t == 0 ? (const c128 *)A_inv_prev : (const c128 *)A_inv_seq + (t - 1) * KK;
      const int64_t pst = t == 0 ? KK : int64_t(T) * KK;
      // AiU^T = U^T (A^-1)^T  (D x K)  and  VhAi = conj(V^T) A^-1  (D x K)
      int rc;
      if (dmma) {
        rc = lrz_chain_gemms_dmma(B, T, t, K, d_max, plan, U, V, prev, pst, ws,
                                  ws + 2 * int64_t(K) * d_max, ws + wb_ws_aux_off(K, d_max), E,
                                  st);
      } else {
        LrzProf p1("chain:gemms", st);
        rc = lrz_zgemm_internal(B, d_max, K, K, 0, (const c128 *)U + t * int64_t(d_max) * K, K,
                                int64_t(T) * d_max * K, 1, prev, K, pst, ws, K, E, st);
        if (!rc)
          rc = lrz_zgemm_internal(B, d_max, K, K, 3, (const c128 *)V + t * int64_t(d_max) * K, K,
                                  int64_t(T) * d_max * K, 0, prev, K, pst,
                                  ws + 2 * int64_t(K) * d_max, K, E, st);
      }
      if (rc) return rc;
      {
        LrzProf p2("chain:wb_core_kernel", st);
        wb_core_kernel<<<unsigned(B), INV_THREADS, smc, st>>>(T, t, K, d_max, plan,
                                                              (const c128 *)V, S, r, ws, fb,
                                                              method, info, dmma ? 1 : 0);
      }
      if (dmma) {
        rc = lrz_chain_T_dmma(B, T, t, K, d_max, fb + B, r, ws + wb_ws_aux_off(K, d_max) +
                              int64_t(d_max) * d_max, ws, ws + int64_t(K) * d_max, E, st);
        if (rc) return rc;
      }
      {
        LrzProf p3("chain:wb_apply_kernel", st);
        wb_apply_kernel<<<unsigned(B * nt * nt), 256, 0, st>>>(
            T, t, K, d_max, plan, (const c128 *)G, prev, pst, (c128 *)A_inv_seq,
            (c128 *)A_state, (const c128 *)U, (const c128 *)V, S, r, ws, fb, method,
            dmma ? 1 : 0);
      }
      if (dmma) {
        rc = lrz_chain_apply_dmma(B, T, t, K, d_max, fb + B, ws + int64_t(K) * d_max,
                                  ws + 2 * int64_t(K) * d_max, E, prev, pst, A_inv_seq, A_state,
                                  U, V, S, r, st);
        if (rc) return rc;
      }
      {
        LrzProf p4("chain:wb_fallback_kernel", st);
        wb_fallback_kernel<<<unsigned(B), INV_THREADS, smf, st>>>(T, t, K, plan,
                                                                  (const c128 *)G,
                                                                  (c128 *)A_inv_seq, fb, method,
                                                                  info);
      }
      if (int rc2 = lrz_launch_status("lrz_chain (step-parallel)")) return rc2;
    }
    return LRZ_OK;
  }
}

extern "C" int lrz_spec_verify(int64_t B, int T, int K, const lrz_arsvd_cfg *cfg,
                               const uint8_t *is_sketch, int32_t *iters_pred,
                               const int32_t *iters_act, int64_t *cursor, const int64_t *cursor0,
                               int32_t *first_unverified, uint8_t *active, int32_t *pending,
                               void *stream) {
  return lrz_spec_verify_vote(B, T, K, cfg, is_sketch, iters_pred, iters_act, cursor, cursor0,
                              first_unverified, active, pending, nullptr, stream);
}

extern "C" int lrz_spec_verify_vote(int64_t B, int T, int K, const lrz_arsvd_cfg *cfg,
                                    const uint8_t *is_sketch, int32_t *iters_pred,
                                    const int32_t *iters_act, int64_t *cursor,
                                    const int64_t *cursor0, int32_t *first_unverified,
                                    uint8_t *active, int32_t *pending, uint8_t *votes,
                                    void *stream) {
  if (B < 0 || T < 1 || K < 1 || !cfg || !is_sketch || !iters_pred || !cursor ||
      !cursor0 || !first_unverified || !active || !pending || cfg->i_max > 30 ||
      (votes && cfg->i_max >= LRZ_SPEC_VOTE_W)) {
    lrz_set_error("lrz_spec_verify: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  ConsumedTab tab;
  tab.v[0] = 0;
  long long k0 = cfg->k_init;
  for (int i = 0; i < cfg->i_max; ++i) {
    const int d = (int)std::min<long long>(k0 + cfg->p, K);
    tab.v[i + 1] = tab.v[i] + 2LL * K * d;
    k0 *= 2;
  }
  const unsigned nb = unsigned((B + 3) / 4);  // one warp per trial
  spec_verify_kernel<<<nb, 128, 0, (cudaStream_t)stream>>>(B, T, K, tab, is_sketch, iters_pred,
                                                           iters_act, cursor, cursor0,
                                                           first_unverified, active, pending,
                                                           votes);
  return lrz_launch_status("lrz_spec_verify");
}
