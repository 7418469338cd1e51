// complex64 precoder W = H^H A^-1 (precoding.py:47) on the 5th-generation
// tensor cores: tcgen05.mma kind::tf32 with a 3xTF32 split, TMA-staged tiles,
// the accumulator in tensor memory (TMEM), for K > 32 (C3-C5 complex64).
//
// Real form.  With q = 2k + c (c = re / im of H[k][n]) and p = 2j + e:
//   D[n][p] = sum_q Aop[n][q] Bop[p][q],   Aop[n][2k + c] = (Hr, Hi)[k][n],
//   Bop[2j][2k] = Ar, Bop[2j][2k+1] = Ai, Bop[2j+1][2k] = Ai, Bop[2j+1][2k+1] = -Ar
// (A = A^-1[k][j]), so D[n][2j] + i D[n][2j+1] = sum_k conj(H[k][n]) A[k][j] =
// W[n][j]: the accumulator rows are W's rows, interleaved complex.
//
// 3xTF32: every operand is split x = hi + lo with hi = x truncated to TF32
// (exactly representable, so the tensor core's own TF32 conversion is a no-op)
// and lo = x - hi (exact in fp32); D += hi_a hi_b + hi_a lo_b + lo_a hi_b, fp32
// accumulation in TMEM: ~2^-21 relative per product, well inside the 1e-4
// complex64 tolerance (plain TF32 would be ~5e-4).
//
// Per CTA: one item x one 128-row tile of n; the reduction (2K floats) is
// streamed in chunks of 16 floats (8 complex k) through an S-stage ring:
//   warp 0   TMA producer: the raw H slab (8 rows x 256 floats, 2-D tensor
//            map) and the pre-split Bop chunk (hi and lo, 2K rows x 16 floats,
//            already in the UMMA canonical K-major layout in global memory:
//            one 2-D TMA each)
//   warps 2-5 convert the raw H slab into Aop hi / lo (transpose + split) in
//            the canonical layout, fence.proxy.async, arrive
//   warp 1   (one elected lane) issues 6 or 12 tcgen05.mma per chunk
//            (2 k-steps x N-halves x 3 split products) and tcgen05.commit's the
//            stage back to the producer; a final commit signals the epilogue
//   warps 2-5 epilogue: tcgen05.ld 32x32b rows of D -> W (complex64) rows,
//            ||W||_F^2 of the stored values as one partial per CTA.
// Canonical K-major SWIZZLE_NONE layout of a (rows x 16 floats) tile: 8-row x
// 16-byte core matrices, address(r, q) = (r/8)*512 + (q/4)*128 + (r%8)*16 +
// (q%4)*4 (LBO = 128 B between the two k core matrices of an instruction,
// SBO = 512 B between 8-row groups).

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"

namespace lrz {

constexpr int TC_M = 128;           // rows of n per CTA (UMMA M)
constexpr int TC_QC = 16;           // reduction floats per chunk
constexpr int TC_THREADS = 192;     // 6 warps

LRZ_DEV uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

LRZ_DEV void mbar_init(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(cnt));
}
LRZ_DEV void mbar_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(tx)
               : "memory");
}
LRZ_DEV void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
LRZ_DEV void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LAB_WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
LRZ_DEV void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
LRZ_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
LRZ_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
LRZ_DEV void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
LRZ_DEV void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   su32(bar))
               : "memory");
}
// smem matrix descriptor: canonical K-major, no swizzle, LBO 128 B, SBO 512 B
LRZ_DEV uint64_t sdesc(const void *p) {
  const uint32_t a = su32(p);
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(512 >> 4) << 32) |
         (uint64_t(1) << 46);
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t tc_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
}
LRZ_DEV float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// accumulator columns per CTA: all 2K when 2K <= 256, else one 256-column half
// (two CTAs per n-tile, so TMEM (512 columns) and shared memory hold two CTAs
// per SM and one CTA's epilogue overlaps the other's MMAs)
__host__ __device__ inline int tc_pc(int K) { return 2 * K < 256 ? 2 * K : 256; }
__host__ __device__ inline int tc_halves(int K) { return 2 * K > 256 ? 2 : 1; }

template <int S>
struct TcSmem {
  // per stage: raw H slab (8 x 256 floats), Aop hi / lo (128 x 16), Bop hi / lo (Pc x 16)
  static constexpr size_t raw = 8 * 256 * 4, aop = TC_M * TC_QC * 4;
  __host__ __device__ static size_t bop(int K) { return size_t(tc_pc(K)) * TC_QC * 4; }
  __host__ __device__ static size_t stage(int K) { return raw + 2 * aop + 2 * bop(K); }
  __host__ __device__ static size_t bytes(int K) { return 128 + S * stage(K) + 256; }
};

// Bop (hi, lo) of every item in the canonical chunk order: chunk c (q in
// [16c, 16c + 16)) of item b is a contiguous 2K x 16-float tile at row
// ((b * nch + c) * K) of a [rows][32 floats] view; lo follows hi after B * nch * K rows.
__global__ void tc_bop_kernel(int64_t B, int K, const c128 *__restrict__ Ainv, int64_t ais,
                              float *__restrict__ bop) {
  const int nch = (2 * K) / TC_QC;
  const int64_t tile = int64_t(2 * K) * TC_QC;  // floats per chunk tile
  const int64_t per_item = tile * nch, total = B * per_item;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / per_item;
    const int64_t r = e - b * per_item;
    const int c = int(r / tile);
    const int w = int(r - int64_t(c) * tile);  // offset inside the canonical tile
    // invert address(p, q4) = (p/8)*128 + (q4/4)*32 + (p%8)*4 + q4%4  (in floats)
    const int g8 = w >> 7, rem = w & 127, qs = rem >> 5, pr = (rem >> 2) & 7, q4 = rem & 3;
    const int p = g8 * 8 + pr, q = c * TC_QC + qs * 4 + q4;
    const int j = p >> 1, e_ = p & 1, k = q >> 1, cc = q & 1;
    const c128 a = Ainv[b * ais + int64_t(k) * K + j];
    const double v = e_ == 0 ? (cc == 0 ? a.re : a.im) : (cc == 0 ? a.im : -a.re);
    const float x = float(v);
    const float hi = tf32_hi(x);
    bop[e] = hi;
    bop[total + e] = x - hi;
  }
}

template <int S>
__global__ void __launch_bounds__(TC_THREADS, 2)
    tc_w_kernel(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_b,
                int K, int N, int64_t B, c64 *__restrict__ W, double *__restrict__ parts) {
  extern __shared__ __align__(128) unsigned char tc_smem_raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 127) & ~uintptr_t(127));
  using L = TcSmem<S>;
  const size_t stage = L::stage(K);
  const size_t bop_b = L::bop(K);
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + S * stage);
  uint64_t *full_tma = bars, *full_cv = bars + S, *empty = bars + 2 * S, *tmem_full = bars + 3 * S;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 3 * S + 1);
  float *red = reinterpret_cast<float *>(bars + 3 * S + 2);  // 4 doubles as 8 floats

  const int halves = tc_halves(K);
  const int tiles = (N / TC_M) * halves;
  const int64_t item = blockIdx.x / tiles;
  const int tl = int(blockIdx.x - item * tiles);
  const int n0 = (tl / halves) * TC_M, half = tl % halves;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (2 * K) / TC_QC;
  const int P = tc_pc(K);                    // accumulator columns of this CTA
  const int NI = P;                          // UMMA N per instruction
  const uint32_t tcols = P <= 32 ? 32u : P <= 64 ? 64u : P <= 128 ? 128u : 256u;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_tma[s], 1);
      mbar_init(&full_cv[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const int64_t hrow = item * K;
      // this CTA's half of each Bop chunk tile: rows of 128 B from half * P / 2
      const int64_t brow_hi = item * nch * int64_t(K) + half * (P / 2);
      const int64_t brow_lo = B * nch * int64_t(K) + brow_hi;
      const uint32_t tx = uint32_t(L::raw + 2 * bop_b);
      for (int c = 0; c < nch; ++c) {
        const int s = c % S;
        if (c >= S) mbar_wait(&empty[s], ((c / S) & 1) ^ 1);
        unsigned char *st = sm + s * stage;
        mbar_expect_tx(&full_tma[s], tx);
        tma_load_2d(st, &map_h, &full_tma[s], 2 * n0, int(hrow + 8 * c));
        unsigned char *bh = st + L::raw + 2 * L::aop;
        tma_load_2d(bh, &map_b, &full_tma[s], 0, int(brow_hi + int64_t(c) * K));
        tma_load_2d(bh + bop_b, &map_b, &full_tma[s], 0, int(brow_lo + int64_t(c) * K));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = tc_idesc(NI);
    for (int c = 0; c < nch; ++c) {
      const int s = c % S;
      mbar_wait(&full_cv[s], (c / S) & 1);
      tc_fence_after();
      if (lane == 0) {
        unsigned char *st = sm + s * stage;
        const unsigned char *ahi = st + L::raw, *alo = ahi + L::aop;
        const unsigned char *bhi = st + L::raw + 2 * L::aop, *blo = bhi + bop_b;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ah = sdesc(ahi + 256 * ks), al = sdesc(alo + 256 * ks);
          const uint64_t bh = sdesc(bhi + 256 * ks), bl = sdesc(blo + 256 * ks);
          tc_mma(tmem, ah, bh, idesc, (c > 0 || ks > 0) ? 1u : 0u);
          tc_mma(tmem, ah, bl, idesc, 1u);
          tc_mma(tmem, al, bh, idesc, 1u);
        }
        tc_commit(&empty[s]);
        if (c == nch - 1) tc_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- converters (warps 2-5), then the epilogue
    const int t = threadIdx.x - 64;  // 0..127 = row n of the tile
    for (int c = 0; c < nch; ++c) {
      const int s = c % S;
      mbar_wait(&full_tma[s], (c / S) & 1);
      unsigned char *st = sm + s * stage;
      const float *raw = reinterpret_cast<const float *>(st);
      float *ahi = reinterpret_cast<float *>(st + L::raw);
      float *alo = reinterpret_cast<float *>(st + L::raw + L::aop);
#pragma unroll
      for (int sc = 0; sc < 4; ++sc) {
        // q = 4 sc .. 4 sc + 3: (Hr, Hi) of rows k = 2 sc, 2 sc + 1 of the slab
        const float2 u = *reinterpret_cast<const float2 *>(raw + (2 * sc) * 256 + 2 * t);
        const float2 v = *reinterpret_cast<const float2 *>(raw + (2 * sc + 1) * 256 + 2 * t);
        float4 x = make_float4(u.x, u.y, v.x, v.y);
        float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
        float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        const int off = (t >> 3) * 128 + sc * 32 + (t & 7) * 4;  // floats
        *reinterpret_cast<float4 *>(ahi + off) = h;
        *reinterpret_cast<float4 *>(alo + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_cv[s]);
    }
    // ---------------- epilogue: row (32 (warp % 4) + lane) of D -> W
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int q4 = warp & 3;
    const int row = 32 * q4 + lane;
    const int n = n0 + row;
    c64 *wrow = W + (item * int64_t(N) + n) * K + half * 128;  // 256 real = 128 complex columns
    double nrm = 0.0;
    for (int col = 0; col < P; col += 32) {
      uint32_t r[32];
      const uint32_t taddr = tmem + (uint32_t(32 * q4) << 16) + uint32_t(col);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
            "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
            "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
            "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
            "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      float4 *dst = reinterpret_cast<float4 *>(wrow + col / 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                     __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        nrm += double(v.x) * v.x + double(v.y) * v.y + double(v.z) * v.z + double(v.w) * v.w;
        if (n < N) dst[i] = v;
      }
    }
    if (n >= N) nrm = 0.0;
    nrm = warp_sum(nrm);
    double *redd = reinterpret_cast<double *>(red);
    if (lane == 0) redd[q4] = nrm;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols));
  }
  if (threadIdx.x == 0 && parts) {
    const double *redd = reinterpret_cast<const double *>(red);
    parts[blockIdx.x] = ((redd[0] + redd[1]) + redd[2]) + redd[3];
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static int make_map_2d(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows,
                       uint64_t row_bytes, uint32_t box_c, uint32_t box_r) {
  auto fn = encode_fn();
  if (!fn) {
    lrz_set_error("cuTensorMapEncodeTiled is unavailable");
    return LRZ_ELAUNCH;
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_c, box_r};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    lrz_set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
    return LRZ_ELAUNCH;
  }
  return LRZ_OK;
}

template <int S>
static int tc_w_launch(const CUtensorMap &mh, const CUtensorMap &mb, int K, int N, int64_t B,
                       c64 *W, double *parts, cudaStream_t s) {
  const size_t sm = TcSmem<S>::bytes(K);
  static size_t reserved = 0;  // largest dynamic shared memory set so far (K-dependent)
  if (sm > reserved) {
    if (cudaFuncSetAttribute(tc_w_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sm)) != cudaSuccess) {
      lrz_set_error("tc_w_kernel: cannot reserve %zu bytes of shared memory", sm);
      return LRZ_ELAUNCH;
    }
    reserved = sm;
  }
  const int64_t grid = B * (N / TC_M) * tc_halves(K);
  tc_w_kernel<S><<<unsigned(grid), TC_THREADS, sm, s>>>(mh, mb, K, N, B, W, parts);
  return lrz_launch_status("tc_w_kernel");
}

}  // namespace lrz

using namespace lrz;

// Whether the tcgen05 path takes a complex64 precoder of this shape.
int lrz_tc_w_ok(int K, int N, int64_t h_stride) {
  return K >= 32 && K <= 256 && K % 8 == 0 && N % TC_M == 0 && h_stride == int64_t(K) * N;
}
// norm partials per item (one per CTA: 128-row tile x column half)
int lrz_tc_w_tiles(int N, int K) { return (N / TC_M) * tc_halves(K); }
// workspace: the pre-split Bop of every item
size_t lrz_tc_w_ws(int64_t B, int K) { return size_t(B) * 2 * (2 * K) * (2 * K) * sizeof(float); }

// W[b] = H[b]^H A_inv[b] (complex64 out), ||W||^2 partials per 128-row tile.
int lrz_tc_precoder_w(int64_t B, int K, int N, const void *H, const void *A_inv, int64_t ais,
                      void *W, double *parts, void *ws, cudaStream_t s) {
  float *bop = (float *)ws;
  {
    LrzProf prof("tc_bop_kernel", s);
    const int64_t tot = B * (2 * K) * int64_t(2 * K);
    const unsigned nb = unsigned(std::min<int64_t>((tot + 255) / 256, 148 * 16));
    tc_bop_kernel<<<nb, 256, 0, s>>>(B, K, (const c128 *)A_inv, ais, bop);
    if (int rc = lrz_launch_status("tc_bop_kernel")) return rc;
  }
  CUtensorMap mh, mb;
  if (int rc = make_map_2d(&mh, H, uint64_t(2) * N, uint64_t(B) * K, uint64_t(N) * 8, 256, 8))
    return rc;
  const uint64_t brows = uint64_t(B) * 2 * ((2 * K) / TC_QC) * K;
  if (int rc = make_map_2d(&mb, bop, 32, brows, 128, 32, uint32_t(tc_pc(K) / 2))) return rc;
  LrzProf prof("tc_w_kernel", s);
  return tc_w_launch<2>(mh, mb, K, N, B, (c64 *)W, parts, s);
}
