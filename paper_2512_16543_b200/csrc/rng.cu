// Device-side sketch streams, bit-exact with numpy's Generator(PCG64).standard_normal.
//
// The reference draws every Omega from a per-(method, trial) numpy Generator
// (lowrank.py:284-286, harness.py:88-92,206-211).  Producing those normals on
// the host costs more than the whole GPU step at C2 and their upload is 16 %
// of the end-to-end bytes, so the GPU reproduces them itself:
//   * PCG64 (128-bit LCG, XSL-RR output) with O(log n) jump-ahead;
//   * numpy's ziggurat for standard normals over numpy's own tables (read from
//     the installed numpy at build time, see rng/tables.py).
// A normal consumes one raw draw 99.3 % of the time and more on the rejection
// and tail paths, so normal n's raw position is data dependent.  Three passes:
//   A  one thread per 256-draw segment: step PCG, record per raw position the
//      draws a normal starting there consumes (c_j); follow the walk that
//      starts at the segment's first draw ("walk 0") and store its normals
//      compacted by rank, with their positions; summarise the walks entering
//      at offsets 0..7 (almost every walk merges into walk 0 within a draw);
//   B  one thread per trial: chain the segment summaries to get each
//      segment's entry offset and the index of its first normal;
//   C  one thread per segment: copy walk 0's normals from the entry's rank on
//      to the output (independent loads); positions off walk 0 (rare) are
//      recomputed from the PCG state.
// lrz_rng_locate turns "normals consumed" into the raw draw offset afterwards,
// so no per-normal position array is written.

#include "common.cuh"
#include "_gen/ziggurat_tables.h"
#include "glibc_log1p.h"

namespace lrz {

typedef unsigned __int128 u128;
constexpr int RNG_SEG = 256;
constexpr int RNG_MAXC = 64;  // a normal consuming more draws aborts the window (never seen)
constexpr int RNG_NE = 8;     // entry offsets summarised per segment by pass A
constexpr int RNG_A_THREADS = 128;
LRZ_DEV u128 pcg_mult() {
  return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
}

LRZ_DEV u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

LRZ_DEV uint64_t pcg_next(u128 &st, u128 inc) {
  st = st * pcg_mult() + inc;
  const uint64_t hi = uint64_t(st >> 64), lo = uint64_t(st);
  const unsigned r = unsigned(st >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> r) | (x << ((64u - r) & 63u));
}

LRZ_DEV double pcg_double(u128 &st, u128 inc) {
  return double(pcg_next(st, inc) >> 11) * (1.0 / 9007199254740992.0);
}

struct ZigTables {
  const double *wi, *fi;
  const uint64_t *ki;
};

// numpy's random_standard_normal given its first raw draw r0 (already taken
// from the stream); further draws come from `st`.  Returns the value and the
// number of raw draws consumed.  Tables in shared memory (lanes index them
// divergently, which would serialise on the constant cache).
LRZ_DEV double zig_from(uint64_t r, u128 st, u128 inc, const ZigTables &t, int &used) {
  used = 1;
  for (;;) {
    const int idx = int(r & 0xff);
    r >>= 8;
    const int sign = int(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = double(rabs) * t.wi[idx];
    if (sign) x = -x;
    if (rabs < t.ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-0.27366123732975828, glibc_log1p(-pcg_double(st, inc)));
        const double yy = -glibc_log1p(-pcg_double(st, inc));
        used += 2;
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(3.6541528853610088 + xx) : 3.6541528853610088 + xx;
        if (used > RNG_MAXC) return 0.0;
      }
    } else {
      const double u = pcg_double(st, inc);
      ++used;
      // numpy's baseline build does not contract this (no FMA): unfused here too.
      // exp: CUDA's and glibc's agree to 1 ulp, so the decision can differ only
      // if the left side falls between the two (p ~ 2^-52 per wedge test)
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(t.fi[idx - 1], t.fi[idx]), u), t.fi[idx]);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
    if (used > RNG_MAXC) return 0.0;
    r = pcg_next(st, inc);
    ++used;
  }
}

struct RngArgs {
  int64_t B;
  int nseg;              // segments per trial
  const uint64_t *st;    // [B][2] lo, hi of the PCG state at raw position 0 of the stream
  const uint64_t *inc;   // [B][2]
  const int64_t *raw0;   // [B] raw position where the window starts
  uint8_t *cons;         // [B][SEG][nseg] draws consumed by a normal starting here
  double *vals0;         // [B][SEG][nseg] walk-0 normals by rank
  uint8_t *pos0;         // [B][SEG][nseg] walk-0 positions by rank
  uint32_t *vis;         // [B][nseg][SEG/32] walk-0 position bitmap
  int32_t *seg_cnt0;     // [B][nseg][RNG_NE] normals in the segment for entry offset e
  int32_t *seg_exit0;    // [B][nseg][RNG_NE] overhang into the next segment for entry e
  int32_t *seg_entry;    // [B][nseg] true entry offset
  int64_t *seg_base;     // [B][nseg] stream index of the segment's first normal
  double *out;           // [B][L]
  int64_t L;
  int32_t *startpos;     // [B][L] raw position (relative to raw0) of each normal
  int32_t *status;       // [B] 0 ok, 1 window too short / overlong normal
};

LRZ_DEV u128 load_u128(const uint64_t *p) { return (u128(p[1]) << 64) | u128(p[0]); }

// per-position arrays are stored [b][j][s] (j = position in segment, s =
// segment) so that a warp of consecutive segments stores contiguously
LRZ_DEV int64_t pos_index(const RngArgs &a, int64_t b, int j, int s) {
  return (b * RNG_SEG + j) * a.nseg + s;
}

__global__ void __launch_bounds__(RNG_A_THREADS) rng_pass_a(RngArgs a) {
  __shared__ double s_wi[256], s_fi[256];
  __shared__ uint64_t s_ki[256];
  __shared__ uint8_t s_c[RNG_A_THREADS][RNG_SEG + 4];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_wi[i] = zig_wi_double[i];
    s_fi[i] = zig_fi_double[i];
    s_ki[i] = zig_ki_double[i];
  }
  __syncthreads();
  const ZigTables tb{s_wi, s_fi, s_ki};
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (tid >= a.B * a.nseg) return;
  const int64_t b = tid / a.nseg;
  const int s = int(tid - b * a.nseg);
  uint8_t *c = s_c[threadIdx.x];
  const u128 inc = load_u128(a.inc + 2 * b);
  u128 st = pcg_advance(load_u128(a.st + 2 * b), inc,
                        uint64_t(a.raw0[b]) + uint64_t(s) * RNG_SEG);
  int over = 0, next0 = 0, cnt0 = 0;
  const int64_t col = pos_index(a, b, 0, s), stride = a.nseg;  // [b][j][s]: j advances by nseg
  uint8_t *pc = a.cons + col, *pp = a.pos0 + col;
  double *pv = a.vals0 + col;
  for (int j = 0; j < RNG_SEG; ++j) {
    const uint64_t r = pcg_next(st, inc);  // raw draw j; st now before draw j + 1
    int used;
    const double x = zig_from(r, st, inc, tb, used);
    if (used > RNG_MAXC) over = 1;
    const uint8_t cu = uint8_t(used > 255 ? 255 : used);
    c[j] = cu;
    pc[int64_t(j) * stride] = cu;
    if (j == next0) {  // walk 0 emits a normal here
      pv[int64_t(cnt0) * stride] = x;
      pp[int64_t(cnt0) * stride] = uint8_t(j);
      ++cnt0;
      next0 = j + cu;
    }
  }
  // walk(0) visited mask, then entries 1..RNG_NE-1 merge into it
  uint32_t vis[RNG_SEG / 32];
#pragma unroll
  for (int i = 0; i < RNG_SEG / 32; ++i) vis[i] = 0;
  int pos = 0;
  while (pos < RNG_SEG) {
    vis[pos >> 5] |= 1u << (pos & 31);
    pos += c[pos];
  }
  const int exit0 = pos - RNG_SEG;
#pragma unroll
  for (int i = 0; i < RNG_SEG / 32; ++i) a.vis[tid * (RNG_SEG / 32) + i] = vis[i];
  int32_t *oc = a.seg_cnt0 + tid * RNG_NE, *oe = a.seg_exit0 + tid * RNG_NE;
  oc[0] = cnt0;
  oe[0] = over ? (1 << 20) : exit0;
  for (int e = 1; e < RNG_NE; ++e) {
    int p = e, k = 0;
    while (p < RNG_SEG && !((vis[p >> 5] >> (p & 31)) & 1u)) {
      ++k;
      p += c[p];
    }
    if (p >= RNG_SEG) {
      oc[e] = k;
      oe[e] = over ? (1 << 20) : p - RNG_SEG;
    } else {  // merged into walk(0) at p: the rest of walk(0) from p on
      int before = 0;
      for (int i = 0; i < (p >> 5); ++i) before += __popc(vis[i]);
      before += __popc(vis[p >> 5] & ((1u << (p & 31)) - 1u));
      oc[e] = k + (cnt0 - before);
      oe[e] = over ? (1 << 20) : exit0;
    }
  }
}

// Pass B: segment s maps an entry offset e < RNG_NE to (exit offset, normals
// emitted) -- pass A's summaries.  These maps compose associatively, so a CTA
// per trial scans them in parallel (per-thread runs of segments, then a
// Hillis-Steele scan of the run maps).  An exit >= RNG_NE (a normal
// overhanging the next segment by >= RNG_NE draws, ~1e-6 per segment) or an
// overlong normal sends the trial through the sequential walk instead.
constexpr int RNG_B_THREADS = 512;
constexpr uint8_t RNG_BIG = 255;

struct SegMap {
  uint8_t ex[RNG_NE];
  int32_t cn[RNG_NE];
};

LRZ_DEV SegMap map_identity() {
  SegMap m;
#pragma unroll
  for (int e = 0; e < RNG_NE; ++e) {
    m.ex[e] = uint8_t(e);
    m.cn[e] = 0;
  }
  return m;
}

// g after f
LRZ_DEV SegMap map_then(const SegMap &f, const SegMap &g) {
  SegMap m;
#pragma unroll
  for (int e = 0; e < RNG_NE; ++e) {
    const uint8_t x = f.ex[e];
    if (x == RNG_BIG) {
      m.ex[e] = RNG_BIG;
      m.cn[e] = 0;
    } else {
      m.ex[e] = g.ex[x];
      m.cn[e] = f.cn[e] + g.cn[x];
    }
  }
  return m;
}

LRZ_DEV SegMap seg_map(const RngArgs &a, int64_t id) {
  SegMap m;
#pragma unroll
  for (int e = 0; e < RNG_NE; ++e) {
    const int ex = a.seg_exit0[id * RNG_NE + e];
    m.ex[e] = (ex >= 0 && ex < RNG_NE) ? uint8_t(ex) : RNG_BIG;
    m.cn[e] = a.seg_cnt0[id * RNG_NE + e];
  }
  return m;
}

// the original sequential walk (fallback)
LRZ_DEV void pass_b_serial(const RngArgs &a, int64_t b) {
  int entry = 0, bad = 0;
  long long base = 0;
  for (int s = 0; s < a.nseg; ++s) {
    const int64_t id = b * a.nseg + s;
    a.seg_entry[id] = entry;
    a.seg_base[id] = base;
    if (entry < RNG_NE) {
      const int ex = a.seg_exit0[id * RNG_NE + entry];
      if (ex >= (1 << 20)) bad = 1;
      base += a.seg_cnt0[id * RNG_NE + entry];
      entry = ex >= (1 << 20) ? 0 : ex;
    } else if (entry >= RNG_SEG) {
      entry -= RNG_SEG;
    } else {  // re-walk from the draw counts
      int pos = entry, cnt = 0;
      while (pos < RNG_SEG) {
        const int cp = a.cons[pos_index(a, b, pos, s)];
        if (cp >= 255) bad = 1;
        ++cnt;
        pos += cp;
      }
      base += cnt;
      entry = pos - RNG_SEG;
    }
  }
  a.status[b] = (bad || base < a.L) ? 1 : 0;
}

__global__ void __launch_bounds__(RNG_B_THREADS) rng_pass_b(RngArgs a) {
  __shared__ SegMap s_map[RNG_B_THREADS];
  __shared__ int s_fallback;
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  const int per = (a.nseg + RNG_B_THREADS - 1) / RNG_B_THREADS;
  const int s0 = min(a.nseg, t * per), s1 = min(a.nseg, s0 + per);
  if (t == 0) s_fallback = 0;
  SegMap run = map_identity();
  for (int s = s0; s < s1; ++s) run = map_then(run, seg_map(a, b * a.nseg + s));
  s_map[t] = run;
  __syncthreads();
  // inclusive Hillis-Steele scan: s_map[t] = run_0 then ... then run_t
  for (int off = 1; off < RNG_B_THREADS; off <<= 1) {
    SegMap left;
    const bool has = t >= off;
    if (has) left = s_map[t - off];
    __syncthreads();
    if (has) s_map[t] = map_then(left, s_map[t]);
    __syncthreads();
  }
  // entry state at this thread's first segment: the scan up to the previous run
  int entry = 0;
  long long base = 0;
  if (t > 0) {
    const SegMap &p = s_map[t - 1];
    if (p.ex[0] == RNG_BIG) {
      s_fallback = 1;
    } else {
      entry = p.ex[0];
      base = p.cn[0];
    }
  }
  for (int s = s0; s < s1; ++s) {
    const int64_t id = b * a.nseg + s;
    a.seg_entry[id] = entry;
    a.seg_base[id] = base;
    const int ex = a.seg_exit0[id * RNG_NE + entry];
    base += a.seg_cnt0[id * RNG_NE + entry];
    if (ex < 0 || ex >= RNG_NE) {  // includes the overlong-normal marker
      if (s + 1 < a.nseg || ex >= (1 << 20)) s_fallback = 1;
      entry = 0;
    } else {
      entry = ex;
    }
  }
  __syncthreads();
  if (s_fallback) {
    if (t == 0) pass_b_serial(a, b);
    return;
  }
  if (t == RNG_B_THREADS - 1) a.status[b] = (base < a.L) ? 1 : 0;
}

constexpr int RNG_C_THREADS = 128;

// rank of position p in walk 0 (number of walk-0 positions before p)
LRZ_DEV int walk0_rank(const uint32_t *vis, int p) {
  int r = 0;
  for (int i = 0; i < (p >> 5); ++i) r += __popc(vis[i]);
  return r + __popc(vis[p >> 5] & ((1u << (p & 31)) - 1u));
}

// the normal starting at raw position `pos` of segment s (off walk 0: rare)
LRZ_DEV double normal_at(const RngArgs &a, int64_t b, int s, int pos, const ZigTables &tb) {
  const u128 inc = load_u128(a.inc + 2 * b);
  u128 st = pcg_advance(load_u128(a.st + 2 * b), inc,
                        uint64_t(a.raw0[b]) + uint64_t(s) * RNG_SEG + uint64_t(pos));
  const uint64_t r = pcg_next(st, inc);
  int used;
  return zig_from(r, st, inc, tb, used);
}

__global__ void __launch_bounds__(RNG_C_THREADS) rng_pass_c(RngArgs a) {
  __shared__ double s_wi[256], s_fi[256];
  __shared__ uint64_t s_ki[256];
  __shared__ double s_v[RNG_C_THREADS][33];
  __shared__ int s_m[RNG_C_THREADS];
  __shared__ int64_t s_n[RNG_C_THREADS];
  __shared__ double *s_o[RNG_C_THREADS];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_wi[i] = zig_wi_double[i];
    s_fi[i] = zig_fi_double[i];
    s_ki[i] = zig_ki_double[i];
  }
  __syncthreads();
  const ZigTables tb{s_wi, s_fi, s_ki};
  const int64_t tid0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool live = tid0 < a.B * a.nseg;
  const int64_t tid = live ? tid0 : 0;
  const int64_t b = tid / a.nseg;
  const int s = int(tid - b * a.nseg);
  int pos = live ? a.seg_entry[tid] : RNG_SEG;
  int64_t n = a.seg_base[tid];
  double *o = a.out + b * a.L;
  uint32_t vis[RNG_SEG / 32];
#pragma unroll
  for (int i = 0; i < RNG_SEG / 32; ++i) vis[i] = a.vis[tid * (RNG_SEG / 32) + i];
  // off walk 0: step the entry's own walk until it joins walk 0
  while (pos < RNG_SEG && n < a.L && !((vis[pos >> 5] >> (pos & 31)) & 1u)) {
    o[n++] = normal_at(a, b, s, pos, tb);
    pos += a.cons[pos_index(a, b, pos, s)];
  }
  // on walk 0 from rank r0: every later walk-0 normal of the segment, in order;
  // copied through shared memory in 32-normal chunks so that each warp writes
  // one segment's 32 consecutive outputs per store (coalesced)
  int r0 = 0, m = 0;
  if (pos < RNG_SEG && n < a.L) {
    r0 = walk0_rank(vis, pos);
    int cnt0 = 0;
#pragma unroll
    for (int i = 0; i < RNG_SEG / 32; ++i) cnt0 += __popc(vis[i]);
    m = int(min(int64_t(cnt0 - r0), a.L - n));
  }
  s_m[threadIdx.x] = m;
  s_n[threadIdx.x] = n;
  s_o[threadIdx.x] = o;
  int mmax = m;
  mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, 16));
  mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, 8));
  mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, 4));
  mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, 2));
  mmax = max(mmax, __shfl_xor_sync(0xffffffffu, mmax, 1));
  const int lane = threadIdx.x & 31, wb = threadIdx.x & ~31;
  const double *src = a.vals0 + pos_index(a, b, r0, s);
  for (int k0 = 0; k0 < mmax; k0 += 32) {   // warp-uniform bound (shfl max)
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk)
      if (k0 + kk < m) s_v[threadIdx.x][kk] = src[int64_t(k0 + kk) * a.nseg];
    __syncwarp();
    for (int u = 0; u < 32; ++u) {            // the warp writes thread u's chunk
      const int mu = s_m[wb + u];
      if (k0 + lane < mu) s_o[wb + u][s_n[wb + u] + k0 + lane] = s_v[wb + u][lane];
    }
    __syncwarp();
  }
}

// raw draws consumed by the first consumed[b] normals of the last window
__global__ void rng_locate_kernel(RngArgs a, const int64_t *__restrict__ consumed,
                                  int64_t *__restrict__ raw_adv) {
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= a.B) return;
  const int64_t c = consumed[b];
  // last segment whose first normal index is <= c
  int lo = 0, hi = a.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.seg_base[b * a.nseg + mid] <= c) lo = mid; else hi = mid - 1;
  }
  const int s = lo;
  const int64_t id = b * a.nseg + s;
  int pos = a.seg_entry[id];
  int64_t n = a.seg_base[id];
  const uint32_t *vis = a.vis + id * (RNG_SEG / 32);
  while (n < c && pos < RNG_SEG) {
    if ((vis[pos >> 5] >> (pos & 31)) & 1u) {  // on walk 0: jump by rank
      const int r = walk0_rank(vis, pos) + int(c - n);
      int cnt0 = 0;
      for (int i = 0; i < RNG_SEG / 32; ++i) cnt0 += __popc(vis[i]);
      if (r < cnt0) {
        pos = a.pos0[pos_index(a, b, r, s)];
        n = c;
      } else {  // past the segment's last normal: its exit
        n += cnt0 - walk0_rank(vis, pos);
        pos = RNG_SEG;
        int p = 0;
        while (p < RNG_SEG) p += a.cons[pos_index(a, b, p, s)];
        pos = p;
      }
      break;
    }
    pos += a.cons[pos_index(a, b, pos, s)];
    ++n;
  }
  raw_adv[b] = int64_t(s) * RNG_SEG + pos;
}

}  // namespace lrz

using namespace lrz;

static int64_t rng_nseg(int64_t L) { return (L + L / 32 + 2048 + RNG_SEG - 1) / RNG_SEG; }

size_t lrz_rng_ws(int64_t B, int64_t L) {
  const int64_t n = B * rng_nseg(L);
  return size_t(n) * RNG_SEG * (8 + 1 + 1) + size_t(n) * (RNG_SEG / 8) +
         size_t(n) * (2 * 4 * RNG_NE + 4 + 8) + 256;
}

static RngArgs rng_args(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                        const int64_t *raw0, void *workspace) {
  RngArgs a;
  a.B = B;
  a.L = L;
  a.nseg = int(rng_nseg(L));
  a.st = state;
  a.inc = inc;
  a.raw0 = raw0;
  const int64_t n = B * a.nseg;
  char *w = (char *)workspace;
  a.vals0 = (double *)w;
  w += size_t(n) * RNG_SEG * 8;
  a.seg_base = (int64_t *)w;
  w += size_t(n) * 8;
  a.seg_cnt0 = (int32_t *)w;
  w += size_t(n) * 4 * RNG_NE;
  a.seg_exit0 = (int32_t *)w;
  w += size_t(n) * 4 * RNG_NE;
  a.seg_entry = (int32_t *)w;
  w += size_t(n) * 4;
  a.vis = (uint32_t *)w;
  w += size_t(n) * (RNG_SEG / 8);
  a.cons = (uint8_t *)w;
  w += size_t(n) * RNG_SEG;
  a.pos0 = (uint8_t *)w;
  a.out = nullptr;
  a.startpos = nullptr;
  a.status = nullptr;
  return a;
}

extern "C" int lrz_rng_normals(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                               const int64_t *raw0, double *out, int32_t *startpos,
                               int32_t *status, void *workspace, void *stream) {
  if (B < 0 || L < 1 || L > (int64_t(1) << 30) || !state || !inc || !raw0 || !out || !status ||
      !workspace) {
    lrz_set_error("lrz_rng_normals: bad arguments");
    return LRZ_EINVAL;
  }
  if (startpos) {
    lrz_set_error("lrz_rng_normals: per-normal positions are not produced; use lrz_rng_locate");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  RngArgs a = rng_args(B, L, state, inc, raw0, workspace);
  a.out = out;
  a.status = status;
  const int64_t n = B * a.nseg;
  cudaStream_t s = (cudaStream_t)stream;
  LrzProf prof("rng_pass_abc", s);
  rng_pass_a<<<unsigned((n + RNG_A_THREADS - 1) / RNG_A_THREADS), RNG_A_THREADS, 0, s>>>(a);
  rng_pass_b<<<unsigned(B), RNG_B_THREADS, 0, s>>>(a);
  rng_pass_c<<<unsigned((n + RNG_C_THREADS - 1) / RNG_C_THREADS), RNG_C_THREADS, 0, s>>>(a);
  return lrz_launch_status("lrz_rng_normals");
}

extern "C" int lrz_rng_locate(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                              const int64_t *raw0, const int64_t *consumed, int64_t *raw_advance,
                              void *workspace, void *stream) {
  if (B < 0 || L < 1 || !consumed || !raw_advance || !workspace) {
    lrz_set_error("lrz_rng_locate: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  RngArgs a = rng_args(B, L, state, inc, raw0, workspace);
  rng_locate_kernel<<<unsigned((B + 127) / 128), 128, 0, (cudaStream_t)stream>>>(a, consumed,
                                                                               raw_advance);
  return lrz_launch_status("lrz_rng_locate");
}
