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
//      draws a normal starting there consumes (c_j) and its value;
//      summarise the segment for a normal starting at its first draw;
//   B  one thread per trial: walk the segment summaries (re-walking a
//      segment only when a multi-draw normal straddles its start) to get each
//      segment's entry offset and the index of its first normal;
//   C  one thread per segment: emit the normals at their stream indices and
//      their raw start positions (used to advance the stream by exactly the
//      normals a chunk consumed).

#include "common.cuh"
#include "_gen/ziggurat_tables.h"

namespace lrz {

typedef unsigned __int128 u128;
constexpr int RNG_SEG = 256;
constexpr int RNG_MAXC = 64;  // a normal consuming more draws aborts the window (never seen)
constexpr int RNG_NE = 8;     // entry offsets summarised per segment by pass A
constexpr int RNG_A_THREADS = 128;
constexpr int RNG_B_CHUNK = 512;  // segments per shared-memory chunk in pass B
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
        const double xx = -0.27366123732975828 * log1p(-pcg_double(st, inc));
        const double yy = -log1p(-pcg_double(st, inc));
        used += 2;
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(3.6541528853610088 + xx) : 3.6541528853610088 + xx;
        if (used > RNG_MAXC) return 0.0;
      }
    } else {
      const double u = pcg_double(st, inc);
      ++used;
      if ((t.fi[idx - 1] - t.fi[idx]) * u + t.fi[idx] < exp(-0.5 * x * x)) return x;
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
  uint8_t *cons;         // [B][nseg * SEG] draws consumed by a normal starting here
  double *val;           // [B][nseg * SEG]
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
  int over = 0;
  for (int j = 0; j < RNG_SEG; ++j) {
    const uint64_t r = pcg_next(st, inc);  // raw draw j; st now before draw j + 1
    int used;
    const double x = zig_from(r, st, inc, tb, used);
    if (used > RNG_MAXC) over = 1;
    const uint8_t cu = uint8_t(used > 255 ? 255 : used);
    c[j] = cu;
    const int64_t q = pos_index(a, b, j, s);
    a.cons[q] = cu;
    a.val[q] = x;
  }
  // walk(0) with a visited mask, then entries 1..RNG_NE-1 merge into it
  uint32_t vis[RNG_SEG / 32];
#pragma unroll
  for (int i = 0; i < RNG_SEG / 32; ++i) vis[i] = 0;
  int pos = 0, cnt0 = 0;
  while (pos < RNG_SEG) {
    vis[pos >> 5] |= 1u << (pos & 31);
    ++cnt0;
    pos += c[pos];
  }
  const int exit0 = pos - RNG_SEG;
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

// one CTA per trial: segment summaries staged in shared memory, thread 0 walks
__global__ void __launch_bounds__(256) rng_pass_b(RngArgs a) {
  __shared__ int32_t s_cnt[RNG_B_CHUNK * RNG_NE], s_exit[RNG_B_CHUNK * RNG_NE];
  __shared__ int s_entry;
  __shared__ long long s_base;
  __shared__ int s_bad;
  const int64_t b = blockIdx.x;
  if (threadIdx.x == 0) {
    s_entry = 0;
    s_base = 0;
    s_bad = 0;
  }
  for (int s0 = 0; s0 < a.nseg; s0 += RNG_B_CHUNK) {
    const int ns = min(RNG_B_CHUNK, a.nseg - s0);
    __syncthreads();
    for (int i = threadIdx.x; i < ns * RNG_NE; i += blockDim.x) {
      const int64_t g = (b * a.nseg + s0) * RNG_NE + i;
      s_cnt[i] = a.seg_cnt0[g];
      s_exit[i] = a.seg_exit0[g];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int entry = s_entry, bad = s_bad;
      long long base = s_base;
      for (int i = 0; i < ns; ++i) {
        const int s = s0 + i;
        const int64_t id = b * a.nseg + s;
        a.seg_entry[id] = entry;
        a.seg_base[id] = base;
        if (entry < RNG_NE) {
          const int ex = s_exit[i * RNG_NE + entry];
          if (ex >= (1 << 20)) bad = 1;
          base += s_cnt[i * RNG_NE + entry];
          entry = ex >= (1 << 20) ? 0 : ex;
        } else if (entry >= RNG_SEG) {
          entry -= RNG_SEG;
        } else {  // rare: re-walk from global memory
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
      s_entry = entry;
      s_base = base;
      s_bad = bad;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.status[b] = (s_bad || s_base < a.L) ? 1 : 0;
}

__global__ void rng_pass_c(RngArgs a) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (tid >= a.B * a.nseg) return;
  const int64_t b = tid / a.nseg;
  const int s = int(tid - b * a.nseg);
  int pos = a.seg_entry[tid];
  int64_t n = a.seg_base[tid];
  double *o = a.out + b * a.L;
  int32_t *sp = a.startpos ? a.startpos + b * a.L : nullptr;
  while (pos < RNG_SEG && n < a.L) {
    const int64_t q = pos_index(a, b, pos, s);
    o[n] = a.val[q];
    if (sp) sp[n] = int32_t(int64_t(s) * RNG_SEG + pos);
    ++n;
    pos += a.cons[q];
  }
}

}  // namespace lrz

using namespace lrz;

size_t lrz_rng_ws(int64_t B, int64_t L) {
  const int64_t nseg = (L + L / 32 + 2048 + RNG_SEG - 1) / RNG_SEG;
  const int64_t n = B * nseg;
  return size_t(n) * RNG_SEG * (1 + 8) + size_t(n) * (2 * 4 * RNG_NE + 4 + 8) + 256;
}

extern "C" int lrz_rng_normals(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                               const int64_t *raw0, double *out, int32_t *startpos,
                               int32_t *status, void *workspace, void *stream) {
  if (B < 0 || L < 1 || L > (int64_t(1) << 30) || !state || !inc || !raw0 || !out || !status ||
      !workspace) {
    lrz_set_error("lrz_rng_normals: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  RngArgs a;
  a.B = B;
  a.L = L;
  a.nseg = int((L + L / 32 + 2048 + RNG_SEG - 1) / RNG_SEG);
  a.st = state;
  a.inc = inc;
  a.raw0 = raw0;
  const int64_t n = B * a.nseg;
  char *w = (char *)workspace;
  a.val = (double *)w;
  w += size_t(n) * RNG_SEG * 8;
  a.seg_base = (int64_t *)w;
  w += size_t(n) * 8;
  a.seg_cnt0 = (int32_t *)w;
  w += size_t(n) * 4 * RNG_NE;
  a.seg_exit0 = (int32_t *)w;
  w += size_t(n) * 4 * RNG_NE;
  a.seg_entry = (int32_t *)w;
  w += size_t(n) * 4;
  a.cons = (uint8_t *)w;
  a.out = out;
  a.startpos = startpos;
  a.status = status;
  cudaStream_t s = (cudaStream_t)stream;
  rng_pass_a<<<unsigned((n + RNG_A_THREADS - 1) / RNG_A_THREADS), RNG_A_THREADS, 0, s>>>(a);
  rng_pass_b<<<unsigned(B), 256, 0, s>>>(a);
  rng_pass_c<<<unsigned((n + 127) / 128), 128, 0, s>>>(a);
  return lrz_launch_status("lrz_rng_normals");
}
