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

// numpy's random_standard_normal on the draw stream starting at `st`
// (`st` advanced past every draw consumed); returns the value, sets used.
LRZ_DEV double zig_normal(u128 &st, u128 inc, int &used) {
  used = 0;
  for (;;) {
    uint64_t r = pcg_next(st, inc);
    ++used;
    const int idx = int(r & 0xff);
    r >>= 8;
    const int sign = int(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = double(rabs) * zig_wi_double[idx];
    if (sign) x = -x;
    if (rabs < zig_ki_double[idx]) return x;
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
      if ((zig_fi_double[idx - 1] - zig_fi_double[idx]) * u + zig_fi_double[idx] <
          exp(-0.5 * x * x))
        return x;
    }
    if (used > RNG_MAXC) return 0.0;
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
  int32_t *seg_cnt0;     // [B][nseg] normals in the segment for entry offset 0
  int32_t *seg_exit0;    // [B][nseg] overhang into the next segment for entry 0
  int32_t *seg_entry;    // [B][nseg] true entry offset
  int64_t *seg_base;     // [B][nseg] stream index of the segment's first normal
  double *out;           // [B][L]
  int64_t L;
  int32_t *startpos;     // [B][L] raw position (relative to raw0) of each normal
  int32_t *status;       // [B] 0 ok, 1 window too short / overlong normal
};

LRZ_DEV u128 load_u128(const uint64_t *p) { return (u128(p[1]) << 64) | u128(p[0]); }

__global__ void rng_pass_a(RngArgs a) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (tid >= a.B * a.nseg) return;
  const int64_t b = tid / a.nseg;
  const int s = int(tid - b * a.nseg);
  const u128 inc = load_u128(a.inc + 2 * b);
  u128 st = pcg_advance(load_u128(a.st + 2 * b), inc,
                        uint64_t(a.raw0[b]) + uint64_t(s) * RNG_SEG);
  uint8_t *c = a.cons + tid * RNG_SEG;
  double *v = a.val + tid * RNG_SEG;
  int pos = 0, cnt = 0, over = 0;  // walk for entry 0
  for (int j = 0; j < RNG_SEG; ++j) {
    u128 probe = st;
    int used;
    const double x = zig_normal(probe, inc, used);
    if (used > RNG_MAXC) over = 1;
    c[j] = uint8_t(used > 255 ? 255 : used);
    v[j] = x;
    if (j == pos) {
      ++cnt;
      pos += used;
    }
    pcg_next(st, inc);  // advance one raw position
  }
  a.seg_cnt0[tid] = cnt;
  a.seg_exit0[tid] = over ? (1 << 20) : pos - RNG_SEG;
}

__global__ void rng_pass_b(RngArgs a) {
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= a.B) return;
  int entry = 0;
  int64_t base = 0;
  int bad = 0;
  for (int s = 0; s < a.nseg; ++s) {
    const int64_t id = b * a.nseg + s;
    a.seg_entry[id] = entry;
    a.seg_base[id] = base;
    if (a.seg_exit0[id] >= (1 << 20)) bad = 1;
    if (entry == 0) {
      base += a.seg_cnt0[id];
      entry = a.seg_exit0[id];
    } else if (entry >= RNG_SEG) {
      entry -= RNG_SEG;  // a very long normal spans the whole segment
    } else {
      const uint8_t *c = a.cons + id * RNG_SEG;
      int pos = entry, cnt = 0;
      while (pos < RNG_SEG) {
        if (c[pos] >= 255) bad = 1;
        ++cnt;
        pos += c[pos];
      }
      base += cnt;
      entry = pos - RNG_SEG;
    }
  }
  if (base < a.L) bad = 1;
  a.status[b] = bad;
}

__global__ void rng_pass_c(RngArgs a) {
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (tid >= a.B * a.nseg) return;
  const int64_t b = tid / a.nseg;
  const int s = int(tid - b * a.nseg);
  int pos = a.seg_entry[tid];
  int64_t n = a.seg_base[tid];
  const uint8_t *c = a.cons + tid * RNG_SEG;
  const double *v = a.val + tid * RNG_SEG;
  double *o = a.out + b * a.L;
  int32_t *sp = a.startpos ? a.startpos + b * a.L : nullptr;
  while (pos < RNG_SEG && n < a.L) {
    o[n] = v[pos];
    if (sp) sp[n] = int32_t(int64_t(s) * RNG_SEG + pos);
    ++n;
    pos += c[pos];
  }
}

}  // namespace lrz

using namespace lrz;

size_t lrz_rng_ws(int64_t B, int64_t L) {
  const int64_t nseg = (L + L / 32 + 2048 + RNG_SEG - 1) / RNG_SEG;
  const int64_t n = B * nseg;
  return size_t(n) * RNG_SEG * (1 + 8) + size_t(n) * (4 + 4 + 4 + 8) + 256;
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
  w += size_t(n) * 4;
  a.seg_exit0 = (int32_t *)w;
  w += size_t(n) * 4;
  a.seg_entry = (int32_t *)w;
  w += size_t(n) * 4;
  a.cons = (uint8_t *)w;
  a.out = out;
  a.startpos = startpos;
  a.status = status;
  cudaStream_t s = (cudaStream_t)stream;
  rng_pass_a<<<unsigned((n + 127) / 128), 128, 0, s>>>(a);
  rng_pass_b<<<unsigned((B + 63) / 64), 64, 0, s>>>(a);
  rng_pass_c<<<unsigned((n + 127) / 128), 128, 0, s>>>(a);
  return lrz_launch_status("lrz_rng_normals");
}
