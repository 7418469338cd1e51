// C-ABI plumbing: error reporting, device check, workspace sizing.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

static thread_local char g_err[512] = "";

void lrz_set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int lrz_launch_status(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    lrz_set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return LRZ_ELAUNCH;
  }
  return LRZ_OK;
}

size_t lrz_arsvd_ws_total(int64_t B, int K, int D);
size_t lrz_precode_ws(int dtype, int64_t B, int K, int N);
size_t lrz_wb_ws(int64_t B, int K, int D);
size_t lrz_rng_ws(int64_t B, int64_t L);
size_t lrz_inverse_blocked_ws(int64_t B, int K);

extern "C" int lrz_version(void) { return 1; }

extern "C" const char *lrz_last_error(void) { return g_err; }

extern "C" int lrz_device_check(int device) {
  cudaDeviceProp p;
  const cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) {
    lrz_set_error("cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    return LRZ_EDEVICE;
  }
  if (p.major != 10 || p.minor != 0) {
    lrz_set_error("device %d is sm_%d%d; this library is built for sm_100a only", device,
                  p.major, p.minor);
    return LRZ_EDEVICE;
  }
  return LRZ_OK;
}

extern "C" size_t lrz_workspace_bytes(int op, int dtype, int64_t B, int K, int N, int d_max) {
  switch (op) {
    case LRZ_WS_INVERSE:
      // per-item redo flags of the fast paths (+ the blocked GJ buffers, K > 64)
      return ((size_t(B) + 255) & ~size_t(255)) +
             ((K >= 64 && K <= 256 && K % 32 == 0) ? lrz_inverse_blocked_ws(B, K) : 0);
    case LRZ_WS_ARSVD:
      return lrz_arsvd_ws_total(B, K, d_max);
    case LRZ_WS_WOODBURY:
    case LRZ_WS_CHAIN:
      return lrz_wb_ws(B, K, d_max);
    case LRZ_WS_PRECODE:
      return lrz_precode_ws(dtype, B, K, N);
    case LRZ_WS_RNG:
      return lrz_rng_ws(B, N);
    default:
      return 0;
  }
}

// ---- per-kernel event profiler (prof.cuh) -----------------------------------
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "prof.cuh"

namespace {
struct ProfState {
  std::mutex mu;
  int on = 0;
  std::vector<cudaEvent_t> pool;  // events handed out since the last collect
  size_t next = 0;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> recs;
  std::string out;
};
ProfState &prof() {
  static ProfState p;
  return p;
}
}  // namespace

int lrz_prof_on() { return prof().on; }

cudaEvent_t lrz_prof_event() {
  ProfState &p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  if (p.next == p.pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p.pool.push_back(e);
  }
  return p.pool[p.next++];
}

void lrz_prof_record(const char *name, cudaEvent_t a, cudaEvent_t b) {
  ProfState &p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  p.recs.push_back({name, {a, b}});
}

extern "C" int lrz_prof_enable(int on) {
  ProfState &p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  p.on = on;
  p.recs.clear();
  p.next = 0;
  return LRZ_OK;
}

extern "C" const char *lrz_prof_collect(void) {
  ProfState &p = prof();
  std::lock_guard<std::mutex> lk(p.mu);
  std::map<std::string, std::pair<double, int>> agg;
  for (auto &r : p.recs) {
    cudaEventSynchronize(r.second.second);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.second.first, r.second.second) != cudaSuccess) ms = -1.f;
    auto &a = agg[r.first];
    a.first += ms;
    a.second += 1;
  }
  p.recs.clear();
  p.next = 0;
  p.out.clear();
  char buf[256];
  for (auto &kv : agg) {
    snprintf(buf, sizeof(buf), "%s=%.6f:%d;", kv.first.c_str(), kv.second.first,
             kv.second.second);
    p.out += buf;
  }
  return p.out.c_str();
}
