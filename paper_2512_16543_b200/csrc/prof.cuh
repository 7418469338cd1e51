// Per-kernel device timing (CUDA events on the launching stream), off by
// default.  lrz_prof_enable(1) starts collecting; every instrumented launch
// site brackets its kernel with a LrzProf scope; lrz_prof_collect() waits on
// the events and returns "name=ms_total:launches;..." -- the per-kernel
// average launch durations bench.py divides the algorithmic work by.
#pragma once

#include <cuda_runtime.h>

int lrz_prof_on();
void lrz_prof_record(const char *name, cudaEvent_t a, cudaEvent_t b);
cudaEvent_t lrz_prof_event();

struct LrzProf {
  const char *name;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  LrzProf(const char *n, cudaStream_t st) : name(n), s(st) {
    if (lrz_prof_on()) {
      a = lrz_prof_event();
      cudaEventRecord(a, s);
    }
  }
  ~LrzProf() {
    if (a) {
      cudaEvent_t b = lrz_prof_event();
      cudaEventRecord(b, s);
      lrz_prof_record(name, a, b);
    }
  }
};
