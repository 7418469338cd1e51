// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double *out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 0.001, b = 1.0000001;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double *o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * double(blocks) * threads;
    printf("DFMA: %.2f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * iters * double(blocks) * (threads / 32);
    printf("DMMA: %.2f TFLOP/s\n", fl / ms / 1e9);
  }
  return 0;
}
