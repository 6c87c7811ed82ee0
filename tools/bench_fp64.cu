// FP64 ceilings on this GPU (developer tool): DFMA issue peak and DMMA (mma.sync m8n8k4 f64)
// peak, so the solve kernels' roofline uses a measured FP64 denominator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_fp64 bench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_peak(double* out, int iters, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-9);
  double t = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 12345.0) out[0] = t;
}

__global__ void dmma_peak(double* out, int iters, double s) {
  const int lane = threadIdx.x & 31;
  double a = lane * 1e-3 + s, b = lane * 2e-3 + s;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  double t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.0) out[0] = t;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  for (int blocks : {148 * 4, 148 * 8}) {
    float ms = timeit([&] { dfma_peak<<<blocks, 256>>>(out, iters, 0.999); });
    double fl = 2.0 * blocks * 256.0 * iters * 16;
    printf("DFMA  blocks=%d: %.3f ms  %.1f TFLOP/s\n", blocks, ms, fl / ms / 1e9);
    ms = timeit([&] { dmma_peak<<<blocks, 256>>>(out, iters, 0.999); });
    fl = 2.0 * blocks * 8.0 * iters * 8 * 256;  // 8x8x4 = 256 FMA per warp-mma
    printf("DMMA  blocks=%d: %.3f ms  %.1f TFLOP/s  (%s)\n", blocks, ms, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
