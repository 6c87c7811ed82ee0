// DMMA throughput against warps per SM scheduler (developer tool): how many resident warps the FP64
// tensor pipe needs to reach its peak, with 24 independent 8x8 accumulator tiles per warp (the solve
// kernel's k-step: 4 m-tiles x 2 n-tiles x 3 products), and whether DFMA work issued by other warps
// adds to it (shared or separate FP64 datapaths).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_dmma_occ bench_dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_k(double* out, int iters, double s, int dfma_warps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  if (warp < dfma_warps) {  // DFMA warps: 2 * NACC independent FMA chains
    double a = lane * 1e-3 + s;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        c[i][0] = fma(c[i][0], s, a);
        c[i][1] = fma(c[i][1], s, a);
      }
  } else {
    double a = lane * 1e-3 + s, b = lane * 2e-3 + s;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < NACC; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1])
                     : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.0) out[0] = t;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wps : {1, 2, 3, 4, 6, 8, 16}) {  // DMMA warps per SM scheduler
    for (int dfps : {0, 1, 2}) {            // DFMA warps per scheduler beside them
      const int warps = 4 * (wps + dfps);
      if (warps > 32) continue;
      auto run = [&] { dmma_k<24><<<sms, 32 * warps>>>(out, iters, 0.999, 4 * dfps); };
      run();
      cudaEventRecord(e0);
      for (int i = 0; i < 3; ++i) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 3;
      const double dmma_fl = 2.0 * 256 * 24.0 * iters * sms * 4 * wps;
      const double dfma_fl = 2.0 * 32 * 48.0 * iters * sms * 4 * dfps;
      printf("dmma warps/SMSP %2d dfma warps/SMSP %d: %.3f ms  DMMA %.1f TF/s  DFMA %.1f TF/s  total %.1f  (%s)\n", wps,
             dfps, ms, dmma_fl / ms / 1e9, dfma_fl / ms / 1e9, (dmma_fl + dfma_fl) / ms / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
