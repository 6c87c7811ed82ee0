// Developer microbenchmark (not part of the library): latencies that bound a lone solve warp.
//  1. DMMA m8n8k4 f64 dependent-chain latency (one accumulator),
//  2. one warp issuing NI independent DMMA chains (throughput of a lone warp),
//  3. cp.async 16 B (LDGSTS.BYPASS) round trip from L2 for one warp,
//  4. ld.global L2 hit round trip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_lat bench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NI>
__global__ void chain(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[NI][2];
  for (int i = 0; i < NI; ++i) d[i][0] = d[i][1] = i;
  __syncwarp();
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int i = 0; i < NI; ++i) dmma(d[i][0], d[i][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < NI; ++i) s += d[i][0] + d[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void cpasync_lat(const double2* src, int n, int iters, long long* cyc, double* out) {
  __shared__ __align__(16) double2 buf[32];
  const int lane = threadIdx.x;
  int idx = lane;
  double acc = 0;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(buf + lane)), "l"(src + idx) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    double2 v = buf[lane];
    acc += v.x;
    idx = (idx + 32 + (int)(v.y)) % n;  // dependent address
  }
  long long t1 = clock64();
  out[lane] = acc;
  if (lane == 0) *cyc = t1 - t0;
}
__global__ void ld_lat(const double2* src, int n, int iters, long long* cyc, double* out) {
  const int lane = threadIdx.x;
  int idx = lane;
  double acc = 0;
  long long t0 = clock64();
  for (int k = 0; k < iters; ++k) {
    double2 v = __ldcg(src + idx);
    acc += v.x;
    idx = (idx + 32 + (int)(v.y)) % n;
  }
  long long t1 = clock64();
  out[lane] = acc;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; double2* src;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 8);
  const int n = 1 << 16;  // 1 MB: L2 resident
  cudaMalloc(&src, n * sizeof(double2)); cudaMemset(src, 0, n * sizeof(double2));
  long long c;
  const int it = 4096;
  auto run = [&](auto kern, int ni, const char* what) {
    kern<<<1, 32>>>(out, it, cyc); kern<<<1, 32>>>(out, it, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per iteration of %d DMMAs (%.1f per DMMA)\n", what, (double)c / it, ni, (double)c / it / ni);
  };
  run(chain<1>, 1, "1 chain");
  run(chain<2>, 2, "2 chains");
  run(chain<4>, 4, "4 chains");
  run(chain<8>, 8, "8 chains");
  run(chain<16>, 16, "16 chains");
  run(chain<32>, 32, "32 chains");
  cpasync_lat<<<1, 32>>>(src, n, 512, cyc, out); cpasync_lat<<<1, 32>>>(src, n, 512, cyc, out);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("cp.async 16B + wait, dependent: %.1f cycles\n", (double)c / 512);
  ld_lat<<<1, 32>>>(src, n, 512, cyc, out); ld_lat<<<1, 32>>>(src, n, 512, cyc, out);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("ld.cg 16B, dependent: %.1f cycles\n", (double)c / 512);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
