// Microbenchmark of the solve kernels' inner product (developer tool, not part of the
// library): each warp computes out[32 rows][RW rhs] = L[32 x K] * X[K x RW] with L streamed
// from HBM (column-major 32-row chunks, one coalesced 512-byte load per column) and X from
// a per-warp shared tile, exactly like fwd_block. Reports DFMA issue rate vs the B200 FP64
// peak and achieved HBM bandwidth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_inner bench_inner.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int RW, int U>
__global__ void __launch_bounds__(256, 2) inner(const double2* L, const double2* X, double2* out, int K, int items) {
  extern __shared__ double2 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* xs = sm + w * 32 * 16;
  const int gw = (blockIdx.x * 256 + threadIdx.x) >> 5, nw = gridDim.x * 8;
  for (int it = gw; it < items; it += nw) {
    const double2* P = L + static_cast<long long>(it) * K * 32;
    double2 acc[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) acc[r] = make_double2(0, 0);
    for (int J = 0; J < K; J += 32) {
      for (int r = 0; r < RW; ++r) xs[lane * RW + r] = X[(J + lane) * RW + r];
      __syncwarp();
      for (int j = 0; j < 32; j += U) {
        double2 l[U];
#pragma unroll
        for (int u = 0; u < U; ++u) l[u] = ld_stream(P + (J + j + u) * 32 + lane);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < RW; ++r) cfma(acc[r], l[u], xs[(j + u) * RW + r]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) out[(static_cast<long long>(it) * 32 + lane) * RW + r] = acc[r];
  }
}


// DMMA variant: factor stored in m8n8k4 A-fragment order (per k-step of 4 columns, 4 m-tiles
// of 8 rows, lane t holds row t>>2, column t&3 as one double2), T tile [k][16] double2 in smem.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int PF>
__global__ void __launch_bounds__(256, 2) inner_mma(const double2* L, const double2* X, double2* out, int K, int items) {
  extern __shared__ double2 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* xs = sm + w * 32 * 16;
  const int gw = (blockIdx.x * 256 + threadIdx.x) >> 5, nw = gridDim.x * 8;
  for (int it = gw; it < items; it += nw) {
    const double2* P = L + static_cast<long long>(it) * K * 32 + lane;
    double acc[4][2][2][2];  // m-tile, n-tile, re/im, 2 regs
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[i][q][c][0] = acc[i][q][c][1] = 0.0;
    const int ks = K / 4;
    double2 a[PF][4];
#pragma unroll
    for (int p = 0; p < PF; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[p][i] = ld_stream(P + (p * 4 + i) * 32);
    for (int J = 0; J < K; J += 32) {
      for (int e = lane; e < 512; e += 32) xs[e] = X[J * 16 + e];
      __syncwarp();
#pragma unroll 1
      for (int s0 = 0; s0 < 8; s0 += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
          const int s = J / 4 + s0 + p;
          double2 cur[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) cur[i] = a[p][i];
          if (s + PF < ks)
#pragma unroll
            for (int i = 0; i < 4; ++i) a[p][i] = ld_stream(P + ((s + PF) * 4 + i) * 32);
          const int kk = (s0 + p) * 4 + (lane & 3);
#pragma unroll
      double2 bb[2];
      double nb[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        bb[q] = xs[kk * 16 + q * 8 + (lane >> 2)];
        nb[q] = -bb[q].y;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma(acc[i][q][0][0], acc[i][q][0][1], cur[i].x, bb[q].x);
          dmma(acc[i][q][1][0], acc[i][q][1][1], cur[i].x, bb[q].y);
        }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma(acc[i][q][0][0], acc[i][q][0][1], cur[i].y, nb[q]);
          dmma(acc[i][q][1][0], acc[i][q][1][1], cur[i].y, bb[q].x);
        }
        }
      }
      __syncwarp();
    }
    double2* o = out + static_cast<long long>(it) * 32 * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          o[(i * 8 + (lane >> 2)) * 16 + q * 8 + (lane & 3) * 2 + e] = make_double2(acc[i][q][0][e], acc[i][q][1][e]);
  }
}
template <int PF>
void run_mma(const double2* L, const double2* X, double2* out, int K, int items, int blocks) {
  cudaFuncSetAttribute(inner_mma<PF>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  inner_mma<PF><<<blocks, 256, 65536>>>(L, X, out, K, items);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) inner_mma<PF><<<blocks, 256, 65536>>>(L, X, out, K, items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double flops = 8.0 * items * 32.0 * K * 16;
  const double bytes = 16.0 * items * 32.0 * K;
  printf("MMA PF=%d blocks=%d: %.3f ms  %.1f TFLOP/s  %.0f GB/s  (err %s)\n", PF, blocks, ms, flops / ms / 1e9,
         bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}


__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(s))), "l"(g));
}
// ring variant: A fragments streamed through a per-warp smem ring of NS k-steps (2 KB each)
template <int NS, int WPC>
__global__ void __launch_bounds__(WPC * 32) inner_ring(const double2* L, const double2* X, double2* out, int K, int items) {
  extern __shared__ double2 sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* xs = sm + w * (32 * 16 + NS * 128);
  double2* ring = xs + 32 * 16;
  const int gw = (blockIdx.x * WPC * 32 + threadIdx.x) >> 5, nw = gridDim.x * WPC;
  for (int it = gw; it < items; it += nw) {
    const double2* P = L + static_cast<long long>(it) * K * 32 + lane;
    double acc[4][2][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc[i][q][c][0] = acc[i][q][c][1] = 0.0;
    const int ks = K / 4;
#pragma unroll
    for (int p = 0; p < NS - 1; ++p) {
      if (p < ks)
#pragma unroll
        for (int i = 0; i < 4; ++i) cp16(ring + p * 128 + i * 32 + lane, P + (p * 4 + i) * 32);
      asm volatile("cp.async.commit_group;");
    }
    for (int s = 0; s < ks; ++s) {
      if ((s & 7) == 0) {
        __syncwarp();
        for (int e = lane; e < 512; e += 32) xs[e] = X[s * 64 + e];
      }
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2));
      __syncwarp();
      const double2* st = ring + (s % NS) * 128 + lane;
      double2 cur[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = st[i * 32];
      __syncwarp();
      const int sn = s + NS - 1;
      if (sn < ks)
#pragma unroll
        for (int i = 0; i < 4; ++i) cp16(ring + (sn % NS) * 128 + i * 32 + lane, P + (sn * 4 + i) * 32);
      asm volatile("cp.async.commit_group;");
      const int kk = (s & 7) * 4 + (lane & 3);
#pragma unroll
      double2 bb[2];
      double nb[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        bb[q] = xs[kk * 16 + q * 8 + (lane >> 2)];
        nb[q] = -bb[q].y;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma(acc[i][q][0][0], acc[i][q][0][1], cur[i].x, bb[q].x);
          dmma(acc[i][q][1][0], acc[i][q][1][1], cur[i].x, bb[q].y);
        }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dmma(acc[i][q][0][0], acc[i][q][0][1], cur[i].y, nb[q]);
          dmma(acc[i][q][1][0], acc[i][q][1][1], cur[i].y, bb[q].x);
        }
    }
    asm volatile("cp.async.wait_group 0;");
    double2* o = out + static_cast<long long>(it) * 32 * 16;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          o[(i * 8 + (lane >> 2)) * 16 + q * 8 + (lane & 3) * 2 + e] = make_double2(acc[i][q][0][e], acc[i][q][1][e]);
  }
}
template <int NS, int WPC>
void run_ring(const double2* L, const double2* X, double2* out, int K, int items) {
  const int smem = WPC * (32 * 16 + NS * 128) * 16;
  cudaFuncSetAttribute(inner_ring<NS, WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_ring<NS, WPC>, WPC * 32, smem);
  const int blocks = 148 * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  inner_ring<NS, WPC><<<blocks, WPC * 32, smem>>>(L, X, out, K, items);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) inner_ring<NS, WPC><<<blocks, WPC * 32, smem>>>(L, X, out, K, items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double flops = 8.0 * items * 32.0 * K * 16;
  const double bytes = 16.0 * items * 32.0 * K;
  printf("RING NS=%d WPC=%d ctas/sm=%d: %.3f ms  %.1f TFLOP/s  %.0f GB/s  (err %s)\n", NS, WPC, per_sm, ms,
         flops / ms / 1e9, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

template <int RW, int U>
void run(const double2* L, const double2* X, double2* out, int K, int items, int blocks) {
  cudaFuncSetAttribute(inner<RW, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  inner<RW, U><<<blocks, 256, 65536>>>(L, X, out, K, items);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) inner<RW, U><<<blocks, 256, 65536>>>(L, X, out, K, items);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double flops = 8.0 * items * 32.0 * K * RW;
  const double bytes = 16.0 * items * 32.0 * K;
  printf("RW=%2d U=%d blocks=%d: %.3f ms  %.1f TFLOP/s  %.0f GB/s  (err %s)\n", RW, U, blocks, ms, flops / ms / 1e9,
         bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const bool only = argc > 1;
  const int K = 64, items = 148 * 16 * 8;
  double2 *L, *X, *out;
  cudaMalloc(&L, sizeof(double2) * items * K * 32);
  cudaMalloc(&X, sizeof(double2) * K * 16);
  cudaMalloc(&out, sizeof(double2) * items * 32 * 16);
  cudaMemset(L, 0, sizeof(double2) * items * K * 32);
  cudaMemset(X, 0, sizeof(double2) * K * 16);
  run_ring<4, 4>(L, X, out, K, items);
  if (only) return 0;
  run_ring<8, 4>(L, X, out, K, items);
  run_ring<4, 2>(L, X, out, K, items);
  run_ring<8, 2>(L, X, out, K, items);
  run_ring<16, 2>(L, X, out, K, items);
  run_ring<6, 4>(L, X, out, K, items);
  for (int blocks : {296}) {
    run<16, 8>(L, X, out, K, items, blocks);
    run_mma<1>(L, X, out, K, items, blocks);
    run_mma<2>(L, X, out, K, items, blocks);
    run_mma<4>(L, X, out, K, items, blocks);
    run<16, 4>(L, X, out, K, items, blocks);
    run<8, 8>(L, X, out, K, items, blocks);
    run<4, 8>(L, X, out, K, items, blocks);
  }
  return 0;
}
