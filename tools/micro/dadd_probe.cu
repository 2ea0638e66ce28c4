// Microbenchmark (dev tool): FP64 add latency and issue cost on this GPU, for
// the quiet-span replay's four sequential DADD chains (engine.cuh
// quiet_steps_fused). Prints cycles per iteration for: one chain, four
// independent chains on all lanes, and the four chains packed one per lane.
#include <cstdio>
#include <cstdint>
__global__ void k(int iters, double* out, long long* cyc, int mode) {
  double a = threadIdx.x * 1e-3, b = 1.0, c = 2.0, d = 3.0;
  const double x = 1e-7, y = 2e-7, z = 3e-7;
  __syncwarp();
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < iters; ++i) { a += x; }
  } else if (mode == 1) {
    for (int i = 0; i < iters; ++i) { a += x; b += y; c += z; d += x; }
  } else {
    const double inc = (threadIdx.x & 3) == 0 ? x : (threadIdx.x & 3) == 1 ? y : z;
    for (int i = 0; i < iters; ++i) { a += inc; }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 * 148 * 16 * 32 * 8); cudaMallocManaged(&cyc, 8 * 148 * 16);
  const int iters = 1 << 16;
  for (int warps_per_sm : {1, 2, 8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      k<<<148 * warps_per_sm, 32>>>(iters, out, cyc, mode);
      cudaDeviceSynchronize();
      double s = 0; for (int i = 0; i < 148 * warps_per_sm; ++i) s += cyc[i];
      printf("warps/SM %2d mode %d (%s): %.2f cycles/iter\n", warps_per_sm, mode,
             mode == 0 ? "1 chain" : mode == 1 ? "4 chains, all lanes" : "4 chains packed per lane",
             s / (148 * warps_per_sm) / iters);
    }
  }
  return 0;
}
