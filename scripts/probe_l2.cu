// L2 capacity probe for the SpMM C-row gathers: random
// 256-byte row gathers (a half-warp per row, 128-bit loads, like the SpMM
// leaf) over a working set of `nrows` rows, uniform over the set.
//   mode 0: every SM gathers from the whole set;
//   mode 1: SMs with smid <  split gather only even rows, the others odd rows;
//   mode 2: SMs with even smid gather only even rows, odd smid odd rows.
// If the effective capacity for data read by all SMs is half the L2 (each
// die's half caching what its own SMs read), modes 1 / 2 with the right SM
// grouping double the working set that still hits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o scripts/libprobe_l2.so scripts/probe_l2.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__global__ void __launch_bounds__(256) k_probe(const double* __restrict__ C, int64_t nrows, int64_t per_warp,
                                                int mode, int split, double* __restrict__ sink) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  int parity = -1;
  if (mode == 1) parity = smid < (unsigned)split ? 0 : 1;
  if (mode == 2) parity = smid & 1;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = 0; i < per_warp; i += 8) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      uint64_t r = mix(gw * 0x9e3779b97f4a7c15ULL + (uint64_t)(i + 2 * u + half)) % (uint64_t)nrows;
      if (parity >= 0) r = (r & ~1ULL) | (uint64_t)parity;
      if (r >= (uint64_t)nrows) r -= 2;
      v[u] = __ldg(reinterpret_cast<const double2*>(C + r * 32) + hl);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) acc.x += v[u].x, acc.y += v[u].y;
  }
  if (acc.x == 12345.678) sink[0] = acc.y;  // keeps the loads
}

extern "C" int probe_l2(const double* C, int64_t nrows, int64_t per_warp, int mode, int split, double* sink,
                        int grid, float* ms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_probe<<<grid, 256>>>(C, nrows, per_warp, mode, split, sink);  // warm
  cudaEventRecord(a);
  k_probe<<<grid, 256>>>(C, nrows, per_warp, mode, split, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (int)cudaGetLastError();
}
