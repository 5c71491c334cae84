// Gather-throughput probe (measurement only, not product code): the SpMM
// leaf's inner pattern -- per position a 256-byte row C[idx[q]] gathered by a
// half-warp with 128-bit loads and FMA'd into a register accumulator -- with
// the row indices streamed from an int32 array like the leaf's crd.  Sweeps
// the gathers in flight per warp (UNR pairs of positions) and the resident
// warps per SM (MINB CTAs of 256 threads) to find the gather ceiling of the
// B200 for L2-resident (small working set) and DRAM-resident rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        -o scripts/libprobe_gather.so scripts/probe_gather.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ldg2_na(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Positions in chunks of 1024 per warp (ticket-free grid stride: the probe has
// no ragged work); 32 indices loaded per lane-window, shuffled out per pair.
template <int UNR, int MINB, bool NA>
__global__ void __launch_bounds__(256, MINB) k_gather(const int32_t* __restrict__ idx, int64_t n,
                                                      const double* __restrict__ C, double* __restrict__ sink) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* Cl = C + 2 * hl;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t base = gw * 32; base < n; base += nw * 32) {
    const int my = __ldg(idx + base + lane);
#pragma unroll 1
    for (int u = 0; u < 32; u += 2 * UNR) {
      double2 v[UNR];
#pragma unroll
      for (int i = 0; i < UNR; i++) {
        const int k = __shfl_sync(0xffffffffu, my, u + 2 * i + half);
        v[i] = NA ? ldg2_na(Cl + (int64_t)k * 32) : ldg2(Cl + (int64_t)k * 32);
      }
#pragma unroll
      for (int i = 0; i < UNR; i++) {
        acc.x = fma(0.5, v[i].x, acc.x);
        acc.y = fma(0.5, v[i].y, acc.y);
      }
    }
  }
  if (acc.x == 12345.678) sink[0] = acc.y;
}

// Software-pipelined variant: the next group's loads are issued before the
// current group is consumed (2*UNR positions in flight per half-warp lane).
template <int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather_pipe(const int32_t* __restrict__ idx, int64_t n,
                                                           const double* __restrict__ C, double* __restrict__ sink) {
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* Cl = C + 2 * hl;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t base = gw * 32; base < n; base += nw * 32) {
    const int my = __ldg(idx + base + lane);
    double2 v[UNR], w[UNR];
#pragma unroll
    for (int i = 0; i < UNR; i++) v[i] = ldg2(Cl + (int64_t)__shfl_sync(0xffffffffu, my, 2 * i + half) * 32);
#pragma unroll
    for (int u = 2 * UNR; u < 32; u += 2 * UNR) {
#pragma unroll
      for (int i = 0; i < UNR; i++) w[i] = ldg2(Cl + (int64_t)__shfl_sync(0xffffffffu, my, u + 2 * i + half) * 32);
#pragma unroll
      for (int i = 0; i < UNR; i++) {
        acc.x = fma(0.5, v[i].x, acc.x);
        acc.y = fma(0.5, v[i].y, acc.y);
        v[i] = w[i];
      }
    }
#pragma unroll
    for (int i = 0; i < UNR; i++) {
      acc.x = fma(0.5, v[i].x, acc.x);
      acc.y = fma(0.5, v[i].y, acc.y);
    }
  }
  if (acc.x == 12345.678) sink[0] = acc.y;
}

template <class K>
static float run(K kern, const int32_t* idx, int64_t n, const double* C, double* sink, int* grid_out) {
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  const int grid = sms * (per_sm > 0 ? per_sm : 1);
  *grid_out = grid;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<grid, 256>>>(idx, n, C, sink);
  cudaEventRecord(a);
  for (int r = 0; r < 5; r++) kern<<<grid, 256>>>(idx, n, C, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? ms / 5 : -1.0f;
}

extern "C" float probe_gather(int variant, const int32_t* idx, int64_t n, const double* C, double* sink, int* grid) {
  switch (variant) {
    case 0: return run(k_gather<4, 4, false>, idx, n, C, sink, grid);
    case 1: return run(k_gather<8, 4, false>, idx, n, C, sink, grid);
    case 2: return run(k_gather<16, 2, false>, idx, n, C, sink, grid);
    case 3: return run(k_gather<4, 6, false>, idx, n, C, sink, grid);
    case 4: return run(k_gather<4, 8, false>, idx, n, C, sink, grid);
    case 5: return run(k_gather<8, 6, false>, idx, n, C, sink, grid);
    case 6: return run(k_gather<4, 4, true>, idx, n, C, sink, grid);
    case 7: return run(k_gather<8, 4, true>, idx, n, C, sink, grid);
    case 8: return run(k_gather_pipe<4, 4>, idx, n, C, sink, grid);
    case 9: return run(k_gather_pipe<8, 3>, idx, n, C, sink, grid);
    case 10: return run(k_gather<2, 8, false>, idx, n, C, sink, grid);
    case 11: return run(k_gather<16, 3, false>, idx, n, C, sink, grid);
  }
  return -2.0f;
}
