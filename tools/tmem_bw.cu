// tmem_bw.cu -- TMEM read bandwidth per SM (tcgen05.ld 32x32b.x32) vs warps per CTA
// (development tool; sizes the S-tile read cost of the fused kernel's passes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -Ipaper_2511_21513_b200/csrc tools/tmem_bw.cu -o tools/tmem_bw
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// mode 0: 2 x (32x32b.x32) then wait; mode 1: 4 x x32 then wait; mode 2: 1 x x32 then wait
template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_bw_kernel(uint64_t* res, uint32_t* sink, int iters) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) & 3) * 128;
  uint32_t acc = 0;
  __syncthreads();
  uint64_t t0 = clk();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int c = 0; c < 128; c += (MODE == 1 ? 128 : (MODE == 0 ? 64 : 32))) {
      uint32_t a[32], b[32];
      if (MODE == 2) {
        tmem_ld32_nowait(base + c, a);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= a[e];
      } else if (MODE == 0) {
        tmem_ld64(base + c, a, b);
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= a[e] + b[e];
      } else {
        uint32_t x[32], y[32];
        tmem_ld32_nowait(base + c, a);
        tmem_ld32_nowait(base + c + 32, b);
        tmem_ld32_nowait(base + c + 64, x);
        tmem_ld32_nowait(base + c + 96, y);
        tmem_wait_ld64(a, b);
        tmem_wait_ld64(x, y);
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= (a[e] + b[e]) ^ (x[e] + y[e]);
      }
    }
  }
  __syncthreads();
  uint64_t t1 = clk();
  if (threadIdx.x == 0) res[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(int nthreads, uint64_t* d_res, uint32_t* d_sink) {
  const int iters = 2000;
  tmem_bw_kernel<MODE><<<148, nthreads>>>(d_res, d_sink, iters);
  cudaError_t e = cudaDeviceSynchronize();
  uint64_t h[148];
  cudaMemcpy(h, d_res, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  // each warp reads 32 lanes x 128 cols x 4 B per iteration
  const double bytes = (double)(nthreads / 32) * 32 * 128 * 4 * iters;
  printf("mode %d warps %2d: %s  %.1f B/cycle/SM  (%.0f cycles per 64 KB)\n", MODE, nthreads / 32,
         cudaGetErrorString(e), bytes / mx, 65536.0 / (bytes / mx));
}

int main() {
  uint64_t* d_res;
  uint32_t* d_sink;
  cudaMalloc(&d_res, 148 * 8);
  cudaMalloc(&d_sink, 4096);
  for (int nt : {128, 256, 384, 512}) {
    run<0>(nt, d_res, d_sink);
    run<1>(nt, d_res, d_sink);
    run<2>(nt, d_res, d_sink);
  }
  return 0;
}
