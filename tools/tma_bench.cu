// tma_bench.cu -- per-SM TMA streaming throughput from an L2-resident buffer
// (development tool).  Every CTA (one per SM) streams `tiles` 16 KB boxes
// (128 rows x 128 B, SWIZZLE_128B) through an NS-stage ring, like the fused
// kernel's K producer, and reports bytes/cycle/SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <int NS>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int tiles,
                                                      int rows_total, uint64_t* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    fence_mbar_init();
  }
  __syncthreads();
  uint64_t t0 = clk();
  if (warp == 0 && lane == 0) {
    int s = 0, ph = 0;
    for (int t = 0; t < tiles; ++t) {
      mbar_wait_spin(empty + s, ph ^ 1);
      mbar_expect_tx(full + s, 16384);
      const int row = ((blockIdx.x * 977 + t * 128) % (rows_total / 128)) * 128;
      tma_load_3d(smem + s * 16384, &tm, full + s, 0, row, 0);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0, ph = 0;
    for (int t = 0; t < tiles; ++t) {
      mbar_wait_spin(full + s, ph);
      mbar_arrive(empty + s);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    out[blockIdx.x] = clk() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int NS>
void run(EncodeFn enc, void* buf, int rows_total, int nsm, uint64_t* d_out) {
  CUtensorMap tm;
  cuuint64_t dims[3] = {128, (cuuint64_t)rows_total, 1};
  cuuint64_t strides[2] = {128, (cuuint64_t)rows_total * 128};
  cuuint32_t box[3] = {128, 128, 1}, es[3] = {1, 1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = NS * 16384 + 1024;
  cudaFuncSetAttribute(stream_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 2000;
  for (int rep = 0; rep < 2; ++rep) stream_kernel<NS><<<nsm, 64, smem>>>(tm, tiles, rows_total, d_out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  stream_kernel<NS><<<nsm, 64, smem>>>(tm, tiles, rows_total, d_out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  uint64_t h[256];
  cudaMemcpy(h, d_out, nsm * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < nsm; ++i) avg += h[i];
  avg /= nsm;
  printf("NS=%d grid=%d: %.1f B/cycle/SM (clock64), chip %.2f TB/s (events)\n", NS, nsm,
         tiles * 16384.0 / avg, (double)nsm * tiles * 16384 / (ms * 1e-3) / 1e12);
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int rows_total = 16 * 1024 * 1024 / 128;  // 16 MB: L2-resident
  void* buf;
  cudaMalloc(&buf, (size_t)rows_total * 128);
  cudaMemset(buf, 1, (size_t)rows_total * 128);
  uint64_t* d_out;
  cudaMalloc(&d_out, 256 * 8);
  run<2>(enc, buf, rows_total, nsm, d_out);
  run<4>(enc, buf, rows_total, nsm, d_out);
  run<8>(enc, buf, rows_total, nsm, d_out);
  run<4>(enc, buf, rows_total, 1, d_out);
  run<8>(enc, buf, rows_total, 1, d_out);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
