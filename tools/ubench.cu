// ubench.cu -- latency microbenchmarks for the fused kernel's primitives on sm_100a
// (development tool; numbers feed DESIGN.md).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include \
//        -I../paper_2511_21513_b200/csrc tools/ubench.cu -o tools/ubench
#include <cstdio>
#include <cstdint>

#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// results[0..] : cycles
__global__ void __launch_bounds__(256, 1) ubench_kernel(uint64_t* res, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(bar + i, 1);
    mbar_init(bar + 3, 3);
    for (int i = 4; i < 8; ++i) mbar_init(bar + i, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 32768 / 4; i += 256) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (warp == 2) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 16384);
  const uint32_t idq = idesc_i8(128, 128, true, true);
  // (a) MMA 128x128x128 int8 issue -> commit-arrive latency, and back-to-back throughput
  if (warp == 1 && lane == 0) {
    uint32_t ph = 0;
    uint64_t best = ~0ull, sum = 0;
    for (int it = 0; it < iters; ++it) {
      uint64_t t0 = clk();
      for (int kk = 0; kk < 4; ++kk)
        mma_i8_ss(tmem, sdesc(sa + kk * 32, 1024, 2), sdesc(sb + kk * 32, 1024, 2), idq, kk > 0);
      tc_commit(bar + 0);
      mbar_wait(bar + 0, ph);
      ph ^= 1;
      uint64_t dt = clk() - t0;
      sum += dt;
      best = dt < best ? dt : best;
    }
    res[0] = best;
    res[1] = sum / iters;
    // 8 tiles back to back, one commit
    uint64_t t0 = clk();
    for (int t = 0; t < 8; ++t)
      for (int kk = 0; kk < 4; ++kk)
        mma_i8_ss(tmem + (t & 3) * 128, sdesc(sa + kk * 32, 1024, 2), sdesc(sb + kk * 32, 1024, 2), idq, kk > 0);
    tc_commit(bar + 0);
    mbar_wait(bar + 0, ph);
    ph ^= 1;
    res[2] = clk() - t0;
    // N=64 tiles back to back (32 tiles), one commit
    const uint32_t id64 = idesc_i8(128, 64, true, true);
    t0 = clk();
    for (int t = 0; t < 32; ++t)
      for (int kk = 0; kk < 4; ++kk)
        mma_i8_ss(tmem + (t & 3) * 64, sdesc(sa + kk * 32, 1024, 2), sdesc(sb + kk * 32, 1024, 2), id64, kk > 0);
    uint64_t t_issue = clk() - t0;
    tc_commit(bar + 0);
    mbar_wait(bar + 0, ph);
    ph ^= 1;
    res[6] = clk() - t0;
    res[7] = t_issue;
    // cost of a wait on an already-completed phase
    t0 = clk();
    for (int r = 0; r < 16; ++r) mbar_wait(bar + 0, ph ^ 1);
    res[9] = (clk() - t0) / 16;
    // issue cost of 4 MMAs + 2 commits with precomputed descriptors
    uint64_t da[4], db[4];
    for (int kk = 0; kk < 4; ++kk) { da[kk] = sdesc(sa + kk * 32, 1024, 2); db[kk] = sdesc(sb + kk * 32, 1024, 2); }
    t0 = clk();
    for (int kk = 0; kk < 4; ++kk) mma_i8_ss(tmem, da[kk], db[kk], id64, kk > 0);
    tc_commit(bar + 2);
    tc_commit(bar + 0);
    res[10] = clk() - t0;
    mbar_wait(bar + 0, ph);
    ph ^= 1;
  }
  __syncthreads();
  // (a3) issue rate of the fused kernel's QK^T step: 24 tiles of {4 MMA (N=128) into a
  // rotating 128-column buffer + 2 commits}, no waits; then completion
  if (warp == 1 && lane == 0) {
    uint64_t da[4], db[4];
    for (int kk = 0; kk < 4; ++kk) { da[kk] = sdesc(sa + kk * 32, 1024, 2); db[kk] = sdesc(sb + kk * 32, 1024, 2); }
    uint64_t t0 = clk(), t3 = 0;
    for (int t = 0; t < 24; ++t) {
      for (int kk = 0; kk < 4; ++kk) mma_i8_ss(tmem + (t % 3) * 128, da[kk], db[kk], idq, kk > 0);
      tc_commit(bar + 4);
      tc_commit(bar + 5);
      if (t == 2) t3 = clk();
    }
    uint64_t t1 = clk();
    tc_commit(bar + 6);
    mbar_wait(bar + 6, 0);
    uint64_t t2 = clk();
    res[16] = t1 - t0;  // issue time, 24 tiles
    res[17] = t3 - t0;  // first 3 tiles
    res[18] = t2 - t0;  // to completion
    // same with 1 commit per tile
    t0 = clk();
    for (int t = 0; t < 24; ++t) {
      for (int kk = 0; kk < 4; ++kk) mma_i8_ss(tmem + (t % 3) * 128, da[kk], db[kk], idq, kk > 0);
      tc_commit(bar + 4);
    }
    t1 = clk();
    tc_commit(bar + 6);
    mbar_wait(bar + 6, 1);
    res[19] = t1 - t0;
    res[20] = clk() - t0;
    // no commits inside
    t0 = clk();
    for (int t = 0; t < 24; ++t)
      for (int kk = 0; kk < 4; ++kk) mma_i8_ss(tmem + (t % 3) * 128, da[kk], db[kk], idq, kk > 0);
    t1 = clk();
    tc_commit(bar + 6);
    mbar_wait(bar + 6, 0);
    res[21] = t1 - t0;
    res[22] = clk() - t0;
  }
  __syncthreads();
  // (a2) 3 warps issuing N=64 MMAs concurrently (32 tiles each) into disjoint TMEM
  if ((warp == 1 || warp == 3 || warp == 5) && lane == 0) {
    const uint32_t id64 = idesc_i8(128, 64, true, true);
    const int wsel = warp == 1 ? 0 : (warp == 3 ? 1 : 2);
    uint64_t t0 = clk();
    for (int t = 0; t < 32; ++t)
      for (int kk = 0; kk < 4; ++kk)
        mma_i8_ss(tmem + wsel * 128 + (t & 1) * 64, sdesc(sa + kk * 32, 1024, 2), sdesc(sb + kk * 32, 1024, 2), id64, kk > 0);
    tc_commit(bar + 3);
    res[11 + wsel] = clk() - t0;
  }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_wait(bar + 3, 0); }
  __syncthreads();
  // (b) tcgen05.ld 32x32b.x32 latency (fused wait), and 2 x32 + one wait
  if (warp == 4) {
    uint32_t v[32], w[32];
    uint64_t best = ~0ull, best2 = ~0ull;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
      uint64_t t0 = clk();
      tmem_ld32(tmem + (it & 3) * 32, v);
      acc += v[0] + v[31];
      uint64_t dt = clk() - t0;
      best = dt < best ? dt : best;
      t0 = clk();
      tmem_ld64(tmem + (it & 1) * 64, v, w);
      acc += v[3] + w[7];
      dt = clk() - t0;
      best2 = dt < best2 ? dt : best2;
    }
    if (lane == 0) { res[3] = best; res[4] = best2; res[14] = acc; }
  }
  __syncthreads();
  // (c) mbarrier arrive (warp 5) -> wake (warp 6) latency
  if (warp == 5 || warp == 6) {
    uint32_t ph = 0;
    uint64_t best = ~0ull;
    for (int it = 0; it < iters; ++it) {
      __syncwarp();
      if (warp == 5) {
        if (lane == 0) {
          volatile uint64_t t0 = clk();
          res[8] = t0;
          mbar_arrive(bar + 1);
        }
      } else {
        if (lane == 0) {
          mbar_wait(bar + 1, ph);
          uint64_t t1 = clk();
          __threadfence_block();
          uint64_t dt = t1 - *((volatile uint64_t*)(res + 8));
          best = dt < best ? dt : best;
        }
      }
      ph ^= 1;
      asm volatile("bar.sync 2, 64;");
    }
    if (warp == 6 && lane == 0) res[5] = best;
  }
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 32 * sizeof(uint64_t));
  cudaMemset(d, 0, 32 * sizeof(uint64_t));
  cudaFuncSetAttribute(ubench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  ubench_kernel<<<1, 256, 40000>>>(d, 64);
  cudaError_t e = cudaDeviceSynchronize();
  uint64_t h[32] = {0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  printf("MMA 128x128x128 i8 issue->commit wait: best %llu avg %llu cycles\n", (unsigned long long)h[0],
         (unsigned long long)h[1]);
  printf("8 MMA tiles back-to-back + commit: %llu cycles (%.1f/tile)\n", (unsigned long long)h[2],
         h[2] / 8.0);
  printf("tcgen05.ld x32 + wait: %llu cycles; 2x x32 + wait: %llu cycles\n", (unsigned long long)h[3],
         (unsigned long long)h[4]);
  printf("mbarrier arrive -> wake (other warp): %llu cycles\n", (unsigned long long)h[5]);
  printf("32 N=64 tiles back-to-back: total %llu (%.1f/tile), issue-only %llu (%.1f/tile)\n",
         (unsigned long long)h[6], h[6] / 32.0, (unsigned long long)h[7], h[7] / 32.0);
  printf("wait on completed phase: %llu cycles; issue 4 MMA + 2 commits: %llu cycles\n",
         (unsigned long long)h[9], (unsigned long long)h[10]);
  printf("3 warps x 32 N=64 tiles concurrently: issue %llu %llu %llu cycles (%.1f/tile each)\n",
         (unsigned long long)h[11], (unsigned long long)h[12], (unsigned long long)h[13], h[11] / 32.0);
  printf("24 tiles {4 MMA + 2 commits}: issue %llu (%.1f/tile; first 3 tiles %llu), to completion %llu (%.1f/tile)\n",
         (unsigned long long)h[16], h[16] / 24.0, (unsigned long long)h[17], (unsigned long long)h[18], h[18] / 24.0);
  printf("24 tiles {4 MMA + 1 commit}: issue %llu (%.1f/tile), completion %llu\n", (unsigned long long)h[19],
         h[19] / 24.0, (unsigned long long)h[20]);
  printf("24 tiles {4 MMA}: issue %llu (%.1f/tile), completion %llu\n", (unsigned long long)h[21], h[21] / 24.0,
         (unsigned long long)h[22]);
  return 0;
}
