// smem_contention.cu -- do tcgen05 SS-MMA operand reads and LDS gathers share the SM's
// shared-memory data pipe?  One CTA per SM: an issuer streams 128x128x128 i8 SS MMAs while
// W warps run conflict-free LDS.32 (or LDS.U8) loops; each side is timed alone and together.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2511_21513_b200/csrc tools/smem_contention.cu -o tools/smem_contention
#include <cstdint>
#include <cstdio>
#include <utility>

#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

// D[tmem] (+)= A[tmem] * B[smem]^T (TS form), kind::i8
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

template <bool U8, int E>
__device__ __forceinline__ uint32_t lds_one(uint32_t a) {
  uint32_t v;
  if (U8) asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(E * 32));
  else asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(E * 128));
  return v;
}
template <bool U8, int... E>
__device__ __forceinline__ void lds_round(uint32_t a, uint32_t& acc, std::integer_sequence<int, E...>) {
  ((acc += lds_one<U8, E>(a)), ...);
}

struct Opt {
  int tiles;   // MMA tiles (0: no MMA stream)
  int lds_it;  // LDS loop iterations of 32 loads per warp (0: no LDS)
  int nw;      // LDS warps
  int u8;      // 1: LDS.U8 gathers from a 32-byte table; 0: LDS.32 conflict-free
  int ts;      // 1: A operand from TMEM (TS form)
  int n;       // MMA N (128 or 64)
};

__global__ void __launch_bounds__(512, 1) k(Opt o, uint64_t* res, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += 512) reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x1f1f1f1fu;
  if (warp == 14) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  uint64_t t0 = clk();
  if (warp == 15) {
    if (lane == 0 && o.tiles) {
      const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 16384);
      const uint32_t id = idesc_i8(128, o.n, true, true);
      uint64_t da[4], db[4];
      for (int kk = 0; kk < 4; ++kk) { da[kk] = sdesc(sa + kk * 32, 1024, 2); db[kk] = sdesc(sb + kk * 32, 1024, 2); }
      // N = 256: B spans 2 x 16 KB (rows 128.. follow at +16 KB: SBO-strided 8-row groups)
      for (int t = 0; t < o.tiles; ++t)
        for (int kk = 0; kk < 4; ++kk) {
          if (o.ts >= 2) { mma_i8_ss(tmem + (t % 3) * 128, da[kk], db[kk], id, kk > 0); __nanosleep(o.ts); }
          else if (o.ts) mma_i8_ts(tmem + (o.n == 256 ? (t & 1) * 256 : (t % 3) * 128), tmem + (o.n == 256 ? 0 : 384) + kk * 8, db[kk], id, kk > 0);
          else mma_i8_ss(tmem + (o.n == 256 ? (t & 1) * 256 : (t % 3) * 128), da[kk], db[kk], id, kk > 0);
        }
      tc_commit(bar);
      mbar_wait(bar, 0);
      res[blockIdx.x * 4 + 0] = clk() - t0;
    }
  } else if (o.lds_it && (o.nw >= 100 ? (warp < o.nw - 100 && (warp & 3) != 3) : warp < o.nw)) {
    uint32_t acc = 0;
    const uint32_t base = smem_u32(smem + 32768);
    const uint32_t a32 = base + lane * 4, a8 = base + ((lane * 7) & 31);  // 32 distinct bytes of one 32-byte row
    for (int it = 0; it < o.lds_it; ++it) {
      if (o.u8 >= 2) {
        // ALU-only (2) / FMA-only (3) work: 8 independent chains x 4 ops per round
        uint32_t x0 = acc + lane, x1 = x0 * 3, x2 = x0 * 5, x3 = x0 * 7, x4 = x0 + 9, x5 = x0 + 11, x6 = x0 + 13, x7 = x0 + 15;
        float f0 = (float)x0, f1 = (float)x1, f2 = (float)x2, f3 = (float)x3, f4 = (float)x4, f5 = (float)x5, f6 = (float)x6, f7 = (float)x7;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (o.u8 == 2) {
            x0 = max((int)x0 + 3, (int)x1); x1 = max((int)x1 + 5, (int)x2); x2 = max((int)x2 + 7, (int)x3); x3 = max((int)x3 + 9, (int)x4);
            x4 = max((int)x4 + 1, (int)x5); x5 = max((int)x5 + 2, (int)x6); x6 = max((int)x6 + 4, (int)x7); x7 = max((int)x7 + 6, (int)x0);
          } else {
            f0 = fmaf(f0, 1.0001f, f1); f1 = fmaf(f1, 1.0001f, f2); f2 = fmaf(f2, 1.0001f, f3); f3 = fmaf(f3, 1.0001f, f4);
            f4 = fmaf(f4, 1.0001f, f5); f5 = fmaf(f5, 1.0001f, f6); f6 = fmaf(f6, 1.0001f, f7); f7 = fmaf(f7, 1.0001f, f0);
          }
        }
        acc += x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
        acc += __float_as_uint(f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7);
      } else if (o.u8) lds_round<true>(a8, acc, std::make_integer_sequence<int, 32>{});
      else lds_round<false>(a32, acc, std::make_integer_sequence<int, 32>{});
    }
    (void)a8;
    if (acc == 0x12345) sink[0] = acc;
    if (lane == 0 && warp == 0) res[blockIdx.x * 4 + 1] = clk() - t0;
    if (lane == 0 && warp == 3) res[blockIdx.x * 4 + 2] = clk() - t0;
  }
  __syncthreads();
  if (warp == 14) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  uint64_t* res;
  int* sink;
  cudaMalloc(&res, 148 * 4 * 8);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  struct V { int tiles, lds_it, nw, u8, ts, n; };
  const V vs[] = {
      {0, 4000, 4, 2, 0, 128},    {2000, 4000, 4, 2, 0, 128},  {2000, 4000, 4, 2, 20, 128}, {2000, 4000, 4, 2, 50, 128},
      {2000, 4000, 4, 2, 80, 128}, {0, 4000, 12, 2, 0, 128},   {2000, 4000, 12, 2, 0, 128}, {2000, 4000, 12, 2, 50, 128},
      {2000, 0, 0, 0, 50, 128},   {2000, 0, 0, 0, 20, 128},
  };
  for (const V& v : vs) {
    Opt o{v.tiles, v.lds_it, v.nw, v.u8, v.ts, v.n};
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(res, 0, 148 * 4 * 8);
      k<<<148, 512, 96 * 1024>>>(o, res, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    uint64_t h[148 * 4];
    cudaMemcpy(h, res, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0, l = 0, l3 = 0;
    for (int i = 0; i < 148; ++i) { m += h[i * 4]; l += h[i * 4 + 1]; l3 += h[i * 4 + 2]; }
    m /= 148; l /= 148; l3 /= 148;
    printf("tiles %4d pace %2d ns, %2d ALU warps (mode %d): MMA %.0f cyc per tile; ALU round: warp 0 %.2f cyc, warp 3 (issuer's sub-partition) %.2f cyc\n",
           v.tiles, v.ts, v.nw, v.u8, v.tiles ? m / v.tiles : 0.0, v.lds_it ? l / v.lds_it : 0.0, v.lds_it ? l3 / v.lds_it : 0.0);
  }
  return 0;
}
