// pipe_bench.cu -- the fused kernel's QK^T -> TMEM -> softmax-warpgroup round trip in
// isolation (development tool): one issuer warp, NWG consumer warpgroups, S buffers
// in TMEM, K/Q tiles static in shared memory, 148 CTAs.  Prints cycles per tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_2511_21513_b200/csrc tools/pipe_bench.cu -o tools/pipe_bench
#include <climits>
#include <cstdint>
#include <cstdio>

#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

struct Opt {
  int nbuf;      // S buffers (= consumer warpgroups), <= 4
  int ncols;     // key tile width N (64 / 128 / 256)
  int work;      // 0: none, 1: pass-1 max/min, 2: pass-2-like idx+lut sum
  int early;     // 1: arrive s_free after the first half (timing only)
  int spin;      // issuer spin-waits
  int ntiles;
  int mode;      // 0: pipeline; 1: issuer only (no waits, no consumers); 2: no MMA (issuer arrives)
  int kst;       // MMA K steps per tile (4 = d 128)
  int cmode;     // consumer: 0 normal; 1 no TMEM loads; 2 spin waits; 3 no tcgen05 fences
  int lean;      // issuer: lane-0-only loop, counters instead of modulo, unrolled K steps
  int kload;     // 1: a producer warp streams 16 KB K tiles (bulk copies from L2) through a 4-stage ring
  int nwg;       // consumer warpgroups (0: = nbuf); WG w takes tiles w, w + nwg, ... (buffer t % nbuf)
};

__device__ uint64_t g_tr[4][768];  // CTA 0 event clocks: issuer start, issuer issued, consumer woke, consumer freed

__global__ void __launch_bounds__(544, 1) pipe_kernel(Opt o, uint64_t* res, int* sink, const uint8_t* kglob) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bars[24];
  __shared__ uint32_t tslot;
  __shared__ uint8_t lut8[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NB = o.nbuf;
  uint64_t* s_full = bars;
  uint64_t* s_free = bars + 8;
  const int NWGC = o.nwg ? o.nwg : o.nbuf;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(s_full + i, 1); mbar_init(s_free + i, 4); }
    for (int i = 16; i < 24; ++i) mbar_init(bars + i, 1);  // k_full[4], k_empty[4]
    fence_mbar_init();
  }
  if (threadIdx.x < 32) lut8[threadIdx.x] = (uint8_t)(255 >> (threadIdx.x / 4));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x3f3f3f3fu;
  const int issuer_warp = 4 * NWGC;
  if (warp == issuer_warp) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int T = o.ntiles;
  const uint32_t bcols = (uint32_t)o.ncols;
  uint64_t t0 = clk();
  uint64_t* k_full = bars + 16;
  uint64_t* k_empty = bars + 20;
  if (warp == issuer_warp + 1) {
    if (o.kload && lane == 0) {  // K producer: 16 KB per tile from an L2-resident buffer
      uint32_t kph = 0;
      for (int t = 0; t < T; ++t) {
        const int st = t & 3;
        if (t >= 4) { mbar_wait(k_empty + st, (kph >> st) & 1u); kph ^= 1u << st; }
        mbar_expect_tx(k_full + st, 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                     ::"r"(smem_u32(smem + 32768 + st * 16384)),
                     "l"(kglob + ((size_t)(blockIdx.x * 7 + t) % 512) * 16384), "r"(smem_u32(k_full + st))
                     : "memory");
      }
    }
    __syncwarp();
  } else if (warp == issuer_warp && o.lean) {
    if (lane == 0) {
      const uint32_t idq = idesc_i8(128, o.ncols > 256 ? 256 : o.ncols, true, true);
      const uint64_t dq = sdesc(smem_u32(smem), 1024, 2);
      uint64_t dk = sdesc(smem_u32(smem + 16384), 1024, 2);
      uint32_t ph = 0, kph = 0;
      int w = 0;
      uint32_t dt = tmem;
      for (int t = 0; t < T; ++t) {
        if (t >= NB && o.mode != 1) {
          mbar_wait(s_free + w, (ph >> w) & 1u);
          ph ^= 1u << w;
        }
        if (o.kload) {
          const int st = t & 3;
          mbar_wait(k_full + st, (kph >> st) & 1u);
          kph ^= 1u << st;
          dk = sdesc(smem_u32(smem + 32768 + st * 16384), 1024, 2);
        }
        tc_fence_after();
        if (o.mode == 2) {
          mbar_arrive(s_full + w);
        } else {
          mma_i8_ss(dt, dq, dk, idq, 0u);
          mma_i8_ss(dt, dq + 2, dk + 2, idq, 1u);
          mma_i8_ss(dt, dq + 4, dk + 4, idq, 1u);
          mma_i8_ss(dt, dq + 6, dk + 6, idq, 1u);
          if (o.kload) tc_commit(k_empty + (t & 3));
          if (o.mode == 0) tc_commit(s_full + w);
        }
        if (++w == NB) { w = 0; dt = tmem; } else dt += bcols;
      }
      if (o.mode == 1) {
        tc_commit(s_full);
        mbar_wait(s_full, 0);
        res[blockIdx.x] = clk() - t0;
      }
    }
    __syncwarp();
  } else if (warp == issuer_warp) {
    const uint32_t idq = idesc_i8(128, o.ncols > 256 ? 256 : o.ncols, true, true);
    const uint64_t dq = sdesc(smem_u32(smem), 1024, 2), dk = sdesc(smem_u32(smem + 16384), 1024, 2);
    uint32_t ph = 0;
    for (int t = 0; t < T; ++t) {
      const int w = t % NB;
      if (blockIdx.x == 0 && lane == 0 && t < 768) g_tr[0][t] = clk();
      if (t >= NB && o.mode != 1) {
        if (o.spin) mbar_wait_spin(s_free + w, (ph >> w) & 1u);
        else mbar_wait(s_free + w, (ph >> w) & 1u);
        ph ^= 1u << w;
      }
      tc_fence_after();
      if (elect_one()) {
        if (o.mode == 2) {
          mbar_arrive(s_full + w);
        } else {
          for (int kk = 0; kk < o.kst; ++kk) mma_i8_ss(tmem + w * bcols, dq + 2 * kk, dk + 2 * kk, idq, kk > 0);
          if (o.mode == 0) tc_commit(s_full + w);
        }
      }
      __syncwarp();
      if (blockIdx.x == 0 && lane == 0 && t < 768) g_tr[1][t] = clk();
    }
    if (o.mode == 1) {
      if (elect_one()) tc_commit(s_full);
      __syncwarp();
      mbar_wait(s_full, 0);
      if (lane == 0) res[blockIdx.x] = clk() - t0;
    }
  } else if (warp < 4 * NWGC && o.mode != 1) {
    const int wg = warp >> 2, quad = warp & 3;
    const uint32_t base0 = tmem + ((uint32_t)(quad * 32) << 16);
    int32_t mx = INT_MIN, mn = INT_MAX;
    uint32_t S = 0;
    uint32_t ph = 0;
    const uint32_t M = 0x2468acefu;
    for (int t = wg; t < T; t += NWGC) {
      const int bf = t % NB;
      const uint32_t base = base0 + bf * bcols;
      if (o.cmode == 2) mbar_wait_spin(s_full + bf, (ph >> bf) & 1u);
      else mbar_wait(s_full + bf, (ph >> bf) & 1u);
      ph ^= 1u << bf;
      if (blockIdx.x == 0 && quad == 0 && lane == 0 && t < 768) g_tr[2][t] = clk();
      if (o.cmode != 3) tc_fence_after();
      const int nh = o.ncols / 64;
#pragma unroll 1
      for (int hb = 0; hb < nh; ++hb) {
        uint32_t va[32], vb[32];
        if (o.cmode == 1) {
          for (int e = 0; e < 32; ++e) { va[e] = e * hb; vb[e] = e + hb; }
        } else {
          tmem_ld64(base + hb * 64, va, vb);
        }
        if ((o.early && hb == 0) || (!o.early && hb == nh - 1)) {
          if (o.cmode != 3) tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + bf);
          if (blockIdx.x == 0 && quad == 0 && lane == 0 && t < 768) g_tr[3][t] = clk();
        }
        if (o.work == 1) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            mx = max(mx, max(max((int32_t)va[e], (int32_t)va[e + 1]), max((int32_t)vb[e], (int32_t)vb[e + 1])));
            mn = min(mn, min(min((int32_t)va[e], (int32_t)va[e + 1]), min((int32_t)vb[e], (int32_t)vb[e + 1])));
          }
        } else if (o.work == 2) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            S += (uint32_t)lut8[(__umulhi(va[e] * 62u + 7u, M) >> 27)] +
                 (uint32_t)lut8[(__umulhi(vb[e] * 62u + 7u, M) >> 27)];
        } else {
          S += va[0] + vb[31];
        }
      }
    }
    if (mx == 12345 || mn == 12345 || S == 12345u) sink[threadIdx.x] = mx + mn + (int)S;
  }
  tc_fence_before();
  __syncthreads();
  uint64_t t1 = clk();
  if (threadIdx.x == 0 && o.mode != 1) res[blockIdx.x] = t1 - t0;
  if (warp == issuer_warp) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  uint64_t* d_res;
  int* d_sink;
  cudaMalloc(&d_res, 148 * 8);
  cudaMalloc(&d_sink, 4096 * 4);
  cudaFuncSetAttribute(pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  uint8_t* kglob;
  cudaMalloc(&kglob, 512 * 16384);
  cudaMemset(kglob, 0x11, 512 * 16384);
  struct V { int nbuf, ncols, work, early, spin, mode, kst, cmode, lean, kload, nwg; };
  const V vs[] = {
      {3, 128, 0, 0, 0, 0, 4, 0, 1, 0, 3}, {3, 128, 0, 0, 0, 0, 4, 0, 1, 1, 3},
      {3, 128, 1, 0, 0, 0, 4, 0, 1, 0, 3}, {3, 128, 1, 0, 0, 0, 4, 0, 1, 1, 3},
      {3, 128, 2, 0, 0, 0, 4, 0, 1, 0, 3}, {3, 128, 2, 0, 0, 0, 4, 0, 1, 1, 3},
      {3, 128, 0, 0, 0, 1, 4, 0, 1, 0, 3}, {3, 128, 0, 0, 0, 1, 4, 0, 1, 1, 3},
  };
  for (const V& v : vs) {
    Opt o{v.nbuf, v.ncols, v.work, v.early, v.spin, 3 * 4 * 64 * (128 / v.ncols), v.mode, v.kst, v.cmode, v.lean, v.kload, v.nwg};
    const int nthreads = 128 * (v.nwg ? v.nwg : v.nbuf) + 64;
    pipe_kernel<<<148, nthreads, 112 * 1024>>>(o, d_res, d_sink, kglob);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[148];
    cudaMemcpy(h, d_res, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    const double per128 = (sum / 148) / o.ntiles * (128.0 / v.ncols);
    static uint64_t tr[4][768];
    cudaMemcpyFromSymbol(tr, g_tr, sizeof(tr));
    if (v.mode != 1) {
      double a = 0, b = 0, c = 0, d = 0; int n = 0;
      for (int t = 100; t < 700; ++t) {
        a += tr[1][t] - tr[0][t];          // issuer: loop top -> issued (incl. s_free wait)
        b += tr[2][t] - tr[1][t];          // issued -> consumer woke
        c += tr[3][t] - tr[2][t];          // consumer woke -> s_free arrive
        d += tr[0][t + 1] - tr[1][t];      // issuer: issued -> next loop top
        ++n;
      }
      printf("   issuer wait+issue %.0f | issue->wake %.0f | wake->free %.0f | issuer gap %.0f\n", a / n, b / n, c / n, d / n);
    }
    printf("kload %d nwg %d lean %d cmode %d mode %d ksteps %d nbuf %d N %3d work %d early %d spin %d: %s  %.0f cycles per tile, %.0f per 128 keys\n",
           v.kload, v.nwg, v.lean, v.cmode, v.mode, v.kst, v.nbuf, v.ncols, v.work, v.early, v.spin, cudaGetErrorString(e), (sum / 148) / o.ntiles, per128);
  }
  return 0;
}
