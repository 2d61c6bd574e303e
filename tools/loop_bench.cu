// loop_bench.cu -- the fused kernel's per-logit softmax loops in isolation (development
// tool): NW warps per CTA (1 CTA per SM, 148 CTAs) read 128x128 int32 tiles from TMEM
// (no MMA running) and run one pass body on them.  Prints cycles per 128-key tile per
// warp for 4 / 8 / 12 / 16 warps (1-4 per SM sub-partition), i.e. the issue rate a
// softmax warp reaches alone and next to its neighbours.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Iinclude \
//        -Ipaper_2511_21513_b200/csrc tools/loop_bench.cu -o tools/loop_bench
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "params.cuh"
#include "ptx.cuh"

using namespace ia;

__device__ __forceinline__ uint64_t clk() {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ float fma_rz(float a, float b, float c) {
  float r;
  asm("fma.rz.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// d = a * b + c on two packed f32 lanes (sm_100 FFMA2)
__device__ __forceinline__ void fma2(float& d0, float& d1, float a0, float a1, float b, float c) {
  uint64_t a, bb, cc, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(bb), "l"(cc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float c) {
  uint64_t a, cc, d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cc) : "f"(c));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(cc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}

struct Args {
  ia_head_params hp;
  int iters, nwarps, m, c_span;  // logits drawn in [m - c_span, m]
  uint64_t* res;
  uint32_t* sink;
};

// MODE 0: no work (TMEM reads only)   1: pass 1 max+min   2: pass 2 unclipped (SHF form)
// 3: pass 2 clipped   4: pass 2 unclipped, shift as IMAD.HI   5: pass 3 unclipped magic9
// 6: pass 3 clipped magic9   7: pass 2 unclipped + IMAD accumulate
// 8: pass 2 with 32-column software-pipelined TMEM loads
template <int MODE>
__global__ void __launch_bounds__(512, 1) loop_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint8_t lut8[256];
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem);            // [56][128] u32
  uint8_t* ptile = smem + 56 * 512;                              // 3 x 16 KB P^ tiles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    lut8[t] = t < 32 ? (uint8_t)(255 >> (t / 4)) : 0;
  for (int t = threadIdx.x; t < 56 * 128; t += blockDim.x) tab[t] = t < 20 * 128 ? (uint32_t)(t & 255) : 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int wg = (warp >> 2) % 3, quad = warp & 3;
  const int row = quad * 32 + lane;
  const uint32_t s_base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(wg * 128);
  if (warp < 12) {  // fill the three S buffers once
    uint32_t h = (uint32_t)(blockIdx.x * 977 + threadIdx.x * 131 + 7);
    for (int c = 0; c < 128; c += 32) {
      uint32_t v[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        h = h * 1664525u + 1013904223u;
        v[e] = (uint32_t)(a.m - (int)((h >> 8) % (uint32_t)(a.c_span + 1)));
      }
      tmem_st32(s_base + c, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp < a.nwarps) {
  const ia_head_params hp = a.hp;
  const uint32_t k = 31;
  IdxMap im;
  im.init(a.m, hp, k);
  const uint32_t tab0 = smem_u32(tab), row4 = (uint32_t)row * 4u;
  const uint32_t m9 = hp.magic9;
  const uint32_t p_row = smem_u32(ptile + wg * 16384) + (uint32_t)row * 128;
  const uint32_t p_xor = (uint32_t)(row & 7);
  uint32_t S = 0;
  int32_t mx = INT_MIN, mn = INT_MAX;
  uint32_t mC = (uint32_t)a.m + 0x4B000000u;  // bits of 2^23 + (m - a) after one subtract
  asm volatile("" : "+r"(mC));
  float rr = 31.0f / (float)hp.c_eff, mf = (float)a.m;
  asm volatile("" : "+f"(rr), "+f"(mf));
  const uint32_t lutoff = smem_u32(lut8) - 0x4B000000u;
  uint32_t mI = (uint32_t)a.m;
  asm volatile("" : "+r"(mI));
  float lutden = __uint_as_float(smem_u32(lut8)), tabden = __uint_as_float(tab0 + 256u), rr9 = rr * 512.0f;
  asm volatile("" : "+f"(lutden), "+f"(tabden), "+f"(rr9));
  const uint32_t taboff = tab0 - 0x46800000u;
  uint32_t one = 1;
  asm volatile("" : "+r"(one));
  const uint64_t t0 = clk();
  for (int it = 0; it < a.iters; ++it) {
    if (MODE == 8) {
      uint32_t b0[32], b1[32];
      tmem_ld32(s_base, b0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t(&cur)[32] = (c & 1) ? b1 : b0;
        uint32_t(&nxt)[32] = (c & 1) ? b0 : b1;
        if (c < 3) tmem_ld32_nowait(s_base + 32 * (c + 1), nxt);
#pragma unroll
        for (int e = 0; e < 32; e += 2)
          S += (uint32_t)lut8[im.idx_u((int32_t)cur[e])] + (uint32_t)lut8[im.idx_u((int32_t)cur[e + 1])];
        if (c < 3) asm volatile("tcgen05.wait::ld.sync.aligned;" : IA_R32(nxt) : : "memory");
      }
      continue;
    }
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      uint32_t va[32], vb[32];
      tmem_ld64(s_base + hb * 64, va, vb);
      if (MODE == 0) {
        S += va[0] ^ vb[31];
      } else if (MODE == 1) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          mx = max(mx, max(max((int32_t)va[e], (int32_t)va[e + 1]), max((int32_t)vb[e], (int32_t)vb[e + 1])));
          mn = min(mn, min(min((int32_t)va[e], (int32_t)va[e + 1]), min((int32_t)vb[e], (int32_t)vb[e + 1])));
        }
      } else if (MODE == 2) {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          S += (uint32_t)lut8[im.idx_u((int32_t)va[e])] + (uint32_t)lut8[im.idx_u((int32_t)vb[e])];
      } else if (MODE == 3) {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          S += (uint32_t)lut8[im.idx_s((int32_t)va[e])] + (uint32_t)lut8[im.idx_s((int32_t)vb[e])];
      } else if (MODE == 4) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const uint32_t na = im.base + im.nk2 * va[e], nb = im.base + im.nk2 * vb[e];
          S += (uint32_t)lut8[__umulhi(__umulhi(na, im.magic), im.mul2)] +
               (uint32_t)lut8[__umulhi(__umulhi(nb, im.magic), im.mul2)];
        }
      } else if (MODE == 7) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          S = (uint32_t)lut8[im.idx_u((int32_t)va[e])] * one + S;
          S = (uint32_t)lut8[im.idx_u((int32_t)vb[e])] * one + S;
        }
      } else if (MODE == 9) {
        // float form: bits(2^23 + delta) by one IMAD, delta_f by FADD, idx in the mantissa of
        // fma(delta_f, r, 2^23); the LUT address is bits + const
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float da = __fadd_rn(__uint_as_float(mC - va[e]), -8388608.0f);
          const float db = __fadd_rn(__uint_as_float(mC - vb[e]), -8388608.0f);
          const uint32_t ia = __float_as_uint(__fmaf_rn(da, rr, 8388608.0f));
          const uint32_t ib = __float_as_uint(__fmaf_rn(db, rr, 8388608.0f));
          S += lds_u8(ia + lutoff) + lds_u8(ib + lutoff);
        }
      } else if (MODE == 10) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float da = __fadd_rn(mf, -__int2float_rn((int32_t)va[e]));
          const float db = __fadd_rn(mf, -__int2float_rn((int32_t)vb[e]));
          const uint32_t ia = __float_as_uint(__fmaf_rn(da, rr, 8388608.0f));
          const uint32_t ib = __float_as_uint(__fmaf_rn(db, rr, 8388608.0f));
          S += lds_u8(ia + lutoff) + lds_u8(ib + lutoff);
        }
      } else if (MODE == 11) {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float da, db, fa, fb;
          add2(da, db, __uint_as_float(mC - va[e]), __uint_as_float(mC - vb[e]), -8388608.0f);
          fma2(fa, fb, da, db, rr, 8388608.0f);
          S += lds_u8(__float_as_uint(fa) + lutoff) + lds_u8(__float_as_uint(fb) + lutoff);
        }
      } else if (MODE == 14) {
        // denormal form: the integer delta IS the f32 denormal delta * 2^-149; one FMA with a
        // denormal addend leaves  RN(delta * r) + lut address  in the result's bit pattern
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float fa, fb;
          fma2(fa, fb, __uint_as_float(mI - va[e]), __uint_as_float(mI - vb[e]), rr, lutden);
          S += lds_u8(__float_as_uint(fa)) + lds_u8(__float_as_uint(fb));
        }
      } else if (MODE == 15) {
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t* v4 = q < 8 ? &va[4 * q] : &vb[4 * (q - 8)];
          uint32_t pw[4];
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            uint64_t a2, b2, c2, d2;
            float f0, f1;
            asm("mov.b64 %0, {%1, %2};" : "=l"(a2) : "r"(mI - v4[e]), "r"(mI - v4[e + 1]));
            asm("mov.b64 %0, {%1, %1};" : "=l"(b2) : "f"(rr9));
            asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(tabden));
            asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(d2) : "l"(a2), "l"(b2), "l"(c2));
            asm("mov.b64 {%0, %1}, %2;" : "=f"(f0), "=f"(f1) : "l"(d2));
            pw[e] = lds_u32(and_or(__float_as_uint(f0), 0xFFFFFE00u, row4));
            pw[e + 1] = lds_u32(and_or(__float_as_uint(f1), 0xFFFFFE00u, row4));
          }
          pk[q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040), __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t x = (uint32_t)(4 * hb + u);
          sts128(p_row + ((x ^ p_xor) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      } else if (MODE == 12 || MODE == 13) {
        uint32_t pk[16];
        const uint32_t nk2 = im.nk2, base = im.base;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t* v4 = q < 8 ? &va[4 * q] : &vb[4 * (q - 8)];
          uint32_t pw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (MODE == 12) {
              const float df = __fadd_rn(__uint_as_float(mC - v4[e]), -8388608.0f);
              const uint32_t hb9 = __float_as_uint(fma_rz(df, rr, 16384.5f));
              pw[e] = lds_u32(taboff + and_or(hb9, 0xFFFFFE00u, row4));
            } else {
              const uint32_t n = base + nk2 * v4[e];
              pw[e] = lds_u32(tab0 + and_or(__umulhi(n, m9), 0xFFFFFE00u, row4));
            }
          }
          if (MODE == 13) pk[q] = (pw[1] * 256u + pw[0]) + (pw[3] * 256u + pw[2]) * 65536u;
          else pk[q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040), __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t x = (uint32_t)(4 * hb + u);
          sts128(p_row + ((x ^ p_xor) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      } else if (MODE == 5 || MODE == 6) {
        uint32_t pk[16];
        const uint32_t nk2 = im.nk2, base = im.base;
        const int32_t lo = im.lo;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t* v4 = q < 8 ? &va[4 * q] : &vb[4 * (q - 8)];
          uint32_t pw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int32_t x = MODE == 6 ? max((int32_t)v4[e], lo) : (int32_t)v4[e];
            const uint32_t n = base + nk2 * (uint32_t)x;
            pw[e] = lds_u32(tab0 + and_or(__umulhi(n, m9), 0xFFFFFE00u, row4));
          }
          pk[q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040), __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t x = (uint32_t)(4 * hb + u);
          sts128(p_row + ((x ^ p_xor) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
    }
  }
  const uint64_t t1 = clk();
  if (lane == 0) a.res[blockIdx.x * 16 + warp] = t1 - t0;
  a.sink[blockIdx.x * 512 + threadIdx.x] = S + (uint32_t)mx + (uint32_t)mn;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
static void run(Args a, const char* name) {
  const size_t smem = 56 * 512 + 3 * 16384 + 1024;
  cudaFuncSetAttribute(loop_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint64_t* h = (uint64_t*)malloc(148 * 16 * 8);
  printf("%-44s", name);
  for (int nw = 4; nw <= 12; nw += 4) {
    a.nwarps = nw;
    cudaMemset(a.res, 0, 148 * 16 * 8);
    loop_kernel<MODE><<<148, 512, smem>>>(a);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf(" error: %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(h, a.res, 148 * 16 * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    int n = 0;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < nw; ++w) { s += (double)h[b * 16 + w]; ++n; }
    printf("  %2d warps: %7.1f cyc/tile/warp (%6.1f /tile/SMSP)", nw, s / n / a.iters, s / n / a.iters / (nw / 4));
  }
  printf("\n");
  free(h);
}

int main(int argc, char** argv) {
  Args a;
  const int64_t c_int = argc > 1 ? atoll(argv[1]) : 48161;
  fill_head_params(c_int, 2 * 128 * 127 * 127, 32, &a.hp);
  a.iters = 2000;
  a.m = 200000;
  a.c_span = (int)(c_int < 1000000 ? c_int : 1000000);  // every logit inside the clip range
  cudaMalloc(&a.res, 148 * 16 * 8);
  cudaMalloc(&a.sink, 148 * 512 * 4);
  printf("c_int %lld use32 %d unc32 %d shift %d magic9 %u\n", (long long)c_int, a.hp.use32, a.hp.unc32,
         a.hp.shift, a.hp.magic9);
  run<0>(a, "0 TMEM reads only");
  run<1>(a, "1 pass 1 max+min");
  run<2>(a, "2 pass 2 unclipped (SHF)");
  run<3>(a, "3 pass 2 clipped (SHF)");
  run<4>(a, "4 pass 2 unclipped (shift on IMAD.HI)");
  run<7>(a, "7 pass 2 unclipped, IMAD accumulate");
  run<8>(a, "8 pass 2 unclipped, 32-col pipelined loads");
  run<9>(a, "9 pass 2 float (IMAD, FADD, FFMA)");
  run<10>(a, "10 pass 2 float (I2F, FADD, FFMA)");
  run<11>(a, "11 pass 2 float packed x2");
  run<14>(a, "14 pass 2 denormal form (ISUB, FFMA2)");
  run<5>(a, "5 pass 3 unclipped magic9 + STS");
  run<15>(a, "15 pass 3 denormal form (ISUB, FFMA2.RZ, LOP3)");
  run<12>(a, "12 pass 3 float (IMAD, FADD, FFMA.RZ, LOP3)");
  run<13>(a, "13 pass 3 magic9, IMAD packing");
  run<6>(a, "6 pass 3 clipped magic9 + STS");
  return 0;
}
