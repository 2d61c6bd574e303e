// gemm_i8.cu -- exact int8 GEMM on tcgen05 (kind::i8, s32 accumulate in TMEM).
//
// C[M, N] int32 = A[M, K] * B[N, K]^T with A s8 or u8 and B s8, both K-major.
// This is the stage-level replacement of the reference's matmul_int8 /
// gemm_qk / gemm_pv (gemm.py:45-133), whose float-BLAS detour is exact by
// construction; integer MMA is exact by definition (|C| < 2^31 under the
// reference's MAX_HEAD_DIM / MAX_SEQ_LEN caps).  The fused attention kernel
// does not use it -- it is the unfused / per-stage path.
//
// One CTA per 128x128 output tile; K streamed in 128-byte (SWIZZLE_128B)
// blocks through a 3-stage TMA ring (97 KB: two CTAs per SM, so one CTA's epilogue
// overlaps the other's main loop); warp 0 = TMA, warp 1 = MMA issuer, warp 2 = TMEM
// allocator (128 columns), warps 4-7 = epilogue (TMEM -> registers -> 16-byte global
// stores, each thread filling whole 128-byte lines of its row).
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace ia {

int make_tmap_2d_u8(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t stride1,
                    uint32_t b0, uint32_t b1, int swizzle_bytes);

constexpr int G_BM = 128, G_BN = 128, G_BK = 128, G_ST = 3, G_THREADS = 256;
constexpr int G_TILE = G_BM * G_BK;  // bytes per A (or B) stage

__global__ void __launch_bounds__(G_THREADS, 2)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                   int32_t* __restrict__ C, int64_t ldc, int M, int N, int K, uint32_t idesc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + G_ST * G_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + G_ST * G_TILE);
  uint64_t* empty = full + G_ST;
  uint64_t* done = empty + G_ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * G_BM, n0 = blockIdx.x * G_BN;
  const int nkb = (K + G_BK - 1) / G_BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tma);
    prefetch_tmap(&tmb);
    for (int s = 0; s < G_ST; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0, s = 0, ph = 0; kb < nkb; ++kb) {
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect_tx(full + s, 2 * G_TILE);
        tma_load_2d(sa + s * G_TILE, &tma, full + s, kb * G_BK, m0);
        tma_load_2d(sb + s * G_TILE, &tmb, full + s, kb * G_BK, n0);
        if (++s == G_ST) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0, s = 0, ph = 0; kb < nkb; ++kb) {
        mbar_wait(full + s, ph);
        tc_fence_after();
        const uint32_t a = smem_u32(sa + s * G_TILE), b = smem_u32(sb + s * G_TILE);
#pragma unroll
        for (int kk = 0; kk < G_BK / 32; ++kk)
          mma_i8_ss(tmem, sdesc(a + kk * 32, 1024, 2u), sdesc(b + kk * 32, 1024, 2u), idesc,
                    (kb | kk) ? 1u : 0u);
        tc_commit(empty + s);
        if (++s == G_ST) { s = 0; ph ^= 1; }
      }
      tc_commit(done);
    }
  } else if (warp >= 4) {
    const int quad = warp & 3;
    const int r = m0 + quad * 32 + lane;
    const bool vec_ok = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
    mbar_wait(done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < G_BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + c, v);
      if (r < M) {
        int32_t* crow = C + (int64_t)r * ldc + n0 + c;
        if (vec_ok && n0 + c + 32 <= N) {  // whole 128-byte line of this row
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<int4*>(crow + e) =
                make_int4((int)v[e], (int)v[e + 1], (int)v[e + 2], (int)v[e + 3]);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (n0 + c + e < N) crow[e] = (int32_t)v[e];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

}  // namespace ia

using namespace ia;

extern "C" int ia_gemm_i8(const void* A, int64_t lda, int a_signed, const int8_t* B, int64_t ldb,
                          int64_t M, int64_t N, int64_t K, int32_t* C, int64_t ldc, void* stream) {
  if (!A || !B || !C || M < 1 || N < 1 || K < 1 || lda < K || ldb < K || ldc < N || (lda & 15) ||
      (ldb & 15) || ((((uintptr_t)A) | ((uintptr_t)B)) & 15))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_gemm_i8: bad arguments");
  if (M > (int64_t)65535 * G_BM || N > (int64_t)0x7fffffff || K > IA_MAX_HEAD_DIM + 65536)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_gemm_i8: problem too large");
  CUtensorMap ta, tb;
  int r;
  if ((r = make_tmap_2d_u8(&ta, A, K, M, lda, G_BK, G_BM, 128))) return r;
  if ((r = make_tmap_2d_u8(&tb, B, K, N, ldb, G_BK, G_BN, 128))) return r;
  const size_t smem = 1024 + 2 * G_ST * G_TILE + 256;
  cudaError_t e =
      cudaFuncSetAttribute(gemm_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e));
  const uint32_t idesc = idesc_i8(G_BM, G_BN, a_signed != 0, true);
  dim3 grid((unsigned)((N + G_BN - 1) / G_BN), (unsigned)((M + G_BM - 1) / G_BM));
  gemm_i8_kernel<<<grid, G_THREADS, smem, (cudaStream_t)stream>>>(ta, tb, C, ldc, (int)M, (int)N,
                                                                   (int)K, idesc);
  return check_launch("gemm_i8_kernel");
}
