// attention.cu -- fused IntAttention forward for sm_100a.
//
// One CTA per (batch, head, 128-row query tile).  Replaces the per-head body of
// the reference's int_attention (pipeline.py:215-253):
//     logits = Q^ K^T (int32)            gemm.py:88-106
//     P^ = IndexSoftmax(logits)  (u8)    softmax.py:131-204
//     acc = P^ V^ (int32)                gemm.py:109-133
//     out = f32(acc) * f32(s_v / 255)    pipeline.py:250-252
// The int32 logits and the u8 probabilities never leave the SM: QK^T lands in
// TMEM (tcgen05.mma kind::i8, s32 accumulate), the integer softmax reads it
// back with tcgen05.ld, and P^ is written back into the same TMEM columns
// (tcgen05.st) as the A operand of the P.V MMA.
//
// IndexSoftmax needs the FINAL row max m (for delta = m - a) and the FINAL
// integer row sum S (for the per-row table round(255 e / S)) before any P^ is
// known, and its LUT values cannot be rescaled exactly, so the FlashAttention
// running-max trick does not apply.  For more than two key tiles the kernel
// therefore makes three passes over the key tiles, recomputing QK^T each pass:
//   pass 1: row max;  pass 2: idx, S;  pass 3: P^ -> TMEM -> P.V MMA.
// With <= 2 key tiles (L <= 256) the logits stay resident in TMEM and QK^T is
// computed once.
//
// Warp roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4-7 / 8-11 = softmax warpgroups 0 / 1.
// Softmax warpgroup w owns key tiles n = w, w+2, ... and TMEM buffer S[w]
// (128 lanes x 128 columns); each thread owns one query row (TMEM lane).
// The two warpgroups merge their partial row max / row sum through smem.
//
// TMEM (512 columns): S[0] = cols [0,128), S[1] = [128,256), O = [256, 256+DP).
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "params.cuh"
#include "ptx.cuh"

namespace ia {

constexpr int BM = 128;  // query rows per tile (= TMEM lanes)
constexpr int BN = 128;  // keys per tile
constexpr int NKST = 3;  // K smem stages
constexpr int NVST = 2;  // V^T smem stages
constexpr int NTHREADS = 384;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t O_COL = 256;

struct AttnDev {
  float* out;
  const ia_head_params* params;
  const int32_t* seq_lens;
  const uint32_t* mask_bits;
  int32_t* dbg_logits;
  uint8_t* dbg_prob;
  int32_t* dbg_acc;
  int B, H, Hkv, L, d, mask_words;
  int causal, nlut, scale_x2, n_qt;
  uint8_t lut[256];
};

template <int DP>
struct Cfg {
  static constexpr int SW = DP >= 128 ? 128 : DP;  // swizzle span (bytes) of Q/K rows
  static constexpr int NSUB = DP / SW;              // 128-row sub-blocks per Q/K tile
  static constexpr uint32_t LAYOUT = SW == 128 ? 2u : (SW == 64 ? 4u : 6u);
  static constexpr uint32_t SBO = 8 * SW;
  static constexpr int SUB_BYTES = 128 * SW;
  static constexpr int Q_BYTES = BM * DP;
  static constexpr int K_BYTES = BN * DP;
  static constexpr int V_BYTES = DP * BN;  // V^T tile: DP rows x 128 keys, SWIZZLE_128B
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = Q_BYTES;
  static constexpr int OFF_V = OFF_K + NKST * K_BYTES;
  static constexpr int OFF_TAB = OFF_V + NVST * V_BYTES;
  static constexpr int KSTEPS = DP / 32;
};

__host__ __device__ constexpr size_t attn_smem_bytes(int dp, int nlut) {
  return 1024 /* alignment slack */ + (size_t)(dp * 128) * (1 + NKST + NVST) +
         (size_t)nlut * 512 /* row tables */ + 1024 /* lut */ + 2048 /* row exchange */ +
         256 /* barriers + tmem slot */;
}

// Masked-key bits for one 32-key chunk starting at j0 for query row i
// (bit e set = key j0+e excluded): causal / length / dense mask.
__device__ __forceinline__ uint32_t chunk_mask(const AttnDev& p, int i, int j0, int lim) {
  uint32_t mb = 0;
  if (j0 + 31 > lim) mb = (lim < j0) ? 0xffffffffu : (0xfffffffeu << (lim - j0));
  if (p.mask_bits && j0 < p.L) mb |= __ldg(p.mask_bits + (size_t)i * p.mask_words + (j0 >> 5));
  return mb;
}

template <int DP, bool DEBUG>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmq,
                    const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnDev p) {
  using C = Cfg<DP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int nlut = p.nlut;
  uint32_t* tab = reinterpret_cast<uint32_t*>(smem + C::OFF_TAB);  // [nlut][128] row tables
  uint32_t* lut_s = tab + nlut * 128;                               // [256]
  int32_t* xmax = reinterpret_cast<int32_t*>(lut_s + 256);          // [2][128]
  uint32_t* xsum = reinterpret_cast<uint32_t*>(xmax + 256);         // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsum + 256);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + NKST;
  uint64_t* v_full = k_empty + NKST;
  uint64_t* v_empty = v_full + NVST;
  uint64_t* s_full = v_empty + NVST;      // [2] MMA -> softmax (QK^T landed)
  uint64_t* s_free_sm = s_full + 2;       // [2] softmax -> MMA (S read, passes 1-2)
  uint64_t* s_free_mma = s_free_sm + 2;   // [2] MMA -> MMA (P.V consumed P^, pass 3)
  uint64_t* p_full = s_free_mma + 2;      // [2] softmax -> MMA (P^ in TMEM)
  uint64_t* o_full = p_full + 2;          // MMA -> epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int BH = p.B * p.H;
  const int bh = blockIdx.x % BH;
  const int qt = p.n_qt - 1 - (int)(blockIdx.x / BH);  // late (heavy causal) tiles first
  const int b = bh / p.H, h = bh - (bh / p.H) * p.H;
  const int kvh = b * p.Hkv + h / (p.H / p.Hkv);
  const int q0 = qt * BM;
  const int len = p.seq_lens ? min(p.seq_lens[b], p.L) : p.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (q0 >= len) {  // the whole query tile is padding: +0.0 rows (pipeline contract)
    const int rows = min(BM, p.L - q0);
    float* o = p.out + ((size_t)bh * p.L + q0) * p.d;
    for (int t = threadIdx.x; t < rows * p.d; t += NTHREADS) o[t] = 0.0f;
    return;
  }
  const int key_end = p.causal ? min(q0 + BM, len) : len;
  const int n_kt = (key_end + BN - 1) / BN;
  const bool resident = n_kt <= 2;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmq);
    prefetch_tmap(&tmk);
    prefetch_tmap(&tmv);
    mbar_init(q_full, 1);
    for (int s = 0; s < NKST; ++s) { mbar_init(k_full + s, 1); mbar_init(k_empty + s, 1); }
    for (int s = 0; s < NVST; ++s) { mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1); }
    for (int w = 0; w < 2; ++w) {
      mbar_init(s_full + w, 1);
      mbar_init(s_free_sm + w, 128);
      mbar_init(s_free_mma + w, 1);
      mbar_init(p_full + w, 128);
    }
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  for (int t = threadIdx.x; t < 256; t += NTHREADS) lut_s[t] = t < nlut ? p.lut[t] : 0u;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int s = 0; s < C::NSUB; ++s)
        tma_load_3d(smem + C::OFF_Q + s * C::SUB_BYTES, &tmq, q_full, s * C::SW, q0, bh);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      const int npass = resident ? 1 : 3;
      for (int pass = 0; pass < npass; ++pass) {
        const bool with_v = pass == npass - 1;
        for (int n = 0; n < n_kt; ++n) {
          mbar_wait(k_empty + ks, kph ^ 1);
          mbar_expect_tx(k_full + ks, C::K_BYTES);
          for (int s = 0; s < C::NSUB; ++s)
            tma_load_3d(smem + C::OFF_K + ks * C::K_BYTES + s * C::SUB_BYTES, &tmk, k_full + ks,
                        s * C::SW, n * BN, kvh);
          if (++ks == NKST) { ks = 0; kph ^= 1; }
          if (with_v) {
            mbar_wait(v_empty + vs, vph ^ 1);
            mbar_expect_tx(v_full + vs, C::V_BYTES);
            tma_load_3d(smem + C::OFF_V + vs * C::V_BYTES, &tmv, v_full + vs, n * BN, 0, kvh);
            if (++vs == NVST) { vs = 0; vph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idq = idesc_i8(BM, BN, true, true);   // s8 x s8 -> s32
      constexpr uint32_t idv = idesc_i8(BM, DP, false, true);  // u8 x s8 -> s32
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      mbar_wait(q_full, 0);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      int prev[2] = {0, 0};  // how S[w]'s last occupant is released: 0 none, 1 softmax, 2 P.V
      uint32_t c_sm[2] = {0, 0}, c_mma[2] = {0, 0}, c_p[2] = {0, 0};
      auto issue_qk = [&](int n, int release) {
        const int w = n & 1;
        if (prev[w] == 1) { mbar_wait(s_free_sm + w, c_sm[w] & 1); ++c_sm[w]; }
        else if (prev[w] == 2) { mbar_wait(s_free_mma + w, c_mma[w] & 1); ++c_mma[w]; }
        mbar_wait(k_full + ks, kph);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + C::OFF_K + ks * C::K_BYTES);
#pragma unroll
        for (int kk = 0; kk < C::KSTEPS; ++kk) {
          const uint32_t off = (kk * 32 / C::SW) * C::SUB_BYTES + (kk * 32) % C::SW;
          mma_i8_ss(tmem + w * 128, sdesc(sq + off, C::SBO, C::LAYOUT),
                    sdesc(sk + off, C::SBO, C::LAYOUT), idq, kk > 0);
        }
        tc_commit(k_empty + ks);
        tc_commit(s_full + w);
        if (++ks == NKST) { ks = 0; kph ^= 1; }
        prev[w] = release;
      };
      auto issue_pv = [&](int n) {
        const int w = n & 1;
        mbar_wait(p_full + w, c_p[w] & 1);
        ++c_p[w];
        mbar_wait(v_full + vs, vph);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + C::OFF_V + vs * C::V_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 32; ++kk)
          mma_i8_ts(tmem + O_COL, tmem + w * 128 + kk * 8, sdesc(sv + kk * 32, 1024, 2u), idv,
                    (n > 0 || kk > 0) ? 1u : 0u);
        tc_commit(v_empty + vs);
        tc_commit(s_free_mma + w);
        if (++vs == NVST) { vs = 0; vph ^= 1; }
      };
      if (!resident) {
        for (int pass = 0; pass < 2; ++pass)
          for (int n = 0; n < n_kt; ++n) issue_qk(n, 1);
        for (int n = 0; n < n_kt; ++n) {
          issue_qk(n, 2);
          if (n >= 1) issue_pv(n - 1);
        }
        issue_pv(n_kt - 1);
      } else {
        for (int n = 0; n < n_kt; ++n) issue_qk(n, 0);
        for (int n = 0; n < n_kt; ++n) issue_pv(n);
      }
      tc_commit(o_full);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ IndexSoftmax warpgroups
    const int wg = (warp - 4) >> 2;
    const int quad = warp & 3;             // TMEM lane quadrant accessible to this warp
    const int row = quad * 32 + lane;
    const int i = q0 + row;
    const bool row_valid = i < len;
    const uint32_t t_lane = (uint32_t)(quad * 32) << 16;
    const uint32_t s_base = tmem + t_lane + (uint32_t)(wg * 128);
    const int lim = p.causal ? min(i, len - 1) : len - 1;  // last unmasked key of this row
    const ia_head_params hp = p.params[bh];
    uint32_t s_cnt = 0;

    // ---- pass 1: row max over unmasked keys (softmax.py:139-143, :174-179)
    int32_t mx = INT_MIN;
    for (int n = wg; n < n_kt; n += 2) {
      mbar_wait(s_full + wg, s_cnt & 1);
      ++s_cnt;
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(s_base + c * 32, v);
        const int j0 = n * BN + c * 32;
        if (DEBUG && p.dbg_logits && i < p.L) {
          for (int e = 0; e < 32; ++e)
            if (j0 + e < p.L) p.dbg_logits[((size_t)bh * p.L + i) * p.L + j0 + e] = (int32_t)v[e];
        }
        if (!row_valid) continue;
        const uint32_t mb = chunk_mask(p, i, j0, lim);
        if (mb == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) mx = max(mx, (int32_t)v[e]);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (!((mb >> e) & 1u)) mx = max(mx, (int32_t)v[e]);
        }
      }
      tc_fence_before();
      if (!resident) mbar_arrive(s_free_sm + wg);
    }
    xmax[wg * 128 + row] = mx;
    named_bar_sync(1, 256);
    int32_t m = max(xmax[row], xmax[128 + row]);
    const bool dead = (m == INT_MIN);  // fully masked row: all-zero P^ (softmax.py:181-184)
    if (dead) m = 0;

    // ---- pass 2: idx, e = lut[idx], S = sum e (softmax.py:144-155)
    const int64_t k64 = nlut - 1;
    IdxMap im;
    im.k2 = 2u * (uint32_t)k64;
    im.magic = hp.magic;
    im.shift = hp.shift;
    im.lo = hp.use32 ? idx_lo(m, hp.c_eff) : 0;
    im.base = (uint32_t)m * im.k2 + (uint32_t)hp.c_eff;
    const bool fast = hp.use32 != 0;
    uint32_t S = 0;
    for (int n = wg; n < n_kt; n += 2) {
      if (!resident) {
        mbar_wait(s_full + wg, s_cnt & 1);
        ++s_cnt;
      }
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(s_base + c * 32, v);
        if (!row_valid || dead) continue;
        const int j0 = n * BN + c * 32;
        const uint32_t mb = chunk_mask(p, i, j0, lim);
        if (fast) {
          if (mb == 0) {
#pragma unroll
            for (int e = 0; e < 32; ++e) S += lut_s[im.idx((int32_t)v[e])];
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              S += lut_s[((mb >> e) & 1u) ? (uint32_t)k64 : im.idx((int32_t)v[e])];
          }
        } else {
          for (int e = 0; e < 32; ++e)
            S += lut_s[((mb >> e) & 1u) ? (uint32_t)k64 : idx_slow(m, (int32_t)v[e], hp.c_eff, k64)];
        }
      }
      tc_fence_before();
      if (!resident) mbar_arrive(s_free_sm + wg);
    }
    xsum[wg * 128 + row] = S;
    named_bar_sync(1, 256);
    S = xsum[row] + xsum[128 + row];
    // per-row normalisation table (softmax.py:157-160): (2*scale*lut[t] + S) // (2S)
    {
      const int half = nlut >> 1;
      const uint32_t two_s = 2u * S;
      for (int t = wg * half; t < (wg + 1) * half; ++t)
        tab[t * 128 + row] = S ? ((uint32_t)p.scale_x2 * lut_s[t] + S) / two_s : 0u;
    }
    named_bar_sync(1, 256);
    const uint32_t* trow = tab + row;

    // ---- pass 3: P^ = rowtab[idx] -> TMEM (in place over S[w]) -> P.V (softmax.py:161-162)
    for (int n = wg; n < n_kt; n += 2) {
      if (!resident) {
        mbar_wait(s_full + wg, s_cnt & 1);
        ++s_cnt;
      }
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(s_base + c * 32, v);
        uint32_t pk[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) pk[q] = 0u;
        const int j0 = n * BN + c * 32;
        if (row_valid && !dead) {
          const uint32_t mb = chunk_mask(p, i, j0, lim);
          if (fast) {
            if (mb == 0) {
#pragma unroll
              for (int e = 0; e < 32; ++e)
                pk[e >> 2] |= trow[im.idx((int32_t)v[e]) * 128] << (8 * (e & 3));
            } else {
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const uint32_t x = ((mb >> e) & 1u) ? (uint32_t)k64 : im.idx((int32_t)v[e]);
                pk[e >> 2] |= trow[x * 128] << (8 * (e & 3));
              }
            }
          } else {
            for (int e = 0; e < 32; ++e) {
              const uint32_t x = ((mb >> e) & 1u) ? (uint32_t)k64 : idx_slow(m, (int32_t)v[e], hp.c_eff, k64);
              pk[e >> 2] |= trow[x * 128] << (8 * (e & 3));
            }
          }
        }
        if (DEBUG && p.dbg_prob && i < p.L) {
          for (int e = 0; e < 32; ++e)
            if (j0 + e < p.L)
              p.dbg_prob[((size_t)bh * p.L + i) * p.L + j0 + e] = (uint8_t)(pk[e >> 2] >> (8 * (e & 3)));
        }
        tmem_st8(s_base + c * 8, pk);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full + wg);
    }

    // ---- epilogue: out = f32(acc) * f32(s_v / scale) (pipeline.py:250-252)
    mbar_wait(o_full, 0);
    tc_fence_after();
    constexpr int HALF = DP / 2;
#pragma unroll 1
    for (int c0 = wg * HALF; c0 < (wg + 1) * HALF; c0 += 16) {
      uint32_t a[16];
      tmem_ld16(tmem + t_lane + O_COL + c0, a);
      if (i < p.L) {
        float* orow = p.out + ((size_t)bh * p.L + i) * p.d;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int col = c0 + e;
          if (col < p.d)
            orow[col] = row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e]), hp.out_scale) : 0.0f;
        }
        if (DEBUG && p.dbg_acc) {
          for (int e = 0; e < 16; ++e)
            p.dbg_acc[((size_t)bh * p.L + i) * DP + c0 + e] = (int32_t)a[e];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
int make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                 uint64_t stride1, uint64_t stride2, uint32_t b0, uint32_t b1, int swizzle_bytes);

template <int DP, bool DEBUG>
static int launch_attn(const ia_attn_args* a, cudaStream_t st) {
  using C = Cfg<DP>;
  CUtensorMap tq, tk, tv;
  const uint64_t BH = a->B * a->H, BHkv = a->B * a->Hkv;
  int r;
  if ((r = make_tmap_3d(&tq, a->q, a->d_pad, a->L, BH, a->d_pad, a->L * a->d_pad, C::SW, BM,
                        C::SW)))
    return r;
  if ((r = make_tmap_3d(&tk, a->k, a->d_pad, a->L, BHkv, a->d_pad, a->L * a->d_pad, C::SW, BN,
                        C::SW)))
    return r;
  if ((r = make_tmap_3d(&tv, a->vt, a->L, a->d_pad, BHkv, a->l_pad, a->d_pad * a->l_pad, BN, DP,
                        128)))
    return r;
  AttnDev dv;
  dv.out = a->out;
  dv.params = a->params;
  dv.seq_lens = a->seq_lens;
  dv.mask_bits = a->mask_bits;
  dv.dbg_logits = a->dbg_logits;
  dv.dbg_prob = a->dbg_prob;
  dv.dbg_acc = a->dbg_acc;
  dv.B = (int)a->B;
  dv.H = (int)a->H;
  dv.Hkv = (int)a->Hkv;
  dv.L = (int)a->L;
  dv.d = (int)a->d;
  dv.mask_words = (int)((a->L + 31) / 32);
  dv.causal = a->causal ? 1 : 0;
  dv.nlut = a->nlut;
  dv.scale_x2 = 2 * a->p_scale;
  dv.n_qt = (int)((a->L + BM - 1) / BM);
  for (int t = 0; t < 256; ++t) dv.lut[t] = t < a->nlut ? a->lut[t] : 0;
  size_t smem = attn_smem_bytes(DP, a->nlut);
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM (it owns all 512 TMEM columns)
  auto kern = attn_fwd_kernel<DP, DEBUG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e));
  const uint64_t grid = (uint64_t)dv.n_qt * BH;
  if (grid > 0x7fffffffull) return fail(IA_ERR_INVALID_ARGUMENT, "grid too large");
  kern<<<(unsigned)grid, NTHREADS, smem, st>>>(tq, tk, tv, dv);
  return check_launch("attn_fwd_kernel");
}

}  // namespace ia

using namespace ia;

extern "C" int ia_attn_fwd(const ia_attn_args* a, void* stream) {
  if (!a || !a->q || !a->k || !a->vt || !a->out || !a->params)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_attn_fwd: null pointer");
  if (a->B < 1 || a->H < 1 || a->Hkv < 1 || a->H % a->Hkv || a->L < 1 || a->d < 1)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_attn_fwd: bad shape");
  if (a->L > IA_MAX_SEQ_LEN) return fail(IA_ERR_SEQ_LEN, "sequence length exceeds 65536");
  if (a->d > IA_FUSED_MAX_HEAD_DIM || a->d_pad < a->d ||
      (a->d_pad != 32 && a->d_pad != 64 && a->d_pad != 128 && a->d_pad != 256))
    return fail(IA_ERR_HEAD_DIM, "fused path needs d <= 256 and d_pad in {32,64,128,256}");
  if (a->l_pad < a->L || (a->l_pad & 15))
    return fail(IA_ERR_INVALID_ARGUMENT, "l_pad must be >= L and a multiple of 16");
  if (a->nlut < 4 || a->nlut > 256 || (a->nlut & (a->nlut - 1)))
    return fail(IA_ERR_INVALID_ARGUMENT, "nlut must be a power of two in [4, 256]");
  if (a->lut[0] != 255 || a->lut[a->nlut - 1] != 0)
    return fail(IA_ERR_LUT, "lookup table endpoints must be 255 and 0");
  if (a->p_scale != 255 && a->p_scale != 127)
    return fail(IA_ERR_INVALID_ARGUMENT, "p_scale must be 255 or 127");
  if ((((uintptr_t)a->q) | ((uintptr_t)a->k) | ((uintptr_t)a->vt)) & 15)
    return fail(IA_ERR_INVALID_ARGUMENT, "operands must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const bool dbg = a->dbg_logits || a->dbg_prob || a->dbg_acc;
  switch (a->d_pad) {
    case 32: return dbg ? launch_attn<32, true>(a, st) : launch_attn<32, false>(a, st);
    case 64: return dbg ? launch_attn<64, true>(a, st) : launch_attn<64, false>(a, st);
    case 128: return dbg ? launch_attn<128, true>(a, st) : launch_attn<128, false>(a, st);
    default: return dbg ? launch_attn<256, true>(a, st) : launch_attn<256, false>(a, st);
  }
}
