// attention.cu -- fused IntAttention forward for sm_100a.
//
// One CTA per (batch, head, 128-row query tile).  Replaces the per-head body of
// the reference's int_attention (pipeline.py:215-253):
//     logits = Q^ K^T (int32)            gemm.py:88-106
//     P^ = IndexSoftmax(logits)  (u8)    softmax.py:131-204
//     acc = P^ V^ (int32)                gemm.py:109-133
//     out = f32(acc) * f32(s_v / 255)    pipeline.py:250-252
// The int32 logits and the u8 probabilities never leave the SM: QK^T lands in
// TMEM (tcgen05.mma kind::i8, s32 accumulate), the integer softmax reads it back
// with tcgen05.ld, and P^ goes to a K-major SWIZZLE_128B shared-memory tile that
// is the A operand of the P.V MMA (SS form, u8 x s8 -> s32 in TMEM).
//
// IndexSoftmax needs the FINAL row max m (for delta = m - a) and the FINAL integer
// row sum S (for the per-row table round(255 e / S)) before any P^ is known, and
// its LUT values cannot be rescaled exactly, so the FlashAttention running-max
// trick does not apply.  For more than NWG key tiles the kernel therefore makes
// three passes over the key tiles, recomputing QK^T each pass:
//   pass 1: row max (+ row min);  pass 2: idx, S;  pass 3: P^ -> smem -> P.V MMA.
// With <= NWG key tiles (L <= 384 for d_pad <= 128) the logits stay resident in
// TMEM and QK^T runs once.  Grouped K (per-row-group key scales, gk_passes) takes
// its group maxima per tile and needs two passes.
//
// Warps (512 threads for d_pad <= 128, 384 for 256): warps 0..4*NWG-1 are NWG = 3
// (2) softmax warpgroups; the last four are the role warps -- K (+Q) TMA producer,
// QK^T MMA issuer, V^T TMA producer + TMEM allocator, P.V MMA issuer -- at the
// highest warp ids, which the scheduler favours.  Softmax warpgroup w owns key
// tiles n = w, w+NWG, ... and TMEM buffer S[w] (128 lanes x 128 columns); each
// thread owns one query row (TMEM lane).  The warpgroups merge their partial row
// max / min / sum through smem at the pass boundaries.
//
// TMEM (512 columns): S[w] = cols [128w, 128w+128), O = [128 NWG, 128 NWG + DP).
// SMEM: Q tile, K ring (NKST stages; in passes 1-2 the idle P^ area adds stages),
// 2 V^T stages, NPB P^ tiles per warpgroup, the per-row normalisation tables, the
// row exchange arrays and the mbarriers (see Cfg and DESIGN.md §5).
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "params.cuh"
#include "ptx.cuh"

// epilogue staging with 16-byte shared-memory accesses (conflict-free pitch)
#ifndef IA_STAGE_V4
#define IA_STAGE_V4 1
#endif

namespace ia {

constexpr int BM = 128;  // query rows per tile (= TMEM lanes)
constexpr int BN = 128;  // keys per tile
constexpr uint32_t TMEM_COLS = 512;

struct AttnDev {
  float* out;
  const ia_head_params* params;
  const int32_t* seq_lens;
  const uint32_t* mask_bits;
  int32_t* dbg_logits;
  uint8_t* dbg_prob;
  int32_t* dbg_acc;
  long long* dbg_times;  // optional per-CTA phase clocks (development instrumentation)
  int B, H, Hkv, L, d, mask_words;
  int causal, nlut, scale_x2, n_qt;
  // development experiments (IA_XFLAGS, read only by the IA_PROFILE build; the release
  // kernel compiles every XF() test to 0 -- results are not exact with any bit set):
  // 1 pass 1 only; 2/4/8/16 spin instead of sleep-waits (QK^T issuer / softmax s_full /
  // P.V issuer / TMA producers); 32 no pass-1 arithmetic; 256 generic index map (no magic9)
  int xflags;
  // grouped K (per-row-group key scales): per (b*H + h, group) {c_eff, magic, shift, use32}
  const int4* kgroup;
  int gs_log2, n_groups;
  uint8_t lut[256];
};

template <int DP>
struct Cfg {
  // softmax warpgroups == TMEM S buffers (one 128-column buffer each); O sits after them.
  // Each warpgroup also owns one smem P^ tile.
  static constexpr int NWG = DP <= 128 ? 3 : 2;
  static constexpr int NKST = DP <= 64 ? 6 : (DP <= 128 ? 3 : 2);  // K smem stages
  static constexpr int NTHREADS = 128 + 128 * NWG;
  static constexpr uint32_t O_COL = 128 * NWG;
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
  static constexpr int NVST = 2;  // V^T smem stages
  static constexpr int OFF_V = OFF_K + NKST * K_BYTES;
  static constexpr int P_BYTES = BM * BN;  // u8 P^ tile, K-major SWIZZLE_128B (A of P.V)
  static constexpr int NPB = DP <= 128 ? 2 : 1;  // P^ buffers per softmax warpgroup
  static constexpr int OFF_P = OFF_V + NVST * V_BYTES;
  static constexpr int OFF_TAB = OFF_P + NWG * NPB * P_BYTES;
  // During passes 1-2 the P^ area is idle, so the K ring borrows it: NKX stages
  // (the NKST regular ones first) instead of NKST.  Pass-3 loads use only the
  // regular stages; every pass-2 QK^T has completed (its S tile was read) before
  // any warpgroup leaves the pass-2 row-sum exchange and writes a P^ tile.
  static constexpr int NKX_RAW = NKST + (NWG * NPB * P_BYTES) / K_BYTES;
  // ring sizes are multiples of NWG so that, with the ring restarting at stage 0 every
  // pass (IA_QK_UNROLL), stage ks of a pass always feeds buffer ks % NWG
  static constexpr int NKX = ((NKX_RAW > 16 ? 16 : NKX_RAW) / NWG) * NWG;
  static_assert(NKST % NWG == 0 && NKX % NWG == 0 && NKX >= NKST, "K ring sizes");
  static constexpr int KSTEPS = DP / 32;
  static constexpr int BAR_BYTES = 8 * (1 + 2 * NKX + 2 * NVST + 2 * NWG + 2 * NWG * NPB + 1) + 4;
  static_assert(BAR_BYTES <= 512, "barrier block");
  __host__ __device__ static constexpr int k_off(int s) {
    return s < NKST ? OFF_K + s * K_BYTES : OFF_P + (s - NKST) * K_BYTES;
  }
  // f32 epilogue staging row pitch (words): 16-byte aligned rows, and 8 consecutive rows'
  // 16-byte units fall in 8 different bank groups (33 r mod 8), so both the per-row STS.128
  // of the writers and the LDS.128 of the coalescing readers are conflict-free (the former
  // DP + 1 pitch made every scalar read-back 4-way conflicted: 8 K wavefronts per CTA)
  static constexpr int STAGE_PITCH = IA_STAGE_V4 ? DP + 4 : DP + 1;
  static_assert(OFF_TAB >= BM * STAGE_PITCH * 4, "epilogue staging must fit in Q/K/V stages");
  static_assert(OFF_TAB % 512 == 0, "row-table base: idx * 512 is OR-ed into the address");
};

// Row tables: u32 [tab_entries][128] (conflict-free gathers) for nlut <= 64, else u8.
// For nlut <= 32 the u32 table is zero-extended to 56 entries so warps whose
// largest reachable index is < 56 can skip the per-logit clip (IdxMap::idx_u).
__host__ __device__ constexpr bool wide_tab(int nlut) { return nlut <= 64; }
__host__ __device__ constexpr int tab_entries(int nlut) { return row_table_entries(nlut); }

template <int DP>
constexpr size_t attn_smem_bytes(int nlut) {
  return 1024 /* alignment slack */ + (size_t)Cfg<DP>::OFF_TAB +
         (size_t)tab_entries(nlut) * (wide_tab(nlut) ? 512 : 128) /* row tables */ +
         3 * 3 * 512 /* row exchange */ + 512 /* barriers + tmem slot (Cfg::BAR_BYTES) */;
}

// Masked-key bits for one 32-key chunk starting at j0 for query row i
// (bit e set = key j0+e excluded): causal / length / dense mask.
__device__ __forceinline__ uint32_t chunk_mask(const AttnDev& p, int i, int j0, int lim) {
  uint32_t mb = 0;
  if (j0 + 31 > lim) mb = (lim < j0) ? 0xffffffffu : (0xfffffffeu << (lim - j0));
  if (p.mask_bits && j0 < p.L) mb |= __ldg(p.mask_bits + (size_t)i * p.mask_words + (j0 >> 5));
  return mb;
}

__host__ __device__ constexpr int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }
__host__ __device__ constexpr int lcm_i(int a, int b) { return a / gcd_i(a, b) * b; }

// f(std::integral_constant<int, 0>{}) ... f(std::integral_constant<int, N - 1>{})
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// (a & b) | c as one LOP3 the compiler cannot re-associate: the row-table address
// (umulhi(n, magic9) & ~511) | row*4 then joins the table base inside the LDS
// ([R + UR + imm] addressing) instead of costing an extra IADD per logit.
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));  // (a & b) | c
  return r;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Phase / wait-time instrumentation (tools/phase_times.py).  Compiled in only
// for the profiling build (make profile -> libintattn_b200_prof.so).
__device__ __forceinline__ long long clk64() {
#if IA_PROFILE
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
#else
  return 0;
#endif
}
// Experiment bits: compile-time 0 outside the profiling build.
#define XF(bits) (IA_PROFILE ? (p.xflags & (bits)) : 0)
#define IA_TMARK(slot)                                                                      \
  do {                                                                                      \
    if (IA_PROFILE && p.dbg_times) p.dbg_times[(size_t)blockIdx.x * 16 + (slot)] = clk64(); \
  } while (0)
// Event timeline of two CTAs (0 and IA_TRACE_CTA2): per-role segments of 2048
// entries after the per-CTA slots, entry = clock << 16 | event << 12 | tile.
#define IA_TRACE_CTA2 1000
#define IA_TRACE(seg, ev, t)                                                                  \
  do {                                                                                        \
    if (IA_PROFILE && p.dbg_times && (blockIdx.x == 0 || blockIdx.x == IA_TRACE_CTA2)) {      \
      long long* tb_ = p.dbg_times + (size_t)gridDim.x * 16 +                                 \
                       ((blockIdx.x ? 16 : 0) + (seg)) * 2048;                                 \
      tb_[trc++ & 2047] = (clk64() << 16) | ((long long)(ev) << 12) | ((t) & 0xfff);          \
    }                                                                                         \
  } while (0)
// Wait-time accumulators live in registers (tacc) and are flushed once at the end,
// so the instrumentation adds no global round trips to the pipeline loops.
#define IA_TADD(slot, v)              \
  do {                                \
    if (IA_PROFILE) tacc[(slot)-8] += (v); \
  } while (0)

// Barrier wait with the suspend hint (default) or a pure poll (spin = true).
__device__ __forceinline__ void bwait(uint64_t* bar, uint32_t parity, bool spin) {
  if (spin) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);
}
// Layout / wait-policy variants (A/B builds):
//   IA_ROLE_FIRST          role warps at warp ids 0-3 (lowest arbitration priority)
//   IA_PRODUCER_BACKOFF_NS TMA producers poll with a fixed back-off (0: suspended try_wait)
//   IA_ISSUER_BACKOFF_NS   MMA issuers likewise
#ifndef IA_ROLE_FIRST
#define IA_ROLE_FIRST 0
#endif
// QK^T issuer unrolled over the K ring (stage / buffer indices compile-time); the K
// ring then restarts at stage 0 every pass (producer and issuer alike)
#ifndef IA_QK_UNROLL
#define IA_QK_UNROLL 1
#endif
// the same for the P.V issuer (measured 0.7 % slower on C4: off)
#ifndef IA_PV_UNROLL
#define IA_PV_UNROLL 0
#endif
// pass-3 16-key group skip below the row's nonzero threshold (rows of >= 16 key tiles)
#ifndef IA_GROUP_SKIP
#define IA_GROUP_SKIP 1
#endif
// float form of the index map in passes 2-3 where it is exact (params.cuh float_idx_ok)
#ifndef IA_FLOAT_IDX
#define IA_FLOAT_IDX 1
#endif
#ifndef IA_SKIP_G
#define IA_SKIP_G 8
#endif
// pass-3 skip decisions for a whole 64-key batch at once (see fgroups)
#ifndef IA_SKIP_MASK
#define IA_SKIP_MASK 1
#endif
// pass-1 row max: independent VIMNMX3 chains per 64-logit batch
// timing-only experiments (never in a shipped build; results are wrong with any bit set):
// 1 pass 2 without its LUT gather, 2 pass 3 without its row-table gather, 4 no P^ stores,
// 8 K producer arrives without loading (stale K tiles)
#ifndef IA_EXP
#define IA_EXP 0
#endif
// warp id made provably uniform (shuffle from lane 0): role loops on the uniform datapath
// (476 -> 77 R2UR, four back-to-back UTCIMMA per tile) -- measured 3-5 % SLOWER on C4
// (2.585 -> 2.68 / 2.72 ms), so off
#ifndef IA_UNIFORM_WARP
#define IA_UNIFORM_WARP 0
#endif
// rows of at least this many key tiles use the pass-3 group skip
// grouped K: batch-level fast path (float form, unmasked) and pass-B chunk skip
#ifndef IA_GK_FAST
#define IA_GK_FAST 1
#endif
// pass 1 (MMA-bound, light softmax work): poll s_full instead of the suspended wait
#ifndef IA_P1_SPIN
#define IA_P1_SPIN 0
#endif
// QK^T issuer polls s_free (1) / k_full (2) instead of the suspended wait (3: C4 2.566 -> 2.552 ms,
// C3 0.086 -> 0.084, C5 2.349 -> 2.343)
#ifndef IA_QK_SPIN
#define IA_QK_SPIN 3
#endif
// experiment: idle the MMA issuers for a while after each tile (QK^T: 100 ns costs 3 %, 300 ns
// 25 % -- its issue latency is on the critical path; P.V: 100 / 300 ns cost 0.3 % / 1.2 %)
#ifndef IA_QK_DELAY_NS
#define IA_QK_DELAY_NS 0
#endif
#ifndef IA_PV_DELAY_NS
#define IA_PV_DELAY_NS 0
#endif
#ifndef IA_SKIP_MIN_KT
#define IA_SKIP_MIN_KT 16
#endif
#ifndef IA_P1_CHAINS
#define IA_P1_CHAINS 2
#endif
#ifndef IA_PRODUCER_BACKOFF_NS
#define IA_PRODUCER_BACKOFF_NS 0
#endif
#ifndef IA_ISSUER_BACKOFF_NS
#define IA_ISSUER_BACKOFF_NS 0
#endif
__device__ __forceinline__ void pwait(uint64_t* bar, uint32_t parity, bool spin) {
  if (IA_PRODUCER_BACKOFF_NS > 0 && !spin) mbar_wait_backoff(bar, parity, IA_PRODUCER_BACKOFF_NS);
  else bwait(bar, parity, spin);
}
__device__ __forceinline__ void iwait(uint64_t* bar, uint32_t parity, bool spin) {
  if (IA_ISSUER_BACKOFF_NS > 0 && !spin) mbar_wait_backoff(bar, parity, IA_ISSUER_BACKOFF_NS);
  else bwait(bar, parity, spin);
}

// ------------------------------------------------------------------ grouped K
// Grouped-K IndexSoftmax (softmax.py:309-399, default per-group-max mode, as the
// per-row-group-K pipeline uses it, pipeline.py:229-246).  Keys are quantised per
// row group of gs keys, so group g has its own clip threshold c_g (from alpha_g =
// s_q s_k[g] / sqrt(d)) and every distance is taken against the group's own row
// max m_g; the LUT and the integer row normalisation are shared.  For gs | 128 no
// group straddles a key tile, so a tile's group maxima come from the tile itself
// and the fused kernel needs two passes instead of three: pass A (S = sum e) and
// pass B (P^ -> P.V), each reading its tile from TMEM twice -- group maxima over
// 8-key chunks, then the per-logit work.  The int32 logits still never leave the SM.

// Excluded-key bits (bit e = key j0 + e masked) for 32 keys of row i.
__device__ __forceinline__ uint32_t gk_mask32(const AttnDev& p, bool row_valid, int i, int j0,
                                              int lim) {
  return row_valid ? chunk_mask(p, i, j0, lim) : 0xffffffffu;
}

// Group maxima of one 128-key tile: gm[c] = max over the unmasked keys of the group
// holding 8-key chunk c (INT_MIN if the row has none there).
__device__ __forceinline__ void gk_group_max(const AttnDev& p, uint32_t s_tile, bool row_valid,
                                             int i, int j0t, int lim, int32_t (&gm)[16]) {
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    uint32_t va[32], vb[32];
    tmem_ld64(s_tile + hb * 64, va, vb);
    const int j0 = j0t + hb * 64;
    const uint32_t ma = gk_mask32(p, row_valid, i, j0, lim);
    const uint32_t mb = gk_mask32(p, row_valid, i, j0 + 32, lim);
    if (!__any_sync(0xffffffffu, (ma | mb) != 0u)) {  // no key masked in the warp: plain maxima
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
        int32_t x = __vimax3_s32((int32_t)v8[0], (int32_t)v8[1], (int32_t)v8[2]);
        x = __vimax3_s32(x, (int32_t)v8[3], (int32_t)v8[4]);
        x = __vimax3_s32(x, (int32_t)v8[5], (int32_t)v8[6]);
        gm[hb * 8 + c] = max(x, (int32_t)v8[7]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
        const uint32_t bits = ((c < 4 ? ma : mb) >> (8 * (c & 3))) & 0xffu;
        int32_t x = INT_MIN;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (!((bits >> e) & 1u)) x = max(x, (int32_t)v8[e]);
        gm[hb * 8 + c] = x;
      }
    }
  }
  // chunks of one group share its maximum (groups of gs/8 = 1..16 chunks)
  const int gs8 = 1 << (p.gs_log2 - 3);
#pragma unroll
  for (int s = 1; s < 16; s <<= 1) {
    if (gs8 > s) {
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (!(c & s)) {
          const int32_t t = max(gm[c], gm[c | s]);
          gm[c] = t;
          gm[c | s] = t;
        }
    }
  }
}

// The same for one 64-key batch already in registers (groups of <= 64 keys never straddle
// a batch, so their maxima need no second TMEM read): gm8[c] for the batch's 8 chunks.
__device__ __forceinline__ void gk_batch_max(const AttnDev& p, const uint32_t (&va)[32],
                                             const uint32_t (&vb)[32], uint32_t ma, uint32_t mb,
                                             bool open, int32_t* gm8) {
  if (open) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
      int32_t x = __vimax3_s32((int32_t)v8[0], (int32_t)v8[1], (int32_t)v8[2]);
      x = __vimax3_s32(x, (int32_t)v8[3], (int32_t)v8[4]);
      x = __vimax3_s32(x, (int32_t)v8[5], (int32_t)v8[6]);
      gm8[c] = max(x, (int32_t)v8[7]);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
      const uint32_t bits = ((c < 4 ? ma : mb) >> (8 * (c & 3))) & 0xffu;
      int32_t x = INT_MIN;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!((bits >> e) & 1u)) x = max(x, (int32_t)v8[e]);
      gm8[c] = x;
    }
  }
  const int gs8 = 1 << (p.gs_log2 - 3);
#pragma unroll
  for (int s = 1; s < 8; s <<= 1) {
    if (gs8 > s) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (!(c & s)) {
          const int32_t t = max(gm8[c], gm8[c | s]);
          gm8[c] = t;
          gm8[c | s] = t;
        }
    }
  }
}

// idx of logit a in a group with row max m (softmax.py:380-386 with the group's c).
struct GkMap {
  int32_t lo;
  uint32_t base, magic, shift;
  int64_t c_eff;
  int32_t m;
  bool use32;
  __device__ __forceinline__ void init(int32_t gmax, int4 g, uint32_t k) {
    c_eff = (int64_t)g.x;
    magic = (uint32_t)g.y;
    shift = (uint32_t)g.z;
    use32 = g.w != 0;
    m = gmax;
    lo = idx_lo(gmax, c_eff);
    base = (uint32_t)gmax * (2u * k) + (uint32_t)c_eff;
  }
  __device__ __forceinline__ uint32_t idx32(int32_t a, uint32_t nk2) const {
    const uint32_t n = base + nk2 * (uint32_t)max(a, lo);
    return __umulhi(n, magic) >> shift;
  }
  __device__ __forceinline__ uint32_t idx(int32_t a, uint32_t nk2, uint32_t k) const {
    return use32 ? idx32(a, nk2) : idx_slow(m, a, c_eff, k);
  }
};

template <int DP, bool DEBUG>
__device__ __forceinline__ void gk_passes(const AttnDev& p, uint8_t* smem, uint32_t* tab,
                                          uint32_t* xsum, const uint8_t* lut8, const uint8_t* lut8r,
                                          uint64_t* s_full,
                                          uint64_t* s_free, uint64_t* p_full, uint64_t* p_free,
                                          uint32_t s_base, int wg, int row, int lane, int i,
                                          int lim, int bh, int n_kt, bool row_valid,
                                          bool resident, uint32_t& s_ph) {
  using C = Cfg<DP>;
  constexpr int NWG = C::NWG;
  constexpr int NWT = 128 * NWG;
  const int nlut = p.nlut;
  const uint32_t k = (uint32_t)(nlut - 1);
  uint32_t nk2 = 0u - 2u * k;
  asm("" : "+r"(nk2));
  const int4* gp = p.kgroup + (size_t)bh * p.n_groups;
  const float lutden = __uint_as_float(smem_u32(lut8r));  // float form, pass A addend: &lut8r[0]

  // ---- pass A: e = lut[idx_g], S = sum e (softmax.py:380-394); the only wait on the
  // MMA when the logits stay resident in TMEM
  uint32_t S = 0;
  for (int n = wg; n < n_kt; n += NWG) {
    mbar_wait(s_full + wg, s_ph);
    s_ph ^= 1u;
    tc_fence_after();
    int32_t gm[16];
    const bool two_reads = p.gs_log2 == 7;  // 128-key groups span both batches of the tile
    if (two_reads) gk_group_max(p, s_base, row_valid, i, n * BN, lim, gm);
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      uint32_t va[32], vb[32];
      tmem_ld64(s_base + hb * 64, va, vb);
      if (hb == 1 && !resident) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free + wg);
      }
      const int j0 = n * BN + hb * 64;
      const uint32_t ma = gk_mask32(p, row_valid, i, j0, lim);
      const uint32_t mb = gk_mask32(p, row_valid, i, j0 + 32, lim);
      const bool open = !__any_sync(0xffffffffu, (ma | mb) != 0u);  // no key masked in the warp
      int32_t gb[8];  // this batch's group maxima per 8-key chunk
      if (two_reads) {
#pragma unroll
        for (int c = 0; c < 8; ++c) gb[c] = hb ? gm[8 + c] : gm[c];
      } else {
        gk_batch_max(p, va, vb, ma, mb, open, gb);
      }
      if (IA_GK_FAST && open) {
        // Batch-level fast path: no key masked and every group of these 64 keys in the float
        // form (warp-uniform) -- straight-line code over the batch, the eight chunks'
        // parameters loaded up front.
        int32_t gcx[8], gry[8];  // c_eff and the f32 ratio bits of each chunk's group
        int allf = 2;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int4 g4 = __ldg(gp + ((j0 + 8 * c) >> p.gs_log2));
          gcx[c] = g4.x;
          gry[c] = g4.y;
          allf &= g4.w;
        }
        if (allf) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
            const float rg = __int_as_float(gry[c]);
            const int32_t nlo = gcx[c] - gb[c];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const uint32_t u0 = (uint32_t)__viaddmax_s32((int32_t)v8[e], nlo, 0);
              const uint32_t u1 = (uint32_t)__viaddmax_s32((int32_t)v8[e + 1], nlo, 0);
              float f0, f1;
              fma_rn_f32x2(f0, f1, __uint_as_float(u0), __uint_as_float(u1), rg, lutden);
              S += lds_u8(__float_as_uint(f0)) + lds_u8(__float_as_uint(f1));
            }
          }
          continue;
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int32_t gmax = gb[c];
        if (gmax == INT_MIN) continue;  // every key of the chunk is masked: e = 0
        const int4 gpar = __ldg(gp + ((j0 + 8 * c) >> p.gs_log2));
        const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
        const uint32_t bits = ((c < 4 ? ma : mb) >> (8 * (c & 3))) & 0xffu;
        if (gpar.w & 2) {
          // float form (params.cuh, as the per-tensor kernel): u = max(a - lo_g, 0), one
          // denormal FMA leaves &lut8r[k - idx] in the result's bits; masked keys take u = 0
          // (idx = k, lut[k] = 0).  Warp-uniform: the group's parameters are.
          const float rg = __int_as_float(gpar.y);
          const int32_t nlo = gpar.x - gmax;
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            uint32_t u0 = (uint32_t)__viaddmax_s32((int32_t)v8[e], nlo, 0);
            uint32_t u1 = (uint32_t)__viaddmax_s32((int32_t)v8[e + 1], nlo, 0);
            if (!open) {
              u0 = ((bits >> e) & 1u) ? 0u : u0;
              u1 = ((bits >> (e + 1)) & 1u) ? 0u : u1;
            }
            float f0, f1;
            fma_rn_f32x2(f0, f1, __uint_as_float(u0), __uint_as_float(u1), rg, lutden);
            S += lds_u8(__float_as_uint(f0)) + lds_u8(__float_as_uint(f1));
          }
          continue;
        }
        GkMap gmap;
        gmap.init(gmax, gpar, k);
        if (open && gmap.use32) {  // warp-uniform: no per-key tests
#pragma unroll
          for (int e = 0; e < 8; ++e) S += lut8[gmap.idx32((int32_t)v8[e], nk2)];
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (!((bits >> e) & 1u)) S += lut8[gmap.idx((int32_t)v8[e], nk2, k)];
        }
      }
    }
  }
  // ---- shared row normalisation table (softmax.py:300-306): (2 scale lut[t] + S) // 2S
  xsum[wg * 128 + row] = S;
  named_bar_sync(1, NWT);
  S = xsum[row];
#pragma unroll
  for (int w = 1; w < NWG; ++w) S += xsum[w * 128 + row];
  {
    const uint32_t two_s = 2u * S;
    const float rden = S ? __frcp_rn((float)two_s) : 0.0f;
    for (int t = wg; t < nlut; t += NWG) {
      const uint32_t lt = lut8[t];
      uint32_t pv = 0u;
      if (S && lt) {
        const uint32_t num = (uint32_t)p.scale_x2 * lt + S;
        int32_t q = __float2int_rz(__fmul_rn((float)num, rden));
        const int32_t r = (int32_t)num - q * (int32_t)two_s;
        q += r < 0 ? -1 : (r >= (int32_t)two_s ? 1 : 0);
        pv = (uint32_t)q;
      }
      tab[((int)k - t) * 128 + row] = pv;  // reversed: entry j = k - idx (the float form's index)
    }
  }
  named_bar_sync(1, NWT);

  // Pass-B skip threshold in the index domain: P^ = rowtab[idx] > 0 only for idx <= t*
  // (t* = the largest t with 2 scale lut[t] >= S, every entry scanned), i.e. only for
  // j = k - idx >= jmin = k - t*; j is monotone in u = a - lo_g, so a chunk whose largest
  // logit maps below jmin in every row of the warp is all zero.  Rows of >= 16 key tiles.
  uint32_t jmin = 0u;  // 0: no chunk is skipped
  if (IA_GK_FAST && n_kt >= IA_SKIP_MIN_KT) {
    int tstar = -1;
    if (row_valid && S)
      for (int t = 0; t < nlut; ++t)
        if ((uint32_t)p.scale_x2 * (uint32_t)lut8[t] >= S) tstar = t;
    jmin = tstar < 0 ? k + 1u : k - (uint32_t)tstar;  // no nonzero entry: nothing is live
  }
  // ---- pass B: P^ = rowtab[idx_g] -> smem -> P.V MMA
  const uint32_t tab_row = smem_u32(tab) + (uint32_t)row * 4u;
  const uint32_t row4 = (uint32_t)row * 4u;
  const float tabden = __uint_as_float(smem_u32(tab) + 256u);  // float form, pass B addend
  const uint32_t p_rows = smem_u32(smem + C::OFF_P + wg * C::NPB * C::P_BYTES) + (uint32_t)row * 128;
  const uint32_t p_xor = (uint32_t)(row & 7);
  int tl = 0;
  for (int n = wg; n < n_kt; n += NWG) {
    if (!resident) {
      mbar_wait(s_full + wg, s_ph);
      s_ph ^= 1u;
    }
    tc_fence_after();
    const int pbl = tl % C::NPB;
    const uint32_t p_row = p_rows + (uint32_t)(pbl * C::P_BYTES);
    mbar_wait(p_free + wg * C::NPB + pbl, ((uint32_t)(tl / C::NPB) & 1u) ^ 1u);
    int32_t gm[16];
    const bool two_reads = p.gs_log2 == 7;
    if (two_reads) gk_group_max(p, s_base, row_valid, i, n * BN, lim, gm);
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      uint32_t va[32], vb[32];
      tmem_ld64(s_base + hb * 64, va, vb);
      if (hb == 1 && !resident) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free + wg);
      }
      const int j0 = n * BN + hb * 64;
      const uint32_t ma = gk_mask32(p, row_valid, i, j0, lim);
      const uint32_t mb = gk_mask32(p, row_valid, i, j0 + 32, lim);
      uint32_t pk[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) pk[q] = 0u;
      const bool open = !__any_sync(0xffffffffu, (ma | mb) != 0u);
      int32_t gb[8];  // this batch's group maxima per 8-key chunk
      if (two_reads) {
#pragma unroll
        for (int c = 0; c < 8; ++c) gb[c] = hb ? gm[8 + c] : gm[c];
      } else {
        gk_batch_max(p, va, vb, ma, mb, open, gb);
      }
      bool fast_done = false;
      if (IA_GK_FAST && open) {
        int32_t gcx[8], gry[8];  // c_eff and the f32 ratio bits of each chunk's group
        int allf = 2;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int4 g4 = __ldg(gp + ((j0 + 8 * c) >> p.gs_log2));
          gcx[c] = g4.x;
          gry[c] = g4.y;
          allf &= g4.w;
        }
        if (allf) {
          // live chunks: the chunk's largest logit reaches an index with a nonzero table
          // entry in some row of the warp (all eight decisions at once, one REDUX.OR)
          uint32_t live = 0xffu;
          if (n_kt >= IA_SKIP_MIN_KT) {
            uint32_t lm = 0u;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
              int32_t cm = __vimax3_s32((int32_t)v8[0], (int32_t)v8[1], (int32_t)v8[2]);
              cm = __vimax3_s32(cm, (int32_t)v8[3], (int32_t)v8[4]);
              cm = __vimax3_s32(cm, (int32_t)v8[5], (int32_t)v8[6]);
              const int32_t nlo = gcx[c] - gb[c];
              const uint32_t um = (uint32_t)__viaddmax_s32(max(cm, (int32_t)v8[7]), nlo, 0);
              const float fj = __fmaf_rn(__uint_as_float(um), __int_as_float(gry[c]), 0.0f);
              lm |= __float_as_uint(fj) >= jmin ? (1u << c) : 0u;
            }
            live = __reduce_or_sync(0xffffffffu, lm);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (!((live >> c) & 1u)) continue;  // pk stays 0
            const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
            const float r9 = __int_as_float(gry[c]) * 512.0f;
            const int32_t nlo = gcx[c] - gb[c];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t pw[4];
#pragma unroll
              for (int e = 0; e < 4; e += 2) {
                const uint32_t u0 = (uint32_t)__viaddmax_s32((int32_t)v8[4 * q + e], nlo, 0);
                const uint32_t u1 = (uint32_t)__viaddmax_s32((int32_t)v8[4 * q + e + 1], nlo, 0);
                float f0, f1;
                fma_rz_f32x2(f0, f1, __uint_as_float(u0), __uint_as_float(u1), r9, tabden);
                pw[e] = lds_u32(and_or(__float_as_uint(f0), 0xFFFFFE00u, row4));
                pw[e + 1] = lds_u32(and_or(__float_as_uint(f1), 0xFFFFFE00u, row4));
              }
              pk[2 * c + q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040),
                                          __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
            }
          }
          fast_done = true;
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (fast_done) break;
        const int32_t gmax = gb[c];
        if (gmax == INT_MIN) continue;
        const int4 gpar = __ldg(gp + ((j0 + 8 * c) >> p.gs_log2));
        const uint32_t* v8 = c < 4 ? &va[8 * c] : &vb[8 * (c - 4)];
        const uint32_t bits = ((c < 4 ? ma : mb) >> (8 * (c & 3))) & 0xffu;
        if (gpar.w & 2) {
          // float form: RZ(u * 512 r + tab0 + 256) = tab0 + (k - idx) * 512 + 9 fraction bits
          const float r9 = __int_as_float(gpar.y) * 512.0f;
          const int32_t nlo = gpar.x - gmax;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            uint32_t pw[4];
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              uint32_t u0 = (uint32_t)__viaddmax_s32((int32_t)v8[4 * q + e], nlo, 0);
              uint32_t u1 = (uint32_t)__viaddmax_s32((int32_t)v8[4 * q + e + 1], nlo, 0);
              if (!open) {
                u0 = ((bits >> (4 * q + e)) & 1u) ? 0u : u0;
                u1 = ((bits >> (4 * q + e + 1)) & 1u) ? 0u : u1;
              }
              float f0, f1;
              fma_rz_f32x2(f0, f1, __uint_as_float(u0), __uint_as_float(u1), r9, tabden);
              pw[e] = lds_u32(and_or(__float_as_uint(f0), 0xFFFFFE00u, row4));
              pw[e + 1] = lds_u32(and_or(__float_as_uint(f1), 0xFFFFFE00u, row4));
            }
            pk[2 * c + q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040),
                                        __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
          }
          continue;
        }
        GkMap gmap;
        gmap.init(gmax, gpar, k);
        if (open && gmap.use32) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t p0 = lds_u32(tab_row + ((k - gmap.idx32((int32_t)v8[4 * q], nk2)) << 9));
            const uint32_t p1 = lds_u32(tab_row + ((k - gmap.idx32((int32_t)v8[4 * q + 1], nk2)) << 9));
            const uint32_t p2 = lds_u32(tab_row + ((k - gmap.idx32((int32_t)v8[4 * q + 2], nk2)) << 9));
            const uint32_t p3 = lds_u32(tab_row + ((k - gmap.idx32((int32_t)v8[4 * q + 3], nk2)) << 9));
            pk[2 * c + q] = __byte_perm(__byte_perm(p0, p1, 0x0040), __byte_perm(p2, p3, 0x0040), 0x5410);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (!((bits >> e) & 1u))
              pk[2 * c + (e >> 2)] |= lds_u32(tab_row + ((k - gmap.idx((int32_t)v8[e], nk2, k)) << 9))
                                      << (8 * (e & 3));
        }
      }
      if (DEBUG && p.dbg_prob && i < p.L) {
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (j0 + e < p.L)
            p.dbg_prob[((size_t)bh * p.L + i) * p.L + j0 + e] = (uint8_t)(pk[e >> 2] >> (8 * (e & 3)));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t x = (uint32_t)(4 * hb + u);
        sts128(p_row + ((x ^ p_xor) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(p_full + wg * C::NPB + pbl);
    ++tl;
  }
}

template <int DP, bool DEBUG, bool SKEL = false, bool QO = false, bool GK = false>
__global__ void __launch_bounds__(Cfg<DP>::NTHREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmq,
                    const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnDev p) {
  using C = Cfg<DP>;
  constexpr int NWG = C::NWG;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint8_t lut8[256];  // static: LDS.U8 [idx + const] in the pass-2 gather
  __shared__ uint8_t lut8r[256];  // reversed: lut8r[j] = lut[k - j] (float form, j = k - idx)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int nlut = p.nlut;
  const bool wtab = wide_tab(nlut);
  uint8_t* tab = smem + C::OFF_TAB;  // row tables [nlut][128], u32 (wide) or u8 entries
  const int ntab = tab_entries(nlut);
  int32_t* xmax = reinterpret_cast<int32_t*>(tab + ntab * (wtab ? 512 : 128));  // [NWG][128]
  int32_t* xmin = xmax + 3 * 128;                                                // [NWG][128]
  uint32_t* xsum = reinterpret_cast<uint32_t*>(xmin + 3 * 128);                  // [NWG][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xsum + 3 * 128);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::NKX;
  uint64_t* v_full = k_empty + C::NKX;
  uint64_t* v_empty = v_full + C::NVST;
  uint64_t* s_full = v_empty + C::NVST;       // [NWG] QK issuer -> softmax (QK^T landed in S[w])
  uint64_t* s_free = s_full + NWG;         // [NWG] softmax -> QK issuer (S[w] fully read)
  uint64_t* p_full = s_free + NWG;         // [NWG*NPB] softmax -> P.V issuer (P^ tile in smem)
  uint64_t* p_free = p_full + NWG * C::NPB;  // [NWG*NPB] P.V issuer -> softmax (tile consumed)
  uint64_t* o_full = p_free + NWG * C::NPB;  // P.V issuer -> epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int BH = p.B * p.H;
  const int bh = blockIdx.x % BH;
  const int qt = p.n_qt - 1 - (int)(blockIdx.x / BH);  // late (heavy causal) tiles first
  const int b = bh / p.H, h = bh - (bh / p.H) * p.H;
  const int kvh = b * p.Hkv + h / (p.H / p.Hkv);
  const int q0 = qt * BM;
  const int len = p.seq_lens ? min(p.seq_lens[b], p.L) : p.L;
  // warp id through a shuffle from lane 0: ptxas then knows it is warp-uniform, so the role
  // branches are uniform branches and the role loops (barrier addresses, smem descriptors,
  // ring counters) run on the uniform datapath instead of R2UR moves per MMA -- the issue
  // loops compete for issue slots with three softmax warps on their SM sub-partition
  const int warp_u = IA_UNIFORM_WARP ? __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0) : (int)(threadIdx.x >> 5);
  // IA_UNIFORM_WARP 2: only the role dispatch sees the uniform id (softmax code unchanged)
  const int warp = IA_UNIFORM_WARP == 1 ? warp_u : (int)(threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  // Softmax warpgroups are warps 0 .. 4*NWG-1; the four role warps come last.  The
  // warp scheduler favours the highest warp id among eligible warps, so the
  // latency-critical TMA / MMA issue loops win their issue slots over the
  // arithmetic-heavy softmax warps sharing their SM sub-partition.
  // role: 0 K producer, 1 QK^T, 2 V^T producer + TMEM alloc, 3 P.V; < 0: softmax warp
  const int rw = IA_ROLE_FIRST ? (warp_u < 4 ? warp_u : -1) : warp_u - 4 * NWG;
  const int sw = IA_ROLE_FIRST ? warp - 4 : warp;  // softmax warp index (when rw < 0)
  const int stid = IA_ROLE_FIRST ? (int)threadIdx.x - 128 : (int)threadIdx.x;

  if (q0 >= len) {  // the whole query tile is padding: +0.0 rows (pipeline contract)
    const int rows = min(BM, p.L - q0);
    float* o = p.out + ((size_t)bh * p.L + q0) * p.d;
    for (int t = threadIdx.x; t < rows * p.d; t += C::NTHREADS) o[t] = 0.0f;
    return;
  }
  if (rw == 0 && lane == 0) IA_TMARK(6);
  const int key_end = p.causal ? min(q0 + BM, len) : len;
  const int n_kt = (key_end + BN - 1) / BN;
  const bool resident = n_kt <= NWG;  // every logit tile fits its own TMEM buffer
  // QO (quant-only comparator, pipeline.py:259-296): an online f32 max / sum-of-exp
  // pass, then the P / P.V pass -- two passes instead of IndexSoftmax's three.
  // GK (grouped K): pass A (S) + pass B (P / P.V), group maxima taken per tile.
  const int npass = resident ? 1 : (XF(1) ? 1 : ((QO || GK) ? 2 : 3));
  constexpr int PV_PASS = (QO || GK) ? 1 : 2;  // tile t >= PV_PASS * n_kt: the P / P.V pass
  const int n_kt_b = (XF(1)) ? 0 : n_kt;  // key tiles of passes 2-3 / P.V

  if (rw == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmq);
      prefetch_tmap(&tmk);
      prefetch_tmap(&tmv);
    }
    // the barriers are one contiguous array: each lane initialises its share (a fixed cost
    // of every CTA, ~40 serial mbarrier.init otherwise).  s_free and p_full take one arrive
    // per warp of a warpgroup, every other barrier one.
    constexpr int NB = 1 + 2 * C::NKX + 2 * C::NVST + 2 * NWG + 2 * NWG * C::NPB + 1;
    constexpr int I4_LO = 1 + 2 * C::NKX + 2 * C::NVST + NWG;  // s_free[0]
    constexpr int I4_HI = I4_LO + NWG + NWG * C::NPB;          // p_free[0]
    for (int bi = lane; bi < NB; bi += 32) mbar_init(bars + bi, (bi >= I4_LO && bi < I4_HI) ? 4 : 1);
    fence_mbar_init();
    __syncwarp();
  }
  if (rw == 2) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  for (int t = threadIdx.x; t < 256; t += C::NTHREADS) {
    lut8[t] = t < nlut ? p.lut[t] : 0;
    lut8r[t] = t < nlut ? p.lut[nlut - 1 - t] : 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = IA_UNIFORM_WARP ? __shfl_sync(0xffffffffu, *tmem_slot, 0) : *tmem_slot;
  int trc = 0;  // trace entry counter (IA_TRACE)
  (void)trc;
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // IA_TADD slots 8..15
  (void)tacc;

  // Four role warps: K producer (warp 0), QK^T issuer (warp 1), V^T producer
  // (warp 2, after the TMEM allocation), P.V issuer (warp 3).  Each role loop runs
  // warp-wide (the waits on every lane, the TMA / MMA issue on one elected lane),
  // with the smem descriptors precomputed: the issue loops sit on the pipeline's
  // critical path, and a lone-lane loop with per-iteration descriptor math was
  // measured to cost ~1000 cycles per tile.  Keeping the two MMA streams in
  // separate warps lets QK^T(n + NWG) start as soon as S[w] is read back,
  // independent of P.V(n) progress.
  if (rw == 0) {
    // ------------------------------------------------------------ K producer (+ Q)
    if (elect_one()) {
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int s = 0; s < C::NSUB; ++s)
        tma_load_3d(smem + C::OFF_Q + s * C::SUB_BYTES, &tmq, q_full, s * C::SW, q0, bh);
    }
    __syncwarp();
    uint32_t kph = 0;  // per-stage phase bits
    int n = 0, ks = 0;
    const int t3 = PV_PASS * n_kt;
    const int nloads = npass * n_kt;
    for (int t = 0; t < nloads; ++t) {
      pwait(k_empty + ks, ((kph >> ks) & 1u) ^ 1u, XF(16));
      kph ^= 1u << ks;
      if ((IA_EXP & 8) && t >= C::NKX) {
        if (elect_one()) mbar_arrive(k_full + ks);
      } else
      if (elect_one()) {
        IA_TRACE(0, 1, t);
        mbar_expect_tx(k_full + ks, C::K_BYTES);
        for (int s = 0; s < C::NSUB; ++s)
          tma_load_3d(smem + C::k_off(ks) + s * C::SUB_BYTES, &tmk, k_full + ks, s * C::SW,
                      n * BN, kvh);
      }
      __syncwarp();
      ++ks;
      if (t + 1 < t3 ? ks == C::NKX : ks == C::NKST) ks = 0;
      if (++n == n_kt) {
        n = 0;
        if (IA_QK_UNROLL) ks = 0;  // every pass starts at stage 0
      }
      if (t + 1 == t3) ks = 0;
    }
  } else if (rw == 2) {
    // ------------------------------------------------------------ V^T producer
    int vs = 0, vph = 0;
    for (int n = 0; n < n_kt_b; ++n) {
      pwait(v_empty + vs, vph ^ 1, XF(16));
      if (elect_one()) {
        IA_TRACE(2, 5, n);
        mbar_expect_tx(v_full + vs, C::V_BYTES);
        tma_load_3d(smem + C::OFF_V + vs * C::V_BYTES, &tmv, v_full + vs, n * BN, 0, kvh);
      }
      __syncwarp();
      if (++vs == C::NVST) { vs = 0; vph ^= 1; }
    }
  } else if (rw == 1) {
    // ------------------------------------------------------------ QK^T issuer
    // Tile n of every pass lives in TMEM buffer / warpgroup w = n % NWG.
    constexpr uint32_t idq = idesc_i8(BM, BN, true, true);  // s8 x s8 -> s32
    const uint64_t dq = sdesc(smem_u32(smem + C::OFF_Q), C::SBO, C::LAYOUT);
    const uint64_t d0 = sdesc(smem_u32(smem), C::SBO, C::LAYOUT);  // + (offset >> 4)
    mbar_wait(q_full, 0);
    uint32_t kph = 0;            // per-stage K phase bits
    uint32_t used = 0, c_s = 0;  // per-buffer occupied bit / s_free phase
#if IA_QK_UNROLL
    // one pass at a time; within a pass tile n uses K stage n % RING and buffer n % NWG,
    // so an unrolled round over the ring has every barrier, descriptor and TMEM column
    // offset as a compile-time constant
    const uint32_t tm = IA_UNIFORM_WARP ? tmem : *tmem_slot;  // (re-read: keeps the loop free of a spilled reload)
    // s_free parity starts at 1: a fresh barrier counts its (nonexistent) previous
    // phase as complete, so every buffer's first use passes without a special case
    uint32_t f_ph = (1u << NWG) - 1u;
    auto qk_tile = [&](auto J) {
      constexpr int ks = decltype(J)::value;
      constexpr int w = ks % NWG;
      const long long t0 = clk64();
      const uint32_t f_ok = mbar_test(s_free + w, (f_ph >> w) & 1u);
      const uint32_t k_ok = mbar_test(k_full + ks, (kph >> ks) & 1u);
      if (!f_ok) iwait(s_free + w, (f_ph >> w) & 1u, (IA_QK_SPIN & 1) || XF(2));
      f_ph ^= 1u << w;
      const long long t1 = clk64();
      if (!k_ok) iwait(k_full + ks, (kph >> ks) & 1u, (IA_QK_SPIN & 2) || XF(2));
      kph ^= 1u << ks;
      IA_TADD(8, t1 - t0);
      IA_TADD(9, clk64() - t1);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t dk = d0 + (uint64_t)(C::k_off(ks) >> 4);
#pragma unroll
        for (int kk = 0; kk < C::KSTEPS; ++kk) {
          const uint32_t off = (kk * 32 / C::SW) * C::SUB_BYTES + (kk * 32) % C::SW;
          mma_i8_ss(tm + (uint32_t)w * 128u, dq + (off >> 4), dk + (off >> 4), idq, kk > 0);
        }
        tc_commit(k_empty + ks);
        tc_commit(s_full + w);
      }
      __syncwarp();
      if (IA_QK_DELAY_NS > 0) __nanosleep(IA_QK_DELAY_NS);
    };
    for (int pass = 0; pass < (resident ? 0 : npass); ++pass) {  // resident: generic loop
      if (pass < PV_PASS) {
        for (int n0 = 0; n0 < n_kt; n0 += C::NKX)
          static_for<C::NKX>([&](auto J) {
            if (n0 + decltype(J)::value < n_kt) qk_tile(J);
          });
      } else {
        for (int n0 = 0; n0 < n_kt; n0 += C::NKST)
          static_for<C::NKST>([&](auto J) {
            if (n0 + decltype(J)::value < n_kt) qk_tile(J);
          });
      }
    }
    if (resident)
#endif
    for (int t = 0, w = 0, n = 0, ks = 0, t3 = PV_PASS * n_kt; t < npass * n_kt; ++t) {
      long long t0 = clk64();
      if (lane == 0) IA_TRACE(1, 2, t);
      // both readiness tests in flight at once; block only on what is not ready yet
      const bool need_free = (used >> w) & 1u;
      const uint32_t f_ok = need_free ? mbar_test(s_free + w, (c_s >> w) & 1u) : 1u;
      const uint32_t k_ok = mbar_test(k_full + ks, (kph >> ks) & 1u);
      if (!f_ok) iwait(s_free + w, (c_s >> w) & 1u, XF(2));
      if (need_free) c_s ^= 1u << w;
      used |= 1u << w;
      if (lane == 0) IA_TRACE(1, 5, t);
      long long t1 = clk64();
      if (!k_ok) iwait(k_full + ks, (kph >> ks) & 1u, (IA_QK_SPIN & 2) || XF(2));
      kph ^= 1u << ks;
      long long t2 = clk64();
      IA_TADD(8, t1 - t0);
      IA_TADD(9, t2 - t1);
      tc_fence_after();
      if (elect_one()) {
        IA_TRACE(1, 3, t);
        const uint64_t dk = d0 + (uint64_t)(C::k_off(ks) >> 4);
        const uint32_t dt = tmem + (uint32_t)w * 128u;
#pragma unroll
        for (int kk = 0; kk < C::KSTEPS; ++kk) {
          const uint32_t off = (kk * 32 / C::SW) * C::SUB_BYTES + (kk * 32) % C::SW;
          mma_i8_ss(dt, dq + (off >> 4), dk + (off >> 4), idq, kk > 0);
        }
        tc_commit(k_empty + ks);
        tc_commit(s_full + w);
        IA_TRACE(1, 4, t);
      }
      __syncwarp();
      if (++w == NWG) w = 0;
      ++ks;
      if (t + 1 < t3 ? ks == C::NKX : ks == C::NKST) ks = 0;
      if (++n == n_kt) {
        n = 0;
        w = 0;
      }
      if (t + 1 == t3) ks = 0;
    }
  } else if (rw == 3) {
    // ------------------------------------------------------------ P.V issuer
    constexpr uint32_t idv = idesc_i8(BM, DP, false, true);  // u8 x s8 -> s32
    const uint64_t dp0 = sdesc(smem_u32(smem + C::OFF_P), 1024, 2u);
    const uint64_t dv0 = sdesc(smem_u32(smem + C::OFF_V), 1024, 2u);
#if IA_PV_UNROLL
    // unrolled over one period of (P^ buffer, V^T stage): tile n uses P^ buffer
    // (n % NWG) * NPB + (n / NWG) % NPB and V^T stage n % NVST -- compile-time in a round
    if (!resident) {
      constexpr int PER = lcm_i(NWG * C::NPB, C::NVST);
      static_assert(PER % C::NVST == 0 && PER % (NWG * C::NPB) == 0, "P.V unroll period");
      const uint32_t tm = *tmem_slot;
      uint32_t pph = 0, vph2 = 0;  // P^ round parity, V^T phase bits per stage
      for (int n0 = 0; n0 < n_kt_b; n0 += PER) {
        static_for<PER>([&](auto J) {
          constexpr int j = decltype(J)::value;
          constexpr int pb = (j % NWG) * C::NPB + (j / NWG) % C::NPB;
          constexpr int vs = j % C::NVST;
          if (n0 + j >= n_kt_b) return;
          iwait(p_full + pb, (pph ^ (uint32_t)((j / (NWG * C::NPB)) & 1)) & 1u, XF(8));
          iwait(v_full + vs, (vph2 >> vs) & 1u, XF(8));
          vph2 ^= 1u << vs;
          tc_fence_after();
          if (elect_one()) {
            const uint64_t dp = dp0 + (uint64_t)((pb * C::P_BYTES) >> 4);
            const uint64_t dv = dv0 + (uint64_t)((vs * C::V_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < BN / 32; ++kk)
              mma_i8_ss(tm + C::O_COL, dp + 2 * kk, dv + 2 * kk, idv,
                        (n0 + j > 0 || kk > 0) ? 1u : 0u);
            tc_commit(v_empty + vs);
            tc_commit(p_free + pb);
          }
          __syncwarp();
        });
        pph ^= (uint32_t)((PER / (NWG * C::NPB)) & 1);
      }
    }
#endif
    int vs = 0, vph = 0, w = 0, tl = 0;  // warpgroup w's local tile counter tl
    for (int n = 0; n < ((IA_PV_UNROLL && !resident) ? 0 : n_kt_b); ++n) {
      const int pb = w * C::NPB + tl % C::NPB;
      long long t0 = clk64();
      iwait(p_full + pb, (uint32_t)(tl / C::NPB) & 1u, XF(8));
      long long t1 = clk64();
      iwait(v_full + vs, vph, XF(8));
      long long t2 = clk64();
      IA_TADD(11, t1 - t0);
      IA_TADD(12, t2 - t1);
      tc_fence_after();
      if (elect_one()) {
        IA_TRACE(3, 7, n);
        const uint64_t dp = dp0 + (uint64_t)((pb * C::P_BYTES) >> 4);
        const uint64_t dv = dv0 + (uint64_t)((vs * C::V_BYTES) >> 4);
#pragma unroll
        for (int kk = 0; kk < BN / 32; ++kk)
          mma_i8_ss(tmem + C::O_COL, dp + 2 * kk, dv + 2 * kk, idv, (n > 0 || kk > 0) ? 1u : 0u);
        tc_commit(v_empty + vs);
        tc_commit(p_free + pb);
      }
      __syncwarp();
      if (IA_PV_DELAY_NS > 0) __nanosleep(IA_PV_DELAY_NS);
      if (++vs == C::NVST) { vs = 0; vph ^= 1; }
      if (++w == NWG) { w = 0; ++tl; }
    }
    if (elect_one()) tc_commit(o_full);
    __syncwarp();
  } else if (rw < 0) {
    // ------------------------------------------------------------ IndexSoftmax warpgroups
    const int wg = sw >> 2;
    const int quad = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int row = quad * 32 + lane;
    const int i = q0 + row;
    const bool row_valid = i < len;
    const uint32_t t_lane = (uint32_t)(quad * 32) << 16;
    const uint32_t s_base = tmem + t_lane + (uint32_t)(wg * 128);
    const int lim = p.causal ? min(i, len - 1) : len - 1;  // last unmasked key of this row
    const ia_head_params hp = p.params[bh];
    const uint32_t k = (uint32_t)(nlut - 1);
    constexpr int NWT = 128 * NWG;  // softmax threads
    uint32_t s_ph = 0;              // phase of s_full[wg]

    // Each tile is read from TMEM in two 64-column batches (two x32 loads in
    // flight per wait); S[w] is handed back to the MMA warp right after the last
    // load of the tile, in every pass.
    const bool tm = (stid == 0);
    const bool trw = IA_PROFILE && lane == 0;  // one trace segment per softmax warp
    if (tm) IA_TMARK(0);
    if constexpr (GK) {
      gk_passes<DP, DEBUG>(p, smem, reinterpret_cast<uint32_t*>(tab), xsum, lut8, lut8r, s_full, s_free,
                           p_full, p_free, s_base, wg, row, lane, i, lim, bh, n_kt, row_valid,
                           resident, s_ph);
    } else {
    // Float (denormal) form of the index map (params.cuh): one path for every row, clip
    // included, so pass 1 needs the row max only.
    const float rf = hp.fratio;  // 0: c_eff too large for the float form
    // (needs the u32 row tables and cut-off masks only: dense masks take the generic path)
    const bool flc = IA_FLOAT_IDX && rf != 0.0f && wtab && !p.mask_bits;
    // ---- pass 1: row max over unmasked keys (softmax.py:139-143, :174-179); for the
    // integer map the row min rides along to size the unclipped index range
    int32_t mx = INT_MIN, mn = INT_MAX;
    // QO: running max (real units) and sum of exp(real - qm); real = f32(a) * alpha in f32
    // as the reference (pipeline.py:277-279); f32(a) * alpha is monotone in a, so the
    // chunk max is taken on the integers.
    const float alpha = QO ? (float)((double)hp.s_q * (double)hp.s_k / sqrt((double)p.d)) : 0.0f;
    constexpr float L2E = 1.4426950408889634f;
    float qm = -INFINITY, qs = 0.0f;
    for (int n = wg; n < n_kt; n += NWG) {
      long long tw0 = clk64();
      bwait(s_full + wg, s_ph, IA_P1_SPIN || XF(4));
      if (trw) IA_TRACE(4 + sw, 8, 0 * n_kt + n);
      s_ph ^= 1u;
      if (tm) IA_TADD(15, clk64() - tw0);
      tc_fence_after();
#pragma unroll 1
      for (int hb = 0; hb < BN / 64; ++hb) {
        uint32_t va[32], vb[32];
        tmem_ld64(s_base + hb * 64, va, vb);
        if (hb == BN / 64 - 1 && !resident) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + wg);
          if (trw) IA_TRACE(4 + sw, 9, 0 * n_kt + n);
        }
        const int j0 = n * BN + hb * 64;
        if (DEBUG && p.dbg_logits && i < p.L) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            int32_t* dl = p.dbg_logits + ((size_t)bh * p.L + i) * p.L + j0;
            if (j0 + e < p.L) dl[e] = (int32_t)va[e];
            if (j0 + 32 + e < p.L) dl[32 + e] = (int32_t)vb[e];
          }
        }
        // Causal / length masking is a per-row cut-off: keys j0 + e with e >= cut are
        // excluded (cut <= 0: whole batch; invalid rows: cut = 0).  Dense masks take
        // the bitmask path.
        const int cut = row_valid ? lim - j0 + 1 : 0;
        if (QO) {
          const uint32_t ma = p.mask_bits ? (row_valid ? chunk_mask(p, i, j0, lim) : ~0u)
                                          : (cut >= 32 ? 0u : (cut <= 0 ? ~0u : (0xffffffffu << cut)));
          const uint32_t mbb = p.mask_bits ? (row_valid ? chunk_mask(p, i, j0 + 32, lim) : ~0u)
                                           : (cut >= 64 ? 0u : (cut <= 32 ? ~0u : (0xffffffffu << (cut - 32))));
          int32_t cmx = INT_MIN;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (!((ma >> e) & 1u)) cmx = max(cmx, (int32_t)va[e]);
            if (!((mbb >> e) & 1u)) cmx = max(cmx, (int32_t)vb[e]);
          }
          if (cmx != INT_MIN) {
            const float cm = __fmul_rn(__int2float_rn(cmx), alpha);
            if (cm > qm) { qs *= ex2_approx(__fmul_rn(qm - cm, L2E)); qm = cm; }
            const float mL = qm * L2E;
            float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float xa = ex2_approx(fmaf(__fmul_rn(__int2float_rn((int32_t)va[e]), alpha), L2E, -mL));
              const float xb = ex2_approx(fmaf(__fmul_rn(__int2float_rn((int32_t)vb[e]), alpha), L2E, -mL));
              acc0 += ((ma >> e) & 1u) ? 0.0f : xa;
              acc1 += ((mbb >> e) & 1u) ? 0.0f : xb;
            }
            qs += acc0 + acc1;
          }
        } else if (XF(32)) {  // experiment: no pass-1 arithmetic
        } else if (!p.mask_bits) {
          if (!__any_sync(0xffffffffu, cut < 64)) {
            // two 3-input VIMNMX3 chains per direction: one instruction per two logits
            int32_t mx1 = mx, mn1 = mn;
            if (flc && IA_P1_CHAINS == 4) {
              int32_t mx2 = mx, mx3 = mx;
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                mx = __vimax3_s32(mx, (int32_t)va[e], (int32_t)va[e + 1]);
                mx1 = __vimax3_s32(mx1, (int32_t)vb[e], (int32_t)vb[e + 1]);
                mx2 = __vimax3_s32(mx2, (int32_t)va[e + 16], (int32_t)va[e + 17]);
                mx3 = __vimax3_s32(mx3, (int32_t)vb[e + 16], (int32_t)vb[e + 17]);
              }
              mx = __vimax3_s32(mx, mx2, mx3);
            } else if (flc) {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                mx = __vimax3_s32(mx, (int32_t)va[e], (int32_t)va[e + 1]);
                mx1 = __vimax3_s32(mx1, (int32_t)vb[e], (int32_t)vb[e + 1]);
              }
            } else {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                mx = __vimax3_s32(mx, (int32_t)va[e], (int32_t)va[e + 1]);
                mx1 = __vimax3_s32(mx1, (int32_t)vb[e], (int32_t)vb[e + 1]);
                mn = __vimin3_s32(mn, (int32_t)va[e], (int32_t)va[e + 1]);
                mn1 = __vimin3_s32(mn1, (int32_t)vb[e], (int32_t)vb[e + 1]);
              }
            }
            mx = max(mx, mx1);
            mn = min(mn, mn1);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (e < cut) { mx = max(mx, (int32_t)va[e]); mn = min(mn, (int32_t)va[e]); }
              if (e + 32 < cut) { mx = max(mx, (int32_t)vb[e]); mn = min(mn, (int32_t)vb[e]); }
            }
          }
        } else if (row_valid) {
          const uint32_t ma = chunk_mask(p, i, j0, lim), mbb = chunk_mask(p, i, j0 + 32, lim);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (!((ma >> e) & 1u)) { mx = max(mx, (int32_t)va[e]); mn = min(mn, (int32_t)va[e]); }
            if (!((mbb >> e) & 1u)) { mx = max(mx, (int32_t)vb[e]); mn = min(mn, (int32_t)vb[e]); }
          }
        }
      }
    }
    if (tm) IA_TMARK(1);
    if (QO) {
      xmax[wg * 128 + row] = __float_as_int(qm);
      xsum[wg * 128 + row] = __float_as_uint(qs);
    } else {
      xmax[wg * 128 + row] = mx;
      xmin[wg * 128 + row] = mn;
    }
    named_bar_sync(1, NWT);
    int32_t m = 0;
    float q_ksc = 0.0f, q_mL = 0.0f;  // QO: p_scale / sum, rowmax * log2(e)
    bool dead;
    if (QO) {
      float M = -INFINITY, Ssum = 0.0f;
#pragma unroll
      for (int w = 0; w < NWG; ++w) M = fmaxf(M, __int_as_float(xmax[w * 128 + row]));
#pragma unroll
      for (int w = 0; w < NWG; ++w) {
        const float mw = __int_as_float(xmax[w * 128 + row]);
        if (mw != -INFINITY) Ssum += __uint_as_float(xsum[w * 128 + row]) * ex2_approx(__fmul_rn(mw - M, L2E));
      }
      dead = !(M > -INFINITY) || !(Ssum > 0.0f);  // fully masked row -> zeros (pipeline.py:122-127)
      q_ksc = dead ? 0.0f : (float)p.scale_x2 * 0.5f / Ssum;
      q_mL = dead ? 0.0f : M * L2E;
      named_bar_sync(1, NWT);  // xsum is reused below
    } else {
      m = xmax[row];
      mn = xmin[row];
#pragma unroll
      for (int w = 1; w < NWG; ++w) {
        m = max(m, xmax[w * 128 + row]);
        mn = min(mn, xmin[w * 128 + row]);
      }
      dead = (m == INT_MIN);  // fully masked row: all-zero P^ (softmax.py:181-184)
    }
    if (dead) m = 0;
    const bool fast = hp.use32 != 0;
    // the clipped distance delta = c_eff itself fits the 32-bit map (it need not when c_eff
    // exceeds every reachable distance): cut-off chunks may then park excluded keys at lo
    const bool fastc = fast && (2 * (int64_t)k + 1) * hp.c_eff < (int64_t(1) << 31);
    IdxMap im;
    im.init(m, hp, k);
    // Largest index any unmasked logit of this warp's rows can reach without the
    // clip; if it fits the zero-extended tables, passes 2-3 skip the clip.
    uint32_t idx_hi = 0;
    if (row_valid && !dead && hp.unc32) {
      const int64_t dmax = (int64_t)m - (int64_t)mn;
      const int64_t hi = (2 * (int64_t)k * dmax + hp.c_eff) / (2 * hp.c_eff);
      idx_hi = hi > 0x7fffffff ? 0x7fffffffu : (uint32_t)hi;
    }
    idx_hi = __reduce_max_sync(0xffffffffu, idx_hi);
    const bool uncl2 = !flc && hp.unc32 && idx_hi < 256u;                      // lut8 has 256 entries
    const bool uncl3 = !flc && hp.unc32 && wtab && idx_hi < (uint32_t)ntab;  // zero-extended row table
    // Float form: u = max(a - lo, 0) = c_eff - delta' (one VIADDMNMX, the clip comes free),
    // read as an f32 bit pattern, IS the denormal u * 2^-149; one FMA with a denormal addend
    // A * 2^-149 leaves j + A in the result's bit pattern, j = k - idx: a shared-memory
    // address into the reversed LUT (pass 2) / reversed row table (pass 3).
    const float rf9 = rf * 512.0f;  // pass 3: j * 512 + 9 fraction bits
    const float lutden = __uint_as_float(smem_u32(lut8r));  // pass 2 addend: &lut8r[0]
    const int32_t nlo = (int32_t)(hp.c_eff - (int64_t)m);    // -lo (flc: |lo| < 2^31)

    // ---- pass 2: idx, e = lut[idx], S = sum e (softmax.py:144-155)
    uint32_t S = 0;
    for (int n = wg; n < (QO ? 0 : n_kt_b); n += NWG) {
      if (!resident) {
        long long tw0 = clk64();
        bwait(s_full + wg, s_ph, XF(4));
        if (trw) IA_TRACE(4 + sw, 8, 1 * n_kt + n);
        s_ph ^= 1u;
        if (tm) IA_TADD(14, clk64() - tw0);
      }
      tc_fence_after();
#pragma unroll 1
      for (int hb = 0; hb < BN / 64; ++hb) {
        uint32_t va[32], vb[32];
        tmem_ld64(s_base + hb * 64, va, vb);
        if (hb == BN / 64 - 1 && !resident) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + wg);
          if (trw) IA_TRACE(4 + sw, 9, 1 * n_kt + n);
        }
        if (SKEL) continue;
        const int j0 = n * BN + hb * 64;
        // masked keys (e >= cut) take idx = k, lut[k] = 0 (softmax.py:187-188); dead /
        // invalid rows (cut = 0) sum to S = 0 and get an all-zero table
        const int cut = (row_valid && !dead) ? lim - j0 + 1 : 0;
        const bool any_cut = __any_sync(0xffffffffu, cut < 64);
        if (!p.mask_bits && fast && (!any_cut || fastc)) {
          if (any_cut) {
            // Cut-off chunk (diagonal / ragged tile): nothing to add if every key of every
            // row is excluded; else excluded keys take the clip floor lo (delta = c_eff ->
            // idx = k, lut[k] = 0) and the chunk runs the clipped fast path.
            if (!__any_sync(0xffffffffu, cut > 0)) continue;
            const uint32_t lo_u = (uint32_t)im.lo;
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              va[e] = e < cut ? va[e] : lo_u;
              vb[e] = e + 32 < cut ? vb[e] : lo_u;
            }
          }
          const bool unc = uncl2 && !any_cut;
          if (flc) {
            // RN(u * r + &lut8r) in denormal units: the bit pattern is &lut8r[k - idx]
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const uint32_t ua = (uint32_t)__viaddmax_s32((int32_t)va[e], nlo, 0);
              const uint32_t ub = (uint32_t)__viaddmax_s32((int32_t)vb[e], nlo, 0);
              float fa, fb;
              fma_rn_f32x2(fa, fb, __uint_as_float(ua), __uint_as_float(ub), rf, lutden);
              if (IA_EXP & 1) S += (__float_as_uint(fa) & 255u) + (__float_as_uint(fb) & 255u);
              else S += lds_u8(__float_as_uint(fa)) + lds_u8(__float_as_uint(fb));
            }
          } else if (unc) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              S += (uint32_t)lut8[im.idx_u((int32_t)va[e])] + (uint32_t)lut8[im.idx_u((int32_t)vb[e])];
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              S += (uint32_t)lut8[im.idx_s((int32_t)va[e])] + (uint32_t)lut8[im.idx_s((int32_t)vb[e])];
          }
        } else if (row_valid && !dead) {
          const uint32_t ma = chunk_mask(p, i, j0, lim), mbb = chunk_mask(p, i, j0 + 32, lim);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (!((ma >> e) & 1u))
              S += lut8[fast ? im.idx((int32_t)va[e]) : idx_slow(m, (int32_t)va[e], hp.c_eff, k)];
            if (!((mbb >> e) & 1u))
              S += lut8[fast ? im.idx((int32_t)vb[e]) : idx_slow(m, (int32_t)vb[e], hp.c_eff, k)];
          }
        }
      }
    }
    if (tm) IA_TMARK(2);
    if (!QO) {
    xsum[wg * 128 + row] = S;
    named_bar_sync(1, NWT);
    S = xsum[row];
#pragma unroll
    for (int w = 1; w < NWG; ++w) S += xsum[w * 128 + row];
    // per-row normalisation table (softmax.py:157-160): (2*scale*lut[t] + S) // (2S)
    {
      // num < 2^25 and 2S < 2^25 (S <= 255 * 65536): the f32 quotient is within 0.02
      // of the exact one, so one remainder check makes it the exact floor
      const uint32_t two_s = 2u * S;
      const float rden = S ? __frcp_rn((float)two_s) : 0.0f;
      // float form: only entries j = k - t, t <= k, are ever addressed (u <= c_eff), so the
      // zero-extension of the integer form's table is not built (short rows: the table
      // build is a fixed cost per CTA)
      const int nbuild = flc ? nlut : ntab;
      // Branch-free, shared-window addressing (a fixed cost of every CTA: ~11 entries per
      // thread).  lt = 0 (a zero LUT entry, t >= nlut, or S = 0) gives num = S, q = 0.
      const uint32_t lut_s = smem_u32(lut8), tab_s = smem_u32(tab);
      const uint32_t sx2 = (uint32_t)p.scale_x2;
      const int kk = (int)k;
      if (wtab) {
        // entry address: (tt * 128 + row) * 4; float form: tt = k - t for t <= k
        const uint32_t a_row = tab_s + (uint32_t)row * 4u;
#pragma unroll 4
        for (int t = wg; t < nbuild; t += NWG) {
          const uint32_t lt = S ? lds_u8(lut_s + (uint32_t)t) : 0u;
          const uint32_t num = sx2 * lt + S;
          int32_t q = __float2int_rz(__fmul_rn((float)num, rden));
          const int32_t r = (int32_t)num - q * (int32_t)two_s;
          q += r < 0 ? -1 : (r >= (int32_t)two_s ? 1 : 0);
          const int tt = (flc && t <= kk) ? kk - t : t;
          sts_u32(a_row + ((uint32_t)tt << 9), S ? (uint32_t)q : 0u);
        }
      } else {
        for (int t = wg; t < nbuild; t += NWG) {
          const uint32_t lt = lut8[t];
          uint32_t pv = 0u;
          if (S && lt) {
            const uint32_t num = sx2 * lt + S;
            int32_t q = __float2int_rz(__fmul_rn((float)num, rden));
            const int32_t r = (int32_t)num - q * (int32_t)two_s;
            q += r < 0 ? -1 : (r >= (int32_t)two_s ? 1 : 0);
            pv = (uint32_t)q;
          }
          tab[t * 128 + row] = (uint8_t)pv;
        }
      }
    }
    named_bar_sync(1, NWT);
    }
    // entry idx of this row: wide: tab_row + idx * 512 (u32), else tab_row + idx * 128 (u8)
    const uint32_t tab_row = smem_u32(tab) + (uint32_t)row * (wtab ? 4u : 1u);
    const uint32_t tab_sh = wtab ? 9u : 7u;
    const uint32_t tab0 = smem_u32(tab), row4 = (uint32_t)row * 4u;
    const uint32_t m9 = (wtab && !(XF(256))) ? hp.magic9 : 0u;
    // Row threshold of the pass-3 group skip: P^ = rowtab[idx] > 0 only for idx <= t*,
    // t* = max{t : 2*scale*lut[t] >= S} (rowtab[t] = (2 scale lut[t] + S) // 2S), i.e.
    // only for delta < T = ceil(c_eff (2t* + 1) / 2k) (idx(delta) > t* from there on),
    // i.e. only for logits a >= theta = m - T + 1.  A group of keys whose largest logit
    // is below theta in every row of the warp is all zero.  Scans every LUT entry, so
    // it holds for any LUT (no monotonicity assumed).
    // Only rows long enough for P^ to be sparse pay the per-row scan (n_kt >= IA_SKIP_MIN_KT);
    // shorter rows keep theta = INT_MIN (no group is skipped).
    int32_t theta = n_kt >= IA_SKIP_MIN_KT ? INT_MAX : INT_MIN;
    if (!QO && (m9 || flc) && n_kt >= IA_SKIP_MIN_KT && row_valid && !dead && S) {
      int tstar = -1;
      for (int t = 0; t < nlut; ++t)
        if ((uint32_t)p.scale_x2 * (uint32_t)lut8[t] >= S) tstar = t;
      if (tstar >= 0) {
        const int64_t T = (hp.c_eff * (2 * (int64_t)tstar + 1) + 2 * (int64_t)k - 1) / (2 * (int64_t)k);
        const int64_t th = (int64_t)m - T + 1;
        theta = th < (int64_t)INT_MIN ? INT_MIN : (th > (int64_t)INT_MAX ? INT_MAX : (int32_t)th);
      }
    }
    // this thread's row of its warpgroup's P^ tile (K-major, 128B swizzle: 16-byte
    // unit x of row r lives at unit x ^ (r % 8))
    const uint32_t p_rows = smem_u32(smem + C::OFF_P + wg * C::NPB * C::P_BYTES) + (uint32_t)row * 128;
    const uint32_t p_xor = (uint32_t)(row & 7);
    int tl = 0;  // this warpgroup's local pass-3 tile counter

    // ---- pass 3: P^ = rowtab[idx] -> smem -> P.V MMA (softmax.py:161-162)
    for (int n = wg; n < n_kt_b; n += NWG) {
      if (!resident) {
        long long tw0 = clk64();
        bwait(s_full + wg, s_ph, XF(4));
        if (trw) IA_TRACE(4 + sw, 8, 2 * n_kt + n);
        s_ph ^= 1u;
        if (tm) IA_TADD(14, clk64() - tw0);
      }
      tc_fence_after();
      const int pbl = tl % C::NPB;
      const uint32_t p_row = p_rows + (uint32_t)(pbl * C::P_BYTES);
      // the P.V that last read this P^ buffer must be done (first use passes at once)
      long long tq0 = clk64();
      mbar_wait(p_free + wg * C::NPB + pbl, ((uint32_t)(tl / C::NPB) & 1u) ^ 1u);
      if (trw) IA_TRACE(4 + sw, 10, 2 * n_kt + n);
      if (tm) IA_TADD(13, clk64() - tq0);
#pragma unroll 1
      for (int hb = 0; hb < BN / 64; ++hb) {
        uint32_t va[32], vb[32];
        tmem_ld64(s_base + hb * 64, va, vb);
        if (hb == BN / 64 - 1 && !resident) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + wg);
          if (trw) IA_TRACE(4 + sw, 9, 2 * n_kt + n);
        }
        const int j0 = n * BN + hb * 64;
        uint32_t pk[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pk[q] = 0u;
        const int cut = (row_valid && !dead) ? lim - j0 + 1 : 0;
        const bool any_cut = __any_sync(0xffffffffu, cut < 64);
        if (SKEL) {
        } else if (QO) {
          // p^ = floor(exp(real - max) * (scale / sum) + 0.5) (pipeline.py:130-140, 281)
          if (row_valid && !dead) {
            const uint32_t ma = p.mask_bits ? chunk_mask(p, i, j0, lim)
                                            : (cut >= 32 ? 0u : (cut <= 0 ? ~0u : (0xffffffffu << cut)));
            const uint32_t mbb = p.mask_bits ? chunk_mask(p, i, j0 + 32, lim)
                                             : (cut >= 64 ? 0u : (cut <= 32 ? ~0u : (0xffffffffu << (cut - 32))));
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float xa = ex2_approx(fmaf(__fmul_rn(__int2float_rn((int32_t)va[e]), alpha), L2E, -q_mL));
              const float xb = ex2_approx(fmaf(__fmul_rn(__int2float_rn((int32_t)vb[e]), alpha), L2E, -q_mL));
              const uint32_t ba = ((ma >> e) & 1u) ? 0u : min(__float2uint_rz(fmaf(xa, q_ksc, 0.5f)), 255u);
              const uint32_t bb = ((mbb >> e) & 1u) ? 0u : min(__float2uint_rz(fmaf(xb, q_ksc, 0.5f)), 255u);
              pk[e >> 2] |= ba << (8 * (e & 3));
              pk[8 + (e >> 2)] |= bb << (8 * (e & 3));
            }
          }
        } else if (!p.mask_bits && fast && wtab && (!any_cut || fastc)) {
          bool live = true;  // some key of some row of the warp is not excluded
          if (any_cut) {
            // cut-off chunk: excluded keys take the clip floor lo (idx = k, table entry 0)
            // and the chunk runs the clipped fast path; all excluded: P^ = 0
            live = __any_sync(0xffffffffu, cut > 0);
            if (live) {
              const uint32_t lo_u = (uint32_t)im.lo;
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                va[e] = e < cut ? va[e] : lo_u;
                vb[e] = e + 32 < cut ? vb[e] : lo_u;
              }
            }
          }
          const bool unc = uncl3 && !any_cut;
          if (!live) {
          } else if (flc) {
            // RZ(u * 512 r + tab0 + 256) in denormal units: tab0 + (k - idx) * 512 + 9
            // fraction bits; the (reversed) row-table address is one LOP3 away
            const float tabden = __uint_as_float(tab0 + 256u);
            auto fgroups = [&](auto skip) {
              constexpr int G = IA_SKIP_G;  // keys per skip group
              // IA_SKIP_MASK: all group maxima first (64 / G independent chains), one
              // warp-wide OR of the per-lane live bits, then uniform branches -- instead
              // of a max chain + vote + branch per group (a serial ~45-cycle chain each)
              uint32_t live_groups = 0xffffffffu;
              if (decltype(skip)::value && IA_SKIP_MASK) {
                uint32_t lm = 0u;
#pragma unroll
                for (int g = 0; g < 64 / G; ++g) {
                  const uint32_t* vg = g < 32 / G ? &va[G * g] : &vb[G * (g - 32 / G)];
                  int32_t gm = (int32_t)vg[0];
#pragma unroll
                  for (int e = 1; e < G; ++e) gm = max(gm, (int32_t)vg[e]);
                  lm |= gm >= theta ? (1u << g) : 0u;
                }
                live_groups = __reduce_or_sync(0xffffffffu, lm);
              }
#pragma unroll
              for (int g = 0; g < 64 / G; ++g) {
                const uint32_t* vg = g < 32 / G ? &va[G * g] : &vb[G * (g - 32 / G)];
                if (decltype(skip)::value && IA_SKIP_MASK) {
                  if (!((live_groups >> g) & 1u)) continue;  // pk stays 0
                } else if (decltype(skip)::value) {
                  int32_t gm = (int32_t)vg[0];
#pragma unroll
                  for (int e = 1; e < G; ++e) gm = max(gm, (int32_t)vg[e]);
                  if (!__any_sync(0xffffffffu, gm >= theta)) continue;  // pk stays 0
                }
#pragma unroll
                for (int q = 0; q < G / 4; ++q) {
                  const uint32_t* v4 = vg + 4 * q;
                  uint32_t pw[4];
#pragma unroll
                  for (int e = 0; e < 4; e += 2) {
                    const uint32_t u0 = (uint32_t)__viaddmax_s32((int32_t)v4[e], nlo, 0);
                    const uint32_t u1 = (uint32_t)__viaddmax_s32((int32_t)v4[e + 1], nlo, 0);
                    float f0, f1;
                    fma_rz_f32x2(f0, f1, __uint_as_float(u0), __uint_as_float(u1), rf9, tabden);
                    if (IA_EXP & 2) {
                      pw[e] = and_or(__float_as_uint(f0), 0xFFFFFE00u, row4) >> 9;
                      pw[e + 1] = and_or(__float_as_uint(f1), 0xFFFFFE00u, row4) >> 9;
                    } else {
                    pw[e] = lds_u32(and_or(__float_as_uint(f0), 0xFFFFFE00u, row4));
                    pw[e + 1] = lds_u32(and_or(__float_as_uint(f1), 0xFFFFFE00u, row4));
                    }
                  }
                  pk[(G / 4) * g + q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040),
                                                    __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
                }
              }
            };
            if (IA_GROUP_SKIP && n_kt >= IA_SKIP_MIN_KT) fgroups(std::true_type{});
            else fgroups(std::false_type{});
          } else if (m9) {
            // address = tab0 + ((umulhi(n, magic9) & ~511) | row*4): IMAD, IMAD.HI, LOP3,
            // LDS per logit (+ the clip VIMNMX when the warp's index range exceeds the
            // table).  Groups of 16 keys below every row's threshold stay zero.
            const uint32_t nk2 = im.nk2, base = im.base;
            const int32_t lo = im.lo;
            auto groups = [&](auto clip, auto skip) {
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                const uint32_t* v16 = g < 2 ? &va[16 * g] : &vb[16 * (g - 2)];
                if (decltype(skip)::value) {
                  int32_t gm = (int32_t)v16[0];
#pragma unroll
                  for (int e = 1; e < 16; ++e) gm = max(gm, (int32_t)v16[e]);
                  if (!__any_sync(0xffffffffu, gm >= theta)) continue;  // pk stays 0
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t* v4 = v16 + 4 * q;
                  uint32_t pw[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const int32_t x = decltype(clip)::value ? max((int32_t)v4[e], lo) : (int32_t)v4[e];
                    const uint32_t n = base + nk2 * (uint32_t)x;
                    pw[e] = lds_u32(tab0 + and_or(__umulhi(n, m9), 0xFFFFFE00u, row4));
                  }
                  pk[4 * g + q] = __byte_perm(__byte_perm(pw[0], pw[1], 0x0040),
                                              __byte_perm(pw[2], pw[3], 0x0040), 0x5410);
                }
              }
            };
            // short rows (theta = INT_MIN) take the branch-free form: all 64 logits
            // interleave freely
            const bool skip = IA_GROUP_SKIP && n_kt >= IA_SKIP_MIN_KT;
            if (unc) {
              if (skip) groups(std::false_type{}, std::true_type{});
              else groups(std::false_type{}, std::false_type{});
            } else {
              if (skip) groups(std::true_type{}, std::true_type{});
              else groups(std::true_type{}, std::false_type{});
            }
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const uint32_t* v4 = q < 8 ? &va[4 * q] : &vb[4 * (q - 8)];
              const uint32_t p0 = lds_u32(tab_row + (im.idx_s((int32_t)v4[0]) << 9));
              const uint32_t p1 = lds_u32(tab_row + (im.idx_s((int32_t)v4[1]) << 9));
              const uint32_t p2 = lds_u32(tab_row + (im.idx_s((int32_t)v4[2]) << 9));
              const uint32_t p3 = lds_u32(tab_row + (im.idx_s((int32_t)v4[3]) << 9));
              pk[q] = __byte_perm(__byte_perm(p0, p1, 0x0040), __byte_perm(p2, p3, 0x0040), 0x5410);
            }
          }
        } else if (row_valid && !dead) {
          const uint32_t ma = chunk_mask(p, i, j0, lim), mbb = chunk_mask(p, i, j0 + 32, lim);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint32_t xa = ((ma >> e) & 1u) ? k
                                : fast ? im.idx((int32_t)va[e])
                                       : idx_slow(m, (int32_t)va[e], hp.c_eff, k);
            const uint32_t xb = ((mbb >> e) & 1u) ? k
                                : fast ? im.idx((int32_t)vb[e])
                                       : idx_slow(m, (int32_t)vb[e], hp.c_eff, k);
            const uint32_t aa = tab_row + (xa << tab_sh), ab = tab_row + (xb << tab_sh);
            pk[e >> 2] |= (wtab ? lds_u32(aa) : lds_u8(aa)) << (8 * (e & 3));
            pk[8 + (e >> 2)] |= (wtab ? lds_u32(ab) : lds_u8(ab)) << (8 * (e & 3));
          }
        }
        if (DEBUG && p.dbg_prob && i < p.L) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (j0 + e < p.L)
              p.dbg_prob[((size_t)bh * p.L + i) * p.L + j0 + e] = (uint8_t)(pk[e >> 2] >> (8 * (e & 3)));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // 16-byte units 4*hb + u of this row
          const uint32_t x = (uint32_t)(4 * hb + u);
          if (!(IA_EXP & 4) || ((pk[4 * u] ^ pk[4 * u + 1] ^ pk[4 * u + 2] ^ pk[4 * u + 3]) == 0x12345u))
          sts128(p_row + ((x ^ p_xor) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full + wg * C::NPB + pbl);
      if (trw) IA_TRACE(4 + sw, 11, 2 * n_kt + n);
      ++tl;
    }
    }  // !GK

    // ---- epilogue: out = f32(acc) * f32(s_v / scale) (pipeline.py:250-252)
    // TMEM -> registers -> smem staging (all TMA/MMA traffic has drained once
    // o_full fires) -> coalesced row-contiguous global stores.
    if (tm) IA_TMARK(3);
    mbar_wait(o_full, 0);
    if (tm) IA_TMARK(4);
    tc_fence_after();
    float* stage = reinterpret_cast<float*>(smem);
    const float osc = hp.out_scale;
#pragma unroll 1
    for (int c0 = wg * 16; c0 < DP; c0 += 16 * NWG) {
      uint32_t a[16];
      tmem_ld16(tmem + t_lane + C::O_COL + c0, a);
      if (IA_STAGE_V4) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          float4 f;
          f.x = row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e]), osc) : 0.0f;
          f.y = row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e + 1]), osc) : 0.0f;
          f.z = row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e + 2]), osc) : 0.0f;
          f.w = row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e + 3]), osc) : 0.0f;
          *reinterpret_cast<float4*>(stage + row * C::STAGE_PITCH + c0 + e) = f;
        }
      } else {
#pragma unroll
      for (int e = 0; e < 16; ++e)
        stage[row * C::STAGE_PITCH + c0 + e] =
            row_valid ? __fmul_rn(__int2float_rn((int32_t)a[e]), osc) : 0.0f;
      }
      if (DEBUG && p.dbg_acc && i < p.L) {
        for (int e = 0; e < 16; ++e)
          p.dbg_acc[((size_t)bh * p.L + i) * DP + c0 + e] = (int32_t)a[e];
      }
    }
    named_bar_sync(1, NWT);
    const int rows = min(BM, p.L - q0);
    float* obase = p.out + ((size_t)bh * p.L + q0) * p.d;
    const int tid = stid;
    if (p.d == DP) {  // compile-time row pitch: shifts instead of a division
      constexpr int D4 = DP / 4;
#pragma unroll 1
      for (int t = tid; t < rows * D4; t += NWT) {
        const int r = t / D4, c4 = (t % D4) * 4;
        const float* s4 = stage + r * C::STAGE_PITCH + c4;
        *reinterpret_cast<float4*>(obase + (size_t)r * DP + c4) =
            IA_STAGE_V4 ? *reinterpret_cast<const float4*>(s4) : make_float4(s4[0], s4[1], s4[2], s4[3]);
      }
    } else if ((p.d & 3) == 0) {
      const int d4 = p.d >> 2;
      for (int t = tid; t < rows * d4; t += NWT) {
        const int r = t / d4, c4 = (t - r * d4) << 2;
        const float* s4 = stage + r * C::STAGE_PITCH + c4;
        *reinterpret_cast<float4*>(obase + (size_t)r * p.d + c4) =
            IA_STAGE_V4 ? *reinterpret_cast<const float4*>(s4) : make_float4(s4[0], s4[1], s4[2], s4[3]);
      }
    } else {
      for (int t = tid; t < rows * p.d; t += NWT) {
        const int r = t / p.d, cc = t - r * p.d;
        obase[(size_t)r * p.d + cc] = stage[r * C::STAGE_PITCH + cc];
      }
    }
  }

  if (IA_PROFILE && p.dbg_times) {
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (tacc[s]) p.dbg_times[(size_t)blockIdx.x * 16 + 8 + s] = tacc[s];
  }
  tc_fence_before();
  __syncthreads();
  if (rw == 0 && lane == 0) { IA_TMARK(5); if (IA_PROFILE && p.dbg_times) p.dbg_times[(size_t)blockIdx.x * 16 + 10] = n_kt; }
  if (rw == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
int make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                 uint64_t stride1, uint64_t stride2, uint32_t b0, uint32_t b1, int swizzle_bytes);

template <int DP>
bool attn_supported(int nlut) {
  return attn_smem_bytes<DP>(nlut) + 256 <= 227 * 1024;
}

template <int DP, bool DEBUG, bool SKEL = false, bool QO = false, bool GK = false>
static int launch_attn(const ia_attn_args* a, cudaStream_t st) {
  using C = Cfg<DP>;
  if (!attn_supported<DP>(a->nlut))
    return fail(IA_ERR_HEAD_DIM, "fused path: d_pad %d with %d LUT entries exceeds shared memory",
                DP, a->nlut);
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
  dv.dbg_times = a->dbg_times;
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
  static const int xflags = dev_knob("IA_XFLAGS", 0);  // always 0 in the release build
  dv.xflags = xflags;
  dv.kgroup = reinterpret_cast<const int4*>(a->kgroup_params);
  dv.gs_log2 = 0;
  dv.n_groups = 0;
  if (GK) {
    int lg = 0;
    while ((1 << lg) < a->k_group_size) ++lg;
    dv.gs_log2 = lg;
    dv.n_groups = (int)((a->L + a->k_group_size - 1) / a->k_group_size);
  }
  for (int t = 0; t < 256; ++t) dv.lut[t] = t < a->nlut ? a->lut[t] : 0;
  size_t smem = attn_smem_bytes<DP>(a->nlut);
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM (it owns all 512 TMEM columns)
  auto kern = attn_fwd_kernel<DP, DEBUG, SKEL, QO, GK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(e));
  const uint64_t grid = (uint64_t)dv.n_qt * BH;
  if (grid > 0x7fffffffull) return fail(IA_ERR_INVALID_ARGUMENT, "grid too large");
  kern<<<(unsigned)grid, C::NTHREADS, smem, st>>>(tq, tk, tv, dv);
  return check_launch("attn_fwd_kernel");
}

}  // namespace ia

using namespace ia;

extern "C" int ia_attn_supported(int64_t d_pad, int nlut) {
  switch (d_pad) {
    case 32: return attn_supported<32>(nlut) ? IA_OK : IA_ERR_HEAD_DIM;
    case 64: return attn_supported<64>(nlut) ? IA_OK : IA_ERR_HEAD_DIM;
    case 128: return attn_supported<128>(nlut) ? IA_OK : IA_ERR_HEAD_DIM;
    case 256: return attn_supported<256>(nlut) ? IA_OK : IA_ERR_HEAD_DIM;
    default: return IA_ERR_HEAD_DIM;
  }
}

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
  if (a->k_group_size && a->softmax_mode != IA_SOFTMAX_INDEX)
    return fail(IA_ERR_INVALID_ARGUMENT, "grouped K is an IndexSoftmax mode");
  if (a->softmax_mode == IA_SOFTMAX_FLOAT) {  // quant-only comparator
    switch (a->d_pad) {
      case 32: return dbg ? launch_attn<32, true, false, true>(a, st) : launch_attn<32, false, false, true>(a, st);
      case 64: return dbg ? launch_attn<64, true, false, true>(a, st) : launch_attn<64, false, false, true>(a, st);
      case 128: return dbg ? launch_attn<128, true, false, true>(a, st) : launch_attn<128, false, false, true>(a, st);
      default: return dbg ? launch_attn<256, true, false, true>(a, st) : launch_attn<256, false, false, true>(a, st);
    }
  }
  if (a->softmax_mode != IA_SOFTMAX_INDEX)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_attn_fwd: unknown softmax_mode %d", a->softmax_mode);
  if (a->k_group_size) {  // grouped K (softmax.py:309-399)
    const int gs = a->k_group_size;
    if (gs < 8 || gs > 128 || (gs & (gs - 1)) || !a->kgroup_params)
      return fail(IA_ERR_INVALID_ARGUMENT,
                  "grouped K needs k_group_size a power of two in [8, 128] and kgroup_params");
    if (a->nlut > 64)
      return fail(IA_ERR_INVALID_ARGUMENT, "grouped K supports LUTs of <= 64 entries");
    switch (a->d_pad) {
      case 32: return dbg ? launch_attn<32, true, false, false, true>(a, st) : launch_attn<32, false, false, false, true>(a, st);
      case 64: return dbg ? launch_attn<64, true, false, false, true>(a, st) : launch_attn<64, false, false, false, true>(a, st);
      case 128: return dbg ? launch_attn<128, true, false, false, true>(a, st) : launch_attn<128, false, false, false, true>(a, st);
      default: return fail(IA_ERR_HEAD_DIM, "grouped K: fused path supports d <= 128");
    }
  }
  switch (a->d_pad) {
    case 32: return dbg ? launch_attn<32, true>(a, st) : launch_attn<32, false>(a, st);
    case 64: return dbg ? launch_attn<64, true>(a, st) : launch_attn<64, false>(a, st);
    case 128:
#if IA_PROFILE
      // IA_EXPERIMENT=1 (profiling build only): timing-only skeleton (softmax reads TMEM,
      // skips the integer work; output is NOT IndexSoftmax).
      if (!dbg && dev_knob("IA_EXPERIMENT", 0) == 1) return launch_attn<128, false, true>(a, st);
#endif
      return dbg ? launch_attn<128, true>(a, st) : launch_attn<128, false>(a, st);
    default: return dbg ? launch_attn<256, true>(a, st) : launch_attn<256, false>(a, st);
  }
}
