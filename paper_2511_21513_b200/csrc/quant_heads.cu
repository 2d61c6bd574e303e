// quant_heads.cu -- per-head dynamic INT8 quantisation of Q, K and V in one launch
// (reference quantize_symmetric, quantize.py:104-123, called three times per head by
// int_attention, pipeline.py:217-219).
//
// The two-kernel path (quantize.cu: grid-wide amax, then quantise) reads every f32
// element from HBM twice.  Here a team of CTAs owns one head slab at a time:
//   pass A: max |x| over the slab's valid rows (HBM read), folded into the slab's
//           amax slot; the team meets at a per-slab arrival counter;
//   pass B: s = max(amax, 1e-12f) / 127f and the quantise pass, re-reading the slab
//           from L2 (teams x slab bytes is kept ~96 MB, under the 126 MB L2, with L2 eviction hints).
// Q^ / K^ are written row-major [L, d_pad] and V^ as the per-head transpose
// [d_pad, l_pad] the fused kernel's P.V operand wants; padding rows / columns are 0.
// Arithmetic is the same IEEE f32 sequence as quantize.cu (bit-identical results).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace ia {

namespace {

__device__ __forceinline__ float qh_scale(uint32_t amax_bits) {
  return __fdiv_rn(fmaxf(__uint_as_float(amax_bits), 1e-12f), 127.0f);  // quantize.py:113
}
// q = clip(round_half_away(x / s), +-127) with the quotient numpy computes (IEEE f32
// x / s, quantize.py:121).  t = x * (1/s) is within |t| 2^-23 <= 2^-16 of it (|t| <= 127
// + an ulp).  y = |t| + 0.5 (the reference's own f32 add, rounding.py:21) is floored by
// one round-toward-zero add of 2^23 -- z = 2^23 + floor(y), the integer sits in z's
// mantissa -- so no FRND / F2I conversion (quarter-rate pipe) is needed; y - floor(y) is
// exact.  Unless that fraction is within 2^-14 of 0 or 1 (|t| near a rounding boundary
// k + 0.5, where the exact quotient is taken instead), the exact quotient's y' lies
// within 2^-15 of y on the same side of every integer, so floor(y') = floor(y): the
// reference's result bit for bit.
__device__ __forceinline__ float qh_add_rz(float a, float b) {
  float r;
  asm("add.rz.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// Fast form; `bad` is raised when the element sits within 2^-14 of a rounding boundary
// and must be redone with the exact quotient (qh_q_exact) -- callers test it once per
// 16 elements, so the common path is branch-free.
__device__ __forceinline__ uint32_t qh_q_fast(float x, float rcp, bool& bad) {
  const float t = __fmul_rn(x, rcp);
  const float y = fminf(__fadd_rn(fabsf(t), 0.5f), 127.5f);  // rounding.py:21; quantize.py:122
  const float z = qh_add_rz(y, 8388608.0f);
  const float fr = __fsub_rn(y, __fsub_rn(z, 8388608.0f));
  bad |= !(fr > 6.103515625e-05f && fr < 0.99993896484375f);
  const uint32_t v = __float_as_uint(z) & 0xffu;  // floor(y) <= 127
  return (t < 0.0f ? 0u - v : v) & 0xffu;
}
// The reference's own sequence on the exact quotient (rare path).
__device__ __noinline__ uint32_t qh_q_exact(float x, float s) {
  const float t = __fdiv_rn(x, s);
  float r = floorf(__fadd_rn(fabsf(t), 0.5f));   // rounding.py:21
  r = fminf(r, 127.0f);                          // quantize.py:122
  const int v = (int)r;
  return (uint32_t)(uint8_t)(int8_t)(t < 0.0f ? -v : v);
}
__device__ __forceinline__ uint32_t qh_pack4_fast(float4 v, float rcp, bool& bad) {
  return qh_q_fast(v.x, rcp, bad) | (qh_q_fast(v.y, rcp, bad) << 8) |
         (qh_q_fast(v.z, rcp, bad) << 16) | (qh_q_fast(v.w, rcp, bad) << 24);
}
__device__ __forceinline__ uint32_t qh_pack4_exact(float4 v, float s) {
  return qh_q_exact(v.x, s) | (qh_q_exact(v.y, s) << 8) | (qh_q_exact(v.z, s) << 16) |
         (qh_q_exact(v.w, s) << 24);
}
__device__ __forceinline__ uint32_t qh_pack4(float4 v, float s, float rcp) {
  bool bad = false;
  const uint32_t w = qh_pack4_fast(v, rcp, bad);
  return bad ? qh_pack4_exact(v, s) : w;
}
__device__ __forceinline__ uint32_t qh_abs(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// L2 eviction hints: the amax pass asks L2 to keep the slab (evict_last) for the quantise
// pass, which reads it with evict_first (done with it) and writes its int8 output as
// streaming data, so neither the pass-B reads nor the outputs push later slabs out.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg_hint(const float4* ptr, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_hint(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

struct QHArgs {
  const float* x[3];
  int8_t* out[3];
  int64_t ngroups[3];  // head slabs per tensor
  int64_t valid_div[3];
  int transpose[3];
  int64_t L, d, d_pad, l_pad;
  const int32_t* valid_rows;
  uint32_t* amax;   // [n_slabs], caller-zeroed
  int32_t* count;   // [n_slabs], caller-zeroed
  float* scales;    // [n_slabs]
  int32_t* err;
  int64_t n_slabs;
  int n_teams, team;
  int kb;    // V^T block: keys per block (multiple of 16, kb/4 * d_pad/4 <= QH_THREADS)
  int mode;  // 0: fused (team barrier), 1: amax only, 2: quantise only (slabs in reverse order)
  int per_tensor;  // split modes only: one amax / scale slot per tensor (ti), not per slab
  int hints;  // mode 0 L2 eviction hints: 1 pass A evict_last, 2 pass B evict_first, 4 stores evict_first
};

constexpr int QH_THREADS = 512;

__global__ void __launch_bounds__(QH_THREADS, 3) quant_heads_kernel(const QHArgs a) {
  __shared__ uint32_t red[QH_THREADS / 32];
  __shared__ float s_sh;
  extern __shared__ __align__(16) uint8_t tile[];  // [d_pad][kb + 4] bytes (V^T blocks)
  const int T = a.team;
  const int team = blockIdx.x / T, rank = blockIdx.x - (blockIdx.x / T) * T;
  // Teams stride over the slabs (split modes with n_teams == n_slabs: one slab each).
  // Split modes: no barrier; the quantise pass walks the slabs in the reverse of the amax
  // pass's order so its first reads hit the slabs still in L2.
  const int64_t s_step = a.n_teams;
  const int tid = threadIdx.x;
  const int64_t L = a.L, d = a.d;
  const int64_t d4 = d >> 2;
  const uint64_t pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();
  const bool hint_a = a.mode == 0 && (a.hints & 1), hint_b = a.mode == 0 && (a.hints & 2);
  const bool hint_st = a.mode == 0 && (a.hints & 4);

  struct Slab {
    int ti;
    int64_t g, nvalid, slot;
    const float4* base;
  };
  auto slab_of = [&](int64_t s) {
    Slab sl;
    sl.ti = 0;
    sl.g = s;
    while (sl.ti < 2 && sl.g >= a.ngroups[sl.ti]) { sl.g -= a.ngroups[sl.ti]; ++sl.ti; }
    sl.nvalid = L;
    if (a.valid_rows) {
      const int64_t v = a.valid_rows[sl.g / a.valid_div[sl.ti]];
      sl.nvalid = v < 0 ? 0 : (v < L ? v : L);
    }
    sl.base = reinterpret_cast<const float4*>(a.x[sl.ti] + sl.g * L * d);
    sl.slot = a.per_tensor ? sl.ti : s;
    return sl;
  };

  // ---- pass A: max |x| over the valid rows (quantize.py:92-101), folded into the slab's
  // amax slot; mode 0: this CTA then arrives at the slab's counter
  auto pass_a = [&](int64_t s) {
    const Slab sl = slab_of(s);
    const float4* base = sl.base;
    const int64_t n4 = sl.nvalid * d4;
    uint32_t m = 0;
    auto fold = [&](const float4& v) {
      m = max(m, max(max(qh_abs(v.x), qh_abs(v.y)), max(qh_abs(v.z), qh_abs(v.w))));
    };
    // four independent 16-byte loads in flight per thread (HBM needs the MLP)
    const int64_t step = (int64_t)T * QH_THREADS;
    int64_t i = (int64_t)rank * QH_THREADS + tid;
    if (hint_a) {
      for (; i + 3 * step < n4; i += 4 * step) {
        const float4 v0 = ldg_hint(base + i, pol_keep), v1 = ldg_hint(base + i + step, pol_keep);
        const float4 v2 = ldg_hint(base + i + 2 * step, pol_keep), v3 = ldg_hint(base + i + 3 * step, pol_keep);
        fold(v0); fold(v1); fold(v2); fold(v3);
      }
      for (; i < n4; i += step) fold(ldg_hint(base + i, pol_keep));
    } else {
      for (; i + 3 * step < n4; i += 4 * step) {
        const float4 v0 = __ldg(base + i), v1 = __ldg(base + i + step);
        const float4 v2 = __ldg(base + i + 2 * step), v3 = __ldg(base + i + 3 * step);
        fold(v0); fold(v1); fold(v2); fold(v3);
      }
      for (; i < n4; i += step) fold(__ldg(base + i));
    }
    m = warp_max_u32(m);
    __syncthreads();  // red[] may still be read by the previous reduction's warp 0
    if ((tid & 31) == 0) red[tid >> 5] = m;
    __syncthreads();
    if (tid < 32) {
      m = tid < QH_THREADS / 32 ? red[tid] : 0u;
      m = warp_max_u32(m);
      if (tid == 0) {
        // NaN bit patterns sort above +inf: a non-finite element lifts m >= 0x7f800000
        if (m >= 0x7f800000u) atomicOr(reinterpret_cast<unsigned int*>(a.err), 1u);
        else if (m) atomicMax(a.amax + sl.slot, m);
        if (a.mode == 0) {
          __threadfence();
          atomicAdd(a.count + s, 1);
        }
      }
    }
  };

  // ---- pass B: the team's amax is final (mode 0: once every CTA of the team has arrived);
  // s = max(amax, 1e-12f) / 127f and the quantise pass (mode 0: slab re-read from L2)
  auto pass_b = [&](int64_t s) {
    const Slab sl = slab_of(s);
    const float4* base = sl.base;
    const int64_t nvalid = sl.nvalid, g = sl.g;
    const int ti = sl.ti;
    if (tid == 0) {
      if (a.mode == 0) {
        // Mode 0 is only ever launched cooperatively (cudaLaunchAttributeCooperative), so
        // every CTA of the grid is co-resident and the wait ends.  The bound is a second
        // line of defence: after ~2^26 polls (seconds) the kernel flags
        // IA_QH_ERR_BARRIER and carries on, so the call fails loudly instead of hanging.
        uint32_t polls = 0;
        while (*reinterpret_cast<volatile int32_t*>(a.count + s) < T) {
          __nanosleep(128);
          if (++polls == (1u << 26)) {
            atomicOr(reinterpret_cast<unsigned int*>(a.err), 2u);
            break;
          }
        }
        __threadfence();
      }
      const float sc0 = qh_scale(*reinterpret_cast<volatile uint32_t*>(a.amax + sl.slot));
      s_sh = sc0;
      if (rank == 0) a.scales[sl.slot] = sc0;  // per tensor: every slab stores the same value
    }
    __syncthreads();
    const float sc = s_sh;
    const float rc = __frcp_rn(sc);
    auto ld = [&](const float4* ptr) { return hint_b ? ldg_hint(ptr, pol_drop) : __ldg(ptr); };
    auto st = [&](void* ptr, uint4 v) {
      if (hint_st) stg_hint(ptr, v, pol_drop);
      else *reinterpret_cast<uint4*>(ptr) = v;
    };
    if (!a.transpose[ti]) {
      const int cpr = (int)(a.d_pad >> 4);  // 16-byte output chunks per row
      int8_t* og = a.out[ti] + g * L * a.d_pad;
      const int64_t nch = L * cpr;
      const int lg = (cpr & (cpr - 1)) == 0 ? __ffs(cpr) - 1 : -1;  // power-of-two row pitch: shifts
      for (int64_t j = (int64_t)rank * QH_THREADS + tid; j < nch; j += (int64_t)T * QH_THREADS) {
        const int64_t r = lg >= 0 ? (j >> lg) : j / cpr;
        const int c0 = (int)(j - r * cpr) << 4;
        uint4 o = make_uint4(0u, 0u, 0u, 0u);
        if (r < nvalid && c0 < d) {
          const float4* xr = base + r * d4 + (c0 >> 2);
          if (c0 + 16 <= d) {
            const float4 v0 = ld(xr), v1 = ld(xr + 1), v2 = ld(xr + 2), v3 = ld(xr + 3);
            bool bad = false;
            o = make_uint4(qh_pack4_fast(v0, rc, bad), qh_pack4_fast(v1, rc, bad),
                           qh_pack4_fast(v2, rc, bad), qh_pack4_fast(v3, rc, bad));
            if (bad)
              o = make_uint4(qh_pack4_exact(v0, sc), qh_pack4_exact(v1, sc), qh_pack4_exact(v2, sc),
                             qh_pack4_exact(v3, sc));
          } else {
            uint32_t w[4] = {0u, 0u, 0u, 0u};
            for (int e = 0; e < 4 && c0 + 4 * e < d; ++e) w[e] = qh_pack4(ld(xr + e), sc, rc);
            o = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        st(og + r * a.d_pad + c0, o);
      }
    } else {
      // V^T: blocks of kb keys.  Each thread loads a 4-key x 4-column patch (four
      // float4, one per key), quantises it, transposes it in registers into four words
      // (four keys of one column) and writes them to the tile [d_pad][kb/4 + 1 words];
      // the odd pitch spreads the scatter over the banks.  The tile then leaves as
      // 16-byte runs of keys for each of the d_pad output rows.
      int8_t* og = a.out[ti] + g * a.d_pad * a.l_pad;
      uint32_t* tw = reinterpret_cast<uint32_t*>(tile);
      const int dp = (int)a.d_pad, cg = dp >> 2, kb = a.kb, pw = (kb >> 2) + 1;
      const int items = (kb >> 2) * cg;  // patches per block (<= QH_THREADS)
      const int nblk = (int)((a.l_pad + kb - 1) / kb);
      for (int rb = rank; rb < nblk; rb += T) {
        const int64_t r0 = (int64_t)rb * kb;
        if (tid < items) {
          const int rg = tid / cg, c4 = (tid - rg * cg) << 2;
          const int64_t rr = r0 + 4 * rg;
          float4 x4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            x4[i] = (rr + i < nvalid && c4 < d) ? ld(base + (rr + i) * d4 + (c4 >> 2))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
          uint32_t w[4];
          bool bad = false;
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] = qh_pack4_fast(x4[i], rc, bad);  // padding: x = 0 -> 0
          if (bad) {
#pragma unroll
            for (int i = 0; i < 4; ++i) w[i] = qh_pack4_exact(x4[i], sc);
          }
          const uint32_t lo01 = __byte_perm(w[0], w[1], 0x5140), hi01 = __byte_perm(w[0], w[1], 0x7362);
          const uint32_t lo23 = __byte_perm(w[2], w[3], 0x5140), hi23 = __byte_perm(w[2], w[3], 0x7362);
          tw[(c4 + 0) * pw + rg] = __byte_perm(lo01, lo23, 0x5410);
          tw[(c4 + 1) * pw + rg] = __byte_perm(lo01, lo23, 0x7632);
          tw[(c4 + 2) * pw + rg] = __byte_perm(hi01, hi23, 0x5410);
          tw[(c4 + 3) * pw + rg] = __byte_perm(hi01, hi23, 0x7632);
        }
        __syncthreads();
        const int cpr = kb >> 4;  // 16-byte runs per output row
        for (int t = tid; t < dp * cpr; t += QH_THREADS) {
          const int c = t / cpr, u = t - c * cpr;
          const int64_t r = r0 + 16 * u;
          if (r < a.l_pad) {
            const uint32_t* src = tw + c * pw + 4 * u;
            st(og + (int64_t)c * a.l_pad + r, make_uint4(src[0], src[1], src[2], src[3]));
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();  // s_sh is rewritten by the next slab's thread 0
  };

  if (a.mode == 1) {
    for (int64_t j = team; j < a.n_slabs; j += s_step) pass_a(j);
  } else if (a.mode == 2) {
    for (int64_t j = team; j < a.n_slabs; j += s_step) pass_b(a.n_slabs - 1 - j);
  } else {
    for (int64_t j = team; j < a.n_slabs; j += s_step) {
      pass_a(j);
      pass_b(j);
    }
  }
}

}  // namespace
}  // namespace ia

using namespace ia;

// amax over every slab, then the quantise pass in reverse slab order; no barriers, so
// the grids need not be resident: ~128 KB of f32 per CTA
static int quant_heads_split(QHArgs a, void (*kern)(const QHArgs), int64_t grid_max,
                             int64_t slab_bytes, size_t smem, cudaStream_t stream) {
  int64_t t2 = (slab_bytes + (128 << 10) - 1) >> 17;
  t2 = t2 < 1 ? 1 : t2;
  a.team = (int)t2;
  a.n_teams = (int)a.n_slabs;
  // IA_QH_WAVES=w > 0 (profiling build): at most w resident waves of teams, each
  // striding over slabs
  static const int waves_env = dev_knob("IA_QH_WAVES", 0);
  if (waves_env > 0) {
    const int64_t cap = grid_max * waves_env / t2;
    if (cap >= 1 && cap < a.n_slabs) a.n_teams = (int)cap;
  }
  const uint64_t g2 = (uint64_t)a.n_teams * t2;
  a.mode = 1;
  kern<<<(unsigned)g2, QH_THREADS, smem, stream>>>(a);
  if (int r = check_launch("quant_heads_kernel (amax)")) return r;
  a.mode = 2;
  kern<<<(unsigned)g2, QH_THREADS, smem, stream>>>(a);
  return check_launch("quant_heads_kernel (quantise)");
}

static int quant_heads_launch(const float* q, const float* k, const float* v, int64_t B,
                              int64_t H, int64_t Hkv, int64_t L, int64_t d,
                              const int32_t* seq_lens, int8_t* qhat, int8_t* khat, int8_t* vt,
                              int64_t d_pad, int64_t l_pad, uint32_t* amax_bits,
                              int32_t* counters, float* scales, int32_t* err_flag, void* stream,
                              int per_tensor) {
  if (!q || !k || !v || !qhat || !khat || !vt || !amax_bits || !scales || !err_flag ||
      (!counters && !per_tensor))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_heads: null pointer");
  if (B < 1 || H < 1 || Hkv < 1 || H % Hkv || L < 1 || d < 1)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_heads: bad shape");
  if ((d & 3) || d > IA_FUSED_MAX_HEAD_DIM || d_pad < d || (d_pad & 15) || d_pad > 256 ||
      l_pad < L || (l_pad & 15))
    return fail(IA_ERR_INVALID_ARGUMENT,
                "ia_quant_heads: needs d %% 4 == 0, d <= d_pad <= 256, d_pad and l_pad %% 16 == 0");
  if ((((uintptr_t)q | (uintptr_t)k | (uintptr_t)v | (uintptr_t)qhat | (uintptr_t)khat |
        (uintptr_t)vt) & 15))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_heads: operands must be 16-byte aligned");
  QHArgs a;
  a.x[0] = q; a.x[1] = k; a.x[2] = v;
  a.out[0] = qhat; a.out[1] = khat; a.out[2] = vt;
  a.ngroups[0] = B * H; a.ngroups[1] = B * Hkv; a.ngroups[2] = B * Hkv;
  a.valid_div[0] = H; a.valid_div[1] = Hkv; a.valid_div[2] = Hkv;
  a.transpose[0] = 0; a.transpose[1] = 0; a.transpose[2] = 1;
  a.L = L; a.d = d; a.d_pad = d_pad; a.l_pad = l_pad;
  a.valid_rows = seq_lens;
  a.amax = amax_bits; a.count = counters; a.scales = scales; a.err = err_flag;
  a.n_slabs = B * H + 2 * B * Hkv;
  // V^T block: one 4x4 patch per thread (kb * d_pad = 16 * QH_THREADS bytes)
  static const int kb_env = dev_knob("IA_QH_KB", 0);
  int kb = (int)(((16 * QH_THREADS) / d_pad) & ~15);
  if (kb_env >= 16 && (kb_env & 15) == 0 && (kb_env / 4) * (d_pad / 4) <= QH_THREADS) kb = kb_env;
  a.kb = kb;
  const size_t smem = (size_t)d_pad * (kb + 4);
  void (*kern)(const QHArgs) = quant_heads_kernel;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                                QH_THREADS, smem);
  if (e != cudaSuccess || per_sm < 1) return fail(IA_ERR_CUDA, "ia_quant_heads: occupancy query");
  // Team barriers need every CTA resident: the grid never exceeds one full wave.
  const int64_t grid_max = (int64_t)num_sms() * per_sm;
  const int64_t slab_bytes = L * d * 4;
  const int64_t slab_elems = L * d;
  // IA_QH_L2MB / IA_QH_TEAM override the L2 budget and team size (A/B runs only)
  static const int l2mb_env = dev_knob("IA_QH_L2MB", 96);
  static const int team_env = dev_knob("IA_QH_TEAM", 0);
  static const int hints_env = dev_knob("IA_QH_HINTS", 7);
  a.hints = hints_env;
  // teams = slabs in flight in L2 (~96 MB: measured best of 32..800 on C4 / C5; smaller
  // teams pay less at each barrier, and the evict_last / evict_first hints keep the re-read hits)
  int64_t target = ((int64_t)l2mb_env << 20) / (slab_bytes > 0 ? slab_bytes : 1);
  target = target < 1 ? 1 : (target > a.n_slabs ? a.n_slabs : target);
  int64_t team = grid_max / target;
  const int64_t want = (slab_elems + QH_THREADS * 16 - 1) / (QH_THREADS * 16);  // >= 16 elem/thread
  team = team < want ? team : want;
  team = team < 1 ? 1 : team;
  if (team_env > 0) team = team_env < grid_max ? team_env : grid_max;
  int64_t n_teams = grid_max / team;
  n_teams = n_teams > a.n_slabs ? a.n_slabs : n_teams;
  a.n_teams = (int)n_teams;
  a.team = (int)team;
  a.mode = 0;
  a.per_tensor = per_tensor;
  // Many small slabs (C3: 96 x 1 MB) spend more on team barriers than on bytes: run the
  // amax and quantise passes as two barrier-free launches instead (IA_QH_SPLIT=0/1
  // forces either form, for A/B checks).
  static const int split_env = dev_knob("IA_QH_SPLIT", -1);
  // Per-tensor scales need every slab's amax first: always the two-launch form.
  const bool split = per_tensor || (split_env >= 0 ? split_env != 0
                                                   : (slab_bytes <= (1 << 20) && a.n_slabs >= 32));
  if (split) return quant_heads_split(a, kern, grid_max, slab_bytes, smem, (cudaStream_t)stream);
  // Cooperative launch: the runtime guarantees every CTA is co-resident (or refuses the
  // launch), which is what the team barrier needs -- an occupancy-sized plain launch is
  // only safe on an otherwise idle device.  If the runtime refuses (kernels on other
  // streams, MPS / green contexts with fewer SMs), run the barrier-free two-launch form.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_teams * team));
  cfg.blockDim = dim3(QH_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e == cudaSuccess) return check_launch("quant_heads_kernel");
  (void)cudaGetLastError();  // clear the refused launch; fall back to the split form
  return quant_heads_split(a, kern, grid_max, slab_bytes, smem, (cudaStream_t)stream);
}

extern "C" int ia_quant_heads(const float* q, const float* k, const float* v, int64_t B, int64_t H,
                              int64_t Hkv, int64_t L, int64_t d, const int32_t* seq_lens,
                              int8_t* qhat, int8_t* khat, int8_t* vt, int64_t d_pad, int64_t l_pad,
                              uint32_t* amax_bits, int32_t* counters, float* scales,
                              int32_t* err_flag, void* stream) {
  return quant_heads_launch(q, k, v, B, H, Hkv, L, d, seq_lens, qhat, khat, vt, d_pad, l_pad,
                            amax_bits, counters, scales, err_flag, stream, 0);
}

extern "C" int ia_quant_tensors(const float* q, const float* k, const float* v, int64_t B,
                                int64_t H, int64_t Hkv, int64_t L, int64_t d,
                                const int32_t* seq_lens, int8_t* qhat, int8_t* khat, int8_t* vt,
                                int64_t d_pad, int64_t l_pad, uint32_t* amax_bits, float* scales,
                                int32_t* err_flag, void* stream) {
  return quant_heads_launch(q, k, v, B, H, Hkv, L, d, seq_lens, qhat, khat, vt, d_pad, l_pad,
                            amax_bits, nullptr, scales, err_flag, stream, 1);
}
