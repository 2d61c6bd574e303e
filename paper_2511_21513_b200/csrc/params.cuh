// params.cuh -- per-(b, head) IndexSoftmax parameters, shared by host and device.
#pragma once
#include <cmath>
#include <climits>
#include <cstdint>
#include <cstring>

#include "intattn_b200.h"

namespace ia {

constexpr int64_t kCIntCap = int64_t(1) << 52;  // softmax.py:47 _C_INT_CAP

// c_int = max(1, min(round_half_away(c / alpha), 2^52)),
// alpha = f64(s_q) * f64(s_k) / sqrt(d)            (gemm.py:105, softmax.py:105-121)
// Every operation is a single IEEE f64 op (no contraction possible), so host
// and device agree bit for bit with Python's float arithmetic.
__host__ __device__ inline int64_t compute_c_int(double c, int64_t d, float s_q, float s_k) {
  double alpha = (double)s_q * (double)s_k;
  alpha = alpha / sqrt((double)d);
  double r = c / alpha;
  double t = floor(fabs(r) + 0.5);
  if (!(t < (double)kCIntCap)) return kCIntCap;
  int64_t ci = (int64_t)t;
  return ci < 1 ? 1 : ci;
}

// Entries of the fused kernel's per-row normalisation table: zero-extended to 56
// for LUTs of <= 32 entries (rows whose largest reachable index is < 56 skip the
// per-logit clip), else one per LUT entry.
__host__ __device__ constexpr int row_table_entries(int nlut) { return nlut <= 32 ? 56 : nlut; }

__host__ __device__ inline int bitlen_u64(uint64_t x) {
  int n = 0;
  while (x) { ++n; x >>= 1; }
  return n;
}

// Float form of the same index map (the fused kernel's fast path for small c_eff).
//
// With lo = m - c (c = c_eff) and u = max(a - lo, 0) = c - delta' in [0, c] (one VIADDMNMX;
// the clip comes free),
//   idx = floor((2k*delta' + c) / (2c)) = k - j,   j = floor((2k*u + c - 1) / (2c))
//       = floor(y0 + 1/2 - 1/(2c)),  y0 = u * k / c:
// j is y0 rounded to the nearest integer with ties going DOWN.  Let r be the largest f32
// strictly below k/c (r = (k/c)(1 - eps), 0 < eps <= 2^-23).  One FMA computes y = u * r =
// y0 (1 - eps) exactly before its single rounding.  y0 + 1/2 is a multiple of 1/(2c), so
// off a tie y0 is at least 1/(2c) above the half-integer below it, and with  c (2k + 1) <
// 2^23  the deficit y0 * eps <= k * 2^-23 stays below that gap:  T - 1/2 < y < T + 1/2 with
// T = j; on a tie (y0 = T + 1/2) y is strictly below T + 1/2, so it rounds down to T = j.
// The kernel feeds the FMA the integer u (< 2^23) reinterpreted as an f32: that bit pattern
// is the denormal u * 2^-149, and with a denormal addend A * 2^-149 the result
// RN(y + A) * 2^-149 has the bit pattern j + A (pass 2: A = the address of a reversed LUT,
// lutr[j] = lut[k - j], so the bits are the entry's address), RZ(512 y + 256 + A) the
// pattern A + 512 j + (9 fraction bits) (pass 3: A = the reversed row table, one LOP3 from
// the entry address, as with magic9).  Denormal FMAs run at full rate and pack two lanes
// per instruction (FFMA2): measured 2x (pass 2) and 1.6x (pass 3) the throughput of the
// IMAD / IMAD.HI form (tools/loop_bench.cu).  Exhaustive check: tests/test_kernel_arith.py.
__host__ __device__ inline bool float_idx_ok(int64_t c_eff, int64_t k) {
  return c_eff > 0 && k > 0 && k < 256 && c_eff < (int64_t(1) << 23) &&
         c_eff * (2 * k + 1) < (int64_t(1) << 23);
}
// Largest f32 strictly below k / c_eff (c_eff < 2^23: the products below are exact in f64).
__host__ __device__ inline float float_idx_ratio(int64_t c_eff, int64_t k) {
  const double rd = (double)k / (double)c_eff;
  float r = (float)rd;  // round to nearest, then step down until r * c_eff < k
  uint32_t bits;
#ifdef __CUDA_ARCH__
  bits = __float_as_uint(r);
#else
  memcpy(&bits, &r, 4);
#endif
  for (int it = 0; it < 4; ++it) {
    float f;
#ifdef __CUDA_ARCH__
    f = __uint_as_float(bits);
#else
    memcpy(&f, &bits, 4);
#endif
    if ((double)f * (double)c_eff < (double)k) return f;
    --bits;
  }
  return 0.0f;  // unreachable for k >= 1
}

// Fill everything except the scales.  k = nlut - 1.
//
// Index map (softmax.py:144-153):  delta = m - a >= 0;  idx = k if delta >= c_int
// else (2*delta*k + c_int) // (2*c_int).  With delta' = min(delta, c) this is
// idx = (2*k*delta' + c) // (2c) for all delta (delta' = c gives k + 1/2 -> k).
//
// c_eff: |a| <= d*127^2 so delta <= dbound = 2*d*127^2.  If c_int > 2k*dbound
// every unmasked idx is 0, and c_eff = 2k*dbound + 1 gives the same (2k*delta
// < c_eff).  Otherwise c_eff = c_int.  Then n = 2k*delta' + c_eff lies in
// [c_eff, n_max], n_max = min((2k+1) c_eff, 2k*dbound + c_eff).
//
// Magic division: D = 2 c_eff, s = max(0, bitlen(n_max*D - 1) - 32),
// M = ceil(2^(32+s) / D), e = M*D - 2^(32+s) in [0, D).  For n <= n_max,
// n*M / 2^(32+s) = n/D + n*e/(D 2^(32+s)) and n*e < n_max*D <= 2^(32+s), so the
// error term is below 1/D and floor(n*M / 2^(32+s)) = floor(n / D).
// use32 requires n_max < 2^31 (then M < 2^32); else the kernels divide in 64-bit.
// When the UNCLAMPED range 2k*dbound + c_eff is also below 2^31 the magic is
// derived for it instead (unc32 = 1): idx = floor(n / D) is then exact for every
// reachable delta without the clip, so a kernel that knows its rows' largest
// delta can drop the per-element min() and read a zero-extended table instead.
// dbound: an upper bound on delta = m - a over the logits this map will see
// (2*d*127^2 for int8 operands; 2^32 - 1 for arbitrary int32 logits).
__host__ __device__ inline void fill_head_params(int64_t c_int, int64_t dbound, int nlut,
                                                 ia_head_params* hp) {
  const int64_t k = nlut - 1;
  const int64_t clamp = 2 * k * dbound + 1;
  const int64_t c_eff = c_int < clamp ? c_int : clamp;
  const int64_t n_unc = 2 * k * dbound + c_eff;  // largest n without the clip
  int64_t n_max = n_unc;
  const int64_t alt = (2 * k + 1) * c_eff;
  if (alt < n_max) n_max = alt;
  hp->unc32 = 0;
  if (n_unc < (int64_t(1) << 31)) {
    n_max = n_unc;
    hp->unc32 = 1;
  }
  hp->c_int = c_int;
  hp->c_eff = c_eff;
  hp->use32 = 0;
  hp->magic = 0;
  hp->shift = 0;
  if (n_max < (int64_t(1) << 31)) {
    const uint64_t D = 2 * (uint64_t)c_eff;
    const uint64_t prod = (uint64_t)n_max * D;  // < 2^63
    int s = bitlen_u64(prod - 1) - 32;            // smallest s with prod <= 2^(32+s)
    if (s < 1) s = 1;  // s >= 1: the device applies >> s as umulhi(q, 2^(32-s))
    const uint64_t num = uint64_t(1) << (32 + s);
    const uint64_t M = (num + D - 1) / D;
    if (s <= 31 && M < (uint64_t(1) << 32)) {
      hp->use32 = 1;
      hp->magic = (uint32_t)M;
      hp->shift = s;
    }
  }
  if (!hp->use32) hp->unc32 = 0;
  hp->fratio = (hp->use32 && float_idx_ok(c_eff, k)) ? float_idx_ratio(c_eff, k) : 0.0f;
  // Scaled magic for every n whose index fits the fused kernel's zero-extended row
  // table (idx <= NT9 = row_table_entries(nlut) - 1: n < 2 c_eff (NT9 + 1)), which
  // covers the clipped range n <= (2k+1) c_eff and the unclipped n of any row whose
  // largest reachable index fits the table: with M9 the magic of shift s9 <= 9 and
  // magic9 = M9 << (9 - s9), umulhi(n, magic9) = idx * 512 + r with r < 512
  // (floor(floor(x * 2^j) / 2^j) = floor(x)), so a row-table address idx * 512 +
  // row * 4 is one LOP3 away.  0 when it does not fit 32 bits.
  hp->magic9 = 0;
  if (hp->use32) {
    const int64_t nt9 = row_table_entries(nlut) - 1;
    const int64_t nmc = 2 * c_eff * (nt9 + 1) - 1;
    if (nmc < (int64_t(1) << 31)) {
      const uint64_t D = 2 * (uint64_t)c_eff;
      int s9 = bitlen_u64((uint64_t)nmc * D - 1) - 32;
      if (s9 < 1) s9 = 1;
      if (s9 <= 9) {
        const uint64_t M9 = ((uint64_t(1) << (32 + s9)) + D - 1) / D;
        const uint64_t m9 = M9 << (9 - s9);
        if (m9 < (uint64_t(1) << 32)) hp->magic9 = (uint32_t)m9;
      }
    }
  }
}

__host__ __device__ inline void make_head_params(double c, int64_t d, int nlut, int p_scale,
                                                 float s_q, float s_k, float s_v,
                                                 ia_head_params* hp) {
  fill_head_params(compute_c_int(c, d, s_q, s_k), 2 * d * 127 * 127, nlut, hp);
  hp->out_scale = (float)((double)s_v / (double)p_scale);  // pipeline.py:250
  hp->s_q = s_q;
  hp->s_k = s_k;
  hp->s_v = s_v;
}

#ifdef __CUDACC__
// lo for a row max m.  If m - c_eff < INT32_MIN no int32 logit is clipped.
__device__ __forceinline__ int32_t idx_lo(int32_t m, int64_t c_eff) {
  const int64_t lo = (int64_t)m - c_eff;
  return lo < (int64_t)INT32_MIN ? INT32_MIN : (int32_t)lo;
}

// Per-element index map (softmax.py:144-153), exact magic-number form (params.cuh).
struct IdxMap {
  int32_t lo;     // max(m - c_eff, INT32_MIN): a' = max(a, lo) clips delta to c_eff
  uint32_t base;  // 2k*m + c_eff (mod 2^32)
  uint32_t nk2;   // -2k (mod 2^32): n = base + nk2 * a' is one IMAD
  uint32_t magic;
  uint32_t mul2;  // 2^(32 - shift): q >> shift == umulhi(q, mul2) (keeps the shift on the FMA pipe)
  uint32_t shift;
  __device__ __forceinline__ void init(int32_t m, const ia_head_params& hp, uint32_t k) {
    nk2 = 0u - 2u * k;
    asm("" : "+r"(nk2));  // keep -2k in a register (a uniform one is re-negated per use)
    magic = hp.magic;
    mul2 = hp.use32 ? (1u << (32 - hp.shift)) : 0u;
    shift = (uint32_t)hp.shift;
    lo = hp.use32 ? idx_lo(m, hp.c_eff) : 0;
    base = (uint32_t)m * (2u * k) + (uint32_t)hp.c_eff;
  }
  // Two forms of the same exact map, to balance the FMA and ALU pipes:
  // idx() does the final >> shift on the FMA pipe (IMAD.HI), idx_s() on the ALU pipe (SHF).
  __device__ __forceinline__ uint32_t idx(int32_t a) const {
    const int32_t ac = max(a, lo);
    const uint32_t n = base + nk2 * (uint32_t)ac;  // n = 2k*delta' + c_eff in [c_eff, n_max]
    return __umulhi(__umulhi(n, magic), mul2);
  }
  __device__ __forceinline__ uint32_t idx_s(int32_t a) const {
    const int32_t ac = max(a, lo);
    const uint32_t n = base + nk2 * (uint32_t)ac;
    return __umulhi(n, magic) >> shift;
  }
  // n for the clipped delta (the operand of magic9)
  __device__ __forceinline__ uint32_t n_clip(int32_t a) const {
    return base + nk2 * (uint32_t)max(a, lo);
  }
  // n without the clip (unc32 rows whose largest index fits the table; operand of magic9)
  __device__ __forceinline__ uint32_t n_unc(int32_t a) const { return base + nk2 * (uint32_t)a; }
  // Unclamped (hp.unc32): floor((2k*delta + c_eff) / (2 c_eff)) for any reachable
  // delta; may exceed k, callers index a table zero-extended past k.
  __device__ __forceinline__ uint32_t idx_u(int32_t a) const {
    const uint32_t n = base + nk2 * (uint32_t)a;
    return __umulhi(n, magic) >> shift;
  }
};

__device__ __forceinline__ uint32_t idx_slow(int64_t m, int32_t a, int64_t c_eff, int64_t k) {
  int64_t dl = m - (int64_t)a;
  if (dl > c_eff) dl = c_eff;
  return (uint32_t)((2 * dl * k + c_eff) / (2 * c_eff));
}

#endif

}  // namespace ia
