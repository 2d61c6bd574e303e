/*
 * intattn_b200.h -- C ABI of the B200 (sm_100a) IntAttention forward path.
 *
 * Plain pointers and sizes only (no torch types).  All device pointers are
 * CUDA device memory; `stream` is a cudaStream_t passed as void*.  Calls are
 * asynchronous and stream-ordered; buffers are caller-allocated.  Every entry
 * point returns an ia_status (0 = ok).  The reference is a Python package
 * (intattn) with no FFI of its own, so each entry point below names the
 * reference operator it replaces (paths relative to
 * /root/reference/pkg/src/intattn/); INTEGRATION.md shows the ctypes binding.
 */
#ifndef INTATTN_B200_H
#define INTATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IA_ABI_VERSION 5  /* 2: ia_head_params gained magic9; 3: ia_attn_args.softmax_mode;
                            4: grouped-K fields of ia_attn_args, ia_group_params;
                            5: ia_head_params.fratio (in the struct's former tail padding) */
#define IA_MAX_SEQ_LEN 65536   /* gemm.py:26 MAX_SEQ_LEN */
#define IA_MAX_HEAD_DIM 131070 /* gemm.py:25 MAX_HEAD_DIM */
#define IA_FUSED_MAX_HEAD_DIM 256

typedef enum ia_status {
  IA_OK = 0,
  IA_ERR_INVALID_ARGUMENT = 1, /* shape/range errors: the reference's ValueError */
  IA_ERR_SEQ_LEN = 2,          /* L > 65536 (pipeline.py:91-92, gemm.py:130-131) */
  IA_ERR_HEAD_DIM = 3,         /* d outside this entry point's range */
  IA_ERR_NONFINITE = 4,        /* non-finite input (quantize.py:109-110) */
  IA_ERR_CUDA = 5,             /* CUDA runtime/driver failure (see ia_last_error) */
  IA_ERR_NO_DEVICE = 6,        /* no sm_100 device */
  IA_ERR_LUT = 7               /* LUT endpoints not 255/0 (softmax.py:230-234) */
} ia_status;

int ia_abi_version(void);
const char* ia_status_string(int status);
/* Human-readable detail of the last failure on the calling thread. */
const char* ia_last_error(void);
/* Returns IA_OK if device `dev` is an sm_100 part this library can run on. */
int ia_device_check(int dev);

/* ------------------------------------------------------------------ quantiser
 * Replaces quantize_symmetric (quantize.py:104-123) and _group_maxabs
 * (quantize.py:92-101).  Two stream-ordered steps: amax (atomic max of the
 * f32 bit pattern into caller-zeroed amax_bits) then quantise.
 *
 * Row layout: x is [n_rowgroups * rows_per_group, cols] f32, row-major.
 * Row group g has valid_rows[g / valid_div] valid rows when valid_rows is
 * non-NULL (seq_lens for padded batches), else rows_per_group.  Its max |x|
 * over valid rows is folded into slot g / slot_div (slot_div = 1: one scale
 * per row group / head; slot_div = n_rowgroups: one global scale).
 * err_flag (device int32) is set to 1 if any valid element is non-finite.
 */
int ia_quant_amax_rows(const float* x, int64_t n_rowgroups, int64_t rows_per_group,
                       int64_t cols, const int32_t* valid_rows, int64_t valid_div,
                       int64_t slot_div, uint32_t* amax_bits, int32_t* err_flag,
                       void* stream);
/* Per-column-group max |x| (per_col_group granularity, quantize.py:99-101). */
int ia_quant_amax_cols(const float* x, int64_t rows, int64_t cols, int64_t col_group,
                       uint32_t* amax_bits, int32_t* err_flag, void* stream);
/* scales[i] = max(amax[i], 1e-12f) / 127f in IEEE f32 (quantize.py:113). */
int ia_quant_scales(const uint32_t* amax_bits, int64_t n, float* scales, void* stream);

#define IA_QMODE_ROWS 0 /* scale index (r / rows_per_group) / slot_div */
#define IA_QMODE_COLS 1 /* scale index c / col_group */
/* values = clip(round_half_away(x / scale), -127, 127) (quantize.py:121-122).
 * transpose = 0: out is [rows, out_pitch] int8; columns [cols, out_pitch) and
 *   invalid rows are written 0 (zero K padding keeps dot products exact).
 * transpose = 1 (ROWS mode only): out holds, per row group g at
 *   out + g * out_group_stride, the [cols, out_pitch] transpose (V^T layout
 *   for the fused kernel's P.V operand); invalid rows are written 0. */
int ia_quantize(const float* x, int64_t n_rowgroups, int64_t rows_per_group, int64_t cols,
                const int32_t* valid_rows, int64_t valid_div, int mode, int64_t slot_div,
                int64_t col_group, const float* scales, int8_t* out, int64_t out_pitch,
                int transpose, int64_t out_group_stride, void* stream);
/* Per-head quantisation of Q, K and V in one launch: the three
 * quantize_symmetric calls of int_attention (pipeline.py:217-219) for every
 * (batch, head) slab of q [B, H, L, d], k and v [B, Hkv, L, d] (f32,
 * row-major, 16-byte aligned, d % 4 == 0, d <= 256).  Writes qhat
 * [B*H, L, d_pad] and khat [B*Hkv, L, d_pad] row-major, vt [B*Hkv, d_pad,
 * l_pad] (per-head V^T), padding zero; rows >= seq_lens[b] are excluded from
 * the amax and written 0.  Slots (amax_bits / counters / scales, each
 * B*H + 2*B*Hkv long; amax_bits and counters caller-zeroed) are Q heads, then
 * K heads, then V heads.  Results are bit-identical to ia_quant_amax_rows +
 * ia_quant_scales + ia_quantize.  Large slabs: one launch, each f32 element read
 * from HBM once (team barrier per slab, L2 re-read); many small slabs: an amax
 * launch and a quantise launch. */
int ia_quant_heads(const float* q, const float* k, const float* v, int64_t B, int64_t H,
                   int64_t Hkv, int64_t L, int64_t d, const int32_t* seq_lens, int8_t* qhat,
                   int8_t* khat, int8_t* vt, int64_t d_pad, int64_t l_pad, uint32_t* amax_bits,
                   int32_t* counters, float* scales, int32_t* err_flag, void* stream);
/* ia_quant_heads with per-TENSOR scales (QuantGranularity per-tensor,
 * quantize.py:26-56,104-123: one max|x| over all heads of Q, of K, of V; the
 * global-scale C2 config).  amax_bits (caller-zeroed) and scales hold 3 slots:
 * Q, K, V.  Two launches (amax over every slab, then quantise from the three
 * scales); bit-identical to ia_quant_amax_rows + ia_quant_scales + ia_quantize
 * with one slot per tensor. */
int ia_quant_tensors(const float* q, const float* k, const float* v, int64_t B, int64_t H,
                     int64_t Hkv, int64_t L, int64_t d, const int32_t* seq_lens, int8_t* qhat,
                     int8_t* khat, int8_t* vt, int64_t d_pad, int64_t l_pad, uint32_t* amax_bits,
                     float* scales, int32_t* err_flag, void* stream);
/* out = f32(values) * scale (quantize.py:126-128), same scale indexing. */
int ia_dequantize(const int8_t* values, int64_t rows, int64_t cols, int mode,
                  int64_t group, const float* scales, float* out, void* stream);

/* ------------------------------------------------------------------ per-head parameters
 * c_int = max(1, min(round_half_away(c / alpha), 2^52)), alpha =
 * f64(s_q) f64(s_k) / sqrt(d) (gemm.py:105, softmax.py:105-121), plus the
 * exact magic-number form of idx = (2 k delta' + c) // (2c) used on device and
 * the output scale f32(f64(s_v) / p_scale) (pipeline.py:250-252). */
typedef struct ia_head_params {
  int64_t c_int;    /* the reference's c_int */
  int64_t c_eff;    /* min(c_int, 2k*2*d*127^2 + 1): same idx for every logit */
  uint32_t magic;   /* idx = umulhi(n, magic) >> shift, n = 2k*delta' + c_eff */
  int32_t shift;
  int32_t use32;    /* 1: the 32-bit magic path is exact for every reachable n */
  float out_scale;
  float s_q, s_k, s_v;
  int32_t unc32;    /* 1: the magic is also exact without the clip (n up to 2k*2*d*127^2 + c_eff) */
  uint32_t magic9;  /* 0, or: idx * 512 = umulhi(n, magic9) & ~511 for the clipped n range */
  float fratio;     /* 0, or the largest f32 below k / c_eff when c_eff (2k + 1) < 2^23: the float
                     * form idx = k - RN(max(a - (m - c_eff), 0) * fratio) is then exact */
} ia_head_params;

int ia_head_params_host(double c, int64_t d, int nlut, int p_scale, float s_q, float s_k,
                        float s_v, ia_head_params* out);
/* Index map of one (query head, key group) of the grouped-K fused kernel: c_eff and
 * the magic numbers of ia_head_params for c_int = round(c / alpha_g), alpha_g =
 * f64(s_q) f64(s_k[g]) / sqrt(d) (softmax.py:370-378).  A group whose c_eff does
 * not fit 31 bits has idx = 0 for every reachable delta and is stored as magic 0.
 * use32 bit 1 set: c_eff (2k + 1) < 2^23, the kernel uses the float form of the map
 * and `magic` holds the bits of its f32 ratio (the largest f32 below k / c_eff). */
typedef struct ia_group_params {
  int32_t c_eff;
  uint32_t magic;
  int32_t shift;
  int32_t use32;
} ia_group_params;
/* out[(b*H + h) * n_groups + g] from q_scales [B*H] and k_scales [B*Hkv, n_groups]
 * (device arrays, stream-ordered). */
int ia_group_params_dev(const float* q_scales, const float* k_scales, int64_t B, int64_t H,
                        int64_t Hkv, int64_t n_groups, int64_t d, double c, int nlut,
                        ia_group_params* out, void* stream);
/* Index-map parameters for a given c_int (clamped to 2^52 as softmax.py:277)
 * and an upper bound on delta = rowmax - logit (2^32 - 1 covers any int32
 * logits); used with ia_index_softmax. */
int ia_softmax_params_host(int64_t c_int, int64_t delta_bound, int nlut, ia_head_params* out);
/* One entry per (b, h) query unit; *_per_head = 0 selects scales[0]. */
int ia_head_params_dev(const float* q_scales, const float* k_scales, const float* v_scales,
                       int q_per_head, int kv_per_head, int64_t B, int64_t H, int64_t Hkv,
                       int64_t d, double c, int nlut, int p_scale, ia_head_params* out,
                       void* stream);

/* Pack a bool [L, L] mask (nonzero = excluded) into bits [L, ceil(L/32)]. */
int ia_mask_pack(const uint8_t* mask, int64_t L, uint32_t* bits, void* stream);

/* ------------------------------------------------------------------ fused attention
 * Replaces the per-head body of int_attention (pipeline.py:215-253):
 * gemm_qk -> index_softmax -> gemm_pv -> rescale, fused per (b, h, 128-row
 * query tile); the int32 logits and u8 probabilities stay in TMEM/registers.
 * Requires d <= 256 and d_pad in {32, 64, 128, 256} (d_pad >= d); L <= 65536;
 * H % Hkv == 0 (query head h reads KV head h / (H / Hkv)). */
typedef struct ia_attn_args {
  const int8_t* q;   /* [B*H, L, d_pad] quantised Q (pad columns zero) */
  const int8_t* k;   /* [B*Hkv, L, d_pad] quantised K (pad columns zero) */
  const int8_t* vt;  /* [B*Hkv, d_pad, l_pad] quantised V, transposed per head */
  float* out;        /* [B*H, L, d] f32 */
  const ia_head_params* params; /* [B*H] device */
  const int32_t* seq_lens;      /* [B] device or NULL: query/key rows >= len are padding */
  const uint32_t* mask_bits;    /* [L, ceil(L/32)] device or NULL (1 = excluded) */
  int64_t B, H, Hkv, L, d, d_pad, l_pad;
  int32_t causal;    /* key j > query i excluded */
  int32_t nlut;      /* 2^b, 4..256 */
  int32_t p_scale;   /* 255 (UINT8X255) or 127 (INT8X127) */
  uint8_t lut[256];  /* ExpLut entries (softmax.py:88-102) */
  int32_t* dbg_logits; /* optional [B*H, L, L] int32 (debug/parity dump) */
  uint8_t* dbg_prob;   /* optional [B*H, L, L] u8 */
  int32_t* dbg_acc;    /* optional [B*H, L, d_pad] int32 */
  long long* dbg_times; /* optional [grid, 16] int64 per-CTA phase clocks (zeroed; profiling) */
  int32_t softmax_mode; /* IA_SOFTMAX_INDEX: IndexSoftmax (softmax.py:265-299, bit-exact);
                           IA_SOFTMAX_FLOAT: the quant-only comparator's dequantise -> f32
                           softmax -> requantise path (pipeline.py:259-296), with MUFU exp2,
                           so P^ matches the reference to float tolerance, not bit for bit */
  /* Grouped K (per-row-group key scales; softmax.py:309-399 default mode, pipeline.py:
   * 229-246): k_group_size keys (a power of two in [8, 128]) share one K scale, and
   * kgroup_params [B*H, ceil(L / k_group_size)] (device, from ia_group_params_dev)
   * holds each (query head, key group)'s index map.  k_group_size = 0: per-head K. */
  const struct ia_group_params* kgroup_params;
  int32_t k_group_size;
} ia_attn_args;
#define IA_SOFTMAX_INDEX 0
#define IA_SOFTMAX_FLOAT 1

int ia_attn_fwd(const ia_attn_args* args, void* stream);
/* IA_OK if the fused kernel supports (d_pad, 2^b LUT entries) within shared
 * memory (d_pad 256 with b >= 6 does not); otherwise use the stage operators. */
int ia_attn_supported(int64_t d_pad, int nlut);

/* ------------------------------------------------------------------ stage operators
 * index_softmax (softmax.py:265-299 / :131-204): logits [rows, cols] int32,
 * optional mask [rows, cols] u8 (nonzero = excluded), out [rows, cols] u8.
 * hp is a HOST pointer (from ia_head_params_host; c_eff/magic/shift/use32). */
int ia_index_softmax(const int32_t* logits, int64_t rows, int64_t cols,
                     const ia_head_params* hp, const uint8_t* lut, int nlut, int p_scale,
                     const uint8_t* mask, uint8_t* out, void* stream);

/* index_softmax_grouped (softmax.py:309-399, default per-group-max mode):
 * group_of_column [cols] int32 (device) maps each column to a group in
 * [0, n_groups), n_groups <= 4096; hp [n_groups] is a DEVICE array of
 * per-group index-map parameters (ia_softmax_params_host(c_int^(g), ...)).
 * Masked columns get e = 0; the row normalisation is shared by all groups. */
int ia_index_softmax_grouped(const int32_t* logits, int64_t rows, int64_t cols,
                             const int32_t* group_of_column, int n_groups,
                             const ia_head_params* hp, const uint8_t* lut, int nlut,
                             int p_scale, const uint8_t* mask, uint8_t* out, void* stream);

/* Exact int8 GEMM on tcgen05 (matmul_int8 / gemm_qk / gemm_pv, gemm.py:45-133):
 * C[M, N] int32 = A[M, K] * B[N, K]^T; A is s8 (a_signed = 1) or u8; B is s8.
 * lda/ldb are byte pitches (multiples of 16); ldc in elements. */
int ia_gemm_i8(const void* A, int64_t lda, int a_signed, const int8_t* B, int64_t ldb,
               int64_t M, int64_t N, int64_t K, int32_t* C, int64_t ldc, void* stream);

/* Host pipeline staging (no reference counterpart; the reference computes on the
 * host): `height` rows of `width` bytes from src (pitch spitch) to dst (pitch dpitch),
 * stream-ordered, either direction (cudaMemcpyDefault).  Used to move the valid rows
 * of every head of a padded batch entry in one copy. */
int ia_copy_rows_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                       int64_t width, int64_t height, void* stream);

/* Zeroes `bytes` bytes of device scratch on the stream (cudaMemsetAsync): the quantiser's
 * amax slots, team arrival counters and error flag must be zero before each call, and a
 * memset node costs no kernel launch of the caller's framework. */
int ia_zero_async(void* dst, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* INTATTN_B200_H */
