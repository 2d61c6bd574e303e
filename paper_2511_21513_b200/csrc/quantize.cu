// quantize.cu -- dynamic symmetric INT8 quantiser (reference quantize.py:92-128).
//
// HBM-bound: f32 read -> int8 write.  Two stream-ordered kernels: a grid-wide
// max|x| (float bit pattern atomics, exact) and the quantise pass.  All f32
// arithmetic uses explicit round-to-nearest intrinsics so the result is the
// IEEE value numpy computes: s = max(amax, 1e-12f) / 127f, t = x / s,
// q = copysign(floor(|t| + 0.5f), t) clipped to [-127, 127].
#include <cstdint>

#include "common.cuh"

namespace ia {

__device__ __forceinline__ float q_scale(uint32_t amax_bits) {
  const float a = __uint_as_float(amax_bits);
  return __fdiv_rn(fmaxf(a, 1e-12f), 127.0f);  // quantize.py:113
}

__device__ __forceinline__ int8_t q_value(float x, float s) {
  const float t = __fdiv_rn(x, s);                     // x / grid (quantize.py:121)
  float r = floorf(__fadd_rn(fabsf(t), 0.5f));         // rounding.py:21
  r = fminf(r, 127.0f);                                // clip (quantize.py:122)
  const int v = (int)r;
  return (int8_t)(t < 0.0f ? -v : v);
}

__device__ __forceinline__ uint32_t absbits(float x) { return __float_as_uint(x) & 0x7fffffffu; }
__device__ __forceinline__ bool nonfinite_bits(uint32_t b) { return b >= 0x7f800000u; }

// grid: (chunks, n_rowgroups).  Each block reduces a strided slice of its row group.
__global__ void amax_rows_kernel(const float* __restrict__ x, int64_t n_rowgroups,
                                 int64_t rows_per_group,
                                 int64_t cols, const int32_t* __restrict__ valid_rows,
                                 int64_t valid_div, int64_t slot_div,
                                 uint32_t* __restrict__ amax_bits, int32_t* __restrict__ err) {
  __shared__ uint32_t red[32];
  for (int64_t g = blockIdx.y; g < n_rowgroups; g += gridDim.y) {
  int64_t nrows = rows_per_group;
  if (valid_rows) {
    const int64_t v = valid_rows[g / valid_div];
    nrows = v < nrows ? (v < 0 ? 0 : v) : nrows;
  }
  const int64_t n = nrows * cols;
  const float* base = x + g * rows_per_group * cols;
  uint32_t m = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((((uintptr_t)base) & 15) == 0) {
    const int64_t n4 = n >> 2;
    const float4* b4 = reinterpret_cast<const float4*>(base);
    for (int64_t i = i0; i < n4; i += stride) {
      const float4 v = __ldg(b4 + i);
      m = max(m, max(max(absbits(v.x), absbits(v.y)), max(absbits(v.z), absbits(v.w))));
    }
    for (int64_t i = (n4 << 2) + i0; i < n; i += stride) m = max(m, absbits(base[i]));
  } else {
    for (int64_t i = i0; i < n; i += stride) m = max(m, absbits(base[i]));
  }
  // NaN bit patterns compare above +inf: any non-finite element lifts m >= 0x7f800000.
  m = warp_max_u32(m);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = m;
  __syncthreads();
  if (w == 0) {
    m = l < (int)(blockDim.x >> 5) ? red[l] : 0u;
    m = warp_max_u32(m);
    if (l == 0) {
      if (nonfinite_bits(m)) {
        atomicOr(reinterpret_cast<unsigned int*>(err), 1u);
      } else if (m) {
        atomicMax(amax_bits + g / slot_div, m);
      }
    }
  }
  __syncthreads();
  }
}

__global__ void amax_cols_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                 int64_t col_group, uint32_t* __restrict__ amax_bits,
                                 int32_t* __restrict__ err) {
  // grid-stride over elements; one atomic per (thread, column group) change.
  const int64_t n = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t b = absbits(x[i]);
    if (nonfinite_bits(b)) atomicOr(reinterpret_cast<unsigned int*>(err), 1u);
    else if (b) atomicMax(amax_bits + (i % cols) / col_group, b);
  }
}

__global__ void scales_kernel(const uint32_t* __restrict__ amax_bits, int64_t n,
                              float* __restrict__ scales) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) scales[i] = q_scale(amax_bits[i]);
}

// Row-major output: thread handles 4 consecutive output columns of one row.
__global__ void quantize_rows_kernel(const float* __restrict__ x, int64_t total_rows,
                                     int64_t rows_per_group, int64_t cols,
                                     const int32_t* __restrict__ valid_rows, int64_t valid_div,
                                     int mode, int64_t slot_div, int64_t col_group,
                                     const float* __restrict__ scales, int8_t* __restrict__ out,
                                     int64_t out_pitch) {
  const int64_t q4 = out_pitch >> 2;
  const int64_t n = total_rows * q4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / q4;
    const int64_t c0 = (i - r * q4) << 2;
    const int64_t g = r / rows_per_group;
    bool valid = true;
    if (valid_rows) valid = (r - g * rows_per_group) < (int64_t)valid_rows[g / valid_div];
    uint32_t packed = 0;
    if (valid) {
      const float* xr = x + r * cols;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t c = c0 + e;
        if (c < cols) {
          const float s = mode == IA_QMODE_ROWS ? scales[g / slot_div] : scales[c / col_group];
          packed |= (uint32_t)(uint8_t)q_value(__ldg(xr + c), s) << (8 * e);
        }
      }
    }
    *reinterpret_cast<uint32_t*>(out + r * out_pitch + c0) = packed;
  }
}

__device__ __forceinline__ uint32_t q_pack4(float4 v, float s) {
  return (uint32_t)(uint8_t)q_value(v.x, s) | ((uint32_t)(uint8_t)q_value(v.y, s) << 8) |
         ((uint32_t)(uint8_t)q_value(v.z, s) << 16) | ((uint32_t)(uint8_t)q_value(v.w, s) << 24);
}

// q_value via x * (1/s), with the IEEE quotient only within 2^-15 of a k + 0.5 rounding
// boundary (same result bit for bit; the argument is at quant_heads.cu:qh_q).
__device__ __forceinline__ int8_t q_value_rcp(float x, float s, float rcp) {
  float t = __fmul_rn(x, rcp);
  const float at = fabsf(t);
  if (fabsf(__fsub_rn(__fsub_rn(at, floorf(at)), 0.5f)) <= 3.0517578125e-05f) t = __fdiv_rn(x, s);
  float r = floorf(__fadd_rn(fabsf(t), 0.5f));
  r = fminf(r, 127.0f);
  const int v = (int)r;
  return (int8_t)(t < 0.0f ? -v : v);
}
__device__ __forceinline__ uint32_t q_pack4_rcp(float4 v, float s, float rcp) {
  return (uint32_t)(uint8_t)q_value_rcp(v.x, s, rcp) | ((uint32_t)(uint8_t)q_value_rcp(v.y, s, rcp) << 8) |
         ((uint32_t)(uint8_t)q_value_rcp(v.z, s, rcp) << 16) |
         ((uint32_t)(uint8_t)q_value_rcp(v.w, s, rcp) << 24);
}

// Vectorised row-major fast path (ROWS mode, cols % 4 == 0, 16-byte aligned
// input, out_pitch % 16 == 0): each thread produces one 16-byte output chunk
// (4 float4 loads -> 16 int8), a row is out_pitch/16 consecutive threads.
__global__ void __launch_bounds__(256) quantize_rows_vec_kernel(
    const float* __restrict__ x, int64_t total_rows, int64_t rows_per_group, int cols,
    const int32_t* __restrict__ valid_rows, int64_t valid_div, int64_t slot_div,
    const float* __restrict__ scales, int8_t* __restrict__ out, int out_pitch) {
  const int chunks = out_pitch >> 4;           // 16-byte chunks per row (<= 64)
  const int rows_per_iter = blockDim.x / chunks;
  const int lr = threadIdx.x / chunks, ch = threadIdx.x - lr * chunks;
  if (lr >= rows_per_iter) return;
  const int c0 = ch << 4;
  for (int64_t r = (int64_t)blockIdx.x * rows_per_iter + lr; r < total_rows;
       r += (int64_t)gridDim.x * rows_per_iter) {
    const int64_t g = r / rows_per_group;
    bool valid = true;
    if (valid_rows) valid = (r - g * rows_per_group) < (int64_t)valid_rows[g / valid_div];
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (valid && c0 < cols) {
      const float s = scales[g / slot_div];
      const float rc = __frcp_rn(s);
      const float4* xr = reinterpret_cast<const float4*>(x + r * cols + c0);
      if (c0 + 16 <= cols) {
        const float4 a = __ldg(xr), b = __ldg(xr + 1), c = __ldg(xr + 2), d = __ldg(xr + 3);
        o = make_uint4(q_pack4_rcp(a, s, rc), q_pack4_rcp(b, s, rc), q_pack4_rcp(c, s, rc),
                       q_pack4_rcp(d, s, rc));
      } else {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        for (int e = 0; e < 4 && c0 + 4 * e < cols; ++e) w[e] = q_pack4_rcp(__ldg(xr + e), s, rc);
        o = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    *reinterpret_cast<uint4*>(out + r * out_pitch + c0) = o;
  }
}

// Vectorised V^T fast path: 64 rows x 64 columns per block, float4 loads along
// the columns, transposed through smem, 16-byte stores along the rows.
__global__ void __launch_bounds__(256) quantize_rows_t_vec_kernel(
    const float* __restrict__ x, int rows_per_group, int cols,
    const int32_t* __restrict__ valid_rows, int64_t valid_div, int64_t slot_div,
    const float* __restrict__ scales, int8_t* __restrict__ out, int out_pitch, int out_rows,
    int64_t out_group_stride) {
  __shared__ uint8_t tile[64][64 + 16];
  const int64_t g = blockIdx.z;
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  int nvalid = rows_per_group;
  if (valid_rows) {
    const int v = valid_rows[g / valid_div];
    nvalid = v < nvalid ? v : nvalid;
  }
  const float s = scales[g / slot_div];
  const float rc = __frcp_rn(s);
  const float* xg = x + g * (int64_t)rows_per_group * cols;
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // 64 rows x 16 float4 = 1024 loads
    const int t = threadIdx.x + k * 256;
    const int rr = t >> 4, c4 = (t & 15) << 2;
    const int r = r0 + rr, c = c0 + c4;
    uint32_t q = 0;
    if (r < nvalid && c < cols) q = q_pack4_rcp(__ldg(reinterpret_cast<const float4*>(xg + (int64_t)r * cols + c)), s, rc);
    tile[c4 + 0][rr] = (uint8_t)q;
    tile[c4 + 1][rr] = (uint8_t)(q >> 8);
    tile[c4 + 2][rr] = (uint8_t)(q >> 16);
    tile[c4 + 3][rr] = (uint8_t)(q >> 24);
  }
  __syncthreads();
  const int cc = threadIdx.x >> 2, r16 = (threadIdx.x & 3) << 4;  // 64 cols x 4 chunks of 16 rows
  const int c = c0 + cc, r = r0 + r16;
  if (c < out_rows && r < out_pitch) {
    const uint32_t* tw = reinterpret_cast<const uint32_t*>(&tile[cc][r16]);
    *reinterpret_cast<uint4*>(out + g * out_group_stride + (int64_t)c * out_pitch + r) =
        make_uint4(tw[0], tw[1], tw[2], tw[3]);
  }
}

// Transposed output per row group: out[g][c][r] (V^T), 64x64 tiles through smem.
__global__ void quantize_rows_t_kernel(const float* __restrict__ x, int64_t rows_per_group,
                                       int64_t cols, const int32_t* __restrict__ valid_rows,
                                       int64_t valid_div, int64_t slot_div,
                                       const float* __restrict__ scales,
                                       int8_t* __restrict__ out, int64_t out_pitch,
                                       int64_t out_group_stride) {
  __shared__ uint8_t tile[64][68];
  const int64_t g = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  int64_t nvalid = rows_per_group;
  if (valid_rows) {
    const int64_t v = valid_rows[g / valid_div];
    nvalid = v < nvalid ? v : nvalid;
  }
  const float s = scales[g / slot_div];
  const float* xg = x + g * rows_per_group * cols;
  for (int t = threadIdx.x; t < 64 * 64; t += blockDim.x) {
    const int rr = t >> 6, cc = t & 63;
    const int64_t r = r0 + rr, c = c0 + cc;
    int8_t q = 0;
    if (r < nvalid && c < cols) q = q_value(__ldg(xg + r * cols + c), s);
    tile[cc][rr] = (uint8_t)q;  // c >= cols (padding rows of V^T) stay 0
  }
  __syncthreads();
  int8_t* og = out + g * out_group_stride;
  const int64_t out_rows = out_group_stride / out_pitch;  // >= cols; rows [cols, out_rows) -> 0
  for (int t = threadIdx.x; t < 64 * 16; t += blockDim.x) {
    const int cc = t >> 4, r4 = (t & 15) << 2;
    const int64_t c = c0 + cc, r = r0 + r4;
    if (c >= out_rows) continue;
    if (r + 3 < out_pitch) {
      uint32_t p = (uint32_t)tile[cc][r4] | ((uint32_t)tile[cc][r4 + 1] << 8) |
                   ((uint32_t)tile[cc][r4 + 2] << 16) | ((uint32_t)tile[cc][r4 + 3] << 24);
      *reinterpret_cast<uint32_t*>(og + c * out_pitch + r) = p;
    } else {
      for (int e = 0; e < 4 && r + e < out_pitch; ++e) og[c * out_pitch + r + e] = (int8_t)tile[cc][r4 + e];
    }
  }
}

__global__ void dequantize_kernel(const int8_t* __restrict__ v, int64_t rows, int64_t cols,
                                  int mode, int64_t group, const float* __restrict__ scales,
                                  float* __restrict__ out) {
  const int64_t n = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    const float s = mode == IA_QMODE_ROWS ? scales[r / group] : scales[c / group];
    out[i] = __fmul_rn((float)v[i], s);  // quantize.py:128
  }
}

}  // namespace ia

using namespace ia;

extern "C" int ia_quant_amax_rows(const float* x, int64_t n_rowgroups, int64_t rows_per_group,
                                  int64_t cols, const int32_t* valid_rows, int64_t valid_div,
                                  int64_t slot_div, uint32_t* amax_bits, int32_t* err_flag,
                                  void* stream) {
  if (!x || !amax_bits || !err_flag || n_rowgroups < 1 || rows_per_group < 1 || cols < 1 ||
      slot_div < 1 || valid_div < 1)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_amax_rows: bad arguments");
  const int64_t per_group = rows_per_group * cols;
  const int threads = 256;
  int64_t chunks = (per_group / 4 + threads * 8 - 1) / (threads * 8);
  const int64_t target = (int64_t)num_sms() * 8;
  const int64_t cap = (target + n_rowgroups - 1) / n_rowgroups;
  chunks = chunks < 1 ? 1 : (chunks > cap ? (cap < 1 ? 1 : cap) : chunks);
  dim3 grid((unsigned)chunks, (unsigned)(n_rowgroups < 65535 ? n_rowgroups : 65535));
  amax_rows_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(
      x, n_rowgroups, rows_per_group, cols, valid_rows, valid_div, slot_div, amax_bits, err_flag);
  return check_launch("amax_rows_kernel");
}

extern "C" int ia_quant_amax_cols(const float* x, int64_t rows, int64_t cols, int64_t col_group,
                                  uint32_t* amax_bits, int32_t* err_flag, void* stream) {
  if (!x || !amax_bits || !err_flag || rows < 1 || cols < 1 || col_group < 1)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_amax_cols: bad arguments");
  const int64_t n = rows * cols;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  amax_cols_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, rows, cols, col_group,
                                                                      amax_bits, err_flag);
  return check_launch("amax_cols_kernel");
}

extern "C" int ia_quant_scales(const uint32_t* amax_bits, int64_t n, float* scales, void* stream) {
  if (!amax_bits || !scales || n < 1) return fail(IA_ERR_INVALID_ARGUMENT, "ia_quant_scales");
  scales_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(amax_bits, n,
                                                                              scales);
  return check_launch("scales_kernel");
}

extern "C" int ia_quantize(const float* x, int64_t n_rowgroups, int64_t rows_per_group,
                           int64_t cols, const int32_t* valid_rows, int64_t valid_div, int mode,
                           int64_t slot_div, int64_t col_group, const float* scales, int8_t* out,
                           int64_t out_pitch, int transpose, int64_t out_group_stride,
                           void* stream) {
  if (!x || !scales || !out || n_rowgroups < 1 || rows_per_group < 1 || cols < 1 ||
      valid_div < 1 || slot_div < 1 || (mode != IA_QMODE_ROWS && mode != IA_QMODE_COLS) ||
      (mode == IA_QMODE_COLS && col_group < 1))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quantize: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (!transpose) {
    if (out_pitch < cols || (out_pitch & 3) || (((uintptr_t)out) & 3))
      return fail(IA_ERR_INVALID_ARGUMENT, "ia_quantize: out_pitch must be >= cols, %4");
    const int64_t rows = n_rowgroups * rows_per_group;
    if (mode == IA_QMODE_ROWS && (cols & 3) == 0 && (out_pitch & 15) == 0 && out_pitch <= 1024 &&
        cols <= 0x7fffffff && (((uintptr_t)x | (uintptr_t)out) & 15) == 0) {
      const int chunks = (int)(out_pitch >> 4);
      const int64_t rows_per_block = 256 / chunks;
      int64_t blocks = (rows + rows_per_block - 1) / rows_per_block;
      if (blocks > (int64_t)num_sms() * 32) blocks = (int64_t)num_sms() * 32;
      quantize_rows_vec_kernel<<<(unsigned)blocks, 256, 0, st>>>(
          x, rows, rows_per_group, (int)cols, valid_rows, valid_div, slot_div, scales, out,
          (int)out_pitch);
      return check_launch("quantize_rows_vec_kernel");
    }
    const int64_t n = rows * (out_pitch >> 2);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    quantize_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(
        x, rows, rows_per_group, cols, valid_rows, valid_div, mode, slot_div, col_group, scales,
        out, out_pitch);
    return check_launch("quantize_rows_kernel");
  }
  if (mode != IA_QMODE_ROWS || out_pitch < rows_per_group || (out_pitch & 3) ||
      n_rowgroups > 65535 || out_group_stride < cols * out_pitch)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_quantize: bad transpose arguments");
  const int64_t out_rows = out_group_stride / out_pitch;
  dim3 grid((unsigned)((rows_per_group + 63) / 64), (unsigned)((out_rows + 63) / 64),
            (unsigned)n_rowgroups);
  if ((cols & 3) == 0 && (out_pitch & 15) == 0 && (out_group_stride & 15) == 0 &&
      rows_per_group < 0x7fffffff && out_pitch < 0x7fffffff &&
      (((uintptr_t)x | (uintptr_t)out) & 15) == 0) {
    quantize_rows_t_vec_kernel<<<grid, 256, 0, st>>>(x, (int)rows_per_group, (int)cols, valid_rows,
                                                     valid_div, slot_div, scales, out,
                                                     (int)out_pitch, (int)out_rows,
                                                     out_group_stride);
    return check_launch("quantize_rows_t_vec_kernel");
  }
  quantize_rows_t_kernel<<<grid, 256, 0, st>>>(x, rows_per_group, cols, valid_rows, valid_div,
                                               slot_div, scales, out, out_pitch,
                                               out_group_stride);
  return check_launch("quantize_rows_t_kernel");
}

extern "C" int ia_dequantize(const int8_t* values, int64_t rows, int64_t cols, int mode,
                             int64_t group, const float* scales, float* out, void* stream) {
  if (!values || !scales || !out || rows < 1 || cols < 1 || group < 1)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_dequantize: bad arguments");
  const int64_t n = rows * cols;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  dequantize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(values, rows, cols, mode,
                                                                       group, scales, out);
  return check_launch("dequantize_kernel");
}
