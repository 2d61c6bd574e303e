// softmax_rows.cu -- standalone IndexSoftmax over a materialised int32 logit
// matrix (the reference's index_softmax operator, softmax.py:265-299 with the
// row kernels :131-204).  Used by the stage-level API (index_softmax) and the
// unfused path; the fused attention kernel never materialises logits.
// One CTA per row: max -> idx/S -> per-row table -> gather.
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "params.cuh"

namespace ia {

constexpr int SR_THREADS = 256;

__global__ void __launch_bounds__(SR_THREADS)
    index_softmax_rows_kernel(const int32_t* __restrict__ logits, int64_t rows, int64_t cols,
                              const ia_head_params hp, const uint8_t* __restrict__ lut_g, int nlut,
                              uint32_t scale_x2, const uint8_t* __restrict__ mask,
                              uint8_t* __restrict__ out) {
  __shared__ uint32_t lut_s[256];
  __shared__ uint32_t tab[256];
  __shared__ int32_t red_i[SR_THREADS / 32];
  __shared__ uint32_t red_u[SR_THREADS / 32];
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int t = tid; t < 256; t += SR_THREADS) lut_s[t] = t < nlut ? lut_g[t] : 0u;
  const uint32_t k = (uint32_t)(nlut - 1);
  __syncthreads();
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int32_t* row = logits + r * cols;
    const uint8_t* mrow = mask ? mask + r * cols : nullptr;
    uint8_t* orow = out + r * cols;
    int32_t mx = INT_MIN;  // softmax.py:139-143 / :174-179
    int seen = 0;
    for (int64_t j = tid; j < cols; j += SR_THREADS)
      if (!mrow || !mrow[j]) { mx = max(mx, row[j]); seen = 1; }
    seen = __syncthreads_or(seen);
    mx = warp_max_i32(mx);
    if (l == 0) red_i[w] = mx;
    __syncthreads();
    mx = red_i[0];
    for (int q = 1; q < SR_THREADS / 32; ++q) mx = max(mx, red_i[q]);
    __syncthreads();
    if (!seen) {  // fully masked row (softmax.py:181-184)
      for (int64_t j = tid; j < cols; j += SR_THREADS) orow[j] = 0;
      continue;
    }
    IdxMap im;
    im.init(mx, hp, k);
    uint32_t s = 0;
    for (int64_t j = tid; j < cols; j += SR_THREADS) {  // softmax.py:144-155
      uint32_t idx;
      if (mrow && mrow[j]) idx = k;
      else idx = hp.use32 ? im.idx(row[j]) : idx_slow(mx, row[j], hp.c_eff, k);
      orow[j] = (uint8_t)idx;
      s += lut_s[idx];
    }
    s = warp_sum_u32(s);
    if (l == 0) red_u[w] = s;
    __syncthreads();
    s = 0;
    for (int q = 0; q < SR_THREADS / 32; ++q) s += red_u[q];
    for (int t = tid; t < nlut; t += SR_THREADS)  // softmax.py:157-160
      tab[t] = (scale_x2 * lut_s[t] + s) / (2u * s);
    __syncthreads();
    for (int64_t j = tid; j < cols; j += SR_THREADS) orow[j] = (uint8_t)tab[orow[j]];
    __syncthreads();
  }
}


// Grouped-key IndexSoftmax (softmax.py:309-399, default per-group-max mode): columns
// are partitioned by group_of_column; group g has its own clip threshold c_int^(g)
// (hp[g].c_eff, from ia_softmax_params_host) and its own row max over the row's
// unmasked columns of g.  The LUT and the integer row normalisation are shared.
// One CTA per row; group maxima live in shared memory (n_groups <= SRG_MAX_GROUPS).
constexpr int SRG_MAX_GROUPS = 4096;

__global__ void __launch_bounds__(SR_THREADS)
    index_softmax_grouped_kernel(const int32_t* __restrict__ logits, int64_t rows, int64_t cols,
                                 const int32_t* __restrict__ group_of_column, int n_groups,
                                 const ia_head_params* __restrict__ hp, const uint8_t* __restrict__ lut_g,
                                 int nlut, uint32_t scale_x2, const uint8_t* __restrict__ mask,
                                 uint8_t* __restrict__ out) {
  __shared__ int32_t gmax[SRG_MAX_GROUPS];
  __shared__ uint32_t lut_s[256];
  __shared__ uint32_t tab[256];
  __shared__ uint32_t red_u[SR_THREADS / 32];
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  for (int t = tid; t < 256; t += SR_THREADS) lut_s[t] = t < nlut ? lut_g[t] : 0u;
  const int64_t k = nlut - 1;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int32_t* row = logits + r * cols;
    const uint8_t* mrow = mask ? mask + r * cols : nullptr;
    uint8_t* orow = out + r * cols;
    for (int g = tid; g < n_groups; g += SR_THREADS) gmax[g] = INT_MIN;
    __syncthreads();
    // per-group row max over unmasked columns (softmax.py:384-390); a thread's run of
    // equal groups is folded locally before the shared atomic
    int cg = -1;
    int32_t cm = INT_MIN;
    for (int64_t j = tid; j < cols; j += SR_THREADS) {
      if (mrow && mrow[j]) continue;
      const int g = group_of_column[j];
      if (g != cg) {
        if (cg >= 0) atomicMax(gmax + cg, cm);
        cg = g;
        cm = INT_MIN;
      }
      cm = max(cm, row[j]);
    }
    if (cg >= 0) atomicMax(gmax + cg, cm);
    __syncthreads();
    // e = lut[(2 k min(m_g - a, c_g) + c_g) // (2 c_g)], masked -> 0 (softmax.py:391-396)
    uint32_t s = 0;
    for (int64_t j = tid; j < cols; j += SR_THREADS) {
      uint32_t e = 0;
      if (!(mrow && mrow[j])) {
        const int g = group_of_column[j];
        e = lut_s[idx_slow(gmax[g], row[j], hp[g].c_eff, k)];
      }
      orow[j] = (uint8_t)e;
      s += e;
    }
    s = warp_sum_u32(s);
    if (l == 0) red_u[w] = s;
    __syncthreads();
    s = 0;
    for (int q = 0; q < SR_THREADS / 32; ++q) s += red_u[q];
    // (2 scale e + s) // max(2s, 1) for every possible e (softmax.py:300-306)
    const uint32_t den = s ? 2u * s : 1u;
    for (int t = tid; t < 256; t += SR_THREADS) tab[t] = (scale_x2 * (uint32_t)t + s) / den;
    __syncthreads();
    for (int64_t j = tid; j < cols; j += SR_THREADS) orow[j] = (uint8_t)tab[orow[j]];
    __syncthreads();
  }
}

}  // namespace ia

using namespace ia;

extern "C" int ia_index_softmax(const int32_t* logits, int64_t rows, int64_t cols,
                                const ia_head_params* hp, const uint8_t* lut, int nlut,
                                int p_scale, const uint8_t* mask, uint8_t* out, void* stream) {
  if (!logits || !hp || !lut || !out || rows < 1 || cols < 1 || nlut < 4 || nlut > 256 ||
      (p_scale != 255 && p_scale != 127))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_index_softmax: bad arguments");
  if (cols > IA_MAX_SEQ_LEN) return fail(IA_ERR_SEQ_LEN, "sequence length exceeds 65536");
  int64_t blocks = rows < (int64_t)num_sms() * 8 ? rows : (int64_t)num_sms() * 8;
  index_softmax_rows_kernel<<<(unsigned)blocks, SR_THREADS, 0, (cudaStream_t)stream>>>(
      logits, rows, cols, *hp, lut, nlut, 2u * (uint32_t)p_scale, mask, out);
  return check_launch("index_softmax_rows_kernel");
}

extern "C" int ia_index_softmax_grouped(const int32_t* logits, int64_t rows, int64_t cols,
                                        const int32_t* group_of_column, int n_groups,
                                        const ia_head_params* hp, const uint8_t* lut, int nlut,
                                        int p_scale, const uint8_t* mask, uint8_t* out,
                                        void* stream) {
  if (!logits || !group_of_column || !hp || !lut || !out || rows < 1 || cols < 1 ||
      n_groups < 1 || nlut < 4 || nlut > 256 || (p_scale != 255 && p_scale != 127))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_index_softmax_grouped: bad arguments");
  if (n_groups > SRG_MAX_GROUPS)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_index_softmax_grouped: more than %d groups",
                SRG_MAX_GROUPS);
  if (cols > IA_MAX_SEQ_LEN) return fail(IA_ERR_SEQ_LEN, "sequence length exceeds 65536");
  int64_t blocks = rows < (int64_t)num_sms() * 8 ? rows : (int64_t)num_sms() * 8;
  index_softmax_grouped_kernel<<<(unsigned)blocks, SR_THREADS, 0, (cudaStream_t)stream>>>(
      logits, rows, cols, group_of_column, n_groups, hp, lut, nlut, 2u * (uint32_t)p_scale, mask,
      out);
  return check_launch("index_softmax_grouped_kernel");
}
