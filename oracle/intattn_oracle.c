/*
 * intattn_oracle.c -- CPU restatement of the reference IntAttention forward
 * path.  TEST INFRASTRUCTURE ONLY: this file is the checker used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm.
 * The product package (paper_2511_21513_b200/) never links, imports or calls
 * it; the product path is the CUDA library and fails loudly without it.
 *
 * Every function restates the reference algorithm in plain C (independent of
 * the reference's Python/numba/OpenBLAS code) and cites the reference lines it
 * follows (paths relative to /root/reference/pkg/src/intattn/).  Integer work
 * is exact (64-bit accumulation / division); the f32 quantiser uses IEEE
 * single-precision division and the same round-half-away rule, so the result
 * is bit-identical to numpy's.  Build with -ffp-contract=off (see Makefile).
 *
 * Pinning: oracle/gen_golden.py imports the reference in this container and
 * writes tests/golden/; tests/test_oracle_golden.py checks this restatement
 * against those vectors and digests (SPEC KATs + all five BASELINE configs).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_NONFINITE 1
#define OR_ERR_ARGS 2

/* quantize.py:19 EPS = 1e-12, applied as np.float32(EPS) (quantize.py:113). */
static const float OR_EPS = 1e-12f;
/* softmax.py:47 _C_INT_CAP */
static const int64_t OR_C_INT_CAP = (int64_t)1 << 52;

int ia_or_abi_version(void) { return 1; }

/* max|x| over n elements (quantize.py:92-101); flags non-finite input
 * (quantize.py:109-110). */
float ia_or_amax(const float* x, int64_t n, int* nonfinite) {
  float m = 0.0f;
  int bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    float a = fabsf(x[i]);
    if (!isfinite(a)) bad = 1;
    if (a > m) m = a;
  }
  if (nonfinite) *nonfinite = bad;
  return m;
}

/* scale = max(eps, amax) / 127 in f32 (quantize.py:113). */
float ia_or_scale(float amax) {
  volatile float a = amax > OR_EPS ? amax : OR_EPS;
  return a / 127.0f;
}

/* values = clip(round_half_away(x / scale), -127, 127) (quantize.py:121-122,
 * rounding.py:21: copysign(floor(|t| + 0.5), t) evaluated in f32). */
void ia_or_quantize(const float* x, int64_t n, float scale, int8_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    float t = x[i] / scale;
    float r = floorf(fabsf(t) + 0.5f);
    if (r > 127.0f) r = 127.0f;
    int v = (int)r;
    out[i] = (int8_t)(t < 0.0f ? -v : v);
  }
}

/* c_int = max(1, min(round_half_away(c / alpha), 2^52)) with
 * alpha = f64(s_q) * f64(s_k) / sqrt(d)  (gemm.py:105, softmax.py:105-121). */
int64_t ia_or_c_int(double c, int64_t d, float s_q, float s_k) {
  volatile double alpha = (double)s_q * (double)s_k;
  alpha = alpha / sqrt((double)d);
  volatile double r = c / alpha;
  double t = floor(fabs(r) + 0.5);
  if (t >= (double)OR_C_INT_CAP) return OR_C_INT_CAP;
  int64_t ci = (int64_t)t;
  return ci < 1 ? 1 : ci;
}

/* Exact int32 a[m,k] @ b_t[n,k]^T (gemm.py:70-85; exact by gemm.py:1-13). */
void ia_or_matmul_s8(const int8_t* a, const int8_t* b_t, int64_t m, int64_t n,
                     int64_t k, int32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    const int8_t* ar = a + i * k;
    for (int64_t j = 0; j < n; ++j) {
      const int8_t* br = b_t + j * k;
      int32_t s = 0;
      for (int64_t t = 0; t < k; ++t) s += (int32_t)ar[t] * (int32_t)br[t];
      out[i * n + j] = s;
    }
  }
}

/* Exact int32 p[m,l] @ v[l,d]; p is uint8 (or int8 in [0,127] for the
 * INT8X127 ablation -- identical bits) (gemm.py:109-133). */
void ia_or_gemm_pv(const uint8_t* p, const int8_t* v, int64_t m, int64_t l,
                   int64_t d, int32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    int32_t* o = out + i * d;
    for (int64_t c = 0; c < d; ++c) o[c] = 0;
    const uint8_t* pr = p + i * l;
    for (int64_t j = 0; j < l; ++j) {
      int32_t pj = pr[j];
      if (!pj) continue;
      const int8_t* vr = v + j * d;
      for (int64_t c = 0; c < d; ++c) o[c] += pj * (int32_t)vr[c];
    }
  }
}

/* One IndexSoftmax row (softmax.py:131-204).  `mrow` (nullable) marks
 * excluded positions (True = masked).  `tmp` is caller scratch of `cols`.
 * Returns 0 if the row was fully masked (all zeros), else the row sum S. */
static uint32_t or_softmax_row(const int32_t* row, const uint8_t* mrow,
                               int64_t cols, int64_t c_int, const uint8_t* lut,
                               int nlut, uint32_t scale_x2, uint8_t* orow) {
  const int64_t last = nlut - 1, k = last;
  int64_t m = 0;
  int seen = 0;
  for (int64_t j = 0; j < cols; ++j) {          /* :139-143, :174-179 */
    if (mrow && mrow[j]) continue;
    if (!seen || (int64_t)row[j] > m) { m = row[j]; seen = 1; }
  }
  if (!seen) {                                   /* :181-184 */
    memset(orow, 0, (size_t)cols);
    return 0;
  }
  uint32_t s = 0;
  for (int64_t j = 0; j < cols; ++j) {          /* :144-155, :186-198 */
    int64_t idx;
    if (mrow && mrow[j]) {
      idx = last;
    } else {
      int64_t delta = m - (int64_t)row[j];
      if (delta >= c_int) idx = last;
      else idx = (2 * delta * k + c_int) / (2 * c_int);
    }
    orow[j] = (uint8_t)idx;
    s += (uint32_t)lut[idx];
  }
  uint8_t rowtab[256];                            /* :157-160 */
  uint32_t two_s = 2u * s;
  for (int t = 0; t < nlut; ++t)
    rowtab[t] = (uint8_t)((scale_x2 * (uint32_t)lut[t] + s) / two_s);
  for (int64_t j = 0; j < cols; ++j) orow[j] = rowtab[orow[j]];   /* :161-162 */
  return s;
}

/* index_softmax over a [rows, cols] int32 logit matrix (softmax.py:265-299).
 * p_scale is 255 (UINT8X255) or 127 (INT8X127). */
void ia_or_index_softmax(const int32_t* logits, int64_t rows, int64_t cols,
                         int64_t c_int, const uint8_t* lut, int nlut,
                         int p_scale, const uint8_t* mask, uint8_t* out) {
  if (c_int > OR_C_INT_CAP) c_int = OR_C_INT_CAP;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < rows; ++i)
    or_softmax_row(logits + i * cols, mask ? mask + i * cols : NULL, cols,
                   c_int, lut, nlut, (uint32_t)(2 * p_scale), out + i * cols);
}

/*
 * Batched attention over (b, h) units -- the reference's int_attention
 * (pipeline.py:202-256) applied per unit, as SURVEY.md §3.5/§8d composes it:
 *   q [B,H,L,d], k/v [B,Hkv,L,d] f32; query head h uses KV head h/(H/Hkv).
 *   scale_mode 0: per (b,head) slab over its valid rows; 1: one global scale
 *   per tensor (over valid rows); 2: given global scales (qs_out[0],
 *   ks_out[0], vs_out[0] are inputs -- the sharded launcher's all-reduced amax).  seq_lens (nullable) [B]: rows >= len are
 *   padding (excluded from amax, masked as keys, zero output as queries).
 *   causal: key j > query i masked.  mask (nullable) [L,L] u8 shared by all
 *   units (True = excluded).  row_stride > 1 computes only rows i with
 *   i % row_stride == 0 (a bounded CPU-baseline sample); other rows untouched.
 * Outputs: out [B,H,L,d] f32; optional qs [B*H], ks/vs [B*Hkv] scales and
 * c_int [B*H] per unit.
 */
int ia_or_attention_batched(const float* q, const float* k, const float* v,
                            int64_t B, int64_t H, int64_t Hkv, int64_t L,
                            int64_t d, const int32_t* seq_lens, int causal,
                            const uint8_t* mask, int scale_mode, double c,
                            const uint8_t* lut, int nlut, int p_scale,
                            int64_t row_stride, int n_threads, float* out,
                            float* qs_out, float* ks_out, float* vs_out,
                            int64_t* cint_out) {
  if (B < 1 || H < 1 || Hkv < 1 || H % Hkv || L < 1 || d < 1 || nlut < 2 ||
      row_stride < 1)
    return OR_ERR_ARGS;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  const int64_t group = H / Hkv;
  const int64_t nq = B * H * L * d, nkv = B * Hkv * L * d;
  int8_t* qh = (int8_t*)malloc((size_t)nq);
  int8_t* kh = (int8_t*)malloc((size_t)nkv);
  int8_t* vh = (int8_t*)malloc((size_t)nkv);
  float* sq = (float*)malloc(sizeof(float) * B * H);
  float* sk = (float*)malloc(sizeof(float) * B * Hkv);
  float* sv = (float*)malloc(sizeof(float) * B * Hkv);
  if (!qh || !kh || !vh || !sq || !sk || !sv) return OR_ERR_ARGS;
  int status = OR_OK;

  /* ---- quantise (quantize.py:104-123) ---- */
  const float* srcs[3] = {q, k, v};
  int8_t* dsts[3] = {qh, kh, vh};
  float* scs[3] = {sq, sk, sv};
  const int64_t heads[3] = {H, Hkv, Hkv};
  for (int t = 0; t < 3; ++t) {
    const int64_t nh = heads[t];
    float* amax = (float*)calloc((size_t)(B * nh), sizeof(float));
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t u = 0; u < B * nh; ++u) {
      int64_t b = u / nh;
      int64_t n = seq_lens ? seq_lens[b] : L;
      int nf = 0;
      amax[u] = ia_or_amax(srcs[t] + u * L * d, n * d, &nf);
      bad |= nf;
    }
    if (bad) status = OR_ERR_NONFINITE;
    if (scale_mode == 2) {
      const float* given[3] = {qs_out, ks_out, vs_out};
      for (int64_t u = 0; u < B * nh; ++u) scs[t][u] = given[t][0];
    } else if (scale_mode == 1) {
      float g = 0.0f;
      for (int64_t u = 0; u < B * nh; ++u) g = amax[u] > g ? amax[u] : g;
      for (int64_t u = 0; u < B * nh; ++u) scs[t][u] = ia_or_scale(g);
    } else {
      for (int64_t u = 0; u < B * nh; ++u) scs[t][u] = ia_or_scale(amax[u]);
    }
    free(amax);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < B * nh; ++u) {
      int64_t b = u / nh;
      int64_t n = seq_lens ? seq_lens[b] : L;
      ia_or_quantize(srcs[t] + u * L * d, n * d, scs[t][u], dsts[t] + u * L * d);
      memset(dsts[t] + u * L * d + n * d, 0, (size_t)((L - n) * d));
    }
  }
  if (status != OR_OK) goto done;
  if (scale_mode != 2) {
    if (qs_out) memcpy(qs_out, sq, sizeof(float) * B * H);
    if (ks_out) memcpy(ks_out, sk, sizeof(float) * B * Hkv);
    if (vs_out) memcpy(vs_out, sv, sizeof(float) * B * Hkv);
  }

  {
    int64_t* cint = (int64_t*)malloc(sizeof(int64_t) * B * H);
    float* oscale = (float*)malloc(sizeof(float) * B * H);
    for (int64_t u = 0; u < B * H; ++u) {
      int64_t b = u / H, h = u % H, ku = b * Hkv + h / group;
      cint[u] = ia_or_c_int(c, d, sq[u], sk[ku]);          /* softmax.py:110-121 */
      volatile double os = (double)sv[ku] / (double)p_scale; /* pipeline.py:250 */
      oscale[u] = (float)os;
    }
    if (cint_out) memcpy(cint_out, cint, sizeof(int64_t) * B * H);

    /* ---- per-row QK^T -> IndexSoftmax -> PV -> rescale ---- */
    const int64_t nrows = B * H * L;
#pragma omp parallel
    {
      int32_t* logit = (int32_t*)malloc(sizeof(int32_t) * L);
      uint8_t* prob = (uint8_t*)malloc((size_t)L);
      uint8_t* mrow = (uint8_t*)malloc((size_t)L);
      int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * d);
#pragma omp for schedule(dynamic, 4)
      for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = r % L, u = r / L, b = u / H, h = u % H;
        if (i % row_stride) continue;
        const int64_t ku = b * Hkv + h / group;
        const int64_t n = seq_lens ? seq_lens[b] : L;
        float* orow = out + (u * L + i) * d;
        if (i >= n) {                       /* padding query row -> +0.0 */
          for (int64_t x = 0; x < d; ++x) orow[x] = 0.0f;
          continue;
        }
        const int64_t ncols = causal ? (i + 1 < n ? i + 1 : n) : n;
        const int8_t* qr = qh + (u * L + i) * d;
        const int8_t* kb = kh + ku * L * d;
        const int8_t* vb = vh + ku * L * d;
        for (int64_t j = 0; j < ncols; ++j) {          /* gemm.py:88-106 */
          const int8_t* kr = kb + j * d;
          int32_t s = 0;
          for (int64_t t = 0; t < d; ++t) s += (int32_t)qr[t] * (int32_t)kr[t];
          logit[j] = s;
        }
        const uint8_t* mp = NULL;
        if (mask) {
          for (int64_t j = 0; j < ncols; ++j) mrow[j] = mask[i * L + j];
          mp = mrow;
        }
        /* Columns >= ncols are masked (causal / padding): they take idx = last,
         * add lut[last] = 0 to S and get P = 0 (softmax.py:187-188), so the row
         * restricted to [0, ncols) is the reference's masked row. */
        int64_t ci = cint[u];
        uint32_t s = or_softmax_row(logit, mp, ncols, ci, lut, nlut,
                                    (uint32_t)(2 * p_scale), prob);
        for (int64_t x = 0; x < d; ++x) acc[x] = 0;
        if (s) {
          for (int64_t j = 0; j < ncols; ++j) {        /* gemm.py:109-133 */
            int32_t p = prob[j];
            if (!p) continue;
            const int8_t* vr = vb + j * d;
            for (int64_t x = 0; x < d; ++x) acc[x] += p * (int32_t)vr[x];
          }
        }
        const float os = oscale[u];
        for (int64_t x = 0; x < d; ++x) orow[x] = (float)acc[x] * os;  /* :250-252 */
      }
      free(logit); free(prob); free(mrow); free(acc);
    }
    free(cint); free(oscale);
  }
done:
  free(qh); free(kh); free(vh); free(sq); free(sk); free(sv);
  return status;
}
