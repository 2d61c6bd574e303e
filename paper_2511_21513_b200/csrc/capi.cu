// capi.cu -- C ABI plumbing: status strings, error detail, device checks,
// per-head parameter kernels and mask packing.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "params.cuh"

namespace ia {

static thread_local char g_err[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return IA_OK;
}

int dev_knob(const char* name, int dflt) {
#if IA_PROFILE
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

int num_sms() {
  static thread_local int cached_dev = -1, cached = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev != cached_dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    cached_dev = dev;
  }
  return cached;
}

__global__ void head_params_kernel(const float* __restrict__ qs, const float* __restrict__ ks,
                                   const float* __restrict__ vs, int q_per_head, int kv_per_head,
                                   int64_t B, int64_t H, int64_t Hkv, int64_t d, double c,
                                   int nlut, int p_scale, ia_head_params* __restrict__ out) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= B * H) return;
  const int64_t b = u / H, h = u % H;
  const int64_t ku = b * Hkv + h / (H / Hkv);
  const float sq = q_per_head ? qs[u] : qs[0];
  const float sk = kv_per_head ? ks[ku] : ks[0];
  const float sv = kv_per_head ? vs[ku] : vs[0];
  ia_head_params hp;
  make_head_params(c, d, nlut, p_scale, sq, sk, sv, &hp);
  out[u] = hp;
}

__global__ void group_params_kernel(const float* __restrict__ qs, const float* __restrict__ ks,
                                    int64_t B, int64_t H, int64_t Hkv, int64_t G, int64_t d,
                                    double c, int nlut, ia_group_params* __restrict__ out) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= B * H * G) return;
  const int64_t bh = u / G, g = u - bh * G;
  const int64_t b = bh / H, h = bh - b * H;
  const int64_t ku = b * Hkv + h / (H / Hkv);
  ia_head_params hp;
  fill_head_params(compute_c_int(c, d, qs[bh], ks[ku * G + g]), 2 * d * 127 * 127, nlut, &hp);
  ia_group_params gp;
  if (hp.c_eff > INT32_MAX) {  // c_int > 2k * dbound: idx = 0 for every reachable delta
    gp.c_eff = INT32_MAX;
    gp.magic = 0u;
    gp.shift = 0;
    gp.use32 = 1;
  } else {
    gp.c_eff = (int32_t)hp.c_eff;
    gp.magic = hp.magic;
    gp.shift = hp.shift;
    gp.use32 = hp.use32;
    // float form of the index map (params.cuh): the fused kernel then needs only c_eff and
    // the ratio, whose bits travel in `magic`
    if (float_idx_ok(hp.c_eff, (int64_t)nlut - 1)) {
      gp.magic = __float_as_uint(float_idx_ratio(hp.c_eff, (int64_t)nlut - 1));
      gp.use32 = hp.use32 | 2;
    }
  }
  out[u] = gp;
}

__global__ void mask_pack_kernel(const uint8_t* __restrict__ mask, int64_t L, int64_t W,
                                 uint32_t* __restrict__ bits) {
  const int64_t n = L * W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t r = i / W, w = i - r * W;
    const uint8_t* m = mask + r * L + w * 32;
    uint32_t v = 0;
    const int64_t lim = L - w * 32 < 32 ? L - w * 32 : 32;
    for (int64_t e = 0; e < lim; ++e) v |= (m[e] ? 1u : 0u) << e;
    bits[i] = v;
  }
}

}  // namespace ia

using namespace ia;

extern "C" int ia_abi_version(void) { return IA_ABI_VERSION; }

extern "C" const char* ia_status_string(int s) {
  switch (s) {
    case IA_OK: return "ok";
    case IA_ERR_INVALID_ARGUMENT: return "invalid argument";
    case IA_ERR_SEQ_LEN: return "sequence length exceeds 65536";
    case IA_ERR_HEAD_DIM: return "unsupported head dimension";
    case IA_ERR_NONFINITE: return "input contains non-finite elements";
    case IA_ERR_CUDA: return "CUDA error";
    case IA_ERR_NO_DEVICE: return "no sm_100 CUDA device";
    case IA_ERR_LUT: return "lookup table endpoints must be 255 and 0";
    default: return "unknown status";
  }
}

extern "C" const char* ia_last_error(void) { return ia::g_err; }

extern "C" int ia_device_check(int dev) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n <= dev)
    return fail(IA_ERR_NO_DEVICE, "no CUDA device %d (%s)", dev,
                e == cudaSuccess ? "count too small" : cudaGetErrorString(e));
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess)
    return fail(IA_ERR_NO_DEVICE, "cudaGetDeviceProperties failed");
  if (p.major != 10 || p.minor != 0)
    return fail(IA_ERR_NO_DEVICE, "device %d is sm_%d%d; this build targets sm_100a", dev,
                p.major, p.minor);
  return IA_OK;
}

extern "C" int ia_head_params_host(double c, int64_t d, int nlut, int p_scale, float s_q,
                                   float s_k, float s_v, ia_head_params* out) {
  if (!out || d < 1 || nlut < 4 || nlut > 256 || (p_scale != 255 && p_scale != 127))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_head_params_host: bad arguments");
  make_head_params(c, d, nlut, p_scale, s_q, s_k, s_v, out);
  return IA_OK;
}

extern "C" int ia_softmax_params_host(int64_t c_int, int64_t delta_bound, int nlut,
                                      ia_head_params* out) {
  if (!out || c_int < 1 || delta_bound < 0 || nlut < 4 || nlut > 256)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_softmax_params_host: bad arguments");
  fill_head_params(c_int < kCIntCap ? c_int : kCIntCap, delta_bound, nlut, out);
  out->out_scale = 0.0f;
  out->s_q = out->s_k = out->s_v = 0.0f;
  return IA_OK;
}

extern "C" int ia_head_params_dev(const float* q_scales, const float* k_scales,
                                  const float* v_scales, int q_per_head, int kv_per_head,
                                  int64_t B, int64_t H, int64_t Hkv, int64_t d, double c,
                                  int nlut, int p_scale, ia_head_params* out, void* stream) {
  if (!q_scales || !k_scales || !v_scales || !out || B < 1 || H < 1 || Hkv < 1 || H % Hkv ||
      d < 1 || nlut < 4 || nlut > 256 || (p_scale != 255 && p_scale != 127))
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_head_params_dev: bad arguments");
  const int64_t n = B * H;
  head_params_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      q_scales, k_scales, v_scales, q_per_head, kv_per_head, B, H, Hkv, d, c, nlut, p_scale,
      out);
  return check_launch("head_params_kernel");
}

extern "C" int ia_group_params_dev(const float* q_scales, const float* k_scales, int64_t B,
                                   int64_t H, int64_t Hkv, int64_t n_groups, int64_t d, double c,
                                   int nlut, ia_group_params* out, void* stream) {
  if (!q_scales || !k_scales || !out || B < 1 || H < 1 || Hkv < 1 || H % Hkv || n_groups < 1 ||
      d < 1 || nlut < 4 || nlut > 256)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_group_params_dev: bad arguments");
  const int64_t n = B * H * n_groups;
  group_params_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      q_scales, k_scales, B, H, Hkv, n_groups, d, c, nlut, out);
  return check_launch("group_params_kernel");
}

extern "C" int ia_mask_pack(const uint8_t* mask, int64_t L, uint32_t* bits, void* stream) {
  if (!mask || !bits || L < 1) return fail(IA_ERR_INVALID_ARGUMENT, "ia_mask_pack");
  const int64_t W = (L + 31) / 32;
  int64_t blocks = (L * W + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  mask_pack_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(mask, L, W, bits);
  return check_launch("mask_pack_kernel");
}

extern "C" int ia_copy_rows_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                                  int64_t width, int64_t height, void* stream) {
  if (!dst || !src || width < 0 || height < 0 || dpitch < width || spitch < width)
    return fail(IA_ERR_INVALID_ARGUMENT, "ia_copy_rows_async: bad arguments");
  if (!width || !height) return IA_OK;
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                    (size_t)height, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "ia_copy_rows_async: %s", cudaGetErrorString(e));
  return IA_OK;
}

extern "C" int ia_zero_async(void* dst, int64_t bytes, void* stream) {
  if (!dst || bytes < 0) return fail(IA_ERR_INVALID_ARGUMENT, "ia_zero_async: bad arguments");
  if (!bytes) return IA_OK;
  cudaError_t e = cudaMemsetAsync(dst, 0, (size_t)bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(IA_ERR_CUDA, "ia_zero_async: %s", cudaGetErrorString(e));
  return IA_OK;
}
