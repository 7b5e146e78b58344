// Stage 5: fused dense Adam (optim.py:29-47,113-130) and densify/prune
// bookkeeping with moment remap (field.py:303-375, optim.py:49-54,101-111).
//
// The field lives in one flat float32 buffer per quantity, class-major:
//   [positions 3N | rotations 4N | log_scales 3N | opacity_logits N | sh 3KN]
// so Adam is a single vectorised pass over params, grads, m and v.
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "ssr_common.cuh"

namespace ssr {

struct AdamConsts {
  float lr[6];  // pos, rot, scale, opacity, sh dc, sh rest
  float bc1[6], bc2[6];
};

template <int K>
__device__ __forceinline__ int adam_class(int64_t idx, int64_t n) {
  if (idx < 3 * n) return 0;
  if (idx < 7 * n) return 1;
  if (idx < 10 * n) return 2;
  if (idx < 11 * n) return 3;
  return ((uint64_t)(idx - 11 * n) % (uint64_t)K) == 0 ? 4 : 5;  // K is a compile-time constant
}

__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, float lr, float bc1, float bc2) {
  m = __fmaf_rn(0.9f, m, 0.1f * g);
  v = __fmaf_rn(0.999f, v, 0.001f * g * g);
  const float mh = m / bc1, vh = v / bc2;
  p -= lr * mh / (sqrtf(vh) + 1e-15f);
}

template <int K>
__global__ void __launch_bounds__(256) k_adam4(int64_t n, int64_t total4, float4* __restrict__ p,
                                               const float4* __restrict__ g, float4* __restrict__ m,
                                               float4* __restrict__ v, AdamConsts c) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total4; q += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = p[q], gg = g[q], mm = m[q], vv = v[q];
    const int64_t i0 = q * 4;
    int cl;
    cl = adam_class<K>(i0, n);
    adam_one(pp.x, gg.x, mm.x, vv.x, c.lr[cl], c.bc1[cl], c.bc2[cl]);
    cl = adam_class<K>(i0 + 1, n);
    adam_one(pp.y, gg.y, mm.y, vv.y, c.lr[cl], c.bc1[cl], c.bc2[cl]);
    cl = adam_class<K>(i0 + 2, n);
    adam_one(pp.z, gg.z, mm.z, vv.z, c.lr[cl], c.bc1[cl], c.bc2[cl]);
    cl = adam_class<K>(i0 + 3, n);
    adam_one(pp.w, gg.w, mm.w, vv.w, c.lr[cl], c.bc1[cl], c.bc2[cl]);
    p[q] = pp;
    m[q] = mm;
    v[q] = vv;
  }
}

template <int K>
__global__ void k_adam1(int64_t n, int64_t start, int64_t total, float* p, const float* g, float* m, float* v,
                        AdamConsts c) {
  const int64_t i = start + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int cl = adam_class<K>(i, n);
  float pp = p[i], mm = m[i], vv = v[i];
  adam_one(pp, g[i], mm, vv, c.lr[cl], c.bc1[cl], c.bc2[cl]);
  p[i] = pp;
  m[i] = mm;
  v[i] = vv;
}

template <int K>
static int launch_adam(int64_t n, float* params, const float* grads, float* m, float* v, const AdamConsts& c,
                       cudaStream_t st) {
  const int64_t total = (int64_t)(11 + 3 * K) * n;
  const bool aligned = ((((uintptr_t)params) | ((uintptr_t)grads) | ((uintptr_t)m) | ((uintptr_t)v)) & 15) == 0;
  int64_t done = 0;
  if (aligned) {
    const int64_t total4 = total / 4;
    if (total4 > 0) {
      int64_t blocks = (total4 + 255) / 256;
      if (blocks > 148 * 8) blocks = 148 * 8;
      k_adam4<K><<<(unsigned)blocks, 256, 0, st>>>(n, total4, (float4*)params, (const float4*)grads, (float4*)m,
                                                   (float4*)v, c);
      SSR_TRY(check_launch("k_adam4"));
    }
    done = total4 * 4;
  }
  if (done < total) {
    const int64_t rem = total - done;
    k_adam1<K><<<(unsigned)((rem + 255) / 256), 256, 0, st>>>(n, done, total, params, grads, m, v, c);
    SSR_TRY(check_launch("k_adam1"));
  }
  return SSR_OK;
}

// field.py:321-327 masks.  flags: bit0 keep, bit1 clone, bit2 split.
__global__ void k_densify_masks(int64_t n, int K, const float* __restrict__ params, const float* __restrict__ stats,
                                double grad_thr, double big_thr, double prune_opa, uint8_t* __restrict__ flags,
                                int32_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* ls = params + 7 * n + i * 3;
  double ms = exp((double)ls[0]);
  ms = fmax(ms, exp((double)ls[1]));
  ms = fmax(ms, exp((double)ls[2]));
  const double logit = (double)params[10 * n + i];
  const bool hot = (double)stats[i] > grad_thr;
  const bool prune = (1.0 / (1.0 + exp(-logit))) < prune_opa;
  const bool big = ms > big_thr;
  const bool clone = hot && !big && !prune;
  const bool split = hot && big && !prune;
  const bool keep = !(split || prune);
  flags[i] = (uint8_t)((keep ? 1 : 0) | (clone ? 2 : 0) | (split ? 4 : 0));
  if (clone) atomicAdd(&counts[0], 1);
  if (split) atomicAdd(&counts[1], 1);
  if (prune) atomicAdd(&counts[2], 1);
}

struct FlagBit {
  int bit;
  __host__ __device__ uint32_t operator()(uint8_t f) const { return (f >> bit) & 1u; }
};

// field.py:329-372 + optim.py:49-54: kept rows, then clones, then split pairs.
__global__ void k_densify_apply(int64_t n, int64_t n_new, int K, const float* __restrict__ src, const float* m,
                                const float* v, const uint8_t* __restrict__ flags,
                                const uint32_t* __restrict__ keep_off, const uint32_t* __restrict__ clone_off,
                                const uint32_t* __restrict__ split_off, const double* __restrict__ eps, double log_shrink, float* __restrict__ dst,
                                float* new_m, float* new_v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t f = flags[i];
  const uint8_t fl = flags[n - 1];
  const uint32_t n_keep = keep_off[n - 1] + (fl & 1);
  const uint32_t n_clone = clone_off[n - 1] + ((fl >> 1) & 1);
  const int width[5] = {3, 4, 3, 1, 3 * K};
  const int64_t so[5] = {0, 3 * n, 7 * n, 10 * n, 11 * n};
  const int64_t dof[5] = {0, 3 * n_new, 7 * n_new, 10 * n_new, 11 * n_new};
  if (f & 1) {
    const int64_t d = keep_off[i];
    for (int c = 0; c < 5; c++)
      for (int j = 0; j < width[c]; j++) {
        const int64_t s = so[c] + i * width[c] + j, t = dof[c] + d * width[c] + j;
        dst[t] = src[s];
        if (new_m) new_m[t] = m[s];
        if (new_v) new_v[t] = v[s];
      }
  }
  if (f & 2) {
    const int64_t d = (int64_t)n_keep + clone_off[i];
    for (int c = 0; c < 5; c++)
      for (int j = 0; j < width[c]; j++) {
        const int64_t t = dof[c] + d * width[c] + j;
        dst[t] = src[so[c] + i * width[c] + j];
        if (new_m) new_m[t] = 0.f;
        if (new_v) new_v[t] = 0.f;
      }
  }
  if (f & 4) {
    const int64_t j2 = split_off[i];
    const float* q = src + so[1] + i * 4;
    double qq[4] = {(double)q[0], (double)q[1], (double)q[2], (double)q[3]};
    double R[9], qn[4], nrm;
    quat_rotmat64(qq, R, qn, &nrm);
    double sc[3];
    for (int a = 0; a < 3; a++) sc[a] = exp((double)src[so[2] + i * 3 + a]);
    for (int c2 = 0; c2 < 2; c2++) {
      const int64_t d = (int64_t)n_keep + n_clone + 2 * j2 + c2;
      const double* e = eps + (2 * j2 + c2) * 3;
      for (int a = 0; a < 3; a++) {
        double off = 0.0;
        for (int b = 0; b < 3; b++) off += R[a * 3 + b] * (sc[b] * e[b]);
        dst[dof[0] + d * 3 + a] = (float)((double)src[so[0] + i * 3 + a] + off);
        dst[dof[2] + d * 3 + a] = (float)((double)src[so[2] + i * 3 + a] - log_shrink);
      }
      for (int a = 0; a < 4; a++) dst[dof[1] + d * 4 + a] = q[a];
      dst[dof[3] + d] = src[so[3] + i];
      for (int a = 0; a < 3 * K; a++) dst[dof[4] + d * 3 * K + a] = src[so[4] + i * 3 * K + a];
      if (new_m || new_v)
        for (int c = 0; c < 5; c++)
          for (int a = 0; a < width[c]; a++) {
            const int64_t t = dof[c] + d * width[c] + a;
            if (new_m) new_m[t] = 0.f;
            if (new_v) new_v[t] = 0.f;
          }
    }
  }
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_adam(int64_t n, int32_t sh_degree, float* params, const float* grads, float* m, float* v,
                        const double* lr, double lr_sh_rest, const double* bc1, const double* bc2, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || !lr || !bc1 || !bc2) {
    set_error("ssr_adam: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  AdamConsts c;
  for (int i = 0; i < 5; i++) {
    c.lr[i] = (float)lr[i];
    c.bc1[i] = (float)bc1[i];
    c.bc2[i] = (float)bc2[i];
  }
  c.lr[5] = (float)lr_sh_rest;
  c.bc1[5] = (float)bc1[4];
  c.bc2[5] = (float)bc2[4];
  cudaStream_t st = (cudaStream_t)stream;
  switch (K) {
    case 1: return launch_adam<1>(n, params, grads, m, v, c, st);
    case 4: return launch_adam<4>(n, params, grads, m, v, c, st);
    case 9: return launch_adam<9>(n, params, grads, m, v, c, st);
    default: return launch_adam<16>(n, params, grads, m, v, c, st);
  }
}

extern "C" int ssr_densify_masks(int64_t n, const float* params, int32_t sh_degree, const float* stats,
                                 double grad_threshold, double big_threshold, double prune_opacity, uint8_t* flags,
                                 int32_t* counts, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3) {
    set_error("ssr_densify_masks: invalid argument");
    return SSR_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SSR_TRY(check_cuda(cudaMemsetAsync(counts, 0, 3 * sizeof(int32_t), st), "densify counts"));
  if (n == 0) return SSR_OK;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  k_densify_masks<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, K, params, stats, grad_threshold, big_threshold,
                                                               prune_opacity, flags, counts);
  return check_launch("k_densify_masks");
}

static size_t densify_scan_bytes(int64_t n) {
  size_t b = 0;
  cub::TransformInputIterator<uint32_t, FlagBit, const uint8_t*> it((const uint8_t*)nullptr, FlagBit{0});
  cub::DeviceScan::ExclusiveSum((void*)nullptr, b, it, (uint32_t*)nullptr, (int)(n > 0 ? n : 1));
  return b;
}

extern "C" int ssr_densify_workspace(int64_t n, int64_t* bytes) {
  *bytes = 3 * align_up(4 * (n > 0 ? n : 1), 256) + align_up((int64_t)densify_scan_bytes(n), 256) + 256;
  return SSR_OK;
}

extern "C" int ssr_densify_apply(int64_t n, int64_t n_new, int32_t sh_degree, const float* params, const float* m,
                                 const float* v, const uint8_t* flags, const double* eps, double log_shrink,
                                 float* new_params, float* new_m, float* new_v, void* workspace,
                                 int64_t workspace_bytes, void* stream) {
  if (n < 0 || n_new < 0 || sh_degree < 0 || sh_degree > 3 || n > INT32_MAX) {
    set_error("ssr_densify_apply: invalid argument");
    return SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_densify_workspace(n, &need);
  if (workspace_bytes < need) {
    set_error("ssr_densify_apply: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  char* w = (char*)workspace;
  uint32_t* offs[3];
  for (int b = 0; b < 3; b++) {
    offs[b] = (uint32_t*)w;
    w += align_up(4 * n, 256);
  }
  size_t tb = densify_scan_bytes(n);
  for (int b = 0; b < 3; b++) {
    cub::TransformInputIterator<uint32_t, FlagBit, const uint8_t*> it(flags, FlagBit{b});
    size_t tb2 = tb;
    SSR_TRY(check_cuda(cub::DeviceScan::ExclusiveSum((void*)w, tb2, it, offs[b], (int)n, st), "densify scan"));
  }
  k_densify_apply<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, n_new, K, params, m, v, flags, offs[0], offs[1],
                                                               offs[2], eps, log_shrink, new_params,
                                                               new_m, new_v);
  return check_launch("k_densify_apply");
}
