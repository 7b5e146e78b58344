// Shared device code for the sm_100a splat rasterizer.
//
// Two numeric regimes live here:
//  * float64 per-Gaussian math (projection, SH, chain) that restates the
//    reference op-for-op (rasterize/projection.py:69-162, sh.py:36-152) so
//    culling, tile rects, depth order and clamp masks come out identical;
//    TUs using it are compiled with -fmad=false.
//  * float32 per-pair blend math used by the forward and both backward
//    layouts; every rounding step is pinned with __f*_rn intrinsics so the
//    backward replays the forward's discrete decisions bit-for-bit.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "../../include/ssr.h"

namespace ssr {

constexpr int TILE = 16;
constexpr int TILE_PX = TILE * TILE;
constexpr int BUCKET = 32;
constexpr double ZNEAR = 0.2;
constexpr double COV2D_DILATION = 0.3;
constexpr double FRUSTUM_EXPAND = 1.3;
constexpr double ALPHA_MIN = 1.0 / 255.0;
constexpr double ALPHA_CAP = 0.99;
constexpr double T_EPS = 1e-4;
constexpr double SOFT_TAU = 0.01;
constexpr float ALPHA_MIN_F = 1.0f / 255.0f;
constexpr float ALPHA_CAP_F = 0.99f;
constexpr float T_EPS_F = 1e-4f;

// Flat parameter / moment / gradient buffers are class-major with every class
// region padded to a row stride that is a multiple of 4, so each region starts
// 16-byte aligned for any N (float4 and TMA bulk paths stay valid after densify).
__host__ __device__ __forceinline__ int64_t row_stride(int64_t n) { return (n + 3) & ~(int64_t)3; }

void set_error(const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
int check_launch(const char* what);

// "Done once" flag kept per device: kernel attributes and __constant__ data
// belong to a device, so a process that drives several GPUs sets each up.
struct DeviceOnce {
  std::atomic<uint64_t> bits{0};
  static int dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool done() const { return (bits.load(std::memory_order_acquire) >> dev()) & 1u; }
  void set() { bits.fetch_or(1ull << dev(), std::memory_order_acq_rel); }
};

#define SSR_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != SSR_OK) return _rc; \
  } while (0)

struct Cam {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  double center[3];
  int width, height;
};

inline Cam to_cam(const ssr_camera& c) {
  Cam o;
  for (int i = 0; i < 9; i++) o.R[i] = c.R[i];
  for (int i = 0; i < 3; i++) {
    o.t[i] = c.t[i];
    o.center[i] = c.center[i];
  }
  o.fx = c.fx;
  o.fy = c.fy;
  o.cx = c.cx;
  o.cy = c.cy;
  o.width = c.width;
  o.height = c.height;
  return o;
}

// ------------------------------------------------------------------ TMA bulk copies
// 1-D cp.async.bulk global <-> shared with an mbarrier (sm_90+/sm_100a): one
// elected thread moves a contiguous block-sized chunk; addresses and sizes
// must be 16-byte multiples.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

// smem -> global bulk store (generic-proxy smem writes are fenced first).
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(smem_src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// ------------------------------------------------------------------ fp64 SH
// sh.py:36-65
__device__ __forceinline__ void sh_basis64(const int deg, const double d[3], double* out) {
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};
  out[0] = 0.28209479177387814;
  if (deg >= 1) {
    double x = d[0], y = d[1], z = d[2];
    out[1] = -0.4886025119029199 * y;
    out[2] = 0.4886025119029199 * z;
    out[3] = -0.4886025119029199 * x;
    if (deg >= 2) {
      double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
      out[4] = C2[0] * xy;
      out[5] = C2[1] * yz;
      out[6] = C2[2] * (2.0 * zz - xx - yy);
      out[7] = C2[3] * xz;
      out[8] = C2[4] * (xx - yy);
      if (deg >= 3) {
        out[9] = C3[0] * y * (3.0 * xx - yy);
        out[10] = C3[1] * xy * z;
        out[11] = C3[2] * y * (4.0 * zz - xx - yy);
        out[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        out[13] = C3[4] * x * (4.0 * zz - xx - yy);
        out[14] = C3[5] * z * (xx - yy);
        out[15] = C3[6] * x * (xx - 3.0 * yy);
      }
    }
  }
}

// sh.py:68-111 ; g[k*3+d]
__device__ __forceinline__ void sh_basis_grad64(int deg, const double dd[3], double* g) {
  const double C1 = 0.4886025119029199;
  const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                        -1.0925484305920792, 0.5462742152960396};
  const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                        0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                        -0.5900435899266435};
  const int K = (deg + 1) * (deg + 1);
  for (int i = 0; i < K * 3; i++) g[i] = 0.0;
  if (deg < 1) return;
  double x = dd[0], y = dd[1], z = dd[2];
  g[1 * 3 + 1] = -C1;
  g[2 * 3 + 2] = C1;
  g[3 * 3 + 0] = -C1;
  if (deg >= 2) {
    g[4 * 3 + 0] = C2[0] * y;
    g[4 * 3 + 1] = C2[0] * x;
    g[5 * 3 + 1] = C2[1] * z;
    g[5 * 3 + 2] = C2[1] * y;
    g[6 * 3 + 0] = C2[2] * (-2.0 * x);
    g[6 * 3 + 1] = C2[2] * (-2.0 * y);
    g[6 * 3 + 2] = C2[2] * (4.0 * z);
    g[7 * 3 + 0] = C2[3] * z;
    g[7 * 3 + 2] = C2[3] * x;
    g[8 * 3 + 0] = C2[4] * (2.0 * x);
    g[8 * 3 + 1] = C2[4] * (-2.0 * y);
  }
  if (deg >= 3) {
    double xx = x * x, yy = y * y, zz = z * z;
    g[9 * 3 + 0] = C3[0] * 6.0 * x * y;
    g[9 * 3 + 1] = C3[0] * (3.0 * xx - 3.0 * yy);
    g[10 * 3 + 0] = C3[1] * y * z;
    g[10 * 3 + 1] = C3[1] * x * z;
    g[10 * 3 + 2] = C3[1] * x * y;
    g[11 * 3 + 0] = C3[2] * (-2.0 * x * y);
    g[11 * 3 + 1] = C3[2] * (4.0 * zz - xx - 3.0 * yy);
    g[11 * 3 + 2] = C3[2] * (8.0 * y * z);
    g[12 * 3 + 0] = C3[3] * (-6.0 * x * z);
    g[12 * 3 + 1] = C3[3] * (-6.0 * y * z);
    g[12 * 3 + 2] = C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    g[13 * 3 + 0] = C3[4] * (4.0 * zz - 3.0 * xx - yy);
    g[13 * 3 + 1] = C3[4] * (-2.0 * x * y);
    g[13 * 3 + 2] = C3[4] * (8.0 * x * z);
    g[14 * 3 + 0] = C3[5] * (2.0 * x * z);
    g[14 * 3 + 1] = C3[5] * (-2.0 * y * z);
    g[14 * 3 + 2] = C3[5] * (xx - yy);
    g[15 * 3 + 0] = C3[6] * (3.0 * xx - 3.0 * yy);
    g[15 * 3 + 1] = C3[6] * (-6.0 * x * y);
  }
}

// field.py:40-60
__device__ __forceinline__ void quat_rotmat64(const double q[4], double r[9], double qn[4], double* nrm_out) {
  double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
  r[0] = 1 - 2 * (y * y + z * z);
  r[1] = 2 * (x * y - w * z);
  r[2] = 2 * (x * z + w * y);
  r[3] = 2 * (x * y + w * z);
  r[4] = 1 - 2 * (x * x + z * z);
  r[5] = 2 * (y * z - w * x);
  r[6] = 2 * (x * z - w * y);
  r[7] = 2 * (y * z + w * x);
  r[8] = 1 - 2 * (x * x + y * y);
  qn[0] = w;
  qn[1] = x;
  qn[2] = y;
  qn[3] = z;
  *nrm_out = nrm;
}

__device__ __forceinline__ long long trunc_i64(double v) {
  // numpy astype(int64) on x86: truncation toward zero, INT64_MIN when out of range
  if (!(v > -9.2e18 && v < 9.2e18)) return (long long)(-9223372036854775807LL - 1);
  return (long long)v;
}
__device__ __forceinline__ long long clip_ll(long long v, long long lo, long long hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

struct Proj64 {
  double cp[3];     // camera-space point
  double u, v;      // projected mean
  double mulx, muly, txc, tyc;
  double cc[9];     // camera-space covariance
  double A, B, C;   // dilated 2D covariance
  double qa, qb, qc; // conic
  double radius;
  int rect[4];
  double rot[9], qn[4], qnorm, sc[3];
};

// projection.py:76-128 for one Gaussian.  Returns true when the splat is kept.
__device__ __forceinline__ bool project64(const Cam& cam, const float* pos, const float* quat,
                                          const float* ls, int tiles_x, int tiles_y, Proj64& o) {
  const double* R = cam.R;
  double p[3] = {(double)pos[0], (double)pos[1], (double)pos[2]};
  for (int j = 0; j < 3; j++)
    o.cp[j] = p[0] * R[j * 3 + 0] + p[1] * R[j * 3 + 1] + p[2] * R[j * 3 + 2] + cam.t[j];
  if (!(o.cp[2] > ZNEAR)) return false;
  const double x = o.cp[0], y = o.cp[1], z = o.cp[2];
  o.u = cam.fx * x / z + cam.cx;
  o.v = cam.fy * y / z + cam.cy;
  const double limx = FRUSTUM_EXPAND * (cam.width / (2.0 * cam.fx));
  const double limy = FRUSTUM_EXPAND * (cam.height / (2.0 * cam.fy));
  const double tx = x / z, ty = y / z;
  o.mulx = (tx > -limx && tx < limx) ? 1.0 : 0.0;
  o.muly = (ty > -limy && ty < limy) ? 1.0 : 0.0;
  o.txc = tx < -limx ? -limx : (tx > limx ? limx : tx);
  o.tyc = ty < -limy ? -limy : (ty > limy ? limy : ty);
  // field.py:71-75  Sigma = M M^T, M = R(q) diag(exp(s))
  const float4 q4 = *reinterpret_cast<const float4*>(quat);  // rotation rows are 16-byte aligned
  double q[4] = {(double)q4.x, (double)q4.y, (double)q4.z, (double)q4.w};
  quat_rotmat64(q, o.rot, o.qn, &o.qnorm);
  double m[9], cw[9];
  for (int j = 0; j < 3; j++) o.sc[j] = exp((double)ls[j]);
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) m[i * 3 + j] = o.rot[i * 3 + j] * o.sc[j];
  for (int i = 0; i < 3; i++)
    for (int k = 0; k < 3; k++) {
      double acc = 0.0;
      for (int j = 0; j < 3; j++) acc += m[i * 3 + j] * m[k * 3 + j];
      cw[i * 3 + k] = acc;
    }
  // einsum("ij,njk,lk->nil", R, Sigma, R)
  for (int a = 0; a < 3; a++)
    for (int l = 0; l < 3; l++) {
      double acc = 0.0;
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) acc += R[a * 3 + j] * cw[j * 3 + k] * R[l * 3 + k];
      o.cc[a * 3 + l] = acc;
    }
  const double fx_z = cam.fx / z, fy_z = cam.fy / z;
  const double j02 = -cam.fx * o.txc / z, j12 = -cam.fy * o.tyc / z;
  const double c00 = o.cc[0], c01 = o.cc[1], c02 = o.cc[2], c11 = o.cc[4], c12 = o.cc[5], c22 = o.cc[8];
  o.A = fx_z * (fx_z * c00 + j02 * c02) + j02 * (fx_z * c02 + j02 * c22) + COV2D_DILATION;
  o.B = fx_z * (fy_z * c01 + j12 * c02) + j02 * (fy_z * c12 + j12 * c22);
  o.C = fy_z * (fy_z * c11 + j12 * c12) + j12 * (fy_z * c12 + j12 * c22) + COV2D_DILATION;
  const double det = o.A * o.C - o.B * o.B;
  bool ok = det > 0.0;
  const double inv_det = ok ? 1.0 / det : 0.0;
  o.qa = o.C * inv_det;
  o.qb = -o.B * inv_det;
  o.qc = o.A * inv_det;
  const double mid = 0.5 * (o.A + o.C);
  const double mm = mid * mid - det;
  const double lam = mid + sqrt(mm > 0.1 ? mm : 0.1);
  o.radius = ceil(3.0 * sqrt(lam));
  long long tx0 = clip_ll(trunc_i64((o.u - o.radius) / TILE), 0, tiles_x);
  long long ty0 = clip_ll(trunc_i64((o.v - o.radius) / TILE), 0, tiles_y);
  long long tx1 = clip_ll(trunc_i64((o.u + o.radius) / TILE) + 1, 0, tiles_x);
  long long ty1 = clip_ll(trunc_i64((o.v + o.radius) / TILE) + 1, 0, tiles_y);
  long long wx = tx1 - tx0 > 0 ? tx1 - tx0 : 0, wy = ty1 - ty0 > 0 ? ty1 - ty0 : 0;
  ok = ok && (o.radius > 0) && (wx * wy > 0);
  o.rect[0] = (int)tx0;
  o.rect[1] = (int)ty0;
  o.rect[2] = (int)tx1;
  o.rect[3] = (int)ty1;
  return ok;
}

// sh.py:114-132: direction, basis, clamped colour and masks.
__device__ __forceinline__ void sh_color64(const Cam& cam, int deg, const float* pos, const float* shrow,
                                           double dir[3], double* rs, double basis[16], double col[3],
                                           bool lo[3], bool hi[3]) {
  const int K = (deg + 1) * (deg + 1);
  double off[3];
  for (int j = 0; j < 3; j++) off[j] = (double)pos[j] - cam.center[j];
  double r = sqrt(off[0] * off[0] + off[1] * off[1] + off[2] * off[2]);
  *rs = r > 1e-12 ? r : 1e-12;
  for (int j = 0; j < 3; j++) dir[j] = off[j] / *rs;
  sh_basis64(deg, dir, basis);
  // degree 3: the row's 48 coefficients as 12 aligned float4 loads (rows are
  // 192 B, class regions 16-byte aligned), issued together
  float cf[48];
  if (K == 16) {
#pragma unroll
    for (int q = 0; q < 12; q++) {
      const float4 v = reinterpret_cast<const float4*>(shrow)[q];
      cf[4 * q] = v.x;
      cf[4 * q + 1] = v.y;
      cf[4 * q + 2] = v.z;
      cf[4 * q + 3] = v.w;
    }
  }
  for (int c = 0; c < 3; c++) {
    double acc = 0.0;
    for (int k = 0; k < K; k++) acc += (double)(K == 16 ? cf[c * 16 + k] : shrow[c * K + k]) * basis[k];
    double raw = acc + 0.5;
    lo[c] = raw < 0.0;
    hi[c] = raw > 1.0;
    col[c] = raw < 0.0 ? 0.0 : (raw > 1.0 ? 1.0 : raw);
  }
}

// ------------------------------------------------------------------ fp32 pair math
// kernels.py:72-80 in base 2.  The staged conic is pre-scaled so that
//   power2 = a2 dx^2 + b2 dx dy + c2 dy^2 = log2(e) * power,
//   a2 = -0.5 a log2e, b2 = -b log2e, c2 = -0.5 c log2e,
// and alpha = opacity * ex2(power2) is one MUFU.EX2.  Every rounding step is
// pinned (__f*_rn, inline ex2.approx) so the forward and both backward
// kernels compute bit-identical alphas and transmittances.
constexpr float LOG2E_F = 1.4426950408889634f;
// pairs with power < -25 (alpha < 1.4e-11 * opacity): no threshold is within
// reach, the soft term equals S0 to 3e-10 and gradient terms are ~1e-10.
constexpr float FAR_POWER2 = -25.0f * 1.4426950408889634f;

// Tile-relative mean split into an exact integer part and a float fraction:
// dx = (px - mi) - mf, where px - mi is exact, so dx carries only one rounding
// (6e-8 relative) instead of the rounding of a float mean near 32 (2e-6 px).
struct StagedMean {
  float xi, xf, yi, yf;
};

__device__ __forceinline__ StagedMean stage_mean(double mx, double my, int x00, int y00) {
  StagedMean s;
  const double rx = mx - (double)x00, ry = my - (double)y00;
  const double ix = rint(rx), iy = rint(ry);
  s.xi = (float)ix;
  s.xf = (float)(rx - ix);
  s.yi = (float)iy;
  s.yf = (float)(ry - iy);
  return s;
}

__device__ __forceinline__ float pair_d(float fp, float mi, float mf) { return __fsub_rn(__fsub_rn(fp, mi), mf); }

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): two round-to-nearest
// lanes per instruction, each lane bit-identical to __fsub_rn / __fmul_rn /
// __fmaf_rn, so two splats' far tests cost one issue slot per operation.
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

struct StagedConic {
  float a2, b2, c2;
};

__device__ __forceinline__ StagedConic stage_conic(float a, float b, float c) {
  StagedConic s;
  s.a2 = __fmul_rn(-0.5f * LOG2E_F, a);
  s.b2 = __fmul_rn(-LOG2E_F, b);
  s.c2 = __fmul_rn(-0.5f * LOG2E_F, c);
  return s;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Returns power2; qpos = a2 dx^2 + c2 dy^2 (<= 0) is the magnitude reference
// for the guard band of the power > 0 decision.
__device__ __forceinline__ float pair_power2(float dxx, float dxy, float dyy, float a2, float b2, float c2,
                                             float& qpos) {
  qpos = __fmaf_rn(c2, dyy, __fmul_rn(a2, dxx));
  return __fmaf_rn(b2, dxy, qpos);
}

__device__ __forceinline__ float pair_alpha2(float opa, float power2) { return __fmul_rn(opa, ex2_approx(power2)); }

// Soft count of the forward (kernels.py:83) is accumulated as
//   n_small * S0 + sum(y * p(y)) + sum(sigmoid(alpha) for alpha >= 2.5e-3),
// y = alpha / SOFT_TAU, S0 = sigmoid(-ALPHA_MIN / SOFT_TAU) in float64 and p a
// degree-3 minimax fit of (sigmoid(y - ALPHA_MIN/TAU) - S0) / y on [0, 0.25]
// (max abs error of y p(y) 3.8e-9, 8.2e-9 with its fp32 evaluation; the error
// shrinks with y, and a pixel's small-alpha pairs sum to well under the 1e-4
// soft-count tolerance).  Long walks (10^4 slots) would otherwise accumulate
// the fp32 rounding of the same ~0.403 term.
constexpr double SOFT_S0 = 0.4031981879117929;
constexpr float SOFT_Y0 = 0.25f;
// Accumulates y p(y) into acc with one final FMA (acc += y * p(y)).
__device__ __forceinline__ float soft_dev_acc(float y, float acc) {
  float p = -2.6635625e-03f;
  p = __fmaf_rn(p, y, -1.8015249e-02f);
  p = __fmaf_rn(p, y, 2.3311704e-02f);
  p = __fmaf_rn(p, y, 2.4062893e-01f);
  return __fmaf_rn(y, p, acc);
}

__device__ __forceinline__ float soft_sigmoid_accurate(float alpha) {
  // ex2.approx (2^-22 rel) + rcp.approx: ~1e-7 abs on a value in [0.5, 1]
  const float e = ex2_approx(__fmul_rn(__fsub_rn(ALPHA_MIN_F, alpha), 100.0f * LOG2E_F));
  return __fdividef(1.0f, 1.0f + e);
}

__device__ __forceinline__ float soft_sigmoid(float alpha) {
  // 1 / (1 + exp(-(alpha - 1/255) / 0.01))   (kernels.py:83)
  const float e = ex2_approx(__fmul_rn(__fsub_rn(ALPHA_MIN_F, alpha), 100.0f * LOG2E_F));
  return __fdividef(1.0f, 1.0f + e);
}

// Adam of optim.py:40-47 for one float32 element: m, v updated in place,
// returns the new parameter.  sqrt.approx (MUFU, 2^-22 relative) keeps v = 0
// (rows never seen) off the IEEE sqrt's special-case path.  Shared by k_adam
// and the fused chain so both paths round identically.
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float adam_update(float p, float g, float& m, float& v, float lr, float ib1, float ib2) {
  m = __fmaf_rn(0.9f, m, 0.1f * g);
  v = __fmaf_rn(0.999f, v, 0.001f * g * g);
  return p - __fdividef(lr * (m * ib1), sqrt_approx(v * ib2) + 1e-15f);
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels launched with launch_pdl may be scheduled while their stream
// predecessor drains (its launch latency hides behind the predecessor's
// tail); each such kernel calls griddep_wait() before anything else, which
// returns once the predecessor has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Zeroes n 32-bit words (a kernel rather than a memset: it keeps the launch
// chain programmatic).
static __global__ void k_zero_words(uint32_t* p, int64_t n) {
  griddep_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0u;
}

// ------------------------------------------------------------------ instance gradient rows
// inst_rows workspace (ssr.h ssr_rows_floats): a 4-word header whose word 0 is
// the generation of the last ssr_backward, then one 10-word row per instance
// (9 gradient terms + the generation that wrote it).  Only instances some
// pixel walked get a row; a row whose tag is not the current generation is
// zero, so the rows of unwalked slots are never written nor zero-filled.
constexpr int ROWS_HEAD = 4;
constexpr int ROW_WORDS = 10;
__device__ __forceinline__ uint32_t rows_generation(const float* rows) {
  return *reinterpret_cast<const volatile uint32_t*>(rows);
}
// 5 x 8-byte loads (global or shared: every row starts 8-byte aligned)
__device__ __forceinline__ void load_row(const float* r, float* v) {
  const float2* p = reinterpret_cast<const float2*>(r);
#pragma unroll
  for (int i = 0; i < ROW_WORDS / 2; i++) {
    const float2 x = p[i];
    v[2 * i] = x.x;
    v[2 * i + 1] = x.y;
  }
}
__device__ __forceinline__ void store_row(float* rows, size_t r, float v0, float v1, float v2, float v3, float v4,
                                          float v5, float v6, float v7, float v8, uint32_t tag) {
  // scalar stores: packing float2 pairs costs the backward 1% (registers)
  float* p = rows + ROWS_HEAD + r * ROW_WORDS;
  p[0] = v0;
  p[1] = v1;
  p[2] = v2;
  p[3] = v3;
  p[4] = v4;
  p[5] = v5;
  p[6] = v6;
  p[7] = v7;
  p[8] = v8;
  p[9] = __uint_as_float(tag);
}

template <typename... KArgs, typename... Args>
static inline int launch_pdl(const char* what, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return SSR_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return check_cuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), what);
}

// ------------------------------------------------------------------ exclusive scan of uint32
// Two launches, no library code: per-4096-element CTA sums, then each CTA sums
// its predecessors' totals directly (no look-back chain) and scans its own
// elements, 16 consecutive per thread.  Totals are 64-bit (out is uint32).
constexpr int SCAN_THREADS = 256, SCAN_ITEMS = 16, SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

static __global__ void __launch_bounds__(SCAN_THREADS) k_u32_tile_sums(int64_t n, const uint32_t* __restrict__ in,
                                                                     uint64_t* __restrict__ sums) {
  __shared__ uint64_t red[SCAN_THREADS / 32];
  uint64_t v = 0;
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const int64_t r = (int64_t)blockIdx.x * SCAN_TILE + i * SCAN_THREADS + threadIdx.x;
    if (r < n) v += in[r];
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < SCAN_THREADS / 32; w++) t += red[w];
    sums[blockIdx.x] = t;
  }
}

static __global__ void __launch_bounds__(SCAN_THREADS) k_u32_scan(int64_t n, const uint32_t* __restrict__ in,
                                                                const uint64_t* __restrict__ sums,
                                                                uint32_t* __restrict__ out) {
  __shared__ uint64_t s_w[SCAN_THREADS / 32], s_p[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t pre = 0;
  for (int t = threadIdx.x; t < (int)blockIdx.x; t += SCAN_THREADS) pre += sums[t];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    v[i] = base + i < n ? in[base + i] : 0u;
    sum += v[i];
  }
  uint64_t incl = sum;
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 31) s_w[warp] = incl;
  if (lane == 0) s_p[warp] = pre;
  __syncthreads();
  uint64_t wb = 0, p = 0;
  for (int w = 0; w < SCAN_THREADS / 32; w++) {
    if (w < warp) wb += s_w[w];
    p += s_p[w];
  }
  uint64_t run = p + wb + incl - sum;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    if (base + i < n) out[base + i] = (uint32_t)run;
    run += v[i];
  }
}

static inline int64_t scan_u32_workspace(int64_t n) { return 8 * ((n + SCAN_TILE - 1) / SCAN_TILE + 1); }

// exclusive scan in -> out of n elements; ws holds scan_u32_workspace(n) bytes
static inline int scan_u32(const uint32_t* in, uint32_t* out, int64_t n, void* ws, cudaStream_t st) {
  if (n <= 0) return SSR_OK;
  const unsigned ctas = (unsigned)((n + SCAN_TILE - 1) / SCAN_TILE);
  k_u32_tile_sums<<<ctas, SCAN_THREADS, 0, st>>>(n, in, (uint64_t*)ws);
  SSR_TRY(check_launch("k_u32_tile_sums"));
  k_u32_scan<<<ctas, SCAN_THREADS, 0, st>>>(n, in, (const uint64_t*)ws, out);
  return check_launch("k_u32_scan");
}

}  // namespace ssr
