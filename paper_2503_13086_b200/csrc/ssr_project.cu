// Stage 1 (per-Gaussian preprocess), float64.
// Compiled with -fmad=false so every multiply/add rounds like the reference's
// numpy float64 expressions (rasterize/projection.py:69-162, sh.py:114-132):
// culling, tile rects, depth order and clamp masks come out identical.
#include "ssr_common.cuh"

namespace ssr {

// projection.py:69-162 + sh.py:114-132 -- one thread per field row.  Templated
// on the SH degree so the basis stays in registers.
//
// STAGED: the CTA's position, rotation, log-scale and SH rows arrive by TMA
// bulk copies issued at entry (~30 KB per CTA at SH3), so the fp64 math reads
// shared memory instead of waiting on per-thread loads; used when the class
// arrays are 16-byte aligned (the flat field layout always is), for every
// full CTA (the last, partial one reads global memory directly).
constexpr int PRE_ROWS = 128;

// SH rows are not staged: only the rows that survive culling read theirs
// (12 float4 loads at degree 3, sh_color64), so culled rows (~40% at config 2)
// cost no SH traffic.  SSR_PRE_STAGE_SH restores staging every row's SH.
#ifdef SSR_PRE_STAGE_SH
constexpr bool PRE_STAGE_SH = true;
#else
constexpr bool PRE_STAGE_SH = false;
#endif

template <int DEG>
__host__ __device__ constexpr int pre_stage_floats() {
  return PRE_ROWS * (3 + 4 + 3 + (PRE_STAGE_SH ? 3 * (DEG + 1) * (DEG + 1) : 0));
}

template <int DEG, bool STAGED>
__global__ void __launch_bounds__(PRE_ROWS, 7) k_preprocess(Cam cam, int64_t n, int tiles_x, int tiles_y,
                                                         const float* __restrict__ pos, const float* __restrict__ rot,
                                                         const float* __restrict__ ls,
                                                         const float* __restrict__ logit,
                                                         const float* __restrict__ sh, ssr_splats o) {
  griddep_wait();
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int W = 3 * K;
  extern __shared__ __align__(16) float s_pre[];  // rot 4R | pos 3R | log-scale 3R | sh W R
  __shared__ uint64_t mbar;
  const int64_t i0 = (int64_t)blockIdx.x * PRE_ROWS;
  const int64_t i = i0 + threadIdx.x;
  const bool staged = STAGED && i0 + PRE_ROWS <= n;
  if (staged) {
    if (threadIdx.x == 0) {
      mbar_init(&mbar, 1);
      constexpr uint32_t bytes = (uint32_t)pre_stage_floats<DEG>() * 4;
      mbar_expect_tx(&mbar, bytes);
      bulk_g2s(s_pre, rot + i0 * 4, PRE_ROWS * 16, &mbar);
      bulk_g2s(s_pre + 4 * PRE_ROWS, pos + i0 * 3, PRE_ROWS * 12, &mbar);
      bulk_g2s(s_pre + 7 * PRE_ROWS, ls + i0 * 3, PRE_ROWS * 12, &mbar);
      if (PRE_STAGE_SH) bulk_g2s(s_pre + 10 * PRE_ROWS, sh + i0 * W, PRE_ROWS * W * 4, &mbar);
    }
    __syncthreads();
    mbar_wait(&mbar, 0);
  }
  if (i >= n) return;
  const int r = threadIdx.x;
  const float* prow = staged ? s_pre + 4 * PRE_ROWS + r * 3 : pos + i * 3;
  const float* qrow = staged ? s_pre + r * 4 : rot + i * 4;
  const float* lrow = staged ? s_pre + 7 * PRE_ROWS + r * 3 : ls + i * 3;
  const float* shrow = staged && PRE_STAGE_SH ? s_pre + 10 * PRE_ROWS + r * W : sh + i * W;
  if (!staged && PRE_STAGE_SH) {
    // start the row's SH coefficients on their way to L2 while the fp64
    // projection runs (culled rows waste 3K floats of L2 fill, visible rows
    // then read them at L2 latency)
    const char* shp = reinterpret_cast<const char*>(shrow);
    for (int off = 0; off < W * 4; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(shp + off));
  }
  Proj64 P;
  if (!project64(cam, prow, qrow, lrow, tiles_x, tiles_y, P)) {
    o.tiles[i] = 0;
    return;
  }
  double dir[3], rs, basis[16], col[3];
  bool lo[3], hi[3];
  sh_color64(cam, DEG, prow, shrow, dir, &rs, basis, col, lo, hi);
  const double opa = 1.0 / (1.0 + exp(-(double)logit[i]));
  reinterpret_cast<double2*>(o.mean)[i] = make_double2(P.u, P.v);
  // near-singular conics (1 - |b|/sqrt(ac) < 1e-3) are the only ones whose fp32
  // power can round across 0; they carry a negative fp32 opacity so the
  // forward can test the power > 0 guard band with a warp-uniform branch
  const bool fragile = 1.0 - fabs(P.qb) / sqrt(P.qa * P.qc) < 1e-3;
  reinterpret_cast<float4*>(o.conic_opa)[i] =
      make_float4((float)P.qa, (float)P.qb, (float)P.qc, fragile ? -(float)opa : (float)opa);
  // .w: bit c set when channel c is not clamped (sh.py:128-131), decided here in
  // float64 so the fp32 chain sees the reference's clamp masks exactly
  const int pass = (!lo[0] && !hi[0] ? 1 : 0) | (!lo[1] && !hi[1] ? 2 : 0) | (!lo[2] && !hi[2] ? 4 : 0);
  reinterpret_cast<float4*>(o.color)[i] = make_float4((float)col[0], (float)col[1], (float)col[2], __int_as_float(pass));
  double2* c64 = reinterpret_cast<double2*>(o.conic_opa64) + 2 * i;
  c64[0] = make_double2(P.qa, P.qb);
  c64[1] = make_double2(P.qc, opa);
  double2* k64 = reinterpret_cast<double2*>(o.color64) + 2 * i;
  k64[0] = make_double2(col[0], col[1]);
  k64[1] = make_double2(col[2], 0.0);
  o.depth[i] = P.cp[2];
  reinterpret_cast<int4*>(o.rect)[i] = make_int4(P.rect[0], P.rect[1], P.rect[2], P.rect[3]);
  o.tiles[i] = (uint32_t)((P.rect[2] - P.rect[0]) * (P.rect[3] - P.rect[1]));
}

// ProjectedSplats retained intermediates (projection.py:40-48), on demand.
__global__ void k_project_aux(Cam cam, int64_t n, int deg, int tiles_x, int tiles_y, const float* pos,
                              const float* rot, const float* ls, const float* sh, const uint32_t* tiles,
                              double* cam_points, double* clamp_mul, double* cov2d, double* cov3d_cam,
                              double* sh_dirs, double* sh_radii, uint8_t* sh_lo, uint8_t* sh_hi,
                              double* radii) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || tiles[i] == 0) return;
  const int K = (deg + 1) * (deg + 1);
  Proj64 P;
  project64(cam, pos + i * 3, rot + i * 4, ls + i * 3, tiles_x, tiles_y, P);
  double dir[3], rs, basis[16], col[3];
  bool lo[3], hi[3];
  sh_color64(cam, deg, pos + i * 3, sh + i * 3 * K, dir, &rs, basis, col, lo, hi);
  for (int j = 0; j < 3; j++) {
    cam_points[i * 3 + j] = P.cp[j];
    sh_dirs[i * 3 + j] = dir[j];
    sh_lo[i * 3 + j] = lo[j];
    sh_hi[i * 3 + j] = hi[j];
  }
  clamp_mul[i * 2] = P.mulx;
  clamp_mul[i * 2 + 1] = P.muly;
  cov2d[i * 3] = P.A;
  cov2d[i * 3 + 1] = P.B;
  cov2d[i * 3 + 2] = P.C;
  for (int j = 0; j < 9; j++) cov3d_cam[i * 9 + j] = P.cc[j];
  sh_radii[i] = rs;
  radii[i] = P.radius;
}

}  // namespace ssr

using namespace ssr;

static inline void tile_dims(const ssr_camera* cam, int* tx, int* ty) {
  *tx = (cam->width + TILE - 1) / TILE;
  *ty = (cam->height + TILE - 1) / TILE;
}

extern "C" int ssr_preprocess(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                              const float* rotations, const float* log_scales, const float* opacity_logits,
                              const float* sh, ssr_splats splats, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3) {
    set_error("ssr_preprocess: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  int tx, ty;
  tile_dims(cam, &tx, &ty);
  const int64_t blocks = (n + PRE_ROWS - 1) / PRE_ROWS;
  const Cam c = to_cam(*cam);
  cudaStream_t st = (cudaStream_t)stream;
  auto al16 = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
  const bool staged = al16(positions) && al16(rotations) && al16(log_scales) && al16(sh);
#define SSR_PRE(D)                                                                                                 \
  do {                                                                                                             \
    if (staged) {                                                                                                  \
      constexpr size_t sm = (size_t)pre_stage_floats<D>() * sizeof(float);                                        \
      static DeviceOnce attr;                                                                                    \
      if (!attr.done()) {                                                                                                 \
        SSR_TRY(check_cuda(                                                                                        \
            cudaFuncSetAttribute(k_preprocess<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),     \
            "k_preprocess smem"));                                                                                 \
        attr.set();                                                                                               \
      }                                                                                                            \
      SSR_TRY(launch_pdl("k_preprocess", k_preprocess<D, true>, dim3((unsigned)blocks), dim3(PRE_ROWS), sm, st, c, \
                         n, tx, ty, positions, rotations, log_scales, opacity_logits, sh, splats));              \
    } else {                                                                                                       \
      SSR_TRY(launch_pdl("k_preprocess", k_preprocess<D, false>, dim3((unsigned)blocks), dim3(PRE_ROWS), 0, st, c, \
                         n, tx, ty, positions, rotations, log_scales, opacity_logits, sh, splats));              \
    }                                                                                                              \
  } while (0)
  switch (sh_degree) {
    case 0: SSR_PRE(0); break;
    case 1: SSR_PRE(1); break;
    case 2: SSR_PRE(2); break;
    default: SSR_PRE(3); break;
  }
#undef SSR_PRE
  return check_launch("k_preprocess");
}

extern "C" int ssr_project_aux(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                               const float* rotations, const float* log_scales, const float* sh,
                               const uint32_t* tiles, double* cam_points, double* clamp_mul, double* cov2d,
                               double* cov3d_cam, double* sh_dirs, double* sh_radii, uint8_t* sh_lo,
                               uint8_t* sh_hi, double* radii, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3) {
    set_error("ssr_project_aux: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  int tx, ty;
  tile_dims(cam, &tx, &ty);
  k_project_aux<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      to_cam(*cam), n, sh_degree, tx, ty, positions, rotations, log_scales, sh, tiles, cam_points, clamp_mul,
      cov2d, cov3d_cam, sh_dirs, sh_radii, sh_lo, sh_hi, radii);
  return check_launch("k_project_aux");
}

