// Stage 1 (per-Gaussian preprocess) and the stage-4 gradient chain, float64.
// Compiled with -fmad=false so every multiply/add rounds like the reference's
// numpy float64 expressions (rasterize/projection.py:69-162,
// rasterize/backward.py:132-259, sh.py:114-152).
#include "ssr_common.cuh"

namespace ssr {

// projection.py:69-162 + sh.py:114-132 -- one thread per field row.
__global__ void __launch_bounds__(256) k_preprocess(Cam cam, int64_t n, int deg, int tiles_x, int tiles_y,
                                                    const float* __restrict__ pos, const float* __restrict__ rot,
                                                    const float* __restrict__ ls, const float* __restrict__ logit,
                                                    const float* __restrict__ sh, ssr_splats o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int K = (deg + 1) * (deg + 1);
  Proj64 P;
  if (!project64(cam, pos + i * 3, rot + i * 4, ls + i * 3, tiles_x, tiles_y, P)) {
    o.tiles[i] = 0;
    return;
  }
  double dir[3], rs, basis[16], col[3];
  bool lo[3], hi[3];
  sh_color64(cam, deg, pos + i * 3, sh + i * 3 * K, dir, &rs, basis, col, lo, hi);
  const double opa = 1.0 / (1.0 + exp(-(double)logit[i]));
  reinterpret_cast<double2*>(o.mean)[i] = make_double2(P.u, P.v);
  // near-singular conics (1 - |b|/sqrt(ac) < 1e-3) are the only ones whose fp32
  // power can round across 0; they carry a negative fp32 opacity so the
  // forward can test the power > 0 guard band with a warp-uniform branch
  const bool fragile = 1.0 - fabs(P.qb) / sqrt(P.qa * P.qc) < 1e-3;
  reinterpret_cast<float4*>(o.conic_opa)[i] =
      make_float4((float)P.qa, (float)P.qb, (float)P.qc, fragile ? -(float)opa : (float)opa);
  reinterpret_cast<float4*>(o.color)[i] = make_float4((float)col[0], (float)col[1], (float)col[2], 0.f);
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

// backward.py:110-206 (geometry half) -- one thread per field row: merge the
// row's instance rows in splat-major (= ascending tile, bincount) order, then
// chain d_mu / d_conic through the projection to position, rotation and
// log-scale in float64.  The merged colour gradient is handed to k_chain_sh
// in the first three floats of the Gaussian's own first instance row.
__global__ void __launch_bounds__(128) k_chain_geo(Cam cam, int64_t n, int K, int tiles_x, int tiles_y,
                                                   const float* __restrict__ pos, const float* __restrict__ rot,
                                                   const float* __restrict__ ls,
                                                   const uint32_t* __restrict__ tiles,
                                                   const uint32_t* __restrict__ offset, float* __restrict__ rows,
                                                   float* __restrict__ grads, int accumulate,
                                                   float* __restrict__ stats) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int S = 11 + 3 * K;
  float* g_pos = grads;
  float* g_rot = grads + 3 * n;
  float* g_ls = grads + 7 * n;
  float* g_logit = grads + 10 * n;
  float* g_screen = grads + (int64_t)S * n;
  float* g_vis = grads + (int64_t)(S + 1) * n;
  const uint32_t nt = tiles[i];
  if (nt == 0) {
    if (!accumulate) {
      for (int j = 0; j < 3; j++) g_pos[i * 3 + j] = 0.f;
      for (int j = 0; j < 4; j++) g_rot[i * 4 + j] = 0.f;
      for (int j = 0; j < 3; j++) g_ls[i * 3 + j] = 0.f;
      g_logit[i] = 0.f;
      g_screen[i] = 0.f;
      g_vis[i] = 0.f;
    }
    return;
  }
  // bincount merge (backward.py:110-118): ascending tile order
  double pr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  float* rw = rows + (int64_t)offset[i] * 9;
  for (uint32_t j = 0; j < nt; j++)
    for (int c = 0; c < 9; c++) pr[c] += (double)rw[j * 9 + c];
  rw[0] = (float)pr[0];
  rw[1] = (float)pr[1];
  rw[2] = (float)pr[2];

  Proj64 P;
  project64(cam, pos + i * 3, rot + i * 4, ls + i * 3, tiles_x, tiles_y, P);
  // conic -> V2: g_v2 = -Q G Q  (backward.py:502-515)
  const double q[4] = {P.qa, P.qb, P.qb, P.qc};
  const double gq[4] = {pr[6], 0.5 * pr[7], 0.5 * pr[7], pr[8]};
  double gv2[4];
  for (int a = 0; a < 2; a++)
    for (int l = 0; l < 2; l++) {
      double acc = 0.0;
      for (int j = 0; j < 2; j++)
        for (int k = 0; k < 2; k++) acc += q[a * 2 + j] * gq[j * 2 + k] * q[k * 2 + l];
      gv2[a * 2 + l] = -acc;
    }
  const double x = P.cp[0], y = P.cp[1], z = P.cp[2];
  const double fx = cam.fx, fy = cam.fy;
  const double J[6] = {fx / z, 0.0, -fx * P.txc / z, 0.0, fy / z, -fy * P.tyc / z};
  double gJ[6], gv3[9], gw[9];
  for (int a = 0; a < 2; a++)
    for (int l = 0; l < 3; l++) {
      double acc = 0.0;
      for (int j = 0; j < 2; j++)
        for (int k = 0; k < 3; k++) acc += gv2[a * 2 + j] * J[j * 3 + k] * P.cc[k * 3 + l];
      gJ[a * 3 + l] = 2.0 * acc;
    }
  for (int a = 0; a < 3; a++)
    for (int l = 0; l < 3; l++) {
      double acc = 0.0;
      for (int j = 0; j < 2; j++)
        for (int k = 0; k < 2; k++) acc += J[j * 3 + a] * gv2[j * 2 + k] * J[k * 3 + l];
      gv3[a * 3 + l] = acc;
    }
  const double* R = cam.R;
  for (int a = 0; a < 3; a++)
    for (int l = 0; l < 3; l++) {
      double acc = 0.0;
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++) acc += R[j * 3 + a] * gv3[j * 3 + k] * R[k * 3 + l];
      gw[a * 3 + l] = acc;
    }
  // backward.py:537-553
  double dcam[3] = {0.0, 0.0, 0.0};
  const double z2 = z * z;
  dcam[0] += gJ[2] * (-fx * P.mulx / z2);
  dcam[1] += gJ[5] * (-fy * P.muly / z2);
  dcam[2] += gJ[0] * (-fx / z2);
  dcam[2] += gJ[4] * (-fy / z2);
  dcam[2] += gJ[2] * fx * (P.mulx * x / z + P.txc) / z2;
  dcam[2] += gJ[5] * fy * (P.muly * y / z + P.tyc) / z2;
  dcam[0] += pr[4] * fx / z;
  dcam[1] += pr[5] * fy / z;
  dcam[2] += -pr[4] * fx * x / z2 - pr[5] * fy * y / z2;
  double dpos[3];
  for (int d = 0; d < 3; d++) dpos[d] = dcam[0] * R[0 * 3 + d] + dcam[1] * R[1 * 3 + d] + dcam[2] * R[2 * 3 + d];

  // _cov_to_rotation_scale (backward.py:562-612)
  double m[9], gs[9], dm[9], drot[9], dls[3];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) m[a * 3 + b] = P.rot[a * 3 + b] * P.sc[b];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) gs[a * 3 + b] = gw[a * 3 + b] + gw[b * 3 + a];
  for (int a = 0; a < 3; a++)
    for (int k = 0; k < 3; k++) {
      double acc = 0.0;
      for (int j = 0; j < 3; j++) acc += gs[a * 3 + j] * m[j * 3 + k];
      dm[a * 3 + k] = acc;
      drot[a * 3 + k] = acc * P.sc[k];
    }
  for (int j = 0; j < 3; j++) {
    double acc = 0.0;
    for (int a = 0; a < 3; a++) acc += dm[a * 3 + j] * P.rot[a * 3 + j];
    dls[j] = acc * P.sc[j];
  }
  const double w_ = P.qn[0], x_ = P.qn[1], y_ = P.qn[2], z_ = P.qn[3];
  const double drw[9] = {0, -z_, y_, z_, 0, -x_, -y_, x_, 0};
  const double drx[9] = {0, y_, z_, y_, -2 * x_, -w_, z_, w_, -2 * x_};
  const double dry[9] = {-2 * y_, x_, w_, x_, 0, z_, -w_, z_, -2 * y_};
  const double drz[9] = {-2 * z_, -w_, x_, w_, -2 * z_, y_, x_, y_, 0};
  double dqn[4] = {0, 0, 0, 0};
  for (int e = 0; e < 9; e++) {
    dqn[0] += drot[e] * (2.0 * drw[e]);
    dqn[1] += drot[e] * (2.0 * drx[e]);
    dqn[2] += drot[e] * (2.0 * dry[e]);
    dqn[3] += drot[e] * (2.0 * drz[e]);
  }
  const double rad = dqn[0] * P.qn[0] + dqn[1] * P.qn[1] + dqn[2] * P.qn[2] + dqn[3] * P.qn[3];
  const double screen =
      sqrt(pr[4] * pr[4] + pr[5] * pr[5]) * (0.5 * (double)(cam.width > cam.height ? cam.width : cam.height));
  if (accumulate) {
    for (int j = 0; j < 3; j++) g_pos[i * 3 + j] += (float)dpos[j];
    for (int j = 0; j < 4; j++) g_rot[i * 4 + j] += (float)((dqn[j] - rad * P.qn[j]) / P.qnorm);
    for (int j = 0; j < 3; j++) g_ls[i * 3 + j] += (float)dls[j];
    g_logit[i] += (float)pr[3];
    g_screen[i] += (float)screen;
    g_vis[i] += 1.f;
  } else {
    for (int j = 0; j < 3; j++) g_pos[i * 3 + j] = (float)dpos[j];
    for (int j = 0; j < 4; j++) g_rot[i * 4 + j] = (float)((dqn[j] - rad * P.qn[j]) / P.qnorm);
    for (int j = 0; j < 3; j++) g_ls[i * 3 + j] = (float)dls[j];
    g_logit[i] = (float)pr[3];
    g_screen[i] = (float)screen;
    g_vis[i] = 1.f;
  }
  if (stats) {
    stats[i] += (float)screen;
    stats[n + i] += 1.f;
  }
}

// sh.py:135-152 (+ backward.py:200) -- SH coefficients and the view-direction
// path into positions.  128 rows per block; the block's coefficient rows and
// their gradients move through shared memory so global traffic is coalesced.
constexpr int CHAIN_SH_ROWS = 128;
__global__ void __launch_bounds__(CHAIN_SH_ROWS) k_chain_sh(Cam cam, int64_t n, int deg,
                                                            const float* __restrict__ pos,
                                                            const float* __restrict__ sh,
                                                            const uint32_t* __restrict__ tiles,
                                                            const uint32_t* __restrict__ offset,
                                                            const float* __restrict__ rows,
                                                            float* __restrict__ grads, int accumulate) {
  extern __shared__ float s_sh[];  // [CHAIN_SH_ROWS * 3K] coefficients, then gradients in place
  const int K = (deg + 1) * (deg + 1);
  const int W = 3 * K;
  const int64_t i0 = (int64_t)blockIdx.x * CHAIN_SH_ROWS;
  const int rows_here = (int)min((int64_t)CHAIN_SH_ROWS, n - i0);
  const int64_t base = i0 * W;
  const int tot = rows_here * W;
  for (int e = threadIdx.x; e < tot; e += blockDim.x) s_sh[e] = sh[base + e];
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  float* my = s_sh + threadIdx.x * W;
  if (threadIdx.x < rows_here) {
    const uint32_t nt = tiles[i];
    if (nt == 0) {
      for (int e = 0; e < W; e++) my[e] = 0.f;
    } else {
      const float* rw = rows + (int64_t)offset[i] * 9;
      double dir[3], rs, basis[16], col[3];
      bool lo[3], hi[3];
      sh_color64(cam, deg, pos + i * 3, my, dir, &rs, basis, col, lo, hi);
      double dcol[3];
      for (int c = 0; c < 3; c++) dcol[c] = (lo[c] || hi[c]) ? 0.0 : (double)rw[c];
      // d_dir = sum_c sum_k dcol_c coeff_ck dY_k/ddir  (sh.py:147-148)
      double gb[48];
      sh_basis_grad64(deg, dir, gb);
      double ddir[3] = {0.0, 0.0, 0.0};
      for (int k = 0; k < K; k++) {
        const double vk = dcol[0] * (double)my[k] + dcol[1] * (double)my[K + k] + dcol[2] * (double)my[2 * K + k];
        ddir[0] += vk * gb[k * 3 + 0];
        ddir[1] += vk * gb[k * 3 + 1];
        ddir[2] += vk * gb[k * 3 + 2];
      }
      const double radial = ddir[0] * dir[0] + ddir[1] * dir[1] + ddir[2] * dir[2];
      float* g_pos = grads + i * 3;
      for (int d = 0; d < 3; d++) g_pos[d] += (float)((ddir[d] - radial * dir[d]) / rs);
      for (int c = 0; c < 3; c++)
        for (int k = 0; k < K; k++) my[c * K + k] = (float)(dcol[c] * basis[k]);
    }
  }
  __syncthreads();
  float* g_sh = grads + 11 * n + base;
  if (accumulate) {
    for (int e = threadIdx.x; e < tot; e += blockDim.x) g_sh[e] += s_sh[e];
  } else {
    for (int e = threadIdx.x; e < tot; e += blockDim.x) g_sh[e] = s_sh[e];
  }
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
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  k_preprocess<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      to_cam(*cam), n, sh_degree, tx, ty, positions, rotations, log_scales, opacity_logits, sh, splats);
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

extern "C" int ssr_chain(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                         const float* rotations, const float* log_scales, const float* sh, ssr_splats splats,
                         const float* inst_rows, float* grads, int32_t accumulate, float* stats, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3 || !grads) {
    set_error("ssr_chain: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  int tx, ty;
  tile_dims(cam, &tx, &ty);
  cudaStream_t st = (cudaStream_t)stream;
  const Cam c = to_cam(*cam);
  const int K = (sh_degree + 1) * (sh_degree + 1);
  // inst_rows is scratch from here on: the geometry pass parks each Gaussian's
  // merged colour gradient in its own first row for the SH pass
  float* rows = const_cast<float*>(inst_rows);
  k_chain_geo<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(c, n, K, tx, ty, positions, rotations, log_scales,
                                                           splats.tiles, splats.offset, rows, grads, accumulate,
                                                           stats);
  SSR_TRY(check_launch("k_chain_geo"));
  const size_t smem = (size_t)CHAIN_SH_ROWS * 3 * K * sizeof(float);
  k_chain_sh<<<(unsigned)((n + CHAIN_SH_ROWS - 1) / CHAIN_SH_ROWS), CHAIN_SH_ROWS, smem, st>>>(
      c, n, sh_degree, positions, sh, splats.tiles, splats.offset, rows, grads, accumulate);
  return check_launch("k_chain_sh");
}
