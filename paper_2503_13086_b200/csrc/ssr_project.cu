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
// log-scale in float64.  Rows are stored in field-row order, so a block's 128
// field rows own one contiguous range of inst_rows, staged through shared
// memory with coalesced loads.  The merged colour gradient is handed to
// k_chain_sh in the first three floats of the Gaussian's own first row.
constexpr int CHAIN_ROWS = 128;
constexpr int CHAIN_STAGE_FLOATS = 9 * 1024;
constexpr uint32_t MERGE_BIG = 32;  // rows above which a Gaussian is merged warp-cooperatively

// Rows of Gaussians touching more than MERGE_BIG tiles (large splats, up to
// thousands of tiles) are summed by a whole warp -- coalesced strided loads,
// fixed-order tree reduction -- and written back into the Gaussian's first
// row, so the chain's per-thread merge stays bounded.  One warp per 32 rows.
__global__ void __launch_bounds__(256) k_merge_big(int64_t n, const uint32_t* __restrict__ tiles,
                                                   const uint32_t* __restrict__ roff, float* __restrict__ rows) {
  const int64_t g0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(int64_t)31;
  const int lane = threadIdx.x & 31;
  if (g0 >= n) return;
  const int64_t gi = g0 + lane;
  const uint32_t mine = gi < n ? tiles[gi] : 0u;
  unsigned big = __ballot_sync(0xffffffffu, mine > MERGE_BIG);
  while (big) {
    const int l = __ffs(big) - 1;
    big &= big - 1;
    const uint32_t nt = __shfl_sync(0xffffffffu, mine, l);
    float* rw = rows + (int64_t)roff[g0 + l] * 9;
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t j = lane; j < nt; j += 32)
#pragma unroll
      for (int c = 0; c < 9; c++) acc[c] += (double)rw[(int64_t)j * 9 + c];
#pragma unroll
    for (int c = 0; c < 9; c++)
      for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    __syncwarp();
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 9; c++) rw[c] = (float)acc[c];
    __syncwarp();
  }
}
// Adam of optim.py:40-47 for one element (FieldOptimizer's fp32 restatement).
struct AdamClass {
  float lr, ib1, ib2;
};
struct AdamArgs {
  AdamClass c[6];  // pos, rot, scale, opacity, sh dc, sh rest
  float* m;
  float* v;
};
__device__ __forceinline__ float adam_apply(float p, float g, float& m, float& v, const AdamClass& c) {
  m = __fmaf_rn(0.9f, m, 0.1f * g);
  v = __fmaf_rn(0.999f, v, 0.001f * g * g);
  return p - __fdividef(c.lr * (m * c.ib1), sqrtf(v * c.ib2) + 1e-15f);
}

// FUSED = false: write FieldGrads (ssr_chain).  FUSED = true (ssr_chain_adam):
// apply Adam to rotations / log-scales / logits in place and park the
// geometric position gradient in floats 3..5 of the row scratch.
template <bool FUSED>
__global__ void __launch_bounds__(CHAIN_ROWS) k_chain_geo(Cam cam, int64_t n, int K, int tiles_x, int tiles_y,
                                                          const float* __restrict__ pos, float* __restrict__ rot,
                                                          float* __restrict__ ls, float* __restrict__ logit_p,
                                                          const uint32_t* __restrict__ tiles,
                                                          const uint32_t* __restrict__ roff, float* __restrict__ rows,
                                                          float* __restrict__ grads, int accumulate,
                                                          float* __restrict__ stats, AdamArgs adam) {
  __shared__ __align__(16) float s_rows[CHAIN_STAGE_FLOATS + 4];
  __shared__ uint64_t mbar;
  const int64_t i0 = (int64_t)blockIdx.x * CHAIN_ROWS;
  const int rows_here = (int)min((int64_t)CHAIN_ROWS, n - i0);
  const int64_t i = i0 + threadIdx.x;
  const bool mine = threadIdx.x < rows_here;
  const uint32_t r_begin = roff[i0];
  const uint32_t r_end = roff[i0 + rows_here - 1] + tiles[i0 + rows_here - 1];
  // the block's rows are one contiguous range: one 16-byte aligned TMA bulk
  // copy when it fits (inst_rows has >= 16 B slack), else direct reads
  const int64_t n_floats = (int64_t)(r_end - r_begin) * 9;
  const int64_t b0 = (int64_t)r_begin * 36, a0 = b0 & ~(int64_t)15;
  const int pad = (int)((b0 - a0) >> 2);
  const int64_t bytes = ((b0 + n_floats * 4 - a0) + 15) & ~(int64_t)15;
  const bool staged = n_floats > 0 && bytes <= (int64_t)sizeof(s_rows);
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (staged) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&mbar, (uint32_t)bytes);
      bulk_g2s(s_rows, reinterpret_cast<const char*>(rows) + a0, (uint32_t)bytes, &mbar);
    }
    mbar_wait(&mbar, 0);
  }
  const uint32_t nt = mine ? tiles[i] : 0u;
  // bincount merge (backward.py:110-118): ascending tile order; Gaussians with
  // more than MERGE_BIG rows were reduced into their first row by k_merge_big
  double pr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (mine && nt > 0) {
    const float* rw = staged ? s_rows + pad + (int64_t)(roff[i] - r_begin) * 9 : rows + (int64_t)roff[i] * 9;
    const uint32_t nr = nt > MERGE_BIG ? 1u : nt;
    for (uint32_t j = 0; j < nr; j++)
#pragma unroll
      for (int c = 0; c < 9; c++) pr[c] += (double)rw[j * 9 + c];
  }
  if (!mine) return;
  const int S = 11 + 3 * K;
  const int64_t ns = row_stride(n);
  float* g_pos = grads;
  float* g_rot = grads + 3 * ns;
  float* g_ls = grads + 7 * ns;
  float* g_logit = grads + 10 * ns;
  float* g_screen = grads + (int64_t)S * ns;
  float* g_vis = grads + (int64_t)(S + 1) * ns;
  if (FUSED && nt == 0) {  // invisible: the reference still steps every row with a zero gradient
    for (int j = 0; j < 4; j++) {
      const int64_t e = 3 * ns + i * 4 + j;
      rot[i * 4 + j] = adam_apply(rot[i * 4 + j], 0.f, adam.m[e], adam.v[e], adam.c[1]);
    }
    for (int j = 0; j < 3; j++) {
      const int64_t e = 7 * ns + i * 3 + j;
      ls[i * 3 + j] = adam_apply(ls[i * 3 + j], 0.f, adam.m[e], adam.v[e], adam.c[2]);
    }
    logit_p[i] = adam_apply(logit_p[i], 0.f, adam.m[10 * ns + i], adam.v[10 * ns + i], adam.c[3]);
    return;
  }
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
  float* dst = rows + (int64_t)roff[i] * 9;
  dst[0] = (float)pr[0];
  dst[1] = (float)pr[1];
  dst[2] = (float)pr[2];

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
  if (FUSED) {
    for (int j = 0; j < 4; j++) {
      const int64_t e = 3 * ns + i * 4 + j;
      rot[i * 4 + j] = adam_apply(rot[i * 4 + j], (float)((dqn[j] - rad * P.qn[j]) / P.qnorm), adam.m[e], adam.v[e],
                                  adam.c[1]);
    }
    for (int j = 0; j < 3; j++) {
      const int64_t e = 7 * ns + i * 3 + j;
      ls[i * 3 + j] = adam_apply(ls[i * 3 + j], (float)dls[j], adam.m[e], adam.v[e], adam.c[2]);
    }
    logit_p[i] = adam_apply(logit_p[i], (float)pr[3], adam.m[10 * ns + i], adam.v[10 * ns + i], adam.c[3]);
    dst[3] = (float)dpos[0];
    dst[4] = (float)dpos[1];
    dst[5] = (float)dpos[2];
  } else if (accumulate) {
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
// Templated on the degree so the basis lives in registers; the direction
// gradient sum_k v_k dY_k/ddir (v_k = sum_c dcol_c coeff_ck) is written out
// term by term (sh.py:68-111) instead of materialising dY/ddir.
constexpr int CHAIN_SH_ROWS = 128;

template <int DEG>
__device__ __forceinline__ void sh_dir_grad(const double* v, double x, double y, double z, double* g) {
  const double C1 = 0.4886025119029199;
  g[0] = g[1] = g[2] = 0.0;
  if (DEG >= 1) {
    g[1] += v[1] * (-C1);
    g[2] += v[2] * C1;
    g[0] += v[3] * (-C1);
  }
  if (DEG >= 2) {
    const double C20 = 1.0925484305920792, C21 = -1.0925484305920792, C22 = 0.31539156525252005,
                 C23 = -1.0925484305920792, C24 = 0.5462742152960396;
    g[0] += v[4] * (C20 * y) + v[6] * (C22 * (-2.0 * x)) + v[7] * (C23 * z) + v[8] * (C24 * (2.0 * x));
    g[1] += v[4] * (C20 * x) + v[5] * (C21 * z) + v[6] * (C22 * (-2.0 * y)) + v[8] * (C24 * (-2.0 * y));
    g[2] += v[5] * (C21 * y) + v[6] * (C22 * (4.0 * z)) + v[7] * (C23 * x);
  }
  if (DEG >= 3) {
    const double C30 = -0.5900435899266435, C31 = 2.890611442640554, C32 = -0.4570457994644658,
                 C33 = 0.3731763325901154, C34 = -0.4570457994644658, C35 = 1.445305721320277,
                 C36 = -0.5900435899266435;
    const double xx = x * x, yy = y * y, zz = z * z;
    g[0] += v[9] * (C30 * 6.0 * x * y) + v[10] * (C31 * y * z) + v[11] * (C32 * (-2.0 * x * y)) +
            v[12] * (C33 * (-6.0 * x * z)) + v[13] * (C34 * (4.0 * zz - 3.0 * xx - yy)) +
            v[14] * (C35 * (2.0 * x * z)) + v[15] * (C36 * (3.0 * xx - 3.0 * yy));
    g[1] += v[9] * (C30 * (3.0 * xx - 3.0 * yy)) + v[10] * (C31 * x * z) + v[11] * (C32 * (4.0 * zz - xx - 3.0 * yy)) +
            v[12] * (C33 * (-6.0 * y * z)) + v[13] * (C34 * (-2.0 * x * y)) + v[14] * (C35 * (-2.0 * y * z)) +
            v[15] * (C36 * (-6.0 * x * y));
    g[2] += v[10] * (C31 * x * y) + v[11] * (C32 * (8.0 * y * z)) + v[12] * (C33 * (6.0 * zz - 3.0 * xx - 3.0 * yy)) +
            v[13] * (C34 * (8.0 * x * z)) + v[14] * (C35 * (xx - yy));
  }
}

// rows per block: 128, or 64 when the Adam moments are staged too (static smem <= 48 KB)
template <bool FUSED>
struct ShRows {
  static constexpr int value = FUSED ? 64 : CHAIN_SH_ROWS;
};

template <int DEG, bool FUSED>
__global__ void __launch_bounds__(ShRows<FUSED>::value) k_chain_sh(Cam cam, int64_t n, float* __restrict__ pos,
                                                            float* __restrict__ sh,
                                                            const uint32_t* __restrict__ tiles,
                                                            const uint32_t* __restrict__ roff,
                                                            const float* __restrict__ rows,
                                                            float* __restrict__ grads, int accumulate, AdamArgs adam) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int W = 3 * K;
  constexpr int ROWS = ShRows<FUSED>::value;
  constexpr int NBUF = FUSED ? 3 : 1;  // coefficients (+ Adam m, v rows when fused)
  __shared__ __align__(16) float s_buf[NBUF][ROWS * W];
  __shared__ uint64_t mbar;
  float* s_sh = s_buf[0];
  const int64_t i0 = (int64_t)blockIdx.x * ROWS;
  const int rows_here = (int)min((int64_t)ROWS, n - i0);
  const int64_t base = i0 * W;
  const int tot = rows_here * W;
  const int64_t ns = row_stride(n);
  float* gsrc[3] = {sh + base, FUSED ? adam.m + 11 * ns + base : nullptr, FUSED ? adam.v + 11 * ns + base : nullptr};
  // TMA bulk loads of the block's coefficient rows (and their moments)
  bool bulk = ((tot * 4) & 15) == 0;
  for (int b = 0; b < NBUF; b++) bulk = bulk && (reinterpret_cast<uintptr_t>(gsrc[b]) & 15) == 0;
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&mbar, (uint32_t)(tot * 4 * NBUF));
      for (int b = 0; b < NBUF; b++) bulk_g2s(s_buf[b], gsrc[b], (uint32_t)(tot * 4), &mbar);
    }
    mbar_wait(&mbar, 0);
  } else {
    for (int b = 0; b < NBUF; b++)
      for (int e = threadIdx.x; e < tot; e += blockDim.x) s_buf[b][e] = gsrc[b][e];
    __syncthreads();
  }
  const int64_t i = i0 + threadIdx.x;
  float* my = s_sh + threadIdx.x * W;
  if (threadIdx.x < rows_here) {
    double dpos_sh[3] = {0.0, 0.0, 0.0};
    double dcol[3] = {0.0, 0.0, 0.0};
    double basis[16];
    const bool vis = tiles[i] != 0;
    const float* rw = rows + (vis ? (int64_t)roff[i] * 9 : 0);
    if (vis) {
      // sh.py:114-132 in float64 (same op order as the preprocess: identical clamp masks)
      double off[3];
      for (int j = 0; j < 3; j++) off[j] = (double)pos[i * 3 + j] - cam.center[j];
      const double r = sqrt(off[0] * off[0] + off[1] * off[1] + off[2] * off[2]);
      const double rs = r > 1e-12 ? r : 1e-12;
      const double dir[3] = {off[0] / rs, off[1] / rs, off[2] / rs};
      sh_basis64(DEG, dir, basis);
#pragma unroll
      for (int c = 0; c < 3; c++) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < K; k++) acc += (double)my[c * K + k] * basis[k];
        const double raw = acc + 0.5;
        dcol[c] = (raw < 0.0 || raw > 1.0) ? 0.0 : (double)rw[c];
      }
      double v[16];
#pragma unroll
      for (int k = 0; k < K; k++)
        v[k] = dcol[0] * (double)my[k] + dcol[1] * (double)my[K + k] + dcol[2] * (double)my[2 * K + k];
      double ddir[3];
      sh_dir_grad<DEG>(v, dir[0], dir[1], dir[2], ddir);
      const double radial = ddir[0] * dir[0] + ddir[1] * dir[1] + ddir[2] * dir[2];
#pragma unroll
      for (int d = 0; d < 3; d++) dpos_sh[d] = (ddir[d] - radial * dir[d]) / rs;
    } else {
#pragma unroll
      for (int k = 0; k < K; k++) basis[k] = 0.0;
    }
    if (FUSED) {
      // positions: geometric part from the geometry kernel + view-direction part
      for (int d = 0; d < 3; d++) {
        const float g = vis ? (float)((double)rw[3 + d] + dpos_sh[d]) : 0.f;
        const int64_t e = i * 3 + d;
        pos[e] = adam_apply(pos[e], g, adam.m[e], adam.v[e], adam.c[0]);
      }
      float* mm = s_buf[FUSED ? 1 : 0] + threadIdx.x * W;
      float* vv = s_buf[FUSED ? 2 : 0] + threadIdx.x * W;
#pragma unroll
      for (int c = 0; c < 3; c++)
#pragma unroll
        for (int k = 0; k < K; k++) {
          const int e = c * K + k;
          my[e] = adam_apply(my[e], (float)(dcol[c] * basis[k]), mm[e], vv[e], adam.c[k == 0 ? 4 : 5]);
        }
    } else if (!vis) {
#pragma unroll
      for (int e = 0; e < W; e++) my[e] = 0.f;
    } else {
      float* g_pos = grads + i * 3;
#pragma unroll
      for (int d = 0; d < 3; d++) g_pos[d] += (float)dpos_sh[d];
#pragma unroll
      for (int c = 0; c < 3; c++)
#pragma unroll
        for (int k = 0; k < K; k++) my[c * K + k] = (float)(dcol[c] * basis[k]);
    }
  }
  __syncthreads();
  float* gdst[3] = {FUSED ? sh + base : grads + 11 * ns + base, FUSED ? adam.m + 11 * ns + base : nullptr,
                    FUSED ? adam.v + 11 * ns + base : nullptr};
  if (!FUSED && accumulate) {
    for (int e = threadIdx.x; e < tot; e += blockDim.x) gdst[0][e] += s_sh[e];
    return;
  }
  bool bulk_out = bulk;
  for (int b = 0; b < NBUF; b++) bulk_out = bulk_out && (reinterpret_cast<uintptr_t>(gdst[b]) & 15) == 0;
  if (bulk_out) {
    if (threadIdx.x == 0)
      for (int b = 0; b < NBUF; b++) bulk_s2g(gdst[b], s_buf[b], (uint32_t)(tot * 4));
  } else {
    for (int b = 0; b < NBUF; b++)
      for (int e = threadIdx.x; e < tot; e += blockDim.x) gdst[b][e] = s_buf[b][e];
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

template <bool FUSED>
static int launch_chain(const ssr_camera* cam, int64_t n, int32_t sh_degree, float* positions, float* rotations,
                        float* log_scales, float* logits, float* sh, ssr_splats splats, float* rows, float* grads,
                        int32_t accumulate, float* stats, const AdamArgs& adam, cudaStream_t st) {
  int tx, ty;
  tile_dims(cam, &tx, &ty);
  const Cam c = to_cam(*cam);
  const int K = (sh_degree + 1) * (sh_degree + 1);
  k_merge_big<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, splats.tiles, splats.row_offset, rows);
  SSR_TRY(check_launch("k_merge_big"));
  const unsigned blocks = (unsigned)((n + CHAIN_ROWS - 1) / CHAIN_ROWS);
  k_chain_geo<FUSED><<<blocks, CHAIN_ROWS, 0, st>>>(c, n, K, tx, ty, positions, rotations, log_scales, logits,
                                                    splats.tiles, splats.row_offset, rows, grads, accumulate, stats,
                                                    adam);
  SSR_TRY(check_launch("k_chain_geo"));
  constexpr int SR = ShRows<FUSED>::value;
  const unsigned sblocks = (unsigned)((n + SR - 1) / SR);
#define SSR_SH(D)                                                                                                \
  k_chain_sh<D, FUSED><<<sblocks, SR, 0, st>>>(c, n, positions, sh, splats.tiles, splats.row_offset, \
                                                          rows, grads, accumulate, adam)
  switch (sh_degree) {
    case 0: SSR_SH(0); break;
    case 1: SSR_SH(1); break;
    case 2: SSR_SH(2); break;
    default: SSR_SH(3); break;
  }
#undef SSR_SH
  return check_launch("k_chain_sh");
}

extern "C" int ssr_chain(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                         const float* rotations, const float* log_scales, const float* sh, ssr_splats splats,
                         const float* inst_rows, float* grads, int32_t accumulate, float* stats, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3 || !grads) {
    set_error("ssr_chain: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  AdamArgs none{};
  // inst_rows is scratch from here on: the geometry pass parks each Gaussian's
  // merged colour gradient in its own first row for the SH pass
  return launch_chain<false>(cam, n, sh_degree, const_cast<float*>(positions), const_cast<float*>(rotations),
                             const_cast<float*>(log_scales), nullptr, const_cast<float*>(sh), splats,
                             const_cast<float*>(inst_rows), grads, accumulate, stats, none, (cudaStream_t)stream);
}

extern "C" int ssr_chain_adam(const ssr_camera* cam, int64_t n, int32_t sh_degree, float* params, float* m, float* v,
                              ssr_splats splats, float* inst_rows, float* stats, const double* lr, double lr_sh_rest,
                              const double* bc1, const double* bc2, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3 || !params || !m || !v || !lr || !bc1 || !bc2) {
    set_error("ssr_chain_adam: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  AdamArgs adam;
  for (int c = 0; c < 5; c++) {
    adam.c[c].lr = (float)lr[c];
    adam.c[c].ib1 = (float)(1.0 / bc1[c]);
    adam.c[c].ib2 = (float)(1.0 / bc2[c]);
  }
  adam.c[5] = adam.c[4];
  adam.c[5].lr = (float)lr_sh_rest;
  adam.m = m;
  adam.v = v;
  const int64_t ns = row_stride(n);
  return launch_chain<true>(cam, n, sh_degree, params, params + 3 * ns, params + 7 * ns, params + 10 * ns,
                            params + 11 * ns, splats, inst_rows, nullptr, 0, stats, adam, (cudaStream_t)stream);
}
