/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the splat rasterizer hot path.
 *
 * A plain-C, float64 restatement of the reference package `splatstream`
 * (the On-the-Fly GS CPU re-statement).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product path (paper_2503_13086_b200) never links or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py
 * imports /root/reference/pkg/src/splatstream in the builder container).
 *
 * Citations are to /root/reference/pkg/src/splatstream/<file>:<line>.
 * Built with -ffp-contract=off so every multiply/add rounds like numpy.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16
#define ZNEAR 0.2
#define COV2D_DILATION 0.3
#define FRUSTUM_EXPAND 1.3
#define ALPHA_MIN (1.0 / 255.0)
#define ALPHA_CAP 0.99
#define T_EPS 1e-4
#define SOFT_TAU 0.01
#define CHUNK 16

typedef struct {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  double center[3];
  int64_t width, height;
} orc_cam;

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* sh.py:36-65 */
static void sh_basis(int deg, const double d[3], double* out) {
  out[0] = SH_C0;
  if (deg >= 1) {
    double x = d[0], y = d[1], z = d[2];
    out[1] = -SH_C1 * y;
    out[2] = SH_C1 * z;
    out[3] = -SH_C1 * x;
    if (deg >= 2) {
      double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
      out[4] = SH_C2[0] * xy;
      out[5] = SH_C2[1] * yz;
      out[6] = SH_C2[2] * (2.0 * zz - xx - yy);
      out[7] = SH_C2[3] * xz;
      out[8] = SH_C2[4] * (xx - yy);
      if (deg >= 3) {
        out[9] = SH_C3[0] * y * (3.0 * xx - yy);
        out[10] = SH_C3[1] * xy * z;
        out[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
        out[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        out[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
        out[14] = SH_C3[5] * z * (xx - yy);
        out[15] = SH_C3[6] * x * (xx - 3.0 * yy);
      }
    }
  }
}

/* sh.py:68-111, g[k*3 + d] */
static void sh_basis_grad(int deg, const double dd[3], double* g) {
  int K = (deg + 1) * (deg + 1);
  for (int i = 0; i < K * 3; i++) g[i] = 0.0;
  if (deg < 1) return;
  double x = dd[0], y = dd[1], z = dd[2];
  g[1 * 3 + 1] = -SH_C1;
  g[2 * 3 + 2] = SH_C1;
  g[3 * 3 + 0] = -SH_C1;
  if (deg >= 2) {
    g[4 * 3 + 0] = SH_C2[0] * y;
    g[4 * 3 + 1] = SH_C2[0] * x;
    g[5 * 3 + 1] = SH_C2[1] * z;
    g[5 * 3 + 2] = SH_C2[1] * y;
    g[6 * 3 + 0] = SH_C2[2] * (-2.0 * x);
    g[6 * 3 + 1] = SH_C2[2] * (-2.0 * y);
    g[6 * 3 + 2] = SH_C2[2] * (4.0 * z);
    g[7 * 3 + 0] = SH_C2[3] * z;
    g[7 * 3 + 2] = SH_C2[3] * x;
    g[8 * 3 + 0] = SH_C2[4] * (2.0 * x);
    g[8 * 3 + 1] = SH_C2[4] * (-2.0 * y);
  }
  if (deg >= 3) {
    double xx = x * x, yy = y * y, zz = z * z;
    g[9 * 3 + 0] = SH_C3[0] * 6.0 * x * y;
    g[9 * 3 + 1] = SH_C3[0] * (3.0 * xx - 3.0 * yy);
    g[10 * 3 + 0] = SH_C3[1] * y * z;
    g[10 * 3 + 1] = SH_C3[1] * x * z;
    g[10 * 3 + 2] = SH_C3[1] * x * y;
    g[11 * 3 + 0] = SH_C3[2] * (-2.0 * x * y);
    g[11 * 3 + 1] = SH_C3[2] * (4.0 * zz - xx - 3.0 * yy);
    g[11 * 3 + 2] = SH_C3[2] * (8.0 * y * z);
    g[12 * 3 + 0] = SH_C3[3] * (-6.0 * x * z);
    g[12 * 3 + 1] = SH_C3[3] * (-6.0 * y * z);
    g[12 * 3 + 2] = SH_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    g[13 * 3 + 0] = SH_C3[4] * (4.0 * zz - 3.0 * xx - yy);
    g[13 * 3 + 1] = SH_C3[4] * (-2.0 * x * y);
    g[13 * 3 + 2] = SH_C3[4] * (8.0 * x * z);
    g[14 * 3 + 0] = SH_C3[5] * (2.0 * x * z);
    g[14 * 3 + 1] = SH_C3[5] * (-2.0 * y * z);
    g[14 * 3 + 2] = SH_C3[5] * (xx - yy);
    g[15 * 3 + 0] = SH_C3[6] * (3.0 * xx - 3.0 * yy);
    g[15 * 3 + 1] = SH_C3[6] * (-6.0 * x * y);
  }
}

/* field.py:40-60 -- rotation matrix of the normalized quaternion (w,x,y,z) */
static void quat_to_rotmat(const double q[4], double r[9], double qn[4], double* norm_out) {
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
  if (qn) {
    qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
  }
  if (norm_out) *norm_out = nrm;
}

/* field.py:71-75 -- Sigma = M M^T, M = R diag(exp(s)) */
static void covariance(const double q[4], const double ls[3], double cov[9]) {
  double r[9], m[9];
  quat_to_rotmat(q, r, NULL, NULL);
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) m[i * 3 + j] = r[i * 3 + j] * exp(ls[j]);
  for (int i = 0; i < 3; i++)
    for (int k = 0; k < 3; k++) {
      double acc = 0.0;
      for (int j = 0; j < 3; j++) acc += m[i * 3 + j] * m[k * 3 + j];
      cov[i * 3 + k] = acc;
    }
}

static int64_t trunc_i64(double v) {
  /* numpy astype(int64): truncation toward zero (x86 cvttsd2si semantics) */
  if (!(v > -9.2e18 && v < 9.2e18)) return INT64_MIN;
  return (int64_t)v;
}
static int64_t clip_i64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/*
 * projection.py:69-162 + sh.py:114-132, per Gaussian (no compaction; the
 * Python glue applies np.nonzero(keep) exactly like projection.py:130-133).
 */
void orc_project(int64_t n, int sh_deg, const double* pos, const double* rot, const double* ls,
                 const double* logit, const double* sh, const orc_cam* cam, uint8_t* keep,
                 double* means2d, double* conics, double* depths, double* radii, double* colors,
                 double* opac, double* cam_pts, double* clamp_mul, double* cov2d, double* cov3d_cam,
                 double* dirs, double* rsafe, uint8_t* lo, uint8_t* hi, int64_t* rect) {
  const int K = (sh_deg + 1) * (sh_deg + 1);
  const int64_t tiles_x = (cam->width + TILE - 1) / TILE;
  const int64_t tiles_y = (cam->height + TILE - 1) / TILE;
  const double* R = cam->R;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    const double* p = pos + i * 3;
    double cp[3];
    for (int j = 0; j < 3; j++) cp[j] = p[0] * R[j * 3 + 0] + p[1] * R[j * 3 + 1] + p[2] * R[j * 3 + 2] + cam->t[j];
    keep[i] = 0;
    if (!(cp[2] > ZNEAR)) continue;
    double x = cp[0], y = cp[1], z = cp[2];
    double u = cam->fx * x / z + cam->cx;
    double v = cam->fy * y / z + cam->cy;
    double limx = FRUSTUM_EXPAND * (cam->width / (2.0 * cam->fx));
    double limy = FRUSTUM_EXPAND * (cam->height / (2.0 * cam->fy));
    double tx = x / z, ty = y / z;
    double mulx = (tx > -limx && tx < limx) ? 1.0 : 0.0;
    double muly = (ty > -limy && ty < limy) ? 1.0 : 0.0;
    double txc = tx < -limx ? -limx : (tx > limx ? limx : tx);
    double tyc = ty < -limy ? -limy : (ty > limy ? limy : ty);
    double cw[9], cc[9];
    covariance(rot + i * 4, ls + i * 3, cw);
    /* einsum("ij,njk,lk->nil", R, cov, R) */
    for (int a = 0; a < 3; a++)
      for (int l = 0; l < 3; l++) {
        double acc = 0.0;
        for (int j = 0; j < 3; j++)
          for (int k = 0; k < 3; k++) acc += R[a * 3 + j] * cw[j * 3 + k] * R[l * 3 + k];
        cc[a * 3 + l] = acc;
      }
    double fx_z = cam->fx / z, fy_z = cam->fy / z;
    double j02 = -cam->fx * txc / z, j12 = -cam->fy * tyc / z;
    double c00 = cc[0], c01 = cc[1], c02 = cc[2], c11 = cc[4], c12 = cc[5], c22 = cc[8];
    double A = fx_z * (fx_z * c00 + j02 * c02) + j02 * (fx_z * c02 + j02 * c22) + COV2D_DILATION;
    double B = fx_z * (fy_z * c01 + j12 * c02) + j02 * (fy_z * c12 + j12 * c22);
    double C = fy_z * (fy_z * c11 + j12 * c12) + j12 * (fy_z * c12 + j12 * c22) + COV2D_DILATION;
    double det = A * C - B * B;
    int ok = det > 0.0;
    double inv_det = ok ? 1.0 / det : 0.0;
    double mid = 0.5 * (A + C);
    double mm = mid * mid - det;
    double lam = mid + sqrt(mm > 0.1 ? mm : 0.1);
    double radius = ceil(3.0 * sqrt(lam));
    int64_t tx0 = clip_i64(trunc_i64((u - radius) / TILE), 0, tiles_x);
    int64_t ty0 = clip_i64(trunc_i64((v - radius) / TILE), 0, tiles_y);
    int64_t tx1 = clip_i64(trunc_i64((u + radius) / TILE) + 1, 0, tiles_x);
    int64_t ty1 = clip_i64(trunc_i64((v + radius) / TILE) + 1, 0, tiles_y);
    int64_t wx = tx1 - tx0 > 0 ? tx1 - tx0 : 0, wy = ty1 - ty0 > 0 ? ty1 - ty0 : 0;
    ok = ok && (radius > 0) && (wx * wy > 0);
    if (!ok) continue;
    keep[i] = 1;
    means2d[i * 2] = u;
    means2d[i * 2 + 1] = v;
    conics[i * 3] = C * inv_det;
    conics[i * 3 + 1] = -B * inv_det;
    conics[i * 3 + 2] = A * inv_det;
    depths[i] = z;
    radii[i] = radius;
    opac[i] = 1.0 / (1.0 + exp(-logit[i]));
    for (int j = 0; j < 3; j++) cam_pts[i * 3 + j] = cp[j];
    clamp_mul[i * 2] = mulx;
    clamp_mul[i * 2 + 1] = muly;
    cov2d[i * 3] = A;
    cov2d[i * 3 + 1] = B;
    cov2d[i * 3 + 2] = C;
    for (int j = 0; j < 9; j++) cov3d_cam[i * 9 + j] = cc[j];
    rect[i * 4] = tx0;
    rect[i * 4 + 1] = ty0;
    rect[i * 4 + 2] = tx1;
    rect[i * 4 + 3] = ty1;
    /* sh.py:114-132 */
    double off[3];
    for (int j = 0; j < 3; j++) off[j] = p[j] - cam->center[j];
    double r = sqrt(off[0] * off[0] + off[1] * off[1] + off[2] * off[2]);
    double rs = r > 1e-12 ? r : 1e-12;
    double d[3] = {off[0] / rs, off[1] / rs, off[2] / rs};
    double basis[16];
    sh_basis(sh_deg, d, basis);
    for (int c = 0; c < 3; c++) {
      double acc = 0.0;
      for (int k = 0; k < K; k++) acc += sh[(i * 3 + c) * K + k] * basis[k];
      double raw = acc + 0.5;
      lo[i * 3 + c] = raw < 0.0;
      hi[i * 3 + c] = raw > 1.0;
      colors[i * 3 + c] = raw < 0.0 ? 0.0 : (raw > 1.0 ? 1.0 : raw);
      dirs[i * 3 + c] = d[c];
    }
    rsafe[i] = rs;
  }
}

typedef struct {
  int64_t tile;
  double depth;
  int64_t order;
  int64_t splat;
} inst_t;

static int inst_cmp(const void* a, const void* b) {
  const inst_t* x = (const inst_t*)a;
  const inst_t* y = (const inst_t*)b;
  if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  return x->order < y->order ? -1 : (x->order > y->order ? 1 : 0);
}

/*
 * projection.py:165-191 -- duplicate per overlapped tile (splat-major, ty outer,
 * tx inner), stable lexsort by (tile, depth), searchsorted tile ranges.
 * rect/depths are over the V visible splats; inst_splat has room for M.
 */
void orc_bin_tiles(int64_t V, int64_t tiles_x, int64_t n_tiles, const int64_t* rect,
                   const double* depths, int64_t M, int64_t* inst_splat, int64_t* tile_starts,
                   int64_t* tile_ends) {
  inst_t* a = (inst_t*)malloc(sizeof(inst_t) * (M > 0 ? M : 1));
  int64_t o = 0;
  for (int64_t i = 0; i < V; i++) {
    for (int64_t ty = rect[i * 4 + 1]; ty < rect[i * 4 + 3]; ty++)
      for (int64_t tx = rect[i * 4]; tx < rect[i * 4 + 2]; tx++) {
        a[o].tile = ty * tiles_x + tx;
        a[o].depth = depths[i];
        a[o].order = o;
        a[o].splat = i;
        o++;
      }
  }
  qsort(a, (size_t)M, sizeof(inst_t), inst_cmp);
  for (int64_t s = 0; s < M; s++) inst_splat[s] = a[s].splat;
  /* searchsorted(side=left/right) for every tile id */
  int64_t s = 0;
  for (int64_t t = 0; t < n_tiles; t++) {
    while (s < M && a[s].tile < t) s++;
    tile_starts[t] = s;
    int64_t e = s;
    while (e < M && a[e].tile <= t) e++;
    tile_ends[t] = e;
    s = e;
  }
  free(a);
}

/* kernels.py:31-103 -- front-to-back blend per pixel */
void orc_forward(int64_t tiles_x, int64_t width, int64_t height, int64_t n_tiles,
                 const int64_t* tile_starts, const int64_t* tile_ends, const int64_t* inst_splat,
                 const double* means2d, const double* conics, const double* opacities,
                 const double* colors, const double* bg, double* img, double* t_final,
                 int64_t* n_walk, uint8_t* terminated, int64_t* hard_count, double* soft_count) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < n_tiles; t++) {
    int64_t s0 = tile_starts[t], s1 = tile_ends[t];
    int64_t y00 = (t / tiles_x) * TILE, x00 = (t % tiles_x) * TILE;
    for (int64_t yy = y00; yy < (y00 + TILE < height ? y00 + TILE : height); yy++)
      for (int64_t xx = x00; xx < (x00 + TILE < width ? x00 + TILE : width); xx++) {
        double trans = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, soft = 0.0;
        int64_t nw = 0, hard = 0;
        int term = 0;
        for (int64_t s = s0; s < s1; s++) {
          int64_t k = s - s0;
          nw = k + 1;
          int64_t g = inst_splat[s];
          double dx = xx - means2d[g * 2], dy = yy - means2d[g * 2 + 1];
          double power = -0.5 * (conics[g * 3] * dx * dx + conics[g * 3 + 2] * dy * dy) - conics[g * 3 + 1] * dx * dy;
          if (power > 0.0) continue;
          double alpha = opacities[g] * exp(power);
          if (alpha > ALPHA_CAP) alpha = ALPHA_CAP;
          soft += 1.0 / (1.0 + exp(-(alpha - ALPHA_MIN) / SOFT_TAU));
          if (alpha < ALPHA_MIN) continue;
          double test_t = trans * (1.0 - alpha);
          if (test_t < T_EPS) {
            term = 1;
            break;
          }
          double w = alpha * trans;
          c0 += colors[g * 3] * w;
          c1 += colors[g * 3 + 1] * w;
          c2 += colors[g * 3 + 2] * w;
          hard += 1;
          trans = test_t;
        }
        int64_t px = yy * width + xx;
        img[px * 3] = c0 + bg[0] * trans;
        img[px * 3 + 1] = c1 + bg[1] * trans;
        img[px * 3 + 2] = c2 + bg[2] * trans;
        t_final[px] = trans;
        n_walk[px] = nw;
        terminated[px] = (uint8_t)term;
        hard_count[px] = hard;
        soft_count[px] = soft;
      }
  }
}

/* kernels.py:106-193 -- pixel-major backward (back to front, T by division) */
void orc_backward_pixel(int64_t tiles_x, int64_t width, int64_t height, int64_t n_tiles,
                        const int64_t* tile_starts, const int64_t* tile_ends,
                        const int64_t* inst_splat, const double* means2d, const double* conics,
                        const double* opacities, const double* colors, const double* bg,
                        const double* w_img, const double* w_soft, const double* t_final,
                        const int64_t* n_walk, const uint8_t* terminated, double* inst_rows) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < n_tiles; t++) {
    int64_t s0 = tile_starts[t], s1 = tile_ends[t];
    if (s1 <= s0) continue;
    int64_t y00 = (t / tiles_x) * TILE, x00 = (t % tiles_x) * TILE;
    for (int64_t yy = y00; yy < (y00 + TILE < height ? y00 + TILE : height); yy++)
      for (int64_t xx = x00; xx < (x00 + TILE < width ? x00 + TILE : width); xx++) {
        int64_t px = yy * width + xx;
        int64_t nw = n_walk[px];
        if (nw == 0) continue;
        int term = terminated[px];
        double trans = t_final[px], ws = w_soft[px];
        double w0 = w_img[px * 3], w1 = w_img[px * 3 + 1], w2 = w_img[px * 3 + 2];
        double sacc0 = bg[0] * trans, sacc1 = bg[1] * trans, sacc2 = bg[2] * trans;
        for (int64_t k = nw - 1; k >= 0; k--) {
          int64_t s = s0 + k;
          int64_t g = inst_splat[s];
          double dx = xx - means2d[g * 2], dy = yy - means2d[g * 2 + 1];
          double ca = conics[g * 3], cb = conics[g * 3 + 1], cc = conics[g * 3 + 2];
          double power = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
          if (power > 0.0) continue;
          double opa = opacities[g];
          double alpha = opa * exp(power);
          int capped = alpha > ALPHA_CAP;
          if (capped) alpha = ALPHA_CAP;
          int blended = alpha >= ALPHA_MIN && !(term == 1 && k == nw - 1);
          double dlda = 0.0;
          double* row = inst_rows + s * 9;
          if (blended) {
            double ti = trans / (1.0 - alpha);
            double aw = alpha * ti;
            row[0] += aw * w0;
            row[1] += aw * w1;
            row[2] += aw * w2;
            double inv = 1.0 / (1.0 - alpha);
            dlda = w0 * (colors[g * 3] * ti - sacc0 * inv) + w1 * (colors[g * 3 + 1] * ti - sacc1 * inv) +
                   w2 * (colors[g * 3 + 2] * ti - sacc2 * inv);
            sacc0 += colors[g * 3] * aw;
            sacc1 += colors[g * 3 + 1] * aw;
            sacc2 += colors[g * 3 + 2] * aw;
            trans = ti;
          }
          if (!capped) {
            double sv = 1.0 / (1.0 + exp(-(alpha - ALPHA_MIN) / SOFT_TAU));
            double gsoft = ws * sv * (1.0 - sv) / SOFT_TAU;
            row[3] += (dlda + gsoft) * alpha * (1.0 - opa);
            if (blended) {
              double gpow = dlda * alpha;
              row[4] += gpow * (ca * dx + cb * dy);
              row[5] += gpow * (cb * dx + cc * dy);
              row[6] += gpow * (-0.5 * dx * dx);
              row[7] += gpow * (-dx * dy);
              row[8] += gpow * (-0.5 * dy * dy);
            }
          }
        }
      }
  }
}

/* kernels.py:196-353 -- splat-major backward: chunked pass A / fixed-order pass B */
void orc_backward_splat(int64_t tiles_x, int64_t width, int64_t height, int64_t n_tiles,
                        const int64_t* tile_starts, const int64_t* tile_ends,
                        const int64_t* inst_splat, const double* means2d, const double* conics,
                        const double* opacities, const double* colors, const double* bg,
                        const double* w_img, const double* w_soft, const double* t_final,
                        const int64_t* n_walk, const uint8_t* terminated, double* inst_rows) {
  const int npx = TILE * TILE;
#pragma omp parallel
  {
    double* staged = (double*)malloc(sizeof(double) * CHUNK * npx * 9);
    double trans[TILE * TILE], sacc[TILE * TILE][3], wpx[TILE * TILE][3], wsf[TILE * TILE];
    double pxs[TILE * TILE], pys[TILE * TILE];
    int64_t nwk[TILE * TILE];
    uint8_t trm[TILE * TILE];
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < n_tiles; t++) {
      int64_t s0 = tile_starts[t], s1 = tile_ends[t];
      if (s1 <= s0) continue;
      int64_t y00 = (t / tiles_x) * TILE, x00 = (t % tiles_x) * TILE;
      int64_t max_walk = 0;
      for (int p = 0; p < npx; p++) {
        int64_t yy = y00 + p / TILE, xx = x00 + p % TILE;
        pxs[p] = (double)xx;
        pys[p] = (double)yy;
        if (yy < height && xx < width) {
          int64_t px = yy * width + xx;
          nwk[p] = n_walk[px];
          trm[p] = terminated[px];
          trans[p] = t_final[px];
          for (int ch = 0; ch < 3; ch++) {
            sacc[p][ch] = bg[ch] * trans[p];
            wpx[p][ch] = w_img[px * 3 + ch];
          }
          wsf[p] = w_soft[px];
          if (nwk[p] > max_walk) max_walk = nwk[p];
        } else {
          nwk[p] = 0;
          trm[p] = 0;
        }
      }
      int64_t k_hi = max_walk;
      while (k_hi > 0) {
        int64_t k_lo = k_hi - CHUNK;
        if (k_lo < 0) k_lo = 0;
        int64_t nc = k_hi - k_lo;
        for (int64_t r = 0; r < nc; r++) {
          int64_t k = k_hi - 1 - r;
          int64_t s = s0 + k;
          int64_t g = inst_splat[s];
          double mx = means2d[g * 2], my = means2d[g * 2 + 1];
          double ca = conics[g * 3], cb = conics[g * 3 + 1], cc = conics[g * 3 + 2];
          double opa = opacities[g];
          double col0 = colors[g * 3], col1 = colors[g * 3 + 1], col2 = colors[g * 3 + 2];
          for (int p = 0; p < npx; p++) {
            double* st = staged + (r * npx + p) * 9;
            for (int j = 0; j < 9; j++) st[j] = 0.0;
            if (k >= nwk[p]) continue;
            double dx = pxs[p] - mx, dy = pys[p] - my;
            double power = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy;
            if (power > 0.0) continue;
            double alpha = opa * exp(power);
            int capped = alpha > ALPHA_CAP;
            if (capped) alpha = ALPHA_CAP;
            int blended = alpha >= ALPHA_MIN && !(trm[p] == 1 && k == nwk[p] - 1);
            double dlda = 0.0;
            if (blended) {
              double ti = trans[p] / (1.0 - alpha);
              double aw = alpha * ti;
              st[0] = aw * wpx[p][0];
              st[1] = aw * wpx[p][1];
              st[2] = aw * wpx[p][2];
              double inv = 1.0 / (1.0 - alpha);
              dlda = wpx[p][0] * (col0 * ti - sacc[p][0] * inv) + wpx[p][1] * (col1 * ti - sacc[p][1] * inv) +
                     wpx[p][2] * (col2 * ti - sacc[p][2] * inv);
              sacc[p][0] += col0 * aw;
              sacc[p][1] += col1 * aw;
              sacc[p][2] += col2 * aw;
              trans[p] = ti;
            }
            if (!capped) {
              double sv = 1.0 / (1.0 + exp(-(alpha - ALPHA_MIN) / SOFT_TAU));
              double gsoft = wsf[p] * sv * (1.0 - sv) / SOFT_TAU;
              st[3] = (dlda + gsoft) * alpha * (1.0 - opa);
              if (blended) {
                double gpow = dlda * alpha;
                st[4] = gpow * (ca * dx + cb * dy);
                st[5] = gpow * (cb * dx + cc * dy);
                st[6] = gpow * (-0.5 * dx * dx);
                st[7] = gpow * (-dx * dy);
                st[8] = gpow * (-0.5 * dy * dy);
              }
            }
          }
        }
        for (int64_t r = 0; r < nc; r++) {
          int64_t s = s0 + k_hi - 1 - r;
          double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
          for (int p = 0; p < npx; p++) {
            const double* st = staged + (r * npx + p) * 9;
            for (int j = 0; j < 9; j++) acc[j] += st[j];
          }
          for (int j = 0; j < 9; j++) inst_rows[s * 9 + j] = acc[j];
        }
        k_hi = k_lo;
      }
    }
    free(staged);
  }
}

/* backward.py:110-118 -- np.bincount per column, instance order */
void orc_merge(int64_t M, int64_t V, const int64_t* inst_splat, const double* rows, double* per) {
  memset(per, 0, sizeof(double) * V * 9);
  for (int64_t s = 0; s < M; s++)
    for (int c = 0; c < 9; c++) per[inst_splat[s] * 9 + c] += rows[s * 9 + c];
}

/*
 * backward.py:132-259 + sh.py:135-152 -- chain per visible splat.
 * Inputs are gathered over the visible splats (index i < V).
 */
void orc_chain(int64_t V, int sh_deg, const orc_cam* cam, const double* sh, const double* quats,
               const double* log_scales, const double* conics, const double* cam_pts,
               const double* clamp_mul, const double* cov3d_cam, const double* dirs,
               const double* rsafe, const uint8_t* lo, const uint8_t* hi, const double* per,
               double* d_pos, double* d_quat, double* d_logscale, double* d_sh) {
  const int K = (sh_deg + 1) * (sh_deg + 1);
  const double fx = cam->fx, fy = cam->fy;
  const double* R = cam->R;
  const double limx = FRUSTUM_EXPAND * (cam->width / (2.0 * fx));
  const double limy = FRUSTUM_EXPAND * (cam->height / (2.0 * fy));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < V; i++) {
    const double* pr = per + i * 9;
    /* SH backward (sh.py:135-152) */
    double dcol[3];
    for (int c = 0; c < 3; c++) dcol[c] = (lo[i * 3 + c] || hi[i * 3 + c]) ? 0.0 : pr[c];
    double basis[16], gb[48];
    sh_basis(sh_deg, dirs + i * 3, basis);
    sh_basis_grad(sh_deg, dirs + i * 3, gb);
    for (int c = 0; c < 3; c++)
      for (int k = 0; k < K; k++) d_sh[(i * 3 + c) * K + k] = dcol[c] * basis[k];
    double ddir[3];
    for (int d = 0; d < 3; d++) {
      double acc = 0.0;
      for (int c = 0; c < 3; c++)
        for (int k = 0; k < K; k++) acc += dcol[c] * sh[(i * 3 + c) * K + k] * gb[k * 3 + d];
      ddir[d] = acc;
    }
    const double* dr = dirs + i * 3;
    double radial = ddir[0] * dr[0] + ddir[1] * dr[1] + ddir[2] * dr[2];
    double dpos_sh[3];
    for (int d = 0; d < 3; d++) dpos_sh[d] = (ddir[d] - radial * dr[d]) / rsafe[i];

    /* conic -> V2: g_v2 = -Q G Q */
    double q[4] = {conics[i * 3], conics[i * 3 + 1], conics[i * 3 + 1], conics[i * 3 + 2]};
    double gq[4] = {pr[6], 0.5 * pr[7], 0.5 * pr[7], pr[8]};
    double gv2[4];
    for (int a = 0; a < 2; a++)
      for (int l = 0; l < 2; l++) {
        double acc = 0.0;
        for (int j = 0; j < 2; j++)
          for (int k = 0; k < 2; k++) acc += q[a * 2 + j] * gq[j * 2 + k] * q[k * 2 + l];
        gv2[a * 2 + l] = -acc;
      }
    const double* p = cam_pts + i * 3;
    double x = p[0], y = p[1], z = p[2];
    double mulx = clamp_mul[i * 2], muly = clamp_mul[i * 2 + 1];
    double txr = x / z, tyr = y / z;
    double txc = txr < -limx ? -limx : (txr > limx ? limx : txr);
    double tyc = tyr < -limy ? -limy : (tyr > limy ? limy : tyr);
    double J[6] = {fx / z, 0.0, -fx * txc / z, 0.0, fy / z, -fy * tyc / z};
    const double* V3 = cov3d_cam + i * 9;
    double gJ[6], gv3[9], gw[9];
    for (int a = 0; a < 2; a++)
      for (int l = 0; l < 3; l++) {
        double acc = 0.0;
        for (int j = 0; j < 2; j++)
          for (int k = 0; k < 3; k++) acc += gv2[a * 2 + j] * J[j * 3 + k] * V3[k * 3 + l];
        gJ[a * 3 + l] = 2.0 * acc;
      }
    for (int a = 0; a < 3; a++)
      for (int l = 0; l < 3; l++) {
        double acc = 0.0;
        for (int j = 0; j < 2; j++)
          for (int k = 0; k < 2; k++) acc += J[j * 3 + a] * gv2[j * 2 + k] * J[k * 3 + l];
        gv3[a * 3 + l] = acc;
      }
    for (int a = 0; a < 3; a++)
      for (int l = 0; l < 3; l++) {
        double acc = 0.0;
        for (int j = 0; j < 3; j++)
          for (int k = 0; k < 3; k++) acc += R[j * 3 + a] * gv3[j * 3 + k] * R[k * 3 + l];
        gw[a * 3 + l] = acc;
      }
    double dcam[3] = {0.0, 0.0, 0.0};
    double z2 = z * z;
    dcam[0] += gJ[2] * (-fx * mulx / z2);
    dcam[1] += gJ[5] * (-fy * muly / z2);
    dcam[2] += gJ[0] * (-fx / z2);
    dcam[2] += gJ[4] * (-fy / z2);
    dcam[2] += gJ[2] * fx * (mulx * x / z + txc) / z2;
    dcam[2] += gJ[5] * fy * (muly * y / z + tyc) / z2;
    dcam[0] += pr[4] * fx / z;
    dcam[1] += pr[5] * fy / z;
    dcam[2] += -pr[4] * fx * x / z2 - pr[5] * fy * y / z2;
    for (int d = 0; d < 3; d++)
      d_pos[i * 3 + d] = dcam[0] * R[0 * 3 + d] + dcam[1] * R[1 * 3 + d] + dcam[2] * R[2 * 3 + d] + dpos_sh[d];

    /* _cov_to_rotation_scale (backward.py:209-259) */
    double rm[9], qn[4], nrm;
    quat_to_rotmat(quats + i * 4, rm, qn, &nrm);
    double sc[3] = {exp(log_scales[i * 3]), exp(log_scales[i * 3 + 1]), exp(log_scales[i * 3 + 2])};
    double m[9];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) m[a * 3 + b] = rm[a * 3 + b] * sc[b];
    double gs[9];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) gs[a * 3 + b] = gw[a * 3 + b] + gw[b * 3 + a];
    double dm[9], drot[9];
    for (int a = 0; a < 3; a++)
      for (int k = 0; k < 3; k++) {
        double acc = 0.0;
        for (int j = 0; j < 3; j++) acc += gs[a * 3 + j] * m[j * 3 + k];
        dm[a * 3 + k] = acc;
        drot[a * 3 + k] = acc * sc[k];
      }
    for (int j = 0; j < 3; j++) {
      double acc = 0.0;
      for (int a = 0; a < 3; a++) acc += dm[a * 3 + j] * rm[a * 3 + j];
      d_logscale[i * 3 + j] = acc * sc[j];
    }
    double w_ = qn[0], x_ = qn[1], y_ = qn[2], z_ = qn[3];
    double drw[9] = {0, -z_, y_, z_, 0, -x_, -y_, x_, 0};
    double drx[9] = {0, y_, z_, y_, -2 * x_, -w_, z_, w_, -2 * x_};
    double dry[9] = {-2 * y_, x_, w_, x_, 0, z_, -w_, z_, -2 * y_};
    double drz[9] = {-2 * z_, -w_, x_, w_, -2 * z_, y_, x_, y_, 0};
    double dqn[4] = {0, 0, 0, 0};
    for (int e = 0; e < 9; e++) {
      dqn[0] += drot[e] * (2.0 * drw[e]);
      dqn[1] += drot[e] * (2.0 * drx[e]);
      dqn[2] += drot[e] * (2.0 * dry[e]);
      dqn[3] += drot[e] * (2.0 * drz[e]);
    }
    double rad = dqn[0] * qn[0] + dqn[1] * qn[1] + dqn[2] * qn[2] + dqn[3] * qn[3];
    for (int e = 0; e < 4; e++) d_quat[i * 4 + e] = (dqn[e] - rad * qn[e]) / nrm;
  }
}

/* optim.py:40-47 -- one bias-corrected Adam update, lr per element */
void orc_adam(int64_t n, double* param, const double* grad, double* m, double* v, const double* lr,
              int64_t step) {
  const double b1 = 0.9, b2 = 0.999, eps = 1e-15;
  double bc1 = 1.0 - pow(b1, (double)step), bc2 = 1.0 - pow(b2, (double)step);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    m[i] = b1 * m[i] + (1.0 - b1) * grad[i];
    v[i] = b2 * v[i] + (1.0 - b2) * grad[i] * grad[i];
    double mh = m[i] / bc1, vh = v[i] / bc2;
    param[i] -= lr[i] * mh / (sqrt(vh) + eps);
  }
}

/* losses.py:415-417 -- scipy correlate1d(mode="constant") along axis 0 then 1, 11 taps */
static void blur(int64_t h, int64_t w, const double* win, const double* a, double* tmp, double* out) {
  const int P = 5;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < h; i++)
    for (int64_t j = 0; j < w; j++) {
      double acc = 0.0;
      for (int t = 0; t < 11; t++) {
        int64_t ii = i + t - P;
        if (ii >= 0 && ii < h) acc += win[t] * a[ii * w + j];
      }
      tmp[i * w + j] = acc;
    }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < h; i++)
    for (int64_t j = 0; j < w; j++) {
      double acc = 0.0;
      for (int t = 0; t < 11; t++) {
        int64_t jj = j + t - P;
        if (jj >= 0 && jj < w) acc += win[t] * tmp[i * w + jj];
      }
      out[i * w + j] = acc;
    }
}

/* losses.py:78-123 -- SSIM value over the interior crop + analytic gradient.
 * x,y are (h,w,nch) interleaved; grad has the same layout. */
double orc_ssim(int64_t h, int64_t w, int64_t nch, const double* x, const double* y, double* grad) {
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  double win[11], gsum = 0.0;
  for (int t = 0; t < 11; t++) {
    double tt = t - 5;
    win[t] = exp(-(tt * tt) / (2.0 * 1.5 * 1.5));
    gsum += win[t];
  }
  for (int t = 0; t < 11; t++) win[t] /= gsum;
  int64_t n = h * w;
  double* buf = (double*)malloc(sizeof(double) * n * 14);
  double *xc = buf, *yc = buf + n, *tmp = buf + 2 * n, *mux = buf + 3 * n, *muy = buf + 4 * n,
         *gx2 = buf + 5 * n, *gy2 = buf + 6 * n, *gxy = buf + 7 * n, *a = buf + 8 * n,
         *dmu = buf + 9 * n, *dg2 = buf + 10 * n, *dxy = buf + 11 * n, *o1 = buf + 12 * n, *o2 = buf + 13 * n;
  int64_t n_crop = (h - 10) * (w - 10);
  double total = 0.0;
  for (int64_t ch = 0; ch < nch; ch++) {
    for (int64_t i = 0; i < n; i++) {
      xc[i] = x[i * nch + ch];
      yc[i] = y[i * nch + ch];
    }
    blur(h, w, win, xc, tmp, mux);
    blur(h, w, win, yc, tmp, muy);
    for (int64_t i = 0; i < n; i++) a[i] = xc[i] * xc[i];
    blur(h, w, win, a, tmp, gx2);
    for (int64_t i = 0; i < n; i++) a[i] = yc[i] * yc[i];
    blur(h, w, win, a, tmp, gy2);
    for (int64_t i = 0; i < n; i++) a[i] = xc[i] * yc[i];
    blur(h, w, win, a, tmp, gxy);
    double csum = 0.0;
    for (int64_t r = 0; r < h; r++)
      for (int64_t c = 0; c < w; c++) {
        int64_t i = r * w + c;
        double vx = gx2[i] - mux[i] * mux[i], vy = gy2[i] - muy[i] * muy[i], cv = gxy[i] - mux[i] * muy[i];
        double a1 = 2.0 * mux[i] * muy[i] + C1, a2 = 2.0 * cv + C2;
        double b1 = mux[i] * mux[i] + muy[i] * muy[i] + C1, b2 = vx + vy + C2;
        double smap = (a1 * a2) / (b1 * b2);
        int in = r >= 5 && r < h - 5 && c >= 5 && c < w - 5;
        if (in) csum += smap;
        double mw = in ? 1.0 / (double)(n_crop * nch) : 0.0;
        dmu[i] = mw * (2.0 * muy[i] * (a2 - a1) / (b1 * b2) - 2.0 * mux[i] * smap * (1.0 / b1 - 1.0 / b2));
        dg2[i] = mw * (-smap / b2);
        dxy[i] = mw * (2.0 * a1 / (b1 * b2));
      }
    total += csum / (double)n_crop;
    blur(h, w, win, dmu, tmp, o1);
    blur(h, w, win, dg2, tmp, o2);
    blur(h, w, win, dxy, tmp, a);
    for (int64_t i = 0; i < n; i++) grad[i * nch + ch] = o1[i] + 2.0 * xc[i] * o2[i] + yc[i] * a[i];
  }
  free(buf);
  return total / (double)nch;
}
