/* A non-Python host of the C ABI (include/ssr.h): renders one view the way
 * INTEGRATION.md section 2 describes, with caller-owned device buffers --
 * ssr_preprocess -> ssr_scan_tiles -> (host reads M) -> ssr_bin_tiles ->
 * ssr_forward -- and writes the image and per-pixel walk lengths.
 *
 *   ssr_render in.bin out.bin [--grad]
 *       in.bin: see main; out.bin: image H x W x 3 float32, then n_walk H x W
 *       int32; with --grad the render keeps the backward state (no soft
 *       counts) and a backward of d_image = 1e-3 + ssr_chain follow, the flat
 *       FieldGrads buffer appended to out.bin
 *   ssr_render in.bin out.bin --train   K training iterations of one view (see train)
 *   ssr_render --query             host-only entry points, no device needed
 *
 * Test infrastructure (tests/test_abi_c.py builds and runs it). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ssr.h"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(2);                                                                 \
    }                                                                          \
  } while (0)
#define SSR(x)                                                                  \
  do {                                                                          \
    int r_ = (x);                                                               \
    if (r_ != 0) {                                                              \
      fprintf(stderr, "%s failed (%d): %s\n", #x, r_, ssr_last_error());        \
      exit(3);                                                                  \
    }                                                                           \
  } while (0)

static void* dalloc(size_t bytes) {
  void* p = NULL;
  CK(cudaMalloc(&p, bytes ? bytes : 16));
  return p;
}

static void* upload(FILE* f, size_t bytes) {
  void* h = malloc(bytes ? bytes : 1);
  if (fread(h, 1, bytes, f) != bytes) {
    fprintf(stderr, "short input\n");
    exit(4);
  }
  void* d = dalloc(bytes);
  CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  free(h);
  return d;
}

static int query(void) {
  int64_t lo = 0, hi = 0, ws = 0;
  printf("version %d\n", ssr_version());
  printf("ckpt_floats %lld\n", (long long)ssr_ckpt_floats(100000, 8160));
  printf("fix_list_ints %lld\n", (long long)ssr_fix_list_ints(1920, 1080, 8160));
  printf("rows_floats %lld\n", (long long)ssr_rows_floats(1000));
  SSR(ssr_scan_workspace(1000000, &ws));
  printf("scan_workspace %lld\n", (long long)ws);
  SSR(ssr_bin_workspace(5000000, 8160, &ws));
  printf("bin_workspace %lld\n", (long long)ws);
  SSR(ssr_exchange_chunk(1003, 4, 3, &lo, &hi));
  printf("exchange_chunk %lld %lld\n", (long long)lo, (long long)hi);
  /* an invalid call returns an error code and sets the message */
  const int rc = ssr_exchange_chunk(10, 0, 0, &lo, &hi);
  printf("invalid %d %s\n", rc, ssr_last_error());
  return 0;
}

/* --train: K training iterations of one view, every stage from C -- render
 * (no soft counts) -> ssr_loss (L1 + D-SSIM on an 8-bit target) ->
 * ssr_backward -> ssr_chain_adam on the class-major flat parameter buffer.
 * in.bin continues after the field with: float64 lr[5] (position rate x scene
 * extent, rotation, scale, opacity, SH DC), lr_sh_rest, beta1, beta2, w_l1,
 * w_ssim; int32 K; the target H x W x 3 uint8.  out.bin: the flat parameters
 * (float32), then the last iteration's 5 loss terms (float64). */
static int train(FILE* f, const char* out_path, int64_t n, int32_t deg, const double* bg, const ssr_camera* cam) {
  const int64_t K = (int64_t)(deg + 1) * (deg + 1), ns = (n + 3) & ~(int64_t)3;
  const int64_t width[5] = {3, 4, 3, 1, 3 * K};
  int64_t off[5], pf = 0;
  for (int c = 0; c < 5; c++) {
    off[c] = pf;
    pf += width[c] * ns;
  }
  /* the class-major flat buffer of the package (field.py class_slices): class c
   * at off[c], n rows, zero padding to a multiple of 4 rows */
  float* hflat = (float*)calloc((size_t)pf, 4);
  for (int c = 0; c < 5; c++)
    if (fread(hflat + off[c], 4, (size_t)(width[c] * n), f) != (size_t)(width[c] * n)) return 4;
  double lr[5], lr_rest, b1, b2, w_l1, w_ssim;
  int32_t iters = 0;
  if (fread(lr, 8, 5, f) != 5 || fread(&lr_rest, 8, 1, f) != 1 || fread(&b1, 8, 1, f) != 1 ||
      fread(&b2, 8, 1, f) != 1 || fread(&w_l1, 8, 1, f) != 1 || fread(&w_ssim, 8, 1, f) != 1 ||
      fread(&iters, 4, 1, f) != 1)
    return 4;
  const int32_t W = cam->width, H = cam->height, tx = (W + 15) / 16, ty = (H + 15) / 16, nt = tx * ty;
  const size_t HW = (size_t)W * H;
  uint8_t* tgt = (uint8_t*)upload(f, 3 * HW);
  float* p = (float*)dalloc(4 * (size_t)pf);
  float* m = (float*)dalloc(4 * (size_t)pf);
  float* v = (float*)dalloc(4 * (size_t)pf);
  CK(cudaMemcpy(p, hflat, 4 * (size_t)pf, cudaMemcpyHostToDevice));
  CK(cudaMemset(m, 0, 4 * (size_t)pf));
  CK(cudaMemset(v, 0, 4 * (size_t)pf));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  ssr_splats sp;
  memset(&sp, 0, sizeof sp);
  sp.mean = (double*)dalloc(16 * n);
  sp.conic_opa = (float*)dalloc(16 * n);
  sp.color = (float*)dalloc(16 * n);
  sp.conic_opa64 = (double*)dalloc(32 * n);
  sp.color64 = (double*)dalloc(32 * n);
  sp.depth = (double*)dalloc(8 * n);
  sp.rect = (int32_t*)dalloc(16 * n);
  sp.tiles = (uint32_t*)dalloc(4 * n);
  sp.offset = (uint32_t*)dalloc(4 * n);
  sp.row_offset = (uint32_t*)dalloc(4 * n);
  sp.depth_order = (uint32_t*)dalloc(4 * n);
  int64_t ws_bytes = 0, loss_bytes = 0;
  SSR(ssr_scan_workspace(n, &ws_bytes));
  SSR(ssr_loss_workspace(W, H, &loss_bytes));
  void* ws = dalloc((size_t)ws_bytes);
  void* lws = dalloc((size_t)loss_bytes);
  uint64_t* total_dev = (uint64_t*)dalloc(8);
  int32_t* ranges = (int32_t*)dalloc(8 * (size_t)nt);
  ssr_frame fr;
  memset(&fr, 0, sizeof fr);
  fr.width = W;
  fr.height = H;
  fr.tiles_x = tx;
  fr.tiles_y = ty;
  for (int c = 0; c < 3; c++) fr.bg[c] = (float)bg[c];
  fr.image = (float*)dalloc(12 * HW);
  fr.t_final = (float*)dalloc(4 * HW);
  fr.n_walk = (int32_t*)dalloc(4 * HW);
  fr.terminated = (uint8_t*)dalloc(HW);
  fr.hard_count = (int32_t*)dalloc(4 * HW);
  fr.soft_count = NULL; /* the objective has no load term */
  fr.flagged = (uint8_t*)dalloc(HW);
  fr.tile_info = (int32_t*)dalloc(16 * (size_t)nt);
  fr.fix_list = (int32_t*)dalloc(4 * (size_t)ssr_fix_list_ints(W, H, nt));
  float* dimg = (float*)dalloc(12 * HW);
  double* loss = (double*)dalloc(8 * 5);
  uint32_t* inst = NULL;
  float* rows = NULL;
  int64_t cap = 0;
  for (int32_t it = 0; it < iters; it++) {
    SSR(ssr_preprocess(cam, n, deg, p + off[0], p + off[1], p + off[2], p + off[3], p + off[4], sp, st));
    SSR(ssr_scan_tiles(n, sp, ws, ws_bytes, total_dev, st));
    uint64_t mm = 0;
    CK(cudaMemcpyAsync(&mm, total_dev, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t M = (int64_t)mm;
    if (M > cap) { /* instance buffers and the rows workspace (zero-filled) for this M */
      if (inst) {
        CK(cudaFree(inst));
        CK(cudaFree(rows));
        CK(cudaFree(fr.ckpt));
      }
      cap = M;
      inst = (uint32_t*)dalloc(4 * (size_t)cap);
      const int64_t rf = ssr_rows_floats(cap);
      rows = (float*)dalloc(4 * (size_t)rf);
      CK(cudaMemset(rows, 0, 4 * (size_t)rf));
      fr.ckpt = (float*)dalloc(4 * (size_t)ssr_ckpt_floats(cap, nt));
    }
    int64_t bin_bytes = 0;
    SSR(ssr_bin_workspace(M, nt, &bin_bytes));
    void* bws = dalloc((size_t)bin_bytes);
    SSR(ssr_bin_tiles(n, M, tx, ty, sp, inst, ranges, bws, bin_bytes, st));
    SSR(ssr_forward(M, sp, inst, ranges, fr, 1e-5f, 1e-4f, st));
    SSR(ssr_loss(W, H, fr.image, tgt, 1, NULL, fr.hard_count, w_l1, w_ssim, 0.0, dimg, NULL, loss, lws,
                 loss_bytes, st));
    SSR(ssr_backward(0, M, sp, inst, ranges, fr, dimg, NULL, rows, st));
    double bc1[5], bc2[5];
    for (int c = 0; c < 5; c++) {
      bc1[c] = 1.0 - pow(b1, (double)(it + 1));
      bc2[c] = 1.0 - pow(b2, (double)(it + 1));
    }
    SSR(ssr_chain_adam(cam, n, deg, p, m, v, sp, rows, NULL, lr, lr_rest, bc1, bc2, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaFree(bws));
  }
  CK(cudaMemcpy(hflat, p, 4 * (size_t)pf, cudaMemcpyDeviceToHost));
  double hl[5];
  CK(cudaMemcpy(hl, loss, 40, cudaMemcpyDeviceToHost));
  FILE* o = fopen(out_path, "wb");
  if (!o) return 1;
  fwrite(hflat, 4, (size_t)pf, o);
  fwrite(hl, 8, 5, o);
  fclose(o);
  printf("trained %d iterations, loss %.6f\n", iters, hl[3]);
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 2 && !strcmp(argv[1], "--query")) return query();
  if (argc == 4 && !strcmp(argv[3], "--train")) {
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 1;
    int64_t n = 0;
    int32_t deg = 0;
    double bg[3];
    ssr_camera cam;
    if (fread(&n, 8, 1, f) != 1 || fread(&deg, 4, 1, f) != 1 || fread(bg, 8, 3, f) != 3 ||
        fread(&cam, sizeof cam, 1, f) != 1)
      return 4;
    const int rc = train(f, argv[2], n, deg, bg, &cam);
    fclose(f);
    return rc;
  }
  const int grad = argc == 4 && !strcmp(argv[3], "--grad");
  if (argc != 3 && !grad) {
    fprintf(stderr, "usage: ssr_render in.bin out.bin [--grad] | --query\n");
    return 1;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  /* in.bin: int64 n, int32 sh_degree, float64 bg[3], ssr_camera, then the
   * field's classes (float32): positions 3n, rotations 4n, log_scales 3n,
   * opacity_logits n, sh 3Kn (channel-major) */
  int64_t n = 0;
  int32_t deg = 0;
  double bg[3];
  ssr_camera cam;
  if (fread(&n, 8, 1, f) != 1 || fread(&deg, 4, 1, f) != 1 || fread(bg, 8, 3, f) != 3 ||
      fread(&cam, sizeof cam, 1, f) != 1)
    return 4;
  const int64_t K = (int64_t)(deg + 1) * (deg + 1);
  float* pos = (float*)upload(f, 4 * 3 * n);
  float* rot = (float*)upload(f, 4 * 4 * n);
  float* lsc = (float*)upload(f, 4 * 3 * n);
  float* opa = (float*)upload(f, 4 * n);
  float* sh = (float*)upload(f, 4 * 3 * K * n);
  fclose(f);

  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  ssr_splats sp;
  memset(&sp, 0, sizeof sp);
  sp.mean = (double*)dalloc(16 * n);
  sp.conic_opa = (float*)dalloc(16 * n);
  sp.color = (float*)dalloc(16 * n);
  sp.conic_opa64 = (double*)dalloc(32 * n);
  sp.color64 = (double*)dalloc(32 * n);
  sp.depth = (double*)dalloc(8 * n);
  sp.rect = (int32_t*)dalloc(16 * n);
  sp.tiles = (uint32_t*)dalloc(4 * n);
  sp.offset = (uint32_t*)dalloc(4 * n);
  sp.row_offset = (uint32_t*)dalloc(4 * n);
  sp.depth_order = (uint32_t*)dalloc(4 * n);
  SSR(ssr_preprocess(&cam, n, deg, pos, rot, lsc, opa, sh, sp, st));

  int64_t ws_bytes = 0;
  SSR(ssr_scan_workspace(n, &ws_bytes));
  void* ws = dalloc((size_t)ws_bytes);
  uint64_t* total_dev = (uint64_t*)dalloc(8);
  SSR(ssr_scan_tiles(n, sp, ws, ws_bytes, total_dev, st));
  uint64_t m = 0;  /* the path's one host read: the instance count */
  CK(cudaMemcpyAsync(&m, total_dev, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));

  const int32_t W = cam.width, H = cam.height, tx = (W + 15) / 16, ty = (H + 15) / 16, nt = tx * ty;
  int64_t bin_bytes = 0;
  SSR(ssr_bin_workspace((int64_t)m, nt, &bin_bytes));
  void* bws = dalloc((size_t)bin_bytes);
  uint32_t* inst = (uint32_t*)dalloc(4 * m);
  int32_t* ranges = (int32_t*)dalloc(8 * (size_t)nt);
  SSR(ssr_bin_tiles(n, (int64_t)m, tx, ty, sp, inst, ranges, bws, bin_bytes, st));

  ssr_frame fr;
  memset(&fr, 0, sizeof fr);
  fr.width = W;
  fr.height = H;
  fr.tiles_x = tx;
  fr.tiles_y = ty;
  for (int c = 0; c < 3; c++) fr.bg[c] = (float)bg[c];
  const size_t HW = (size_t)W * H;
  fr.image = (float*)dalloc(12 * HW);
  fr.t_final = (float*)dalloc(4 * HW);
  fr.n_walk = (int32_t*)dalloc(4 * HW);
  fr.terminated = (uint8_t*)dalloc(HW);
  fr.hard_count = (int32_t*)dalloc(4 * HW);
  fr.soft_count = grad ? NULL : (double*)dalloc(8 * HW); /* training: no soft counts */
  fr.flagged = (uint8_t*)dalloc(HW);
  fr.tile_info = (int32_t*)dalloc(16 * (size_t)nt);
  /* render only: no backward state; training: the bucket checkpoints */
  fr.ckpt = grad ? (float*)dalloc(4 * (size_t)ssr_ckpt_floats((int64_t)m, nt)) : NULL;
  fr.fix_list = (int32_t*)dalloc(4 * (size_t)ssr_fix_list_ints(W, H, nt));
  SSR(ssr_forward((int64_t)m, sp, inst, ranges, fr, 1e-5f, 1e-4f, st));
  CK(cudaStreamSynchronize(st));

  float* img = (float*)malloc(12 * HW);
  int32_t* nw = (int32_t*)malloc(4 * HW);
  CK(cudaMemcpy(img, fr.image, 12 * HW, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(nw, fr.n_walk, 4 * HW, cudaMemcpyDeviceToHost));
  FILE* o = fopen(argv[2], "wb");
  if (!o) return 1;
  fwrite(img, 4, 3 * HW, o);
  fwrite(nw, 4, HW, o);
  if (grad) {
    /* dL/d(image) = 1e-3 everywhere -> instance rows -> the chain */
    float* dimg_h = (float*)malloc(12 * HW);
    for (size_t i = 0; i < 3 * HW; i++) dimg_h[i] = 1e-3f;
    float* dimg = (float*)dalloc(12 * HW);
    CK(cudaMemcpy(dimg, dimg_h, 12 * HW, cudaMemcpyHostToDevice));
    /* the rows workspace: zero-filled once, then reused by every backward */
    const int64_t rows_n = ssr_rows_floats((int64_t)m);
    float* rows = (float*)dalloc(4 * (size_t)rows_n);
    CK(cudaMemset(rows, 0, 4 * (size_t)rows_n));
    const int64_t ns = (n + 3) & ~(int64_t)3;
    const size_t g_floats = (size_t)(11 + 3 * K + 2) * ns;
    float* g = (float*)dalloc(4 * g_floats);
    SSR(ssr_backward(0, (int64_t)m, sp, inst, ranges, fr, dimg, NULL, rows, st));
    SSR(ssr_chain(&cam, n, deg, pos, rot, lsc, sh, sp, rows, g, 0, NULL, NULL, st));
    CK(cudaStreamSynchronize(st));
    float* gh = (float*)malloc(4 * g_floats);
    CK(cudaMemcpy(gh, g, 4 * g_floats, cudaMemcpyDeviceToHost));
    fwrite(gh, 4, g_floats, o);
  }
  fclose(o);
  printf("rendered %dx%d, %lld instances\n", W, H, (long long)m);
  return 0;
}
