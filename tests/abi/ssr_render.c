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
 *   ssr_render --query             host-only entry points, no device needed
 *
 * Test infrastructure (tests/test_abi_c.py builds and runs it). */
#include <cuda_runtime.h>
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

int main(int argc, char** argv) {
  if (argc == 2 && !strcmp(argv[1], "--query")) return query();
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
    SSR(ssr_chain(&cam, n, deg, pos, rot, lsc, sh, sp, rows, g, 0, NULL, st));
    CK(cudaStreamSynchronize(st));
    float* gh = (float*)malloc(4 * g_floats);
    CK(cudaMemcpy(gh, g, 4 * g_floats, cudaMemcpyDeviceToHost));
    fwrite(gh, 4, g_floats, o);
  }
  fclose(o);
  printf("rendered %dx%d, %lld instances\n", W, H, (long long)m);
  return 0;
}
