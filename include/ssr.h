/*
 * ssr.h -- C ABI of the B200 (sm_100a) splat rasterizer ("splatstream raster").
 *
 * Drop-in boundary for the reference package's Python operator API
 * (/root/reference/pkg/src/splatstream/...):
 *
 *   render(field, cam, bg, workers)            rasterize/forward.py:66-114
 *     = ssr_preprocess -> ssr_scan_tiles -> ssr_bin_tiles -> ssr_forward
 *   project_field(field, cam)                  rasterize/projection.py:69-191
 *     = ssr_preprocess -> ssr_scan_tiles -> ssr_bin_tiles (+ ssr_project_aux)
 *   backward(field, out, d_image, d_soft, ...) rasterize/backward.py:41-129
 *     = ssr_backward (kernels.py:106-353) -> ssr_chain (backward.py:110-259)
 *   FieldOptimizer.step(fld, grads, rate)      optim.py:113-130  = ssr_adam
 *   GaussianField.densify_and_prune(...)       field.py:303-375
 *     = ssr_densify_masks -> ssr_densify_apply (+ optim.py:101-111 remap)
 *   total_loss(rendered, target, out, w)       losses.py:147-173 = ssr_loss
 *
 * Rules: every pointer is DEVICE memory unless documented otherwise; buffers
 * are caller-owned (workspace sizes come from the *_workspace queries); no
 * function allocates, frees or synchronises (except where a host-visible
 * result is documented); all work is ordered on `stream` (a cudaStream_t);
 * the only global state is the per-thread error string.  Every function
 * returns 0 on success, non-zero on failure; ssr_last_error() describes it.
 * `workers` of the reference API has no counterpart (the GPU grid is fixed).
 */
#ifndef SSR_H
#define SSR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSR_OK 0
#define SSR_ERR_INVALID 1 /* maps to InvalidParameter */
#define SSR_ERR_CUDA 2    /* a CUDA launch/runtime failure */
#define SSR_ERR_CAPACITY 3 /* instance count overflow etc. */

#define SSR_TILE 16
#define SSR_BUCKET 32 /* splats per backward bucket / checkpoint interval */

/* Pinhole camera, world-to-camera x_cam = R x_world + t (camera.py:11-52).
 * Kept in float64 end to end (the reference rejects fp32-rounded poses). */
typedef struct ssr_camera {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  double center[3]; /* -R^T t */
  int32_t width, height;
} ssr_camera;

/* Per-Gaussian preprocess outputs (indexed by field row, N entries each).
 * Rows with tiles[i] == 0 are culled (projection.py:76-133) and left unwritten. */
typedef struct ssr_splats {
  double* mean;        /* N x 2  projected mean (u, v), fp64 */
  float* conic_opa;    /* N x 4  (conic a, b, c, opacity), fp32 */
  float* color;        /* N x 4  clamped SH colour (r, g, b), .w = int bits: channel c not clamped */
  double* conic_opa64; /* N x 4  fp64 copies for the guard-band fix-up */
  double* color64;     /* N x 4 */
  double* depth;       /* N      camera-space z, fp64 */
  int32_t* rect;       /* N x 4  tile rect (tx0, ty0, tx1, ty1), exclusive upper */
  uint32_t* tiles;     /* N      tiles touched (0 = culled) */
  uint32_t* offset;    /* N      first instance id: tiles scanned in (fp64 depth, row) order */
  uint32_t* row_offset; /* N     first gradient row: tiles scanned in field-row order, so a
                            block of consecutive rows owns one contiguous range of inst_rows */
  uint32_t* depth_order; /* N    field row of the r-th Gaussian in (fp64 depth, row) order (culled
                            rows last); written by ssr_scan_tiles, read by ssr_bin_tiles */
} ssr_splats;

/* Render-time per-pixel / per-tile state retained for the backward. */
typedef struct ssr_frame {
  int32_t width, height, tiles_x, tiles_y;
  float bg[3];
  float* image;        /* H x W x 3 */
  float* t_final;      /* H x W */
  int32_t* n_walk;     /* H x W */
  uint8_t* terminated; /* H x W */
  int32_t* hard_count; /* H x W */
  double* soft_count;  /* H x W  float64: counts reach 10^4, the bar is 1e-4 absolute.  NULL:
                        * no soft counts (the walk culls pairs below 1/255); ssr_backward
                        * layout 0 then takes no d_soft */
  uint8_t* flagged;    /* H x W  1 = pixel re-walked in fp64 (guard band) */
  int32_t* tile_info;  /* n_tiles x 4  (max n_walk, flagged pixel count, max n_walk of a flagged pixel, 0) */
  float* ckpt;         /* ssr_ckpt_floats(M, n_tiles) floats: (T, C_front rgb) per bucket/pixel */
  int32_t* fix_list;   /* ssr_fix_list_ints(W, H, n_tiles) int32, written by ssr_forward: [0] flagged
                        * pixels, [1] flagged tiles, [2] backward fix-up buckets, [3] spare,
                        * then n_tiles slots (first pixel entry of each
                        * flagged tile, unordered), n_tiles bucket-plan
                        * slots, then W*H pixel entries (tile << 8 | pixel in tile),
                        * contiguous per tile, in a fixed order within it */
} ssr_frame;

const char* ssr_last_error(void);
int ssr_version(void);
/* sm count / compute capability of the current device (host-visible). */
int ssr_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* ---------------------------------------------------------- stage 1 */
/* projection.py:69-162 + sh.py:114-132: EWA projection, conic, radius, tile
 * rect, SH colour; float64 arithmetic on float32 storage. */
int ssr_preprocess(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                   const float* rotations, const float* log_scales, const float* opacity_logits,
                   const float* sh, ssr_splats splats, void* stream);

/* Retained intermediates of ProjectedSplats (projection.py:40-48), N-indexed,
 * fp64; for API completeness -- the hot path recomputes them in ssr_chain. */
int ssr_project_aux(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
                    const float* rotations, const float* log_scales, const float* sh,
                    const uint32_t* tiles, double* cam_points, double* clamp_mul, double* cov2d,
                    double* cov3d_cam, double* sh_dirs, double* sh_radii, uint8_t* sh_lo,
                    uint8_t* sh_hi, double* radii, void* stream);

/* ---------------------------------------------------------- stage 2 */
/* Hand-written (no library sort or scan).  Depth pre-sort of the N rows: three
 * stable 8-bit radix passes over a 24-bit monotone key of fp32(depth) with an
 * fp64 (depth, row) tie-fix -> splats.depth_order; then one launch with two
 * decoupled-look-back scans of splats.tiles: in depth order into splats.offset
 * (each row's instances are emitted at depth-ordered positions) and in field-row
 * order into splats.row_offset.  *total_dev gets M, summed in 64 bits; M is
 * computed first and stored by a kernel into mapped pinned host memory ahead of
 * the depth sort (no copy engine: it cannot queue behind the caller's uploads),
 * so a following ssr_bin_tiles_capacity on the same host thread waits for that
 * store alone while the device still sorts. */
int ssr_scan_workspace(int64_t n, int64_t* bytes);
int ssr_scan_tiles(int64_t n, ssr_splats splats, void* workspace, int64_t workspace_bytes,
                   uint64_t* total_dev, void* stream);

/* projection.py:165-191: duplicate each visible splat per overlapped tile at
 * its depth-ordered offset, two stable 8-bit radix passes over the tile id
 * (<= 65536 tiles) -> (tile, fp64 depth, row) order, searchsorted tile ranges.
 * M must be below 2^30 (SSR_ERR_CAPACITY otherwise).  Outputs:
 *   inst_gauss[M]   field row of each sorted instance
 *   tile_ranges[2*n_tiles]  (start, end) per tile, searchsorted semantics */
int ssr_bin_workspace(int64_t m, int32_t n_tiles, int64_t* bytes);
int ssr_bin_tiles(int64_t n, int64_t m, int32_t tiles_x, int32_t tiles_y, ssr_splats splats,
                  uint32_t* inst_gauss, int32_t* tile_ranges, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* ssr_bin_tiles with the instance count read here: copies *total_dev (from
 * ssr_scan_tiles) to the host, synchronises the stream, stores M in *m_out and,
 * when M <= capacity, bins into inst_gauss / workspace sized for `capacity`
 * instances (ssr_bin_workspace(capacity, ...)).  Returns SSR_ERR_CAPACITY
 * without launching when M > capacity (the caller then sizes the buffers for
 * *m_out and calls ssr_bin_tiles).  Lets the binning start without a round
 * trip through the host language after the path's one synchronisation.
 * `stream` must be the stream of the preceding ssr_scan_tiles: the binning reads
 * its depth order and offsets, ordered after them by that stream only. */
int ssr_bin_tiles_capacity(int64_t n, int64_t capacity, int32_t tiles_x, int32_t tiles_y, ssr_splats splats,
                           const uint64_t* total_dev, int64_t* m_out, uint32_t* inst_gauss, int32_t* tile_ranges,
                           void* workspace, int64_t workspace_bytes, void* stream);

/* Floats needed for the checkpoint buffer of a frame with M instances. */
int64_t ssr_ckpt_floats(int64_t m, int32_t n_tiles);

/* ---------------------------------------------------------- stage 3 */
/* kernels.py:31-103: 16x16-tile front-to-back blend (fp32) with an fp64
 * guard-band re-walk of pixels whose discrete decisions sit within a relative
 * band of a threshold: band_alpha around the alpha >= 1/255
 * gate and the 0.99 cap, band_t around the T(1 - alpha) < 1e-4 termination. */
/* Size of ssr_frame.fix_list. */
int64_t ssr_fix_list_ints(int32_t width, int32_t height, int32_t n_tiles);

int ssr_forward(int64_t m, ssr_splats splats, const uint32_t* inst_gauss,
                const int32_t* tile_ranges, ssr_frame frame, float band_alpha, float band_t,
                void* stream);

/* ---------------------------------------------------------- stage 4 */
/* kernels.py:106-353: per-instance rows [dcolor rgb, dlogit, dmu xy,
 * dconic abc] (9 floats) stored at the instance's splat-major position
 * (splats.row_offset[g] + local tile index).  layout 0 = splat-parallel
 * (Taming-style warp per 32-splat bucket), 1 = pixel-parallel.  Rows of
 * guard-band pixels are added by an fp64 pixel walk.
 *
 * inst_rows is a WORKSPACE of ssr_rows_floats(M) floats that the caller
 * zero-fills once when it allocates it and then hands unchanged to every
 * ssr_backward / ssr_chain pair (it may be regrown: zero-fill the new one).
 * Word 0 holds a generation counter, then each instance has a 10-word row: the
 * 9 terms and the generation that wrote it.  ssr_backward writes rows only for
 * the slots some pixel walked (slot < tile_info.x); a row with a stale tag is
 * zero to ssr_chain.  This skips the scattered zero-fill of unwalked slots
 * (~30% of the rows at config 2, ~80% at config 4).  One buffer per stream (and host
 * thread issuing backward / chain pairs). */
int64_t ssr_rows_floats(int64_t m);

int ssr_backward(int32_t layout, int64_t m, ssr_splats splats, const uint32_t* inst_gauss,
                 const int32_t* tile_ranges, ssr_frame frame, const float* d_image,
                 const float* d_soft, float* inst_rows, void* stream);

/* backward.py:110-259 + sh.py:135-152: merge rows per splat (bincount
 * order) and chain through projection/SH in fp32 (ssr_chain.cu).  grads is the flat
 * FieldGrads buffer [pos 3N | rot 4N | logscale 3N | logit N | sh 3KN |
 * screen_norm N | visible N].  accumulate!=0 adds into it (view batches);
 * stats (optional, 2N: grad_accum, grad_count) get += screen_norm/visible.
 * inst_rows is the workspace ssr_backward just filled; it is consumed (the
 * chain parks merged colour gradients in it between its kernels).  row_list
 * (optional, N + 1 uint32 of scratch; used with accumulate != 0): the SH pass
 * then runs over the rows this view sees only (full warps), listed there. */
int ssr_chain(const ssr_camera* cam, int64_t n, int32_t sh_degree, const float* positions,
              const float* rotations, const float* log_scales, const float* sh, ssr_splats splats,
              const float* inst_rows, float* grads, int32_t accumulate, float* stats, uint32_t* row_list,
              void* stream);

/* backward.py:110-259 fused with optim.py:40-47,113-130: the chain of ssr_chain
 * followed by the dense Adam step of ssr_adam, without materialising
 * FieldGrads: rotations / log-scales / logits are stepped by the geometry
 * kernel, SH rows (+ their m, v, staged with TMA bulk copies) and positions by
 * the SH kernel; invisible rows get the zero-gradient update.  params, m, v
 * are the flat buffers of ssr_adam; lr, bc1, bc2 HOST arrays as there. */
int ssr_chain_adam(const ssr_camera* cam, int64_t n, int32_t sh_degree, float* params, float* m, float* v,
                   ssr_splats splats, float* inst_rows, float* stats, const double* lr,
                   double lr_sh_rest, const double* bc1, const double* bc2, void* stream);

/* ---------------------------------------------------------- stage 5 */
/* optim.py:29-47,113-130: dense bias-corrected Adam over the flat parameter
 * buffer [pos | rot | logscale | logit | sh] (n rows, K sh coeffs).
 * lr[5] = (pos, rot, scale, opacity, sh_dc), sh rest lr = lr_sh_rest;
 * bc1/bc2[5] = 1 - beta^step per class.  lr, bc1, bc2 are HOST arrays. */
int ssr_adam(int64_t n, int32_t sh_degree, float* params, const float* grads, float* m, float* v,
             const double* lr, double lr_sh_rest, const double* bc1, const double* bc2, void* stream);

/* ssr_adam restricted to the flat elements [lo, hi) of the same class-major
 * buffers: the owner's share of a sharded (reduce-scatter -> Adam -> all-gather)
 * view-batch step.  grads[e - grads_offset] is element e's gradient,
 * so a rank passes just its reduced chunk (grads_offset = lo). */
int ssr_adam_range(int64_t n, int32_t sh_degree, float* params, const float* grads, int64_t grads_offset,
                   float* m, float* v, int64_t lo, int64_t hi, const double* lr, double lr_sh_rest,
                   const double* bc1, const double* bc2, void* stream);

/* The sharded view-batch exchange fused into one kernel per rank,
 * over peer memory instead of reduce-scatter -> ssr_adam_range -> all-gather.
 * grads / params: HOST arrays of `world` (<= 8) DEVICE pointers, entry q = rank
 * q's FieldGrads flat buffer / field parameter buffer, mapped into this process
 * (CUDA IPC over NVLink / NVSwitch; on one device, that device's memory).
 * Rank `rank` owns the flat parameter elements ssr_exchange_chunk(P, world,
 * rank) (P = (11+3K) * row_stride(n)): it sums their gradients over the ranks in
 * rank order, runs Adam on params[rank] with its own m, v (current only in its
 * chunk, like ssr_adam_range) and stores the result into every params[q]; the
 * densify statistics [screen_norms | visible] are summed over the ranks the
 * same way (its chunk of the 2 * row_stride(n) floats after P) and the sum is
 * stored into every grads[q].  Caller contract: a barrier that orders every
 * rank's gradient writes before any rank's call, and one after every rank's
 * call before any replica is read (e.g. a 1-element NCCL all-reduce on the
 * stream, which the kernel's stores precede by stream order).  lr, bc1, bc2 as ssr_adam. */
int ssr_exchange_adam(int64_t n, int32_t sh_degree, int32_t world, int32_t rank, float* const* grads,
                      float* const* params, float* m, float* v, const double* lr, double lr_sh_rest,
                      const double* bc1, const double* bc2, void* stream);
/* Peer buffers for ssr_exchange_adam (CUDA IPC).  ssr_ipc_export: the
 * SSR_IPC_HANDLE_BYTES-byte handle of the device allocation holding ptr and
 * ptr's offset in it.  ssr_ipc_open (another process): maps that allocation on
 * the CURRENT device with lazy peer access and returns the buffer's address;
 * opening one allocation twice shares the mapping (reference-counted).
 * ssr_ipc_close: drops one reference (unmapping at zero). */
#define SSR_IPC_HANDLE_BYTES 64
int ssr_ipc_export(const void* ptr, uint8_t* handle, int64_t* offset);
int ssr_ipc_open(const uint8_t* handle, int64_t offset, void** ptr);
int ssr_ipc_close(const uint8_t* handle);
/* [lo, hi) of rank's chunk of `total` floats: 16-byte aligned equal chunks,
 * the last rank also owning the remainder (used by ssr_exchange_adam). */
int ssr_exchange_chunk(int64_t total, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);

/* field.py:303-375: per-row flags (bit0 keep, bit1 clone, bit2 split) and
 * counts[3] = (n_clone, n_split, n_prune) in device memory. stats = the
 * already averaged grad_accum / max(count, 1) (pipeline.py:209-210). */
int ssr_densify_masks(int64_t n, const float* params, int32_t sh_degree, const float* stats,
                      double grad_threshold, double big_threshold, double prune_opacity,
                      uint8_t* flags, int32_t* counts, void* stream);
int ssr_densify_workspace(int64_t n, int64_t* bytes);
/* Compacts params (+ Adam m, v when non-null) into the new buffers: kept rows,
 * clones, split pairs (field.py:329-372, optim.py:49-54).  eps = (2*n_split)x3
 * standard normals drawn on the host from the session RNG (field.py:340). */
int ssr_densify_apply(int64_t n, int64_t n_new, int32_t sh_degree, const float* params,
                      const float* m, const float* v, const uint8_t* flags, const double* eps,
                      double log_shrink, float* new_params, float* new_m, float* new_v,
                      void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------- spatial index */
/* Exact k-NN distances (cKDTree.query replacement; field.py:111-161,279-289):
 * for every query the k smallest Euclidean distances to the pool, ascending,
 * +inf when the pool has fewer points.  float64, dense uniform grid:
 * grid = HOST {bmin x, y, z, cell size} covering pool AND queries, dims = HOST
 * {nx, ny, nz} (<= 2^26 cells); 1 <= k <= 8. */
int ssr_knn_workspace(int64_t n_pool, int64_t n_cells, int64_t* bytes);
int ssr_knn(const double* pool, int64_t n_pool, const double* queries, int64_t n_q, int32_t k,
            const double* grid, const int32_t* dims, double* out_dist, void* workspace,
            int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------- field snapshot */
/* io/ply.py:29-124: the flat float32 parameter buffer <-> PLY vertex records,
 * n x ssr_ply_properties(deg) doubles in property order x y z nx ny nz
 * f_dc_0..2 f_rest_* (channel-major) opacity scale_0..2 rot_0..3.  Pack widens
 * exactly (bit-exact round trip); unpack rounds to nearest float32.  Device
 * pointers; the host writes / parses the header (paper_2503_13086_b200/ply.py). */
int32_t ssr_ply_properties(int32_t sh_degree);
int ssr_ply_pack(int64_t n, int32_t sh_degree, const float* params, double* records, void* stream);
int ssr_ply_unpack(int64_t n, int32_t sh_degree, const double* records, float* params, void* stream);

/* ---------------------------------------------------------- loss */
/* losses.py:55-173: w_l1 * L1 + w_ssim * (1 - SSIM) + w_load * std(soft).
 * target: H x W x 3 float32 in [0, 1], or 8-bit (target_u8 != 0; value / 255,
 * like the reference's image loader io/images.py).
 * Writes d_image (HxWx3), d_soft (HxW) and out[5] = (l1, ssim_loss, load,
 * total, hard_count_std) as float64 in device memory.  soft_count may be NULL
 * when w_load == 0 and d_soft == NULL (a render without soft counts).
 * workspace: ssr_loss_workspace() bytes of device memory, 16-byte aligned
 * (its adjoint maps are read back by TMA). */
int ssr_loss_workspace(int32_t width, int32_t height, int64_t* bytes);
int ssr_loss(int32_t width, int32_t height, const float* image, const void* target, int32_t target_u8,
             const double* soft_count, const int32_t* hard_count, double w_l1, double w_ssim,
             double w_load, float* d_image, float* d_soft, double* out, void* workspace,
             int64_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSR_H */
