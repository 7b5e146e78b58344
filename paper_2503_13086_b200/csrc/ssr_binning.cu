// Stage 2: tile-key duplication, prefix scan, 64-bit (tile, depth) radix
// sort, tie-fix and searchsorted tile ranges (rasterize/projection.py:165-191).
//
// Key = (tile << 32) | float_bits(fp32(depth64)).  fp64 -> fp32 rounding is
// monotone, so the fp32 key never inverts the reference's fp64 order; it can
// only create ties, which the tie-fix pass re-orders by (fp64 depth, field
// row).  The radix sort is stable and instances are emitted in field-row
// order, which is exactly the reference's np.lexsort tie-break.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ssr_common.cuh"

namespace ssr {

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

__global__ void k_scan_total(int64_t n, const uint32_t* tiles, const uint32_t* offset, uint32_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *total = n ? offset[n - 1] + tiles[n - 1] : 0u;
}

// One thread per field row writes its tiles.  Emission order inside a row is
// ty-outer / tx-inner (projection.py:175-182).
__global__ void __launch_bounds__(256) k_duplicate(int64_t n, int tiles_x, const uint32_t* __restrict__ tiles,
                                                   const uint32_t* __restrict__ offset,
                                                   const int4* __restrict__ rect, const double* __restrict__ depth,
                                                   unsigned long long* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t nt = tiles[i];
  if (nt == 0) return;
  const int4 r = rect[i];
  const unsigned long long dbits = (unsigned long long)__float_as_uint(__double2float_rn(depth[i]));
  uint32_t o = offset[i];
  for (int ty = r.y; ty < r.w; ty++) {
    const unsigned long long row = (unsigned long long)ty * tiles_x;
    for (int tx = r.x; tx < r.z; tx++) {
      keys[o] = ((row + tx) << 32) | dbits;
      vals[o] = (uint32_t)i;
      o++;
    }
  }
}

// Tie-fix + searchsorted ranges, one thread per sorted instance.
__global__ void __launch_bounds__(256) k_tiefix_ranges(int64_t m, int n_tiles,
                                                       const unsigned long long* __restrict__ keys,
                                                       uint32_t* __restrict__ vals, const double* __restrict__ depth,
                                                       int32_t* __restrict__ ranges) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  const unsigned long long key = keys[s];
  const int tile = (int)(key >> 32);
  const int prev = s > 0 ? (int)(keys[s - 1] >> 32) : -1;
  // searchsorted(left) start of every tile in (prev, tile]; searchsorted(right)
  // end of every tile in [prev, tile)
  if (tile != prev) {
    for (int t = prev + 1; t <= tile; t++) ranges[2 * t] = (int32_t)s;
    for (int t = prev < 0 ? 0 : prev; t < tile; t++) ranges[2 * t + 1] = (int32_t)s;
  }
  if (s == m - 1) {
    for (int t = tile + 1; t < n_tiles; t++) ranges[2 * t] = (int32_t)m;
    for (int t = tile; t < n_tiles; t++) ranges[2 * t + 1] = (int32_t)m;
  }
  // tie-fix: the head of a run of equal keys insertion-sorts it by fp64 depth
  // (stable, so equal fp64 depths stay in field-row order)
  const bool head = (s == 0) || (keys[s - 1] != key);
  if (head && s + 1 < m && keys[s + 1] == key) {
    int64_t e = s + 1;
    while (e < m && keys[e] == key) e++;
    for (int64_t a = s + 1; a < e; a++) {
      const uint32_t v = vals[a];
      const double d = depth[v];
      int64_t b = a - 1;
      while (b >= s && depth[vals[b]] > d) {
        vals[b + 1] = vals[b];
        b--;
      }
      vals[b + 1] = v;
    }
  }
}

static int tile_bits(int n_tiles) {
  int b = 0;
  while ((1LL << b) < (long long)n_tiles) b++;
  return b;
}

static size_t sort_temp_bytes(int64_t m, int n_tiles) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (int)(m > 0 ? m : 1), 0, 32 + tile_bits(n_tiles));
  return bytes;
}

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_scan_workspace(int64_t n, int64_t* bytes) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)(n > 0 ? n : 1));
  *bytes = (int64_t)b;
  return SSR_OK;
}

extern "C" int ssr_scan_tiles(int64_t n, ssr_splats splats, void* workspace, int64_t workspace_bytes,
                              uint32_t* total_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n > INT32_MAX) {
    set_error("ssr_scan_tiles: n out of range");
    return SSR_ERR_INVALID;
  }
  if (n > 0) {
    size_t b = (size_t)workspace_bytes;
    SSR_TRY(check_cuda(cub::DeviceScan::ExclusiveSum(workspace, b, splats.tiles, splats.offset, (int)n, st),
                       "scan tiles"));
  }
  k_scan_total<<<1, 32, 0, st>>>(n, splats.tiles, splats.offset, total_dev);
  return check_launch("k_scan_total");
}

extern "C" int ssr_bin_workspace(int64_t m, int32_t n_tiles, int64_t* bytes) {
  int64_t b = 0;
  b += align_up(8 * (m > 0 ? m : 1), 256);  // keys in
  b += align_up(8 * (m > 0 ? m : 1), 256);  // keys out
  b += align_up(4 * (m > 0 ? m : 1), 256);  // vals in
  b += align_up((int64_t)sort_temp_bytes(m, n_tiles), 256);
  *bytes = b;
  return SSR_OK;
}

extern "C" int ssr_bin_tiles(int64_t n, int64_t m, int32_t tiles_x, int32_t tiles_y, ssr_splats splats,
                             uint32_t* inst_gauss, int32_t* tile_ranges, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int n_tiles = tiles_x * tiles_y;
  if (n < 0 || m < 0 || m > INT32_MAX || n_tiles <= 0) {
    set_error("ssr_bin_tiles: invalid sizes (instance count must fit int32)");
    return m > INT32_MAX ? SSR_ERR_CAPACITY : SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_bin_workspace(m, n_tiles, &need);
  if (workspace_bytes < need) {
    set_error("ssr_bin_tiles: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (m == 0) {
    return check_cuda(cudaMemsetAsync(tile_ranges, 0, sizeof(int32_t) * 2 * n_tiles, st), "ranges memset");
  }
  char* w = (char*)workspace;
  unsigned long long* keys_in = (unsigned long long*)w;
  w += align_up(8 * m, 256);
  unsigned long long* keys_out = (unsigned long long*)w;
  w += align_up(8 * m, 256);
  uint32_t* vals_in = (uint32_t*)w;
  w += align_up(4 * m, 256);
  size_t temp = sort_temp_bytes(m, n_tiles);

  k_duplicate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, tiles_x, splats.tiles, splats.offset,
                                                           (const int4*)splats.rect, splats.depth, keys_in, vals_in);
  SSR_TRY(check_launch("k_duplicate"));
  SSR_TRY(check_cuda(cub::DeviceRadixSort::SortPairs((void*)w, temp, keys_in, keys_out, vals_in, inst_gauss, (int)m,
                                                     0, 32 + tile_bits(n_tiles), st),
                     "radix sort"));
  k_tiefix_ranges<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, n_tiles, keys_out, inst_gauss, splats.depth,
                                                               tile_ranges);
  return check_launch("k_tiefix_ranges");
}

extern "C" int64_t ssr_ckpt_floats(int64_t m, int32_t n_tiles) {
  return (m / BUCKET + (int64_t)n_tiles + 1) * TILE_PX * 4;
}
