// Stage 2: tile-key duplication, prefix scan and the (tile, depth) sort
// (rasterize/projection.py:165-191), as a depth pre-sort + stable tile sort:
//
//  1. the N Gaussians are radix-sorted by a 24-bit monotone key of
//     fp32(depth64) (culled rows keyed last); runs of equal keys are
//     re-ordered by (fp64 depth, field row).  Rounding and the key map are
//     monotone, so this is exactly the reference's fp64 depth order with
//     row-index tie-break;
//  2. tiles-touched counts are scanned in that order, so every Gaussian's
//     instances are emitted at depth-ordered positions (splats.offset);
//  3. one stable LSD radix sort over the tile id alone (ceil(log2 n_tiles)
//     bits) turns the depth-ordered instance list into (tile, depth, row)
//     order -- np.lexsort((depth, tile)) over splat-major instances;
//  4. searchsorted tile ranges from the sorted tile ids.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ssr_common.cuh"

namespace ssr {

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// 24-bit depth keys (3 radix passes instead of 4): the fp32 bit pattern of a
// kept depth (> ZNEAR > 0, so monotone in the depth) minus that of ZNEAR,
// shifted right by DEPTH_KEY_SHIFT (16 consecutive fp32 depths per key, ~1e-6
// relative) and clamped below the culled key.  The mapping is monotone, so
// equal-key runs only need re-ordering by (fp64 depth, row): k_depth_tiefix.
constexpr int DEPTH_KEY_BITS = 24;
constexpr int DEPTH_KEY_SHIFT = 4;
constexpr uint32_t DEPTH_KEY_CULLED = (1u << DEPTH_KEY_BITS) - 1u;

// The per-Gaussian passes below handle BIN_PER elements per thread, block-
// strided (each step coalesced across the warp), so several independent
// loads are in flight per thread.
constexpr int BIN_PER = 4;
constexpr int BIN_THREADS = 256;

__global__ void __launch_bounds__(BIN_THREADS) k_depth_keys(int64_t n, const uint32_t* __restrict__ tiles,
                                                            const double* __restrict__ depth,
                                                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t base = (int64_t)blockIdx.x * BIN_THREADS * BIN_PER + threadIdx.x;
  uint32_t t[BIN_PER];
  double d[BIN_PER];
#pragma unroll
  for (int k = 0; k < BIN_PER; k++) {
    const int64_t i = base + k * BIN_THREADS;
    t[k] = i < n ? tiles[i] : 0u;
    d[k] = i < n ? depth[i] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < BIN_PER; k++) {
    const int64_t i = base + k * BIN_THREADS;
    if (i >= n) break;
    uint32_t key = DEPTH_KEY_CULLED;
    if (t[k]) {
      const uint32_t b = __float_as_uint(__double2float_rn(d[k])) - __float_as_uint((float)ZNEAR);
      key = min(b >> DEPTH_KEY_SHIFT, DEPTH_KEY_CULLED - 1u);
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

// Runs of equal fp32 depth keys: re-ordered by fp64 depth (stable, so equal
// fp64 depths keep field-row order).  Also gathers the tile counts in depth
// order (cnt[s] = tiles[order[s]]) once each position's entry is final: a
// run's head writes the whole run after sorting it.  Runs of up to TIE_MAX
// (nearly all) are loaded with independent loads and sorted in registers
// (stable bubble network); longer ones fall back to an insertion sort in
// place.
constexpr int TIE_MAX = 8;

__device__ __noinline__ void tiefix_long_run(int64_t s, int64_t n, uint32_t key, const uint32_t* __restrict__ keys,
                                             uint32_t* __restrict__ order, const double* __restrict__ depth,
                                             const uint32_t* __restrict__ tiles, uint32_t* __restrict__ cnt) {
  int64_t e = s + 1;
  while (e < n && keys[e] == key) e++;
  for (int64_t a = s + 1; a < e; a++) {
    const uint32_t v = order[a];
    const double d = depth[v];
    int64_t b = a - 1;
    while (b >= s && depth[order[b]] > d) {
      order[b + 1] = order[b];
      b--;
    }
    order[b + 1] = v;
  }
  for (int64_t a = s; a < e; a++) cnt[a] = tiles[order[a]];
}

__global__ void __launch_bounds__(256) k_depth_tiefix(int64_t n, const uint32_t* __restrict__ keys,
                                                      uint32_t* __restrict__ order, const double* __restrict__ depth,
                                                      const uint32_t* __restrict__ tiles, uint32_t* __restrict__ cnt) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t key = keys[s];
  const bool head = (s == 0) || (keys[s - 1] != key);
  if (key == DEPTH_KEY_CULLED || !head || s + 1 >= n || keys[s + 1] != key) {
    if (key == DEPTH_KEY_CULLED || head) cnt[s] = tiles[order[s]];  // culled or a run of one
    return;
  }
  // run length (>= 2): the next TIE_MAX keys at once
  uint32_t kk[TIE_MAX];
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++) kk[j] = s + 1 + j < n ? keys[s + 1 + j] : UINT32_MAX;
  int len = 1;
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++)
    if (len == j + 1 && kk[j] == key) len++;
  if (len > TIE_MAX) {
    tiefix_long_run(s, n, key, keys, order, depth, tiles, cnt);
    return;
  }
  uint32_t o[TIE_MAX];
  double d[TIE_MAX];
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++) o[j] = j < len ? order[s + j] : 0u;
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++) d[j] = j < len ? depth[o[j]] : __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
  for (int i = 0; i < TIE_MAX - 1; i++)
#pragma unroll
    for (int j = 0; j < TIE_MAX - 1 - i; j++)
      if (d[j] > d[j + 1]) {
        const double td = d[j];
        d[j] = d[j + 1];
        d[j + 1] = td;
        const uint32_t to = o[j];
        o[j] = o[j + 1];
        o[j + 1] = to;
      }
  uint32_t tc[TIE_MAX];
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++) tc[j] = j < len ? tiles[o[j]] : 0u;
#pragma unroll
  for (int j = 0; j < TIE_MAX; j++)
    if (j < len) {
      order[s + j] = o[j];
      cnt[s + j] = tc[j];
    }
}

__global__ void __launch_bounds__(256) k_scatter_offsets(int64_t n, const uint32_t* __restrict__ order,
                                                         const uint32_t* __restrict__ cnt,
                                                         const uint32_t* __restrict__ off_sorted,
                                                         uint32_t* __restrict__ offset, uint32_t* __restrict__ total,
                                                         uint32_t* __restrict__ depth_order) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t g = order[r];
  offset[g] = off_sorted[r];
  if (depth_order) depth_order[r] = g;
  if (r == n - 1) *total = off_sorted[r] + cnt[r];
}

__global__ void k_zero_total(uint32_t* total) {
  if (threadIdx.x == 0) *total = 0u;
}

// Every field row writes its tiles at its depth-ordered offset; emission order
// inside a row is ty-outer / tx-inner (projection.py:175-182).  Two roles per
// thread r:
//  * small Gaussians (<= DUP_SMALL tiles) in depth order (depth_order[r]): a
//    warp's 32 consecutive ranks own (up to the large ones among them) one
//    contiguous output range, so the warp enumerates its small instances
//    k = 0 .. sum-1 (lane-order prefix of the counts, 5-step shuffle search)
//    and lanes write consecutive slots: coalesced stores;
//  * large Gaussians in field-row order (row r): written by the whole warp,
//    lane-strided over the Gaussian's own contiguous range.  Field order
//    spreads adjacent-in-depth large splats over different warps.
constexpr uint32_t DUP_SMALL = 32;

__global__ void __launch_bounds__(256) k_duplicate(int64_t n, int tiles_x, const uint32_t* __restrict__ tiles,
                                                   const uint32_t* __restrict__ offset, const int4* __restrict__ rect,
                                                   const uint32_t* __restrict__ order, uint32_t* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const unsigned FULLM = 0xffffffffu;
  // ---- small Gaussians, depth order
  {
    uint32_t g = 0, cnt = 0, off = 0;
    int4 rc = make_int4(0, 0, 1, 1);
    if (r < n) {
      g = order[r];
      cnt = tiles[g];
      if (cnt > DUP_SMALL) cnt = 0;  // written by the field-order role
      if (cnt) {
        off = offset[g];
        rc = rect[g];
      }
    }
    uint32_t incl = cnt;  // inclusive prefix of the small counts in lane order
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(FULLM, incl, d);
      if (lane >= d) incl += o;
    }
    const uint32_t total = __shfl_sync(FULLM, incl, 31);
    const uint32_t excl = incl - cnt;
    const uint32_t w = (uint32_t)(rc.z - rc.x);
    for (uint32_t k0 = 0; k0 < total; k0 += 32) {
      const uint32_t k = k0 + lane;
      // last lane whose exclusive prefix <= k (for k < total that lane has a
      // nonzero count: a zero-count lane shares its prefix with the next lane)
      int src = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t e = __shfl_sync(FULLM, excl, src + step);
        if (e <= k) src += step;
      }
      const uint32_t se = __shfl_sync(FULLM, excl, src), so = __shfl_sync(FULLM, off, src);
      const uint32_t sw = __shfl_sync(FULLM, w, src), sg = __shfl_sync(FULLM, g, src);
      const int sx = __shfl_sync(FULLM, rc.x, src), sy = __shfl_sync(FULLM, rc.y, src);
      if (k < total) {
        const uint32_t q = k - se;  // < 32: q / sw from a float reciprocal is exact
        const uint32_t row = __float2uint_rz(((float)q + 0.5f) * __frcp_rn((float)sw));
        keys[so + q] = ((uint32_t)sy + row) * (uint32_t)tiles_x + (uint32_t)sx + (q - row * sw);
        vals[so + q] = sg;
      }
    }
  }
  // ---- large Gaussians, field-row order, warp-cooperative
  const uint32_t nt = r < n ? tiles[r] : 0u;
  unsigned big = __ballot_sync(FULLM, nt > DUP_SMALL);
  while (big) {
    const int l = __ffs(big) - 1;
    big &= big - 1;
    const int64_t g = r - lane + l;
    const int4 rc = rect[g];
    const uint32_t o = offset[g];
    const uint32_t w = (uint32_t)(rc.z - rc.x), cnt = __shfl_sync(FULLM, nt, l);
    // (row, col) of instance j = lane + 32 i advanced incrementally (no division per instance)
    uint32_t row = (uint32_t)lane / w, col = (uint32_t)lane - row * w;
    const uint32_t drow = 32u / w, dcol = 32u - drow * w;
    uint32_t key = ((uint32_t)rc.y + row) * (uint32_t)tiles_x + (uint32_t)rc.x + col;
    for (uint32_t j = lane; j < cnt; j += 32) {
      keys[o + j] = key;
      vals[o + j] = (uint32_t)g;
      col += dcol;
      row += drow;
      if (col >= w) {
        col -= w;
        row++;
      }
      key = ((uint32_t)rc.y + row) * (uint32_t)tiles_x + (uint32_t)rc.x + col;
    }
  }
}

// searchsorted(left/right) for every tile id from the sorted tile keys;
// RANGE_KEYS consecutive keys per thread.
constexpr int RANGE_KEYS = 8;

__global__ void __launch_bounds__(256) k_ranges(int64_t m, int n_tiles, const uint32_t* __restrict__ keys,
                                                int32_t* __restrict__ ranges) {
  const int64_t s0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * RANGE_KEYS;
  if (s0 >= m) return;
  int prev = s0 > 0 ? (int)keys[s0 - 1] : -1;
  uint32_t kk[RANGE_KEYS];
#pragma unroll
  for (int j = 0; j < RANGE_KEYS; j++) kk[j] = s0 + j < m ? keys[s0 + j] : 0u;
#pragma unroll
  for (int j = 0; j < RANGE_KEYS; j++) {
    const int64_t s = s0 + j;
    if (s >= m) break;
    const int tile = (int)kk[j];
    if (tile != prev) {
      for (int t = prev + 1; t <= tile; t++) ranges[2 * t] = (int32_t)s;
      for (int t = prev < 0 ? 0 : prev; t < tile; t++) ranges[2 * t + 1] = (int32_t)s;
    }
    if (s == m - 1) {
      for (int t = tile + 1; t < n_tiles; t++) ranges[2 * t] = (int32_t)m;
      for (int t = tile; t < n_tiles; t++) ranges[2 * t + 1] = (int32_t)m;
    }
    prev = tile;
  }
}

static int tile_bits(int n_tiles) {
  int b = 1;
  while ((1LL << b) < (long long)n_tiles) b++;
  return b;
}

static size_t sort32_temp_bytes(int64_t m, int end_bit) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(m > 0 ? m : 1), 0, end_bit);
  return bytes;
}

static size_t scan_temp_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum((void*)nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)(n > 0 ? n : 1));
  return b;
}

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_scan_workspace(int64_t n, int64_t* bytes) {
  const int64_t a = align_up(4 * (n > 0 ? n : 1), 256);
  *bytes = 6 * a + align_up((int64_t)sort32_temp_bytes(n, 32), 256) + align_up((int64_t)scan_temp_bytes(n), 256);
  return SSR_OK;
}

extern "C" int ssr_scan_tiles(int64_t n, ssr_splats splats, void* workspace, int64_t workspace_bytes,
                              uint32_t* total_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n > INT32_MAX) {
    set_error("ssr_scan_tiles: n out of range");
    return SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_scan_workspace(n, &need);
  if (workspace_bytes < need) {
    set_error("ssr_scan_tiles: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (n == 0) {
    k_zero_total<<<1, 32, 0, st>>>(total_dev);
    return check_launch("k_zero_total");
  }
  const int64_t a = align_up(4 * n, 256);
  char* w = (char*)workspace;
  uint32_t* keys_in = (uint32_t*)w;
  uint32_t* keys_out = (uint32_t*)(w + a);
  uint32_t* vals_in = (uint32_t*)(w + 2 * a);
  uint32_t* order = (uint32_t*)(w + 3 * a);
  uint32_t* cnt = (uint32_t*)(w + 4 * a);
  uint32_t* off_sorted = (uint32_t*)(w + 5 * a);
  char* temp = w + 6 * a;
  const unsigned blocks = (unsigned)((n + BIN_THREADS * BIN_PER - 1) / (BIN_THREADS * BIN_PER));
  k_depth_keys<<<blocks, BIN_THREADS, 0, st>>>(n, splats.tiles, splats.depth, keys_in, vals_in);
  SSR_TRY(check_launch("k_depth_keys"));
  size_t tb = sort32_temp_bytes(n, DEPTH_KEY_BITS);
  SSR_TRY(check_cuda(cub::DeviceRadixSort::SortPairs((void*)temp, tb, keys_in, keys_out, vals_in, order, (int)n, 0,
                                                     DEPTH_KEY_BITS, st),
                     "depth sort"));
  const unsigned blocks1 = (unsigned)((n + 255) / 256);
  k_depth_tiefix<<<blocks1, 256, 0, st>>>(n, keys_out, order, splats.depth, splats.tiles, cnt);
  SSR_TRY(check_launch("k_depth_tiefix"));
  size_t sb = scan_temp_bytes(n);
  SSR_TRY(check_cuda(cub::DeviceScan::ExclusiveSum((void*)temp, sb, cnt, off_sorted, (int)n, st), "scan tiles"));
  k_scatter_offsets<<<blocks1, 256, 0, st>>>(n, order, cnt, off_sorted, splats.offset, total_dev,
                                            splats.depth_order);
  SSR_TRY(check_launch("k_scatter_offsets"));
  // gradient-row offsets in field-row order (contiguous per block of rows for the chain)
  size_t sb2 = scan_temp_bytes(n);
  return check_cuda(cub::DeviceScan::ExclusiveSum((void*)temp, sb2, splats.tiles, splats.row_offset, (int)n, st),
                    "row-order scan");
}

extern "C" int ssr_bin_workspace(int64_t m, int32_t n_tiles, int64_t* bytes) {
  const int64_t a = align_up(4 * (m > 0 ? m : 1), 256);
  *bytes = 3 * a + align_up((int64_t)sort32_temp_bytes(m, tile_bits(n_tiles > 0 ? n_tiles : 1)), 256);
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
  const int64_t a = align_up(4 * m, 256);
  char* w = (char*)workspace;
  uint32_t* keys_in = (uint32_t*)w;
  uint32_t* keys_out = (uint32_t*)(w + a);
  uint32_t* vals_in = (uint32_t*)(w + 2 * a);
  const int bits = tile_bits(n_tiles);
  size_t temp = sort32_temp_bytes(m, bits);
  if (!splats.depth_order) {
    set_error("ssr_bin_tiles: splats.depth_order (from ssr_scan_tiles) is required");
    return SSR_ERR_INVALID;
  }
  k_duplicate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, tiles_x, splats.tiles, splats.offset,
                                                           (const int4*)splats.rect, splats.depth_order, keys_in,
                                                           vals_in);
  SSR_TRY(check_launch("k_duplicate"));
  SSR_TRY(check_cuda(cub::DeviceRadixSort::SortPairs((void*)(w + 3 * a), temp, keys_in, keys_out, vals_in, inst_gauss,
                                                     (int)m, 0, bits, st),
                     "tile sort"));
  const int64_t rthreads = (m + RANGE_KEYS - 1) / RANGE_KEYS;
  k_ranges<<<(unsigned)((rthreads + 255) / 256), 256, 0, st>>>(m, n_tiles, keys_out, tile_ranges);
  return check_launch("k_ranges");
}

extern "C" int ssr_bin_tiles_capacity(int64_t n, int64_t capacity, int32_t tiles_x, int32_t tiles_y,
                                      ssr_splats splats, const uint32_t* total_dev, int64_t* m_out,
                                      uint32_t* inst_gauss, int32_t* tile_ranges, void* workspace,
                                      int64_t workspace_bytes, void* stream) {
  if (!total_dev || !m_out) {
    set_error("ssr_bin_tiles_capacity: total_dev and m_out are required");
    return SSR_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // one pinned word per host thread for the instance total
  static thread_local uint32_t* host_total = nullptr;
  if (!host_total) SSR_TRY(check_cuda(cudaMallocHost(&host_total, sizeof(uint32_t)), "pinned total"));
  SSR_TRY(check_cuda(cudaMemcpyAsync(host_total, total_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, st),
                     "instance total"));
  SSR_TRY(check_cuda(cudaStreamSynchronize(st), "instance total"));
  const int64_t m = (int64_t)*host_total;
  *m_out = m;
  if (m > capacity) {
    set_error("ssr_bin_tiles_capacity: instance count exceeds the capacity");
    return SSR_ERR_CAPACITY;
  }
  return ssr_bin_tiles(n, m, tiles_x, tiles_y, splats, m ? inst_gauss : nullptr, tile_ranges, workspace,
                       workspace_bytes, stream);
}

extern "C" int64_t ssr_ckpt_floats(int64_t m, int32_t n_tiles) {
  return (m / BUCKET + (int64_t)n_tiles + 1) * TILE_PX * 4;
}
