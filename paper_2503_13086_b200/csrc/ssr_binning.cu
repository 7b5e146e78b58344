// Stage 2: tile-key duplication, prefix scans and the (tile, depth) sort
// (rasterize/projection.py:165-191), hand-written for sm_100a: no library
// sort or scan.  The order is built as a depth pre-sort followed by a stable
// tile sort:
//
//  1. the N Gaussians are sorted by a 24-bit monotone key of fp32(depth64)
//     (culled rows keyed last) with three stable 8-bit radix passes; runs of
//     equal keys are then re-ordered by (fp64 depth, field row).  Rounding and
//     the key map are monotone, so this is exactly the reference's fp64 depth
//     order with the row-index tie-break;
//  2. tiles-touched counts are scanned in that order, so every Gaussian's
//     instances are emitted at depth-ordered positions (splats.offset); the
//     same launches scan them in field-row order for the backward's
//     per-instance gradient rows (splats.row_offset) and yield M;
//  3. two stable 8-bit radix passes over the tile id alone (ceil(log2
//     n_tiles) <= 16 bits) turn the depth-ordered instance list into
//     (tile, depth, row) order -- np.lexsort((depth, tile)) over the
//     splat-major instance list;
//  4. searchsorted tile ranges from the sorted tile ids.
//
// Radix passes: reduce-then-scan per 8-bit digit (k_radix_up ->
// k_digit_scan -> k_radix_down, see below); no tile ever waits on another.
// The scans are summed in 64 bits (totals past the 2^30 instance limit are
// reported, never wrapped).
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
constexpr int DEPTH_PASSES = DEPTH_KEY_BITS / 8;
constexpr uint32_t DEPTH_KEY_CULLED = (1u << DEPTH_KEY_BITS) - 1u;
constexpr int TILE_PASSES = 2;  // tile ids up to 16 bits
// the radix look-back status words hold 30-bit counts
constexpr int64_t MAX_INSTANCES = (1LL << 30) - 1;

constexpr unsigned FULLM = 0xffffffffu;

__device__ __forceinline__ uint32_t depth_key(uint32_t tiles, double depth) {
  // branch-free, so the depth load is never made dependent on the tiles load
  const uint32_t b = __float_as_uint(__double2float_rn(depth)) - __float_as_uint((float)ZNEAR);
  const uint32_t k = min(b >> DEPTH_KEY_SHIFT, DEPTH_KEY_CULLED - 1u);
  return tiles ? k : DEPTH_KEY_CULLED;
}

// ---------------------------------------------------------------- radix passes
// One stable 8-bit LSD pass = three launches, reduce-then-scan (no look-back
// chains, so no tile waits on a predecessor):
//  k_radix_up:   per 4096-key tile, its digit counts -> counts[digit][tile];
//  k_digit_scan: per digit (one CTA each), exclusive scan over the tiles plus
//                the digit's bucket base (totals of the smaller digits);
//  k_radix_down: per tile, stable per-warp ranking (ballot-built peer masks,
//                items ranked in input order), staging in shared memory in
//                digit order, coalesced stores of each digit run.
constexpr int RX_THREADS = 512;
constexpr int RX_WARPS = RX_THREADS / 32;
constexpr int RX_ITEMS = 8;
constexpr int RX_TILE = RX_THREADS * RX_ITEMS;  // keys per CTA

// MODE 0: keys from an array.  MODE 1: depth keys made on the fly from
// (tiles, depth) of field row idx (pass 0 of the depth sort; values = row).
template <int MODE>
__device__ __forceinline__ uint32_t rx_key(int64_t idx, int64_t n, const uint32_t* __restrict__ keys_in,
                                           const uint32_t* __restrict__ tiles, const double* __restrict__ depth) {
  if (idx >= n) return 0u;
  if (MODE == 1) return depth_key(tiles[idx], depth[idx]);
  return keys_in[idx];
}

// Exclusive block-wide scan of one value per thread (RX_THREADS threads);
// returns the exclusive prefix, *total gets the sum.  `red` is RX_WARPS
// shared words.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* red, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(FULLM, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  uint32_t wbase = 0, sum = 0;
#pragma unroll
  for (int w = 0; w < RX_WARPS; w++) {
    const uint32_t r = red[w];
    if (w < warp) wbase += r;
    sum += r;
  }
  *total = sum;
  return wbase + incl - v;
}

// NB: bits of this pass's digit (<= 8; the tile sort splits its key's bits
// evenly over its passes, so no ballot or bucket is spent on bits that are
// always zero).
template <int MODE, int NB>
__global__ void __launch_bounds__(RX_THREADS) k_radix_up(int64_t n, int shift, const uint32_t* __restrict__ keys_in,
                                                         const uint32_t* __restrict__ tiles,
                                                         const double* __restrict__ depth,
                                                         uint32_t* __restrict__ counts,
                                                         uint32_t* __restrict__ hist, int n_ctas) {
  griddep_wait();
  __shared__ uint32_t s_hist[RX_WARPS][256];  // one histogram per warp: no cross-warp contention
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * RX_TILE + (int64_t)warp * (RX_ITEMS * 32) + lane;
  uint32_t key[RX_ITEMS];  // requested before the histogram set-up (latency overlap)
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) key[i] = rx_key<MODE>(base + i * 32, n, keys_in, tiles, depth);
  for (int i = threadIdx.x; i < RX_WARPS * 256; i += RX_THREADS) (&s_hist[0][0])[i] = 0u;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++)
    if (base + i * 32 < n) atomicAdd(&s_hist[warp][(key[i] >> shift) & ((1u << NB) - 1u)], 1u);
  __syncthreads();
  if (threadIdx.x < 256) {
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < RX_WARPS; w++) c += s_hist[w][threadIdx.x];
    counts[(size_t)threadIdx.x * n_ctas + blockIdx.x] = c;
    if (c) atomicAdd(&hist[threadIdx.x], c);
  }
}

// blockIdx.x = digit d: offsets[d][t] = (keys with a smaller digit: the
// pass histogram, accumulated by k_radix_up) + (digit-d keys in tiles < t).
__global__ void __launch_bounds__(RX_THREADS) k_digit_scan(const uint32_t* __restrict__ counts,
                                                           const uint32_t* __restrict__ hist, int n_ctas,
                                                           uint32_t* __restrict__ offsets) {
  griddep_wait();
  __shared__ uint32_t s_red[RX_WARPS];
  __shared__ uint32_t s_base;
  const int d = blockIdx.x;
  uint32_t tot;
  const uint32_t below = block_excl_scan(threadIdx.x < 256 ? hist[threadIdx.x] : 0u, s_red, &tot);
  if ((int)threadIdx.x == d) s_base = below;
  __syncthreads();
  uint32_t run = s_base;
  const uint32_t* c = counts + (size_t)d * n_ctas;
  uint32_t* o = offsets + (size_t)d * n_ctas;
  for (int t0 = 0; t0 < n_ctas; t0 += RX_THREADS) {
    __syncthreads();  // s_red reuse
    const int t = t0 + threadIdx.x;
    const uint32_t v = t < n_ctas ? c[t] : 0u;
    const uint32_t ex = block_excl_scan(v, s_red, &tot);
    if (t < n_ctas) o[t] = run + ex;
    run += tot;
  }
}

template <int MODE, int NB>
__global__ void __launch_bounds__(RX_THREADS, 2) k_radix_down(
    int64_t n, int shift, const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    const uint32_t* __restrict__ tiles, const double* __restrict__ depth, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ offsets, int n_ctas) {
  griddep_wait();
  constexpr uint32_t DMASK = (1u << NB) - 1u;
  __shared__ uint32_t s_keys[RX_TILE];
  __shared__ uint32_t s_vals[RX_TILE];
  __shared__ uint16_t s_whist[RX_WARPS][256];  // per-warp digit counts, then warp offsets (< 4096)
  __shared__ uint32_t s_start[256];  // first staged slot of each digit in this tile
  __shared__ uint32_t s_gbase[256];  // global slot of the tile's digit run minus s_start
  __shared__ uint32_t s_red[RX_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  // the tile's keys are requested first: their latency overlaps the setup
  const int64_t base = (int64_t)tile * RX_TILE + (int64_t)warp * (RX_ITEMS * 32) + lane;
  uint32_t key[RX_ITEMS];  // values are read again at staging time (cache hits), saving registers
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) key[i] = rx_key<MODE>(base + i * 32, n, keys_in, tiles, depth);
  for (int i = threadIdx.x; i < RX_WARPS * 256; i += RX_THREADS) (&s_whist[0][0])[i] = 0u;
  const uint32_t goff = threadIdx.x < 256 ? offsets[(size_t)threadIdx.x * n_ctas + tile] : 0u;
  __syncthreads();
  // ---- stable per-warp ranking (items in input order: item-major, lane-minor)
  const unsigned lt = (1u << lane) - 1u;
  uint32_t rank[RX_ITEMS];
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    const bool valid = base + i * 32 < n;
    const uint32_t d = (key[i] >> shift) & DMASK;
    unsigned peers = __ballot_sync(FULLM, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < NB; b++) {
      const unsigned bal = __ballot_sync(FULLM, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    uint32_t before = 0;
    if (valid) before = s_whist[warp][d];
    __syncwarp();
    const int leader = 31 - __clz(peers);
    if (valid && lane == leader) s_whist[warp][d] = (uint16_t)(before + __popc(peers));
    __syncwarp();
    rank[i] = before + __popc(peers & lt);
  }
  __syncthreads();
  // ---- per digit (thread = digit): exclusive offsets of the warps, tile count
  const int dg = threadIdx.x;
  uint32_t cnt = 0;
  if (dg < 256) {
#pragma unroll
    for (int w = 0; w < RX_WARPS; w++) {
      const uint32_t c = s_whist[w][dg];
      s_whist[w][dg] = (uint16_t)cnt;
      cnt += c;
    }
  }
  uint32_t tot;
  const uint32_t start = block_excl_scan(cnt, s_red, &tot);
  if (dg < 256) {
    s_start[dg] = start;
    s_gbase[dg] = goff - start;
  }
  __syncthreads();
  // ---- stage the tile in digit order: keys and their slot in the input tile
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    if (base + i * 32 < n) {
      const uint32_t d = (key[i] >> shift) & DMASK;
      const uint32_t pos = s_start[d] + s_whist[warp][d] + rank[i];
      s_keys[pos] = key[i];
      s_vals[pos] = (uint32_t)(warp * (RX_ITEMS * 32) + i * 32 + lane);
    }
  }
  __syncthreads();
  // ---- coalesced stores of each digit run; the values are gathered from the
  // tile's own 16 KB of input (L1/L2 hits), all loads of a thread in flight at once
  const int64_t tile0 = (int64_t)tile * RX_TILE;
  const int valid_n = (int)min((int64_t)RX_TILE, n - tile0);
  uint32_t kv[RX_ITEMS], vv[RX_ITEMS];
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    const int j = i * RX_THREADS + threadIdx.x;
    kv[i] = j < valid_n ? s_keys[j] : 0u;
    const uint32_t src = j < valid_n ? s_vals[j] : 0u;
    vv[i] = j < valid_n ? (MODE == 1 ? (uint32_t)(tile0 + src) : vals_in[tile0 + src]) : 0u;
  }
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    const int j = i * RX_THREADS + threadIdx.x;
    if (j < valid_n) {
      const uint32_t o = s_gbase[(kv[i] >> shift) & DMASK] + (uint32_t)j;
      keys_out[o] = kv[i];
      vals_out[o] = vv[i];
    }
  }
}

// ---------------------------------------------------------------- depth tie-fix
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
  griddep_wait();
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

// ---------------------------------------------------------------- the two scans
// Two independent exclusive scans of tile counts over 4096-item CTAs:
//  scan A (depth order): cnt[s] -> splats.offset[order[s]];
//  scan B (field-row order): tiles[i] -> splats.row_offset[i], and M.
// k_tile_sums writes each CTA's 64-bit sum; k_scan2's CTA t then sums the
// sums of CTAs < t itself (independent loads, no chain through the
// predecessors) and scans its items.  Blocks [0, n_per) scan A, the rest B.
__global__ void __launch_bounds__(RX_THREADS) k_tile_sums(int64_t n, const uint32_t* __restrict__ src,
                                                          uint64_t* __restrict__ sums,
                                                          unsigned long long* __restrict__ total) {
  griddep_wait();
  __shared__ uint64_t s_red[RX_WARPS];
  const int64_t base = (int64_t)blockIdx.x * RX_TILE + threadIdx.x;
  uint64_t v = 0;
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    const int64_t idx = base + i * RX_THREADS;
    if (idx < n) v += src[idx];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
#pragma unroll
    for (int w = 0; w < RX_WARPS; w++) t += s_red[w];
    sums[blockIdx.x] = t;
    if (total) atomicAdd(total, (unsigned long long)t);
  }
}

__global__ void __launch_bounds__(RX_THREADS) k_scan2(int64_t n, const uint32_t* __restrict__ cnt,
                                                      const uint32_t* __restrict__ order,
                                                      const uint32_t* __restrict__ tiles,
                                                      uint32_t* __restrict__ offset, uint32_t* __restrict__ row_offset,
                                                      const uint64_t* __restrict__ sums, int n_per) {
  griddep_wait();
  __shared__ uint64_t s_red[RX_WARPS];
  __shared__ uint64_t s_pre[RX_WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool a = (int)blockIdx.x < n_per;
  const int tile = a ? blockIdx.x : blockIdx.x - n_per;
  const uint64_t* my_sums = sums + (a ? 0 : n_per);
  // prefix of the preceding CTAs
  uint64_t pre = 0;
  for (int t = threadIdx.x; t < tile; t += RX_THREADS) pre += my_sums[t];
  // blocked: thread j owns items [tile*4096 + j*16, +16)
  const int64_t base = (int64_t)tile * RX_TILE + (int64_t)threadIdx.x * RX_ITEMS;
  const uint32_t* src = a ? cnt : tiles;
  uint32_t v[RX_ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    v[i] = base + i < n ? src[base + i] : 0u;
    sum += v[i];
  }
  uint64_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(FULLM, incl, d);
    if (lane >= d) incl += o;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(FULLM, pre, o);
  if (lane == 31) s_red[warp] = incl;
  if (lane == 0) s_pre[warp] = pre;
  __syncthreads();
  uint64_t wbase = 0, tile_sum = 0, prefix = 0;
#pragma unroll
  for (int w = 0; w < RX_WARPS; w++) {
    if (w < warp) wbase += s_red[w];
    tile_sum += s_red[w];
    prefix += s_pre[w];
  }
  uint64_t run = prefix + wbase + incl - sum;
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    const int64_t idx = base + i;
    if (idx < n) {
      if (a)
        offset[order[idx]] = (uint32_t)run;
      else
        row_offset[idx] = (uint32_t)run;
    }
    run += v[i];
  }
}

// ---------------------------------------------------------------- duplication
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
  griddep_wait();
  const int lane = threadIdx.x & 31;
  {
    const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
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
          const uint32_t key = ((uint32_t)sy + row) * (uint32_t)tiles_x + (uint32_t)sx + (q - row * sw);
          keys[so + q] = key;
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
}

// searchsorted(left/right) for every tile id from the sorted tile keys;
// RANGE_KEYS consecutive keys per thread.
constexpr int RANGE_KEYS = 8;

__global__ void __launch_bounds__(256) k_ranges(int64_t m, int n_tiles, const uint32_t* __restrict__ keys,
                                                int32_t* __restrict__ ranges) {
  griddep_wait();
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

static inline int64_t rx_ctas(int64_t n) { return (n + RX_TILE - 1) / RX_TILE; }

// The instance total M of the last ssr_scan_tiles of this host thread: stored
// by a one-thread kernel straight into mapped pinned host memory right after
// it is computed, with an event behind it.  No copy engine is involved, so the
// read cannot queue behind a caller's host-to-device uploads (an 8-bit target
// frame in flight delayed a cudaMemcpyAsync of these 8 bytes by ~20 us).
__global__ void k_publish_total(const uint64_t* __restrict__ total_dev, volatile uint64_t* host) {
  griddep_wait();
  if (threadIdx.x == 0) {
    *host = *total_dev;
    __threadfence_system();
  }
}

struct PendingTotal {
  uint64_t* host = nullptr;
  uint64_t* host_dev = nullptr;  // device alias of the mapped host word
  cudaEvent_t ev = nullptr;
  const uint64_t* dev = nullptr;
  int device = -1;
  bool armed = false;
};

static PendingTotal& pending_total() {
  static thread_local PendingTotal pt;
  return pt;
}

static int arm_pending_total(const uint64_t* total_dev, cudaStream_t st) {
  PendingTotal& pt = pending_total();
  int dev = 0;
  SSR_TRY(check_cuda(cudaGetDevice(&dev), "cudaGetDevice"));
  if (!pt.host) {
    SSR_TRY(check_cuda(cudaHostAlloc(&pt.host, sizeof(uint64_t), cudaHostAllocMapped | cudaHostAllocPortable),
                       "mapped total"));
    SSR_TRY(check_cuda(cudaHostGetDevicePointer(&pt.host_dev, pt.host, 0), "mapped total"));
  }
  if (pt.ev && pt.device != dev) {
    cudaEventDestroy(pt.ev);
    pt.ev = nullptr;
  }
  if (!pt.ev) SSR_TRY(check_cuda(cudaEventCreateWithFlags(&pt.ev, cudaEventDisableTiming), "total event"));
  pt.device = dev;
  SSR_TRY(launch_pdl("k_publish_total", k_publish_total, dim3(1), dim3(32), 0, st, total_dev,
                     (volatile uint64_t*)pt.host_dev));
  SSR_TRY(check_cuda(cudaEventRecord(pt.ev, st), "total event record"));
  pt.dev = total_dev;
  pt.armed = true;
  return SSR_OK;
}

// One stable radix pass: counts -> digit scan -> ranked scatter.
template <int MODE, int NB>
static int radix_pass(int64_t n, int shift, const uint32_t* keys_in, const uint32_t* vals_in, const uint32_t* tiles,
                      const double* depth, uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts,
                      uint32_t* offsets, uint32_t* hist, cudaStream_t st) {
  const int ctas = (int)rx_ctas(n);
  SSR_TRY(launch_pdl("k_radix_up", k_radix_up<MODE, NB>, dim3(ctas), dim3(RX_THREADS), 0, st, n, shift, keys_in,
                     tiles, depth, counts, hist, ctas));
  SSR_TRY(launch_pdl("k_digit_scan", k_digit_scan, dim3(1u << NB), dim3(RX_THREADS), 0, st, (const uint32_t*)counts,
                     (const uint32_t*)hist, ctas, offsets));
  return launch_pdl("k_radix_down", k_radix_down<MODE, NB>, dim3(ctas), dim3(RX_THREADS), 0, st, n, shift, keys_in,
                    vals_in, tiles, depth, keys_out, vals_out, (const uint32_t*)offsets, ctas);
}

// A tile-sort pass over nb (1..8) digit bits.
static int tile_pass(int nb, int64_t m, int shift, const uint32_t* keys_in, const uint32_t* vals_in,
                     uint32_t* keys_out, uint32_t* vals_out, uint32_t* counts, uint32_t* offsets, uint32_t* hist,
                     cudaStream_t st) {
#define SSR_TP(B)                                                                                              \
  case B:                                                                                                      \
    return radix_pass<0, B>(m, shift, keys_in, vals_in, nullptr, nullptr, keys_out, vals_out, counts, offsets, \
                            hist, st)
  switch (nb) {
    SSR_TP(1);
    SSR_TP(2);
    SSR_TP(3);
    SSR_TP(4);
    SSR_TP(5);
    SSR_TP(6);
    SSR_TP(7);
    default: SSR_TP(8);
  }
#undef SSR_TP
}

// scan workspace: [zeroed: hist 3 x 256 u32] [counts 256 x ctas | offsets 256 x ctas u32 | sums 2 x ctas u64]
//                 [keys_a | vals_a | keys_b | cnt]  (N u32 each)
struct ScanLayout {
  int64_t ctas, zero_bytes, counts, offsets, sums, keys_a, vals_a, keys_b, cnt, bytes;
};

static ScanLayout scan_layout(int64_t n) {
  ScanLayout L;
  const int64_t nn = n > 0 ? n : 1;
  L.ctas = rx_ctas(nn);
  L.zero_bytes = align_up(4 * DEPTH_PASSES * 256, 256);
  L.counts = L.zero_bytes;
  L.offsets = align_up(L.counts + 4 * 256 * L.ctas, 256);
  L.sums = align_up(L.offsets + 4 * 256 * L.ctas, 256);
  const int64_t a = align_up(4 * nn, 256);
  L.keys_a = align_up(L.sums + 8 * 2 * L.ctas, 256);
  L.vals_a = L.keys_a + a;
  L.keys_b = L.vals_a + a;
  L.cnt = L.keys_b + a;
  L.bytes = L.cnt + a;
  return L;
}

// bin workspace: [zeroed: hist 2 x 256] [counts | offsets 256 x ctas] [keys_a | vals_a | keys_b | vals_b] (M u32)
struct BinLayout {
  int64_t ctas, zero_bytes, counts, offsets, keys_a, vals_a, keys_b, vals_b, bytes;
};

static BinLayout bin_layout(int64_t m) {
  BinLayout L;
  const int64_t mm = m > 0 ? m : 1;
  L.ctas = rx_ctas(mm);
  L.zero_bytes = align_up(4 * TILE_PASSES * 256, 256);
  L.counts = L.zero_bytes;
  L.offsets = align_up(L.counts + 4 * 256 * L.ctas, 256);
  const int64_t a = align_up(4 * mm, 256);
  L.keys_a = align_up(L.offsets + 4 * 256 * L.ctas, 256);
  L.vals_a = L.keys_a + a;
  L.keys_b = L.vals_a + a;
  L.vals_b = L.keys_b + a;
  L.bytes = L.vals_b + a;
  return L;
}

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_scan_workspace(int64_t n, int64_t* bytes) {
  *bytes = scan_layout(n).bytes;
  return SSR_OK;
}

extern "C" int ssr_scan_tiles(int64_t n, ssr_splats splats, void* workspace, int64_t workspace_bytes,
                              uint64_t* total_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n > INT32_MAX) {
    set_error("ssr_scan_tiles: n out of range");
    return SSR_ERR_INVALID;
  }
  const ScanLayout L = scan_layout(n);
  if (workspace_bytes < L.bytes || !splats.depth_order || !splats.offset || !splats.row_offset) {
    set_error("ssr_scan_tiles: workspace too small or splats.offset / row_offset / depth_order missing");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return check_cuda(cudaMemsetAsync(total_dev, 0, sizeof(uint64_t), st), "total memset");
  char* w = (char*)workspace;
  uint32_t* hist = (uint32_t*)w;
  uint32_t* counts = (uint32_t*)(w + L.counts);
  uint32_t* offsets = (uint32_t*)(w + L.offsets);
  uint64_t* sums = (uint64_t*)(w + L.sums);
  uint32_t* keys_a = (uint32_t*)(w + L.keys_a);
  uint32_t* vals_a = (uint32_t*)(w + L.vals_a);
  uint32_t* keys_b = (uint32_t*)(w + L.keys_b);
  uint32_t* cnt = (uint32_t*)(w + L.cnt);
  SSR_TRY(launch_pdl("scan workspace zero", k_zero_words, dim3(1), dim3(256), 0, st, (uint32_t*)w,
                     (int64_t)(L.zero_bytes / 4)));
  SSR_TRY(launch_pdl("total zero", k_zero_words, dim3(1), dim3(32), 0, st, (uint32_t*)total_dev, (int64_t)2));
  const int ctas = (int)L.ctas;
  // M first (field-row tile sums, summed into *total_dev), then its copy to
  // the host and an event: the host waits for M (ssr_bin_tiles_capacity) while
  // the device runs the depth sort queued behind the event
  SSR_TRY(launch_pdl("k_tile_sums rows", k_tile_sums, dim3(ctas), dim3(RX_THREADS), 0, st, n,
                     (const uint32_t*)splats.tiles, sums + ctas, (unsigned long long*)total_dev));
  SSR_TRY(arm_pending_total(total_dev, st));
  // pass 0: keys from (tiles, depth) -> (keys_a, vals_a); pass 1 -> (keys_b, cnt as scratch);
  // pass 2 -> (keys_a, depth_order); the tie-fix then fixes depth_order in place and fills cnt
  SSR_TRY((radix_pass<1, 8>(n, 0, nullptr, nullptr, splats.tiles, splats.depth, keys_a, vals_a, counts, offsets, hist,
                        st)));
  SSR_TRY((radix_pass<0, 8>(n, 8, keys_a, vals_a, nullptr, nullptr, keys_b, cnt, counts, offsets, hist + 256, st)));
  SSR_TRY((radix_pass<0, 8>(n, 16, keys_b, cnt, nullptr, nullptr, keys_a, splats.depth_order, counts, offsets,
                        hist + 512, st)));
  SSR_TRY(launch_pdl("k_depth_tiefix", k_depth_tiefix, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, n,
                     (const uint32_t*)keys_a, splats.depth_order, (const double*)splats.depth,
                     (const uint32_t*)splats.tiles, cnt));
  SSR_TRY(launch_pdl("k_tile_sums depth", k_tile_sums, dim3(ctas), dim3(RX_THREADS), 0, st, n, (const uint32_t*)cnt,
                     sums, (unsigned long long*)nullptr));
  return launch_pdl("k_scan2", k_scan2, dim3(2 * ctas), dim3(RX_THREADS), 0, st, n, (const uint32_t*)cnt,
                    (const uint32_t*)splats.depth_order, (const uint32_t*)splats.tiles, splats.offset,
                    splats.row_offset, (const uint64_t*)sums, ctas);
}

extern "C" int ssr_bin_workspace(int64_t m, int32_t n_tiles, int64_t* bytes) {
  (void)n_tiles;
  *bytes = bin_layout(m).bytes;
  return SSR_OK;
}

extern "C" int ssr_bin_tiles(int64_t n, int64_t m, int32_t tiles_x, int32_t tiles_y, ssr_splats splats,
                             uint32_t* inst_gauss, int32_t* tile_ranges, void* workspace, int64_t workspace_bytes,
                             void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
  if (n < 0 || m < 0 || n_tiles <= 0 || n_tiles > 65536) {
    set_error("ssr_bin_tiles: invalid sizes (1..65536 tiles)");
    return SSR_ERR_INVALID;
  }
  if (m > MAX_INSTANCES) {
    set_error("ssr_bin_tiles: instance count exceeds 2^30 - 1");
    return SSR_ERR_CAPACITY;
  }
  const BinLayout L = bin_layout(m);
  if (workspace_bytes < L.bytes) {
    set_error("ssr_bin_tiles: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (m == 0) {
    return check_cuda(cudaMemsetAsync(tile_ranges, 0, sizeof(int32_t) * 2 * n_tiles, st), "ranges memset");
  }
  if (!splats.depth_order) {
    set_error("ssr_bin_tiles: splats.depth_order (from ssr_scan_tiles) is required");
    return SSR_ERR_INVALID;
  }
  char* w = (char*)workspace;
  uint32_t* hist = (uint32_t*)w;
  uint32_t* counts = (uint32_t*)(w + L.counts);
  uint32_t* offsets = (uint32_t*)(w + L.offsets);
  uint32_t* keys_a = (uint32_t*)(w + L.keys_a);
  uint32_t* vals_a = (uint32_t*)(w + L.vals_a);
  uint32_t* keys_b = (uint32_t*)(w + L.keys_b);
  uint32_t* vals_b = (uint32_t*)(w + L.vals_b);
  SSR_TRY(launch_pdl("bin workspace zero", k_zero_words, dim3(1), dim3(256), 0, st, (uint32_t*)w,
                     (int64_t)(L.zero_bytes / 4)));
  SSR_TRY(launch_pdl("k_duplicate", k_duplicate, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, n,
                     (int)tiles_x, (const uint32_t*)splats.tiles, (const uint32_t*)splats.offset,
                     (const int4*)splats.rect, (const uint32_t*)splats.depth_order, keys_a, vals_a));
  // stable LSD sort over the tile id's bits: one pass up to 256 tiles, else
  // two passes splitting the bits evenly (7 + 6 for the 8160 tiles of 1080p)
  int bits = 1;
  while ((1 << bits) < n_tiles) bits++;
  const uint32_t* sorted_keys;
  if (bits <= 8) {
    SSR_TRY(tile_pass(bits, m, 0, keys_a, vals_a, keys_b, inst_gauss, counts, offsets, hist, st));
    sorted_keys = keys_b;
  } else {
    const int b0 = bits <= 14 ? (bits + 1) / 2 : bits - 8;  // high pass <= 8 bits
    SSR_TRY(tile_pass(b0, m, 0, keys_a, vals_a, keys_b, vals_b, counts, offsets, hist, st));
    SSR_TRY(tile_pass(bits - b0, m, b0, keys_b, vals_b, keys_a, inst_gauss, counts, offsets, hist + 256, st));
    sorted_keys = keys_a;
  }
  const int64_t rthreads = (m + RANGE_KEYS - 1) / RANGE_KEYS;
  return launch_pdl("k_ranges", k_ranges, dim3((unsigned)((rthreads + 255) / 256)), dim3(256), 0, st, m,
                    (int)n_tiles, sorted_keys, tile_ranges);
}

extern "C" int ssr_bin_tiles_capacity(int64_t n, int64_t capacity, int32_t tiles_x, int32_t tiles_y,
                                      ssr_splats splats, const uint64_t* total_dev, int64_t* m_out,
                                      uint32_t* inst_gauss, int32_t* tile_ranges, void* workspace,
                                      int64_t workspace_bytes, void* stream) {
  if (!total_dev || !m_out) {
    set_error("ssr_bin_tiles_capacity: total_dev and m_out are required");
    return SSR_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  PendingTotal& pt = pending_total();
  int64_t m;
  if (pt.armed && pt.dev == total_dev) {
    // the copy was queued by ssr_scan_tiles ahead of its depth sort: wait for
    // it alone, so the binning is launched while the device still sorts
    SSR_TRY(check_cuda(cudaEventSynchronize(pt.ev), "instance total"));
    m = (int64_t)*(volatile uint64_t*)pt.host;
    pt.armed = false;
  } else {
    static thread_local uint64_t* host_total = nullptr;
    if (!host_total) SSR_TRY(check_cuda(cudaMallocHost(&host_total, sizeof(uint64_t)), "pinned total"));
    SSR_TRY(check_cuda(cudaMemcpyAsync(host_total, total_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, st),
                       "instance total"));
    SSR_TRY(check_cuda(cudaStreamSynchronize(st), "instance total"));
    m = (int64_t)*host_total;
  }
  *m_out = m;
  if (m > MAX_INSTANCES) {
    set_error("ssr_bin_tiles_capacity: instance count exceeds 2^30 - 1");
    return SSR_ERR_CAPACITY;
  }
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
