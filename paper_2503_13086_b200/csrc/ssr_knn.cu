// Exact k-nearest-neighbour distances on a dense uniform grid:
// the GPU replacement of the reference's cKDTree queries used by field
// expansion -- insert_points' 3-NN scale init (field.py:279-289), the novelty
// filter (field.py:139-151) and median_nn_spacing (field.py:154-161).
//
// Build: counting sort of the pool by cell (histogram -> scan -> scatter),
// coordinates copied into cell order.  Query: one warp per query walks
// Chebyshev rings of cells around its cell and keeps the k smallest squared
// distances; after ring r every unseen point is at least r*h away (the query
// lies inside its own cell, the bbox covers pool and queries), so the walk
// stops once the k-th distance is <= r*h.  float64 throughout, so distances
// are those of a float64 k-d tree.
#include <math_constants.h>

#include "ssr_common.cuh"

namespace ssr {

constexpr int KNN_MAX_K = 8;

struct Grid {
  double bx, by, bz, h, inv_h;
  int dx, dy, dz;
};

__device__ __forceinline__ int cell_coord(double v, double b, double inv_h, int d) {
  int c = (int)floor((v - b) * inv_h);
  return c < 0 ? 0 : (c >= d ? d - 1 : c);
}

__global__ void k_knn_count(int64_t n, const double* __restrict__ pool, Grid g, uint32_t* __restrict__ cell_of,
                            uint32_t* __restrict__ count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int cx = cell_coord(pool[i * 3], g.bx, g.inv_h, g.dx);
  const int cy = cell_coord(pool[i * 3 + 1], g.by, g.inv_h, g.dy);
  const int cz = cell_coord(pool[i * 3 + 2], g.bz, g.inv_h, g.dz);
  const uint32_t c = ((uint32_t)cz * g.dy + cy) * g.dx + cx;
  cell_of[i] = c;
  atomicAdd(&count[c], 1u);
}

__global__ void k_knn_scatter(int64_t n, const double* __restrict__ pool, const uint32_t* __restrict__ cell_of,
                              uint32_t* __restrict__ cursor, double* __restrict__ sorted) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t pos = atomicAdd(&cursor[cell_of[i]], 1u);
  sorted[(int64_t)pos * 3] = pool[i * 3];
  sorted[(int64_t)pos * 3 + 1] = pool[i * 3 + 1];
  sorted[(int64_t)pos * 3 + 2] = pool[i * 3 + 2];
}

// One warp per query: the rows of cells of each Chebyshev ring are split over
// the lanes (each lane keeps its own k smallest squared distances), and after
// every ring the warp merges the lanes' lists to test the stop condition, so
// a query whose nearest points are many rings away is searched 32 cells at a
// time.  The k smallest distances of a set do not depend on the visiting
// order, so the result equals the one-thread walk's.
constexpr int KNN_WARPS = 4;

// k-th smallest (1-based kk) of the union of the lanes' sorted lists, without
// consuming them (work on copies), warp-uniform result.
__device__ __forceinline__ double warp_kth(const double* best, int k) {
  double head[KNN_MAX_K];
  for (int j = 0; j < KNN_MAX_K; j++) head[j] = best[j];
  int pos = 0;
  double v = CUDART_INF;
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < k; j++) {
    const double mine = pos < k ? head[pos] : CUDART_INF;
    double m = mine;
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    v = m;
    // the lowest lane holding the minimum pops it
    const unsigned who = __ballot_sync(0xffffffffu, mine == m);
    if (lane == __ffs(who) - 1) pos++;
  }
  return v;
}

__global__ void __launch_bounds__(KNN_WARPS * 32) k_knn_query(int64_t nq, const double* __restrict__ queries, int k,
                                                              Grid g, const uint32_t* __restrict__ start,
                                                              const double* __restrict__ sorted,
                                                              double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t)blockIdx.x * KNN_WARPS + (threadIdx.x >> 5);
  if (qi >= nq) return;
  const double qx = queries[qi * 3], qy = queries[qi * 3 + 1], qz = queries[qi * 3 + 2];
  const int cx = cell_coord(qx, g.bx, g.inv_h, g.dx);
  const int cy = cell_coord(qy, g.by, g.inv_h, g.dy);
  const int cz = cell_coord(qz, g.bz, g.inv_h, g.dz);
  double best[KNN_MAX_K];
  for (int j = 0; j < KNN_MAX_K; j++) best[j] = CUDART_INF;
  int found = 0;
  const int rmax = max(g.dx, max(g.dy, g.dz));
  for (int r = 0; r <= rmax; r++) {
    const int side = 2 * r + 1;
    // rows (oz, oy) of the ring, lane-strided; a face row holds all x, an
    // interior row only x = -r and x = +r
    for (int row = lane; row < side * side; row += 32) {
      const int oz = row / side - r, oy = row % side - r;
      const int z = cz + oz, y = cy + oy;
      if (z < 0 || z >= g.dz || y < 0 || y >= g.dy) continue;
      const bool face = (oz == -r || oz == r || oy == -r || oy == r);
      const int step = (face || r == 0) ? 1 : 2 * r;
      for (int ox = -r; ox <= r; ox += step) {
        const int x = cx + ox;
        if (x < 0 || x >= g.dx) continue;
        const uint32_t c = ((uint32_t)z * g.dy + y) * g.dx + x;
        const uint32_t e = start[c + 1];
        for (uint32_t p = start[c]; p < e; p++) {
          const double ddx = sorted[(int64_t)p * 3] - qx;
          const double ddy = sorted[(int64_t)p * 3 + 1] - qy;
          const double ddz = sorted[(int64_t)p * 3 + 2] - qz;
          const double d2 = ddx * ddx + ddy * ddy + ddz * ddz;
          if (d2 < best[k - 1]) {
            int j = k - 1;
            while (j > 0 && best[j - 1] > d2) {
              best[j] = best[j - 1];
              j--;
            }
            best[j] = d2;
          }
          found++;
        }
      }
    }
    int total = found;
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (total >= k) {
      const double reach = (double)r * g.h;
      if (warp_kth(best, k) <= reach * reach) break;
    }
  }
  // the k smallest of the lanes' lists, in ascending order
  int pos = 0;
  for (int j = 0; j < k; j++) {
    const double mine = pos < k ? best[pos] : CUDART_INF;
    double m = mine;
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    const unsigned who = __ballot_sync(0xffffffffu, mine == m);
    if (lane == __ffs(who) - 1) pos++;
    if (lane == 0) out[qi * k + j] = sqrt(m);
  }
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static size_t knn_scan_bytes(int64_t n_cells) { return (size_t)scan_u32_workspace(n_cells + 1); }

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_knn_workspace(int64_t n_pool, int64_t n_cells, int64_t* bytes) {
  const int64_t c = align_up(4 * (n_cells + 1), 256);
  *bytes = 3 * c + align_up(4 * (n_pool > 0 ? n_pool : 1), 256) + align_up(24 * (n_pool > 0 ? n_pool : 1), 256) +
           align_up((int64_t)knn_scan_bytes(n_cells), 256);
  return SSR_OK;
}

extern "C" int ssr_knn(const double* pool, int64_t n_pool, const double* queries, int64_t n_q, int32_t k,
                       const double* grid, const int32_t* dims, double* out_dist, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  if (n_pool < 0 || n_q < 0 || k < 1 || k > KNN_MAX_K || !grid || !dims || !(grid[3] > 0.0) || dims[0] < 1 ||
      dims[1] < 1 || dims[2] < 1) {
    set_error("ssr_knn: invalid argument (1 <= k <= 8, positive cell size and dims)");
    return SSR_ERR_INVALID;
  }
  const int64_t n_cells = (int64_t)dims[0] * dims[1] * dims[2];
  if (n_cells > (1LL << 26)) {
    set_error("ssr_knn: too many grid cells");
    return SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_knn_workspace(n_pool, n_cells, &need);
  if (workspace_bytes < need) {
    set_error("ssr_knn: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (n_q == 0) return SSR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Grid g;
  g.bx = grid[0];
  g.by = grid[1];
  g.bz = grid[2];
  g.h = grid[3];
  g.inv_h = 1.0 / grid[3];
  g.dx = dims[0];
  g.dy = dims[1];
  g.dz = dims[2];
  const int64_t c = align_up(4 * (n_cells + 1), 256);
  char* w = (char*)workspace;
  uint32_t* count = (uint32_t*)w;
  uint32_t* start = (uint32_t*)(w + c);
  uint32_t* cursor = (uint32_t*)(w + 2 * c);
  uint32_t* cell_of = (uint32_t*)(w + 3 * c);
  double* sorted = (double*)(w + 3 * c + align_up(4 * (n_pool > 0 ? n_pool : 1), 256));
  char* temp = (char*)sorted + align_up(24 * (n_pool > 0 ? n_pool : 1), 256);
  SSR_TRY(check_cuda(cudaMemsetAsync(count, 0, 4 * (n_cells + 1), st), "knn count memset"));
  if (n_pool > 0) {
    k_knn_count<<<(unsigned)((n_pool + 255) / 256), 256, 0, st>>>(n_pool, pool, g, cell_of, count);
    SSR_TRY(check_launch("k_knn_count"));
  }
  SSR_TRY(scan_u32(count, start, n_cells + 1, temp, st));
  SSR_TRY(check_cuda(cudaMemcpyAsync(cursor, start, 4 * (n_cells + 1), cudaMemcpyDeviceToDevice, st), "knn cursor"));
  if (n_pool > 0) {
    k_knn_scatter<<<(unsigned)((n_pool + 255) / 256), 256, 0, st>>>(n_pool, pool, cell_of, cursor, sorted);
    SSR_TRY(check_launch("k_knn_scatter"));
  }
  k_knn_query<<<(unsigned)((n_q + KNN_WARPS - 1) / KNN_WARPS), KNN_WARPS * 32, 0, st>>>(n_q, queries, k, g, start,
                                                                                      sorted, out_dist);
  return check_launch("k_knn_query");
}
