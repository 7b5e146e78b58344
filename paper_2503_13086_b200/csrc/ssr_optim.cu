// Stage 5: fused dense Adam (optim.py:29-47,113-130) and densify/prune
// bookkeeping with moment remap (field.py:303-375, optim.py:49-54,101-111).
//
// The field lives in one flat float32 buffer per quantity, class-major:
//   [positions 3N | rotations 4N | log_scales 3N | opacity_logits N | sh 3KN]
// so Adam is a single vectorised pass over params, grads, m and v.
#include "ssr_common.cuh"

namespace ssr {

// One launch; blocks are assigned to class regions so every block has a
// uniform learning rate and bias correction (no per-element class lookup).
struct AdamRegion {
  int64_t start, count;  // element range in the flat buffer
  int64_t phase0;        // start of the class region (sh coefficient index = (e - phase0) % K)
  int64_t block0;        // first block of this region
  float lr, lr_rest;     // sh region: lr = DC rate, lr_rest = rest rate
  float inv_bc1, inv_bc2;
  int is_sh;
};
struct AdamPlan {
  AdamRegion r[5];
};

constexpr int ADAM_THREADS = 256;
constexpr int ADAM_PER_THREAD = 8;  // two float4 per thread
constexpr int64_t ADAM_PER_BLOCK = (int64_t)ADAM_THREADS * ADAM_PER_THREAD;

__device__ __forceinline__ float adam_one(float p, float g, float& m, float& v, float lr, float ib1, float ib2) {
  return adam_update(p, g, m, v, lr, ib1, ib2);
}

// g is indexed by (e - goff): a rank of a sharded step holds only its chunk
// of the reduced gradients (ssr_adam_range).
template <int K>
__global__ void __launch_bounds__(ADAM_THREADS) k_adam(AdamPlan plan, float* __restrict__ p,
                                                       const float* __restrict__ g_base, int64_t goff,
                                                       float* __restrict__ m, float* __restrict__ v) {
  griddep_wait();
  const float* __restrict__ g = g_base - goff;
  const int64_t bid = blockIdx.x;
  int ri = 0;
#pragma unroll
  for (int i = 1; i < 5; i++)
    if (bid >= plan.r[i].block0) ri = i;
  const AdamRegion R = plan.r[ri];
  const int64_t e0 = R.start + (bid - R.block0) * ADAM_PER_BLOCK;
  const int64_t e_end = R.start + R.count;
  const bool vec = ((R.start & 3) == 0) && ((goff & 3) == 0);
  if (vec && e0 + ADAM_PER_BLOCK <= e_end) {
#pragma unroll
    for (int u = 0; u < ADAM_PER_THREAD / 4; u++) {
      const int64_t e = e0 + (int64_t)(u * ADAM_THREADS + threadIdx.x) * 4;
      float4 pp = *reinterpret_cast<float4*>(p + e);
      const float4 gg = *reinterpret_cast<const float4*>(g + e);
      float4 mm = *reinterpret_cast<float4*>(m + e);
      float4 vv = *reinterpret_cast<float4*>(v + e);
      float lr0 = R.lr, lr1 = R.lr, lr2 = R.lr, lr3 = R.lr;
      if (R.is_sh) {
        const int64_t j = e - R.phase0;
        lr0 = ((j + 0) % K) == 0 ? R.lr : R.lr_rest;
        lr1 = ((j + 1) % K) == 0 ? R.lr : R.lr_rest;
        lr2 = ((j + 2) % K) == 0 ? R.lr : R.lr_rest;
        lr3 = ((j + 3) % K) == 0 ? R.lr : R.lr_rest;
      }
      pp.x = adam_one(pp.x, gg.x, mm.x, vv.x, lr0, R.inv_bc1, R.inv_bc2);
      pp.y = adam_one(pp.y, gg.y, mm.y, vv.y, lr1, R.inv_bc1, R.inv_bc2);
      pp.z = adam_one(pp.z, gg.z, mm.z, vv.z, lr2, R.inv_bc1, R.inv_bc2);
      pp.w = adam_one(pp.w, gg.w, mm.w, vv.w, lr3, R.inv_bc1, R.inv_bc2);
      *reinterpret_cast<float4*>(p + e) = pp;
      *reinterpret_cast<float4*>(m + e) = mm;
      *reinterpret_cast<float4*>(v + e) = vv;
    }
  } else {
    for (int u = 0; u < ADAM_PER_THREAD; u++) {
      const int64_t e = e0 + (int64_t)u * ADAM_THREADS + threadIdx.x;
      if (e >= e_end) break;
      const float lr = (R.is_sh && ((e - R.phase0) % K) != 0) ? R.lr_rest : R.lr;
      float mm = m[e], vv = v[e];
      p[e] = adam_one(p[e], g[e], mm, vv, lr, R.inv_bc1, R.inv_bc2);
      m[e] = mm;
      v[e] = vv;
    }
  }
}

// field.py:321-327 masks.  flags: bit0 keep, bit1 clone, bit2 split.
__global__ void k_densify_masks(int64_t n, int K, const float* __restrict__ params, const float* __restrict__ stats,
                                double grad_thr, double big_thr, double prune_opa, uint8_t* __restrict__ flags,
                                int32_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t ns = row_stride(n);
  const float* ls = params + 7 * ns + i * 3;
  double ms = exp((double)ls[0]);
  ms = fmax(ms, exp((double)ls[1]));
  ms = fmax(ms, exp((double)ls[2]));
  const double logit = (double)params[10 * ns + i];
  const bool hot = (double)stats[i] > grad_thr;
  const bool prune = (1.0 / (1.0 + exp(-logit))) < prune_opa;
  const bool big = ms > big_thr;
  const bool clone = hot && !big && !prune;
  const bool split = hot && big && !prune;
  const bool keep = !(split || prune);
  flags[i] = (uint8_t)((keep ? 1 : 0) | (clone ? 2 : 0) | (split ? 4 : 0));
  if (clone) atomicAdd(&counts[0], 1);
  if (split) atomicAdd(&counts[1], 1);
  if (prune) atomicAdd(&counts[2], 1);
}

// Exclusive scans of the three flag bits (keep, clone, split) over the rows,
// hand-written: k_flag_sums gives each 4096-row CTA its three counts, then
// k_flag_scan's CTA t sums its predecessors' counts directly (no look-back
// chain) and scans its own rows, thread j owning 16 consecutive rows.
constexpr int FS_THREADS = 256, FS_ITEMS = 16, FS_ROWS = FS_THREADS * FS_ITEMS;

__global__ void __launch_bounds__(FS_THREADS) k_flag_sums(int64_t n, const uint8_t* __restrict__ flags,
                                                          uint32_t* __restrict__ sums) {
  __shared__ uint32_t red[3][FS_THREADS / 32];
  uint32_t c[3] = {0u, 0u, 0u};
  for (int i = 0; i < FS_ITEMS; i++) {
    const int64_t r = (int64_t)blockIdx.x * FS_ROWS + i * FS_THREADS + threadIdx.x;
    if (r < n) {
      const uint32_t f = flags[r];
      c[0] += f & 1u;
      c[1] += (f >> 1) & 1u;
      c[2] += (f >> 2) & 1u;
    }
  }
#pragma unroll
  for (int b = 0; b < 3; b++) {
    for (int o = 16; o > 0; o >>= 1) c[b] += __shfl_xor_sync(0xffffffffu, c[b], o);
    if ((threadIdx.x & 31) == 0) red[b][threadIdx.x >> 5] = c[b];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    uint32_t t = 0;
    for (int w = 0; w < FS_THREADS / 32; w++) t += red[threadIdx.x][w];
    sums[(size_t)blockIdx.x * 3 + threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(FS_THREADS) k_flag_scan(int64_t n, const uint8_t* __restrict__ flags,
                                                          const uint32_t* __restrict__ sums, uint32_t* __restrict__ o0,
                                                          uint32_t* __restrict__ o1, uint32_t* __restrict__ o2) {
  __shared__ uint32_t s_w[3][FS_THREADS / 32], s_p[3][FS_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t pre[3] = {0u, 0u, 0u};
  for (int t = threadIdx.x; t < (int)blockIdx.x; t += FS_THREADS)
#pragma unroll
    for (int b = 0; b < 3; b++) pre[b] += sums[(size_t)t * 3 + b];
  const int64_t base = (int64_t)blockIdx.x * FS_ROWS + (int64_t)threadIdx.x * FS_ITEMS;
  uint8_t f[FS_ITEMS];
  uint32_t sum[3] = {0u, 0u, 0u};
#pragma unroll
  for (int i = 0; i < FS_ITEMS; i++) {
    f[i] = base + i < n ? flags[base + i] : (uint8_t)0;
#pragma unroll
    for (int b = 0; b < 3; b++) sum[b] += (f[i] >> b) & 1u;
  }
  uint32_t incl[3];
#pragma unroll
  for (int b = 0; b < 3; b++) {
    incl[b] = sum[b];
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl[b], d);
      if (lane >= d) incl[b] += o;
    }
    for (int o = 16; o > 0; o >>= 1) pre[b] += __shfl_xor_sync(0xffffffffu, pre[b], o);
    if (lane == 31) s_w[b][warp] = incl[b];
    if (lane == 0) s_p[b][warp] = pre[b];
  }
  __syncthreads();
  uint32_t run[3];
#pragma unroll
  for (int b = 0; b < 3; b++) {
    uint32_t wb = 0, p = 0;
    for (int w = 0; w < FS_THREADS / 32; w++) {
      if (w < warp) wb += s_w[b][w];
      p += s_p[b][w];
    }
    run[b] = p + wb + incl[b] - sum[b];
  }
  uint32_t* outs[3] = {o0, o1, o2};
#pragma unroll
  for (int i = 0; i < FS_ITEMS; i++) {
    if (base + i < n)
#pragma unroll
      for (int b = 0; b < 3; b++) outs[b][base + i] = run[b];
#pragma unroll
    for (int b = 0; b < 3; b++) run[b] += (f[i] >> b) & 1u;
  }
}

// field.py:329-372 + optim.py:49-54: kept rows, then clones, then split pairs.
// Kept rows (field.py:303-375 compaction): one warp per 32 source rows copies
// each class region's 32 * width contiguous source floats lane-strided
// (coalesced reads; the kept rows land contiguously, so the writes are too)
// into their compacted positions, for the parameters and both moments.
template <int W>
__device__ __forceinline__ void keep_copy(const float* __restrict__ src, float* __restrict__ dst, int64_t i0,
                                          int rows, unsigned keep, uint32_t my_off, int lane) {
  for (int e0 = 0; e0 < rows * W; e0 += 32) {  // same trip count on every lane (the shuffle)
    const int e = e0 + lane;
    const int r = min(e / W, 31), j = e - (e / W) * W;
    const uint32_t off = __shfl_sync(0xffffffffu, my_off, r);
    if (e < rows * W && ((keep >> r) & 1u)) dst[(int64_t)off * W + j] = src[(i0 + r) * W + j];
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_densify_keep(int64_t n, int64_t n_new, const float* __restrict__ src,
                                                      const float* __restrict__ m, const float* __restrict__ v,
                                                      const uint8_t* __restrict__ flags,
                                                      const uint32_t* __restrict__ keep_off, float* __restrict__ dst,
                                                      float* __restrict__ new_m, float* __restrict__ new_v) {
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
  if (i0 >= n) return;
  const int rows = (int)min((int64_t)32, n - i0);
  const bool mine = lane < rows;
  const bool kp = mine && (flags[i0 + lane] & 1);
  const unsigned keep = __ballot_sync(0xffffffffu, kp);
  if (!keep) return;
  const uint32_t my_off = mine ? keep_off[i0 + lane] : 0u;
  const int64_t ns = row_stride(n), nns = row_stride(n_new);
  const float* srcs[3] = {src, m, v};
  float* dsts[3] = {dst, new_m, new_v};
#pragma unroll
  for (int b = 0; b < 3; b++) {
    if (!dsts[b]) continue;
    const float* sb = srcs[b];
    float* db = dsts[b];
    keep_copy<3>(sb, db, i0, rows, keep, my_off, lane);
    keep_copy<4>(sb + 3 * ns, db + 3 * nns, i0, rows, keep, my_off, lane);
    keep_copy<3>(sb + 7 * ns, db + 7 * nns, i0, rows, keep, my_off, lane);
    keep_copy<1>(sb + 10 * ns, db + 10 * nns, i0, rows, keep, my_off, lane);
    keep_copy<3 * K>(sb + 11 * ns, db + 11 * nns, i0, rows, keep, my_off, lane);
  }
}

__global__ void k_densify_apply(int64_t n, int64_t n_new, int K, const float* __restrict__ src, const float* m,
                                const float* v, const uint8_t* __restrict__ flags,
                                const uint32_t* __restrict__ keep_off, const uint32_t* __restrict__ clone_off,
                                const uint32_t* __restrict__ split_off, const double* __restrict__ eps, double log_shrink, float* __restrict__ dst,
                                float* new_m, float* new_v) {
  // kept rows are copied by k_densify_keep; this kernel writes the clones and
  // the split children
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t f = flags[i];
  const uint8_t fl = flags[n - 1];
  const uint32_t n_keep = keep_off[n - 1] + (fl & 1);
  const uint32_t n_clone = clone_off[n - 1] + ((fl >> 1) & 1);
  const int width[5] = {3, 4, 3, 1, 3 * K};
  const int64_t ns = row_stride(n), nns = row_stride(n_new);
  const int64_t so[5] = {0, 3 * ns, 7 * ns, 10 * ns, 11 * ns};
  const int64_t dof[5] = {0, 3 * nns, 7 * nns, 10 * nns, 11 * nns};
  if (f & 2) {
    const int64_t d = (int64_t)n_keep + clone_off[i];
    for (int c = 0; c < 5; c++)
      for (int j = 0; j < width[c]; j++) {
        const int64_t t = dof[c] + d * width[c] + j;
        dst[t] = src[so[c] + i * width[c] + j];
        if (new_m) new_m[t] = 0.f;
        if (new_v) new_v[t] = 0.f;
      }
  }
  if (f & 4) {
    const int64_t j2 = split_off[i];
    const float* q = src + so[1] + i * 4;
    double qq[4] = {(double)q[0], (double)q[1], (double)q[2], (double)q[3]};
    double R[9], qn[4], nrm;
    quat_rotmat64(qq, R, qn, &nrm);
    double sc[3];
    for (int a = 0; a < 3; a++) sc[a] = exp((double)src[so[2] + i * 3 + a]);
    for (int c2 = 0; c2 < 2; c2++) {
      const int64_t d = (int64_t)n_keep + n_clone + 2 * j2 + c2;
      const double* e = eps + (2 * j2 + c2) * 3;
      for (int a = 0; a < 3; a++) {
        double off = 0.0;
        for (int b = 0; b < 3; b++) off += R[a * 3 + b] * (sc[b] * e[b]);
        dst[dof[0] + d * 3 + a] = (float)((double)src[so[0] + i * 3 + a] + off);
        dst[dof[2] + d * 3 + a] = (float)((double)src[so[2] + i * 3 + a] - log_shrink);
      }
      for (int a = 0; a < 4; a++) dst[dof[1] + d * 4 + a] = q[a];
      dst[dof[3] + d] = src[so[3] + i];
      for (int a = 0; a < 3 * K; a++) dst[dof[4] + d * 3 * K + a] = src[so[4] + i * 3 * K + a];
      if (new_m || new_v)
        for (int c = 0; c < 5; c++)
          for (int a = 0; a < width[c]; a++) {
            const int64_t t = dof[c] + d * width[c] + a;
            if (new_m) new_m[t] = 0.f;
            if (new_v) new_v[t] = 0.f;
          }
    }
  }
}

// ------------------------------------------------------------------ fused exchange + Adam over peer memory
// The sharded step of a view batch as one kernel per rank instead
// of reduce-scatter -> Adam -> all-gather: rank r owns the flat elements of
// its chunk; each thread loads the gradients of its elements from every
// rank's buffer (peer memory over NVLink / NVSwitch, mapped by CUDA IPC), sums
// them in rank order, runs Adam on its own replica's element and stores the
// new value into every rank's replica.  Reads and writes use the two link
// directions at once, the reduced gradient is never written, and the Adam
// pass over the chunk rides on the transfer.  The densify statistics
// (screen_norms, visible) are summed the same way and the sum stored into
// every rank's gradient buffer.  Ranks must not read their replicas until
// every rank's kernel is done (a stream-ordered barrier after it), nor launch
// it before every rank's gradients are final (one before it).  One-GPU
// timing with the peers as local buffers (tools/exchange_bench.py, 3 M
// Gaussians): 5.6 TB/s of HBM traffic at W = 2, 6.4 TB/s at W = 8.
constexpr int MAX_PEERS = 8;
struct PeerSet {
  const float* g[MAX_PEERS];
  float* p[MAX_PEERS];
  float* gs[MAX_PEERS];  // writable view of the same gradient buffers (statistics)
  int world;
};

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

template <int K>
__global__ void __launch_bounds__(ADAM_THREADS) k_exchange_adam(AdamPlan plan, PeerSet ps, int own,
                                                                float* __restrict__ m, float* __restrict__ v,
                                                                int64_t s_lo, int64_t s_hi, int64_t s_block0) {
  griddep_wait();
  const int64_t bid = blockIdx.x;
  const int W = ps.world;
  if (bid >= s_block0) {
    // statistics: sum over the ranks, stored into every rank's buffer
    const int64_t e0 = s_lo + (bid - s_block0) * ADAM_PER_BLOCK;
    for (int u = 0; u < ADAM_PER_THREAD; u++) {
      const int64_t e = e0 + (int64_t)u * ADAM_THREADS + threadIdx.x;
      if (e >= s_hi) break;
      float g = ps.g[0][e];
      for (int q = 1; q < W; q++) g += ps.g[q][e];
      for (int q = 0; q < W; q++) ps.gs[q][e] = g;
    }
    return;
  }
  int ri = 0;
#pragma unroll
  for (int i = 1; i < 5; i++)
    if (bid >= plan.r[i].block0) ri = i;
  const AdamRegion R = plan.r[ri];
  const int64_t e0 = R.start + (bid - R.block0) * ADAM_PER_BLOCK;
  const int64_t e_end = R.start + R.count;
  float* __restrict__ p = ps.p[own];
  if ((R.start & 3) == 0 && e0 + ADAM_PER_BLOCK <= e_end) {
#pragma unroll
    for (int u = 0; u < ADAM_PER_THREAD / 4; u++) {
      const int64_t e = e0 + (int64_t)(u * ADAM_THREADS + threadIdx.x) * 4;
      float4 gq[MAX_PEERS];
#pragma unroll
      for (int q = 0; q < MAX_PEERS; q++)  // all loads in flight before the sum
        if (q < W) gq[q] = *reinterpret_cast<const float4*>(ps.g[q] + e);
      float4 gg = gq[0];
#pragma unroll
      for (int q = 1; q < MAX_PEERS; q++)
        if (q < W) gg = f4_add(gg, gq[q]);
      float4 pp = *reinterpret_cast<const float4*>(p + e);
      float4 mm = *reinterpret_cast<float4*>(m + e);
      float4 vv = *reinterpret_cast<float4*>(v + e);
      float lr0 = R.lr, lr1 = R.lr, lr2 = R.lr, lr3 = R.lr;
      if (R.is_sh) {
        const int64_t j = e - R.phase0;
        lr0 = ((j + 0) % K) == 0 ? R.lr : R.lr_rest;
        lr1 = ((j + 1) % K) == 0 ? R.lr : R.lr_rest;
        lr2 = ((j + 2) % K) == 0 ? R.lr : R.lr_rest;
        lr3 = ((j + 3) % K) == 0 ? R.lr : R.lr_rest;
      }
      pp.x = adam_one(pp.x, gg.x, mm.x, vv.x, lr0, R.inv_bc1, R.inv_bc2);
      pp.y = adam_one(pp.y, gg.y, mm.y, vv.y, lr1, R.inv_bc1, R.inv_bc2);
      pp.z = adam_one(pp.z, gg.z, mm.z, vv.z, lr2, R.inv_bc1, R.inv_bc2);
      pp.w = adam_one(pp.w, gg.w, mm.w, vv.w, lr3, R.inv_bc1, R.inv_bc2);
      *reinterpret_cast<float4*>(m + e) = mm;
      *reinterpret_cast<float4*>(v + e) = vv;
#pragma unroll
      for (int q = 0; q < MAX_PEERS; q++)
        if (q < W) *reinterpret_cast<float4*>(ps.p[q] + e) = pp;
    }
  } else {
    for (int u = 0; u < ADAM_PER_THREAD; u++) {
      const int64_t e = e0 + (int64_t)u * ADAM_THREADS + threadIdx.x;
      if (e >= e_end) break;
      float g = ps.g[0][e];
      for (int q = 1; q < W; q++) g += ps.g[q][e];
      const float lr = (R.is_sh && ((e - R.phase0) % K) != 0) ? R.lr_rest : R.lr;
      float mm = m[e], vv = v[e];
      const float np = adam_one(p[e], g, mm, vv, lr, R.inv_bc1, R.inv_bc2);
      m[e] = mm;
      v[e] = vv;
      for (int q = 0; q < W; q++) ps.p[q][e] = np;
    }
  }
  // No per-thread system fence: the stores are performed by the time the
  // grid completes (the next kernel on the stream -- the barrier -- starts only
  // then), and the barrier's cross-GPU synchronisation orders them before any
  // peer's later reads.  A fence per thread tripled the kernel's time.
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace ssr

using namespace ssr;

// Region plan of Adam over the flat elements [lo, hi) (padding rows excluded);
// returns the block count.
static int64_t adam_plan(AdamPlan& plan, int64_t n, int32_t sh_degree, int64_t lo, int64_t hi, const double* lr,
                         double lr_sh_rest, const double* bc1, const double* bc2) {
  const int K = (sh_degree + 1) * (sh_degree + 1);
  const int64_t widths[5] = {3, 4, 3, 1, 3 * (int64_t)K};
  int64_t start = 0, blocks = 0;
  const int64_t ns = row_stride(n);
  for (int c = 0; c < 5; c++) {
    AdamRegion& R = plan.r[c];
    const int64_t a = start > lo ? start : lo;
    const int64_t b0 = start + widths[c] * n;
    const int64_t b = b0 < hi ? b0 : hi;
    R.start = a;
    R.count = b > a ? b - a : 0;
    R.phase0 = start;
    R.block0 = blocks;
    R.lr = (float)lr[c];
    R.lr_rest = (float)lr_sh_rest;
    R.inv_bc1 = (float)(1.0 / bc1[c]);
    R.inv_bc2 = (float)(1.0 / bc2[c]);
    R.is_sh = c == 4;
    start += widths[c] * ns;
    blocks += (R.count + ADAM_PER_BLOCK - 1) / ADAM_PER_BLOCK;
  }
  return blocks;
}

// Adam over the flat elements [lo, hi) of the class-major buffers (padding
// rows excluded); grads[e - goff] is the gradient of element e.
static int launch_adam(int64_t n, int32_t sh_degree, float* params, const float* grads, int64_t goff, float* m,
                       float* v, int64_t lo, int64_t hi, const double* lr, double lr_sh_rest, const double* bc1,
                       const double* bc2, cudaStream_t st) {
  const int K = (sh_degree + 1) * (sh_degree + 1);
  AdamPlan plan;
  const int64_t blocks = adam_plan(plan, n, sh_degree, lo, hi, lr, lr_sh_rest, bc1, bc2);
  if (blocks == 0) return SSR_OK;
  switch (K) {
    case 1: return launch_pdl("k_adam", k_adam<1>, dim3((unsigned)blocks), dim3(ADAM_THREADS), 0, st, plan, params,
                          grads, goff, m, v);
    case 4: return launch_pdl("k_adam", k_adam<4>, dim3((unsigned)blocks), dim3(ADAM_THREADS), 0, st, plan, params,
                          grads, goff, m, v);
    case 9: return launch_pdl("k_adam", k_adam<9>, dim3((unsigned)blocks), dim3(ADAM_THREADS), 0, st, plan, params,
                          grads, goff, m, v);
    default: return launch_pdl("k_adam", k_adam<16>, dim3((unsigned)blocks), dim3(ADAM_THREADS), 0, st, plan, params,
                          grads, goff, m, v);
  }
}


extern "C" int ssr_adam(int64_t n, int32_t sh_degree, float* params, const float* grads, float* m, float* v,
                        const double* lr, double lr_sh_rest, const double* bc1, const double* bc2, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || !lr || !bc1 || !bc2) {
    set_error("ssr_adam: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  return launch_adam(n, sh_degree, params, grads, 0, m, v, 0, INT64_MAX, lr, lr_sh_rest, bc1, bc2,
                     (cudaStream_t)stream);
}

extern "C" int ssr_adam_range(int64_t n, int32_t sh_degree, float* params, const float* grads, int64_t grads_offset,
                              float* m, float* v, int64_t lo, int64_t hi, const double* lr, double lr_sh_rest,
                              const double* bc1, const double* bc2, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || !lr || !bc1 || !bc2 || lo < 0 || hi < lo || grads_offset > lo) {
    set_error("ssr_adam_range: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0 || hi == lo) return SSR_OK;
  return launch_adam(n, sh_degree, params, grads, grads_offset, m, v, lo, hi, lr, lr_sh_rest, bc1, bc2,
                     (cudaStream_t)stream);
}

extern "C" int ssr_exchange_chunk(int64_t total, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  if (world < 1 || rank < 0 || rank >= world || total < 0 || !lo || !hi) {
    set_error("ssr_exchange_chunk: invalid argument");
    return SSR_ERR_INVALID;
  }
  const int64_t chunk = total / (4 * (int64_t)world) * 4;  // 16-byte aligned chunks
  *lo = rank * chunk;
  *hi = rank == world - 1 ? total : (rank + 1) * chunk;  // the last rank also owns the tail
  return SSR_OK;
}

extern "C" int ssr_exchange_adam(int64_t n, int32_t sh_degree, int32_t world, int32_t rank, float* const* grads,
                                 float* const* params, float* m, float* v, const double* lr, double lr_sh_rest,
                                 const double* bc1, const double* bc2, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || world < 1 || world > MAX_PEERS || rank < 0 || rank >= world ||
      !grads || !params || !m || !v || !lr || !bc1 || !bc2) {
    set_error("ssr_exchange_adam: invalid argument (world must be 1..8)");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  PeerSet ps = {};
  ps.world = world;
  for (int q = 0; q < world; q++) {
    if (!grads[q] || !params[q]) {
      set_error("ssr_exchange_adam: null peer pointer");
      return SSR_ERR_INVALID;
    }
    ps.g[q] = grads[q];
    ps.gs[q] = grads[q];
    ps.p[q] = params[q];
  }
  const int K = (sh_degree + 1) * (sh_degree + 1);
  const int64_t ns = row_stride(n);
  const int64_t p_floats = (11 + 3 * (int64_t)K) * ns;
  int64_t lo, hi, s_lo, s_hi;
  SSR_TRY(ssr_exchange_chunk(p_floats, world, rank, &lo, &hi));
  SSR_TRY(ssr_exchange_chunk(2 * ns, world, rank, &s_lo, &s_hi));
  s_lo += p_floats;  // statistics: [screen_norms | visible] after the parameter classes
  s_hi += p_floats;
  AdamPlan plan;
  const int64_t blocks = adam_plan(plan, n, sh_degree, lo, hi, lr, lr_sh_rest, bc1, bc2);
  const int64_t total = blocks + (s_hi - s_lo + ADAM_PER_BLOCK - 1) / ADAM_PER_BLOCK;
  if (total == 0) return SSR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (K) {
    case 1: return launch_pdl("k_exchange_adam", k_exchange_adam<1>, dim3((unsigned)total), dim3(ADAM_THREADS), 0,
                              st, plan, ps, (int)rank, m, v, s_lo, s_hi, blocks);
    case 4: return launch_pdl("k_exchange_adam", k_exchange_adam<4>, dim3((unsigned)total), dim3(ADAM_THREADS), 0,
                              st, plan, ps, (int)rank, m, v, s_lo, s_hi, blocks);
    case 9: return launch_pdl("k_exchange_adam", k_exchange_adam<9>, dim3((unsigned)total), dim3(ADAM_THREADS), 0,
                              st, plan, ps, (int)rank, m, v, s_lo, s_hi, blocks);
    default: return launch_pdl("k_exchange_adam", k_exchange_adam<16>, dim3((unsigned)total), dim3(ADAM_THREADS), 0,
                               st, plan, ps, (int)rank, m, v, s_lo, s_hi, blocks);
  }
}

extern "C" int ssr_densify_masks(int64_t n, const float* params, int32_t sh_degree, const float* stats,
                                 double grad_threshold, double big_threshold, double prune_opacity, uint8_t* flags,
                                 int32_t* counts, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3) {
    set_error("ssr_densify_masks: invalid argument");
    return SSR_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SSR_TRY(check_cuda(cudaMemsetAsync(counts, 0, 3 * sizeof(int32_t), st), "densify counts"));
  if (n == 0) return SSR_OK;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  k_densify_masks<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, K, params, stats, grad_threshold, big_threshold,
                                                               prune_opacity, flags, counts);
  return check_launch("k_densify_masks");
}

extern "C" int ssr_densify_workspace(int64_t n, int64_t* bytes) {
  const int64_t nn = n > 0 ? n : 1;
  *bytes = 3 * align_up(4 * nn, 256) + align_up(12 * ((nn + FS_ROWS - 1) / FS_ROWS), 256) + 256;
  return SSR_OK;
}

extern "C" int ssr_densify_apply(int64_t n, int64_t n_new, int32_t sh_degree, const float* params, const float* m,
                                 const float* v, const uint8_t* flags, const double* eps, double log_shrink,
                                 float* new_params, float* new_m, float* new_v, void* workspace,
                                 int64_t workspace_bytes, void* stream) {
  if (n < 0 || n_new < 0 || sh_degree < 0 || sh_degree > 3 || n > INT32_MAX) {
    set_error("ssr_densify_apply: invalid argument");
    return SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_densify_workspace(n, &need);
  if (workspace_bytes < need) {
    set_error("ssr_densify_apply: workspace too small");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  char* w = (char*)workspace;
  uint32_t* offs[3];
  for (int b = 0; b < 3; b++) {
    offs[b] = (uint32_t*)w;
    w += align_up(4 * n, 256);
  }
  const unsigned fs = (unsigned)((n + FS_ROWS - 1) / FS_ROWS);
  uint32_t* fsums = (uint32_t*)w;
  k_flag_sums<<<fs, FS_THREADS, 0, st>>>(n, flags, fsums);
  SSR_TRY(check_launch("k_flag_sums"));
  k_flag_scan<<<fs, FS_THREADS, 0, st>>>(n, flags, fsums, offs[0], offs[1], offs[2]);
  SSR_TRY(check_launch("k_flag_scan"));
  const unsigned kb = (unsigned)((n + 255) / 256);
  switch (K) {
    case 1: k_densify_keep<1><<<kb, 256, 0, st>>>(n, n_new, params, m, v, flags, offs[0], new_params, new_m, new_v); break;
    case 4: k_densify_keep<4><<<kb, 256, 0, st>>>(n, n_new, params, m, v, flags, offs[0], new_params, new_m, new_v); break;
    case 9: k_densify_keep<9><<<kb, 256, 0, st>>>(n, n_new, params, m, v, flags, offs[0], new_params, new_m, new_v); break;
    default: k_densify_keep<16><<<kb, 256, 0, st>>>(n, n_new, params, m, v, flags, offs[0], new_params, new_m, new_v); break;
  }
  SSR_TRY(check_launch("k_densify_keep"));
  k_densify_apply<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, n_new, K, params, m, v, flags, offs[0], offs[1],
                                                               offs[2], eps, log_shrink, new_params,
                                                               new_m, new_v);
  return check_launch("k_densify_apply");
}
