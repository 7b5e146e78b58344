// Stage 4 gradient chain (rasterize/backward.py:110-259, sh.py:68-152) in
// float32: merge each splat's instance rows (bincount order), chain d_mu /
// d_conic through the EWA projection into position, rotation and log-scale,
// and d_colour through the SH evaluation into the coefficients and position.
//
// The preprocess (ssr_project.cu) must reproduce the reference's fp64 culling,
// rects and depth order bit for bit, so it runs in float64; the chain only has
// to meet the 1e-3 relative-L2 gradient bar, so it runs in float32 (~1e-6
// relative), which halves its registers and lets it stream at HBM rate.
//
// Two kernels per call:
//  * k_chain_geo: one thread per field row, 128 rows per CTA; the CTA's rows
//    own one contiguous range of inst_rows (field-row order), staged into
//    shared memory by one TMA bulk copy.  Writes the geometric gradients and
//    parks the merged colour gradient (and, fused, the geometric position
//    gradient) in the row's first instance row for the SH kernel.
//  * k_chain_sh: four lanes per row, each owning a quarter of every colour
//    channel's coefficients, read and written as coalesced float4 streams
//    straight from HBM (no shared-memory transpose); channel sums and the
//    direction gradient are reduced over the four lanes with shuffles.
// Fused (ssr_chain_adam): the dense Adam step is applied in place instead of
// writing FieldGrads, so the gradient buffer's write and read disappear.  The
// geometry kernel then also stages its CTA's rotation / log-scale / logit rows
// and their moments by TMA, and k_chain_sh_adam (same lane layout as
// k_chain_sh) stages the SH, position and moment rows: every Adam stream is
// a few large bulk copies per CTA instead of per-thread loads.
#include <climits>

#include "ssr_common.cuh"

namespace ssr {

constexpr unsigned FULLMASK = 0xffffffffu;

struct CamF {
  float R[9], t[3], fx, fy, center[3];
  int width, height;
};

static CamF to_camf(const ssr_camera& c) {
  CamF o;
  for (int i = 0; i < 9; i++) o.R[i] = (float)c.R[i];
  for (int i = 0; i < 3; i++) {
    o.t[i] = (float)c.t[i];
    o.center[i] = (float)c.center[i];
  }
  o.fx = (float)c.fx;
  o.fy = (float)c.fy;
  o.width = c.width;
  o.height = c.height;
  return o;
}

// Adam of optim.py:40-47 for one element (same expression as k_adam).
struct AdamClassF {
  float lr, ib1, ib2;
};
struct AdamArgsF {
  AdamClassF c[6];  // pos, rot, scale, opacity, sh dc, sh rest
  float* m;
  float* v;
};
__device__ __forceinline__ float adam_step(float p, float g, float& m, float& v, const AdamClassF& c) {
  return adam_update(p, g, m, v, c.lr, c.ib1, c.ib2);
}

// ------------------------------------------------------------------ merge of large splats
// Rows of Gaussians touching more than MERGE_BIG tiles (large splats, up to
// the whole image) are pre-summed before the chain, load-balanced over the
// instance rows: the rows (field-row order, contiguous per Gaussian) are cut
// into MERGE_CHUNK-row chunks and every warp takes a contiguous run of chunks.
// Each large Gaussian's rows inside one chunk are summed by the warp (fixed
// order: flat coalesced loads, then a shuffle tree) into the first of those
// rows -- the Gaussian's first row or a chunk boundary.  The geometry kernel
// adds those heads in ascending order, so the merge is deterministic and no
// warp waits on another.
constexpr uint32_t MERGE_BIG = 32;
constexpr uint32_t MERGE_CHUNK = 256;
constexpr int MERGE_WARPS = 8;

// Sum of nr contiguous instance rows (ROW_WORDS floats each) over a warp: lane l
// reads rows l, l + 32, ... (two rows, 20 loads, in flight), then a
// reduce-scatter butterfly over 16 zero-padded channels (16 shuffles instead
// of 9 x 5).  Lanes 2c and 2c + 1 of the bit-reversed lane order end up with
// channel c; the return value is the lane's channel sum, *ch its channel.
// Rows whose tag is not `gen` belong to slots no pixel walked: zero.
__device__ __forceinline__ float merge_rows_warp(const float* __restrict__ rw, uint32_t nr, int lane, int* ch,
                                                 uint32_t gen) {
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; c++) acc[c] = 0.f;
  uint32_t j = lane;
  for (; j + 32 < nr; j += 64) {
    float v0[ROW_WORDS], v1[ROW_WORDS];
    load_row(rw + (int64_t)j * ROW_WORDS, v0);
    load_row(rw + (int64_t)(j + 32) * ROW_WORDS, v1);
    const bool w0 = __float_as_uint(v0[9]) == gen, w1 = __float_as_uint(v1[9]) == gen;
#pragma unroll
    for (int c = 0; c < 9; c++) acc[c] += (w0 ? v0[c] : 0.f) + (w1 ? v1[c] : 0.f);
  }
  if (j < nr) {
    float v[ROW_WORDS];
    load_row(rw + (int64_t)j * ROW_WORDS, v);
    const bool ok = __float_as_uint(v[9]) == gen;
#pragma unroll
    for (int c = 0; c < 9; c++) acc[c] += ok ? v[c] : 0.f;
  }
  // level xor 16: keep half 8 channels, receive the partner's copy of them
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
    const bool hi = lane & (2 * w);
#pragma unroll
    for (int k = 0; k < w; k++) {
      const float keep = hi ? acc[w + k] : acc[k];
      const float give = hi ? acc[k] : acc[w + k];
      acc[k] = keep + __shfl_xor_sync(FULLMASK, give, 2 * w);
    }
  }
  *ch = ((lane >> 4) & 1) << 3 | ((lane >> 3) & 1) << 2 | ((lane >> 2) & 1) << 1 | ((lane >> 1) & 1);
  return acc[0] + __shfl_xor_sync(FULLMASK, acc[0], 1);
}

// First Gaussian whose rows end after instance row `lo` (ends = roff + tiles
// are non-decreasing): 32-ary warp search, warp-uniform result.
__device__ __forceinline__ int64_t merge_find(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ roff,
                                              int64_t n, uint32_t lo, int lane) {
  int64_t a = 0, b = n - 1;  // the answer is in [a, b]; rows end after lo at b
  while (b - a >= 32) {
    const int64_t step = (b - a + 31) / 32;
    const int64_t p = min(a + (int64_t)lane * step, b);
    const unsigned m = __ballot_sync(FULLMASK, roff[p] + tiles[p] > lo);
    if (m & 1u) return a;
    if (m == 0u) {
      a = min(a + 31 * step, b) + 1;
    } else {
      const int f = __ffs(m) - 1;
      b = min(a + (int64_t)f * step, b);
      a = a + (int64_t)(f - 1) * step + 1;
    }
  }
  const int64_t p = a + lane;
  const unsigned m = __ballot_sync(FULLMASK, p <= b && roff[p] + tiles[p] > lo);
  return a + (__ffs(m) - 1);
}

__global__ void __launch_bounds__(MERGE_WARPS * 32, 4) k_merge_big(int64_t n, const uint32_t* __restrict__ tiles,
                                                                const uint32_t* __restrict__ roff,
                                                                float* __restrict__ rows) {
  griddep_wait();
  const uint32_t gen = rows_generation(rows);
  rows += ROWS_HEAD;
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * MERGE_WARPS;
  const int64_t w = (int64_t)blockIdx.x * MERGE_WARPS + (threadIdx.x >> 5);
  const uint32_t m_rows = roff[n - 1] + tiles[n - 1];
  const int64_t n_chunks = (m_rows + MERGE_CHUNK - 1) / MERGE_CHUNK;
  const int64_t c0 = w * n_chunks / n_warps, c1 = (w + 1) * n_chunks / n_warps;
  if (c0 >= c1) return;
  const uint32_t lo0 = (uint32_t)(c0 * MERGE_CHUNK), hi1 = (uint32_t)min((int64_t)m_rows, c1 * MERGE_CHUNK);
  int64_t g = merge_find(tiles, roff, n, lo0, lane);
  while (g < n) {
    const int64_t gl = g + lane;
    uint32_t s = UINT32_MAX, nt = 0;
    if (gl < n) {
      s = roff[gl];
      nt = tiles[gl];
    }
    const bool in = gl < n && s < hi1;
    unsigned big = __ballot_sync(FULLMASK, in && nt > MERGE_BIG);
    while (big) {
      const int l = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t sl = __shfl_sync(FULLMASK, s, l), el = sl + __shfl_sync(FULLMASK, nt, l);
      // the Gaussian's rows inside this warp's range, one portion per chunk
      uint32_t p0 = max(sl, lo0);
      while (p0 < min(el, hi1)) {
        const uint32_t p1 = min(min(el, hi1), (p0 / MERGE_CHUNK + 1) * MERGE_CHUNK);
        float* rw = rows + (int64_t)p0 * ROW_WORDS;
        int ch;
        const float v = merge_rows_warp(rw, p1 - p0, lane, &ch, gen);
        __syncwarp();  // every lane's reads of the head row are done before it is overwritten
        if (!(lane & 1) && ch < 9) rw[ch] = v;
        p0 = p1;
      }
    }
    if (__ballot_sync(FULLMASK, in) != FULLMASK) break;
    g += 32;
  }
}

// ------------------------------------------------------------------ geometry chain
constexpr int CHAIN_ROWS = 64;
constexpr int CHAIN_STAGE_FLOATS = ROW_WORDS * 448;  // 17.5 KB: 10 CTAs per SM

template <bool FUSED>
__global__ void __launch_bounds__(CHAIN_ROWS) k_chain_geo(CamF cam, int64_t n, const float* __restrict__ pos,
                                                          float* __restrict__ rot, float* __restrict__ ls,
                                                          float* __restrict__ logit_p,
                                                          const uint32_t* __restrict__ tiles,
                                                          const uint32_t* __restrict__ roff, float* __restrict__ rows,
                                                          float* __restrict__ grads, int S, int accumulate,
                                                          float* __restrict__ stats, AdamArgsF adam) {
  griddep_wait();
  const uint32_t gen = rows_generation(rows);
  rows += ROWS_HEAD;
  __shared__ __align__(16) float s_rows[CHAIN_STAGE_FLOATS + 4];
  __shared__ uint64_t mbar;
  const int64_t i0 = (int64_t)blockIdx.x * CHAIN_ROWS;
  const int rows_here = (int)min((int64_t)CHAIN_ROWS, n - i0);
  const int64_t i = i0 + threadIdx.x;
  const bool mine = threadIdx.x < rows_here;
  const uint32_t r_begin = roff[i0];
  const uint32_t r_end = roff[i0 + rows_here - 1] + tiles[i0 + rows_here - 1];
  // the CTA's rows are one contiguous range: one 16-byte aligned TMA bulk
  // copy when it fits (inst_rows has >= 16 B slack), else direct reads
  const int64_t n_floats = (int64_t)(r_end - r_begin) * ROW_WORDS;
  const int64_t b0 = (int64_t)r_begin * ROW_WORDS * 4 + ROWS_HEAD * 4, a0 = b0 & ~(int64_t)15;
  const int pad = (int)((b0 - a0) >> 2);
  const int64_t bytes = ((b0 + n_floats * 4 - a0) + 15) & ~(int64_t)15;
  const bool staged = n_floats > 0 && bytes <= (int64_t)sizeof(s_rows);
  const int64_t ns = row_stride(n);
  // fused: the CTA's rotation / log-scale / logit rows and their moments come
  // in by TMA bulk copies next to the instance rows ([param | m | v] x
  // [rot 4 | log-scale 3 | logit 1] x CHAIN_ROWS, dynamic shared memory)
  extern __shared__ __align__(16) float s_adam[];
  if (threadIdx.x == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (staged || FUSED) {
    if (threadIdx.x == 0) {
      const uint32_t rows4 = (uint32_t)min((int64_t)CHAIN_ROWS, ns - i0);
      mbar_expect_tx(&mbar, (staged ? (uint32_t)bytes : 0u) + (FUSED ? 3u * 32u * rows4 : 0u));
      if (staged) bulk_g2s(s_rows, reinterpret_cast<const char*>(rows - ROWS_HEAD) + a0, (uint32_t)bytes, &mbar);
      if (FUSED) {
        const float* src[3] = {rot, adam.m + 3 * ns, adam.v + 3 * ns};
        for (int t = 0; t < 3; t++) {
          const float* base = src[t];  // rotation region; log-scales at +4ns, logits at +7ns
          float* d = s_adam + t * 8 * CHAIN_ROWS;
          bulk_g2s(d, base + i0 * 4, rows4 * 16, &mbar);
          bulk_g2s(d + 4 * CHAIN_ROWS, base + 4 * ns + i0 * 3, rows4 * 12, &mbar);
          bulk_g2s(d + 7 * CHAIN_ROWS, base + 7 * ns + i0, rows4 * 4, &mbar);
        }
      }
    }
  }
  // the row's own global reads are issued before waiting for the bulk copies
  uint32_t nt = 0, s0 = 0;
  float px = 0.f, py = 0.f, pz = 0.f, st0 = 0.f, st1 = 0.f;
  if (mine) {
    nt = tiles[i];
    s0 = roff[i];
    px = pos[i * 3];
    py = pos[i * 3 + 1];
    pz = pos[i * 3 + 2];
    if (stats) {
      st0 = stats[i];
      st1 = stats[n + i];
    }
  }
  // accumulating (view batches): the gradient entries this row adds to are
  // requested now, so their latency overlaps the staging wait and the chain
  float acc[13];
  if (!FUSED && accumulate && mine && nt > 0) {
    const float* gb[6] = {grads + i * 3, grads + 3 * ns + i * 4, grads + 7 * ns + i * 3, grads + 10 * ns + i,
                          grads + (int64_t)S * ns + i, grads + (int64_t)(S + 1) * ns + i};
    const int cnt[6] = {3, 4, 3, 1, 1, 1};
    int e = 0;
#pragma unroll
    for (int b = 0; b < 6; b++)
#pragma unroll
      for (int j = 0; j < cnt[b]; j++) acc[e++] = gb[b][j];
  }
  if (staged || FUSED) mbar_wait(&mbar, 0);
  if (!mine) return;
  // bincount merge (backward.py:110-118): ascending tile order; Gaussians with
  // more than MERGE_BIG rows were reduced into their first row by k_merge_big
  float pr[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (nt > 0) {
    const float* rw = staged ? s_rows + pad + (int64_t)(s0 - r_begin) * ROW_WORDS : rows + (int64_t)s0 * ROW_WORDS;
    if (nt <= MERGE_BIG) {
      // rows of slots no pixel walked carry a stale tag: zero.  Separate
      // shared / global loops so the staged one compiles to LDS.64.
      auto merge = [&](const float* r) {
        for (uint32_t j = 0; j < nt; j++) {
          float v[ROW_WORDS];
          load_row(r + j * ROW_WORDS, v);
          const bool ok = __float_as_uint(v[9]) == gen;
#pragma unroll
          for (int c = 0; c < 9; c++) pr[c] += ok ? v[c] : 0.f;
        }
      };
      if (staged)
        merge(s_rows + pad + (int64_t)(s0 - r_begin) * ROW_WORDS);
      else
        merge(rows + (int64_t)s0 * ROW_WORDS);
    } else {
      // k_merge_big left one partial sum per chunk the rows span: the first
      // row and every chunk boundary inside the range
#pragma unroll
      for (int c = 0; c < 9; c++) pr[c] = rw[c];
      for (uint32_t h = (s0 / MERGE_CHUNK + 1) * MERGE_CHUNK; h < s0 + nt; h += MERGE_CHUNK)
#pragma unroll
        for (int c = 0; c < 9; c++) pr[c] += rw[(int64_t)(h - s0) * ROW_WORDS + c];
    }
  }
  float* g_pos = grads;
  float* g_rot = grads + 3 * ns;
  float* g_ls = grads + 7 * ns;
  float* g_logit = grads + 10 * ns;
  float* g_screen = grads + (int64_t)S * ns;
  float* g_vis = grads + (int64_t)(S + 1) * ns;
  const int tr = threadIdx.x;
  const float* s_p = s_adam;
  const float* s_m = s_adam + 8 * CHAIN_ROWS;
  const float* s_v = s_adam + 16 * CHAIN_ROWS;
  const float4 q4 = FUSED ? *reinterpret_cast<const float4*>(s_p + tr * 4)
                          : *reinterpret_cast<const float4*>(rot + i * 4);
  float grot[4] = {0.f, 0.f, 0.f, 0.f}, dls[3] = {0.f, 0.f, 0.f}, dpos[3] = {0.f, 0.f, 0.f}, screen = 0.f;
  float* dst = rows + (int64_t)roff[i] * ROW_WORDS;
  if (nt > 0) {
    dst[0] = pr[0];
    dst[1] = pr[1];
    dst[2] = pr[2];

    // ---- forward quantities of projection.py:76-128 (float32 restatement)
    const float* R = cam.R;
    const float x = R[0] * px + R[1] * py + R[2] * pz + cam.t[0];
    const float y = R[3] * px + R[4] * py + R[5] * pz + cam.t[1];
    const float z = R[6] * px + R[7] * py + R[8] * pz + cam.t[2];
    const float fx = cam.fx, fy = cam.fy;
    const float limx = 1.3f * ((float)cam.width / (2.f * fx)), limy = 1.3f * ((float)cam.height / (2.f * fy));
    const float iz = 1.f / z;
    const float txr = x * iz, tyr = y * iz;
    const float mulx = (txr > -limx && txr < limx) ? 1.f : 0.f;
    const float muly = (tyr > -limy && tyr < limy) ? 1.f : 0.f;
    const float txc = fminf(fmaxf(txr, -limx), limx), tyc = fminf(fmaxf(tyr, -limy), limy);
    // field.py:40-75: R(q) from the normalised quaternion, M = R diag(e^s)
    const float qnorm = sqrtf(q4.x * q4.x + q4.y * q4.y + q4.z * q4.z + q4.w * q4.w);
    const float iq = 1.f / qnorm;
    const float qw = q4.x * iq, qx = q4.y * iq, qy = q4.z * iq, qz = q4.w * iq;
    float rm[9];
    rm[0] = 1.f - 2.f * (qy * qy + qz * qz);
    rm[1] = 2.f * (qx * qy - qw * qz);
    rm[2] = 2.f * (qx * qz + qw * qy);
    rm[3] = 2.f * (qx * qy + qw * qz);
    rm[4] = 1.f - 2.f * (qx * qx + qz * qz);
    rm[5] = 2.f * (qy * qz - qw * qx);
    rm[6] = 2.f * (qx * qz - qw * qy);
    rm[7] = 2.f * (qy * qz + qw * qx);
    rm[8] = 1.f - 2.f * (qx * qx + qy * qy);
    const float* lsr = FUSED ? s_p + 4 * CHAIN_ROWS + tr * 3 : ls + i * 3;
    const float sc[3] = {__expf(lsr[0]), __expf(lsr[1]), __expf(lsr[2])};
    float m[9], cw[9], tmp[9], cc[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) m[a * 3 + b] = rm[a * 3 + b] * sc[b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) cw[a * 3 + b] = m[a * 3] * m[b * 3] + m[a * 3 + 1] * m[b * 3 + 1] + m[a * 3 + 2] * m[b * 3 + 2];
    // cc = R cw R^T
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) tmp[a * 3 + b] = R[a * 3] * cw[b] + R[a * 3 + 1] * cw[3 + b] + R[a * 3 + 2] * cw[6 + b];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) cc[a * 3 + b] = tmp[a * 3] * R[b * 3] + tmp[a * 3 + 1] * R[b * 3 + 1] + tmp[a * 3 + 2] * R[b * 3 + 2];
    const float fx_z = fx * iz, fy_z = fy * iz;
    const float j02 = -fx * txc * iz, j12 = -fy * tyc * iz;
    const float A = fx_z * (fx_z * cc[0] + j02 * cc[2]) + j02 * (fx_z * cc[2] + j02 * cc[8]) + 0.3f;
    const float B = fx_z * (fy_z * cc[1] + j12 * cc[2]) + j02 * (fy_z * cc[5] + j12 * cc[8]);
    const float C = fy_z * (fy_z * cc[4] + j12 * cc[5]) + j12 * (fy_z * cc[5] + j12 * cc[8]) + 0.3f;
    const float idet = 1.f / (A * C - B * B);
    const float qa = C * idet, qb = -B * idet, qc = A * idet;

    // ---- backward.py:502-515: conic -> V2, g_v2 = -Q G Q
    const float g00 = pr[6], g01 = 0.5f * pr[7], g11 = pr[8];
    const float t00 = qa * g00 + qb * g01, t01 = qa * g01 + qb * g11;
    const float t10 = qb * g00 + qc * g01, t11 = qb * g01 + qc * g11;
    const float gv2[4] = {-(t00 * qa + t01 * qb), -(t00 * qb + t01 * qc), -(t10 * qa + t11 * qb),
                          -(t10 * qb + t11 * qc)};
    const float J[6] = {fx_z, 0.f, j02, 0.f, fy_z, j12};
    // gJ = 2 gv2 J cc ; gv3 = J^T gv2 J
    float jc[6];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) jc[a * 3 + l] = J[a * 3] * cc[l] + J[a * 3 + 1] * cc[3 + l] + J[a * 3 + 2] * cc[6 + l];
    float gJ[6];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) gJ[a * 3 + l] = 2.f * (gv2[a * 2] * jc[l] + gv2[a * 2 + 1] * jc[3 + l]);
    float gj[6];  // gv2 J
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) gj[a * 3 + l] = gv2[a * 2] * J[l] + gv2[a * 2 + 1] * J[3 + l];
    float gv3[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) gv3[a * 3 + l] = J[a] * gj[l] + J[3 + a] * gj[3 + l];
    // gw = R^T gv3 R
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) tmp[a * 3 + l] = R[a] * gv3[l] + R[3 + a] * gv3[3 + l] + R[6 + a] * gv3[6 + l];
    float gw[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int l = 0; l < 3; l++) gw[a * 3 + l] = tmp[a * 3] * R[l] + tmp[a * 3 + 1] * R[3 + l] + tmp[a * 3 + 2] * R[6 + l];
    // backward.py:537-553: J and the projected mean -> camera point -> world
    const float iz2 = iz * iz;
    float dcx = gJ[2] * (-fx * mulx * iz2);
    float dcy = gJ[5] * (-fy * muly * iz2);
    float dcz = gJ[0] * (-fx * iz2) + gJ[4] * (-fy * iz2) + gJ[2] * fx * (mulx * x * iz + txc) * iz2 +
                gJ[5] * fy * (muly * y * iz + tyc) * iz2;
    dcx += pr[4] * fx * iz;
    dcy += pr[5] * fy * iz;
    dcz += -pr[4] * fx * x * iz2 - pr[5] * fy * y * iz2;
    dpos[0] = dcx * R[0] + dcy * R[3] + dcz * R[6];
    dpos[1] = dcx * R[1] + dcy * R[4] + dcz * R[7];
    dpos[2] = dcx * R[2] + dcy * R[5] + dcz * R[8];
    // _cov_to_rotation_scale (backward.py:562-612)
    float gs[9], dm[9], drot[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int b = 0; b < 3; b++) gs[a * 3 + b] = gw[a * 3 + b] + gw[b * 3 + a];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
      for (int k = 0; k < 3; k++) {
        dm[a * 3 + k] = gs[a * 3] * m[k] + gs[a * 3 + 1] * m[3 + k] + gs[a * 3 + 2] * m[6 + k];
        drot[a * 3 + k] = dm[a * 3 + k] * sc[k];
      }
#pragma unroll
    for (int j = 0; j < 3; j++) dls[j] = (dm[j] * rm[j] + dm[3 + j] * rm[3 + j] + dm[6 + j] * rm[6 + j]) * sc[j];
    const float dqw = 2.f * (-qz * drot[1] + qy * drot[2] + qz * drot[3] - qx * drot[5] - qy * drot[6] + qx * drot[7]);
    const float dqx = 2.f * (qy * drot[1] + qz * drot[2] + qy * drot[3] - 2.f * qx * drot[4] - qw * drot[5] +
                             qz * drot[6] + qw * drot[7] - 2.f * qx * drot[8]);
    const float dqy = 2.f * (-2.f * qy * drot[0] + qx * drot[1] + qw * drot[2] + qx * drot[3] + qz * drot[5] -
                             qw * drot[6] + qz * drot[7] - 2.f * qy * drot[8]);
    const float dqz = 2.f * (-2.f * qz * drot[0] - qw * drot[1] + qx * drot[2] + qw * drot[3] - 2.f * qz * drot[4] +
                             qy * drot[5] + qx * drot[6] + qy * drot[7]);
    const float rad = dqw * qw + dqx * qx + dqy * qy + dqz * qz;
    grot[0] = (dqw - rad * qw) * iq;
    grot[1] = (dqx - rad * qx) * iq;
    grot[2] = (dqy - rad * qy) * iq;
    grot[3] = (dqz - rad * qz) * iq;
    screen = sqrtf(pr[4] * pr[4] + pr[5] * pr[5]) * (0.5f * (float)max(cam.width, cam.height));
  }  // visible
  const bool vis = nt > 0;
  if (FUSED) {
    // dense Adam: invisible rows step with a zero gradient like the reference
    float4 m_rot = *reinterpret_cast<const float4*>(s_m + tr * 4);
    float4 v_rot = *reinterpret_cast<const float4*>(s_v + tr * 4);
    float4 qn;
    qn.x = adam_step(q4.x, grot[0], m_rot.x, v_rot.x, adam.c[1]);
    qn.y = adam_step(q4.y, grot[1], m_rot.y, v_rot.y, adam.c[1]);
    qn.z = adam_step(q4.z, grot[2], m_rot.z, v_rot.z, adam.c[1]);
    qn.w = adam_step(q4.w, grot[3], m_rot.w, v_rot.w, adam.c[1]);
    *reinterpret_cast<float4*>(rot + i * 4) = qn;
    *reinterpret_cast<float4*>(adam.m + 3 * ns + i * 4) = m_rot;
    *reinterpret_cast<float4*>(adam.v + 3 * ns + i * 4) = v_rot;
#pragma unroll
    for (int j = 0; j < 3; j++) {
      float mj = s_m[4 * CHAIN_ROWS + tr * 3 + j], vj = s_v[4 * CHAIN_ROWS + tr * 3 + j];
      ls[i * 3 + j] = adam_step(s_p[4 * CHAIN_ROWS + tr * 3 + j], dls[j], mj, vj, adam.c[2]);
      adam.m[7 * ns + i * 3 + j] = mj;
      adam.v[7 * ns + i * 3 + j] = vj;
    }
    float m_lo = s_m[7 * CHAIN_ROWS + tr], v_lo = s_v[7 * CHAIN_ROWS + tr];
    logit_p[i] = adam_step(s_p[7 * CHAIN_ROWS + tr], pr[3], m_lo, v_lo, adam.c[3]);
    adam.m[10 * ns + i] = m_lo;
    adam.v[10 * ns + i] = v_lo;
    if (vis) {
      dst[3] = dpos[0];
      dst[4] = dpos[1];
      dst[5] = dpos[2];
    }
  } else if (accumulate) {
    if (vis) {  // acc: the entries read at entry (same order as below)
#pragma unroll
      for (int j = 0; j < 3; j++) g_pos[i * 3 + j] = acc[j] + dpos[j];
#pragma unroll
      for (int j = 0; j < 4; j++) g_rot[i * 4 + j] = acc[3 + j] + grot[j];
#pragma unroll
      for (int j = 0; j < 3; j++) g_ls[i * 3 + j] = acc[7 + j] + dls[j];
      g_logit[i] = acc[10] + pr[3];
      g_screen[i] = acc[11] + screen;
      g_vis[i] = acc[12] + 1.f;
    }
  } else {
    for (int j = 0; j < 3; j++) g_pos[i * 3 + j] = dpos[j];
    *reinterpret_cast<float4*>(g_rot + i * 4) = make_float4(grot[0], grot[1], grot[2], grot[3]);
    for (int j = 0; j < 3; j++) g_ls[i * 3 + j] = dls[j];
    g_logit[i] = pr[3];
    g_screen[i] = screen;
    g_vis[i] = vis ? 1.f : 0.f;
  }
  if (stats && vis) {
    stats[i] = st0 + screen;
    stats[n + i] = st1 + 1.f;
  }
}

// ------------------------------------------------------------------ SH chain
// sh.py:36-65 basis in float32.
template <int DEG>
__device__ __forceinline__ void sh_basis32(float x, float y, float z, float* b) {
  b[0] = 0.28209479177387814f;
  if (DEG >= 1) {
    b[1] = -0.4886025119029199f * y;
    b[2] = 0.4886025119029199f * z;
    b[3] = -0.4886025119029199f * x;
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = 1.0925484305920792f * (x * y);
    b[5] = -1.0925484305920792f * (y * z);
    b[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    b[7] = -1.0925484305920792f * (x * z);
    b[8] = 0.5462742152960396f * (xx - yy);
    if (DEG >= 3) {
      b[9] = -0.5900435899266435f * y * (3.f * xx - yy);
      b[10] = 2.890611442640554f * (x * y) * z;
      b[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
      b[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
      b[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
      b[14] = 1.445305721320277f * z * (xx - yy);
      b[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
    }
  }
}

// sum_k v_k dY_k/ddir (sh.py:68-111), written term by term.
template <int DEG>
__device__ __forceinline__ void sh_dir_grad32(const float* v, float x, float y, float z, float* g) {
  const float C1 = 0.4886025119029199f;
  g[0] = g[1] = g[2] = 0.f;
  if (DEG >= 1) {
    g[1] += v[1] * (-C1);
    g[2] += v[2] * C1;
    g[0] += v[3] * (-C1);
  }
  if (DEG >= 2) {
    const float C20 = 1.0925484305920792f, C21 = -1.0925484305920792f, C22 = 0.31539156525252005f,
                C23 = -1.0925484305920792f, C24 = 0.5462742152960396f;
    g[0] += v[4] * (C20 * y) + v[6] * (C22 * (-2.f * x)) + v[7] * (C23 * z) + v[8] * (C24 * (2.f * x));
    g[1] += v[4] * (C20 * x) + v[5] * (C21 * z) + v[6] * (C22 * (-2.f * y)) + v[8] * (C24 * (-2.f * y));
    g[2] += v[5] * (C21 * y) + v[6] * (C22 * (4.f * z)) + v[7] * (C23 * x);
  }
  if (DEG >= 3) {
    const float C30 = -0.5900435899266435f, C31 = 2.890611442640554f, C32 = -0.4570457994644658f,
                C33 = 0.3731763325901154f, C34 = -0.4570457994644658f, C35 = 1.445305721320277f,
                C36 = -0.5900435899266435f;
    const float xx = x * x, yy = y * y, zz = z * z;
    g[0] += v[9] * (C30 * 6.f * x * y) + v[10] * (C31 * y * z) + v[11] * (C32 * (-2.f * x * y)) +
            v[12] * (C33 * (-6.f * x * z)) + v[13] * (C34 * (4.f * zz - 3.f * xx - yy)) +
            v[14] * (C35 * (2.f * x * z)) + v[15] * (C36 * (3.f * xx - 3.f * yy));
    g[1] += v[9] * (C30 * (3.f * xx - 3.f * yy)) + v[10] * (C31 * x * z) + v[11] * (C32 * (4.f * zz - xx - 3.f * yy)) +
            v[12] * (C33 * (-6.f * y * z)) + v[13] * (C34 * (-2.f * x * y)) + v[14] * (C35 * (-2.f * y * z)) +
            v[15] * (C36 * (-6.f * x * y));
    g[2] += v[10] * (C31 * x * y) + v[11] * (C32 * (8.f * y * z)) + v[12] * (C33 * (6.f * zz - 3.f * xx - 3.f * yy)) +
            v[13] * (C34 * (8.f * x * z)) + v[14] * (C35 * (xx - yy));
  }
}

constexpr int SH_LANES = 4;
constexpr int SH_THREADS = 256;
constexpr int SH_ROWS = SH_THREADS / SH_LANES;

// Accumulating (view batches): the field rows the view sees, listed (any
// order: every row's update is independent), so the SH pass runs full warps
// over them alone.  list[0] = count (zeroed beforehand), rows from list[1].
constexpr int LIST_THREADS = 1024;
__global__ void __launch_bounds__(LIST_THREADS) k_list_visible(int64_t n, const uint32_t* __restrict__ tiles,
                                                               uint32_t* __restrict__ list) {
  griddep_wait();
  __shared__ uint32_t s_cnt[LIST_THREADS / 32];
  __shared__ uint32_t s_base;
  const int64_t i = (int64_t)blockIdx.x * LIST_THREADS + threadIdx.x;
  const bool vis = i < n && tiles[i] != 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(FULLMASK, vis);
  if (lane == 0) s_cnt[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {  // one counter update per CTA, the warps' offsets in order
    uint32_t run = 0;
    for (int w = 0; w < LIST_THREADS / 32; w++) {
      const uint32_t c = s_cnt[w];
      s_cnt[w] = run;
      run += c;
    }
    s_base = run ? atomicAdd(list, run) : 0u;
  }
  __syncthreads();
  if (vis) list[1 + s_base + s_cnt[warp] + __popc(b & ((1u << lane) - 1u))] = (uint32_t)i;
}

// Lane q of a row owns coefficients k = q*KL + j (j < KL, k < K) of every
// channel; at SH3 that is one float4 per channel, read and written directly.
// list (optional, accumulating): the rows to process, from k_list_visible.
template <int DEG>
__global__ void __launch_bounds__(SH_THREADS, 4) k_chain_sh(CamF cam, int64_t n, float* __restrict__ pos,
                                                         float* __restrict__ sh, const uint32_t* __restrict__ tiles,
                                                         const uint32_t* __restrict__ roff,
                                                         const float4* __restrict__ color,
                                                         const float* __restrict__ rows, float* __restrict__ grads,
                                                         int accumulate, const uint32_t* __restrict__ list) {
  griddep_wait();
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int W = 3 * K;
  constexpr int KL = (K + 3) / 4;
  constexpr bool VEC = (K == 16);
  const int64_t slot = (int64_t)blockIdx.x * SH_ROWS + (threadIdx.x >> 2);
  const int64_t n_slots = list ? (int64_t)list[0] : n;
  if ((int64_t)blockIdx.x * SH_ROWS >= n_slots) return;  // the whole CTA is past the listed rows
  const int64_t i = list ? (slot < n_slots ? (int64_t)list[1 + slot] : n) : slot;
  const int q = threadIdx.x & 3;
  const bool row_ok = i < n;
  const int64_t ii = row_ok ? i : n - 1;  // out-of-range lanes shadow the last row (shuffles need them)
  const int64_t ns = row_stride(n);
  const bool vis = row_ok && tiles[ii] != 0;
  const float* rw = rows + ROWS_HEAD + (vis ? (int64_t)roff[ii] * ROW_WORDS : 0);
  float* shrow = sh + ii * W;
  float* grow = grads + 11 * ns + ii * W;
  // the lane's coefficients: c[ch][j] = sh[ch*K + q*KL + j] (an invisible
  // row's gradient is zero: no coefficient or position is read for it)
  float cf[3][KL];
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    if (!vis) {
#pragma unroll
      for (int j = 0; j < KL; j++) cf[ch][j] = 0.f;
    } else if (VEC) {
      const float4 v4 = *reinterpret_cast<const float4*>(shrow + ch * K + q * 4);
      cf[ch][0] = v4.x;
      cf[ch][1] = v4.y;
      cf[ch][2] = v4.z;
      cf[ch][3] = v4.w;
    } else {
#pragma unroll
      for (int j = 0; j < KL; j++) {
        const int k = q * KL + j;
        cf[ch][j] = k < K ? shrow[ch * K + k] : 0.f;
      }
    }
  }
  // direction (sh.py:114-124), recomputed by each lane
  const float ox = vis ? pos[ii * 3] - cam.center[0] : 1.f, oy = vis ? pos[ii * 3 + 1] - cam.center[1] : 0.f,
              oz = vis ? pos[ii * 3 + 2] - cam.center[2] : 0.f;
  const float r = sqrtf(ox * ox + oy * oy + oz * oz);
  const float rs = fmaxf(r, 1e-12f);
  const float irs = 1.f / rs;
  const float dx = ox * irs, dy = oy * irs, dz = oz * irs;
  float basis[16];
  sh_basis32<DEG>(dx, dy, dz, basis);
  float bown[KL];  // basis of the lane's coefficients
#pragma unroll
  for (int j = 0; j < KL; j++) {
    float b = 0.f;
#pragma unroll
    for (int qq = 0; qq < 4; qq++)
      if (qq * KL + j < K) b = (q == qq) ? basis[qq * KL + j] : b;
    bown[j] = (q * KL + j < K) ? b : 0.f;
  }
  // colour gradient through the clamp (sh.py:128-131); the masks were decided
  // by the float64 preprocess (colour .w bits), not re-derived in fp32
  float dcol[3] = {0.f, 0.f, 0.f};
  if (vis) {
    const int pass = __float_as_int(color[ii].w);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) dcol[ch] = (pass >> ch) & 1 ? rw[ch] : 0.f;
  }
  // direction gradient: v_k = sum_c dcol_c coeff_ck for the lane's k (zero
  // elsewhere), contracted with dY/ddir, reduced over the 4 lanes
  float vfull[16];
#pragma unroll
  for (int k = 0; k < 16; k++) vfull[k] = 0.f;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const int qq = k / KL, j = k % KL;
    const float vk = dcol[0] * cf[0][j] + dcol[1] * cf[1][j] + dcol[2] * cf[2][j];
    vfull[k] = (q == qq) ? vk : 0.f;
  }
  float gd[3];
  sh_dir_grad32<DEG>(vfull, dx, dy, dz, gd);
#pragma unroll
  for (int d = 0; d < 3; d++) {
    gd[d] += __shfl_xor_sync(FULLMASK, gd[d], 1);
    gd[d] += __shfl_xor_sync(FULLMASK, gd[d], 2);
  }
  const float radial = gd[0] * dx + gd[1] * dy + gd[2] * dz;
  const float dpos_sh[3] = {(gd[0] - radial * dx) * irs, (gd[1] - radial * dy) * irs, (gd[2] - radial * dz) * irs};
  // accumulating (view batches): an invisible row adds exact zeros -- skip
  // its read-modify-write of the gradient rows
  if (!row_ok || (accumulate && !vis)) return;
  if (q == 0 && vis) {
    float* g_pos = grads + i * 3;
#pragma unroll
    for (int d = 0; d < 3; d++) g_pos[d] += dpos_sh[d];
  }
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    if (VEC) {
      float4 g4 = make_float4(dcol[ch] * bown[0], dcol[ch] * bown[1], dcol[ch] * bown[2], dcol[ch] * bown[3]);
      float4* dstp = reinterpret_cast<float4*>(grow + ch * K + q * 4);
      if (accumulate) {
        const float4 o = *dstp;
        g4.x += o.x;
        g4.y += o.y;
        g4.z += o.z;
        g4.w += o.w;
      }
      *dstp = g4;
    } else {
#pragma unroll
      for (int j = 0; j < KL; j++) {
        const int k = q * KL + j;
        if (k < K) {
          const float g = dcol[ch] * bown[j];
          grow[ch * K + k] = accumulate ? grow[ch * K + k] + g : g;
        }
      }
    }
  }
}

// Fused SH chain + Adam with the CTA's parameter, first- and second-moment
// rows (and the position rows) staged by TMA bulk copies issued at entry: six
// contiguous ranges per CTA, ~39 KB in flight per CTA at SH3, so the dense
// Adam stream is not bounded by per-thread load latency.  The per-row gathers
// of the chain (tile count, merged colour / position gradient, clamp bits)
// overlap the copies.  Results are stored straight to global memory.
constexpr int SHA_ROWS = 64;  // 4 lanes per row, 256 threads

template <int DEG>
__global__ void __launch_bounds__(SH_THREADS, 4) k_chain_sh_adam(CamF cam, int64_t n, float* __restrict__ pos,
                                                              float* __restrict__ sh,
                                                              const uint32_t* __restrict__ tiles,
                                                              const uint32_t* __restrict__ roff,
                                                              const float4* __restrict__ color,
                                                              const float* __restrict__ rows, AdamArgsF adam) {
  griddep_wait();
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int W = 3 * K;
  constexpr int KL = (K + 3) / 4;
  constexpr bool VEC = (K == 16);
  extern __shared__ __align__(16) float s_st[];  // sh | m | v  (SHA_ROWS*W each), pos | mpos | vpos (SHA_ROWS*3)
  __shared__ uint64_t mbar;
  float* s_sh = s_st;
  float* s_m = s_st + SHA_ROWS * W;
  float* s_v = s_st + 2 * SHA_ROWS * W;
  float* s_p = s_st + 3 * SHA_ROWS * W;
  float* s_mp = s_p + SHA_ROWS * 3;
  float* s_vp = s_p + 2 * SHA_ROWS * 3;
  const int64_t i0 = (int64_t)blockIdx.x * SHA_ROWS;
  const int64_t ns = row_stride(n);
  // rows rounded up to 4: the class regions are padded to 4-row strides, so the
  // byte counts stay multiples of 16 and the copies stay inside each region
  const int rows4 = (int)min((int64_t)SHA_ROWS, ns - i0);
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    const uint32_t bw = (uint32_t)rows4 * W * 4, bp = (uint32_t)rows4 * 12;
    mbar_expect_tx(&mbar, 3 * bw + 3 * bp);
    bulk_g2s(s_sh, sh + i0 * W, bw, &mbar);
    bulk_g2s(s_m, adam.m + 11 * ns + i0 * W, bw, &mbar);
    bulk_g2s(s_v, adam.v + 11 * ns + i0 * W, bw, &mbar);
    bulk_g2s(s_p, pos + i0 * 3, bp, &mbar);
    bulk_g2s(s_mp, adam.m + i0 * 3, bp, &mbar);
    bulk_g2s(s_vp, adam.v + i0 * 3, bp, &mbar);
  }
  const int rl = threadIdx.x >> 2, q = threadIdx.x & 3;
  const int64_t i = i0 + rl;
  const bool row_ok = i < n;
  const int64_t ii = row_ok ? i : n - 1;  // out-of-range lanes shadow the last row (shuffles need them)
  const bool vis = row_ok && tiles[ii] != 0;
  const float* rw = rows + ROWS_HEAD + (vis ? (int64_t)roff[ii] * ROW_WORDS : 0);
  // colour gradient through the clamp (sh.py:128-131), masks from the fp64 preprocess
  float dcol[3] = {0.f, 0.f, 0.f}, gp_geo = 0.f;
  if (vis) {
    const int pass = __float_as_int(color[ii].w);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) dcol[ch] = (pass >> ch) & 1 ? rw[ch] : 0.f;
    if (q < 3) gp_geo = rw[3 + q];
  }
  __syncthreads();  // barrier init visible before anyone waits on it
  mbar_wait(&mbar, 0);
  const float* srow = s_sh + rl * W;
  float cf[3][KL];
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    if (VEC) {
      const float4 v4 = *reinterpret_cast<const float4*>(srow + ch * K + q * 4);
      cf[ch][0] = v4.x;
      cf[ch][1] = v4.y;
      cf[ch][2] = v4.z;
      cf[ch][3] = v4.w;
    } else {
#pragma unroll
      for (int j = 0; j < KL; j++) {
        const int k = q * KL + j;
        cf[ch][j] = k < K ? srow[ch * K + k] : 0.f;
      }
    }
  }
  // direction (sh.py:114-124)
  const float px = s_p[rl * 3], py = s_p[rl * 3 + 1], pz = s_p[rl * 3 + 2];
  const float ox = px - cam.center[0], oy = py - cam.center[1], oz = pz - cam.center[2];
  const float r = sqrtf(ox * ox + oy * oy + oz * oz);
  const float rs = fmaxf(r, 1e-12f);
  const float irs = 1.f / rs;
  const float dx = ox * irs, dy = oy * irs, dz = oz * irs;
  float basis[16];
  sh_basis32<DEG>(dx, dy, dz, basis);
  float bown[KL];
#pragma unroll
  for (int j = 0; j < KL; j++) {
    float b = 0.f;
#pragma unroll
    for (int qq = 0; qq < 4; qq++)
      if (qq * KL + j < K) b = (q == qq) ? basis[qq * KL + j] : b;
    bown[j] = (q * KL + j < K) ? b : 0.f;
  }
  float vfull[16];
#pragma unroll
  for (int k = 0; k < 16; k++) vfull[k] = 0.f;
#pragma unroll
  for (int k = 0; k < K; k++) {
    const int qq = k / KL, j = k % KL;
    const float vk = dcol[0] * cf[0][j] + dcol[1] * cf[1][j] + dcol[2] * cf[2][j];
    vfull[k] = (q == qq) ? vk : 0.f;
  }
  float gd[3];
  sh_dir_grad32<DEG>(vfull, dx, dy, dz, gd);
#pragma unroll
  for (int d = 0; d < 3; d++) {
    gd[d] += __shfl_xor_sync(FULLMASK, gd[d], 1);
    gd[d] += __shfl_xor_sync(FULLMASK, gd[d], 2);
  }
  if (!row_ok) return;
  const float radial = gd[0] * dx + gd[1] * dy + gd[2] * dz;
  // positions: lane q < 3 owns coordinate q (geometric part from k_chain_geo
  // plus the view-direction part)
  if (q < 3) {
    const float gq = q == 0 ? gd[0] : (q == 1 ? gd[1] : gd[2]);
    const float dq = q == 0 ? dx : (q == 1 ? dy : dz);
    const float g = vis ? gp_geo + (gq - radial * dq) * irs : 0.f;
    float mq = s_mp[rl * 3 + q], vq = s_vp[rl * 3 + q];
    const float pq = q == 0 ? px : (q == 1 ? py : pz);
    const int64_t e = i * 3 + q;
    pos[e] = adam_step(pq, g, mq, vq, adam.c[0]);
    adam.m[e] = mq;
    adam.v[e] = vq;
  }
  float* shrow = sh + i * W;
  float* mrow = adam.m + 11 * ns + i * W;
  float* vrow = adam.v + 11 * ns + i * W;
  const float* smr = s_m + rl * W;
  const float* svr = s_v + rl * W;
  const AdamClassF c_dc = adam.c[4], c_rest = adam.c[5];
#pragma unroll
  for (int ch = 0; ch < 3; ch++) {
    float mf[KL], vf[KL], pn[KL];
    if (VEC) {
      const float4 a4 = *reinterpret_cast<const float4*>(smr + ch * K + q * 4);
      const float4 b4 = *reinterpret_cast<const float4*>(svr + ch * K + q * 4);
      mf[0] = a4.x, mf[1] = a4.y, mf[2] = a4.z, mf[3] = a4.w;
      vf[0] = b4.x, vf[1] = b4.y, vf[2] = b4.z, vf[3] = b4.w;
    } else {
#pragma unroll
      for (int j = 0; j < KL; j++) {
        const int k = q * KL + j;
        mf[j] = k < K ? smr[ch * K + k] : 0.f;
        vf[j] = k < K ? svr[ch * K + k] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < KL; j++)
      pn[j] = adam_step(cf[ch][j], dcol[ch] * bown[j], mf[j], vf[j], (q * KL + j == 0) ? c_dc : c_rest);
    if (VEC) {
      *reinterpret_cast<float4*>(shrow + ch * K + q * 4) = make_float4(pn[0], pn[1], pn[2], pn[3]);
      *reinterpret_cast<float4*>(mrow + ch * K + q * 4) = make_float4(mf[0], mf[1], mf[2], mf[3]);
      *reinterpret_cast<float4*>(vrow + ch * K + q * 4) = make_float4(vf[0], vf[1], vf[2], vf[3]);
    } else {
#pragma unroll
      for (int j = 0; j < KL; j++) {
        const int k = q * KL + j;
        if (k < K) {
          shrow[ch * K + k] = pn[j];
          mrow[ch * K + k] = mf[j];
          vrow[ch * K + k] = vf[j];
        }
      }
    }
  }
}

template <int DEG>
static size_t sh_adam_smem() {
  constexpr int K = (DEG + 1) * (DEG + 1);
  return (size_t)(3 * SHA_ROWS * 3 * K + 3 * SHA_ROWS * 3) * sizeof(float);
}

}  // namespace ssr

using namespace ssr;

template <bool FUSED>
static int launch_chain(const ssr_camera* cam, int64_t n, int32_t sh_degree, float* positions, float* rotations,
                        float* log_scales, float* logits, float* sh, ssr_splats splats, float* rows, float* grads,
                        int32_t accumulate, float* stats, const AdamArgsF& adam, cudaStream_t st,
                        uint32_t* row_list = nullptr) {
  const CamF c = to_camf(*cam);
  const int K = (sh_degree + 1) * (sh_degree + 1);
  static int merge_blocks = 0;
  if (!merge_blocks) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_merge_big, MERGE_WARPS * 32, 0);
    merge_blocks = (sms > 0 ? sms : 148) * (occ > 0 ? occ : 4);  // one resident wave
  }
  SSR_TRY(launch_pdl("k_merge_big", k_merge_big, dim3(merge_blocks), dim3(MERGE_WARPS * 32), 0, st, n,
                     (const uint32_t*)splats.tiles, (const uint32_t*)splats.row_offset, rows));
  SSR_TRY(check_launch("k_merge_big"));
  const unsigned blocks = (unsigned)((n + CHAIN_ROWS - 1) / CHAIN_ROWS);
  const size_t geo_smem = FUSED ? 3 * 8 * CHAIN_ROWS * sizeof(float) : 0;
  if (FUSED) {
    static DeviceOnce attr;
    if (!attr.done()) {
      SSR_TRY(check_cuda(cudaFuncSetAttribute(k_chain_geo<FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)geo_smem),
                         "k_chain_geo smem"));
      attr.set();
    }
  }
  SSR_TRY(launch_pdl("k_chain_geo", k_chain_geo<FUSED>, dim3(blocks), dim3(CHAIN_ROWS), geo_smem, st, c, n, positions,
                     rotations, log_scales, logits, (const uint32_t*)splats.tiles, (const uint32_t*)splats.row_offset,
                     rows, grads, 11 + 3 * K, (int)accumulate, stats, adam));
  SSR_TRY(check_launch("k_chain_geo"));
  if (FUSED) {
    const unsigned ablocks = (unsigned)((n + SHA_ROWS - 1) / SHA_ROWS);
#define SSR_SHA(D)                                                                                                \
  do {                                                                                                            \
    const size_t sm = sh_adam_smem<D>();                                                                          \
    static DeviceOnce attr;                                                                                     \
    if (!attr.done()) {                                                                                                  \
      SSR_TRY(check_cuda(cudaFuncSetAttribute(k_chain_sh_adam<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                              (int)sm),                                                           \
                         "k_chain_sh_adam smem"));                                                                \
      attr.set();                                                                                                \
    }                                                                                                             \
    SSR_TRY(launch_pdl("k_chain_sh_adam", k_chain_sh_adam<D>, dim3(ablocks), dim3(SH_THREADS), sm, st, c, n,     \
                       positions, sh, (const uint32_t*)splats.tiles, (const uint32_t*)splats.row_offset,           \
                       (const float4*)splats.color, (const float*)rows, adam));                                  \
  } while (0)
    switch (sh_degree) {
      case 0: SSR_SHA(0); break;
      case 1: SSR_SHA(1); break;
      case 2: SSR_SHA(2); break;
      default: SSR_SHA(3); break;
    }
#undef SSR_SHA
    return check_launch("k_chain_sh_adam");
  }
  const unsigned sblocks = (unsigned)((n + SH_ROWS - 1) / SH_ROWS);
  const uint32_t* list = nullptr;
  if (accumulate && row_list) {  // the view's visible rows only (full warps)
    SSR_TRY(launch_pdl("row list zero", k_zero_words, dim3(1), dim3(32), 0, st, row_list, (int64_t)1));
    SSR_TRY(launch_pdl("k_list_visible", k_list_visible, dim3((unsigned)((n + LIST_THREADS - 1) / LIST_THREADS)),
                       dim3(LIST_THREADS), 0, st, n, (const uint32_t*)splats.tiles, row_list));
    list = row_list;
  }
#define SSR_SH(D)                                                                                         \
  SSR_TRY(launch_pdl("k_chain_sh", k_chain_sh<D>, dim3(sblocks), dim3(SH_THREADS), 0, st, c, n, positions, sh, \
                     (const uint32_t*)splats.tiles, (const uint32_t*)splats.row_offset,                       \
                     (const float4*)splats.color, (const float*)rows, grads, (int)accumulate, list))
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
                         const float* inst_rows, float* grads, int32_t accumulate, float* stats, uint32_t* row_list,
                         void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3 || !grads) {
    set_error("ssr_chain: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  AdamArgsF none{};
  // inst_rows is scratch from here on: the geometry pass parks each Gaussian's
  // merged colour gradient in its own first row for the SH pass
  return launch_chain<false>(cam, n, sh_degree, const_cast<float*>(positions), const_cast<float*>(rotations),
                             const_cast<float*>(log_scales), nullptr, const_cast<float*>(sh), splats,
                             const_cast<float*>(inst_rows), grads, accumulate, stats, none, (cudaStream_t)stream,
                             row_list);
}

extern "C" int ssr_chain_adam(const ssr_camera* cam, int64_t n, int32_t sh_degree, float* params, float* m, float* v,
                              ssr_splats splats, float* inst_rows, float* stats, const double* lr, double lr_sh_rest,
                              const double* bc1, const double* bc2, void* stream) {
  if (!cam || n < 0 || sh_degree < 0 || sh_degree > 3 || !params || !m || !v || !lr || !bc1 || !bc2) {
    set_error("ssr_chain_adam: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  AdamArgsF adam;
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
