// Fused training objective on device (losses.py:55-173):
//   w_l1 * L1 + w_ssim * (1 - SSIM) + w_load * std(soft_count)
// with the analytic SSIM gradient (11-tap sigma=1.5 separable Gaussian,
// zero padding, mean over the interior crop, channel-averaged).
//
// k_ssim_fwd: 32x32 output tile per CTA with a 5-pixel halo in shared
// memory; computes the five blurred moments, the SSIM map and the three
// per-pixel adjoint maps (d_mu, d_gx2, d_gxy), plus per-CTA L1 / SSIM /
// soft-count partial sums (fp64, no atomics).  k_loss_finalize adds them in a
// fixed order (so the scalars and d_soft are bit-identical run to run) and
// turns them into the scalars.  k_ssim_bwd blurs the adjoint maps (the window is self-adjoint)
// and writes d_image and d_soft.
#include <cuda.h>

#include "ssr_common.cuh"

namespace ssr {

constexpr int LT = 32;           // output tile edge
constexpr int HALO = 5;          // (11 - 1) / 2
constexpr int LH = LT + 2 * HALO; // 42
constexpr int LOSS_TERMS = 6;  // l1, ssim, soft d, soft d^2, hard d, hard d^2 per CTA

struct LossAcc {
  double l1_sum, ssim_sum, soft_d, soft_d2, hard_d, hard_d2, soft0, hard0;
  double mean_soft, std_soft;
};

__constant__ float c_win[11];

// Target pixels: float32 in [0, 1], or 8-bit (the reference's image files are
// 8-bit; io/images.py divides by 255) converted on load.  The kernels are
// templated on the format, so the per-element test is resolved at compile time.
struct Target {
  const void* p;
  int u8;
};

template <bool U8>
__device__ __forceinline__ float tgt_at(const Target& t, int i) {
  return U8 ? (float)reinterpret_cast<const uint8_t*>(t.p)[i] * (1.f / 255.f) : reinterpret_cast<const float*>(t.p)[i];
}

__device__ __forceinline__ double block_sum64(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += red[i];
  return s;
}

// Register-blocked separable blur: the horizontal pass gives each thread 8
// consecutive outputs of one row (18 loads per map for 88 taps), the vertical
// pass 4 consecutive outputs of one column (14 loads per map for 44 taps), so
// shared-memory traffic is ~1/4 of a per-output 11-tap loop.
constexpr int HSEG = 8;                 // horizontal outputs per thread
constexpr int HITEMS = LH * (LT / HSEG);  // 168
constexpr int VSEG = 4;                 // vertical outputs per thread (32 x 8 = 256 items)
constexpr int HZS = LT + 1;             // padded row stride of the horizontal results

// The adjoint maps are stored with a zero border of HALO columns on the left
// and HALO rows on top (written by the forward) and rows padded to 4 floats
// (16-byte TMA global strides).  The backward loads each channel's three halo
// tiles with one 3-D TMA copy at non-negative coordinates (a negative tile
// origin faults on this hardware), its rows BP floats apart (16-byte multiple;
// the columns past LH are loaded and not read); past the right and bottom edges
// the copy fills zeros.  Both are the SSIM window's zero padding.
__host__ __device__ __forceinline__ int map_pitch(int W) { return (W + HALO + 3) & ~3; }
__host__ __device__ __forceinline__ size_t map_stride(int W, int H) { return (size_t)map_pitch(W) * (H + HALO); }
constexpr int BP = 44;
constexpr uint32_t BW_TILE_BYTES = 3 * LH * BP * 4;
constexpr uint32_t BW_BUF_BYTES = (BW_TILE_BYTES + 127) & ~127u;  // TMA destinations: 128-byte aligned

template <bool U8>
__global__ void __launch_bounds__(256, 4) k_ssim_fwd(int W, int H, const float* __restrict__ img,
                                                  const Target tgt, const double* __restrict__ soft,
                                                  const int32_t* __restrict__ hard, float* __restrict__ dmaps,
                                                  double* __restrict__ partials) {
  griddep_wait();
  __shared__ float sx[LH][LH + 1], sy[LH][LH + 1];
  __shared__ float hz[5][LH][HZS];
  __shared__ double red[8];
  const int c0 = blockIdx.x * LT, r0 = blockIdx.y * LT;
  const int tid = threadIdx.x;
  const int Wp = map_pitch(W);
  const size_t MS = map_stride(W, H);
  const int n_crop_w = W - 2 * HALO, n_crop_h = H - 2 * HALO;
  // the maps' zero borders: top rows by the first CTA row, left columns by the
  // first CTA column
  if (blockIdx.y == 0) {
    for (int e = tid; e < 9 * HALO * (LT + HALO); e += blockDim.x) {
      const int k = e / (HALO * (LT + HALO)), rr = (e / (LT + HALO)) % HALO, cc = e % (LT + HALO);
      const int col = cc < HALO ? (blockIdx.x == 0 ? cc : -1) : (c0 + cc - HALO < W ? c0 + cc : -1);
      if (col >= 0) dmaps[k * MS + (size_t)rr * Wp + col] = 0.f;
    }
  }
  if (blockIdx.x == 0) {
    for (int e = tid; e < 9 * LT * HALO; e += blockDim.x) {
      const int k = e / (LT * HALO), rr = (e / HALO) % LT, cc = e % HALO;
      if (r0 + rr < H) dmaps[k * MS + (size_t)(r0 + rr + HALO) * Wp + cc] = 0.f;
    }
  }
  const double mw = 1.0 / ((double)n_crop_w * n_crop_h * 3.0);
  const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
  float wv[11];
#pragma unroll
  for (int t = 0; t < 11; t++) wv[t] = c_win[t];
  double l1 = 0.0, ss = 0.0;
  // the thread's halo columns (lane and lane + 32 < LH), fixed for every row
  const int ca = tid & 31, cb = ca + 32;
  const int gca = c0 - HALO + ca, gcb = c0 - HALO + cb;
  const bool ina = gca >= 0 && gca < W, inb = cb < LH && gcb >= 0 && gcb < W;
  for (int ch = 0; ch < 3; ch++) {
    const float* imc = img + ch;
    float* dm0 = dmaps + (size_t)(ch * 3 + 0) * MS + HALO * Wp + HALO;  // pixel (0, 0)
    float* dm1 = dmaps + (size_t)(ch * 3 + 1) * MS + HALO * Wp + HALO;
    float* dm2 = dmaps + (size_t)(ch * 3 + 2) * MS + HALO * Wp + HALO;
    // two rows per pass, all eight loads issued before the stores
    for (int r = tid >> 5; r < LH; r += 16) {
      float v[2][4];
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int rr = r + 8 * u;
        const int gr = r0 - HALO + rr;
        const bool rin = rr < LH && gr >= 0 && gr < H;
        const int row = gr * W;
        v[u][0] = rin && ina ? imc[3 * (row + gca)] : 0.f;
        v[u][1] = rin && ina ? tgt_at<U8>(tgt, 3 * (row + gca) + ch) : 0.f;
        v[u][2] = rin && inb ? imc[3 * (row + gcb)] : 0.f;
        v[u][3] = rin && inb ? tgt_at<U8>(tgt, 3 * (row + gcb) + ch) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int rr = r + 8 * u;
        if (rr >= LH) break;
        sx[rr][ca] = v[u][0];
        sy[rr][ca] = v[u][1];
        if (cb < LH) {
          sx[rr][cb] = v[u][2];
          sy[rr][cb] = v[u][3];
        }
      }
    }
    __syncthreads();
    if (tid < HITEMS) {
      const int r = tid / (LT / HSEG), cs = (tid % (LT / HSEG)) * HSEG;
      float2 xy[HSEG + 10];
#pragma unroll
      for (int j = 0; j < HSEG + 10; j++) xy[j] = make_float2(sx[r][cs + j], sy[r][cs + j]);
      // maps (x, y) and (x^2, y^2) as packed lane pairs (FFMA2, each lane the
      // scalar FMA chain), then x y: the map's inputs are formed once per input
      // element, then 11 FMAs per output
#pragma unroll
      for (int k = 0; k < 2; k++) {
        float2 in[HSEG + 10];
#pragma unroll
        for (int j = 0; j < HSEG + 10; j++) in[j] = k == 0 ? xy[j] : f2_mul(xy[j], xy[j]);
#pragma unroll
        for (int o = 0; o < HSEG; o++) {
          float2 v = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < 11; t++) v = f2_fma(make_float2(wv[t], wv[t]), in[o + t], v);
          hz[2 * k][r][cs + o] = v.x;
          hz[2 * k + 1][r][cs + o] = v.y;
        }
      }
      {
        float in[HSEG + 10];
#pragma unroll
        for (int j = 0; j < HSEG + 10; j++) in[j] = xy[j].x * xy[j].y;
#pragma unroll
        for (int o = 0; o < HSEG; o++) {
          float v = 0.f;
#pragma unroll
          for (int t = 0; t < 11; t++) v = fmaf(wv[t], in[o + t], v);
          hz[4][r][cs + o] = v;
        }
      }
    }
    __syncthreads();
    {
      const int c = tid % LT, rs = (tid / LT) * VSEG;
      float mom[5][VSEG];
#pragma unroll
      for (int k = 0; k < 4; k += 2) {  // maps (k, k + 1) as lane pairs
        float2 col[VSEG + 10];
#pragma unroll
        for (int j = 0; j < VSEG + 10; j++) col[j] = make_float2(hz[k][rs + j][c], hz[k + 1][rs + j][c]);
#pragma unroll
        for (int o = 0; o < VSEG; o++) {
          float2 v = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < 11; t++) v = f2_fma(make_float2(wv[t], wv[t]), col[o + t], v);
          mom[k][o] = v.x;
          mom[k + 1][o] = v.y;
        }
      }
      {
        float col[VSEG + 10];
#pragma unroll
        for (int j = 0; j < VSEG + 10; j++) col[j] = hz[4][rs + j][c];
#pragma unroll
        for (int o = 0; o < VSEG; o++) {
          float v = 0.f;
#pragma unroll
          for (int t = 0; t < 11; t++) v = fmaf(wv[t], col[o + t], v);
          mom[4][o] = v;
        }
      }
      float l1f = 0.f, ssf = 0.f;  // <= 4 terms per channel: fp32 partials, fp64 from here on
#pragma unroll
      for (int o = 0; o < VSEG; o++) {
        const int r = rs + o;
        const int gr = r0 + r, gc = c0 + c;
        if (gr >= H || gc >= W) continue;
        const float mx = mom[0][o], my = mom[1][o], gx2 = mom[2][o], gy2 = mom[3][o], gxy = mom[4][o];
        const float vx = gx2 - mx * mx, vy = gy2 - my * my, cv = gxy - mx * my;
        const float a1 = 2.f * mx * my + C1, a2 = 2.f * cv + C2;
        const float b1 = mx * mx + my * my + C1, b2 = vx + vy + C2;
        const float i1 = __frcp_rn(b1), i2 = __frcp_rn(b2), i12 = i1 * i2;
        const float smap = (a1 * a2) * i12;
        const bool crop = gr >= HALO && gr < H - HALO && gc >= HALO && gc < W - HALO;
        const int pi = gr * Wp + gc;
        float dmu = 0.f, dg2 = 0.f, dxy = 0.f;
        if (crop) {
          ssf += smap;
          const float m = (float)mw;
          dmu = m * (2.f * my * (a2 - a1) * i12 - 2.f * mx * smap * (i1 - i2));
          dg2 = m * (-smap * i2);
          dxy = m * (2.f * a1 * i12);
        }
        dm0[pi] = dmu;
        dm1[pi] = dg2;
        dm2[pi] = dxy;
        l1f += fabsf(sx[r + HALO][c + HALO] - sy[r + HALO][c + HALO]);
      }
      l1 += (double)l1f;
      ss += (double)ssf;
    }
    __syncthreads();
  }
  double sd = 0.0, sd2 = 0.0, hd = 0.0, hd2 = 0.0;
  const double s0 = soft ? soft[0] : 0.0;  // soft == NULL: the render computed no soft counts (load weight 0)
  const int32_t h0 = hard[0];
  for (int e = tid; e < LT * LT; e += blockDim.x) {
    const int gr = r0 + e / LT, gc = c0 + e % LT;
    if (gr >= H || gc >= W) continue;
    const size_t pi = (size_t)gr * W + gc;
    const double d = soft ? soft[pi] - s0 : 0.0;
    sd += d;
    sd2 += d * d;
    const double dh = (double)(hard[pi] - h0);
    hd += dh;
    hd2 += dh * dh;
  }
  // per-CTA partial sums (no atomics): k_loss_finalize adds them in a fixed
  // order, so the scalar terms -- and d_soft, which depends on them -- are
  // bit-identical run to run
  double* part = partials + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * LOSS_TERMS;
  const double vals[LOSS_TERMS] = {l1, ss, sd, sd2, hd, hd2};
#pragma unroll
  for (int j = 0; j < LOSS_TERMS; j++) {
    const double v = block_sum64(vals[j], red);
    if (tid == 0) part[j] = v;
  }
}

constexpr int FIN_THREADS = 256;

__global__ void __launch_bounds__(FIN_THREADS) k_loss_finalize(int W, int H, double w_l1, double w_ssim,
                                                               double w_load, const double* soft,
                                                               const double* __restrict__ partials, int n_parts,
                                                               LossAcc* acc, double* out) {
  griddep_wait();
  // fixed-order sums of the per-CTA partials: thread t adds parts t, t + 256,
  // ... in order, then a fixed shuffle / warp-order tree
  __shared__ double red[FIN_THREADS / 32][LOSS_TERMS];
  double tsum[LOSS_TERMS] = {0, 0, 0, 0, 0, 0};
  for (int c = threadIdx.x; c < n_parts; c += FIN_THREADS)
#pragma unroll
    for (int j = 0; j < LOSS_TERMS; j++) tsum[j] += partials[(size_t)c * LOSS_TERMS + j];
#pragma unroll
  for (int j = 0; j < LOSS_TERMS; j++) {
    for (int o = 16; o > 0; o >>= 1) tsum[j] += __shfl_xor_sync(0xffffffffu, tsum[j], o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][j] = tsum[j];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
#pragma unroll
  for (int j = 0; j < LOSS_TERMS; j++) {
    double v = 0.0;
    for (int w = 0; w < FIN_THREADS / 32; w++) v += red[w][j];
    tsum[j] = v;
  }
  acc->l1_sum = tsum[0];
  acc->ssim_sum = tsum[1];
  acc->soft_d = tsum[2];
  acc->soft_d2 = tsum[3];
  acc->hard_d = tsum[4];
  acc->hard_d2 = tsum[5];
  const double n = (double)W * H;
  const double n_crop = (double)(W - 2 * HALO) * (H - 2 * HALO);
  const double l1 = acc->l1_sum / (n * 3.0);
  const double ssim = acc->ssim_sum / (n_crop * 3.0);
  const double md = acc->soft_d / n;
  double var = acc->soft_d2 / n - md * md;
  double sd = var > 0.0 ? sqrt(var) : 0.0;
  const double mh = acc->hard_d / n;
  double varh = acc->hard_d2 / n - mh * mh;
  acc->mean_soft = (soft ? soft[0] : 0.0) + md;
  acc->std_soft = sd;
  const double load = w_load > 0.0 ? sd : 0.0;
  out[0] = l1;
  out[1] = 1.0 - ssim;
  out[2] = load;
  out[3] = w_l1 * l1 + w_ssim * (1.0 - ssim) + w_load * load;
  out[4] = varh > 0.0 ? sqrt(varh) : 0.0;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(smem_dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(mbar))
      : "memory");
}

// Dynamic shared memory of k_ssim_bwd: two channel buffers of the three halo
// tiles (TMA destinations, 128-byte aligned), the horizontal results, two
// mbarriers.
constexpr size_t BW_SMEM = 2 * (size_t)BW_BUF_BYTES + sizeof(float) * 3 * LH * HZS + 16;

// One elected thread loads channel 0 and 1's adjoint tiles by TMA at entry
// and channel 2's into the first buffer once channel 0's horizontal pass has
// read it, so every tile load overlaps the blur of the previous channel.
template <bool U8>
__global__ void __launch_bounds__(256) k_ssim_bwd(const __grid_constant__ CUtensorMap tmap, int W, int H,
                                                  const float* __restrict__ img, const Target tgt,
                                                  const double* __restrict__ soft, const LossAcc* __restrict__ acc,
                                                  double w_l1, double w_ssim, double w_load,
                                                  float* __restrict__ d_image, float* __restrict__ d_soft) {
  extern __shared__ __align__(128) unsigned char smem[];
  float(*buf[2])[LH][BP] = {reinterpret_cast<float(*)[LH][BP]>(smem),
                            reinterpret_cast<float(*)[LH][BP]>(smem + BW_BUF_BYTES)};
  float(*hz)[LH][HZS] = reinterpret_cast<float(*)[LH][HZS]>(smem + 2 * BW_BUF_BYTES);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 2 * BW_BUF_BYTES + sizeof(float) * 3 * LH * HZS);
  const int c0 = blockIdx.x * LT, r0 = blockIdx.y * LT;
  const int tid = threadIdx.x;
  const size_t HW = (size_t)W * H;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
  }
  __syncthreads();
  griddep_wait();  // the maps are the forward's output
  if (tid == 0) {
#pragma unroll
    for (int ch = 0; ch < 2; ch++) {
      mbar_expect_tx(&mbar[ch], BW_TILE_BYTES);
      tma_load_3d(&buf[ch][0][0][0], &tmap, c0, r0, ch * 3, &mbar[ch]);  // padded coordinates
    }
  }
  const float gl1 = (float)(w_l1 / (double)(HW * 3));
  const float gss = (float)w_ssim;
  float wv[11];
#pragma unroll
  for (int t = 0; t < 11; t++) wv[t] = c_win[t];
  for (int ch = 0; ch < 3; ch++) {
    const int b = ch & 1;
    mbar_wait(&mbar[b], ch >> 1);
    float(*sm)[LH][BP] = buf[b];
    if (tid < HITEMS) {
      const int r = tid / (LT / HSEG), cs = (tid % (LT / HSEG)) * HSEG;
      // 18 consecutive floats of a row: four 16-byte and one 8-byte load
      // (conflict-free: the rows are 44 floats apart)
      float row[3][HSEG + 10];
#pragma unroll
      for (int k = 0; k < 3; k++) {
        const float4* q = reinterpret_cast<const float4*>(&sm[k][r][cs]);
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const float4 x = q[v];
          row[k][4 * v] = x.x;
          row[k][4 * v + 1] = x.y;
          row[k][4 * v + 2] = x.z;
          row[k][4 * v + 3] = x.w;
        }
        const float2 x = *reinterpret_cast<const float2*>(&sm[k][r][cs + 16]);
        row[k][16] = x.x;
        row[k][17] = x.y;
      }
      {  // maps 0 and 1 as lane pairs, then map 2
        float2 xv[HSEG + 10];
#pragma unroll
        for (int j = 0; j < HSEG + 10; j++) xv[j] = make_float2(row[0][j], row[1][j]);
#pragma unroll
        for (int o = 0; o < HSEG; o++) {
          float2 v = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < 11; t++) v = f2_fma(make_float2(wv[t], wv[t]), xv[o + t], v);
          hz[0][r][cs + o] = v.x;
          hz[1][r][cs + o] = v.y;
        }
      }
#pragma unroll
      for (int o = 0; o < HSEG; o++) {
        float v = 0.f;
#pragma unroll
        for (int t = 0; t < 11; t++) v = fmaf(wv[t], row[2][o + t], v);
        hz[2][r][cs + o] = v;
      }
    }
    __syncthreads();
    if (ch == 0 && tid == 0) {  // buffer 0 is free: channel 2's tiles
      mbar_expect_tx(&mbar[0], BW_TILE_BYTES);
      tma_load_3d(&buf[0][0][0][0], &tmap, c0, r0, 6, &mbar[0]);
    }
    {
      const int c = tid % LT, rs = (tid / LT) * VSEG;
      float bm[3][VSEG];
      {  // maps 0 and 1 as lane pairs, then map 2
        float2 col[VSEG + 10];
#pragma unroll
        for (int j = 0; j < VSEG + 10; j++) col[j] = make_float2(hz[0][rs + j][c], hz[1][rs + j][c]);
#pragma unroll
        for (int o = 0; o < VSEG; o++) {
          float2 v = make_float2(0.f, 0.f);
#pragma unroll
          for (int t = 0; t < 11; t++) v = f2_fma(make_float2(wv[t], wv[t]), col[o + t], v);
          bm[0][o] = v.x;
          bm[1][o] = v.y;
        }
      }
      {
        float col[VSEG + 10];
#pragma unroll
        for (int j = 0; j < VSEG + 10; j++) col[j] = hz[2][rs + j][c];
#pragma unroll
        for (int o = 0; o < VSEG; o++) {
          float v = 0.f;
#pragma unroll
          for (int t = 0; t < 11; t++) v = fmaf(wv[t], col[o + t], v);
          bm[2][o] = v;
        }
      }
#pragma unroll
      for (int o = 0; o < VSEG; o++) {
        const int gr = r0 + rs + o, gc = c0 + c;
        if (gr >= H || gc >= W) continue;
        const int pi = gr * W + gc;
        const float x = img[pi * 3 + ch], y = tgt_at<U8>(tgt, pi * 3 + ch);
        const float gs = bm[0][o] + 2.f * x * bm[1][o] + y * bm[2][o];  // d SSIM / d x
        const float diff = x - y;
        const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
        d_image[pi * 3 + ch] = gl1 * sgn - gss * gs;
      }
    }
    __syncthreads();
  }
  if (d_soft) {
    const double sd = acc->std_soft, mean = acc->mean_soft;
    const double scale = (w_load > 0.0 && sd > 0.0) ? w_load / ((double)HW * sd) : 0.0;
    for (int e = tid; e < LT * LT; e += blockDim.x) {
      const int gr = r0 + e / LT, gc = c0 + e % LT;
      if (gr >= H || gc >= W) continue;
      const size_t pi = (size_t)gr * W + gc;
      d_soft[pi] = (float)((soft[pi] - mean) * scale);
    }
  }
}

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static int ensure_window() {
  static DeviceOnce done;
  if (done.done()) return SSR_OK;
  float w[11];
  double g[11], s = 0.0;
  for (int t = 0; t < 11; t++) {
    const double tt = t - 5;
    g[t] = exp(-(tt * tt) / (2.0 * 1.5 * 1.5));
    s += g[t];
  }
  for (int t = 0; t < 11; t++) w[t] = (float)(g[t] / s);
  SSR_TRY(check_cuda(cudaMemcpyToSymbol(c_win, w, sizeof(w)), "ssim window"));
  done.set();
  return SSR_OK;
}

}  // namespace ssr

using namespace ssr;

static int64_t loss_ctas(int32_t width, int32_t height) {
  return (int64_t)((width + LT - 1) / LT) * ((height + LT - 1) / LT);
}

static int64_t maps_bytes(int32_t width, int32_t height) {
  return align_up((int64_t)9 * map_stride(width, height) * 4, 256);
}

// The 3-D tensor map over the nine adjoint maps (x: column, y: row, z: map),
// box = one channel's three halo tiles.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int maps_tensor_map(CUtensorMap* m, float* dmaps, int32_t width, int32_t height) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    SSR_TRY(check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
                       "cuTensorMapEncodeTiled entry point"));
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("ssr_loss: cuTensorMapEncodeTiled unavailable");
      return SSR_ERR_CUDA;
    }
    encode = (EncodeTiledFn)fn;
  }
  const cuuint64_t pitch = (cuuint64_t)map_pitch(width) * 4;
  const cuuint64_t dims[3] = {(cuuint64_t)width + HALO, (cuuint64_t)height + HALO, 9};
  const cuuint64_t strides[2] = {pitch, (cuuint64_t)map_stride(width, height) * 4};
  const cuuint32_t box[3] = {BP, LH, 3};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dmaps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("ssr_loss: cuTensorMapEncodeTiled failed");
    return SSR_ERR_CUDA;
  }
  return SSR_OK;
}

extern "C" int ssr_loss_workspace(int32_t width, int32_t height, int64_t* bytes) {
  *bytes = maps_bytes(width, height) + align_up(sizeof(LossAcc), 256) +
           align_up(loss_ctas(width, height) * LOSS_TERMS * 8, 256);
  return SSR_OK;
}

extern "C" int ssr_loss(int32_t width, int32_t height, const float* image, const void* target, int32_t target_u8,
                        const double* soft_count, const int32_t* hard_count, double w_l1, double w_ssim, double w_load,
                        float* d_image, float* d_soft, double* out, void* workspace, int64_t workspace_bytes,
                        void* stream) {
  if (width < 11 || height < 11) {
    set_error("ssr_loss: image smaller than the 11-tap SSIM window");
    return SSR_ERR_INVALID;
  }
  if ((int64_t)width * height * 3 > INT32_MAX) {
    set_error("ssr_loss: image larger than 715 megapixels (32-bit pixel indexing)");
    return SSR_ERR_INVALID;
  }
  int64_t need = 0;
  ssr_loss_workspace(width, height, &need);
  if (workspace_bytes < need || ((uintptr_t)workspace & 15)) {
    set_error("ssr_loss: workspace too small or not 16-byte aligned");
    return SSR_ERR_INVALID;
  }
  if (!soft_count && (w_load > 0.0 || d_soft)) {
    set_error("ssr_loss: soft_count is required for a load term or a d_soft output");
    return SSR_ERR_INVALID;
  }
  SSR_TRY(ensure_window());
  cudaStream_t st = (cudaStream_t)stream;
  float* dmaps = (float*)workspace;
  LossAcc* acc = (LossAcc*)((char*)workspace + maps_bytes(width, height));
  double* partials = (double*)((char*)acc + align_up(sizeof(LossAcc), 256));
  dim3 grid((width + LT - 1) / LT, (height + LT - 1) / LT);
  const Target tg{target, target_u8 ? 1 : 0};
  if (tg.u8)
    SSR_TRY(launch_pdl("k_ssim_fwd", k_ssim_fwd<true>, grid, dim3(256), 0, st, width, height, image, tg, soft_count,
                       hard_count, dmaps, partials));
  else
    SSR_TRY(launch_pdl("k_ssim_fwd", k_ssim_fwd<false>, grid, dim3(256), 0, st, width, height, image, tg, soft_count,
                       hard_count, dmaps, partials));
  SSR_TRY(check_launch("k_ssim_fwd"));
  SSR_TRY(launch_pdl("k_loss_finalize", k_loss_finalize, dim3(1), dim3(FIN_THREADS), 0, st, width, height, w_l1,
                     w_ssim, w_load, soft_count, (const double*)partials, (int)loss_ctas(width, height), acc, out));
  SSR_TRY(check_launch("k_loss_finalize"));
  CUtensorMap tmap;
  SSR_TRY(maps_tensor_map(&tmap, dmaps, width, height));
  static DeviceOnce attr;
  if (!attr.done()) {
    SSR_TRY(check_cuda(cudaFuncSetAttribute(k_ssim_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)BW_SMEM),
                       "k_ssim_bwd smem"));
    SSR_TRY(check_cuda(cudaFuncSetAttribute(k_ssim_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)BW_SMEM),
                       "k_ssim_bwd smem"));
    attr.set();
  }
  if (tg.u8)
    SSR_TRY(launch_pdl("k_ssim_bwd", k_ssim_bwd<true>, grid, dim3(256), BW_SMEM, st, tmap, width, height, image, tg,
                       soft_count, (const LossAcc*)acc, w_l1, w_ssim, w_load, d_image, d_soft));
  else
    SSR_TRY(launch_pdl("k_ssim_bwd", k_ssim_bwd<false>, grid, dim3(256), BW_SMEM, st, tmap, width, height, image, tg,
                       soft_count, (const LossAcc*)acc, w_l1, w_ssim, w_load, d_image, d_soft));
  return check_launch("k_ssim_bwd");
}
