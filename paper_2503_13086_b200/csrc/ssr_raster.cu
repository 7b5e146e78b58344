// Stages 3 and 4: 16x16-tile alpha-blend forward and the two backward layouts
// (rasterize/kernels.py:31-353), plus the float64 guard-band fix-up.
//
// Forward: one CTA per tile, one thread per pixel, 512-splat batches staged in
// shared memory, block-wide early exit on transmittance.  Every 32 walked
// slots (64 without soft counts: only the two-slot backward can follow) each
// live pixel checkpoints (T, C_front) so the splat-parallel backward can start
// any bucket without replaying the tile.
//
// Backward: per-instance gradient rows (10 words: 9 terms + the generation
// tag of ssr_common.cuh) written once each, for the walked slots only.
//
// Guard band: the fp32 walk flags a pixel when any discrete
// decision (power>0 skip, alpha >= 1/255 gate, alpha > 0.99 cap, T(1-a) < 1e-4
// termination) is within `band` (relative) of its threshold.  Flagged pixels
// are re-walked in float64 by one warp each (forward fix-up) and their
// gradient rows are added by an fp64 pixel walk (backward fix-up); the fp32
// backward kernels skip them, so fp32 never has to agree with fp64 near a
// threshold.
#include <climits>

#include "ssr_common.cuh"

namespace ssr {

constexpr unsigned FULL = 0xffffffffu;

struct RasterArgs {
  int width, height, tiles_x, tiles_y;
  float bg[3];
  double bg64[3];
  float band, band_t;
  const double2* mean;
  const float4* conic_opa;
  const float4* color;
  const double2* conic_opa64;
  const double2* color64;
  const int4* rect;
  const uint32_t* row_offset;
  const uint32_t* inst;
  const int2* ranges;
  float* image;
  float* t_final;
  int* n_walk;
  uint8_t* term;
  int* hard;
  double* soft;
  uint8_t* flagged;
  int4* tile_info;  // (max n_walk, flagged pixels, max fp64 n_walk of a flagged pixel, first flagged slot)
  float4* ckpt;
  int* fix;  // fix_list: [0] pixels, [1] tiles, [2] fix-up buckets, [3] spare, tile slots, bucket plan,
             // pixel entries
  int n_tiles;
};

constexpr int FIX_HEAD = 4;

__device__ __forceinline__ int* fix_tiles(const RasterArgs& a) { return a.fix + FIX_HEAD; }
__device__ __forceinline__ int* fix_plan(const RasterArgs& a) { return a.fix + FIX_HEAD + a.n_tiles; }
__device__ __forceinline__ int* fix_pixels(const RasterArgs& a) { return a.fix + FIX_HEAD + 2 * a.n_tiles; }
// per pixel (y * W + x): the walk slot of a flagged pixel's first ambiguous decision
__device__ __forceinline__ int* fix_kflag(const RasterArgs& a) {
  return a.fix + FIX_HEAD + 2 * a.n_tiles + (size_t)a.width * a.height;
}

// Splat-major position of the instance of field row g in tile (tx, ty).
__device__ __forceinline__ uint32_t inst_row(const RasterArgs& a, uint32_t g, int tx, int ty) {
  const int4 r = a.rect[g];
  return a.row_offset[g] + (uint32_t)((ty - r.y) * (r.z - r.x) + (tx - r.x));
}

__device__ __forceinline__ size_t ckpt_base(int s0, int t) { return ((size_t)(s0 >> 5) + (size_t)t) * TILE_PX; }

// ------------------------------------------------------------------ forward (fp32)
// Per-pixel walk state of the fp32 forward.
struct FwdState {
  float T, c0, c1, c2, sdev;
  double sbig;
  // every walked slot is exactly one of: far or small-alpha (soft term S0 +
  // deviation), skipped fragile (no term), or large-alpha (exact sigmoid), so
  // the S0 count is n_walk - n_big and the common paths count nothing
  int hard, nwk, nbig;
  bool term, flag;
};

// One walked slot past the far test (kernels.py:68-95): fragile guard,
// small-alpha soft deviation, or the large path (exact sigmoid, guard bands,
// blend).  w100 = staged +-100 opacity (sign: fragile).  Returns false once
// the pixel terminated or was flagged.
template <bool FRAGILE, bool SOFT>
__device__ __forceinline__ bool fwd_slot(FwdState& q, float p2, float qpos, float w100, const float4* sB, int j,
                                         int k0, float band, float band_t) {
  if (FRAGILE) {
    // SOFT = false stages the signed opacity in sB[j].w instead of +-100 opacity
    const bool fragile = SOFT ? w100 < 0.f : sB[j].w < 0.f;
    if (fragile) {
      // only near-singular conics can round to power > 0: flag near that decision
      if (p2 > 1e-6f * qpos && qpos != 0.f) {
        q.flag = true;
        q.nwk = k0 + j;  // flagged: the slot of the ambiguous decision
        return false;
      }
      if (p2 > 0.f) {
        q.nbig++;  // skipped: no soft term (counted out of the S0 total)
        return true;
      }
    }
  }
  // y = 100 alpha costs one product; alpha itself (= opacity * 2^p2, the
  // decisions' operand) only on the large path.  y may differ from
  // fl(alpha * 100) in the last bit: that only moves a pair between the
  // deviation fit and the exact sigmoid (|diff| < 2e-10).
  const float e2 = ex2_approx(p2);
  if (SOFT) {
    const float y = __fmul_rn(fabsf(w100), e2);
    if (y < SOFT_Y0) {
      q.sdev = soft_dev_acc(y, q.sdev);
      return true;
    }
  }
  const float4 B = sB[j];
  float alpha = __fmul_rn(SOFT ? B.w : fabsf(B.w), e2);
  const bool fa = (fabsf(alpha - ALPHA_MIN_F) < ALPHA_MIN_F * band) | (fabsf(alpha - ALPHA_CAP_F) < ALPHA_CAP_F * band);
  alpha = fminf(alpha, ALPHA_CAP_F);
  if (SOFT) {
    q.nbig++;  // (also for a slot flagged here: the fix-up recomputes a flagged pixel)
    q.sbig += (double)soft_sigmoid_accurate(alpha);
  }
  // blend without a branch (most large-path lanes blend): a lane below
  // 1/255 runs it with alpha = 0, i.e. T * 1 and colour + B * 0
  const bool bl = alpha >= ALPHA_MIN_F;
  const float ab = bl ? alpha : 0.f;
  const float test = __fmul_rn(q.T, __fsub_rn(1.f, ab));
  const bool ft = bl & (fabsf(test - T_EPS_F) < T_EPS_F * band_t);
  // one exit: an alpha guard band, a transmittance guard band, or termination
  if (fa | ft | (bl & (test < T_EPS_F))) {
    if (fa | ft) {
      q.flag = true;
      q.nwk = k0 + j;
    } else {
      q.term = true;
      q.nwk = k0 + j + 1;
    }
    return false;
  }
  const float w = __fmul_rn(ab, q.T);
  q.c0 = __fmaf_rn(B.x, w, q.c0);
  q.c1 = __fmaf_rn(B.y, w, q.c1);
  q.c2 = __fmaf_rn(B.z, w, q.c2);
  q.hard += bl ? 1 : 0;
  q.T = test;
  return true;
}

// kernels.py:68-95 over slots [j0, jend) of the staged batch (walk index
// k0 + j), two slots at a time: the staged pair (j, j + 1) holds
// {x int, x frac}, {y int, y frac}, {a2, b2}, {c2, +-100 opacity} as lane
// pairs, so the far test of both splats is 7 packed operations; slots that
// pass it run fwd_slot in walk order.  FRAGILE: the batch holds a
// near-singular conic (negative staged opacity), so the power > 0 guard band
// is tested; batches without one (the common case) skip that test entirely.
// Returns false once the pixel terminated or was flagged.
// SOFT = false (no soft-count output): the far test uses each splat's own
// cut (D.z / D.w = log2(0.999 / (255 opacity)), clamped to the soft far
// power): a pair below it has alpha < 1/255 and, without soft counts,
// contributes nothing -- the same bound the backward's non-soft path uses.
template <bool FRAGILE, bool FULL, bool SOFT>
__device__ __forceinline__ bool fwd_walk(FwdState& q, const float4* sP, const float4* sB, int j0, int jend, int k0,
                                         float fpx, float fpy, float band, float band_t) {
  // FULL: a whole 32-slot bucket, constant trip count (no per-slot bound test)
  const int nj = FULL ? BUCKET : jend - j0;
  const float2 px2 = make_float2(fpx, fpx), py2 = make_float2(fpy, fpy);
#pragma unroll 4
  for (int jj = 0; jj < nj; jj += 2) {
    const int j = j0 + jj;  // even: pair j / 2
    const float4* P = sP + 2 * j;
    const float4 MX = P[0], MY = P[1], C = P[2], D = P[3];
    const float2 dx = f2_sub(f2_sub(px2, make_float2(MX.x, MX.y)), make_float2(MX.z, MX.w));
    const float2 dy = f2_sub(f2_sub(py2, make_float2(MY.x, MY.y)), make_float2(MY.z, MY.w));
    const float2 dxx = f2_mul(dx, dx), dxy = f2_mul(dx, dy), dyy = f2_mul(dy, dy);
    const float2 qp = f2_fma(make_float2(D.x, D.y), dyy, f2_mul(make_float2(C.x, C.y), dxx));
    const float2 p2 = f2_fma(make_float2(C.z, C.w), dxy, qp);
    // far (power < -25): soft term S0 only, nothing else
    const float cut_x = SOFT ? FAR_POWER2 : D.z, cut_y = SOFT ? FAR_POWER2 : D.w;
    if (!(p2.x < cut_x) && !fwd_slot<FRAGILE, SOFT>(q, p2.x, qp.x, D.z, sB, j, k0, band, band_t)) return false;
    if ((FULL || jj + 1 < nj) && !(p2.y < cut_y) &&
        !fwd_slot<FRAGILE, SOFT>(q, p2.y, qp.y, D.w, sB, j + 1, k0, band, band_t))
      return false;
  }
  return true;
}

// Splats staged per batch: two per thread (half the barriers of one per thread).
#ifndef SSR_FWD_PER
#define SSR_FWD_PER 2
#endif
constexpr int FWD_BATCH = SSR_FWD_PER * TILE_PX;

// CK = false: render-only (view_psnr, pipeline.py:180-182): no bucket
// checkpoints are written (the backward's seeds, ~16 B per live pixel-bucket).
template <bool CK, bool SOFT>
__global__ void __launch_bounds__(256) k_forward(RasterArgs a) {
  griddep_wait();
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int x00 = tx * TILE, y00 = ty * TILE;
  // warp w covers the 8x4 pixel block (w & 1, w >> 1) of the tile: a splat's
  // footprint splits the lanes of a compact block less often than a 16x2 strip
  const int lane_ = tid & 31, wrp = tid >> 5;
  const int lx = (wrp & 1) * 8 + (lane_ & 7), ly = (wrp >> 1) * 4 + (lane_ >> 3);
  const int pidx = ly * TILE + lx;  // row-major pixel index in the tile (checkpoints, fix list)
  const int px = x00 + lx, py = y00 + ly;
  const bool inside = px < a.width && py < a.height;
  const int2 rg = a.ranges[t];
  const int s0 = rg.x, s1 = rg.y;
  const float fpx = (float)lx, fpy = (float)ly;
  const float band = a.band, band_t = a.band_t;

  // staged splat pairs (fwd_walk): {xi}, {xf}, {yi}, {yf}, {a2}, {b2}, {c2},
  // {100 opacity, < 0 marks a fragile conic} as lane pairs, 4 float4 per pair
  __shared__ float4 sP[2 * FWD_BATCH];
  __shared__ float4 sB[FWD_BATCH];  // r, g, b, opacity
  __shared__ int sMax[8];

  FwdState q;
  q.T = 1.f;
  q.c0 = q.c1 = q.c2 = q.sdev = 0.f;
  q.sbig = 0.0;
  q.hard = 0;
  q.nwk = s1 - s0;
  q.nbig = 0;
  q.term = q.flag = false;
  bool done = !inside;
  float4* ck = CK ? a.ckpt + ckpt_base(s0, t) + pidx : nullptr;

  for (int base = s0; base < s1; base += FWD_BATCH) {
    if (__syncthreads_count(done) == TILE_PX) break;
    bool fragile = false;
#pragma unroll
    for (int u = 0; u < FWD_BATCH / TILE_PX; u++) {
      const int e = u * TILE_PX + tid;
      const int s = base + e;
      if (s < s1) {
        const uint32_t g = a.inst[s];
        const double2 m = a.mean[g];
        const float4 co = a.conic_opa[g];
        const float4 col = a.color[g];
        const StagedConic sc = stage_conic(co.x, co.y, co.z);
        const StagedMean sm = stage_mean(m.x, m.y, x00, y00);
        float* P = reinterpret_cast<float*>(sP + 2 * (e & ~1)) + (e & 1);
        P[0] = sm.xi;
        P[2] = sm.xf;
        P[4] = sm.yi;
        P[6] = sm.yf;
        P[8] = sc.a2;
        P[10] = sc.b2;
        P[12] = sc.c2;
        if (SOFT) {
          P[14] = __fmul_rn(co.w, 100.f);  // < 0 marks a fragile conic
          sB[e] = make_float4(col.x, col.y, col.z, fabsf(co.w));
        } else {  // the pair's far cut; the staged opacity keeps the fragile sign
          P[14] = fmaxf(FAR_POWER2, __log2f(0.999f * ALPHA_MIN_F / fabsf(co.w)));
          sB[e] = make_float4(col.x, col.y, col.z, co.w);
        }
        fragile |= co.w < 0.f;
      }
    }
    const bool batch_fragile = __syncthreads_or(fragile);
    if (!done) {
      const int n = min(FWD_BATCH, s1 - base);
      const int k0 = base - s0;
      for (int j0 = 0; j0 < n; j0 += BUCKET) {
        if (k0 + j0) {  // checkpoint for the splat-parallel backward: its
          // buckets hold 64 slots, so every other 32-slot boundary (the fp64
          // fix-up writes its flagged pixels' own at every 32)
          if (CK && ((k0 + j0) & 63) == 0)
            ck[(size_t)((k0 + j0) >> 5) * TILE_PX] = make_float4(q.T, q.c0, q.c1, q.c2);
          q.sbig += (double)q.sdev;
          q.sdev = 0.f;
        }
        const int jend = min(j0 + BUCKET, n);
        bool go;
        if (jend - j0 == BUCKET)
          go = batch_fragile ? fwd_walk<true, true, SOFT>(q, sP, sB, j0, jend, k0, fpx, fpy, band, band_t)
                             : fwd_walk<false, true, SOFT>(q, sP, sB, j0, jend, k0, fpx, fpy, band, band_t);
        else
          go = batch_fragile ? fwd_walk<true, false, SOFT>(q, sP, sB, j0, jend, k0, fpx, fpy, band, band_t)
                             : fwd_walk<false, false, SOFT>(q, sP, sB, j0, jend, k0, fpx, fpy, band, band_t);
        if (!go) {
          done = true;
          break;
        }
      }
    }
  }
  float T = q.T, c0 = q.c0, c1 = q.c1, c2 = q.c2, sdev = q.sdev;
  double sbig = q.sbig;
  int hard = q.hard, nwk = q.nwk, nbig = q.nbig;
  const bool term = q.term, flag = q.flag;
  if (inside) {
    const size_t pix = (size_t)py * a.width + px;
    a.image[pix * 3 + 0] = c0 + a.bg[0] * T;
    a.image[pix * 3 + 1] = c1 + a.bg[1] * T;
    a.image[pix * 3 + 2] = c2 + a.bg[2] * T;
    a.t_final[pix] = T;
    a.n_walk[pix] = nwk;
    a.term[pix] = term ? 1 : 0;
    a.hard[pix] = hard;
    if (SOFT) a.soft[pix] = (double)(nwk - nbig) * SOFT_S0 + (sbig + (double)sdev);
    a.flagged[pix] = flag ? 1 : 0;
    // every decision before the flagged slot was unambiguous, so the fp32
    // backward handles those slots of a flagged pixel and the fp64 fix-up the rest
    if (flag) fix_kflag(a)[pix] = nwk;
  }
  // per-tile (max n_walk over unflagged pixels, flagged count, first flagged slot)
  int mw = (inside && !flag) ? nwk : 0;
  int kf = (inside && flag) ? nwk : INT_MAX;
  for (int o = 16; o > 0; o >>= 1) {
    mw = max(mw, __shfl_xor_sync(FULL, mw, o));
    kf = min(kf, __shfl_xor_sync(FULL, kf, o));
  }
  const bool fl = inside && flag;
  const unsigned fm = __ballot_sync(FULL, fl);
  __shared__ int sCnt[8], sKf[8];
  __shared__ int sBase;
  if ((tid & 31) == 0) {
    sMax[tid >> 5] = mw;
    sCnt[tid >> 5] = __popc(fm);
    sKf[tid >> 5] = kf;
  }
  const int nflag = __syncthreads_count(fl);
  if (tid == 0) {
    int m = 0, kmin = INT_MAX;
    for (int w = 0; w < 8; w++) {
      m = max(m, sMax[w]);
      kmin = min(kmin, sKf[w]);
    }
    a.tile_info[t] = make_int4(m, nflag, 0, kmin);
    if (nflag) {  // reserve this tile's block of the compact fix-up lists
      sBase = atomicAdd(&a.fix[0], nflag);
      fix_tiles(a)[atomicAdd(&a.fix[1], 1)] = sBase;
    }
  }
  if (nflag) {
    __syncthreads();
    if (fl) {
      int r = __popc(fm & ((1u << (tid & 31)) - 1u));
      for (int w = 0; w < (tid >> 5); w++) r += sCnt[w];
      fix_pixels(a)[sBase + r] = (t << 8) | pidx;
    }
  }
}

// ------------------------------------------------------------------ fp64 pixel walk (warp)
__device__ __forceinline__ double warp_sum64(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

struct Slot64 {
  bool valid, skip, capped, cand;
  double alpha, sv, dx, dy, qa, qb, qc, opa, col[3];
  uint32_t g;
};

// The per-slot field data a float64 walk needs (independent of the pixel).
struct SlotRaw {
  bool valid;
  uint32_t g;
  double2 m, c0, c1, k0, k1;
};

__device__ __forceinline__ void load_slot(const RasterArgs& a, int s, int s1, SlotRaw& r) {
  r.valid = s < s1;
  if (!r.valid) return;
  r.g = a.inst[s];
  r.m = a.mean[r.g];
  r.c0 = a.conic_opa64[2 * r.g];
  r.c1 = a.conic_opa64[2 * r.g + 1];
  r.k0 = a.color64[2 * r.g];
  r.k1 = a.color64[2 * r.g + 1];
}

// kernels.py:68-89 for one slot in float64, mirroring the reference's op order.
// `with_sv` = false skips the soft-count sigmoid (only the backward fix-up
// without a soft-count gradient does that; q.sv is then 0).
__device__ __forceinline__ void eval_slot(const SlotRaw& r, bool valid, double xx, double yy, Slot64& q,
                                          bool with_sv = true) {
  q.valid = valid;
  q.skip = true;
  q.cand = false;
  q.capped = false;
  q.alpha = 0.0;
  q.sv = 0.0;
  if (!valid) return;
  q.g = r.g;
  q.qa = r.c0.x;
  q.qb = r.c0.y;
  q.qc = r.c1.x;
  q.opa = r.c1.y;
  q.dx = __dsub_rn(xx, r.m.x);
  q.dy = __dsub_rn(yy, r.m.y);
  const double t1 = __dmul_rn(__dmul_rn(q.qa, q.dx), q.dx);
  const double t2 = __dmul_rn(__dmul_rn(q.qc, q.dy), q.dy);
  const double power = __dsub_rn(__dmul_rn(-0.5, __dadd_rn(t1, t2)), __dmul_rn(__dmul_rn(q.qb, q.dx), q.dy));
  if (power > 0.0) return;
  q.skip = false;
  double alpha = __dmul_rn(q.opa, exp(power));
  q.capped = alpha > ALPHA_CAP;
  if (q.capped) alpha = ALPHA_CAP;
  q.alpha = alpha;
  if (with_sv) {
    // the soft-count term only has to meet the value tolerance (the walk's
    // decisions above stay float64): the fp32 forward's split -- the float64
    // constant S0 plus the fitted small-alpha deviation, the fp32 sigmoid
    // above -- so no float64 exp / divide per slot and no systematic fp32
    // rounding of S0 summed over long walks
    const float af = (float)alpha;
    const float y = __fmul_rn(af, 100.f);
    q.sv = y < SOFT_Y0 ? SOFT_S0 + (double)soft_dev_acc(y, 0.f) : (double)soft_sigmoid_accurate(af);
  }
  q.cand = alpha >= ALPHA_MIN;
  q.col[0] = r.k0.x;
  q.col[1] = r.k0.y;
  q.col[2] = r.k1.x;
}

struct Pix64 {
  double T, C[3], soft;
  int hard, nw, term;
};

// Front-to-back walk of one pixel by one warp (lanes = 32 consecutive slots).
// When ck != nullptr the fp32 bucket checkpoint (T, C_front) of every chunk
// boundary is written for the backward fix-up (chunks coincide with buckets).
//
// `kfast`: walk slots before which every decision is known to agree with the
// fp32 walk (a flagged pixel's first ambiguous slot): whole chunks before it
// cannot terminate, so they skip the termination test and the per-chunk
// colour / soft-count reductions (each lane accumulates its own terms, reduced
// once when the light chunks end) and keep the fp32 forward's checkpoints.
__device__ void walk_pixel64(const RasterArgs& a, int s0, int s1, double xx, double yy, Pix64& r,
                             float4* ck = nullptr, int kfast = 0) {
  const int lane = threadIdx.x & 31;
  double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, soft = 0.0;
  double lc0 = 0.0, lc1 = 0.0, lc2 = 0.0, lsoft = 0.0;  // light-chunk per-lane sums
  bool light_pending = false;
  int hard = 0, nw = s1 - s0, term = 0;
  // Two-stage prefetch: the next chunk's field data and the index of the one
  // after it are in flight while the current chunk is evaluated.
  SlotRaw cur;
  load_slot(a, s0 + lane, s1, cur);
  uint32_t g_next = s0 + 32 + lane < s1 ? a.inst[s0 + 32 + lane] : 0u;
  for (int cb = s0; cb < s1; cb += 32) {
    const bool light = cb - s0 + 32 <= kfast;
    if (!light && light_pending) {  // leaving the light chunks: reduce their per-lane sums
      C0 += warp_sum64(lc0);
      C1 += warp_sum64(lc1);
      C2 += warp_sum64(lc2);
      soft += warp_sum64(lsoft);
      light_pending = false;
    }
    if (ck && cb > s0 && !light && lane == 0)
      ck[(size_t)((cb - s0) >> 5) * TILE_PX] = make_float4((float)T, (float)C0, (float)C1, (float)C2);
    SlotRaw nxt;
    nxt.valid = cb + 32 + lane < s1;
    if (nxt.valid) {
      nxt.g = g_next;
      nxt.m = a.mean[g_next];
      nxt.c0 = a.conic_opa64[2 * g_next];
      nxt.c1 = a.conic_opa64[2 * g_next + 1];
      nxt.k0 = a.color64[2 * g_next];
      nxt.k1 = a.color64[2 * g_next + 1];
    }
    g_next = cb + 64 + lane < s1 ? a.inst[cb + 64 + lane] : 0u;
    Slot64 q;
    eval_slot(cur, cur.valid, xx, yy, q);
    const double f = q.cand ? (1.0 - q.alpha) : 1.0;
    double P = f;
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(FULL, P, d);
      if (lane >= d) P *= o;
    }
    double Pex = __shfl_up_sync(FULL, P, 1);
    if (lane == 0) Pex = 1.0;
    const double Tb = T * Pex;
    if (light) {
      const double wgt = q.cand ? q.alpha * Tb : 0.0;
      lc0 += q.col[0] * wgt;
      lc1 += q.col[1] * wgt;
      lc2 += q.col[2] * wgt;
      lsoft += q.skip ? 0.0 : q.sv;
      hard += __popc(__ballot_sync(FULL, q.cand));
      light_pending = true;
      T = T * __shfl_sync(FULL, P, 31);
      cur = nxt;
      continue;
    }
    const bool tc = q.cand && (Tb * (1.0 - q.alpha) < T_EPS);
    const unsigned tm = __ballot_sync(FULL, tc);
    const int tl = tm ? __ffs(tm) - 1 : 32;
    const bool bl = q.cand && lane < tl;
    const double wgt = bl ? q.alpha * Tb : 0.0;
    C0 += warp_sum64(bl ? q.col[0] * wgt : 0.0);
    C1 += warp_sum64(bl ? q.col[1] * wgt : 0.0);
    C2 += warp_sum64(bl ? q.col[2] * wgt : 0.0);
    soft += warp_sum64((!q.skip && lane <= tl) ? q.sv : 0.0);
    hard += __popc(__ballot_sync(FULL, bl));
    if (tm) {
      term = 1;
      nw = cb - s0 + tl + 1;
      T = __shfl_sync(FULL, Tb, tl);
      break;
    }
    T = T * __shfl_sync(FULL, P, 31);
    cur = nxt;
  }
  if (light_pending) {  // the walk ended inside the light chunks
    C0 += warp_sum64(lc0);
    C1 += warp_sum64(lc1);
    C2 += warp_sum64(lc2);
    soft += warp_sum64(lsoft);
  }
  r.T = T;
  r.C[0] = C0;
  r.C[1] = C1;
  r.C[2] = C2;
  r.soft = soft;
  r.hard = hard;
  r.nw = nw;
  r.term = term;
}

// Forward fix-up: persistent grid, one warp per flagged pixel of the compact
// list k_forward built (pixels are independent).
__global__ void __launch_bounds__(256) k_forward_fixup(RasterArgs a) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int nw_total = gridDim.x * 8, count = a.fix[0];
  const int* px_list = fix_pixels(a);
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < count; i += nw_total) {
    const int e = px_list[i];
    const int t = e >> 8, p = e & 255;
    const int tx = t % a.tiles_x, ty = t / a.tiles_x;
    const int px = tx * TILE + (p & 15), py = ty * TILE + (p >> 4);
    const size_t pix = (size_t)py * a.width + px;
    const int2 rg = a.ranges[t];
    Pix64 r;
    walk_pixel64(a, rg.x, rg.y, (double)px, (double)py, r, a.ckpt ? a.ckpt + ckpt_base(rg.x, t) + p : nullptr,
                 fix_kflag(a)[pix]);
    if (lane == 0) {
      a.image[pix * 3 + 0] = (float)(r.C[0] + a.bg64[0] * r.T);
      a.image[pix * 3 + 1] = (float)(r.C[1] + a.bg64[1] * r.T);
      a.image[pix * 3 + 2] = (float)(r.C[2] + a.bg64[2] * r.T);
      a.t_final[pix] = (float)r.T;
      a.n_walk[pix] = r.nw;
      a.term[pix] = (uint8_t)r.term;
      a.hard[pix] = r.hard;
      if (a.soft) a.soft[pix] = r.soft;
      // tile_info.x stays an upper bound of the tile's n_walk (buckets to visit);
      // .z bounds the buckets the backward fix-up visits for this tile
      atomicMax(&a.tile_info[t].x, r.nw);
      atomicMax(&a.tile_info[t].z, r.nw);
    }
  }
}

// Reset of the fix-up list heads (a kernel, so the launch chain stays programmatic).
__global__ void k_fix_reset(int* fix) {
  griddep_wait();
  if (threadIdx.x < FIX_HEAD) fix[threadIdx.x] = 0;
}

// ------------------------------------------------------------------ backward, splat-parallel (fp32)
// Taming-style: one warp per (tile, 64-splat bucket); lane l owns slots
// 64b+2l and 64b+2l+1 and accumulates their 9 gradient terms in registers
// while the bucket's live pixels stream through the warp as a systolic
// pipeline: at step i lane l handles live pixel i-l and receives that pixel's
// running (T, H = w.C_front) from lane l-1 by shuffle.  Lane 0 seeds each pixel
// from the forward's checkpoint at the bucket start.  No atomics; each
// instance row is written once.
//
// The pixel list of a bucket is padded with 32 sentinel entries on both sides
// (pixel 256: blend limit 0), so the stream needs no bounds checks.  The mean
// gradient is accumulated as sum(gp dx), sum(gp dy) and mapped through the
// conic once per row (linear), so a contributing pair costs ~30 instructions.
//
// Without a soft-count gradient: 80 registers, 24 warps per SM (2 blocks:
// 125 registers, no faster).  With one the soft pair block needs more: 125
// registers, 16 warps per SM (3 blocks rematerialise addresses in the loop:
// 2.6 % slower; the former one-slot kernel with 32-slot buckets: 1.3 %).
constexpr int BW2_MIN_BLOCKS = 3;
constexpr int BW2_SOFT_MIN_BLOCKS = 2;
constexpr int BW_PAD = 32;
constexpr int BW_LIST = BW_PAD + TILE_PX + BW_PAD;

struct BwSplat {
  StagedMean sm;
  StagedConic q;
  float opa, cr, cg, cbl, p2_min;
};

struct BwAcc {
  float g0, g1, g2, g3, sx, sy, g6, g7, g8;
};

// One bucket's stream.  SOFT = false: the tile carries no soft-count gradient,
// so only blended pairs contribute; B.w holds the blend limit n_walk - term.
// SOFT = true: B.w holds n_walk << 1 | terminated and every walked pair with
// alpha below the cap adds its soft term.  The pixel list holds byte offsets
// (p * 16) shared by both per-pixel arrays; the next step's records are
// fetched one step ahead.
// Per-pixel records of the tile being differentiated (k_backward_splat2), at
// file scope so the stream addresses them as list offset + constant base.
// sPA: dL/dr, dL/dg, dL/db, dL/dsoft; sPB: pixel x, y (tile-relative),
// w . image, walk limit; entry [256] = sentinel.  One array, so a pixel's two
// records sit at one register address plus an immediate offset.
__shared__ float4 sPix[2 * (TILE_PX + 1)];
#define sPA (sPix)
#define sPB (sPix + TILE_PX + 1)

// One (pixel, slot) pair of the splat-parallel backward: the pixel record
// (PB: x, y, w . image, walk limit; w: dL/dRGB, dL/dsoft), the slot k, the
// lane's splat; T / H (transmittance, w . C_front) enter and leave updated.
template <bool SOFT>
__device__ __forceinline__ void bw_pair(const float4& PB, const float4& w, int k, const BwSplat& s, BwAcc& g,
                                        float& T, float& H) {
  const int lim = __float_as_int(PB.w);
  const float dx = pair_d(PB.x, s.sm.xi, s.sm.xf), dy = pair_d(PB.y, s.sm.yi, s.sm.yf);
  const float dxx = __fmul_rn(dx, dx), dxy = __fmul_rn(dx, dy), dyy = __fmul_rn(dy, dy);
  float qpos;
  const float p2 = pair_power2(dxx, dxy, dyy, s.q.a2, s.q.b2, s.q.c2, qpos);
  if (!SOFT) {
    const float araw = pair_alpha2(s.opa, p2);
    // (araw >= 1/255 implies p2 >= p2_min: no separate far test here; lanes
    // past the walks have opacity 0).  Branch-free: some lane of the warp
    // nearly always contributes, so the block runs anyway; a lane that does
    // not contributes exactly zero (alpha = 0: T, H and every sum unchanged).
    const bool c = (k < lim) & (p2 <= 0.f) & (araw >= ALPHA_MIN_F);
    const float alpha = c ? fminf(araw, ALPHA_CAP_F) : 0.f;
    const float wc = w.x * s.cr + w.y * s.cg + w.z * s.cbl;
    const float aT = alpha * T;
    g.g0 = fmaf(aT, w.x, g.g0);
    g.g1 = fmaf(aT, w.y, g.g1);
    g.g2 = fmaf(aT, w.z, g.g2);
    const float one_m = __fsub_rn(1.f, alpha);  // >= 0.01
    const float awc = aT * wc;
    const float sdot = PB.z - H - awc;  // w . (colour behind this splat)
    const float dlda = fmaf(T, wc, -sdot * rcp_approx(one_m));
    H = c ? H + awc : H;
    T = __fmul_rn(T, one_m);
    // capped: no opacity/geometry path; a lane that does not blend has
    // alpha = 0 and a finite dlda, so its gp is already zero
    const float gp = araw <= ALPHA_CAP_F ? dlda * alpha : 0.f;
    g.g3 += gp;
    g.sx = fmaf(gp, dx, g.sx);
    g.sy = fmaf(gp, dy, g.sy);
    g.g6 = fmaf(gp, dxx, g.g6);
    g.g8 = fmaf(gp, dyy, g.g8);
    g.g7 = fmaf(gp, dxy, g.g7);
  } else {
    // same branch-free form with the soft-count term of every walked pair
    // below the cap
    const int nw = lim >> 1;
    const bool walked = (k < nw) & (p2 <= 0.f) & (p2 >= s.p2_min);
    const float araw = pair_alpha2(s.opa, p2);
    const bool capped = araw > ALPHA_CAP_F;
    const float alpha = capped ? ALPHA_CAP_F : araw;
    // the terminating slot (k == nw - 1 of a terminated walk) is never blended
    const bool blended = walked & (alpha >= ALPHA_MIN_F) & (k < nw - (lim & 1));
    const float ab = blended ? alpha : 0.f;
    const float wc = w.x * s.cr + w.y * s.cg + w.z * s.cbl;
    const float aT = ab * T;
    g.g0 = fmaf(aT, w.x, g.g0);
    g.g1 = fmaf(aT, w.y, g.g1);
    g.g2 = fmaf(aT, w.z, g.g2);
    const float one_m = __fsub_rn(1.f, ab);
    const float awc = aT * wc;
    const float sdot = PB.z - H - awc;
    const float dlda = blended ? fmaf(T, wc, -sdot * rcp_approx(one_m)) : 0.f;
    H = blended ? H + awc : H;
    T = __fmul_rn(T, one_m);
    const bool soft_ok = walked & !capped;
    const float sv = soft_sigmoid(alpha);
    g.g3 = soft_ok ? fmaf(fmaf(w.w * sv * (1.f - sv), 100.f, dlda), alpha, g.g3) : g.g3;
    const float gp = (soft_ok & blended) ? dlda * alpha : 0.f;
    g.sx = fmaf(gp, dx, g.sx);
    g.sy = fmaf(gp, dy, g.sy);
    g.g6 = fmaf(gp, dxx, g.g6);
    g.g7 = fmaf(gp, dxy, g.g7);
    g.g8 = fmaf(gp, dyy, g.g8);
  }
}

// Two consecutive slots per lane (64-slot buckets, k_backward_splat2): lane l
// owns slots k and k + 1; each pixel record read from shared memory and each
// (T, H) hand-off by shuffle serves two pairs (a one-slot stream ran at 86%
// of the LSU wavefront peak; this one at 49%, limited by occupancy).
template <bool SOFT>
__device__ __forceinline__ void bw_stream2(const uint16_t* __restrict__ list, const float2* __restrict__ seed,
                                           int n_live, int lane, int k, const BwSplat& s0, const BwSplat& s1,
                                           BwAcc& g0, BwAcc& g1) {
  float T = 1.f, H = 0.f;
  const int n_steps = n_live + 31;
  const bool lane0 = lane == 0;
  int jn = BW_PAD - lane;
  int on = list[jn];
  const char* sPixb = reinterpret_cast<const char*>(sPix);
  constexpr int B_OFF = (TILE_PX + 1) * sizeof(float4);
  float4 PBn = *reinterpret_cast<const float4*>(sPixb + on + B_OFF), PAn = *reinterpret_cast<const float4*>(sPixb + on);
#pragma unroll 2
  for (int i = 0; i < n_steps; i++) {
    float Tin = __shfl_up_sync(FULL, T, 1);
    float Hin = __shfl_up_sync(FULL, H, 1);
    const float2 sd = seed[i];
    T = lane0 ? sd.x : Tin;
    H = lane0 ? sd.y : Hin;
    const float4 PB = PBn, w = PAn;
    jn++;
    on = list[jn];
    PBn = *reinterpret_cast<const float4*>(sPixb + on + B_OFF);
    PAn = *reinterpret_cast<const float4*>(sPixb + on);
    bw_pair<SOFT>(PB, w, k, s0, g0, T, H);
    bw_pair<SOFT>(PB, w, k + 1, s1, g1, T, H);
  }
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_backward_splat2(RasterArgs a, const float* __restrict__ d_image,
                                                        const float* __restrict__ d_soft, float* __restrict__ rows) {
  griddep_wait();
  const int t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2 rg = a.ranges[t];
  const int s0 = rg.x, len = rg.y - rg.x;
  if (len == 0) return;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int x00 = tx * TILE, y00 = ty * TILE;
  const int maxw = a.tile_info[t].x;
  const uint32_t gen = rows_generation(rows) + 1;  // k_fix_plan publishes it after this grid

  __shared__ float2 sSeed[8][TILE_PX + 32];  // per warp: (T, H) entering the bucket, i-th live pixel
  __shared__ uint16_t sList[8][BW_LIST];     // per warp: byte offsets of the bucket's live pixel records, padded
  bool soft_px = false;
  {
    const int px = x00 + (tid & 15), py = y00 + (tid >> 4);
    int nw = 0, term = 0;
    float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
    float wimg = 0.f;
    if (px < a.width && py < a.height) {
      const size_t pix = (size_t)py * a.width + px;
      if (!a.flagged[pix]) {
        nw = a.n_walk[pix];
        term = a.term[pix] ? 1 : 0;
      } else {
        nw = fix_kflag(a)[pix];  // slots before the ambiguous one; the fp64 fix-up adds the rest
      }
      w = make_float4(d_image[pix * 3], d_image[pix * 3 + 1], d_image[pix * 3 + 2], d_soft ? d_soft[pix] : 0.f);
      wimg = w.x * a.image[pix * 3] + w.y * a.image[pix * 3 + 1] + w.z * a.image[pix * 3 + 2];
    }
    soft_px = w.w != 0.f;
    sPA[tid] = w;
    // does any pixel of the tile carry a soft-count gradient?  If not, pairs
    // with alpha < 1/255 (and terminating slots) contribute exactly nothing.
    const bool us = __syncthreads_or(soft_px);
    const int lim = us ? ((nw << 1) | term) : nw - term;
    sPB[tid] = make_float4((float)(tid & 15), (float)(tid >> 4), wimg, __int_as_float(lim));
    if (tid < 8)
      for (int e = 0; e < BW_PAD; e++) {
        sList[tid][e] = TILE_PX * sizeof(float4);
        sList[tid][BW_PAD + TILE_PX + e] = TILE_PX * sizeof(float4);
      }
    if (tid == 0) {
      sPA[TILE_PX] = make_float4(0.f, 0.f, 0.f, 0.f);
      sPB[TILE_PX] = make_float4(0.f, 0.f, 0.f, __int_as_float(0));
    }
    soft_px = us;
  }
  __syncthreads();
  const bool use_soft = soft_px;

  const int nb = (maxw + 63) >> 6;  // 64-slot buckets: two slots per lane
  const float4* ckt = a.ckpt + ckpt_base(s0, t);
  const unsigned lt_mask = (1u << lane) - 1u;
  uint16_t* const myList = sList[warp] + BW_PAD;
  float2* const mySeed = sSeed[warp];
  // buckets over the CTA's warps and, for images of few tiles, over gridDim.y
  // CTAs of the same tile (each a copy of the pixel set-up)
  for (int b = warp + 8 * (int)blockIdx.y; b < nb; b += 8 * (int)gridDim.y) {
    const int kb = b * 64;
    int n_live = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) {
      const int p = c * 32 + lane;
      const int lim = __float_as_int(sPB[p].w);
      const bool lv = (use_soft ? (lim >> 1) : lim) > kb;
      const unsigned msk = __ballot_sync(FULL, lv);
      if (lv) myList[n_live + __popc(msk & lt_mask)] = (uint16_t)(p * sizeof(float4));
      n_live += __popc(msk);
    }
    if (n_live + lane < TILE_PX) myList[n_live + lane] = TILE_PX * sizeof(float4);
    __syncwarp();
    for (int j = lane; j < n_live; j += 32) {
      const int p = myList[j] / sizeof(float4);
      float2 sd = make_float2(1.f, 0.f);
      if (b > 0) {  // the forward's checkpoint at slot kb (every other 32-slot checkpoint)
        const float4 c = ckt[(size_t)(2 * b) * TILE_PX + p];
        const float4 w = sPA[p];
        sd = make_float2(c.x, w.x * c.y + w.y * c.z + w.z * c.w);
      }
      mySeed[j] = sd;
    }
    mySeed[n_live + lane] = make_float2(1.f, 0.f);
    __syncwarp();
    const int k = kb + 2 * lane;
    BwSplat sp[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      BwSplat& sv = sp[h];
      sv.sm = {0.f, 0.f, 0.f, 0.f};
      sv.q = {0.f, 0.f, 0.f};
      sv.opa = sv.cr = sv.cg = sv.cbl = 0.f;
      sv.p2_min = __int_as_float(0x7f800000);
      if (k + h < maxw) {
        const uint32_t g = a.inst[s0 + k + h];
        const double2 m = a.mean[g];
        const float4 co = a.conic_opa[g];
        const float4 col = a.color[g];
        sv.sm = stage_mean(m.x, m.y, x00, y00);
        sv.opa = fabsf(co.w);
        sv.q = stage_conic(co.x, co.y, co.z);
        sv.cr = col.x;
        sv.cg = col.y;
        sv.cbl = col.z;
        sv.p2_min = use_soft ? FAR_POWER2 : fmaxf(FAR_POWER2, __log2f(0.999f * ALPHA_MIN_F / sv.opa));
      }
    }
    BwAcc g[2] = {{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}};
    if (use_soft)
      bw_stream2<true>(sList[warp], mySeed, n_live, lane, k, sp[0], sp[1], g[0], g[1]);
    else
      bw_stream2<false>(sList[warp], mySeed, n_live, lane, k, sp[0], sp[1], g[0], g[1]);
    // the row index and conic are re-read after the stream (registers are the limit)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (k + h < maxw) {
        const uint32_t gi = a.inst[s0 + k + h];
        const float4 co = a.conic_opa[gi];
        store_row(rows, inst_row(a, gi, tx, ty), g[h].g0, g[h].g1, g[h].g2, g[h].g3 * (1.f - fabsf(co.w)),
                  co.x * g[h].sx + co.y * g[h].sy, co.y * g[h].sx + co.z * g[h].sy, -0.5f * g[h].g6, -g[h].g7,
                  -0.5f * g[h].g8, gen);
      }
    }
    __syncwarp();
  }
  // slots k >= maxw: no row (their tag stays stale, ssr_common.cuh)
}

// ------------------------------------------------------------------ backward, pixel-parallel (fp32)
// The no_splat_parallel ablation (pipeline.py:130-131): thread per pixel,
// each slot's 9 terms reduced across the warp by shuffles, per-warp partials
// summed in a fixed order (deterministic), one row write per slot.
__global__ void __launch_bounds__(256) k_backward_pixel(RasterArgs a, const float* __restrict__ d_image,
                                                        const float* __restrict__ d_soft, float* __restrict__ rows) {
  griddep_wait();
  const int t = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2 rg = a.ranges[t];
  const int s0 = rg.x, len = rg.y - rg.x;
  if (len == 0) return;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int x00 = tx * TILE, y00 = ty * TILE;
  const int maxw = a.tile_info[t].x;
  const uint32_t gen = rows_generation(rows) + 1;  // k_fix_plan publishes it after this grid
  __shared__ float4 sA[32], sB[32];
  __shared__ float4 sQ[32], sM[32];
  __shared__ uint32_t sRow[32];
  __shared__ float part[8][32][9];

  const int px = x00 + (tid & 15), py = y00 + (tid >> 4);
  int nw = 0, term = 0;
  float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
  float wimg = 0.f;
  if (px < a.width && py < a.height) {
    const size_t pix = (size_t)py * a.width + px;
    if (!a.flagged[pix]) {
      nw = a.n_walk[pix];
      term = a.term[pix];
    } else {
      nw = fix_kflag(a)[pix];  // slots before the ambiguous one; the fp64 fix-up adds the rest
    }
    w = make_float4(d_image[pix * 3], d_image[pix * 3 + 1], d_image[pix * 3 + 2], d_soft ? d_soft[pix] : 0.f);
    wimg = w.x * a.image[pix * 3] + w.y * a.image[pix * 3 + 1] + w.z * a.image[pix * 3 + 2];
  }
  const float fpx = (float)(tid & 15), fpy = (float)(tid >> 4);
  float T = 1.f, H = 0.f;
  for (int kb = 0; kb < maxw; kb += 32) {
    if (tid < 32 && kb + tid < maxw) {
      const uint32_t g = a.inst[s0 + kb + tid];
      const double2 m = a.mean[g];
      const float4 co = a.conic_opa[g];
      const float4 col = a.color[g];
      const StagedConic q = stage_conic(co.x, co.y, co.z);
      const StagedMean sm = stage_mean(m.x, m.y, x00, y00);
      sM[tid] = make_float4(sm.xi, sm.xf, sm.yi, sm.yf);
      sA[tid] = make_float4(0.f, 0.f, co.x, co.y);
      sB[tid] = make_float4(co.z, fabsf(co.w), col.x, col.y);
      sQ[tid] = make_float4(q.a2, q.b2, q.c2, col.z);
      sRow[tid] = inst_row(a, g, tx, ty);
    }
    __syncthreads();
    const int nc = min(32, maxw - kb);
    for (int j = 0; j < nc; j++) {
      const int k = kb + j;
      float c[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (k < nw) {
        const float4 A = sA[j], B = sB[j], Q = sQ[j], M = sM[j];
        const float dx = pair_d(fpx, M.x, M.y), dy = pair_d(fpy, M.z, M.w);
        const float dxx = __fmul_rn(dx, dx), dxy = __fmul_rn(dx, dy), dyy = __fmul_rn(dy, dy);
        float qpos;
        const float p2 = pair_power2(dxx, dxy, dyy, Q.x, Q.y, Q.z, qpos);
        if (p2 <= 0.f && p2 >= FAR_POWER2) {
          const float araw = pair_alpha2(B.y, p2);
          const bool capped = araw > ALPHA_CAP_F;
          const float alpha = capped ? ALPHA_CAP_F : araw;
          const bool blended = alpha >= ALPHA_MIN_F && !(term && k == nw - 1);
          float dlda = 0.f;
          if (blended) {
            const float wc = w.x * B.z + w.y * B.w + w.z * Q.w;
            const float aT = alpha * T;
            c[0] = aT * w.x;
            c[1] = aT * w.y;
            c[2] = aT * w.z;
            const float one_m = __fsub_rn(1.f, alpha);
            dlda = T * wc - __fdividef(wimg - H - aT * wc, one_m);
            H += aT * wc;
            T = __fmul_rn(T, one_m);
          }
          if (!capped) {
            const float sv = soft_sigmoid(alpha);
            c[3] = (dlda + w.w * sv * (1.f - sv) * 100.f) * alpha * (1.f - B.y);
            if (blended) {
              const float gp = dlda * alpha;
              c[4] = gp * (A.z * dx + A.w * dy);
              c[5] = gp * (A.w * dx + B.x * dy);
              c[6] = gp * (-0.5f * dxx);
              c[7] = gp * (-dxy);
              c[8] = gp * (-0.5f * dyy);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 9; q++) {
        float v = c[q];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        c[q] = v;
      }
      if (lane == 0)
        for (int q = 0; q < 9; q++) part[warp][j][q] = c[q];
    }
    __syncthreads();
    for (int e = tid; e < nc * ROW_WORDS; e += blockDim.x) {
      const int j = e / ROW_WORDS, q = e % ROW_WORDS;
      float v = __uint_as_float(gen);
      if (q < 9) {
        v = 0.f;
        for (int ww = 0; ww < 8; ww++) v += part[ww][j][q];
      }
      rows[ROWS_HEAD + (size_t)sRow[j] * ROW_WORDS + q] = v;
    }
    __syncthreads();
  }
  // slots k >= maxw: no row (their tag stays stale, ssr_common.cuh)
}

// ------------------------------------------------------------------ backward fix-up (fp64)
// Adds the float64 pixel-walk gradient terms of guard-band pixels
// (kernels.py:149-193 semantics, front to back) into the rows the fp32 kernel
// wrote.  One warp per (tile, 32-slot bucket): it seeds each flagged pixel of
// the tile from the bucket checkpoint the forward fix-up wrote, evaluates the
// bucket's slots in float64 (lanes = slots), and accumulates the pixels'
// terms in a fixed (pixel) order before one add per slot -- deterministic
// without atomics, and parallel over buckets.  Backward decisions do not
// depend on T (termination comes from n_walk / terminated), so fp32 seeds only
// perturb gradient values, never which slots blend.
// Buckets of flagged tile slot `it` the backward fix-up visits: from the one
// holding the tile's first flagged slot to the end of its longest flagged walk.
__device__ __forceinline__ int fix_tile_buckets(const RasterArgs& a, int it) {
  const int4 ti = a.tile_info[fix_pixels(a)[fix_tiles(a)[it]] >> 8];
  return max(0, ((ti.z + 31) >> 5) - (ti.w >> 5));
}

// Bucket plan of the backward fix-up: exclusive prefix over the flagged tiles
// of their bucket counts (one CTA; <= n_tiles entries), total in fix[2].
__global__ void __launch_bounds__(1024) k_fix_plan(RasterArgs a, float* rows) {
  griddep_wait();
  // the backward grid has finished reading the old generation: publish the new one
  if (threadIdx.x == 0) *reinterpret_cast<uint32_t*>(rows) = rows_generation(rows) + 1;
  __shared__ int s_part[32];
  const int n_ft = a.fix[1];
  const int per = (n_ft + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(lo + per, n_ft);
  int sum = 0;
  for (int it = lo; it < hi; it++) sum += fix_tile_buckets(a, it);
  // block exclusive scan of the per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = sum;
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(FULL, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) s_part[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = s_part[lane], vi = v;
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(FULL, vi, d);
      if (lane >= d) vi += o;
    }
    s_part[lane] = vi - v;
    if (lane == 31) a.fix[2] = vi;
  }
  __syncthreads();
  int run = s_part[warp] + incl - sum;
  for (int it = lo; it < hi; it++) {
    fix_plan(a)[it] = run;
    run += fix_tile_buckets(a, it);
  }
}

// Work items are the (flagged tile, bucket) pairs of the plan, strided
// statically over every warp of a persistent grid (no tile-sized serial
// chains; deterministic).  A warp loads its bucket's 32 slots and the tile's
// flagged-pixel inputs (lane f holds pixel f, broadcast by shuffles) in
// parallel, walks the flagged pixels in pixel order (seeded from the
// checkpoints the forward fix-up wrote) and adds each slot's float64 sum to its
// row with one plain add: every row is owned by exactly one item.
__global__ void __launch_bounds__(256, 2) k_backward_fixup(RasterArgs a, const float* __restrict__ d_image,
                                                           const float* __restrict__ d_soft, float* __restrict__ rows) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int n_ft = a.fix[1];
  const int n_items = a.fix[2];
  const int n_warps = gridDim.x * (blockDim.x >> 5);
  const bool soft_grad = d_soft != nullptr;
  const int* plan = fix_plan(a);
  for (int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < n_items; item += n_warps) {
    // tile of this item: the last plan entry <= item (the plan is
    // non-decreasing), by a 32-way warp search: each level narrows the range
    // 32x with one load per lane (3 dependent loads at 8160 tiles, not 13)
    int lo = 0, hi = n_ft;
    while (hi - lo > 1) {
      const int step = (hi - lo + 31) >> 5;
      const int idx = lo + lane * step;
      const unsigned ok = __ballot_sync(FULL, idx < hi && plan[idx] <= item);  // lane 0 always
      lo += (31 - __clz(ok)) * step;
      hi = min(hi, lo + step);
    }
    const int it = lo;
    const int start = fix_tiles(a)[it];
    const int* plist = fix_pixels(a) + start;
    const int t = plist[0] >> 8;
    const int4 ti = a.tile_info[t];
    const int nflag = ti.y;
    const int b = (ti.w >> 5) + item - plan[lo];
    const int kb = b * 32, k = kb + lane;
    const int tx = t % a.tiles_x, ty = t / a.tiles_x;
    const int2 rg = a.ranges[t];
    const int s0 = rg.x, s1 = rg.y;
    const float4* ckt = a.ckpt + ckpt_base(s0, t);
    SlotRaw raw;
    load_slot(a, s0 + k, s1, raw);
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int f0 = 0; f0 < nflag; f0 += 32) {
      // lane f - f0 loads flagged pixel f's inputs
      int my_p = 0, my_nw = 0, my_term = 0, my_kf = 0;
      double my_w0 = 0.0, my_w1 = 0.0, my_w2 = 0.0, my_ws = 0.0, my_wimg = 0.0;
      float4 my_ck = make_float4(1.f, 0.f, 0.f, 0.f);
      if (f0 + lane < nflag) {
        my_p = plist[f0 + lane] & 255;
        const size_t pix = (size_t)(ty * TILE + (my_p >> 4)) * a.width + tx * TILE + (my_p & 15);
        my_nw = a.n_walk[pix];
        my_term = a.term[pix];
        my_kf = fix_kflag(a)[pix];
        my_w0 = d_image[pix * 3];
        my_w1 = d_image[pix * 3 + 1];
        my_w2 = d_image[pix * 3 + 2];
        my_ws = soft_grad ? (double)d_soft[pix] : 0.0;
        my_wimg = my_w0 * (double)a.image[pix * 3] + my_w1 * (double)a.image[pix * 3 + 1] +
                  my_w2 * (double)a.image[pix * 3 + 2];
        if (b > 0 && my_nw > kb) my_ck = ckt[(size_t)b * TILE_PX + my_p];
      }
      // pixels whose fp64 part [kflag, n_walk) meets this bucket
      const unsigned walks = __ballot_sync(FULL, f0 + lane < nflag && my_nw > kb && my_kf < kb + 32);
      for (unsigned rem = walks; rem; rem &= rem - 1) {
        const int f = __ffs(rem) - 1;
        const int p = __shfl_sync(FULL, my_p, f), nw = __shfl_sync(FULL, my_nw, f);
        const int term = __shfl_sync(FULL, my_term, f), kf = __shfl_sync(FULL, my_kf, f);
        const double w0 = __shfl_sync(FULL, my_w0, f), w1 = __shfl_sync(FULL, my_w1, f),
                     w2 = __shfl_sync(FULL, my_w2, f), ws = __shfl_sync(FULL, my_ws, f),
                     wimg = __shfl_sync(FULL, my_wimg, f);
        const float ckx = __shfl_sync(FULL, my_ck.x, f), cky = __shfl_sync(FULL, my_ck.y, f),
                    ckz = __shfl_sync(FULL, my_ck.z, f), ckw = __shfl_sync(FULL, my_ck.w, f);
        const int px = tx * TILE + (p & 15), py = ty * TILE + (p >> 4);
        const double T = (double)ckx;
        const double H = w0 * cky + w1 * ckz + w2 * ckw;
        Slot64 sl;
        eval_slot(raw, k < nw && raw.valid, (double)px, (double)py, sl, soft_grad);
        const bool bl = sl.cand && !(term && k == nw - 1);
        const double f1 = bl ? (1.0 - sl.alpha) : 1.0;
        double P = f1;
        for (int d = 1; d < 32; d <<= 1) {
          const double o = __shfl_up_sync(FULL, P, d);
          if (lane >= d) P *= o;
        }
        double Pex = __shfl_up_sync(FULL, P, 1);
        if (lane == 0) Pex = 1.0;
        const double Tb = T * Pex;
        const double wc = bl ? (w0 * sl.col[0] + w1 * sl.col[1] + w2 * sl.col[2]) : 0.0;
        const double e = bl ? sl.alpha * Tb * wc : 0.0;
        double E = e;  // inclusive prefix sum of w.(c alpha T)
        for (int d = 1; d < 32; d <<= 1) {
          const double o = __shfl_up_sync(FULL, E, d);
          if (lane >= d) E += o;
        }
        const double Hb = H + (E - e);
        if (sl.valid && !sl.skip && k >= kf) {  // earlier slots: the fp32 backward's
          double dlda = 0.0;
          if (bl) {
            const double aT = sl.alpha * Tb;
            acc[0] += aT * w0;
            acc[1] += aT * w1;
            acc[2] += aT * w2;
            dlda = Tb * wc - (wimg - Hb - aT * wc) / (1.0 - sl.alpha);
          }
          if (!sl.capped) {
            acc[3] += (dlda + ws * sl.sv * (1.0 - sl.sv) / SOFT_TAU) * sl.alpha * (1.0 - sl.opa);
            if (bl) {
              const double gp = dlda * sl.alpha;
              acc[4] += gp * (sl.qa * sl.dx + sl.qb * sl.dy);
              acc[5] += gp * (sl.qb * sl.dx + sl.qc * sl.dy);
              acc[6] += gp * (-0.5 * sl.dx * sl.dx);
              acc[7] += gp * (-sl.dx * sl.dy);
              acc[8] += gp * (-0.5 * sl.dy * sl.dy);
            }
          }
        }
      }
    }
    if (raw.valid) {
      float* row = rows + ROWS_HEAD + (size_t)inst_row(a, raw.g, tx, ty) * ROW_WORDS;
      for (int j = 0; j < 9; j++)
        if (acc[j] != 0.0) row[j] += (float)acc[j];
    }
  }
}

static int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

extern "C" int64_t ssr_rows_floats(int64_t m) {
  return ROWS_HEAD + (m > 0 ? m : 1) * ROW_WORDS + 4;  // +4: the chain's 16-byte aligned TMA windows
}

extern "C" int64_t ssr_fix_list_ints(int32_t width, int32_t height, int32_t n_tiles) {
  return FIX_HEAD + 2 * (int64_t)n_tiles + 2 * (int64_t)width * height;
}

static RasterArgs make_args(ssr_splats sp, const uint32_t* inst, const int32_t* ranges, const ssr_frame& f,
                            float band, float band_t) {
  RasterArgs a;
  a.width = f.width;
  a.height = f.height;
  a.tiles_x = f.tiles_x;
  a.tiles_y = f.tiles_y;
  for (int i = 0; i < 3; i++) {
    a.bg[i] = f.bg[i];
    a.bg64[i] = (double)f.bg[i];
  }
  a.band = band;
  a.band_t = band_t;
  a.mean = (const double2*)sp.mean;
  a.conic_opa = (const float4*)sp.conic_opa;
  a.color = (const float4*)sp.color;
  a.conic_opa64 = (const double2*)sp.conic_opa64;
  a.color64 = (const double2*)sp.color64;
  a.rect = (const int4*)sp.rect;
  a.row_offset = sp.row_offset;
  a.inst = inst;
  a.ranges = (const int2*)ranges;
  a.image = f.image;
  a.t_final = f.t_final;
  a.n_walk = f.n_walk;
  a.term = f.terminated;
  a.hard = f.hard_count;
  a.soft = f.soft_count;
  a.flagged = f.flagged;
  a.tile_info = (int4*)f.tile_info;
  a.ckpt = (float4*)f.ckpt;
  a.fix = f.fix_list;
  a.n_tiles = f.tiles_x * f.tiles_y;
  return a;
}

}  // namespace ssr

using namespace ssr;

extern "C" int ssr_forward(int64_t m, ssr_splats splats, const uint32_t* inst_gauss, const int32_t* tile_ranges,
                           ssr_frame frame, float band_alpha, float band_t, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int n_tiles = frame.tiles_x * frame.tiles_y;
  if (n_tiles <= 0 || frame.width <= 0 || frame.height <= 0 || m < 0 || !(band_alpha >= 0.f) || !(band_t >= 0.f)) {
    set_error("ssr_forward: invalid argument");
    return SSR_ERR_INVALID;
  }
  RasterArgs a = make_args(splats, inst_gauss, tile_ranges, frame, band_alpha, band_t);
  if (!frame.fix_list) {
    set_error("ssr_forward: frame.fix_list is required");
    return SSR_ERR_INVALID;
  }
  SSR_TRY(launch_pdl("k_fix_reset", k_fix_reset, dim3(1), dim3(32), 0, st, frame.fix_list));
  // frame.ckpt == NULL: render-only (no backward state beyond the per-pixel outputs)
  // frame.soft_count == NULL: no soft-count output (the caller's loss does not
  // read it); the walk then culls pairs below 1/255 at the packed far test
  if (frame.ckpt)
    if (frame.soft_count)
      SSR_TRY(launch_pdl("k_forward", k_forward<true, true>, dim3(n_tiles), dim3(TILE_PX), 0, st, a));
    else
      SSR_TRY(launch_pdl("k_forward", k_forward<true, false>, dim3(n_tiles), dim3(TILE_PX), 0, st, a));
  else if (frame.soft_count)
    SSR_TRY(launch_pdl("k_forward", k_forward<false, true>, dim3(n_tiles), dim3(TILE_PX), 0, st, a));
  else
    SSR_TRY(launch_pdl("k_forward", k_forward<false, false>, dim3(n_tiles), dim3(TILE_PX), 0, st, a));
  SSR_TRY(check_launch("k_forward"));
  return launch_pdl("k_forward_fixup", k_forward_fixup, dim3(num_sms() * 4), dim3(256), 0, st, a);
}

extern "C" int ssr_backward(int32_t layout, int64_t m, ssr_splats splats, const uint32_t* inst_gauss,
                            const int32_t* tile_ranges, ssr_frame frame, const float* d_image, const float* d_soft,
                            float* inst_rows, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int n_tiles = frame.tiles_x * frame.tiles_y;
  if (n_tiles <= 0 || (layout != 0 && layout != 1) || !d_image) {
    set_error("ssr_backward: invalid argument (layout must be 0=splat or 1=pixel)");
    return SSR_ERR_INVALID;
  }
  if (m == 0) return SSR_OK;
  if (!frame.ckpt) {
    set_error("ssr_backward: the frame was rendered without checkpoints (render-only)");
    return SSR_ERR_INVALID;
  }
  if (d_soft && !frame.soft_count && layout == 0) {
    set_error("ssr_backward: a soft-count gradient needs a frame rendered with soft counts");
    return SSR_ERR_INVALID;
  }
  if (!frame.fix_list || !inst_rows) {
    set_error("ssr_backward: frame.fix_list and inst_rows are required");
    return SSR_ERR_INVALID;
  }
  RasterArgs a = make_args(splats, inst_gauss, tile_ranges, frame, 0.f, 0.f);
  // few tiles (small images): split each tile's buckets over up to 8 CTAs so
  // the grid still fills the GPU (bucket rows are disjoint: no conflicts)
  const int split = max(1, min(8, (num_sms() * 4 + n_tiles - 1) / n_tiles));
  if (layout == 0) {
    // two slots per lane, 64-slot buckets; the soft pair block (d_soft given)
    // needs more registers
    if (!d_soft)
      SSR_TRY(launch_pdl("k_backward_splat2", k_backward_splat2<BW2_MIN_BLOCKS>, dim3(n_tiles, split), dim3(TILE_PX), 0,
                         st, a, d_image, d_soft, inst_rows));
    else
      SSR_TRY(launch_pdl("k_backward_splat2", k_backward_splat2<BW2_SOFT_MIN_BLOCKS>, dim3(n_tiles, split),
                         dim3(TILE_PX), 0, st, a, d_image, d_soft, inst_rows));
  }
  else
    SSR_TRY(launch_pdl("k_backward_pixel", k_backward_pixel, dim3(n_tiles), dim3(TILE_PX), 0, st, a, d_image, d_soft,
                       inst_rows));
  SSR_TRY(check_launch(layout == 0 ? "k_backward_splat2" : "k_backward_pixel"));
  SSR_TRY(launch_pdl("k_fix_plan", k_fix_plan, dim3(1), dim3(1024), 0, st, a, inst_rows));
  return launch_pdl("k_backward_fixup", k_backward_fixup, dim3(num_sms() * 2), dim3(256), 0, st, a, d_image, d_soft,
                    inst_rows);
}
