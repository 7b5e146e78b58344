// Field snapshot records (io/ply.py:29-54 / 57-124 of the reference): the
// flat class-major float32 parameter buffer <-> the PLY body, one vertex of
// doubles per Gaussian in property order
//   x y z nx ny nz f_dc_0..2 f_rest_0..3(K-1)-1 opacity scale_0..2 rot_0..3
// with the rest coefficients channel-major (io/ply.py:43).  float32 -> float64
// is exact, so a pack/unpack round trip reproduces every parameter bit for
// bit; unpack rounds foreign doubles to nearest float32.
//
// One thread per (vertex, property): the record array is written (packed) or
// read (unpacked) fully coalesced, the class-major side is a strided gather
// that the L2 absorbs (HBM-bound either way; a snapshot is not on the
// per-iteration path).
#include "ssr_common.cuh"

namespace ssr {

// Flat-buffer element of property j of row i (-1: the zero normals).
__device__ __forceinline__ int64_t ply_src(int64_t i, int j, int K, int64_t ns) {
  const int n_rest = 3 * (K - 1);
  if (j < 3) return i * 3 + j;                        // x y z
  if (j < 6) return -1;                               // nx ny nz
  if (j < 9) return 11 * ns + i * 3 * K + (j - 6) * K;  // f_dc_c = sh[c][0]
  if (j < 9 + n_rest) {                               // f_rest_r, r = c (K-1) + (k-1)
    const int r = j - 9, c = r / (K - 1), k = r % (K - 1) + 1;
    return 11 * ns + i * 3 * K + c * K + k;
  }
  const int q = j - 9 - n_rest;
  if (q == 0) return 10 * ns + i;                     // opacity (logit)
  if (q < 4) return 7 * ns + i * 3 + (q - 1);         // scale_0..2 (log scales)
  return 3 * ns + i * 4 + (q - 4);                    // rot_0..3
}

__global__ void __launch_bounds__(256) k_ply_pack(int64_t n, int K, const float* __restrict__ params,
                                                  double* __restrict__ rec) {
  const int P = 17 + 3 * (K - 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * P) return;
  const int64_t i = e / P;
  const int j = (int)(e - i * P);
  const int64_t s = ply_src(i, j, K, row_stride(n));
  rec[e] = s < 0 ? 0.0 : (double)params[s];
}

__global__ void __launch_bounds__(256) k_ply_unpack(int64_t n, int K, const double* __restrict__ rec,
                                                    float* __restrict__ params) {
  const int P = 17 + 3 * (K - 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * P) return;
  const int64_t i = e / P;
  const int j = (int)(e - i * P);
  const int64_t s = ply_src(i, j, K, row_stride(n));
  if (s >= 0) params[s] = __double2float_rn(rec[e]);
}

}  // namespace ssr

using namespace ssr;

extern "C" int32_t ssr_ply_properties(int32_t sh_degree) {
  if (sh_degree < 0 || sh_degree > 3) return -1;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  return 17 + 3 * (K - 1);
}

extern "C" int ssr_ply_pack(int64_t n, int32_t sh_degree, const float* params, double* records, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || (n > 0 && (!params || !records))) {
    set_error("ssr_ply_pack: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  const int64_t total = n * ssr_ply_properties(sh_degree);
  k_ply_pack<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, K, params, records);
  return check_launch("k_ply_pack");
}

extern "C" int ssr_ply_unpack(int64_t n, int32_t sh_degree, const double* records, float* params, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || (n > 0 && (!params || !records))) {
    set_error("ssr_ply_unpack: invalid argument");
    return SSR_ERR_INVALID;
  }
  if (n == 0) return SSR_OK;
  const int K = (sh_degree + 1) * (sh_degree + 1);
  const int64_t total = n * ssr_ply_properties(sh_degree);
  k_ply_unpack<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, K, records, params);
  return check_launch("k_ply_unpack");
}
