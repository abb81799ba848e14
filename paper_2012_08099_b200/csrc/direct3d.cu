// direct3d.cu -- the reference's direct engines on the device (not the hot path).
//
// The reference registers three engines (moments3d.py:267-271): the projection
// method dpm_moments, and two direct evaluations of Eq. 2 it cross-checks it
// with, naive_moments (moments3d.py:78-139: every voxel times every moment's
// in-plane monomial, Theta(#moments * LMN) multiplications) and
// factored_moments (moments3d.py:142-198: x-rows -> y-slices -> z, K
// multiplications per voxel).  Here both are exact sums on the device, so the
// drop-in's ENGINES holds all three and verify_engines cross-checks them the
// way the reference does.  Arithmetic is mod 2^128 (unsigned __int128), exact
// for every moment inside the envelope dpm_check_envelope guards (< 2^126).
//
//   stage 1 (direct_planes_kernel, one CTA per (volume, plane z)):
//     P_pq(z) = sum_{y,x} V(x,y,z) x^p y^q   for p + q <= K
//     NAIVE:    per voxel, every (p, q) monomial x^p y^q multiplied in
//     FACTORED: per row y, R_p = sum_x V x^p; then R_p y^q per row
//     -> 32-bit limb sums in uint64 (the moments2d accumulator format)
//   stage 2 (direct_volume_kernel, one CTA per (volume, moment)):
//     M_pqr = sum_z P_pq(z) (z + z0)^r
#include "derive_dev.cuh"

namespace dpm {

constexpr int DT_THREADS = 128;

struct DirectParams {
  const void* vox;
  int64_t L, M, N, B;
  int64_t sy, sz, sb;
  int32_t offset, dtype;
  int64_t z0;
  uint64_t* planes;   // [B][N][n2d][4]
  int64_t* out_i128;  // [B][n3d][2]
  double* out_f64;    // [B][n3d]
};

__device__ __forceinline__ uint32_t dt_voxel(const DirectParams& p, int64_t off) {
  switch (p.dtype) {
    case DPM_U8: return static_cast<const uint8_t*>(p.vox)[off];
    case DPM_U16: return static_cast<const uint16_t*>(p.vox)[off];
    default: return (uint32_t)((int32_t) static_cast<const int16_t*>(p.vox)[off] + p.offset);
  }
}

// CTA-wide sum of per-thread 128-bit values (mod 2^128) as four 32-bit limb sums
template <int NV>
__device__ __forceinline__ void dt_reduce_store(const unsigned __int128 (&v)[NV], uint64_t* out, uint64_t* red) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NWARP = DT_THREADS / 32;
  #pragma unroll
  for (int i = 0; i < NV; ++i) {
    #pragma unroll
    for (int l = 0; l < 4; ++l) {
      uint64_t s = (uint32_t)(v[i] >> (32 * l));
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[(w * NV + i) * 4 + l] = s;
    }
  }
  __syncthreads();
  for (int j = tid; j < NV * 4; j += DT_THREADS) {
    uint64_t s = 0;
    #pragma unroll
    for (int ww = 0; ww < NWARP; ++ww) s += red[ww * NV * 4 + j];
    out[j] = s;
  }
}

template <int K, bool NAIVE>
__global__ void __launch_bounds__(DT_THREADS) direct_planes_kernel(DirectParams p) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  __shared__ uint64_t red[(DT_THREADS / 32) * N2 * 4];
  typedef unsigned __int128 u128;
  const int64_t b = blockIdx.x / p.N, z = blockIdx.x - b * p.N;
  u128 acc[N2];
  #pragma unroll
  for (int i = 0; i < N2; ++i) acc[i] = 0;
  for (int64_t y = threadIdx.x; y < p.M; y += DT_THREADS) {
    const int64_t row = b * p.sb + z * p.sz + y * p.sy;
    u128 yq[K + 1];
    yq[0] = 1;
    #pragma unroll
    for (int q = 1; q <= K; ++q) yq[q] = yq[q - 1] * (u128)(uint64_t)y;
    if constexpr (NAIVE) {
      for (int64_t x = 0; x < p.L; ++x) {
        const uint32_t v = dt_voxel(p, row + x);
        if (v == 0) continue;
        u128 xp = 1;
        int i = 0;
        #pragma unroll
        for (int pp = 0; pp <= K; ++pp) {
          #pragma unroll
          for (int q = 0; q <= K - pp; ++q, ++i) acc[i] += (u128)v * xp * yq[q];   // the (p, q) monomial, term by term
          xp *= (u128)(uint64_t)x;
        }
      }
    } else {
      u128 R[K + 1];
      #pragma unroll
      for (int pp = 0; pp <= K; ++pp) R[pp] = 0;
      for (int64_t x = 0; x < p.L; ++x) {
        const uint32_t v = dt_voxel(p, row + x);
        if (v == 0) continue;
        u128 t = v;
        #pragma unroll
        for (int pp = 0; pp <= K; ++pp) { R[pp] += t; t *= (u128)(uint64_t)x; }
      }
      int i = 0;
      #pragma unroll
      for (int pp = 0; pp <= K; ++pp) {
        #pragma unroll
        for (int q = 0; q <= K - pp; ++q, ++i) acc[i] += R[pp] * yq[q];
      }
    }
  }
  dt_reduce_store<N2>(acc, p.planes + (blockIdx.x * (int64_t)N2) * 4, red);
}

template <int K>
__global__ void __launch_bounds__(DT_THREADS) direct_volume_kernel(DirectParams p) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  constexpr int N3 = (K + 1) * (K + 2) * (K + 3) / 6;
  __shared__ uint64_t red[(DT_THREADS / 32) * 4];
  __shared__ uint64_t fin[4];
  typedef unsigned __int128 u128;
  const int64_t b = blockIdx.x / N3;
  const int m = (int)(blockIdx.x - b * N3);
  int pp = 0, qq = 0, rr = 0;
  {   // moment m in moment_indices order (moments3d.py:46-54)
    int n = 0;
    for (int a = 0; a <= K; ++a)
      for (int c = 0; c <= K - a; ++c)
        for (int e = 0; e <= K - a - c; ++e, ++n)
          if (n == m) { pp = a; qq = c; rr = e; }
  }
  const int slot = idx2(K, pp, qq);
  u128 acc[1] = {0};
  for (int64_t z = threadIdx.x; z < p.N; z += DT_THREADS) {
    const uint64_t* l = p.planes + ((b * p.N + z) * N2 + slot) * 4;
    const u128 P = (u128)l[0] + ((u128)l[1] << 32) + ((u128)l[2] << 64) + ((u128)l[3] << 96);
    u128 zr = 1;
    for (int e = 0; e < rr; ++e) zr *= (u128)(uint64_t)(z + p.z0);
    acc[0] += P * zr;
  }
  dt_reduce_store<1>(acc, fin, red);
  __syncthreads();
  if (threadIdx.x == 0) {
    const u128 v = (u128)fin[0] + ((u128)fin[1] << 32) + ((u128)fin[2] << 64) + ((u128)fin[3] << 96);
    p.out_i128[(b * N3 + m) * 2 + 0] = (int64_t)(uint64_t)v;
    p.out_i128[(b * N3 + m) * 2 + 1] = (int64_t)(uint64_t)(v >> 64);
    if (p.out_f64) p.out_f64[b * N3 + m] = i128_to_f64((i128)v);
  }
}

template <int K>
static void direct_launch(const DirectParams& p, bool naive, cudaStream_t st) {
  constexpr int N3 = (K + 1) * (K + 2) * (K + 3) / 6;
  if (naive) direct_planes_kernel<K, true><<<(unsigned)(p.B * p.N), DT_THREADS, 0, st>>>(p);
  else direct_planes_kernel<K, false><<<(unsigned)(p.B * p.N), DT_THREADS, 0, st>>>(p);
  direct_volume_kernel<K><<<(unsigned)(p.B * N3), DT_THREADS, 0, st>>>(p);
}

int launch_direct3d(const dpm_volume_desc* d, const void* vox, int order, bool naive, uint64_t* planes,
                    int64_t* out_i128, double* out_f64, cudaStream_t st) {
  DirectParams p;
  p.vox = vox; p.L = d->L; p.M = d->M; p.N = d->N; p.B = d->B;
  p.sy = d->stride_y; p.sz = d->stride_z; p.sb = d->B > 1 ? d->stride_b : 0;
  p.offset = d->offset; p.dtype = d->dtype; p.z0 = d->z0;
  p.planes = planes; p.out_i128 = out_i128; p.out_f64 = out_f64;
  if (p.B * p.N > 0x7fffffffLL) return DPM_EINVAL;
  switch (order) {
    case 3: direct_launch<3>(p, naive, st); break;
    case 4: direct_launch<4>(p, naive, st); break;
    case 5: direct_launch<5>(p, naive, st); break;
    default: direct_launch<6>(p, naive, st); break;
  }
  note_launches(2);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
