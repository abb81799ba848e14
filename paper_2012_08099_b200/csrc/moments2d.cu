// moments2d.cu -- exact 2D raw moments of every projection image.
//
// M_pq = sum_j (j+aj)^q * sum_i I[j][i] (i+ai)^p   for p + q <= K.
//
// Replaces the reference's 1D-integral route (drt2d.integrals/assemble_2d,
// drt2d.py:92-174, plus shift_origin :196-208 and exact.weighted_power_sums,
// exact.py:63-82).  That route caps at 2D order 4; this one reaches the order 6
// the extension needs and stays exact:
//   stage 1 (per column i, per chunk of <= 256 rows):
//       C_q[i] = sum_j I[j][i] (j+aj)^q, with (j+aj)^q split into 24-bit limbs
//       held in a per-CTA shared table, so every product is one IMAD.WIDE.U32
//       (32 x 24 -> 56 bits) accumulated into a uint64 that cannot overflow in
//       256 rows;
//   stage 2 (per column): C_q as a 128-bit integer times (i+ai)^p (signed),
//       reduced over the CTA's columns and added into four 32-bit limb
//       accumulators per moment with 64-bit atomics (exact, order independent).
// The host checks the exactness envelope first (dpm_check_envelope), so every
// partial sum is below 2^126 and arithmetic mod 2^128 is exact.
#include <mutex>
#include "dpm_common.cuh"

namespace dpm {

constexpr int M2_THREADS = 128;
constexpr int M2_CHUNK = 8;   // moments per stage-2 reduction round (4 * M2_CHUNK == M2_THREADS / 4)

template <int JB> struct Limbs {
  __host__ __device__ static constexpr int nl(int q) { return q == 0 ? 1 : (q * JB + 23) / 24; }
  __host__ __device__ static constexpr int off(int q) { int s = 0; for (int a = 0; a < q; ++a) s += nl(a); return s; }
};

struct M2Params {
  ImageSet s;
  int64_t B;
  int64_t rc;                              // rows per chunk (<= 256)
  int64_t blocks_img[DPM_MAX_IMAGES + 1];  // prefix sums of blocks per image (per volume)
  int64_t cblocks[DPM_MAX_IMAGES];         // column blocks per image
  uint64_t* acc;                           // [B][n_img][n2][4]
};

template <int K, int JB>
__global__ void __launch_bounds__(M2_THREADS) moments2d_kernel(M2Params p) {
  using LP = Limbs<JB>;
  constexpr int NT = LP::off(K + 1);        // total limbs across q = 0..K
  constexpr int NTP = (NT + 3) & ~3;        // padded to uint4
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  // table (stage 1) and red (stage 2) are live in disjoint phases: one buffer
  extern __shared__ __align__(16) uint32_t m2_smem[];
  uint32_t (*table)[NTP] = reinterpret_cast<uint32_t (*)[NTP]>(m2_smem);
  uint32_t (*red)[M2_THREADS + 1] = reinterpret_cast<uint32_t (*)[M2_THREADS + 1]>(m2_smem);

  const int64_t per_vol = p.blocks_img[p.s.n_img];
  const int64_t b = blockIdx.x / per_vol;
  int64_t r = blockIdx.x - b * per_vol;
  int k = 0;
  while (r >= p.blocks_img[k + 1]) ++k;
  r -= p.blocks_img[k];
  const int64_t rb = r / p.cblocks[k], cb = r - rb * p.cblocks[k];
  const int64_t W = p.s.W[k], H = p.s.H[k], ai = p.s.ai[k], aj = p.s.aj[k];
  const int64_t j0 = rb * p.rc;
  const int rows = (int)imin64(p.rc, H - j0);
  const int tid = threadIdx.x;

  // row-power limb table: (j + aj)^q as 24-bit limbs
  for (int rr = tid; rr < rows; rr += M2_THREADS) {
    const unsigned __int128 y = (unsigned __int128)(uint64_t)(j0 + rr + aj);
    unsigned __int128 pw = 1;
    #pragma unroll
    for (int q = 0; q <= K; ++q) {
      unsigned __int128 t = pw;
      #pragma unroll
      for (int l = 0; l < LP::nl(q); ++l) { table[rr][LP::off(q) + l] = (uint32_t)(t & 0xFFFFFFu); t >>= 24; }
      pw *= y;
    }
    #pragma unroll
    for (int l = NT; l < NTP; ++l) table[rr][l] = 0;
  }
  __syncthreads();

  const int64_t i = cb * M2_THREADS + tid;
  uint64_t acc[NTP];
  #pragma unroll
  for (int l = 0; l < NTP; ++l) acc[l] = 0;
  if (i < W) {
    const uint32_t* col = p.s.img[k] + b * W * H + j0 * W + i;
    #pragma unroll 4
    for (int rr = 0; rr < rows; ++rr) {
      const uint64_t v = __ldg(col + (int64_t)rr * W);
      const uint4* tr = reinterpret_cast<const uint4*>(&table[rr][0]);
      #pragma unroll
      for (int l4 = 0; l4 < NTP / 4; ++l4) {
        const uint4 t = tr[l4];
        acc[4 * l4 + 0] += v * t.x;
        acc[4 * l4 + 1] += v * t.y;
        acc[4 * l4 + 2] += v * t.z;
        acc[4 * l4 + 3] += v * t.w;
      }
    }
  }

  __syncthreads();  // table dead from here on; its storage becomes red
  // stage 2: C_q (mod 2^128) times (i + ai)^p, p + q <= K, reduced over the
  // CTA's columns M2_CHUNK moments at a time (keeps the shared buffer small,
  // so occupancy is set by the 16 KB row table, not by the reduction)
  unsigned __int128 C[K + 1];
  #pragma unroll
  for (int q = 0; q <= K; ++q) {
    unsigned __int128 c = 0;
    #pragma unroll
    for (int l = 0; l < LP::nl(q); ++l) c += ((unsigned __int128)acc[LP::off(q) + l]) << (24 * l);
    C[q] = (i < W) ? c : 0;
  }
  unsigned __int128 xp[K + 1];
  {
    const __int128 x = (__int128)(i + ai);
    __int128 t = 1;
    #pragma unroll
    for (int pp = 0; pp <= K; ++pp) { xp[pp] = (unsigned __int128)t; t *= x; }
  }
  uint64_t* out = p.acc + ((b * p.s.n_img + k) * N2) * 4;
  #pragma unroll
  for (int m0 = 0; m0 < N2; m0 += M2_CHUNK) {
    int m = 0;
    #pragma unroll
    for (int pp = 0; pp <= K; ++pp) {
      #pragma unroll
      for (int q = 0; q <= K - pp; ++q, ++m) {
        if (m < m0 || m >= m0 + M2_CHUNK) continue;
        const unsigned __int128 v = C[q] * xp[pp];
        const int e = m - m0;
        red[4 * e + 0][tid] = (uint32_t)v;
        red[4 * e + 1][tid] = (uint32_t)(v >> 32);
        red[4 * e + 2][tid] = (uint32_t)(v >> 64);
        red[4 * e + 3][tid] = (uint32_t)(v >> 96);
      }
    }
    __syncthreads();
    // 4 threads per limb row: 32 columns each, then a 4-lane shuffle sum
    {
      const int e = tid >> 2, part = tid & 3;
      uint64_t sum = 0;
      if (e < 4 * M2_CHUNK) {
        #pragma unroll 8
        for (int t = part * 32; t < part * 32 + 32; ++t) sum += red[e][t];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      const int gm = m0 + (e >> 2);
      if (part == 0 && e < 4 * M2_CHUNK && gm < N2 && sum)
        atomicAdd(reinterpret_cast<unsigned long long*>(out + 4 * m0 + e), (unsigned long long)sum);
    }
    __syncthreads();
  }
}

template <int K, int JB>
static void launch_kj(dim3 grid, cudaStream_t st, const M2Params& p) {
  constexpr int NT = Limbs<JB>::off(K + 1);
  constexpr int NTP = (NT + 3) & ~3;
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  constexpr size_t t_bytes = 256 * NTP * 4, r_bytes = (size_t)M2_CHUNK * 4 * (M2_THREADS + 1) * 4;
  constexpr size_t bytes = t_bytes > r_bytes ? t_bytes : r_bytes;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(moments2d_kernel<K, JB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  });
  moments2d_kernel<K, JB><<<grid, M2_THREADS, bytes, st>>>(p);
}

template <int K>
static void launch_k(int jb, dim3 grid, cudaStream_t st, const M2Params& p) {
  if (jb <= 12) launch_kj<K, 12>(grid, st, p);
  else if (jb <= 16) launch_kj<K, 16>(grid, st, p);
  else launch_kj<K, 21>(grid, st, p);
}

int launch_moments2d(const ImageSet& s, int64_t B, int order, int jbits, uint64_t* acc, cudaStream_t st) {
  M2Params p;
  p.s = s; p.B = B; p.acc = acc;
  // rows per chunk: the largest of 256/128/64 that still gives >= 8 CTAs per SM
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.rc = 64;
  for (int64_t rc = 256; rc >= 128; rc >>= 1) {
    int64_t nb = 0;
    for (int k = 0; k < s.n_img; ++k) nb += ((s.W[k] + M2_THREADS - 1) / M2_THREADS) * ((s.H[k] + rc - 1) / rc);
    if (nb * B >= 8 * (int64_t)sms) { p.rc = rc; break; }
  }
  p.blocks_img[0] = 0;
  for (int k = 0; k < s.n_img; ++k) {
    p.cblocks[k] = (s.W[k] + M2_THREADS - 1) / M2_THREADS;
    const int64_t rblocks = (s.H[k] + p.rc - 1) / p.rc;
    p.blocks_img[k + 1] = p.blocks_img[k] + p.cblocks[k] * rblocks;
  }
  for (int k = s.n_img + 1; k <= DPM_MAX_IMAGES; ++k) p.blocks_img[k] = p.blocks_img[s.n_img];
  const int64_t nblocks = p.blocks_img[s.n_img] * B;
  if (nblocks == 0) return DPM_OK;
  if (nblocks > 0x7fffffffLL) return DPM_EINVAL;
  dim3 grid((unsigned)nblocks);
  switch (order) {
    case 3: launch_k<3>(jbits, grid, st, p); break;
    case 4: launch_k<4>(jbits, grid, st, p); break;
    case 5: launch_k<5>(jbits, grid, st, p); break;
    default: launch_k<6>(jbits, grid, st, p); break;
  }
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

// 1D exact moments of the y-summed profile (moments pipeline, DPM_ACC_PROFILE):
//   M_a = sum_i P[i] (i + ai)^a,  a = 0..K,
// into the q = 0 entries of accumulator slot `slot` ([B][n_img][n2d][4] limb
// sums, zeroed by the caller).  Each term is formed mod 2^128 and split into
// four 32-bit limbs summed in uint64, as in moments2d_kernel.
constexpr int PM_THREADS = 256;

template <int K>
__global__ void __launch_bounds__(PM_THREADS) profile_moments_kernel(const unsigned long long* prof, int64_t WQ,
                                                                    int64_t B, int64_t ai, int n_img, int slot,
                                                                    uint64_t* acc) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  for (int64_t b = blockIdx.y; b < B; b += gridDim.y) {
  uint64_t l[K + 1][4];
  #pragma unroll
  for (int a = 0; a <= K; ++a) { l[a][0] = l[a][1] = l[a][2] = l[a][3] = 0; }
  for (int64_t i = (int64_t)blockIdx.x * PM_THREADS + threadIdx.x; i < WQ; i += (int64_t)gridDim.x * PM_THREADS) {
    const unsigned long long v = prof[b * WQ + i];
    if (v == 0) continue;
    const __int128 x = (__int128)(i + ai);
    __int128 pw = 1;
    #pragma unroll
    for (int a = 0; a <= K; ++a) {
      const unsigned __int128 t = (unsigned __int128)v * (unsigned __int128)pw;
      l[a][0] += (uint32_t)t;
      l[a][1] += (uint32_t)(t >> 32);
      l[a][2] += (uint32_t)(t >> 64);
      l[a][3] += (uint32_t)(t >> 96);
      pw *= x;
    }
  }
  uint64_t* out = acc + ((b * n_img + slot) * N2) * 4;
  #pragma unroll
  for (int a = 0; a <= K; ++a) {
    #pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint64_t v = l[a][k];
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(out + idx2(K, a, 0) * 4 + k),
                                                  (unsigned long long)v);
    }
  }
  }
}

int launch_profile_moments(const unsigned long long* prof, int64_t WQ, int64_t B, int64_t ai, int order, int n_img,
                           int slot, uint64_t* acc, cudaStream_t st) {
  const unsigned gx = (unsigned)imin64((WQ + PM_THREADS - 1) / PM_THREADS, 64);
  const dim3 grid(gx, (unsigned)imin64(B, 65535));
  switch (order) {
    case 3: profile_moments_kernel<3><<<grid, PM_THREADS, 0, st>>>(prof, WQ, B, ai, n_img, slot, acc); break;
    case 4: profile_moments_kernel<4><<<grid, PM_THREADS, 0, st>>>(prof, WQ, B, ai, n_img, slot, acc); break;
    case 5: profile_moments_kernel<5><<<grid, PM_THREADS, 0, st>>>(prof, WQ, B, ai, n_img, slot, acc); break;
    default: profile_moments_kernel<6><<<grid, PM_THREADS, 0, st>>>(prof, WQ, B, ai, n_img, slot, acc); break;
  }
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
