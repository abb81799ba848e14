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
#include "derive_dev.cuh"

namespace dpm {

constexpr int M2_THREADS = 128;
constexpr int M2_CHUNK = 8;   // moments per stage-2 reduction round (4 * M2_CHUNK == M2_THREADS / 4)
#ifndef DPM_M2_UNROLL
#define DPM_M2_UNROLL 16
#endif
constexpr int M2_UNROLL = DPM_M2_UNROLL;   // pixel loads in flight per thread (stage 1)

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
  // moments pipeline: the profile's 1D moments in the same launch (pblocks
  // extra blocks per volume, into the q = 0 entries of slot DPM_IMG_ZX)
  const unsigned long long* prof;          // [B][WQ] or null
  int sgn;                                 // signed-exact int16: int32 pixels, int64 profile cells
  OffsetBox box;                           // offset x box moments added by the epilogue (sgn only)
  int64_t WQ, prof_ai, pblocks;
  // fused epilogue: the last block of each volume (counter cnt[b], zeroed by
  // the caller) runs derive_volume for it; null out_i128 = separate derive3d
  unsigned int* cnt;
  int64_t* out_i128;
  double* out_f64;
  int32_t* status;
  int kind;
};

// one block's share of the profile's 1D moments (cells chunk, chunk + pblocks, ...)
template <int K>
__device__ __forceinline__ void profile_block(const M2Params& p, int64_t b, int64_t chunk, int tid) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  uint64_t l[K + 1][4];
  #pragma unroll
  for (int a = 0; a <= K; ++a) { l[a][0] = l[a][1] = l[a][2] = l[a][3] = 0; }
  for (int64_t i = chunk * M2_THREADS + tid; i < p.WQ; i += p.pblocks * M2_THREADS) {
    const unsigned long long v = p.prof[b * p.WQ + i];
    if (v == 0) continue;
    const __int128 x = (__int128)(i + p.prof_ai);
    __int128 pw = 1;
    // signed cells (sgn): the uint64 is a two's-complement int64
    const unsigned __int128 vv = p.sgn ? (unsigned __int128)(__int128)(long long)v : (unsigned __int128)v;
    #pragma unroll
    for (int a = 0; a <= K; ++a) {
      const unsigned __int128 t = vv * (unsigned __int128)pw;
      l[a][0] += (uint32_t)t;
      l[a][1] += (uint32_t)(t >> 32);
      l[a][2] += (uint32_t)(t >> 64);
      l[a][3] += (uint32_t)(t >> 96);
      pw *= x;
    }
  }
  uint64_t* out = p.acc + ((b * p.s.n_img + DPM_IMG_ZX) * N2) * 4;
  #pragma unroll
  for (int a = 0; a <= K; ++a) {
    #pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint64_t v = l[a][q];
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(out + idx2(K, a, 0) * 4 + q),
                                          (unsigned long long)v);
    }
  }
}

#ifdef DPM_M2_MINB
#define DPM_M2_BOUNDS __launch_bounds__(M2_THREADS, DPM_M2_MINB)   // register cap for A/B builds
#else
#define DPM_M2_BOUNDS __launch_bounds__(M2_THREADS)
#endif
template <int K, int JB>
__global__ void DPM_M2_BOUNDS moments2d_kernel(M2Params p) {
  using LP = Limbs<JB>;
  constexpr int NT = LP::off(K + 1);        // total limbs across q = 0..K
  constexpr int NTP = (NT + 3) & ~3;        // padded to uint4
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  // table (stage 1) and red (stage 2) are live in disjoint phases: one buffer
  extern __shared__ __align__(16) uint32_t m2_smem[];
  uint32_t (*table)[NTP] = reinterpret_cast<uint32_t (*)[NTP]>(m2_smem);
  uint32_t (*red)[M2_THREADS + 1] = reinterpret_cast<uint32_t (*)[M2_THREADS + 1]>(m2_smem);

  const int64_t per_img = p.blocks_img[p.s.n_img];
  const int64_t per_vol = per_img + p.pblocks;
  const int64_t b = blockIdx.x / per_vol;
  int64_t r = blockIdx.x - b * per_vol;
  const int tid = threadIdx.x;
  pdl_trigger();
  if (r >= per_img) {
    pdl_wait();   // the profile is complete once the projection grid is
    profile_block<K>(p, b, r - per_img, tid);
  } else {
  int k = 0;
  while (r >= p.blocks_img[k + 1]) ++k;
  r -= p.blocks_img[k];
  const int64_t rb = r / p.cblocks[k], cb = r - rb * p.cblocks[k];
  const int64_t W = p.s.W[k], H = p.s.H[k], ai = p.s.ai[k], aj = p.s.aj[k];
  const int64_t j0 = rb * p.rc;
  const int rows = (int)imin64(p.rc, H - j0);

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
  pdl_wait();   // images complete (the row-power table above overlapped the projection's tail)

  const int64_t i = cb * M2_THREADS + tid;
  uint64_t acc[NTP];
  #pragma unroll
  for (int l = 0; l < NTP; ++l) acc[l] = 0;
  if (i < W) {
    const uint32_t* col = p.s.img[k] + b * W * H + j0 * W + i;
    // one 32 x 32 -> 64 multiply-add per limb (IMAD.WIDE): the pixel stays a
    // 32-bit operand in both variants (a uint64 pixel times a limb costs three)
    auto column = [&]<bool SGN>() {
      #pragma unroll M2_UNROLL
      for (int rr = 0; rr < rows; ++rr) {
        const uint32_t raw = __ldg(col + (int64_t)rr * W);
        const uint4* tr = reinterpret_cast<const uint4*>(&table[rr][0]);
        #pragma unroll
        for (int l4 = 0; l4 < NTP / 4; ++l4) {
          const uint4 t = tr[l4];
          const uint32_t tl[4] = {t.x, t.y, t.z, t.w};
          #pragma unroll
          for (int e = 0; e < 4; ++e) {
            // signed pixels (sgn): the limb sums stay exact int64 (|v t| < 2^55, 256 rows)
            if constexpr (SGN) acc[4 * l4 + e] += (uint64_t)((int64_t)(int32_t)raw * (int64_t)(int32_t)tl[e]);
            else acc[4 * l4 + e] += (uint64_t)raw * (uint64_t)tl[e];
          }
        }
      }
    };
    if (p.sgn) column.template operator()<true>();
    else column.template operator()<false>();
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
    for (int l = 0; l < LP::nl(q); ++l)
      c += (p.sgn ? (unsigned __int128)(__int128)(int64_t)acc[LP::off(q) + l] : (unsigned __int128)acc[LP::off(q) + l])
           << (24 * l);
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
  }   // image block
  if (p.out_i128) {   // fused epilogue: the volume's last block derives its 3D moments
    __shared__ int last;
    __shared__ int32_t sst;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      last = atomicAdd(p.cnt + b, 1u) == (unsigned)(per_vol - 1);
    }
    __syncthreads();
    if (last) {
      __threadfence();
      derive_volume<K>(p.acc + b * p.s.n_img * N2 * 4, b, p.s.n_img, p.kind, p.out_i128, p.out_f64,
                       p.status, reinterpret_cast<uint64_t*>(m2_smem), &sst, true, p.sgn ? &p.box : nullptr);
    }
  }
}

template <int K, int JB>
static int launch_kj(dim3 grid, cudaStream_t st, const M2Params& p) {
  constexpr int NT = Limbs<JB>::off(K + 1);
  constexpr int NTP = (NT + 3) & ~3;
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  constexpr size_t t_bytes = 256 * NTP * 4, r_bytes = (size_t)M2_CHUNK * 4 * (M2_THREADS + 1) * 4;
  constexpr size_t bytes = t_bytes > r_bytes ? t_bytes : r_bytes;
  static std::atomic<uint64_t> attr_mask{0};
  if (ensure_smem(moments2d_kernel<K, JB>, bytes, attr_mask)) return DPM_ECUDA;
  if (launch_pdl(moments2d_kernel<K, JB>, grid, dim3(M2_THREADS), bytes, st, p) != cudaSuccess) return DPM_ECUDA;
  return DPM_OK;
}

template <int K>
static int launch_k(int jb, dim3 grid, cudaStream_t st, const M2Params& p) {
  if (jb <= 12) return launch_kj<K, 12>(grid, st, p);
  if (jb <= 16) return launch_kj<K, 16>(grid, st, p);
  return launch_kj<K, 21>(grid, st, p);
}

// off * S_e(L), S_e(M), S_e(N), S_e(n) = sum_{k < n} k^e, summed directly mod
// 2^128 (no division, so exact in the ring the epilogue works in; the true
// moments are below 2^126).  The last box is cached per thread: graph capture
// and repeated calls on one geometry pay the O(L + M + N) loop once.
static OffsetBox offset_box(int64_t off, int64_t L, int64_t M, int64_t N) {
  thread_local int64_t key[4] = {-1, -1, -1, -1};
  thread_local OffsetBox cached;
  if (key[0] == off && key[1] == L && key[2] == M && key[3] == N) return cached;
  OffsetBox bx;
  const int64_t dims[3] = {L, M, N};
  for (int a = 0; a < 3; ++a) {
    unsigned __int128 S[DPM_MAX_ORDER + 1] = {};
    for (int64_t k = 0; k < dims[a]; ++k) {
      unsigned __int128 pw = 1;
      for (int e = 0; e <= DPM_MAX_ORDER; ++e) { S[e] += pw; pw *= (unsigned __int128)k; }
    }
    for (int e = 0; e <= DPM_MAX_ORDER; ++e) {
      const unsigned __int128 v = a == 0 ? S[e] * (unsigned __int128)(__int128)off : S[e];
      bx.s[a][e][0] = (int64_t)(uint64_t)v;
      bx.s[a][e][1] = (int64_t)(uint64_t)(v >> 64);
    }
  }
  key[0] = off; key[1] = L; key[2] = M; key[3] = N;
  cached = bx;
  return bx;
}

int launch_moments2d(const ImageSet& s, int64_t B, int order, int jbits, uint64_t* acc, cudaStream_t st,
                     const M2Extra* ex) {
  M2Params p;
  p.s = s; p.B = B; p.acc = acc;
  p.prof = ex ? ex->prof : nullptr;
  p.sgn = ex ? ex->sgn : 0;
  if (p.sgn) p.box = offset_box(ex->off, ex->L, ex->M, ex->N);
  p.WQ = ex ? ex->WQ : 0;
  p.prof_ai = ex ? ex->ai : 0;
  p.pblocks = p.prof ? imin64((p.WQ + M2_THREADS - 1) / M2_THREADS, 16) : 0;
  p.cnt = ex ? ex->cnt : nullptr;
  p.out_i128 = ex ? ex->out_i128 : nullptr;
  p.out_f64 = ex ? ex->out_f64 : nullptr;
  p.status = ex ? ex->status : nullptr;
  p.kind = ex ? ex->kind : DPM_ACC_PROFILE;
  // rows per chunk: the largest of 256/128/64 that still gives >= 8 CTAs per SM
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifndef DPM_M2_TARGET
#define DPM_M2_TARGET 8    // row chunk: the longest that still gives this many CTAs per SM
#endif
#ifndef DPM_M2_MIN_RC
#define DPM_M2_MIN_RC 16   // small images: shorter row chunks, more CTAs in flight (cfg1 graph 22.9 -> 18.8 us)
#endif
  p.rc = DPM_M2_MIN_RC;
  for (int64_t rc = 256; rc > DPM_M2_MIN_RC; rc >>= 1) {
    int64_t nb = 0;
    for (int k = 0; k < s.n_img; ++k) nb += ((s.W[k] + M2_THREADS - 1) / M2_THREADS) * ((s.H[k] + rc - 1) / rc);
    if (nb * B >= DPM_M2_TARGET * (int64_t)sms) { p.rc = rc; break; }
  }
  p.blocks_img[0] = 0;
  for (int k = 0; k < s.n_img; ++k) {
    p.cblocks[k] = (s.W[k] + M2_THREADS - 1) / M2_THREADS;
    const int64_t rblocks = (s.H[k] + p.rc - 1) / p.rc;
    p.blocks_img[k + 1] = p.blocks_img[k] + p.cblocks[k] * rblocks;
  }
  for (int k = s.n_img + 1; k <= DPM_MAX_IMAGES; ++k) p.blocks_img[k] = p.blocks_img[s.n_img];
  const int64_t nblocks = (p.blocks_img[s.n_img] + p.pblocks) * B;
  if (nblocks == 0) return DPM_OK;
  if (nblocks > 0x7fffffffLL) return DPM_EINVAL;
  dim3 grid((unsigned)nblocks);
  int rc;
  switch (order) {
    case 3: rc = launch_k<3>(jbits, grid, st, p); break;
    case 4: rc = launch_k<4>(jbits, grid, st, p); break;
    case 5: rc = launch_k<5>(jbits, grid, st, p); break;
    default: rc = launch_k<6>(jbits, grid, st, p); break;
  }
  if (rc) return rc;
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
