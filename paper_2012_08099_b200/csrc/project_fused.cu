// project_fused.cu -- the whole moments pipeline of small uint8 volumes in ONE
// launch: projection pass, 2D / 1D moments and the 3D epilogue.
//
// Replaces, per volume, projection._accumulate (projection.py:139-186) +
// drt2d.integrals/assemble_2d/shift_origin (drt2d.py:92-208) + moments3d._place /
// _cross_axis_moments (moments3d.py:201-229), for order 3 (the reference's
// default, moments3d.py:232-264) on volumes of at most 128 x M x 128 uint8
// voxels -- BASELINE configs 1 (64^3) and 4 (1024 x 128^3).
//
// Why a separate kernel: for such volumes one row-step (one y, every x and z)
// completes an image row of XY and of DIAG and a column of YZ, so the rows never
// need to exist in HBM.  The streaming pass would store them (single-tile mode)
// and a second launch would read them back: 1.31x the algorithmic DRAM bytes
// and a moments launch that is 13 % of the cfg4 step.  Here each completed row
// is folded straight into per-thread y-power accumulators, and the volume's
// moments are reduced, added to its limb accumulator, and -- by the last CTA to
// finish the volume -- turned into the 3D moments (derive_volume, the K3 code).
//
// Packed bytes (SWAR).  A lane owns 4 consecutive x of a plane row (one 32-bit
// word).  Two PRMTs split the word into e = (x0, x2) and o = (x1, x3) as two
// 16-bit fields, and every sum below adds two voxels per 32-bit add:
//   XY   (x, y)     e, o summed over the warp's planes (fields <= 128*255)
//   DIAG (x + z, y) the word of plane t and the odd half of plane t-1 cover the
//                   same cell pair (c, c+2): ONE add per plane and one
//                   red.shared into a packed CTA row (two rows A/B so that no
//                   two pairs share a word; immediate offsets, conflict-free)
//   prof (x - z, summed over y)  a packed register window, e of plane t and o
//                   of plane t+1 share a cell pair: one 3-input add per plane;
//                   flushed to a CTA row every 128 rows (fields <= 128*2*255)
//   YZ   (y, z)     byte sums of two planes packed by IDP (FMA pipe), one
//                   REDUX per two planes
// so a voxel costs ~1.1 ALU ops instead of ~2.8 unpacked.
//
// Row reduction (per row-step, after the CTA barrier): thread j owns XY cell
// x = j, DIAG cells g = j (+128) and YZ plane z = j, and accumulates
//   T_q[x] += XY[y][x] y^q,  D_q[g] += DIAG[y][g] y^q,  S_p[z] += YZ[z][y] y^p
// (IMAD.WIDE, exact in uint64 for M <= 1024).  At the end of the CTA's run
// through a volume: M_pq = sum x^p T_q (and likewise), each thread's 128-bit
// partial split into 16-bit pieces, reduced per warp by REDUX (exact: 32 x
// 2^16 < 2^21), summed over the warps, and added into the volume's limb
// accumulator [4 images][n2d][4 x uint64] (the moments2d format, so the
// epilogue is unchanged).  A per-volume counter of finished rows elects the CTA
// that runs the epilogue.
//
// Exactness: integer sums throughout; the 16-bit fields never carry (bounds
// above), the uint64 accumulators stay below 2^56 (checked by the eligibility
// rule), and the 128-bit moments are formed mod 2^128 like moments2d's.
#include <cudaTypedefs.h>
#include "derive_dev.cuh"
#include "ptx.cuh"

namespace dpm {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();   // project_stream.cu

namespace fb {
constexpr int X = 128, Z = 128;           // the tile is the whole volume: L <= 128, N <= 128
constexpr int K = 3;
constexpr int N2 = (K + 1) * (K + 2) / 2;  // 10
constexpr int NIMG = 4;                    // XY, YZ, (profile in the ZX slot), DIAG
constexpr int NMOM = 3 * N2 + (K + 1);     // XY, YZ, DIAG 2D moments + the profile's 1D moments
constexpr int PIECES = 8;                  // 16-bit pieces of a 128-bit value
constexpr int ROWW = 384;                  // row buffer: XY [0,128) | DIAG A [128,256) | DIAG B [256,384)
constexpr int PROFW = 256;                 // profile row (L + N - 1 <= 255 cells)
constexpr int MAXM = 1024;                 // y^3 < 2^30, accumulators < 2^56

template <int NW> struct Geo {
  static constexpr int THREADS = 32 * NW;
  static constexpr int ZP = Z / NW;        // planes per warp
  static constexpr int CTAS = 16 / NW;     // CTAs per SM
  static constexpr int STAGE = X * Z;      // bytes per row-step
  static constexpr int NPQ = ZP + 1;       // packed profile cell pairs per lane
  static constexpr int NDG = 256 / THREADS;   // DIAG cells per thread
  static constexpr int REDW = NW * NMOM * PIECES;
  static constexpr int FIXED = 3 * ROWW * 4 + PROFW * 4 + REDW * 4 + NIMG * N2 * 4 * 8 + 256;
  static constexpr int BUDGET = (CTAS == 1 ? 220 : 224 / CTAS) * 1024;
  static constexpr int FIT = (BUDGET - FIXED) / STAGE;
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + FIXED;
};
}  // namespace fb

struct FBParams {
  int32_t L, M, N;
  int64_t B, total;        // volumes, row-steps (B * M)
  uint64_t* acc;           // [B][4][10][4]
  unsigned int* cnt;       // [B] finished rows per volume
  int64_t* out_i128;
  double* out_f64;
  int32_t* status;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
  return d;
}

// word (in the row buffer) of the packed DIAG pair with base cell g = 4a + m
__host__ __device__ constexpr int diag_word(int m, int a) { return (m >= 2 ? 256 : 128) + 64 * (m & 1) + a; }

template <int NW>
__global__ void __launch_bounds__(32 * NW, 16 / NW) fused_batch_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                      const FBParams p) {
  using G = fb::Geo<NW>;
  constexpr int ZP = G::ZP, S = G::STAGES, T = G::THREADS, NPQ = G::NPQ, NDG = G::NDG;
  constexpr int N2 = fb::N2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* rows = reinterpret_cast<uint32_t*>(smem + (size_t)S * G::STAGE);   // [3][ROWW]
  uint32_t* prow = rows + 3 * fb::ROWW;                                         // [PROFW]
  uint32_t* red = prow + fb::PROFW;                                             // [NW][NMOM][PIECES]
  uint64_t* sa = reinterpret_cast<uint64_t*>(red + G::REDW);                    // epilogue staging
  uint64_t* full = sa + fb::NIMG * N2 * 4;                                      // [S]
  int32_t* flags = reinterpret_cast<int32_t*>(full + S);                        // [0] last, [1] epilogue status
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  const int64_t r0 = p.total * blockIdx.x / gridDim.x, r1 = p.total * (blockIdx.x + 1) / gridDim.x;
  if (r0 >= r1) return;
  for (int i = tid; i < 3 * fb::ROWW + fb::PROFW; i += T) rows[i] = 0;
  // refill cursor (thread 0): the next row to fetch, advanced row by row -- no
  // division in the row loop (a 64-bit division is a call, and a call site in
  // the loop costs every thread registers)
  int32_t ib = (int32_t)(r0 / p.M);
  int32_t iy = (int32_t)(r0 - (int64_t)ib * p.M);
  auto issue = [&](int k) {
    ptx::mbar_arrive_expect_tx(&full[k], G::STAGE);
    ptx::tma_load_4d_hint(stages + (size_t)k * G::STAGE, &tmap, &full[k], 0, iy, 0, ib, ptx::policy_evict_first());
    if (++iy == (int32_t)p.M) { iy = 0; ++ib; }
  };
  if (tid == 0) {
    ptx::prefetch_tmap(&tmap);
    for (int i = 0; i < S; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
    for (int h = 0; h < S && r0 + h < r1; ++h) issue(h);
  }
  __syncthreads();

  // ---- per-thread ownership (fixed for the whole run) ----
  const uint32_t rows_a = ptx::smem_addr(rows), prow_a = ptx::smem_addr(prow);
  const uint32_t stage_a = ptx::smem_addr(stages) + (uint32_t)(ZP * w * fb::X + 4 * lane);
  // DIAG emission: pair base g = 4 lane + ZP w + t -> word diag_word(t % 4, lane + ZP w / 4 + t / 4)
  const uint32_t dlane = 4u * (uint32_t)(lane + ZP * w / 4);
  // profile window: packed pair c covers global cells base + c and base + c + 2,
  // global index x - z + (N - 1); base = 4 lane - ZP w + N - ZP
  const int32_t pbase = 4 * lane - ZP * w + p.N - ZP;
  // XY cell x = tid: word (x & 1) * 64 + x / 4, field (x & 2) ? hi : lo
  const bool own_xy = tid < fb::X && tid < p.L;
  const uint32_t xy_w = 4u * (uint32_t)((tid & 1) * 64 + (tid >> 2));
  const uint32_t xy_sh = (tid & 2) ? 16u : 0u;
  // DIAG cells g = tid + T c: lo field of the pair based at g, hi field of the pair based at g - 2
  uint32_t dg_lo[NDG], dg_hi[NDG];
  bool dg_hi_ok[NDG];
  #pragma unroll
  for (int c = 0; c < NDG; ++c) {
    const int g = tid + T * c;
    dg_lo[c] = 4u * (uint32_t)diag_word(g & 3, g >> 2);
    dg_hi_ok[c] = g >= 2;
    dg_hi[c] = g >= 2 ? 4u * (uint32_t)diag_word((g - 2) & 3, (g - 2) >> 2) : 0u;
  }
  const bool own_yz = lane < ZP;   // plane z = ZP w + lane

  uint32_t PQ[NPQ];
  #pragma unroll
  for (int c = 0; c < NPQ; ++c) PQ[c] = 0;
  uint64_t Txy[4], Dg[NDG][4], Syz[4];
  auto zero_acc = [&]() {
    #pragma unroll
    for (int q = 0; q < 4; ++q) {
      Txy[q] = 0; Syz[q] = 0;
      #pragma unroll
      for (int c = 0; c < NDG; ++c) Dg[c][q] = 0;
    }
  };
  zero_acc();

  // packed profile registers -> CTA profile row (u32 cells)
  auto flush_pq = [&]() {
    #pragma unroll
    for (int c = 0; c < NPQ; ++c) {
      const uint32_t v = PQ[c];
      PQ[c] = 0;
      if (v == 0) continue;
      const int32_t i = pbase + c;
      if ((v & 0xFFFFu) && i >= 0 && i < fb::PROFW) ptx::red_shared_add_dyn(prow_a + 4u * (uint32_t)i, v & 0xFFFFu);
      if ((v >> 16) && i + 2 >= 0 && i + 2 < fb::PROFW) ptx::red_shared_add_dyn(prow_a + 4u * (uint32_t)(i + 2), v >> 16);
    }
  };

  // end of this CTA's rows of volume vb: partial moments -> limb accumulator;
  // the CTA that completes the volume runs the epilogue
  auto volume_end = [&](int64_t vb, int32_t rows_done) {
    pdl_wait();   // accumulator and counters zeroed by the preceding kernel (no-op after the first volume)
    flush_pq();
    __syncthreads();
    // profile cells of this thread (read and re-zero the CTA row)
    uint32_t pv[NDG];
    #pragma unroll
    for (int c = 0; c < NDG; ++c) {
      const int i = tid + T * c;
      pv[c] = prow[i];
      prow[i] = 0;
    }
    typedef unsigned __int128 u128;
    int m = 0;
    auto reduce_one = [&](u128 v) {   // this thread's 128-bit partial of moment m -> red[w][m][*]
      #pragma unroll
      for (int j = 0; j < fb::PIECES; ++j) {
        const uint32_t piece = (uint32_t)(v >> (16 * j)) & 0xFFFFu;
        const uint32_t s = __reduce_add_sync(0xffffffffu, piece);
        if (lane == 0) red[(w * fb::NMOM + m) * fb::PIECES + j] = s;
      }
      ++m;
    };
    const uint64_t x = (uint64_t)tid;
    // XY: M_pq = sum_x x^p T_q
    #pragma unroll
    for (int pp = 0; pp <= fb::K; ++pp) {
      #pragma unroll
      for (int q = 0; q <= fb::K - pp; ++q) {
        uint64_t xp = 1;
        #pragma unroll
        for (int e = 0; e < pp; ++e) xp *= x;
        reduce_one(own_xy ? (u128)xp * Txy[q] : (u128)0);
      }
    }
    // YZ (stored [z][y]: i = y, j = z): M_pq = sum_z z^q S_p
    const uint64_t z = (uint64_t)(ZP * w + lane);
    #pragma unroll
    for (int pp = 0; pp <= fb::K; ++pp) {
      #pragma unroll
      for (int q = 0; q <= fb::K - pp; ++q) {
        uint64_t zq = 1;
        #pragma unroll
        for (int e = 0; e < q; ++e) zq *= z;
        reduce_one(own_yz ? (u128)zq * Syz[pp] : (u128)0);
      }
    }
    // DIAG: M_pq = sum_g g^p D_q
    #pragma unroll
    for (int pp = 0; pp <= fb::K; ++pp) {
      #pragma unroll
      for (int q = 0; q <= fb::K - pp; ++q) {
        u128 v = 0;
        #pragma unroll
        for (int c = 0; c < NDG; ++c) {
          const uint64_t g = (uint64_t)(tid + T * c);
          uint64_t gp = 1;
          #pragma unroll
          for (int e = 0; e < pp; ++e) gp *= g;
          v += (u128)gp * Dg[c][q];
        }
        reduce_one(v);
      }
    }
    // profile: sum_i P[i] (i - (N - 1))^a  (signed coordinate, two's complement mod 2^128)
    #pragma unroll
    for (int a = 0; a <= fb::K; ++a) {
      u128 v = 0;
      #pragma unroll
      for (int c = 0; c < NDG; ++c) {
        const __int128 xc = (__int128)(tid + T * c) - (__int128)(p.N - 1);
        __int128 t = 1;
        #pragma unroll
        for (int e = 0; e < a; ++e) t *= xc;
        v += (u128)((__int128)pv[c] * t);
      }
      reduce_one(v);
    }
    zero_acc();
    __syncthreads();
    // sum over the warps, add into the volume's limb accumulator
    uint64_t* accb = p.acc + vb * (fb::NIMG * N2 * 4);
    for (int e = tid; e < fb::NMOM * fb::PIECES; e += T) {
      const int mm = e / fb::PIECES, j = e % fb::PIECES;
      uint64_t s = 0;
      #pragma unroll
      for (int ww = 0; ww < NW; ++ww) s += red[(ww * fb::NMOM + mm) * fb::PIECES + j];
      if (s == 0) continue;
      int img, slot;
      if (mm < 3 * N2) {
        img = mm < N2 ? DPM_IMG_XY : mm < 2 * N2 ? DPM_IMG_YZ : DPM_IMG_DIAG;
        slot = mm % N2;   // p-major (p, q) order == idx2
      } else {
        img = DPM_IMG_ZX;
        slot = idx2(fb::K, mm - 3 * N2, 0);
      }
      atomicAdd(reinterpret_cast<unsigned long long*>(accb + (img * N2 + slot) * 4 + j / 2),
                (unsigned long long)(s << (16 * (j & 1))));
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned int old = atomicAdd(p.cnt + vb, (unsigned int)rows_done);
      flags[0] = old + (unsigned int)rows_done == (unsigned int)p.M;
    }
    __syncthreads();
    if (flags[0]) {
      __threadfence();
      derive_volume<fb::K>(accb, vb, fb::NIMG, DPM_ACC_PROFILE, p.out_i128, p.out_f64, p.status, sa, flags + 1, true);
    }
  };

  int64_t b = (int32_t)(r0 / p.M);
  int32_t y = (int32_t)(r0 - b * p.M);
  int32_t seg_rows = 0, pq_rows = 0;
  int k = 0, buf = 0;
  uint32_t ph = 0;
  for (int64_t r = r0; r < r1; ++r) {
    ptx::mbar_wait_addr(ptx::smem_addr(&full[k]), ph);
    const uint32_t ra = rows_a + (uint32_t)(buf * fb::ROWW * 4);
    const uint32_t sa_k = stage_a + (uint32_t)(k * G::STAGE);
    uint32_t cse = 0, cso = 0, yz2 = 0, oprev = 0, eprev = 0;
    #pragma unroll
    for (int t = 0; t < ZP; t += 2) {
      const uint32_t w0 = ptx::lds_u32(sa_k + (uint32_t)(t * fb::X));
      const uint32_t w1 = ptx::lds_u32(sa_k + (uint32_t)((t + 1) * fb::X));
      const uint32_t e0 = prmt(w0, 0x4240u), o0 = prmt(w0, 0x4341u);
      const uint32_t e1 = prmt(w1, 0x4240u), o1 = prmt(w1, 0x4341u);
      // XY: column sums, two voxels per add
      cse = cse + e0 + e1;
      cso = cso + o0 + o1;
      // YZ: byte sums of planes t, t+1 packed in one word, one REDUX; lane t/2 keeps it
      const uint32_t s2 = __dp4a(w0, 0x01010101u, __dp4a(w1, 0x01010101u, 0u) << 16);
      const uint32_t rs = __reduce_add_sync(0xffffffffu, s2);
      yz2 = lane == (t >> 1) ? rs : yz2;
      // DIAG: pair (x+z) based at 4 lane + ZP w + t gets e_t and o_{t-1}
      ptx::red_shared_add_dyn(ra + dlane + 4u * (uint32_t)diag_word(t & 3, t >> 2), e0 + oprev);
      ptx::red_shared_add_dyn(ra + dlane + 4u * (uint32_t)diag_word((t + 1) & 3, (t + 1) >> 2), e1 + o0);
      oprev = o1;
      // profile (x - z): pair c = ZP - 1 - t gets e_t and o_{t+1}
      if (t == 0) PQ[ZP] += o0;
      else PQ[ZP - t] = PQ[ZP - t] + eprev + o0;   // e_{t-1} + o_t
      PQ[ZP - 1 - t] = PQ[ZP - 1 - t] + e0 + o1;
      eprev = e1;
    }
    PQ[0] += eprev;
    ptx::red_shared_add_dyn(ra + dlane + 4u * (uint32_t)diag_word(ZP & 3, ZP >> 2), oprev);
    ptx::red_shared_add_dyn(ra + 4u * (uint32_t)lane, cse);
    ptx::red_shared_add_dyn(ra + 4u * (uint32_t)(64 + lane), cso);
    // plane ZP w + lane's sum: lane's pair sits with lane / 2
    const uint32_t yzp = __shfl_sync(0xffffffffu, yz2, lane >> 1);
    const uint32_t yzv = (lane & 1) ? (yzp >> 16) : (yzp & 0xFFFFu);
    __syncthreads();
    if (tid == 0 && r + S < r1) issue(k);
    if (++k == S) { k = 0; ph ^= 1u; }

    // ---- fold the completed rows of this row-step into the y-power accumulators ----
    const uint32_t y1 = (uint32_t)y, y2 = y1 * y1, y3 = y2 * y1;
    const uint32_t* rw = rows + buf * fb::ROWW;
    if (own_xy) {
      const uint32_t v = (rw[xy_w / 4] >> xy_sh) & 0xFFFFu;
      Txy[0] += v;
      Txy[1] += (uint64_t)v * y1;
      Txy[2] += (uint64_t)v * y2;
      Txy[3] += (uint64_t)v * y3;
    }
    #pragma unroll
    for (int c = 0; c < NDG; ++c) {
      const uint32_t v = (rw[dg_lo[c] / 4] & 0xFFFFu) + (dg_hi_ok[c] ? (rw[dg_hi[c] / 4] >> 16) : 0u);
      Dg[c][0] += v;
      Dg[c][1] += (uint64_t)v * y1;
      Dg[c][2] += (uint64_t)v * y2;
      Dg[c][3] += (uint64_t)v * y3;
    }
    if (own_yz) {
      Syz[0] += yzv;
      Syz[1] += (uint64_t)yzv * y1;
      Syz[2] += (uint64_t)yzv * y2;
      Syz[3] += (uint64_t)yzv * y3;
    }
    // zero the buffer read in the previous row-step (next written two row-steps on)
    {
      uint32_t* zb = rows + (buf == 0 ? 2 : buf - 1) * fb::ROWW;
      for (int i = tid; i < fb::ROWW; i += T) zb[i] = 0;
    }
    buf = buf == 2 ? 0 : buf + 1;
    ++seg_rows;
    if (++pq_rows == 128) { flush_pq(); pq_rows = 0; }   // 16-bit fields: <= 128 rows x 510
    if (++y == p.M || r + 1 == r1) {
      volume_end(b, seg_rows);
      ++b;
      y = 0;
      seg_rows = 0;
      pq_rows = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

#ifndef DPM_FB_NW
#define DPM_FB_NW 4   // warps per CTA (4: 32 planes per warp, 4 CTAs per SM; 8: 16 planes, 2 CTAs)
#endif

bool fused_batch_eligible(const dpm_volume_desc* d, const void* vox, int order) {
  if (order != fb::K || d->dtype != DPM_U8 || d->offset != 0 || d->z0 != 0) return false;
  if (d->L < 4 || d->L > fb::X || d->L % 4 || d->N < 1 || d->N > fb::Z || d->M < 1 || d->M > fb::MAXM) return false;
  if (d->stride_y % 16 || d->stride_z % 16 || (d->B > 1 && d->stride_b % 16)) return false;
  if (reinterpret_cast<uintptr_t>(vox) % 16) return false;
  if (d->B > 0x7fffffffLL) return false;
  return tensor_map_encoder() != nullptr;
}

template <int NW>
static int launch_fb(const dpm_volume_desc* d, const void* vox, const FBParams& p, int sms, cudaStream_t st) {
  using G = fb::Geo<NW>;
  static_assert(G::STAGES >= 2, "at least two stages");
  static_assert(G::SMEM <= (G::CTAS == 1 ? 227 : 227 / G::CTAS) * 1024, "shared memory budget");
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)d->L, (cuuint64_t)d->M, (cuuint64_t)d->N, (cuuint64_t)d->B};
  const cuuint64_t strides[3] = {(cuuint64_t)d->stride_y, (cuuint64_t)d->stride_z,
                                 (cuuint64_t)(d->B > 1 ? d->stride_b : d->stride_z * d->N)};
  const cuuint32_t box[4] = {(cuuint32_t)fb::X, 1, (cuuint32_t)fb::Z, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(vox), dims, strides,
                                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;
  static std::atomic<uint64_t> attr_mask{0};
  if (ensure_smem(fused_batch_kernel<NW>, G::SMEM, attr_mask)) return DPM_ECUDA;
  const int grid = (int)imin64((int64_t)sms * G::CTAS, p.total);
  if (launch_pdl(fused_batch_kernel<NW>, dim3(grid), dim3(G::THREADS), G::SMEM, st, map, p) != cudaSuccess)
    return DPM_ECUDA;
  return DPM_OK;
}

// one-launch moments pass (order 3, uint8, x and z extents <= 128).  The caller
// zeroed acc [B][4][10][4] and cnt [B]; *handled = false leaves it to the
// streaming pipeline.
int launch_fused_batch(const dpm_volume_desc* d, const void* vox, int order, uint64_t* acc, unsigned int* cnt,
                       int64_t* out_i128, double* out_f64, int32_t* status, cudaStream_t st, bool* handled) {
  *handled = false;
  if (!fused_batch_eligible(d, vox, order)) return DPM_OK;
  FBParams p;
  p.L = (int32_t)d->L; p.M = (int32_t)d->M; p.N = (int32_t)d->N;
  p.B = d->B;
  p.total = d->B * d->M;
  p.acc = acc; p.cnt = cnt;
  p.out_i128 = out_i128; p.out_f64 = out_f64; p.status = status;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int rc = DPM_FB_NW == 8 ? launch_fb<8>(d, vox, p, sms, st) : launch_fb<4>(d, vox, p, sms, st);
  if (rc < 0) return DPM_OK;
  if (rc) return rc;
  note_launches(1);
  *handled = true;
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
