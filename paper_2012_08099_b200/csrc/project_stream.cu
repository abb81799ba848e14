// project_stream.cu -- the streaming projection pass (one read of every voxel).
//
// Replaces projection._accumulate (projection.py:139-186), which sweeps the
// volume at least four times (three numpy reductions plus a chunked shear
// copy), with a single pass that builds all P images at once (the paper's
// Listing 1).
//
// Decomposition ("K1 project_stream"):
//   column   = (volume b, x-tile of SX = 32*VX voxels, z-tile of SZ = 8*NW planes)
//   row-step = one y of one column: an SX (x) x SZ (z) slice of plane-rows,
//              fetched by ONE 4-D TMA box (x SX, y 1, z SZ, b 1) into a
//              shared-memory stage of a STAGES-deep mbarrier pipeline (zero
//              fill out of bounds; L2 evict_first so the stream does not evict
//              the image rows being reduced into).
//   CTA      = NW warps, warp w owns planes Z0+8w..+7, lane l owns x = X0+VX*l..+VX-1:
//              each lane reduces a VX (x) x 8 (z) patch per row-step (VX = 8, or
//              4 for narrow volumes such as the 128^3 batch).  NW = 12 (3 warps
//              per scheduler, <= 168 registers; 16 for 4-wide lanes at order 3).
//              The TMA producer is lane 0 of warp NW/2 (the row flush lands on
//              warps 0-3).
//   Two modes (template PROF):
//   PROF = 0 (dpm_project: the reference's images)
//     ZX (x,z) sum over y: 8*VX registers per lane, persistent across the
//             row-steps of a column (adds on the FMA pipe), flushed at the end
//             of the CTA's run through the column: an 8x8 shfl.xor transpose
//             per 8-lane group makes every red.global cover 32-byte runs of z.
//             At order 6 the (x +- 2z) images are folded in a second pass over
//             the same stage to stay within the register budget.
//   PROF = 1 (the moments pipeline)
//     no ZX; the profile P[x + t z] = sum_y V (t = -1, 2, -2, 3 at 4..7 images)
//             is a VX + 7|t| register window folded with IMAD-by-1 (FMA pipe),
//             summed over the rows of a column run, then added to a CTA shared
//             row (conflict-free transposed layout) and to the uint64 global
//             profile with one coalesced pass of atomics per column and y-band.
//             Order 6 runs in one pass.
//   XY and the oblique images (x + t z, y), t = 1, -1, 2, -2: plane pairs are
//             folded into VX / VX+7 / VX+14-cell register windows with 3-input
//             adds, and every lane adds its WHOLE window to the CTA row with
//             red.shared.  Rows are stored transposed (cell i at
//             (i%VX)*S + i/VX, S = 32/VX mod 32), so window cell c of the 32
//             lanes is 32 consecutive words: conflict-free, and the overlaps
//             between neighbouring lanes (and the tile halo) are resolved by
//             the atomics themselves.  After one __syncthreads per row-step the
//             rows are flushed to global memory (LDS.128 + coalesced red.global)
//             and re-zeroed; rows are double-buffered.
//   YZ (y,z)  per-plane lane sums, one warp redux per plane inside the fold
//             loop, one red.global per (z,y) (orders <= 5: staged per 8
//             consecutive y in shared memory, flushed coalesced).
// Work split: row-steps are grouped into y-bands sized so a band's image rows
// stay L2-resident; within a band the (column, y) sequence is cut into equal
// contiguous runs, one per persistent CTA, iterated as runs of consecutive
// rows of one column.
// Exactness: uint32 ray sums (the C ABI rejects shapes whose longest ray could
// reach 2^32) and associative integer atomics: bit-identical to the reference.
#include <cudaTypedefs.h>
#include <mutex>
#include "dpm_common.cuh"
#include "ptx.cuh"

namespace dpm {

// Pipe balance.  The fold adds are 3-input IADD3 on the ALU pipe; a window
// listed in DPM_FMA_FOLDS (bit 0 DIAG, 1 ANTI, 2 X2P, 3 X2M, 4 profile) is
// folded with single IMAD-by-1 adds on the otherwise idle FMA pipe instead.
#ifndef DPM_FMA_FOLDS
#define DPM_FMA_FOLDS 16
#endif
// DPM_UNPACK_MIX: 16-bit unpack as hi = SHF (ALU), lo = IMAD (FMA) instead of LOP3 + SHF
// single-tile volumes store complete image rows instead of adding them
#ifndef DPM_SINGLE_TILE
#define DPM_SINGLE_TILE 1
#endif
#ifndef DPM_UNPACK_MIX
#define DPM_UNPACK_MIX 0
#endif

struct StreamParams {
  int64_t L, M, N, B;
  int32_t offset;
  int64_t ntx, ntz, ncol;      // tiles along x, z; columns = B * ntz * ntx
  int64_t band;                // rows per y-band
  uint32_t one;                // == 1 at run time: keeps the ZX adds on the FMA pipe (IMAD)
  ImageSet s;
  // profile mode: the y-summed profile P[x + t z] (uint64 [B][WQ]) replaces
  // the ZX image; qoff = |t| (N - 1) for t < 0, else 0
  unsigned long long* prof;
  int64_t WQ, qoff;
  // single-tile moments pass (one x-tile and one z-tile per volume): every image
  // row is completed by the one CTA that owns its row-step, so rows are stored
  // (no zeroing, no read-modify-write in L2) instead of added
  uint32_t single;
};

// Profile direction t of the moments pass (x + t z, summed over y), by image
// count: the next (x, z) direction after the oblique images of the order --
// order 3: -1, order 4: 2, order 5: -2, order 6: 3 ("profile").
template <int NI> struct ProfT { static constexpr int value = NI <= 4 ? -1 : NI == 5 ? 2 : NI == 6 ? -2 : 3; };

// ---- VX-voxel lane vectors --------------------------------------------------
template <typename T, int VX> struct Vec;
template <> struct Vec<uint16_t, 8> { using type = uint4; };
template <> struct Vec<int16_t, 8>  { using type = uint4; };
template <> struct Vec<uint8_t, 8>  { using type = uint2; };
template <> struct Vec<uint16_t, 4> { using type = uint2; };
template <> struct Vec<int16_t, 4>  { using type = uint2; };
template <> struct Vec<uint8_t, 4>  { using type = uint32_t; };

template <typename T, int VX> struct Unpack;
template <int VX> struct Unpack<uint16_t, VX> {
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t, uint32_t one16) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < VX / 2; ++i) {
      v[2 * i + 1] = w[i] >> 16;
      v[2 * i] = DPM_UNPACK_MIX ? ptx::mad_u32(v[2 * i + 1], 0u - one16, w[i]) : (w[i] & 0xFFFFu);
    }
  }
};
// signed 16-bit plus offset: lo half sign-extended by one PRMT (sign-replicate
// selector), hi half by an arithmetic shift, then the offset.  The caller
// passes off = 0 for out-of-bounds planes / lanes, whose TMA zero fill must
// stay 0 -- one select per plane instead of one per voxel.
template <int VX> struct Unpack<int16_t, VX> {
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t off, uint32_t) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < VX / 2; ++i) {
      uint32_t lo;   // prmt with sign-replicate selector nibbles (__byte_perm ignores the sign bit)
      asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(lo) : "r"(w[i]));
      v[2 * i] = lo + (uint32_t)off;
      v[2 * i + 1] = (uint32_t)((int32_t)w[i] >> 16) + (uint32_t)off;
    }
  }
};
template <int VX> struct Unpack<uint8_t, VX> {
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t, uint32_t) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < VX / 4; ++i) {
      #pragma unroll
      for (int j = 0; j < 4; ++j) v[4 * i + j] = __byte_perm(w[i], 0u, 0x4440u + j);   // one PRMT per byte
    }
  }
};

// Sum of a lane's VX voxels of one plane straight from the packed vector:
// byte dot products with ones (IDP, FMA pipe), independent of the unpack, and
// two planes per redux.  Used for 8-wide uint8 lanes only: measured faster
// there (1024^3 u8 K3 -12 %), slower for 4-wide u8 lanes (cfg4 +3 %) and for
// uint16 with __dp2a (cfg5 +3 %) -- tools/EXPERIMENTS.md v25.
template <typename T, int VX> struct PlaneSum {
  static constexpr bool packed = sizeof(T) == 1 && VX == 8;
  template <typename V> __device__ __forceinline__ static uint32_t run(const V& d) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    uint32_t s = 0;
    if constexpr (sizeof(T) == 1) {
      #pragma unroll
      for (int i = 0; i < VX / 4; ++i) s = __dp4a(w[i], 0x01010101u, s);
    } else {
      #pragma unroll
      for (int i = 0; i < VX / 2; ++i) s = __dp2a_lo(w[i], 0x0101u, s);
    }
    return s;
  }
};

// win[c] += a[c - OA] + b[c - OB] over the cells the plane pair reaches (a =
// plane t, b = plane t+1); OA/OB are constants after unrolling.
//   DIAG c = k + t:        OA = t,        OB = t + 1
//   ANTI c = k - t + 7:    OA = 7 - t,    OB = 6 - t
//   X2P  c = k + 2t:       OA = 2t,       OB = 2t + 2
//   X2M  c = k - 2t + 14:  OA = 14 - 2t,  OB = 12 - 2t
template <int NW, int VX>
__device__ __forceinline__ void fold_pair(uint32_t* win, const uint32_t* a, const uint32_t* b, int OA, int OB) {
  #pragma unroll
  for (int c = 0; c < NW; ++c) {
    const int ka = c - OA, kb = c - OB;
    const bool ha = ka >= 0 && ka < VX, hb = kb >= 0 && kb < VX;
    if (ha && hb) win[c] += a[ka] + b[kb];
    else if (ha) win[c] += a[ka];
    else if (hb) win[c] += b[kb];
  }
}

// fold_pair with single adds on the FMA pipe (IMAD by a run-time 1)
template <int NW, int VX>
__device__ __forceinline__ void fold_pair_fma(uint32_t* win, const uint32_t* a, const uint32_t* b, int OA, int OB,
                                              uint32_t one);
template <int BIT, int NW, int VX>
__device__ __forceinline__ void fold(uint32_t* win, const uint32_t* a, const uint32_t* b, int OA, int OB, uint32_t one) {
  if constexpr (((DPM_FMA_FOLDS >> BIT) & 1) != 0) fold_pair_fma<NW, VX>(win, a, b, OA, OB, one);
  else fold_pair<NW, VX>(win, a, b, OA, OB);
}
template <int NW, int VX>
__device__ __forceinline__ void fold_pair_fma(uint32_t* win, const uint32_t* a, const uint32_t* b, int OA, int OB,
                                              uint32_t one) {
  #pragma unroll
  for (int c = 0; c < NW; ++c) {
    const int ka = c - OA, kb = c - OB;
    if (ka >= 0 && ka < VX) win[c] = ptx::mad_u32(a[ka], one, win[c]);
    if (kb >= 0 && kb < VX) win[c] = ptx::mad_u32(b[kb], one, win[c]);
  }
}

// owned cells VX*g .. VX*g+VX-1 of a transposed region with stride S: word c*S + g;
// `addr` = region byte address + 4*g
template <int S, int VX>
__device__ __forceinline__ void add_owned(uint32_t addr, const uint32_t* win) {
  #pragma unroll
  for (int c = 0; c < VX; ++c) ptx::red_shared_add_dyn(addr + 4 * c * S, win[c]);
}

// whole window: cell c of lane g goes to word (c % VX) * S + g + c / VX --
// for a fixed c the 32 lanes hit 32 consecutive words (no bank conflict);
// overlaps between neighbouring lanes and the top lanes' halo are resolved
// by the shared-memory atomics themselves (no shuffles, no per-lane branches)
template <int S, int VX, int NW>
__device__ __forceinline__ void add_window(uint32_t addr, const uint32_t* win) {
  #pragma unroll
  for (int c = 0; c < NW; ++c) ptx::red_shared_add_dyn(addr + 4 * ((c % VX) * S + c / VX), win[c]);
}

// VX-value sums with 3-input adds
template <int VX> __device__ __forceinline__ uint32_t sumv(const uint32_t* v) {
  if (VX == 8) {
    const uint32_t s0 = v[0] + v[1] + v[2];
    const uint32_t s1 = s0 + v[3] + v[4];
    const uint32_t s2 = s1 + v[5] + v[6];
    return s2 + v[7];
  }
  return (v[0] + v[1] + v[2]) + v[VX - 1];
}

// Per-CTA cursor over its row-steps: bands in order; inside a band the CTA's
// contiguous run of the (column, y) sequence.  Advances incrementally (the
// 64-bit divisions happen once per band, not per row-step).
struct Cursor {
  int32_t y0, yb, c, yoff, left;
  bool done;
  // floor(seq * i / g) without a 64-bit division (a call: call sites reachable
  // from the row-step loop cost the loop its register allocation); the host
  // guarantees seq < 2^31 (a row-step is >= 4 KB of voxels)
  static __device__ __forceinline__ uint32_t share(uint32_t seq, uint32_t i, uint32_t g) {
    const uint32_t q = seq / g, r = seq - q * g;
    return q * i + (r * i) / g;
  }
  __device__ __forceinline__ void band_setup(const StreamParams& p) {
    while (y0 < p.M) {
      yb = (int32_t)imin64(p.band, p.M - y0);
      const uint32_t seq = (uint32_t)p.ncol * (uint32_t)yb;
      const uint32_t s = share(seq, blockIdx.x, gridDim.x);
      const uint32_t e = share(seq, blockIdx.x + 1, gridDim.x);
      if (s < e) { c = (int32_t)(s / (uint32_t)yb); yoff = (int32_t)(s - (uint32_t)c * (uint32_t)yb); left = (int32_t)(e - s); done = false; return; }
      y0 += (int32_t)p.band;
    }
    done = true;
  }
  __device__ void init(const StreamParams& p) { y0 = 0; band_setup(p); }
  __device__ __forceinline__ void advance(const StreamParams& p) {
    if (--left == 0) { y0 += (int32_t)p.band; band_setup(p); return; }
    if (++yoff == yb) { yoff = 0; ++c; }
  }
  __device__ __forceinline__ int32_t y() const { return y0 + yoff; }
  // rows left in the current column within this band and this CTA's run
  __device__ __forceinline__ int32_t run() const { return left < yb - yoff ? left : yb - yoff; }
  __device__ __forceinline__ void advance_by(const StreamParams& p, int32_t n) {
    left -= n;
    if (left == 0) { y0 += (int32_t)p.band; band_setup(p); return; }
    yoff += n;
    if (yoff == yb) { yoff = 0; ++c; }
  }
};


// Per-(NI, NW, VX) geometry of the CTA rows (transposed layout, see header).
__host__ __device__ constexpr int stride_for(int need, int VX) {
  // smallest S >= need with S = 32/VX (mod 32)
  return ((need - (32 / VX) + 31) / 32) * 32 + (32 / VX);
}
template <int NI, int NW, int VX, int ZP = 8> struct Geo {
  static constexpr int SX = 32 * VX;                   // x-tile
  static constexpr int SZ = ZP * NW;                   // z-tile (ZP planes per warp)
  static constexpr int W1 = SX + SZ - 1;               // DIAG/ANTI row footprint
  static constexpr int W2 = SX + 2 * SZ - 2;           // X2P/X2M row footprint
  static constexpr int SXY = stride_for(32 + 1, VX);
  static constexpr int SOB = stride_for(((W2 + VX - 1) / VX + 3) / 4 * 4 + 2, VX);
  static constexpr int XY = 0, DG = VX * SXY, AN = DG + VX * SOB, XP = AN + VX * SOB, XM = XP + VX * SOB;
  static constexpr int WORDS = NI <= 4 ? DG + VX * SOB : NI == 5 ? AN + VX * SOB : NI == 6 ? XP + VX * SOB : XM + VX * SOB;
  static constexpr int THREADS = 32 * NW;
  // YZ plane sums staged per 8 consecutive y in shared memory (orders <= 5; at
  // order 6 the extra code costs more than the scattered atomics it saves)
  static constexpr int YZT = NI <= 6 ? SZ * 8 : 0;
  // profile mode: the CTA's profile row (x + t z over the SX x SZ tile), in the
  // same transposed layout (cell i at (i % VX) * SPQ + i / VX)
  static constexpr int AQ = ProfT<NI>::value < 0 ? -ProfT<NI>::value : ProfT<NI>::value;
  static constexpr int WQC = SX + AQ * (SZ - 1);
  static constexpr int SPQ = (WQC + VX - 1) / VX;
  static constexpr int PW = VX * SPQ;
};

struct ColGeom {
  int64_t X0, Z0;
  int32_t b;
  int zc;
  bool xok;
  __device__ __forceinline__ void set(const StreamParams& p, int32_t col, int SX, int SZ, int VX, int ZP, int w,
                                      int lane) {
    const int32_t per = (int32_t)(p.ntz * p.ntx);
    b = col / per;
    const int32_t r = col - b * per;
    Z0 = (int64_t)(r / (int32_t)p.ntx) * SZ;
    X0 = (int64_t)(r % (int32_t)p.ntx) * SX;
    zc = (int)imax64(0, imin64(ZP, p.N - (Z0 + ZP * w)));
    xok = X0 + VX * lane < p.L;
  }
};

// one transposed region of a CTA row buffer -> global image row.  Cell c sits
// at word (c % VX) * S + c / VX, so one 16-byte word group of residue row r
// holds cells VX*q + r + {0, VX, 2VX, 3VX}: one LDS.128 / STS.128 and four
// immediate-offset reds per 4 cells.  `g` points at local cell 0 of the
// global row; [lo, hi) is the part of the padded extent inside the row.
// Cells past NCELL are never written (zero), so reducing them is harmless.
template <int VX, int S, int NCELL, int THREADS>
__device__ __forceinline__ void flush_region(uint32_t* rw, int tid, uint32_t* g, int lo, int hi, bool single) {
  constexpr int WORDS = (NCELL + VX - 1) / VX;
  constexpr int QCH = (WORDS + 3) / 4;
  constexpr int NCH = VX * QCH;
  static_assert(4 * QCH <= S, "row stride must cover the padded word groups");
  const bool interior = lo == 0 && hi >= 4 * QCH * VX;    // uniform per CTA
  #pragma unroll
  for (int it = 0; it < (NCH + THREADS - 1) / THREADS; ++it) {
    const int j = tid + it * THREADS;
    if ((NCH % THREADS) != 0 && j >= NCH) break;
    const int r = j % VX, q = 4 * (j / VX);
    uint4* wp = reinterpret_cast<uint4*>(rw + r * S + q);
    const uint4 v = *wp;
    *wp = make_uint4(0u, 0u, 0u, 0u);
    const int c0 = VX * q + r;
    uint32_t* gp = g + c0;
    if (single) {
      ptx::st_global_if(gp, v.x, c0 >= lo && c0 < hi);
      ptx::st_global_if(gp + VX, v.y, c0 + VX >= lo && c0 + VX < hi);
      ptx::st_global_if(gp + 2 * VX, v.z, c0 + 2 * VX >= lo && c0 + 2 * VX < hi);
      ptx::st_global_if(gp + 3 * VX, v.w, c0 + 3 * VX >= lo && c0 + 3 * VX < hi);
    } else if (interior) {
      ptx::red_global_add_off<0>(gp, v.x);
      ptx::red_global_add_off<4 * VX>(gp, v.y);
      ptx::red_global_add_off<8 * VX>(gp, v.z);
      ptx::red_global_add_off<12 * VX>(gp, v.w);
    } else {
      ptx::red_global_add_if(gp, v.x, c0 >= lo && c0 < hi);
      ptx::red_global_add_if(gp + VX, v.y, c0 + VX >= lo && c0 + VX < hi);
      ptx::red_global_add_if(gp + 2 * VX, v.z, c0 + 2 * VX >= lo && c0 + 2 * VX < hi);
      ptx::red_global_add_if(gp + 3 * VX, v.w, c0 + 3 * VX >= lo && c0 + 3 * VX < hi);
    }
  }
}

// per-column flush geometry of one region: global offset of local cell 0 and
// the local range [lo, hi) that lies inside the image row
struct RegionCol {
  int64_t g0;
  int lo, hi;
  __device__ __forceinline__ void set(int64_t g0_, int64_t W) {
    g0 = g0_;
    lo = (int)imax64(0, -g0_);
    hi = (int)imin64(1 << 30, W - g0_);
  }
};

// ZP: planes per warp (8, or 16 for the 4-wide-lane batch variant, profile
// mode only); CTAS: resident CTAs per SM
template <typename T, int NI, int NW, int VX, int STAGES, bool PROF, int ZP, int CTAS>
__global__ void __launch_bounds__(32 * NW, CTAS)
project_stream_kernel(const __grid_constant__ CUtensorMap tmap, const StreamParams p) {
  static_assert(ZP == 8 || ((ZP == 16 || ZP == 32) && PROF && NI <= 5), "16/32-plane warps: profile mode, orders <= 4");
  using G = Geo<NI, NW, VX, ZP>;
  using V = typename Vec<T, VX>::type;
  constexpr int SX = G::SX, SZ = G::SZ, THREADS = G::THREADS;
  constexpr int N1 = VX + ZP - 1, N2 = VX + 2 * (ZP - 1);   // oblique window widths
#ifndef DPM_PROF_TWO_PASS
#define DPM_PROF_TWO_PASS 0
#endif
  // +-2z images in a second pass over the stage (the ZX registers leave no room
  // for them in the first); the profile mode frees those registers
  constexpr bool TWO_PASS = NI >= 6 && VX == 8 && NW > 8 && (!PROF || DPM_PROF_TWO_PASS);
  constexpr int TQ = ProfT<NI>::value, AQ = TQ < 0 ? -TQ : TQ;
  constexpr int NQ = PROF ? VX + (ZP - 1) * AQ : 1;    // profile window width
  constexpr uint32_t STAGE_BYTES = SX * SZ * sizeof(T);
  constexpr int YZT = G::YZT;   // words of one YZ tile (0: YZ goes straight to global)
  // TMA producer: lane 0 of a middle warp.  The row flushes start at thread 0,
  // so warps 0-3 carry them; keeping the producer's per-row-step work off those
  // warps shortens the slowest warp (cfg5 -5.7 %, tools/EXPERIMENTS.md v14)
  constexpr int PROD = 32 * (NW / 2);
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* rows = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES);   // [2][G::WORDS]
  uint32_t* yzb = rows + 2 * G::WORDS;                                          // [2][SZ][8] plane sums by y % 8
  uint64_t* full = reinterpret_cast<uint64_t*>(yzb + 2 * YZT);                  // [STAGES]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t rows_addr = ptx::smem_addr(rows), full_addr = ptx::smem_addr(full);
  const bool single = PROF && p.single != 0;

  for (int i = tid; i < 2 * G::WORDS + 2 * YZT; i += THREADS) rows[i] = 0;
  if constexpr (PROF) {
    uint32_t* pr = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_BYTES + (2 * G::WORDS + 2 * YZT) * 4 +
                                               STAGES * 8 + 64 + 160);
    for (int i = tid; i < G::PW; i += THREADS) pr[i] = 0;
  }
  if (tid == 0) {
    ptx::prefetch_tmap(&tmap);
    for (int i = 0; i < STAGES; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();

  // producer (lane 0 of warp NW/2): STAGES row-steps ahead; refills after each
  // row-step barrier.  For the 7-image kernel its cursor lives in shared memory
  // instead of registers every thread would reserve (-1.4 % at order 6; the
  // extra latency costs more than it saves for the smaller kernels).
  constexpr bool PROD_SMEM = NI >= 7;
  struct ProdState { Cursor cur; int pst; };
  ProdState* ps = reinterpret_cast<ProdState*>(full + STAGES);
  ProdState preg;
  preg.cur.done = true;
  preg.pst = 0;
  uint64_t evict_first = 0;
  auto issue_from = [&](ProdState& st) {
    const int32_t per = (int32_t)(p.ntz * p.ntx);
    const int32_t b = st.cur.c / per, r = st.cur.c - b * per;
    const int32_t zt = r / (int32_t)p.ntx;
    const int k = st.pst;
    ptx::mbar_arrive_expect_tx(&full[k], STAGE_BYTES);
    ptx::tma_load_4d_hint(stages + k * STAGE_BYTES, &tmap, &full[k], (r - zt * (int32_t)p.ntx) * SX, st.cur.y(),
                          zt * SZ, b, PROD_SMEM ? ptx::policy_evict_first() : evict_first);
    st.cur.advance(p);
    st.pst = k + 1 == STAGES ? 0 : k + 1;
  };
  if (tid == PROD) {
    if (!PROD_SMEM) evict_first = ptx::policy_evict_first();
    ProdState st;
    st.cur.init(p);
    st.pst = 0;
    for (int i = 0; i < STAGES && !st.cur.done; ++i) issue_from(st);
    if (PROD_SMEM) *ps = st; else preg = st;
  }
  auto issue = [&]() {
    if (PROD_SMEM) {
      ProdState st = *ps;
      if (!st.cur.done) { issue_from(st); *ps = st; }
    } else if (!preg.cur.done) {
      issue_from(preg);
    }
  };

  Cursor cur;
  cur.init(p);
  uint32_t zx[8][PROF ? 1 : VX];
  uint32_t wq[NQ];                // profile window (x + TQ z over this lane's patch), summed over y
  #pragma unroll
  for (int i = 0; i < NQ; ++i) wq[i] = 0;
  int32_t col = -1, band_y0 = -1;
  ColGeom g;
  g.X0 = g.Z0 = 0; g.b = 0; g.zc = 0; g.xok = false;
  uint32_t* zx_col = nullptr;
  uint32_t* yz_col = nullptr;
  // flush geometry of the current column: identical for all threads, so it
  // lives in shared memory (two slots by column parity: thread 0 fills the
  // next column's slot while others may still flush the previous column)
  RegionCol* rcs = reinterpret_cast<RegionCol*>(reinterpret_cast<uint8_t*>(full + STAGES) + 64);
  uint32_t* prow = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(full + STAGES) + 64 + 160);   // [G::PW]
  int rslot = 0;
  int cst = 0, parity = 0, yzpar = 0;
  uint32_t cphase = 0;

  // ZX flush at the end of a column segment.  Lane l = 8g + j holds the sums
  // of x = X0 + VX*l + k, planes t = 0..7.  Per k, an 8x8 shfl.xor butterfly
  // transposes (lane-in-group, plane) so that afterwards lane j holds plane j of
  // the 8 x's of its group: every red.global then covers 4 runs of 8
  // consecutive z (32 B each) instead of 32 scattered words.
  auto flush_zx = [&]() {
    if constexpr (!PROF) {
    if (col < 0) return;
    const int j = lane & 7, g8 = lane >> 3;
    uint32_t* base = p.s.img[DPM_IMG_ZX] + (int64_t)g.b * p.L * p.N + (g.X0 + VX * 8 * g8) * p.N + g.Z0 + 8 * w + j;
    const bool zok = j < g.zc;
    const int64_t xg = g.X0 + VX * 8 * g8;
    #pragma unroll
    for (int k = 0; k < VX; ++k) {
      uint32_t r[8];
      #pragma unroll
      for (int t = 0; t < 8; ++t) r[t] = zx[t][k];
      #pragma unroll
      for (int sft = 4; sft >= 1; sft >>= 1) {
        const bool up = (j & sft) != 0;
        #pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (t & sft) continue;
          const uint32_t send = up ? r[t] : r[t | sft];
          const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, sft);
          if (up) r[t] = recv; else r[t | sft] = recv;
        }
      }
      #pragma unroll
      for (int i = 0; i < 8; ++i)   // r[i] = plane j of x = xg + VX*i + k
        ptx::red_global_add_if(base + (int64_t)(VX * i + k) * p.N, r[i], r[i] != 0 && zok && xg + VX * i + k < p.L);
    }
    }
  };

  // profile flush (per column and y-band, CTA-uniform): every lane adds its
  // window to the CTA's profile row (cell VX*lane + 8*w*TQ + c, or with
  // 8*(NW-1-w)*|TQ| for TQ < 0; transposed, so conflict-free), then the CTA
  // adds the row to the global profile with one coalesced pass of 64-bit
  // atomics (row cell 0 = global index X0 + TQ Z0, or X0 - |TQ|(Z0 + SZ - 1) + qoff).
  // Only real voxels contribute, so every non-zero cell lies inside [0, WQ).
  auto flush_prof = [&]() {
    if constexpr (PROF) {
      if (col < 0) return;
      const uint32_t pa = ptx::smem_addr(prow) + 4u * lane;
      const int lb = TQ > 0 ? ZP * w * TQ : ZP * (NW - 1 - w) * AQ;   // warp's first row cell - VX*lane
      #pragma unroll
      for (int c = 0; c < NQ; ++c) {
        const int i = lb + c;   // + VX * lane
        if (wq[c] != 0) ptx::red_shared_add_dyn(pa + 4u * ((i % VX) * G::SPQ + i / VX), wq[c]);
        wq[c] = 0;
      }
      __syncthreads();
      unsigned long long* gq = p.prof + (int64_t)g.b * p.WQ +
                               (TQ > 0 ? g.X0 + TQ * g.Z0 : g.X0 - AQ * (g.Z0 + SZ - 1) + p.qoff);
      for (int i = tid; i < G::WQC; i += THREADS) {
        uint32_t* cell = prow + (i % VX) * G::SPQ + i / VX;
        const uint32_t v = *cell;
        *cell = 0;
        if (v) atomicAdd(gq + i, (unsigned long long)v);
      }
      __syncthreads();
    }
  };

  while (!cur.done) {
    if (PROF && (cur.c != col || cur.y0 != band_y0)) {   // per column and y-band: <= 4096 rows per window sum
      flush_prof();
      band_y0 = cur.y0;
    }
    if (cur.c != col) {
      flush_zx();
      col = cur.c;
      g.set(p, col, SX, SZ, VX, ZP, w, lane);
      if constexpr (!PROF) {
        #pragma unroll
        for (int t = 0; t < 8; ++t) {
          #pragma unroll
          for (int k = 0; k < VX; ++k) zx[t][k] = 0;
        }
      }
      zx_col = p.s.img[DPM_IMG_ZX] + (int64_t)g.b * p.L * p.N + (g.X0 + VX * lane) * p.N + g.Z0 + ZP * w;
      yz_col = p.s.img[DPM_IMG_YZ] + (int64_t)g.b * p.M * p.N + (g.Z0 + ZP * w + (lane & (ZP - 1))) * p.M;
      rslot ^= 1;
      if (tid == 0) {
        RegionCol* rc = rcs + 5 * rslot;
        rc[0].set(g.X0, p.L);
        rc[1].set(g.X0 + g.Z0, p.s.W[DPM_IMG_DIAG]);
        if (NI > DPM_IMG_ANTI) rc[2].set(g.X0 - g.Z0 - (SZ - 1) + p.N - 1, p.s.W[DPM_IMG_ANTI]);
        if (NI > DPM_IMG_X2P) rc[3].set(g.X0 + 2 * g.Z0, p.s.W[DPM_IMG_X2P]);
        if (NI > DPM_IMG_X2M) rc[4].set(g.X0 - 2 * g.Z0 - 2 * (SZ - 1) + 2 * (p.N - 1), p.s.W[DPM_IMG_X2M]);
      }
    }
    // consecutive rows of this column: no column or band logic per row-step
    const int32_t y_first = cur.y(), y_end = y_first + cur.run();
    for (int32_t y = y_first; y < y_end; ++y) {
    if (g.zc > 0) {   // warp-uniform: warps past the volume's last plane only join the barrier
    ptx::mbar_wait_addr(full_addr + 8u * cst, cphase);
    const T* tile = reinterpret_cast<const T*>(stages + cst * STAGE_BYTES) + (ZP * w) * SX + VX * lane;

    uint32_t cs[VX];
    uint32_t yzmine = 0;   // lane t < 8: this warp's plane t sum (YZ), reduced as each plane pair is folded
    uint32_t wd[N1], wa[N1], wp[N2], wm[N2];
    #pragma unroll
    for (int i = 0; i < VX; ++i) cs[i] = 0;
    #pragma unroll
    for (int i = 0; i < N1; ++i) { wd[i] = 0; wa[i] = 0; }
    #pragma unroll
    for (int i = 0; i < N2; ++i) { wp[i] = 0; wm[i] = 0; }
    V dv[ZP];
    #pragma unroll
    for (int t = 0; t < 4; ++t) dv[t] = *reinterpret_cast<const V*>(tile + t * SX);
    #pragma unroll
    for (int tp = 0; tp < ZP / 2; ++tp) {
      const int t0 = 2 * tp, t1 = t0 + 1;
      if (tp >= 1 && 2 * tp + 3 < ZP) {   // two plane pairs in flight (16 fewer live registers than all 8 up front)
        #pragma unroll
        for (int t = 2 * tp + 2; t < 2 * tp + 4; ++t) dv[t] = *reinterpret_cast<const V*>(tile + t * SX);
      }
      uint32_t a[VX], bb[VX];
      // signed input: out-of-bounds (zero-filled) voxels get no offset
      Unpack<T, VX>::run(dv[t0], a, g.xok && t0 < g.zc ? p.offset : 0, p.one << 16);
      Unpack<T, VX>::run(dv[t1], bb, g.xok && t1 < g.zc ? p.offset : 0, p.one << 16);
      #pragma unroll
      for (int k = 0; k < VX; ++k) {
        if constexpr (!PROF) {
          zx[t0][k] = ptx::mad_u32(a[k], p.one, zx[t0][k]);
          zx[t1][k] = ptx::mad_u32(bb[k], p.one, zx[t1][k]);
        }
        cs[k] += a[k] + bb[k];
      }
      if constexpr (PROF) {   // profile x + TQ z: window cell k + TQ t (TQ > 0) or k + |TQ| (7 - t)
        // plane pair 3 of orders <= 5 folds the profile with IADD3 (ALU), the
        // rest with IMAD (FMA): the pipe balance measured best (EXPERIMENTS.md v24)
        constexpr int ALU_PAIRS = NI >= 7 ? 0 : 8;
        if (((ALU_PAIRS >> tp) & 1) != 0) {
          if (TQ > 0) fold_pair<NQ, VX>(wq, a, bb, TQ * t0, TQ * t1);
          else fold_pair<NQ, VX>(wq, a, bb, AQ * (ZP - 1 - t0), AQ * (ZP - 1 - t1));
        } else {
          if (TQ > 0) fold<4, NQ, VX>(wq, a, bb, TQ * t0, TQ * t1, p.one);
          else fold<4, NQ, VX>(wq, a, bb, AQ * (ZP - 1 - t0), AQ * (ZP - 1 - t1), p.one);
        }
      }
      {   // YZ: warp-wide redux of the plane sums (one REDUX per plane)
        if constexpr (PlaneSum<T, VX>::packed && sizeof(T) == 1) {
          // u8: both plane sums in one redux (16-bit fields: 32 lanes x VX x 255 < 2^16)
          const uint32_t r = __reduce_add_sync(0xffffffffu, ptx::mad_u32(PlaneSum<T, VX>::run(dv[t1]), p.one << 16,
                                                                         PlaneSum<T, VX>::run(dv[t0])));
          yzmine = lane == t0 ? (r & 0xFFFFu) : (lane == t1 ? (r >> 16) : yzmine);
        } else {
          const uint32_t s0 = __reduce_add_sync(0xffffffffu, PlaneSum<T, VX>::packed ? PlaneSum<T, VX>::run(dv[t0]) : sumv<VX>(a));
          const uint32_t s1 = __reduce_add_sync(0xffffffffu, PlaneSum<T, VX>::packed ? PlaneSum<T, VX>::run(dv[t1]) : sumv<VX>(bb));
          yzmine = lane == t0 ? s0 : (lane == t1 ? s1 : yzmine);
        }
      }
      fold<0, N1, VX>(wd, a, bb, t0, t0 + 1, p.one);
      if (NI > DPM_IMG_ANTI) fold<1, N1, VX>(wa, a, bb, ZP - 1 - t0, ZP - 2 - t0, p.one);
      if (!TWO_PASS && NI > DPM_IMG_X2P) fold<2, N2, VX>(wp, a, bb, 2 * t0, 2 * t0 + 2, p.one);
      if (!TWO_PASS && NI > DPM_IMG_X2M) fold<3, N2, VX>(wm, a, bb, 2 * (ZP - 1) - 2 * t0, 2 * (ZP - 2) - 2 * t0, p.one);
    }

    // ---- YZ: lane t < 8 holds plane t of this warp (reduced in the fold loop)
    if (YZT > 0) {
      if (lane < ZP) yzb[yzpar * SZ * 8 + (ZP * w + lane) * 8 + (y & 7)] = yzmine;
    } else {
      if (single) ptx::st_global_if(yz_col + y, yzmine, lane < ZP && lane < g.zc);
      else ptx::red_global_add_if(yz_col + y, yzmine, lane < ZP && yzmine != 0 && lane < g.zc);
    }

    // ---- add the XY column sums and the oblique windows to the CTA rows
    {
      const uint32_t rp = rows_addr + (uint32_t)(parity * G::WORDS * 4);
      add_owned<G::SXY, VX>(rp + 4 * (G::XY + lane), cs);
      {
        const uint32_t base = rp + 4 * (G::DG + lane + (ZP / VX) * w);
        add_window<G::SOB, VX, N1>(base, wd);
      }
      if (NI > DPM_IMG_ANTI) {
        const uint32_t base = rp + 4 * (G::AN + lane + (ZP / VX) * (NW - 1 - w));
        add_window<G::SOB, VX, N1>(base, wa);
      }
      if (TWO_PASS) {
        // second pass over the same stage for the (x +- 2z, y) images: keeps the
        // live register set of order 6 within the 12-warp budget
        #pragma unroll
        for (int i = 0; i < N2; ++i) { wp[i] = 0; wm[i] = 0; }
        #pragma unroll
        for (int tp = 0; tp < 4; ++tp) {
          const int t0 = 2 * tp, t1 = t0 + 1;
          uint32_t a[VX], bb[VX];
          Unpack<T, VX>::run(*reinterpret_cast<const V*>(tile + t0 * SX), a, g.xok && t0 < g.zc ? p.offset : 0,
                             p.one << 16);
          Unpack<T, VX>::run(*reinterpret_cast<const V*>(tile + t1 * SX), bb, g.xok && t1 < g.zc ? p.offset : 0,
                             p.one << 16);
          fold<2, N2, VX>(wp, a, bb, 2 * t0, 2 * t0 + 2, p.one);
          fold<3, N2, VX>(wm, a, bb, 14 - 2 * t0, 12 - 2 * t0, p.one);
        }
      }
      if (NI > DPM_IMG_X2P) {
        const uint32_t base = rp + 4 * (G::XP + lane + (2 * ZP / VX) * w);
        add_window<G::SOB, VX, N2>(base, wp);
      }
      if (NI > DPM_IMG_X2M) {
        const uint32_t base = rp + 4 * (G::XM + lane + (2 * ZP / VX) * (NW - 1 - w));
        add_window<G::SOB, VX, N2>(base, wm);
      }
    }
    }  // g.zc > 0

    __syncthreads();
    if (tid == PROD) issue();   // every warp is done with stage `cst`

    // ---- flush this row-step's CTA rows -------------------------------------
    {
      uint32_t* rw = rows + parity * G::WORDS;
      // 32-bit row index and widths (the host checks B*M and W < 2^31 for this
      // kernel): one IMAD.WIDE.U32 per region instead of 64-bit multiplies
      const uint32_t rowid = (uint32_t)g.b * (uint32_t)p.M + (uint32_t)y;
      auto row = [&](int k, uint32_t w32, int64_t g0) { return p.s.img[k] + ((uint64_t)rowid * w32 + g0); };
      const RegionCol* rc = rcs + 5 * rslot;   // written before this column's first barrier
      flush_region<VX, G::SXY, SX, THREADS>(rw + G::XY, tid, row(DPM_IMG_XY, (uint32_t)p.L, rc[0].g0), rc[0].lo, rc[0].hi, single);
      const uint32_t Wd = (uint32_t)p.s.W[DPM_IMG_DIAG];
      flush_region<VX, G::SOB, G::W1, THREADS>(rw + G::DG, tid, row(DPM_IMG_DIAG, Wd, rc[1].g0), rc[1].lo, rc[1].hi, single);
      if (NI > DPM_IMG_ANTI)
        flush_region<VX, G::SOB, G::W1, THREADS>(rw + G::AN, tid, row(DPM_IMG_ANTI, Wd, rc[2].g0), rc[2].lo, rc[2].hi, single);
      if (NI > DPM_IMG_X2P) {
        const uint32_t W2g = (uint32_t)p.s.W[DPM_IMG_X2P];
        flush_region<VX, G::SOB, G::W2, THREADS>(rw + G::XP, tid, row(DPM_IMG_X2P, W2g, rc[3].g0), rc[3].lo, rc[3].hi, single);
        if (NI > DPM_IMG_X2M)
          flush_region<VX, G::SOB, G::W2, THREADS>(rw + G::XM, tid, row(DPM_IMG_X2M, W2g, rc[4].g0), rc[4].lo, rc[4].hi, single);
      }
    }
    parity ^= 1;
    if (++cst == STAGES) { cst = 0; cphase ^= 1u; }
    // YZ tile -> image once 8 consecutive y are in (or the run of y ends):
    // 8 threads cover 32 contiguous bytes of a z-row
    if (YZT > 0 && (y + 1 == y_end || ((y + 1) & 7) == 0)) {
      uint32_t* tb = yzb + yzpar * SZ * 8;
      uint32_t* gy = p.s.img[DPM_IMG_YZ] + (int64_t)g.b * p.M * p.N + g.Z0 * p.M + (y & ~7);
      const int ty = tid;   // (spreading the flushes over all warps measured slower: 4 %)
      #pragma unroll
      for (int it = 0; it < (SZ * 8 + THREADS - 1) / THREADS; ++it) {
        const int i = ty + it * THREADS;
        if ((SZ * 8) % THREADS != 0 && i >= SZ * 8) break;
        const uint32_t v = tb[i];
        tb[i] = 0;
        if (single) {   // only this run's rows of the group, only planes inside the volume
          const int32_t yy = (y & ~7) + (i & 7);
          ptx::st_global_if(gy + (int64_t)(i >> 3) * p.M + (i & 7), v,
                            yy >= y_first && yy <= y && g.Z0 + (i >> 3) < p.N);
        } else {
          ptx::red_global_add_if(gy + (int64_t)(i >> 3) * p.M + (i & 7), v, v != 0);
        }
      }
      yzpar ^= 1;
    }
    }  // rows of the run
    cur.advance_by(p, y_end - y_first);
  }
  flush_zx();
  flush_prof();
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

static int lane_width(const dpm_volume_desc* d) { return d->L > 128 ? 8 : 4; }

static bool stream_eligible(const dpm_volume_desc* d, const void* vox) {
  const int64_t es = d->dtype == DPM_U8 ? 1 : 2;
  if (d->L < 32 || d->N < 8) return false;
  if ((d->stride_y * es) % 16 || (d->stride_z * es) % 16) return false;
  if (d->B > 1 && (d->stride_b * es) % 16) return false;
  if (d->L % lane_width(d)) return false;  // a lane vector never straddles the row end
  if (reinterpret_cast<uintptr_t>(vox) % 16) return false;
  if (d->L > 0x7fffffffLL || d->M > 0x7fffffffLL || d->N > 0x7fffffffLL || d->B > 0x7fffffffLL) return false;
  if (d->B * d->M > 0x7fffffffLL || d->L + 2 * d->N > 0x7fffffffLL) return false;   // 32-bit row ids / widths
  return tensor_map_encoder() != nullptr;
}

size_t project_stream_workspace(const dpm_volume_desc*, int) { return 0; }

// warps per CTA: 12 (3 warps/SMSP, <= 168 registers) unless the 8-wide lanes
// of orders >= 5 need more registers (then 8 warps, <= 255 registers); the
// 4-wide lanes of order 3 fit 128 registers, so 16 warps (128-plane z-tiles)
#ifndef DPM_BATCH_ZP
#define DPM_BATCH_ZP 32  // planes per warp of the 4-wide-lane order-3 profile variant: 32 = 4 warps x 4 CTAs/SM (v27, v29)
#endif
// 8-wide uint8 lanes at orders 3-4 likewise (16 planes, 6 warps x 2 CTAs/SM:
// 1024^3 u8 K3 -3 %); for uint16 the 2-CTA shared-memory budget leaves 1-2
// stages of 48 KB, which loses (+20 %) -- tools/EXPERIMENTS.md v28
#ifndef DPM_WIDE_ZP
#define DPM_WIDE_ZP 16
#endif
// SMALL: few row-steps in total (tiny volumes): the latency of one row-step
// dominates, so 8 planes per warp (16 warps, 1 CTA) beats the batch layout
template <typename T, int NI, int VX, bool PROF, bool SMALL = false> struct CfgFor {
  static constexpr bool batch16 = DPM_BATCH_ZP >= 16 && VX == 4 && NI == 4 && PROF && !SMALL;
  static constexpr bool wide16 = DPM_WIDE_ZP == 16 && VX == 8 && NI <= 5 && PROF && sizeof(T) == 1;
  // batch layout: z-tile 128 = NW x ZP, 16 warps per SM over 16 / NW CTAs
  // (16-bit voxels: 16 planes, so a CTA's quarter of shared memory still holds 2+ stages)
  static constexpr int BZP = sizeof(T) == 1 ? DPM_BATCH_ZP : 16;
  static constexpr int ZP = batch16 ? BZP : wide16 ? 16 : 8;
  static constexpr int NW = batch16 ? 128 / BZP : wide16 ? 6 : (VX == 4 && NI == 4) ? 16 : 12;
  static constexpr int CTAS = batch16 ? 16 / NW : wide16 ? 2 : 1;
};

// stages: as many 4-D boxes as fit next to the row buffers
template <typename T, int NI, int VX, bool PROF, bool SMALL = false> struct StagesFor {
  using C = CfgFor<T, NI, VX, PROF, SMALL>;
  static constexpr int NW = C::NW;
  using GG = Geo<NI, NW, VX, C::ZP>;
  static constexpr int BOX = 32 * VX * C::ZP * NW * (int)sizeof(T);
  static constexpr int ROWS = 2 * GG::WORDS * 4 + 2 * GG::YZT * 4 + (PROF ? GG::PW * 4 : 0);
  static constexpr int FIT = ((C::CTAS == 1 ? 220 : 222 / C::CTAS) * 1024 - ROWS) / BOX;
  static constexpr int value = FIT > 12 ? 12 : FIT;
};

template <typename T, int NI, int VX, bool PROF, bool SMALL = false>
static int launch_one(const dpm_volume_desc* d, const void* vox, int grid, cudaStream_t st, StreamParams p) {
  using C = CfgFor<T, NI, VX, PROF, SMALL>;
  constexpr int NW = C::NW, ZP = C::ZP, CTAS = C::CTAS;
  constexpr int S = StagesFor<T, NI, VX, PROF, SMALL>::value;
  using G = Geo<NI, NW, VX, ZP>;
  constexpr size_t bytes = (size_t)S * G::SX * G::SZ * sizeof(T) + 2 * G::WORDS * 4 + 2 * G::YZT * 4 + S * 8 + 64 + 160 +
                           (PROF ? G::PW * 4 : 0);
  static_assert(bytes <= (CTAS == 1 ? 227 : 224 / CTAS) * 1024, "shared memory budget");
  const int64_t es = sizeof(T);
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)d->L, (cuuint64_t)d->M, (cuuint64_t)d->N, (cuuint64_t)d->B};
  const cuuint64_t strides[3] = {(cuuint64_t)(d->stride_y * es), (cuuint64_t)(d->stride_z * es),
                                 (cuuint64_t)((d->B > 1 ? d->stride_b : d->stride_z * d->N) * es)};
  const cuuint32_t box[4] = {(cuuint32_t)G::SX, 1, (cuuint32_t)G::SZ, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = tensor_map_encoder()(&map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16,
                                 4, const_cast<void*>(vox), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;  // not describable by TMA: generic path
  if (PROF) {   // CTA profile row cells (u32) sum <= SZ voxels per row-step: bound the rows per flush
    const int64_t vmax = sizeof(T) == 1 ? 255 : 65535;
    p.band = imax64(1, imin64(p.band, (int64_t)0xFFFFFFFFll / (G::SZ * vmax)));
  }
  p.ntx = (d->L + G::SX - 1) / G::SX;
  p.ntz = (d->N + G::SZ - 1) / G::SZ;
  p.ncol = p.ntx * p.ntz * d->B;
  if (p.ncol * d->M >= 0x7fffffffLL) return -1;   // 32-bit row-step positions (Cursor); not reachable in 180 GB
  p.single = (DPM_SINGLE_TILE && PROF && p.ntx == 1 && p.ntz == 1) ? 1u : 0u;
  static std::atomic<uint64_t> attr_mask{0};
  if (ensure_smem(project_stream_kernel<T, NI, NW, VX, S, PROF, ZP, CTAS>, bytes, attr_mask)) return DPM_ECUDA;
  project_stream_kernel<T, NI, NW, VX, S, PROF, ZP, CTAS>
      <<<(int)imin64((int64_t)grid * CTAS, p.ncol * d->M), 32 * NW, bytes, st>>>(map, p);
  return DPM_OK;
}

template <typename T, int VX, bool PROF>
static int launch_typed(int n_img, const dpm_volume_desc* d, const void* vox, int grid, cudaStream_t st,
                        const StreamParams& p) {
  switch (n_img) {
    case 4: return launch_one<T, 4, VX, PROF>(d, vox, grid, st, p);
    case 5: return launch_one<T, 5, VX, PROF>(d, vox, grid, st, p);
    case 6: return launch_one<T, 6, VX, PROF>(d, vox, grid, st, p);
    default: return launch_one<T, 7, VX, PROF>(d, vox, grid, st, p);
  }
}

template <typename T>
static int launch_vx(int n_img, const dpm_volume_desc* d, const void* vox, int grid, cudaStream_t st,
                     const StreamParams& p) {
  if (p.prof && n_img == 4 && lane_width(d) == 4) {
    // batch layout (32 planes per warp, 4 CTAs per SM) unless the whole pass is
    // only a few row-steps (cfg1: 64), where per-row-step latency dominates
    const int64_t rowsteps = ((d->L + 127) / 128) * ((d->N + 127) / 128) * d->B * d->M;
    if (rowsteps < 8 * (int64_t)grid) return launch_one<T, 4, 4, true, true>(d, vox, grid, st, p);
  }
  if (p.prof)
    return lane_width(d) == 8 ? launch_typed<T, 8, true>(n_img, d, vox, grid, st, p)
                              : launch_typed<T, 4, true>(n_img, d, vox, grid, st, p);
  return lane_width(d) == 8 ? launch_typed<T, 8, false>(n_img, d, vox, grid, st, p)
                            : launch_typed<T, 4, false>(n_img, d, vox, grid, st, p);
}

int profile_shift(int n_img) {
  return n_img <= 4 ? ProfT<4>::value : n_img == 5 ? ProfT<5>::value : n_img == 6 ? ProfT<6>::value : ProfT<7>::value;
}

bool project_stream_eligible(const dpm_volume_desc* d, const void* vox) { return stream_eligible(d, vox); }

template <typename T, int VX> static int64_t ztile_for(int n_img) {
  switch (n_img) {
    case 4: return (int64_t)CfgFor<T, 4, VX, true>::ZP * CfgFor<T, 4, VX, true>::NW;
    case 5: return (int64_t)CfgFor<T, 5, VX, true>::ZP * CfgFor<T, 5, VX, true>::NW;
    case 6: return (int64_t)CfgFor<T, 6, VX, true>::ZP * CfgFor<T, 6, VX, true>::NW;
    default: return (int64_t)CfgFor<T, 7, VX, true>::ZP * CfgFor<T, 7, VX, true>::NW;
  }
}

// true when the moments pass will run the streaming kernel with ONE x-tile and
// ONE z-tile per volume: it then stores complete image rows (p.single), and the
// caller need not zero the images
bool project_stream_single_tile(const dpm_volume_desc* d, const void* vox, int n_img) {
  if (!DPM_SINGLE_TILE || n_img < 4 || !stream_eligible(d, vox)) return false;
  const int vx = lane_width(d);
  int64_t sz;
  if (d->dtype == DPM_U8) sz = vx == 8 ? ztile_for<uint8_t, 8>(n_img) : ztile_for<uint8_t, 4>(n_img);
  else if (d->dtype == DPM_U16) sz = vx == 8 ? ztile_for<uint16_t, 8>(n_img) : ztile_for<uint16_t, 4>(n_img);
  else sz = vx == 8 ? ztile_for<int16_t, 8>(n_img) : ztile_for<int16_t, 4>(n_img);
  return d->L <= 32 * vx && d->N <= sz;
}

// prof != nullptr: moments mode (images except ZX + the profile along x + t z
// summed over y, t = profile_shift(n_img)); the caller zeroed images and profile
int launch_project_stream(const dpm_volume_desc* d, const void* vox, const ImageSet& s, unsigned long long* prof,
                          cudaStream_t st, bool* handled) {
  *handled = false;
  if (s.n_img < 4 || !stream_eligible(d, vox)) return DPM_OK;
  StreamParams p;
  p.L = d->L; p.M = d->M; p.N = d->N; p.B = d->B; p.offset = d->offset;
  p.ntx = p.ntz = p.ncol = 0;  // set per lane width / warp count in launch_one
  p.one = 1;
  p.s = s;
  p.prof = prof;
  {
    const int t = profile_shift(s.n_img), at = t < 0 ? -t : t;
    p.WQ = d->L + at * (d->N - 1);
    p.qoff = t < 0 ? at * (d->N - 1) : 0;
  }
  // y-band: keep one band's image rows (plus the YZ cells) within ~40 MB of L2
  int64_t row_bytes = 0;
  for (int k = 0; k < s.n_img; ++k)
    if (k != DPM_IMG_YZ && k != DPM_IMG_ZX) row_bytes += s.W[k] * 4 * d->B;
  row_bytes += d->N * 4 * d->B;
  p.band = imax64(16, imin64(d->M, (40ll << 20) / imax64(row_bytes, 1)));

  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int rc;
  switch (d->dtype) {
    case DPM_U8: rc = launch_vx<uint8_t>(s.n_img, d, vox, sms, st, p); break;
    case DPM_U16: rc = launch_vx<uint16_t>(s.n_img, d, vox, sms, st, p); break;
    default: rc = launch_vx<int16_t>(s.n_img, d, vox, sms, st, p); break;
  }
  if (rc < 0) return DPM_OK;   // TMA could not describe it: generic kernel
  note_launches(1);
  *handled = true;
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
