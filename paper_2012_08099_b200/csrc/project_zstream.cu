// project_zstream.cu -- the moments pipeline's projection pass, streaming along z.
//
// Replaces projection._accumulate (projection.py:139-186) for dpm_moments.  The
// moments pipeline needs projections only as an intermediate (their 2D moments
// are recombined into the 3D moments), so it is free to choose WHICH
// projections to build.  It builds the reference method's image set of the
// volume with x and z exchanged ("layout T"):
//
//   slot XY   (z, y)   sum over x        stored [y][z]          W = N
//   slot YZ   (y, x)   sum over z        stored [x][y]          W = M, H = L
//   DIAG      z + x         (s = +1)     stored [y][z + x]
//   ANTI      z - x         (s = -1)     stored [y][z - x + (L-1)]
//   X2P       z + 2x        (s = +2)     stored [y][z + 2x]                  (orders 5-6)
//   X2M       z - 2x        (s = -2)     stored [y][z - 2x + 2(L-1)]         (order 6)
//   profile   z + s_P x, summed over y   s_P = -1, 2, -2, 3 at orders 3..6
//
// i.e. exactly the images dpm_project would build for the volume V'(x', y, z')
// = V(z', y, x'); the 2D moments and the epilogue are the classic ones with
// the output relabelled M_pqr = M'_rqp (derive_dev.cuh).
//
// Why z: every oblique form here is z + s x, so as a lane's 8-plane patch
// advances one step in z, its register window over the form's cells slides
// by exactly 8 cells whatever s is.  The 8 cells that leave the window are
// complete for that lane and are emitted (8 shared atomics per form per step,
// 0.125 per voxel -- vs 0.23-0.34 for a per-row-step window), and nothing
// about the window depends on the other warps:
//
//   CTA      = NW warps; warp w owns image row y = Y0 + w (one y per warp), all
//              warps share the column's x-tile (SX = 32 VX voxels) and z range.
//   step     = 8 planes: ONE 4-D TMA box (x SX, y NW, z 8, b 1) per step into a
//              STAGES-deep ring with full/empty mbarriers.  No CTA barrier per
//              step: each warp releases a stage by arriving on its empty
//              barrier as soon as the step's last planes are in registers
//              (mid-step); thread 0 refills the stage at the end of its own
//              step once all warps released it, so warps drift freely within
//              the ring.
//   lane     = VX consecutive x of the warp's row, 8 planes per step.
//   forms    = register windows of 8 + |s|(VX-1) cells, slid by 8 cells per
//              step; the 8 completed cells go to a warp-private ring of image
//              cells in shared memory (red.shared, conflict-free: the 32 lanes'
//              blocks are consecutive ring slots), and the warp flushes the one
//              ring block that completes per step to global memory (8 cells per
//              form, red.global).  The profile window goes to a CTA-shared
//              ring (it is summed over the warps' y), flushed block by block
//              by the warps in turn once every warp is past the block.
//   XY slot  = per-plane lane sums, one warp redux per plane, 8 plane sums of
//              row y per step (red.global, partial over x-tiles).
//   YZ slot  = the lane's VX x-sums over all planes of the segment (registers),
//              flushed at the end of the segment.
// Work split: the (column, step) space (a column = one (volume, y-group,
// x-tile), a step = 8 of its planes) is cut into equal contiguous runs, one
// per persistent CTA; a segment = the part of a run inside one column.
// Exactness: uint32 ray sums (the C ABI rejects shapes whose longest ray could
// reach 2^32), integer atomics: order independent, bit-identical.
#include <cudaTypedefs.h>
#include <atomic>
#include <mutex>
#include "dpm_common.cuh"
#include "ptx.cuh"

#ifndef DPM_ZS_HALF
#define DPM_ZS_HALF 1   // orders 5-6: windows spanning one fold group, emitted per group, 12 warps (v33)
#endif
#ifndef DPM_ZS_CTAS6
#define DPM_ZS_CTAS6 1   // CTAs per SM at orders 5-6
#endif
__host__ __device__ constexpr int zs_ctas(int K) { return K >= 5 ? DPM_ZS_CTAS6 : 1; }
#ifndef DPM_ZS_XY_SMEM
#define DPM_ZS_XY_SMEM 1   // XY-slot plane sums through a per-warp shared word each instead of lane selects (x37)
#endif
#ifndef DPM_ZS_SLEEP
#define DPM_ZS_SLEEP 0   // suspend-time hint (ns) of the stage waits; 0 = plain try_wait polling
#endif
#ifndef DPM_ZS_HALF_MINK
#define DPM_ZS_HALF_MINK 5   // lowest order that uses the group-wise windows
#endif
#ifndef DPM_ZS_SPLIT
#define DPM_ZS_SPLIT 0   // group-wise windows: fetch each step as two half boxes with their own barriers
#endif
__host__ __device__ constexpr int zs_spl(int K) { return (DPM_ZS_SPLIT && DPM_ZS_HALF && K >= DPM_ZS_HALF_MINK) ? 2 : 1; }
#ifndef DPM_ZS_NW34
#define DPM_ZS_NW34 12       // warps per CTA at orders 3-4
#endif
#ifndef DPM_ZS_XT_MAJOR_MB
#define DPM_ZS_XT_MAJOR_MB 96   // image sets above this size (MB): columns ordered x-tile outermost (v39)
#endif
#ifndef DPM_ZS_EARLY_REL
#define DPM_ZS_EARLY_REL 1   // release a stage once the step's last plane group is in registers, refill it at the step's end (x42: cfg5 -3 %)
#endif

#ifndef DPM_ZS_CS_FMA
#define DPM_ZS_CS_FMA 0   // YZ-slot x sums with IMAD-by-1 (FMA pipe) instead of 3-input adds
#endif
#ifndef DPM_ZS_XY_IDP
#define DPM_ZS_XY_IDP 1   // XY-slot plane sums by IDP dot products on the FMA pipe (x30: cfg5 -1 %)
#endif
#include <type_traits>
#ifndef DPM_ZS_GP
#define DPM_ZS_GP 4   // planes per fold group when a |s| >= 2 form is folded on the ALU pipe
#endif

namespace dpm {

// profile direction s_P of layout T by order (the transposed classic t)
__host__ __device__ constexpr int zs_prof_s(int K) { return K <= 3 ? -1 : K == 4 ? 2 : K == 5 ? -2 : 3; }
__host__ __device__ constexpr int zs_form_s(int j) { return j == 0 ? 1 : j == 1 ? -1 : j == 2 ? 2 : -2; }
__host__ __device__ constexpr int zs_abs(int v) { return v < 0 ? -v : v; }

struct ZParams {
  int64_t L, M, N, B;
  int32_t offset;
  int32_t n_xt, n_yg, ns;        // x-tiles, y-groups, z-steps per column
  int64_t ncol;                  // B * n_yg * n_xt
  int32_t yb;                    // column order: y-groups per block (zdecode)
  uint32_t one;                  // == 1 at run time (IMAD-by-1 folds on the FMA pipe)
  uint32_t* img[DPM_MAX_IMAGES];
  int64_t W[DPM_MAX_IMAGES];     // stored widths (layout T)
  unsigned long long* prof;      // [B][WQ]
  int64_t WQ;
};

// ---- geometry ---------------------------------------------------------------
template <int AS> struct Ring {
  static constexpr int R = 32 * AS;     // logical blocks (>= live span 31 AS + 1)
  static constexpr int RP = R + 1;      // word stride between cell rows (conflict-free flush)
  static constexpr int WORDS = 8 * RP;
  // slot index of block b: lanes' blocks n + AS l map to consecutive slots
  static __device__ __forceinline__ int idx(int b) {
    const uint32_t m = (uint32_t)b % (uint32_t)R;
    return (int)((m % AS) * 32 + m / AS);
  }
};
// CTA profile ring: live span 31 AS + 1 plus the warps' drift (< STAGES steps)
// plus the flush lag (a block is flushed STAGES, with early release STAGES + 1, steps after it completes).
// R is a power of two (a multiple of 32): for odd AS the lanes' blocks n + AS l
// are 32 distinct banks as they are; for AS = 2 the two parity classes are
// split into halves (slot (m & 1) R/2 + m/2), so no division by AS at all
__host__ __device__ constexpr int zs_pow2_at_least(int v) { int r = 32; while (r < v) r *= 2; return r; }
template <int AS, int STAGES> struct PRing {
  static constexpr int R = zs_pow2_at_least(32 * AS + 2 * STAGES + 4);
  static constexpr int RP = R + 1;
  static constexpr int WORDS = 8 * RP;
  static __device__ __forceinline__ int idx(int b) {
    const uint32_t m = (uint32_t)b & (uint32_t)(R - 1);
    if constexpr (AS % 2 == 1) return (int)m;
    else return (int)((m & 1u) * (R / 2) + (m >> 1));
  }
};

template <typename T, int K, int NW, int VX, int STAGES> struct ZGeo {
  static constexpr int NOB = K <= 3 ? 1 : K - 2;               // oblique images (DIAG, ANTI, X2P, X2M)
  static constexpr int SP = zs_prof_s(K), ASP = zs_abs(SP);
  static constexpr int SX = 32 * VX;
  static constexpr int STAGE_BYTES = SX * NW * 8 * (int)sizeof(T);
  static constexpr int ring_words(int j) { return 8 * (32 * zs_abs(zs_form_s(j)) + 1); }
  static constexpr int ring_off(int j) { int o = 0; for (int i = 0; i < j; ++i) o += ring_words(i); return o; }
  static constexpr int WARP_RING = ring_off(NOB);               // words per warp
  static constexpr int PR_WORDS = PRing<ASP, STAGES>::WORDS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + (size_t)NW * WARP_RING * 4 + PR_WORDS * 4 + 8 +
                                 4 * STAGES * 8 + 128 + 64 * NW + 96 * STAGES + 32 * NW + 16;   // + producer state, cursors, XY-slot sums
};

// ---- lane vectors ------------------------------------------------------------
// s16: int16 voxels summed SIGNED, without the offset (dpm_moments adds
// offset x the box's moments to the 3D moments exactly; capi.cu "signed-exact
// int16"): cells hold two's-complement sums mod 2^32, the profile is sign-extended
struct s16 { int16_t v; };
template <typename T> struct ZSigned { static constexpr bool value = false; };
template <> struct ZSigned<s16> { static constexpr bool value = true; };
// a shared-memory u32 cell as the uint64 the profile atomics add
template <typename T> __device__ __forceinline__ unsigned long long zprof64(uint32_t v) {
  if constexpr (ZSigned<T>::value) return (unsigned long long)(long long)(int32_t)v;
  else return (unsigned long long)v;
}

template <typename T, int VX> struct ZVec;
template <> struct ZVec<uint16_t, 8> { using type = uint4; };
template <> struct ZVec<s16, 8>      { using type = uint4; };
template <> struct ZVec<int16_t, 8>  { using type = uint4; };
template <> struct ZVec<uint8_t, 8>  { using type = uint2; };

template <typename T> struct ZUnpack;
// 16-bit halves by PRMT: one ALU op per voxel that ptxas does not fuse into the
// adds (a plain shift becomes LEA.HI acc + (w >> 16) at EVERY use: one 2-input
// add per voxel-add instead of 3-input pairs)
#ifndef DPM_ZS_UNPACK_FMA
#define DPM_ZS_UNPACK_FMA 0
#endif
// DPM_ZS_UNPACK_FMA: the halves on the FMA pipe instead -- hi = mul.hi(w, 2^16),
// lo = w - hi * 2^16 (a run-time 2^16 keeps ptxas from turning them back into
// shifts): the folds saturate the ALU pipe, the FMA pipe idles
template <> struct ZUnpack<uint16_t> {
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t, uint32_t k16) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (DPM_ZS_UNPACK_FMA == 1) {
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(v[2 * i + 1]) : "r"(w[i]), "r"(k16));
        v[2 * i] = ptx::mad_u32(v[2 * i + 1], 0u - k16, w[i]);
      } else if (DPM_ZS_UNPACK_FMA == 2) {   // hi on the FMA pipe, lo on the ALU pipe
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(v[2 * i + 1]) : "r"(w[i]), "r"(k16));
        asm("prmt.b32 %0, %1, 0, 0x4410;" : "=r"(v[2 * i]) : "r"(w[i]));
      } else {
        asm("prmt.b32 %0, %1, 0, 0x4410;" : "=r"(v[2 * i]) : "r"(w[i]));
        asm("prmt.b32 %0, %1, 0, 0x4432;" : "=r"(v[2 * i + 1]) : "r"(w[i]));
      }
    }
  }
};
template <> struct ZUnpack<int16_t> {   // sign-extend, add the offset (0 for zero-filled voxels)
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t off, uint32_t) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t lo;
      asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(lo) : "r"(w[i]));
      v[2 * i] = lo + (uint32_t)off;
      v[2 * i + 1] = (uint32_t)((int32_t)w[i] >> 16) + (uint32_t)off;
    }
  }
};
template <> struct ZUnpack<s16> {   // sign-extend only: both halves by PRMT with sign replication
  // (an arithmetic shift for the high half is fused into EVERY add that uses it
  // as LEA.HI.SX32, a 2-input add: twice the adds of the 3-input pairs)
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t, uint32_t) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(v[2 * i]) : "r"(w[i]));
      asm("prmt.b32 %0, %1, 0, 0xBB32;" : "=r"(v[2 * i + 1]) : "r"(w[i]));
    }
  }
};
template <> struct ZUnpack<uint8_t> {
  template <typename V> __device__ __forceinline__ static void run(const V& d, uint32_t* v, int32_t, uint32_t) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&d);
    #pragma unroll
    for (int i = 0; i < 2; ++i) {
      #pragma unroll
      for (int j = 0; j < 4; ++j) v[4 * i + j] = __byte_perm(w[i], 0u, 0x4440u + j);
    }
  }
};

// window cell of voxel (plane t of the step, lane element k) for form s
template <int S, int VX> __device__ __forceinline__ constexpr int zcell(int t, int k) {
  return t + zs_abs(S) * (S > 0 ? k : VX - 1 - k);
}

// Fold a group of GP planes (P[g][k], planes t0 + g) into the window of form S.
// FMA = true: single IMAD-by-1 adds (FMA pipe); else the contributions of a
// cell are summed with 3-input adds (ALU pipe).
template <int S, int VX, int GP, bool FMA, int NWIN>
__device__ __forceinline__ void zfold(uint32_t (&win)[NWIN], const uint32_t (&P)[GP][VX], int t0, uint32_t one) {
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) {
    if constexpr (FMA) {
      #pragma unroll
      for (int g = 0; g < GP; ++g) {
        #pragma unroll
        for (int k = 0; k < VX; ++k)
          if (zcell<S, VX>(t0 + g, k) == c) win[c] = ptx::mad_u32(P[g][k], one, win[c]);
      }
    } else {
      uint32_t acc = win[c];
      uint32_t pend = 0;
      bool have = false;
      #pragma unroll
      for (int g = 0; g < GP; ++g) {
        #pragma unroll
        for (int k = 0; k < VX; ++k) {
          if (zcell<S, VX>(t0 + g, k) == c) {
            if (have) { acc = acc + pend + P[g][k]; have = false; }
            else { pend = P[g][k]; have = true; }
          }
        }
      }
      if (have) acc += pend;
      win[c] = acc;
    }
  }
}

// emit window cells [0, 8) of form S into ring slots of block (n + AS l'),
// then slide the window by 8 cells
template <int S, int NWIN, typename RingT>
__device__ __forceinline__ void zemit_slide(uint32_t (&win)[NWIN], uint32_t ring_addr, int blk) {
  const uint32_t a = ring_addr + 4u * (uint32_t)RingT::idx(blk);
  #pragma unroll
  for (int k = 0; k < 8; ++k) ptx::red_shared_add_dyn(a + 4u * (uint32_t)(k * RingT::RP), win[k]);
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) win[c] = c + 8 < NWIN ? win[c + 8] : 0u;
}

// emit ALL window cells (segment end), cell c into block blk + c/8
template <int S, int NWIN, typename RingT>
__device__ __forceinline__ void zemit_all(uint32_t (&win)[NWIN], uint32_t ring_addr, int blk) {
  #pragma unroll
  for (int c = 0; c < NWIN - 8; ++c) {   // cells [NWIN-8, NWIN) are zero after the last slide
    if (win[c] != 0)
      ptx::red_shared_add_dyn(ring_addr + 4u * (uint32_t)(RingT::idx(blk + c / 8) + (c % 8) * RingT::RP), win[c]);
  }
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) win[c] = 0;
}

// ---- windows as rings of 8-cell blocks ------------------------------------------
// A form's register window is NB blocks of 8 cells; logical block j of the
// window at step phase R (= step mod ZU) lives in physical block (j + R) mod NB.
// The step loop is unrolled ZU times, so every index is a compile-time constant
// and the window slides by one block per step without a single register move
// (the emitted block becomes the window's last block).  NB divides ZU.
// DPM_ZS_UNROLL = 1 keeps one loop body and slides the windows with register
// moves (measured faster: the 4-phase body overflows the instruction cache --
// ncu no_instruction stalls 1.0 per issue -- and costs more than the ~60 moves
// per step it saves; tools/EXPERIMENTS.md z7)
#ifndef DPM_ZS_UNROLL
#define DPM_ZS_UNROLL 1
#endif
constexpr int ZU = DPM_ZS_UNROLL;
__host__ __device__ constexpr int zs_nb(int as) { return ZU == 1 ? (as == 1 ? 2 : as == 2 ? 3 : 4) : (as == 1 ? 2 : 4); }
template <int NB, int R> __device__ __forceinline__ constexpr int zphys(int c) { return (((c >> 3) + R) % NB) * 8 + (c & 7); }

template <int S, int VX, int GP, bool FMA, int NB, int R>
__device__ __forceinline__ void zfold_r(uint32_t (&win)[NB * 8], const uint32_t (&P)[GP][VX], int t0, uint32_t one) {
  constexpr int NWIN = 8 + zs_abs(S) * (VX - 1);
  static_assert(NWIN <= NB * 8, "window ring too small");
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) {
    const int pc = zphys<NB, R>(c);
    if constexpr (FMA) {
      #pragma unroll
      for (int g = 0; g < GP; ++g) {
        #pragma unroll
        for (int k = 0; k < VX; ++k)
          if (zcell<S, VX>(t0 + g, k) == c) win[pc] = ptx::mad_u32(P[g][k], one, win[pc]);
      }
    } else {
      uint32_t acc = win[pc];
      uint32_t pend = 0;
      bool have = false;
      #pragma unroll
      for (int g = 0; g < GP; ++g) {
        #pragma unroll
        for (int k = 0; k < VX; ++k) {
          if (zcell<S, VX>(t0 + g, k) == c) {
            if (have) { acc = acc + pend + P[g][k]; have = false; }
            else { pend = P[g][k]; have = true; }
          }
        }
      }
      if (have) acc += pend;
      win[pc] = acc;
    }
  }
}
// emit logical block 0 (8 red.shared into ring block blk) and clear it: it is the
// window's last block at the next phase
template <int NB, int R, typename RingT>
__device__ __forceinline__ void zemit_r(uint32_t (&win)[NB * 8], uint32_t ring_addr, int blk) {
  const uint32_t a = ring_addr + 4u * (uint32_t)RingT::idx(blk);
  #pragma unroll
  for (int k = 0; k < 8; ++k) {
    ptx::red_shared_add_dyn(a + 4u * (uint32_t)(k * RingT::RP), win[zphys<NB, R>(k)]);
    win[zphys<NB, R>(k)] = 0u;
  }
  if constexpr (ZU == 1) {   // one loop body: slide by 8 cells with moves
    #pragma unroll
    for (int c = 0; c < NB * 8; ++c) win[c] = c + 8 < NB * 8 ? win[c + 8] : 0u;
  }
}
// segment end at phase R: emit every remaining cell, logical cell c into block blk + c/8
template <int S, int VX, int NB, int R, typename RingT>
__device__ __forceinline__ void zemit_all_r(uint32_t (&win)[NB * 8], uint32_t ring_addr, int blk) {
  constexpr int NWIN = 8 + zs_abs(S) * (VX - 1);
  #pragma unroll
  for (int c = 0; c < NWIN - 8; ++c) {
    const uint32_t v = win[zphys<NB, R>(c)];
    if (v != 0) ptx::red_shared_add_dyn(ring_addr + 4u * (uint32_t)(RingT::idx(blk + c / 8) + (c % 8) * RingT::RP), v);
  }
  #pragma unroll
  for (int c = 0; c < NB * 8; ++c) win[c] = 0u;
}

// ---- group-wise windows (DPM_ZS_HALF) -------------------------------------------
// The window of a form only has to span ONE fold group of GP planes: after the
// group, its first GP cells are complete for this lane (every later plane of
// the step lands at a higher cell), so they are emitted -- ring rows GP h ..
// GP h + GP - 1 of the step's block -- and the window slides by GP cells.
// GP + |s|(VX - 1) cells instead of 8 + |s|(VX - 1): the order-6 windows need
// 83 registers instead of 103, which lets 12 warps (3 per scheduler) fit.
template <int S, int VX, int GP> __host__ __device__ constexpr int zs_gwin() { return GP + zs_abs(S) * (VX - 1); }
template <int GP, int NWIN, typename RingT>
__device__ __forceinline__ void zemit_group(uint32_t (&win)[NWIN], uint32_t ring_addr, int blk, int h) {
  const uint32_t a = ring_addr + 4u * (uint32_t)RingT::idx(blk);
  #pragma unroll
  for (int k = 0; k < GP; ++k) ptx::red_shared_add_dyn(a + 4u * (uint32_t)((GP * h + k) * RingT::RP), win[k]);
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) win[c] = c + GP < NWIN ? win[c + GP] : 0u;
}
// segment end (after the last group's slide): cells [0, 7|s|) belong to blocks blk + c / 8
template <int S, int VX, int NWIN, typename RingT>
__device__ __forceinline__ void zemit_group_tail(uint32_t (&win)[NWIN], uint32_t ring_addr, int blk) {
  #pragma unroll
  for (int c = 0; c < zs_abs(S) * (VX - 1); ++c) {
    const uint32_t v = win[c];
    if (v != 0) ptx::red_shared_add_dyn(ring_addr + 4u * (uint32_t)(RingT::idx(blk + c / 8) + (c % 8) * RingT::RP), v);
  }
  #pragma unroll
  for (int c = 0; c < NWIN; ++c) win[c] = 0u;
}

// Segment iterator shared by the producer and the consumers: the CTA's
// sequence of (column, n0, n1) step ranges -- its equal contiguous run of the
// flattened (column, step) space, cut at the column ends.  All of it fits 32
// bits (a step is >= 16 KB of voxels: 2^31 steps would be 32 TB), and must:
// a 64-bit division is a ~100-instruction call, and call sites inside the
// step loop cost the whole loop registers (x47: cfg5 pass -4 %)
struct ZSeg {
  uint32_t col;
  int32_t n0, n1;
  uint32_t pos, end;     // position in the flattened step space, end of the run
  bool done;
  __device__ __forceinline__ void first(const ZParams& p) {
    const uint64_t W = (uint64_t)p.ncol * (uint64_t)p.ns;
    pos = (uint32_t)(W * blockIdx.x / gridDim.x);
    end = (uint32_t)(W * (blockIdx.x + 1) / gridDim.x);
    set_run(p);
  }
  __device__ __forceinline__ void next(const ZParams& p) {
    pos += (uint32_t)(n1 - n0);
    set_run(p);
  }
  __device__ __forceinline__ void set_run(const ZParams& p) {
    done = pos >= end;
    if (done) return;
    col = pos / (uint32_t)p.ns;
    n0 = (int32_t)(pos - col * (uint32_t)p.ns);
    n1 = (int32_t)umin((uint32_t)p.ns, (uint32_t)n0 + (end - pos));
  }
};

// producer state (thread 0's refill cursor), kept in shared memory to spare registers
struct ZProd {
  ZSeg seg;
  int32_t n, k;          // next step to issue (within seg), its stage (sub-stage with DPM_ZS_SPLIT)
  int32_t xt, yg, b;     // decoded column of seg
  int32_t hh;            // next half of step n (DPM_ZS_SPLIT)
};
// Column order: volume, then blocks of p.yb y-groups, then the x-tile, then the
// y-group inside the block.  yb = 1 is x-tile innermost: a CTA's run walks the
// x-tiles of one y-group one after the other (they add into the same image
// rows a column later; fine while the image set fits in L2).  For larger image
// sets the x-tiles of a y-group should run on DIFFERENT CTAs at the SAME time,
// so that a row's partial sums meet in L2: two columns run simultaneously when
// their indices differ by a multiple of the run length R = ncol / grid, so the
// host picks yb = round(m R) for the small m with the least rounding error
// (cfg5: R = 9.24, yb = 37 = 4.003 R); yb = n_yg is plain x-tile-outermost order.
__device__ __forceinline__ void zdecode(const ZParams& p, uint32_t col, int32_t& xt, int32_t& yg, int32_t& b) {
  const uint32_t per_vol = (uint32_t)p.n_yg * (uint32_t)p.n_xt;
  const uint32_t bb = col / per_vol, c = col - bb * per_vol;
  const uint32_t per_blk = (uint32_t)p.yb * (uint32_t)p.n_xt;
  const uint32_t blk = c / per_blk, w = c - blk * per_blk;
  const uint32_t ybt = umin((uint32_t)p.yb, (uint32_t)p.n_yg - blk * (uint32_t)p.yb);   // the last block may be short
  const uint32_t x = w / ybt;
  xt = (int32_t)x;
  yg = (int32_t)(blk * (uint32_t)p.yb + (w - x * ybt));
  b = (int32_t)bb;
}

// Who refills a stage (DPM_ZS_PWARP):
//   0: thread 0, for stage g - ZLAG, from inside its own step loop (waits on
//      the stage's empty mbarrier);
//   1: one extra warp that only produces (refills a stage the moment the last
//      compute warp releases it) -- costs a register-file quarter per SMSP;
//   2: the compute warp that releases a stage LAST refills it (per-stage release
//      counters; every stage has its own cursor, advanced STAGES steps per use,
//      so refills of different stages never share state).
#ifndef DPM_ZS_PWARP
#define DPM_ZS_PWARP 0   // measured: 1 spills (the fourth warp per SMSP caps registers at 168), 2 is 8 % slower (x25)
#endif
constexpr int ZPW = DPM_ZS_PWARP == 1 ? 1 : 0;
constexpr bool ZLAST = DPM_ZS_PWARP == 2;

// barrier over the NW compute warps only (the producer warp never joins it)
template <int NW> __device__ __forceinline__ void zs_sync() {
  if constexpr (ZPW) asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
  else __syncthreads();
}

template <typename T, int K, int NW, int VX, int STAGES, int FMAMASK>
__global__ void __launch_bounds__(32 * (NW + ZPW), zs_ctas(K)) zstream_kernel(const __grid_constant__ CUtensorMap tmap, const ZParams p) {
  using G = ZGeo<T, K, NW, VX, STAGES>;
  using V = typename ZVec<T, VX>::type;
  constexpr int NOB = G::NOB, SX = G::SX;
  constexpr int SP = G::SP, ASP = G::ASP;
  constexpr int S0 = zs_form_s(0), S1 = zs_form_s(1), S2 = zs_form_s(2), S3 = zs_form_s(3);
  constexpr int NW0 = 8 + zs_abs(S0) * (VX - 1), NW1 = 8 + zs_abs(S1) * (VX - 1);
  constexpr int NW2 = 8 + zs_abs(S2) * (VX - 1), NW3 = 8 + zs_abs(S3) * (VX - 1);
  constexpr int NWP = 8 + ASP * (VX - 1);
  // planes per fold group: 3-input pairs are planes (t, t+1) for |s| = 1, (t, t+2)
  // for |s| = 2, (t, t+3) for |s| = 3 -- groups of 4 when a form with |s| >= 2 is
  // folded on the ALU pipe, 2 (fewer live registers) when those go to the FMA pipe
  constexpr int GP = (NOB <= 2 || (FMAMASK & 12) == 12) && ((FMAMASK & 16) || ASP == 1) ? 2 : DPM_ZS_GP;
  constexpr bool HALF = DPM_ZS_HALF && K >= DPM_ZS_HALF_MINK;   // group-wise windows (see zemit_group)
  // DPM_ZS_SPLIT: each step's box is fetched as two half boxes of 4 planes with
  // their own barriers, one per fold group: a half-stage is released (and
  // refilled) after its group, half a step earlier than a whole stage
  constexpr int SPL = zs_spl(K);
  static_assert(SPL == 1 || (HALF && GP == 4), "half-box stages need the 4-plane group-wise windows");
  constexpr int NSUB = STAGES * SPL;
  constexpr uint32_t SUB_BYTES = G::STAGE_BYTES / SPL;
  constexpr int PPS = 8 / SPL;   // planes per (sub-)stage
  using PR = PRing<ASP, STAGES>;
  constexpr uint32_t R0 = G::ring_off(0) * 4, R1 = G::ring_off(1) * 4, R2 = G::ring_off(2) * 4,
                     R3 = G::ring_off(3) * 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint32_t* rings = reinterpret_cast<uint32_t*>(smem + (size_t)STAGES * G::STAGE_BYTES);
  uint32_t* pring = rings + NW * G::WARP_RING;
  uint64_t* full = reinterpret_cast<uint64_t*>(pring + G::PR_WORDS + ((G::PR_WORDS & 1) ? 1 : 0));
  uint64_t* empty = full + NSUB;
  ZProd* prod = reinterpret_cast<ZProd*>(empty + NSUB);     // producer state (thread 0 only)
  ZSeg* segs = reinterpret_cast<ZSeg*>(prod + 1);            // [NW] each warp's segment cursor
  ZProd* prods = reinterpret_cast<ZProd*>(segs + NW);        // [STAGES] per-stage cursors (ZLAST)
  uint32_t* rel = reinterpret_cast<uint32_t*>(prods + STAGES);   // [STAGES] release counters (ZLAST)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t* xyv = rel + STAGES + 8 * w;                          // [NW][8] this warp's XY-slot plane sums

  if (w < NW)
    for (int i = tid; i < NW * G::WARP_RING + G::PR_WORDS; i += 32 * NW) rings[i] = 0;
  auto issue = [&]() {   // thread 0: the next step (half step with SPL = 2) of the sequence into its stage
    ZProd st = *prod;
    if (st.seg.done) return;
    const int k = st.k;
    ptx::mbar_arrive_expect_tx(&full[k], SUB_BYTES);
    ptx::tma_load_4d_hint(stages + (size_t)k * SUB_BYTES, &tmap, &full[k], st.xt * SX, st.yg * NW, st.n * 8 + PPS * st.hh,
                          st.b, ptx::policy_evict_first());
    st.k = k + 1 == NSUB ? 0 : k + 1;
    if (SPL == 2 && st.hh == 0) { st.hh = 1; *prod = st; return; }
    st.hh = 0;
    if (++st.n == st.seg.n1) {
      st.seg.next(p);
      if (!st.seg.done) { st.n = st.seg.n0; zdecode(p, st.seg.col, st.xt, st.yg, st.b); }
    }
    *prod = st;
  };
  auto advance1 = [&](ZProd& st) {
    if (st.seg.done) return;
    if (++st.n == st.seg.n1) {
      st.seg.next(p);
      if (!st.seg.done) { st.n = st.seg.n0; zdecode(p, st.seg.col, st.xt, st.yg, st.b); }
    }
  };
  // ZLAST: stage k's cursor -> TMA into stage k, then advance it STAGES steps
  auto issue_stage = [&](int k) {
    ZProd st = prods[k];
    if (st.seg.done) return;
    ptx::mbar_arrive_expect_tx(&full[k], G::STAGE_BYTES);
    ptx::tma_load_4d_hint(stages + (size_t)k * G::STAGE_BYTES, &tmap, &full[k], st.xt * SX, st.yg * NW, st.n * 8,
                          st.b, ptx::policy_evict_first());
    #pragma unroll 1
    for (int i = 0; i < STAGES; ++i) advance1(st);
    prods[k] = st;
  };
  if (tid == 0) {
    ptx::prefetch_tmap(&tmap);
    for (int i = 0; i < NSUB; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], NW); }
    ptx::fence_barrier_init();
    ZProd st;
    st.k = 0;
    st.hh = 0;
    st.seg.first(p);
    if (!st.seg.done) { st.n = st.seg.n0; zdecode(p, st.seg.col, st.xt, st.yg, st.b); }
    if constexpr (ZLAST) {
      for (int h = 0; h < STAGES; ++h) { prods[h] = st; rel[h] = 0; advance1(st); }
      for (int h = 0; h < STAGES; ++h) issue_stage(h);
    } else {
      *prod = st;
      for (int h = 0; h < NSUB; ++h) issue();
    }
  }
  if (lane == 0 && w < NW) segs[w].first(p);
  pdl_trigger();    // the moments launch may start its prologue while this grid drains
  __syncthreads();
  pdl_wait();       // images / profile zeroed by the preceding kernel (the first TMA loads are in flight)
  if constexpr (ZPW) {
    if (w == NW) {   // producer warp: refill each stage as soon as every compute warp released it
      if (lane == 0) {
        int kk = 0;
        uint32_t ph = 0;
        while (!prod->seg.done) {
          ptx::mbar_wait_addr(ptx::smem_addr(empty) + 8u * (uint32_t)kk, ph);
          issue();
          if (++kk == NSUB) { kk = 0; ph ^= 1u; }
        }
      }
      return;
    }
  }

  const uint32_t bar_a = ptx::smem_addr(full);               // full[k] at +8k, empty[k] at +8(STAGES + k)
  const uint32_t wring_a = ptx::smem_addr(rings + w * G::WARP_RING);
  const uint32_t pring_a = ptx::smem_addr(pring);
  const uint32_t stage_a = ptx::smem_addr(stages) + 2u * (uint32_t)(w * SX + VX * lane) * (uint32_t)sizeof(T) / 2u;
  // this lane's share of the per-step ring flush: form fj, cell fk of the completed block
  const int fj = lane >> 3, fk = lane & 7;
  const int fas = fj < 2 ? 1 : 2;                     // |s| of form fj
  const uint32_t fring_a = wring_a + (fj == 0 ? R0 : fj == 1 ? R1 : fj == 2 ? R2 : R3) + 4u * (uint32_t)(fk * (32 * fas + 1));
  const int lpp = lane, lpm = 31 - lane;             // lane l' of forms with s > 0 / s < 0

  // step counter (all warps): step g in stage k / phase ph; step g - ZLAG in stage kl /
  // phase phl; warp pw flushes the profile block of step g
#ifndef DPM_ZS_ZLAG
#define DPM_ZS_ZLAG (K >= 6 ? 2 : 1)   // measured best per order (x26)
#endif
  // early release: the stage goes back to the producer once the step's last
  // plane group is in registers, half a step before the step ends
  constexpr bool EREL = DPM_ZS_EARLY_REL && zs_spl(K) == 1 && !ZLAST && !ZPW;
  // ... and thread 0 refills it at the END of its own step (lag 0: it only waits
  // for warps more than half a step behind it); without early release the
  // refill is at the step's top, ZLAG steps behind
  constexpr int ZLAG = EREL ? 0 : STAGES >= 4 ? DPM_ZS_ZLAG : 1;
  // a refilled stage proves every warp RELEASED step g - STAGES; released early,
  // that only proves step g - STAGES - 1 was emitted completely
  constexpr int PLAG = STAGES + (EREL ? 1 : 0);
  constexpr int ZLAGS = ZLAG * SPL;   // the same lag in sub-stages
  static_assert(sizeof(ZProd) <= 96, "stage cursor budget (ZGeo::SMEM)");
  int k = 0, pw = 0, kl = 0, lagc = 0;
  uint32_t ph = 0, phl = 0;
  while (true) {
    const ZSeg seg = segs[w];
    if (seg.done) break;
    int32_t xt, yg, bi;
    zdecode(p, seg.col, xt, yg, bi);
    const int64_t b = bi;
    const int32_t X0 = xt * SX;
    const int32_t y = yg * NW + w;
    const bool yok = y < p.M;
    const int32_t xl = X0 + VX * lane;          // lane's first x
    const int32_t Zs = 8 * seg.n0;
    const int32_t n0 = seg.n0, nsteps = seg.n1 - seg.n0;
    // global cell index of local cell 0, per form (s > 0: Zs + s X0; s < 0: Zs + |s|(L - X0 - SX))
    auto base_of = [&](int s) -> int32_t { return s > 0 ? Zs + s * X0 : Zs + (-s) * ((int32_t)p.L - X0 - SX); };
    const int64_t rowid = b * p.M + y;
    const int32_t off_lane = (xl < p.L && yok) ? p.offset : 0;
    // per-lane flush targets of this segment
    const int32_t fW = fj < NOB ? (int32_t)p.W[DPM_IMG_DIAG + fj] : 0;
    uint32_t* const frow = fj < NOB && yok ? p.img[DPM_IMG_DIAG + fj] + rowid * fW : nullptr;
    const int32_t fi0 = base_of(zs_form_s(fj)) + fk;
    uint32_t* const xyrow = lane < 8 && yok ? p.img[DPM_IMG_XY] + rowid * p.N + Zs + lane : nullptr;
    // the steps whose flushed cell i = fi0 + 8 rn lies in [0, fW), and whose XY-slot
    // plane z + lane < N: one unsigned compare per step instead of four
    const int32_t frlo = fi0 >= 0 ? 0 : (7 - fi0) / 8;
    const int32_t frhi = frow != nullptr && fW > fi0 ? (fW - fi0 + 7) / 8 : 0;
    const uint32_t frange = frhi > frlo ? (uint32_t)(frhi - frlo) : 0u;
    uint32_t* const fptr = frow != nullptr ? frow + fi0 : nullptr;
    const int32_t xylim = xyrow != nullptr && p.N - Zs - lane > 0 ? (int32_t)((p.N - Zs - lane + 7) / 8) : 0;
    const int32_t pbase = base_of(SP);
    unsigned long long* const prow = p.prof + b * p.WQ;

    constexpr int NB0 = zs_nb(zs_abs(S0)), NB1 = zs_nb(zs_abs(S1)), NB2 = zs_nb(zs_abs(S2)), NB3 = zs_nb(zs_abs(S3));
    constexpr int NBP = zs_nb(ASP);
    constexpr int WS0 = HALF ? zs_gwin<S0, VX, GP>() : NB0 * 8, WS1 = HALF ? zs_gwin<S1, VX, GP>() : NB1 * 8;
    constexpr int WS2 = HALF ? zs_gwin<S2, VX, GP>() : NB2 * 8, WS3 = HALF ? zs_gwin<S3, VX, GP>() : NB3 * 8;
    constexpr int WSP = HALF ? zs_gwin<SP, VX, GP>() : NBP * 8;
    uint32_t w0[WS0], w1[WS1], w2[WS2], w3[WS3], wq[WSP], cs[VX];
    #pragma unroll
    for (int i = 0; i < WS0; ++i) w0[i] = 0;
    #pragma unroll
    for (int i = 0; i < WS1; ++i) w1[i] = 0;
    #pragma unroll
    for (int i = 0; i < WS2; ++i) w2[i] = 0;
    #pragma unroll
    for (int i = 0; i < WS3; ++i) w3[i] = 0;
    #pragma unroll
    for (int i = 0; i < WSP; ++i) wq[i] = 0;
    #pragma unroll
    for (int i = 0; i < VX; ++i) cs[i] = 0;

    // one step (8 planes) at window phase R = rn mod ZU
    // the producer (thread 0): once every warp released sub-stage g - ZLAGS,
    // refill it with sub-step g - ZLAGS + NSUB.  The lag leaves the other warps
    // ZLAGS - 1 sub-steps of slack before the producer waits for the slowest.
    auto produce = [&]() {
      if (!ZPW && !ZLAST && tid == 0) {
        if (lagc >= ZLAGS) {
          ptx::mbar_wait_addr(bar_a + 8u * (uint32_t)(NSUB + kl), phl);
          issue();
          if (++kl == NSUB) { kl = 0; phl ^= 1u; }
        } else {
          ++lagc;
        }
      }
    };
    // step g's (last) sub-stage was refilled only after every warp released
    // step g - STAGES: profile blocks <= rn - PLAG are complete; warp g mod NW
    // flushes that one
    auto flush_profile_block = [&](const int rn) {
      if (w == pw && rn >= PLAG && lane < 8) {
        const int blk = rn - PLAG;
        const uint32_t a = pring_a + 4u * (uint32_t)(PR::idx(blk) + lane * PR::RP);
        const uint32_t v = ptx::lds_u32(a);
        ptx::sts_u32(a, 0u);
        const int32_t i = pbase + 8 * blk + lane;
        if (v != 0 && i >= 0 && i < p.WQ) atomicAdd(prow + i, zprof64<T>(v));
      }
    };
    auto release = [&]() {   // this warp is done with (sub-)stage k
      __syncwarp();
      if (lane == 0) {
        if constexpr (ZLAST) {   // the last of the NW warps to release stage k refills it
          uint32_t old;
          asm volatile("atom.shared.inc.u32 %0, [%1], %2;" : "=r"(old) : "r"(ptx::smem_addr(rel + k)), "r"((uint32_t)(NW - 1)) : "memory");
          if (old == (uint32_t)(NW - 1)) issue_stage(k);
        } else {
          ptx::mbar_arrive_addr(bar_a + 8u * (uint32_t)(NSUB + k));
        }
      }
      if (++k == NSUB) { k = 0; ph ^= 1u; }
    };
    // one step (8 planes) at window phase R = rn mod ZU
    auto step = [&]<int R>(const int rn) {
      const int32_t z = 8 * (n0 + rn);
      uint32_t yzmine = 0;
      uint32_t tile_a = 0;
      if constexpr (SPL == 1) {
        if constexpr (!EREL) produce();
        if constexpr (DPM_ZS_SLEEP > 0) ptx::mbar_wait_addr_sleep(bar_a + 8u * (uint32_t)k, ph, DPM_ZS_SLEEP);
        else ptx::mbar_wait_addr(bar_a + 8u * (uint32_t)k, ph);
        flush_profile_block(rn);
        tile_a = stage_a + (uint32_t)k * G::STAGE_BYTES;
      }
      #pragma unroll
      for (int h = 0; h < 8 / GP; ++h) {
        if constexpr (SPL == 2) {   // group h = half-stage k
          produce();
          ptx::mbar_wait_addr(bar_a + 8u * (uint32_t)k, ph);
          if (h == 1) flush_profile_block(rn);
          tile_a = stage_a + (uint32_t)k * SUB_BYTES;
        }
        uint32_t P[GP][VX];
        V draw[GP];
        #pragma unroll
        for (int gg = 0; gg < GP; ++gg) {
          const int t = GP * h + gg;
          const int ts = SPL == 2 ? gg : t;   // plane within the (sub-)stage
          const V d = ptx::lds_vec<V>(tile_a + (uint32_t)(ts * NW * SX * (int)sizeof(T)));
          draw[gg] = d;
          ZUnpack<T>::run(d, P[gg], z + t < p.N ? off_lane : 0, p.one << 16);
        }
        // XY slot: plane sums over the lane's x, one warp redux per plane
        #pragma unroll
        for (int gg = 0; gg < GP; ++gg) {
          uint32_t sm = 0;
          if constexpr (DPM_ZS_XY_IDP && !std::is_same_v<T, int16_t>) {
            // byte / halfword dot products with ones on the FMA pipe, straight
            // from the packed words (the ALU pipe carries the folds)
            const uint32_t* wd = reinterpret_cast<const uint32_t*>(&draw[gg]);
            if constexpr (ZSigned<T>::value)   // signed halves (sum mod 2^32 == the u32 cell arithmetic)
              sm = (uint32_t)__dp2a_lo((int)wd[0], 0x0101, __dp2a_lo((int)wd[1], 0x0101, __dp2a_lo((int)wd[2], 0x0101, __dp2a_lo((int)wd[3], 0x0101, 0))));
            else if constexpr (sizeof(T) == 2) sm = __dp2a_lo(wd[0], 0x0101u, __dp2a_lo(wd[1], 0x0101u, __dp2a_lo(wd[2], 0x0101u, __dp2a_lo(wd[3], 0x0101u, 0u))));
            else sm = __dp4a(wd[0], 0x01010101u, __dp4a(wd[1], 0x01010101u, 0u));
          } else if constexpr (VX == 8) {
            sm = (P[gg][0] + P[gg][1] + P[gg][2]) + (P[gg][3] + P[gg][4]) + (P[gg][5] + P[gg][6]) + P[gg][7];
          }
          const uint32_t r = __reduce_add_sync(0xffffffffu, sm);
          if constexpr (DPM_ZS_XY_SMEM) ptx::sts_u32(ptx::smem_addr(xyv + GP * h + gg), r);   // uniform value, one word
          else yzmine = lane == GP * h + gg ? r : yzmine;
        }
        if constexpr (EREL) {
          // every plane of the stage has been read AND used (the reductions above
          // consumed each lane's loaded words), so the stage can be refilled now
          if (h == 8 / GP - 1) release();
        }
        // YZ slot: x-sums over z
        #pragma unroll
        for (int kk = 0; kk < VX; ++kk) {
          if constexpr (DPM_ZS_CS_FMA) {
            #pragma unroll
            for (int gg = 0; gg < GP; ++gg) cs[kk] = ptx::mad_u32(P[gg][kk], p.one, cs[kk]);
          } else if constexpr (GP == 4) cs[kk] = cs[kk] + (P[0][kk] + P[1][kk]) + (P[2][kk] + P[3][kk]);
          else cs[kk] = cs[kk] + P[0][kk] + P[GP - 1][kk];
        }
        if constexpr (HALF) {
          // fold the group into windows spanning one group, emit its completed cells, slide
          zfold<S0, VX, GP, (FMAMASK & 1) != 0, WS0>(w0, P, 0, p.one);
          if constexpr (NOB > 1) zfold<S1, VX, GP, (FMAMASK & 2) != 0, WS1>(w1, P, 0, p.one);
          if constexpr (NOB > 2) zfold<S2, VX, GP, (FMAMASK & 4) != 0, WS2>(w2, P, 0, p.one);
          if constexpr (NOB > 3) zfold<S3, VX, GP, (FMAMASK & 8) != 0, WS3>(w3, P, 0, p.one);
          zfold<SP, VX, GP, (FMAMASK & 16) != 0, WSP>(wq, P, 0, p.one);
          if constexpr (SPL == 2) release();   // every value of this half-stage is in registers and used
          zemit_group<GP, WS0, Ring<zs_abs(S0)>>(w0, wring_a + R0, rn + zs_abs(S0) * (S0 > 0 ? lpp : lpm), h);
          if constexpr (NOB > 1) zemit_group<GP, WS1, Ring<zs_abs(S1)>>(w1, wring_a + R1, rn + zs_abs(S1) * (S1 > 0 ? lpp : lpm), h);
          if constexpr (NOB > 2) zemit_group<GP, WS2, Ring<zs_abs(S2)>>(w2, wring_a + R2, rn + zs_abs(S2) * (S2 > 0 ? lpp : lpm), h);
          if constexpr (NOB > 3) zemit_group<GP, WS3, Ring<zs_abs(S3)>>(w3, wring_a + R3, rn + zs_abs(S3) * (S3 > 0 ? lpp : lpm), h);
          zemit_group<GP, WSP, PR>(wq, pring_a, rn + ASP * (SP > 0 ? lpp : lpm), h);
        } else {
          zfold_r<S0, VX, GP, (FMAMASK & 1) != 0, NB0, R % NB0>(w0, P, GP * h, p.one);
          if constexpr (NOB > 1) zfold_r<S1, VX, GP, (FMAMASK & 2) != 0, NB1, R % NB1>(w1, P, GP * h, p.one);
          if constexpr (NOB > 2) zfold_r<S2, VX, GP, (FMAMASK & 4) != 0, NB2, R % NB2>(w2, P, GP * h, p.one);
          if constexpr (NOB > 3) zfold_r<S3, VX, GP, (FMAMASK & 8) != 0, NB3, R % NB3>(w3, P, GP * h, p.one);
          zfold_r<SP, VX, GP, (FMAMASK & 16) != 0, NBP, R % NBP>(wq, P, GP * h, p.one);
        }
      }
      if constexpr (!HALF) {
        // emit the completed cells (block rn + AS l' of each form); the window slides by rotation
        zemit_r<NB0, R % NB0, Ring<zs_abs(S0)>>(w0, wring_a + R0, rn + zs_abs(S0) * (S0 > 0 ? lpp : lpm));
        if constexpr (NOB > 1) zemit_r<NB1, R % NB1, Ring<zs_abs(S1)>>(w1, wring_a + R1, rn + zs_abs(S1) * (S1 > 0 ? lpp : lpm));
        if constexpr (NOB > 2) zemit_r<NB2, R % NB2, Ring<zs_abs(S2)>>(w2, wring_a + R2, rn + zs_abs(S2) * (S2 > 0 ? lpp : lpm));
        if constexpr (NOB > 3) zemit_r<NB3, R % NB3, Ring<zs_abs(S3)>>(w3, wring_a + R3, rn + zs_abs(S3) * (S3 > 0 ? lpp : lpm));
        zemit_r<NBP, R % NBP, PR>(wq, pring_a, rn + ASP * (SP > 0 ? lpp : lpm));
      }
      // XY slot row y: 8 consecutive z (partial over x-tiles)
      if constexpr (DPM_ZS_XY_SMEM) {
        __syncwarp();
        yzmine = lane < 8 ? ptx::lds_u32(ptx::smem_addr(xyv + (lane & 7))) : 0u;
      }
      ptx::red_global_add_if(xyrow + 8 * rn, yzmine, rn < xylim && yzmine != 0);
      __syncwarp();
      // the ring block this step completed: lanes 8j..8j+7 flush form j's 8 cells
      if (fj < NOB) {
        const int m = rn & (32 * fas - 1);
        const uint32_t a = fring_a + 4u * (uint32_t)((m & (fas - 1)) * 32 + (m >> (fas - 1)));
        const uint32_t v = ptx::lds_u32(a);
        ptx::sts_u32(a, 0u);
        ptx::red_global_add_if(fptr + 8 * rn, v, v != 0 && (uint32_t)(rn - frlo) < frange);
      }
      if constexpr (SPL == 1 && !EREL) release();
      else __syncwarp();
      if constexpr (EREL) produce();
      if (++pw == NW) pw = 0;
    };
    auto end_emit = [&]<int R>(const int rn_end) {
      if constexpr (HALF) {
        zemit_group_tail<S0, VX, WS0, Ring<zs_abs(S0)>>(w0, wring_a + R0, rn_end + zs_abs(S0) * (S0 > 0 ? lpp : lpm));
        if constexpr (NOB > 1) zemit_group_tail<S1, VX, WS1, Ring<zs_abs(S1)>>(w1, wring_a + R1, rn_end + zs_abs(S1) * (S1 > 0 ? lpp : lpm));
        if constexpr (NOB > 2) zemit_group_tail<S2, VX, WS2, Ring<zs_abs(S2)>>(w2, wring_a + R2, rn_end + zs_abs(S2) * (S2 > 0 ? lpp : lpm));
        if constexpr (NOB > 3) zemit_group_tail<S3, VX, WS3, Ring<zs_abs(S3)>>(w3, wring_a + R3, rn_end + zs_abs(S3) * (S3 > 0 ? lpp : lpm));
        zemit_group_tail<SP, VX, WSP, PR>(wq, pring_a, rn_end + ASP * (SP > 0 ? lpp : lpm));
      } else {
      zemit_all_r<S0, VX, NB0, R % NB0, Ring<zs_abs(S0)>>(w0, wring_a + R0, rn_end + zs_abs(S0) * (S0 > 0 ? lpp : lpm));
      if constexpr (NOB > 1) zemit_all_r<S1, VX, NB1, R % NB1, Ring<zs_abs(S1)>>(w1, wring_a + R1, rn_end + zs_abs(S1) * (S1 > 0 ? lpp : lpm));
      if constexpr (NOB > 2) zemit_all_r<S2, VX, NB2, R % NB2, Ring<zs_abs(S2)>>(w2, wring_a + R2, rn_end + zs_abs(S2) * (S2 > 0 ? lpp : lpm));
      if constexpr (NOB > 3) zemit_all_r<S3, VX, NB3, R % NB3, Ring<zs_abs(S3)>>(w3, wring_a + R3, rn_end + zs_abs(S3) * (S3 > 0 ? lpp : lpm));
      zemit_all_r<SP, VX, NBP, R % NBP, PR>(wq, pring_a, rn_end + ASP * (SP > 0 ? lpp : lpm));
      }
    };
    static_assert(ZU == 1 || ZU == 4, "the step loop is written for 1 or 4 phases");
    int rn = 0;
    int rem = 0;
    if constexpr (ZU == 1) {
      for (; rn < nsteps; ++rn) step.template operator()<0>(rn);
    } else {
      for (; rn + ZU <= nsteps; rn += ZU) {
        step.template operator()<0>(rn);
        step.template operator()<1>(rn + 1);
        step.template operator()<2>(rn + 2);
        step.template operator()<3>(rn + 3);
      }
      rem = nsteps - rn;
      if (rem > 0) step.template operator()<0>(rn);
      if (rem > 1) step.template operator()<1>(rn + 1);
      if (rem > 2) step.template operator()<2>(rn + 2);
    }

    // ---- segment end: emit the rest of every window, flush the rings ----
    const int rn_end = nsteps;
    if constexpr (ZU == 1) {
      end_emit.template operator()<0>(rn_end);
    } else {
      switch (rem) {
        case 0: end_emit.template operator()<0>(rn_end); break;
        case 1: end_emit.template operator()<1>(rn_end); break;
        case 2: end_emit.template operator()<2>(rn_end); break;
        default: end_emit.template operator()<3>(rn_end); break;
      }
    }
    __syncwarp();
    #pragma unroll
    for (int j = 0; j < NOB; ++j) {
      const int s = zs_form_s(j), as = zs_abs(s);
      const uint32_t roff = j == 0 ? R0 : j == 1 ? R1 : j == 2 ? R2 : R3;
      const int32_t base = base_of(s), Wj = (int32_t)p.W[DPM_IMG_DIAG + j];
      uint32_t* const rowj = p.img[DPM_IMG_DIAG + j] + rowid * Wj;
      #pragma unroll
      for (int c = lane; c < 8 * 32 * as; c += 32) {
        const int blk = rn_end + c / 8, kk = c % 8;
        const int idx = as == 1 ? Ring<1>::idx(blk) : Ring<2>::idx(blk);
        const uint32_t a = wring_a + roff + 4u * (uint32_t)(idx + kk * (as == 1 ? Ring<1>::RP : Ring<2>::RP));
        const uint32_t v = ptx::lds_u32(a);
        ptx::sts_u32(a, 0u);
        const int32_t i = base + 8 * blk + kk;
        if (v != 0 && yok && i >= 0 && i < Wj) atomicAdd(rowj + i, v);
      }
    }
    // YZ slot [x][y]: the lane's x-sums over the segment's planes
    #pragma unroll
    for (int kk = 0; kk < VX; ++kk)
      if (cs[kk] != 0 && yok && xl + kk < p.L) atomicAdd(p.img[DPM_IMG_YZ] + (b * p.L + xl + kk) * p.M + y, cs[kk]);
    // CTA profile ring: every warp has emitted all of the segment; flush what is left
    zs_sync<NW>();
    {
      const int first = rn_end >= PLAG ? rn_end - PLAG : 0;   // blocks the step loop did not flush
      const int nblk = rn_end + 32 * ASP - first;
      for (int c = tid; c < 8 * nblk; c += 32 * NW) {
        const int blk = first + c / 8, kk = c % 8;
        const uint32_t a = pring_a + 4u * (uint32_t)(PR::idx(blk) + kk * PR::RP);
        const uint32_t v = ptx::lds_u32(a);
        ptx::sts_u32(a, 0u);
        const int32_t i = pbase + 8 * blk + kk;
        if (v != 0 && i >= 0 && i < p.WQ) atomicAdd(prow + i, zprof64<T>(v));
      }
    }
    if (lane == 0) segs[w].next(p);
    zs_sync<NW>();
  }
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();   // project_stream.cu

#ifndef DPM_ZS_FMAMASK
#define DPM_ZS_FMAMASK 0   // forms folded with IMAD on the FMA pipe: bit j = oblique j, bit 4 = profile
#endif
#ifndef DPM_ZS_FMAMASK6
#define DPM_ZS_FMAMASK6 28 // order 6 at 12 warps: X2P, X2M and the profile on the FMA pipe (2-plane groups)
#endif

#ifndef DPM_ZS_NW6
#define DPM_ZS_NW6 (DPM_ZS_HALF ? 12 : 8)   // warps (= image rows) per CTA at orders 5-6
#endif
template <typename T, int K> struct ZCfg {
  static constexpr int VX = 8;
  static constexpr int NW = K >= 5 ? DPM_ZS_NW6 : DPM_ZS_NW34;
  static constexpr int FMAMASK = K >= 5 && NW > 8 && !DPM_ZS_HALF ? DPM_ZS_FMAMASK6 : DPM_ZS_FMAMASK;
  static constexpr int STAGE = 32 * VX * NW * 8 * (int)sizeof(T);
  static constexpr int RINGS = NW * ZGeo<T, K, NW, VX, 1>::WARP_RING * 4 + 8 * 200 * 4;
  static constexpr int FIT = ((zs_ctas(K) == 1 ? 225 : 226 / zs_ctas(K)) * 1024 - RINGS) / STAGE;
  static constexpr int STAGES = FIT > 6 ? 6 : FIT;
};

bool zstream_eligible(const dpm_volume_desc* d, const void* vox) {
  const int64_t es = d->dtype == DPM_U8 ? 1 : 2;
  if (d->L < 192 || d->L % 8) return false;
  if ((d->stride_y * es) % 16 || (d->stride_z * es) % 16) return false;
  if (d->B > 1 && (d->stride_b * es) % 16) return false;
  if (reinterpret_cast<uintptr_t>(vox) % 16) return false;
  if (d->L > 0x7fffffffLL || d->M > 0x7fffffffLL || d->N > 0x7fffffffLL || d->B > 0x7fffffffLL) return false;
  return tensor_map_encoder() != nullptr;
}

template <typename T, int K>
static int launch_zs(const dpm_volume_desc* d, const void* vox, const ImageSet& s, unsigned long long* prof,
                     int64_t WQ, int sms, cudaStream_t st) {
  using C = ZCfg<T, K>;
  constexpr int NW = C::NW, VX = C::VX, S = C::STAGES;
  using G = ZGeo<T, K, NW, VX, S>;
  static_assert(G::SMEM <= 227 * 1024, "shared memory budget");
  const int64_t es = sizeof(T);
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)d->L, (cuuint64_t)d->M, (cuuint64_t)d->N, (cuuint64_t)d->B};
  const cuuint64_t strides[3] = {(cuuint64_t)(d->stride_y * es), (cuuint64_t)(d->stride_z * es),
                                 (cuuint64_t)((d->B > 1 ? d->stride_b : d->stride_z * d->N) * es)};
  const cuuint32_t box[4] = {(cuuint32_t)G::SX, (cuuint32_t)NW, (cuuint32_t)(8 / zs_spl(K)), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = tensor_map_encoder()(&map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16,
                                          4, const_cast<void*>(vox), dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -1;
  ZParams p;
  memset(&p, 0, sizeof(p));
  p.L = d->L; p.M = d->M; p.N = d->N; p.B = d->B; p.offset = d->offset;
  p.n_xt = (int32_t)((d->L + G::SX - 1) / G::SX);
  p.n_yg = (int32_t)((d->M + NW - 1) / NW);
  p.ns = (int32_t)((d->N + 7) / 8);
  p.ncol = d->B * p.n_yg * p.n_xt;
  p.one = 1;
  for (int k = 0; k < DPM_MAX_IMAGES; ++k) { p.img[k] = s.img[k]; p.W[k] = s.W[k]; }
  p.prof = prof;
  p.WQ = WQ;
  // schedule: equal contiguous runs of the (column, step) space, one per CTA
  // (32-bit positions: see ZSeg); column order by the size of the image set
  if (p.ncol * p.ns >= 0x7fffffffLL) return -1;   // not reachable with < 32 TB of voxels: the classic pass takes it
  int64_t img_bytes = 0;
  for (int k = 0; k < s.n_img; ++k) img_bytes += s.W[k] * s.H[k] * 4 * d->B;
  const int64_t G_ = (int64_t)sms * zs_ctas(K);
  const int grid = (int)imin64(G_, p.ncol * p.ns);
  // (the threshold can be overridden at run time, e.g. 0 to test the order on small volumes)
  static const int64_t xt_mb = [] { const char* e = getenv("DPM_ZS_XT_MAJOR_MB"); return e ? (int64_t)atoll(e) : (int64_t)DPM_ZS_XT_MAJOR_MB; }();
  static const int yb_forced = [] { const char* e = getenv("DPM_ZS_YB"); return e ? atoi(e) : 0; }();
  p.yb = 1;
  if (img_bytes > (xt_mb << 20) && p.n_xt > 1) {
    const double R = (double)p.ncol / grid;
    double best = 1e9;
    p.yb = p.n_yg;
    for (int m = 1; m <= 8; ++m) {
      const int yb = (int)(m * R + 0.5);
      if (yb < 1 || yb > p.n_yg) continue;
      const double err = fabs(yb - m * R);
      if (err < best - 1e-9) { best = err; p.yb = yb; }
    }
    if (yb_forced > 0) p.yb = (int)imin64(yb_forced, p.n_yg);
  }
  static std::atomic<uint64_t> attr_mask{0};
  if (ensure_smem(zstream_kernel<T, K, NW, VX, S, C::FMAMASK>, G::SMEM, attr_mask)) return DPM_ECUDA;
  if (launch_pdl(zstream_kernel<T, K, NW, VX, S, C::FMAMASK>, dim3(grid), dim3(32 * (NW + ZPW)), G::SMEM, st, map, p) !=
      cudaSuccess)
    return DPM_ECUDA;
  return DPM_OK;
}

template <typename T>
static int launch_zs_k(int order, const dpm_volume_desc* d, const void* vox, const ImageSet& s,
                       unsigned long long* prof, int64_t WQ, int sms, cudaStream_t st) {
  switch (order) {
    case 3: return launch_zs<T, 3>(d, vox, s, prof, WQ, sms, st);
    case 4: return launch_zs<T, 4>(d, vox, s, prof, WQ, sms, st);
    case 5: return launch_zs<T, 5>(d, vox, s, prof, WQ, sms, st);
    default: return launch_zs<T, 6>(d, vox, s, prof, WQ, sms, st);
  }
}

// layout-T moments projection pass; the caller zeroed the images and profile
int launch_project_zstream(const dpm_volume_desc* d, const void* vox, int order, const ImageSet& s,
                           unsigned long long* prof, int64_t WQ, cudaStream_t st, bool* handled, bool signed_i16) {
  *handled = false;
  if (!zstream_eligible(d, vox)) return DPM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int rc;
  switch (d->dtype) {
    case DPM_U8: rc = launch_zs_k<uint8_t>(order, d, vox, s, prof, WQ, sms, st); break;
    case DPM_U16: rc = launch_zs_k<uint16_t>(order, d, vox, s, prof, WQ, sms, st); break;
    default:
      rc = signed_i16 ? launch_zs_k<s16>(order, d, vox, s, prof, WQ, sms, st)
                      : launch_zs_k<int16_t>(order, d, vox, s, prof, WQ, sms, st);
      break;
  }
  if (rc < 0) return DPM_OK;
  if (rc) return rc;
  note_launches(1);
  *handled = true;
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
