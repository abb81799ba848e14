// derive_dev.cuh -- the device epilogue as a device function, shared by the
// derive3d kernel and the fused tail of the moments kernel (moments2d.cu).
// See derive3d.cu for the method.
#pragma once
#include "dpm_common.cuh"

namespace dpm {

typedef __int128 i128;

// DPM_DERIVE_PROBE (development builds only, tools/microbench/derive_probe.cu):
// %globaltimer stamps at the epilogue's phase boundaries, per warp
#ifdef DPM_DERIVE_PROBE
__device__ unsigned long long g_derive_probe[64][8];
__device__ __forceinline__ void derive_probe(int w, int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if ((threadIdx.x & 31) == 0 && w < 64) g_derive_probe[w][i] = t;
}
#define DPM_PROBE(i) derive_probe(w, i)
#else
#define DPM_PROBE(i) ((void)0)
#endif

__device__ __forceinline__ i128 acc_to_i128(const uint64_t* a) {
  unsigned __int128 v = (unsigned __int128)a[0];
  v += ((unsigned __int128)a[1]) << 32;
  v += ((unsigned __int128)a[2]) << 64;
  v += ((unsigned __int128)a[3]) << 96;
  return (i128)v;
}

__device__ __forceinline__ double i128_to_f64(i128 v) {
  const bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-v) : (unsigned __int128)v;
  const uint64_t hi = (uint64_t)(u >> 64), lo = (uint64_t)u;
  double d = (double)hi * 18446744073709551616.0 + (double)lo;
  return neg ? -d : d;
}

// Exact division by a small positive constant d = 2^s * o (o odd) without the
// 128-bit software divide: the low s bits must be zero; the odd part uses the
// inverse of o modulo 2^128, and the quotient is exact iff q * o does not
// overflow 128 bits (then q * o == |num| exactly).
__device__ __forceinline__ bool div_exact(i128 num, int64_t d, i128* out) {
  typedef unsigned __int128 u128;
  const int s = __ffsll(d) - 1;
  const uint64_t o = (uint64_t)d >> s;
  if (s > 0 && ((u128)num & (((u128)1 << s) - 1)) != 0) return false;
  const i128 n1 = num >> s;
  const bool neg = n1 < 0;
  const u128 a = neg ? (u128)(-n1) : (u128)n1;
  u128 inv;
  switch (o) {   // the odd parts that occur (2, 6, 12 and C(p, c), p <= 6): 1, 3, 5, 15
    case 1: inv = 1; break;
    case 3: inv = ((u128)0xAAAAAAAAAAAAAAAAull << 64) | 0xAAAAAAAAAAAAAAABull; break;
    case 5: inv = ((u128)0xCCCCCCCCCCCCCCCCull << 64) | 0xCCCCCCCCCCCCCCCDull; break;
    case 15: inv = ((u128)0xEEEEEEEEEEEEEEEEull << 64) | 0xEEEEEEEEEEEEEEEFull; break;
    default:
      inv = o;                                   // Newton: 3 -> 6 -> ... -> 192 correct bits
      for (int i = 0; i < 6; ++i) inv *= (u128)2 - (u128)o * inv;
  }
  const u128 q = a * inv;
  const uint64_t ql = (uint64_t)q, qh = (uint64_t)(q >> 64);
  const u128 t = (u128)ql * o;
  const u128 hi = (u128)qh * o + (t >> 64);
  if ((hi >> 64) != 0) return false;
  *out = neg ? -(i128)q : (i128)q;
  return true;
}

__device__ __forceinline__ int64_t binom(int n, int k) {
  constexpr int64_t t[7][7] = {{1, 0, 0, 0, 0, 0, 0},  {1, 1, 0, 0, 0, 0, 0},   {1, 2, 1, 0, 0, 0, 0},
                                     {1, 3, 3, 1, 0, 0, 0},  {1, 4, 6, 4, 1, 0, 0},   {1, 5, 10, 10, 5, 1, 0},
                                     {1, 6, 15, 20, 15, 6, 1}};
  return t[n][k];
}


// One CTA per volume.  The volume's limb accumulator (n_img x n2d x 4 words,
// <= 6.3 KB) is staged in shared memory by one coalesced load; threads then
// take the placement / duplicate-route checks of the moments with a zero
// index, and warp w solves the cross-axis groups g = w (mod warps) (group
// (q, a): all unknowns M_{a-c,q,c}, c = 1..a-1) on lane 0 — warp-uniform
// control flow, so the groups run concurrently instead of serialising on
// lane divergence.
// `a` = this volume's accumulator; `sa` = shared staging of n_img * n2d * 4
// words; `sst` = a shared status word.  All threads of the CTA call it.
// `coherent`: read `a` through L2 (written by other CTAs' atomics in the same
// grid, the fused tail of moments2d).
// Signed-exact int16 (capi.cu): the pass summed the raw signed voxels; the
// offset's share of every moment is off * S_P(L) S_Q(M) S_R(N) (power sums
// S_e(n) = sum_{k < n} k^e of the box), added at placement in true (x, y, z) order.
// off * S_e(L), S_e(M), S_e(N) (e = 0..6) as (lo, hi) int64 pairs, formed on
// the host (capi.cu offset_box) so the epilogue only multiplies
struct OffsetBox { int64_t s[3][DPM_MAX_ORDER + 1][2]; };
__device__ __forceinline__ i128 box_sum(const OffsetBox& bx, int axis, int e) {
  return (i128)(((unsigned __int128)(uint64_t)bx.s[axis][e][1] << 64) | (uint64_t)bx.s[axis][e][0]);
}

template <int K>
__device__ void derive_volume(const uint64_t* a, int64_t b, int n_img, int kind, int64_t* out_i128, double* out_f64,
                              int32_t* status, uint64_t* sa, int32_t* sst_p, bool coherent,
                              const OffsetBox* box = nullptr) {
  // DPM_ACC_PROFILE_T: the accumulator holds the layout-T image set (the volume
  // with x and z exchanged); the solve yields M'_pqr = M_rqp, stored relabelled
  const bool prof = kind == DPM_ACC_PROFILE || kind == DPM_ACC_PROFILE_T;
  const bool tr = kind == DPM_ACC_PROFILE_T;
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  constexpr int N3 = (K + 1) * (K + 2) * (K + 3) / 6;
  int32_t& sst = *sst_p;
  const int nthreads = blockDim.x, nwarps = nthreads >> 5;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  DPM_PROBE(0);
  for (int i = tid; i < n_img * N2 * 4; i += nthreads) sa[i] = coherent ? __ldcg(a + i) : a[i];
  if (tid == 0) sst = 0;
  __syncthreads();
  DPM_PROBE(1);
  int32_t st = 0;
  auto m2 = [&](int img, int p, int q) -> i128 { return acc_to_i128(sa + (img * N2 + idx2(K, p, q)) * 4); };
  auto put = [&](int p, int q, int r, i128 v) {
    const int i = tr ? idx3(K, r, q, p) : idx3(K, p, q, r);
    if (box) {   // true (x, y, z) exponents; the offset is folded into the x sums
      const int P = tr ? r : p, R = tr ? p : r;
      v += box_sum(*box, 0, P) * box_sum(*box, 1, q) * box_sum(*box, 2, R);
    }
    const unsigned __int128 u = (unsigned __int128)v;
    out_i128[(b * N3 + i) * 2 + 0] = (int64_t)(uint64_t)u;
    out_i128[(b * N3 + i) * 2 + 1] = (int64_t)(uint64_t)(u >> 64);
    if (out_f64) out_f64[b * N3 + i] = i128_to_f64(v);
  };
  if (tid > 0 && tid < n_img && m2(tid, 0, 0) != m2(0, 0, 0)) st |= DPM_ST_MASS;

  // placement: XY -> (p,q,0), YZ -> (0,p,q), ZX -> (q,0,p); first route wins, others must agree
  // (one moment per thread: n3d <= 84 <= blockDim; the index is decoded, not
  // searched with a run-time modulo per candidate -- that loop was most of the
  // epilogue's latency)
  // (counted from the LAST thread: warp 0 takes the costliest solve group below)
  for (int n = nthreads - 1 - tid; n < N3; n += nthreads) {
    int p = 0, rem = n;
    while (rem >= (K - p + 1) * (K - p + 2) / 2) { rem -= (K - p + 1) * (K - p + 2) / 2; ++p; }
    int q = 0;
    while (rem >= K - p - q + 1) { rem -= K - p - q + 1; ++q; }
    const int r = rem;
    if (p > 0 && r > 0 && (q > 0 || prof)) continue;
    bool have = false;
    i128 v = 0;
    auto route = [&](i128 x) {
      if (!have) { have = true; v = x; }
      else if (x != v) st |= DPM_ST_DISAGREE;
    };
    if (r == 0) route(m2(DPM_IMG_XY, p, q));
    if (p == 0) route(m2(DPM_IMG_YZ, q, r));
    if (q == 0 && !prof) route(m2(DPM_IMG_ZX, r, p));
    put(p, q, r, v);
  }

  DPM_PROBE(2);
  // cross-axis groups (q, a = p + r): unknowns u_c = C(a,c) M_{a-c,q,c}, c = 1..a-1, from
  //   f_t = M^t_{a,q} - M_{a,q,0} - t^a M_{0,q,a} = sum_c t^c u_c
  // over the oblique images t = 1, -1, 2, -2 (and, for q = 0 in profile mode,
  // the profile as the next t).  Groups with a = 1 only check.
  // Group (q, p) runs on lane q of warp (K - p) mod nwarps: the lanes of a warp
  // share p, so they share the solve path (n = p - 1 unknowns) and run the
  // groups of a p side by side (one lane each) instead of one after another;
  // the costliest p (the most unknowns) get warps of their own first.
  {
    const int tv[5] = {1, -1, 2, -2, 3};
    const int n_obl = n_img - 3;
    const int q = lane;
    for (int p = K - w; p >= 1; p -= nwarps) {
        if (q < (prof ? 0 : 1) || q > K - p) continue;
        const int n = p - 1;                               // unknowns
        const int avail = (q == 0) ? n_obl + 1 : n_obl;    // equations (q = 0 only in profile mode)
        const i128 mxy = m2(DPM_IMG_XY, p, q), myz = m2(DPM_IMG_YZ, q, p);
        i128 f[5] = {0, 0, 0, 0, 0};
        #pragma unroll
        for (int k = 0; k < 5; ++k) {
          if (k < avail) {
            i128 tp = 1;
            for (int e = 0; e < p; ++e) tp *= tv[k];
            const int slot = k < n_obl ? DPM_IMG_DIAG + k : DPM_IMG_ZX;   // profile in the ZX slot
            f[k] = m2(slot, p, q) - mxy - tp * myz;
          }
        }
        i128 u[6] = {0, 0, 0, 0, 0, 0};
        bool ok = true;
        if (n == 1) {
          u[1] = f[0];
        } else if (n == 2) {
          ok &= div_exact(f[0] + f[1], 2, &u[2]);
          ok &= div_exact(f[0] - f[1], 2, &u[1]);
        } else if (n == 3) {
          const i128 S = f[0] + f[1], D = f[0] - f[1];
          ok &= div_exact(S, 2, &u[2]);
          ok &= div_exact(f[2] - 2 * S - D, 6, &u[3]);
          i128 h; ok &= div_exact(D, 2, &h); u[1] = h - u[3];
        } else if (n >= 4) {
          i128 E1, E2, O1, O2;
          ok &= div_exact(f[0] + f[1], 2, &E1); ok &= div_exact(f[2] + f[3], 2, &E2);
          ok &= div_exact(f[0] - f[1], 2, &O1); ok &= div_exact(f[2] - f[3], 2, &O2);
          ok &= div_exact(E2 - 4 * E1, 12, &u[4]); u[2] = E1 - u[4];
          if (n == 4) {
            ok &= div_exact(O2 - 2 * O1, 6, &u[3]); u[1] = O1 - u[3];
          } else {   // n == 5: odd unknowns u1, u3, u5 from t = +-1, +-2 and 3
            i128 P2, F, A3, B5;
            ok &= div_exact(O2, 2, &P2);                              // u1 + 4 u3 + 16 u5
            ok &= div_exact(f[4] - 9 * u[2] - 81 * u[4], 3, &F);      // u1 + 9 u3 + 81 u5
            ok &= div_exact(P2 - O1, 3, &A3);                         // u3 + 5 u5
            ok &= div_exact(F - P2, 5, &B5);                          // u3 + 13 u5
            ok &= div_exact(B5 - A3, 8, &u[5]);
            u[3] = A3 - 5 * u[5];
            u[1] = O1 - u[3] - u[5];
          }
        }
        // equations the solve did not use must agree with it
        #pragma unroll
        for (int k = 0; k < 5; ++k) {
          if (k >= n && k < avail) {
            i128 pred = 0, tc = 1;
            for (int c = 1; c <= n; ++c) { tc *= tv[k]; pred += tc * u[c]; }
            if (pred != f[k]) st |= DPM_ST_DISAGREE;
          }
        }
        #pragma unroll
        for (int c = 1; c <= 5; ++c) {
          if (c <= n) {
            i128 m = 0;
            ok &= div_exact(u[c], binom(p, c), &m);
            put(p - c, q, c, m);
          }
        }
        if (!ok) st |= DPM_ST_NONEXACT;
      }
  }
  DPM_PROBE(3);
  st = __reduce_or_sync(0xffffffffu, (unsigned)st);
  if (lane == 0 && st) atomicOr(&sst, st);
  __syncthreads();
  DPM_PROBE(4);
  if (tid == 0) status[b] = sst;
}

}  // namespace dpm
