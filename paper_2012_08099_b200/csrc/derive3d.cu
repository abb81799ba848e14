// derive3d.cu -- device epilogue: 2D moments -> 3D moments, exact.
//
// Placement follows moments3d.dpm_moments (moments3d.py:255-261) with the
// duplicate-route check of _place (moments3d.py:223-229): XY -> (p,q,0),
// YZ -> (0,p,q), ZX -> (q,0,p).  The moments with all three indices >= 1 come
// from the oblique images (x + t z, y), t = 1, -1, 2, -2:
//   f_t = M^t_{p,q} - M_{p,q,0} - t^p M_{0,q,p} = sum_{c=1}^{p-1} C(p,c) t^c M_{p-c,q,c}
// solved in closed form (exact integer divisions).  At order 4 these are the
// reference's formulas (moments3d.py:213-219; note the oracle-pinned sum/
// difference association, test_moments3d.py:116-147).  Orders 5-6 extend the
// same scheme.
#include "dpm_common.cuh"

namespace dpm {

typedef __int128 i128;

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

__device__ __forceinline__ bool div_exact(i128 num, int64_t d, i128* q) {
  *q = num / d;
  return (*q) * d == num;
}

template <int K>
__global__ void derive3d_kernel(const uint64_t* acc, int64_t B, int n_img, int64_t* out_i128,
                                double* out_f64, int32_t* status) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  constexpr int N3 = (K + 1) * (K + 2) * (K + 3) / 6;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const uint64_t* a = acc + b * n_img * N2 * 4;
  i128 out[N3];
  bool have[N3];
  for (int i = 0; i < N3; ++i) { out[i] = 0; have[i] = false; }
  int32_t st = 0;
  auto m2 = [&](int img, int p, int q) -> i128 { return acc_to_i128(a + (img * N2 + idx2(K, p, q)) * 4); };
  const i128 mass = m2(0, 0, 0);
  for (int k = 1; k < n_img; ++k)
    if (m2(k, 0, 0) != mass) st |= DPM_ST_MASS;
  auto place = [&](int p, int q, int r, i128 v) {
    const int i = idx3(K, p, q, r);
    if (!have[i]) { have[i] = true; out[i] = v; }
    else if (out[i] != v) st |= DPM_ST_DISAGREE;
  };
  for (int p = 0; p <= K; ++p)
    for (int q = 0; q <= K - p; ++q) place(p, q, 0, m2(DPM_IMG_XY, p, q));
  for (int p = 0; p <= K; ++p)
    for (int q = 0; q <= K - p; ++q) place(0, p, q, m2(DPM_IMG_YZ, p, q));
  for (int p = 0; p <= K; ++p)
    for (int q = 0; q <= K - p; ++q) place(q, 0, p, m2(DPM_IMG_ZX, p, q));

  const int tv[4] = {1, -1, 2, -2};
  for (int q = 1; q <= K - 2; ++q) {
    for (int p = 2; p <= K - q; ++p) {
      const int n = p - 1;
      i128 f[4] = {0, 0, 0, 0};
      for (int k = 0; k < n; ++k) {
        i128 tp = 1;
        for (int e = 0; e < p; ++e) tp *= tv[k];
        f[k] = m2(DPM_IMG_DIAG + k, p, q) - out[idx3(K, p, q, 0)] - tp * out[idx3(K, 0, q, p)];
      }
      i128 u[5] = {0, 0, 0, 0, 0};
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
      } else {
        i128 E1, E2, O1, O2;
        ok &= div_exact(f[0] + f[1], 2, &E1); ok &= div_exact(f[2] + f[3], 2, &E2);
        ok &= div_exact(f[0] - f[1], 2, &O1); ok &= div_exact(f[2] - f[3], 2, &O2);
        ok &= div_exact(E2 - 4 * E1, 12, &u[4]); u[2] = E1 - u[4];
        ok &= div_exact(O2 - 2 * O1, 6, &u[3]); u[1] = O1 - u[3];
      }
      int64_t binom = 1;
      for (int c = 1; c <= n; ++c) {
        binom = binom * (p - c + 1) / c;
        i128 m;
        ok &= div_exact(u[c], binom, &m);
        out[idx3(K, p - c, q, c)] = m;
        have[idx3(K, p - c, q, c)] = true;
      }
      if (!ok) st |= DPM_ST_NONEXACT;
    }
  }
  for (int i = 0; i < N3; ++i) {
    const unsigned __int128 u = (unsigned __int128)out[i];
    out_i128[(b * N3 + i) * 2 + 0] = (int64_t)(uint64_t)u;
    out_i128[(b * N3 + i) * 2 + 1] = (int64_t)(uint64_t)(u >> 64);
    if (out_f64) out_f64[b * N3 + i] = i128_to_f64(out[i]);
  }
  status[b] = st;
}

int launch_derive3d(const uint64_t* acc, int64_t B, int n_img, int order, int64_t* out_i128,
                    double* out_f64, int32_t* status, cudaStream_t st) {
  const int threads = 64;
  const unsigned grid = (unsigned)((B + threads - 1) / threads);
  switch (order) {
    case 3: derive3d_kernel<3><<<grid, threads, 0, st>>>(acc, B, n_img, out_i128, out_f64, status); break;
    case 4: derive3d_kernel<4><<<grid, threads, 0, st>>>(acc, B, n_img, out_i128, out_f64, status); break;
    case 5: derive3d_kernel<5><<<grid, threads, 0, st>>>(acc, B, n_img, out_i128, out_f64, status); break;
    default: derive3d_kernel<6><<<grid, threads, 0, st>>>(acc, B, n_img, out_i128, out_f64, status); break;
  }
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
