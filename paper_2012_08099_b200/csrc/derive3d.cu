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
//
// Accumulator kinds.  DPM_ACC_IMAGES: slot 2 holds the ZX image's moments
// (dpm_moments2d over the reference's image set).  DPM_ACC_PROFILE (the
// moments pipeline): slot 2 holds the 1D moments of the y-summed profile
// P[x + t z], t = profile_shift (-1, 2, -2, 3 at orders 3..6), so the q = 0
// family M_{p,0,r} (p, r >= 1) is solved like the others, from the obliques'
// q = 0 rows plus the profile as the next direction t (order 6, p + r = 6:
// five unknowns from t = 1, -1, 2, -2, 3).  Every equation a group does not
// need is checked against the solution (DPM_ST_DISAGREE), including the
// p + r = 1 rows, which have no unknowns at all.
#include "derive_dev.cuh"

namespace dpm {

constexpr int kDeriveWarps = 16;   // solve/check groups (<= 21 at order 6) are dealt round-robin

template <int K>
__global__ void __launch_bounds__(32 * kDeriveWarps) derive3d_kernel(const uint64_t* acc, int64_t B, int n_img,
                                                                    int kind, int64_t* out_i128, double* out_f64,
                                                                    int32_t* status) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  __shared__ uint64_t sa[DPM_MAX_IMAGES * N2 * 4];
  __shared__ int32_t sst;
  const int64_t b = blockIdx.x;
  derive_volume<K>(acc + b * n_img * N2 * 4, b, n_img, kind, out_i128, out_f64, status, sa, &sst, false);
}

int launch_derive3d(const uint64_t* acc, int64_t B, int n_img, int order, int kind, int64_t* out_i128,
                    double* out_f64, int32_t* status, cudaStream_t st) {
  const int threads = 32 * kDeriveWarps;   // one CTA per volume
  const unsigned grid = (unsigned)B;
  switch (order) {
    case 3: derive3d_kernel<3><<<grid, threads, 0, st>>>(acc, B, n_img, kind, out_i128, out_f64, status); break;
    case 4: derive3d_kernel<4><<<grid, threads, 0, st>>>(acc, B, n_img, kind, out_i128, out_f64, status); break;
    case 5: derive3d_kernel<5><<<grid, threads, 0, st>>>(acc, B, n_img, kind, out_i128, out_f64, status); break;
    default: derive3d_kernel<6><<<grid, threads, 0, st>>>(acc, B, n_img, kind, out_i128, out_f64, status); break;
  }
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
