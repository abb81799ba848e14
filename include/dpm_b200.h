/*
 * dpm_b200.h -- C ABI of the B200-native Discrete Projection Moment (DPM) hot path.
 *
 * The drop-in boundary for the reference package `volmoments`
 * (/root/reference/pkg/src/volmoments).  Each entry point replaces one stage of
 * the reference's hot path; the reference interface it stands in for is cited
 * beside it.  Plain pointers and sizes only: no torch types cross this ABI.
 *
 * Conventions
 *   - Every pointer named `d_*` is a CUDA device pointer; every other pointer is
 *     host memory.  The caller owns (allocates and frees) every buffer.  The
 *     library never allocates device memory, never frees, never synchronises:
 *     all work is enqueued on the `stream` argument (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).
 *   - Volumes are x-fastest: voxel (x, y, z, b) lives at element offset
 *     x + y*stride_y + z*stride_z + b*stride_b (reference volume.py:1-6).
 *   - Images are row-major uint32 `pixels[j][i]` with the reference's stored
 *     index maps (projection.py:7-14; ANTI stored at x-z+N-1).  The order-5/6
 *     extension adds X2P (x+2z, y) and X2M (x-2z+2(N-1), y).
 *   - Moments are exact signed 128-bit integers returned as (lo, hi) int64
 *     pairs, plus the same values rounded to fp64.  3D moments are ordered like
 *     moment_indices (moments3d.py:46-54): lexicographic (p, q, r), p+q+r <= K.
 *   - Return value: DPM_OK or a DPM_E* code (dpm_strerror).  Device-side
 *     consistency failures are reported through the int32 `d_status` word,
 *     which the host maps to volmoments.InconsistencyError (errors.py:8-15).
 *   - Reentrant; no global mutable state except a one-time lazy kernel
 *     attribute setup guarded by std::call_once.
 */
#ifndef DPM_B200_H
#define DPM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DPM_API __attribute__((visibility("default")))
#else
#define DPM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define DPM_OK 0
#define DPM_EINVAL 1       /* bad argument: maps to ValueError (moments3d.py:57-59, volume.py:34-35) */
#define DPM_EOVERFLOW 2    /* exactness envelope exceeded: maps to OverflowError (moments3d.py:121-127) */
#define DPM_ECUDA 3        /* a CUDA launch/runtime error: maps to RuntimeError */
#define DPM_EWORKSPACE 4   /* workspace too small */

/* device status word bits (d_status), mapped to InconsistencyError */
#define DPM_ST_DISAGREE 1  /* two projection routes disagree (moments3d.py:223-229) */
#define DPM_ST_NONEXACT 2  /* an exact division left a remainder (drt2d.py:133-137) */
#define DPM_ST_MASS 4      /* image masses differ (drt2d.py:160-161) */

/* ---- voxel types --------------------------------------------------------- */
#define DPM_U8 1
#define DPM_U16 2
#define DPM_I16 3          /* signed 16-bit plus `offset` (CT volumes: +1024) */

/* ---- image tags (index into every per-image array) ----------------------- */
#define DPM_IMG_XY 0
#define DPM_IMG_YZ 1
#define DPM_IMG_ZX 2
#define DPM_IMG_DIAG 3
#define DPM_IMG_ANTI 4
#define DPM_IMG_X2P 5
#define DPM_IMG_X2M 6
#define DPM_MAX_IMAGES 7
#define DPM_MAX_ORDER 6

/* ---- limb-accumulator kinds (what slot DPM_IMG_ZX of d_acc holds) ---------- */
#define DPM_ACC_IMAGES 0   /* the ZX image's 2D moments (dpm_moments2d on dpm_project's images) */
#define DPM_ACC_PROFILE 1  /* the y-summed profile's 1D moments (dpm_moments_partial, dpm_moments2d_profile) */
#define DPM_ACC_PROFILE_T 2 /* the same for layout T (x and z exchanged, see dpm_moments_acc_kind) */

/* A (batch of) volume(s), or a z-slab of one.  Strides are in elements. */
typedef struct dpm_volume_desc {
  int64_t L, M, N;        /* extents along x, y, z (of this slab) */
  int64_t B;              /* number of volumes (1 unless batched) */
  int64_t stride_y;       /* usually L */
  int64_t stride_z;       /* usually L*M */
  int64_t stride_b;       /* usually L*M*N */
  int32_t dtype;          /* DPM_U8 / DPM_U16 / DPM_I16 */
  int32_t offset;         /* added to every voxel before accumulation */
  int64_t z0;             /* global z of this slab's first plane (0: whole volume) */
} dpm_volume_desc;

/* Number of projection images the DPM method needs at `order`
 * (4 at K<=3, 5 at K=4: moments3d.py:242-245; 6 at K=5, 7 at K=6). */
DPM_API int dpm_num_images(int order);

/* Number of 3D / 2D raw moments with total order <= `order`. */
DPM_API int dpm_num_moments3d(int order);
DPM_API int dpm_num_moments2d(int order);

/* Geometry of image `img` for `desc`: width W (index i), height H (index j),
 * and the offsets (ai, aj) mapping stored (i, j) to logical global
 * coordinates (i + ai, j + aj).  Replaces the size rules of projection.py:7-14
 * and the ANTI origin_offset of projection.py:189-191. */
DPM_API int dpm_image_layout(const dpm_volume_desc* desc, int img,
                     int64_t* W, int64_t* H, int64_t* ai, int64_t* aj);

/* Projection pass.  Replaces projection._accumulate / project_subset
 * (projection.py:139-210): builds images 0..n_img-1 of every volume in one
 * streaming read of the voxels.  `d_images[k]` holds B * W_k * H_k uint32
 * (volume b at offset b*W_k*H_k); the call zeroes them first.  `d_ws` is
 * scratch of dpm_project_workspace_bytes() bytes (may be NULL when that is 0). */
DPM_API size_t dpm_project_workspace_bytes(const dpm_volume_desc* desc, int n_img);
DPM_API int dpm_project(const dpm_volume_desc* desc, const void* d_voxels, int n_img,
                uint32_t* const* d_images, void* d_ws, size_t ws_bytes, void* stream);

/* The same projection pass through the shape-generic brick kernel only (never
 * the TMA streaming kernel): an independent second implementation, registered
 * as the "dpm_generic" engine so verify_engines (harness.py:101-120) has two
 * device engines to cross-check, as the reference cross-checks its three. */
DPM_API int dpm_project_generic(const dpm_volume_desc* desc, const void* d_voxels, int n_img,
                uint32_t* const* d_images, void* stream);

/* Exact 2D raw moments M_pq = sum I[j][i] (i+ai)^p (j+aj)^q, p+q <= order, of
 * images laid out by `desc`.  Replaces drt2d.integrals + assemble_2d +
 * shift_origin (drt2d.py:92-208) and exact.weighted_power_sums (exact.py:63-82).
 * Output `d_acc` is B * n_img * n2d * 4 uint64 limb sums: the moment is
 * sum_k acc[k] * 2^(32k) mod 2^128, read as two's complement.  The call zeroes
 * d_acc first. */
DPM_API int dpm_moments2d(const dpm_volume_desc* desc, int n_img, const uint32_t* const* d_images,
                  int order, uint64_t* d_acc, void* stream);

/* Exact 2D raw moments of ONE stand-alone device image, pixels[j][i]
 * (contiguous rows of W uint32), about additive origins (ai, aj >= 0):
 *   M_pq = sum_{i,j} I[j][i] (i + ai)^p (j + aj)^q,  p + q <= order (3..6).
 * Replaces drt2d.brute_force_2d and assemble_2d(integrals(image))
 * (drt2d.py:140-193) for device images: same values, any order up to 6.
 * d_acc: n2d(order) * 4 uint64 limb sums, zeroed by the call (read as in
 * dpm_moments2d).  The caller checks the exactness envelope
 * (mass * max|coordinate|^order < 2^126); DPM_EOVERFLOW if H - 1 + aj >= 2^21. */
DPM_API int dpm_image_moments2d(const uint32_t* d_pixels, int64_t W, int64_t H, int64_t ai, int64_t aj,
                                int order, uint64_t* d_acc, void* stream);

/* ---- the moments pipeline ------------------------------------------------
 * dpm_moments does not build the ZX image: the q = 0 moments M_{p,0,r} come
 * from the obliques' q = 0 rows plus ONE extra direction, the profile
 *   P[x + t z] = sum_y V(x, y, z),  t = -1, 2, -2, 3 at orders 3, 4, 5, 6,
 * a 1D array of WQ = L + |t|(N-1) uint64 per volume (stored index x + t z, plus
 * |t|(N-1) when t < 0; logical coordinate = stored index + ai).  Per voxel the
 * pass folds the profile into a register window summed over y instead of
 * keeping the 8 x VX ZX accumulators of dpm_project.
 *
 * Layout T.  Wide volumes (L >= 192) build that image set for the volume with
 * x and z EXCHANGED, V'(x', y, z') = V(z', y, x'), with the z-streaming kernel:
 * XY slot (z, y) stored [y][z]; YZ slot (y, x) stored [x][y]; DIAG z + x,
 * ANTI z - x + (L-1), X2P z + 2x, X2M z - 2x + 2(L-1) stored [y][.]; the
 * profile P[z + t x] (+|t|(L-1) when t < 0), WQ = N + |t|(L-1).  Their
 * accumulators are DPM_ACC_PROFILE_T (the epilogue relabels M_pqr = M'_rqp).
 * The layout depends on the geometry only, so all z-slabs of one volume agree.
 * dpm_moments_image_layout / dpm_profile_layout give the geometry of the
 * moments pipeline's images and profile for either layout. */
DPM_API int dpm_profile_layout(const dpm_volume_desc* desc, int order, int64_t* WQ, int64_t* ai, int* t);
/* Accumulator kind (DPM_ACC_PROFILE or DPM_ACC_PROFILE_T) that
 * dpm_moments_partial / dpm_moments2d_profile produce for `desc`, to pass to
 * dpm_derive3d; negative on a bad argument. */
DPM_API int dpm_moments_acc_kind(const dpm_volume_desc* desc, int order);
/* Geometry of image `img` (not DPM_IMG_ZX) of the moments pipeline at `order`
 * (as dpm_image_layout, for the layout dpm_moments_acc_kind names). */
DPM_API int dpm_moments_image_layout(const dpm_volume_desc* desc, int order, int img,
                int64_t* W, int64_t* H, int64_t* ai, int64_t* aj);
/* Projection pass of the moments pipeline: images 0..num_images(order)-1
 * except DPM_IMG_ZX (d_images[2] is ignored) plus the profile (B * WQ
 * uint64).  Zeroes its outputs first. */
DPM_API int dpm_project_profile(const dpm_volume_desc* desc, const void* d_voxels, int order,
                uint32_t* const* d_images, uint64_t* d_profile, void* stream);
/* The same two halves separately, for callers that keep the buffers and
 * re-zero them right after their moments are taken (engine.GraphedSlabStages:
 * the zeroing rides the moments stage, the projection stage is the pass alone):
 * dpm_zero_profile_buffers zeroes the images and the profile (one launch),
 * dpm_project_profile_zeroed runs the pass on buffers the caller zeroed. */
DPM_API int dpm_zero_profile_buffers(const dpm_volume_desc* desc, int order, uint32_t* const* d_images,
                uint64_t* d_profile, void* stream);
DPM_API int dpm_project_profile_zeroed(const dpm_volume_desc* desc, const void* d_voxels, int order,
                uint32_t* const* d_images, uint64_t* d_profile, void* stream);
/* Exact moments of those images (2D) and of the profile (1D, into the q = 0
 * entries of slot DPM_IMG_ZX): a DPM_ACC_PROFILE accumulator, zeroed first. */
DPM_API int dpm_moments2d_profile(const dpm_volume_desc* desc, int order, const uint32_t* const* d_images,
                const uint64_t* d_profile, uint64_t* d_acc, void* stream);
/* The same, ending with the epilogue in the same launch (the last block of each
 * volume derives it, like dpm_moments): for a single device, where no
 * accumulator exchange sits between the moments and the epilogue.
 * d_counters: B uint32 scratch (zeroed by the call). */
DPM_API int dpm_moments2d_profile_derive(const dpm_volume_desc* desc, int order, const uint32_t* const* d_images,
                const uint64_t* d_profile, uint64_t* d_acc, uint32_t* d_counters, int64_t* d_m3d_i128,
                double* d_m3d_f64, int32_t* d_status, void* stream);
/* Both steps on caller scratch of dpm_partial_workspace_bytes() bytes: the
 * per-slab partial of the multi-GPU / streaming drivers (accumulators of
 * z-slabs taken in global coordinates add elementwise). */
DPM_API size_t dpm_partial_workspace_bytes(const dpm_volume_desc* desc, int order);
DPM_API int dpm_moments_partial(const dpm_volume_desc* desc, const void* d_voxels, int order,
                void* d_ws, size_t ws_bytes, uint64_t* d_acc, void* stream);

/* Device epilogue: placement + duplicate-route checks + cross-axis solve.
 * Replaces moments3d._place / _cross_axis_moments / dpm_moments:255-264
 * (moments3d.py:201-264).  Reads d_acc of kind `acc_kind` (DPM_ACC_IMAGES as
 * written by dpm_moments2d, DPM_ACC_PROFILE as written by dpm_moments_partial),
 * writes per volume n3d exact moments to d_m3d_i128 (B * n3d * 2 int64, lo/hi)
 * and fp64 copies to d_m3d_f64 (B * n3d, may be NULL), and ORs DPM_ST_* bits
 * into d_status[b] (B int32, zeroed by the call).  Every equation the solve
 * does not need is checked against it (DPM_ST_DISAGREE). */
DPM_API int dpm_derive3d(const dpm_volume_desc* desc, const uint64_t* d_acc, int order, int acc_kind,
                 int64_t* d_m3d_i128, double* d_m3d_f64, int32_t* d_status, void* stream);

/* Whole pipeline (dpm_moments_partial -> dpm_derive3d) for a volume, a batch of
 * volumes, or a z-slab in global coordinates.  Replaces moments3d.dpm_moments
 * (moments3d.py:232-264).  Needs dpm_workspace_bytes() of scratch. */
DPM_API size_t dpm_workspace_bytes(const dpm_volume_desc* desc, int order);
DPM_API int dpm_moments(const dpm_volume_desc* desc, const void* d_voxels, int order,
                void* d_ws, size_t ws_bytes, int64_t* d_m3d_i128, double* d_m3d_f64,
                int32_t* d_status, void* stream);

/* Exactness envelope: DPM_OK when every moment of a volume/slab with the given
 * global extent and voxel maximum fits the signed 128-bit accumulators (and,
 * at order 6, the profile solve's intermediates: mass * max(L,M,N)^6 < 2^116),
 * else DPM_EOVERFLOW (the analogue of the reference's int64 guards,
 * moments3d.py:121-127, 158-161, drt2d.py:181-184). */
DPM_API int dpm_check_envelope(int64_t L, int64_t M, int64_t N_global, int64_t vmax, int order);

/* Sum `count` limb arrays elementwise into d_acc_out (used by host drivers to
 * combine per-slab partials before dpm_derive3d on one device). */
DPM_API int dpm_acc_add(uint64_t* d_acc_out, const uint64_t* d_acc_in, int64_t count, void* stream);

/* Synthetic config-5 volume: smooth multi-octave lattice value noise mapped by
 * a fixed affine map to 0..65535, generated independently per global z plane
 * so every z-slab is reproducible on any rank.  Writes L*M*n_planes uint16
 * starting at global plane z0. */
DPM_API int dpm_synth_noise_u16(uint16_t* d_out, int64_t L, int64_t M, int64_t z0, int64_t n_planes,
                        uint64_t seed, void* stream);

/* Number of kernels the last dpm_* call on this thread enqueued (bench evidence). */
DPM_API int dpm_last_launch_count(void);

/* ---- the reference's direct engines (cross-checks, not the hot path) ------
 * Exact Eq. 2 sums M_pqr = sum V x^p y^q (z + z0)^r on the device, the
 * counterparts of naive_moments (moments3d.py:78-139: every voxel times every
 * in-plane monomial) and factored_moments (moments3d.py:142-198: x-rows, then
 * y-slices, then z).  `method`: DPM_DIRECT_NAIVE or DPM_DIRECT_FACTORED.
 * d_ws: dpm_direct_workspace_bytes() of scratch (per-plane limb sums). */
#define DPM_DIRECT_NAIVE 0
#define DPM_DIRECT_FACTORED 1
DPM_API size_t dpm_direct_workspace_bytes(const dpm_volume_desc* desc, int order);
DPM_API int dpm_direct_moments(const dpm_volume_desc* desc, const void* d_voxels, int order, int method,
                               void* d_ws, size_t ws_bytes, int64_t* d_m3d_i128, double* d_m3d_f64, void* stream);

DPM_API const char* dpm_strerror(int code);

#ifdef __cplusplus
}
#endif

#endif /* DPM_B200_H */
