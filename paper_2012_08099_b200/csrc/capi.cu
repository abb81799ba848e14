// capi.cu -- the C ABI (include/dpm_b200.h): argument validation, workspace
// carving and stage dispatch.  No allocation, no synchronisation.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "dpm_common.cuh"

namespace dpm {

static thread_local int g_launches = 0;
// DPM_DEBUG=1 in the environment: CUDA errors behind DPM_ECUDA are printed
void report_cuda_error(cudaError_t e, const char* where) {
  static const bool on = getenv("DPM_DEBUG") != nullptr;
  if (on) fprintf(stderr, "[dpm] CUDA error in %s: %s\n", where, cudaGetErrorString(e));
}
void note_launches(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

int launch_project_generic(const dpm_volume_desc* d, const void* vox, const ImageSet& s, unsigned long long* prof,
                           cudaStream_t st, bool transposed = false);
int launch_project_zstream(const dpm_volume_desc* d, const void* vox, int order, const ImageSet& s,
                           unsigned long long* prof, int64_t WQ, cudaStream_t st, bool* handled,
                           bool signed_i16 = false);
bool zstream_eligible(const dpm_volume_desc* d, const void* vox);
bool fused_batch_eligible(const dpm_volume_desc* d, const void* vox, int order);
int launch_fused_batch(const dpm_volume_desc* d, const void* vox, int order, uint64_t* acc, unsigned int* cnt,
                       int64_t* out_i128, double* out_f64, int32_t* status, cudaStream_t st, bool* handled);
int launch_project_stream(const dpm_volume_desc* d, const void* vox, const ImageSet& s, unsigned long long* prof,
                          cudaStream_t st, bool* handled);
int profile_shift(int n_img);
bool project_stream_single_tile(const dpm_volume_desc* d, const void* vox, int n_img);
bool project_stream_eligible(const dpm_volume_desc* d, const void* vox);
int launch_pad_copy(const dpm_volume_desc* d, const void* vox, int64_t z, int64_t n, int64_t Lp, void* dst,
                    cudaStream_t st);
size_t project_stream_workspace(const dpm_volume_desc* d, int n_img);
int launch_moments2d(const ImageSet& s, int64_t B, int order, int jbits, uint64_t* acc, cudaStream_t st,
                     const M2Extra* ex = nullptr);
int launch_derive3d(const uint64_t* acc, int64_t B, int n_img, int order, int kind, int64_t* out_i128,
                    double* out_f64, int32_t* status, cudaStream_t st);
int launch_synth_noise(uint16_t* out, int64_t L, int64_t M, int64_t z0, int64_t nz, uint64_t seed, cudaStream_t st);
int launch_direct3d(const dpm_volume_desc* d, const void* vox, int order, bool naive, uint64_t* planes,
                    int64_t* out_i128, double* out_f64, cudaStream_t st);

static int check_desc(const dpm_volume_desc* d) {
  if (!d) return DPM_EINVAL;
  if (d->L < 1 || d->M < 1 || d->N < 1 || d->B < 1) return DPM_EINVAL;
  if (d->dtype != DPM_U8 && d->dtype != DPM_U16 && d->dtype != DPM_I16) return DPM_EINVAL;
  if (d->stride_y < d->L || d->stride_z < d->stride_y * (d->M - 1) + d->L) return DPM_EINVAL;
  if (d->B > 1 && d->stride_b < d->stride_z * (d->N - 1) + d->stride_y * (d->M - 1) + d->L) return DPM_EINVAL;
  if (d->z0 < 0) return DPM_EINVAL;
  // u32 ray sums: the longest ray times the largest voxel must stay below 2^32
  const int64_t vmax = d->dtype == DPM_U8 ? 255 : 65535;
  int64_t ray = d->L > d->M ? d->L : d->M;
  ray = ray > d->N ? ray : d->N;
  if (ray * vmax >= (int64_t(1) << 32)) return DPM_EOVERFLOW;
  // int16 + offset must land in 0..65535 for every int16 value the data may hold:
  // checked by the host wrapper on the actual data range; here only sanity.
  return DPM_OK;
}

struct ZeroList {
  uint8_t* p[DPM_MAX_IMAGES + 2];
  uint64_t bytes[DPM_MAX_IMAGES + 2];
  int n;
};

// grid-stride zeroing of up to 9 buffers (16-byte stores, byte tail); starts
// its dependent (PDL) immediately
__global__ void zero_kernel(const ZeroList z) {
  pdl_trigger();
  const size_t stride = (size_t)gridDim.x * blockDim.x, t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int b = 0; b < z.n; ++b) {
    uint4* q = reinterpret_cast<uint4*>(z.p[b]);
    const size_t n16 = z.bytes[b] / 16;
    for (size_t i = t0; i < n16; i += stride) q[i] = make_uint4(0u, 0u, 0u, 0u);
    for (size_t i = n16 * 16 + t0; i < z.bytes[b]; i += stride) z.p[b][i] = 0;
  }
}

static int zero_list_async(const ZeroList& z, cudaStream_t st) {
  size_t total = 0;
  for (int b = 0; b < z.n; ++b) total += z.bytes[b];
  if (total == 0) return DPM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t want = (total / 16 + 255) / 256;
  const unsigned grid = (unsigned)(want < (size_t)sms * 4 ? (want > 0 ? want : 1) : (size_t)sms * 4);
  zero_kernel<<<grid, 256, 0, st>>>(z);
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

int zero_async(void* p, size_t bytes, cudaStream_t st) {
  ZeroList z;
  z.n = 1;
  z.p[0] = static_cast<uint8_t*>(p);
  z.bytes[0] = bytes;
  return zero_list_async(z, st);
}

#ifndef DPM_SIGNED_I16
#define DPM_SIGNED_I16 1
#endif

static int check_order(int order) { return (order >= 3 && order <= DPM_MAX_ORDER) ? DPM_OK : DPM_EINVAL; }

// Moments-pipeline layout.  Wide volumes use layout T: the
// method's image set of the volume with x and z exchanged, built by the
// z-streaming kernel (project_zstream.cu); the epilogue relabels the result.
// A pure function of the geometry (never of pointers), so the z-slabs of one
// volume -- whose accumulators are summed across ranks -- always agree.
// (DPM_LAYOUT_T_MIN_L in the environment moves the threshold: A/B timing only)
static int64_t layout_t_min_l() {
  static const int64_t v = [] {
    const char* e = getenv("DPM_LAYOUT_T_MIN_L");
    return e ? (int64_t)atoll(e) : (int64_t)192;
  }();
  return v;
}
static bool layout_t(const dpm_volume_desc* d) { return d->L >= layout_t_min_l(); }

// stored geometry of image k of the moments pipeline (slot ZX unused)
static ImageGeom mgeom(const dpm_volume_desc* d, int k) {
  if (!layout_t(d)) return image_geom(d->L, d->M, d->N, d->z0, k);
  // transposed volume V'(x', y, z') = V(z', y, x'): L' = N, N' = L; the slab's
  // global z offset shifts x', i.e. every image index that contains x'
  ImageGeom g = image_geom(d->N, d->M, d->L, 0, k);
  if (k == DPM_IMG_XY || k >= DPM_IMG_DIAG) g.ai += d->z0;
  return g;
}

// no_zx: moments-pipeline image set (slot 2 empty: W = H = 0, no pointer; layout per mgeom)
static ImageSet make_set(const dpm_volume_desc* d, int n_img, uint32_t* const* imgs, bool no_zx = false) {
  ImageSet s;
  memset(&s, 0, sizeof(s));
  s.n_img = n_img;
  for (int k = 0; k < n_img; ++k) {
    if (no_zx && k == DPM_IMG_ZX) continue;
    const ImageGeom g = no_zx ? mgeom(d, k) : image_geom(d->L, d->M, d->N, d->z0, k);
    s.img[k] = imgs ? imgs[k] : nullptr;
    s.W[k] = g.W; s.H[k] = g.H; s.ai[k] = g.ai; s.aj[k] = g.aj;
  }
  return s;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t images_bytes(const dpm_volume_desc* d, int n_img, size_t* offs, bool no_zx = false) {
  size_t total = 0;
  for (int k = 0; k < n_img; ++k) {
    const ImageGeom g = no_zx ? mgeom(d, k) : image_geom(d->L, d->M, d->N, d->z0, k);
    if (offs) offs[k] = total;
    if (no_zx && k == DPM_IMG_ZX) continue;
    total += align256((size_t)(g.W * g.H * d->B) * sizeof(uint32_t));
  }
  return total;
}

static size_t acc_bytes_of(const dpm_volume_desc* d, int order) {
  return align256((size_t)(d->B * num_images(order) * n2d(order) * 4) * sizeof(uint64_t));
}

// the y-summed profile of the moments pipeline: direction t, stored length WQ,
// logical coordinate = stored index + ai (global z: ai includes t * z0)
struct ProfGeom { int t; int64_t WQ, ai; };
static ProfGeom profile_geom(const dpm_volume_desc* d, int order) {
  ProfGeom g;
  g.t = profile_shift(num_images(order));
  const int64_t at = g.t < 0 ? -g.t : g.t;
  if (layout_t(d)) {   // P[z + t x] (+|t|(L-1) for t < 0); the slab offset shifts z
    g.WQ = d->N + at * (d->L - 1);
    g.ai = (g.t > 0 ? 0 : -at * (d->L - 1)) + d->z0;
  } else {
    g.WQ = d->L + at * (d->N - 1);
    g.ai = g.t > 0 ? g.t * d->z0 : -at * (d->N - 1) - at * d->z0;
  }
  return g;
}

static int acc_kind_of(const dpm_volume_desc* d) { return layout_t(d) ? DPM_ACC_PROFILE_T : DPM_ACC_PROFILE; }

static int jbits_for(const dpm_volume_desc* d, int n_img, bool moments_set = false) {
  int64_t jmax = 0;
  for (int k = 0; k < n_img; ++k) {
    if (moments_set && k == DPM_IMG_ZX) continue;
    const ImageGeom g = moments_set ? mgeom(d, k) : image_geom(d->L, d->M, d->N, d->z0, k);
    jmax = imax64(jmax, g.H - 1 + g.aj);
  }
  int b = 0;
  while ((int64_t(1) << b) <= jmax) ++b;
  return b;
}

}  // namespace dpm

using namespace dpm;

extern "C" {

int dpm_num_images(int order) { return check_order(order) ? 0 : num_images(order); }
int dpm_num_moments3d(int order) { return n3d(order); }
int dpm_num_moments2d(int order) { return n2d(order); }

int dpm_image_layout(const dpm_volume_desc* desc, int img, int64_t* W, int64_t* H, int64_t* ai, int64_t* aj) {
  if (!desc || img < 0 || img >= DPM_MAX_IMAGES) return DPM_EINVAL;
  const ImageGeom g = image_geom(desc->L, desc->M, desc->N, desc->z0, img);
  if (W) *W = g.W;
  if (H) *H = g.H;
  if (ai) *ai = g.ai;
  if (aj) *aj = g.aj;
  return DPM_OK;
}

size_t dpm_project_workspace_bytes(const dpm_volume_desc* desc, int n_img) {
  if (check_desc(desc)) return 0;
  return project_stream_workspace(desc, n_img);
}

int dpm_project(const dpm_volume_desc* desc, const void* d_voxels, int n_img, uint32_t* const* d_images,
                void* d_ws, size_t ws_bytes, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (n_img < 3 || n_img > DPM_MAX_IMAGES || !d_images || !d_voxels) return DPM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ImageSet s = make_set(desc, n_img, d_images);
  for (int k = 0; k < n_img; ++k) {
    if (!s.img[k]) return DPM_EINVAL;
    if (cudaMemsetAsync(s.img[k], 0, (size_t)(s.W[k] * s.H[k] * desc->B) * sizeof(uint32_t), st) != cudaSuccess)
      return DPM_ECUDA;
  }
  (void)d_ws; (void)ws_bytes;
  bool handled = false;
  rc = launch_project_stream(desc, d_voxels, s, nullptr, st, &handled);
  if (rc || handled) return rc;
  return launch_project_generic(desc, d_voxels, s, nullptr, st);
}

int dpm_project_generic(const dpm_volume_desc* desc, const void* d_voxels, int n_img, uint32_t* const* d_images,
                        void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (n_img < 3 || n_img > DPM_MAX_IMAGES || !d_images || !d_voxels) return DPM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ImageSet s = make_set(desc, n_img, d_images);
  for (int k = 0; k < n_img; ++k) {
    if (!s.img[k]) return DPM_EINVAL;
    if (cudaMemsetAsync(s.img[k], 0, (size_t)(s.W[k] * s.H[k] * desc->B) * sizeof(uint32_t), st) != cudaSuccess)
      return DPM_ECUDA;
  }
  return launch_project_generic(desc, d_voxels, s, nullptr, st);
}

int dpm_profile_layout(const dpm_volume_desc* desc, int order, int64_t* WQ, int64_t* ai, int* t) {
  if (check_desc(desc) || check_order(order)) return DPM_EINVAL;
  const ProfGeom g = profile_geom(desc, order);
  if (WQ) *WQ = g.WQ;
  if (ai) *ai = g.ai;
  if (t) *t = g.t;
  return DPM_OK;
}

// moments-pipeline projection kernel on a zeroed profile and zeroed images
// (images_zeroed == false: the caller skipped them because the streaming
// kernel stores complete rows -- zero them here if it declines)
static int project_profile_launch(const dpm_volume_desc* desc, const void* d_voxels, int order,
                                  uint32_t* const* d_images, uint64_t* d_profile, cudaStream_t st,
                                  bool images_zeroed = true, bool signed_i16 = false) {
  ImageSet s = make_set(desc, num_images(order), d_images, true);
  unsigned long long* prof = reinterpret_cast<unsigned long long*>(d_profile);
  bool handled = false;
  if (layout_t(desc)) {
    const int rc = launch_project_zstream(desc, d_voxels, order, s, prof, profile_geom(desc, order).WQ, st, &handled,
                                          signed_i16);
    if (rc || handled) return rc;
    // shapes the z-streaming kernel cannot read (unaligned rows): the generic
    // brick kernel on the transposed view builds the same layout-T images
    return launch_project_generic(desc, d_voxels, s, prof, st, true);
  }
  const int rc = launch_project_stream(desc, d_voxels, s, prof, st, &handled);
  if (rc || handled) return rc;
  if (!images_zeroed)
    for (int k = 0; k < s.n_img; ++k)
      if (k != DPM_IMG_ZX &&
          cudaMemsetAsync(s.img[k], 0, (size_t)(s.W[k] * s.H[k] * desc->B) * sizeof(uint32_t), st) != cudaSuccess)
        return DPM_ECUDA;
  return launch_project_generic(desc, d_voxels, s, prof, st);
}

// image + profile moments (one launch) into an already zeroed DPM_ACC_PROFILE
// accumulator; with `fused` (counters zeroed, outputs) the same launch ends
// with the epilogue
struct FusedOut { unsigned int* cnt; int64_t* i128; double* f64; int32_t* status; };
static int moments2d_profile_launch(const dpm_volume_desc* desc, int order, const uint32_t* const* d_images,
                                    const uint64_t* d_profile, uint64_t* d_acc, cudaStream_t st,
                                    const FusedOut* fused = nullptr, bool signed_i16 = false) {
  const int n_img = num_images(order);
  ImageSet s = make_set(desc, n_img, const_cast<uint32_t* const*>(d_images), true);
  const int jb = jbits_for(desc, n_img, true);
  if (jb > 21) return DPM_EOVERFLOW;
  const ProfGeom pg = profile_geom(desc, order);
  M2Extra ex;
  ex.sgn = signed_i16 ? 1 : 0;
  ex.off = desc->offset;
  ex.L = desc->L; ex.M = desc->M; ex.N = desc->N;
  ex.kind = acc_kind_of(desc);
  ex.prof = reinterpret_cast<const unsigned long long*>(d_profile);
  ex.WQ = pg.WQ;
  ex.ai = pg.ai;
  ex.cnt = fused ? fused->cnt : nullptr;
  ex.out_i128 = fused ? fused->i128 : nullptr;
  ex.out_f64 = fused ? fused->f64 : nullptr;
  ex.status = fused ? fused->status : nullptr;
  return launch_moments2d(s, desc->B, order, jb, d_acc, st, &ex);
}

static int zero_profile_buffers(const dpm_volume_desc* desc, int order, uint32_t* const* d_images,
                                uint64_t* d_profile, cudaStream_t st) {
  const int n_img = num_images(order);
  ImageSet s = make_set(desc, n_img, d_images, true);
  ZeroList z;
  z.n = 0;
  for (int k = 0; k < n_img; ++k) {
    if (k == DPM_IMG_ZX) continue;
    if (!s.img[k]) return DPM_EINVAL;
    z.p[z.n] = reinterpret_cast<uint8_t*>(s.img[k]);
    z.bytes[z.n++] = (uint64_t)(s.W[k] * s.H[k] * desc->B) * sizeof(uint32_t);
  }
  const ProfGeom pg = profile_geom(desc, order);
  z.p[z.n] = reinterpret_cast<uint8_t*>(d_profile);
  z.bytes[z.n++] = (uint64_t)(pg.WQ * desc->B) * sizeof(uint64_t);
  return zero_list_async(z, st);
}

int dpm_zero_profile_buffers(const dpm_volume_desc* desc, int order, uint32_t* const* d_images, uint64_t* d_profile,
                             void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_images || !d_profile) return DPM_EINVAL;
  return zero_profile_buffers(desc, order, d_images, d_profile, static_cast<cudaStream_t>(stream));
}

int dpm_project_profile_zeroed(const dpm_volume_desc* desc, const void* d_voxels, int order, uint32_t* const* d_images,
                               uint64_t* d_profile, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_images || !d_voxels || !d_profile) return DPM_EINVAL;
  for (int k = 0; k < num_images(order); ++k)
    if (k != DPM_IMG_ZX && !d_images[k]) return DPM_EINVAL;
  return project_profile_launch(desc, d_voxels, order, d_images, d_profile, static_cast<cudaStream_t>(stream));
}

int dpm_project_profile(const dpm_volume_desc* desc, const void* d_voxels, int order, uint32_t* const* d_images,
                        uint64_t* d_profile, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_images || !d_voxels || !d_profile) return DPM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = zero_profile_buffers(desc, order, d_images, d_profile, st);   // the pass starts while it drains (PDL)
  if (rc) return rc;
  return project_profile_launch(desc, d_voxels, order, d_images, d_profile, st);
}

int dpm_moments2d_profile(const dpm_volume_desc* desc, int order, const uint32_t* const* d_images,
                          const uint64_t* d_profile, uint64_t* d_acc, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_images || !d_profile || !d_acc) return DPM_EINVAL;
  const int n_img = num_images(order);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = zero_async(d_acc, (size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t), st);
  if (rc) return rc;
  return moments2d_profile_launch(desc, order, d_images, d_profile, d_acc, st);
}

int dpm_moments2d_profile_derive(const dpm_volume_desc* desc, int order, const uint32_t* const* d_images,
                                 const uint64_t* d_profile, uint64_t* d_acc, uint32_t* d_counters,
                                 int64_t* d_m3d_i128, double* d_m3d_f64, int32_t* d_status, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_images || !d_profile || !d_acc || !d_counters || !d_m3d_i128 || !d_status)
    return DPM_EINVAL;
  const int n_img = num_images(order);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ZeroList z;
  z.n = 2;
  z.p[0] = reinterpret_cast<uint8_t*>(d_acc);
  z.bytes[0] = (uint64_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t);
  z.p[1] = reinterpret_cast<uint8_t*>(d_counters);
  z.bytes[1] = (uint64_t)desc->B * sizeof(uint32_t);
  rc = zero_list_async(z, st);
  if (rc) return rc;
  FusedOut f;
  f.cnt = d_counters;
  f.i128 = d_m3d_i128;
  f.f64 = d_m3d_f64;
  f.status = d_status;
  return moments2d_profile_launch(desc, order, d_images, d_profile, d_acc, st, &f);
}

size_t dpm_partial_workspace_bytes(const dpm_volume_desc* desc, int order) {
  if (check_desc(desc) || check_order(order)) return 0;
  const ProfGeom pg = profile_geom(desc, order);
  return images_bytes(desc, num_images(order), nullptr, true) + align256((size_t)(pg.WQ * desc->B) * sizeof(uint64_t));
}

// fused (dpm_moments): the workspace is [images | profile | counters | acc]
// (acc_adjacent: d_acc directly follows the counters), and the moments launch
// ends with the epilogue; the profile, counters and accumulator are then one
// contiguous range to zero
static int moments_partial_impl(const dpm_volume_desc* desc, const void* d_voxels, int order, void* d_ws,
                                size_t ws_bytes, uint64_t* d_acc, void* stream, bool acc_adjacent,
                                const FusedOut* fused = nullptr, bool zero_acc = true) {
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_voxels || !d_acc) return DPM_EINVAL;
  if (ws_bytes < dpm_partial_workspace_bytes(desc, order) || !d_ws) return DPM_EWORKSPACE;
  const int n_img = num_images(order);
  size_t offs[DPM_MAX_IMAGES];
  const size_t ib = images_bytes(desc, n_img, offs, true);
  uint32_t* imgs[DPM_MAX_IMAGES];
  char* base = static_cast<char*>(d_ws);
  for (int k = 0; k < n_img; ++k) imgs[k] = k == DPM_IMG_ZX ? nullptr : reinterpret_cast<uint32_t*>(base + offs[k]);
  uint64_t* prof = reinterpret_cast<uint64_t*>(base + ib);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // one zeroing of the contiguous images + profile scratch, one of the accumulator
  // (or none when the caller's accumulator directly precedes it: dpm_moments)
  // (single-tile volumes: the images are stored whole by the kernel, zero only the profile and counters)
  const bool single = !layout_t(desc) && project_stream_single_tile(desc, d_voxels, n_img);
  const size_t tail = dpm_partial_workspace_bytes(desc, order) - ib +
                      (fused ? align256((size_t)desc->B * sizeof(unsigned int)) : 0);
  char* z0 = single ? reinterpret_cast<char*>(prof) : base;
  const size_t zb = (single ? 0 : ib) + tail + (acc_adjacent ? acc_bytes_of(desc, order) : 0);
  reset_launches();
  if (!acc_adjacent && zero_acc &&
      cudaMemsetAsync(d_acc, 0, (size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t), st) != cudaSuccess)
    return DPM_ECUDA;
  rc = zero_async(z0, zb, st);   // last before the projection kernel: it starts while this drains (PDL)
  if (rc) return rc;
  // signed-exact int16 (whole volumes through dpm_moments, layout T): the pass
  // sums the raw signed voxels -- no per-voxel offset add, the 16-bit unpack costs
  // what uint16's does -- and the epilogue adds offset x the box's moments
  // (derive_volume's OffsetBox), exactly
  const bool sgn = fused && desc->dtype == DPM_I16 && desc->offset != 0 && desc->z0 == 0 && layout_t(desc) &&
                   zstream_eligible(desc, d_voxels) && DPM_SIGNED_I16;
  rc = project_profile_launch(desc, d_voxels, order, imgs, prof, st, !single, sgn);
  if (rc) return rc;
  return moments2d_profile_launch(desc, order, imgs, prof, d_acc, st, fused, sgn);
}

int dpm_moments_partial(const dpm_volume_desc* desc, const void* d_voxels, int order, void* d_ws, size_t ws_bytes,
                        uint64_t* d_acc, void* stream) {
  return moments_partial_impl(desc, d_voxels, order, d_ws, ws_bytes, d_acc, stream, false);
}

int dpm_moments2d(const dpm_volume_desc* desc, int n_img, const uint32_t* const* d_images, int order,
                  uint64_t* d_acc, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || n_img < 3 || n_img > DPM_MAX_IMAGES || !d_images || !d_acc) return DPM_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ImageSet s = make_set(desc, n_img, const_cast<uint32_t* const*>(d_images));
  const int jb = jbits_for(desc, n_img);
  if (jb > 21) return DPM_EOVERFLOW;
  if (cudaMemsetAsync(d_acc, 0, (size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t), st) != cudaSuccess)
    return DPM_ECUDA;
  return launch_moments2d(s, desc->B, order, jb, d_acc, st);
}

int dpm_image_moments2d(const uint32_t* d_pixels, int64_t W, int64_t H, int64_t ai, int64_t aj, int order,
                        uint64_t* d_acc, void* stream) {
  reset_launches();
  if (!d_pixels || !d_acc || W < 1 || H < 1 || aj < 0 || check_order(order)) return DPM_EINVAL;
  int jb = 0;
  while ((int64_t(1) << jb) <= H - 1 + aj) ++jb;
  if (jb > 21) return DPM_EOVERFLOW;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ImageSet s{};
  s.n_img = 1;
  s.img[0] = const_cast<uint32_t*>(d_pixels);
  s.W[0] = W; s.H[0] = H; s.ai[0] = ai; s.aj[0] = aj;
  if (cudaMemsetAsync(d_acc, 0, (size_t)n2d(order) * 4 * sizeof(uint64_t), st) != cudaSuccess) return DPM_ECUDA;
  return launch_moments2d(s, 1, order, jb, d_acc, st);
}

int dpm_derive3d(const dpm_volume_desc* desc, const uint64_t* d_acc, int order, int acc_kind, int64_t* d_m3d_i128,
                 double* d_m3d_f64, int32_t* d_status, void* stream) {
  reset_launches();
  if (!desc || desc->B < 1 || check_order(order) || !d_acc || !d_m3d_i128 || !d_status) return DPM_EINVAL;
  if (acc_kind != DPM_ACC_IMAGES && acc_kind != DPM_ACC_PROFILE && acc_kind != DPM_ACC_PROFILE_T) return DPM_EINVAL;
  return launch_derive3d(d_acc, desc->B, num_images(order), order, acc_kind, d_m3d_i128, d_m3d_f64, d_status,
                         static_cast<cudaStream_t>(stream));
}

// Staged moments pass for single volumes the streaming (TMA) kernel cannot
// read in place -- row pitch not a multiple of 16 bytes, width not a multiple
// of the lane width (e.g. the odd cube sides of the reference's bench sweep):
// z-slabs are copied into a zero-padded pitched scratch (int16 + offset is
// converted to uint16 on the way), each slab runs the streaming moments pass
// in global coordinates into one accumulator, and the epilogue runs once.
// The padding columns are zero, so images are only wider, moments identical.
struct Staged {
  bool use;
  int64_t Lp, S;            // padded width, planes per slab
  dpm_volume_desc slab;     // geometry of a full slab (N = S)
};
static constexpr size_t kStagedSlabBytes = size_t(256) << 20;   // scratch budget per slab
static Staged staged_plan(const dpm_volume_desc* d) {
  Staged g;
  memset(&g, 0, sizeof(g));
  if (d->B != 1 || d->L < 32 || d->N < 8) return g;        // tiny / batched: the generic kernel
  const int64_t es_out = d->dtype == DPM_U8 ? 1 : 2;
  const int64_t es_in = d->dtype == DPM_U8 ? 1 : 2;
  const bool pitch_ok = (d->stride_y * es_in) % 16 == 0 && (d->stride_z * es_in) % 16 == 0;
  const int64_t lw = d->L > 128 ? 8 : 4;
  if (pitch_ok && d->L % lw == 0) return g;                  // the streaming kernel reads it in place
  const int64_t a = 16 / es_out;                             // pitch multiple (elements)
  g.Lp = (d->L + a - 1) / a * a;
  const int64_t plane = g.Lp * d->M * es_out;
  int64_t S = (int64_t)(kStagedSlabBytes / (size_t)plane);
  if (S >= 96) S = S / 96 * 96;                              // whole z-tiles of the streaming kernel
  S = imax64(8, imin64(S, d->N));
  g.S = S;
  g.slab = *d;
  g.slab.L = g.Lp;
  g.slab.N = S;
  g.slab.B = 1;
  g.slab.stride_y = g.Lp;
  g.slab.stride_z = g.Lp * d->M;
  g.slab.stride_b = g.Lp * d->M * S;
  g.slab.dtype = d->dtype == DPM_U8 ? DPM_U8 : DPM_U16;
  g.slab.offset = 0;
  g.use = true;
  return g;
}

size_t dpm_workspace_bytes(const dpm_volume_desc* desc, int order) {
  if (check_desc(desc) || check_order(order)) return 0;
  const int n_img = num_images(order);
  const size_t base = align256((size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t)) +
                      dpm_partial_workspace_bytes(desc, order) + align256((size_t)desc->B * sizeof(unsigned int));
  const Staged g = staged_plan(desc);
  if (!g.use) return base;
  const int64_t es_out = g.slab.dtype == DPM_U8 ? 1 : 2;
  const size_t staged = align256((size_t)(n_img * n2d(order) * 4) * sizeof(uint64_t)) +
                        dpm_partial_workspace_bytes(&g.slab, order) +
                        align256((size_t)(g.Lp * desc->M * g.S * es_out));
  return base > staged ? base : staged;
}

static int moments_staged(const dpm_volume_desc* desc, const Staged& g, const void* d_voxels, int order, void* d_ws,
                          int64_t* d_m3d_i128, double* d_m3d_f64, int32_t* d_status, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n_img = num_images(order);
  // workspace: [acc | slab images + profile | scratch]
  char* base = static_cast<char*>(d_ws);
  uint64_t* acc = reinterpret_cast<uint64_t*>(base);
  const size_t acc_bytes = align256((size_t)(n_img * n2d(order) * 4) * sizeof(uint64_t));
  char* pws = base + acc_bytes;
  const size_t pbytes = dpm_partial_workspace_bytes(&g.slab, order);
  char* scratch = pws + pbytes;
  if (cudaMemsetAsync(acc, 0, acc_bytes, st) != cudaSuccess) return DPM_ECUDA;
  int launches = 0;
  for (int64_t z = 0; z < desc->N; z += g.S) {
    dpm_volume_desc sd = g.slab;
    sd.N = imin64(g.S, desc->N - z);
    sd.stride_b = g.Lp * desc->M * sd.N;
    sd.z0 = desc->z0 + z;
    int rc = launch_pad_copy(desc, d_voxels, z, sd.N, g.Lp, scratch, st);
    if (rc) return rc;
    launches += 1;
    rc = moments_partial_impl(&sd, scratch, order, pws, pbytes, acc, stream, false, nullptr, false);
    launches += dpm_last_launch_count();
    if (rc) return rc;
  }
  const int rc = dpm_derive3d(desc, acc, order, acc_kind_of(&g.slab), d_m3d_i128, d_m3d_f64, d_status, stream);
  g_launches = launches + dpm_last_launch_count();
  return rc;
}

int dpm_check_envelope(int64_t L, int64_t M, int64_t N_global, int64_t vmax, int order) {
  if (L < 1 || M < 1 || N_global < 1 || vmax < 0 || check_order(order)) return DPM_EINVAL;
  // every |moment| and every partial sum <= mass * cmax^K, cmax = largest |logical coordinate|
  const long double mass = (long double)vmax * L * M * N_global;
  // (x +- 2z images of the classic layout, z +- 2x of layout T)
  const int64_t cmax = imax64(imax64(L, M), imax64(L + 2 * N_global, N_global + 2 * L));
  long double bound = mass;
  for (int k = 0; k < order; ++k) bound *= (long double)cmax;
  if (bound >= 0x1p126L) return DPM_EOVERFLOW;
  if (order == 6) {
    // the order-6 profile solve (derive3d, five unknowns) forms sums of up to
    // 2016 x the largest 3D moment: keep mass * max(L, M, N)^6 < 2^116
    const int64_t c3 = imax64(imax64(L, M), N_global);
    long double b6 = mass;
    for (int k = 0; k < 6; ++k) b6 *= (long double)c3;
    if (b6 >= 0x1p116L) return DPM_EOVERFLOW;
  }
  return DPM_OK;
}

int dpm_moments(const dpm_volume_desc* desc, const void* d_voxels, int order, void* d_ws, size_t ws_bytes,
                int64_t* d_m3d_i128, double* d_m3d_f64, int32_t* d_status, void* stream) {
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_voxels || !d_m3d_i128 || !d_status) return DPM_EINVAL;
  if (ws_bytes < dpm_workspace_bytes(desc, order) || !d_ws) return DPM_EWORKSPACE;
  const Staged g = staged_plan(desc);
  if (g.use) return moments_staged(desc, g, d_voxels, order, d_ws, d_m3d_i128, d_m3d_f64, d_status, stream);
  // workspace: [images | profile | counters | acc]
  char* pws = static_cast<char*>(d_ws);
  const size_t pbytes = dpm_partial_workspace_bytes(desc, order);
  const size_t cbytes = align256((size_t)desc->B * sizeof(unsigned int));
  uint64_t* acc = reinterpret_cast<uint64_t*>(pws + pbytes + cbytes);
  FusedOut f;
  f.cnt = reinterpret_cast<unsigned int*>(pws + pbytes);
  f.i128 = d_m3d_i128;
  f.f64 = d_m3d_f64;
  f.status = d_status;
  if (fused_batch_eligible(desc, d_voxels, order)) {
    // small uint8 volumes (<= 128 wide and deep, order 3): one memset of
    // [counters | acc] and ONE launch for projection, moments and epilogue
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    reset_launches();
    rc = zero_async(f.cnt, cbytes + acc_bytes_of(desc, order), st);
    if (rc) return rc;
    bool handled = false;
    rc = launch_fused_batch(desc, d_voxels, order, acc, f.cnt, d_m3d_i128, d_m3d_f64, d_status, st, &handled);
    if (rc || handled) return rc;
  }
  // memset, projection pass, one moments launch that ends with the epilogue
  return moments_partial_impl(desc, d_voxels, order, pws, pbytes, acc, stream, true, &f);
}

int dpm_acc_add(uint64_t* d_acc_out, const uint64_t* d_acc_in, int64_t count, void* stream);

int dpm_synth_noise_u16(uint16_t* d_out, int64_t L, int64_t M, int64_t z0, int64_t n_planes, uint64_t seed,
                        void* stream) {
  reset_launches();
  if (!d_out || L < 1 || M < 1 || z0 < 0 || n_planes < 1) return DPM_EINVAL;
  return launch_synth_noise(d_out, L, M, z0, n_planes, seed, static_cast<cudaStream_t>(stream));
}

int dpm_moments_acc_kind(const dpm_volume_desc* desc, int order) {
  if (check_desc(desc) || check_order(order)) return -DPM_EINVAL;
  return acc_kind_of(desc);
}

int dpm_moments_image_layout(const dpm_volume_desc* desc, int order, int img, int64_t* W, int64_t* H, int64_t* ai,
                             int64_t* aj) {
  if (check_desc(desc) || check_order(order) || img < 0 || img >= num_images(order) || img == DPM_IMG_ZX)
    return DPM_EINVAL;
  const ImageGeom g = mgeom(desc, img);
  if (W) *W = g.W;
  if (H) *H = g.H;
  if (ai) *ai = g.ai;
  if (aj) *aj = g.aj;
  return DPM_OK;
}

size_t dpm_direct_workspace_bytes(const dpm_volume_desc* desc, int order) {
  if (check_desc(desc) || check_order(order)) return 0;
  return align256((size_t)(desc->B * desc->N * n2d(order) * 4) * sizeof(uint64_t));
}

int dpm_direct_moments(const dpm_volume_desc* desc, const void* d_voxels, int order, int method, void* d_ws,
                       size_t ws_bytes, int64_t* d_m3d_i128, double* d_m3d_f64, void* stream) {
  reset_launches();
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_voxels || !d_m3d_i128 || (method != DPM_DIRECT_NAIVE && method != DPM_DIRECT_FACTORED))
    return DPM_EINVAL;
  if (!d_ws || ws_bytes < dpm_direct_workspace_bytes(desc, order)) return DPM_EWORKSPACE;
  return launch_direct3d(desc, d_voxels, order, method == DPM_DIRECT_NAIVE, static_cast<uint64_t*>(d_ws),
                         d_m3d_i128, d_m3d_f64, static_cast<cudaStream_t>(stream));
}

int dpm_last_launch_count(void) { return g_launches; }

const char* dpm_strerror(int code) {
  switch (code) {
    case DPM_OK: return "ok";
    case DPM_EINVAL: return "invalid argument";
    case DPM_EOVERFLOW: return "exactness envelope exceeded (accumulator would overflow)";
    case DPM_ECUDA: return "CUDA error";
    case DPM_EWORKSPACE: return "workspace too small";
    default: return "unknown error";
  }
}

}  // extern "C"

// elementwise uint64 add (combining per-slab limb partials on one device)
namespace dpm {
__global__ void acc_add_kernel(uint64_t* out, const uint64_t* in, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] += in[i];
}
}  // namespace dpm

extern "C" int dpm_acc_add(uint64_t* d_acc_out, const uint64_t* d_acc_in, int64_t count, void* stream) {
  dpm::reset_launches();
  if (!d_acc_out || !d_acc_in || count < 0) return DPM_EINVAL;
  if (count == 0) return DPM_OK;
  const int threads = 256;
  const unsigned grid = (unsigned)dpm::imin64((count + threads - 1) / threads, 1024);
  dpm::acc_add_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(d_acc_out, d_acc_in, count);
  dpm::note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}
