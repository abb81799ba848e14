// capi.cu -- the C ABI (include/dpm_b200.h): argument validation, workspace
// carving and stage dispatch.  No allocation, no synchronisation.
#include <cstring>
#include "dpm_common.cuh"

namespace dpm {

static thread_local int g_launches = 0;
void note_launches(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

int launch_project_generic(const dpm_volume_desc* d, const void* vox, const ImageSet& s, cudaStream_t st);
int launch_project_stream(const dpm_volume_desc* d, const void* vox, const ImageSet& s, void* ws, size_t ws_bytes,
                          cudaStream_t st, bool* handled);
size_t project_stream_workspace(const dpm_volume_desc* d, int n_img);
int launch_moments2d(const ImageSet& s, int64_t B, int order, int jbits, uint64_t* acc, cudaStream_t st);
int launch_derive3d(const uint64_t* acc, int64_t B, int n_img, int order, int64_t* out_i128,
                    double* out_f64, int32_t* status, cudaStream_t st);
int launch_synth_noise(uint16_t* out, int64_t L, int64_t M, int64_t z0, int64_t nz, uint64_t seed, cudaStream_t st);

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

static int check_order(int order) { return (order >= 3 && order <= DPM_MAX_ORDER) ? DPM_OK : DPM_EINVAL; }

static ImageSet make_set(const dpm_volume_desc* d, int n_img, uint32_t* const* imgs) {
  ImageSet s;
  memset(&s, 0, sizeof(s));
  s.n_img = n_img;
  for (int k = 0; k < n_img; ++k) {
    const ImageGeom g = image_geom(d->L, d->M, d->N, d->z0, k);
    s.img[k] = imgs ? imgs[k] : nullptr;
    s.W[k] = g.W; s.H[k] = g.H; s.ai[k] = g.ai; s.aj[k] = g.aj;
  }
  return s;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t images_bytes(const dpm_volume_desc* d, int n_img, size_t* offs) {
  size_t total = 0;
  for (int k = 0; k < n_img; ++k) {
    const ImageGeom g = image_geom(d->L, d->M, d->N, d->z0, k);
    if (offs) offs[k] = total;
    total += align256((size_t)(g.W * g.H * d->B) * sizeof(uint32_t));
  }
  return total;
}

static int jbits_for(const dpm_volume_desc* d, int n_img) {
  int64_t jmax = 0;
  for (int k = 0; k < n_img; ++k) {
    const ImageGeom g = image_geom(d->L, d->M, d->N, d->z0, k);
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
  bool handled = false;
  rc = launch_project_stream(desc, d_voxels, s, d_ws, ws_bytes, st, &handled);
  if (rc || handled) return rc;
  return launch_project_generic(desc, d_voxels, s, st);
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
  return launch_project_generic(desc, d_voxels, s, st);
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

int dpm_derive3d(const dpm_volume_desc* desc, const uint64_t* d_acc, int order, int64_t* d_m3d_i128,
                 double* d_m3d_f64, int32_t* d_status, void* stream) {
  reset_launches();
  if (!desc || desc->B < 1 || check_order(order) || !d_acc || !d_m3d_i128 || !d_status) return DPM_EINVAL;
  return launch_derive3d(d_acc, desc->B, num_images(order), order, d_m3d_i128, d_m3d_f64, d_status,
                         static_cast<cudaStream_t>(stream));
}

size_t dpm_workspace_bytes(const dpm_volume_desc* desc, int order) {
  if (check_desc(desc) || check_order(order)) return 0;
  const int n_img = num_images(order);
  size_t total = images_bytes(desc, n_img, nullptr);
  total += align256((size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t));
  total += align256(project_stream_workspace(desc, n_img));
  return total;
}

int dpm_check_envelope(int64_t L, int64_t M, int64_t N_global, int64_t vmax, int order) {
  if (L < 1 || M < 1 || N_global < 1 || vmax < 0 || check_order(order)) return DPM_EINVAL;
  // every |moment| and every partial sum <= mass * cmax^K, cmax = largest |logical coordinate|
  const long double mass = (long double)vmax * L * M * N_global;
  const int64_t cmax = imax64(imax64(L, M), L + 2 * N_global);
  long double bound = mass;
  for (int k = 0; k < order; ++k) bound *= (long double)cmax;
  return bound < 0x1p126L ? DPM_OK : DPM_EOVERFLOW;
}

int dpm_moments(const dpm_volume_desc* desc, const void* d_voxels, int order, void* d_ws, size_t ws_bytes,
                int64_t* d_m3d_i128, double* d_m3d_f64, int32_t* d_status, void* stream) {
  int rc = check_desc(desc);
  if (rc) return rc;
  if (check_order(order) || !d_voxels || !d_m3d_i128 || !d_status) return DPM_EINVAL;
  if (ws_bytes < dpm_workspace_bytes(desc, order) || !d_ws) return DPM_EWORKSPACE;
  const int n_img = num_images(order);
  size_t offs[DPM_MAX_IMAGES];
  const size_t ib = images_bytes(desc, n_img, offs);
  uint32_t* imgs[DPM_MAX_IMAGES];
  char* base = static_cast<char*>(d_ws);
  for (int k = 0; k < n_img; ++k) imgs[k] = reinterpret_cast<uint32_t*>(base + offs[k]);
  uint64_t* acc = reinterpret_cast<uint64_t*>(base + ib);
  const size_t acc_bytes = align256((size_t)(desc->B * n_img * n2d(order) * 4) * sizeof(uint64_t));
  void* pws = base + ib + acc_bytes;
  const size_t pws_bytes = ws_bytes - ib - acc_bytes;
  int launches = 0;
  rc = dpm_project(desc, d_voxels, n_img, imgs, pws, pws_bytes, stream);
  launches += dpm_last_launch_count();
  if (rc) return rc;
  rc = dpm_moments2d(desc, n_img, imgs, order, acc, stream);
  launches += dpm_last_launch_count();
  if (rc) return rc;
  rc = dpm_derive3d(desc, acc, order, d_m3d_i128, d_m3d_f64, d_status, stream);
  launches += dpm_last_launch_count();
  g_launches = launches;
  return rc;
}

int dpm_acc_add(uint64_t* d_acc_out, const uint64_t* d_acc_in, int64_t count, void* stream);

int dpm_synth_noise_u16(uint16_t* d_out, int64_t L, int64_t M, int64_t z0, int64_t n_planes, uint64_t seed,
                        void* stream) {
  reset_launches();
  if (!d_out || L < 1 || M < 1 || z0 < 0 || n_planes < 1) return DPM_EINVAL;
  return launch_synth_noise(d_out, L, M, z0, n_planes, seed, static_cast<cudaStream_t>(stream));
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
