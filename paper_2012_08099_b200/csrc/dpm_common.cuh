// dpm_common.cuh -- shared geometry and launch plumbing for the DPM kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/dpm_b200.h"

namespace dpm {

// Stored image geometry and logical-origin offsets.  Index maps follow the
// reference (projection.py:7-14): XY (x,y), YZ (y,z), ZX (z,x), DIAG (x+z,y),
// ANTI (x-z+N-1,y); the order-5/6 extension adds X2P (x+2z,y) and
// X2M (x-2z+2(N-1),y).  (ai, aj) shift stored indices to logical global
// coordinates of a z-slab starting at global plane z0; for a whole
// volume (z0 = 0) ai of ANTI is -(N-1), the reference's origin_offset
// (projection.py:189-191, drt2d.py:196-208).
struct ImageGeom { int64_t W, H, ai, aj; };

__host__ __device__ inline ImageGeom image_geom(int64_t L, int64_t M, int64_t N, int64_t z0, int img) {
  switch (img) {
    case DPM_IMG_XY:   return {L, M, 0, 0};
    case DPM_IMG_YZ:   return {M, N, 0, z0};
    case DPM_IMG_ZX:   return {N, L, z0, 0};
    case DPM_IMG_DIAG: return {L + N - 1, M, z0, 0};
    case DPM_IMG_ANTI: return {L + N - 1, M, -(N - 1) - z0, 0};
    case DPM_IMG_X2P:  return {L + 2 * N - 2, M, 2 * z0, 0};
    default:           return {L + 2 * N - 2, M, -2 * (N - 1) - 2 * z0, 0};
  }
}

__host__ __device__ inline int num_images(int order) { return order <= 3 ? 4 : order + 1; }
__host__ __device__ inline int n2d(int order) { return (order + 1) * (order + 2) / 2; }
__host__ __device__ inline int n3d(int order) { return (order + 1) * (order + 2) * (order + 3) / 6; }

// p-major 2D moment slot: p then q (q <= K-p).
__host__ __device__ inline int idx2(int order, int p, int q) { return p * (order + 1) - p * (p - 1) / 2 + q; }

// lexicographic (p,q,r) slot == moment_indices (moments3d.py:46-54).
__host__ __device__ inline int idx3(int order, int p, int q, int r) {
  int n = 0;
  for (int a = 0; a < p; ++a) { int s = order - a; n += (s + 1) * (s + 2) / 2; }
  int s = order - p;
  for (int b = 0; b < q; ++b) n += s - b + 1;
  return n + r;
}

// Per-image pointer/geometry pack passed by value to kernels.
struct ImageSet {
  uint32_t* img[DPM_MAX_IMAGES];
  int64_t W[DPM_MAX_IMAGES];
  int64_t H[DPM_MAX_IMAGES];
  int64_t ai[DPM_MAX_IMAGES];
  int64_t aj[DPM_MAX_IMAGES];
  int n_img;
};

template <typename T> struct VoxelTraits;
template <> struct VoxelTraits<uint8_t>  { static __device__ __forceinline__ uint32_t get(uint8_t v, int32_t) { return v; } };
template <> struct VoxelTraits<uint16_t> { static __device__ __forceinline__ uint32_t get(uint16_t v, int32_t) { return v; } };
template <> struct VoxelTraits<int16_t>  { static __device__ __forceinline__ uint32_t get(int16_t v, int32_t off) { return (uint32_t)((int32_t)v + off); } };

// Optional parts of the moments kernel launch (launch_moments2d): the
// profile's 1D moments in the same grid, and the fused epilogue (the last
// block of each volume runs derive_volume; cnt[B] zeroed by the caller).
struct M2Extra {
  // signed-exact int16: pixels are int32 (two's complement sums), the profile
  // int64, and the epilogue adds off * (the box's moments); off = 0: plain
  int sgn;
  int64_t off, L, M, N;
  const unsigned long long* prof;
  int64_t WQ, ai;
  int kind;                 // accumulator kind of the fused epilogue (DPM_ACC_PROFILE / _T)
  unsigned int* cnt;
  int64_t* out_i128;
  double* out_f64;
  int32_t* status;
};

// thread-local count of kernels the last C-ABI call enqueued
void note_launches(int n);
void reset_launches();

}  // namespace dpm

namespace dpm { void report_cuda_error(cudaError_t e, const char* where); }
#define DPM_CUDA_CHECK_LAUNCH()                                  \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) {                                     \
      dpm::report_cuda_error(_e, __FILE__);                      \
      return DPM_ECUDA;                                          \
    }                                                            \
  } while (0)

namespace dpm {
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
}  // namespace dpm

namespace dpm {
// Programmatic dependent launch (PDL).  The pipeline's kernels are launched
// with programmatic stream serialisation, so a kernel starts while its
// predecessor drains: it runs its prologue (shared-memory setup, barrier
// init, the first TMA loads of the VOLUME, which earlier stream work
// produced) and calls pdl_wait() before it touches anything the predecessor
// writes (zeroed images / accumulators, images to reduce).  Predecessors call
// pdl_trigger() early.  Without a programmatic dependency both are no-ops.
// DPM_PDL=0 launches everything with plain stream order (A/B).
#ifndef DPM_PDL
#define DPM_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... ExpTypes, typename... ActTypes>
inline cudaError_t launch_pdl(void (*kern)(ExpTypes...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              ActTypes&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = DPM_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<ActTypes&&>(args)...);
}

// zero `bytes` at `p` (256-byte aligned) with a kernel that lets its
// dependent start right away (cudaMemsetAsync is not a kernel, so it cannot
// take part in PDL); counts as one launch
int zero_async(void* p, size_t bytes, cudaStream_t st);

// Dynamic shared-memory opt-in of one kernel, set once per DEVICE (the
// attribute lives in that device's context; a process-wide once-flag would
// leave a second GPU unconfigured).  `mask` is the kernel's own bit set of
// configured device ordinals.
template <typename KernelT>
inline int ensure_smem(KernelT kern, size_t bytes, std::atomic<uint64_t>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DPM_ECUDA;
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return DPM_OK;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    report_cuda_error(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    return DPM_ECUDA;
  }
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return DPM_OK;
}
}  // namespace dpm
