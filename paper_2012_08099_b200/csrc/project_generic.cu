// project_generic.cu -- shape-agnostic projection pass (any L, M, N, strides,
// batch, dtype).  Used for shapes the streaming kernel does not tile
// (unaligned rows, tiny volumes) and as an independent cross-check of it.
//
// One CTA owns a GBX x GBY x GBZ brick and privatises every image's footprint
// in shared memory (red.shared), then flushes non-zero cells with one
// red.global per cell.  Integer addition makes the result independent of
// scheduling.  Index maps: projection.py:7-14.
#include "dpm_common.cuh"

namespace dpm {

constexpr int GBX = 64, GBY = 4, GBZ = 16;
constexpr int GW1 = GBX + GBZ - 1;        // DIAG/ANTI brick footprint width
constexpr int GW2 = GBX + 2 * GBZ - 2;    // X2P/X2M brick footprint width
constexpr int GWQ = GBX + 3 * (GBZ - 1);  // profile footprint width (|t| <= 3)

struct GenericParams {
  const void* vox;
  int64_t L, M, N, B;
  int64_t sx, sy, sz, sb;   // element strides (sx = 1 except for the transposed view)
  int32_t offset;
  int64_t nbx, nby, nbz;
  ImageSet s;
  // moments mode: profile P[x + tq z] summed over y (uint64 [B][WQ]) instead of ZX
  unsigned long long* prof;
  int tq;
  int64_t WQ, qoff;
};

template <typename T>
__global__ void __launch_bounds__(256) project_generic_kernel(GenericParams p) {
  __shared__ uint32_t yz_s[GBZ][GBY];
  __shared__ uint32_t zx_s[GBX][GBZ + 1];
  __shared__ uint32_t dg_s[GBY][GW1];
  __shared__ uint32_t an_s[GBY][GW1];
  __shared__ uint32_t xp_s[GBY][GW2];
  __shared__ uint32_t xm_s[GBY][GW2];
  __shared__ uint32_t pq_s[GWQ];
  const int n_img = p.s.n_img;
  const bool prof = p.prof != nullptr;
  const int aq = p.tq < 0 ? -p.tq : p.tq;
  const int tid = threadIdx.x;
  const int xl = tid % GBX, yl = tid / GBX;
  const int64_t bricks_per_vol = p.nbx * p.nby * p.nbz;
  const int64_t total = bricks_per_vol * p.B;
  const T* vox = static_cast<const T*>(p.vox);

  for (int64_t brick = blockIdx.x; brick < total; brick += gridDim.x) {
    const int64_t b = brick / bricks_per_vol;
    int64_t r = brick - b * bricks_per_vol;
    const int64_t bz = r / (p.nbx * p.nby); r -= bz * p.nbx * p.nby;
    const int64_t by = r / p.nbx;
    const int64_t bx = r - by * p.nbx;
    const int64_t x0 = bx * GBX, y0 = by * GBY, z0 = bz * GBZ;

    for (int i = tid; i < GBZ * GBY; i += blockDim.x) (&yz_s[0][0])[i] = 0;
    for (int i = tid; i < GBX * (GBZ + 1); i += blockDim.x) (&zx_s[0][0])[i] = 0;
    for (int i = tid; i < GWQ; i += blockDim.x) pq_s[i] = 0;
    for (int i = tid; i < GBY * GW1; i += blockDim.x) { (&dg_s[0][0])[i] = 0; (&an_s[0][0])[i] = 0; }
    for (int i = tid; i < GBY * GW2; i += blockDim.x) { (&xp_s[0][0])[i] = 0; (&xm_s[0][0])[i] = 0; }
    __syncthreads();

    const int64_t x = x0 + xl, y = y0 + yl;
    const bool valid = (x < p.L) && (y < p.M);
    const T* row = vox + b * p.sb + y * p.sy + x * p.sx;
    uint32_t xy = 0;
    const int zcount = (int)imin64(GBZ, p.N - z0);
    for (int zl = 0; zl < zcount; ++zl) {
      uint32_t v = valid ? VoxelTraits<T>::get(row[(z0 + zl) * p.sz], p.offset) : 0u;
      xy += v;
      uint32_t s = v;
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((tid & 31) == 0 && s) atomicAdd(&yz_s[zl][yl], s);
      if (v) {
        if (prof) atomicAdd(&pq_s[p.tq > 0 ? xl + p.tq * zl : xl + aq * (GBZ - 1 - zl)], v);
        else atomicAdd(&zx_s[xl][zl], v);
        atomicAdd(&dg_s[yl][xl + zl], v);
        if (n_img > DPM_IMG_ANTI) atomicAdd(&an_s[yl][xl - zl + GBZ - 1], v);
        if (n_img > DPM_IMG_X2P) atomicAdd(&xp_s[yl][xl + 2 * zl], v);
        if (n_img > DPM_IMG_X2M) atomicAdd(&xm_s[yl][xl - 2 * zl + 2 * (GBZ - 1)], v);
      }
    }
    __syncthreads();

    // flush: brick-local cells -> global stored indices (bounds-checked)
    if (valid && xy) atomicAdd(p.s.img[DPM_IMG_XY] + b * p.s.W[0] * p.s.H[0] + y * p.L + x, xy);
    for (int i = tid; i < GBZ * GBY; i += blockDim.x) {
      const int zl = i / GBY, yy = i % GBY;
      const uint32_t v = yz_s[zl][yy];
      if (v) atomicAdd(p.s.img[DPM_IMG_YZ] + b * p.s.W[1] * p.s.H[1] + (z0 + zl) * p.M + (y0 + yy), v);
    }
    if (prof) {
      // local d -> stored x + tq z (tq > 0) or x - |tq| z + qoff (tq < 0)
      const int64_t g0 = p.tq > 0 ? x0 + p.tq * z0 : x0 - aq * (GBZ - 1) - aq * z0 + p.qoff;
      for (int i = tid; i < GWQ; i += blockDim.x) {
        const uint32_t v = pq_s[i];
        if (v) atomicAdd(p.prof + b * p.WQ + g0 + i, (unsigned long long)v);
      }
    } else {
      for (int i = tid; i < GBX * GBZ; i += blockDim.x) {
        const int xx = i / GBZ, zl = i % GBZ;
        const uint32_t v = zx_s[xx][zl];
        if (v) atomicAdd(p.s.img[DPM_IMG_ZX] + b * p.s.W[2] * p.s.H[2] + (x0 + xx) * p.N + (z0 + zl), v);
      }
    }
    for (int i = tid; i < GBY * GW1; i += blockDim.x) {
      const int yy = i / GW1, d = i % GW1;
      const uint32_t vd = dg_s[yy][d];
      const int64_t W = p.s.W[DPM_IMG_DIAG];
      if (vd) atomicAdd(p.s.img[DPM_IMG_DIAG] + b * W * p.M + (y0 + yy) * W + (x0 + z0 + d), vd);
      if (n_img > DPM_IMG_ANTI) {
        const uint32_t va = an_s[yy][d];
        // local a = xl - zl + GBZ-1  ->  stored x - z + N - 1
        if (va) atomicAdd(p.s.img[DPM_IMG_ANTI] + b * W * p.M + (y0 + yy) * W + (d + x0 - z0 + p.N - GBZ), va);
      }
    }
    if (n_img > DPM_IMG_X2P) {
      for (int i = tid; i < GBY * GW2; i += blockDim.x) {
        const int yy = i / GW2, d = i % GW2;
        const int64_t W = p.s.W[DPM_IMG_X2P];
        const uint32_t vp = xp_s[yy][d];
        if (vp) atomicAdd(p.s.img[DPM_IMG_X2P] + b * W * p.M + (y0 + yy) * W + (x0 + 2 * z0 + d), vp);
        if (n_img > DPM_IMG_X2M) {
          const uint32_t vm = xm_s[yy][d];
          // local a = xl - 2zl + 2(GBZ-1)  ->  stored x - 2z + 2(N-1)
          if (vm) atomicAdd(p.s.img[DPM_IMG_X2M] + b * W * p.M + (y0 + yy) * W + (d + x0 - 2 * z0 + 2 * p.N - 2 * GBZ), vm);
        }
      }
    }
    __syncthreads();
  }
}

int profile_shift(int n_img);

// prof != nullptr: moments mode (the profile along x + t z replaces ZX).
// transposed: the volume is read as V'(x', y, z') = V(z', y, x') -- the
// moments pipeline's layout T (capi.cu) for shapes the z-streaming kernel
// cannot read; `s` then carries the layout-T geometry
int launch_project_generic(const dpm_volume_desc* d, const void* vox, const ImageSet& s, unsigned long long* prof,
                           cudaStream_t st, bool transposed) {
  GenericParams p;
  p.vox = vox; p.M = d->M; p.B = d->B;
  p.sy = d->stride_y; p.sb = d->stride_b; p.offset = d->offset;
  if (transposed) { p.L = d->N; p.N = d->L; p.sx = d->stride_z; p.sz = 1; }
  else { p.L = d->L; p.N = d->N; p.sx = 1; p.sz = d->stride_z; }
  p.prof = prof;
  p.tq = profile_shift(s.n_img);
  {
    const int at = p.tq < 0 ? -p.tq : p.tq;
    p.WQ = p.L + at * (p.N - 1);
    p.qoff = p.tq < 0 ? at * (p.N - 1) : 0;
  }
  p.nbx = (p.L + GBX - 1) / GBX; p.nby = (p.M + GBY - 1) / GBY; p.nbz = (p.N + GBZ - 1) / GBZ;
  p.s = s;
  const int64_t total = p.nbx * p.nby * p.nbz * p.B;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)imin64(total, (int64_t)sms * 8);
  switch (d->dtype) {
    case DPM_U8:  project_generic_kernel<uint8_t><<<grid, 256, 0, st>>>(p); break;
    case DPM_U16: project_generic_kernel<uint16_t><<<grid, 256, 0, st>>>(p); break;
    default:      project_generic_kernel<int16_t><<<grid, 256, 0, st>>>(p); break;
  }
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

// ---- staged copies for the moments pass (capi.cu, moments_staged) ----------
// planes [z, z+n) of one volume -> zero-padded pitched scratch [n][M][Lp]; int16
// + offset becomes uint16 (the caller guarantees 0..65535), so the slab runs
// the streaming kernel with offset 0.  One warp per row, coalesced both ways.
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) pad_copy_kernel(const Tin* src, int64_t sy, int64_t sz, int64_t L, int64_t M,
                                                       int64_t n, int32_t offset, Tout* dst, int64_t Lp) {
  const int64_t rows = M * n;
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * 8) {
    const int64_t zz = r / M, yy = r - zz * M;
    const Tin* s = src + zz * sz + yy * sy;
    Tout* d = dst + r * Lp;
    for (int64_t x = lane; x < Lp; x += 32) {
      uint32_t v = 0;
      if (x < L) v = (uint32_t)((int32_t)s[x] + offset);
      d[x] = (Tout)v;
    }
  }
}

int launch_pad_copy(const dpm_volume_desc* d, const void* vox, int64_t z, int64_t n, int64_t Lp, void* dst,
                    cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t rows = d->M * n;
  const int grid = (int)imax64(1, imin64((rows + 7) / 8, (int64_t)sms * 16));
  switch (d->dtype) {
    case DPM_U8:
      pad_copy_kernel<uint8_t, uint8_t><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(vox) + z * d->stride_z,
                                                            d->stride_y, d->stride_z, d->L, d->M, n, 0,
                                                            static_cast<uint8_t*>(dst), Lp);
      break;
    case DPM_U16:
      pad_copy_kernel<uint16_t, uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(vox) + z * d->stride_z,
                                                              d->stride_y, d->stride_z, d->L, d->M, n, 0,
                                                              static_cast<uint16_t*>(dst), Lp);
      break;
    default:
      pad_copy_kernel<int16_t, uint16_t><<<grid, 256, 0, st>>>(static_cast<const int16_t*>(vox) + z * d->stride_z,
                                                             d->stride_y, d->stride_z, d->L, d->M, n, d->offset,
                                                             static_cast<uint16_t*>(dst), Lp);
  }
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
