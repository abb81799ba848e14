// Microbenchmarks that size the projection kernel's design choices on B200:
// streaming read bandwidth, L2 reduction (red.global) throughput, shared-memory
// atomic throughput, shuffle throughput.  Standalone; not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void read_bw(const uint4* __restrict__ p, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  #pragma unroll 8
  for (; i < n; i += stride) { uint4 v = __ldcs(p + i); acc += v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void red_global(uint32_t* img, uint32_t mask, int iters, int spread) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t a = tid * spread;
  for (int k = 0; k < iters; ++k) {
    atomicAdd(img + ((a + k * 7919u * spread) & mask), a + k);
  }
}

__global__ void atom_shared(uint32_t* out, int iters) {
  __shared__ uint32_t s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t base = threadIdx.x;
  #pragma unroll 4
  for (int k = 0; k < iters; ++k) atomicAdd(&s[(base + k * 37) & 8191], base + k);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}

__global__ void lds_sts(uint32_t* out, int iters) {
  __shared__ uint4 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_uint4(i, 0, 0, 0);
  __syncthreads();
  uint32_t acc = 0;
  uint32_t idx = threadIdx.x;
  #pragma unroll 8
  for (int k = 0; k < iters; ++k) { uint4 v = s[(idx + k * 32) & 2047]; acc += v.x + v.y + v.z + v.w; }
  if (acc == 7) out[0] = acc;
}

__global__ void shfl_tp(uint32_t* out, int iters) {
  uint32_t a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  #pragma unroll 8
  for (int k = 0; k < iters; ++k) {
    a += __shfl_down_sync(0xffffffffu, b, 1);
    b += __shfl_down_sync(0xffffffffu, c, 1);
    c += __shfl_down_sync(0xffffffffu, d, 1);
    d += __shfl_down_sync(0xffffffffu, a, 1);
  }
  if ((a ^ b ^ c ^ d) == 7) out[0] = a;
}

__global__ void iadd_tp(uint32_t* out, int iters, uint32_t x) {
  uint32_t a[8];
  #pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  #pragma unroll 4
  for (int k = 0; k < iters; ++k) {
    #pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + x + a[(i + 1) & 7];
  }
  uint32_t r = 0;
  #pragma unroll
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 7) out[0] = r;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d L2 %d MB smem/blk optin %zu clock %d kHz\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin, prop.clockRate);
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  uint32_t* out; CK(cudaMalloc(&out, 1 << 20));
  // 1. streaming read bandwidth
  size_t bytes = 8ull << 30;
  uint4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  for (int bpsm : {2, 4, 8}) for (int thr : {256, 512}) {
    int grid = sms * bpsm;
    read_bw<<<grid, thr>>>(buf, bytes / 16, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) read_bw<<<grid, thr>>>(buf, bytes / 16, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("read_bw grid=%d thr=%d: %.1f GB/s\n", grid, thr, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  // 2. red.global throughput (addresses in L2)
  uint32_t* img; CK(cudaMalloc(&img, 64 << 20)); CK(cudaMemset(img, 0, 64 << 20));
  for (int spread : {1, 33}) for (uint32_t mask : {(1u << 20) - 1, (1u << 24) - 1}) {
    int grid = sms * 8, thr = 256, iters = 256;
    red_global<<<grid, thr>>>(img, mask, iters, spread);
    cudaEventRecord(e0);
    red_global<<<grid, thr>>>(img, mask, iters, spread);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * thr * iters;
    printf("red_global spread=%d span=%u words: %.1f G atomics/s\n", spread, mask + 1, n / (ms * 1e-3) / 1e9);
  }
  // 3. shared atomics
  {
    int grid = sms * 4, thr = 512, iters = 4096;
    atom_shared<<<grid, thr>>>(out, iters);
    cudaEventRecord(e0); atom_shared<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * thr * iters;
    printf("atom_shared: %.1f G lane-atomics/s (%.2f per SM per ns)\n", n / (ms * 1e-3) / 1e9, n / (ms * 1e6) / sms);
  }
  {
    int grid = sms * 4, thr = 512, iters = 4096;
    lds_sts<<<grid, thr>>>(out, iters);
    cudaEventRecord(e0); lds_sts<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * thr * iters * 16;
    printf("lds128: %.1f TB/s (%.1f B per SM per ns)\n", n / (ms * 1e-3) / 1e12, n / (ms * 1e6) / sms);
  }
  {
    int grid = sms * 4, thr = 512, iters = 4096;
    shfl_tp<<<grid, thr>>>(out, iters);
    cudaEventRecord(e0); shfl_tp<<<grid, thr>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * thr * iters * 4;
    printf("shfl: %.1f G lane-shfl/s (%.2f per SM per ns)\n", n / (ms * 1e-3) / 1e9, n / (ms * 1e6) / sms);
  }
  {
    int grid = sms * 4, thr = 512, iters = 4096;
    iadd_tp<<<grid, thr>>>(out, iters, 3);
    cudaEventRecord(e0); iadd_tp<<<grid, thr>>>(out, iters, 3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)grid * thr * iters * 8;
    printf("iadd3: %.1f T lane-ops/s (%.2f per SM per ns)\n", n / (ms * 1e-3) / 1e12, n / (ms * 1e6) / sms);
  }
  return 0;
}
