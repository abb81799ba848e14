// TMA access-pattern ceiling: 4-D boxes (x 256, y YB, z ZB, b 1) of uint16 streamed
// through S shared-memory stages by a persistent grid, consumers touch the data
// (one LDS.128 per lane per row) and release stages with a CTA barrier.
//   ZITER = 0: a CTA walks consecutive y (box = x-tile x 1 row x ZB planes): round-1 kernel
//   ZITER = 1: a CTA walks consecutive z-steps of one (x-tile, y-group) column: z-stream kernel
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred d;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1;\n@!d bra W_%=;\n}" ::"r"(bar), "r"(ph) : "memory");
}

template <int S, int YB, int ZB, int ZITER>
__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ CUtensorMap map, int L, int M, int N, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr uint32_t BYTES = 256 * YB * ZB * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * BYTES);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int ntx = L / 256, nty = M / YB, ntz = N / ZB;
  const long long total = (long long)ntx * nty * ntz;   // boxes
  long long s0, s1;
  s0 = total * blockIdx.x / gridDim.x; s1 = total * (blockIdx.x + 1) / gridDim.x;
  auto issue = [&](long long s, int st) {
    int x, y, z;
    if (ZITER) { z = (int)(s % ntz); long long c = s / ntz; x = (int)(c % ntx); y = (int)(c / ntx); }
    else { y = (int)(s % nty); long long c = s / nty; x = (int)(c % ntx); z = (int)(c / ntx); }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(BYTES));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(sa(sm + st * BYTES)), "l"((uint64_t)&map), "r"(x * 256), "r"(y * YB), "r"(z * ZB), "r"(0), "r"(sa(&full[st])) : "memory");
  };
  long long next = s0;
  if (tid == 0) for (int i = 0; i < S && next < s1; ++i) issue(next++, i);
  uint32_t acc = 0;
  int st = 0; uint32_t ph = 0;
  for (long long s = s0; s < s1; ++s) {
    wait(sa(&full[st]), ph);
    const uint4* tile = reinterpret_cast<const uint4*>(sm + st * BYTES);
    for (int t = warp; t < YB * ZB; t += 8) { uint4 v = tile[t * 32 + lane]; acc += v.x ^ v.y ^ v.z ^ v.w; }
    __syncthreads();
    if (tid == 0 && next < s1) issue(next++, st);
    if (++st == S) { st = 0; ph ^= 1; }
  }
  if (acc == 0x1234567u) out[0] = acc;
}

template <int S, int YB, int ZB, int ZITER>
int run(void* ptr, int L, int M, int N, int grid, uint32_t* out, PFN_cuTensorMapEncodeTiled_v12000 enc) {
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)L, (cuuint64_t)M, (cuuint64_t)N, 1};
  cuuint64_t str[3] = {(cuuint64_t)L * 2, (cuuint64_t)L * M * 2, (cuuint64_t)L * M * N * 2};
  cuuint32_t box[4] = {256, YB, ZB, 1}, es[4] = {1, 1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode fail\n"); return 1; }
  size_t smem = (size_t)S * 256 * YB * ZB * 2 + S * 8;
  CK(cudaFuncSetAttribute(k<S, YB, ZB, ZITER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<S, YB, ZB, ZITER><<<grid, 256, smem>>>(map, L, M, N, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<S, YB, ZB, ZITER><<<grid, 256, smem>>>(map, L, M, N, out);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("S=%d box y%d z%d %s grid=%d smem=%zuKB: %.0f GB/s\n", S, YB, ZB, ZITER ? "z-iter" : "y-iter", grid, smem >> 10,
         5.0 * L * M * (double)N * 2 / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int L = 2048, M = 2048, N = 1024;   // 8 GiB of uint16
  void* ptr; CK(cudaMalloc(&ptr, (size_t)L * M * N * 2)); CK(cudaMemset(ptr, 1, (size_t)L * M * N * 2));
  uint32_t* out; CK(cudaMalloc(&out, 64));
  run<4, 1, 96, 0>(ptr, L, M, 960, 148, out, enc);
  run<4, 1, 64, 0>(ptr, L, M, N, 148, out, enc);
  run<4, 8, 8, 1>(ptr, L, M, N, 148, out, enc);
  run<5, 8, 8, 1>(ptr, L, M, N, 148, out, enc);
  run<6, 8, 8, 1>(ptr, L, M, N, 148, out, enc);
  run<4, 8, 8, 0>(ptr, L, M, N, 148, out, enc);
  run<3, 16, 8, 1>(ptr, L, M, N, 148, out, enc);
  run<4, 4, 16, 1>(ptr, L, M, N, 148, out, enc);
  run<4, 2, 32, 1>(ptr, L, M, N, 148, out, enc);
  run<4, 32, 2, 1>(ptr, L, M, N, 148, out, enc);
  return 0;
}
