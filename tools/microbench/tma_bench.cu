// Ceiling of the projection kernel's TMA pattern: 4-D boxes (x 256, y 1, z ZB, b 1) of uint16
// streamed through S shared-memory stages by a persistent grid; consumers touch the data
// (one LDS.128 per lane per plane) and release stages either with a CTA barrier per step
// (MODE 0) or with an mbarrier "empty" protocol (MODE 1).
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

template <int S, int ZB, int MODE>
__global__ void __launch_bounds__(512, 1) k(const __grid_constant__ CUtensorMap map, int L, int M, int N, uint32_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr uint32_t BYTES = 256 * ZB * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * BYTES);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(sa(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int ntx = L / 256, ntz = N / ZB;
  const long long total = (long long)ntx * ntz * M;
  const long long s0 = total * blockIdx.x / gridDim.x, s1 = total * (blockIdx.x + 1) / gridDim.x;
  auto issue = [&](long long s, int st) {
    const int col = (int)(s / M), y = (int)(s % M);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(BYTES));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(sa(sm + st * BYTES)), "l"((uint64_t)&map), "r"((col % ntx) * 256), "r"(y), "r"((col / ntx) * ZB), "r"(0), "r"(sa(&full[st])) : "memory");
  };
  long long next = s0;
  if (tid == 0) for (int i = 0; i < S && next < s1; ++i) issue(next++, i);
  uint32_t acc = 0;
  int st = 0; uint32_t ph = 0;
  for (long long s = s0; s < s1; ++s) {
    wait(sa(&full[st]), ph);
    const uint4* tile = reinterpret_cast<const uint4*>(sm + st * BYTES);
    for (int t = warp; t < ZB; t += 16) { uint4 v = tile[t * 32 + lane]; acc += v.x ^ v.y ^ v.z ^ v.w; }
    if (MODE == 0) {
      __syncthreads();
      if (tid == 0 && next < s1) issue(next++, st);
    } else {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
      if (tid == 0 && next < s1) { wait(sa(&empty[st]), ph); issue(next++, st); }
    }
    if (++st == S) { st = 0; ph ^= 1; }
  }
  if (acc == 0x1234567u) out[0] = acc;
}

template <int S, int ZB, int MODE>
int run(CUtensorMap* maps, void* ptr, int L, int M, int N, int grid, uint32_t* out, PFN_cuTensorMapEncodeTiled_v12000 enc) {
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)L, (cuuint64_t)M, (cuuint64_t)N, 1};
  cuuint64_t str[3] = {(cuuint64_t)L * 2, (cuuint64_t)L * M * 2, (cuuint64_t)L * M * N * 2};
  cuuint32_t box[4] = {256, 1, ZB, 1}, es[4] = {1, 1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode fail\n"); return 1; }
  size_t smem = (size_t)S * 256 * ZB * 2 + 2 * S * 8;
  CK(cudaFuncSetAttribute(k<S, ZB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<S, ZB, MODE><<<grid, 512, smem>>>(map, L, M, N, out);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<S, ZB, MODE><<<grid, 512, smem>>>(map, L, M, N, out);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("S=%d ZB=%d mode=%d grid=%d smem=%zuKB: %.0f GB/s\n", S, ZB, MODE, grid, smem >> 10, 5.0 * L * M * (double)N * 2 / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int L = 1024, M = 1024, N = 2048;   // 4 GiB of uint16
  void* ptr; CK(cudaMalloc(&ptr, (size_t)L * M * N * 2)); CK(cudaMemset(ptr, 1, (size_t)L * M * N * 2));
  uint32_t* out; CK(cudaMalloc(&out, 64));
  run<4, 64, 0>(nullptr, ptr, L, M, N, 148, out, enc);
  run<5, 64, 0>(nullptr, ptr, L, M, N, 148, out, enc);
  run<6, 64, 0>(nullptr, ptr, L, M, N, 148, out, enc);
  run<4, 64, 1>(nullptr, ptr, L, M, N, 148, out, enc);
  run<6, 64, 1>(nullptr, ptr, L, M, N, 148, out, enc);
  run<8, 32, 0>(nullptr, ptr, L, M, N, 148, out, enc);
  run<12, 32, 1>(nullptr, ptr, L, M, N, 148, out, enc);
  run<12, 16, 1>(nullptr, ptr, L, M, N, 148, out, enc);
  run<3, 64, 0>(nullptr, ptr, L, M, N, 296, out, enc);
  run<6, 32, 1>(nullptr, ptr, L, M, N, 296, out, enc);
  return 0;
}
