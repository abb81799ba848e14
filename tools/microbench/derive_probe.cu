// Phase timing of the device epilogue (derive_volume) on an all-zero
// accumulator (every check passes, every solve path runs): globaltimer stamps
// per warp, printed as the slowest warp's phase durations.
//   nvcc -DDPM_DERIVE_PROBE -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a \
//        --expt-relaxed-constexpr -I. tools/microbench/derive_probe.cu -o /tmp/derive_probe
#include <cstdio>
#include <vector>
#include "../../paper_2012_08099_b200/csrc/derive_dev.cuh"

using namespace dpm;

template <int K, int WARPS>
__global__ void probe_kernel(const uint64_t* acc, int n_img, int kind, int64_t* out_i128, double* out_f64, int32_t* status) {
  constexpr int N2 = (K + 1) * (K + 2) / 2;
  __shared__ uint64_t sa[DPM_MAX_IMAGES * N2 * 4];
  __shared__ int32_t sst;
  derive_volume<K>(acc, 0, n_img, kind, out_i128, out_f64, status, sa, &sst, false);
}

template <int K, int WARPS>
void run(const char* name) {
  const int n_img = K <= 3 ? 4 : K + 1;
  uint64_t* acc; int64_t* o; double* f; int32_t* st;
  cudaMalloc(&acc, 8 * 4 * 28 * 4 * 8); cudaMemset(acc, 0, 8 * 4 * 28 * 4 * 8);
  cudaMalloc(&o, 2 * 84 * 8); cudaMalloc(&f, 84 * 8); cudaMalloc(&st, 4);
  unsigned long long best[5] = {~0ull, ~0ull, ~0ull, ~0ull, ~0ull};
  for (int rep = 0; rep < 12; ++rep) {   // fastest of 10 warm replays, per phase
    probe_kernel<K, WARPS><<<1, 32 * WARPS>>>(acc, n_img, DPM_ACC_PROFILE, o, f, st);
    cudaDeviceSynchronize();
    unsigned long long h[64][8];
    cudaMemcpyFromSymbol(h, g_derive_probe, sizeof(h));
    unsigned long long t0 = ~0ull, m[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < WARPS; ++w) t0 = h[w][0] < t0 ? h[w][0] : t0;
    for (int w = 0; w < WARPS; ++w)
      for (int i = 1; i < 5; ++i) m[i] = h[w][i] - t0 > m[i] ? h[w][i] - t0 : m[i];
    if (rep >= 2)
      for (int i = 1; i < 5; ++i) best[i] = m[i] < best[i] ? m[i] : best[i];
  }
  unsigned long long* mx = best;
  int s; cudaMemcpy(&s, st, 4, cudaMemcpyDeviceToHost);
  printf("%s: staged %llu ns, placed %llu ns, solved (slowest warp) %llu ns, end %llu ns, status %d (%s)\n", name,
         mx[1], mx[2], mx[3], mx[4], s, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<3, 4>("K3 4 warps");
  run<3, 16>("K3 16 warps");
  run<4, 16>("K4 16 warps");
  run<6, 4>("K6 4 warps");
  run<6, 16>("K6 16 warps");
  return 0;
}
