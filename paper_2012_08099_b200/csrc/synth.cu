// synth.cu -- deterministic synthetic config-5 volume on the device.
//
// Smooth value noise: 4 octaves on integer lattices of spacing 128/64/32/16
// with amplitudes 8/4/2/1.  Lattice values are a 64-bit integer hash of
// (seed, octave, lattice point); interpolation is trilinear with a quantised
// smoothstep weight w(f) = floor(65536 * f^2 (3S - 2f) / S^3).  Everything is
// integer arithmetic, so paper_2012_08099_b200/synth.py:noise_slab_numpy
// reproduces it bit for bit.  The map to 0..65535 is fixed (sum / 15), not
// data-dependent, so z-slabs are generated independently on any rank.
#include "dpm_common.cuh"

namespace dpm {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t lattice(uint64_t seed, int o, int64_t cx, int64_t cy, int64_t cz) {
  uint64_t h = seed ^ ((uint64_t)o << 56);
  h = mix64(h ^ ((uint64_t)cx * 0x8CB92BA72F3D8DD7ull));
  h = mix64(h ^ ((uint64_t)cy * 0xA24BAED4963EE407ull));
  h = mix64(h ^ ((uint64_t)cz * 0x9FB21C651E98DF25ull));
  return h >> 48;  // 16-bit lattice value
}

__device__ __forceinline__ uint64_t sweight(int64_t f, int64_t S) {
  return (uint64_t)((f * f * (3 * S - 2 * f)) * 65536 / (S * S * S));
}

__global__ void synth_noise_kernel(uint16_t* out, int64_t L, int64_t M, int64_t z0, int64_t nz, uint64_t seed) {
  const int64_t total = L * M * nz;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = idx % L;
    const int64_t y = (idx / L) % M;
    const int64_t z = idx / (L * M) + z0;
    uint64_t sum = 0;
    #pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int64_t S = 128 >> o;
      const int64_t cx = x / S, cy = y / S, cz = z / S;
      const uint64_t wx = sweight(x - cx * S, S), wy = sweight(y - cy * S, S), wz = sweight(z - cz * S, S);
      uint64_t c[2];
      #pragma unroll
      for (int dz = 0; dz < 2; ++dz) {
        uint64_t b[2];
        #pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
          const uint64_t h0 = lattice(seed, o, cx, cy + dy, cz + dz);
          const uint64_t h1 = lattice(seed, o, cx + 1, cy + dy, cz + dz);
          b[dy] = h0 * (65536 - wx) + h1 * wx;                 // < 2^32
        }
        c[dz] = b[0] * (65536 - wy) + b[1] * wy;               // < 2^48
      }
      const uint64_t v = (c[0] * (65536 - wz) + c[1] * wz) >> 48;  // < 2^64 before shift
      sum += v << (3 - o);                                     // amplitudes 8, 4, 2, 1
    }
    out[idx] = (uint16_t)(sum / 15);
  }
}

int launch_synth_noise(uint16_t* out, int64_t L, int64_t M, int64_t z0, int64_t nz, uint64_t seed, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  synth_noise_kernel<<<sms * 16, 256, 0, st>>>(out, L, M, z0, nz, seed);
  note_launches(1);
  DPM_CUDA_CHECK_LAUNCH();
  return DPM_OK;
}

}  // namespace dpm
