// fill.cu -- device side of the seeded input generator (synth/dlrm_gen.py documents the recipe).
// NOT the method: it only writes procedural table values W_g[row][d] so the product's fused
// kernel has tables to read.  The oracle (oracle/oracle.c) and the host generator
// (synth/dlrm_gen.py) implement the same counter-based formula independently; tests pin all
// three against each other on sampled (g, row, d).
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(float* __restrict__ dst, long long n, int D, long long g,
                            unsigned long long seed_mix, int mode) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / D;
    const long long d = e - row * D;
    const unsigned long long key =
        ((unsigned long long)g * 8388608ull + (unsigned long long)row) * 1024ull +
        (unsigned long long)d;
    const unsigned long long x = sm64(key ^ seed_mix);
    float v;
    if (mode == 1) v = (float)((long long)(x >> 60) - 8);
    else if (mode == 2) v = (float)((double)((long long)(x >> 56) - 128) * (1.0 / 128.0));
    else v = (float)((double)((long long)(x >> 40) - 8388608ll) * (1.0 / 8388608.0));
    dst[e] = v;
  }
}

extern "C" int synth_fill_table(float* dst, long long rows, int D, long long g,
                                unsigned long long seed, int mode, void* stream) {
  if (rows >= (1ll << 23) || D > 1024 || D < 1) return 1;
  const long long n = rows * (long long)D;
  unsigned long long z = seed + 0x9E3779B97F4A7C15ull;     // host splitmix64(seed)
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= (z >> 31);
  fill_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(dst, n, D, g, z, mode);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// GEMM operands of the fused AllGather + GEMM (synth/gemm_gen.py documents the recipe):
// x = splitmix64(key ^ splitmix64(seed)), key = ((tensor << 24) + row) << 16 | col; mode 0:
// ((x >> 57) - 64) * 2^-6, mode 1: (x >> 61) - 4 -- both exact in bfloat16, written as bf16 bits.
__global__ void fill_gemm_kernel(unsigned short* __restrict__ dst, long long rows, long long cols,
                                 long long row0, long long tensor, unsigned long long seed_mix,
                                 int mode) {
  const long long n = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols;
    const long long c = e - r * cols;
    const unsigned long long key =
        ((((unsigned long long)tensor << 24) + (unsigned long long)(row0 + r)) << 16) |
        (unsigned long long)c;
    const unsigned long long x = sm64(key ^ seed_mix);
    float v = mode == 1 ? (float)((long long)(x >> 61) - 4)
                        : (float)((long long)(x >> 57) - 64) * 0.015625f;
    dst[e] = (unsigned short)(__float_as_uint(v) >> 16);   // exact: v has <= 8 significant bits
  }
}

extern "C" int synth_fill_gemm_bf16(void* dst, long long rows, long long cols, long long row0,
                                    long long tensor, unsigned long long seed, int mode,
                                    void* stream) {
  if (row0 < 0 || row0 + rows > (1ll << 24) || cols > (1ll << 16) || cols < 1 || rows < 0)
    return 1;
  unsigned long long z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= (z >> 31);
  if (rows == 0) return 0;
  fill_gemm_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>((unsigned short*)dst, rows, cols,
                                                              row0, tensor, z, mode);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
