// Random 4-byte load throughput from an L2-resident array (the k-core's
// alive-bitmap tests), with and without a concurrent streaming read.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return uint32_t(x);
}
template <int K, bool STREAM, bool REL>
__global__ void __launch_bounds__(1024, 1) k(const uint32_t* a, uint32_t mask, uint64_t iters,
                                             const uint32_t* st, uint64_t stn, uint32_t* sink) {
  const uint64_t t = blockIdx.x * 1024ull + threadIdx.x, T = gridDim.x * 1024ull;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < iters; ++i) {
    uint32_t idx[K], v[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      idx[j] = mix((i * K + j) * T + t) & mask;
      if (STREAM) idx[j] ^= st[((i * K + j) * T + t) % stn] & 1;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (REL) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v[j]) : "l"(a + idx[j]));
      else v[j] = a[idx[j]];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) acc += v[j];
  }
  if (acc == 0x12345) sink[0] = acc;
}
int main() {
  uint32_t *a, *st, *sink;
  const uint64_t stbytes = 4ull << 30;
  cudaMalloc(&a, 64ull << 20); cudaMalloc(&st, stbytes); cudaMalloc(&sink, 4);
  cudaMemset(a, 1, 64ull << 20); cudaMemset(st, 0, stbytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int stream = 0; stream < 2; ++stream)
    for (int rel = 0; rel < 2; ++rel)
      for (uint64_t mb : {1ull, 4ull, 16ull, 64ull}) {
        const uint32_t mask = uint32_t((mb << 20) / 4 - 1);
        const uint64_t iters = 64;
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          if (stream) { if (rel) k<8, true, true><<<148, 1024>>>(a, mask, iters, st, stbytes / 4, sink);
                        else k<8, true, false><<<148, 1024>>>(a, mask, iters, st, stbytes / 4, sink); }
          else { if (rel) k<8, false, true><<<148, 1024>>>(a, mask, iters, st, stbytes / 4, sink);
                 else k<8, false, false><<<148, 1024>>>(a, mask, iters, st, stbytes / 4, sink); }
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        const double ops = 148.0 * 1024 * iters * 8;
        printf("array %3llu MB %s %s: %.1f G loads/s (%.3f ms)\n", (unsigned long long)mb,
               rel ? "ld.relaxed.gpu" : "ld (L1)       ", stream ? "+4B stream" : "          ",
               ops / best / 1e6, best);
      }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
