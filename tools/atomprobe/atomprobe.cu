// Random returning atomicSub throughput on a u32 array of S bytes, with a
// concurrent streaming read (like the k-core's big rounds): is the degree
// array's residency in L2 (16-bit degrees) worth it?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return uint32_t(x);
}
template <int K, bool RET, bool STREAM>
__global__ void __launch_bounds__(1024, 1) k(uint32_t* a, uint32_t mask, uint64_t iters,
                                             const uint4* st, uint64_t stn, uint32_t* sink) {
  const uint64_t t = blockIdx.x * 1024ull + threadIdx.x, T = gridDim.x * 1024ull;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < iters; ++i) {
    uint32_t idx[K];
    uint4 sv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      idx[j] = mix((i * K + j) * T + t) & mask;
      if (STREAM) sv[j] = st[((i * K + j) * T + t) % stn];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (STREAM) idx[j] ^= (sv[j].x & 1);
      if (RET) acc += atomicSub(&a[idx[j]], 1u);
      else atomicSub(&a[idx[j]], 1u);
    }
  }
  if (acc == 0x12345) sink[0] = acc;
}
int main() {
  uint32_t* a; uint4* st; uint32_t* sink;
  const uint64_t stbytes = 4ull << 30;
  cudaMalloc(&a, 512ull << 20); cudaMalloc(&st, stbytes); cudaMalloc(&sink, 4);
  cudaMemset(a, 0x7f, 512ull << 20); cudaMemset(st, 0, stbytes);
  cudaFuncSetAttribute(k<8, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int stream = 0; stream < 2; ++stream)
  for (uint64_t mb : {4ull, 16ull, 32ull, 64ull, 96ull, 128ull, 256ull}) {
    const uint32_t mask = uint32_t((mb << 20) / 4 - 1);
    const uint64_t iters = 64;
    for (int ret = 0; ret < 2; ++ret) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (stream) { if (ret) k<8, true, true><<<148, 1024>>>(a, mask, iters, st, stbytes / 16, sink);
                      else k<8, false, true><<<148, 1024>>>(a, mask, iters, st, stbytes / 16, sink); }
        else { if (ret) k<8, true, false><<<148, 1024>>>(a, mask, iters, st, stbytes / 16, sink);
               else k<8, false, false><<<148, 1024>>>(a, mask, iters, st, stbytes / 16, sink); }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      const double ops = 148.0 * 1024 * iters * 8;
      printf("array %4llu MB %s %s: %.1f G atomics/s (%.3f ms)\n", (unsigned long long)mb,
             ret ? "atom(ret)" : "red     ", stream ? "+16B stream" : "           ",
             ops / best / 1e6, best);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
