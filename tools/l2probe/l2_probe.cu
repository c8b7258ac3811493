// L2 latency by address chunk, seen from one chosen SM (experiment).
// Launch one CTA per SM; only the CTA on SM `sm` works: for every 64 KB chunk
// of a buffer it warms 8 lines (one pass), then times a dependent chain of
// loads over those lines (L2 hits).  Prints per-chunk cycles/load.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void probe(unsigned* buf, size_t chunk_words, size_t nchunks, unsigned sm,
                      unsigned long long* out) {
  if (smid() != sm || threadIdx.x != 0) return;
  for (size_t c = 0; c < nchunks; ++c) {
    unsigned* base = buf + c * chunk_words;
    // chain over 8 lines spread in the chunk: base[k*stride] holds next index
    const size_t stride = chunk_words / 8;
    unsigned idx = 0;
    for (int k = 0; k < 8; ++k) idx = __ldcg(&base[idx]);  // warm (L2)
    idx = 0;
    long long t0 = clock64();
    for (int rep = 0; rep < 4; ++rep)
      for (int k = 0; k < 8; ++k) idx = __ldcg(&base[idx]);
    long long t1 = clock64();
    out[c] = (unsigned long long)(t1 - t0) / 32 + (idx == 0xdeadbeef);
    (void)stride;
  }
}

__global__ void init(unsigned* buf, size_t chunk_words, size_t nchunks) {
  size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  unsigned* base = buf + c * chunk_words;
  const size_t stride = chunk_words / 8;
  for (int k = 0; k < 8; ++k) base[k * stride] = unsigned(((k + 1) % 8) * stride);
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 64;
  const size_t chunk = argc > 2 ? atoi(argv[2]) : 65536;
  const size_t words = mb * (1 << 20) / 4, cw = chunk / 4, nch = words / cw;
  unsigned* buf;
  cudaMalloc(&buf, words * 4);
  unsigned long long* out;
  cudaMalloc(&out, nch * 8);
  init<<<(nch + 255) / 256, 256>>>(buf, cw, nch);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::vector<unsigned long long> h(nch);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  if (argc > 3) {  // mean over all SMs (chunks given by argv[1..2])
    std::vector<double> m(nsm);
    for (int sm = 0; sm < nsm; ++sm) {
      probe<<<nsm, 32, 150 * 1024>>>(buf, cw, nch, sm, out);
      cudaMemcpy(h.data(), out, nch * 8, cudaMemcpyDeviceToHost);
      double sum = 0;
      for (auto x : h) sum += double(x);
      m[sm] = sum / nch;
    }
    for (int sm = 0; sm < nsm; ++sm) printf("%d:%.0f%s", sm, m[sm], sm % 16 == 15 ? "\n" : " ");
    printf("\n");
    return 0;
  }
  for (unsigned sm : {0u, 1u, 73u, 74u, 146u, 147u}) {
    probe<<<nsm, 32, 150 * 1024>>>(buf, cw, nch, sm, out);  // one CTA per SM
    cudaMemcpy(h.data(), out, nch * 8, cudaMemcpyDeviceToHost);
    size_t lo = 0, hi = 0;
    unsigned long long mn = ~0ULL, mx = 0, sum = 0;
    for (auto x : h) {
      mn = x < mn ? x : mn;
      mx = x > mx ? x : mx;
      sum += x;
    }
    const unsigned long long mid = (mn + mx) / 2;
    for (auto x : h) (x < mid ? lo : hi)++;
    printf("sm %3u: chunks %zu  min %llu max %llu mean %.0f  below-mid %zu above %zu  first 24:", sm,
           nch, mn, mx, double(sum) / nch, lo, hi);
    for (size_t i = 0; i < 24 && i < nch; ++i) printf(" %llu", h[i]);
    printf("\n");
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
