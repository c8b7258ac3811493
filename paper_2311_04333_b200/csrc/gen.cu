// gen.cu -- seeded synthetic inputs on the device (BASELINE.json configs).
// Counter-based splitmix64 streams with integer thresholds; bit-identical to
// the host generators in oracle/dg_oracle.c (pinned by tests).
#include "internal.cuh"

namespace dgb {

namespace {

// RMAT quadrant thresholds on 32-bit draws: a=.57 b=.19 c=.19 d=.05
constexpr uint32_t TA = 2448131358u, TAB = 3264175144u, TABC = 4080218930u;

__global__ void k_rmat(uint32_t scale, uint64_t samples, uint64_t sk, uint64_t* u, uint64_t* v) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < samples;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a = 0, b = 0;
    for (uint32_t l = 0; l < scale; l += 2) {
      const uint64_t r = mix64(sk ^ ((k << 5) | (l >> 1)));
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        if (l + h >= scale) break;
        const uint32_t d = h ? uint32_t(r >> 32) : uint32_t(r);
        const uint32_t bu = d >= TAB, bv = (d >= TA && d < TAB) || d >= TABC;
        a = (a << 1) | bu;
        b = (b << 1) | bv;
      }
    }
    u[k] = a;
    v[k] = b;
  }
}

__device__ __forceinline__ uint64_t cl_endpoint(uint64_t r, double R, uint64_t n) {
  const double x = __dmul_rn(double(r >> 11), 1.0 / 9007199254740992.0);
  const double t = __dmul_rn(x, __dadd_rn(R, -1.0));
  const double y = __dadd_rn(1.0, t);
  const double y2 = __dmul_rn(y, y);
  const double y4 = __dmul_rn(y2, y2);
  const double y8 = __dmul_rn(y4, y4);
  const double y10 = __dmul_rn(y8, y2);
  const double z = __dmul_rn(y10, y);
  uint64_t id = uint64_t(z);
  id = id >= 1 ? id - 1 : 0;
  return id < n ? id : n - 1;
}

__global__ void k_chung_lu(uint64_t n, uint64_t pairs, double R, uint64_t sc, uint64_t* u,
                           uint64_t* v) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < pairs;
       k += uint64_t(gridDim.x) * blockDim.x) {
    u[k] = cl_endpoint(mix64(sc ^ (2 * k)), R, n);
    v[k] = cl_endpoint(mix64(sc ^ (2 * k + 1)), R, n);
  }
}

}  // namespace

void gen_rmat_device(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* d_u,
                     uint64_t* d_v) {
  if (!samples) return;
  k_rmat<<<grid_for(samples, 256, 16), 256, 0, stream()>>>(scale, samples,
                                                           mix64(seed ^ 0x524d4154ULL), d_u, d_v);
  DG_CHECK_LAUNCH();
}

void gen_chung_lu_device(uint64_t n, uint64_t pairs, double R, uint64_t seed, uint64_t* d_u,
                         uint64_t* d_v) {
  if (!pairs) return;
  k_chung_lu<<<grid_for(pairs, 256, 16), 256, 0, stream()>>>(n, pairs, R,
                                                             mix64(seed ^ 0x434cULL), d_u, d_v);
  DG_CHECK_LAUNCH();
}

}  // namespace dgb
