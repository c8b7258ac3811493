// gen.cuh -- per-sample device functions of the seeded generators (gen.cu),
// shared by the pair generators and the streamed CSR build (graph_stream.cu).
// Counter-based splitmix64 streams with integer thresholds; bit-identical to
// the host generators in oracle/dg_oracle.c (pinned by tests).
#pragma once

#include "internal.cuh"

namespace dgb {

// RMAT quadrant thresholds on 32-bit draws: a=.57 b=.19 c=.19 d=.05
constexpr uint32_t kRmatTA = 2448131358u, kRmatTAB = 3264175144u, kRmatTABC = 4080218930u;

struct RmatGen {
  uint32_t scale;
  uint64_t sk;  // mix64(seed ^ 0x524d4154)
  __device__ __forceinline__ void operator()(uint64_t k, uint64_t& a, uint64_t& b) const {
    a = 0;
    b = 0;
    for (uint32_t l = 0; l < scale; l += 2) {
      const uint64_t r = mix64(sk ^ ((k << 5) | (l >> 1)));
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        if (l + h >= scale) break;
        const uint32_t d = h ? uint32_t(r >> 32) : uint32_t(r);
        const uint32_t bu = d >= kRmatTAB, bv = (d >= kRmatTA && d < kRmatTAB) || d >= kRmatTABC;
        a = (a << 1) | bu;
        b = (b << 1) | bv;
      }
    }
  }
  uint64_t id_bound() const { return 1ULL << scale; }
};

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

struct ChungLuGen {
  uint64_t n;
  double R;     // n^(1/11)
  uint64_t sc;  // mix64(seed ^ 0x434c)
  __device__ __forceinline__ void operator()(uint64_t k, uint64_t& a, uint64_t& b) const {
    a = cl_endpoint(mix64(sc ^ (2 * k)), R, n);
    b = cl_endpoint(mix64(sc ^ (2 * k + 1)), R, n);
  }
  uint64_t id_bound() const { return n; }
};

}  // namespace dgb
