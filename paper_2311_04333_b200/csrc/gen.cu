// gen.cu -- seeded synthetic inputs on the device (BASELINE.json configs):
// the pair arrays of the generators in gen.cuh.
#include "gen.cuh"

namespace dgb {

namespace {

// samples [first, first + count) of the stream -> u[0..count), v[0..count)
template <class Gen>
__global__ void k_gen_pairs(Gen gen, uint64_t first, uint64_t count, uint64_t* u, uint64_t* v) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < count;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t a, b;
    gen(first + k, a, b);
    u[k] = a;
    v[k] = b;
  }
}

}  // namespace

void gen_rmat_device(uint32_t scale, uint64_t samples, uint64_t seed, uint64_t* d_u,
                     uint64_t* d_v, uint64_t first) {
  if (!samples) return;
  const RmatGen gen{scale, mix64(seed ^ 0x524d4154ULL)};
  k_gen_pairs<<<grid_for(samples, 256, 16), 256, 0, stream()>>>(gen, first, samples, d_u, d_v);
  DG_CHECK_LAUNCH();
}

void gen_chung_lu_device(uint64_t n, uint64_t pairs, double R, uint64_t seed, uint64_t* d_u,
                         uint64_t* d_v) {
  if (!pairs) return;
  const ChungLuGen gen{n, R, mix64(seed ^ 0x434cULL)};
  k_gen_pairs<<<grid_for(pairs, 256, 16), 256, 0, stream()>>>(gen, 0, pairs, d_u, d_v);
  DG_CHECK_LAUNCH();
}

}  // namespace dgb
