// peel_cluster.cuh -- Greedy++ batch peel over a thread-block CLUSTER, for
// cores whose keys do not fit one SM's shared memory (e.g. RMAT-26's
// 83,682-vertex ceil(kmax/2)-core, RMAT-22's 35,367-vertex one).
//
// Same semantics and key ranges as peel_kernel.cuh (refine.cpp:20-156, fused
// Alg. 3 charges).  The vertex range is split into CS contiguous blocks of NC
// = 2^sh ids; CTA r of the cluster owns keys [r*NC, (r+1)*NC) (and their u32
// row offsets) in its shared memory.  Per batch:
//   S1  every CTA scans its own keys (128-bit loads), CTA-level (min, count)
//       via redux.sync + one CTA barrier, published in its shared memory
//   --- cluster barrier A
//   S2  every warp reads the CS CTA summaries through DSMEM (one remote load
//       per lane) -> global min, batch size, its CTA's offset; owners write
//       the batch in ascending id (CTA order = id order) into perm, the raw
//       charge key_at_removal into raw[pos], and broadcast (v, row offset,
//       degree) of the first 32 members into every CTA's staging slots
//   --- cluster barrier B
//   S3  the cluster's warps share the members' rows (16-byte quads); every
//       neighbour's key is decremented with a DSMEM reduction on its owner
//       CTA (atom.shared::cluster when same-batch neighbours must be told
//       apart, whose decrements then go to raw[pos] in global memory)
//   --- cluster barrier C
#pragma once

#include <cooperative_groups.h>

namespace dgb {
namespace peelc {

namespace cg = cooperative_groups;
using peelk::Range;

constexpr int PT = 1024;
constexpr int NW = PT / 32;
constexpr int UQ = 2;
constexpr int SB = 32;  // staged (small) batch members

struct Args {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  const uint64_t* loads;
  uint64_t base;
  int one;
  uint32_t sh;     // NC = 1 << sh ids per CTA
  uint32_t chunk;  // keys per thread = NC / PT (multiple of 4 when >= 4)
  int offs_smem;   // row offsets staged in shared memory (u32)
  uint32_t* perm;
  uint64_t* raw;
  unsigned long long* batches;
  unsigned long long* prof;  // [8] rank-0 thread-0 cycles: S1, S2, S3, batches
};

struct Fixed {
  uint32_t bv[SB];
  uint64_t boff[SB];
  uint32_t bdeg[SB];
  uint32_t wmin[NW];
  uint32_t wcnt[NW];
  uint32_t cmin, ccnt;  // this CTA's summary (read remotely)
  uint32_t wmap[SB][NW];
};

template <int CS>
__global__ void __launch_bounds__(PT, 1) k_peel_cluster(Args a) {
  using R = Range<uint32_t>;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t NC = 1u << a.sh;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
  uint32_t* soffs = keys + NC;  // NC + 1 entries when staged
  Fixed& s = *reinterpret_cast<Fixed*>(smem + ((size_t(NC) * 4 * (a.offs_smem ? 2 : 1) + 4 + 15) &
                                              ~size_t(15)));
  const uint4* adj4 = reinterpret_cast<const uint4*>(a.adj);
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const uint32_t n = a.n, c = a.chunk, lo = tid * c, hi = lo + c;
  const uint32_t gbase = rank << a.sh;  // first global id owned by this CTA
  const bool vec = (c & 3u) == 0;

  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t g = gbase + i;
    if (g < n) {
      const uint64_t o0 = a.offs[g], o1 = a.offs[g + 1];
      keys[i] = uint32_t(a.loads[g] - a.base + (o1 - o0));
      if (a.offs_smem) soffs[i] = uint32_t(o0);
    } else {
      keys[i] = R::DEAD;
      if (a.offs_smem) soffs[i] = uint32_t(a.offs[n]);
    }
  }
  if (a.offs_smem && tid == 0) soffs[NC] = uint32_t(a.offs[min(n, gbase + NC)]);
  for (uint32_t e = tid; e < SB * NW; e += PT) {
    const uint32_t b = e / NW + 1, ww = e % NW, gw = rank * NW + ww;
    const uint32_t jj = gw % b;
    // (member, rank among its warps, #warps serving it) over the cluster's warps
    // 8-bit member, 12-bit rank, 12-bit warp count (cluster has up to 512 warps)
    s.wmap[b - 1][ww] = jj | ((gw / b) << 8) | (((CS * NW - 1 - jj) / b + 1) << 20);
  }
  cl.sync();

  uint32_t removed = 0, pos = 0;
  bool marked = false;
  unsigned long long nbat = 0;
  const bool P = rank == 0 && tid == 0;
  long long c1 = 0, c2 = 0, c3 = 0, tm = clock64();
  while (removed < n) {
    // ---- S1: CTA summary
    uint32_t lmin = R::DEAD, lcnt = 0;
    if (vec) {
      const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
      for (uint32_t q = 0; q < (c >> 2); ++q) {
        const uint4 v = kv[q];
        lmin = min(min(lmin, min(v.x, v.y)), min(v.z, v.w));
      }
      for (uint32_t q = 0; q < (c >> 2); ++q) {
        const uint4 v = kv[q];
        lcnt += uint32_t(v.x == lmin) + uint32_t(v.y == lmin) + uint32_t(v.z == lmin) +
                uint32_t(v.w == lmin);
      }
    } else {
      for (uint32_t i = lo; i < hi; ++i) lmin = min(lmin, keys[i]);
      for (uint32_t i = lo; i < hi; ++i) lcnt += keys[i] == lmin;
    }
    if (!R::alive(lmin)) lmin = R::DEAD, lcnt = 0;
    const uint32_t wm = __reduce_min_sync(~0u, lmin);
    const uint32_t wc = __reduce_add_sync(~0u, lmin == wm ? lcnt : 0u);
    if (lane == 0) {
      s.wmin[w] = wm;
      s.wcnt[w] = wc;
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t x = s.wmin[lane];
      const uint32_t cm = __reduce_min_sync(~0u, x);
      const uint32_t ccnt = __reduce_add_sync(~0u, x == cm ? s.wcnt[lane] : 0u);
      if (lane == 0) {
        s.cmin = cm;
        s.ccnt = ccnt;
      }
    }
    cl.sync();  // A
    if (P) {
      const long long t = clock64();
      c1 += t - tm;
      tm = t;
    }
    // ---- S2: cluster min, batch size, offsets; owners write the batch
    uint32_t rmin = R::DEAD, rcnt = 0;
    if (lane < CS) {
      const Fixed* rs = cl.map_shared_rank(&s, lane);
      rmin = rs->cmin;
      rcnt = rs->ccnt;
    }
    const uint32_t gmin = __reduce_min_sync(~0u, rmin);
    const uint32_t total = __reduce_add_sync(~0u, rmin == gmin ? rcnt : 0u);
    const uint32_t bs = a.one ? 1u : total;
    if (marked) {
      for (uint32_t i = lo; i < hi; ++i)
        if (R::in_batch(keys[i])) keys[i] = R::DEAD;
      marked = false;
    }
    if (s.cmin == gmin && wm == gmin) {  // this warp owns part of the batch
      const uint32_t cta_off = __reduce_add_sync(~0u, (lane < rank && rmin == gmin) ? rcnt : 0u);
      const uint32_t xw = s.wmin[lane];
      const uint32_t woff = __reduce_add_sync(~0u, (lane < w && xw == gmin) ? s.wcnt[lane] : 0u);
      const bool mine = lmin == gmin && lcnt;
      const uint32_t mm = __ballot_sync(~0u, mine);
      uint32_t my = cta_off + woff;
      if (__popc(mm) > 1) {
        const uint32_t v = mine ? lcnt : 0u;
        my += warp_incl_scan(v) - v;
      }
      if (mine) {
        for (uint32_t i = lo; i < hi && my < bs; ++i) {
          if (keys[i] != gmin) continue;
          const uint32_t g = gbase + i;
          a.perm[pos + my] = g;
          a.raw[pos + my] = gmin;  // same-batch smaller neighbours are subtracted in S3
          keys[i] = bs == 1 ? R::DEAD : R::BATCH;
          marked = bs != 1;
          if (my < SB) {
            uint64_t r0, r1;
            if (a.offs_smem) {
              r0 = soffs[i];
              r1 = soffs[i + 1];
            } else {
              r0 = a.offs[g];
              r1 = a.offs[g + 1];
            }
            for (int q = 0; q < CS; ++q) {  // broadcast into every CTA's staging slot
              Fixed* rs = cl.map_shared_rank(&s, q);
              rs->bv[my] = g;
              rs->boff[my] = r0;
              rs->bdeg[my] = uint32_t(r1 - r0);
            }
          }
          ++my;
        }
      }
    }
    cl.sync();  // B
    if (P) {
      const long long t = clock64();
      c2 += t - tm;
      tm = t;
    }
    // ---- S3: the cluster's warps share the members' rows
    const uint32_t msk = NC - 1;
    auto dec = [&](uint32_t u, uint32_t vj, uint32_t pj) {
      uint32_t* rk = cl.map_shared_rank(keys, u >> a.sh) + (u & msk);
      if (bs == 1) {
        atomicAdd(rk, 0xffffffffu);
      } else {
        const uint32_t old = atomicAdd(rk, 0xffffffffu);
        if (R::in_batch(old) && u < vj)
          atomicAdd(reinterpret_cast<unsigned long long*>(&a.raw[pos + pj]), ~0ULL);
      }
    };
    if (bs <= SB) {
      const uint32_t wm3 = s.wmap[bs - 1][w];
      const uint32_t j = wm3 & 0xffu, rk = (wm3 >> 8) & 0xfffu, nwj = wm3 >> 20;
      const uint64_t oj = s.boff[j], ej = oj + s.bdeg[j];
      const uint32_t vj = s.bv[j];
      const uint64_t q1 = (ej + 3) >> 2, stride = uint64_t(nwj) * 32;
      for (uint64_t b0 = (oj >> 2) + uint64_t(rk) * 32; b0 < q1; b0 += stride * UQ) {
        uint4 x[UQ];
#pragma unroll
        for (int k = 0; k < UQ; ++k) {
          const uint64_t q = b0 + k * stride + lane;
          if (q < q1) x[k] = __ldg(adj4 + q);
        }
#pragma unroll
        for (int k = 0; k < UQ; ++k) {
          const uint64_t q = b0 + k * stride + lane;
          if (q >= q1) continue;
          const uint32_t us[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint64_t p = (q << 2) + e;
            if (p >= oj && p < ej) dec(us[e], vj, j);
          }
        }
      }
    } else {
      // large batch: CTA r takes members j = r, r + CS, ...; its warps split a row
      for (uint32_t j = rank; j < bs; j += CS) {
        const uint32_t vj = a.perm[pos + j];
        const uint64_t oj = a.offs[vj], ej = a.offs[vj + 1];
        for (uint64_t p = oj + tid; p < ej; p += PT) dec(a.adj[p], vj, j);
      }
    }
    cl.sync();  // C
    if (P) {
      const long long t = clock64();
      c3 += t - tm;
      tm = t;
    }
    pos += bs;
    removed += bs;
    ++nbat;
  }
  if (P) {
    *a.batches = nbat;
    if (a.prof) {
      a.prof[0] = c1;
      a.prof[1] = c2;
      a.prof[2] = c3;
      a.prof[3] = nbat;
      a.prof[4] = a.prof[5] = a.prof[6] = 0;
      a.prof[7] = CS;
    }
  }
}

inline size_t smem_bytes(uint32_t sh, bool offs_smem) {
  const size_t NC = size_t(1) << sh;
  return ((NC * 4 * (offs_smem ? 2 : 1) + 4 + 15) & ~size_t(15)) + sizeof(Fixed);
}

}  // namespace peelc
}  // namespace dgb
