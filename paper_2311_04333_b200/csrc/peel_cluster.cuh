// peel_cluster.cuh -- Greedy++ batch peel over a thread-block CLUSTER, for
// cores whose keys do not fit one SM's shared memory (e.g. RMAT-26's
// 83,682-vertex ceil(kmax/2)-core, RMAT-28's 122K one).
//
// Same semantics and key ranges as peel_kernel.cuh (refine.cpp:20-156, fused
// Alg. 3 charges).  The vertex range is split into CS contiguous blocks of NC
// ids (a multiple of the CTA size); CTA r of the cluster owns keys [r*NC, (r+1)*NC) (and their u32
// row offsets) in its shared memory.
//
// Owner-applied decrements.  Every CTA streams the removed members' rows
// (16-byte quads from L2) and applies only the decrements whose target lies
// in its own block, with shared-memory atomics on its own keys: no atomic
// ever crosses the cluster, and the row is read CS times from L2 (a few KB
// per member, far below L2 bandwidth).
//
// Per batch (no cluster-wide barrier on the common path):
//   S1  every CTA scans its own keys: (min, count, first id at the min, its
//       degree and row start) = its 32-byte summary, which warp 0 PUSHES
//       into every CTA's shared memory with st.async (slot [parity][rank])
//       completing bytes on the receiver's mbarrier; each CTA waits on its
//       own mbarrier for the CS summaries (no cluster.sync: that costs
//       ~380 cycles plus an L1 invalidate, and reading the summaries
//       remotely queues every warp's requests on one SM's shared memory)
//   S2  every warp decodes the local summaries -> global min, owner CTAs,
//       batch size.  Simple batch (each owner CTA holds exactly one
//       member, or one-at-a-time): the summaries name the batch in
//       ascending id (CTA order = id order), so every CTA starts removing at
//       once.  Otherwise owners write the batch and push (v, degree, row
//       start) of each member into every CTA's staging slots (again
//       st.async on a second mbarrier pair).
//   S3  removal, owner-applied (above); batches beyond SB members decrement
//       through DSMEM instead (remote atomics between cluster barriers)
//   --- CTA barrier (the next S1 reads only this CTA's keys)
// Slots are double-buffered by batch parity: a CTA pushes batch b+2's
// summary only after receiving every CTA's b+1 summary, which each CTA
// sends after it has decoded batch b.
// Raw charges (key_at_removal - #same-batch neighbours with a smaller id)
// are accumulated with atomics into a zeroed raw[]: the owner adds the key,
// every CTA subtracts the same-batch arcs it sees, in any order.
#pragma once

#include <cooperative_groups.h>

namespace dgb {
namespace peelc {

namespace cg = cooperative_groups;
using peelk::Range;

constexpr int MAXW = 32;  // warps per CTA at most (PT <= 1024)
constexpr int SB = 32;  // staged (small) batch members
#ifndef DG_SLICE_MIN
#define DG_SLICE_MIN 2048
#endif
// simple batches read only the CTA's slice of rows at least this long
constexpr uint32_t kSliceMin = DG_SLICE_MIN;
// 1024-thread CTAs look their slice up in the global table (a dependent
// round trip before the row's) and cover 4K arcs per pass
#ifndef DG_SLICE_MIN_1024
#define DG_SLICE_MIN_1024 2048
#endif
constexpr uint32_t kSliceMin1024 = DG_SLICE_MIN_1024;
// DG_PEEL_PROF=1 (a tuning build: python build.py prof -DDG_PEEL_PROF=1)
// records rank-0 phase cycles into Args::prof; the production kernel carries
// none of those live registers.
#ifndef DG_PEEL_PROF
#define DG_PEEL_PROF 0
#endif
#ifndef DG_SC_FILL
#define DG_SC_FILL 1
#endif
#ifndef DG_SC_HIT
#define DG_SC_HIT 1
#endif
#ifndef DG_SC_GEN
#define DG_SC_GEN 1
#endif
#ifndef DG_ROW_PREFETCH
#define DG_ROW_PREFETCH 1
#endif

struct Args {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  const uint64_t* loads;
  uint64_t base;
  int one;
  uint32_t nc;     // NC key slots per CTA (a multiple of PT)
  uint32_t chunk;  // keys per thread = NC / PT (<= 32)
  uint32_t no;     // NO <= NC ids owned per CTA: [rank*NO, (rank+1)*NO)
  int offs_smem;   // row offsets staged in shared memory (u32)
  uint32_t* perm;
  uint64_t* raw;   // zeroed by the launcher
  // seg[v*(CS+1) + r]: offset inside row v of its first neighbour owned by
  // CTA r (rows ascend, so CTA r's targets are [seg[r], seg[r+1]))
  const uint32_t* seg;
  int slice_smem;  // this CTA's slice bounds of EVERY row staged in shared memory
                   // (u16 start | u16 end << 16; rows shorter than 2^16)
  uint32_t slotq;  // slice cache: 16-byte quads per slot (0: no cache; 512-thread CTAs
                   // with slice_smem only)
  unsigned long long* batches;
  unsigned long long* prof;  // [8] rank-0 thread-0 cycles: S1, S2, S3, batches, simple
};

// CTA summary: min key, #keys at the min, first id at the min, its degree,
// its row start (u64) -- two 16-byte st.async
struct __align__(16) Summary {
  uint32_t cmin, ccnt, cfirst, cdeg;
  uint32_t r0lo, r0hi, pad0, pad1;
};

// staged member of a general batch: id, degree, row start
struct __align__(16) Member {
  uint32_t v, deg, r0lo, r0hi;
};

struct Fixed {
  unsigned long long mbA[2], mbB[2];  // summaries / staged members, by parity
  // the summaries' halves in separate arrays, [parity][CTA rank]: lane q's
  // 16-byte loads sit at a 16-byte stride (conflict free; the 32-byte stride
  // of whole Summary slots doubled their wavefronts)
  uint4 sumA[2][16];                  // min key, count, first id, degree
  uint4 sumB[2][16];                  // row start (u64), pad
  Member stage[2][SB];                // [parity][member]
  // per-warp summary: {min key, #keys at it, first index at it, its row start}
  // and that row's degree (row bounds only with offsets staged in shared memory)
  uint4 wsum[MAXW];
  uint32_t wdeg[MAXW];
  // warp -> member map over this CTA's warps for batches of b <= SB members:
  // wmap[b-1][w] = j | rank << 8 | nwj << 16 (j = w % b, rank = w / b,
  // nwj = #warps serving member j); batches of more than NW members are
  // removed as one flat quad range (remove_flat)
  uint32_t wmap[MAXW][MAXW];
  // slice cache (see k_peel_cluster): one mbarrier and one tag word per slot,
  // tag = cached vertex id | phase parity of its copy << 31 (kNoTag: empty)
  unsigned long long mbS[16];
  uint32_t ctag[16];
#if DG_PEEL_PROF
  uint32_t prevc[2][16];  // previous batch's CTA candidates (slice-cache hit estimate)
#endif
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
// shared::cluster address of `local` in CTA `r`
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(local), "r"(r));
  return o;
}
__device__ __forceinline__ void st_async(uint32_t raddr, const uint4& v, uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::
          "r"(raddr),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
constexpr uint32_t kNoTag = 0x7fffffffu;  // no vertex id reaches 2^31 - 1 (n < 2^28)
// this CTA's shared memory <- global, completing bytes on the CTA's mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// row [oj, oj + dj) of member vj, quads [rk*32 + lane, ...) step nwj*32:
// decrement the targets in this CTA's block [gbase, gbase + NC)
template <bool ONE, int UQ, class Off = uint64_t>
__device__ __forceinline__ void remove_local(const uint4* adj4, uint32_t keys_s, Off oj,
                                             uint32_t dj, uint32_t vj, uint32_t rk, uint32_t nwj,
                                             uint32_t lane, uint32_t gbase, uint32_t NC,
                                             unsigned long long* rawj) {
  const Off ej = oj + dj, q1 = (ej + 3) >> 2, stride = Off(nwj) * 32;
  for (Off b0 = (oj >> 2) + Off(rk) * 32 + lane; b0 < q1; b0 += stride * UQ) {
    uint4 x[UQ];
#pragma unroll
    for (int k = 0; k < UQ; ++k)
      if (b0 + k * stride < q1) x[k] = __ldg(adj4 + b0 + k * stride);
#pragma unroll
    for (int k = 0; k < UQ; ++k) {
      const Off q = b0 + k * stride;
      if (q >= q1) break;
      const uint32_t us[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
      bool ok[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const Off p = (q << 2) + e;
        ok[e] = p >= oj && p < ej && us[e] - gbase < NC;
      }
      if (ONE) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (ok[e])
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(keys_s + ((us[e] - gbase) << 2)),
                         "r"(0xffffffffu)
                         : "memory");
      } else {
        uint32_t old[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // all atomics in flight before any test
          old[e] = 0;
          if (ok[e])
            asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                         : "=r"(old[e])
                         : "r"(keys_s + ((us[e] - gbase) << 2)), "r"(0xffffffffu)
                         : "memory");
        }
        unsigned long long c = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) c += (ok[e] && Range<uint32_t>::in_batch(old[e]) && us[e] < vj);
        if (c) atomicAdd(rawj, 0ULL - c);
      }
    }
  }
}

// the same from a slice-cache slot: the slot holds the aligned quads that
// cover the slice [oj, oj + dj) of member vj's row, the slice starting at arc
// (oj & 3) of the slot
#ifndef DG_SC_INLINE
#define DG_SC_INLINE __forceinline__
#endif
template <bool ONE>
__device__ DG_SC_INLINE void remove_cached(uint32_t slot_s, uint32_t keys_s, uint32_t a0,
                                              uint32_t dj, uint32_t vj, uint32_t rk, uint32_t nwj,
                                              uint32_t lane, uint32_t gbase, uint32_t NC,
                                              unsigned long long* rawj) {
  const uint32_t a1 = a0 + dj, nq = (a1 + 3) >> 2;
  for (uint32_t q = rk * 32 + lane; q < nq; q += nwj * 32) {
    uint32_t us[4];
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(us[0]), "=r"(us[1]), "=r"(us[2]), "=r"(us[3])
                 : "r"(slot_s + (q << 4)));
    bool ok[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t p = (q << 2) + e;
      ok[e] = p >= a0 && p < a1 && us[e] - gbase < NC;
    }
    if (ONE) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (ok[e])
          asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(keys_s + ((us[e] - gbase) << 2)),
                       "r"(0xffffffffu)
                       : "memory");
    } else {
      uint32_t old[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        old[e] = 0;
        if (ok[e])
          asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                       : "=r"(old[e])
                       : "r"(keys_s + ((us[e] - gbase) << 2)), "r"(0xffffffffu)
                       : "memory");
      }
      unsigned long long c = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) c += (ok[e] && Range<uint32_t>::in_batch(old[e]) && us[e] < vj);
      if (c) atomicAdd(rawj, 0ULL - c);
    }
  }
}

// removal of a multi-member batch (bs <= 32) as ONE flat range of 16-byte
// quads: the members' rows concatenated (lane j of every warp holds member
// j: id, degree, row start), 2 quads per thread per round over the CTA, each
// quad's member found by a 5-step binary search over the lanes' prefix
// sums.  Every thread gets the same share however the batch's degrees vary.
template <int PT, class Off = uint64_t>
__device__ __forceinline__ void remove_flat(const uint4* adj4, uint32_t keys_s, uint32_t bs,
                                            uint32_t mv, uint32_t mdeg, Off mr0,
                                            uint32_t w, uint32_t lane, uint32_t gbase,
                                            uint32_t NC, unsigned long long* rawpos) {
  const uint32_t nq = lane < bs ? (uint32_t(mr0 & 3) + mdeg + 3) >> 2 : 0u;
  const uint32_t incl = warp_incl_scan(nq), excl = incl - nq;
  const uint32_t totq = __shfl_sync(~0u, incl, 31);
  for (uint32_t base = w * 32; base < totq; base += 2 * PT) {
    uint4 x[2];
    uint32_t m[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t t = base + k * PT + lane;
      uint32_t lo = 0, hi = bs - 1;  // largest member with excl <= t
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        const uint32_t e = __shfl_sync(~0u, excl, mid);
        if (e <= t) lo = mid; else hi = mid - 1;
      }
      m[k] = lo;
      const Off r0 = __shfl_sync(~0u, mr0, lo);
      const uint32_t ex = __shfl_sync(~0u, excl, lo);
      if (t < totq) x[k] = __ldg(adj4 + (r0 >> 2) + (t - ex));
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t t = base + k * PT + lane;
      const Off r0 = __shfl_sync(~0u, mr0, m[k]);
      const uint32_t d = __shfl_sync(~0u, mdeg, m[k]), v = __shfl_sync(~0u, mv, m[k]);
      const uint32_t ex = __shfl_sync(~0u, excl, m[k]);
      if (t >= totq) continue;
      const Off q = (r0 >> 2) + (t - ex);
      const uint32_t us[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
      uint32_t old[4];
      bool ok[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const Off pp = (q << 2) + e;
        ok[e] = pp >= r0 && pp < r0 + d && us[e] - gbase < NC;
        old[e] = 0;
        if (ok[e])
          asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                       : "=r"(old[e])
                       : "r"(keys_s + ((us[e] - gbase) << 2)), "r"(0xffffffffu)
                       : "memory");
      }
      unsigned long long c = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) c += (ok[e] && Range<uint32_t>::in_batch(old[e]) && us[e] < v);
      if (c) atomicAdd(rawpos + m[k], 0ULL - c);
    }
  }
}

// S1 over KR >= c keys held in registers: retire this thread's batch marks,
// then the minimum and the mask of keys at it
template <int KR, class R>
__device__ __forceinline__ void scan_regs(uint32_t* keys, uint32_t lo, uint32_t c, bool& marked,
                                          uint32_t& lmin, uint32_t& bits) {
  uint32_t k[KR];
  if (KR == 8 && c == 8) {  // two 16-byte vectors (lo is a multiple of 4)
#pragma unroll
    for (int q = 0; q < KR / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(keys + lo)[q];
      k[4 * q] = v.x, k[4 * q + 1] = v.y, k[4 * q + 2] = v.z, k[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < KR; ++j) k[j] = uint32_t(j) < c ? keys[lo + j] : R::DEAD;
  }
  if (marked) {
#pragma unroll
    for (int j = 0; j < KR; ++j)
      if (uint32_t(j) < c && R::in_batch(k[j])) k[j] = keys[lo + j] = R::DEAD;
    marked = false;
  }
#pragma unroll
  for (int j = 0; j < KR; ++j) lmin = min(lmin, k[j]);
#pragma unroll
  for (int j = 0; j < KR; ++j) bits |= uint32_t(k[j] == lmin) << j;
}

// O64: row offsets beyond 32 bits (2m + 16 >= 2^32); the usual core's fit a
// u32, which halves the offset arithmetic and shuffles on the batch's chain
template <int CS, int PT, bool O64>
__global__ void __launch_bounds__(PT, 1) k_peel_cluster(Args a) {
  using Off = std::conditional_t<O64, uint64_t, uint32_t>;
  constexpr uint32_t NW = PT / 32;
  // quads in flight per thread: 64 registers at 1024 threads allow 2; 512-thread
  // CTAs mostly remove slices of at most one or two quads per thread, and one
  // quad leaves the registers the slice cache needs (17.9K core: 1.906 us/batch
  // at 4, 1.878 at 2, 1.849 at 1)
#ifndef DG_UQ512
#define DG_UQ512 1
#endif
  // (1024 threads: one quad too -- RMAT-26's 84K core 3.42 -> 3.12 us/batch,
  // RMAT-28's 122K core 3.52 -> 3.19, 56 registers instead of 64: a pass of the
  // CTA covers 4K arcs, so the second quad was almost always predicated off)
#ifndef DG_UQ1024
#define DG_UQ1024 1
#endif
  constexpr int UQ = PT >= 1024 ? DG_UQ1024 : DG_UQ512;
  static_assert(CS <= 16, "summary slots");
  static_assert(sizeof(Fixed) % 16 == 0, "cache slots follow Fixed, 16-byte aligned");
  using R = Range<uint32_t>;
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t NC = a.nc;
  const uint32_t NO = a.no;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
  uint32_t* soffs = keys + NC;  // NC + 1 entries when staged
  const size_t head = (size_t(NC) * 4 * (a.offs_smem ? 2 : 1) + 4 + 15) & ~size_t(15);
  uint32_t* sslice = reinterpret_cast<uint32_t*>(smem + head);  // n entries when staged
  Fixed& s = *reinterpret_cast<Fixed*>(
      smem + head + (PT == 512 && a.slice_smem ? ((size_t(a.n) * 4 + 15) & ~size_t(15)) : 0));
  const uint4* adj4 = reinterpret_cast<const uint4*>(a.adj);
  // Slice cache (512-thread CTAs with the slice bounds in shared memory).  A
  // CTA's candidate that loses a batch is a likely member of the next ones
  // (RMAT-26's 17.9K core: 3 of 4 members were their CTA's candidate one batch
  // earlier), so after the decode the last warp copies this CTA's slice of
  // every such candidate's row into slot q (q = the candidate's CTA) with
  // cp.async.bulk, completing on the slot's mbarrier; a member whose id matches
  // a slot's tag is removed from shared memory instead of paying the L2 / HBM
  // round trip of its row on the batch's critical path.
  constexpr bool CACHE = PT == 512;
  const uint32_t slotq = CACHE && a.slice_smem ? a.slotq : 0u;
  uint4* cdata = reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(&s) + sizeof(Fixed));
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const uint32_t n = a.n, c = a.chunk, lo = tid * c, hi = lo + c;
  const uint32_t gbase = rank * NO;  // first global id owned by this CTA
  const bool vec = (c & 3u) == 0;
  const uint32_t keys_s = smem_u32(keys);

  const uint32_t gend = min(n, gbase + NO);  // end of the owned range
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t g = gbase + i;
    if (g < gend) {
      const uint64_t o0 = a.offs[g], o1 = a.offs[g + 1];
      keys[i] = uint32_t(a.loads[g] - a.base + (o1 - o0));
      if (a.offs_smem) soffs[i] = uint32_t(o0);
    } else {
      keys[i] = R::DEAD;
      if (a.offs_smem) soffs[i] = uint32_t(a.offs[gend]);
    }
  }
  if (a.offs_smem && tid == 0) soffs[NC] = uint32_t(a.offs[gend]);
  if (PT == 512 && a.slice_smem)  // removal reads its row slices without a global round trip
    for (uint32_t v = tid; v < n; v += PT) {
      const uint32_t* sg = a.seg + size_t(v) * (CS + 1) + rank;
      sslice[v] = sg[0] | (sg[1] << 16);
    }
  for (uint32_t e = tid; e < NW * NW; e += PT) {
    const uint32_t b = e / NW + 1, ww = e % NW;
    const uint32_t jj = ww % b;
    s.wmap[b - 1][ww] = jj | ((ww / b) << 8) | (((NW - 1 - jj) / b + 1) << 16);
  }
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(smem_u32(&s.mbA[k]));
      mbar_init(smem_u32(&s.mbB[k]));
    }
    if constexpr (CACHE)
      for (int k = 0; k < 16; ++k) {
        mbar_init(smem_u32(&s.mbS[k]));
        s.ctag[k] = kNoTag | (1u << 31);  // parity 1: "the previous phase" of a fresh mbarrier
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // every CTA's mbarriers exist before the first push
#ifndef DG_WMAP_REG
#define DG_WMAP_REG 1
#endif
  // this warp's column of the warp -> member map, lane b - 1 <- wmap[b - 1][w]:
  // a shuffle per batch instead of a dependent shared load (512-thread CTAs)
  uint32_t wmreg = 0;
  if (DG_WMAP_REG && PT == 512 && lane < NW) wmreg = s.wmap[lane][w];

  // CTA `rank`'s slice [s0, s1) of row v (offsets inside the row)
  // (512-thread CTAs only: the cores large enough for 1024-thread CTAs never
  // fit every row's slices, and their 64-register budget has no room)
  auto slice_of = [&](uint32_t v, uint32_t& s0, uint32_t& s1) {
    if (PT == 512 && a.slice_smem) {
      const uint32_t x = sslice[v];
      s0 = x & 0xffffu;
      s1 = x >> 16;
    } else {
      const uint32_t* sg = a.seg + size_t(v) * (CS + 1) + rank;
      s0 = sg[0];
      s1 = sg[1];
    }
  };
  uint32_t removed = 0, pos = 0, useB = 0;  // useB bit k: phase parity of mbB[k]
  bool marked = false;  // my chunk holds BATCH marks of the previous batch
  unsigned long long nbat = 0, nsimple = 0, nlarge = 0, clarge = 0, mlarge = 0;
  const bool P = DG_PEEL_PROF && rank == 0 && tid == 0;
  // DG_PEEL_PROF timeline: every CTA's thread 0 stamps (SM clock) batches
  // [arm - 1, arm + 7) into prof[16 + ((batch * 16) + rank) * 8 + k]:
  // k = 0 loop top, 1 summary pushed, 2 summaries arrived, 3 removal done, 4 end
  const unsigned long long arm = (DG_PEEL_PROF && a.prof) ? a.prof[15] : 0ULL;
  auto stamp = [&](unsigned long long b, int k) {
    if (DG_PEEL_PROF && tid == 0 && arm && b + 1 >= arm && b + 1 < arm + 8)
      a.prof[16 + ((b + 1 - arm) * 16 + rank) * 12 + k] = clock64();
  };
  long long c1 = 0, c2 = 0, c3 = 0, tm = DG_PEEL_PROF ? clock64() : 0;
#if DG_PEEL_PROF
  unsigned long long chit[2] = {0, 0}, cmem[2] = {0, 0};
#endif
  while (removed < n) {
    stamp(nbat, 0);
    const uint32_t par = uint32_t(nbat & 1);
    const uint32_t mbA = smem_u32(&s.mbA[par]), mbB = smem_u32(&s.mbB[par]);
    // ---- retire my BATCH marks (no decrement of this CTA's keys runs
    // between the last CTA barrier and the next removal), then
    // ---- S1: CTA summary
    uint32_t lmin = R::DEAD, bits = 0;  // bits: my keys at lmin (chunk <= 32)
    // up to 8 keys per thread: one round of loads into registers serves the
    // retirement, the minimum and the match mask (17.9K core: 2.37 -> 1.99
    // us/batch against reloading the keys for each; a register array of the
    // exact tier, since predicated slots cost issue slots on every batch)
    if (c <= 4) {
      scan_regs<4, R>(keys, lo, c, marked, lmin, bits);
    } else if (c <= 8) {
      scan_regs<8, R>(keys, lo, c, marked, lmin, bits);
    } else if (vec) {
      if (marked) {
        for (uint32_t i = lo; i < hi; ++i)
          if (R::in_batch(keys[i])) keys[i] = R::DEAD;
        marked = false;
      }
      const uint4* kv = reinterpret_cast<const uint4*>(keys) + (lo >> 2);
      for (uint32_t q = 0; q < (c >> 2); ++q) {
        const uint4 v = kv[q];
        lmin = min(min(lmin, min(v.x, v.y)), min(v.z, v.w));
      }
      for (uint32_t q = 0; q < (c >> 2); ++q) {
        const uint4 v = kv[q];
        bits |= ((v.x == lmin) | ((v.y == lmin) << 1) | ((v.z == lmin) << 2) |
                 (uint32_t(v.w == lmin) << 3))
                << (4 * q);
      }
    } else {
      if (marked) {
        for (uint32_t i = lo; i < hi; ++i)
          if (R::in_batch(keys[i])) keys[i] = R::DEAD;
        marked = false;
      }
      for (uint32_t i = lo; i < hi; ++i) lmin = min(lmin, keys[i]);
      for (uint32_t i = lo; i < hi; ++i) bits |= uint32_t(keys[i] == lmin) << (i - lo);
    }
    uint32_t lcnt = __popc(bits);
    const uint32_t lfirst = lo + __ffs(bits) - 1;
    if (!R::alive(lmin)) lmin = R::DEAD, lcnt = 0;
    // my first minimum's row bounds, loaded while the warp reduces (the CTA
    // summary then needs no dependent shared loads after the barrier)
    uint32_t q0 = 0, q1 = 0;
    if (a.offs_smem) {
      q0 = soffs[lfirst];
      q1 = soffs[lfirst + 1];
    }
    const uint32_t wm = __reduce_min_sync(~0u, lmin);
    const uint32_t fl = __ffs(__ballot_sync(~0u, lmin == wm)) - 1;
    const uint32_t wc = __reduce_add_sync(~0u, lmin == wm ? lcnt : 0u);
    if (lane == fl) {
      s.wsum[w] = make_uint4(wm, wc, lfirst, q0);
      s.wdeg[w] = q1 - q0;
    }
    stamp(nbat, 5);
    if (tid == 0) mbar_expect(mbA, CS * uint32_t(sizeof(Summary)));
    __syncthreads();
    stamp(nbat, 6);
    if (w == 0) {  // CTA summary, pushed to every CTA (lane q -> CTA q)
      const uint4 ws = lane < NW ? s.wsum[lane] : make_uint4(R::DEAD, 0u, 0u, 0u);
      const uint32_t wd = lane < NW ? s.wdeg[lane] : 0u;
      const uint32_t x = ws.x;
      const uint32_t cm = __reduce_min_sync(~0u, x);
      const uint32_t fw = __ffs(__ballot_sync(~0u, x == cm)) - 1;
      const uint32_t ccnt = __reduce_add_sync(~0u, x == cm ? ws.y : 0u);
      const uint32_t f = __shfl_sync(~0u, ws.z, fw);
      uint64_t r0 = __shfl_sync(~0u, ws.w, fw), r1 = r0 + __shfl_sync(~0u, wd, fw);
      if (!R::alive(cm)) {
        r0 = r1 = 0;
      } else if (!a.offs_smem) {
        r0 = a.offs[gbase + f];
        r1 = a.offs[gbase + f + 1];
      }
#if DG_ROW_PREFETCH
      // the CTA's candidate is a likely member of this or an early batch:
      // pull its row into L2 while the summaries travel (cores whose
      // adjacency exceeds L2 -- RMAT-26's -- would otherwise pay an HBM
      // round trip on the removal's critical path)
      // (1024-thread CTAs only: at 512 the slice cache's fills bring the losers'
      // rows in, and the prefetch sits on the push path -- 17.9K core 1.833 ->
      // 1.802 without it)
      if (PT >= 1024 && lane == 0 && R::alive(cm) && r1 > r0) {
        const uint64_t b0 = (r0 * 4) & ~uint64_t(15);
        const uint64_t b1 = min((r1 * 4 + 15) & ~uint64_t(15), b0 + (uint64_t(1) << 16));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         reinterpret_cast<const char*>(a.adj) + b0),
                     "r"(uint32_t(b1 - b0))
                     : "memory");
      }
#endif
      stamp(nbat, 7);
      if (lane < CS) {
        const uint32_t bar = mapa(mbA, lane);
        st_async(mapa(smem_u32(&s.sumA[par][rank]), lane),
                 make_uint4(cm, ccnt, gbase + f, uint32_t(r1 - r0)), bar);
        st_async(mapa(smem_u32(&s.sumB[par][rank]), lane),
                 make_uint4(uint32_t(r0), uint32_t(r0 >> 32), 0u, 0u), bar);
      }
    }
    stamp(nbat, 1);
    mbar_wait(mbA, uint32_t(nbat >> 1) & 1u);
    stamp(nbat, 2);
    if (P) {
      const long long t = clock64();
      c1 += t - tm;
      tm = t;
    }
    // ---- S2: every warp decodes the CS summaries (lane q <- CTA q)
    uint32_t rmin = R::DEAD, rcnt = 0, rfirst = 0, rdeg = 0;
    Off rr0 = 0;
    uint32_t ctreg = kNoTag;  // lane q: tag word of cache slot q
    if (lane < CS) {
      if (CACHE && slotq) ctreg = s.ctag[lane];
      const uint4 p0 = s.sumA[par][lane], p1 = s.sumB[par][lane];
      rmin = p0.x;
      rcnt = p0.y;
      rfirst = p0.z;
      rdeg = p0.w;
      rr0 = O64 ? Off(uint64_t(p1.x) | (uint64_t(p1.y) << 32)) : Off(p1.x);
    }
    const uint32_t gmin = __reduce_min_sync(~0u, rmin);
    const bool own = lane < CS && rmin == gmin;
    const uint32_t ownmask = __ballot_sync(~0u, own);
    const uint32_t total = __reduce_add_sync(~0u, own ? rcnt : 0u);
    const uint32_t bs = a.one ? 1u : total;
    if (DG_SC_FILL && CACHE && slotq && w == NW - 1 && lane < CS && R::alive(rmin) && !own &&
        (ctreg & kNoTag) != rfirst) {
      // slot `lane` <- this CTA's slice of CTA `lane`'s candidate (no member of
      // this batch is owned by that CTA, so nobody reads the slot now)
      uint32_t s0, s1;
      slice_of(rfirst, s0, s1);
      const Off qa = (rr0 + s0) >> 2, qb = (rr0 + s1 + 3) >> 2;
      const uint32_t bar = smem_u32(&s.mbS[lane]);
      uint32_t ph = ctreg >> 31, tag = kNoTag;
      if (s1 > s0 && qb - qa <= slotq) {
        mbar_wait(bar, ph);  // the slot's previous copy has landed
        ph ^= 1u;
        const uint32_t bytes = uint32_t(qb - qa) * 16u;
        mbar_expect(bar, bytes);
        bulk_g2s(smem_u32(cdata + lane * slotq), adj4 + qa, bytes, bar);
        tag = rfirst;
      }
      s.ctag[lane] = tag | (ph << 31);
    }
#if DG_PEEL_PROF
    if (rank == 0 && w == 0) {  // would a cache of last batch's candidates' slices hit?
      const bool hit = own && nbat && s.prevc[par][lane] == rfirst;
      const uint32_t hm = __ballot_sync(~0u, hit);
      if (lane < CS) s.prevc[par ^ 1][lane] = rfirst;
      if (lane == 0) {
        const bool simple = a.one || total == uint32_t(__popc(ownmask));
        chit[simple] += __popc(hm);
        cmem[simple] += simple ? bs : uint32_t(__popc(ownmask));
      }
    }
#endif
    if (a.one || total == uint32_t(__popc(ownmask))) {
      // ---- simple batch: owner lane L (CTA L) holds member #(owners below L)
      if (P) ++nsimple;
      const uint32_t rkl = __popc(ownmask & ((1u << lane) - 1u));
      // my CTA's member (if any): every warp marks it before its own
      // decrements (a later mark by another warp only rewrites a batch key)
      const uint32_t mrk = __popc(ownmask & ((1u << rank) - 1u));
      if (((ownmask >> rank) & 1u) && mrk < bs) {
        const uint32_t mv = __shfl_sync(~0u, rfirst, rank);
        if (lane == 0) {
          keys[mv - gbase] = bs == 1 ? R::DEAD : R::BATCH;
          if (w == 0) {
            a.perm[pos + mrk] = mv;
            atomicAdd(reinterpret_cast<unsigned long long*>(&a.raw[pos + mrk]),
                      (unsigned long long)gmin);
          }
        }
        if (bs != 1 && mv - gbase - lo < c) marked = true;
      }
      __syncwarp();
      if (bs <= NW) {
        const uint32_t wm3 = DG_WMAP_REG && PT == 512 ? __shfl_sync(~0u, wmreg, bs - 1)
                                                      : s.wmap[bs - 1][w];
        const uint32_t j = wm3 & 0xffu, rk = (wm3 >> 8) & 0xffu, nwj = wm3 >> 16;
        const uint32_t lj = __ffs(__ballot_sync(~0u, own && rkl == j)) - 1;
        const uint32_t vj = __shfl_sync(~0u, rfirst, lj);
        uint32_t dj = __shfl_sync(~0u, rdeg, lj);
        Off oj = __shfl_sync(~0u, rr0, lj);
        uint32_t tg = kNoTag;  // the tag of the member's CTA's slot
        if constexpr (CACHE) tg = __shfl_sync(~0u, ctreg, lj);
        const bool hit = DG_SC_HIT && CACHE && slotq && (tg & kNoTag) == vj;
        unsigned long long* rawj = reinterpret_cast<unsigned long long*>(&a.raw[pos + j]);
        stamp(nbat, 8);
        if (!hit) {
          // long row: only this CTA's slice; every row when the slice bounds are a
          // shared load away (RMAT-22's 9.1K core in cluster mode 1.814 -> 1.767)
          if (dj >= (PT >= 1024 ? kSliceMin1024 : kSliceMin) || (PT == 512 && a.slice_smem)) {
            uint32_t s0, s1;
            slice_of(vj, s0, s1);
            oj += s0;
            dj = s1 - s0;
          }
          if (bs == 1)
            remove_local<true, UQ, Off>(adj4, keys_s, oj, dj, vj, rk, nwj, lane, gbase, NO, rawj);
          else
            remove_local<false, UQ, Off>(adj4, keys_s, oj, dj, vj, rk, nwj, lane, gbase, NO, rawj);
        } else {  // this CTA's slice of the row sits in cache slot lj
          uint32_t s0, s1;
          slice_of(vj, s0, s1);
          const uint32_t a0 = (uint32_t(oj) + s0) & 3u;
          mbar_wait(smem_u32(&s.mbS[lj]), tg >> 31);
          const uint32_t slot_s = smem_u32(cdata + lj * slotq);
          if (bs == 1)
            remove_cached<true>(slot_s, keys_s, a0, s1 - s0, vj, rk, nwj, lane, gbase, NO, rawj);
          else
            remove_cached<false>(slot_s, keys_s, a0, s1 - s0, vj, rk, nwj, lane, gbase, NO, rawj);
        }
      } else if constexpr (NW < 32) {  // lane j <- member j (the owner lane of rank j)
        const uint32_t lj = (lane < bs ? __fns(ownmask, 0, int(lane) + 1) : 0u) & 31u;
        remove_flat<PT, Off>(adj4, keys_s, bs, __shfl_sync(~0u, rfirst, lj), __shfl_sync(~0u, rdeg, lj),
                    __shfl_sync(~0u, rr0, lj), w, lane, gbase, NO,
                    reinterpret_cast<unsigned long long*>(&a.raw[pos]));
      }
      if (P) {
        const long long t = clock64();
        c2 += t - tm;
        tm = t;
      }
      stamp(nbat, 3);
      __syncthreads();
    } else {
      // ---- general batch (bs >= 2): owners write the batch in ascending id
      if (tid == 0 && bs <= SB) mbar_expect(mbB, bs * uint32_t(sizeof(Member)));
      if (((ownmask >> rank) & 1u) && wm == gmin) {  // this warp owns part of the batch
        const uint32_t cta_off = __reduce_add_sync(~0u, (lane < rank && own) ? rcnt : 0u);
        const uint4 wsl = lane < NW ? s.wsum[lane] : make_uint4(R::DEAD, 0u, 0u, 0u);
        const uint32_t woff = __reduce_add_sync(~0u, (lane < w && wsl.x == gmin) ? wsl.y : 0u);
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
            atomicAdd(reinterpret_cast<unsigned long long*>(&a.raw[pos + my]),
                      (unsigned long long)gmin);
            keys[i] = R::BATCH;
            marked = true;
            if (my < SB && bs <= SB) {
              uint64_t r0, r1;
              if (a.offs_smem) {
                r0 = soffs[i];
                r1 = soffs[i + 1];
              } else {
                r0 = a.offs[g];
                r1 = a.offs[g + 1];
              }
              const uint4 rec = make_uint4(g, uint32_t(r1 - r0), uint32_t(r0), uint32_t(r0 >> 32));
              const uint32_t src = smem_u32(&s.stage[par][my]);
              for (uint32_t q = 0; q < CS; ++q) st_async(mapa(src, q), rec, mapa(mbB, q));
            }
            ++my;
          }
        }
      }
      if (bs <= SB) {
        __syncthreads();  // this CTA's batch marks before its decrements
        mbar_wait(mbB, (useB >> par) & 1u);
        useB ^= 1u << par;
        if (P) {
          const long long t = clock64();
          c2 += t - tm;
          tm = t;
        }
        if (bs <= NW) {
          const uint32_t wm3 = s.wmap[bs - 1][w];
          const uint32_t j = wm3 & 0xffu;
          const Member& mj = s.stage[par][j];
          // only this CTA's slice of the member's row
          uint32_t s0, s1;
          slice_of(mj.v, s0, s1);
          uint32_t hm = 0;
          if constexpr (CACHE && DG_SC_GEN)
            if (slotq) hm = __ballot_sync(~0u, (ctreg & kNoTag) == mj.v);
          if (hm) {
            const uint32_t sl = __ffs(hm) - 1;
            mbar_wait(smem_u32(&s.mbS[sl]), __shfl_sync(~0u, ctreg, sl) >> 31);
            remove_cached<false>(smem_u32(cdata + sl * slotq), keys_s, (mj.r0lo + s0) & 3u, s1 - s0,
                                 mj.v, (wm3 >> 8) & 0xffu, wm3 >> 16, lane, gbase, NO,
                                 reinterpret_cast<unsigned long long*>(&a.raw[pos + j]));
          } else {
            remove_local<false, UQ, Off>(
                adj4, keys_s,
                (O64 ? Off(uint64_t(mj.r0lo) | (uint64_t(mj.r0hi) << 32)) : Off(mj.r0lo)) + s0,
                s1 - s0, mj.v, (wm3 >> 8) & 0xffu, wm3 >> 16, lane, gbase, NO,
                reinterpret_cast<unsigned long long*>(&a.raw[pos + j]));
          }
        } else if constexpr (NW < SB) {
          Member mj = {0u, 0u, 0u, 0u};
          uint32_t s0 = 0, s1 = 0;
          if (lane < bs) {
            mj = s.stage[par][lane];
            slice_of(mj.v, s0, s1);
          }
          remove_flat<PT, Off>(
              adj4, keys_s, bs, mj.v, s1 - s0,
              (O64 ? Off(uint64_t(mj.r0lo) | (uint64_t(mj.r0hi) << 32)) : Off(mj.r0lo)) + s0, w, lane,
              gbase, NO, reinterpret_cast<unsigned long long*>(&a.raw[pos]));
        }
        __syncthreads();
      } else {
        // large batch: every warp takes members w, w + NW, ... and applies
        // the decrements of its slice of their rows to this CTA's keys
        const long long tl0 = P ? clock64() : 0;
        cl.sync();  // perm and every batch mark written
        // 512-thread CTAs: groups of 32 members, each removed as ONE flat
        // range of quads over the whole CTA (lane j of every warp holds member
        // j of the group): the member loads of a group are in flight
        // together, and every thread gets the same share however the slices
        // vary (RMAT-22's 35K core 2.99 -> 2.89 us/batch)
        if constexpr (PT == 512) {
          for (uint32_t g0 = 0; g0 < bs; g0 += 32) {
            const uint32_t gb = min(32u, bs - g0);
            uint32_t mv = 0, s0 = 0, s1 = 0;
            Off o = 0;
            if (lane < gb) {
              mv = a.perm[pos + g0 + lane];
              o = Off(a.offs[mv]);
              slice_of(mv, s0, s1);
            }
            remove_flat<PT, Off>(adj4, keys_s, gb, mv, s1 - s0, o + s0, w, lane, gbase, NO,
                            reinterpret_cast<unsigned long long*>(&a.raw[pos + g0]));
          }
        } else {
          // 1024-thread CTAs (32 warps): a warp per member -- the flat form
          // does not fit their 64-register budget without spilling, and
          // measured no faster there (84K core 3.83 vs 3.78 us/batch)
          for (uint32_t j = w; j < bs; j += NW) {
            const uint32_t vj = a.perm[pos + j];
            const Off oj = Off(a.offs[vj]);
            uint32_t s0, s1;
            slice_of(vj, s0, s1);
            remove_local<false, UQ, Off>(adj4, keys_s, oj + s0, s1 - s0, vj, 0, 1, lane, gbase, NO,
                                    reinterpret_cast<unsigned long long*>(&a.raw[pos + j]));
          }
        }
        __syncthreads();
        if (P) ++nlarge, clarge += clock64() - tl0, mlarge += bs;
      }
    }
    if (P) {
      const long long t = clock64();
      c3 += t - tm;
      tm = t;
    }
    stamp(nbat, 4);
    pos += bs;
    removed += bs;
    ++nbat;
  }
  if (CACHE && slotq && w == NW - 1 && lane < CS)  // no copy in flight at exit
    mbar_wait(smem_u32(&s.mbS[lane]), s.ctag[lane] >> 31);
  if (rank == 0 && tid == 0) *a.batches = nbat;
  if (P) {
    if (a.prof) {
      a.prof[0] = c1;
      a.prof[1] = c2;
      a.prof[2] = c3;
      a.prof[3] = nbat;
      a.prof[4] = nsimple;
      a.prof[5] = nlarge;
      a.prof[6] = clarge;
      a.prof[8] = mlarge;
      a.prof[7] = CS;
    }
  }
#if DG_PEEL_PROF
  if (rank == 0 && tid == 0 && a.prof) {
    a.prof[9] = chit[1], a.prof[10] = cmem[1], a.prof[11] = chit[0], a.prof[12] = cmem[0];
  }
#endif
  cl.sync();  // no CTA exits while a push into it could be in flight
}

inline size_t smem_bytes(uint32_t nc, bool offs_smem, uint64_t slice_n = 0, uint32_t slotq = 0) {
  const size_t NC = nc;
  return ((NC * 4 * (offs_smem ? 2 : 1) + 4 + 15) & ~size_t(15)) +
         ((slice_n * 4 + 15) & ~size_t(15)) + sizeof(Fixed) + size_t(slotq) * 16 * 16;
}

}  // namespace peelc
}  // namespace dgb
