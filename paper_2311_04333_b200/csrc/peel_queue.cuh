// peel_queue.cuh -- Greedy++ batch peel with a shared-memory candidate list
// (the B200 form of the reference's bucket queue, refine.cpp:60-120
// `peel_buckets`): one CTA, u32 keys in shared memory, batch mode.
//
// Semantics, key ranges and the fused Alg. 3 charge are those of
// peel_kernel.cuh (refine.cpp:20-156).  What changes is how the minimum is
// found.  k_peel rescans every key of the core for every batch; here the CTA
// keeps a window [.., thr) just above the minimum:
//
//   invariant: every alive vertex whose key is < thr is in list[0, lcount)
//
// so the batch minimum is the minimum over the list (all other alive keys
// are >= thr), and a batch is the list entries at that key.  Keys only
// decrease, so a vertex enters the window exactly once, when a decrement
// takes its key from thr to thr - 1; removal decrements are atom.shared.add
// and the returned key detects that crossing (append).  When the list holds
// no alive vertex, overflows, or the tie group at the minimum is too large to
// stage, a full scan REBASES: global minimum gm, window width W adapted so
// ~1K vertices fall below thr = gm + W, list rebuilt in ascending id.
//
// Per list batch:
//   S1  each thread reads its <= 4 list entries and their keys: (min, count)
//       -> redux.sync -> warp table            --- barrier A
//   S2  every warp reduces the table (gmin, batch size); threads holding a
//       member stage (v, row, degree) and mark it BATCH (DEAD if alone)
//                                                --- barrier B
//   S3  warp w serves member w mod bs (16-byte adjacency quads, atom.shared
//       decrements: same-batch counting + window crossings); the last warp
//       ranks the members by id -> perm (the reference's ascending-id order)
//                                                --- barrier C
//   the batch's raw charges and BATCH -> DEAD retirement run in the next S1.
// Tie groups beyond MCAP members take an ordered full-scan batch (owners
// write the batch in id order, removal in slices of 1024 members).
#pragma once

namespace dgb {
namespace peelq {

using peelk::Range;
constexpr int PT = 1024;
constexpr uint32_t NW = PT / 32;
constexpr int UQ = 2;              // adjacency quads in flight per thread
constexpr uint32_t LCAP = 4096;    // candidate list capacity
constexpr uint32_t LPT = LCAP / PT;
#ifndef DG_PEEL_LTARGET
#define DG_PEEL_LTARGET 512
#endif
constexpr uint32_t LTARGET = DG_PEEL_LTARGET;  // list size the window width aims at
constexpr uint32_t MCAP = PT;      // members staged per list batch
using R = Range<uint32_t>;

struct Args {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  const uint64_t* loads;
  uint64_t base;
  uint32_t* perm;
  uint64_t* raw;
  unsigned long long* batches;
  unsigned long long* prof;  // [9] rebases, [10] full-scan batches, [11] list batches
};

struct Q {
  uint32_t list[2][LCAP];  // double-buffered: S2 compacts into the other buffer
  uint32_t mem[MCAP];   // batch members (arrival order)
  uint64_t moff[MCAP];  // their row starts
  uint32_t mdeg[MCAP];
  uint32_t mcnt[MCAP];  // same-batch neighbours with a smaller id
  uint32_t mrank[MCAP]; // ascending-id rank inside the batch
  uint64_t pre[PT];
  uint64_t ws[33];
  uint32_t wmin[NW], wcnt[NW];
  uint32_t wmap[NW][NW];  // as peel_kernel.cuh: j | rank << 8 | nwj << 16
  struct alignas(16) Hdr {
    uint32_t lcount[2], nmem, overflow;  // read together (uint4)
  } h;
  uint32_t gmin[2];  // red.shared.min of the scanning warps' minima, by list-batch parity
  alignas(16) uint32_t cmd[4];  // S2 -> all warps: batch size (0: rebase), gmin, thr
};

template <int VQ, bool OFFS>
constexpr size_t smem_bytes() {
  constexpr size_t npad = size_t(4 * VQ) * PT;
  return npad * 4 + (OFFS ? (((npad + 1) * 4 + 15) & ~size_t(15)) : 0) + sizeof(Q);
}

__device__ __forceinline__ void append(Q& q, uint32_t buf, uint32_t u) {
  const uint32_t s = atomicAdd(&q.h.lcount[buf], 1u);
  if (s < LCAP)
    q.list[buf][s] = u;
  else
    q.h.overflow = 1;
}

// decrement key u, returning the old key
__device__ __forceinline__ uint32_t dec_atom(uint32_t keys_s, uint32_t u) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(keys_s + (u << 2)), "r"(0xffffffffu)
               : "memory");
  return old;
}

// the old key tells same-batch members (BATCH range) and window crossings
// (old == thr) apart
template <bool ONE>
__device__ __forceinline__ void dec_check(uint32_t old, uint32_t u, uint32_t vj, uint32_t* cnt,
                                          uint32_t thr, Q& q, uint32_t buf) {
  if (!ONE && R::in_batch(old) && u < vj) atomicAdd(cnt, 1u);
  if (old == thr) append(q, buf, u);
}

template <bool ONE>
__device__ __forceinline__ void dec(uint32_t keys_s, uint32_t u, uint32_t vj, uint32_t* cnt,
                                    uint32_t thr, Q& q, uint32_t buf) {
  dec_check<ONE>(dec_atom(keys_s, u), u, vj, cnt, thr, q, buf);
}

template <bool ONE>
__device__ __forceinline__ void remove_row(const uint4* adj4, uint32_t keys_s, uint64_t oj,
                                           uint32_t dj, uint32_t vj, uint32_t rank, uint32_t nwj,
                                           uint32_t lane, uint32_t* cnt, uint32_t thr, Q& q,
                                           uint32_t buf) {
  const uint4* row = adj4 + (oj >> 2);
  const uint32_t head = uint32_t(oj & 3), end = head + dj;  // valid elements [head, end)
  const uint32_t nq = (end + 3) >> 2, stride = nwj * 32;
  for (uint32_t b = rank * 32 + lane; b < nq; b += stride * UQ) {
    uint4 x[UQ];
#pragma unroll
    for (int k = 0; k < UQ; ++k)
      if (b + k * stride < nq) x[k] = __ldg(row + b + k * stride);
#pragma unroll
    for (int k = 0; k < UQ; ++k) {
      const uint32_t t = b + k * stride;
      if (t >= nq) break;
      const uint32_t e0 = t << 2;
      if (e0 >= head && e0 + 4 <= end) {  // full quad: four atomics in flight, then checks
        const uint32_t o0 = dec_atom(keys_s, x[k].x), o1 = dec_atom(keys_s, x[k].y);
        const uint32_t o2 = dec_atom(keys_s, x[k].z), o3 = dec_atom(keys_s, x[k].w);
        dec_check<ONE>(o0, x[k].x, vj, cnt, thr, q, buf);
        dec_check<ONE>(o1, x[k].y, vj, cnt, thr, q, buf);
        dec_check<ONE>(o2, x[k].z, vj, cnt, thr, q, buf);
        dec_check<ONE>(o3, x[k].w, vj, cnt, thr, q, buf);
      } else {
        const uint32_t us[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e0 + e >= head && e0 + e < end) dec<ONE>(keys_s, us[e], vj, cnt, thr, q, buf);
      }
    }
  }
}

// removal of staged members [0, sl) -- every thread calls it (barriers
// inside).  The members' rows are concatenated as 16-byte quads (a CTA scan
// over per-member quad counts); warps take 32-quad chunks, a lane finds its
// member by stepping forward from the chunk's first member (rows are long,
// so usually zero steps), loads its quad and decrements its valid arcs.
__device__ __forceinline__ void remove_slice(const uint32_t* adj, uint32_t keys_s, uint32_t sl,
                                             uint32_t tid, uint32_t lane, uint32_t w,
                                             uint32_t thr, Q& q, uint32_t buf) {
  const uint4* adj4 = reinterpret_cast<const uint4*>(adj);
  const uint64_t nqj =
      tid < sl ? ((q.moff[tid] & 3) + q.mdeg[tid] + 3) >> 2 : 0;  // quads of member tid
  uint64_t tot;
  const uint64_t ex = block_excl_scan(nqj, q.ws, &tot);
  q.pre[tid] = ex;  // first quad of member tid (exclusive prefix)
  __syncthreads();
  const uint64_t nch = (tot + 31) / 32;
  for (uint64_t c = w; c < nch; c += NW) {
    const uint64_t x0 = c * 32;
    // chunk's first member: largest j with pre[j] <= x0 (lane-parallel search)
    uint32_t j0 = 0;
    {
      uint32_t lo = 0, hi = sl - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (q.pre[mid] <= x0)
          lo = mid;
        else
          hi = mid - 1;
      }
      j0 = lo;
    }
    const uint64_t x = x0 + lane;
    if (x >= tot) continue;
    uint32_t j = j0;
    while (j + 1 < sl && q.pre[j + 1] <= x) ++j;
    const uint64_t oj = q.moff[j];
    const uint32_t head = uint32_t(oj & 3), end = head + q.mdeg[j];
    const uint32_t qi = uint32_t(x - q.pre[j]);
    const uint4 v4 = __ldg(adj4 + (oj >> 2) + qi);
    const uint32_t us[4] = {v4.x, v4.y, v4.z, v4.w};
    const uint32_t vj = q.mem[j];
    uint32_t old[4];
    const uint32_t e0 = qi << 2;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      old[e] = (e0 + e >= head && e0 + e < end) ? dec_atom(keys_s, us[e]) : R::DEAD;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e0 + e >= head && e0 + e < end) dec_check<false>(old[e], us[e], vj, &q.mcnt[j], thr, q, buf);
  }
}

template <bool OFFS, int VQ, bool TR>
__global__ void __launch_bounds__(PT, 1) k_peel_queue(Args a) {
  extern __shared__ __align__(16) unsigned char raw_smem[];
  constexpr uint32_t C = 4 * VQ;
  constexpr uint32_t npad = C * PT;
  uint32_t* keys = reinterpret_cast<uint32_t*>(raw_smem);
  size_t o = size_t(npad) * 4;
  uint32_t* soffs = reinterpret_cast<uint32_t*>(raw_smem + o);  // u32 row starts, n+1
  if (OFFS) o += ((size_t(npad) + 1) * 4 + 15) & ~size_t(15);
  Q& q = *reinterpret_cast<Q*>(raw_smem + o);
  const uint4* adj4 = reinterpret_cast<const uint4*>(a.adj);
  const uint32_t keys_s = peelk::smem_addr(keys);
  const uint32_t tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const uint32_t n = a.n, lo = tid * C;

  for (uint32_t i = lo; i < lo + C; ++i) {
    if (i < n) {
      const uint64_t o0 = a.offs[i], o1 = a.offs[i + 1];
      keys[i] = uint32_t(a.loads[i] - a.base + (o1 - o0));
      if (OFFS) soffs[i] = uint32_t(o0);
    } else {
      keys[i] = R::DEAD;
    }
  }
  if (OFFS && tid == 0) soffs[n] = uint32_t(a.offs[n]);
  for (uint32_t e = tid; e < NW * NW; e += PT) {
    const uint32_t b = e / NW + 1, ww = e % NW, jj = ww % b;
    q.wmap[b - 1][ww] = jj | ((ww / b) << 8) | (((NW - 1 - jj) / b + 1) << 16);
  }
  if (tid == 0) {
    q.h.lcount[0] = q.h.lcount[1] = q.h.nmem = q.h.overflow = 0;
    q.gmin[0] = q.gmin[1] = R::DEAD;
  }
  __syncthreads();

  const unsigned long long tr_first = TR ? a.prof[15] : 0;
#define PQ_STAMP(k, dep)                                                          \
  if constexpr (TR) {                                                             \
    if (tr_first && lane == 0) peelk::stamp(a.prof, tr_first, nbat, w, k, dep); \
  }
  uint32_t removed = 0, pos = 0, thr = 0, W = 64, lp = 0, gp = 0;  // list buffer S1 reads, gmin slot
  bool valid = false;                           // list invariant established (uniform)
  uint32_t pnm = 0, ppos = 0, pkey = 0;         // previous list batch (deferred work)
  unsigned long long nbat = 0, nreb = 0, nfull = 0, nlist = 0;
  while (removed < n) {
    PQ_STAMP(0, q.h.nmem);
    // ---- deferred: raw charges and BATCH -> DEAD of the previous list batch
    // (no decrements run between barriers C and B)
    if (tid < pnm) {
      a.raw[ppos + q.mrank[tid]] = uint64_t(pkey) - q.mcnt[tid];
      keys[q.mem[tid]] = R::DEAD;
    }
    pnm = 0;
    // Dependent shared-memory steps dominate a batch on this part (measured:
    // LDS ~75, redux.sync ~97, returning shared atomic ~139, barrier ~80
    // cycles), so the control path is short and runs on the ns warps that
    // hold list entries (128 each); the other warps wait at barrier B.
    const uint4 hdr = *reinterpret_cast<const uint4*>(&q.h);  // lcount[2], nmem, overflow
    const bool listok = valid && hdr.w == 0;
    const uint32_t lc = listok ? min(lp ? hdr.y : hdr.x, LCAP) : 0u;
    const uint32_t ns = max(1u, min(NW, (lc + 127) / 128));
    // window width for this batch's compaction: the list aims at LTARGET
    if (lc > 2 * LTARGET)
      W = max(1u, W >> 1);
    else if (lc < LTARGET / 2)
      W = min(W << 1, 1u << 24);
    PQ_STAMP(6, lc);
    if (w < ns) {
      // ---- S1: minimum over the candidate list
      uint32_t lv[LPT], lk[LPT];
#pragma unroll
      for (uint32_t k = 0; k < LPT; ++k) {
        const uint32_t i = w * 128 + k * 32 + lane;
        lv[k] = i < lc ? q.list[lp][i] : 0u;
      }
#pragma unroll
      for (uint32_t k = 0; k < LPT; ++k) lk[k] = w * 128 + k * 32 + lane < lc ? keys[lv[k]] : R::DEAD;
      PQ_STAMP(7, lk[0]);
      uint32_t lmin = R::DEAD, lfv = 0;
#pragma unroll
      for (uint32_t k = 0; k < LPT; ++k) lmin = min(lmin, lk[k]);
#pragma unroll
      for (int k = LPT - 1; k >= 0; --k)
        if (lk[k] == lmin) lfv = lv[k];
      // row bounds of my first minimum, issued now (overlaps the reduction)
      uint64_t pf0 = 0, pf1 = 0;
      if (R::alive(lmin)) {
        pf0 = OFFS ? uint64_t(soffs[lfv]) : a.offs[lfv];
        pf1 = OFFS ? uint64_t(soffs[lfv + 1]) : a.offs[lfv + 1];
      }
      const uint32_t wm = __reduce_min_sync(~0u, lmin);
      PQ_STAMP(8, wm);
      if (lane == 0 && R::alive(wm))
        asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(peelk::smem_addr(&q.gmin[gp])), "r"(wm)
                     : "memory");
      if (tid == 0) {
        q.h.nmem = 0;
        q.h.lcount[lp ^ 1] = 0;  // the compaction target (read last by the previous batch)
      }
      PQ_STAMP(1, 0);
      asm volatile("bar.sync 1, %0;" ::"r"(ns * 32) : "memory");  // A (scanning warps)
      // ---- S2: stage the members (list entries at gmin); compact the list
      const uint32_t gmin = q.gmin[gp];
      PQ_STAMP(2, gmin);
      if (R::alive(gmin)) {
        if (lmin == gmin) {
#pragma unroll
          for (uint32_t k = 0; k < LPT; ++k) {
            if (lk[k] != gmin) continue;
            const uint32_t v = lv[k], s = atomicAdd(&q.h.nmem, 1u);
            if (s >= MCAP) continue;  // tie group beyond the staging: full-scan batch
            uint64_t r0 = pf0, r1 = pf1;
            if (v != lfv) {
              r0 = OFFS ? uint64_t(soffs[v]) : a.offs[v];
              r1 = OFFS ? uint64_t(soffs[v + 1]) : a.offs[v + 1];
            }
            q.mem[s] = v;
            q.moff[s] = r0;
            q.mdeg[s] = uint32_t(r1 - r0);
            q.mcnt[s] = 0;
            keys[v] = R::BATCH;  // dead before any decrement
          }
        }
        // compaction into the other buffer: alive entries below the (possibly
        // lowered) threshold tn, minus this batch's members.  Lowering keeps
        // the invariant: a dropped entry can only come back below tn by a
        // decrement crossing tn, which S3 appends.
        const uint32_t tn = uint32_t(min(uint64_t(thr), uint64_t(gmin) + W));
        uint32_t m[LPT], tot = 0;
#pragma unroll
        for (uint32_t k = 0; k < LPT; ++k) {
          m[k] = __ballot_sync(~0u, lk[k] < tn && lk[k] != gmin);  // alive and kept
          tot += __popc(m[k]);
        }
        uint32_t base = 0;
        if (lane == 0 && tot) base = atomicAdd(&q.h.lcount[lp ^ 1], tot);
        base = __shfl_sync(~0u, base, 0);
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (uint32_t k = 0; k < LPT; ++k) {
          if (m[k] >> lane & 1u) q.list[lp ^ 1][base + __popc(m[k] & lt)] = lv[k];
          base += __popc(m[k]);
        }
        if (tid == 0) q.cmd[2] = tn;
      }
    }
    PQ_STAMP(3, 0);
    __syncthreads();  // B
    const uint32_t gmin = q.gmin[gp], bs = q.h.nmem;
    const uint64_t moff0 = q.moff[0];
    const uint32_t mdeg0 = q.mdeg[0];
    PQ_STAMP(4, bs);
    if (R::alive(gmin) && bs <= MCAP) {
      thr = q.cmd[2];
      lp ^= 1;  // S3 appends to the compacted buffer, the next S1 reads it
      ++nlist;
      if (tid == 0) q.gmin[gp ^ 1] = R::DEAD;  // last read before the previous barrier C
      gp ^= 1;
      // ---- S3: ranks (ascending id -> perm) and removal
      const uint32_t rt = bs <= 32 ? tid - (PT - 32) : tid;  // the last warp for small batches
      if (rt < bs) {
        const uint32_t v = q.mem[rt];
        uint32_t r = 0;
        for (uint32_t s = 0; s < bs; ++s) r += q.mem[s] < v;
        q.mrank[rt] = r;
        a.perm[pos + r] = v;
      }
      if (bs == 1) {
        remove_row<true>(adj4, keys_s, moff0, mdeg0, 0, w, NW, lane, nullptr, thr, q, lp);
      } else if (bs <= NW) {
        const uint32_t wm3 = q.wmap[bs - 1][w];
        const uint32_t j = wm3 & 0xffu, rank = (wm3 >> 8) & 0xffu, nwj = wm3 >> 16;
        remove_row<false>(adj4, keys_s, q.moff[j], q.mdeg[j], q.mem[j], rank, nwj, lane,
                          &q.mcnt[j], thr, q, lp);
      } else {
        remove_slice(a.adj, keys_s, bs, tid, lane, w, thr, q, lp);
      }
      PQ_STAMP(5, 0);
      __syncthreads();  // C
      pnm = bs;
      ppos = pos;
      pkey = gmin;
      pos += bs;
      removed += bs;
      ++nbat;
      continue;
    }
    if (R::alive(gmin)) {
      // tie group beyond the staging: undo the staged marks, rebase (the full
      // scan then runs an ordered full-scan batch)
      if (tid < MCAP) keys[q.mem[tid]] = gmin;
      valid = false;
    }
    if (tid == 0) q.gmin[gp] = R::DEAD;  // every warp has read it (barrier B)
    __syncthreads();
    // ---- rebase: full scan for the global minimum
    ++nreb;
    uint32_t fmin = R::DEAD, fcnt = 0, ffirst = lo;
    if (lo < n) peelk::chunk_min_count<VQ>(keys, lo, C, fmin, fcnt, ffirst);
    if (!R::alive(fmin)) fmin = R::DEAD, fcnt = 0;
    {
      const uint32_t m = __reduce_min_sync(~0u, fmin);
      const uint32_t c = __reduce_add_sync(~0u, fmin == m ? fcnt : 0u);
      if (lane == 0) {
        q.wmin[w] = m;
        q.wcnt[w] = c;
      }
    }
    __syncthreads();
    const uint32_t gm = __reduce_min_sync(~0u, q.wmin[lane]);
    const uint32_t cgm = __reduce_add_sync(~0u, q.wmin[lane] == gm ? q.wcnt[lane] : 0u);
    if (cgm <= MCAP) {
      // rebuild the window [gm, gm + Wt) with about LTARGET vertices
      uint32_t Wt = W;
      for (;;) {
        const uint32_t t = uint32_t(min(uint64_t(gm) + Wt, uint64_t(R::ALIVE_END)));
        uint32_t c = 0;
        if (lo < n)
          for (uint32_t i = lo; i < lo + C; ++i) c += keys[i] < t;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(c, reinterpret_cast<uint32_t*>(q.ws), &tot);
        if (tot > LTARGET && Wt > 1) {
          Wt >>= 1;
          __syncthreads();  // ws reuse
          continue;
        }
        // tot <= LTARGET, or Wt == 1 (then tot == cgm <= MCAP <= LCAP)
        uint32_t s = ex;
        if (c)
          for (uint32_t i = lo; i < lo + C; ++i)
            if (keys[i] < t) q.list[lp][s++] = i;
        if (tid == 0) {
          q.h.lcount[lp] = tot;
          q.h.overflow = 0;
        }
        thr = t;
        W = tot < LTARGET / 4 ? min(Wt * 2, 1u << 24) : Wt;
        break;
      }
      valid = true;
      __syncthreads();
      continue;
    }
    // ---- full-scan batch: the tie group at gm exceeds the staging; owners
    // write it in ascending id, removal in slices of PT members
    ++nfull;
    valid = false;
    {
      uint32_t bsf;
      const uint32_t ex = block_excl_scan(fmin == gm ? fcnt : 0u, reinterpret_cast<uint32_t*>(q.ws),
                                          &bsf);
      if (fmin == gm) {
        uint32_t s = pos + ex;
        for (uint32_t i = lo; i < lo + C; ++i)
          if (keys[i] == gm) {
            a.perm[s++] = i;
            keys[i] = R::BATCH;
          }
      }
      __syncthreads();
      for (uint32_t s0 = 0; s0 < bsf; s0 += PT) {
        const uint32_t sl = min(uint32_t(PT), bsf - s0);
        if (tid < sl) {
          const uint32_t v = a.perm[pos + s0 + tid];
          const uint64_t r0 = OFFS ? soffs[v] : a.offs[v];
          const uint64_t r1 = OFFS ? soffs[v + 1] : a.offs[v + 1];
          q.mem[tid] = v;
          q.moff[tid] = r0;
          q.mdeg[tid] = uint32_t(r1 - r0);
          q.mcnt[tid] = 0;
        }
        __syncthreads();
        remove_slice(a.adj, keys_s, sl, tid, lane, w, R::ALIVE_END, q, lp);
        __syncthreads();
        if (tid < sl) a.raw[pos + s0 + tid] = uint64_t(gm) - q.mcnt[tid];
        __syncthreads();
      }
      for (uint32_t s = tid; s < bsf; s += PT) keys[a.perm[pos + s]] = R::DEAD;
      __syncthreads();
      pos += bsf;
      removed += bsf;
      ++nbat;
    }
  }
#undef PQ_STAMP
  if (tid < pnm) a.raw[ppos + q.mrank[tid]] = uint64_t(pkey) - q.mcnt[tid];
  if (tid == 0) {
    *a.batches = nbat;
    if (a.prof) {
      a.prof[3] = nbat;
      a.prof[9] = nreb;
      a.prof[10] = nfull;
      a.prof[11] = nlist;
    }
  }
}

}  // namespace peelq
}  // namespace dgb
