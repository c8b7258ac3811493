// kcore.cu -- exact / approximate coreness as ONE persistent cooperative
// kernel (reference core.cpp:18-131).
//
// Semantics reproduced exactly (labels, kmax, peel_rounds):
//   round at bound b: every alive vertex with residual degree <= b leaves
//   (label = current label), then alive neighbours lose one degree per removed
//   neighbour.  A round is "non-empty" iff it removes something; when none is
//   left at b the bound advances (exact: to the minimum alive degree, which
//   is what the reference's ++bound loop reaches; approximate: geometric
//   phases t_{i+1} = max(t_i + 1, ceil(c t_i)) until b >= min degree).
//
// B200 mapping:
//   * frontier of round r+1 = vertices whose degree crossed b+1 -> b during
//     round r, detected by the atomicSub return value (no bucket rescans);
//   * frontier entries carry an exclusive arc prefix, and a "chunk-start"
//     table cse[c] = entry holding arc c*CH, so the expansion is perfectly
//     load balanced over warps (hub rows are spread over many warps) with
//     one coalesced adjacency pass;
//   * appends are aggregated in shared memory and published with ONE packed
//     64-bit atomic per CTA per tile: (count << 36) | arcs;  a CTA whose
//     buffer overflows leaves the vertex unlabelled and raises a flag, and an
//     extra collect phase picks those up from the live list;
//   * the live list (alive vertices) is compacted at every level advance, so
//     min-degree scans shrink with the graph;
//   * one generation barrier per round (two per level advance).
#include <cooperative_groups.h>

#include "internal.cuh"

namespace dgb {

namespace {

constexpr int KC_THREADS = 1024;
constexpr uint32_t CH = 128;   // arcs per warp work chunk (4 per lane)
constexpr uint32_t BUF = 6144; // per-CTA crossing buffer
constexpr uint32_t kUnset = 0xffffffffu;
constexpr uint64_t M36 = (1ULL << 36) - 1;

struct Acc {
  unsigned long long front;  // (count << 36) | arcs of the frontier being built
  unsigned long long live;   // live-list entries written
  uint32_t minv;             // min alive degree (level advance)
  uint32_t ovf;              // some CTA buffer overflowed while building
};

struct KcArgs {
  const uint64_t* offs;
  const uint32_t* adj;
  uint32_t n;
  uint32_t* deg;
  uint32_t* labels;
  uint32_t* live0;
  uint32_t* live1;
  uint32_t* fr0;
  uint32_t* fr1;
  uint64_t* fa0;
  uint64_t* fa1;
  uint32_t* cse0;
  uint32_t* cse1;
  Acc* acc;  // [3]
  GridBarrier* bar;
  uint32_t* out;  // kmax, rounds, err
  int approx;
  uint64_t c_num, c_den;
};

struct Smem {
  uint32_t id[BUF];
  uint32_t dg[BUF];
  uint64_t tileA[KC_THREADS];
  uint64_t ws[33];
  uint32_t ws32[33];
  uint32_t cnt;
  unsigned long long baseF, baseL;
  uint32_t minv;
  // phase scalars fetched by thread 0 after each grid barrier
  uint32_t abort;
  unsigned long long b_front, b_live;
  uint32_t b_minv, b_ovf;
};

__device__ __forceinline__ void fetch_acc(Smem& s, Acc* acc) {
  s.b_front = ld_relaxed_u64(&acc->front);
  s.b_live = ld_relaxed_u64(&acc->live);
  s.b_minv = ld_relaxed_u32(&acc->minv);
  s.b_ovf = ld_relaxed_u32(&acc->ovf);
}

__device__ __forceinline__ uint32_t deg_full(const uint64_t* offs, uint32_t v) {
  return uint32_t(offs[v + 1] - offs[v]);
}

// All threads of the CTA call this with a per-thread candidate (isF, v, d).
// Publishes the tile's entries into frontier (fr, fa) with one atomic,
// labels them, and fills the chunk-start table for the tile's arc range.
__device__ __forceinline__ void emit_front_tile(bool isF, uint32_t v, uint32_t d, uint32_t label,
                                                const KcArgs& a, uint32_t* fr, uint64_t* fa,
                                                uint32_t* cse, Acc* acc, Smem& s) {
  uint64_t pk = isF ? ((1ULL << 36) | d) : 0ULL;
  uint64_t tot;
  uint64_t ex = block_excl_scan(pk, s.ws, &tot);
  if (tot == 0) return;  // uniform: nothing in this tile (block_excl_scan synced)
  if (threadIdx.x == 0) s.baseF = atomicAdd(&acc->front, (unsigned long long)tot);
  __syncthreads();
  const uint64_t base = s.baseF;
  const uint64_t e0 = base >> 36, A0 = base & M36;
  if (isF) {
    uint64_t k = ex >> 36, A = A0 + (ex & M36);
    fr[e0 + k] = v;
    fa[e0 + k] = A;
    a.labels[v] = label;
    s.tileA[k] = A;
  }
  __syncthreads();
  const uint64_t cnt = tot >> 36, TA = tot & M36;
  if (TA) {
    const uint64_t c_lo = (A0 + CH - 1) / CH, c_hi = (A0 + TA - 1) / CH;
    for (uint64_t c = c_lo + threadIdx.x; c <= c_hi; c += blockDim.x) {
      const uint64_t x = c * CH;
      uint64_t lo = 0, hi = cnt - 1;  // largest k with tileA[k] <= x
      while (lo < hi) {
        uint64_t mid = (lo + hi + 1) >> 1;
        if (s.tileA[mid] <= x)
          lo = mid;
        else
          hi = mid - 1;
      }
      cse[c] = uint32_t(e0 + lo);
    }
  }
  __syncthreads();
}

// Scan the live list: alive vertices with deg <= bound join the frontier,
// the other alive ones are compacted into live_out.
__device__ void collect(const KcArgs& a, uint32_t livec, bool implicit, const uint32_t* live_in,
                        uint32_t* live_out, uint32_t bound, uint32_t label, uint32_t* fr,
                        uint64_t* fa, uint32_t* cse, Acc* acc, Smem& s) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x; base < livec; base += stride) {
    const uint64_t i = base + threadIdx.x;
    uint32_t v = 0, d = 0;
    bool isF = false, isL = false;
    if (i < livec) {
      v = implicit ? uint32_t(i) : live_in[i];
      if (a.labels[v] == kUnset) {
        if (a.deg[v] <= bound) {
          isF = true;
          d = deg_full(a.offs, v);
        } else {
          isL = true;
        }
      }
    }
    uint32_t totL;
    uint32_t exL = block_excl_scan<uint32_t>(isL ? 1u : 0u, s.ws32, &totL);
    if (threadIdx.x == 0 && totL) s.baseL = atomicAdd(&acc->live, (unsigned long long)totL);
    __syncthreads();
    if (isL) live_out[s.baseL + exL] = v;
    emit_front_tile(isF, v, d, label, a, fr, fa, cse, acc, s);
  }
}

__global__ void __launch_bounds__(KC_THREADS, 1) k_coreness(KcArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const uint32_t nb = gridDim.x;
  const uint32_t lane = lane_id();
  const uint64_t gwarp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;

  uint32_t f = 0;       // frontier generation
  uint32_t lv = 0;      // live buffer holding the current live list
  uint32_t livec = a.n;
  bool implicit = true; // live list = 0..n-1 until the first compaction
  uint64_t bound = 0, label = 0, t = 1;
  uint64_t remaining = a.n;
  uint32_t kmax = 0, rounds = 0;
  uint32_t Fc = 0;
  uint64_t Ftot = 0;
  uint64_t guard = 0;

  for (;;) {
    if (++guard > 4ULL * a.n + 64) {
      if (blockIdx.x == 0 && threadIdx.x == 0) a.out[2] = 1;
      break;
    }
    if (Fc == 0) {
      if (remaining == 0) break;
      // ---- level advance: min alive degree over the live list
      Acc* acc = a.acc + (f % 3);
      const uint32_t* live_in = lv ? a.live1 : a.live0;
      uint32_t lmin = kUnset;
      for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < livec;
           i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t v = implicit ? uint32_t(i) : live_in[i];
        if (a.labels[v] == kUnset) lmin = min(lmin, a.deg[v]);
      }
      lmin = warp_min(lmin);
      if (lane == 0) s.ws32[threadIdx.x >> 5] = lmin;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t x = threadIdx.x < (blockDim.x >> 5) ? s.ws32[threadIdx.x] : kUnset;
        x = warp_min(x);
        if (threadIdx.x == 0 && x != kUnset) atomicMin(&acc->minv, x);
      }
      if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, acc); })) break;
      const uint64_t gmin = s.b_minv;
      if (gmin == kUnset) {  // remaining > 0 but nothing alive: inconsistent
        if (blockIdx.x == 0 && threadIdx.x == 0) a.out[2] = 2;
        break;
      }
      while (gmin > bound) {
        if (!a.approx) {
          bound = gmin;
          label = gmin;
        } else {  // core.cpp:105-110
          label = t;
          uint64_t ct = (t * a.c_num) / a.c_den + ((t * a.c_num) % a.c_den != 0);
          uint64_t nt = t + 1 > ct ? t + 1 : ct;
          bound = nt - 1;
          t = nt;
        }
      }
      uint32_t* fr = (f & 1) ? a.fr1 : a.fr0;
      uint64_t* fa = (f & 1) ? a.fa1 : a.fa0;
      uint32_t* cse = (f & 1) ? a.cse1 : a.cse0;
      collect(a, livec, implicit, live_in, lv ? a.live0 : a.live1, uint32_t(bound),
              uint32_t(label), fr, fa, cse, acc, s);
      if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, acc); })) break;
      const unsigned long long pk = s.b_front;
      Fc = uint32_t(pk >> 36);
      Ftot = pk & M36;
      livec = uint32_t(s.b_live);
      lv ^= 1;
      implicit = false;
      if (Fc == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.out[2] = 3;
        break;
      }
    }

    // ---- expand frontier f into frontier f+1
    ++rounds;
    if (label > kmax) kmax = uint32_t(label);
    remaining -= Fc;
    Acc* nacc = a.acc + ((f + 1) % 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      Acc* r = a.acc + ((f + 2) % 3);
      r->front = 0;
      r->live = 0;
      r->minv = kUnset;
      r->ovf = 0;
    }
    if (threadIdx.x == 0) s.cnt = 0;
    __syncthreads();
    {
      const uint32_t* F = (f & 1) ? a.fr1 : a.fr0;
      const uint64_t* FA = (f & 1) ? a.fa1 : a.fa0;
      const uint32_t* CS = (f & 1) ? a.cse1 : a.cse0;
      const uint32_t b32 = uint32_t(bound);
      const uint64_t nchunks = (Ftot + CH - 1) / CH;
      for (uint64_t c = gwarp; c < nchunks; c += nwarps) {
        const uint32_t e0 = CS[c];
        const uint32_t elast = (c + 1 < nchunks) ? CS[c + 1] : Fc - 1;
        const uint64_t a0 = c * CH;
        uint32_t us[CH / 32];
#pragma unroll
        for (int j = 0; j < int(CH / 32); ++j) {
          const uint64_t x = a0 + j * 32 + lane;
          us[j] = kUnset;
          if (x < Ftot) {
            uint32_t lo = e0, hi = elast;
            while (lo < hi) {  // largest e with FA[e] <= x
              uint32_t mid = (lo + hi + 1) >> 1;
              if (FA[mid] <= x)
                lo = mid;
              else
                hi = mid - 1;
            }
            const uint32_t v = F[lo];
            us[j] = a.adj[a.offs[v] + (x - FA[lo])];
          }
        }
#pragma unroll
        for (int j = 0; j < int(CH / 32); ++j) {
          const uint32_t u = us[j];
          if (u == kUnset) continue;
          if (a.deg[u] <= b32) continue;  // dead, or already at/below the bound
          const uint32_t old = atomicSub(&a.deg[u], 1u);
          if (old == b32 + 1) {  // crossed: joins the next round
            const uint32_t slot = atomicAdd(&s.cnt, 1u);
            if (slot < BUF) {
              s.id[slot] = u;
              s.dg[slot] = deg_full(a.offs, u);
            } else {
              nacc->ovf = 1;  // left unlabelled; the overflow collect finds it
            }
          }
        }
      }
    }
    __syncthreads();
    {
      const uint32_t cnt = min(s.cnt, BUF);
      uint32_t* fr = ((f + 1) & 1) ? a.fr1 : a.fr0;
      uint64_t* fa = ((f + 1) & 1) ? a.fa1 : a.fa0;
      uint32_t* cse = ((f + 1) & 1) ? a.cse1 : a.cse0;
      for (uint32_t b0 = 0; b0 < cnt; b0 += blockDim.x) {
        const uint32_t i = b0 + threadIdx.x;
        const bool ok = i < cnt;
        emit_front_tile(ok, ok ? s.id[i] : 0, ok ? s.dg[i] : 0, uint32_t(label), a, fr, fa, cse,
                        nacc, s);
      }
    }
    if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, nacc); })) break;
    ++f;
    if (s.b_ovf) {
      uint32_t* fr = (f & 1) ? a.fr1 : a.fr0;
      uint64_t* fa = (f & 1) ? a.fa1 : a.fa0;
      uint32_t* cse = (f & 1) ? a.cse1 : a.cse0;
      collect(a, livec, implicit, lv ? a.live1 : a.live0, lv ? a.live0 : a.live1, uint32_t(bound),
              uint32_t(label), fr, fa, cse, nacc, s);
      if (!grid_sync(a.bar, nb, &s.abort, [&] { fetch_acc(s, nacc); })) break;
      livec = uint32_t(s.b_live);
      lv ^= 1;
      implicit = false;
    }
    const unsigned long long pk = s.b_front;
    Fc = uint32_t(pk >> 36);
    Ftot = pk & M36;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out[0] = kmax;
    a.out[1] = rounds;
    if (ld_relaxed_u32(&a.bar->abort)) a.out[2] = 4;
  }
}

__global__ void k_init_deg(const uint64_t* offs, uint64_t n, uint32_t* deg, uint32_t* labels) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    deg[i] = uint32_t(offs[i + 1] - offs[i]);
    labels[i] = kUnset;
  }
}

__global__ void k_init_acc(Acc* acc, GridBarrier* bar) {
  if (threadIdx.x < 3) {
    acc[threadIdx.x].front = 0;
    acc[threadIdx.x].live = 0;
    acc[threadIdx.x].minv = kUnset;
    acc[threadIdx.x].ovf = 0;
  }
  if (threadIdx.x == 0) *bar = GridBarrier{0, 0, 0, 0};
}

}  // namespace

CoreOut coreness(const dg_graph& g, bool approx, uint64_t c_num, uint64_t c_den,
                 uint32_t* d_labels) {
  if (g.n == 0) throw DgError(DG_E_EMPTY, "coreness of empty graph");
  if (approx && (c_den == 0 || c_num <= c_den))
    throw DgError(DG_E_PARAM, "approximation factor must be > 1");
  if (g.n >= (1ULL << 28) || 2 * g.m >= (1ULL << 36))
    throw DgError(DG_E_PARAM, "graph too large for the single-GPU coreness kernel");
  const uint64_t n = g.n;
  DevBuf<uint32_t> deg(n), live0(n), live1(n), fr0(n), fr1(n);
  DevBuf<uint64_t> fa0(n), fa1(n);
  const uint64_t nch = (2 * g.m) / CH + 2;
  DevBuf<uint32_t> cse0(nch), cse1(nch);
  DevBuf<Acc> acc(3);
  DevBuf<GridBarrier> bar(1);
  DevBuf<uint32_t> out(3);
  out.zero();
  k_init_deg<<<grid_for(n, 256), 256, 0, stream()>>>(g.offs.get(), n, deg.get(), d_labels);
  DG_CHECK_LAUNCH();
  k_init_acc<<<1, 32, 0, stream()>>>(acc.get(), bar.get());
  DG_CHECK_LAUNCH();

  const size_t smem = sizeof(Smem);
  static bool attr_set = false;
  if (!attr_set) {
    DG_CUDA(cudaFuncSetAttribute(k_coreness, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    attr_set = true;
  }
  int occ = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coreness, KC_THREADS, smem));
  if (occ < 1) throw DgError(DG_E_CUDA, "coreness kernel does not fit on an SM");
  const unsigned blocks = unsigned(num_sms()) * unsigned(occ > 1 ? 1 : occ);

  KcArgs args{g.offs.get(), g.adj.get(), uint32_t(n), deg.get(), d_labels, live0.get(),
              live1.get(), fr0.get(), fr1.get(), fa0.get(), fa1.get(), cse0.get(), cse1.get(),
              acc.get(), bar.get(), out.get(), approx ? 1 : 0, c_num, c_den};
  void* params[] = {&args};
  cudaEvent_t e0, e1;
  DG_CUDA(cudaEventCreate(&e0));
  DG_CUDA(cudaEventCreate(&e1));
  DG_CUDA(cudaEventRecord(e0, stream()));
  DG_CUDA(cudaLaunchCooperativeKernel((void*)k_coreness, dim3(blocks), dim3(KC_THREADS), params,
                                      smem, stream()));
  DG_CUDA(cudaEventRecord(e1, stream()));
  uint32_t h[3];
  d2h(h, out.get(), 3);
  stream_sync();
  CoreOut r;
  DG_CUDA(cudaEventElapsedTime(&r.kernel_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (h[2]) {
    char buf[128];
    snprintf(buf, sizeof buf, "coreness kernel failed internal check (code %u)", h[2]);
    throw DgError(DG_E_INVARIANT, buf);
  }
  r.kmax = h[0];
  r.rounds = h[1];
  return r;
}

}  // namespace dgb
