// parse.cu -- SNAP-style edge-list text -> canonical pairs on the device
// (reference io.cpp:25-60 parse_edge_list tokenisation; the CSR build that
// follows is graph.cu's build_from_pairs, io.cpp:62-92).
//
// Rules reproduced byte for byte: lines end at '\n' (the last one may not);
// one trailing '\r' is dropped; leading spaces / tabs are skipped; an empty
// line or one whose first other byte is the comment character is skipped;
// tokens are maximal runs of bytes other than ' ' and '\t' and must each be a
// complete std::from_chars u64 (decimal digits, no sign, no overflow); exactly
// two tokens, else ParseError at the FIRST such line; self-loops are dropped
// after validation.
//
// B200 mapping (byte work, HBM-bound; one pass over the text): a CTA takes
// 8 KB tiles of the 16-byte-aligned address space (grid-stride over a
// persistent grid) and stages tile + 256-byte halo into shared memory with
// coalesced 16-byte loads, the next tile's loads in flight (registers) while
// the current one is parsed.  Each of its 256 threads owns a 32-byte window
// and classifies it with exact SWAR byte compares into bit masks (newline,
// blank, digit), published in shared memory; a line that starts in the
// window and ends within the next window is parsed from the masks (token
// count and digits-only by bit arithmetic, the trailing-CR rule by one byte
// check, values by SWAR 8-digit conversion); longer lines and tokens of 17+
// digits take a byte state machine (shared memory, then global memory past
// the halo).  Pairs go to per-thread slots in shared memory (<= 8 per window:
// an emitting line takes >= 4 bytes) and, after a CTA scan, to global memory
// at an offset taken by ONE atomicAdd per tile -- the CSR build sorts, so the
// order of pairs between tiles does not matter.  Capacity: one pair per line
// (a vectorised newline count).  The first malformed line is the minimum
// byte offset of a bad line start (atomicMin); its number is the count of
// '\n' before it.
#include "internal.cuh"

namespace dgb {
namespace {

#ifndef DG_PARSE_MINB
#define DG_PARSE_MINB 4  // resident CTAs per SM the register budget is cut for
#endif

constexpr uint32_t kThreads = 256, kWin = 32, kTile = kThreads * kWin;  // 8 KB tiles
constexpr uint32_t kHalo = 256, kSpan = 16 + kTile + kHalo;               // staged bytes
constexpr uint32_t kSlots = kWin / 4;  // pairs per window (an emitting line takes >= 4 bytes)

// Per-line state of the byte machine (io.cpp:25-60 rules, see the header).
struct Line {
  uint64_t start, x, id0, id1;
  uint32_t ntok;
  bool active, intok, skip, err;
};

__device__ __forceinline__ void line_begin(Line& L, uint64_t i) {
  L.start = i;
  L.x = L.id0 = L.id1 = 0;
  L.ntok = 0;
  L.active = true;
  L.intok = L.skip = L.err = false;
}

// one byte c at position i of an active line; next = the byte after it (only
// read for a '\r'); returns true when the line ended at this byte
__device__ __forceinline__ bool line_byte(Line& L, uint8_t c, uint64_t i, uint64_t len,
                                          uint8_t next, uint8_t comment) {
  constexpr uint64_t kCut = 0xffffffffffffffffULL / 10;  // 1844674407370955161
  if (c == '\n') return true;
  // a CR ends the line only before LF / the end of the text (one trailing CR
  // is dropped); elsewhere it is a token byte
  if (c == '\r' && (i + 1 >= len || next == '\n')) return false;
  if (L.skip) return false;
  if (c == ' ' || c == '\t') {
    L.intok = false;
    return false;
  }
  if (!L.intok) {  // a token starts
    if (L.ntok == 0 && c == comment) {
      L.skip = true;
      return false;
    }
    L.intok = true;
    ++L.ntok;
    L.x = 0;
    if (L.ntok > 2) L.err = true;
  }
  const uint32_t d = uint32_t(c) - '0';
  if (d > 9 || L.x > kCut || (L.x == kCut && d > 5)) L.err = true;
  L.x = L.x * 10 + d;
  if (L.ntok == 1) L.id0 = L.x;
  if (L.ntok == 2) L.id1 = L.x;
  return false;
}

// 0xFF/0x00 per byte -> 4-bit mask (bits 7, 15, 23, 31 gathered to 28..31)
__device__ __forceinline__ uint32_t bytemask4(uint32_t v) {
  return ((v & 0x80808080u) * 0x00204081u) >> 28;
}

// Character classes of a 32-byte window as bit masks (bit k = byte k).
struct Classes {
  uint32_t nl, bl, dg;
};

// bit 7 of each byte set where the byte equals the byte of c (exact SWAR:
// no carries between bytes)
__device__ __forceinline__ uint32_t eq_bytes(uint32_t v, uint32_t c) {
  const uint32_t x = v ^ c;
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}

__device__ __forceinline__ Classes classify(const uint4& qa, const uint4& qb) {
  const uint32_t w[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
  Classes c{0, 0, 0};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t v = w[j];
    const uint32_t lo = v & 0x7f7f7f7fu;
    // '0' <= b <= '9': b + 0x50 carries into bit 7 and b + 0x46 does not
    const uint32_t dg = (lo + 0x50505050u) & ~(lo + 0x46464646u) & ~v & 0x80808080u;
    c.nl |= bytemask4(eq_bytes(v, 0x0a0a0a0au)) << (4 * j);
    c.bl |= bytemask4(eq_bytes(v, 0x20202020u) | eq_bytes(v, 0x09090909u)) << (4 * j);
    c.dg |= bytemask4(dg) << (4 * j);
  }
  return c;
}

// value of the decimal token of la <= 16 digits ending at byte `end` of the
// span (bytes before the token read as '0'): SWAR 8-digit conversion of one
// or two 8-byte words gathered from aligned 8-byte shared loads
__device__ __forceinline__ uint64_t swar8(uint64_t v) {  // 8 ASCII digits, first at byte 0
  v -= 0x3030303030303030ULL;
  v = (v * 10) + (v >> 8);  // pairs
  v = (((v & 0x000000FF000000FFULL) * (100 + (1000000ULL << 32))) +
       (((v >> 16) & 0x000000FF000000FFULL) * (1 + (10000ULL << 32)))) >> 32;
  return v;
}

__device__ __forceinline__ uint64_t load8(const uint8_t* sm, uint32_t pos) {  // bytes [pos, pos+8)
  const uint64_t* q = reinterpret_cast<const uint64_t*>(sm);
  const uint32_t k = pos >> 3, sh = 8 * (pos & 7);
  const uint64_t lo = q[k];
  if (sh == 0) return lo;
  return (lo >> sh) | (q[k + 1] << (64 - sh));
}

__device__ __forceinline__ uint64_t token_value(const uint8_t* sm, uint32_t end, int la) {
  // the last min(la, 8) digits
  const int l0 = la < 8 ? la : 8;
  uint64_t w = load8(sm, end - 8);
  const uint64_t keep = ~0ULL << (8 * (8 - l0));
  uint64_t x = swar8((w & keep) | (0x3030303030303030ULL & ~keep));
  if (la > 8) {  // the leading la - 8 digits
    const int l1 = la - 8;
    uint64_t w1 = load8(sm, end - 16);
    const uint64_t k1 = ~0ULL << (8 * (8 - l1));
    x += swar8((w1 & k1) | (0x3030303030303030ULL & ~k1)) * 100000000ULL;
  }
  return x;
}

// positions outside [0, len) read as newlines (virtual line ends before the
// text and at its end) and nothing else
__device__ __forceinline__ void clip(Classes& c, int64_t i0, uint64_t len) {
  uint32_t inv = 0;
  if (i0 < 0) inv |= i0 <= -32 ? ~0u : ((1u << uint32_t(-i0)) - 1);
  const int64_t hi = int64_t(len) - i0;  // first invalid bit
  if (hi < 32) inv |= hi <= 0 ? ~0u : ~((1u << uint32_t(hi)) - 1);
  c.nl |= inv;
  c.bl &= ~inv;
  c.dg &= ~inv;
}

__global__ void __launch_bounds__(kThreads, DG_PARSE_MINB) k_parse_tiles(const uint8_t* __restrict__ t,
                                                          uint64_t len, uint8_t comment,
                                                          uint64_t* __restrict__ pu,
                                                          uint64_t* __restrict__ pv,
                                                          unsigned long long* cnt,
                                                          unsigned long long* bad) {
  __shared__ __align__(16) uint8_t sm[kSpan];
  __shared__ uint64_t su[kThreads * kSlots], sv[kThreads * kSlots];
  __shared__ uint32_t cls[3][kThreads + 1];  // window classes (+ the first halo window)
  __shared__ uint32_t wsum[kThreads / 32];
  __shared__ unsigned long long tbase;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // positions are taken relative to the 16-byte-aligned address below the
  // text: rel = i + mis, so every window and staged chunk is aligned
  const uintptr_t tb = reinterpret_cast<uintptr_t>(t);
  const uint32_t mis = uint32_t(tb & 15);
  const uint8_t* abase = t - mis;
  const uint64_t relend = len + mis;
  const uint64_t ntiles = (relend + kTile - 1) / kTile;
  uint4* sm16 = reinterpret_cast<uint4*>(sm);
  uint64_t* myu = su + tid * kSlots;
  uint64_t* myv = sv + tid * kSlots;
  // the next tile's chunks are loaded into registers while this one is parsed
  constexpr uint32_t kChunks = kSpan / 16, kPer = (kChunks + kThreads - 1) / kThreads;
  uint4 pre[kPer];
  auto fetch = [&](uint64_t tile) {
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j) {
      const uint32_t ch = tid + j * kThreads;
      const int64_t rel = int64_t(tile * kTile) - 16 + 16 * int64_t(ch);
      if (ch < kChunks && tile < ntiles && rel >= 0 && uint64_t(rel) < relend)
        pre[j] = __ldg(reinterpret_cast<const uint4*>(abase + rel));
    }
  };
  fetch(blockIdx.x);
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t r0 = tile * kTile;  // sm[k] holds rel r0 - 16 + k
#pragma unroll
    for (uint32_t j = 0; j < kPer; ++j)
      if (tid + j * kThreads < kChunks) sm16[tid + j * kThreads] = pre[j];
    __syncthreads();
    fetch(tile + gridDim.x);
    auto at = [&](uint64_t i) -> uint8_t {  // text byte i (i < len)
      const uint64_t k = i + mis + 16 - r0;
      return k < kSpan ? sm[k] : __ldg(t + i);
    };
    const int64_t i0 = int64_t(r0 + uint64_t(tid) * kWin) - int64_t(mis);  // window start
    {
      Classes c = classify(sm16[1 + 2 * tid], sm16[2 + 2 * tid]);
      clip(c, i0, len);
      cls[0][tid] = c.nl, cls[1][tid] = c.bl, cls[2][tid] = c.dg;
      if (tid == 0) {  // the first halo window
        Classes h = classify(sm16[1 + 2 * kThreads], sm16[2 + 2 * kThreads]);
        clip(h, i0 + int64_t(kTile), len);
        cls[0][kThreads] = h.nl, cls[1][kThreads] = h.bl, cls[2][kThreads] = h.dg;
      }
    }
    __syncthreads();
    const uint64_t NL = cls[0][tid] | uint64_t(cls[0][tid + 1]) << 32;
    const uint64_t BL = cls[1][tid] | uint64_t(cls[1][tid + 1]) << 32;
    const uint64_t DG = cls[2][tid] | uint64_t(cls[2][tid + 1]) << 32;
    // newline before the window: the previous window's top bit, or the byte
    // before the tile (virtual newline before the text)
    bool prev_nl;
    if (tid > 0) {
      prev_nl = cls[0][tid - 1] >> 31;
    } else {
      prev_nl = i0 <= 0 || sm[15] == '\n';
    }
    // lines that start in this window: valid position after a newline
    uint32_t valid = ~0u;
    if (i0 < 0) valid &= i0 <= -32 ? 0u : ~((1u << uint32_t(-i0)) - 1);
    if (int64_t(len) - i0 < 32)
      valid &= int64_t(len) - i0 <= 0 ? 0u : ((1u << uint32_t(int64_t(len) - i0)) - 1);
    uint32_t starts = valid & ((uint32_t(NL) << 1) | uint32_t(prev_nl));
    const uint8_t* wb = sm + 16 + kWin * tid;  // byte k of the 64-byte span
    uint32_t c = 0;
    while (starts) {
      const int s = __ffs(starts) - 1;
      starts &= starts - 1;
      const uint64_t ls = uint64_t(i0 + s);
      // ---- fast path: the line ends inside the 64-byte span
      const uint64_t after = NL >> s;
      int kind = -1;  // -1 slow path, 0 skip, 1 pair, 2 malformed
      uint64_t a = 0, b = 0;
      if (after) {
        int e = s + __ffsll(after) - 1;
        if (e > s && wb[e - 1] == '\r') --e;  // one trailing CR
        const uint64_t lm = ((1ull << e) - 1) & ~((1ull << s) - 1);
        const uint64_t nb = lm & ~BL;
        if (!nb) {
          kind = 0;
        } else {
          const int f = __ffsll(nb) - 1;
          if (wb[f] == comment) {
            kind = 0;
          } else {
            const uint64_t st = nb & ~(nb << 1);
            if ((nb & ~DG) || __popcll(st) != 2) {
              kind = 2;
            } else {
              const int b0 = __ffsll(st & (st - 1)) - 1;
              const int la = __ffsll(~(nb >> f)) - 1, lb = __ffsll(~(nb >> b0)) - 1;
              if (la <= 16 && lb <= 16) {  // 16 digits cannot overflow u64
                const uint32_t wo = 16 + kWin * tid;  // span byte 0 in sm
                a = token_value(sm, wo + f + la, la);
                b = token_value(sm, wo + b0 + lb, lb);
                kind = a != b;  // self-loops dropped after validation
              }
            }
          }
        }
      }
      // ---- slow path: byte machine (long lines, 20-digit tokens)
      if (kind < 0) {
        Line L;
        line_begin(L, ls);
        for (uint64_t i = ls;; ++i) {
          if (i >= len) break;
          const uint8_t ch = at(i);
          const uint8_t nx = (ch == '\r' && i + 1 < len) ? at(i + 1) : 0;
          if (line_byte(L, ch, i, len, nx, comment)) break;
        }
        if (L.skip || L.ntok == 0) {
          kind = 0;
        } else if (L.err || L.ntok != 2) {
          kind = 2;
        } else {
          a = L.id0, b = L.id1;
          kind = a != b;
        }
      }
      if (kind == 2) atomicMin(bad, (unsigned long long)ls);
      if (kind == 1) {
        myu[c] = a;
        myv[c] = b;
        ++c;
      }
    }
    // CTA exclusive scan of the pair counts, one atomicAdd per tile
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(~0u, incl, o);
      if (lane >= uint32_t(o)) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (uint32_t x = 0; x < kThreads / 32; ++x) {
      const uint32_t y = wsum[x];
      wpre += x < warp ? y : 0;
      total += y;
    }
    if (tid == 0 && total) tbase = atomicAdd(cnt, (unsigned long long)total);
    __syncthreads();
    const unsigned long long base = tbase + wpre + incl - c;
    for (uint32_t j = 0; j < c; ++j) {
      pu[base + j] = myu[j];
      pv[base + j] = myv[j];
    }
    __syncthreads();  // sm / cls / wsum / tbase reused by the next tile
  }
}

// number of '\n' bytes in [0, lim): 16-byte loads, four byte compares per
// instruction (__vcmpeq4); unaligned head and tail bytewise
__global__ void k_count_newlines(const uint8_t* __restrict__ t, uint64_t lim,
                                 unsigned long long* out) {
  const uint64_t mis = (16 - (reinterpret_cast<uintptr_t>(t) & 15)) & 15;
  const uint64_t head = mis < lim ? mis : lim;
  const uint64_t nch = (lim - head) / 16, tail0 = head + 16 * nch;
  const uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t c = 0;
  if (g < head) c += t[g] == '\n';
  if (g < lim - tail0) c += t[tail0 + g] == '\n';
  const uint4* v = reinterpret_cast<const uint4*>(t + head);
  for (uint64_t k = g; k < nch; k += stride) {
    const uint4 x = __ldg(v + k);
    c += (__popc(__vcmpeq4(x.x, 0x0a0a0a0au)) + __popc(__vcmpeq4(x.y, 0x0a0a0a0au)) +
          __popc(__vcmpeq4(x.z, 0x0a0a0a0au)) + __popc(__vcmpeq4(x.w, 0x0a0a0a0au))) >> 3;
  }
  c = __reduce_add_sync(~0u, c);
  if (lane_id() == 0 && c) atomicAdd(out, (unsigned long long)c);
}

}  // namespace

GraphPtr parse_edge_list(const uint8_t* d_text, uint64_t len, uint8_t comment,
                         uint64_t* bad_line) {
  *bad_line = 0;
  if (len == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  // counters: [0] newlines of the text, [1] pairs written, [2] bad offset, [3] newlines before it
  DevBuf<unsigned long long> ctr(4);
  const unsigned long long init[4] = {0ULL, 0ULL, ~0ULL, 0ULL};
  h2d(ctr.get(), init, 4);
  k_count_newlines<<<num_sms() * 8, 256, 0, stream()>>>(d_text, len, ctr.get());
  DG_CHECK_LAUNCH();
  unsigned long long lines = 0;
  d2h(&lines, ctr.get(), 1);
  stream_sync();
  const uint64_t cap = lines + 1;  // at most one pair per line
  DevBuf<uint64_t> pu(cap), pv(cap);
  const uint64_t ntiles = (len + 15 + kTile - 1) / kTile;
  int per_sm = 0;
  DG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_parse_tiles, kThreads, 0));
  const unsigned grid =
      unsigned(std::min<uint64_t>(ntiles, uint64_t(num_sms()) * uint64_t(std::max(per_sm, 1))));
  k_parse_tiles<<<grid, kThreads, 0, stream()>>>(d_text, len, comment, pu.get(), pv.get(),
                                                 ctr.get() + 1, ctr.get() + 2);
  DG_CHECK_LAUNCH();
  unsigned long long h[2];
  d2h(h, ctr.get() + 1, 2);
  stream_sync();
  if (h[1] != ~0ULL) {  // the first malformed line: its number
    if (h[1]) {
      k_count_newlines<<<num_sms() * 8, 256, 0, stream()>>>(d_text, h[1], ctr.get() + 3);
      DG_CHECK_LAUNCH();
    }
    unsigned long long nl = 0;
    d2h(&nl, ctr.get() + 3, 1);
    stream_sync();
    *bad_line = nl + 1;
    throw DgError(DG_E_PARSE, "expected two non-negative integers");
  }
  const uint64_t k = h[0];
  if (k == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  return build_from_pairs(pu.get(), pv.get(), k);
}

}  // namespace dgb
