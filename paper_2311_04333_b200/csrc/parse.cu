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
// B200 mapping (byte work, HBM-bound): the text is cut into 256-byte windows,
// one thread per window parses every line that STARTS in its window (reading
// past the window end if the line does).  Pass 1 counts pairs per window and
// takes the minimum byte offset of a bad line start (atomicMin); a CUB scan
// gives each window its output offset; pass 2 writes the pairs.  A bad line's
// number is the count of '\n' before its start (one more pass over a prefix).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace dgb {
namespace {

constexpr uint32_t PW = 256;  // window bytes per thread

__device__ __forceinline__ bool blank(uint8_t c) { return c == ' ' || c == '\t'; }

// One forward scan per line from its first byte p: returns the start of the
// next line in *next and 0: skip, 1: pair (a, b), 2: malformed.  A '\r' ends
// the line only when '\n' or the end of the text follows (the reference drops
// ONE trailing '\r' before tokenising); anywhere else it is a token byte.
// u64 overflow (from_chars out_of_range) is two comparisons, no division.
__device__ __forceinline__ int parse_line(const uint8_t* __restrict__ t, uint64_t len, uint64_t p,
                                          uint8_t comment, uint64_t& a, uint64_t& b,
                                          uint64_t* next) {
  constexpr uint64_t kCut = 0xffffffffffffffffULL / 10;  // 1844674407370955161
  uint64_t q = p;
  auto at_eol = [&](uint64_t i) {  // line end at i (excluding a trailing CR)
    if (i >= len) return true;
    const uint8_t c = __ldg(t + i);
    return c == '\n' || (c == '\r' && (i + 1 >= len || __ldg(t + i + 1) == '\n'));
  };
  auto skip_line = [&](uint64_t i) {
    while (i < len && __ldg(t + i) != '\n') ++i;
    *next = i + 1;
  };
  while (!at_eol(q) && blank(__ldg(t + q))) ++q;
  if (at_eol(q)) {
    skip_line(q);
    return 0;
  }
  if (__ldg(t + q) == comment) {
    skip_line(q);
    return 0;
  }
  uint64_t id[2] = {0, 0};
  int tok = 0;
  while (!at_eol(q)) {
    if (tok == 2) {  // a third token
      skip_line(q);
      return 2;
    }
    uint64_t x = 0;
    while (!at_eol(q)) {
      const uint8_t c = __ldg(t + q);
      if (blank(c)) break;
      const uint32_t d = uint32_t(c) - '0';
      if (d > 9 || x > kCut || (x == kCut && d > 5)) {
        skip_line(q);
        return 2;
      }
      x = x * 10 + d;
      ++q;
    }
    id[tok++] = x;
    while (!at_eol(q) && blank(__ldg(t + q))) ++q;
  }
  skip_line(q);
  if (tok != 2) return 2;
  if (id[0] == id[1]) return 0;  // self-loop
  a = id[0];
  b = id[1];
  return 1;
}

template <bool WRITE>
__global__ void k_parse(const uint8_t* __restrict__ t, uint64_t len, uint8_t comment,
                        uint64_t* cnt, const uint64_t* off, uint64_t* pu, uint64_t* pv,
                        unsigned long long* bad) {
  const uint64_t nwin = (len + PW - 1) / PW;
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < nwin;
       w += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t w0 = w * PW, w1 = min(w0 + PW, len);
    uint64_t p = w0;
    if (p > 0 && __ldg(t + p - 1) != '\n') {  // the line in progress belongs to an earlier window
      while (p < w1 && __ldg(t + p) != '\n') ++p;
      ++p;
    }
    uint64_t c = 0, o = WRITE ? off[w] : 0;
    while (p < w1) {
      uint64_t a, b, nx;
      const int k = parse_line(t, len, p, comment, a, b, &nx);
      if (k == 1) {
        if (WRITE) {
          pu[o + c] = a;
          pv[o + c] = b;
        }
        ++c;
      } else if (k == 2 && !WRITE) {
        atomicMin(bad, (unsigned long long)p);
      }
      p = nx;
    }
    if (!WRITE) cnt[w] = c;
  }
}

// number of '\n' bytes in [0, lim)
__global__ void k_count_newlines(const uint8_t* __restrict__ t, uint64_t lim,
                                 unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < lim;
       i += uint64_t(gridDim.x) * blockDim.x)
    c += t[i] == '\n';
  c = __reduce_add_sync(~0u, uint32_t(c));
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

}  // namespace

GraphPtr parse_edge_list(const uint8_t* d_text, uint64_t len, uint8_t comment,
                         uint64_t* bad_line) {
  *bad_line = 0;
  const uint64_t nwin = (len + PW - 1) / PW;
  if (nwin == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  DevBuf<uint64_t> cnt(nwin), off(nwin);
  DevBuf<unsigned long long> bad(2);
  const unsigned long long init[2] = {~0ULL, 0ULL};
  h2d(bad.get(), init, 2);
  const unsigned grid = grid_for(nwin, 256);
  k_parse<false><<<grid, 256, 0, stream()>>>(d_text, len, comment, cnt.get(), nullptr, nullptr,
                                              nullptr, bad.get());
  DG_CHECK_LAUNCH();
  unsigned long long b0 = 0;
  d2h(&b0, bad.get(), 1);
  stream_sync();
  if (b0 != ~0ULL) {  // the first malformed line: its number
    if (b0) {
      k_count_newlines<<<grid_for(b0, 256), 256, 0, stream()>>>(d_text, b0, bad.get() + 1);
      DG_CHECK_LAUNCH();
    }
    unsigned long long nl = 0;
    d2h(&nl, bad.get() + 1, 1);
    stream_sync();
    *bad_line = nl + 1;
    throw DgError(DG_E_PARSE, "expected two non-negative integers");
  }
  size_t tmp = 0;
  DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt.get(), off.get(), nwin, stream()));
  DevBuf<unsigned char> scratch(tmp);
  DG_CUDA(cub::DeviceScan::ExclusiveSum(scratch.get(), tmp, cnt.get(), off.get(), nwin, stream()));
  uint64_t last[2];
  d2h(&last[0], off.get() + nwin - 1, 1);
  d2h(&last[1], cnt.get() + nwin - 1, 1);
  stream_sync();
  const uint64_t k = last[0] + last[1];
  if (k == 0) throw DgError(DG_E_EMPTY, "no edges after removing self-loops and duplicates");
  DevBuf<uint64_t> pu(k), pv(k);
  k_parse<true><<<grid, 256, 0, stream()>>>(d_text, len, comment, nullptr, off.get(), pu.get(),
                                             pv.get(), nullptr);
  DG_CHECK_LAUNCH();
  return build_from_pairs(pu.get(), pv.get(), k);
}

}  // namespace dgb
