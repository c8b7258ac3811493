// io.hpp -- drop-in ingest API (reference proj/include/densegraph/io.hpp:10-31).
// Text tokenising and the binary cache are host I/O plumbing; the CSR build
// (sort / dedup / relabel / fill, io.cpp:51-92) runs on the device through
// dg_graph_build.  Cache layout "DGRC0001": magic, n, m, source hash,
// payload FNV-1a hash, then little-endian orig u64[n], offs u64[n+1],
// adj u32[2m] -- byte-compatible with the reference's cache files.
#pragma once

#include <bit>
#include <charconv>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <string>
#include <vector>

#include "densegraph/graph.hpp"

namespace densegraph {

static_assert(std::endian::native == std::endian::little, "cache I/O assumes a little-endian host");

struct ParseOptions {
  char comment = '#';
};

// Tokenised on the device (dg_parse_edge_list, csrc/parse.cu) with the
// reference's rules; the message of a ParseError carries the line's text.
inline Graph parse_edge_list(std::istream& in, const ParseOptions& opts = {}) {
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad()) throw IoError("read failure while parsing edge list");
  dg_graph* h = nullptr;
  uint64_t bad = 0;
  const dg_status st =
      dg_parse_edge_list(text.data(), text.size(), opts.comment, 0, &h, &bad);
  if (st == DG_E_PARSE && bad) {
    std::size_t b = 0;
    for (uint64_t l = 1; l < bad; ++l) b = text.find('\n', b) + 1;
    std::size_t e = text.find('\n', b);
    std::string line = text.substr(b, e == std::string::npos ? std::string::npos : e - b);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    throw ParseError(std::size_t(bad), "expected two non-negative integers, got \"" + line + "\"");
  }
  detail::check(st);
  return Graph::from_device(h);
}

inline Graph parse_edge_list_file(const std::string& path, const ParseOptions& opts = {}) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  return parse_edge_list(in, opts);
}

inline void write_edge_list(const Graph& g, std::ostream& out) {
  for (u64 v = 0; v < g.n; ++v)
    for (u32 u : g.neighbors(u32(v)))
      if (u > v) out << g.orig[v] << ' ' << g.orig[u] << '\n';
}

inline u64 fnv1a64(const void* data, std::size_t size, u64 seed = 14695981039346656037ULL) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < size; ++i) seed = (seed ^ p[i]) * 1099511628211ULL;
  return seed;
}

inline u64 hash_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  std::vector<char> buf(1 << 16);
  u64 h = 14695981039346656037ULL;
  while (in) {
    in.read(buf.data(), std::streamsize(buf.size()));
    h = fnv1a64(buf.data(), std::size_t(in.gcount()), h);
  }
  if (in.bad()) throw IoError("read failure on " + path);
  return h;
}

namespace detail {
inline constexpr char kCacheMagic[8] = {'D', 'G', 'R', 'C', '0', '0', '0', '1'};
inline u64 payload_hash(const Graph& g) {
  u64 h = fnv1a64(g.orig.data(), g.orig.size() * 8);
  h = fnv1a64(g.offs.data(), g.offs.size() * 8, h);
  return fnv1a64(g.adj.data(), g.adj.size() * 4, h);
}
template <class T>
void read_exact(std::istream& in, T* p, std::size_t count) {
  in.read(reinterpret_cast<char*>(p), std::streamsize(count * sizeof(T)));
  if (std::size_t(in.gcount()) != count * sizeof(T)) throw IoError("truncated cache file");
}
}  // namespace detail

inline bool is_cache_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  char m[8];
  return in && in.read(m, 8) && std::memcmp(m, detail::kCacheMagic, 8) == 0;
}

inline void write_cache(const Graph& g, const std::string& path, u64 source_hash) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path + " for writing");
  const u64 head[4] = {g.n, g.m, source_hash, detail::payload_hash(g)};
  out.write(detail::kCacheMagic, 8);
  out.write(reinterpret_cast<const char*>(head), sizeof head);
  out.write(reinterpret_cast<const char*>(g.orig.data()), std::streamsize(g.orig.size() * 8));
  out.write(reinterpret_cast<const char*>(g.offs.data()), std::streamsize(g.offs.size() * 8));
  out.write(reinterpret_cast<const char*>(g.adj.data()), std::streamsize(g.adj.size() * 4));
  if (!out) throw IoError("write failure on " + path);
}

inline Graph read_cache(const std::string& path, u64* source_hash = nullptr) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path);
  char m[8];
  in.read(m, 8);
  if (in.gcount() != 8 || std::memcmp(m, detail::kCacheMagic, 8) != 0)
    throw IoError(path + " is not a graph cache file");
  u64 head[4];
  detail::read_exact(in, head, 4);
  Graph g;
  g.n = head[0];
  g.m = head[1];
  g.orig.resize(g.n);
  g.offs.resize(g.n + 1);
  g.adj.resize(2 * g.m);
  detail::read_exact(in, g.orig.data(), g.n);
  detail::read_exact(in, g.offs.data(), g.n + 1);
  detail::read_exact(in, g.adj.data(), 2 * g.m);
  if (detail::payload_hash(g) != head[3]) throw CacheHashError(path + ": cache payload corrupt");
  if (source_hash) *source_hash = head[2];
  return g;
}

}  // namespace densegraph
