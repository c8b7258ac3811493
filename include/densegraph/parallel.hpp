// parallel.hpp -- host-side helpers kept for API parity with the reference
// (proj/include/densegraph/parallel.hpp).  Parallelism lives on the B200;
// the OpenMP thread count has no effect on the device path, so
// set_threads / max_threads only record the request.
#pragma once

#include <cstdint>

#include "densegraph/density.hpp"

namespace densegraph {

namespace detail {
inline int& thread_request() {
  static int t = 0;
  return t;
}
}  // namespace detail

inline int max_threads() { return detail::thread_request() > 0 ? detail::thread_request() : 1; }
inline void set_threads(int t) { detail::thread_request() = t > 0 ? t : 0; }

// splitmix64 (the reference's seeded sampling stream)
inline u64 mix64(u64 x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace densegraph
