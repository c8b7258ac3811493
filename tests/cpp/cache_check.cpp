// DGRC0001 cache checks for include/densegraph/io.hpp (host-only code paths;
// runs without a GPU).  Usage:
//   cache_check roundtrip <in.dgrc> <out.dgrc>   read, print "n m source_hash", write back
//   cache_check hash <file>                      print hash_file(file)
//   cache_check is <file>                        print is_cache_file(file)
//   cache_check fnv <string>                     print fnv1a64 of its bytes
// Exit codes follow the reference CLI mapping (densest.cpp:305-329):
// Io 3, Invariant 4, CacheHash 6.
#include <cstdio>
#include <string>

#include "densegraph/io.hpp"

int main(int argc, char** argv) {
  using namespace densegraph;
  if (argc < 3) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "roundtrip" && argc == 4) {
      u64 src = 0;
      Graph g = read_cache(argv[2], &src);
      std::printf("%llu %llu %llu\n", (unsigned long long)g.n, (unsigned long long)g.m,
                  (unsigned long long)src);
      write_cache(g, argv[3], src);
      return 0;
    }
    if (mode == "hash") {
      std::printf("%llu\n", (unsigned long long)hash_file(argv[2]));
      return 0;
    }
    if (mode == "fnv") {  // fnv1a64 of the argument's bytes
      const std::string x = argv[2];
      std::printf("%llu\n", (unsigned long long)fnv1a64(x.data(), x.size()));
      return 0;
    }
    if (mode == "is") {
      std::printf("%d\n", int(is_cache_file(argv[2])));
      return 0;
    }
  } catch (const CacheHashError& e) {
    std::printf("CacheHashError: %s\n", e.what());
    return 6;
  } catch (const IoError& e) {
    std::printf("IoError: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 4;
  }
  return 2;
}
