// shard.cuh -- a GPU's shard of the 1D vertex-range partition (shard.cu) and
// the peer-visible state block the other shards decrement into.
#pragma once

#include <vector>

#include "internal.cuh"

// Cross-shard control block: one per shard block; every shard uses shard 0's
// (mapped into every process: NVLink peer memory, or this GPU for shards of
// one process).  A flip barrier word and rotating reduction slots.
struct alignas(128) XCtrl {
  uint32_t arrive;               // flip barrier of the cross-shard episodes
  uint32_t abort;                // raised by a participant that timed out
  uint32_t arrive2;              // flip barrier of the mid-round phase (one launch)
  uint32_t pad0[29];
  unsigned long long sum[4];     // per barrier episode (mod 4): sums
  unsigned int minv[4];          // per barrier episode (mod 4): minima
  uint32_t pad1[20];
};
static_assert(sizeof(XCtrl) == 256, "XCtrl is two cache lines");

// device view of one shard's peer block
struct PeerView {
  uint32_t* deg;
  uint32_t* labels;
  uint32_t* q[2];               // frontier queues (round parity)
  unsigned long long* ctr;      // [2] queue counters
  XCtrl* x;                     // the block's control block
};

struct dg_shard {
  uint64_t n = 0;  // global vertex count
  uint64_t lo = 0, hi = 0;
  uint32_t rank = 0;
  dgb::DevBuf<uint64_t> offs;  // the rank's own rows: local offsets, n_local + 1
  dgb::DevBuf<uint32_t> adj;   // neighbour ids (global dense ids)
  void* block = nullptr;       // peer-visible state (cudaMalloc: IPC-exportable)
  PeerView own{};
  uint32_t cur = 0;            // queue holding the current frontier
  dgb::DevBuf<unsigned long long> cnt;  // [0] next size, [1] min, [2..] per-rank counts
  uint64_t nfront = 0;
  dgb::DevBuf<uint64_t> bounds;  // rank boundaries (P + 1)
  std::vector<uint64_t> hbounds;
  uint32_t P = 0;
  std::vector<PeerView> peers;   // per rank (own entry included)
  std::vector<void*> opened;     // IPC mappings to close
  dgb::DevBuf<PeerView> d_peers;
  bool peers_ready = false;
  ~dg_shard() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    if (block) cudaFree(block);
  }
};

// block layout: ctr u64[2] (+ pad to 128) | XCtrl | deg | labels | q0 | q1 (u32[nl] each)
inline size_t shard_block_bytes(uint64_t nl) { return 128 + sizeof(XCtrl) + 16 * (nl ? nl : 1); }
inline PeerView shard_block_view(void* block, uint64_t nl) {
  char* b = static_cast<char*>(block);
  const uint64_t w = nl ? nl : 1;
  PeerView v;
  v.ctr = reinterpret_cast<unsigned long long*>(b);
  v.x = reinterpret_cast<XCtrl*>(b + 128);
  v.deg = reinterpret_cast<uint32_t*>(b + 128 + sizeof(XCtrl));
  v.labels = v.deg + w;
  v.q[0] = v.labels + w;
  v.q[1] = v.q[0] + w;
  return v;
}

namespace dgb {
// the peer views of every shard as seen from this process (uploads once)
const PeerView* shard_device_peers(dg_shard* s);
}  // namespace dgb
