// Physical pool shared by the C-ABI allocator calls (oc_alloc/oc_map/...)
// and the executor.
#pragma once
#include <deque>
#include <set>
#include <unordered_map>
#include <vector>

#include "cuda_util.hpp"

namespace oc {

struct Span {
  uint64_t handle = 0;
  CUdeviceptr va = 0;
  uint64_t m_r = 0, m_a = 0, offset = 0;
  uint32_t k = 0;
  std::vector<uint32_t> bound;   // chunks logically owned (between map and unmap)
  std::vector<uint32_t> mapped;  // chunks the driver currently maps at va
  bool live = false;
  cudaEvent_t ev = nullptr;      // release event of the span's last use
  bool ev_used = false;
};

struct MemPool {
  int device = 0;
  oc_alloc_model model{};
  uint32_t flags = 0;
  Driver* drv = nullptr;
  size_t gran = 0;
  CUmemAllocationProp prop{};
  CUmemAccessDesc access{};
  // VA
  uint64_t m_c = 0;
  uint32_t n_chunks = 0;
  std::vector<CUmemGenericAllocationHandle> chunk;
  std::vector<cudaEvent_t> chunk_ev;
  std::vector<uint8_t> chunk_ev_used;
  std::deque<uint32_t> free_q;
  std::vector<uint64_t> deferred;  // spans awaiting an eager unmap
  // arena
  CUdeviceptr slab = 0;
  uint64_t slab_bytes = 0;
  CUmemGenericAllocationHandle slab_h = 0;
  ArenaPlacer placer;
  struct Released { uint64_t start, end; cudaEvent_t ev; };
  std::vector<Released> released;   // arena: byte ranges whose release has not completed yet
  std::vector<cudaEvent_t> ev_pool;  // recycled release events
  cudaEvent_t take_event();
  void poll_released();              // drop (and recycle) releases whose event has completed
  // spans
  std::unordered_map<uint64_t, Span> spans;
  std::set<uint64_t> freed;
  uint64_t next_handle = 1;
  // stats
  uint64_t live_requested = 0, live_allocated = 0, peak_mapped = 0, live_if = 0, if_peak = 0;
  uint32_t live_count = 0, n_max = 0;
  uint64_t n_driver_map = 0, n_driver_unmap = 0, n_map_calls = 0, n_map_memo_hits = 0;
  double map_us = 0, unmap_us = 0;

  Status init(int dev, const oc_alloc_model& m, uint32_t flags);
  Status ensure_chunk(uint32_t c);
  Status reserve(uint64_t m_a, CUdeviceptr& va);
  Status bind(Span& s, const std::vector<uint32_t>& chunks);  // memoised map + setaccess
  Status driver_unmap(Span& s);
  void poll_deferred();
  void destroy();
};

}  // namespace oc

struct oc_mem {
  oc::MemPool p;
};
