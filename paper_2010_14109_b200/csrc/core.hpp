// Internal host-side structures of liboocore: graph, variable-sequence,
// schedule and allocator replay.  No CUDA here — this part runs (and is
// tested) on a machine without a GPU.
#pragma once
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "json.hpp"
#include "oocore.h"

namespace oc {

constexpr int64_t NONE = -1;

struct Status {
  int code = OC_OK;
  uint32_t fn = UINT32_MAX, var = UINT32_MAX;
  uint64_t needed = 0, free_bytes = 0;
  int cuda = 0;
  std::string msg;
  static Status ok() { return Status(); }
  static Status make(int c, std::string m) {
    Status s;
    s.code = c;
    s.msg = std::move(m);
    return s;
  }
  bool good() const { return code == OC_OK; }
  void fill(oc_err* e) const {
    if (!e) return;
    e->code = code;
    e->fn = fn;
    e->var = var;
    e->needed = needed;
    e->free_bytes = free_bytes;
    e->cuda = cuda;
    std::strncpy(e->msg, msg.c_str(), sizeof(e->msg) - 1);
    e->msg[sizeof(e->msg) - 1] = 0;
  }
};

struct Function {
  std::string name;
  std::vector<uint32_t> in, out;
  std::string op_json;  // raw op descriptor ("" if none)
  JVal op;              // parsed op descriptor
  uint32_t decl = 0;    // declaration index
};

struct Graph {
  std::vector<std::string> var_names;
  std::vector<uint64_t> var_bytes;
  std::vector<uint8_t> persistent, pinned;
  std::vector<Function> fns;        // execution order after finalize
  std::vector<uint32_t> decl_to_pos;
  bool finalized = false;

  // variable-sequence v over non-pinned variables
  std::vector<uint32_t> occ;
  std::vector<uint64_t> occ_bytes;
  std::vector<int64_t> l, e;        // span of f_i: [l_i, e_i]; e_i = l_i - 1 if empty
  std::vector<int64_t> next_use;    // next occurrence of the same variable or NONE
  uint64_t pinned_bytes = 0;

  uint32_t nv() const { return (uint32_t)var_names.size(); }
  uint32_t nf() const { return (uint32_t)fns.size(); }
};

Status graph_from_json(const char* s, size_t n, Graph& g);
Status graph_finalize(Graph& g);
uint64_t graph_in_core_peak(const Graph& g);

// ------------------------------------------------------------- schedule
enum ArrivalKind : uint8_t { ARRIVE_H2D = 0, ARRIVE_ALLOC = 1 };

struct Arrival {
  uint32_t var;
  uint8_t kind;
  // allocator placement decided by the replay
  uint64_t offset = 0;            // arena: byte offset in the slab
  std::vector<uint32_t> chunks;   // VA: chunk indices (FIFO order)
  uint32_t slot = 0;              // index over all arrivals of the step
};

struct Departure {                // a surviving reservation
  uint32_t var;
  uint8_t dirty;                  // host copy stale at reservation time
  int32_t wait_fn;                // function before which it is waited (-1 = end)
};

struct FnSchedule {
  std::vector<Arrival> in;
  std::vector<uint32_t> wait_out;
  std::vector<Departure> reserve_out;
  std::vector<uint32_t> free;
};

struct ReplayStats {
  uint64_t peak_phys = 0, peak_alloc = 0, if_peak = 0;
  uint32_t n_max = 0;
  int32_t oom_fn = -1, oom_var = -1;
  uint64_t oom_request = 0, oom_free = 0;
};

struct Schedule {
  const Graph* g = nullptr;
  uint64_t budget = 0, window = 0;
  uint32_t distance = 0;      // > 0: prior-art function-distance window (F1)
  oc_alloc_model alloc{};
  std::vector<int64_t> r;
  std::vector<FnSchedule> fn;
  std::vector<uint32_t> end_wait;
  uint64_t bytes_h2d = 0, bytes_alloc = 0, bytes_d2h = 0, bytes_d2h_dirty = 0, peak_sched = 0;
  uint32_t n_in_h2d = 0, n_in_alloc = 0, n_out = 0, n_arrivals = 0;
  ReplayStats replay;
};

// Caching best-/first-fit arena placer, shared by
// the plan-time replay and the runtime arena.
struct ArenaPlacer {
  struct Blk { uint64_t start, size, seg; bool free; };
  uint64_t cap = 0, align = 512, tail = 0, allocated = 0;
  bool best = true;
  std::vector<Blk> blocks;                // sorted by start
  std::map<uint64_t, uint64_t> live;      // key -> block start
  void init(uint64_t capacity, uint64_t al, bool best_fit) {
    cap = capacity; align = al; best = best_fit; tail = allocated = 0; blocks.clear(); live.clear();
  }
  bool alloc(uint64_t key, uint64_t m_r, uint64_t& off);
  uint64_t free(uint64_t key);            // returns the freed block size
  uint64_t free_bytes() const;
};

std::vector<int64_t> window_ends(const Graph& g, uint64_t W);
std::vector<int64_t> window_ends_distance(const Graph& g, uint32_t d);
uint64_t min_feasible_budget(const Graph& g, uint64_t W, uint32_t distance = 0);
Status max_feasible_window(const Graph& g, uint64_t budget, uint64_t& W);
Status build_schedule(const Graph& g, uint64_t budget, uint64_t W, Schedule& s, uint32_t distance = 0);
Status replay_allocator(const Graph& g, Schedule& s);
std::string schedule_json(const Schedule& s);

}  // namespace oc

// opaque handles of the C ABI
struct oc_graph {
  oc::Graph g;
};
struct oc_schedule {
  oc::Schedule s;
  const oc_graph* owner;
};
