// Executor of one out-of-core training step under a window schedule.
//
// Per function f_i, in the paper's order (reading Z9):
//   wait_out[i]  compute stream waits the D2H completion of each waited
//                variable ("waits for the Swap-out right before f_i", P:86b);
//                its memory is released at that point
//   in[i]        H2D stream: wait the release points of the memory the
//                arrival reuses (static, from the allocator replay), map the
//                chunks (VA, memoised), copy host->device (h2d) or only
//                materialise (alloc); record ev_in
//   f_i          compute stream waits ev_in of V̂_i, launches f_i's kernels,
//                records ev_done[i]
//   reserve_out  D2H stream waits ev_done[i], copies device->host
//                ("Swap-out is reserved right after the previous function
//                using the variable", P:86b); records ev_out
//   free[i]      memory released at ev_done[i]
// Addresses are fixed per arrival slot and identical every step, so after the
// first step no driver call is made (memoised VA) and the host only issues
// copies, event waits and kernels.
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <dlfcn.h>
#include <sstream>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <fstream>

#include "mem.hpp"
#include "ops.hpp"
#include "pack.hpp"

namespace oc {

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// a release point: compute event after f_j, or the D2H completion of departure d
struct Ref {
  enum { DONE, OUT } type;
  uint32_t idx;
  bool operator==(const Ref& o) const { return type == o.type && idx == o.idx; }
};

struct Slot {
  uint32_t var = 0, fn = 0;
  uint8_t kind = ARRIVE_H2D;
  CUdeviceptr addr = 0;
  Span span;                       // VA mode: fixed span of this arrival slot
  std::vector<uint32_t> chunks;    // VA mode: chunks from the replay
  std::vector<Ref> waits;          // release points of reused memory
  int32_t host_dep = -1;           // departure whose D2H must land before this H2D
  bool packed = false;             // moved by the function's unpack kernel (A7)
};

struct Dep {
  uint32_t fn, var;
  uint8_t dirty;
  int32_t wait_fn;
  int32_t slot = -1;               // arrival slot holding the variable when it leaves
  bool packed = false;             // moved by the function's pack kernel (A7)
};

struct XVar {
  uint64_t bytes = 0;
  bool pinned = false, persistent = false;
  void* dev_fixed = nullptr;       // pinned variables: bound by the caller
  int64_t host_off = -1;
  int32_t cur_slot = -1;
  bool need_wait = false;
  int32_t async_fn = -1;           // produced by an allreduce still running on the comm stream
};

struct XFn {
  const OpDesc* op = nullptr;
  std::vector<std::vector<uint32_t>> role_vars;  // per role, variables
  std::vector<int32_t> dep_of_wait;              // parallel to wait_out: departure ids
  std::vector<uint32_t> dep_reserve;             // departure ids reserved after f_i
  uint32_t pin_off = 0, pin_n = 0;               // unpack entries (small arrivals) in pack_tab
  uint32_t pout_off = 0, pout_n = 0;             // pack entries (small departures)
  bool is_allreduce = false;                     // gradient exchange (comm stream when attached)
};

// NUMA node of a GPU's PCIe root (sysfs), -1 if unknown
int gpu_numa_node(int dev) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
  std::string b(bus);
  for (char& c : b) c = (char)std::tolower((unsigned char)c);
  std::ifstream f("/sys/bus/pci/devices/" + b + "/numa_node");
  int n = -1;
  if (!(f >> n)) return -1;
  return n;
}

// The pinned host pool on the GPU's NUMA node (each replica's
// host copies local to its PCIe link): anonymous pages with a preferred-node
// policy (mbind), faulted in there, then page-locked and mapped for the
// device (cudaHostRegister).  Falls back to cudaHostAlloc when the node is
// unknown or any step fails.
struct HostPool {
  char* p = nullptr;
  uint64_t bytes = 0;
  int node = -1;
  bool registered = false;
  Status alloc(int dev, uint64_t n) {
    bytes = n;
    node = gpu_numa_node(dev);
    if (node >= 0 && node < 1024) {
      void* m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (m != MAP_FAILED) {
        unsigned long mask[16] = {0};
        mask[node / 64] |= 1UL << (node % 64);
        const long rc = syscall(SYS_mbind, m, n, 1 /* MPOL_PREFERRED */, mask, 1024, 0);
        std::memset(m, 0, n);   // fault the pages in on the preferred node
        if (rc == 0 && cudaHostRegister(m, n, cudaHostRegisterPortable | cudaHostRegisterMapped) == cudaSuccess) {
          p = (char*)m;
          registered = true;
          return Status::ok();
        }
        (void)cudaGetLastError();
        munmap(m, n);
      }
      node = -1;
    }
    OC_CUDA(cudaHostAlloc((void**)&p, n, cudaHostAllocPortable | cudaHostAllocMapped));
    std::memset(p, 0, n);
    return Status::ok();
  }
  void release() {
    if (!p) return;
    if (registered) {
      cudaHostUnregister(p);
      munmap(p, bytes);
    } else {
      cudaFreeHost(p);
    }
    p = nullptr;
  }
};

struct Interval { double a, b; };

double union_len(std::vector<Interval> v) {
  std::sort(v.begin(), v.end(), [](const Interval& x, const Interval& y) { return x.a < y.a; });
  double tot = 0, ca = -1e300, cb = -1e300;
  for (auto& x : v) {
    if (x.a > cb) { if (cb > ca) tot += cb - ca; ca = x.a; cb = x.b; }
    else cb = std::max(cb, x.b);
  }
  if (cb > ca) tot += cb - ca;
  return tot;
}

std::vector<Interval> merge(std::vector<Interval> v) {
  std::sort(v.begin(), v.end(), [](const Interval& x, const Interval& y) { return x.a < y.a; });
  std::vector<Interval> out;
  for (auto& x : v) {
    if (out.empty() || x.a > out.back().b) out.push_back(x);
    else out.back().b = std::max(out.back().b, x.b);
  }
  return out;
}

double inter_len(const std::vector<Interval>& A, const std::vector<Interval>& B) {
  auto a = merge(A), b = merge(B);
  size_t i = 0, j = 0;
  double t = 0;
  while (i < a.size() && j < b.size()) {
    double lo = std::max(a[i].a, b[j].a), hi = std::min(a[i].b, b[j].b);
    if (hi > lo) t += hi - lo;
    if (a[i].b < b[j].b) ++i; else ++j;
  }
  return t;
}

}  // namespace

// the largest per-function workspace of the graph's ops (oc_graph_workspace_bytes)
size_t graph_workspace(const Graph& g) {
  size_t ws = 0;
  for (const Function& f : g.fns) {
    if (f.op.kind != JVal::OBJ) continue;
    const OpDesc* d = find_op(f.op.gets("kind"));
    const JVal* attrs = f.op.get("attrs");
    if (d && d->workspace && attrs) ws = std::max(ws, d->workspace(*attrs));
  }
  return ws;
}

struct Exec {
  int device = 0;
  const Graph* g = nullptr;
  const Schedule* s = nullptr;
  MemPool* mem = nullptr;
  cudaStream_t cs = nullptr, hs = nullptr, ds = nullptr;
  oc_exec_options opt{};
  std::vector<XVar> vars;
  std::vector<XFn> fns;
  std::vector<Slot> slots;
  std::vector<Dep> deps;
  std::vector<int32_t> end_deps;
  std::vector<cudaEvent_t> ev_done, ev_in, ev_out;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_fork = nullptr;
  cudaGraphExec_t gexec = nullptr;    // captured step (opt.use_graph)
  uint64_t g_bytes_h2d = 0, g_bytes_d2h = 0;
  uint32_t g_n_h2d = 0, g_n_d2h = 0, g_n_kernels = 0;
  bool have_prev = false;
  char* host = nullptr;
  uint64_t host_bytes = 0;
  HostPool host_pool;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  PackEntry* pack_tab = nullptr;   // device copy of all pack/unpack entries (static addresses)
  // timeline (opt.timeline)
  std::vector<cudaEvent_t> tl_fn0, tl_fn1, tl_in0, tl_in1, tl_out0, tl_out1;
  std::vector<uint8_t> tl_in_used, tl_out_used;
  std::vector<int32_t> tl_in_ref, tl_out_ref;   // slot / departure whose events time this one (pack kernels)
  std::vector<KernelTimer> tl_k;   // per function: the contraction kernel launches
  // NCCL
  void* nccl_lib = nullptr;
  void* nccl_comm = nullptr;
  void* nccl_allreduce = nullptr;
  void* nccl_destroy = nullptr;
  void* nccl_group_start = nullptr, *nccl_group_end = nullptr;
  oc_allreduce_fn comm_fn = nullptr;   // custom communicator (tests, other transports)
  void* comm_user = nullptr;
  // gradient exchange on its own stream: an allreduce function f_i (a bucket of
  // gradients) runs on comm_s, forked from the compute stream after f_i's
  // inputs are produced; ev_done[i] is recorded on comm_s, so every consumer of
  // the bucket (the SGD placed one bucket later, swap-outs, memory reuse) waits
  // for the exchange while the compute stream runs the next layers' backward
  cudaStream_t comm_s = nullptr;
  cudaEvent_t ev_cfork = nullptr, ev_cjoin = nullptr;
  Status ensure_comm_stream() {
    if (comm_s) return Status::ok();
    OC_CUDA(cudaSetDevice(device));
    OC_CUDA(cudaStreamCreateWithFlags(&comm_s, cudaStreamNonBlocking));
    OC_CUDA(cudaEventCreateWithFlags(&ev_cfork, cudaEventDisableTiming));
    OC_CUDA(cudaEventCreateWithFlags(&ev_cjoin, cudaEventDisableTiming));
    return Status::ok();
  }
  uint64_t step_index = 0;
  // layer-local inspection hook (oc_exec_set_hook; tests only)
  oc_fn_hook hook = nullptr;
  void* hook_user = nullptr;
  bool tl_created = false;   // timeline events exist (created with opt.timeline)

  Status create(int dev, const Graph* graph, const Schedule* sch, MemPool* m, const oc_streams& st,
                const oc_exec_options* o);
  Status run(oc_step_metrics* out);
  void destroy();
  void* addr_of(uint32_t v) const {
    const XVar& x = vars[v];
    if (x.pinned) return x.dev_fixed;
    return x.cur_slot >= 0 ? (void*)slots[x.cur_slot].addr : nullptr;
  }
};

Status Exec::create(int dev, const Graph* graph, const Schedule* sch, MemPool* m, const oc_streams& st,
                    const oc_exec_options* o) {
  device = dev;
  g = graph;
  s = sch;
  mem = m;
  cs = (cudaStream_t)st.compute;
  hs = (cudaStream_t)st.h2d;
  ds = (cudaStream_t)st.d2h;
  if (o) opt = *o;
  OC_CUDA(cudaSetDevice(dev));
  if (s->replay.oom_fn >= 0) return Status::make(OC_E_DEVICE_OOM, "schedule's allocator replay ran out of memory");
  const auto& am = s->alloc;
  if (am.mode != m->model.mode) return Status::make(OC_E_ARG, "schedule and memory pool use different allocator modes");
  if (am.mode == OC_ALLOC_VA && am.chunk_bytes != m->m_c)
    return Status::make(OC_E_ARG, "schedule chunk size differs from the pool's");
  const uint64_t phys = am.phys_bytes ? am.phys_bytes : (s->budget - g->pinned_bytes);
  if (am.mode == OC_ALLOC_VA && phys / am.chunk_bytes > m->n_chunks)
    return Status::make(OC_E_ARG, "memory pool has fewer chunks than the schedule's replay");
  if (am.mode != OC_ALLOC_VA && m->slab_bytes < s->replay.peak_phys)
    return Status::make(OC_E_ARG, "arena slab smaller than the schedule's peak");

  // variables
  vars.resize(g->nv());
  for (uint32_t v = 0; v < g->nv(); ++v) {
    vars[v].bytes = g->var_bytes[v];
    vars[v].pinned = g->pinned[v];
    vars[v].persistent = g->persistent[v];
  }
  // host copies: persistent variables and every variable ever swapped out
  std::vector<uint8_t> needs_host(g->nv(), 0);
  for (uint32_t v = 0; v < g->nv(); ++v) needs_host[v] = g->persistent[v] && !g->pinned[v];
  for (auto& F : s->fn)
    for (auto& d : F.reserve_out) needs_host[d.var] = 1;
  host_bytes = 0;
  for (uint32_t v = 0; v < g->nv(); ++v)
    if (needs_host[v]) {
      vars[v].host_off = (int64_t)host_bytes;
      host_bytes += (g->var_bytes[v] + 255) / 256 * 256;
    }
  if (host_bytes) {
    // mapped: the pack/unpack kernel addresses it directly (UVA: same pointer on the device)
    OC_TRY(host_pool.alloc(dev, host_bytes));
    host = host_pool.p;
  }

  // departures
  const uint32_t n = g->nf();
  fns.resize(n);
  for (uint32_t i = 0; i < n; ++i)
    for (auto& d : s->fn[i].reserve_out) {
      fns[i].dep_reserve.push_back((uint32_t)deps.size());
      deps.push_back(Dep{i, d.var, d.dirty, d.wait_fn});
    }
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t v : s->fn[i].wait_out) {
      int32_t id = -1;
      for (uint32_t d = 0; d < deps.size(); ++d)
        if (deps[d].wait_fn == (int32_t)i && deps[d].var == v) { id = (int32_t)d; break; }
      if (id < 0) return Status::make(OC_E_INVARIANT, "wait without a departure");
      fns[i].dep_of_wait.push_back(id);
    }
  for (uint32_t v : s->end_wait) {
    int32_t id = -1;
    for (uint32_t d = 0; d < deps.size(); ++d)
      if (deps[d].wait_fn == -1 && deps[d].var == v) { id = (int32_t)d; break; }
    if (id < 0) return Status::make(OC_E_INVARIANT, "end wait without a departure");
    end_deps.push_back(id);
  }

  // arrival slots and the static hazard analysis over the replay's placements
  slots.resize(s->n_arrivals);
  const bool va = am.mode == OC_ALLOC_VA;
  std::vector<Ref> chunk_rel;                 // VA: last release point per chunk
  std::vector<uint8_t> chunk_has;
  struct Range { uint64_t a, b; Ref r; };
  std::vector<Range> ranges;                  // arena: released byte ranges
  if (va) { chunk_rel.resize(m->n_chunks); chunk_has.assign(m->n_chunks, 0); }
  std::vector<int32_t> var_slot(g->nv(), -1), var_last_dep(g->nv(), -1);
  auto release = [&](uint32_t v, Ref r) {
    const Slot& sl = slots[var_slot[v]];
    if (va) {
      for (uint32_t c : sl.chunks) { chunk_rel[c] = r; chunk_has[c] = 1; }
    } else {
      uint64_t off = sl.addr - m->slab;
      uint64_t al = am.align ? am.align : 512;
      ranges.push_back(Range{off, off + (vars[v].bytes + al - 1) / al * al, r});
    }
    var_slot[v] = -1;
  };
  for (uint32_t i = 0; i < n; ++i) {
    const FnSchedule& F = s->fn[i];
    for (size_t k = 0; k < F.wait_out.size(); ++k) {
      uint32_t v = F.wait_out[k];
      release(v, Ref{Ref::OUT, (uint32_t)fns[i].dep_of_wait[k]});
    }
    for (const Arrival& a : F.in) {
      Slot& sl = slots[a.slot];
      sl.var = a.var;
      sl.fn = i;
      sl.kind = a.kind;
      auto add = [&](Ref r) {
        if (r.type == Ref::DONE && r.idx >= i) return;  // cannot happen; defensive
        if (std::find(sl.waits.begin(), sl.waits.end(), r) == sl.waits.end()) sl.waits.push_back(r);
      };
      if (va) {
        sl.chunks = a.chunks;
        for (uint32_t c : a.chunks)
          if (chunk_has[c]) add(chunk_rel[c]);
        sl.span.m_r = vars[a.var].bytes;
        sl.span.k = (uint32_t)a.chunks.size();
        sl.span.m_a = (uint64_t)sl.span.k * m->m_c;
        OC_TRY(m->reserve(sl.span.m_a, sl.span.va));
        sl.addr = sl.span.va;
      } else {
        sl.addr = m->slab + a.offset;
        uint64_t al = am.align ? am.align : 512;
        uint64_t lo = a.offset, hi = a.offset + (vars[a.var].bytes + al - 1) / al * al;
        for (size_t k = 0; k < ranges.size();) {
          if (ranges[k].a < hi && lo < ranges[k].b) {
            add(ranges[k].r);
            if (lo <= ranges[k].a && ranges[k].b <= hi) { ranges[k] = ranges.back(); ranges.pop_back(); continue; }
          }
          ++k;
        }
      }
      if (a.kind == ARRIVE_H2D && var_last_dep[a.var] >= 0) sl.host_dep = var_last_dep[a.var];
      var_slot[a.var] = (int32_t)a.slot;
    }
    for (uint32_t d : fns[i].dep_reserve) {
      var_last_dep[deps[d].var] = (int32_t)d;
      deps[d].slot = var_slot[deps[d].var];
    }
    for (uint32_t v : F.free) release(v, Ref{Ref::DONE, i});
  }

  // pack/unpack tables (A7): static entries per function, addresses fixed per slot
  if (opt.pack_threshold) {
    std::vector<PackEntry> tab;
    for (uint32_t i = 0; i < n; ++i) {
      XFn& X = fns[i];
      X.pin_off = (uint32_t)tab.size();
      for (const Arrival& a : s->fn[i].in) {
        Slot& sl = slots[a.slot];
        const XVar& xv = vars[sl.var];
        if (sl.kind != ARRIVE_H2D || xv.bytes > opt.pack_threshold) continue;
        sl.packed = true;
        tab.push_back(PackEntry{(const unsigned char*)(host + xv.host_off), (unsigned char*)sl.addr, xv.bytes});
      }
      X.pin_n = (uint32_t)tab.size() - X.pin_off;
      X.pout_off = (uint32_t)tab.size();
      for (uint32_t d : X.dep_reserve) {
        Dep& D = deps[d];
        const XVar& xv = vars[D.var];
        if (xv.bytes > opt.pack_threshold || !(D.dirty || !opt.elide_clean)) continue;
        D.packed = true;
        tab.push_back(PackEntry{(const unsigned char*)slots[D.slot].addr, (unsigned char*)(host + xv.host_off),
                                xv.bytes});
      }
      X.pout_n = (uint32_t)tab.size() - X.pout_off;
    }
    if (!tab.empty()) {
      OC_CUDA(cudaMalloc((void**)&pack_tab, tab.size() * sizeof(PackEntry)));
      OC_CUDA(cudaMemcpy(pack_tab, tab.data(), tab.size() * sizeof(PackEntry), cudaMemcpyHostToDevice));
    }
  }

  // ops
  size_t ws_need = graph_workspace(*g);
  for (uint32_t i = 0; i < n; ++i) {
    const Function& f = g->fns[i];
    if (f.op.kind != JVal::OBJ) continue;  // a function without compute (planner-only graphs)
    std::string kind = f.op.gets("kind");
    const OpDesc* d = find_op(kind);
    if (!d) {
      Status e = Status::make(OC_E_UNSUPPORTED, "function " + f.name + ": unknown op kind '" + kind + "'");
      e.fn = i;
      return e;
    }
    fns[i].op = d;
    fns[i].is_allreduce = kind == "allreduce";
    const JVal* args = f.op.get("args");
    fns[i].role_vars.resize(d->roles.size());
    for (size_t r = 0; r < d->roles.size(); ++r) {
      const JVal* a = args ? args->get(d->roles[r]) : nullptr;
      if (!a || a->kind == JVal::NUL) continue;
      std::vector<const JVal*> items;
      if (a->kind == JVal::ARR) for (auto& x : a->arr) items.push_back(&x);
      else items.push_back(a);
      for (const JVal* x : items) {
        uint32_t v = UINT32_MAX;
        for (uint32_t j = 0; j < g->nv(); ++j)
          if (g->var_names[j] == x->s) { v = j; break; }
        if (v == UINT32_MAX || x->kind != JVal::STR) {
          Status e = Status::make(OC_E_INVALID, "function " + f.name + ": role " + d->roles[r] + " names no variable");
          e.fn = i;
          return e;
        }
        bool used = std::find(f.in.begin(), f.in.end(), v) != f.in.end() ||
                    std::find(f.out.begin(), f.out.end(), v) != f.out.end();
        if (!used) {
          Status e = Status::make(OC_E_INVALID, "function " + f.name + ": op reads " + x->s + " which is not in V̂_i");
          e.fn = i;
          e.var = v;
          return e;
        }
        fns[i].role_vars[r].push_back(v);
      }
    }
  }
  ws_bytes = ws_need;
  if (ws_bytes) OC_CUDA(cudaMalloc(&ws, ws_bytes));

  // events
  auto mk = [&](std::vector<cudaEvent_t>& v, size_t cnt, bool timing) -> Status {
    v.assign(cnt, nullptr);
    for (auto& e : v) OC_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    return Status::ok();
  };
  OC_TRY(mk(ev_done, n, false));
  OC_TRY(mk(ev_in, slots.size(), false));
  OC_TRY(mk(ev_out, deps.size(), false));
  OC_CUDA(cudaEventCreate(&ev_start));
  OC_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  OC_CUDA(cudaEventCreate(&ev_end));
  if (opt.timeline) {
    OC_TRY(mk(tl_fn0, n, true));
    OC_TRY(mk(tl_fn1, n, true));
    OC_TRY(mk(tl_in0, slots.size(), true));
    OC_TRY(mk(tl_in1, slots.size(), true));
    OC_TRY(mk(tl_out0, deps.size(), true));
    OC_TRY(mk(tl_out1, deps.size(), true));
    tl_k.resize(n);
    tl_created = true;
  }
  return Status::ok();
}

Status Exec::run(oc_step_metrics* out) {
  OC_CUDA(cudaSetDevice(device));
  for (uint32_t v = 0; v < vars.size(); ++v) {
    if (vars[v].pinned && !vars[v].dev_fixed) {
      Status e = Status::make(OC_E_ARG, "pinned variable " + g->var_names[v] + " has no bound device address");
      e.var = v;
      return e;
    }
    vars[v].cur_slot = -1;
    vars[v].need_wait = false;
    vars[v].async_fn = -1;
  }
  const double t_host0 = now_ms();
  const double map0 = mem->map_us, unmap0 = mem->unmap_us;
  uint64_t bytes_h2d = 0, bytes_d2h = 0;
  uint32_t n_h2d = 0, n_d2h = 0, n_kernels = 0;
  tl_in_used.assign(slots.size(), 0);
  tl_out_used.assign(deps.size(), 0);
  tl_in_ref.resize(slots.size());
  tl_out_ref.resize(deps.size());
  for (size_t k = 0; k < slots.size(); ++k) tl_in_ref[k] = (int32_t)k;
  for (size_t k = 0; k < deps.size(); ++k) tl_out_ref[k] = (int32_t)k;
  auto ev_of = [&](const Ref& r) { return r.type == Ref::DONE ? ev_done[r.idx] : ev_out[r.idx]; };

  // The whole step is issued by `issue`: eagerly, or once into a CUDA graph
  // (opt.use_graph, after one eager step has memoised every VA mapping) that
  // later steps replay with a single launch.
  const uint32_t n = g->nf();
  auto issue = [&]() -> Status {
  // the previous step (incl. its end waits) is complete on the compute stream
  OC_CUDA(cudaEventRecord(ev_fork, cs));
  OC_CUDA(cudaStreamWaitEvent(hs, ev_fork, 0));
  OC_CUDA(cudaStreamWaitEvent(ds, ev_fork, 0));
  for (uint32_t i = 0; i < n; ++i) {
    const FnSchedule& F = s->fn[i];
    XFn& X = fns[i];
    // (b) waits before f_i
    for (size_t k = 0; k < X.dep_of_wait.size(); ++k) {
      OC_CUDA(cudaStreamWaitEvent(cs, ev_out[X.dep_of_wait[k]], 0));
      vars[F.wait_out[k]].cur_slot = -1;  // swapped out: no longer resident
    }
    // (a) arrivals; small H2D arrivals go through one unpack kernel (A7).
    // Paper trigger (opt.trigger = 1): the arrivals of f_i are issued at the
    // function boundary — after f_{i-1} and the swap-outs waited in (b).
    auto paper_gate = [&](cudaStream_t h) -> Status {
      if (opt.trigger != 1) return Status::ok();
      if (i > 0) OC_CUDA(cudaStreamWaitEvent(h, ev_done[i - 1], 0));
      for (int32_t d : X.dep_of_wait) OC_CUDA(cudaStreamWaitEvent(h, ev_out[d], 0));
      return Status::ok();
    };
    for (const Arrival& a : F.in) {
      Slot& sl = slots[a.slot];
      if (s->alloc.mode == OC_ALLOC_VA) OC_TRY(mem->bind(sl.span, sl.chunks));
      if (sl.packed) continue;
      cudaStream_t h = hs;
      for (const Ref& r : sl.waits) OC_CUDA(cudaStreamWaitEvent(h, ev_of(r), 0));
      OC_TRY(paper_gate(h));
      if (sl.kind == ARRIVE_H2D) {
        if (sl.host_dep >= 0) OC_CUDA(cudaStreamWaitEvent(h, ev_out[sl.host_dep], 0));
        XVar& xv = vars[sl.var];
        if (opt.timeline) { OC_CUDA(cudaEventRecord(tl_in0[a.slot], h)); tl_in_used[a.slot] = 1; }
        OC_CUDA(cudaMemcpyAsync((void*)sl.addr, host + xv.host_off, xv.bytes, cudaMemcpyHostToDevice, h));
        if (opt.timeline) OC_CUDA(cudaEventRecord(tl_in1[a.slot], h));
        bytes_h2d += xv.bytes;
        ++n_h2d;
      }
      OC_CUDA(cudaEventRecord(ev_in[a.slot], h));
      vars[sl.var].cur_slot = (int32_t)a.slot;
      vars[sl.var].need_wait = true;
    }
    if (X.pin_n) {
      int32_t first = -1;
      for (const Arrival& a : F.in) {
        Slot& sl = slots[a.slot];
        if (!sl.packed) continue;
        if (first < 0) first = (int32_t)a.slot;
        for (const Ref& r : sl.waits) OC_CUDA(cudaStreamWaitEvent(hs, ev_of(r), 0));
        if (sl.host_dep >= 0) OC_CUDA(cudaStreamWaitEvent(hs, ev_out[sl.host_dep], 0));
        bytes_h2d += vars[sl.var].bytes;
      }
      OC_TRY(paper_gate(hs));
      if (opt.timeline) { OC_CUDA(cudaEventRecord(tl_in0[first], hs)); tl_in_used[first] = 1; }
      OC_TRY(pack_launch(pack_tab + X.pin_off, (int)X.pin_n, hs));
      if (opt.timeline) OC_CUDA(cudaEventRecord(tl_in1[first], hs));
      ++n_h2d;
      ++n_kernels;
      for (const Arrival& a : F.in) {
        Slot& sl = slots[a.slot];
        if (!sl.packed) continue;
        if (opt.timeline) { tl_in_used[a.slot] = 1; tl_in_ref[a.slot] = first; }
        OC_CUDA(cudaEventRecord(ev_in[a.slot], hs));
        vars[sl.var].cur_slot = (int32_t)a.slot;
        vars[sl.var].need_wait = true;
      }
    }
    // f_i on the compute stream
    const Function& f = g->fns[i];
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t v : (pass == 0 ? f.in : f.out)) {
        XVar& xv = vars[v];
        if (xv.async_fn >= 0) {   // a gradient bucket still being exchanged
          OC_CUDA(cudaStreamWaitEvent(cs, ev_done[xv.async_fn], 0));
          xv.async_fn = -1;
        }
        if (xv.pinned) continue;
        if (xv.cur_slot < 0) {
          Status e = Status::make(OC_E_INVARIANT, "variable " + g->var_names[v] + " not resident at " + f.name);
          e.fn = i;
          e.var = v;
          return e;
        }
        if (xv.need_wait) {
          OC_CUDA(cudaStreamWaitEvent(cs, ev_in[xv.cur_slot], 0));
          xv.need_wait = false;
        }
      }
    if (hook) {
      OC_CUDA(cudaDeviceSynchronize());
      hook(hook_user, i, 0);
    }
    const bool on_comm = X.is_allreduce && comm_s && (nccl_comm || comm_fn);
    cudaStream_t fs = on_comm ? comm_s : cs;
    if (on_comm) {
      OC_CUDA(cudaEventRecord(ev_cfork, cs));
      OC_CUDA(cudaStreamWaitEvent(comm_s, ev_cfork, 0));
    }
    if (opt.timeline) OC_CUDA(cudaEventRecord(tl_fn0[i], fs));
    if (X.op) {
      OpArgs oa;
      oa.ptr.resize(X.role_vars.size());
      oa.bytes.resize(X.role_vars.size());
      for (size_t r = 0; r < X.role_vars.size(); ++r)
        for (uint32_t v : X.role_vars[r]) {
          oa.ptr[r].push_back(addr_of(v));
          oa.bytes[r].push_back(vars[v].bytes);
        }
      oa.attrs = f.op.get("attrs");
      oa.ws = ws;
      oa.ws_bytes = ws_bytes;
      oa.stream = fs;
      oa.nccl_comm = nccl_comm;
      oa.nccl_allreduce = nccl_allreduce;
      oa.nccl_group_start = nccl_group_start;
      oa.nccl_group_end = nccl_group_end;
      oa.comm_fn = comm_fn;
      oa.comm_user = comm_user;
      if (opt.timeline) {
        tl_k[i].used = 0;
        oa.ktimer = &tl_k[i];
      }
      Status st = X.op->launch(oa);
      if (!st.good()) {
        st.fn = i;
        st.msg = f.name + ": " + st.msg;
        return st;
      }
      n_kernels += oa.n_kernels;
    }
    if (hook) {
      OC_CUDA(cudaDeviceSynchronize());
      hook(hook_user, i, 1);
    }
    if (opt.timeline) OC_CUDA(cudaEventRecord(tl_fn1[i], fs));
    OC_CUDA(cudaEventRecord(ev_done[i], fs));
    if (on_comm)
      for (uint32_t v : f.out) vars[v].async_fn = (int32_t)i;
    // (c) reserved swap-outs after f_i; small ones through one pack kernel (A7)
    if (!X.dep_reserve.empty()) OC_CUDA(cudaStreamWaitEvent(ds, ev_done[i], 0));
    if (X.pout_n) {
      uint32_t first = X.dep_reserve[0];   // the pack kernel is timed on its first packed departure
      for (uint32_t d : X.dep_reserve)
        if (deps[d].packed) { first = d; break; }
      if (opt.timeline) { OC_CUDA(cudaEventRecord(tl_out0[first], ds)); tl_out_used[first] = 1; }
      OC_TRY(pack_launch(pack_tab + X.pout_off, (int)X.pout_n, ds));
      if (opt.timeline) OC_CUDA(cudaEventRecord(tl_out1[first], ds));
      ++n_d2h;
      ++n_kernels;
      for (uint32_t d : X.dep_reserve)
        if (deps[d].packed) {
          bytes_d2h += vars[deps[d].var].bytes;
          if (opt.timeline) { tl_out_used[d] = 1; tl_out_ref[d] = (int32_t)first; }
        }
    }
    for (uint32_t d : X.dep_reserve) {
      const Dep& D = deps[d];
      XVar& xv = vars[D.var];
      if (D.packed) {
        OC_CUDA(cudaEventRecord(ev_out[d], ds));
        continue;
      }
      cudaStream_t dsk = ds;
      if (D.dirty || !opt.elide_clean) {
        if (opt.timeline) { OC_CUDA(cudaEventRecord(tl_out0[d], dsk)); tl_out_used[d] = 1; }
        OC_CUDA(cudaMemcpyAsync(host + xv.host_off, addr_of(D.var), xv.bytes, cudaMemcpyDeviceToHost, dsk));
        if (opt.timeline) OC_CUDA(cudaEventRecord(tl_out1[d], dsk));
        bytes_d2h += xv.bytes;
        ++n_d2h;
      }
      OC_CUDA(cudaEventRecord(ev_out[d], dsk));
    }
    // frees: nothing to issue; the memory is released at ev_done[i]
    for (uint32_t v : F.free) vars[v].cur_slot = -1;
  }
  for (int32_t d : end_deps) OC_CUDA(cudaStreamWaitEvent(cs, ev_out[d], 0));
  if (comm_s) {   // the step ends when its last gradient exchange has
    OC_CUDA(cudaEventRecord(ev_cjoin, comm_s));
    OC_CUDA(cudaStreamWaitEvent(cs, ev_cjoin, 0));
  }
  return Status::ok();
  };

  if (opt.use_graph && !gexec && step_index >= 1 && !opt.timeline && !hook && !comm_fn) {
    const uint64_t maps_before = mem->n_driver_map;
    OC_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    Status st = issue();
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (!st.good()) return st;
    if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamEndCapture");
    if (mem->n_driver_map != maps_before) return Status::make(OC_E_INVARIANT, "VA mapping changed during capture");
    OC_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
    cudaGraphDestroy(graph);
    g_bytes_h2d = bytes_h2d; g_bytes_d2h = bytes_d2h; g_n_h2d = n_h2d; g_n_d2h = n_d2h; g_n_kernels = n_kernels;
  }
  OC_CUDA(cudaEventRecord(ev_start, cs));
  if (gexec && !hook && !opt.timeline && !comm_fn) {
    OC_CUDA(cudaGraphLaunch(gexec, cs));
    bytes_h2d = g_bytes_h2d; bytes_d2h = g_bytes_d2h; n_h2d = g_n_h2d; n_d2h = g_n_d2h; n_kernels = g_n_kernels;
  } else {
    OC_TRY(issue());
  }
  OC_CUDA(cudaEventRecord(ev_end, cs));
  const double t_host1 = now_ms();
  OC_CUDA(cudaEventSynchronize(ev_end));
  ++step_index;
  if (out) {
    std::memset(out, 0, sizeof(*out));
    float ms = 0;
    OC_CUDA(cudaEventElapsedTime(&ms, ev_start, ev_end));
    out->step_ms = ms;
    out->bytes_h2d = bytes_h2d;
    out->bytes_d2h = bytes_d2h;
    out->n_h2d = n_h2d;
    out->n_d2h = n_d2h;
    out->n_kernels = n_kernels;
    out->host_issue_ms = t_host1 - t_host0;
    out->map_us = mem->map_us - map0;
    out->unmap_us = mem->unmap_us - unmap0;
    if (opt.timeline) {
      std::vector<Interval> C, H, D, T;
      auto iv = [&](cudaEvent_t a, cudaEvent_t b) {
        float x = 0, y = 0;
        cudaEventElapsedTime(&x, ev_start, a);
        cudaEventElapsedTime(&y, ev_start, b);
        return Interval{x, y};
      };
      for (uint32_t i = 0; i < n; ++i)
        if (fns[i].op) C.push_back(iv(tl_fn0[i], tl_fn1[i]));
      // packed transfers share their kernel's events (tl_*_ref); the unions dedupe them
      for (size_t k = 0; k < slots.size(); ++k)
        if (tl_in_used[k]) H.push_back(iv(tl_in0[tl_in_ref[k]], tl_in1[tl_in_ref[k]]));
      for (size_t k = 0; k < deps.size(); ++k)
        if (tl_out_used[k]) D.push_back(iv(tl_out0[tl_out_ref[k]], tl_out1[tl_out_ref[k]]));
      T = H;
      T.insert(T.end(), D.begin(), D.end());
      out->compute_busy_ms = union_len(C);
      out->h2d_busy_ms = union_len(H);
      out->d2h_busy_ms = union_len(D);
      double tl = union_len(T);
      out->overlap_frac = tl > 0 ? inter_len(T, C) / tl : 1.0;
      out->stall_ms = out->step_ms - out->compute_busy_ms;
      (void)cudaGetLastError();   // timing queries are best effort; leave no sticky error behind
    }
  }
  return Status::ok();
}

void Exec::destroy() {
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  for (auto& k : tl_k) k.destroy();
  for (auto& sl : slots) {
    if (sl.span.va) {
      if (!sl.span.mapped.empty()) mem->driver_unmap(sl.span);
      mem->drv->MemAddressFree(sl.span.va, sl.span.m_a);
    }
  }
  auto kill = [](std::vector<cudaEvent_t>& v) { for (auto e : v) if (e) cudaEventDestroy(e); v.clear(); };
  kill(ev_done); kill(ev_in); kill(ev_out);
  kill(tl_fn0); kill(tl_fn1); kill(tl_in0); kill(tl_in1); kill(tl_out0); kill(tl_out1);
  if (ev_start) cudaEventDestroy(ev_start);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (gexec) cudaGraphExecDestroy(gexec);
  if (ev_end) cudaEventDestroy(ev_end);
  host_pool.release();
  host = nullptr;
  if (ws) cudaFree(ws);
  if (pack_tab) cudaFree(pack_tab);
  if (nccl_comm && nccl_destroy) ((int (*)(void*))nccl_destroy)(nccl_comm);
  if (comm_s) cudaStreamDestroy(comm_s);
  if (ev_cfork) cudaEventDestroy(ev_cfork);
  if (ev_cjoin) cudaEventDestroy(ev_cjoin);
}

}  // namespace oc

using namespace oc;

struct oc_exec {
  Exec x;
};

extern "C" {

int oc_exec_create(int device, const oc_graph* g, const oc_schedule* s, oc_mem* m, const oc_streams* st,
                   const oc_exec_options* opt, oc_exec** out, oc_err* err) {
  if (!g || !s || !m || !st || !out) return OC_E_ARG;
  *out = nullptr;
  oc_exec* x = new oc_exec();
  Status r = x->x.create(device, &g->g, &s->s, &m->p, *st, opt);
  if (!r.good()) {
    r.fill(err);
    x->x.destroy();
    delete x;
    return r.code;
  }
  *out = x;
  return OC_OK;
}

int oc_exec_bind_device(oc_exec* x, uint32_t var, void* dev_ptr, oc_err* err) {
  if (!x || var >= x->x.vars.size() || !x->x.vars[var].pinned) {
    Status::make(OC_E_ARG, "oc_exec_bind_device: not a pinned variable").fill(err);
    return OC_E_ARG;
  }
  x->x.vars[var].dev_fixed = dev_ptr;
  return OC_OK;
}

int oc_exec_host_ptr(oc_exec* x, uint32_t var, void** host_ptr, oc_err* err) {
  if (!x || !host_ptr || var >= x->x.vars.size() || x->x.vars[var].host_off < 0) {
    Status::make(OC_E_ARG, "oc_exec_host_ptr: variable has no host copy").fill(err);
    return OC_E_ARG;
  }
  *host_ptr = x->x.host + x->x.vars[var].host_off;
  return OC_OK;
}

int oc_run_step(oc_exec* x, oc_step_metrics* out, oc_err* err) {
  if (!x) return OC_E_ARG;
  Status st = x->x.run(out);
  st.fill(err);
  return st.code;
}

uint64_t oc_graph_workspace_bytes(const oc_graph* g) { return g ? graph_workspace(g->g) : 0; }

int oc_exec_host_info(oc_exec* x, uint64_t* host_bytes, int* numa_node) {
  if (!x) return OC_E_ARG;
  if (host_bytes) *host_bytes = x->x.host_bytes;
  if (numa_node) *numa_node = x->x.host_pool.node;
  return OC_OK;
}

int oc_exec_set_timeline(oc_exec* x, int on) {
  if (!x || (on && !x->x.tl_created)) return OC_E_ARG;
  x->x.opt.timeline = on ? 1 : 0;
  return OC_OK;
}

int oc_exec_set_hook(oc_exec* x, oc_fn_hook hook, void* user) {
  if (!x) return OC_E_ARG;
  x->x.hook = hook;
  x->x.hook_user = user;
  return OC_OK;
}

int oc_exec_read_var(oc_exec* x, uint32_t var, void* host, uint64_t bytes, oc_err* err) {
  if (!x || !host || var >= x->x.vars.size() || bytes > x->x.vars[var].bytes) {
    Status::make(OC_E_ARG, "oc_exec_read_var: unknown variable or size").fill(err);
    return OC_E_ARG;
  }
  void* d = x->x.addr_of(var);
  if (!d) {
    Status e = Status::make(OC_E_ARG, "oc_exec_read_var: variable " + x->x.g->var_names[var] + " is not resident");
    e.var = var;
    e.fill(err);
    return OC_E_ARG;
  }
  cudaSetDevice(x->x.device);
  cudaError_t ce = cudaMemcpy(host, d, bytes, cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) {
    Status s = cuda_status(ce, "oc_exec_read_var");
    s.fill(err);
    return s.code;
  }
  return OC_OK;
}

// the launch probes of f_i's contraction kernels: Σ in-kernel spans and the SM clock
static std::string probe_json(const Exec& X, uint32_t i) {
  if (i >= X.tl_k.size() || !X.tl_k[i].dprobe) return "";
  double span = 0, mhz = 0;
  X.tl_k[i].probe_summary(span, mhz);
  std::ostringstream o;
  o << ",\"k_span_ms\":" << span << ",\"k_mhz\":" << mhz;
  return o.str();
}

int oc_exec_timeline(oc_exec* xh, char* buf, size_t cap, size_t* need) {
  if (!xh) return OC_E_ARG;
  Exec& X = xh->x;
  std::ostringstream o;
  if (X.opt.timeline) {
    auto t = [&](cudaEvent_t e) { float v = 0; cudaEventElapsedTime(&v, X.ev_start, e); return v; };
    for (uint32_t i = 0; i < X.fns.size(); ++i)
      if (X.fns[i].op)
        o << "{\"t0\":" << t(X.tl_fn0[i]) << ",\"t1\":" << t(X.tl_fn1[i]) << ",\"stream\":\"compute\",\"id\":\""
          << X.g->fns[i].name << "\",\"fn\":" << i << ",\"k_ms\":" << (i < X.tl_k.size() ? X.tl_k[i].ms() : 0.0f)
          << ",\"k_n\":" << (i < X.tl_k.size() ? X.tl_k[i].used / 2 : 0) << probe_json(X, i) << "}\n";
    // transfers: "slot" = arrival slot (allocator-replay order), "fn" = the
    // function whose step (a) issued it; departures: "fn" = the function after
    // which the swap-out was reserved (c), "slot" = the slot it leaves;
    // "packed": moved by that function's pack/unpack kernel (one interval)
    for (size_t k = 0; k < X.slots.size(); ++k)
      if (k < X.tl_in_used.size() && X.tl_in_used[k]) {
        const int32_t r = X.tl_in_ref[k];
        o << "{\"t0\":" << t(X.tl_in0[r]) << ",\"t1\":" << t(X.tl_in1[r]) << ",\"stream\":\"h2d\",\"id\":\""
          << X.g->var_names[X.slots[k].var] << "\",\"slot\":" << k << ",\"fn\":" << X.slots[k].fn
          << ",\"packed\":" << (X.slots[k].packed ? 1 : 0) << "}\n";
      }
    for (size_t k = 0; k < X.deps.size(); ++k)
      if (k < X.tl_out_used.size() && X.tl_out_used[k]) {
        const int32_t r = X.tl_out_ref[k];
        o << "{\"t0\":" << t(X.tl_out0[r]) << ",\"t1\":" << t(X.tl_out1[r]) << ",\"stream\":\"d2h\",\"id\":\""
          << X.g->var_names[X.deps[k].var] << "\",\"dep\":" << k << ",\"fn\":" << X.deps[k].fn
          << ",\"slot\":" << X.deps[k].slot << ",\"packed\":" << (X.deps[k].packed ? 1 : 0) << "}\n";
      }
  }
  std::string j = o.str();
  if (need) *need = j.size();
  if (!buf || cap < j.size() + 1) return buf ? OC_E_BUFFER_TOO_SMALL : OC_OK;
  std::memcpy(buf, j.c_str(), j.size() + 1);
  return OC_OK;
}

void oc_exec_destroy(oc_exec* x) {
  if (!x) return;
  x->x.destroy();
  delete x;
}

// ---------------------------------------------------------------- NCCL
typedef struct { char internal[128]; } nccl_uid;
typedef int (*nccl_get_uid_t)(nccl_uid*);
typedef int (*nccl_init_rank_t)(void**, int, nccl_uid, int);

static void* open_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  return h;
}

int oc_nccl_unique_id(void* out, oc_err* err) {
  void* h = open_nccl();
  if (!h || !out) { Status::make(OC_E_NCCL, "libnccl.so.2 not loadable").fill(err); return OC_E_NCCL; }
  auto f = (nccl_get_uid_t)dlsym(h, "ncclGetUniqueId");
  if (!f) { Status::make(OC_E_NCCL, "ncclGetUniqueId missing").fill(err); return OC_E_NCCL; }
  int r = f((nccl_uid*)out);
  if (r) { Status s = Status::make(OC_E_NCCL, "ncclGetUniqueId failed"); s.cuda = r; s.fill(err); return OC_E_NCCL; }
  return OC_OK;
}

int oc_exec_attach_nccl(oc_exec* xh, const void* uid, int rank, int nranks, oc_err* err) {
  if (!xh || !uid) return OC_E_ARG;
  Exec& X = xh->x;
  void* h = open_nccl();
  if (!h) { Status::make(OC_E_NCCL, "libnccl.so.2 not loadable").fill(err); return OC_E_NCCL; }
  auto init = (nccl_init_rank_t)dlsym(h, "ncclCommInitRank");
  X.nccl_allreduce = dlsym(h, "ncclAllReduce");
  X.nccl_destroy = dlsym(h, "ncclCommDestroy");
  X.nccl_group_start = dlsym(h, "ncclGroupStart");
  X.nccl_group_end = dlsym(h, "ncclGroupEnd");
  if (!init || !X.nccl_allreduce) { Status::make(OC_E_NCCL, "NCCL symbols missing").fill(err); return OC_E_NCCL; }
  cudaSetDevice(X.device);
  nccl_uid id;
  std::memcpy(&id, uid, sizeof(id));
  int r = init(&X.nccl_comm, nranks, id, rank);
  if (r) { Status s = Status::make(OC_E_NCCL, "ncclCommInitRank failed"); s.cuda = r; s.fill(err); return OC_E_NCCL; }
  Status st = X.ensure_comm_stream();
  st.fill(err);
  return st.code;
}

int oc_exec_attach_comm(oc_exec* xh, oc_allreduce_fn fn, void* user, oc_err* err) {
  if (!xh || !fn) return OC_E_ARG;
  Exec& X = xh->x;
  X.comm_fn = fn;
  X.comm_user = user;
  Status st = X.ensure_comm_stream();
  st.fill(err);
  return st.code;
}

}  // extern "C"
