// extern "C" surface of the host-side part of liboocore (graph, planning).
// See include/oocore.h for the contract of each call.
#include <algorithm>
#include <cstring>
#include <new>

#include "core.hpp"

using namespace oc;

extern "C" {

const char* oc_strerror(int code) {
  switch (code) {
    case OC_OK: return "ok";
    case OC_E_PARSE: return "parse error";
    case OC_E_INVALID: return "invalid graph";
    case OC_E_INFEASIBLE_BUDGET: return "infeasible budget";
    case OC_E_DEVICE_OOM: return "device out of memory";
    case OC_E_UNKNOWN_HANDLE: return "unknown handle";
    case OC_E_DOUBLE_FREE: return "double free";
    case OC_E_CUDA: return "CUDA error";
    case OC_E_BUFFER_TOO_SMALL: return "buffer too small";
    case OC_E_INVARIANT: return "invariant violated";
    case OC_E_ARG: return "bad argument";
    case OC_E_UNSUPPORTED: return "unsupported";
    case OC_E_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

int oc_abi_version(void) { return OC_ABI_VERSION; }

int oc_graph_from_json(const char* utf8, size_t len, oc_graph** out, oc_err* err) {
  if (!utf8 || !out) { Status::make(OC_E_ARG, "null argument").fill(err); return OC_E_ARG; }
  *out = nullptr;
  oc_graph* h = new (std::nothrow) oc_graph();
  if (!h) return OC_E_ARG;
  Status st = graph_from_json(utf8, len, h->g);
  if (!st.good()) {
    st.fill(err);
    delete h;
    return st.code;
  }
  *out = h;
  return OC_OK;
}

int oc_graph_create(oc_graph** out) {
  if (!out) return OC_E_ARG;
  *out = new (std::nothrow) oc_graph();
  return *out ? OC_OK : OC_E_ARG;
}

int oc_graph_add_var(oc_graph* h, const char* name, uint64_t bytes, uint32_t flags, uint32_t* id) {
  if (!h || !name || h->g.finalized) return OC_E_ARG;
  if (bytes < 1) return OC_E_INVALID;
  for (auto& n : h->g.var_names)
    if (n == name) return OC_E_INVALID;
  if (id) *id = h->g.nv();
  h->g.var_names.push_back(name);
  h->g.var_bytes.push_back(bytes);
  h->g.persistent.push_back((flags & OC_VAR_PERSISTENT) ? 1 : 0);
  h->g.pinned.push_back((flags & OC_VAR_PINNED) ? 1 : 0);
  return OC_OK;
}

int oc_graph_add_fn(oc_graph* h, const char* name, const uint32_t* in, uint32_t n_in, const uint32_t* out,
                    uint32_t n_out, const char* op_json, uint32_t* id) {
  if (!h || !name || h->g.finalized || (n_in && !in) || (n_out && !out)) return OC_E_ARG;
  if (n_in + n_out == 0) return OC_E_INVALID;
  for (auto& f : h->g.fns)
    if (f.name == name) return OC_E_INVALID;
  Function f;
  f.name = name;
  for (uint32_t k = 0; k < n_in; ++k) {
    if (in[k] >= h->g.nv() || std::count(in, in + k, in[k])) return OC_E_INVALID;
    f.in.push_back(in[k]);
  }
  for (uint32_t k = 0; k < n_out; ++k) {
    if (out[k] >= h->g.nv() || std::count(out, out + k, out[k])) return OC_E_INVALID;
    f.out.push_back(out[k]);
  }
  if (op_json && *op_json) {
    std::string perr;
    JParser P(op_json, std::strlen(op_json));
    if (!P.parse(f.op, perr)) return OC_E_PARSE;
  }
  f.decl = h->g.nf();
  if (id) *id = f.decl;
  h->g.fns.push_back(std::move(f));
  return OC_OK;
}

int oc_graph_finalize(oc_graph* h, oc_err* err) {
  if (!h) return OC_E_ARG;
  Status st = graph_finalize(h->g);
  st.fill(err);
  return st.code;
}

void oc_graph_destroy(oc_graph* h) { delete h; }

uint32_t oc_graph_num_vars(const oc_graph* h) { return h ? h->g.nv() : 0; }
uint32_t oc_graph_num_fns(const oc_graph* h) { return h ? h->g.nf() : 0; }
uint64_t oc_graph_var_bytes(const oc_graph* h, uint32_t v) {
  return (h && v < h->g.nv()) ? h->g.var_bytes[v] : 0;
}
uint32_t oc_graph_fn_position(const oc_graph* h, uint32_t d) {
  return (h && d < h->g.decl_to_pos.size()) ? h->g.decl_to_pos[d] : UINT32_MAX;
}
uint64_t oc_graph_in_core_peak(const oc_graph* h) { return h ? graph_in_core_peak(h->g) : 0; }

void oc_graph_footprint(const oc_graph* h, uint64_t* total, uint64_t* max_fn) {
  if (!h) return;
  const Graph& g = h->g;
  uint64_t t = 0, m = 0;
  for (uint64_t b : g.var_bytes) t += b;
  std::vector<uint32_t> mark(g.nv(), UINT32_MAX);
  for (uint32_t i = 0; i < g.nf(); ++i) {
    uint64_t s = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t v : (pass == 0 ? g.fns[i].in : g.fns[i].out))
        if (mark[v] != i) { mark[v] = i; s += g.var_bytes[v]; }
    m = std::max(m, s);
  }
  if (total) *total = t;
  if (max_fn) *max_fn = m;
}

int oc_plan_schedule(const oc_graph* h, const oc_plan_params* p, oc_schedule** out, oc_err* err) {
  if (!h || !p || !out || !h->g.finalized) { Status::make(OC_E_ARG, "null or unfinalized").fill(err); return OC_E_ARG; }
  *out = nullptr;
  uint64_t W = p->window_bytes;
  if (p->distance) W = 0;
  else if (W == OC_WINDOW_MAX_FEASIBLE) {
    Status st = max_feasible_window(h->g, p->budget_bytes, W);
    if (!st.good()) { st.fill(err); return st.code; }
  }
  oc_schedule* s = new (std::nothrow) oc_schedule();
  if (!s) return OC_E_ARG;
  s->owner = h;
  s->s.alloc = p->alloc;
  Status st = build_schedule(h->g, p->budget_bytes, W, s->s, p->distance);
  if (!st.good()) {
    st.fill(err);
    delete s;
    return st.code;
  }
  st = replay_allocator(h->g, s->s);
  *out = s;
  st.fill(err);
  return st.code;
}

void oc_schedule_destroy(oc_schedule* s) { delete s; }

uint64_t oc_min_feasible_budget(const oc_graph* h, uint64_t window) {
  return h ? min_feasible_budget(h->g, window) : 0;
}

uint64_t oc_min_feasible_budget_distance(const oc_graph* h, uint32_t distance) {
  return (h && distance) ? min_feasible_budget(h->g, 0, distance) : 0;
}

int oc_max_feasible_window(const oc_graph* h, uint64_t budget, uint64_t* window, oc_err* err) {
  if (!h || !window) return OC_E_ARG;
  Status st = max_feasible_window(h->g, budget, *window);
  st.fill(err);
  return st.code;
}

int oc_schedule_json(const oc_schedule* s, char* buf, size_t cap, size_t* need) {
  if (!s) return OC_E_ARG;
  std::string j = schedule_json(s->s);
  if (need) *need = j.size();
  if (!buf || cap < j.size() + 1) return buf ? OC_E_BUFFER_TOO_SMALL : OC_OK;
  std::memcpy(buf, j.c_str(), j.size() + 1);
  return OC_OK;
}

int oc_schedule_stats(const oc_schedule* h, oc_sched_stats* o) {
  if (!h || !o) return OC_E_ARG;
  const Schedule& s = h->s;
  std::memset(o, 0, sizeof(*o));
  o->budget = s.budget;
  o->window = s.window;
  o->bytes_h2d = s.bytes_h2d;
  o->bytes_alloc = s.bytes_alloc;
  o->bytes_d2h = s.bytes_d2h;
  o->bytes_d2h_dirty = s.bytes_d2h_dirty;
  o->peak_sched = s.peak_sched;
  o->pinned_bytes = h->owner->g.pinned_bytes;
  o->peak_phys = s.replay.peak_phys;
  o->peak_alloc = s.replay.peak_alloc;
  o->if_peak = s.replay.if_peak;
  o->n_max = s.replay.n_max;
  o->oom_fn = s.replay.oom_fn;
  o->oom_var = s.replay.oom_var;
  o->oom_request = s.replay.oom_request;
  o->oom_free_bytes = s.replay.oom_free;
  o->n_in_h2d = s.n_in_h2d;
  o->n_in_alloc = s.n_in_alloc;
  o->n_out = s.n_out;
  o->n_fns = (uint32_t)s.fn.size();
  return OC_OK;
}

int oc_schedule_window_ends(const oc_schedule* s, int64_t* r, size_t n) {
  if (!s || !r || n < s->s.r.size()) return OC_E_ARG;
  std::copy(s->s.r.begin(), s->s.r.end(), r);
  return OC_OK;
}

// oracle/simulator.py, operation for operation (float64, same order)
int oc_simulate(const oc_schedule* sh, const double* fn_ms, size_t n, const oc_link_model* link, oc_sim_result* out,
                double* stall_ms) {
  if (!sh || !fn_ms || !link || !out || link->h2d_gbs <= 0 || link->d2h_gbs <= 0) return OC_E_ARG;
  const Schedule& s = sh->s;
  const Graph& g = *s.g;
  if (n != s.fn.size()) return OC_E_ARG;
  std::vector<double> ready(g.nv(), 0.0), out_done(g.nv(), 0.0);
  double h2d_free = 0.0, d2h_free = 0.0, end_prev = 0.0;
  oc_sim_result r{};
  if (link->model == 1) {
    // executor ordering (oracle/simulator.simulate_exec)
    const bool va = s.alloc.mode == OC_ALLOC_VA;
    const uint64_t al = s.alloc.align ? s.alloc.align : 1;
    std::vector<double> rel_chunk;
    struct Iv { uint64_t lo, hi; double t; };
    std::vector<Iv> rel_iv;
    std::vector<const Arrival*> held(g.nv(), nullptr);
    std::vector<double> host_ready(g.nv(), 0.0);
    auto range_of = [&](const Arrival& a) {
      const uint64_t size = (g.var_bytes[a.var] + al - 1) / al * al;
      return std::make_pair(a.offset, a.offset + size);
    };
    auto mem_ready = [&](const Arrival& a) {
      double t = 0.0;
      if (va) {
        for (uint32_t c : a.chunks)
          if (c < rel_chunk.size()) t = std::max(t, rel_chunk[c]);
      } else {
        const auto rg = range_of(a);
        for (const Iv& iv : rel_iv)
          if (iv.lo < rg.second && rg.first < iv.hi) t = std::max(t, iv.t);
      }
      return t;
    };
    auto release = [&](const Arrival* a, double t) {
      if (!a) return;
      if (va) {
        for (uint32_t c : a->chunks) {
          if (c >= rel_chunk.size()) rel_chunk.resize(c + 1, 0.0);
          rel_chunk[c] = t;
        }
      } else {
        const auto rg = range_of(*a);
        rel_iv.push_back(Iv{rg.first, rg.second, t});
      }
    };
    for (size_t i = 0; i < n; ++i) {
      const FnSchedule& F = s.fn[i];
      double t_wait = 0.0;
      for (uint32_t v : F.wait_out) {
        t_wait = std::max(t_wait, out_done[v]);
        release(held[v], out_done[v]);
        held[v] = nullptr;
      }
      for (const Arrival& a : F.in) {
        double t = std::max(h2d_free, mem_ready(a));
        if (a.kind == ARRIVE_H2D) {
          t = std::max(t, host_ready[a.var]);
          const double dur = link->h2d_fixed_us * 1e-3 + (double)g.var_bytes[a.var] / (link->h2d_gbs * 1e6);
          t = t + dur;
          r.h2d_busy_ms += dur;
        }
        h2d_free = t;
        ready[a.var] = t;
        held[a.var] = &a;
      }
      double need = 0.0;
      for (int64_t k = g.l[i]; k <= g.e[i]; ++k) {
        const uint32_t v = g.occ[k];
        if (!g.pinned[v]) need = std::max(need, ready[v]);
      }
      const double start = std::max(std::max(end_prev, t_wait), need);
      if (stall_ms) stall_ms[i] = start - end_prev;
      r.stall_ms += start - end_prev;
      const double end = start + fn_ms[i];
      r.compute_ms += fn_ms[i];
      for (const Departure& d : F.reserve_out) {
        double t = std::max(d2h_free, end);
        if (d.dirty || !link->elide_clean) {
          const double dur = link->d2h_fixed_us * 1e-3 + (double)g.var_bytes[d.var] / (link->d2h_gbs * 1e6);
          t = t + dur;
          r.d2h_busy_ms += dur;
          host_ready[d.var] = t;
        }
        d2h_free = t;
        out_done[d.var] = t;
      }
      for (uint32_t v : F.free) {
        release(held[v], end);
        held[v] = nullptr;
      }
      end_prev = end;
    }
    double makespan = end_prev;
    for (uint32_t v : s.end_wait) makespan = std::max(makespan, out_done[v]);
    r.makespan_ms = makespan;
    *out = r;
    return OC_OK;
  }
  for (size_t i = 0; i < n; ++i) {
    const FnSchedule& F = s.fn[i];
    double t_wait = 0.0;
    for (uint32_t v : F.wait_out) t_wait = std::max(t_wait, out_done[v]);
    const double t_trig = std::max(end_prev, t_wait);
    for (const Arrival& a : F.in) {
      if (a.kind == ARRIVE_H2D) {
        const double start = std::max(h2d_free, t_trig);
        const double dur = link->h2d_fixed_us * 1e-3 + (double)g.var_bytes[a.var] / (link->h2d_gbs * 1e6);
        h2d_free = start + dur;
        r.h2d_busy_ms += dur;
        ready[a.var] = h2d_free;
      } else {
        ready[a.var] = t_trig;
      }
    }
    double need = 0.0;
    for (int64_t k = g.l[i]; k <= g.e[i]; ++k) {
      const uint32_t v = g.occ[k];
      if (!g.pinned[v]) need = std::max(need, ready[v]);
    }
    const double start = std::max(std::max(end_prev, t_wait), need);
    if (stall_ms) stall_ms[i] = start - end_prev;
    r.stall_ms += start - end_prev;
    const double end = start + fn_ms[i];
    r.compute_ms += fn_ms[i];
    for (const Departure& d : F.reserve_out) {
      if (link->elide_clean && !d.dirty) {
        out_done[d.var] = end;
        continue;
      }
      const double s0 = std::max(d2h_free, end);
      const double dur = link->d2h_fixed_us * 1e-3 + (double)g.var_bytes[d.var] / (link->d2h_gbs * 1e6);
      d2h_free = s0 + dur;
      r.d2h_busy_ms += dur;
      out_done[d.var] = d2h_free;
    }
    end_prev = end;
  }
  double makespan = end_prev;
  for (uint32_t v : s.end_wait) makespan = std::max(makespan, out_done[v]);
  r.makespan_ms = makespan;
  *out = r;
  return OC_OK;
}

}  // extern "C"
