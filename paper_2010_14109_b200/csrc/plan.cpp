// Schedule-window planner (§3) and allocator replay (§4).
//
//   window   v[l_i : r_i], r_i = max{r : Σ_{k=l_i..r} b_k ≤ W}, r_i ≥ e_i   (Z1, Z2)
//   (a)      swap-in {v ∈ v[r_{i-1}+1 : r_i] | σ(v) = 1}                      (Fig.2a)
//   (b)      complete the oldest reserved swap-outs while scheduled > budget  (Fig.2b)
//   (c)/(d)  reserve swap-out of V̂_i after f_i; free if never used again;
//            skip if the next use is inside the window; an arrival cancels a
//            pending reservation                                            (P:86c-d)
//   replay   free(wait_out) -> alloc(in) -> f_i -> free(free); end_wait      (Z9)
//            VA: k = ⌈m_r/m_c⌉ chunks from a FIFO pool
//            arena: caching best-/first-fit with segment-local coalescing
#include <algorithm>
#include <deque>
#include <map>
#include <sstream>

#include "core.hpp"

namespace oc {

std::vector<int64_t> window_ends(const Graph& g, uint64_t W) {
  const int64_t N = (int64_t)g.occ.size();
  std::vector<int64_t> r(g.nf());
  int64_t lo = 0, j = 0;  // current sum covers occ[lo .. j-1]
  uint64_t sum = 0;
  for (uint32_t i = 0; i < g.nf(); ++i) {
    const int64_t li = g.l[i];
    if (j < li) { j = li; sum = 0; lo = li; }
    while (lo < li) sum -= g.occ_bytes[lo++];
    while (j < N && g.occ_bytes[j] <= W - sum) sum += g.occ_bytes[j++];
    r[i] = std::max(g.e[i], j - 1);
  }
  return r;
}

// Prior-art window by function count: r_i = e_{min(i+d, n−1)};
// d = 1 is vDNN's prefetch-one-layer-ahead, a fixed d LMS's graph
// distance.  Steps (a)-(c) are unchanged.
std::vector<int64_t> window_ends_distance(const Graph& g, uint32_t d) {
  const uint32_t n = g.nf();
  std::vector<int64_t> r(n);
  for (uint32_t i = 0; i < n; ++i) r[i] = g.e[std::min<uint64_t>((uint64_t)i + d, n - 1)];
  return r;
}

// B_i(W): bytes of the distinct variables in v[l_i : r_i]; both ends move forward
static std::vector<uint64_t> window_bytes(const Graph& g, const std::vector<int64_t>& r) {
  std::vector<uint32_t> cnt(g.nv(), 0);
  std::vector<uint64_t> out(g.nf(), 0);
  int64_t a = 0, b = -1;  // covered occurrence range [a, b]
  uint64_t cur = 0;
  for (uint32_t i = 0; i < g.nf(); ++i) {
    while (a < g.l[i]) {
      if (a <= b && --cnt[g.occ[a]] == 0) cur -= g.var_bytes[g.occ[a]];
      ++a;
    }
    if (b < a - 1) b = a - 1;
    while (b < r[i]) {
      ++b;
      if (cnt[g.occ[b]]++ == 0) cur += g.var_bytes[g.occ[b]];
    }
    out[i] = (r[i] >= g.l[i]) ? cur : 0;
  }
  return out;
}

uint64_t min_feasible_budget(const Graph& g, uint64_t W, uint32_t distance) {
  auto r = distance ? window_ends_distance(g, distance) : window_ends(g, W);
  auto B = window_bytes(g, r);
  uint64_t m = 0;
  for (uint64_t x : B) m = std::max(m, x);
  return m + g.pinned_bytes;
}

Status max_feasible_window(const Graph& g, uint64_t budget, uint64_t& W) {
  if (min_feasible_budget(g, 0) > budget) {
    Status s = Status::make(OC_E_INFEASIBLE_BUDGET, "budget infeasible even at window 0");
    s.needed = min_feasible_budget(g, 0);
    return s;
  }
  uint64_t lo = 0, hi = 0;
  for (uint64_t b : g.occ_bytes) hi += b;
  while (lo < hi) {  // largest W with max_i B_i(W) + pinned <= budget (monotone in W)
    uint64_t mid = lo + (hi - lo + 1) / 2;
    if (min_feasible_budget(g, mid) <= budget) lo = mid;
    else hi = mid - 1;
  }
  W = lo;
  return Status::ok();
}

Status build_schedule(const Graph& g, uint64_t budget, uint64_t W, Schedule& s, uint32_t distance) {
  const uint32_t n = g.nf(), nv = g.nv();
  s.g = &g;
  s.budget = budget;
  s.window = distance ? 0 : W;
  s.distance = distance;
  s.r = distance ? window_ends_distance(g, distance) : window_ends(g, W);
  s.fn.assign(n, FnSchedule());
  s.end_wait.clear();
  // B_s = B − pinned (Z10); may be negative, then the first function fails in (b)
  const int64_t Bs = (int64_t)budget - (int64_t)g.pinned_bytes;

  struct Res { uint32_t fn, var; bool cancelled = false, waited = false, dirty = false; int32_t wait_fn = -1; };
  std::vector<Res> res;
  std::deque<uint32_t> fifo;                 // reservation ids, oldest first
  std::vector<int64_t> pending(nv, -1);      // var -> live reservation id
  std::vector<uint8_t> on_dev(nv, 0), written(nv, 0), host_valid(nv, 0);
  for (uint32_t v = 0; v < nv; ++v) host_valid[v] = g.persistent[v];
  uint64_t R = 0, peak = 0;
  int64_t r_prev = -1;
  std::vector<int64_t> last_in_span(nv, -1);
  std::vector<uint32_t> seen;

  for (uint32_t i = 0; i < n; ++i) {
    FnSchedule& F = s.fn[i];
    // (a) swap-in for the variables entering the window
    for (int64_t k = r_prev + 1; k <= s.r[i]; ++k) {
      const uint32_t v = g.occ[k];
      if (pending[v] >= 0) {
        res[pending[v]].cancelled = true;
        pending[v] = -1;
      } else if (!on_dev[v]) {
        Arrival a;
        a.var = v;
        a.kind = (g.persistent[v] || written[v]) ? ARRIVE_H2D : ARRIVE_ALLOC;
        F.in.push_back(a);
        on_dev[v] = 1;
        R += g.var_bytes[v];
      }
    }
    // (b) complete the oldest reserved swap-outs until the budget holds
    while ((int64_t)R > Bs) {
      while (!fifo.empty() && res[fifo.front()].cancelled) fifo.pop_front();
      if (fifo.empty()) {
        Status st = Status::make(OC_E_INFEASIBLE_BUDGET, "function " + g.fns[i].name + " does not fit the budget");
        st.fn = i;
        std::vector<uint8_t> mark(nv, 0);
        uint64_t need = 0;
        for (int64_t k = g.l[i]; k <= s.r[i]; ++k)
          if (!mark[g.occ[k]]) { mark[g.occ[k]] = 1; need += g.var_bytes[g.occ[k]]; }
        st.needed = need + g.pinned_bytes;
        return st;
      }
      Res& x = res[fifo.front()];
      fifo.pop_front();
      x.waited = true;
      x.wait_fn = (int32_t)i;
      F.wait_out.push_back(x.var);
      pending[x.var] = -1;
      on_dev[x.var] = 0;
      host_valid[x.var] = 1;
      R -= g.var_bytes[x.var];
    }
    peak = std::max(peak, R);
    // f_i runs: its outputs become stale on the host
    for (uint32_t v : g.fns[i].out)
      if (!g.pinned[v]) { written[v] = 1; host_valid[v] = 0; }
    // (c)/(d)
    seen.clear();
    for (int64_t k = g.l[i]; k <= g.e[i]; ++k) {
      const uint32_t v = g.occ[k];
      if (last_in_span[v] < g.l[i]) seen.push_back(v);
      last_in_span[v] = k;  // Z7: the last occurrence inside f_i decides
    }
    for (uint32_t v : seen) {
      const int64_t nx = g.next_use[last_in_span[v]];
      if (nx == NONE) {
        if (g.persistent[v] && !host_valid[v]) {  // write-back of a modified persistent variable
          Res x; x.fn = i; x.var = v; x.dirty = true;
          pending[v] = (int64_t)res.size();
          fifo.push_back((uint32_t)res.size());
          res.push_back(x);
        } else {
          F.free.push_back(v);
          on_dev[v] = 0;
          R -= g.var_bytes[v];
        }
      } else if (nx <= s.r[i]) {
        // already inside the window: stays resident (Fig.2d)
      } else {
        Res x; x.fn = i; x.var = v; x.dirty = !host_valid[v];
        pending[v] = (int64_t)res.size();
        fifo.push_back((uint32_t)res.size());
        res.push_back(x);
      }
    }
    r_prev = s.r[i];
  }
  for (uint32_t id : fifo) {
    if (res[id].cancelled) continue;
    res[id].waited = true;
    res[id].wait_fn = -1;
    s.end_wait.push_back(res[id].var);
  }
  // compaction: only reservations that are eventually waited survive
  s.bytes_h2d = s.bytes_alloc = s.bytes_d2h = s.bytes_d2h_dirty = 0;
  s.n_in_h2d = s.n_in_alloc = s.n_out = s.n_arrivals = 0;
  for (const Res& x : res) {
    if (!x.waited) continue;
    s.fn[x.fn].reserve_out.push_back(Departure{x.var, (uint8_t)x.dirty, x.wait_fn});
    s.bytes_d2h += g.var_bytes[x.var];
    if (x.dirty) s.bytes_d2h_dirty += g.var_bytes[x.var];
    ++s.n_out;
  }
  for (auto& F : s.fn)
    for (auto& a : F.in) {
      a.slot = s.n_arrivals++;
      if (a.kind == ARRIVE_H2D) { s.bytes_h2d += g.var_bytes[a.var]; ++s.n_in_h2d; }
      else { s.bytes_alloc += g.var_bytes[a.var]; ++s.n_in_alloc; }
    }
  s.peak_sched = peak + g.pinned_bytes;
  return Status::ok();
}

// ------------------------------------------------------------- allocators

namespace {

struct VAModel {
  uint64_t m_c;
  uint32_t n_chunks;
  std::deque<uint32_t> free_q;
  std::map<uint32_t, std::pair<uint64_t, std::vector<uint32_t>>> live;  // var -> (m_r, chunks)
  uint64_t live_if = 0;
  ReplayStats* st;
  bool alloc(uint32_t var, uint64_t m_r, std::vector<uint32_t>& chunks) {
    uint64_t k = (m_r + m_c - 1) / m_c;  // k = ⌈m_r/m_c⌉ (Eq.1)
    if (free_q.size() < k) return false;
    chunks.assign(free_q.begin(), free_q.begin() + k);
    free_q.erase(free_q.begin(), free_q.begin() + k);
    live[var] = {m_r, chunks};
    live_if += k * m_c - m_r;
    uint64_t mapped = n_chunks - free_q.size();
    st->peak_phys = std::max(st->peak_phys, mapped * m_c);
    st->if_peak = std::max(st->if_peak, live_if);
    st->n_max = std::max<uint32_t>(st->n_max, (uint32_t)live.size());
    return true;
  }
  void free(uint32_t var) {
    auto it = live.find(var);
    live_if -= it->second.second.size() * m_c - it->second.first;
    for (uint32_t c : it->second.second) free_q.push_back(c);
    live.erase(it);
  }
  uint64_t free_bytes() const { return free_q.size() * m_c; }
};

}  // namespace

bool ArenaPlacer::alloc(uint64_t key, uint64_t m_r, uint64_t& off) {
  const uint64_t s = (m_r + align - 1) / align * align;
  int64_t pick = -1;
  for (size_t b = 0; b < blocks.size(); ++b) {
    if (!blocks[b].free || blocks[b].size < s) continue;
    if (pick < 0) { pick = (int64_t)b; if (!best) break; continue; }
    if (blocks[b].size < blocks[pick].size) pick = (int64_t)b;  // ties keep the lower address
  }
  if (pick >= 0) {
    Blk& B = blocks[pick];
    if (B.size > s) {  // split: the remainder stays cached in the same segment
      Blk rest{B.start + s, B.size - s, B.seg, true};
      B.size = s;
      blocks.insert(blocks.begin() + pick + 1, rest);
    }
    blocks[pick].free = false;
    off = blocks[pick].start;
  } else if (cap - tail >= s) {  // carve a new segment from the untouched tail
    blocks.push_back(Blk{tail, s, tail, false});
    off = tail;
    tail += s;
  } else {
    return false;  // external fragmentation when free_bytes() >= s
  }
  live[key] = off;
  allocated += s;
  return true;
}

uint64_t ArenaPlacer::free(uint64_t key) {
  const uint64_t off = live[key];
  live.erase(key);
  size_t b = 0;
  while (blocks[b].start != off) ++b;
  blocks[b].free = true;
  const uint64_t sz = blocks[b].size;
  allocated -= sz;
  // coalesce only with address-adjacent free blocks of the same segment
  if (b + 1 < blocks.size() && blocks[b + 1].free && blocks[b + 1].seg == blocks[b].seg) {
    blocks[b].size += blocks[b + 1].size;
    blocks.erase(blocks.begin() + b + 1);
  }
  if (b > 0 && blocks[b - 1].free && blocks[b - 1].seg == blocks[b].seg) {
    blocks[b - 1].size += blocks[b].size;
    blocks.erase(blocks.begin() + b);
  }
  return sz;
}

uint64_t ArenaPlacer::free_bytes() const {
  uint64_t f = cap - tail;
  for (auto& B : blocks)
    if (B.free) f += B.size;
  return f;
}

Status replay_allocator(const Graph& g, Schedule& s) {
  s.replay = ReplayStats();
  ReplayStats& st = s.replay;
  const oc_alloc_model& am = s.alloc;
  uint64_t phys = am.phys_bytes ? am.phys_bytes : (s.budget - g.pinned_bytes);
  VAModel va{};
  ArenaPlacer ar;
  const bool is_va = am.mode == OC_ALLOC_VA;
  if (is_va) {
    if (am.chunk_bytes == 0) return Status::make(OC_E_ARG, "chunk_bytes must be > 0");
    va.m_c = am.chunk_bytes;
    va.n_chunks = (uint32_t)(phys / am.chunk_bytes);
    for (uint32_t c = 0; c < va.n_chunks; ++c) va.free_q.push_back(c);
    va.st = &st;
  } else if (am.mode == OC_ALLOC_ARENA_BEST || am.mode == OC_ALLOC_ARENA_FIRST) {
    ar.init(phys, am.align ? am.align : 512, am.mode == OC_ALLOC_ARENA_BEST);
  } else {
    return Status::make(OC_E_ARG, "unknown allocator mode");
  }
  auto do_free = [&](uint32_t v) { if (is_va) va.free(v); else ar.free(v); };
  for (uint32_t i = 0; i < g.nf(); ++i) {
    FnSchedule& F = s.fn[i];
    for (uint32_t v : F.wait_out) do_free(v);
    for (Arrival& a : F.in) {
      bool ok = is_va ? va.alloc(a.var, g.var_bytes[a.var], a.chunks) : ar.alloc(a.var, g.var_bytes[a.var], a.offset);
      if (ok && !is_va) {
        st.peak_alloc = std::max(st.peak_alloc, ar.allocated);
        st.peak_phys = std::max(st.peak_phys, ar.tail);
      }
      if (!ok) {
        st.oom_fn = (int32_t)i;
        st.oom_var = (int32_t)a.var;
        st.oom_request = g.var_bytes[a.var];
        st.oom_free = is_va ? va.free_bytes() : ar.free_bytes();
        Status e = Status::make(OC_E_DEVICE_OOM, "allocator replay: " + g.var_names[a.var] + " does not fit at " + g.fns[i].name);
        e.fn = i;
        e.var = a.var;
        e.needed = st.oom_request;
        e.free_bytes = st.oom_free;
        return e;
      }
    }
    for (uint32_t v : F.free) do_free(v);
  }
  for (uint32_t v : s.end_wait) do_free(v);
  if (is_va) st.peak_alloc = st.peak_phys;
  return Status::ok();
}

std::string schedule_json(const Schedule& s) {
  std::ostringstream o;
  o << "{\"v\":1,\"budget\":" << s.budget << ",\"window\":" << s.window;
  if (s.distance) o << ",\"distance\":" << s.distance;
  o << ",\"fn\":[";
  for (size_t i = 0; i < s.fn.size(); ++i) {
    const FnSchedule& F = s.fn[i];
    if (i) o << ',';
    o << "{\"in\":[";
    for (size_t k = 0; k < F.in.size(); ++k)
      o << (k ? "," : "") << '[' << F.in[k].var << ",\"" << (F.in[k].kind == ARRIVE_H2D ? "h2d" : "alloc") << "\"]";
    o << "],\"wait_out\":[";
    for (size_t k = 0; k < F.wait_out.size(); ++k) o << (k ? "," : "") << F.wait_out[k];
    o << "],\"reserve_out\":[";
    for (size_t k = 0; k < F.reserve_out.size(); ++k) o << (k ? "," : "") << F.reserve_out[k].var;
    o << "],\"free\":[";
    for (size_t k = 0; k < F.free.size(); ++k) o << (k ? "," : "") << F.free[k];
    o << "]}";
  }
  o << "],\"end_wait\":[";
  for (size_t k = 0; k < s.end_wait.size(); ++k) o << (k ? "," : "") << s.end_wait[k];
  o << "],\"stats\":{\"bytes_h2d\":" << s.bytes_h2d << ",\"bytes_alloc\":" << s.bytes_alloc
    << ",\"bytes_d2h\":" << s.bytes_d2h << ",\"bytes_d2h_clean_elided\":" << s.bytes_d2h_dirty
    << ",\"peak_sched\":" << s.peak_sched << "}}";
  return o.str();
}

}  // namespace oc
