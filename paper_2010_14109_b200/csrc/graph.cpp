// Graph document -> validated function-sequence and variable-sequence.
//   P:44  network = DAG of functions, executed f_1..f_n in topological order
//   P:60  v = flatten([V̂_1..V̂_n]), duplicates kept; b_v bytes per variable
//   S:44-65 validation, ordering (ties by smallest index), next_use scan
#include <algorithm>
#include <map>
#include <queue>
#include <set>
#include <unordered_map>

#include "core.hpp"

namespace oc {

static Status invalid(const std::string& m) { return Status::make(OC_E_INVALID, m); }
static Status parse_err(const std::string& m) { return Status::make(OC_E_PARSE, m); }

Status graph_from_json(const char* s, size_t n, Graph& g) {
  JVal doc;
  std::string perr;
  JParser P(s, n);
  if (!P.parse(doc, perr)) return parse_err(perr);
  const JVal* vars = doc.kind == JVal::OBJ ? doc.get("variables") : nullptr;
  const JVal* fns = doc.kind == JVal::OBJ ? doc.get("functions") : nullptr;
  if (!vars || !fns || vars->kind != JVal::ARR || fns->kind != JVal::ARR)
    return parse_err("expected an object with 'variables' and 'functions' lists");
  std::unordered_map<std::string, uint32_t> index;
  for (const JVal& v : vars->arr) {
    const JVal* id = v.kind == JVal::OBJ ? v.get("id") : nullptr;
    if (!id || id->kind != JVal::STR) return parse_err("variable without string id");
    const JVal* b = v.get("bytes");
    if (!b || b->kind != JVal::NUM || !b->is_int) return parse_err("variable " + id->s + ": bytes must be an integer");
    if (index.count(id->s)) return invalid("duplicate variable id " + id->s);
    if (b->i < 1) return invalid("variable " + id->s + ": bytes must be >= 1");
    index[id->s] = (uint32_t)g.var_names.size();
    g.var_names.push_back(id->s);
    g.var_bytes.push_back((uint64_t)b->i);
    g.persistent.push_back(v.getb("persistent") ? 1 : 0);
    g.pinned.push_back(v.getb("pinned") ? 1 : 0);
  }
  std::set<std::string> fn_seen;
  for (const JVal& f : fns->arr) {
    const JVal* id = f.kind == JVal::OBJ ? f.get("id") : nullptr;
    if (!id || id->kind != JVal::STR) return parse_err("function without string id");
    if (fn_seen.count(id->s)) return invalid("duplicate function id " + id->s);
    fn_seen.insert(id->s);
    const JVal* ins = f.get("in");
    const JVal* outs = f.get("out");
    if ((ins && ins->kind != JVal::ARR) || (outs && outs->kind != JVal::ARR))
      return parse_err("function " + id->s + ": in/out must be lists");
    Function fn;
    fn.name = id->s;
    size_t n_in = ins ? ins->arr.size() : 0, n_out = outs ? outs->arr.size() : 0;
    if (n_in + n_out == 0) return invalid("function " + id->s + " uses no variable");
    for (int pass = 0; pass < 2; ++pass) {
      const JVal* lst = pass == 0 ? ins : outs;
      if (!lst) continue;
      std::set<std::string> seen;
      for (const JVal& x : lst->arr) {
        if (x.kind != JVal::STR) return parse_err("function " + id->s + ": variable ids must be strings");
        if (seen.count(x.s)) return invalid("function " + id->s + ": variable repeated in one list");
        seen.insert(x.s);
      }
      for (const JVal& x : lst->arr) {
        auto it = index.find(x.s);
        if (it == index.end()) return invalid("function " + id->s + ": undeclared variable " + x.s);
        (pass == 0 ? fn.in : fn.out).push_back(it->second);
      }
    }
    const JVal* op = f.get("op");
    if (op) fn.op = *op;
    fn.decl = (uint32_t)g.fns.size();
    g.fns.push_back(std::move(fn));
  }
  return graph_finalize(g);
}

// index in `order` of the first function reading a non-persistent, non-pinned
// variable that no earlier function wrote; -1 if none
static int64_t read_before_write(const Graph& g, const std::vector<uint32_t>& order) {
  std::vector<uint8_t> written(g.nv(), 0);
  for (size_t p = 0; p < order.size(); ++p) {
    const Function& f = g.fns[order[p]];
    for (uint32_t v : f.in)
      if (!g.persistent[v] && !g.pinned[v] && !written[v]) return (int64_t)p;
    for (uint32_t v : f.out) written[v] = 1;
  }
  return -1;
}

Status graph_finalize(Graph& g) {
  if (g.finalized) return Status::make(OC_E_ARG, "graph already finalized");
  std::vector<uint8_t> used(g.nv(), 0);
  for (auto& f : g.fns) {
    for (uint32_t v : f.in) used[v] = 1;
    for (uint32_t v : f.out) used[v] = 1;
  }
  for (uint32_t v = 0; v < g.nv(); ++v)
    if (!used[v]) return invalid("variable " + g.var_names[v] + " is used by no function");

  const uint32_t n = g.nf();
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  if (read_before_write(g, order) >= 0) {
    // Kahn over writer -> reader edges, smallest listed index first
    std::vector<int64_t> writer(g.nv(), -1);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t v : g.fns[i].out) {
        if (writer[v] >= 0) return invalid("listed order reads before write and a variable has several writers");
        writer[v] = i;
      }
    std::vector<std::set<uint32_t>> succ(n);
    std::vector<uint32_t> indeg(n, 0);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t v : g.fns[i].in)
        if (writer[v] >= 0 && (uint32_t)writer[v] != i && succ[writer[v]].insert(i).second) ++indeg[i];
    std::priority_queue<uint32_t, std::vector<uint32_t>, std::greater<uint32_t>> ready;
    for (uint32_t i = 0; i < n; ++i)
      if (!indeg[i]) ready.push(i);
    order.clear();
    while (!ready.empty()) {
      uint32_t i = ready.top();
      ready.pop();
      order.push_back(i);
      for (uint32_t j : succ[i])
        if (--indeg[j] == 0) ready.push(j);
    }
    if (order.size() != n) return invalid("cycle in the function graph");
    if (read_before_write(g, order) >= 0) return invalid("a variable is read but never written and is not persistent");
  }
  std::vector<Function> fns(n);
  g.decl_to_pos.assign(n, 0);
  for (uint32_t p = 0; p < n; ++p) {
    fns[p] = std::move(g.fns[order[p]]);
    g.decl_to_pos[fns[p].decl] = p;
  }
  g.fns = std::move(fns);

  // variable-sequence without pinned variables (Z10); next_use scan
  g.occ.clear();
  g.occ_bytes.clear();
  g.l.assign(n, 0);
  g.e.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i) {
    g.l[i] = (int64_t)g.occ.size();
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t v : (pass == 0 ? g.fns[i].in : g.fns[i].out)) {
        if (g.pinned[v]) continue;
        g.occ.push_back(v);
        g.occ_bytes.push_back(g.var_bytes[v]);
      }
    g.e[i] = (int64_t)g.occ.size() - 1;
  }
  g.next_use.assign(g.occ.size(), NONE);
  std::vector<int64_t> last(g.nv(), NONE);
  for (int64_t k = (int64_t)g.occ.size() - 1; k >= 0; --k) {
    g.next_use[k] = last[g.occ[k]];
    last[g.occ[k]] = k;
  }
  g.pinned_bytes = 0;
  for (uint32_t v = 0; v < g.nv(); ++v)
    if (g.pinned[v]) g.pinned_bytes += g.var_bytes[v];
  g.finalized = true;
  return Status::ok();
}

uint64_t graph_in_core_peak(const Graph& g) {
  // live bytes at f_i with allocation at first use and release after last use (Z21)
  std::vector<int64_t> first(g.nv(), -1), last(g.nv(), -1);
  for (uint32_t i = 0; i < g.nf(); ++i)
    for (int pass = 0; pass < 2; ++pass)
      for (uint32_t v : (pass == 0 ? g.fns[i].in : g.fns[i].out)) {
        if (first[v] < 0) first[v] = i;
        last[v] = i;
      }
  std::vector<int64_t> delta(g.nf() + 1, 0);
  for (uint32_t v = 0; v < g.nv(); ++v) {
    if (g.pinned[v] || first[v] < 0) continue;
    delta[first[v]] += (int64_t)g.var_bytes[v];
    delta[last[v] + 1] -= (int64_t)g.var_bytes[v];
  }
  int64_t live = 0, peak = 0;
  for (uint32_t i = 0; i < g.nf(); ++i) {
    live += delta[i];
    peak = std::max(peak, live);
  }
  return (uint64_t)peak + g.pinned_bytes;
}

}  // namespace oc
