"""Oracle: network graph, execution order and variable-sequence.

Follows PAPER.md §2: a network is a DAG of functions executed in a
topological order f_1..f_n; and §3: the variable-sequence
v = flatten([V̂_1, ..., V̂_n]), duplicates kept, each variable with a size
b_v in bytes.

Graph document (JSON, UTF-8) — the same format `oc_graph_from_json` reads
(include/oocore.h):
  {"variables": [{"id": str, "bytes": int>=1, "persistent": bool?, "pinned": bool?}, ...],
   "functions": [{"id": str, "in": [var id...], "out": [var id...], "op": {...}?}, ...]}
V̂_i (the "uses" of f_i) = in + out, in that order ("inputs then
outputs").  A variable listed in both `in` and `out` of one function is an
in-place read-modify-write and contributes two occurrences.

Flags (reading Z10): `persistent` = the variable's authoritative copy lives on
the host between steps (inputs, labels, and — for swappable parameters — the
parameters themselves); it starts on the host with valid data.  `pinned` =
never swapped: it is removed from the variable-sequence and its bytes are
subtracted from the budget.
"""
import json


class GraphError(Exception):
    """Parse or validation failure."""

    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind  # "parse" or "invalid"


class Graph:
    """Validated graph.  Variables and functions are indexed by declaration
    order; that index is the `id` used in the canonical schedule JSON."""

    def __init__(self, var_names, var_bytes, persistent, pinned, fn_names, fn_in, fn_out, fn_op):
        self.var_names = var_names
        self.var_bytes = var_bytes
        self.persistent = persistent
        self.pinned = pinned
        self.fn_names = fn_names
        self.fn_in = fn_in
        self.fn_out = fn_out
        self.fn_op = fn_op

    @property
    def n_vars(self):
        return len(self.var_names)

    @property
    def n_fns(self):
        return len(self.fn_names)

    def uses(self, i):
        """V̂_i as an ordered list with duplicates: inputs then outputs."""
        return list(self.fn_in[i]) + list(self.fn_out[i])


def load_graph(text):
    """Parse and validate a graph document."""
    try:
        doc = json.loads(text)
    except (ValueError, TypeError) as e:
        raise GraphError("parse", str(e))
    if not isinstance(doc, dict) or not isinstance(doc.get("variables"), list) \
            or not isinstance(doc.get("functions"), list):
        raise GraphError("parse", "expected an object with 'variables' and 'functions' lists")

    var_names, var_bytes, persistent, pinned = [], [], [], []
    index = {}
    for v in doc["variables"]:
        if not isinstance(v, dict) or not isinstance(v.get("id"), str):
            raise GraphError("parse", "variable without string id")
        b = v.get("bytes")
        if not isinstance(b, int) or isinstance(b, bool):
            raise GraphError("parse", f"variable {v['id']}: bytes must be an integer")
        if v["id"] in index:
            raise GraphError("invalid", f"duplicate variable id {v['id']}")
        if b < 1:
            raise GraphError("invalid", f"variable {v['id']}: bytes must be >= 1")
        index[v["id"]] = len(var_names)
        var_names.append(v["id"])
        var_bytes.append(b)
        persistent.append(bool(v.get("persistent", False)))
        pinned.append(bool(v.get("pinned", False)))

    fn_names, fn_in, fn_out, fn_op = [], [], [], []
    fn_seen = set()
    for f in doc["functions"]:
        if not isinstance(f, dict) or not isinstance(f.get("id"), str):
            raise GraphError("parse", "function without string id")
        if f["id"] in fn_seen:
            raise GraphError("invalid", f"duplicate function id {f['id']}")
        fn_seen.add(f["id"])
        ins, outs = f.get("in", []), f.get("out", [])
        if not isinstance(ins, list) or not isinstance(outs, list):
            raise GraphError("parse", f"function {f['id']}: in/out must be lists")
        if len(ins) + len(outs) == 0:
            raise GraphError("invalid", f"function {f['id']} uses no variable")
        for lst in (ins, outs):
            if len(set(lst)) != len(lst):
                raise GraphError("invalid", f"function {f['id']}: variable repeated in one list")
            for vid in lst:
                if vid not in index:
                    raise GraphError("invalid", f"function {f['id']}: undeclared variable {vid}")
        fn_names.append(f["id"])
        fn_in.append([index[x] for x in ins])
        fn_out.append([index[x] for x in outs])
        fn_op.append(f.get("op"))

    used = set()
    for i in range(len(fn_names)):
        used.update(fn_in[i])
        used.update(fn_out[i])
    for j, name in enumerate(var_names):
        if j not in used:
            raise GraphError("invalid", f"variable {name} is used by no function")

    g = Graph(var_names, var_bytes, persistent, pinned, fn_names, fn_in, fn_out, fn_op)
    order = execution_order(g)
    # Re-index functions in execution order so that f_1..f_n is the list order.
    g = Graph(var_names, var_bytes, persistent, pinned,
              [fn_names[i] for i in order], [fn_in[i] for i in order],
              [fn_out[i] for i in order], [fn_op[i] for i in order])
    return g


def _read_before_write(g, order):
    """Index of the first function in `order` that reads a non-persistent,
    non-pinned variable no earlier function wrote; None if there is none."""
    written = set()
    for pos, i in enumerate(order):
        for v in g.fn_in[i]:
            if not g.persistent[v] and not g.pinned[v] and v not in written:
                return pos
        written.update(g.fn_out[i])
    return None


def execution_order(g):
    """A topological order of the functions ("Through topological
    ordering, we can index all functions in ascending order").

    The listed order is used when it is executable (no read-before-write).
    Otherwise, when every variable has at most one writer, edges run from the
    writer of v to every other function reading v and Kahn's algorithm takes
    the smallest listed index first.  Anything else is invalid."""
    listed = list(range(g.n_fns))
    if _read_before_write(g, listed) is None:
        return listed
    writers = {}
    for i in listed:
        for v in g.fn_out[i]:
            writers.setdefault(v, []).append(i)
    if any(len(w) > 1 for w in writers.values()):
        raise GraphError("invalid", "listed order reads before write and a variable has several writers")
    succ = {i: set() for i in listed}
    indeg = {i: 0 for i in listed}
    for i in listed:
        for v in g.fn_in[i]:
            if v in writers and writers[v][0] != i:
                w = writers[v][0]
                if i not in succ[w]:
                    succ[w].add(i)
                    indeg[i] += 1
    order = []
    ready = sorted(i for i in listed if indeg[i] == 0)
    while ready:
        i = ready.pop(0)
        order.append(i)
        for j in sorted(succ[i]):
            indeg[j] -= 1
            if indeg[j] == 0:
                ready.append(j)
                ready.sort()
    if len(order) != len(listed):
        raise GraphError("invalid", "cycle in the function graph")
    if _read_before_write(g, order) is not None:
        raise GraphError("invalid", "a variable is read but never written and is not persistent")
    return order


class Sequence:
    """The variable-sequence v of P:60 with per-function spans and next_use.

    occ[k]      variable index of occurrence k (pinned variables removed, Z10)
    owner[k]    function index owning occurrence k
    l[i], e[i]  first and last occurrence index of f_i (e[i] = l[i]-1 when
                f_i touches only pinned variables)
    next_use[k] index of the next occurrence of the same variable, or None
    """

    def __init__(self, occ, owner, l, e, next_use):
        self.occ = occ
        self.owner = owner
        self.l = l
        self.e = e
        self.next_use = next_use


def build_sequence(g):
    """v = flatten([V̂_1..V̂_n]); next_use by one backward scan."""
    occ, owner, l, e = [], [], [], []
    for i in range(g.n_fns):
        l.append(len(occ))
        for v in g.uses(i):
            if g.pinned[v]:
                continue
            occ.append(v)
            owner.append(i)
        e.append(len(occ) - 1)
    next_use = [None] * len(occ)
    last_seen = {}
    for k in range(len(occ) - 1, -1, -1):
        next_use[k] = last_seen.get(occ[k])
        last_seen[occ[k]] = k
    return Sequence(occ, owner, l, e, next_use)


def footprint_stats(g):
    """total bytes of distinct variables, and max_i bytes(distinct V̂_i)."""
    total = sum(g.var_bytes)
    max_fn = max(sum(g.var_bytes[v] for v in set(g.uses(i))) for i in range(g.n_fns))
    return {"total_bytes": total, "max_function_bytes": max_fn}


def in_core_peak(g):
    """F_peak (reading Z21): peak over functions of the bytes of variables
    live at f_i when every variable is allocated at its first use and freed
    after its last use, no swapping; pinned variables count throughout."""
    first, last = {}, {}
    for i in range(g.n_fns):
        for v in g.uses(i):
            first.setdefault(v, i)
            last[v] = i
    pinned = sum(b for v, b in enumerate(g.var_bytes) if g.pinned[v])
    peak = 0
    for i in range(g.n_fns):
        live = sum(g.var_bytes[v] for v in first
                   if not g.pinned[v] and first[v] <= i <= last[v])
        peak = max(peak, live + pinned)
    return peak
