"""Oracle: exhaustive search over all swap schedules of a tiny graph.

P:62: "At each function, we must consider which variables are on GPU.
Therefore, the entire search space can be represented as
O(Π_i 2^{|V \\ V'_i|})" — this module enumerates exactly that space: the
resident set S_i ⊇ V̂_i held on the device while f_i runs, for every i, and
takes the cheapest sequence by dynamic programming over (S_i, dirty bits).

Cost model (the same bytes the greedy's stats count):
  * a variable entering S costs b_v if its data exists (persistent, or
    produced by an earlier function) — an H2D copy; 0 otherwise (alloc only);
  * a variable leaving S costs b_v if it is dirty (written since its host
    copy was last valid) and still needed (used later, or persistent) — a D2H
    copy; 0 otherwise (dropped);
  * after f_n every dirty persistent variable is written back.
Constraint: bytes(S_i) + pinned bytes <= B for every i ("doesn't exceed
the physical GPU memory budget").

Limits: <= 7 non-pinned variables, <= 8 functions.
"""
from itertools import combinations

INF = float("inf")


def _subsets_containing(base, universe):
    rest = [v for v in universe if v not in base]
    for k in range(len(rest) + 1):
        for extra in combinations(rest, k):
            yield frozenset(base) | frozenset(extra)


def optimal_cost(g, budget):
    """Minimum transfer bytes over all schedules at budget B, or None if no
    schedule fits the budget."""
    vars_ = [v for v in range(g.n_vars) if not g.pinned[v]]
    if len(vars_) > 7 or g.n_fns > 8:
        raise ValueError("instance exceeds brute-force limits")
    b = g.var_bytes
    pinned = sum(x for v, x in enumerate(b) if g.pinned[v])
    cap = budget - pinned
    n = g.n_fns
    uses = [set(v for v in g.uses(i) if not g.pinned[v]) for i in range(n)]
    later = [set() for _ in range(n + 1)]          # variables used by f_j, j > i
    for i in range(n - 1, -1, -1):
        later[i] = later[i + 1] | uses[i]
    # used after f_i  = later[i+1]
    written_before = [set() for _ in range(n + 1)]  # produced by f_j, j < i
    for i in range(n):
        written_before[i + 1] = written_before[i] | set(v for v in g.fn_out[i] if not g.pinned[v])

    def has_data(v, i):
        return g.persistent[v] or v in written_before[i]

    def needed_after(v, i):
        return v in later[i + 1] or g.persistent[v]

    # state before f_0: nothing resident
    frontier = {(frozenset(), frozenset()): 0}   # (S, dirty) -> cost
    for i in range(n):
        nxt = {}
        for (S, dirty), cost in frontier.items():
            for S2 in _subsets_containing(uses[i], vars_):
                if sum(b[v] for v in S2) > cap:
                    continue
                c = cost
                for v in S - S2:                     # leaves before f_i
                    if v in dirty and needed_after(v, i - 1):
                        c += b[v]
                for v in S2 - S:                     # enters before f_i
                    if has_data(v, i):
                        c += b[v]
                d2 = (dirty & S2) | set(v for v in g.fn_out[i] if not g.pinned[v])
                key = (S2, frozenset(d2))
                if c < nxt.get(key, INF):
                    nxt[key] = c
        frontier = nxt
        if not frontier:
            return None
    best = INF
    for (S, dirty), cost in frontier.items():
        c = cost + sum(b[v] for v in dirty if g.persistent[v])
        best = min(best, c)
    return best


def min_budget_all_schedules(g):
    """Smallest B for which some schedule exists, by scanning B upward."""
    total = sum(g.var_bytes)
    for B in range(0, total + 1):
        if optimal_cost(g, B) is not None:
            return B
    return None


class _Sch:
    """Minimal schedule record in the scheduler's format (for the simulator)."""

    def __init__(self, n):
        self.ins = [[] for _ in range(n)]
        self.wait_out = [[] for _ in range(n)]
        self.reserve_out = [[] for _ in range(n)]
        self.reserve_dirty = [[] for _ in range(n)]
        self.free = [[] for _ in range(n)]
        self.end_wait = []


def _schedule_of(g, seq, sets):
    """The swap schedule realising resident sets S_0..S_{n-1} (S_i held while
    f_i runs): arrivals S_i − S_{i−1} before f_i, ordered by next use;
    departures S_{i−1} − S_i that are still needed (used later, or
    persistent) reserved after their last use (copied if dirty, else
    elidable) and waited before f_i, others dropped; dirty persistent
    variables written back at the end — the same event vocabulary as the
    greedy."""
    n = g.n_fns
    sch = _Sch(n)
    uses = [set(seq.occ[seq.l[i]:seq.e[i] + 1]) for i in range(n)]
    first_occ = {}
    for k, v in enumerate(seq.occ):
        first_occ.setdefault((v, k), k)
    written = set()
    dirty, last_use = {}, {}
    later = [set() for _ in range(n + 1)]           # used by f_j, j >= i
    for i in range(n - 1, -1, -1):
        later[i] = later[i + 1] | uses[i]
    prev = frozenset()
    for i in range(n):
        S = sets[i]
        for v in sorted(prev - S):
            if v in last_use and (v in later[i] or g.persistent[v]):   # still needed: swap out
                sch.reserve_out[last_use[v]].append(v)
                sch.reserve_dirty[last_use[v]].append(bool(dirty.get(v)))
                sch.wait_out[i].append(v)
            dirty.pop(v, None)
            last_use.pop(v, None)

        def next_use(v):
            for j in range(i, n):
                if v in uses[j]:
                    return j
            return n
        for v in sorted(S - prev, key=lambda v: (next_use(v), v)):
            sch.ins[i].append((v, "h2d" if (g.persistent[v] or v in written) else "alloc"))
        for v in uses[i]:
            if not g.pinned[v]:
                last_use[v] = i
        for v in g.fn_out[i]:
            if not g.pinned[v]:
                dirty[v] = True
                written.add(v)
        prev = S
    for v in sorted(prev):
        if g.persistent[v] and dirty.get(v):
            sch.reserve_out[last_use[v]].append(v)
            sch.reserve_dirty[last_use[v]].append(True)
            sch.end_wait.append(v)
    return sch


def optimal_makespan(g, seq, budget, fn_ms, h2d_gbs, d2h_gbs, elide_clean=True):
    """Minimum simulated makespan (oracle/simulator.simulate, the paper's
    boundary semantics) over every sequence of resident sets S_i ⊇ V̂_i with
    bytes(S_i) + pinned <= B (the P:62 search space), or None.  Limits: <= 4
    functions, <= 5 non-pinned variables."""
    from . import simulator
    vars_ = [v for v in range(g.n_vars) if not g.pinned[v]]
    if len(vars_) > 5 or g.n_fns > 4:
        raise ValueError("instance exceeds brute-force limits")
    b = g.var_bytes
    cap = budget - sum(x for v, x in enumerate(b) if g.pinned[v])
    n = g.n_fns
    uses = [set(v for v in seq.occ[seq.l[i]:seq.e[i] + 1] if not g.pinned[v]) for i in range(n)]
    choices = [[S for S in _subsets_containing(uses[i], vars_) if sum(b[v] for v in S) <= cap] for i in range(n)]
    if any(not c for c in choices):
        return None
    best = [INF, None]

    def rec(i, sets):
        if i == n:
            sch = _schedule_of(g, seq, sets)
            m = simulator.simulate(g, seq, sch, fn_ms, h2d_gbs, d2h_gbs, 0.0, 0.0, elide_clean)["makespan_ms"]
            if m < best[0]:
                best[0], best[1] = m, list(sets)
            return
        for S in choices[i]:
            rec(i + 1, sets + [S])

    rec(0, [])
    return best[0]
