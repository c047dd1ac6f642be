"""Oracle: the paper's schedule-window greedy (§3).

Straight-line restatement of the algorithm, in the paper's order and notation:

  window at f_i:  v[l:r], l = first occurrence of V̂_i, r = the maximum index
                  with  Σ_{k=l..r} b_{v_k} ≤ schedule-window
                  floored at the end of f_i's own span (reading Z2)
  step (a)        schedule Swap-in for {v ∈ v[r⁻+1 : r] | σ(v) = 1}       (Fig.2a)
  step (b)        complete previously scheduled Swap-outs, oldest first,
                  until the budget holds; the waits go before f_i         (Fig.2b)
  step (c)        reserve Swap-out for V̂_i right after f_i               (Fig.2c)
  step (d)        skip it if the variable is never used again (free) or
                  already inside the window ("already reserved as
                  Swap-in"); a later arrival cancels a pending reservation (P:86d)

Readings of the paper's silences (Z1-Z12) are marked inline.
"""
import json

HOST, DEV = 1, 0  # σ(v) = 1 if v is on the CPU


class InfeasibleBudget(Exception):
    """Step (b) cannot bring the scheduled bytes under the budget."""

    def __init__(self, fn, needed):
        super().__init__(f"InfeasibleBudget at function {fn}: needs {needed} bytes")
        self.fn = fn
        self.needed = needed


def window_ends(seq, window):
    """r_i for every function.  Z1: the sum runs over occurrences,
    duplicates counted.  Z2: r_i >= e_i (the window always covers V̂_i)."""
    b = seq.occ_bytes
    r = []
    for i in range(len(seq.l)):
        li = seq.l[i]
        best = li - 1          # the empty sub-sequence always satisfies the bound
        acc = 0
        k = li
        while k < len(seq.occ):
            acc += b[k]
            if acc > window:
                break
            best = k
            k += 1
        r.append(max(seq.e[i], best))
    return r


def window_ends_distance(seq, distance):
    """Prior-art window of SURVEY §8(f) F1, by function count instead of bytes:
    r_i = e_{min(i+d, n-1)}.  d = 1 is vDNN's "prefetch one layer ahead"
    (P:46); a fixed d is LMS's fixed graph distance.  The rest of
    the sweep — (a) arrivals, (b) oldest-first waits, (c) reservations — is
    unchanged, so only the window rule differs from the paper's method."""
    n = len(seq.l)
    return [seq.e[min(i + distance, n - 1)] for i in range(n)]


def window_bytes(g, seq, window):
    """B_i(W): bytes of the distinct variables in v[l_i : r_i]."""
    r = window_ends(seq, window)
    out = []
    for i in range(len(seq.l)):
        distinct = set(seq.occ[seq.l[i]:r[i] + 1])
        out.append(sum(g.var_bytes[v] for v in distinct))
    return out


def pinned_bytes(g):
    return sum(b for v, b in enumerate(g.var_bytes) if g.pinned[v])


def attach_bytes(g, seq):
    seq.occ_bytes = [g.var_bytes[v] for v in seq.occ]
    return seq


class Schedule:
    def __init__(self, n_fns):
        self.budget = None
        self.window = None
        self.ins = [[] for _ in range(n_fns)]        # (a): [(v, "h2d"|"alloc")]
        self.wait_out = [[] for _ in range(n_fns)]   # (b): waits placed before f_i
        self.reserve_out = [[] for _ in range(n_fns)]  # (c): surviving reservations after f_i
        self.free = [[] for _ in range(n_fns)]       # (d): never used again -> released after f_i
        self.end_wait = []
        self.stats = {}
        self.r = []


def build_schedule(g, seq, budget, window, distance=0):
    """Sweep f_1..f_n performing (a) -> (b) -> (c) at each function.

    `budget` is the physical budget B; pinned variables are resident all step,
    so the scheduler works against B_s = B - Σ pinned (reading Z10).
    distance > 0 replaces the byte window by the prior-art function-distance
    window (window_ends_distance; `window` is then ignored and reported 0)."""
    attach_bytes(g, seq)
    n = len(seq.l)
    b = g.var_bytes
    if distance:
        window = 0
        r = window_ends_distance(seq, distance)
    else:
        r = window_ends(seq, window)
    budget_s = budget - pinned_bytes(g)

    sigma = [HOST] * g.n_vars          # Z4: every variable starts on the host
    written = [False] * g.n_vars       # has f_j (j < i) produced the variable?
    host_valid = [g.persistent[v] for v in range(g.n_vars)]  # host copy up to date
    pend = []                          # FIFO of reservations: [v, fn, id, dirty_at_reserve]
    cancelled = set()                  # reservation ids dropped by a later arrival
    reservations = []                  # (fn, v, id)
    R = 0                              # scheduled resident bytes (Z5)
    peak = 0
    sch = Schedule(n)
    sch.budget, sch.window, sch.r = budget, window, r
    sch.distance = distance
    bytes_h2d = bytes_alloc = 0
    waited = {}                        # reservation id -> dirty_at_reserve (survivors)

    r_prev = -1
    for i in range(n):
        # (a) Swap-in for the new variables coming into the window  (Fig.2a)
        for k in range(r_prev + 1, r[i] + 1):
            v = seq.occ[k]
            hit = [p for p in pend if p[0] == v]
            if hit:
                # "already reserved": the pending Swap-out is cancelled, v stays (P:86d, Z8)
                pend.remove(hit[0])
                cancelled.add(hit[0][2])
            elif sigma[v] == HOST:
                # Z4: a non-persistent variable not yet produced needs no copy
                kind = "h2d" if (g.persistent[v] or written[v]) else "alloc"
                sch.ins[i].append((v, kind))
                if kind == "h2d":
                    bytes_h2d += b[v]
                else:
                    bytes_alloc += b[v]
                sigma[v] = DEV
                R += b[v]
        # (b) complete the oldest scheduled Swap-outs until the budget holds (Fig.2b)
        while R > budget_s:
            if not pend:
                needed = sum(b[v] for v in set(seq.occ[seq.l[i]:r[i] + 1]))
                raise InfeasibleBudget(i, needed + pinned_bytes(g))
            v, _, rid, dirty = pend.pop(0)
            sch.wait_out[i].append(v)
            waited[rid] = dirty
            sigma[v] = HOST
            host_valid[v] = True
            R -= b[v]
        peak = max(peak, R)
        # f_i executes: its outputs are (re)written
        for v in g.fn_out[i]:
            if not g.pinned[v]:
                written[v] = True
                host_valid[v] = False
        # (c)/(d) reserve Swap-out for V̂_i after f_i, or skip it (Fig.2c, 2d)
        seen = []
        for k in range(seq.l[i], seq.e[i] + 1):
            if seq.occ[k] not in seen:
                seen.append(seq.occ[k])
        for v in seen:
            last_k = max(k for k in range(seq.l[i], seq.e[i] + 1) if seq.occ[k] == v)  # Z7
            nx = seq.next_use[last_k]
            if nx is None:
                if g.persistent[v] and not host_valid[v]:
                    # a modified persistent variable is written back (Z10)
                    rid = len(reservations)
                    reservations.append((i, v, rid))
                    pend.append([v, i, rid, True])
                else:
                    sch.free[i].append(v)       # "never used in future" (P:86d)
                    sigma[v] = HOST
                    R -= b[v]
            elif nx <= r[i]:
                pass                            # already inside the window (P:86d, Z8)
            else:
                rid = len(reservations)
                reservations.append((i, v, rid))
                pend.append([v, i, rid, not host_valid[v]])
        r_prev = r[i]

    for v, _, rid, dirty in pend:
        sch.end_wait.append(v)
        waited[rid] = dirty
    # compaction: only reservations that are eventually waited survive
    sch.reserve_dirty = [[] for _ in range(n)]   # host copy stale at reservation (Z19), per entry
    for (i, v, rid) in reservations:
        if rid in waited:
            sch.reserve_out[i].append(v)
            sch.reserve_dirty[i].append(bool(waited[rid]))
    bytes_d2h = sum(b[v] for (i, v, rid) in reservations if rid in waited)
    bytes_d2h_dirty = sum(b[v] for (i, v, rid) in reservations if rid in waited and waited[rid])
    sch.stats = {"bytes_h2d": bytes_h2d, "bytes_alloc": bytes_alloc, "bytes_d2h": bytes_d2h,
                 "bytes_d2h_clean_elided": bytes_d2h_dirty, "peak_sched": peak + pinned_bytes(g)}
    return sch


def canonical_json(sch):
    """The canonical schedule bytes: fixed key order, no
    whitespace, decimal integers, ids = declaration index, lists in trigger
    order."""
    fns = []
    for i in range(len(sch.ins)):
        fns.append('{"in":[' + ",".join(f'[{v},"{k}"]' for v, k in sch.ins[i]) + '],'
                   '"wait_out":[' + ",".join(str(v) for v in sch.wait_out[i]) + '],'
                   '"reserve_out":[' + ",".join(str(v) for v in sch.reserve_out[i]) + '],'
                   '"free":[' + ",".join(str(v) for v in sch.free[i]) + ']}')
    s = sch.stats
    dist = ',"distance":%d' % sch.distance if getattr(sch, "distance", 0) else ""
    return ('{"v":1,"budget":%d,"window":%d%s,"fn":[%s],"end_wait":[%s],"stats":{"bytes_h2d":%d,'
            '"bytes_alloc":%d,"bytes_d2h":%d,"bytes_d2h_clean_elided":%d,"peak_sched":%d}}'
            % (sch.budget, sch.window, dist, ",".join(fns), ",".join(str(v) for v in sch.end_wait),
               s["bytes_h2d"], s["bytes_alloc"], s["bytes_d2h"], s["bytes_d2h_clean_elided"],
               s["peak_sched"]))


def min_feasible_budget(g, seq, window, distance=0):
    """Smallest budget B for which build_schedule succeeds at this window,
    found by binary search over B (budget monotonicity S:157)."""
    attach_bytes(g, seq)
    lo = pinned_bytes(g)
    hi = pinned_bytes(g) + sum(b for v, b in enumerate(g.var_bytes) if not g.pinned[v])

    def ok(B):
        try:
            build_schedule(g, seq, B, window, distance)
            return True
        except InfeasibleBudget:
            return False

    while lo < hi:
        mid = (lo + hi) // 2
        if ok(mid):
            hi = mid
        else:
            lo = mid + 1
    return lo


def max_feasible_window(g, seq, budget):
    """Largest schedule-window W at which the budget is feasible (reading
    Z12), by binary search over W in [0, Σ occurrence bytes]; None if even
    W = 0 is infeasible."""
    attach_bytes(g, seq)

    def ok(W):
        try:
            build_schedule(g, seq, budget, W)
            return True
        except InfeasibleBudget:
            return False

    top = sum(seq.occ_bytes)
    if not ok(0):
        return None
    lo, hi = 0, top
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if ok(mid):
            lo = mid
        else:
            hi = mid - 1
    return lo


def schedule_dict(sch):
    return json.loads(canonical_json(sch))
