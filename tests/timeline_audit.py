"""Audit of an executed out-of-core step's timeline against the paper's
execution semantics (north_star invariants "every tensor is resident when
read" and "no transfer overlaps a use"; Fig.2(b): "waits for the
Swap-out right before f_i": swap-ins performed before executing f_i).

Input: the timeline in oc_exec_timeline's format — compute intervals per
function position ("fn"), H2D intervals per arrival slot ("slot", "fn" = the
function whose step (a) issued it), D2H intervals per departure ("dep", "fn" =
the function after which it was reserved) — plus the schedule and the
allocator placements (oracle/allocators.replay, bit-exact with the C-ABI
replay, tests/test_plan_parity.py) that say which memory each arrival slot
occupies.  Checks, with times compared exactly (events on the same device
clock):

  R1 residency   every H2D arrival ends before the first function >= its
                 issuing function that uses the variable starts
  R2 reuse       no write into a slot's memory (its H2D, or for an alloc-only
                 arrival its first compute use) starts before every reader of
                 the memory's previous occupants ended: the functions that used
                 them while resident there and their swap-outs (D2H) from there
  R3 swap-out    every D2H starts after the function it was reserved after ends
  R4 write-back  an H2D of a variable starts after the latest earlier D2H of
                 the same variable ended (the host copy it reads is complete)
  R5 trigger     (paper trigger mode only, oc_exec_options.trigger = 1) every
                 H2D issued by f_i's step (a) starts after f_{i-1} ended
                 ("We trigger Swap-in operations at a function f_i")

Test helper (tests/ only); returns a list of violation strings."""


def _units(mode, p, nbytes, align):
    if mode == "va":
        return ("c", frozenset(p))
    size = -(-nbytes // align) * align
    return ("r", (p, p + size))


def _overlap(u, w):
    if u[0] == "c":
        return bool(u[1] & w[1])
    return u[1][0] < w[1][1] and w[1][0] < u[1][1]


def audit(g, sch, placements, mode, timeline, align=512, paper_trigger=False):
    n = len(sch.ins)
    uses = [set(g.uses(i)) for i in range(n)]
    comp = {e["fn"]: (e["t0"], e["t1"]) for e in timeline if e["stream"] == "compute"}
    h2d = {e["slot"]: e for e in timeline if e["stream"] == "h2d"}
    d2h = {e["dep"]: e for e in timeline if e["stream"] == "d2h"}
    bad = []

    # departures in executor order: for each f_i, its reserve_out list
    deps = []
    for i in range(n):
        for v in sch.reserve_out[i]:
            deps.append((i, v))

    # slots: placements in arrival order; residency [arrival fn, release]
    slots = []
    for k, (ia, v, p) in enumerate(placements):
        readers_fn, rel = [], None
        for j in range(ia, n):
            if j > ia and v in sch.wait_out[j]:
                rel = ("wait", j)
                break
            if v in uses[j]:
                readers_fn.append(j)
            if v in sch.free[j]:
                rel = ("free", j)
                break
        end = rel[1] if rel else n
        readers_dep = [d for d, (i, u) in enumerate(deps) if u == v and ia <= i < end]
        kind = dict(sch.ins[ia])[v]
        slots.append({"k": k, "fn": ia, "var": v, "kind": kind, "units": _units(mode, p, g.var_bytes[v], align),
                      "readers_fn": readers_fn, "readers_dep": readers_dep})

    for s in slots:
        k, v = s["k"], s["var"]
        first_use = s["readers_fn"][0] if s["readers_fn"] else None
        # R1
        if s["kind"] == "h2d":
            if k not in h2d:
                bad.append(f"R1 slot {k} ({g.var_names[v]}): H2D not in the timeline")
                continue
            if first_use is not None and first_use in comp and h2d[k]["t1"] > comp[first_use][0]:
                bad.append(f"R1 slot {k} ({g.var_names[v]}): H2D ends {h2d[k]['t1']:.4f} after f{first_use} "
                           f"starts {comp[first_use][0]:.4f}")
        # R2: the write into this slot's memory
        if s["kind"] == "h2d":
            t_write = h2d[k]["t0"]
        elif first_use is not None and first_use in comp:
            t_write = comp[first_use][0]
        else:
            t_write = None
        if t_write is not None:
            for q in slots[:k]:
                if not _overlap(q["units"], s["units"]):
                    continue
                for f in q["readers_fn"]:
                    if f in comp and comp[f][1] > t_write:
                        bad.append(f"R2 slot {k} ({g.var_names[v]}) written at {t_write:.4f} while f{f} "
                                   f"(reads {g.var_names[q['var']]} in slot {q['k']}) ends {comp[f][1]:.4f}")
                for d in q["readers_dep"]:
                    if d in d2h and d2h[d]["t1"] > t_write:
                        bad.append(f"R2 slot {k} ({g.var_names[v]}) written at {t_write:.4f} while the swap-out "
                                   f"of {g.var_names[q['var']]} from slot {q['k']} ends {d2h[d]['t1']:.4f}")
        # R4
        if s["kind"] == "h2d":
            prev = [d for d, (i, u) in enumerate(deps) if u == v and i < s["fn"] and d in d2h]
            if prev and d2h[prev[-1]]["t1"] > h2d[k]["t0"]:
                bad.append(f"R4 slot {k} ({g.var_names[v]}): H2D starts before its write-back ended")
    # R5
    if paper_trigger:
        for k, e in h2d.items():
            i = e["fn"]
            if i > 0 and i - 1 in comp and e["t0"] < comp[i - 1][1]:
                bad.append(f"R5 slot {k}: H2D issued by f{i} starts {e['t0']:.4f} before f{i - 1} ends "
                           f"{comp[i - 1][1]:.4f}")
    # R3
    for d, (i, v) in enumerate(deps):
        if d in d2h and i in comp and d2h[d]["t0"] < comp[i][1]:
            bad.append(f"R3 dep {d} ({g.var_names[v]}): D2H starts {d2h[d]['t0']:.4f} before f{i} ends "
                       f"{comp[i][1]:.4f}")
    return bad
