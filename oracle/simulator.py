"""Oracle: makespan model of one out-of-core step.

Test infrastructure only (see oracle/__init__.py).  A deterministic
discrete-event replay of a schedule with one compute stream and two copy
channels (host->device, device->host), following the paper's execution
semantics: functions run f_1..f_n in order; before f_i the
swap-outs promoted in (b) must have completed (their memory is what the
arrivals of (a) reuse); the arrivals of (a) are enqueued FIFO on the H2D
channel once f_{i−1} has ended and those waits are done; f_i starts when
f_{i−1} ended, its waits completed and every variable of V̂_i has arrived;
the surviving reservations of (c) enqueue FIFO on the D2H channel when f_i
ends (clean ones move no bytes when elide_clean, Z19); the step ends when
f_n and the end-of-step write-backs are done.

Times are float64 milliseconds, accumulated in a fixed order, so the C++
model (oc_simulate) must reproduce them exactly.  Transfer time =
fixed latency + bytes / bandwidth; compute time of f_i = fn_ms[i] (measured
per-function durations, or any cost model the caller chooses).
"""


def simulate(g, seq, sch, fn_ms, h2d_gbs, d2h_gbs, h2d_us=0.0, d2h_us=0.0, elide_clean=True):
    b = g.var_bytes
    n = len(sch.ins)
    ready = {}          # var -> time its device copy is complete
    out_done = {}       # var -> completion of its pending swap-out
    h2d_free = d2h_free = 0.0
    end_prev = 0.0
    stall = []
    busy = {"compute": 0.0, "h2d": 0.0, "d2h": 0.0}
    events = []
    for i in range(n):
        t_wait = 0.0
        for v in sch.wait_out[i]:
            t_wait = max(t_wait, out_done.pop(v))
        t_trig = max(end_prev, t_wait)
        for v, kind in sch.ins[i]:
            if kind == "h2d":
                start = max(h2d_free, t_trig)
                dur = h2d_us * 1e-3 + b[v] / (h2d_gbs * 1e6)
                h2d_free = start + dur
                busy["h2d"] += dur
                ready[v] = h2d_free
                events.append((start, h2d_free, "h2d", v))
            else:
                ready[v] = t_trig
        need = 0.0
        for v in set(seq.occ[seq.l[i]:seq.e[i] + 1]):
            if not g.pinned[v]:
                need = max(need, ready[v])
        start = max(end_prev, t_wait, need)
        stall.append(start - end_prev)
        end = start + fn_ms[i]
        busy["compute"] += fn_ms[i]
        events.append((start, end, "compute", i))
        for v, dirty in zip(sch.reserve_out[i], sch.reserve_dirty[i]):
            if elide_clean and not dirty:
                out_done[v] = end
                continue
            s0 = max(d2h_free, end)
            dur = d2h_us * 1e-3 + b[v] / (d2h_gbs * 1e6)
            d2h_free = s0 + dur
            busy["d2h"] += dur
            out_done[v] = d2h_free
            events.append((s0, d2h_free, "d2h", v))
        end_prev = end
    makespan = end_prev
    for v in sch.end_wait:
        makespan = max(makespan, out_done[v])
    return {"makespan_ms": makespan, "stall_ms": stall, "busy_ms": busy, "events": events}


def lower_bounds(g, sch, fn_ms, h2d_gbs, d2h_gbs):
    """Σ compute, H2D bytes / bandwidth, D2H bytes / bandwidth."""
    return {"compute": sum(fn_ms), "h2d": sch.stats["bytes_h2d"] / (h2d_gbs * 1e6),
            "d2h": sch.stats["bytes_d2h_clean_elided"] / (d2h_gbs * 1e6)}


def simulate_exec(g, seq, sch, placements, mode, fn_ms, h2d_gbs, d2h_gbs, h2d_us=0.0, d2h_us=0.0,
                  elide_clean=True, align=512):
    """Placement-aware variant: the executor's ordering instead of the paper's
    boundary semantics.  An arrival is not held until f_{i−1} ends; it waits
    only for the memory it reuses — the chunks (VA) or byte range (arena) the
    allocator replay gave it (`placements`, from allocators.replay), released
    at the end of the function that freed the previous occupant or at the
    completion of its swap-out — and, for a variable written back, for that
    copy.  Each copy channel is one in-order stream: an alloc-only arrival or a
    clean (elided) swap-out occupies no transfer time but still passes the
    stream in order.  Compute as in simulate()."""
    b = g.var_bytes
    n = len(sch.ins)
    place = iter(placements)
    rel_chunk, rel_iv, held = {}, [], {}
    ready, out_done, host_ready = {}, {}, {}
    h2d_free = d2h_free = end_prev = 0.0

    def units_of(v, p):
        if mode == "va":
            return ("c", list(p))
        size = -(-b[v] // align) * align
        return ("r", (p, p + size))

    def mem_ready(u):
        t = 0.0
        if u[0] == "c":
            for c in u[1]:
                t = max(t, rel_chunk.get(c, 0.0))
        else:
            lo, hi = u[1]
            for (a, z, tr) in rel_iv:
                if a < hi and lo < z:
                    t = max(t, tr)
        return t

    def release(u, t):
        if u[0] == "c":
            for c in u[1]:
                rel_chunk[c] = t
        else:
            rel_iv.append((u[1][0], u[1][1], t))

    stall = []
    events = []        # timeline in the executor's format (oc_exec_timeline): slot / dep ids
    slot = dep = 0
    for i in range(n):
        t_wait = 0.0
        for v in sch.wait_out[i]:
            t_wait = max(t_wait, out_done[v])
            release(held.pop(v), out_done[v])
        for v, kind in sch.ins[i]:
            i2, v2, p = next(place)
            assert (i2, v2) == (i, v)
            u = units_of(v, p)
            t = max(h2d_free, mem_ready(u))
            if kind == "h2d":
                t = max(t, host_ready.get(v, 0.0))
                t0 = t
                t = t + (h2d_us * 1e-3 + b[v] / (h2d_gbs * 1e6))
                events.append({"t0": t0, "t1": t, "stream": "h2d", "slot": slot, "fn": i, "var": v})
            h2d_free = t
            ready[v] = t
            held[v] = u
            slot += 1
        need = 0.0
        for v in set(seq.occ[seq.l[i]:seq.e[i] + 1]):
            if not g.pinned[v]:
                need = max(need, ready[v])
        start = max(end_prev, t_wait, need)
        stall.append(start - end_prev)
        end = start + fn_ms[i]
        events.append({"t0": start, "t1": end, "stream": "compute", "fn": i})
        for v, dirty in zip(sch.reserve_out[i], sch.reserve_dirty[i]):
            t = max(d2h_free, end)
            if dirty or not elide_clean:
                t0 = t
                t = t + (d2h_us * 1e-3 + b[v] / (d2h_gbs * 1e6))
                host_ready[v] = t
                events.append({"t0": t0, "t1": t, "stream": "d2h", "dep": dep, "fn": i, "var": v})
            d2h_free = t
            out_done[v] = t
            dep += 1
        for v in sch.free[i]:
            release(held.pop(v), end)
        end_prev = end
    makespan = end_prev
    for v in sch.end_wait:
        makespan = max(makespan, out_done[v])
    return {"makespan_ms": makespan, "stall_ms": stall, "events": events}
