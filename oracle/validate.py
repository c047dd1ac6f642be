"""Oracle: replay validator of a schedule.

Replays the schedule event by event in the executor order
  wait_out[i] -> in[i] -> f_i -> reserve_out[i] -> free[i],   end: end_wait
and checks, independently of how the schedule was built:
  (1) every variable of V̂_i is on the device when f_i runs       (S:140 (1))
  (2) scheduled resident bytes <= budget at every point           (S:140 (2))
  (3) no reservation of a variable never used again unless it is a
      modified persistent variable (write-back); no swap-in of a
      resident variable                                           (S:140 (3),(4))
  (4) every reservation has exactly one later wait and the variable
      is not used between them
  (5) conservation: Σ in bytes = Σ waited bytes + Σ freed bytes
  (6) r_i non-decreasing (reading Z3)
Returns (True, None) or (False, "<first violation>").
"""


def validate(g, seq, sch, budget):
    b = g.var_bytes
    pinned = sum(x for v, x in enumerate(g.var_bytes) if g.pinned[v])
    budget_s = budget - pinned
    on_dev = set()
    pending = {}        # v -> function index of the reservation
    waited_once = set()
    R = 0
    bytes_in = bytes_waited = bytes_freed = 0
    last_use = {}
    for i in range(g.n_fns):
        for v in g.uses(i):
            last_use[v] = i
    for i in range(1, len(sch.r)):
        if sch.r[i] < sch.r[i - 1]:
            return False, f"window end decreases at f{i}"
    res_at = {}
    for i in range(g.n_fns):
        for v in sch.reserve_out[i]:
            res_at.setdefault(v, []).append(i)

    def wait(v, where):
        nonlocal R, bytes_waited
        if v not in pending:
            return f"{where}: wait for var {v} without a pending reservation"
        del pending[v]
        on_dev.discard(v)
        R -= b[v]
        bytes_waited += b[v]
        return None

    for i in range(g.n_fns):
        for v in sch.wait_out[i]:
            err = wait(v, f"f{i}")
            if err:
                return False, err
        for v, kind in sch.ins[i]:
            if v in on_dev:
                return False, f"f{i}: swap-in of resident var {v}"
            if g.pinned[v]:
                return False, f"f{i}: swap-in of pinned var {v}"
            on_dev.add(v)
            R += b[v]
            bytes_in += b[v]
        if R > budget_s:
            return False, f"f{i}: resident {R} exceeds budget {budget_s}"
        for v in g.uses(i):
            if not g.pinned[v] and v not in on_dev:
                return False, f"f{i}: var {v} not resident when f{i} runs"
            if v in pending:
                return False, f"f{i}: var {v} used while its swap-out is in flight"
        for v in sch.reserve_out[i]:
            if v not in set(g.uses(i)):
                return False, f"f{i}: reservation of var {v} not used by f{i}"
            if last_use[v] == i and not g.persistent[v]:
                return False, f"f{i}: swap-out of dead var {v}"
            if v in pending:
                return False, f"f{i}: var {v} reserved twice"
            pending[v] = i
        for v in sch.free[i]:
            if last_use[v] != i:
                return False, f"f{i}: free of var {v} that is used later"
            if v not in on_dev or v in pending:
                return False, f"f{i}: free of non-resident var {v}"
            on_dev.discard(v)
            R -= b[v]
            bytes_freed += b[v]
    for v in sch.end_wait:
        err = wait(v, "end")
        if err:
            return False, err
    if pending:
        return False, f"reservations never waited: {sorted(pending)}"
    if on_dev:
        return False, f"variables left on device at the end: {sorted(on_dev)}"
    if bytes_in != bytes_waited + bytes_freed:
        return False, "conservation violated"
    return True, None
