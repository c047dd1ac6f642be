"""Seeded random graph documents for planner tests (S:462 replay-safety suite,
S:416-424 workload shapes).  Output is the JSON graph document read by both
`oracle.graph.load_graph` and `oc_graph_from_json`."""
import json

import numpy as np


def doc(variables, functions):
    return json.dumps({"variables": variables, "functions": functions}, separators=(",", ":"))


def random_graph(seed, n_fns=None, n_vars=None, max_bytes=64, p_persistent=0.2, p_pinned=0.0,
                 max_in=3, p_inplace=0.1):
    """A random executable function sequence: each function reads up to
    `max_in` earlier-produced (or persistent) variables and writes 0-2 new
    ones; some functions update a variable in place.  Sizes U{1..max_bytes}."""
    rng = np.random.default_rng(seed)
    if n_fns is None:
        n_fns = int(rng.integers(1, 50))
    if n_vars is None:
        n_vars = int(rng.integers(1, 100))
    variables = []
    for j in range(n_vars):
        variables.append({"id": f"v{j}", "bytes": int(rng.integers(1, max_bytes + 1)),
                          "persistent": bool(rng.random() < p_persistent),
                          "pinned": bool(rng.random() < p_pinned)})
    readable = [j for j in range(n_vars) if variables[j]["persistent"] or variables[j]["pinned"]]
    unwritten = [j for j in range(n_vars) if j not in readable]
    functions = []
    for i in range(n_fns):
        ins = []
        if readable:
            k = int(rng.integers(0, min(max_in, len(readable)) + 1))
            ins = [int(x) for x in rng.choice(readable, size=k, replace=False)]
        outs = []
        n_new = int(rng.integers(0, 3))
        for _ in range(n_new):
            if unwritten:
                outs.append(unwritten.pop(0))
        if ins and rng.random() < p_inplace:
            outs.append(ins[int(rng.integers(0, len(ins)))])
        if not ins and not outs:
            if unwritten:
                outs.append(unwritten.pop(0))
            elif readable:
                ins = [int(rng.choice(readable))]
        for o in outs:
            if o not in readable:
                readable.append(o)
        functions.append({"id": f"f{i}", "in": [f"v{x}" for x in ins], "out": [f"v{x}" for x in outs]})
    used = set()
    for f in functions:
        used.update(f["in"])
        used.update(f["out"])
    # every declared variable must be used: give leftovers to a last function
    left = [v["id"] for v in variables if v["id"] not in used]
    if left:
        functions.append({"id": f"f{len(functions)}", "in": [], "out": left})
    return doc(variables, functions)


def chain_graph(sizes, persistent_first=False):
    """f1=[v1], f_i=[v_{i-1}, v_i]: the chain layout of SURVEY E0."""
    variables = [{"id": f"v{j + 1}", "bytes": s, "persistent": persistent_first and j == 0}
                 for j, s in enumerate(sizes)]
    functions = [{"id": "f1", "in": [], "out": ["v1"]}]
    for i in range(1, len(sizes)):
        functions.append({"id": f"f{i + 1}", "in": [f"v{i}"], "out": [f"v{i + 1}"]})
    return doc(variables, functions)


def train_mirror_chain(depth, act_bytes, param_bytes=0, grad_bytes=None):
    """A training-step-shaped chain (S:407 train_mirror): forward f_1..f_d
    producing a_1..a_d from x, a loss, then backward functions in reverse,
    each reading the saved activation and producing the next gradient."""
    grad_bytes = act_bytes if grad_bytes is None else grad_bytes
    variables = [{"id": "x", "bytes": act_bytes, "persistent": True}]
    functions = []
    prev = "x"
    for i in range(1, depth + 1):
        variables.append({"id": f"a{i}", "bytes": act_bytes})
        functions.append({"id": f"fwd{i}", "in": [prev], "out": [f"a{i}"]})
        prev = f"a{i}"
    variables.append({"id": "L", "bytes": 4})
    functions.append({"id": "loss", "in": [prev], "out": ["L"]})
    variables.append({"id": f"g{depth}", "bytes": grad_bytes})
    functions.append({"id": f"bwd{depth}", "in": [prev, "L"], "out": [f"g{depth}"]})
    for i in range(depth - 1, 0, -1):
        variables.append({"id": f"g{i}", "bytes": grad_bytes})
        functions.append({"id": f"bwd{i}", "in": [f"a{i}", f"g{i + 1}"], "out": [f"g{i}"]})
    return doc(variables, functions)
