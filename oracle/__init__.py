"""CPU oracle for arXiv 2010.14109 (out-of-core training with a locally adaptive
swap window and virtual addressing).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
under `oracle/`.  The product (`paper_2010_14109_b200/`, the C-ABI library
`liboocore.so`) never imports, links or executes it, and the oracle never
imports the product.  The two share only the seeded input generators in
`synth/`, which contain none of the method's arithmetic.

Every function here is written to be checked against the paper by eye: plain
Python loops / numpy, no blocking, no fusion, each citing the passage it
follows.  Citations: `P:n` = line n of the paper text, `S:n` = line
n of SPEC.md, `Z<k>` = the k-th reading listed in DESIGN.md §3 (the paper's
silences and how they are read).

Modules
  graph       — DAG of functions, execution order, variable-sequence
  scheduler   — schedule-window greedy, steps (a)-(d)
  allocators  — virtual-addressing chunk pool and caching
                best-/first-fit arenas; replay of a schedule
  validate    — replay validator of a schedule
  bruteforce  — exhaustive search on tiny graphs (P:62 search space)
  numerics    — fp64 reference forward/backward/update with bf16/fp32
                rounding emulation (standard training-step definitions)

Parity status (DESIGN.md §4 lists each pin):
  graph, scheduler, allocators, validate, bruteforce, numerics — pinned.
  No function in this package is "parity unpinned".
"""
