/*
 * oocore.h — C ABI of the out-of-core training step of arXiv 2010.14109
 * ("Out-of-core Training for Extremely Large-Scale Neural Networks With
 * Adaptive Window-Based Scheduling"), B200 (sm_100a) implementation.
 *
 * Citations: P:n = line n of the paper text; S:n = line n of the
 * SPEC.md written from it; Z<k> = reading k in DESIGN.md §3.
 *
 * The calls follow the paper's problem statement:
 * given a function-sequence over sized variables and a physical memory
 * budget, decide which variables to swap in and out and when
 * (oc_plan_schedule); place swapped variables in a virtual-addressing chunk
 * allocator (oc_alloc / oc_map / oc_unmap); execute the training
 * step under that schedule (oc_run_step).
 *
 * Conventions
 *   - Every call returns 0 (OC_OK) or a negative oc_status.  No C++
 *     exception crosses the ABI.  When `err` is non-NULL it is filled on
 *     failure (code, indices, byte counts, CUDA/driver status, message).
 *   - Objects (oc_graph, oc_schedule, oc_mem, oc_exec) are owned by the
 *     library and released by their *_destroy call.  Input buffers are owned
 *     by the caller and only read during the call.
 *   - Variable ids = declaration index in the graph document; function ids =
 *     position in execution order (the document's order when executable,
 *     else Kahn's order, see oc_graph_from_json).
 *   - Streams and events are CUDA runtime handles passed as void*; they are
 *     borrowed, never destroyed by the library.
 *   - Thread safety: oc_graph and oc_schedule are immutable after creation and
 *     may be shared across threads.  oc_mem and oc_exec are not
 *     re-entrant; serialise calls per object.
 *   - The library loads without a GPU (CUDA runtime linked statically, the
 *     driver API resolved at first use, NCCL opened with dlopen on demand);
 *     only oc_mem_*, oc_exec_* and oc_nccl_* need a device.
 */
#ifndef OOCORE_H
#define OOCORE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define OC_ABI_VERSION 1

/* ------------------------------------------------------------------ errors */
typedef enum oc_status {
  OC_OK = 0,
  OC_E_PARSE = -1,              /* malformed graph document */
  OC_E_INVALID = -2,            /* cycle, undeclared id, bytes < 1, duplicate id,
                                   unused variable, read before write */
  OC_E_INFEASIBLE_BUDGET = -3,  /* step (b) cannot meet the budget at fn
                                   (P:93); err->needed = B_i(W) + pinned */
  OC_E_DEVICE_OOM = -4,         /* allocator cannot place a request */
  OC_E_UNKNOWN_HANDLE = -5,
  OC_E_DOUBLE_FREE = -6,
  OC_E_CUDA = -7,               /* CUDA runtime / driver failure; err->cuda */
  OC_E_BUFFER_TOO_SMALL = -8,   /* caller buffer shorter than *need */
  OC_E_INVARIANT = -9,          /* internal consistency check failed */
  OC_E_ARG = -10,               /* bad argument (NULL, out of range) */
  OC_E_UNSUPPORTED = -11,       /* op kind / configuration not implemented */
  OC_E_NCCL = -12               /* NCCL failure or library not loadable */
} oc_status;

typedef struct oc_err {
  int code;            /* oc_status */
  uint32_t fn;         /* function index involved, or UINT32_MAX */
  uint32_t var;        /* variable index involved, or UINT32_MAX */
  uint64_t needed;     /* bytes needed (infeasible budget / OOM request) */
  uint64_t free_bytes; /* bytes free at an OOM */
  int cuda;            /* cudaError_t / CUresult / ncclResult_t, 0 if none */
  char msg[256];
} oc_err;

/* Static string for a status code. */
const char* oc_strerror(int code);
/* ABI version of the loaded library (OC_ABI_VERSION at build time). */
int oc_abi_version(void);

/* ------------------------------------------------------------------ graph
 * The network as a DAG of functions over sized variables (Fig.1).
 *
 * Document (JSON, UTF-8):
 *   {"variables": [{"id": str, "bytes": int >= 1,
 *                   "persistent": bool (default false),
 *                   "pinned": bool (default false)} ...],
 *    "functions": [{"id": str, "in": [var id ...], "out": [var id ...],
 *                   "op": {...} (optional; read by the executor)} ...]}
 * V̂_i = in ++ out; a variable in both lists is updated in place and
 * occurs twice in the variable-sequence.
 * persistent: authoritative copy on the host between steps; starts on the
 *   host with valid data; written back after modification (Z10).
 * pinned: resident for the whole step, never swapped; removed from the
 *   variable-sequence; its bytes are subtracted from the budget (Z10).
 * Order: the listed order when no function reads a non-persistent variable
 * before some earlier function wrote it; otherwise Kahn's algorithm over
 * writer->reader edges with the smallest listed index first,
 * allowed only when every variable has at most one writer.
 */
typedef struct oc_graph oc_graph;

int oc_graph_from_json(const char* utf8, size_t len, oc_graph** out, oc_err* err);
/* Incremental construction; ids are returned in declaration order. */
int oc_graph_create(oc_graph** out);
int oc_graph_add_var(oc_graph* g, const char* name, uint64_t bytes, uint32_t flags, uint32_t* id);
#define OC_VAR_PERSISTENT 1u
#define OC_VAR_PINNED 2u
int oc_graph_add_fn(oc_graph* g, const char* name, const uint32_t* in, uint32_t n_in,
                    const uint32_t* out, uint32_t n_out, const char* op_json, uint32_t* id);
int oc_graph_finalize(oc_graph* g, oc_err* err); /* validates and orders; required before use */
void oc_graph_destroy(oc_graph* g);

uint32_t oc_graph_num_vars(const oc_graph* g);
uint32_t oc_graph_num_fns(const oc_graph* g);
uint64_t oc_graph_var_bytes(const oc_graph* g, uint32_t var);
/* Position of the function declared `decl_index`-th in execution order. */
uint32_t oc_graph_fn_position(const oc_graph* g, uint32_t decl_index);
/* F_peak: in-core peak live bytes, alloc at first use / free at last use (Z21). */
uint64_t oc_graph_in_core_peak(const oc_graph* g);
/* Σ distinct variable bytes and max_i bytes(distinct V̂_i). */
void oc_graph_footprint(const oc_graph* g, uint64_t* total_bytes, uint64_t* max_function_bytes);
/* Bytes of the executor's compute workspace for this graph: the largest
 * per-function scratch of its ops (bf16 weight copies, re-laid-out narrow
 * input slices, split-K partials, reduction partials).  Allocated once per
 * executor outside the swap pool (like a cuDNN workspace), so a physical
 * device budget B_p = pinned bytes + pool + this.  0 for graphs without ops. */
uint64_t oc_graph_workspace_bytes(const oc_graph* g);

/* --------------------------------------------------------------- planning
 * The schedule-window greedy of P:91-93 / Fig.2:
 *   window at f_i = v[l_i : r_i], r_i = max index with Σ_{k=l_i..r} b ≤ W,
 *   floored at the end of f_i's span (Z1, Z2);
 *   (a) swap-in every σ=1 variable in v[r_{i-1}+1 : r_i];
 *   (b) complete the oldest reserved swap-outs until the scheduled bytes
 *       ≤ budget − pinned; the waits are placed before f_i;
 *   (c) reserve swap-out of V̂_i after f_i, except (d): free it if never used
 *       again (write back if persistent and modified), skip it if its next use
 *       is inside the window; a later arrival cancels a pending reservation.
 * Then replays the allocator calls wait_out -> in -> [f_i] -> free (Z9)
 * through the chosen allocator model to predict the physical peak,
 * internal/external fragmentation and DeviceOOM.
 */
typedef enum oc_alloc_mode {
  OC_ALLOC_VA = 0,          /* chunked virtual addressing, m_c = chunk_bytes */
  OC_ALLOC_ARENA_BEST = 1,  /* caching best-fit */
  OC_ALLOC_ARENA_FIRST = 2  /* caching first-fit */
} oc_alloc_mode;

typedef struct oc_alloc_model {
  uint32_t mode;         /* oc_alloc_mode */
  uint32_t align;        /* arena request rounding in bytes (default 512); ignored by VA */
  uint64_t chunk_bytes;  /* m_c: VA chunk size, a multiple of the driver granularity
                            (2 MiB on B200); paper default 40 MiB */
  uint64_t phys_bytes;   /* B_p: physical pool for swappable variables (pinned
                            variables live outside it) */
} oc_alloc_model;

#define OC_WINDOW_MAX_FEASIBLE UINT64_MAX

typedef struct oc_plan_params {
  uint64_t budget_bytes; /* B: physical budget incl. pinned variables */
  uint64_t window_bytes; /* schedule-window W, or OC_WINDOW_MAX_FEASIBLE (Z12) */
  oc_alloc_model alloc;
  /* 0: the paper's byte window.  d >= 1: the prior-art window by
   * function count, r_i = e_{min(i+d, n-1)}: d = 1 is
   * vDNN's prefetch-one-layer-ahead, a fixed d the LMS graph distance
   * (P:48-50); window_bytes is then ignored.  Steps (a)-(c) are unchanged. */
  uint32_t distance;
  uint32_t reserved; /* must be 0 */
} oc_plan_params;

typedef struct oc_schedule oc_schedule;

/* Returns OC_OK, OC_E_INFEASIBLE_BUDGET (no schedule; *out = NULL) or
 * OC_E_DEVICE_OOM (the schedule exists but the allocator replay fails:
 * *out is set — usable for stats / JSON, refused by oc_exec_create). */
int oc_plan_schedule(const oc_graph* g, const oc_plan_params* p, oc_schedule** out, oc_err* err);
void oc_schedule_destroy(oc_schedule* s);

/* max_i B_i(W) + pinned bytes: the smallest feasible budget at window W
 * (DESIGN.md §4 closed form). */
uint64_t oc_min_feasible_budget(const oc_graph* g, uint64_t window);
/* The same for the function-distance window d >= 1 (F1): max_i bytes of the
 * distinct variables of f_i .. f_{i+d}, plus pinned bytes. */
uint64_t oc_min_feasible_budget_distance(const oc_graph* g, uint32_t distance);
/* Largest W with oc_min_feasible_budget(W) ≤ budget; OC_E_INFEASIBLE_BUDGET
 * when even W = 0 does not fit. */
int oc_max_feasible_window(const oc_graph* g, uint64_t budget, uint64_t* window, oc_err* err);

/* Canonical schedule bytes: {"v":1,"budget":..,"window":..,
 * "fn":[{"in":[[id,"h2d"|"alloc"]..],"wait_out":[..],"reserve_out":[..],
 * "free":[..]}..],"end_wait":[..],"stats":{..}}.  Two-call size query:
 * *need = length (no NUL); copies when cap >= *need + 1 (NUL-terminated). */
int oc_schedule_json(const oc_schedule* s, char* buf, size_t cap, size_t* need);

typedef struct oc_sched_stats {
  uint64_t budget, window;
  uint64_t bytes_h2d;       /* swap-in bytes that copy (host data valid) */
  uint64_t bytes_alloc;     /* materialisations (no copy) */
  uint64_t bytes_d2h;       /* surviving reservations, paper-literal */
  uint64_t bytes_d2h_dirty; /* of which the host copy was stale (clean ones elided, Z19) */
  uint64_t peak_sched;      /* max_i scheduled bytes after (b), incl. pinned */
  uint64_t pinned_bytes;
  /* allocator replay */
  uint64_t peak_phys;       /* VA: peak mapped chunks × m_c; arena: carved high-water */
  uint64_t peak_alloc;      /* arena: peak allocated bytes; VA: = peak_phys */
  uint64_t if_peak;         /* VA: peak Σ live (m_a − m_r) (Eq.1/2) */
  uint32_t n_max;           /* VA: max live allocations (Eq.2 N_max) */
  int32_t oom_fn, oom_var;  /* -1 when the replay succeeded */
  uint64_t oom_request, oom_free_bytes;
  uint32_t n_in_h2d, n_in_alloc, n_out; /* transfer counts */
  uint32_t n_fns;
} oc_sched_stats;
int oc_schedule_stats(const oc_schedule* s, oc_sched_stats* out);
/* r_i of every function (n = number of functions). */
int oc_schedule_window_ends(const oc_schedule* s, int64_t* r, size_t n);

/* Makespan model of one step (the paper's execution
 * semantics P:86): one compute stream running f_1..f_n in order and two
 * FIFO copy channels.  Before f_i the swap-outs promoted in (b) must have
 * completed; the arrivals of (a) enter the H2D channel once f_{i-1} has
 * ended and those waits are done; f_i starts when f_{i-1} ended, its waits
 * completed and every variable of V̂_i has arrived; the reservations of (c)
 * enter the D2H channel when f_i ends (clean ones move nothing when
 * elide_clean, Z19).  Transfer time = fixed latency + bytes / bandwidth.
 * fn_ms: the n compute times in ms (measured per-function durations, or any
 * cost model); stall_ms (nullable, n entries): f_i's wait after f_{i-1}.
 * Deterministic float64 arithmetic in a fixed order (the oracle,
 * oracle/simulator.py, reproduces it bit for bit).  OC_E_ARG on n mismatch. */
typedef struct oc_link_model {
  double h2d_gbs, d2h_gbs;           /* bandwidth per direction, GB/s (1e9 B/s), > 0 */
  double h2d_fixed_us, d2h_fixed_us; /* per-transfer latency */
  uint32_t elide_clean;
  /* 0: the paper's boundary semantics above.  1: the executor's ordering —
   * an arrival waits only for the memory the allocator replay gave it (VA
   * chunks / arena byte range) to be released (end of the freeing function,
   * or completion of the previous occupant's swap-out) and, for a variable
   * written back, for that copy; each channel is one in-order stream on
   * which alloc-only arrivals and elided swap-outs pass without transfer
   * time (oracle/simulator.simulate_exec). */
  uint32_t model;
} oc_link_model;
typedef struct oc_sim_result {
  double makespan_ms, compute_ms, h2d_busy_ms, d2h_busy_ms, stall_ms;
} oc_sim_result;
int oc_simulate(const oc_schedule* s, const double* fn_ms, size_t n, const oc_link_model* link, oc_sim_result* out,
                double* stall_ms);

/* ------------------------------------------------------------------ memory
 * Virtual-addressing allocator on the CUDA driver VMM API:
 * a pool of ⌊phys_bytes / m_c⌋ physical chunks (cuMemCreate, created lazily);
 * oc_alloc reserves a VA span of m_a = ⌈m_r/m_c⌉·m_c bytes (once, address
 * stable for the span's life); oc_map binds ⌈m_r/m_c⌉ free chunks (FIFO,
 * oldest released first) to it and makes `consumer_stream` wait on each
 * chunk's release event; oc_unmap returns the chunks and records their
 * release event on `release_stream` (the stream of the last use).  Driver unmaps are deferred: a span keeps
 * its mapping until it is re-mapped to different chunks (memoised mode,
 * default) or until its release event completes (OC_MEM_EAGER_UNMAP).
 * Arena modes place requests in one slab with the same best/first-fit rules
 * as the planner's replay; oc_map then only orders the consumer stream after
 * the release events of the block's previous occupants.
 */
typedef struct oc_mem oc_mem;

#define OC_MEM_EAGER_UNMAP 1u   /* paper-literal: unmap every released span */

typedef struct oc_span {
  uint64_t handle;
  uint64_t va;   /* device address (CUdeviceptr); stable for VA spans */
  uint64_t m_r;  /* requested bytes */
  uint64_t m_a;  /* VA: k·m_c; arena: rounded size */
} oc_span;

typedef struct oc_mem_stats {
  uint64_t n_chunks, free_chunks, chunk_bytes;
  uint64_t live_requested, live_allocated, peak_mapped_bytes;
  uint64_t internal_frag, if_peak;
  uint32_t live_count, n_max;
  uint64_t n_driver_map, n_driver_unmap, n_map_calls, n_map_memo_hits;
  uint64_t arena_carved, arena_free_cached;
  double map_us, unmap_us;  /* host time spent in driver map/setaccess and unmap */
} oc_mem_stats;

int oc_mem_create(int device, const oc_alloc_model* model, uint32_t flags, oc_mem** out, oc_err* err);
int oc_alloc(oc_mem* m, uint64_t bytes, oc_span* out, oc_err* err);
int oc_map(oc_mem* m, uint64_t handle, void* consumer_stream, oc_span* out, oc_err* err);
int oc_unmap(oc_mem* m, uint64_t handle, void* release_stream, oc_err* err);
int oc_free(oc_mem* m, uint64_t handle, oc_err* err);
int oc_mem_get_stats(oc_mem* m, oc_mem_stats* out);
/* Return the free-chunk FIFO to its initial order (all chunks must be free);
 * makes every step's chunk assignment identical. */
int oc_mem_reset_order(oc_mem* m, oc_err* err);
void oc_mem_destroy(oc_mem* m);

/* ---------------------------------------------------------------- executor
 * Runs one training step f_1..f_n under a schedule:
 *   per f_i: waits of wait_out[i] (device-side) -> release -> swap-ins of
 *   in[i] on the H2D stream (map + copy, or map only for "alloc") ->
 *   compute stream waits the arrivals of V̂_i -> f_i's kernels ->
 *   D2H of reserve_out[i] on the D2H stream after f_i -> release of free[i].
 * Host copies of every non-pinned variable live in pinned host memory owned
 * by the executor (oc_exec_host_ptr).  Pinned variables need device
 * addresses bound by the caller (oc_exec_bind_device) before the first step.
 */
typedef struct oc_exec oc_exec;

typedef struct oc_streams {
  void* compute; /* cudaStream_t */
  void* h2d;
  void* d2h;
} oc_streams;

typedef struct oc_exec_options {
  uint32_t timeline;       /* 1: record CUDA events around every function and transfer */
  uint32_t elide_clean;    /* 1: skip D2H of variables whose host copy is valid (Z19) */
  uint32_t check;          /* 1: verify residency on the host while issuing (debug) */
  uint32_t pack_threshold; /* bytes; swaps of variables up to this size are grouped per
                              function into one SM-driven pack/unpack kernel that
                              copies 16-byte vectors between device memory and the
                              mapped pinned host copies; 0 = off */
  uint32_t use_graph;      /* 1: after one eager step (all VA mappings memoised), capture
                              the step's issue — copies, event waits, kernels, NCCL — into a
                              CUDA graph once and replay it every later step; ignored with
                              timeline */
  uint32_t trigger;        /* when step (a)'s swap-ins of f_i start on the H2D stream:
                              0 = as soon as the memory they reuse is released (the
                                  previous occupant's last use or swap-out) and their
                                  host copy is complete — the executor's default;
                              1 = the paper's trigger ("We trigger Swap-in
                                  operations at a function f_i", Fig.2): also after
                                  f_{i-1} has finished and the swap-outs f_i waits for
                                  in (b) are complete — the boundary semantics of
                                  oc_simulate model 0 */
} oc_exec_options;

typedef struct oc_step_metrics {
  double step_ms;          /* compute-stream event time of the step */
  double compute_busy_ms;  /* union of function intervals (timeline) */
  double h2d_busy_ms, d2h_busy_ms; /* union of transfer intervals per direction */
  double overlap_frac;     /* |T ∩ C| / |T|, T = transfer union, C = compute union */
  double stall_ms;         /* compute-stream idle time inside the step */
  uint64_t bytes_h2d, bytes_d2h;
  uint32_t n_h2d, n_d2h, n_kernels;
  double host_issue_ms;    /* host time spent issuing the step */
  double map_us, unmap_us; /* driver VMM time during the step */
} oc_step_metrics;

int oc_exec_create(int device, const oc_graph* g, const oc_schedule* s, oc_mem* m,
                   const oc_streams* streams, const oc_exec_options* opt, oc_exec** out,
                   oc_err* err);
int oc_exec_bind_device(oc_exec* x, uint32_t var, void* dev_ptr, oc_err* err);
int oc_exec_host_ptr(oc_exec* x, uint32_t var, void** host_ptr, oc_err* err);
/* The executor's pinned host pool: its size, and the NUMA node its pages were
 * placed on (the GPU's PCIe-local node read from sysfs, MPOL_PREFERRED), or -1
 * when the node is unknown and the pool came from cudaHostAlloc. */
int oc_exec_host_info(oc_exec* x, uint64_t* host_bytes, int* numa_node);
int oc_run_step(oc_exec* x, oc_step_metrics* out, oc_err* err);
/* Per-event timeline of the last step as JSON lines (S:358 format):
 * {"t0":ms,"t1":ms,"stream":"compute|h2d|d2h","id":"<fn or var>"} */
int oc_exec_timeline(oc_exec* x, char* buf, size_t cap, size_t* need);
/* Switch the per-event timeline on or off for later steps (the executor must
 * have been created with options.timeline = 1, which creates the events;
 * OC_E_ARG otherwise).  Off: steps replay the captured CUDA graph when
 * options.use_graph is set; on: steps are issued eagerly with events, so one
 * executor serves both the timed and the instrumented passes of a bench. */
int oc_exec_set_timeline(oc_exec* x, int on);
void oc_exec_destroy(oc_exec* x);

/* ---------------------------------------------------- layer-local inspection
 * Test infrastructure for the layer-local parity harness
 * (tests/test_gpu_layerwise.py): the out-of-core step's functions are the
 * ordinary training step's, so each f_i can be checked on its own —
 * its outputs against the definition applied to the values it read.
 * With a hook set, oc_run_step issues the step eagerly (no CUDA-graph
 * capture), synchronises the device before and after the kernels of each
 * function f_i and calls hook(user, i, 0) before them and hook(user, i, 1)
 * after them (i = execution position, oc_graph_fn_position).  Inside the hook
 * oc_exec_read_var copies the current device bytes of a variable of V̂_i —
 * resident by construction (swap-ins complete before f_i) — or of a
 * pinned variable to host memory (blocking cudaMemcpy; `host` is caller
 * memory of at least `bytes`).  Errors: OC_E_ARG (unknown variable, not
 * resident, bytes larger than the variable), OC_E_CUDA.  hook = NULL removes
 * it.  Not for timed runs. */
typedef void (*oc_fn_hook)(void* user, uint32_t fn, int phase);
int oc_exec_set_hook(oc_exec* x, oc_fn_hook hook, void* user);
int oc_exec_read_var(oc_exec* x, uint32_t var, void* host, uint64_t bytes, oc_err* err);

/* ---------------------------------------------------- data parallel (NCCL)
 * Functions with op {"kind":"allreduce", ...} sum their pinned gradient
 * buffers across replicas with NCCL on the compute stream.
 * Without an attached communicator they are no-ops (single replica).
 */
int oc_nccl_unique_id(void* out_128_bytes, oc_err* err);
int oc_exec_attach_nccl(oc_exec* x, const void* unique_id_128_bytes, int rank, int nranks,
                        oc_err* err);
/* A caller-provided communicator instead of NCCL (other transports; the
 * multi-process tests exchange through torch.distributed gloo): fn(user, buf,
 * count, stream) must replace the `count` fp32 values at device address `buf`
 * by their mean over the replicas, ordered after the work already issued on
 * `stream` (a cudaStream_t), and return 0 (non-zero -> OC_E_NCCL).  Steps then
 * run eagerly (no CUDA-graph capture).  The user pointer is borrowed.
 *
 * With a communicator attached (NCCL or custom) every allreduce function — a
 * bucket of gradients, graphs.build(dp_bucket_bytes=...) — runs on the
 * executor's communication stream, forked from the compute stream after its
 * inputs; everything that consumes the bucket (its SGD, swap-outs, reuse of
 * its memory) waits for the exchange, while the compute stream continues with
 * the next layers' backward.  NCCL buckets are one ncclGroup. */
typedef int (*oc_allreduce_fn)(void* user, void* buf, uint64_t count, void* stream);
int oc_exec_attach_comm(oc_exec* x, oc_allreduce_fn fn, void* user, oc_err* err);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* OOCORE_H */
