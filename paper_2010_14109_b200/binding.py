"""ctypes binding of liboocore.so — argument marshalling only, same names as
include/oocore.h.  Every step of the planning and the training step runs in
the library; nothing here computes.  Loading fails loudly when the library is
missing (there is no Python fallback)."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboocore.so")

OC_OK = 0
OC_E_PARSE, OC_E_INVALID, OC_E_INFEASIBLE_BUDGET, OC_E_DEVICE_OOM = -1, -2, -3, -4
OC_E_UNKNOWN_HANDLE, OC_E_DOUBLE_FREE, OC_E_CUDA, OC_E_BUFFER_TOO_SMALL = -5, -6, -7, -8
OC_E_INVARIANT, OC_E_ARG, OC_E_UNSUPPORTED, OC_E_NCCL = -9, -10, -11, -12
OC_ALLOC_VA, OC_ALLOC_ARENA_BEST, OC_ALLOC_ARENA_FIRST = 0, 1, 2
OC_WINDOW_MAX_FEASIBLE = 2 ** 64 - 1
OC_VAR_PERSISTENT, OC_VAR_PINNED = 1, 2
OC_MEM_EAGER_UNMAP = 1


class oc_err(C.Structure):
    _fields_ = [("code", C.c_int), ("fn", C.c_uint32), ("var", C.c_uint32), ("needed", C.c_uint64),
                ("free_bytes", C.c_uint64), ("cuda", C.c_int), ("msg", C.c_char * 256)]


class oc_alloc_model(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("align", C.c_uint32), ("chunk_bytes", C.c_uint64),
                ("phys_bytes", C.c_uint64)]


class oc_plan_params(C.Structure):
    _fields_ = [("budget_bytes", C.c_uint64), ("window_bytes", C.c_uint64), ("alloc", oc_alloc_model),
                ("distance", C.c_uint32), ("reserved", C.c_uint32)]


class oc_link_model(C.Structure):
    _fields_ = [("h2d_gbs", C.c_double), ("d2h_gbs", C.c_double), ("h2d_fixed_us", C.c_double),
                ("d2h_fixed_us", C.c_double), ("elide_clean", C.c_uint32), ("model", C.c_uint32)]


class oc_sim_result(C.Structure):
    _fields_ = [("makespan_ms", C.c_double), ("compute_ms", C.c_double), ("h2d_busy_ms", C.c_double),
                ("d2h_busy_ms", C.c_double), ("stall_ms", C.c_double)]


class oc_sched_stats(C.Structure):
    _fields_ = [("budget", C.c_uint64), ("window", C.c_uint64), ("bytes_h2d", C.c_uint64),
                ("bytes_alloc", C.c_uint64), ("bytes_d2h", C.c_uint64), ("bytes_d2h_dirty", C.c_uint64),
                ("peak_sched", C.c_uint64), ("pinned_bytes", C.c_uint64), ("peak_phys", C.c_uint64),
                ("peak_alloc", C.c_uint64), ("if_peak", C.c_uint64), ("n_max", C.c_uint32),
                ("oom_fn", C.c_int32), ("oom_var", C.c_int32), ("oom_request", C.c_uint64),
                ("oom_free_bytes", C.c_uint64), ("n_in_h2d", C.c_uint32), ("n_in_alloc", C.c_uint32),
                ("n_out", C.c_uint32), ("n_fns", C.c_uint32)]


class oc_span(C.Structure):
    _fields_ = [("handle", C.c_uint64), ("va", C.c_uint64), ("m_r", C.c_uint64), ("m_a", C.c_uint64)]


class oc_mem_stats(C.Structure):
    _fields_ = [("n_chunks", C.c_uint64), ("free_chunks", C.c_uint64), ("chunk_bytes", C.c_uint64),
                ("live_requested", C.c_uint64), ("live_allocated", C.c_uint64),
                ("peak_mapped_bytes", C.c_uint64), ("internal_frag", C.c_uint64), ("if_peak", C.c_uint64),
                ("live_count", C.c_uint32), ("n_max", C.c_uint32), ("n_driver_map", C.c_uint64),
                ("n_driver_unmap", C.c_uint64), ("n_map_calls", C.c_uint64), ("n_map_memo_hits", C.c_uint64),
                ("arena_carved", C.c_uint64), ("arena_free_cached", C.c_uint64), ("map_us", C.c_double),
                ("unmap_us", C.c_double)]


class oc_streams(C.Structure):
    _fields_ = [("compute", C.c_void_p), ("h2d", C.c_void_p), ("d2h", C.c_void_p)]


class oc_exec_options(C.Structure):
    _fields_ = [("timeline", C.c_uint32), ("elide_clean", C.c_uint32), ("check", C.c_uint32),
                ("pack_threshold", C.c_uint32), ("use_graph", C.c_uint32), ("trigger", C.c_uint32)]


class oc_step_metrics(C.Structure):
    _fields_ = [("step_ms", C.c_double), ("compute_busy_ms", C.c_double), ("h2d_busy_ms", C.c_double),
                ("d2h_busy_ms", C.c_double), ("overlap_frac", C.c_double), ("stall_ms", C.c_double),
                ("bytes_h2d", C.c_uint64), ("bytes_d2h", C.c_uint64), ("n_h2d", C.c_uint32),
                ("n_d2h", C.c_uint32), ("n_kernels", C.c_uint32), ("host_issue_ms", C.c_double),
                ("map_us", C.c_double), ("unmap_us", C.c_double)]


P = C.c_void_p
E = C.POINTER(oc_err)
OC_FN_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_uint32, C.c_int)
OC_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_SIGS = {
    "oc_strerror": (C.c_char_p, [C.c_int]),
    "oc_abi_version": (C.c_int, []),
    "oc_graph_from_json": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P), E]),
    "oc_graph_create": (C.c_int, [C.POINTER(P)]),
    "oc_graph_add_var": (C.c_int, [P, C.c_char_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32)]),
    "oc_graph_add_fn": (C.c_int, [P, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_uint32),
                                  C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32)]),
    "oc_graph_finalize": (C.c_int, [P, E]),
    "oc_graph_destroy": (None, [P]),
    "oc_graph_num_vars": (C.c_uint32, [P]),
    "oc_graph_num_fns": (C.c_uint32, [P]),
    "oc_graph_var_bytes": (C.c_uint64, [P, C.c_uint32]),
    "oc_graph_fn_position": (C.c_uint32, [P, C.c_uint32]),
    "oc_graph_in_core_peak": (C.c_uint64, [P]),
    "oc_graph_footprint": (None, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "oc_graph_workspace_bytes": (C.c_uint64, [P]),
    "oc_plan_schedule": (C.c_int, [P, C.POINTER(oc_plan_params), C.POINTER(P), E]),
    "oc_schedule_destroy": (None, [P]),
    "oc_min_feasible_budget": (C.c_uint64, [P, C.c_uint64]),
    "oc_min_feasible_budget_distance": (C.c_uint64, [P, C.c_uint32]),
    "oc_max_feasible_window": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_uint64), E]),
    "oc_schedule_json": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "oc_schedule_stats": (C.c_int, [P, C.POINTER(oc_sched_stats)]),
    "oc_schedule_window_ends": (C.c_int, [P, C.POINTER(C.c_int64), C.c_size_t]),
    "oc_simulate": (C.c_int, [P, C.POINTER(C.c_double), C.c_size_t, C.POINTER(oc_link_model), C.POINTER(oc_sim_result),
                              C.POINTER(C.c_double)]),
    "oc_mem_create": (C.c_int, [C.c_int, C.POINTER(oc_alloc_model), C.c_uint32, C.POINTER(P), E]),
    "oc_alloc": (C.c_int, [P, C.c_uint64, C.POINTER(oc_span), E]),
    "oc_map": (C.c_int, [P, C.c_uint64, P, C.POINTER(oc_span), E]),
    "oc_unmap": (C.c_int, [P, C.c_uint64, P, E]),
    "oc_free": (C.c_int, [P, C.c_uint64, E]),
    "oc_mem_get_stats": (C.c_int, [P, C.POINTER(oc_mem_stats)]),
    "oc_mem_reset_order": (C.c_int, [P, E]),
    "oc_mem_destroy": (None, [P]),
    "oc_exec_create": (C.c_int, [C.c_int, P, P, P, C.POINTER(oc_streams), C.POINTER(oc_exec_options),
                                 C.POINTER(P), E]),
    "oc_exec_bind_device": (C.c_int, [P, C.c_uint32, P, E]),
    "oc_exec_host_ptr": (C.c_int, [P, C.c_uint32, C.POINTER(P), E]),
    "oc_exec_host_info": (C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
    "oc_run_step": (C.c_int, [P, C.POINTER(oc_step_metrics), E]),
    "oc_exec_timeline": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "oc_exec_destroy": (None, [P]),
    "oc_exec_set_timeline": (C.c_int, [P, C.c_int]),
    "oc_exec_set_hook": (C.c_int, [P, OC_FN_HOOK, P]),
    "oc_exec_read_var": (C.c_int, [P, C.c_uint32, P, C.c_uint64, E]),
    "oc_nccl_unique_id": (C.c_int, [P, E]),
    "oc_exec_attach_nccl": (C.c_int, [P, P, C.c_int, C.c_int, E]),
    "oc_exec_attach_comm": (C.c_int, [P, OC_ALLREDUCE_FN, P, E]),
}

_lib = None


def lib():
    """Load liboocore.so (raises if it is missing — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2010_14109_b200.build` "
                               "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIGS)


class OcError(Exception):
    def __init__(self, code, err):
        self.code = code
        self.fn = err.fn
        self.var = err.var
        self.needed = err.needed
        self.free_bytes = err.free_bytes
        self.cuda = err.cuda
        self.msg = err.msg.decode(errors="replace")
        super().__init__(f"{lib().oc_strerror(code).decode()} ({code}): {self.msg}")


def check(code, err):
    if code != OC_OK:
        raise OcError(code, err)


# ------------------------------------------------------------ thin wrappers


class Mem:
    """The allocator C-ABI (oc_mem_create / oc_alloc / oc_map / oc_unmap /
    oc_free / oc_mem_get_stats, include/oocore.h): VA chunk pool
    or caching best/first-fit arena.  Argument marshalling only;
    streams are raw cudaStream_t values (e.g. torch.cuda.Stream.cuda_stream)."""

    def __init__(self, device=0, mode=OC_ALLOC_VA, chunk_bytes=2 << 20, phys_bytes=64 << 20, align=512, flags=0):
        self.h = P()
        err = oc_err()
        model = oc_alloc_model(mode=mode, align=align, chunk_bytes=chunk_bytes, phys_bytes=phys_bytes)
        check(lib().oc_mem_create(device, C.byref(model), flags, C.byref(self.h), C.byref(err)), err)

    def alloc(self, nbytes):
        sp, err = oc_span(), oc_err()
        check(lib().oc_alloc(self.h, nbytes, C.byref(sp), C.byref(err)), err)
        return sp

    def map(self, handle, stream=0):
        sp, err = oc_span(), oc_err()
        check(lib().oc_map(self.h, handle, P(stream), C.byref(sp), C.byref(err)), err)
        return sp

    def unmap(self, handle, stream=0):
        err = oc_err()
        check(lib().oc_unmap(self.h, handle, P(stream), C.byref(err)), err)

    def free(self, handle):
        err = oc_err()
        check(lib().oc_free(self.h, handle, C.byref(err)), err)

    def stats(self):
        st = oc_mem_stats()
        check(lib().oc_mem_get_stats(self.h, C.byref(st)), oc_err())
        return {k: getattr(st, k) for k, _ in oc_mem_stats._fields_}

    def close(self):
        if getattr(self, "h", None):
            lib().oc_mem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:
            pass


class Graph:
    def __init__(self, doc):
        self.h = P()
        err = oc_err()
        b = doc.encode() if isinstance(doc, str) else doc
        check(lib().oc_graph_from_json(b, len(b), C.byref(self.h), C.byref(err)), err)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().oc_graph_destroy(self.h)
            except TypeError:      # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    @property
    def n_vars(self):
        return lib().oc_graph_num_vars(self.h)

    @property
    def n_fns(self):
        return lib().oc_graph_num_fns(self.h)

    def in_core_peak(self):
        return lib().oc_graph_in_core_peak(self.h)

    def workspace_bytes(self):
        return lib().oc_graph_workspace_bytes(self.h)

    def footprint(self):
        t, m = C.c_uint64(), C.c_uint64()
        lib().oc_graph_footprint(self.h, C.byref(t), C.byref(m))
        return {"total_bytes": t.value, "max_function_bytes": m.value}

    def min_feasible_budget(self, window, distance=0):
        if distance:
            return lib().oc_min_feasible_budget_distance(self.h, distance)
        return lib().oc_min_feasible_budget(self.h, window)

    def max_feasible_window(self, budget):
        w = C.c_uint64()
        err = oc_err()
        check(lib().oc_max_feasible_window(self.h, budget, C.byref(w), C.byref(err)), err)
        return w.value

    def plan(self, budget, window=OC_WINDOW_MAX_FEASIBLE, mode=OC_ALLOC_VA, chunk_bytes=40 << 20,
             phys_bytes=0, align=512, allow_oom=False, distance=0):
        """distance = 0: the paper's byte window; d >= 1: prior-art function-distance window (F1)."""
        p = oc_plan_params(budget, window, oc_alloc_model(mode, align, chunk_bytes, phys_bytes), distance, 0)
        h = P()
        err = oc_err()
        rc = lib().oc_plan_schedule(self.h, C.byref(p), C.byref(h), C.byref(err))
        if rc == OC_E_DEVICE_OOM and allow_oom and h:
            return Schedule(h, self, oom=OcError(rc, err))
        check(rc, err)
        return Schedule(h, self)


class Schedule:
    def __init__(self, h, graph, oom=None):
        self.h = h
        self.graph = graph   # keeps the graph alive
        self.oom = oom

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().oc_schedule_destroy(self.h)
            except TypeError:      # interpreter shutdown
                pass
            self.h = None

    def json(self):
        need = C.c_size_t()
        lib().oc_schedule_json(self.h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value + 1)
        rc = lib().oc_schedule_json(self.h, buf, need.value + 1, C.byref(need))
        if rc != OC_OK:
            raise RuntimeError(rc)
        return buf.value.decode()

    def stats(self):
        s = oc_sched_stats()
        lib().oc_schedule_stats(self.h, C.byref(s))
        return {k: getattr(s, k) for k, _ in oc_sched_stats._fields_}

    def window_ends(self):
        n = self.graph.n_fns
        arr = (C.c_int64 * max(n, 1))()
        lib().oc_schedule_window_ends(self.h, arr, n)
        return list(arr[:n])

    def simulate(self, fn_ms, h2d_gbs, d2h_gbs, h2d_us=0.0, d2h_us=0.0, elide_clean=True, model=0):
        """Makespan model of the step (oc_simulate); model 0 = the
        paper's boundary semantics, 1 = the executor's placement-aware ordering."""
        n = self.graph.n_fns
        fn = (C.c_double * max(n, 1))(*[float(x) for x in fn_ms])
        stall = (C.c_double * max(n, 1))()
        res = oc_sim_result()
        link = oc_link_model(h2d_gbs, d2h_gbs, h2d_us, d2h_us, 1 if elide_clean else 0, model)
        rc = lib().oc_simulate(self.h, fn, n, C.byref(link), C.byref(res), stall)
        if rc != OC_OK:
            raise OcError(rc, oc_err())
        out = {k: getattr(res, k) for k, _ in oc_sim_result._fields_}
        out["stall_per_fn_ms"] = list(stall[:n])
        return out
