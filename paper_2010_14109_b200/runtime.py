"""Python front end of the out-of-core step: plans a schedule (oc_plan_schedule),
creates the VA pool (oc_mem_create) and the executor (oc_exec_create) on CUDA
streams owned by PyTorch, binds device-resident (pinned) variables to torch
tensors, and exposes the executor's host copies as numpy views.  Marshalling
only — every step of the path runs in liboocore."""
import ctypes as C
import json

import numpy as np
import torch

from . import binding as B

_NP = {"f32": np.float32, "i32": np.int32, "u8": np.uint8, "bf16": np.uint16}


class OutOfCoreStep:
    def __init__(self, doc, budget, window=B.OC_WINDOW_MAX_FEASIBLE, mode="va", chunk_bytes=40 << 20,
                 phys_bytes=0, device=0, timeline=False, elide_clean=True, align=512, meta=None,
                 pack_threshold=64 << 10, use_graph=False, distance=0, trigger=0):
        if not torch.cuda.is_available():
            raise RuntimeError("OutOfCoreStep needs a CUDA device (no CPU fallback)")
        self.device = device
        self.doc = doc
        d = json.loads(doc)
        self.names = [v["id"] for v in d["variables"]]
        self.var_bytes = {v["id"]: v["bytes"] for v in d["variables"]}
        self.pinned = {v["id"] for v in d["variables"] if v.get("pinned")}
        self.id = {n: i for i, n in enumerate(self.names)}
        self.meta = meta or {}
        self.graph = B.Graph(doc)
        m = {"va": B.OC_ALLOC_VA, "best": B.OC_ALLOC_ARENA_BEST, "first": B.OC_ALLOC_ARENA_FIRST}[mode]
        self.mode = mode
        self.sched = self.graph.plan(budget, window, m, chunk_bytes=chunk_bytes, phys_bytes=phys_bytes, align=align,
                                     distance=distance)
        st = self.sched.stats()
        self.stats = st
        pool = phys_bytes or (budget - st["pinned_bytes"])
        if mode != "va":
            pool = max(pool, st["peak_phys"])
        torch.cuda.set_device(device)
        self.streams = [torch.cuda.Stream(device) for _ in range(3)]
        self.mem = B.P()
        err = B.oc_err()
        B.check(B.lib().oc_mem_create(device, C.byref(B.oc_alloc_model(m, align, chunk_bytes, pool)), 0,
                                      C.byref(self.mem), C.byref(err)), err)
        self.exec = B.P()
        ss = B.oc_streams(self.streams[0].cuda_stream, self.streams[1].cuda_stream, self.streams[2].cuda_stream)
        opt = B.oc_exec_options(1 if timeline else 0, 1 if elide_clean else 0, 0, int(pack_threshold),
                                1 if use_graph else 0, int(trigger))
        B.check(B.lib().oc_exec_create(device, self.graph.h, self.sched.h, self.mem, C.byref(ss), C.byref(opt),
                                       C.byref(self.exec), C.byref(err)), err)
        # device-resident (pinned) variables live in torch tensors bound to the executor
        self.dev = {}
        for n in self.pinned:
            t = torch.zeros(self.var_bytes[n], dtype=torch.uint8, device=f"cuda:{device}")
            self.dev[n] = t
            B.check(B.lib().oc_exec_bind_device(self.exec, self.id[n], C.c_void_p(t.data_ptr()), C.byref(err)), err)

    # ----------------------------------------------------------- data access
    def host(self, name, dtype=np.float32):
        """numpy view of the executor's pinned host copy of a variable."""
        p = C.c_void_p()
        err = B.oc_err()
        B.check(B.lib().oc_exec_host_ptr(self.exec, self.id[name], C.byref(p), C.byref(err)), err)
        n = self.var_bytes[name] // np.dtype(dtype).itemsize
        buf = (C.c_char * self.var_bytes[name]).from_address(p.value)
        return np.frombuffer(buf, dtype=dtype, count=n)

    def device_tensor(self, name, dtype=torch.float32):
        return self.dev[name].view(dtype)

    def write(self, name, array):
        """Copy values into a variable (host copy, or device tensor if pinned)."""
        a = np.ascontiguousarray(array)
        if name in self.pinned:
            t = torch.from_numpy(a.view(np.uint8).reshape(-1).copy())
            self.dev[name].copy_(t)
        else:
            self.host(name, a.dtype)[:] = a.reshape(-1)

    def read(self, name, dtype=np.float32):
        if name in self.pinned:
            torch.cuda.synchronize(self.device)
            return self.dev[name].cpu().numpy().view(dtype).copy()
        return self.host(name, dtype).copy()

    # ----------------------------------------------------------- execution
    def step(self):
        m = B.oc_step_metrics()
        err = B.oc_err()
        B.check(B.lib().oc_run_step(self.exec, C.byref(m), C.byref(err)), err)
        return {k: getattr(m, k) for k, _ in B.oc_step_metrics._fields_}

    def host_info(self):
        """(pinned host pool bytes, NUMA node of its pages or -1)."""
        n, node = C.c_uint64(), C.c_int()
        B.lib().oc_exec_host_info(self.exec, C.byref(n), C.byref(node))
        return n.value, node.value

    def set_timeline(self, on):
        """Per-event timeline on/off for the next steps (created with timeline=True)."""
        rc = B.lib().oc_exec_set_timeline(self.exec, 1 if on else 0)
        if rc != B.OC_OK:
            raise RuntimeError("set_timeline: the executor was created without timeline events")

    def timeline(self):
        need = C.c_size_t()
        B.lib().oc_exec_timeline(self.exec, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value + 1)
        B.lib().oc_exec_timeline(self.exec, buf, need.value + 1, C.byref(need))
        return [json.loads(x) for x in buf.value.decode().splitlines() if x]

    def mem_stats(self):
        s = B.oc_mem_stats()
        B.lib().oc_mem_get_stats(self.mem, C.byref(s))
        return {k: getattr(s, k) for k, _ in B.oc_mem_stats._fields_}

    # ------------------------------------------------ layer-local inspection
    def set_hook(self, fn):
        """fn(position, phase) is called before (0) and after (1) the kernels of
        each function, device synchronised, eager issue (oc_exec_set_hook).
        None removes it."""
        if fn is None:
            self._hook = B.OC_FN_HOOK()
        else:
            self._hook = B.OC_FN_HOOK(lambda user, i, phase: fn(int(i), int(phase)))
        B.check(B.lib().oc_exec_set_hook(self.exec, self._hook, None), B.oc_err())

    def read_device(self, name, dtype=np.uint8):
        """Current device bytes of a resident (or pinned) variable (oc_exec_read_var)."""
        n = self.var_bytes[name]
        out = np.empty(n, dtype=np.uint8)
        err = B.oc_err()
        B.check(B.lib().oc_exec_read_var(self.exec, self.id[name], out.ctypes.data_as(C.c_void_p), n,
                                         C.byref(err)), err)
        return out.view(dtype)

    def attach_nccl(self, uid_bytes, rank, nranks):
        err = B.oc_err()
        buf = C.create_string_buffer(bytes(uid_bytes), 128)
        B.check(B.lib().oc_exec_attach_nccl(self.exec, buf, rank, nranks, C.byref(err)), err)

    def attach_comm(self, fn):
        """Custom communicator (oc_exec_attach_comm): fn(dev_ptr, count, stream)
        averages `count` fp32 values at the device address over the replicas."""
        self._comm = B.OC_ALLREDUCE_FN(lambda user, buf, count, stream: int(fn(buf, int(count), stream) or 0))
        err = B.oc_err()
        B.check(B.lib().oc_exec_attach_comm(self.exec, self._comm, None, C.byref(err)), err)

    def close(self):
        if getattr(self, "exec", None):
            B.lib().oc_exec_destroy(self.exec)
            self.exec = None
        if getattr(self, "mem", None):
            B.lib().oc_mem_destroy(self.mem)
            self.mem = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id():
    buf = C.create_string_buffer(128)
    err = B.oc_err()
    B.check(B.lib().oc_nccl_unique_id(buf, C.byref(err)), err)
    return buf.raw
