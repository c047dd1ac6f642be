"""Data-parallel step with TWO replica processes on the one GPU of the test box
(SURVEY §8(e)): each rank runs its own out-of-core executor (own budget, VA
pool, host copies) on its shard of the batch, and the gradient buckets are
averaged through the executor's allreduce functions on its communication
stream — with a custom communicator (oc_exec_attach_comm) that exchanges
through torch.distributed gloo, since NCCL needs one GPU per rank.  This runs
the whole DP plumbing of the executor: bucket functions, the comm stream
fork/join, consumers waiting for the exchange, deferred multi-tensor SGD.

Checked against the DP oracle C7 (per-replica BN statistics, gradients
averaged, then SGD): fp32 mode (CUDA-core convs) within 1e-5 on every updated
parameter; and in bf16 with tensor cores, two replicas on IDENTICAL shards
must reproduce the single-replica step bitwise (the mean of equal fp32
gradients is exact)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numerics as nm
from synth import nets

MiB = 1 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cudart():
    for name in ("libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12", "libcudart.so"):
        try:
            return C.CDLL(name)
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def _replica(rank, world, port, spec, shards, identical, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    rt = _cudart()
    rt.cudaStreamSynchronize.argtypes = [C.c_void_p]
    rt.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    n_calls = [0]

    def gloo_mean(buf, count, stream):
        rt.cudaStreamSynchronize(stream)
        host = np.empty(count, np.float32)
        assert rt.cudaMemcpy(host.ctypes.data, buf, count * 4, 2) == 0
        t = torch.from_numpy(host)
        dist.all_reduce(t)
        t /= world
        assert rt.cudaMemcpy(buf, host.ctypes.data, count * 4, 1) == 0
        n_calls[0] += 1
        return 0

    local = dict(spec, batch=spec["batch"] // world)
    doc, info = graphs.build(local, params="persistent", dp_bucket_bytes=64 << 10)
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(0), G.in_core_peak() // 3)
    probe = G.plan(budget, B.OC_WINDOW_MAX_FEASIBLE, B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=1 << 40,
                   allow_oom=True).stats()
    st = OutOfCoreStep(doc, budget, B.OC_WINDOW_MAX_FEASIBLE, mode="va", chunk_bytes=2 * MiB,
                       phys_bytes=probe["peak_phys"] + 2 * MiB)
    st.attach_comm(gloo_mean)
    x, y = shards[0 if identical else rank]
    p = nets.make_params(spec)
    st.write(info["x"], x.astype(np.float32) if spec["mode"] == "fp32"
             else torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    met = st.step()
    res = {k: st.read(info["params"][k]).reshape(p[k].shape) for k in p}
    n_buckets = sum(1 for f in __import__("json").loads(doc)["functions"] if f["op"]["kind"] == "allreduce")
    st.close()
    if rank == 0:
        out_q.put({"params": res, "bytes_d2h": met["bytes_d2h"], "calls": n_calls[0], "buckets": n_buckets})
    dist.destroy_process_group()


def _run_dp(spec, shards, identical=False, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica, args=(r, world, port, spec, shards, identical, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def _shards(spec, world=2):
    x, y = nets.make_inputs(spec)
    n = spec["batch"] // world
    return [(x[r * n:(r + 1) * n], y[r * n:(r + 1) * n]) for r in range(world)]


@pytest.mark.gpu
def test_dp_two_replicas_fp32_matches_dp_oracle():
    spec = nets.tiny_resnet(batch=8, image=16, classes=10, mode="fp32")
    shards = _shards(spec)
    out = _run_dp(spec, shards)
    assert out["bytes_d2h"] > 0 and out["buckets"] > 1
    # oracle C7: per-replica steps (own BN statistics), gradients averaged, SGD from zero momentum
    p = nets.make_params(spec)
    half = dict(spec, batch=spec["batch"] // 2)
    gs = [nm.train_step(half, p, x, y)["grads"] for x, y in shards]
    lr, mu = spec["sgd"]["lr"], spec["sgd"]["momentum"]
    for k in p:
        g = nm.round_fp32((gs[0][k] + gs[1][k]) / 2)
        want = nm.round_fp32(np.asarray(p[k], np.float64) - lr * g)
        assert nm.rel_l2(out["params"][k], want) <= 1e-5, k


@pytest.mark.gpu
def test_dp_identical_shards_bf16_equals_single_replica():
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from paper_2010_14109_b200.runtime import OutOfCoreStep
    spec = nets.tiny_resnet(batch=8, image=16, classes=10)
    shards = _shards(spec)
    out = _run_dp(spec, shards, identical=True)
    # the single replica on the same shard, no communicator, per-layer updates
    local = dict(spec, batch=spec["batch"] // 2)
    doc, info = graphs.build(local, params="persistent")
    G = B.Graph(doc)
    peak = G.in_core_peak()
    st = OutOfCoreStep(doc, peak, 0, mode="best", phys_bytes=peak * 2)
    x, y = shards[0]
    p = nets.make_params(spec)
    st.write(info["x"], torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy())
    st.write(info["labels"], y)
    for k, v in p.items():
        st.write(info["params"][k], v)
        st.write(info["momentum"][k], np.zeros_like(v))
    st.step()
    for k in p:
        assert np.array_equal(st.read(info["params"][k]).reshape(p[k].shape), out["params"][k]), k
    st.close()
