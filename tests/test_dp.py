"""Data-parallel replicas: host-side logic on CPU with the
gloo backend at world size 2, the DP oracle (C7), and the NCCL path of the
executor on one GPU (world size 1: ncclAvg over one rank is the identity)."""
import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numerics as nm
from synth import nets


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dp_oracle_average_equals_full_batch_for_mlp():
    """C7: for a net without batch statistics the mean of the per-replica
    gradients over equal shards equals the full-batch gradient (fp64)."""
    spec = nets.mlp6(batch=8, width=32, classes=10)
    spec["mode"] = "fp64"
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    full = nm.train_step(spec, p, x, y)["grads"]
    half = dict(spec, batch=4)
    g0 = nm.train_step(half, p, x[:4], y[:4])["grads"]
    g1 = nm.train_step(half, p, x[4:], y[4:])["grads"]
    for k in p:
        assert np.allclose((g0[k] + g1[k]) / 2, full[k], rtol=1e-12, atol=1e-15)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    # every replica plans the identical schedule (identical shapes) — compare hashes
    spec = nets.resnet(18, batch=64)
    doc, _ = graphs.build(spec, params="persistent")
    G = B.Graph(doc)
    budget = G.in_core_peak() // 4
    s = G.plan(budget, G.max_feasible_window(budget), B.OC_ALLOC_VA, chunk_bytes=2 << 20,
               phys_bytes=budget * 4, allow_oom=True)
    h = hashlib.sha256(s.json().encode()).hexdigest()
    hs = [None] * world
    dist.all_gather_object(hs, h)
    # the bench's NCCL unique-id exchange: rank 0's 128 bytes reach every rank
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    # per-replica shard of the MLP through the oracle, gradients averaged (the NCCL ncclAvg step)
    mspec = nets.mlp6(batch=8, width=32, classes=10)
    mspec["mode"] = "fp64"
    x, y = nets.make_inputs(mspec)
    p = nets.make_params(mspec)
    shard = dict(mspec, batch=8 // world)
    lo = rank * (8 // world)
    g = nm.train_step(shard, p, x[lo:lo + 8 // world], y[lo:lo + 8 // world])["grads"]
    avg = {}
    for k in sorted(g):
        t = torch.from_numpy(np.ascontiguousarray(g[k]))
        dist.all_reduce(t)
        avg[k] = (t / world).numpy()
    if rank == 0:
        full = nm.train_step(mspec, p, x, y)["grads"]
        err = max(float(np.max(np.abs(avg[k] - full[k]))) for k in full)
        out.put({"hashes": hs, "uid_ok": uid[0] == bytes(range(128)), "max_err": err})
    dist.destroy_process_group()


def test_dp_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = q.get(timeout=300)
    for p_ in ps:
        p_.join(timeout=60)
    assert len(set(res["hashes"])) == 1
    assert res["uid_ok"]
    assert res["max_err"] < 1e-12


@pytest.mark.gpu
def test_nccl_single_rank_step_identical():
    """The executor's NCCL path: a communicator over one rank makes every
    per-layer allreduce(avg) an identity, so the step equals the no-NCCL step
    bitwise."""
    from paper_2010_14109_b200 import graphs
    from paper_2010_14109_b200.runtime import OutOfCoreStep, nccl_unique_id
    spec = nets.mlp6()
    doc, info = graphs.build(spec, params="persistent")
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    outs = []
    for use_nccl in (False, True):
        st = OutOfCoreStep(doc, 4 << 20, 2 ** 64 - 1, mode="best", phys_bytes=8 << 20)
        if use_nccl:
            st.attach_nccl(nccl_unique_id(), 0, 1)
        st.write(info["x"], x)
        st.write(info["labels"], y)
        for k, v in p.items():
            st.write(info["params"][k], v)
            st.write(info["momentum"][k], np.zeros_like(v))
        st.step()
        outs.append({k: st.read(info["params"][k]) for k in p})
        st.close()
    for k in p:
        assert np.array_equal(outs[0][k], outs[1][k]), k


@pytest.mark.gpu
def test_nccl_single_rank_bucketed_resnet_identical():
    """The bench's N > 1 configuration on one rank: a bf16 tiny ResNet with
    bucketed allreduce functions (graphs.build(dp_bucket_bytes=...), one
    ncclGroup per bucket on the executor's communication stream, SGD one
    bucket later) under a swap-forcing budget; a one-rank NCCL communicator
    makes every exchange an identity, so the step equals the step without a
    communicator bitwise — the NCCL plumbing (dlopen, unique id, comm init,
    group calls, comm-stream ordering) runs on the GPU."""
    from paper_2010_14109_b200 import binding as B
    from paper_2010_14109_b200 import graphs
    from paper_2010_14109_b200.runtime import OutOfCoreStep, nccl_unique_id
    spec = nets.tiny_resnet(batch=4, image=16, classes=10)
    doc, info = graphs.build(spec, params="persistent", dp_bucket_bytes=16 << 10)
    assert sum(1 for f in json.loads(doc)["functions"] if f["op"]["kind"] == "allreduce") > 1
    G = B.Graph(doc)
    budget = max(G.min_feasible_budget(0), int(G.in_core_peak() * 0.5))
    x, y = nets.make_inputs(spec)
    p = nets.make_params(spec)
    phys = G.plan(budget, 0, B.OC_ALLOC_VA, chunk_bytes=2 << 20, phys_bytes=8 * budget + (1 << 30),
                  allow_oom=True).stats()["peak_phys"] + (2 << 20)
    xb = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).view(torch.int16).numpy()
    outs = []
    for use_nccl in (False, True):
        st = OutOfCoreStep(doc, budget, 0, mode="va", chunk_bytes=2 << 20, phys_bytes=phys)
        if use_nccl:
            st.attach_nccl(nccl_unique_id(), 0, 1)
        st.write(info["x"], xb)
        st.write(info["labels"], y)
        for k, v in p.items():
            st.write(info["params"][k], v)
            st.write(info["momentum"][k], np.zeros_like(v))
        m = st.step()
        assert m["bytes_d2h"] > 0
        outs.append({k: st.read(info["params"][k]) for k in p})
        st.close()
    for k in p:
        assert np.array_equal(outs[0][k], outs[1][k]), k
