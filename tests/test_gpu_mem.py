"""The allocator C-ABI on the GPU (SURVEY §8(b) "Memory" row; A4): the VA
chunk pool on the CUDA VMM API and the caching arena, called directly through
oc_mem_create / oc_alloc / oc_map / oc_unmap / oc_free — Eq.1 sizes and
internal fragmentation, OOM iff free chunks < k,
error codes, data written through one mapping read back after a
remap, the paper-literal eager unmap (OC_MEM_EAGER_UNMAP) and the best-fit
external-fragmentation example."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2010_14109_b200 import binding as B

MiB = 1 << 20


def _cudart():
    from cuda.bindings import runtime as rt
    return rt


def _h2d(va, arr):
    rt = _cudart()
    (e,) = rt.cudaMemcpy(va, arr.ctypes.data, arr.nbytes, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
    assert int(e) == 0


def _d2h(va, nbytes):
    rt = _cudart()
    out = np.empty(nbytes, np.uint8)
    (e,) = rt.cudaMemcpy(out.ctypes.data, va, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert int(e) == 0
    return out


def _code(fn):
    with pytest.raises(B.OcError) as ei:
        fn()
    return ei.value.code


@pytest.mark.gpu
def test_va_pool_eq1_oom_and_remap():
    torch.cuda.init()
    m = B.Mem(mode=B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=8 * MiB)   # 4 chunks
    a = m.alloc(5 * MiB)                       # Eq.1: k = 3, m_a = 6 MiB, IF = 1 MiB
    assert (a.m_r, a.m_a) == (5 * MiB, 6 * MiB)
    b = m.alloc(3 * MiB)                       # k = 2
    sa = m.map(a.handle)
    assert sa.va == a.va != 0
    st = m.stats()
    assert st["free_chunks"] == 1 and st["internal_frag"] == 1 * MiB and st["live_count"] == 1
    assert _code(lambda: m.map(b.handle)) == B.OC_E_DEVICE_OOM    # 1 free chunk < k = 2
    rng = np.random.default_rng(0)
    data = rng.integers(0, 256, 5 * MiB, dtype=np.uint8)
    _h2d(sa.va, data)
    assert np.array_equal(_d2h(sa.va, 5 * MiB), data)
    m.unmap(a.handle)
    torch.cuda.synchronize()
    sb = m.map(b.handle)                       # chunks reused after a's release (physical memory recycled)
    assert sb.va == b.va and m.stats()["free_chunks"] == 2
    data_b = rng.integers(0, 256, 3 * MiB, dtype=np.uint8)
    _h2d(sb.va, data_b)
    assert np.array_equal(_d2h(sb.va, 3 * MiB), data_b)
    assert _code(lambda: m.map(a.handle)) == B.OC_E_DEVICE_OOM    # 2 free chunks < k = 3
    m.unmap(b.handle)
    m.free(b.handle)
    assert _code(lambda: m.free(b.handle)) == B.OC_E_DOUBLE_FREE
    assert _code(lambda: m.map(12345)) == B.OC_E_UNKNOWN_HANDLE
    m.free(a.handle)
    st = m.stats()
    assert st["live_count"] == 0 and st["n_max"] >= 1 and st["if_peak"] >= 1 * MiB
    m.close()


@pytest.mark.gpu
def test_va_pool_exact_multiples_have_no_internal_fragmentation():
    torch.cuda.init()
    m = B.Mem(mode=B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=16 * MiB)
    spans = [m.alloc(k * 2 * MiB) for k in (1, 2, 3)]
    for s in spans:
        m.map(s.handle)
    st = m.stats()
    assert st["internal_frag"] == 0 and st["free_chunks"] == 2 and st["live_count"] == 3
    for s in spans:
        m.unmap(s.handle)
        m.free(s.handle)
    m.close()


@pytest.mark.gpu
def test_va_eager_unmap_releases_mappings():
    torch.cuda.init()
    m = B.Mem(mode=B.OC_ALLOC_VA, chunk_bytes=2 * MiB, phys_bytes=8 * MiB, flags=B.OC_MEM_EAGER_UNMAP)
    a = m.alloc(4 * MiB)
    m.map(a.handle)
    m.unmap(a.handle)
    torch.cuda.synchronize()
    b = m.alloc(2 * MiB)
    m.map(b.handle)                            # polls the deferred list: a's completed release is unmapped
    st = m.stats()
    assert st["n_driver_unmap"] >= 1 and st["n_driver_map"] >= 2
    m.unmap(b.handle)
    m.free(a.handle)
    m.free(b.handle)
    m.close()


@pytest.mark.gpu
def test_arena_best_fit_external_fragmentation():
    """S:258 with MiB units: capacity 10, A = 10 freed, B = 6, C = 5 -> OOM
    although 4 MiB are cached free (no coalescing with fresh capacity)."""
    torch.cuda.init()
    m = B.Mem(mode=B.OC_ALLOC_ARENA_BEST, phys_bytes=10 * MiB, align=512)
    a = m.alloc(10 * MiB)
    m.free(a.handle)
    b = m.alloc(6 * MiB)
    assert _code(lambda: m.alloc(5 * MiB)) == B.OC_E_DEVICE_OOM
    st = m.stats()
    assert st["arena_free_cached"] == 4 * MiB
    data = np.arange(6 * MiB, dtype=np.uint8)
    _h2d(b.va, data)
    assert np.array_equal(_d2h(b.va, 6 * MiB), data)
    m.free(b.handle)
    m.close()
