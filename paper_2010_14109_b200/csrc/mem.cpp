// Virtual-addressing chunk allocator on the CUDA driver VMM API (§4,
// P:104-120) and the caching-arena alternative.
//
//   VA:    physical chunks of m_c bytes (cuMemCreate, lazily) are mapped to a
//          span of consecutive virtual addresses reserved per request
//          (cuMemAddressReserve); m_a = ⌈m_r/m_c⌉·m_c (Eq.1).  A released span
//          returns its chunks to a FIFO pool ("cache physical memories for the
//          future requests").  Driver calls are the cost the paper
//          names; measured on B200: cuMemSetAccess ≈150 µs and
//          cuMemUnmap ≈100 µs per chunk mapping, cuMemMap ≈1 µs
//          (profiles/r01_box_phase0.txt) — so mappings are memoised: a span
//          keeps its chunk mapping after release and is re-mapped only when it
//          next receives different chunks (or eagerly, OC_MEM_EAGER_UNMAP).
//   arena: one slab, best-/first-fit placement with the planner's rules.
// Device-side hazards are ordered with per-chunk (VA) or per-range (arena)
// release events; nothing here blocks the host on the device except the
// unmap of a span whose last use has not finished.
#include "mem.hpp"

#include <chrono>
#include <cstring>
#include <mutex>

namespace oc {

static std::once_flag g_drv_once;
static Driver g_drv;
static std::string g_drv_msg;

bool driver(Driver*& d, std::string& msg) {
  std::call_once(g_drv_once, [] {
    cudaDriverEntryPointQueryResult q;
    auto get = [&](const char* name, void** fn) {
      cudaError_t e = cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q);
      if (e != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        g_drv_msg += std::string("missing driver entry point ") + name + "; ";
        return false;
      }
      return true;
    };
    bool ok = true;
    ok &= get("cuMemCreate", (void**)&g_drv.MemCreate);
    ok &= get("cuMemRelease", (void**)&g_drv.MemRelease);
    ok &= get("cuMemAddressReserve", (void**)&g_drv.MemAddressReserve);
    ok &= get("cuMemAddressFree", (void**)&g_drv.MemAddressFree);
    ok &= get("cuMemMap", (void**)&g_drv.MemMap);
    ok &= get("cuMemUnmap", (void**)&g_drv.MemUnmap);
    ok &= get("cuMemSetAccess", (void**)&g_drv.MemSetAccess);
    ok &= get("cuMemGetAllocationGranularity", (void**)&g_drv.MemGetAllocationGranularity);
    ok &= get("cuGetErrorString", (void**)&g_drv.GetErrorString);
    ok &= get("cuTensorMapEncodeTiled", (void**)&g_drv.TensorMapEncodeTiled);
    ok &= get("cuTensorMapEncodeIm2col", (void**)&g_drv.TensorMapEncodeIm2col);
    g_drv.loaded = ok;
  });
  d = &g_drv;
  msg = g_drv_msg;
  return g_drv.loaded;
}

Status cu_status(CUresult r, const char* what) {
  const char* s = "unknown";
  if (g_drv.GetErrorString) g_drv.GetErrorString(r, &s);
  Status st = Status::make(OC_E_CUDA, std::string(what) + ": " + s);
  st.cuda = (int)r;
  return st;
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Status MemPool::init(int dev, const oc_alloc_model& m, uint32_t fl) {
  device = dev;
  model = m;
  flags = fl;
  OC_CUDA(cudaSetDevice(dev));
  OC_CUDA(cudaFree(0));
  std::string msg;
  if (!driver(drv, msg)) return Status::make(OC_E_CUDA, msg);
  std::memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  OC_CU(drv->MemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  std::memset(&access, 0, sizeof(access));
  access.location = prop.location;
  access.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (m.mode == OC_ALLOC_VA) {
    if (m.chunk_bytes == 0 || m.chunk_bytes % gran)
      return Status::make(OC_E_ARG, "chunk_bytes must be a positive multiple of the VMM granularity (" +
                                        std::to_string(gran) + ")");
    m_c = m.chunk_bytes;
    n_chunks = (uint32_t)(m.phys_bytes / m_c);
    chunk.assign(n_chunks, 0);
    chunk_ev.assign(n_chunks, nullptr);
    chunk_ev_used.assign(n_chunks, 0);
    for (uint32_t c = 0; c < n_chunks; ++c) {
      free_q.push_back(c);
      OC_CUDA(cudaEventCreateWithFlags(&chunk_ev[c], cudaEventDisableTiming));
    }
  } else if (m.mode == OC_ALLOC_ARENA_BEST || m.mode == OC_ALLOC_ARENA_FIRST) {
    slab_bytes = (m.phys_bytes + gran - 1) / gran * gran;
    if (slab_bytes) {
      OC_CU(drv->MemCreate(&slab_h, slab_bytes, &prop, 0));
      OC_CU(drv->MemAddressReserve(&slab, slab_bytes, 0, 0, 0));
      OC_CU(drv->MemMap(slab, slab_bytes, 0, slab_h, 0));
      OC_CU(drv->MemSetAccess(slab, slab_bytes, &access, 1));
    }
    placer.init(m.phys_bytes, m.align ? m.align : 512, m.mode == OC_ALLOC_ARENA_BEST);
  } else {
    return Status::make(OC_E_ARG, "unknown allocator mode");
  }
  return Status::ok();
}

Status MemPool::ensure_chunk(uint32_t c) {
  if (!chunk[c]) OC_CU(drv->MemCreate(&chunk[c], m_c, &prop, 0));
  return Status::ok();
}

Status MemPool::reserve(uint64_t m_a, CUdeviceptr& va) {
  OC_CU(drv->MemAddressReserve(&va, m_a, 0, 0, 0));
  return Status::ok();
}

Status MemPool::driver_unmap(Span& s) {
  if (s.mapped.empty()) return Status::ok();
  double t0 = now_us();
  OC_CU(drv->MemUnmap(s.va, s.mapped.size() * m_c));
  unmap_us += now_us() - t0;
  ++n_driver_unmap;
  s.mapped.clear();
  return Status::ok();
}

Status MemPool::bind(Span& s, const std::vector<uint32_t>& chunks) {
  ++n_map_calls;
  if (s.mapped == chunks) {  // memoised: the span already maps exactly these chunks
    ++n_map_memo_hits;
    return Status::ok();
  }
  if (!s.mapped.empty()) {
    // the span's previous use must be complete before its VA is re-pointed
    if (s.ev_used) OC_CUDA(cudaEventSynchronize(s.ev));
    OC_TRY(driver_unmap(s));
  }
  double t0 = now_us();
  for (size_t j = 0; j < chunks.size(); ++j) {
    OC_TRY(ensure_chunk(chunks[j]));
    OC_CU(drv->MemMap(s.va + j * m_c, m_c, 0, chunk[chunks[j]], 0));
  }
  OC_CU(drv->MemSetAccess(s.va, chunks.size() * m_c, &access, 1));
  map_us += now_us() - t0;
  ++n_driver_map;
  s.mapped = chunks;
  return Status::ok();
}

void MemPool::poll_deferred() {
  for (size_t k = 0; k < deferred.size();) {
    Span& s = spans[deferred[k]];
    if (!s.ev_used || cudaEventQuery(s.ev) == cudaSuccess) {
      driver_unmap(s);
      deferred[k] = deferred.back();
      deferred.pop_back();
    } else {
      ++k;
    }
  }
}

cudaEvent_t MemPool::take_event() {
  if (!ev_pool.empty()) {
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

void MemPool::poll_released() {
  for (size_t k = 0; k < released.size();) {
    if (cudaEventQuery(released[k].ev) == cudaSuccess) {
      ev_pool.push_back(released[k].ev);
      released[k] = released.back();
      released.pop_back();
      continue;
    }
    ++k;
  }
  (void)cudaGetLastError();   // cudaErrorNotReady from the queries is not an error
}

void MemPool::destroy() {
  cudaSetDevice(device);
  cudaDeviceSynchronize();
  for (auto& kv : spans) {
    Span& s = kv.second;
    if (!s.mapped.empty()) drv->MemUnmap(s.va, s.mapped.size() * m_c);
    if (s.va) drv->MemAddressFree(s.va, s.m_a);
    if (s.ev) cudaEventDestroy(s.ev);
  }
  spans.clear();
  for (auto& r : released)
    if (r.ev) cudaEventDestroy(r.ev);
  released.clear();
  for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  ev_pool.clear();
  for (uint32_t c = 0; c < chunk.size(); ++c) {
    if (chunk[c]) drv->MemRelease(chunk[c]);
    if (chunk_ev[c]) cudaEventDestroy(chunk_ev[c]);
  }
  chunk.clear();
  if (slab) {
    drv->MemUnmap(slab, slab_bytes);
    drv->MemAddressFree(slab, slab_bytes);
    drv->MemRelease(slab_h);
    slab = 0;
  }
}

}  // namespace oc

using namespace oc;

extern "C" {

int oc_mem_create(int device, const oc_alloc_model* model, uint32_t flags, oc_mem** out, oc_err* err) {
  if (!model || !out) return OC_E_ARG;
  *out = nullptr;
  oc_mem* m = new oc_mem();
  Status st = m->p.init(device, *model, flags);
  if (!st.good()) {
    st.fill(err);
    m->p.destroy();
    delete m;
    return st.code;
  }
  *out = m;
  return OC_OK;
}

int oc_alloc(oc_mem* m, uint64_t bytes, oc_span* out, oc_err* err) {
  if (!m || !out || bytes == 0) return OC_E_ARG;
  MemPool& P = m->p;
  cudaSetDevice(P.device);
  Span s;
  s.m_r = bytes;
  if (P.model.mode == OC_ALLOC_VA) {
    s.k = (uint32_t)((bytes + P.m_c - 1) / P.m_c);
    s.m_a = (uint64_t)s.k * P.m_c;
    Status st = P.reserve(s.m_a, s.va);
    if (!st.good()) { st.fill(err); return st.code; }
    cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming);
  } else {
    uint64_t off = 0;
    uint64_t h = P.next_handle;
    if (!P.placer.alloc(h, bytes, off)) {
      Status st = Status::make(OC_E_DEVICE_OOM, "arena: no block fits");
      st.needed = bytes;
      st.free_bytes = P.placer.free_bytes();
      st.fill(err);
      return st.code;
    }
    s.offset = off;
    s.va = P.slab + off;
    s.m_a = (bytes + P.placer.align - 1) / P.placer.align * P.placer.align;
    s.live = true;
  }
  s.handle = P.next_handle++;
  P.live_requested += bytes;
  P.live_allocated += s.m_a;
  out->handle = s.handle;
  out->va = s.va;
  out->m_r = s.m_r;
  out->m_a = s.m_a;
  P.spans[s.handle] = s;
  return OC_OK;
}

int oc_map(oc_mem* m, uint64_t handle, void* consumer_stream, oc_span* out, oc_err* err) {
  if (!m) return OC_E_ARG;
  MemPool& P = m->p;
  cudaSetDevice(P.device);
  auto it = P.spans.find(handle);
  if (it == P.spans.end()) {
    Status st = Status::make(P.freed.count(handle) ? OC_E_DOUBLE_FREE : OC_E_UNKNOWN_HANDLE, "oc_map: bad handle");
    st.fill(err);
    return st.code;
  }
  Span& s = it->second;
  cudaStream_t cs = (cudaStream_t)consumer_stream;
  if (P.model.mode == OC_ALLOC_VA) {
    if (s.live) { Status::make(OC_E_ARG, "span already mapped").fill(err); return OC_E_ARG; }
    P.poll_deferred();
    if (P.free_q.size() < s.k) {
      Status st = Status::make(OC_E_DEVICE_OOM, "VA pool: not enough free chunks");
      st.needed = s.m_r;
      st.free_bytes = P.free_q.size() * P.m_c;
      st.fill(err);
      return st.code;
    }
    std::vector<uint32_t> chunks(P.free_q.begin(), P.free_q.begin() + s.k);
    P.free_q.erase(P.free_q.begin(), P.free_q.begin() + s.k);
    Status st = P.bind(s, chunks);
    if (!st.good()) { st.fill(err); return st.code; }
    for (uint32_t c : chunks)
      if (P.chunk_ev_used[c]) cudaStreamWaitEvent(cs, P.chunk_ev[c], 0);
    s.bound = chunks;
    s.live = true;
    uint64_t mapped = (P.n_chunks - P.free_q.size()) * P.m_c;
    P.peak_mapped = std::max(P.peak_mapped, mapped);
    P.live_count++;
    P.n_max = std::max(P.n_max, P.live_count);
    P.live_if += s.m_a - s.m_r;
    P.if_peak = std::max(P.if_peak, P.live_if);
  } else {
    // wait for every earlier occupant of the block's bytes whose release is
    // still in flight (completed releases are dropped first, so the list holds
    // only in-flight ranges and does not grow with the number of maps)
    P.poll_released();
    const uint64_t a = s.offset, b = s.offset + s.m_a;
    for (size_t k = 0; k < P.released.size();) {
      auto& r = P.released[k];
      if (r.start < b && a < r.end) {
        cudaStreamWaitEvent(cs, r.ev, 0);
        if (a <= r.start && r.end <= b) {  // fully covered: this block's release will imply it
          P.ev_pool.push_back(r.ev);
          P.released[k] = P.released.back();
          P.released.pop_back();
          continue;
        }
      }
      ++k;
    }
    P.live_count++;
    P.n_max = std::max(P.n_max, P.live_count);
    P.peak_mapped = std::max(P.peak_mapped, P.placer.tail);
  }
  if (out) { out->handle = s.handle; out->va = s.va; out->m_r = s.m_r; out->m_a = s.m_a; }
  return OC_OK;
}

int oc_unmap(oc_mem* m, uint64_t handle, void* release_stream, oc_err* err) {
  if (!m) return OC_E_ARG;
  MemPool& P = m->p;
  cudaSetDevice(P.device);
  auto it = P.spans.find(handle);
  if (it == P.spans.end()) {
    Status st = Status::make(P.freed.count(handle) ? OC_E_DOUBLE_FREE : OC_E_UNKNOWN_HANDLE, "oc_unmap: bad handle");
    st.fill(err);
    return st.code;
  }
  Span& s = it->second;
  cudaStream_t rs = (cudaStream_t)release_stream;
  if (!s.live) { Status::make(OC_E_ARG, "span not mapped").fill(err); return OC_E_ARG; }
  if (P.model.mode == OC_ALLOC_VA) {
    cudaEventRecord(s.ev, rs);
    s.ev_used = true;
    for (uint32_t c : s.bound) {
      cudaEventRecord(P.chunk_ev[c], rs);
      P.chunk_ev_used[c] = 1;
      P.free_q.push_back(c);
    }
    s.bound.clear();
    P.live_if -= s.m_a - s.m_r;
    if (P.flags & OC_MEM_EAGER_UNMAP) P.deferred.push_back(handle);
    P.poll_deferred();
  } else {
    MemPool::Released r;
    r.start = s.offset;
    r.end = s.offset + s.m_a;
    r.ev = P.take_event();
    cudaEventRecord(r.ev, rs);
    P.released.push_back(r);
  }
  s.live = false;
  P.live_count--;
  return OC_OK;
}

int oc_free(oc_mem* m, uint64_t handle, oc_err* err) {
  if (!m) return OC_E_ARG;
  MemPool& P = m->p;
  cudaSetDevice(P.device);
  auto it = P.spans.find(handle);
  if (it == P.spans.end()) {
    Status st = Status::make(P.freed.count(handle) ? OC_E_DOUBLE_FREE : OC_E_UNKNOWN_HANDLE, "oc_free: bad handle");
    st.fill(err);
    return st.code;
  }
  Span& s = it->second;
  if (P.model.mode == OC_ALLOC_VA) {
    if (s.live) { Status::make(OC_E_ARG, "free of a mapped span: unmap first").fill(err); return OC_E_ARG; }
    if (s.ev_used) cudaEventSynchronize(s.ev);
    Status st = P.driver_unmap(s);
    if (!st.good()) { st.fill(err); return st.code; }
    for (size_t k = 0; k < P.deferred.size(); ++k)
      if (P.deferred[k] == handle) { P.deferred[k] = P.deferred.back(); P.deferred.pop_back(); break; }
    P.drv->MemAddressFree(s.va, s.m_a);
    cudaEventDestroy(s.ev);
  } else {
    if (s.live) {  // arena: free without unmap releases at the current device point
      P.live_count--;
    }
    P.placer.free(handle);
  }
  P.live_requested -= s.m_r;
  P.live_allocated -= s.m_a;
  P.freed.insert(handle);
  P.spans.erase(it);
  return OC_OK;
}

int oc_mem_get_stats(oc_mem* m, oc_mem_stats* o) {
  if (!m || !o) return OC_E_ARG;
  MemPool& P = m->p;
  std::memset(o, 0, sizeof(*o));
  o->n_chunks = P.n_chunks;
  o->free_chunks = P.free_q.size();
  o->chunk_bytes = P.m_c;
  o->live_requested = P.live_requested;
  o->live_allocated = P.live_allocated;
  o->peak_mapped_bytes = P.peak_mapped;
  o->internal_frag = P.live_if;
  o->if_peak = P.if_peak;
  o->live_count = P.live_count;
  o->n_max = P.n_max;
  o->n_driver_map = P.n_driver_map;
  o->n_driver_unmap = P.n_driver_unmap;
  o->n_map_calls = P.n_map_calls;
  o->n_map_memo_hits = P.n_map_memo_hits;
  o->arena_carved = P.placer.tail;
  o->arena_free_cached = P.placer.free_bytes() - (P.placer.cap - P.placer.tail);
  o->map_us = P.map_us;
  o->unmap_us = P.unmap_us;
  return OC_OK;
}

int oc_mem_reset_order(oc_mem* m, oc_err* err) {
  if (!m) return OC_E_ARG;
  MemPool& P = m->p;
  if (P.free_q.size() != P.n_chunks) {
    Status::make(OC_E_ARG, "oc_mem_reset_order: chunks still mapped").fill(err);
    return OC_E_ARG;
  }
  for (uint32_t c = 0; c < P.n_chunks; ++c) P.free_q[c] = c;
  return OC_OK;
}

void oc_mem_destroy(oc_mem* m) {
  if (!m) return;
  m->p.destroy();
  delete m;
}

}  // extern "C"
