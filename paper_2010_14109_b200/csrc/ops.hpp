// Op registry: the compute of one function f_i (the layer kernels of the
// training step).  An op descriptor in the graph
// document looks like
//   {"kind": "linear_fwd", "args": {"x": var, "w": var, ...}, "attrs": {...}}
// `args` binds the op's roles to variables (a role may take a list of
// variables); `attrs` holds shapes and flags.  The executor resolves roles to
// device addresses before each launch.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "core.hpp"
#include "cuda_util.hpp"

namespace oc {

// Event pairs around the main contraction kernel launches of one function
// (timeline mode only): the bench's roofline divides algorithmic FLOPs by the
// kernel's own launch durations, without the operand re-layout kernels.
struct KernelTimer {
  std::vector<cudaEvent_t> ev;   // 2 per launch, created on demand, reused every step
  size_t used = 0;
  // in-kernel launch probes (tc_util.cuh KProbe): 4 u64 per launch, kMaxProbes launches
  static constexpr size_t kMaxProbes = 64;
  unsigned long long* dprobe = nullptr;
  unsigned long long* probe_slot(cudaStream_t s) {
    const size_t k = used / 2;
    if (k >= kMaxProbes) return nullptr;
    if (!dprobe && cudaMalloc((void**)&dprobe, kMaxProbes * 4 * sizeof(unsigned long long)) != cudaSuccess) {
      dprobe = nullptr;
      return nullptr;
    }
    unsigned long long* p = dprobe + 4 * k;
    cudaMemsetAsync(p, 0xFF, 8, s);
    cudaMemsetAsync(p + 1, 0, 24, s);
    return p;
  }
  // Σ launch spans (ms) and the SM clock the launches ran at (MHz), after the step
  void probe_summary(double& span_ms, double& mhz) const {
    span_ms = 0;
    mhz = 0;
    const size_t n = std::min(used / 2, kMaxProbes);
    if (!dprobe || n == 0) return;
    std::vector<unsigned long long> h(4 * n);
    if (cudaMemcpy(h.data(), dprobe, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
      return;
    double clk = 0, ns = 0;
    for (size_t k = 0; k < n; ++k) {
      if (h[4 * k + 1] < h[4 * k]) continue;   // launch without a probe
      span_ms += (double)(h[4 * k + 1] - h[4 * k]) * 1e-6;
      clk += (double)h[4 * k + 2];
      ns += (double)h[4 * k + 3];
    }
    mhz = ns > 0 ? clk / ns * 1e3 : 0;
  }
  void begin(cudaStream_t s) {
    if (used + 2 > ev.size())
      for (int k = 0; k < 2; ++k) {
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        ev.push_back(e);
      }
    cudaEventRecord(ev[used], s);
  }
  void end(cudaStream_t s) {
    cudaEventRecord(ev[used + 1], s);
    used += 2;
  }
  float ms() const {
    float t = 0;
    for (size_t k = 0; k + 1 < used; k += 2) {
      float v = 0;
      cudaEventElapsedTime(&v, ev[k], ev[k + 1]);
      t += v;
    }
    return t;
  }
  void destroy() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
    used = 0;
    if (dprobe) cudaFree(dprobe);
    dprobe = nullptr;
  }
};

struct OpArgs {
  KernelTimer* ktimer = nullptr;   // non-null in timeline mode
  // one entry per role in OpDesc::roles order; list roles hold several
  std::vector<std::vector<void*>> ptr;
  std::vector<std::vector<uint64_t>> bytes;
  const JVal* attrs = nullptr;
  void* ws = nullptr;            // executor workspace (outside the budget)
  size_t ws_bytes = 0;
  cudaStream_t stream = nullptr;
  void* nccl_comm = nullptr;     // attached communicator (allreduce)
  void* nccl_allreduce = nullptr;
  void* nccl_group_start = nullptr, *nccl_group_end = nullptr;   // one NCCL group per bucket
  oc_allreduce_fn comm_fn = nullptr;   // custom communicator (oc_exec_attach_comm)
  void* comm_user = nullptr;
  uint32_t n_kernels = 0;        // incremented by launch()
  void* p(size_t role, size_t k = 0) const {
    return (role < ptr.size() && k < ptr[role].size()) ? ptr[role][k] : nullptr;
  }
};

struct OpDesc {
  const char* kind;
  std::vector<const char*> roles;
  Status (*launch)(OpArgs& a);
  size_t (*workspace)(const JVal& attrs);  // may be null
};

const OpDesc* find_op(const std::string& kind);
void register_ops(std::vector<const OpDesc*>& out);

inline int64_t A(const OpArgs& a, const char* k, int64_t d = 0) { return a.attrs ? a.attrs->geti(k, d) : d; }
inline double Ad(const OpArgs& a, const char* k, double d = 0) { return a.attrs ? a.attrs->getd(k, d) : d; }
inline bool Ab(const OpArgs& a, const char* k, bool d = false) { return a.attrs ? a.attrs->getb(k, d) : d; }
inline std::string As(const OpArgs& a, const char* k, const char* d = "") { return a.attrs ? a.attrs->gets(k, d) : d; }

#define OC_LAUNCH_CHECK(a)                                   \
  do {                                                       \
    cudaError_t e_ = cudaGetLastError();                     \
    if (e_ != cudaSuccess) return oc::cuda_status(e_, "kernel launch"); \
    (a).n_kernels++;                                         \
  } while (0)

}  // namespace oc
