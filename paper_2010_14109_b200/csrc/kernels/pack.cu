// SM-driven pack/unpack copy: moves a batch of small
// swapped variables between device memory and their pinned host copies in
// ONE kernel instead of one copy-engine operation each.  Pinned host memory
// is addressable from the device (UVA), so the kernel reads/writes it
// directly over PCIe with 16-byte vectors; many 16-byte requests in flight
// per SM hide the link latency.  Bytes per launch = Σ entry bytes (roofline:
// host link).
#include "../pack.hpp"
#include "common.cuh"

namespace oc {

__global__ void __launch_bounds__(256) pack_copy_kernel(const PackEntry* __restrict__ ents, int n) {
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    const PackEntry E = ents[e];
    const uint64_t n16 = E.bytes >> 4;
    const uint4* __restrict__ s = reinterpret_cast<const uint4*>(E.src);
    uint4* __restrict__ d = reinterpret_cast<uint4*>(E.dst);
    uint64_t i = threadIdx.x;
    // 4 independent 16-byte loads in flight per thread before the stores
    for (; i + 3 * 256 < n16; i += 4 * 256) {
      uint4 a = s[i], b = s[i + 256], c = s[i + 512], f = s[i + 768];
      d[i] = a;
      d[i + 256] = b;
      d[i + 512] = c;
      d[i + 768] = f;
    }
    for (; i < n16; i += 256) d[i] = s[i];
    const uint64_t tail = E.bytes & 15;
    if (threadIdx.x < tail) E.dst[(n16 << 4) + threadIdx.x] = E.src[(n16 << 4) + threadIdx.x];
  }
}

Status pack_launch(const PackEntry* dev_table, int n, cudaStream_t s) {
  if (n <= 0) return Status::ok();
  const int grid = n < 4 * kNumSMs ? n : 4 * kNumSMs;
  pack_copy_kernel<<<grid, 256, 0, s>>>(dev_table, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e, "pack_copy_kernel");
  return Status::ok();
}

}  // namespace oc
