// Probe: pinned host <-> device copy bandwidth into VMM-mapped memory as a
// function of how the VA range is backed (cudaMalloc vs k separate physical
// chunks of m_c; mapping pieces of one allocation at offsets is unsupported).
// Not part of the product; results go to profiles/.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

static int bw(void* dptr, void* hptr, size_t bytes, const char* what) {
  cudaStream_t s; RK(cudaStreamCreate(&s));
  cudaEvent_t a, b; RK(cudaEventCreate(&a)); RK(cudaEventCreate(&b));
  for (int dir = 0; dir < 2; ++dir) {
    for (int w = 0; w < 2; ++w)
      RK(cudaMemcpyAsync(dir ? hptr : dptr, dir ? dptr : hptr, bytes, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, s));
    RK(cudaEventRecord(a, s));
    const int reps = 5;
    for (int r = 0; r < reps; ++r)
      RK(cudaMemcpyAsync(dir ? hptr : dptr, dir ? dptr : hptr, bytes, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, s));
    RK(cudaEventRecord(b, s));
    RK(cudaEventSynchronize(b));
    float ms = 0; RK(cudaEventElapsedTime(&ms, a, b));
    printf("%-40s %s %6.2f GB/s\n", what, dir ? "d2h" : "h2d", bytes * reps / (ms * 1e6));
  }
  cudaStreamDestroy(s);
  return 0;
}

int main() {
  RK(cudaFree(0));
  CUdevice dev; CK(cuCtxGetDevice(&dev));
  const size_t bytes = 256ull << 20;
  void* h; RK(cudaHostAlloc(&h, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  void* d; RK(cudaMalloc(&d, bytes));
  if (bw(d, h, bytes, "cudaMalloc")) return 1;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  CUmemAccessDesc acc = {};
  acc.location = prop.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t mc : {(size_t)2 << 20, (size_t)8 << 20, (size_t)32 << 20}) {
    const size_t k = bytes / mc;
    CUdeviceptr va; CK(cuMemAddressReserve(&va, bytes, 0, 0, 0));
    std::vector<CUmemGenericAllocationHandle> hh(k);
    for (size_t i = 0; i < k; ++i) { CK(cuMemCreate(&hh[i], mc, &prop, 0)); CK(cuMemMap(va + i * mc, mc, 0, hh[i], 0)); }
    CK(cuMemSetAccess(va, bytes, &acc, 1));
    char name[64]; snprintf(name, 64, "VMM %zu separate %zu MiB chunks", k, mc >> 20);
    if (bw((void*)va, h, bytes, name)) return 1;
    CK(cuMemUnmap(va, bytes));
    for (auto x : hh) CK(cuMemRelease(x));
    CK(cuMemAddressFree(va, bytes));
  }
  return 0;
}
