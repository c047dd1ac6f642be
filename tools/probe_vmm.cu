// Phase-0 box probe (hard part H2): VMM granularity and the
// host-side cost of cuMemCreate / cuMemMap / cuMemSetAccess / cuMemUnmap, and
// whether cuMemSetAccess / cuMemUnmap block the host while a long kernel runs
// on another stream.  Not part of the product; results go to profiles/.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  RK(cudaFree(0));
  CUdevice dev; CK(cuCtxGetDevice(&dev));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gmin = 0, grec = 0;
  CK(cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CK(cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("granularity_min %zu recommended %zu\n", gmin, grec);
  int async_engines = 0; cudaDeviceGetAttribute(&async_engines, cudaDevAttrAsyncEngineCount, 0);
  printf("asyncEngineCount %d\n", async_engines);

  for (size_t mc : {(size_t)2 << 20, (size_t)40 << 20}) {
    const int nchunks = 64;
    std::vector<CUmemGenericAllocationHandle> h(nchunks);
    double t0 = now_us();
    for (int i = 0; i < nchunks; ++i) CK(cuMemCreate(&h[i], mc, &prop, 0));
    double t1 = now_us();
    CUdeviceptr va; CK(cuMemAddressReserve(&va, mc * nchunks, 0, 0, 0));
    double t2 = now_us();
    for (int i = 0; i < nchunks; ++i) CK(cuMemMap(va + i * mc, mc, 0, h[i], 0));
    double t3 = now_us();
    CUmemAccessDesc acc = {};
    acc.location = prop.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int i = 0; i < nchunks; ++i) CK(cuMemSetAccess(va + i * mc, mc, &acc, 1));
    double t4 = now_us();
    for (int i = 0; i < nchunks; ++i) CK(cuMemUnmap(va + i * mc, mc));
    double t5 = now_us();
    // one big map of all chunks then one setaccess
    for (int i = 0; i < nchunks; ++i) CK(cuMemMap(va + i * mc, mc, 0, h[i], 0));
    double t6 = now_us();
    CK(cuMemSetAccess(va, mc * nchunks, &acc, 1));
    double t7 = now_us();
    CK(cuMemUnmap(va, mc * nchunks));
    double t8 = now_us();
    printf("m_c %zu MiB: create %.1f us/chunk, reserve %.1f us, map %.1f us/chunk, setaccess %.1f us/chunk, unmap %.1f us/chunk | "
           "batched: map %.1f us/chunk, setaccess(all) %.1f us, unmap(all) %.1f us\n",
           mc >> 20, (t1 - t0) / nchunks, t2 - t1, (t3 - t2) / nchunks, (t4 - t3) / nchunks, (t5 - t4) / nchunks,
           (t6 - t5) / nchunks, t7 - t6, t8 - t7);

    // Does SetAccess/Unmap stall behind a long kernel on another stream?
    cudaStream_t s; RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    long long cyc = (long long)clk_khz * 200;  // ~200 ms
    spin<<<1, 1, 0, s>>>(cyc);
    double a0 = now_us();
    CK(cuMemMap(va, mc, 0, h[0], 0));
    double a1 = now_us();
    CK(cuMemSetAccess(va, mc, &acc, 1));
    double a2 = now_us();
    CK(cuMemUnmap(va, mc));
    double a3 = now_us();
    RK(cudaStreamSynchronize(s));
    double a4 = now_us();
    printf("  during 200ms kernel: map %.1f us, setaccess %.1f us, unmap %.1f us, remaining kernel %.1f us\n",
           a1 - a0, a2 - a1, a3 - a2, a4 - a3);
    RK(cudaStreamDestroy(s));
    CK(cuMemAddressFree(va, mc * nchunks));
    for (int i = 0; i < nchunks; ++i) CK(cuMemRelease(h[i]));
  }
  return 0;
}
