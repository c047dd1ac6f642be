// CUDA runtime/driver helpers.  The driver API (VMM calls) is resolved at
// first use through cudaGetDriverEntryPoint so that liboocore.so loads on a
// machine without libcuda (the CPU build/test box).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "core.hpp"

namespace oc {

struct Driver {
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*TensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  CUresult (*TensorMapEncodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  bool loaded = false;
};

// Loads the entry points once; returns false (with msg) if unavailable.
bool driver(Driver*& d, std::string& msg);

inline Status cuda_status(cudaError_t e, const char* what) {
  Status s = Status::make(OC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  s.cuda = (int)e;
  return s;
}
Status cu_status(CUresult r, const char* what);

#define OC_CUDA(call)                                      \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return oc::cuda_status(e_, #call); \
  } while (0)

#define OC_CU(call)                                        \
  do {                                                     \
    CUresult r_ = (call);                                  \
    if (r_ != CUDA_SUCCESS) return oc::cu_status(r_, #call); \
  } while (0)

#define OC_TRY(expr)                    \
  do {                                  \
    oc::Status s_ = (expr);             \
    if (!s_.good()) return s_;          \
  } while (0)

}  // namespace oc
