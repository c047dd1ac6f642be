// Pack/unpack copy entries (kernels/pack.cu).
#pragma once
#include <cuda_runtime.h>

#include "cuda_util.hpp"

namespace oc {

struct PackEntry {
  const unsigned char* src;   // device or mapped pinned host address (16-byte aligned)
  unsigned char* dst;
  uint64_t bytes;
};

Status pack_launch(const PackEntry* dev_table, int n, cudaStream_t s);

}  // namespace oc
