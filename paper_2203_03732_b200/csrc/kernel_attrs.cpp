// kernel_attrs.cpp — per-device bookkeeping of kernel attributes (internal).
#include <map>
#include <mutex>
#include <utility>

#include <cuda_runtime.h>

#include "kernels.h"

namespace otprg {

cudaError_t smem_attr_raise(const void* fn, size_t bytes) {
  // (also below 48 KB: the default limit covers static + dynamic shared memory,
  // so a kernel with static shared memory needs the opt-in earlier)
  if (bytes == 0) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = set[{dev, fn}];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

}  // namespace otprg
