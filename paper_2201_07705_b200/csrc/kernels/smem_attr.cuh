// Dynamic shared memory attribute of a kernel with a dynamic shared-memory footprint:
// set ONCE to the most the device allows next to the kernel's static shared memory,
// instead of the size of its latest launch.  A kernel launched twice per step with
// different sizes (e.g. top-k over YOLO and Faster R-CNN rows) then keeps both captured
// graph nodes valid when a tool (ncu) re-launches a node with the function's current
// attribute.  The size a launch actually uses is still its own (occupancy unchanged).
#pragma once
#include <cuda_runtime.h>

namespace gemel {

template <class Kernel>
inline cudaError_t allow_max_dyn_smem(Kernel kernel) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - int(fa.sharedSizeBytes));
}

}  // namespace gemel
