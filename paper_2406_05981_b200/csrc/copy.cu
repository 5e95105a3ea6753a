// copy.cu -- §8(d) e2e transfers: a kernel copy between device and pinned host memory (UVA
// maps page-locked host memory into the device address space, so a load or store from the
// SMs goes over PCIe).  For the kilobytes a batch-1 decode step moves each way, this costs
// one PCIe round trip inside the step's PDL chain instead of a copy-engine memcpy node.
#include "common.cuh"

namespace shiftadd {
namespace {

constexpr int kCopyThreads = 256;

// One 16-B chunk per thread.  SRC_READY: src does not depend on the upstream kernel, so it is
// read before griddepcontrol.wait; dst is always written after it (the upstream kernel may
// still read the old dst).
__global__ void __launch_bounds__(kCopyThreads) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                            size_t n16, int pdl, int src_ready) {
  if (pdl) pdl_launch_dependents();
  const size_t i = (size_t)blockIdx.x * kCopyThreads + threadIdx.x;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (src_ready && i < n16) v = src[i];
  if (pdl) pdl_wait();
  if (!src_ready && i < n16) v = src[i];
  if (i < n16) dst[i] = v;
}

}  // namespace

cudaError_t launch_copy(void* dst, const void* src, size_t bytes, bool pdl, bool src_ready, cudaStream_t stream) {
  const size_t n16 = bytes / 16;
  if (n16 == 0) return cudaSuccess;
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3((unsigned)((n16 + kCopyThreads - 1) / kCopyThreads));
  c.blockDim = dim3(kCopyThreads);
  c.stream = stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  c.attrs = &attr;
  c.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&c, copy_kernel, reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n16,
                            pdl ? 1 : 0, src_ready ? 1 : 0);
}

}  // namespace shiftadd
