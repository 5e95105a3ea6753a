// LUT-build microbenchmark (development tool): cycles per 2-slot build in one CTA of 16 warps.
//   A: fp32 entries, STS.32 (the kernels' build_lut_slot)
//   B: fp16 entries of two slices interleaved in one 32-bit word, STS.32 (half the stores)
//   C: fp32 entries, STS.128 (each lane writes 4 consecutive columns of one key)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lutbuild.bin tools/lutbuild.cu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

template <int MODE>
__global__ void __launch_bounds__(512) k(const __half* x, int iters, long long* out, float* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float xv[2][8];
  for (int t = 0; t < 2; ++t)
    for (int b = 0; b < 8; ++b) xv[t][b] = __half2float(x[t * 256 + 8 * lane + b]);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 1) {
      float L[2][16], H[2];
      for (int t = 0; t < 2; ++t) {
        const float A[4] = {-xv[t][0] - xv[t][1], xv[t][0] - xv[t][1], xv[t][1] - xv[t][0], xv[t][0] + xv[t][1]};
        const float B[4] = {-xv[t][2] - xv[t][3], xv[t][2] - xv[t][3], xv[t][3] - xv[t][2], xv[t][2] + xv[t][3]};
#pragma unroll
        for (int lo = 0; lo < 16; ++lo) L[t][lo] = A[lo & 3] + B[lo >> 2];
        const int hi = warp;
        H[t] = ((hi & 1 ? xv[t][4] : -xv[t][4]) + (hi & 2 ? xv[t][5] : -xv[t][5])) +
               ((hi & 4 ? xv[t][6] : -xv[t][6]) + (hi & 8 ? xv[t][7] : -xv[t][7]));
      }
      if (MODE == 0) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int lo = 0; lo < 16; ++lo)
            sts32(base + t * 128 + 4 * lane + ((warp * 16 + lo) << 8), __float_as_uint(L[t][lo] + H[t] + (float)it));
      } else {
#pragma unroll
        for (int lo = 0; lo < 16; ++lo) {
          const __half2 v = __floats2half2_rn(L[0][lo] + H[0] + (float)it, L[1][lo] + H[1]);
          sts32(base + 4 * lane + ((warp * 16 + lo) << 7), *reinterpret_cast<const uint32_t*>(&v));
        }
      }
    } else {
      // lane: 4 columns c0 = 4*(lane & 7) of slice t = (lane >> 3) & 1, keys: lo block (lane >> 4)
      const int t = (lane >> 3) & 1, c0 = 4 * (lane & 7), kb = lane >> 4;
      float4 acc;
#pragma unroll
      for (int lo = 0; lo < 8; ++lo) {
        const int key = warp * 16 + kb * 8 + lo;
        acc.x = xv[t][0] + (float)key + (float)it;
        acc.y = xv[t][1] + (float)key;
        acc.z = xv[t][2] + (float)key;
        acc.w = xv[t][3] + (float)key;
        sts128(base + t * 128 + 4 * c0 + (key << 8), acc);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (threadIdx.x == 0) sink[blockIdx.x] = *(float*)sm;
}

int main() {
  __half* x; long long* out; float* sink;
  cudaMalloc(&x, 4096); cudaMemset(x, 0, 4096); cudaMalloc(&out, 8 * 148); cudaMalloc(&sink, 4 * 148);
  const char* names[3] = {"A fp32 STS.32", "B fp16x2 STS.32 (half the bytes)", "C fp32 STS.128"};
  for (int m = 0; m < 3; ++m) {
    auto f = m == 0 ? k<0> : m == 1 ? k<1> : k<2>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    f<<<148, 512, 65536>>>(x, 200, out, sink);
    long long h[148];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-36s %lld cycles per 2-slot build (%s)\n", names[m], h[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
