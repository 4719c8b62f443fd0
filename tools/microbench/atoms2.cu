// ATOMS wavefronts on a large dynamic window (the deposit's layout: lo limbs at
// word 0.., hi limbs at +7681 words): conflict-free / random patterns.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
template <int PAT>
__global__ void k(unsigned* out, int n, int words) {
  extern __shared__ unsigned s[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < n; i++) {
    unsigned a;
    if (PAT == 0) a = (hash(i * 64 + warp) % (words / 32 - 1)) * 32 + lane;     // conflict-free anywhere
    else if (PAT == 1) a = hash(i * 1024 + threadIdx.x) % 7680;               // random in lo region
    else a = hash(i * 1024 + threadIdx.x) % 7680 + 7681;                      // random in hi region
    atomicAdd(&s[a], 1u);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; cudaMalloc(&out, 64 << 20);
  const int words = 15362, smem = words * 4;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<0><<<nsm * 3, 256, smem>>>(out, 1024, words);
  k<1><<<nsm * 3, 256, smem>>>(out, 1024, words);
  k<2><<<nsm * 3, 256, smem>>>(out, 1024, words);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
