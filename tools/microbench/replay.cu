// Replays dumped deposit lane addresses (one ATOMS per recorded instruction)
// to measure the hardware wavefronts of those exact address sets.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void k(const unsigned* __restrict__ addr, int ninstr, int reps, unsigned* out, unsigned off) {
  extern __shared__ unsigned s[];
  for (int i = threadIdx.x; i < 51200; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = gridDim.x * blockDim.x / 32;
  for (int r = 0; r < reps; r++)
    for (int i = warp; i < ninstr; i += nw) atomicAdd(&s[off + (addr[(size_t)i * 32 + lane] & 16383)], 1u);
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  std::vector<unsigned> h;
  unsigned v;
  while (fread(&v, 4, 1, f) == 1) h.push_back(v);
  fclose(f);
  int ninstr = (int)(h.size() / 32);
  unsigned *d, *out;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&out, 1 << 24);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 204800);
  for (unsigned off : {0u, 7681u, 18432u, 25113u, 34816u})
    k<<<148, 256, 204800>>>(d, ninstr, 4, out, off);
  cudaDeviceSynchronize();
  printf("replayed %d instr x 4 reps: %s\n", ninstr, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
