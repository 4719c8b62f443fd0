// L1 data-pipe cost of warp-wide 128-bit global loads vs lane address pattern.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
// PAT 0: all lanes the same 16 B; 1: 4 distinct 16-B chunks in one 128-B line;
// 2: 32 consecutive chunks (4 lines); 3: 8 distinct lines (4 lanes each, same chunk);
// 4: 8 lines, lanes on distinct chunks; 5: 2 lines x 2 chunks
template <int PAT>
__global__ void k(const double2* __restrict__ f, int n, double* out) {
  const unsigned lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0;
  for (int i = 0; i < n; i++) {
    unsigned base = (hash(i * 4096 + warp) & 4095) * 64;  // 64 chunks = 1 KB blocks, L1-resident set (4 MB?)
    base &= (1u << 16) - 1;                               // 1 MB footprint: L2 hits, mostly L1 after warmup
    unsigned c;
    if (PAT == 0) c = 0;
    else if (PAT == 1) c = lane & 3;
    else if (PAT == 2) c = lane;
    else if (PAT == 3) c = (lane >> 2) * 8;
    else if (PAT == 4) c = (lane >> 2) * 8 + (lane & 3);
    else c = (lane & 1) + 8 * ((lane >> 1) & 1);
    double2 v = f[base + c];
    acc += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double2* f; cudaMalloc(&f, 64 << 20); cudaMemset(f, 0, 64 << 20);
  double* out; cudaMalloc(&out, 64 << 20);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  k<0><<<nsm * 4, 256>>>(f, 2048, out); k<1><<<nsm * 4, 256>>>(f, 2048, out); k<2><<<nsm * 4, 256>>>(f, 2048, out);
  k<3><<<nsm * 4, 256>>>(f, 2048, out); k<4><<<nsm * 4, 256>>>(f, 2048, out); k<5><<<nsm * 4, 256>>>(f, 2048, out);
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
