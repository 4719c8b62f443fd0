// Shared-memory ATOMS.ADD cost vs lane address pattern (calibrates tools/bank_sim.py).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int W = 8192;  // words of the smem window
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
// pattern: 0 conflict-free, 1 all lanes one word, 2 two lanes per bank (distinct words),
// 3 four lanes per bank (distinct), 4 groups of 4 lanes on one word (8 banks), 5 random,
// 6 groups of 2 lanes on one word, 7 eight lanes per bank (distinct)
template <int PAT>
__global__ void k(unsigned* out, int n) {
  __shared__ unsigned s[W];
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = 0; i < n; i++) {
    unsigned base = (hash(i * 64 + warp) & (W / 64 - 1)) * 32;  // varies per iteration, 32-aligned
    unsigned a;
    if (PAT == 0) a = base + lane;
    else if (PAT == 1) a = base;
    else if (PAT == 2) a = base + (lane & 15) + 32 * (lane >> 4) * 3;
    else if (PAT == 3) a = base + (lane & 7) + 32 * (lane >> 3) * 3;
    else if (PAT == 4) a = base + (lane >> 2);
    else if (PAT == 5) a = hash(i * 1024 + threadIdx.x) & (W - 1);
    else if (PAT == 6) a = base + (lane >> 1);
    else if (PAT == 7) a = base + (lane & 3) + 32 * (lane >> 2) * 3;
    else if (PAT == 8) a = base + (lane & 7) + 32 * (lane < 16 ? 0 : (lane < 24 ? 1 : 2));  // 2 same + 1 + 1 per bank
    else if (PAT == 9) a = base + (lane & 7) + 32 * (lane < 24 ? 0 : 1);                   // 3 same + 1 per bank
    else a = base + (lane & 15) + 32 * (lane < 16 ? 0 : 1) * (lane & 1);                    // mixed
    atomicAdd(&s[a & (W - 1)], 1u);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned* out; cudaMalloc(&out, 64 << 20);
  const int B = nsm * 4, T = 512, N = 4096;
  auto run = [&](const char* name, auto kern) {
    kern<<<B, T>>>(out, N); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); kern<<<B, T>>>(out, N); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = (double)B * (T / 32) * N;
    printf("%-28s %8.3f ms  %6.3f clk per warp-ATOMS per SM\n", name, ms, ms * 1e-3 * clk * 1e3 * nsm / instr);
  };
  run("0 conflict-free", k<0>);
  run("1 all one word", k<1>);
  run("2 two lanes/bank distinct", k<2>);
  run("3 four lanes/bank distinct", k<3>);
  run("7 eight lanes/bank distinct", k<7>);
  run("6 pairs on one word", k<6>);
  run("4 quads on one word", k<4>);
  run("5 random in 8K words", k<5>);
  run("8 per bank 2same+1+1", k<8>);
  run("9 per bank 3same+1", k<9>);
  return 0;
}
