// Semantics and cost of __match_any_sync + __reduce_add_sync with per-group
// (disjoint) member masks: the warp-aggregation step of a deposit variant.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
__global__ void check(int* bad) {
  const unsigned lane = threadIdx.x & 31;
  for (int t = 0; t < 64; t++) {
    unsigned key = hash(lane * 7 + t * 131) % (1 + t % 8);   // 1..8 groups, arbitrary membership
    unsigned m = __match_any_sync(0xffffffffu, key);
    unsigned s = __reduce_add_sync(m, lane + 1);
    unsigned ref = 0;
    for (int l = 0; l < 32; l++) if ((m >> l) & 1) ref += l + 1;
    if (s != ref) atomicAdd(bad, 1);
  }
}
template <int MODE>
__global__ void bench(unsigned* out, int n) {
  const unsigned lane = threadIdx.x & 31;
  unsigned acc = 0;
  for (int i = 0; i < n; i++) {
    unsigned key = (lane + i) >> 3;  // 4 groups of 8
    if (MODE >= 1) {
      unsigned m = __match_any_sync(0xffffffffu, key);
      if (MODE == 2) acc += __reduce_add_sync(m, acc + i);
      else acc += m;
    } else acc += key * 3 + i;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  check<<<148, 256>>>(bad);
  int h = -1; cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
  printf("disjoint-mask reduce mismatches: %d\n", h);
  unsigned* out; cudaMalloc(&out, 64 << 20);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int B = nsm * 8, T = 256, N = 4096;
  auto run = [&](const char* nm, auto k) {
    k<<<B, T>>>(out, N); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<B, T>>>(out, N); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double wi = (double)B * (T / 32) * N;  // warp-iterations
    printf("%-22s %.3f ms  %.2f clk per warp-iteration per SM\n", nm, ms, ms * 1e-3 * clk * 1e3 * nsm / wi);
  };
  run("alu only", bench<0>);
  run("match_any", bench<1>);
  run("match_any + redux", bench<2>);
  return 0;
}
