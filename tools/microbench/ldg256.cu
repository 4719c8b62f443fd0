// L1 data-pipe cost of a warp-wide gather of 96-byte field records (the
// push's (node j, node j+1) x 2 planes x 3 components in fp64) with
//   A: 48-byte node records, 6 x LDG.128 per record (the product layout)
//   B: 64-byte padded node records, 4 x LDG.256 per record
//   C: 96-byte duplicated pair records (node j's record holds j and j+1),
//      3 x LDG.256 per record
// Lanes of a warp pick nodes among a few consecutive ones (cell-sorted
// markers).  L1-resident footprint; time per warp-record in SM clocks.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned hash(unsigned x) { x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x; }
__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
template <int MODE, int SPREAD, int CLUSTERS = 1>
__global__ void __launch_bounds__(256, 2) k(const double* __restrict__ f, int n, double* out) {
  const unsigned lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0;
  for (int i = 0; i < n; i++) {
    unsigned h = hash(i * 4096 + warp);
    unsigned node = (h & 255) * 4 + (hash(h + lane) % SPREAD);  // 1K nodes
    if (CLUSTERS > 1) node += 1024 * (hash(h + 77 * lane) % CLUSTERS);  // e.g. two rings
    if (MODE == 0) {
      const double2* q = reinterpret_cast<const double2*>(f + node * 6);
#pragma unroll
      for (int c = 0; c < 6; c++) { double2 v = __ldg(q + c); acc += v.x * v.y; }
    } else if (MODE == 1) {
      const double* q = f + node * 8;
      double a, b, c, d;
      ld256(q, a, b, c, d); acc += a * b + c * d;
      ld256(q + 4, a, b, c, d); acc += a * b;
      ld256(q + 8, a, b, c, d); acc += a * b + c * d;
      ld256(q + 12, a, b, c, d); acc += a * b;
    } else {
      const double* q = f + node * 12;
      double a, b, c, d;
      ld256(q, a, b, c, d); acc += a * b + c * d;
      ld256(q + 4, a, b, c, d); acc += a * b + c * d;
      ld256(q + 8, a, b, c, d); acc += a * b + c * d;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* f; cudaMalloc(&f, 64 << 20); cudaMemset(f, 0, 64 << 20);  // 2 clusters: nodes < 2.1K
  double* out; cudaMalloc(&out, 64 << 20);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int B = nsm * 2, T = 256, N = 4096;
  auto run = [&](const char* nm, auto kern) {
    kern<<<B, T>>>(f, N, out); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); kern<<<B, T>>>(f, N, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double wr = (double)B * (T / 32) * N / nsm;  // warp-records per SM
    printf("%-34s %.3f ms  %.2f clk per warp-record per SM\n", nm, ms, ms * 1e-3 * clk * 1e3 / wr);
  };
  run("A 6xLDG.128 48B nodes, spread 1", k<0, 1>);
  run("B 4xLDG.256 64B nodes, spread 1", k<1, 1>);
  run("C 3xLDG.256 96B pairs, spread 1", k<2, 1>);
  run("A 6xLDG.128 48B nodes, spread 2", k<0, 2>);
  run("B 4xLDG.256 64B nodes, spread 2", k<1, 2>);
  run("C 3xLDG.256 96B pairs, spread 2", k<2, 2>);
  run("A 6xLDG.128 48B nodes, spread 4", k<0, 4>);
  run("B 4xLDG.256 64B nodes, spread 4", k<1, 4>);
  run("C 3xLDG.256 96B pairs, spread 4", k<2, 4>);
  run("A 6xLDG.128 48B nodes, spread 32", k<0, 32>);
  run("A spread 2, 2 clusters (rings)", k<0, 2, 2>);
  run("A spread 4, 2 clusters (rings)", k<0, 4, 2>);
  run("A spread 8", k<0, 8>);
  run("A spread 16", k<0, 16>);
  run("B 4xLDG.256 64B nodes, spread 32", k<1, 32>);
  run("C 3xLDG.256 96B pairs, spread 32", k<2, 32>);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
