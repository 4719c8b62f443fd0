// Standalone single-GPU harness for the shift kernels (gtcp_shift.cu): times
// classify / pack / count-holes / backfill on synthetic particles with a given
// mover fraction, so they can be profiled with ncu without a multi-rank run.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -I include \
//   -I <nccl include> -o tools/shift_bench tools/shift_bench.cu paper_1510_05546_b200/csrc/gtcp_shift.cu \
//   paper_1510_05546_b200/csrc/gtcp_kernels.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1510_05546_b200/csrc/gtcp_internal.cuh"

using namespace gtcp;

__global__ void init_zeta(double* z, long long n, double frac_move, double dz_dom, unsigned seed) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = (unsigned long long)p + 0x9E3779B97F4A7C15ull * (seed + 1);
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
        // most particles inside domain 0 [0, dz_dom), a fraction just beyond its right edge
        z[p] = (u < frac_move) ? dz_dom * (1.0 + 0.01 * u / frac_move) : dz_dom * u;
    }
}

int main(int argc, char** argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 483000000LL;
    double frac = argc > 2 ? atof(argv[2]) : 0.003;
    int reps = argc > 3 ? atoi(argv[3]) : 3;
    const int mode = argc > 4 ? atoi(argv[4]) : 0;  // 0 toroidal, 1 radial (psi = zeta values here)
    Geo g{};
    g.mzetamax = 64; g.ntor = 2; g.P = 32; g.rank_t = 0;
    g.cz = 64 / GTCP_TWO_PI; g.dzeta = GTCP_TWO_PI / 64;
    // radial mode: two windows split at r = sqrt(2 * 32 dzeta) (so the zeta
    // generator's domain edge is the radial boundary in psi)
    g.nrad = 2; g.rank_r = 0;
    g.rbound[0] = 0.0; g.rbound[1] = sqrt(2.0 * 32 * g.dzeta); g.rbound[2] = 1e30;
    for (int b = 0; b < 9; b++) g.rbound2[b] = g.rbound[b] * g.rbound[b];
    const int nattr = 11;
    double* a[11];
    for (int d = 0; d < nattr; d++) cudaMalloc(&a[d], n * sizeof(double));
    init_zeta<<<148 * 16, 256>>>(a[2], n, frac, 32 * g.dzeta, 7);
    long long cap = (long long)(0.02 * n) + 1024;
    double *sL[11], *sR[11];
    for (int d = 0; d < nattr; d++) { cudaMalloc(&sL[d], cap * 8); cudaMalloc(&sR[d], cap * 8); }
    unsigned char* cls; cudaMalloc(&cls, n);
    int nb = shift_chunks(n);
    unsigned *cnt, *scan_tmp, *holes;
    cudaMalloc(&cnt, 8LL * (nb + 1) * sizeof(unsigned));
    cudaMalloc(&scan_tmp, (nb / 4096 + 2) * sizeof(unsigned));
    cudaMalloc(&holes, cap * sizeof(unsigned));
    unsigned *fills, *midx;
    cudaMalloc(&fills, cap * sizeof(unsigned));
    cudaMalloc(&midx, 2 * cap * sizeof(unsigned));
    long long *nkeep, *counts, *far_flag; cudaMalloc(&nkeep, 8); cudaMalloc(&counts, 64); cudaMalloc(&far_flag, 8);
    unsigned *cL = cnt, *cR = cL + nb + 1, *cH = cR + nb + 1, *cF = cH + nb + 1, *oL = cF + nb + 1, *oR = oL + nb + 1,
             *oH = oR + nb + 1, *oF = oH + nb + 1;
    cudaEvent_t e[8];
    for (auto& x : e) cudaEventCreate(&x);
    for (int r = 0; r < reps; r++) {
        init_zeta<<<148 * 16, 256>>>(a[2], n, frac, 32 * g.dzeta, 7 + r);
        cudaEventRecord(e[0]);
        launch_shift_classify(g, a[2], a[2], mode, n, cls, cL, cR, far_flag, 0);
        launch_scan_u32(cL, oL, nb, scan_tmp, 0);
        launch_scan_u32(cR, oR, nb, scan_tmp, 0);
        launch_shift_nkeep(n, oL + nb, oR + nb, nkeep, counts, 0);
        cudaEventRecord(e[1]);
        long long hc0[2];
        cudaMemcpy(hc0, counts, 16, cudaMemcpyDeviceToHost);
        cudaEventRecord(e[1]);
        launch_shift_pack(a, nattr, nullptr, cls, n, oL, oR, sL, sR, nullptr, nullptr, midx, hc0[0], hc0[1], 0);
        cudaEventRecord(e[2]);
        launch_shift_count_holes(cls, n, nkeep, cH, cF, 0);
        launch_scan_u32(cH, oH, nb, scan_tmp, 0);
        launch_scan_u32(cF, oF, nb, scan_tmp, 0);
        cudaEventRecord(e[3]);
        launch_shift_backfill(a, nattr, nullptr, cls, n, nkeep, oH, oF, holes, fills, hc0[0] + hc0[1], 0);
        cudaEventRecord(e[4]);
        cudaEventSynchronize(e[4]);
        long long hc[2];
        cudaMemcpy(hc, counts, 16, cudaMemcpyDeviceToHost);
        float t[4];
        for (int i = 0; i < 4; i++) cudaEventElapsedTime(&t[i], e[i], e[i + 1]);
        printf("n=%lld movers L=%lld R=%lld  classify+scan %.3f  pack %.3f  holes+scan %.3f  backfill %.3f ms  (%s)\n",
               n, hc[0], hc[1], t[0], t[1], t[2], t[3], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
