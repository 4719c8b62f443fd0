// gtcp_shift.cu -- toroidal particle shift kernels (H-1..H-3).
//
// One pass of the shift on rank t of ntor toroidal domains:
//   classify : destination domain d = floor(kg / P) (same kg as the charge,
//              bit-exact with the oracle); class 0 keep, 1 left, 2 right (the
//              shorter way round the torus; a multi-hop mover is forwarded
//              again by the next pass).  Per-block mover counts.
//   scan     : exclusive scans of the per-block counts (left, right, holes).
//   pack     : movers -> SoA send segments (warp ballot + block prefix: no
//              global atomics, deterministic order).
//   backfill : holes below n_keep are filled by keepers from [n_keep, n)
//              (k-th hole <- k-th tail keeper), so the owned particles stay
//              contiguous; arrivals are then received straight behind them.
#include "gtcp_internal.cuh"

namespace gtcp {

static constexpr int kShiftBlock = 1024;

__device__ __forceinline__ int shift_plane(const Geo& g, double zeta) {
    double tg = __dmul_rn(zeta, g.cz);
    int k = (int)floor(tg);
    return min(max(k, 0), g.mzetamax - 1);
}

// cls[p] and per-block counts cnt[b] = (left, right, holes_below_nkeep unknown yet -> 0)
__global__ void __launch_bounds__(kShiftBlock) k_shift_classify(Geo g, const double* __restrict__ zeta, long long n,
                                                                unsigned char* __restrict__ cls,
                                                                unsigned* __restrict__ cntL,
                                                                unsigned* __restrict__ cntR) {
    __shared__ unsigned sL[32], sR[32];
    long long p = (long long)blockIdx.x * kShiftBlock + threadIdx.x;
    unsigned char c = 0;
    if (p < n) {
        int d = shift_plane(g, zeta[p]) / g.P;
        int rel = d - g.rank_t;
        if (rel < 0) rel += g.ntor;
        if (rel != 0) c = (rel <= g.ntor / 2) ? 2 : 1;
        cls[p] = c;
    }
    unsigned bl = __ballot_sync(0xffffffffu, c == 1), br = __ballot_sync(0xffffffffu, c == 2);
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sL[w] = __popc(bl); sR[w] = __popc(br); }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned a = 0, b = 0;
        for (int i = 0; i < kShiftBlock / 32; i++) { a += sL[i]; b += sR[i]; }
        cntL[blockIdx.x] = a;
        cntR[blockIdx.x] = b;
    }
}

// holes: movers at p < n_keep; fillers: keepers at p >= n_keep.  Counts per block.
__global__ void __launch_bounds__(kShiftBlock) k_shift_count_holes(const unsigned char* __restrict__ cls, long long n,
                                                                   const long long* __restrict__ nkeep_p,
                                                                   unsigned* __restrict__ cntH,
                                                                   unsigned* __restrict__ cntF) {
    __shared__ unsigned sH[32], sF[32];
    const long long nkeep = *nkeep_p;
    long long p = (long long)blockIdx.x * kShiftBlock + threadIdx.x;
    bool hole = false, fill = false;
    if (p < n) {
        unsigned char c = cls[p];
        hole = (p < nkeep) && c != 0;
        fill = (p >= nkeep) && c == 0;
    }
    unsigned bh = __ballot_sync(0xffffffffu, hole), bf = __ballot_sync(0xffffffffu, fill);
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sH[w] = __popc(bh); sF[w] = __popc(bf); }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned a = 0, b = 0;
        for (int i = 0; i < kShiftBlock / 32; i++) { a += sH[i]; b += sF[i]; }
        cntH[blockIdx.x] = a;
        cntF[blockIdx.x] = b;
    }
}

// block-local exclusive rank of `flag` among the block's threads (warp ballot + smem)
__device__ __forceinline__ unsigned block_rank(bool flag, unsigned* sw) {
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned b = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) sw[w] = __popc(b);
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned v = (threadIdx.x < kShiftBlock / 32) ? sw[threadIdx.x] : 0u;
        unsigned x = v;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (threadIdx.x >= o) x += y;
        }
        sw[threadIdx.x] = x - v;
    }
    __syncthreads();
    unsigned r = sw[w] + __popc(b & ((1u << lane) - 1u));
    __syncthreads();
    return r;
}

struct ShiftAttrs {
    double* a[11];
    int nattr;
    unsigned long long* id;
};

// movers -> send segments (SoA, stride cap)
__global__ void __launch_bounds__(kShiftBlock) k_shift_pack(ShiftAttrs A, const unsigned char* __restrict__ cls, long long n,
                                                            const unsigned* __restrict__ offL,
                                                            const unsigned* __restrict__ offR, ShiftAttrs sendL,
                                                            ShiftAttrs sendR) {
    __shared__ unsigned sw[32];
    long long p = (long long)blockIdx.x * kShiftBlock + threadIdx.x;
    unsigned char c = (p < n) ? cls[p] : 0;
    unsigned rl = block_rank(c == 1, sw);
    unsigned rr = block_rank(c == 2, sw);
    if (c == 1 || c == 2) {
        const ShiftAttrs& S = (c == 1) ? sendL : sendR;
        long long q = (long long)((c == 1) ? offL[blockIdx.x] + rl : offR[blockIdx.x] + rr);
        for (int d = 0; d < A.nattr; d++) S.a[d][q] = A.a[d][p];
        if (A.id) S.id[q] = A.id[p];
    }
}

// list hole positions in index order
__global__ void __launch_bounds__(kShiftBlock) k_shift_list_holes(const unsigned char* __restrict__ cls, long long n,
                                                                  const long long* __restrict__ nkeep_p,
                                                                  const unsigned* __restrict__ offH,
                                                                  unsigned* __restrict__ holes) {
    __shared__ unsigned sw[32];
    const long long nkeep = *nkeep_p;
    long long p = (long long)blockIdx.x * kShiftBlock + threadIdx.x;
    bool hole = (p < n) && (p < nkeep) && cls[p] != 0;
    unsigned r = block_rank(hole, sw);
    if (hole) holes[offH[blockIdx.x] + r] = (unsigned)p;
}

// k-th tail keeper -> k-th hole
__global__ void __launch_bounds__(kShiftBlock) k_shift_fill(ShiftAttrs A, const unsigned char* __restrict__ cls, long long n,
                                                            const long long* __restrict__ nkeep_p,
                                                            const unsigned* __restrict__ offF,
                                                            const unsigned* __restrict__ holes) {
    __shared__ unsigned sw[32];
    const long long nkeep = *nkeep_p;
    long long p = (long long)blockIdx.x * kShiftBlock + threadIdx.x;
    bool fill = (p < n) && (p >= nkeep) && cls[p] == 0;
    unsigned r = block_rank(fill, sw);
    if (fill) {
        long long dst = holes[offF[blockIdx.x] + r];
        for (int d = 0; d < A.nattr; d++) A.a[d][dst] = A.a[d][p];
        if (A.id) A.id[dst] = A.id[p];
    }
}

// n_keep = n - (total left + total right), written on the device
__global__ void k_shift_nkeep(long long n, const unsigned* totL, const unsigned* totR, long long* nkeep,
                              long long* counts_out) {
    long long l = *totL, r = *totR;
    *nkeep = n - l - r;
    counts_out[0] = l;
    counts_out[1] = r;
}

// ---------------------------------------------------------------------------
void launch_shift_classify(const Geo& g, const double* zeta, long long n, unsigned char* cls, unsigned* cntL,
                           unsigned* cntR, cudaStream_t st) {
    int nb = (int)std::max<long long>(1, (n + kShiftBlock - 1) / kShiftBlock);
    k_shift_classify<<<nb, kShiftBlock, 0, st>>>(g, zeta, n, cls, cntL, cntR);
    g_launches++;
}

void launch_shift_nkeep(long long n, const unsigned* totL, const unsigned* totR, long long* nkeep, long long* counts,
                        cudaStream_t st) {
    k_shift_nkeep<<<1, 1, 0, st>>>(n, totL, totR, nkeep, counts);
    g_launches++;
}

void launch_shift_count_holes(const unsigned char* cls, long long n, const long long* nkeep, unsigned* cntH,
                              unsigned* cntF, cudaStream_t st) {
    int nb = (int)std::max<long long>(1, (n + kShiftBlock - 1) / kShiftBlock);
    k_shift_count_holes<<<nb, kShiftBlock, 0, st>>>(cls, n, nkeep, cntH, cntF);
    g_launches++;
}

static ShiftAttrs mk(double* const* a, int nattr, unsigned long long* id) {
    ShiftAttrs s;
    for (int d = 0; d < 11; d++) s.a[d] = d < nattr ? a[d] : nullptr;
    s.nattr = nattr;
    s.id = id;
    return s;
}

void launch_shift_pack(double* const* attrs, int nattr, unsigned long long* id, const unsigned char* cls, long long n,
                       const unsigned* offL, const unsigned* offR, double* const* sendL, double* const* sendR,
                       unsigned long long* idL, unsigned long long* idR, cudaStream_t st) {
    int nb = (int)std::max<long long>(1, (n + kShiftBlock - 1) / kShiftBlock);
    k_shift_pack<<<nb, kShiftBlock, 0, st>>>(mk(attrs, nattr, id), cls, n, offL, offR, mk(sendL, nattr, idL),
                                             mk(sendR, nattr, idR));
    g_launches++;
}

void launch_shift_backfill(double* const* attrs, int nattr, unsigned long long* id, const unsigned char* cls,
                           long long n, const long long* nkeep, const unsigned* offH, const unsigned* offF,
                           unsigned* holes, cudaStream_t st) {
    int nb = (int)std::max<long long>(1, (n + kShiftBlock - 1) / kShiftBlock);
    k_shift_list_holes<<<nb, kShiftBlock, 0, st>>>(cls, n, nkeep, offH, holes);
    k_shift_fill<<<nb, kShiftBlock, 0, st>>>(mk(attrs, nattr, id), cls, n, nkeep, offF, holes);
    g_launches += 2;
}

int shift_block() { return kShiftBlock; }

}  // namespace gtcp
