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

// Every kernel below walks a chunk of kChunk consecutive particles per block:
// warp w owns the kSub = kChunk/32 particles [base + w*kSub, base + (w+1)*kSub)
// in kIt coalesced steps of 32, keeps its per-step ballot masks in registers,
// and a single block-level scan of the 32 warp totals gives every warp its
// output offset (one barrier per chunk).
static constexpr int kChunk = 16 * kShiftBlock;
static constexpr int kSub = kChunk / 32;  // particles per warp
static constexpr int kIt = kSub / 32;     // steps per warp

// exclusive scan of one value per warp over the block; returns this warp's
// offset and the block total (all threads call it)
__device__ __forceinline__ unsigned warp_offsets(unsigned v, unsigned* sw, unsigned* total) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sw[w] = v;
    __syncthreads();
    if (w == 0) {
        unsigned x = sw[lane], y = x;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        sw[lane] = y - x;
        if (lane == 31) sw[32] = y;
    }
    __syncthreads();
    unsigned off = sw[w];
    *total = sw[32];
    __syncthreads();
    return off;
}

__device__ __forceinline__ long long warp_p(long long base, int it) {
    return base + (long long)(threadIdx.x >> 5) * kSub + it * 32 + (threadIdx.x & 31);
}

// H-2: radial domain of a gyrocentre radius r = sqrt(2 psi) (IEEE sqrt and
// exact comparisons against the ring radii of the window boundaries)
__device__ __forceinline__ int radial_domain(const Geo& g, double psi) {
    const double r = sqrt(__dmul_rn(2.0, psi));
    int d = 0;
    for (int b = 1; b < g.nrad; b++) d += (r >= g.rbound[b]) ? 1 : 0;
    return d;
}

// classify: cls[p] in {0 keep, 1 left, 2 right}; per-chunk mover counts.
// mode 0: toroidal (periodic ring, the shorter way round); mode 1: radial
// (inner = left, outer = right, not periodic)
template <class R>
__global__ void __launch_bounds__(kShiftBlock) k_shift_classify(Geo g, const double* __restrict__ zeta,
                                                                const double* __restrict__ psi, int mode, long long n,
                                                                unsigned char* __restrict__ cls,
                                                                unsigned* __restrict__ cntL,
                                                                unsigned* __restrict__ cntR) {
    __shared__ unsigned sw[33];
    const long long base = (long long)blockIdx.x * kChunk;
    const double* key = mode ? psi : zeta;
    double z[kIt];
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        z[it] = (p < n) ? (double)__ldcs(reinterpret_cast<const R*>(key) + p) : 0.0;
    }
    unsigned a = 0, b = 0;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        unsigned char c = 0;
        if (p < n) {
            if (mode == 0) {
                int d = shift_plane(g, z[it]) / g.P;
                int rel = d - g.rank_t;
                if (rel < 0) rel += g.ntor;
                if (rel != 0) c = (rel <= g.ntor / 2) ? 2 : 1;
            } else {
                int rel = radial_domain(g, z[it]) - g.rank_r;
                if (rel != 0) c = (rel > 0) ? 2 : 1;
            }
            cls[p] = c;
        }
        a += __popc(__ballot_sync(0xffffffffu, c == 1));
        b += __popc(__ballot_sync(0xffffffffu, c == 2));
    }
    unsigned ta, tb;
    warp_offsets(a, sw, &ta);
    warp_offsets(b, sw, &tb);
    if (threadIdx.x == 0) {
        cntL[blockIdx.x] = ta;
        cntR[blockIdx.x] = tb;
    }
}

// holes: movers at p < n_keep; fillers: keepers at p >= n_keep (per chunk)
__global__ void __launch_bounds__(kShiftBlock) k_shift_count_holes(const unsigned char* __restrict__ cls, long long n,
                                                                   const long long* __restrict__ nkeep_p,
                                                                   unsigned* __restrict__ cntH,
                                                                   unsigned* __restrict__ cntF) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long base = (long long)blockIdx.x * kChunk;
    unsigned a = 0, b = 0;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        unsigned char c = (p < n) ? cls[p] : 0;
        a += __popc(__ballot_sync(0xffffffffu, (p < n) && (p < nkeep) && c != 0));
        b += __popc(__ballot_sync(0xffffffffu, (p < n) && (p >= nkeep) && c == 0));
    }
    unsigned ta, tb;
    warp_offsets(a, sw, &ta);
    warp_offsets(b, sw, &tb);
    if (threadIdx.x == 0) {
        cntH[blockIdx.x] = ta;
        cntF[blockIdx.x] = tb;
    }
}

struct ShiftAttrs {
    double* a[11];
    int nattr;
    unsigned long long* id;
};

// movers -> index lists (left list, right list), in index order
// (deterministic); the attribute copies run in k_shift_copy with one thread
// per (particle, attribute) so the sparse reads are all in flight at once.
__global__ void __launch_bounds__(kShiftBlock) k_shift_pack(const unsigned char* __restrict__ cls, long long n,
                                                            const unsigned* __restrict__ offL,
                                                            const unsigned* __restrict__ offR,
                                                            unsigned* __restrict__ idxL, unsigned* __restrict__ idxR) {
    __shared__ unsigned sw[33];
    const long long base = (long long)blockIdx.x * kChunk;
    const int lane = threadIdx.x & 31;
    unsigned mL[kIt], mR[kIt];
    unsigned a = 0, b = 0;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        unsigned char c = (p < n) ? cls[p] : 0;
        mL[it] = __ballot_sync(0xffffffffu, c == 1);
        mR[it] = __ballot_sync(0xffffffffu, c == 2);
        a += __popc(mL[it]);
        b += __popc(mR[it]);
    }
    unsigned t;
    unsigned ol = offL[blockIdx.x] + warp_offsets(a, sw, &t);
    unsigned orr = offR[blockIdx.x] + warp_offsets(b, sw, &t);
    if (a + b == 0) return;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        const unsigned p = (unsigned)warp_p(base, it);
        if ((mL[it] >> lane) & 1) idxL[ol + __popc(mL[it] & lt)] = p;
        if ((mR[it] >> lane) & 1) idxR[orr + __popc(mR[it] & lt)] = p;
        ol += __popc(mL[it]);
        orr += __popc(mR[it]);
    }
}

// dst.a[d][q] = src.a[d][idx[q]] (gather; dst contiguous) or, with scatter,
// dst.a[d][didx[q]] = src.a[d][idx[q]]; one thread per (q, d), d = blockIdx.y
template <class R>
__global__ void k_shift_copy(ShiftAttrs src, ShiftAttrs dst, const unsigned* __restrict__ idx,
                             const unsigned* __restrict__ didx, long long m, const unsigned* __restrict__ m_dev) {
    const int d = blockIdx.y;
    if (m_dev) m = min(m, (long long)*m_dev);  // exact count known on the device only
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < m; q += (long long)gridDim.x * blockDim.x) {
        const long long s = idx[q];
        const long long o = didx ? (long long)didx[q] : q;
        if (d < src.nattr) {
            R v = 0;
#pragma unroll
            for (int e = 0; e < 11; e++)
                if (e == d) v = reinterpret_cast<const R*>(src.a[e])[s];
#pragma unroll
            for (int e = 0; e < 11; e++)
                if (e == d) reinterpret_cast<R*>(dst.a[e])[o] = v;
        } else if (src.id) {
            dst.id[o] = src.id[s];
        }
    }
}

// list hole positions in index order
__global__ void __launch_bounds__(kShiftBlock) k_shift_list_holes(const unsigned char* __restrict__ cls, long long n,
                                                                  const long long* __restrict__ nkeep_p,
                                                                  const unsigned* __restrict__ offH,
                                                                  unsigned* __restrict__ holes) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long base = (long long)blockIdx.x * kChunk;
    if (base >= nkeep) return;  // no holes in this chunk (uniform per block)
    const int lane = threadIdx.x & 31;
    unsigned m[kIt];
    unsigned a = 0;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        bool hole = (p < n) && (p < nkeep) && cls[p] != 0;
        m[it] = __ballot_sync(0xffffffffu, hole);
        a += __popc(m[it]);
    }
    unsigned t;
    unsigned oh = offH[blockIdx.x] + warp_offsets(a, sw, &t);
    if (a == 0) return;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        if ((m[it] >> lane) & 1) holes[oh + __popc(m[it] & ((1u << lane) - 1u))] = (unsigned)warp_p(base, it);
        oh += __popc(m[it]);
    }
}

// list tail-keeper (filler) positions in index order; the k-th filler moves
// into the k-th hole (k_shift_copy with scatter)
__global__ void __launch_bounds__(kShiftBlock) k_shift_list_fill(const unsigned char* __restrict__ cls, long long n,
                                                                 const long long* __restrict__ nkeep_p,
                                                                 const unsigned* __restrict__ offF,
                                                                 unsigned* __restrict__ fills) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long base = (long long)blockIdx.x * kChunk;
    if (base + kChunk <= nkeep) return;  // no fillers in this chunk (uniform per block)
    const int lane = threadIdx.x & 31;
    unsigned m[kIt];
    unsigned a = 0;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        long long p = warp_p(base, it);
        bool fill = (p < n) && (p >= nkeep) && cls[p] == 0;
        m[it] = __ballot_sync(0xffffffffu, fill);
        a += __popc(m[it]);
    }
    unsigned t;
    unsigned of = offF[blockIdx.x] + warp_offsets(a, sw, &t);
    if (a == 0) return;
#pragma unroll
    for (int it = 0; it < kIt; it++) {
        if ((m[it] >> lane) & 1) fills[of + __popc(m[it] & ((1u << lane) - 1u))] = (unsigned)warp_p(base, it);
        of += __popc(m[it]);
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

int shift_chunks(long long n) { return (int)std::max<long long>(1, (n + kChunk - 1) / kChunk); }

// ---------------------------------------------------------------------------
void launch_shift_classify(const Geo& g, const double* zeta, const double* psi, int mode, long long n,
                           unsigned char* cls, unsigned* cntL, unsigned* cntR, cudaStream_t st) {
    int nb = shift_chunks(n);
    if (g.prec32) k_shift_classify<float><<<nb, kShiftBlock, 0, st>>>(g, zeta, psi, mode, n, cls, cntL, cntR);
    else k_shift_classify<double><<<nb, kShiftBlock, 0, st>>>(g, zeta, psi, mode, n, cls, cntL, cntR);
    g_launches++;
}

void launch_shift_nkeep(long long n, const unsigned* totL, const unsigned* totR, long long* nkeep, long long* counts,
                        cudaStream_t st) {
    k_shift_nkeep<<<1, 1, 0, st>>>(n, totL, totR, nkeep, counts);
    g_launches++;
}

void launch_shift_count_holes(const unsigned char* cls, long long n, const long long* nkeep, unsigned* cntH,
                              unsigned* cntF, cudaStream_t st) {
    int nb = shift_chunks(n);
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
                       unsigned long long* idL, unsigned long long* idR, unsigned* idx, long long nL, long long nR,
                       cudaStream_t st) {
    int nb = shift_chunks(n);
    unsigned* idxL = idx;
    unsigned* idxR = idx + nL;
    k_shift_pack<<<nb, kShiftBlock, 0, st>>>(cls, n, offL, offR, idxL, idxR);
    g_launches++;
    ShiftAttrs A = mk(attrs, nattr, id);
    for (int side = 0; side < 2; side++) {
        long long m = side ? nR : nL;
        if (m == 0) continue;
        int gx = (int)std::min<long long>((m + 255) / 256, 148LL * 8);
        dim3 grid(gx, nattr + (id ? 1 : 0));
        if (g_prec32)
            k_shift_copy<float><<<grid, 256, 0, st>>>(A, side ? mk(sendR, nattr, idR) : mk(sendL, nattr, idL),
                                                      side ? idxR : idxL, nullptr, m, nullptr);
        else
            k_shift_copy<double><<<grid, 256, 0, st>>>(A, side ? mk(sendR, nattr, idR) : mk(sendL, nattr, idL),
                                                       side ? idxR : idxL, nullptr, m, nullptr);
        g_launches++;
    }
}

void launch_shift_backfill(double* const* attrs, int nattr, unsigned long long* id, const unsigned char* cls,
                           long long n, const long long* nkeep, const unsigned* offH, const unsigned* offF,
                           unsigned* holes, unsigned* fills, long long nholes, cudaStream_t st) {
    int nb = shift_chunks(n);
    const unsigned* nholes_dev = offH + nb;  // scan total = number of holes
    k_shift_list_holes<<<nb, kShiftBlock, 0, st>>>(cls, n, nkeep, offH, holes);
    k_shift_list_fill<<<nb, kShiftBlock, 0, st>>>(cls, n, nkeep, offF, fills);
    g_launches += 2;
    if (nholes > 0) {
        ShiftAttrs A = mk(attrs, nattr, id);
        int gx = (int)std::min<long long>((nholes + 255) / 256, 148LL * 8);
        dim3 grid(gx, nattr + (id ? 1 : 0));
        if (g_prec32) k_shift_copy<float><<<grid, 256, 0, st>>>(A, A, fills, holes, nholes, nholes_dev);
        else k_shift_copy<double><<<grid, 256, 0, st>>>(A, A, fills, holes, nholes, nholes_dev);
        g_launches++;
    }
}

}  // namespace gtcp
