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


__device__ __forceinline__ int shift_plane(const Geo& g, double zeta) {
    double tg = __dmul_rn(zeta, g.cz);
    int k = (int)floor(tg);
    return min(max(k, 0), g.mzetamax - 1);
}

// Every kernel below works on chunks of kChunk consecutive particles (the
// granularity of the per-chunk mover / hole / filler counts and their scans).
static constexpr int kChunk = 16384;  // == 1 << kShiftChunkLog2 of the fused classification in k_push

// The list/count kernels: one block of kLT threads per chunk; thread t owns
// particles [base + kPer t, base + kPer (t+1)) of its chunk (thread order =
// index order) and reads their class bytes with kPer/16 16-byte loads.  Many
// small blocks per SM keep enough chunks in flight (the work is latency-bound).
static constexpr int kLT = 256;
static constexpr int kPer = kChunk / kLT;  // 64 particles per thread
static_assert(kPer == 64, "four uint4 of class bytes per thread");

// class bytes of [p0, p0 + kPer) as 16 packed words (zero past n)
__device__ __forceinline__ void load_cls(const unsigned char* __restrict__ cls, long long n, long long p0,
                                         unsigned w[kPer / 4]) {
    if (p0 + kPer <= n) {
#pragma unroll
        for (int u = 0; u < kPer / 16; u++) {
            const uint4 v = *reinterpret_cast<const uint4*>(cls + p0 + 16 * u);
            w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < kPer / 4; i++) {
            unsigned x = 0;
            for (int b = 0; b < 4; b++) {
                const long long p = p0 + 4 * i + b;
                if (p < n) x |= (unsigned)cls[p] << (8 * b);
            }
            w[i] = x;
        }
    }
}

// class bytes (0, 1, 2) of a word -> 4 bits (one per byte, bit = predicate):
// the predicate lands in bit 0 of each byte, then one multiply gathers bits
// 0, 8, 16, 24 into bits 21..24 (distinct partial products, no carries)
__device__ __forceinline__ unsigned gather4(unsigned t) { return ((t * 0x00204081u) >> 21) & 0xfu; }
// bits of the class bytes equal to v in {1, 2} (KIND 0), nonzero (KIND 1), zero (KIND 2)
template <int KIND>
__device__ __forceinline__ unsigned long long cls_bits(const unsigned w[kPer / 4], unsigned v = 0) {
    unsigned long long m = 0;
#pragma unroll
    for (int i = 0; i < kPer / 4; i++) {
        const unsigned x = w[i];
        const unsigned t = KIND == 0 ? (v == 1u ? (x & ~(x >> 1)) : ((x >> 1) & ~x)) & 0x01010101u
                         : KIND == 1 ? (x | (x >> 1)) & 0x01010101u
                                     : ~(x | (x >> 1)) & 0x01010101u;
        m |= (unsigned long long)gather4(t) << (4 * i);
    }
    return m;
}
// bits q with lo <= p0 + q < hi
__device__ __forceinline__ unsigned long long range_bits(long long p0, long long lo, long long hi) {
    const long long a = min(max(lo - p0, 0LL), (long long)kPer), b = min(max(hi - p0, 0LL), (long long)kPer);
    if (b <= a) return 0ull;
    const unsigned long long top = b == 64 ? ~0ull : ((1ull << b) - 1ull);
    const unsigned long long bot = a == 64 ? ~0ull : ((1ull << a) - 1ull);
    return top & ~bot;
}

// exclusive scan of one value per thread over the block (index order) and the
// block total; all threads call it
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* sw, unsigned* total) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sw[w] = x;
    __syncthreads();
    if (w == 0) {
        const unsigned t = lane < nw ? sw[lane] : 0u;
        unsigned y = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += u;
        }
        if (lane < nw) sw[lane] = y - t;
        if (lane == 31) sw[32] = y;
    }
    __syncthreads();
    const unsigned off = sw[w] + x - v;
    *total = sw[32];
    __syncthreads();
    return off;
}

// write p0 + (bit positions of m) to out[off..]
__device__ __forceinline__ void emit_bits(unsigned long long m, long long p0, unsigned* __restrict__ out,
                                          unsigned off) {
    while (m) {
        const int q = __ffsll((long long)m) - 1;
        out[off++] = (unsigned)(p0 + q);
        m &= m - 1;
    }
}



// H-2: radial domain of a gyrocentre radius r = sqrt(2 psi) (IEEE sqrt and
// exact comparisons against the ring radii of the window boundaries)
__device__ __forceinline__ int radial_domain(const Geo& g, double psi) {
    // the decision is that of IEEE sqrt(2 psi) >= r_b; away from a boundary
    // (relative margin 1e-12, far above the rounding of 2 psi and r_b^2) it is
    // taken on 2 psi vs r_b^2 without the square root
    const double x = __dmul_rn(2.0, psi);
    int d = 0;
    for (int b = 1; b < g.nrad; b++) {
        const double r2 = g.rbound2[b];
        if (x > r2 * (1.0 + 1e-12)) d++;
        else if (x >= r2 * (1.0 - 1e-12)) d += (sqrt(x) >= g.rbound[b]) ? 1 : 0;
    }
    return d;
}

// classify: cls[p] in {0 keep, 1 left, 2 right}; per-chunk mover counts.
// mode 0: toroidal (periodic ring, the shorter way round); mode 1: radial
// (inner = left, outer = right, not periodic).  One kLT-thread block per
// chunk; each warp walks a contiguous 2048-marker slice in coalesced steps.
template <class R>
__global__ void __launch_bounds__(kLT) k_shift_classify(Geo g, const double* __restrict__ zeta,
                                                        const double* __restrict__ psi, int mode, long long n,
                                                        unsigned char* __restrict__ cls,
                                                        unsigned* __restrict__ cntL,
                                                        unsigned* __restrict__ cntR, long long* far) {
    __shared__ unsigned sw[33];
    const long long base = (long long)blockIdx.x * kChunk;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kWarps = kLT / 32, kSlice = kChunk / kWarps;
    const R* key = reinterpret_cast<const R*>(mode ? psi : zeta);
    unsigned a = 0, b = 0;
    // batches of kB independent loads in flight per warp, then the decisions
    constexpr int kB = 8;
    for (int it0 = 0; it0 < kSlice / 32; it0 += kB) {
        const long long p0 = base + (long long)w * kSlice + it0 * 32 + lane;
        double z[kB];
#pragma unroll
        for (int j = 0; j < kB; j++) z[j] = p0 + 32 * j < n ? (double)__ldcs(key + p0 + 32 * j) : 0.0;
#pragma unroll
        for (int j = 0; j < kB; j++) {
            const long long p = p0 + 32 * j;
            unsigned char c = 0;
            if (p < n) {
                if (mode == 0) {
                    int d = shift_plane(g, z[j]) / g.P;
                    int rel = d - g.rank_t;
                    if (rel < 0) rel += g.ntor;
                    if (rel != 0) c = (rel <= g.ntor / 2) ? 2 : 1;
                    if (rel > 1 && rel < g.ntor - 1) *far = 1;  // beyond a neighbour: multi-hop
                } else {
                    int rel = radial_domain(g, z[j]) - g.rank_r;
                    if (rel != 0) c = (rel > 0) ? 2 : 1;
                    if (rel > 1 || rel < -1) *far = 1;
                }
                cls[p] = c;
            }
            a += __popc(__ballot_sync(0xffffffffu, c == 1));
            b += __popc(__ballot_sync(0xffffffffu, c == 2));
        }
    }
    unsigned ta, tb;
    block_excl_scan(lane == 0 ? a : 0u, sw, &ta);
    block_excl_scan(lane == 0 ? b : 0u, sw, &tb);
    if (threadIdx.x == 0) {
        cntL[blockIdx.x] = ta;
        cntR[blockIdx.x] = tb;
    }
}

// holes: movers at p < n_keep; fillers: keepers at p >= n_keep (per chunk)
__global__ void __launch_bounds__(kLT) k_shift_count_holes(const unsigned char* __restrict__ cls, long long n,
                                                                   const long long* __restrict__ nkeep_p,
                                                                   unsigned* __restrict__ cntH,
                                                                   unsigned* __restrict__ cntF) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long ch = blockIdx.x;
    const long long p0 = ch * kChunk + (long long)threadIdx.x * kPer;
    unsigned w[kPer / 4];
    load_cls(cls, n, p0, w);
    const unsigned h = __popcll(cls_bits<1>(w) & range_bits(p0, 0, min(n, nkeep)));
    const unsigned f = __popcll(cls_bits<2>(w) & range_bits(p0, nkeep, n));
    unsigned th, tf;
    block_excl_scan(h, sw, &th);
    block_excl_scan(f, sw, &tf);
    if (threadIdx.x == 0) {
        cntH[ch] = th;
        cntF[ch] = tf;
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
__global__ void __launch_bounds__(kLT) k_shift_pack(const unsigned char* __restrict__ cls, long long n,
                                                            const unsigned* __restrict__ offL,
                                                            const unsigned* __restrict__ offR,
                                                            unsigned* __restrict__ idxL, unsigned* __restrict__ idxR) {
    __shared__ unsigned sw[33];
    const long long ch = blockIdx.x;
    const long long p0 = ch * kChunk + (long long)threadIdx.x * kPer;
    unsigned w[kPer / 4];
    load_cls(cls, n, p0, w);
    const unsigned long long in = range_bits(p0, 0, n);
    const unsigned long long mL = cls_bits<0>(w, 1u) & in;
    const unsigned long long mR = cls_bits<0>(w, 2u) & in;
    unsigned t;
    const unsigned ol = offL[ch] + block_excl_scan(__popcll(mL), sw, &t);
    const unsigned orr = offR[ch] + block_excl_scan(__popcll(mR), sw, &t);
    emit_bits(mL, p0, idxL, ol);
    emit_bits(mR, p0, idxR, orr);
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
__global__ void __launch_bounds__(kLT) k_shift_list_holes(const unsigned char* __restrict__ cls, long long n,
                                                                  const long long* __restrict__ nkeep_p,
                                                                  const unsigned* __restrict__ offH,
                                                                  unsigned* __restrict__ holes) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long ch = blockIdx.x;
    if (ch * kChunk >= nkeep) return;  // holes lie below n_keep (uniform per block)
    const long long p0 = ch * kChunk + (long long)threadIdx.x * kPer;
    unsigned w[kPer / 4];
    load_cls(cls, n, p0, w);
    const unsigned long long m = cls_bits<1>(w) & range_bits(p0, 0, min(n, nkeep));
    unsigned t;
    const unsigned o = offH[ch] + block_excl_scan(__popcll(m), sw, &t);
    emit_bits(m, p0, holes, o);
}

// list tail-keeper (filler) positions in index order; the k-th filler moves
// into the k-th hole (k_shift_copy with scatter)
__global__ void __launch_bounds__(kLT) k_shift_list_fill(const unsigned char* __restrict__ cls, long long n,
                                                                 const long long* __restrict__ nkeep_p,
                                                                 const unsigned* __restrict__ offF,
                                                                 unsigned* __restrict__ fills) {
    __shared__ unsigned sw[33];
    const long long nkeep = *nkeep_p;
    const long long ch = blockIdx.x;
    if ((ch + 1) * kChunk <= nkeep) return;  // fillers lie at or above n_keep (uniform per block)
    const long long p0 = ch * kChunk + (long long)threadIdx.x * kPer;
    unsigned w[kPer / 4];
    load_cls(cls, n, p0, w);
    const unsigned long long m = cls_bits<2>(w) & range_bits(p0, nkeep, n);
    unsigned t;
    const unsigned o = offF[ch] + block_excl_scan(__popcll(m), sw, &t);
    emit_bits(m, p0, fills, o);
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
                           unsigned char* cls, unsigned* cntL, unsigned* cntR, long long* far, cudaStream_t st) {
    int nb = shift_chunks(n);
    if (g.prec32) k_shift_classify<float><<<nb, kLT, 0, st>>>(g, zeta, psi, mode, n, cls, cntL, cntR, far);
    else k_shift_classify<double><<<nb, kLT, 0, st>>>(g, zeta, psi, mode, n, cls, cntL, cntR, far);
    g_launches++;
}

void launch_shift_nkeep(long long n, const unsigned* totL, const unsigned* totR, long long* nkeep, long long* counts,
                        cudaStream_t st) {
    k_shift_nkeep<<<1, 1, 0, st>>>(n, totL, totR, nkeep, counts);
    g_launches++;
}

void launch_shift_count_holes(const unsigned char* cls, long long n, const long long* nkeep, unsigned* cntH,
                              unsigned* cntF, cudaStream_t st) {
    k_shift_count_holes<<<shift_chunks(n), kLT, 0, st>>>(cls, n, nkeep, cntH, cntF);
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
    unsigned* idxL = idx;
    unsigned* idxR = idx + nL;
    k_shift_pack<<<shift_chunks(n), kLT, 0, st>>>(cls, n, offL, offR, idxL, idxR);
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
    const int nchunk = shift_chunks(n);
    const unsigned* nholes_dev = offH + nchunk;  // scan total = number of holes
    k_shift_list_holes<<<nchunk, kLT, 0, st>>>(cls, n, nkeep, offH, holes);
    k_shift_list_fill<<<nchunk, kLT, 0, st>>>(cls, n, nkeep, offF, fills);
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
