// gtcp_kernels.cu -- particle kernels of the B200 GTC-P hot path (sm_100a).
//
//   charge : k_deposit_tiled  -- persistent CTAs over cell-sorted tiles; each
//            tile's deposition footprint (all local planes x a radial band x a
//            label window per ring) lives in shared memory as 64-bit fixed
//            point split into two 32-bit limbs updated with native ATOMS.ADD
//            (24 ops/SM/clk measured, vs 5/SM/clk for the fp64 CAS loop), then
//            flushed once with REDG.ADD.64 into an L2-resident int64 grid.
//            Contributions outside the window go straight to L2.
//            Deterministic: integer sums are order-independent.
//   push   : k_push           -- fused gather (4-point gyro-average of the
//            gradient from the interval-interleaved field) + RK2 stage.
//   bin    : counting sort by cell key (H-4) + permutation + tile build.
//   load   : counter-based Philox marker loader (L-1..L-3 recipe).
//
// Paper passages: charge P:201-209; push P:224-227, P:374-378,
// Eqs. 2-8; bin P:317-318.  Readings: SURVEY §8(c).
#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

#include "gtcp_internal.cuh"

#ifdef GTCP_DEBUG
#include <cassert>
#define DCHECK(c) assert(c)
#else
#define DCHECK(c) ((void)0)
#endif

namespace gtcp {

std::atomic<long long> g_launches{0};
thread_local int g_prec32 = 0;  // precision of the particle store of the context being driven (set per call)

static constexpr double kInvTwoPi = 1.0 / GTCP_TWO_PI;
static constexpr double kInvPi = 2.0 / GTCP_TWO_PI;

// theta is kept in [0, 2 pi) (U-8 wrap), so sin/cos go through the pi-scaled
// forms: exact argument reduction, no large-argument path (about half the
// instructions of sincos(theta)); the one rounding of theta/pi is far below
// the P-0 tolerance.
__device__ __forceinline__ double cos_theta(double theta) { return cospi(theta * kInvPi); }
__device__ __forceinline__ void sincos_theta(double theta, double* s, double* c) { sincospi(theta * kInvPi, s, c); }
static constexpr int kMaxRings = 16;   // radial band of one tile window
static constexpr int kDepositThreads = 256;
// plane stride of a tile window = kPlanePad (mod 32) words: picked with the
// bank-conflict model tools/bank_sim.py (mean 4.1 wavefronts per ATOMS over
// A and B/2, B/4, B/8 windows vs 4.7 for 16 mod 32, whose stride aligns with
// the ~16-column rings of the B/4 windows)
#ifndef GTCP_PLANE_PAD
#define GTCP_PLANE_PAD 4
#endif
static constexpr int kPlanePad = GTCP_PLANE_PAD;

// round-to-nearest-even integer of a*b for |a*b| < 2^51 (1.5*2^52 magic
// constant, one fused rounding).  Explicit intrinsics: every kernel computes
// bit-identical contributions, so tiled and direct deposits agree bitwise.
__device__ __forceinline__ long long fx_round(double a, double b) {
    const double M = 6755399441055744.0;
    double t = __fma_rn(a, b, M);
    return __double_as_longlong(t) - __double_as_longlong(M);
}

// floor of x (|x| < 2^51) with fp64 adds only: x + 1.5*2^52 rounded toward
// -inf is exactly 1.5*2^52 + floor(x), whose low word is the integer; the
// difference is floor(x) as a double.  Bitwise the same as floor() and a
// (double)(int) round trip, without the F2I / I2F / FRND conversions whose
// variable latency stalls the issue on the short scoreboard.  Callers make
// sure x is finite (the deposit skips non-finite markers; the push flags them).
__device__ __forceinline__ double floor_fx(double x, int* i) {
    const double M = 6755399441055744.0;
    const double t = __dadd_rd(x, M);
    *i = __double2loint(t);
    return __dsub_rn(t, M);
}
// (double)i for 0 <= i < 2^31, the same way round: the bits of 1.5*2^52 + i
// minus the constant (exact)
__device__ __forceinline__ double i2d_fx(int i) {
    return __dsub_rn(__hiloint2double(0x43380000, i), 6755399441055744.0);
}

// Q-2 / H-1: global plane interval and its upper weight.  Same operation
// sequence as the oracle (single rounded multiply, floor), bit-exact.
__device__ __forceinline__ int plane_of(const Geo& g, double zeta, double* wz1) {
    double tg = __dmul_rn(zeta, g.cz);
    int k;
    floor_fx(tg, &k);
    k = min(max(k, 0), g.mzetamax - 1);
    *wz1 = __dsub_rn(tg, i2d_fx(k));
    return k;
}

// Q-3..Q-5: the 4 gyro-points x 2 bounding rings of a particle.  For each
// (point, ring) calls fn(m, j, mt, a0, a1) with a0/a1 = 1/4 * wp * wt0/wt1,
// the weights of label nodes j and j+1 (j+1 may equal mt: the duplicate).
template <class Fn>
__device__ __forceinline__ void gyro_point(const Geo& g, double r, double theta, double zeta, double rho,
                                           double inv_r, int l, Fn&& fn);

template <class Fn>
__device__ __forceinline__ void gyro_stencil(const Geo& g, double r, double theta, double zeta, double rho,
                                             double inv_r, Fn&& fn) {
#pragma unroll
    for (int l = 0; l < 4; l++) gyro_point(g, r, theta, zeta, rho, inv_r, l, fn);
}

// one gyro-point l of gyro_stencil (explicit roundings: the same bits in
// every kernel that inlines this)
template <class Fn>
__device__ __forceinline__ void gyro_point(const Geo& g, double r, double theta, double zeta, double rho,
                                           double inv_r, int l, Fn&& fn) {
    const double rho_r = __dmul_rn(rho, inv_r);
    {
        double rl = r, tl = theta;
        if (l == 0) rl = __dadd_rn(r, rho);
        if (l == 2) rl = __dsub_rn(r, rho);
        if (l == 1) tl = __dadd_rn(theta, rho_r);
        if (l == 3) tl = __dsub_rn(theta, rho_r);
        rl = fmin(fmax(rl, g.a0), g.a1);
        double x = __dmul_rn(__dsub_rn(rl, g.a0), g.inv_dr);
        int i;
        floor_fx(x, &i);
        i = min(max(i, 0), g.mpsi - 1);
        double wp1 = __dsub_rn(x, i2d_fx(i));
#pragma unroll
        for (int mm = 0; mm < 2; mm++) {
            int m = i + mm;
            double qt = __ldg(g.qtinv + m);
            int mt = __ldg(g.mtheta + m);
            double s = __dmul_rn(__fma_rn(-zeta, qt, tl), kInvTwoPi);
            int jw;
            s = __dsub_rn(s, floor_fx(s, &jw));
            s = __dmul_rn(s, (double)mt);
            int j;
            floor_fx(s, &j);
            j = (int)min((unsigned)j, (unsigned)(mt - 1));
            double wt1 = __dsub_rn(s, i2d_fx(j));
            double wp = mm ? wp1 : __dsub_rn(1.0, wp1);
            fn(m, j, mt, __dmul_rn(__dmul_rn(0.25, wp), __dsub_rn(1.0, wt1)), __dmul_rn(__dmul_rn(0.25, wp), wt1));
        }
    }
}

// per-particle gyroradius inputs with explicit roundings (shared by all kernels)
__device__ __forceinline__ void gyro_radius(const Geo& g, double psi, double ct, double mu, double* r, double* invB,
                                            double* rho, double* inv_r) {
    // one reciprocal square root per radicand: sqrt(x) = x * rsqrt(x) (within
    // an ulp of sqrt; psi >= a0^2/2 > 0 always, the gyro radicand may be 0)
    const double two_psi = __dmul_rn(2.0, psi);
    *inv_r = rsqrt(two_psi);
    *r = __dmul_rn(two_psi, *inv_r);
    *invB = __fma_rn(__dmul_rn(*r, g.inv_R0), ct, 1.0);
    const double rad = __dmul_rn(__dmul_rn(2.0, mu), *invB);
    *rho = rad > 0.0 ? __dmul_rn(__dmul_rn(rad, rsqrt(rad)), g.inv_omega0) : 0.0;
}

// Global fixed-point grid index of canonical node (kk, m, j), j < mt.  On a
// single toroidal domain the seam plane P is folded into plane 0 with the
// exact label rotation j -> (j + itran_m) mod mt (G-4).
__device__ __forceinline__ long long fx_node(const Geo& g, int kk, int m, int j, int mt) {
    if (g.ntor == 1 && kk == g.P) {
        kk = 0;
        j += __ldg(g.itran + m);
        j -= (j / mt) * mt;
    }
    DCHECK(kk >= 0 && kk <= g.P && m >= 0 && m <= g.mpsi && j >= 0 && j < mt);
    return (long long)kk * g.mgrid + __ldg(g.igrid + m) + j;
}

__device__ __forceinline__ void red_i64(long long* p, long long v) {
    DCHECK(p != nullptr);
    atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// shared-memory 2-limb fixed-point add, no return value needed:
//   v = hi * 2^16 + lo,  lo = v & (2^16 - 1) in [0, 2^16),  hi = v >> 16.
// With |v| < 2^31 and at most 4 * 16384 = 2^16 contributions per node per
// tile (a marker's 4 gyro-points can share a node; tiles hold <= 16384
// markers), sum(lo) < 2^32 and |sum(hi)| < 2^31: both limbs are exact
// (native 32-bit ATOMS.ADD).
static constexpr int kLimbBits = 16;
__device__ __forceinline__ void smem_add(unsigned* lo, int* hi, int slot, long long v) {
    atomicAdd(lo + slot, (unsigned)v & ((1u << kLimbBits) - 1u));
    atomicAdd(hi + slot, (int)(v >> kLimbBits));
}

__device__ __forceinline__ double fx_scale(const DevCounters* dc) { return scalbn(1.0, dc->fx_shift); }

// particle storage of type R (double for precision 64, float for 32): the
// arithmetic is always fp64 (fp32 state, fp64 index/weight math)
template <class R>
__device__ __forceinline__ double ldp(const double* a, long long p) { return (double)reinterpret_cast<const R*>(a)[p]; }
template <class R>
__device__ __forceinline__ double ldp_cs(const double* a, long long p) {
    return (double)__ldcs(reinterpret_cast<const R*>(a) + p);
}
template <class R>
__device__ __forceinline__ void stp(double* a, long long p, double v) { reinterpret_cast<R*>(a)[p] = (R)v; }
template <class R>
__device__ __forceinline__ void stp_cs(double* a, long long p, double v) { __stcs(reinterpret_cast<R*>(a) + p, (R)v); }

// ---------------------------------------------------------------------------
// charge: fixed-point scale.  F = 33 - e with max|w| in [2^(e-1), 2^e), so
// |w| 2^F < 2^33 and every contribution (<= |w|/4) rounds to an integer of
// magnitude below 2^31 (31-bit contributions; precision analysis DESIGN.md §3).
// ---------------------------------------------------------------------------
__global__ void k_fx_scale(DevCounters* dc, int headroom) {
    double wmax = __longlong_as_double((long long)dc->wmax_bits);
    int F = 33;
    if (wmax > 0.0 && isfinite(wmax)) {
        int e;
        frexp(wmax, &e);  // wmax in [2^(e-1), 2^e)
        F = 33 - e - headroom;
    }
    F = max(-60, min(F, 60));
    dc->fx_shift = F;
    dc->fallback = 0;
    dc->tile_next = 0;
}

void launch_fx_scale(DevCounters* dc, cudaStream_t st, int headroom) {
    k_fx_scale<<<1, 1, 0, st>>>(dc, headroom);
    g_launches++;
}

// ---------------------------------------------------------------------------
// charge: direct deposit (every contribution is one REDG.ADD.64 into L2).
// Used for particles outside any tile (arrivals after a shift) and as the
// reference mode 1.
// ---------------------------------------------------------------------------
template <class R>
__global__ void __launch_bounds__(256) k_deposit_direct(Geo g, PSet s, long long begin, long long n,
                                                        long long* __restrict__ fx, DevCounters* dc) {
    const double scale = fx_scale(dc);
    long long clamps = 0;
    for (long long p = begin + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        double psi = ldp<R>(s.x[0], p), theta = ldp<R>(s.x[1], p), zeta = ldp<R>(s.x[2], p), w = ldp<R>(s.x[4], p),
               mu = ldp<R>(s.mu, p);
        if (!isfinite((psi + theta + zeta + mu) * 0.0 + w)) continue;  // flagged by the push; never deposited
        double r, invB, rho, inv_r;
        gyro_radius(g, psi, cos_theta(theta), mu, &r, &invB, &rho, &inv_r);
        double wz1;
        int kg = plane_of(g, zeta, &wz1);
        int k = kg - g.k0;
        if (k < 0 || k > g.P - 1) { clamps++; k = min(max(k, 0), g.P - 1); }
        double ws = __dmul_rn(w, scale);
        double wz[2] = {__dmul_rn(__dsub_rn(1.0, wz1), ws), __dmul_rn(wz1, ws)};
        gyro_stencil(g, r, theta, zeta, rho, inv_r, [&](int m, int j, int mt, double a0, double a1) {
            int j1 = (j + 1 == mt) ? 0 : j + 1;
#pragma unroll
            for (int kk = 0; kk < 2; kk++) {
                long long v0 = fx_round(wz[kk], a0), v1 = fx_round(wz[kk], a1);
                if (v0) red_i64(fx + fx_node(g, k + kk, m, j, mt), v0);
                if (v1) red_i64(fx + fx_node(g, k + kk, m, j1, mt), v1);
            }
        });
    }
    if (clamps) atomicAdd((unsigned long long*)&dc->plane_clamps, (unsigned long long)clamps);
}

void launch_deposit_direct(const Geo& g, const PSet& s, long long begin, long long n, long long* fx,
                           DevCounters* dc, cudaStream_t st) {
    if (n <= begin) return;
    long long work = n - begin;
    int blocks = (int)std::min<long long>((work + 255) / 256, 148LL * 16);
    if (g.prec32) k_deposit_direct<float><<<blocks, 256, 0, st>>>(g, s, begin, n, fx, dc);
    else k_deposit_direct<double><<<blocks, 256, 0, st>>>(g, s, begin, n, fx, dc);
    g_launches++;
}

// ---------------------------------------------------------------------------
// charge: tiled deposit.
// ---------------------------------------------------------------------------
// Tile window (all local planes x rings m_lo..m_hi x a label window per ring):
// ring halo h from the gyroradius cutoff; label half-width on ring m =
// tile half-width + field-line skew over +-dzeta + theta-point margin (rings
// i-1..i+2) + one cell of drift since the bin.
__device__ __forceinline__ int win_halo(const Geo& g, double rho_cut) {
    int h = (int)ceil(rho_cut * g.inv_dr) + 1;
    return min(h, (kMaxRings - 2) / 2);
}

__device__ __forceinline__ double win_halfwidth(const Geo& g, int i, int c0, int c1, int m, double rho_cut,
                                                double* dq_out) {
    int mti = __ldg(g.mtheta + i);
    double half0 = 0.5 * (double)(c1 + 1 - c0) / mti;
    double dq = (__ldg(g.qtinv + i) - __ldg(g.qtinv + m)) * kInvTwoPi;
    double rm = g.a0 + m * g.dr;
    double thm = (m >= i - 1 && m <= i + 2) ? rho_cut / rm * kInvTwoPi : 0.0;
    *dq_out = dq;
    return half0 + g.dzeta * fabs(dq) + thm + g.drift_cells / __ldg(g.mtheta + m);
}

__device__ __forceinline__ int win_width(const Geo& g, int i, int c0, int c1, int m, double rho_cut) {
    double dq;
    double hw = win_halfwidth(g, i, c0, c1, m, rho_cut, &dq);
    int mt = __ldg(g.mtheta + m);
    return min((int)ceil(2.0 * hw * mt) + 2, mt);
}

__device__ __forceinline__ int win_nodes(const Geo& g, int i, int c0, int c1, double rho_cut) {
    int h = win_halo(g, rho_cut);
    int m_lo = max(0, i - h), m_hi = min(g.mpsi, i + 1 + h);
    int S = 0;
    for (int m = m_lo; m <= m_hi; m++) S += win_width(g, i, c0, c1, m, rho_cut) + 1;  // + trash column
    S += (kPlanePad - (S & 31) + 32) & 31;  // the plane-stride padding of k_deposit_tiled
    return S * (g.P + 1);
}

static double deposit_rho_cut(const Geo& g) { return g.rho_cut_th / g.omega0; }

struct WinTables {
    int m_lo, nr, S, total;
    int2 WO[kMaxRings];  // (window width W, column offset) per ring of the band
    int mt[kMaxRings];
    long long start, end;
    int tile;
};

// per-ring constants of the tile band (index nr = the "outside the band" ring:
// W = 0, so every contribution lands in the trash slot and is redone via L2)
struct RingT {  // 16 bytes: one LDS.128 per (gyro-point, ring)
    double qt;
    int mt, W;
};

// limbs of the fixed-point value v = round(a*b) taken straight from the bits of
// t = fma(a, b, 1.5*2^52): the low 16 bits of v are the low 16 bits of t, and
// v >> 16 (|v| < 2^31) is bits 16..47 of t read as a signed int (the 2^51
// offset of the magic constant vanishes mod 2^32).
__device__ __forceinline__ double fx_magic(double a, double b) { return __fma_rn(a, b, 6755399441055744.0); }
__device__ __forceinline__ unsigned fx_lo(double t) { return (unsigned)__double2loint(t) & ((1u << kLimbBits) - 1u); }
__device__ __forceinline__ int fx_hi(double t) {
    return (int)__funnelshift_r((unsigned)__double2loint(t), (unsigned)__double2hiint(t), kLimbBits);
}
__device__ __forceinline__ long long fx_val(double t) {
    return __double_as_longlong(t) - __double_as_longlong(6755399441055744.0);
}

// (j - js) mod mt for j, js in [0, mt): unsigned min of the two candidates
__device__ __forceinline__ unsigned wrap_diff(int j, int js, int mt) {
    const unsigned d = (unsigned)(j - js);
    return min(d, d + (unsigned)mt);
}

// Shared-memory layout of k_deposit_tiled (dynamic): low limbs [kDepCap + 1]
// (index kDepCap = trash slot), high limbs at the fixed distance kDepStride
// (an immediate offset in the ATOMS), interval row table [P x kITStride] of
// int2 = (row of plane k, row of plane k + 1) for plane interval k and ring
// q, column -> ring bytes.  A row packs the label window start (bits 0..12)
// and the word offset of the window row (bits 13..31), so one LDS.64 gives a
// marker both of its planes' rows: the table lookups were ~36 % of the
// L1/shared data-pipe wavefronts that bound this kernel (ncu, r02).
// kITStride = 24 entries (48 banks = 16 mod 32 per interval): the rows of
// intervals k and k+1 for rings q and q+1 never share a bank.
static constexpr int kITStride = 24;
static constexpr int kRowXBits = 13;  // label window start < 8192 (mthetamax < 8192, checked at init)
__device__ __forceinline__ int row_x(int row) { return row & ((1 << kRowXBits) - 1); }
__device__ __forceinline__ int row_y(int row) { return (int)((unsigned)row >> kRowXBits) << 2; }  // byte offset
#ifdef GTCP_DUMP_ADDR
// debug build only: word offsets of the lo-limb ATOMS of the first 8 iterations
// of the 8 warps of 64 tiles spread over the launch ([tile][iter][warp][32][32])
__device__ unsigned g_addr_dump[64 * 8 * 8 * 32 * 32];
extern "C" int gtcp_debug_addr_dump(unsigned* host) {
    return (int)cudaMemcpyFromSymbol(host, g_addr_dump, sizeof(g_addr_dump));
}
#endif

// SURVEY §8(f) #1, fused stage pipeline (an option, gtcp_set_fused): the
// push of one RK2 stage and the deposit of the NEXT stage's charge in one
// persistent kernel over the bin's tiles -- each marker is pushed (same
// push_one as k_push) and its new position deposited straight from registers,
// so the deposit's 40 B/particle re-read of the state and one launch go away.
struct RingTab;
template <int GU = 8, class FT = double, int MODE = 0>
__device__ __forceinline__ void push_one(const Geo& g, const RingTab* __restrict__ rt, double psi, double theta,
                                         double zeta, double rho_par, double w, double mu, const double* base,
                                         double h, const double* __restrict__ gf, double* X, long long& refl,
                                         long long& clamps, double* gio = nullptr);
__device__ __forceinline__ void load_ring_tab(const Geo& g, RingTab* rt);
__device__ __forceinline__ void push_epilogue(DevCounters* dc, double wmax, long long refl, long long clamps,
                                              int nonfinite);
struct FusePush {
    const double* src[5];
    const double* base[5];
    double* out[5];
    const double* gf;
    double h;
    int s1;      // stage 1: the source is the base (read once)
    int rt_off;  // byte offset of the push's ring table in dynamic shared memory
};

#ifndef GTCP_FUSED_NB  // experiment builds: CTAs per SM / gather unroll of the fused push + deposit
#define GTCP_FUSED_NB 2
#endif
#ifndef GTCP_FUSED_GU
#define GTCP_FUSED_GU 8
#endif
template <class R, int NB, bool FUSE = false>
__global__ void __launch_bounds__(kDepositThreads, NB)
    k_deposit_tiled(Geo g, PSet s, long long n, const Tile* __restrict__ tiles, const int* ntiles_p,
                    long long* __restrict__ fx, DevCounters* dc, int cap_nodes, double rho_cut, FusePush fp = {}) {
    constexpr int kDepCap = FUSE ? deposit_cap_nodes(3) : deposit_cap_nodes(NB);  // fused: the NB=3 window
    constexpr int kDepStride = kDepCap + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned* slo = reinterpret_cast<unsigned*>(smem_raw);
    int* shi = reinterpret_cast<int*>(slo + kDepStride);
    int2* itab = reinterpret_cast<int2*>(slo + 2 * kDepStride);  // 8-byte aligned: 2*kDepStride is even
    unsigned char* colq = reinterpret_cast<unsigned char*>(itab + g.P * kITStride);  // [S] ring of column
    __shared__ WinTables T;
    __shared__ __align__(16) RingT RT[kMaxRings + 1];
    __shared__ unsigned long long s_fallback;
    const double scale = fx_scale(dc);
    const int ntiles = *ntiles_p;
    const int P1 = g.P + 1;
    const int lane = threadIdx.x & 31;
    const int b2 = (lane >> 2) & 1, b3 = (lane >> 3) & 1, b4 = (lane >> 4) & 1;
    if (threadIdx.x == 0) s_fallback = 0;
    // fused push: its ring table, and its per-thread counters
    const RingTab* prt = reinterpret_cast<const RingTab*>(smem_raw + fp.rt_off);
    if constexpr (FUSE) load_ring_tab(g, reinterpret_cast<RingTab*>(smem_raw + fp.rt_off));
    double p_wmax = 0.0;
    long long p_refl = 0, p_clamps = 0;
    int p_nonfinite = 0;

    for (;;) {
        if (threadIdx.x == 0) T.tile = atomicAdd(&dc->tile_next, 1);
        __syncthreads();
        const int t = T.tile;
        if (t >= ntiles) break;
        const Tile tl = tiles[t];
        // ---- window of this tile: rings m_lo..m_lo+nr-1, a label window per (plane, ring).
        // One thread per ring computes its width, then every thread forms the
        // (<= 16-term) column prefix itself.
        {
            const int i = tl.ring;
            const int h = win_halo(g, rho_cut);
            const int m_lo = max(0, i - h), m_hi = min(g.mpsi, i + 1 + h);
            const int nr = m_hi - m_lo + 1;
            if (threadIdx.x < nr) {
                const int m = m_lo + threadIdx.x;
                T.WO[threadIdx.x] = make_int2(win_width(g, i, tl.c0, tl.c1, m, rho_cut), 0);
                T.mt[threadIdx.x] = __ldg(g.mtheta + m);
            }
            __syncthreads();
            int S = 0;
            for (int q = 0; q < nr; q++) S += T.WO[q].x + 1;  // column W of each ring: its trash column
            // pad the plane stride to kPlanePad (mod 32) words (4: measured best
            // of the bank-model candidates)
            S += (kPlanePad - (S & 31) + 32) & 31;
            const bool fits = S * P1 <= cap_nodes;  // else: everything via L2
            __syncthreads();
            if (threadIdx.x == 0) {
                T.m_lo = m_lo;
                T.nr = nr;
                T.start = tl.start;
                T.end = min(tl.end, n);
                T.S = fits ? S : 0;
                T.total = fits ? S * P1 : 0;
                int off = 0;
                for (int q = 0; q < nr; q++) {
                    const int W = T.WO[q].x;
                    T.WO[q] = fits ? make_int2(W, off) : make_int2(0, 0);
                    off += W + 1;
                }
            }
            __syncthreads();
        }
        {
            const int i = tl.ring;
            const int mti = __ldg(g.mtheta + i);
            const double fc = 0.5 * (double)(tl.c0 + tl.c1 + 1) / mti;
            const int nr = T.nr, S = T.S;
            // packed row of plane kk, ring q: (label window start, word offset);
            // outside the band or without a window: the trash slot
            auto row_of = [&](int kk, int q) -> int {
                if (q < nr && S > 0) {
                    int m = T.m_lo + q;
                    int mt = T.mt[q];
                    double dq;
                    double hw = win_halfwidth(g, i, tl.c0, tl.c1, m, rho_cut, &dq);
                    double zk = (double)(g.k0 + kk) * g.dzeta;
                    double f = fc + zk * dq - hw;
                    f = f - floor(f);
                    const int x = min(max((int)floor(f * mt), 0), mt - 1);
                    return x | ((kk * S + T.WO[q].y) << kRowXBits);
                }
                return kDepCap << kRowXBits;
            };
            for (int e = threadIdx.x; e < g.P * kITStride; e += blockDim.x) {
                const int k = e / kITStride, q = e - k * kITStride;
                itab[e] = make_int2(row_of(k, q), row_of(k + 1, q));
            }
            if (threadIdx.x <= kMaxRings) {
                const int q = threadIdx.x;
                RingT rt;
                if (q < nr) {
                    const int m = T.m_lo + q;
                    rt.qt = __ldg(g.qtinv + m);
                    rt.mt = T.mt[q];
                    rt.W = T.WO[q].x;
                } else {
                    rt.qt = 0.0;
                    rt.mt = 1;
                    rt.W = 0;
                }
                RT[q] = rt;
            }
            for (int x = threadIdx.x; x < S; x += blockDim.x) colq[x] = 0xFF;  // trash / padding columns
            __syncthreads();
            for (int q = 0; q < nr; q++)
                for (int x = threadIdx.x; x < T.WO[q].x; x += blockDim.x) colq[T.WO[q].y + x] = (unsigned char)q;
            uint4* z4 = reinterpret_cast<uint4*>(slo);
            for (int e = threadIdx.x; e < (T.total + 3) / 4; e += blockDim.x) {
                if (4 * e + 3 < T.total) {
                    z4[e] = make_uint4(0, 0, 0, 0);
                } else {
                    for (int u = 4 * e; u < T.total; u++) slo[u] = 0u;
                }
            }
            for (int e = threadIdx.x; e < T.total; e += blockDim.x) shi[e] = 0;
        }
        __syncthreads();
        // ---- deposit the tile's particles (Q-1..Q-6)
        const int m_lo = T.m_lo, nr = T.nr;
        unsigned long long fb = 0;
        long long clamps = 0;
        // software pipelined: the next particle's five loads are in flight
        // while this one deposits
        const long long pend = T.end;
        long long p = T.start + threadIdx.x;
        double n_psi = 0.0, n_theta = 0.0, n_zeta = 0.0, n_w = 0.0, n_mu = 0.0;
        if (!FUSE && p < pend) {
            n_psi = ldp_cs<R>(s.x[0], p); n_theta = ldp_cs<R>(s.x[1], p); n_zeta = ldp_cs<R>(s.x[2], p);
            n_w = ldp_cs<R>(s.x[4], p); n_mu = ldp_cs<R>(s.mu, p);
        }
        for (; p < pend; p += blockDim.x) {
            double psi, theta, zeta, w, mu;
            if constexpr (FUSE) {
                // push this marker (RK2 stage), store its new state, deposit it
                double base[5], X[5];
#pragma unroll
                for (int d = 0; d < 5; d++) base[d] = ldp_cs<double>(fp.base[d], p);
                mu = ldp_cs<double>(s.mu, p);
                if (fp.s1) {
                    push_one<GTCP_FUSED_GU, double, 0>(g, prt, base[0], base[1], base[2], base[3], base[4], mu, base,
                                                       fp.h, fp.gf, X, p_refl, p_clamps, nullptr);
                } else {
                    push_one<GTCP_FUSED_GU, double, 0>(g, prt, ldp_cs<double>(fp.src[0], p), ldp_cs<double>(fp.src[1], p),
                                           ldp_cs<double>(fp.src[2], p), ldp_cs<double>(fp.src[3], p),
                                           ldp_cs<double>(fp.src[4], p), mu, base, fp.h, fp.gf, X, p_refl, p_clamps,
                                           nullptr);
                }
                if (!isfinite((X[0] + X[1] + X[2] + X[3]) * 0.0 + X[4])) p_nonfinite = 1;
#pragma unroll
                for (int d = 0; d < 5; d++) stp_cs<double>(fp.out[d], p, X[d]);
                p_wmax = fmax(p_wmax, fabs(X[4]));
                psi = X[0];
                theta = X[1];
                zeta = X[2];
                w = X[4];
            } else {
                psi = n_psi; theta = n_theta; zeta = n_zeta; w = n_w; mu = n_mu;
                const long long pn = p + blockDim.x;
                if (pn < pend) {
                    n_psi = ldp_cs<R>(s.x[0], pn); n_theta = ldp_cs<R>(s.x[1], pn); n_zeta = ldp_cs<R>(s.x[2], pn);
                    n_w = ldp_cs<R>(s.x[4], pn); n_mu = ldp_cs<R>(s.mu, pn);
                }
            }
            // a non-finite marker (flagged by the push) is never deposited
            if (!isfinite((psi + theta + zeta + mu) * 0.0 + w)) continue;
            double r, invB, rho, inv_r;
            gyro_radius(g, psi, cos_theta(theta), mu, &r, &invB, &rho, &inv_r);
            double wz1;
            const int kg = plane_of(g, zeta, &wz1);
            int k = kg - g.k0;
            if (k < 0 || k > g.P - 1) { clamps++; k = min(max(k, 0), g.P - 1); }
            const double ws = __dmul_rn(w, scale);
            const double wzl = __dmul_rn(__dsub_rn(1.0, wz1), ws), wzu = __dmul_rn(wz1, ws);
            const double rho_r = __dmul_rn(rho, inv_r);
            // lane-rotated plane order, fixed for the whole particle: pass A uses
            // plane k + b3, pass B plane k + 1 - b3
            const double wzA = b3 ? wzu : wzl, wzB = b3 ? wzl : wzu;
            const int2* itk = itab + k * kITStride;  // rows of planes k, k + 1 (pass A = plane k + b3)
            int bad = -1;  // max over contributions of (window offset - W): >= 0 iff one hit a trash column
#pragma unroll
            for (int lq = 0; lq < 4; lq++) {
                // lane-rotated gyro-point: l = (lq + lane) mod 4.  r +- rho and
                // theta +- rho/r as fma(sign, x, y): one rounding, bit-identical
                // to the add/sub of the direct kernel (sign in {-1, 0, 1})
                const int l = (lq + lane) & 3;
                const double sr = (double)(((l + 1) & 1) * (1 - (l & 2)));
                const double stt = (double)((l & 1) * (1 - (l & 2)));
                double rl = __fma_rn(sr, rho, r);
                const double tl2 = __fma_rn(stt, rho_r, theta);
                rl = fmin(fmax(rl, g.a0), g.a1);
                const double x = __dmul_rn(__dsub_rn(rl, g.a0), g.inv_dr);
                int ir;
                floor_fx(x, &ir);
                ir = min(max(ir, 0), g.mpsi - 1);
                const double wp1 = __dsub_rn(x, i2d_fx(ir));
                // both rings' table entries and window rows are fetched before
                // any use, so the shared-memory latency overlaps the arithmetic
                int qcs[2];
                RingT rts[2];
                int rows[2][2];
#pragma unroll
                for (int mq = 0; mq < 2; mq++) {
                    const int q = ir + (mq ^ b2) - m_lo;
                    qcs[mq] = (unsigned)q < (unsigned)nr ? q : nr;
                    {  // one 16-byte load: (qt lo, qt hi, mt, W)
                        const int4 raw = reinterpret_cast<const int4*>(RT)[qcs[mq]];
                        rts[mq].qt = __hiloint2double(raw.y, raw.x);
                        rts[mq].mt = raw.z;
                        rts[mq].W = raw.w;
                    }
                    const int2 it = itk[qcs[mq]];
                    rows[mq][0] = b3 ? it.y : it.x;
                    rows[mq][1] = b3 ? it.x : it.y;
                }
#pragma unroll
                for (int mq = 0; mq < 2; mq++) {
                    const int mm = mq ^ b2;  // lane-rotated ring choice
                    const RingT rt = rts[mq];
                    double sl = __dmul_rn(__fma_rn(-zeta, rt.qt, tl2), kInvTwoPi);
                    int jw;
                    sl = __dsub_rn(sl, floor_fx(sl, &jw));
                    sl = __dmul_rn(sl, i2d_fx(rt.mt));
                    int j;
                    floor_fx(sl, &j);
                    j = (int)min((unsigned)j, (unsigned)(rt.mt - 1));
                    const double wt1 = __dsub_rn(sl, i2d_fx(j));
                    // wp = mm ? wp1 : 1 - wp1, and the node weights rotated by lane
                    // bit 4, each as one exact fma(+-1, x, {0, 1})
                    const double sm = mm ? 1.0 : -1.0, s4 = b4 ? 1.0 : -1.0;
                    const double wp = __fma_rn(sm, wp1, mm ? 0.0 : 1.0);
                    const double qw = __dmul_rn(0.25, wp);
                    const double aa = __dmul_rn(qw, __fma_rn(s4, wt1, b4 ? 0.0 : 1.0));
                    const double ab = __dmul_rn(qw, __fma_rn(-s4, wt1, b4 ? 1.0 : 0.0));
                    const int j1 = (j + 1 == rt.mt) ? 0 : j + 1;
                    const int ja = b4 ? j1 : j, jb = b4 ? j : j1;
#pragma unroll
                    for (int kq = 0; kq < 2; kq++) {
                        const int row = rows[mq][kq];
                        const int rx = row_x(row), ry = row_y(row);
                        const unsigned da = wrap_diff(ja, rx, rt.mt), db = wrap_diff(jb, rx, rt.mt);
                        bad = max(bad, (int)max(da, db) - rt.W);
                        const int oa = ry + 4 * (int)min(da, (unsigned)rt.W);
                        const int ob = ry + 4 * (int)min(db, (unsigned)rt.W);
                        const double wzk = kq ? wzB : wzA;
                        const double ta = fx_magic(wzk, aa), tb = fx_magic(wzk, ab);
                        unsigned char* base = reinterpret_cast<unsigned char*>(slo);
#ifdef GTCP_DUMP_ADDR  // tools/dump_addr.py: lane word offsets of sampled tiles
                        {
                            const int tstride = max(1, ntiles / 64), ts = t / tstride;
                            if (t % tstride == 0 && ts < 64 && p < T.start + 2048) {
                                const int it = (int)((p - T.start) / blockDim.x), wi = threadIdx.x >> 5;
                                const int ins = ((lq * 2 + mq) * 2 + kq) * 2;
                                if (it < 8) {
                                    unsigned* d = g_addr_dump + (((size_t)(ts * 8 + it) * 8 + wi) * 32 + ins) * 32 + lane;
                                    d[0] = oa >> 2;
                                    d[32] = ob >> 2;
                                }
                            }
                        }
#endif
#ifdef GTCP_DEP_CARRY
                        // one 32-bit word takes the whole contribution v (|v| < 2^31, the
                        // low word of the magic sum); a signed wrap of that word, seen in
                        // the returned old value, moves +-2^32 into the high word.  The
                        // node value hi * 2^32 + lo is the exact sum in any order.
                        {
                            const int va = __double2loint(ta), vb = __double2loint(tb);
                            const int pa = atomicAdd(reinterpret_cast<int*>(base + oa), va);
                            const int pb = atomicAdd(reinterpret_cast<int*>(base + ob), vb);
                            const int na = pa + va, nb = pb + vb;
                            if (((pa ^ na) & (va ^ na)) < 0)
                                atomicAdd(reinterpret_cast<int*>(base + oa + 4 * kDepStride), va < 0 ? -1 : 1);
                            if (((pb ^ nb) & (vb ^ nb)) < 0)
                                atomicAdd(reinterpret_cast<int*>(base + ob + 4 * kDepStride), vb < 0 ? -1 : 1);
                        }
#else
                        atomicAdd(reinterpret_cast<unsigned*>(base + oa), fx_lo(ta));
                        atomicAdd(reinterpret_cast<int*>(base + oa + 4 * kDepStride), fx_hi(ta));
                        atomicAdd(reinterpret_cast<unsigned*>(base + ob), fx_lo(tb));
                        atomicAdd(reinterpret_cast<int*>(base + ob + 4 * kDepStride), fx_hi(tb));
#endif
                    }
                }
            }
            if (__builtin_expect(bad >= 0, 0)) {
                // rare: some contributions fell outside the tile window (trash
                // columns).  Redo exactly those, with the same arithmetic, into L2.
                const int kp0 = k + b3, kp1 = k + 1 - b3;
#pragma unroll 1
                for (int lq = 0; lq < 4; lq++) {
                    const int l = (lq + lane) & 3;
                    const double sr = (double)(((l + 1) & 1) * (1 - (l & 2)));
                    const double stt = (double)((l & 1) * (1 - (l & 2)));
                    double rl = __fma_rn(sr, rho, r);
                    const double tl2 = __fma_rn(stt, rho_r, theta);
                    rl = fmin(fmax(rl, g.a0), g.a1);
                    const double x = __dmul_rn(__dsub_rn(rl, g.a0), g.inv_dr);
                    const int ir = min(max((int)floor(x), 0), g.mpsi - 1);
                    const double wp1 = __dsub_rn(x, (double)ir);
#pragma unroll 1
                    for (int mm = 0; mm < 2; mm++) {
                        const int m = ir + mm, q = m - m_lo;
                        const int qc = (unsigned)q < (unsigned)nr ? q : nr;
                        const RingT rt = RT[qc];
                        const double qt = __ldg(g.qtinv + m);
                        const int mt = __ldg(g.mtheta + m);
                        double sl = __dmul_rn(__fma_rn(-zeta, qt, tl2), kInvTwoPi);
                        sl = __dsub_rn(sl, floor(sl));
                        sl = __dmul_rn(sl, (double)mt);
                        const int j = min((int)floor(sl), mt - 1);
                        const double wt1 = __dsub_rn(sl, (double)j);
                        const double wp = mm ? wp1 : __dsub_rn(1.0, wp1);
                        const double qw = __dmul_rn(0.25, wp);
                        const double a0 = __dmul_rn(qw, __dsub_rn(1.0, wt1)), a1 = __dmul_rn(qw, wt1);
                        const int j1 = (j + 1 == mt) ? 0 : j + 1;
#pragma unroll 1
                        for (int kq = 0; kq < 2; kq++) {
                            const int2 it = itk[qc];
                            const int rx = row_x((kq ^ b3) ? it.y : it.x);
                            const double wzk = kq ? wzB : wzA;
#pragma unroll 1
                            for (int u = 0; u < 2; u++) {
                                const int ju = u ? j1 : j;
                                // same test as the fast path: in the band and inside the window
                                const bool in = qc < nr && wrap_diff(ju, rx, rt.mt) < (unsigned)rt.W;
                                if (in) continue;
                                const long long v = fx_val(fx_magic(wzk, u ? a1 : a0));
                                if (v) { red_i64(fx + fx_node(g, kq ? kp1 : kp0, m, ju, mt), v); fb++; }
                            }
                        }
                    }
                }
            }
        }
        if (fb) atomicAdd(&s_fallback, fb);
        if (clamps) atomicAdd((unsigned long long*)&dc->plane_clamps, (unsigned long long)clamps);
        __syncthreads();
        // ---- flush the window to L2 (one REDG.ADD.64 per nonzero node)
        const int S = T.S;
        if (S > 0) {
            int kk = threadIdx.x / S, x = threadIdx.x - kk * S;
            const int bdiv = blockDim.x / S, bmod = blockDim.x - bdiv * S;
            for (int e = threadIdx.x; e < T.total; e += blockDim.x) {
                const int q = colq[x];
                if (q != 0xFF) {
#ifdef GTCP_DEP_CARRY
                    long long v = (long long)shi[e] * (1LL << 32) + (long long)(int)slo[e];
#else
                    long long v = (long long)shi[e] * (1LL << kLimbBits) + (long long)slo[e];
#endif
                    if (v != 0) {
                        DCHECK(x >= 0 && x < S && kk >= 0 && kk < P1 && q < nr);
                        const int mt = T.mt[q];
                        int j = row_x(kk < g.P ? itab[kk * kITStride + q].x : itab[(g.P - 1) * kITStride + q].y) +
                                (x - T.WO[q].y);
                        if (j >= mt) j -= mt;
                        red_i64(fx + fx_node(g, kk, m_lo + q, j, mt), v);
                    }
                }
                x += bmod;
                kk += bdiv;
                if (x >= S) { x -= S; kk++; }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && s_fallback) atomicAdd((unsigned long long*)&dc->fallback, s_fallback);
    if constexpr (FUSE) push_epilogue(dc, p_wmax, p_refl, p_clamps, p_nonfinite);
}

// ---------------------------------------------------------------------------
// charge ablation: the paper's Fermi/Kepler "update
// binning" deposit.  Every charge, the 4 gyro-points of every
// particle are binned by the cell of the point itself (super-cell = one label
// cell c of ring i in plane interval k), which turns the gyrokinetic deposit
// into a standard one whose footprint spans one cell: then each thread of a
// CTA deposits all the points of one super-cell, consecutive threads take
// adjacent super-cells, and threads of even and odd index accumulate into two
// separate copies of the CTA's partial grid in shared memory (the paper's
// twin copies), flushed to the global grid once.  Same contributions and
// fixed-point arithmetic as the product kernels (bitwise-identical grid).
// ---------------------------------------------------------------------------
// point key = (k * mgrid + igrid_i + c) of gyro-point l of the particle
__device__ __forceinline__ unsigned point_key(const Geo& g, double r, double theta, double zeta, double rho,
                                              double inv_r, int l, int k) {
    const double rho_r = __dmul_rn(rho, inv_r);
    double rl = r, tl = theta;
    if (l == 0) rl = __dadd_rn(r, rho);
    if (l == 2) rl = __dsub_rn(r, rho);
    if (l == 1) tl = __dadd_rn(theta, rho_r);
    if (l == 3) tl = __dsub_rn(theta, rho_r);
    rl = fmin(fmax(rl, g.a0), g.a1);
    const double x = __dmul_rn(__dsub_rn(rl, g.a0), g.inv_dr);
    int i;
    floor_fx(x, &i);
    i = min(max(i, 0), g.mpsi - 1);
    const int mt = __ldg(g.mtheta + i);
    double sl = __dmul_rn(__fma_rn(-zeta, __ldg(g.qtinv + i), tl), kInvTwoPi);
    int jw;
    sl = __dsub_rn(sl, floor_fx(sl, &jw));
    sl = __dmul_rn(sl, (double)mt);
    int c;
    floor_fx(sl, &c);
    c = (int)min((unsigned)c, (unsigned)(mt - 1));
    return (unsigned)(k * g.mgrid + __ldg(g.igrid + i) + c);
}

template <class R>
__global__ void k_point_keys(Geo g, PSet s, long long n, unsigned* __restrict__ pkey, unsigned* __restrict__ prank,
                             unsigned* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    for (long long q0 = (long long)blockIdx.x * blockDim.x; q0 < 4 * n; q0 += (long long)gridDim.x * blockDim.x) {
        const long long q = q0 + threadIdx.x;  // point q = 4 p + l
        const bool act = q < 4 * n;
        unsigned key = 0xffffffffu;
        if (act) {
            const long long p = q >> 2;
            const double psi = ldp<R>(s.x[0], p), theta = ldp<R>(s.x[1], p), zeta = ldp<R>(s.x[2], p),
                         mu = ldp<R>(s.mu, p);
            double r, invB, rho, inv_r;
            gyro_radius(g, psi, cos_theta(theta), mu, &r, &invB, &rho, &inv_r);
            double wz1;
            int k = plane_of(g, zeta, &wz1) - g.k0;
            k = min(max(k, 0), g.P - 1);
            key = point_key(g, r, theta, zeta, rho, inv_r, (int)(q & 3), k);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (act && lane == leader) base = atomicAdd(count + key, (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (act) {
            pkey[q] = key;
            prank[q] = base + __popc(peers & ((1u << lane) - 1u));
        }
    }
}

__global__ void k_point_scatter(const unsigned* __restrict__ pkey, const unsigned* __restrict__ prank,
                                const unsigned* __restrict__ offset, long long npts, unsigned* __restrict__ rec) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < npts; q += (long long)gridDim.x * blockDim.x)
        rec[offset[pkey[q]] + prank[q]] = (unsigned)q;
}

// One CTA per segment of up to blockDim super-cells of one (interval, ring):
// window = planes k, k+1 x rings i, i+1 x label ranges, twin copies.
static constexpr int kPtWin = 1280;  // window nodes per copy (2 planes x 2 rings x labels)
template <class R>
__global__ void __launch_bounds__(256) k_deposit_points(Geo g, PSet s, const unsigned* __restrict__ offset,
                                                      const unsigned* __restrict__ rec, const int4* __restrict__ segs,
                                                      long long* __restrict__ fx, DevCounters* dc) {
    __shared__ unsigned slo[2][kPtWin + 1];
    __shared__ int shi[2][kPtWin + 1];
    __shared__ int s_x[2], s_w[2];  // window start label and width per ring (i, i + 1)
    const double scale = fx_scale(dc);
    // segment = (interval k, ring i, cells c0..c1), a geometry table
    const int4 sg = segs[blockIdx.x];
    const int k = sg.x, i = sg.y, c0 = sg.z, c1 = sg.w;
    const int mti = __ldg(g.mtheta + i);
    // label windows: ring i cells c0..c1+1; ring i+1 the same angular range
    // (ratio mt'/mt, field-line skew over one interval) with a 2-label margin
    if (threadIdx.x < 2) {
        const int m = i + threadIdx.x, mt = __ldg(g.mtheta + m);
        if (threadIdx.x == 0) {
            s_x[0] = c0;
            s_w[0] = min(c1 - c0 + 2, mt);
        } else {
            const double dq = (__ldg(g.qtinv + i) - __ldg(g.qtinv + m)) * kInvTwoPi;
            const double z0 = (double)(g.k0 + k) * g.dzeta;
            double f0 = (double)c0 / mti + z0 * dq - 2.0 / mt - g.dzeta * fabs(dq);
            f0 -= floor(f0);
            s_x[1] = min(max((int)floor(f0 * mt), 0), mt - 1);
            const double span = (double)(c1 + 1 - c0) / mti + 4.0 / mt + 2.0 * g.dzeta * fabs(dq);
            s_w[1] = min((int)ceil(span * mt) + 2, mt);
        }
    }
    for (int e = threadIdx.x; e < 2 * (kPtWin + 1); e += blockDim.x) {
        (&slo[0][0])[e] = 0u;
        (&shi[0][0])[e] = 0;
    }
    __syncthreads();
    const int W0 = s_w[0], W1 = s_w[1];
    const bool fits = 2 * (W0 + W1) <= kPtWin;
    const int cp = threadIdx.x & 1;  // twin copy of this thread (even / odd)
    const int c = c0 + (int)threadIdx.x;
    unsigned long long fb = 0;
    if (c <= c1) {
        const unsigned key = (unsigned)(k * g.mgrid + __ldg(g.igrid + i) + c);
        for (unsigned e = offset[key]; e < offset[key + 1]; e++) {
            const unsigned q = rec[e];
            const long long p = q >> 2;
            const int l = (int)(q & 3);
            const double psi = ldp<R>(s.x[0], p), theta = ldp<R>(s.x[1], p), zeta = ldp<R>(s.x[2], p),
                         w = ldp<R>(s.x[4], p), mu = ldp<R>(s.mu, p);
            if (!isfinite((psi + theta + zeta + mu) * 0.0 + w)) continue;
            double r, invB, rho, inv_r;
            gyro_radius(g, psi, cos_theta(theta), mu, &r, &invB, &rho, &inv_r);
            double wz1;
            int kk = plane_of(g, zeta, &wz1) - g.k0;
            kk = min(max(kk, 0), g.P - 1);
            const double ws = __dmul_rn(w, scale);
            const double wz[2] = {__dmul_rn(__dsub_rn(1.0, wz1), ws), __dmul_rn(wz1, ws)};
            // this point only: the 2 rings x 2 label nodes x 2 planes
            gyro_point(g, r, theta, zeta, rho, inv_r, l, [&](int m, int j, int mt, double a0, double a1) {
                const int rr = m - i;  // 0 or 1 for this point's cell
                const int j1 = (j + 1 == mt) ? 0 : j + 1;
#pragma unroll
                for (int pl = 0; pl < 2; pl++) {
                    const long long v0 = fx_val(fx_magic(wz[pl], a0)), v1 = fx_val(fx_magic(wz[pl], a1));
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const int ju = u ? j1 : j;
                        const long long v = u ? v1 : v0;
                        if (!v) continue;
                        const unsigned d = (rr == 0 || rr == 1) ? wrap_diff(ju, s_x[rr], mt) : 0xffffffffu;
                        const int Wr = rr == 0 ? W0 : W1;
                        if (fits && (unsigned)rr < 2u && d < (unsigned)Wr) {
                            const int slot = pl * (W0 + W1) + (rr ? W0 : 0) + (int)d;
                            atomicAdd(&slo[cp][slot], (unsigned)v & 0xffffu);
                            atomicAdd(&shi[cp][slot], (int)(v >> 16));
                        } else {
                            red_i64(fx + fx_node(g, kk + pl, m, ju, mt), v);
                            fb++;
                        }
                    }
                }
            });
        }
    }
    __syncthreads();
    if (fits)
        for (int e = threadIdx.x; e < 2 * (W0 + W1); e += blockDim.x) {
            const long long v = (long long)shi[0][e] * 65536 + (long long)slo[0][e] + (long long)shi[1][e] * 65536 +
                                (long long)slo[1][e];
            if (!v) continue;
            const int pl = e / (W0 + W1), x = e - pl * (W0 + W1);
            const int rr = x < W0 ? 0 : 1, d = rr ? x - W0 : x;
            const int m = i + rr, mt = __ldg(g.mtheta + m);
            int j = s_x[rr] + d;
            if (j >= mt) j -= mt;
            red_i64(fx + fx_node(g, k + pl, m, j, mt), v);
        }
    if (fb) atomicAdd((unsigned long long*)&dc->fallback, fb);
}

// host: point binning (keys, scan, scatter) + segmented twin-copy deposit
void launch_deposit_points(const Geo& g, const PSet& s, long long n, long long* fx, DevCounters* dc, unsigned* pkey,
                           unsigned* prank, unsigned* rec, unsigned* count, unsigned* offset, unsigned* scan_tmp,
                           const int4* segs, int nseg, cudaStream_t st) {
    if (n <= 0) return;
    const long long nkeys = (long long)g.P * g.mgrid;
    cudaMemsetAsync(count, 0, (nkeys + 1) * sizeof(unsigned), st);
    const int blocks = (int)std::min<long long>((4 * n + 255) / 256, 148LL * 16);
    if (g.prec32) k_point_keys<float><<<blocks, 256, 0, st>>>(g, s, n, pkey, prank, count);
    else k_point_keys<double><<<blocks, 256, 0, st>>>(g, s, n, pkey, prank, count);
    launch_scan_u32(count, offset, nkeys, scan_tmp, st);
    k_point_scatter<<<blocks, 256, 0, st>>>(pkey, prank, offset, 4 * n, rec);
    if (g.prec32) k_deposit_points<float><<<nseg, 256, 0, st>>>(g, s, offset, rec, segs, fx, dc);
    else k_deposit_points<double><<<nseg, 256, 0, st>>>(g, s, offset, rec, segs, fx, dc);
    g_launches += 3;
}

template <int NB>
static cudaError_t configure_nb(size_t smem_bytes) {
    cudaError_t e = cudaFuncSetAttribute(k_deposit_tiled<double, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_bytes);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_deposit_tiled<float, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_bytes);
}

cudaError_t configure_deposit_tiled(size_t smem_bytes, int nb) {
    return nb == 2 ? configure_nb<2>(smem_bytes) : configure_nb<3>(smem_bytes);
}

int deposit_tiled_ctas_per_sm(size_t smem_bytes, int nb) {
    int r = 0;
    cudaError_t e = nb == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_deposit_tiled<double, 2>,
                                                                          kDepositThreads, smem_bytes)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_deposit_tiled<double, 3>,
                                                                          kDepositThreads, smem_bytes);
    return e == cudaSuccess ? r : 0;
}

size_t deposit_tiled_smem(int P, int nb) {
    const int cap = deposit_cap_nodes(nb);
    return (size_t)(2 * (cap + 1)) * 4 + (size_t)P * kITStride * 8 + (size_t)(cap / (P + 1) + 64);
}

void launch_deposit_tiled(const Geo& g, const PSet& s, long long n, const Tile* tiles, int max_tiles,
                          long long* fx, DevCounters* dc, int ctas, size_t smem_bytes, int cap_nodes, int nb,
                          cudaStream_t st) {
    (void)max_tiles;
    double rho_cut = deposit_rho_cut(g);
#define GTCP_DEP(RT, NBV) \
    k_deposit_tiled<RT, NBV><<<ctas, kDepositThreads, smem_bytes, st>>>(g, s, n, tiles, &dc->ntiles, fx, dc, cap_nodes, rho_cut)
    if (g.prec32) {
        if (nb == 2) GTCP_DEP(float, 2); else GTCP_DEP(float, 3);
    } else {
        if (nb == 2) GTCP_DEP(double, 2); else GTCP_DEP(double, 3);
    }
#undef GTCP_DEP
    g_launches++;
}

// fused push + next-stage deposit: 2 CTAs/SM (the push's
// 128 registers), the 3-CTA window capacity, the push's ring table behind the
// deposit's shared memory
size_t push_deposit_smem(const Geo& g, size_t* rt_off) {
    const size_t off = (deposit_tiled_smem(g.P, 3) + 15) & ~(size_t)15;
    if (rt_off) *rt_off = off;
    return off + (size_t)(g.mpsi + 1) * 16;
}

int configure_push_deposit(const Geo& g) {
    const size_t smem = push_deposit_smem(g, nullptr);
    if (cudaFuncSetAttribute(k_deposit_tiled<double, GTCP_FUSED_NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int r = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_deposit_tiled<double, GTCP_FUSED_NB, true>, kDepositThreads, smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return std::min(r, GTCP_FUSED_NB);
}

void launch_push_deposit(const Geo& g, const PSet& s, long long n, const Tile* tiles, long long* fx, DevCounters* dc,
                         int ctas, int cap_nodes, const double* const src[5], const double* const base[5],
                         double* const out[5], const double* gf, double h, cudaStream_t st) {
    FusePush fp;
    for (int d = 0; d < 5; d++) {
        fp.src[d] = src[d];
        fp.base[d] = base[d];
        fp.out[d] = out[d];
    }
    fp.gf = gf;
    fp.h = h;
    fp.s1 = src[0] == base[0];
    size_t off = 0;
    const size_t smem = push_deposit_smem(g, &off);
    fp.rt_off = (int)off;
    k_deposit_tiled<double, GTCP_FUSED_NB, true><<<ctas, kDepositThreads, smem, st>>>(g, s, n, tiles, &dc->ntiles, fx, dc, cap_nodes,
                                                                        deposit_rho_cut(g), fp);
    g_launches++;
}

// fixed point -> fp64 on planes 0..planes-1 (canonical and duplicate nodes)
__global__ void k_fx_to_real(Geo g, const long long* __restrict__ fx, double* __restrict__ rho,
                             const DevCounters* dc, int planes) {
    const double inv = scalbn(1.0, -dc->fx_shift);
    long long total = (long long)planes * g.mgrid;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x)
        rho[e] = (double)fx[e] * inv;
}

void launch_fx_to_real(const Geo& g, const long long* fx, double* rho, const DevCounters* dc, int planes,
                       cudaStream_t st) {
    long long total = (long long)planes * g.mgrid;
    int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
    k_fx_to_real<<<blocks, 256, 0, st>>>(g, fx, rho, dc, planes);
    g_launches++;
}

// ---------------------------------------------------------------------------
// push: fused gather + RK2 stage (U-1..U-8).
//   stage 1: out = src + dt/2 F(src)     (src = live X, out = other buffer)
//   stage 2: out = base + dt F(src)      (src = midpoint, base = out = saved X0)
// gfield layout: interval k, node n -> 6 doubles (plane k: gr gth gpar,
// plane k+1: gr gth gpar); label nodes j, j+1 are 96 contiguous bytes.
// ---------------------------------------------------------------------------
// per-ring geometry in shared memory (one 16-byte record per ring)
struct RingTab {
    double qtinv;
    int mtheta, igrid;
};

__device__ __forceinline__ void load_ring_tab(const Geo& g, RingTab* rt) {
    for (int i = threadIdx.x; i <= g.mpsi; i += blockDim.x) {
        RingTab t;
        t.qtinv = g.qtinv[i];
        t.mtheta = g.mtheta[i];
        t.igrid = g.igrid[i];
        rt[i] = t;
    }
    __syncthreads();
}

struct PushPtrs {
    const double* src[5];
    const double* base[5];
    double* out[5];
    const double* mu;
    // optional fused toroidal shift classification (H-1) of the new state:
    // cls[p] in {0 keep, 1 left, 2 right}, per-16384-particle-chunk mover counts
    unsigned char* cls;
    unsigned* cntL;
    unsigned* cntR;
    long long* far;  // set to 1 if any particle moves beyond a neighbouring domain
};

#ifndef GTCP_PUSH_MINB  // experiment builds: CTAs per SM / gather unroll of the fp64 push
#define GTCP_PUSH_MINB 2
#endif
#ifndef GTCP_PUSH_GU
#define GTCP_PUSH_GU 8
#endif
static constexpr int kShiftChunkLog2 = 14;  // == log2(kChunk) of gtcp_shift.cu

// same expression as the shift's classify (mode 0): destination toroidal domain
// floor(kg / P) of the new zeta, the shorter way round the torus
// far: the destination is beyond the neighbouring domain (a multi-hop mover)
__device__ __forceinline__ unsigned char toroidal_class(const Geo& g, double zeta, bool* far) {
    double wz1;
    const int d = plane_of(g, zeta, &wz1) / g.P;
    int rel = d - g.rank_t;
    if (rel < 0) rel += g.ntor;
    *far = rel > 1 && rel < g.ntor - 1;
    if (rel == 0) return 0;
    return (rel <= g.ntor / 2) ? 2 : 1;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One RK2 stage of one particle (U-1..U-8): returns the new state X[5] from
// the source state (psi, theta, zeta, rho_par, w), mu and the base state.
// Counts reflections / plane clamps into the caller's registers.
// FT: storage type of the gather field (double; float with the fp32 particle
// state of precision 32), arithmetic always fp64.
// MODE 0: fused gather + update (the product).  Loop-fission ablation of the
// paper's Xeon Phi push: MODE 1 only gathers gbar into gio[0..2],
// MODE 2 only updates from gio.
template <int GU, class FT, int MODE>
__device__ __forceinline__ void push_one(const Geo& g, const RingTab* __restrict__ rt, double psi, double theta,
                                         double zeta, double rho_par, double w, double mu, const double* base,
                                         double h, const double* __restrict__ gf, double* X, long long& refl,
                                         long long& clamps, double* gio) {
    // U-1
    double st, ct;
    sincos_theta(theta, &st, &ct);
    double r, invB, rho, inv_r;
    gyro_radius(g, psi, ct, mu, &r, &invB, &rho, &inv_r);
    const double eps = r * g.inv_R0;
    const double q = g.q0 + g.q2 * r * r;
    const double inv_qB = 1.0 / (q * invB);  // one division: 1/q and B follow
    const double B = q * inv_qB;
    const double inv_q = invB * inv_qB;
    // U-2 gather
    double gr, gt, gp;
    if constexpr (MODE == 2) {
        gr = gio[0];
        gt = gio[1];
        gp = gio[2];
    } else {
    double wz1;
    int kg = plane_of(g, zeta, &wz1);
    int k = kg - g.k0;
    if (k < 0 || k > g.P - 1) { clamps++; k = min(max(k, 0), g.P - 1); }
    const double wz0 = 1.0 - wz1;
    // phase 1: the 8 (gyro-point, ring) stencil records (ring tables in smem)
    int node[8];
    double wa[8], wb[8];
    {
        const double rho_r = rho * inv_r;
#pragma unroll
        for (int l = 0; l < 4; l++) {
            double rl = r, tl = theta;
            if (l == 0) rl = r + rho;
            if (l == 2) rl = r - rho;
            if (l == 1) tl = theta + rho_r;
            if (l == 3) tl = theta - rho_r;
            rl = fmin(fmax(rl, g.a0), g.a1);
            const double x = (rl - g.a0) * g.inv_dr;
            int i;
            floor_fx(x, &i);
            i = min(max(i, 0), g.mpsi - 1);
            const double wp1 = x - i2d_fx(i);
#pragma unroll
            for (int mm = 0; mm < 2; mm++) {
                const RingTab t = rt[i + mm];
                double s = (tl - zeta * t.qtinv) * kInvTwoPi;
                int jw;
                s = s - floor_fx(s, &jw);
                s = s * (double)t.mtheta;
                int j;
                floor_fx(s, &j);
                j = (int)min((unsigned)j, (unsigned)(t.mtheta - 1));
                const double wt1 = s - i2d_fx(j);
                const double wp = mm ? wp1 : 1.0 - wp1;
                node[2 * l + mm] = t.igrid + j;
                wa[2 * l + mm] = wp * (1.0 - wt1);
                wb[2 * l + mm] = wp * wt1;
            }
        }
    }
    // phase 2: 8 x 96 contiguous bytes of the interval-interleaved field; each
    // bounding plane accumulated separately, plane weights and 1/4 applied once
    double r0 = 0.0, t0 = 0.0, p0 = 0.0, r1 = 0.0, t1 = 0.0, p1 = 0.0;
    using V2 = typename std::conditional<std::is_same<FT, float>::value, float2, double2>::type;
    const FT* gk = reinterpret_cast<const FT*>(gf) + (long long)k * g.gstride * 6;
#pragma unroll GU
    for (int q = 0; q < 8; q++) {
        const V2* qq = reinterpret_cast<const V2*>(gk + (long long)node[q] * 6);
        const V2 v0 = qq[0], v1 = qq[1], v2 = qq[2];
        const V2 v3 = qq[3], v4 = qq[4], v5 = qq[5];
        const double a0 = wa[q], a1 = wb[q];
        // node j: (v0.x v0.y v1.x) plane k, (v1.y v2.x v2.y) plane k+1; node j+1 likewise in v3..v5
        r0 = fma(a0, v0.x, fma(a1, v3.x, r0));
        t0 = fma(a0, v0.y, fma(a1, v3.y, t0));
        p0 = fma(a0, v1.x, fma(a1, v4.x, p0));
        r1 = fma(a0, v1.y, fma(a1, v4.y, r1));
        t1 = fma(a0, v2.x, fma(a1, v5.x, t1));
        p1 = fma(a0, v2.y, fma(a1, v5.y, p1));
    }
    const double wz0q = 0.25 * wz0, wz1q = 0.25 * wz1;
    gr = wz0q * r0 + wz1q * r1;
    gt = wz0q * t0 + wz1q * t1;
    gp = wz0q * p0 + wz1q * p1;
    if constexpr (MODE == 1) {
        gio[0] = gr;
        gio[1] = gt;
        gio[2] = gp;
        return;
    }
    }
    // U-3 drifts
    const double vpar = g.omega0 * B * rho_par;
    const double iOB = g.inv_omega0 * invB;  // 1 / (omega0 B)
    double vEr = 0.0, vEt = 0.0, vdr = 0.0, vdt = 0.0;
    if (g.drifts) {
        vEr = -gt * inv_r * iOB;
        vEt = gr * iOB;
        const double Cd = (vpar * vpar + mu * B) * g.inv_omega0_R0;
        vdr = -Cd * st;
        vdt = -Cd * ct;
    }
    // U-4
    const double rdot = vEr + vdr;
    const double psidot = r * rdot;
    const double thdot = vpar * B * inv_q * g.inv_R0 + (vEt + vdt) * inv_r;
    const double zdot = vpar * B * g.inv_R0;
    // U-5
    double vdot = -mu * B * B * B * r * st * inv_q * g.inv_R0 * g.inv_R0;
    if (g.paranl) {
        double par = -(B * g.inv_R0) * gp;
        if (g.drifts) par += vpar * g.inv_omega0_R0 * (st * gr + ct * gt * inv_r);
        vdot += par;
    }
    const double dBdr = -B * B * ct * g.inv_R0;
    const double dBdt = B * B * eps * st;
    const double Bdot = rdot * dBdr + thdot * dBdt;
    const double rhodot = (vdot - vpar * Bdot * invB) * iOB;
    // U-6 delta-f weight
    const double Ekin = 0.5 * vpar * vpar + mu * B;
    const double x6 = (r - 0.5) * (1.0 / 0.35);
    const double x2 = x6 * x6;
    const double prof = exp(-(x2 * x2 * x2));
    const double kappa = prof * (g.rln + (Ekin - 1.5) * g.rlt) * g.inv_R0;
    const double wdot = (1.0 - (double)g.paranl * w) *
                        (vEr * kappa - (vpar * (B * g.inv_R0) * gp + vdr * gr + vdt * gt * inv_r));
    // U-7 update
    const double F[5] = {psidot, thdot, zdot, rhodot, wdot};
#pragma unroll
    for (int d = 0; d < 5; d++) X[d] = base[d] + h * F[d];
    // U-8 wrap angles (same operation sequence as the oracle) and reflect r
#pragma unroll
    for (int d = 1; d <= 2; d++) {
        // X in [0, 2 pi): floor(X / 2 pi) = 0 and the oracle's expression returns X itself
        if (X[d] < 0.0 || X[d] >= GTCP_TWO_PI) {
            double t = __dsub_rn(X[d], __dmul_rn(GTCP_TWO_PI, floor(__ddiv_rn(X[d], GTCP_TWO_PI))));
            if (t >= GTCP_TWO_PI) t = 0.0;
            X[d] = t;
        }
    }
    // r = sqrt(2 psi) only when it may leave [a0, a1] (psi bounds padded by a
    // few ulps; the decision itself is taken on r as in the oracle)
    if (!(X[0] > g.psi_lo && X[0] < g.psi_hi)) {
        double rn = sqrt(2.0 * fmax(X[0], 0.0));
        bool rf = false;
        if (rn > g.a1) { rn = 2.0 * g.a1 - rn; rf = true; }
        if (rn < g.a0) { rn = 2.0 * g.a0 - rn; rf = true; }
        if (rf) { X[0] = 0.5 * rn * rn; refl++; }
    }
}

__device__ __forceinline__ void push_epilogue(DevCounters* dc, double wmax, long long refl, long long clamps,
                                              int nonfinite) {
    wmax = warp_max(wmax);
    if ((threadIdx.x & 31) == 0 && wmax > 0.0)
        atomicMax(&dc->wmax_bits, (unsigned long long)__double_as_longlong(wmax));
    if (refl) atomicAdd((unsigned long long*)&dc->reflections, (unsigned long long)refl);
    if (clamps) atomicAdd((unsigned long long*)&dc->plane_clamps, (unsigned long long)clamps);
    if (nonfinite) dc->nonfinite = 1;
}

template <int MINB, bool CS, int GU = 8, class R = double, class FT = R, int MODE = 0, bool S1 = false>
__global__ void __launch_bounds__(256, MINB) k_push(Geo g, PushPtrs pp, long long n, double h,
                                             const double* __restrict__ gf, DevCounters* dc,
                                             double* __restrict__ g3 = nullptr) {
    extern __shared__ RingTab rt_dyn[];
    load_ring_tab(g, rt_dyn);
    double wmax = 0.0;
    long long refl = 0, clamps = 0;
    int nonfinite = 0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        // CS: particle streams evict-first (.cs) so they do not push the field out of L2
        auto ld = [&](const double* a) { return CS ? ldp_cs<R>(a, p) : ldp<R>(a, p); };
        double base[5], X[5];
#pragma unroll
        for (int d = 0; d < 5; d++) base[d] = ld(pp.base[d]);
        if constexpr (MODE == 1) {  // fission, gather loop: gbar to HBM (3 arrays)
            double gio[3];
            push_one<GU, FT, 1>(g, rt_dyn, ld(pp.src[0]), ld(pp.src[1]), ld(pp.src[2]), 0.0, 0.0, ld(pp.mu), base, h,
                                gf, X, refl, clamps, gio);
            __stcs(g3 + p, gio[0]);
            __stcs(g3 + n + p, gio[1]);
            __stcs(g3 + 2 * n + p, gio[2]);
            continue;
        }
        if constexpr (MODE == 2) {  // fission, update loop: gbar from HBM
            double gio[3] = {__ldcs(g3 + p), __ldcs(g3 + n + p), __ldcs(g3 + 2 * n + p)};
            push_one<GU, FT, 2>(g, rt_dyn, ld(pp.src[0]), ld(pp.src[1]), ld(pp.src[2]), ld(pp.src[3]), ld(pp.src[4]),
                                ld(pp.mu), base, h, gf, X, refl, clamps, gio);
        } else {
            // S1 (stage 1: X + dt/2 F(X)): the source is the base, read once
            auto lds = [&](int d) { return S1 ? base[d] : ld(pp.src[d]); };
            push_one<GU, FT>(g, rt_dyn, lds(0), lds(1), lds(2), lds(3), lds(4), ld(pp.mu), base, h, gf, X, refl,
                             clamps);
        }
        // one test: a NaN or Inf in any component survives the product with 0
        if (!isfinite((X[0] + X[1] + X[2] + X[3]) * 0.0 + X[4])) nonfinite = 1;
#pragma unroll
        for (int d = 0; d < 5; d++) {
            if (CS) stp_cs<R>(pp.out[d], p, X[d]);
            else stp<R>(pp.out[d], p, X[d]);
        }
        if (pp.cls) {
            // classify on the value as stored (fp32 state rounds zeta)
            bool far;
            const unsigned char c = toroidal_class(g, (double)(R)X[2], &far);
            pp.cls[p] = c;
            if (far) *pp.far = 1;
            // the 32 lanes of a warp hold consecutive p inside one chunk
            const unsigned act = __activemask();
            const unsigned bl = __ballot_sync(act, c == 1), br = __ballot_sync(act, c == 2);
            if ((threadIdx.x & 31) == __ffs(act) - 1) {
                if (bl) atomicAdd(pp.cntL + (p >> kShiftChunkLog2), (unsigned)__popc(bl));
                if (br) atomicAdd(pp.cntR + (p >> kShiftChunkLog2), (unsigned)__popc(br));
            }
        }
        wmax = fmax(wmax, fabs((double)(R)X[4]));
    }
    push_epilogue(dc, wmax, refl, clamps, nonfinite);
}

void launch_push3(const Geo& g, const double* const src[5], const double* const base[5], double* const out[5],
                  const double* mu, long long n, double h, const double* gfield, DevCounters* dc,
                  cudaStream_t st, unsigned char* cls, unsigned* cntL, unsigned* cntR, double* g3, long long* far) {
    if (n <= 0) return;
    PushPtrs pp;
    for (int d = 0; d < 5; d++) {
        pp.src[d] = src[d];
        pp.base[d] = base[d];
        pp.out[d] = out[d];
    }
    pp.mu = mu;
    pp.cls = cls;
    pp.cntL = cntL;
    pp.cntR = cntR;
    pp.far = far;
    // one particle per thread, 2 CTAs of 256 per SM (128 registers); measured
    // alternatives (3 CTAs, 96-register shapes, TMA- or smem-staged streams and
    // field windows, a texture-path gather) were all slower
    // exactly the resident CTAs (2 per SM), each striding over the particles:
    // no partial last wave (measured 148 x 2 / 4 / 8 / 16 / 32 CTAs at A:
    // 19.58 / 19.58 / 19.97 / 20.47 / 20.75 ms/step)
    static const int pgm = getenv("GTCP_PUSH_GRID") ? atoi(getenv("GTCP_PUSH_GRID")) : 2;  // experiments
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * pgm);
    size_t smr = (g.mpsi + 1) * sizeof(RingTab);
    if (g3 && !g.prec32 && !g.f32field) {
        // loop-fission ablation: gather loop, then update loop
        k_push<2, true, 8, double, double, 1><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc, g3);
        k_push<2, true, 8, double, double, 2><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc, g3);
        g_launches++;
    } else if (src[0] == base[0]) {  // stage 1: the source is the base (read once)
        if (g.prec32) k_push<2, true, 8, float, float, 0, true><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
        else if (g.f32field) k_push<2, true, 8, double, float, 0, true><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
        else k_push<GTCP_PUSH_MINB, true, GTCP_PUSH_GU, double, double, 0, true><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
    } else if (g.prec32) k_push<2, true, 8, float><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
    else if (g.f32field) k_push<2, true, 8, double, float><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
    else k_push<GTCP_PUSH_MINB, true, GTCP_PUSH_GU, double><<<blocks, 256, smr, st>>>(g, pp, n, h, gfield, dc);
    g_launches++;
}

template <class R>
__global__ void k_wmax(const double* __restrict__ w, long long n, DevCounters* dc) {
    double m = 0.0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(ldp<R>(w, p)));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(&dc->wmax_bits, (unsigned long long)__double_as_longlong(m));
}

void launch_wmax(const double* w, long long n, DevCounters* dc, cudaStream_t st) {
    int blocks = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8));
    if (g_prec32) k_wmax<float><<<blocks, 256, 0, st>>>(w, n, dc);
    else k_wmax<double><<<blocks, 256, 0, st>>>(w, n, dc);
    g_launches++;
}

// ---------------------------------------------------------------------------
// bin (H-4): key = (igrid_i + c) * P + k, same operation sequence as the
// oracle so the key is bit-exact; counting sort by key.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned bin_key(const Geo& g, double psi, double theta, double zeta, double mu) {
    double r = sqrt(__dmul_rn(2.0, psi));
    double x = __ddiv_rn(__dsub_rn(r, g.a0), g.dr);
    int i = (int)floor(x);
    i = min(max(i, 0), g.mpsi - 1);
    double s = __ddiv_rn(__dsub_rn(theta, __dmul_rn(zeta, __ldg(g.qtinv + i))), GTCP_TWO_PI);
    s = __dsub_rn(s, floor(s));
    int mt = __ldg(g.mtheta + i);
    s = __dmul_rn(s, (double)mt);
    int c = (int)floor(s);
    c = min(max(c, 0), mt - 1);
    double wz1;
    int k = plane_of(g, zeta, &wz1) - g.k0;
    k = min(max(k, 0), g.P - 1);
    int mb = 0;  // magnetic-moment bin (constant per marker): gyroradius-coherent warps
    for (int b = 0; b < g.nmu - 1; b++) mb += (mu >= g.mu_thr[b]);
    return (unsigned)(((__ldg(g.igrid + i) + c) * g.P + k) * g.nmu + mb);
}

template <class R>
__global__ void k_bin_keys(Geo g, PSet s, long long n, unsigned* __restrict__ key, unsigned* __restrict__ rank,
                           unsigned* __restrict__ count) {
    // cell-sorted input repeats a key ~100 times in a row: aggregate equal keys
    // of a warp into one atomic (leader adds the group size, peers take offsets)
    const int lane = threadIdx.x & 31;
    for (long long p0 = (long long)blockIdx.x * blockDim.x; p0 < n; p0 += (long long)gridDim.x * blockDim.x) {
        const long long p = p0 + threadIdx.x;
        const bool act = p < n;
        unsigned kk = act ? bin_key(g, ldp<R>(s.x[0], p), ldp<R>(s.x[1], p), ldp<R>(s.x[2], p), ldp<R>(s.mu, p)) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, kk);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (act && lane == leader) base = atomicAdd(count + kk, (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (act) {
            key[p] = kk;
            rank[p] = base + __popc(peers & ((1u << lane) - 1u));
        }
    }
}

void launch_bin_keys(const Geo& g, const PSet& s, long long n, unsigned* key, unsigned* rank, unsigned* count,
                     cudaStream_t st) {
    if (n <= 0) return;
    // measured at A (ms per bin) for 148 x {4, 8, 16, 32, 64, 128} CTAs: 2.37 /
    // 2.40 / 1.95 / 1.94 / 1.84 / 1.84
    static const int gm = getenv("GTCP_KEYS_GRID") ? atoi(getenv("GTCP_KEYS_GRID")) : 64;  // experiments
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * gm);
    if (g.prec32) k_bin_keys<float><<<blocks, 256, 0, st>>>(g, s, n, key, rank, count);
    else k_bin_keys<double><<<blocks, 256, 0, st>>>(g, s, n, key, rank, count);
    g_launches++;
}

// exclusive scan of n u32 -> out[0..n] (out[n] = total); 3 kernels
static constexpr int kScanChunk = 4096;

__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* sm, unsigned* total) {
    // blockDim.x == 1024
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned x = v;
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned t = sm[lane];
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        sm[lane] = t;
    }
    __syncthreads();
    unsigned excl = x - v + (wid ? sm[wid - 1] : 0u);
    if (total) *total = sm[31];
    __syncthreads();
    return excl;
}

__global__ void __launch_bounds__(1024) k_scan_reduce(const unsigned* __restrict__ in, long long n,
                                                      unsigned* __restrict__ bsum) {
    __shared__ unsigned sm[32];
    long long base = (long long)blockIdx.x * kScanChunk;
    unsigned v = 0;
    for (int e = threadIdx.x; e < kScanChunk; e += 1024) {
        long long q = base + e;
        if (q < n) v += in[q];
    }
    unsigned tot;
    block_exclusive_scan(v, sm, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_bsum(unsigned* bsum, int nb, unsigned* total_out) {
    __shared__ unsigned sm[32];
    unsigned carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        int b = b0 + threadIdx.x;
        unsigned v = b < nb ? bsum[b] : 0u;
        unsigned tot;
        unsigned ex = block_exclusive_scan(v, sm, &tot);
        if (b < nb) bsum[b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

__global__ void __launch_bounds__(1024) k_scan_final(const unsigned* __restrict__ in, long long n,
                                                     const unsigned* __restrict__ bsum, unsigned* __restrict__ out) {
    __shared__ unsigned sm[32];
    long long base = (long long)blockIdx.x * kScanChunk;
    constexpr int per = kScanChunk / 1024;
    unsigned v[per];
    unsigned s = 0;
    for (int e = 0; e < per; e++) {
        long long q = base + (long long)threadIdx.x * per + e;
        v[e] = q < n ? in[q] : 0u;
        s += v[e];
    }
    unsigned ex = block_exclusive_scan(s, sm, nullptr) + bsum[blockIdx.x];
    for (int e = 0; e < per; e++) {
        long long q = base + (long long)threadIdx.x * per + e;
        if (q < n) out[q] = ex;
        ex += v[e];
    }
}

void launch_scan_u32(const unsigned* in, unsigned* out, long long n, unsigned* block_tmp, cudaStream_t st) {
    int nb = (int)((n + kScanChunk - 1) / kScanChunk);
    k_scan_reduce<<<nb, 1024, 0, st>>>(in, n, block_tmp);
    k_scan_bsum<<<1, 1024, 0, st>>>(block_tmp, nb, out + n);
    k_scan_final<<<nb, 1024, 0, st>>>(in, n, block_tmp, out);
    g_launches += 3;
}

// inverse permutation straight from key and rank: inv[offset[key] + rank] = p
// (the destination of p is never stored)
__global__ void k_bin_inverse(const unsigned* __restrict__ key, const unsigned* __restrict__ rank,
                              const unsigned* __restrict__ offset, long long n, unsigned* __restrict__ inv) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        inv[offset[key[p]] + rank[p]] = (unsigned)p;
}
void launch_bin_inverse(const unsigned* key, const unsigned* rank, const unsigned* offset, long long n,
                        unsigned* inv, cudaStream_t st) {
    if (n <= 0) return;
    // measured at A (ms per bin) for 148 x {1, 2, 3, 4, 6, 8, 16, 64} CTAs:
    // 1.58 / 0.91 / 0.71 / 0.68 / 1.17 / 1.35 / 1.30 / 1.20 (the scattered
    // 4-byte writes of the inverse merge best with 4 resident CTAs per SM)
    static const int gm = getenv("GTCP_INV_GRID") ? atoi(getenv("GTCP_INV_GRID")) : 4;  // experiments
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * gm);
    k_bin_inverse<<<blocks, 256, 0, st>>>(key, rank, offset, n, inv);
    g_launches++;
}

// gather form of the permutation: dst[i] = src[inv[i]] (coalesced writes)
template <class T>
__global__ void k_gather_perm(const T* __restrict__ src, T* __restrict__ dst, const unsigned* __restrict__ inv,
                              long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        dst[i] = __ldg(src + inv[i]);
}

// all attribute arrays in one pass: dst_a[i] = src_a[inv[i]] for every a
struct PermArrays {
    const double* src[12];
    double* dst[12];
    int na;
    const unsigned long long* id_src;
    unsigned long long* id_dst;
};

template <class R>
__global__ void k_gather_perm_multi(PermArrays A, const unsigned* __restrict__ inv, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long s = inv[i];
        R v[12];
#pragma unroll
        for (int a = 0; a < 12; a++)
            if (a < A.na) v[a] = __ldg(reinterpret_cast<const R*>(A.src[a]) + s);
        unsigned long long id = A.id_src ? __ldg(A.id_src + s) : 0ull;
#pragma unroll
        for (int a = 0; a < 12; a++)
            if (a < A.na) __stcs(reinterpret_cast<R*>(A.dst[a]) + i, v[a]);
        if (A.id_src) A.id_dst[i] = id;
    }
}


void launch_gather_perm_multi(const double* const* src, double* const* dst, int na, const unsigned long long* id_src,
                              unsigned long long* id_dst, const unsigned* inv, long long n, cudaStream_t st) {
    if (n <= 0) return;
    PermArrays A;
    for (int a = 0; a < 12; a++) {
        A.src[a] = a < na ? src[a] : nullptr;
        A.dst[a] = a < na ? dst[a] : nullptr;
    }
    A.na = na;
    A.id_src = id_src;
    A.id_dst = id_dst;
    // measured (ms per bin) for 148 x {2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 24} CTAs:
    // class A 10.5 / 7.6 / 6.2 / 5.4 / 4.9 / 7.1 / 6.4 / 5.5 / 5.4 / 5.4 / 5.3;
    // the class-B grid at 241 M markers: x6 5.7, x16 6.2
    static const int gm = getenv("GTCP_PERM_GRID") ? atoi(getenv("GTCP_PERM_GRID")) : 6;  // experiments
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * gm);
    if (g_prec32) k_gather_perm_multi<float><<<blocks, 256, 0, st>>>(A, inv, n);
    else k_gather_perm_multi<double><<<blocks, 256, 0, st>>>(A, inv, n);
    g_launches++;
}

void launch_gather_perm_f64(const double* src, double* dst, const unsigned* inv, long long n, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (g_prec32)
        k_gather_perm<float><<<blocks, 256, 0, st>>>(reinterpret_cast<const float*>(src), reinterpret_cast<float*>(dst),
                                                     inv, n);
    else k_gather_perm<double><<<blocks, 256, 0, st>>>(src, dst, inv, n);
    g_launches++;
}

void launch_gather_perm_u64(const unsigned long long* src, unsigned long long* dst, const unsigned* inv, long long n,
                            cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_gather_perm<unsigned long long><<<blocks, 256, 0, st>>>(src, dst, inv, n);
    g_launches++;
}

__global__ void k_permute_f64(const double* __restrict__ src, double* __restrict__ dst,
                              const unsigned* __restrict__ dest, long long n) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        dst[dest[p]] = src[p];
}

void launch_permute_f64(const double* src, double* dst, const unsigned* dest, long long n, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_permute_f64<<<blocks, 256, 0, st>>>(src, dst, dest, n);
    g_launches++;
}

__global__ void k_permute_u64(const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst,
                              const unsigned* __restrict__ dest, long long n) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        dst[dest[p]] = src[p];
}

void launch_permute_u64(const unsigned long long* src, unsigned long long* dst, const unsigned* dest,
                        long long n, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_permute_u64<<<blocks, 256, 0, st>>>(src, dst, dest, n);
    g_launches++;
}

// Tiles.  max_span[i] = the widest label-cell span of ring i whose window
// (all planes, radial band, label windows) fits the shared-memory capacity;
// a geometry constant, computed once at init by a 32-ary search (one
// candidate span per lane).
__global__ void k_tile_spans(Geo g, int cap_nodes, double rho_cut, int* __restrict__ span) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= g.mpsi) return;
    const int mt = __ldg(g.mtheta + i);
    int lo = 1, hi = mt;  // answer in [lo, hi]; span 1 assumed to fit (else one-cell tiles go via L2)
    while (lo < hi) {
        const int c = lo + (int)(((long long)(hi - lo) * (lane + 1) + 31) / 32);  // in (lo, hi]
        const bool fits = win_nodes(g, i, 0, c - 1, rho_cut) <= cap_nodes;
        const unsigned fm = __ballot_sync(0xffffffffu, fits), nm = __ballot_sync(0xffffffffu, !fits);
        // candidates increase with the lane: the fitting ones form a prefix
        const int nlo = fm ? __shfl_sync(0xffffffffu, c, 31 - __clz(fm)) : lo;
        const int nhi = nm ? __shfl_sync(0xffffffffu, c, __ffs(nm) - 1) - 1 : hi;
        lo = nlo;
        hi = nhi;
    }
    if (lane == 0) span[i] = lo;
}

void launch_tile_spans(const Geo& g, int cap_nodes, int* span, cudaStream_t st) {
    k_tile_spans<<<(g.mpsi + 3) / 4, 128, 0, st>>>(g, cap_nodes, deposit_rho_cut(g), span);
    g_launches++;
}

// One warp per ring: the lanes fetch 32 cells' particle extents at a time
// (cell c of ring i owns keys [(igrid_i+c)P, (igrid_i+c+1)P)), lane 0 packs
// consecutive cells greedily into tiles of at most tile_max particles and at
// most max_span cells.  Returns the ring's tile count (written if out).
__device__ int ring_tiles_warp(const Geo& g, int i, const unsigned* __restrict__ offset, int tile_max,
                               int max_span, Tile* out, int max_out) {
    const int lane = threadIdx.x & 31;
    const int mt = __ldg(g.mtheta + i), ig = __ldg(g.igrid + i);
    int nt = 0, c0 = 0;
    const long long ks = (long long)g.P * g.nmu;  // keys per cell
    long long cur = 0, tstart = offset[(long long)ig * ks];
    auto emit = [&](int a, int b, long long s0, long long s1) {
        if (s1 <= s0) return;
        if (out && nt < max_out) {
            Tile t;
            t.ring = i; t.c0 = a; t.c1 = b; t.pad = 0; t.start = s0; t.end = s1;
            out[nt] = t;
        }
        nt++;
    };
    for (int cb = 0; cb < mt; cb += 32) {
        const int cl = cb + lane;
        unsigned cs_l = 0, ce_l = 0;
        if (cl < mt) {
            cs_l = offset[(long long)(ig + cl) * ks];
            ce_l = offset[(long long)(ig + cl + 1) * ks];
        }
        const int nq = min(32, mt - cb);
        for (int q = 0; q < nq; q++) {
            const long long cs = __shfl_sync(0xffffffffu, cs_l, q);
            const long long ce = __shfl_sync(0xffffffffu, ce_l, q);
            if (lane != 0) continue;
            const int c = cb + q;
            const long long cnt = ce - cs;
            if (cnt == 0) continue;
            if (cur > 0 && (cur + cnt > tile_max || c - c0 + 1 > max_span)) {
                emit(c0, c - 1 < c0 ? c0 : c - 1, tstart, cs);
                cur = 0;
                tstart = cs;
                c0 = c;
            }
            if (cur == 0) { tstart = cs; c0 = c; }
            cur += cnt;
            while (cur > tile_max) {
                emit(c0, c, tstart, tstart + tile_max);
                tstart += tile_max;
                cur -= tile_max;
                c0 = c;
            }
        }
    }
    if (lane == 0 && cur > 0) emit(c0, mt - 1, tstart, tstart + cur);
    return __shfl_sync(0xffffffffu, nt, 0);
}

// pass 1: tile count per ring (rings with gyrocentres: 0..mpsi-1, the bin key
// uses the floor ring), one warp per ring spread over the SMs
__global__ void k_tiles_count(Geo g, const unsigned* __restrict__ offset, int tile_max, const int* __restrict__ span,
                              int* __restrict__ ring_cnt) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= g.mpsi) return;
    const int n = ring_tiles_warp(g, i, offset, tile_max, span[i], nullptr, 0);
    if ((threadIdx.x & 31) == 0) ring_cnt[i] = n;
}

// pass 2: each warp sums the counts of the rings before its own, then writes
__global__ void k_tiles_write(Geo g, const unsigned* __restrict__ offset, int tile_max, const int* __restrict__ span,
                              const int* __restrict__ ring_cnt, Tile* tiles, int max_tiles, DevCounters* dc) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= g.mpsi) return;
    int acc = 0;
    for (int q = lane; q < i; q += 32) acc += ring_cnt[q];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int room = max_tiles - acc;
    if (room > 0) ring_tiles_warp(g, i, offset, tile_max, span[i], tiles + acc, room);
    if (i == g.mpsi - 1 && lane == 0) dc->ntiles = min(acc + ring_cnt[i], max_tiles);
}

void launch_build_tiles(const Geo& g, const unsigned* offset, int tile_max, Tile* tiles, int max_tiles,
                        DevCounters* dc, const int* span, int* ring_cnt, cudaStream_t st) {
    const int blocks = (g.mpsi + 3) / 4;
    k_tiles_count<<<blocks, 128, 0, st>>>(g, offset, tile_max, span, ring_cnt);
    k_tiles_write<<<blocks, 128, 0, st>>>(g, offset, tile_max, span, ring_cnt, tiles, max_tiles, dc);
    g_launches += 2;
}

// deterministic sum: fixed grid of partials, then one block in fixed order
template <class R>
__global__ void k_sum_partial(const double* __restrict__ x, long long n, double* __restrict__ partial) {
    double s = 0.0;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
        s += ldp<R>(x, p);
    __shared__ double sm[32];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += sm[w];
        partial[blockIdx.x] = t;
    }
}

__global__ void k_sum_final(const double* __restrict__ partial, int nb, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < nb; b++) t += partial[b];
        out[0] = t;
    }
}

void launch_sum_f64(const double* x, long long n, double* out, double* partial, cudaStream_t st) {
    const int nb = 592;
    if (g_prec32) k_sum_partial<float><<<nb, 256, 0, st>>>(x, n, partial);
    else k_sum_partial<double><<<nb, 256, 0, st>>>(x, n, partial);
    k_sum_final<<<1, 32, 0, st>>>(partial, nb, out);
    g_launches += 2;
}

// ---------------------------------------------------------------------------
// diagnostics (SPEC S:578-586 history record): the delta-f ion heat flux
// Q = sum_p w_p E_kin,p v_E,r(p) (E_kin = v_par^2/2 + mu B, v_E,r =
// -gbar_theta / (r Omega0 B), gbar the 4-point gyro-averaged gradient of the
// current field, U-2/U-3) and the field energy sum phi^2 over canonical nodes.
// Fixed grid of per-block partials, summed in block order (deterministic).
// ---------------------------------------------------------------------------
template <class R, class FT>
__global__ void k_heat_flux(Geo g, PSet s, long long n, const double* __restrict__ gf, double* __restrict__ partial) {
    double acc = 0.0;
    const FT* gff = reinterpret_cast<const FT*>(gf);
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const double psi = ldp<R>(s.x[0], p), theta = ldp<R>(s.x[1], p), zeta = ldp<R>(s.x[2], p),
                     rho_par = ldp<R>(s.x[3], p), w = ldp<R>(s.x[4], p), mu = ldp<R>(s.mu, p);
        if (!isfinite((psi + theta + zeta + rho_par + mu) * 0.0 + w)) continue;
        double r, invB, rho, inv_r;
        gyro_radius(g, psi, cos_theta(theta), mu, &r, &invB, &rho, &inv_r);
        double wz1;
        int k = plane_of(g, zeta, &wz1) - g.k0;
        k = min(max(k, 0), g.P - 1);
        const double wz0 = 1.0 - wz1;
        double gt = 0.0;
        const FT* gk = gff + (long long)k * g.gstride * 6;
        gyro_stencil(g, r, theta, zeta, rho, inv_r, [&](int m, int j, int mt, double a0, double a1) {
            const FT* rj = gk + ((long long)__ldg(g.igrid + m) + j) * 6;  // nodes j, j + 1 (duplicate at mt)
            gt += a0 * (wz0 * (double)rj[1] + wz1 * (double)rj[4]) + a1 * (wz0 * (double)rj[7] + wz1 * (double)rj[10]);
            (void)mt;
        });
        const double B = 1.0 / invB;
        const double vpar = g.omega0 * B * rho_par;
        const double vEr = g.drifts ? -gt * inv_r * g.inv_omega0 * invB : 0.0;
        acc += w * (0.5 * vpar * vpar + mu * B) * vEr;
    }
    __shared__ double sm[32];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int wq = 0; wq < (int)(blockDim.x >> 5); wq++) t += sm[wq];
        partial[blockIdx.x] = t;
    }
}

// sum of phi^2 over the canonical nodes (j < mtheta) of the owned planes 0..P-1
__global__ void k_field_energy(Geo g, const double* __restrict__ phi, double* __restrict__ partial) {
    double acc = 0.0;
    const long long total = (long long)g.P * g.mgrid;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int node = (int)(e % g.mgrid);
        const int i = __ldg(g.node_ring + node);
        if (node - __ldg(g.igrid + i) == __ldg(g.mtheta + i)) continue;  // duplicate node
        const double v = phi[e];
        acc += v * v;
    }
    __shared__ double sm[32];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int wq = 0; wq < (int)(blockDim.x >> 5); wq++) t += sm[wq];
        partial[blockIdx.x] = t;
    }
}

void launch_heat_flux(const Geo& g, const PSet& s, long long n, const double* gf, double* out, double* partial,
                      cudaStream_t st) {
    const int nb = 592;
    if (g.prec32) k_heat_flux<float, float><<<nb, 256, 0, st>>>(g, s, n, gf, partial);
    else if (g.f32field) k_heat_flux<double, float><<<nb, 256, 0, st>>>(g, s, n, gf, partial);
    else k_heat_flux<double, double><<<nb, 256, 0, st>>>(g, s, n, gf, partial);
    k_sum_final<<<1, 32, 0, st>>>(partial, nb, out);
    g_launches += 2;
}

void launch_field_energy(const Geo& g, const double* phi, double* out, double* partial, cudaStream_t st) {
    const int nb = 592;
    k_field_energy<<<nb, 256, 0, st>>>(g, phi, partial);
    k_sum_final<<<1, 32, 0, st>>>(partial, nb, out);
    g_launches += 2;
}

__global__ void k_sum_i64_pair(const long long* in2, long long* out) { out[0] = in2[0] + in2[1]; }

void launch_sum_i64_pair(const long long* in2, long long* out, cudaStream_t st) {
    k_sum_i64_pair<<<1, 1, 0, st>>>(in2, out);
    g_launches++;
}

template <class R>
__global__ void k_fill_f64(double* __restrict__ x, long long n, double v) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
        stp<R>(x, p, v);
}

void launch_fill_f64(double* x, long long n, double v, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (g_prec32) k_fill_f64<float><<<blocks, 256, 0, st>>>(x, n, v);
    else k_fill_f64<double><<<blocks, 256, 0, st>>>(x, n, v);
    g_launches++;
}

template <class R>
__global__ void k_gather_f64(const double* __restrict__ src, const long long* __restrict__ idx, long long m,
                             double* __restrict__ out) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < m; q += (long long)gridDim.x * blockDim.x)
        out[q] = ldp<R>(src, idx[q]);
}

void launch_gather_f64(const double* src, const long long* idx, long long m, double* out, cudaStream_t st) {
    int blocks = (int)std::max<long long>(1, std::min<long long>((m + 255) / 256, 148LL * 8));
    if (g_prec32) k_gather_f64<float><<<blocks, 256, 0, st>>>(src, idx, m, out);
    else k_gather_f64<double><<<blocks, 256, 0, st>>>(src, idx, m, out);
    g_launches++;
}

// 8-byte ids: always 64-bit elements, whatever the particle store precision
__global__ void k_gather_u64(const unsigned long long* __restrict__ src, const long long* __restrict__ idx, long long m,
                             unsigned long long* __restrict__ out) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < m; q += (long long)gridDim.x * blockDim.x)
        out[q] = src[idx[q]];
}

void launch_gather_u64(const unsigned long long* src, const long long* idx, long long m, unsigned long long* out,
                       cudaStream_t st) {
    int blocks = (int)std::max<long long>(1, std::min<long long>((m + 255) / 256, 148LL * 8));
    k_gather_u64<<<blocks, 256, 0, st>>>(src, idx, m, out);
    g_launches++;
}

// ---------------------------------------------------------------------------
// load: Philox4x32-10 counter-based generator; counter = (id lo, id hi, draw, 0)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
    const unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        unsigned hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        unsigned hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += W0;
        k.y += W1;
    }
    return c;
}

struct Philox {
    uint2 key;
    unsigned id_lo, id_hi, draw;
    uint4 buf;
    int used;
    __device__ double u53() {  // uniform in [0, 1)
        if (used >= 4) { buf = philox4x32_10(make_uint4(id_lo, id_hi, draw++, 0u), key); used = 0; }
        unsigned a = (&buf.x)[used], b = (&buf.x)[used + 1];
        used += 2;
        unsigned long long m = ((unsigned long long)(a >> 5) << 26) | (b >> 6);
        return (double)m * (1.0 / 9007199254740992.0);
    }
};

template <class R>
__global__ void k_load(Geo g, PSet s, long long n, unsigned long long seed, long long id0, double w_amp,
                       double vcut, double zlo, double zhi, double rlo, double rhi) {
    const double jmax = (1.0 + g.a1 * g.inv_R0) * (1.0 + g.a1 * g.inv_R0);
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        unsigned long long gid = (unsigned long long)(id0 + p);
        Philox rng;
        rng.key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
        rng.id_lo = (unsigned)gid;
        rng.id_hi = (unsigned)(gid >> 32);
        rng.draw = 0;
        rng.used = 4;
        double r, th;
        for (;;) {
            r = sqrt(rlo * rlo + (rhi * rhi - rlo * rlo) * rng.u53());
            if (r >= rhi && rhi < g.a1) continue;  // radial window [rlo, rhi) (last window closed)
            th = GTCP_TWO_PI * rng.u53();
            double J = 1.0 + r * g.inv_R0 * cos(th);
            J *= J;
            if (rng.u53() * jmax < J) break;
        }
        double ze = zlo + (zhi - zlo) * rng.u53();
        if (ze >= zhi) ze = zlo;
        double vpar;
        do {
            double u1 = 1.0 - rng.u53(), u2 = rng.u53();
            vpar = sqrt(-2.0 * log(u1)) * cos(GTCP_TWO_PI * u2);
        } while (fabs(vpar) > vcut);
        double vperp;
        do {
            vperp = sqrt(-2.0 * log(1.0 - rng.u53()));
        } while (vperp > vcut);
        double B = 1.0 / (1.0 + r * g.inv_R0 * cos(th));
        stp<R>(s.x[0], p, 0.5 * r * r);
        stp<R>(s.x[1], p, th);
        stp<R>(s.x[2], p, ze);
        stp<R>(s.x[3], p, vpar / (g.omega0 * B));
        stp<R>(s.x[4], p, w_amp * (2.0 * rng.u53() - 1.0));
        stp<R>(s.mu, p, vperp * vperp / (2.0 * B));
        if (s.id) s.id[p] = gid;
    }
}

void launch_load(const Geo& g, const PSet& s, long long n, unsigned long long seed, long long id0, double w_amp,
                 double vcut, double zlo, double zhi, double rlo, double rhi, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (g.prec32) k_load<float><<<blocks, 256, 0, st>>>(g, s, n, seed, id0, w_amp, vcut, zlo, zhi, rlo, rhi);
    else k_load<double><<<blocks, 256, 0, st>>>(g, s, n, seed, id0, w_amp, vcut, zlo, zhi, rlo, rhi);
    g_launches++;
}

}  // namespace gtcp
