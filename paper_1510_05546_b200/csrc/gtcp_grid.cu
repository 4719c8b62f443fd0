// gtcp_grid.cu -- LIGHT grid kernels: normalisation, smooth, gyro-averaged
// Poisson (weighted Jacobi), zonal solve, field gradients (
// readings F-1..F-5, Q-8 in DESIGN.md §3).  One thread per grid node; the
// per-plane work scales with mgrid, not with particles.
//
// Arrays with halo planes ("H" arrays) hold planes -1..P+1 of this rank's
// domain: plane k lives at offset (k+1)*mgrid.  Plain arrays hold planes 0..P-1.
#include "gtcp_internal.cuh"

namespace gtcp {

static constexpr double kInvTwoPi = 1.0 / GTCP_TWO_PI;

__device__ __forceinline__ int ring_of(const Geo& g, int node) { return __ldg(g.node_ring + node); }

static int blocks_for(long long n, int t = 256) {
    long long b = (n + t - 1) / t;
    return (int)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

#define GRID_LOOP(e, total) \
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (total); e += (long long)gridDim.x * blockDim.x)

// value of plane array `pl` on ring m at physical angle th (plane angle zk),
// linear in the label index, periodic.
__device__ __forceinline__ double ring_interp(const Geo& g, const double* pl, int m, double th, double zk) {
    int mt = __ldg(g.mtheta + m);
    double s = (th - zk * __ldg(g.qtinv + m)) * kInvTwoPi;
    s = s - floor(s);
    s = s * mt;
    int j = min((int)floor(s), mt - 1);
    double wt1 = s - j;
    int j1 = (j + 1 == mt) ? 0 : j + 1;
    const double* ring = pl + __ldg(g.igrid + m);
    return (1.0 - wt1) * ring[j] + wt1 * ring[j1];
}


// copy canonical j=0 into the duplicate j=mtheta on `planes` planes (ncomp interleaved)
__global__ void k_fill_dup(Geo g, double* f, int planes, int ncomp) {
    long long total = (long long)planes * (g.mpsi + 1) * ncomp;
    GRID_LOOP(e, total) {
        int c = (int)(e % ncomp);
        long long t = e / ncomp;
        int i = (int)(t % (g.mpsi + 1));
        int k = (int)(t / (g.mpsi + 1));
        long long a = ((long long)k * g.mgrid + __ldg(g.igrid + i)) * ncomp + c;
        f[a + (long long)__ldg(g.mtheta + i) * ncomp] = f[a];
    }
}

void launch_fill_dup(const Geo& g, double* f, int planes, int ncomp, cudaStream_t st) {
    long long total = (long long)planes * (g.mpsi + 1) * ncomp;
    k_fill_dup<<<blocks_for(total), 256, 0, st>>>(g, f, planes, ncomp);
    g_launches++;
}

// dst(j) = src((j + sign*itran) mod mt) over one plane, all nodes incl. duplicates
// (seam identity G-4: node(k + mzetamax, j) == node(k, j + itran)).
__global__ void k_seam_rotate(Geo g, const double* __restrict__ src, double* __restrict__ dst, int sign) {
    GRID_LOOP(e, (long long)g.mgrid) {
        int node = (int)e;
        int i = ring_of(g, node);
        int mt = __ldg(g.mtheta + i);
        int j = node - __ldg(g.igrid + i);
        int jj = (j + sign * __ldg(g.itran + i)) % mt;
        if (jj < 0) jj += mt;
        dst[node] = src[__ldg(g.igrid + i) + jj];
    }
}

void launch_seam_rotate(const Geo& g, const double* src, double* dst, int sign, cudaStream_t st) {
    k_seam_rotate<<<blocks_for(g.mgrid), 256, 0, st>>>(g, src, dst, sign);
    g_launches++;
}

// int64 plane add with rotation: dst(canonical (j + sign*itran) mod mt) += src(j)
__global__ void k_rotate_add_i64(Geo g, const long long* __restrict__ src, long long* __restrict__ dst, int sign) {
    GRID_LOOP(e, (long long)g.mgrid) {
        int node = (int)e;
        int i = ring_of(g, node);
        int mt = __ldg(g.mtheta + i);
        int j = node - __ldg(g.igrid + i);
        if (j >= mt) continue;
        int jj = (j + sign * __ldg(g.itran + i)) % mt;
        if (jj < 0) jj += mt;
        long long v = src[node];
        if (v) dst[__ldg(g.igrid + i) + jj] += v;
    }
}

void launch_rotate_add_i64(const Geo& g, const long long* src, long long* dst, int sign, cudaStream_t st) {
    k_rotate_add_i64<<<blocks_for(g.mgrid), 256, 0, st>>>(g, src, dst, sign);
    g_launches++;
}

// Q-8: dn(k, node) = rho(k, node) / n_m(ring) on planes 0..P-1 -> H array
__global__ void k_normalize(Geo g, const double* __restrict__ rho, const double* __restrict__ nm,
                            double* __restrict__ dnH) {
    long long total = (long long)g.P * g.mgrid;
    GRID_LOOP(e, total) {
        int node = (int)(e % g.mgrid);
        int i = ring_of(g, node);
        dnH[e + g.mgrid] = rho[e] / nm[i];
    }
}

void launch_normalize(const Geo& g, const double* rho, const double* nm, double* dn, cudaStream_t st) {
    k_normalize<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, rho, nm, dn);
    g_launches++;
}

// F-4 theta pass on owned planes (H arrays), writes canonical + duplicate
__global__ void k_smooth_theta(Geo g, const double* __restrict__ in, double* __restrict__ out) {
    long long total = (long long)g.P * g.mgrid;
    GRID_LOOP(e, total) {
        int k = (int)(e / g.mgrid), node = (int)(e % g.mgrid);
        int i = ring_of(g, node);
        int mt = __ldg(g.mtheta + i), ig = __ldg(g.igrid + i);
        int j = node - ig;
        if (j == mt) j = 0;
        const double* ring = in + (long long)(k + 1) * g.mgrid + ig;
        int jm = (j == 0) ? mt - 1 : j - 1, jp = (j + 1 == mt) ? 0 : j + 1;
        out[e + g.mgrid] = 0.25 * ring[jm] + 0.5 * ring[j] + 0.25 * ring[jp];
    }
}

void launch_smooth_theta(const Geo& g, const double* in, double* out, cudaStream_t st) {
    k_smooth_theta<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, in, out);
    g_launches++;
}

// F-4 radial pass at the same physical angle; boundary rings unchanged
__global__ void k_smooth_r(Geo g, const double* __restrict__ in, double* __restrict__ out) {
    long long total = (long long)g.P * g.mgrid;
    GRID_LOOP(e, total) {
        int k = (int)(e / g.mgrid), node = (int)(e % g.mgrid);
        int i = ring_of(g, node);
        const double* pl = in + (long long)(k + 1) * g.mgrid;
        double v = pl[node];
        if (i > 0 && i < g.mpsi) {
            int mt = __ldg(g.mtheta + i);
            int j = node - __ldg(g.igrid + i);
            if (j == mt) j = 0;
            double zk = (double)(g.k0 + k) * g.dzeta;
            double th = j * (GTCP_TWO_PI / mt) + zk * __ldg(g.qtinv + i);
            v = 0.25 * ring_interp(g, pl, i - 1, th, zk) + 0.5 * pl[__ldg(g.igrid + i) + j] +
                0.25 * ring_interp(g, pl, i + 1, th, zk);
        }
        out[e + g.mgrid] = v;
    }
}

void launch_smooth_r(const Geo& g, const double* in, double* out, cudaStream_t st) {
    k_smooth_r<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, in, out);
    g_launches++;
}

// F-4 pass along the field line: same label on planes k-1, k, k+1 (halos filled)
__global__ void k_smooth_par(Geo g, const double* __restrict__ in, double* __restrict__ out) {
    long long total = (long long)g.P * g.mgrid;
    GRID_LOOP(e, total) {
        long long a = e + g.mgrid;
        out[a] = 0.25 * in[a - g.mgrid] + 0.5 * in[a] + 0.25 * in[a + g.mgrid];
    }
}

void launch_smooth_par(const Geo& g, const double* in, double* out, cudaStream_t st) {
    k_smooth_par<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, in, out);
    g_launches++;
}

// per-ring sums over owned planes and canonical nodes of an H array
__global__ void k_ring_sum(Geo g, const double* __restrict__ fH, double* __restrict__ ringsum) {
    int i = blockIdx.x;
    int mt = __ldg(g.mtheta + i), ig = __ldg(g.igrid + i);
    double s = 0.0;
    // plane by plane (no index division; consecutive threads read consecutive
    // labels), a fixed summation order: deterministic
    for (int k = 0; k < g.P; k++) {
        const double* row = fH + (long long)(k + 1) * g.mgrid + ig;
        for (int j = threadIdx.x; j < mt; j += blockDim.x) s += row[j];
    }
    __shared__ double sm[32];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) ringsum[i] = s;
    }
}

void launch_ring_sum(const Geo& g, const double* f, double* ringsum, cudaStream_t st) {
    k_ring_sum<<<g.mpsi + 1, 1024, 0, st>>>(g, f, ringsum);
    g_launches++;
}

// ring sums of a plain (non-halo) plane-major array over planes 0..P-1
void launch_marker_from_rho(const Geo& g, const double* rho, double* ringsum, cudaStream_t st) {
    // rho has planes 0..P at offset k*mgrid: view it as an H array shifted by one plane
    k_ring_sum<<<g.mpsi + 1, 1024, 0, st>>>(g, rho - g.mgrid, ringsum);
    g_launches++;
}

__global__ void k_ring_mean(Geo g, const double* ringsum, double* nm) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= g.mpsi) nm[i] = ringsum[i] / ((double)g.mzetamax * __ldg(g.mtheta + i));
}

void launch_ring_mean(const Geo& g, const double* ringsum, double* nm, cudaStream_t st) {
    k_ring_mean<<<(g.mpsi + 256) / 256, 256, 0, st>>>(g, ringsum, nm);
    g_launches++;
}

// F-2 init: rhs = dn - <dn>_ring, phi0 = rhs / (1 + 1/tau), phi = 0 on boundary rings
__global__ void k_jacobi_init(Geo g, const double* __restrict__ dnH, const double* __restrict__ ringsum,
                              double* __restrict__ rhs, double* __restrict__ phi) {
    long long total = (long long)g.P * g.mgrid;
    const double c0 = 1.0 + 1.0 / g.tau;
    GRID_LOOP(e, total) {
        int node = (int)(e % g.mgrid);
        int i = ring_of(g, node);
        double nbar = ringsum[i] / ((double)g.mzetamax * __ldg(g.mtheta + i));
        double rr = dnH[e + g.mgrid] - nbar;
        rhs[e] = rr;
        phi[e] = (i == 0 || i == g.mpsi) ? 0.0 : rr / c0;
    }
}

void launch_jacobi_init(const Geo& g, const double* dn, const double* ringsum, double* rhs, double* phi,
                        cudaStream_t st) {
    k_jacobi_init<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, dn, ringsum, rhs, phi);
    g_launches++;
}

// value of a ring at fractional label s in [0, mt): linear in the label, periodic
__device__ __forceinline__ double lerp_ring(const double* ring, int mt, double s) {
    const int j0 = min((int)floor(s), mt - 1);
    const double w = s - j0;
    const int j1 = (j0 + 1 == mt) ? 0 : j0 + 1;
    return (1.0 - w) * ring[j0] + w * ring[j1];
}

// F-1 four-point gyro-average at node (ring i, label j) of plane pl at plane
// angle zk: points (r_i +- rhoG, theta) interpolated between their bounding
// rings, (r_i, theta +- rhoG / r_i) on ring i (r = r_i: radial weight 1), each
// label from the per-ring constants with one fma.
__device__ __forceinline__ double gyro_value_tab(const PoisRing* __restrict__ R, const double* pl, int j,
                                                 double zk) {
    const int mt = R->mt;
    const double* ring = pl + R->ig;
    double s = (double)j + R->dlab;
    if (s >= mt) s -= mt;
    double v = lerp_ring(ring, mt, s);
    s = (double)j - R->dlab;
    if (s < 0.0) s += mt;
    v += lerp_ring(ring, mt, s);
#pragma unroll
    for (int sg = 0; sg < 2; sg++) {
        const double wp = R->wp[sg];
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const int t = 2 * sg + q;
            const int mtm = R->mtm[t];
            double y = fma((double)j, R->ratio[t], zk * R->cz[t]) * R->inv_mt[t];
            y = (y - floor(y)) * mtm;
            acc += (q ? wp : 1.0 - wp) * lerp_ring(pl + R->igm[t], mtm, y);
        }
        v += acc;
    }
    return 0.25 * v;
}

// F-1 on planes kbeg..kend-1 of the plain arrays; grid (nodes, plane groups):
// each thread does kGyroKP planes of its node, so the ring lookups and the
// plane-independent labels are shared and the planes' gathers are in flight
// together (the kernel is bound by its dependent load chains: ncu long
// scoreboard 10 per issue with one plane per thread).  Same arithmetic per
// (node, plane); a group's tail planes repeat the last plane's work.
// Measured at class A (Poisson ms/step): 1 plane 2.77 / 2.69 (32 regs),
// 2 planes 2.51 (48 regs, 5 CTAs/SM), 2.60 (40), 4 planes 3.0-3.5.
static constexpr int kGyroKP = 2;
static constexpr int kGyroMinBlocks = 5;
__global__ void __launch_bounds__(256, kGyroMinBlocks) k_gyro(Geo g, const PoisRing* __restrict__ pr, const double* __restrict__ in,
                       double* __restrict__ out, int kbeg, int kend) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.mgrid) return;
    const int kq = kbeg + blockIdx.y * kGyroKP;
    const int i = ring_of(g, node);
    const PoisRing* R = pr + i;
    int j = node - R->ig;
    if (j == R->mt) j = 0;
    double v[kGyroKP];
#pragma unroll
    for (int q = 0; q < kGyroKP; q++) {
        const int k = min(kq + q, kend - 1);
        v[q] = gyro_value_tab(R, in + (long long)k * g.mgrid, j, (double)(g.k0 + k) * g.dzeta);
    }
#pragma unroll
    for (int q = 0; q < kGyroKP; q++)
        if (kq + q < kend) out[(long long)(kq + q) * g.mgrid + node] = v[q];
}

static dim3 grid_nodes_planes(const Geo& g, int kcount) {
    return dim3((unsigned)((g.mgrid + 255) / 256), (unsigned)((kcount + kGyroKP - 1) / kGyroKP));
}

void launch_gyro(const Geo& g, const PoisRing* pr, const double* in, double* out, int kbeg, int kcount,
                 cudaStream_t st) {
    if (kcount <= 0) return;
    k_gyro<<<grid_nodes_planes(g, kcount), 256, 0, st>>>(g, pr, in, out, kbeg, kbeg + kcount);
    g_launches++;
}

// second G application fused with the Jacobi update (F-2):
// phi <- (1-omega) phi + omega (rhs + G(g1)) / (1 + 1/tau), phi = 0 on rings 0, mpsi
__global__ void __launch_bounds__(256, kGyroMinBlocks) k_gyro_jacobi(Geo g, const PoisRing* __restrict__ pr, const double* __restrict__ g1,
                              const double* __restrict__ rhs, double* __restrict__ phi, double omega, int kbeg,
                              int kend) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.mgrid) return;
    const int kq = kbeg + blockIdx.y * kGyroKP;
    const int i = ring_of(g, node);
    if (i == 0 || i == g.mpsi) {
#pragma unroll
        for (int q = 0; q < kGyroKP; q++)
            if (kq + q < kend) phi[(long long)(kq + q) * g.mgrid + node] = 0.0;
        return;
    }
    const double c0 = 1.0 + 1.0 / g.tau;
    const PoisRing* R = pr + i;
    int j = node - R->ig;
    if (j == R->mt) j = 0;
    double v[kGyroKP];
#pragma unroll
    for (int q = 0; q < kGyroKP; q++) {
        const int k = min(kq + q, kend - 1);
        v[q] = gyro_value_tab(R, g1 + (long long)k * g.mgrid, j, (double)(g.k0 + k) * g.dzeta);
    }
#pragma unroll
    for (int q = 0; q < kGyroKP; q++) {
        if (kq + q < kend) {
            const long long e = (long long)(kq + q) * g.mgrid + node;
            phi[e] = (1.0 - omega) * phi[e] + omega * (rhs[e] + v[q]) / c0;
        }
    }
}

void launch_gyro_jacobi(const Geo& g, const PoisRing* pr, const double* g1, const double* rhs, double* phi,
                        double omega, int kbeg, int kcount, cudaStream_t st) {
    if (kcount <= 0) return;
    k_gyro_jacobi<<<grid_nodes_planes(g, kcount), 256, 0, st>>>(g, pr, g1, rhs, phi, omega, kbeg, kbeg + kcount);
    g_launches++;
}

// F-3 zonal flow: -rho_i^2 (1/r)(r phi00')' = <dn>, Dirichlet ends, Thomas algorithm.
// ringsum holds the global ring sums of dn (mean = sum / (mzetamax * mtheta)).
__global__ void k_zonal(Geo g, const double* __restrict__ ringsum, double* __restrict__ phi00, double* work) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int M = g.mpsi;
    double rho2 = 1.0 / (g.omega0 * g.omega0);
    double* b = work;
    double* d = work + (M + 1);
    double* a = work + 2 * (M + 1);
    double* c = work + 3 * (M + 1);
    for (int i = 1; i < M; i++) {
        double r = g.a0 + i * g.dr;
        double f = rho2 / (r * g.dr * g.dr);
        a[i] = -f * (r - 0.5 * g.dr);
        b[i] = f * ((r + 0.5 * g.dr) + (r - 0.5 * g.dr));
        c[i] = -f * (r + 0.5 * g.dr);
        d[i] = ringsum[i] / ((double)g.mzetamax * __ldg(g.mtheta + i));
    }
    for (int i = 2; i < M; i++) {
        double m = a[i] / b[i - 1];
        b[i] -= m * c[i - 1];
        d[i] -= m * d[i - 1];
    }
    phi00[0] = 0.0;
    phi00[M] = 0.0;
    if (M >= 2) phi00[M - 1] = d[M - 1] / b[M - 1];
    for (int i = M - 2; i >= 1; i--) phi00[i] = (d[i] - c[i] * phi00[i + 1]) / b[i];
}

void launch_zonal(const Geo& g, const double* ringsum, double* phi00, cudaStream_t st) {
    // phi00 buffer has room for (mpsi+1) outputs followed by 4*(mpsi+1) scratch
    k_zonal<<<1, 32, 0, st>>>(g, ringsum, phi00, phi00 + (g.mpsi + 1));
    g_launches++;
}

// phi (plain, from Jacobi) + phi00(ring) -> H array planes 0..P-1
__global__ void k_add_zonal(Geo g, const double* __restrict__ phi00, const double* __restrict__ phi,
                            double* __restrict__ phiH) {
    long long total = (long long)g.P * g.mgrid;
    GRID_LOOP(e, total) {
        int node = (int)(e % g.mgrid);
        phiH[e + g.mgrid] = phi[e] + phi00[ring_of(g, node)];
    }
}

void launch_add_zonal2(const Geo& g, const double* phi00, const double* phi, double* phiH, cudaStream_t st) {
    k_add_zonal<<<blocks_for((long long)g.P * g.mgrid), 256, 0, st>>>(g, phi00, phi, phiH);
    g_launches++;
}

// F-5 field on planes 0..P from phi H array (planes -1..P+1 filled) into the
// gather layout gf[interval][node][plane-of-interval][3].
template <class FT>
__global__ void k_field(Geo g, const double* __restrict__ phiH, FT* __restrict__ gf) {
    long long total = (long long)(g.P + 1) * g.mgrid;
    const double inv2dz = 1.0 / (2.0 * g.dzeta);
    GRID_LOOP(e, total) {
        int k = (int)(e / g.mgrid), node = (int)(e % g.mgrid);
        int i = ring_of(g, node);
        int mt = __ldg(g.mtheta + i), ig = __ldg(g.igrid + i);
        int j = node - ig;
        if (j == mt) j = 0;
        const double* pl = phiH + (long long)(k + 1) * g.mgrid;
        double zk = (double)(g.k0 + k) * g.dzeta;
        double dth = GTCP_TWO_PI / mt;
        double th = j * dth + zk * __ldg(g.qtinv + i);
        double here = pl[ig + j];
        double gr;
        if (i == 0)
            gr = (ring_interp(g, pl, 1, th, zk) - here) * g.inv_dr;
        else if (i == g.mpsi)
            gr = (here - ring_interp(g, pl, g.mpsi - 1, th, zk)) * g.inv_dr;
        else
            gr = (ring_interp(g, pl, i + 1, th, zk) - ring_interp(g, pl, i - 1, th, zk)) * (0.5 * g.inv_dr);
        int jp = (j + 1 == mt) ? 0 : j + 1, jm = (j == 0) ? mt - 1 : j - 1;
        double gt = (pl[ig + jp] - pl[ig + jm]) / (2.0 * dth);
        double gp = (pl[g.mgrid + ig + j] - pl[-(long long)g.mgrid + ig + j]) * inv2dz;
        if (k < g.P) {
            FT* o = gf + ((long long)k * g.gstride + node) * 6;
            o[0] = (FT)gr; o[1] = (FT)gt; o[2] = (FT)gp;
        }
        if (k > 0) {
            FT* o = gf + ((long long)(k - 1) * g.gstride + node) * 6 + 3;
            o[0] = (FT)gr; o[1] = (FT)gt; o[2] = (FT)gp;
        }
    }
}

void launch_field(const Geo& g, const double* phi, double* gfield, cudaStream_t st) {
    // precision 32: the gather field is stored in fp32 next to the fp32 particle state
    if (g.f32field) k_field<float><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, phi, (float*)gfield);
    else k_field<double><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, phi, gfield);
    g_launches++;
}

// gather layout -> (P+1) x mgrid x 3 plane-major
template <class FT>
__global__ void k_gfield_export(Geo g, const FT* __restrict__ gf, double* __restrict__ out) {
    long long total = (long long)(g.P + 1) * g.mgrid;
    GRID_LOOP(e, total) {
        int k = (int)(e / g.mgrid), node = (int)(e % g.mgrid);
        const FT* s = (k < g.P) ? gf + ((long long)k * g.gstride + node) * 6
                                : gf + ((long long)(k - 1) * g.gstride + node) * 6 + 3;
        out[e * 3 + 0] = s[0];
        out[e * 3 + 1] = s[1];
        out[e * 3 + 2] = s[2];
    }
}

void launch_gfield_export(const Geo& g, const double* gfield, double* out, cudaStream_t st) {
    if (g.f32field)
        k_gfield_export<float><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, (const float*)gfield, out);
    else k_gfield_export<double><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, gfield, out);
    g_launches++;
}

template <class FT>
__global__ void k_gfield_import(Geo g, const double* __restrict__ in, FT* __restrict__ gf) {
    long long total = (long long)(g.P + 1) * g.mgrid;
    GRID_LOOP(e, total) {
        int k = (int)(e / g.mgrid), node = (int)(e % g.mgrid);
        for (int c = 0; c < 3; c++) {
            double v = in[e * 3 + c];
            if (k < g.P) gf[((long long)k * g.gstride + node) * 6 + c] = (FT)v;
            if (k > 0) gf[((long long)(k - 1) * g.gstride + node) * 6 + 3 + c] = (FT)v;
        }
    }
}

void launch_gfield_import(const Geo& g, const double* in, double* gfield, cudaStream_t st) {
    if (g.f32field)
        k_gfield_import<float><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, in, (float*)gfield);
    else k_gfield_import<double><<<blocks_for((long long)(g.P + 1) * g.mgrid), 256, 0, st>>>(g, in, gfield);
    g_launches++;
}

}  // namespace gtcp
