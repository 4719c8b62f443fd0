/*
 * gtcp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct, single-threaded fp64 CPU oracle of the
 * GTC-P gyrokinetic PIC hot path described in arXiv:1510.05546.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1510_05546_b200/) never imports, links or executes it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; the readings of points
 * where the paper is silent are the SURVEY.md §8(c) items (G-*, Q-*, F-*, U-*,
 * H-*) and are listed in DESIGN.md §3.  Compile with -ffp-contract=off so that
 * every a*b+c is two rounded operations (shift destinations must be bit-exact).
 *
 * Grid layout used here (oracle-private): plane-major, node index
 *   node(k, i, j) = k*mgrid + igrid[i] + j,  j = 0..mtheta[i]  (j = mtheta[i]
 * duplicates j = 0, G-2).  Vector fields are stored node-major with 3
 * components (g_r, g_theta, g_par).
 *
 * Parity status of every function is given in its comment ("pinned by ..." or
 * "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TWO_PI (2.0 * 3.14159265358979323846)

typedef struct {
    int32_t mpsi, mthetamax, mzetamax;
    int32_t paranl;         /* 1: velocity-space nonlinearity      */
    int32_t drifts;         /* 1 normally; 0 = test-only drift-off flag (U-*)  */
    int32_t poisson_iters;  /* fixed Jacobi count (F-2)                        */
    double a0, a1;          /* radial boundaries r = 0.1a, 0.9a   */
    double R0;              /* major radius / a (reading C-4)                  */
    double omega0;          /* a / rho_i (C-1, C-2)                            */
    double q0, q2;          /* q(r) = q0 + q2 r^2 (C-5)                 */
    double rln, rlt;        /* R0/L_n, R0/L_T                          */
    double tau;             /* T_e / T_i                                       */
    double dt;              /* time step (C-3)                                 */
    double jacobi_omega;    /* weighted-Jacobi weight (F-2)             */
} orc_params;

/* ------------------------------------------------------------------ */
/* Geometry (P:170-173 field-line-following grid; G-1..G-4)            */
/* ------------------------------------------------------------------ */

static double orc_dr(const orc_params* p) { return (p->a1 - p->a0) / p->mpsi; }
static double orc_ring_r(const orc_params* p, int i) { return p->a0 + i * orc_dr(p); }
static double orc_q(const orc_params* p, double r) { return p->q0 + p->q2 * r * r; }

/* Fill mtheta[0..mpsi], igrid[0..mpsi+1], itran[0..mpsi], qtinv[0..mpsi];
 * return mgrid.  G-1: rings uniform in r; G-2: mtheta_i =
 * 2*floor(mthetamax*r_i/(2*a1) + 1/2) (pinned exactly by Tab.2 mgrid);
 * G-4: itran_i = floor(mtheta_i/q(r_i) + 1/2), qtinv_i = itran_i/mtheta_i. */
int64_t orc_geometry(const orc_params* p, int32_t* mtheta, int64_t* igrid,
                     int32_t* itran, double* qtinv) {
    igrid[0] = 0;
    for (int i = 0; i <= p->mpsi; i++) {
        double r = orc_ring_r(p, i);
        mtheta[i] = 2 * (int32_t)floor(p->mthetamax * r / (2.0 * p->a1) + 0.5);
        itran[i] = (int32_t)floor(mtheta[i] / orc_q(p, r) + 0.5);
        qtinv[i] = (double)itran[i] / (double)mtheta[i];
        igrid[i + 1] = igrid[i] + mtheta[i] + 1;
    }
    return igrid[p->mpsi + 1];
}

/* Internal geometry bundle. */
typedef struct {
    int32_t* mtheta;
    int64_t* igrid;
    int32_t* itran;
    double* qtinv;
    int64_t mgrid;
} orc_geom;

static void geom_build(const orc_params* p, orc_geom* g) {
    g->mtheta = (int32_t*)malloc(sizeof(int32_t) * (p->mpsi + 1));
    g->igrid = (int64_t*)malloc(sizeof(int64_t) * (p->mpsi + 2));
    g->itran = (int32_t*)malloc(sizeof(int32_t) * (p->mpsi + 1));
    g->qtinv = (double*)malloc(sizeof(double) * (p->mpsi + 1));
    g->mgrid = orc_geometry(p, g->mtheta, g->igrid, g->itran, g->qtinv);
}
static void geom_free(orc_geom* g) {
    free(g->mtheta); free(g->igrid); free(g->itran); free(g->qtinv);
}

/* Equilibrium (G-5; circular, large aspect ratio, low beta: P:123). */
static double orc_B(const orc_params* p, double r, double theta) {
    return 1.0 / (1.0 + r / p->R0 * cos(theta));
}

/* Gradient drive profile (C-6; "exp{-[(r-0.5a)/0.35a]^6}"). */
double orc_prof(double r) {
    double x = (r - 0.5) / 0.35;
    return exp(-(x * x * x * x * x * x));
}

double orc_qprofile(const orc_params* p, double r) { return orc_q(p, r); }
double orc_bfield(const orc_params* p, double r, double theta) { return orc_B(p, r, theta); }

/* ------------------------------------------------------------------ */
/* The 4-point gyro-averaged stencil shared by charge and  */
/* gather.  Q-1..Q-6.                                      */
/* ------------------------------------------------------------------ */

/* One contribution = node index within a P+1-plane local grid + weight. */
typedef struct {
    int64_t node[32];
    double wgt[32];
    int n;
    int clamped_plane;   /* 1 if the plane index had to be clamped (Q-2) */
} orc_stencil;

/* Q-2 / H-1: global plane index kg and its weight.  The constant
 * mzetamax/(2 pi) is rounded to fp64 once; t_g = zeta * that constant. */
static void orc_plane(const orc_params* p, double zeta, int32_t* kg, double* wz1) {
    double cz = p->mzetamax / TWO_PI;
    double tg = zeta * cz;
    double f = floor(tg);
    int32_t k = (int32_t)f;
    if (k > p->mzetamax - 1) k = p->mzetamax - 1;
    if (k < 0) k = 0;
    *kg = k;
    *wz1 = tg - (double)k;
}

/* Build the <=32 (node, weight) pairs of one particle on the local grid of
 * planes k0..k0+P (P+1 planes stored).  Weights include the 1/4 of each
 * gyro-point (Q-6) but not the particle weight w. */
static void orc_build_stencil(const orc_params* p, const orc_geom* g,
                              double psi, double theta, double zeta, double mu,
                              int32_t k0, int32_t P, orc_stencil* st) {
    double dr = orc_dr(p);
    /* Q-1 */
    double r = sqrt(2.0 * psi);
    double B = orc_B(p, r, theta);
    double rho = sqrt(2.0 * mu / B) / p->omega0;
    /* Q-2 */
    int32_t kg;
    double wz1;
    orc_plane(p, zeta, &kg, &wz1);
    int32_t k = kg - k0;
    st->clamped_plane = 0;
    if (k < 0) { k = 0; st->clamped_plane = 1; }
    if (k > P - 1) { k = P - 1; st->clamped_plane = 1; }
    double wz[2] = {1.0 - wz1, wz1};
    /* Q-3: four points (dr, dtheta) = (rho,0), (0,rho/r), (-rho,0), (0,-rho/r) */
    double pdr[4] = {rho, 0.0, -rho, 0.0};
    double pdt[4] = {0.0, rho / r, 0.0, -rho / r};
    st->n = 0;
    for (int l = 0; l < 4; l++) {
        double rl = r + pdr[l];
        if (rl < p->a0) rl = p->a0;
        if (rl > p->a1) rl = p->a1;
        double tl = theta + pdt[l];
        /* Q-4 radial cell */
        double x = (rl - p->a0) / dr;
        int32_t i = (int32_t)floor(x);
        if (i < 0) i = 0;
        if (i > p->mpsi - 1) i = p->mpsi - 1;
        double wp1 = x - i;
        double wp[2] = {1.0 - wp1, wp1};
        for (int mm = 0; mm < 2; mm++) {
            int32_t m = i + mm;
            /* Q-5 field-aligned label index on ring m */
            double s = (tl - zeta * g->qtinv[m]) / TWO_PI;
            s = s - floor(s);
            s = s * g->mtheta[m];
            int32_t j = (int32_t)floor(s);
            if (j < 0) j = 0;
            if (j > g->mtheta[m] - 1) j = g->mtheta[m] - 1;
            double wt1 = s - j;
            double wt[2] = {1.0 - wt1, wt1};
            /* Q-6 */
            for (int kk = 0; kk < 2; kk++) {
                for (int jj = 0; jj < 2; jj++) {
                    st->node[st->n] = (int64_t)(k + kk) * g->mgrid + g->igrid[m] + j + jj;
                    st->wgt[st->n] = 0.25 * wz[kk] * wp[mm] * wt[jj];
                    st->n++;
                }
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* Charge deposition (Q-1..Q-6).                            */
/* Pinned by: charge conservation, hand cases 1-2, brute-force         */
/* node-centric deposit, 8..32 unique nodes (tests/test_oracle_*.py).  */
/* ------------------------------------------------------------------ */

/* grid has (P+1)*mgrid entries and is ACCUMULATED into (caller zeroes it).
 * Returns the number of particles whose plane had to be clamped. */
int64_t orc_deposit(const orc_params* p, int64_t n, const double* psi, const double* theta,
                    const double* zeta, const double* mu, const double* w,
                    int32_t k0, int32_t P, double* grid) {
    orc_geom g;
    geom_build(p, &g);
    int64_t nclamp = 0;
    orc_stencil st;
    for (int64_t ip = 0; ip < n; ip++) {
        orc_build_stencil(p, &g, psi[ip], theta[ip], zeta[ip], mu[ip], k0, P, &st);
        nclamp += st.clamped_plane;
        for (int c = 0; c < st.n; c++) grid[st.node[c]] += w[ip] * st.wgt[c];
    }
    geom_free(&g);
    return nclamp;
}

/* Q-7 on a single-domain (global) grid of mzetamax+1 planes:
 * fold the duplicate node j=mtheta into j=0; add the seam plane mzetamax into
 * plane 0 with the exact label rotation j -> (j + itran) mod mtheta (G-4);
 * then copy canonical values back to duplicates and to the seam plane. */
void orc_charge_reduce_global(const orc_params* p, double* grid) {
    orc_geom g;
    geom_build(p, &g);
    int32_t K = p->mzetamax;
    for (int32_t k = 0; k <= K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++) {
            double* ring = grid + (int64_t)k * g.mgrid + g.igrid[i];
            ring[0] += ring[g.mtheta[i]];
            ring[g.mtheta[i]] = 0.0;
        }
    for (int32_t i = 0; i <= p->mpsi; i++) {
        double* seam = grid + (int64_t)K * g.mgrid + g.igrid[i];
        double* first = grid + g.igrid[i];
        for (int32_t j = 0; j < g.mtheta[i]; j++)
            first[(j + g.itran[i]) % g.mtheta[i]] += seam[j];
    }
    for (int32_t k = 0; k < K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++) {
            double* ring = grid + (int64_t)k * g.mgrid + g.igrid[i];
            ring[g.mtheta[i]] = ring[0];
        }
    for (int32_t i = 0; i <= p->mpsi; i++) {
        double* seam = grid + (int64_t)K * g.mgrid + g.igrid[i];
        double* first = grid + g.igrid[i];
        for (int32_t j = 0; j <= g.mtheta[i]; j++)
            seam[j] = first[(j + g.itran[i]) % g.mtheta[i]];
    }
    geom_free(&g);
}

/* Q-8 (reading; paper silent): marker density per ring = flux-surface mean
 * (over planes 0..mzetamax-1 and canonical nodes) of the reduced charge
 * deposited with w = 1.  Pinned by conservation and by the closed form of
 * markers sitting on nodes with mu = 0 (tests/test_oracle_charge.py). */
void orc_marker_norm(const orc_params* p, int64_t n, const double* psi, const double* theta,
                     const double* zeta, const double* mu, double* nm) {
    orc_geom g;
    geom_build(p, &g);
    int64_t sz = (int64_t)(p->mzetamax + 1) * g.mgrid;
    double* grid = (double*)calloc(sz, sizeof(double));
    double* ones = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int64_t ip = 0; ip < n; ip++) ones[ip] = 1.0;
    orc_deposit(p, n, psi, theta, zeta, mu, ones, 0, p->mzetamax, grid);
    orc_charge_reduce_global(p, grid);
    for (int32_t i = 0; i <= p->mpsi; i++) {
        double s = 0.0;
        for (int32_t k = 0; k < p->mzetamax; k++)
            for (int32_t j = 0; j < g.mtheta[i]; j++)
                s += grid[(int64_t)k * g.mgrid + g.igrid[i] + j];
        nm[i] = s / ((double)p->mzetamax * g.mtheta[i]);
    }
    free(ones);
    free(grid);
    geom_free(&g);
}

/* ------------------------------------------------------------------ */
/* Grid kernels: poisson / smooth / field (F-1..F-5) */
/* All operate on the global grid (mzetamax+1 planes, seam plane last). */
/* ------------------------------------------------------------------ */

/* Value of f on plane k, ring m, at physical angle th (label interpolation,
 * linear in the label index, periodic through the duplicate node). */
static double ring_interp(const orc_params* p, const orc_geom* g, const double* plane,
                          int32_t m, double th, double zeta_k) {
    double s = (th - zeta_k * g->qtinv[m]) / TWO_PI;
    s = s - floor(s);
    s = s * g->mtheta[m];
    int32_t j = (int32_t)floor(s);
    if (j < 0) j = 0;
    if (j > g->mtheta[m] - 1) j = g->mtheta[m] - 1;
    double wt1 = s - j;
    const double* ring = plane + g->igrid[m];
    int32_t j1 = (j + 1) % g->mtheta[m];
    return (1.0 - wt1) * ring[j] + wt1 * ring[j1];
    (void)p;
}

/* Bilinear value of f on plane k at (r, th): radial cell as Q-4. */
static double plane_interp(const orc_params* p, const orc_geom* g, const double* plane,
                           double r, double th, double zeta_k) {
    double dr = orc_dr(p);
    if (r < p->a0) r = p->a0;
    if (r > p->a1) r = p->a1;
    double x = (r - p->a0) / dr;
    int32_t i = (int32_t)floor(x);
    if (i < 0) i = 0;
    if (i > p->mpsi - 1) i = p->mpsi - 1;
    double wp1 = x - i;
    return (1.0 - wp1) * ring_interp(p, g, plane, i, th, zeta_k) +
           wp1 * ring_interp(p, g, plane, i + 1, th, zeta_k);
}

/* F-1: four-point gyro-average operator on one plane with radius
 * rho_G = sqrt(2)/omega0 (so that G^2 ~ Gamma_0 to O(b)).  Parity:
 * pinned by "constant in -> constant out", G(r) = r, the rho -> 0 limit,
 * G(r^2) = r^2 + rho_G^2/2 (radius) and second-order convergence of
 * G cos(m theta) to cos(m theta)[1/2 + 1/2 cos(m rho_G/r)] (angular offset
 * rho_G/r) -- tests/test_oracle_closed_forms.py. */
static void gyro_op(const orc_params* p, const orc_geom* g, const double* in, double* out,
                    int32_t k) {
    double zeta_k = k * (TWO_PI / p->mzetamax);
    double rhoG = sqrt(2.0) / p->omega0;
    for (int32_t i = 0; i <= p->mpsi; i++) {
        double r = orc_ring_r(p, i);
        double dth = TWO_PI / g->mtheta[i];
        for (int32_t j = 0; j < g->mtheta[i]; j++) {
            double th = j * dth + zeta_k * g->qtinv[i];
            double v = plane_interp(p, g, in, r + rhoG, th, zeta_k) +
                       plane_interp(p, g, in, r, th + rhoG / r, zeta_k) +
                       plane_interp(p, g, in, r - rhoG, th, zeta_k) +
                       plane_interp(p, g, in, r, th - rhoG / r, zeta_k);
            out[g->igrid[i] + j] = 0.25 * v;
        }
        out[g->igrid[i] + g->mtheta[i]] = out[g->igrid[i]];
    }
}

/* Copy canonical values to duplicate nodes and the seam plane (G-2, G-4). */
static void fill_dup_and_seam(const orc_params* p, const orc_geom* g, double* f, int ncomp) {
    int32_t K = p->mzetamax;
    for (int32_t k = 0; k < K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int c = 0; c < ncomp; c++) {
                int64_t a = ((int64_t)k * g->mgrid + g->igrid[i]) * ncomp + c;
                f[a + (int64_t)g->mtheta[i] * ncomp] = f[a];
            }
    for (int32_t i = 0; i <= p->mpsi; i++)
        for (int32_t j = 0; j <= g->mtheta[i]; j++)
            for (int c = 0; c < ncomp; c++)
                f[((int64_t)K * g->mgrid + g->igrid[i] + j) * ncomp + c] =
                    f[(g->igrid[i] + (j + g->itran[i]) % g->mtheta[i]) * ncomp + c];
}

/* Value at (k, i, j) for any integer plane k, using the seam identity
 * node(k + mzetamax, i, j) == node(k, i, (j + itran_i) mod mtheta_i) (G-4). */
static double plane_value(const orc_params* p, const orc_geom* g, const double* f,
                          int32_t k, int32_t i, int32_t j) {
    int32_t K = p->mzetamax, mt = g->mtheta[i];
    while (k < 0) { k += K; j = ((j - g->itran[i]) % mt + mt) % mt; }
    while (k >= K) { k -= K; j = (j + g->itran[i]) % mt; }
    return f[(int64_t)k * g->mgrid + g->igrid[i] + j];
}

/* F-4 smooth (reading; "a filter"): one (1/4,1/2,1/4) pass along theta
 * (periodic), then along r at the same physical angle (boundary rings
 * fixed), then along the field line (same label, neighbouring planes, seam
 * rotation).  Pinned: constants preserved, linearity, the exact response
 * 1/2 + 1/2 cos(2 pi m/mt) of a ring Fourier mode with the seam-rotated
 * parallel pass on planes 0 and K-1, and r^2 -> r^2 + dr^2/2 for the radial
 * pass (tests/test_oracle_closed_forms.py). */
void orc_smooth(const orc_params* p, double* f) {
    orc_geom g;
    geom_build(p, &g);
    int32_t K = p->mzetamax;
    int64_t sz = (int64_t)(K + 1) * g.mgrid;
    double* t = (double*)malloc(sizeof(double) * sz);
    /* theta */
    memcpy(t, f, sizeof(double) * sz);
    for (int32_t k = 0; k < K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++) {
            int32_t mt = g.mtheta[i];
            const double* src = t + (int64_t)k * g.mgrid + g.igrid[i];
            double* dst = f + (int64_t)k * g.mgrid + g.igrid[i];
            for (int32_t j = 0; j < mt; j++)
                dst[j] = 0.25 * src[(j - 1 + mt) % mt] + 0.5 * src[j] + 0.25 * src[(j + 1) % mt];
        }
    fill_dup_and_seam(p, &g, f, 1);
    /* r */
    memcpy(t, f, sizeof(double) * sz);
    for (int32_t k = 0; k < K; k++) {
        double zeta_k = k * (TWO_PI / K);
        const double* src = t + (int64_t)k * g.mgrid;
        for (int32_t i = 1; i < p->mpsi; i++) {
            double dth = TWO_PI / g.mtheta[i];
            for (int32_t j = 0; j < g.mtheta[i]; j++) {
                double th = j * dth + zeta_k * g.qtinv[i];
                f[(int64_t)k * g.mgrid + g.igrid[i] + j] =
                    0.25 * ring_interp(p, &g, src, i - 1, th, zeta_k) +
                    0.5 * src[g.igrid[i] + j] +
                    0.25 * ring_interp(p, &g, src, i + 1, th, zeta_k);
            }
        }
    }
    fill_dup_and_seam(p, &g, f, 1);
    /* along the field line */
    memcpy(t, f, sizeof(double) * sz);
    for (int32_t k = 0; k < K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int32_t j = 0; j < g.mtheta[i]; j++)
                f[(int64_t)k * g.mgrid + g.igrid[i] + j] =
                    0.25 * plane_value(p, &g, t, k - 1, i, j) + 0.5 * t[(int64_t)k * g.mgrid + g.igrid[i] + j] +
                    0.25 * plane_value(p, &g, t, k + 1, i, j);
    fill_dup_and_seam(p, &g, f, 1);
    free(t);
    geom_free(&g);
}

/* F-3 zonal flow (reading): -rho_i^2 (1/r) d/dr (r dphi00/dr) =
 * <dn>_ring with phi00 = 0 at both boundary rings; second-order finite
 * differences, Thomas algorithm.  Pinned: residual of the discrete equation
 * and a closed-form solution test. */
void orc_zonal_solve(const orc_params* p, const double* nbar, double* phi00) {
    int32_t M = p->mpsi;
    double dr = orc_dr(p);
    double rho2 = 1.0 / (p->omega0 * p->omega0);
    double* a = (double*)calloc(M + 1, sizeof(double));
    double* b = (double*)calloc(M + 1, sizeof(double));
    double* c = (double*)calloc(M + 1, sizeof(double));
    double* d = (double*)calloc(M + 1, sizeof(double));
    for (int32_t i = 1; i < M; i++) {
        double r = orc_ring_r(p, i);
        double rp = r + 0.5 * dr, rm = r - 0.5 * dr;
        double f = rho2 / (r * dr * dr);
        a[i] = -f * rm;          /* coefficient of phi_{i-1} */
        b[i] = f * (rp + rm);    /* coefficient of phi_i     */
        c[i] = -f * rp;          /* coefficient of phi_{i+1} */
        d[i] = nbar[i];
    }
    /* forward elimination over i = 1..M-1 (phi_0 = phi_M = 0) */
    for (int32_t i = 2; i < M; i++) {
        double m = a[i] / b[i - 1];
        b[i] = b[i] - m * c[i - 1];
        d[i] = d[i] - m * d[i - 1];
    }
    phi00[0] = 0.0;
    phi00[M] = 0.0;
    if (M >= 2) phi00[M - 1] = d[M - 1] / b[M - 1];
    for (int32_t i = M - 2; i >= 1; i--) phi00[i] = (d[i] - c[i] * phi00[i + 1]) / b[i];
    free(a); free(b); free(c); free(d);
}

/* poisson_smooth (Eq.14 with adiabatic electrons; P:176-177 four-
 * point operator + weighted Jacobi; readings F-1..F-4, Q-8):
 *   dn = charge / nm(ring); smooth(dn); nbar = ring mean of dn;
 *   per plane solve (1 + 1/tau) phi - G(G(phi)) = dn - nbar by
 *   poisson_iters weighted-Jacobi sweeps from phi0 = rhs/(1+1/tau), phi = 0 on
 *   rings 0 and mpsi; add the zonal solution phi00(ring); smooth(phi).
 * charge is the reduced global grid (mzetamax+1 planes); phi likewise. */
void orc_poisson_smooth(const orc_params* p, const double* charge, const double* nm, double* phi) {
    orc_geom g;
    geom_build(p, &g);
    int32_t K = p->mzetamax;
    int64_t sz = (int64_t)(K + 1) * g.mgrid;
    double* dn = (double*)calloc(sz, sizeof(double));
    for (int32_t k = 0; k <= K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int32_t j = 0; j <= g.mtheta[i]; j++) {
                int64_t a = (int64_t)k * g.mgrid + g.igrid[i] + j;
                dn[a] = charge[a] / nm[i];
            }
    orc_smooth(p, dn);
    double* nbar = (double*)calloc(p->mpsi + 1, sizeof(double));
    for (int32_t i = 0; i <= p->mpsi; i++) {
        double s = 0.0;
        for (int32_t k = 0; k < K; k++)
            for (int32_t j = 0; j < g.mtheta[i]; j++) s += dn[(int64_t)k * g.mgrid + g.igrid[i] + j];
        nbar[i] = s / ((double)K * g.mtheta[i]);
    }
    double c0 = 1.0 + 1.0 / p->tau;
    double* rhs = (double*)calloc(g.mgrid, sizeof(double));
    double* g1 = (double*)calloc(g.mgrid, sizeof(double));
    double* g2 = (double*)calloc(g.mgrid, sizeof(double));
    for (int32_t k = 0; k < K; k++) {
        double* ph = phi + (int64_t)k * g.mgrid;
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int32_t j = 0; j <= g.mtheta[i]; j++) {
                int64_t a = g.igrid[i] + j;
                rhs[a] = dn[(int64_t)k * g.mgrid + a] - nbar[i];
                ph[a] = (i == 0 || i == p->mpsi) ? 0.0 : rhs[a] / c0;
            }
        for (int it = 0; it < p->poisson_iters; it++) {
            gyro_op(p, &g, ph, g1, k);
            gyro_op(p, &g, g1, g2, k);
            for (int32_t i = 0; i <= p->mpsi; i++)
                for (int32_t j = 0; j <= g.mtheta[i]; j++) {
                    int64_t a = g.igrid[i] + j;
                    double v = (1.0 - p->jacobi_omega) * ph[a] +
                               p->jacobi_omega * (rhs[a] + g2[a]) / c0;
                    ph[a] = (i == 0 || i == p->mpsi) ? 0.0 : v;
                }
        }
    }
    double* phi00 = (double*)calloc(p->mpsi + 1, sizeof(double));
    orc_zonal_solve(p, nbar, phi00);
    for (int32_t k = 0; k < K; k++)
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int32_t j = 0; j <= g.mtheta[i]; j++)
                phi[(int64_t)k * g.mgrid + g.igrid[i] + j] += phi00[i];
    fill_dup_and_seam(p, &g, phi, 1);
    orc_smooth(p, phi);
    free(phi00); free(rhs); free(g1); free(g2); free(nbar); free(dn);
    geom_free(&g);
}

/* Unsmoothed single-plane Jacobi (exposed for the dense-LU pin). */
void orc_jacobi_plane(const orc_params* p, int32_t k, const double* rhs, double* ph) {
    orc_geom g;
    geom_build(p, &g);
    double c0 = 1.0 + 1.0 / p->tau;
    double* g1 = (double*)calloc(g.mgrid, sizeof(double));
    double* g2 = (double*)calloc(g.mgrid, sizeof(double));
    for (int32_t i = 0; i <= p->mpsi; i++)
        for (int32_t j = 0; j <= g.mtheta[i]; j++) {
            int64_t a = g.igrid[i] + j;
            ph[a] = (i == 0 || i == p->mpsi) ? 0.0 : rhs[a] / c0;
        }
    for (int it = 0; it < p->poisson_iters; it++) {
        gyro_op(p, &g, ph, g1, k);
        gyro_op(p, &g, g1, g2, k);
        for (int32_t i = 0; i <= p->mpsi; i++)
            for (int32_t j = 0; j <= g.mtheta[i]; j++) {
                int64_t a = g.igrid[i] + j;
                double v = (1.0 - p->jacobi_omega) * ph[a] + p->jacobi_omega * (rhs[a] + g2[a]) / c0;
                ph[a] = (i == 0 || i == p->mpsi) ? 0.0 : v;
            }
    }
    free(g1); free(g2);
    geom_free(&g);
}

/* Exposed single application of F-1 on plane k (for the operator pins). */
void orc_gyro_op(const orc_params* p, int32_t k, const double* in, double* out) {
    orc_geom g;
    geom_build(p, &g);
    gyro_op(p, &g, in, out, k);
    geom_free(&g);
}

/* F-5 field (reading): gradient triplets (g_r, g_theta, g_par) at
 * every node of planes 0..mzetamax-1, then duplicates and the seam plane.
 *   g_r   = d phi/dr at the node's physical angle (neighbour rings
 *           interpolated at that angle), centred; one-sided at rings 0, mpsi;
 *   g_th  = (phi_{j+1} - phi_{j-1}) / (2 dtheta_i), periodic;
 *   g_par = (phi(k+1) - phi(k-1)) / (2 dzeta) at the same label (seam rotation).
 * Pinned: constant phi -> 0; sin(m theta) -> second-order convergent g_theta;
 * linear-in-r phi -> exact g_r; r cos(theta) -> g_r = cos(theta) at the
 * physical angle (second order); cos(n theta - l zeta) -> second-order
 * g_par on every plane, through the seam rotation
 * (tests/test_oracle_grid.py, tests/test_oracle_closed_forms.py). */
void orc_field(const orc_params* p, const double* phi, double* gradphi) {
    orc_geom g;
    geom_build(p, &g);
    int32_t K = p->mzetamax;
    double dr = orc_dr(p), dz = TWO_PI / K;
    for (int32_t k = 0; k < K; k++) {
        double zeta_k = k * dz;
        const double* pl = phi + (int64_t)k * g.mgrid;
        for (int32_t i = 0; i <= p->mpsi; i++) {
            int32_t mt = g.mtheta[i];
            double dth = TWO_PI / mt;
            for (int32_t j = 0; j < mt; j++) {
                double th = j * dth + zeta_k * g.qtinv[i];
                double here = pl[g.igrid[i] + j];
                double gr;
                if (i == 0)
                    gr = (ring_interp(p, &g, pl, 1, th, zeta_k) - here) / dr;
                else if (i == p->mpsi)
                    gr = (here - ring_interp(p, &g, pl, p->mpsi - 1, th, zeta_k)) / dr;
                else
                    gr = (ring_interp(p, &g, pl, i + 1, th, zeta_k) -
                          ring_interp(p, &g, pl, i - 1, th, zeta_k)) / (2.0 * dr);
                double gt = (pl[g.igrid[i] + (j + 1) % mt] - pl[g.igrid[i] + (j - 1 + mt) % mt]) / (2.0 * dth);
                double gp = (plane_value(p, &g, phi, k + 1, i, j) - plane_value(p, &g, phi, k - 1, i, j)) / (2.0 * dz);
                int64_t a = ((int64_t)k * g.mgrid + g.igrid[i] + j) * 3;
                gradphi[a + 0] = gr;
                gradphi[a + 1] = gt;
                gradphi[a + 2] = gp;
            }
        }
    }
    fill_dup_and_seam(p, &g, gradphi, 3);
    geom_free(&g);
}

/* ------------------------------------------------------------------ */
/* Gather + push (Eqs. 2-8; U-1..U-8)              */
/* ------------------------------------------------------------------ */

/* U-2: gyro-averaged gradient at the particle from a local field of P+1
 * planes (layout node-major x 3).  Pinned: constant field -> exact; mu = 0 at
 * a node -> nodal value; adjointness with orc_deposit. */
void orc_gather(const orc_params* p, int64_t n, const double* psi, const double* theta,
                const double* zeta, const double* mu, int32_t k0, int32_t P,
                const double* gradphi, double* gbar) {
    orc_geom g;
    geom_build(p, &g);
    orc_stencil st;
    for (int64_t ip = 0; ip < n; ip++) {
        orc_build_stencil(p, &g, psi[ip], theta[ip], zeta[ip], mu[ip], k0, P, &st);
        double s[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < st.n; c++)
            for (int d = 0; d < 3; d++) s[d] += st.wgt[c] * gradphi[st.node[c] * 3 + d];
        gbar[ip * 3 + 0] = s[0];
        gbar[ip * 3 + 1] = s[1];
        gbar[ip * 3 + 2] = s[2];
    }
    geom_free(&g);
}

/* Right-hand side F(X) of the gyrocenter equations of motion for
 * X = (psi, theta, zeta, rho_par, w), magnetic moment mu and gyro-averaged
 * gradient gbar = (g_r, g_theta, g_par):
 *   U-1 r = sqrt(2 psi), B, dB/dr, dB/dtheta (G-5), q(r), v_par = omega0 B rho_par
 *   U-3 v_E = b x grad(phi_bar)/B (Eq.5): v_Er = -g_th/(r omega0 B), v_Eth = g_r/(omega0 B)
 *       v_d = (v_par^2/Omega + mu/Z)(b x grad B)/B (Eq.8): C_d = (v_par^2 + mu B)/(omega0 R0),
 *       v_dr = -C_d sin(theta), v_dth = -C_d cos(theta)
 *   U-4 dR/dt = v_par b + v_E + v_d (Eq.2)
 *   U-5 dv_par/dt = -b*.(mu grad B + grad phi_bar) (Eqs.3-4)
 *   U-6 dw/dt = (1 - paranl w) [v_Er kappa - (v_par b + v_d).grad(phi_bar)]
 * The drift-off test flag (drifts = 0) removes v_E, v_d and the
 * (v_par/Omega) b x grad B / B part of b*.  Pinned: E = 0 energy
 * conservation and RK2 order, static-potential energy conservation, drift-
 * off closed form, w constant for E = 0 (tests/test_oracle_push.py). */
void orc_rhs(const orc_params* p, const double* X, double mu, const double* gbar, double* dX) {
    double psi = X[0], theta = X[1], rho_par = X[3], w = X[4];
    double r = sqrt(2.0 * psi);
    double st = sin(theta), ct = cos(theta);
    double B = 1.0 / (1.0 + r / p->R0 * ct);
    double dBdr = -B * B * ct / p->R0;
    double dBdt = B * B * (r / p->R0) * st;
    double q = orc_q(p, r);
    double vpar = p->omega0 * B * rho_par;
    double gr = gbar[0], gt = gbar[1], gp = gbar[2];
    double vEr = 0.0, vEt = 0.0, vdr = 0.0, vdt = 0.0;
    if (p->drifts) {
        vEr = -gt / (r * p->omega0 * B);
        vEt = gr / (p->omega0 * B);
        double Cd = (vpar * vpar + mu * B) / (p->omega0 * p->R0);
        vdr = -Cd * st;
        vdt = -Cd * ct;
    }
    double rdot = vEr + vdr;
    double psidot = r * rdot;
    double thdot = vpar * B / (q * p->R0) + (vEt + vdt) / r;
    double zdot = vpar * B / p->R0;
    double vdot = -mu * B * B * B * r * st / (q * p->R0 * p->R0);
    if (p->paranl) {
        double par = -(B / p->R0) * gp;
        if (p->drifts) par += (vpar / (p->omega0 * p->R0)) * (st * gr + ct * gt / r);
        vdot += par;
    }
    double Bdot = rdot * dBdr + thdot * dBdt;
    double rhodot = (vdot - vpar * Bdot / B) / (p->omega0 * B);
    double Ekin = 0.5 * vpar * vpar + mu * B;
    double kappa = orc_prof(r) * (p->rln + (Ekin - 1.5) * p->rlt) / p->R0;
    double wdot = (1.0 - p->paranl * w) *
                  (vEr * kappa - (vpar * (B / p->R0) * gp + vdr * gr + vdt * gt / r));
    dX[0] = psidot;
    dX[1] = thdot;
    dX[2] = zdot;
    dX[3] = rhodot;
    dX[4] = wdot;
}

/* U-8: wrap theta, zeta into [0, 2 pi); reflect r at a0, a1 (reading A-17).
 * Returns 1 if a reflection happened.  Pinned: one outward and one inward
 * crossing against the closed form r' = 2 a1 - r / 2 a0 - r
 * (tests/test_oracle_closed_forms.py). */
static int orc_post(const orc_params* p, double* X) {
    double t = X[1] - TWO_PI * floor(X[1] / TWO_PI);
    if (t >= TWO_PI) t = 0.0;
    X[1] = t;
    double z = X[2] - TWO_PI * floor(X[2] / TWO_PI);
    if (z >= TWO_PI) z = 0.0;
    X[2] = z;
    double r = sqrt(2.0 * (X[0] > 0.0 ? X[0] : 0.0));
    int refl = 0;
    if (r > p->a1) { r = 2.0 * p->a1 - r; refl = 1; }
    if (r < p->a0) { r = 2.0 * p->a0 - r; refl = 1; }
    if (refl) X[0] = 0.5 * r * r;
    return refl;
}

/* One RK2 stage (U-7, "second order Runge Kutta"):
 *   stage 1: Xb = Xa + (dt/2) F(Xa)
 *   stage 2: Xa = Xa + dt F(Xb)
 * Xa[5], Xb[5] are SoA pointer arrays (psi, theta, zeta, rho_par, w); the
 * field is local (planes k0..k0+P).  mu is never written.  Returns the number
 * of radial reflections. */
int64_t orc_push(const orc_params* p, int32_t stage, int64_t n, double* const* Xa,
                 double* const* Xb, const double* mu, int32_t k0, int32_t P,
                 const double* gradphi) {
    orc_geom g;
    geom_build(p, &g);
    orc_stencil st;
    int64_t nrefl = 0;
    for (int64_t ip = 0; ip < n; ip++) {
        double xa[5], xb[5], x[5], F[5], gb[3] = {0.0, 0.0, 0.0};
        for (int d = 0; d < 5; d++) { xa[d] = Xa[d][ip]; xb[d] = Xb[d][ip]; }
        const double* src = (stage == 1) ? xa : xb;
        orc_build_stencil(p, &g, src[0], src[1], src[2], mu[ip], k0, P, &st);
        for (int c = 0; c < st.n; c++)
            for (int d = 0; d < 3; d++) gb[d] += st.wgt[c] * gradphi[st.node[c] * 3 + d];
        orc_rhs(p, src, mu[ip], gb, F);
        double h = (stage == 1) ? 0.5 * p->dt : p->dt;
        for (int d = 0; d < 5; d++) x[d] = xa[d] + h * F[d];
        nrefl += orc_post(p, x);
        double* const* dst = (stage == 1) ? Xb : Xa;
        for (int d = 0; d < 5; d++) dst[d][ip] = x[d];
    }
    geom_free(&g);
    return nrefl;
}

/* Diagnostic (fig:convergence P:718-729): delta-f ion heat
 * flux Q = sum_p w_p E_kin,p v_E,r(p), E_kin = v_par^2/2 + mu B and
 * v_E,r = -gbar_theta / (r omega0 B) with the gyro-averaged gradient of the
 * local field (U-2, U-3; v_E,r = 0 with the drift-off flag).  Pinned: phi = 0
 * or w = 0 gives 0; a field with constant g_theta gives the closed form
 * sum w E_kin (-g_theta / (r omega0 B)) (tests/test_oracle_push.py). */
double orc_heat_flux(const orc_params* p, int64_t n, const double* psi, const double* theta,
                     const double* zeta, const double* rho_par, const double* w, const double* mu,
                     int32_t k0, int32_t P, const double* gradphi) {
    orc_geom g;
    geom_build(p, &g);
    orc_stencil st;
    double q = 0.0;
    for (int64_t ip = 0; ip < n; ip++) {
        orc_build_stencil(p, &g, psi[ip], theta[ip], zeta[ip], mu[ip], k0, P, &st);
        double gt = 0.0;
        for (int c = 0; c < st.n; c++) gt += st.wgt[c] * gradphi[st.node[c] * 3 + 1];
        double r = sqrt(2.0 * psi[ip]);
        double B = orc_B(p, r, theta[ip]);
        double vpar = p->omega0 * B * rho_par[ip];
        double vEr = p->drifts ? -gt / (r * p->omega0 * B) : 0.0;
        q += w[ip] * (0.5 * vpar * vpar + mu[ip] * B) * vEr;
    }
    geom_free(&g);
    return q;
}

/* ------------------------------------------------------------------ */
/* Shift and bin (H-1, H-4)                          */
/* ------------------------------------------------------------------ */

/* H-1: destination toroidal domain of each particle: floor(kg / P) with the
 * same kg as Q-2.  Pinned against a brute-force exact-rational owner test. */
void orc_shift_dest(const orc_params* p, int64_t n, const double* zeta, int32_t P, int32_t* dest) {
    for (int64_t ip = 0; ip < n; ip++) {
        int32_t kg;
        double wz1;
        orc_plane(p, zeta[ip], &kg, &wz1);
        dest[ip] = kg / P;
    }
}

/* G-6 ("the radial domain decomposition ... each subdomain has
 * roughly the same area"): K radial windows split the
 * annulus a0 < r < a1 into equal areas, r_k = sqrt(a0^2 + (k/K)(a1^2 - a0^2)),
 * each boundary snapped to the nearest ring (floor((r_k - a0)/dr + 1/2)).
 * bound[0..K] are ring indices, bound[0] = 0, bound[K] = mpsi.
 * Pinned: class D at K = 2 splits at ring 519 with owned sum(mtheta)
 * 1,201,004 / 1,205,110 (SURVEY G-6 [computed]); exact-decimal recomputation
 * of the snapped boundaries (tests/test_oracle_radial.py). */
void orc_radial_windows(const orc_params* p, int32_t K, int32_t* bound) {
    double dr = orc_dr(p);
    bound[0] = 0;
    for (int32_t k = 1; k < K; k++) {
        double rk = sqrt(p->a0 * p->a0 + ((double)k / K) * (p->a1 * p->a1 - p->a0 * p->a0));
        int32_t b = (int32_t)floor((rk - p->a0) / dr + 0.5);
        if (b < 0) b = 0;
        if (b > p->mpsi) b = p->mpsi;
        bound[k] = b;
    }
    bound[K] = p->mpsi;
}

/* H-2 (P:244-249 radial domains; SPEC S:553 toroidal first, then radial):
 * radial owner of each particle = the window k whose boundary radii bracket
 * its gyrocentre radius r = sqrt(2 psi): r(bound[k]) <= r < r(bound[k+1]),
 * r(b) = a0 + b dr; the last window also owns r = a1.  Pinned against an
 * exact-decimal brute-force owner test (tests/test_oracle_radial.py). */
void orc_radial_dest(const orc_params* p, int64_t n, const double* psi, int32_t K, const int32_t* bound,
                     int32_t* dest) {
    double dr = orc_dr(p);
    for (int64_t ip = 0; ip < n; ip++) {
        double r = sqrt(2.0 * psi[ip]);
        int32_t d = 0;
        for (int32_t k = 1; k < K; k++)
            if (r >= p->a0 + bound[k] * dr) d = k;
        dest[ip] = d;
    }
}

/* H-4 (reading; "sorting particles based on their cell
 * association"): cell key = (igrid_i + c) * P + k where i is the gyrocenter's
 * radial cell (Q-4 formula), c = floor(frac((theta - zeta qtinv_i)/2 pi) *
 * mtheta_i) its label cell on ring i and k its local plane interval; refined
 * by nmu magnetic-moment sub-bins (DESIGN H-4): key * nmu + b, b = number of
 * thresholds -ln(1 - q/nmu), q = 1..nmu-1, that mu reaches.  nmu = 1: the
 * plain cell key (mu may be NULL). */
void orc_bin_key(const orc_params* p, int64_t n, const double* psi, const double* theta,
                 const double* zeta, const double* mu, int32_t k0, int32_t P, int32_t nmu, int64_t* key) {
    orc_geom g;
    geom_build(p, &g);
    double dr = orc_dr(p);
    for (int64_t ip = 0; ip < n; ip++) {
        double r = sqrt(2.0 * psi[ip]);
        double x = (r - p->a0) / dr;
        int32_t i = (int32_t)floor(x);
        if (i < 0) i = 0;
        if (i > p->mpsi - 1) i = p->mpsi - 1;
        double s = (theta[ip] - zeta[ip] * g.qtinv[i]) / TWO_PI;
        s = s - floor(s);
        s = s * g.mtheta[i];
        int32_t c = (int32_t)floor(s);
        if (c < 0) c = 0;
        if (c > g.mtheta[i] - 1) c = g.mtheta[i] - 1;
        int32_t kg;
        double wz1;
        orc_plane(p, zeta[ip], &kg, &wz1);
        int32_t k = kg - k0;
        if (k < 0) k = 0;
        if (k > P - 1) k = P - 1;
        int32_t b = 0;
        for (int32_t q = 1; q < nmu; q++)
            if (mu[ip] >= -log(1.0 - (double)q / nmu)) b++;
        key[ip] = ((g.igrid[i] + c) * (int64_t)P + k) * nmu + b;
    }
    geom_free(&g);
}
