/*
 * gtcp.h -- C ABI of the B200-native GTC-P hot-path library (libgtcp.so).
 *
 * Implements the data-parallel hot path of the gyrokinetic PIC time step of
 * Wang et al., "Modern Gyrokinetic Particle-In-Cell Simulation of Fusion
 * Plasmas on Top Supercomputers" (arXiv:1510.05546; "P:n" = PAPER.md line n):
 *   charge  -- 4-point gyro-averaged deposition onto the two bounding
 *              poloidal planes of the field-line-following grid,
 *   push    -- field gather + RK2 update of psi, theta, zeta, rho_par and the
 *              delta-f weight (Eqs. 2-8),
 *   shift   -- toroidal particle migration with periodic
 *              binning by cell,
 * plus the light grid kernels poisson/smooth/field.
 * Readings of points the paper leaves open are SURVEY.md §8(c) items, listed
 * in DESIGN.md §3.
 *
 * Conventions
 *  - Every call returns gtcp_status (0 = OK).  No C++ exception crosses the ABI.
 *  - Device failures (GTCP_ECUDA / GTCP_ENCCL) are sticky: every later call on
 *    the same context returns GTCP_ESTATE; gtcp_strerror() gives the message.
 *  - All device work is enqueued on the CUDA stream given to gtcp_init and is
 *    asynchronous, except calls that take or return HOST buffers
 *    (set/get_particles, set/get_grid, stats, timings, step_host), which
 *    synchronise that stream before returning.
 *  - The context owns all device memory.  The caller owns every host buffer;
 *    the library never keeps a host pointer after a call returns.
 *  - Particle attributes on the host are always fp64 SoA arrays in the
 *    canonical order of enum gtcp_attr.
 *  - Grid arrays on the host use the plane-major layout
 *      value(k, i, j) = buf[k * mgrid + igrid[i] + j],  j = 0..mtheta[i]
 *    (j = mtheta[i] duplicates j = 0, SURVEY G-2), local planes k = 0..P
 *    (plane P = first plane of the right neighbour / the seam, G-3, G-4).
 *    GRADPHI holds 3 components per node: (d/dr, d/dtheta, d/dzeta along b).
 */
#ifndef GTCP_H
#define GTCP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gtcp_ctx_s* gtcp_ctx;

typedef enum {
    GTCP_OK = 0,
    GTCP_EINVAL = 1,      /* bad pointer, size or argument                         */
    GTCP_EINVARIANT = 2,  /* parameters violate an invariant (e.g. mzetamax % ntoroidal) */
    GTCP_ENOMEM = 3,      /* device or pinned-host allocation failed               */
    GTCP_ECUDA = 4,       /* CUDA error (sticky)                                   */
    GTCP_ENCCL = 5,       /* NCCL error (sticky)                                   */
    GTCP_ECAPACITY = 6,   /* particle capacity / shift buffer overflow             */
    GTCP_ENONFINITE = 7,  /* non-finite particle state detected                    */
    GTCP_ESTATE = 8       /* call out of order, or context already failed          */
} gtcp_status;

/* Canonical particle attribute order: live state X = (psi, theta, zeta,
 * rho_par, w), magnetic moment mu, and the RK2 saved state X0 (U-7). */
enum gtcp_attr {
    GTCP_PSI = 0, GTCP_THETA, GTCP_ZETA, GTCP_RHO, GTCP_W, GTCP_MU,
    GTCP_PSI0, GTCP_THETA0, GTCP_ZETA0, GTCP_RHO0, GTCP_W0,
    GTCP_NATTR = 11
};

/* Grid selectors for gtcp_get_grid / gtcp_set_grid. */
enum gtcp_grid {
    GTCP_GRID_CHARGE = 0,   /* reduced charge density rho, (P+1) x mgrid         */
    GTCP_GRID_PHI = 1,      /* potential phi after poisson_smooth, (P+1) x mgrid */
    GTCP_GRID_GRADPHI = 2,  /* gradient triplets, (P+1) x mgrid x 3              */
    GTCP_GRID_MARKER = 3    /* marker density per ring n_m(i), mpsi+1 (Q-8)     */
};

typedef struct {
    /* grid and particle sizes (north_star gtcp_init arguments; Tab.2) */
    int32_t mpsi, mthetamax, mzetamax, micell;
    /* decomposition: ntoroidal * nradial * npartdom == nranks;
     * rank = (toroidal * nradial + radial) * npartdom + particle replica.
     * Radial domains: equal-area windows snapped to rings (G-6). */
    int32_t ntoroidal, npartdom, nradial;
    int32_t bin_mu;         /* magnetic-moment sub-bins of the bin key, 1..16 (H-4): markers of
                             * one (cell, plane) are further ordered by their mu quantile
                             * (Exp(1) quantiles) so that a warp shares gyroradii; 4 */
    int32_t precision;      /* 64: fp64 state; 32: fp32 state (class D), fp64 arithmetic */
    int32_t bin_every;      /* bin by cell every bin_every steps; 3 */
    int32_t poisson_iters;  /* fixed weighted-Jacobi sweeps (F-2)              */
    int32_t paranl;         /* velocity-space nonlinearity on      */
    int32_t drifts;         /* 1; 0 = test-only drift-off flag                 */
    int32_t track_ids;      /* carry a uint64 id per particle (parity runs)    */
    double a0, a1;          /* radial boundaries 0.1, 0.9         */
    double R0;              /* major radius / a = 2.78 (reading C-4)           */
    double omega0;          /* a / rho_i = 125 * mpsi / 90 (C-2)        */
    double q0, q2;          /* q = q0 + q2 r^2 (C-5)                    */
    double rln, rlt;        /* R0/L_n = 2.2, R0/L_T = 6.9              */
    double tau;             /* T_e / T_i = 1                                   */
    double dt;              /* 0.06 (C-3)                               */
    double jacobi_omega;    /* 1.0 (F-2)                                       */
    double w_init_amp;      /* 1e-3 initial weight amplitude (L-3)             */
    double vcut;            /* velocity cutoff 5 v_th (L-3)                    */
    double capacity_factor; /* particle-array headroom for shift arrivals      */
    uint64_t seed;          /* gtcp_load Philox key                            */
    int32_t field_f32;      /* store the gather field in fp32 with an fp64 state (experiment;
                             * precision 32 always does); 0 */
    int32_t reserved2;
} gtcp_params;

/* Per-context sizes and counters.  Host copy; filled by gtcp_info / gtcp_stats. */
typedef struct {
    int64_t mgrid;          /* poloidal nodes per plane incl. duplicates       */
    int32_t P;              /* local planes (mzetamax / ntoroidal)             */
    int32_t k0;             /* global index of local plane 0                   */
    int32_t rank_toroidal, rank_particle;
    int32_t rank_radial;    /* radial domain of this rank                        */
    int32_t ring_lo, ring_hi; /* owned gyrocentre radii [r(ring_lo), r(ring_hi)) */
    int32_t reserved1;
    int64_t n_local;        /* particles currently owned by this rank          */
    int64_t capacity;       /* particle array capacity                         */
    int32_t stage_next;     /* 1 or 2: RK2 stage the next push expects         */
    int32_t steps_done;
} gtcp_info_t;

typedef struct {
    int64_t n_local;        /* particles owned                                  */
    int64_t n_global;       /* sum over all ranks                               */
    double sum_w;           /* sum of weights over all ranks                    */
    double max_abs_w;       /* max |w| on this rank                             */
    int64_t movers_sent;    /* cumulative particles sent by shift               */
    int64_t movers_recv;    /* cumulative particles received by shift           */
    int64_t reflections;    /* cumulative radial reflections (U-8)              */
    int64_t plane_clamps;   /* cumulative charge-plane clamps (Q-2)             */
    int64_t charge_global_fallback; /* contributions outside smem tiles (last charge) */
    int32_t fx_shift;       /* fixed-point scale F of the last charge (2^-F units) */
} gtcp_stats_t;

/* Physics diagnostics of the current state (SPEC S:578-586 history record;
 * paper fig:convergence P:718-729 plots chi in gyro-Bohm units).  Host copy,
 * filled by gtcp_diag. */
typedef struct {
    double field_energy;    /* sum of phi^2 over the canonical nodes of all planes (phi of the
                             * last poisson_smooth)                                            */
    double heat_flux;       /* Q = sum_p w_p (v_par^2/2 + mu B) v_E,r(p): delta-f ion heat flux with
                             * the gather field of the last gtcp_field (U-2, U-3), all ranks       */
    double chi_gb;          /* chi_i / chi_GB = (Q / N) / |dT/dr|(0.5a) * omega0^2: the flux per
                             * marker over the temperature gradient R0/L_T / R0, in units of
                             * rho_i^2 c_s / a (qualitative; absolute values out of scope)        */
    double sum_w;           /* sum of weights over all ranks                                    */
    int64_t n_global;       /* markers over all ranks                                           */
} gtcp_diag_t;

/* Phase timers (CUDA events on the context stream), cumulative milliseconds
 * since the last gtcp_timings_reset. */
enum gtcp_phase {
    GTCP_T_CHARGE = 0,      /* deposit kernel(s)                                */
    GTCP_T_CHARGE_RED,      /* fixed-point finalize, ghost-plane merge, allreduce */
    GTCP_T_POISSON,         /* poisson_smooth                                   */
    GTCP_T_FIELD,           /* field                                            */
    GTCP_T_PUSH,            /* gather + push kernel                             */
    GTCP_T_SHIFT,           /* shift: classify, compact, exchange, backfill     */
    GTCP_T_BIN,             /* bin: key, counting sort, permutation, tiles      */
    GTCP_NPHASE
};

typedef struct {
    double ms[GTCP_NPHASE];
    int64_t calls[GTCP_NPHASE];
    int64_t launches;       /* kernels launched by the library (all phases)     */
    int64_t comm_bytes[GTCP_NPHASE]; /* bytes this rank moved between GPUs per phase,
                             * counted by the library (NCCL bus-byte convention:
                             * send/recv payload, allreduce 2(n-1)/n x size,
                             * broadcast size); 0 on one GPU                    */
} gtcp_timings_t;

/* Fill *out with the preset of size 'T','A','B','C','D' (BASELINE.json
 * configs) or 'a'..'d' (paper Tab.2 sizes) and the Cyclone physics
 * of SURVEY §8(c) C-1..C-7.  EINVAL for an unknown size or NULL. */
gtcp_status gtcp_default_params(char size, gtcp_params* out);

/* Geometry tables (G-1..G-4) for params p: mtheta[mpsi+1], igrid[mpsi+2],
 * itran[mpsi+1], qtinv[mpsi+1]; any pointer may be NULL.  Host only. */
gtcp_status gtcp_geometry(const gtcp_params* p, int32_t* mtheta, int64_t* igrid,
                          int32_t* itran, double* qtinv, int64_t* mgrid);

/* 128-byte NCCL unique id for rank 0 to broadcast (torch.distributed). */
gtcp_status gtcp_nccl_unique_id(void* out128);

/* Create a context for rank `rank` of `nranks` (nranks ==
 * ntoroidal*nradial*npartdom; toroidal domain = rank / (nradial*npartdom),
 * radial domain = (rank / npartdom) % nradial, replica = rank % npartdom).
 * nccl_id: the 128-byte id from gtcp_nccl_unique_id, NULL iff nranks == 1.
 * cuda_stream: a cudaStream_t (NULL = legacy default stream) on which all work
 * is enqueued; the current CUDA device must be set by the caller.
 * EINVARIANT if mzetamax % ntoroidal != 0 or the product != nranks. */
gtcp_status gtcp_init(const gtcp_params* p, int rank, int nranks, const void* nccl_id,
                      void* cuda_stream, gtcp_ctx* out);
/* Free the context and everything it allocated (device memory, pinned
 * buffers, communicators); NULL is a no-op. */
void gtcp_destroy(gtcp_ctx ctx);
/* Text of the last error set on this context ("null context" for NULL);
 * owned by the context, valid until the next call on it. */
const char* gtcp_strerror(gtcp_ctx ctx);
/* Sizes, ranks and state of the context into *out (host copy, no sync). */
gtcp_status gtcp_info(gtcp_ctx ctx, gtcp_info_t* out);

/* Load this rank's markers on the device (L-1..L-3 recipe, counter-based
 * Philox keyed by params.seed): micell*(mgrid-mpsi) per plane interval
 * (pinned by P:522), divided over the npartdom replicas; then the marker
 * density (Q-8) and the first bin.  Statistically identical to the host
 * generator used for parity; not bit-identical. */
gtcp_status gtcp_load(gtcp_ctx ctx);

/* Upload n particles (host fp64 SoA): attr[GTCP_PSI..GTCP_MU] (6 arrays,
 * live state + mu); id may be NULL unless track_ids.  Particles must lie in
 * this rank's toroidal (and radial) domain.  Recomputes the marker density from these
 * particles (collective over ranks) and bins.  ECAPACITY if n > capacity. */
gtcp_status gtcp_set_particles(gtcp_ctx ctx, int64_t n, const double* const* attr, const uint64_t* id);

/* Download the owned particles: *n = count; attr[0..GTCP_NATTR) may contain
 * NULL entries to skip attributes; id may be NULL.  ECAPACITY if cap < count. */
gtcp_status gtcp_get_particles(gtcp_ctx ctx, int64_t cap, int64_t* n, double* const* attr, uint64_t* id);

/* Sampled read for full-size parity: copy particles idx[0..m) (indices into
 * the current owned order, 0 <= idx < n_local) of every non-NULL attr[] to
 * the host, and their ids if id != NULL and track_ids.  EINVAL on a bad index. */
gtcp_status gtcp_sample_particles(gtcp_ctx ctx, int64_t m, const int64_t* idx, double* const* attr, uint64_t* id);

/* Hot-path phases.  gtcp_charge deposits the CURRENT live state (X before
 * stage 1, the midpoint state before stage 2) and performs the reductions
 * (Q-7): duplicate fold, ghost-plane merge with the right neighbour (seam
 * rotation at zeta = 2 pi), particle-replica allreduce. */
gtcp_status gtcp_charge(gtcp_ctx ctx);
/* Gyrokinetic Poisson equation and smoothing (§2 Eq. 14
 * and P:221 §3.1; readings F-1..F-4): the charge of the last
 * gtcp_charge (or gtcp_set_grid CHARGE) normalised by the marker density
 * (Q-8) and smoothed (F-4); the flux-surface mean removed; poisson_iters
 * weighted-Jacobi sweeps of (1 + 1/tau) phi - G(G(phi)) = dn with G the
 * 4-point gyro-average (F-1, F-2); the zonal component added from its 1-D
 * radial solve (F-3); phi smoothed again (F-4).  Result: the potential of
 * the local planes with their halo planes (gtcp_get_grid PHI), consumed by
 * gtcp_field.  Collectives: ring sums over the toroidal ring, the plane
 * split of the sweeps over a section's ranks, halo exchanges.  Errors:
 * GTCP_ECUDA, GTCP_ENCCL. */
gtcp_status gtcp_poisson_smooth(gtcp_ctx ctx);
/* Field (§3.1, reading F-5): the gradient triplet (g_r = dphi/dr at
 * the node's physical angle, g_theta = dphi/dtheta, g_par = dphi/dzeta at
 * fixed field-line label, centred differences) of the current phi on planes
 * 0..P of this rank,
 * written into the push's gather layout (interval-interleaved records,
 * DESIGN.md §5; gtcp_get_grid GRADPHI returns it plane-major).  Errors:
 * GTCP_ECUDA. */
gtcp_status gtcp_field(gtcp_ctx ctx);
/* stage 1: X0 <- X, X <- X + dt/2 F(X);  stage 2: X <- X0 + dt F(X) (U-7).
 * ESTATE if stage is not the one expected. */
gtcp_status gtcp_push(gtcp_ctx ctx, int stage);
/* Migrate particles to their owner domain (H-1 toroidal, then H-2 radial;
 * multi-hop with guard: GTCP_EINVARIANT if movers remain after ntoroidal + 1
 * passes), then bin by cell when the schedule says so (after stage 2 every
 * bin_every steps).  ECAPACITY on a send-buffer or particle-capacity overflow. */
gtcp_status gtcp_shift(gtcp_ctx ctx);
/* Force a bin (cell sort, H-4) now. */
gtcp_status gtcp_bin(gtcp_ctx ctx);
/* nsteps x [for stage in (1,2): charge, poisson_smooth, field, push(stage), shift]
 * (with gtcp_set_fused(1) a stage's push also deposits the next charge).
 * Synchronises the stream once at the end and returns GTCP_ENONFINITE if a
 * push produced a non-finite state (checked without waiting after every
 * step as well, so a long call stops within about a step of the event). */
gtcp_status gtcp_step(gtcp_ctx ctx, int nsteps);
/* End-to-end offload call: upload n particles from host buffers attr[0..6)
 * (live state + mu), run nsteps steps, download the owned particles' live
 * state AND mu (a bin or a shift inside the steps reorders them together)
 * back into the same buffers, whose capacity is cap elements each.
 * *n_out = the owned count after the steps (differs from n when a decomposed
 * run migrated particles).  ECAPACITY, with nothing downloaded, if that count
 * exceeds cap.  The tiles of the previous bin are kept: they are exact for a
 * state returned by the previous call (same order); any other order stays
 * exact through the deposit's out-of-window path, only slower.  Synchronises. */
gtcp_status gtcp_step_host(gtcp_ctx ctx, int64_t n, int64_t cap, double* const* attr, int nsteps, int64_t* n_out);

/* Download a grid (GTCP_GRID_*): CHARGE / PHI as (planes 0..P) x mgrid
 * doubles, GRADPHI as (planes 0..P) x mgrid x 3, MARKER as mpsi + 1 ring
 * densities.  ECAPACITY if cap is below the size; synchronises. */
gtcp_status gtcp_get_grid(gtcp_ctx ctx, int which, int64_t cap, double* host);
/* Prescribe a grid (tests): CHARGE (then poisson_smooth uses it), PHI (then
 * field uses it) or GRADPHI (then push gathers it). */
gtcp_status gtcp_set_grid(gtcp_ctx ctx, int which, int64_t n, const double* host);

/* Counters of the context (global particle count, sum of w, reflections,
 * clamps, fallback contributions, fixed-point scale...) into *out;
 * GTCP_ENONFINITE if a push flagged a non-finite state; synchronises. */
gtcp_status gtcp_stats(gtcp_ctx ctx, gtcp_stats_t* out);
/* Diagnostics of the current live state against the current gather field
 * (call after gtcp_field, before the push, for the fields of this stage);
 * collective over all ranks; synchronises.  EINVAL if out is NULL. */
gtcp_status gtcp_diag(gtcp_ctx ctx, gtcp_diag_t* out);
/* Accumulated per-phase CUDA-event times and library-counted inter-GPU bytes
 * since the last reset (phases timed only while gtcp_set_timing is on). */
gtcp_status gtcp_timings(gtcp_ctx ctx, gtcp_timings_t* out);
gtcp_status gtcp_timings_reset(gtcp_ctx ctx);
/* Enable (1) / disable (0) per-phase CUDA-event timing (default off). */
gtcp_status gtcp_set_timing(gtcp_ctx ctx, int enable);

/* Test-only transport (SURVEY §4 "loopback"): nranks contexts of ONE process
 * on ONE device, one host thread per context, share a hub instead of NCCL.
 * Every exchange of the decomposed step (ghost-plane charge merge, section
 * and ring allreduces, potential halos, Poisson plane broadcasts, shift
 * counts and payload) then runs as one cudaMemcpyAsync per message between
 * the contexts' device buffers (allreduce: one small kernel summing the
 * members' staged buffers in member order), so the decomposition can be
 * parity-checked on a single GPU.  gtcp_loopback_create returns the hub
 * (EINVAL for nranks outside 1..16); gtcp_init_loopback is gtcp_init with the
 * hub in place of the NCCL id (same rank layout and invariants; the stream
 * should be a distinct non-blocking stream per context).  The hub must
 * outlive every context created on it; gtcp_loopback_destroy frees it. */
gtcp_status gtcp_loopback_create(int nranks, void** hub);
void gtcp_loopback_destroy(void* hub);
gtcp_status gtcp_init_loopback(const gtcp_params* p, int rank, int nranks, void* hub, void* cuda_stream,
                               gtcp_ctx* out);

/* Test / ablation hooks: select the charge kernel -- 0 = smem-tiled (the
 * product), 1 = direct global fixed-point atomics (the paper's Kepler-style
 * cooperative atomics), 2 = the paper's Fermi update binning
 * (P:336-353): the 4 gyro-points of every particle binned by their own cell at
 * every charge, one thread per super-cell, even/odd twin shared-memory copies.
 * All three give the bitwise-identical fixed-point grid. */
gtcp_status gtcp_set_charge_mode(gtcp_ctx ctx, int mode);
/* Ablation hook: 0 = fused gather + push (default); 1 = the
 * paper's Xeon Phi loop fission: a gather kernel writes the
 * gyro-averaged gradient (3 doubles per particle) to HBM, an update kernel
 * reads it (fp64 state only; other precisions stay fused).  Same results. */
gtcp_status gtcp_set_push_mode(gtcp_ctx ctx, int mode);
/* SURVEY §8(f) #1, fused stage pipeline: 1 = gtcp_step pushes each RK2 stage
 * and deposits the NEXT stage's charge from the new state in one kernel over
 * the bin's tiles (no re-read of the state for the charge, one launch less);
 * 0 = separate push and charge (default).  One rank, tiled charge, fp64 state
 * only (GTCP_EINVAL otherwise); applies inside gtcp_step, the first charge of
 * each gtcp_step call after gtcp_load / set_particles / step_host / set_grid
 * is deposited separately.  The fused charge uses one bit less fixed-point
 * scale (the new max|w| is not known before it is deposited); results match
 * the unfused step within the fixed-point rounding (2^-31 of max|w|/4 per
 * contribution). */
gtcp_status gtcp_set_fused(gtcp_ctx ctx, int on);

#ifdef __cplusplus
}
#endif
#endif /* GTCP_H */
