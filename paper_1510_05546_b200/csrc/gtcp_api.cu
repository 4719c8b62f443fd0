// gtcp_api.cu -- host orchestration behind the C ABI of include/gtcp.h.
//
// One context per rank (one process per GPU).  All device work is enqueued on
// the context stream; NCCL runs on the same stream, so ordering is implicit.
// Geometry (G-1..G-4) is rebuilt here on the host from the paper's rules
// (product-side code; the oracle has its own independent implementation).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gtcp_internal.cuh"

#include <nvtx3/nvToolsExt.h>

using namespace gtcp;

struct gtcp_ctx_s {
    gtcp_params prm;
    int rank, nranks, rank_t, rank_p, rank_r;
    std::vector<int> rad_ring;    // radial window boundaries (ring indices), nradial+1
    Comm sect, rad;  // same toroidal domain; same (toroidal, replica)
    cudaStream_t st;
    int device;
    Comm world, tor;  // all ranks; toroidal ring (same radial window and replica)
    LoopHub* hub = nullptr;  // loopback transport (test-only), not owned
    long long comm_bytes[GTCP_NPHASE] = {};  // bytes moved by this rank per phase (NCCL bus-byte convention)
    int cur_phase = GTCP_T_CHARGE_RED;       // phase the comm calls are charged to
    std::string err;
    gtcp_status sticky = GTCP_OK;
    // geometry (host + device)
    std::vector<int> mtheta, igrid, itran;
    std::vector<double> qtinv;
    int mgrid = 0, P = 0, k0 = 0;
    int *d_mtheta = nullptr, *d_igrid = nullptr, *d_itran = nullptr;
    unsigned short* d_node_ring = nullptr;
    PoisRing* d_pois = nullptr;  // F-1 per-ring constants (Poisson operator)
    double* d_qtinv = nullptr;
    Geo geo;
    // particles
    long long n = 0, cap = 0;
    double* bufA[5] = {};
    double* bufB[5] = {};
    double* live[5] = {};
    double* saved[5] = {};
    double* mu = nullptr;
    double* scratch = nullptr;
    unsigned long long* id = nullptr;
    unsigned long long* id_scratch = nullptr;
    int stage_next = 1;
    int steps_done = 0;
    // binning
    long long nkeys = 0;
    unsigned *key = nullptr, *rankbuf = nullptr, *inv = nullptr, *count = nullptr, *offset = nullptr,
             *scan_tmp = nullptr;
    Tile* tiles = nullptr;
    int max_tiles = 0;
    int* tile_span = nullptr;  // per ring: widest cell span whose window fits smem; then per-ring tile counts
    long long n_binned = 0;  // particles [0, n_binned) are covered by tiles
    int tile_max = 16384;  // <= 16384: bounds the smem limb sums (gtcp_kernels.cu smem_add)
    // grids
    long long* fx = nullptr;   // (P+1) * mgrid fixed-point charge
    double *rhoH = nullptr, *dnH = nullptr, *tmpH = nullptr, *phiH = nullptr;
    double *rhs = nullptr, *jphi = nullptr, *g1 = nullptr, *g2 = nullptr;
    double* gfield = nullptr;  // P * gstride * 6 (interval-interleaved gather layout)
    double* nm = nullptr;      // mpsi+1 marker density
    double* ringsum = nullptr; // mpsi+1
    double* phi00 = nullptr;   // 5 * (mpsi+1)
    double* halo_buf = nullptr;  // 3 * mgrid receive buffer
    long long* fx_recv = nullptr;  // mgrid
    DevCounters* dc = nullptr;
    DevCounters* h_dc = nullptr;  // pinned host mirror
    int* h_nonfinite = nullptr;   // pinned mirror of dc->nonfinite, refreshed after every push
    double* d_scalar = nullptr;   // small device scratch (sums)
    double* d_partial = nullptr;  // 1024 partial sums
    double* h_scalar = nullptr;   // pinned
    // shift buffers
    long long shift_cap = 0;
    double* sendL[12] = {};
    double* sendR[12] = {};
    double* recvL[12] = {};
    double* recvR[12] = {};
    unsigned long long *sidL = nullptr, *sidR = nullptr, *ridL = nullptr, *ridR = nullptr;
    unsigned char* cls = nullptr;
    unsigned* bcount = nullptr;  // per-block counts and offsets (8 arrays of shift_blocks+1)
    unsigned* holes = nullptr;   // hole positions, shift_cap
    unsigned* fills = nullptr;   // filler positions, shift_cap
    unsigned* midx = nullptr;    // mover positions (left list, right list), 2 shift_cap
    long long* d_nkeep = nullptr;
    long long* d_counts = nullptr;  // [myL, myR, fromRight, fromLeft, mine, total]
    long long* h_counts = nullptr;  // pinned mirror
    int shift_blocks = 0;
    bool cls_ready = false;  // cls + per-chunk counts of the toroidal shift were produced by the push
    long long movers_sent = 0, movers_recv = 0;
    // charge config
    int charge_mode = 0;
    int push_mode = 0;          // 1: loop-fission ablation of the push
    int fused = 0;              // gtcp_set_fused: push + next-stage deposit in one kernel
    int fused_ctas = 0;
    int fx_pending = 0;         // RK2 stage whose charge the last fused push already deposited into fx (0: none)
    // charge mode 2 (update-binning ablation): point records and segments
    unsigned *pkey = nullptr, *prank = nullptr, *prec = nullptr;
    int4* psegs = nullptr;
    int npsegs = 0;
    double* g3 = nullptr;       // its gbar arrays (3 x cap), allocated on first use
    int dep_ctas = 0, dep_cap_nodes = 0, dep_nb = 3;
    size_t dep_smem = 0;
    // timing
    bool timing = false;
    struct Pending { int phase; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    double t_ms[GTCP_NPHASE] = {};
    long long t_calls[GTCP_NPHASE] = {};
    long long launches0 = 0;
};

// ----------------------------------------------------------------------------
// error helpers
// ----------------------------------------------------------------------------
static gtcp_status set_err(gtcp_ctx c, gtcp_status s, const std::string& msg) {
    if (c) {
        c->err = msg;
        if (s == GTCP_ECUDA || s == GTCP_ENCCL) c->sticky = s;
    }
    return s;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (call);                                                                   \
        if (_e != cudaSuccess)                                                                     \
            return set_err(c, GTCP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
    } while (0)
#define NC(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t _r = (call);                                                                  \
        if (_r != ncclSuccess)                                                                     \
            return set_err(c, GTCP_ENCCL, std::string(#call) + ": " + comm_error_string(_r));      \
    } while (0)
#define CHECK_CTX(c)                                                                               \
    do {                                                                                           \
        if (!(c)) return GTCP_EINVAL;                                                              \
        if ((c)->sticky != GTCP_OK) return GTCP_ESTATE;                                            \
        gtcp::g_prec32 = (c)->geo.prec32;                                                          \
    } while (0)
#define KCHECK()                                                                                   \
    do {                                                                                           \
        cudaError_t _e = cudaGetLastError();                                                       \
        if (_e != cudaSuccess) return set_err(c, GTCP_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

// ----------------------------------------------------------------------------
// timing (CUDA events on the context stream)
// ----------------------------------------------------------------------------
static cudaEvent_t get_event(gtcp_ctx c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

static void fold_pending(gtcp_ctx c) {
    for (auto& p : c->pending) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        c->t_ms[p.phase] += ms;
        c->t_calls[p.phase]++;
        c->event_pool.push_back(p.a);
        c->event_pool.push_back(p.b);
    }
    c->pending.clear();
}

// NVTX ranges name every phase on the host timeline (nsys / ncu --nvtx);
// header-only NVTX 3, a no-op unless a tool injects itself
static const char* const kPhaseName[GTCP_NPHASE] = {"gtcp charge", "gtcp charge_red", "gtcp poisson_smooth",
                                                   "gtcp field", "gtcp push", "gtcp shift", "gtcp bin"};
struct PhaseTimer {
    gtcp_ctx c;
    int phase;
    cudaEvent_t a = nullptr;
    int prev_phase;
    PhaseTimer(gtcp_ctx c_, int ph) : c(c_), phase(ph) {
        nvtxRangePushA(kPhaseName[ph]);
        prev_phase = c->cur_phase;
        c->cur_phase = ph;
        if (c->timing) {
            a = get_event(c);
            cudaEventRecord(a, c->st);
        }
    }
    ~PhaseTimer() {
        nvtxRangePop();
        c->cur_phase = prev_phase;
        if (c->timing) {
            cudaEvent_t b = get_event(c);
            cudaEventRecord(b, c->st);
            c->pending.push_back({phase, a, b});
            if (c->pending.size() > 4096) fold_pending(c);
        }
    }
};

// ----------------------------------------------------------------------------
// geometry (G-1..G-4; Tab.2) -- product-side host implementation
// ----------------------------------------------------------------------------
static long long build_geometry(const gtcp_params* p, std::vector<int>& mtheta, std::vector<int>& igrid,
                                std::vector<int>& itran, std::vector<double>& qtinv) {
    int M = p->mpsi;
    mtheta.assign(M + 1, 0);
    igrid.assign(M + 2, 0);
    itran.assign(M + 1, 0);
    qtinv.assign(M + 1, 0.0);
    double dr = (p->a1 - p->a0) / M;
    long long acc = 0;
    for (int i = 0; i <= M; i++) {
        double r = p->a0 + i * dr;
        int mt = 2 * (int)std::floor(p->mthetamax * r / (2.0 * p->a1) + 0.5);
        double q = p->q0 + p->q2 * r * r;
        mtheta[i] = mt;
        itran[i] = (int)std::floor(mt / q + 0.5);
        qtinv[i] = (double)itran[i] / (double)mt;
        igrid[i] = (int)acc;
        acc += mt + 1;
    }
    igrid[M + 1] = (int)acc;
    return acc;
}

extern "C" gtcp_status gtcp_default_params(char size, gtcp_params* out) {
    if (!out) return GTCP_EINVAL;
    int mpsi, mth, mze = 64, micell = 100;
    switch (size) {
        case 'T': mpsi = 16; mth = 64; mze = 2; micell = 10; break;
        case 'A': case 'a': mpsi = 90; mth = 640; break;
        case 'B': mpsi = 192; mth = 1408; break;
        case 'C': mpsi = 384; mth = 2816; break;
        case 'D': mpsi = 768; mth = 5632; break;
        case 'b': mpsi = 180; mth = 1280; break;
        case 'c': mpsi = 360; mth = 2560; break;
        case 'd': mpsi = 720; mth = 5120; break;
        default: return GTCP_EINVAL;
    }
    gtcp_params p;
    memset(&p, 0, sizeof(p));
    p.mpsi = mpsi; p.mthetamax = mth; p.mzetamax = mze; p.micell = micell;
    p.ntoroidal = 1; p.npartdom = 1; p.nradial = 1;
    p.precision = 64; p.bin_every = 3; p.bin_mu = 4; p.poisson_iters = 20; p.paranl = 1; p.drifts = 1; p.track_ids = 0;
    p.a0 = 0.1; p.a1 = 0.9; p.R0 = 2.78; p.omega0 = 125.0 * mpsi / 90.0;
    p.q0 = 0.854; p.q2 = 2.184; p.rln = 2.2; p.rlt = 6.9; p.tau = 1.0; p.dt = 0.06;
    p.jacobi_omega = 1.0; p.w_init_amp = 1e-3; p.vcut = 5.0; p.capacity_factor = 1.0;
    p.seed = 2;
    *out = p;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_geometry(const gtcp_params* p, int32_t* mtheta, int64_t* igrid, int32_t* itran,
                                     double* qtinv, int64_t* mgrid) {
    if (!p || p->mpsi < 2 || p->mthetamax < 4) return GTCP_EINVAL;
    std::vector<int> mt, ig, it;
    std::vector<double> qt;
    long long mg = build_geometry(p, mt, ig, it, qt);
    for (int i = 0; i <= p->mpsi; i++) {
        if (mtheta) mtheta[i] = mt[i];
        if (itran) itran[i] = it[i];
        if (qtinv) qtinv[i] = qt[i];
    }
    if (igrid)
        for (int i = 0; i <= p->mpsi + 1; i++) igrid[i] = ig[i];
    if (mgrid) *mgrid = mg;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_nccl_unique_id(void* out128) {
    if (!out128) return GTCP_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return GTCP_ENCCL;
    memcpy(out128, &id, sizeof(id));
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// init / destroy
// ----------------------------------------------------------------------------
template <class T>
static cudaError_t dalloc(T** p, size_t count) {
    return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

static gtcp_status init_ctx(const gtcp_params* p, int rank, int nranks, const void* nccl_id, LoopHub* hub,
                            void* cuda_stream, gtcp_ctx* out) {
    if (!p || !out || nranks < 1 || rank < 0 || rank >= nranks) return GTCP_EINVAL;
    if (p->precision != 64 && p->precision != 32) return GTCP_EINVAL;
    if (p->mpsi < 2 || p->mthetamax < 4 || p->mzetamax < 2 || p->micell < 0) return GTCP_EINVAL;
    const int nrad = p->nradial < 1 ? 1 : p->nradial;
    if (p->ntoroidal < 1 || p->npartdom < 1 || nrad > 8) return GTCP_EINVAL;
    if (p->bin_mu < 1 || p->bin_mu > 16) return GTCP_EINVAL;
    if (p->mzetamax % p->ntoroidal != 0 || p->ntoroidal * nrad * p->npartdom != nranks) return GTCP_EINVARIANT;
    if (p->mzetamax / p->ntoroidal < 2) return GTCP_EINVARIANT;
    if (nranks > 1 && !nccl_id && !hub) return GTCP_EINVAL;
    if (hub && loop_hub_size(hub) != nranks) return GTCP_EINVAL;
    gtcp_ctx c = new gtcp_ctx_s();
    c->prm = *p;
    c->prm.nradial = nrad;
    c->rank = rank;
    c->nranks = nranks;
    c->rank_t = rank / (nrad * p->npartdom);
    c->rank_r = (rank / p->npartdom) % nrad;
    c->rank_p = rank % p->npartdom;
    c->st = (cudaStream_t)cuda_stream;
    cudaGetDevice(&c->device);
    *out = c;
    c->mgrid = (int)build_geometry(p, c->mtheta, c->igrid, c->itran, c->qtinv);
    c->P = p->mzetamax / p->ntoroidal;
    c->k0 = c->rank_t * c->P;
    // G-6: equal-area radial windows r_k = sqrt(a0^2 + (k/K)(a1^2 - a0^2)), snapped to the nearest ring
    c->rad_ring.assign(nrad + 1, 0);
    for (int kk = 0; kk <= nrad; kk++) {
        double rk = std::sqrt(p->a0 * p->a0 + (double)kk / nrad * (p->a1 * p->a1 - p->a0 * p->a0));
        int b = (int)std::floor((rk - p->a0) / ((p->a1 - p->a0) / p->mpsi) + 0.5);
        c->rad_ring[kk] = std::min(std::max(b, 0), p->mpsi);
    }
    c->rad_ring[0] = 0;
    c->rad_ring[nrad] = p->mpsi;
    const int M = p->mpsi, mg = c->mgrid, P = c->P;
    CU(dalloc(&c->d_mtheta, M + 1));
    CU(dalloc(&c->d_igrid, M + 2));
    CU(dalloc(&c->d_itran, M + 1));
    CU(dalloc(&c->d_qtinv, M + 1));
    CU(cudaMemcpy(c->d_mtheta, c->mtheta.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_igrid, c->igrid.data(), sizeof(int) * (M + 2), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_itran, c->itran.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_qtinv, c->qtinv.data(), sizeof(double) * (M + 1), cudaMemcpyHostToDevice));
    {
        std::vector<unsigned short> nr(mg);
        for (int i = 0; i <= M; i++)
            for (int j = c->igrid[i]; j < c->igrid[i + 1]; j++) nr[j] = (unsigned short)i;
        CU(dalloc(&c->d_node_ring, mg));
        CU(cudaMemcpy(c->d_node_ring, nr.data(), sizeof(unsigned short) * mg, cudaMemcpyHostToDevice));
    }
    Geo& g = c->geo;
    g.mpsi = M; g.mzetamax = p->mzetamax; g.P = P; g.k0 = c->k0; g.ntor = p->ntoroidal; g.rank_t = c->rank_t;
    g.mgrid = mg; g.paranl = p->paranl; g.drifts = p->drifts;
    // gather-field interval stride: 3 (mod 8) nodes.  A 16-byte load of a
    // quarter-warp costs one L1 wavefront per distinct line on each of the 8
    // 16-byte chunk positions (tools/microbench/ldg256.cu); records are 48 B
    // (3 chunks), so lanes at the same label in intervals k and k + d collide
    // when 3 d gstride = 0 (mod 8).  3 mod 8 keeps d = 1, 2 apart (mgrid itself
    // is 1 mod 8 at class A: neighbouring labels across an interval collided).
    g.gstride = mg + ((3 - mg % 8) + 8) % 8;
    if (const char* e = getenv("GTCP_GSTRIDE_RES")) {  // experiments: residue mod 8, or -1 for mgrid
        const int r = atoi(e);
        g.gstride = r < 0 ? mg : mg + ((r - mg % 8) % 8 + 8) % 8;
    }
    g.prec32 = (p->precision == 32);
    g.f32field = g.prec32 || p->field_f32 != 0;
    gtcp::g_prec32 = g.prec32;
    const size_t es = g.prec32 ? sizeof(float) : sizeof(double);  // particle element size
    g.a0 = p->a0; g.a1 = p->a1; g.dr = (p->a1 - p->a0) / M; g.inv_dr = 1.0 / g.dr;
    g.R0 = p->R0; g.inv_R0 = 1.0 / p->R0; g.omega0 = p->omega0; g.q0 = p->q0; g.q2 = p->q2;
    g.rln = p->rln; g.rlt = p->rlt; g.tau = p->tau; g.dt = p->dt;
    g.cz = p->mzetamax / GTCP_TWO_PI;
    g.psi_lo = 0.5 * g.a0 * g.a0 * (1.0 + 1e-12);
    g.nmu = p->bin_mu;  // H-4 mu sub-bins: thresholds at the Exp(1) quantiles b / nmu
    for (int b = 1; b < g.nmu; b++) g.mu_thr[b - 1] = -std::log(1.0 - (double)b / g.nmu);
    g.psi_hi = 0.5 * g.a1 * g.a1 * (1.0 - 1e-12);
    g.dzeta = GTCP_TWO_PI / p->mzetamax;
    g.rhoG = std::sqrt(2.0) / p->omega0;
    // deposit tile windows: a label-drift margin of 1 cell since the bin and a
    // radial band for gyroradii up to 3 thermal radii (~1 % of the markers, with
    // v_perp > 3 v_th, redo some contributions through L2); measured best at A
    // against drift 0.5 and bands of 3.5 and 4
    g.drift_cells = 1.0;
    g.rho_cut_th = 3.0;
    if (const char* e = getenv("GTCP_DRIFT_CELLS")) g.drift_cells = std::max(0.0, atof(e));  // experiments
    if (const char* e = getenv("GTCP_RHO_CUT")) g.rho_cut_th = std::max(1.0, atof(e));       // experiments
    g.inv_omega0 = 1.0 / p->omega0;
    g.inv_omega0_R0 = 1.0 / (p->omega0 * p->R0);
    g.nrad = nrad;
    g.rank_r = c->rank_r;
    for (int b = 0; b < 9; b++) g.rbound[b] = p->a1 + 1.0;
    for (int b = 0; b <= nrad; b++) g.rbound[b] = p->a0 + c->rad_ring[b] * g.dr;
    for (int b = 0; b < 9; b++) g.rbound2[b] = g.rbound[b] * g.rbound[b];
    g.mtheta = c->d_mtheta; g.igrid = c->d_igrid; g.itran = c->d_itran; g.qtinv = c->d_qtinv;
    g.node_ring = c->d_node_ring;
    {
        // F-1 per-ring constants, same point definitions as the oracle's operator:
        // theta-points (r_i, theta +- rhoG/r_i), radial points (r_i +- rhoG, theta)
        std::vector<PoisRing> pr(M + 1);
        for (int i = 0; i <= M; i++) {
            PoisRing& R = pr[i];
            const double r = g.a0 + i * g.dr;
            const int mt = c->mtheta[i];
            R.mt = mt;
            R.ig = c->igrid[i];
            R.dlab = g.rhoG / r * mt / GTCP_TWO_PI;
            for (int sg = 0; sg < 2; sg++) {
                double rs = sg == 0 ? r + g.rhoG : r - g.rhoG;
                rs = std::min(std::max(rs, g.a0), g.a1);
                const double x = (rs - g.a0) * g.inv_dr;
                const int m = std::min(std::max((int)std::floor(x), 0), M - 1);
                R.m[sg] = m;
                R.wp[sg] = x - m;
                for (int q = 0; q < 2; q++) {
                    const int mm = m + q, t = 2 * sg + q;
                    R.mtm[t] = c->mtheta[mm];
                    R.igm[t] = c->igrid[mm];
                    R.ratio[t] = (double)c->mtheta[mm] / mt;
                    R.cz[t] = (c->qtinv[i] - c->qtinv[mm]) * c->mtheta[mm] / GTCP_TWO_PI;
                    R.inv_mt[t] = 1.0 / c->mtheta[mm];
                }
            }
        }
        CU(dalloc(&c->d_pois, M + 1));
        CU(cudaMemcpy(c->d_pois, pr.data(), sizeof(PoisRing) * (M + 1), cudaMemcpyHostToDevice));
    }
    // particle capacity: the loaded count plus headroom for shift imbalance
    long long per_plane = (long long)p->micell * (mg - M);
    long long n_load = per_plane * P / p->npartdom;
    if (nrad > 1) {
        // marker density ~ r (1 + r^2 / (2 R0^2)) (theta-average of J): share of this window
        auto Mr = [&](double r) { return 0.5 * r * r + r * r * r * r / (8.0 * p->R0 * p->R0); };
        double tot = Mr(p->a1) - Mr(p->a0);
        double mx = 0.0;
        for (int kk = 0; kk < nrad; kk++)
            mx = std::max(mx, (Mr(p->a0 + c->rad_ring[kk + 1] * g.dr) - Mr(p->a0 + c->rad_ring[kk] * g.dr)) / tot);
        n_load = (long long)std::ceil(per_plane * P * mx / p->npartdom);
    }
    double headroom = nranks > 1 ? 0.10 : 0.0;
    c->cap = (long long)std::ceil(n_load * (p->capacity_factor + headroom)) + 1024;
    c->cap = (c->cap + 255) / 256 * 256;  // whole 256-particle blocks (and 16-byte aligned class-byte loads)
    // particle arrays hold `es`-byte reals (fp64 or fp32 state); typed double* for plumbing only
    auto palloc = [&](double** ptr, long long count) { return cudaMalloc((void**)ptr, std::max<long long>(count, 1) * es); };
    for (int d = 0; d < 5; d++) {
        CU(palloc(&c->bufA[d], c->cap));
        CU(palloc(&c->bufB[d], c->cap));
        c->live[d] = c->bufA[d];
        c->saved[d] = c->bufB[d];
    }
    CU(palloc(&c->mu, c->cap));
    CU(palloc(&c->scratch, c->cap));
    if (p->track_ids) {
        CU(dalloc(&c->id, c->cap));
        CU(dalloc(&c->id_scratch, c->cap));
    }
    // binning
    c->nkeys = (long long)mg * P * c->geo.nmu;
    CU(dalloc(&c->key, c->cap));
    CU(dalloc(&c->rankbuf, c->cap));
    CU(dalloc(&c->inv, c->cap));
    CU(dalloc(&c->count, c->nkeys + 1));
    CU(dalloc(&c->offset, c->nkeys + 1));
    CU(dalloc(&c->scan_tmp, (c->nkeys + 4095) / 4096 + 1));
    c->max_tiles = (int)std::min<long long>((long long)mg + c->cap / 1024 + M + 16, 1LL << 30);
    CU(dalloc(&c->tiles, c->max_tiles));
    CU(dalloc(&c->tile_span, 2LL * M));  // [M] max label span per ring, [M] tiles per ring
    // grids
    long long HP = (long long)(P + 3) * mg;
    CU(dalloc(&c->fx, (long long)(P + 1) * mg));
    CU(dalloc(&c->rhoH, HP));
    CU(dalloc(&c->dnH, HP));
    CU(dalloc(&c->tmpH, HP));
    CU(dalloc(&c->phiH, HP));
    CU(cudaMemset(c->rhoH, 0, HP * sizeof(double)));
    CU(cudaMemset(c->dnH, 0, HP * sizeof(double)));
    CU(cudaMemset(c->tmpH, 0, HP * sizeof(double)));
    CU(cudaMemset(c->phiH, 0, HP * sizeof(double)));
    CU(dalloc(&c->rhs, (long long)P * mg));
    CU(dalloc(&c->jphi, (long long)P * mg));
    CU(dalloc(&c->g1, (long long)P * mg));
    CU(dalloc(&c->g2, (long long)P * mg));
    CU(dalloc(&c->gfield, (long long)P * c->geo.gstride * 6));
    CU(cudaMemset(c->gfield, 0, (long long)P * c->geo.gstride * 6 * sizeof(double)));
    CU(dalloc(&c->nm, M + 1));
    CU(dalloc(&c->ringsum, M + 1));
    CU(dalloc(&c->phi00, 5 * (M + 1)));
    CU(dalloc(&c->halo_buf, 3LL * mg));
    CU(dalloc(&c->fx_recv, mg));
    CU(dalloc(&c->dc, 1));
    CU(cudaMemset(c->dc, 0, sizeof(DevCounters)));
    CU(cudaMallocHost((void**)&c->h_dc, sizeof(DevCounters)));
    CU(cudaMallocHost((void**)&c->h_nonfinite, sizeof(int)));
    c->h_nonfinite[0] = 0;
    CU(dalloc(&c->d_scalar, 32));
    CU(dalloc(&c->d_partial, 1024));
    CU(cudaMallocHost((void**)&c->h_scalar, 32 * sizeof(double)));
    {
        std::vector<double> ones(M + 1, 1.0);
        CU(cudaMemcpy(c->nm, ones.data(), sizeof(double) * (M + 1), cudaMemcpyHostToDevice));
    }
    // tiled deposit launch configuration: 3 CTAs of 256 threads per SM
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    // dynamic smem: 2 limb arrays of kDepCap+1 words, row table [(P+1) x 17], column -> ring bytes
    {
        const char* e = getenv("GTCP_DEPOSIT_CTAS");  // 3 (default) or 2 CTAs per SM
        c->dep_nb = (e && atoi(e) == 2) ? 2 : 3;
    }
    {
        // tiles of ~2.5-5 label cells: 16384 markers with many local planes,
        // 8192 with few (measured: A -4 % charge with 16384; B on 4 GPUs, P = 16,
        // 2 % faster with 8192)
        c->tile_max = P >= 32 ? 16384 : 8192;
        const char* e = getenv("GTCP_TILE_MAX");  // experiments
        if (e) c->tile_max = std::max(256, std::min(16384, atoi(e)));
    }
    c->dep_cap_nodes = gtcp::deposit_cap_nodes(c->dep_nb);
    c->dep_smem = gtcp::deposit_tiled_smem(P, c->dep_nb);
    if (c->dep_smem > (size_t)smem_optin) c->dep_cap_nodes = 0;
    c->dep_ctas = nsm * c->dep_nb;
    if (P + 1 > 80 || c->dep_cap_nodes < 1024 || p->mthetamax >= 8192) {  // packed rows: labels < 2^13
        c->charge_mode = 1;
    } else {
        CU(configure_deposit_tiled(c->dep_smem, c->dep_nb));
        int per_sm = gtcp::deposit_tiled_ctas_per_sm(c->dep_smem, c->dep_nb);
        if (per_sm < 1) c->charge_mode = 1;
        else c->dep_ctas = nsm * std::min(per_sm, c->dep_nb);
    }
    gtcp::launch_tile_spans(c->geo, c->dep_cap_nodes, c->tile_span, c->st);
    c->launches0 = gtcp::g_launches;
    // NCCL communicators
    if (nranks > 1) {
        if (hub) {
            c->hub = hub;
            c->world = loop_world(hub, rank);
        } else {
            ncclUniqueId uid;
            memcpy(&uid, nccl_id, sizeof(uid));
            NC(comm_init_nccl(&c->world, nranks, uid, rank));
        }
        // toroidal ring: same (radial, replica); section: same toroidal domain;
        // radial line: same (toroidal, replica)
        NC(comm_split(c->world, c->rank_r * p->npartdom + c->rank_p, c->rank_t, &c->tor));
        NC(comm_split(c->world, c->rank_t, c->rank_r * p->npartdom + c->rank_p, &c->sect));
        NC(comm_split(c->world, c->rank_t * p->npartdom + c->rank_p, c->rank_r, &c->rad));
    }
    // shift buffers (movers per stage ~1% at 8 domains; allocate generously)
    if (p->ntoroidal > 1 || nrad > 1) {
        c->shift_cap = std::max<long long>(1 << 16, (long long)(0.08 * c->cap));
        for (int d = 0; d < 11; d++) {
            CU(palloc(&c->sendL[d], c->shift_cap));
            CU(palloc(&c->sendR[d], c->shift_cap));
        }
        if (p->track_ids) {
            CU(dalloc(&c->sidL, c->shift_cap));
            CU(dalloc(&c->sidR, c->shift_cap));
        }
        CU(dalloc(&c->cls, c->cap));
        c->shift_blocks = (int)((c->cap + 1023) / 1024);
        CU(dalloc(&c->bcount, 8LL * (c->shift_blocks + 1)));
        CU(dalloc(&c->holes, 2 * c->shift_cap));
        CU(dalloc(&c->fills, 2 * c->shift_cap));
        CU(dalloc(&c->midx, 2 * c->shift_cap));
        CU(dalloc(&c->d_nkeep, 1));
        CU(dalloc(&c->d_counts, 8));
        CU(cudaMallocHost((void**)&c->h_counts, 8 * sizeof(long long)));
        // scan scratch must cover the per-block count arrays too
        if ((c->shift_blocks + 4095) / 4096 + 1 > (c->nkeys + 4095) / 4096 + 1) {
            cudaFree(c->scan_tmp);
            CU(dalloc(&c->scan_tmp, (c->shift_blocks + 4095) / 4096 + 1));
        }
    }
    CU(cudaDeviceSynchronize());
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_init(const gtcp_params* p, int rank, int nranks, const void* nccl_id,
                                 void* cuda_stream, gtcp_ctx* out) {
    return init_ctx(p, rank, nranks, nccl_id, nullptr, cuda_stream, out);
}

extern "C" gtcp_status gtcp_loopback_create(int nranks, void** hub) {
    if (!hub || nranks < 1 || nranks > 16) return GTCP_EINVAL;
    *hub = loop_hub_create(nranks);
    return GTCP_OK;
}

extern "C" void gtcp_loopback_destroy(void* hub) { loop_hub_destroy(static_cast<LoopHub*>(hub)); }

extern "C" gtcp_status gtcp_init_loopback(const gtcp_params* p, int rank, int nranks, void* hub, void* cuda_stream,
                                          gtcp_ctx* out) {
    if (!hub) return GTCP_EINVAL;
    return init_ctx(p, rank, nranks, nullptr, static_cast<LoopHub*>(hub), cuda_stream, out);
}

extern "C" void gtcp_destroy(gtcp_ctx c) {
    if (!c) return;
    cudaStreamSynchronize(c->st);
    fold_pending(c);
    for (auto e : c->event_pool) cudaEventDestroy(e);
    auto F = [](void* p) { if (p) cudaFree(p); };
    // the live/saved/mu/scratch pointers are always a permutation of the original allocations
    for (int d = 0; d < 5; d++) { F(c->live[d]); F(c->saved[d]); }
    F(c->mu); F(c->scratch); F(c->id); F(c->id_scratch);
    F(c->key); F(c->rankbuf); F(c->inv); F(c->count); F(c->offset); F(c->scan_tmp); F(c->tiles); F(c->tile_span);
    F(c->fx); F(c->rhoH); F(c->dnH); F(c->tmpH); F(c->phiH); F(c->rhs); F(c->jphi); F(c->g1); F(c->g2);
    F(c->gfield); F(c->nm); F(c->ringsum); F(c->phi00); F(c->halo_buf); F(c->fx_recv); F(c->dc); F(c->d_scalar); F(c->d_partial);
    F(c->d_mtheta); F(c->d_igrid); F(c->d_itran); F(c->d_qtinv); F(c->d_node_ring); F(c->d_pois);
    for (int d = 0; d < 12; d++) { F(c->sendL[d]); F(c->sendR[d]); F(c->recvL[d]); F(c->recvR[d]); }
    F(c->sidL); F(c->sidR); F(c->ridL); F(c->ridR); F(c->cls); F(c->bcount); F(c->holes); F(c->fills); F(c->midx); F(c->d_nkeep);
    F(c->d_counts); F(c->g3); F(c->pkey); F(c->prank); F(c->prec); F(c->psegs);
    if (c->h_counts) cudaFreeHost(c->h_counts);
    if (c->h_dc) cudaFreeHost(c->h_dc);
    if (c->h_nonfinite) cudaFreeHost(c->h_nonfinite);
    if (c->h_scalar) cudaFreeHost(c->h_scalar);
    comm_destroy(&c->sect);
    comm_destroy(&c->rad);
    comm_destroy(&c->tor);
    comm_destroy(&c->world);
    delete c;
}

extern "C" const char* gtcp_strerror(gtcp_ctx c) { return c ? c->err.c_str() : "null context"; }

extern "C" gtcp_status gtcp_info(gtcp_ctx c, gtcp_info_t* out) {
    if (!c || !out) return GTCP_EINVAL;
    out->mgrid = c->mgrid;
    out->P = c->P;
    out->k0 = c->k0;
    out->rank_toroidal = c->rank_t;
    out->rank_particle = c->rank_p;
    out->rank_radial = c->rank_r;
    out->ring_lo = c->rad_ring[c->rank_r];
    out->ring_hi = c->rad_ring[c->rank_r + 1];
    out->n_local = c->n;
    out->capacity = c->cap;
    out->stage_next = c->stage_next;
    out->steps_done = c->steps_done;
    return GTCP_OK;
}

// host fp64 <-> device particle array (fp64, or fp32 state converted on the host)
static cudaError_t upload_reals(gtcp_ctx c, double* dev, const double* host, long long n) {
    if (n <= 0) return cudaSuccess;
    if (!c->geo.prec32) return cudaMemcpyAsync(dev, host, n * sizeof(double), cudaMemcpyHostToDevice, c->st);
    std::vector<float> tmp(host, host + n);
    cudaError_t e = cudaMemcpyAsync(dev, tmp.data(), n * sizeof(float), cudaMemcpyHostToDevice, c->st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(c->st);  // tmp dies here
}

static cudaError_t download_reals(gtcp_ctx c, double* host, const double* dev, long long n) {
    if (n <= 0) return cudaSuccess;
    if (!c->geo.prec32) return cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->st);
    std::vector<float> tmp(n);
    cudaError_t e = cudaMemcpyAsync(tmp.data(), dev, n * sizeof(float), cudaMemcpyDeviceToHost, c->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
    if (e != cudaSuccess) return e;
    for (long long i = 0; i < n; i++) host[i] = tmp[i];
    return cudaSuccess;
}

// a new particle state: clear the non-finite flag on the device and its host
// mirror (after the stream drained, so no older flag copy lands afterwards)
static cudaError_t reset_nonfinite(gtcp_ctx c) {
    cudaError_t e = cudaMemsetAsync(&c->dc->nonfinite, 0, sizeof(int), c->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
    c->h_nonfinite[0] = 0;
    return e;
}

// pointer to element `count` of a particle array of the context's element size
static double* pofs(double* base, long long count) {
    return reinterpret_cast<double*>(reinterpret_cast<char*>(base) + count * (gtcp::g_prec32 ? 4 : 8));
}

static PSet live_set(gtcp_ctx c) {
    PSet s;
    for (int d = 0; d < 5; d++) { s.x[d] = c->live[d]; s.x0[d] = c->saved[d]; }
    s.mu = c->mu;
    s.id = c->id;
    return s;
}

// ----------------------------------------------------------------------------
// halo exchange of an H array (planes -1..P+1): plane -1 <- left neighbour's
// P-1; planes P, P+1 <- right neighbour's 0, 1; seam rotation at zeta = 2 pi.
// ----------------------------------------------------------------------------
static gtcp_status halo_exchange(gtcp_ctx c, double* H) {
    const Geo& g = c->geo;
    const long long mg = c->mgrid;
    const int P = c->P;
    double* pm1 = H;                       // plane -1
    double* p0 = H + mg;                   // plane 0
    double* pP = H + (long long)(P + 1) * mg;
    if (c->prm.ntoroidal == 1) {
        launch_seam_rotate(g, H + (long long)P * mg, pm1, -1, c->st);       // plane P-1 -> -1
        launch_seam_rotate(g, p0, pP, +1, c->st);                            // plane 0 -> P
        launch_seam_rotate(g, p0 + mg, pP + mg, +1, c->st);                  // plane 1 -> P+1
        KCHECK();
        return GTCP_OK;
    }
    int nt = c->prm.ntoroidal;
    int left = (c->rank_t - 1 + nt) % nt, right = (c->rank_t + 1) % nt;
    double* rb = c->halo_buf;  // [0]: from left (their P-1), [1..2]: from right (their 0, 1)
    // sends: left then right; receives: right then left -- with two domains
    // left == right and NCCL pairs same-peer messages in posting order.
    long long* acct = &c->comm_bytes[c->cur_phase];
    NC(comm_group_start());
    NC(comm_send(c->tor, p0, 2 * mg, ncclDouble, left, c->st, acct));
    NC(comm_send(c->tor, H + (long long)P * mg, mg, ncclDouble, right, c->st, acct));
    NC(comm_recv(c->tor, rb + mg, 2 * mg, ncclDouble, right, c->st, acct));
    NC(comm_recv(c->tor, rb, mg, ncclDouble, left, c->st, acct));
    NC(comm_group_end());
    if (c->rank_t == 0) launch_seam_rotate(g, rb, pm1, -1, c->st);
    else CU(cudaMemcpyAsync(pm1, rb, mg * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    if (c->rank_t == nt - 1) {
        launch_seam_rotate(g, rb + mg, pP, +1, c->st);
        launch_seam_rotate(g, rb + 2 * mg, pP + mg, +1, c->st);
    } else {
        CU(cudaMemcpyAsync(pP, rb + mg, 2 * mg * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    }
    KCHECK();
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// charge
// ----------------------------------------------------------------------------
static thread_local bool g_unit_weight = false;  // marker-density deposit (w == 1)

static gtcp_status deposit_fx(gtcp_ctx c) {
    const Geo& g = c->geo;
    PSet s = live_set(c);
    if (g_unit_weight) {
        // w == 1: point the weight array at a constant-one buffer (scratch)
        s.x[4] = c->scratch;
    }
#ifndef GTCP_NO_FX_AGREE  // (defined only in the regression-demonstration build of tools/fx_agree_demo.sh)
    if (c->nranks > 1 && !g_unit_weight) {
        // one fixed-point scale F for every rank whose grids are summed (the
        // ghost-plane merge, the section allreduce): F follows the GLOBAL
        // max|w| (8 bytes; positive doubles order like their bit patterns)
        NC(comm_allreduce(c->world, &c->dc->wmax_bits, &c->dc->wmax_bits, 1, ncclUint64, ncclMax, c->st,
                          &c->comm_bytes[c->cur_phase]));
    }
#endif
    launch_fx_scale(c->dc, c->st);
    CU(cudaMemsetAsync(c->fx, 0, (size_t)(c->P + 1) * c->mgrid * sizeof(long long), c->st));
    long long tiled_end = 0;
    if (c->charge_mode == 2) {
        launch_deposit_points(g, s, c->n, c->fx, c->dc, c->pkey, c->prank, c->prec, c->count, c->offset, c->scan_tmp,
                              c->psegs, c->npsegs, c->st);
        KCHECK();
        return GTCP_OK;
    }
    if (c->charge_mode == 0 && c->n_binned > 0) {
        launch_deposit_tiled(g, s, std::min(c->n, c->n_binned), c->tiles, c->max_tiles, c->fx, c->dc, c->dep_ctas,
                             c->dep_smem, c->dep_cap_nodes, c->dep_nb, c->st);
        tiled_end = std::min(c->n, c->n_binned);
    }
    launch_deposit_direct(g, s, tiled_end, c->n, c->fx, c->dc, c->st);
    KCHECK();
    return GTCP_OK;
}

// Q-7 reductions on the fixed-point grid, then fp64 rho (H array, planes 0..P
// plus halos).
static gtcp_status charge_reduce(gtcp_ctx c) {
    const Geo& g = c->geo;
    const long long mg = c->mgrid;
    const int P = c->P;
    if (c->prm.ntoroidal > 1) {
        int nt = c->prm.ntoroidal;
        int left = (c->rank_t - 1 + nt) % nt, right = (c->rank_t + 1) % nt;
        long long* acct = &c->comm_bytes[c->cur_phase];
        NC(comm_group_start());
        NC(comm_send(c->tor, c->fx + (long long)P * mg, mg, ncclInt64, right, c->st, acct));
        NC(comm_recv(c->tor, c->fx_recv, mg, ncclInt64, left, c->st, acct));
        NC(comm_group_end());
        launch_rotate_add_i64(g, c->fx_recv, c->fx, c->rank_t == 0 ? +1 : 0, c->st);
    }
    if (c->prm.npartdom * c->prm.nradial > 1) {
        // particle replicas and radial domains of one toroidal domain hold partial
        // charges of the same (replicated) grid: exact int64 sum
        NC(comm_allreduce(c->sect, c->fx, c->fx, (size_t)P * mg, ncclInt64, ncclSum, c->st,
                          &c->comm_bytes[c->cur_phase]));
    }
    launch_fx_to_real(g, c->fx, c->rhoH + mg, c->dc, P, c->st);
    launch_fill_dup(g, c->rhoH + mg, P, 1, c->st);
    KCHECK();
    return halo_exchange(c, c->rhoH);
}

static gtcp_status compute_marker_norm(gtcp_ctx c) {
    // deposit with w == 1 (Q-8): scratch := 1, wmax := 1
    const Geo& g = c->geo;
    {
        double v1 = 1.0;
        memcpy(&c->h_scalar[8], &v1, 8);
        CU(cudaMemcpyAsync(&c->dc->wmax_bits, &c->h_scalar[8], 8, cudaMemcpyHostToDevice, c->st));
        launch_fill_f64(c->scratch, c->n, 1.0, c->st);
    }
    g_unit_weight = true;
    gtcp_status s = deposit_fx(c);
    g_unit_weight = false;
    if (s != GTCP_OK) return s;
    s = charge_reduce(c);
    if (s != GTCP_OK) return s;
    launch_ring_sum(g, c->rhoH, c->ringsum, c->st);
    if (c->prm.ntoroidal > 1)
        NC(comm_allreduce(c->tor, c->ringsum, c->ringsum, g.mpsi + 1, ncclDouble, ncclSum, c->st,
                          &c->comm_bytes[c->cur_phase]));
    launch_ring_mean(g, c->ringsum, c->nm, c->st);
    // restore max|w| of the real weights
    CU(cudaMemsetAsync(&c->dc->wmax_bits, 0, 8, c->st));
    launch_wmax(c->live[4], c->n, c->dc, c->st);
    KCHECK();
    return GTCP_OK;
}

static gtcp_status charge_impl(gtcp_ctx c);
extern "C" gtcp_status gtcp_charge(gtcp_ctx c) {
    CHECK_CTX(c);
    c->fx_pending = 0;
    return charge_impl(c);
}

static gtcp_status charge_impl(gtcp_ctx c) {
    {
        PhaseTimer t(c, GTCP_T_CHARGE);
        gtcp_status s = deposit_fx(c);
        if (s != GTCP_OK) return s;
    }
    PhaseTimer t(c, GTCP_T_CHARGE_RED);
    return charge_reduce(c);
}

// ----------------------------------------------------------------------------
// poisson_smooth / field
// ----------------------------------------------------------------------------
// F-4 smooth of H array `f` (owned planes), result back in `f`; uses tmpH.
static gtcp_status smooth_H(gtcp_ctx c, double* f) {
    const Geo& g = c->geo;
    launch_smooth_theta(g, f, c->tmpH, c->st);
    launch_smooth_r(g, c->tmpH, f, c->st);
    KCHECK();
    gtcp_status s = halo_exchange(c, f);
    if (s != GTCP_OK) return s;
    launch_smooth_par(g, f, c->tmpH, c->st);
    CU(cudaMemcpyAsync(f + c->mgrid, c->tmpH + c->mgrid, (size_t)c->P * c->mgrid * sizeof(double),
                       cudaMemcpyDeviceToDevice, c->st));
    KCHECK();
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_poisson_smooth(gtcp_ctx c) {
    CHECK_CTX(c);
    PhaseTimer t(c, GTCP_T_POISSON);
    const Geo& g = c->geo;
    launch_normalize(g, c->rhoH + c->mgrid, c->nm, c->dnH, c->st);
    gtcp_status s = smooth_H(c, c->dnH);
    if (s != GTCP_OK) return s;
    launch_ring_sum(g, c->dnH, c->ringsum, c->st);
    if (c->prm.ntoroidal > 1)
        NC(comm_allreduce(c->tor, c->ringsum, c->ringsum, g.mpsi + 1, ncclDouble, ncclSum, c->st,
                          &c->comm_bytes[c->cur_phase]));
    launch_jacobi_init(g, c->dnH, c->ringsum, c->rhs, c->jphi, c->st);
    // the Poisson equation is 2-D per plane: the ranks of a section (radial
    // windows and particle replicas of one toroidal domain hold the same grid)
    // split the planes of the Jacobi sweeps and then share the result
    const int S = c->prm.nradial * c->prm.npartdom, s_me = c->rank_r * c->prm.npartdom + c->rank_p;
    auto kb = [&](int r) { return (int)((long long)r * c->P / S); };
    for (int it = 0; it < c->prm.poisson_iters; it++) {
        launch_gyro(g, c->d_pois, c->jphi, c->g1, kb(s_me), kb(s_me + 1) - kb(s_me), c->st);
        launch_gyro_jacobi(g, c->d_pois, c->g1, c->rhs, c->jphi, c->prm.jacobi_omega, kb(s_me),
                           kb(s_me + 1) - kb(s_me), c->st);
    }
    if (S > 1) {
        NC(comm_group_start());
        for (int r = 0; r < S; r++) {
            double* bp = c->jphi + (long long)kb(r) * c->mgrid;
            const size_t cnt = (size_t)(kb(r + 1) - kb(r)) * c->mgrid;
            if (cnt) NC(comm_bcast(c->sect, bp, bp, cnt, ncclDouble, r, c->st, &c->comm_bytes[c->cur_phase]));
        }
        NC(comm_group_end());
    }
    launch_zonal(g, c->ringsum, c->phi00, c->st);
    launch_add_zonal2(g, c->phi00, c->jphi, c->phiH, c->st);
    launch_fill_dup(g, c->phiH + c->mgrid, c->P, 1, c->st);
    KCHECK();
    s = halo_exchange(c, c->phiH);
    if (s != GTCP_OK) return s;
    s = smooth_H(c, c->phiH);
    if (s != GTCP_OK) return s;
    return halo_exchange(c, c->phiH);
}

extern "C" gtcp_status gtcp_field(gtcp_ctx c) {
    CHECK_CTX(c);
    PhaseTimer t(c, GTCP_T_FIELD);
    launch_field(c->geo, c->phiH, c->gfield, c->st);
    KCHECK();
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// push
// ----------------------------------------------------------------------------
#define CU_VOID(call) do { (void)(call); } while (0)

// push over [0, n): the binned part tile by tile (field windows staged in
// shared memory), the tail (shift arrivals beyond the last bin) plainly
static void push_range(gtcp_ctx c, double* const* src, double* const* base, double* const* out, double h) {
    // fused toroidal classification for the shift that follows
    const bool fuse = c->prm.ntoroidal > 1 && c->cls != nullptr;
    unsigned* cntL = c->bcount;
    unsigned* cntR = cntL + (c->shift_blocks + 1);
    if (fuse) {
        CU_VOID(cudaMemsetAsync(cntL, 0, 2 * (c->shift_blocks + 1) * sizeof(unsigned), c->st));
        CU_VOID(cudaMemsetAsync(c->d_counts + 5, 0, sizeof(long long), c->st));  // multi-hop flag
    }
    c->cls_ready = fuse;
    if (c->n > 0)
        launch_push3(c->geo, src, base, out, c->mu, c->n, h, c->gfield, c->dc, c->st, fuse ? c->cls : nullptr,
                     fuse ? cntL : nullptr, fuse ? cntR : nullptr, c->push_mode == 1 ? c->g3 : nullptr,
                     fuse ? c->d_counts + 5 : nullptr);
}

static gtcp_status push_impl(gtcp_ctx c, int stage);
extern "C" gtcp_status gtcp_push(gtcp_ctx c, int stage) {
    CHECK_CTX(c);
    c->fx_pending = 0;
    return push_impl(c, stage);
}

// can this stage's push also deposit the next stage's charge?
static bool fused_ok(gtcp_ctx c) {
    return c->fused && c->fused_ctas > 0 && c->nranks == 1 && c->charge_mode == 0 && c->push_mode == 0 &&
           !c->geo.prec32 && !c->geo.f32field && c->n_binned == c->n && c->n > 0;
}

// the fused stage: X <- X + h F (as push_impl) and, from the new state in
// registers, the fixed-point charge of the next RK2 stage.  Its scale F
// follows the pre-push max|w| with one bit of headroom (the new weights are
// not known before the deposit; |w| may grow within a stage).
static gtcp_status push_fused(gtcp_ctx c, int stage) {
    if (stage != c->stage_next) return set_err(c, GTCP_ESTATE, "push: unexpected RK2 stage");
    PhaseTimer t(c, GTCP_T_PUSH);
    launch_fx_scale(c->dc, c->st, 1);
    CU(cudaMemsetAsync(c->fx, 0, (size_t)(c->P + 1) * c->mgrid * sizeof(long long), c->st));
    CU(cudaMemsetAsync(&c->dc->wmax_bits, 0, 8, c->st));
    double* src[5];
    double* base[5];
    double* out[5];
    const double h = stage == 1 ? 0.5 * c->prm.dt : c->prm.dt;
    for (int d = 0; d < 5; d++) {
        src[d] = c->live[d];
        base[d] = stage == 1 ? c->live[d] : c->saved[d];
        out[d] = c->saved[d];
    }
    launch_push_deposit(c->geo, live_set(c), c->n, c->tiles, c->fx, c->dc, c->fused_ctas, c->dep_cap_nodes, src, base,
                        out, c->gfield, h, c->st);
    for (int d = 0; d < 5; d++) std::swap(c->live[d], c->saved[d]);
    c->stage_next = stage == 1 ? 2 : 1;
    c->fx_pending = c->stage_next;
    CU(cudaMemcpyAsync(c->h_nonfinite, &c->dc->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    KCHECK();
    return GTCP_OK;
}

static gtcp_status push_impl(gtcp_ctx c, int stage) {
    if (stage != c->stage_next) return set_err(c, GTCP_ESTATE, "push: unexpected RK2 stage");
    PhaseTimer t(c, GTCP_T_PUSH);
    CU(cudaMemsetAsync(&c->dc->wmax_bits, 0, 8, c->st));
    if (stage == 1) {
        // X0 <- X (buffer swap), X <- X + dt/2 F(X)
        double* src[5];
        double* out[5];
        for (int d = 0; d < 5; d++) { src[d] = c->live[d]; out[d] = c->saved[d]; }
        push_range(c, src, src, out, 0.5 * c->prm.dt);
        for (int d = 0; d < 5; d++) std::swap(c->live[d], c->saved[d]);
        c->stage_next = 2;
    } else {
        // X <- X0 + dt F(X_mid): read live (midpoint) + saved, write saved, swap
        double* src[5];
        double* base[5];
        for (int d = 0; d < 5; d++) { src[d] = c->live[d]; base[d] = c->saved[d]; }
        push_range(c, src, base, base, c->prm.dt);
        for (int d = 0; d < 5; d++) std::swap(c->live[d], c->saved[d]);
        c->stage_next = 1;
    }
    CU(cudaMemcpyAsync(c->h_nonfinite, &c->dc->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    KCHECK();
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// bin (H-4): counting sort of the live particles by cell key, tiles
// ----------------------------------------------------------------------------
static gtcp_status do_bin(gtcp_ctx c) {
    const Geo& g = c->geo;
    c->cls_ready = false;
    PSet s = live_set(c);
    // GTCP_PROFILE_BIN=1: per-kernel event times of the bin on stderr (diagnostics)
    static const bool prof = getenv("GTCP_PROFILE_BIN") != nullptr;
    cudaEvent_t ev[8];
    int nev = 0;
    auto mark = [&]() {
        if (!prof) return;
        cudaEventCreate(&ev[nev]);
        cudaEventRecord(ev[nev++], c->st);
    };
    mark();
    CU(cudaMemsetAsync(c->count, 0, (c->nkeys + 1) * sizeof(unsigned), c->st));
    launch_bin_keys(g, s, c->n, c->key, c->rankbuf, c->count, c->st);
    mark();
    launch_scan_u32(c->count, c->offset, c->nkeys, c->scan_tmp, c->st);
    mark();
    // gather form: inv[dest[p]] = p once, then every array is written coalesced
    // (scatter forms measured slower: plain 40 %, smem-staged chunks 7 %)
    launch_bin_inverse(c->key, c->rankbuf, c->offset, c->n, c->inv, c->st);
    mark();
    // permute live state, mu (and the saved state when mid-step) in one fused
    // gather pass into the other ping-pong set + spare arrays, then swap pointers
    std::vector<double**> arrs;
    for (int d = 0; d < 5; d++) arrs.push_back(&c->live[d]);
    arrs.push_back(&c->mu);
    if (c->stage_next == 2)
        for (int d = 0; d < 5; d++) arrs.push_back(&c->saved[d]);
    if (c->stage_next == 1) {
        // saved[] is dead between steps: use it (and the scratch array) as destinations
        const double* src[6];
        double* dst[6];
        for (int d = 0; d < 5; d++) { src[d] = c->live[d]; dst[d] = c->saved[d]; }
        src[5] = c->mu;
        dst[5] = c->scratch;
        launch_gather_perm_multi(src, dst, 6, c->id, c->id ? c->id_scratch : nullptr, c->inv, c->n, c->st);
        for (int d = 0; d < 5; d++) std::swap(c->live[d], c->saved[d]);
        std::swap(c->mu, c->scratch);
        if (c->id) std::swap(c->id, c->id_scratch);
    } else {
        for (double** a : arrs) {
            launch_gather_perm_f64(*a, c->scratch, c->inv, c->n, c->st);
            double* old = *a;
            *a = c->scratch;
            c->scratch = old;
        }
        if (c->id) {
            launch_gather_perm_u64(c->id, c->id_scratch, c->inv, c->n, c->st);
            std::swap(c->id, c->id_scratch);
        }
    }
    mark();
    launch_build_tiles(g, c->offset, c->tile_max, c->tiles, c->max_tiles, c->dc, c->tile_span,
                       c->tile_span + c->geo.mpsi, c->st);
    mark();
    c->n_binned = c->n;
    KCHECK();
    if (prof) {
        cudaStreamSynchronize(c->st);
        fprintf(stderr, "[bin r%d n=%lld] keys/scan/inverse/permute/tiles ms:", c->rank, c->n);
        for (int i = 1; i < nev; i++) {
            float ms;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %.3f", ms);
        }
        fprintf(stderr, "\n");
        for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    }
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_bin(gtcp_ctx c) {
    CHECK_CTX(c);
    PhaseTimer t(c, GTCP_T_BIN);
    return do_bin(c);
}

// ----------------------------------------------------------------------------
// shift (H-1..H-3): implemented in gtcp_shift_host below
// ----------------------------------------------------------------------------
gtcp_status shift_exchange(gtcp_ctx c, int dir);

extern "C" gtcp_status gtcp_shift(gtcp_ctx c) {
    CHECK_CTX(c);
    {
        PhaseTimer t(c, GTCP_T_SHIFT);
        // toroidal first, then radial (H-2)
        if (c->prm.ntoroidal > 1) {
            gtcp_status s = shift_exchange(c, 0);
            if (s != GTCP_OK) return s;
        }
        if (c->prm.nradial > 1) {
            gtcp_status s = shift_exchange(c, 1);
            if (s != GTCP_OK) return s;
        }
    }
    if (c->stage_next == 1) {  // a full step has completed
        c->steps_done++;
        if (c->prm.bin_every > 0 && c->steps_done % c->prm.bin_every == 0) {
            PhaseTimer t(c, GTCP_T_BIN);
            return do_bin(c);
        }
    }
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_step(gtcp_ctx c, int nsteps) {
    CHECK_CTX(c);
    if (c->stage_next != 1) return set_err(c, GTCP_ESTATE, "step: a stage is in progress");
    for (int s = 0; s < nsteps; s++) {
        for (int stage = 1; stage <= 2; stage++) {
            gtcp_status r;
            if (c->fx_pending == stage) {  // deposited by the previous (fused) push
                PhaseTimer t(c, GTCP_T_CHARGE_RED);
                r = charge_reduce(c);
            } else {
                r = charge_impl(c);
            }
            c->fx_pending = 0;
            if (r != GTCP_OK) return r;
            if ((r = gtcp_poisson_smooth(c)) != GTCP_OK) return r;
            if ((r = gtcp_field(c)) != GTCP_OK) return r;
            if ((r = fused_ok(c) ? push_fused(c, stage) : push_impl(c, stage)) != GTCP_OK) return r;
            if ((r = gtcp_shift(c)) != GTCP_OK) return r;
        }
        // the push raises a device flag on a non-finite state; its
        // pinned mirror is refreshed after every push, checked here without
        // waiting (a copy still in flight shows up one step later) ...
        if (c->h_nonfinite[0]) return set_err(c, GTCP_ENONFINITE, "step: non-finite particle state");
    }
    // ... and exactly once per call
    CU(cudaStreamSynchronize(c->st));
    if (c->h_nonfinite[0]) return set_err(c, GTCP_ENONFINITE, "step: non-finite particle state");
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// particles in / out
// ----------------------------------------------------------------------------
extern "C" gtcp_status gtcp_load(gtcp_ctx c) {
    CHECK_CTX(c);
    const gtcp_params& p = c->prm;
    const long long per_plane = (long long)p.micell * (c->mgrid - p.mpsi);
    const long long n_dom = per_plane * c->P;
    // radial windows take the share of the marker density r (1 + r^2/(2 R0^2))
    // (theta-average of J) between their boundary rings
    const double dr = (p.a1 - p.a0) / p.mpsi;
    auto Mr = [&](double r) { return 0.5 * r * r + r * r * r * r / (8.0 * p.R0 * p.R0); };
    const double tot = Mr(p.a1) - Mr(p.a0);
    long long n_rad = n_dom, id_rad = 0;
    if (p.nradial > 1) {
        long long acc = 0;
        for (int kk = 0; kk < p.nradial; kk++) {
            long long nk = (kk == p.nradial - 1)
                               ? n_dom - acc
                               : (long long)std::floor(n_dom * (Mr(p.a0 + c->rad_ring[kk + 1] * dr) -
                                                                 Mr(p.a0 + c->rad_ring[kk] * dr)) / tot);
            if (kk == c->rank_r) { n_rad = nk; id_rad = acc; }
            acc += nk;
        }
    }
    const long long n = n_rad / p.npartdom + (c->rank_p < n_rad % p.npartdom ? 1 : 0);
    if (n > c->cap) return set_err(c, GTCP_ECAPACITY, "load: capacity");
    const long long id0 = (long long)c->rank_t * n_dom + id_rad + (long long)c->rank_p * (n_rad / p.npartdom) +
                          std::min<long long>(c->rank_p, n_rad % p.npartdom);
    c->n = n;
    c->stage_next = 1;
    c->fx_pending = 0;
    CU(reset_nonfinite(c));
    PSet s = live_set(c);
    const double zlo = c->k0 * (GTCP_TWO_PI / p.mzetamax), zhi = (c->k0 + c->P) * (GTCP_TWO_PI / p.mzetamax);
    const double rlo = p.a0 + c->rad_ring[c->rank_r] * dr;
    const double rhi = (c->rank_r == p.nradial - 1) ? p.a1 : p.a0 + c->rad_ring[c->rank_r + 1] * dr;
    launch_load(c->geo, s, n, p.seed, id0, p.w_init_amp, p.vcut, zlo, zhi, rlo, rhi, c->st);
    KCHECK();
    gtcp_status r = do_bin(c);
    if (r != GTCP_OK) return r;
    r = compute_marker_norm(c);
    if (r != GTCP_OK) return r;
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_particles(gtcp_ctx c, int64_t n, const double* const* attr, const uint64_t* id) {
    CHECK_CTX(c);
    if (n < 0 || (n > 0 && !attr)) return set_err(c, GTCP_EINVAL, "set_particles: bad args");
    if (n > c->cap) return set_err(c, GTCP_ECAPACITY, "set_particles: n exceeds capacity");
    if (c->prm.track_ids && n > 0 && !id) return set_err(c, GTCP_EINVAL, "set_particles: ids required");
    for (int d = 0; d < 6; d++)
        if (n > 0 && !attr[d]) return set_err(c, GTCP_EINVAL, "set_particles: null attribute");
    for (int d = 0; d < 5; d++) CU(upload_reals(c, c->live[d], attr[d], n));
    CU(upload_reals(c, c->mu, attr[5], n));
    if (c->id && id) CU(cudaMemcpyAsync(c->id, id, n * sizeof(uint64_t), cudaMemcpyHostToDevice, c->st));
    c->n = n;
    c->stage_next = 1;
    c->fx_pending = 0;
    CU(reset_nonfinite(c));
    gtcp_status r = do_bin(c);
    if (r != GTCP_OK) return r;
    r = compute_marker_norm(c);
    if (r != GTCP_OK) return r;
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_get_particles(gtcp_ctx c, int64_t cap, int64_t* n, double* const* attr, uint64_t* id) {
    CHECK_CTX(c);
    if (!n) return set_err(c, GTCP_EINVAL, "get_particles: n is null");
    *n = c->n;
    if (cap < c->n) return set_err(c, GTCP_ECAPACITY, "get_particles: cap < n");
    if (attr) {
        const double* src[11];
        for (int d = 0; d < 5; d++) { src[d] = c->live[d]; src[6 + d] = c->saved[d]; }
        src[5] = c->mu;
        for (int d = 0; d < 11; d++)
            if (attr[d]) CU(download_reals(c, attr[d], src[d], c->n));
    }
    if (id && c->id) CU(cudaMemcpyAsync(id, c->id, c->n * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_sample_particles(gtcp_ctx c, int64_t m, const int64_t* idx, double* const* attr,
                                             uint64_t* id) {
    CHECK_CTX(c);
    if (m < 0 || (m > 0 && !idx)) return set_err(c, GTCP_EINVAL, "sample_particles: bad args");
    for (int64_t q = 0; q < m; q++)
        if (idx[q] < 0 || idx[q] >= c->n) return set_err(c, GTCP_EINVAL, "sample_particles: index out of range");
    if (m == 0) return GTCP_OK;
    long long* d_idx;
    double* d_out;
    CU(cudaMallocAsync((void**)&d_idx, m * sizeof(long long), c->st));
    CU(cudaMallocAsync((void**)&d_out, m * sizeof(double), c->st));
    CU(cudaMemcpyAsync(d_idx, idx, m * sizeof(long long), cudaMemcpyHostToDevice, c->st));
    const double* src[11];
    for (int d = 0; d < 5; d++) { src[d] = c->live[d]; src[6 + d] = c->saved[d]; }
    src[5] = c->mu;
    for (int d = 0; d < 11; d++) {
        if (!attr || !attr[d]) continue;
        launch_gather_f64(src[d], d_idx, m, d_out, c->st);
        CU(cudaMemcpyAsync(attr[d], d_out, m * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    }
    if (id && c->id) {
        launch_gather_u64(c->id, d_idx, m, reinterpret_cast<unsigned long long*>(d_out), c->st);
        CU(cudaMemcpyAsync(id, d_out, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->st));
    }
    CU(cudaFreeAsync(d_idx, c->st));
    CU(cudaFreeAsync(d_out, c->st));
    KCHECK();
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_step_host(gtcp_ctx c, int64_t n, int64_t cap, double* const* attr, int nsteps,
                                      int64_t* n_out) {
    CHECK_CTX(c);
    if (n < 0 || n > c->cap || cap < 0 || !attr || !n_out) return set_err(c, GTCP_EINVAL, "step_host: bad args");
    for (int d = 0; d < 6; d++)
        if (!attr[d]) return set_err(c, GTCP_EINVAL, "step_host: null attribute");
    for (int d = 0; d < 5; d++) CU(upload_reals(c, c->live[d], attr[d], n));
    CU(upload_reals(c, c->mu, attr[5], n));
    c->n = n;
    c->stage_next = 1;
    c->fx_pending = 0;  // a foreign state: the next charge is deposited afresh
    // the tiles of the last bin stay: they are exact for a state returned by
    // the previous step_host (same order); for any other order the deposit's
    // out-of-window path keeps the charge exact (slower)
    c->n_binned = std::min<long long>(c->n_binned, n);
    CU(reset_nonfinite(c));
    CU(cudaMemsetAsync(&c->dc->wmax_bits, 0, 8, c->st));
    launch_wmax(c->live[4], c->n, c->dc, c->st);
    gtcp_status r = gtcp_step(c, nsteps);
    if (r != GTCP_OK) return r;
    *n_out = c->n;
    if (c->n > cap) return set_err(c, GTCP_ECAPACITY, "step_host: owned count exceeds cap");
    // live state and mu: a bin or a shift inside the steps reorders them together
    for (int d = 0; d < 5; d++) CU(download_reals(c, attr[d], c->live[d], c->n));
    CU(download_reals(c, attr[5], c->mu, c->n));
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// grids in / out
// ----------------------------------------------------------------------------
extern "C" gtcp_status gtcp_get_grid(gtcp_ctx c, int which, int64_t cap, double* host) {
    CHECK_CTX(c);
    const long long mg = c->mgrid;
    const long long planes = c->P + 1;
    if (!host) return set_err(c, GTCP_EINVAL, "get_grid: null buffer");
    switch (which) {
        case GTCP_GRID_CHARGE:
        case GTCP_GRID_PHI: {
            if (cap < planes * mg) return set_err(c, GTCP_ECAPACITY, "get_grid: cap");
            const double* H = which == GTCP_GRID_CHARGE ? c->rhoH : c->phiH;
            CU(cudaMemcpyAsync(host, H + mg, planes * mg * sizeof(double), cudaMemcpyDeviceToHost, c->st));
            break;
        }
        case GTCP_GRID_GRADPHI: {
            if (cap < planes * mg * 3) return set_err(c, GTCP_ECAPACITY, "get_grid: cap");
            double* buf;  // stream-ordered scratch for the plane-major export
            CU(cudaMallocAsync((void**)&buf, planes * mg * 3 * sizeof(double), c->st));
            launch_gfield_export(c->geo, c->gfield, buf, c->st);
            CU(cudaMemcpyAsync(host, buf, planes * mg * 3 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
            CU(cudaFreeAsync(buf, c->st));
            break;
        }
        case GTCP_GRID_MARKER: {
            if (cap < c->prm.mpsi + 1) return set_err(c, GTCP_ECAPACITY, "get_grid: cap");
            CU(cudaMemcpyAsync(host, c->nm, (c->prm.mpsi + 1) * sizeof(double), cudaMemcpyDeviceToHost, c->st));
            break;
        }
        default: return set_err(c, GTCP_EINVAL, "get_grid: unknown grid");
    }
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_grid(gtcp_ctx c, int which, int64_t n, const double* host) {
    CHECK_CTX(c);
    c->fx_pending = 0;
    const long long mg = c->mgrid;
    const long long planes = c->P + 1;
    if (!host) return set_err(c, GTCP_EINVAL, "set_grid: null buffer");
    switch (which) {
        case GTCP_GRID_CHARGE:
        case GTCP_GRID_PHI: {
            if (n != planes * mg) return set_err(c, GTCP_EINVAL, "set_grid: size");
            double* H = which == GTCP_GRID_CHARGE ? c->rhoH : c->phiH;
            CU(cudaMemcpyAsync(H + mg, host, planes * mg * sizeof(double), cudaMemcpyHostToDevice, c->st));
            gtcp_status s = halo_exchange(c, H);
            if (s != GTCP_OK) return s;
            break;
        }
        case GTCP_GRID_GRADPHI: {
            if (n != planes * mg * 3) return set_err(c, GTCP_EINVAL, "set_grid: size");
            double* buf;
            CU(cudaMallocAsync((void**)&buf, planes * mg * 3 * sizeof(double), c->st));
            CU(cudaMemcpyAsync(buf, host, planes * mg * 3 * sizeof(double), cudaMemcpyHostToDevice, c->st));
            launch_gfield_import(c->geo, buf, c->gfield, c->st);
            CU(cudaFreeAsync(buf, c->st));
            break;
        }
        case GTCP_GRID_MARKER: {
            if (n != c->prm.mpsi + 1) return set_err(c, GTCP_EINVAL, "set_grid: size");
            CU(cudaMemcpyAsync(c->nm, host, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
            break;
        }
        default: return set_err(c, GTCP_EINVAL, "set_grid: unknown grid");
    }
    KCHECK();
    CU(cudaStreamSynchronize(c->st));
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// stats / timings
// ----------------------------------------------------------------------------
extern "C" gtcp_status gtcp_stats(gtcp_ctx c, gtcp_stats_t* out) {
    CHECK_CTX(c);
    if (!out) return GTCP_EINVAL;
    launch_sum_f64(c->live[4], c->n, c->d_scalar, c->d_partial, c->st);
    long long nl = c->n;
    CU(cudaMemcpyAsync(c->d_scalar + 1, &nl, 8, cudaMemcpyHostToDevice, c->st));
    if (c->nranks > 1) {
        NC(comm_allreduce(c->world, c->d_scalar, c->d_scalar + 2, 1, ncclDouble, ncclSum, c->st, nullptr));
        NC(comm_allreduce(c->world, c->d_scalar + 1, c->d_scalar + 3, 1, ncclInt64, ncclSum, c->st, nullptr));
    } else {
        CU(cudaMemcpyAsync(c->d_scalar + 2, c->d_scalar, 16, cudaMemcpyDeviceToDevice, c->st));
    }
    CU(cudaMemcpyAsync(c->h_scalar, c->d_scalar, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CU(cudaMemcpyAsync(c->h_dc, c->dc, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->st));
    CU(cudaStreamSynchronize(c->st));
    KCHECK();
    out->n_local = c->n;
    long long ng;
    memcpy(&ng, &c->h_scalar[3], 8);
    out->n_global = ng;
    out->sum_w = c->h_scalar[2];
    double wm;
    memcpy(&wm, &c->h_dc->wmax_bits, 8);
    out->max_abs_w = wm;
    out->movers_sent = c->movers_sent;
    out->movers_recv = c->movers_recv;
    out->reflections = c->h_dc->reflections;
    out->plane_clamps = c->h_dc->plane_clamps;
    out->charge_global_fallback = c->h_dc->fallback;
    out->fx_shift = c->h_dc->fx_shift;
    if (c->h_dc->nonfinite) return set_err(c, GTCP_ENONFINITE, "non-finite particle state");
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_diag(gtcp_ctx c, gtcp_diag_t* out) {
    CHECK_CTX(c);
    if (!out) return GTCP_EINVAL;
    // [0] heat flux, [1] field energy, [2] sum w, [3] n (as double); [4..7] reduced
    PSet s = live_set(c);
    launch_heat_flux(c->geo, s, c->n, c->gfield, c->d_scalar + 8, c->d_partial, c->st);
    launch_field_energy(c->geo, c->phiH + c->mgrid, c->d_scalar + 9, c->d_partial, c->st);
    launch_sum_f64(c->live[4], c->n, c->d_scalar + 10, c->d_partial, c->st);
    const double nl = (double)c->n;
    CU(cudaMemcpyAsync(c->d_scalar + 11, &nl, 8, cudaMemcpyHostToDevice, c->st));
    if (c->nranks > 1) {
        // particles are partitioned over all ranks; the grid over the toroidal
        // ring only (replicas and radial windows hold copies of it)
        NC(comm_allreduce(c->world, c->d_scalar + 8, c->d_scalar + 12, 1, ncclDouble, ncclSum, c->st, nullptr));
        NC(comm_allreduce(c->tor, c->d_scalar + 9, c->d_scalar + 13, 1, ncclDouble, ncclSum, c->st, nullptr));
        NC(comm_allreduce(c->world, c->d_scalar + 10, c->d_scalar + 14, 2, ncclDouble, ncclSum, c->st, nullptr));
    } else {
        CU(cudaMemcpyAsync(c->d_scalar + 12, c->d_scalar + 8, 4 * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    }
    CU(cudaMemcpyAsync(c->h_scalar + 8, c->d_scalar + 12, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    KCHECK();
    CU(cudaStreamSynchronize(c->st));
    const gtcp_params& p = c->prm;
    out->heat_flux = c->h_scalar[8];
    out->field_energy = c->h_scalar[9];
    out->sum_w = c->h_scalar[10];
    out->n_global = (int64_t)c->h_scalar[11];
    // chi_i = <Q> / |dT/dr|(0.5 a), <Q> the mean flux per marker (markers
    // sample n0), |dT/dr| = (R0/L_T)/R0 at r = 0.5 a (prof = 1, T0 = 1);
    // gyro-Bohm unit chi_GB = rho_i^2 c_s / a = 1 / omega0^2 (tau = 1)
    const double grad_t = p.rlt / p.R0;
    out->chi_gb = out->n_global > 0 ? out->heat_flux / (double)out->n_global / grad_t * p.omega0 * p.omega0 : 0.0;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_timings(gtcp_ctx c, gtcp_timings_t* out) {
    CHECK_CTX(c);
    if (!out) return GTCP_EINVAL;
    CU(cudaStreamSynchronize(c->st));
    fold_pending(c);
    for (int i = 0; i < GTCP_NPHASE; i++) {
        out->ms[i] = c->t_ms[i];
        out->calls[i] = c->t_calls[i];
    }
    out->launches = gtcp::g_launches - c->launches0;
    for (int i = 0; i < GTCP_NPHASE; i++) out->comm_bytes[i] = c->comm_bytes[i];
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_timings_reset(gtcp_ctx c) {
    CHECK_CTX(c);
    CU(cudaStreamSynchronize(c->st));
    fold_pending(c);
    for (int i = 0; i < GTCP_NPHASE; i++) { c->t_ms[i] = 0; c->t_calls[i] = 0; c->comm_bytes[i] = 0; }
    c->launches0 = gtcp::g_launches;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_timing(gtcp_ctx c, int enable) {
    CHECK_CTX(c);
    c->timing = enable != 0;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_push_mode(gtcp_ctx c, int mode) {
    CHECK_CTX(c);
    if (mode != 0 && mode != 1) return GTCP_EINVAL;
    if (mode == 1 && !c->g3) CU(dalloc(&c->g3, 3 * c->cap));
    c->push_mode = mode;
    c->fx_pending = 0;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_fused(gtcp_ctx c, int on) {
    CHECK_CTX(c);
    if (on != 0 && on != 1) return GTCP_EINVAL;
    c->fx_pending = 0;
    if (on && !c->fused_ctas) {
        if (c->nranks != 1 || c->charge_mode != 0 || c->geo.prec32 || c->geo.f32field || c->dep_cap_nodes == 0)
            return set_err(c, GTCP_EINVAL, "set_fused: one rank, tiled charge, fp64 state only");
        const int per_sm = gtcp::configure_push_deposit(c->geo);
        if (per_sm < 1) return set_err(c, GTCP_EINVAL, "set_fused: the fused kernel does not fit an SM");
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        c->fused_ctas = nsm * per_sm;
    }
    c->fused = on;
    return GTCP_OK;
}

extern "C" gtcp_status gtcp_set_charge_mode(gtcp_ctx c, int mode) {
    CHECK_CTX(c);
    c->fx_pending = 0;
    if (mode < 0 || mode > 2) return GTCP_EINVAL;
    if (mode == 2 && !c->pkey) {
        // point records (4 per particle) and the (interval, ring, 256-cell) segments
        if (4 * c->cap >= (1LL << 32)) return set_err(c, GTCP_ECAPACITY, "charge mode 2: too many points");
        CU(dalloc(&c->pkey, 4 * c->cap));
        CU(dalloc(&c->prank, 4 * c->cap));
        CU(dalloc(&c->prec, 4 * c->cap));
        std::vector<int4> sg;
        for (int k = 0; k < c->P; k++)
            for (int i = 0; i < c->prm.mpsi; i++)
                for (int c0 = 0; c0 < c->mtheta[i]; c0 += 256)
                    sg.push_back(make_int4(k, i, c0, std::min(c0 + 255, c->mtheta[i] - 1)));
        c->npsegs = (int)sg.size();
        CU(dalloc(&c->psegs, sg.size()));
        CU(cudaMemcpy(c->psegs, sg.data(), sizeof(int4) * sg.size(), cudaMemcpyHostToDevice));
    }
    c->charge_mode = mode;
    return GTCP_OK;
}

// ----------------------------------------------------------------------------
// shift over NCCL (toroidal ring neighbours), H-1..H-3
// ----------------------------------------------------------------------------
gtcp_status shift_exchange(gtcp_ctx c, int dir) {
    static const bool prof = getenv("GTCP_PROFILE_SHIFT") != nullptr;
    cudaEvent_t ev[16];
    int nev = 0;
    auto mark = [&]() {
        if (prof && nev < 16) {
            cudaEventCreate(&ev[nev]);
            cudaEventRecord(ev[nev], c->st);
            nev++;
        }
    };
    mark();
    const Geo& g = c->geo;
    // dir 0: toroidal ring (periodic); dir 1: radial line (inner = left, outer = right)
    const int nt = dir ? c->prm.nradial : c->prm.ntoroidal;
    const int me = dir ? c->rank_r : c->rank_t;
    const Comm& comm = dir ? c->rad : c->tor;
    long long* acct = &c->comm_bytes[c->cur_phase];
    const int left = dir ? (me > 0 ? me - 1 : -1) : (me - 1 + nt) % nt;
    const int right = dir ? (me < nt - 1 ? me + 1 : -1) : (me + 1) % nt;
    // movers carry the live state and mu, plus the saved RK2 state mid-step (H-3)
    const int nattr = (c->stage_next == 2) ? 11 : 6;
    long long start = 0;  // first pass scans everything, later passes only the arrivals
    bool settled = false;
    // multi-hop guard: a particle crosses at most nt domains in one
    // shift, so pass nt + 1 must find no movers
    for (int iter = 0; iter <= nt + 1; iter++) {
        double* attrs[11];
        for (int d = 0; d < 5; d++) attrs[d] = pofs(c->live[d], start);
        attrs[5] = pofs(c->mu, start);
        for (int d = 0; d < 5; d++) attrs[6 + d] = pofs(c->saved[d], start);
        unsigned long long* idp = c->id ? c->id + start : nullptr;
        const long long n = c->n - start;
        const int nb = shift_chunks(n);
        unsigned* cntL = c->bcount;
        unsigned* cntR = cntL + (c->shift_blocks + 1);
        unsigned* cntH = cntR + (c->shift_blocks + 1);
        unsigned* cntF = cntH + (c->shift_blocks + 1);
        unsigned* offL = cntF + (c->shift_blocks + 1);
        unsigned* offR = offL + (c->shift_blocks + 1);
        unsigned* offH = offR + (c->shift_blocks + 1);
        unsigned* offF = offH + (c->shift_blocks + 1);
        if (dir == 0 && iter == 0 && c->cls_ready) {
            // classification, per-chunk counts and the multi-hop flag came fused out of the push
        } else {
            CU(cudaMemsetAsync(c->d_counts + 5, 0, sizeof(long long), c->st));
            launch_shift_classify(g, attrs[2], attrs[0], dir, n, c->cls, cntL, cntR, c->d_counts + 5, c->st);
        }
        if (dir == 0) c->cls_ready = false;
        launch_scan_u32(cntL, offL, nb, c->scan_tmp, c->st);
        launch_scan_u32(cntR, offR, nb, c->scan_tmp, c->st);
        launch_shift_nkeep(n, offL + nb, offR + nb, c->d_nkeep, c->d_counts, c->st);
        if (iter == 0) mark();
        // counts: mine (left, right) out; theirs in; global mover total
        CU(cudaMemsetAsync(c->d_counts + 2, 0, 2 * sizeof(long long), c->st));
        NC(comm_group_start());
        if (left >= 0) NC(comm_send(comm, c->d_counts + 0, 1, ncclInt64, left, c->st, acct));
        if (right >= 0) NC(comm_send(comm, c->d_counts + 1, 1, ncclInt64, right, c->st, acct));
        if (right >= 0) NC(comm_recv(comm, c->d_counts + 2, 1, ncclInt64, right, c->st, acct));  // right's left-movers
        if (left >= 0) NC(comm_recv(comm, c->d_counts + 3, 1, ncclInt64, left, c->st, acct));    // left's right-movers
        NC(comm_group_end());
        launch_sum_i64_pair(c->d_counts, c->d_counts + 4, c->st);
        // [mine, multi-hop flag] summed over the ring / line -> [total, any multi-hop]
        NC(comm_allreduce(comm, c->d_counts + 4, c->d_counts + 6, 2, ncclInt64, ncclSum, c->st, acct));
        CU(cudaMemcpyAsync(c->h_counts, c->d_counts, 8 * sizeof(long long), cudaMemcpyDeviceToHost, c->st));
        if (iter == 0) mark();
        CU(cudaStreamSynchronize(c->st));
        const long long nL = c->h_counts[0], nR = c->h_counts[1], rR = c->h_counts[2], rL = c->h_counts[3];
        const long long total = c->h_counts[6];
        const bool multi_hop = c->h_counts[7] != 0;
        if (total == 0) {
            settled = true;
            break;
        }
        if (iter == nt + 1) break;
        if (nL > c->shift_cap || nR > c->shift_cap)
            return set_err(c, GTCP_ECAPACITY, "shift: send buffer overflow");
        const long long nkeep = n - nL - nR;
        if (start + nkeep + rL + rR > c->cap) return set_err(c, GTCP_ECAPACITY, "shift: particle capacity exceeded");
        if (iter == 0) mark();
        if (nL + nR > 0) {
            launch_shift_pack(attrs, nattr, idp, c->cls, n, offL, offR, c->sendL, c->sendR, c->sidL, c->sidR, c->midx, nL, nR,
                              c->st);
            if (iter == 0) mark();
            launch_shift_count_holes(c->cls, n, c->d_nkeep, cntH, cntF, c->st);
            launch_scan_u32(cntH, offH, nb, c->scan_tmp, c->st);
            launch_scan_u32(cntF, offF, nb, c->scan_tmp, c->st);
            if (iter == 0) mark();
            // holes below n_keep == movers below n_keep == fillers above it; their count is
            // min(nL + nR, ...) -- bounded by the movers, so size the copy by nL + nR (extra threads idle)
            launch_shift_backfill(attrs, nattr, idp, c->cls, n, c->d_nkeep, offH, offF, c->holes, c->fills, nL + nR, c->st);
        }
        KCHECK();
        if (iter == 0) mark();
        // payload: straight into the particle arrays behind the keepers
        NC(comm_group_start());
        for (int d = 0; d < nattr; d++) {
            const ncclDataType_t ty = g.prec32 ? ncclFloat : ncclDouble;
            if (left >= 0) NC(comm_send(comm, c->sendL[d], nL, ty, left, c->st, acct));
            if (right >= 0) NC(comm_send(comm, c->sendR[d], nR, ty, right, c->st, acct));
            if (right >= 0) NC(comm_recv(comm, pofs(attrs[d], nkeep), rR, ty, right, c->st, acct));
            if (left >= 0) NC(comm_recv(comm, pofs(attrs[d], nkeep + rR), rL, ty, left, c->st, acct));
        }
        if (idp) {
            if (left >= 0) NC(comm_send(comm, c->sidL, nL, ncclUint64, left, c->st, acct));
            if (right >= 0) NC(comm_send(comm, c->sidR, nR, ncclUint64, right, c->st, acct));
            if (right >= 0) NC(comm_recv(comm, idp + nkeep, rR, ncclUint64, right, c->st, acct));
            if (left >= 0) NC(comm_recv(comm, idp + nkeep + rR, rL, ncclUint64, left, c->st, acct));
        }
        NC(comm_group_end());
        if (iter == 0) mark();
        c->movers_sent += nL + nR;
        c->movers_recv += rL + rR;
        c->n = start + nkeep + rL + rR;
        start = start + nkeep;  // only the arrivals can still be misplaced
        // no mover went beyond a neighbouring domain anywhere on the ring /
        // line: every arrival is home, the re-check pass would find none
        if (!multi_hop) {
            settled = true;
            break;
        }
    }
    if (!settled) return set_err(c, GTCP_EINVARIANT, "shift: movers left after the multi-hop guard");
    // (the fixed-point charge scale needs max|w| of the new particle set: the
    // next deposit takes the max over all ranks, which bounds the arrivals too)
    mark();
    KCHECK();
    if (prof) {
        cudaStreamSynchronize(c->st);
        fprintf(stderr, "[shift%d r%d n=%lld]", dir, c->rank, c->n);
        for (int i = 1; i < nev; i++) {
            float ms;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %.3f", ms);
        }
        fprintf(stderr, "\n");
        for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
    }
    return GTCP_OK;
}
