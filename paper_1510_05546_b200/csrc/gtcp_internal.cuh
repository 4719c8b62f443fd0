// gtcp_internal.cuh -- private declarations of the B200 GTC-P library.
// Product code: shares nothing with oracle/ (see DESIGN.md §2).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <atomic>

#include <string>
#include <vector>

#include "../../include/gtcp.h"
#include "gtcp_comm.cuh"

#define GTCP_TWO_PI (2.0 * 3.14159265358979323846)

// Geometry + physics constants passed by value to every kernel.
struct Geo {
    int mpsi, mzetamax, P, k0;     // rings, global planes, local planes, first local plane
    int nmu;                       // magnetic-moment bins in the bin key (1 = off)
    double mu_thr[15];             // their thresholds (Exp(1) quantiles of mu)
    int ntor, rank_t;              // toroidal domains, this rank's toroidal index
    int nrad, rank_r;              // radial domains, this rank's radial index
    double rbound[9];              // radial domain boundaries r(b_0 = ring 0) .. r(b_nrad = ring mpsi)
    double rbound2[9];             // their squares (fast classification away from a boundary)
    int mgrid;                     // nodes per plane incl. duplicates (< 2^31)
    int gstride;                   // nodes per interval of the push's gather field (mgrid padded to 3 mod 8)
    int paranl, drifts;
    int prec32;                    // particle store in fp32 (arithmetic stays fp64)
    int f32field;                  // gather field stored in fp32 (precision 32, or field_f32)
    double a0, a1, dr, inv_dr, R0, inv_R0, omega0, q0, q2, rln, rlt, tau, dt;
    double cz;                     // mzetamax / (2 pi), rounded once (Q-2, H-1)
    double psi_lo, psi_hi;         // a0^2/2, a1^2/2 padded inwards: psi strictly inside needs no reflection test
    double dzeta;                  // 2 pi / mzetamax
    double rhoG;                   // sqrt(2) / omega0 (F-1)
    double drift_cells;            // label-drift margin of the deposit tile windows (cells since the bin)
    double rho_cut_th;             // radial band of the tile windows: gyroradii up to rho_cut_th thermal radii
    double inv_omega0, inv_omega0_R0;
    const int* mtheta;             // [mpsi+1]
    const int* igrid;              // [mpsi+2]
    const int* itran;              // [mpsi+1]
    const double* qtinv;           // [mpsi+1]
    const unsigned short* node_ring;  // [mgrid] ring of each node (replaces a binary search)
};

// One charge tile: particles [start, end) of the cell-sorted store whose
// gyrocentre cell (ring, label) lay in ring `ring`, cells [c0, c1] at bin time.
// Per-ring constants of the F-1 gyro-average on the grid (Poisson operator),
// host-computed once: the theta-points' label offset on the node's own ring,
// and for the radial points r_i +- rhoG (s = 0, 1) their floor ring m_s, upper
// weight and, for rings m_s + q, the label map j -> j * ratio + zk * cz.
struct PoisRing {
    double dlab;
    double wp[2];
    double ratio[4], cz[4], inv_mt[4];
    int m[2];
    int mt, ig;
    int mtm[4], igm[4];
};

struct Tile {
    int ring, c0, c1, pad;
    long long start, end;
};

// SoA particle set: live state x[5] (psi, theta, zeta, rho_par, w), saved x0[5], mu.
struct PSet {
    double* x[5];
    double* x0[5];
    double* mu;
    unsigned long long* id;        // may be null
};

// Device counters (one allocation, zeroed at init).
struct DevCounters {
    unsigned long long wmax_bits;  // max |w| of the live state (bits of a positive double)
    long long reflections;
    long long plane_clamps;
    long long fallback;            // contributions that went straight to L2 in the last charge
    int fx_shift;                  // fixed-point F of the last charge
    int tile_next;                 // persistent-CTA tile counter
    int ntiles;                    // tiles built by the last bin
    int nonfinite;
    long long n_send[2];           // shift: movers to left / right
    long long n_keep;
    long long n_holes;
};

namespace gtcp {

// ---- kernels (gtcp_kernels.cu) -------------------------------------------
// tiled deposit, nb = CTAs per SM (3: 80 registers, 2: 128 registers and a
// larger window); limb capacity (nodes) of one window for each
__host__ __device__ constexpr int deposit_cap_nodes(int nb) { return nb == 2 ? 12288 : 7680; }
void launch_deposit_tiled(const Geo& g, const PSet& s, long long n, const Tile* tiles, int max_tiles,
                          long long* fx, DevCounters* dc, int ctas, size_t smem_bytes, int cap_nodes, int nb,
                          cudaStream_t st);
cudaError_t configure_deposit_tiled(size_t smem_bytes, int nb);
size_t deposit_tiled_smem(int P, int nb);
int deposit_tiled_ctas_per_sm(size_t smem_bytes, int nb);  // after configure_deposit_tiled
// fused RK2 stage push + deposit of the next stage's charge;
// configure returns the CTAs per SM it runs at (0: not available)
size_t push_deposit_smem(const Geo& g, size_t* rt_off);
int configure_push_deposit(const Geo& g);
void launch_push_deposit(const Geo& g, const PSet& s, long long n, const Tile* tiles, long long* fx, DevCounters* dc,
                         int ctas, int cap_nodes, const double* const src[5], const double* const base[5],
                         double* const out[5], const double* gf, double h, cudaStream_t st);
void launch_deposit_direct(const Geo& g, const PSet& s, long long begin, long long n, long long* fx,
                           DevCounters* dc, cudaStream_t st);
// charge ablation: the paper's update-binning deposit (points binned by cell
// every charge, one thread per super-cell, twin shared-memory copies)
void launch_deposit_points(const Geo& g, const PSet& s, long long n, long long* fx, DevCounters* dc, unsigned* pkey,
                           unsigned* prank, unsigned* rec, unsigned* count, unsigned* offset, unsigned* scan_tmp,
                           const int4* segs, int nseg, cudaStream_t st);
void launch_fx_scale(DevCounters* dc, cudaStream_t st, int headroom = 0);
void launch_fx_to_real(const Geo& g, const long long* fx, double* rho, const DevCounters* dc, int planes,
                       cudaStream_t st);
void launch_push3(const Geo& g, const double* const src[5], const double* const base[5], double* const out[5],
                  const double* mu, long long n, double h, const double* gfield, DevCounters* dc, cudaStream_t st,
                  unsigned char* cls = nullptr, unsigned* cntL = nullptr, unsigned* cntR = nullptr,
                  double* g3 = nullptr, long long* far = nullptr);  // g3 != null: loop-fission ablation (3 n doubles of gbar)
void launch_wmax(const double* w, long long n, DevCounters* dc, cudaStream_t st);
void launch_bin_keys(const Geo& g, const PSet& s, long long n, unsigned* key, unsigned* rank, unsigned* count,
                     cudaStream_t st);
void launch_scan_u32(const unsigned* in, unsigned* out, long long n, unsigned* block_tmp, cudaStream_t st);
void launch_bin_inverse(const unsigned* key, const unsigned* rank, const unsigned* offset, long long n,
                        unsigned* inv, cudaStream_t st);
void launch_gather_perm_multi(const double* const* src, double* const* dst, int na, const unsigned long long* id_src,
                              unsigned long long* id_dst, const unsigned* inv, long long n, cudaStream_t st);
void launch_gather_perm_f64(const double* src, double* dst, const unsigned* inv, long long n, cudaStream_t st);
void launch_gather_perm_u64(const unsigned long long* src, unsigned long long* dst, const unsigned* inv, long long n,
                            cudaStream_t st);
void launch_permute_f64(const double* src, double* dst, const unsigned* dest, long long n, cudaStream_t st);
void launch_permute_u64(const unsigned long long* src, unsigned long long* dst, const unsigned* dest,
                        long long n, cudaStream_t st);
void launch_build_tiles(const Geo& g, const unsigned* offset, int tile_max, Tile* tiles, int max_tiles,
                        DevCounters* dc, const int* span, int* ring_cnt, cudaStream_t st);
void launch_tile_spans(const Geo& g, int cap_nodes, int* span, cudaStream_t st);  // once, at init
void launch_load(const Geo& g, const PSet& s, long long n, unsigned long long seed, long long id0,
                 double w_amp, double vcut, double zlo, double zhi, double rlo, double rhi, cudaStream_t st);
// grid kernels (gtcp_grid.cu)
void launch_fill_dup(const Geo& g, double* f, int planes, int ncomp, cudaStream_t st);
void launch_seam_rotate(const Geo& g, const double* src, double* dst, int shift_sign, cudaStream_t st);
void launch_rotate_add_i64(const Geo& g, const long long* src, long long* dst, int shift_sign, cudaStream_t st);
void launch_normalize(const Geo& g, const double* rho, const double* nm, double* dn, cudaStream_t st);
void launch_smooth_theta(const Geo& g, const double* in, double* out, cudaStream_t st);
void launch_smooth_r(const Geo& g, const double* in, double* out, cudaStream_t st);
void launch_smooth_par(const Geo& g, const double* in, double* out, cudaStream_t st);
void launch_ring_sum(const Geo& g, const double* f, double* ringsum, cudaStream_t st);
void launch_jacobi_init(const Geo& g, const double* dn, const double* ringsum, double* rhs, double* phi,
                        cudaStream_t st);
void launch_gyro(const Geo& g, const PoisRing* pr, const double* in, double* out, int kbeg, int kcount,
                 cudaStream_t st);
void launch_gyro_jacobi(const Geo& g, const PoisRing* pr, const double* g1, const double* rhs, double* phi,
                        double omega, int kbeg, int kcount, cudaStream_t st);
void launch_zonal(const Geo& g, const double* ringsum, double* phi00, cudaStream_t st);
void launch_add_zonal2(const Geo& g, const double* phi00, const double* phi, double* phiH, cudaStream_t st);
void launch_field(const Geo& g, const double* phi, double* gfield, cudaStream_t st);
void launch_gfield_export(const Geo& g, const double* gfield, double* out, cudaStream_t st);
void launch_gfield_import(const Geo& g, const double* in, double* gfield, cudaStream_t st);
void launch_marker_from_rho(const Geo& g, const double* rho, double* ringsum, cudaStream_t st);
void launch_ring_mean(const Geo& g, const double* ringsum, double* nm, cudaStream_t st);
void launch_sum_f64(const double* x, long long n, double* out, double* partial, cudaStream_t st);
void launch_sum_i64_pair(const long long* in2, long long* out, cudaStream_t st);
// diagnostics: heat flux sum_p w E_kin v_E,r with the current gather field;
// field energy sum phi^2 over the owned planes' canonical nodes (phi: plane 0)
void launch_heat_flux(const Geo& g, const PSet& s, long long n, const double* gf, double* out, double* partial,
                      cudaStream_t st);
void launch_field_energy(const Geo& g, const double* phi, double* out, double* partial, cudaStream_t st);
// shift (gtcp_shift.cu)
int shift_chunks(long long n);
void launch_shift_classify(const Geo& g, const double* zeta, const double* psi, int mode, long long n,
                           unsigned char* cls, unsigned* cntL, unsigned* cntR, long long* far, cudaStream_t st);
void launch_shift_nkeep(long long n, const unsigned* totL, const unsigned* totR, long long* nkeep, long long* counts,
                        cudaStream_t st);
void launch_shift_count_holes(const unsigned char* cls, long long n, const long long* nkeep, unsigned* cntH,
                              unsigned* cntF, cudaStream_t st);
void launch_shift_pack(double* const* attrs, int nattr, unsigned long long* id, const unsigned char* cls, long long n,
                       const unsigned* offL, const unsigned* offR, double* const* sendL, double* const* sendR,
                       unsigned long long* idL, unsigned long long* idR, unsigned* idx, long long nL, long long nR,
                       cudaStream_t st);
void launch_shift_backfill(double* const* attrs, int nattr, unsigned long long* id, const unsigned char* cls,
                           long long n, const long long* nkeep, const unsigned* offH, const unsigned* offF,
                           unsigned* holes, unsigned* fills, long long nholes, cudaStream_t st);
void launch_fill_f64(double* x, long long n, double v, cudaStream_t st);
void launch_gather_f64(const double* src, const long long* idx, long long m, double* out, cudaStream_t st);
void launch_gather_u64(const unsigned long long* src, const long long* idx, long long m, unsigned long long* out,
                       cudaStream_t st);

extern std::atomic<long long> g_launches;  // kernels launched (for the bench's gpu_launches claim)
extern thread_local int g_prec32;         // precision of the current context's particle store

}  // namespace gtcp
