/*
 * gtcp_oracle_omp.c -- TEST INFRASTRUCTURE ONLY (bench.py cpu_baseline).
 *
 * The paper's CPU charge method run over all host cores: every OpenMP thread
 * deposits a contiguous share of the particles into its OWN copy of the grid,
 * and the copies are then summed in thread order (§5: per-thread grid
 * replication, the private copies summed at the end of the charge phase in a
 * chosen order; the fixed order also makes the result deterministic).
 * The arithmetic is the oracle's: each thread calls orc_deposit / orc_push
 * of gtcp_oracle.c on its particle range (no new formula here).  The push and
 * the shift destination are embarrassingly parallel over particles.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int64_t orc_deposit(const void* p, int64_t n, const double* psi, const double* theta, const double* zeta,
                    const double* mu, const double* w, int32_t k0, int32_t P, double* grid);
int64_t orc_push(const void* p, int32_t stage, int64_t n, double* const* Xa, double* const* Xb, const double* mu,
                 int32_t k0, int32_t P, const double* gradphi);
void orc_shift_dest(const void* p, int64_t n, const double* zeta, int32_t P, int32_t* dest);

int orc_omp_threads(void) { return omp_get_max_threads(); }

/* grid (gsize doubles) is ACCUMULATED into, as orc_deposit. */
int64_t orc_deposit_replicas(const void* p, int64_t n, const double* psi, const double* theta, const double* zeta,
                             const double* mu, const double* w, int32_t k0, int32_t P, double* grid, int64_t gsize) {
    int nt = omp_get_max_threads();
    double** rep = (double**)calloc(nt, sizeof(double*));
    int64_t nclamp = 0;
#pragma omp parallel reduction(+ : nclamp)
    {
        int t = omp_get_thread_num(), T = omp_get_num_threads();
        int64_t lo = n * t / T, hi = n * (t + 1) / T;
        rep[t] = (double*)calloc(gsize, sizeof(double));
        nclamp += orc_deposit(p, hi - lo, psi + lo, theta + lo, zeta + lo, mu + lo, w + lo, k0, P, rep[t]);
#pragma omp barrier
        /* fixed-order merge: each thread owns a slice of the grid and adds the
         * replicas in thread order 0, 1, ..., T-1 */
        int64_t glo = gsize * t / T, ghi = gsize * (t + 1) / T;
        for (int q = 0; q < T; q++)
            for (int64_t a = glo; a < ghi; a++) grid[a] += rep[q][a];
#pragma omp barrier
        free(rep[t]);
    }
    free(rep);
    return nclamp;
}

int64_t orc_push_omp(const void* p, int32_t stage, int64_t n, double* const* Xa, double* const* Xb, const double* mu,
                     int32_t k0, int32_t P, const double* gradphi) {
    int64_t nrefl = 0;
#pragma omp parallel reduction(+ : nrefl)
    {
        int t = omp_get_thread_num(), T = omp_get_num_threads();
        int64_t lo = n * t / T, hi = n * (t + 1) / T;
        double* a[5];
        double* b[5];
        for (int d = 0; d < 5; d++) { a[d] = Xa[d] + lo; b[d] = Xb[d] + lo; }
        nrefl += orc_push(p, stage, hi - lo, a, b, mu + lo, k0, P, gradphi);
    }
    return nrefl;
}

void orc_shift_dest_omp(const void* p, int64_t n, const double* zeta, int32_t P, int32_t* dest) {
#pragma omp parallel
    {
        int t = omp_get_thread_num(), T = omp_get_num_threads();
        int64_t lo = n * t / T, hi = n * (t + 1) / T;
        orc_shift_dest(p, hi - lo, zeta + lo, P, dest + lo);
    }
}
