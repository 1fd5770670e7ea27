/*
 * vrp_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this library: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, and only as the checker or
 * as the timed CPU baseline.
 *
 * Every function restates one reference function (file:line given below,
 * relative to /root/reference/pkg/src/vrp_rpd/).  Parity of this restatement
 * is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, run in the build container where the
 * reference is importable) -- see tests/test_oracle_golden.py.
 *
 * Data conventions (shared with include/vrp_rpd.h):
 *   d      (n+1)*(n+1) row-major fp64 travel times, depot = 0
 *   p      (n+1) fp64 processing times, p[0] = 0
 *   op     2*(c-1) + kind, kind 0 = dropoff (D), 1 = pickup (P)   (brkga.py:73-75)
 *   ops    one candidate = m routes concatenated vehicle-major, lengths len[m]
 *   status 0 OK, 1 CAPACITY, 2 DEADLOCK, 3 MALFORMED
 */
#ifndef VRP_ORACLE_H
#define VRP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_CAPACITY = 1, ORC_DEADLOCK = 2, ORC_MALFORMED = 3 };

/* numpy.random.Philox bit-generator state + numpy's buffered uint32 half.
 * Field-for-field the same as Generator(Philox).bit_generator.state. */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buffer[4];
    int32_t buffer_pos;
    int32_t has_uint32;
    uint32_t uinteger;
    uint32_t _pad;
} orc_philox;

uint64_t orc_philox_next64(orc_philox *s);
uint32_t orc_philox_next32(orc_philox *s);
double orc_philox_next_double(orc_philox *s);
/* Generator.integers(0, n) for 1 <= n <= 2^32 (Lemire, 32-bit, numpy semantics) */
uint64_t orc_philox_integers(orc_philox *s, uint64_t n);
void orc_philox_fill_double(orc_philox *s, double *out, int64_t count);

int orc_route_initial_load(const int32_t *route, int32_t L, int32_t k, int32_t *q0);
int orc_validate(int32_t n, int32_t m, const int32_t *ops, const int32_t *len);

int orc_exact_makespan(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                       const int32_t *ops, const int32_t *len, double *z, double *returns);
int orc_evaluate(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                 const int32_t *ops, const int32_t *len, double *z, double *returns,
                 double *arrival, double *time, int32_t *q0);
int orc_two_pass(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                 const int32_t *ops, const int32_t *len, double *z);

/* batch drivers: candidates are padded rows of stride 2n ops, m lens.
 * mode 0 = exact_makespan, 1 = evaluate (validating), 2 = two_pass_estimate.
 * threads <= 0 means all available. */
void orc_makespan_batch(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                        const int32_t *ops, const int32_t *len, int64_t N, int32_t mode,
                        double *z, int32_t *status, double *returns, int32_t threads);

int32_t orc_default_threads(void);
void orc_stable_argsort(const double *x, int64_t count, int64_t *order);
int32_t orc_hint_vehicle(int32_t m, double gene);
void orc_decode(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                const double *genes, int32_t relax, double penalty,
                int32_t *ops_out, int32_t *len_out, double *fitness, double *makespan,
                int32_t *scheduled, int64_t *visits);
void orc_decode_batch(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                      const double *genes, int64_t N, int32_t relax, double penalty,
                      int32_t *ops_out, int32_t *len_out, double *fitness, double *makespan,
                      int32_t *scheduled, int64_t *visits, int32_t threads);

/* returns 0, or -1 (PopulationTooSmall) */
int orc_evolve(const double *pop, const double *fit, int64_t N, int64_t G,
               double elite_frac, double mutant_frac, double bias, orc_philox *rng,
               double *out);

/* insertion.py restatement (insertion_oracle.c) */
double orc_py_sum(const double *x, int cnt);
int orc_reinsert_all(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                     int32_t *ops, int32_t *lens, const int32_t *removed, int32_t nremoved,
                     int32_t regret_k, orc_philox *rng);
int orc_remove_customers(int32_t n, int32_t m, int32_t k, int32_t *ops, int32_t *lens,
                         const int32_t *customers, int32_t ncust, int32_t *removed_out);

#ifdef __cplusplus
}
#endif
#endif
