/*
 * vrp_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see vrp_oracle.h).  Compiled with
 * -ffp-contract=off so that every a*b+c is two roundings, as in CPython.
 *
 * Reference files are /root/reference/pkg/src/vrp_rpd/<file>:<line>.
 */
#include "vrp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* minimal dynamic parallel-for over [0, N) in chunks (pthreads, no OpenMP) */
typedef struct {
    int64_t N, chunk;
    int64_t next;
    pthread_mutex_t mu;
    void (*body)(void *ctx, int64_t i);
    void *ctx;
} pfor_t;

static void *pfor_worker(void *arg) {
    pfor_t *pf = (pfor_t *)arg;
    for (;;) {
        pthread_mutex_lock(&pf->mu);
        int64_t lo = pf->next;
        pf->next += pf->chunk;
        pthread_mutex_unlock(&pf->mu);
        if (lo >= pf->N) break;
        int64_t hi = lo + pf->chunk < pf->N ? lo + pf->chunk : pf->N;
        for (int64_t i = lo; i < hi; ++i) pf->body(pf->ctx, i);
    }
    return NULL;
}

int32_t orc_default_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int32_t)c : 1;
}

static void parallel_for(int64_t N, int64_t chunk, int32_t threads,
                         void (*body)(void *, int64_t), void *ctx) {
    if (threads <= 0) threads = orc_default_threads();
    if (threads > 256) threads = 256;
    pfor_t pf = {N, chunk, 0, PTHREAD_MUTEX_INITIALIZER, body, ctx};
    if (threads == 1 || N <= chunk) { pfor_worker(&pf); return; }
    pthread_t tid[256];
    for (int32_t t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, pfor_worker, &pf);
    for (int32_t t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

#define OP_C(op) (((op) >> 1) + 1)
#define OP_IS_PICK(op) ((op) & 1)

/* ------------------------------------------------------------------------- */
/* numpy Philox4x64-10 + Generator draws (numpy/random/src/philox, distributions.c) */
/* ------------------------------------------------------------------------- */

static inline uint64_t mulhilo64(uint64_t a, uint64_t b, uint64_t *hi) {
    __uint128_t prod = (__uint128_t)a * (__uint128_t)b;
    *hi = (uint64_t)(prod >> 64);
    return (uint64_t)prod;
}

static void philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t hi0, hi1;
        uint64_t lo0 = mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0);
        uint64_t lo1 = mulhilo64(0xCA5A826395121157ULL, c2, &hi1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t orc_philox_next64(orc_philox *s) {
    if (s->buffer_pos < 4) return s->buffer[s->buffer_pos++];
    if (++s->ctr[0] == 0)
        if (++s->ctr[1] == 0)
            if (++s->ctr[2] == 0) ++s->ctr[3];
    philox_block(s->ctr, s->key, s->buffer);
    s->buffer_pos = 1;
    return s->buffer[0];
}

uint32_t orc_philox_next32(orc_philox *s) {
    if (s->has_uint32) {
        s->has_uint32 = 0;
        return s->uinteger;
    }
    uint64_t x = orc_philox_next64(s);
    s->has_uint32 = 1;
    s->uinteger = (uint32_t)(x >> 32);
    return (uint32_t)(x & 0xffffffffULL);
}

double orc_philox_next_double(orc_philox *s) {
    return (double)(orc_philox_next64(s) >> 11) * (1.0 / 9007199254740992.0);
}

uint64_t orc_philox_integers(orc_philox *s, uint64_t n) {
    /* integers(0, n): inclusive range rng = n - 1 */
    uint64_t rng = n - 1;
    if (rng == 0) return 0;
    if (rng == 0xffffffffULL) return orc_philox_next32(s);
    uint32_t excl = (uint32_t)(rng + 1);
    uint64_t prod = (uint64_t)orc_philox_next32(s) * excl;
    uint32_t left = (uint32_t)prod;
    if (left < excl) {
        uint32_t thresh = (uint32_t)((0xffffffffULL - rng) % excl);
        while (left < thresh) {
            prod = (uint64_t)orc_philox_next32(s) * excl;
            left = (uint32_t)prod;
        }
    }
    return prod >> 32;
}

void orc_philox_fill_double(orc_philox *s, double *out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = orc_philox_next_double(s);
}

/* ------------------------------------------------------------------------- */
/* schedule.py                                                               */
/* ------------------------------------------------------------------------- */

/* schedule.py:159-185 route_initial_load: minimal feasible initial load. */
int orc_route_initial_load(const int32_t *route, int32_t L, int32_t k, int32_t *q0) {
    int32_t s = 0, lo = 0, hi = k;
    for (int32_t i = 0; i < L; ++i) {
        if (!OP_IS_PICK(route[i])) {
            if (1 - s > lo) lo = 1 - s;
            if (lo > hi) return ORC_CAPACITY;
            --s;
        } else {
            if (k - 1 - s < hi) hi = k - 1 - s;
            if (lo > hi) return ORC_CAPACITY;
            ++s;
        }
    }
    if (q0) *q0 = lo;
    return ORC_OK;
}

/* schedule.py:134-156 validate_solution (tour count is structural here). */
int orc_validate(int32_t n, int32_t m, const int32_t *ops, const int32_t *len) {
    int64_t total = 0;
    for (int32_t v = 0; v < m; ++v) {
        if (len[v] < 0) return ORC_MALFORMED;
        total += len[v];
    }
    if (total != 2 * (int64_t)n) return ORC_MALFORMED;
    unsigned char *seen = (unsigned char *)calloc((size_t)(2 * n + 1), 1);
    int st = ORC_OK;
    for (int64_t i = 0; i < total; ++i) {
        int32_t op = ops[i];
        if (op < 0 || op >= 2 * n || seen[op]) { st = ORC_MALFORMED; break; }
        seen[op] = 1;
    }
    free(seen);
    return st;
}

/* Shared event-driven simulator: schedule.py:265-316 exact_makespan, and
 * (with arrival/time records) schedule.py:188-257 evaluate.  Round-robin over
 * vehicles, each advancing until a pickup whose dropoff is not yet done. */
static int simulate(int32_t n, int32_t m, const double *d, const double *p,
                    const int32_t *ops, const int32_t *len, double *z, double *returns,
                    double *arrival, double *time_out) {
    const int64_t W = n + 1;
    int64_t off[64];
    int32_t pos[64], loc[64];
    double tv[64];
    int64_t remaining = 0;
    for (int32_t v = 0; v < m; ++v) {
        off[v] = remaining;
        remaining += len[v];
        pos[v] = 0; loc[v] = 0; tv[v] = 0.0;
    }
    double *t_drop = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    unsigned char *done = (unsigned char *)calloc((size_t)(n + 1), 1);
    int st = ORC_OK;
    while (remaining) {
        int progress = 0;
        for (int32_t v = 0; v < m; ++v) {
            int32_t i = pos[v], L = len[v], at = loc[v];
            double t = tv[v];
            const int32_t *route = ops + off[v];
            while (i < L) {
                int32_t op = route[i];
                int32_t c = OP_C(op);
                if (!OP_IS_PICK(op)) {
                    t += d[at * W + c];
                    t_drop[c] = t;
                    done[c] = 1;
                    if (arrival) { arrival[off[v] + i] = t; time_out[off[v] + i] = t; }
                } else {
                    if (!done[c]) break;
                    double arr = t + d[at * W + c];
                    double ready = t_drop[c] + p[c];
                    t = arr >= ready ? arr : ready;
                    if (arrival) { arrival[off[v] + i] = arr; time_out[off[v] + i] = t; }
                }
                at = c;
                ++i;
            }
            if (i != pos[v]) {
                remaining -= i - pos[v];
                pos[v] = i;
                tv[v] = t;
                loc[v] = at;
                progress = 1;
            }
        }
        if (!progress) { st = ORC_DEADLOCK; break; }
    }
    if (st == ORC_OK) {
        double best = 0.0;
        for (int32_t v = 0; v < m; ++v) {
            double r = 0.0;
            if (len[v]) {
                r = tv[v] + d[(int64_t)loc[v] * W];
                if (r > best) best = r;
            }
            if (returns) returns[v] = r;
        }
        *z = best;
    }
    free(t_drop);
    free(done);
    return st;
}

int orc_exact_makespan(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                       const int32_t *ops, const int32_t *len, double *z, double *returns) {
    int64_t off = 0;
    for (int32_t v = 0; v < m; ++v) {
        if (orc_route_initial_load(ops + off, len[v], k, NULL) != ORC_OK) return ORC_CAPACITY;
        off += len[v];
    }
    /* exact_makespan has no structural check; guard memory only */
    for (int64_t i = 0; i < off; ++i)
        if (ops[i] < 0 || ops[i] >= 2 * n) return ORC_MALFORMED;
    return simulate(n, m, d, p, ops, len, z, returns, NULL, NULL);
}

int orc_evaluate(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                 const int32_t *ops, const int32_t *len, double *z, double *returns,
                 double *arrival, double *time, int32_t *q0) {
    if (orc_validate(n, m, ops, len) != ORC_OK) return ORC_MALFORMED;
    int64_t off = 0;
    for (int32_t v = 0; v < m; ++v) {
        if (orc_route_initial_load(ops + off, len[v], k, q0 ? q0 + v : NULL) != ORC_OK)
            return ORC_CAPACITY;
        off += len[v];
    }
    return simulate(n, m, d, p, ops, len, z, returns, arrival, time);
}

/* schedule.py:345-393 two_pass_estimate */
int orc_two_pass(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                 const int32_t *ops, const int32_t *len, double *z) {
    if (orc_validate(n, m, ops, len) != ORC_OK) return ORC_MALFORMED;
    const int64_t W = n + 1;
    int64_t off = 0;
    for (int32_t v = 0; v < m; ++v) {
        if (orc_route_initial_load(ops + off, len[v], k, NULL) != ORC_OK) return ORC_CAPACITY;
        off += len[v];
    }
    /* same-route pickup before its own dropoff (schedule.py:362-369) */
    int32_t *route_of_drop = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    unsigned char *seen = (unsigned char *)calloc((size_t)(n + 1), 1);
    double *ready = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    off = 0;
    for (int32_t v = 0; v < m; ++v) {
        for (int32_t i = 0; i < len[v]; ++i)
            if (!OP_IS_PICK(ops[off + i])) route_of_drop[OP_C(ops[off + i])] = v;
        off += len[v];
    }
    int st = ORC_OK;
    off = 0;
    for (int32_t v = 0; v < m && st == ORC_OK; ++v) {
        for (int32_t i = 0; i < len[v]; ++i) {
            int32_t op = ops[off + i], c = OP_C(op);
            if (!OP_IS_PICK(op)) seen[c] = 1;
            else if (route_of_drop[c] == v && !seen[c]) { st = ORC_DEADLOCK; break; }
        }
        off += len[v];
    }
    if (st == ORC_OK) {
        off = 0;
        for (int32_t v = 0; v < m; ++v) {
            double t = 0.0;
            int32_t at = 0;
            for (int32_t i = 0; i < len[v]; ++i) {
                int32_t op = ops[off + i], c = OP_C(op);
                t += d[at * W + c];
                at = c;
                if (!OP_IS_PICK(op)) ready[c] = t + p[c];
            }
            off += len[v];
        }
        double best = 0.0;
        off = 0;
        for (int32_t v = 0; v < m; ++v) {
            if (len[v]) {
                double t = 0.0;
                int32_t at = 0;
                for (int32_t i = 0; i < len[v]; ++i) {
                    int32_t op = ops[off + i], c = OP_C(op);
                    t += d[at * W + c];
                    at = c;
                    if (OP_IS_PICK(op) && ready[c] > t) t = ready[c];
                }
                t += d[(int64_t)at * W];
                if (t > best) best = t;
            }
            off += len[v];
        }
        *z = best;
    }
    free(route_of_drop);
    free(seen);
    free(ready);
    return st;
}

typedef struct {
    int32_t n, m, k, mode;
    const double *d, *p;
    const int32_t *ops, *len;
    double *z, *returns;
    int32_t *status;
} mk_ctx;

static void mk_body(void *vctx, int64_t i) {
    mk_ctx *c = (mk_ctx *)vctx;
    const int32_t *o = c->ops + i * 2 * (int64_t)c->n;
    const int32_t *l = c->len + i * (int64_t)c->m;
    double zi = 0.0;
    double *ret = c->returns ? c->returns + i * (int64_t)c->m : NULL;
    int st;
    if (c->mode == 0) st = orc_exact_makespan(c->n, c->m, c->k, c->d, c->p, o, l, &zi, ret);
    else if (c->mode == 1) st = orc_evaluate(c->n, c->m, c->k, c->d, c->p, o, l, &zi, ret, NULL, NULL, NULL);
    else st = orc_two_pass(c->n, c->m, c->k, c->d, c->p, o, l, &zi);
    c->z[i] = st == ORC_OK ? zi : 0.0;
    c->status[i] = st;
}

void orc_makespan_batch(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                        const int32_t *ops, const int32_t *len, int64_t N, int32_t mode,
                        double *z, int32_t *status, double *returns, int32_t threads) {
    mk_ctx c = {n, m, k, mode, d, p, ops, len, z, returns, status};
    parallel_for(N, 64, threads, mk_body, &c);
}

/* ------------------------------------------------------------------------- */
/* brkga.py                                                                  */
/* ------------------------------------------------------------------------- */

/* numpy.argsort(kind="stable"): ascending, ties by index, NaN last. */
static int less_key(double a, int64_t ia, double b, int64_t ib) {
    int na = isnan(a), nb = isnan(b);
    if (na || nb) {
        if (na && nb) return ia < ib;
        return nb;  /* non-NaN < NaN */
    }
    if (a < b) return 1;
    if (a > b) return 0;
    return ia < ib;
}

void orc_stable_argsort(const double *x, int64_t count, int64_t *order) {
    /* bottom-up merge sort on indices */
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(count > 0 ? count : 1));
    for (int64_t i = 0; i < count; ++i) order[i] = i;
    for (int64_t w = 1; w < count; w *= 2) {
        for (int64_t lo = 0; lo < count; lo += 2 * w) {
            int64_t mid = lo + w < count ? lo + w : count;
            int64_t hi = lo + 2 * w < count ? lo + 2 * w : count;
            int64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (less_key(x[order[b]], order[b], x[order[a]], order[a])) tmp[o++] = order[b++];
                else tmp[o++] = order[a++];
            }
            while (a < mid) tmp[o++] = order[a++];
            while (b < hi) tmp[o++] = order[b++];
        }
        memcpy(order, tmp, sizeof(int64_t) * (size_t)count);
    }
    free(tmp);
}

/* brkga.py:82-89 _hint_vehicle */
int32_t orc_hint_vehicle(int32_t m, double gene) {
    double x = (double)m * gene;
    int64_t h = (int64_t)x;
    if (x - (double)h > 1.0 - 1e-9) h += 1;
    return (int32_t)(h < m ? h : m - 1);
}

/* brkga.py:92-207 decode */
void orc_decode(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                const double *genes, int32_t relax, double penalty,
                int32_t *ops_out, int32_t *len_out, double *fitness, double *makespan,
                int32_t *scheduled, int64_t *visits_out) {
    const int64_t W = n + 1;
    const int32_t two_n = 2 * n;
    const double *pi = genes, *alpha = genes + two_n;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)two_n);
    orc_stable_argsort(pi, two_n, order);
    int32_t *pending = (int32_t *)malloc(sizeof(int32_t) * (size_t)two_n);
    int32_t npend = two_n;
    for (int32_t i = 0; i < two_n; ++i) pending[i] = (int32_t)order[i];
    free(order);

    double t[64], comp_v[64];
    int32_t loc[64], net[64], lo[64], hi[64], feas[64];
    for (int32_t v = 0; v < m; ++v) { t[v] = 0.0; loc[v] = 0; net[v] = 0; lo[v] = 0; hi[v] = k; }
    double *t_drop = (double *)calloc((size_t)(n + 1), sizeof(double));
    unsigned char *dropped = (unsigned char *)calloc((size_t)(n + 1), 1);
    /* schedule sequence (op, vehicle), compacted vehicle-major at the end */
    int32_t *seq_op = (int32_t *)malloc(sizeof(int32_t) * (size_t)two_n);
    int32_t *seq_v = (int32_t *)malloc(sizeof(int32_t) * (size_t)two_n);
    int32_t nseq = 0;
    int64_t visits = 0;

    for (int32_t pass = 0; pass < two_n; ++pass) {
        if (!npend) break;
        int32_t ndef = 0, progressed = 0;
        for (int32_t j = 0; j < npend; ++j) {
            int32_t op = pending[j];
            ++visits;
            int32_t c = OP_C(op), is_pick = OP_IS_PICK(op);
            if (is_pick && !dropped[c]) { pending[ndef++] = op; continue; }
            double ready = is_pick ? t_drop[c] + p[c] : 0.0;
            int32_t nf = 0;
            for (int32_t v = 0; v < m; ++v) {
                if (is_pick) {
                    int32_t room = k - 1 - net[v];
                    if (!(lo[v] <= (room < hi[v] ? room : hi[v]))) continue;
                    if (relax) {
                        double arr = t[v] + d[loc[v] * W + c];
                        comp_v[nf] = arr >= ready ? arr : ready;
                        feas[nf++] = v;
                    } else if (t[v] >= ready) {
                        comp_v[nf] = t[v] + d[loc[v] * W + c];
                        feas[nf++] = v;
                    }
                } else {
                    int32_t need = 1 - net[v];
                    if ((need > lo[v] ? need : lo[v]) <= hi[v]) {
                        comp_v[nf] = t[v] + d[loc[v] * W + c];
                        feas[nf++] = v;
                    }
                }
            }
            if (!nf) { pending[ndef++] = op; continue; }
            int32_t hint = orc_hint_vehicle(m, alpha[op]);
            int32_t pick = -1;
            double pc = 0.0;
            for (int32_t f = 0; f < nf; ++f)
                if (feas[f] == hint) { pick = hint; pc = comp_v[f]; break; }
            if (pick < 0) {
                int32_t bd = 0;
                for (int32_t f = 0; f < nf; ++f) {
                    int32_t v = feas[f], dist = v > hint ? v - hint : hint - v;
                    if (pick < 0 || comp_v[f] < pc || (comp_v[f] == pc && (dist < bd || (dist == bd && v < pick)))) {
                        pick = v; pc = comp_v[f]; bd = dist;
                    }
                }
            }
            int32_t v = pick;
            t[v] = pc;
            loc[v] = c;
            if (is_pick) {
                int32_t room = k - 1 - net[v];
                if (room < hi[v]) hi[v] = room;
                net[v] += 1;
            } else {
                int32_t need = 1 - net[v];
                if (need > lo[v]) lo[v] = need;
                net[v] -= 1;
                dropped[c] = 1;
                t_drop[c] = pc;
            }
            seq_op[nseq] = op;
            seq_v[nseq] = v;
            ++nseq;
            progressed = 1;
        }
        npend = ndef;
        if (!progressed) break;
    }
    double z = 0.0;
    for (int32_t v = 0; v < m; ++v) {
        double r = t[v] + d[(int64_t)loc[v] * W];
        if (v == 0 || r > z) z = r;
    }
    /* vehicle-major compaction, then -1 padding to 2n */
    int32_t o = 0;
    for (int32_t v = 0; v < m; ++v) {
        int32_t cnt = 0;
        for (int32_t i = 0; i < nseq; ++i)
            if (seq_v[i] == v) { ops_out[o++] = seq_op[i]; ++cnt; }
        len_out[v] = cnt;
    }
    for (; o < two_n; ++o) ops_out[o] = -1;
    *fitness = z + penalty * (double)npend;
    *makespan = z;
    *scheduled = two_n - npend;
    *visits_out = visits;
    free(pending); free(t_drop); free(dropped); free(seq_op); free(seq_v);
}

typedef struct {
    int32_t n, m, k, relax;
    const double *d, *p, *genes;
    double penalty;
    int32_t *ops_out, *len_out, *scheduled;
    double *fitness, *makespan;
    int64_t *visits;
} dec_ctx;

static void dec_body(void *vctx, int64_t i) {
    dec_ctx *c = (dec_ctx *)vctx;
    orc_decode(c->n, c->m, c->k, c->d, c->p, c->genes + i * 4 * (int64_t)c->n, c->relax,
               c->penalty, c->ops_out + i * 2 * (int64_t)c->n, c->len_out + i * (int64_t)c->m,
               c->fitness + i, c->makespan + i, c->scheduled + i, c->visits + i);
}

void orc_decode_batch(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                      const double *genes, int64_t N, int32_t relax, double penalty,
                      int32_t *ops_out, int32_t *len_out, double *fitness, double *makespan,
                      int32_t *scheduled, int64_t *visits, int32_t threads) {
    dec_ctx c = {n, m, k, relax, d, p, genes, penalty, ops_out, len_out, scheduled,
                 fitness, makespan, visits};
    parallel_for(N, 4, threads, dec_body, &c);
}

/* brkga.py:231-252 evolve */
int orc_evolve(const double *pop, const double *fit, int64_t N, int64_t G,
               double elite_frac, double mutant_frac, double bias, orc_philox *rng,
               double *out) {
    int64_t n_elite = (int64_t)(elite_frac * (double)N);
    int64_t n_mutant = (int64_t)(mutant_frac * (double)N);
    int64_t n_off = N - n_elite - n_mutant;
    if (n_elite < 1 || N - n_elite < 1) return -1;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    orc_stable_argsort(fit, N, order);
    for (int64_t i = 0; i < n_elite; ++i)
        memcpy(out + i * G, pop + order[i] * G, sizeof(double) * (size_t)G);
    orc_philox_fill_double(rng, out + n_elite * G, n_mutant * G);
    int64_t *e_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_off > 0 ? n_off : 1));
    int64_t *o_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_off > 0 ? n_off : 1));
    for (int64_t i = 0; i < n_off; ++i) e_idx[i] = (int64_t)orc_philox_integers(rng, (uint64_t)n_elite);
    for (int64_t i = 0; i < n_off; ++i) o_idx[i] = (int64_t)orc_philox_integers(rng, (uint64_t)(N - n_elite));
    for (int64_t i = 0; i < n_off; ++i) {
        const double *e = pop + order[e_idx[i]] * G;
        const double *q = pop + order[n_elite + o_idx[i]] * G;
        double *dst = out + (n_elite + n_mutant + i) * G;
        for (int64_t g = 0; g < G; ++g) {
            double u = orc_philox_next_double(rng);
            dst[g] = u < bias ? e[g] : q[g];
        }
    }
    free(order); free(e_idx); free(o_idx);
    return 0;
}
