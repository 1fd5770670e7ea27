/*
 * insertion_oracle.c -- CPU restatement of the reference's insertion scoring
 * and repair (/root/reference/pkg/src/vrp_rpd/insertion.py) and of the
 * removal cascade.  TEST INFRASTRUCTURE ONLY (see vrp_oracle.h).
 *
 *   InsertionContext   insertion.py:52-350  (_pass1/_pass2/_refresh_aggregates,
 *                                            cost_of, eval_gaps, eval_pair_gaps,
 *                                            ret_after_drop, tentative_drop)
 *   remove_customers   insertion.py:379-397 (with _first_capacity_break 358-376)
 *   _pick_windowed     insertion.py:414-426
 *   customer_options   insertion.py:429-472
 *   reinsert_all       insertion.py:484-516
 *   CPython 3.12 sum() (Neumaier compensation) where the reference sums floats.
 *
 * Routes are op-code arrays (2(c-1)+kind).  Compiled with -ffp-contract=off.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "vrp_oracle.h"

#define OPC(op) (((op) >> 1) + 1)
#define ISP(op) ((op) & 1)
#define NEG_BIG (-(1 << 28))
#define POS_BIG (1 << 28)
#define MAXM 32

typedef struct {
    int L;
    int *seq;          /* op codes, capacity 2n+2 */
    double *T, *dep, *M;
    int *sp, *lo_pre, *hi_pre, *lo_suf, *hi_suf, *drops_suf; /* L+1 */
    double ret, exit_leg;
} route_t;

typedef struct {
    int n, m, k;
    const double *d, *p;
    route_t r[MAXM];
    double *ready;      /* n+1 */
    unsigned char *has_ready;
    int *pos_v, *pos_i; /* dropoff position per customer, -1 when absent */
    double sum_ret;
    double omax[MAXM];
} ictx_t;

/* CPython 3.12 builtin sum over floats with int start 0 (bltinmodule.c) */
double orc_py_sum(const double *x, int cnt) {
    if (cnt <= 0) return 0.0;
    double f = x[0], c = 0.0;
    for (int i = 1; i < cnt; ++i) {
        double t = f + x[i];
        if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

static void route_alloc(route_t *R, int cap) {
    R->seq = (int *)malloc(sizeof(int) * cap);
    R->T = (double *)malloc(sizeof(double) * cap);
    R->dep = (double *)malloc(sizeof(double) * cap);
    R->M = (double *)malloc(sizeof(double) * cap);
    R->sp = (int *)malloc(sizeof(int) * (cap + 1));
    R->lo_pre = (int *)malloc(sizeof(int) * (cap + 1));
    R->hi_pre = (int *)malloc(sizeof(int) * (cap + 1));
    R->lo_suf = (int *)malloc(sizeof(int) * (cap + 1));
    R->hi_suf = (int *)malloc(sizeof(int) * (cap + 1));
    R->drops_suf = (int *)malloc(sizeof(int) * (cap + 1));
    R->L = 0;
    R->ret = R->exit_leg = 0.0;
}

static void route_free(route_t *R) {
    free(R->seq); free(R->T); free(R->dep); free(R->M); free(R->sp); free(R->lo_pre);
    free(R->hi_pre); free(R->lo_suf); free(R->hi_suf); free(R->drops_suf);
}

static void route_copy(route_t *dst, const route_t *src) {
    int L = src->L;
    dst->L = L;
    memcpy(dst->seq, src->seq, sizeof(int) * L);
    memcpy(dst->T, src->T, sizeof(double) * L);
    memcpy(dst->dep, src->dep, sizeof(double) * L);
    memcpy(dst->M, src->M, sizeof(double) * L);
    memcpy(dst->sp, src->sp, sizeof(int) * (L + 1));
    memcpy(dst->lo_pre, src->lo_pre, sizeof(int) * (L + 1));
    memcpy(dst->hi_pre, src->hi_pre, sizeof(int) * (L + 1));
    memcpy(dst->lo_suf, src->lo_suf, sizeof(int) * (L + 1));
    memcpy(dst->hi_suf, src->hi_suf, sizeof(int) * (L + 1));
    memcpy(dst->drops_suf, src->drops_suf, sizeof(int) * (L + 1));
    dst->ret = src->ret;
    dst->exit_leg = src->exit_leg;
}

/* insertion.py:68-76 */
static void pass1(ictx_t *X, int v) {
    const int W = X->n + 1;
    route_t *R = &X->r[v];
    double t = 0.0;
    int loc = 0;
    for (int i = 0; i < R->L; ++i) {
        int op = R->seq[i], c = OPC(op);
        t += X->d[loc * W + c];
        loc = c;
        if (!ISP(op)) {
            X->ready[c] = t + X->p[c];
            X->has_ready[c] = 1;
            X->pos_v[c] = v;
            X->pos_i[c] = i;
        }
    }
}

/* insertion.py:78-144 */
static void pass2(ictx_t *X, int v) {
    const int W = X->n + 1, k = X->k;
    route_t *R = &X->r[v];
    int L = R->L;
    for (int g = 0; g <= L; ++g) {
        R->sp[g] = 0; R->lo_pre[g] = 0; R->hi_pre[g] = k;
        R->lo_suf[g] = NEG_BIG; R->hi_suf[g] = POS_BIG; R->drops_suf[g] = 0;
    }
    if (!L) { R->ret = 0.0; R->exit_leg = 0.0; return; }
    double t = 0.0, runmax = 0.0;
    int loc = 0, s = 0, lo = 0, hi = k;
    for (int i = 0; i < L; ++i) {
        int op = R->seq[i], c = OPC(op);
        t += X->d[loc * W + c];
        loc = c;
        R->T[i] = t;
        if (ISP(op)) {
            double base = X->ready[c] - t;
            if (base > runmax) runmax = base;
            int room = k - 1 - s;
            if (room < hi) hi = room;
            s += 1;
        } else {
            int need = 1 - s;
            if (need > lo) lo = need;
            s -= 1;
        }
        R->dep[i] = t + runmax;
        R->sp[i + 1] = s;
        R->lo_pre[i + 1] = lo;
        R->hi_pre[i + 1] = hi;
    }
    double sufmax = -INFINITY;
    int slo = NEG_BIG, shi = POS_BIG, ndrops = 0;
    for (int i = L - 1; i >= 0; --i) {
        int op = R->seq[i], c = OPC(op);
        if (ISP(op)) {
            double base = X->ready[c] - R->T[i];
            if (base > sufmax) sufmax = base;
            int room = k - 1 - R->sp[i];
            if (room < shi) shi = room;
        } else {
            int need = 1 - R->sp[i];
            if (need > slo) slo = need;
            ndrops += 1;
        }
        R->M[i] = sufmax;
        R->lo_suf[i] = slo;
        R->hi_suf[i] = shi;
        R->drops_suf[i] = ndrops;
    }
    R->exit_leg = X->d[OPC(R->seq[L - 1]) * W + 0];
    R->ret = R->dep[L - 1] + R->exit_leg;
}

/* insertion.py:146-156 */
static void refresh(ictx_t *X) {
    double rets[MAXM];
    for (int v = 0; v < X->m; ++v) rets[v] = X->r[v].ret;
    X->sum_ret = orc_py_sum(rets, X->m);
    double top1 = 0.0, top2 = 0.0;
    int arg1 = -1;
    for (int v = 0; v < X->m; ++v) {
        if (rets[v] > top1) { top2 = top1; top1 = rets[v]; arg1 = v; }
        else if (rets[v] > top2) top2 = rets[v];
    }
    for (int v = 0; v < X->m; ++v) X->omax[v] = v == arg1 ? top2 : top1;
}

static void rebuild_all(ictx_t *X) {
    memset(X->has_ready, 0, (size_t)(X->n + 1));
    for (int c = 0; c <= X->n; ++c) { X->pos_v[c] = -1; X->pos_i[c] = -1; X->ready[c] = 0.0; }
    for (int v = 0; v < X->m; ++v) pass1(X, v);
    for (int v = 0; v < X->m; ++v) pass2(X, v);
    refresh(X);
}

static void rebuild_route(ictx_t *X, int v) {
    pass1(X, v);
    pass2(X, v);
    refresh(X);
}

static double cost_of(const ictx_t *X, int v, double new_ret) {
    double other = X->omax[v];
    double mk = new_ret > other ? new_ret : other;
    return mk + 1e-6 * ((X->sum_ret - X->r[v].ret) + new_ret);
}

static int imax3(int a, int b, int c) { int x = a > b ? a : b; return x > c ? x : c; }
static int imin3(int a, int b, int c) { int x = a < b ? a : b; return x < c ? x : c; }

/* insertion.py:193-242; returns count; outputs g, new_ret, stale */
static int eval_gaps(const ictx_t *X, int v, int c, int pick, int min_gap, int *og, double *oret, int *ostale) {
    const int W = X->n + 1, k = X->k;
    const route_t *R = &X->r[v];
    int L = R->L;
    double ready_c = X->has_ready[c] ? X->ready[c] : 0.0;
    if (pick && X->pos_v[c] == v && X->pos_i[c] + 1 > min_gap) min_gap = X->pos_i[c] + 1;
    double t_last = L ? R->T[L - 1] + R->exit_leg : 0.0;
    int cnt = 0;
    for (int g = min_gap; g <= L; ++g) {
        int sp_g = R->sp[g], lo, hi;
        if (!pick) {
            lo = imax3(R->lo_pre[g], 1 - sp_g, R->lo_suf[g] == NEG_BIG ? NEG_BIG : R->lo_suf[g] + 1);
            hi = imin3(R->hi_pre[g], R->hi_suf[g] == POS_BIG ? POS_BIG : R->hi_suf[g] + 1, k);
        } else {
            lo = imax3(R->lo_pre[g], R->lo_suf[g] == NEG_BIG ? NEG_BIG : R->lo_suf[g] - 1, 0);
            hi = imin3(R->hi_pre[g], k - 1 - sp_g, R->hi_suf[g] == POS_BIG ? POS_BIG : R->hi_suf[g] - 1);
        }
        if (lo > hi) continue;
        double prev_dep = g ? R->dep[g - 1] : 0.0;
        int prev_loc = g ? OPC(R->seq[g - 1]) : 0;
        double arr = prev_dep + X->d[prev_loc * W + c];
        double dep_x = (!pick || arr >= ready_c) ? arr : ready_c;
        double new_ret;
        int stale;
        if (g == L) {
            new_ret = dep_x + X->d[c * W + 0];
            stale = 0;
        } else {
            double s_entry = dep_x + X->d[c * W + OPC(R->seq[g])];
            double tail = s_entry - R->T[g];
            double mg = R->M[g];
            new_ret = t_last + (tail > mg ? tail : mg);
            double old_entry = prev_dep + (R->T[g] - (g ? R->T[g - 1] : 0.0));
            stale = s_entry > old_entry + 1e-12 ? R->drops_suf[g] : 0;
        }
        og[cnt] = g; oret[cnt] = new_ret; ostale[cnt] = stale;
        ++cnt;
    }
    return cnt;
}

/* insertion.py:244-272 */
static int eval_pair_gaps(const ictx_t *X, int v, int c, int *og, double *oret, int *ostale) {
    const int W = X->n + 1, k = X->k;
    const route_t *R = &X->r[v];
    int L = R->L, cnt = 0;
    for (int g = 0; g <= L; ++g) {
        int sp_g = R->sp[g];
        int lo = imax3(R->lo_pre[g], R->lo_suf[g], 1 - sp_g);
        int hi = imin3(R->hi_pre[g], R->hi_suf[g], k - sp_g);
        if (lo > hi) continue;
        double prev_dep = g ? R->dep[g - 1] : 0.0;
        int prev_loc = g ? OPC(R->seq[g - 1]) : 0;
        double dep_x = prev_dep + X->d[prev_loc * W + c] + X->p[c];
        double new_ret;
        int stale;
        if (g == L) {
            new_ret = dep_x + X->d[c * W + 0];
            stale = 0;
        } else {
            double s_entry = dep_x + X->d[c * W + OPC(R->seq[g])];
            double tail = s_entry - R->T[g];
            double mg = R->M[g];
            new_ret = R->T[L - 1] + (tail > mg ? tail : mg) + R->exit_leg;
            double old_entry = (g ? R->dep[g - 1] : 0.0) + (R->T[g] - (g ? R->T[g - 1] : 0.0));
            stale = s_entry > old_entry + 1e-12 ? R->drops_suf[g] : 0;
        }
        og[cnt] = g; oret[cnt] = new_ret; ostale[cnt] = stale;
        ++cnt;
    }
    return cnt;
}

/* insertion.py:274-310; over[] sized n+1 scratch */
static double ret_after_drop(const ictx_t *X, int v, int gap, int c, double *over, unsigned char *has_over) {
    const int W = X->n + 1;
    const route_t *R = &X->r[v];
    int L = R->L;
    if (!L) return X->d[0 * W + c] + X->d[c * W + 0];
    memset(has_over, 0, (size_t)(X->n + 1));
    over[c] = 0.0; has_over[c] = 1;
    double t = 0.0;
    int loc = 0;
    for (int j = 0; j <= L; ++j) {
        int cc, isp;
        if (j == gap) { cc = c; isp = 0; }
        else { int op = R->seq[j > gap ? j - 1 : j]; cc = OPC(op); isp = ISP(op); }
        t += X->d[loc * W + cc];
        loc = cc;
        if (!isp) { over[cc] = t + X->p[cc]; has_over[cc] = 1; }
    }
    t = 0.0; loc = 0;
    for (int j = 0; j <= L; ++j) {
        int cc, isp;
        if (j == gap) { cc = c; isp = 0; }
        else { int op = R->seq[j > gap ? j - 1 : j]; cc = OPC(op); isp = ISP(op); }
        t += X->d[loc * W + cc];
        loc = cc;
        if (isp) {
            double r = has_over[cc] ? over[cc] : (X->has_ready[cc] ? X->ready[cc] : 0.0);
            if (r > t) t = r;
        }
    }
    return t + X->d[loc * W + 0];
}

/* ---- key comparisons (tuples) ---- */
typedef struct { double cost; int stale; int a; int b; } key4;  /* (cost, stale, a, b) */

static int key_lt(const key4 *x, const key4 *y) {
    if (x->cost != y->cost) return x->cost < y->cost;
    if (x->stale != y->stale) return x->stale < y->stale;
    if (x->a != y->a) return x->a < y->a;
    return x->b < y->b;
}

/* insertion.py:414-426 on a key list; returns chosen index */
static int pick_windowed(const key4 *keys, int cnt, orc_philox *rng) {
    int best = 0;
    for (int i = 1; i < cnt; ++i) if (key_lt(&keys[i], &keys[best])) best = i;
    if (!rng) return best;  /* first equal to the min (keys are unique here) */
    double limit = keys[best].cost * (1.0 + 0.02) + 1e-12;
    int wcnt = 0;
    for (int i = 0; i < cnt; ++i) if (keys[i].cost <= limit) ++wcnt;
    if (wcnt == 1) {
        for (int i = 0; i < cnt; ++i) if (keys[i].cost <= limit) return i;
    }
    int pick = (int)orc_philox_integers(rng, (uint64_t)wcnt);
    for (int i = 0; i < cnt; ++i)
        if (keys[i].cost <= limit) { if (pick == 0) return i; --pick; }
    return best;
}

typedef struct { double cost; int stale, vd, gd, vp, gp, pair; } option_t;

static int opt_lt(const option_t *x, const option_t *y) {
    if (x->cost != y->cost) return x->cost < y->cost;
    if (x->stale != y->stale) return x->stale < y->stale;
    if (x->vd != y->vd) return x->vd < y->vd;
    return x->gd < y->gd;
}

/* scratch shared by the option search */
typedef struct {
    int *g; double *ret; int *stale;   /* gap lists, capacity 2n+2 */
    key4 *keys;                        /* capacity m*(2n+2) */
    int *pl_a, *pl_b;
    double *over; unsigned char *has_over;
    /* tentative-drop save area */
    route_t saved;
    double *s_ready; unsigned char *s_has; int *s_pv, *s_pi;
} scratch_t;

static void insert_op(route_t *R, int gap, int op) {
    memmove(R->seq + gap + 1, R->seq + gap, sizeof(int) * (R->L - gap));
    R->seq[gap] = op;
    R->L += 1;
}

/* insertion.py:429-472 */
static int customer_options(ictx_t *X, int c, orc_philox *rng, scratch_t *S, option_t *opts) {
    const int m = X->m, n = X->n;
    int nopt = 0;
    for (int vd = 0; vd < m; ++vd) {
        int cnt = eval_gaps(X, vd, c, 0, 0, S->g, S->ret, S->stale);
        if (!cnt) continue;
        /* sort gaps by (cost_of(vd, ret), stale, g): insertion sort (stable) */
        for (int i = 1; i < cnt; ++i) {
            int gg = S->g[i], st = S->stale[i];
            double rr = S->ret[i];
            key4 ki = {cost_of(X, vd, rr), st, gg, 0};
            int j = i - 1;
            while (j >= 0) {
                key4 kj = {cost_of(X, vd, S->ret[j]), S->stale[j], S->g[j], 0};
                if (!key_lt(&ki, &kj)) break;
                S->g[j + 1] = S->g[j]; S->ret[j + 1] = S->ret[j]; S->stale[j + 1] = S->stale[j];
                --j;
            }
            S->g[j + 1] = gg; S->ret[j + 1] = rr; S->stale[j + 1] = st;
        }
        int short_n = cnt < 3 ? cnt : 3;
        key4 dk[3];
        int dg[3];
        for (int i = 0; i < short_n; ++i) {
            int g_drop = S->g[i];
            double r = ret_after_drop(X, vd, g_drop, c, S->over, S->has_over);
            dk[i].cost = cost_of(X, vd, r);
            dk[i].stale = S->stale[i];
            dk[i].a = g_drop;
            dk[i].b = 0;
            dg[i] = g_drop;
        }
        int di = pick_windowed(dk, short_n, rng);
        int d_stale = dk[di].stale, g_drop = dg[di];
        /* tentative_drop (insertion.py:326-338): save, insert, rebuild route vd only */
        route_copy(&S->saved, &X->r[vd]);
        memcpy(S->s_ready, X->ready, sizeof(double) * (n + 1));
        memcpy(S->s_has, X->has_ready, (size_t)(n + 1));
        memcpy(S->s_pv, X->pos_v, sizeof(int) * (n + 1));
        memcpy(S->s_pi, X->pos_i, sizeof(int) * (n + 1));
        double s_sum = X->sum_ret, s_omax[MAXM];
        memcpy(s_omax, X->omax, sizeof(double) * m);
        insert_op(&X->r[vd], g_drop, 2 * (c - 1));
        rebuild_route(X, vd);
        int np = 0;
        for (int vp = 0; vp < m; ++vp) {
            int pc = eval_gaps(X, vp, c, 1, 0, S->g, S->ret, S->stale);
            for (int i = 0; i < pc; ++i) {
                S->keys[np].cost = cost_of(X, vp, S->ret[i]);
                S->keys[np].stale = d_stale + S->stale[i];
                S->keys[np].a = vp;
                S->keys[np].b = S->g[i];
                ++np;
            }
        }
        int pick = np ? pick_windowed(S->keys, np, rng) : -1;
        key4 pk = np ? S->keys[pick] : (key4){0, 0, 0, 0};
        /* restore (insertion.py:340-347) */
        route_copy(&X->r[vd], &S->saved);
        memcpy(X->ready, S->s_ready, sizeof(double) * (n + 1));
        memcpy(X->has_ready, S->s_has, (size_t)(n + 1));
        memcpy(X->pos_v, S->s_pv, sizeof(int) * (n + 1));
        memcpy(X->pos_i, S->s_pi, sizeof(int) * (n + 1));
        X->sum_ret = s_sum;
        memcpy(X->omax, s_omax, sizeof(double) * m);
        if (np) {
            option_t o = {pk.cost, pk.stale, vd, g_drop, pk.a, pk.b, 0};
            opts[nopt++] = o;
        }
    }
    if (!nopt) {
        for (int v = 0; v < m; ++v) {
            int cnt = eval_pair_gaps(X, v, c, S->g, S->ret, S->stale);
            for (int i = 0; i < cnt; ++i) {
                option_t o = {cost_of(X, v, S->ret[i]), S->stale[i], v, S->g[i], v, S->g[i] + 1, 1};
                opts[nopt++] = o;
            }
        }
    }
    /* stable sort by (cost, stale, vd, gd) */
    for (int i = 1; i < nopt; ++i) {
        option_t x = opts[i];
        int j = i - 1;
        while (j >= 0 && opt_lt(&x, &opts[j])) { opts[j + 1] = opts[j]; --j; }
        opts[j + 1] = x;
    }
    return nopt;
}

static void apply_option(ictx_t *X, int c, const option_t *o) {
    if (o->pair) {
        insert_op(&X->r[o->vd], o->gd, 2 * (c - 1) + 1);
        insert_op(&X->r[o->vd], o->gd, 2 * (c - 1));
        rebuild_all(X);
    } else {
        insert_op(&X->r[o->vd], o->gd, 2 * (c - 1));
        rebuild_all(X);
        insert_op(&X->r[o->vp], o->gp, 2 * (c - 1) + 1);
        rebuild_all(X);
    }
}

/* insertion.py:484-516.  ops/lens: partial solution in, repaired out (ops
 * capacity 2n).  removed: customers (any order, duplicates allowed).
 * rng may be NULL (deterministic argmin).  Returns 0 or 1 (RepairFailed). */
int orc_reinsert_all(int32_t n, int32_t m, int32_t k, const double *d, const double *p,
                     int32_t *ops, int32_t *lens, const int32_t *removed, int32_t nremoved,
                     int32_t regret_k, orc_philox *rng) {
    ictx_t X;
    X.n = n; X.m = m; X.k = k; X.d = d; X.p = p;
    const int cap = 2 * n + 2;
    int off = 0;
    for (int v = 0; v < m; ++v) {
        route_alloc(&X.r[v], cap);
        X.r[v].L = lens[v];
        memcpy(X.r[v].seq, ops + off, sizeof(int) * lens[v]);
        off += lens[v];
    }
    X.ready = (double *)calloc((size_t)(n + 1), sizeof(double));
    X.has_ready = (unsigned char *)calloc((size_t)(n + 1), 1);
    X.pos_v = (int *)malloc(sizeof(int) * (n + 1));
    X.pos_i = (int *)malloc(sizeof(int) * (n + 1));
    scratch_t S;
    S.g = (int *)malloc(sizeof(int) * cap);
    S.ret = (double *)malloc(sizeof(double) * cap);
    S.stale = (int *)malloc(sizeof(int) * cap);
    S.keys = (key4 *)malloc(sizeof(key4) * (size_t)m * cap);
    S.over = (double *)malloc(sizeof(double) * (n + 1));
    S.has_over = (unsigned char *)malloc((size_t)(n + 1));
    route_alloc(&S.saved, cap);
    S.s_ready = (double *)malloc(sizeof(double) * (n + 1));
    S.s_has = (unsigned char *)malloc((size_t)(n + 1));
    S.s_pv = (int *)malloc(sizeof(int) * (n + 1));
    S.s_pi = (int *)malloc(sizeof(int) * (n + 1));
    option_t *opts = (option_t *)malloc(sizeof(option_t) * (size_t)m * cap);
    option_t *best_opts = (option_t *)malloc(sizeof(option_t) * (size_t)(n + 1));
    int *remaining = (int *)malloc(sizeof(int) * (size_t)(nremoved > 0 ? nremoved : 1));
    key4 *gk = (key4 *)malloc(sizeof(key4) * (size_t)(nremoved > 0 ? nremoved : 1));
    double *rbuf = (double *)malloc(sizeof(double) * (size_t)m * cap);
    int nrem = 0, status = 0;
    /* sorted(set(removed)) */
    unsigned char *seen = (unsigned char *)calloc((size_t)(n + 1), 1);
    for (int i = 0; i < nremoved; ++i) {
        int c = removed[i];
        if (c >= 1 && c <= n && !seen[c]) { seen[c] = 1; }
    }
    for (int c = 1; c <= n; ++c) if (seen[c]) remaining[nrem++] = c;
    free(seen);

    rebuild_all(&X);
    while (nrem) {
        int chosen_i = -1;
        option_t chosen_opt;
        if (regret_k == 0) {
            for (int i = 0; i < nrem; ++i) {
                int no = customer_options(&X, remaining[i], rng, &S, opts);
                if (!no) { status = 1; goto done; }
                best_opts[i] = opts[0];
                gk[i].cost = opts[0].cost; gk[i].stale = opts[0].stale; gk[i].a = remaining[i]; gk[i].b = 0;
            }
            chosen_i = pick_windowed(gk, nrem, rng);
            chosen_opt = best_opts[chosen_i];
        } else {
            double bk_r = 0, bk_c = 0;
            int bk_s = 0, bk_cust = 0, have = 0;
            for (int i = 0; i < nrem; ++i) {
                int c = remaining[i];
                int no = customer_options(&X, c, rng, &S, opts);
                if (!no) { status = 1; goto done; }
                double regret;
                if (no < regret_k) regret = INFINITY;
                else {
                    double c1 = opts[0].cost;
                    for (int h = 1; h < regret_k; ++h) rbuf[h - 1] = opts[h].cost - c1;
                    regret = orc_py_sum(rbuf, regret_k - 1);
                }
                double nr = -regret;
                /* key (-regret, c1, stale, c) */
                int better = !have || nr < bk_r || (nr == bk_r && (opts[0].cost < bk_c ||
                             (opts[0].cost == bk_c && (opts[0].stale < bk_s ||
                             (opts[0].stale == bk_s && c < bk_cust)))));
                if (better) {
                    have = 1; bk_r = nr; bk_c = opts[0].cost; bk_s = opts[0].stale; bk_cust = c;
                    chosen_i = i; chosen_opt = opts[0];
                }
            }
        }
        apply_option(&X, remaining[chosen_i], &chosen_opt);
        memmove(remaining + chosen_i, remaining + chosen_i + 1, sizeof(int) * (nrem - chosen_i - 1));
        --nrem;
    }
done:
    if (!status) {
        int o = 0;
        for (int v = 0; v < m; ++v) {
            memcpy(ops + o, X.r[v].seq, sizeof(int) * X.r[v].L);
            lens[v] = X.r[v].L;
            o += X.r[v].L;
        }
    }
    for (int v = 0; v < m; ++v) route_free(&X.r[v]);
    route_free(&S.saved);
    free(X.ready); free(X.has_ready); free(X.pos_v); free(X.pos_i);
    free(S.g); free(S.ret); free(S.stale); free(S.keys); free(S.over); free(S.has_over);
    free(S.s_ready); free(S.s_has); free(S.s_pv); free(S.s_pi);
    free(opts); free(best_opts); free(remaining); free(gk); free(rbuf);
    return status;
}

/* insertion.py:358-397: remove both ops of `customers`, cascade capacity
 * casualties; ops/lens rewritten in place, removed_out receives sorted set.
 * Returns the number removed. */
int orc_remove_customers(int32_t n, int32_t m, int32_t k, int32_t *ops, int32_t *lens,
                         const int32_t *customers, int32_t ncust, int32_t *removed_out) {
    unsigned char *rem = (unsigned char *)calloc((size_t)(n + 1), 1);
    for (int i = 0; i < ncust; ++i) if (customers[i] >= 1 && customers[i] <= n) rem[customers[i]] = 1;
    for (;;) {
        /* filter */
        int o = 0, off = 0;
        for (int v = 0; v < m; ++v) {
            int keep = 0;
            for (int i = 0; i < lens[v]; ++i) {
                int op = ops[off + i];
                if (!rem[OPC(op)]) { ops[o + keep] = op; ++keep; }
            }
            off += lens[v];
            lens[v] = keep;
            o += keep;
        }
        /* first capacity break, tours in order */
        int broken = 0;
        off = 0;
        for (int v = 0; v < m && !broken; ++v) {
            int s = 0, lo = 0, hi = k;
            for (int i = 0; i < lens[v]; ++i) {
                int op = ops[off + i];
                if (!ISP(op)) { if (1 - s > lo) lo = 1 - s; s -= 1; }
                else { if (k - 1 - s < hi) hi = k - 1 - s; s += 1; }
                if (lo > hi) { broken = OPC(op); break; }
            }
            off += lens[v];
        }
        if (!broken) break;
        rem[broken] = 1;
    }
    int cnt = 0;
    for (int c = 1; c <= n; ++c) if (rem[c]) removed_out[cnt++] = c;
    free(rem);
    return cnt;
}
