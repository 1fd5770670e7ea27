// repair_team.cuh -- K5 with a CTA (TEAM_WARPS warps) per repair instance:
// insertion.reinsert_all (insertion.py:484-516) with every customer_options
// evaluation of a round running concurrently.
//
// The warp-per-instance K5 (repair_core.cuh) follows customer_options
// (:429-472) literally: for each remaining customer, for each dropoff
// vehicle vd, a D-gap scan, the top-3 re-timing, a windowed draw, a
// tentative drop of route vd, a P-gap scan over every route and a second
// windowed draw -- one warp, serially, q(q+1)/2 customer calls per repair.
// At n = 999 that is ~1.5 M clocks per call on one warp.
//
// Everything in a round except the draws is a deterministic function of the
// round's context, so a round splits into
//   AB (all warps, one (customer, vd) unit at a time, dynamic):
//      D gaps -> shortlist keys -> the drop window (members, no draw); for
//      every window member (only the argmin without an rng) a PRIVATE
//      tentative drop -- route vd rebuilt with c's dropoff in per-warp
//      scratch, the aggregates refreshed privately -- and the P scan over all
//      routes: argmin key, feasible count, pick-window size;
//   C1 (warp 0): the draws in the reference's order (customer -> vd -> drop
//      draw -> pick draw), which need only the window SIZES; stops at the
//      first customer without any option (RepairFailed) exactly where the
//      reference raises;
//   D  (all warps): for each (c, vd) whose pick draw chose a non-argmin
//      member, the private drop again and a scan for that member;
//   C2 (warp 0): per-customer option lists (pair fallback included), the
//      stable sort, the greedy window / regret choice -- the reference's code
//      path with the options already known;
//   E  (all warps): apply_option and rebuild_all with one warp per route.
// Results, and the generator state, are bit-identical to the serial order.
// Integral instances with long routes only (use_scan(): the prefix passes
// are warp scans whose partial sums are exact integers).
#pragma once
#include "repair_core.cuh"
#ifdef VRP_TEAM_TIMERS
#include <cstdio>
#endif

namespace {

// warps per repair CTA: the batched repair kernel (repair.cu) runs 32 (1024
// threads; 64 registers, a few spills, measured 1.3x faster than 16 at
// n = 999), the ALNS iteration kernel 16 (its destroy / replay code spills
// too much at 64 registers: 16 measured 1.2x faster there)
constexpr int TEAM_WARPS = 16;
constexpr int REPAIR_TEAM_WARPS = 32;

// The team path: integral instances with long routes (use_scan) and n >= 72
// (2n >= 24 m at m = 6); VRP_TEAM_MIN_N (compile-time) moves the threshold.
#ifndef VRP_TEAM_MIN_N
#define VRP_TEAM_MIN_N 0
#endif
__host__ __device__ inline bool use_team(const DevInstance &I) { return use_scan(I) && I.n >= VRP_TEAM_MIN_N; }

// One route's pass-2 aggregates, read-only view (InsertionContext._Route).
struct RouteA {
    const int *seq;
    const double *T, *dep, *M;
    const int *sp, *lo_pre, *hi_pre, *lo_suf, *hi_suf, *drops;
    int L;
    double exit_leg;
};

__device__ __forceinline__ RouteA route_of(const Ctx &X, int v) {
    const size_t o = (size_t)v * X.C, o1 = (size_t)v * (X.C + 1);
    return RouteA{X.seq + o, X.T + o, X.dep + o, X.M + o, X.sp + o1, X.lo_pre + o1, X.hi_pre + o1,
                  X.lo_suf + o1, X.hi_suf + o1, X.drops + o1, X.Lr[v], X.exit_leg[v]};
}

// One insertion gap g of a route, packed for the gap scans (three 16-byte
// loads instead of a dozen scattered ones): the terms of insertion.py:193-242
// that do not depend on the inserted customer, and the capacity-interval
// verdicts, which do not either (bit 0: a pickup fits, bit 1: a dropoff fits).
struct __align__(16) GapRec {
    double prev_dep;  // dep[g-1] (0 at g = 0)
    double T;         // T[g] (g < L)
    double M;         // M[g] (g < L)
    double dT;        // T[g] - T[g-1] (the old entry's leg)
    int prev_loc, next_loc, drops, flags;
};

// records of gaps 0..L of one route from its pass-2 arrays (warp-wide)
__device__ void pack_recs(const RouteA &R, int k, int lane, GapRec *out) {
    for (int g = lane; g <= R.L; g += 32) {
        GapRec r;
        const int sp_g = R.sp[g], ls = R.lo_suf[g], hs = R.hi_suf[g], lp = R.lo_pre[g], hp = R.hi_pre[g];
        const int plo = imax3(lp, ls == NEG_BIG ? NEG_BIG : ls - 1, 0);
        const int phi = imin3(hp, k - 1 - sp_g, hs == POS_BIG ? POS_BIG : hs - 1);
        const int dlo = imax3(lp, 1 - sp_g, ls == NEG_BIG ? NEG_BIG : ls + 1);
        const int dhi = imin3(hp, hs == POS_BIG ? POS_BIG : hs + 1, k);
        r.flags = (plo <= phi ? 1 : 0) | (dlo <= dhi ? 2 : 0);
        r.prev_dep = g ? R.dep[g - 1] : 0.0;
        r.prev_loc = g ? opc(R.seq[g - 1]) : 0;
        if (g < R.L) {
            r.T = R.T[g];
            r.M = R.M[g];
            r.dT = R.T[g] - (g ? R.T[g - 1] : 0.0);
            r.next_loc = opc(R.seq[g]);
            r.drops = R.drops[g];
        } else {
            r.T = r.M = r.dT = 0.0;
            r.next_loc = 0;
            r.drops = 0;
        }
        out[g] = r;
    }
}

// gap g from its record: insertion.py:217-241 for a pickup (pick = true, the
// vehicle waits for ready_c) or a dropoff; same operation order as gap_eval.
// base = T[L-1] + exit_leg of the route.
// The customer's two distance rows (integral instances): to_c[x] = d[x][c]
// (the transpose's row c) and from_c[x] = d[c][x].
struct CRows {
    const int32_t *to_c, *from_c;
};

__device__ __forceinline__ CRows crows(const Ctx &X, int c) {
    const size_t o = (size_t)c * X.W;
    return CRows{X.I->d32t + o, X.I->d32 + o};
}

__device__ __forceinline__ bool gap_rec(const CRows &R, const GapRec &r, int g, int L, double base, bool pick,
                                        double ready_c, double &new_ret, int &stale) {
    new_ret = 0.0;
    stale = 0;
    if (!(r.flags & (pick ? 1 : 2))) return false;
    const double arr = r.prev_dep + (double)R.to_c[r.prev_loc];
    const double dep_x = (!pick || arr >= ready_c) ? arr : ready_c;
    if (g == L) {
        new_ret = dep_x + (double)R.from_c[0];
    } else {
        const double s_entry = dep_x + (double)R.from_c[r.next_loc];
        const double tail = s_entry - r.T;
        new_ret = base + (tail > r.M ? tail : r.M);
        const double old_entry = r.prev_dep + r.dT;
        stale = s_entry > old_entry + 1e-12 ? r.drops : 0;
    }
    return true;
}

__device__ __forceinline__ double route_base(const RouteA &R) { return R.L ? R.T[R.L - 1] + R.exit_leg : 0.0; }

// Per-warp scratch (global memory, L1/L2 resident).
struct TeamWS {
    int *gl_g, *gl_stale;
    double *gl_ret;
    Key *keys;
    double *walk, *pcost;
    int *seq;  // the private route: vd with c's dropoff inserted
    double *T, *dep, *M;
    int *sp, *lo_pre, *hi_pre, *lo_suf, *hi_suf, *drops;
    double *aret, *aomax, *asum;  // private aggregates (ret, other-max, sum of returns)
    int *pstart;                  // flat P-gap start of each route [MAXM + 1]
    GapRec *recs;                 // the private route's gap records [C + 1]
    int L;
    double exit_leg, ret, base, ready_c;  // base = T'[L-1] + exit_leg; ready_c = T'[g] + p(c)
};

__host__ __device__ inline size_t team_ws_bytes(int n, int m) {
    const size_t C = 2 * (size_t)n + 2, PF = 2 * (size_t)n + m + 2;
    size_t o = 0;
    auto take = [&](size_t b) { o += al8(b); };
    take(4 * C); take(4 * C); take(8 * C); take(sizeof(Key) * C);
    take(8 * C); take(8 * PF);
    take(4 * C); take(8 * C); take(8 * C); take(8 * C);
    for (int i = 0; i < 6; ++i) take(4 * (C + 1));
    take(8 * MAXM); take(8 * MAXM); take(8);
    take(4 * (MAXM + 1));
    take(sizeof(GapRec) * (C + 1));
    return o;
}

__device__ inline TeamWS bind_ws(unsigned char *b, int n, int m) {
    const size_t C = 2 * (size_t)n + 2, PF = 2 * (size_t)n + m + 2;
    size_t o = 0;
    auto take = [&](size_t bytes) { unsigned char *p = b + o; o += al8(bytes); return p; };
    TeamWS W;
    W.gl_g = (int *)take(4 * C); W.gl_stale = (int *)take(4 * C); W.gl_ret = (double *)take(8 * C);
    W.keys = (Key *)take(sizeof(Key) * C);
    W.walk = (double *)take(8 * C); W.pcost = (double *)take(8 * PF);
    W.seq = (int *)take(4 * C); W.T = (double *)take(8 * C); W.dep = (double *)take(8 * C);
    W.M = (double *)take(8 * C);
    W.sp = (int *)take(4 * (C + 1)); W.lo_pre = (int *)take(4 * (C + 1)); W.hi_pre = (int *)take(4 * (C + 1));
    W.lo_suf = (int *)take(4 * (C + 1)); W.hi_suf = (int *)take(4 * (C + 1)); W.drops = (int *)take(4 * (C + 1));
    W.aret = (double *)take(8 * MAXM); W.aomax = (double *)take(8 * MAXM); W.asum = (double *)take(8);
    W.pstart = (int *)take(4 * (MAXM + 1));
    W.recs = (GapRec *)take(sizeof(GapRec) * (C + 1));
    W.L = 0; W.exit_leg = 0.0; W.ret = 0.0;
    return W;
}

// Per (customer, dropoff vehicle) results of phase AB.
struct UnitRes {
    Key dk[3];     // re-timed shortlist keys (cost, d_stale, g_drop) in shortlist order
    Key pbest[3];  // per shortlist entry: argmin pickup key (cost, stale, vp, gp)
    int ns, dbest, dwin, dmask;
    int np[3], pwin[3], prank[3];
    int4 sum;      // what the draw pass reads, packed for one 16-byte load:
                   // x = ns | dbest << 4 | dwin << 8 | dmask << 12 | (np[j] > 0) << (16 + j);
                   // y, z, w = pwin[j] | prank[j] << 16 (both < 2^16: P gaps <= 2n + m + 2)
};

// Phase C1 decisions per (customer, vd).
struct UnitPick {
    Key pk;     // the chosen pickup key (after phase D when jp >= 0)
    int alt;    // chosen shortlist entry, -1: no dropoff gap on vd
    int jp;     // pending pick-window member index, -1: pk final
    int has;    // an option exists for this vd
    int pad;
};

// Per context route position i (pickups): the ready time the pass-2 walk
// uses (insertion.py:128) and the position of the customer's dropoff when it
// is on the same route (else -1) -- the inputs of a tentative drop's re-walk.
struct TeamCx {
    double *r;
    int *dp;
};

__host__ __device__ inline size_t team_bytes(int n, int m, int nw) {
    const size_t C = 2 * (size_t)n + 2;
    return (size_t)nw * team_ws_bytes(n, m) + al8(sizeof(UnitRes) * (size_t)n * m) +
           al8(sizeof(UnitPick) * (size_t)n * m) + al8(sizeof(GapRec) * (size_t)m * (C + 1)) +
           al8(8 * (size_t)m * C) + al8(4 * (size_t)m * C);
}

// Bind warp `warp`'s view: the context is shared, the scan scratch is the
// warp's own (gl_*, keys, walk), plus the round's unit tables.
__device__ inline TeamWS bind_team(Ctx &X, unsigned char *tb, int n, int m, int warp, int nw, UnitRes *&units,
                                   UnitPick *&picks, GapRec *&crecs, TeamCx &cx) {
    const size_t wsb = team_ws_bytes(n, m);
    TeamWS W = bind_ws(tb + (size_t)warp * wsb, n, m);
    X.gl_g = W.gl_g; X.gl_ret = W.gl_ret; X.gl_stale = W.gl_stale; X.keys = W.keys; X.walk = W.walk;
    unsigned char *q = tb + (size_t)nw * wsb;
    units = (UnitRes *)q;
    q += al8(sizeof(UnitRes) * (size_t)n * m);
    picks = (UnitPick *)q;
    q += al8(sizeof(UnitPick) * (size_t)n * m);
    crecs = (GapRec *)q;  // [m][C + 1]: the context routes' gap records
    q += al8(sizeof(GapRec) * (size_t)m * (2 * n + 3));
    cx.r = (double *)q;
    q += al8(8 * (size_t)m * (2 * n + 2));
    cx.dp = (int *)q;
    return W;
}

// Block-shared control of the team loop.
struct TeamCtl {
    int nrem, st, next, nfail_at, chosen, npend;
};

__device__ __forceinline__ double cost_priv(const TeamWS &W, int v, double new_ret) {
    const double other = W.aomax[v];
    const double mk = new_ret > other ? new_ret : other;
    return mk + 1e-6 * ((*W.asum - W.aret[v]) + new_ret);
}

// A tentative dropoff of c at gap g of route vd (insertion.py:326-338 ->
// rebuild_route(vd), :68-144) seen from the context's pass-2 arrays.  Integral
// instances only (exact integer sums, so any association gives the
// reference's value): inserting c between a and b shifts every later no-wait
// time by delta = d(a,c) + d(c,b) - d(a,b); the ready time of a pickup moves
// by delta too when its dropoff sits on vd at or after g; the load before
// every later op drops by one.  So nothing before g changes, and after g:
//   T'     = T + delta,   sp' = sp - 1,   lo_suf'/hi_suf' = +1,  drops' = drops
//   runmax, lo_pre, hi_pre: prefix scans from g (carried in from g - 1)
//   M (suffix max of ready - T over pickups): a suffix scan from L - 1 to g.
struct DropGeo {
    double T_ins, delta, run0, dep_ins;
    int a, L;
};

__device__ __forceinline__ DropGeo drop_geo(const Ctx &X, int vd, int g, int c) {
    const size_t o = (size_t)vd * X.C;
    const int *sq = X.seq + o;
    const double *T = X.T + o;
    DropGeo G;
    G.L = X.Lr[vd];
    G.a = g ? opc(sq[g - 1]) : 0;
    const double Tp = g ? T[g - 1] : 0.0;
    G.T_ins = Tp + X.d(G.a, c);
    G.delta = g < G.L ? (G.T_ins + X.d(c, opc(sq[g]))) - T[g] : 0.0;
    G.run0 = g ? X.dep[o + g - 1] - Tp : 0.0;
    G.dep_ins = G.T_ins + G.run0;
    return G;
}

// ready - T' of the old op i (>= g) after the insertion; -inf for dropoffs
__device__ __forceinline__ double shifted_base(const Ctx &X, const TeamCx &cx, size_t o, int i, int g, double delta) {
    const int op = X.seq[o + i];
    if (!(op & 1)) return -INFINITY;
    const double r = cx.dp[o + i] >= g ? cx.r[o + i] + delta : cx.r[o + i];
    return r - (X.T[o + i] + delta);
}

// ret_after_drop (insertion.py:274-310) = the tentative route's return
// dep'[L] + exit': one max-reduction over the ops after g
__device__ double rad_fast(const Ctx &X, const TeamCx &cx, int vd, int g, int c) {
    const DropGeo G = drop_geo(X, vd, g, c);
    const size_t o = (size_t)vd * X.C;
    if (g == G.L) return G.dep_ins + X.d(c, 0);
    double sm = -INFINITY;
    for (int i = g + X.lane; i < G.L; i += 32) {
        const double b = shifted_base(X, cx, o, i, g, G.delta);
        sm = b > sm ? b : sm;
    }
    sm = warp_max(sm);
    const double run = sm > G.run0 ? sm : G.run0;
    return ((X.T[o + G.L - 1] + G.delta) + run) + X.d(opc(X.seq[o + G.L - 1]), 0);
}

// the private tentative route's P-gap records g+1 .. L+1, its return and the
// refreshed aggregates (insertion.py:146-156)
__device__ void priv_fast(const Ctx &X, TeamWS &W, const TeamCx &cx, int vd, int g, int c) {
    const int lane = X.lane, k = X.k;
    const DropGeo G = drop_geo(X, vd, g, c);
    const int L = G.L, Lp = L + 1;
    const size_t o = (size_t)vd * X.C, o1 = (size_t)vd * (X.C + 1);
    const int *sq = X.seq + o, *sp = X.sp + o1, *lo_suf = X.lo_suf + o1, *hi_suf = X.hi_suf + o1;
    const int *drops = X.drops + o1;
    const double *T = X.T + o;
    const double delta = G.delta;
    auto sh_lo = [](int x) { return x == NEG_BIG ? NEG_BIG : x + 1; };
    auto sh_hi = [](int x) { return x == POS_BIG ? POS_BIG : x + 1; };
    // suffix max of the shifted bases over old ops i >= g -> W.M[i]
    double csuf = -INFINITY;
    for (int ch = (L - 1 - g) >> 5; ch >= 0 && L > g; --ch) {
        const int i = g + (ch << 5) + lane;
        const bool in = i < L;
        double mx = rscan_max(in ? shifted_base(X, cx, o, i, g, delta) : -INFINITY, lane);
        if (csuf > mx) mx = csuf;
        if (in) W.M[i] = mx;
        csuf = __shfl_sync(VRP_FULL_MASK, mx, 0);
    }
    __syncwarp();
    const int lo0 = imax3(X.lo_pre[o1 + g], 1 - sp[g], NEG_BIG), hi0 = X.hi_pre[o1 + g];
    // the gap right after the new dropoff
    auto write_rec = [&](int Gp, double prev_dep, int prev_loc, double Tprev, int lo_pre, int hi_pre) {
        GapRec r;
        r.prev_dep = prev_dep;
        r.prev_loc = prev_loc;
        const int j = Gp - 1;  // old index of the op after the gap
        int sp_g, ls, hs;
        if (j < L) {
            r.T = T[j] + delta;
            r.M = W.M[j];
            r.dT = r.T - Tprev;
            r.next_loc = opc(sq[j]);
            r.drops = drops[j];
            sp_g = sp[j] - 1; ls = sh_lo(lo_suf[j]); hs = sh_hi(hi_suf[j]);
        } else {
            r.T = r.M = r.dT = 0.0;
            r.next_loc = 0;
            r.drops = 0;
            sp_g = sp[L] - 1; ls = NEG_BIG; hs = POS_BIG;
        }
        const int plo = imax3(lo_pre, ls == NEG_BIG ? NEG_BIG : ls - 1, 0);
        const int phi = imin3(hi_pre, k - 1 - sp_g, hs == POS_BIG ? POS_BIG : hs - 1);
        r.flags = plo <= phi ? 1 : 0;
        W.recs[Gp] = r;
    };
    if (lane == 0) write_rec(g + 1, G.dep_ins, c, G.T_ins, lo0, hi0);
    // prefix scans over old ops i = g .. L-1 -> the records of gaps i + 2
    double crun = G.run0;
    int clo = lo0, chi = hi0;
    double dep_last = G.dep_ins;
    for (int base = g; base < L; base += 32) {
        const int i = base + lane;
        const bool in = i < L;
        const int op = in ? sq[i] : 0;
        const bool isp = in && (op & 1), isd = in && !(op & 1);
        const int spi = in ? sp[i] : 0;
        double run = scan_max(isp ? shifted_base(X, cx, o, i, g, delta) : -INFINITY, lane);
        if (crun > run) run = crun;
        int lo = scan_maxi(isd ? 2 - spi : NEG_BIG, lane);
        if (clo > lo) lo = clo;
        int hi = scan_mini(isp ? k - spi : POS_BIG, lane);
        if (chi < hi) hi = chi;
        if (in) {
            const double Ti = T[i] + delta;
            write_rec(i + 2, Ti + run, opc(op), Ti, lo, hi);
        }
        crun = __shfl_sync(VRP_FULL_MASK, run, 31);
        clo = __shfl_sync(VRP_FULL_MASK, lo, 31);
        chi = __shfl_sync(VRP_FULL_MASK, hi, 31);
    }
    if (L > g) dep_last = (T[L - 1] + delta) + crun;
    __syncwarp();
    const int last = g < L ? opc(sq[L - 1]) : c;
    W.L = Lp;
    W.exit_leg = X.d(last, 0);
    W.base = (g < L ? T[L - 1] + delta : G.T_ins) + W.exit_leg;
    W.ret = dep_last + W.exit_leg;
    W.ready_c = G.T_ins + X.p(c);
    if (lane == 0) {
        for (int v = 0; v < X.m; ++v) W.aret[v] = v == vd ? W.ret : X.ret[v];
        *W.asum = py_sum(W.aret, X.m);
        double top1 = 0.0, top2 = 0.0;
        int arg1 = -1;
        for (int v = 0; v < X.m; ++v) {
            const double r = W.aret[v];
            if (r > top1) { top2 = top1; top1 = r; arg1 = v; }
            else if (r > top2) top2 = r;
        }
        for (int v = 0; v < X.m; ++v) W.aomax[v] = v == arg1 ? top2 : top1;
        int s = 0;
        for (int v = 0; v < X.m; ++v) {
            W.pstart[v] = s;
            const int first = v == vd ? g + 1 : 0;
            const int Lv = v == vd ? Lp : X.Lr[v];
            const int cnt = Lv + 1 - first;
            s += cnt > 0 ? cnt : 0;
        }
        W.pstart[X.m] = s;
    }
    __syncwarp();
}


// The P scan of customer_options after the private drop (insertion.py:456-466),
// in pick_keys_all's flat order (routes ascending, gaps ascending).
//   select < 0: argmin key, feasible count, and (want_win) the pick-window
//               size of _pick_windowed (keys with cost <= best*1.02 + 1e-12)
//   select >= 0: the select-th window member (limit given)
struct PScan {
    Key best;
    int np, win, brank;  // brank: window members before the argmin (flat order)
};

__device__ PScan pscan(const Ctx &X, TeamWS &W, const GapRec *crecs, int vd, int g_drop, int c, int d_stale,
                       bool want_win, int select, double limit) {
    const int lane = X.lane, m = X.m;
    const size_t CR = (size_t)X.C + 1;
    const double ready_c = W.ready_c;
    const double asum = *W.asum;
    const CRows R = crows(X, c);
    Key bk{};
    bool have = false;
    int cnt = 0, seen = 0, F0 = 0;
    PScan out{};
    out.np = 0; out.win = 0; out.brank = 0; out.best = Key{0, 0, -1, -1, 0};
    for (int v = 0; v < m; ++v) {
        const bool priv = v == vd;
        const int L = priv ? W.L : X.Lr[v];
        const int first = priv ? g_drop + 1 : 0;
        const GapRec *rec = priv ? W.recs : crecs + (size_t)v * CR;
        const double base = priv ? W.base : (L ? X.T[(size_t)v * X.C + L - 1] + X.exit_leg[v] : 0.0);
        const double other = W.aomax[v], rest = asum - W.aret[v];
        auto key_at = [&](int g, const GapRec &r, Key &key) -> bool {
            double nr;
            int st;
            if (!gap_rec(R, r, g, L, base, true, ready_c, nr, st)) return false;
            const double mk = nr > other ? nr : other;  // cost_of (insertion.py:188-191)
            key = Key{mk + 1e-6 * (rest + nr), d_stale + st, v, g, 0};
            return true;
        };
        if (select < 0) {
            // chunks of the route (U in flight per iteration; 1 measured best: register pressure)
            constexpr int U = 1;
            for (int g0 = first; g0 <= L; g0 += 32 * U) {
                GapRec rr[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int g = g0 + 32 * u + lane;
                    if (g <= L) rr[u] = rec[g];
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int g = g0 + 32 * u + lane;
                    Key key{};
                    const bool ok = g <= L && key_at(g, rr[u], key);
                    if (want_win && g <= L) W.pcost[F0 + (g - first)] = ok ? key.cost : INFINITY;
                    if (ok && (!have || key_lt(key, bk))) { have = true; bk = key; }
                    cnt += ok;
                }
            }
        } else {
            for (int g0 = first; g0 <= L; g0 += 32) {
                const int g = g0 + lane;
                Key key{};
                const bool ok = g <= L && key_at(g, rec[g], key);
                const bool in = ok && key.cost <= limit;
                const unsigned mk = __ballot_sync(VRP_FULL_MASK, in);
                if (select < seen + __popc(mk)) {
                    unsigned x = mk;
                    for (int r = select - seen; r > 0; --r) x &= x - 1;
                    const int src = __ffs(x) - 1;
                    out.best.cost = __shfl_sync(VRP_FULL_MASK, key.cost, src);
                    out.best.stale = __shfl_sync(VRP_FULL_MASK, key.stale, src);
                    out.best.a = __shfl_sync(VRP_FULL_MASK, key.a, src);
                    out.best.b = __shfl_sync(VRP_FULL_MASK, key.b, src);
                    out.np = 1;
                    return out;
                }
                seen += __popc(mk);
            }
        }
        F0 += L + 1 - first > 0 ? L + 1 - first : 0;
    }
    if (select >= 0) return out;  // not reached for a valid select
    for (int o = 16; o; o >>= 1) {
        const int oh = __shfl_xor_sync(VRP_FULL_MASK, (int)have, o);
        Key ok;
        ok.cost = __shfl_xor_sync(VRP_FULL_MASK, bk.cost, o);
        ok.stale = __shfl_xor_sync(VRP_FULL_MASK, bk.stale, o);
        ok.a = __shfl_xor_sync(VRP_FULL_MASK, bk.a, o);
        ok.b = __shfl_xor_sync(VRP_FULL_MASK, bk.b, o);
        if (oh && (!have || key_lt(ok, bk))) { have = true; bk = ok; }
    }
    out.np = warp_sum(cnt);
    out.best = bk;
    if (want_win && out.np) {
        __syncwarp();
        const double lim = bk.cost * (1.0 + 0.02) + 1e-12;
        const int Fb = W.pstart[bk.a] + (bk.b - (bk.a == vd ? g_drop + 1 : 0));  // the argmin's flat index
        int w = 0, wb = 0;
        for (int F = lane; F < F0; F += 32) {
            const bool in = W.pcost[F] <= lim;
            w += in;
            wb += in && F < Fb;
        }
        out.win = warp_sum(w);
        out.brank = warp_sum(wb);
    }
    return out;
}

#ifdef VRP_TEAM_TIMERS
__device__ long long g_ut[5];
#define VRP_UT(j) do { if (X.lane == 0 && threadIdx.x == 0 && blockIdx.x == 0) { const long long t1 = clock64(); g_ut[j] += t1 - ut0; ut0 = t1; } } while (0)
#else
#define VRP_UT(j) do {} while (0)
#endif

// Phase AB for one (customer c, dropoff vehicle vd): customer_options'
// per-vehicle body (insertion.py:443-465) without the draws.
__device__ void unit_ab(Ctx &X, TeamWS &W, const GapRec *crecs, const TeamCx &cx, int c, int vd, bool use_rng,
                        UnitRes &U) {
    const int lane = X.lane;
#ifdef VRP_TEAM_TIMERS
    long long ut0 = clock64();
    if (X.lane == 0 && threadIdx.x == 0 && blockIdx.x == 0) g_ut[4] += 1;
#endif
    // eval_gaps(vd, c, D) (insertion.py:193-242) from the gap records, keyed
    // (cost_of, stale, g) in gap order into X.keys
    int cnt = 0;
    {
        const int L = X.Lr[vd];
        const GapRec *rec = crecs + (size_t)vd * (X.C + 1);
        const double base = L ? X.T[(size_t)vd * X.C + L - 1] + X.exit_leg[vd] : 0.0;
        const unsigned lt = lanemask_lt();
        const CRows R = crows(X, c);
        for (int g0 = 0; g0 <= L; g0 += 32) {
            const int g = g0 + lane;
            double nr = 0.0;
            int st = 0;
            const bool ok = g <= L && gap_rec(R, rec[g], g, L, base, false, 0.0, nr, st);
            const unsigned mk = __ballot_sync(VRP_FULL_MASK, ok);
            if (ok) X.keys[cnt + __popc(mk & lt)] = Key{cost_of(X, vd, nr), st, g, 0, 0};
            cnt += __popc(mk);
        }
    }
    if (!cnt) {
        if (lane == 0) { U.ns = 0; U.sum = make_int4(0, 0, 0, 0); }
        __syncwarp();
        return;
    }
    __syncwarp();
    const int s0 = warp_argmin(X.keys, cnt, lane);
    const int s1 = cnt > 1 ? warp_argmin(X.keys, cnt, lane, s0) : -1;
    const int s2 = cnt > 2 ? warp_argmin(X.keys, cnt, lane, s0, s1) : -1;
    const int ns = cnt < 3 ? cnt : 3;
    const int sel[3] = {s0, s1, s2};
    VRP_UT(0);
    Key dk[3];
    for (int j = 0; j < ns; ++j) {
        const int gd = X.keys[sel[j]].a, stl = X.keys[sel[j]].stale;
        const double r = rad_fast(X, cx, vd, gd, c);
        dk[j] = Key{cost_of(X, vd, r), stl, gd, 0, 0};
    }
    VRP_UT(1);
    // _pick_windowed over the shortlist: argmin, then the window members
    int best = 0;
    for (int j = 1; j < ns; ++j)
        if (key_lt(dk[j], dk[best])) best = j;
    int mask = 1 << best, wcount = 1;
    if (use_rng) {
        const double lim = dk[best].cost * (1.0 + 0.02) + 1e-12;
        mask = 0; wcount = 0;
        for (int j = 0; j < ns; ++j)
            if (dk[j].cost <= lim) { mask |= 1 << j; ++wcount; }
    }
    if (lane == 0) {
        U.ns = ns; U.dbest = best; U.dwin = wcount; U.dmask = mask;
        for (int j = 0; j < ns; ++j) { U.dk[j] = dk[j]; U.np[j] = 0; U.pwin[j] = 0; }
    }
    for (int j = 0; j < ns; ++j) {
        if (!(mask >> j & 1)) continue;
        priv_fast(X, W, cx, vd, dk[j].a, c);
        VRP_UT(2);
        const PScan ps = pscan(X, W, crecs, vd, dk[j].a, c, dk[j].stale, use_rng, -1, 0.0);
        VRP_UT(3);
        if (lane == 0) { U.np[j] = ps.np; U.pwin[j] = ps.win; U.prank[j] = ps.brank; U.pbest[j] = ps.best; }
        __syncwarp();
    }
    if (lane == 0) {
        int x = ns | best << 4 | wcount << 8 | mask << 12;
        for (int j = 0; j < ns; ++j)
            if ((mask >> j & 1) && U.np[j] > 0) x |= 1 << (16 + j);
        auto pw = [&](int j) { return (mask >> j & 1) ? (U.pwin[j] | U.prank[j] << 16) : 0; };
        U.sum = make_int4(x, pw(0), pw(1), pw(2));
    }
    __syncwarp();
}

// rebuild_all (insertion.py:158-165) with one warp per route
__device__ void rebuild_all_team(Ctx &X, GapRec *crecs, const TeamCx &cx, int warp, int nw) {
    const int tid = warp * 32 + X.lane;
    for (int c = tid; c <= X.n; c += nw * 32) {
        X.has_ready[c] = 0; X.pos_v[c] = -1; X.pos_i[c] = -1; X.ready[c] = 0.0;
    }
    __syncthreads();
    for (int v = warp; v < X.m; v += nw) pass1_warp(X, v);
    __syncthreads();
    for (int v = warp; v < X.m; v += nw) {
        pass2_warp(X, v);
        pack_recs(route_of(X, v), X.k, X.lane, crecs + (size_t)v * (X.C + 1));
        const size_t o = (size_t)v * X.C;
        for (int i = X.lane; i < X.Lr[v]; i += 32) {
            const int op = X.seq[o + i];
            if (!(op & 1)) continue;
            const int cc = opc(op);
            cx.r[o + i] = X.has_ready[cc] ? X.ready[cc] : 0.0;
            cx.dp[o + i] = X.pos_v[cc] == v ? X.pos_i[cc] : -1;
        }
    }
    __syncthreads();
    if (warp == 0 && X.lane == 0) refresh(X);
    __syncthreads();
}

// insertion.py:484-516 on the context's current routes (already rebuilt) and
// X.remaining[0..nrem); called by every warp of the block with the same
// arguments (gen is read only by warp 0, lane 0).  Returns 0 or 1 (RepairFailed).
__device__ int reinsert_team(Ctx &X, TeamWS &W, TeamCtl &T, UnitRes *units, UnitPick *picks, GapRec *crecs,
                             const TeamCx &cx, int nrem_in,
                             int rk, PhiloxGen *gen, bool use_rng, int warp, int nw) {
    const int lane = X.lane, m = X.m;
    if (warp == 0 && lane == 0) { T.nrem = nrem_in; T.st = 0; }
    __syncthreads();
#ifdef VRP_TEAM_TIMERS
    long long tt[6] = {0, 0, 0, 0, 0, 0}, t0 = clock64();
#define VRP_TT(j) do { if (warp == 0 && lane == 0) { const long long t1 = clock64(); tt[j] += t1 - t0; t0 = t1; } } while (0)
#else
#define VRP_TT(j) do {} while (0)
#endif
    while (T.nrem > 0 && !T.st) {
        const int nrem = T.nrem;
        VRP_TT(4);
        // ---- AB: every (customer, vd) unit, dynamically shared out
        if (warp == 0 && lane == 0) T.next = 0;
        __syncthreads();
        for (;;) {
            int u = 0;
            if (lane == 0) u = atomicAdd(&T.next, 1);
            u = __shfl_sync(VRP_FULL_MASK, u, 0);
            if (u >= nrem * m) break;
            const int i = u / m, vd = u - i * m;
            unit_ab(X, W, crecs, cx, X.remaining[i], vd, use_rng, units[u]);
        }
        __syncthreads();
        VRP_TT(0);
        // ---- C1: the draws, in the reference's order.  The warp loads 32 unit
        // summaries at a time; lane 0 walks them in (customer, vd) order via
        // shuffles, draws, and records the decisions.
        if (warp == 0) {
            int fail_at = -1, npend = 0, nopt = 0;
            const int total = nrem * m;
            for (int base = 0; base < total && fail_at < 0; base += 32) {
                const int uu = base + lane;
                const int4 su = uu < total ? units[uu].sum : make_int4(0, 0, 0, 0);
                const int lim = total - base < 32 ? total - base : 32;
                for (int j = 0; j < lim; ++j) {
                    const int x = __shfl_sync(VRP_FULL_MASK, su.x, j);
                    const int pw0 = __shfl_sync(VRP_FULL_MASK, su.y, j);
                    const int pw1 = __shfl_sync(VRP_FULL_MASK, su.z, j);
                    const int pw2 = __shfl_sync(VRP_FULL_MASK, su.w, j);
                    const int u = base + j, vd = u % m;
                    if (lane == 0) {
                        const int ns = x & 15;
                        int alt = -1, jp = -1, has = 0;
                        if (ns) {
                            alt = (x >> 4) & 15;
                            if (use_rng) {
                                const int dwin = (x >> 8) & 15;
                                const int jd = dwin > 1 ? (int)gen->integers((uint32_t)dwin) : 0;
                                unsigned mk = (unsigned)(x >> 12) & 7u;
                                for (int r = jd; r > 0; --r) mk &= mk - 1;
                                alt = __ffs(mk) - 1;
                            }
                            if (x >> (16 + alt) & 1) {
                                has = 1;
                                ++nopt;
                                const int pp = alt == 0 ? pw0 : alt == 1 ? pw1 : pw2;
                                const int pw = pp & 0xFFFF, brank = pp >> 16;
                                if (use_rng && pw > 1) {
                                    jp = (int)gen->integers((uint32_t)pw);
                                    if (jp == brank) jp = -1;  // the draw chose the argmin: no phase-D work
                                    else ++npend;
                                }
                            }
                        }
                        UnitPick &P = picks[u];
                        P.alt = alt; P.jp = jp; P.has = has;
                    }
                    if (vd == m - 1) {  // the customer is complete: pair fallback when it has no option
                        const int any = __shfl_sync(VRP_FULL_MASK, nopt, 0);
                        if (!any) {
                            const int i = u / m;
                            int pairs = 0;
                            for (int v = 0; v < m && !pairs; ++v) pairs = eval_gaps(X, v, X.remaining[i], false, true);
                            if (!pairs) { fail_at = i; break; }
                        }
                        nopt = 0;
                    }
                }
            }
            npend = __shfl_sync(VRP_FULL_MASK, npend, 0);
            if (lane == 0) { T.nfail_at = fail_at; T.npend = npend; T.next = 0; }
        }
        __syncthreads();
        if (T.nfail_at >= 0) {
            if (warp == 0 && lane == 0) T.st = 1;
            __syncthreads();
            break;
        }
        VRP_TT(1);
        // ---- D: the non-argmin pick-window members
        if (T.npend) {
            for (;;) {
                int u = 0;
                if (lane == 0) u = atomicAdd(&T.next, 1);
                u = __shfl_sync(VRP_FULL_MASK, u, 0);
                if (u >= nrem * m) break;
                UnitPick &P = picks[u];
                if (P.jp < 0) continue;
                const UnitRes &U = units[u];
                const int i = u / m, vd = u - i * m, c = X.remaining[i];
                const Key dk = U.dk[P.alt];
                priv_fast(X, W, cx, vd, dk.a, c);
                const double lim = U.pbest[P.alt].cost * (1.0 + 0.02) + 1e-12;
                const PScan ps = pscan(X, W, crecs, vd, dk.a, c, dk.stale, true, P.jp, lim);
                if (lane == 0) P.pk = ps.best;
                __syncwarp();
            }
            __syncthreads();
        }
        VRP_TT(2);
        // ---- C2: option lists, stable sort, greedy window / regret choice
        if (warp == 0) {
            int chosen = -1;
            double bk_r = 0.0, bk_c = 0.0;
            int bk_s = 0, bk_cust = 0;
            bool have = false;
            for (int i = 0; i < nrem; ++i) {
                const int c = X.remaining[i];
                // lane vd gathers its option (the chosen pickup: the argmin, or
                // phase D's window member), compacted in vd order
                bool has = false;
                Opt mine{};
                if (lane < m) {
                    const UnitPick &P = picks[i * m + lane];
                    has = P.has;
                    if (has) {
                        const UnitRes &U = units[i * m + lane];
                        const Key pk = P.jp >= 0 ? P.pk : U.pbest[P.alt];
                        mine = Opt{pk.cost, pk.stale, lane, U.dk[P.alt].a, pk.a, pk.b, 0};
                    }
                }
                const unsigned hm = __ballot_sync(VRP_FULL_MASK, has);
                int nopt = __popc(hm);
                if (has) X.opts[__popc(hm & lanemask_lt())] = mine;
                __syncwarp();
                if (!nopt) {
                    for (int v = 0; v < m; ++v) {
                        const int cnt = eval_gaps(X, v, c, false, true);
                        for (int j = lane; j < cnt; j += 32)
                            X.opts[nopt + j] = Opt{cost_of(X, v, X.gl_ret[j]), X.gl_stale[j], v, X.gl_g[j], v,
                                                   X.gl_g[j] + 1, 1};
                        nopt += cnt;
                        __syncwarp();
                    }
                }
                if (lane == 0 && nopt > 1) {
                    for (int a = 1; a < nopt; ++a) {
                        const Opt x = X.opts[a];
                        int j = a - 1;
                        while (j >= 0 && opt_lt(x, X.opts[j])) { X.opts[j + 1] = X.opts[j]; --j; }
                        X.opts[j + 1] = x;
                    }
                }
                __syncwarp();
                if (rk == 0) {
                    if (lane == 0) X.best[i] = X.opts[0];
                } else if (lane == 0) {
                    double regret;
                    if (nopt < rk) {
                        regret = INFINITY;
                    } else {
                        double buf[MAXM];
                        const double c1 = X.opts[0].cost;
                        for (int h = 1; h < rk; ++h) buf[h - 1] = X.opts[h].cost - c1;
                        regret = py_sum(buf, rk - 1);
                    }
                    const double nr2 = -regret;
                    const Opt &o0 = X.opts[0];
                    const bool better = !have || nr2 < bk_r ||
                        (nr2 == bk_r && (o0.cost < bk_c || (o0.cost == bk_c &&
                         (o0.stale < bk_s || (o0.stale == bk_s && c < bk_cust)))));
                    if (better) {
                        have = true; bk_r = nr2; bk_c = o0.cost; bk_s = o0.stale; bk_cust = c;
                        chosen = i;
                        X.best[nrem] = o0;
                    }
                }
                __syncwarp();
            }
            if (rk == 0) {
                for (int i = lane; i < nrem; i += 32)
                    X.keys[i] = Key{X.best[i].cost, X.best[i].stale, X.remaining[i], 0, 0};
                __syncwarp();
                chosen = pick_windowed(X.keys, nrem, lane, gen, use_rng);
            } else {
                chosen = __shfl_sync(VRP_FULL_MASK, chosen, 0);
            }
            if (lane == 0) T.chosen = chosen;
            // apply_option (insertion.py:475-481): first insertion(s)
            const Opt o = rk == 0 ? X.best[chosen] : X.best[nrem];
            const int c = X.remaining[chosen];
            if (o.pair) {
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1) + 1);
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1));
            } else {
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1));
            }
        }
        __syncthreads();
        VRP_TT(3);
        rebuild_all_team(X, crecs, cx, warp, nw);
        {
            const Opt o = X.best[rk == 0 ? T.chosen : nrem];
            if (!o.pair) {
                if (warp == 0) insert_op_warp(X, o.vp, o.gp, 2 * (X.remaining[T.chosen] - 1) + 1);
                __syncthreads();
                rebuild_all_team(X, crecs, cx, warp, nw);
            }
        }
        if (warp == 0) {
            if (lane == 0) {
                for (int i = T.chosen; i + 1 < nrem; ++i) X.remaining[i] = X.remaining[i + 1];
                T.nrem = nrem - 1;
            }
            __syncwarp();
        }
        __syncthreads();
    }
    VRP_TT(4);
#ifdef VRP_TEAM_TIMERS
    if (warp == 0 && lane == 0 && blockIdx.x == 0)
        printf("team timers (clocks): AB %lld C1 %lld D %lld C2 %lld E %lld | warp0 units: dscan+top3 %lld rad %lld priv %lld pscan %lld n %lld\n",
               tt[0], tt[1], tt[2], tt[3], tt[4], g_ut[0], g_ut[1], g_ut[2], g_ut[3], g_ut[4]);
#endif
    const int st = T.st;
    __syncthreads();
    return st;
}

}  // namespace
