// repair_core.cuh -- the per-instance ALNS repair machinery (insertion.py:52-516)
// shared by K5 (csrc/repair.cu, batched repair) and the device-resident ALNS
// iteration (csrc/alns_step.cu).  One warp owns one instance; see repair.cu
// for the design.
#pragma once
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "philox.cuh"

namespace {


constexpr int NEG_BIG = -(1 << 28);
constexpr int POS_BIG = (1 << 28);
constexpr int MAXM = 32;

struct Key {
    double cost;
    int stale, a, b, pad;
};

struct Opt {
    double cost;
    int stale, vd, gd, vp, gp, pair;
};

__device__ __forceinline__ bool key_lt(const Key &x, const Key &y) {
    if (x.cost != y.cost) return x.cost < y.cost;
    if (x.stale != y.stale) return x.stale < y.stale;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
}

__device__ __forceinline__ bool opt_lt(const Opt &x, const Opt &y) {
    if (x.cost != y.cost) return x.cost < y.cost;
    if (x.stale != y.stale) return x.stale < y.stale;
    if (x.vd != y.vd) return x.vd < y.vd;
    return x.gd < y.gd;
}

__host__ __device__ inline size_t al8(size_t x) { return (x + 15) & ~size_t(15); }

// Scratch layout of one instance (bytes).  C = route capacity = 2n + 2.
struct Layout {
    size_t seq, T, dep, M, sp, lo_pre, hi_pre, lo_suf, hi_suf, drops;  // [m][C] / [m][C+1]
    size_t ret, exit_leg, omax, sum_ret;                                // [m] / 1
    size_t ready, has_ready, pos_v, pos_i;                              // [n+1]
    size_t s_seq, s_T, s_dep, s_M, s_sp, s_lo_pre, s_hi_pre, s_lo_suf, s_hi_suf, s_drops;
    size_t s_misc, s_ready, s_has, s_pv, s_pi;
    size_t gl_g, gl_ret, gl_stale;                                      // gap list [C]
    size_t keys, opts, best, remaining, walk;                           // [m*C] / [n] / 3*[C]
    size_t total;
    int C;
};

__host__ __device__ inline Layout make_layout(int n, int m) {
    Layout L;
    const int C = 2 * n + 2;
    L.C = C;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += al8(bytes); return at; };
    L.seq = take(4ull * m * C);
    L.T = take(8ull * m * C);
    L.dep = take(8ull * m * C);
    L.M = take(8ull * m * C);
    L.sp = take(4ull * m * (C + 1));
    L.lo_pre = take(4ull * m * (C + 1));
    L.hi_pre = take(4ull * m * (C + 1));
    L.lo_suf = take(4ull * m * (C + 1));
    L.hi_suf = take(4ull * m * (C + 1));
    L.drops = take(4ull * m * (C + 1));
    L.ret = take(8ull * m);
    L.exit_leg = take(8ull * m);
    L.omax = take(8ull * m);
    L.sum_ret = take(8);
    L.ready = take(8ull * (n + 1));
    L.has_ready = take(4ull * (n + 1));
    L.pos_v = take(4ull * (n + 1));
    L.pos_i = take(4ull * (n + 1));
    L.s_seq = take(4ull * C);
    L.s_T = take(8ull * C);
    L.s_dep = take(8ull * C);
    L.s_M = take(8ull * C);
    L.s_sp = take(4ull * (C + 1));
    L.s_lo_pre = take(4ull * (C + 1));
    L.s_hi_pre = take(4ull * (C + 1));
    L.s_lo_suf = take(4ull * (C + 1));
    L.s_hi_suf = take(4ull * (C + 1));
    L.s_drops = take(4ull * (C + 1));
    L.s_misc = take(8ull * (2 * m + 4));  // L, ret, exit_leg, sum_ret, omax[m]
    L.s_ready = take(8ull * C);  // per route position (+1 slot for the inserted customer)
    L.s_has = take(4ull * C);
    L.s_pv = take(4ull * C);
    L.s_pi = take(4ull * C);
    L.gl_g = take(4ull * C);
    L.gl_ret = take(8ull * C);
    L.gl_stale = take(4ull * C);
    L.keys = take(sizeof(Key) * (size_t)m * C);
    L.opts = take(sizeof(Opt) * (size_t)m * C);
    L.best = take(sizeof(Opt) * (size_t)(n + 1));
    L.remaining = take(4ull * (n + 1));
    L.walk = take(8ull * 3 * C);
    L.total = o;
    return L;
}

// The warp's view of one instance.
struct Ctx {
    const DevInstance *I;
    int n, m, k, C, W, lane;
    int *seq;
    double *T, *dep, *M;
    int *sp, *lo_pre, *hi_pre, *lo_suf, *hi_suf, *drops;
    int *Lr;  // route lengths (in shared memory, warp-private)
    double *ret, *exit_leg, *omax, *sum_ret;
    double *ready;
    int *has_ready, *pos_v, *pos_i;
    int *s_seq;
    double *s_T, *s_dep, *s_M;
    int *s_sp, *s_lo_pre, *s_hi_pre, *s_lo_suf, *s_hi_suf, *s_drops;
    double *s_misc, *s_ready;
    int *s_has, *s_pv, *s_pi;
    int *gl_g, *gl_stale;
    double *gl_ret;
    Key *keys;
    Opt *opts, *best;
    int *remaining;
    double *walk;
    const double *dm, *pv;  // I->d, I->p
    int pad_;

    __device__ double d(int a, int b) const { return dm[(int64_t)a * W + b]; }
    __device__ double p(int c) const { return pv[c]; }
};

__device__ __forceinline__ int opc(int op) { return (op >> 1) + 1; }

// ---------------------------------------------------------------------------
// Warp-parallel passes for integral instances.  Every quantity the passes
// form -- prefix sums of integer travel times, ready - T, T + runmax -- is an
// exact integer below 2^53, so a tree-ordered scan gives the bit-identical
// double the reference's left-to-right loop does; max/min/int scans are exact
// for any data.  Non-integral instances keep the one-lane loops.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double scan_add(double x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const double y = __shfl_up_sync(VRP_FULL_MASK, x, o); if (lane >= o) x += y; }
    return x;
}
__device__ __forceinline__ double scan_max(double x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const double y = __shfl_up_sync(VRP_FULL_MASK, x, o); if (lane >= o && y > x) x = y; }
    return x;
}
__device__ __forceinline__ int scan_addi(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(VRP_FULL_MASK, x, o); if (lane >= o) x += y; }
    return x;
}
__device__ __forceinline__ int scan_maxi(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(VRP_FULL_MASK, x, o); if (lane >= o && y > x) x = y; }
    return x;
}
__device__ __forceinline__ int scan_mini(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(VRP_FULL_MASK, x, o); if (lane >= o && y < x) x = y; }
    return x;
}
__device__ __forceinline__ double rscan_max(double x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const double y = __shfl_down_sync(VRP_FULL_MASK, x, o); if (lane + o < 32 && y > x) x = y; }
    return x;
}
__device__ __forceinline__ int rscan_addi(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(VRP_FULL_MASK, x, o); if (lane + o < 32) x += y; }
    return x;
}
__device__ __forceinline__ int rscan_maxi(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(VRP_FULL_MASK, x, o); if (lane + o < 32 && y > x) x = y; }
    return x;
}
__device__ __forceinline__ int rscan_mini(int x, int lane) {
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_down_sync(VRP_FULL_MASK, x, o); if (lane + o < 32 && y < x) x = y; }
    return x;
}

// pass1 (insertion.py:68-76), warp-wide
__device__ void pass1_warp(Ctx &X, int v) {
    const int L = X.Lr[v], lane = X.lane;
    const int *sq = X.seq + (size_t)v * X.C;
    double carry = 0.0;
    int cprev = 0;
    for (int base = 0; base < L; base += 32) {
        const int i = base + lane;
        const bool in = i < L;
        const int op = in ? sq[i] : 0, c = opc(op);
        int pc = __shfl_up_sync(VRP_FULL_MASK, c, 1);
        if (lane == 0) pc = cprev;
        const double t = carry + scan_add(in ? X.d(pc, c) : 0.0, lane);
        if (in && !(op & 1)) {
            X.ready[c] = t + X.p(c);
            X.has_ready[c] = 1;
            X.pos_v[c] = v;
            X.pos_i[c] = i;
        }
        carry = __shfl_sync(VRP_FULL_MASK, t, 31);
        cprev = __shfl_sync(VRP_FULL_MASK, c, 31);
    }
}

// pass2 (insertion.py:78-144), warp-wide; the arrays' untouched defaults
// (sp/lo_pre/hi_pre at 0, the suffix arrays at L) are the only init writes
__device__ void pass2_warp(Ctx &X, int v) {
    const int k = X.k, L = X.Lr[v], lane = X.lane;
    const size_t o = (size_t)v * X.C, o1 = (size_t)v * (X.C + 1);
    const int *sq = X.seq + o;
    double *T = X.T + o, *dep = X.dep + o, *M = X.M + o;
    int *sp = X.sp + o1, *lo_pre = X.lo_pre + o1, *hi_pre = X.hi_pre + o1;
    int *lo_suf = X.lo_suf + o1, *hi_suf = X.hi_suf + o1, *drops = X.drops + o1;
    if (lane == 0) {
        sp[0] = 0; lo_pre[0] = 0; hi_pre[0] = k;
        lo_suf[L] = NEG_BIG; hi_suf[L] = POS_BIG; drops[L] = 0;
        if (!L) { X.ret[v] = 0.0; X.exit_leg[v] = 0.0; }
    }
    if (!L) { __syncwarp(); return; }
    double ct = 0.0, crun = 0.0;
    int cs = 0, clo = 0, chi = k, cprev = 0;
    for (int base = 0; base < L; base += 32) {
        const int i = base + lane;
        const bool in = i < L;
        const int op = in ? sq[i] : 0, c = opc(op);
        const bool isp = in && (op & 1), isd = in && !(op & 1);
        int pc = __shfl_up_sync(VRP_FULL_MASK, c, 1);
        if (lane == 0) pc = cprev;
        const double t = ct + scan_add(in ? X.d(pc, c) : 0.0, lane);
        double run = scan_max(isp ? X.ready[c] - t : -INFINITY, lane);
        if (crun > run) run = crun;
        const int delta = isp ? 1 : (isd ? -1 : 0);
        const int s_in = cs + scan_addi(delta, lane), s_bef = s_in - delta;
        int lo = scan_maxi(isd ? 1 - s_bef : NEG_BIG, lane);
        if (clo > lo) lo = clo;
        int hi = scan_mini(isp ? k - 1 - s_bef : POS_BIG, lane);
        if (chi < hi) hi = chi;
        if (in) {
            T[i] = t;
            dep[i] = t + run;
            sp[i + 1] = s_in;
            lo_pre[i + 1] = lo;
            hi_pre[i + 1] = hi;
        }
        ct = __shfl_sync(VRP_FULL_MASK, t, 31);
        crun = __shfl_sync(VRP_FULL_MASK, run, 31);
        cs = __shfl_sync(VRP_FULL_MASK, s_in, 31);
        clo = __shfl_sync(VRP_FULL_MASK, lo, 31);
        chi = __shfl_sync(VRP_FULL_MASK, hi, 31);
        cprev = __shfl_sync(VRP_FULL_MASK, c, 31);
    }
    __syncwarp();
    double csuf = -INFINITY;
    int cslo = NEG_BIG, cshi = POS_BIG, cnd = 0;
    for (int ch = (L - 1) >> 5; ch >= 0; --ch) {
        const int i = (ch << 5) + lane;
        const bool in = i < L;
        const int op = in ? sq[i] : 0, c = opc(op);
        const bool isp = in && (op & 1), isd = in && !(op & 1);
        const int spi = in ? sp[i] : 0;
        double mx = rscan_max(isp ? X.ready[c] - T[i] : -INFINITY, lane);
        if (csuf > mx) mx = csuf;
        int slo = rscan_maxi(isd ? 1 - spi : NEG_BIG, lane);
        if (cslo > slo) slo = cslo;
        int shi = rscan_mini(isp ? k - 1 - spi : POS_BIG, lane);
        if (cshi < shi) shi = cshi;
        const int nd = cnd + rscan_addi(isd ? 1 : 0, lane);
        if (in) {
            M[i] = mx;
            lo_suf[i] = slo;
            hi_suf[i] = shi;
            drops[i] = nd;
        }
        csuf = __shfl_sync(VRP_FULL_MASK, mx, 0);
        cslo = __shfl_sync(VRP_FULL_MASK, slo, 0);
        cshi = __shfl_sync(VRP_FULL_MASK, shi, 0);
        cnd = __shfl_sync(VRP_FULL_MASK, nd, 0);
    }
    __syncwarp();
    if (lane == 0) {
        X.exit_leg[v] = X.d(opc(sq[L - 1]), 0);
        X.ret[v] = dep[L - 1] + X.exit_leg[v];
    }
    __syncwarp();
}

// insert_op, warp-wide: shift [gap, L) up by one, chunks from the end
__device__ void insert_op_warp(Ctx &X, int v, int gap, int op) {
    int *sq = X.seq + (size_t)v * X.C;
    const int L = X.Lr[v];
    for (int hi = L; hi > gap; hi -= 32) {
        const int i = hi - X.lane;
        const bool in = i > gap;
        const int val = in ? sq[i - 1] : 0;
        __syncwarp();
        if (in) sq[i] = val;
        __syncwarp();
    }
    if (X.lane == 0) {
        sq[gap] = op;
        X.Lr[v] = L + 1;
    }
    __syncwarp();
}

// ret_after_drop (insertion.py:274-310), warp-wide: walk 1 is a prefix sum;
// walk 2's t = max(t + d, r) unrolls to max(D_L, max_j (r_j - D_j) + D_L)
__device__ double ret_after_drop_warp(const Ctx &X, int v, int gap, int c) {
    const int L = X.Lr[v], lane = X.lane;
    if (!L) return X.d(0, c) + X.d(c, 0);
    const int *sq = X.seq + (size_t)v * X.C;
    double *w = X.walk;
    double carry = 0.0;
    int cprev = 0;
    for (int base = 0; base <= L; base += 32) {
        const int j = base + lane;
        const bool in = j <= L;
        const int cc = in ? (j == gap ? c : opc(sq[j > gap ? j - 1 : j])) : 0;
        int pc = __shfl_up_sync(VRP_FULL_MASK, cc, 1);
        if (lane == 0) pc = cprev;
        const double t = carry + scan_add(in ? X.d(pc, cc) : 0.0, lane);
        if (in) w[j] = t;
        carry = __shfl_sync(VRP_FULL_MASK, t, 31);
        cprev = __shfl_sync(VRP_FULL_MASK, cc, 31);
    }
    __syncwarp();
    double xm = -INFINITY;
    for (int j = lane; j <= L; j += 32) {
        if (j == gap) continue;
        const int op = sq[j > gap ? j - 1 : j];
        if (!(op & 1)) continue;
        const int cc = opc(op);
        double r;
        if (X.pos_v[cc] == v) {
            const int di = X.pos_i[cc] + (X.pos_i[cc] >= gap ? 1 : 0);
            r = w[di] + X.p(cc);
        } else {
            r = X.has_ready[cc] ? X.ready[cc] : 0.0;
        }
        const double val = r - w[j];
        if (val > xm) xm = val;
    }
    xm = warp_max(xm);
    const double DL = w[L];
    const int last = L == gap ? c : opc(sq[L - 1]);
    const double t = xm > 0.0 ? DL + xm : DL;
    __syncwarp();
    return t + X.d(last, 0);
}

// insertion.py:68-76 (one lane)
__device__ void pass1(Ctx &X, int v) {
    const int *sq = X.seq + (size_t)v * X.C;
    double t = 0.0;
    int loc = 0;
    for (int i = 0; i < X.Lr[v]; ++i) {
        const int op = sq[i], c = opc(op);
        t += X.d(loc, c);
        loc = c;
        if (!(op & 1)) {
            X.ready[c] = t + X.p(c);
            X.has_ready[c] = 1;
            X.pos_v[c] = v;
            X.pos_i[c] = i;
        }
    }
}

// insertion.py:78-144 (one lane)
__device__ void pass2(Ctx &X, int v) {
    const int k = X.k, L = X.Lr[v];
    const size_t o = (size_t)v * X.C, o1 = (size_t)v * (X.C + 1);
    const int *sq = X.seq + o;
    double *T = X.T + o, *dep = X.dep + o, *M = X.M + o;
    int *sp = X.sp + o1, *lo_pre = X.lo_pre + o1, *hi_pre = X.hi_pre + o1;
    int *lo_suf = X.lo_suf + o1, *hi_suf = X.hi_suf + o1, *drops = X.drops + o1;
    for (int g = 0; g <= L; ++g) {
        sp[g] = 0; lo_pre[g] = 0; hi_pre[g] = k;
        lo_suf[g] = NEG_BIG; hi_suf[g] = POS_BIG; drops[g] = 0;
    }
    if (!L) { X.ret[v] = 0.0; X.exit_leg[v] = 0.0; return; }
    double t = 0.0, runmax = 0.0;
    int loc = 0, s = 0, lo = 0, hi = k;
    for (int i = 0; i < L; ++i) {
        const int op = sq[i], c = opc(op);
        t += X.d(loc, c);
        loc = c;
        T[i] = t;
        if (op & 1) {
            const double base = X.ready[c] - t;
            if (base > runmax) runmax = base;
            const int room = k - 1 - s;
            if (room < hi) hi = room;
            s += 1;
        } else {
            const int need = 1 - s;
            if (need > lo) lo = need;
            s -= 1;
        }
        dep[i] = t + runmax;
        sp[i + 1] = s;
        lo_pre[i + 1] = lo;
        hi_pre[i + 1] = hi;
    }
    double sufmax = -INFINITY;
    int slo = NEG_BIG, shi = POS_BIG, nd = 0;
    for (int i = L - 1; i >= 0; --i) {
        const int op = sq[i], c = opc(op);
        if (op & 1) {
            const double base = X.ready[c] - T[i];
            if (base > sufmax) sufmax = base;
            const int room = k - 1 - sp[i];
            if (room < shi) shi = room;
        } else {
            const int need = 1 - sp[i];
            if (need > slo) slo = need;
            nd += 1;
        }
        M[i] = sufmax;
        lo_suf[i] = slo;
        hi_suf[i] = shi;
        drops[i] = nd;
    }
    X.exit_leg[v] = X.d(opc(sq[L - 1]), 0);
    X.ret[v] = dep[L - 1] + X.exit_leg[v];
}

// CPython 3.12 sum() over floats (Neumaier), int start 0
__device__ double py_sum(const double *x, int cnt) {
    if (cnt <= 0) return 0.0;
    double f = x[0], c = 0.0;
    for (int i = 1; i < cnt; ++i) {
        const double t = f + x[i];
        if (fabs(f) >= fabs(x[i])) c += (f - t) + x[i];
        else c += (x[i] - t) + f;
        f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    return f;
}

// insertion.py:146-156 (one lane)
__device__ void refresh(Ctx &X) {
    *X.sum_ret = py_sum(X.ret, X.m);
    double top1 = 0.0, top2 = 0.0;
    int arg1 = -1;
    for (int v = 0; v < X.m; ++v) {
        const double r = X.ret[v];
        if (r > top1) { top2 = top1; top1 = r; arg1 = v; }
        else if (r > top2) top2 = r;
    }
    for (int v = 0; v < X.m; ++v) X.omax[v] = v == arg1 ? top2 : top1;
}

template <bool SCAN>
__device__ void rebuild_all(Ctx &X) {
    for (int c = X.lane; c <= X.n; c += 32) {
        X.has_ready[c] = 0; X.pos_v[c] = -1; X.pos_i[c] = -1; X.ready[c] = 0.0;
    }
    __syncwarp();
    if (SCAN) {
        for (int v = 0; v < X.m; ++v) pass1_warp(X, v);
        __syncwarp();
        for (int v = 0; v < X.m; ++v) pass2_warp(X, v);
    } else {
        for (int v = X.lane; v < X.m; v += 32) pass1(X, v);
        __syncwarp();
        for (int v = X.lane; v < X.m; v += 32) pass2(X, v);
    }
    __syncwarp();
    if (X.lane == 0) refresh(X);
    __syncwarp();
}

__device__ __forceinline__ double cost_of(const Ctx &X, int v, double new_ret) {
    const double other = X.omax[v];
    const double mk = new_ret > other ? new_ret : other;
    return mk + 1e-6 * ((*X.sum_ret - X.ret[v]) + new_ret);
}

__device__ __forceinline__ int imax3(int a, int b, int c) { int x = a > b ? a : b; return x > c ? x : c; }
__device__ __forceinline__ int imin3(int a, int b, int c) { int x = a < b ? a : b; return x < c ? x : c; }

// One insertion gap g of route v for customer c (insertion.py:193-272):
// capacity interval, new return and stale count.  Returns feasibility.
__device__ __forceinline__ bool gap_eval(const Ctx &X, int v, int g, int c, bool pick, bool pair, double ready_c,
                                         double &new_ret, int &stale) {
    const int k = X.k, L = X.Lr[v];
    const size_t o = (size_t)v * X.C, o1 = (size_t)v * (X.C + 1);
    const int *sq = X.seq + o;
    const double *T = X.T + o;
    const int sp_g = X.sp[o1 + g];
    const int ls = X.lo_suf[o1 + g], hs = X.hi_suf[o1 + g];
    const int lp = X.lo_pre[o1 + g], hp = X.hi_pre[o1 + g];
    int lo, hi;
    if (pair) {
        lo = imax3(lp, ls, 1 - sp_g);
        hi = imin3(hp, hs, k - sp_g);
    } else if (!pick) {
        lo = imax3(lp, 1 - sp_g, ls == NEG_BIG ? NEG_BIG : ls + 1);
        hi = imin3(hp, hs == POS_BIG ? POS_BIG : hs + 1, k);
    } else {
        lo = imax3(lp, ls == NEG_BIG ? NEG_BIG : ls - 1, 0);
        hi = imin3(hp, k - 1 - sp_g, hs == POS_BIG ? POS_BIG : hs - 1);
    }
    new_ret = 0.0;
    stale = 0;
    if (lo > hi) return false;
    const double prev_dep = g ? X.dep[o + g - 1] : 0.0;
    const int prev_loc = g ? opc(sq[g - 1]) : 0;
    double dep_x;
    if (pair) {
        dep_x = prev_dep + X.d(prev_loc, c) + X.p(c);
    } else {
        const double arr = prev_dep + X.d(prev_loc, c);
        dep_x = (!pick || arr >= ready_c) ? arr : ready_c;
    }
    if (g == L) {
        new_ret = dep_x + X.d(c, 0);
    } else {
        const double s_entry = dep_x + X.d(c, opc(sq[g]));
        const double tail = s_entry - T[g];
        const double mg = X.M[o + g];
        if (pair) new_ret = T[L - 1] + (tail > mg ? tail : mg) + X.exit_leg[v];
        else new_ret = (T[L - 1] + X.exit_leg[v]) + (tail > mg ? tail : mg);
        const double old_entry = prev_dep + (T[g] - (g ? T[g - 1] : 0.0));
        stale = s_entry > old_entry + 1e-12 ? X.drops[o1 + g] : 0;
    }
    return true;
}

// insertion.py:193-242 (pair = false) and :244-272 (pair = true); warp-wide,
// one gap per lane, compacted in gap order into gl_*; returns the count.
__device__ int eval_gaps(Ctx &X, int v, int c, bool pick, bool pair) {
    const int L = X.Lr[v];
    const double ready_c = X.has_ready[c] ? X.ready[c] : 0.0;
    int min_gap = 0;
    if (pick && X.pos_v[c] == v && X.pos_i[c] + 1 > min_gap) min_gap = X.pos_i[c] + 1;
    const unsigned lt = lanemask_lt();
    int cnt = 0;
    for (int base = min_gap; base <= L; base += 32) {
        const int g = base + X.lane;
        double new_ret = 0.0;
        int stale = 0;
        const bool ok = g <= L && gap_eval(X, v, g, c, pick, pair, ready_c, new_ret, stale);
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, ok);
        if (ok) {
            const int at = cnt + __popc(mk & lt);
            X.gl_g[at] = g;
            X.gl_ret[at] = new_ret;
            X.gl_stale[at] = stale;
        }
        cnt += __popc(mk);
    }
    __syncwarp();
    return cnt;
}

// The pickup gaps of every route in one warp pass (the P scan of a
// tentative drop, insertion.py:456-466): flat gap index over the routes in
// order, gaps ascending -- the order of m eval_gaps calls -- keyed straight
// into keys[0..): (cost, d_stale + stale, vp, g).  Returns the count.
__device__ int pick_keys_all(Ctx &X, int c, int d_stale) {
    const int m = X.m, lane = X.lane;
    int first = 0, cntv = 0;
    if (lane < m) {
        first = X.pos_v[c] == lane ? X.pos_i[c] + 1 : 0;
        cntv = X.Lr[lane] + 1 - first;
        if (cntv < 0) cntv = 0;
    }
    int ex = cntv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(VRP_FULL_MASK, ex, o);
        if (lane >= o) ex += y;
    }
    const int total = __shfl_sync(VRP_FULL_MASK, ex, m - 1);
    ex -= cntv;  // exclusive start of route `lane`
    const double ready_c = X.has_ready[c] ? X.ready[c] : 0.0;
    const unsigned lt = lanemask_lt();
    int np = 0;
    for (int base = 0; base < total; base += 32) {
        const int F = base + lane;
        int v = 0;
        for (int u = 1; u < m; ++u) {  // the route holding flat gap F
            const int eu = __shfl_sync(VRP_FULL_MASK, ex, u);
            const int cu = __shfl_sync(VRP_FULL_MASK, cntv, u);
            if (cu > 0 && F >= eu) v = u;
        }
        const int g = __shfl_sync(VRP_FULL_MASK, first, v) + (F - __shfl_sync(VRP_FULL_MASK, ex, v));
        double new_ret = 0.0;
        int stale = 0;
        const bool ok = F < total && gap_eval(X, v, g, c, true, false, ready_c, new_ret, stale);
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, ok);
        if (ok) X.keys[np + __popc(mk & lt)] = Key{cost_of(X, v, new_ret), d_stale + stale, v, g, 0};
        np += __popc(mk);
    }
    __syncwarp();
    return np;
}

// warp argmin of keys[0..cnt), excluding indices in `skip` (up to 3)
__device__ int warp_argmin(const Key *keys, int cnt, int lane, int s0 = -1, int s1 = -1) {
    int bi = -1;
    Key bk{};
    for (int i = lane; i < cnt; i += 32) {
        if (i == s0 || i == s1) continue;
        if (bi < 0 || key_lt(keys[i], bk)) { bi = i; bk = keys[i]; }
    }
    for (int o = 16; o; o >>= 1) {
        const int oi = __shfl_xor_sync(VRP_FULL_MASK, bi, o);
        Key ok;
        ok.cost = __shfl_xor_sync(VRP_FULL_MASK, bk.cost, o);
        ok.stale = __shfl_xor_sync(VRP_FULL_MASK, bk.stale, o);
        ok.a = __shfl_xor_sync(VRP_FULL_MASK, bk.a, o);
        ok.b = __shfl_xor_sync(VRP_FULL_MASK, bk.b, o);
        if (oi >= 0 && (bi < 0 || key_lt(ok, bk))) { bi = oi; bk = ok; }
    }
    return bi;
}

// insertion.py:414-426: returns the chosen index (warp-uniform); lane 0 draws
__device__ int pick_windowed(const Key *keys, int cnt, int lane, PhiloxGen *gen, bool use_rng) {
    const int best = warp_argmin(keys, cnt, lane);
    if (!use_rng) return best;
    const double limit = keys[best].cost * (1.0 + 0.02) + 1e-12;
    const unsigned lt = lanemask_lt();
    int wcnt = 0;
    for (int base = 0; base < cnt; base += 32) {
        const int i = base + lane;
        wcnt += __popc(__ballot_sync(VRP_FULL_MASK, i < cnt && keys[i].cost <= limit));
    }
    int j = 0;
    if (wcnt > 1) {
        if (lane == 0) j = (int)gen->integers((uint32_t)wcnt);
        j = __shfl_sync(VRP_FULL_MASK, j, 0);
    }
    int seen = 0;
    for (int base = 0; base < cnt; base += 32) {
        const int i = base + lane;
        const bool in = i < cnt && keys[i].cost <= limit;
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, in);
        if (j < seen + __popc(mk)) {
            const unsigned want = mk;
            // the (j - seen)-th set bit
            unsigned x = want;
#pragma unroll 1
            for (int r = j - seen; r > 0; --r) x &= x - 1;
            return base + __ffs(x) - 1;
        }
        seen += __popc(mk);
    }
    return best;
}

// insertion.py:274-310, walk on one lane; t1 = scratch of C doubles
__device__ double ret_after_drop(const Ctx &X, int v, int gap, int c, double *t1) {
    const int L = X.Lr[v];
    if (!L) return X.d(0, c) + X.d(c, 0);
    const int *sq = X.seq + (size_t)v * X.C;
    double t = 0.0;
    int loc = 0;
    for (int j = 0; j <= L; ++j) {
        const int cc = j == gap ? c : opc(sq[j > gap ? j - 1 : j]);
        t += X.d(loc, cc);
        loc = cc;
        t1[j] = t;
    }
    t = 0.0;
    loc = 0;
    for (int j = 0; j <= L; ++j) {
        int cc, isp;
        if (j == gap) { cc = c; isp = 0; }
        else { const int op = sq[j > gap ? j - 1 : j]; cc = opc(op); isp = op & 1; }
        t += X.d(loc, cc);
        loc = cc;
        if (isp) {
            double r;
            if (X.pos_v[cc] == v) {  // its dropoff is on this route: pass-1 time there
                const int di = X.pos_i[cc] + (X.pos_i[cc] >= gap ? 1 : 0);
                r = t1[di] + X.p(cc);
            } else {
                r = X.has_ready[cc] ? X.ready[cc] : 0.0;
            }
            if (r > t) t = r;
        }
    }
    return t + X.d(loc, 0);
}

__device__ void insert_op(Ctx &X, int v, int gap, int op) {  // one lane
    int *sq = X.seq + (size_t)v * X.C;
    for (int i = X.Lr[v]; i > gap; --i) sq[i] = sq[i - 1];
    sq[gap] = op;
    X.Lr[v] += 1;
}

// tentative_drop save / restore (insertion.py:326-347), warp-wide copies.
// pass1 on route v only rewrites the per-customer entries of v's dropoffs and
// of the inserted customer c, so only those are saved (by route position; c
// at position L) -- O(L) instead of O(n) per tentative drop.
template <bool SAVE>
__device__ void swap_state(Ctx &X, int v, int c) {
    const int L = SAVE ? X.Lr[v] : (int)X.s_misc[0];
    const size_t o = (size_t)v * X.C, o1 = (size_t)v * (X.C + 1);
    for (int i = X.lane; i <= L; i += 32) {
        if (i < L) {
            if (SAVE) { X.s_seq[i] = X.seq[o + i]; X.s_T[i] = X.T[o + i]; X.s_dep[i] = X.dep[o + i]; X.s_M[i] = X.M[o + i]; }
            else { X.seq[o + i] = X.s_seq[i]; X.T[o + i] = X.s_T[i]; X.dep[o + i] = X.s_dep[i]; X.M[o + i] = X.s_M[i]; }
        }
        if (SAVE) {
            X.s_sp[i] = X.sp[o1 + i]; X.s_lo_pre[i] = X.lo_pre[o1 + i]; X.s_hi_pre[i] = X.hi_pre[o1 + i];
            X.s_lo_suf[i] = X.lo_suf[o1 + i]; X.s_hi_suf[i] = X.hi_suf[o1 + i]; X.s_drops[i] = X.drops[o1 + i];
        } else {
            X.sp[o1 + i] = X.s_sp[i]; X.lo_pre[o1 + i] = X.s_lo_pre[i]; X.hi_pre[o1 + i] = X.s_hi_pre[i];
            X.lo_suf[o1 + i] = X.s_lo_suf[i]; X.hi_suf[o1 + i] = X.s_hi_suf[i]; X.drops[o1 + i] = X.s_drops[i];
        }
    }
    for (int i = X.lane; i <= L; i += 32) {
        int cu;
        if (i < L) {
            const int op = SAVE ? X.seq[o + i] : X.s_seq[i];
            if (op & 1) continue;
            cu = opc(op);
        } else {
            cu = c;
        }
        if (SAVE) { X.s_ready[i] = X.ready[cu]; X.s_has[i] = X.has_ready[cu]; X.s_pv[i] = X.pos_v[cu]; X.s_pi[i] = X.pos_i[cu]; }
        else { X.ready[cu] = X.s_ready[i]; X.has_ready[cu] = X.s_has[i]; X.pos_v[cu] = X.s_pv[i]; X.pos_i[cu] = X.s_pi[i]; }
    }
    if (X.lane == 0) {
        if (SAVE) {
            X.s_misc[0] = (double)X.Lr[v]; X.s_misc[1] = X.ret[v]; X.s_misc[2] = X.exit_leg[v];
            X.s_misc[3] = *X.sum_ret;
            for (int u = 0; u < X.m; ++u) X.s_misc[4 + u] = X.omax[u];
        } else {
            X.Lr[v] = (int)X.s_misc[0]; X.ret[v] = X.s_misc[1]; X.exit_leg[v] = X.s_misc[2];
            *X.sum_ret = X.s_misc[3];
            for (int u = 0; u < X.m; ++u) X.omax[u] = X.s_misc[4 + u];
        }
    }
    __syncwarp();
}

// insertion.py:429-472; options in X.opts, returns the count (warp-uniform)
template <bool SCAN>
__device__ int customer_options(Ctx &X, int c, PhiloxGen *gen, bool use_rng) {
    const int m = X.m, lane = X.lane;
    int nopt = 0;
    for (int vd = 0; vd < m; ++vd) {
        const int cnt = eval_gaps(X, vd, c, false, false);
        if (!cnt) continue;
        // top 3 by (cost_of(vd, ret), stale, g): keys into X.keys
        for (int i = lane; i < cnt; i += 32)
            X.keys[i] = Key{cost_of(X, vd, X.gl_ret[i]), X.gl_stale[i], X.gl_g[i], 0, 0};
        __syncwarp();
        const int s0 = warp_argmin(X.keys, cnt, lane);
        const int s1 = cnt > 1 ? warp_argmin(X.keys, cnt, lane, s0) : -1;
        const int s2 = cnt > 2 ? warp_argmin(X.keys, cnt, lane, s0, s1) : -1;
        const int ns = cnt < 3 ? cnt : 3;
        const int sel[3] = {s0, s1, s2};
        // re-score the shortlist exactly, one lane each; drop keys -> keys[cnt..cnt+3)
        Key dk = Key{0, 0, 0, 0, 0};
        if (SCAN) {
            for (int j = 0; j < ns; ++j) {
                const int si = sel[j];
                const int gd = X.keys[si].a, stl = X.keys[si].stale;
                const double r = ret_after_drop_warp(X, vd, gd, c);
                if (lane == j) dk = Key{cost_of(X, vd, r), stl, gd, 0, 0};
            }
        } else if (lane < ns) {
            const int si = sel[lane];
            const int g_drop = X.keys[si].a;
            const double r = ret_after_drop(X, vd, g_drop, c, X.walk + (size_t)lane * X.C);
            dk = Key{cost_of(X, vd, r), X.keys[si].stale, g_drop, 0, 0};
        }
        __syncwarp();
        if (lane < ns) X.keys[lane] = dk;  // shortlist order = the sorted order
        __syncwarp();
        const int di = pick_windowed(X.keys, ns, lane, gen, use_rng);
        const int d_stale = X.keys[di].stale, g_drop = X.keys[di].a;
        __syncwarp();
        // tentative_drop: save, insert D, rebuild route vd only
        swap_state<true>(X, vd, c);
        if (SCAN) {
            insert_op_warp(X, vd, g_drop, 2 * (c - 1));
            pass1_warp(X, vd);
            __syncwarp();
            pass2_warp(X, vd);
            if (lane == 0) refresh(X);
        } else if (lane == 0) {
            insert_op(X, vd, g_drop, 2 * (c - 1));
            pass1(X, vd);
            pass2(X, vd);
            refresh(X);
        }
        __syncwarp();
        const int np = pick_keys_all(X, c, d_stale);
        Key pk{};
        if (np) {
            const int pi = pick_windowed(X.keys, np, lane, gen, use_rng);
            pk = X.keys[pi];
        }
        __syncwarp();
        swap_state<false>(X, vd, c);  // restore
        if (np) {
            if (lane == 0) X.opts[nopt] = Opt{pk.cost, pk.stale, vd, g_drop, pk.a, pk.b, 0};
            ++nopt;
        }
        __syncwarp();
    }
    if (!nopt) {
        for (int v = 0; v < m; ++v) {
            const int cnt = eval_gaps(X, v, c, false, true);
            for (int i = lane; i < cnt; i += 32)
                X.opts[nopt + i] = Opt{cost_of(X, v, X.gl_ret[i]), X.gl_stale[i], v, X.gl_g[i], v,
                                       X.gl_g[i] + 1, 1};
            nopt += cnt;
            __syncwarp();
        }
    }
    if (lane == 0 && nopt > 1) {  // stable sort by (cost, stale, vd, gd)
        for (int i = 1; i < nopt; ++i) {
            const Opt x = X.opts[i];
            int j = i - 1;
            while (j >= 0 && opt_lt(x, X.opts[j])) { X.opts[j + 1] = X.opts[j]; --j; }
            X.opts[j + 1] = x;
        }
    }
    __syncwarp();
    return nopt;
}


// Warp-scan passes (SCAN = true) need an integral instance (every partial sum
// an exact integer) and pay off once routes are long enough: 2n/m >= 24
// (measured: eil51's ~17-op routes run faster with the one-lane loops, whose
// compact code also suits the instruction cache when 8 warps share an SM).
__host__ __device__ inline bool use_scan(const DevInstance &I) { return I.integral && 2 * I.n >= 24 * I.m; }

// Bind a Ctx to one instance's scratch block `b` (make_layout(n, m) bytes).
__device__ __forceinline__ void bind_ctx(Ctx &X, const DevInstance *I, unsigned char *b, int *Lr, int lane) {
    const Layout Ly = make_layout(I->n, I->m);
    X.I = I; X.n = I->n; X.m = I->m; X.k = I->k; X.C = Ly.C; X.W = I->W; X.lane = lane;
    X.seq = (int *)(b + Ly.seq); X.T = (double *)(b + Ly.T); X.dep = (double *)(b + Ly.dep);
    X.M = (double *)(b + Ly.M); X.sp = (int *)(b + Ly.sp); X.lo_pre = (int *)(b + Ly.lo_pre);
    X.hi_pre = (int *)(b + Ly.hi_pre); X.lo_suf = (int *)(b + Ly.lo_suf); X.hi_suf = (int *)(b + Ly.hi_suf);
    X.drops = (int *)(b + Ly.drops); X.Lr = Lr;
    X.ret = (double *)(b + Ly.ret); X.exit_leg = (double *)(b + Ly.exit_leg);
    X.omax = (double *)(b + Ly.omax); X.sum_ret = (double *)(b + Ly.sum_ret);
    X.ready = (double *)(b + Ly.ready); X.has_ready = (int *)(b + Ly.has_ready);
    X.pos_v = (int *)(b + Ly.pos_v); X.pos_i = (int *)(b + Ly.pos_i);
    X.s_seq = (int *)(b + Ly.s_seq); X.s_T = (double *)(b + Ly.s_T); X.s_dep = (double *)(b + Ly.s_dep);
    X.s_M = (double *)(b + Ly.s_M); X.s_sp = (int *)(b + Ly.s_sp); X.s_lo_pre = (int *)(b + Ly.s_lo_pre);
    X.s_hi_pre = (int *)(b + Ly.s_hi_pre); X.s_lo_suf = (int *)(b + Ly.s_lo_suf);
    X.s_hi_suf = (int *)(b + Ly.s_hi_suf); X.s_drops = (int *)(b + Ly.s_drops);
    X.s_misc = (double *)(b + Ly.s_misc); X.s_ready = (double *)(b + Ly.s_ready);
    X.s_has = (int *)(b + Ly.s_has); X.s_pv = (int *)(b + Ly.s_pv); X.s_pi = (int *)(b + Ly.s_pi);
    X.gl_g = (int *)(b + Ly.gl_g); X.gl_ret = (double *)(b + Ly.gl_ret); X.gl_stale = (int *)(b + Ly.gl_stale);
    X.keys = (Key *)(b + Ly.keys); X.opts = (Opt *)(b + Ly.opts); X.best = (Opt *)(b + Ly.best);
    X.remaining = (int *)(b + Ly.remaining); X.walk = (double *)(b + Ly.walk);
    X.dm = I->d; X.pv = I->p;
}

// remaining = sorted customers c with flag[c] != 0 (insertion.py:488); returns the count
__device__ __forceinline__ int compact_flags(Ctx &X, const int *flag) {
    int nrem = 0;
    const unsigned lt = lanemask_lt();
    for (int base = 1; base <= X.n; base += 32) {
        const int c = base + X.lane;
        const bool in = c <= X.n && flag[c];
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, in);
        if (in) X.remaining[nrem + __popc(mk & lt)] = c;
        nrem += __popc(mk);
    }
    __syncwarp();
    return nrem;
}

// insertion.py:484-516 on the context's current routes (already rebuilt) and
// X.remaining[0..nrem).  Returns 0, or 1 for RepairFailed.
template <bool SCAN>
__device__ int reinsert_core(Ctx &X, int nrem, int rk, PhiloxGen *gen, bool use_rng) {
    const int lane = X.lane;
    int st = 0;
    while (nrem) {
        int chosen = -1;
        if (rk == 0) {
            for (int i = 0; i < nrem; ++i) {
                const int c = X.remaining[i];
                const int no = customer_options<SCAN>(X, c, gen, use_rng);
                if (!no) { st = 1; break; }
                if (lane == 0) X.best[i] = X.opts[0];
                __syncwarp();
            }
            if (st) break;
            // greedy outer window over (c1, stale, c) -- keys reuse X.keys
            for (int i = lane; i < nrem; i += 32)
                X.keys[i] = Key{X.best[i].cost, X.best[i].stale, X.remaining[i], 0, 0};
            __syncwarp();
            chosen = pick_windowed(X.keys, nrem, lane, gen, use_rng);
        } else {
            double bk_r = 0.0, bk_c = 0.0;
            int bk_s = 0, bk_cust = 0;
            bool have = false;
            for (int i = 0; i < nrem; ++i) {
                const int c = X.remaining[i];
                const int no = customer_options<SCAN>(X, c, gen, use_rng);
                if (!no) { st = 1; break; }
                if (lane == 0) {
                    double regret;
                    if (no < rk) {
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
                        X.best[0] = o0;
                    }
                }
                __syncwarp();
            }
            if (st) break;
            chosen = __shfl_sync(VRP_FULL_MASK, chosen, 0);
        }
        // apply_option (insertion.py:475-481) + remaining.remove(chosen)
        const Opt o = rk == 0 ? X.best[chosen] : X.best[0];
        const int c = X.remaining[chosen];
        if (o.pair) {
            if (SCAN) {
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1) + 1);
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1));
            } else {
                if (lane == 0) { insert_op(X, o.vd, o.gd, 2 * (c - 1) + 1); insert_op(X, o.vd, o.gd, 2 * (c - 1)); }
                __syncwarp();
            }
            rebuild_all<SCAN>(X);
        } else {
            if (SCAN) {
                insert_op_warp(X, o.vd, o.gd, 2 * (c - 1));
            } else {
                if (lane == 0) insert_op(X, o.vd, o.gd, 2 * (c - 1));
                __syncwarp();
            }
            rebuild_all<SCAN>(X);
            if (SCAN) {
                insert_op_warp(X, o.vp, o.gp, 2 * (c - 1) + 1);
            } else {
                if (lane == 0) insert_op(X, o.vp, o.gp, 2 * (c - 1) + 1);
                __syncwarp();
            }
            rebuild_all<SCAN>(X);
        }
        if (lane == 0)
            for (int i = chosen; i + 1 < nrem; ++i) X.remaining[i] = X.remaining[i + 1];
        --nrem;
        __syncwarp();
    }
    return st;
}

}  // namespace
