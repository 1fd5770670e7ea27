// alns_step.cu -- K6 + the device-resident ALNS iteration (alns.py:536-640).
//
// One warp owns one ALNS worker (one trajectory) and runs a whole stretch of
// iterations [it_begin, it_end] without returning to the host:
//
//   roulette selection of the destroy / repair operators (alns.py:130-142)
//   destroy (alns.py:182-251): random (Fisher-Yates, :172-179), worst (power-6
//       picks over removal_gains, insertion.py:538-569), shaw (relatedness over
//       the exact schedule, :145-155), cluster, route, critical_path
//   remove_customers + capacity cascade (insertion.py:358-397)
//   repair: insertion.reinsert_all on a fresh context (repair_core.cuh, K5)
//   exact_makespan of the candidate (schedule.py:265-316), lanes = vehicles
//   simulated-annealing acceptance, scores, cooling, reheat, weight updates
//
// Everything the host has to do between iterations -- the local-search pair
// (every 200 / 500 iterations), pool share polling and merging -- sits at
// stretch boundaries the host chooses, so a stretch is a pure function of the
// worker state.  The generator is numpy's Generator(Philox) state advanced
// draw for draw like the reference's single rng (lane 0 owns it).
//
// Scratch per worker: the K5 repair layout + the destroy layout below.
// fp64 in the reference's order (-fmad=false).  Two documented last-ulp
// caveats: the power-6 pick uses a double-double x^6 rounded once, and the SA
// test uses a correctly rounded exp (ddexp.cuh) where the host uses glibc's,
// which misrounds ~0.07 % of inputs; a disagreement needs such an input AND a
// uniform draw inside that one ulp (p < 2^-63 per test).
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "repair_core.cuh"
#include "repair_team.cuh"
#include "ddexp.cuh"

namespace {

constexpr int NOPS = 10;  // DESTROY_OPERATORS (6) + REPAIR_OPERATORS (4), alns.py:28-29
enum { D_RANDOM = 0, D_WORST, D_SHAW, D_CLUSTER, D_ROUTE, D_CRITICAL };
constexpr int ROW_VALS = 2 + NOPS;  // z_best, temperature, weights

struct DLayout {
    size_t tw, ready, gains, mind, tdrop, ret, dveh, pveh, flag, mark, list, posd, posp, off, total;
};

__host__ __device__ inline DLayout make_dlayout(int n, int m) {
    DLayout L;
    const int C = 2 * n + 2;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o += al8(bytes); return at; };
    L.tw = take(8ull * m * C);
    L.ready = take(8ull * (n + 1));
    L.gains = take(8ull * (n + 1));
    L.mind = take(8ull * (n + 1));
    L.tdrop = take(8ull * (n + 1));
    L.ret = take(8ull * MAXM);
    L.dveh = take(4ull * (n + 1));
    L.pveh = take(4ull * (n + 1));
    L.flag = take(4ull * (n + 1));
    L.mark = take(4ull * (n + 1));
    L.list = take(4ull * (n + 1));
    L.posd = take(4ull * (n + 1));
    L.posp = take(4ull * (n + 1));
    L.off = take(4ull * (MAXM + 1));
    L.total = o;
    return L;
}

struct Dx {
    double *tw, *ready, *gains, *mind, *tdrop, *ret;
    int *dveh, *pveh, *flag, *mark, *list, *posd, *posp, *off;
};

__host__ __device__ inline size_t alns_scratch_bytes_dev(int n, int m) {
    return make_layout(n, m).total + make_dlayout(n, m).total;
}

__device__ __forceinline__ Dx bind_dx(unsigned char *b, int n, int m) {
    const DLayout L = make_dlayout(n, m);
    Dx D;
    D.tw = (double *)(b + L.tw); D.ready = (double *)(b + L.ready); D.gains = (double *)(b + L.gains);
    D.mind = (double *)(b + L.mind); D.tdrop = (double *)(b + L.tdrop); D.ret = (double *)(b + L.ret);
    D.dveh = (int *)(b + L.dveh); D.pveh = (int *)(b + L.pveh); D.flag = (int *)(b + L.flag);
    D.mark = (int *)(b + L.mark); D.list = (int *)(b + L.list); D.posd = (int *)(b + L.posd);
    D.posp = (int *)(b + L.posp); D.off = (int *)(b + L.off);
    return D;
}

template <bool INTD>
__device__ __forceinline__ double dd(const DevInstance &I, int a, int b) { return dist<INTD>(I, a, b); }
__device__ __forceinline__ double pp(const DevInstance &I, int c) { return __ldg(I.p + c); }

// x ** 6.0 (alns.py:167-169 `rng.random() ** power`): double-double product
// rounded once.
__device__ __forceinline__ double pow6(double x) {
    const double h2 = x * x, l2 = fma(x, x, -h2);
    const double h4 = h2 * h2, l4 = fma(h2, h2, -h4) + 2.0 * h2 * l2;
    const double h6 = h4 * h2, l6 = fma(h4, h2, -h6) + (h4 * l2 + l4 * h2);
    return h6 + l6;
}

// roulette_select (alns.py:130-142); w = the operator group's weights
__device__ int roulette(const double *w, int cnt, PhiloxGen &gen) {
    const double total = py_sum(w, cnt);
    const double x = gen.next_double() * total;
    double acc = 0.0;
    for (int i = 0; i < cnt; ++i) {
        acc += w[i];
        if (x < acc) return i;
    }
    return cnt - 1;
}

// warp argmin over customers c in 1..n with flag[c] == 0 of (key(c), c); 0 if none
template <class F>
__device__ int argmin_customers(int n, const int *flag, int lane, F key) {
    double bv = 0.0;
    int bc = 0;
    for (int c = lane + 1; c <= n; c += 32) {
        if (flag[c]) continue;
        const double v = key(c);
        if (!bc || v < bv) { bv = v; bc = c; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(VRP_FULL_MASK, bv, o);
        const int oc = __shfl_xor_sync(VRP_FULL_MASK, bc, o);
        if (oc && (!bc || ov < bv || (ov == bv && oc < bc))) { bv = ov; bc = oc; }
    }
    return bc;
}

// ascending list of customers with mark[c] != 0; returns the count
__device__ int compact_marked(const int *mark, int *list, int n, int lane) {
    int cnt = 0;
    const unsigned lt = lanemask_lt();
    for (int base = 1; base <= n; base += 32) {
        const int c = base + lane;
        const bool in = c <= n && mark[c];
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, in);
        if (in) list[cnt + __popc(mk & lt)] = c;
        cnt += __popc(mk);
    }
    __syncwarp();
    return cnt;
}

// exclusive prefix of per-lane lengths (lanes >= m contribute 0)
__device__ __forceinline__ int lane_offset(int L, int lane) {
    int s = L;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(VRP_FULL_MASK, s, o);
        if (lane >= o) s += y;
    }
    return s - L;
}

// schedule.exact_makespan (schedule.py:265-316) / the timing half of
// evaluate (:188-257), lanes = vehicles: route_initial_load of every route
// first (CapacityViolation), then lockstep rounds in which every vehicle
// advances as far as its pickups allow; a round without progress is the
// reference's Deadlock.  Drop times are order-independent, so the result is
// the reference's for any interleaving.  row = this lane's route, L its length.
// Returns 0 / VRP_CAPACITY / VRP_DEADLOCK; *z = makespan (all lanes).
template <bool INTD>
__device__ int replay(const DevInstance &I, const int *row, int L, int lane, Dx &D, bool want_veh,
                      bool want_ret, double *z) {
    const int k = I.k, n = I.n;
    bool bad = false;
    {
        int s = 0, lo = 0, hi = k;
        for (int i = 0; i < L; ++i) {
            if (!(row[i] & 1)) {
                const int need = 1 - s;
                if (need > lo) lo = need;
                s -= 1;
            } else {
                const int room = k - 1 - s;
                if (room < hi) hi = room;
                s += 1;
            }
            if (lo > hi) { bad = true; break; }
        }
    }
    if (__any_sync(VRP_FULL_MASK, bad)) return VRP_CAPACITY;
    volatile double *td = D.tdrop;
    for (int c = lane; c <= n; c += 32) td[c] = NAN;
    __syncwarp();
    int i = 0, at = 0;
    double t = 0.0;
    while (true) {
        const int i0 = i;
        while (i < L) {
            const int op = row[i], c = opc(op);
            if (!(op & 1)) {
                t += dd<INTD>(I, at, c);
                td[c] = t;
                if (want_veh) D.dveh[c] = lane;
            } else {
                const double tdc = td[c];
                if (isnan(tdc)) break;
                const double arr = t + dd<INTD>(I, at, c);
                const double ready = tdc + pp(I, c);
                t = arr >= ready ? arr : ready;
                if (want_veh) D.pveh[c] = lane;
            }
            at = c;
            ++i;
        }
        const bool prog = i != i0, left = i < L;
        __syncwarp();
        if (!__any_sync(VRP_FULL_MASK, left)) break;
        if (!__any_sync(VRP_FULL_MASK, prog)) return VRP_DEADLOCK;
    }
    const double r = L ? t + dd<INTD>(I, at, 0) : 0.0;
    if (want_ret && lane < I.m) D.ret[lane] = r;
    *z = warp_max(r);  // lanes >= m carry 0.0 (the reference's best = 0.0 start)
    __syncwarp();
    return 0;
}

// insertion.removal_gains (insertion.py:538-569) on the current solution
// (flat vehicle-major ops `cur`, lane v's route at D.off[v]).  Each
// customer's new return is re-walked from its first removed position and
// stops as soon as the walk rejoins the original one (same time at the same
// op), which leaves the remainder -- and the result -- bit-identical.
template <bool INTD>
__device__ void removal_gains(const DevInstance &I, const int *cur, const int *lens, Dx &D, int C,
                              int lane) {
    const int n = I.n, m = I.m;
    const int L = lane < m ? lens[lane] : 0;
    const int *row = cur + (lane < m ? D.off[lane] : 0);
    for (int c = lane; c <= n; c += 32) D.posd[c] = D.posp[c] = -1;  // absent from a partial solution
    __syncwarp();
    {
        double t = 0.0;
        int loc = 0;
        for (int i = 0; i < L; ++i) {
            const int op = row[i], c = opc(op);
            t += dd<INTD>(I, loc, c);
            loc = c;
            if (!(op & 1)) {
                D.ready[c] = t + pp(I, c);
                D.posd[c] = (lane << 16) | i;
            } else {
                D.posp[c] = (lane << 16) | i;
            }
        }
    }
    __syncwarp();
    double r = 0.0;
    if (lane < m) {
        double t = 0.0;
        int loc = 0;
        double *tw = D.tw + (size_t)lane * C;
        for (int i = 0; i < L; ++i) {
            const int op = row[i], c = opc(op);
            t += dd<INTD>(I, loc, c);
            loc = c;
            if (op & 1) {
                const double rd = D.ready[c];
                if (rd > t) t = rd;
            }
            tw[i] = t;
        }
        r = L ? t + dd<INTD>(I, loc, 0) : 0.0;
        D.ret[lane] = r;
    }
    __syncwarp();
    double cur_mk = D.ret[0];
    for (int v = 1; v < m; ++v)
        if (D.ret[v] > cur_mk) cur_mk = D.ret[v];
    for (int c = lane + 1; c <= n; c += 32) {
        const int pd = D.posd[c], pk = D.posp[c];
        const int vd = pd >= 0 ? pd >> 16 : -1, vp = pk >= 0 ? pk >> 16 : -1;
        bool have = false;
        double nm = 0.0;
        for (int v = 0; v < m; ++v) {
            if (v == vd || v == vp) continue;
            if (!have || D.ret[v] > nm) { nm = D.ret[v]; have = true; }
        }
        for (int a = 0; a < 2; ++a) {
            const int v = a ? vp : vd;
            if (a && vp == vd) break;
            if (v < 0) continue;
            const int *rv = cur + D.off[v];
            const int Lv = lens[v];
            int i0, i1, cnt;
            if (vd == vp) {
                const int x = pd & 0xffff, y = pk & 0xffff;
                i0 = x < y ? x : y; i1 = x < y ? y : x; cnt = 2;
            } else {
                i0 = i1 = (v == vd ? pd : pk) & 0xffff; cnt = 1;
            }
            double rr;
            if (Lv - cnt == 0) {
                rr = 0.0;
            } else {
                const double *tw = D.tw + (size_t)v * C;
                double t = i0 ? tw[i0 - 1] : 0.0;
                int loc = i0 ? opc(rv[i0 - 1]) : 0;
                bool joined = false;
                for (int j = i0 + 1; j < Lv; ++j) {
                    const int op = rv[j], cc = opc(op);
                    if (cc == c) continue;
                    t += dd<INTD>(I, loc, cc);
                    loc = cc;
                    if (op & 1) {
                        const double rd = D.ready[cc];
                        if (rd > t) t = rd;
                    }
                    if (j > i1 && t == tw[j]) { joined = true; break; }
                }
                rr = joined ? D.ret[v] : t + dd<INTD>(I, loc, 0);
            }
            if (rr > nm) nm = rr;
        }
        D.gains[c] = cur_mk - nm;
    }
    __syncwarp();
}

// flat current solution -> context rows without the flagged customers, then
// the capacity cascade of remove_customers (insertion.py:358-397)
__device__ void remove_flagged(Ctx &X, const int *cur, const int *lens, Dx &D) {
    const int lane = X.lane, m = X.m, k = X.k;
    const unsigned lt = lanemask_lt();
    for (int v = 0; v < m; ++v) {
        const int L = lens[v];
        const int *row = cur + D.off[v];
        int *out = X.seq + (size_t)v * X.C;
        int cnt = 0;
        for (int base = 0; base < L; base += 32) {
            const int i = base + lane;
            const int op = i < L ? row[i] : 0;
            const bool keep = i < L && !D.flag[opc(op)];
            const unsigned mk = __ballot_sync(VRP_FULL_MASK, keep);
            if (keep) out[cnt + __popc(mk & lt)] = op;
            cnt += __popc(mk);
        }
        if (lane == 0) X.Lr[v] = cnt;
    }
    __syncwarp();
    while (true) {
        int brk = 0;
        if (lane < m) {
            const int *row = X.seq + (size_t)lane * X.C;
            int s = 0, lo = 0, hi = k;
            for (int i = 0; i < X.Lr[lane]; ++i) {
                const int op = row[i];
                if (!(op & 1)) {
                    const int need = 1 - s;
                    if (need > lo) lo = need;
                    s -= 1;
                } else {
                    const int room = k - 1 - s;
                    if (room < hi) hi = room;
                    s += 1;
                }
                if (lo > hi) { brk = opc(op); break; }
            }
        }
        const unsigned mk = __ballot_sync(VRP_FULL_MASK, brk != 0);
        if (!mk) break;
        const int broken = __shfl_sync(VRP_FULL_MASK, brk, __ffs(mk) - 1);
        if (lane == 0) D.flag[broken] = 1;
        for (int v = 0; v < m; ++v) {
            int *row = X.seq + (size_t)v * X.C;
            const int L = X.Lr[v];
            int cnt = 0;
            for (int base = 0; base < L; base += 32) {
                const int i = base + lane;
                const int op = i < L ? row[i] : 0;
                const bool keep = i < L && opc(op) != broken;
                const unsigned km = __ballot_sync(VRP_FULL_MASK, keep);
                __syncwarp();
                if (keep) row[cnt + __popc(km & lt)] = op;
                cnt += __popc(km);
            }
            __syncwarp();
            if (lane == 0) X.Lr[v] = cnt;
            __syncwarp();
        }
    }
    __syncwarp();
}

// context rows -> flat (ops, lens)
__device__ void store_rows(const Ctx &X, int *ops, int *lens) {
    int off = 0;
    for (int v = 0; v < X.m; ++v) {
        const int L = X.Lr[v];
        const int *row = X.seq + (size_t)v * X.C;
        for (int i = X.lane; i < L; i += 32) ops[off + i] = row[i];
        off += L;
    }
    if (X.lane < X.m) lens[X.lane] = X.Lr[X.lane];
}

// destroy (alns.py:182-251): sets D.flag[c] = 1 for the picked customers
template <bool INTD>
__device__ void destroy(const DevInstance &I, int op, int q, int q_min, const int *cur, const int *lens,
                        Dx &D, int C, int lane, PhiloxGen &gen) {
    const int n = I.n, m = I.m;
    for (int c = lane; c <= n; c += 32) D.flag[c] = 0;
    __syncwarp();
    if (op == D_RANDOM) {
        for (int i = lane; i < n; i += 32) D.list[i] = i + 1;
        __syncwarp();
        if (lane == 0) {
            for (int i = 0; i < q; ++i) {
                const int j = i + (int)gen.integers((uint32_t)(n - i));
                const int a = D.list[i];
                D.list[i] = D.list[j];
                D.list[j] = a;
            }
            for (int i = 0; i < q; ++i) D.flag[D.list[i]] = 1;
        }
    } else if (op == D_WORST) {
        removal_gains<INTD>(I, cur, lens, D, C, lane);
        // ranked = sorted(customers, key=(-gain, c)): rank by counting
        for (int c = lane + 1; c <= n; c += 32) {
            const double g = D.gains[c];
            int r = 0;
            for (int c2 = 1; c2 <= n; ++c2) {
                const double g2 = D.gains[c2];
                r += (g2 > g) || (g2 == g && c2 < c);
            }
            D.list[r] = c;
        }
        __syncwarp();
        int len = n;
        for (int pick = 0; pick < q; ++pick) {
            int idx = 0;
            if (lane == 0) {
                const double x = pow6(gen.next_double()) * (double)len;
                idx = (int)x;
                if (idx > len - 1) idx = len - 1;
                D.flag[D.list[idx]] = 1;
            }
            idx = __shfl_sync(VRP_FULL_MASK, idx, 0);
            __syncwarp();
            for (int base = idx; base < len - 1; base += 32) {  // ranked.remove(c)
                const int i = base + lane;
                const int nxt = i < len - 1 ? D.list[i + 1] : 0;
                __syncwarp();
                if (i < len - 1) D.list[i] = nxt;
                __syncwarp();
            }
            --len;
        }
    } else if (op == D_SHAW) {
        const int L = lane < m ? lens[lane] : 0;
        double z;
        replay<INTD>(I, cur + (lane < m ? D.off[lane] : 0), L, lane, D, true, false, &z);
        int cnt = 1;
        if (lane == 0) {
            const int seed = 1 + (int)gen.integers((uint32_t)n);
            D.list[0] = seed;
            D.flag[seed] = 1;
        }
        __syncwarp();
        while (cnt < q && cnt < n) {
            int ref = 0;
            if (lane == 0) ref = D.list[gen.integers((uint32_t)cnt)];
            ref = __shfl_sync(VRP_FULL_MASK, ref, 0);
            const double tr = D.tdrop[ref];
            const int dvr = D.dveh[ref], pvr = D.pveh[ref];
            const int best = argmin_customers(n, D.flag, lane, [&](int c) {
                double r = 9.0 * dd<INTD>(I, ref, c);  // shaw_relatedness, alns.py:145-155
                r += 3.0 * fabs(tr - D.tdrop[c]);
                if (dvr != D.dveh[c]) r += 2.5;
                if (pvr != D.pveh[c]) r += 2.5;
                return r;
            });
            if (lane == 0) { D.flag[best] = 1; D.list[cnt] = best; }
            ++cnt;
            __syncwarp();
        }
    } else if (op == D_CLUSTER) {
        int center = 0;
        if (lane == 0) {
            center = 1 + (int)gen.integers((uint32_t)n);
            D.flag[center] = 1;
        }
        center = __shfl_sync(VRP_FULL_MASK, center, 0);
        __syncwarp();
        for (int i = 0; i < q - 1; ++i) {
            const int best = argmin_customers(n, D.flag, lane, [&](int c) { return dd<INTD>(I, center, c); });
            if (lane == 0) D.flag[best] = 1;
            __syncwarp();
        }
    } else if (op == D_ROUTE) {
        const int L = lane < m ? lens[lane] : 0;
        const unsigned ne = __ballot_sync(VRP_FULL_MASK, lane < m && L > 0);
        int v = 0;
        if (lane == 0) {
            int j = (int)gen.integers((uint32_t)__popc(ne));
            unsigned x = ne;
            while (j--) x &= x - 1;
            v = __ffs(x) - 1;
        }
        v = __shfl_sync(VRP_FULL_MASK, v, 0);
        const int Lv = lens[v];
        const int *row = cur + D.off[v];
        for (int i = lane; i < Lv; i += 32) D.flag[opc(row[i])] = 1;
        __syncwarp();
        int cnt = 0;
        for (int c = lane + 1; c <= n; c += 32) cnt += D.flag[c];
        cnt = warp_sum(cnt);
        if (cnt < q_min) {
            const int np = compact_marked(D.flag, D.list, n, lane);
            for (int c = lane + 1; c <= n; c += 32) {
                if (D.flag[c]) continue;
                double mn = dd<INTD>(I, c, D.list[0]);
                for (int j = 1; j < np; ++j) {
                    const double x = dd<INTD>(I, c, D.list[j]);
                    if (x < mn) mn = x;
                }
                D.mind[c] = mn;
            }
            __syncwarp();
            while (cnt < q_min && cnt < n) {
                const int best = argmin_customers(n, D.flag, lane, [&](int c) { return D.mind[c]; });
                if (lane == 0) D.flag[best] = 1;
                __syncwarp();
                ++cnt;
                for (int c = lane + 1; c <= n; c += 32) {
                    if (D.flag[c]) continue;
                    const double x = dd<INTD>(I, c, best);
                    if (x < D.mind[c]) D.mind[c] = x;
                }
                __syncwarp();
            }
        }
    } else {  // D_CRITICAL
        const int L = lane < m ? lens[lane] : 0;
        double z;
        replay<INTD>(I, cur + (lane < m ? D.off[lane] : 0), L, lane, D, false, true, &z);
        int v = 0;
        for (int u = 1; u < m; ++u)
            if (D.ret[u] > D.ret[v]) v = u;  // Schedule.bottleneck, schedule.py:105-110
        for (int c = lane; c <= n; c += 32) D.mark[c] = 0;
        __syncwarp();
        const int Lv = lens[v];
        const int *row = cur + D.off[v];
        for (int i = lane; i < Lv; i += 32) D.mark[opc(row[i])] = 1;
        __syncwarp();
        const int cntR = compact_marked(D.mark, D.list, n, lane);
        if (cntR >= q) {
            if (lane == 0) {
                for (int i = 0; i < q; ++i) {
                    const int j = i + (int)gen.integers((uint32_t)(cntR - i));
                    const int a = D.list[i];
                    D.list[i] = D.list[j];
                    D.list[j] = a;
                }
                for (int i = 0; i < q; ++i) D.flag[D.list[i]] = 1;
            }
            __syncwarp();
        } else {
            for (int i = lane; i < cntR; i += 32) D.flag[D.list[i]] = 1;
            __syncwarp();
            if (cntR < q_min) {
                removal_gains<INTD>(I, cur, lens, D, C, lane);
                for (int i = 0; i < q_min - cntR && i < n - cntR; ++i) {
                    const int best = argmin_customers(n, D.flag, lane, [&](int c) { return -D.gains[c]; });
                    if (lane == 0) D.flag[best] = 1;
                    __syncwarp();
                }
            }
        }
    }
    __syncwarp();
}

// Out-of-line copies of the once-per-iteration steps.  The warp-scan (SCAN)
// instantiation calls these -- keeping its per-customer repair loop compact
// in the instruction cache measured faster (kroA100/a280) -- while the
// one-lane instantiation inlines them (faster at eil51's short routes).
template <bool INTD>
__device__ __noinline__ void destroy_ool(const DevInstance &I, int op, int q, int q_min, const int *cur,
                                         const int *lens, Dx &D, int C, int lane, PhiloxGen &gen) {
    destroy<INTD>(I, op, q, q_min, cur, lens, D, C, lane, gen);
}
__device__ __noinline__ void remove_flagged_ool(Ctx &X, const int *cur, const int *lens, Dx &D) {
    remove_flagged(X, cur, lens, D);
}
template <bool INTD>
__device__ __noinline__ int replay_ool(const DevInstance &I, const int *row, int L, int lane, Dx &D, double *z) {
    return replay<INTD>(I, row, L, lane, D, false, false, z);
}
__device__ __noinline__ void store_rows_ool(const Ctx &X, int *ops, int *lens) { store_rows(X, ops, lens); }

// TEAM: a CTA of TEAM_WARPS warps per worker -- warp 0 runs the iteration,
// every warp joins the context rebuilds and the repair (repair_team.cuh).
template <bool INTD, bool SCAN, bool TEAM = false>
__global__ void __launch_bounds__(TEAM ? 32 * TEAM_WARPS : 32)
alns_kernel(DevInstance I, vrp_alns_params P, vrp_alns_worker *__restrict__ workers, int32_t nw,
            int32_t *__restrict__ cur_ops, int32_t *__restrict__ cur_lens, int32_t *__restrict__ best_ops,
            int32_t *__restrict__ best_lens, const int32_t *__restrict__ q_draws, int64_t q_stride,
            int64_t it_begin, int64_t it_end, int32_t *__restrict__ trace_it, double *__restrict__ trace_z,
            int64_t trace_cap, int32_t *__restrict__ rows_it, double *__restrict__ rows_val,
            int64_t rows_cap, unsigned char *__restrict__ scratch, size_t per) {
    __shared__ int s_len[MAXM];
    __shared__ vrp_alns_worker S;
    __shared__ TeamCtl T;
    __shared__ int s_nrem, s_rk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int w = blockIdx.x;
    if (w >= nw) return;
    const int n = I.n, m = I.m, C = 2 * n + 2;
    unsigned char *b = scratch + (size_t)w * per;
    Ctx X;
    bind_ctx(X, &I, b, s_len, lane);
    Dx D = bind_dx(b + make_layout(n, m).total, n, m);
    UnitRes *units = nullptr;
    UnitPick *picks = nullptr;
    TeamWS W{};
    GapRec *crecs = nullptr;
    TeamCx cx{};
    if (TEAM) W = bind_team(X, b + al8(alns_scratch_bytes_dev(n, m)), n, m, warp, nwarps, units, picks, crecs, cx);

    int32_t *cur = cur_ops + (int64_t)w * 2 * n, *clen = cur_lens + (int64_t)w * m;
    int32_t *best = best_ops + (int64_t)w * 2 * n, *blen = best_lens + (int64_t)w * m;
#ifdef VRP_PHASE_TIMERS
    long long tph[6] = {0, 0, 0, 0, 0, 0};  // destroy, rebuild, repair, replay, removed, options calls
#endif
    PhiloxGen gen;
    if (warp == 0 && lane == 0) {
        S = workers[w];
        gen.s = S.rng;
        S.n_trace = 0;
        S.n_rows = 0;
    }
    __syncwarp();

    for (int64_t it = it_begin; it <= it_end; ++it) {
        int dop = 0, rop = 0, q = 0, nrem = 0, rk = 0, st = 0;
        double zc = 0.0;
      if (warp == 0) {
        // operator selection (alns.py:567-571)
        if (lane == 0) {
            dop = roulette(S.weights, 6, gen);
            rop = roulette(S.weights + 6, 4, gen);
            S.attempts[dop] += 1;
            S.attempts[6 + rop] += 1;
            q = q_draws[(int64_t)w * q_stride + (it - 1)];
            if (q > n) q = n;
        }
        dop = __shfl_sync(VRP_FULL_MASK, dop, 0);
        rop = __shfl_sync(VRP_FULL_MASK, rop, 0);
        q = __shfl_sync(VRP_FULL_MASK, q, 0);
        {
            const int L = lane < m ? clen[lane] : 0;
            const int o = lane_offset(L, lane);
            if (lane < m) D.off[lane] = o;
            __syncwarp();
        }
#ifdef VRP_PHASE_TIMERS
        long long tq = clock64();
#define VRP_TICK(j) do { const long long t2 = clock64(); tph[j] += t2 - tq; tq = t2; } while (0)
#else
#define VRP_TICK(j) do {} while (0)
#endif
        // destroy + remove_customers (alns.py:574; insertion.py:379-397)
        if (SCAN) {
            destroy_ool<INTD>(I, dop, q, P.q_min, cur, clen, D, C, lane, gen);
            remove_flagged_ool(X, cur, clen, D);
        } else {
            destroy<INTD>(I, dop, q, P.q_min, cur, clen, D, C, lane, gen);
            remove_flagged(X, cur, clen, D);
        }
        VRP_TICK(0);
        // repair (alns.py:258-274): reinsert_all, then exact_makespan
        rk = rop == 0 ? 0 : rop == 1 ? 2 : rop == 2 ? 3 : m;
        if (!TEAM) {
            rebuild_all<SCAN>(X);
            nrem = compact_flags(X, D.flag);
            VRP_TICK(1);
            st = reinsert_core<SCAN>(X, nrem, rk, &gen, true);
            VRP_TICK(2);
        }
      }
        if (TEAM) {
            __syncthreads();
            rebuild_all_team(X, crecs, cx, warp, nwarps);
            if (warp == 0) {
                nrem = compact_flags(X, D.flag);
                if (lane == 0) { s_nrem = nrem; s_rk = rk; }
            }
            __syncthreads();
            st = reinsert_team(X, W, T, units, picks, crecs, cx, s_nrem, s_rk, &gen, true, warp, nwarps);
        }
      if (warp == 0) {
        if (!st) {
            const int *row = X.seq + (size_t)(lane < m ? lane : 0) * C;
            const int L = lane < m ? X.Lr[lane] : 0;
            st = SCAN ? replay_ool<INTD>(I, row, L, lane, D, &zc) : replay<INTD>(I, row, L, lane, D, false, false, &zc);
        }
        VRP_TICK(3);
#ifdef VRP_PHASE_TIMERS
        tph[4] += nrem;
        tph[5] += (long long)nrem * (nrem + 1) / 2;
#endif
        // acceptance + bookkeeping (alns.py:577-611)
        int acc = 0, nb = 0;
        if (lane == 0) {
            const int r6 = 6 + rop;
            if (st) {
                S.rejected += 1;
            } else if (zc < S.z) {
                acc = 1;
                S.z = zc;
                S.scores[dop] += P.sigma2;
                S.scores[r6] += P.sigma2;
                S.accepted += 1;
                if (zc < S.z_best) {
                    S.scores[dop] += P.sigma1 - P.sigma2;
                    S.scores[r6] += P.sigma1 - P.sigma2;
                    nb = 1;
                    S.z_best = zc;
                    S.stagnation = 0;
                    S.best_it = it;
                    if (S.n_trace < trace_cap) {
                        trace_it[(int64_t)w * trace_cap + S.n_trace] = (int32_t)it;
                        trace_z[(int64_t)w * trace_cap + S.n_trace] = zc;
                    }
                    S.n_trace += 1;
                }
            } else if (S.temperature > 0 && gen.next_double() < ddexp::exp_cr(-(zc - S.z) / S.temperature)) {
                acc = 1;
                S.z = zc;
                S.scores[dop] += P.sigma3;
                S.scores[r6] += P.sigma3;
                S.accepted += 1;
            }
            S.temperature *= P.alpha;
            S.stagnation += 1;
            if (S.stagnation >= P.stagnation_threshold && S.temperature < 0.01 * S.t_init) {
                S.temperature = P.reheat_factor * P.t0 * S.z_best;
                S.stagnation = 0;
                S.reheats += 1;
            }
            if (it % P.weight_interval == 0) {  // update_weights, alns.py:112-127
                for (int j = 0; j < NOPS; ++j) {
                    const int64_t a = S.attempts[j];
                    const double avg = a ? S.scores[j] / (double)a : 0.0;
                    const double nwt = (1.0 - P.reaction) * S.weights[j] + P.reaction * avg;
                    S.weights[j] = nwt > P.min_weight ? nwt : P.min_weight;
                    S.scores[j] = 0.0;
                    S.attempts[j] = 0;
                }
                if (S.n_rows < rows_cap) {
                    const int64_t r = (int64_t)w * rows_cap + S.n_rows;
                    rows_it[r] = (int32_t)it;
                    double *rv = rows_val + r * ROW_VALS;
                    rv[0] = S.z_best;
                    rv[1] = S.temperature;
                    for (int j = 0; j < NOPS; ++j) rv[2 + j] = S.weights[j];
                }
                S.n_rows += 1;
            }
        }
        acc = __shfl_sync(VRP_FULL_MASK, acc, 0);
        nb = __shfl_sync(VRP_FULL_MASK, nb, 0);
        if (acc) { if (SCAN) store_rows_ool(X, cur, clen); else store_rows(X, cur, clen); }
        if (nb) { if (SCAN) store_rows_ool(X, best, blen); else store_rows(X, best, blen); }
        __syncwarp();
      }
    }
    if (warp == 0 && lane == 0) {
        S.rng = gen.s;
        workers[w] = S;
#ifdef VRP_PHASE_TIMERS  // debug builds: phase clocks into the trace buffer
        for (int j = 0; j < 6 && j < trace_cap; ++j) trace_z[(int64_t)w * trace_cap + j] = (double)tph[j];
#endif
    }
}

// K6 alone: destroy + remove_customers on N independent solutions
// (alns.py:182-251 -> insertion.py:379-397).
template <bool INTD>
__global__ void __launch_bounds__(32)
destroy_kernel(DevInstance I, const int32_t *__restrict__ ops, int64_t stride, const int32_t *__restrict__ lens,
               const int32_t *__restrict__ opcode, const int32_t *__restrict__ qv, int32_t q_min,
               vrp_philox *__restrict__ states, int32_t *__restrict__ out_ops, int64_t ostride,
               int32_t *__restrict__ out_lens, int32_t *__restrict__ removed, int64_t rstride,
               int32_t *__restrict__ nremoved, unsigned char *__restrict__ scratch, size_t per, int64_t N,
               const int32_t *__restrict__ picked, int64_t pstride, const int32_t *__restrict__ npicked) {
    __shared__ int s_len[MAXM];
    const int lane = threadIdx.x;
    const int64_t w = blockIdx.x;
    if (w >= N) return;
    const int n = I.n, m = I.m, C = 2 * n + 2;
    unsigned char *b = scratch + (size_t)w * per;
    Ctx X;
    bind_ctx(X, &I, b, s_len, lane);
    Dx D = bind_dx(b + make_layout(n, m).total, n, m);
    const int32_t *cur = ops + w * stride, *clen = lens + w * m;
    {
        const int L = lane < m ? clen[lane] : 0;
        const int o = lane_offset(L, lane);
        if (lane < m) D.off[lane] = o;
        __syncwarp();
    }
    PhiloxGen gen;
    if (picked) {  // remove_customers alone: the caller's customers (insertion.py:379-397)
        for (int c = lane; c <= n; c += 32) D.flag[c] = 0;
        __syncwarp();
        const int np = npicked[w];
        for (int i = lane; i < np; i += 32) {
            const int c = picked[w * pstride + i];
            if (c >= 1 && c <= n) D.flag[c] = 1;
        }
        __syncwarp();
    } else {
        if (lane == 0) gen.s = states[w];
        int q = qv[w];
        if (q > n) q = n;
        destroy<INTD>(I, opcode[w], q, q_min < n ? q_min : n, cur, clen, D, C, lane, gen);
    }
    remove_flagged(X, cur, clen, D);
    int32_t *oo = out_ops + w * ostride;
    store_rows(X, oo, out_lens + w * m);
    int tot = 0;
    for (int v = 0; v < m; ++v) tot += X.Lr[v];
    for (int i = tot + lane; i < 2 * n; i += 32) oo[i] = -1;
    const int nr = compact_marked(D.flag, removed + w * rstride, n, lane);
    if (lane == 0) {
        nremoved[w] = nr;
        if (!picked) states[w] = gen.s;
    }
}

// insertion.removal_gains (insertion.py:538-569) alone: gains[w][c], c = 1..n
// (gains[w][0] = 0)
template <bool INTD>
__global__ void __launch_bounds__(32)
gains_kernel(DevInstance I, const int32_t *__restrict__ ops, int64_t stride, const int32_t *__restrict__ lens,
             double *__restrict__ gains, int64_t gstride, unsigned char *__restrict__ scratch, size_t per,
             int64_t N) {
    const int lane = threadIdx.x;
    const int64_t w = blockIdx.x;
    if (w >= N) return;
    const int n = I.n, m = I.m, C = 2 * n + 2;
    Dx D = bind_dx(scratch + (size_t)w * per, n, m);
    const int32_t *cur = ops + w * stride, *clen = lens + w * m;
    {
        const int L = lane < m ? clen[lane] : 0;
        const int o = lane_offset(L, lane);
        if (lane < m) D.off[lane] = o;
        __syncwarp();
    }
    removal_gains<INTD>(I, cur, clen, D, C, lane);
    double *g = gains + w * gstride;
    for (int c = lane; c <= n; c += 32) g[c] = c ? D.gains[c] : 0.0;
}

}  // namespace

size_t alns_scratch_bytes(int n, int m) { return alns_scratch_bytes_dev(n, m); }

int launch_alns(const DevInstance &I, const vrp_alns_params &P, vrp_alns_worker *workers, int32_t nw,
                int32_t *cur_ops, int32_t *cur_lens, int32_t *best_ops, int32_t *best_lens,
                const int32_t *q_draws, int64_t q_stride, int64_t it_begin, int64_t it_end,
                int32_t *trace_it, double *trace_z, int64_t trace_cap, int32_t *rows_it,
                double *rows_val, int64_t rows_cap, cudaStream_t stream) {
    if (nw <= 0 || it_end < it_begin) return 0;
    const bool team = use_team(I);
    const size_t per = al8(alns_scratch_bytes(I.n, I.m)) + (team ? team_bytes(I.n, I.m, TEAM_WARPS) : 0);
    unsigned char *scratch = nullptr;
    if (cudaMallocAsync(&scratch, per * (size_t)nw, stream) != cudaSuccess) return -1;
#define VRP_ALNS_ARGS I, P, workers, nw, cur_ops, cur_lens, best_ops, best_lens, q_draws, q_stride, it_begin, \
        it_end, trace_it, trace_z, trace_cap, rows_it, rows_val, rows_cap, scratch, per
    if (team) alns_kernel<true, true, true><<<nw, 32 * TEAM_WARPS, 0, stream>>>(VRP_ALNS_ARGS);
    else if (use_scan(I)) alns_kernel<true, true><<<nw, 32, 0, stream>>>(VRP_ALNS_ARGS);
    else if (I.integral) alns_kernel<true, false><<<nw, 32, 0, stream>>>(VRP_ALNS_ARGS);
    else alns_kernel<false, false><<<nw, 32, 0, stream>>>(VRP_ALNS_ARGS);
#undef VRP_ALNS_ARGS
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(scratch, stream);
    return e == cudaSuccess ? 0 : -1;
}

int launch_destroy(const DevInstance &I, const int32_t *ops, int64_t stride, const int32_t *lens,
                   const int32_t *opcode, const int32_t *q, int32_t q_min, vrp_philox *states,
                   int32_t *out_ops, int64_t ostride, int32_t *out_lens, int32_t *removed,
                   int64_t rstride, int32_t *nremoved, int64_t N, cudaStream_t stream,
                   const int32_t *picked, int64_t pstride, const int32_t *npicked) {
    if (N <= 0) return 0;
    const size_t per = al8(alns_scratch_bytes(I.n, I.m));
    unsigned char *scratch = nullptr;
    if (cudaMallocAsync(&scratch, per * (size_t)N, stream) != cudaSuccess) return -1;
    if (I.integral)
        destroy_kernel<true><<<(unsigned)N, 32, 0, stream>>>(I, ops, stride, lens, opcode, q, q_min, states,
                                                             out_ops, ostride, out_lens, removed, rstride,
                                                             nremoved, scratch, per, N, picked, pstride,
                                                             npicked);
    else
        destroy_kernel<false><<<(unsigned)N, 32, 0, stream>>>(I, ops, stride, lens, opcode, q, q_min, states,
                                                              out_ops, ostride, out_lens, removed, rstride,
                                                              nremoved, scratch, per, N, picked, pstride,
                                                              npicked);
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(scratch, stream);
    return e == cudaSuccess ? 0 : -1;
}

namespace {
__global__ void sa_exp_kernel(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = ddexp::exp_cr(x[i]);
}
}  // namespace

int launch_gains(const DevInstance &I, const int32_t *ops, int64_t stride, const int32_t *lens, double *gains,
                 int64_t gstride, int64_t N, cudaStream_t stream) {
    if (N <= 0) return 0;
    const size_t per = al8(make_dlayout(I.n, I.m).total);
    unsigned char *scratch = nullptr;
    if (cudaMallocAsync(&scratch, per * (size_t)N, stream) != cudaSuccess) return -1;
    if (I.integral)
        gains_kernel<true><<<(unsigned)N, 32, 0, stream>>>(I, ops, stride, lens, gains, gstride, scratch, per, N);
    else
        gains_kernel<false><<<(unsigned)N, 32, 0, stream>>>(I, ops, stride, lens, gains, gstride, scratch, per, N);
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(scratch, stream);
    return e == cudaSuccess ? 0 : -1;
}

int launch_sa_exp(const double *x, double *y, int64_t n, cudaStream_t stream) {
    if (n <= 0) return 0;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    sa_exp_kernel<<<(unsigned)blocks, 256, 0, stream>>>(x, y, n);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
