// makespan.cu -- K1 (exact event-driven makespan, schedule.py:188-316) and
// K2 (two-pass estimate, schedule.py:345-393) over batches of candidates.
//
// Mapping.  A warp carries G = floor(32/m) candidates at once; lane g*m+v owns
// route v of candidate g (30 of 32 lanes busy for m = 6).  Persistent grid.
//
// Windowed staging.  Each route has a WIN-position window in shared memory
// holding its op codes and legs d[prev][c].  Whenever some lane has consumed
// the older half of its window, the WHOLE WARP refills: for up to
// REFILL_BATCH routes at a time, 32 lanes stream the next CHUNK op codes of a
// route (coalesced), exchange the predecessor op with a shuffle and gather the
// legs from the L2-resident matrix -- all loads of a round are issued before
// any is consumed.  Refills are warp-uniform (no divergence) and the per-lane
// replay loop below touches shared memory only.  Per candidate this costs the
// ready table (8(n+1) B) plus m*WIN*(4+2) B of window, ~10 KB at n = 999, so
// ~20 candidates are in flight per SM.
//
// Replay (exact / evaluate): lockstep dataflow.  Every iteration each lane
// executes the next op of its route unless it is a pickup whose dropoff has
// not happened yet (ready < 0):
//     dropoff  t = t + leg;                 ready[c] = t + p[c]
//     pickup   arr = t + leg;  t = arr >= ready[c] ? arr : ready[c]
// Writes become visible to the other lanes at the __syncwarp() ending the
// iteration, so the iteration count is the depth of the precedence DAG.  A
// candidate whose lanes all stall while ops remain is a circular wait
// (Deadlock, schedule.py:243-245 / :308-309).  Each value depends only on its
// DAG predecessors; integral instances keep times in int64 (exact), others in
// fp64 with the reference's operation order -- bit-identical either way.
//
// Capacity (route_initial_load, schedule.py:159-185) is the running interval
// [lo, hi] of feasible initial loads; lo only grows and hi only shrinks, so
// "empty at some prefix" == "empty at the end" and the test rides along with
// the replay (finished past a deadlock by a capacity-only scan).  Status
// precedence: MALFORMED > CAPACITY > DEADLOCK.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int MODE_EXACT = 0, MODE_EVAL = 1, MODE_TWO = 2;
constexpr int ST_OK = 0, ST_CAP = 1, ST_DEAD = 2, ST_MAL = 3;
constexpr int WIN = 64;           // staged positions per route (power of two)
constexpr int CHUNK = 32;         // positions staged per refill (= warp width)
constexpr int REFILL_BATCH = 4;   // routes refilled per round (loads in flight)

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <bool INTD>
using TimeT = typename std::conditional<INTD, long long, double>::type;  // event times
template <bool INTD>
using LegT = typename std::conditional<INTD, int32_t, double>::type;     // staged legs

// Per candidate: ready table, route windows, plus (validating modes) an op
// bitmap and (two-pass) the (route, position) of every dropoff.
struct CandLayout {
    size_t ready, wleg, wop, bits, posd, total;
};

__host__ __device__ inline CandLayout cand_layout(int n, int m, bool intd, int mode) {
    CandLayout L;
    size_t o = 0;
    L.ready = o; o += align16(8 * (size_t)(n + 1));
    L.wleg = o;  o += align16((intd ? 4 : 8) * (size_t)m * WIN);
    L.wop = o;   o += align16(2 * (size_t)m * WIN);
    L.bits = o;  if (mode != MODE_EXACT) o += align16(4 * (size_t)((2 * n + 31) / 32));
    L.posd = o;  if (mode == MODE_TWO) o += align16(4 * (size_t)(n + 1));
    L.total = o;
    return L;
}

__host__ __device__ inline size_t block_p_bytes(int n) { return align16(8 * (size_t)(n + 1)); }

__device__ __forceinline__ void cap_step(int op, int k, int &s, int &lo, int &hi) {
    if (op & 1) { int room = k - 1 - s; hi = room < hi ? room : hi; ++s; }
    else        { int need = 1 - s;     lo = need > lo ? need : lo; --s; }
}

// Per-lane view of its route.
struct Route {
    int64_t re;   // element index of position 0 in the ops buffer
    int L;        // length
    int i;        // next position to execute
    int staged;   // positions [staged - WIN, staged) are in the window
};

// Stage the next CHUNK positions of every route in `need` (a lane mask),
// REFILL_BATCH routes per round.  Warp-uniform; returns (uniformly) the lanes
// whose newly staged op codes were out of range.
template <typename OpT, bool INTD>
__device__ __forceinline__ unsigned refill(const DevInstance &I, const OpT *__restrict__ ops,
                                           unsigned need, Route &R, int lane, int m,
                                           unsigned char *wbase, const CandLayout &CL, int two_n) {
    using LT = LegT<INTD>;
    unsigned badmask = 0;
    while (need) {
        int rl[REFILL_BATCH], pos[REFILL_BATCH], op[REFILL_BATCH];
        unsigned served = 0;
#pragma unroll
        for (int b = 0; b < REFILL_BATCH; ++b) {
            rl[b] = need ? __ffs(need) - 1 : -1;
            if (rl[b] >= 0) { served |= 1u << rl[b]; need &= need - 1; }
        }
        // op codes: coalesced; every round's loads in flight together
#pragma unroll
        for (int b = 0; b < REFILL_BATCH; ++b) {
            const int src = rl[b] < 0 ? lane : rl[b];
            const int s = __shfl_sync(VRP_FULL_MASK, R.staged, src);
            const int L = __shfl_sync(VRP_FULL_MASK, R.L, src);
            const long long re = __shfl_sync(VRP_FULL_MASK, (long long)R.re, src);
            pos[b] = s + lane;
            const bool ok = rl[b] >= 0 && pos[b] < L;
            op[b] = ok ? (int)__ldg(ops + re + pos[b]) : -1;
            if (!ok) pos[b] = -1;
        }
        LT leg[REFILL_BATCH];
#pragma unroll
        for (int b = 0; b < REFILL_BATCH; ++b) {
            const int src = rl[b] < 0 ? 0 : rl[b];
            const int gg = src / m, vv = src - (src / m) * m;
            const uint16_t *wop = reinterpret_cast<const uint16_t *>(wbase + (size_t)gg * CL.total + CL.wop) + vv * WIN;
            const bool bad = pos[b] >= 0 && (unsigned)op[b] >= (unsigned)two_n;
            if (bad) op[b] = 0;
            if (__any_sync(VRP_FULL_MASK, bad) && rl[b] >= 0) badmask |= 1u << rl[b];
            int prev = __shfl_up_sync(VRP_FULL_MASK, op[b], 1);
            if (lane == 0) prev = pos[b] > 0 ? (int)wop[(pos[b] - 1) & (WIN - 1)] : -1;
            const int a = prev < 0 ? 0 : op_customer(prev);
            const int idx = a * I.W + op_customer(op[b] < 0 ? 0 : op[b]);
            if (pos[b] >= 0) leg[b] = INTD ? (LT)__ldcg(I.d32 + idx) : (LT)__ldcg(I.d + idx);
            else leg[b] = (LT)0;
        }
#pragma unroll
        for (int b = 0; b < REFILL_BATCH; ++b) {
            if (pos[b] < 0) continue;
            const int gg = rl[b] / m, vv = rl[b] - (rl[b] / m) * m;
            unsigned char *cb = wbase + (size_t)gg * CL.total;
            reinterpret_cast<uint16_t *>(cb + CL.wop)[vv * WIN + (pos[b] & (WIN - 1))] = (uint16_t)op[b];
            reinterpret_cast<LT *>(cb + CL.wleg)[vv * WIN + (pos[b] & (WIN - 1))] = leg[b];
        }
        if ((served >> lane) & 1u) R.staged += CHUNK;
        __syncwarp();
    }
    return badmask;
}

// Lanes whose window can take (and still lacks) their next chunk.
__device__ __forceinline__ bool wants_chunk(const Route &R, bool run) {
    return run && R.staged < R.L && R.i >= R.staged - WIN + CHUNK;
}

template <typename OpT, bool INTD, int MODE, bool REC>
__global__ void __launch_bounds__(256)
makespan_kernel(DevInstance I, const OpT *__restrict__ ops, int64_t stride,
                const int32_t *__restrict__ lens, int64_t N, int G, double *__restrict__ z_out,
                int32_t *__restrict__ status_out, double *__restrict__ returns_out,
                int32_t *__restrict__ bottleneck_out, double *__restrict__ arrival_out,
                double *__restrict__ time_out, int32_t *__restrict__ q0_out) {
    using TT = TimeT<INTD>;
    using LT = LegT<INTD>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int n = I.n, m = I.m, k = I.k, two_n = 2 * n;
    const CandLayout CL = cand_layout(n, m, INTD, MODE);
    TT *s_p = reinterpret_cast<TT *>(smem);
    unsigned char *wbase = smem + block_p_bytes(n) + (size_t)warp * G * CL.total;

    const int g = lane / m, v = lane - (lane / m) * m;
    const bool glane = g < G;
    const unsigned gmask = glane ? (((m == 32) ? 0xffffffffu : ((1u << m) - 1u)) << (g * m)) : 0u;
    const int leader = g * m;  // lane holding route 0 of this lane's candidate
    unsigned char *cbase = wbase + (size_t)(glane ? g : 0) * CL.total;
    TT *s_ready = reinterpret_cast<TT *>(cbase + CL.ready);
    uint32_t *s_posd = reinterpret_cast<uint32_t *>(cbase + CL.posd);
    const LT *w_leg = reinterpret_cast<const LT *>(cbase + CL.wleg) + (glane ? v : 0) * WIN;
    const uint16_t *w_op = reinterpret_cast<const uint16_t *>(cbase + CL.wop) + (glane ? v : 0) * WIN;

    for (int c = threadIdx.x; c <= n; c += blockDim.x)
        s_p[c] = INTD ? (TT)__ldg(I.p32 + c) : (TT)__ldg(I.p + c);
    __syncthreads();

    const int64_t step = (int64_t)gridDim.x * wpb * G;
    for (int64_t base = ((int64_t)blockIdx.x * wpb + warp) * G; base < N; base += step) {
        const int64_t cand = base + g;
        const bool live = glane && cand < N;
        // ---- route offsets: lane v sums the lengths of routes 0..v-1
        int L = 0, off = 0, total = 0;
        bool mal = false;
        if (live) {
            const int32_t *lr = lens + cand * m;
            for (int u = 0; u < m; ++u) {
                const int x = __ldg(lr + u);
                mal |= x < 0;
                if (u < v) off += x;
                if (u == v) L = x;
                total += x;
            }
            mal |= total > two_n || total > stride || (MODE != MODE_EXACT && total != two_n);
        }

        // ---- shared tables: ready = -1 (dropoff not done); validation bitmap
        for (int gg = 0; gg < G; ++gg) {
            TT *rd = reinterpret_cast<TT *>(wbase + (size_t)gg * CL.total + CL.ready);
            for (int c = lane; c <= n; c += 32) rd[c] = (TT)-1;
            if (MODE != MODE_EXACT) {
                uint32_t *bt = reinterpret_cast<uint32_t *>(wbase + (size_t)gg * CL.total + CL.bits);
                for (int w = lane; w < (two_n + 31) / 32; w += 32) bt[w] = 0u;
            }
        }
        __syncwarp();
        if (MODE != MODE_EXACT) {
            // duplicates / range (schedule.py:134-156): the whole warp streams
            // each candidate's ops, coalesced
            for (int gg = 0; gg < G; ++gg) {
                const int64_t cg = base + gg;
                const int tg = __shfl_sync(VRP_FULL_MASK, total, gg * m);
                const int mg = __shfl_sync(VRP_FULL_MASK, (int)mal, gg * m);
                if (cg >= N || mg) continue;
                uint32_t *bt = reinterpret_cast<uint32_t *>(wbase + (size_t)gg * CL.total + CL.bits);
                bool dup = false;
                for (int j = lane; j < tg; j += 32) {
                    const int op = (int)__ldg(ops + cg * stride + j);
                    if (op < 0 || op >= two_n) { dup = true; continue; }
                    const uint32_t bit = 1u << (op & 31);
                    dup |= (atomicOr(&bt[op >> 5], bit) & bit) != 0;
                }
                const bool anyd = __any_sync(VRP_FULL_MASK, dup);
                if (glane && g == gg) mal |= anyd;
            }
        }
        mal = (__ballot_sync(VRP_FULL_MASK, live && mal) & gmask) != 0;
        const bool run = live && !mal;

        Route R;
        R.re = (live ? cand : 0) * stride + off;
        R.L = run ? L : 0;
        R.i = 0;
        R.staged = 0;
        unsigned bad = 0;  // lanes whose route holds an out-of-range op code
        TT t = 0;
        int s = 0, lo = 0, hi = k, lastc = 0;
        bool dead = false;

        if (MODE == MODE_TWO) {
            // pass 1: no-wait walk; ready = dropoff time + p (schedule.py:371-378)
            for (;;) {
                const unsigned need = __ballot_sync(VRP_FULL_MASK, wants_chunk(R, run));
                if (need) bad |= refill<OpT, INTD>(I, ops, need, R, lane, m, wbase, CL, two_n);
                const bool active = R.i < R.L;
                if (!__any_sync(VRP_FULL_MASK, active)) break;
                if (active) {
                    const int slot = R.i & (WIN - 1);
                    const int op = w_op[slot];
                    const int c = op_customer(op);
                    t = t + (TT)w_leg[slot];
                    if (!(op & 1)) {
                        s_ready[c] = t + s_p[c];
                        s_posd[c] = ((uint32_t)v << 16) | (uint32_t)R.i;
                    }
                    cap_step(op, k, s, lo, hi);
                    ++R.i;
                }
            }
            __syncwarp();
            // pass 2: waits at pickups (schedule.py:380-393), and the same-route
            // pickup-before-its-dropoff Deadlock (:362-369)
            R.i = 0;
            R.staged = 0;
            t = 0;
            for (;;) {
                const unsigned need = __ballot_sync(VRP_FULL_MASK, wants_chunk(R, run));
                if (need) refill<OpT, INTD>(I, ops, need, R, lane, m, wbase, CL, two_n);
                const bool active = R.i < R.L;
                if (!__any_sync(VRP_FULL_MASK, active)) break;
                if (active) {
                    const int slot = R.i & (WIN - 1);
                    const int op = w_op[slot];
                    const int c = op_customer(op);
                    t = t + (TT)w_leg[slot];
                    if (op & 1) {
                        const TT r = s_ready[c];
                        if (r > t) t = r;
                        const uint32_t pd = s_posd[c];
                        dead |= (int)(pd >> 16) == v && (int)(pd & 0xffffu) > R.i;
                    }
                    lastc = c;
                    ++R.i;
                }
            }
        } else {
            for (;;) {
                const unsigned need = __ballot_sync(VRP_FULL_MASK, wants_chunk(R, run && !dead));
                if (need) bad |= refill<OpT, INTD>(I, ops, need, R, lane, m, wbase, CL, two_n);
                const bool active = run && !dead && R.i < R.L;
                const int slot = R.i & (WIN - 1);
                const int op = active ? (int)w_op[slot] : 0;
                const TT lg = (TT)w_leg[slot];
                const int c = op_customer(op);
                const bool pick = op & 1;
                const TT r = s_ready[c];
                const TT pc = s_p[c];
                const bool go = active && !(pick && r < (TT)0);
                const TT arr = t + lg;
                const TT tn = (pick && !(arr >= r)) ? r : arr;
                if (go) {
                    if (!pick) s_ready[c] = tn + pc;
                    if (REC) {
                        const int64_t at = R.re + R.i;
                        arrival_out[at] = (double)arr;
                        time_out[at] = (double)tn;
                    }
                    t = tn;
                    lastc = c;
                    cap_step(op, k, s, lo, hi);
                    ++R.i;
                }
                const unsigned moved = __ballot_sync(VRP_FULL_MASK, go);
                const unsigned left = __ballot_sync(VRP_FULL_MASK, active && R.i < R.L);
                __syncwarp();
                if (!left) break;
                if ((left & gmask) && !(moved & gmask)) dead = true;  // this candidate is stuck
            }
            if (dead)  // finish the capacity test past the stuck position
                for (int j = R.i; j < R.L; ++j) {
                    const int op = (int)__ldg(ops + R.re + j);
                    if ((unsigned)op >= (unsigned)two_n) bad |= 1u << lane;
                    cap_step(op, k, s, lo, hi);
                }
        }
        mal = mal || ((__reduce_or_sync(VRP_FULL_MASK, bad) & gmask) != 0);
        const bool capfail = (__ballot_sync(VRP_FULL_MASK, live && lo > hi) & gmask) != 0;
        const bool gdead = (__ballot_sync(VRP_FULL_MASK, live && dead) & gmask) != 0;
        const int st = mal ? ST_MAL : (capfail ? ST_CAP : (gdead ? ST_DEAD : ST_OK));

        double ret = 0.0;
        if (live && st == ST_OK && L > 0) {
            if (INTD) ret = (double)(t + (TT)__ldg(I.d32 + (int64_t)lastc * I.W));
            else ret = (double)t + __ldg(I.d + (int64_t)lastc * I.W);
        }
        double z = 0.0;  // returns are >= 0; empty routes count as 0
        for (int u = 0; u < m; ++u) {
            const double x = __shfl_sync(VRP_FULL_MASK, ret, glane ? leader + u : lane);
            z = x > z ? x : z;
        }
        const unsigned bm = __ballot_sync(VRP_FULL_MASK, live && ret == z) & gmask;
        if (live && v == 0) {
            z_out[cand] = st == ST_OK ? z : 0.0;
            status_out[cand] = st;
            if (bottleneck_out) bottleneck_out[cand] = bm ? __ffs(bm) - 1 - leader : 0;
        }
        if (live && returns_out) returns_out[cand * m + v] = st == ST_OK ? ret : 0.0;
        if (REC && live && q0_out) q0_out[cand * m + v] = lo;
        __syncwarp();
    }
}

// (candidates per warp, warps per block) maximising resident candidates per SM
struct Shape {
    int G, wpb, blocks;
    size_t smem;
};

template <typename Kern>
int plan(Kern kern, int n, int m, bool intd, int mode, Shape &out) {
    const size_t per_cand = cand_layout(n, m, intd, mode).total;
    const size_t pbytes = block_p_bytes(n);
    const int gmax = 32 / m;
    long best = -1;
    for (int G = gmax; G >= 1; --G) {
        for (int w = 8; w >= 1; --w) {
            const size_t bytes = pbytes + (size_t)w * G * per_cand;
            if (bytes > 227 * 1024) continue;
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
                return -1;
            int blocks = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * w, bytes) != cudaSuccess)
                return -1;
            // most resident candidates; among equals, fewer warps (fewer issued instructions)
            const long score = (long)blocks * w * G * 64 - (long)blocks * w;
            if (blocks > 0 && score > best) { best = score; out = {G, w, blocks, bytes}; }
        }
    }
    if (best < 0) return -2;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out.smem) == cudaSuccess ? 0 : -1;
}

template <typename OpT, bool INTD, int MODE, bool REC>
int launch_t(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
             int64_t N, double *z, int32_t *status, double *returns, int32_t *bottleneck,
             double *arrival, double *timev, int32_t *q0, cudaStream_t stream, int sm_count) {
    auto kern = makespan_kernel<OpT, INTD, MODE, REC>;
    static int cached_n = -1, cached_m = -1;
    static Shape sh;
    if (cached_n != I.n || cached_m != I.m) {
        const int rc = plan(kern, I.n, I.m, INTD, MODE, sh);
        if (rc) return rc;
        cached_n = I.n;
        cached_m = I.m;
    }
    const int64_t per_block = (int64_t)sh.wpb * sh.G;
    const int64_t want = (N + per_block - 1) / per_block;
    int64_t grid = (int64_t)sh.blocks * sm_count;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * sh.wpb, sh.smem, stream>>>(
        I, static_cast<const OpT *>(ops), stride, lens, N, sh.G, z, status, returns, bottleneck,
        arrival, timev, q0);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

template <typename OpT, bool INTD>
int dispatch_mode(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
                  int64_t N, int mode, bool rec, double *z, int32_t *status, double *returns,
                  int32_t *bottleneck, double *arrival, double *timev, int32_t *q0,
                  cudaStream_t stream, int sm_count) {
    if (rec)
        return launch_t<OpT, INTD, MODE_EVAL, true>(I, ops, stride, lens, N, z, status, returns,
                                                    bottleneck, arrival, timev, q0, stream, sm_count);
    switch (mode) {
        case MODE_EXACT:
            return launch_t<OpT, INTD, MODE_EXACT, false>(I, ops, stride, lens, N, z, status, returns,
                                                          bottleneck, nullptr, nullptr, nullptr, stream, sm_count);
        case MODE_EVAL:
            return launch_t<OpT, INTD, MODE_EVAL, false>(I, ops, stride, lens, N, z, status, returns,
                                                         bottleneck, nullptr, nullptr, nullptr, stream, sm_count);
        default:
            return launch_t<OpT, INTD, MODE_TWO, false>(I, ops, stride, lens, N, z, status, returns,
                                                        bottleneck, nullptr, nullptr, nullptr, stream, sm_count);
    }
}

}  // namespace

int launch_makespan(const DevInstance &I, const void *ops, int op_bytes, int64_t stride,
                    const int32_t *lens, int64_t N, int mode, bool rec, double *z, int32_t *status,
                    double *returns, int32_t *bottleneck, double *arrival, double *timev,
                    int32_t *q0, cudaStream_t stream, int sm_count) {
    if (op_bytes == 2) {
        if (I.integral)
            return dispatch_mode<int16_t, true>(I, ops, stride, lens, N, mode, rec, z, status, returns,
                                                bottleneck, arrival, timev, q0, stream, sm_count);
        return dispatch_mode<int16_t, false>(I, ops, stride, lens, N, mode, rec, z, status, returns,
                                             bottleneck, arrival, timev, q0, stream, sm_count);
    }
    if (I.integral)
        return dispatch_mode<int32_t, true>(I, ops, stride, lens, N, mode, rec, z, status, returns,
                                            bottleneck, arrival, timev, q0, stream, sm_count);
    return dispatch_mode<int32_t, false>(I, ops, stride, lens, N, mode, rec, z, status, returns,
                                         bottleneck, arrival, timev, q0, stream, sm_count);
}
