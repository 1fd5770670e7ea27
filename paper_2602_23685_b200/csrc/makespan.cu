// makespan.cu -- K1 (exact event-driven makespan, schedule.py:188-316) and
// K2 (two-pass estimate, schedule.py:345-393) over batches of candidates.
//
// One warp per candidate, persistent grid (148 SMs x resident blocks).
//
//  stage   all 32 lanes: stream the candidate's ops into shared memory
//          (coalesced, evict-first), validate (range / duplicates / count),
//          and gather every leg d[prev][c] from the L2-resident matrix into
//          shared memory -- the gathers do not depend on any time value, so
//          they are issued with full memory-level parallelism;
//  walk    lane v = vehicle v replays its route from shared memory:
//          dropoff  t += leg,  ready[c] = t + p[c]
//          pickup   t = max(t + leg, ready[c])   (blocked while ready[c] unset)
//          Lanes advance in rounds; a round in which no lane advances while
//          ops remain is a circular wait (Deadlock, schedule.py:243-245/308-309).
//          Every value depends only on its DAG predecessors, computed with the
//          reference's operation order, so the result is bit-identical to the
//          reference's round-robin replay whatever the interleaving.
//  reduce  returns = t + d[last][0] (0 for an empty route), z = max, bottleneck
//          = first argmax, status precedence MALFORMED > CAPACITY > DEADLOCK.
//
// The capacity test (route_initial_load, schedule.py:159-185) is the running
// interval [lo, hi] of feasible initial loads; lo only grows and hi only
// shrinks, so "empty at some prefix" == "empty at the end" and the test is
// fused into the walk (finished past a deadlock by a capacity-only scan).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int MODE_EXACT = 0, MODE_EVAL = 1, MODE_TWO = 2;
constexpr uint16_t START_BIT = 0x8000;  // marks the first op of a route in s_op
constexpr int ST_OK = 0, ST_CAP = 1, ST_DEAD = 2, ST_MAL = 3;
constexpr int GATHER_BATCH = 16;         // independent L2 gathers in flight per lane

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <bool INTD>
struct LegType { using T = double; };
template <>
struct LegType<true> { using T = int32_t; };

// Per-warp shared-memory slots (one candidate in flight per warp) ...
struct WarpLayout {
    size_t ready, leg, op, posd, total;
};

__host__ __device__ inline WarpLayout warp_layout(int n, bool intd, int mode) {
    WarpLayout L;
    size_t o = 0;
    L.ready = o; o += align16(sizeof(double) * (size_t)(n + 1));
    L.leg = o;   o += align16((intd ? 4 : 8) * (size_t)(2 * n + 2));   // +2: prefetch overrun
    L.op = o;    o += align16(sizeof(uint16_t) * (size_t)(2 * n + 2));
    L.posd = o;  if (mode == MODE_TWO) o += align16(sizeof(uint16_t) * (size_t)(n + 1));
    L.total = o;
    return L;
}

// ... plus one block-shared copy of p (processing times), read on every dropoff.
__host__ __device__ inline size_t block_p_bytes(int n, bool intd) {
    return align16((intd ? 4 : 8) * (size_t)(n + 1));
}

__device__ __forceinline__ void cap_step(int op, int k, int &s, int &lo, int &hi) {
    if (op & 1) { int room = k - 1 - s; hi = room < hi ? room : hi; ++s; }
    else        { int need = 1 - s;     lo = need > lo ? need : lo; --s; }
}

template <typename OpT, bool INTD, int MODE, bool REC>
__global__ void __launch_bounds__(256)
makespan_kernel(DevInstance I, const OpT *__restrict__ ops, int64_t stride,
                const int32_t *__restrict__ lens, int64_t N, double *__restrict__ z_out,
                int32_t *__restrict__ status_out, double *__restrict__ returns_out,
                int32_t *__restrict__ bottleneck_out, double *__restrict__ arrival_out,
                double *__restrict__ time_out, int32_t *__restrict__ q0_out) {
    using LegT = typename LegType<INTD>::T;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int n = I.n, m = I.m, k = I.k, two_n = 2 * n;
    const WarpLayout Lw = warp_layout(n, INTD, MODE);
    LegT *s_p = reinterpret_cast<LegT *>(smem);
    unsigned char *base = smem + block_p_bytes(n, INTD) + (size_t)warp * Lw.total;
    double *s_ready = reinterpret_cast<double *>(base + Lw.ready);
    uint32_t *s_bits = reinterpret_cast<uint32_t *>(base + Lw.ready);  // validation bitmap (aliases ready)
    LegT *s_leg = reinterpret_cast<LegT *>(base + Lw.leg);
    uint16_t *s_op = reinterpret_cast<uint16_t *>(base + Lw.op);
    uint16_t *s_posd = reinterpret_cast<uint16_t *>(base + Lw.posd);
    const bool vlane = lane < m;

    for (int c = threadIdx.x; c <= n; c += blockDim.x)
        s_p[c] = INTD ? (LegT)__ldg(I.p32 + c) : (LegT)__ldg(I.p + c);
    __syncthreads();

    for (int64_t cand = (int64_t)blockIdx.x * wpb + warp; cand < N;
         cand += (int64_t)gridDim.x * wpb) {
        const OpT *row = ops + cand * stride;
        // ---- route offsets (lane v owns route v)
        int L = vlane ? __ldg(lens + cand * m + lane) : 0;
        int off = L;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(VRP_FULL_MASK, off, o);
            if (lane >= o) off += y;
        }
        const int total = __shfl_sync(VRP_FULL_MASK, off, 31);
        off -= L;  // exclusive
        bool bad = __any_sync(VRP_FULL_MASK, L < 0) || total > two_n ||
                   (MODE != MODE_EXACT && total != two_n) || total > stride;

        // ---- stage ops (streaming loads) + validation
        if (MODE != MODE_EXACT && !bad) {
            for (int w = lane; w < (two_n + 31) / 32; w += 32) s_bits[w] = 0u;
            __syncwarp();
        }
        if (!bad) {
            bool mine_bad = false;
#pragma unroll 4
            for (int j = lane; j < total; j += 32) {
                int op = (int)load_stream(row + j);
                if (op < 0 || op >= two_n) { mine_bad = true; op = 0; }
                s_op[j] = (uint16_t)op;
                if (MODE != MODE_EXACT) {
                    uint32_t bit = 1u << (op & 31);
                    uint32_t prev = atomicOr(&s_bits[op >> 5], bit);
                    if (prev & bit) mine_bad = true;
                }
            }
            bad = __any_sync(VRP_FULL_MASK, mine_bad);
        }
        if (bad) {
            if (lane == 0) {
                z_out[cand] = 0.0;
                status_out[cand] = ST_MAL;
                if (bottleneck_out) bottleneck_out[cand] = 0;
            }
            if (returns_out && vlane) returns_out[cand * m + lane] = 0.0;
            __syncwarp();
            continue;
        }
        __syncwarp();
        if (vlane && L > 0) s_op[off] |= START_BIT;
        __syncwarp();

        // ---- gather legs d[prev][c]: independent of all times, so issue
        // GATHER_BATCH loads per lane before consuming any of them
        for (int j0 = lane; j0 < total; j0 += 32 * GATHER_BATCH) {
            int64_t addr[GATHER_BATCH];
#pragma unroll
            for (int u = 0; u < GATHER_BATCH; ++u) {
                const int j = j0 + 32 * u;
                addr[u] = 0;
                if (j < total) {
                    const int raw = s_op[j];
                    const int c = op_customer(raw & 0x7fff);
                    const int prev = (raw & START_BIT) ? 0 : op_customer(s_op[j - 1] & 0x7fff);
                    addr[u] = (int64_t)prev * I.W + c;
                    if (MODE == MODE_TWO && !(raw & 1)) s_posd[c] = (uint16_t)j;
                }
            }
            LegT v[GATHER_BATCH];
#pragma unroll
            for (int u = 0; u < GATHER_BATCH; ++u)
                v[u] = INTD ? (LegT)__ldg(I.d32 + addr[u]) : (LegT)__ldg(I.d + addr[u]);
#pragma unroll
            for (int u = 0; u < GATHER_BATCH; ++u)
                if (j0 + 32 * u < total) s_leg[j0 + 32 * u] = v[u];
        }
        for (int c = lane; c <= n; c += 32) s_ready[c] = -1.0;  // -1: dropoff not done
        __syncwarp();

        const int end = off + L;
        double t = 0.0;
        int s = 0, lo = 0, hi = k;
        bool dead = false;
        if (MODE == MODE_TWO) {
            // pass 1: no-wait walk, ready = dropoff time + p (schedule.py:371-378);
            // same-route pickup before its own dropoff => Deadlock (:362-369)
            if (vlane) {
                for (int i = off; i < end; ++i) {
                    const int op = s_op[i] & 0x7fff;
                    const int c = op_customer(op);
                    const bool pick = op & 1;
                    t = t + (double)s_leg[i];
                    const double pc = (double)s_p[c];
                    const int pd = s_posd[c];
                    if (!pick) s_ready[c] = t + pc;
                    dead |= pick && pd > i && pd < end;
                    cap_step(op, k, s, lo, hi);
                }
            }
            dead = __any_sync(VRP_FULL_MASK, dead);
            __syncwarp();
            // pass 2: waits at pickups (schedule.py:380-393)
            t = 0.0;
            if (vlane && !dead) {
                for (int i = off; i < end; ++i) {
                    const int op = s_op[i] & 0x7fff;
                    t = t + (double)s_leg[i];
                    const double r = s_ready[op_customer(op)];
                    if ((op & 1) && r > t) t = r;
                }
            }
        } else {
            // Lockstep dataflow replay: every iteration each lane executes the
            // next op of its route unless it is a pickup whose dropoff has not
            // happened yet; writes become visible to the other lanes at the
            // __syncwarp() ending the iteration, so the iteration count is the
            // depth of the precedence DAG.  An iteration in which no lane moves
            // while ops remain is a circular wait.  Branch-free body: both op
            // kinds are evaluated and the result selected.
            int i = off;
            int raw0 = s_op[i], raw1 = s_op[i + 1];
            double leg0 = (double)s_leg[i], leg1 = (double)s_leg[i + 1];
            for (;;) {
                const bool active = vlane && i < end;
                const int op = active ? (raw0 & 0x7fff) : 0;  // past the end: stale slot
                const int c = op_customer(op);
                const bool pick = op & 1;
                const double r = s_ready[c];
                const double pc = (double)s_p[c];
                const bool go = active && !(pick && r < 0.0);
                const double arr = t + leg0;
                const double tn = (pick && !(arr >= r)) ? r : arr;
                if (go) {
                    if (!pick) s_ready[c] = tn + pc;
                    if (REC) { arrival_out[cand * stride + i] = arr; time_out[cand * stride + i] = tn; }
                    t = tn;
                    cap_step(op, k, s, lo, hi);
                    ++i;
                    raw0 = raw1; leg0 = leg1;
                    raw1 = s_op[i + 1];
                    leg1 = (double)s_leg[i + 1];
                }
                const unsigned moved = __ballot_sync(VRP_FULL_MASK, go);
                const unsigned left = __ballot_sync(VRP_FULL_MASK, vlane && i < end);
                __syncwarp();
                if (!left) break;
                if (!moved) { dead = true; break; }
            }
            if (dead && vlane)  // finish the capacity test past the stuck position
                for (int j = i; j < end; ++j) cap_step(s_op[j] & 0x7fff, k, s, lo, hi);
        }
        const bool capfail = __any_sync(VRP_FULL_MASK, vlane && lo > hi);
        const int st = capfail ? ST_CAP : (dead ? ST_DEAD : ST_OK);

        double ret = 0.0;
        if (st == ST_OK && vlane && L > 0)
            ret = t + dist<INTD>(I, op_customer(s_op[end - 1] & 0x7fff), 0);
        double z = warp_max(ret);  // returns are >= 0; empty routes count as 0
        if (st != ST_OK) z = 0.0;
        const unsigned bmask = __ballot_sync(VRP_FULL_MASK, vlane && ret == z);
        if (lane == 0) {
            z_out[cand] = z;
            status_out[cand] = st;
            if (bottleneck_out) bottleneck_out[cand] = bmask ? __ffs(bmask) - 1 : 0;
        }
        if (returns_out && vlane) returns_out[cand * m + lane] = st == ST_OK ? ret : 0.0;
        if (REC && q0_out && vlane) q0_out[cand * m + lane] = lo;
        __syncwarp();
    }
}

template <typename OpT, bool INTD, int MODE, bool REC>
int launch_t(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
             int64_t N, double *z, int32_t *status, double *returns, int32_t *bottleneck,
             double *arrival, double *timev, int32_t *q0, cudaStream_t stream, int sm_count) {
    auto kern = makespan_kernel<OpT, INTD, MODE, REC>;
    const size_t per_warp = warp_layout(I.n, INTD, MODE).total;
    const size_t shared_p = block_p_bytes(I.n, INTD);
    // choose warps/block maximising resident warps per SM under the smem
    // budget; cached per instantiation for the last per-warp footprint
    static size_t cached_pw = 0;
    static int cached_w = 0, cached_blocks = 0;
    int best_w = 1, best_res = 0, best_blocks = 1;
    const bool hit = cached_pw == per_warp;
    if (hit) { best_w = cached_w; best_blocks = cached_blocks; best_res = 1; }
    for (int w = 8; w >= 1 && !hit; --w) {
        size_t bytes = shared_p + per_warp * (size_t)w;
        if (bytes > 227 * 1024) continue;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
            return -1;
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * w, bytes) != cudaSuccess)
            return -1;
        if (blocks * w > best_res) { best_res = blocks * w; best_w = w; best_blocks = blocks; }
    }
    if (best_res == 0) return -2;
    size_t bytes = shared_p + per_warp * (size_t)best_w;
    if (cached_pw != per_warp) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        cached_pw = per_warp; cached_w = best_w; cached_blocks = best_blocks;
    }
    int64_t want = (N + best_w - 1) / best_w;
    int64_t grid = (int64_t)best_blocks * sm_count;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * best_w, bytes, stream>>>(
        I, static_cast<const OpT *>(ops), stride, lens, N, z, status, returns, bottleneck,
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
