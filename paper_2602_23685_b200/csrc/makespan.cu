// makespan.cu -- K1 (exact event-driven makespan, schedule.py:188-316) and
// K2 (two-pass estimate, schedule.py:345-393) over batches of candidates.
//
// Mapping: a warp carries G = floor(32/m) candidates at once, lane g*m+v owns
// route v of candidate g (30 of 32 lanes busy for m = 6); persistent grid.
//
// Each lane streams its own route through a register pipeline -- op codes
// loaded OPS_AHEAD positions ahead (read-only path, L1 line reuse), legs
// d[prev][c] gathered from the L2-resident matrix LEGS_AHEAD positions ahead --
// so the only shared memory a candidate needs is its ready table
// ready[c] = t_drop[c] + p[c] (fp64, n+1 slots) plus one block-shared copy of
// p.  That keeps ~25 candidates in flight per SM at n = 999.
//
// Replay (exact / evaluate): lockstep dataflow.  Every iteration each lane
// executes the next op of its route unless it is a pickup whose dropoff has
// not happened yet (ready < 0):
//     dropoff  t = t + leg;                 ready[c] = t + p[c]
//     pickup   arr = t + leg;  t = arr >= ready[c] ? arr : ready[c]
// Writes become visible to the other lanes at the __syncwarp() closing the
// iteration, so the iteration count is the depth of the precedence DAG.  A
// candidate whose lanes all stall while ops remain is a circular wait
// (Deadlock, schedule.py:243-245 / :308-309).  Each value depends only on its
// DAG predecessors and is computed with the reference's fp64 operation order,
// so results are bit-identical to the reference's round-robin replay.
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
constexpr int ST_RETRY = 4;                 // internal: narrow ready table overflowed
constexpr uint32_t NOT_READY32 = 0xFFFFFFFFu;
constexpr int OPS_AHEAD = 8;   // op codes in registers (positions i .. i+7)
constexpr int LEGS_AHEAD = 4;  // gathered legs in registers (positions i .. i+3)
#ifndef K2_LEGS_AHEAD
#define K2_LEGS_AHEAD 12  // two-pass (K2) pipeline depths: shared memory caps K2 at 8 warps/SM (LS cross pass at n = 999, legs / ops: 4 / 8 1.78 s, 8 / 12 1.70 s; after the pass-1 duplicate check 8 / 12 1.53 s, 12 / 16 1.48 s)
#endif
#ifndef K2_OPS_AHEAD
#define K2_OPS_AHEAD 16
#endif
#ifndef VRP_K1_RA
#define VRP_K1_RA 0  // run-ahead ops per lockstep round (exact mode, slot table); measured slower, see DESIGN.md
#endif

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Per candidate: ready table, plus (validating modes) an op bitmap and (two-
// pass) the (route, position) of every dropoff.
struct CandLayout {
    size_t ready, vals, freem, bits, posd, total;
};

// COMPACT: ready[] becomes a u8 slot id per customer (0xFF = not dropped) into
// SLOTS uint32 ready values (see makespan_kernel).
constexpr int SLOTS = 32;  // ready slots per candidate

__host__ __device__ inline CandLayout cand_layout(int n, int mode, int ready_bytes = 8, bool compact = false) {
    CandLayout L;
    size_t o = 0;
    L.ready = o;
    if (compact) {  // u8 slot id per customer + SLOTS ready values
        o += align16((size_t)(n + 1));
        L.vals = o; o += align16(sizeof(uint32_t) * SLOTS);
        L.freem = o;
    } else {
        o += align16((size_t)ready_bytes * (size_t)(n + 1));
        L.vals = L.freem = 0;
    }
    L.bits = o;  if (mode != MODE_EXACT) o += align16(sizeof(uint32_t) * (size_t)((2 * n + 31) / 32));
    // two-pass: the dropoff route of every customer, u8 (bit 7: passed by pass 2)
    L.posd = o;  if (mode == MODE_TWO) o += align16((size_t)(n + 1));
    L.total = o;
    return L;
}

__host__ __device__ inline size_t block_p_bytes(int n) { return align16(sizeof(double) * (size_t)(n + 1)); }

// a << b with PTX semantics: b >= 32 gives 0 (C++ leaves it undefined)
__device__ __forceinline__ unsigned shl_clamped(unsigned a, unsigned b) {
    unsigned r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

__device__ __forceinline__ void cap_step(int op, int k, int &s, int &lo, int &hi) {
    if (op & 1) { int room = k - 1 - s; hi = room < hi ? room : hi; ++s; }
    else        { int need = 1 - s;     lo = need > lo ? need : lo; --s; }
}

// One route's op codes and legs, streamed through registers.  Loads enter at
// the back of the pipeline and are only consumed stages later, so neither the
// op load (L1) nor the leg gather (L2) sits on the per-iteration critical
// path: an op code is range-checked when it reaches the gather stage
// (LEGS_AHEAD-1), a gathered leg is converted to fp64 when it reaches stage 0.
// Positions past the end read as -1; out-of-range codes set `bad` and are
// replaced by op 0 so that no gather leaves the matrix.
template <bool INTD>
struct LegRaw { using T = double; };
template <>
struct LegRaw<true> { using T = int32_t; };

template <bool INTD>
__device__ __forceinline__ typename LegRaw<INTD>::T gather_leg(const DevInstance &I, int a, int b) {
    // L2-only load: the random d gathers must not evict the op-stream lines from L1.
    // 32-bit index: n <= 8192 (vrp_instance_create), so W^2 < 2^27
    const uint32_t idx = (uint32_t)a * (uint32_t)I.W + (uint32_t)b;
    if (INTD) return (typename LegRaw<INTD>::T)__ldcg(I.d32 + idx);
    return (typename LegRaw<INTD>::T)__ldcg(I.d + idx);
}

// Event-time arithmetic: integral instances (every d and p an integer < 2^31,
// all TSPLIB types) keep times in int64 -- exact, hence bit-identical to the
// reference's fp64 sums, with short ALU latencies on the replay's critical
// path; other instances use fp64 in the reference's operation order.
template <bool INTD>
using TimeT = typename std::conditional<INTD, long long, double>::type;

template <typename OpT, bool INTD, int OA = OPS_AHEAD, int LA = LEGS_AHEAD>
struct RouteStream {
    using LT = typename LegRaw<INTD>::T;
    using TT = TimeT<INTD>;
    const OpT *rp;
    int L, i, two_n, lastp;
    int o[OA];
    LT l[LA];
    bool bad;

    // Loads never feed a select: positions past the end re-read the last op
    // (in bounds); the -1 sentinel is applied by checked() stages later.
    __device__ __forceinline__ int fetch(int pos) const { return (int)__ldg(rp + (pos < L ? pos : lastp)); }
    // validate the op at route position `pos` (past the end -> -1 sentinel)
    __device__ __forceinline__ int checked(int op, int pos) {
        if (pos >= L) return -1;
        if ((unsigned)op >= (unsigned)two_n) { bad = true; return 0; }
        return op;
    }
    __device__ __forceinline__ LT leg(const DevInstance &I, int prev_op, int op) const {
        if (op < 0) return (LT)0;
        return gather_leg<INTD>(I, prev_op < 0 ? 0 : op_customer(prev_op), op_customer(op));
    }
    __device__ __forceinline__ TT leg0() const { return (TT)l[0]; }
    __device__ __forceinline__ void init(const DevInstance &I, const OpT *route, int len, int n2) {
        rp = route; L = len; i = 0; two_n = n2; bad = false;
        lastp = len > 0 ? len - 1 : 0;  // len == 0: rp points inside the row, never consumed
#pragma unroll
        for (int q = 0; q < OA; ++q) o[q] = fetch(q);
#pragma unroll
        for (int q = 0; q < LA; ++q) o[q] = checked(o[q], q);
        l[0] = leg(I, -1, o[0]);
#pragma unroll
        for (int q = 1; q < LA; ++q) l[q] = leg(I, o[q - 1], o[q]);
    }
    __device__ __forceinline__ void advance(const DevInstance &I) {
        ++i;
#pragma unroll
        for (int q = 0; q + 1 < OA; ++q) o[q] = o[q + 1];
        o[OA - 1] = fetch(i + OA - 1);
        o[LA - 1] = checked(o[LA - 1], i + LA - 1);
#pragma unroll
        for (int q = 0; q + 1 < LA; ++q) l[q] = l[q + 1];
        l[LA - 1] = leg(I, o[LA - 2], o[LA - 1]);
    }
    // re-read and validate the op at `pos` (capacity scan past a deadlock)
    __device__ __forceinline__ int checked_at(int pos) { return checked(fetch(pos), pos); }
};

// NARROW (integral instances, exact/evaluate): the ready table stores uint32
// (NOT_READY32 = not yet dropped) -- half the shared memory per candidate,
// twice the resident candidates.  Times are still computed in int64; a value
// that does not fit marks the candidate ST_RETRY and the launcher re-runs just
// those candidates with the 64-bit table (`fixup`), so results stay exact.
//
// COMPACT (with NARROW, when m*k <= SLOTS): resources are conserved, so at
// any point of any replay order the customers whose dropoff is done and
// pickup is not number sum_v (q0_v - load_v) <= sum_v lo_v <= m*k for a
// capacity-feasible candidate.  The ready table then needs only SLOTS values:
// the candidate's free-slot mask is a register replicated over its lanes;
// lanes dropping in the same iteration take the lowest free slots in lane
// order (ballot rank), record the slot in a u8-per-customer map, and pickups
// read the map, then the value, and return the slot (a rotation OR over the
// candidate's lanes).  ~1.3 KB instead of 4 KB per candidate at n = 999, so
// residency is set by registers, not shared memory.  A candidate that runs
// out of slots is capacity-infeasible (status CAPACITY regardless) -- or,
// should that reasoning ever fail, goes to the 64-bit fix-up pass (ST_RETRY).
//
// MC > 0 fixes the fleet size at compile time (MC == I.m; the m = 6 fleets of
// every benchmark config beyond gr17): lane/candidate indexing, the slot
// classes and the rotation OR then cost no run-time tests.
template <typename OpT, bool INTD, int MODE, bool REC, bool NARROW, bool COMPACT = false, int MC = 0, int RA = 0>
__global__ void __launch_bounds__(256)
makespan_kernel(DevInstance I, const OpT *__restrict__ ops, int64_t stride,
                const int32_t *__restrict__ lens, int64_t N, int G, double *__restrict__ z_out,
                int32_t *__restrict__ status_out, double *__restrict__ returns_out,
                int32_t *__restrict__ bottleneck_out, double *__restrict__ arrival_out,
                double *__restrict__ time_out, int32_t *__restrict__ q0_out, int fixup) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int n = I.n, m = MC ? MC : I.m, k = I.k, two_n = 2 * n;
    // NARROW: event times in uint32 (every value the narrow table can hold);
    // a wrap-around is detected and sends the candidate to the 64-bit pass
    using TT = typename std::conditional<NARROW, uint32_t, TimeT<INTD>>::type;
    using RT = typename std::conditional<NARROW, uint32_t, TT>::type;
    const CandLayout CL = cand_layout(n, MODE, (int)sizeof(RT), COMPACT);
    TT *s_p = reinterpret_cast<TT *>(smem);
    unsigned char *wbase = smem + block_p_bytes(n) + (size_t)warp * G * CL.total;

    const int g = lane / m, v = lane - (lane / m) * m;
    const bool glane = g < G;
    const unsigned gmask = glane ? (((m == 32) ? 0xffffffffu : ((1u << m) - 1u)) << (g * m)) : 0u;
    const int leader = g * m;  // lane holding route 0 of this lane's candidate
    unsigned char *cbase = wbase + (size_t)(glane ? g : 0) * CL.total;
    RT *s_ready = reinterpret_cast<RT *>(cbase + CL.ready);
    uint8_t *s_sid = cbase + CL.ready;
    uint32_t *s_val = reinterpret_cast<uint32_t *>(cbase + CL.vals);
    uint8_t *s_posd = cbase + CL.posd;

    for (int c = threadIdx.x; c <= n; c += blockDim.x)
        s_p[c] = INTD ? (TT)__ldg(I.p32 + c) : (TT)__ldg(I.p + c);
    __syncthreads();

    const int64_t step = (int64_t)gridDim.x * wpb * G;
    for (int64_t base = ((int64_t)blockIdx.x * wpb + warp) * G; base < N; base += step) {
        const int64_t cand = base + g;
        const bool live = glane && cand < N && (!fixup || status_out[cand] == ST_RETRY);
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
        const OpT *row = ops + (live ? cand : 0) * stride;

        // ---- shared tables: ready = -1 (dropoff not done); validation bitmap
        for (int gg = 0; gg < G; ++gg) {
            if (COMPACT) {
                uint32_t *sd = reinterpret_cast<uint32_t *>(wbase + (size_t)gg * CL.total + CL.ready);
                for (int w = lane; w < (n + 4) / 4; w += 32) sd[w] = 0xFFFFFFFFu;
            } else {
                RT *rd = reinterpret_cast<RT *>(wbase + (size_t)gg * CL.total + CL.ready);
                for (int c = lane; c <= n; c += 32) rd[c] = NARROW ? (RT)NOT_READY32 : (RT)-1;
            }
            if (MODE != MODE_EXACT) {
                uint32_t *bt = reinterpret_cast<uint32_t *>(wbase + (size_t)gg * CL.total + CL.bits);
                for (int w = lane; w < (two_n + 31) / 32; w += 32) bt[w] = 0u;
            }
        }
        __syncwarp();
        if (MODE == MODE_EVAL) {
            // duplicates / range (schedule.py:134-156): the whole warp streams
            // each candidate's ops, coalesced (two-pass: inside pass 1, below)
            for (int gg = 0; gg < G; ++gg) {
                const int64_t cg = base + gg;
                const int tg = __shfl_sync(VRP_FULL_MASK, total, gg * m);
                const int mg = __shfl_sync(VRP_FULL_MASK, (int)mal, gg * m);
                if (cg >= N || mg) continue;
                uint32_t *bt = reinterpret_cast<uint32_t *>(wbase + (size_t)gg * CL.total + CL.bits);
                bool dup = false;
                // VB op codes in flight per lane (the first touch of the row
                // comes from HBM; one load per shared atomic left the warp
                // waiting on every load)
                constexpr int VB = 8;
                for (int j0 = 0; j0 < tg; j0 += 32 * VB) {
                    int ov[VB];
#pragma unroll
                    for (int u = 0; u < VB; ++u) {
                        const int j = j0 + u * 32 + lane;
                        ov[u] = j < tg ? (int)__ldg(ops + cg * stride + j) : 0;
                    }
#pragma unroll
                    for (int u = 0; u < VB; ++u) {
                        if (j0 + u * 32 + lane >= tg) continue;
                        const int op = ov[u];
                        if (op < 0 || op >= two_n) { dup = true; continue; }
                        const uint32_t bit = 1u << (op & 31);
                        dup |= (atomicOr(&bt[op >> 5], bit) & bit) != 0;
                    }
                }
                const bool anyd = __any_sync(VRP_FULL_MASK, dup);
                if (glane && g == gg) mal |= anyd;
            }
        }
        mal = (__ballot_sync(VRP_FULL_MASK, live && mal) & gmask) != 0;
        const bool run = live && !mal;

        RouteStream<OpT, INTD, MODE == MODE_TWO ? K2_OPS_AHEAD : OPS_AHEAD, MODE == MODE_TWO ? K2_LEGS_AHEAD : LEGS_AHEAD> rs;
        rs.init(I, row + (run && L > 0 ? off : 0), run ? L : 0, two_n);
        TT t = 0;
        int s = 0, lo = 0, hi = k, lastc = 0;
        bool dead = false, bad_ops = false, ovf = false, dup = false;

        if (MODE == MODE_TWO) {
            // pass 1: no-wait walk; ready = dropoff time + p (schedule.py:371-378).
            // Each lane also marks its route's ops in the candidate's bitmap:
            // a second mark is a duplicate (the reference's structural check,
            // schedule.py:134-156; ranges are checked by the stream)
            uint32_t *bt = reinterpret_cast<uint32_t *>(cbase + CL.bits);
            while (rs.i < rs.L) {
                const int op = rs.o[0];
                const int c = op_customer(op);
                {
                    const uint32_t bit = 1u << (op & 31);
                    dup |= (atomicOr(&bt[op >> 5], bit) & bit) != 0;
                }
                const TT tn = t + (TT)rs.leg0();
                if (NARROW) ovf |= tn < t;  // uint32 wrap -> 64-bit fix-up pass
                t = tn;
                if (!(op & 1)) {
                    const TT rv = t + s_p[c];
                    if (NARROW) ovf |= rv < t;
                    s_ready[c] = (RT)rv;
                    s_posd[c] = (uint8_t)v;  // every customer's dropoff route (valid candidates: each once)
                }
                cap_step(op, k, s, lo, hi);
                lastc = c;
                rs.advance(I);
            }
            bad_ops = rs.bad;
            __syncwarp();
            // pass 2: waits at pickups (schedule.py:380-393), and the same-route
            // pickup-before-its-dropoff Deadlock (:362-369)
            rs.init(I, row + (run && L > 0 ? off : 0), run ? L : 0, two_n);
            t = 0;
            while (rs.i < rs.L) {
                const int op = rs.o[0];
                const int c = op_customer(op);
                const TT tn = t + (TT)rs.leg0();
                if (NARROW) ovf |= tn < t;
                t = tn;
                if (op & 1) {
                    const TT r = (TT)s_ready[c];
                    if (r > t) t = r;
                    // its dropoff is on this route and not passed yet: a pickup before it
                    const int pd = s_posd[c];
                    dead |= (pd & 0x7F) == v && !(pd & 0x80);
                } else {
                    s_posd[c] = (uint8_t)(v | 0x80);  // only this lane touches route v's dropoffs
                }
                rs.advance(I);
            }
        } else {
            // COMPACT: the free-slot mask (replicated over the candidate's lanes) and
            // the rotation partners of its OR: after step s lane v holds v .. v+2^s-1 (mod m)
            unsigned freem = ~0u;
            const int pt1 = glane ? leader + (v + 1) % m : lane, pt2 = glane ? leader + (v + 2) % m : lane;
            const int pt4 = glane ? leader + (v + 4) % m : lane, pt8 = glane ? leader + (v + 8) % m : lane;
            const int pt16 = glane ? leader + (v + 16) % m : lane;
            unsigned cls = 0, cls_next = 0;  // slot classes {v, v+m, ...} of this and the next route
            for (int q = v; q < SLOTS; q += m) cls |= 1u << q;
            for (int q = (v + 1) % m; q < SLOTS; q += m) cls_next |= 1u << q;
            for (;;) {
                const bool active = run && !dead && rs.i < rs.L;
                const int op = active ? rs.o[0] : 0;
                const int c = op_customer(op);
                const bool pick = op & 1;
                TT r;
                bool rdy;  // a pickup's dropoff has happened (dropoffs: always)
                int sid = 0xFF;
                if (COMPACT) {
                    sid = s_sid[c];
                    rdy = !pick || sid != 0xFF;
                    r = (TT)s_val[sid & (SLOTS - 1)];
                } else {
                    const RT rraw = s_ready[c];
                    r = (TT)rraw;
                    rdy = NARROW ? (!pick || rraw != (RT)NOT_READY32) : !(pick && r < (TT)0);
                }
                const TT pc = s_p[c];
                const bool go = active && rdy;
                const TT arr = t + (TT)rs.leg0();
                if (NARROW) ovf |= arr < t;  // uint32 wrap
                const TT tn = (pick && !(arr >= r)) ? r : arr;
                int slot = SLOTS;
                if (COMPACT) {
                    // a dropping lane takes the lowest free slot of its own class
                    // (slots = v mod m), so lanes never collide; if some lane's class
                    // is exhausted, every dropping lane of the warp takes the
                    // rank-th lowest free slot of its candidate instead (rare)
                    const bool dgo = go && !pick;
                    const unsigned mine = freem & cls;
                    const bool own = dgo && mine;
                    if (own) slot = __ffs(mine) - 1;
                    const bool need = dgo && !mine;
                    if (__any_sync(VRP_FULL_MASK, need)) {
                        // borrow from the next route's class: its lowest free slot, or
                        // the second lowest when that route takes its own lowest now
                        const bool nxt_own = __shfl_sync(VRP_FULL_MASK, own, pt1);
                        const unsigned nx = freem & cls_next;
                        const unsigned cand = nxt_own ? (nx & (nx - 1)) : nx;
                        if (need && cand) slot = __ffs(cand) - 1;
                        const bool stuck = need && !cand;
                        if (__any_sync(VRP_FULL_MASK, stuck)) {  // (only ever after a borrow)
                            const unsigned dm = __ballot_sync(VRP_FULL_MASK, dgo) & gmask;
                            unsigned x = freem;
                            const int below = __popc(dm & lanemask_lt());
                            slot = SLOTS;
                            for (int q = 0, kq = __popc(dm); q < kq && x; ++q) {
                                if (q == below && dgo) slot = __ffs(x) - 1;
                                x &= x - 1;
                            }
                        }
                    }
                    // slots taken (were free) and returned by pickups (were taken)
                    // flip; the XOR of all of them is one OR over the candidate's lanes
                    // (PTX shl clamps shift amounts >= 32 to a zero result: slot = SLOTS
                    // means none taken, sid = 0xFF none returned)
                    unsigned tg = shl_clamped(1u, dgo ? (unsigned)slot : 32u) |
                                  shl_clamped(1u, (go && pick) ? (unsigned)sid : 32u);
                    tg |= __shfl_sync(VRP_FULL_MASK, tg, pt1);
                    if (m > 2) tg |= __shfl_sync(VRP_FULL_MASK, tg, pt2);
                    if (m > 4) tg |= __shfl_sync(VRP_FULL_MASK, tg, pt4);
                    if (m > 8) tg |= __shfl_sync(VRP_FULL_MASK, tg, pt8);
                    if (m > 16) tg |= __shfl_sync(VRP_FULL_MASK, tg, pt16);
                    freem ^= tg;
                }
                if (go) {
                    if (COMPACT) {
                        if (!pick) {
                            const TT rv = tn + pc;
                            ovf |= slot >= SLOTS || rv < tn || rv == (TT)NOT_READY32;
                            if (slot < SLOTS) {
                                s_val[slot] = (uint32_t)rv;
                                s_sid[c] = (uint8_t)slot;
                            }
                        }
                    } else if (!pick) {
                        const TT rv = tn + pc;
                        if (NARROW) {
                            ovf |= rv < tn || rv == (TT)NOT_READY32;
                            s_ready[c] = (RT)rv;
                        } else {
                            s_ready[c] = (RT)rv;
                        }
                    }
                    if (REC) {
                        const int64_t at = cand * stride + off + rs.i;
                        arrival_out[at] = (double)arr;
                        time_out[at] = (double)tn;
                    }
                    t = tn;
                    lastc = c;
                    cap_step(op, k, s, lo, hi);
                    rs.advance(I);
                }
                if (RA > 0) {
                    // Run-ahead (exact mode, slot table): a lane that moved keeps
                    // executing its route -- up to RA more ops -- while its pickups'
                    // dropoffs are visible and its own slot class has room, with no
                    // warp collective per op.  Visibility: the __syncwarp publishes
                    // this round's first ops; a run-ahead drop writes its value, then
                    // a block fence, then the slot id, and a run-ahead pickup reads
                    // the slot id, fences, then the value (message passing), so a
                    // pickup either sees its dropoff complete or stops.  Values only
                    // depend on DAG predecessors, so results are unchanged.  Slot
                    // bookkeeping: a lane toggles slots of its own class (takes, and
                    // releases of its own customers) and releases foreign slots; per
                    // round a slot has at most one net own-class toggle (its class
                    // owner) and at most one foreign release (a slot freed by another
                    // lane is invisible to its owner until the merge), so
                    // start ^ OR(own toggles) ^ OR(foreign toggles) is the exact new
                    // free mask.
                    __syncwarp();
                    const unsigned f0 = freem;
                    unsigned flips = 0;
                    volatile uint8_t *vsid = s_sid;
                    volatile uint32_t *vval = s_val;
                    for (int ra = 0; ra < RA && go && rs.i < rs.L; ++ra) {
                        const int op2 = rs.o[0];
                        const int c2 = op_customer(op2);
                        const TT arr2 = t + (TT)rs.leg0();
                        TT tn2 = arr2;
                        if (op2 & 1) {
                            const int sid2 = vsid[c2];
                            if (sid2 == 0xFF) break;
                            __threadfence_block();
                            const TT r2 = (TT)vval[sid2 & (SLOTS - 1)];
                            if (!(arr2 >= r2)) tn2 = r2;
                            const unsigned bit = 1u << (sid2 & (SLOTS - 1));
                            flips ^= bit;
                            freem ^= bit;
                        } else {
                            const unsigned av = freem & cls;
                            if (!av) break;
                            const int sl = __ffs(av) - 1;
                            const TT rv = arr2 + s_p[c2];
                            ovf |= rv < arr2 || rv == (TT)NOT_READY32;
                            vval[sl] = (uint32_t)rv;
                            __threadfence_block();
                            vsid[c2] = (uint8_t)sl;
                            flips ^= 1u << sl;
                            freem ^= 1u << sl;
                        }
                        ovf |= arr2 < t;
                        t = tn2;
                        lastc = c2;
                        cap_step(op2, k, s, lo, hi);
                        rs.advance(I);
                    }
                    if (__any_sync(VRP_FULL_MASK, flips != 0)) {
                        unsigned tk = flips & cls, rl = flips & ~cls;
                        tk |= __shfl_sync(VRP_FULL_MASK, tk, pt1);
                        rl |= __shfl_sync(VRP_FULL_MASK, rl, pt1);
                        if (m > 2) { tk |= __shfl_sync(VRP_FULL_MASK, tk, pt2); rl |= __shfl_sync(VRP_FULL_MASK, rl, pt2); }
                        if (m > 4) { tk |= __shfl_sync(VRP_FULL_MASK, tk, pt4); rl |= __shfl_sync(VRP_FULL_MASK, rl, pt4); }
                        if (m > 8) { tk |= __shfl_sync(VRP_FULL_MASK, tk, pt8); rl |= __shfl_sync(VRP_FULL_MASK, rl, pt8); }
                        if (m > 16) { tk |= __shfl_sync(VRP_FULL_MASK, tk, pt16); rl |= __shfl_sync(VRP_FULL_MASK, rl, pt16); }
                        freem = f0 ^ tk ^ rl;
                    } else {
                        freem = f0;
                    }
                }
                const unsigned moved = __ballot_sync(VRP_FULL_MASK, go);
                const unsigned left = __ballot_sync(VRP_FULL_MASK, active && rs.i < rs.L);
                __syncwarp();
                if (!left) break;
                if ((left & gmask) && !(moved & gmask)) dead = true;  // this candidate is stuck
            }
            if (dead)  // finish the capacity test past the stuck position
                for (int j = rs.i; j < rs.L; ++j) cap_step(rs.checked_at(j), k, s, lo, hi);
            bad_ops = rs.bad;
        }
        mal = mal || ((__ballot_sync(VRP_FULL_MASK, live && (bad_ops || dup)) & gmask) != 0);
        const bool capfail = (__ballot_sync(VRP_FULL_MASK, live && lo > hi) & gmask) != 0;
        const bool gdead = (__ballot_sync(VRP_FULL_MASK, live && dead) & gmask) != 0;
        const bool govf = NARROW && (__ballot_sync(VRP_FULL_MASK, live && ovf) & gmask) != 0;
        const int st = mal ? ST_MAL : (govf ? ST_RETRY : (capfail ? ST_CAP : (gdead ? ST_DEAD : ST_OK)));

        double ret = 0.0;
        if (live && st == ST_OK && L > 0) {
            if (INTD) ret = (double)((long long)t + (long long)__ldg(I.d32 + (int64_t)lastc * I.W));
            else ret = (double)t + __ldg(I.d + (int64_t)lastc * I.W);
        }
        double z = 0.0;  // returns are >= 0; empty routes count as 0
        for (int u = 0; u < m; ++u) {
            const double x = __shfl_sync(VRP_FULL_MASK, ret, glane ? leader + u : lane);
            z = x > z ? x : z;
        }
        const unsigned bm = __ballot_sync(VRP_FULL_MASK, live && ret == z) & gmask;
        __syncwarp();  // every lane has read status_out (fixup) before lane 0 rewrites it
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

#ifndef VRP_K1_SERIAL
#define VRP_K1_SERIAL 0  // thread-per-candidate exact replay; measured slower, see DESIGN.md
#endif
#if VRP_K1_SERIAL
// ---------------------------------------------------------------------------
// Thread-per-candidate exact replay (integral instances, m = M fixed, m*k <=
// SLOTS) -- the round-2 A/B against the lockstep warp replay above, compiled
// out (VRP_K1_SERIAL=0): bit-exact (the parity suite passes with it) but
// 20.6 M evals/s against 44.5 M at n = 999.  The per-candidate slot table
// (1.1 KB of shared memory per thread) caps residency at 6 warps/SM, and
// advancing one of six register-resident route pipelines without branching
// costs ~150 instructions per route-round in register moves and selects
// (13.5 k warp instructions per evaluation, IPC 0.91; DESIGN.md §3 K1).
//
// One thread owns one candidate and all M of its routes; each round visits
// the routes in order 0..M-1 and executes the next op of each that can go.
// Everything the lockstep warp replay spends on lane coordination -- ballots,
// the slot-mask rotation OR, shuffles, __syncwarp per round -- disappears:
// the free-slot mask is one register of the thread, and a dropoff executed on
// route v is visible to a pickup on route w > v in the same round (program
// order), so rounds <= the lockstep's DAG depth.  Results depend only on the
// precedence DAG (every value is a max-plus function of its predecessors), so
// they equal the reference's round-robin replay (schedule.py:265-316).
//
// The M route streams (op codes OA ahead, L2 leg gathers LA ahead) live in
// registers (full unroll over the compile-time fleet); shared memory holds the
// candidate's slot table: a u8 slot id per customer (0xFF = not dropped, 0xFE
// = already picked up) and SLOTS uint32 ready values, laid out so that the 32
// threads of a warp always hit 32 distinct banks (word index = x * 32 + lane).
// Event times are uint32; a wrap, an exhausted slot mask (capacity-infeasible
// by the conservation argument above) or a second pickup of one customer send
// the candidate to the 64-bit fix-up pass (ST_RETRY), so results stay exact.
// predicated loads: the replay advances a route only when its op executes,
// without branching the warp
__device__ __forceinline__ int ldg_if(const int16_t *p, bool pr, int old) {
    int r = old;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.s16 %0, [%1];\n\t}"
                 : "+r"(r) : "l"(p), "r"((int)pr));
    return r;
}
__device__ __forceinline__ int ldg_if(const int32_t *p, bool pr, int old) {
    int r = old;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.b32 %0, [%1];\n\t}"
                 : "+r"(r) : "l"(p), "r"((int)pr));
    return r;
}
__device__ __forceinline__ int ldcg_if(const int32_t *p, bool pr, int old) {
    int r = old;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.b32 %0, [%1];\n\t}"
                 : "+r"(r) : "l"(p), "r"((int)pr));
    return r;
}

// One route of the thread-per-candidate replay: op codes OA ahead, and at the
// gather stage (LA-1) the leg d[prev][c] from L2 plus p[c] (used by dropoffs),
// so nothing the replay reads at stage 0 is a fresh load.  advance_if(go)
// moves the pipeline only when go (selects + predicated loads, no branch).
template <typename OpT, int OA, int LA>
struct SerialRoute {
    const OpT *rp;
    int L, i, lastp, two_n;
    bool bad;
    int o[OA];
    int32_t l[LA], pp[LA];

    __device__ __forceinline__ const OpT *at(int pos) const { return rp + (pos < L ? pos : lastp); }
    __device__ __forceinline__ int checked(int op, int pos) {
        if (pos >= L) return -1;
        if ((unsigned)op >= (unsigned)two_n) { bad = true; return 0; }
        return op;
    }
    __device__ __forceinline__ uint32_t gidx(const DevInstance &I, int prev_op, int op) const {
        const int a = prev_op < 0 ? 0 : op_customer(prev_op);
        return (uint32_t)a * (uint32_t)I.W + (uint32_t)op_customer(op < 0 ? 0 : op);
    }
    __device__ __forceinline__ void init(const DevInstance &I, const OpT *route, int len, int n2) {
        rp = route; L = len; i = 0; two_n = n2; bad = false;
        lastp = len > 0 ? len - 1 : 0;
#pragma unroll
        for (int q = 0; q < OA; ++q) o[q] = (int)__ldg(at(q));
#pragma unroll
        for (int q = 0; q < LA; ++q) o[q] = checked(o[q], q);
#pragma unroll
        for (int q = 0; q < LA; ++q) {
            l[q] = o[q] < 0 ? 0 : __ldcg(I.d32 + gidx(I, q ? o[q - 1] : -1, o[q]));
            pp[q] = __ldg(I.p32 + op_customer(o[q] < 0 ? 0 : o[q]));
        }
    }
    __device__ __forceinline__ void advance_if(const DevInstance &I, bool go) {
        i += go ? 1 : 0;
#pragma unroll
        for (int q = 0; q + 1 < OA; ++q) o[q] = go ? o[q + 1] : o[q];
        o[OA - 1] = ldg_if(at(i + OA - 1), go, o[OA - 1]);
        const int h = checked(o[LA - 1], i + LA - 1);  // o[LA-1] was raw (one stage behind)
        o[LA - 1] = go ? h : o[LA - 1];
#pragma unroll
        for (int q = 0; q + 1 < LA; ++q) { l[q] = go ? l[q + 1] : l[q]; pp[q] = go ? pp[q + 1] : pp[q]; }
        const bool g2 = go && h >= 0;
        l[LA - 1] = ldcg_if(I.d32 + gidx(I, o[LA - 2], h), g2, go ? 0 : l[LA - 1]);
        pp[LA - 1] = ldg_if(I.p32 + op_customer(h < 0 ? 0 : h), g2, pp[LA - 1]);
    }
};

template <typename OpT, int M, int OA, int LA>
__global__ void __launch_bounds__(32)
serial_exact_kernel(DevInstance I, const OpT *__restrict__ ops, int64_t stride,
                    const int32_t *__restrict__ lens, int64_t N, double *__restrict__ z_out,
                    int32_t *__restrict__ status_out, double *__restrict__ returns_out,
                    int32_t *__restrict__ bottleneck_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    const int n = I.n, k = I.k, two_n = 2 * n;
    const int mwords = (n + 4) >> 2;  // slot ids of customers 0..n, 4 per word
    unsigned char *s_map = smem + lane * 4;  // customer c: byte (c & ~3) * 32 + (c & 3)
    uint32_t *s_mapw = reinterpret_cast<uint32_t *>(smem) + lane;
    // slot q: [q * 32]; slot SLOTS is a scratch target for the unconditional store
    uint32_t *s_val = reinterpret_cast<uint32_t *>(smem + (size_t)mwords * 128) + lane;

    for (int64_t base = (int64_t)blockIdx.x * 32; base < N; base += (int64_t)gridDim.x * 32) {
        const int64_t cand = base + lane;
        const bool live = cand < N;
        int L[M], off[M];
        int total = 0;
        bool mal = false;
#pragma unroll
        for (int v = 0; v < M; ++v) {
            const int x = live ? __ldg(lens + cand * M + v) : 0;
            mal |= x < 0;
            L[v] = x;
            off[v] = total;
            total += x;
        }
        mal |= total > two_n || total > stride;
        const bool run = live && !mal;
        const OpT *row = ops + (run ? cand : 0) * stride;
        SerialRoute<OpT, OA, LA> rs[M];
#pragma unroll
        for (int v = 0; v < M; ++v) rs[v].init(I, row + (run && L[v] > 0 ? off[v] : 0), run ? L[v] : 0, two_n);
        for (int w = 0; w < mwords; ++w) s_mapw[w * 32] = 0xFFFFFFFFu;

        uint32_t t[M];
        int lastc[M], sc[M], lo[M], hi[M];
#pragma unroll
        for (int v = 0; v < M; ++v) { t[v] = 0; lastc[v] = 0; sc[v] = 0; lo[v] = 0; hi[v] = k; }
        uint32_t freem = ~0u;
        bool dead = false, ovf = false;
        if (run) {
            for (;;) {
                bool moved = false, left = false;
#pragma unroll
                for (int v = 0; v < M; ++v) {
                    const bool act = rs[v].i < rs[v].L;
                    const int op = rs[v].o[0];  // -1 past the end: customer 0 (unused map entry)
                    const int c = op_customer(op);
                    const bool pick = op & 1;
                    unsigned char *mp = s_map + ((c & ~3) << 5) + (c & 3);
                    const int sid = *mp;
                    const uint32_t r = s_val[(sid & (SLOTS - 1)) * 32];
                    const uint32_t arr = t[v] + (uint32_t)rs[v].l[0];
                    const int slot = __ffs(freem) - 1;
                    const bool go = act && (!pick || sid < SLOTS);
                    const uint32_t rv = arr + (uint32_t)rs[v].pp[0];
                    ovf |= act && (arr < t[v] || (pick ? sid == 0xFE : (slot < 0 || rv < arr)));
                    const uint32_t tn = (pick && r > arr) ? r : arr;
                    const bool dgo = go && !pick;
                    s_val[((dgo && slot >= 0) ? slot : SLOTS) * 32] = rv;
                    *mp = (unsigned char)(go ? (pick ? 0xFE : slot) : sid);
                    freem = go ? (pick ? (freem | (1u << (sid & (SLOTS - 1)))) : (freem & (freem - 1))) : freem;
                    t[v] = go ? tn : t[v];
                    lastc[v] = go ? c : lastc[v];
                    const int room = k - 1 - sc[v], need = 1 - sc[v];
                    hi[v] = (go && pick && room < hi[v]) ? room : hi[v];
                    lo[v] = (dgo && need > lo[v]) ? need : lo[v];
                    sc[v] += go ? (pick ? 1 : -1) : 0;
                    rs[v].advance_if(I, go);
                    moved |= go;
                    left |= rs[v].i < rs[v].L;
                }
                if (!left || ovf) break;
                if (!moved) { dead = true; break; }
            }
        }
        bool bad = false, capfail = false;
#pragma unroll
        for (int v = 0; v < M; ++v) {
            if (dead)  // finish the capacity test past the stuck position
                for (int j = rs[v].i; j < rs[v].L; ++j)
                    cap_step(rs[v].checked((int)__ldg(rs[v].at(j)), j), k, sc[v], lo[v], hi[v]);
            bad |= rs[v].bad;
            capfail |= lo[v] > hi[v];
        }
        mal |= bad;
        const int st = mal ? ST_MAL : (ovf ? ST_RETRY : (capfail ? ST_CAP : (dead ? ST_DEAD : ST_OK)));
        double ret[M], z = 0.0;
#pragma unroll
        for (int v = 0; v < M; ++v) {
            ret[v] = 0.0;
            if (live && st == ST_OK && L[v] > 0)
                ret[v] = (double)((long long)t[v] + (long long)__ldg(I.d32 + (int64_t)lastc[v] * I.W));
            z = ret[v] > z ? ret[v] : z;
        }
        if (live) {
            int bn = 0;
#pragma unroll
            for (int v = M - 1; v >= 0; --v) bn = ret[v] == z ? v : bn;
            z_out[cand] = st == ST_OK ? z : 0.0;
            status_out[cand] = st;
            if (bottleneck_out) bottleneck_out[cand] = bn;
            if (returns_out)
#pragma unroll
                for (int v = 0; v < M; ++v) returns_out[cand * M + v] = ret[v];
        }
    }
}

#ifndef VRP_K1S_OA
#define VRP_K1S_OA 8
#endif
#ifndef VRP_K1S_LA
#define VRP_K1S_LA 4
#endif

struct SerialShape {
    int blocks;
    size_t smem;
};

template <typename OpT, int M>
int launch_serial(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens, int64_t N,
                  double *z, int32_t *status, double *returns, int32_t *bottleneck, cudaStream_t stream,
                  int sm_count) {
    auto kern = serial_exact_kernel<OpT, M, VRP_K1S_OA, VRP_K1S_LA>;
    static PlanCache<SerialShape> cache;
    SerialShape sh;
    const int rc = cache.get(I.n, sh, [&](SerialShape &out) {
        out.smem = (size_t)((I.n + 4) >> 2) * 128 + (size_t)(SLOTS + 1) * 128;
        if (out.smem > 227 * 1024) return -2;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out.smem) != cudaSuccess)
            return -1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out.blocks, kern, 32, out.smem) != cudaSuccess)
            return -1;
        return out.blocks > 0 ? 0 : -2;
    });
    if (rc) return rc;
    int64_t grid = (int64_t)sh.blocks * sm_count;
    const int64_t want = (N + 31) / 32;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32, sh.smem, stream>>>(I, static_cast<const OpT *>(ops), stride, lens, N, z, status,
                                                   returns, bottleneck);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

#endif  // VRP_K1_SERIAL

// (candidates per warp, warps per block) maximising resident candidates per SM
struct Shape {
    int G, wpb, blocks;
    size_t smem;
};

template <typename Kern>
int plan(Kern kern, int n, int m, int mode, int ready_bytes, bool compact, Shape &out) {
    const size_t per_cand = cand_layout(n, mode, ready_bytes, compact).total;
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
            // most resident candidates; among equals, fewer warps (fewer instructions)
            const long score = (long)blocks * w * G * 64 - (long)blocks * w;
            if (blocks > 0 && score > best) { best = score; out = {G, w, blocks, bytes}; }
        }
    }
    if (best < 0) return -2;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out.smem) == cudaSuccess ? 0 : -1;
}

template <typename OpT, bool INTD, int MODE, bool REC, bool NARROW, bool COMPACT = false, int MC = 0, int RA = 0>
int launch_t(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
             int64_t N, double *z, int32_t *status, double *returns, int32_t *bottleneck,
             double *arrival, double *timev, int32_t *q0, cudaStream_t stream, int sm_count,
             int fixup) {
    auto kern = makespan_kernel<OpT, INTD, MODE, REC, NARROW, COMPACT, MC, RA>;
    static PlanCache<Shape> cache;  // per instantiation, per device
    Shape sh;
    const int rc = cache.get(((int64_t)I.n << 8) | I.m, sh, [&](Shape &out) {
        using RT = typename std::conditional<NARROW, uint32_t, TimeT<INTD>>::type;
        return plan(kern, I.n, I.m, MODE, (int)sizeof(RT), COMPACT, out);
    });
    if (rc) return rc;
    const int64_t per_block = (int64_t)sh.wpb * sh.G;
    const int64_t want = (N + per_block - 1) / per_block;
    int64_t grid = (int64_t)sh.blocks * sm_count;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * sh.wpb, sh.smem, stream>>>(
        I, static_cast<const OpT *>(ops), stride, lens, N, sh.G, z, status, returns, bottleneck,
        arrival, timev, q0, fixup);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

// integral exact/evaluate: narrow pass, then the 64-bit kernel over the
// (normally zero) candidates whose ready times did not fit in 32 bits
template <typename OpT, int MODE>
int launch_narrow(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
                  int64_t N, double *z, int32_t *status, double *returns, int32_t *bottleneck,
                  cudaStream_t stream, int sm_count) {
    int rc = -1;
    bool done = false;
#if VRP_K1_SERIAL
    if (MODE == MODE_EXACT && I.m == 6 && I.k <= SLOTS / 6) {  // thread per candidate (A/B, compiled out)
        rc = launch_serial<OpT, 6>(I, ops, stride, lens, N, z, status, returns, bottleneck, stream, sm_count);
        done = true;
    }
#endif
    if (done) {
    } else if (MODE != MODE_TWO && I.m == 6 && I.k <= SLOTS / 6)  // slot table, m fixed at 6 (+ run-ahead: exact)
        rc = launch_t<OpT, true, MODE, false, true, true, 6, MODE == MODE_EXACT ? VRP_K1_RA : 0>(
            I, ops, stride, lens, N, z, status, returns, bottleneck, nullptr, nullptr, nullptr, stream, sm_count, 0);
    else if (MODE != MODE_TWO && I.m * I.k <= SLOTS)  // slot table (see makespan_kernel: COMPACT)
        rc = launch_t<OpT, true, MODE, false, true, true>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                                          nullptr, nullptr, nullptr, stream, sm_count, 0);
    else
        rc = launch_t<OpT, true, MODE, false, true>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                                    nullptr, nullptr, nullptr, stream, sm_count, 0);
    if (rc) return rc;
    return launch_t<OpT, true, MODE, false, false>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                                   nullptr, nullptr, nullptr, stream, sm_count, 1);
}

template <typename OpT, bool INTD>
int dispatch_mode(const DevInstance &I, const void *ops, int64_t stride, const int32_t *lens,
                  int64_t N, int mode, bool rec, double *z, int32_t *status, double *returns,
                  int32_t *bottleneck, double *arrival, double *timev, int32_t *q0,
                  cudaStream_t stream, int sm_count) {
    if (rec)
        return launch_t<OpT, INTD, MODE_EVAL, true, false>(I, ops, stride, lens, N, z, status, returns,
                                                           bottleneck, arrival, timev, q0, stream,
                                                           sm_count, 0);
    if (INTD && mode == MODE_EXACT)
        return launch_narrow<OpT, MODE_EXACT>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                              stream, sm_count);
    if (INTD && mode == MODE_EVAL)
        return launch_narrow<OpT, MODE_EVAL>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                             stream, sm_count);
    if (INTD && mode == MODE_TWO)  // the two-pass tables need every dropoff: narrow, not compact
        return launch_narrow<OpT, MODE_TWO>(I, ops, stride, lens, N, z, status, returns, bottleneck,
                                            stream, sm_count);
    switch (mode) {
        case MODE_EXACT:
            return launch_t<OpT, INTD, MODE_EXACT, false, false>(I, ops, stride, lens, N, z, status, returns,
                                                                 bottleneck, nullptr, nullptr, nullptr,
                                                                 stream, sm_count, 0);
        case MODE_EVAL:
            return launch_t<OpT, INTD, MODE_EVAL, false, false>(I, ops, stride, lens, N, z, status, returns,
                                                                bottleneck, nullptr, nullptr, nullptr,
                                                                stream, sm_count, 0);
        default:
            return launch_t<OpT, INTD, MODE_TWO, false, false>(I, ops, stride, lens, N, z, status, returns,
                                                               bottleneck, nullptr, nullptr, nullptr,
                                                               stream, sm_count, 0);
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
