// decode.cu -- K3: BRKGA multi-pass decoder (brkga.py:92-207) over a batch
// of chromosomes, one warp per chromosome.
//
//  sort    stable argsort of the 2n priority genes (brkga.py:116) on the
//          strict total order (order-preserving u64 key, index) -- equal to
//          numpy's stable sort (-0.0 canonicalised to +0.0, NaN last): a
//          bucketed counting sort with per-bucket insertion sorts, or, for a
//          chromosome whose priorities cluster, a bitonic network in shared
//          memory.
//  decode  lane v = vehicle v holds (t, loc, net, lo, hi) in registers.  The
//          pending list is scanned 32 ops at a time: a dropoff is deferred iff
//          no vehicle can take one (the capacity test does not depend on the
//          customer), a pickup iff its dropoff is unscheduled or no vehicle can
//          take it -- so every lane classifies its own op with one shared-
//          memory read, and the warp jumps straight to the first schedulable
//          op (ballot + ffs), writing the deferred ones back in visit order
//          (in place, stable).  The schedulable op is placed by the lanes in
//          parallel: feasibility, completion max(t + d, ready), hint-first
//          choice, else the lexicographic min of (completion, |v-hint|, v)
//          via a butterfly reduction (brkga.py:149-176).
//  emit    (op, vehicle) events are compacted vehicle-major with ballots.
#include <float.h>
#include <limits.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline int pow2_at_least(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Sort kernel smem per warp: P2 keys (u64) + P2 indices (u16).
__host__ __device__ inline size_t sort_bytes(int n) {
    const int P2 = pow2_at_least(2 * n);
    return align16(8 * (size_t)P2) + align16(2 * (size_t)P2);
}

// Decode kernel smem per warp: the pending list and the ready table only --
// the (op, vehicle) event log goes to a global scratch row, so residency is
// set by 2*(2n) + 8*(n+1) bytes (12 KB at n = 999).
struct DecodeLayout {
    size_t pend, ready, total;
};

// ready_bytes = 0: the compact slot table (a u8 slot id per customer + 32
// uint32 values, see decode_multi_kernel's CT)
__host__ __device__ inline DecodeLayout decode_layout(int n, int ready_bytes = 8) {
    DecodeLayout L;
    L.pend = 0;
    L.ready = align16(2 * (size_t)(2 * n));
    L.total = L.ready + (ready_bytes ? align16((size_t)ready_bytes * (size_t)(n + 1))
                                     : align16((size_t)(n + 1)) + 4 * 32);
    return L;
}

constexpr uint32_t NOT_DROPPED32 = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t order_key(double x) {
    if (x != x) return 0xFFFFFFFFFFFFFFFEull;  // NaN: after every number
    if (x == 0.0) x = 0.0;                    // -0.0 ties with +0.0
    uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// brkga.py:82-89 _hint_vehicle, with explicit round-to-nearest ops (no FMA)
__device__ __forceinline__ int hint_vehicle(int m, double g) {
    double x = __dmul_rn((double)m, g);
    long long h = (long long)x;
    if (__dsub_rn(x, (double)h) > 1.0 - 1e-9) h += 1;
    // any negative hint orders vehicles like -1 does (|v - h| = v - h) and is
    // never feasible, so it is clamped to -1 (keeps |v - h| < 64 for the keys)
    return h < 0 ? -1 : (int)(h < m ? h : m - 1);
}

__device__ __forceinline__ void bitonic_sort(uint64_t *key, uint16_t *idx, int P2, int lane) {
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < (P2 >> 1); i += 32) {
                int a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                int b = a + j;
                uint64_t ka = key[a], kb = key[b];
                uint16_t ia = idx[a], ib = idx[b];
                bool a_gt_b = ka > kb || (ka == kb && ia > ib);
                bool up = (a & k) == 0;
                if (a_gt_b == up) {
                    key[a] = kb; key[b] = ka;
                    idx[a] = ib; idx[b] = ia;
                }
            }
            __syncwarp();
        }
    }
}

// warp-uniform: can any vehicle take a dropoff / a pickup now, and (strict
// mode) the latest clock among vehicles that can take a pickup
// mhalf: the max runs over lanes [0, 2 mhalf) (which hold the m vehicles) and
// is broadcast from lane 0 -- 3 butterfly levels instead of 5 at m = 6
__device__ __forceinline__ void fleet_flags(bool vlane, double t, int net, int lo, int hi, int k,
                                            int relax, bool &any_drop, bool &any_pick,
                                            double &pick_maxT, int mhalf = 16) {
    int need = 1 - net, room = k - 1 - net;
    bool cd = vlane && ((need > lo ? need : lo) <= hi);
    bool cp = vlane && (lo <= (room < hi ? room : hi));
    any_drop = __any_sync(VRP_FULL_MASK, cd);
    any_pick = __any_sync(VRP_FULL_MASK, cp);
    if (relax) {
        pick_maxT = 0.0;
    } else if (mhalf >= 16) {
        pick_maxT = warp_max(cp ? t : -DBL_MAX);
    } else {
        double x = cp ? t : -DBL_MAX;
        for (int o = mhalf; o; o >>= 1) {
            const double y = __shfl_xor_sync(VRP_FULL_MASK, x, o);
            x = y > x ? y : x;
        }
        pick_maxT = __shfl_sync(VRP_FULL_MASK, x, 0);
    }
}

// Stable argsort of every chromosome's 2n priorities (brkga.py:116), one warp
// per chromosome; writes the order as u16 op indices to order_out[N][2n].
__global__ void __launch_bounds__(256)
sort_kernel(const double *__restrict__ genes, int64_t gstride, int64_t N, int two_n,
            uint16_t *__restrict__ order_out, const uint8_t *__restrict__ only) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int P2 = pow2_at_least(two_n);
    unsigned char *base = smem + (size_t)warp * (align16(8 * (size_t)P2) + align16(2 * (size_t)P2));
    uint64_t *s_key = reinterpret_cast<uint64_t *>(base);
    uint16_t *s_idx = reinterpret_cast<uint16_t *>(base + align16(8 * (size_t)P2));
    for (int64_t chrom = (int64_t)blockIdx.x * wpb + warp; chrom < N; chrom += (int64_t)gridDim.x * wpb) {
        if (only && !only[chrom]) continue;  // fallback pass of bucket_sort_kernel
        const double *g = genes + chrom * gstride;
        for (int i = lane; i < P2; i += 32) {
            s_key[i] = i < two_n ? order_key(__ldg(g + i)) : ~0ull;
            s_idx[i] = (uint16_t)i;
        }
        __syncwarp();
        bitonic_sort(s_key, s_idx, P2, lane);
        uint16_t *o = order_out + chrom * (int64_t)two_n;
        for (int i = lane; i < two_n; i += 32) o[i] = s_idx[i];
        __syncwarp();
    }
}

// NARROW (integral instances): the ready table holds uint32 (NOT_DROPPED32 =
// not dropped) -- 8 KB instead of 12 KB per warp at n = 999, so more warps
// per SM.  A ready time that does not fit sets retry[chrom]; the launcher's
// second (wide, `only = retry`) pass re-decodes exactly those chromosomes.
// Bucketed stable argsort (same order as sort_kernel): NB buckets monotone in
// the key (x < 0 | [0,1) in NB-2 equal slices | >= 1, inf, NaN), counted and
// scattered with shared atomics, then every bucket insertion-sorted by
// (order key, index) -- O(n) for BRKGA's [0, 1) genes instead of the bitonic
// network's O(n log^2 n).  A chromosome with a bucket of more than MAXB
// entries (many equal or clustered priorities) is flagged for sort_kernel.
constexpr int MAXB = 48;
constexpr int SU = 8;  // priorities loaded per lane per batch

// bucket count: a power of two near n (about two priorities per bucket), 64..1024
#ifndef VRP_BUCKET_PER
#define VRP_BUCKET_PER 2  // priorities per bucket (target)
#endif
#ifndef VRP_BUCKET_MAX
#define VRP_BUCKET_MAX 1024
#endif
__host__ __device__ inline int bucket_count(int two_n) {
    const int b = pow2_at_least(two_n / VRP_BUCKET_PER);
    return b < 64 ? 64 : (b > VRP_BUCKET_MAX ? VRP_BUCKET_MAX : b);
}

__device__ __forceinline__ int bucket_of(double x, int nb) {
    if (x < 0.0) return 0;
    if (!(x < 1.0)) return nb - 1;  // >= 1, +inf, NaN
    return 1 + (int)(x * (double)(nb - 2));
}

// per warp: bucket counters, the scattered indices and their keys' upper 32
// bits (the insertion sort compares those in shared memory and reads the full
// keys only on a tie of the upper halves)
__host__ __device__ inline size_t bucket_sort_bytes(int n) {
    return align16(4 * (size_t)bucket_count(2 * n)) + align16(2 * (size_t)(2 * n)) + align16(4 * (size_t)(2 * n));
}

__global__ void __launch_bounds__(256)
bucket_sort_kernel(const double *__restrict__ genes, int64_t gstride, int64_t N, int two_n,
                   uint16_t *__restrict__ order_out, uint8_t *__restrict__ fallback) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    unsigned char *base = smem + (size_t)warp * bucket_sort_bytes(two_n / 2);
    const int NB = bucket_count(two_n);
    int *cnt = reinterpret_cast<int *>(base);
    uint16_t *out = reinterpret_cast<uint16_t *>(base + align16(4 * (size_t)NB));
    uint32_t *khi = reinterpret_cast<uint32_t *>(base + align16(4 * (size_t)NB) + align16(2 * (size_t)two_n));
    for (int64_t chrom = (int64_t)blockIdx.x * wpb + warp; chrom < N; chrom += (int64_t)gridDim.x * wpb) {
        const double *g = genes + chrom * gstride;
        for (int b = lane; b < NB; b += 32) cnt[b] = 0;
        __syncwarp();
        // the priorities are read in batches of SU per lane, so SU loads are in
        // flight instead of one per shared-memory atomic
        for (int i0 = 0; i0 < two_n; i0 += 32 * SU) {
            double x[SU];
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int i = i0 + u * 32 + lane;
                x[u] = i < two_n ? __ldg(g + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SU; ++u)
                if (i0 + u * 32 + lane < two_n) atomicAdd(&cnt[bucket_of(x[u], NB)], 1);
        }
        __syncwarp();
        // exclusive prefix over the buckets, 32 consecutive buckets per step
        // (lane = bucket: conflict-free), and the largest bucket
        int carry = 0, big = 0;
        for (int j = 0; j < NB; j += 32) {
            const int c = cnt[j + lane];
            big = c > big ? c : big;
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(VRP_FULL_MASK, incl, o);
                if (lane >= o) incl += y;
            }
            cnt[j + lane] = carry + incl - c;  // bucket start, advanced by the scatter
            carry += __shfl_sync(VRP_FULL_MASK, incl, 31);
        }
        for (int o = 16; o; o >>= 1) {
            const int y = __shfl_xor_sync(VRP_FULL_MASK, big, o);
            big = y > big ? y : big;
        }
        if (big > MAXB) {  // clustered priorities: leave it to the bitonic pass
            if (lane == 0) fallback[chrom] = 1;
            __syncwarp();
            continue;
        }
        __syncwarp();
        for (int i0 = 0; i0 < two_n; i0 += 32 * SU) {
            double x[SU];
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int i = i0 + u * 32 + lane;
                x[u] = i < two_n ? __ldg(g + i) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int i = i0 + u * 32 + lane;
                if (i < two_n) {
                    const int pos = atomicAdd(&cnt[bucket_of(x[u], NB)], 1);
                    out[pos] = (uint16_t)i;
                    khi[pos] = (uint32_t)(order_key(x[u]) >> 32);
                }
            }
        }
        __syncwarp();
        // cnt[b] is now bucket b's end; sort each bucket by (key, index) --
        // upper key halves from shared memory, full keys only on a tie of those
        for (int b = lane; b < NB; b += 32) {
            const int e = cnt[b], s0 = b ? cnt[b - 1] : 0;
            for (int i = s0 + 1; i < e; ++i) {
                const uint16_t xi = out[i];
                const uint32_t hx = khi[i];
                int j = i - 1;
                while (j >= s0) {
                    const uint16_t yj = out[j];
                    const uint32_t hy = khi[j];
                    bool before = hy < hx;  // y sorts before x: stop
                    if (hy == hx) {
                        const uint64_t kx = order_key(__ldg(g + xi)), ky = order_key(__ldg(g + yj));
                        before = ky < kx || (ky == kx && yj < xi);
                    }
                    if (before) break;
                    out[j + 1] = yj;
                    khi[j + 1] = hy;
                    --j;
                }
                out[j + 1] = xi;
                khi[j + 1] = hx;
            }
        }
        __syncwarp();
        uint16_t *o = order_out + chrom * (int64_t)two_n;
        for (int i = lane; i < two_n; i += 32) o[i] = out[i];
        if (lane == 0) fallback[chrom] = 0;
        __syncwarp();
    }
}

#ifndef VRP_DECODE_WPF
#define VRP_DECODE_WPF 1  // next-window op + hint-gene prefetch (12.56 -> 11.89 ms per 24k decodes at n = 999, with MINB 4)
#endif
#ifndef VRP_DECODE_MINB
#define VRP_DECODE_MINB 4  // decode_kernel launch bounds (4: <= 64 registers; 5 (48) measured best without the window prefetch, which needs the registers)
#endif
// MC > 0 fixes the fleet size at compile time (MC == I.m): the argmin
// butterfly, the hint product and the vehicle-major emit loop are unrolled.
template <bool INTD, typename OutT, bool NARROW = false, int MC = 0, bool CT = false>
__global__ void __launch_bounds__(256, VRP_DECODE_MINB)
decode_kernel(DevInstance I, const double *__restrict__ genes, int64_t gstride, int64_t N,
              int relax, double penalty, double *__restrict__ fitness_out,
              double *__restrict__ makespan_out, int32_t *__restrict__ scheduled_out,
              int64_t *__restrict__ visits_out, OutT *__restrict__ ops_out, int64_t ostride,
              int32_t *__restrict__ lens_out, const uint16_t *__restrict__ order,
              uint32_t *__restrict__ seq_scratch, uint8_t *__restrict__ retry,
              const uint8_t *__restrict__ only) {
    using RT = typename std::conditional<NARROW, uint32_t, double>::type;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const int n = I.n, m = MC ? MC : I.m, k = I.k, two_n = 2 * n;
    const DecodeLayout Ly = decode_layout(n, CT ? 0 : (int)sizeof(RT));
    unsigned char *base = smem + (size_t)warp * Ly.total;
    volatile RT *s_ready = reinterpret_cast<volatile RT *>(base + Ly.ready);
    volatile uint8_t *s_sid = reinterpret_cast<volatile uint8_t *>(base + Ly.ready);
    volatile uint32_t *s_val = reinterpret_cast<volatile uint32_t *>(base + Ly.ready + align16((size_t)(n + 1)));
    uint16_t *s_pend = reinterpret_cast<uint16_t *>(base + Ly.pend);
    const bool vlane = lane < m;
    const unsigned lt = lanemask_lt();
    int mhalf = 1;  // argmin butterfly over lanes [0, 2*mhalf) ⊇ the m vehicle lanes
    while (2 * mhalf < m) mhalf <<= 1;
    if (m == 1) mhalf = 0;

    for (int64_t chrom = (int64_t)blockIdx.x * wpb + warp; chrom < N;
         chrom += (int64_t)gridDim.x * wpb) {
        if (only && !only[chrom]) continue;  // fix-up pass: just the flagged chromosomes
        const double *g = genes + chrom * gstride;
        uint32_t *seq = seq_scratch + chrom * (int64_t)two_n;  // (op | vehicle << 16) log
        bool ovf = false;
        // ---- pending list = the stable priority order (sort_kernel)
        const uint16_t *ord = order + chrom * (int64_t)two_n;
        for (int i = lane; i < two_n; i += 32) s_pend[i] = __ldg(ord + i);
        if (CT) {
            volatile uint32_t *w4 = reinterpret_cast<volatile uint32_t *>(s_sid);
            for (int c = lane; c < (n + 4) / 4; c += 32) w4[c] = 0xFFFFFFFFu;
        } else {
            for (int c = lane; c <= n; c += 32) s_ready[c] = NARROW ? (RT)NOT_DROPPED32 : (RT)-1.0;  // not dropped
        }
        __syncwarp();
        unsigned freem = 0xFFFFFFFFu;  // CT: free slots (warp-uniform)

        // ---- vehicle state (lane v = vehicle v)
        double t = 0.0;
        int loc = 0, net = 0, lo = 0, hi = k, cnt = 0;
        bool any_drop, any_pick;
        double pick_maxT;
        fleet_flags(vlane, t, net, lo, hi, k, relax, any_drop, any_pick, pick_maxT, mhalf);

        int npend = two_n, nseq = 0;
        int64_t visits = 0;
        for (int pass = 0; pass < two_n && npend; ++pass) {
            visits += npend;
            int nw = 0;
            bool progressed = false;
#if VRP_DECODE_WPF
            // the next window's ops and hint genes are loaded one window ahead
            // (deferrals only rewrite positions below the current window's end)
            int nxt_op = lane < npend ? s_pend[lane] : 0;
            double nxt_gene = lane < npend ? __ldg(g + two_n + nxt_op) : 0.0;
#endif
            for (int wbase = 0; wbase < npend; wbase += 32) {
                const int j = wbase + lane;
                const bool valid = j < npend;
#if VRP_DECODE_WPF
                const int op = valid ? nxt_op : 0;
                const double gene = nxt_gene;
                {
                    const int j2 = j + 32;
                    nxt_op = j2 < npend ? s_pend[j2] : 0;
                    nxt_gene = j2 < npend ? __ldg(g + two_n + nxt_op) : 0.0;
                }
#else
                const int op = valid ? s_pend[j] : 0;
                const double gene = valid ? __ldg(g + two_n + op) : 0.0;
#endif
                const int c = op_customer(op);
                const bool pk = op & 1;
                // the op's hint vehicle, computed with the window (off the placement chain)
                const int hj = valid ? hint_vehicle(m, gene) : 0;
                const double pj = valid && !pk ? __ldg(I.p + c) : 0.0;  // dropoff processing time
                // the pickup's ready time, read once per window; a dropoff placed
                // inside the window updates its pickup's copy in registers
                RT rr;
                if (CT) {
                    const int sd = pk ? (int)s_sid[c] : 0xFF;
                    rr = pk ? (sd == 0xFF ? (RT)NOT_DROPPED32 : (RT)s_val[sd & 31]) : (RT)0;
                } else {
                    rr = pk ? s_ready[c] : (RT)0;
                }
                unsigned todo = __ballot_sync(VRP_FULL_MASK, valid);
                __syncwarp();
                while (todo) {
                    const bool dropped = NARROW ? rr != (RT)NOT_DROPPED32 : (double)rr >= 0.0;
                    const double r = (double)rr;
                    const bool feas = pk ? (dropped && any_pick && (relax || pick_maxT >= r)) : any_drop;
                    const unsigned fm = __ballot_sync(VRP_FULL_MASK, feas) & todo;
                    const unsigned defm = fm ? (todo & ((1u << (__ffs(fm) - 1)) - 1u)) : todo;
                    if ((defm >> lane) & 1u) s_pend[nw + __popc(defm & lt)] = (uint16_t)op;
                    nw += __popc(defm);
                    if (!fm) break;
                    const int f = __ffs(fm) - 1;
                    todo &= ~((2u << f) - 1u);
                    // ---- place op f (brkga.py:148-193)
                    const int opf = __shfl_sync(VRP_FULL_MASK, op, f);
                    const double rf = __shfl_sync(VRP_FULL_MASK, r, f);
                    const int cf = op_customer(opf);
                    const bool pickf = opf & 1;
                    const double pf = __shfl_sync(VRP_FULL_MASK, pj, f);
                    double comp = 0.0;
                    bool fv = false;
                    if (vlane) {
                        const double leg = dist<INTD>(I, loc, cf);
                        const double arr = t + leg;
                        if (pickf) {
                            int room = k - 1 - net;
                            bool cp = lo <= (room < hi ? room : hi);
                            fv = cp && (relax || t >= rf);
                            comp = relax ? (arr >= rf ? arr : rf) : arr;
                        } else {
                            int need = 1 - net;
                            fv = (need > lo ? need : lo) <= hi;
                            comp = arr;
                        }
                    }
                    const int hint = __shfl_sync(VRP_FULL_MASK, hj, f);
                    const unsigned fmask = __ballot_sync(VRP_FULL_MASK, fv);
                    int vstar;
                    if (hint >= 0 && hint < 32 && ((fmask >> hint) & 1u)) {
                        vstar = hint;
                    } else if (INTD) {
                        // integral completions (< 2^53, exact): one u64 key
                        // (comp, |v - hint|, v), min over the m vehicle lanes
                        const int dh = lane > hint ? lane - hint : hint - lane;
                        uint64_t key = fv ? ((uint64_t)comp << 11) | ((uint64_t)dh << 5) | (uint64_t)lane : ~0ull;
                        for (int o = mhalf; o; o >>= 1) {
                            const uint64_t ok = __shfl_xor_sync(VRP_FULL_MASK, key, o);
                            key = ok < key ? ok : key;
                        }
                        vstar = __shfl_sync(VRP_FULL_MASK, (int)(key & 31u), 0);
                    } else {
                        double kc = fv ? comp : DBL_MAX;
                        int kd = fv ? (lane > hint ? lane - hint : hint - lane) : INT_MAX;
                        int kv = fv ? lane : INT_MAX;
                        for (int o = mhalf; o; o >>= 1) {
                            double oc = __shfl_xor_sync(VRP_FULL_MASK, kc, o);
                            int od = __shfl_xor_sync(VRP_FULL_MASK, kd, o);
                            int ov = __shfl_xor_sync(VRP_FULL_MASK, kv, o);
                            bool better = oc < kc || (oc == kc && (od < kd || (od == kd && ov < kv)));
                            if (better) { kc = oc; kd = od; kv = ov; }
                        }
                        vstar = __shfl_sync(VRP_FULL_MASK, kv, 0);
                    }
                    const double cstar = __shfl_sync(VRP_FULL_MASK, comp, vstar);
                    if (lane == vstar) {
                        t = cstar;
                        loc = cf;
                        if (pickf) { int room = k - 1 - net; hi = room < hi ? room : hi; ++net; }
                        else { int need = 1 - net; lo = need > lo ? need : lo; --net; }
                        ++cnt;
                    }
                    if (!pickf) {
                        const double rv = cstar + pf;
                        RT rs;
                        if (NARROW) {
                            ovf |= !(rv < 4294967295.0);  // warp-uniform
                            rs = (RT)(ovf ? 0.0 : rv);
                        } else {
                            rs = (RT)rv;
                        }
                        if (CT) {
                            ovf |= freem == 0u;  // no free slot: the wide fix-up pass decodes it
                            const int slot = freem ? __ffs(freem) - 1 : 0;
                            freem &= ~(1u << slot);
                            if (lane == 0) { s_val[slot] = (uint32_t)rs; s_sid[cf] = (uint8_t)slot; }
                        } else {
                            if (lane == 0) s_ready[cf] = rs;
                        }
                        if (op == opf + 1) rr = rs;  // this window holds the pickup
                    } else if (CT) {
                        const int sd = (int)s_sid[cf];  // its dropoff's slot is free again
                        freem |= 1u << (sd & 31);
                    }
                    if (lane == 0 && seq_scratch) seq[nseq] = (uint32_t)opf | ((uint32_t)vstar << 16);
                    ++nseq;
                    progressed = true;
                    fleet_flags(vlane, t, net, lo, hi, k, relax, any_drop, any_pick, pick_maxT, mhalf);
                    __syncwarp();
                }
                __syncwarp();
            }
            npend = nw;
            if (!progressed) break;
        }

        // ---- fitness (brkga.py:198-200): unused vehicles return at 0 + d[0][0]
        double ret = vlane ? t + dist<INTD>(I, loc, 0) : -DBL_MAX;
        const double z = warp_max(ret);
        if (NARROW && lane == 0) retry[chrom] = ovf ? 1 : 0;
        if (lane == 0) {
            fitness_out[chrom] = z + penalty * (double)npend;
            if (makespan_out) makespan_out[chrom] = z;
            if (scheduled_out) scheduled_out[chrom] = two_n - npend;
            if (visits_out) visits_out[chrom] = visits;
        }
        // ---- emit the solution vehicle-major
        if (ops_out) {
            int off = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(VRP_FULL_MASK, off, o);
                if (lane >= o) off += y;
            }
            off -= cnt;  // exclusive start of route `lane`
            OutT *row = ops_out + chrom * ostride;
            for (int sb = 0; sb < nseq; sb += 32) {
                const int j = sb + lane;
                const bool valid = j < nseq;
                const uint32_t e = valid ? seq[j] : 0u;
                const int op = (int)(e & 0xffffu);
                const int v = valid ? (int)(e >> 16) : -1;
                for (int u = 0; u < m; ++u) {
                    const unsigned mk = __ballot_sync(VRP_FULL_MASK, v == u);
                    const int ou = __shfl_sync(VRP_FULL_MASK, off, u);
                    if (v == u) row[ou + __popc(mk & lt)] = (OutT)op;
                    if (lane == u) off += __popc(mk);
                }
            }
            for (int j = nseq + lane; j < two_n; j += 32) row[j] = (OutT)-1;
            if (lens_out && vlane) lens_out[chrom * m + lane] = cnt;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Segmented decode: G = 32 / P chromosomes per warp, P = pow2 >= m lanes each
// (lane sl < m of a segment = vehicle sl).  Every segment runs the same
// algorithm as decode_kernel on its own P-op window, in lockstep: one step =
// classify the window, defer the unschedulable prefix, place the first
// schedulable op.  The per-step ballots, shuffles and the argmin butterfly
// (log2 P levels) serve G chromosomes at once.  Hint vehicles are staged in
// shared memory (u8 per gene) with the pending list and the ready table, so a
// window refill reads shared memory only.
struct MultiLayout {
    size_t pend, ready, hint, total;
};

// ready_bytes = 0: the compact slot table (CT) -- a u8 slot id per customer
// plus MULTI_SLOTS uint32 ready values (see decode_multi_kernel)
constexpr int MULTI_SLOTS = 32;

__host__ __device__ inline MultiLayout multi_layout(int n, int ready_bytes) {
    MultiLayout L;
    L.pend = 0;
    L.ready = align16(2 * (size_t)(2 * n));
    const size_t rb = ready_bytes ? align16((size_t)ready_bytes * (size_t)(n + 1))
                                  : align16((size_t)(n + 1)) + 4 * MULTI_SLOTS;
    L.hint = L.ready + rb;
    L.total = L.hint + align16((size_t)(2 * n));
    return L;
}

template <int P>
__device__ __forceinline__ double seg_max(double x) {
#pragma unroll
    for (int o = P / 2; o; o >>= 1) {
        double y = __shfl_xor_sync(VRP_FULL_MASK, x, o);
        x = y > x ? y : x;
    }
    return x;
}

template <int P>
__device__ __forceinline__ void seg_flags(bool vlane, double t, int net, int lo, int hi, int k, int relax,
                                          unsigned smask, bool &any_drop, bool &any_pick, double &pick_maxT) {
    int need = 1 - net, room = k - 1 - net;
    bool cd = vlane && ((need > lo ? need : lo) <= hi);
    bool cp = vlane && (lo <= (room < hi ? room : hi));
    any_drop = (__ballot_sync(VRP_FULL_MASK, cd) & smask) != 0u;
    any_pick = (__ballot_sync(VRP_FULL_MASK, cp) & smask) != 0u;
    pick_maxT = relax ? 0.0 : seg_max<P>(cp ? t : -DBL_MAX);
}

// CT (with NARROW): the ready table is a slot table, as in K1 -- customers
// dropped but not yet picked up number at most sum_v q0_v <= m k (the decoder
// keeps every vehicle's load interval feasible), so m k <= 32 slots of uint32
// values and a u8 slot id per customer replace the (n+1)-entry table: 5 KB
// less shared memory per chromosome at n = 999, twice the resident
// chromosomes.  A chromosome that finds no free slot goes to the wide fix-up
// pass like a 32-bit overflow.
template <bool INTD, typename OutT, bool NARROW, int P, int MC = 0, bool CT = false>  // MC: as decode_kernel
__global__ void __launch_bounds__(256, 4)
decode_multi_kernel(DevInstance I, const double *__restrict__ genes, int64_t gstride, int64_t N,
                    int relax, double penalty, double *__restrict__ fitness_out,
                    double *__restrict__ makespan_out, int32_t *__restrict__ scheduled_out,
                    int64_t *__restrict__ visits_out, OutT *__restrict__ ops_out, int64_t ostride,
                    int32_t *__restrict__ lens_out, const uint16_t *__restrict__ order,
                    uint32_t *__restrict__ seq_scratch, uint8_t *__restrict__ retry,
                    const uint8_t *__restrict__ only) {
    using RT = typename std::conditional<NARROW, uint32_t, double>::type;
    constexpr int G = 32 / P;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const int seg = lane / P, sl = lane % P, sbase = seg * P;
    const unsigned smask = (P == 32) ? 0xffffffffu : (((1u << P) - 1u) << sbase);
    const int n = I.n, m = MC ? MC : I.m, k = I.k, two_n = 2 * n;
    const MultiLayout Ly = multi_layout(n, CT ? 0 : (int)sizeof(RT));
    unsigned char *base = smem + ((size_t)warp * G + seg) * Ly.total;
    volatile RT *s_ready = reinterpret_cast<volatile RT *>(base + Ly.ready);
    volatile uint8_t *s_sid = reinterpret_cast<volatile uint8_t *>(base + Ly.ready);
    volatile uint32_t *s_val = reinterpret_cast<volatile uint32_t *>(base + Ly.ready + align16((size_t)(n + 1)));
    uint16_t *s_pend = reinterpret_cast<uint16_t *>(base + Ly.pend);
    int8_t *s_hint = reinterpret_cast<int8_t *>(base + Ly.hint);
    const bool vlane = sl < m;
    const unsigned lt = lanemask_lt();
    int mhalf = 1;  // argmin butterfly over segment lanes [0, 2*mhalf) ⊇ the m vehicles
    while (2 * mhalf < m) mhalf <<= 1;
    if (m == 1) mhalf = 0;

    for (int64_t c0 = ((int64_t)blockIdx.x * wpb + warp) * G; c0 < N; c0 += (int64_t)gridDim.x * wpb * G) {
        const int64_t chrom = c0 + seg;
        const bool real = chrom < N && !(only && !only[chrom]);
        const int64_t cx = real ? chrom : c0;
        const double *g = genes + cx * gstride;
        uint32_t *seq = seq_scratch ? seq_scratch + cx * (int64_t)two_n : nullptr;
        if (real) {
            const uint16_t *ord = order + cx * (int64_t)two_n;
            for (int i = sl; i < two_n; i += P) {
                s_pend[i] = __ldg(ord + i);
                s_hint[i] = (int8_t)hint_vehicle(m, __ldg(g + two_n + i));
            }
            if (CT) {
                volatile uint32_t *w4 = reinterpret_cast<volatile uint32_t *>(s_sid);
                for (int c = sl; c < (n + 4) / 4; c += P) w4[c] = 0xFFFFFFFFu;
            } else {
                for (int c = sl; c <= n; c += P) s_ready[c] = NARROW ? (RT)NOT_DROPPED32 : (RT)-1.0;
            }
        }
        __syncwarp();
        unsigned freem = 0xFFFFFFFFu;  // CT: free slots (segment-uniform)

        double t = 0.0;
        int loc = 0, net = 0, lo = 0, hi = k, cnt = 0;
        bool any_drop, any_pick;
        double pick_maxT;
        seg_flags<P>(vlane, t, net, lo, hi, k, relax, smask, any_drop, any_pick, pick_maxT);

        // segment-uniform progress state
        int npend = two_n, nw = 0, wbase = -P, pass = 0, nseq = 0;
        int64_t visits = two_n;
        bool progressed = false, ovf = false, done = !real || two_n == 0;
        unsigned todo = 0u;
        // this lane's op of its segment's window
        int op = 0, c = 0, hj = 0;
        bool pk = false;
        double pj = 0.0;
        RT rr = (RT)0;
        while (!__all_sync(VRP_FULL_MASK, done)) {
            __syncwarp();
            // ---- refill exhausted windows (a pass ends when its list is exhausted)
            bool refill = !done && todo == 0u;
            if (__any_sync(VRP_FULL_MASK, refill)) {
                if (refill) {
                    wbase += P;
                    if (wbase >= npend) {
                        npend = nw;
                        ++pass;
                        if (!progressed || npend == 0 || pass >= two_n) {
                            done = true;
                        } else {
                            visits += npend;
                            nw = 0;
                            wbase = 0;
                            progressed = false;
                        }
                    }
                }
                refill = refill && !done;
                const int j = wbase + sl;
                const bool valid = refill && j < npend;
                if (refill) {
                    op = valid ? s_pend[j] : 0;
                    c = op_customer(op);
                    pk = op & 1;
                    hj = valid ? s_hint[op] : 0;
                    pj = valid && !pk ? __ldg(I.p + c) : 0.0;
                    if (CT) {
                        const int sd = pk ? (int)s_sid[c] : 0xFF;
                        rr = pk ? (sd == 0xFF ? (RT)NOT_DROPPED32 : (RT)s_val[sd & (MULTI_SLOTS - 1)]) : (RT)0;
                    } else {
                        rr = pk ? s_ready[c] : (RT)0;
                    }
                }
                const unsigned vb = __ballot_sync(VRP_FULL_MASK, valid);
                if (refill) todo = vb & smask;
            }
            // ---- classify, defer the unschedulable prefix (in visit order)
            const bool dropped = NARROW ? rr != (RT)NOT_DROPPED32 : (double)rr >= 0.0;
            const double r = (double)rr;
            const bool feas = pk ? (dropped && any_pick && (relax || pick_maxT >= r)) : any_drop;
            const unsigned fm = __ballot_sync(VRP_FULL_MASK, feas) & todo;
            const unsigned defm = fm ? (todo & ((1u << (__ffs(fm) - 1)) - 1u)) : todo;
            if ((defm >> lane) & 1u) s_pend[nw + __popc(defm & lt)] = (uint16_t)op;
            nw += __popc(defm);
            const bool place = fm != 0u;
            const int f = place ? __ffs(fm) - 1 : sbase;
            todo = place ? (todo & ~((2u << f) - 1u)) : 0u;
            // ---- place op f (brkga.py:148-193) in every segment that has one
            const int opf = __shfl_sync(VRP_FULL_MASK, op, f);
            const double rf = __shfl_sync(VRP_FULL_MASK, r, f);
            const double pf = __shfl_sync(VRP_FULL_MASK, pj, f);
            const int hint = __shfl_sync(VRP_FULL_MASK, hj, f);
            const int cf = op_customer(opf);
            const bool pickf = opf & 1;
            double comp = 0.0;
            bool fv = false;
            if (vlane && place) {
                const double leg = dist<INTD>(I, loc, cf);
                const double arr = t + leg;
                if (pickf) {
                    int room = k - 1 - net;
                    bool cp = lo <= (room < hi ? room : hi);
                    fv = cp && (relax || t >= rf);
                    comp = relax ? (arr >= rf ? arr : rf) : arr;
                } else {
                    int need = 1 - net;
                    fv = (need > lo ? need : lo) <= hi;
                    comp = arr;
                }
            }
            const unsigned fmask = (__ballot_sync(VRP_FULL_MASK, fv) & smask) >> sbase;
            const bool hintok = hint >= 0 && ((fmask >> hint) & 1u);
            int vstar = hint;
            if (__any_sync(VRP_FULL_MASK, place && !hintok)) {
                int am;
                if (INTD) {
                    // integral completions (< 2^53, exact): one u64 key (comp, |v - hint|, v)
                    const int dh = sl > hint ? sl - hint : hint - sl;
                    uint64_t key = fv ? ((uint64_t)comp << 11) | ((uint64_t)dh << 5) | (uint64_t)sl : ~0ull;
                    for (int o = mhalf; o; o >>= 1) {
                        const uint64_t ok = __shfl_xor_sync(VRP_FULL_MASK, key, o);
                        key = ok < key ? ok : key;
                    }
                    am = (int)(key & 31u);
                } else {
                    double kc = fv ? comp : DBL_MAX;
                    int kd = fv ? (sl > hint ? sl - hint : hint - sl) : INT_MAX;
                    int kv = fv ? sl : INT_MAX;
                    for (int o = mhalf; o; o >>= 1) {
                        double oc = __shfl_xor_sync(VRP_FULL_MASK, kc, o);
                        int od = __shfl_xor_sync(VRP_FULL_MASK, kd, o);
                        int ov = __shfl_xor_sync(VRP_FULL_MASK, kv, o);
                        bool better = oc < kc || (oc == kc && (od < kd || (od == kd && ov < kv)));
                        if (better) { kc = oc; kd = od; kv = ov; }
                    }
                    am = kv;
                }
                am = __shfl_sync(VRP_FULL_MASK, am, sbase);
                if (!hintok) vstar = am;
            }
            const double cstar = __shfl_sync(VRP_FULL_MASK, comp, sbase + (vstar & (P - 1)));
            if (place) {
                if (sl == vstar) {
                    t = cstar;
                    loc = cf;
                    if (pickf) { int room = k - 1 - net; hi = room < hi ? room : hi; ++net; }
                    else { int need = 1 - net; lo = need > lo ? need : lo; --net; }
                    ++cnt;
                }
                if (!pickf) {
                    const double rv = cstar + pf;
                    RT rs;
                    if (NARROW) {
                        ovf |= !(rv < 4294967295.0);  // segment-uniform
                        rs = (RT)(ovf ? 0.0 : rv);
                    } else {
                        rs = (RT)rv;
                    }
                    if (CT) {
                        ovf |= freem == 0u;  // no free slot: the wide fix-up pass decodes it
                        const int slot = freem ? __ffs(freem) - 1 : 0;
                        freem &= ~(1u << slot);
                        if (sl == 0) { s_val[slot] = (uint32_t)rs; s_sid[cf] = (uint8_t)slot; }
                    } else {
                        if (sl == 0) s_ready[cf] = rs;
                    }
                    if (op == opf + 1) rr = rs;  // the window holds the pickup
                } else if (CT) {
                    const int sd = (int)s_sid[cf];  // its dropoff's slot is free again
                    freem |= 1u << (sd & (MULTI_SLOTS - 1));
                }
                if (sl == 0 && seq) seq[nseq] = (uint32_t)opf | ((uint32_t)vstar << 16);
                ++nseq;
                progressed = true;
            }
            seg_flags<P>(vlane, t, net, lo, hi, k, relax, smask, any_drop, any_pick, pick_maxT);
        }

        // ---- fitness (brkga.py:198-200): unused vehicles return at 0 + d[0][0]
        double ret = vlane ? t + dist<INTD>(I, loc, 0) : -DBL_MAX;
        const double z = seg_max<P>(ret);
        if (real && sl == 0) {
            if (NARROW) retry[chrom] = ovf ? 1 : 0;
            fitness_out[chrom] = z + penalty * (double)npend;
            if (makespan_out) makespan_out[chrom] = z;
            if (scheduled_out) scheduled_out[chrom] = two_n - npend;
            if (visits_out) visits_out[chrom] = visits;
        }
        // ---- emit every chromosome's solution vehicle-major, one at a time
        if (ops_out) {
            int off = cnt;
#pragma unroll
            for (int o = 1; o < P; o <<= 1) {
                int y = __shfl_up_sync(VRP_FULL_MASK, off, o, P);
                if (sl >= o) off += y;
            }
            off -= cnt;  // exclusive start of route sl of this segment's chromosome
            __syncwarp();
            for (int gi = 0; gi < G; ++gi) {
                const int64_t ch = c0 + gi;
                if (ch >= N || (only && !only[ch])) continue;  // warp-uniform
                const int ns = __shfl_sync(VRP_FULL_MASK, nseq, gi * P);
                const uint32_t *sq = seq_scratch + ch * (int64_t)two_n;
                OutT *row = ops_out + ch * ostride;
                for (int sb = 0; sb < ns; sb += 32) {
                    const int j = sb + lane;
                    const bool valid = j < ns;
                    const uint32_t e = valid ? sq[j] : 0u;
                    const int o2 = (int)(e & 0xffffu);
                    const int v = valid ? (int)(e >> 16) : -1;
                    for (int u = 0; u < m; ++u) {
                        const unsigned mk = __ballot_sync(VRP_FULL_MASK, v == u);
                        const int ou = __shfl_sync(VRP_FULL_MASK, off, gi * P + u);
                        if (v == u) row[ou + __popc(mk & lt)] = (OutT)o2;
                        if (lane == gi * P + u) off += __popc(mk);
                    }
                }
                for (int j = ns + lane; j < two_n; j += 32) row[j] = (OutT)-1;
            }
            if (real && lens_out && vlane) lens_out[chrom * m + sl] = cnt;
        }
        __syncwarp();
    }
}

// (warps per block, resident blocks) maximising resident warps per SM for a
// dynamic shared-memory footprint of per_warp bytes per warp
struct DecodePlan {
    int w, blocks;
};

template <typename Kern>
int plan_decode(Kern kern, size_t per_warp, DecodePlan &out) {
    int best_w = 0, best_res = 0, best_blocks = 0;
    for (int w = 8; w >= 1; --w) {
        const size_t bytes = per_warp * (size_t)w;
        if (bytes > 227 * 1024) continue;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
            return -1;
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * w, bytes) != cudaSuccess) return -1;
        if (blocks * w > best_res) { best_res = blocks * w; best_w = w; best_blocks = blocks; }
    }
    if (!best_res) return -2;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per_warp * best_w)) != cudaSuccess)
        return -1;
    out = DecodePlan{best_w, best_blocks};
    return 0;
}

template <bool INTD, typename OutT, bool NARROW, int P, int MC = 0, bool CT = false>
int launch_m(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
             double penalty, double *fitness, double *makespan, int32_t *scheduled, int64_t *visits,
             void *ops_out, int64_t ostride, int32_t *lens_out, const uint16_t *order, uint32_t *seq,
             uint8_t *retry, const uint8_t *only, cudaStream_t stream, int sm_count) {
    constexpr int G = 32 / P;
    auto kern = decode_multi_kernel<INTD, OutT, NARROW, P, MC, CT>;
    const size_t per_warp = multi_layout(I.n, CT ? 0 : (NARROW ? 4 : 8)).total * G;
    static PlanCache<DecodePlan> cache;
    DecodePlan pl;
    const int rc = cache.get((int64_t)per_warp, pl, [&](DecodePlan &out) { return plan_decode(kern, per_warp, out); });
    if (rc) return rc;
    const int cached_w = pl.w, cached_blocks = pl.blocks;
    const size_t bytes = per_warp * (size_t)cached_w;
    const int64_t nwarps = (N + G - 1) / G;
    int64_t want = (nwarps + cached_w - 1) / cached_w;
    int64_t grid = (int64_t)cached_blocks * sm_count;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * cached_w, bytes, stream>>>(I, genes, gstride, N, relax, penalty, fitness,
                                                         makespan, scheduled, visits,
                                                         static_cast<OutT *>(ops_out), ostride, lens_out,
                                                         order, seq, retry, only);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

// one decode_kernel launch, occupancy planned once per (instantiation, n)
template <bool INTD, typename OutT, bool NARROW, int MC = 0, bool CT = false>
int launch_k(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
             double penalty, double *fitness, double *makespan, int32_t *scheduled, int64_t *visits,
             void *ops_out, int64_t ostride, int32_t *lens_out, const uint16_t *order, uint32_t *seq,
             uint8_t *retry, const uint8_t *only, cudaStream_t stream, int sm_count) {
    auto kern = decode_kernel<INTD, OutT, NARROW, MC, CT>;
    const size_t per_warp = decode_layout(I.n, CT ? 0 : (NARROW ? 4 : 8)).total;
    static PlanCache<DecodePlan> cache;
    DecodePlan pl;
    const int rc = cache.get((int64_t)per_warp, pl, [&](DecodePlan &out) { return plan_decode(kern, per_warp, out); });
    if (rc) return rc;
    const int cached_w = pl.w, cached_blocks = pl.blocks;
    const size_t bytes = per_warp * (size_t)cached_w;
    int64_t want = (N + cached_w - 1) / cached_w;
    int64_t grid = (int64_t)cached_blocks * sm_count;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 32 * cached_w, bytes, stream>>>(I, genes, gstride, N, relax, penalty, fitness,
                                                         makespan, scheduled, visits,
                                                         static_cast<OutT *>(ops_out), ostride, lens_out,
                                                         order, seq, retry, only);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

// segmented kernel for m <= 16 (G = 32 / P chromosomes per warp), the
// warp-per-chromosome kernel above that, or when VRP_DECODE_SINGLE is set
template <bool INTD, typename OutT, bool NARROW>
int launch_any(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
               double penalty, double *fitness, double *makespan, int32_t *scheduled, int64_t *visits,
               void *ops_out, int64_t ostride, int32_t *lens_out, const uint16_t *order, uint32_t *seq,
               uint8_t *retry, const uint8_t *only, cudaStream_t stream, int sm_count) {
    const char *single = getenv("VRP_DECODE_SINGLE");
    const char *noct = getenv("VRP_DECODE_NO_CT");  // (ablation knob)
    const char *wnoct = getenv("VRP_DECODE_WARP_NO_CT");  // (ablation knob: warp kernel only)
    // the compact slot table (narrow pass, m k <= 32 slots, m = 6): 5 KB of
    // shared memory per chromosome at n = 999 instead of 10 KB
    const bool ct = NARROW && I.m == 6 && I.m * I.k <= MULTI_SLOTS && !(noct && noct[0] && noct[0] != '0');
    // below n = 500 (a280: 2.8 KB of shared memory per chromosome; the slot
    // table measured +15 % generations/s there).  At n = 999 the warp-per-
    // chromosome kernel wins: 2.8x with the full table, and still 2x with the
    // slot table (random chromosomes defer ~11 ops per placement there, and
    // its 32-op pending window scans 4x faster than a segment's 8-op window)
    const bool seg = !(single && single[0] && single[0] != '0') && I.n < 500;
    if (seg && ct)
        return launch_m<INTD, OutT, NARROW, 8, 6, true>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                                        scheduled, visits, ops_out, ostride, lens_out, order, seq,
                                                        retry, only, stream, sm_count);
    if (seg && I.m == 6)  // the fleet of every benchmark config beyond gr17
        return launch_m<INTD, OutT, NARROW, 8, 6>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                                  scheduled, visits, ops_out, ostride, lens_out, order, seq, retry,
                                                  only, stream, sm_count);
    if (seg && I.m <= 4)
        return launch_m<INTD, OutT, NARROW, 4>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                               visits, ops_out, ostride, lens_out, order, seq, retry, only,
                                               stream, sm_count);
    if (seg && I.m <= 8)
        return launch_m<INTD, OutT, NARROW, 8>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                               visits, ops_out, ostride, lens_out, order, seq, retry, only,
                                               stream, sm_count);
    if (seg && I.m <= 16)
        return launch_m<INTD, OutT, NARROW, 16>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                                scheduled, visits, ops_out, ostride, lens_out, order, seq, retry,
                                                only, stream, sm_count);
    if (ct && !(wnoct && wnoct[0] && wnoct[0] != '0'))  // the slot table in the warp kernel too
        return launch_k<INTD, OutT, NARROW, 6, true>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                                     scheduled, visits, ops_out, ostride, lens_out, order, seq,
                                                     retry, only, stream, sm_count);
    if (I.m == 6)  // the fleet of every benchmark config beyond gr17
        return launch_k<INTD, OutT, NARROW, 6>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                               visits, ops_out, ostride, lens_out, order, seq, retry, only, stream,
                                               sm_count);
    return launch_k<INTD, OutT, NARROW>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                        visits, ops_out, ostride, lens_out, order, seq, retry, only, stream,
                                        sm_count);
}

template <bool INTD, typename OutT>
int launch_t(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
             double penalty, double *fitness, double *makespan, int32_t *scheduled, int64_t *visits,
             void *ops_out, int64_t ostride, int32_t *lens_out, cudaStream_t stream, int sm_count) {
    // scratch: priority order (u16), the (op | vehicle << 16) event log when the
    // solution is wanted, and (integral instances) the narrow pass's retry flags
    const int two_n = 2 * I.n;
    uint16_t *order = nullptr;
    uint32_t *seq = nullptr;
    uint8_t *retry = nullptr, *fb = nullptr;
    auto release = [&]() {  // every exit path frees the scratch
        if (order) cudaFreeAsync(order, stream);
        if (fb) cudaFreeAsync(fb, stream);
        if (seq) cudaFreeAsync(seq, stream);
        if (retry) cudaFreeAsync(retry, stream);
    };
    // the sort kernels' shared memory per warp; as many warps per block as fit
    const size_t bper = bucket_sort_bytes(I.n), sper = sort_bytes(I.n);
    if (bper > 227 * 1024 || sper > 227 * 1024) return -2;  // n beyond the sort's shared-memory footprint
    // narrow tables where shared memory limits residency (measured: a280
    // +25 % with the segmented kernel; below n ~ 200 registers bound it)
    const char *nm = getenv("VRP_DECODE_NARROW_MIN");  // (ablation knob)
    const bool narrow = INTD && I.n >= (nm ? atoi(nm) : 200);
    if (cudaMallocAsync(&order, sizeof(uint16_t) * (size_t)N * two_n, stream) != cudaSuccess ||
        (ops_out && cudaMallocAsync(&seq, sizeof(uint32_t) * (size_t)N * two_n, stream) != cudaSuccess) ||
        (narrow && cudaMallocAsync(&retry, (size_t)N, stream) != cudaSuccess) ||
        cudaMallocAsync(&fb, (size_t)N, stream) != cudaSuccess) {
        release();
        return -1;
    }
    {
        auto fit = [](size_t per) { int w = 4; while (w > 1 && per * w > 227 * 1024) --w; return w; };
        const int bw = fit(bper), sw = fit(sper);
        const size_t bbytes = bper * bw, sbytes = sper * sw;
        struct SortPlan { int bblocks, sblocks; };
        static PlanCache<SortPlan> cache;
        SortPlan sp;
        const int rc0 = cache.get(I.n, sp, [&](SortPlan &out) {
            if (cudaFuncSetAttribute(bucket_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bbytes) != cudaSuccess ||
                cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes) != cudaSuccess)
                return -1;
            out.bblocks = out.sblocks = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out.bblocks, bucket_sort_kernel, 32 * bw, bbytes);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&out.sblocks, sort_kernel, 32 * sw, sbytes);
            return 0;
        });
        if (rc0) { release(); return rc0; }
        int64_t bgrid = (int64_t)(sp.bblocks > 0 ? sp.bblocks : 1) * sm_count, bwant = (N + bw - 1) / bw;
        if (bgrid > bwant) bgrid = bwant;
        bucket_sort_kernel<<<(unsigned)bgrid, 32 * bw, bbytes, stream>>>(genes, gstride, N, two_n, order, fb);
        // the (normally few) chromosomes whose priorities cluster: bitonic network
        int64_t sgrid = (int64_t)(sp.sblocks > 0 ? sp.sblocks : 1) * sm_count, swant = (N + sw - 1) / sw;
        if (sgrid > swant) sgrid = swant;
        sort_kernel<<<(unsigned)sgrid, 32 * sw, sbytes, stream>>>(genes, gstride, N, two_n, order, fb);
    }
    int rc;
    if (narrow) {  // narrow pass, then the wide kernel over the (normally no) flagged chromosomes
        rc = launch_any<INTD, OutT, true>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                        visits, ops_out, ostride, lens_out, order, seq, retry, nullptr, stream,
                                        sm_count);
        if (!rc)
            rc = launch_any<INTD, OutT, false>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                             scheduled, visits, ops_out, ostride, lens_out, order, seq,
                                             nullptr, retry, stream, sm_count);
    } else {
        rc = launch_any<INTD, OutT, false>(I, genes, gstride, N, relax, penalty, fitness, makespan, scheduled,
                                         visits, ops_out, ostride, lens_out, order, seq, nullptr, nullptr,
                                         stream, sm_count);
    }
    release();
    return rc;
}

}  // namespace

int launch_decode(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
                  double penalty, double *fitness, double *makespan, int32_t *scheduled,
                  int64_t *visits, void *ops_out, int op_bytes, int64_t ostride,
                  int32_t *lens_out, cudaStream_t stream, int sm_count) {
    if (op_bytes == 2) {
        if (I.integral)
            return launch_t<true, int16_t>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                           scheduled, visits, ops_out, ostride, lens_out, stream, sm_count);
        return launch_t<false, int16_t>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                        scheduled, visits, ops_out, ostride, lens_out, stream, sm_count);
    }
    if (I.integral)
        return launch_t<true, int32_t>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                       scheduled, visits, ops_out, ostride, lens_out, stream, sm_count);
    return launch_t<false, int32_t>(I, genes, gstride, N, relax, penalty, fitness, makespan,
                                    scheduled, visits, ops_out, ostride, lens_out, stream, sm_count);
}
