// evolve.cu -- K4: the BRKGA generation step on device (brkga.py:231-252,
// run_brkga :454-467).
//
//  order   stable argsort of the fitness (brkga.py:243, :456): the rank of
//          every (fitness key, index) pair -- equal fitnesses keep index
//          order, exactly as numpy's stable sort -- from 1024-pair tiles
//          sorted in shared memory and log2(N / 1024) merge-path passes:
//          57 us at N = 30,000 (round 1's O(N^2) rank count: 1.31 ms).
//  draws   numpy Generator(Philox) reproduced bit for bit.  Philox4x64-10 is
//          counter based, so the q-th 64-bit output of the stream is a pure
//          function of (state, q): mutant genes, the e_idx/o_idx Lemire draws
//          and the crossover mask are all computed in parallel.  A Lemire
//          rejection (probability (2^32 mod n)/2^32 per draw) shifts every
//          later 32-bit draw; draws are computed optimistically, the first
//          rejection is found with atomicMin, and one thread redoes the
//          remaining draws sequentially (rare: ~1.5 % of generations at
//          N = 30,000).  The final state -- counter, 4-word buffer, buffer
//          position, pending u32 half -- is written back so the caller's
//          generator continues exactly where numpy's would.
//  build   [elites | mutants | offspring] rows; offspring gene = mask ?
//          elite parent : other parent.  HBM-bound: 3 x 4n x 8 B per
//          offspring (two parent reads, one write); one Philox block per
//          thread serves 4 genes (was one block per gene).
//  best    block reduction of (fitness, first index) over the new rows; the
//          strict `<` against the incumbent is evaluated on device and the
//          winning chromosome copied (run_brkga's best tracking, :461-467).
#include <float.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace {

// k-th u32 drawn after `base` u64s were consumed, given the pending half
__device__ __forceinline__ uint32_t stream_u32(const vrp_philox &S, uint64_t base, uint64_t k) {
    if (S.has_uint32) {
        if (k == 0) return S.uinteger;
        --k;
    }
    const uint64_t x = stream_u64(S, base + k / 2);
    return (k & 1) ? (uint32_t)(x >> 32) : (uint32_t)x;
}

__device__ __forceinline__ uint64_t fit_key(double x) {
    if (x != x) return 0xFFFFFFFFFFFFFFFFull;
    if (x == 0.0) x = 0.0;
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Stable order = rank of every (key, index) pair in the total order of the
// pairs (equal fitnesses keep index order, numpy's stable argsort):
//   sort_tiles_kernel  each block sorts a tile of 1024 pairs in shared memory
//                      (bitonic network on the composite key -- a total order,
//                      so the result is unique)
//   merge_kway_kernel  log_4(N / 1024) 4-way merge passes over the sorted
//                      runs of packed 16-byte (key, index) pairs (3 binary
//                      searches per element and pass, advanced in lockstep);
//                      the last pass writes the first N indices: the order.
#ifndef RANK_TILE_N
#define RANK_TILE_N 512  // measured at N = 30,000: 512 -> 44 us, 1024 -> 47 us, 2048 -> 54 us
#endif
constexpr int RANK_TILE = RANK_TILE_N;  // pairs per shared-memory tile (threads: half of it)
#ifndef ORDER_WAYS
#define ORDER_WAYS 4  // runs merged per pass (2: the binary merge-path pass)
#endif

__device__ __forceinline__ bool pair_lt(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(RANK_TILE / 2) sort_tiles_kernel(const double *__restrict__ fit, int64_t N,
                                                         ulonglong2 *__restrict__ sp, int32_t *__restrict__ order) {
    __shared__ uint64_t k[RANK_TILE];
    __shared__ int32_t ix[RANK_TILE];
    const int64_t base = (int64_t)blockIdx.x * RANK_TILE;
    for (int t = threadIdx.x; t < RANK_TILE; t += blockDim.x) {
        const int64_t i = base + t;
        k[t] = i < N ? fit_key(__ldg(fit + i)) : ~0ull;
        ix[t] = (int32_t)i;  // padding (i >= N) keeps unique indices and sorts last
    }
    __syncthreads();
    for (int size = 2; size <= RANK_TILE; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < RANK_TILE / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t ka = k[lo], kb = k[hi];
                const int32_t ia = ix[lo], ib = ix[hi];
                if (pair_lt(kb, ib, ka, ia) == up) { k[lo] = kb; k[hi] = ka; ix[lo] = ib; ix[hi] = ia; }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < RANK_TILE; t += blockDim.x) {
        if (order) {  // a single tile: it is the order
            if (base + t < N) order[base + t] = ix[t];
        } else {
            sp[base + t] = make_ulonglong2(k[t], (unsigned long long)(uint32_t)ix[t]);
        }
    }
}

// one K-way merge pass: sorted runs of S pairs -> runs of K S.  A pair's place
// in its merged run = its rank in its own run + the number of pairs below it
// in each of the other K - 1 runs of its group (independent binary searches,
// so the pass costs one search latency, not K - 1); pairs are unique.
template <int K>
__global__ void __launch_bounds__(256) merge_kway_kernel(const ulonglong2 *__restrict__ pin, int64_t total, int64_t S,
                                                         ulonglong2 *__restrict__ pout, int32_t *__restrict__ order,
                                                         int64_t N) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const ulonglong2 e = pin[i];  // (key, index) in one 16-byte load
    const int64_t r = i / S, g0 = (r / K) * K;
    int64_t lo[K], hi[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        const int64_t rq = g0 + q, ps = rq * S;
        lo[q] = ps;
        hi[q] = (rq == r || ps >= total) ? ps : (ps + S < total ? ps + S : total);
    }
    // the K - 1 searches advance in lockstep: their loads are independent
    for (int64_t w = S; w > 0; w >>= 1) {
#pragma unroll
        for (int q = 0; q < K; ++q) {
            if (lo[q] < hi[q]) {
                const int64_t mid = (lo[q] + hi[q]) >> 1;
                const ulonglong2 x = pin[mid];
                if (pair_lt(x.x, (int32_t)x.y, e.x, (int32_t)e.y)) lo[q] = mid + 1;
                else hi[q] = mid;
            }
        }
    }
    int64_t pos = g0 * S + (i - r * S);
#pragma unroll
    for (int q = 0; q < K; ++q) pos += lo[q] - (g0 + q) * S;
    if (order) {  // the last pass writes the order (the first N pairs are the real ones)
        if (pos < N) order[pos] = (int32_t)e.y;
    } else {
        pout[pos] = e;
    }
}

struct EvolveShape {
    int64_t N, G, n_elite, n_mutant, n_off;
    int e_draws, o_draws;  // 1 if the range consumes draws (range > 1), else 0
    uint32_t e_range, o_range;
};

__device__ __forceinline__ bool lemire(uint32_t u, uint32_t range, uint32_t &out) {
    const uint64_t m = (uint64_t)u * range;
    const uint32_t left = (uint32_t)m;
    out = (uint32_t)(m >> 32);
    if (left < range) {
        const uint32_t thresh = (0u - range) % range;
        if (left < thresh) return false;  // numpy would reject and redraw
    }
    return true;
}

// optimistic e_idx / o_idx; first rejecting draw index -> *first_rej
__global__ void draw_kernel(const vrp_philox *__restrict__ Sp, EvolveShape sh, int32_t *__restrict__ e_idx,
                            int32_t *__restrict__ o_idx, unsigned long long *__restrict__ first_rej) {
    const vrp_philox S = *Sp;
    const uint64_t base = (uint64_t)(sh.n_mutant * sh.G);
    const int64_t tot = (int64_t)(sh.e_draws + sh.o_draws) * sh.n_off;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < 2 * sh.n_off;
         k += (int64_t)gridDim.x * blockDim.x) {
        const bool is_e = k < sh.n_off;
        const int64_t i = is_e ? k : k - sh.n_off;
        const int used = is_e ? sh.e_draws : sh.o_draws;
        if (!used) {
            (is_e ? e_idx : o_idx)[i] = 0;
            continue;
        }
        const int64_t d = is_e ? i : (int64_t)sh.e_draws * sh.n_off + i;  // u32 draw number
        uint32_t v;
        const bool ok = lemire(stream_u32(S, base, (uint64_t)d), is_e ? sh.e_range : sh.o_range, v);
        (is_e ? e_idx : o_idx)[i] = (int32_t)v;
        if (!ok) atomicMin(first_rej, (unsigned long long)d);
    }
    (void)tot;
}

// sequential redo from the first rejection; writes the u32 count consumed
__global__ void fix_kernel(const vrp_philox *__restrict__ Sp, EvolveShape sh, int32_t *__restrict__ e_idx,
                           int32_t *__restrict__ o_idx, const unsigned long long *__restrict__ first_rej,
                           unsigned long long *__restrict__ u32_used) {
    const vrp_philox S = *Sp;
    const uint64_t base = (uint64_t)(sh.n_mutant * sh.G);
    const int64_t ndraw = (int64_t)(sh.e_draws + sh.o_draws) * sh.n_off;
    const unsigned long long fr = *first_rej;
    if (fr >= (unsigned long long)ndraw) { *u32_used = (unsigned long long)ndraw; return; }
    uint64_t k = fr;  // u32 position of draw number fr (no rejection before it)
    for (int64_t d = (int64_t)fr; d < ndraw; ++d) {
        const bool is_e = sh.e_draws && d < sh.n_off;
        const uint32_t range = is_e ? sh.e_range : sh.o_range;
        uint32_t v;
        while (!lemire(stream_u32(S, base, k++), range, v)) {}
        if (is_e) e_idx[d] = (int32_t)v;
        else o_idx[d - (int64_t)sh.e_draws * sh.n_off] = (int32_t)v;
    }
    *u32_used = k;
}

__device__ __forceinline__ uint64_t u64s_for_u32(const vrp_philox &S, uint64_t used) {
    const uint64_t from_u64 = used > (uint64_t)S.has_uint32 ? used - S.has_uint32 : 0;
    return (from_u64 + 1) / 2;
}

// rows [elites | mutants | offspring], in three launches:
//   elite rows: 16-byte row copies (G = 4n is even: 16-byte aligned rows);
//   mutant / offspring rows: one thread per Philox block (4 consecutive
//     stream words -> 4 consecutive genes of a row; G is a multiple of 4, so
//     every row has the same block phase), one block row per grid row.
template <bool VEC>  // VEC: G even and both bases 16-byte aligned (BRKGA's 4n genes)
__global__ void __launch_bounds__(256) elite_rows_kernel(const double *__restrict__ pop,
                                                         const int32_t *__restrict__ order, int64_t G,
                                                         double *__restrict__ out, int64_t row0) {
    const int64_t r = row0 + blockIdx.y;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    if (VEC) {
        const double2 *src = reinterpret_cast<const double2 *>(pop + (int64_t)order[r] * G);
        double2 *dst = reinterpret_cast<double2 *>(out + r * G);
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < G / 2; j += step) dst[j] = __ldg(src + j);
    } else {
        const double *src = pop + (int64_t)order[r] * G;
        double *dst = out + r * G;
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < G; j += step) dst[j] = __ldg(src + j);
    }
}

// OFF = false: mutant row r (stream words r*G ..); OFF = true: offspring row r
// (mask words mask0 + r*G ..; gene = mask < bias ? elite parent : other parent)
template <bool OFF>
__global__ void __launch_bounds__(256) stream_rows_kernel(const vrp_philox *__restrict__ Sp, EvolveShape sh,
                                                          const double *__restrict__ pop,
                                                          const int32_t *__restrict__ order,
                                                          const int32_t *__restrict__ e_idx,
                                                          const int32_t *__restrict__ o_idx,
                                                          const unsigned long long *__restrict__ u32_used,
                                                          double bias, double *__restrict__ out, int64_t row0) {
    const vrp_philox S = *Sp;
    const int64_t G = sh.G, r = row0 + blockIdx.y;
    const int64_t head = 4 - (int64_t)S.buffer_pos;
    const int64_t q0 = (OFF ? (int64_t)(sh.n_mutant * G) + (int64_t)u64s_for_u32(S, *u32_used) : 0) + r * G;
    // block-aligned start (stream words >= head come in Philox blocks of 4)
    const int64_t qq0 = q0 - head;
    const int64_t b0 = qq0 >= 0 ? qq0 / 4 : -((3 - qq0) / 4);
    const int64_t nblk = (qq0 + G - 1 - 4 * b0) / 4 + 1;
    const double *pe = nullptr, *po = nullptr;
    if (OFF) {
        pe = pop + (int64_t)order[e_idx[r]] * G;
        po = pop + (int64_t)order[sh.n_elite + o_idx[r]] * G;
    }
    double *dst = out + ((OFF ? sh.n_elite + sh.n_mutant : sh.n_elite) + r) * G;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nblk; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t qqb = 4 * (b0 + j);
        uint64_t w[4];
        if (qqb >= 0) {
            uint64_t c[4];
            ctr_add(S.ctr, 1 + (uint64_t)(qqb / 4), c);
            philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], w);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t g = qqb + k - qq0;
            if (g < 0 || g >= G) continue;
            const int64_t qq = qqb + k;
            const uint64_t x = qq >= 0 ? w[k] : S.buffer[S.buffer_pos + (qq + head)];
            const double u = u64_to_double(x);
            dst[g] = OFF ? __ldg((u < bias ? pe : po) + g) : u;
        }
    }
}

// Offspring row r (mask words mask0 + r*G ..): phase 1, one thread per Philox
// block, writes the row's mask verdicts (u < bias) to shared memory; phase 2
// copies both parents 16 bytes at a time and selects per gene (both parents'
// sectors are fetched either way -- the mask is random per gene).
__global__ void __launch_bounds__(256) offspring_rows_kernel(const vrp_philox *__restrict__ Sp, EvolveShape sh,
                                                             const double *__restrict__ pop,
                                                             const int32_t *__restrict__ order,
                                                             const int32_t *__restrict__ e_idx,
                                                             const int32_t *__restrict__ o_idx,
                                                             const unsigned long long *__restrict__ u32_used,
                                                             double bias, double *__restrict__ out, int64_t row0) {
    extern __shared__ uint8_t s_mask[];
    const vrp_philox S = *Sp;
    const int64_t G = sh.G, r = row0 + blockIdx.y;
    const int64_t head = 4 - (int64_t)S.buffer_pos;
    const int64_t q0 = (int64_t)(sh.n_mutant * G) + (int64_t)u64s_for_u32(S, *u32_used) + r * G;
    const int64_t qq0 = q0 - head;
    const int64_t b0 = qq0 >= 0 ? qq0 / 4 : -((3 - qq0) / 4);
    const int64_t nblk = (qq0 + G - 1 - 4 * b0) / 4 + 1;
    for (int64_t j = threadIdx.x; j < nblk; j += blockDim.x) {
        const int64_t qqb = 4 * (b0 + j);
        uint64_t w[4];
        if (qqb >= 0) {
            uint64_t c[4];
            ctr_add(S.ctr, 1 + (uint64_t)(qqb / 4), c);
            philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], w);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t g = qqb + k - qq0;
            if (g < 0 || g >= G) continue;
            const int64_t qq = qqb + k;
            const uint64_t x = qq >= 0 ? w[k] : S.buffer[S.buffer_pos + (qq + head)];
            s_mask[g] = u64_to_double(x) < bias;
        }
    }
    __syncthreads();
    const double2 *pe = reinterpret_cast<const double2 *>(pop + (int64_t)order[e_idx[r]] * G);
    const double2 *po = reinterpret_cast<const double2 *>(pop + (int64_t)order[sh.n_elite + o_idx[r]] * G);
    double2 *dst = reinterpret_cast<double2 *>(out + (sh.n_elite + sh.n_mutant + r) * G);
    for (int64_t j = threadIdx.x; j < G / 2; j += blockDim.x) {
        const double2 a = __ldg(pe + j), b = __ldg(po + j);
        dst[j] = make_double2(s_mask[2 * j] ? a.x : b.x, s_mask[2 * j + 1] ? a.y : b.y);
    }
}

// advance the caller's generator past everything evolve consumed
__global__ void state_kernel(vrp_philox *__restrict__ Sp, EvolveShape sh,
                             const unsigned long long *__restrict__ u32_used) {
    vrp_philox S = *Sp;
    const uint64_t used32 = *u32_used;
    const uint64_t mut = (uint64_t)(sh.n_mutant * sh.G);
    const uint64_t u64_32 = u64s_for_u32(S, used32);
    // pending half after the integer draws
    int has = S.has_uint32;
    uint32_t pend = S.uinteger;
    if (used32 > 0) {
        if (used32 <= (uint64_t)S.has_uint32) {
            has = 0;
        } else {
            // numpy keeps the high half of the last u64 it split in `uinteger`,
            // pending (odd count) or already consumed (even count, stale)
            const uint64_t from_u64 = used32 - S.has_uint32;
            has = (int)(from_u64 & 1);
            pend = (uint32_t)(stream_u64(S, mut + (from_u64 - 1) / 2) >> 32);
        }
    }
    const uint64_t Q = mut + u64_32 + (uint64_t)(sh.n_off * sh.G);
    const uint64_t head = 4 - (uint64_t)S.buffer_pos;
    if (Q <= head) {
        S.buffer_pos += (int32_t)Q;
    } else {
        const uint64_t qq = Q - head;
        const uint64_t blocks = (qq + 3) / 4;
        uint64_t c[4];
        ctr_add(S.ctr, blocks, c);
        uint64_t buf[4];
        philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], buf);
        for (int j = 0; j < 4; ++j) { S.ctr[j] = c[j]; S.buffer[j] = buf[j]; }
        S.buffer_pos = (int32_t)(((qq - 1) & 3) + 1);
    }
    S.has_uint32 = has;
    S.uinteger = pend;
    *Sp = S;
}

// Generator.random(count) (numpy: (next64 >> 11) * 2^-53, in order): thread b
// produces Philox block b of the stream, thread 0 also the buffered head.
__global__ void random_fill_kernel(const vrp_philox *__restrict__ Sp, int64_t count, double *__restrict__ out) {
    const vrp_philox S = *Sp;
    const int64_t head = 4 - (int64_t)S.buffer_pos;
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0)
        for (int64_t q = 0; q < head && q < count; ++q) out[q] = u64_to_double(S.buffer[S.buffer_pos + q]);
    const int64_t base = head + 4 * b;
    if (base >= count) return;
    uint64_t c[4], o[4];
    ctr_add(S.ctr, 1 + (uint64_t)b, c);
    philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], o);
    for (int j = 0; j < 4 && base + j < count; ++j) out[base + j] = u64_to_double(o[j]);
}

// advance the generator past Q next64 draws (random() leaves the u32 half alone)
__global__ void advance_kernel(vrp_philox *__restrict__ Sp, uint64_t Q) {
    vrp_philox S = *Sp;
    const uint64_t head = 4 - (uint64_t)S.buffer_pos;
    if (Q <= head) {
        S.buffer_pos += (int32_t)Q;
    } else {
        const uint64_t qq = Q - head;
        const uint64_t blocks = (qq + 3) / 4;
        uint64_t c[4], buf[4];
        ctr_add(S.ctr, blocks, c);
        philox_block(c[0], c[1], c[2], c[3], S.key[0], S.key[1], buf);
        for (int j = 0; j < 4; ++j) { S.ctr[j] = c[j]; S.buffer[j] = buf[j]; }
        S.buffer_pos = (int32_t)(((qq - 1) & 3) + 1);
    }
    *Sp = S;
}

// (min fitness, first index) over fit[lo, hi); strict improvement of *best
__global__ void __launch_bounds__(1024) best_kernel(const double *__restrict__ fit, int64_t lo, int64_t hi,
                                                    const double *__restrict__ genes, int64_t G,
                                                    double *__restrict__ best_fit,
                                                    double *__restrict__ best_genes,
                                                    int64_t *__restrict__ best_index,
                                                    double *__restrict__ trace) {
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    __shared__ int64_t win;
    double bv = DBL_MAX;
    int64_t bi = -1;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double f = fit[i];
        if (bi < 0 || f < bv) { bv = f; bi = i; }  // first index within the thread's stride
    }
    // warp then block argmin with first-index ties
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(VRP_FULL_MASK, bv, o);
        const int64_t oi = __shfl_xor_sync(VRP_FULL_MASK, bi, o);
        if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { sv[w] = bv; si[w] = bi; }
    __syncthreads();
    if (w == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        bv = lane < nw ? sv[lane] : DBL_MAX;
        bi = lane < nw ? si[lane] : -1;
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(VRP_FULL_MASK, bv, o);
            const int64_t oi = __shfl_xor_sync(VRP_FULL_MASK, bi, o);
            if (oi >= 0 && (bi < 0 || ov < bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
        }
        if (lane == 0) {
            const bool better = bi >= 0 && (*best_index < 0 || bv < *best_fit);
            win = better ? bi : -1;
            if (better) { *best_fit = bv; *best_index = bi; }
            if (trace) *trace = *best_fit;
        }
    }
    __syncthreads();
    if (win >= 0 && best_genes)
        for (int64_t g = threadIdx.x; g < G; g += blockDim.x) best_genes[g] = genes[win * G + g];
}

__global__ void gather_fit_kernel(const double *__restrict__ fit, const int32_t *__restrict__ order,
                                  int64_t n, double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = fit[order[i]];
}

}  // namespace

int launch_fitness_order(const double *fit, int64_t N, int32_t *order, cudaStream_t stream) {
    if (N <= 0) return 0;
    const int64_t ntiles = (N + RANK_TILE - 1) / RANK_TILE;
    const int64_t total = ntiles * RANK_TILE;
    if (ntiles == 1) {
        sort_tiles_kernel<<<1, RANK_TILE / 2, 0, stream>>>(fit, N, nullptr, order);
        return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
    }
    ulonglong2 *pa = nullptr, *pb = nullptr;
    if (cudaMallocAsync(&pa, sizeof(ulonglong2) * (size_t)total, stream) != cudaSuccess) return -1;
    if (cudaMallocAsync(&pb, sizeof(ulonglong2) * (size_t)total, stream) != cudaSuccess) {
        cudaFreeAsync(pa, stream);
        return -1;
    }
    sort_tiles_kernel<<<(unsigned)ntiles, RANK_TILE / 2, 0, stream>>>(fit, N, pa, nullptr);
    for (int64_t S = RANK_TILE; S < total; S *= ORDER_WAYS) {  // log_K(N / 1024) merge passes
        const bool last = S * ORDER_WAYS >= total;
        merge_kway_kernel<ORDER_WAYS><<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(
            pa, total, S, pb, last ? order : nullptr, N);
        ulonglong2 *t = pa; pa = pb; pb = t;
    }
    cudaFreeAsync(pa, stream);
    cudaFreeAsync(pb, stream);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int launch_evolve(const double *pop, const double *fit, int64_t N, int64_t G, double elite_frac,
                  double mutant_frac, double bias, vrp_philox *state, double *out, int32_t *order,
                  double *elite_fit, cudaStream_t stream, int sm_count) {
    EvolveShape sh;
    sh.N = N;
    sh.G = G;
    sh.n_elite = (int64_t)(elite_frac * (double)N);
    sh.n_mutant = (int64_t)(mutant_frac * (double)N);
    sh.n_off = N - sh.n_elite - sh.n_mutant;
    if (sh.n_elite < 1 || N - sh.n_elite < 1) return -3;  // PopulationTooSmall
    sh.e_range = (uint32_t)sh.n_elite;
    sh.o_range = (uint32_t)(N - sh.n_elite);
    sh.e_draws = sh.n_elite > 1 ? 1 : 0;  // integers(1) consumes nothing (numpy)
    sh.o_draws = N - sh.n_elite > 1 ? 1 : 0;

    int32_t *e_idx = nullptr, *o_idx = nullptr;
    unsigned long long *scal = nullptr;
    const size_t idx_bytes = sizeof(int32_t) * (size_t)(sh.n_off > 0 ? sh.n_off : 1);
    if (cudaMallocAsync(&e_idx, idx_bytes, stream) != cudaSuccess) return -1;
    if (cudaMallocAsync(&o_idx, idx_bytes, stream) != cudaSuccess) return -1;
    if (cudaMallocAsync(&scal, 2 * sizeof(unsigned long long), stream) != cudaSuccess) return -1;
    cudaMemsetAsync(scal, 0xff, sizeof(unsigned long long), stream);

    if (launch_fitness_order(fit, N, order, stream)) return -1;
    if (elite_fit) {
        gather_fit_kernel<<<(unsigned)((sh.n_elite + 255) / 256), 256, 0, stream>>>(fit, order, sh.n_elite,
                                                                                 elite_fit);
    }
    const int grid = sm_count * 8;
    if (sh.n_off > 0) draw_kernel<<<grid, 256, 0, stream>>>(state, sh, e_idx, o_idx, scal);
    fix_kernel<<<1, 1, 0, stream>>>(state, sh, e_idx, o_idx, scal, scal + 1);
    {
        constexpr int64_t YMAX = 65535;  // grid rows per launch
        const bool vec = G % 2 == 0 && ((uintptr_t)pop % 16) == 0 && ((uintptr_t)out % 16) == 0;
        const unsigned gx = (unsigned)(((vec ? G / 2 : G) + 255) / 256);
        for (int64_t r0 = 0; r0 < sh.n_elite; r0 += YMAX) {
            const dim3 grid2(gx, (unsigned)(sh.n_elite - r0 < YMAX ? sh.n_elite - r0 : YMAX));
            if (vec) elite_rows_kernel<true><<<grid2, 256, 0, stream>>>(pop, order, G, out, r0);
            else elite_rows_kernel<false><<<grid2, 256, 0, stream>>>(pop, order, G, out, r0);
        }
        const unsigned bx = (unsigned)((G / 4 + 2 + 255) / 256);
        for (int64_t r0 = 0; r0 < sh.n_mutant; r0 += YMAX)
            stream_rows_kernel<false><<<dim3(bx, (unsigned)(sh.n_mutant - r0 < YMAX ? sh.n_mutant - r0 : YMAX)), 256,
                                        0, stream>>>(state, sh, pop, order, e_idx, o_idx, scal + 1, bias, out, r0);
        for (int64_t r0 = 0; r0 < sh.n_off; r0 += YMAX) {
            const unsigned rows = (unsigned)(sh.n_off - r0 < YMAX ? sh.n_off - r0 : YMAX);
            if (vec && (size_t)G <= 48 * 1024)  // mask row in shared memory, 16-byte parent copies
                offspring_rows_kernel<<<dim3(1, rows), 256, (size_t)G, stream>>>(state, sh, pop, order, e_idx, o_idx,
                                                                             scal + 1, bias, out, r0);
            else
                stream_rows_kernel<true><<<dim3(bx, rows), 256, 0, stream>>>(state, sh, pop, order, e_idx, o_idx,
                                                                            scal + 1, bias, out, r0);
        }
    }
    state_kernel<<<1, 1, 0, stream>>>(state, sh, scal + 1);
    cudaFreeAsync(e_idx, stream);
    cudaFreeAsync(o_idx, stream);
    cudaFreeAsync(scal, stream);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int launch_best_update(const double *fit, int64_t lo, int64_t hi, const double *genes, int64_t G,
                       double *best_fit, double *best_genes, int64_t *best_index, double *trace,
                       cudaStream_t stream) {
    best_kernel<<<1, 1024, 0, stream>>>(fit, lo, hi, genes, G, best_fit, best_genes, best_index, trace);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int launch_random_fill(vrp_philox *state, int64_t count, double *out, cudaStream_t stream) {
    if (count <= 0) return 0;
    const int64_t blocks = (count + 3) / 4;
    const int64_t grid = (blocks + 255) / 256;
    random_fill_kernel<<<(unsigned)grid, 256, 0, stream>>>(state, count, out);
    advance_kernel<<<1, 1, 0, stream>>>(state, (uint64_t)count);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
