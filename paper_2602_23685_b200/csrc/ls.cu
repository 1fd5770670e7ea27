// ls.cu -- candidate builder for the batched local search (alns.py:416-487,
// SURVEY §8(f) row 1): pickup_repositioning and cross_agent_relocation
// neighbourhoods materialised on the device, straight into the int16/int32
// batch layout that K2 (two_pass_estimate) and K1 (exact_makespan) consume.
//
// One warp per candidate.  The move is decoded from the candidate's global
// index in the reference's generation order, then the 2n ops are written with
// a branch-free position map (coalesced reads of the L2-resident base
// solution, coalesced writes):
//   pickup move  (entry = worker, v, i, fi): drop the pickup at route position
//       i of vehicle v (flat fi), re-insert it at every (w, g) of the reduced
//       solution except (v, i): K = 2n + m - 2 candidates per entry
//   cross move   (entry = worker, c, w, f1, f2): strip customer c's two ops
//       (flat f1 < f2), insert D at gd and P at gp > gd on vehicle w:
//       (L+1)(L+2)/2 candidates per entry, gd-major
// and the two_opt_improve neighbourhoods (baselines.py:372-455):
//   2-opt        (entry = worker, v): reverse positions i < j of route v,
//       L(L-1)/2 candidates, i-major
//   swap         (entry = worker): swap flat ops a < b, 2n(2n-1)/2, a-major
// (its relocation neighbourhood is the pickup move applied to every op)
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace {

// t-th pair (x, y), 0 <= x < y < K, in x-major order: S(x) = x (K-1) - x (x-1) / 2
__device__ __forceinline__ void tri_decode(int64_t t, int K, int &x, int &y) {
    const double A = 2.0 * K - 1.0;
    int g = (int)floor((A - sqrt(A * A - 8.0 * (double)t)) / 2.0);
    if (g < 0) g = 0;
    if (g > K - 2) g = K - 2;
    auto S = [&](int64_t q) { return q * (K - 1) - q * (q - 1) / 2; };
    while (g > 0 && S(g) > t) --g;
    while (g < K - 2 && S(g + 1) <= t) ++g;
    x = g;
    y = g + 1 + (int)(t - S(g));
}

template <typename OpT>
__global__ void __launch_bounds__(256)
ls_build_kernel(int kind, int n, int m, const int32_t *__restrict__ base_ops, const int32_t *__restrict__ base_lens,
                const int32_t *__restrict__ entries, const int64_t *__restrict__ entry_start, int64_t n_entries,
                const int64_t *__restrict__ index_list, int64_t first, int64_t count,
                OpT *__restrict__ out_ops, int32_t *__restrict__ out_lens) {
    const int lane = threadIdx.x & 31;
    const int64_t cand = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (cand >= count) return;
    const int64_t gidx = index_list ? index_list[cand] : first + cand;
    const int n2 = 2 * n;
    // ---- decode (all lanes redundantly; warp-uniform)
    int64_t e;
    if (kind == 0) {
        e = gidx / (int64_t)(n2 + m - 2);
    } else {
        int64_t lo = 0, hi = n_entries - 1;  // last entry with start <= gidx
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (entry_start[mid] <= gidx) lo = mid; else hi = mid - 1;
        }
        e = lo;
    }
    const int32_t *E = entries + e * 5;
    const int worker = E[0];
    const int32_t *ops = base_ops + (int64_t)worker * n2;
    const int32_t *lens = base_lens + (int64_t)worker * m;
    int L_lane = lane < m ? lens[lane] : 0;
    OpT *oo = out_ops + cand * n2;
    int32_t *ol = out_lens + cand * m;
    if (kind == 0) {
        const int v = E[1], i = E[2], fi = E[3];
        const int op = ops[fi];
        int j = (int)(gidx - e * (int64_t)(n2 + m - 2));
        // base lens, enumeration of (w, g) with (v, i) excluded
        const int lb_lane = L_lane - (lane == v ? 1 : 0);
        int ex = 0, w = 0, g = 0, boff = 0;
        for (int u = 0; u < v; ++u) ex += __shfl_sync(VRP_FULL_MASK, lb_lane, u) + 1;
        ex += i;
        if (j >= ex) ++j;
        for (int u = 0; u < m; ++u) {
            const int gaps = __shfl_sync(VRP_FULL_MASK, lb_lane, u) + 1;
            if (j < gaps) { w = u; g = j; break; }
            j -= gaps;
            boff += gaps - 1;
        }
        const int p = boff + g;
        for (int o = lane; o < n2; o += 32) {
            const int x = o < p ? o : o - 1;  // base index (unused when o == p)
            const int val = o == p ? op : ops[x < fi ? x : x + 1];
            oo[o] = (OpT)val;
        }
        if (lane < m) ol[lane] = lb_lane + (lane == w ? 1 : 0);
    } else if (kind == 2 || kind == 3) {
        // kind 2: reverse positions i..j of route E[1]; kind 3: swap flat ops a < b
        const int64_t t = gidx - entry_start[e];
        int lo, hi;
        if (kind == 2) {
            const int v = E[1];
            int off = 0;
            for (int u = 0; u < v; ++u) off += __shfl_sync(VRP_FULL_MASK, L_lane, u);
            const int Lv = __shfl_sync(VRP_FULL_MASK, L_lane, v);
            int i, j;
            tri_decode(t, Lv, i, j);
            lo = off + i;
            hi = off + j;
            for (int o = lane; o < n2; o += 32) oo[o] = (OpT)ops[(o >= lo && o <= hi) ? lo + hi - o : o];
        } else {
            tri_decode(t, n2, lo, hi);
            for (int o = lane; o < n2; o += 32) oo[o] = (OpT)ops[o == lo ? hi : (o == hi ? lo : o)];
        }
        if (lane < m) ol[lane] = L_lane;
    } else {
        const int c = E[1], w = E[2], f1 = E[3], f2 = E[4];
        const int64_t t = gidx - entry_start[e];
        // stripped lens: c's ops removed from whichever routes hold them
        int sl_lane = L_lane;
        {
            // route of flat position f: the lane whose [off, off+L) holds it
            int off = L_lane;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(VRP_FULL_MASK, off, o);
                if (lane >= o) off += y;
            }
            off -= L_lane;
            if (lane < m) sl_lane -= (f1 >= off && f1 < off + L_lane) + (f2 >= off && f2 < off + L_lane);
        }
        int soff = 0;
        for (int u = 0; u < w; ++u) soff += __shfl_sync(VRP_FULL_MASK, sl_lane, u);
        const int Lw = __shfl_sync(VRP_FULL_MASK, sl_lane, w);
        int gd, gp;  // D at gd, P at gp: pairs of [0, Lw + 1]
        tri_decode(t, Lw + 2, gd, gp);
        const int pd = soff + gd, pp = soff + gp;
        const int dop = 2 * (c - 1), pop = dop + 1;
        for (int o = lane; o < n2; o += 32) {
            int val;
            if (o == pd) val = dop;
            else if (o == pp) val = pop;
            else {
                const int x = o < pd ? o : (o < pp ? o - 1 : o - 2);  // stripped index
                val = ops[x + (x >= f1) + (x >= f2 - 1)];
            }
            oo[o] = (OpT)val;
        }
        if (lane < m) ol[lane] = sl_lane + (lane == w ? 2 : 0);
    }
}

// ---- per-solution top-K of the local-search survivors (alns.py:401-413: the
// stable sort by estimate + [:_VERIFY_LIMIT] over candidates in generation
// order == the K smallest (estimate, generation index) pairs)
constexpr int LS_SEG = 2048;  // candidates per segment (one worker each)

__device__ __forceinline__ bool zi_lt(double za, int64_t ia, double zb, int64_t ib) {
    return za < zb || (za == zb && ia < ib);
}

// segment s: the K smallest survivors (status 0, z < zthr[worker]) of
// candidates [seg_begin, seg_end) -- K rounds of block argmin above the last pick
__global__ void __launch_bounds__(256)
ls_seg_topk_kernel(const double *__restrict__ z, const int32_t *__restrict__ status, int64_t first,
                   const double *__restrict__ zthr, const int32_t *__restrict__ seg_worker,
                   const int64_t *__restrict__ seg_begin, const int64_t *__restrict__ seg_end, int K,
                   double *__restrict__ out_z, int64_t *__restrict__ out_i, int32_t *__restrict__ out_n) {
    __shared__ double sz[8];
    __shared__ int64_t si[8];
    constexpr int PER = LS_SEG / 256;
    const int s = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b = seg_begin[s], e = seg_end[s];
    const double thr = zthr[seg_worker[s]];
    double vz[PER];
    int64_t vi[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int64_t g = b + threadIdx.x + 256 * k;
        const bool ok = g < e && status[g - first] == 0 && z[g - first] < thr;
        vz[k] = ok ? z[g - first] : INFINITY;
        vi[k] = ok ? g : INT64_MAX;
    }
    double lz = -INFINITY;
    int64_t li = -1;
    int cnt = 0;
    for (int r = 0; r < K; ++r) {
        double bz = INFINITY;
        int64_t bi = INT64_MAX;
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (vi[k] != INT64_MAX && zi_lt(lz, li, vz[k], vi[k]) && zi_lt(vz[k], vi[k], bz, bi)) { bz = vz[k]; bi = vi[k]; }
        for (int o = 16; o; o >>= 1) {
            const double oz = __shfl_xor_sync(VRP_FULL_MASK, bz, o);
            const int64_t oi = __shfl_xor_sync(VRP_FULL_MASK, bi, o);
            if (zi_lt(oz, oi, bz, bi)) { bz = oz; bi = oi; }
        }
        if (lane == 0) { sz[warp] = bz; si[warp] = bi; }
        __syncthreads();
        bz = INFINITY; bi = INT64_MAX;
        for (int w = 0; w < 8; ++w)
            if (zi_lt(sz[w], si[w], bz, bi)) { bz = sz[w]; bi = si[w]; }
        __syncthreads();
        if (bi == INT64_MAX) break;
        if (threadIdx.x == 0) { out_z[(int64_t)s * K + r] = bz; out_i[(int64_t)s * K + r] = bi; }
        lz = bz; li = bi;
        ++cnt;
    }
    if (threadIdx.x == 0) out_n[s] = cnt;
}

// worker w: merge its running list with its segments' lists (warp per worker)
__global__ void __launch_bounds__(32)
ls_merge_topk_kernel(const int32_t *__restrict__ workers, const int32_t *__restrict__ wseg_first,
                     const int32_t *__restrict__ wseg_count, int K, const double *__restrict__ seg_z,
                     const int64_t *__restrict__ seg_i, const int32_t *__restrict__ seg_n,
                     double *__restrict__ top_z, int64_t *__restrict__ top_i, int32_t *__restrict__ top_n) {
    const int lane = threadIdx.x;
    const int w = workers[blockIdx.x];
    const int s0 = wseg_first[blockIdx.x], ns = wseg_count[blockIdx.x];
    const int tot = (ns + 1) * K;  // slot j < K: running list; then K per segment
    auto at = [&](int j, double &zz, int64_t &ii) -> bool {
        const int src = j / K, r = j - src * K;
        if (src == 0) {
            if (r >= top_n[w]) return false;
            zz = top_z[(int64_t)w * K + r]; ii = top_i[(int64_t)w * K + r];
            return true;
        }
        const int s = s0 + src - 1;
        if (r >= seg_n[s]) return false;
        zz = seg_z[(int64_t)s * K + r]; ii = seg_i[(int64_t)s * K + r];
        return true;
    };
    double lz = -INFINITY, pz[16];
    int64_t li = -1, pi[16];
    int cnt = 0;
    for (int r = 0; r < K; ++r) {
        double bz = INFINITY;
        int64_t bi = INT64_MAX;
        for (int j = lane; j < tot; j += 32) {
            double zz;
            int64_t ii;
            if (at(j, zz, ii) && zi_lt(lz, li, zz, ii) && zi_lt(zz, ii, bz, bi)) { bz = zz; bi = ii; }
        }
        for (int o = 16; o; o >>= 1) {
            const double oz = __shfl_xor_sync(VRP_FULL_MASK, bz, o);
            const int64_t oi = __shfl_xor_sync(VRP_FULL_MASK, bi, o);
            if (zi_lt(oz, oi, bz, bi)) { bz = oz; bi = oi; }
        }
        if (bi == INT64_MAX) break;
        pz[r] = bz; pi[r] = bi;
        lz = bz; li = bi;
        ++cnt;
    }
    __syncwarp();  // every lane has read the running list before lane 0 rewrites it
    if (lane == 0) {
        for (int r = 0; r < cnt; ++r) { top_z[(int64_t)w * K + r] = pz[r]; top_i[(int64_t)w * K + r] = pi[r]; }
        top_n[w] = cnt;
    }
}

// ---- the neighbourhood entries of every solution, built on the device from
// the evaluate returns (alns.py:416-487's generation order), so the local
// search never copies solutions back to the host.  Block (one warp) per
// solution; count phase (eoff == null): entries and candidates per solution;
// fill phase: entries[e] and entry_start[e] at the host-scanned offsets.
//   kind 0 (pickup_repositioning, :416-450): solutions with z > 0, vehicles
//     whose return >= 0.9 z, every pickup in route order:
//     {w, v, i, flat, 0}, 2n + m - 2 candidates each
//   kind 1 (cross_agent_relocation, :453-487): b = first argmax of the
//     returns; customers of route b ascending; every other vehicle u:
//     {w, c, u, f1, f2} (f1 < f2: c's flat positions), (L+1)(L+2)/2
//     candidates, L = route u's length without c's ops
__global__ void __launch_bounds__(32)
ls_entries_kernel(int kind, int n, int m, const int32_t *__restrict__ base_ops, const int32_t *__restrict__ base_lens,
                  const double *__restrict__ z, const double *__restrict__ returns,
                  const uint8_t *__restrict__ active, const int64_t *__restrict__ eoff,
                  const int64_t *__restrict__ coff, int32_t *__restrict__ ecount, int64_t *__restrict__ ccount,
                  int32_t *__restrict__ entries, int64_t *__restrict__ starts) {
    extern __shared__ int32_t s_first[];  // kind 1: first / second flat position of each customer
    const int w = blockIdx.x, lane = threadIdx.x, n2 = 2 * n;
    const int32_t *ops = base_ops + (int64_t)w * n2;
    const int32_t *lens = base_lens + (int64_t)w * m;
    const double *ret = returns + (int64_t)w * m;
    const bool fill = eoff != nullptr;
    const int64_t e0 = fill ? eoff[w] : 0, c0 = fill ? coff[w] : 0;
    int ne = 0;
    int64_t nc = 0;
    if (active[w] && kind == 0) {
        const double zw = z[w];
        if (!(zw <= 0.0)) {
            const int64_t K = n2 + m - 2;
            int off = 0;
            for (int v = 0; v < m; ++v) {
                const int Lv = lens[v];
                if (ret[v] >= 0.9 * zw) {
                    for (int b = 0; b < Lv; b += 32) {
                        const int i = b + lane;
                        const bool pk = i < Lv && (ops[off + i] & 1);
                        const unsigned bal = __ballot_sync(VRP_FULL_MASK, pk);
                        if (fill && pk) {
                            const int64_t r = ne + __popc(bal & lanemask_lt());
                            int32_t *E = entries + (e0 + r) * 5;
                            E[0] = w; E[1] = v; E[2] = i; E[3] = off + i; E[4] = 0;
                            starts[e0 + r] = c0 + r * K;
                        }
                        ne += __popc(bal);
                    }
                }
                off += Lv;
            }
            nc = (int64_t)ne * K;
        }
    } else if (active[w] && kind == 1 && m > 1) {
        int b = 0;
        for (int v = 1; v < m; ++v) b = ret[v] > ret[b] ? v : b;  // np.argmax: first maximum
        int offb = 0, total = 0;
        for (int v = 0; v < m; ++v) {
            if (v < b) offb += lens[v];
            total += lens[v];
        }
        const int Lb = lens[b];
        int32_t *f1 = s_first, *f2 = s_first + n + 1;
        for (int c = lane; c <= n; c += 32) { f1[c] = INT32_MAX; f2[c] = INT32_MAX; }
        __syncwarp();
        for (int q = lane; q < total; q += 32) atomicMin(&f1[op_customer(ops[q])], q);
        __syncwarp();
        for (int q = lane; q < total; q += 32) {
            const int c = op_customer(ops[q]);
            if (q != f1[c]) atomicMin(&f2[c], q);
        }
        __syncwarp();
        for (int cb = 1; cb <= n; cb += 32) {
            const int c = cb + lane;
            const int p1 = c <= n ? f1[c] : INT32_MAX, p2 = c <= n ? f2[c] : INT32_MAX;
            const bool onb = (p1 >= offb && p1 < offb + Lb) || (p2 >= offb && p2 < offb + Lb);
            const unsigned bal = __ballot_sync(VRP_FULL_MASK, onb);
            if (!bal) continue;
            int64_t mine = 0;
            if (onb) {
                int off = 0;
                for (int u = 0; u < m; ++u) {
                    const int Lu = lens[u];
                    if (u != b) {
                        const int L = Lu - (p1 >= off && p1 < off + Lu) - (p2 >= off && p2 < off + Lu);
                        mine += (int64_t)(L + 1) * (L + 2) / 2;
                    }
                    off += Lu;
                }
            }
            int64_t incl = mine;  // inclusive scan over the lanes (customer order)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(VRP_FULL_MASK, incl, o);
                if (lane >= o) incl += y;
            }
            if (fill && onb) {
                int64_t r = ne + (int64_t)__popc(bal & lanemask_lt()) * (m - 1);
                int64_t st = c0 + nc + incl - mine;
                int off = 0;
                for (int u = 0; u < m; ++u) {
                    const int Lu = lens[u];
                    if (u != b) {
                        const int L = Lu - (p1 >= off && p1 < off + Lu) - (p2 >= off && p2 < off + Lu);
                        int32_t *E = entries + (e0 + r) * 5;
                        E[0] = w; E[1] = c; E[2] = u; E[3] = p1; E[4] = p2;
                        starts[e0 + r] = st;
                        st += (int64_t)(L + 1) * (L + 2) / 2;
                        ++r;
                    }
                    off += Lu;
                }
            }
            ne += __popc(bal) * (m - 1);
            nc += __shfl_sync(VRP_FULL_MASK, incl, 31);
        }
    }
    if (!fill && lane == 0) { ecount[w] = ne; ccount[w] = nc; }
}

}  // namespace

int launch_ls_build(int kind, int n, int m, const int32_t *base_ops, const int32_t *base_lens,
                    const int32_t *entries, const int64_t *entry_start, int64_t n_entries,
                    const int64_t *index_list, int64_t first, int64_t count, void *out_ops, int op_bytes,
                    int32_t *out_lens, cudaStream_t stream) {
    if (count <= 0) return 0;
    const int wpb = 8;
    const int64_t blocks = (count + wpb - 1) / wpb;
    if (op_bytes == 2)
        ls_build_kernel<int16_t><<<(unsigned)blocks, 32 * wpb, 0, stream>>>(
            kind, n, m, base_ops, base_lens, entries, entry_start, n_entries, index_list, first, count,
            (int16_t *)out_ops, out_lens);
    else
        ls_build_kernel<int32_t><<<(unsigned)blocks, 32 * wpb, 0, stream>>>(
            kind, n, m, base_ops, base_lens, entries, entry_start, n_entries, index_list, first, count,
            (int32_t *)out_ops, out_lens);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

int launch_ls_topk(const double *z, const int32_t *status, int64_t first, const double *zthr,
                   const int32_t *seg_worker, const int64_t *seg_begin, const int64_t *seg_end, int64_t nseg,
                   const int32_t *workers, const int32_t *wseg_first, const int32_t *wseg_count, int32_t nworkers,
                   int32_t K, double *top_z, int64_t *top_i, int32_t *top_n, cudaStream_t stream) {
    if (nseg <= 0 || nworkers <= 0) return 0;
    double *sz = nullptr;
    int64_t *si = nullptr;
    int32_t *sn = nullptr;
    if (cudaMallocAsync(&sz, sizeof(double) * (size_t)nseg * K, stream) != cudaSuccess) return -1;
    if (cudaMallocAsync(&si, sizeof(int64_t) * (size_t)nseg * K, stream) != cudaSuccess ||
        cudaMallocAsync(&sn, sizeof(int32_t) * (size_t)nseg, stream) != cudaSuccess) {
        cudaFreeAsync(sz, stream);
        if (si) cudaFreeAsync(si, stream);
        return -1;
    }
    ls_seg_topk_kernel<<<(unsigned)nseg, 256, 0, stream>>>(z, status, first, zthr, seg_worker, seg_begin, seg_end, K,
                                                           sz, si, sn);
    ls_merge_topk_kernel<<<(unsigned)nworkers, 32, 0, stream>>>(workers, wseg_first, wseg_count, K, sz, si, sn,
                                                                top_z, top_i, top_n);
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(sz, stream);
    cudaFreeAsync(si, stream);
    cudaFreeAsync(sn, stream);
    return e == cudaSuccess ? 0 : -1;
}

int launch_ls_entries(int kind, int n, int m, const int32_t *base_ops, const int32_t *base_lens, const double *z,
                      const double *returns, const uint8_t *active, int32_t W, const int64_t *entry_off,
                      const int64_t *cand_off, int32_t *entry_count, int64_t *cand_count, int32_t *entries,
                      int64_t *entry_start, cudaStream_t stream) {
    if (W <= 0) return 0;
    const size_t smem = kind == 1 ? sizeof(int32_t) * 2 * (size_t)(n + 1) : 0;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(ls_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    ls_entries_kernel<<<(unsigned)W, 32, smem, stream>>>(kind, n, m, base_ops, base_lens, z, returns, active,
                                                          entry_off, cand_off, entry_count, cand_count, entries,
                                                          entry_start);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}
