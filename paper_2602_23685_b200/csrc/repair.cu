// repair.cu -- K5: ALNS repair (insertion.reinsert_all, insertion.py:484-516)
// for a batch of independent repair instances, one warp per instance.
//
// Each instance is a partial solution, its removed customers, the repair
// operator's regret_k (0 = greedy) and its own numpy-Philox generator.  The
// warp keeps the reference's InsertionContext (insertion.py:52-350) in a
// global scratch block (L1/L2 resident: per route seq, T, dep, M and the
// capacity prefix/suffix bounds; ready / pos_d per customer) and follows the
// reference's control flow exactly, so RNG draws happen in the reference's
// order (customer -> dropoff vehicle -> drop window -> pick window, then the
// greedy outer window):
//   * every gap scan (eval_gaps / eval_pair_gaps, :193-272) runs one gap per
//     lane, results compacted in gap order with ballots;
//   * the three shortlisted dropoff gaps are re-scored by ret_after_drop
//     (:274-310) on three lanes in parallel;
//   * argmin / top-3 / selection windows (_pick_windowed, :414-426) are warp
//     reductions over (cost, stale, a, b) keys; the draw itself is lane 0
//     advancing the instance's generator (Generator.integers semantics);
//   * rebuild_all runs one route per lane; tentative_drop saves and restores
//     the touched state with warp-wide copies.
// Arithmetic is fp64 in the reference's order (-fmad=false), CPython's
// compensated sum() where the reference sums floats (_refresh_aggregates,
// regret), so results are bit-identical for any instance.
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.h"

#include "repair_core.cuh"
#include "repair_team.cuh"

namespace {

template <bool SCAN>
__global__ void __launch_bounds__(128)
repair_kernel(DevInstance I, const int32_t *__restrict__ pops, int64_t pstride,
              const int32_t *__restrict__ plens, const int32_t *__restrict__ removed, int64_t rstride,
              const int32_t *__restrict__ nremoved, const int32_t *__restrict__ regret_k,
              vrp_philox *__restrict__ states, int32_t *__restrict__ out_ops, int64_t ostride,
              int32_t *__restrict__ out_lens, int32_t *__restrict__ status,
              unsigned char *__restrict__ scratch, int64_t N) {
    __shared__ int s_len[4][MAXM];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t inst = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (inst >= N) return;
    const int n = I.n, m = I.m;
    const Layout Ly = make_layout(n, m);
    unsigned char *b = scratch + (size_t)inst * Ly.total;
    Ctx X;
    bind_ctx(X, &I, b, s_len[warp], lane);

    // ---- load the partial solution
    const int32_t *po = pops + inst * pstride;
    const int32_t *pl = plens + inst * m;
    if (lane < m) s_len[warp][lane] = pl[lane];
    __syncwarp();
    int off = 0;
    bool bad = false;
    for (int v = 0; v < m; ++v) {
        const int L = s_len[warp][v];
        bad |= L < 0 || off + L > 2 * n;
        if (!bad)
            for (int i = lane; i < L; i += 32) {
                const int op = po[off + i];
                bad |= op < 0 || op >= 2 * n;
                X.seq[(size_t)v * X.C + i] = op;
            }
        off += L > 0 ? L : 0;
    }
    bad = __any_sync(VRP_FULL_MASK, bad);
    const bool use_rng = states != nullptr;
    PhiloxGen gen;
    if (use_rng && lane == 0) gen.s = states[inst];
    int st = 0;
    if (bad) {
        st = 2;  // malformed partial
    } else {
        rebuild_all<SCAN>(X);
        // remaining = sorted(set(removed)) (insertion.py:488): mark, then compact
        for (int c = lane; c <= n; c += 32) X.s_has[c] = 0;
        __syncwarp();
        const int nr = nremoved[inst];
        for (int i = lane; i < nr; i += 32) {
            const int c = removed[inst * rstride + i];
            if (c >= 1 && c <= n) X.s_has[c] = 1;
        }
        __syncwarp();
        const int nrem = compact_flags(X, X.s_has);
        st = reinsert_core<SCAN>(X, nrem, regret_k[inst], &gen, use_rng);
    }
    // ---- write back
    int32_t *oo = out_ops + inst * ostride;
    off = 0;
    for (int v = 0; v < m; ++v) {
        const int L = st ? 0 : s_len[warp][v];
        for (int i = lane; i < L; i += 32) oo[off + i] = X.seq[(size_t)v * X.C + i];
        off += L;
    }
    for (int i = off + lane; i < 2 * n; i += 32) oo[i] = -1;
    if (lane < m) out_lens[inst * m + lane] = st ? 0 : s_len[warp][lane];
    if (lane == 0) {
        status[inst] = st;
        if (use_rng) states[inst] = gen.s;
    }
}

// The same repair with a CTA of REPAIR_TEAM_WARPS warps per instance (repair_team.cuh):
// integral instances with long routes (use_scan).
__global__ void __launch_bounds__(32 * REPAIR_TEAM_WARPS)
repair_team_kernel(DevInstance I, const int32_t *__restrict__ pops, int64_t pstride,
                   const int32_t *__restrict__ plens, const int32_t *__restrict__ removed, int64_t rstride,
                   const int32_t *__restrict__ nremoved, const int32_t *__restrict__ regret_k,
                   vrp_philox *__restrict__ states, int32_t *__restrict__ out_ops, int64_t ostride,
                   int32_t *__restrict__ out_lens, int32_t *__restrict__ status,
                   unsigned char *__restrict__ scratch, size_t per, int64_t N) {
    __shared__ int s_len[MAXM];
    __shared__ TeamCtl T;
    __shared__ int s_bad, s_nrem;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t inst = blockIdx.x;
    if (inst >= N) return;
    const int n = I.n, m = I.m;
    const Layout Ly = make_layout(n, m);
    unsigned char *b = scratch + (size_t)inst * per;
    Ctx X;
    bind_ctx(X, &I, b, s_len, lane);
    UnitRes *units;
    UnitPick *picks;
    GapRec *crecs;
    TeamCx cx;
    TeamWS W = bind_team(X, b + al8(Ly.total), n, m, warp, nw, units, picks, crecs, cx);
    const bool use_rng = states != nullptr;
    PhiloxGen gen;
    if (warp == 0) {
        const int32_t *po = pops + inst * pstride;
        const int32_t *pl = plens + inst * m;
        if (lane < m) s_len[lane] = pl[lane];
        __syncwarp();
        int off = 0;
        bool bad = false;
        for (int v = 0; v < m; ++v) {
            const int L = s_len[v];
            bad |= L < 0 || off + L > 2 * n;
            if (!bad)
                for (int i = lane; i < L; i += 32) {
                    const int op = po[off + i];
                    bad |= op < 0 || op >= 2 * n;
                    X.seq[(size_t)v * X.C + i] = op;
                }
            off += L > 0 ? L : 0;
        }
        bad = __any_sync(VRP_FULL_MASK, bad);
        if (lane == 0) s_bad = bad;
        if (use_rng && lane == 0) gen.s = states[inst];
    }
    __syncthreads();
    int st = 0;
    if (s_bad) {
        st = 2;
    } else {
        rebuild_all_team(X, crecs, cx, warp, nw);
        if (warp == 0) {
            for (int c = lane; c <= n; c += 32) X.s_has[c] = 0;
            __syncwarp();
            const int nr = nremoved[inst];
            for (int i = lane; i < nr; i += 32) {
                const int c = removed[inst * rstride + i];
                if (c >= 1 && c <= n) X.s_has[c] = 1;
            }
            __syncwarp();
            const int nrem = compact_flags(X, X.s_has);
            if (lane == 0) s_nrem = nrem;
        }
        __syncthreads();
        st = reinsert_team(X, W, T, units, picks, crecs, cx, s_nrem, regret_k[inst], &gen, use_rng, warp, nw);
    }
    if (warp == 0) {
        int32_t *oo = out_ops + inst * ostride;
        int off = 0;
        for (int v = 0; v < m; ++v) {
            const int L = st ? 0 : s_len[v];
            for (int i = lane; i < L; i += 32) oo[off + i] = X.seq[(size_t)v * X.C + i];
            off += L;
        }
        for (int i = off + lane; i < 2 * n; i += 32) oo[i] = -1;
        if (lane < m) out_lens[inst * m + lane] = st ? 0 : s_len[lane];
        if (lane == 0) {
            status[inst] = st;
            if (use_rng) states[inst] = gen.s;
        }
    }
}

}  // namespace

size_t repair_scratch_bytes(int n, int m) { return make_layout(n, m).total; }

int launch_repair(const DevInstance &I, const int32_t *pops, int64_t pstride, const int32_t *plens,
                  const int32_t *removed, int64_t rstride, const int32_t *nremoved,
                  const int32_t *regret_k, vrp_philox *states, int32_t *out_ops, int64_t ostride,
                  int32_t *out_lens, int32_t *status, int64_t N, cudaStream_t stream) {
    if (N <= 0) return 0;
    if (use_team(I)) {
        const size_t per = al8(make_layout(I.n, I.m).total) + team_bytes(I.n, I.m, REPAIR_TEAM_WARPS);
        unsigned char *scratch = nullptr;
        if (cudaMallocAsync(&scratch, per * (size_t)N, stream) != cudaSuccess) return -1;
        repair_team_kernel<<<(unsigned)N, 32 * REPAIR_TEAM_WARPS, 0, stream>>>(I, pops, pstride, plens, removed, rstride,
                                                                      nremoved, regret_k, states, out_ops, ostride,
                                                                      out_lens, status, scratch, per, N);
        const cudaError_t e = cudaPeekAtLastError();
        cudaFreeAsync(scratch, stream);
        return e == cudaSuccess ? 0 : -1;
    }
    const size_t per = make_layout(I.n, I.m).total;
    unsigned char *scratch = nullptr;
    if (cudaMallocAsync(&scratch, per * (size_t)N, stream) != cudaSuccess) return -1;
    const int wpb = 4;
    const int64_t blocks = (N + wpb - 1) / wpb;
    if (use_scan(I))
        repair_kernel<true><<<(unsigned)blocks, 32 * wpb, 0, stream>>>(I, pops, pstride, plens, removed, rstride,
                                                                     nremoved, regret_k, states, out_ops, ostride,
                                                                     out_lens, status, scratch, N);
    else
        repair_kernel<false><<<(unsigned)blocks, 32 * wpb, 0, stream>>>(I, pops, pstride, plens, removed, rstride,
                                                                      nremoved, regret_k, states, out_ops, ostride,
                                                                      out_lens, status, scratch, N);
    const cudaError_t e = cudaPeekAtLastError();
    cudaFreeAsync(scratch, stream);
    return e == cudaSuccess ? 0 : -1;
}
