// capi.cu -- the extern "C" boundary declared in include/vrp_rpd.h.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>

#include "../../include/vrp_rpd.h"
#include "kernels.h"

struct vrp_instance {
    DevInstance dev;
    double *d = nullptr;
    int32_t *d32 = nullptr;
    int32_t *d32t = nullptr;
    double *p = nullptr;
    int32_t *p32 = nullptr;
    int device = 0;
    int sm_count = 148;
};

namespace {
thread_local char g_err[512] = "";

__global__ void probe_kernel() {}
const void *probe_kernel_ptr() { return reinterpret_cast<const void *>(&probe_kernel); }

int fail(int code, const char *fmt, const char *arg = "") {
    snprintf(g_err, sizeof(g_err), fmt, arg);
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return VRP_ECUDA;
}

// Every handle-taking entry point runs on the handle's device (the calling
// thread's current device is restored on return), so one process can drive
// several GPUs with one instance handle per device.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int launch_result(int rc, const char *what) {
    if (rc == 0) return 0;
    cudaError_t e = cudaGetLastError();
    if (rc == -2) return fail(VRP_EUNSUPPORTED, "%s: shared-memory footprint exceeds the SM", what);
    snprintf(g_err, sizeof(g_err), "%s launch failed: %s", what, cudaGetErrorString(e));
    return VRP_ECUDA;
}
}  // namespace

extern "C" {

int vrp_version(int32_t *abi_version, int32_t *compiled_arch) {
    if (abi_version) *abi_version = 1;
    if (compiled_arch) {
        // the SASS architecture of this library's kernels (100 = sm_100a), times 10
        cudaFuncAttributes fa;
        *compiled_arch = cudaFuncGetAttributes(&fa, probe_kernel_ptr()) == cudaSuccess ? fa.binaryVersion * 10 : 1000;
    }
    return 0;
}

const char *vrp_last_error(void) { return g_err; }

int vrp_instance_create(int32_t n, int32_t m, int32_t k, const double *d_host, const double *p_host,
                        vrp_instance_t *out) {
    if (!out || !d_host || !p_host) return fail(VRP_EINVAL, "null argument%s");
    // the binding per-kernel limit: K3's bitonic argsort fallback holds a chromosome's
    // 2n keys (+ indices) padded to a power of two in one warp's shared memory
    // (10 B x 16384 at n = 8192); K1's 64-bit fix-up table fits to n ~ 14.5 k,
    // K2's to ~13 k
    if (n < 1 || n > VRP_MAX_N) return fail(VRP_EUNSUPPORTED, "n must lie in [1, 8192]%s");
    if (m < 1 || m > 32) return fail(VRP_EUNSUPPORTED, "m must lie in [1, 32] (lanes = vehicles)%s");
    if (k < 1) return fail(VRP_EINVAL, "k must be >= 1%s");
    const size_t cells = (size_t)(n + 1) * (size_t)(n + 1);
    bool integral = true;
    for (size_t i = 0; i < cells && integral; ++i) {
        double x = d_host[i];
        if (!(x >= 0.0 && x < 2147483648.0 && x == std::floor(x))) integral = false;
        if (std::signbit(x)) integral = false;  // keep -0.0 bit-exact in the fp64 table
    }
    for (int32_t i = 0; i <= n && integral; ++i) {
        double x = p_host[i];
        if (!(x >= 0.0 && x < 2147483648.0 && x == std::floor(x)) || std::signbit(x)) integral = false;
    }
    vrp_instance *h = new (std::nothrow) vrp_instance();
    if (!h) return fail(VRP_EINVAL, "out of host memory%s");
    cudaError_t e = cudaGetDevice(&h->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
    if (e == cudaSuccess) {
        // kernels take their scratch from the stream-ordered pool; keep freed
        // blocks cached instead of unmapping them at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, h->device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    if (e == cudaSuccess) e = cudaMalloc(&h->d, cells * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&h->p, (size_t)(n + 1) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(h->d, d_host, cells * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->p, p_host, (size_t)(n + 1) * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && integral) {
        int32_t *tmp = new (std::nothrow) int32_t[cells];
        if (!tmp) { vrp_instance_destroy(h); return fail(VRP_EINVAL, "out of host memory%s"); }
        for (size_t i = 0; i < cells; ++i) tmp[i] = (int32_t)d_host[i];
        e = cudaMalloc(&h->d32, cells * sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMemcpy(h->d32, tmp, cells * sizeof(int32_t), cudaMemcpyHostToDevice);
        // the transpose: column c of d as a contiguous row (the repair scans read
        // d[x][c] and d[c][x] for one c over every gap: two L1-resident rows)
        const size_t W = (size_t)n + 1;
        for (size_t a = 0; a < W; ++a)
            for (size_t b = 0; b < W; ++b) tmp[b * W + a] = (int32_t)d_host[a * W + b];
        if (e == cudaSuccess) e = cudaMalloc(&h->d32t, cells * sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMemcpy(h->d32t, tmp, cells * sizeof(int32_t), cudaMemcpyHostToDevice);
        for (int32_t i = 0; i <= n; ++i) tmp[i] = (int32_t)p_host[i];
        if (e == cudaSuccess) e = cudaMalloc(&h->p32, (size_t)(n + 1) * sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMemcpy(h->p32, tmp, (size_t)(n + 1) * sizeof(int32_t), cudaMemcpyHostToDevice);
        delete[] tmp;
    }
    if (e != cudaSuccess) {
        vrp_instance_destroy(h);
        return cuda_fail(e, "vrp_instance_create");
    }
    h->dev.n = n; h->dev.m = m; h->dev.k = k; h->dev.W = n + 1;
    h->dev.d = h->d; h->dev.d32 = h->d32; h->dev.d32t = h->d32t; h->dev.p = h->p; h->dev.p32 = h->p32;
    h->dev.integral = integral ? 1 : 0;
    *out = h;
    return 0;
}

int vrp_instance_destroy(vrp_instance_t h) {
    if (!h) return 0;
    if (h->d) cudaFree(h->d);
    if (h->d32) cudaFree(h->d32);
    if (h->d32t) cudaFree(h->d32t);
    if (h->p) cudaFree(h->p);
    if (h->p32) cudaFree(h->p32);
    delete h;
    return 0;
}

int vrp_instance_info(vrp_instance_t h, int32_t *n, int32_t *m, int32_t *k, int32_t *integral) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (n) *n = h->dev.n;
    if (m) *m = h->dev.m;
    if (k) *k = h->dev.k;
    if (integral) *integral = h->dev.integral;
    return 0;
}

int vrp_makespan_batch(vrp_instance_t h, const void *ops, int32_t op_bytes, int64_t op_stride,
                       const int32_t *lens, int64_t N, int32_t mode, double *z, int32_t *status,
                       double *returns, int32_t *bottleneck, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0 || (N > 0 && (!ops || !lens || !z || !status)))
        return fail(VRP_EINVAL, "vrp_makespan_batch: null buffer%s");
    if (op_bytes != 2 && op_bytes != 4) return fail(VRP_EINVAL, "op_bytes must be 2 or 4%s");
    if (mode < 0 || mode > 2) return fail(VRP_EINVAL, "unknown mode%s");
    if (N == 0) return 0;
    int rc = launch_makespan(h->dev, ops, op_bytes, op_stride, lens, N, mode, false, z, status,
                             returns, bottleneck, nullptr, nullptr, nullptr,
                             static_cast<cudaStream_t>(stream), h->sm_count);
    return launch_result(rc, "vrp_makespan_batch");
}

int vrp_evaluate_records(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                         int64_t N, double *z, int32_t *status, double *returns, double *arrival,
                         double *time, int32_t *q0, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0 || (N > 0 && (!ops || !lens || !z || !status || !arrival || !time)))
        return fail(VRP_EINVAL, "vrp_evaluate_records: null buffer%s");
    if (N == 0) return 0;
    int rc = launch_makespan(h->dev, ops, 4, op_stride, lens, N, 1, true, z, status, returns,
                             nullptr, arrival, time, q0, static_cast<cudaStream_t>(stream), h->sm_count);
    return launch_result(rc, "vrp_evaluate_records");
}

int vrp_decode_batch(vrp_instance_t h, const double *genes, int64_t gene_stride, int64_t N,
                     int32_t relax, double penalty, double *fitness, double *makespan,
                     int32_t *scheduled, int64_t *visits, void *ops_out, int32_t op_bytes,
                     int64_t out_stride, int32_t *lens_out, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0 || (N > 0 && (!genes || !fitness))) return fail(VRP_EINVAL, "vrp_decode_batch: null buffer%s");
    if (ops_out && op_bytes != 2 && op_bytes != 4) return fail(VRP_EINVAL, "op_bytes must be 2 or 4%s");
    if (ops_out && out_stride < 2 * (int64_t)h->dev.n) return fail(VRP_EINVAL, "out_stride < 2n%s");
    if (gene_stride < 4 * (int64_t)h->dev.n) return fail(VRP_EINVAL, "gene_stride < 4n%s");
    if (N == 0) return 0;
    int rc = launch_decode(h->dev, genes, gene_stride, N, relax, penalty, fitness, makespan, scheduled,
                           visits, ops_out, ops_out ? op_bytes : 4, out_stride, lens_out,
                           static_cast<cudaStream_t>(stream), h->sm_count);
    return launch_result(rc, "vrp_decode_batch");
}

int vrp_fitness_order(const double *fitness, int64_t N, int32_t *order, void *stream) {
    if (N < 0 || (N > 0 && (!fitness || !order))) return fail(VRP_EINVAL, "vrp_fitness_order: null buffer%s");
    if (N > 0x7fffffff) return fail(VRP_EUNSUPPORTED, "population too large%s");
    return launch_result(launch_fitness_order(fitness, N, order, static_cast<cudaStream_t>(stream)),
                         "vrp_fitness_order");
}

int vrp_evolve(const double *pop, const double *fitness, int64_t N, int64_t genes,
               double elite_fraction, double mutant_fraction, double elite_bias,
               vrp_philox *state, double *pop_out, int32_t *order_out,
               double *elite_fitness_out, void *stream) {
    if (!pop || !fitness || !state || !pop_out || !order_out || N < 1 || genes < 1)
        return fail(VRP_EINVAL, "vrp_evolve: bad argument%s");
    if (N > 0x7fffffff) return fail(VRP_EUNSUPPORTED, "population too large%s");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int rc = launch_evolve(pop, fitness, N, genes, elite_fraction, mutant_fraction, elite_bias,
                                 state, pop_out, order_out, elite_fitness_out,
                                 static_cast<cudaStream_t>(stream), sms);
    if (rc == -3) return fail(VRP_EINVAL, "PopulationTooSmall: population %s cannot sustain elites", "");
    return launch_result(rc, "vrp_evolve");
}

int vrp_best_update(const double *fitness, int64_t lo, int64_t hi, const double *genes,
                    int64_t genes_per_row, double *best_fitness, double *best_genes,
                    int64_t *best_index, double *trace_slot, void *stream) {
    if (!fitness || !best_fitness || !best_index || lo < 0 || hi < lo)
        return fail(VRP_EINVAL, "vrp_best_update: bad argument%s");
    return launch_result(launch_best_update(fitness, lo, hi, genes, genes_per_row, best_fitness,
                                            best_genes, best_index, trace_slot,
                                            static_cast<cudaStream_t>(stream)),
                         "vrp_best_update");
}

int vrp_repair_batch(vrp_instance_t h, const int32_t *partial_ops, int64_t partial_stride,
                     const int32_t *partial_lens, const int32_t *removed, int64_t removed_stride,
                     const int32_t *nremoved, const int32_t *regret_k, vrp_philox *states,
                     int32_t *out_ops, int64_t out_stride, int32_t *out_lens, int32_t *status,
                     int64_t N, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0 || (N > 0 && (!partial_ops || !partial_lens || !removed || !nremoved || !regret_k ||
                            !out_ops || !out_lens || !status)))
        return fail(VRP_EINVAL, "vrp_repair_batch: null buffer%s");
    if (out_stride < 2 * (int64_t)h->dev.n) return fail(VRP_EINVAL, "out_stride < 2n%s");
    if (N == 0) return 0;
    return launch_result(launch_repair(h->dev, partial_ops, partial_stride, partial_lens, removed,
                                       removed_stride, nremoved, regret_k, states, out_ops, out_stride,
                                       out_lens, status, N, static_cast<cudaStream_t>(stream)),
                         "vrp_repair_batch");
}

int vrp_alns_iterate(vrp_instance_t h, const vrp_alns_params *params, vrp_alns_worker *workers,
                     int32_t nw, int32_t *cur_ops, int32_t *cur_lens, int32_t *best_ops,
                     int32_t *best_lens, const int32_t *q_draws, int64_t q_stride, int64_t it_begin,
                     int64_t it_end, int32_t *trace_it, double *trace_z, int64_t trace_cap,
                     int32_t *rows_it, double *rows_val, int64_t rows_cap, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (!params) return fail(VRP_EINVAL, "vrp_alns_iterate: null params%s");
    if (nw < 0 || it_begin < 1) return fail(VRP_EINVAL, "vrp_alns_iterate: bad worker count / iteration%s");
    if (nw == 0 || it_end < it_begin) return 0;
    if (!workers || !cur_ops || !cur_lens || !best_ops || !best_lens || !q_draws || !trace_it ||
        !trace_z || !rows_it || !rows_val)
        return fail(VRP_EINVAL, "vrp_alns_iterate: null buffer%s");
    if (q_stride < it_end) return fail(VRP_EINVAL, "vrp_alns_iterate: q_stride < it_end%s");
    if (params->weight_interval < 1) return fail(VRP_EINVAL, "vrp_alns_iterate: weight_interval < 1%s");
    return launch_result(launch_alns(h->dev, *params, workers, nw, cur_ops, cur_lens, best_ops, best_lens,
                                     q_draws, q_stride, it_begin, it_end, trace_it, trace_z, trace_cap,
                                     rows_it, rows_val, rows_cap, static_cast<cudaStream_t>(stream)),
                         "vrp_alns_iterate");
}

int vrp_destroy_batch(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                      const int32_t *opcode, const int32_t *q, int32_t q_min, vrp_philox *states,
                      int32_t *out_ops, int64_t out_stride, int32_t *out_lens, int32_t *removed,
                      int64_t removed_stride, int32_t *nremoved, int64_t N, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0) return fail(VRP_EINVAL, "vrp_destroy_batch: N < 0%s");
    if (N == 0) return 0;
    if (!ops || !lens || !opcode || !q || !states || !out_ops || !out_lens || !removed || !nremoved)
        return fail(VRP_EINVAL, "vrp_destroy_batch: null buffer%s");
    const int64_t n = h->dev.n;
    if (op_stride < 2 * n || out_stride < 2 * n || removed_stride < n)
        return fail(VRP_EINVAL, "vrp_destroy_batch: stride too small%s");
    return launch_result(launch_destroy(h->dev, ops, op_stride, lens, opcode, q, q_min, states, out_ops,
                                        out_stride, out_lens, removed, removed_stride, nremoved, N,
                                        static_cast<cudaStream_t>(stream)),
                         "vrp_destroy_batch");
}

int vrp_remove_batch(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                     const int32_t *picked, int64_t picked_stride, const int32_t *npicked, int32_t *out_ops,
                     int64_t out_stride, int32_t *out_lens, int32_t *removed, int64_t removed_stride,
                     int32_t *nremoved, int64_t N, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0) return fail(VRP_EINVAL, "vrp_remove_batch: N < 0%s");
    if (N == 0) return 0;
    if (!ops || !lens || !picked || !npicked || !out_ops || !out_lens || !removed || !nremoved)
        return fail(VRP_EINVAL, "vrp_remove_batch: null buffer%s");
    const int64_t n = h->dev.n;
    if (op_stride < 2 * n || out_stride < 2 * n || removed_stride < n || picked_stride < 0)
        return fail(VRP_EINVAL, "vrp_remove_batch: stride too small%s");
    return launch_result(launch_destroy(h->dev, ops, op_stride, lens, nullptr, nullptr, 0, nullptr, out_ops,
                                        out_stride, out_lens, removed, removed_stride, nremoved, N,
                                        static_cast<cudaStream_t>(stream), picked, picked_stride, npicked),
                         "vrp_remove_batch");
}

int vrp_removal_gains(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                      double *gains, int64_t gains_stride, int64_t N, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (N < 0) return fail(VRP_EINVAL, "vrp_removal_gains: N < 0%s");
    if (N == 0) return 0;
    if (!ops || !lens || !gains) return fail(VRP_EINVAL, "vrp_removal_gains: null buffer%s");
    if (op_stride < 2 * (int64_t)h->dev.n || gains_stride < (int64_t)h->dev.n + 1)
        return fail(VRP_EINVAL, "vrp_removal_gains: stride too small%s");
    return launch_result(launch_gains(h->dev, ops, op_stride, lens, gains, gains_stride, N,
                                      static_cast<cudaStream_t>(stream)),
                         "vrp_removal_gains");
}

int vrp_sa_exp(const double *x, double *y, int64_t n, void *stream) {
    if (n < 0) return fail(VRP_EINVAL, "vrp_sa_exp: n < 0%s");
    if (n && (!x || !y)) return fail(VRP_EINVAL, "vrp_sa_exp: null buffer%s");
    return launch_result(launch_sa_exp(x, y, n, static_cast<cudaStream_t>(stream)), "vrp_sa_exp");
}

int vrp_ls_build(vrp_instance_t h, int32_t kind, const int32_t *base_ops, const int32_t *base_lens,
                 const int32_t *entries, const int64_t *entry_start, int64_t n_entries,
                 const int64_t *index_list, int64_t first, int64_t count, void *out_ops,
                 int32_t op_bytes, int32_t *out_lens, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (kind < 0 || kind > 3) return fail(VRP_EINVAL, "vrp_ls_build: kind must lie in 0..3%s");
    if (op_bytes != 2 && op_bytes != 4) return fail(VRP_EINVAL, "vrp_ls_build: op_bytes must be 2 or 4%s");
    if (count < 0 || n_entries < 0) return fail(VRP_EINVAL, "vrp_ls_build: negative count%s");
    if (count == 0) return 0;
    if (!base_ops || !base_lens || !entries || !out_ops || !out_lens || (kind != 0 && !entry_start) ||
        n_entries == 0)
        return fail(VRP_EINVAL, "vrp_ls_build: null buffer%s");
    if (op_bytes == 2 && 2 * (int64_t)h->dev.n > 32767)
        return fail(VRP_EUNSUPPORTED, "vrp_ls_build: int16 ops need 2n <= 32767%s");
    return launch_result(launch_ls_build(kind, h->dev.n, h->dev.m, base_ops, base_lens, entries, entry_start,
                                         n_entries, index_list, first, count, out_ops, op_bytes, out_lens,
                                         static_cast<cudaStream_t>(stream)),
                         "vrp_ls_build");
}

int vrp_ls_entries(vrp_instance_t h, int32_t kind, const int32_t *base_ops, const int32_t *base_lens,
                   const double *z, const double *returns, const uint8_t *active, int32_t W,
                   const int64_t *entry_off, const int64_t *cand_off, int32_t *entry_count, int64_t *cand_count,
                   int32_t *entries, int64_t *entry_start, void *stream) {
    if (!h) return fail(VRP_EINVAL, "null instance%s");
    DeviceGuard dg(h->device);
    if (kind != 0 && kind != 1) return fail(VRP_EINVAL, "vrp_ls_entries: kind must be 0 or 1%s");
    if (W < 0) return fail(VRP_EINVAL, "vrp_ls_entries: W < 0%s");
    if (W == 0) return 0;
    if (!base_ops || !base_lens || !z || !returns || !active)
        return fail(VRP_EINVAL, "vrp_ls_entries: null buffer%s");
    if ((entry_off == nullptr) != (cand_off == nullptr) ||
        (entry_off ? (!entries || !entry_start) : (!entry_count || !cand_count)))
        return fail(VRP_EINVAL, "vrp_ls_entries: count phase needs entry_count/cand_count, fill phase "
                                "entry_off/cand_off/entries/entry_start%s");
    if (kind == 1 && 8 * ((int64_t)h->dev.n + 1) > 227 * 1024)
        return fail(VRP_EUNSUPPORTED, "vrp_ls_entries: cross entries need 8 (n + 1) bytes of shared memory%s");
    return launch_result(launch_ls_entries(kind, h->dev.n, h->dev.m, base_ops, base_lens, z, returns, active, W,
                                           entry_off, cand_off, entry_count, cand_count, entries, entry_start,
                                           static_cast<cudaStream_t>(stream)),
                         "vrp_ls_entries");
}

int vrp_ls_topk(const double *z, const int32_t *status, int64_t first, const double *zthr,
                const int32_t *seg_worker, const int64_t *seg_begin, const int64_t *seg_end, int64_t nseg,
                const int32_t *workers, const int32_t *wseg_first, const int32_t *wseg_count, int32_t nworkers,
                int32_t K, double *top_z, int64_t *top_i, int32_t *top_n, void *stream) {
    if (nseg < 0 || nworkers < 0) return fail(VRP_EINVAL, "vrp_ls_topk: negative count%s");
    if (K < 1 || K > 16) return fail(VRP_EINVAL, "vrp_ls_topk: K must lie in 1..16%s");
    if (nseg == 0 || nworkers == 0) return 0;
    if (!z || !status || !zthr || !seg_worker || !seg_begin || !seg_end || !workers || !wseg_first || !wseg_count ||
        !top_z || !top_i || !top_n)
        return fail(VRP_EINVAL, "vrp_ls_topk: null buffer%s");
    return launch_result(launch_ls_topk(z, status, first, zthr, seg_worker, seg_begin, seg_end, nseg, workers,
                                        wseg_first, wseg_count, nworkers, K, top_z, top_i, top_n,
                                        static_cast<cudaStream_t>(stream)),
                         "vrp_ls_topk");
}

int vrp_random_fill(vrp_philox *state, int64_t count, double *out, void *stream) {
    if (count < 0) return fail(VRP_EINVAL, "vrp_random_fill: count < 0%s");
    if (count == 0) return 0;
    if (!state || !out) return fail(VRP_EINVAL, "vrp_random_fill: null buffer%s");
    return launch_result(launch_random_fill(state, count, out, static_cast<cudaStream_t>(stream)),
                         "vrp_random_fill");
}

}  // extern "C"
