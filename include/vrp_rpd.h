/*
 * vrp_rpd.h -- C-ABI of the B200-native VRP-RPD candidate-scoring library
 * (libvrprpd.so, built from paper_2602_23685_b200/csrc/ for sm_100a).
 *
 * The reference (arxiv 2602.23685, /root/reference/pkg/src/vrp_rpd/) is pure
 * Python with no FFI of its own; these entry points are what its hot-path
 * functions would bind (ctypes stub in INTEGRATION.md).  Each export names the
 * reference function it replaces.
 *
 * Conventions
 *  - Every call returns an int error code: 0 = OK, VRP_EINVAL, VRP_ECUDA,
 *    VRP_EUNSUPPORTED.  vrp_last_error() gives a message.  No C++ exception
 *    crosses the ABI.
 *  - Per-candidate outcomes are status codes, replacing the reference's
 *    exceptions: VRP_OK, VRP_CAPACITY (CapacityViolation), VRP_DEADLOCK
 *    (Deadlock), VRP_MALFORMED (MalformedSolution)  (schedule.py:32-45).
 *  - Batch buffers (ops, lens, genes, outputs) are DEVICE pointers owned by the
 *    caller; `stream` is a cudaStream_t (NULL = legacy default stream).  Calls
 *    are asynchronous on that stream.
 *  - Ops: op code = 2*(customer-1) + kind, kind 0 = dropoff, 1 = pickup
 *    (brkga.py:73-75 op_index).  One candidate = its m routes concatenated
 *    vehicle-major; row i starts at ops + i*op_stride elements; lens[i*m + v]
 *    is route v's length.  op_bytes selects int16 (2) or int32 (4) codes.
 *  - Times are fp64 and follow the reference's operation order, so results
 *    are bit-identical to the reference for any input, integer or not.
 */
#ifndef VRP_RPD_H
#define VRP_RPD_H
#include <stdint.h>

#define VRP_MAX_N 8192  /* largest instance (customers) every kernel supports */

#ifdef __cplusplus
extern "C" {
#endif

#define VRP_EINVAL 1
#define VRP_ECUDA 2
#define VRP_EUNSUPPORTED 3

#define VRP_OK 0
#define VRP_CAPACITY 1
#define VRP_DEADLOCK 2
#define VRP_MALFORMED 3

/* makespan modes */
#define VRP_MODE_EXACT 0    /* schedule.exact_makespan  (schedule.py:265-316) */
#define VRP_MODE_EVALUATE 1 /* schedule.evaluate        (schedule.py:188-257), validating */
#define VRP_MODE_TWO_PASS 2 /* schedule.two_pass_estimate (schedule.py:345-393) */

typedef struct vrp_instance *vrp_instance_t;

/* numpy.random.Philox bit-generator state, field for field
 * (Generator(Philox).bit_generator.state: counter, key, buffer, buffer_pos,
 * has_uint32, uinteger).  Device-resident when passed to vrp_evolve. */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buffer[4];
    int32_t buffer_pos;
    int32_t has_uint32;
    uint32_t uinteger;
    uint32_t reserved;
} vrp_philox;

/* Library / device info.  Returns the compiled arch (e.g. 1000 for sm_100a). */
int vrp_version(int32_t *abi_version, int32_t *compiled_arch);
const char *vrp_last_error(void);

/* Upload an instance (instance.py:82-156 Instance): host d[(n+1)*(n+1)], p[n+1].
 * The handle owns the device copies; d is also kept as int32 when every entry
 * is an integer in [0, 2^31) (all TSPLIB distance types), which halves the
 * L2 footprint of the gathers.  Requires 1 <= m <= 32, 1 <= n <= VRP_MAX_N (8192: the
 * tightest per-kernel shared-memory bound, K3's bitonic argsort fallback). */
int vrp_instance_create(int32_t n, int32_t m, int32_t k, const double *d_host,
                        const double *p_host, vrp_instance_t *out);
int vrp_instance_destroy(vrp_instance_t h);
int vrp_instance_info(vrp_instance_t h, int32_t *n, int32_t *m, int32_t *k, int32_t *integral);

/* K1/K2: score N candidates.  mode = VRP_MODE_*.
 * Replaces schedule.exact_makespan / evaluate / two_pass_estimate.
 *   z[N]            makespan (0 where status != OK)
 *   status[N]       VRP_OK / CAPACITY / DEADLOCK / MALFORMED
 *   returns[N*m]    per-vehicle depot return (nullable)      (Schedule.returns)
 *   bottleneck[N]   first argmax of returns (nullable)       (Schedule.bottleneck, schedule.py:105-110) */
int vrp_makespan_batch(vrp_instance_t h, const void *ops, int32_t op_bytes, int64_t op_stride,
                       const int32_t *lens, int64_t N, int32_t mode, double *z, int32_t *status,
                       double *returns, int32_t *bottleneck, void *stream);

/* Full event records for evaluate (schedule.py:188-257): per op (same layout as
 * ops) the arrival and execution time, per vehicle the minimal initial load
 * (route_initial_load, schedule.py:159-185).  Validating (MODE_EVALUATE).
 * Records are defined for candidates with status VRP_OK (every op executed),
 * as the reference's Schedule exists only for those. */
int vrp_evaluate_records(vrp_instance_t h, const int32_t *ops, int64_t op_stride,
                         const int32_t *lens, int64_t N, double *z, int32_t *status,
                         double *returns, double *arrival, double *time, int32_t *q0,
                         void *stream);

/* K3: BRKGA decode (brkga.py:92-207) of N chromosomes genes[N][gene_stride]
 * (4n fp64: priorities then hints).  relax = wait_relaxation, penalty =
 * infeasibility_penalty.  Outputs: fitness/makespan[N], scheduled[N] (ops
 * placed), visits[N] (op_visits), and the decoded solution as ops_out (op_bytes
 * 2|4, row stride out_stride, vehicle-major, unscheduled tail = -1) + lens_out[N*m].
 * ops_out/lens_out may be NULL when only fitness is needed. */
int vrp_decode_batch(vrp_instance_t h, const double *genes, int64_t gene_stride, int64_t N,
                     int32_t relax, double penalty, double *fitness, double *makespan,
                     int32_t *scheduled, int64_t *visits, void *ops_out, int32_t op_bytes,
                     int64_t out_stride, int32_t *lens_out, void *stream);

/* K4: stable argsort of a fitness vector (numpy argsort kind="stable",
 * brkga.py:243/:456): order[N] int32 (device). */
int vrp_fitness_order(const double *fitness, int64_t N, int32_t *order, void *stream);

/* K4: one BRKGA generation, brkga.evolve (brkga.py:231-252), fully on device.
 * pop[N][genes] and fitness[N] in; pop_out[N][genes] = [elites | mutants |
 * offspring]; order_out[N] = the stable fitness order; elite_fitness_out
 * (nullable) = fitness of the elites in order (run_brkga :456-460).  `state`
 * is a DEVICE pointer to the generator; it is advanced exactly as numpy's
 * Generator(Philox) would be by mutants = random((n_mutant, genes)),
 * e_idx = integers(n_elite, n_off), o_idx = integers(N - n_elite, n_off),
 * mask = random((n_off, genes)) < elite_bias.  Returns VRP_EINVAL for
 * PopulationTooSmall (n_elite < 1 or N - n_elite < 1). */
int vrp_evolve(const double *pop, const double *fitness, int64_t N, int64_t genes,
               double elite_fraction, double mutant_fraction, double elite_bias,
               vrp_philox *state, double *pop_out, int32_t *order_out,
               double *elite_fitness_out, void *stream);

/* run_brkga best tracking (brkga.py:446-467): the first index of the minimum
 * of fitness[lo, hi) replaces the incumbent when strictly better (or when
 * *best_index < 0); its chromosome (row of genes[., genes_per_row]) is copied
 * to best_genes; *trace_slot (nullable) receives the incumbent fitness. */
int vrp_best_update(const double *fitness, int64_t lo, int64_t hi, const double *genes,
                    int64_t genes_per_row, double *best_fitness, double *best_genes,
                    int64_t *best_index, double *trace_slot, void *stream);

/* Generator.random(count) on the device: out[i] = the i-th (next64 >> 11) *
 * 2^-53 draw of the numpy Philox stream in *state (DEVICE), which is then
 * advanced past the count draws -- bit-identical to rng.random(count) for the
 * BRKGA populations (brkga.py:436-437 random init, :418 warm-start fill). */
int vrp_random_fill(vrp_philox *state, int64_t count, double *out, void *stream);

/* K5: ALNS repair, insertion.reinsert_all (insertion.py:484-516) on a fresh
 * InsertionContext of each partial solution, N independent instances.
 *   partial_ops[N][partial_stride] int32 + partial_lens[N][m]   (vehicle-major)
 *   removed[N][removed_stride] int32 customers, nremoved[N]       (any order)
 *   regret_k[N]: 0 = greedy, k >= 2 = regret-k (alns.py:258/:266)
 *   states[N]: per-instance numpy-Philox generators (DEVICE), advanced exactly
 *              as the reference's rng; NULL = deterministic (rng=None)
 *   out_ops[N][out_stride] (-1 padded), out_lens[N][m]
 *   status[N]: 0 OK, 1 RepairFailed (some customer has no insertion), 2 malformed input
 * The repaired solution is NOT re-scored here (the reference's _repair_scored,
 * alns.py:261-274, follows with exact_makespan: use vrp_makespan_batch). */
int vrp_repair_batch(vrp_instance_t h, const int32_t *partial_ops, int64_t partial_stride,
                     const int32_t *partial_lens, const int32_t *removed, int64_t removed_stride,
                     const int32_t *nremoved, const int32_t *regret_k, vrp_philox *states,
                     int32_t *out_ops, int64_t out_stride, int32_t *out_lens, int32_t *status,
                     int64_t N, void *stream);

/* K6: alns.destroy (alns.py:182-251) followed by insertion.remove_customers
 * (insertion.py:379-397, capacity cascade included) on N solutions.
 *   ops[N][op_stride] + lens[N][m]  complete solutions (vehicle-major, DEVICE)
 *   opcode[N]: 0 random, 1 worst, 2 shaw, 3 cluster, 4 route, 5 critical_path
 *   q[N] (clamped to n), q_min = removal_bounds(n)[0]
 *   states[N]: per-solution generators (DEVICE), advanced like the reference's rng
 *   out_ops[N][out_stride] (-1 padded) + out_lens[N][m]: the partial solutions
 *   removed[N][removed_stride] (>= n) sorted removed customers, nremoved[N] */
int vrp_destroy_batch(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                      const int32_t *opcode, const int32_t *q, int32_t q_min, vrp_philox *states,
                      int32_t *out_ops, int64_t out_stride, int32_t *out_lens, int32_t *removed,
                      int64_t removed_stride, int32_t *nremoved, int64_t N, void *stream);

/* insertion.remove_customers (insertion.py:379-397) alone, on N solutions:
 * both ops of the picked customers (picked[N][picked_stride], npicked[N]) are
 * removed and the capacity cascade runs; outputs as vrp_destroy_batch. */
int vrp_remove_batch(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                     const int32_t *picked, int64_t picked_stride, const int32_t *npicked,
                     int32_t *out_ops, int64_t out_stride, int32_t *out_lens, int32_t *removed,
                     int64_t removed_stride, int32_t *nremoved, int64_t N, void *stream);

/* insertion.removal_gains (insertion.py:538-569): the makespan reduction of
 * removing each customer under fixed ready times, gains[N][gains_stride]
 * (index c = 1..n; index 0 = 0) for N complete solutions (DEVICE). */
int vrp_removal_gains(vrp_instance_t h, const int32_t *ops, int64_t op_stride, const int32_t *lens,
                      double *gains, int64_t gains_stride, int64_t N, void *stream);

/* Local-search neighbourhoods (alns.py:416-487 pickup_repositioning /
 * cross_agent_relocation; baselines.py:372-455 two_opt_improve) materialised
 * as a candidate batch for
 * vrp_makespan_batch (K2 estimate, K1 verify).  Candidates are numbered in the
 * reference's generation order:
 *   kind 0 (pickup move): entries[e] = {worker, v, i, fi, 0} -- the pickup at
 *     position i of vehicle v (flat index fi of the worker's solution) is
 *     removed and re-inserted at every (w, g) of the reduced solution except
 *     (v, i): 2n + m - 2 candidates per entry, index = e * (2n+m-2) + j
 *   kind 1 (cross move): entries[e] = {worker, c, w, f1, f2} -- customer c
 *     (flat op positions f1 < f2) is stripped and re-inserted as D at gd, P at
 *     gp (0 <= gd < gp <= L_w + 1) on vehicle w: entry_start[e] = first index
 *   kind 2 (2-opt, baselines.py:393-406): entries[e] = {worker, v, 0, 0, 0} --
 *     reverse positions i < j of route v, L_v (L_v - 1) / 2 candidates, i-major
 *   kind 3 (swap, baselines.py:431-443): entries[e] = {worker, 0, 0, 0, 0} --
 *     swap flat ops a < b, 2n (2n - 1) / 2 candidates, a-major
 *   (two_opt_improve's relocation, :408-429, is kind 0 over every op)
 *   base_ops[W][2n], base_lens[W][m]: the workers' solutions (DEVICE)
 *   index_list (nullable): explicit candidate indices; else first .. first+count-1
 *   out_ops[count][2n] (op_bytes 2 or 4), out_lens[count][m] */
int vrp_ls_build(vrp_instance_t h, int32_t kind, const int32_t *base_ops, const int32_t *base_lens,
                 const int32_t *entries, const int64_t *entry_start, int64_t n_entries,
                 const int64_t *index_list, int64_t first, int64_t count, void *out_ops,
                 int32_t op_bytes, int32_t *out_lens, void *stream);

/* The simulated-annealing acceptance threshold exp(x) of alns.py:588
 * (`rng.random() < math.exp(-delta / T)`) as vrp_alns_iterate computes it:
 * fp64 exp rounded correctly (double-double evaluation, csrc/ddexp.cuh).
 * x, y: n DEVICE doubles. */
int vrp_sa_exp(const double *x, double *y, int64_t n, void *stream);

/* The local-search neighbourhood entries of W solutions, built on the device
 * from their evaluate returns (alns.py:416-450 pickup_repositioning, kind 0;
 * :453-487 cross_agent_relocation, kind 1), in the reference's generation
 * order, in the layout vrp_ls_build consumes:
 *   kind 0: solutions with z > 0, vehicles with return >= 0.9 z, each pickup
 *     in route order -> {w, v, i, flat, 0}, 2n + m - 2 candidates each
 *   kind 1: b = first argmax of the returns, customers of route b ascending,
 *     every vehicle u != b -> {w, c, u, f1, f2}, (L+1)(L+2)/2 candidates
 *   base_ops[W][2n], base_lens[W][m], z[W], returns[W][m], active[W] (u8) DEVICE
 * Two calls: count phase (entry_off = cand_off = NULL) writes entry_count[W]
 * and cand_count[W]; the fill phase, given their exclusive prefix sums
 * entry_off[W] / cand_off[W], writes entries[E][5] and entry_start[E]. */
int vrp_ls_entries(vrp_instance_t h, int32_t kind, const int32_t *base_ops, const int32_t *base_lens,
                   const double *z, const double *returns, const uint8_t *active, int32_t W,
                   const int64_t *entry_off, const int64_t *cand_off, int32_t *entry_count, int64_t *cand_count,
                   int32_t *entries, int64_t *entry_start, void *stream);

/* The verification shortlist of the batched local search (alns.py:401-413:
 * stable sort of the survivors by estimate, first _VERIFY_LIMIT), per solution,
 * over a chunk of estimated candidates: candidates with status 0 and
 * z < zthr[worker] are merged into each solution's running list of its K
 * smallest (estimate, generation index) pairs (K <= 16).
 *   z/status[count]            K2 output for candidates first .. first+count-1 (DEVICE)
 *   seg_worker/seg_begin/seg_end[nseg]  host-planned segments of <= 2048
 *                              candidates of one solution each (global indices)
 *   workers/wseg_first/wseg_count[nworkers]  solutions with segments in this
 *                              chunk and their segment ranges
 *   top_z/top_i[W][K], top_n[W] running lists, sorted (DEVICE, in/out) */
int vrp_ls_topk(const double *z, const int32_t *status, int64_t first, const double *zthr,
                const int32_t *seg_worker, const int64_t *seg_begin, const int64_t *seg_end, int64_t nseg,
                const int32_t *workers, const int32_t *wseg_first, const int32_t *wseg_count, int32_t nworkers,
                int32_t K, double *top_z, int64_t *top_i, int32_t *top_n, void *stream);

/* One ALNS worker (alns.py:536-640 run_alns locals), DEVICE-resident.
 * weights/scores/attempts are indexed in the reference's operator order:
 * random, worst, shaw, cluster, route, critical_path, greedy, regret2,
 * regret3, regretm (alns.py:28-29). */
typedef struct {
    vrp_philox rng;           /* the worker's generator (alns.py:541) */
    double z, z_best, temperature, t_init;
    double weights[10], scores[10];
    int64_t attempts[10];
    int64_t stagnation, accepted, rejected, reheats;
    int64_t best_it;          /* iteration of the last z_best improvement */
    int32_t n_trace, n_rows;  /* records written by the last vrp_alns_iterate */
} vrp_alns_worker;

/* AlnsParams (alns.py:42-70) fields the device loop reads. */
typedef struct {
    double t0, alpha, reheat_factor, reaction, sigma1, sigma2, sigma3, min_weight;
    int64_t stagnation_threshold, weight_interval;
    int32_t q_min; /* min(removal_bounds(n)[0], n) (alns.py:102-109, :190) */
    int32_t reserved;
} vrp_alns_params;

/* K6 + device-resident ALNS: iterations it_begin..it_end (1-based, inclusive)
 * of run_alns's loop body (alns.py:566-611: roulette, destroy, repair,
 * exact_makespan, SA acceptance, cooling/reheat, update_weights) for nw
 * independent workers, one warp each.  Host-side steps (local search every
 * pickup_reposition / cross_agent interval, pool share polling) belong at the
 * iteration boundaries the caller chooses.
 *   workers[nw]                      device, in/out
 *   cur_ops/best_ops[nw][2n], cur_lens/best_lens[nw][m]  device, in/out (vehicle-major)
 *   q_draws[nw][q_stride]            device: the worker's pre-drawn q (alns.py:556)
 *   trace_it/trace_z[nw][trace_cap]  out: (iteration, z_best) per improvement
 *   rows_it[nw][rows_cap], rows_val[nw][rows_cap][12]  out: weight rows
 *                                    (z_best, temperature, 10 weights)
 * workers[i].n_trace / n_rows receive the record counts of this call. */
int vrp_alns_iterate(vrp_instance_t h, const vrp_alns_params *params, vrp_alns_worker *workers,
                     int32_t nw, int32_t *cur_ops, int32_t *cur_lens, int32_t *best_ops,
                     int32_t *best_lens, const int32_t *q_draws, int64_t q_stride, int64_t it_begin,
                     int64_t it_end, int32_t *trace_it, double *trace_z, int64_t trace_cap,
                     int32_t *rows_it, double *rows_val, int64_t rows_cap, void *stream);

#ifdef __cplusplus
}
#endif
#endif
