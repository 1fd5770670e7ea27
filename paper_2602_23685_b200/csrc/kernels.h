// kernels.h -- host-side launchers implemented by the kernel translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vrp_rpd.h"
#include "common.cuh"

// makespan.cu (K1/K2); mode 0 exact, 1 evaluate, 2 two-pass; rec = event records
int launch_makespan(const DevInstance &I, const void *ops, int op_bytes, int64_t stride,
                    const int32_t *lens, int64_t N, int mode, bool rec, double *z, int32_t *status,
                    double *returns, int32_t *bottleneck, double *arrival, double *timev,
                    int32_t *q0, cudaStream_t stream, int sm_count);

// decode.cu (K3)
int launch_decode(const DevInstance &I, const double *genes, int64_t gstride, int64_t N, int relax,
                  double penalty, double *fitness, double *makespan, int32_t *scheduled,
                  int64_t *visits, void *ops_out, int op_bytes, int64_t ostride,
                  int32_t *lens_out, cudaStream_t stream, int sm_count);

// evolve.cu (K4)
int launch_fitness_order(const double *fit, int64_t N, int32_t *order, cudaStream_t stream);
int launch_evolve(const double *pop, const double *fit, int64_t N, int64_t G, double elite_frac,
                  double mutant_frac, double bias, vrp_philox *state, double *out, int32_t *order,
                  double *elite_fit, cudaStream_t stream, int sm_count);
int launch_best_update(const double *fit, int64_t lo, int64_t hi, const double *genes, int64_t G,
                       double *best_fit, double *best_genes, int64_t *best_index, double *trace,
                       cudaStream_t stream);

int launch_random_fill(vrp_philox *state, int64_t count, double *out, cudaStream_t stream);

// repair.cu (K5)
size_t repair_scratch_bytes(int n, int m);
int launch_repair(const DevInstance &I, const int32_t *pops, int64_t pstride, const int32_t *plens,
                  const int32_t *removed, int64_t rstride, const int32_t *nremoved,
                  const int32_t *regret_k, vrp_philox *states, int32_t *out_ops, int64_t ostride,
                  int32_t *out_lens, int32_t *status, int64_t N, cudaStream_t stream);

// alns_step.cu (K6 + device ALNS iterations)
size_t alns_scratch_bytes(int n, int m);
int launch_alns(const DevInstance &I, const vrp_alns_params &P, vrp_alns_worker *workers, int32_t nw,
                int32_t *cur_ops, int32_t *cur_lens, int32_t *best_ops, int32_t *best_lens,
                const int32_t *q_draws, int64_t q_stride, int64_t it_begin, int64_t it_end,
                int32_t *trace_it, double *trace_z, int64_t trace_cap, int32_t *rows_it,
                double *rows_val, int64_t rows_cap, cudaStream_t stream);
int launch_destroy(const DevInstance &I, const int32_t *ops, int64_t stride, const int32_t *lens,
                   const int32_t *opcode, const int32_t *q, int32_t q_min, vrp_philox *states,
                   int32_t *out_ops, int64_t ostride, int32_t *out_lens, int32_t *removed,
                   int64_t rstride, int32_t *nremoved, int64_t N, cudaStream_t stream,
                   const int32_t *picked = nullptr, int64_t pstride = 0, const int32_t *npicked = nullptr);
int launch_gains(const DevInstance &I, const int32_t *ops, int64_t stride, const int32_t *lens, double *gains,
                 int64_t gstride, int64_t N, cudaStream_t stream);

int launch_sa_exp(const double *x, double *y, int64_t n, cudaStream_t stream);

// ls.cu (batched local-search candidate builder)
int launch_ls_build(int kind, int n, int m, const int32_t *base_ops, const int32_t *base_lens,
                    const int32_t *entries, const int64_t *entry_start, int64_t n_entries,
                    const int64_t *index_list, int64_t first, int64_t count, void *out_ops, int op_bytes,
                    int32_t *out_lens, cudaStream_t stream);
int launch_ls_entries(int kind, int n, int m, const int32_t *base_ops, const int32_t *base_lens, const double *z,
                      const double *returns, const uint8_t *active, int32_t W, const int64_t *entry_off,
                      const int64_t *cand_off, int32_t *entry_count, int64_t *cand_count, int32_t *entries,
                      int64_t *entry_start, cudaStream_t stream);
int launch_ls_topk(const double *z, const int32_t *status, int64_t first, const double *zthr,
                   const int32_t *seg_worker, const int64_t *seg_begin, const int64_t *seg_end, int64_t nseg,
                   const int32_t *workers, const int32_t *wseg_first, const int32_t *wseg_count, int32_t nworkers,
                   int32_t K, double *top_z, int64_t *top_i, int32_t *top_n, cudaStream_t stream);
