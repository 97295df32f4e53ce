/*
 * teccl_b200.h — C ABI of the B200-native TE-CCL LP engine.
 *
 * The reference (arXiv 2305.13479 artifact, package `collsched`) solves the
 * copy-free time-expanded multi-commodity-flow LP on the CPU:
 *
 *   build_lp_model(t, d, cfg, opts)   pkg/src/collsched/lp.py:22-136
 *   solve(m, opts)  -> scipy HiGHS    pkg/src/collsched/solver.py:86-143
 *   lp_completion_epoch(sol)          pkg/src/collsched/lp.py:139-153
 *   simulate(sched, t, d, opts)       pkg/src/collsched/simulator.py:58-235
 *
 * Each entry point below replaces one of those steps. Every argument is a
 * plain pointer or size; host pointers unless the name says `_dev`. All
 * functions return 0 on success and a nonzero TECCL_E* code on failure;
 * teccl_last_error() then holds a one-line message (thread-local).
 *
 * Variable and row order of a built LP are exactly the reference's
 * (see DESIGN.md "LP layout"), so solution vectors can be handed back to the
 * reference's own post-processing unchanged.
 */
#ifndef TECCL_B200_H
#define TECCL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TECCL_OK 0
#define TECCL_EINVAL 1    /* bad argument / inconsistent description */
#define TECCL_ECUDA 2     /* CUDA runtime failure */
#define TECCL_ENOMEM 3    /* device allocation failed */
#define TECCL_ENODEV 4    /* no usable sm_100 device */

/* solve status (teccl_pdlp_result.status) */
#define TECCL_OPTIMAL 0        /* gap <= eps_rel, residuals <= min(eps_rel, eps_res) */
#define TECCL_ITER_LIMIT 1     /* max_iters reached */
#define TECCL_TIME_LIMIT 2     /* time_limit reached */
#define TECCL_PRIMAL_INFEASIBLE 3  /* Farkas certificate found (see eps_infeas) */
#define TECCL_NUMERICAL 4
#define TECCL_PEER_TIMEOUT 5    /* a peer rank stopped answering (row-partitioned solve) */

typedef struct teccl_ctx teccl_ctx; /* one device + one stream */
typedef struct teccl_lp teccl_lp;   /* device-resident LP: CSR, CSC, bounds, costs */

const char* teccl_last_error(void);
const char* teccl_version(void);

int teccl_ctx_create(int device, teccl_ctx** out);
int teccl_ctx_destroy(teccl_ctx* ctx);
int teccl_ctx_sync(teccl_ctx* ctx);

/* ---------------------------------------------------------------------------
 * (1) Time-expanded constraint-matrix builder.
 * Replaces build_lp_model (pkg/src/collsched/lp.py:22-136): the host passes
 * the compact topology/demand tables (node kinds, edges with delay and
 * per-epoch capacity, sorted sources, sorted (source,dst) pairs); the device
 * emits CSR and CSC directly in HBM, with the reference's variable order,
 * row order, bounds and (minimisation) objective.
 */
typedef struct {
  int32_t num_nodes;            /* all nodes, reference node order */
  int32_t num_edges;            /* reference edge order */
  int32_t num_sources;          /* sources sorted by str() as lp.py:34 */
  int32_t num_pairs;            /* (s,d) pairs sorted as lp.py:60 */
  int32_t K;                    /* epochs 0..K-1 */
  const uint8_t* node_is_switch;  /* [num_nodes] */
  const int32_t* edge_src;        /* [E] node index */
  const int32_t* edge_dst;        /* [E] node index */
  const int32_t* edge_delta;      /* [E] ceil(alpha/tau), epochs.py:58-64 */
  const double* edge_cap;         /* [E*K] chunks/epoch, cap_chunks(), row e*K+k */
  const int32_t* source_node;     /* [S] node index of each source slot */
  const int32_t* pair_source;     /* [P] source slot */
  const int32_t* pair_dst;        /* [P] node index */
  const double* pair_units;       /* [P] demanded chunks of the pair */
  double buffer_limit;            /* < 0: no Appendix-B buffer rows */
  int32_t phase1;                 /* 1: feasibility LP -- maximise sum_p Rc(p,K-1) with
                                     Rc(p,K-1) in [0,u] (feasible iff it reaches sum u) */
} teccl_te_desc;

int teccl_lp_build_te(teccl_ctx* ctx, const teccl_te_desc* desc, teccl_lp** out);

/* Row-partitioned build (north_star: a single LP row-partitioned by epoch
 * block over GPUs). Rank `rank` of `world` builds only its epoch block of the
 * LP in epoch-major numbering: owned rows and
 * columns plus the halo windows its SpMVs gather from. info[16] receives
 * {own_c0, own_c1, own_r0, own_r1, win_c0, win_c1, win_r0, win_r1, k0, k1,
 *  total_cols, total_rows, delta_max, nnz_csr, nnz_csc, cols_per_epoch}. */
int teccl_lp_build_te_part(teccl_ctx* ctx, const teccl_te_desc* desc, int32_t world,
                           int32_t rank, teccl_lp** out, int64_t* info);

/* Peer exchange for a row-partitioned LP (one process per GPU). Each rank
 * exports a blob (CUDA IPC handle of its exchange arena + layout, *blob_len
 * bytes, <= 512), the host all-gathers the blobs in rank order and every
 * rank connects to all of them; teccl_pdlp_solve then runs the partitioned
 * solve on all ranks together, halo vectors and KKT scalars moving through
 * peer memory over NVLink. */
int teccl_dist_export(teccl_ctx* ctx, teccl_lp* lp, uint8_t* blob, int64_t* blob_len);
int teccl_dist_connect(teccl_ctx* ctx, teccl_lp* lp, const uint8_t* blobs, int64_t blob_len);

/* Source-partitioned solve of a WHOLE LP from teccl_lp_build_te (every rank
 * holds it; setup is the single-device one, redundant on every rank). Rank
 * `rank` of `world` updates the columns of sources [s0, s1) and of their
 * pairs and the init / conservation / cumulative rows of those; the capacity
 * (and buffer-limit) rows couple the sources: every iteration each rank
 * stores its partial row sums into every rank's buffer over peer memory and
 * all ranks take those rows' dual step identically. No reference
 * counterpart (new). info8 = {s0, s1, p0, p1, c0, c1, q0, q1}: own sources,
 * pairs, flow+buffer columns [c0, c1) and Rd/Rc columns [q0, q1). Then
 * export / all-gather / connect the blobs (rank order) as for
 * teccl_dist_*, and call teccl_pdlp_solve; x/y come back whole, valid on
 * this rank's columns / rows. */
int teccl_src_setup(teccl_ctx* ctx, teccl_lp* lp, int32_t world, int32_t rank, int64_t* info8);
int teccl_src_export(teccl_ctx* ctx, teccl_lp* lp, uint8_t* blob, int64_t* blob_len);
int teccl_src_connect(teccl_ctx* ctx, teccl_lp* lp, const uint8_t* blobs, int64_t blob_len);

/* Generic LP upload (minimise obj.x s.t. row_lo <= A x <= row_hi,
 * var_lb <= x <= var_ub; +-INFINITY allowed). Replaces the matrix assembly of
 * collsched.solver.solve (solver.py:100-121) for any Model the reference
 * builds. row_ptr has m+1 entries; columns need not be sorted. */
int teccl_lp_from_csr(teccl_ctx* ctx, int32_t m, int32_t n, int64_t nnz,
                      const int64_t* row_ptr, const int32_t* col, const double* val,
                      const double* row_lo, const double* row_hi,
                      const double* var_lb, const double* var_ub, const double* obj,
                      teccl_lp** out);

int teccl_lp_dims(const teccl_lp* lp, int32_t* m, int32_t* n, int64_t* nnz);
/* Copy the built LP back to the host (CSR, columns ascending in each row).
 * Any output pointer may be NULL. val gets explicit coefficients. */
int teccl_lp_export(const teccl_lp* lp, int64_t* row_ptr, int32_t* col, double* val,
                    double* row_lo, double* row_hi, double* var_lb, double* var_ub,
                    double* obj);
/* Copy the CSC (rows ascending in each column) back to the host. */
int teccl_lp_export_csc(const teccl_lp* lp, int64_t* col_ptr, int32_t* row, double* val);
int teccl_lp_destroy(teccl_lp* lp);

/* ---------------------------------------------------------------------------
 * (2)+(3) Restarted Halpern primal-dual hybrid gradient (PDLP family).
 * Replaces the HiGHS call in collsched.solver.solve (solver.py:128-143) for
 * LPs. Termination: relative duality gap <= eps_rel and relative primal and
 * dual residuals <= min(eps_rel, eps_res) (definitions in DESIGN.md); primal
 * infeasibility is certified on the device (eps_infeas) and reported as
 * TECCL_PRIMAL_INFEASIBLE, the reference's "infeasible" (solver.py:133-134).
 */
typedef struct {
  double eps_rel;          /* e.g. 1e-4 */
  int64_t max_iters;       /* hard iteration cap */
  double time_limit;       /* seconds */
  int32_t check_every;     /* iterations between restart/termination checks (64) */
  int32_t ruiz_iters;      /* Ruiz equilibration passes (10) */
  int32_t lookahead;       /* chunks queued ahead of the host poll (4) */
  int32_t verbose;         /* print progress to stderr every N checks (0 = quiet) */
  double reflection;       /* Halpern reflection coefficient in [0,1] (1.0) */
  int32_t use_graphs;      /* 1: replay each chunk from a CUDA graph */
  int32_t warm_start;      /* 1: start from x_inout / y_inout */
  double restart_sufficient;  /* restart when r <= this * r0 (0.3) */
  double restart_necessary;   /* ... or r <= this * r0 and r grew (0.9) */
  double restart_artificial;  /* ... or inner iterations >= this * total (0.36) */
  double omega_theta;         /* primal-weight proportional gain at restarts, 0..1 (0.6) */
  double omega_scale;         /* multiplies the initial primal weight (1.0) */
  double omega_ki;            /* integral gain of the primal-weight PID (0) */
  double omega_kd;            /* derivative gain of the primal-weight PID (0) */
  int32_t col_pipeline;       /* 1: software-pipelined column half-step kernel (1) */
  int32_t matrix_free;        /* LPs from teccl_lp_build_te apply A / A^T from the
                                 topology tables instead of the stored matrix:
                                 0 off, 1 auto (stored matrix below 3M columns, where
                                 the iteration is L2-resident; mode 4 above), 2 one
                                 thread per entry, 3 segment kernels, 4 per-entry
                                 columns + segment rows (1). Blocks of row-partitioned
                                 LPs: 2-4 select the epoch-major matrix-free operator,
                                 auto the stored matrix */
  int32_t pdl;                /* 1: programmatic dependent launch between the iteration
                                 kernels (prologue of one overlaps the tail of the last) (1) */
  int32_t fused_halo;         /* row-partitioned solves: the half-step kernels store their
                                 boundary outputs into the neighbours' windows over peer
                                 memory and signal, instead of separate halo kernels (1) */
  double eps_res;             /* > 0: primal and dual residual tolerance min(eps_rel, eps_res),
                                 the duality gap keeps eps_rel -- the parity bar (gap 1e-4,
                                 residuals 1e-6); 0: eps_rel for all three (1e-6) */
  double eps_infeas;          /* primal-infeasibility certificate margin: the solve stops with
                                 TECCL_PRIMAL_INFEASIBLE once the change of the dual iterate
                                 between two evaluations is a Farkas ray whose value exceeds
                                 this fraction of its terms' magnitude; 0 disables (1e-6).
                                 Single-device solves only */
  int32_t infeas_every;       /* checks between certificate evaluations (4) */
  int32_t persist;            /* 1: run each chunk of iterations as one persistent cooperative
                                 kernel (dense state in shared memory, grid barriers between
                                 half-steps) when the LP is on the stored operator and every
                                 block's share fits in shared memory -- L2-resident LPs such as
                                 configs[1]; same arithmetic per entry, partial sums of the
                                 restart metrics in another order) (0: measured slower) */
  double omega_bias;          /* multiplies the primal-weight target dy/dx at restarts (1.0) */
  double step_safety;         /* eta = step_safety / (power-iteration estimate of
                                 ||E^1/2 A D^1/2||_2), in (0, 1) (0.998) */
} teccl_pdlp_opts;

typedef struct {
  int32_t status;
  int32_t restarts;
  int64_t iters;
  double primal_obj;       /* c.x of the returned point (minimisation form) */
  double dual_obj;
  double rel_gap;
  double rel_primal_res;
  double rel_dual_res;
  double solve_seconds;    /* device time, scaling + iterations + unscaling */
  double omega;            /* final primal weight */
  double step;             /* eta = step_safety / ||E^1/2 A D^1/2||_2 estimate */
  int64_t spmv_launches;   /* all kernel launches issued by the solve (setup + chunks) */
  double infeas_cert;      /* last Farkas certificate value / magnitude (> eps_infeas:
                              TECCL_PRIMAL_INFEASIBLE); 0 before the first evaluation */
} teccl_pdlp_result;

void teccl_pdlp_default_opts(teccl_pdlp_opts* o);
/* x_inout [n] / y_inout [m] host buffers (either may be NULL): read when
 * warm_start, written with the solution on return. */
int teccl_pdlp_solve(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                     double* x_inout, double* y_inout, teccl_pdlp_result* res);
/* Device-pointer variant: x_dev/y_dev are device buffers owned by the caller. */
int teccl_pdlp_solve_dev(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                         double* x_dev, double* y_dev, teccl_pdlp_result* res);

/* One A.x then one A^T.y over the LP's unit/explicit CSR and CSC, `reps`
 * times, timed with CUDA events on the context stream. Reports mean
 * milliseconds per pair and the algorithmic bytes of one pair. */
int teccl_spmv_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* ms_per_pair,
                     double* bytes_per_pair);

/* out = A.in (transpose = 0, length m) or A^T.in (transpose = 1, length n)
 * through the stored CSR/CSC (matrix_free = 0) or, for LPs from
 * teccl_lp_build_te, the per-entry matrix-free operator (1) or the segment
 * walkers the PDLP kernels use (2), with the row bounds /
 * column bounds and costs that path uses (lo/hi/cost may be NULL; cost only
 * for transpose = 1). Host buffers. The parity tests pin the two paths to
 * each other bit for bit. */
int teccl_lp_apply(teccl_ctx* ctx, teccl_lp* lp, int32_t transpose, int32_t matrix_free,
                   const double* in, double* out, double* lo, double* hi, double* cost);

/* Time the two fused PDLP iteration kernels alone (after the real scaling
 * setup), `reps` launches each, CUDA events on the context stream.
 * out6 = {ms per column-kernel launch, ms per row-kernel launch, algorithmic
 * bytes per column launch, per row launch, operator (0 stored + bound arrays,
 * 1 stored matrix + bound dictionaries, 2/3/4 the matrix-free mode used),
 * SELL slice}. */
int teccl_pdlp_step_bench(teccl_ctx* ctx, teccl_lp* lp, int32_t reps, double* out6);
/* Same with explicit options (NULL = defaults): the operator (`matrix_free`),
 * `col_pipeline` and `pdl` select the kernels that are timed. */
int teccl_pdlp_step_bench_opts(teccl_ctx* ctx, teccl_lp* lp, const teccl_pdlp_opts* opts,
                               int32_t reps, double* out6);

/* ---------------------------------------------------------------------------
 * (4) Exact-integer schedule checker for a time-expanded LP solution: the
 * flow-level counterpart of simulate() (simulator.py:58-235), on the GPU:
 * flows are quantised to `quantum` units per chunk (int64) and the replay is
 * exact: per (edge,epoch) capacity, per (source,node,epoch) buffer >= 0
 * (causality), switches hold nothing across epochs, every pair's cumulative
 * reads reach its demand. `slack_units` is the per-check integer tolerance
 * (0 = exact). x is the LP solution in the builder's variable order.
 */
typedef struct {
  int64_t capacity_violations;
  int64_t causality_violations;   /* negative buffer at a GPU */
  int64_t switch_violations;      /* switch in != out */
  int64_t unmet_pairs;            /* cumulative reads short of demand */
  int32_t completion_epoch;       /* max over pairs of first epoch reads reach demand; -1 if none */
  int64_t max_capacity_excess;    /* units */
  int64_t max_buffer_deficit;     /* units */
} teccl_check_report;

int teccl_check_te(teccl_ctx* ctx, const teccl_te_desc* desc, const double* x_host,
                   int64_t quantum, int64_t slack_units, teccl_check_report* out);
int teccl_check_te_dev(teccl_ctx* ctx, const teccl_te_desc* desc, const double* x_dev,
                       int64_t quantum, int64_t slack_units, teccl_check_report* out);

/* ---------------------------------------------------------------------------
 * Rate -> schedule decomposition (host CPU, one thread per source). Replaces
 * lp_rates_to_schedule (pkg/src/collsched/lp.py:156-301) on an LP solution x
 * in the builder's variable order. in_ptr/in_edges: in-edges of every node in
 * str(sender) order; pair_chunk_ptr/pair_chunks: demanded chunk ids of every
 * pair in (str(source), chunk, str(dst)) order; pair_order: pairs in the order
 * the reference visits them; source_rank/node_rank: positions in str() order.
 * tol: entries at or below it count as empty while tracing; need_tol: unserved
 * remainder accepted per chunk. On success *out holds the merged, sorted
 * events; teccl_schedule_fetch copies them out (src_slot = source slot,
 * edge = edge index) and frees the handle. */
int teccl_schedule_te(const teccl_te_desc* desc, const double* x, double tol, double need_tol,
                      const int32_t* in_ptr, const int32_t* in_edges,
                      const int32_t* pair_chunk_ptr, const int32_t* pair_chunks,
                      const int32_t* pair_order, const int32_t* source_rank,
                      const int32_t* node_rank, int32_t threads, void** out, int64_t* n_events);
int teccl_schedule_fetch(void* handle, int32_t* src_slot, int32_t* chunk, int32_t* edge,
                         int32_t* epoch, double* frac);

/* ---------------------------------------------------------------------------
 * (4b) Event-level schedule replay (host CPU, one thread per commodity).
 * Replaces simulate() (pkg/src/collsched/simulator.py:58-208 with
 * _check_capacity :211-223 and _check_switch_rest :226-235) for copy /
 * no-copy switches: the emitted event list is replayed -- sends of data the
 * sender does not hold (causality), per-(edge, window) capacity, switch
 * arrivals left over after their one forwarding epoch, unmet demand. The
 * caller computes each edge's delay, capacity window and window budget with
 * the reference's exact rational arithmetic (simulator.py:80-92).
 */
typedef struct {
  int32_t num_nodes;
  const uint8_t* node_is_switch;  /* [num_nodes] */
  int32_t num_edges;
  const int32_t* edge_delta;      /* [E] ceil(alpha/tau) + window widening */
  const int32_t* edge_window;     /* [E] capacity window in epochs (kap) */
  const double* edge_budget;      /* [E] float(kap * capacity*tau/chunk) */
  int64_t num_entries;            /* demanded (source, chunk, destination) entries */
  const int32_t* entry_source;    /* [num_entries] node index */
  const int32_t* entry_chunk;
  const int32_t* entry_dst;       /* node index */
  int32_t switch_mode;            /* 0 copy, 1 no-copy */
  double tolerance;               /* SimOptions.tolerance (1e-6) */
} teccl_sim_desc;

/* Events (source node, chunk, src node, dst node, edge index, epoch,
 * fraction) in any order; source_rank / node_rank: position of each node in
 * str() order (the replay order is (epoch, str(source), str(src), str(dst),
 * chunk), stable). counts4 = {causality, capacity, switch-rest violations,
 * entries}; teccl_simulate_fetch copies them out -- causality as event ids in
 * replay order, capacity as (edge, epoch) pairs in (edge, epoch) order,
 * switch rest as (source, chunk, switch node, usable epoch), per-entry
 * completion epochs (-1 = unmet) -- and frees the handle. */
int teccl_simulate(const teccl_sim_desc* desc, int64_t n_events, const int32_t* ev_source,
                   const int32_t* ev_chunk, const int32_t* ev_src, const int32_t* ev_dst,
                   const int32_t* ev_edge, const int32_t* ev_epoch, const double* ev_frac,
                   const int32_t* source_rank, const int32_t* node_rank, int32_t threads,
                   void** out, int64_t* counts4);
int teccl_simulate_fetch(void* handle, int64_t* causality, int64_t* capacity, int64_t* sw_rest,
                         int32_t* entry_done);

#ifdef __cplusplus
}
#endif
#endif /* TECCL_B200_H */
