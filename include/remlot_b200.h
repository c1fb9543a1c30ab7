/*
 * remlot_b200.h -- C ABI of the B200 VND hot path (libremlot_b200.so).
 *
 * Drop-in boundary for the reference package `remlot`, whose operator API is
 * its set of numba kernels called with flat numpy buffers
 * (reference pkg/src/remlot/_kernels.py) plus the VND driver (vnd.py).  Each
 * entry point below names the reference interface it replaces.  Plain C
 * types only: host pointers unless the name ends in _device (device
 * pointers, asynchronous on the given cudaStream_t passed as void*).
 *
 * Conventions (mirroring the reference):
 *   - setup plans are two bool (uint8 0/1) K x T C-order matrices;
 *   - instance matrices are int64 K x T C-order; cost vectors int64[K] in the
 *     order setup_m, setup_r, holding_m, holding_r, unit_m, unit_r;
 *   - costs are int64 cents, RL_INFEASIBLE = 1 << 62 (_kernels.py:11);
 *   - caller-allocated outputs; return 0 on success, negative on error
 *     (RL_E*), message in rl_last_error() (thread-local);
 *   - a handle is bound to the CUDA device that was current at creation;
 *   - thread safety: every entry point taking a handle holds the handle's
 *     mutex for the call (single calls may come from any thread); no entry
 *     point synchronises the whole device.  Multi-call sequences over state
 *     kept on the handle (rl_vnd_device + rl_vnd_collect, the rl_gvns_*
 *     session) need one handle per concurrent user.
 */
#ifndef REMLOT_B200_H
#define REMLOT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RL_INFEASIBLE ((int64_t)1 << 62)

#define RL_OK 0
#define RL_EINVAL -1   /* bad argument (reference raises ValueError/IndexError) */
#define RL_ECUDA -2    /* CUDA runtime error (message says which) */
#define RL_ERANGE -4   /* instance values outside the exact int64 range */

typedef struct rl_instance rl_instance;

/* Upload an instance once; the handle owns its device memory.
 * Replaces the Instance arrays handed to every kernel call
 * (reference model.py:28-72, vnd.py:141-145, plan.py:120-123).
 * 1 <= T <= 16000.  The move-scoring entry points keep one product's
 * horizon in shared memory (~26 B per period with int32 values, ~38 B with
 * int64): horizons beyond ~8,000 (int32) / ~5,800 (int64) periods return
 * RL_EINVAL from rl_vnd / rl_scan_products / rl_product_costs. */
int rl_instance_create(int64_t K, int64_t T, const int64_t *demand, const int64_t *returns,
                       const int64_t *setup_m, const int64_t *setup_r,
                       const int64_t *hold_m, const int64_t *hold_r,
                       const int64_t *unit_m, const int64_t *unit_r, rl_instance **out);
/* Re-upload new data of the same K x T into an existing handle. */
int rl_instance_update(rl_instance *h, const int64_t *demand, const int64_t *returns,
                       const int64_t *setup_m, const int64_t *setup_r,
                       const int64_t *hold_m, const int64_t *hold_r,
                       const int64_t *unit_m, const int64_t *unit_r);
void rl_instance_destroy(rl_instance *h);
/* _kernels.oracle_product / oracle.enumerate_optimal (_kernels.py:347-371,
 * oracle.py:19-44): per product the minimum cost over all 2^(2T) setup
 * patterns (lowest (m, r) mask pair on ties) and that pattern; T <= 10
 * (larger T -> RL_EINVAL like the reference's ValueError). */
int rl_oracle_optimal(rl_instance *h, int64_t *cost, uint8_t *sm, uint8_t *sr);

/* Kernel variants of rl_vnd (results are identical; for A/B measurement and
 * tests).  Bit 0: reserved (was two products per warp; removed, RL_EINVAL).
 * Bit 1: T > 63 never uses one CTA per product (by default
 * a CTA per product is used when K <= 2 x SMs, a warp per product above).
 * Bits 2/3: T <= 63 slack skip always / never (default: per launch).
 * Bit 4: int64 values and int64 costs whatever the range proof allows (the
 * general path; the narrow exact widths are the default).
 * Bit 5: reserved (lane kernel off, the default).  Bit 6: T <= 63 runs the
 * lane-per-product kernel (k_vnd_lane; exact, slower at C3: DESIGN.md 5).
 * Bit 7: never the 16-bit long-horizon rows.  Bit 8: T > 63 always one CTA
 * per product (measured slower at C4: 203 vs 137 ms). */
int rl_instance_set_variant(rl_instance *h, int variant);
/* info[0..5] = K, T, bytes per period value (4|8), bytes per cost (4|8),
 * SM count, warps per CTA of the resident VND kernel. */
int rl_instance_info(const rl_instance *h, int64_t *info);

/* _kernels.product_costs(lo, hi, ...) (_kernels.py:171-175) / plan.evaluate
 * (plan.py:117-126): out[k] for k in [lo, hi), RL_INFEASIBLE if infeasible.
 * sm/sr are full K x T plans; out has K entries. */
int rl_product_costs(rl_instance *h, int64_t lo, int64_t hi, const uint8_t *sm,
                     const uint8_t *sr, int64_t *out);

/* _kernels.scan_products(lo, hi, ..., nbh, out_*) (_kernels.py:261-325):
 * best strictly improving move of neighborhood nbh per product in [lo, hi);
 * out_* have K entries, only [lo, hi) is written.  m0/r0 (m1/r1) are 0 where
 * no move won (where p1 < 0); the reference leaves them unwritten.
 * *evals (may be NULL) = number of candidate moves scored. */
int rl_scan_products(rl_instance *h, int64_t lo, int64_t hi, const uint8_t *sm,
                     const uint8_t *sr, int nbh, int64_t *dec, int64_t *p0, uint8_t *m0,
                     uint8_t *r0, int64_t *p1, uint8_t *m1, uint8_t *r1, int64_t *evals);

/* _kernels.apply_scan(lo, hi, ...) (_kernels.py:328-344): writes winners into
 * sm/sr (K x T, in place) and returns the product-ordered sum in *diff. */
int rl_apply_scan(rl_instance *h, int64_t lo, int64_t hi, const int64_t *dec,
                  const int64_t *p0, const uint8_t *m0, const uint8_t *r0, const int64_t *p1,
                  const uint8_t *m1, const uint8_t *r1, uint8_t *sm, uint8_t *sr,
                  int64_t *diff);

/* _kernels.list_moves(nbh, sm_row, sr_row, mp0, mm0, mr0, mp1, mm1, mr1)
 * (_kernels.py:188-258) for one product row of length T; buffers hold 2T
 * entries; *n = move count.  mm1/mr1 are 0 for single-period moves. */
int rl_list_moves(int nbh, int64_t T, const uint8_t *sm_row, const uint8_t *sr_row,
                  int64_t *mp0, uint8_t *mm0, uint8_t *mr0, int64_t *mp1, uint8_t *mm1,
                  uint8_t *mr1, int64_t *n);

/* vnd.vnd(inst, plan, k_max) (vnd.py:253-289): descend to a local optimum of
 * N1..Nk_max.  Bit-identical plan, cost and trace to the reference's
 * lockstep loop.  trace gets 1 + k_max*sweeps entries (*n_trace; if it
 * exceeds trace_cap only trace_cap are written).  stats[0..7] = final cost,
 * start cost, sweeps, candidate evaluations performed, reference-equivalent
 * evaluations (lockstep count), moves applied, products,
 * kernel time in ns, sum over feasible products of their final move counts
 * (stats has 9 entries). */
int rl_vnd(rl_instance *h, int k_max, const uint8_t *sm_in, const uint8_t *sr_in,
           uint8_t *sm_out, uint8_t *sr_out, int64_t *trace, int64_t trace_cap,
           int64_t *n_trace, int64_t *stats);

/* Device-resident variant: plans are device pointers; enqueued on stream
 * (cudaStream_t as void*, NULL = the handle's stream) without host sync.
 * Read results with rl_vnd_collect afterwards. */
int rl_vnd_device(rl_instance *h, int k_max, const uint8_t *d_sm_in, const uint8_t *d_sr_in,
                  uint8_t *d_sm_out, uint8_t *d_sr_out, void *stream);
int rl_vnd_collect(rl_instance *h, int64_t *trace, int64_t trace_cap, int64_t *n_trace,
                   int64_t *stats);

/* Per-product results of the last descent on h (K entries each): own
 * sweeps, moves applied and candidate evaluations performed.  Diagnostic
 * (work distribution); no reference counterpart. */
int rl_vnd_product_stats(rl_instance *h, int32_t *sweeps, int32_t *moves, int64_t *evals);

/* rl_instance_update + rl_vnd in one call (same arguments and results): the
 * host->device copies of the instance and plan rows are cut into product
 * chunks and overlapped with the descent of the chunks before them on two
 * compute streams (the e2e path of bench.py; pinned host buffers give the
 * overlap).  Falls back to the two calls when the new data need wider exact
 * integers than the handle holds. */
int rl_vnd_host(rl_instance *h, int k_max, const int64_t *demand, const int64_t *returns,
                const int64_t *setup_m, const int64_t *setup_r, const int64_t *hold_m,
                const int64_t *hold_r, const int64_t *unit_m, const int64_t *unit_r,
                const uint8_t *sm_in, const uint8_t *sr_in, uint8_t *sm_out, uint8_t *sr_out,
                int64_t *trace, int64_t trace_cap, int64_t *n_trace, int64_t *stats);

/* model.generate_instance(GeneratorConfig(...)) (model.py:115-153) on the
 * device: the same numpy Philox stream and Lemire draws, bit-identical
 * arrays.  ranges = {setup lo, hi, holding lo, hi, unit lo, hi} (inclusive).
 * The handle keeps products [lo, hi) of the K-product instance (lo = 0,
 * hi = K for all of it).  RL_EINVAL for configs GeneratorConfig rejects and
 * for ranges of 2^32-1 or more (numpy's 64-bit draw path). */
int rl_generate_instance(int64_t K, int64_t T, uint64_t seed, int64_t demand_max,
                         double return_ratio, const int64_t *ranges, int64_t lo, int64_t hi,
                         rl_instance **out);

/* The handle's instance back in host arrays (K x T, K x T, six K-vectors). */
int rl_instance_download(rl_instance *h, int64_t *demand, int64_t *returns, int64_t *setup_m,
                         int64_t *setup_r, int64_t *hold_m, int64_t *hold_r, int64_t *unit_m,
                         int64_t *unit_r);

/* plan.initial_solution(inst) (plan.py:140-167): lot-for-lot start. */
int rl_initial_solution(rl_instance *h, uint8_t *sm, uint8_t *sr);
int rl_initial_solution_device(rl_instance *h, uint8_t *d_sm, uint8_t *d_sr, void *stream);

/* plan.decode (plan.py:99-114, _kernels.row_decode :100-168): per period
 * quantities x_m, x_r and stocks y_m, y_r (K x T each) and per product cost;
 * rows of infeasible products are zero and their cost RL_INFEASIBLE. */
int rl_decode(rl_instance *h, const uint8_t *sm, const uint8_t *sr, int64_t *x_m,
              int64_t *x_r, int64_t *y_m, int64_t *y_r, int64_t *cost);

/* ---- device GVNS (reference gvns.py:88-244) ----------------------------
 * rl_gvns_begin uploads an incumbent plan (must be feasible), computes the
 * lot-for-lot start and F = the VND image of the incumbent, sets strength 1.
 * workers = W local workers with global indices worker_offset.., k_max =
 * shake strength bound, k_vnd_max in 1..4, seed = the solver seed (used mod
 * 2^64 like gvns.py:89).  *inc_cost = evaluate(inc). */
int rl_gvns_begin(rl_instance *h, int workers, int64_t worker_offset, int k_max, int k_vnd_max,
                  uint64_t seed, const uint8_t *sm, const uint8_t *sr, int64_t *inc_cost);
/* rl_gvns_begin with speculative batches of `batch` (1..32) rounds for
 * rl_gvns_run: B x W worker slots; the round counter starts at 0. */
int rl_gvns_begin_batch(rl_instance *h, int workers, int batch, int64_t worker_offset, int k_max,
                        int k_vnd_max, uint64_t seed, const uint8_t *sm, const uint8_t *sr,
                        int64_t *inc_cost);
/* Overwrite the shake strength k (worker_round(..., k, ...)). */
int rl_gvns_set_strength(rl_instance *h, int64_t strength);
/* One round (worker_round, gvns.py:147-174) with round index round_index;
 * accept = 1 also applies the GVNS step (gvns.py:207-215) on the device
 * (accept strict improvement, next_strength).  Asynchronous. */
int rl_gvns_round(rl_instance *h, int64_t round_index, int accept);
/* The gvns loop body (gvns.py:200-215) for up to `batch` rounds starting at
 * the device round counter, never past max_rounds: every round of the batch
 * shakes the incumbent with the strength it has if the rounds before it do
 * not improve; the join applies the rounds in order and stops at the first
 * accepted one (later rounds are re-run by the next call), so the result is
 * the sequential trajectory.  Asynchronous; the counter is info[6]. */
int rl_gvns_run(rl_instance *h, int64_t max_rounds);
/* The whole gvns loop (gvns.py:200-215) on the device: speculative batches
 * inside a CUDA-graph conditional WHILE node until the device round counter
 * reaches max_rounds or budget_ns nanoseconds of device time (%globaltimer,
 * from the launch) have passed, checked between batches (the reference
 * checks between rounds; a batch is at most 4 rounds, each the round the
 * sequential loop would run).  One graph launch; synchronous. */
int rl_gvns_run_until(rl_instance *h, int64_t max_rounds, int64_t budget_ns);
/* which = 0: incumbent, 1: last round's winning candidate (accept = 0).
 * info[0..6] = incumbent cost, strength, last best cost, last best worker,
 * accepted rounds, shake fallbacks in the last round, rounds completed.
 * sm/sr may be NULL. */
int rl_gvns_state(rl_instance *h, int which, uint8_t *sm, uint8_t *sr, int64_t *info);
/* Sharded rounds (one rank per GPU, workers split in blocks): after
 * rl_gvns_round(h, r, 0), rl_gvns_candidate copies this rank's winning
 * candidate plan (2KT bytes: m rows then r rows) to device memory d_plan
 * (may be NULL) and writes best[0] = its cost, best[1] = its global worker;
 * rl_gvns_import(h, d_plan, cost) makes the job's winner (a VND fixpoint,
 * device memory) the incumbent. */
int rl_gvns_candidate(rl_instance *h, uint8_t *d_plan, int64_t *best);
int rl_gvns_import(rl_instance *h, const uint8_t *d_plan, int64_t cost);
/* Sharded rounds in speculative batches (one collective per batch): after
 * rl_gvns_begin_batch(h, W_local, B, ...) and rl_gvns_set_strength(h, k),
 * rl_gvns_run_local runs rounds round0 .. round0+nb-1 (nb <= B) of this
 * rank's worker block, each shaking the incumbent with the strength it has
 * if the rounds before it do not improve, without acceptance; out[3j..3j+2]
 * = round j's best (cost, global worker, local slot) for j < *n_out (fewer
 * than nb when the fallback slots ran out; the caller re-runs the rest).
 * rl_gvns_export copies round jr's best candidate (2KT bytes, device memory)
 * for the winner's broadcast; the job's winner is adopted with
 * rl_gvns_import.  Both synchronous. */
int rl_gvns_run_local(rl_instance *h, int64_t round0, int nb, int64_t *out, int64_t *n_out);
int rl_gvns_export(rl_instance *h, int jr, uint8_t *d_plan);
/* Test hook: numpy-exact Philox stream of SeedSequence((seed, round,
 * worker)) on the device: out = 4 raw next64, choice(pop, size,
 * replace=False), shuffle of [1, 4, 7, ...] (shuffle_n), one more next64. */
int rl_rng_probe(uint64_t seed, uint64_t round, uint64_t worker, int64_t pop, int64_t size,
                 int64_t shuffle_n, int64_t *out);

/* Measured INT32 throughput of the current device (integer ops/s; IMAD +
 * LOP3 chains over all SMs): the roofline denominator of the ALU-bound VND
 * kernel. */
int rl_int_peak(double *ops_per_s);

/* Number of kernel launches issued by this handle since creation. */
int64_t rl_launch_count(const rl_instance *h);

const char *rl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
