/*
 * phylograd.h -- C ABI of the B200 (sm_100a) branch-length gradient library.
 *
 * One instance evaluates, for a fixed tree topology and substitution model,
 *   logL = sum_c w_c log sum_r P(gamma_r) pi' p_{root,r,c}       (Eq. 3)
 * and its gradient with respect to all 2N-2 branch lengths
 *   d/db_i logL = sum_c w_c [sum_r gamma_r P(gamma_r) p'Q'q] / [sum_r P(gamma_r) p'q]
 *                                                                 (Eq. 6-8)
 * in O(N) work per pattern: a post-order pass (Eq. 2), a pre-order pass
 * (Eq. 4) and a per-edge reduction over patterns and rate categories.
 * Equation and line numbers refer to PAPER.md (arXiv 2303.04390):
 * Eq. 1, Eq. 2, Eq. 3, Eq. 4 P:242-262,
 * Eq. 5, Eq. 6-8, numbering P:197-201, patterns P:191-193.
 *
 * Conventions
 *  - Node numbering (P:197-201, 0-based): tips 0..N-1, internal nodes
 *    N..2N-3, root 2N-2.  Branch i (0 <= i < 2N-2) is the edge above node i.
 *  - Matrices are row-major doubles.  The transition matrix of branch i,
 *    category r is P = V diag(exp(gamma_r b_i lambda)) V^{-1} (Eq. 1); entry
 *    (s, t) is the probability of child state t given parent state s.
 *  - Every host input is COPIED at the set_* call; the library keeps no
 *    pointer to caller memory.  Outputs are written to caller buffers.
 *  - One instance is bound to one CUDA device and one stream and is not
 *    thread-safe.  All device work is ordered on that stream.  Every call
 *    switches to the instance's device and restores the caller's current
 *    device before returning.
 *  - Errors: every call returns PG_OK (0) or a PG_ERR_* code; the message of
 *    the last failure is pg_last_error(instance).  A failed call leaves the
 *    instance's previous state unchanged.
 *  - The library does not normalise Q, pi, the category rates or weights
 *    (that is the caller's job); it does not clamp transition probabilities.
 *  - Underflow: partial likelihoods are rescaled by exact powers of two per
 *    (node, pattern), shared across categories; results equal the unscaled
 *    arithmetic (no extra rounding).  Not in the paper (reading R4).
 */
#ifndef PHYLOGRAD_H
#define PHYLOGRAD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define PG_OK                   0
#define PG_ERR_ARG              1  /* NULL pointer, size or index out of range     */
#define PG_ERR_DOMAIN           2  /* negative branch length, rate <= 0, weight < 0 */
#define PG_ERR_TOPOLOGY         3  /* op list is not a rooted bifurcating tree      */
#define PG_ERR_SEQUENCE         4  /* compute before all inputs were set            */
#define PG_ERR_ZERO_LIKELIHOOD  5  /* some pattern has L_c = 0 (logL = -inf)        */
#define PG_ERR_CUDA             6  /* CUDA runtime failure (message has details)    */
#define PG_ERR_UNSUPPORTED      7  /* configuration outside what the build supports */
#define PG_ERR_MEMORY           8  /* device/host allocation failed or too small    */

/* ---- precision --------------------------------------------------------- */
#define PG_FP64 0   /* partials and arithmetic in double                          */
#define PG_FP32 1   /* partials in float; logL and gradient reductions in double */

/* ---- flags ------------------------------------------------------------- */
#define PG_FLAG_TIP_PARTIALS  1u  /* reserve space for pg_set_tip_partials     */

typedef struct pg_instance pg_instance;

typedef struct {
    int32_t tips;        /* N >= 2                                              */
    int32_t patterns;    /* C >= 1 unique site patterns             */
    int32_t states;      /* S, 2 <= S <= 128 (4, <=16, <=64, <=128 paths)      */
    int32_t categories;  /* R, 1 <= R <= 16 rate categories         */
    int32_t precision;   /* PG_FP64 or PG_FP32                                  */
    int32_t device;      /* CUDA device ordinal                                 */
    uint32_t flags;      /* PG_FLAG_*                                           */
} pg_config;

/* Library ABI version (major*10000 + minor*100 + patch). */
int pg_version(void);

/* Device bytes an instance with this configuration needs.  Use it to hand
 * pg_create a caller-allocated workspace (e.g. a torch tensor).
 * Errors: PG_ERR_ARG, PG_ERR_UNSUPPORTED. */
int pg_workspace_bytes(const pg_config *cfg, size_t *bytes);

/* Create an instance.
 *   cuda_stream     cudaStream_t to order all work on; NULL => the library
 *                   creates (and owns) a non-blocking stream.
 *   dev_workspace   device memory of >= pg_workspace_bytes() bytes, owned by
 *                   the caller and kept alive until pg_destroy; NULL => the
 *                   library allocates (and frees) its own.  Nucleotide (S <= 4)
 *                   instances with state tips also get library-allocated
 *                   staging buffers for the post-order pass (per internal
 *                   node one step record of its matrices, ~2 KB at R = 4 fp64,
 *                   and per CTA its tip-code windows, ~0.2 KB per CTA and
 *                   node), freed by pg_destroy.
 * Errors: PG_ERR_ARG, PG_ERR_UNSUPPORTED, PG_ERR_MEMORY, PG_ERR_CUDA. */
int pg_create(const pg_config *cfg, void *cuda_stream, void *dev_workspace,
              size_t workspace_bytes, pg_instance **out);

/* Destroy an instance (synchronises its stream).  NULL is a no-op. */
int pg_destroy(pg_instance *inst);

/* Observed states of one tip: states[c] in 0..S-1, or S for missing data
 * (all-ones partial).  P:613-614 (tips as compressed integer states).
 * Errors: PG_ERR_ARG (tip out of range, state outside 0..S). */
int pg_set_tip_states(pg_instance *inst, int32_t tip, const int32_t *states /*[C]*/);

/* Arbitrary tip partial vectors (ambiguity codes, hidden states of
 * Markov-modulated models): partials[c*S + s] >= 0, pattern-major.
 * Requires PG_FLAG_TIP_PARTIALS.  Errors: PG_ERR_ARG, PG_ERR_DOMAIN. */
int pg_set_tip_partials(pg_instance *inst, int32_t tip, const double *partials /*[C][S]*/);

/* Site-pattern weights w_c >= 0 (counts from compression; 0 allowed).
 * Errors: PG_ERR_ARG, PG_ERR_DOMAIN. */
int pg_set_pattern_weights(pg_instance *inst, const double *weights /*[C]*/);

/* Root prior pi (Eq. 3; q_root = pi in Eq. 4).  Errors: ARG, DOMAIN. */
int pg_set_state_frequencies(pg_instance *inst, const double *pi /*[S]*/);

/* Real eigensystem of Q: Q = V diag(lambda) V^{-1} (Eq. 1).  evec = V and
 * ievec = V^{-1} row-major [S][S], eval = lambda [S].  Q itself is formed
 * from these.  Errors: PG_ERR_ARG (NULL / non-finite). */
int pg_set_eigen(pg_instance *inst, const double *evec, const double *ievec,
                 const double *eval);

/* Category rates gamma_r > 0 and weights P(gamma_r) >= 0. */
int pg_set_category_rates(pg_instance *inst, const double *rates /*[R]*/);
int pg_set_category_weights(pg_instance *inst, const double *weights /*[R]*/);

/* Post-order operation list: n_ops = N-1 triples (dest, child1, child2),
 * children defined before they are used, last dest = root (2N-2).
 * Re-plans the traversal (stack schedule) and re-captures the CUDA graph.
 * Errors: PG_ERR_ARG, PG_ERR_TOPOLOGY. */
int pg_set_operations(pg_instance *inst, const int32_t *ops /*[n_ops][3]*/, int32_t n_ops);

/* Branch lengths b_i >= 0 indexed by child node, i = 0..2N-3.  May
 * change between computes (the HMC use case).  The host copy goes through a
 * pinned staging buffer and is uploaded inside the next pg_compute /
 * pg_compute_device.  If a previous pg_compute_device's upload from that
 * buffer is still queued on the stream, this call first waits for it (so an
 * evaluation always sees the values set before it).
 * Errors: PG_ERR_ARG, PG_ERR_DOMAIN, PG_ERR_CUDA. */
int pg_set_branch_lengths(pg_instance *inst, const double *b /*[2N-2]*/);

/* Same, from DEVICE memory: a stream-ordered device-to-device copy (no
 * validation of the values).  For callers whose branch lengths live on the
 * GPU (device-resident HMC, benchmarks). */
int pg_set_branch_lengths_device(pg_instance *inst, const double *d_b /*[2N-2]*/);

/* Evaluate logL and the gradient; synchronous, host outputs (not allowed
 * while the instance stream is being captured: PG_ERR_SEQUENCE).
 *   gradient  [2N-2] or NULL (logL only is still a full evaluation).
 * On PG_ERR_ZERO_LIKELIHOOD *log_likelihood = -inf, the gradient is not
 * written, and pg_last_error names the first such pattern.
 * Errors: PG_ERR_SEQUENCE, PG_ERR_ZERO_LIKELIHOOD, PG_ERR_CUDA. */
int pg_compute(pg_instance *inst, double *log_likelihood, double *gradient);

/* Asynchronous evaluation into DEVICE memory: d_out[0] = this instance's
 * logL, d_out[1 + i] = gradient entry i (2N-1 doubles), stream-ordered, no
 * host synchronisation.  These are the partial sums over this instance's
 * patterns (Eq. 6 is a sum over patterns), ready for an
 * allreduce(sum) across pattern shards.  Zero likelihoods are
 * recorded on the device; read them with pg_check_status.
 * Stream capture: normally the evaluation is replayed from a CUDA graph the
 * library captured itself.  If the CALLER is capturing the instance stream
 * (cudaStreamBeginCapture), the kernels are enqueued straight into the
 * caller's graph instead, so one graph can hold [pg_set_branch_lengths_device,
 * pg_compute_device, ncclAllReduce].  Under capture the call must not need
 * host uploads: run one evaluation outside capture first (else
 * PG_ERR_SEQUENCE); host-staged branch lengths become memcpy nodes that
 * re-read the pinned staging buffer at every replay.
 * Errors: PG_ERR_SEQUENCE, PG_ERR_CUDA. */
int pg_compute_device(pg_instance *inst, double *d_out /*[2N-1]*/);

/* ---- Time-tree ("clock") parameterisation of the branch lengths ----------
 * a branch length "can ... be the difference between the
 * parent and child node heights measured in time-units multiplied by a
 * (possibly branch-specific) evolutionary rate scalar":
 *     b_i = rho_i * tau_i,   tau_i = h_parent(i) - h_i,   i = 0..2N-3.
 * The gradient w.r.t. these parameters is the chain rule on g = dlogL/db
 * (HMC over rate scalars and node heights,
 * P:967-968; strict clock "reduce the partial derivatives across a set of
 * branches").  Node numbering and parents come from the operation
 * list (pg_set_operations must have been called).
 *
 * pg_set_node_heights: host heights [2N-1] (tips may be non-zero: serially
 * sampled data) and rate scalars [2N-2] (NULL = all 1), validated
 * (h_parent >= h_child, rho >= 0, finite; else PG_ERR_DOMAIN), copied, and
 * b is formed on the device inside the next compute.
 * pg_set_node_heights_device: the same from DEVICE pointers, stream-ordered,
 * no validation (a child above its parent yields b < 0: undefined results).
 * Both replace any branch lengths set before. */
int pg_set_node_heights(pg_instance *inst, const double *heights /*[2N-1]*/, const double *rates /*[2N-2]*/);
int pg_set_node_heights_device(pg_instance *inst, const double *d_heights, const double *d_rates);

/* Branch sets for clock-rate sums: set_of_branch[i] in -1..n_sets-1 (-1 = in
 * no set), 1 <= n_sets <= 2N-2.  Default (never called): one set holding
 * every branch, i.e. the strict clock b_i = r tau_i.  Errors: PG_ERR_ARG. */
int pg_set_branch_sets(pg_instance *inst, const int32_t *set_of_branch /*[2N-2]*/, int32_t n_sets);

/* Chain rule on the device, on the instance stream, from d_out = [logL, g]
 * as written by pg_compute_device (after any allreduce), using the heights
 * and rates of the last pg_set_node_heights[_device]:
 *   d_grad_rates[i]   = dlogL/drho_i = tau_i g_i                    [2N-2]
 *   d_grad_heights[k] = dlogL/dh_k   = sum_{c: parent(c) = k} rho_c g_c
 *                                      - [k != root] rho_k g_k       [2N-1]
 *   d_set_sums[s]     = sum_{i in set s} tau_i g_i   (= dlogL/dr for
 *                       b_i = r tau_i on the set, fixed-order sum)  [n_sets]
 * Any output may be NULL (skipped).  Device pointers, caller-owned.
 * Errors: PG_ERR_ARG, PG_ERR_SEQUENCE (no heights set), PG_ERR_CUDA. */
int pg_clock_gradient_device(pg_instance *inst, const double *d_out, double *d_grad_rates,
                             double *d_grad_heights, double *d_set_sums);

/* Device-resident HMC leapfrog over theta = log b (the
 * paper's use of the BLS gradient).  Target
 *   log pi(theta) = logL(b = exp(theta)) + sum_i theta_i
 * (logL of Eq. 3 plus the log-Jacobian of b = e^theta; flat prior on b), so
 *   grad_i = b_i dlogL/db_i + 1.
 * Runs n_steps >= 0 leapfrog steps of size eps with diagonal inverse mass:
 *   p += eps/2 grad; repeat { theta += eps M^-1 p; p += eps grad } ... with the
 * last kick eps/2 -- n_steps + 1 full evaluations (each the captured graph),
 * all on the instance stream, no host synchronisation.  In/out: d_theta,
 * d_p [2N-2]; d_inv_mass [2N-2] or NULL (identity).  Out: d_out [2N-1] =
 * [logL, dlogL/db] at the final position; d_grad_theta [2N-2] (or NULL) =
 * grad of log pi at the final position.  Device pointers, caller-owned; the
 * instance's branch lengths become exp(theta_final).  The log-likelihood of
 * a zero-likelihood pattern makes the trajectory meaningless: check with
 * pg_check_status afterwards.  Errors: PG_ERR_ARG (NULL, n_steps < 0,
 * eps not finite), PG_ERR_SEQUENCE, PG_ERR_CUDA. */
int pg_hmc_leapfrog(pg_instance *inst, double *d_theta, double *d_p, const double *d_inv_mass, double eps,
                    int32_t n_steps, double *d_out, double *d_grad_theta);

/* Synchronise the stream and report the first zero-likelihood pattern of the
 * most recent evaluation (-1 if none).  Returns PG_ERR_ZERO_LIKELIHOOD if
 * one occurred. */
int pg_check_status(pg_instance *inst, int32_t *zero_pattern);

/* Number of kernels one evaluation launches (for launch accounting). */
int pg_kernels_per_eval(const pg_instance *inst, int32_t *n);

/* Per-kernel device timing.  When enabled, CUDA events bracket each kernel
 * of an evaluation (event-record nodes inside the captured graph, on the
 * instance stream); pg_get_kernel_times synchronises and returns the
 * durations in milliseconds of the most recent evaluation:
 * ms[0] = transition matrices (A1), ms[1] = traversal (A2-A5),
 * ms[2] = reduction (A6).  Enabling/disabling re-captures the graph. */
int pg_set_kernel_timing(pg_instance *inst, int enable);
int pg_get_kernel_times(pg_instance *inst, float *ms /*[3]*/);

/* Plan statistics after pg_set_operations: post- and pre-order stack depths
 * and the traversal kernel's launch shape. */
typedef struct {
    int32_t post_depth, pre_depth;   /* per-thread stack slots used        */
    int32_t grid, block;             /* traversal kernel launch shape      */
    int32_t smem_bytes;              /* dynamic shared memory per CTA      */
    int32_t prefetch_depth;          /* pre-order prefetch ring stages     */
    int32_t padded_patterns;         /* C rounded up to the CTA tile       */
    int32_t kernel_variant;          /* 0 = small-S, 1 = large-S SIMT,
                                        2 = codon FP64 tensor path        */
    int32_t flow_tiles;              /* codon: 32-pattern tiles per item of
                                        the one-launch dataflow schedule;
                                        0 = one launch per tree level     */
    int32_t flow_version;            /* codon: 2 = warp-specialised TMA ring,
                                        1 = round-1 flow kernel            */
    int32_t flow_stages;             /* codon flow v2: ring stages (1 or 2) */
    int32_t flow_pdl;                /* codon flow v2: launched behind A1
                                        with programmatic dependent launch */
} pg_plan_info;
int pg_get_plan_info(const pg_instance *inst, pg_plan_info *info);

/* Host-only topology check and schedule statistics (no device needed):
 * validates an op list exactly as pg_set_operations does and reports the
 * stack depths of the post- and pre-order traversal plans. */
int pg_plan_check(int32_t tips, const int32_t *ops, int32_t n_ops,
                  int32_t *post_depth, int32_t *pre_depth);

const char *pg_last_error(const pg_instance *inst);
const char *pg_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* PHYLOGRAD_H */
