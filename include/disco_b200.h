/*
 * disco_b200.h -- C-ABI of the B200-native DisCo candidate-scoring path.
 *
 * The reference (`fuseopt`, pure Python) exposes this path as Python
 * callbacks and functions; each entry point below names the reference
 * interface it replaces (paths relative to the reference's pkg/src/fuseopt/).
 * Plain pointers and sizes only; no torch types.  Every function returns an
 * fo_status; fo_last_error() gives a thread-local message for the last
 * failure on the calling thread.
 *
 * Index conventions (identical to build_graph's sort order, graph.py:314-316):
 *   ops        0..V-1 in ascending op id order
 *   edges      0..E-1 sorted by (src, dst)
 *   allreduces 0..A-1 in ascending AllReduce id order
 * A candidate fusion state is three int32 arrays:
 *   normal_gid[V]   group id of each op's normal membership
 *   replica_gid[V]  group id of its replica membership, or -1
 *   bucket_of[A]    bucket id of each AllReduce
 * Group ids lie in [0, gid_bound) and bucket ids in [0, A); only their ORDER
 * is observable (simulator tie-breaks, graph.py:269-273), so callers map the
 * reference's ids to these ranges with any monotone relabelling.
 */
#ifndef DISCO_B200_H
#define DISCO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> fuseopt.errors classes (errors.py:4-53). */
typedef enum {
    FO_OK = 0,
    FO_CYCLE = 1,             /* CycleError: schedule deadlock (simulator.py:133) */
    FO_MISSING_COST = 2,      /* MissingCost (simulator.py:45-46, estimator.py:815-818) */
    FO_NEGATIVE_DURATION = 3, /* ValueError (simulator.py:48-49) */
    FO_DIM_MISMATCH = 4,      /* DimensionMismatch (estimator.py:358-360) */
    FO_INVALID_ARG = 5,       /* malformed input (ids out of range, bad sizes) */
    FO_CUDA_ERROR = 6,        /* CUDA runtime failure */
    FO_UNSUPPORTED = 7        /* configuration outside the device path */
} fo_status;

/* Cost providers (simulator.py:28-35). */
enum {
    FO_PROVIDER_PROFILE = 0,  /* make_cost_providers(profile, comm, model), estimator.py:801-824 */
    FO_PROVIDER_HW_ORACLE = 1 /* oracle_providers(hw), noise == 0, workloads.py:294-304 */
};
/* Fused-op estimator variants (estimator.py:254-257). */
enum {
    FO_EST_INVALID = -2, /* model whose shapes disagree: fused groups raise DimensionMismatch */
    FO_EST_NONE = -1,    /* model=None: fused groups raise MissingCost (estimator.py:815) */
    FO_EST_ANALYTIC = 0,
    FO_EST_LINEAR = 1,
    FO_EST_MESSAGE_PASSING = 2
};
/* Estimator arithmetic on the device. */
enum {
    FO_PREC_FP32 = 0, /* FP32 FFMA message passing: throughput mode, <= 1e-4 rel */
    FO_PREC_FP64 = 1  /* FP64 message passing: decision-exact mode for the search */
};

/* Static graph (replaces HloGraph's ops/edges/allreduces, graph.py:277-299,
 * plus the per-op profile lookup of estimator.py:63-69 resolved once). */
typedef struct {
    int32_t n_ops, n_edges, n_allreduces;
    const int32_t *op_kind;       /* [V] 0 compute, 1 parameter, 2 control (graph.py:29-32) */
    const int64_t *op_out_bytes;  /* [V] OpNode.out_bytes */
    const double *op_profile_us;  /* [V] lookup(profile, op); NaN when the profile has no entry */
    const double *op_compute_us;  /* [V] OpNode.compute_us; NaN for None */
    const int32_t *edge_src;      /* [E] op indices */
    const int32_t *edge_dst;      /* [E] */
    const int64_t *edge_bytes;    /* [E] */
    const int32_t *ar_producer;   /* [A] producer op index */
    const int64_t *ar_bytes;      /* [A] tensor bytes */
} fo_graph_desc;

/* Cost model: what make_cost_providers / oracle_providers close over. */
typedef struct {
    int32_t provider;            /* FO_PROVIDER_* */
    int32_t variant;             /* FO_EST_* (ignored by the hardware oracle) */
    double comm_C, comm_D;       /* CommModelParams (comm.py:20-49) */
    double launch_us;            /* analytic launch_overhead_us / HardwareParams.launch_overhead_us */
    double mem_us_per_byte;      /* analytic mem_us_per_byte / HardwareParams.mem_us_per_byte */
    int32_t layers, hidden, feat_dim; /* message passing hyper-parameters (estimator.py:264-278) */
    const int32_t *op_vocab_slot;     /* [V] one-hot slot of each op's op_code (estimator.py:326-337) */
    /* MESSAGE_PASSING: W_emb[h*F], W_1..W_L[L*h*h], W_r[h*h], A1[h*h], c1[h],
     *                  A2[h*h], c2[h], a3[h], c3[1]   (row-major, estimator.py:554-576)
     * LINEAR:          w[12], b[1]                    (estimator.py:557-561) */
    const double *params;
    int64_t n_params;
    const double *norm_mean; /* node_norm (MP, F entries) or agg_norm (LINEAR, 12); NULL = none */
    const double *norm_std;
    double out_scale;
    /* hardware-oracle jitter (workloads.py:254-291), used when provider ==
     * FO_PROVIDER_HW_ORACLE and hw_noise > 0: every group's oracle time is
     * multiplied by 1 + noise * (2u - 1), u = blake2b-64("{seed}|{content key}")
     * / 2^64 with the content key of _group_content_key (workloads.py:267-273). */
    double hw_noise;              /* HardwareParams.noise in [0, 0.5] */
    const char *hw_key_prefix;    /* UTF-8 "{seed}|" */
    int32_t hw_key_prefix_len;
    const char *op_key_bytes;     /* per op, UTF-8 "{op_code}:{input_shape_key}:{compute_us}" (Python str()) */
    const int64_t *op_key_off;    /* [V + 1] offsets into op_key_bytes */
} fo_cost_model;

typedef struct fo_graph fo_graph;

/* ---- graph handle ------------------------------------------------------ */
int fo_graph_create(const fo_graph_desc *desc, int32_t device, fo_graph **out);
int fo_graph_destroy(fo_graph *g);
/* Replaces make_cost_providers(...) / oracle_providers(...) (estimator.py:801, workloads.py:294). */
int fo_graph_set_cost_model(fo_graph *g, const fo_cost_model *model);

/* Per-round best of a scored batch (device pointers, async): out_pair[2] =
 * {min cost, id_offset + argmin}, lowest id among equal costs (strict-<,
 * search.py:124, :214); candidates with a non-OK status are skipped.  This is
 * the 16-byte value the multi-GPU exchange all-gathers. */
int fo_batch_best(const double *cost, const int32_t *status, int32_t K, int64_t id_offset, double *out_pair,
                  void *stream);
/* Lexicographic min over n (cost, id) pairs, e.g. the all-gathered exchange
 * buffer of every rank's fo_batch_best. */
int fo_pairs_best(const double *pairs, int32_t n, double *out_pair, void *stream);

/* ---- estimator memo ---------------------------------------------------- */
/* Message-passing predictions are a pure function of the fused group's member
 * set (estimator.py:157-191, :363-389); the device caches them per handle.
 * fo_memo_clear empties the cache, ordered on `stream` (NULL: the handle's own
 * stream, which fo_score_host / fo_simulate use); fo_memo_enable(0) turns it off. */
int fo_memo_clear(fo_graph *g, void *stream);
int fo_memo_enable(fo_graph *g, int32_t enable);

/* ---- feature-level prediction ------------------------------------------ */
/* predict_fused(model, featurize(g, group, profile)) (estimator.py:462-470,
 * :157-191) for ONE group given by its features, with the estimator loaded by
 * fo_graph_set_cost_model (profile provider; any variant).  Host buffers,
 * synchronous.  n member ops (local ids 0..n-1 in featurize's node order):
 * op_slot[n] vocab slot (message passing only; else ignored), compute_us[n],
 * in_bytes[n], out_bytes[n]; m internal edges as (src, dst) local pairs in the
 * graph's edge order; aggregates[6] = SubgraphFeatures.aggregate_vector()
 * {member_count, total_compute_us, internal, ext_in, ext_out, longest_path}
 * (estimator.py:117-128).  The MP variant embeds the node features on the device exactly as
 * the per-op table is built at fo_graph_set_cost_model, so the result equals
 * the prediction the scoring kernels make for that group. */
int fo_predict_features(fo_graph *g, int32_t n, const int32_t *op_slot, const double *compute_us,
                        const int64_t *in_bytes, const int64_t *out_bytes, int32_t m, const int32_t *edges,
                        const double *aggregates, int32_t precision, double *pred_out);

/* ---- scoring ----------------------------------------------------------- */
/* cost() for K candidates (simulator.py:143-145 over K fresh graphs).
 * Device pointers; asynchronous on `stream` (cudaStream_t, NULL = legacy).
 * ngid/rgid: [K*V], bkt: [K*A], cost_out: [K] fp64, status_out: [K] fo_status. */
int fo_score(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K,
             int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out, void *stream);
/* int16 encodings (gid_bound and A <= 32767): half the bytes in HBM and over PCIe. */
int fo_score_i16(fo_graph *g, const int16_t *ngid, const int16_t *rgid, const int16_t *bkt, int32_t K,
                 int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out, void *stream);
/* Same through host buffers (pinned or pageable): H2D, kernel, D2H, synchronous. */
int fo_score_host(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K,
                  int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out);
int fo_score_host_i16(fo_graph *g, const int16_t *ngid, const int16_t *rgid, const int16_t *bkt, int32_t K,
                      int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out);

/* simulate() of one candidate with its Timeline (simulator.py:53-140).
 * durations: NULL -> device cost model; else host fp64 durations in schedule
 * node order [groups by id | buckets by id] (custom CostProviders; negative
 * values -> FO_NEGATIVE_DURATION).  Event buffers are host arrays of
 * capacity 2V (compute) and A (comm); ids written are the caller's ids.
 * bad_node_out: first failing schedule node index (or -1). */
int fo_simulate(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t gid_bound,
                int32_t precision, const double *durations, int32_t *c_id, double *c_start, double *c_end,
                int32_t *n_compute, int32_t *b_id, double *b_start, double *b_end, int32_t *n_comm,
                double *makespan, int32_t *bad_node_out);

/* Per-node durations of one candidate as the device computes them
 * (_duration for every schedule node, simulator.py:62): dur_out [G+B] in node
 * order, n_groups_out = G.  Used for predict_fused parity (estimator.py:462). */
int fo_node_durations(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt,
                      int32_t gid_bound, int32_t precision, double *dur_out, int32_t *n_groups_out,
                      int32_t *bad_node_out);

/* ---- native batch-expand (rewrite.py:222-263, search.py:88-119) -------- */
/* Candidate k: random.Random(seeds[k]) then, for each enabled method in
 * (nondup, dup, ar), n = randint(0, beta) accumulating random_apply steps,
 * starting from the base state (NULL = unfused default).  Output states use
 * compact group ids < gid_bound_out (returned).  Host threads: n_threads. */
int fo_make_candidates(fo_graph *g, const int32_t *base_ngid, const int32_t *base_rgid, const int32_t *base_bkt,
                       const uint64_t *seeds, int32_t K, int32_t beta, int32_t methods_mask, int32_t n_threads,
                       int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out, int32_t *gid_bound_out);

/* Sparse (delta) candidates.  A candidate of a search or batch usually
 * differs from its parent in a handful of entries (13 of 1,505 at ResNet-50,
 * 10 of 101,000 at 50k ops), so the parent state stays resident on the
 * device and each candidate travels as (index, value) int32 pairs over the
 * concatenated ngid[V] | rgid[V] | bkt[A] index space.
 *   fo_set_parent         parent state (host arrays, any ids; ranked like the
 *                         engine's base state; NULL = unfused default)
 *   fo_make_candidates_delta   fo_make_candidates' batch as changes against
 *                         the same base: offsets_out[K+1], changes_out[2 * n]
 *                         (capacity cap_pairs pairs; offsets_out[K] = n even
 *                         when the capacity is too small -> FO_INVALID_ARG)
 *   fo_score_delta        device offsets / changes / outputs, async on stream
 *   fo_score_delta_host   host (pinned) buffers, synchronous
 * Indices within one candidate must be distinct. */
int fo_set_parent(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt);
int fo_make_candidates_delta(fo_graph *g, const int32_t *base_ngid, const int32_t *base_rgid, const int32_t *base_bkt,
                             const uint64_t *seeds, int32_t K, int32_t beta, int32_t methods_mask, int32_t n_threads,
                             int32_t *offsets_out, int32_t *changes_out, int64_t cap_pairs);
int fo_score_delta(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                   double *cost_out, int32_t *status_out, void *stream);
int fo_score_delta_host(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                        double *cost_out, int32_t *status_out);
/* fo_score_delta on scratch set `slot` (0 .. 3; 0 is fo_score_delta's): batches
 * on different slots may run concurrently on different streams.  clear_memo
 * empties the slot's memo table of this precision first (on `stream`).
 * Slots > 0 need groups that fit the estimator scratch (V <= 2048). */
int fo_score_delta_slot(fo_graph *g, int32_t slot, const int32_t *offsets, const int32_t *changes, int32_t K,
                        int32_t precision, int32_t clear_memo, double *cost_out, int32_t *status_out, void *stream);
/* Pipelined fo_score_delta_host for streams of batches: enqueues H2D of the
 * candidates (host buffers, pinned for overlap), [if clear_memo, an
 * fo_memo_clear of this precision's table], the score and the D2H of cost_out / status_out, and returns a
 * ticket.  Four submissions may be in flight, each on its own compute
 * stream with its own scratch and memo tables (consecutive batches overlap);
 * a fifth waits for the oldest.  Results are valid, and the input buffers reusable, after
 * fo_score_wait(g, ticket).  Same semantics per batch as
 * fo_score_delta_host (simulator.py:143-145 per candidate). */
int fo_score_delta_submit(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                          int32_t clear_memo, double *cost_out, int32_t *status_out, int64_t *ticket_out);
int fo_score_wait(fo_graph *g, int64_t ticket);

/* random_apply (rewrite.py:222-263) on one state in place, driven by a
 * CPython random.Random state: mt_state = getstate()[1] (624 words + index). */
int fo_random_apply(fo_graph *g, int32_t *ngid, int32_t *rgid, int32_t *bkt, int32_t method, int32_t n,
                    uint32_t *mt_state, int32_t *applied_out);
/* Every accepted single rewrite of a state in exhaustive_search's enumeration
 * order (search.py:185-206): nondup / dup per fusible pair, then AllReduce
 * fusion per bucket pair.  Outputs up to cap states; n_out = count. */
int fo_expand_all(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t cap,
                  int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out, int32_t *n_out);

/* ---- rewrite primitives (rewrite.py:49-219) ----------------------------- */
/* Ids are ranks of the state's group / bucket ids (0..G-1 / 0..B-1 in id
 * order).  fo_rewrite_pairs: kind 0 fusible_pairs, 1 fusible pairs after the
 * duplicate-fusion filter, 2 bucket_pairs, 3 every contracted (group,
 * predecessor) pair (graph.py:161-179); (a, b) pairs in the reference's
 * order into pairs_out[2 * cap]; n_out = count (FO_INVALID_ARG when cap is
 * short).  fo_rewrite_apply: method 0 fuse_nondup(a, b), 1 fuse_dup(a, b)
 * (a consumer, b predecessor group), 2 fuse_allreduce(a, b) (buckets; the
 * caller checks that b neighbours a); applied_out = 0 for a rejected rewrite,
 * else the state arrays are rewritten (engine ids). */
int fo_rewrite_pairs(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t kind,
                     int32_t *pairs_out, int32_t cap, int32_t *n_out);
int fo_rewrite_apply(fo_graph *g, int32_t *ngid, int32_t *rgid, int32_t *bkt, int32_t method, int32_t a, int32_t b,
                     int32_t *applied_out);

/* ---- heuristic baselines (search.py:228-302) ---------------------------- */
/* greedy_postorder_fusion (search.py:228-244): every op in reverse contracted
 * topological order; its normal group is non-duplicate-fused with the first
 * predecessor group (ascending id) whose rewrite is valid.  FO_CYCLE when the
 * input's group graph is cyclic. */
int fo_greedy_postorder(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt,
                        int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out);

/* topo_order (graph.py:536-556): the group ids (compact, as in ngid) in the
 * deterministic topological order of the contracted group graph -- Kahn's
 * algorithm, ties to the group with the smallest member op.  gid_out holds
 * one entry per group; *n_out receives the count.  FO_CYCLE when the
 * contracted graph is cyclic. */
int fo_topo_order(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t *gid_out,
                  int32_t *n_out);
/* threshold_allreduce_fusion (search.py:247-302): buckets scanned in production
 * order -- order[n_order] = bucket ids sorted by simulated start (the cp path,
 * search.py:264-267), or NULL for the contracted topological production key
 * (search.py:268-281) -- merging consecutive neighbours while the merged size
 * stays <= threshold_bytes (> 0, else FO_INVALID_ARG). */
int fo_threshold_ar(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int64_t threshold_bytes,
                    const int32_t *order, int32_t n_order, int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out);

/* Canonical fusion-state hash (equality semantics of canonical_hash, graph.py:559-580). */
int fo_state_hash(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K,
                  uint64_t *hash_out);

/* ---- backtracking search, lock-stepped seeds (search.py:84-155) -------- */
typedef struct {
    double alpha;
    int32_t beta, max_unchanged, methods_mask; /* bit 0 nondup, bit 1 dup, bit 2 ar */
    int32_t precision;                          /* FO_PREC_* for the estimator */
    int32_t n_threads;                          /* host threads for the batch-expand */
} fo_search_cfg;

typedef struct {
    int32_t step;
    int32_t method; /* 0 nondup, 1 dup, 2 ar */
    double cost_us, best_cost_us;
    int32_t queue_len;
    int32_t enqueued;
} fo_trace_rec;

typedef struct fo_search fo_search;
/* R independent searches (seeds[r]) from the same start state (NULL = default). */
int fo_search_create(fo_graph *g, const fo_search_cfg *cfg, const uint64_t *seeds, int32_t R,
                     const int32_t *ngid0, const int32_t *rgid0, const int32_t *bkt0, fo_search **out);
/* One round: every active search does one step of Alg. 1; all their
 * candidates are scored in ONE device batch.  active_out = searches still
 * running; best_out[R] / best_cost_out: per-search best costs after the round. */
int fo_search_round(fo_search *s, int32_t *active_out, double *best_cost_out);
/* The initial evaluation of the start state for every seed (search.py:101-102)
 * without a step -- idempotent; fo_search_round / _run call it too. */
int fo_search_start(fo_search *s, double *best_cost_out);
/* Run every search to completion (max_rounds <= 0: unbounded) natively.  With
 * R >= 2 the seeds run in two halves whose device batches overlap the other
 * half's host-side expand; each seed's step sequence is unchanged. */
int fo_search_run(fo_search *s, int64_t max_rounds, int32_t *active_out);
/* fo_search_run with a hook after every round (every seed advanced one step):
 * fn(ctx, round, active, best[R], R) with the seeds' best costs so far -- the
 * multi-GPU driver posts its per-round exchange from it.  A nonzero return
 * stops the run with FO_INVALID_ARG.  fn must not call back into this handle. */
typedef int32_t (*fo_round_fn)(void *ctx, int64_t round, int32_t active, const double *best, int32_t R);
int fo_search_run_cb(fo_search *s, int64_t max_rounds, fo_round_fn fn, void *ctx, int32_t *active_out);

/* ---- multi-GPU search exchange over NCCL (parallel.py ShardedSearch) ------
 * One communicator per rank (NCCL bound at run time).  An attached search
 * posts, every `every` rounds, its best (cost, global seed id) and live-seed
 * count -- one ncclAllGather of 3 doubles per rank on the exchange's stream,
 * waited `lag` exchanges late -- and every rank records the global best of
 * each exchange (strict <: lowest id among equal costs, search.py:124).
 * fo_xchg_finish (every rank, after its run) keeps posting 0-live exchanges
 * until all ranks are done, so all ranks post the same number. */
typedef struct fo_xchg fo_xchg;
int fo_xchg_unique_id(uint8_t *out128); /* rank 0; broadcast to the others */
int fo_xchg_create(const uint8_t *id128, int32_t rank, int32_t world, int32_t device, int32_t lag, fo_xchg **out);
int fo_xchg_attach(fo_search *s, fo_xchg *x, int64_t seed_offset, int32_t every);
int fo_xchg_finish(fo_xchg *x);
/* out2[2 * i] = global best cost of exchange i, out2[2 * i + 1] its seed id */
int fo_xchg_history(fo_xchg *x, double *out2, int64_t cap, int64_t *n_out);
int fo_xchg_destroy(fo_xchg *x);
/* Counters: steps, candidates_evaluated, candidates_enqueued, trace length. */
int fo_search_result(fo_search *s, int32_t r, double *best_cost, int64_t *counters4, int32_t *best_ngid,
                     int32_t *best_rgid, int32_t *best_bkt, fo_trace_rec *trace, int64_t trace_cap);
/* Per-round device time (ms) of the scoring kernels and host expand time (ms). */
int fo_search_timing(fo_search *s, double *device_ms, double *expand_ms, int64_t *scored);
/* Rounds (device batches of lock-stepped steps) executed so far by
 * fo_search_round / fo_search_run. */
int fo_search_rounds(fo_search *s, int64_t *rounds_out);
int fo_search_destroy(fo_search *s);

/* ---- misc -------------------------------------------------------------- */
const char *fo_last_error(void);
/* Device kernel launches issued by this process (for the bench's gpu_launches). */
int64_t fo_kernel_launches(void);
/* Measurement hook (phase timing in bench.py): subsequent launches on g return
 * after K1 contraction (phase 1) or K2 estimation (phase 2) with cost 0 /
 * status OK; 0 restores full scoring. */
int fo_set_phase_stop(fo_graph *g, int32_t phase);
/* Sparse-candidate scoring mode: 1 (default) scores each candidate as a patch
 * of the resident parent's contracted DAG (incremental kernel, MP estimator
 * with profile lookups; anything else falls back per candidate), 0 always
 * runs the general kernel.  Results are identical; for A/B measurement.
 * 2 is diagnostic: incremental kernel only, candidates it would hand to the
 * general kernel keep status 101. */
int fo_set_delta_mode(fo_graph *g, int32_t mode);
/* Event-loop fast-forward counters of the incremental kernel, accumulated
 * over mode-2 launches since the last call (then reset; synchronizes the
 * device): out6 = {candidates that reached the event loop, candidates that
 * started from a parent snapshot, parent iterations skipped in total, the
 * parent loop's iterations, snapshots held, iterations between snapshots}
 * for the plan of this precision. */
int fo_inc_stats(fo_graph *g, int32_t precision, int64_t *out6);
/* Arithmetic of the FP32 message-passing layer transforms (estimator.py:375):
 * 0 FP32 FFMA (default), 1 TF32 tensor cores (mma.sync m16n8k8), 2 3xTF32
 * tensor cores (split operands).  The FP64 estimator is unaffected.  The
 * estimator memo is per handle: empty it when switching. */
int fo_set_estimator_arith(fo_graph *g, int32_t mode);
/* Introspection: the launch geometry a K-candidate batch takes (before the
 * workspace cap): out4 = {block-per-candidate (1) or warp-per-candidate (0),
 * grid, resident blocks per SM, shared-memory arena bytes per candidate}. */
int fo_score_geometry(fo_graph *g, int32_t K, int32_t precision, int32_t *out4);

#ifdef __cplusplus
}
#endif
#endif /* DISCO_B200_H */
