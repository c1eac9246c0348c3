/*
 * sw_plan.h -- C ABI of the B200-native StreamWise plan evaluator (libsw_plan.so).
 *
 * The library evaluates, in batch on B200 GPUs, every candidate serving plan of
 * one podcast-video request: per scene (or block of scenes) a quality level, a
 * parallelism degree k and a GPU pool.  It scores each with the paper's
 * latency/cost model and reduces the results to SLO/budget-constrained winners
 * and a 3-D Pareto front.  Citations: P:n = arXiv 2603.05800 PAPER.md line n,
 * SPEC = the spec written from it, R<n> = readings listed in DESIGN.md.
 *
 *   - the estimator the paper's provisioner runs per setting: "For each setting,
 *     we use the greedy algorithm to estimate the latency and cost";
 *     a greedy DAG simulation with deadline-ordered scenes
 *     (P:970), shortest-expected-runtime instance choice,
 *     adaptive per-scene quality, USP parallel degree;
 *   - objective, SLO steering and "closest solution", the
 *     latency/cost/quality Pareto frontier;
 *   - metrics TTFF / TTFF_eff, Table 3 prices.
 *
 * Conventions (every entry point):
 *   - No exceptions cross the ABI; every call returns an sw_status.  Negative =
 *     error (nothing changed unless stated), 0 = OK, positive = soft status.
 *     The library never exits the process.  sw_last_error() gives a message.
 *   - All pointer arguments of sw_plan_create are HOST pointers; create deep-
 *     copies them (the caller may free them on return) and uploads them once.
 *   - A handle owns its device tables, record buffer, Pareto front and scratch
 *     (allocated with cudaMallocAsync on its stream, or the caller's allocator;
 *     with the default allocator, create sets the device's default memory pool
 *     release threshold to UINT64_MAX so freed blocks stay pooled).
 *   - eval is asynchronous on the handle's stream; select / pareto_get / digest /
 *     detail synchronise that stream and write caller HOST memory.
 *   - Multi-GPU: with nranks > 1 every rank makes the same call sequence with the
 *     same arguments (like NCCL); eval takes the GLOBAL index range and shards it
 *     internally; select / pareto_get / digest are collectives over nccl_comm.
 *   - A handle is not thread-safe; distinct handles are independent.
 *   - Integer semantics everywhere: times in microseconds (u64), money in
 *     milli-cents (u64), quality in ms x score (u32).  Results are bit-exact
 *     and independent of grid size, rank count and range splitting.
 */
#ifndef SW_PLAN_H
#define SW_PLAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sw_plan sw_plan; /* opaque: one request's plan space on one rank */
typedef int32_t sw_status;

enum {
    SW_OK = 0,
    SW_CLOSEST = 1,   /* no feasible plan: the closest one is returned (SPEC exit 2) */
    SW_TRUNCATED = 2, /* output buffer too small; *n_out holds the required count */
    SW_EMPTY = 3,     /* nothing evaluated yet (no records in the handle) */
    SW_EINVAL = -1,   /* bad argument / shape: k > G_p, heads % k != 0, S = 0, duration 0,
                         G_p > SW_MAX_GPUS_PER_POOL, overlapping eval range, ... */
    SW_ERANGE = -2,   /* space size >= 2^63, an overflow bound fails, or records exceed
                         record_capacity (SPEC "InstanceTooLarge") */
    SW_ENOMEM = -3,
    SW_ECUDA = -4,
    SW_ENCCL = -5,    /* a collective failed, a peer rank reported an asynchronous NCCL
                         error, or a wait exceeded SW_NCCL_TIMEOUT_S seconds (default 600):
                         the communicator is then aborted (do not use it again) */
    SW_ESTATE = -6 /* wrong call order or handle misuse; multi-rank: the ranks made
                      different collective calls (arguments or evaluated ranges differ),
                      detected on every rank */
};

#define SW_MAX_SCENES 64
#define SW_MAX_DIGITS 16
#define SW_MAX_CHOICES 64          /* per digit */
#define SW_MAX_POOLS 4
#define SW_MAX_GPUS_PER_POOL 32 /* <= 8: lane-per-prefix fast path; 9..32: the warp-per-candidate
                                   generic path (no fused stream mode, no greedy planner) */
#define SW_MAX_QUERIES 8           /* per sw_plan_select_batch call */

/* Scene list: the refined DAG of one request, scenes in playback order. */
typedef struct {
    uint32_t n_scenes;          /* S, 1..SW_MAX_SCENES */
    const uint64_t *dur_us;     /* [S] playback duration of each scene, > 0 */
    const uint64_t *llm_us;     /* [S] screenplay (LLM) time per scene (Table 4 Gemma) */
    const uint64_t *tts_us;     /* [S] audio (TTS) time per scene (Table 4 Kokoro) */
    uint64_t overhead_us;       /* front end before the LLM starts (Table 4 StreamCast) */
    uint32_t scene0_static;     /* 1: scene 0 is a static intro, no GPU work */
    uint64_t static_ready_us;   /* its ready time (e.g. 500 ms) */
} sw_scene_list;

/* One choice of a digit: applied to every scene of the digit's block. */
typedef struct {
    uint8_t level;   /* index into level_score */
    uint8_t degree;  /* k GPUs (USP degree); must divide heads.
                        0 = the STATIC rung: no video stage and no GPU, the scene is
                        ready with its text and audio, R_s = a_s ("If not enough, we
                        switch to static content"; reading R33);
                        pair it with a level whose score is 0 (R12) */
    uint8_t pool;    /* GPU pool index (< n_pools; unused by a STATIC choice) */
    uint8_t vae;     /* 0: the VAE runs inside the V+A stage (R1).  v + 1: FramePack-style
                        DiT/VAE disaggregation, "FramePack DiT streams latent outputs to the
                        VAE for decoding ... pipelined execution, independent scaling"
                        (reading R37): the V+A stage is the DiT (k GPUs of `pool`)
                        and a separate VAE stage runs on pool v, one GPU (the VAE is not
                        parallelised), as soon as the scene's DiT finished and a GPU
                        of pool v is free; needs tables->vae_us */
} sw_choice;

/* Profiled tables (on-boarding profiles) expanded per candidate choice.
 * Digit b covers scenes [first_scene[b], first_scene[b+1]); blocks are contiguous,
 * start at scene scene0_static and end at S.  Index order: MSD = earliest block (R19). */
typedef struct {
    uint32_t n_digits;          /* B, 1..SW_MAX_DIGITS */
    const uint32_t *radix;      /* [B] r_b, 1..SW_MAX_CHOICES */
    const uint32_t *first_scene;/* [B+1] */
    const sw_choice *choices;   /* [sum r_b] concatenated per digit */
    const uint64_t *va_us;      /* V+A stage time, block-major: digit b, scene s in
                                   block, choice c -> va_us[off_b + (s-first_b)*r_b + c], >= 1
                                   (= 0 exactly for STATIC choices, else SW_EINVAL) */
    uint32_t n_levels;
    const uint32_t *level_score;/* [n_levels] quality score per level (R12) */
    uint32_t heads;             /* attention heads for the divisibility check;
                                   0 = no check */
    const uint64_t *vae_us;     /* NULL, or laid out like va_us: the VAE stage time of each
                                   (scene, choice) with a VAE stage (1 .. 2^32 - 1 us), 0 for
                                   the others (R37) */
} sw_profile_tables;

/* Pools and prices (Table 3) in integer milli-cents per GPU-hour. */
typedef struct {
    uint32_t n_pools;                       /* 1..SW_MAX_POOLS */
    const uint32_t *gpus;                   /* [n_pools] G_p, 1..SW_MAX_GPUS_PER_POOL */
    const uint64_t *price_mc_per_gpu_hour;  /* [n_pools] reserved or spot column */
    uint64_t fixed_cost_mc;                 /* LLM/TTS instances */
    uint32_t billing;    /* 0 RESERVED: G_p x pool span (GPU idle time billed);
                            1 BUSY: sum k x t (GPU-seconds) -- reading R10 */
    uint32_t objective;  /* 0 QUALITY_FIRST: (-Q, cost, ttff_eff, index);
                            1 COST_X_TTFF: (cost x ttff_eff, -Q, index) -- R13 */
    const uint64_t *pool_ready_us;  /* [n_pools] or NULL: time at which every GPU of pool p
                            is free -- model load + warm-up, "~30 seconds ... ~80 seconds"
                            (reading R31); NULL = all 0
                            (warm pools, R18).  An unused pool is neither billed nor
                            counted in the makespan. */
    const uint32_t *evict_risk_permille;  /* [n_pools] or NULL: Spot eviction risk rho_p of
                            pool p over the request, in 1/1000 (0 <= rho_p < 1000).  "We
                            proportionally increase the number of allocated resources to the
                            eviction risk" ("ceil(replicas /
                            (1 - risk))"; reading R32): pool p is billed for
                            G'_p = ceil(G_p * 1000 / (1000 - rho_p)) GPUs while the schedule
                            runs on G_p (the spares stand by for evicted GPUs).  Pair it with
                            the Spot column of Table 3.  RESERVED billing only: a non-zero
                            rho_p with BUSY billing is SW_EINVAL.  NULL = all 0. */
    uint32_t metric;     /* 0: records carry cost in milli-cents (the prices above).
                            1: ENERGY in microjoules instead ("optimizing for energy,
                            TTFF, and other combinations (e.g., Energy x TTFF)"; P:701-724;
                            reading R38): busy GPUs draw power_active_w, a pool's other rented
                            GPUs power_idle_w until its last finish (RESERVED; BUSY: busy time
                            only); fixed_cost_mc is then the fixed stages' energy (uJ), query
                            budgets are energy budgets, and COST_X_TTFF minimises Energy x
                            TTFF_eff.  Record field cost_mc holds the energy. */
    const uint32_t *power_active_w; /* [n_pools] (metric 1): busy GPU power, W (the TDP) */
    const uint32_t *power_idle_w;   /* [n_pools] (metric 1): idle GPU power, W */
} sw_price_table;

typedef void *(*sw_alloc_fn)(size_t bytes, void *stream, void *ctx);
typedef void (*sw_free_fn)(void *ptr, void *stream, void *ctx);

typedef struct {
    int32_t device;           /* CUDA device ordinal */
    void *stream;             /* cudaStream_t to run on; NULL = the handle creates one */
    void *nccl_comm;          /* ncclComm_t (from sw_comm_init) or NULL when nranks == 1 */
    int32_t rank, nranks;
    uint64_t record_capacity; /* records retained per rank; 0 = this rank's share of
                                 the whole space */
    sw_alloc_fn alloc;        /* NULL = cudaMallocAsync on the stream */
    sw_free_fn free;
    void *alloc_ctx;
} sw_runtime;

/* Per-candidate record, 32 B, the HBM traffic of the eval kernel. */
typedef struct {
    uint64_t ttff_us;     /* time to first frame */
    uint64_t stall_us;    /* ttff_eff - ttff: total playback pause (R8) */
    uint64_t cost_mc;     /* milli-cents */
    uint32_t quality;     /* sum over scenes of duration_ms x level score (R12) */
    uint16_t stall_count; /* rebuffering events: new strict maxima of R_s - P_s, s >= 1 */
    uint8_t flags;        /* bit p: pool p used */
    uint8_t pad;
} sw_record;

typedef struct {
    uint64_t slo_startup_us; /* feasible iff ttff <= slo_startup  (UINT64_MAX = none) */
    uint64_t slo_stall_us;   /*          and stall <= slo_stall */
    uint64_t budget_mc;      /*          and cost <= budget */
} sw_query;

/* A selected plan with its full metrics (recomputed on the GPU from its index). */
typedef struct {
    int32_t status;                 /* SW_OK, SW_CLOSEST or SW_EMPTY */
    uint32_t pad;
    uint64_t index;                 /* global candidate index */
    sw_record rec;
    uint64_t ttff_eff_us;           /* max_s (R_s - P_s) */
    uint64_t makespan_us;           /* last finish over pools and scene 0 */
    uint64_t pool_end_us[SW_MAX_POOLS];
    uint8_t digit[SW_MAX_DIGITS];   /* decoded choice per digit */
} sw_selection;

typedef struct {
    uint64_t index, ttff_eff_us, cost_mc;
    uint32_t quality, pad;
} sw_pareto_point;

/* ---- lifecycle ---------------------------------------------------------- */

/* Validate inputs, check overflow bounds (R25), upload and pack the tables on the
 * device (fixed-stage ready times a_s and deadlines P_s are computed there), and
 * allocate the record buffer.  EINVAL / ERANGE / ENOMEM / ECUDA; *out untouched
 * on error. */
sw_status sw_plan_create(const sw_profile_tables *tables, const sw_scene_list *scenes,
                         const sw_price_table *prices, const sw_runtime *rt, sw_plan **out);
sw_status sw_plan_destroy(sw_plan *h);
/* Drop all records and the running Pareto front (the tables stay). */
sw_status sw_plan_reset(sw_plan *h);
/* Chunked sweeps: fold every evaluated record into the running Pareto front, then
 * drop the records (the front persists; later evals append to it). */
sw_status sw_plan_release_records(sw_plan *h);

/* N = prod r_b (the number of candidate plans). */
sw_status sw_plan_space_size(const sw_plan *h, uint64_t *n);

/* ---- evaluation (a1-a8) --------------------------------------------------- */

/* Evaluate global candidates [begin, end): this rank's shard is decoded, scored and
 * its 32 B records stored; the shard is folded into the running Pareto front.
 * Asynchronous on the handle's stream.  EINVAL if the range is outside [0,N) or
 * overlaps one evaluated before; ERANGE if the records would exceed capacity. */
sw_status sw_plan_eval(sw_plan *h, uint64_t begin, uint64_t end);

/* ---- reductions (a9, a10) ------------------------------------------------- */

/* Constrained argmin over every record evaluated since create/reset (all ranks).
 * Returns SW_OK with the winner, SW_CLOSEST with the closest plan when nothing is
 * feasible, SW_EMPTY when nothing was evaluated.  Collective when nranks > 1. */
sw_status sw_plan_select(sw_plan *h, uint64_t slo_startup_us, uint64_t slo_stall_us,
                         uint64_t budget_mc, sw_selection *out);

/* Several queries in one pass over the records (n_queries <= SW_MAX_QUERIES);
 * out[q].status per query.  Return value: the worst soft status, or an error. */
sw_status sw_plan_select_batch(sw_plan *h, uint32_t n_queries, const sw_query *queries,
                               sw_selection *out);

/* Chunked sweep of global candidates [begin, end) for spaces larger than the record
 * buffer (C5: 1.2e10 plans = 391 GB of records): for each chunk of `chunk` global
 * candidates (0 = as many as record_capacity allows on every rank), eval -> one fused
 * select + Pareto-fold scan -> (optional) digest -> records dropped.  Per-query
 * winners of the chunks are merged with the query's total order (sw_selection_merge)
 * into out[0, n_queries); the running Pareto front persists (sw_pareto_get after);
 * *digest (may be NULL) receives the digest of [begin, end).  The handle must hold no
 * records (fresh, reset or released) -- else SW_ESTATE; n_queries may be 0 (front
 * and digest only).  Collective when nranks > 1.  Returns the worst soft status. */
sw_status sw_plan_sweep(sw_plan *h, uint64_t begin, uint64_t end, uint64_t chunk,
                        uint32_t n_queries, const sw_query *queries, sw_selection *out,
                        uint64_t *digest);


/* Fused streaming evaluation of global candidates [begin, end) (
 * BJ (4)): every candidate is decoded, scored (a1-a6) and handed from
 * registers straight to the select predicate (a9) and the Pareto DLT filter (a8) inside
 * one kernel per strided tile pass -- NO records are stored (no record capacity used),
 * for spaces beyond HBM and the lowest latency.  Winners of the n_queries queries over
 * [begin, end) (all ranks) go to out[0, n_queries) exactly as sw_plan_select_batch would
 * report them; the range is folded into the running Pareto front (sw_pareto_get).  The
 * handle must hold no records (else SW_ESTATE); records cannot be inspected afterwards.
 * SW_ERANGE if a pass's DLT survivors or a query's reported candidates exceed the
 * handle's buffers (sw_plan_sweep then gives the same results through records).
 * Synchronous; collective when nranks > 1.  Returns the worst soft status. */
sw_status sw_plan_stream(sw_plan *h, uint64_t begin, uint64_t end, uint32_t n_queries,
                         const sw_query *queries, sw_selection *out);

/* The running 3-D Pareto front over (ttff_eff min, cost min, quality max), exact
 * duplicates keeping the lowest index (R14), sorted by (ttff_eff asc, cost asc,
 * quality desc, index asc).  Two-call idiom: cap = 0 returns *n_out; a short
 * buffer returns SW_TRUNCATED with *n_out = the required count.  Collective. */
sw_status sw_pareto_get(sw_plan *h, sw_pareto_point *out, uint64_t cap, uint64_t *n_out);

/* Order-independent 64-bit digest of all records evaluated (all ranks):
 * sum_i mix64(i ^ rotl(ttff,7) ^ rotl(stall,19) ^ rotl(cost,31) ^
 * (flags<<48 | quality<<16 | stall_count)) mod 2^64.  Collective. */
sw_status sw_plan_digest(sw_plan *h, uint64_t *digest);

/* Full metrics of any candidate (GPU kernel), e.g. to inspect a what-if plan.
 * ready_us may be NULL or point to S entries (scene ready times R_s). */
sw_status sw_plan_detail(sw_plan *h, uint64_t index, sw_selection *out, uint64_t *ready_us);

/* Zero-copy view of this rank's records: the device pointer of the record buffer and
 * *n = the record SLOTS in use.  Records are stored in a TILED layout: an
 * eval call (a "segment", see sw_plan_segments) covers whole tiles of 32 rows of `row`
 * candidates; the record of global index i = H * row + j (row H, in-row offset j) of a
 * segment sits at slot  offset + ((H / 32 - tile0) * row + j) * 32 + H % 32.  Slots of a
 * segment's first / last tile outside [shard_begin, shard_end) are padding (undefined). */
sw_status sw_plan_records(const sw_plan *h, const sw_record **dev_ptr, uint64_t *n);

/* Segment table of this rank's records (one entry per eval call since create/reset/
 * release), for consumers of the zero-copy view.  Two-call idiom as sw_pareto_get. */
typedef struct {
    uint64_t global_begin, global_end;  /* the eval call's global range */
    uint64_t shard_begin, shard_end;    /* this rank's candidates of it */
    uint64_t offset;                    /* record slot of the segment's first tile */
    uint64_t tile0, ntiles;             /* tiles of 32 rows covering the shard */
    uint64_t row;                       /* candidates per row */
} sw_segment;
sw_status sw_plan_segments(const sw_plan *h, sw_segment *out, uint64_t cap, uint64_t *n_out);

/* Host helper: the digit (choice index within its digit's list) of candidate `index`
 * for every scene, choice_per_scene[S] (a static intro scene gets 0).  Mixed-radix,
 * MSD = earliest block (R19).  EINVAL if index >= N.  No device work. */
sw_status sw_plan_decode(const sw_plan *h, uint64_t index, uint8_t *choice_per_scene);
/* Copy n records starting at GLOBAL index `index` (must lie in one evaluated local
 * segment) into host memory. */
sw_status sw_plan_copy_records(sw_plan *h, uint64_t index, uint64_t n, sw_record *host_out);

/* ---- greedy + iterative refinement planner ------------ */

/* The paper's provisioner on the batched evaluator: start from the
 * cost-efficient baseline (start_index = UINT64_MAX: per digit the choice with the
 * smallest (level score, k, pool price)) or from start_index (a warm start,
 * P:1341), then repeatedly evaluate every single-digit change in parallel (one GPU
 * thread each) and move to the best one under the query's total order (R13)
 * while it is strictly better; stop at a local optimum (reading R28).  Needs no
 * records (runs on the tables).  *out = the plan with full detail; status SW_OK
 * (feasible) or SW_CLOSEST; *iterations = moves made, *evaluations = plans evaluated
 * (either may be NULL).  Synchronises; replicated (no collective) when nranks > 1. */
sw_status sw_plan_greedy(sw_plan *h, uint64_t slo_startup_us, uint64_t slo_stall_us,
                         uint64_t budget_mc, uint64_t start_index, sw_selection *out,
                         uint32_t *iterations, uint64_t *evaluations);

/* ---- host-only helpers (no device needed) ---------------------------------- */

/* Size of the plan space N = prod r_b and the row size (candidates per eval-kernel
 * thread: the product of the last two digits' radices, digits left-padded with
 * radix 1 to B >= 3) of a profile table, without creating a handle.  Only
 * tables->n_digits and tables->radix are read.  EINVAL on a bad shape, ERANGE when
 * N >= 2^63. */
sw_status sw_space_shape(const sw_profile_tables *tables, uint64_t *n, uint64_t *row);

/* Device memory of destroyed handles stays cached in the device's default stream-ordered
 * memory pool (the library allocates with cudaMallocAsync), so that re-creating a handle
 * of the same shape maps no new memory.  sw_trim_device_memory synchronises the device
 * and returns the cached, unused part of that pool to the driver (cudaMemPoolTrimTo 0), so
 * that cudaMemGetInfo shows it as free again -- e.g. before sizing a record capacity from
 * free memory.  Memory of live handles is untouched.  ECUDA on a CUDA error. */
sw_status sw_trim_device_memory(int32_t device);

/* Associative, commutative merge of two selections of the SAME query (q) over
 * disjoint candidate sets, e.g. the winners of successive chunks of a chunked sweep
 * (eval -> select -> release_records, R13) or of independent handles.  *out = the
 * better of *a and *b under the query's total order (R13): feasible plans
 * by the objective key (objective as in sw_price_table), else the closest plan by
 * (startup+stall violation, budget violation, key), the lower index breaking ties;
 * an SW_EMPTY input loses.  out->status is recomputed (SW_OK feasible, SW_CLOSEST
 * not, SW_EMPTY if both are empty) and returned.  out may alias a or b.  Host only. */
sw_status sw_selection_merge(uint32_t objective, const sw_query *q, const sw_selection *a,
                             const sw_selection *b, sw_selection *out);

/* ---- fleet batch (BASELINE configs[3], C4) -------------------------------- */

/* A batch of independent requests (e.g. 256 podcasts of 5-15 min, each with its own SLO
 * and budget) evaluated and selected together: sw_fleet_eval is ONE kernel launch over
 * every request's whole plan space (each request's records in its own handle),
 * sw_fleet_select ONE scan launch with one query per request, a merge kernel, a batched
 * winner-detail kernel and, with nranks > 1, ONE allgather of the n winners (every
 * request's space is sharded over the ranks like sw_plan_eval).  Each request keeps a
 * full sw_plan handle (sw_fleet_plan: Pareto front, digest, records, detail), owned by
 * the fleet.  Arrays of sw_fleet_create have n entries (host, deep-copied); the runtime
 * is shared (record_capacity applies per request). */
typedef struct sw_fleet sw_fleet;
#define SW_MAX_FLEET 4096
sw_status sw_fleet_create(uint32_t n, const sw_profile_tables *tables, const sw_scene_list *scenes,
                          const sw_price_table *prices, const sw_runtime *rt, sw_fleet **out);
sw_status sw_fleet_destroy(sw_fleet *f);
sw_status sw_fleet_size(const sw_fleet *f, uint32_t *n);
/* Borrowed handle of request i (valid until sw_fleet_destroy; do not destroy it). */
sw_status sw_fleet_plan(sw_fleet *f, uint32_t i, sw_plan **out);
/* Evaluate every request's whole space (this rank's shard of each); asynchronous.
 * Handles must hold no records (fresh or sw_fleet_reset) -- else SW_ESTATE. */
sw_status sw_fleet_eval(sw_fleet *f);
/* queries[i] selects request i's winner into out[i] (status per request as in
 * sw_plan_select).  Collective when nranks > 1; synchronises; returns the worst soft
 * status.  The Pareto fronts are folded lazily by sw_pareto_get on sw_fleet_plan(i). */
sw_status sw_fleet_select(sw_fleet *f, const sw_query *queries, sw_selection *out);
sw_status sw_fleet_reset(sw_fleet *f);
/* As sw_plan_kernel_time, for the fleet-wide launches. */
sw_status sw_fleet_kernel_time(sw_fleet *f, uint32_t kind, uint64_t *n_launches, double *total_ms,
                               uint64_t *bytes);
uint64_t sw_fleet_launch_count(const sw_fleet *f);

/* ---- shared-pool fleet (reading R36) ------------------ */

/* Several requests contend for the SAME GPU pools.  "To coordinate multiple requests,
 * model instances maintain local queues that prioritize tasks by deadline ... an early
 * scene from a new request before a later scene from an earlier request if it has a
 * tighter deadline"; heterogeneous SLOs -- real-time, 50% relaxed, batch --
 * let the scheduler "prioritize real-time requests".  Reading R36: request r
 * arrives at arrival_us; its scene s is released at arrival + a_s (its own LLM/TTS) and
 * due at arrival + slo_startup_us + P_s (UINT64_MAX: batch); every pool is an online,
 * non-preemptive EDF queue of gang tasks (the head = smallest (deadline, request, scene)
 * among released tasks takes the k earliest-free GPUs; a more urgent task released
 * before the head can start takes the decision).  A request with fixed_index != UINT64_MAX
 * is background load with that fixed plan; the others are FREE and their plans are
 * enumerated jointly (joint index: mixed radix over the free requests' digits, MSD = the
 * first free request's first digit).  The fleet RECORD of a joint plan:
 *   ttff_us  = max_r sat(ttff_r - slo_startup_r)  (worst startup lateness; ttff_r relative
 *              to the request's arrival)
 *   stall_us = max_r sat(stall_r - slo_stall_r)   (worst stall lateness)
 *   cost_mc  = sum_r fixed_cost_mc[r] + sum_p pool cost over the fleet (billing of pools)
 *   quality = sum_r Q_r, stall_count = sum_r count_r, flags = pools used,
 * so sw_plan_select(h, 0, 0, budget) finds the best joint plan meeting EVERY request's SLO
 * within the fleet budget (closest = least lateness).
 * The result is an ordinary sw_plan handle (row = 1): eval / select / select_batch / sweep /
 * sw_pareto_get / digest / records / detail / reset work unchanged (detail: the fleet
 * record, pool ends, joint digits); stream and greedy are SW_EINVAL.  Limits: <= 16
 * requests, <= 128 scenes in all, <= 16 joint digits.  tables/scenes/fixed_cost_mc/reqs
 * have n entries (host, deep-copied); pools gives the shared pools (n_pools, gpus, prices,
 * billing, objective, pool_ready_us; no eviction risk) -- every request's choices index
 * them.  Collective like sw_plan_create when nranks > 1 (the joint space is sharded). */
typedef struct {
    uint64_t arrival_us;      /* T0_r */
    uint64_t slo_startup_us;  /* deadline base and startup SLO (UINT64_MAX: batch) */
    uint64_t slo_stall_us;    /* stall SLO */
    uint64_t fixed_index;     /* background plan, or UINT64_MAX = free (enumerated) */
} sw_shared_request;
sw_status sw_shared_create(uint32_t n, const sw_profile_tables *tables, const sw_scene_list *scenes,
                           const uint64_t *fixed_cost_mc, const sw_shared_request *reqs,
                           const sw_price_table *pools, const sw_runtime *rt, sw_plan **out);
/* Per-request metrics of joint candidate `index`: per_request[n] = (ttff, stall relative to
 * the request's arrival, cost = its fixed cost, quality, stall count, flags 0) and, if
 * ready_abs is not NULL, the absolute ready time of every scene, request-major. */
sw_status sw_shared_detail(sw_plan *h, uint64_t index, sw_record *per_request, uint64_t *ready_abs);

/* ---- multi-GPU --------------------------------------------- */

/* Row-aligned contiguous shard of [begin, end) for `rank` of `nranks`: whole rows
 * of `row` candidates are split evenly, a ragged head goes to rank 0 and a ragged
 * tail to rank nranks-1.  Pure host arithmetic on indices. */
sw_status sw_shard_range(uint64_t begin, uint64_t end, uint64_t row, int32_t rank,
                         int32_t nranks, uint64_t *shard_begin, uint64_t *shard_end);
/* Candidates per row of this plan (the unit the eval kernel gives one thread). */
sw_status sw_plan_row_size(const sw_plan *h, uint64_t *row);

/* NCCL bootstrap: rank 0 creates a 128-byte unique id, the caller broadcasts it
 * (e.g. torch.distributed), every rank calls sw_comm_init on its device. */
sw_status sw_comm_unique_id(void *id128);
sw_status sw_comm_init(const void *id128, int32_t rank, int32_t nranks, int32_t device,
                       void **comm_out);
/* Destroys an NCCL communicator of sw_comm_init (one the library aborted after
 * SW_ENCCL is only forgotten) or a loopback rank (the group goes with its last rank). */
sw_status sw_comm_destroy(void *comm);
/* TEST/EMULATION: an in-process loopback group of nranks ranks.  comms_out[r] is passed
 * as sw_runtime.nccl_comm of rank r's handle (rank = r, nranks = nranks); each rank is
 * driven by its own host thread making the same call sequence, and all ranks may live on
 * ONE device (NCCL refuses duplicate GPUs).  The collectives (allgather / allreduce) are
 * enqueued on each handle's stream with NCCL's ordering (peers' send buffers are read
 * after the work that wrote them; later writes wait for the peers' copies), so the
 * multi-rank device merge path runs unchanged.  Destroy each rank with sw_comm_destroy. */
sw_status sw_comm_loopback_create(int32_t nranks, void **comms_out);

/* ---- diagnostics ------------------------------------------------------------ */
const char *sw_status_str(sw_status s);
const char *sw_last_error(const sw_plan *h); /* h may be NULL: last global error */
/* Number of kernels this handle launched since create (for the bench's claim). */
uint64_t sw_plan_launch_count(const sw_plan *h);
/* Per-launch eval-kernel time of the last sw_plan_eval on this rank (CUDA events
 * recorded on the handle's stream around the eval kernel), milliseconds. */
sw_status sw_plan_last_eval_ms(sw_plan *h, float *ms);
/* Launch statistics of one kernel kind since create: launches, their summed
 * CUDA-event time (ms; events recorded on the handle's stream around each launch) and
 * their ALGORITHMIC bytes (32 B per record written by eval / read by a scan, tile
 * padding included for scans).  Synchronises the last recorded launch. */
enum {
    SW_KERNEL_EVAL = 0,   /* eval_kernel: a1-a7 */
    SW_KERNEL_SCAN = 1,   /* scan_kernel: a8+a9 */
    SW_KERNEL_STREAM = 2  /* stream_kernel: a1-a6 + a8 filter + a9, no records (bytes: 0) */
};
sw_status sw_plan_kernel_time(sw_plan *h, uint32_t kind, uint64_t *n_launches, double *total_ms,
                              uint64_t *bytes);
int32_t sw_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SW_PLAN_H */
