/*
 * oracle/sw_oracle.c -- CPU ORACLE for the StreamWise batched plan evaluator.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg / `--impl reference` arm may load, call or link this file.
 * The product path (paper_2603_05800_b200/) never imports it and shares no
 * code, header, table or helper with it; the only shared artefact is the
 * seeded input generator (swgen/), which holds none of the method's arithmetic.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md):
 *   - fixed-stage ready times a_s: LLM streams scenes in order and each finished
 *     scene triggers its downstream stages; one FIFO TTS server
 *     (Table 4; readings R2/R3);
 *   - per-scene V+A max-plus step on the k earliest-free GPUs of the chosen pool
 *     (greedy DAG simulation P:898-900, EDF/scene order P:970 P:983-986,
 *     shortest expected runtime P:990, parallel degree P:588-596, adaptive
 *     quality per scene P:994-997);
 *   - playback metrics: TTFF, TTFF_eff = max over scenes of
 *     ready - deadline (scene-granular deadlines P:338-341), stall
 *     = TTFF_eff - TTFF (reading R8);
 *   - a STATIC rung (degree k = 0): no video stage and no GPU, R_s = a_s (P:997,
 *     P:823-825; reading R33);
 *   - cost from Table 3 prices billed per pool (reading R10);
 *     Spot pools over-provisioned by eviction risk (reading R32);
 *   - quality = sum of duration_ms x level score (R12);
 *   - constrained selection: objective, SLO steering and "closest solution"
 *     when infeasible (reading R13);
 *   - 3-D Pareto front over (ttff_eff, cost, quality) (R14);
 *   - an order-independent record digest (test tool).
 *
 * Every candidate is evaluated independently by FULL RECOMPUTE from its linear
 * index; reductions are naive.  Nothing is blocked, fused or reordered.
 * Parity pins: see tests/test_oracle_pins.py (every function below is pinned).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    uint32_t S;                       /* scenes */
    const uint64_t *dur_us;           /* [S] scene durations (us) */
    const uint64_t *llm_us;           /* [S] LLM (screenplay) time per scene */
    const uint64_t *tts_us;           /* [S] TTS time per scene */
    uint64_t overhead_us;             /* StreamCast front end before the LLM */
    uint32_t scene0_static;           /* 1: scene 0 is a static intro */
    uint64_t static_ready_us;         /* its ready time */
    uint32_t n_pools;
    const uint32_t *gpus;             /* [n_pools] GPUs per pool */
    const uint64_t *price_mc;         /* [n_pools] milli-cents per GPU-hour */
    uint64_t fixed_cost_mc;           /* LLM/TTS instances */
    uint32_t billing;                 /* 0 RESERVED, 1 BUSY */
    uint32_t objective;               /* 0 QUALITY_FIRST, 1 COST_X_TTFF */
    uint32_t n_levels;
    const uint32_t *level_score;      /* [n_levels] */
    uint32_t B;                       /* digits */
    const uint32_t *radix;            /* [B] */
    const uint32_t *first_scene;      /* [B+1] */
    const uint32_t *choice_level;     /* [sum radix] */
    const uint32_t *choice_k;         /* [sum radix] */
    const uint32_t *choice_pool;      /* [sum radix] */
    const uint64_t *va_us;            /* block-major: b, (s - first_b), c */
    const uint64_t *pool_ready_us;    /* [n_pools] or NULL: pool p's GPUs free from this time
                                         (model load + warm-up; reading R31) */
    const uint32_t *evict_risk_permille; /* [n_pools] or NULL: Spot eviction risk of pool p
                                         over the request, 1/1000 (reading R32) */
    const uint64_t *vae_us;           /* NULL, or block-major like va_us: the VAE stage time of a
                                         disaggregated choice (reading R37) */
    const uint32_t *choice_vae_pool;  /* NULL, or [sum radix]: pool running the choice's VAE
                                         stage on 1 GPU; UINT32_MAX = VAE folded into V+A */
    uint32_t metric;                  /* 0: cost in milli-cents; 1: energy in microjoules
                                         (reading R38) */
    const uint32_t *power_active_w;   /* [n_pools] busy GPU power (metric 1) */
    const uint32_t *power_idle_w;     /* [n_pools] idle GPU power (metric 1) */
} or_problem;

typedef struct {
    uint64_t ttff_us;
    uint64_t stall_us;
    uint64_t cost_mc;
    uint32_t quality;
    uint16_t stall_count;
    uint8_t flags;   /* bit p: pool p used */
    uint8_t pad;
} or_record;

typedef struct {
    uint64_t slo_startup_us, slo_stall_us, budget_mc;
} or_query;

typedef struct {
    uint64_t index;
    or_record rec;
    int32_t status; /* 0 feasible winner, 1 closest (nothing feasible), -1 empty range */
    int32_t pad;
} or_winner;

typedef struct {
    uint64_t index, ttff_eff_us, cost_mc;
    uint32_t quality, pad;
} or_point;

#define OR_MAXP 8
#define OR_MAXG 64

/* ---- a2: fixed-stage ready times (Table 4) ---------- */
/* L = overhead; for each non-static scene in order: the LLM finishes scene s at
 * L += llm_s; the single TTS server starts it when both the text exists and
 * the server is free: A = max(L, A) + tts_s; a_s = A is the earliest V+A start. */
void or_fixed_stages(const or_problem *pb, uint64_t *a_out) {
    uint64_t L = pb->overhead_us, A = 0;
    for (uint32_t s = 0; s < pb->S; s++) {
        if (s == 0 && pb->scene0_static) { a_out[s] = 0; continue; }
        L = L + pb->llm_us[s];
        A = (L > A ? L : A) + pb->tts_us[s];
        a_out[s] = A;
    }
}

/* ---- scene deadlines relative to the first frame: P_s = sum_{j<s} d_j */
void or_deadlines(const or_problem *pb, uint64_t *P_out) {
    uint64_t acc = 0;
    for (uint32_t s = 0; s < pb->S; s++) { P_out[s] = acc; acc += pb->dur_us[s]; }
}

/* ---- a1: mixed-radix decode, MSD = earliest scene block (reading R19) ------- */
void or_decode(const or_problem *pb, uint64_t index, uint32_t *digits) {
    for (int b = (int)pb->B - 1; b >= 0; b--) {
        digits[b] = (uint32_t)(index % pb->radix[b]);
        index /= pb->radix[b];
    }
}

uint64_t or_space_size(const or_problem *pb) {
    uint64_t n = 1;
    for (uint32_t b = 0; b < pb->B; b++) n *= pb->radix[b];
    return n;
}

static int cmp_u64(const void *x, const void *y) {
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* cost of one pool: round-half-up of X_p * price_p / 3.6e9 us-per-hour (Table 3;
 * reading R10/R11): (X*price + 1.8e9) / 3.6e9 in integer milli-cents. */
static uint64_t pool_cost(uint64_t X, uint64_t price) {
    return (X * price + 1800000000ull) / 3600000000ull;
}

/* ---- a4-a7: evaluate ONE candidate by full recompute ----------------------- */
/* Spot over-provisioning ("We proportionally increase the number of allocated
 * resources to the eviction risk"; reading R32): allocate the fewest GPUs n
 * whose expected survivors n * (1 - rho) still cover the G the schedule runs on, i.e. the
 * smallest n >= G with n * (1000 - rho) >= G * 1000.  All n are billed (RESERVED). */
static uint64_t billed_gpus(const or_problem *pb, uint32_t p) {
    uint64_t G = pb->gpus[p], rho = pb->evict_risk_permille ? pb->evict_risk_permille[p] : 0;
    uint64_t n = G;
    while (n * (1000 - rho) < G * 1000) n++;
    return n;
}

/* Optional detail outputs (any may be NULL): ready_us[S], pool_end[n_pools],
 * makespan, ttff_eff. */
void or_eval_detail(const or_problem *pb, const uint64_t *a, const uint64_t *P,
                    uint64_t index, or_record *rec, uint64_t *ready_us,
                    uint64_t *pool_end_us, uint64_t *makespan_us, uint64_t *ttff_eff_us) {
    uint32_t digits[64];
    or_decode(pb, index, digits);

    uint64_t F[OR_MAXP][OR_MAXG]; /* ascending free times of each pool's GPUs */
    uint64_t busy[OR_MAXP];
    uint32_t used = 0;
    for (uint32_t p = 0; p < pb->n_pools; p++) {
        /* every GPU of pool p is free once the pool is loaded and warmed up (P:608-611,
           R31); warm pools (R18) start at 0 */
        for (uint32_t g = 0; g < pb->gpus[p]; g++) F[p][g] = pb->pool_ready_us ? pb->pool_ready_us[p] : 0;
        busy[p] = 0;
    }
    uint64_t R0 = 0, Q = 0, last = 0; /* last: latest ready time of a STATIC scene */
    int64_t M = 0;
    uint32_t cnt = 0;
    uint32_t s0 = 0;
    if (pb->scene0_static) { /* static intro, no GPU, quality 0 (R15) */
        R0 = pb->static_ready_us;
        M = (int64_t)R0;
        s0 = 1;
        if (ready_us) ready_us[0] = R0;
    }
    uint32_t coff = 0, voff = 0, b = 0;
    /* walk digits/blocks in scene order */
    for (uint32_t s = s0; s < pb->S; s++) {
        while (!(pb->first_scene[b] <= s && s < pb->first_scene[b + 1])) {
            coff += pb->radix[b];
            voff += (pb->first_scene[b + 1] - pb->first_scene[b]) * pb->radix[b];
            b++;
        }
        uint32_t c = digits[b];
        uint32_t l = pb->choice_level[coff + c];
        uint32_t k = pb->choice_k[coff + c];
        uint32_t p = pb->choice_pool[coff + c];
        uint64_t t = pb->va_us[voff + (s - pb->first_scene[b]) * pb->radix[b] + c];
        if (k == 0) {
            /* STATIC rung ("If not enough, we switch to static content", P:823-825;
               reading R33): no video stage and no GPU -- the scene (slides over its
               narration) is ready once its text and audio are, R_s = a_s */
            uint64_t e = a[s];
            if (ready_us) ready_us[s] = e;
            if (e > last) last = e;
            if (s == 0) {
                R0 = e;
                M = (int64_t)e;
            } else if ((int64_t)e - (int64_t)P[s] > M) {
                M = (int64_t)e - (int64_t)P[s];
                cnt++;
            }
            Q += (pb->dur_us[s] / 1000) * pb->level_score[l];
            continue;
        }
        /* the scene needs its text+audio (a_s) and k GPUs: the k earliest free */
        uint64_t fk = F[p][k - 1];
        uint64_t st = a[s] > fk ? a[s] : fk;
        uint64_t e = st + t;
        /* F_p <- sort(F_p[k:] ++ [e]*k): the gang of k GPUs is busy until e */
        uint64_t nf[OR_MAXG];
        uint32_t G = pb->gpus[p], n = 0;
        for (uint32_t g = k; g < G; g++) nf[n++] = F[p][g];
        for (uint32_t g = 0; g < k; g++) nf[n++] = e;
        qsort(nf, n, sizeof(uint64_t), cmp_u64);
        for (uint32_t g = 0; g < G; g++) F[p][g] = nf[g];
        used |= 1u << p;
        busy[p] += (uint64_t)k * t;
        uint32_t vp = pb->choice_vae_pool ? pb->choice_vae_pool[coff + c] : UINT32_MAX;
        if (vp != UINT32_MAX) {
            /* "FramePack DiT streams latent outputs to the VAE for decoding ... This enables
               pipelined execution" (reading R37): the scene's VAE runs on its own
               pool, one GPU (the VAE is not parallelised), once its DiT finished and
               a VAE GPU is free; the DiT pool meanwhile serves the next scene */
            uint64_t tv = pb->vae_us[voff + (s - pb->first_scene[b]) * pb->radix[b] + c];
            uint64_t fv = F[vp][0];
            uint64_t ev = (e > fv ? e : fv) + tv;
            uint32_t Gv = pb->gpus[vp], m = 0;
            for (uint32_t g = 1; g < Gv; g++) nf[m++] = F[vp][g];
            nf[m++] = ev;
            qsort(nf, m, sizeof(uint64_t), cmp_u64);
            for (uint32_t g = 0; g < Gv; g++) F[vp][g] = nf[g];
            used |= 1u << vp;
            busy[vp] += tv;
            e = ev;
        }
        if (ready_us) ready_us[s] = e;
        if (s == 0) {
            R0 = e;
            M = (int64_t)e;
        } else if ((int64_t)e - (int64_t)P[s] > M) { /* new rebuffering event */
            M = (int64_t)e - (int64_t)P[s];
            cnt++;
        }
        Q += (pb->dur_us[s] / 1000) * pb->level_score[l];
    }
    uint64_t cost = pb->fixed_cost_mc, mk = R0 > last ? R0 : last; /* makespan: last scene ready */
    for (uint32_t p = 0; p < pb->n_pools; p++) {
        uint64_t end = 0; /* an unused pool is not provisioned: no end, no bill (R31) */
        if (used & (1u << p))
            for (uint32_t g = 0; g < pb->gpus[p]; g++) if (F[p][g] > end) end = F[p][g];
        if (pool_end_us) pool_end_us[p] = end;
        if (end > mk) mk = end;
        if (used & (1u << p)) {
            if (pb->metric == 1) {
                /* energy ("optimizing for energy"; reading R38): busy GPUs draw their
                   active power (TDP, "average power remains within 10% of the peak"),
                   the pool's other rented GPUs their idle power ("63W when idle")
                   until the pool's last finish (RESERVED); BUSY: busy GPU time only.  W x us
                   = microjoules, exact */
                uint64_t idle_us = pb->billing == 0 ? billed_gpus(pb, p) * end - busy[p] : 0;
                cost += (uint64_t)pb->power_active_w[p] * busy[p] + (uint64_t)pb->power_idle_w[p] * idle_us;
            } else {
                uint64_t X = pb->billing == 0 ? billed_gpus(pb, p) * end : busy[p];
                cost += pool_cost(X, pb->price_mc[p]);
            }
        }
    }
    rec->ttff_us = R0;
    rec->stall_us = (uint64_t)M - R0;
    rec->cost_mc = cost;
    rec->quality = (uint32_t)Q;
    rec->stall_count = (uint16_t)cnt;
    rec->flags = (uint8_t)used;
    rec->pad = 0;
    if (makespan_us) *makespan_us = mk;
    if (ttff_eff_us) *ttff_eff_us = (uint64_t)M;
}

void or_eval_range(const or_problem *pb, uint64_t begin, uint64_t end, or_record *out) {
    uint64_t *a = malloc(sizeof(uint64_t) * pb->S), *P = malloc(sizeof(uint64_t) * pb->S);
    or_fixed_stages(pb, a);
    or_deadlines(pb, P);
    for (uint64_t i = begin; i < end; i++)
        or_eval_detail(pb, a, P, i, &out[i - begin], NULL, NULL, NULL, NULL);
    free(a);
    free(P);
}

/* ---- a9: selection keys (reading R13) --------------------------- */
static uint64_t sat_sub(uint64_t x, uint64_t y) { return x > y ? x - y : 0; }

/* objective key comparison; returns <0 if (ia,a) is better than (ib,b) */
static int obj_cmp(uint32_t objective, uint64_t ia, const or_record *a, uint64_t ib,
                   const or_record *b) {
    uint64_t ta = a->ttff_us + a->stall_us, tb = b->ttff_us + b->stall_us;
    if (objective == 0) { /* QUALITY_FIRST: (-Q, cost, ttff_eff, index) */
        if (a->quality != b->quality) return a->quality > b->quality ? -1 : 1;
        if (a->cost_mc != b->cost_mc) return a->cost_mc < b->cost_mc ? -1 : 1;
        if (ta != tb) return ta < tb ? -1 : 1;
    } else { /* COST_X_TTFF: (cost * ttff_eff as u128, -Q, index) -- "$ x seconds" */
        unsigned __int128 xa = (unsigned __int128)a->cost_mc * ta;
        unsigned __int128 xb = (unsigned __int128)b->cost_mc * tb;
        if (xa != xb) return xa < xb ? -1 : 1;
        if (a->quality != b->quality) return a->quality > b->quality ? -1 : 1;
    }
    if (ia != ib) return ia < ib ? -1 : 1;
    return 0;
}

static int feasible(const or_query *q, const or_record *r) {
    return r->ttff_us <= q->slo_startup_us && r->stall_us <= q->slo_stall_us &&
           r->cost_mc <= q->budget_mc;
}

/* closest-solution order when nothing is feasible: (V_t, V_c, objective key, index) */
static int closest_cmp(uint32_t objective, const or_query *q, uint64_t ia,
                       const or_record *a, uint64_t ib, const or_record *b) {
    uint64_t vta = sat_sub(a->ttff_us, q->slo_startup_us) + sat_sub(a->stall_us, q->slo_stall_us);
    uint64_t vtb = sat_sub(b->ttff_us, q->slo_startup_us) + sat_sub(b->stall_us, q->slo_stall_us);
    if (vta != vtb) return vta < vtb ? -1 : 1;
    uint64_t vca = sat_sub(a->cost_mc, q->budget_mc), vcb = sat_sub(b->cost_mc, q->budget_mc);
    if (vca != vcb) return vca < vcb ? -1 : 1;
    return obj_cmp(objective, ia, a, ib, b);
}

/* ---- a8: 3-D dominance with the lowest-index duplicate rule (reading R14) --- */
static int dominates(const or_point *y, const or_point *x) {
    if (!(y->ttff_eff_us <= x->ttff_eff_us && y->cost_mc <= x->cost_mc &&
          y->quality >= x->quality))
        return 0;
    if (y->ttff_eff_us < x->ttff_eff_us || y->cost_mc < x->cost_mc || y->quality > x->quality)
        return 1;
    return y->index < x->index;
}

typedef struct {
    or_point *v;
    uint64_t n, cap;
} front_t;

static void front_offer(front_t *f, const or_point *x) {
    for (uint64_t j = 0; j < f->n; j++) {
        if (dominates(&f->v[j], x)) {
            if (j > 0) { /* move the dominator forward: a plain search heuristic */
                or_point tmp = f->v[j];
                f->v[j] = f->v[0];
                f->v[0] = tmp;
            }
            return;
        }
    }
    uint64_t w = 0;
    for (uint64_t j = 0; j < f->n; j++)
        if (!dominates(x, &f->v[j])) f->v[w++] = f->v[j];
    f->n = w;
    if (f->n == f->cap) {
        f->cap = f->cap ? 2 * f->cap : 64;
        f->v = realloc(f->v, f->cap * sizeof(or_point));
    }
    f->v[f->n++] = *x;
}

static int point_order(const void *xa, const void *xb) {
    const or_point *a = xa, *b = xb;
    if (a->ttff_eff_us != b->ttff_eff_us) return a->ttff_eff_us < b->ttff_eff_us ? -1 : 1;
    if (a->cost_mc != b->cost_mc) return a->cost_mc < b->cost_mc ? -1 : 1;
    if (a->quality != b->quality) return a->quality > b->quality ? -1 : 1;
    return a->index < b->index ? -1 : (a->index > b->index ? 1 : 0);
}

/* ---- record digest (test tool): sum_i mix64(i ^ rotl(ttff,7) ^ rotl(stall,19)
 *      ^ rotl(cost,31) ^ (flags<<48 | Q<<16 | cnt)) mod 2^64 -------------------- */
static uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t or_record_hash(uint64_t index, const or_record *r) {
    uint64_t w = ((uint64_t)r->flags << 48) | ((uint64_t)r->quality << 16) | r->stall_count;
    return mix64(index ^ rotl(r->ttff_us, 7) ^ rotl(r->stall_us, 19) ^ rotl(r->cost_mc, 31) ^ w);
}

/* ---- the full sweep: evaluate [begin,end), select, Pareto, digest --------- */
typedef void (*or_eval_fn)(const void *ctx, uint64_t index, or_record *rec);

typedef struct {
    const or_problem *pb;
    const uint64_t *a, *P;
    uint64_t begin, end;
    or_eval_fn fn; /* NULL: one request's candidate (or_eval_detail), else fn(ctx, i, &r) */
    const void *ctx;
    uint32_t objective;
    uint32_t nq;
    const or_query *q;
    or_winner feas[64], close[64];
    front_t front;
    uint64_t digest;
} sweep_job;

static void *sweep_worker(void *arg) {
    sweep_job *j = arg;
    const uint32_t objective = j->objective;
    for (uint32_t k = 0; k < j->nq; k++) { j->feas[k].status = -1; j->close[k].status = -1; }
    for (uint64_t i = j->begin; i < j->end; i++) {
        or_record r;
        if (j->fn) j->fn(j->ctx, i, &r);
        else or_eval_detail(j->pb, j->a, j->P, i, &r, NULL, NULL, NULL, NULL);
        j->digest += or_record_hash(i, &r);
        for (uint32_t k = 0; k < j->nq; k++) {
            const or_query *q = &j->q[k];
            if (feasible(q, &r)) {
                if (j->feas[k].status < 0 ||
                    obj_cmp(objective, i, &r, j->feas[k].index, &j->feas[k].rec) < 0) {
                    j->feas[k].index = i; j->feas[k].rec = r; j->feas[k].status = 0;
                }
            } else {
                if (j->close[k].status < 0 ||
                    closest_cmp(objective, q, i, &r, j->close[k].index, &j->close[k].rec) < 0) {
                    j->close[k].index = i; j->close[k].rec = r; j->close[k].status = 1;
                }
            }
        }
        or_point x = {i, r.ttff_us + r.stall_us, r.cost_mc, r.quality, 0};
        front_offer(&j->front, &x);
    }
    return NULL;
}

/* Evaluate [begin, end) with the given evaluator (fn NULL: candidates of pb), select,
 * Pareto, digest.  Returns 0 on success, 1 if the front did not fit. */
static int sweep_generic(const or_problem *pb, or_eval_fn fn, const void *ctx, uint32_t objective,
                         uint64_t begin, uint64_t end, uint32_t nthreads,
                         uint32_t nq, const or_query *queries, or_winner *winners,
                         or_point *front_out, uint64_t front_cap, uint64_t *front_n, uint64_t *digest) {
    if (nthreads < 1) nthreads = 1;
    if (nq > 64) return -1;
    uint64_t *a = NULL, *P = NULL;
    if (pb) {
        a = malloc(sizeof(uint64_t) * pb->S);
        P = malloc(sizeof(uint64_t) * pb->S);
        or_fixed_stages(pb, a);
        or_deadlines(pb, P);
    }
    sweep_job *jobs = calloc(nthreads, sizeof(sweep_job));
    pthread_t *th = calloc(nthreads, sizeof(pthread_t));
    uint64_t n = end > begin ? end - begin : 0;
    for (uint32_t t = 0; t < nthreads; t++) {
        jobs[t].pb = pb; jobs[t].a = a; jobs[t].P = P;
        jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].objective = objective;
        jobs[t].begin = begin + n * t / nthreads;
        jobs[t].end = begin + n * (t + 1) / nthreads;
        jobs[t].nq = nq; jobs[t].q = queries;
        pthread_create(&th[t], NULL, sweep_worker, &jobs[t]);
    }
    for (uint32_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    /* merge: per query, best feasible over threads, else best closest */
    uint64_t dg = 0;
    for (uint32_t t = 0; t < nthreads; t++) dg += jobs[t].digest;
    *digest = dg;
    for (uint32_t k = 0; k < nq; k++) {
        or_winner best = {0};
        best.status = -1;
        for (uint32_t t = 0; t < nthreads; t++) {
            or_winner *w = &jobs[t].feas[k];
            if (w->status == 0 && (best.status != 0 ||
                obj_cmp(objective, w->index, &w->rec, best.index, &best.rec) < 0))
                best = *w;
        }
        if (best.status != 0) {
            for (uint32_t t = 0; t < nthreads; t++) {
                or_winner *w = &jobs[t].close[k];
                if (w->status == 1 && (best.status != 1 ||
                    closest_cmp(objective, &queries[k], w->index, &w->rec, best.index, &best.rec) < 0))
                    best = *w;
            }
        }
        winners[k] = best;
    }
    /* Pareto: union of the per-thread fronts, then the plain definition */
    uint64_t tot = 0;
    for (uint32_t t = 0; t < nthreads; t++) tot += jobs[t].front.n;
    or_point *all = malloc((tot + 1) * sizeof(or_point));
    uint64_t m = 0;
    for (uint32_t t = 0; t < nthreads; t++) {
        memcpy(all + m, jobs[t].front.v, jobs[t].front.n * sizeof(or_point));
        m += jobs[t].front.n;
        free(jobs[t].front.v);
    }
    or_point *fr = malloc((tot + 1) * sizeof(or_point));
    uint64_t nf = 0;
    for (uint64_t x = 0; x < m; x++) {
        int dom = 0;
        for (uint64_t y = 0; y < m && !dom; y++)
            if (y != x && dominates(&all[y], &all[x])) dom = 1;
        if (!dom) fr[nf++] = all[x];
    }
    qsort(fr, nf, sizeof(or_point), point_order);
    *front_n = nf;
    int rc = 0;
    if (nf > front_cap) rc = 1;
    else memcpy(front_out, fr, nf * sizeof(or_point));
    free(all); free(fr); free(jobs); free(th); free(a); free(P);
    return rc;
}

int or_sweep(const or_problem *pb, uint64_t begin, uint64_t end, uint32_t nthreads,
             uint32_t nq, const or_query *queries, or_winner *winners,
             or_point *front_out, uint64_t front_cap, uint64_t *front_n, uint64_t *digest) {
    return sweep_generic(pb, NULL, NULL, pb->objective, begin, end, nthreads, nq, queries, winners,
                         front_out, front_cap, front_n, digest);
}

/* Pareto front of an explicit point list (plain O(n^2) definition, sorted output). */
uint64_t or_pareto_points(const or_point *pts, uint64_t n, or_point *out) {
    uint64_t nf = 0;
    for (uint64_t x = 0; x < n; x++) {
        int dom = 0;
        for (uint64_t y = 0; y < n && !dom; y++)
            if (y != x && dominates(&pts[y], &pts[x])) dom = 1;
        if (!dom) out[nf++] = pts[x];
    }
    qsort(out, nf, sizeof(or_point), point_order);
    return nf;
}

/* ---- greedy + iterative refinement planner -------------
 * The paper's provisioner: "Initial provisioning: we start with a
 * cost-efficient baseline configuration that leverages inexpensive models and
 * lower-cost GPUs. Each model instance ... is assigned a single GPU";
 * "Iterative refinement: ... systematically exploring the latency-cost trade-off
 * space. For each setting, we use the greedy algorithm to estimate the latency and
 * cost", switching GPU types, models and GPU allocation per instance
 * (P:906-911), minimising the objective and steering toward the SLO, "If we cannot
 * find feasible solutions, it returns the closest solution".
 * Reading R28: the baseline takes, in every digit, the choice with the
 * smallest (level score, k, pool price, choice index); a refinement step evaluates
 * every single-digit change of the current plan (switch model = level, GPU type =
 * pool, parallelism = k) and moves to the best one under the query's total order
 * (feasible first by the objective key, else closest) if it is strictly better than
 * the current plan; it stops when none is (steepest descent to a local optimum). */
static int query_better(uint32_t objective, const or_query *q, uint64_t ia, const or_record *a,
                        uint64_t ib, const or_record *b) {
    int fa = feasible(q, a), fb = feasible(q, b);
    if (fa != fb) return fa;
    if (fa) return obj_cmp(objective, ia, a, ib, b) < 0;
    return closest_cmp(objective, q, ia, a, ib, b) < 0;
}

int or_greedy(const or_problem *pb, const or_query *q, uint64_t start, uint64_t *out_index,
              or_record *out_rec, int32_t *status, uint32_t *iterations, uint64_t *evaluations) {
    uint64_t *a = malloc(sizeof(uint64_t) * pb->S), *P = malloc(sizeof(uint64_t) * pb->S);
    or_fixed_stages(pb, a);
    or_deadlines(pb, P);
    uint64_t place[64];
    uint64_t pl = 1;
    for (int b = (int)pb->B - 1; b >= 0; b--) { place[b] = pl; pl *= pb->radix[b]; }
    uint32_t dig[64];
    if (start == UINT64_MAX) { /* cost-efficient baseline */
        uint32_t coff = 0;
        start = 0;
        for (uint32_t b = 0; b < pb->B; b++) {
            uint32_t best = 0;
            for (uint32_t c = 1; c < pb->radix[b]; c++) {
                uint32_t x = coff + c, y = coff + best;
                uint64_t kx[3] = {pb->level_score[pb->choice_level[x]], pb->choice_k[x], pb->price_mc[pb->choice_pool[x]]};
                uint64_t ky[3] = {pb->level_score[pb->choice_level[y]], pb->choice_k[y], pb->price_mc[pb->choice_pool[y]]};
                int lt = 0;
                for (int i = 0; i < 3; i++) if (kx[i] != ky[i]) { lt = kx[i] < ky[i]; goto decided; }
                lt = 0; /* equal keys: keep the lower choice index */
            decided:
                if (lt) best = c;
            }
            start += best * place[b];
            coff += pb->radix[b];
        }
    }
    uint64_t cur = start;
    or_record rc;
    or_eval_detail(pb, a, P, cur, &rc, NULL, NULL, NULL, NULL);
    uint64_t evals = 1;
    uint32_t it = 0;
    for (;;) {
        or_decode(pb, cur, dig);
        uint64_t bi = UINT64_MAX;
        or_record br;
        for (uint32_t b = 0; b < pb->B; b++)
            for (uint32_t c = 0; c < pb->radix[b]; c++) {
                if (c == dig[b]) continue;
                uint64_t x = cur - (uint64_t)dig[b] * place[b] + (uint64_t)c * place[b];
                or_record r;
                or_eval_detail(pb, a, P, x, &r, NULL, NULL, NULL, NULL);
                evals++;
                if (bi == UINT64_MAX || query_better(pb->objective, q, x, &r, bi, &br)) { bi = x; br = r; }
            }
        if (bi == UINT64_MAX || !query_better(pb->objective, q, bi, &br, cur, &rc)) break;
        cur = bi;
        rc = br;
        it++;
    }
    *out_index = cur;
    *out_rec = rc;
    *status = feasible(q, &rc) ? 0 : 1;
    *iterations = it;
    *evaluations = evals;
    free(a);
    free(P);
    return 0;
}

/* ---- shared-pool fleet (reading R36) ------------------------
 * "To coordinate multiple requests, model instances maintain local queues that
 * prioritize tasks by deadline.  For example, the image generation model may process an
 * early scene from a new request before a later scene from an earlier request if it has
 * a tighter deadline"; per-node deadlines come from the request's SLO: "a
 * real-time video podcast with a TTFF of 5 seconds and 10-minute duration sets the final
 * node's deadline at t_now+605"; heterogeneous SLOs -- real-time, 50% relaxed,
 * batch (no SLO) -- let the deadline-aware scheduler "prioritize real-time requests"
 * (P:1449-1451).  Reading R36:
 *   - requests r arrive at T0_r, each with its own fixed stages (own LLM / TTS, so its
 *     scene s is released at T0_r + a_s), scenes, tables and a plan; the n_pools GPU pools
 *     are SHARED by all requests;
 *   - scene s of request r is due at d_rs = T0_r + slo_startup_r + P_s (UINT64_MAX for a
 *     batch request, whose scenes then rank after every deadline-bearing task);
 *   - every pool is an online, non-preemptive EDF queue of gang tasks: whenever it
 *     decides at time t, the head is the released (release <= t), unstarted task with the
 *     smallest (deadline, request, scene); it starts at max(t, F[k-1]) on the k
 *     earliest-free GPUs (the single-request recurrence's gang rule, no backfill)
 *     unless a more urgent task is released at or before that start, which then takes the
 *     decision; decisions are made in time order;
 *   - a request's metrics are its own, relative to T0_r (TTFF, TTFF_eff, stall, count,
 *     quality as for one request); the FLEET record of a joint plan is
 *       ttff  = max_r sat(ttff_r - slo_startup_r)   (worst startup lateness)
 *       stall = max_r sat(stall_r - slo_stall_r)    (worst stall lateness)
 *       cost  = sum_r fixed_r + sum_p pool cost (RESERVED: billed G_p x the pool's last
 *               finish, from t = 0; BUSY: sum k t), Q = sum_r Q_r, count = sum_r count_r,
 *       flags = pools used,
 *     so the query (0, 0, budget) asks "every request meets its SLO within the fleet
 *     budget" and the closest tier minimises lateness.
 * A joint candidate index enumerates the plans of the FREE requests (fixed_index[r] =
 * UINT64_MAX), MSD = the first free request's first digit; fixed requests are the
 * background load. */
typedef struct {
    uint32_t n_req;
    const or_problem *req;          /* [n_req]: scenes, tables, fixed cost, level scores of
                                       each request; their pool fields are ignored */
    const uint64_t *arrival_us;     /* [n_req] T0_r */
    const uint64_t *slo_startup_us; /* [n_req] (UINT64_MAX: batch) */
    const uint64_t *slo_stall_us;   /* [n_req] */
    const uint64_t *fixed_index;    /* [n_req] plan of a background request, UINT64_MAX = free */
    uint32_t n_pools;
    const uint32_t *gpus;
    const uint64_t *price_mc;
    const uint64_t *pool_ready_us;  /* or NULL */
    uint32_t billing;
    uint32_t objective;
} or_shared;

#define OR_MAXREQ 16

static uint64_t sat_add(uint64_t a, uint64_t b) { return a > UINT64_MAX - b ? UINT64_MAX : a + b; }

uint64_t or_shared_space_size(const or_shared *sh) {
    uint64_t n = 1;
    for (uint32_t r = 0; r < sh->n_req; r++)
        if (sh->fixed_index[r] == UINT64_MAX) n *= or_space_size(&sh->req[r]);
    return n;
}

/* Joint index -> one plan index per request (last free request = least significant). */
void or_shared_decode(const or_shared *sh, uint64_t index, uint64_t *plan) {
    for (int r = (int)sh->n_req - 1; r >= 0; r--) {
        if (sh->fixed_index[r] != UINT64_MAX) { plan[r] = sh->fixed_index[r]; continue; }
        uint64_t n = or_space_size(&sh->req[r]);
        plan[r] = index % n;
        index /= n;
    }
}

typedef struct { uint32_t r, s, k, pool; uint64_t rel, dl, t; int started; } sh_task;

static int task_before(const sh_task *x, const sh_task *y) { /* (deadline, request, scene) */
    if (x->dl != y->dl) return x->dl < y->dl;
    if (x->r != y->r) return x->r < y->r;
    return x->s < y->s;
}

/* Evaluate one joint candidate: fleet record, per-request records (may be NULL) and
 * absolute scene ready times ready[r * 64 + s] (may be NULL). */
void or_shared_eval(const or_shared *sh, uint64_t index, or_record *fleet, or_record *per_req,
                    uint64_t *ready_abs) {
    uint64_t plan[OR_MAXREQ];
    or_shared_decode(sh, index, plan);
    static const uint32_t MAXT = OR_MAXREQ * 64;
    sh_task *tasks = malloc(sizeof(sh_task) * MAXT);
    uint64_t ready[OR_MAXREQ][64];
    uint64_t a[OR_MAXREQ][64], P[OR_MAXREQ][64];
    uint32_t lvl[OR_MAXREQ][64];
    uint32_t nt = 0;
    /* 1. every request's fixed stages and its scenes' choices */
    for (uint32_t r = 0; r < sh->n_req; r++) {
        const or_problem *pb = &sh->req[r];
        or_fixed_stages(pb, a[r]);
        or_deadlines(pb, P[r]);
        uint32_t digits[64];
        or_decode(pb, plan[r], digits);
        uint32_t coff = 0, voff = 0, b = 0;
        uint32_t s0 = pb->scene0_static ? 1 : 0;
        if (s0) { ready[r][0] = sat_add(sh->arrival_us[r], pb->static_ready_us); lvl[r][0] = UINT32_MAX; }
        for (uint32_t s = s0; s < pb->S; s++) {
            while (!(pb->first_scene[b] <= s && s < pb->first_scene[b + 1])) {
                coff += pb->radix[b];
                voff += (pb->first_scene[b + 1] - pb->first_scene[b]) * pb->radix[b];
                b++;
            }
            uint32_t c = digits[b];
            lvl[r][s] = pb->choice_level[coff + c];
            uint32_t k = pb->choice_k[coff + c], p = pb->choice_pool[coff + c];
            uint64_t t = pb->va_us[voff + (s - pb->first_scene[b]) * pb->radix[b] + c];
            uint64_t rel = sh->arrival_us[r] + a[r][s];
            if (k == 0) { ready[r][s] = rel; continue; } /* STATIC rung: R = a (R33) */
            sh_task x = {r, s, k, p, rel, 0, t, 0};
            x.dl = sh->slo_startup_us[r] == UINT64_MAX ? UINT64_MAX
                   : sat_add(sat_add(sh->arrival_us[r], sh->slo_startup_us[r]), P[r][s]);
            tasks[nt++] = x;
        }
    }
    /* 2. every pool: online non-preemptive EDF of gang tasks */
    uint32_t used = 0;
    uint64_t cost = 0;
    for (uint32_t p = 0; p < sh->n_pools; p++) {
        uint64_t F[OR_MAXG];
        uint32_t G = sh->gpus[p];
        for (uint32_t g = 0; g < G; g++) F[g] = sh->pool_ready_us ? sh->pool_ready_us[p] : 0;
        uint64_t busy = 0, tnow = 0;
        int any = 0;
        for (;;) {
            int h = -1, left = 0;
            for (uint32_t i = 0; i < nt; i++) {
                if (tasks[i].pool != p || tasks[i].started) continue;
                left = 1;
                if (tasks[i].rel <= tnow && (h < 0 || task_before(&tasks[i], &tasks[h]))) h = (int)i;
            }
            if (!left) break;
            if (h < 0) { /* nothing released: wait for the next release */
                uint64_t nr = UINT64_MAX;
                for (uint32_t i = 0; i < nt; i++)
                    if (tasks[i].pool == p && !tasks[i].started && tasks[i].rel < nr) nr = tasks[i].rel;
                tnow = nr;
                continue;
            }
            sh_task *x = &tasks[h];
            uint64_t fk = F[x->k - 1];
            uint64_t st = tnow > fk ? tnow : fk;
            /* a more urgent task released by the head's start takes the decision */
            uint64_t u = UINT64_MAX;
            for (uint32_t i = 0; i < nt; i++)
                if (tasks[i].pool == p && !tasks[i].started && tasks[i].rel > tnow && task_before(&tasks[i], x) &&
                    tasks[i].rel < u)
                    u = tasks[i].rel;
            if (u <= st) { tnow = u; continue; }
            uint64_t e = st + x->t;
            uint64_t nf[OR_MAXG];
            uint32_t n = 0;
            for (uint32_t g = x->k; g < G; g++) nf[n++] = F[g];
            for (uint32_t g = 0; g < x->k; g++) nf[n++] = e;
            qsort(nf, n, sizeof(uint64_t), cmp_u64);
            for (uint32_t g = 0; g < G; g++) F[g] = nf[g];
            busy += (uint64_t)x->k * x->t;
            ready[x->r][x->s] = e;
            x->started = 1;
            tnow = st;
            any = 1;
        }
        if (any) {
            used |= 1u << p;
            uint64_t end = 0;
            for (uint32_t g = 0; g < G; g++) if (F[g] > end) end = F[g];
            uint64_t X = sh->billing == 0 ? (uint64_t)G * end : busy;
            cost += pool_cost(X, sh->price_mc[p]);
        }
    }
    /* 3. per-request playback metrics in scene order (relative to T0_r), fleet record */
    uint64_t late_t = 0, late_s = 0, Qs = 0, cnts = 0;
    for (uint32_t r = 0; r < sh->n_req; r++) {
        const or_problem *pb = &sh->req[r];
        uint64_t R0 = 0, Q = 0;
        int64_t M = 0;
        uint32_t cnt = 0;
        for (uint32_t s = 0; s < pb->S; s++) {
            uint64_t e = ready[r][s] - sh->arrival_us[r];
            if (ready_abs) ready_abs[r * 64 + s] = ready[r][s];
            if (s == 0) { R0 = e; M = (int64_t)e; }
            else if ((int64_t)e - (int64_t)P[r][s] > M) { M = (int64_t)e - (int64_t)P[r][s]; cnt++; }
            if (lvl[r][s] != UINT32_MAX) Q += (pb->dur_us[s] / 1000) * pb->level_score[lvl[r][s]];
        }
        uint64_t stall = (uint64_t)M - R0;
        cost += pb->fixed_cost_mc;
        if (per_req) {
            per_req[r].ttff_us = R0; per_req[r].stall_us = stall; per_req[r].cost_mc = pb->fixed_cost_mc;
            per_req[r].quality = (uint32_t)Q; per_req[r].stall_count = (uint16_t)cnt; per_req[r].flags = 0;
            per_req[r].pad = 0;
        }
        uint64_t lt = sat_sub(R0, sh->slo_startup_us[r]), ls = sat_sub(stall, sh->slo_stall_us[r]);
        if (lt > late_t) late_t = lt;
        if (ls > late_s) late_s = ls;
        Qs += Q;
        cnts += cnt;
    }
    fleet->ttff_us = late_t;
    fleet->stall_us = late_s;
    fleet->cost_mc = cost;
    fleet->quality = (uint32_t)Qs;
    fleet->stall_count = (uint16_t)cnts;
    fleet->flags = (uint8_t)used;
    fleet->pad = 0;
    free(tasks);
}

static void shared_eval_fn(const void *ctx, uint64_t i, or_record *r) {
    or_shared_eval((const or_shared *)ctx, i, r, NULL, NULL);
}

int or_shared_sweep(const or_shared *sh, uint64_t begin, uint64_t end, uint32_t nthreads, uint32_t nq,
                    const or_query *queries, or_winner *winners, or_point *front_out, uint64_t front_cap,
                    uint64_t *front_n, uint64_t *digest) {
    return sweep_generic(NULL, shared_eval_fn, sh, sh->objective, begin, end, nthreads, nq, queries, winners,
                         front_out, front_cap, front_n, digest);
}

/* Merge of two winners of the SAME query over disjoint candidate sets (e.g. pieces of a
 * long full-space sweep run one after the other): the same rule or_sweep applies across
 * its threads -- a feasible winner beats a closest one, feasible by the objective key,
 * closest by (V_t, V_c, key, index) (reading R13); an empty one (status -1)
 * loses. */
void or_winner_merge(uint32_t objective, const or_query *q, const or_winner *a, const or_winner *b,
                     or_winner *out) {
    if (a->status < 0) { *out = *b; return; }
    if (b->status < 0) { *out = *a; return; }
    if (a->status != b->status) { *out = a->status == 0 ? *a : *b; return; }
    int c = a->status == 0 ? obj_cmp(objective, a->index, &a->rec, b->index, &b->rec)
                           : closest_cmp(objective, q, a->index, &a->rec, b->index, &b->rec);
    *out = c <= 0 ? *a : *b;
}

int or_abi_version(void) { return 1; }
uint32_t or_sizeof_record(void) { return (uint32_t)sizeof(or_record); }
uint32_t or_sizeof_winner(void) { return (uint32_t)sizeof(or_winner); }
uint32_t or_sizeof_point(void) { return (uint32_t)sizeof(or_point); }
