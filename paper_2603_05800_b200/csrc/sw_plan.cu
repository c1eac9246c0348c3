// sw_plan.cu -- host runtime + C ABI of libsw_plan.so (see include/sw_plan.h).
//
// Host code here only validates inputs, does index bookkeeping (digit padding,
// place values, shard ranges, segment table), moves bytes and launches kernels.
// Every step of the method -- fixed-stage ready times, decode, the max-plus scan,
// metrics, cost, selection, Pareto and the cross-rank merge -- runs in the CUDA
// kernels of sw_kernels.cuh.  There is no CPU fallback: without a device every
// call that needs one returns SW_ECUDA.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "sw_coll.cuh"
#include <nvtx3/nvToolsExt.h>

#include "sw_kernels.cuh"
#include "sw_shared.cuh"
#include "sw_wide.cuh"
#include "sw_plan.h"

using namespace sw;

namespace {

thread_local std::string g_last_error;

// NVTX range around every public entry point (visible in nsys / ncu timelines; a no-op
// when no tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct Segment {
    uint64_t gbegin, gend;  // global range of the eval call
    uint64_t begin, end;    // this rank's shard
    uint64_t offset;        // record slot of the segment's first tile
    uint64_t tile0, ntiles; // tiles of 32 rows covering this rank's shard (tiled layout)
    bool folded;            // already folded into the Pareto front
};

}  // namespace

struct SharedHost {
    std::vector<sw_plan*> reqs;      // per request: tables only (t_tables_only handles)
    std::vector<uint32_t> S, sc_off; // scenes and their offset in the joint ready array
    SharedDev* d_dev = nullptr;
    SharedDetailOut* d_full = nullptr;  // [SW_MAX_QUERIES]
};

struct sw_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ncclComm_t comm = nullptr;
    LoopComm* loop = nullptr;  // in-process loopback rank (tests), instead of comm
    int rank = 0, nranks = 1;
    sw_alloc_fn alloc = nullptr;
    sw_free_fn free_fn = nullptr;
    void* alloc_ctx = nullptr;

    DevHeader h{};  // host image of the index bookkeeping
    uint32_t NP = 1, S = 0, B_user = 0, pad_digits = 0;
    uint64_t N = 0, row = 1;
    uint32_t n_va = 0, va_bytes = 0;
    int num_sms = 148;
    int eval_grid = 0;
    size_t eval_smem = 0;

    DevHeader* d_hdr = nullptr;
    VaEntry* d_va = nullptr;
    Rec4* d_rec = nullptr;
    uint64_t rec_cap = 0, rec_used = 0;  // record SLOTS (tiled layout incl. padding)
    uint64_t cand_cap = 0, cand_used = 0;  // candidates retained (record_capacity)
    std::vector<Segment> segs;

    // Pareto
    PPoint* d_front = nullptr;
    uint64_t front_n = 0;
    uint64_t front_cap = 1ull << 17;
    uint64_t surv_cap = 1ull << 18;  // 2^17 overflowed in the first passes of 3 G-record C5 shards (a refold: 2x the scan)
    PPoint* d_work = nullptr;  // front_cap + surv_cap
    PPoint* d_tmp = nullptr;   // front_cap + surv_cap (the merge's t-sorted input)
    uint32_t* d_rhist = nullptr;  // kRedBuckets (the merge's bucket sort)
    uint32_t* d_qsort = nullptr;  // kDltSortMax + 1: the DLT's sorted front qualities, then its done counter
    uint8_t* d_keep = nullptr;
    ParetoCtl* d_ctl = nullptr;
    Dlt* d_dlt = nullptr;
    PPoint* d_gather = nullptr;  // multi-rank padded fronts
    PPoint* d_tmp2 = nullptr;    // front_cap + surv_cap (block-local fronts)
    PPoint* d_surv = nullptr;    // surv_cap survivors of filter passes
    PPoint* d_dltc = nullptr;    // DLT survivors of a scan pass (deferred exact test), allocated on first fold
    uint64_t dltc_cap = 0;
    bool fuse_pareto = true;     // fold unfolded segments inside select scans
    bool cxt_front_ok = false;   // COST_X_TTFF: every record has cost > 0 and ttff_eff > 0 (R35)
    bool wide = false;           // a pool of > 8 GPUs: the warp-per-candidate generic path (sw_wide.cuh)
    uint64_t chunk = 1ull << 25; // records per fold chunk (the front improves per chunk)
    uint64_t fold_passes = 0;    // diagnostics: filter passes run
    uint64_t epoch = 1;          // bumped by every change of records or front
    bool released = false;       // records dropped since create/reset: the front covers more
    uint64_t merged_epoch = 0, merged_n = 0;  // multi-rank merged front cached in d_gather
    // state epoch that changes only with calls every rank makes (eval, reset, release,
    // stream): the merged-front cache is keyed on it, so every rank takes the same
    // (cached or collective) branch whatever its local refolds did
    uint64_t gepoch = 1;
    bool debug = false;          // SW_DEBUG=1: per-pass fold statistics on stderr
    uint64_t first_pass = 8ull << 20;  // SW_FIRST_PASS: records of the first strided fold pass (about)
    uint64_t max_pass = 1ull << 29;    // SW_MAX_PASS: a fold level of more records is split ...
    uint64_t sub_pass = 1ull << 28;    // SW_SUB_PASS: ... into sub-passes of about this many
    uint32_t fold_kmin = 1;      // SW_FOLD_KMIN: fewest strided fold levels (passes - 1); a first pass stays <= ~8 M records
    const char* dump_merge = nullptr;  // SW_DUMP_MERGE=<prefix>: every fold merge's input -> <prefix>_<n>.bin
    bool coop_reduce = true;        // merge in one cooperative launch (SW_COOP_REDUCE=0: 5 launches)
    uint32_t coop_grid = 0;
    bool trace = false;             // SW_TRACE=1: per-phase CUDA-event times of each select on stderr
    std::vector<std::pair<const char*, cudaEvent_t>> tr;  // (phase that ENDS at the event, event)
    uint64_t* d_counts = nullptr;
    uint32_t* d_gfeas = nullptr;  // grid-wide "feasible seen" flags + closest keys of a select (kGSelWords)
    GreedyOut* d_greedy = nullptr;
    std::vector<uint32_t> level_score;  // for the greedy baseline (host copy of the input)

    // select / detail / digest
    Cand* d_partial = nullptr;
    uint32_t scan_grid = 0;
    uint32_t max_partial = 0;
    Cand* d_cand = nullptr;
    Cand* d_cand_all = nullptr;
    DetailOut* d_detail = nullptr;  // [SW_MAX_QUERIES]
    EvalJob* d_selfjob = nullptr;   // this handle's tables as a 1-entry job list
    unsigned long long* d_digest = nullptr;

    // CUDA events around every eval-kernel launch, on the handle's stream: a ring of
    // pairs harvested (synchronised and summed) when full or on sw_plan_eval_time
    static constexpr int kEvPairs = 64;
    cudaEvent_t ev[2 * kEvPairs] = {};
    uint32_t ev_kind[kEvPairs] = {};   // SW_KERNEL_EVAL / SW_KERNEL_SCAN
    uint64_t ev_bytes[kEvPairs] = {};  // algorithmic bytes of the launch (32 B x records)
    int ev_used = 0;          // pairs recorded since the last harvest
    int ev_last = -1;         // pair of the last eval launch
    float last_eval_ms = 0.f;
    bool have_eval_ev = false;
    uint64_t k_launches[3] = {0, 0, 0};
    double k_ms[3] = {0.0, 0.0, 0.0};
    uint64_t k_bytes[3] = {0, 0, 0};
    uint64_t launches = 0;
    std::string err;

    // shared-pool fleet (sw_shared_create): the requests' table handles + device descriptor
    struct SharedHost* shared = nullptr;

    // fused stream (sw_plan_stream): per-query reported candidates, allocated on first use
    Cand* d_scand = nullptr;       // [SW_MAX_QUERIES][scand_cap]
    uint32_t* d_scand_n = nullptr;  // [SW_MAX_QUERIES]
    unsigned long long* d_skey = nullptr;  // [3][SW_MAX_QUERIES] pruning keys (StreamArgs::gkey)
    uint64_t* h_pass_surv = nullptr;       // pinned: survivors of each stream pass (<= 21 levels)
    uint32_t scand_cap = 1u << 18;
    size_t stream_smem = 0;
    int stream_occ[3] = {1, 1, 1};  // resident stream blocks per SM, per eval path
    uint64_t stream_passes = 0;    // diagnostics
};

namespace {

sw_status fail(sw_plan* h, sw_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    if (h) h->err = buf;
    return s;
}

#define CK(h, call)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail((h), SW_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

#define CKL(h)                                                                                \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess)                                                                \
            return fail((h), SW_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                  \
        (h)->launches++;                                                                      \
    } while (0)

#define CKN(h, call)                                                                          \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail((h), SW_ENCCL, "%s failed: %s", #call, ncclGetErrorString(r_));        \
    } while (0)

// The handle's collective context (NCCL or loopback) on its stream.
Coll coll_of(const sw_plan* h) {
    Coll c;
    c.nccl = h->comm;
    c.loop = h->loop;
    c.stream = h->stream;
    c.rank = h->rank;
    c.nranks = h->nranks;
    return c;
}

// a10 collectives and the stream wait of collective calls (async NCCL errors, timeout)
#define CKC(h, call)                                                                           \
    do {                                                                                       \
        const char* why_ = "";                                                                 \
        sw_status s_ = (call);                                                                 \
        if (s_ != SW_OK) return fail((h), s_, "%s failed: %s (%s:%d)", #call, why_, __FILE__, __LINE__); \
    } while (0)
#define SYNC(h)                                                                               \
    do {                                                                                      \
        const char* why_ = "";                                                                \
        sw_status s_ = coll_sync(coll_of(h), &why_);                                          \
        if (s_ != SW_OK) return fail((h), s_, "stream synchronisation failed: %s (%s:%d)", why_, __FILE__, __LINE__); \
    } while (0)

// Timing events outlive handles: a process-wide pool (per device), filled lazily and
// refilled at destroy -- 128 cudaEventCreate + cudaEventDestroy per handle were about a
// third of an end-to-end step's create/destroy host time.
namespace {
std::mutex g_ev_mu;
std::vector<std::pair<int, cudaEvent_t>> g_ev_free;
cudaError_t event_get(int dev, cudaEvent_t* e) {
    {
        std::lock_guard<std::mutex> g(g_ev_mu);
        for (size_t i = g_ev_free.size(); i-- > 0;)
            if (g_ev_free[i].first == dev) {
                *e = g_ev_free[i].second;
                g_ev_free[i] = g_ev_free.back();
                g_ev_free.pop_back();
                return cudaSuccess;
            }
    }
    return cudaEventCreate(e);
}
void event_put(int dev, cudaEvent_t e) {  // the handle's stream is idle (synchronised)
    std::lock_guard<std::mutex> g(g_ev_mu);
    g_ev_free.push_back({dev, e});
}
}  // namespace

void* dev_alloc(sw_plan* h, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (h->alloc) return h->alloc(bytes, h->stream, h->alloc_ctx);
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, h->stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void dev_free(sw_plan* h, void* p) {
    if (!p) return;
    if (h->free_fn) h->free_fn(p, h->stream, h->alloc_ctx);
    else cudaFreeAsync(p, h->stream);
}

template <typename T>
sw_status alloc_n(sw_plan* h, T** p, uint64_t n, const char* what) {
    *p = (T*)dev_alloc(h, (size_t)(n * sizeof(T)));
    if (!*p) return fail(h, SW_ENOMEM, "device allocation of %s (%llu bytes) failed", what,
                         (unsigned long long)(n * sizeof(T)));
    return SW_OK;
}

template <typename F>
sw_status launch_np(sw_plan* h, F&& f) {
    switch (h->NP) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        default: return fail(h, SW_EINVAL, "bad pool count");
    }
    return SW_OK;
}

using u128 = unsigned __int128;

}  // namespace

static sw_status fold_pending(sw_plan* h);
static sw_status global_front(sw_plan* h, const PPoint** res_out, uint64_t* n_out);
static sw_status ensure_dltc(sw_plan* h, uint64_t candidates);
static constexpr uint64_t kMaxSegs = 16;  // segments with tile padding budgeted per handle

// Tiles [t_lo, t_hi) (relative to the segment) of a segment as a scan view.
static SegView view_of(const sw_plan* h, const Segment& g, uint64_t t_lo, uint64_t t_hi) {
    SegView v;
    v.recs = h->d_rec + g.offset + t_lo * kTileRows * h->row;
    v.t0 = g.tile0 + t_lo;
    v.ntiles = t_hi - t_lo;
    v.row = h->row;
    v.ib = g.begin;
    v.ie = g.end;
    v.pass = 0;
    v.upt = 1;
    v.levels = 0;
    v.j0 = 0;
    v.j1 = 0xffffffffu;
    v.pad_ = 0;
    return v;
}
static cudaError_t set_scan_smem_attrs();
static cudaError_t set_scan_smem_attrs_once(int device);

static sw_status create_common(sw_plan* h, const sw_runtime* rt);
static thread_local bool t_tables_only = false;  // sw_shared_create: per-request table handles

// ============================================================================ create
extern "C" sw_status sw_plan_create(const sw_profile_tables* tb, const sw_scene_list* sc,
                                    const sw_price_table* pr, const sw_runtime* rt, sw_plan** out) {
    const NvtxRange nvtx_("sw_plan_create");
    if (!tb || !sc || !pr || !rt || !out) return fail(nullptr, SW_EINVAL, "null argument");
    const uint32_t S = sc->n_scenes;
    if (S < 1 || S > SW_MAX_SCENES) return fail(nullptr, SW_EINVAL, "n_scenes %u not in 1..%d", S, SW_MAX_SCENES);
    if (!sc->dur_us || !sc->llm_us || !sc->tts_us) return fail(nullptr, SW_EINVAL, "null scene array");
    for (uint32_t s = 0; s < S; s++)
        if (sc->dur_us[s] == 0) return fail(nullptr, SW_EINVAL, "scene %u has duration 0", s);
    const uint32_t B = tb->n_digits;
    if (B < 1 || B > SW_MAX_DIGITS) return fail(nullptr, SW_EINVAL, "n_digits %u not in 1..%d", B, SW_MAX_DIGITS);
    if (!tb->radix || !tb->first_scene || !tb->choices || !tb->va_us || !tb->level_score)
        return fail(nullptr, SW_EINVAL, "null table array");
    const uint32_t NP = pr->n_pools;
    if (NP < 1 || NP > SW_MAX_POOLS) return fail(nullptr, SW_EINVAL, "n_pools %u not in 1..%d", NP, SW_MAX_POOLS);
    if (!pr->gpus || !pr->price_mc_per_gpu_hour) return fail(nullptr, SW_EINVAL, "null price array");
    for (uint32_t p = 0; p < NP; p++)
        if (pr->gpus[p] < 1 || pr->gpus[p] > SW_MAX_GPUS_PER_POOL)
            return fail(nullptr, SW_EINVAL, "pool %u has %u GPUs (1..%d supported)", p, pr->gpus[p],
                        SW_MAX_GPUS_PER_POOL);
    if (pr->billing > 1 || pr->objective > 1 || pr->metric > 1)
        return fail(nullptr, SW_EINVAL, "bad billing/objective/metric");
    if (pr->metric && (!pr->power_active_w || !pr->power_idle_w))
        return fail(nullptr, SW_EINVAL, "the energy metric needs power_active_w and power_idle_w");
    if (pr->metric)
        for (uint32_t p = 0; p < NP; p++)
            if (pr->power_idle_w[p] > pr->power_active_w[p])
                return fail(nullptr, SW_EINVAL, "pool %u: idle power above active power", p);
    // Spot over-provisioning (R32): billed GPUs G'_p = ceil(G_p * 1000 / (1000 - rho_p))
    uint32_t gbill[SW_MAX_POOLS];
    for (uint32_t p = 0; p < NP; p++) {
        const uint32_t rho = pr->evict_risk_permille ? pr->evict_risk_permille[p] : 0;
        if (rho >= 1000) return fail(nullptr, SW_EINVAL, "pool %u: eviction risk %u per mille not < 1000", p, rho);
        if (rho && pr->billing) return fail(nullptr, SW_EINVAL, "pool %u: eviction risk needs RESERVED billing", p);
        gbill[p] = (uint32_t)(((uint64_t)pr->gpus[p] * 1000 + (999 - rho)) / (1000 - rho));
    }
    if (tb->n_levels < 1) return fail(nullptr, SW_EINVAL, "n_levels = 0");
    const uint32_t s0 = sc->scene0_static ? 1u : 0u;
    if (s0 && S < 2) return fail(nullptr, SW_EINVAL, "a static intro needs S >= 2");
    if (tb->first_scene[0] != s0 || tb->first_scene[B] != S)
        return fail(nullptr, SW_EINVAL, "digit blocks must cover scenes [%u, %u)", s0, S);
    uint64_t N = 1;
    uint32_t n_choice = 0;
    uint64_t n_va = 0;
    for (uint32_t b = 0; b < B; b++) {
        const uint32_t r = tb->radix[b];
        if (r < 1 || r > SW_MAX_CHOICES) return fail(nullptr, SW_EINVAL, "radix[%u] = %u not in 1..%d", b, r, SW_MAX_CHOICES);
        if (tb->first_scene[b + 1] <= tb->first_scene[b])
            return fail(nullptr, SW_EINVAL, "digit %u has an empty scene block", b);
        if ((u128)N * r >= ((u128)1 << 63)) return fail(nullptr, SW_ERANGE, "plan space >= 2^63 (InstanceTooLarge)");
        N *= r;
        n_choice += r;
        n_va += (uint64_t)(tb->first_scene[b + 1] - tb->first_scene[b]) * r;
    }
    for (uint32_t c = 0; c < n_choice; c++) {
        const sw_choice& ch = tb->choices[c];
        if (ch.level >= tb->n_levels) return fail(nullptr, SW_EINVAL, "choice %u: level %u >= n_levels", c, ch.level);
        if (ch.pool >= NP) return fail(nullptr, SW_EINVAL, "choice %u: pool %u >= n_pools", c, ch.pool);
        if (ch.vae) {  // DiT/VAE disaggregation (R37): the VAE stage runs on pool vae - 1
            if (!tb->vae_us) return fail(nullptr, SW_EINVAL, "choice %u has a VAE stage but vae_us is NULL", c);
            if (ch.vae > NP) return fail(nullptr, SW_EINVAL, "choice %u: VAE pool %u >= n_pools", c, ch.vae - 1);
            if (ch.degree == 0) return fail(nullptr, SW_EINVAL, "choice %u: a STATIC choice has no VAE stage", c);
        }
        if (ch.degree == 0) continue;  // STATIC rung: no video stage, no GPU (R33)
        if (ch.degree > pr->gpus[ch.pool])
            return fail(nullptr, SW_EINVAL, "choice %u: k = %u exceeds G_p = %u", c, ch.degree, pr->gpus[ch.pool]);
        if (tb->heads && tb->heads % ch.degree)
            return fail(nullptr, SW_EINVAL, "choice %u: k = %u does not divide %u heads (P:748)", c, ch.degree, tb->heads);
    }
    {  // a video stage takes time (va >= 1); a STATIC choice has none (va = 0)
        uint64_t i = 0, coff = 0;
        for (uint32_t b = 0; b < B; b++) {
            const uint32_t r = tb->radix[b];
            for (uint32_t s = tb->first_scene[b]; s < tb->first_scene[b + 1]; s++)
                for (uint32_t c = 0; c < r; c++, i++) {
                    const bool stat = tb->choices[coff + c].degree == 0;
                    if (stat != (tb->va_us[i] == 0))
                        return fail(nullptr, SW_EINVAL, "va_us[%llu] = %llu for a %s choice", (unsigned long long)i,
                                    (unsigned long long)tb->va_us[i], stat ? "STATIC" : "video");
                    if (tb->vae_us) {  // a VAE stage takes time (1 .. 2^32 - 1 us); none: 0
                        const bool vae = tb->choices[coff + c].vae != 0;
                        if (vae != (tb->vae_us[i] != 0) || tb->vae_us[i] >= (1ull << 32))
                            return fail(nullptr, SW_EINVAL, "vae_us[%llu] = %llu for a choice %s a VAE stage",
                                        (unsigned long long)i, (unsigned long long)tb->vae_us[i],
                                        vae ? "with" : "without");
                    }
                }
            coff += r;
        }
    }
    // ---- overflow bounds (R25): every intermediate fits its integer type
    {
        u128 fixed = (u128)sc->overhead_us + sc->static_ready_us;
        u128 dsum = 0, qsum = 0;
        uint32_t max_score = 0;
        for (uint32_t l = 0; l < tb->n_levels; l++) max_score = std::max(max_score, tb->level_score[l]);
        for (uint32_t s = 0; s < S; s++) {
            fixed += (u128)sc->llm_us[s] + sc->tts_us[s];
            dsum += sc->dur_us[s];
            qsum += (u128)(sc->dur_us[s] / 1000) * max_score;
        }
        u128 tmax = fixed;
        if (pr->pool_ready_us)  // a start offset delays every later finish (R31)
            for (uint32_t p = 0; p < pr->n_pools; p++) tmax = std::max<u128>(tmax, fixed + pr->pool_ready_us[p]);
        uint64_t off = 0;
        for (uint32_t b = 0; b < B; b++) {
            const uint32_t r = tb->radix[b];
            for (uint32_t s = tb->first_scene[b]; s < tb->first_scene[b + 1]; s++) {
                uint64_t mx = 0;
                for (uint32_t c = 0; c < r; c++) {
                    const uint64_t j = off + (s - tb->first_scene[b]) * r + c;
                    mx = std::max(mx, tb->va_us[j] + (tb->vae_us ? tb->vae_us[j] : 0));
                }
                tmax += mx;
            }
            off += (uint64_t)(tb->first_scene[b + 1] - tb->first_scene[b]) * r;
        }
        const u128 lim62 = (u128)1 << 62;
        if (tmax >= lim62 || dsum >= lim62) return fail(nullptr, SW_ERANGE, "time bound exceeds 2^62 us");
        if (qsum >= ((u128)1 << 32) - 1) return fail(nullptr, SW_ERANGE, "quality bound exceeds 2^32 - 2");
        u128 cmax = pr->fixed_cost_mc;
        for (uint32_t p = 0; p < NP; p++) {
            const u128 X = (u128)gbill[p] * tmax;  // >= busy and >= G' * span (G' >= G)
            const u128 prod = pr->metric ? X * ((u128)pr->power_active_w[p] + pr->power_idle_w[p])  // energy, uJ
                                         : X * pr->price_mc_per_gpu_hour[p] + kHalfHour;
            if (prod >= ((u128)1 << 64)) return fail(nullptr, SW_ERANGE, "cost bound of pool %u exceeds 2^64", p);
            cmax += pr->metric ? prod : prod / kUsPerHour;
        }
        if (cmax >= ((u128)1 << 64)) return fail(nullptr, SW_ERANGE, "cost bound exceeds 2^64");
    }
    if (rt->nranks < 1 || rt->rank < 0 || rt->rank >= rt->nranks)
        return fail(nullptr, SW_EINVAL, "bad rank %d of %d", rt->rank, rt->nranks);
    if (rt->nranks > 1 && !rt->nccl_comm) return fail(nullptr, SW_EINVAL, "nranks > 1 needs nccl_comm");
    if (LoopComm* lc = as_loop(rt->nccl_comm))
        if (lc->g->n != rt->nranks || lc->rank != rt->rank)
            return fail(nullptr, SW_EINVAL, "loopback communicator is rank %d of %d, runtime says %d of %d", lc->rank,
                        lc->g->n, rt->rank, rt->nranks);

    sw_plan* h = new sw_plan();
    h->device = rt->device;
    h->loop = as_loop(rt->nccl_comm);
    h->comm = h->loop ? nullptr : (ncclComm_t)rt->nccl_comm;
    h->rank = rt->rank;
    h->nranks = rt->nranks;
    h->alloc = rt->alloc;
    h->free_fn = rt->free;
    h->alloc_ctx = rt->alloc_ctx;
    h->NP = NP;
    h->S = S;
    h->B_user = B;
    for (uint32_t p = 0; p < NP; p++) h->wide |= pr->gpus[p] > (uint32_t)kMaxG;
    {  // R35: cost >= fixed cost > 0; ttff_eff >= ttff = R_0 > 0 (a static intro's ready
       // time; else a_0 = overhead + llm_0 + tts_0, plus t >= 1 for a video choice)
        bool t_pos = s0 ? sc->static_ready_us > 0 : sc->overhead_us + sc->llm_us[0] + sc->tts_us[0] > 0;
        if (!s0 && !t_pos) {
            t_pos = true;  // scene 0 lies in digit 0's block: every choice must run a video stage
            for (uint32_t c = 0; c < tb->radix[0]; c++) t_pos &= tb->choices[c].degree > 0;
        }
        h->cxt_front_ok = pr->fixed_cost_mc > 0 && t_pos;
    }
    h->N = N;
    auto bail = [&](sw_status s) {
        sw_plan_destroy(h);
        return s;
    };
    if (cudaSetDevice(h->device) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(nullptr, SW_ECUDA, "cudaSetDevice(%d) failed (no CUDA device?)", h->device));
    }
    if (rt->stream) {
        h->stream = (cudaStream_t)rt->stream;
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(nullptr, SW_ECUDA, "cudaStreamCreate failed"));
        h->own_stream = true;
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
    if (!h->alloc) {  // keep freed blocks in the stream-ordered pool (repeated create/destroy)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, h->device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }

    // ---- index bookkeeping: left-pad digits to B >= 3 with radix-1 empty blocks
    DevHeader& H = h->h;
    memset(&H, 0, sizeof H);
    const uint32_t pad = B >= 3 ? 0 : 3 - B;
    const uint32_t BP = B + pad;
    h->pad_digits = pad;
    H.S = S;
    H.B = BP;
    H.NP = NP;
    bool any_vae = false;
    for (uint32_t c = 0; c < n_choice; c++) any_vae |= tb->choices[c].vae != 0;
    H.flags = (s0 ? 1u : 0u) | (pr->billing ? 2u : 0u) | (pr->objective ? 4u : 0u) | (pr->metric ? 8u : 0u) |
              (any_vae ? 16u : 0u);
    H.s0 = s0;
    H.R0_static = s0 ? sc->static_ready_us : 0;
    H.fixed_cost = pr->fixed_cost_mc;
    H.N = N;
    H.choice[0] = 0u | (1u << 8) | (0u << 16);  // dummy choice of the virtual digits
    uint32_t coff = 1, voff = 0;
    for (uint32_t b = 0; b < BP; b++) {
        if (b < pad) {
            H.radix[b] = 1;
            H.first[b] = s0;
            H.coff[b] = 0;
            H.voff[b] = 0;
        } else {
            const uint32_t ub = b - pad;
            H.radix[b] = tb->radix[ub];
            H.first[b] = tb->first_scene[ub];
            H.coff[b] = coff;
            H.voff[b] = voff;
            for (uint32_t c = 0; c < tb->radix[ub]; c++) {
                const sw_choice& ch = tb->choices[coff - 1 + c];
                H.choice[coff + c] = (uint32_t)ch.level | ((uint32_t)ch.degree << 8) | ((uint32_t)ch.pool << 16) |
                                     ((uint32_t)ch.vae << 24);
            }
            coff += tb->radix[ub];
            voff += (tb->first_scene[ub + 1] - tb->first_scene[ub]) * tb->radix[ub];
        }
    }
    H.first[BP] = S;
    H.n_choice = coff;
    if (H.first[BP] - H.first[BP - 1] == 1 && H.first[BP - 1] != 0) H.flags |= 32u;  // LSD fast path
    {  // group the LSD digit's choices by (pool, k) in first-appearance order
        const uint32_t bl = BP - 1, r = H.radix[bl];
        std::vector<uint32_t> keys;
        std::vector<std::vector<uint32_t>> members;
        for (uint32_t c = 0; c < r; c++) {
            const uint32_t ch = H.choice[H.coff[bl] + c];
            const uint32_t key = ch_pool(ch) | (ch_k(ch) << 8);
            size_t gi = std::find(keys.begin(), keys.end(), key) - keys.begin();
            if (gi == keys.size()) {
                keys.push_back(key);
                members.emplace_back();
            }
            members[gi].push_back(c);
        }
        H.lsd_ngroups = (uint32_t)keys.size();
        uint32_t o = 0;
        for (size_t gi = 0; gi < keys.size(); gi++) {
            H.lsd_goff[gi] = o;
            H.lsd_pk[gi] = keys[gi];
            for (uint32_t c : members[gi]) H.lsd_dl[o++] = c;
        }
        H.lsd_goff[keys.size()] = o;
    }
    H.n_va = (uint32_t)n_va;
    H.va_bytes = n_va * sizeof(VaEntry);
    h->row = (uint64_t)H.radix[BP - 2] * H.radix[BP - 1];
    H.row = h->row;
    H.n_rows = N / h->row;
    {
        uint64_t pl = 1;
        for (int b = (int)BP - 3; b >= 0; b--) {
            H.place[b] = pl;
            pl *= H.radix[b];
        }
    }
    for (uint32_t p = 0; p < NP; p++) {
        H.G[p] = pr->gpus[p];
        H.Gbill[p] = gbill[p];
        H.price[p] = pr->price_mc_per_gpu_hour[p];
        H.ready[p] = pr->pool_ready_us ? pr->pool_ready_us[p] : 0;  // load + warm-up (R31)
        H.Pact[p] = pr->metric ? pr->power_active_w[p] : 0;       // energy metric (R38)
        H.Pidle[p] = pr->metric ? pr->power_idle_w[p] : 0;
    }
    h->n_va = (uint32_t)n_va;
    h->va_bytes = (uint32_t)(n_va * sizeof(VaEntry));

    // ---- upload raw inputs + header, pack on the device (a2 runs in pack_kernel)
    std::vector<uint32_t> va_scene(n_va), va_choice(n_va);
    {
        uint64_t i = 0;
        for (uint32_t b = 0; b < B; b++) {
            const uint32_t r = tb->radix[b];
            for (uint32_t s = tb->first_scene[b]; s < tb->first_scene[b + 1]; s++)
                for (uint32_t c = 0; c < r; c++, i++) {
                    va_scene[i] = s;
                    va_choice[i] = H.coff[b + pad] + c;
                }
        }
    }
    const bool has_vae = tb->vae_us != nullptr;
    const size_t n_raw64 = 3 * (size_t)S + n_va + (has_vae ? n_va : 0);
    const size_t raw_bytes = n_raw64 * 8 + (size_t)tb->n_levels * 4 + 2 * (size_t)n_va * 4;
    std::vector<uint8_t> raw(raw_bytes);
    size_t o = 0;
    auto put = [&](const void* src, size_t bytes) {
        memcpy(raw.data() + o, src, bytes);
        o += bytes;
    };
    put(sc->dur_us, 8 * (size_t)S);
    put(sc->llm_us, 8 * (size_t)S);
    put(sc->tts_us, 8 * (size_t)S);
    put(tb->va_us, 8 * (size_t)n_va);
    if (has_vae) put(tb->vae_us, 8 * (size_t)n_va);
    put(tb->level_score, 4 * (size_t)tb->n_levels);
    put(va_scene.data(), 4 * (size_t)n_va);
    put(va_choice.data(), 4 * (size_t)n_va);
    uint8_t* d_raw = nullptr;
    sw_status st;
    if ((st = alloc_n(h, &h->d_hdr, 1, "header")) < 0) return bail(st);
    if ((st = alloc_n(h, &h->d_va, std::max<uint64_t>(n_va, 1), "va table")) < 0) return bail(st);
    if ((st = alloc_n(h, &d_raw, raw_bytes, "raw inputs")) < 0) return bail(st);
    if (cudaMemcpyAsync(h->d_hdr, &H, sizeof H, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
        cudaMemcpyAsync(d_raw, raw.data(), raw_bytes, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
        cudaGetLastError();
        dev_free(h, d_raw);
        return bail(fail(nullptr, SW_ECUDA, "table upload failed"));
    }
    RawDesc rd;
    {
        const uint64_t* r64 = (const uint64_t*)d_raw;
        rd.dur = r64;
        rd.llm = r64 + S;
        rd.tts = r64 + 2 * S;
        rd.va = r64 + 3 * S;
        rd.vae = has_vae ? r64 + 3 * S + n_va : nullptr;
        const uint32_t* r32 = (const uint32_t*)(r64 + 3 * S + n_va + (has_vae ? n_va : 0));
        rd.score = r32;
        rd.va_scene = r32 + tb->n_levels;
        rd.va_choice = r32 + tb->n_levels + n_va;
        rd.overhead = sc->overhead_us;
        rd.n_va = (uint32_t)n_va;
    }
    pack_kernel<<<1, 256, 0, h->stream>>>(rd, h->d_hdr, h->d_va);
    if (cudaGetLastError() != cudaSuccess) {
        dev_free(h, d_raw);
        return bail(fail(nullptr, SW_ECUDA, "pack_kernel launch failed"));
    }
    h->launches++;
    dev_free(h, d_raw);
    // keep the host mirror's a/P unused (device-owned); fetch nothing back.
    if (t_tables_only) {  // a request's tables for a shared-pool fleet: nothing else
        if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
            cudaGetLastError();
            return bail(fail(nullptr, SW_ECUDA, "create: device work failed"));
        }
        *out = h;
        return SW_OK;
    }

    // ---- eval launch configuration: persistent grid sized by occupancy x SMs
    h->eval_smem = sizeof(DevHeader) + h->va_bytes;
    {
        int occ = 0;
        cudaError_t e = cudaSuccess;
        launch_np(h, [&](auto np) {
            constexpr int NPc = decltype(np)::value;
            // the attribute is per kernel, not per handle: set the device maximum so
            // that every handle's table size stays launchable (occupancy below uses
            // this handle's actual size)
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
            auto setup = [&](auto kern) {  // every billing mode's instantiation (fleets use mode 2)
                cudaFuncAttributes fa{};
                cudaError_t r = cudaFuncGetAttributes(&fa, kern);
                const size_t dyn_max = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
                if (r == cudaSuccess)
                    r = dyn_max < h->eval_smem ? cudaErrorInvalidValue
                                               : cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                      (int)dyn_max);
                int o = 0;
                if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kEvalThreads, h->eval_smem);
                if (r != cudaSuccess && e == cudaSuccess) e = r;
                return o;
            };
            const int o[3] = {setup(eval_kernel<NPc, 0>), setup(eval_kernel<NPc, 1>), setup(eval_kernel<NPc, 2>)};
            setup(eval_kernel<NPc, 3>);
            const int ow = setup(eval_wide_kernel<NPc>);
            occ = h->wide ? ow : o[eval_mode(h->h.flags)];
        });
        if (e != cudaSuccess || occ < 1) {
            cudaGetLastError();
            return bail(fail(nullptr, SW_ECUDA, "eval kernel cannot launch (%s, occupancy %d)",
                             cudaGetErrorString(e), occ));
        }
        h->eval_grid = occ * h->num_sms;
    }
    h->level_score.assign(tb->level_score, tb->level_score + tb->n_levels);
    if ((st = create_common(h, rt)) < 0) return bail(st);
    *out = h;
    return SW_OK;
}

// Everything after the tables: scan configuration, record buffer, reduction scratch,
// events (shared by sw_plan_create and sw_shared_create).
static sw_status create_common(sw_plan* h, const sw_runtime* rt) {
    sw_status st;
    h->scan_grid = (uint32_t)h->num_sms;  // scan kernels: one TMA-pipelined block per SM
    if (const char* ev = getenv("SW_PARETO_CHUNK")) h->chunk = std::max<uint64_t>(1, strtoull(ev, nullptr, 10));
    if (const char* ev = getenv("SW_FUSE_PARETO")) h->fuse_pareto = atoi(ev) != 0;
    if (const char* ev = getenv("SW_DEBUG")) h->debug = atoi(ev) != 0;
    h->dump_merge = getenv("SW_DUMP_MERGE");
    if (const char* ev = getenv("SW_SUB_PASS")) h->sub_pass = std::max<uint64_t>(1 << 20, strtoull(ev, nullptr, 10));
    if (const char* ev = getenv("SW_MAX_PASS")) h->max_pass = std::max<uint64_t>(1 << 20, strtoull(ev, nullptr, 10));
    if (const char* ev = getenv("SW_FIRST_PASS")) h->first_pass = std::max<uint64_t>(1 << 16, strtoull(ev, nullptr, 10));
    if (const char* ev = getenv("SW_FOLD_KMIN")) h->fold_kmin = (uint32_t)std::min(std::max(atoi(ev), 1), 9);
    if (const char* ev = getenv("SW_TRACE")) h->trace = atoi(ev) != 0;
    if (const char* ev = getenv("SW_COOP_REDUCE")) h->coop_reduce = atoi(ev) != 0;
    if (const char* ev = getenv("SW_SURV_CAP")) {  // test hook: "<cap>[@<rank>]" (>= 256)
        char* end = nullptr;
        const uint64_t c = strtoull(ev, &end, 10);
        const int only = (end && *end == '@') ? atoi(end + 1) : -1;
        if (c >= 256 && (only < 0 || only == h->rank)) h->surv_cap = c;
    }
    {  // the cooperative merge needs all its blocks co-resident
        int occ = 0, coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pareto_reduce_kernel, kRedThreads, 0) != cudaSuccess ||
            occ < 1 || !coop) {
            cudaGetLastError();
            h->coop_reduce = false;
        }
        h->coop_grid = (uint32_t)(std::min(occ, 1) * h->num_sms);  // one block per SM
        if (const char* ev = getenv("SW_COOP_GRID"))
            h->coop_grid = std::min<uint32_t>(h->coop_grid, std::max(1, atoi(ev)));
    }
    if (cudaError_t se = set_scan_smem_attrs_once(h->device); se != cudaSuccess) {
        cudaGetLastError();
        return (fail(nullptr, SW_ECUDA, "scan kernels cannot launch one block per SM (%s; smem %zu/%zu B)",
                         cudaGetErrorString(se), ring_bytes(true) + sizeof(Dlt),
                         ring_bytes(false)));
    }

    // ---- record buffer + reduction scratch
    uint64_t cap = rt->record_capacity;
    // default: this rank's largest possible shard (whole rows split evenly, plus a
    // ragged head or tail of under a row each)
    if (cap == 0) cap = h->N / (uint64_t)h->nranks + 3 * h->row;
    h->cand_cap = cap;
    {  // slots: whole tiles of 32 rows plus 2 tiles of padding for each of up to
       // kMaxSegs segments (each eval call adds at most 2 partial tiles)
        const uint64_t per_tile = kTileRows * h->row;
        const uint64_t tiles = (cap + per_tile - 1) / per_tile + 2 * kMaxSegs;
        cap = tiles * per_tile;
    }
    h->rec_cap = cap;
    if ((st = alloc_n(h, &h->d_rec, cap, "records")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_front, h->front_cap, "pareto front")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_work, h->front_cap + h->surv_cap, "pareto work")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_tmp, h->front_cap + h->surv_cap, "pareto tmp")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_keep, h->front_cap + h->surv_cap, "pareto flags")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_rhist, kRedBuckets, "merge buckets")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_qsort, kDltSortMax + 1, "dlt quality sort")) < 0) return (st);
    if (cudaMemsetAsync(h->d_qsort + kDltSortMax, 0, sizeof(uint32_t), h->stream) != cudaSuccess)
        return (fail(nullptr, SW_ECUDA, "dlt counter init failed"));
    if ((st = alloc_n(h, &h->d_tmp2, h->front_cap + h->surv_cap, "pareto tmp2")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_surv, h->surv_cap, "pareto survivors")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_ctl, 1, "pareto ctl")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_dlt, 1, "dlt")) < 0) return (st);
    h->max_partial = h->scan_grid * 256;  // up to 256 scan launches (chunks x fold passes) per select
    if ((st = alloc_n(h, &h->d_partial, (uint64_t)h->max_partial * SW_MAX_QUERIES, "partials")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_cand, SW_MAX_QUERIES, "winners")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_cand_all, (uint64_t)SW_MAX_QUERIES * h->nranks, "winners all")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_detail, SW_MAX_QUERIES, "detail")) < 0) return (st);
    if (h->d_hdr) {  // this handle's tables as a 1-entry job list (winner details)
        if ((st = alloc_n(h, &h->d_selfjob, 1, "self job")) < 0) return (st);
        const EvalJob sj{h->d_hdr, h->d_va, h->va_bytes, 0, 0, nullptr};
        if (cudaMemcpyAsync(h->d_selfjob, &sj, sizeof sj, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
            return (fail(nullptr, SW_ECUDA, "self job upload failed"));
    }
    if ((st = alloc_n(h, &h->d_digest, 1, "digest")) < 0) return (st);
    // [0, R) gathered counts, [R] mine, [R+1] saved local front size, [R+2] merged size,
    // [R+3] pad overflow flag of the asynchronous merge, [R+4, R+4+kStatusWords) the
    // max-reduced status words of a multi-rank call
    if ((st = alloc_n(h, &h->d_counts, (uint64_t)h->nranks + 4 + kStatusWords, "counts")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_gfeas, kGSelWords, "select flags")) < 0) return (st);
    if ((st = alloc_n(h, &h->d_greedy, 1, "greedy result")) < 0) return (st);
        if (h->nranks > 1)
        if ((st = alloc_n(h, &h->d_gather, h->front_cap * (uint64_t)h->nranks, "front gather")) < 0) return (st);
    if (cudaMemsetAsync(h->d_ctl, 0, sizeof(ParetoCtl), h->stream) != cudaSuccess)
        return (fail(nullptr, SW_ECUDA, "ctl init failed"));
    for (int i = 0; i < 2 * sw_plan::kEvPairs; i++)
        if (event_get(h->device, &h->ev[i]) != cudaSuccess) return (fail(nullptr, SW_ECUDA, "cudaEventCreate failed"));
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
        cudaGetLastError();
        return (fail(nullptr, SW_ECUDA, "create: device work failed"));
    }
    return SW_OK;
}

extern "C" sw_status sw_plan_destroy(sw_plan* h) {
    if (!h) return SW_OK;
    if (h->stream) {
        cudaSetDevice(h->device);
        void* bufs[] = {h->d_hdr,   h->d_va,      h->d_rec,     h->d_front, h->d_work,
                        h->d_tmp,   h->d_keep,    h->d_ctl,     h->d_dlt,
                        h->d_partial, h->d_cand,  h->d_cand_all, h->d_detail, h->d_digest, h->d_selfjob,
                        h->d_counts, h->d_gather, h->d_tmp2, h->d_surv, h->d_gfeas, h->d_greedy,
                        h->d_scand, h->d_scand_n, h->d_skey, h->d_dltc, h->d_rhist, h->d_qsort};
        for (void* b : bufs) dev_free(h, b);
        cudaStreamSynchronize(h->stream);
        if (h->h_pass_surv) cudaFreeHost(h->h_pass_surv);
        for (cudaEvent_t e : h->ev)
            if (e) event_put(h->device, e);
        if (h->shared) {
            for (sw_plan* r : h->shared->reqs) sw_plan_destroy(r);
            cudaFree(h->shared->d_dev);
            cudaFree(h->shared->d_full);
        }
        if (h->own_stream) cudaStreamDestroy(h->stream);
        cudaGetLastError();
    }
    delete h->shared;
    delete h;
    return SW_OK;
}

extern "C" sw_status sw_plan_reset(sw_plan* h) {
    if (!h) return fail(nullptr, SW_EINVAL, "null handle");
    h->epoch++;
    h->gepoch++;
    h->segs.clear();
    h->rec_used = 0;
    h->cand_used = 0;
    h->front_n = 0;
    h->released = false;
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaMemsetAsync(h->d_ctl, 0, sizeof(ParetoCtl), h->stream));
    return SW_OK;
}

extern "C" sw_status sw_plan_release_records(sw_plan* h) {
    if (!h) return fail(nullptr, SW_EINVAL, "null handle");
    // fold pending records into the running front first (the front survives)
    sw_status st = fold_pending(h);
    if (st < 0) return st;
    h->segs.clear();
    h->rec_used = 0;
    h->cand_used = 0;
    h->released = true;
    h->epoch++;
    h->gepoch++;
    return SW_OK;
}

extern "C" sw_status sw_plan_space_size(const sw_plan* h, uint64_t* n) {
    if (!h || !n) return fail(nullptr, SW_EINVAL, "null argument");
    *n = h->N;
    return SW_OK;
}

extern "C" sw_status sw_plan_row_size(const sw_plan* h, uint64_t* row) {
    if (!h || !row) return fail(nullptr, SW_EINVAL, "null argument");
    *row = h->row;
    return SW_OK;
}

// ============================================================================ shard
extern "C" sw_status sw_shard_range(uint64_t begin, uint64_t end, uint64_t row, int32_t rank,
                                    int32_t nranks, uint64_t* sb, uint64_t* se) {
    if (!sb || !se || nranks < 1 || rank < 0 || rank >= nranks || row == 0 || end < begin)
        return fail(nullptr, SW_EINVAL, "bad shard arguments");
    const uint64_t r0 = (begin + row - 1) / row;  // first whole row
    const uint64_t r1 = end / row;                // one past the last whole row
    if (r1 <= r0) {  // no whole row: everything on rank 0
        *sb = rank == 0 ? begin : end;
        *se = end;
        if (rank != 0) *sb = *se = end;
        return SW_OK;
    }
    const uint64_t nr = r1 - r0;
    const uint64_t a = r0 + (uint64_t)((u128)nr * (uint64_t)rank / (uint64_t)nranks);
    const uint64_t b = r0 + (uint64_t)((u128)nr * (uint64_t)(rank + 1) / (uint64_t)nranks);
    *sb = rank == 0 ? begin : a * row;
    *se = rank == nranks - 1 ? end : b * row;
    return SW_OK;
}

// ============================================================================ eval
// Sum the recorded eval-kernel event pairs into the totals and free the ring.
static sw_status harvest_eval_events(sw_plan* h) {
    if (h->ev_used == 0) return SW_OK;
    CK(h, cudaEventSynchronize(h->ev[2 * (h->ev_used - 1) + 1]));
    for (int i = 0; i < h->ev_used; i++) {
        float ms = 0.f;
        CK(h, cudaEventElapsedTime(&ms, h->ev[2 * i], h->ev[2 * i + 1]));
        const uint32_t k = h->ev_kind[i];
        h->k_launches[k]++;
        h->k_ms[k] += ms;
        h->k_bytes[k] += h->ev_bytes[i];
        if (i == h->ev_last) h->last_eval_ms = ms;
    }
    h->ev_used = 0;
    h->ev_last = -1;
    return SW_OK;
}

// Event pair around one timed launch: begin_timed() before, end_timed() after.
static sw_status begin_timed(sw_plan* h, uint32_t kind, uint64_t bytes, int* pair) {
    if (h->ev_used == sw_plan::kEvPairs) {
        sw_status hs = harvest_eval_events(h);
        if (hs < 0) return hs;
    }
    const int pr = h->ev_used++;
    h->ev_kind[pr] = kind;
    h->ev_bytes[pr] = bytes;
    CK(h, cudaEventRecord(h->ev[2 * pr], h->stream));
    *pair = pr;
    return SW_OK;
}

static sw_status end_timed(sw_plan* h, int pair) {
    CK(h, cudaEventRecord(h->ev[2 * pair + 1], h->stream));
    return SW_OK;
}

// SW_TRACE: mark the end of a phase on the stream (no-op unless tracing).
static void trace_mark(sw_plan* h, const char* phase) {
    if (!h->trace) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, h->stream);
    h->tr.emplace_back(phase, e);
}

// After a sync: print the phase durations and drop the events.
static void trace_dump(sw_plan* h, const char* what) {
    if (!h->trace || h->tr.empty()) return;
    std::string line = std::string("[sw trace] rank ") + std::to_string(h->rank) + " " + what + ":";
    for (size_t i = 1; i < h->tr.size(); i++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->tr[i - 1].second, h->tr[i].second);
        char buf[96];
        snprintf(buf, sizeof buf, " %s %.3f", h->tr[i].first, ms);
        line += buf;
    }
    fprintf(stderr, "%s ms\n", line.c_str());
    for (auto& pe : h->tr) cudaEventDestroy(pe.second);
    h->tr.clear();
}

extern "C" sw_status sw_plan_eval(sw_plan* h, uint64_t begin, uint64_t end) {
    const NvtxRange nvtx_("sw_plan_eval");
    if (!h) return fail(nullptr, SW_EINVAL, "null handle");
    if (begin > end || end > h->N)
        return fail(h, SW_EINVAL, "range [%llu, %llu) outside [0, %llu)", (unsigned long long)begin,
                    (unsigned long long)end, (unsigned long long)h->N);
    if (begin == end) return SW_OK;
    for (const Segment& g : h->segs)
        if (begin < g.gend && g.gbegin < end) return fail(h, SW_EINVAL, "range overlaps an evaluated range");
    uint64_t b, e;
    sw_status st = sw_shard_range(begin, end, h->row, h->rank, h->nranks, &b, &e);
    if (st < 0) return st;
    const uint64_t n = e - b;
    const uint64_t rb = b / h->row, re = (e + h->row - 1) / h->row;
    const uint64_t t0 = rb / kTileRows, t1 = (re + kTileRows - 1) / kTileRows;
    const uint64_t slots = n ? (t1 - t0) * kTileRows * h->row : 0;
    if (h->cand_used + n > h->cand_cap)
        return fail(h, SW_ERANGE, "records would exceed capacity (%llu + %llu > %llu): reset or chunk",
                    (unsigned long long)h->cand_used, (unsigned long long)n, (unsigned long long)h->cand_cap);
    if (h->rec_used + slots > h->rec_cap)
        return fail(h, SW_ERANGE, "record buffer fragmented by more than %llu eval calls: reset or chunk",
                    (unsigned long long)kMaxSegs);
    Segment sg{begin, end, b, e, h->rec_used, t0, n ? t1 - t0 : 0, false};
    h->epoch++;
    h->gepoch++;
    CK(h, cudaSetDevice(h->device));
    if (n > 0) {
        const uint64_t need = (sg.ntiles * kTileRows + kEvalThreads - 1) / kEvalThreads;  // one warp per tile
        const uint32_t grid = (uint32_t)std::min<uint64_t>(need, (uint64_t)h->eval_grid);
        Rec4* outp = h->d_rec + h->rec_used;
        int pr = 0;
        sw_status ts = begin_timed(h, SW_KERNEL_EVAL, n * sizeof(Rec4), &pr);
        if (ts < 0) return ts;
        if (h->wide) {  // pools of > 8 GPUs: one warp per candidate (sw_wide.cuh)
            launch_np(h, [&](auto np) {
                constexpr int NPc = decltype(np)::value;
                eval_wide_kernel<NPc><<<grid, kEvalThreads, h->eval_smem, h->stream>>>(
                    EvalJob{h->d_hdr, h->d_va, h->va_bytes, t0, t1, outp});
            });
        } else if (h->shared) {  // shared-pool fleet: one thread per joint candidate (row = 1)
            const uint64_t thr = sg.ntiles * kTileRows;
            const uint32_t sgrid = (uint32_t)std::min<uint64_t>((thr + kShThreads - 1) / kShThreads, 8ull * h->num_sms);
            shared_eval_kernel<<<sgrid, kShThreads, 0, h->stream>>>(h->shared->d_dev, t0, t1, h->N, outp);
        } else {
            launch_np(h, [&](auto np) {
                constexpr int NPc = decltype(np)::value;
                const EvalJob job{h->d_hdr, h->d_va, h->va_bytes, t0, t1, outp};
                switch (eval_mode(h->h.flags)) {
                    case 0: eval_kernel<NPc, 0><<<grid, kEvalThreads, h->eval_smem, h->stream>>>(job, nullptr); break;
                    case 1: eval_kernel<NPc, 1><<<grid, kEvalThreads, h->eval_smem, h->stream>>>(job, nullptr); break;
                    default: eval_kernel<NPc, 2><<<grid, kEvalThreads, h->eval_smem, h->stream>>>(job, nullptr); break;
                }
            });
        }
        CKL(h);
        ts = end_timed(h, pr);
        if (ts < 0) return ts;
        h->ev_last = pr;
        h->have_eval_ev = true;
        h->rec_used += slots;
        h->cand_used += n;
    }
    h->segs.push_back(sg);
    return SW_OK;
}

extern "C" sw_status sw_plan_last_eval_ms(sw_plan* h, float* ms) {
    if (!h || !ms) return fail(nullptr, SW_EINVAL, "null argument");
    if (!h->have_eval_ev) return fail(h, SW_ESTATE, "no eval launched yet");
    if (h->ev_last >= 0) {
        CK(h, cudaEventSynchronize(h->ev[2 * h->ev_last + 1]));
        CK(h, cudaEventElapsedTime(&h->last_eval_ms, h->ev[2 * h->ev_last], h->ev[2 * h->ev_last + 1]));
    }
    *ms = h->last_eval_ms;
    return SW_OK;
}

extern "C" sw_status sw_plan_kernel_time(sw_plan* h, uint32_t kind, uint64_t* n_launches, double* total_ms,
                                         uint64_t* bytes) {
    if (!h || !n_launches || !total_ms || !bytes) return fail(nullptr, SW_EINVAL, "null argument");
    if (kind > SW_KERNEL_STREAM) return fail(h, SW_EINVAL, "bad kernel kind %u", kind);
    sw_status st = harvest_eval_events(h);
    if (st < 0) return st;
    *n_launches = h->k_launches[kind];
    *total_ms = h->k_ms[kind];
    *bytes = h->k_bytes[kind];
    return SW_OK;
}

// ============================================================================ select
static void detail_to_selection(const sw_plan* h, uint64_t index, const DetailOut& d, sw_selection* out,
                                uint64_t* ready);

// Full metrics of the winners d_cand[0, nw) into d_detail (one launch).
static sw_status launch_detail(sw_plan* h, uint32_t nw) {
    if (h->wide) {
        launch_np(h, [&](auto npc) {
            constexpr int NPc = decltype(npc)::value;
            wide_detail_kernel<NPc><<<nw, 32, 0, h->stream>>>(h->d_hdr, h->d_va, h->d_cand, nw, h->d_detail);
        });
    } else if (h->shared) {
        shared_detail_kernel<<<1, 32, 0, h->stream>>>(h->shared->d_dev, h->d_cand, nw, h->d_detail, h->shared->d_full);
    } else {
        launch_np(h, [&](auto npc) {
            constexpr int NPc = decltype(npc)::value;
            detail_fleet_kernel<NPc><<<1, 32, 0, h->stream>>>(h->d_selfjob, h->d_cand, nw, h->d_detail);
        });
    }
    CKL(h);
    return SW_OK;
}

static sw_status fill_detail(sw_plan* h, uint64_t index, sw_selection* out, uint64_t* ready) {
    if (h->shared || h->wide) {
        Cand c{};
        c.idx = index;
        CK(h, cudaMemcpyAsync(h->d_cand, &c, sizeof c, cudaMemcpyHostToDevice, h->stream));
        sw_status ds = launch_detail(h, 1);
        if (ds < 0) return ds;
    } else {
        launch_np(h, [&](auto np) {
            constexpr int NPc = decltype(np)::value;
            detail_kernel<NPc><<<1, 32, 0, h->stream>>>(h->d_hdr, h->d_va, index, h->d_detail);
        });
        CKL(h);
    }
    DetailOut d;
    CK(h, cudaMemcpyAsync(&d, h->d_detail, sizeof d, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    detail_to_selection(h, index, d, out, ready);
    return SW_OK;
}

static void detail_to_selection(const sw_plan* h, uint64_t index, const DetailOut& d, sw_selection* out,
                                uint64_t* ready) {
    out->index = index;
    out->rec.ttff_us = d.rec.w0;
    out->rec.stall_us = d.rec.w1;
    out->rec.cost_mc = d.rec.w2;
    out->rec.quality = (uint32_t)d.rec.w3;
    out->rec.stall_count = (uint16_t)(d.rec.w3 >> 32);
    out->rec.flags = (uint8_t)(d.rec.w3 >> 48);
    out->rec.pad = 0;
    out->ttff_eff_us = d.ttff_eff;
    out->makespan_us = d.makespan;
    for (int p = 0; p < SW_MAX_POOLS; p++) out->pool_end_us[p] = p < (int)h->NP ? d.pool_end[p] : 0;
    memset(out->digit, 0, sizeof out->digit);
    for (uint32_t b = 0; b < h->B_user; b++) out->digit[b] = (uint8_t)d.digit[b + h->pad_digits];
    if (ready) memcpy(ready, d.ready, sizeof(uint64_t) * h->S);
}

template <int NQ, bool PARETO>
static void launch_scan(uint32_t grid, size_t smem, cudaStream_t st, const SegView& v, const SelParams& P,
                        Cand* partial, const ParetoArgs& pa) {
    if (P.objective) scan_kernel<NQ, PARETO, 1><<<grid, kScanBlock, smem, st>>>(v, P, partial, pa, nullptr);
    else scan_kernel<NQ, PARETO, 0><<<grid, kScanBlock, smem, st>>>(v, P, partial, pa, nullptr);
}

// Scan kernels are specialised for NQ in {0, 1, 2, 4, 8} queries: a batch of another size
// runs with the next larger NQ, the extra slots holding copies of its last query (their
// partial winners are never read).
template <bool PARETO>
static void launch_scan_nq(uint32_t nq, uint32_t grid, size_t smem, cudaStream_t st, const SegView& v,
                           const SelParams& P0, Cand* partial, const ParetoArgs& pa) {
    SelParams P = P0;
    const uint32_t nqs = nq <= 2 ? nq : nq <= 4 ? 4 : 8;
    for (uint32_t j = nq; j < nqs; j++) P.q[j] = P.q[nq - 1];
    switch (nqs) {
        case 0: launch_scan<0, PARETO>(grid, smem, st, v, P, partial, pa); break;
        case 1: launch_scan<1, PARETO>(grid, smem, st, v, P, partial, pa); break;
        case 2: launch_scan<2, PARETO>(grid, smem, st, v, P, partial, pa); break;
        case 4: launch_scan<4, PARETO>(grid, smem, st, v, P, partial, pa); break;
        default: launch_scan<8, PARETO>(grid, smem, st, v, P, partial, pa); break;
    }
}

static constexpr size_t kScanSmemPareto = ring_bytes(true) + sizeof(Dlt);
static constexpr size_t kRingBytes = ring_bytes(false);

template <int NQ, int OBJ>
static cudaError_t set_attr_one() {
    cudaError_t a = cudaFuncSetAttribute(scan_kernel<NQ, true, OBJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kScanSmemPareto);
    cudaError_t b = cudaFuncSetAttribute(scan_kernel<NQ, false, OBJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kRingBytes);
    if (a != cudaSuccess) return a;
    if (b != cudaSuccess) return b;
    // the persistent scan needs one resident block per SM (registers x 512 threads + smem)
    int o1 = 0, o2 = 0;
    a = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, scan_kernel<NQ, true, OBJ>, kScanBlock, kScanSmemPareto);
    b = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, scan_kernel<NQ, false, OBJ>, kScanBlock, kRingBytes);
    if (a != cudaSuccess) return a;
    if (b != cudaSuccess) return b;
    return (o1 < 1 || o2 < 1) ? cudaErrorLaunchOutOfResources : cudaSuccess;
}

static cudaError_t set_scan_smem_attrs() {
    cudaError_t e = cudaFuncSetAttribute(pareto_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)exact_smem_bytes());
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(dlt_qtop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kDltSortMax * sizeof(uint32_t)));
    cudaError_t r[] = {set_attr_one<0, 0>(), set_attr_one<1, 0>(), set_attr_one<2, 0>(), set_attr_one<4, 0>(),
                       set_attr_one<8, 0>(), set_attr_one<0, 1>(), set_attr_one<1, 1>(), set_attr_one<2, 1>(),
                       set_attr_one<4, 1>(), set_attr_one<8, 1>()};
    for (cudaError_t x : r)
        if (x != cudaSuccess && e == cudaSuccess) e = x;
    // fleet scans: one query per request, objective per request at run time
    cudaError_t f = cudaFuncSetAttribute(scan_kernel<1, false, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kRingBytes);
    return f != cudaSuccess ? f : e;
}

// Function attributes are context-wide: set once per device (they were redone, with the
// occupancy queries, at every create -- part of an end-to-end step's create time).
static cudaError_t set_scan_smem_attrs_once(int device) {
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> g(mu);
    if (device >= 0 && device < 64 && done[device]) return cudaSuccess;
    const cudaError_t e = set_scan_smem_attrs();
    if (e == cudaSuccess && device >= 0 && device < 64) done[device] = true;
    return e;
}

static ParetoArgs pareto_args(sw_plan* h) {
    ParetoArgs pa;
    pa.dlt = h->d_dlt;
    pa.front = h->d_front;
    pa.ctl = h->d_ctl;
    pa.surv = h->d_surv;
    pa.cap = h->surv_cap;
    pa.cand = h->d_dltc;
    pa.cand_cap = h->dltc_cap;
    pa.gfeas = h->d_gfeas;
    pa.debug = h->debug ? 1u : 0u;
    return pa;
}

// The DLT of the current front: quality tops + q map (one block), then the t edges, t map
// and cells (kDltT blocks).
static sw_status dlt_build_async(sw_plan* h) {
    dlt_qtop_kernel<<<kDltQtopGrid, kDltQThreads, kDltSortMax * sizeof(uint32_t), h->stream>>>(
        h->d_front, h->d_ctl, h->d_dlt, h->d_qsort, h->d_qsort + kDltSortMax);
    CKL(h);
    dlt_build_kernel<<<kDltQ, kDltBuildThreads, 0, h->stream>>>(h->d_front, h->d_ctl, h->d_dlt);
    CKL(h);
    return SW_OK;
}

// ---- the device-sized merge pipeline: work[0, ctl.m_in) -> exact front in `out`
// (two block-local passes in smem, a global O(m'^2) mark, compaction, rank sort).
// Grids are sized for the capacity; blocks beyond the live count exit at once.
static sw_status reduce_async(sw_plan* h, PPoint* out) {
    if (h->coop_reduce) {  // one cooperative launch for the whole merge
        PPoint* work = h->d_work;
        PPoint* tmp2 = h->d_tmp2;
        uint8_t* keep = h->d_keep;
        ParetoCtl* ctl = h->d_ctl;
        uint64_t cap = h->front_cap;
        PPoint* sorted = h->d_tmp;
        uint32_t* hist = h->d_rhist;
        void* args[] = {&work, &tmp2, &keep, &out, &ctl, &cap, &sorted, &hist};
        CK(h, cudaLaunchCooperativeKernel((const void*)pareto_reduce_kernel, dim3(h->coop_grid), dim3(kRedThreads),
                                          args, 0, h->stream));
        h->launches++;
        return SW_OK;
    }
    const uint64_t U = h->front_cap + h->surv_cap;
    ParetoCtl* c = h->d_ctl;
    const uint32_t gl = (uint32_t)((U + kLocal - 1) / kLocal), gs = (uint32_t)((U + kScanThreads - 1) / kScanThreads);
    const uint32_t gls = (uint32_t)((U + kLocalSmall - 1) / kLocalSmall);
    CK(h, cudaMemsetAsync(&c->m_loc, 0, 3 * sizeof(uint32_t), h->stream));  // m_loc, m_loc2, m_cmp
    (void)gl;
    pareto_local_kernel<kLocalSmall><<<gls, kLocalSmall, 0, h->stream>>>(h->d_work, &c->m_in, h->d_tmp2, &c->m_loc,
                                                                         h->d_keep);
    CKL(h);
    pareto_mark2d_kernel<<<2 * h->num_sms, kScanThreads, 0, h->stream>>>(h->d_tmp2, &c->m_loc, h->d_keep);
    CKL(h);
    // compaction first: the O(m^2) rank sort then runs over the (few hundred) kept points
    // only (a fused compact+rank over all m measured 7x slower)
    pareto_compact_kernel<<<gs, kScanThreads, 0, h->stream>>>(h->d_tmp2, &c->m_loc, h->d_keep, h->d_work, &c->m_cmp);
    CKL(h);
    pareto_rank_kernel<<<gs, kScanThreads, 0, h->stream>>>(h->d_work, &c->m_cmp, out, c, h->front_cap);
    CKL(h);
    return SW_OK;
}

// Seed the running front from a strided sample of a segment (async).
static sw_status seed_async(sw_plan* h, const Segment& g) {
    const uint64_t n = g.end - g.begin;
    // a strided sample seeds the running front (its exact front is cheap to reduce)
    // (a larger sample for large segments: a better first front cuts the first pass's
    // survivors and its merge)
    uint64_t want = n >= (1ull << 26) ? 32768 : 16384;
    if (const char* ev = getenv("SW_SEED_N")) want = std::max<uint64_t>(1024, strtoull(ev, nullptr, 10));  // experiments
    const uint32_t ns = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(n, want), h->front_cap + h->surv_cap);
    CK(h, cudaMemsetAsync(&h->d_ctl->m_in, 0, sizeof(uint32_t), h->stream));
    pareto_sample_kernel<<<(ns + 255) / 256, 256, 0, h->stream>>>(view_of(h, g, 0, g.ntiles), ns, h->d_work, h->d_ctl);
    CKL(h);
    return reduce_async(h, h->d_front);
}

// Fold a segment chunk by chunk: DLT from the current front, one filter pass over the
// chunk (fused with nq select queries when nq > 0), survivors merged on the device.
// The DLT-survivor buffer of the deferred exact Pareto test: 1/8 of the candidates a pass
// can cover (records held, or a stream shard), 256 K..128 M points -- a pass whose DLT
// survivors overflow it is refolded / re-run; 1/8 is ~5x the DLT pass rate measured (1.5%
// on C3 against the final front).  Grown on demand.
static sw_status ensure_dltc(sw_plan* h, uint64_t candidates) {
    const uint64_t want = std::min<uint64_t>(std::max<uint64_t>(candidates / 8, 1ull << 18), 1ull << 27);
    if (h->d_dltc && h->dltc_cap >= want) return SW_OK;
    if (h->d_dltc) {
        dev_free(h, h->d_dltc);
        h->d_dltc = nullptr;
        h->dltc_cap = 0;
    }
    for (uint64_t c = want;; c /= 2) {
        h->d_dltc = (PPoint*)dev_alloc(h, c * sizeof(PPoint));
        if (h->d_dltc) {
            h->dltc_cap = c;
            return SW_OK;
        }
        if (c <= (1ull << 18)) return fail(h, SW_ENOMEM, "DLT survivor buffer allocation failed");
    }
}

static sw_status fold_chunks_async(sw_plan* h, const Segment& g, uint32_t nq, const SelParams& P, uint32_t* np) {
    if (sw_status st = ensure_dltc(h, h->rec_cap); st < 0) return st;
    const size_t psmem = kScanSmemPareto;
    // strided passes: units of upt tiles (a whole number of scan stages); pass 1 = every
    // 8^K-th unit (about kFirstPass records, at most 1/64 of the segment), each further
    // pass the multiples of the next smaller power of 8 not yet scanned (8x more) -- each a
    // uniform sample of the segment, so the front (and its DLT filter) is close to final
    // early and every pass's survivors stay bounded.  Small segments: one pass.
    const uint64_t per_tile = kTileRows * h->row;
    uint32_t upt = 1;
    while ((upt * per_tile) % kUnitAlign) upt++;
    const uint64_t unit_recs = upt * per_tile;
    const uint64_t total = g.ntiles * per_tile;
    const uint64_t nunits = (total + unit_recs - 1) / unit_recs;
    // K levels: the first pass covers about kFirstPass records (>= 1/64 of the segment)
    const uint64_t kFirstPass = h->first_pass;
    // a level of more than kMaxPassRecs records is folded in sub-passes of h->sub_pass: for
    // segments of >= 2^31 records (a big chunk) every level above 256 M -- its survivors
    // against the front of the levels before overflowed the survivor buffer and forced a
    // refold (C5 213 -> 188 ms, same box); smaller segments only above 512 M (C2's 376 M
    // last level unsplit: splitting it cost 1.3%)
    const uint64_t kMaxPassRecs = g.ntiles * kTileRows * h->row >= (1ull << 31) ? h->sub_pass : h->max_pass;
    uint32_t K = h->fold_kmin;
    while (K < 10 && (nunits >> (3 * K)) * unit_recs > kFirstPass) K++;
    const bool strided = nunits >= 256;
    const uint64_t last_short = nunits * unit_recs - total;  // missing slots of the last unit
    const uint32_t npass = strided ? K + 1 : 1;
    for (uint32_t pi = 0; pi < npass; pi++) {
        const uint32_t pass = strided ? pi + 1 : 0;
        const uint32_t lvl = pi, sh = 3 * (K - lvl);
        uint64_t units = nunits;
        bool has_last = true;
        if (strided) {
            const uint64_t c_here = (nunits + (1ull << sh) - 1) >> sh;
            const uint64_t c_up = lvl ? (nunits + (1ull << (sh + 3)) - 1) >> (sh + 3) : 0;
            units = c_here - c_up;
            const uint64_t L = nunits - 1;  // does this pass hold the (possibly short) last unit?
            has_last = (L % (1ull << sh) == 0) && (lvl == 0 || L % (1ull << (sh + 3)) != 0);
        }
        const uint64_t recs_level = units * unit_recs - (has_last ? last_short : 0);
        // a huge pass (a big chunk's last level) is folded in sub-passes of <= kMaxPassRecs:
        // its survivors of the exact test against a front from much fewer records would
        // overflow the survivor buffer and force a refold (a second read of the pass)
        const uint64_t nsub = strided && recs_level > kMaxPassRecs
                                  ? (recs_level + h->sub_pass - 1) / h->sub_pass : 1;
        for (uint64_t si = 0; si < nsub; si++) {
        const uint64_t j0 = units * si / nsub, j1 = units * (si + 1) / nsub;
        const uint64_t recs = nsub == 1 ? recs_level
                                        : (j1 - j0) * unit_recs - (has_last && j1 == units ? last_short : 0);
        SegView v = view_of(h, g, 0, g.ntiles);
        v.pass = pass;
        v.upt = upt;
        v.levels = K;
        v.j0 = (uint32_t)j0;
        v.j1 = nsub == 1 ? 0xffffffffu : (uint32_t)j1;
        if (sw_status ds = dlt_build_async(h); ds < 0) return ds;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(1, recs / (kStageRecs * kCW)), h->scan_grid);
        Cand* part = h->d_partial;
        if (nq) {
            if (*np + grid > h->max_partial) return fail(h, SW_ERANGE, "too many chunks for one select");
            part = h->d_partial + (uint64_t)*np * SW_MAX_QUERIES;
            *np += grid;
        }
        int pr = 0;
        sw_status ts = begin_timed(h, SW_KERNEL_SCAN, recs * sizeof(Rec4), &pr);
        if (ts < 0) return ts;
        trace_mark(h, "dlt");
        launch_scan_nq<true>(nq, grid, psmem, h->stream, v, P, part, pareto_args(h));
        CKL(h);
        if ((ts = end_timed(h, pr)) < 0) return ts;
        trace_mark(h, pass == 1 ? "scan1" : pass == 2 ? "scan2" : pass == 3 ? "scan3" : pass == 4 ? "scan4" : "scan");
        // the pass's DLT survivors: exact test against the running front (grid-stride over
        // the device-side count)
        pareto_exact_kernel<<<h->num_sms, kExactThreads, exact_smem_bytes(), h->stream>>>(
            h->d_dltc, h->dltc_cap, h->d_front, h->d_ctl, h->d_surv, h->surv_cap);
        CKL(h);
        trace_mark(h, "exact");
        pareto_append_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_front, h->d_surv, h->surv_cap, h->d_work,
                                                               h->d_ctl);
        CKL(h);
        if (h->dump_merge) {  // diagnostics only (merge experiments): the merge input, raw PPoints
            ParetoCtl c;
            CK(h, cudaMemcpyAsync(&c, h->d_ctl, sizeof c, cudaMemcpyDeviceToHost, h->stream));
            SYNC(h);
            std::vector<PPoint> buf(c.m_in);
            CK(h, cudaMemcpy(buf.data(), h->d_work, sizeof(PPoint) * c.m_in, cudaMemcpyDeviceToHost));
            char path[512];
            snprintf(path, sizeof path, "%s_%llu.bin", h->dump_merge, (unsigned long long)h->fold_passes + 1);
            if (FILE* f = fopen(path, "wb")) {
                fwrite(&c.front_n, sizeof(uint64_t), 1, f);  // the running front = the first front_n points
                fwrite(buf.data(), sizeof(PPoint), buf.size(), f);
                fclose(f);
            }
        }
        sw_status st = reduce_async(h, h->d_front);
        if (st < 0) return st;
        trace_mark(h, "merge");
        h->fold_passes++;
        h->epoch++;
        if (h->debug) {  // diagnostics only: synchronises every pass
            ParetoCtl c;
            CK(h, cudaMemcpyAsync(&c, h->d_ctl, sizeof c, cudaMemcpyDeviceToHost, h->stream));
            SYNC(h);
            fprintf(stderr, "[sw] dlt passed %llu records in this pass\n", (unsigned long long)c.dlt_n);
            fprintf(stderr, "[sw] fold pass %llu: stride pass %u, %llu records, survivors %llu merge-in %u local %u/%u front %llu"
                            " | merge phases us: init %.1f local %.1f mark %.1f compact %.1f rank(b0) %.1f\n",
                    (unsigned long long)h->fold_passes, pass, (unsigned long long)recs,
                    (unsigned long long)c.surv, c.m_in, c.m_loc, c.m_loc2, (unsigned long long)c.front_n,
                    1e-3 * (double)(c.stamp[1] - c.stamp[0]), 1e-3 * (double)(c.stamp[2] - c.stamp[1]),
                    1e-3 * (double)(c.stamp[3] - c.stamp[2]), 1e-3 * (double)(c.stamp[4] - c.stamp[3]),
                    1e-3 * (double)(c.stamp[5] - c.stamp[4]));
        }
        }  // sub-passes
    }
    return SW_OK;
}

// Read back the pipeline state (sync).  Returns SW_ERANGE on a front overflow; sets
// *overflow if some filter pass had more survivors than capacity (refold needed).
static sw_status sync_ctl(sw_plan* h, bool* overflow) {
    ParetoCtl c;
    CK(h, cudaMemcpyAsync(&c, h->d_ctl, sizeof c, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    if (c.front_overflow) return fail(h, SW_ERANGE, "Pareto front exceeds %llu points", (unsigned long long)h->front_cap);
    h->front_n = c.front_n;
    *overflow = c.surv_overflow != 0;
    if (c.surv_overflow) CK(h, cudaMemsetAsync(&h->d_ctl->surv_overflow, 0, sizeof(uint32_t), h->stream));
    if (c.dlt_max > h->dltc_cap) {  // a loose DLT (e.g. discrete qualities): grow the buffer so
                                    // the refold does not drop survivors again
        sw_status st = ensure_dltc(h, c.dlt_max * 10);
        if (st < 0) return st;
    }
    return SW_OK;
}

// The exact global front, launched asynchronously: 1 rank -> the running front and its
// device-side size; several -> counts and fronts padded to kMergePad points allgathered,
// concatenated and merged on the device into d_gather (size in d_counts[R+2]); the local
// front size is saved and restored on the device.  Cached per state epoch.  Collective.
// After the caller's sync, finish_global_front() records the cache or reports that some
// front exceeded the pad (then the synchronous global_front() redoes the merge).
static constexpr uint32_t kMergePad = 4096;

static sw_status global_front_async(sw_plan* h, const PPoint** res, const uint64_t** d_n, bool* launched) {
    *launched = false;
    if (h->nranks == 1) {
        *res = h->d_front;
        *d_n = &h->d_ctl->front_n;
        return SW_OK;
    }
    const int R = h->nranks;
    *res = h->d_gather;
    *d_n = h->d_counts + R + 2;
    if (h->merged_epoch == h->gepoch) return SW_OK;  // cached merge, size already on device
    ParetoCtl* c = h->d_ctl;
    CK(h, cudaMemcpyAsync(h->d_counts + R, &c->front_n, 8, cudaMemcpyDeviceToDevice, h->stream));
    CK(h, cudaMemcpyAsync(h->d_counts + R + 1, &c->front_n, 8, cudaMemcpyDeviceToDevice, h->stream));
    CKC(h, coll_allgather(coll_of(h), h->d_counts + R, h->d_counts, 8, &why_));
    CKC(h, coll_allgather(coll_of(h), h->d_front, h->d_gather, (size_t)kMergePad * sizeof(PPoint), &why_));
    const uint64_t all = (uint64_t)kMergePad * R;
    front_gather_pad_kernel<<<(uint32_t)((all + 255) / 256), 256, 0, h->stream>>>(
        h->d_gather, h->d_counts, R, kMergePad, h->d_work, c, h->d_counts + R + 3);
    CKL(h);
    sw_status st = reduce_async(h, h->d_gather);
    if (st < 0) return st;
    CK(h, cudaMemcpyAsync(h->d_counts + R + 2, &c->front_n, 8, cudaMemcpyDeviceToDevice, h->stream));
    CK(h, cudaMemcpyAsync(&c->front_n, h->d_counts + R + 1, 8, cudaMemcpyDeviceToDevice, h->stream));
    *launched = true;
    return SW_OK;
}

// Winners of front-answerable queries (R30) from the exact global front, synchronous
// (fallback path).  Collective.
static sw_status front_answer(sw_plan* h, uint32_t nq, const sw_query* qs, sw_selection* out) {
    const PPoint* fr = nullptr;
    uint64_t n = 0;
    sw_status st = global_front(h, &fr, &n);
    if (st < 0) return st;
    SelParams P{};
    P.nq = nq;
    P.objective = (h->h.flags & 4u) ? 1u : 0u;
    for (uint32_t q = 0; q < nq; q++) P.q[q] = QueryDev{qs[q].slo_startup_us, qs[q].slo_stall_us, qs[q].budget_mc};
    select_front_kernel<<<1, kScanThreads, 0, h->stream>>>(fr, n, nullptr, P, h->d_cand);
    CKL(h);
    if (sw_status ds = launch_detail(h, nq); ds < 0) return ds;
    Cand win[SW_MAX_QUERIES];
    DetailOut det[SW_MAX_QUERIES];
    CK(h, cudaMemcpyAsync(win, h->d_cand, sizeof(Cand) * nq, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(det, h->d_detail, sizeof(DetailOut) * nq, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    sw_status worst = SW_OK;
    for (uint32_t q = 0; q < nq; q++) {
        memset(&out[q], 0, sizeof(sw_selection));
        if (win[q].idx == kInf64) {
            out[q].status = SW_EMPTY;
        } else {
            detail_to_selection(h, win[q].idx, det[q], &out[q], nullptr);
            out[q].status = win[q].pad ? SW_CLOSEST : SW_OK;
        }
        worst = std::max<sw_status>(worst, out[q].status);
    }
    return worst;
}

// A query is front-answerable (R30) when it bounds neither startup nor stall under the
// QUALITY_FIRST objective (and the handle's front covers exactly its records).
// Under COST_X_TTFF the same holds when every record has cost > 0 and ttff_eff > 0
// (reading R35): then a dominating point has a strictly smaller cost x ttff_eff product
// unless only its quality is better, which the key's -Q breaks in its favour.
static bool front_query(const sw_plan* h, const sw_query& q) {
    return h->fuse_pareto && (!(h->h.flags & 4u) || h->cxt_front_ok) && q.slo_startup_us == UINT64_MAX &&
           q.slo_stall_us == UINT64_MAX;
}

// Select over the held records.  Scan queries (S) ride on the fused select + Pareto-fold
// scans (or a plain scan of already folded segments); front-answerable queries (F, when
// allow_front) are reduced over the exact global front.  Everything -- scans, folds,
// merges, allgathers, every winner's detail -- is launched asynchronously and read back
// with ONE synchronisation; a Pareto capacity overflow falls back to the synchronous
// refold + front answer.  Collective when nranks > 1.
// Fingerprint of a collective call's arguments (order-sensitive 64-bit mix): ranks that
// disagree are detected by the status-word reduction and fail with SW_ESTATE together.
static uint64_t fp_mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}
static uint64_t call_fingerprint(const sw_plan* h, uint32_t kind, uint32_t nq, const sw_query* qs, uint64_t a,
                                 uint64_t b) {
    uint64_t f = fp_mix(0x5357u, kind);
    f = fp_mix(f, h->N);
    f = fp_mix(f, nq);
    for (uint32_t q = 0; q < nq; q++) {
        f = fp_mix(f, qs[q].slo_startup_us);
        f = fp_mix(f, qs[q].slo_stall_us);
        f = fp_mix(f, qs[q].budget_mc);
    }
    f = fp_mix(f, a);
    f = fp_mix(f, b);
    for (const Segment& g : h->segs) {
        f = fp_mix(f, g.gbegin);
        f = fp_mix(f, g.gend);
    }
    return f;
}

// Launch the status words of this call and max-reduce them over the ranks (no-op at one
// rank); the caller reads them back with its answers.
static sw_status status_exchange(sw_plan* h, const uint32_t* cand_n, uint32_t nq, uint32_t cap, uint64_t host_flag,
                                 uint64_t fp) {
    if (h->nranks == 1) return SW_OK;
    uint64_t* d_st = h->d_counts + h->nranks + 4;
    status_words_kernel<<<1, 1, 0, h->stream>>>(h->d_ctl, cand_n, nq, cap, host_flag, fp, d_st);
    CKL(h);
    CKC(h, coll_allreduce_u64(coll_of(h), d_st, kStatusWords, 1, &why_));
    return SW_OK;
}

static sw_status select_impl(sw_plan* h, uint32_t nq, const sw_query* qs, sw_selection* out, bool allow_front) {
    uint32_t fi[SW_MAX_QUERIES], si[SW_MAX_QUERIES], nf = 0, ns = 0;
    for (uint32_t q = 0; q < nq; q++) {
        if (allow_front && front_query(h, qs[q])) fi[nf++] = q;
        else si[ns++] = q;
    }
    SelParams PS{}, PF{};
    PS.objective = PF.objective = (h->h.flags & 4u) ? 1u : 0u;
    PS.nq = ns;
    PF.nq = nf;
    for (uint32_t j = 0; j < ns; j++)
        PS.q[j] = QueryDev{qs[si[j]].slo_startup_us, qs[si[j]].slo_stall_us, qs[si[j]].budget_mc};
    for (uint32_t j = 0; j < nf; j++)
        PF.q[j] = QueryDev{qs[fi[j]].slo_startup_us, qs[fi[j]].slo_stall_us, qs[fi[j]].budget_mc};
    uint32_t np = 0;
    std::vector<size_t> fused;
    trace_mark(h, "start");
    CK(h, cudaMemsetAsync(h->d_gfeas, 0, sizeof(uint32_t) * kGSelWords, h->stream));
    bool seeded = h->front_n > 0;
    for (size_t si_ = 0; si_ < h->segs.size(); si_++) {
        Segment& g = h->segs[si_];
        const uint64_t n = g.end - g.begin;
        if (n == 0) continue;
        if (h->fuse_pareto && !g.folded) {  // a8 rides on the same 32 B loads as a9
            if (!seeded) {
                sw_status st = seed_async(h, g);
                if (st < 0) return st;
                seeded = true;
                trace_mark(h, "seed");
            }
            sw_status st = fold_chunks_async(h, g, ns, PS, &np);
            if (st < 0) return st;
            g.folded = true;
            fused.push_back(si_);
        } else if (ns) {
            const uint32_t grid = (uint32_t)std::min<uint64_t>(g.ntiles, h->scan_grid);
            if (np + grid > h->max_partial) return fail(h, SW_ERANGE, "too many segments for one select");
            int pr = 0;
            sw_status ts = begin_timed(h, SW_KERNEL_SCAN, g.ntiles * kTileRows * h->row * sizeof(Rec4), &pr);
            if (ts < 0) return ts;
            launch_scan_nq<false>(ns, grid, kRingBytes, h->stream, view_of(h, g, 0, g.ntiles), PS,
                                  h->d_partial + (uint64_t)np * SW_MAX_QUERIES, pareto_args(h));
            CKL(h);
            if ((ts = end_timed(h, pr)) < 0) return ts;
            np += grid;
        }
    }
    trace_mark(h, "folds");
    if (ns) {
        if (np == 0) {  // empty local contribution: a row of "none" candidates
            std::vector<Cand> none(SW_MAX_QUERIES);
            for (auto& c : none) c.idx = kInf64;
            CK(h, cudaMemcpyAsync(h->d_partial, none.data(), sizeof(Cand) * SW_MAX_QUERIES, cudaMemcpyHostToDevice,
                                  h->stream));
            np = 1;
        }
        select_final_kernel<<<1, kScanThreads, 0, h->stream>>>(h->d_partial, np, PS, h->d_cand);
        CKL(h);
        if (h->nranks > 1) {  // a10: allgather per-rank winners over NVLink, replicated merge
            CKC(h, coll_allgather(coll_of(h), h->d_cand, h->d_cand_all, sizeof(Cand) * SW_MAX_QUERIES, &why_));
            select_final_kernel<<<1, kScanThreads, 0, h->stream>>>(h->d_cand_all, (uint32_t)h->nranks, PS, h->d_cand);
            CKL(h);
        }
    }
    trace_mark(h, "select");
    {
        sw_status st = status_exchange(h, nullptr, 0, 0, 0, call_fingerprint(h, 1, nq, qs, allow_front, 0));
        if (st < 0) return st;
    }
    bool merged_now = false;
    if (nf) {
        const PPoint* fr = nullptr;
        const uint64_t* d_n = nullptr;
        sw_status st = global_front_async(h, &fr, &d_n, &merged_now);
        if (st < 0) return st;
        trace_mark(h, "front_merge");
        select_front_kernel<<<1, kScanThreads, 0, h->stream>>>(fr, 0, d_n, PF, h->d_cand + ns);
        CKL(h);
    }
    // every winner's full metrics in one launch, read back with the winners (one sync)
    const uint32_t nw = ns + nf;
    if (sw_status ds = launch_detail(h, nw); ds < 0) return ds;
    Cand win[SW_MAX_QUERIES];
    DetailOut det[SW_MAX_QUERIES];
    ParetoCtl cc;
    // merged front size, pad overflow, then the max-reduced status words (multi-rank)
    uint64_t aux[2 + kStatusWords] = {};
    CK(h, cudaMemcpyAsync(win, h->d_cand, sizeof(Cand) * nw, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(det, h->d_detail, sizeof(DetailOut) * nw, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(&cc, h->d_ctl, sizeof cc, cudaMemcpyDeviceToHost, h->stream));
    if (h->nranks > 1)
        CK(h, cudaMemcpyAsync(aux, h->d_counts + h->nranks + 2, sizeof aux, cudaMemcpyDeviceToHost, h->stream));
    trace_mark(h, "answers");
    SYNC(h);
    trace_dump(h, "select");
    // every branch below that leads to another collective is taken on the status words
    // reduced over ALL ranks, so the ranks stay in step (a rank-local overflow would
    // otherwise send only that rank into the exact front redo's collectives)
    const uint64_t* gst = aux + 2;
    const bool g_surv = h->nranks > 1 ? gst[0] != 0 : cc.surv_overflow != 0;
    const bool g_front = h->nranks > 1 ? gst[1] != 0 : cc.front_overflow != 0;
    if (h->nranks > 1 && gst[4] != ~gst[5])
        return fail(h, SW_ESTATE, "ranks made different select calls (arguments or evaluated ranges differ)");
    if (g_front) return fail(h, SW_ERANGE, "Pareto front exceeds %llu points", (unsigned long long)h->front_cap);
    h->front_n = cc.front_n;
    bool redo_front = false;
    if (cc.surv_overflow) {  // a local filter pass overflowed: the local front is valid but incomplete
        CK(h, cudaMemsetAsync(&h->d_ctl->surv_overflow, 0, sizeof(uint32_t), h->stream));
        for (size_t x : fused) h->segs[x].folded = false;
    }
    if (g_surv) redo_front = nf > 0;  // some rank's front is incomplete: every rank redoes
    if (merged_now) {
        if (aux[1]) redo_front = nf > 0;  // some rank's front exceeded the pad
        else if (!g_surv) {
            h->merged_epoch = h->gepoch;
            h->merged_n = aux[0];
        }
    }
    sw_status worst = SW_OK;
    for (uint32_t j = 0; j < nw; j++) {
        const uint32_t q = j < ns ? si[j] : fi[j - ns];
        memset(&out[q], 0, sizeof(sw_selection));
        if (win[j].idx == kInf64) {
            out[q].status = SW_EMPTY;
        } else {
            detail_to_selection(h, win[j].idx, det[j], &out[q], nullptr);
            out[q].status = win[j].pad ? SW_CLOSEST : SW_OK;  // feasibility flag set on device
        }
        worst = std::max<sw_status>(worst, out[q].status);
    }
    if (redo_front) {  // rare: exact refold, full-size merge, answer again
        sw_query qf[SW_MAX_QUERIES];
        sw_selection of[SW_MAX_QUERIES];
        for (uint32_t j = 0; j < nf; j++) qf[j] = qs[fi[j]];
        sw_status st = front_answer(h, nf, qf, of);
        if (st < 0) return st;
        worst = SW_OK;
        for (uint32_t j = 0; j < nf; j++) out[fi[j]] = of[j];
        for (uint32_t q = 0; q < nq; q++) worst = std::max<sw_status>(worst, out[q].status);
    }
    return worst;
}

extern "C" sw_status sw_plan_select_batch(sw_plan* h, uint32_t nq, const sw_query* qs, sw_selection* out) {
    const NvtxRange nvtx_("sw_plan_select_batch");
    if (!h || !qs || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (nq < 1 || nq > SW_MAX_QUERIES) return fail(h, SW_EINVAL, "n_queries %u not in 1..%d", nq, SW_MAX_QUERIES);
    CK(h, cudaSetDevice(h->device));
    return select_impl(h, nq, qs, out, !h->released);
}

extern "C" sw_status sw_plan_select(sw_plan* h, uint64_t slo_startup_us, uint64_t slo_stall_us, uint64_t budget_mc,
                                    sw_selection* out) {
    sw_query q{slo_startup_us, slo_stall_us, budget_mc};
    return sw_plan_select_batch(h, 1, &q, out);
}

extern "C" sw_status sw_plan_detail(sw_plan* h, uint64_t index, sw_selection* out, uint64_t* ready_us) {
    const NvtxRange nvtx_("sw_plan_detail");
    if (!h || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (index >= h->N) return fail(h, SW_EINVAL, "index out of range");
    CK(h, cudaSetDevice(h->device));
    memset(out, 0, sizeof *out);
    sw_status st = fill_detail(h, index, out, ready_us);
    if (st < 0) return st;
    out->status = SW_OK;
    return SW_OK;
}

// ============================================================================ chunked sweep
extern "C" sw_status sw_plan_sweep(sw_plan* h, uint64_t begin, uint64_t end, uint64_t chunk, uint32_t nq,
                                   const sw_query* qs, sw_selection* out, uint64_t* digest) {
    const NvtxRange nvtx_("sw_plan_sweep");
    if (!h || (nq && (!qs || !out))) return fail(nullptr, SW_EINVAL, "null argument");
    if (nq > SW_MAX_QUERIES) return fail(h, SW_EINVAL, "n_queries %u > %d", nq, SW_MAX_QUERIES);
    if (begin > end || end > h->N) return fail(h, SW_EINVAL, "range outside [0, N)");
    if (!h->segs.empty()) return fail(h, SW_ESTATE, "sweep needs a handle without records (reset/release)");
    // largest global chunk whose every rank shard fits the per-rank capacity: whole
    // rows per rank, at most cand_cap - row candidates each (ragged ends fit the slack)
    // one rank: the shard is the chunk; several: whole rows split evenly (<= one extra
    // row per rank) plus a ragged head / tail of under a row each
    uint64_t max_chunk = h->cand_cap;
    if (h->nranks > 1)
        max_chunk = h->cand_cap > 3 * h->row ? (h->cand_cap - 3 * h->row) / h->row * h->row * (uint64_t)h->nranks : 0;
    if (chunk == 0) chunk = max_chunk;
    if (chunk == 0 || chunk > max_chunk)
        return fail(h, SW_ERANGE, "chunk %llu exceeds what record_capacity %llu allows (%llu)",
                    (unsigned long long)chunk, (unsigned long long)h->cand_cap, (unsigned long long)max_chunk);
    for (uint32_t q = 0; q < nq; q++) {
        memset(&out[q], 0, sizeof(sw_selection));
        out[q].status = SW_EMPTY;
    }
    uint64_t dsum = 0;
    sw_selection tmp[SW_MAX_QUERIES];
    // front-answerable queries (R30) are answered once from the final front when that
    // front covers exactly [begin, end) (empty front at the start); the others per chunk
    const bool front_ok = h->front_n == 0 && !h->released && h->segs.empty();
    uint32_t fi[SW_MAX_QUERIES], si[SW_MAX_QUERIES], nf = 0, ns = 0;
    sw_query qsn[SW_MAX_QUERIES];
    for (uint32_t q = 0; q < nq; q++) {
        if (front_ok && front_query(h, qs[q])) fi[nf++] = q;
        else qsn[ns] = qs[q], si[ns++] = q;
    }
    if (front_ok && nf && end - begin <= chunk && !digest) {
        // one chunk: the front after its fold covers exactly [begin, end), so every query
        // goes through one select (front-answerable ones from that front, one readback)
        sw_status st = sw_plan_eval(h, begin, end);
        if (st < 0) return st;
        const sw_status sel = select_impl(h, nq, qs, out, true);
        if (sel < 0) return sel;
        if ((st = sw_plan_release_records(h)) < 0) return st;
        return sel;
    }
    for (uint64_t c0 = begin; c0 < end;) {
        const uint64_t c1 = end - c0 > chunk ? c0 + chunk : end;
        sw_status st = sw_plan_eval(h, c0, c1);
        if (st < 0) return st;
        if (ns) {
            st = select_impl(h, ns, qsn, tmp, false);  // also folds the chunk into the front
            if (st < 0) return st;
            for (uint32_t j = 0; j < ns; j++)
                sw_selection_merge(h->h.flags & 4u ? 1u : 0u, &qsn[j], &out[si[j]], &tmp[j], &out[si[j]]);
        }
        if (digest) {
            uint64_t d = 0;
            st = sw_plan_digest(h, &d);
            if (st < 0) return st;
            dsum += d;
        }
        st = sw_plan_release_records(h);  // folds whatever is still pending, drops the records
        if (st < 0) return st;
        c0 = c1;
    }
    if (nf) {
        sw_query qf[SW_MAX_QUERIES];
        for (uint32_t j = 0; j < nf; j++) qf[j] = qs[fi[j]];
        sw_status st = front_answer(h, nf, qf, tmp);
        if (st < 0) return st;
        for (uint32_t j = 0; j < nf; j++) out[fi[j]] = tmp[j];
    }
    if (digest) *digest = dsum;
    sw_status worst = SW_OK;
    for (uint32_t q = 0; q < nq; q++) worst = std::max<sw_status>(worst, out[q].status);
    return worst;
}

// ============================================================================ fused stream
// §8(f) row 1: decode + score + select + Pareto filter in one kernel per strided tile
// pass, no records.  A fresh front is first seeded from 16K candidates spread over the
// shard (evaluated one per thread); the tile hierarchy then mirrors the fold passes
// (fold_chunks_async): pass 0 = every 8^K-th tile of the shard (~1/64), each further pass
// 8x more tiles, each with a DLT from the front so far.
static sw_status stream_setup(sw_plan* h) {
    if (h->d_scand) return SW_OK;
    sw_status st;
    if ((st = alloc_n(h, &h->d_scand, (uint64_t)SW_MAX_QUERIES * h->scand_cap, "stream candidates")) < 0) return st;
    if ((st = alloc_n(h, &h->d_scand_n, SW_MAX_QUERIES, "stream candidate counts")) < 0) return st;
    if ((st = alloc_n(h, &h->d_skey, 3 * SW_MAX_QUERIES, "stream pruning keys")) < 0) return st;
    CK(h, cudaMallocHost((void**)&h->h_pass_surv, 64 * sizeof(uint64_t)));  // [lvl] survivors, [32+lvl] DLT survivors
    h->stream_smem = ((sizeof(DevHeader) + h->va_bytes + 127) & ~(size_t)127) + sizeof(Dlt);
    cudaError_t e = cudaSuccess;
    launch_np(h, [&](auto np) {
        constexpr int NPc = decltype(np)::value;
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
        auto setup = [&](auto kern) {
            cudaFuncAttributes fa{};
            cudaError_t r = cudaFuncGetAttributes(&fa, kern);
            const size_t dyn_max = (size_t)optin > fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
            if (r == cudaSuccess)
                r = dyn_max < h->stream_smem ? cudaErrorInvalidValue
                                             : cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                                    (int)dyn_max);
            int occ = 0;
            if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStreamThreads, h->stream_smem);
            if (r == cudaSuccess && occ < 1) r = cudaErrorLaunchOutOfResources;
            if (r != cudaSuccess && e == cudaSuccess) e = r;
            return occ;
        };
        h->stream_occ[0] = setup(stream_kernel<NPc, 0>);
        h->stream_occ[1] = setup(stream_kernel<NPc, 1>);
        h->stream_occ[2] = setup(stream_kernel<NPc, 2>);
    });
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(h, SW_ECUDA, "stream kernel cannot launch (%s)", cudaGetErrorString(e));
    }
    return SW_OK;
}

extern "C" sw_status sw_plan_stream(sw_plan* h, uint64_t begin, uint64_t end, uint32_t nq, const sw_query* qs,
                                    sw_selection* out) {
    const NvtxRange nvtx_("sw_plan_stream");
    if (!h || (nq && (!qs || !out))) return fail(nullptr, SW_EINVAL, "null argument");
    if (nq > SW_MAX_QUERIES) return fail(h, SW_EINVAL, "n_queries %u > %d", nq, SW_MAX_QUERIES);
    if (begin > end || end > h->N) return fail(h, SW_EINVAL, "range outside [0, N)");
    if (!h->segs.empty()) return fail(h, SW_ESTATE, "stream needs a handle without records (reset/release)");
    if (h->shared) return fail(h, SW_EINVAL, "the fused stream mode is not available for shared-pool fleets");
    if (h->wide) return fail(h, SW_EINVAL, "the fused stream mode needs pools of <= 8 GPUs (use sw_plan_sweep)");
    CK(h, cudaSetDevice(h->device));
    h->gepoch++;  // the stream folds new candidates into the front (every rank makes this call)
    sw_status st = stream_setup(h);
    if (st < 0) return st;
    // front-answerable queries (R30) come from the front when it covers exactly [begin, end)
    const bool front_ok = h->front_n == 0 && !h->released;
    uint32_t fi[SW_MAX_QUERIES], si[SW_MAX_QUERIES], nf = 0, ns = 0;
    for (uint32_t q = 0; q < nq; q++) {
        if (front_ok && front_query(h, qs[q])) fi[nf++] = q;
        else si[ns++] = q;
    }
    SelParams PS{}, PF{};
    PS.objective = PF.objective = (h->h.flags & 4u) ? 1u : 0u;
    PS.nq = ns;
    PF.nq = nf;
    for (uint32_t j = 0; j < ns; j++)
        PS.q[j] = QueryDev{qs[si[j]].slo_startup_us, qs[si[j]].slo_stall_us, qs[si[j]].budget_mc};
    for (uint32_t j = 0; j < nf; j++)
        PF.q[j] = QueryDev{qs[fi[j]].slo_startup_us, qs[fi[j]].slo_stall_us, qs[fi[j]].budget_mc};
    uint64_t b, e;
    if ((st = sw_shard_range(begin, end, h->row, h->rank, h->nranks, &b, &e)) < 0) return st;
    if ((st = ensure_dltc(h, e - b)) < 0) return st;
    trace_mark(h, "start");
    uint64_t host_err = 0;
    CK(h, cudaMemsetAsync(h->d_scand_n, 0, sizeof(uint32_t) * SW_MAX_QUERIES, h->stream));
    CK(h, cudaMemsetAsync(h->d_skey, 0, sizeof(unsigned long long) * 3 * SW_MAX_QUERIES, h->stream));
    if (e > b) {
        const uint64_t rb = b / h->row, re = (e + h->row - 1) / h->row;
        const uint64_t t0 = rb / kTileRows, t1 = (re + kTileRows - 1) / kTileRows, nt = t1 - t0;
        const uint64_t per_tile = kTileRows * h->row;
        auto up = [](uint64_t n, uint32_t sh) { return (n + (1ull << sh) - 1) >> sh; };  // ceil(n / 2^sh)
        // K levels: pass 0 = about 1/64 of the tiles (its DLT comes from the seed), each
        // further pass 8x more; more levels only while pass 0 alone would exceed the
        // survivor budget if nothing were filtered
        uint32_t K = nt >= 4096 ? 2 : nt >= 64 ? 1 : 0;
        while (K < 20 && up(nt, 3 * K) * per_tile > 64 * (uint64_t)h->surv_cap) K++;
        if (h->front_n == 0) {  // fresh front: seed it from 16K (64K from 2^26 on) candidates spread over the shard
            const uint32_t ns = (uint32_t)std::min<uint64_t>(e - b, (e - b) >> 26 ? 65536 : 16384);
            CK(h, cudaMemsetAsync(&h->d_ctl->m_in, 0, sizeof(uint32_t), h->stream));
            launch_np(h, [&](auto npc) {
                constexpr int NPc = decltype(npc)::value;
                stream_seed_kernel<NPc><<<(ns + 127) / 128, 128, 0, h->stream>>>(h->d_hdr, h->d_va, b, e, ns, h->d_work,
                                                                                h->d_ctl);
            });
            CKL(h);
            if ((st = reduce_async(h, h->d_front)) < 0) return st;
            trace_mark(h, "seed");
        }
        // one pass: DLT from the running front, the fused kernel over the pass's tiles,
        // survivors merged into the front; the pass's survivor count lands in pinned memory
        auto run_pass = [&](uint32_t lvl, uint64_t ntp) -> sw_status {
            if (sw_status ds = dlt_build_async(h); ds < 0) return ds;
            StreamArgs sa{};
            sa.dlt = h->d_dlt;
            sa.gkey = h->d_skey;
            sa.ctl = h->d_ctl;
            sa.pts = h->d_dltc;
            sa.pts_cap = h->dltc_cap;
            sa.cand = h->d_scand;
            sa.cand_n = h->d_scand_n;
            sa.cand_cap = h->scand_cap;
            sa.levels = K;
            sa.lvl = lvl;
            sa.ntiles_pass = ntp;
            sa.ib = b;
            sa.ie = e;
            sa.P = PS;
            const uint64_t warps_per_block = kStreamThreads / 32;
            const uint64_t max_blocks = (uint64_t)h->num_sms * std::max(1, h->stream_occ[eval_mode(h->h.flags)]);
            // a warp works a whole tile (32 rows x row candidates): a pass of few tiles is
            // split into MID-digit slices so that it has >= 2 work items per warp slot
            const uint64_t slots = max_blocks * warps_per_block;
            const uint32_t rm = h->h.radix[h->h.B - 2];
            sa.msplit = (uint32_t)std::min<uint64_t>(rm, std::max<uint64_t>(1, (2 * slots + ntp - 1) / ntp));
            const uint64_t nwork = ntp * sa.msplit;
            const uint32_t grid = (uint32_t)std::min<uint64_t>((nwork + warps_per_block - 1) / warps_per_block, max_blocks);
            int pr = 0;
            sw_status ts = begin_timed(h, SW_KERNEL_STREAM, 0, &pr);
            if (ts < 0) return ts;
            launch_np(h, [&](auto npc) {
                constexpr int NPc = decltype(npc)::value;
                const EvalJob job{h->d_hdr, h->d_va, h->va_bytes, t0, t1, nullptr};
                switch (eval_mode(h->h.flags)) {
                    case 0: stream_kernel<NPc, 0><<<grid, kStreamThreads, h->stream_smem, h->stream>>>(job, sa); break;
                    case 1: stream_kernel<NPc, 1><<<grid, kStreamThreads, h->stream_smem, h->stream>>>(job, sa); break;
                    default: stream_kernel<NPc, 2><<<grid, kStreamThreads, h->stream_smem, h->stream>>>(job, sa); break;
                }
            });
            CKL(h);
            if ((ts = end_timed(h, pr)) < 0) return ts;
            trace_mark(h, "stream");
            // the pass's DLT survivors: exact test against the running front
            pareto_exact_kernel<<<h->num_sms, kExactThreads, exact_smem_bytes(), h->stream>>>(
                h->d_dltc, h->dltc_cap, h->d_front, h->d_ctl, h->d_surv, h->surv_cap);
            CKL(h);
            trace_mark(h, "exact");
            CK(h, cudaMemcpyAsync(&h->h_pass_surv[lvl], &h->d_ctl->surv, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                  h->stream));
            CK(h, cudaMemcpyAsync(&h->h_pass_surv[32 + lvl], &h->d_ctl->dlt_n, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                  h->stream));
            pareto_append_kernel<<<h->num_sms, 256, 0, h->stream>>>(h->d_front, h->d_surv, h->surv_cap, h->d_work,
                                                                   h->d_ctl);
            CKL(h);
            if ((ts = reduce_async(h, h->d_front)) < 0) return ts;
            trace_mark(h, "merge");
            h->stream_passes++;
            h->epoch++;
            if (h->debug) {
                ParetoCtl c;
                uint32_t cn[SW_MAX_QUERIES];
                CK(h, cudaMemcpyAsync(&c, h->d_ctl, sizeof c, cudaMemcpyDeviceToHost, h->stream));
                CK(h, cudaMemcpyAsync(cn, h->d_scand_n, sizeof cn, cudaMemcpyDeviceToHost, h->stream));
                SYNC(h);
                fprintf(stderr, "[sw] stream pass %u/%u: %llu tiles, survivors %llu front %llu, candidates reported",
                        lvl, K, (unsigned long long)ntp, (unsigned long long)c.surv, (unsigned long long)c.front_n);
                for (uint32_t q = 0; q < ns; q++) fprintf(stderr, " %u", cn[q]);
                fprintf(stderr, "\n");
            }
            return SW_OK;
        };
        auto ntiles_of = [&](uint32_t lvl) {
            const uint32_t sh = 3 * (K - lvl);
            return up(nt, sh) - (lvl ? up(nt, sh + 3) : 0);
        };
        // A pass whose survivors overflowed dropped some: the merged front is valid (real
        // candidates) but may miss points.  Re-running that pass against the better front
        // is exact -- a record already in the front is removed by its identical entry --
        // and its survivors shrink with the front; it is redone at once (one readback per
        // pass), before the next, larger pass would build on the weaker front.
        // (passes are rank-local: a pass that still overflows after 8 re-runs only sets
        // this rank's error flag; the ranks agree on the outcome after the collectives)
        for (uint32_t lvl = 0; lvl <= K && !host_err; lvl++) {
            const uint64_t ntp = ntiles_of(lvl);
            if (ntp == 0) continue;
            for (int round = 0;; round++) {
                if ((st = run_pass(lvl, ntp)) < 0) return st;
                SYNC(h);
                if (h->h_pass_surv[lvl] <= h->surv_cap && h->h_pass_surv[32 + lvl] <= h->dltc_cap) break;
                if (h->h_pass_surv[32 + lvl] > h->dltc_cap && (st = ensure_dltc(h, h->h_pass_surv[32 + lvl] * 10)) < 0)
                    return st;
                if (round == 8) {
                    host_err = 1;
                    break;
                }
                CK(h, cudaMemsetAsync(&h->d_ctl->surv_overflow, 0, sizeof(uint32_t), h->stream));
            }
        }
    }
    h->released = true;  // the front now covers candidates without records
    if ((st = status_exchange(h, h->d_scand_n, ns, h->scand_cap, host_err,
                              call_fingerprint(h, 2, nq, qs, begin, end))) < 0)
        return st;
    if (ns) {
        stream_select_final_kernel<<<ns, kScanThreads, 0, h->stream>>>(h->d_scand, h->d_scand_n, h->scand_cap, PS,
                                                                      h->d_cand);
        CKL(h);
        if (h->nranks > 1) {  // a10: allgather per-rank winners, replicated merge
            CKC(h, coll_allgather(coll_of(h), h->d_cand, h->d_cand_all, sizeof(Cand) * SW_MAX_QUERIES, &why_));
            select_final_kernel<<<1, kScanThreads, 0, h->stream>>>(h->d_cand_all, (uint32_t)h->nranks, PS, h->d_cand);
            CKL(h);
        }
    }
    bool merged_now = false;
    if (nf) {
        const PPoint* fr = nullptr;
        const uint64_t* d_n = nullptr;
        if ((st = global_front_async(h, &fr, &d_n, &merged_now)) < 0) return st;
        select_front_kernel<<<1, kScanThreads, 0, h->stream>>>(fr, 0, d_n, PF, h->d_cand + ns);
        CKL(h);
    }
    const uint32_t nw = ns + nf;
    if (nw) {
        if (sw_status ds = launch_detail(h, nw); ds < 0) return ds;
    }
    Cand win[SW_MAX_QUERIES];
    DetailOut det[SW_MAX_QUERIES];
    uint32_t cn[SW_MAX_QUERIES];
    ParetoCtl cc;
    uint64_t aux[2 + kStatusWords] = {};  // merged front size, pad overflow, status words
    if (nw) {
        CK(h, cudaMemcpyAsync(win, h->d_cand, sizeof(Cand) * nw, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaMemcpyAsync(det, h->d_detail, sizeof(DetailOut) * nw, cudaMemcpyDeviceToHost, h->stream));
    }
    CK(h, cudaMemcpyAsync(cn, h->d_scand_n, sizeof cn, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(&cc, h->d_ctl, sizeof cc, cudaMemcpyDeviceToHost, h->stream));
    if (h->nranks > 1)
        CK(h, cudaMemcpyAsync(aux, h->d_counts + h->nranks + 2, sizeof aux, cudaMemcpyDeviceToHost, h->stream));
    trace_mark(h, "answers");
    SYNC(h);
    trace_dump(h, "stream");
    // the outcome is decided on the status words reduced over ALL ranks: every rank
    // returns the same status (an error on one rank fails the call everywhere)
    bool g_front = cc.front_overflow != 0, g_surv = cc.surv_overflow != 0 || host_err, g_cand = false;
    for (uint32_t q = 0; q < ns; q++) g_cand |= cn[q] > h->scand_cap;
    if (h->nranks > 1) {
        const uint64_t* gst = aux + 2;
        if (gst[4] != ~gst[5]) return fail(h, SW_ESTATE, "ranks made different stream calls");
        g_front = gst[1] != 0;
        g_surv = gst[0] != 0 || gst[3] != 0;
        g_cand = gst[2] != 0;
    }
    h->front_n = cc.front_n;
    if (cc.surv_overflow) CK(h, cudaMemsetAsync(&h->d_ctl->surv_overflow, 0, sizeof(uint32_t), h->stream));
    if (g_front) return fail(h, SW_ERANGE, "Pareto front exceeds %llu points", (unsigned long long)h->front_cap);
    if (g_surv)
        return fail(h, SW_ERANGE, "stream pass survivors exceeded %llu (on some rank): use sw_plan_sweep",
                    (unsigned long long)h->surv_cap);
    if (g_cand) return fail(h, SW_ERANGE, "stream select candidates exceeded %u (on some rank): use sw_plan_sweep",
                            h->scand_cap);
    if (merged_now && !aux[1]) {
        h->merged_epoch = h->gepoch;
        h->merged_n = aux[0];
    }
    sw_status worst = SW_OK;
    for (uint32_t j = 0; j < nw; j++) {
        const uint32_t q = j < ns ? si[j] : fi[j - ns];
        memset(&out[q], 0, sizeof(sw_selection));
        if (win[j].idx == kInf64) {
            out[q].status = SW_EMPTY;
        } else {
            detail_to_selection(h, win[j].idx, det[j], &out[q], nullptr);
            out[q].status = win[j].pad ? SW_CLOSEST : SW_OK;
        }
        worst = std::max<sw_status>(worst, out[q].status);
    }
    if (merged_now && aux[1] && nf) {  // some rank's front exceeded the merge pad: exact redo
        sw_query qf[SW_MAX_QUERIES];
        sw_selection of[SW_MAX_QUERIES];
        for (uint32_t j = 0; j < nf; j++) qf[j] = qs[fi[j]];
        if ((st = front_answer(h, nf, qf, of)) < 0) return st;
        for (uint32_t j = 0; j < nf; j++) out[fi[j]] = of[j];
        worst = SW_OK;
        for (uint32_t q = 0; q < nq; q++) worst = std::max<sw_status>(worst, out[q].status);
    }
    return worst;
}

// ============================================================================ digest
extern "C" sw_status sw_plan_digest(sw_plan* h, uint64_t* digest) {
    const NvtxRange nvtx_("sw_plan_digest");
    if (!h || !digest) return fail(nullptr, SW_EINVAL, "null argument");
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaMemsetAsync(h->d_digest, 0, sizeof(unsigned long long), h->stream));
    for (const Segment& g : h->segs) {
        if (g.end == g.begin) continue;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(g.ntiles, (uint64_t)h->num_sms * 8);
        digest_kernel<<<grid, kScanThreads, 0, h->stream>>>(view_of(h, g, 0, g.ntiles), h->d_digest);
        CKL(h);
    }
    if (h->nranks > 1)
        CKC(h, coll_allreduce_u64(coll_of(h), (uint64_t*)h->d_digest, 1, 0, &why_));
    unsigned long long v = 0;
    CK(h, cudaMemcpyAsync(&v, h->d_digest, sizeof v, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    *digest = v;
    return SW_OK;
}

// ============================================================================ Pareto
static sw_status fold_segment(sw_plan* h, const Segment& g) {
    if (g.end == g.begin) return SW_OK;
    SelParams P{};
    for (int pass = 0; pass < 16; pass++) {
        if (h->front_n == 0) {
            sw_status st = seed_async(h, g);
            if (st < 0) return st;
        }
        sw_status st = fold_chunks_async(h, g, 0, P, nullptr);
        if (st < 0) return st;
        bool overflow = false;
        st = sync_ctl(h, &overflow);
        if (st < 0) return st;
        if (!overflow) return SW_OK;
        // survivors overflowed: the merged front is a better filter -> refilter
    }
    return fail(h, SW_ERANGE, "Pareto filter did not converge");
}

static sw_status fold_pending(sw_plan* h) {
    CK(h, cudaSetDevice(h->device));
    for (Segment& g : h->segs) {
        if (g.folded) continue;
        sw_status st = fold_segment(h, g);
        if (st < 0) return st;
        g.folded = true;
    }
    return SW_OK;
}

// The exact front of all records since create/reset over ALL ranks: folds pending
// segments, and with nranks > 1 merges the per-rank fronts (allgather of counts, then of
// padded fronts, exact merge; cached until the state changes).  Collective.
static sw_status global_front(sw_plan* h, const PPoint** res_out, uint64_t* n_out) {
    sw_status st = fold_pending(h);
    if (st < 0 && h->nranks == 1) return st;
    const PPoint* res = h->d_front;
    uint64_t n = h->front_n;
    if (h->nranks > 1 && h->merged_epoch == h->gepoch) {  // same state: the cached merge
        if (st < 0) return st;  // (cannot happen: the cache implies complete fronts)
        n = h->merged_n;
        res = h->d_gather;
    } else if (h->nranks > 1) {  // a10: allgather counts, then padded fronts; exact merge
        // a rank whose fold failed still takes part in the count exchange (count = max
        // marks the failure), so every rank fails together instead of hanging its peers
        const std::string err = st < 0 ? h->err : std::string();
        uint64_t mine = st < 0 ? ~0ull : h->front_n;
        CK(h, cudaMemcpyAsync(h->d_counts + h->nranks, &mine, 8, cudaMemcpyHostToDevice, h->stream));
        CKC(h, coll_allgather(coll_of(h), h->d_counts + h->nranks, h->d_counts, 8, &why_));
        std::vector<uint64_t> counts(h->nranks);
        CK(h, cudaMemcpyAsync(counts.data(), h->d_counts, 8 * h->nranks, cudaMemcpyDeviceToHost, h->stream));
        SYNC(h);
        uint64_t maxc = 1, tot = 0;
        for (uint64_t c : counts) {
            if (c == ~0ull)
                return fail(h, st < 0 ? st : SW_ERANGE, "%s", st < 0 ? err.c_str() : "a peer rank's Pareto fold failed");
            maxc = std::max(maxc, c);
            tot += c;
        }
        if (tot > h->front_cap + h->surv_cap) return fail(h, SW_ERANGE, "merged fronts too large");
        CKC(h, coll_allgather(coll_of(h), h->d_front, h->d_gather, maxc * sizeof(PPoint), &why_));
        const uint64_t all = maxc * (uint64_t)h->nranks;
        pareto_gather_kernel<<<(uint32_t)((all + 255) / 256), 256, 0, h->stream>>>(h->d_gather, h->d_counts,
                                                                                  h->nranks, maxc, h->d_work);
        CKL(h);
        uint32_t tot32 = (uint32_t)tot;
        CK(h, cudaMemcpyAsync(&h->d_ctl->m_in, &tot32, sizeof tot32, cudaMemcpyHostToDevice, h->stream));
        // merged front into the gather buffer; the local running front stays intact
        st = reduce_async(h, h->d_gather);
        if (st < 0) return st;
        bool overflow = false;
        st = sync_ctl(h, &overflow);
        if (st < 0) return st;
        n = h->front_n;
        res = h->d_gather;
        h->front_n = mine;
        h->merged_epoch = h->gepoch;
        h->merged_n = n;
        CK(h, cudaMemcpyAsync(&h->d_ctl->front_n, &mine, sizeof mine, cudaMemcpyHostToDevice, h->stream));
        // the asynchronous path reads the cached merge's size from the device
        CK(h, cudaMemcpyAsync(h->d_counts + h->nranks + 2, &n, sizeof n, cudaMemcpyHostToDevice, h->stream));
        SYNC(h);
    }
    *res_out = res;
    *n_out = n;
    return SW_OK;
}

extern "C" sw_status sw_pareto_get(sw_plan* h, sw_pareto_point* out, uint64_t cap, uint64_t* n_out) {
    const NvtxRange nvtx_("sw_pareto_get");
    if (!h || !n_out || (cap && !out)) return fail(nullptr, SW_EINVAL, "null argument");
    const PPoint* res = nullptr;
    uint64_t n = 0;
    sw_status st = global_front(h, &res, &n);
    if (st < 0) return st;
    *n_out = n;
    if (cap == 0) return SW_OK;
    if (cap < n) return SW_TRUNCATED;
    CK(h, cudaMemcpyAsync(out, res, n * sizeof(PPoint), cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    return SW_OK;
}

// ============================================================================ views
extern "C" sw_status sw_plan_records(const sw_plan* h, const sw_record** dev_ptr, uint64_t* n) {
    if (!h || !dev_ptr || !n) return fail(nullptr, SW_EINVAL, "null argument");
    *dev_ptr = (const sw_record*)h->d_rec;
    *n = h->rec_used;
    return SW_OK;
}

extern "C" sw_status sw_plan_segments(const sw_plan* h, sw_segment* out, uint64_t cap, uint64_t* n_out) {
    if (!h || !n_out || (cap && !out)) return fail(nullptr, SW_EINVAL, "null argument");
    *n_out = h->segs.size();
    if (cap == 0) return SW_OK;
    if (cap < h->segs.size()) return SW_TRUNCATED;
    for (size_t i = 0; i < h->segs.size(); i++) {
        const Segment& g = h->segs[i];
        out[i] = sw_segment{g.gbegin, g.gend, g.begin, g.end, g.offset, g.tile0, g.ntiles, h->row};
    }
    return SW_OK;
}

extern "C" sw_status sw_plan_copy_records(sw_plan* h, uint64_t index, uint64_t n, sw_record* host_out) {
    if (!h || (n && !host_out)) return fail(nullptr, SW_EINVAL, "null argument");
    for (const Segment& g : h->segs) {
        if (index >= g.begin && index + n <= g.end) {
            if (n == 0) return SW_OK;
            CK(h, cudaSetDevice(h->device));
            Rec4* tmp = nullptr;
            sw_status st = alloc_n(h, &tmp, n, "record staging");
            if (st < 0) return st;
            gather_records_kernel<<<(uint32_t)((n + 255) / 256), 256, 0, h->stream>>>(view_of(h, g, 0, g.ntiles), index,
                                                                                     n, tmp);
            cudaError_t e1 = cudaGetLastError();
            h->launches++;
            cudaError_t e2 = cudaMemcpyAsync(host_out, tmp, n * sizeof(sw_record), cudaMemcpyDeviceToHost, h->stream);
            dev_free(h, tmp);
            cudaError_t e3 = cudaStreamSynchronize(h->stream);
            if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
                return fail(h, SW_ECUDA, "copy_records failed: %s", cudaGetErrorString(e1 ? e1 : e2 ? e2 : e3));
            return SW_OK;
        }
    }
    return fail(h, SW_EINVAL, "range not inside one local segment");
}

// ============================================================================ greedy planner
extern "C" sw_status sw_plan_greedy(sw_plan* h, uint64_t slo_startup_us, uint64_t slo_stall_us, uint64_t budget_mc,
                                    uint64_t start_index, sw_selection* out, uint32_t* iterations,
                                    uint64_t* evaluations) {
    const NvtxRange nvtx_("sw_plan_greedy");
    if (!h || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (start_index != UINT64_MAX && start_index >= h->N) return fail(h, SW_EINVAL, "start index out of range");
    if (h->shared) return fail(h, SW_EINVAL, "the greedy planner is not available for shared-pool fleets");
    if (h->wide) return fail(h, SW_EINVAL, "the greedy planner needs pools of <= 8 GPUs");
    if (h->level_score.size() > (size_t)kMaxLevels) return fail(h, SW_EINVAL, "greedy supports <= %d levels", kMaxLevels);
    CK(h, cudaSetDevice(h->device));
    GreedyArgs A{};
    A.q = QueryDev{slo_startup_us, slo_stall_us, budget_mc};
    A.objective = (h->h.flags & 4u) ? 1u : 0u;
    A.n_levels = (uint32_t)h->level_score.size();
    for (size_t l = 0; l < h->level_score.size(); l++) A.score[l] = h->level_score[l];
    A.start = start_index == UINT64_MAX ? kInf64 : start_index;
    A.max_iter = 1u << 20;
    launch_np(h, [&](auto np) {
        constexpr int NPc = decltype(np)::value;
        greedy_kernel<NPc><<<1, kGreedyThreads, 0, h->stream>>>(h->d_hdr, h->d_va, A, h->d_greedy);
    });
    CKL(h);
    GreedyOut g;
    CK(h, cudaMemcpyAsync(&g, h->d_greedy, sizeof g, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    sw_status st = fill_detail(h, g.index, out, nullptr);
    if (st < 0) return st;
    out->status = g.feasible ? SW_OK : SW_CLOSEST;
    if (iterations) *iterations = g.iterations;
    if (evaluations) *evaluations = g.evaluations;
    return out->status;
}

// ============================================================================ host helpers
extern "C" sw_status sw_plan_decode(const sw_plan* h, uint64_t index, uint8_t* choice_per_scene) {
    if (!h || !choice_per_scene) return fail(nullptr, SW_EINVAL, "null argument");
    if (h->shared) return fail(nullptr, SW_EINVAL, "sw_plan_decode: a shared-pool fleet has joint digits (sw_shared_detail)");
    if (index >= h->N) return fail(nullptr, SW_EINVAL, "index %llu outside [0, %llu)", (unsigned long long)index,
                                   (unsigned long long)h->N);
    // mixed-radix digits, MSD = earliest block (R19); padded virtual digits have radix 1
    const DevHeader& H = h->h;
    uint64_t rem = index;
    uint32_t dig[kMaxDigits] = {};
    for (int b = (int)H.B - 1; b >= 0; b--) {
        dig[b] = (uint32_t)(rem % H.radix[b]);
        rem /= H.radix[b];
    }
    memset(choice_per_scene, 0, h->S);
    for (uint32_t b = h->pad_digits; b < H.B; b++)
        for (uint32_t s = H.first[b]; s < H.first[b + 1]; s++) choice_per_scene[s] = (uint8_t)dig[b];
    return SW_OK;
}

extern "C" sw_status sw_space_shape(const sw_profile_tables* tb, uint64_t* n, uint64_t* row) {
    if (!tb || !n || !row || !tb->radix) return fail(nullptr, SW_EINVAL, "null argument");
    const uint32_t B = tb->n_digits;
    if (B < 1 || B > SW_MAX_DIGITS) return fail(nullptr, SW_EINVAL, "n_digits %u not in 1..%d", B, SW_MAX_DIGITS);
    uint64_t N = 1;
    for (uint32_t b = 0; b < B; b++) {
        const uint32_t r = tb->radix[b];
        if (r < 1 || r > SW_MAX_CHOICES) return fail(nullptr, SW_EINVAL, "radix[%u] = %u not in 1..%d", b, r, SW_MAX_CHOICES);
        if ((u128)N * r >= ((u128)1 << 63)) return fail(nullptr, SW_ERANGE, "plan space >= 2^63 (InstanceTooLarge)");
        N *= r;
    }
    // digits left-padded with radix 1 to B >= 3: the row is the last two digits
    *row = B == 1 ? (uint64_t)tb->radix[0] : (uint64_t)tb->radix[B - 2] * tb->radix[B - 1];
    *n = N;
    return SW_OK;
}

static Rec4 rec4_of(const sw_record& r) {
    Rec4 x;
    x.w0 = r.ttff_us;
    x.w1 = r.stall_us;
    x.w2 = r.cost_mc;
    x.w3 = (uint64_t)r.quality | ((uint64_t)r.stall_count << 32) | ((uint64_t)r.flags << 48);
    return x;
}

extern "C" sw_status sw_selection_merge(uint32_t objective, const sw_query* q, const sw_selection* a,
                                        const sw_selection* b, sw_selection* out) {
    if (!q || !a || !b || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (objective > 1) return fail(nullptr, SW_EINVAL, "bad objective %u", objective);
    for (const sw_selection* s : {a, b})
        if (s->status != SW_OK && s->status != SW_CLOSEST && s->status != SW_EMPTY)
            return fail(nullptr, SW_EINVAL, "selection status %d is not OK/CLOSEST/EMPTY", s->status);
    const QueryDev qd{q->slo_startup_us, q->slo_stall_us, q->budget_mc};
    const uint64_t ia = a->status == SW_EMPTY ? kInf64 : a->index;
    const uint64_t ib = b->status == SW_EMPTY ? kInf64 : b->index;
    const Rec4 ra = rec4_of(a->rec), rb = rec4_of(b->rec);
    // same total order as the scan / merge kernels (cand_better is __host__ __device__)
    const bool take_b = cand_better(qd, objective, ib, rb, ia, ra);
    const sw_selection w = take_b ? *b : *a;
    *out = w;
    if ((take_b ? ib : ia) == kInf64) out->status = SW_EMPTY;
    else out->status = feasible(qd, take_b ? rb : ra) ? SW_OK : SW_CLOSEST;
    return out->status;
}

// ============================================================================ shared-pool fleet
// SURVEY §8(f) row 4 (reading R36): requests contending for the same pools through per-pool
// EDF queues.  The handle is an ordinary sw_plan over the JOINT plan space of
// the free requests (row = 1, one thread per candidate): eval / select / Pareto / digest /
// sweep / records work unchanged on its fleet records; each request's tables live in a
// tables-only handle (validated and packed -- a_s, P_s, V+A entries -- by sw_plan_create).
extern "C" sw_status sw_shared_create(uint32_t n, const sw_profile_tables* tables, const sw_scene_list* scenes,
                                      const uint64_t* fixed_cost_mc, const sw_shared_request* reqs,
                                      const sw_price_table* pools, const sw_runtime* rt, sw_plan** out) {
    const NvtxRange nvtx_("sw_shared_create");
    if (!tables || !scenes || !reqs || !pools || !rt || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (n < 1 || n > (uint32_t)kShMaxReq) return fail(nullptr, SW_EINVAL, "shared fleet of %u requests (1..%d)", n, kShMaxReq);
    if (pools->evict_risk_permille) return fail(nullptr, SW_EINVAL, "shared pools take no eviction risk");
    if (pools->metric) return fail(nullptr, SW_EINVAL, "shared-pool fleets use the money metric");
    for (uint32_t p = 0; p < pools->n_pools; p++)
        if (pools->gpus[p] > (uint32_t)kMaxG) return fail(nullptr, SW_EINVAL, "shared pools of <= %d GPUs", kMaxG);
    for (uint32_t r = 0; r < n; r++)
        if (tables[r].vae_us) return fail(nullptr, SW_EINVAL, "request %u: DiT/VAE stages are not supported in shared-pool fleets", r);
    if (rt->nranks < 1 || rt->rank < 0 || rt->rank >= rt->nranks)
        return fail(nullptr, SW_EINVAL, "bad rank %d of %d", rt->rank, rt->nranks);
    if (rt->nranks > 1 && !rt->nccl_comm) return fail(nullptr, SW_EINVAL, "nranks > 1 needs nccl_comm");
    uint32_t tot_s = 0, nd = 0;
    uint64_t N = 1;
    for (uint32_t r = 0; r < n; r++) {
        tot_s += scenes[r].n_scenes;
        if (reqs[r].fixed_index == UINT64_MAX) {
            nd += tables[r].n_digits;
            for (uint32_t b = 0; b < tables[r].n_digits && tables[r].radix; b++) {
                if ((u128)N * tables[r].radix[b] >= ((u128)1 << 63))
                    return fail(nullptr, SW_ERANGE, "joint plan space >= 2^63");
                N *= tables[r].radix[b];
            }
        }
    }
    if (tot_s > (uint32_t)kShMaxScenes) return fail(nullptr, SW_EINVAL, "%u scenes over all requests (max %d)", tot_s, kShMaxScenes);
    if (nd > SW_MAX_DIGITS) return fail(nullptr, SW_EINVAL, "%u joint digits over the free requests (max %d)", nd, SW_MAX_DIGITS);
    sw_plan* h = new sw_plan();
    h->shared = new SharedHost();
    auto bail = [&](sw_status st) {
        sw_plan_destroy(h);
        return st;
    };
    h->device = rt->device;
    h->loop = as_loop(rt->nccl_comm);
    h->comm = h->loop ? nullptr : (ncclComm_t)rt->nccl_comm;
    h->rank = rt->rank;
    h->nranks = rt->nranks;
    h->alloc = rt->alloc;
    h->free_fn = rt->free;
    h->alloc_ctx = rt->alloc_ctx;
    if (cudaSetDevice(h->device) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(nullptr, SW_ECUDA, "cudaSetDevice(%d) failed (no CUDA device?)", h->device));
    }
    if (rt->stream) {
        h->stream = (cudaStream_t)rt->stream;
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(nullptr, SW_ECUDA, "cudaStreamCreate failed"));
        h->own_stream = true;
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
    // every request's tables, validated against the shared pools and packed on the device
    SharedDev D{};
    D.R = n;
    D.NP = pools->n_pools;
    D.billing = pools->billing;
    D.nd = nd;
    u128 tbound = 0, qsum = 0, maxT0 = 0;
    uint32_t sc_off = 0, dg = 0;
    for (uint32_t r = 0; r < n; r++) {
        sw_price_table pr = *pools;
        pr.fixed_cost_mc = fixed_cost_mc ? fixed_cost_mc[r] : 0;
        sw_runtime rr{};
        rr.device = rt->device;
        rr.stream = h->stream;
        rr.rank = 0;
        rr.nranks = 1;
        sw_plan* q = nullptr;
        t_tables_only = true;
        sw_status st = sw_plan_create(&tables[r], &scenes[r], &pr, &rr, &q);
        t_tables_only = false;
        if (st < 0) {
            const std::string msg = "request " + std::to_string(r) + ": " + g_last_error;
            bail(st);
            return fail(nullptr, st, "%s", msg.c_str());
        }
        h->shared->reqs.push_back(q);
        if (reqs[r].fixed_index != UINT64_MAX && reqs[r].fixed_index >= q->N)
            return bail(fail(nullptr, SW_EINVAL, "request %u: background plan %llu outside [0, %llu)", r,
                             (unsigned long long)reqs[r].fixed_index, (unsigned long long)q->N));
        SharedReqDev& R = D.req[r];
        R.hdr = q->d_hdr;
        R.va = q->d_va;
        R.T0 = reqs[r].arrival_us;
        R.slo_t = reqs[r].slo_startup_us;
        R.slo_s = reqs[r].slo_stall_us;
        R.S = q->S;
        R.s0 = scenes[r].scene0_static ? 1u : 0u;
        R.B = q->B_user;
        R.pad_digits = q->pad_digits;
        R.free_ = reqs[r].fixed_index == UINT64_MAX ? 1u : 0u;
        R.dig0 = dg;
        R.sc_off = sc_off;
        if (R.free_) {
            for (uint32_t b = 0; b < q->B_user; b++) D.jradix[dg + b] = tables[r].radix[b];
            dg += q->B_user;
        } else {  // the background plan's digits (mixed radix, MSD = earliest block)
            uint64_t rem = reqs[r].fixed_index;
            for (int b = (int)q->B_user - 1; b >= 0; b--) {
                R.fixed_dig[b] = (uint32_t)(rem % tables[r].radix[b]);
                rem /= tables[r].radix[b];
            }
        }
        h->shared->S.push_back(q->S);
        h->shared->sc_off.push_back(sc_off);
        sc_off += q->S;
        // overflow bounds (R25 over the fleet): every task of every request may queue behind
        // every other one -> time bound = latest arrival + pool offset + sum of all stage times
        u128 tr = scenes[r].overhead_us + scenes[r].static_ready_us;
        for (uint32_t s = 0; s < q->S; s++) tr += (u128)scenes[r].llm_us[s] + scenes[r].tts_us[s];
        uint64_t off = 0;
        for (uint32_t b = 0; b < tables[r].n_digits; b++) {
            const uint32_t rb = tables[r].radix[b];
            for (uint32_t s = tables[r].first_scene[b]; s < tables[r].first_scene[b + 1]; s++) {
                uint64_t mx = 0;
                for (uint32_t c = 0; c < rb; c++) mx = std::max(mx, tables[r].va_us[off + (s - tables[r].first_scene[b]) * rb + c]);
                tr += mx;
            }
            off += (uint64_t)(tables[r].first_scene[b + 1] - tables[r].first_scene[b]) * rb;
        }
        tbound += tr;
        maxT0 = std::max<u128>(maxT0, reqs[r].arrival_us);
        uint32_t max_score = 0;
        for (uint32_t l = 0; l < tables[r].n_levels; l++) max_score = std::max(max_score, tables[r].level_score[l]);
        for (uint32_t s = 0; s < q->S; s++) qsum += (u128)(scenes[r].dur_us[s] / 1000) * max_score;
    }
    {
        u128 ready_max = 0;
        for (uint32_t p = 0; p < pools->n_pools; p++) {
            D.G[p] = pools->gpus[p];
            D.price[p] = pools->price_mc_per_gpu_hour[p];
            D.ready[p] = pools->pool_ready_us ? pools->pool_ready_us[p] : 0;
            ready_max = std::max<u128>(ready_max, D.ready[p]);
        }
        tbound += maxT0 + ready_max;
        if (tbound >= ((u128)1 << 62)) return bail(fail(nullptr, SW_ERANGE, "fleet time bound exceeds 2^62 us"));
        if (qsum >= ((u128)1 << 32) - 1) return bail(fail(nullptr, SW_ERANGE, "fleet quality bound exceeds 2^32 - 2"));
        if (tot_s >= (1u << 16)) return bail(fail(nullptr, SW_ERANGE, "fleet stall-count bound"));
        u128 cmax = 0;
        for (uint32_t r = 0; r < n; r++) cmax += fixed_cost_mc ? fixed_cost_mc[r] : 0;
        for (uint32_t p = 0; p < pools->n_pools; p++) {
            const u128 prod = (u128)D.G[p] * tbound * D.price[p] + kHalfHour;
            if (prod >= ((u128)1 << 64)) return bail(fail(nullptr, SW_ERANGE, "cost bound of pool %u exceeds 2^64", p));
            cmax += prod / kUsPerHour;
        }
        if (cmax >= ((u128)1 << 64)) return bail(fail(nullptr, SW_ERANGE, "fleet cost bound exceeds 2^64"));
    }
    // the handle over the joint space: row = 1 (tiles of 32 consecutive candidates)
    h->NP = pools->n_pools;
    h->S = std::min<uint32_t>(tot_s, SW_MAX_SCENES);
    h->B_user = nd;
    h->pad_digits = 0;
    h->N = N;
    h->row = 1;
    DevHeader& H = h->h;
    memset(&H, 0, sizeof H);
    H.flags = (pools->billing ? 2u : 0u) | (pools->objective ? 4u : 0u);
    H.N = N;
    H.row = 1;
    H.n_rows = N;
    h->cxt_front_ok = false;  // lateness can be 0: cost x lateness ties (R35 does not apply)
    if (cudaMalloc(&h->shared->d_dev, sizeof(SharedDev)) != cudaSuccess ||
        cudaMalloc(&h->shared->d_full, sizeof(SharedDetailOut) * SW_MAX_QUERIES) != cudaSuccess ||
        cudaMemcpyAsync(h->shared->d_dev, &D, sizeof D, cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(nullptr, SW_ENOMEM, "shared fleet descriptor allocation failed"));
    }
    sw_status st = create_common(h, rt);
    if (st < 0) return bail(st);
    *out = h;
    return SW_OK;
}

extern "C" sw_status sw_shared_detail(sw_plan* h, uint64_t index, sw_record* per_request, uint64_t* ready_abs) {
    if (!h || !per_request) return fail(nullptr, SW_EINVAL, "null argument");
    if (!h->shared) return fail(h, SW_EINVAL, "not a shared-pool fleet handle");
    if (index >= h->N) return fail(h, SW_EINVAL, "index out of range");
    CK(h, cudaSetDevice(h->device));
    Cand c{};
    c.idx = index;
    CK(h, cudaMemcpyAsync(h->d_cand, &c, sizeof c, cudaMemcpyHostToDevice, h->stream));
    sw_status ds = launch_detail(h, 1);
    if (ds < 0) return ds;
    SharedDetailOut d;
    CK(h, cudaMemcpyAsync(&d, h->shared->d_full, sizeof d, cudaMemcpyDeviceToHost, h->stream));
    SYNC(h);
    const uint32_t n = (uint32_t)h->shared->reqs.size();
    for (uint32_t r = 0; r < n; r++) {
        sw_record& o = per_request[r];
        o.ttff_us = d.per[r].w0;
        o.stall_us = d.per[r].w1;
        o.cost_mc = d.per[r].w2;
        o.quality = (uint32_t)d.per[r].w3;
        o.stall_count = (uint16_t)(d.per[r].w3 >> 32);
        o.flags = 0;
        o.pad = 0;
        if (ready_abs)
            for (uint32_t s = 0; s < h->shared->S[r]; s++) ready_abs[h->shared->sc_off[r] + s] = d.ready[h->shared->sc_off[r] + s];
    }
    return SW_OK;
}

// ============================================================================ fleet (C4)
// A batch of requests evaluated and selected together: ONE eval launch for every
// request's space (grid.y = request, each CTA stages its own request's tables), ONE
// select scan (grid.y = request, one query per request), one merge kernel, one batched
// winner-detail kernel and -- multi-GPU -- one allgather of the n winners.  The per-request
// handles stay usable (Pareto front, digest, records, detail) through sw_fleet_plan.
struct sw_fleet {
    std::vector<sw_plan*> plans;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ncclComm_t comm = nullptr;
    LoopComm* loop = nullptr;
    int rank = 0, nranks = 1;
    uint32_t np_max = 1;
    int bmode = -1;  // eval path (eval_mode) shared by every request, else 3 (runtime)
    size_t eval_smem = 0;
    int eval_occ = 1, num_sms = 148;
    uint32_t gx = 1;  // scan blocks per request
    EvalJob* d_ejobs = nullptr;
    ScanJob* d_sjobs = nullptr;
    Cand* d_partial = nullptr;
    Cand* d_win = nullptr;
    Cand* d_win_all = nullptr;
    DetailOut* d_det = nullptr;
    uint32_t* d_gfeas = nullptr;
    bool evaluated = false;
    cudaEvent_t ev[4] = {};
    uint64_t k_launches[2] = {0, 0};
    double k_ms[2] = {0.0, 0.0};
    uint64_t k_bytes[2] = {0, 0};
};

template <typename F>
static sw_status launch_np_n(uint32_t np, sw_plan* h, F&& f) {
    switch (np) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 3: f(std::integral_constant<int, 3>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        default: return fail(h, SW_EINVAL, "bad pool count");
    }
    return SW_OK;
}

extern "C" sw_status sw_fleet_destroy(sw_fleet* f) {
    if (!f) return SW_OK;
    if (f->stream) {
        cudaSetDevice(f->device);
        void* bufs[] = {f->d_ejobs, f->d_sjobs, f->d_partial, f->d_win, f->d_win_all, f->d_det, f->d_gfeas};
        for (void* b : bufs)
            if (b) cudaFreeAsync(b, f->stream);
        for (cudaEvent_t e : f->ev)
            if (e) cudaEventDestroy(e);
    }
    for (sw_plan* p : f->plans) sw_plan_destroy(p);
    if (f->stream) {
        cudaStreamSynchronize(f->stream);
        if (f->own_stream) cudaStreamDestroy(f->stream);
    }
    cudaGetLastError();
    delete f;
    return SW_OK;
}

extern "C" sw_status sw_fleet_create(uint32_t n, const sw_profile_tables* tables, const sw_scene_list* scenes,
                                     const sw_price_table* prices, const sw_runtime* rt, sw_fleet** out) {
    const NvtxRange nvtx_("sw_fleet_create");
    if (!tables || !scenes || !prices || !rt || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (n < 1 || n > SW_MAX_FLEET) return fail(nullptr, SW_EINVAL, "fleet size %u not in 1..%d", n, SW_MAX_FLEET);
    sw_fleet* f = new sw_fleet();
    f->device = rt->device;
    f->loop = as_loop(rt->nccl_comm);
    f->comm = f->loop ? nullptr : (ncclComm_t)rt->nccl_comm;
    f->rank = rt->rank;
    f->nranks = rt->nranks;
    auto bail = [&](sw_status s) {
        sw_fleet_destroy(f);
        return s;
    };
    if (cudaSetDevice(f->device) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(nullptr, SW_ECUDA, "cudaSetDevice(%d) failed (no CUDA device?)", f->device));
    }
    if (rt->stream) {
        f->stream = (cudaStream_t)rt->stream;
    } else {
        if (cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(nullptr, SW_ECUDA, "cudaStreamCreate failed"));
        f->own_stream = true;
    }
    sw_runtime prt = *rt;
    prt.stream = f->stream;
    for (uint32_t i = 0; i < n; i++) {
        sw_plan* p = nullptr;
        sw_status st = sw_plan_create(&tables[i], &scenes[i], &prices[i], &prt, &p);
        if (st < 0) {
            const std::string msg = "request " + std::to_string(i) + ": " + g_last_error;
            bail(st);
            return fail(nullptr, st, "%s", msg.c_str());
        }
        f->plans.push_back(p);
        if (p->wide) {
            bail(SW_EINVAL);
            return fail(nullptr, SW_EINVAL, "request %u: fleets need pools of <= %d GPUs", i, kMaxG);
        }
        f->np_max = std::max(f->np_max, p->NP);
        const int bm = eval_mode(p->h.flags);
        f->bmode = f->bmode < 0 ? bm : (f->bmode == bm ? bm : 3);
        f->eval_smem = std::max(f->eval_smem, p->eval_smem);
    }
    sw_plan* h = f->plans[0];
    f->num_sms = h->num_sms;
    {
        cudaError_t e = cudaSuccess;
        int occ = 0;
        launch_np_n(f->np_max, h, [&](auto np) {
            constexpr int NPc = decltype(np)::value;
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, f->device);
            auto setup = [&](auto kern) {
                cudaFuncAttributes fa{};
                cudaError_t r = cudaFuncGetAttributes(&fa, kern);
                if (r == cudaSuccess)
                    r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             optin - (int)fa.sharedSizeBytes);
                int o = 0;
                if (r == cudaSuccess) r = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kEvalThreads, f->eval_smem);
                if (r != cudaSuccess && e == cudaSuccess) e = r;
                return o;
            };
            const int o[4] = {setup(eval_kernel<NPc, 0>), setup(eval_kernel<NPc, 1>), setup(eval_kernel<NPc, 2>),
                              setup(eval_kernel<NPc, 3>)};
            occ = o[f->bmode];
        });
        if (e != cudaSuccess || occ < 1) {
            cudaGetLastError();
            return bail(fail(nullptr, SW_ECUDA, "fleet eval kernel cannot launch (%s)", cudaGetErrorString(e)));
        }
        f->eval_occ = occ;
    }
    f->gx = (uint32_t)std::min<uint64_t>(64, std::max<uint64_t>(1, (8ull * f->num_sms + n - 1) / n));
    auto alloc = [&](void** p, size_t bytes) {
        return cudaMallocAsync(p, bytes, f->stream) == cudaSuccess;
    };
    if (!alloc((void**)&f->d_ejobs, sizeof(EvalJob) * n) || !alloc((void**)&f->d_sjobs, sizeof(ScanJob) * n) ||
        !alloc((void**)&f->d_partial, sizeof(Cand) * SW_MAX_QUERIES * (size_t)n * f->gx) ||
        !alloc((void**)&f->d_win, sizeof(Cand) * SW_MAX_QUERIES * (size_t)n) ||
        !alloc((void**)&f->d_win_all, sizeof(Cand) * SW_MAX_QUERIES * (size_t)n * f->nranks) ||
        !alloc((void**)&f->d_det, sizeof(DetailOut) * (size_t)n) ||
        !alloc((void**)&f->d_gfeas, sizeof(uint32_t) * kGSelWords * (size_t)n)) {
        cudaGetLastError();
        return bail(fail(nullptr, SW_ENOMEM, "fleet scratch allocation failed"));
    }
    for (cudaEvent_t& e : f->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(nullptr, SW_ECUDA, "cudaEventCreate failed"));
    if (cudaStreamSynchronize(f->stream) != cudaSuccess) return bail(fail(nullptr, SW_ECUDA, "fleet create failed"));
    *out = f;
    return SW_OK;
}

extern "C" sw_status sw_fleet_size(const sw_fleet* f, uint32_t* n) {
    if (!f || !n) return fail(nullptr, SW_EINVAL, "null argument");
    *n = (uint32_t)f->plans.size();
    return SW_OK;
}

extern "C" sw_status sw_fleet_plan(sw_fleet* f, uint32_t i, sw_plan** out) {
    if (!f || !out) return fail(nullptr, SW_EINVAL, "null argument");
    if (i >= f->plans.size()) return fail(nullptr, SW_EINVAL, "request %u of %zu", i, f->plans.size());
    *out = f->plans[i];
    return SW_OK;
}

extern "C" sw_status sw_fleet_reset(sw_fleet* f) {
    if (!f) return fail(nullptr, SW_EINVAL, "null fleet");
    for (sw_plan* p : f->plans) {
        sw_status st = sw_plan_reset(p);
        if (st < 0) return st;
    }
    f->evaluated = false;
    return SW_OK;
}

static sw_status fleet_harvest(sw_fleet* f, int kind, uint64_t bytes) {
    sw_plan* h = f->plans[0];
    float ms = 0.f;
    CK(h, cudaEventSynchronize(f->ev[2 * kind + 1]));
    CK(h, cudaEventElapsedTime(&ms, f->ev[2 * kind], f->ev[2 * kind + 1]));
    f->k_launches[kind]++;
    f->k_ms[kind] += ms;
    f->k_bytes[kind] += bytes;
    return SW_OK;
}

extern "C" sw_status sw_fleet_eval(sw_fleet* f) {
    const NvtxRange nvtx_("sw_fleet_eval");
    if (!f) return fail(nullptr, SW_EINVAL, "null fleet");
    sw_plan* h = f->plans[0];
    const uint32_t n = (uint32_t)f->plans.size();
    for (sw_plan* p : f->plans)
        if (!p->segs.empty()) return fail(h, SW_ESTATE, "fleet eval needs handles without records (sw_fleet_reset)");
    CK(h, cudaSetDevice(f->device));
    std::vector<EvalJob> jobs(n);
    uint64_t max_tiles = 0, recs = 0;
    for (uint32_t i = 0; i < n; i++) {  // every request's capacity first: nothing changes on error
        sw_plan* p = f->plans[i];
        uint64_t b, e;
        sw_status st = sw_shard_range(0, p->N, p->row, p->rank, p->nranks, &b, &e);
        if (st < 0) return st;
        const uint64_t m = e - b;
        const uint64_t rb = b / p->row, re = (e + p->row - 1) / p->row;
        const uint64_t t0 = rb / kTileRows, t1 = (re + kTileRows - 1) / kTileRows;
        const uint64_t slots = m ? (t1 - t0) * kTileRows * p->row : 0;
        if (m > p->cand_cap || slots > p->rec_cap)
            return fail(h, SW_ERANGE, "request %u: records exceed its capacity", i);
    }
    for (uint32_t i = 0; i < n; i++) {
        sw_plan* p = f->plans[i];
        uint64_t b, e;
        sw_shard_range(0, p->N, p->row, p->rank, p->nranks, &b, &e);
        const uint64_t m = e - b;
        const uint64_t rb = b / p->row, re = (e + p->row - 1) / p->row;
        const uint64_t t0 = rb / kTileRows, t1 = (re + kTileRows - 1) / kTileRows;
        const uint64_t slots = m ? (t1 - t0) * kTileRows * p->row : 0;
        p->segs.push_back(Segment{0, p->N, b, e, 0, t0, m ? t1 - t0 : 0, false});
        p->rec_used = slots;
        p->cand_used = m;
        jobs[i] = EvalJob{p->d_hdr, p->d_va, p->va_bytes, t0, m ? t1 : t0, p->d_rec};
        max_tiles = std::max<uint64_t>(max_tiles, m ? t1 - t0 : 0);
        recs += m;
    }
    CK(h, cudaMemcpyAsync(f->d_ejobs, jobs.data(), sizeof(EvalJob) * n, cudaMemcpyHostToDevice, f->stream));
    f->evaluated = true;
    if (max_tiles == 0) return SW_OK;
    // one warp per tile: blocks per request = ceil(max tiles / warps per block)
    const uint32_t gxe = (uint32_t)((max_tiles * kTileRows + kEvalThreads - 1) / kEvalThreads);
    CK(h, cudaEventRecord(f->ev[0], f->stream));
    launch_np_n(f->np_max, h, [&](auto np) {
        constexpr int NPc = decltype(np)::value;
        switch (f->bmode) {
            case 0: eval_kernel<NPc, 0><<<dim3(gxe, n), kEvalThreads, f->eval_smem, f->stream>>>(EvalJob{}, f->d_ejobs); break;
            case 1: eval_kernel<NPc, 1><<<dim3(gxe, n), kEvalThreads, f->eval_smem, f->stream>>>(EvalJob{}, f->d_ejobs); break;
            case 2: eval_kernel<NPc, 2><<<dim3(gxe, n), kEvalThreads, f->eval_smem, f->stream>>>(EvalJob{}, f->d_ejobs); break;
            default: eval_kernel<NPc, 3><<<dim3(gxe, n), kEvalThreads, f->eval_smem, f->stream>>>(EvalJob{}, f->d_ejobs); break;
        }
    });
    CKL(h);
    CK(h, cudaEventRecord(f->ev[1], f->stream));
    return fleet_harvest(f, SW_KERNEL_EVAL, recs * sizeof(Rec4));
}

extern "C" sw_status sw_fleet_select(sw_fleet* f, const sw_query* queries, sw_selection* out) {
    const NvtxRange nvtx_("sw_fleet_select");
    if (!f || !queries || !out) return fail(nullptr, SW_EINVAL, "null argument");
    sw_plan* h = f->plans[0];
    if (!f->evaluated) return fail(h, SW_ESTATE, "sw_fleet_eval first");
    const uint32_t n = (uint32_t)f->plans.size();
    CK(h, cudaSetDevice(f->device));
    std::vector<ScanJob> jobs(n);
    uint64_t slots = 0;
    for (uint32_t i = 0; i < n; i++) {
        sw_plan* p = f->plans[i];
        if (p->segs.size() != 1) return fail(h, SW_ESTATE, "request %u: records changed since sw_fleet_eval", i);
        const Segment& g = p->segs[0];
        jobs[i].v = view_of(p, g, 0, g.ntiles);
        memset(&jobs[i].P, 0, sizeof(SelParams));
        jobs[i].P.nq = 1;
        jobs[i].P.objective = (p->h.flags & 4u) ? 1u : 0u;
        jobs[i].P.q[0] = QueryDev{queries[i].slo_startup_us, queries[i].slo_stall_us, queries[i].budget_mc};
        slots += g.ntiles * kTileRows * p->row;
    }
    CK(h, cudaMemcpyAsync(f->d_sjobs, jobs.data(), sizeof(ScanJob) * n, cudaMemcpyHostToDevice, f->stream));
    CK(h, cudaMemsetAsync(f->d_gfeas, 0, sizeof(uint32_t) * kGSelWords * n, f->stream));
    ParetoArgs pa{};
    pa.gfeas = f->d_gfeas;
    CK(h, cudaEventRecord(f->ev[2], f->stream));
    scan_kernel<1, false, -1><<<dim3(f->gx, n), kScanBlock, kRingBytes, f->stream>>>(SegView{}, SelParams{}, f->d_partial,
                                                                                pa, f->d_sjobs);
    CKL(h);
    CK(h, cudaEventRecord(f->ev[3], f->stream));
    select_merge_kernel<<<n, kScanThreads, 0, f->stream>>>(f->d_partial, f->gx, SW_MAX_QUERIES,
                                                           (uint64_t)f->gx * SW_MAX_QUERIES, f->d_sjobs, f->d_win);
    CKL(h);
    if (f->nranks > 1) {  // a10: one allgather of the n winners, replicated merge
        CKC(h, coll_allgather(coll_of(h), f->d_win, f->d_win_all, sizeof(Cand) * SW_MAX_QUERIES * n, &why_));
        select_merge_kernel<<<n, kScanThreads, 0, f->stream>>>(f->d_win_all, (uint32_t)f->nranks,
                                                               (uint64_t)n * SW_MAX_QUERIES, SW_MAX_QUERIES, f->d_sjobs,
                                                               f->d_win);
        CKL(h);
    }
    launch_np_n(f->np_max, h, [&](auto np) {
        constexpr int NPc = decltype(np)::value;
        detail_fleet_kernel<NPc><<<n, 32, 0, f->stream>>>(f->d_ejobs, f->d_win, 1, f->d_det);
    });
    CKL(h);
    std::vector<Cand> win((size_t)n * SW_MAX_QUERIES);
    std::vector<DetailOut> det(n);
    CK(h, cudaMemcpyAsync(win.data(), f->d_win, sizeof(Cand) * win.size(), cudaMemcpyDeviceToHost, f->stream));
    CK(h, cudaMemcpyAsync(det.data(), f->d_det, sizeof(DetailOut) * n, cudaMemcpyDeviceToHost, f->stream));
    sw_status st = fleet_harvest(f, SW_KERNEL_SCAN, slots * sizeof(Rec4));  // synchronises the scan
    if (st < 0) return st;
    SYNC(h);
    sw_status worst = SW_OK;
    for (uint32_t i = 0; i < n; i++) {
        const Cand& c = win[(size_t)i * SW_MAX_QUERIES];
        sw_selection& o = out[i];
        memset(&o, 0, sizeof o);
        if (c.idx == kInf64) {
            o.status = SW_EMPTY;
        } else {
            const sw_plan* p = f->plans[i];
            const DetailOut& d = det[i];
            o.status = c.pad ? SW_CLOSEST : SW_OK;
            o.index = c.idx;
            o.rec.ttff_us = d.rec.w0;
            o.rec.stall_us = d.rec.w1;
            o.rec.cost_mc = d.rec.w2;
            o.rec.quality = (uint32_t)d.rec.w3;
            o.rec.stall_count = (uint16_t)(d.rec.w3 >> 32);
            o.rec.flags = (uint8_t)(d.rec.w3 >> 48);
            o.ttff_eff_us = d.ttff_eff;
            o.makespan_us = d.makespan;
            for (uint32_t q = 0; q < SW_MAX_POOLS; q++) o.pool_end_us[q] = q < p->NP ? d.pool_end[q] : 0;
            for (uint32_t b = 0; b < p->B_user; b++) o.digit[b] = (uint8_t)d.digit[b + p->pad_digits];
        }
        worst = std::max<sw_status>(worst, o.status);
    }
    return worst;
}

extern "C" sw_status sw_fleet_kernel_time(sw_fleet* f, uint32_t kind, uint64_t* n_launches, double* total_ms,
                                          uint64_t* bytes) {
    if (!f || !n_launches || !total_ms || !bytes) return fail(nullptr, SW_EINVAL, "null argument");
    if (kind > SW_KERNEL_SCAN) return fail(nullptr, SW_EINVAL, "bad kernel kind %u", kind);
    *n_launches = f->k_launches[kind];
    *total_ms = f->k_ms[kind];
    *bytes = f->k_bytes[kind];
    return SW_OK;
}

extern "C" uint64_t sw_fleet_launch_count(const sw_fleet* f) {
    uint64_t s = 0;
    if (f)
        for (const sw_plan* p : f->plans) s += p->launches;
    return s;
}

// ============================================================================ NCCL
extern "C" sw_status sw_comm_unique_id(void* id128) {
    if (!id128) return fail(nullptr, SW_EINVAL, "null argument");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, SW_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "nccl unique id size");
    memcpy(id128, &id, 128);
    return SW_OK;
}

extern "C" sw_status sw_comm_init(const void* id128, int32_t rank, int32_t nranks, int32_t device, void** comm_out) {
    if (!id128 || !comm_out) return fail(nullptr, SW_EINVAL, "null argument");
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        return fail(nullptr, SW_ECUDA, "cudaSetDevice(%d) failed", device);
    }
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclComm_t c = nullptr;
    ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) return fail(nullptr, SW_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    *comm_out = (void*)c;
    return SW_OK;
}

extern "C" sw_status sw_comm_loopback_create(int32_t nranks, void** comms_out) {
    if (!comms_out || nranks < 1 || nranks > 1024) return fail(nullptr, SW_EINVAL, "bad loopback arguments");
    LoopGroup* g = new LoopGroup();
    g->n = g->alive = nranks;
    g->send.assign(nranks, nullptr);
    g->ready.assign(nranks, nullptr);
    g->done.assign(nranks, nullptr);
    for (int r = 0; r < nranks; r++) {
        if (cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            for (cudaEvent_t e : g->ready)
                if (e) cudaEventDestroy(e);
            for (cudaEvent_t e : g->done)
                if (e) cudaEventDestroy(e);
            delete g;
            return fail(nullptr, SW_ECUDA, "loopback: cudaEventCreate failed (no CUDA device?)");
        }
    }
    std::lock_guard<std::mutex> lk(loop_registry_mu());
    for (int r = 0; r < nranks; r++) {
        LoopComm* c = new LoopComm{kLoopMagic, g, r};
        loop_registry().insert(c);
        comms_out[r] = c;
    }
    return SW_OK;
}

extern "C" sw_status sw_trim_device_memory(int32_t device) {
    cudaMemPool_t pool;
    if (cudaSetDevice(device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
        cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess || cudaMemPoolTrimTo(pool, 0) != cudaSuccess) {
        cudaGetLastError();
        return fail(nullptr, SW_ECUDA, "trimming the device memory pool of device %d failed", device);
    }
    return SW_OK;
}

extern "C" sw_status sw_comm_destroy(void* comm) {
    if (!comm) return SW_OK;
    if (LoopComm* lc = as_loop(comm)) {  // a loopback rank: the group goes with its last rank
        LoopGroup* g = lc->g;
        bool last = false;
        {
            std::lock_guard<std::mutex> lk(loop_registry_mu());
            loop_registry().erase(comm);
            last = --g->alive == 0;
        }
        delete lc;
        if (last) {
            for (cudaEvent_t e : g->ready) cudaEventDestroy(e);
            for (cudaEvent_t e : g->done) cudaEventDestroy(e);
            delete g;
        }
        return SW_OK;
    }
    {
        std::lock_guard<std::mutex> lk(loop_registry_mu());
        if (aborted_registry().erase(comm)) return SW_OK;  // already aborted by the library
    }
    ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
    if (r != ncclSuccess) return fail(nullptr, SW_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
    return SW_OK;
}

// ============================================================================ diagnostics
extern "C" const char* sw_status_str(sw_status s) {
    switch (s) {
        case SW_OK: return "SW_OK";
        case SW_CLOSEST: return "SW_CLOSEST";
        case SW_TRUNCATED: return "SW_TRUNCATED";
        case SW_EMPTY: return "SW_EMPTY";
        case SW_EINVAL: return "SW_EINVAL";
        case SW_ERANGE: return "SW_ERANGE";
        case SW_ENOMEM: return "SW_ENOMEM";
        case SW_ECUDA: return "SW_ECUDA";
        case SW_ENCCL: return "SW_ENCCL";
        case SW_ESTATE: return "SW_ESTATE";
        default: return "SW_UNKNOWN";
    }
}

extern "C" const char* sw_last_error(const sw_plan* h) {
    if (h && !h->err.empty()) return h->err.c_str();
    return g_last_error.c_str();
}

extern "C" uint64_t sw_plan_launch_count(const sw_plan* h) { return h ? h->launches : 0; }

extern "C" int32_t sw_abi_version(void) { return 6; }  // 2: pool_ready_us; 3: evict_risk_permille; 4: loopback, decode, segments; 5: shared-pool fleets; 6: VAE stages, energy metric
