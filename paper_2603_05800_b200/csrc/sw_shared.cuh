// sw_shared.cuh -- shared-pool fleet evaluation (reading R36).
//
// Several requests contend for the SAME GPU pools: "model instances maintain local queues
// that prioritize tasks by deadline ... the image generation model may process an early
// scene from a new request before a later scene from an earlier request if it has a
// tighter deadline".  A candidate is a JOINT plan of the free requests (the
// others are fixed background load); one thread evaluates one candidate:
//   1. decode the joint index (MSD = the first free request's first digit);
//   2. every pool is an online, non-preemptive EDF queue of gang tasks: at decision time
//      t the head is the released (release <= t), unstarted task with the smallest
//      (deadline, request, scene); it starts at max(t, F[k-1]) on the k earliest-free GPUs
//      (the single-request gang rule, no backfill) unless a more urgent task is released at
//      or before that start, which then takes the decision; decisions are in time order.
//      Within a request a pool's tasks are in scene order with non-decreasing release and
//      increasing deadline, so only each request's next task on the pool (its "head")
//      competes: O(R) per decision;
//   3. per request, playback metrics in scene order relative to its arrival; the fleet
//      record (worst startup lateness, worst stall lateness, fleet cost, total quality,
//      total rebuffering events, pools used) goes to the tiled record buffer (row = 1), so
//      select / Pareto / digest / sweep run unchanged on it.
// Product code of libsw_plan.so; shares nothing with oracle/.
#pragma once
#include "sw_kernels.cuh"

namespace sw {

constexpr int kShMaxReq = 16;
constexpr int kShMaxScenes = 128;  // scenes over all requests (per-thread ready times)
constexpr int kShThreads = 128;

struct SharedReqDev {
    const DevHeader* hdr;  // the request's packed tables (a_s, P_s, choices, VA entries)
    const VaEntry* va;
    uint64_t T0, slo_t, slo_s;
    uint32_t S, s0, B, pad_digits;  // B = the request's digits (header digits minus padding)
    uint32_t free_, dig0, sc_off, pad;  // dig0: first joint digit (free requests)
    uint32_t fixed_dig[SW_MAX_DIGITS];  // a background request's plan
};

struct SharedDev {
    uint32_t R, NP, billing, nd;  // nd: joint digits
    uint32_t G[kMaxP];
    uint64_t price[kMaxP];
    uint64_t ready[kMaxP];
    uint32_t jradix[SW_MAX_DIGITS];  // radix of joint digit j (MSD first)
    SharedReqDev req[kShMaxReq];
};

struct SharedDetailOut {
    Rec4 fleet;
    Rec4 per[kShMaxReq];  // per request: ttff, stall, fixed cost, Q | cnt << 32
    uint64_t ready[kShMaxScenes];  // absolute ready times, request-major (sc_off + s)
    uint64_t pool_end[kMaxP];
    uint64_t makespan;  // latest scene ready time over all requests (absolute)
    uint32_t digit[SW_MAX_DIGITS];
};

__device__ __forceinline__ uint64_t sat_add64(uint64_t a, uint64_t b) { return a > ~b ? kInf64 : a + b; }

// Digit of request r's block b for this candidate.
__device__ __forceinline__ uint32_t sh_digit(const SharedReqDev& q, const uint32_t* jd, uint32_t b) {
    return q.free_ ? jd[q.dig0 + b] : q.fixed_dig[b];
}

// Choice (level | k << 8 | pool << 16) and V+A entry of request r's scene s (s >= s0).
__device__ __forceinline__ void sh_scene(const SharedReqDev& q, const uint32_t* jd, uint32_t s, uint32_t& ch,
                                         VaEntry& v) {
    const DevHeader& h = *q.hdr;
    uint32_t b = q.pad_digits;
    while (s >= h.first[b + 1]) b++;
    const uint32_t c = sh_digit(q, jd, b - q.pad_digits);
    ch = h.choice[h.coff[b] + c];
    v = q.va[h.voff[b] + (s - h.first[b]) * h.radix[b] + c];
}

// next scene >= s of request q on pool p with a video stage (S if none)
__device__ __forceinline__ uint32_t sh_next(const SharedReqDev& q, const uint32_t* jd, uint32_t s, uint32_t p) {
    for (; s < q.S; s++) {
        uint32_t ch;
        VaEntry v;
        sh_scene(q, jd, s, ch, v);
        if (ch_k(ch) != 0 && ch_pool(ch) == p) return s;
    }
    return q.S;
}

__device__ __forceinline__ uint64_t sh_deadline(const SharedReqDev& q, uint32_t s) {
    return q.slo_t == kInf64 ? kInf64 : sat_add64(sat_add64(q.T0, q.slo_t), q.hdr->P[s]);
}

// One joint candidate: fleet record (+ optional detail).
__device__ Rec4 shared_eval_one(const SharedDev& D, uint64_t index, SharedDetailOut* det) {
    uint32_t jd[SW_MAX_DIGITS];
    {
        uint64_t rem = index;
        for (int j = (int)D.nd - 1; j >= 0; j--) {
            const uint32_t r = D.jradix[j];
            jd[j] = (uint32_t)(rem % r);
            rem /= r;
        }
    }
    uint64_t ready[kShMaxScenes];
    uint32_t used = 0;
    uint64_t cost = 0;
    // STATIC scenes and the static intro: ready with their text and audio (R33, R15)
    for (uint32_t r = 0; r < D.R; r++) {
        const SharedReqDev& q = D.req[r];
        if (q.s0) ready[q.sc_off] = q.T0 + q.hdr->R0_static;
        for (uint32_t s = q.s0; s < q.S; s++) {
            uint32_t ch;
            VaEntry v;
            sh_scene(q, jd, s, ch, v);
            if (ch_k(ch) == 0) ready[q.sc_off + s] = q.T0 + q.hdr->a[s];
        }
    }
    // every pool: online non-preemptive EDF of gang tasks over the requests' heads
    for (uint32_t p = 0; p < D.NP; p++) {
        uint64_t F[kMaxG];
#pragma unroll
        for (int g = 0; g < kMaxG; g++) F[g] = (uint32_t)g < D.G[p] ? D.ready[p] : kInf64;
        uint64_t busy = 0, tnow = 0;
        bool any = false;
        uint32_t cur[kShMaxReq];
        for (uint32_t r = 0; r < D.R; r++) cur[r] = sh_next(D.req[r], jd, D.req[r].s0, p);
        for (;;) {
            int h = -1;
            uint64_t hdl = 0, nrel = kInf64;
            bool left = false;
            for (uint32_t r = 0; r < D.R; r++) {
                const SharedReqDev& q = D.req[r];
                if (cur[r] >= q.S) continue;
                left = true;
                const uint64_t rel = q.T0 + q.hdr->a[cur[r]];
                if (rel <= tnow) {
                    const uint64_t dl = sh_deadline(q, cur[r]);
                    if (h < 0 || dl < hdl) {  // requests in index order: ties keep the lower r
                        h = (int)r;
                        hdl = dl;
                    }
                } else {
                    nrel = umin64(nrel, rel);
                }
            }
            if (!left) break;
            if (h < 0) {  // nothing released: wait for the next release
                tnow = nrel;
                continue;
            }
            const SharedReqDev& qh = D.req[h];
            uint32_t ch;
            VaEntry v;
            sh_scene(qh, jd, cur[h], ch, v);
            const uint32_t k = ch_k(ch);
            const uint64_t st = umax64(tnow, sel_dyn(F, k - 1));
            // a more urgent task released by the head's start takes the decision
            uint64_t u = kInf64;
            for (uint32_t r = 0; r < D.R; r++) {
                const SharedReqDev& q = D.req[r];
                if (cur[r] >= q.S || (int)r == h) continue;
                const uint64_t rel = q.T0 + q.hdr->a[cur[r]];
                if (rel <= tnow) continue;
                const uint64_t dl = sh_deadline(q, cur[r]);
                if (dl < hdl || (dl == hdl && (int)r < h)) u = umin64(u, rel);
            }
            if (u <= st) {
                tnow = u;
                continue;
            }
            const uint64_t e = st + v.t_us;
            gang_update_dyn(F, e, k);
            busy += (uint64_t)k * v.t_us;
            ready[qh.sc_off + cur[h]] = e;
            tnow = st;
            any = true;
            cur[h] = sh_next(qh, jd, cur[h] + 1, p);
        }
        uint64_t end = 0;
        if (any) {
            used |= 1u << p;
#pragma unroll
            for (int g = 0; g < kMaxG; g++)
                if ((uint32_t)g < D.G[p]) end = umax64(end, F[g]);
            const uint64_t X = D.billing ? busy : (uint64_t)D.G[p] * end;
            cost += pool_cost(X, D.price[p]);
        }
        if (det) det->pool_end[p] = end;
    }
    // per request: playback metrics in scene order, relative to its arrival (R7-R9)
    uint64_t late_t = 0, late_s = 0, Qs = 0, cnts = 0;
    for (uint32_t r = 0; r < D.R; r++) {
        const SharedReqDev& q = D.req[r];
        uint64_t R0 = 0, Q = 0;
        int64_t M = 0;
        uint32_t cnt = 0;
        for (uint32_t s = 0; s < q.S; s++) {
            const uint64_t e = ready[q.sc_off + s] - q.T0;
            if (s == 0) {
                R0 = e;
                M = (int64_t)e;
            } else if ((int64_t)e - (int64_t)q.hdr->P[s] > M) {
                M = (int64_t)e - (int64_t)q.hdr->P[s];
                cnt++;
            }
            if (s >= q.s0) {
                uint32_t ch;
                VaEntry v;
                sh_scene(q, jd, s, ch, v);
                Q += v.q;
            }
        }
        const uint64_t stall = (uint64_t)M - R0;
        cost += q.hdr->fixed_cost;
        late_t = umax64(late_t, sat_sub(R0, q.slo_t));
        late_s = umax64(late_s, sat_sub(stall, q.slo_s));
        Qs += Q;
        cnts += cnt;
        if (det) {
            det->per[r].w0 = R0;
            det->per[r].w1 = stall;
            det->per[r].w2 = q.hdr->fixed_cost;
            det->per[r].w3 = Q | ((uint64_t)cnt << 32);
        }
    }
    Rec4 out;
    if (det) {
        uint64_t mk = 0;
        for (uint32_t r = 0; r < D.R; r++)
            for (uint32_t s = 0; s < D.req[r].S; s++) mk = umax64(mk, ready[D.req[r].sc_off + s]);
        det->makespan = mk;
    }
    out.w0 = late_t;
    out.w1 = late_s;
    out.w2 = cost;
    out.w3 = Qs | (cnts << 32) | ((uint64_t)used << 48);
    if (det) {
        det->fleet = out;
        for (uint32_t r = 0; r < D.R; r++)
            for (uint32_t s = 0; s < D.req[r].S; s++) det->ready[D.req[r].sc_off + s] = ready[D.req[r].sc_off + s];
        for (uint32_t j = 0; j < D.nd; j++) det->digit[j] = jd[j];
    }
    return out;
}

// Records of joint candidates of tiles [tile_begin, tile_end) (row = 1: tile t holds
// candidates t*32 .. t*32+31 in order); candidates past the space write their padding slot.
__global__ void __launch_bounds__(kShThreads) shared_eval_kernel(const SharedDev* __restrict__ D, uint64_t tile_begin,
                                                                 uint64_t tile_end, uint64_t n, Rec4* __restrict__ out) {
    const uint64_t first = tile_begin * kTileRows, last = tile_end * kTileRows;
    for (uint64_t i = first + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < last;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const Rec4 r = shared_eval_one(*D, i < n ? i : n - 1, nullptr);
        st_global_256(out + (i - first), r);
    }
}

// Full detail of the winners cand[q].idx (q < nq) -> DetailOut (fleet record, pool ends,
// joint digits; ready = the first 64 scenes' absolute ready times).
__global__ void shared_detail_kernel(const SharedDev* __restrict__ D, const Cand* __restrict__ cand, uint32_t nq,
                                     DetailOut* __restrict__ out, SharedDetailOut* __restrict__ full) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t idx = cand[q].idx;
    if (idx == kInf64) return;
    SharedDetailOut* d = full + q;
    shared_eval_one(*D, idx, d);
    DetailOut& o = out[q];
    o.rec = d->fleet;
    o.ttff_eff = d->fleet.w0 + d->fleet.w1;
    o.makespan = d->makespan;
    for (uint32_t p = 0; p < kMaxP; p++) o.pool_end[p] = p < D->NP ? d->pool_end[p] : 0;
    for (uint32_t i = 0; i < SW_MAX_SCENES; i++) o.ready[i] = d->ready[i];
    for (uint32_t j = 0; j < kMaxDigits; j++) o.digit[j] = j < D->nd ? d->digit[j] : 0;
}

}  // namespace sw
