// sw_wide.cuh -- the generic path for pools of 9..32 GPUs (SURVEY §8(a) layout note, §8(b)
// "G_p <= 8 fast path, <= 32 generic").
//
// The fast path holds each pool's <= 8 free times in a lane's registers (lane per prefix).
// A wider pool does not fit, so here a WARP evaluates one candidate at a time with the
// pool's GPU slots on its lanes: lane j holds F_p[j] of every pool (+inf for j >= G_p).  A
// scene step on (pool p, k GPUs) is the same gang identity as the fast path,
//   F'[j] = max(F[j], min(e, F[j + k])),  e = max(a_s, F[k-1]) + t   (R5; F[>= 32] = inf),
// with F[k-1] one shuffle and F[j + k] a shuffle-down: ~15 warp instructions per scene-step
// for one candidate.  Everything else (metrics, cost, the record) is warp-uniform.  The warp
// walks a tile of 32 rows; per row it simulates the HI prefix once and iterates the MID and
// LSD digits with state copies (prefix sharing as on the fast path); lane 0 stores each
// record into the same tiled layout, so the scans, select, Pareto and digest are unchanged.
#pragma once
#include "sw_kernels.cuh"

namespace sw {

constexpr int kWideMaxG = 32;

template <int NP>
struct WState {
    uint64_t F[NP];  // this lane's slot of each pool's ascending free-time multiset
    uint64_t end[NP], busy[NP];
    uint64_t R0;
    int64_t M;
    uint32_t cnt, Q, used;
};

template <int NP>
__device__ __forceinline__ void wide_init(WState<NP>& s, const DevHeader& h, uint32_t lane) {
#pragma unroll
    for (int q = 0; q < NP; q++) {
        s.F[q] = lane < h.G[q] ? h.ready[q] : kInf64;
        s.end[q] = 0;
        s.busy[q] = 0;
    }
    s.R0 = h.R0_static;
    s.M = (int64_t)h.R0_static;
    s.cnt = s.Q = s.used = 0;
}

// Gang update of one pool's multiset held across the warp (k warp-uniform, 1..32).
__device__ __forceinline__ uint64_t wide_gang(uint64_t& Fq, uint32_t k, uint64_t a, uint64_t t, uint32_t lane) {
    const uint64_t fk = __shfl_sync(0xffffffffu, Fq, k - 1);
    const uint64_t e = umax64(a, fk) + t;
    uint64_t up = __shfl_down_sync(0xffffffffu, Fq, k);
    if (lane + k >= 32) up = kInf64;
    Fq = umax64(Fq, umin64(e, up));
    return e;
}

// One scene on choice ch (pool, k, optional VAE stage R37); returns R_s.  ch is warp-uniform.
template <int NP>
__device__ __forceinline__ uint64_t wide_step(WState<NP>& s, uint32_t ch, uint64_t a, const VaEntry& v,
                                              uint32_t lane) {
    const uint32_t p = ch_pool(ch), k = ch_k(ch), vae = ch_vae(ch);
    if (k == 0) return a;  // STATIC rung (R33)
    uint64_t e = 0;
#pragma unroll
    for (int q = 0; q < NP; q++)
        if ((uint32_t)q == p) {
            e = wide_gang(s.F[q], k, a, v.t_us, lane);
            s.end[q] = umax64(s.end[q], e);
            s.busy[q] += (uint64_t)k * v.t_us;
        }
    s.used |= 1u << p;
    if (vae) {  // the VAE stage on pool vae - 1, one GPU, after the DiT
        uint64_t ev = e;
#pragma unroll
        for (int q = 0; q < NP; q++)
            if ((uint32_t)q == vae - 1) {
                ev = wide_gang(s.F[q], 1, e, v.t_vae, lane);
                s.end[q] = umax64(s.end[q], ev);
                s.busy[q] += v.t_vae;
            }
        s.used |= 1u << (vae - 1);
        e = ev;
    }
    return e;
}

template <int NP>
__device__ __forceinline__ void wide_block(WState<NP>& s, const DevHeader& h, uint32_t ch, uint32_t f0, uint32_t f1,
                                           const VaEntry* vb, uint32_t r, uint32_t lane, uint64_t* ready = nullptr) {
    for (uint32_t sc = f0; sc < f1; sc++) {
        const VaEntry v = vb[(sc - f0) * r];
        const uint64_t e = wide_step<NP>(s, ch, h.a[sc], v, lane);
        scene_metrics(s, sc, e, h.P[sc], v.q);
        if (ready) ready[sc] = e;
    }
}

template <int NP>
__device__ __forceinline__ uint64_t wide_cost(const WState<NP>& s, const DevHeader& h) {
    uint64_t c = h.fixed_cost;
    const int mode = cost_mode(h.flags);
#pragma unroll
    for (int p = 0; p < NP; p++) {
        switch (mode) {
            case 0: c += pool_term<0>(h, p, s.end[p], s.busy[p]); break;
            case 1: c += pool_term<1>(h, p, s.end[p], s.busy[p]); break;
            case 2: c += pool_term<2>(h, p, s.end[p], s.busy[p]); break;
            default: c += pool_term<3>(h, p, s.end[p], s.busy[p]); break;
        }
    }
    return c;
}

template <int NP>
__device__ __forceinline__ Rec4 wide_record(const WState<NP>& s, const DevHeader& h) {
    Rec4 r;
    r.w0 = s.R0;
    r.w1 = (uint64_t)s.M - s.R0;
    r.w2 = wide_cost(s, h);
    r.w3 = (uint64_t)s.Q | ((uint64_t)s.cnt << 32) | ((uint64_t)s.used << 48);
    return r;
}

// a1-a7 for handles with a pool of more than 8 GPUs: warp <-> tile of 32 rows, one row at a
// time (HI prefix once per row), MID x LSD candidates in odometer order.
template <int NP>
__global__ void __launch_bounds__(kEvalThreads) eval_wide_kernel(EvalJob job) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar;
    DevHeader& h = *reinterpret_cast<DevHeader*>(smem);
    VaEntry* va = reinterpret_cast<VaEntry*>(smem + sizeof(DevHeader));
    stage_tables(job.hdr, job.va, &h, va, (uint32_t)job.va_bytes, &bar);
    const uint32_t bm = h.B - 2, bl = h.B - 1;
    const uint32_t rm = h.radix[bm], rl = h.radix[bl];
    const uint64_t row = h.row, n_rows = h.n_rows;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = job.tile_begin + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); t < job.tile_end;
         t += nwarps) {
        Rec4* tile_out = job.out + (t - job.tile_begin) * kTileRows * row;
        for (uint32_t rr = 0; rr < kTileRows; rr++) {
            const uint64_t H = t * kTileRows + rr;
            if (H >= n_rows) break;  // warp-uniform
            WState<NP> st;
            wide_init<NP>(st, h, lane);
            uint64_t rem = H;
            for (uint32_t b = 0; b < bm; b++) {  // HI prefix (MSD = earliest block, R19)
                const uint64_t pl = h.place[b];
                const uint32_t c = (uint32_t)(rem / pl);
                rem -= (uint64_t)c * pl;
                wide_block<NP>(st, h, h.choice[h.coff[b] + c], h.first[b], h.first[b + 1], va + h.voff[b] + c,
                               h.radix[b], lane);
            }
            for (uint32_t dm = 0; dm < rm; dm++) {
                WState<NP> s2 = st;
                wide_block<NP>(s2, h, h.choice[h.coff[bm] + dm], h.first[bm], h.first[bm + 1], va + h.voff[bm] + dm,
                               rm, lane);
                for (uint32_t dl = 0; dl < rl; dl++) {
                    WState<NP> s3 = s2;
                    wide_block<NP>(s3, h, h.choice[h.coff[bl] + dl], h.first[bl], h.first[bl + 1],
                                   va + h.voff[bl] + dl, rl, lane);
                    const Rec4 r = wide_record(s3, h);
                    if (lane == 0) st_global_256(tile_out + ((size_t)dm * rl + dl) * kTileRows + rr, r);
                }
            }
        }
    }
}

// Full detail of winners cand[q].idx (one warp each) -> DetailOut.
template <int NP>
__global__ void wide_detail_kernel(const DevHeader* __restrict__ g_hdr, const VaEntry* __restrict__ g_va,
                                   const Cand* __restrict__ cand, uint32_t nq, DetailOut* __restrict__ out) {
    const uint32_t q = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    if (q >= nq || threadIdx.x >= 32) return;
    const uint64_t index = cand[q].idx;
    if (index == kInf64) return;
    const DevHeader& h = *g_hdr;
    DetailOut* o = out + q;
    WState<NP> st;
    wide_init<NP>(st, h, lane);
    uint32_t dig[kMaxDigits];
    uint64_t rem = index;
    for (int b = (int)h.B - 1; b >= 0; b--) {
        dig[b] = (uint32_t)(rem % h.radix[b]);
        rem /= h.radix[b];
    }
    uint64_t ready[SW_MAX_SCENES];
    if (h.flags & 1u) ready[0] = h.R0_static;
    for (uint32_t b = 0; b < h.B; b++)
        wide_block<NP>(st, h, h.choice[h.coff[b] + dig[b]], h.first[b], h.first[b + 1], g_va + h.voff[b] + dig[b],
                       h.radix[b], lane, ready);
    if (lane != 0) return;
    uint64_t mk = st.R0;
    for (int p = 0; p < NP; p++) {
        o->pool_end[p] = st.end[p];
        mk = umax64(mk, st.end[p]);
    }
    for (uint32_t s = 0; s < h.S; s++) {
        o->ready[s] = ready[s];
        mk = umax64(mk, ready[s]);
    }
    for (uint32_t b = 0; b < h.B; b++) o->digit[b] = dig[b];
    o->rec = wide_record(st, h);
    o->ttff_eff = (uint64_t)st.M;
    o->makespan = mk;
}

}  // namespace sw
