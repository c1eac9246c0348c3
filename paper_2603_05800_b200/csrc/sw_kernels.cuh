// sw_kernels.cuh -- sm_100a kernels of libsw_plan.so.
//
// pack_kernel     : a2 fixed-stage ready times + deadlines + 16 B VA/quality entries
// eval_kernel<NP> : a1 decode, a3 TMA-staged tables, a4 max-plus scan, a5-a7 metrics,
//                   cost and the 32 B record store
// detail_kernel   : one candidate's full metrics (winner report, what-if inspection)
// select_*        : a9 constrained argmin (multi-query, warp/block/grid reductions)
// pareto_*        : a8 exact 3-D Pareto front (DLT filter + exact dominance merge)
// digest_kernel   : order-independent record digest (full-space parity tool)
#pragma once
#include <cooperative_groups.h>
#include <type_traits>

#include "sw_device.cuh"

namespace sw {

constexpr int kEvalThreads = 128;
constexpr uint32_t kTileRows = 32;  // rows per record tile (= lanes per warp)

// Tiled record layout: a segment's records live in tiles of 32 consecutive rows; within
// a tile the record of (row tile*32 + lane, in-row offset j) is at j * 32 + lane.
// Index of the record at position pos of a tile-aligned segment starting at tile t0:
__device__ __forceinline__ uint64_t tiled_index(uint64_t t0, uint64_t row, uint64_t tile, uint32_t pos_in_tile) {
    return ((t0 + tile) * kTileRows + (pos_in_tile & 31u)) * row + (pos_in_tile >> 5);
}

// A tile range of one segment's records, plus the global index range it owns
// (records outside [ib, ie) -- tile padding -- are skipped by every scan).
struct SegView {
    const Rec4* recs;  // first record of tile t0
    uint64_t t0;       // absolute index of the first tile
    uint64_t ntiles;
    uint64_t row;
    uint64_t ib, ie;
    // Strided fold passes (scan kernels only): the view is cut into units of `upt`
    // tiles (a whole number of scan stages).  With K levels, pass 1 scans the units
    // u % 8^K == 0, pass l+1 (l = 1..K) the units that are multiples of 8^(K-l) but not of
    // 8^(K-l+1) -- each pass a uniform sample of the whole segment, 8x the previous one,
    // so the Pareto filter sees every region early and each pass's survivors stay
    // bounded.  pass 0: the whole view in order.
    uint32_t pass, upt, levels;
    // a huge pass is folded in sub-passes: this one covers the pass's units [j0, j1)
    // (pass-local unit order; j1 = ~0: to the end)
    uint32_t j0, j1, pad_;
};
constexpr int kScanThreads = 256;
constexpr int kDltT = 255;  // dominance lookup table: ttff_eff bins (front quantiles; <= 255: u8 map)
constexpr int kDltQ = 128;  //                         quality bins (tops at front quality values)
constexpr int kDltCols = kDltQ + 1;  // + the "above every front q" column
constexpr int kDltQMap = 1024;  // q map: linear cells over the quality tops' range
constexpr int kDltMap = 2048;  // t direct map: 128 cells per octave over 16 octaves
constexpr int kDltTShift = 16; // t cell key = float bits >> 16 (7 mantissa bits)

// ============================================================================ a2 + packing
struct RawDesc {
    const uint64_t* dur;
    const uint64_t* llm;
    const uint64_t* tts;
    const uint64_t* va;      // raw block-major stage times (host layout)
    const uint32_t* score;   // level scores
    const uint32_t* va_scene;  // scene of each raw va entry (index bookkeeping from host)
    const uint32_t* va_choice; // global choice slot of each raw va entry
    const uint64_t* vae;       // raw VAE stage times (R37), or null
    uint64_t overhead;
    uint32_t n_va;
};

// One block.  Thread 0 runs the sequential fixed-stage recurrence (plan-independent,
// S <= 64 steps): the LLM streams scenes in order and each finished scene triggers its
// downstream stages; one FIFO TTS server (Table 4; R2/R3):
//   L += llm_s ; A = max(L, A) + tts_s ; a_s = A.
// Deadlines P_s = sum_{j<s} d_j.  All threads fill the VA entries with the
// quality contribution q = dur_ms(s) * score(level) (R12).
__global__ void pack_kernel(RawDesc raw, DevHeader* __restrict__ hdr, VaEntry* __restrict__ va) {
    if (threadIdx.x == 0) {
        uint64_t L = raw.overhead, A = 0, acc = 0;
        const bool stat = hdr->flags & 1u;
        for (uint32_t s = 0; s < hdr->S; s++) {
            if (s == 0 && stat) {
                hdr->a[s] = 0;
            } else {
                L = L + raw.llm[s];
                A = (L > A ? L : A) + raw.tts[s];
                hdr->a[s] = A;
            }
            hdr->P[s] = acc;
            acc += raw.dur[s];
        }
    }
    for (uint32_t p = threadIdx.x; p < hdr->NP; p += blockDim.x) {
        hdr->Gprice[p] = (uint64_t)hdr->Gbill[p] * hdr->price[p];
        hdr->PidleG[p] = (uint64_t)hdr->Gbill[p] * hdr->Pidle[p];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < raw.n_va; i += blockDim.x) {
        const uint32_t s = raw.va_scene[i];
        const uint32_t lv = ch_level(hdr->choice[raw.va_choice[i]]);
        VaEntry e;
        e.t_us = raw.va[i];
        e.q = (uint32_t)((raw.dur[s] / 1000ull) * raw.score[lv]);
        e.t_vae = raw.vae ? (uint32_t)raw.vae[i] : 0u;  // < 2^32, validated at create
        va[i] = e;
    }
    __syncthreads();
    // LSD table in (pool, k)-group order (single-scene last block only)
    const uint32_t bl = hdr->B - 1;
    if (hdr->first[bl + 1] - hdr->first[bl] == 1) {
        const int mode = cost_mode(hdr->flags);
        for (uint32_t j = threadIdx.x; j < hdr->radix[bl]; j += blockDim.x) {
            const uint32_t dl = hdr->lsd_dl[j];
            const uint32_t ch = hdr->choice[hdr->coff[bl] + dl];
            const uint32_t p = ch_pool(ch), k = ch_k(ch);
            const VaEntry v = va[hdr->voff[bl] + dl];
            LsdEntry le;
            le.t_us = v.t_us;
            le.q = v.q;
            le.dl = dl;
            if (mode <= 1) {  // money: X_t = G price t (RESERVED) or k price t (BUSY) = cq D + cr
                const uint64_t X = mode ? (uint64_t)k * v.t_us * hdr->price[p] : v.t_us * hdr->Gprice[p];
                le.x1 = X / kUsPerHour;
                le.x2 = X % kUsPerHour;
            } else if (mode == 2) {  // energy, RESERVED: idle G' end + (active - idle) busy
                const uint64_t B = (hdr->Pact[p] - hdr->Pidle[p]) * k * v.t_us;
                le.x1 = hdr->PidleG[p] * v.t_us + B;  // the choice ends the pool: end grows by t too
                le.x2 = B;
            } else {  // energy, BUSY: active x busy
                le.x1 = le.x2 = hdr->Pact[p] * k * v.t_us;
            }
            hdr->lsd[j] = le;
        }
    }
}

#ifndef SW_LSD_UNROLL
#define SW_LSD_UNROLL 2  // 1 and 4 measured 1-2% slower (eval C2, C5; tools/build_variant.py)
#endif
constexpr int kLsdUnroll = SW_LSD_UNROLL;
// ============================================================================ LSD fast path
// The last digit's block is a single scene: only pool p of the chosen (p, k) changes,
// so per candidate  e = max(a_s, F_p[k-1]) + t,  end_p' = max(end_p, e),
// cost = sum_{q != p} cost_q + round((G_p price_p end_p' + 1.8e9) / 3.6e9)  (RESERVED)
// or busy_p + k t (BUSY), the playback metrics of the new scene and one 32 B store.
// Choices are visited grouped by (p, k) (create-time table), and everything that does
// not depend on the choice's stage time t is hoisted into per-group thresholds:
//   e > end_p          <=>  t > end_p - st0           (st0 = max(a_s, F_p[k-1]))
//   R_s - P_s > M      <=>  t > M - (st0 - P_s)       (a new rebuffering maximum, R8)
//   cost carry         <=>  cr >= 3.6e9 - rY          (rY: remainder of the hoisted part)
// so a candidate costs two 16 B table loads, a few 64-bit compares/selects and the store.
template <int K, int NP>
__device__ __forceinline__ uint64_t fk_of(const State<NP>& st, const MidState& m, uint32_t p) {
    // F_p[K-1], pool p's free times taken from the MID copy when p is the MID pool
    uint64_t r = m.F[K - 1];
#pragma unroll
    for (int q = 0; q < NP; q++)
        if ((uint32_t)q == p && p != m.pm) r = st.F[q][K - 1];
    return r;
}

template <int NP>
__device__ __forceinline__ uint64_t fk_pool(const State<NP>& st, const MidState& m, uint32_t p, uint32_t k) {
    switch (k) {
        case 1: return fk_of<1, NP>(st, m, p);
        case 2: return fk_of<2, NP>(st, m, p);
        case 4: return fk_of<4, NP>(st, m, p);
        case 8: return fk_of<8, NP>(st, m, p);
        default: {
            uint64_t r = sel_dyn(m.F, k - 1);
#pragma unroll
            for (int q = 0; q < NP; q++)
                if ((uint32_t)q == p && p != m.pm) r = sel_dyn(st.F[q], k - 1);
            return r;
        }
    }
}

template <int NP, bool ACC, class Put>
__device__ __forceinline__ void lsd_fast(const DevHeader& h, const State<NP>& st, const MidState& m, Put&& put) {
    const uint32_t bl = h.B - 1;
    const uint32_t s = h.first[bl];  // s >= 1 on this path
    const uint64_t as = h.a[s];
    const int64_t Ps = (int64_t)h.P[s];
    // cost mode (cost_mode): 0 without busy accumulation; else 1..3 (uniform over the launch)
    const int mode = ACC ? cost_mode(h.flags) : 0;
    uint64_t pc[NP], endq[NP], busyq[NP];
    uint64_t pcsum = h.fixed_cost;
#pragma unroll
    for (int q = 0; q < NP; q++) {
        endq[q] = (uint32_t)q == m.pm ? m.end : st.end[q];
        busyq[q] = (uint32_t)q == m.pm ? m.busy : st.busy[q];
        if (!ACC) pc[q] = pool_term<0>(h, q, endq[q], 0);
        else if (mode == 1) pc[q] = pool_term<1>(h, q, 0, busyq[q]);
        else if (mode == 2) pc[q] = pool_term<2>(h, q, endq[q], busyq[q]);
        else pc[q] = pool_term<3>(h, q, 0, busyq[q]);
        pcsum += pc[q];
    }
    const uint64_t R0 = m.R0;
    const int64_t M0 = m.M;
    const uint64_t B1 = (uint64_t)M0 - R0;  // w1 = stall when the scene sets no new maximum
    const uint64_t w3base = (uint64_t)m.Q | ((uint64_t)m.cnt << 32) | ((uint64_t)(st.used | m.used) << 48);
    const uint32_t ng = h.lsd_ngroups;
#pragma unroll 1
    for (uint32_t g = 0; g < ng; g++) {
        const uint32_t pk = h.lsd_pk[g];
        const uint32_t p = pk & 0xffu, k = pk >> 8;
        const uint32_t j0 = h.lsd_goff[g], j1 = h.lsd_goff[g + 1];
        if (k == 0) {  // STATIC rung (R33): R_s = a_s, no pool touched, nothing billed
            const int64_t d = (int64_t)as - Ps;
            const bool nm = d > M0;
            Rec4 r;
            r.w0 = R0;
            r.w1 = (uint64_t)(nm ? d : M0) - R0;
            r.w2 = pcsum;
            const uint64_t w3s = w3base + (nm ? (1ull << 32) : 0ull);
            for (uint32_t j = j0; j < j1; j++) {
                const LsdEntry E = h.lsd[j];
                r.w3 = w3s + E.q;
                put(E.dl, E.dl * (kTileRows * (uint32_t)sizeof(Rec4)), r);
            }
            continue;
        }
        uint64_t endp = 0, busyp = 0, pcp = 0;
#pragma unroll
        for (int q = 0; q < NP; q++)
            if ((uint32_t)q == p) {
                endp = endq[q];
                busyp = busyq[q];
                pcp = pc[q];
            }
        const uint64_t st0 = umax64(as, fk_pool<NP>(st, m, p, k));
        const uint64_t base = pcsum - pcp;
        const int64_t dd0 = (int64_t)st0 - Ps;
        const int64_t thrE = (int64_t)endp - (int64_t)st0;  // e > end_p <=> t > thrE
        const int64_t thrM = M0 - dd0;                     // new maximum <=> t > thrM
        const uint64_t A1 = (uint64_t)(dd0 - (int64_t)R0);  // w1 on a new maximum: A1 + t
        const uint64_t w3g = w3base | ((uint64_t)(1u << p) << 48);
        // the cost of the choice's pool, hoisted: cost = U1 + x1 (+ carry) when the scene
        // ends the pool (t > thrE; always for the busy-only modes), else U2 + x2
        uint64_t U1, U2 = 0;
        uint32_t Dm = 0;
        if (mode <= 1) {  // money: Y = (prefix part of X_p) price + 1.8e9 = qY D + rY
            const uint64_t Y = (mode ? busyp * h.price[p] : h.Gprice[p] * st0) + kHalfHour;
            const uint64_t qY = Y / kUsPerHour, rY = Y - qY * kUsPerHour;
            U1 = base + qY;
            U2 = base + pcp;
            Dm = (uint32_t)(kUsPerHour - rY);  // carry iff cr >= Dm (rY + cr >= D)
        } else if (mode == 2) {  // energy RESERVED: PidleG max(end_p, e) + (Pact - Pidle)(busy_p + k t)
            const uint64_t Bb = (h.Pact[p] - h.Pidle[p]) * busyp;
            U1 = base + h.PidleG[p] * st0 + Bb;
            U2 = base + h.PidleG[p] * endp + Bb;
        } else {  // energy BUSY: Pact (busy_p + k t)
            U1 = base + h.Pact[p] * busyp;
        }
        auto emit = [&](const LsdEntry& E, uint64_t cost) {
            const int64_t t = (int64_t)E.t_us;
            const bool nm = t > thrM;
            Rec4 r;
            r.w0 = R0;
            r.w1 = nm ? A1 + (uint64_t)t : B1;
            r.w2 = cost;
            r.w3 = (w3g + E.q) + (nm ? (1ull << 32) : 0ull);
            put(E.dl, E.dl * (kTileRows * (uint32_t)sizeof(Rec4)), r);  // a7 store, or the stream filter
        };
        if (mode == 0) {
            // the eval store unrolls (ILP); the stream filter does not (registers)
            constexpr int kUnr = std::decay_t<Put>::kUnroll;
#pragma unroll kUnr
            for (uint32_t j = j0; j < j1; j++) {
                const LsdEntry E = h.lsd[j];
                const uint64_t cnew = U1 + E.x1 + ((uint32_t)E.x2 >= Dm ? 1u : 0u);
                emit(E, (int64_t)E.t_us > thrE ? cnew : U2);
            }
        } else if (ACC && mode == 1) {
            for (uint32_t j = j0; j < j1; j++) {
                const LsdEntry E = h.lsd[j];
                emit(E, U1 + E.x1 + ((uint32_t)E.x2 >= Dm ? 1u : 0u));
            }
        } else if (ACC && mode == 2) {
            for (uint32_t j = j0; j < j1; j++) {
                const LsdEntry E = h.lsd[j];
                emit(E, (int64_t)E.t_us > thrE ? U1 + E.x1 : U2 + E.x2);
            }
        } else if (ACC) {
            for (uint32_t j = j0; j < j1; j++) {
                const LsdEntry E = h.lsd[j];
                emit(E, U1 + E.x1);
            }
        }
    }
}

// Scenes [f0, f1) of one digit's block with choice ch (pool, k, optional VAE stage R37), gang
// update specialised for K (K = 0: runtime k).  ACC: accumulate busy GPU time.
// VAE: compile the VAE stage in (the fast eval path never has one).
template <int NP, int K, bool ACC = true, bool VAE = true>
__device__ __forceinline__ void run_block(State<NP>& st, const DevHeader& h, uint32_t ch, uint32_t f0, uint32_t f1,
                                          const VaEntry* vb, uint32_t r, uint64_t* ready = nullptr) {
    const uint32_t p = ch_pool(ch), k = ch_k(ch), vae = VAE ? ch_vae(ch) : 0u;
#pragma unroll 1  // one copy of the step per K: the gang updates dominate the code size
    for (uint32_t s = f0; s < f1; s++) {
        const VaEntry v = vb[(s - f0) * r];
        uint64_t e = scene_step<NP, K, ACC>(st, p, k, h.a[s], v.t_us);
        if (VAE && vae) e = vae_step<NP, ACC>(st, vae - 1, e, v.t_vae);
        scene_metrics(st, s, e, h.P[s], v.q);
        if (ready) ready[s] = e;
    }
}

// run_block with a warp-uniform runtime k dispatched to the compile-time specialisations.
template <int NP, bool ACC = true>
__device__ __forceinline__ void run_block_uniform(State<NP>& st, const DevHeader& h, uint32_t ch, uint32_t f0,
                                                  uint32_t f1, const VaEntry* vb, uint32_t r,
                                                  uint64_t* ready = nullptr) {
    switch (ch_k(ch)) {
        case 1: run_block<NP, 1, ACC>(st, h, ch, f0, f1, vb, r, ready); break;
        case 2: run_block<NP, 2, ACC>(st, h, ch, f0, f1, vb, r, ready); break;
        case 4: run_block<NP, 4, ACC>(st, h, ch, f0, f1, vb, r, ready); break;
        case 8: run_block<NP, 8, ACC>(st, h, ch, f0, f1, vb, r, ready); break;
        default: run_block<NP, 0, ACC>(st, h, ch, f0, f1, vb, r, ready); break;
    }
}

// MID block scenes [f0, f1) on the MID copy, compile-time K.
template <int K, bool BUSY>
__device__ __forceinline__ void mid_block(MidState& m, const DevHeader& h, uint32_t k, uint32_t f0, uint32_t f1,
                                          const VaEntry* vb, uint32_t r) {
#pragma unroll 1
    for (uint32_t s = f0; s < f1; s++) {
        const VaEntry v = vb[(s - f0) * r];
        const uint64_t e = mid_step<K, BUSY>(m, k, h.a[s], v.t_us);
        scene_metrics(m, s, e, h.P[s], v.q);
    }
}

// ============================================================================ a1-a7 eval
// Lane <-> row H: the candidates [H*row, (H+1)*row) share their HI digits (digits
// 0..B-3); a warp owns a tile of 32 consecutive rows (tiled record layout, sw_plan.h).
// The thread simulates the HI scenes once (per-lane choices, runtime k/pool), then
// iterates the MID digit and the LSD digit in lock-step with the other lanes: (k, pool)
// is warp-uniform there, so the gang update uses compile-time slot indices and the LSD
// step (the dominant loop) is a few integer ops + one 32 B store.
// Amortised scene-steps per candidate: L_LSD + L_MID / r_LSD + L_HI / row.
// One eval launch's work for one request: its tables and the tile range to write.
struct EvalJob {
    const DevHeader* hdr;
    const VaEntry* va;
    uint64_t va_bytes;
    uint64_t tile_begin, tile_end;
    Rec4* out;
};

// One tile (32 consecutive rows, lane <-> row H = t * 32 + lane) of candidates: record
// (dm, dl) of the lane's row goes to emit.at(dm, live)(dl, off, r) -- the 32 B store of
// the eval kernel, or the fused select + Pareto filter of the stream kernel.
// BUSY: accumulate busy GPU time (every cost mode but money + RESERVED).  DIS (the
// "generic" path): full-state MID pass and per-candidate LSD blocks, for handles whose LSD
// block has several scenes (or starts at scene 0) or that have DiT/VAE disaggregated
// choices (R37); the fast path (single-pool MID copy + lsd_fast) is a separate
// instantiation, so neither carries the other's code or registers.
// [slice of nslice]: only the MID digits [slice rm / nslice, (slice + 1) rm / nslice) (the
// stream kernel splits small passes' tiles so that they fill the GPU).
template <int NP, bool BUSY, bool DIS, class Emit>
__device__ __forceinline__ void eval_tile_b(const DevHeader& h, const VaEntry* va, uint64_t t, Emit&& emit,
                                            uint32_t slice = 0, uint32_t nslice = 1) {
    const uint32_t bm = h.B - 2, bl = h.B - 1;
    const uint32_t rm = h.radix[bm], rl = h.radix[bl];
    const uint32_t dm0 = slice * rm / nslice, dm1 = (slice + 1) * rm / nslice;
    const uint32_t mfirst = h.first[bm], mlast = h.first[bm + 1];
    const uint32_t lfirst = h.first[bl], llast = h.first[bl + 1];
    const uint64_t n_rows = h.n_rows;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t Hraw = t * kTileRows + lane;
    const bool live = Hraw < n_rows;  // the last tile may run past the space
    const uint64_t H = live ? Hraw : n_rows - 1;
    State<NP> st;
    state_init(st, h);
    // ---- HI prefix: decode the row index (MSD = earliest block, R19) and simulate
    uint64_t rem = H;
    for (uint32_t b = 0; b < bm; b++) {
        const uint64_t pl = h.place[b];
        uint32_t c;
        if ((rem >> 32) == 0 && (pl >> 32) == 0) c = (uint32_t)rem / (uint32_t)pl;
        else c = (uint32_t)(rem / pl);
        rem -= (uint64_t)c * pl;
        const uint32_t ch = h.choice[h.coff[b] + c];
        const uint32_t k = ch_k(ch), p = ch_pool(ch);
        const uint32_t f0 = h.first[b], f1 = h.first[b + 1], r = h.radix[b];
        const VaEntry* vb = va + h.voff[b] + c;
        // lanes are 32 consecutive rows: the high digits usually agree across the
        // warp -- then (k, p) is warp-uniform and the compile-time gang update runs;
        // otherwise the runtime-k update (a divergent switch over the compile-time
        // variants measured 12% slower overall on C2)
        if (__all_sync(0xffffffffu, ch == __shfl_sync(0xffffffffu, ch, 0))) {
            switch (k) {
                case 1: run_block<NP, 1, BUSY, DIS>(st, h, ch, f0, f1, vb, r); break;
                case 2: run_block<NP, 2, BUSY, DIS>(st, h, ch, f0, f1, vb, r); break;
                case 4: run_block<NP, 4, BUSY, DIS>(st, h, ch, f0, f1, vb, r); break;
                case 8: run_block<NP, 8, BUSY, DIS>(st, h, ch, f0, f1, vb, r); break;
                default: run_block<NP, 0, BUSY, DIS>(st, h, ch, f0, f1, vb, r); break;
            }
        } else {
            run_block<NP, 0, BUSY, DIS>(st, h, ch, f0, f1, vb, r);
        }
    }
    if (DIS) {
        // ---- DiT/VAE disaggregated choices (R37) touch two pools per scene: MID and LSD
        // digits on full state copies (no single-pool MID copy, no LSD fast path)
        for (uint32_t dm = dm0; dm < dm1; dm++) {
            State<NP> s2 = st;
            const uint32_t chm = h.choice[h.coff[bm] + dm];
            run_block_uniform<NP, BUSY>(s2, h, chm, mfirst, mlast, va + h.voff[bm] + dm, rm);
            auto put = emit.at(dm, live);
            for (uint32_t dl = 0; dl < rl; dl++) {
                State<NP> s3 = s2;
                const uint32_t chl = h.choice[h.coff[bl] + dl];
                run_block_uniform<NP, BUSY>(s3, h, chl, lfirst, llast, va + h.voff[bl] + dl, rl);
                Rec4 r;
                r.w0 = s3.R0;
                r.w1 = (uint64_t)s3.M - s3.R0;
                r.w2 = state_cost(s3, h);
                r.w3 = (uint64_t)s3.Q | ((uint64_t)s3.cnt << 32) | ((uint64_t)s3.used << 48);
                put(dl, dl * kTileRows * (uint32_t)sizeof(Rec4), r);
            }
        }
        return;
    }
    // ---- MID digit: warp-uniform choice (k, pm) on a copy of pool pm only
    for (uint32_t dm = dm0; dm < dm1; dm++) {
        const uint32_t ch = h.choice[h.coff[bm] + dm];
        const uint32_t k = ch_k(ch), pm = ch_pool(ch);
        MidState m;
        mid_init<NP>(m, st, pm);
        {
            const VaEntry* vb = va + h.voff[bm] + dm;
            switch (k) {
                case 1: mid_block<1, BUSY>(m, h, k, mfirst, mlast, vb, rm); break;
                case 2: mid_block<2, BUSY>(m, h, k, mfirst, mlast, vb, rm); break;
                case 4: mid_block<4, BUSY>(m, h, k, mfirst, mlast, vb, rm); break;
                case 8: mid_block<8, BUSY>(m, h, k, mfirst, mlast, vb, rm); break;
                default: mid_block<0, BUSY>(m, h, k, mfirst, mlast, vb, rm); break;
            }
        }
        lsd_fast<NP, BUSY>(h, st, m, emit.at(dm, live));  // record (dm, dl) of this lane's row
    }
}

template <int NP, class Emit>
__device__ __forceinline__ void eval_tile(const DevHeader& h, const VaEntry* va, uint64_t t, Emit&& emit) {
    // busy GPU time is needed by every cost mode but money + RESERVED (uniform branch)
    switch (eval_mode(h.flags)) {
        case 0: eval_tile_b<NP, false, false>(h, va, t, emit); break;
        case 1: eval_tile_b<NP, true, false>(h, va, t, emit); break;
        default: eval_tile_b<NP, true, true>(h, va, t, emit); break;
    }
}

// a7: the 32 B store.  Record (dm, dl) of the lane's row lands at tile_out + (dm * rl +
// dl) * 32: a warp store covers 32 consecutive records (1 KB, fully coalesced).  Lanes past
// the end of the space (last tile only) write their tile-padding slot (the tile is
// allocated whole; scans skip indices outside the segment), so the store is unconditional.
struct StoreEmit {
    Rec4* tile_out;  // this lane's first slot in its tile
    uint32_t rl;
    struct Put {
        static constexpr int kUnroll = kLsdUnroll;
        char* lane_out;
        __device__ __forceinline__ void operator()(uint32_t, uint32_t off, const Rec4& r) const {
            st_global_256(lane_out + off, r);
        }
    };
    __device__ __forceinline__ Put at(uint32_t dm, bool) const {
        return Put{reinterpret_cast<char*>(tile_out + (size_t)dm * rl * kTileRows)};
    }
};

// Resident CTAs per SM the register allocation is sized for, per pool count: the state
// grows with the pools (NP + 1 pools of 8 free times live in the MID/LSD loops), and
// these are the largest occupancies whose hot loops do not spill (ptxas -v).
// fast path (BM 0/1) vs generic path (BM 2/3, full-state copies)
#ifndef SW_EVAL_MINB1
#define SW_EVAL_MINB1 4  // (experiments: tools/build_variant.py)
#endif
__host__ __device__ constexpr int eval_min_blocks(int np, int bm) {
    return bm <= 1 ? (np == 1 ? SW_EVAL_MINB1 : np == 2 ? 4 : np == 3 ? 3 : 2) : (np <= 1 ? 4 : np == 2 ? 3 : 2);
}

// jobs == nullptr: one request (job); else request blockIdx.y of a fleet (jobs[y]), each
// CTA staging its own request's tables -- a whole fleet in one launch.
// BM: path of the launch (eval_mode) -- 0 fast path without busy time (money + RESERVED),
// 1 fast path with busy time (BUSY billing or the energy metric), 2 generic path, 3 per
// request at run time (a fleet mixing them).  Compile-time for single requests: one copy of
// the tile code per kernel (a runtime switch inside multiplied the code and cost
// instruction-cache misses and registers).

template <int NP, int BM = 3>
__global__ void __launch_bounds__(kEvalThreads, eval_min_blocks(NP, BM)) eval_kernel(EvalJob job, const EvalJob* __restrict__ jobs) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar;
    if (jobs) job = jobs[blockIdx.y];
    const uint64_t tile_begin = job.tile_begin, tile_end = job.tile_end;
    Rec4* __restrict__ out = job.out;
    DevHeader& h = *reinterpret_cast<DevHeader*>(smem);
    VaEntry* va = reinterpret_cast<VaEntry*>(smem + sizeof(DevHeader));
    stage_tables(job.hdr, job.va, &h, va, (uint32_t)job.va_bytes, &bar);
    const uint64_t row = h.row;
    const uint32_t rl = h.radix[h.B - 1];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    // warp <-> tile of 32 consecutive rows; lane <-> row H = tile * 32 + lane
    for (uint64_t t = tile_begin + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); t < tile_end;
         t += nwarps) {
        const StoreEmit em{out + (t - tile_begin) * kTileRows * row + lane, rl};
        if (BM == 3) eval_tile<NP>(h, va, t, em);
        else eval_tile_b<NP, BM != 0, BM == 2>(h, va, t, em);
    }
}

// ============================================================================ detail
struct DetailOut {
    Rec4 rec;
    uint64_t ttff_eff, makespan;
    uint64_t pool_end[kMaxP];
    uint64_t ready[SW_MAX_SCENES];
    uint32_t digit[kMaxDigits];
};

template <int NP>
__device__ void detail_one(const DevHeader* __restrict__ g_hdr, const VaEntry* __restrict__ g_va, uint64_t index,
                           DetailOut* __restrict__ out) {
    const DevHeader& h = *g_hdr;
    State<NP> st;
    state_init(st, h);
    uint32_t dig[kMaxDigits];
    uint64_t rem = index;
    for (int b = (int)h.B - 1; b >= 0; b--) {  // a1: i mod r_b, LSD first
        dig[b] = (uint32_t)(rem % h.radix[b]);
        rem /= h.radix[b];
    }
    if (h.flags & 1u) out->ready[0] = h.R0_static;
    for (uint32_t b = 0; b < h.B; b++) {
        const uint32_t c = dig[b];
        out->digit[b] = c;
        const uint32_t ch = h.choice[h.coff[b] + c];
        const uint32_t k = ch_k(ch), p = ch_pool(ch);
        const VaEntry* vb = g_va + h.voff[b] + c;
        const uint32_t f0 = h.first[b], f1 = h.first[b + 1], r = h.radix[b];
        switch (k) {  // compile-time gang updates (a single thread: no divergence cost)
            case 1: run_block<NP, 1>(st, h, ch, f0, f1, vb, r, out->ready); break;
            case 2: run_block<NP, 2>(st, h, ch, f0, f1, vb, r, out->ready); break;
            case 4: run_block<NP, 4>(st, h, ch, f0, f1, vb, r, out->ready); break;
            case 8: run_block<NP, 8>(st, h, ch, f0, f1, vb, r, out->ready); break;
            default: run_block<NP, 0>(st, h, ch, f0, f1, vb, r, out->ready); break;
        }
    }
    uint64_t mk = st.R0;
    for (int p = 0; p < NP; p++) {
        out->pool_end[p] = st.end[p];
        mk = umax64(mk, st.end[p]);
    }
    for (uint32_t s = 0; s < h.S; s++) mk = umax64(mk, out->ready[s]);  // STATIC scenes (R33)
    out->rec.w0 = st.R0;
    out->rec.w1 = (uint64_t)st.M - st.R0;
    out->rec.w2 = state_cost(st, h);
    out->rec.w3 = (uint64_t)st.Q | ((uint64_t)st.cnt << 32) | ((uint64_t)st.used << 48);
    out->ttff_eff = (uint64_t)st.M;
    out->makespan = mk;
}

template <int NP>
__global__ void detail_kernel(const DevHeader* __restrict__ g_hdr, const VaEntry* __restrict__ g_va,
                              uint64_t index, DetailOut* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    detail_one<NP>(g_hdr, g_va, index, out);
}

// ============================================================================ a9 select
struct QueryDev {
    uint64_t slo_t, slo_s, budget;
};
struct SelParams {
    uint32_t nq, objective;
    QueryDev q[SW_MAX_QUERIES];
};
struct Cand {
    uint64_t idx;  // kInf64 = none
    uint64_t pad;
    Rec4 r;
};

// The comparison functions below are __host__ __device__: the same code ranks candidates
// in the scan kernels, the cross-rank merge kernel and the host-side sw_selection_merge.
__host__ __device__ __forceinline__ uint64_t sat_sub(uint64_t x, uint64_t y) { return x > y ? x - y : 0; }

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ bool feasible(const QueryDev& q, const Rec4& r) {
    return r.w0 <= q.slo_t && r.w1 <= q.slo_s && r.w2 <= q.budget;
}

// Objective order (R13): true iff a precedes b.
__host__ __device__ __forceinline__ int obj_cmp(uint32_t obj, uint64_t ia, const Rec4& a, uint64_t ib,
                                       const Rec4& b) {
    const uint64_t ta = a.w0 + a.w1, tb = b.w0 + b.w1;
    const uint32_t qa = rec_Q(a), qb = rec_Q(b);
    if (obj == 0) {  // QUALITY_FIRST (-Q, cost, ttff_eff, index)
        if (qa != qb) return qa > qb ? -1 : 1;
        if (a.w2 != b.w2) return a.w2 < b.w2 ? -1 : 1;
        if (ta != tb) return ta < tb ? -1 : 1;
    } else {  // COST_X_TTFF (cost x ttff_eff as 128-bit, -Q, index)
        const uint64_t lo_a = a.w2 * ta, hi_a = mulhi64(a.w2, ta);
        const uint64_t lo_b = b.w2 * tb, hi_b = mulhi64(b.w2, tb);
        if (hi_a != hi_b) return hi_a < hi_b ? -1 : 1;
        if (lo_a != lo_b) return lo_a < lo_b ? -1 : 1;
        if (qa != qb) return qa > qb ? -1 : 1;
    }
    if (ia != ib) return ia < ib ? -1 : 1;
    return 0;
}

// Total order of a query: feasible plans by objective; then (nothing feasible)
// the closest plan by (V_t, V_c, objective, index) ("returns the closest
// solution").  Invalid candidates (idx = inf) are last.
__host__ __device__ __forceinline__ bool cand_better(const QueryDev& q, uint32_t obj, uint64_t ia,
                                            const Rec4& a, uint64_t ib, const Rec4& b) {
    if (ib == kInf64) return ia != kInf64;
    if (ia == kInf64) return false;
    const bool fa = feasible(q, a), fb = feasible(q, b);
    if (fa != fb) return fa;
    if (!fa) {
        const uint64_t vta = sat_sub(a.w0, q.slo_t) + sat_sub(a.w1, q.slo_s);
        const uint64_t vtb = sat_sub(b.w0, q.slo_t) + sat_sub(b.w1, q.slo_s);
        if (vta != vtb) return vta < vtb;
        const uint64_t vca = sat_sub(a.w2, q.budget), vcb = sat_sub(b.w2, q.budget);
        if (vca != vcb) return vca < vcb;
    }
    return obj_cmp(obj, ia, a, ib, b) < 0;
}

__device__ __forceinline__ void shfl_cand(uint64_t& idx, Rec4& r, int off) {
    const uint64_t i2 = __shfl_down_sync(0xffffffffu, idx, off);
    Rec4 o;
    o.w0 = __shfl_down_sync(0xffffffffu, r.w0, off);
    o.w1 = __shfl_down_sync(0xffffffffu, r.w1, off);
    o.w2 = __shfl_down_sync(0xffffffffu, r.w2, off);
    o.w3 = __shfl_down_sync(0xffffffffu, r.w3, off);
    idx = i2;
    r = o;
}

// Block-level argmin of per-thread candidates; result valid in thread 0.
__device__ __forceinline__ void block_reduce_cand(const QueryDev& q, uint32_t obj, uint64_t& idx,
                                                  Rec4& r, Cand* s_tmp /* [32] */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        uint64_t oi = idx;
        Rec4 orr = r;
        shfl_cand(oi, orr, off);
        if (lane + off < 32 && cand_better(q, obj, oi, orr, idx, r)) {
            idx = oi;
            r = orr;
        }
    }
    __syncthreads();
    if (lane == 0) {
        s_tmp[warp].idx = idx;
        s_tmp[warp].r = r;
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        if (lane < nw) {
            idx = s_tmp[lane].idx;
            r = s_tmp[lane].r;
        } else {
            idx = kInf64;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            uint64_t oi = idx;
            Rec4 orr = r;
            shfl_cand(oi, orr, off);
            if (lane + off < 32 && cand_better(q, obj, oi, orr, idx, r)) {
                idx = oi;
                r = orr;
            }
        }
    }
}

// Reduce n_partial candidates per query (strided by SW_MAX_QUERIES) -> out[q].
// Used after the scan (per-block partials) and for the cross-rank merge (a10).
__global__ void __launch_bounds__(kScanThreads) select_final_kernel(
    const Cand* __restrict__ partial, uint32_t n_partial, SelParams P, Cand* __restrict__ out) {
    __shared__ Cand s_tmp[32];
    for (uint32_t q = 0; q < P.nq; q++) {
        uint64_t idx = kInf64;
        Rec4 r{};
        for (uint32_t j = threadIdx.x; j < n_partial; j += blockDim.x) {
            const Cand c = partial[(uint64_t)j * SW_MAX_QUERIES + q];
            if (cand_better(P.q[q], P.objective, c.idx, c.r, idx, r)) {
                idx = c.idx;
                r = c.r;
            }
        }
        block_reduce_cand(P.q[q], P.objective, idx, r, s_tmp);
        if (threadIdx.x == 0) {
            out[q].idx = idx;
            out[q].r = r;
            // status flag for the host: 1 = closest (nothing feasible)
            out[q].pad = (idx != kInf64 && !feasible(P.q[q], r)) ? 1ull : 0ull;
        }
        __syncthreads();
    }
}

// ============================================================================ digest
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(kScanThreads) digest_kernel(SegView v, unsigned long long* __restrict__ acc) {
    uint64_t sum = 0;
    const uint32_t per_tile = (uint32_t)(kTileRows * v.row);
    for (uint64_t t = blockIdx.x; t < v.ntiles; t += gridDim.x) {
        const Rec4* tp = v.recs + t * per_tile;
        for (uint32_t p = threadIdx.x; p < per_tile; p += blockDim.x) {
            const uint64_t idx = tiled_index(v.t0, v.row, t, p);
            if (idx < v.ib || idx >= v.ie) continue;
            const Rec4 r = ld_global_nc_256(tp + p);
            // w3 = Q | cnt << 32 | flags << 48  ->  flags << 48 | Q << 16 | cnt
            const uint64_t w = ((r.w3 >> 48) << 48) | ((r.w3 & 0xffffffffull) << 16) | ((r.w3 >> 32) & 0xffffull);
            sum += mix64(idx ^ rotl64(r.w0, 7) ^ rotl64(r.w1, 19) ^ rotl64(r.w2, 31) ^ w);
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)sum);
}

// ============================================================================ a8 Pareto
struct __align__(16) PPoint {  // == sw_pareto_point
    uint64_t idx, t, c;
    uint32_t q, pad;
};

// y dominates x: <= in ttff_eff and cost, >= in quality, one strict; exact duplicates
// keep the lowest index (R14); identical entries (same index) keep the first position.
__device__ __forceinline__ bool pdom(const PPoint& y, uint32_t py, const PPoint& x, uint32_t px) {
    // branch-free, so that unrolled loops overlap several tests
    const bool le = (y.t <= x.t) & (y.c <= x.c) & (y.q >= x.q);
    const bool strict = (y.t < x.t) | (y.c < x.c) | (y.q > x.q);
    const bool tie = (y.idx < x.idx) | ((y.idx == x.idx) & (py < px));
    return le & (strict | tie);
}

// Device-side sizes of the Pareto merge pipeline: every kernel below reads its input
// count from here, so a whole merge runs without a host round trip.
struct ParetoCtl {
    unsigned long long surv;  // survivors appended by the current filter pass
    uint32_t m_in, m_loc, m_loc2, m_cmp;
    uint64_t front_n;         // size of the running front (d_front)
    uint32_t surv_overflow;   // a filter pass had more survivors than capacity
    uint32_t front_overflow;  // the front exceeded its capacity
    uint64_t stamp[6];        // diagnostics: %globaltimer at the merge kernel's phase ends
    unsigned long long dlt_pass;  // diagnostics: records the DLT did not rule out (all passes)
    unsigned long long dlt_n;     // DLT survivors appended by the current scan pass (deferred exact test)
    unsigned long long dlt_max;   // the largest dlt_n of any pass since the host last looked (buffer growth)
    uint32_t rkmin, rkmax;        // merge: range of the t sort keys (bucket sort before the local fronts)
};

// Per-call status words of a multi-rank call, max-reduced over the ranks BEFORE any rank
// takes a branch that involves another collective (a rank-local decision next to a
// collective hangs or mispairs the peers): [0] a filter pass of this call overflowed its
// survivor buffer (refold + exact front redo), [1] the front overflowed its capacity,
// [2] a stream query's candidate list overflowed, [3] a host-side error of this rank,
// [4] the call's argument fingerprint and [5] its complement (after the max-reduction
// max(fp) == ~max(~fp) iff every rank made the same call with the same arguments).
constexpr uint32_t kStatusWords = 6;
__global__ void status_words_kernel(const ParetoCtl* __restrict__ ctl, const uint32_t* __restrict__ cand_n,
                                    uint32_t nq, uint32_t cap, uint64_t host_flag, uint64_t fp,
                                    uint64_t* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t over = 0;
    for (uint32_t q = 0; q < nq; q++) over |= cand_n[q] > cap ? 1ull : 0ull;
    out[0] = ctl->surv_overflow ? 1ull : 0ull;
    out[1] = ctl->front_overflow ? 1ull : 0ull;
    out[2] = over;
    out[3] = host_flag;
    out[4] = fp;
    out[5] = ~fp;
}

// keep[x] = no other point of pts[0,m) dominates x.  O(m^2), tiles through smem.
__global__ void __launch_bounds__(kScanThreads) pareto_mark_kernel(const PPoint* __restrict__ pts,
                                                                   const uint32_t* __restrict__ d_m,
                                                                   uint8_t* __restrict__ keep) {
    __shared__ PPoint tile[kScanThreads];
    const uint32_t m = *d_m;
    if (blockIdx.x * blockDim.x >= m) return;
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    PPoint px{};
    if (x < m) px = pts[x];
    bool dom = x >= m;
    for (uint32_t base = 0; base < m; base += blockDim.x) {
        if (__syncthreads_and(dom)) break;
        const uint32_t y = base + threadIdx.x;
        if (y < m) tile[threadIdx.x] = pts[y];
        __syncthreads();
        const uint32_t lim = min((uint32_t)blockDim.x, m - base);
        if (!dom)
            for (uint32_t j = 0; j < lim; j++)
                if (base + j != x && pdom(tile[j], base + j, px, x)) {
                    dom = true;
                    break;
                }
        __syncthreads();
    }
    if (x < m) keep[x] = dom ? 0 : 1;
}

__global__ void pareto_compact_kernel(const PPoint* __restrict__ pts, const uint32_t* __restrict__ d_m,
                                      const uint8_t* __restrict__ keep, PPoint* __restrict__ out,
                                      uint32_t* __restrict__ count) {
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < *d_m && keep[x]) out[atomicAdd(count, 1u)] = pts[x];
}

__device__ __forceinline__ bool pkey_less(const PPoint& a, const PPoint& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.c != b.c) return a.c < b.c;
    if (a.q != b.q) return a.q > b.q;
    return a.idx < b.idx;
}

// out[rank(x)] = x with rank = #{y : key(y) < key(x)}: deterministic ordering of a
// front (indices are unique) by (ttff_eff asc, cost asc, quality desc, index asc).
// Publishes the new front size; flags an overflow of the front capacity.
__global__ void __launch_bounds__(kScanThreads) pareto_rank_kernel(const PPoint* __restrict__ pts,
                                                                   const uint32_t* __restrict__ d_m,
                                                                   PPoint* __restrict__ out, ParetoCtl* ctl,
                                                                   uint64_t cap) {
    __shared__ PPoint tile[kScanThreads];
    const uint32_t m = *d_m;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->front_n = m <= cap ? m : 0;
        if (m > cap) ctl->front_overflow = 1;
    }
    if (m > cap || blockIdx.x * blockDim.x >= m) return;
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    PPoint px{};
    if (x < m) px = pts[x];
    uint32_t rank = 0;
    for (uint32_t base = 0; base < m; base += blockDim.x) {
        const uint32_t y = base + threadIdx.x;
        if (y < m) tile[threadIdx.x] = pts[y];
        __syncthreads();
        const uint32_t lim = min((uint32_t)blockDim.x, m - base);
        for (uint32_t j = 0; j < lim; j++) rank += pkey_less(tile[j], px) ? 1u : 0u;
        __syncthreads();
    }
    if (x < m) out[rank] = px;
}

// Dominance lookup table (DLT) from the current front (sorted by ttff_eff).
// t-bins: quantile edges of the front's t (tedge ascending, bin b holds t >= tedge[b]);
// q-bins: (qtop[j-1], qtop[j]] with tops at front quality values (dlt_qtop_kernel).
// cell[b][j] = min cost over front points f with f.t <= tedge[b] and f.q >= the largest
// q of bin j, as u32 (0xffffffff = none / too big).  A record (t, c, q) in cell (b, j)
// with cell < c is strictly dominated by a real candidate (f.t <= t, f.q >= q, f.c < c),
// so it cannot be on the front.  Lookup is O(1) and conservative: the t bin comes from a
// fine direct map of the float exponent + 8 mantissa bits (the bin of the map cell's
// lower end), the q bin is a shift.
struct Dlt {
    int32_t kbase;         // t key of tmap[0]
    uint32_t qbase;        // q of qmap[0]'s lower end (= qtop[0])
    uint32_t qmshift;      // q map cell width 2^qmshift
    uint32_t ntop;         // quality bin tops in use (<= kDltQ)
    uint32_t cshift, pad_[3];
    uint64_t tedge[kDltT + 1];
    // t map cell k: lo = #edges <= the cell's lower end, hi = #edges <= its upper end
    // (packed lo | hi << 8).  A record's bin count is hi when t >= tedge[hi - 1] (the
    // cell's largest edge), else lo -- exact also when many front points share one t
    // (e.g. every stall-free plan behind a static intro)
    uint16_t tmap[kDltMap];
    // cell[b1][j] (row b1 = t bin + 1, column j = q bin): min cost >> cshift, rounded down;
    // 0xffff = none.  Row 0 (no front point has t <= the record's t) and column kDltQ (q
    // above every front point's) are all "none", so the lookup needs no range checks.  A
    // record with cost c is strictly dominated when min(c >> cshift, 0xffff) > cell, i.e.
    // c >= (cell + 1) << cshift > the true minimum.
    uint16_t cell[(kDltT + 1) * kDltCols];
    // quality bins (round 2): bin j = (qtop[j-1], qtop[j]], the tops are front quality
    // values (all distinct ones, or quantiles of them), so a column needs f.q >= qtop[j]
    // and a front point of the record's OWN quality still counts (linear bins of width 2^k
    // needed f.q >= the bin's top and missed same-quality dominators -- the common case
    // with discrete quality levels).  q map: kDltQMap linear cells of 2^qmshift from qbase
    // over the tops' range; cell k: lo = #tops < its lower end, hi = #tops <= its upper
    // end; a record's column is lo when q <= qtop[lo], else hi (exact when the cell holds
    // <= 1 top, else conservative: column hi needs f.q >= qtop[hi] >= q).  Packed per cell
    // as {qtop[lo] (~0 when lo = ntop), lo | hi << 8}: one 8 B shared load per lookup.
    uint32_t qtop[kDltQ];
    uint2 qmap[kDltQMap];
};
static_assert(sizeof(Dlt) % 16 == 0, "Dlt is staged in 16 B vectors");

__device__ __forceinline__ int32_t dlt_tkey(uint64_t t) {
    return (int32_t)(__float_as_uint(__ull2float_rz(t)) >> kDltTShift);
}

// The DLT's scalar fields, held in registers by the scan consumers.
struct DltHot {
    int32_t kbase;
    uint32_t qbase, qmshift, cshift;
};

__device__ __forceinline__ bool dlt_dominated(const Dlt& d, const DltHot& hs, uint64_t t, uint64_t c, uint32_t q) {
    // branch-free and check-free: the map's cell 0 lies below the front's smallest t (so a
    // clamped t below it gets row 0), column kDltQ catches q above the front's
    const int32_t k = dlt_tkey(t) - hs.kbase;
    const uint32_t kc = (uint32_t)min(max(k, 0), kDltMap - 1);
    const uint2 qm = d.qmap[min((max(q, hs.qbase) - hs.qbase) >> hs.qmshift, (uint32_t)kDltQMap - 1)];
    const uint32_t loq = qm.y & 0xffu, hiq = qm.y >> 8;
    const uint32_t j = q > qm.x ? hiq : loq;  // #tops < q (column; kDltQ = none)
    const uint32_t lh = d.tmap[kc];
    const uint32_t lo = lh & 0xffu, hi = lh >> 8;
    const uint32_t b1 = (hi > lo && t >= d.tedge[hi > 0 ? hi - 1 : 0]) ? hi : lo;  // t bin + 1
    const uint32_t cell = d.cell[b1 * kDltCols + j];
    const uint64_t cs = c >> hs.cshift;
    return (uint32_t)(cs < 0xffffull ? cs : 0xffffull) > cell;
}

// Quality bin tops and the q map of the DLT (before dlt_build_kernel): the front's quality
// values rank-sorted over the grid (rank = #smaller + #equal at a lower position, 16
// threads per value), then the last block to finish takes the distinct ones -- all, or
// kDltQ quantiles of them -- as tops.  Fronts above kDltSortMax points take kDltQ linear
// tops over [qmin, qmax] instead (still exact: a column only ever counts f.q >= its top).
constexpr uint32_t kDltSortMax = 16384;
constexpr int kDltQThreads = 1024;
constexpr int kDltQtopGrid = 64;  // the rank sort's blocks (64 values per block step)
__global__ void __launch_bounds__(kDltQThreads) dlt_qtop_kernel(const PPoint* __restrict__ front,
                                                                const ParetoCtl* __restrict__ ctl, Dlt* __restrict__ d,
                                                                uint32_t* __restrict__ qsorted,
                                                                uint32_t* __restrict__ done) {
    extern __shared__ uint32_t qs[];  // kDltSortMax
    __shared__ uint32_t s_nd, s_qmin, s_qmax;
    __shared__ uint32_t s_wsum[32];
    __shared__ uint32_t s_top[kDltQ];
    __shared__ uint32_t s_cnt[64];
    __shared__ bool s_last;
    const uint32_t m = (uint32_t)ctl->front_n, tid = threadIdx.x;
    const bool sortable = m > 0 && m <= kDltSortMax;
    if (sortable) {  // (1) rank sort over the grid: 64 values per block step, 16 threads each
        const uint32_t pl = tid % 64, part = tid / 64;
        for (uint32_t base = blockIdx.x * 64; base < m; base += gridDim.x * 64) {
            const uint32_t p = base + pl;
            const uint32_t v = p < m ? __ldg(&front[p].q) : 0u;
            if (tid < 64) s_cnt[tid] = 0;
            __syncthreads();
            uint32_t r = 0;  // #{j: q_j < v} + #{j < p: q_j = v}
            if (p < m)
#pragma unroll 4
                for (uint32_t j = part; j < m; j += kDltQThreads / 64) {
                    const uint32_t w = __ldg(&front[j].q);
                    r += (w < v || (w == v && j < p)) ? 1u : 0u;
                }
            atomicAdd(&s_cnt[pl], r);
            __syncthreads();
            if (tid < 64 && p < m) qsorted[s_cnt[tid]] = v;
            __syncthreads();
        }
    }
    // (2) the last block to finish derives the tops and the q map from the sorted values
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    if (tid == 0) *done = 0;  // re-armed for the next launch (stream-ordered)
    __threadfence();
    uint32_t ntop = 0;
    if (sortable) {
        for (uint32_t i = tid; i < m; i += blockDim.x) qs[i] = __ldcg(&qsorted[i]);
        __syncthreads();
        // distinct values, compacted in place: thread tid owns kDltPer consecutive slots
        // (held in registers across the barrier), a block scan gives its output offset
        constexpr uint32_t kDltPer = kDltSortMax / kDltQThreads;
        uint32_t v[kDltPer], fresh = 0, cnt = 0;
#pragma unroll
        for (uint32_t r = 0; r < kDltPer; r++) {
            const uint32_t i = tid * kDltPer + r;
            v[r] = i < m ? qs[i] : 0;
            if (i < m && (i == 0 || qs[i] != qs[i - 1])) {
                fresh |= 1u << r;
                cnt++;
            }
        }
        const uint32_t lane = tid & 31, wid = tid >> 5;
        uint32_t inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (lane == 31) s_wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = s_wsum[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= (uint32_t)o) wi += y;
            }
            s_wsum[lane] = wi - w;  // exclusive
            if (lane == 31) s_nd = wi;
        }
        __syncthreads();
        uint32_t off = s_wsum[wid] + inc - cnt;
#pragma unroll
        for (uint32_t r = 0; r < kDltPer; r++)
            if (fresh & (1u << r)) qs[off++] = v[r];
        __syncthreads();
        const uint32_t nd = s_nd;
        ntop = min(nd, (uint32_t)kDltQ);
        for (uint32_t jj = tid; jj < ntop; jj += blockDim.x)
            s_top[jj] = nd <= (uint32_t)kDltQ ? qs[jj] : qs[((uint64_t)(jj + 1) * nd) / kDltQ - 1];
    } else if (m > 0) {
        if (tid == 0) {
            s_qmin = 0xffffffffu;
            s_qmax = 0;
        }
        __syncthreads();
        uint32_t lo = 0xffffffffu, hi = 0;
        for (uint32_t i = tid; i < m; i += blockDim.x) {
            lo = min(lo, front[i].q);
            hi = max(hi, front[i].q);
        }
        atomicMin(&s_qmin, lo);
        atomicMax(&s_qmax, hi);
        __syncthreads();
        const uint64_t qmin = s_qmin, span = (uint64_t)s_qmax - s_qmin + 1;
        ntop = kDltQ;
        for (uint32_t jj = tid; jj < (uint32_t)kDltQ; jj += blockDim.x)
            s_top[jj] = (uint32_t)(qmin + ((uint64_t)(jj + 1) * span - 1) / kDltQ);
    }
    __syncthreads();
    for (uint32_t jj = tid; jj < (uint32_t)kDltQ; jj += blockDim.x) d->qtop[jj] = jj < ntop ? s_top[jj] : 0xffffffffu;
    const uint32_t qbase = ntop ? s_top[0] : 0;
    uint32_t qsh = 0;
    if (ntop)
        while (((uint64_t)(s_top[ntop - 1] - qbase) >> qsh) >= (uint64_t)kDltQMap) qsh++;
    if (tid == 0) {
        d->qbase = qbase;
        d->qmshift = qsh;
        d->ntop = ntop;
    }
    auto count_lt = [&](uint64_t L) -> uint32_t {  // #tops < L
        uint32_t a = 0, e = ntop;
        while (a < e) {
            const uint32_t mid = (a + e) >> 1;
            if ((uint64_t)s_top[mid] < L) a = mid + 1;
            else e = mid;
        }
        return a;
    };
    // the q map (cell 0 also takes q below qbase, the last cell everything above)
    for (uint32_t k = tid; k < (uint32_t)kDltQMap; k += blockDim.x) {
        const uint64_t L = k ? (uint64_t)qbase + ((uint64_t)k << qsh) : 0;
        const bool last = k == (uint32_t)kDltQMap - 1;
        const uint32_t lo = count_lt(L);
        const uint32_t hi = last ? ntop : count_lt((uint64_t)qbase + ((uint64_t)(k + 1) << qsh));
        d->qmap[k] = make_uint2(lo < ntop ? s_top[lo] : 0xffffffffu, lo | (hi << 8));
    }
}

// One launch builds the rest of the DLT: block j (256 threads) owns quality column j;
// thread r takes the front's t slice (te[r-1], te[r]] (the front is sorted by t: an index
// range, two binary searches), the min cost of its points with q >= qtop[j], and a block
// prefix-min over r turns slices into the cell's "t <= te[r]" minimum.  Every block also
// builds a 1/kDltQ share of the t map; block 0 writes the header, the t edges and the
// "none" row and column.  The quality tops come from dlt_qtop_kernel (launched before).
constexpr int kDltBuildThreads = 256;
static_assert(kDltT < kDltBuildThreads, "one thread per t bin");
__global__ void __launch_bounds__(kDltBuildThreads) dlt_build_kernel(const PPoint* __restrict__ front,
                                                                     ParetoCtl* __restrict__ ctl,
                                                                     Dlt* __restrict__ d) {
    __shared__ uint64_t te[kDltT];
    __shared__ unsigned long long s_cmax;
    __shared__ unsigned long long s_wmin[kDltBuildThreads / 32];
    const uint32_t m = (uint32_t)ctl->front_n;
    const uint32_t j = blockIdx.x, r = threadIdx.x, lane = r & 31, wid = r >> 5;
    if (r == 0) s_cmax = 0;
    for (uint32_t i = r; i < kDltT; i += blockDim.x) te[i] = m ? front[((uint64_t)i * m) / kDltT].t : kInf64;
    __syncthreads();
    uint64_t cmx = 0;
    for (uint32_t i = r; i < m; i += blockDim.x) cmx = umax64(cmx, front[i].c);
    cmx = umax64(cmx, __shfl_xor_sync(0xffffffffu, cmx, 16));
    cmx = umax64(cmx, __shfl_xor_sync(0xffffffffu, cmx, 8));
    cmx = umax64(cmx, __shfl_xor_sync(0xffffffffu, cmx, 4));
    cmx = umax64(cmx, __shfl_xor_sync(0xffffffffu, cmx, 2));
    cmx = umax64(cmx, __shfl_xor_sync(0xffffffffu, cmx, 1));
    if (lane == 0) atomicMax(&s_cmax, (unsigned long long)cmx);
    __syncthreads();
    uint32_t csh = 0;
    while ((s_cmax >> csh) >= 0xffffull) csh++;  // every front cost fits below the 0xffff "none"
    // map cell 0 sits just below the front's smallest t: it holds no edge
    const int32_t kbase = m ? dlt_tkey(front[0].t) - 1 : 0x7fffffff;
    if (j == 0) {
        if (r == 0) {
            d->kbase = kbase;
            d->cshift = csh;
            // the coming pass's counters (the previous pass's were consumed before this
            // launch): folded in here instead of two memset launches per pass
            ctl->surv = 0;
            ctl->dlt_n = 0;
        }
        for (uint32_t i = r; i < kDltT; i += blockDim.x) d->tedge[i] = te[i];
        for (uint32_t i = r; i <= (uint32_t)kDltT; i += blockDim.x) d->cell[i * kDltCols + kDltQ] = 0xffff;
    }
    if (r == 0) d->cell[j] = 0xffff;  // row 0: no front point has t <= the record's t
    // the t map, dealt over the grid: #edges <= lower end of cell k
    for (uint32_t k = j * blockDim.x + r; k < (uint32_t)kDltMap; k += gridDim.x * blockDim.x) {
        const int32_t key = kbase + (int32_t)k;
        auto lower_end = [&](int32_t kk) -> uint64_t {  // smallest integer t with key(t) >= kk
            return (kk >= (0x7f800000 >> kDltTShift)) ? kInf64 : (uint64_t)ceilf(__uint_as_float((uint32_t)kk << kDltTShift));
        };
        auto count_le = [&](uint64_t L) -> uint32_t {  // #edges <= L
            uint32_t a = 0, e = kDltT;
            while (a < e) {
                const uint32_t mid = (a + e) >> 1;
                if (te[mid] <= L) a = mid + 1;
                else e = mid;
            }
            return a;
        };
        const uint64_t L = lower_end(key), Lnext = lower_end(key + 1);
        // the last map cell also covers everything above it
        const uint64_t U = (k == (uint32_t)kDltMap - 1 || Lnext == kInf64) ? kInf64 : Lnext - 1;
        const uint32_t lo = m ? count_le(L) : 0, hi = m ? count_le(U) : 0;
        d->tmap[k] = (uint16_t)(lo | (hi << 8));
    }
    // slice of t bin r: front indices [#t <= te[r-1], #t <= te[r]).  te[r] is the t of
    // front point (r m) / kDltT, so #t <= te[r] is found by galloping forward from there
    // (a step or two; long runs of equal t take a doubling search)
    auto count_le_from = [&](uint32_t start) -> uint32_t {  // front[start].t = v; #t <= v
        const uint64_t v = __ldg(&front[start].t);
        uint32_t a = start + 1, b = a, step = 1;  // invariant: t[a - 1] <= v
        while (b < m && __ldg(&front[b].t) <= v) {
            a = b + 1;
            b = a + step;
            step <<= 1;
        }
        b = min(b, m);
        while (a < b) {  // t[a - 1] <= v < t[b] (or b = m)
            const uint32_t mid = (a + b) >> 1;
            if (__ldg(&front[mid].t) <= v) a = mid + 1;
            else b = mid;
        }
        return a;
    };
    const uint32_t ntop = d->ntop;
    const uint64_t qthr = j < ntop ? (uint64_t)d->qtop[j] : (1ull << 33);
    uint64_t best = kInf64;
    if (r < (uint32_t)kDltT && m && j < ntop) {
        const uint32_t i0 = r ? count_le_from((uint32_t)(((uint64_t)(r - 1) * m) / kDltT)) : 0;
        const uint32_t i1 = count_le_from((uint32_t)(((uint64_t)r * m) / kDltT));
        for (uint32_t i = i0; i < i1; i++)
            if ((uint64_t)__ldg(&front[i].q) >= qthr) best = umin64(best, __ldg(&front[i].c));
    }
    // inclusive prefix-min over the t bins (warp scan, then across the warps)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, best, o);
        if (lane >= (uint32_t)o) best = umin64(best, y);
    }
    if (lane == 31) s_wmin[wid] = best;
    __syncthreads();
    for (uint32_t w = 0; w < wid; w++) best = umin64(best, s_wmin[w]);
    // row r + 1 holds t bin r
    if (r < (uint32_t)kDltT)
        d->cell[(r + 1) * kDltCols + j] = best == kInf64 ? (uint16_t)0xffff : (uint16_t)(best >> csh);
}

// work = front[0, front_n) ++ surv[0, min(surv, cap)); m_in = its size.
__global__ void pareto_append_kernel(const PPoint* __restrict__ front, const PPoint* __restrict__ surv,
                                     uint64_t cap, PPoint* __restrict__ work, ParetoCtl* ctl) {
    const uint64_t fn = ctl->front_n;
    const unsigned long long sv = ctl->surv;
    const uint64_t ns = sv < cap ? sv : cap;
    const uint64_t tot = fn + ns;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (uint64_t)gridDim.x * blockDim.x)
        work[x] = x < fn ? front[x] : surv[x - fn];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->m_in = (uint32_t)tot;
        if (sv > cap) ctl->surv_overflow = 1;
    }
}

// Strided sample of a record segment -> points (seed for the first DLT).
__global__ void pareto_sample_kernel(SegView v, uint32_t ns, PPoint* __restrict__ out, ParetoCtl* ctl) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ns) return;
    const uint64_t per_tile = kTileRows * v.row;
    const uint64_t npos = v.ntiles * per_tile;
    const uint64_t pos = (uint64_t)((unsigned __int128)j * npos / ns);
    const uint64_t t = pos / per_tile;
    const uint32_t pin = (uint32_t)(pos - t * per_tile);
    const uint64_t idx = tiled_index(v.t0, v.row, t, pin);
    if (idx < v.ib || idx >= v.ie) return;
    const Rec4 r = ld_global_nc_256(v.recs + pos);
    PPoint p;
    p.idx = idx;
    p.t = r.w0 + r.w1;
    p.c = r.w2;
    p.q = rec_Q(r);
    p.pad = 0;
    out[atomicAdd(&ctl->m_in, 1u)] = p;
}

// Device-sized variant for the asynchronous cross-rank merge: fronts allgathered padded to
// `pad` points (counts allgathered alongside); each rank's first min(count, pad) points are
// concatenated into out, ctl->m_in = their total, *pad_over = 1 if some front exceeded pad
// (the host then redoes the merge at full size).
__global__ void front_gather_pad_kernel(const PPoint* __restrict__ padded, const uint64_t* __restrict__ counts,
                                        int nranks, uint32_t pad, PPoint* __restrict__ out, ParetoCtl* ctl,
                                        uint64_t* __restrict__ pad_over) {
    const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t r = x / pad, j = x % pad;
    if (x == 0) {
        uint64_t tot = 0, over = 0;
        for (int q = 0; q < nranks; q++) {
            tot += counts[q] < pad ? counts[q] : pad;
            over |= counts[q] > pad ? 1ull : 0ull;
        }
        ctl->m_in = (uint32_t)tot;
        *pad_over = over;
    }
    if ((int)r >= nranks) return;
    const uint64_t cr = counts[r] < pad ? counts[r] : pad;
    if (j >= cr) return;
    uint64_t off = 0;
    for (uint64_t q = 0; q < r; q++) off += counts[q] < pad ? counts[q] : pad;
    out[off + j] = padded[x];
}

// Gather variable-size per-rank fronts (allgathered, padded to maxc) into one array.
__global__ void pareto_gather_kernel(const PPoint* __restrict__ padded, const uint64_t* __restrict__ counts,
                                     int nranks, uint64_t maxc, PPoint* __restrict__ out) {
    const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t r = x / maxc, j = x % maxc;
    if ((int)r >= nranks || j >= counts[r]) return;
    uint64_t off = 0;
    for (uint64_t q = 0; q < r; q++) off += counts[q];
    out[off + j] = padded[x];
}


// Block-local front: each CTA reduces a chunk of kLocal points in shared memory and
// appends its non-dominated points.  front(A u B) = front(front(A) u front(B)), so a
// global mark over the (much smaller) union stays exact.
// BS = points per block: a first pass with small blocks spreads the O(BS^2) work of a
// large survivor set over many SMs; a second pass with large blocks shrinks the rest.
constexpr int kLocal = 1024;
constexpr int kLocalSmall = 256;
template <int BS>
__global__ void __launch_bounds__(BS) pareto_local_kernel(const PPoint* __restrict__ pts,
                                                          const uint32_t* __restrict__ d_m,
                                                          PPoint* __restrict__ out,
                                                          uint32_t* __restrict__ count,
                                                          uint8_t* __restrict__ keep_init) {
    __shared__ PPoint sp[BS];
    const uint32_t m = *d_m;
    const uint32_t base = blockIdx.x * BS;
    if (base >= m) return;
    const uint32_t cnt = min((uint32_t)BS, m - base);
    if (threadIdx.x < cnt) sp[threadIdx.x] = pts[base + threadIdx.x];
    __syncthreads();
    if (threadIdx.x >= cnt) return;
    const PPoint p = sp[threadIdx.x];
    for (uint32_t j = 0; j < cnt; j++)
        if (j != threadIdx.x && pdom(sp[j], base + j, p, base + threadIdx.x)) return;
    const uint32_t slot = atomicAdd(count, 1u);
    out[slot] = p;
    if (keep_init) keep_init[slot] = 1;
}

// keep[x] = 0 for every x of pts[0, m) dominated by another point.  The m x m dominance
// tests are cut into 256 x 256 tiles dealt to a persistent grid, so even a few thousand
// points spread over all SMs (keep[] must hold 1 for [0, m) on entry).
__global__ void __launch_bounds__(kScanThreads) pareto_mark2d_kernel(const PPoint* __restrict__ pts,
                                                                     const uint32_t* __restrict__ d_m,
                                                                     uint8_t* __restrict__ keep) {
    __shared__ PPoint tile[kScanThreads];
    const uint32_t m = *d_m;
    const uint32_t nb = (m + kScanThreads - 1) / kScanThreads;
    const uint64_t items = (uint64_t)nb * nb;
    for (uint64_t w = blockIdx.x; w < items; w += gridDim.x) {
        const uint32_t xb = (uint32_t)(w / nb), yb = (uint32_t)(w - (uint64_t)xb * nb);
        const uint32_t x = xb * kScanThreads + threadIdx.x;
        const uint32_t y0 = yb * kScanThreads;
        __syncthreads();
        if (y0 + threadIdx.x < m) tile[threadIdx.x] = pts[y0 + threadIdx.x];
        __syncthreads();
        if (x >= m || !keep[x]) continue;  // already known dominated: skip the work
        const PPoint px = pts[x];
        const uint32_t lim = min((uint32_t)kScanThreads, m - y0);
        for (uint32_t j = 0; j < lim; j++)
            if (y0 + j != x && pdom(tile[j], y0 + j, px, x)) {
                keep[x] = 0;
                break;
            }
    }
}

// a9 from the front (reading R30): a QUALITY_FIRST query that bounds neither startup nor
// stall has its winner -- feasible (cost <= budget) or closest (least budget overshoot)
// -- on the exact 3-D Pareto front, so it is reduced over the front points only.
__global__ void __launch_bounds__(kScanThreads) select_front_kernel(const PPoint* __restrict__ front, uint64_t n,
                                                                    const uint64_t* __restrict__ d_n, SelParams P,
                                                                    Cand* __restrict__ out) {
    __shared__ Cand s_tmp[32];
    if (d_n) n = *d_n;  // front size produced on the device by the preceding merge
    for (uint32_t q = 0; q < P.nq; q++) {
        uint64_t idx = kInf64;
        Rec4 r{};
        for (uint64_t j = threadIdx.x; j < n; j += blockDim.x) {
            const PPoint pt = front[j];
            Rec4 x;
            x.w0 = pt.t;  // ttff_eff as ttff with zero stall: unbounded in this query
            x.w1 = 0;
            x.w2 = pt.c;
            x.w3 = pt.q;
            if (cand_better(P.q[q], P.objective, pt.idx, x, idx, r)) {
                idx = pt.idx;
                r = x;
            }
        }
        block_reduce_cand(P.q[q], P.objective, idx, r, s_tmp);
        if (threadIdx.x == 0) {
            out[q].idx = idx;
            out[q].r = r;
            out[q].pad = (idx != kInf64 && !feasible(P.q[q], r)) ? 1ull : 0ull;
        }
        __syncthreads();
    }
}

// The whole exact merge work[0, ctl.m_in) -> sorted front in `out`, in ONE cooperative
// launch (a persistent grid of 1024-thread blocks, phases separated by grid-wide
// barriers): (0) a bucket sort of the input by ttff_eff into `sorted` (kRedBuckets
// buckets of the float key of t over its range: counts, one block's scan, scatter) -- a
// point's dominators mostly have about its t, so (1) the 256-point block-local fronts of
// t-sorted chunks keep ~4x fewer points than chunks in arrival order (measured on the C3
// merges: 30 K in -> 3.9 K vs 16.9 K kept), which cuts the quadratic mark ~19x; the order
// only affects speed, every phase is exact whatever it is; (1) local fronts into tmp2,
// (2) the m x m dominance mark in
// 256 x 256 tiles, (3) compaction into work, (4) rank sort into out; publishes front_n /
// front_overflow.  Every 256-point tile is worked by 4 threads per point (64 tests each,
// 8 independent tests per step): the phases are latency chains, not throughput, so the
// critical path is what counts.  Reads of data other blocks wrote in an earlier phase
// bypass L1 (__ldcg).
constexpr int kRedThreads = 1024;
constexpr int kRedParts = kRedThreads / kScanThreads;  // threads per point
constexpr uint32_t kRedSpan = kScanThreads / kRedParts;  // candidates per thread per tile

__device__ __forceinline__ PPoint ldcg_point(const PPoint* p) {
    PPoint x;
    x.idx = __ldcg(&p->idx);
    x.t = __ldcg(&p->t);
    x.c = __ldcg(&p->c);
    x.q = __ldcg(&p->q);
    x.pad = 0;
    return x;
}

// Does any of tile[j0, j0 + kRedSpan) (restricted to j < lim, position y0 + j != px)
// dominate x?  Branch-free groups of 8 tests.
__device__ __forceinline__ bool span_dominated(const PPoint* tile, uint32_t j0, uint32_t lim, uint32_t y0,
                                               const PPoint& x, uint32_t px) {
    bool dom = false;
    for (uint32_t g = 0; g < kRedSpan && !dom; g += 8) {
#pragma unroll
        for (uint32_t u = 0; u < 8; u++) {
            const uint32_t j = j0 + g + u;
            const bool ok = (j < lim) & (y0 + j != px);
            dom |= ok & pdom(tile[ok ? j : 0], y0 + j, x, px);
        }
    }
    return dom;
}

constexpr uint32_t kRedBuckets = 4096;
constexpr uint32_t kRedSortMin = 12288;
__device__ __forceinline__ uint32_t red_tkey(uint64_t t) { return __float_as_uint(__ull2float_rz(t)); }

__global__ void __launch_bounds__(kRedThreads, 1) pareto_reduce_kernel(PPoint* __restrict__ work,
                                                                       PPoint* __restrict__ tmp2,
                                                                       uint8_t* __restrict__ keep,
                                                                       PPoint* __restrict__ out, ParetoCtl* ctl,
                                                                       uint64_t cap, PPoint* __restrict__ sorted,
                                                                       uint32_t* __restrict__ hist) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ PPoint tile[kScanThreads];
    __shared__ uint8_t s_dom[kScanThreads];
    __shared__ uint32_t s_rank[kScanThreads];
    const uint32_t tid = threadIdx.x;
    const uint32_t pt = tid % kScanThreads, part = tid / kScanThreads;
    auto stamp = [&](int i) {
        if (blockIdx.x == 0 && tid == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            ctl->stamp[i] = t;
        }
    };
    stamp(0);
    if (blockIdx.x == 0) {
        if (tid == 0) {
            ctl->m_loc = 0;
            ctl->m_cmp = 0;
            ctl->rkmin = 0xffffffffu;
            ctl->rkmax = 0;
        }
        for (uint32_t i = tid; i < kRedBuckets; i += blockDim.x) hist[i] = 0;
    }
    grid.sync();
    const uint32_t m = __ldcg(&ctl->m_in);
    const uint32_t gsz = gridDim.x * blockDim.x, gid = blockIdx.x * blockDim.x + tid;
    // (0) bucket sort by t (inputs of >= kRedSortMin points; smaller ones are cheap to mark
    // as they come): key range, counts, scan (block 0), scatter.  m is grid-uniform.
    const bool do_sort = m >= kRedSortMin;
    if (do_sort) {
        uint32_t lo = 0xffffffffu, hi = 0;
        for (uint32_t x = gid; x < m; x += gsz) {
            const uint32_t k = red_tkey(work[x].t);
            lo = min(lo, k);
            hi = max(hi, k);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((tid & 31) == 0 && hi >= lo) {
            atomicMin(&ctl->rkmin, lo);
            atomicMax(&ctl->rkmax, hi);
        }
        grid.sync();
        const uint32_t kmin = __ldcg(&ctl->rkmin), kmax = __ldcg(&ctl->rkmax);
        uint32_t sh = 0;
        while (kmax > kmin && ((kmax - kmin) >> sh) >= kRedBuckets) sh++;
        for (uint32_t x = gid; x < m; x += gsz) atomicAdd(&hist[(red_tkey(work[x].t) - kmin) >> sh], 1u);
        grid.sync();
        if (blockIdx.x == 0) {  // exclusive scan of the counts, kRedBuckets / 1024 per thread
            constexpr uint32_t kPer = kRedBuckets / kRedThreads;
            uint32_t v[kPer], sum = 0;
#pragma unroll
            for (uint32_t r = 0; r < kPer; r++) {
                v[r] = __ldcg(&hist[tid * kPer + r]);
                sum += v[r];
            }
            uint32_t inc = sum;
            const uint32_t lane = tid & 31, wid = tid >> 5;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= (uint32_t)o) inc += y;
            }
            if (lane == 31) s_rank[wid] = inc;
            __syncthreads();
            if (wid == 0) {
                const uint32_t w = s_rank[lane];
                uint32_t wi = w;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= (uint32_t)o) wi += y;
                }
                s_rank[lane] = wi - w;
            }
            __syncthreads();
            uint32_t off = s_rank[wid] + inc - sum;
#pragma unroll
            for (uint32_t r = 0; r < kPer; r++) {
                hist[tid * kPer + r] = off;
                off += v[r];
            }
        }
        grid.sync();
        for (uint32_t x = gid; x < m; x += gsz) {
            const PPoint p = work[x];
            sorted[atomicAdd(&hist[(red_tkey(p.t) - kmin) >> sh], 1u)] = p;
        }
        grid.sync();
    }
    stamp(1);
    // (1) block-local fronts of 256-point chunks of the t-sorted input
    for (uint32_t base = blockIdx.x * kScanThreads; base < m; base += gridDim.x * kScanThreads) {
        const uint32_t cnt = min((uint32_t)kScanThreads, m - base);
        __syncthreads();
        if (part == 0) {
            if (pt < cnt) tile[pt] = ldcg_point(do_sort ? &sorted[base + pt] : &work[base + pt]);
            s_dom[pt] = 0;
        }
        __syncthreads();
        if (pt < cnt && span_dominated(tile, part * kRedSpan, cnt, base, tile[pt], base + pt)) s_dom[pt] = 1;
        __syncthreads();
        // the chunk's kept points: one global atomic per chunk (ballots + a block offset)
        // -- one per kept point serialised ~10 us on 30 K-point C3 merges
        if (part == 0) {
            const bool kp = pt < cnt && !s_dom[pt];
            const unsigned bal = __ballot_sync(0xffffffffu, kp);
            if ((tid & 31) == 0) s_rank[tid >> 5] = __popc(bal);  // per-warp counts (8 warps)
            __syncwarp();
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t acc = 0;
            for (uint32_t w = 0; w < kScanThreads / 32; w++) {
                const uint32_t c = s_rank[w];
                s_rank[w] = acc;
                acc += c;
            }
            s_rank[kScanThreads / 32] = acc ? atomicAdd(&ctl->m_loc, acc) : 0u;
        }
        __syncthreads();
        if (part == 0) {  // whole warps (tid < 256): the ballot sees every lane
            const bool kp = pt < cnt && !s_dom[pt];
            const unsigned bal = __ballot_sync(0xffffffffu, kp);
            if (kp) {
                const uint32_t slot =
                    s_rank[kScanThreads / 32] + s_rank[tid >> 5] + __popc(bal & ((1u << (tid & 31)) - 1u));
                tmp2[slot] = tile[pt];
                keep[slot] = 1;
            }
        }
    }
    grid.sync();
    stamp(2);
    const uint32_t ml = __ldcg(&ctl->m_loc);
    // (2) dominance mark over 256 x 256 tiles
    const uint32_t nb = (ml + kScanThreads - 1) / kScanThreads;
    const uint64_t items = (uint64_t)nb * nb;
    for (uint64_t w = blockIdx.x; w < items; w += gridDim.x) {
        const uint32_t xb = (uint32_t)(w / nb), yb = (uint32_t)(w - (uint64_t)xb * nb);
        const uint32_t x = xb * kScanThreads + pt, y0 = yb * kScanThreads;
        __syncthreads();
        if (part == 0 && y0 + pt < ml) tile[pt] = ldcg_point(&tmp2[y0 + pt]);
        __syncthreads();
        if (x >= ml || !__ldcg(&keep[x])) continue;
        const PPoint px = ldcg_point(&tmp2[x]);
        const uint32_t lim = min((uint32_t)kScanThreads, ml - y0);
        if (span_dominated(tile, part * kRedSpan, lim, y0, px, x)) keep[x] = 0;
    }
    grid.sync();
    stamp(3);
    // (3) compaction of the kept points into work
    for (uint32_t x0 = blockIdx.x * blockDim.x; x0 < ml; x0 += gridDim.x * blockDim.x) {  // one atomic per warp
        const uint32_t x = x0 + tid;
        const bool kp = x < ml && __ldcg(&keep[x]);
        const unsigned bal = __ballot_sync(0xffffffffu, kp);
        uint32_t wb = 0;
        if ((tid & 31) == 0 && bal) wb = atomicAdd(&ctl->m_cmp, (uint32_t)__popc(bal));
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if (kp) work[wb + __popc(bal & ((1u << (tid & 31)) - 1u))] = ldcg_point(&tmp2[x]);
    }
    grid.sync();
    stamp(4);
    const uint32_t mc = __ldcg(&ctl->m_cmp);
    if (blockIdx.x == 0 && tid == 0) {
        ctl->front_n = mc <= cap ? mc : 0;
        if (mc > cap) ctl->front_overflow = 1;
    }
    if (mc > cap) return;
    // (4) rank sort by (t asc, c asc, q desc, index asc) -- indices are unique (a bitonic
    // sort of the few hundred points in one block measured slower: ~45 barrier steps).
    // 64 points per block, 16 threads per point (each 1/16 of every 256-point tile), so a
    // front of m points keeps m / 64 blocks busy.
    constexpr uint32_t kRankPts = 64, kRankParts = kRedThreads / kRankPts;
    const uint32_t rp = tid % kRankPts, rpart = tid / kRankPts;
    for (uint32_t xb = blockIdx.x; xb * kRankPts < mc; xb += gridDim.x) {
        const uint32_t x = xb * kRankPts + rp;
        __syncthreads();
        if (tid < kRankPts) s_rank[tid] = 0;
        const PPoint px = x < mc ? ldcg_point(&work[x]) : PPoint{};
        uint32_t rank = 0;
        for (uint32_t base = 0; base < mc; base += kScanThreads) {
            __syncthreads();
            if (tid < kScanThreads && base + tid < mc) tile[tid] = ldcg_point(&work[base + tid]);
            __syncthreads();
            const uint32_t lim = min((uint32_t)kScanThreads, mc - base);
#pragma unroll 4
            for (uint32_t g = rpart; g < (uint32_t)kScanThreads; g += kRankParts)
                rank += ((g < lim) & pkey_less(tile[g < lim ? g : 0], px)) ? 1u : 0u;
        }
        atomicAdd(&s_rank[rp], rank);
        __syncthreads();
        if (tid < kRankPts && x < mc) out[s_rank[tid]] = px;
    }
    if (blockIdx.x == 0) stamp(5);  // block 0's own share of the rank sort done
}

// ============================================================================ fused scan
// One pass over a record segment serves (a9) up to NQ select queries and, when PARETO,
// (a8) the front filter: (1) the DLT prefilter, O(1) per record; (2) for DLT survivors
// an exact warp-cooperative dominance test against up to m_sm front points held in
// shared memory (32 per step, __any_sync early exit).  A record dominated by a real
// candidate cannot be on the front, so the survivors always contain every true front
// point of the segment whatever front subset is used: the later merge stays exact.
constexpr uint32_t kFrontSmem = 512;  // front points held in smem for the exact filter
constexpr uint32_t kBlockSurv = 256;  // this block's own survivors, kept in smem as a second filter

struct ParetoArgs {  // scan auxiliaries: Pareto filter state + grid-wide select flags
    const Dlt* dlt;
    const PPoint* front;
    ParetoCtl* ctl;  // front_n (read) and the DLT-survivor counter dlt_n (atomics)
    PPoint* surv;
    uint64_t cap;
    PPoint* cand;       // DLT survivors of the pass, exact-tested by pareto_exact_kernel
    uint64_t cand_cap;
    uint32_t* gfeas;  // [SW_MAX_QUERIES] per request: a feasible record was seen (or null)
    uint32_t debug;     // count DLT passes (SW_DEBUG)
};

// The deferred exact Pareto test of a scan pass (DLT survivors, appended by the scan).
// Every WARP walks its own contiguous run of the candidate buffer, 32 candidates at a time,
// with no block-wide barrier:
//  (1) each lane tests its candidate x against the 8 front points just below x.t (the
//      front is sorted by t; only points with t <= x.t can dominate x, and the dominator
//      the DLT missed is almost always just below x.t, in x's own t bin);
//  (2) the still undecided candidates (rare) are tested by the whole warp against the rest
//      of the front, 32 points per step, early exit on a hit;
//  (3) a candidate not dominated by the front is tested by the warp against the warp's own
//      earlier survivors (neighbouring records often dominate each other) and, if it
//      passes, joins that list at once; lists are flushed to surv (ctl->surv) when full and
//      at the end.  An identical entry (same index) also removes x: it is already kept.
// A survivor list only loosens a filter (a record dominated by a real candidate is never a
// front point), so the merge after the pass stays exact.  Dropped DLT survivors (candidate
// buffer full) set surv_overflow: the merged front is then valid but incomplete and the pass
// is refolded.  The front (<= kExactFront points) and the lists live in dynamic shared
// memory as arrays (t, c, idx, q), with a position map of the front's t (the float key of
// t, kDltMap cells of 1/128 octave: cell k -> [#front t below it, #front t up to its
// end]) so that x's position in the front is a map load plus a search of one cell's
// range (usually empty) instead of an 11-step binary search of dependent smem loads.
// 24 warps per block (one block per SM: the front copy is shared by all of them).
#ifndef SW_EXACT_FRONT
#define SW_EXACT_FRONT 4096  // C5 fronts (3021 points) in smem with their staircases: C5 182 -> 177 ms
#endif
#ifndef SW_EXACT_LIST
#define SW_EXACT_LIST 64  // (128 and 64 measured equal on C2/C3)
#endif
constexpr uint32_t kExactFront = SW_EXACT_FRONT;  // front points staged in smem (larger fronts: from L2)
constexpr uint32_t kExactList = SW_EXACT_LIST;    // per-warp survivor list
constexpr int kExactThreads = 768;
constexpr int kExactWarps = kExactThreads / 32;
#ifndef SW_EXACT_NEAR
#define SW_EXACT_NEAR 24  // 8..48 measured with the staircases: 24 best (C3 exact tests 0.40 -> 0.28 ms)
#endif
constexpr uint32_t kExactNear = SW_EXACT_NEAR;  // front points below x.t tested per lane first
__host__ __device__ constexpr size_t exact_smem_bytes() {
    return (size_t)(kExactFront + kExactWarps * kExactList) * (3 * sizeof(uint64_t) + sizeof(uint32_t)) +
           (size_t)kDltMap * sizeof(uint32_t) + (size_t)kExactFront * (sizeof(uint32_t) + sizeof(uint64_t));
}
struct PArrays {  // a point list as arrays in shared memory
    uint64_t *t, *c, *i;
    uint32_t* q;
    __device__ __forceinline__ PPoint get(uint32_t j) const {
        PPoint y;
        y.t = t[j];
        y.c = c[j];
        y.idx = i[j];
        y.q = q[j];
        y.pad = 0;
        return y;
    }
    __device__ __forceinline__ void put(uint32_t j, const PPoint& x) const {
        t[j] = x.t;
        c[j] = x.c;
        i[j] = x.idx;
        q[j] = x.q;
    }
};
__device__ __forceinline__ PArrays parrays(unsigned char* base, uint32_t n) {
    PArrays a;
    a.t = reinterpret_cast<uint64_t*>(base);
    a.c = a.t + n;
    a.i = a.c + n;
    a.q = reinterpret_cast<uint32_t*>(a.i + n);
    return a;
}

__global__ void __launch_bounds__(kExactThreads, 1) pareto_exact_kernel(const PPoint* __restrict__ cand, uint64_t cand_cap,
                                                                        const PPoint* __restrict__ front, ParetoCtl* ctl,
                                                                        PPoint* __restrict__ surv, uint64_t surv_cap) {
    extern __shared__ __align__(16) unsigned char xsm[];
    const PArrays F = parrays(xsm, kExactFront);
    const unsigned long long nd = ctl->dlt_n;
    const uint64_t n = nd < cand_cap ? nd : cand_cap;
    const uint32_t m = (uint32_t)ctl->front_n;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (nd > cand_cap) ctl->surv_overflow = 1;
        atomicMax(&ctl->dlt_max, nd);
    }
    const uint64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
    if (r0 >= r1) return;
    const bool f_smem = m <= kExactFront;
    uint32_t* pmap = reinterpret_cast<uint32_t*>(xsm + (size_t)(kExactFront + kExactWarps * kExactList) * 28);
    const int32_t pkbase = m ? dlt_tkey(front[0].t) : 0;  // cell 0 holds the smallest front t
    if (f_smem) {
        for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) F.put(j, front[j]);
        __syncthreads();
        auto count_le = [&](uint64_t v) {  // #front points with t <= v
            uint32_t a = 0, e = m;
            while (a < e) {
                const uint32_t mid = (a + e) >> 1;
                if (F.t[mid] <= v) a = mid + 1;
                else e = mid;
            }
            return a;
        };
        for (uint32_t k = threadIdx.x; k < (uint32_t)kDltMap; k += blockDim.x) {
            // cell k: keys pkbase + k (the last cell: everything above); lo = #t below the
            // cell's lower end L, hi = #t <= its upper end
            const int32_t key = pkbase + (int32_t)k;
            auto lower_end = [&](int32_t kk) -> uint64_t {  // smallest integer t with key(t) >= kk
                return (kk >= (0x7f800000 >> kDltTShift)) ? kInf64
                                                          : (uint64_t)ceilf(__uint_as_float((uint32_t)kk << kDltTShift));
            };
            const uint64_t L = lower_end(key), Ln = lower_end(key + 1);
            const uint32_t lo = (k == 0 || L == 0) ? 0 : count_le(L - 1);
            const uint32_t hi = (k == (uint32_t)kDltMap - 1 || Ln == kInf64) ? m : count_le(Ln - 1);
            pmap[k] = lo | (hi << 16);
        }
    }
    // per 32-point block of the t-sorted front: its qualities sorted descending (sq) and the
    // running min cost over them (sc) -- "is any point of this block >= q and < c?" is then
    // one binary search, so a candidate the nearest points leave undecided is settled by
    // one lookup per block (a lane each) instead of a scan of the whole front below it
    uint32_t* sq = pmap + kDltMap;
    uint64_t* sc = reinterpret_cast<uint64_t*>(sq + kExactFront);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (f_smem) {
        __syncthreads();  // F staged
        for (uint32_t kb = warp; kb * 32 < m; kb += kExactWarps) {
            const uint32_t p = kb * 32 + lane;
            const uint32_t q = p < m ? F.q[p] : 0u;
            const uint64_t c = p < m ? F.c[p] : kInf64;
            uint32_t r = 0;  // rank: higher q first, ties by lane
            for (uint32_t o = 0; o < 32; o++) {
                const uint32_t oq = __shfl_sync(0xffffffffu, q, o);
                r += (oq > q || (oq == q && o < lane)) ? 1u : 0u;
            }
            sq[kb * 32 + r] = q;
            sc[kb * 32 + r] = c;
            __syncwarp();
            uint64_t mn = sc[kb * 32 + lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, mn, o);
                if (lane >= (uint32_t)o) mn = umin64(mn, y);
            }
            sc[kb * 32 + lane] = mn;
            __syncwarp();
        }
    }
    __syncthreads();
    const PArrays L = parrays(xsm + (size_t)kExactFront * 28 + (size_t)warp * kExactList * 28, kExactList);
    auto fget = [&](uint32_t j) { return f_smem ? F.get(j) : front[j]; };
    // this warp's run of the block's range
    const uint64_t w0 = r0 + (r1 - r0) * warp / kExactWarps, w1 = r0 + (r1 - r0) * (warp + 1) / kExactWarps;
    uint32_t nl = 0;  // warp-uniform list fill
    auto flush = [&]() {
        unsigned long long b = 0;
        if (lane == 0 && nl) b = atomicAdd(&ctl->surv, (unsigned long long)nl);
        b = __shfl_sync(0xffffffffu, b, 0);
        for (uint32_t j = lane; j < nl; j += 32)
            if (b + j < surv_cap) surv[b + j] = L.get(j);
        __syncwarp();
        nl = 0;
    };
    for (uint64_t base = w0; base < w1; base += 32) {
        const uint64_t i = base + lane;
        const bool valid = i < w1;
        PPoint x{};
        uint32_t lo = 0;
        bool dom = !valid;
        if (valid) {
            x = cand[i];
            uint32_t hi = m;  // lo = #front points with t <= x.t
            if (f_smem) {  // narrowed by the position map (t below the front's smallest: lo = 0)
                const int32_t k = dlt_tkey(x.t) - pkbase;
                const uint32_t pm = pmap[min(max(k, 0), kDltMap - 1)];
                lo = k < 0 ? 0 : pm & 0xffffu;
                hi = k < 0 ? 0 : pm >> 16;
            }
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((f_smem ? F.t[mid] : front[mid].t) <= x.t) lo = mid + 1;
                else hi = mid;
            }
            // (1) the nearest points below x.t, 4 independent tests per step
            const uint32_t stop = lo > kExactNear ? lo - kExactNear : 0;
            uint32_t j = lo;
            for (; j >= stop + 4 && !dom; j -= 4)
                dom = pdom(fget(j - 1), 0, x, 1) | pdom(fget(j - 2), 0, x, 1) | pdom(fget(j - 3), 0, x, 1) |
                      pdom(fget(j - 4), 0, x, 1);
            for (; j > stop && !dom; j--) dom = pdom(fget(j - 1), 0, x, 1);
        }
        const uint32_t top = lo > kExactNear ? lo - kExactNear : 0;  // still to test: [0, top)
        // (2) undecided candidates (rare): the whole warp against the rest of the front
        unsigned hard = __ballot_sync(0xffffffffu, !dom && top > 0);
        while (hard) {
            const int src = __ffs(hard) - 1;
            hard &= hard - 1;
            PPoint y;
            y.t = __shfl_sync(0xffffffffu, x.t, src);
            y.c = __shfl_sync(0xffffffffu, x.c, src);
            y.idx = __shfl_sync(0xffffffffu, x.idx, src);
            y.q = __shfl_sync(0xffffffffu, x.q, src);
            y.pad = 0;
            const uint32_t ytop = __shfl_sync(0xffffffffu, top, src);
            const uint32_t kfull = f_smem ? ytop >> 5 : 0;  // whole blocks below ytop: by summary
            bool d;
            {  // the rest above them: direct tests, a lane each
                const uint32_t j = (kfull << 5) + lane;
                d = __any_sync(0xffffffffu, j < ytop && pdom(fget(j < ytop ? j : 0), 0, y, 1));
            }
            if (!d && kfull) {
                bool hit = false, unsure = false;
                for (uint32_t kb = lane; kb < kfull; kb += 32) {
                    const uint32_t* qa = sq + kb * 32;  // descending
                    uint32_t a = 0;                     // #points of block kb with q >= y.q
#pragma unroll
                    for (uint32_t st = 16; st > 0; st >>= 1) a += qa[a + st - 1] >= y.q ? st : 0u;
                    a += qa[a] >= y.q ? 1u : 0u;  // a <= 31 here: the last element
                    if (a) {
                        const uint64_t mc = sc[kb * 32 + a - 1];
                        hit |= mc < y.c;      // t <= y.t, q >= y.q, c < y.c: dominates
                        unsure |= mc == y.c;  // equal cost: strictness decided point by point
                    }
                }
                d = __any_sync(0xffffffffu, hit);
                if (!d && __any_sync(0xffffffffu, unsure))
                    for (uint32_t j1 = kfull << 5; j1 > 0 && !d;) {  // rare: the exact scan
                        const uint32_t j0 = j1 - 32, j = j0 + lane;
                        d = __any_sync(0xffffffffu, pdom(fget(j), 0, y, 1));
                        j1 = j0;
                    }
            }
            if (!f_smem)  // front beyond smem: the downward scan from L2
                for (uint32_t j1 = ytop; j1 > 0 && !d;) {
                    const uint32_t j0 = j1 > 32 ? j1 - 32 : 0;
                    const uint32_t j = j0 + lane;
                    d = __any_sync(0xffffffffu, j < j1 && pdom(fget(j < j1 ? j : 0), 0, y, 1));
                    j1 = j0;
                }
            if (lane == src) dom = d;
        }
        // (3) front survivors: against the warp's earlier survivors, then join the list
        unsigned keep = __ballot_sync(0xffffffffu, !dom);
        while (keep) {
            const int src = __ffs(keep) - 1;
            keep &= keep - 1;
            PPoint y;
            y.t = __shfl_sync(0xffffffffu, x.t, src);
            y.c = __shfl_sync(0xffffffffu, x.c, src);
            y.idx = __shfl_sync(0xffffffffu, x.idx, src);
            y.q = __shfl_sync(0xffffffffu, x.q, src);
            y.pad = 0;
            bool d = false;
            for (uint32_t j0 = 0; j0 < nl && !d; j0 += 32) {
                const uint32_t j = j0 + lane;
                d = __any_sync(0xffffffffu, j < nl && pdom(L.get(j), 0, y, 1));
            }
            if (d) continue;
            if (nl == kExactList) flush();
            if (lane == 0) L.put(nl, y);
            __syncwarp();
            nl++;
        }
    }
    flush();
}// objective keys only (ties keep the earlier = lower index within a thread's scan)
__device__ __forceinline__ bool obj_strict_better(uint32_t obj, const Rec4& a, const Rec4& b) {
    const uint32_t qa = rec_Q(a), qb = rec_Q(b);
    if (obj == 0) {
        if (qa != qb) return qa > qb;
        if (a.w2 != b.w2) return a.w2 < b.w2;
        return a.w0 + a.w1 < b.w0 + b.w1;
    }
    const uint64_t ta = a.w0 + a.w1, tb = b.w0 + b.w1;
    const uint64_t hi_a = __umul64hi(a.w2, ta), hi_b = __umul64hi(b.w2, tb);
    if (hi_a != hi_b) return hi_a < hi_b;
    const uint64_t lo_a = a.w2 * ta, lo_b = b.w2 * tb;
    if (lo_a != lo_b) return lo_a < lo_b;
    return qa > qb;
}

__device__ __forceinline__ bool closest_strict_better(const QueryDev& q, uint32_t obj, const Rec4& a,
                                                      const Rec4& b) {
    const uint64_t vta = sat_sub(a.w0, q.slo_t) + sat_sub(a.w1, q.slo_s);
    const uint64_t vtb = sat_sub(b.w0, q.slo_t) + sat_sub(b.w1, q.slo_s);
    if (vta != vtb) return vta < vtb;
    const uint64_t vca = sat_sub(a.w2, q.budget), vcb = sat_sub(b.w2, q.budget);
    if (vca != vcb) return vca < vcb;
    return obj_strict_better(obj, a, b);
}

// TMA-pipelined scan: the segment's records (a flat run of ntiles * 32 * row slots, tile
// padding included) are dealt to the WARPS of the grid in 4 KB stages (128 records),
// round-robin (warp w of block b takes stages b * kCW + w + i * gridDim.x * kCW).  Every
// warp owns its own ring slots and full mbarriers: its lane 0 issues the cp.async.bulk
// of the warp's next stage the moment the warp has moved the current one into registers.
// No producer warp, no empty barriers, and no coupling between warps -- a warp that
// spends longer on a stage (select candidates, exact Pareto tests) delays only its own
// stream (measured: group-owned 32 KB stages, refilled after the group's slowest warp,
// left fast warps spinning on their next stage).  kRPT records per thread per stage
// (independent chains: ILP).
//
// Select (a9) per record and query costs a few integer ops in the common case: the block
// shares, per query, a threshold in shared memory -- the best quality of any FEASIBLE
// record seen (QUALITY_FIRST) or a "feasible seen" flag (COST_X_TTFF).  A record of lower
// quality (resp. an infeasible record once a feasible one exists) is strictly worse than
// a record this block will report, so it is skipped; the full total-order comparison
// (cand_better) runs only for the rare records that pass.
constexpr int kCW = 16;                         // warps per block (4 per SMSP, up to 128 registers)
constexpr int kScanBlock = kCW * 32;
constexpr int kRPT = 4;                         // records per thread per stage
constexpr uint32_t kStageRecs = 32 * kRPT;      // one warp's stage: 128 records (4 KB)
constexpr uint32_t kUnitAlign = 1024;           // strided fold units: multiples of this many records
constexpr int kWarpSlots = 3;        // plain scans: 16 warps x 3 x 4 KB = 192 KB ring
constexpr int kWarpSlotsPareto = 2;  // scans carrying the DLT + front subset in smem: 128 KB
static_assert(kUnitAlign % kStageRecs == 0, "units are whole stages");
__host__ __device__ constexpr size_t ring_bytes(bool pareto) {
    return (size_t)kCW * (pareto ? kWarpSlotsPareto : kWarpSlots) * kStageRecs * sizeof(Rec4);
}

struct __align__(16) StageMeta {
    uint32_t gf[SW_MAX_QUERIES];  // grid-wide "feasible seen" flags, copied by the stage's TMA
    // ... and right behind them the grid-wide closest-tier keys, complemented (~key of the
    // best closest-tier record any block has seen; 0 = none): a block's own closest bound
    // starts at ~0 and tightens slowly where a query is infeasible in its shard, the grid's
    // is known after a few stages
    unsigned long long gneg[SW_MAX_QUERIES];
    uint64_t pos0;       // flat slot of the stage's first record
    uint32_t cnt;        // records in the stage; 0 = end of stream
    uint16_t all_valid;  // no tile padding inside: skip per-record range checks
    uint16_t pad;
};
static_assert(sizeof(uint32_t) * SW_MAX_QUERIES % 16 == 0, "flags are bulk-copied");
// global layout per request (pa.gfeas): gf[SW_MAX_QUERIES] u32 then gneg[SW_MAX_QUERIES] u64
constexpr uint32_t kGSelWords = SW_MAX_QUERIES + 2 * SW_MAX_QUERIES;
static_assert(offsetof(StageMeta, gneg) == sizeof(uint32_t) * SW_MAX_QUERIES, "gf and gneg are one bulk copy");

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Global index of flat slot P of a segment view (division only on rare paths).
__device__ __forceinline__ uint64_t flat_index(const SegView& v, uint32_t per_tile, uint64_t P) {
    const uint64_t t = P / per_tile;
    return tiled_index(v.t0, v.row, t, (uint32_t)(P - t * per_tile));
}

// QUALITY_FIRST prefilter key: higher is better in (-Q, cost) order up to the cost clamp.
__device__ __forceinline__ uint64_t qc_key(const Rec4& r) {
    const uint32_t c32 = r.w2 > 0xffffffffull ? 0xffffffffu : (uint32_t)r.w2;
    return ((uint64_t)rec_Q(r) << 32) | (uint64_t)(~c32);
}

// COST_X_TTFF prefilter key: ~min(cost x ttff_eff, 2^64 - 1) -- higher is better; a
// record whose key is below the best feasible record's has a strictly larger product.
__device__ __forceinline__ uint64_t cxt_key(const Rec4& r) {
    const uint64_t t = r.w0 + r.w1;
    return __umul64hi(r.w2, t) ? 0ull : ~(r.w2 * t);
}
// The objective's prefilter key (OBJ 0 / 1 compile-time, -1: runtime obj_q -- fleets).
template <int OBJ>
__device__ __forceinline__ uint64_t obj_key(bool obj_q, const Rec4& r) {
    if (OBJ == 0) return qc_key(r);
    if (OBJ == 1) return cxt_key(r);
    return obj_q ? qc_key(r) : cxt_key(r);
}

// Closest-tier prefilter key (lower is better): saturated (V_t, V_c) packed in 64 bits.
__device__ __forceinline__ uint64_t closest_pack(const Rec4& r, uint64_t slo_t, uint64_t slo_s, uint64_t bud) {
    const uint64_t vt = sat_sub(r.w0, slo_t) + sat_sub(r.w1, slo_s);
    const uint64_t vc = sat_sub(r.w2, bud);
    return (umin64(vt, 0xffffffffull) << 32) | umin64(vc, 0xffffffffull);
}

// Select predicate of kRPT records for one query: bit u set iff record u is valid,
// feasible (only the bounds in AM are compared) and its objective prefilter key (packed
// (Q, ~cost) under QUALITY_FIRST, ~sat(cost x ttff_eff) under COST_X_TTFF) is >= the
// block's best feasible key thr (thr == 0: none yet, every key passes).  Ties pass: they
// are settled by the full total order.
template <int AM, int OBJ>
__device__ __forceinline__ uint32_t pred_pass(const Rec4 (&r)[kRPT], const bool (&valid)[kRPT],
                                              unsigned long long thr, bool obj_q,
                                              uint64_t slo_t, uint64_t slo_s, uint64_t bud) {
    uint32_t need = 0;
#pragma unroll
    for (int u = 0; u < kRPT; u++) {
        bool f = valid[u];
        if (AM & 1) f &= r[u].w0 <= slo_t;
        if (AM & 2) f &= r[u].w1 <= slo_s;
        if (AM & 4) f &= r[u].w2 <= bud;
        f &= obj_key<OBJ>(obj_q, r[u]) >= thr;
        need |= (uint32_t)f << u;
    }
    return need;
}

// A fleet scan: request blockIdx.y scans its own records with its own queries.
struct ScanJob {
    SegView v;
    SelParams P;
};

// OBJ: the handle's objective at compile time (0 QUALITY_FIRST, 1 COST_X_TTFF) or -1 =
// per request at run time (fleet scans, whose requests may differ).
template <int NQ, bool PARETO, int OBJ>
__global__ void __launch_bounds__(kScanBlock, 1) scan_kernel(SegView v, SelParams P, Cand* __restrict__ partial,
                                                             ParetoArgs pa, const ScanJob* __restrict__ jobs) {
    if (jobs) {  // fleet: request y (never with PARETO)
        v = jobs[blockIdx.y].v;
        P = jobs[blockIdx.y].P;
        if (pa.gfeas) pa.gfeas += (uint64_t)blockIdx.y * kGSelWords;
    }
    const uint64_t out_block = (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
    constexpr int NQA = NQ > 0 ? NQ : 1;
    uint32_t amask[NQA];  // per query: bit 0 ttff bound set, bit 1 stall bound, bit 2 budget
#pragma unroll
    for (int q = 0; q < NQA; q++)
        amask[q] = NQ == 0 ? 0u
                           : (P.q[q].slo_t != kInf64 ? 1u : 0u) | (P.q[q].slo_s != kInf64 ? 2u : 0u) |
                                 (P.q[q].budget != kInf64 ? 4u : 0u);
    extern __shared__ __align__(128) unsigned char fsm[];
    __shared__ Cand s_tmp[32];
    constexpr int WS = PARETO ? kWarpSlotsPareto : kWarpSlots;  // ring slots per warp
    constexpr int NS = kCW * WS;
    __shared__ __align__(8) uint64_t full_bar[NS];
    __shared__ StageMeta meta[NS];
    // per query: the objective prefilter key (obj_key) of this block's best FEASIBLE
    // record: Q << 32 | ~min(cost, 2^32-1) (QUALITY_FIRST) or ~sat(cost x ttff_eff)
    // (COST_X_TTFF); 0 = none yet
    __shared__ unsigned long long s_thr[NQA];
    // per query, while no feasible record is known: the smallest closest-tier key
    // (min(V_t, 2^32-1) << 32 | min(V_c, 2^32-1), V_t the startup+stall violation and V_c the
    // budget violation -- the closest tier's order) of any best in this block; a record
    // with a larger key cannot win.  (V_t alone let every record of a shard through where
    // a query is infeasible and many records tie on V_t: C3's last quarter at 4 ranks
    // scanned at half speed.)
    __shared__ unsigned long long s_vt[NQA];
    Rec4* ring = reinterpret_cast<Rec4*>(fsm);
    Dlt& d = *reinterpret_cast<Dlt*>(fsm + ring_bytes(PARETO));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int st = 0; st < NS; st++) mbar_init(&full_bar[st], 1);
    }
    if (threadIdx.x < NQA) {
        s_thr[threadIdx.x] = 0;
        s_vt[threadIdx.x] = ~0ull;
    }
    if (PARETO) {  // stage the whole DLT (16 B vectors)
        const uint4* src = reinterpret_cast<const uint4*>(pa.dlt);
        uint4* dst = reinterpret_cast<uint4*>(&d);
        for (uint32_t i = threadIdx.x; i < sizeof(Dlt) / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    DltHot dh{0, 0, 0, 0};
    if (PARETO) dh = DltHot{d.kbase, d.qbase, d.qmshift, d.cshift};
    const uint32_t per_tile = (uint32_t)(kTileRows * v.row);
    const uint64_t total = v.ntiles * per_tile;
    // stage sg of this view/pass -> flat slot of its first record (kInf64: none)
    const uint64_t unit_recs = (uint64_t)v.upt * per_tile;
    const uint64_t spu = v.pass ? unit_recs / kStageRecs : 1;
    const uint64_t nunits = v.pass ? (total + unit_recs - 1) / unit_recs : 0;
    // level of this pass: 0 = multiples of 8^K; l >= 1 = multiples of 8^(K-l), not of 8^(K-l+1)
    const uint32_t lvl = v.pass ? v.pass - 1 : 0;
    const uint32_t sh = v.pass ? 3 * (v.levels - lvl) : 0;  // log2 of the unit stride
    const uint64_t c_here = v.pass ? (nunits + (1ull << sh) - 1) >> sh : 0;
    const uint64_t c_up = (v.pass && lvl > 0) ? (nunits + (1ull << (sh + 3)) - 1) >> (sh + 3) : 0;
    const uint64_t units_here = c_here - c_up;
    const uint64_t j_end = v.j1 < units_here ? v.j1 : units_here;
    const uint64_t nstages = v.pass == 0 ? (total + kStageRecs - 1) / kStageRecs
                                         : (j_end > v.j0 ? spu * (j_end - v.j0) : 0);
    // stage sg -> flat slot of its first record: with sg = j * spu + part (pass 0: spu = 1),
    // pos = (m << sh) * unit_recs + part * kStageRecs, m = the j-th unit of this pass
    // (pass 0: sh = 0 and unit_recs = kStageRecs, so pos = sg * kStageRecs)
    const uint64_t unit_pos = v.pass ? unit_recs : kStageRecs;
    const uint32_t spu32 = (uint32_t)spu;
    auto stage_pos = [&](uint32_t jl, uint32_t part) -> uint64_t {
        const uint32_t j = jl + (v.pass ? v.j0 : 0u);  // the pass's j-th unit
        const uint64_t m = lvl == 0 ? (uint64_t)j : (uint64_t)(j / 7) * 8 + (j % 7) + 1;  // j-th non-multiple of 8
        const uint64_t pos = (m << sh) * unit_pos + part * kStageRecs;
        return pos < total ? pos : kInf64;
    };
    // one running best per query under the query's total order (feasible first)
    uint64_t bi[NQA];
    Rec4 br[NQA];
    bool bf[NQA];
#pragma unroll
    for (int q = 0; q < NQA; q++) {
        bi[q] = kInf64;
        br[q] = Rec4{};
        bf[q] = false;
    }

    // ---------------- this warp's pipeline: slots warp*WS .. warp*WS+WS-1
    // Iteration k of the warp consumes global stage sg = gw + k * (gridDim.x * kCW) from
    // slot warp*WS + k % WS; lane 0 refills the slot with iteration k + WS as soon as the
    // warp holds the stage in registers.
    // lane 0 walks the warp's stages in order (one issue per iteration): a cursor sg =
    // c_j * spu + c_part advanced by nw per issue -- no divisions on the stream
    const uint32_t gw = blockIdx.x * kCW + warp, nw = gridDim.x * kCW;
    const uint32_t dj = nw / spu32, dp = nw - dj * spu32;
    uint64_t c_sg = gw;
    uint32_t c_j = gw / spu32, c_part = gw - c_j * spu32;
    auto issue = [&](uint32_t slot) {  // lane 0: fill slot with the warp's next stage
        const uint64_t sg = c_sg;
        const uint32_t j = c_j, part = c_part;
        c_sg += nw;
        c_j += dj;
        c_part += dp;
        if (c_part >= spu32) {
            c_part -= spu32;
            c_j++;
        }
        if (sg >= nstages) {  // end of this warp's stream
            meta[slot].pos0 = 0;
            meta[slot].cnt = 0;
            mbar_arrive(&full_bar[slot]);
            return;
        }
        const uint64_t pos0 = stage_pos(j, part);
        if (pos0 == kInf64) {  // a stage past a partial last unit: nothing to read
            meta[slot].pos0 = kInf64;
            meta[slot].cnt = 0;
            mbar_arrive(&full_bar[slot]);
            return;
        }
        const uint32_t cnt = (uint32_t)umin64(kStageRecs, total - pos0);
        // tile padding lives only in the first and the last tile of a segment
        const bool edge = pos0 < per_tile || pos0 + cnt > total - per_tile;
        meta[slot].pos0 = pos0;
        meta[slot].cnt = cnt;
        meta[slot].all_valid = (edge || cnt != kStageRecs) ? 0 : 1;  // a full stage, no padding
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA write
        // the grid-wide feasibility flags ride on the stage's own transaction: no thread
        // waits on a global load
        const uint32_t gf_bytes =
            (NQ > 0 && pa.gfeas) ? (uint32_t)(sizeof(meta[slot].gf) + sizeof(meta[slot].gneg)) : 0u;
        mbar_expect_tx(&full_bar[slot], cnt * (uint32_t)sizeof(Rec4) + gf_bytes);
        if (gf_bytes) tma_bulk_g2s(meta[slot].gf, pa.gfeas, gf_bytes, &full_bar[slot]);
        tma_bulk_g2s(ring + (size_t)slot * kStageRecs, v.recs + pos0, cnt * (uint32_t)sizeof(Rec4), &full_bar[slot]);
    };
    if (lane == 0)
        for (int j = 0; j < WS; j++) issue(warp * WS + j);
    {
        // ---------------- consume
        for (uint32_t k = 0;; k++) {
            const uint32_t st = warp * WS + k % WS;
            mbar_wait(&full_bar[st], (k / WS) & 1);
            const StageMeta mt = meta[st];
            if (mt.cnt == 0 && mt.pos0 == 0) break;  // end of the warp's stream
            if (mt.cnt == 0) {                        // empty stage: refill and go on
                __syncwarp();
                if (lane == 0) issue(st);
                continue;
            }
            Rec4 r[kRPT];
            bool valid[kRPT];
            if (mt.all_valid) {  // a full stage without tile padding (warp-uniform)
#pragma unroll
                for (int u = 0; u < kRPT; u++) {
                    valid[u] = true;
                    r[u] = ring[(size_t)st * kStageRecs + lane + u * 32];
                }
            } else {
#pragma unroll
                for (int u = 0; u < kRPT; u++) {
                    const uint32_t o = lane + u * 32;
                    valid[u] = o < mt.cnt;
                    if (valid[u]) {
                        const uint64_t i0 = flat_index(v, per_tile, mt.pos0 + o);
                        valid[u] = i0 >= v.ib && i0 < v.ie;
                    }
                    // unconditional: a slot past cnt holds stale bytes that valid[] masks out
                    r[u] = ring[(size_t)st * kStageRecs + o];
                }
            }
            // the warp has the stage in registers: lane 0 refills the slot
            __syncwarp();
            if (lane == 0) issue(st);
            const bool obj_q = OBJ >= 0 ? OBJ == 0 : P.objective == 0;
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                // predicate pass (branch-free, bitwise): which records can still beat this
                // block's best for query q?  The full comparison runs only for those.
                //  - once a feasible record is known (this thread, this block or -- via
                //    the stage meta -- any block) only feasible records can win, and under
                //    QUALITY_FIRST only those at least as good in (Q desc, cost asc) as
                //    the block's best feasible key;
                //  - before that, only records whose startup+stall violation does not
                //    exceed the block's best closest-tier violation.
                const unsigned long long thr = s_thr[q];
                const bool anyf = (thr != 0) | bf[q] | (pa.gfeas != nullptr && mt.gf[q] != 0);
                const uint64_t slo_t = P.q[q].slo_t, slo_s = P.q[q].slo_s, bud = P.q[q].budget;
                // only the bounds the query actually sets are compared (uniform dispatch)
                uint32_t need;
                switch (amask[q]) {
                    case 0: need = pred_pass<0, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 1: need = pred_pass<1, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 2: need = pred_pass<2, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 3: need = pred_pass<3, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 4: need = pred_pass<4, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 5: need = pred_pass<5, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    case 6: need = pred_pass<6, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                    default: need = pred_pass<7, OBJ>(r, valid, thr, obj_q, slo_t, slo_s, bud); break;
                }
                if (__any_sync(0xffffffffu, !anyf)) {  // closest tier still open somewhere
                    const unsigned long long gv = pa.gfeas ? ~mt.gneg[q] : ~0ull;
                    const unsigned long long vmax = s_vt[q] < gv ? s_vt[q] : gv;
#pragma unroll
                    for (int u = 0; u < kRPT; u++)
                        need |= (uint32_t)(valid[u] & !anyf & (closest_pack(r[u], slo_t, slo_s, bud) <= vmax)) << u;
                }
                if (__any_sync(0xffffffffu, need != 0)) {
#pragma unroll
                    for (int u = 0; u < kRPT; u++) {
                        if (!((need >> u) & 1u)) continue;
                        const bool f = feasible(P.q[q], r[u]);
                        const uint64_t idx = flat_index(v, per_tile, mt.pos0 + lane + u * 32);
                        if (cand_better(P.q[q], P.objective, idx, r[u], bi[q], br[q])) {
                            bi[q] = idx;
                            br[q] = r[u];
                            if (f) {
                                if (!bf[q] && pa.gfeas) atomicOr(&pa.gfeas[q], 1u);
                                atomicMax(&s_thr[q], (unsigned long long)obj_key<OBJ>(obj_q, r[u]));
                            } else {
                                const unsigned long long ck =
                                    closest_pack(r[u], P.q[q].slo_t, P.q[q].slo_s, P.q[q].budget);
                                if (ck < atomicMin(&s_vt[q], ck) && pa.gfeas)  // a block improvement
                                    atomicMax(reinterpret_cast<unsigned long long*>(pa.gfeas + SW_MAX_QUERIES) + q,
                                              ~ck);
                            }
                            bf[q] = f;
                        }
                    }
                }
            }
            if (PARETO) {
                uint32_t keepm = 0;  // DLT survivors, all kRPT lookups first (independent: ILP)
#pragma unroll
                for (int u = 0; u < kRPT; u++)
                    keepm |= (uint32_t)(valid[u] & !dlt_dominated(d, dh, r[u].w0 + r[u].w1, r[u].w2, rec_Q(r[u]))) << u;
                if (!__any_sync(0xffffffffu, keepm != 0)) continue;
                // deferred exact test: the stage's DLT survivors (rare) are appended to the
                // pass's candidate buffer -- one atomic per warp -- and tested after the pass
                // by pareto_exact_kernel, so this streaming loop stays HBM-bound
                const uint32_t mine = __popc(keepm);
                uint32_t incl = mine;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += v;
                }
                unsigned long long base = 0;
                if (lane == 31) base = atomicAdd(&pa.ctl->dlt_n, (unsigned long long)incl);
                base = __shfl_sync(0xffffffffu, base, 31);
                uint64_t slot = base + incl - mine;
#pragma unroll
                for (int u = 0; u < kRPT; u++) {
                    if (!((keepm >> u) & 1u)) continue;
                    if (slot < pa.cand_cap) {
                        PPoint x;
                        x.idx = flat_index(v, per_tile, mt.pos0 + lane + u * 32);
                        x.t = r[u].w0 + r[u].w1;
                        x.c = r[u].w2;
                        x.q = rec_Q(r[u]);
                        x.pad = 0;
                        pa.cand[slot] = x;
                    }
                    slot++;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; q++) {
        uint64_t idx = bi[q];
        Rec4 rr = br[q];
        block_reduce_cand(P.q[q], P.objective, idx, rr, s_tmp);
        if (threadIdx.x == 0) {
            partial[out_block * SW_MAX_QUERIES + q].idx = idx;
            partial[out_block * SW_MAX_QUERIES + q].r = rr;
        }
    }
}

// Fleet merge: block b reduces, for each of its request's queries q, the `count`
// candidates in[b * stride_block + j * stride_item + q] (j < count) -> out[b * SW_MAX_QUERIES
// + q], with the closest flag in .pad.  Per-block partials after a fleet scan
// (stride_item = SW_MAX_QUERIES) and the cross-rank merge of allgathered winners
// (stride_item = n_requests * SW_MAX_QUERIES) both use it.
__global__ void __launch_bounds__(kScanThreads) select_merge_kernel(const Cand* __restrict__ in, uint32_t count,
                                                                    uint64_t stride_item, uint64_t stride_block,
                                                                    const ScanJob* __restrict__ jobs,
                                                                    Cand* __restrict__ out) {
    __shared__ Cand s_tmp[32];
    const SelParams& P = jobs[blockIdx.x].P;
    const Cand* base = in + (uint64_t)blockIdx.x * stride_block;
    for (uint32_t q = 0; q < P.nq; q++) {
        uint64_t idx = kInf64;
        Rec4 r{};
        for (uint32_t j = threadIdx.x; j < count; j += blockDim.x) {
            const Cand c = base[(uint64_t)j * stride_item + q];
            if (cand_better(P.q[q], P.objective, c.idx, c.r, idx, r)) {
                idx = c.idx;
                r = c.r;
            }
        }
        block_reduce_cand(P.q[q], P.objective, idx, r, s_tmp);
        if (threadIdx.x == 0) {
            Cand& o = out[(uint64_t)blockIdx.x * SW_MAX_QUERIES + q];
            o.idx = idx;
            o.r = r;
            o.pad = (idx != kInf64 && !feasible(P.q[q], r)) ? 1ull : 0ull;
        }
        __syncthreads();
    }
}

// Fleet winners' full metrics: block b recomputes query q's winner of request b into
// out[b * nq + q] (winners strided by SW_MAX_QUERIES).
template <int NP>
__global__ void detail_fleet_kernel(const EvalJob* __restrict__ jobs, const Cand* __restrict__ win, uint32_t nq,
                                    DetailOut* __restrict__ out) {
    const uint32_t b = blockIdx.x;
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        const Cand c = win[(uint64_t)b * SW_MAX_QUERIES + q];
        if (c.idx != kInf64) detail_one<NP>(jobs[b].hdr, jobs[b].va, c.idx, out + (uint64_t)b * nq + q);
    }
}

// ============================================================================ fused stream
// Evaluation with NO record store: every candidate's record goes straight from registers
// to the a9 select predicate and the a8 Pareto filter (one kernel per strided tile pass).
//  - a9: per query a pruning key, higher = better, of the candidates already reported --
//    QUALITY_FIRST: the packed (Q, ~min(cost, 2^32-1)) key of a feasible one; COST_X_TTFF:
//    ~sat(cost x ttff_eff); while none is feasible, ~(packed saturated (V_t, V_c)) of a
//    closest-tier one.  A record whose key is below the best reported key is strictly
//    worse than a reported candidate and cannot win; the others (rare) are reduced per
//    warp with the query's total order (cand_better) and the warp's best is appended to
//    the query's candidate list (stream_select_final_kernel reduces it).  The keys live in
//    shared memory per block and in global memory across blocks and passes (atomicMax,
//    read at block start).  Saturation and ties only let more records through (the
//    filter stays conservative); a full candidate list is reported (cand_n > cap).
//  - a8: records the DLT does not rule out get the scan's exact warp-cooperative test
//    against the front (smem subset + L2) and this block's earlier survivors; the rest
//    are appended to the block's survivor list, flushed to the pass's survivor buffer,
//    which the usual pipeline merges into the front after the pass.
struct StreamArgs {
    const Dlt* dlt;
    ParetoCtl* ctl;  // dlt_n: DLT survivors appended (atomics)
    PPoint* pts;     // DLT survivors of the pass (exact-tested by pareto_exact_kernel)
    uint64_t pts_cap;
    Cand* cand;        // [SW_MAX_QUERIES][cand_cap] reported candidates per query
    uint32_t* cand_n;  // [SW_MAX_QUERIES]
    uint32_t cand_cap;
    unsigned long long* gkey;  // [3][SW_MAX_QUERIES]: key, closest key, feasible flag (all 0 = none)
    // tile hierarchy of the shard's tiles [tile_begin, tile_end): pass lvl of levels K
    // (lvl 0 = tiles u with u % 8^K == 0; lvl l >= 1 = multiples of 8^(K-l), not of 8^(K-l+1))
    uint32_t levels, lvl;
    uint64_t ntiles_pass;  // tiles in this pass
    uint32_t msplit;       // work items per tile (MID-digit slices): small passes fill the GPU
    uint64_t ib, ie;       // the shard's global candidate range
    SelParams P;
};

__device__ __forceinline__ uint64_t sat_mul64(uint64_t a, uint64_t b) {
    return __umul64hi(a, b) ? ~0ull : a * b;
}
// pruning keys (higher = better) of a feasible record and of a closest-tier record
__device__ __forceinline__ uint64_t prune_key(uint32_t obj, const Rec4& r) {
    return obj == 0 ? qc_key(r) : ~sat_mul64(r.w2, r.w0 + r.w1);
}
__device__ __forceinline__ uint64_t closest_key(const QueryDev& q, const Rec4& r) {
    const uint64_t vt = sat_sub(r.w0, q.slo_t) + sat_sub(r.w1, q.slo_s), vc = sat_sub(r.w2, q.budget);
    return ~((umin64(vt, 0xffffffffull) << 32) | umin64(vc, 0xffffffffull));
}

constexpr int kStreamThreads = 256;  // each block stages the DLT (~80 KB) + tables
struct StreamShared {
    // per warp and query: the best candidate this warp passed to the query's filter (total
    // order cand_better), kept by the warp's lane 0 (the only thread that touches it) and
    // appended to the query's list once, when the warp is done -- a report per improvement
    // overflowed the lists when many records tie on the pruning key
    Cand wb[kStreamThreads / 32][SW_MAX_QUERIES];
    QueryDev q[SW_MAX_QUERIES];
    unsigned long long key[SW_MAX_QUERIES];   // best pruning key of a reported feasible candidate
    unsigned long long ckey[SW_MAX_QUERIES];  // best closest-tier key of a reported candidate
    uint32_t feas[SW_MAX_QUERIES];            // a feasible candidate was reported
};

struct StreamEmit {
    const StreamArgs* sa;
    StreamShared* ss;
    const Dlt* d;
    DltHot dh;
    uint64_t rowbase;  // global index of this lane's row's first candidate
    uint32_t rl;
    bool edge;         // the row crosses the shard boundary: check each index
    bool allf;         // at the tile's start every query had a feasible report ...
    unsigned long long kmin;  // ... and this was the smallest of their pruning keys
    struct Put {
        static constexpr int kUnroll = 1;
        const StreamEmit* e;
        uint64_t base;  // index of candidate (dm, 0)
        bool live;
        __device__ __forceinline__ void operator()(uint32_t dl, uint32_t, const Rec4& r) const {
            const StreamArgs& a = *e->sa;
            StreamShared& S = *e->ss;
            const uint32_t lane = threadIdx.x & 31;
            const uint64_t idx = base + dl;
            const bool valid = live && (!e->edge || (idx >= a.ib && idx < a.ie));
            const uint32_t obj = a.P.objective;
            // ---- a9: which records can still beat what was reported?  Once every query has
            // a feasible report: only a record feasible for some query q with a pruning key
            // >= q's (keys only rise, so a stale read is a weaker filter, never a wrong one)
            bool pre = valid;
            if (e->allf) {
                const uint64_t key = prune_key(obj, r);
                bool any = false;
                for (uint32_t q = 0; q < a.P.nq; q++) {
                    const QueryDev& Q = S.q[q];
                    any |= (key >= S.key[q]) & (r.w2 <= Q.budget) & (r.w0 <= Q.slo_t) & (r.w1 <= Q.slo_s);
                }
                pre &= any;
            }
            const uint32_t nq = __any_sync(0xffffffffu, pre) ? a.P.nq : 0u;
            for (uint32_t q = 0; q < nq; q++) {
                const QueryDev Q = S.q[q];
                const bool f = valid & (r.w0 <= Q.slo_t) & (r.w1 <= Q.slo_s) & (r.w2 <= Q.budget);
                bool pass = f & (prune_key(obj, r) >= *(volatile unsigned long long*)&S.key[q]);
                if (!*(volatile uint32_t*)&S.feas[q])
                    pass |= valid & !f & (closest_key(Q, r) >= *(volatile unsigned long long*)&S.ckey[q]);
                if (!__any_sync(0xffffffffu, pass)) continue;
                uint64_t ci = pass ? idx : kInf64;  // the warp's best passing record
                Rec4 cr = r;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    uint64_t oi = ci;
                    Rec4 orr = cr;
                    shfl_cand(oi, orr, off);
                    if (lane + off < 32 && cand_better(Q, obj, oi, orr, ci, cr)) {
                        ci = oi;
                        cr = orr;
                    }
                }
                if (lane == 0 && ci != kInf64) {
                    Cand& wb = S.wb[threadIdx.x >> 5][q];
                    if (cand_better(Q, obj, ci, cr, wb.idx, wb.r)) {
                        wb.idx = ci;
                        wb.r = cr;
                    }
                    if (feasible(Q, cr)) {
                        const unsigned long long k = prune_key(obj, cr);
                        S.feas[q] = 1u;
                        atomicMax(&S.key[q], k);
                        atomicMax(&a.gkey[q], k);
                        a.gkey[2 * SW_MAX_QUERIES + q] = 1ull;
                    } else {
                        const unsigned long long k = closest_key(Q, cr);
                        atomicMax(&S.ckey[q], k);
                        atomicMax(&a.gkey[SW_MAX_QUERIES + q], k);
                    }
                }
                __syncwarp();
            }
            // ---- a8: the DLT filter; its (rare) survivors go to the pass's candidate
            // buffer -- one atomic per warp -- and are exact-tested after the pass by
            // pareto_exact_kernel (deferred, as in the scan)
            const bool cand = valid && !dlt_dominated(*e->d, e->dh, r.w0 + r.w1, r.w2, rec_Q(r));
            const unsigned pend = __ballot_sync(0xffffffffu, cand);
            if (!pend) return;
            const int ldr = __ffs(pend) - 1;
            unsigned long long b0 = 0;
            if (lane == ldr) b0 = atomicAdd(&a.ctl->dlt_n, (unsigned long long)__popc(pend));
            b0 = __shfl_sync(0xffffffffu, b0, ldr);
            const uint64_t slot = b0 + __popc(pend & ((1u << lane) - 1u));
            if (cand && slot < a.pts_cap) {
                PPoint pt;
                pt.idx = idx;
                pt.t = r.w0 + r.w1;
                pt.c = r.w2;
                pt.q = rec_Q(r);
                pt.pad = 0;
                a.pts[slot] = pt;
            }
        }
    };
    __device__ __forceinline__ Put at(uint32_t dm, bool live) const { return Put{this, rowbase + (uint64_t)dm * rl, live}; }
};

// registers: the eval path plus the in-kernel filters (2 blocks/SM only for one pool)
#ifndef SW_STREAM_MINB1
#define SW_STREAM_MINB1 2
#endif
#ifndef SW_STREAM_MINB2
#define SW_STREAM_MINB2 2  // 2 blocks (128 registers, ~0.7 KB spills) beat 1 block by 10% on C3
#endif
#ifndef SW_STREAM_MINB3
#define SW_STREAM_MINB3 1
#endif
__host__ __device__ constexpr int stream_min_blocks(int np, int bm) {
    return (np == 1 && bm < 2) ? SW_STREAM_MINB1 : (np == 2 && bm < 2) ? SW_STREAM_MINB2 : (np == 3 && bm < 2) ? SW_STREAM_MINB3 : 1;
}

// BM: the eval path (eval_mode) at compile time, as in eval_kernel.
template <int NP, int BM>
__global__ void __launch_bounds__(kStreamThreads, stream_min_blocks(NP, BM)) stream_kernel(EvalJob job, const __grid_constant__ StreamArgs sa) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ StreamShared ss;
    DevHeader& h = *reinterpret_cast<DevHeader*>(smem);
    VaEntry* va = reinterpret_cast<VaEntry*>(smem + sizeof(DevHeader));
    Dlt* d = reinterpret_cast<Dlt*>(smem + ((sizeof(DevHeader) + job.va_bytes + 127) & ~(size_t)127));
    {  // the DLT (16 B vectors) and the queries
        const uint4* src = reinterpret_cast<const uint4*>(sa.dlt);
        uint4* dst = reinterpret_cast<uint4*>(d);
        for (uint32_t i = threadIdx.x; i < sizeof(Dlt) / 16; i += blockDim.x) dst[i] = src[i];
    }
    if ((threadIdx.x & 31) == 0)  // each warp's lane 0 alone writes and reads its bests
        for (uint32_t q = 0; q < SW_MAX_QUERIES; q++) ss.wb[threadIdx.x >> 5][q].idx = kInf64;
    if (threadIdx.x < SW_MAX_QUERIES) {
        ss.q[threadIdx.x] = sa.P.q[threadIdx.x];
        ss.key[threadIdx.x] = sa.gkey[threadIdx.x];
        ss.ckey[threadIdx.x] = sa.gkey[SW_MAX_QUERIES + threadIdx.x];
        ss.feas[threadIdx.x] = sa.gkey[2 * SW_MAX_QUERIES + threadIdx.x] ? 1u : 0u;
    }
    stage_tables(job.hdr, job.va, &h, va, (uint32_t)job.va_bytes, &bar);  // ends with a barrier
    const DltHot dh{d->kbase, d->qbase, d->qmshift, d->cshift};
    const uint64_t row = h.row;
    const uint32_t rl = h.radix[h.B - 1];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t sh = 3 * (sa.levels - sa.lvl);
    const uint64_t nwork = sa.ntiles_pass * sa.msplit;
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwork; w += nwarps) {
        const uint64_t j = w / sa.msplit;  // the pass's j-th tile, MID slice w % msplit
        const uint32_t slice = (uint32_t)(w - j * sa.msplit);
        const uint64_t u = sa.lvl == 0 ? j << sh : ((j / 7) * 8 + (j % 7) + 1) << sh;  // tile of the pass
        const uint64_t t = job.tile_begin + u;
        if (t >= job.tile_end) break;  // warp-uniform; tiles grow with j
        if (lane < sa.P.nq) {  // other blocks' reported keys (global, monotone) tighten ours
            const unsigned long long* g = sa.gkey;
            atomicMax(&ss.key[lane], *(volatile const unsigned long long*)&g[lane]);
            atomicMax(&ss.ckey[lane], *(volatile const unsigned long long*)&g[SW_MAX_QUERIES + lane]);
            if (*(volatile const unsigned long long*)&g[2 * SW_MAX_QUERIES + lane]) ss.feas[lane] = 1u;
        }
        __syncwarp();
        const uint64_t H = t * kTileRows + lane;
        const uint64_t rb = H * row;
        bool allf = true;
        unsigned long long kmin = ~0ull;
        for (uint32_t q = 0; q < sa.P.nq; q++) {
            allf &= *(volatile uint32_t*)&ss.feas[q] != 0;
            kmin = min(kmin, *(volatile unsigned long long*)&ss.key[q]);
        }
        const StreamEmit em{&sa, &ss, d, dh, rb, rl, rb < sa.ib || rb + row > sa.ie, allf, kmin};
        eval_tile_b<NP, BM != 0, BM == 2>(h, va, t, em, slice, sa.msplit);
    }
    if (lane == 0)  // this warp's best per query -> the query's list (lane 0 wrote them)
        for (uint32_t q = 0; q < sa.P.nq; q++) {
            const Cand& wb = ss.wb[threadIdx.x >> 5][q];
            if (wb.idx == kInf64) continue;
            const uint32_t slot = atomicAdd(&sa.cand_n[q], 1u);
            if (slot < sa.cand_cap) {
                Cand c = wb;
                c.pad = 0;
                sa.cand[(uint64_t)q * sa.cand_cap + slot] = c;
            }
        }
}

// One candidate from scratch (a1-a7 for a single index; plain loads from global/L2).
template <int NP>
__device__ __forceinline__ Rec4 eval_one(const DevHeader& h, const VaEntry* __restrict__ va, uint64_t index) {
    State<NP> st;
    state_init(st, h);
    uint32_t dig[kMaxDigits];
    uint64_t rem = index;
    for (int b = (int)h.B - 1; b >= 0; b--) {  // a1: i mod r_b, LSD first
        dig[b] = (uint32_t)(rem % h.radix[b]);
        rem /= h.radix[b];
    }
    for (uint32_t b = 0; b < h.B; b++) {
        const uint32_t ch = h.choice[h.coff[b] + dig[b]];
        const uint32_t k = ch_k(ch), p = ch_pool(ch);
        run_block<NP, 0>(st, h, ch, h.first[b], h.first[b + 1], va + h.voff[b] + dig[b], h.radix[b]);
    }
    Rec4 r;
    r.w0 = st.R0;
    r.w1 = (uint64_t)st.M - st.R0;
    r.w2 = state_cost(st, h);
    r.w3 = (uint64_t)st.Q | ((uint64_t)st.cnt << 32) | ((uint64_t)st.used << 48);
    return r;
}

// Seed of a stream: ns candidates spread evenly over [b, e) -> work[ctl->m_in++] (their
// exact front, reduced next, gives the first pass a useful DLT).
template <int NP>
__global__ void stream_seed_kernel(const DevHeader* __restrict__ hdr, const VaEntry* __restrict__ va, uint64_t b,
                                   uint64_t e, uint32_t ns, PPoint* __restrict__ work, ParetoCtl* ctl) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ns) return;
    const uint64_t idx = b + (uint64_t)((unsigned __int128)(e - b) * j / ns);
    const Rec4 r = eval_one<NP>(*hdr, va, idx);
    PPoint p;
    p.idx = idx;
    p.t = r.w0 + r.w1;
    p.c = r.w2;
    p.q = rec_Q(r);
    p.pad = 0;
    work[atomicAdd(&ctl->m_in, 1u)] = p;
}

// Per query q (block q): reduce the reported candidates of stream passes -> out[q] (the
// closest flag in .pad), like select_final_kernel.
__global__ void __launch_bounds__(kScanThreads) stream_select_final_kernel(const Cand* __restrict__ cand,
                                                                           const uint32_t* __restrict__ cand_n,
                                                                           uint32_t cap, SelParams P,
                                                                           Cand* __restrict__ out) {
    __shared__ Cand s_tmp[32];
    const uint32_t q = blockIdx.x;
    const uint32_t n = min(cand_n[q], cap);
    uint64_t idx = kInf64;
    Rec4 r{};
    for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
        const Cand c = cand[(uint64_t)q * cap + j];
        if (cand_better(P.q[q], P.objective, c.idx, c.r, idx, r)) {
            idx = c.idx;
            r = c.r;
        }
    }
    block_reduce_cand(P.q[q], P.objective, idx, r, s_tmp);
    if (threadIdx.x == 0) {
        out[q].idx = idx;
        out[q].r = r;
        out[q].pad = (idx != kInf64 && !feasible(P.q[q], r)) ? 1ull : 0ull;
    }
}

// ============================================================================ greedy planner
// The paper's provisioner on the batched evaluator:
// a cost-efficient baseline -- per digit the choice with the smallest (level score, k,
// pool price, index): cheap models, one GPU, cheap GPUs -- then iterative
// refinement: every single-digit change of the current plan (switch model / GPU type /
// parallelism) is evaluated by one thread in parallel, the best under the
// query's total order is taken if strictly better; stop at a local optimum.
// One CTA runs the whole search (R28).
constexpr int kGreedyThreads = 1024;
constexpr int kMaxLevels = 16;

struct GreedyArgs {
    QueryDev q;
    uint32_t objective, n_levels;
    uint64_t start;  // kInf64: the cost-efficient baseline
    uint32_t score[kMaxLevels];
    uint32_t max_iter;
};
struct GreedyOut {
    uint64_t index;
    Rec4 rec;
    uint64_t evaluations;
    uint32_t iterations, feasible;
};

// One candidate's record by full recompute (compile-time gang updates per block).
template <int NP>
__device__ Rec4 full_eval(const DevHeader& h, const VaEntry* __restrict__ va, uint64_t index) {
    State<NP> st;
    state_init(st, h);
    uint32_t dig[kMaxDigits];
    uint64_t rem = index;
    for (int b = (int)h.B - 1; b >= 0; b--) {
        dig[b] = (uint32_t)(rem % h.radix[b]);
        rem /= h.radix[b];
    }
    for (uint32_t b = 0; b < h.B; b++) {
        const uint32_t ch = h.choice[h.coff[b] + dig[b]];
        const uint32_t k = ch_k(ch), p = ch_pool(ch);
        const VaEntry* vb = va + h.voff[b] + dig[b];
        const uint32_t f0 = h.first[b], f1 = h.first[b + 1], r = h.radix[b];
        switch (k) {
            case 1: run_block<NP, 1>(st, h, ch, f0, f1, vb, r); break;
            case 2: run_block<NP, 2>(st, h, ch, f0, f1, vb, r); break;
            case 4: run_block<NP, 4>(st, h, ch, f0, f1, vb, r); break;
            case 8: run_block<NP, 8>(st, h, ch, f0, f1, vb, r); break;
            default: run_block<NP, 0>(st, h, ch, f0, f1, vb, r); break;
        }
    }
    Rec4 o;
    o.w0 = st.R0;
    o.w1 = (uint64_t)st.M - st.R0;
    o.w2 = state_cost(st, h);
    o.w3 = (uint64_t)st.Q | ((uint64_t)st.cnt << 32) | ((uint64_t)st.used << 48);
    return o;
}

template <int NP>
__global__ void __launch_bounds__(kGreedyThreads) greedy_kernel(const DevHeader* __restrict__ g_hdr,
                                                               const VaEntry* __restrict__ g_va, GreedyArgs A,
                                                               GreedyOut* __restrict__ out) {
    __shared__ Cand s_tmp[32];
    __shared__ uint64_t s_place[kMaxDigits];
    __shared__ uint32_t s_dig[kMaxDigits], s_nboff[kMaxDigits + 1];
    __shared__ uint64_t s_cur;
    __shared__ Rec4 s_rec;
    __shared__ int s_done;
    const DevHeader& h = *g_hdr;
    const uint32_t B = h.B;
    if (threadIdx.x == 0) {
        uint64_t pl = 1;
        for (int b = (int)B - 1; b >= 0; b--) {
            s_place[b] = pl;
            pl *= h.radix[b];
        }
        s_nboff[0] = 0;
        for (uint32_t b = 0; b < B; b++) s_nboff[b + 1] = s_nboff[b] + h.radix[b] - 1;
        uint64_t cur = A.start;
        if (cur == kInf64) {  // cost-efficient baseline
            cur = 0;
            for (uint32_t b = 0; b < B; b++) {
                uint32_t best = 0;
                for (uint32_t c = 1; c < h.radix[b]; c++) {
                    const uint32_t x = h.choice[h.coff[b] + c], y = h.choice[h.coff[b] + best];
                    const uint32_t sx = A.score[ch_level(x)], sy = A.score[ch_level(y)];
                    const uint64_t px = h.price[ch_pool(x)], py = h.price[ch_pool(y)];
                    const bool lt = sx != sy ? sx < sy : (ch_k(x) != ch_k(y) ? ch_k(x) < ch_k(y) : px < py);
                    if (lt) best = c;
                }
                cur += best * s_place[b];
            }
        }
        s_cur = cur;
        s_rec = full_eval<NP>(h, g_va, cur);
        s_done = 0;
    }
    __syncthreads();
    uint32_t iters = 0;
    uint64_t evals = 1;
    const uint32_t n_nb = s_nboff[B];
    while (true) {
        if (threadIdx.x == 0) {
            uint64_t rem = s_cur;
            for (int b = (int)B - 1; b >= 0; b--) {
                s_dig[b] = (uint32_t)(rem % h.radix[b]);
                rem /= h.radix[b];
            }
        }
        __syncthreads();
        uint64_t idx = kInf64;
        Rec4 r{};
        for (uint32_t t = threadIdx.x; t < n_nb; t += blockDim.x) {  // one neighbour per thread
            uint32_t b = 0;
            while (t >= s_nboff[b + 1]) b++;
            uint32_t c = t - s_nboff[b];
            if (c >= s_dig[b]) c++;  // skip the current choice
            const uint64_t x = s_cur - (uint64_t)s_dig[b] * s_place[b] + (uint64_t)c * s_place[b];
            const Rec4 rx = full_eval<NP>(h, g_va, x);
            if (cand_better(A.q, A.objective, x, rx, idx, r)) {
                idx = x;
                r = rx;
            }
        }
        block_reduce_cand(A.q, A.objective, idx, r, s_tmp);
        evals += n_nb;
        if (threadIdx.x == 0) {
            if (idx != kInf64 && iters < A.max_iter && cand_better(A.q, A.objective, idx, r, s_cur, s_rec)) {
                s_cur = idx;
                s_rec = r;
            } else {
                s_done = 1;
            }
        }
        __syncthreads();
        if (s_done) break;
        iters++;
    }
    if (threadIdx.x == 0) {
        out->index = s_cur;
        out->rec = s_rec;
        out->iterations = iters;
        out->evaluations = evals;
        out->feasible = feasible(A.q, s_rec) ? 1u : 0u;
    }
}

// Linearise n records [index, index + n) of a tiled segment (host views / tests).
__global__ void gather_records_kernel(SegView v, uint64_t index, uint64_t n, Rec4* __restrict__ out) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint64_t i = index + k;
    const uint64_t H = i / v.row, j = i - H * v.row;
    const uint64_t t = H / kTileRows - v.t0, lane = H % kTileRows;
    out[k] = v.recs[t * kTileRows * v.row + j * kTileRows + lane];
}

}  // namespace sw
