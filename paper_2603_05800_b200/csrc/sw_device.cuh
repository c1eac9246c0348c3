// sw_device.cuh -- device-side layout and the per-scene max-plus step.
//
// Product code of libsw_plan.so.  Shares nothing with oracle/ (the CPU checker).
// Citations: P:n = PAPER.md line n; R<n> = DESIGN.md reading n.
#pragma once
#include <cstdint>

#include "sw_plan.h"

namespace sw {

constexpr uint64_t kInf64 = 0xFFFFFFFFFFFFFFFFull;
constexpr int kMaxG = 8;  // register slots per pool on the fast path (pools of <= 8 GPUs; wider: sw_wide.cuh)
constexpr int kMaxP = SW_MAX_POOLS;
constexpr int kMaxDigits = SW_MAX_DIGITS + 2;  // + up to 2 virtual radix-1 digits
constexpr int kMaxChoiceTotal = SW_MAX_DIGITS * SW_MAX_CHOICES;
constexpr uint64_t kUsPerHour = 3600000000ull;
constexpr uint64_t kHalfHour = 1800000000ull;

// Table entry for (scene, choice): V+A stage time and the quality contribution
// dur_ms(s) x score(level) (R12).  16 B -> one LDS.128 per scene-step.
struct __align__(16) VaEntry {
    uint64_t t_us;
    uint32_t q;
    uint32_t t_vae;  // VAE stage time of a disaggregated choice (R37; 0 = none), < 2^32 us
};

// LSD table entry (32 B), stored in (pool, k)-group order: the last scene's stage time
// and quality for choice dl, and X_t = G_p price_p t (RESERVED) or k price_p t (BUSY)
// split as X_t = cq * 3.6e9 + cr, so a candidate's pool cost needs no multiply/divide:
// floor((Y + X_t) / D) = qY + cq + (rY + cr >= D) for Y = qY * D + rY.
struct __align__(16) LsdEntry {
    uint64_t t_us;
    uint64_t x1;   // money: cq; energy: the choice's own term when it ends the pool (see lsd_fast)
    uint64_t x2;   // money: cr (< 3.6e9); energy: the term when it does not
    uint32_t q;
    uint32_t dl;
};

// Per-request constants, packed ON THE DEVICE by pack_kernel, staged into shared
// memory by every eval CTA with one TMA bulk copy (cp.async.bulk + mbarrier).
// Digits are left-padded with virtual radix-1 / empty-block digits so that
// B >= 3: digits [0, B-2) are the per-thread "row" prefix (HI), digit B-2 is the
// warp-uniform MID loop and digit B-1 the warp-uniform LSD loop.
struct __align__(16) DevHeader {
    uint32_t S, B, NP, flags;     // flags: 1 scene0 static, 2 BUSY billing, 4 COST_X_TTFF
    uint32_t s0, n_va, n_choice, pad0;
    uint64_t R0_static, fixed_cost;
    uint64_t va_bytes;            // n_va * 16
    uint64_t row;                 // r_{B-2} * r_{B-1}: candidates per thread-row
    uint64_t n_rows;              // N / row
    uint64_t N;
    uint64_t place[kMaxDigits];   // place value of digit b within a ROW index (b < B-2)
    uint32_t radix[kMaxDigits];
    uint32_t first[kMaxDigits + 2];
    uint32_t coff[kMaxDigits];    // choice offset of digit b
    uint32_t voff[kMaxDigits];    // va offset of digit b
    uint32_t G[kMaxP];
    uint32_t Gbill[kMaxP];        // billed GPUs G'_p >= G_p (Spot over-provisioning, R32)
    uint64_t price[kMaxP];
    uint64_t Gprice[kMaxP];       // G'_p * price_p (device-computed in pack_kernel)
    uint64_t ready[kMaxP];        // pool p's GPUs free from this time (load + warm-up, R31)
    uint64_t Pact[kMaxP];         // energy metric (R38): busy power of a GPU of pool p (W)
    uint64_t Pidle[kMaxP];        //   idle power (W)
    uint64_t PidleG[kMaxP];       //   idle power x billed GPUs
    // LSD choices grouped by (pool, k) so the inner loop has neither: group g covers
    // lsd_dl[lsd_goff[g] .. lsd_goff[g+1]) with pool/k packed in lsd_pk[g] (p | k << 8)
    uint32_t lsd_ngroups, pad1;
    uint32_t lsd_goff[SW_MAX_CHOICES + 1];
    uint32_t lsd_pk[SW_MAX_CHOICES];
    uint32_t lsd_dl[SW_MAX_CHOICES];
    LsdEntry lsd[SW_MAX_CHOICES];  // device-computed in pack_kernel
    uint64_t a[SW_MAX_SCENES];    // fixed-stage ready times (a2), device-computed
    uint64_t P[SW_MAX_SCENES];    // deadline offsets P_s = sum_{j<s} d_j
    uint32_t choice[kMaxChoiceTotal];  // level | k << 8 | pool << 16
};
static_assert(sizeof(DevHeader) % 16 == 0, "TMA bulk copies need 16 B multiples");

__host__ __device__ __forceinline__ uint32_t ch_level(uint32_t c) { return c & 0xff; }
__host__ __device__ __forceinline__ uint32_t ch_k(uint32_t c) { return (c >> 8) & 0xff; }
__host__ __device__ __forceinline__ uint32_t ch_pool(uint32_t c) { return (c >> 16) & 0xff; }
// VAE pool + 1 of a disaggregated choice (FramePack DiT -> VAE, R37); 0 = VAE folded into V+A
__host__ __device__ __forceinline__ uint32_t ch_vae(uint32_t c) { return c >> 24; }

// DevHeader.flags: 1 scene0 static, 2 BUSY billing, 4 COST_X_TTFF, 8 energy metric (R38),
// 16 some choice has a separate VAE stage (R37), 32 the LSD fast path applies.  Cost modes of the kernels: bit 0 =
// BUSY billing, bit 1 = energy (0 money RESERVED, 1 money BUSY, 2 energy RESERVED,
// 3 energy BUSY); every mode but 0 accumulates busy GPU time.
__host__ __device__ __forceinline__ int cost_mode(uint32_t flags) {
    return ((flags & 2u) ? 1 : 0) | ((flags & 8u) ? 2 : 0);
}
// Eval path: 0 fast path, money + RESERVED (no busy time); 1 fast path with busy time;
// 2 generic path -- flag 32 (set at create) says the fast path applies: the last digit's
// block is one scene >= 1 and no choice has a VAE stage (flag 16).
__host__ __device__ __forceinline__ int eval_mode(uint32_t flags) {
    return ((flags & 16u) || !(flags & 32u)) ? 2 : cost_mode(flags) ? 1 : 0;
}

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Pool cost, round-half-up to milli-cents: (X * price + 1.8e9) / 3.6e9 (Table 3,
// P:623-641; R10/R11).  Division by a compile-time constant -> mul.hi sequence.
__device__ __forceinline__ uint64_t pool_cost(uint64_t X, uint64_t price) {
    return (X * price + kHalfHour) / kUsPerHour;
}

// Evaluation state after a prefix of scenes.  F[p][*] is the ascending multiset of
// the free times of pool p's GPUs (slots >= G_p hold +inf so they are never taken).
template <int NP>
struct State {
    uint64_t F[NP][kMaxG];
    uint64_t end[NP];   // max F[p] (pool span end)
    uint64_t busy[NP];  // sum k * t (GPU-us), BUSY billing
    uint64_t R0;        // ready time of scene 0 (TTFF)
    int64_t M;          // max_s (R_s - P_s) so far: TTFF_eff
    uint32_t cnt;       // rebuffering events
    uint32_t Q;         // quality
    uint32_t used;      // pool-used mask
};

template <int NP>
__device__ __forceinline__ void state_init(State<NP>& st, const DevHeader& h) {
#pragma unroll
    for (int p = 0; p < NP; p++) {
#pragma unroll
        for (int g = 0; g < kMaxG; g++) st.F[p][g] = (uint32_t)g < h.G[p] ? h.ready[p] : kInf64;
        st.end[p] = 0;
        st.busy[p] = 0;
    }
    st.R0 = h.R0_static;  // static intro ready time, 0 otherwise
    st.M = (int64_t)h.R0_static;
    st.cnt = 0;
    st.Q = 0;
    st.used = 0;
}

// F[k-1] for a runtime k (select chain, no local-memory indexing).
__device__ __forceinline__ uint64_t sel_dyn(const uint64_t (&F)[kMaxG], uint32_t i) {
    uint64_t r = F[0];
#pragma unroll
    for (int j = 1; j < kMaxG; j++) r = (i == (uint32_t)j) ? F[j] : r;
    return r;
}

// The k-earliest-free gang update (a4), branch-free in registers:
//   F' = sort(F[k:] ++ [e]*k)   <=>   F'[j] = max(F[j], min(e, F[j+k]))   (F[>=G] = inf)
// since e >= F[k-1] >= F[0..k-1]: slot j keeps F[j+k] while F[j+k] < e, then takes
// e for k slots, then keeps F[j].
template <int K>
__device__ __forceinline__ void gang_update_static(uint64_t (&F)[kMaxG], uint64_t e) {
#pragma unroll
    for (int j = 0; j < kMaxG; j++) {
        uint64_t up = (j + K < kMaxG) ? F[j + K] : kInf64;
        F[j] = umax64(F[j], umin64(e, up));
    }
}

__device__ __forceinline__ void gang_update_dyn(uint64_t (&F)[kMaxG], uint64_t e, uint32_t k) {
    uint64_t sh[kMaxG];
#pragma unroll
    for (int j = 0; j < kMaxG; j++) sh[j] = F[j];
    // barrel shift left by k (k in 1..8), vacated slots +inf
#pragma unroll
    for (int bit = 0; bit < 4; bit++) {
        const int d = 1 << bit;
        const bool on = (k >> bit) & 1u;
#pragma unroll
        for (int j = 0; j < kMaxG; j++) {
            uint64_t v = (j + d < kMaxG) ? sh[j + d] : kInf64;
            sh[j] = on ? v : sh[j];
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxG; j++) F[j] = umax64(F[j], umin64(e, sh[j]));
}

// One scene-step on pool p with degree k; returns the scene's ready time e = R_s.
// KS > 0: k is a compile-time constant (warp-uniform MID/LSD loops); KS == 0: runtime.
// BUSY: accumulate k x t (BUSY billing); RESERVED billing never reads it.
// The VAE stage of a disaggregated choice (R37; "FramePack DiT streams latent outputs to the
// VAE for decoding ... pipelined execution"): on pool vp, one GPU (the VAE is not
// parallelised), once the DiT finished at e and a VAE GPU is free.
template <int NP, bool BUSY>
__device__ __forceinline__ uint64_t vae_step(State<NP>& st, uint32_t vp, uint64_t e, uint64_t tv) {
    uint64_t ev = e;
#pragma unroll
    for (int q = 0; q < NP; q++) {
        if ((uint32_t)q == vp) {
            ev = umax64(e, st.F[q][0]) + tv;
            gang_update_static<1>(st.F[q], ev);
            st.end[q] = umax64(st.end[q], ev);
            if (BUSY) st.busy[q] += tv;
        }
    }
    st.used |= 1u << vp;
    return ev;
}

template <int NP, int KS, bool BUSY = true>
__device__ __forceinline__ uint64_t scene_step(State<NP>& st, uint32_t p, uint32_t k,
                                               uint64_t a, uint64_t t) {
    // STATIC rung (k = 0, runtime path only): no video stage, no GPU -- the scene is
    // ready with its text and audio, R_s = a_s (reading R33)
    if (KS == 0 && k == 0) return a;
    uint64_t e = 0;
#pragma unroll
    for (int q = 0; q < NP; q++) {
        if ((uint32_t)q == p) {
            // the scene needs its text+audio (a_s) and the k earliest-free GPUs
            const uint64_t fk = KS ? st.F[q][KS - 1] : sel_dyn(st.F[q], k - 1);
            e = umax64(a, fk) + t;
            if (KS) gang_update_static<KS>(st.F[q], e);
            else gang_update_dyn(st.F[q], e, k);
            st.end[q] = umax64(st.end[q], e);
            if (BUSY) st.busy[q] += (uint64_t)k * t;
        }
    }
    st.used |= 1u << p;
    return e;
}

// Playback metrics after scene s ready at e (R7-R9); St = State<NP> or MidState.
template <class St>
__device__ __forceinline__ void scene_metrics(St& st, uint32_t s, uint64_t e,
                                              uint64_t Ps, uint32_t q) {
    if (s == 0) {
        st.R0 = e;
        st.M = (int64_t)e;
    } else {
        const int64_t d = (int64_t)e - (int64_t)Ps;
        if (d > st.M) {
            st.M = d;
            st.cnt++;
        }
    }
    st.Q += q;
}

// Dispatch a runtime k to a compile-time specialisation (k warp-uniform => no
// divergence; k in {1,2,4,8} covers USP degrees dividing the 40 heads).
template <int NP, bool BUSY = true>
__device__ __forceinline__ uint64_t scene_step_uniform(State<NP>& st, uint32_t p, uint32_t k,
                                                       uint64_t a, uint64_t t) {
    switch (k) {
        case 1: return scene_step<NP, 1, BUSY>(st, p, k, a, t);
        case 2: return scene_step<NP, 2, BUSY>(st, p, k, a, t);
        case 4: return scene_step<NP, 4, BUSY>(st, p, k, a, t);
        case 8: return scene_step<NP, 8, BUSY>(st, p, k, a, t);
        default: return scene_step<NP, 0, BUSY>(st, p, k, a, t);
    }
}

// MID state (eval tiles): the HI state of a row is shared by its rm MID choices, and a
// MID choice (k, pool pm) changes only pool pm -- so the MID pass works on a copy of
// that one pool's free times (the other pools are read from the HI state).  Keeps the
// live state at (NP + 1) pools instead of 2 NP (no spills with 3-4 pools).
struct MidState {
    uint64_t F[kMaxG];
    uint64_t end, busy;
    uint64_t R0;
    int64_t M;
    uint32_t cnt, Q, used, pm;
};

template <int NP>
__device__ __forceinline__ void mid_init(MidState& m, const State<NP>& st, uint32_t pm) {
#pragma unroll
    for (int g = 0; g < kMaxG; g++) m.F[g] = st.F[0][g];
    m.end = st.end[0];
    m.busy = st.busy[0];
#pragma unroll
    for (int q = 1; q < NP; q++)
        if ((uint32_t)q == pm) {
#pragma unroll
            for (int g = 0; g < kMaxG; g++) m.F[g] = st.F[q][g];
            m.end = st.end[q];
            m.busy = st.busy[q];
        }
    m.R0 = st.R0;
    m.M = st.M;
    m.cnt = st.cnt;
    m.Q = st.Q;
    m.used = st.used;
    m.pm = pm;
}

// One MID scene step on pool pm (KS compile-time k; KS == 0: runtime k incl. STATIC).
template <int KS, bool BUSY>
__device__ __forceinline__ uint64_t mid_step(MidState& m, uint32_t k, uint64_t a, uint64_t t) {
    if (KS == 0 && k == 0) return a;  // STATIC rung (R33)
    const uint64_t fk = KS ? m.F[KS - 1] : sel_dyn(m.F, k - 1);
    const uint64_t e = umax64(a, fk) + t;
    if (KS) gang_update_static<KS>(m.F, e);
    else gang_update_dyn(m.F, e, k);
    m.end = umax64(m.end, e);
    if (BUSY) m.busy += (uint64_t)k * t;
    m.used |= 1u << m.pm;
    return e;
}

// The full state after the MID pass (generic LSD path).
template <int NP>
__device__ __forceinline__ State<NP> merge_mid(const State<NP>& st, const MidState& m) {
    State<NP> s2 = st;
#pragma unroll
    for (int q = 0; q < NP; q++)
        if ((uint32_t)q == m.pm) {
#pragma unroll
            for (int g = 0; g < kMaxG; g++) s2.F[q][g] = m.F[g];
            s2.end[q] = m.end;
            s2.busy[q] = m.busy;
        }
    s2.R0 = m.R0;
    s2.M = m.M;
    s2.cnt = m.cnt;
    s2.Q = m.Q;
    s2.used = m.used;
    return s2;
}

// Packed 32 B record: {ttff, stall, cost, Q | cnt << 32 | flags << 48}.
struct __align__(32) Rec4 {
    uint64_t w0, w1, w2, w3;
};

// Pool term of the record's cost field: money (Table 3 prices, round half up, R10/R11) or
// energy in microjoules (R38: busy GPUs at P_act, the pool's other rented GPUs idle at
// P_idle until its last finish under RESERVED; BUSY: busy time only).
template <int MODE>
__device__ __forceinline__ uint64_t pool_term(const DevHeader& h, int q, uint64_t end, uint64_t busy) {
    if (MODE == 0) return (end * h.Gprice[q] + kHalfHour) / kUsPerHour;
    if (MODE == 1) return pool_cost(busy, h.price[q]);
    if (MODE == 2) return h.PidleG[q] * end + (h.Pact[q] - h.Pidle[q]) * busy;
    return h.Pact[q] * busy;
}

template <int NP>
__device__ __forceinline__ uint64_t state_cost(const State<NP>& st, const DevHeader& h) {
    uint64_t c = h.fixed_cost;
    const int mode = cost_mode(h.flags);
#pragma unroll
    for (int p = 0; p < NP; p++) {
        switch (mode) {  // an unused pool: end = busy = 0 -> 0
            case 0: c += pool_term<0>(h, p, st.end[p], st.busy[p]); break;
            case 1: c += pool_term<1>(h, p, st.end[p], st.busy[p]); break;
            case 2: c += pool_term<2>(h, p, st.end[p], st.busy[p]); break;
            default: c += pool_term<3>(h, p, st.end[p], st.busy[p]); break;
        }
    }
    return c;
}

__device__ __forceinline__ void st_global_256(void* ptr, const Rec4& r) {
    asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "l"(r.w0), "l"(r.w1),
                 "l"(r.w2), "l"(r.w3)
                 : "memory");
}

__device__ __forceinline__ Rec4 ld_global_nc_256(const void* ptr) {
    Rec4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2), "=l"(r.w3)
                 : "l"(ptr));
    return r;
}

__host__ __device__ __forceinline__ uint32_t rec_Q(const Rec4& r) { return (uint32_t)r.w3; }

// ---- TMA bulk staging (cp.async.bulk global -> shared, completion on an mbarrier) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Bulk prefetch of [src, src + bytes) into L2 (no completion tracking; bytes % 16 == 0).
__device__ __forceinline__ void tma_prefetch_l2(const void* src_gmem, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}

// Waits with a suspend-time hint: the warp sleeps until the phase completes (or the hint
// expires) instead of re-issuing try_wait -- hot spinning consumers cost ~20% of the scan's
// issued instructions.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase), "r"(20000u)
            : "memory");
    } while (!done);
}

// Stage header + used VA entries into shared memory (one elected thread issues the
// bulk copies; everyone waits on the mbarrier).  bytes multiples of 16 (static_assert
// above; va entries are 16 B).
__device__ __forceinline__ void stage_tables(const DevHeader* __restrict__ g_hdr,
                                             const VaEntry* __restrict__ g_va, DevHeader* s_hdr,
                                             VaEntry* s_va, uint32_t va_bytes, uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const uint32_t hb = (uint32_t)sizeof(DevHeader);
        mbar_expect_tx(bar, hb + va_bytes);
        tma_bulk_g2s(s_hdr, g_hdr, hb, bar);
        if (va_bytes) tma_bulk_g2s(s_va, g_va, va_bytes, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
}

}  // namespace sw
