// B200 (sm_100a) CFR / CFR+ iteration: device kernels, CUDA-Graph orchestration
// and the solver half of the C ABI (include/cfr_b200.h).
//
// One iteration (§3.2), all state resident in HBM:
//   k_fwd  level l = 1..D-1  : reach factors of the decision nodes of depth l
//                              (Eq 2 pi_check and Eq 4 pi_hat per player, the
//                              paper's Pi_check / Pi_hat recurrences Eq 13, P:266,
//                              P:281) -- child-centric, terminals never touched.
//   k_bwd  level L = D-1..0  : one CTA per tile of whole infosets: node values
//                              (Eq 1 / Eq 11), the cancelled-form
//                              regret terms of Eq 7 (matrix form P:313) and
//                              pi_bar of Eq 5 summed EXACTLY in int64
//                              slices, then -- because the infoset is complete
//                              and its sigma is no longer needed this iteration --
//                              the fused update: cumulative regret (Eq 8/15 or
//                              CFR+), average-strategy sums (Eq 10/14) and regret
//                              matching (Eq 9).
//   k_deferred               : the same update for infosets that span depths or
//                              tiles (accumulated globally with int64 atomics).
// No tensor cores: the path is a sparse gather/scatter at < 1 flop/byte.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "game.hpp"

namespace cfrb {

// Device tile / segment records (built by the solver from the game's TileH /
// SegH plus the precision-dependent staging layout).
struct TileD {
    long long s0, s1;    // slot range
    int seg0, seg1;      // segments
    int npairs;          // (h, a) pairs of the tile's segments
    int staged;          // 0: children read from global; 1: uniform rows, chunked; 2: generic rows
    int rowlen;          // elements per row (mode 1)
    int cpr;             // chunks per row (mode 1)
    int stride;          // row stride in elements (mode 1)
    float inv_cpr;       // 1 / cpr
    int contrib;         // 1: add this tile's deferred partial sums (trunk tiles: rank 0 only)
    int pad;
};
struct SegD {
    long long h, qb;     // internal infoset, qbase[h]
    long long sb, se;    // member slots
    long long dq, dh;    // compact accumulator pair base / infoset index (deferred only)
    int pair_off, n, owner, fused;
};

enum { MODE_CFR = 0, MODE_VALUES = 1, MODE_BR = 2 };

template <class R, class I>
struct DG {
    R* U;          // [V * Pc] node values, canonical order; terminal rows = u
    R* reach;      // [ND][2P] AoS, canonical decision order: pi_check(., 1..P), pi_hat(., 1..P)
    R* sig;        // [Q + C] sigma_ext = current strategy (internal q order) | chance
    R* regret;     // [Q] cumulative regret
    R* snum;       // [Q] sum_t w_t pi_bar sigma
    R* sden;       // [H] sum_t w_t pi_bar
    unsigned long long* acc_r;  // [ndef pairs][3] exact slices of the deferred infosets (compact)
    unsigned long long* acc_p;  // [ndef][3]; acc_r and acc_p are one contiguous exchange block
    const long long* dqbase;    // [ndef + 1] compact pair base of each deferred infoset
    const I* f_parent;            // [NS] slot order: parent slot, incoming sigma_ext edge, parent actor
    const I* f_e;
    const unsigned char* f_pact;
    const I* s_node;              // [NS] backward pass (slot order)
    const I* s_cb;
    const int* s_n;
    const I* s_ebase;
    const unsigned char* s_actor;
    const I* s_dec;
    const int* s_coff;
    const I* qbase;               // [H+1] internal
    const unsigned char* owner;   // [H]
    const TileD* tiles;
    const SegD* segs;
    const I* deferred;            // [ndef]
    long long* ctrl;              // [0] iterations done, [1] first bad iteration, [2] done counter
    unsigned long long* lcnt;     // [D][4] streaming-level work counters (updated / visited infosets, pairs)
    long long ndef;
    int P;
    int variant;
    int upd_player;               // alternating updates (variant 4): the player updated by this pass; 0 = all
    double sc0, rc[3];            // 2^(40-E), 2^(E-40k): regret / BR sums
    double scp0, rcp[3];          // same with E = 1: pi_bar sums
};

// ---------------------------------------------------------------- exact sums
// Three 40-bit slices per term:
// c_k = rint(x * 2^(40k-E)), x <- x - c_k 2^(E-40k).  Implemented with FP64 adds
// only: y = x*2^(40-E) is exact; rint(y) = (y + 1.5*2^52) - 1.5*2^52 (round half
// to even, |y| < 2^51); y - c is exact and y' = (y - c) * 2^40 is the next slice's
// input, identical to x_k * 2^(40(k+1)-E).  The slices are integers, so partial
// sums of <= 2^13 of them are exact in binary64; they are converted to int64 only
// for global accumulation.  decode = ((C1 2^(E-40) + C2 2^(E-80)) + C3 2^(E-120)).
__device__ __forceinline__ double rint_magic(double y) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    return (y + M) - M;
}
__device__ __forceinline__ void xadd(double& a0, double& a1, double& a2, double x, double sc0) {
    double y = x * sc0;
    const double c0 = rint_magic(y);
    y = (y - c0) * 1099511627776.0;   // 2^40
    const double c1 = rint_magic(y);
    y = (y - c1) * 1099511627776.0;
    const double c2 = rint_magic(y);
    a0 += c0;
    a1 += c1;
    a2 += c2;
}
__device__ __forceinline__ double xdec(double c0, double c1, double c2, const double (&rc)[3]) {
    return (c0 * rc[0] + c1 * rc[1]) + c2 * rc[2];
}
__device__ __forceinline__ double xdec_ll(long long c0, long long c1, long long c2, const double (&rc)[3]) {
    return (__ll2double_rn(c0) * rc[0] + __ll2double_rn(c1) * rc[1]) + __ll2double_rn(c2) * rc[2];
}

// cp.async (LDGSTS): global -> shared without register staging, many in flight.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Programmatic dependent launch (PDL): a kernel lets its successor launch early
// (launch_dependents) and waits for its predecessor's completion + memory flush
// (wait) only before touching data the predecessor may write.  Both are no-ops
// without a programmatic dependency.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// L2 eviction-priority policies (createpolicy) for loads / stores with a cache hint:
// streams read or written once go first, small reused gather tables stay
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_normal() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
template <class T>
__device__ __forceinline__ T ld_hint(const T* p, unsigned long long pol);
template <>
__device__ __forceinline__ double ld_hint<double>(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ float ld_hint<float>(const float* p, unsigned long long pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;\n" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ int ld_hint<int>(const int* p, unsigned long long pol) {
    int v;
    asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;\n" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ long long ld_hint<long long>(const long long* p, unsigned long long pol) {
    long long v;
    asm volatile("ld.global.L2::cache_hint.s64 %0, [%1], %2;\n" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ unsigned char ld_hint<unsigned char>(const unsigned char* p, unsigned long long pol) {
    unsigned short v;
    asm volatile("ld.global.L2::cache_hint.u8 %0, [%1], %2;\n" : "=h"(v) : "l"(p), "l"(pol));
    return (unsigned char)v;
}
__device__ __forceinline__ void st_hint_v2(double2* p, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_hint_v2(float2* p, float2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
                 : "memory");
}

template <class R>
__device__ __forceinline__ bool finite_(R x) {
    return isfinite(x);
}

// Per-iteration update rule (cfr_solver_config.variant): 0 CFR (Eq 8/15
// cumulative, reading Q4), 1 CFR+ (RM+, w_t = t; reading Q6) and 4 its
// alternating-update form (reading Q19: same rule, one player per pass), 2 linear CFR and 3
// DCFR(3/2, 0, 2) -- Brown & Sandholm's discounting of Eq 14/15 (reading
// Q18): after iteration t's terms are added, positive regrets x t^a/(t^a+1),
// others x t^b/(t^b+1), both average-strategy sums x (t/(t+1))^g.  Only correctly
// rounded operations (t^(3/2) = t * sqrt(t)), so CPU and GPU agree bit for bit.
template <class R>
struct Upd {
    int variant;
    R w;                  // weight of pi_bar inside the average sums: t for CFR+, else 1
    R dpos, dneg, dsum;   // discount factors (variants 2, 3)
};
template <class R>
__device__ __forceinline__ Upd<R> make_upd(int variant, long long t) {
    Upd<R> u;
    u.variant = variant;
    u.w = (variant == 1 || variant == 4) ? (R)t : (R)1;
    u.dpos = u.dneg = u.dsum = (R)1;
    const R tt = (R)t;
    if (variant == 2) {
        const R f = tt / (tt + (R)1);
        u.dpos = f;
        u.dneg = f;
        u.dsum = f;
    } else if (variant == 3) {
        const R a = tt * sqrt(tt);
        u.dpos = a / (a + (R)1);
        u.dneg = (R)1 / ((R)1 + (R)1);
        const R f = tt / (tt + (R)1);
        u.dsum = f * f;
    }
    return u;
}
template <class R>
__device__ __forceinline__ R upd_regret(const Upd<R>& u, R reg, R rt) {
    const R x = reg + rt;
    if (u.variant == 0) return x;
    if (u.variant == 1 || u.variant == 4) {
        R r = (x > (R)0) ? x : (R)0;
        if (!finite_(x)) r = x;
        return r;
    }
    return (x > (R)0) ? x * u.dpos : x * u.dneg;
}
// S_num (add = (w pi_bar) sigma) or S_den (add = w pi_bar)
template <class R>
__device__ __forceinline__ R upd_sum(const Upd<R>& u, R s, R add) {
    return (u.variant == 2 || u.variant == 3) ? (s + add) * u.dsum : s + add;
}

// ------------------------------------------------------------ forward pass
// Decision nodes of one depth in canonical order (streaming reads of the
// parents' rows, streaming writes).  Eq 2: pi_check(v,i) =
// pi_check(parent,i) * (sigma if the parent's actor != i else 1); Eq 4 (P:97,
// reading Q1): pi_hat(v,i) = pi_hat(parent,i) * (sigma if actor == i else 1).
// compact != 0 (two players, the deepest decision level when its backward pass
// is the streaming kernel): no forward level reads these rows, and the backward
// pass needs only the acting player's pi_check and pi_hat -- 2 values per slot
// are written at reach + d_begin*2P + (d - d_begin)*2 instead of the 2P-value row.
template <class R, class I, int PT>
__device__ __forceinline__ void fwd_body(const DG<R, I>& g, const R* __restrict__ sig, long long d_begin,
                                         long long d_end, int compact) {
    const int P = (PT > 0) ? PT : g.P;
    const long long stride = (long long)gridDim.x * blockDim.x;
    pdl_trigger();
    if (PT == 2) {
        // two players: 4-value rows (32 B) moved as two 16-byte vectors; FW rows
        // per thread with every load issued before the first use (the parent rows
        // are gathers: memory-level parallelism, not bandwidth, bounds this pass)
#ifndef CFR_FWD_FW
#define CFR_FWD_FW 4
#endif
        constexpr int FW = CFR_FWD_FW;
        using V2 = typename std::conditional<sizeof(R) == 8, double2, float2>::type;
        const long long n = d_end - d_begin;
        const long long chunk = (long long)blockDim.x * FW;
#ifndef CFR_FWD_HINTS
#define CFR_FWD_HINTS 1
#endif
        const unsigned long long pf = CFR_FWD_HINTS ? policy_evict_first() : policy_evict_normal();
        const unsigned long long pl = CFR_FWD_HINTS ? policy_evict_last() : policy_evict_normal();
        pdl_wait();
        for (long long base = (long long)blockIdx.x * chunk; base < n; base += (long long)gridDim.x * chunk) {
            long long p[FW];
            long long e[FW];
            int act[FW], own[FW];
#pragma unroll
            for (int k = 0; k < FW; ++k) {
                const long long i = base + k * blockDim.x + threadIdx.x;
                const long long d = d_begin + (i < n ? i : 0);
                p[k] = (long long)ld_hint(g.f_parent + d, pf);
                e[k] = (long long)ld_hint(g.f_e + d, pf);
                act[k] = ld_hint(g.f_pact + d, pf);
                own[k] = compact ? (int)ld_hint(g.s_actor + d, pf) : 0;
            }
            V2 a[FW], b[FW];
            R x[FW];
#pragma unroll
            for (int k = 0; k < FW; ++k) {
                if (sizeof(R) == 8) {
                    // the whole 32-byte parent row in one 256-bit load (one L1 request)
                    double r0, r1, r2, r3;
                    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
                                 : "=d"(r0), "=d"(r1), "=d"(r2), "=d"(r3)
                                 : "l"(g.reach + p[k] * 4));
                    a[k].x = (R)r0;   // pi_check(1), pi_check(2)
                    a[k].y = (R)r1;
                    b[k].x = (R)r2;   // pi_hat(1), pi_hat(2)
                    b[k].y = (R)r3;
                } else {
                    const V2* src = reinterpret_cast<const V2*>(g.reach + p[k] * 4);
                    a[k] = src[0];
                    b[k] = src[1];
                }
                x[k] = ld_hint(sig + e[k], pl);   // the edge's sigma: reused by every member of the parent's infoset
            }
#pragma unroll
            for (int k = 0; k < FW; ++k) {
                const long long i = base + k * blockDim.x + threadIdx.x;
                if (i >= n) continue;
                V2 ca, cb;
                ca.x = (act[k] != 1) ? a[k].x * x[k] : a[k].x;
                ca.y = (act[k] != 2) ? a[k].y * x[k] : a[k].y;
                cb.x = (act[k] == 1) ? b[k].x * x[k] : b[k].x;
                cb.y = (act[k] == 2) ? b[k].y * x[k] : b[k].y;
                if (compact) {
                    // the slot's actor: (pi_check, pi_hat) of that player only
                    V2 c2;
                    c2.x = (own[k] == 2) ? ca.y : ca.x;
                    c2.y = (own[k] == 2) ? cb.y : cb.x;
                    st_hint_v2(reinterpret_cast<V2*>(g.reach + d_begin * 4 + i * 2), c2, pf);
                    continue;
                }
                if (sizeof(R) == 8) {
                    // the 32-byte row in one 256-bit store
                    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(
                                     g.reach + (d_begin + i) * 4),
                                 "d"((double)ca.x), "d"((double)ca.y), "d"((double)cb.x), "d"((double)cb.y), "l"(pf)
                                 : "memory");
                } else {
                    V2* dst = reinterpret_cast<V2*>(g.reach + (d_begin + i) * 4);
                    st_hint_v2(dst, ca, pf);
                    st_hint_v2(dst + 1, cb, pf);
                }
            }
        }
        return;
    }
    pdl_wait();
    for (long long d = d_begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; d < d_end; d += stride) {
        const long long p = (long long)g.f_parent[d];
        const R x = sig[g.f_e[d]];
        const int act = g.f_pact[d];
        const R* __restrict__ src = g.reach + p * 2 * P;
        R* __restrict__ dst = g.reach + d * 2 * P;
#pragma unroll
        for (int j = 0; j < ((PT > 0) ? PT : 16); ++j) {
            if (PT == 0 && j >= P) break;
            const R pc = src[j];
            const R ph = src[P + j];
            dst[j] = (act != j + 1) ? pc * x : pc;
            dst[P + j] = (act == j + 1) ? ph * x : ph;
        }
    }
}

template <class R, class I, int PT>
__global__ void __launch_bounds__(256) k_fwd(DG<R, I> g, const R* __restrict__ sig, long long d_begin,
                                             long long d_end, int compact) {
    fwd_body<R, I, PT>(g, sig, d_begin, d_end, compact);
}

// ----------------------------------------------------------- backward pass
// One CTA (kTileSlots threads) per tile of whole infosets.  Global memory is
// touched in three dependency steps only (metadata; reach + sigma + children +
// update state; writes), everything else runs out of shared memory.
struct SegS {
    long long h;     // internal infoset
    long long qb;    // qbase[h]
    long long dq, dh;  // compact accumulator indices (deferred)
    int sb, se;      // tile-local member slots
    int pair_off;    // first pair of the segment in the tile
    int n;           // |A(h)|
    int owner;       // acting player
    int fused;
};

// Shared-memory layout of one backward launch (per level: sized by the
// level's largest tile so small tiles leave room for more resident CTAs).
struct SmemLayout {
    int ch, sv, spc, sph, ssig, sreg, ssn, pib, zs, sden, seg, soff, best, scoff, spoff, sn, scb, pseg, cm, ccnt;
    int bytes;
};
template <class R>
struct TileView {
    R *ch, *sv, *spc, *sph, *ssig, *sreg, *ssn, *pib, *zs, *sden;
    SegS* seg;
    int *soff, *best, *scoff, *spoff, *sn;
    long long* scb;
    unsigned char* pseg;
    short* cm;     // per segment: members with nonzero pi_check (tile-local slots)
    int* ccnt;
};
template <class R>
__device__ __forceinline__ TileView<R> make_view(unsigned char* b, const SmemLayout& L) {
    TileView<R> v;
    v.ch = (R*)(b + L.ch);
    v.sv = (R*)(b + L.sv);
    v.spc = (R*)(b + L.spc);
    v.sph = (R*)(b + L.sph);
    v.ssig = (R*)(b + L.ssig);
    v.sreg = (R*)(b + L.sreg);
    v.ssn = (R*)(b + L.ssn);
    v.pib = (R*)(b + L.pib);
    v.zs = (R*)(b + L.zs);
    v.sden = (R*)(b + L.sden);
    v.seg = (SegS*)(b + L.seg);
    v.soff = (int*)(b + L.soff);
    v.best = (int*)(b + L.best);
    v.scoff = (int*)(b + L.scoff);
    v.spoff = (int*)(b + L.spoff);
    v.sn = (int*)(b + L.sn);
    v.scb = (long long*)(b + L.scb);
    v.pseg = (unsigned char*)(b + L.pseg);
    v.cm = (short*)(b + L.cm);
    v.ccnt = (int*)(b + L.ccnt);
    return v;
}

// rt / pos alias ch after phase B (the host sizes ch >= 2 * pairs)

__device__ __forceinline__ int seg_of_pair(const int* soff, int nseg, int p) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (soff[mid] <= p) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <class R, class I, int PC, int MODE>
__device__ __forceinline__ void bwd_tile(const DG<R, I>& g, const R* __restrict__ sig, long long tile, int br_player,
                                         int last, const SmemLayout& lay, unsigned char* smem_raw) {
    const TileView<R> sm = make_view<R>(smem_raw, lay);
    const TileD T = g.tiles[tile];
    const int nslot = (int)(T.s1 - T.s0);
    const int nseg = T.seg1 - T.seg0;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
    const int P = g.P;
    R* const rt = sm.ch;                  // valid after phase B
    R* const pos = sm.ch + (lay.sreg - lay.ssig) / (int)sizeof(R);  // = ch + (pairs capacity)
    const bool sig_staged = T.npairs <= kTilePairs;
    const bool staged = T.staged != 0;
    constexpr int CH = (sizeof(R) == 8) ? 16 : 8;     // cp.async chunk (bytes) of uniform tiles
    constexpr int CE = CH / (int)sizeof(R);            // elements per chunk

    // ---- step 1: per-slot metadata (thread = slot), owner reach, segment + run tables
    // (metadata is constant: loaded before waiting for the previous kernel)
    pdl_trigger();
    long long my_node = 0, my_cb = 0, my_eb = 0, my_dec = 0;
    int my_n = 0, my_actor = 0;
    if (tid < nslot) {
        const long long s = T.s0 + tid;
        my_node = (long long)g.s_node[s];
        my_cb = (long long)g.s_cb[s];
        my_n = g.s_n[s];
        my_eb = (long long)g.s_ebase[s];
        my_actor = g.s_actor[s];
        my_dec = (long long)g.s_dec[s];
        sm.scoff[tid] = g.s_coff[s];
        sm.scb[tid] = my_cb;
        sm.sn[tid] = my_n;
        sm.spoff[tid] = -1;
    }
    pdl_wait();
    const long long t_iter = (MODE == MODE_CFR) ? g.ctrl[0] + 1 : 0;
    if (tid < nslot && MODE != MODE_VALUES && my_actor >= 1) {
        sm.spc[tid] = g.reach[my_dec * 2 * P + (my_actor - 1)];
        sm.sph[tid] = g.reach[my_dec * 2 * P + P + (my_actor - 1)];
    }
    if (tid < nseg) {
        const SegD sg = g.segs[T.seg0 + tid];
        SegS ss;
        ss.h = sg.h;
        ss.qb = sg.qb;
        ss.dq = sg.dq;
        ss.dh = sg.dh;
        ss.n = sg.n;
        ss.owner = sg.owner;
        ss.sb = (int)(sg.sb - T.s0);
        ss.se = (int)(sg.se - T.s0);
        ss.pair_off = sg.pair_off;
        ss.fused = sg.fused;
        sm.seg[tid] = ss;
        sm.soff[tid] = sg.pair_off;
        if (MODE == MODE_CFR && sg.fused) sm.sden[tid] = g.sden[sg.h];
    }
    if (tid == 0) sm.soff[nseg] = T.npairs;
    __syncthreads();

    // ---- step 2: children (cp.async, every lane keeps issuing; nothing waits
    // until cp.async.wait_all), sigma and update state of the tile's pairs
    if (T.staged == 1) {
        // uniform rows: flat loop over 16-B (f64) / 8-B (f32) chunks, all lanes busy
        const int total = nslot * T.cpr;
        for (int c = tid; c < total; c += nth) {
            const int row = __float2int_rd(((float)c + 0.5f) * T.inv_cpr);
            const int k = c - row * T.cpr;
            cp_async<CH>(sm.ch + row * T.stride + k * CE, g.U + sm.scb[row] * PC + k * CE);
        }
    } else if (T.staged == 2) {
        // generic rows: a warp per row, lanes over the row's elements
        for (int ls = warp; ls < nslot; ls += nwarps) {
            const R* __restrict__ src = g.U + sm.scb[ls] * PC;
            R* dst = sm.ch + sm.scoff[ls];
            const int cnt = sm.sn[ls] * PC;
            for (int e = lane; e < cnt; e += 32) cp_async<(int)sizeof(R)>(dst + e, src + e);
        }
    }
    if (sig_staged) {
        for (int p = tid; p < T.npairs; p += nth) {
            const int k = seg_of_pair(sm.soff, nseg, p);
            sm.pseg[p] = (unsigned char)k;
            const long long q = sm.seg[k].qb + (p - sm.soff[k]);
            sm.ssig[p] = sig[q];
            if (MODE == MODE_CFR && sm.seg[k].fused) {
                sm.sreg[p] = g.regret[q];
                sm.ssn[p] = g.snum[q];
            }
        }
    }
    for (int k = warp; k < nseg; k += nwarps)
        for (int s = sm.seg[k].sb + lane; s < sm.seg[k].se; s += 32) sm.spoff[s] = sm.soff[k];
    cp_async_wait_all();
    __syncthreads();

    // ---- phase A: node values, Eq 1 in ascending action order from +0
    if (tid < nslot) {
        R v[PC];
#pragma unroll
        for (int j = 0; j < PC; ++j) v[j] = (R)0;
        const int po = sig_staged ? sm.spoff[tid] : -1;
        if (staged && po >= 0) {
            const R* row = sm.ch + sm.scoff[tid];
            const R* sg = sm.ssig + po;
            for (int a = 0; a < my_n; ++a) {
                const R x = sg[a];
#pragma unroll
                for (int j = 0; j < PC; ++j) v[j] = v[j] + x * row[a * PC + j];
            }
        } else {
            for (int a = 0; a < my_n; ++a) {
                const R x = (po >= 0) ? sm.ssig[po + a] : sig[my_eb + a];
#pragma unroll
                for (int j = 0; j < PC; ++j) {
                    const R u = staged ? sm.ch[sm.scoff[tid] + a * PC + j] : g.U[(my_cb + a) * PC + j];
                    v[j] = v[j] + x * u;
                }
            }
        }
        const bool skip = (MODE == MODE_BR) && (my_actor == br_player);
        if (!skip) {
#pragma unroll
            for (int j = 0; j < PC; ++j) g.U[my_node * PC + j] = v[j];
        }
#pragma unroll
        for (int j = 0; j < PC; ++j) sm.sv[tid * PC + j] = v[j];
    }
    if (MODE == MODE_VALUES) return;
    // members with pi_check == 0 add exact zeros to every sum: compact them away
    for (int k = warp; k < nseg; k += nwarps) {
        const int sb = sm.seg[k].sb, se = sm.seg[k].se;
        int cnt = 0;
        for (int base = sb; base < se; base += 32) {
            const int s2 = base + lane;
            const bool f = (s2 < se) && (sm.spc[s2] != (R)0);
            const unsigned m = __ballot_sync(0xffffffffu, f);
            if (f) sm.cm[sb + cnt + __popc(m & ((1u << lane) - 1u))] = (short)s2;
            cnt += __popc(m);
        }
        if (lane == 0) sm.ccnt[k] = cnt;
    }
    __syncthreads();

    // ---- phase B: exact sums.  Work items: every (infoset, action) pair (r~ or BR
    // sums) plus one pi_bar item per segment (CFR mode).  Each item is split over
    // `ns` adjacent lanes (members strided); partial slice sums are exact
    // integer-valued doubles combined with shuffles.  The player-2 sign of the
    // zero-sum storage (u2 = -u1) is applied to the sums: slices of -t are -slices of t.
    const int nitems = T.npairs + ((MODE == MODE_CFR) ? nseg : 0);
    int ns = 1;
    int lns = 0;                      // ns = 2^lns (shifts, no integer division)
    while (ns < 8 && nitems * ns * 2 <= nth) { ns <<= 1; ++lns; }
    const int rounds = (nitems * ns + nth - 1) / nth;
    double kr0 = 0, kr1 = 0, kr2 = 0, kr3 = 0, kr4 = 0;
    for (int rd = 0; rd < rounds; ++rd) {
        const int wi = rd * nth + tid;
        const int it = wi >> lns, part = wi & (ns - 1);
        double c0 = 0, c1 = 0, c2 = 0;
        int k = 0, a = 0;
        bool is_pair = false, neg = false, active = false;
        if (it < T.npairs) {
            k = sig_staged ? (int)sm.pseg[it] : seg_of_pair(sm.soff, nseg, it);
            a = it - sm.soff[k];
            is_pair = true;
            const int i = sm.seg[k].owner;
            active = !(MODE == MODE_BR && i != br_player);
            neg = (PC == 1) && (i == 2) && (MODE == MODE_CFR);
        } else if (it < nitems) {
            k = it - T.npairs;
            active = true;
        }
        if (active) {
            const SegS& sg = sm.seg[k];
            const int col = (PC == 1) ? 0 : sg.owner - 1;
            if (!is_pair) {
                for (int ls = sg.sb + part; ls < sg.se; ls += ns) xadd(c0, c1, c2, (double)sm.sph[ls], g.scp0);
            } else if (staged) {
                double e0 = 0, e1 = 0, e2 = 0;   // second independent chain (ILP)
                const short* mem = sm.cm + sg.sb;
                const int cnt = sm.ccnt[k];
                int j = part;
                for (; j + ns < cnt; j += 2 * ns) {
                    const int la = mem[j], lb = mem[j + ns];
                    const R ua = sm.ch[sm.scoff[la] + a * PC + col];
                    const R ub = sm.ch[sm.scoff[lb] + a * PC + col];
                    const R ta = (MODE == MODE_CFR) ? sm.spc[la] * (ua - sm.sv[la * PC + col]) : sm.spc[la] * ua;
                    const R tb = (MODE == MODE_CFR) ? sm.spc[lb] * (ub - sm.sv[lb * PC + col]) : sm.spc[lb] * ub;
                    xadd(c0, c1, c2, (double)ta, g.sc0);
                    xadd(e0, e1, e2, (double)tb, g.sc0);
                }
                if (j < cnt) {
                    const int la = mem[j];
                    const R ua = sm.ch[sm.scoff[la] + a * PC + col];
                    const R ta = (MODE == MODE_CFR) ? sm.spc[la] * (ua - sm.sv[la * PC + col]) : sm.spc[la] * ua;
                    xadd(c0, c1, c2, (double)ta, g.sc0);
                }
                c0 += e0;
                c1 += e1;
                c2 += e2;
            } else {
                const short* mem = sm.cm + sg.sb;
                for (int j = part; j < sm.ccnt[k]; j += ns) {
                    const int ls = mem[j];
                    const R uc = g.U[(sm.scb[ls] + a) * PC + col];
                    const R t = (MODE == MODE_CFR) ? sm.spc[ls] * (uc - sm.sv[ls * PC + col]) : sm.spc[ls] * uc;
                    xadd(c0, c1, c2, (double)t, g.sc0);
                }
            }
            if (neg) { c0 = -c0; c1 = -c1; c2 = -c2; }
        }
        // combine the ns partial sums (exact: integer-valued doubles < 2^53)
        for (int o = 1; o < ns; o <<= 1) {
            c0 += __shfl_xor_sync(0xffffffffu, c0, o);
            c1 += __shfl_xor_sync(0xffffffffu, c1, o);
            c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        }
        if (active && part == 0) {
            const bool keep = (MODE == MODE_BR) || sm.seg[k].fused;
            if (keep) {
                const double x = is_pair ? xdec(c0, c1, c2, g.rc) : xdec(c0, c1, c2, g.rcp);
                if (rd == 0) kr0 = x;
                else if (rd == 1) kr1 = x;
                else if (rd == 2) kr2 = x;
                else if (rd == 3) kr3 = x;
                else kr4 = x;
            } else if (MODE == MODE_CFR && T.contrib) {
                if (is_pair) {
                    const long long q = sm.seg[k].dq + a;
                    atomicAdd(&g.acc_r[q * 3 + 0], (unsigned long long)(long long)c0);
                    atomicAdd(&g.acc_r[q * 3 + 1], (unsigned long long)(long long)c1);
                    atomicAdd(&g.acc_r[q * 3 + 2], (unsigned long long)(long long)c2);
                } else {
                    const long long h = sm.seg[k].dh;
                    atomicAdd(&g.acc_p[h * 3 + 0], (unsigned long long)(long long)c0);
                    atomicAdd(&g.acc_p[h * 3 + 1], (unsigned long long)(long long)c1);
                    atomicAdd(&g.acc_p[h * 3 + 2], (unsigned long long)(long long)c2);
                }
            }
        }
    }
    __syncthreads();   // all reads of sm.ch done: rt / pos alias it from here on
    if (sig_staged) {
        for (int rd = 0; rd < rounds && rd < 5; ++rd) {
            const int wi = rd * nth + tid;
            const int it = wi >> lns, part = wi & (ns - 1);
            if (it < nitems && part == 0) {
                const double x = rd == 0 ? kr0 : rd == 1 ? kr1 : rd == 2 ? kr2 : rd == 3 ? kr3 : kr4;
                if (it < T.npairs) rt[it] = (R)x;
                else sm.pib[it - T.npairs] = (R)x;
            }
        }
    }
    __syncthreads();

    if (MODE == MODE_BR) {
        // argmax per segment (ties to the lowest action); for u2 = -u1 storage the
        // stored sums are negated, so player 2 takes the argmin.
        for (int k = tid; k < nseg; k += nth) {
            if (sm.seg[k].owner != br_player) continue;
            const int n = sm.seg[k].n;
            const bool neg = (PC == 1) && (br_player == 2);
            int best = 0;
            R bv = rt[sm.soff[k]];
            for (int a = 1; a < n; ++a) {
                const R x = rt[sm.soff[k] + a];
                if (neg ? (x < bv) : (x > bv)) { bv = x; best = a; }
            }
            sm.best[k] = best;
        }
        __syncthreads();
        for (int k = 0; k < nseg; ++k) {
            if (sm.seg[k].owner != br_player) continue;
            const int best = sm.best[k];
            for (int ls = sm.seg[k].sb + tid; ls < sm.seg[k].se; ls += nth) {
                const long long s = T.s0 + ls;
                const long long src = ((long long)g.s_cb[s] + best) * PC;
                const long long dst = (long long)g.s_node[s] * PC;
#pragma unroll
                for (int j = 0; j < PC; ++j) g.U[dst + j] = g.U[src + j];
            }
        }
        return;
    }

    // ---- phase C: fused update of complete single-depth infosets
    const Upd<R> up = make_upd<R>(g.variant, t_iter);
    const R w = up.w;
    if (!sig_staged) {   // split tile: every segment is deferred
        if (last) {
            __syncthreads();
            if (tid == 0) g.ctrl[0] = t_iter;
        }
        return;
    }
    auto upd_seg = [&](int k) {   // fused and (alternating updates) owned by this pass's player
        return sm.seg[k].fused && (g.upd_player == 0 || sm.seg[k].owner == g.upd_player);
    };
    for (int p = tid; p < T.npairs; p += nth) {
        const int k = sm.pseg[p];
        if (!upd_seg(k)) continue;
        const long long q = sm.seg[k].qb + (p - sm.soff[k]);
        const R r_t = rt[p];
        const R r = upd_regret(up, sm.sreg[p], r_t);   // Eq 8/15 (Q4) / CFR+ (Q6) / Q18
        g.regret[q] = r;
        const R wp = w * sm.pib[k];
        g.snum[q] = upd_sum(up, sm.ssn[p], wp * sm.ssig[p]);   // Eq 10 numerator
        pos[p] = (r > (R)0) ? r : (R)0;
    }
    __syncthreads();
    for (int k = tid; k < nseg; k += nth) {
        if (!upd_seg(k)) continue;
        g.sden[sm.seg[k].h] = upd_sum(up, sm.sden[k], w * sm.pib[k]);   // Eq 10 denominator
        R z = (R)0;
        for (int p = sm.soff[k]; p < sm.soff[k + 1]; ++p) z = z + pos[p];
        sm.zs[k] = z;
    }
    __syncthreads();
    bool bad = false;
    for (int p = tid; p < T.npairs; p += nth) {
        const int k = sm.pseg[p];
        if (!upd_seg(k)) continue;
        const int a = p - sm.soff[k];
        const R z = sm.zs[k];
        const R nsig = (z > (R)0) ? pos[p] / z : (R)1 / (R)sm.seg[k].n;   // Eq 9
        g.sig[sm.seg[k].qb + a] = nsig;
        if (!finite_(rt[p]) || !finite_(nsig) || !finite_(z)) bad = true;
    }
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (last) {
        __syncthreads();
        if (tid == 0) g.ctrl[0] = t_iter;
    }
}

template <class R, class I, int PC, int MODE>
__global__ void __launch_bounds__(kTileSlots) k_bwd(DG<R, I> g, const R* __restrict__ sig, long long tile0,
                                                    int br_player, int last, SmemLayout lay) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    bwd_tile<R, I, PC, MODE>(g, sig, tile0 + blockIdx.x, br_player, last, lay, smem_raw);
}

// ------------------------------------------------- pipelined backward pass
// Persistent variant of k_bwd (MODE_CFR) for levels whose tiles are all "fast":
// uniform child rows staged in 16/8-byte chunks, every infoset complete in its
// tile (fused update), no chance nodes.  Each CTA walks tiles blockIdx.x,
// blockIdx.x + gridDim.x, ... with a three-stage cp.async pipeline: while tile i
// is computed, the data of tile i+1 and the metadata record of tile i+2 are in
// flight, so the global-memory latency of one tile hides behind another's work.
// The arithmetic is the same as k_bwd's (same order of every FP operation).
struct FastHdr {
    long long s0;    // first slot
    int nslot, nseg, npairs, pad;
};
struct FastSeg {
    long long h, qb;
    int pair_off, n, owner, sb, se, pad;
};
struct FastLevel {
    long long tile0, ntiles;   // tiles of the level
    long long rec;             // byte offset of the level's records in the record pool
    int recsize;               // bytes per record (16-byte multiple)
    int maxslot, maxseg, maxpairs, maxch;
    int rowlen, cpr, stride;   // uniform child rows
    float inv_cpr;
    int last;                  // 1: this launch ends the iteration
    int pad;
};

// Shared-memory plan of k_bwd_fast: 3 metadata records, 2 data buffers (each
// holding ch | ssig | sreg | ssn | spc | sph | sden), then per-tile work arrays.
// Buffers are addressed as base + index * stride (no dynamically indexed
// pointer arrays, which would live in local memory).
struct FastPlan {
    int meta, mstride;        // meta record k at meta + k * mstride
    int data, dstride;        // data buffer k at data + k * dstride
    int o_ssig, o_sreg, o_ssn, o_spc, o_sph, o_sden;   // offsets inside a data buffer
    int sv, pib, zs, spoff, pseg, cm, ccnt;
    int bytes;
};
__host__ __device__ inline FastPlan fast_plan(const FastLevel& L, int Pc, int w) {
    FastPlan f;
    auto al = [](int x) { return (x + 15) & ~15; };
    const int pairs_b = al(L.maxpairs * w);
    f.meta = 0;
    f.mstride = al(L.recsize);
    f.data = 3 * f.mstride;
    int o = al(L.maxch * w > 2 * pairs_b ? L.maxch * w : 2 * pairs_b);
    f.o_ssig = o; o += pairs_b;
    f.o_sreg = o; o += pairs_b;
    f.o_ssn = o; o += pairs_b;
    f.o_spc = o; o += al(L.maxslot * w);
    f.o_sph = o; o += al(L.maxslot * w);
    f.o_sden = o; o += al(L.maxseg * w);
    f.dstride = o;
    int x = f.data + 2 * f.dstride;
    f.sv = x; x += al(L.maxslot * Pc * w);
    f.pib = x; x += al(L.maxseg * w);
    f.zs = x; x += al(L.maxseg * w);
    f.spoff = x; x += al(L.maxslot * 4);
    f.pseg = x; x += al(L.maxpairs);
    f.cm = x; x += al(L.maxslot * 2);
    f.ccnt = x; x += al(L.maxseg * 4);
    f.bytes = x;
    return f;
}

// t = tile index within the level (records are level-local)
template <class R, class I, int PC>
__device__ __forceinline__ void fast_issue_meta(const unsigned char* __restrict__ pool, const FastLevel& L, long long t,
                                                unsigned char* dst) {
    const unsigned char* src = pool + L.rec + t * (long long)L.recsize;
    for (int c = threadIdx.x; c < L.recsize / 16; c += blockDim.x) cp_async<16>(dst + c * 16, src + c * 16);
}

template <class R, class I, int PC>
__device__ __forceinline__ void fast_issue_data(const DG<R, I>& g, const FastLevel& L, const unsigned char* meta,
                                                R* ch, R* ssig, R* sreg, R* ssn, R* spc, R* sph, R* sden) {
    constexpr int CH = (sizeof(R) == 8) ? 16 : 8;
    constexpr int CE = CH / (int)sizeof(R);
    const FastHdr& hd = *reinterpret_cast<const FastHdr*>(meta);
    const FastSeg* seg = reinterpret_cast<const FastSeg*>(meta + 32);
    const I* node = reinterpret_cast<const I*>(meta + 32 + hd.nseg * (int)sizeof(FastSeg));
    const I* cb = node + hd.nslot;
    const I* dec = cb + hd.nslot;
    const unsigned char* sseg = reinterpret_cast<const unsigned char*>(dec + hd.nslot);
    const unsigned char* pseg = sseg + hd.nslot;
    (void)node;
    const int P = g.P;
    {
        // 2-D walk: thread -> (row r0 + j * rpp, chunk k), no per-chunk division
        const int rpp = blockDim.x / L.cpr;
        const int r0 = threadIdx.x / L.cpr, k = threadIdx.x - r0 * L.cpr;
        if (r0 < rpp)
            for (int row = r0; row < hd.nslot; row += rpp)
                cp_async<CH>(ch + row * L.stride + k * CE, g.U + (long long)cb[row] * PC + k * CE);
    }
    for (int s = threadIdx.x; s < hd.nslot; s += blockDim.x) {
        const int k = sseg[s];
        const long long d = (long long)dec[s];
        const int i = seg[k].owner;
        cp_async<(int)sizeof(R)>(spc + s, g.reach + d * 2 * P + (i - 1));
        cp_async<(int)sizeof(R)>(sph + s, g.reach + d * 2 * P + P + (i - 1));
    }
    for (int p = threadIdx.x; p < hd.npairs; p += blockDim.x) {
        const int k = pseg[p];
        const long long q = seg[k].qb + (p - seg[k].pair_off);
        cp_async<(int)sizeof(R)>(ssig + p, g.sig + q);
        cp_async<(int)sizeof(R)>(sreg + p, g.regret + q);
        cp_async<(int)sizeof(R)>(ssn + p, g.snum + q);
    }
    for (int k = threadIdx.x; k < hd.nseg; k += blockDim.x) cp_async<(int)sizeof(R)>(sden + k, g.sden + seg[k].h);
    asm volatile("cp.async.commit_group;\n" ::);
}

template <class R, class I, int PC>
__global__ void __launch_bounds__(2 * kTileSlots, 4) k_bwd_fast(DG<R, I> g, const unsigned char* __restrict__ pool,
                                                         FastLevel L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const FastPlan F = fast_plan(L, PC, (int)sizeof(R));
    unsigned char* const B = smem_raw;
    auto META = [&](int k) { return B + F.meta + k * F.mstride; };
    auto DATA = [&](int k) { return B + F.data + k * F.dstride; };
    R* const sv_ = (R*)(B + F.sv);
    R* const pib_ = (R*)(B + F.pib);
    R* const zs_ = (R*)(B + F.zs);
    int* const spoff_ = (int*)(B + F.spoff);
    unsigned char* const pseg_ = B + F.pseg;
    short* const cm_ = (short*)(B + F.cm);      // members with nonzero pi_check, per segment
    int* const ccnt_ = (int*)(B + F.ccnt);
    auto ISSUE = [&](int mk, int dk) {
        unsigned char* d = DATA(dk);
        fast_issue_data<R, I, PC>(g, L, META(mk), (R*)d, (R*)(d + F.o_ssig), (R*)(d + F.o_sreg), (R*)(d + F.o_ssn),
                                  (R*)(d + F.o_spc), (R*)(d + F.o_sph), (R*)(d + F.o_sden));
    };
    const int tid = threadIdx.x, nth = blockDim.x;
    pdl_trigger();
    long long t = blockIdx.x;
    if (t >= L.ntiles) return;
    // prologue: meta(t) (constant records: before the PDL wait) -> data(t), meta(t + G)
    fast_issue_meta<R, I, PC>(pool, L, t, META(0));
    asm volatile("cp.async.commit_group;\n" ::);
    pdl_wait();
    const long long t_iter = g.ctrl[0] + 1;
    const Upd<R> up = make_upd<R>(g.variant, t_iter);
    const R w = up.w;
    cp_async_wait_all();
    __syncthreads();
    ISSUE(0, 0);
    if (t + gridDim.x < L.ntiles) fast_issue_meta<R, I, PC>(pool, L, t + gridDim.x, META(1));
    asm volatile("cp.async.commit_group;\n" ::);
    bool bad = false;
    for (int it = 0;; ++it) {
        const int mb = it % 3, db = it & 1;
        const long long tn = t + gridDim.x, tnn = t + 2 * (long long)gridDim.x;
        cp_async_wait_all();      // data(t) and meta(tn) have landed
        __syncthreads();
        if (tn < L.ntiles) {
            ISSUE((it + 1) % 3, db ^ 1);
            if (tnn < L.ntiles) fast_issue_meta<R, I, PC>(pool, L, tnn, META((it + 2) % 3));
            asm volatile("cp.async.commit_group;\n" ::);
        }
        // ---- compute tile t
        const unsigned char* meta = META(mb);
        const FastHdr hd = *reinterpret_cast<const FastHdr*>(meta);
        const FastSeg* seg = reinterpret_cast<const FastSeg*>(meta + 32);
        const I* node = reinterpret_cast<const I*>(meta + 32 + hd.nseg * (int)sizeof(FastSeg));
        const unsigned char* rsseg = reinterpret_cast<const unsigned char*>(node + 3 * hd.nslot);
        const unsigned char* rpseg = rsseg + hd.nslot;
        unsigned char* dbuf = DATA(db);
        R* ch = (R*)dbuf;
        const R* ssig = (const R*)(dbuf + F.o_ssig);
        const R* sreg = (const R*)(dbuf + F.o_sreg);
        const R* ssn = (const R*)(dbuf + F.o_ssn);
        const R* spc = (const R*)(dbuf + F.o_spc);
        const R* sph = (const R*)(dbuf + F.o_sph);
        const R* sden = (const R*)(dbuf + F.o_sden);
        const int nslot = hd.nslot, nseg = hd.nseg, npairs = hd.npairs;
        (void)pseg_;
        (void)spoff_;
        // phase A: node values (Eq 1), ascending actions from +0
        if (tid < nslot) {
            R v[PC];
#pragma unroll
            for (int j = 0; j < PC; ++j) v[j] = (R)0;
            const R* row = ch + tid * L.stride;
            const R* sg = ssig + seg[rsseg[tid]].pair_off;
            const int n = L.rowlen / PC;
            for (int a = 0; a < n; ++a) {
                const R x = sg[a];
#pragma unroll
                for (int j = 0; j < PC; ++j) v[j] = v[j] + x * row[a * PC + j];
            }
            const long long nd = (long long)node[tid];
#pragma unroll
            for (int j = 0; j < PC; ++j) {
                g.U[nd * PC + j] = v[j];
                sv_[tid * PC + j] = v[j];
            }
        }
        // members whose pi_check is zero contribute exact zeros to every r~ sum
        // (slices of +-0 are 0): compact them away (warp ballot per segment)
        {
            const int lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
            for (int k = warp; k < nseg; k += nwarps) {
                const int sb = seg[k].sb, se = seg[k].se;
                int cnt = 0;
                for (int base = sb; base < se; base += 32) {
                    const int s2 = base + lane;
                    const bool f = (s2 < se) && (spc[s2] != (R)0);
                    const unsigned m = __ballot_sync(0xffffffffu, f);
                    if (f) cm_[sb + cnt + __popc(m & ((1u << lane) - 1u))] = (short)s2;
                    cnt += __popc(m);
                }
                if (lane == 0) ccnt_[k] = cnt;
            }
        }
        __syncthreads();
        // phase B: exact sums (pairs, then one pi_bar item per segment)
        const int nitems = npairs + nseg;
        int ns = 1;
        int lns = 0;                  // ns = 2^lns (shifts, no integer division)
        while (ns < 8 && nitems * ns * 2 <= nth) { ns <<= 1; ++lns; }
        const int rounds = (nitems * ns + nth - 1) / nth;
        double kr0 = 0, kr1 = 0, kr2 = 0, kr3 = 0, kr4 = 0;
        for (int rd = 0; rd < rounds; ++rd) {
            const int wi = rd * nth + tid;
            const int itm = wi >> lns, part = wi & (ns - 1);
            double c0 = 0, c1 = 0, c2 = 0;
            bool is_pair = false, neg = false;
            int k = 0, a = 0;
            if (itm < npairs) {
                k = rpseg[itm];
                a = itm - seg[k].pair_off;
                is_pair = true;
                neg = (PC == 1) && (seg[k].owner == 2);
            } else if (itm < nitems) {
                k = itm - npairs;
            }
            if (itm < nitems) {
                const int col = (PC == 1) ? 0 : seg[k].owner - 1;
                const int sb = seg[k].sb, se = seg[k].se;
                if (!is_pair) {
                    for (int ls = sb + part; ls < se; ls += ns) xadd(c0, c1, c2, (double)sph[ls], g.scp0);
                } else {
                    // two independent slice chains (ILP); integer-valued partial sums
                    // combine exactly
                    double e0 = 0, e1 = 0, e2 = 0;
                    const short* mem = cm_ + sb;
                    const int cnt = ccnt_[k];
                    int j = part;
                    for (; j + ns < cnt; j += 2 * ns) {
                        const int la = mem[j], lb = mem[j + ns];
                        const R ua = ch[la * L.stride + a * PC + col];
                        const R ub = ch[lb * L.stride + a * PC + col];
                        const R ta = spc[la] * (ua - sv_[la * PC + col]);
                        const R tb = spc[lb] * (ub - sv_[lb * PC + col]);
                        xadd(c0, c1, c2, (double)ta, g.sc0);
                        xadd(e0, e1, e2, (double)tb, g.sc0);
                    }
                    if (j < cnt) {
                        const int la = mem[j];
                        const R ua = ch[la * L.stride + a * PC + col];
                        const R ta = spc[la] * (ua - sv_[la * PC + col]);
                        xadd(c0, c1, c2, (double)ta, g.sc0);
                    }
                    c0 += e0;
                    c1 += e1;
                    c2 += e2;
                }
                if (neg) { c0 = -c0; c1 = -c1; c2 = -c2; }
            }
            for (int o = 1; o < ns; o <<= 1) {
                c0 += __shfl_xor_sync(0xffffffffu, c0, o);
                c1 += __shfl_xor_sync(0xffffffffu, c1, o);
                c2 += __shfl_xor_sync(0xffffffffu, c2, o);
            }
            if (itm < nitems && part == 0) {
                const double x = is_pair ? xdec(c0, c1, c2, g.rc) : xdec(c0, c1, c2, g.rcp);
                if (rd == 0) kr0 = x;
                else if (rd == 1) kr1 = x;
                else if (rd == 2) kr2 = x;
                else if (rd == 3) kr3 = x;
                else kr4 = x;
            }
        }
        __syncthreads();   // reads of ch done: rt / pos alias it
        R* rt = ch;
        R* pos = ch + (((npairs * (int)sizeof(R) + 15) & ~15) / (int)sizeof(R));
        for (int rd = 0; rd < rounds && rd < 5; ++rd) {
            const int wi = rd * nth + tid;
            const int itm = wi >> lns, part = wi & (ns - 1);
            if (itm < nitems && part == 0) {
                const double x = rd == 0 ? kr0 : rd == 1 ? kr1 : rd == 2 ? kr2 : rd == 3 ? kr3 : kr4;
                if (itm < npairs) rt[itm] = (R)x;
                else pib_[itm - npairs] = (R)x;
            }
        }
        __syncthreads();
        // phase C: fused update (Eq 8/15 or CFR+, Eq 10, Eq 9)
        for (int p = tid; p < npairs; p += nth) {
            const int k = rpseg[p];
            if (g.upd_player != 0 && seg[k].owner != g.upd_player) continue;   // alternating updates
            const long long q = seg[k].qb + (p - seg[k].pair_off);
            const R r_t = rt[p];
            const R r = upd_regret(up, sreg[p], r_t);
            g.regret[q] = r;
            const R wp = w * pib_[k];
            g.snum[q] = upd_sum(up, ssn[p], wp * ssig[p]);
            pos[p] = (r > (R)0) ? r : (R)0;
        }
        __syncthreads();
        for (int k = tid; k < nseg; k += nth) {
            if (g.upd_player != 0 && seg[k].owner != g.upd_player) continue;
            g.sden[seg[k].h] = upd_sum(up, sden[k], w * pib_[k]);
            R z = (R)0;
            for (int p = seg[k].pair_off; p < seg[k].pair_off + seg[k].n; ++p) z = z + pos[p];
            zs_[k] = z;
        }
        __syncthreads();
        for (int p = tid; p < npairs; p += nth) {
            const int k = rpseg[p];
            if (g.upd_player != 0 && seg[k].owner != g.upd_player) continue;
            const int a = p - seg[k].pair_off;
            const R z = zs_[k];
            const R nsig = (z > (R)0) ? pos[p] / z : (R)1 / (R)seg[k].n;
            g.sig[seg[k].qb + a] = nsig;
            if (!finite_(rt[p]) || !finite_(nsig) || !finite_(z)) bad = true;
        }
        __syncthreads();   // buffers of tile t may be refilled from here on
        t = tn;
        if (t >= L.ntiles) break;
    }
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (L.last) {
        // last-block-done: the iteration counter advances once every CTA is done
        if (tid == 0) {
            __threadfence();
            const unsigned long long prev = atomicAdd((unsigned long long*)&g.ctrl[2], 1ULL);
            if (prev == gridDim.x - 1) {
                g.ctrl[0] = t_iter;
                g.ctrl[2] = 0;
            }
        }
    }
}

// ------------------------------------------------- streaming backward pass
// k_bwd_stream (MODE_CFR) serves levels whose slots are all player nodes with one
// |A(h)| = n and whose infosets are complete in the level (fused update).  In the
// slot-ordered device layout (u_rows) a tile of whole infosets reads ONE
// contiguous block from every stream: child rows, reach rows, sigma / R / S_num of
// its (h, a) pairs, S_den / owner of its infosets and the infosets' member starts.
// A producer warp moves the blocks with TMA bulk copies (cp.async.bulk, mbarrier
// complete_tx) into an S-stage ring; eight consumer warps compute the tile: Eq 1
// values (phase A), exact sums of the cancelled-form regret terms (Eq 7, matrix
// form P:313) and of pi_hat (Eq 5) (phase B), and the fused update Eq 8/15 + Eq 10
// + Eq 9 (phase C).  Every FP operation and its order is k_bwd's.
struct StreamLevel {
    long long s0;           // first slot of the level
    long long h0, q0;       // first internal infoset of the level, qbase[h0]
    long long row0;         // U row of the level's first child row
    long long ntiles;
    long long rec;          // int4 offset of the level's tile records {k0, k1, m0, m1} in the pool
    long long hs;           // int offset of the level's infoset member starts hs[nh + 1] in the pool
    int n, rowlen;          // |A(h)|, n * Pc
    int maxm, maxseg;       // per-tile maxima (members, infosets)
    int stages, stage_bytes;
    int o_rows, o_reach, o_sig, o_reg, o_snum, o_sden, o_own, o_hs, o_node;   // byte offsets inside a stage
    int fused;              // 1: deepest decision level -- its forward pass (Eq 2 / Eq 4) is fused here
    int o_pact, o_gsig;     // fused: parent actors, gathered incoming-edge sigma (reach area = parent rows)
    unsigned ndiv_m;        // p / n == (p * ndiv_m) >> ndiv_s (64-bit) for p < 2^16 (host-verified)
    int ndiv_s;
    int umem;               // > 0: every infoset of the level has umem members (m / umem by udiv)
    unsigned udiv_m;
    int udiv_s;
    int o_sv, o_cm, o_rt, o_pos, o_pib, o_zs, o_ccnt, o_bar;          // work arrays / barriers
    int bytes;              // dynamic shared memory
    int last;
    int debug;              // timing experiments only: 1 consumers skip compute, 2 producer skips loads
    int level;              // parent level (work counters)
    int compact;            // 1: reach rows of this level are compact (pi_check, pi_hat of the actor; k_fwd compact)
};
constexpr int kStreamConsumers = 256;   // 8 consumer warps
constexpr int kStreamThreads = kStreamConsumers + 32;   // + 1 producer warp

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(void* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy of a 16-byte-aligned window; completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, void* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kStreamConsumers) : "memory"); }

// 16-byte window [lo, hi) around [p, p + bytes): returns lo, sets the window size
// and the element offset of p inside it
template <class T>
__device__ __forceinline__ const unsigned char* window16(const T* p, long long count, unsigned* wbytes, int* off) {
    const unsigned long long a = (unsigned long long)p;
    const unsigned long long lo = a & ~15ull;
    const unsigned long long hi = (a + (unsigned long long)count * sizeof(T) + 15ull) & ~15ull;
    *wbytes = (unsigned)(hi - lo);
    *off = (int)((a - lo) / sizeof(T));
    return reinterpret_cast<const unsigned char*>(lo);
}

#ifdef CFR_STREAM_PROFILE
__device__ unsigned long long g_stream_prof[80];   // [warp][8] cycles, [64] tiles
extern "C" int cfr_debug_stream_profile(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_stream_prof, sizeof(g_stream_prof));
    if (reset) {
        unsigned long long z[80] = {0};
        cudaMemcpyToSymbol(g_stream_prof, z, sizeof(z));
    }
    return 0;
}
#endif
struct StreamHdr {
    int k0, nseg, m0, M;        // first infoset (level-relative), infosets, first member, members
    int po, ho, oo, hso;        // element offsets inside the windows: pairs, S_den, owner, hs
    int no, pao, ro, rro;       // node-row / parent-actor / child-row / reach-row window offsets
};

#ifndef CFR_STREAM_MINB
#define CFR_STREAM_MINB 2
#endif
template <class R, class I, int PC>
__global__ void __launch_bounds__(kStreamThreads, CFR_STREAM_MINB) k_bwd_stream(DG<R, I> g, const int* __restrict__ pool,
                                                                   StreamLevel L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char* const B = smem_raw;
    unsigned long long* const full = reinterpret_cast<unsigned long long*>(B + L.o_bar);
    unsigned long long* const empty = full + L.stages;
    const int tid = threadIdx.x;
    const int P = g.P;
    const int n = L.n;
    pdl_trigger();
    if (tid == 0) {
        for (int s = 0; s < L.stages; ++s) {
            mbar_init(&full[s], L.fused ? 33 : 1);   // fused: + the producer lanes' cp.async arrivals
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    {
        int* ccnt = reinterpret_cast<int*>(B + L.o_ccnt);
        for (int k = tid; k < 4 * L.maxseg; k += blockDim.x) ccnt[k] = 0;   // two tile buffers
    }
    __syncthreads();
    pdl_wait();
    const long long G = gridDim.x;

    if (tid >= kStreamConsumers) {
        // ------------------------------------------------------------ producer
        // Lane 0 arms the stage and issues the TMA bulk copies.  On the fused level
        // all 32 lanes also gather each member's parent reach row and incoming-edge
        // sigma (cp.async, completion counted on the same barrier); the parent /
        // edge indices of the next tile are prefetched into registers meanwhile.
        const int plane = tid - kStreamConsumers;
        if (!L.fused && plane != 0) return;   // lane 0 alone issues
        const int4* recs = reinterpret_cast<const int4*>(pool) + L.rec;
        const int* hs = pool + L.hs;
        constexpr int GMAX = kStreamConsumers / 32;   // members per lane (maxm <= kStreamConsumers)
        long long t = blockIdx.x;
        int4 rec = (t < L.ntiles) ? recs[t] : make_int4(0, 0, 0, 0);
        long long fp[GMAX], fe[GMAX];
        auto prefetch = [&](const int4& r) {
#pragma unroll
            for (int q = 0; q < GMAX; ++q) {
                const int m = q * 32 + plane;
                const long long s = L.s0 + r.z + m;
                fp[q] = (m < r.w - r.z) ? (long long)g.f_parent[s] : 0;
                fe[q] = (m < r.w - r.z) ? (long long)g.f_e[s] : 0;
            }
        };
        if (L.fused && t < L.ntiles) prefetch(rec);
        int st = 0;
        unsigned ph = 0;   // ring pass (parity of the empty barrier's phase to wait for)
        for (int it = 0; t < L.ntiles; ++it, t += G) {
            const int4 cur = rec;
            if (t + G < L.ntiles) rec = recs[t + G];    // next record in flight during the wait
            if (it >= L.stages) mbar_wait(&empty[st], (ph - 1u) & 1u);
            unsigned char* S = B + (size_t)st * L.stage_bytes;
            const int k0 = cur.x, k1 = cur.y, m0 = cur.z, m1 = cur.w;
            const int nseg = k1 - k0, M = m1 - m0;
            const long long slot = L.s0 + m0;
            if (plane == 0) {
                const long long q = L.q0 + (long long)k0 * n;
                const long long h = L.h0 + k0;
                unsigned b_rows, b_reach = 0, b_sig, b_reg, b_snum, b_sden, b_own, b_hs, b_node, b_pact = 0;
                int o_rows, o_reach = 0, po, po2, po3, ho, oo, hso, no, pao = 0;
                const unsigned char* w_rows = window16(g.U + (L.row0 + (long long)m0 * n) * PC, (long long)M * L.rowlen, &b_rows, &o_rows);
                const unsigned char* w_reach = nullptr;
                const unsigned char* w_pact = nullptr;
                if (L.fused) w_pact = window16(g.f_pact + slot, M, &b_pact, &pao);
                else if (L.compact) w_reach = window16(g.reach + L.s0 * 2 * P + (long long)m0 * 2, (long long)M * 2, &b_reach, &o_reach);
                else w_reach = window16(g.reach + slot * 2 * P, (long long)M * 2 * P, &b_reach, &o_reach);
                const unsigned char* w_sig = window16(g.sig + q, (long long)nseg * n, &b_sig, &po);
                const unsigned char* w_reg = window16(g.regret + q, (long long)nseg * n, &b_reg, &po2);
                const unsigned char* w_snum = window16(g.snum + q, (long long)nseg * n, &b_snum, &po3);
                const unsigned char* w_sden = window16(g.sden + h, nseg, &b_sden, &ho);
                const unsigned char* w_own = window16(g.owner + h, nseg, &b_own, &oo);
                const unsigned char* w_hs = window16(hs + k0, nseg + 1, &b_hs, &hso);
                const unsigned char* w_node = window16(g.s_node + slot, M, &b_node, &no);
                StreamHdr* hd = reinterpret_cast<StreamHdr*>(S);
                hd->k0 = k0;
                hd->nseg = nseg;
                hd->m0 = m0;
                hd->M = M;
                hd->po = po;
                hd->ho = ho;
                hd->oo = oo;
                hd->hso = hso;
                hd->no = no;
                hd->pao = pao;
                hd->ro = o_rows;
                hd->rro = o_reach;
                (void)po2; (void)po3;   // sigma / R / S_num share the pair window offset (same base alignment)
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                if (L.debug == 2) {   // timing experiment: no loads (consumers compute on stale data)
                    mbar_expect_tx(&full[st], 0);
                } else {
                    mbar_expect_tx(&full[st], b_rows + b_reach + b_sig + b_reg + b_snum + b_sden + b_own + b_hs + b_node + b_pact);
                    bulk_g2s(S + L.o_node, w_node, b_node, &full[st]);
                    bulk_g2s(S + L.o_rows, w_rows, b_rows, &full[st]);
                    if (L.fused) bulk_g2s(S + L.o_pact, w_pact, b_pact, &full[st]);
                    else bulk_g2s(S + L.o_reach, w_reach, b_reach, &full[st]);
                    bulk_g2s(S + L.o_sig, w_sig, b_sig, &full[st]);
                    bulk_g2s(S + L.o_reg, w_reg, b_reg, &full[st]);
                    bulk_g2s(S + L.o_snum, w_snum, b_snum, &full[st]);
                    bulk_g2s(S + L.o_sden, w_sden, b_sden, &full[st]);
                    bulk_g2s(S + L.o_own, w_own, b_own, &full[st]);
                    bulk_g2s(S + L.o_hs, w_hs, b_hs, &full[st]);
                }
            }
            if (L.fused) {
                // gathers: parent reach row (2P values, 16-byte pieces) and sigma of
                // the incoming edge, per member, into the stage
                constexpr int RB = 2 * 2 * (int)sizeof(R);   // P = 2 fast path is the common case
                R* prow = reinterpret_cast<R*>(S + L.o_reach);
                R* gsig = reinterpret_cast<R*>(S + L.o_gsig);
                const int rowb = 2 * P * (int)sizeof(R);
                (void)RB;
#pragma unroll
                for (int q = 0; q < GMAX; ++q) {
                    const int m = q * 32 + plane;
                    if (m < M) {
                        const unsigned char* src = reinterpret_cast<const unsigned char*>(g.reach + fp[q] * 2 * P);
                        unsigned char* dst = reinterpret_cast<unsigned char*>(prow + (long long)m * 2 * P);
                        for (int c = 0; c < rowb; c += 16) cp_async<16>(dst + c, src + c);
                        cp_async<(int)sizeof(R)>(gsig + m, g.sig + fe[q]);
                    }
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[st]))
                             : "memory");
                if (t + G < L.ntiles) prefetch(rec);
            }
            if (++st == L.stages) { st = 0; ++ph; }
        }
        return;
    }

    // -------------------------------------------------------------- consumers
    const int lane = tid & 31;
#ifdef CFR_STREAM_PROFILE
    // timing experiment: per consumer warp, cycles between the marks below
    unsigned long long sp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto sp_clock = []() {
        long long c;
        asm volatile("mov.u64 %0, %%clock64;\n" : "=l"(c)::"memory");
        return c;
    };
    long long sp_last = sp_clock();
#define SPROF(k)                                      \
    do {                                              \
        const long long now_ = sp_clock();            \
        sp_acc[k] += (unsigned long long)(now_ - sp_last); \
        sp_last = now_;                               \
    } while (0)
#else
#define SPROF(k) do { } while (0)
#endif
    R* const sv = reinterpret_cast<R*>(B + L.o_sv);
    short* const cm = reinterpret_cast<short*>(B + L.o_cm);
    R* const rt = reinterpret_cast<R*>(B + L.o_rt);
    R* const pos = reinterpret_cast<R*>(B + L.o_pos);
    R* const pib = reinterpret_cast<R*>(B + L.o_pib);
    // compaction counters [pi_check | pi_hat][maxseg], double-buffered by tile parity:
    // a tile's buffer is zeroed after its end barrier, while the next tile uses the other
    int* const ccnt_buf = reinterpret_cast<int*>(B + L.o_ccnt);
    int tpar = 0;
    const long long t_iter = g.ctrl[0] + 1;
    const Upd<R> up = make_upd<R>(g.variant, t_iter);
    const R w = up.w;
    bool bad = false;
    const bool all_live = g.variant >= 2;   // discounting changes every infoset: no identity updates
    const R inv_n = (R)1 / (R)n;   // uniform strategy of the level's infosets (Eq 9, z = 0)
    const int rs = L.compact ? 2 : 2 * P;   // reach row stride in the stage (elements)
    unsigned long long live_h = 0, all_h = 0;   // updated / visited infosets (thread 0)
    long long t = blockIdx.x;
    int st = 0;
    unsigned ph = 0;
    for (; t < L.ntiles; t += G) {
        unsigned char* S = B + (size_t)st * L.stage_bytes;
        const StreamHdr* hdp = reinterpret_cast<const StreamHdr*>(S);
        int* const ccnt = ccnt_buf + tpar * 2 * L.maxseg;
        SPROF(0); mbar_wait(&full[st], ph & 1u); SPROF(1);
        const StreamHdr hd = *hdp;
        const R* rows = reinterpret_cast<const R*>(S + L.o_rows) + hd.ro;
        const R* reach = reinterpret_cast<const R*>(S + L.o_reach) + hd.rro;
        // 16-byte row reads need 16-byte aligned rows in the stage
        const bool vec_rows = (((unsigned)L.rowlen * (unsigned)sizeof(R)) & 15u) == 0 &&
                              (((unsigned)hd.ro * (unsigned)sizeof(R)) & 15u) == 0;
        const R* ssig = reinterpret_cast<const R*>(S + L.o_sig) + hd.po;
        const R* sreg = reinterpret_cast<const R*>(S + L.o_reg) + hd.po;
        const R* ssn = reinterpret_cast<const R*>(S + L.o_snum) + hd.po;
        const R* sden = reinterpret_cast<const R*>(S + L.o_sden) + hd.ho;
        const unsigned char* own = reinterpret_cast<const unsigned char*>(S + L.o_own) + hd.oo;
        const int* hs = reinterpret_cast<const int*>(S + L.o_hs) + hd.hso;   // level-relative member starts
        const I* snode = reinterpret_cast<const I*>(S + L.o_node) + hd.no;   // U rows of the members
        const unsigned char* pact = reinterpret_cast<const unsigned char*>(S + L.o_pact) + hd.pao;   // fused only
        const R* gsig = reinterpret_cast<const R*>(S + L.o_gsig);                                  // fused only
        const int nseg = hd.nseg, M = hd.M, m0 = hd.m0;

        if (L.debug == 1) {   // timing experiment: data movement only
            consumers_sync();
            if (tid == 0) mbar_arrive(&empty[st]);
            if (++st == L.stages) { st = 0; ++ph; }
            tpar ^= 1;
            continue;
        }

        // ---- phase A: node values (Eq 1, ascending actions from +0); compaction of
        // the members with nonzero pi_check (their regret terms are exact zeros)
        // and of those with nonzero pi_hat (their pi_bar terms are exact zeros)
        for (int base = 0; base < M; base += kStreamConsumers) {
            const int m = base + tid;
            const bool active = m < M;
            int k = 0;
            R pc = (R)0, ph = (R)0;
            if (active) {
                const long long node = (long long)snode[m];
                if (L.umem > 0) {
                    // every infoset of the level has umem members: k = m / umem
                    k = (int)(((unsigned long long)(unsigned)m * L.udiv_m) >> L.udiv_s);
                } else {
                    int lo = 0, hi = nseg - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (hs[mid] - m0 <= m) lo = mid; else hi = mid - 1;
                    }
                    k = lo;
                }
                R v[PC];
#pragma unroll
                for (int j = 0; j < PC; ++j) v[j] = (R)0;
                const R* row = rows + (long long)m * L.rowlen;
                const R* sg = ssig + k * n;
                if (L.debug & 16) {   // timing experiment: no value loop
                } else if (PC == 1 && vec_rows) {
                    // 16-byte row reads (vec_rows: rows 16-byte aligned in the stage)
                    using V = typename std::conditional<sizeof(R) == 8, double2, float4>::type;
                    constexpr int E = 16 / (int)sizeof(R);
                    const V* row4 = reinterpret_cast<const V*>(row);
                    if ((reinterpret_cast<unsigned long long>(sg) & 15ull) == 0) {
                        // sigma row 16-byte aligned: vector loads of it too.  Row chunks
                        // are read in pairs, each lane starting with chunk 2j + d, d =
                        // bit 2 of the member: rows of 8 consecutive members then fall
                        // in 8 distinct 16-byte bank groups (a row of an even number of
                        // chunks would otherwise give 2-way conflicts); the additions
                        // stay in ascending action order
                        const V* sg4 = reinterpret_cast<const V*>(sg);
                        const int d = (m >> 2) & 1;
                        const int nc = n / E;
                        int c = 0;
                        for (; c + 1 < nc; c += 2) {
                            const V p0 = row4[c + d];
                            const V p1 = row4[c + 1 - d];
                            const V x0 = sg4[c], x1 = sg4[c + 1];
                            const R* ua = reinterpret_cast<const R*>(d ? &p1 : &p0);
                            const R* ub = reinterpret_cast<const R*>(d ? &p0 : &p1);
                            const R* xa = reinterpret_cast<const R*>(&x0);
                            const R* xb = reinterpret_cast<const R*>(&x1);
#pragma unroll
                            for (int e = 0; e < E; ++e) v[0] = v[0] + xa[e] * ua[e];
#pragma unroll
                            for (int e = 0; e < E; ++e) v[0] = v[0] + xb[e] * ub[e];
                        }
                        if (c < nc) {
                            const V u = row4[c];
                            const V x = sg4[c];
                            const R* ue = reinterpret_cast<const R*>(&u);
                            const R* xe = reinterpret_cast<const R*>(&x);
#pragma unroll
                            for (int e = 0; e < E; ++e) v[0] = v[0] + xe[e] * ue[e];
                        }
                    } else {
                        for (int a = 0; a < n; a += E) {
                            const V u = row4[a / E];
                            const R* ue = reinterpret_cast<const R*>(&u);
#pragma unroll
                            for (int e = 0; e < E; ++e) v[0] = v[0] + sg[a + e] * ue[e];
                        }
                    }
                } else {
                    for (int a = 0; a < n; ++a) {
                        const R x = sg[a];
#pragma unroll
                        for (int j = 0; j < PC; ++j) v[j] = v[j] + x * row[a * PC + j];
                    }
                }
                SPROF(2);
#pragma unroll
                for (int j = 0; j < PC; ++j) {
                    if (!(L.debug & 4)) g.U[node * PC + j] = v[j];   // (debug bit 4: timing experiment)
                    sv[m * PC + j] = v[j];
                }
                const int i = own[k];
                if (L.fused) {
                    // forward pass of this member (Eq 2 pi_check and Eq 4 pi_hat, reading
                    // Q1; the k_fwd arithmetic) from its gathered parent row and edge
                    // sigma; the actor's two factors replace the parent row in place
                    R* prow = const_cast<R*>(reach) + (long long)m * 2 * P;
                    const R x = gsig[m];
                    const int act = pact[m];
                    const R pcp = prow[i - 1], php = prow[P + i - 1];
                    pc = (act != i) ? pcp * x : pcp;
                    ph = (act == i) ? php * x : php;
                    prow[0] = pc;
                    prow[1] = ph;
                } else {
                    pc = reach[(long long)m * rs + (L.compact ? 0 : i - 1)];
                    ph = reach[(long long)m * rs + (L.compact ? 1 : P + i - 1)];
                }
            }
            SPROF(3);
            if (L.debug & 32) continue;   // timing experiment: no compaction
            // a warp whose members all have zero reach has nothing to compact
            if (__ballot_sync(0xffffffffu, active && (pc != (R)0 || ph != (R)0)) == 0u) continue;
            const int key = active ? k : -1;
            const unsigned grp = __match_any_sync(0xffffffffu, key);
            const int leader = __ffs(grp) - 1;
            const unsigned lt = (1u << lane) - 1u;
            const unsigned nzc = grp & __ballot_sync(0xffffffffu, active && pc != (R)0);
            const unsigned nzh = grp & __ballot_sync(0xffffffffu, active && ph != (R)0);
            int bc = 0, bh = 0;
            if (lane == leader && key >= 0) {
                if (nzc) bc = atomicAdd(&ccnt[k], __popc(nzc));
                if (nzh) bh = atomicAdd(&ccnt[L.maxseg + k], __popc(nzh));
            }
            bc = __shfl_sync(0xffffffffu, bc, leader);
            bh = __shfl_sync(0xffffffffu, bh, leader);
            if (active && pc != (R)0) cm[(hs[k] - m0) + bc + __popc(nzc & lt)] = (short)m;
            if (active && ph != (R)0) cm[L.maxm + (hs[k] - m0) + bh + __popc(nzh & lt)] = (short)m;
        }
        SPROF(4); consumers_sync(); SPROF(5);

        // ---- phases B + C, a warp per LIVE infoset (no CTA barrier in between).
        // Live: some member has a nonzero pi_check (r~ may be nonzero) or pi_hat
        // (pi_bar may be nonzero).  For a dead infoset every term is an exact zero:
        // r~ = +0 and pi_bar = +0, so R, S_num, S_den and sigma keep their bits and
        // its update (and its writes) are skipped.  (Splitting a live infoset's
        // members over several warps, combined after a CTA barrier, was measured
        // slower: live infosets mostly have few live members.)
        const long long qt = L.q0 + (long long)hd.k0 * n;
        const long long ht = L.h0 + hd.k0;
        {
            const int warp = tid >> 5;
            const unsigned live = __ballot_sync(
                0xffffffffu, lane < nseg && (g.upd_player == 0 || own[lane] == g.upd_player) &&
                                 (all_live || ccnt[lane] != 0 || ccnt[L.maxseg + lane] != 0));
            if (tid == 0) {
                live_h += __popc(live);
                all_h += nseg;
            }
            // phase B items of one infoset: n pairs (r~) + 1 pi_bar, ns lanes each
            int ns = 1, lns = 0;
            while (ns < 32 && (n + 1) * ns * 2 <= 32) { ns <<= 1; ++lns; }
            const int ipr = 32 >> lns;   // items per round
            int j = 0;
            for (unsigned lm = live; lm; lm &= lm - 1u, ++j) {
                if ((j & (kStreamConsumers / 32 - 1)) != warp) continue;
                const int k = __ffs(lm) - 1;
                const int i = own[k];
                const int col = (PC == 1) ? 0 : i - 1;
                const int sb = hs[k] - m0;
                const int cntc = ccnt[k], cnth = ccnt[L.maxseg + k];
                const short* memc = cm + sb;
                const short* memh = cm + L.maxm + sb;
                const bool two = L.fused || L.compact;
                const int oc = two ? 0 : i - 1, oh = two ? 1 : P + i - 1;   // pi_check / pi_hat in a reach row
                // ---- phase B: exact sums (slices of integer-valued doubles combine
                // exactly in any order)
                for (int base = 0; base <= n; base += ipr) {
                    const int itm = base + (lane >> lns), part = lane & (ns - 1);
                    double c0 = 0, c1 = 0, c2 = 0;
                    if (itm < n) {
                        const int a = itm;
                        double e0 = 0, e1 = 0, e2 = 0;   // second independent slice chain (ILP)
                        int jj = part;
                        for (; jj + ns < cntc; jj += 2 * ns) {
                            const int la = memc[jj], lb = memc[jj + ns];
                            const R ua = rows[(long long)la * L.rowlen + a * PC + col];
                            const R ub = rows[(long long)lb * L.rowlen + a * PC + col];
                            const R ta = reach[(long long)la * rs + oc] * (ua - sv[la * PC + col]);
                            const R tb = reach[(long long)lb * rs + oc] * (ub - sv[lb * PC + col]);
                            xadd(c0, c1, c2, (double)ta, g.sc0);
                            xadd(e0, e1, e2, (double)tb, g.sc0);
                        }
                        if (jj < cntc) {
                            const int la = memc[jj];
                            const R ua = rows[(long long)la * L.rowlen + a * PC + col];
                            const R ta = reach[(long long)la * rs + oc] * (ua - sv[la * PC + col]);
                            xadd(c0, c1, c2, (double)ta, g.sc0);
                        }
                        c0 += e0;
                        c1 += e1;
                        c2 += e2;
                        if (PC == 1 && i == 2) { c0 = -c0; c1 = -c1; c2 = -c2; }   // u2 = -u1 storage
                    } else if (itm == n) {
                        for (int jj = part; jj < cnth; jj += ns)
                            xadd(c0, c1, c2, (double)reach[(long long)memh[jj] * rs + oh], g.scp0);
                    }
                    for (int o = 1; o < ns; o <<= 1) {
                        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
                        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
                        c2 += __shfl_xor_sync(0xffffffffu, c2, o);
                    }
                    if (part == 0) {
                        if (itm < n) rt[k * n + itm] = (R)xdec(c0, c1, c2, g.rc);
                        else if (itm == n) pib[k] = (R)xdec(c0, c1, c2, g.rcp);
                    }
                }
                __syncwarp();
                // ---- phase C: Eq 8/15 or CFR+, Eq 10, then Eq 9 (z ascending)
                const R wp = w * pib[k];
                for (int c = 0; c < n; c += 32) {
                    const int a = c + lane;
                    if (a < n) {
                        const int p = k * n + a;
                        const R r_t = rt[p];
                        const R r = upd_regret(up, sreg[p], r_t);   // Eq 8/15 (Q4) / CFR+ (Q6) / Q18
                        if (!(L.debug & 8)) {   // (debug bit 8: timing experiment)
                            g.regret[qt + p] = r;
                            g.snum[qt + p] = upd_sum(up, ssn[p], wp * ssig[p]);  // Eq 10 numerator
                        }
                        pos[p] = (r > (R)0) ? r : (R)0;
                    }
                }
                __syncwarp();
                R z = (R)0;
                const R* pk = pos + k * n;
#pragma unroll 4
                for (int b = 0; b < n; ++b) z = z + pk[b];   // broadcast reads, ascending
                if (lane == 0 && !(L.debug & 8)) g.sden[ht + k] = upd_sum(up, sden[k], wp);   // Eq 10 denominator
                for (int c = 0; c < n; c += 32) {
                    const int a = c + lane;
                    if (a < n) {
                        const int p = k * n + a;
                        const R nsig = (z > (R)0) ? pos[p] / z : inv_n;   // Eq 9
                        if (!(L.debug & 8)) g.sig[qt + p] = nsig;
                        if (!finite_(rt[p]) || !finite_(nsig) || !finite_(z)) bad = true;
                    }
                }
            }
        }
        SPROF(6); consumers_sync();   // every read of this stage is done
        SPROF(7);
        if (tid == 0) mbar_arrive(&empty[st]);
        for (int k = tid; k < 2 * L.maxseg; k += kStreamConsumers) ccnt[k] = 0;   // for the tile after next
        tpar ^= 1;
        if (++st == L.stages) { st = 0; ++ph; }
    }
#ifdef CFR_STREAM_PROFILE
    if (lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&g_stream_prof[(tid >> 5) * 8 + k], sp_acc[k]);
    if (tid == 0) atomicAdd(&g_stream_prof[64], (unsigned long long)((L.ntiles - blockIdx.x + G - 1) / G));
#endif
#undef SPROF
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (tid == 0) {
        // cumulative: infosets updated / visited by the streaming levels (bench.py's
        // byte model counts update writes of live infosets only)
        unsigned long long* c = g.lcnt + 4 * L.level;
        atomicAdd(c + 0, live_h);
        atomicAdd(c + 1, live_h * (unsigned long long)n);
        atomicAdd(c + 2, all_h);
        atomicAdd(c + 3, all_h * (unsigned long long)n);
    }
    if (L.last) {
        consumers_sync();
        if (tid == 0) {
            __threadfence();
            const unsigned long long prev = atomicAdd((unsigned long long*)&g.ctrl[2], 1ULL);
            if (prev == gridDim.x - 1) {
                g.ctrl[0] = t_iter;
                g.ctrl[2] = 0;
            }
        }
    }
}

// Update of deferred infosets (span several depths / tiles): decode the global
// exact sums, then the same Eq 8/15, Eq 10, Eq 9 steps; zero the accumulators.
template <class R, class I>
__device__ __forceinline__ void deferred_body(const DG<R, I>& g, int last) {
    pdl_trigger();
    pdl_wait();
    const long long t_iter = g.ctrl[0] + 1;
    const Upd<R> up = make_upd<R>(g.variant, t_iter);
    const R w = up.w;
    bool bad = false;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < g.ndef; idx += stride) {
        const long long h = (long long)g.deferred[idx];
        const long long qb = (long long)g.qbase[h];
        const int n = (int)((long long)g.qbase[h + 1] - qb);
        const long long dq = g.dqbase[idx];
        const long long p0 = (long long)g.acc_p[idx * 3 + 0], p1 = (long long)g.acc_p[idx * 3 + 1],
                        p2 = (long long)g.acc_p[idx * 3 + 2];
        g.acc_p[idx * 3 + 0] = 0;
        g.acc_p[idx * 3 + 1] = 0;
        g.acc_p[idx * 3 + 2] = 0;
        if (g.upd_player != 0 && g.owner[h] != g.upd_player) {
            // alternating updates: another player's infoset -- zero its sums only
            for (int a = 0; a < 3 * n; ++a) g.acc_r[dq * 3 + a] = 0;
            continue;
        }
        const R pib = (R)xdec_ll(p0, p1, p2, g.rcp);
        const R wp = w * pib;
        R z = (R)0;
        for (int a = 0; a < n; ++a) {
            const long long q = qb + a;
            const long long cq = dq + a;
            const long long c0 = (long long)g.acc_r[cq * 3 + 0], c1 = (long long)g.acc_r[cq * 3 + 1],
                            c2 = (long long)g.acc_r[cq * 3 + 2];
            g.acc_r[cq * 3 + 0] = 0;
            g.acc_r[cq * 3 + 1] = 0;
            g.acc_r[cq * 3 + 2] = 0;
            const R rt = (R)xdec_ll(c0, c1, c2, g.rc);
            g.regret[q] = upd_regret(up, g.regret[q], rt);
            g.snum[q] = upd_sum(up, g.snum[q], wp * g.sig[q]);
        }
        g.sden[h] = upd_sum(up, g.sden[h], wp);
        for (int a = 0; a < n; ++a) {
            const R r = g.regret[qb + a];
            z = z + ((r > (R)0) ? r : (R)0);
        }
        for (int a = 0; a < n; ++a) {
            const R r = g.regret[qb + a];
            const R pos = (r > (R)0) ? r : (R)0;
            const R nsig = (z > (R)0) ? pos / z : (R)1 / (R)n;
            g.sig[qb + a] = nsig;
            if (!finite_(r) || !finite_(nsig)) bad = true;
        }
    }
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (last) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned long long prev = atomicAdd((unsigned long long*)&g.ctrl[2], 1ULL);
            if (prev == gridDim.x - 1) {
                g.ctrl[0] = t_iter;
                g.ctrl[2] = 0;
            }
        }
    }
}

template <class R, class I>
__global__ void __launch_bounds__(256) k_deferred(DG<R, I> g, int last) {
    deferred_body<R, I>(g, last);
}

// --------------------------------------------------- persistent iteration
// Small games are launch-latency bound (2D kernels per iteration).  k_persist runs
// T whole iterations in ONE cooperative launch: every CTA is resident; the levels
// of an iteration are separated by grid-wide barriers (the same forward, tile and
// deferred bodies as the per-level kernels, so the arithmetic is identical).
struct PLevel {
    long long s0, s1;   // slots of depth l (forward pass of level l)
    long long t0, t1;   // tiles of parent depth L (backward pass)
    SmemLayout lay;     // tile shared-memory layout of depth L
};

// Sense-free grid barrier: bar[0] arrivals, bar[1] generation.  Thread 0 arrives
// after a gpu-scope fence (the block's writes are visible) and leaves after one
// (other blocks' writes are visible to the block, L1 included).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g0) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

template <class R, class I, int PC, int PT>
__global__ void __launch_bounds__(kTileSlots) k_persist(DG<R, I> g, const PLevel* __restrict__ lv, int D, int has_def,
                                                         long long T, unsigned* bar) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    long long t_done = g.ctrl[0];
    for (long long it = 0; it < T; ++it) {
        for (int l = 1; l < D; ++l) {   // forward pass, depth 1 .. D-1
            const long long s0 = lv[l].s0, s1 = lv[l].s1;
            if (s1 <= s0) continue;
            fwd_body<R, I, PT>(g, g.sig, s0, s1, 0);
            grid_sync(bar);
        }
        for (int L = D - 1; L >= 0; --L) {   // backward pass, parent depth D-1 .. 0
            const long long t0 = lv[L].t0, t1 = lv[L].t1;
            if (t1 <= t0) continue;
            const SmemLayout lay = lv[L].lay;
            for (long long t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
                __syncthreads();   // the previous tile's shared-memory reads are done
                bwd_tile<R, I, PC, MODE_CFR>(g, g.sig, t, 0, 0, lay, smem_raw);
            }
            grid_sync(bar);
        }
        if (has_def) {
            deferred_body<R, I>(g, 0);
            grid_sync(bar);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) g.ctrl[0] = ++t_done;   // the iteration is complete
        else ++t_done;
        grid_sync(bar);
    }
}

// ------------------------------------------------------------- tiny games
// Games whose whole mutable state fits in one CTA's shared memory (Kuhn; Leduc in
// f32) are bound by per-level latency, not bytes.  k_tiny runs T iterations in
// ONE CTA: U, reach, sigma, R, S_num, S_den (and the per-level r~ / pi_bar) live
// in shared memory; levels are separated by __syncthreads; read-only metadata
// comes from global memory through L1.  Same operations, same order as the
// per-level kernels (requires depth-homogeneous infosets: an infoset's members
// are the contiguous slots mem_of[2h] .. mem_of[2h+1] of one level).
struct TinyLevel {
    long long s0, s1;   // slots of depth l
    long long h0, h1;   // internal infosets at depth l (consecutive)
};
struct TinyPlan {
    long long U, reach, sig, reg, snum, sden, rt, pib;   // element offsets in shared memory (R units)
    long long nU, nreach, nsig, Q, H;
    int bytes;
};

template <class R, class I, int PC>
__global__ void __launch_bounds__(1024) k_tiny(DG<R, I> g, const TinyLevel* __restrict__ lv, const I* __restrict__ mem_of,
                                                int D, long long T, TinyPlan tp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* const sm = reinterpret_cast<R*>(smem_raw);
    R* const U = sm + tp.U;
    R* const reach = sm + tp.reach;
    R* const sig = sm + tp.sig;
    R* const reg = sm + tp.reg;
    R* const snum = sm + tp.snum;
    R* const sden = sm + tp.sden;
    R* const rtb = sm + tp.rt;
    R* const pibb = sm + tp.pib;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int P = g.P;
    pdl_trigger();
    pdl_wait();
    for (long long k = tid; k < tp.nU; k += nth) U[k] = g.U[k];
    for (long long k = tid; k < tp.nreach; k += nth) reach[k] = g.reach[k];
    for (long long k = tid; k < tp.nsig; k += nth) sig[k] = g.sig[k];
    for (long long k = tid; k < tp.Q; k += nth) {
        reg[k] = g.regret[k];
        snum[k] = g.snum[k];
    }
    for (long long k = tid; k < tp.H; k += nth) sden[k] = g.sden[k];
    __syncthreads();
    long long t_iter = g.ctrl[0];
    bool bad = false;
    for (long long it = 0; it < T; ++it) {
        ++t_iter;
        const Upd<R> up = make_upd<R>(g.variant, t_iter);
        const R w = up.w;
        const int passes = (g.variant == 4) ? P : 1;
        for (int pass = 1; pass <= passes; ++pass) {
            const int upl = (passes > 1) ? pass : 0;
            for (int l = 1; l < D; ++l) {   // forward (Eq 2, Eq 4 with reading Q1)
                for (long long s = lv[l].s0 + tid; s < lv[l].s1; s += nth) {
                    const long long p = (long long)g.f_parent[s];
                    const R x = sig[g.f_e[s]];
                    const int act = g.f_pact[s];
                    for (int j = 0; j < P; ++j) {
                        const R pc = reach[p * 2 * P + j], ph = reach[p * 2 * P + P + j];
                        reach[s * 2 * P + j] = (act != j + 1) ? pc * x : pc;
                        reach[s * 2 * P + P + j] = (act == j + 1) ? ph * x : ph;
                    }
                }
                __syncthreads();
            }
            for (int L = D - 1; L >= 0; --L) {
                for (long long s = lv[L].s0 + tid; s < lv[L].s1; s += nth) {   // values (Eq 1)
                    const long long cb = (long long)g.s_cb[s], eb = (long long)g.s_ebase[s];
                    const int nch = g.s_n[s];
                    R v[PC];
#pragma unroll
                    for (int j = 0; j < PC; ++j) v[j] = (R)0;
                    for (int a = 0; a < nch; ++a) {
                        const R x = sig[eb + a];
#pragma unroll
                        for (int j = 0; j < PC; ++j) v[j] = v[j] + x * U[(cb + a) * PC + j];
                    }
                    const long long node = (long long)g.s_node[s];
#pragma unroll
                    for (int j = 0; j < PC; ++j) U[node * PC + j] = v[j];
                }
                __syncthreads();
                const long long h0 = lv[L].h0, h1 = lv[L].h1;
                if (h1 > h0) {
                    const long long q0 = (long long)g.qbase[h0], q1 = (long long)g.qbase[h1];
                    const long long items = (q1 - q0) + (h1 - h0);
                    for (long long x = tid; x < items; x += nth) {   // exact sums
                        double c0 = 0, c1 = 0, c2 = 0;
                        if (x < q1 - q0) {
                            const long long q = q0 + x;
                            long long lo = h0, hi = h1 - 1;
                            while (lo < hi) {
                                const long long mid = (lo + hi + 1) >> 1;
                                if ((long long)g.qbase[mid] <= q) lo = mid; else hi = mid - 1;
                            }
                            const long long h = lo;
                            const int i = g.owner[h];
                            if (upl != 0 && i != upl) continue;
                            const int a = (int)(q - (long long)g.qbase[h]);
                            const int col = (PC == 1) ? 0 : i - 1;
                            for (long long d = (long long)mem_of[2 * h]; d < (long long)mem_of[2 * h + 1]; ++d) {
                                const R pc = reach[d * 2 * P + (i - 1)];
                                if (pc == (R)0) continue;   // exact zero terms
                                const R u = U[((long long)g.s_cb[d] + a) * PC + col];
                                const R v = U[(long long)g.s_node[d] * PC + col];
                                xadd(c0, c1, c2, (double)(pc * (u - v)), g.sc0);
                            }
                            if (PC == 1 && i == 2) { c0 = -c0; c1 = -c1; c2 = -c2; }   // u2 = -u1 storage
                            rtb[q] = (R)xdec(c0, c1, c2, g.rc);
                        } else {
                            const long long h = h0 + (x - (q1 - q0));
                            const int i = g.owner[h];
                            if (upl != 0 && i != upl) continue;
                            for (long long d = (long long)mem_of[2 * h]; d < (long long)mem_of[2 * h + 1]; ++d)
                                xadd(c0, c1, c2, (double)reach[d * 2 * P + P + (i - 1)], g.scp0);
                            pibb[h] = (R)xdec(c0, c1, c2, g.rcp);
                        }
                    }
                    __syncthreads();
                    for (long long h = h0 + tid; h < h1; h += nth) {   // update (Eq 8/15 / CFR+ / Q18, Eq 10, Eq 9)
                        const int i = g.owner[h];
                        if (upl != 0 && i != upl) continue;
                        const long long qb = (long long)g.qbase[h];
                        const int n = (int)((long long)g.qbase[h + 1] - qb);
                        const R wp = w * pibb[h];
                        R z = (R)0;
                        for (int a = 0; a < n; ++a) {
                            const long long q = qb + a;
                            const R r = upd_regret(up, reg[q], rtb[q]);
                            reg[q] = r;
                            snum[q] = upd_sum(up, snum[q], wp * sig[q]);
                            z = z + ((r > (R)0) ? r : (R)0);
                        }
                        sden[h] = upd_sum(up, sden[h], wp);
                        for (int a = 0; a < n; ++a) {
                            const long long q = qb + a;
                            const R r = reg[q];
                            const R pos = (r > (R)0) ? r : (R)0;
                            const R nsig = (z > (R)0) ? pos / z : (R)1 / (R)n;
                            sig[q] = nsig;
                            if (!finite_(rtb[q]) || !finite_(nsig) || !finite_(z)) bad = true;
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
    // write the state back (readbacks and later launches read it from global)
    for (long long k = tid; k < tp.nU; k += nth) g.U[k] = U[k];
    for (long long k = tid; k < tp.nreach; k += nth) g.reach[k] = reach[k];
    for (long long k = tid; k < tp.nsig; k += nth) g.sig[k] = sig[k];
    for (long long k = tid; k < tp.Q; k += nth) {
        g.regret[k] = reg[k];
        g.snum[k] = snum[k];
    }
    for (long long k = tid; k < tp.H; k += nth) g.sden[k] = sden[k];
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (tid == 0) g.ctrl[0] = t_iter;
}

// sigma_bar (Eq 10, reading Q5) into an evaluation strategy buffer: S_num/S_den,
// uniform where S_den = 0.  Chance part copied.
template <class R, class I>
__global__ void k_average(DG<R, I> g, R* out, long long H, long long Q, long long C) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < H; h += stride) {
        const long long qb = (long long)g.qbase[h];
        const int n = (int)((long long)g.qbase[h + 1] - qb);
        const R den = g.sden[h];
        for (int a = 0; a < n; ++a) out[qb + a] = (den > (R)0) ? g.snum[qb + a] / den : (R)1 / (R)n;
    }
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < C; c += stride) out[Q + c] = g.sig[Q + c];
}

// Multi-GPU exchange 1: cut-level decision values.  Each row is
// written by exactly one rank (others contribute zeros), so a sum-allreduce is exact.
template <class R>
__global__ void k_cut_pack(const R* __restrict__ U, const long long* __restrict__ rows,
                           const unsigned char* __restrict__ owned, R* __restrict__ buf, long long n, int Pc) {
    pdl_trigger();
    pdl_wait();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        for (int j = 0; j < Pc; ++j) buf[i * Pc + j] = owned[i] ? U[rows[i] * Pc + j] : (R)0;
}
template <class R>
__global__ void k_cut_unpack(R* __restrict__ U, const long long* __restrict__ rows, const R* __restrict__ buf, long long n,
                             int Pc) {
    pdl_trigger();
    pdl_wait();
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        for (int j = 0; j < Pc; ++j) U[rows[i] * Pc + j] = buf[i * Pc + j];
}
// Readback combination: zero the (h, a) entries this rank does not report.
template <class R, class I>
__global__ void k_mask_q(R* __restrict__ out, const I* __restrict__ qbase, const unsigned char* __restrict__ report,
                         long long H) {
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < H; h += (long long)gridDim.x * blockDim.x)
        if (!report[h])
            for (long long q = (long long)qbase[h]; q < (long long)qbase[h + 1]; ++q) out[q] = (R)0;
}
template <class R>
__global__ void k_mask_h(R* __restrict__ out, const unsigned char* __restrict__ report, long long H) {
    for (long long h = (long long)blockIdx.x * blockDim.x + threadIdx.x; h < H; h += (long long)gridDim.x * blockDim.x)
        if (!report[h]) out[h] = (R)0;
}

// --------------------------------------------------------------- host side
#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            cfrb_set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return CFR_ERR_CUDA;                                                                   \
        }                                                                                          \
    } while (0)

// Launch with the programmatic-stream-serialization attribute (PDL) when `pdl`.
template <typename... KArgs, typename... Args>
static cudaError_t launch(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

struct SolverBase {
    virtual ~SolverBase() {}
    virtual cfr_status enqueue(int64_t iters) = 0;
    virtual cfr_status sync() = 0;
    virtual cfr_status iteration(int64_t* T) = 0;
    virtual cfr_status strategy(int which, double* out) = 0;   // 0 avg, 1 current
    virtual cfr_status get_state(double* regret, double* snum, double* sden) = 0;
    virtual cfr_status expected_values(int which, double* out) = 0;
    virtual cfr_status exploitability(double* nc, double* ex, double* br) = 0;
    virtual cfr_status launches(int64_t* n) = 0;
    virtual cfr_status profile(int64_t iters, double* out) = 0;
    virtual cfr_status model_bytes(double* out) = 0;
    virtual cfr_status level_kernels(int32_t* out, int32_t max_levels, int32_t* num_levels) = 0;
    virtual cfr_status counters(int64_t* out, int32_t max_levels, int32_t* num_levels) = 0;
    virtual cfr_status level_profile(double* out, int32_t max_levels, int32_t* num_levels) = 0;
    virtual cfr_status phase(int ph, double* out) = 0;
    virtual cfr_status exchange_size(int which, size_t* bytes) = 0;
    virtual cfr_status exchange(int which, int put, void* host, size_t bytes) = 0;
    virtual cfr_status shard_info(int64_t* out) = 0;
};

struct Layout {
    size_t off = 0;
    template <class T>
    size_t take(size_t n) {
        off = (off + 255) & ~size_t(255);
        const size_t o = off;
        off += n * sizeof(T);
        return o;
    }
};

// U rows of depth l start at u_off[l] (rows), each level aligned to 32 bytes so
// that uniform child rows can be staged with 16-byte cp.async chunks.
static std::vector<int64_t> u_layout(const Game& g, size_t elem) {
    const int64_t rowbytes = (int64_t)g.Pc * (int64_t)elem;
    int64_t a = 32, b = rowbytes;
    while (b) { const int64_t t = a % b; a = b; b = t; }
    const int64_t m = 32 / a;   // rows per alignment unit
    std::vector<int64_t> off(g.D + 2, 0);
    for (int l = 0; l <= g.D; ++l) {
        const int64_t n = g.level_ptr[l + 1] - g.level_ptr[l];
        off[l + 1] = ((off[l] + n + m - 1) / m) * m;
    }
    return off;
}

// Device row order.  Row 0 is the root; the rows of depth L+1 are
// the children of the depth-L slots taken in SLOT order (each slot's children
// contiguous, in action order).  A backward tile's child rows are then one
// contiguous block, as are its reach rows (reach is indexed by slot) and its
// (h, a) state: every stream of the backward pass is sequential.  Only the
// per-node value write (into the parent's row) scatters.
// node_u[s] / cb_u[s]: U row of slot s's node / first child.
static void u_rows(const Game& g, const std::vector<int64_t>& uoff, std::vector<int64_t>& node_u,
                   std::vector<int64_t>& cb_u) {
    node_u.assign(g.NS, 0);
    cb_u.assign(g.NS, 0);
    std::vector<int64_t> sod(g.ND, -1);   // slot of each dec index
    for (int64_t s = 0; s < g.NS; ++s) sod[g.s_dec[s]] = s;
    for (int L = 0; L < g.D; ++L) {
        int64_t run = 0;
        for (int64_t s = g.slot_ptr[L]; s < g.slot_ptr[L + 1]; ++s) {
            cb_u[s] = uoff[L + 1] + run;
            run += g.s_n[s];
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < g.NS; ++s) {
        const int64_t d = g.s_dec[s];
        const int64_t pd = g.f_parent[d];
        if (pd < 0) { node_u[s] = 0; continue; }   // the root
        const int64_t ps = sod[pd];
        node_u[s] = cb_u[ps] + (g.f_e[d] - g.s_ebase[ps]);   // f_e = parent's edge base + action
    }
}

// Staging layout per tile (precision dependent): uniform rows whose starts and
// lengths are multiples of the cp.async chunk use chunked copies with an odd
// number of chunks per row stride (<= 2-way bank conflicts); others fall back to
// generic rows (odd element strides) or, if too large, to global reads.
template <class R>
static void stage_tiles(const Game& g, const std::vector<int64_t>& cb_u, const std::vector<uint8_t>& contrib,
                        std::vector<TileD>& tiles, std::vector<int32_t>& s_coff) {
    const int CH = (sizeof(R) == 8) ? 16 : 8;
    const int CE = CH / (int)sizeof(R);
    s_coff = g.s_coff;
    tiles.assign(g.tiles.size(), TileD{});
    for (size_t t = 0; t < g.tiles.size(); ++t) {
        const TileH& th = g.tiles[t];
        TileD td{};
        td.s0 = th.s0;
        td.s1 = th.s1;
        td.seg0 = th.seg0;
        td.seg1 = th.seg1;
        td.npairs = th.npairs;
        td.staged = th.staged ? 2 : 0;
        td.contrib = contrib.empty() ? 1 : (int)contrib[t];
        if (th.staged) {
            const int rowlen = g.s_n[th.s0] * g.Pc;
            bool uni = (rowlen % CE) == 0;
            for (int64_t s = th.s0; s < th.s1 && uni; ++s)
                uni = (g.s_n[s] * g.Pc == rowlen) && ((cb_u[s] * g.Pc) % CE == 0);
            if (uni) {
                const int cpr = rowlen / CE;
                const int cstride = (cpr % 2 == 0) ? cpr + 1 : cpr;
                const int64_t need = (int64_t)(th.s1 - th.s0) * cstride * CE;
                if (need <= kTileChildren) {
                    td.staged = 1;
                    td.rowlen = rowlen;
                    td.cpr = cpr;
                    td.stride = cstride * CE;
                    td.inv_cpr = 1.0f / (float)cpr;
                    for (int64_t s = th.s0; s < th.s1; ++s) s_coff[s] = (int32_t)((s - th.s0) * td.stride);
                }
            }
        }
        tiles[t] = td;
    }
}

// Levels served by the pipelined k_bwd_fast: every tile chunk-staged, fused,
// player-only, one row length across the level, and enough tiles to pipeline.
template <class R, class I>
static std::vector<FastLevel> fast_levels(const Game& g, const std::vector<TileD>& tiles, size_t* pool_bytes) {
    std::vector<FastLevel> out(g.D, FastLevel{});
    size_t pool = 0;
    for (int L = 0; L < g.D; ++L) {
        FastLevel f{};
        f.tile0 = g.tile_ptr[L];
        f.ntiles = g.tile_ptr[L + 1] - g.tile_ptr[L];
        f.recsize = 0;
        bool ok = f.ntiles >= 2 * 148;
        int rowlen = -1, maxslot = 1, maxseg = 1, maxpairs = 1, maxch = 0;
        for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1] && ok; ++t) {
            const TileD& td = tiles[t];
            if (td.staged != 1 || td.npairs > kTilePairs || td.cpr > 2 * kTileSlots) { ok = false; break; }
            if (rowlen < 0) rowlen = td.rowlen;
            if (td.rowlen != rowlen) { ok = false; break; }
            int64_t members = 0;
            for (int k = td.seg0; k < td.seg1; ++k) {
                if (!g.segs[k].fused) ok = false;
                members += g.segs[k].se - g.segs[k].sb;
            }
            if (members != td.s1 - td.s0) ok = false;   // a chance slot
            const int nslot = (int)(td.s1 - td.s0);
            maxslot = std::max(maxslot, nslot);
            maxseg = std::max(maxseg, td.seg1 - td.seg0);
            maxpairs = std::max(maxpairs, td.npairs);
            maxch = std::max(maxch, nslot * td.stride);
        }
        if (ok && f.ntiles > 0) {
            const TileD& t0 = tiles[g.tile_ptr[L]];
            f.maxslot = maxslot;
            f.maxseg = maxseg;
            f.maxpairs = maxpairs;
            f.maxch = maxch;
            f.rowlen = t0.rowlen;
            f.cpr = t0.cpr;
            f.stride = t0.stride;
            f.inv_cpr = t0.inv_cpr;
            f.recsize = (int)((32 + (int64_t)maxseg * sizeof(FastSeg) + 3 * sizeof(I) * (int64_t)maxslot + maxslot +
                               maxpairs + 15) & ~int64_t(15));
            f.rec = (long long)pool;
            pool += (size_t)f.recsize * (size_t)f.ntiles;
        }
        out[L] = f;
    }
    *pool_bytes = pool;
    return out;
}

// Shared-memory plan of k_bwd_stream for one level (stage ring + work arrays +
// barriers).  Every block is 16-byte aligned; windows get 16 bytes of slack.
static void stream_plan(StreamLevel& f, int P, int Pc, int w, int ix, int stages) {
    auto al = [](long long x) { return (int)((x + 15) & ~15ll); };
    const int maxpairs = f.maxm > 0 ? f.maxseg * f.n : 0;
    int o = al(sizeof(StreamHdr));
    f.o_rows = o; o += al((long long)f.maxm * f.rowlen * w + 16);
    f.o_reach = o; o += al((long long)f.maxm * 2 * P * w + 16);
    f.o_sig = o; o += al((long long)maxpairs * w + 16);
    f.o_reg = o; o += al((long long)maxpairs * w + 16);
    f.o_snum = o; o += al((long long)maxpairs * w + 16);
    f.o_sden = o; o += al((long long)f.maxseg * w + 16);
    f.o_own = o; o += al((long long)f.maxseg + 16);
    f.o_hs = o; o += al((long long)(f.maxseg + 1) * 4 + 16);
    f.o_node = o; o += al((long long)f.maxm * ix + 16);
    f.o_pact = o; o += f.fused ? al((long long)f.maxm + 16) : 0;
    f.o_gsig = o; o += f.fused ? al((long long)f.maxm * w) : 0;
    f.stages = stages;
    f.stage_bytes = o;
    int x = stages * o;
    f.o_sv = x; x += al((long long)f.maxm * Pc * w);
    f.o_cm = x; x += al((long long)f.maxm * 4);          // two compaction lists (pi_check, pi_hat)
    f.o_rt = x; x += al((long long)maxpairs * w);
    f.o_pos = x; x += al((long long)maxpairs * w);
    f.o_pib = x; x += al((long long)f.maxseg * w);
    f.o_zs = x; x += al((long long)f.maxseg * w);
    f.o_ccnt = x; x += al((long long)f.maxseg * 16);   // 2 counters x 2 tile buffers
    f.o_bar = x; x += al(2 * stages * 8);
    f.bytes = x;
}

// Levels served by k_bwd_stream: every slot a player node inside a fused segment,
// consecutive internal infosets with one |A(h)|, <= kStreamConsumers members per
// infoset, 16-byte rows.  Tiles pack whole infosets (<= kStreamConsumers members).
// Appends the tile records (int4 {k0, k1, m0, m1}) and member starts to `pool`.
template <class R, class I>
static std::vector<StreamLevel> stream_levels(const Game& g, const std::vector<int64_t>& cb_u, std::vector<int>* pool,
                                              int min_tiles, int stages, int tile_target, bool fuse_forward,
                                              bool compact_reach) {
    const int w = (int)sizeof(R), P = g.P, Pc = g.Pc, ix = (int)sizeof(I);
    std::vector<StreamLevel> out(g.D, StreamLevel{});
    for (int L = 0; L < g.D; ++L) {
        StreamLevel f{};
        const int64_t s0 = g.slot_ptr[L], s1 = g.slot_ptr[L + 1];
        if (s1 <= s0) { out[L] = f; continue; }
        bool ok = s1 < INT32_MAX;
        std::vector<int> hs;
        int64_t h_prev = -1, next = s0;
        int n = -1;
        for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1] && ok; ++t)
            for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1 && ok; ++k) {
                const SegH& sg = g.segs[k];
                const int nn = (int)(g.qbase_int[sg.h + 1] - g.qbase_int[sg.h]);
                if (!sg.fused || sg.sb != next || (h_prev >= 0 && sg.h != h_prev + 1) || (n >= 0 && nn != n) ||
                    sg.se - sg.sb > tile_target)
                    ok = false;
                n = nn;
                hs.push_back((int)(sg.sb - s0));
                h_prev = sg.h;
                next = sg.se;
            }
        if (!ok || next != s1 || n <= 0) { out[L] = f; continue; }
        const int64_t row0 = cb_u[s0];
        // (rows and reach rows of any alignment: the TMA windows are 16-byte aligned
        // supersets and the consumers apply the element offsets).  Rows shorter than
        // 16 bytes stay on the tile kernel: their per-member work is too small to
        // amortise the streaming pipeline (measured on Goofspiel-6's one-action levels).
        if ((int64_t)n * Pc * w < 16) { out[L] = f; continue; }
        for (int64_t s = s0; s < s1 && ok; ++s) ok = (cb_u[s] == row0 + (s - s0) * n);
        if (!ok) { out[L] = f; continue; }
        const int nh = (int)hs.size();
        hs.push_back((int)(s1 - s0));
        // tiles: greedy runs of whole infosets, <= kStreamConsumers members, <= 32 infosets
        std::vector<int> tk = {0};
        for (int k = 0; k < nh; ++k) {
            const int k0 = tk.back();
            if (k > k0 && (hs[k + 1] - hs[k0] > tile_target || k + 1 - k0 > 32)) tk.push_back(k);
        }
        tk.push_back(nh);
        f.ntiles = (long long)tk.size() - 1;
        if (f.ntiles < min_tiles) { out[L] = StreamLevel{}; continue; }
        f.s0 = s0;
        f.h0 = g.segs[g.tiles[g.tile_ptr[L]].seg0].h;
        f.q0 = g.qbase_int[f.h0];
        f.row0 = row0;
        f.n = n;
        f.rowlen = n * Pc;
        {
            // p / n by a 64-bit multiply and shift (round-up reciprocal), verified for p < 2^16
            int l = 0;
            while ((1 << l) < n) ++l;
            f.ndiv_s = 16 + l;
            f.ndiv_m = (unsigned)((((unsigned long long)1 << (16 + l)) + (unsigned long long)n - 1) / (unsigned long long)n);
            for (unsigned x = 0; x < 65536u && ok; ++x)
                ok = (unsigned)(((unsigned long long)x * f.ndiv_m) >> f.ndiv_s) == x / (unsigned)n;
            if (!ok) { out[L] = StreamLevel{}; continue; }
        }
        for (long long t = 0; t < f.ntiles; ++t) {
            f.maxm = std::max(f.maxm, hs[tk[t + 1]] - hs[tk[t]]);
            f.maxseg = std::max(f.maxseg, tk[t + 1] - tk[t]);
        }
        if (pool) {
            while (pool->size() % 4) pool->push_back(0);
            f.rec = (long long)(pool->size() / 4);
            for (long long t = 0; t < f.ntiles; ++t) {
                pool->push_back(tk[t]);
                pool->push_back(tk[t + 1]);
                pool->push_back(hs[tk[t]]);
                pool->push_back(hs[tk[t + 1]]);
            }
            f.hs = (long long)pool->size();
            pool->insert(pool->end(), hs.begin(), hs.end());
        }
        if ((int64_t)f.maxseg * n + f.maxseg >= 65536) { out[L] = StreamLevel{}; continue; }   // item ids < 2^16
        {
            // uniform member count: member -> infoset by multiply-shift (verified)
            int um = hs[1] - hs[0];
            for (int k = 1; k < nh && um > 0; ++k)
                if (hs[k + 1] - hs[k] != um) um = 0;
            if (um > 0) {
                int l = 0;
                while ((1 << l) < um) ++l;
                f.udiv_s = 16 + l;
                f.udiv_m = (unsigned)((((unsigned long long)1 << (16 + l)) + (unsigned long long)um - 1) / (unsigned long long)um);
                bool uok = true;
                for (unsigned x = 0; x < 65536u && uok; ++x)
                    uok = (unsigned)(((unsigned long long)x * f.udiv_m) >> f.udiv_s) == x / (unsigned)um;
                f.umem = uok ? um : 0;
            }
        }
        // the deepest decision level: no decision children, so no other forward
        // level reads its reach rows -- its forward pass runs inside this kernel
        f.fused = (fuse_forward && L == g.D - 1 && f.maxm <= kStreamConsumers && (2 * P * w) % 16 == 0) ? 1 : 0;   // gathers: <= 8 per lane, 16-byte pieces
        f.level = L;
        f.compact = (!f.fused && P == 2 && L == g.D - 1 && compact_reach) ? 1 : 0;
        stream_plan(f, P, Pc, w, ix, stages);
        out[L] = f;
    }
    if (pool) pool->resize(pool->size() + 8, 0);   // bulk-copy window slack
    return out;
}

// ints of the stream tables: per level <= 4 (ntiles <= infosets) + 1 per infoset,
// + per-level alignment / terminators and the window slack
static size_t stream_pool_bound(const Game& g) { return (size_t)(5 * g.H + 10 * (int64_t)g.D + 64); }

template <class R, class I>
static size_t fast_pool_bytes(const Game& g, const ShardInfo* sh) {
    const std::vector<int64_t> uoff = u_layout(g, sizeof(R));
    std::vector<int64_t> nu, cu;
    u_rows(g, uoff, nu, cu);
    std::vector<TileD> tiles;
    std::vector<int32_t> coff;
    static const std::vector<uint8_t> none;
    stage_tiles<R>(g, cu, sh ? sh->tile_contrib : none, tiles, coff);
    size_t pool = 0;
    fast_levels<R, I>(g, tiles, &pool);
    return pool;
}

template <class R, class I>
struct Plan {
    size_t U, reach, sig, sig_eval, regret, snum, sden, acc_r, acc_p, dqbase;
    size_t f_parent, f_e, f_pact;
    size_t s_node, s_cb, s_n, s_ebase, s_actor, s_dec, s_coff;
    size_t qbase, owner, tiles, segs, deferred, ctrl, lcnt, out;
    size_t cutbuf, cutrow, cutown, report, pool, spool, plev, gbar, tlev, tmem_of;
    size_t total;
    explicit Plan(const Game& g, const ShardInfo* sh = nullptr) {
        Layout L;
        const size_t NS = (size_t)g.NS, ND = (size_t)g.ND, Q = (size_t)g.Q, H = (size_t)g.H, C = (size_t)g.C;
        U = L.take<R>((size_t)u_layout(g, sizeof(R)).back() * g.Pc + 8);
        reach = L.take<R>(2 * (size_t)g.P * ND);
        sig = L.take<R>(Q + C);
        sig_eval = L.take<R>(Q + C);
        regret = L.take<R>(Q);
        snum = L.take<R>(Q);
        sden = L.take<R>(H);
        const size_t ndq = g.dqbase.empty() ? 0 : (size_t)g.dqbase.back();
        acc_r = L.take<unsigned long long>(3 * ndq + 3 * g.deferred_list.size());   // one exchange block
        acc_p = acc_r + 3 * ndq * sizeof(unsigned long long);
        dqbase = L.take<long long>(g.deferred_list.size() + 1);
        f_parent = L.take<I>(ND);
        f_e = L.take<I>(ND);
        f_pact = L.take<unsigned char>(ND);
        s_node = L.take<I>(NS);
        s_cb = L.take<I>(NS);
        s_n = L.take<int>(NS);
        s_ebase = L.take<I>(NS);
        s_actor = L.take<unsigned char>(NS);
        s_dec = L.take<I>(NS);
        s_coff = L.take<int>(NS);
        qbase = L.take<I>(H + 1);
        owner = L.take<unsigned char>(H);
        tiles = L.take<TileD>(g.tiles.size());
        segs = L.take<SegD>(g.segs.size());
        deferred = L.take<I>(g.deferred_list.size());
        ctrl = L.take<long long>(8);
        lcnt = L.take<unsigned long long>(4 * (size_t)g.D + 4);
        out = L.take<R>(std::max<size_t>(Q + C, (size_t)g.P * 2 + 8));
        const size_t ncut = sh ? sh->cut_row.size() : 0;
        cutbuf = L.take<R>(ncut * g.Pc + 1);
        cutrow = L.take<long long>(ncut + 1);
        cutown = L.take<unsigned char>(ncut + 1);
        report = L.take<unsigned char>(H + 1);
        pool = L.take<unsigned char>(fast_pool_bytes<R, I>(g, sh) + 16);
        spool = L.take<int>(stream_pool_bound(g));
        plev = L.take<PLevel>((size_t)g.D + 1);
        gbar = L.take<unsigned>(4);
        tlev = L.take<TinyLevel>((size_t)g.D + 1);
        tmem_of = L.take<I>(g.V <= (int64_t(1) << 20) ? 2 * H + 2 : 2);
        total = L.off + 256;
    }
};

template <class T, class S>
static std::vector<T> narrow(const std::vector<S>& v) {
    std::vector<T> o(v.size());
    for (size_t k = 0; k < v.size(); ++k) o[k] = (T)v[k];
    return o;
}

template <class R, class I>
struct Solver final : SolverBase {
    const Game* gp;               // the (local) game this rank iterates
    const Game* full;             // the whole game (caller order readbacks)
    cfr_solver_config cfg;
    cudaStream_t stream;
    cudaStream_t cap_stream = nullptr;
    unsigned char* ws;
    const ShardInfo* sh;          // multi-GPU view (cut = -1 on one GPU)
    Plan<R, I> plan;
    DG<R, I> dg;
    cudaGraphExec_t gexec = nullptr;
    int E = 1;
    int64_t launches_per_iter = 0;
    bool use_graph = true;
    bool persist_ = false;        // small game: whole iterations in one cooperative launch (k_persist)
    bool tiny_ = false;           // tiny game: whole iterations in one CTA, state in shared memory (k_tiny)
    TinyPlan tiny_plan_{};
    int persist_grid_ = 0, persist_smem_ = 0;
    bool use_fast_ = true;
    bool use_stream_ = true;
    int stream_debug_ = 0;   // CFR_STREAM_DEBUG (timing experiments; results are garbage when set)
    bool pdl_ = true;
    int num_sms_ = 148;
    int world = 1, rank = 0;
    bool external = false;        // world > 1 without NCCL: the caller runs the exchanges
    ncclComm_t comm = nullptr;

    Solver(const Game* g, const Game* f, const ShardInfo* s_, const cfr_solver_config& c, void* w, cudaStream_t s)
        : gp(g), full(f), cfg(c), stream(s), ws((unsigned char*)w), sh(s_), plan(*g, s_) {
        world = sh->world;
        rank = sh->rank;
    }

    ~Solver() override {
        if (pinned_) cudaFreeHost(pinned_);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (cap_stream) cudaStreamDestroy(cap_stream);
        if (comm) ncclCommDestroy(comm);
    }
    bool sharded() const { return sh->cut >= 0; }
    int64_t ncut() const { return (int64_t)sh->cut_row.size(); }

    template <class T>
    T* at(size_t off) { return reinterpret_cast<T*>(ws + off); }

    template <class T>
    cfr_status up(size_t off, const std::vector<T>& v) {
        if (!v.empty()) CU(cudaMemcpyAsync(ws + off, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
        return CFR_OK;
    }

    size_t acc_bytes() const {
        const size_t ndq = gp->dqbase.empty() ? 0 : (size_t)gp->dqbase.back();
        return (3 * ndq + 3 * gp->deferred_list.size()) * sizeof(unsigned long long);
    }
    std::vector<uint8_t> tile_contrib_;   // set by the sharded path; empty = all tiles contribute
    int contrib_of_tile(size_t t) const { return tile_contrib_.empty() ? 1 : (int)tile_contrib_[t]; }
    std::vector<SmemLayout> lay_;   // per parent level
    int max_smem_ = 0;
    int max_smem_stream_ = 0;
    std::vector<FastLevel> fast_;   // per parent level: recsize > 0 -> pipelined kernel
    std::vector<StreamLevel> stream_;   // per parent level: ntiles > 0 -> streaming (TMA) kernel

    SmemLayout make_layout(int maxch, int maxslot, int maxpairs, int maxseg) const {
        const int Pc = gp->Pc;
        const int w = (int)sizeof(R);
        int off = 0;
        auto take = [&](int bytes) {
            const int o = off;
            off = (off + bytes + 15) & ~15;
            return o;
        };
        const int pairs_b = ((maxpairs * w + 15) & ~15);
        SmemLayout L{};
        L.ch = take(std::max(maxch * w, 2 * pairs_b));
        L.sv = take(maxslot * Pc * w);
        L.spc = take(maxslot * w);
        L.sph = take(maxslot * w);
        L.ssig = take(pairs_b);
        L.sreg = take(pairs_b);
        L.ssn = take(pairs_b);
        L.pib = take(maxseg * w);
        L.zs = take(maxseg * w);
        L.sden = take(maxseg * w);
        L.seg = take(maxseg * (int)sizeof(SegS));
        L.soff = take((maxseg + 1) * 4);
        L.best = take(maxseg * 4);
        L.scoff = take(maxslot * 4);
        L.spoff = take(maxslot * 4);
        L.sn = take(maxslot * 4);
        L.scb = take(maxslot * 8);
        L.pseg = take(maxpairs);
        L.cm = take(maxslot * 2);
        L.ccnt = take(maxseg * 4);
        L.bytes = off;
        return L;
    }

    void build_layouts(const std::vector<TileD>& tiles) {
        const Game& g = *gp;
        lay_.assign(g.D, SmemLayout{});
        max_smem_ = 0;
        for (int L = 0; L < g.D; ++L) {
            int maxch = 0, maxslot = 1, maxpairs = 1, maxseg = 1;
            for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1]; ++t) {
                const TileD& td = tiles[t];
                const int nslot = (int)(td.s1 - td.s0);
                maxslot = std::max(maxslot, nslot);
                maxseg = std::max(maxseg, td.seg1 - td.seg0);
                if (td.npairs <= kTilePairs) maxpairs = std::max(maxpairs, td.npairs);
                int ch = 0;
                if (td.staged == 1) ch = nslot * td.stride;
                else if (td.staged == 2) {
                    for (int64_t s = td.s0; s < td.s1; ++s) ch += (g.s_n[s] * g.Pc) | 1;
                }
                maxch = std::max(maxch, ch);
            }
            lay_[L] = make_layout(maxch, maxslot, maxpairs, maxseg);
            max_smem_ = std::max(max_smem_, lay_[L].bytes);
        }
    }

    cfr_status init(const void* nccl_id) {
        const Game& g = *gp;
        tile_contrib_ = sh->tile_contrib;
        if (world > 1) {
            if (nccl_id) {
                ncclUniqueId id;
                std::memcpy(&id, nccl_id, sizeof(id));
                const ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
                if (r != ncclSuccess) {
                    cfrb_set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
                    return CFR_ERR_NCCL;
                }
            } else {
                external = true;   // the caller performs the two exchanges (cfr_solver_phase)
            }
        }
        if (g.Pc > 4) {
            cfrb_set_error("non-zero-sum games with more than 4 players are not supported by the device kernels");
            return CFR_ERR_UNSUPPORTED;
        }
        if (external && cfg.variant == CFR_PLUS_ALT) {
            cfrb_set_error("alternating updates need the in-graph (NCCL) exchanges when sharded");
            return CFR_ERR_UNSUPPORTED;
        }
        use_graph = !(cfg.flags & CFR_FLAG_NO_GRAPH);
        use_fast_ = !(cfg.flags & CFR_FLAG_NO_PIPELINE);
        use_stream_ = !(cfg.flags & CFR_FLAG_NO_STREAM);
        pdl_ = !(cfg.flags & CFR_FLAG_NO_PDL);
        {
            int dev = 0;
            CU(cudaGetDevice(&dev));
            CU(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, dev));
        }
        // exact-accumulation exponent from the utilities in working precision
        double m = 0.0;
        for (double u : g.util_c) m = std::max(m, std::fabs((double)(R)u));
        if (g.zero_sum_2p) { /* column 2 = -column 1: same max */ }
        E = game_exponent(m);
        dg.U = at<R>(plan.U);
        dg.reach = at<R>(plan.reach);
        dg.sig = at<R>(plan.sig);
        dg.regret = at<R>(plan.regret);
        dg.snum = at<R>(plan.snum);
        dg.sden = at<R>(plan.sden);
        dg.acc_r = at<unsigned long long>(plan.acc_r);
        dg.acc_p = at<unsigned long long>(plan.acc_p);
        dg.dqbase = at<long long>(plan.dqbase);
        dg.f_parent = at<I>(plan.f_parent);
        dg.f_e = at<I>(plan.f_e);
        dg.f_pact = at<unsigned char>(plan.f_pact);
        dg.s_node = at<I>(plan.s_node);
        dg.s_cb = at<I>(plan.s_cb);
        dg.s_n = at<int>(plan.s_n);
        dg.s_ebase = at<I>(plan.s_ebase);
        dg.s_actor = at<unsigned char>(plan.s_actor);
        dg.s_dec = at<I>(plan.s_dec);
        dg.s_coff = at<int>(plan.s_coff);
        dg.qbase = at<I>(plan.qbase);
        dg.owner = at<unsigned char>(plan.owner);
        dg.tiles = at<TileD>(plan.tiles);
        dg.segs = at<SegD>(plan.segs);
        dg.deferred = at<I>(plan.deferred);
        dg.ctrl = at<long long>(plan.ctrl);
        dg.lcnt = at<unsigned long long>(plan.lcnt);
        dg.ndef = (long long)g.deferred_list.size();
        dg.P = g.P;
        dg.variant = cfg.variant;
        dg.upd_player = 0;
        dg.sc0 = std::ldexp(1.0, 40 - E);
        dg.scp0 = std::ldexp(1.0, 40 - 1);
        for (int k = 0; k < 3; ++k) {
            dg.rc[k] = std::ldexp(1.0, E - 40 * (k + 1));
            dg.rcp[k] = std::ldexp(1.0, 1 - 40 * (k + 1));
        }
        // ---- uploads
        cfr_status st;
        // ---- U in device row order (u_rows), per-level 32-byte alignment (u_layout)
        const std::vector<int64_t> uoff = u_layout(g, sizeof(R));
        std::vector<int64_t> s_node_u, s_cb_u;
        u_rows(g, uoff, s_node_u, s_cb_u);
        {
            std::vector<R> u((size_t)uoff.back() * g.Pc + 8, (R)0);
            for (int j = 0; j < g.Pc; ++j) u[j] = (R)g.util_c[j];   // the root (a one-node game)
            const int Pc = g.Pc;
#pragma omp parallel for schedule(static)
            for (int64_t s = 0; s < g.NS; ++s)
                for (int64_t a = 0; a < g.s_n[s]; ++a)
                    for (int j = 0; j < Pc; ++j)
                        u[(size_t)(s_cb_u[s] + a) * Pc + j] = (R)g.util_c[(size_t)(g.s_cb[s] + a) * Pc + j];
            if ((st = up(plan.U, u))) return st;
        }
        // reach rows are indexed by slot: the forward pass walks each level in slot
        // order (parent slot, incoming edge, parent actor per slot)
        std::vector<int64_t> fs_parent(g.NS, -1), fs_e(g.NS, -1), fs_dec(g.NS);
        std::vector<uint8_t> fs_pact(g.NS, 0);
        {
            std::vector<int64_t> sod(g.ND, -1);
            for (int64_t s = 0; s < g.NS; ++s) sod[g.s_dec[s]] = s;
#pragma omp parallel for schedule(static)
            for (int64_t s = 0; s < g.NS; ++s) {
                const int64_t d = g.s_dec[s];
                fs_dec[s] = s;
                fs_parent[s] = g.f_parent[d] < 0 ? -1 : sod[g.f_parent[d]];
                fs_e[s] = g.f_e[d];
                fs_pact[s] = g.f_pact[d];
            }
        }
        std::vector<int32_t> s_coff;
        std::vector<TileD> tiles;
        stage_tiles<R>(g, s_cb_u, tile_contrib_, tiles, s_coff);
        {
            // records of the pipelined levels
            size_t pool = 0;
            fast_ = fast_levels<R, I>(g, tiles, &pool);
            std::vector<unsigned char> rec(pool, 0);
            for (int L = 0; L < g.D; ++L) {
                const FastLevel& f = fast_[L];
                if (f.recsize == 0) continue;
                for (int64_t t = 0; t < f.ntiles; ++t) {
                    const TileH& th = g.tiles[f.tile0 + t];
                    unsigned char* r = rec.data() + f.rec + t * f.recsize;
                    FastHdr hd{th.s0, (int)(th.s1 - th.s0), th.seg1 - th.seg0, th.npairs, 0};
                    std::memcpy(r, &hd, sizeof(hd));
                    FastSeg* sg = reinterpret_cast<FastSeg*>(r + 32);
                    for (int k = th.seg0; k < th.seg1; ++k) {
                        const SegH& shh = g.segs[k];
                        FastSeg fs{};
                        fs.h = shh.h;
                        fs.qb = g.qbase_int[shh.h];
                        fs.pair_off = shh.pair_off;
                        fs.n = (int)(g.qbase_int[shh.h + 1] - g.qbase_int[shh.h]);
                        fs.owner = g.owner_int[shh.h];
                        fs.sb = (int)(shh.sb - th.s0);
                        fs.se = (int)(shh.se - th.s0);
                        sg[k - th.seg0] = fs;
                    }
                    I* node = reinterpret_cast<I*>(r + 32 + (th.seg1 - th.seg0) * sizeof(FastSeg));
                    I* cb = node + (th.s1 - th.s0);
                    I* dec = cb + (th.s1 - th.s0);
                    for (int64_t s = th.s0; s < th.s1; ++s) {
                        node[s - th.s0] = (I)s_node_u[s];
                        cb[s - th.s0] = (I)s_cb_u[s];
                        dec[s - th.s0] = (I)s;   // reach row = slot
                    }
                    // segment of every slot and of every pair (no searches on the device)
                    unsigned char* sseg = reinterpret_cast<unsigned char*>(dec + (th.s1 - th.s0));
                    unsigned char* pseg = sseg + (th.s1 - th.s0);
                    for (int k = th.seg0; k < th.seg1; ++k) {
                        const SegH& shh = g.segs[k];
                        for (int64_t s = shh.sb; s < shh.se; ++s) sseg[s - th.s0] = (unsigned char)(k - th.seg0);
                        const int n = (int)(g.qbase_int[shh.h + 1] - g.qbase_int[shh.h]);
                        for (int a = 0; a < n; ++a) pseg[shh.pair_off + a] = (unsigned char)(k - th.seg0);
                    }
                }
            }
            if ((st = up(plan.pool, rec))) return st;
        }
        {
            // tables of the streaming levels
            std::vector<int> sp;
            int stages = 2;
            if (const char* e = std::getenv("CFR_STREAM_STAGES")) stages = std::max(2, std::min(8, std::atoi(e)));
            if (const char* e = std::getenv("CFR_STREAM_DEBUG")) stream_debug_ = std::atoi(e);
            // members per tile: ~240 f64 / ~480 f32 keeps two CTAs (2-stage rings of
            // ~50 KB) resident per SM (measured best, tools/stream_sweep.py)
            int tile = (sizeof(R) == 4 && !(cfg.flags & CFR_FLAG_FUSED_FORWARD)) ? 2 * kStreamConsumers : kStreamConsumers;
            if (const char* e = std::getenv("CFR_STREAM_TILE")) tile = std::max(32, std::min(1024, std::atoi(e)));
            stream_ = stream_levels<R, I>(g, s_cb_u, &sp, (cfg.flags & CFR_FLAG_FORCE_STREAM) ? 1 : num_sms_, stages, tile,
                                          (cfg.flags & CFR_FLAG_FUSED_FORWARD) != 0, std::getenv("CFR_NO_COMPACT") == nullptr);
            if (sp.size() > stream_pool_bound(g)) {
                cfrb_set_error("internal: stream table bound");
                return CFR_ERR_INVALID_ARG;
            }
            if ((st = up(plan.spool, sp))) return st;
            for (const StreamLevel& f : stream_) max_smem_stream_ = std::max(max_smem_stream_, f.bytes);
        }
        std::vector<SegD> segs(g.segs.size());
        for (size_t k = 0; k < g.segs.size(); ++k) {
            const SegH& sh = g.segs[k];
            SegD sd{};
            sd.h = sh.h;
            sd.qb = g.qbase_int[sh.h];
            sd.n = (int)(g.qbase_int[sh.h + 1] - g.qbase_int[sh.h]);
            sd.owner = g.owner_int[sh.h];
            sd.sb = sh.sb;
            sd.se = sh.se;
            sd.dq = g.dpos[sh.h] >= 0 ? g.dqbase[g.dpos[sh.h]] : -1;
            sd.dh = g.dpos[sh.h];
            sd.pair_off = sh.pair_off;
            sd.fused = sh.fused;
            segs[k] = sd;
        }
        if ((st = up(plan.f_parent, narrow<I>(fs_parent)))) return st;
        if ((st = up(plan.f_e, narrow<I>(fs_e)))) return st;
        if ((st = up(plan.f_pact, fs_pact))) return st;
        if ((st = up(plan.s_node, narrow<I>(s_node_u)))) return st;
        if ((st = up(plan.s_cb, narrow<I>(s_cb_u)))) return st;
        if ((st = up(plan.s_n, g.s_n))) return st;
        if ((st = up(plan.s_ebase, narrow<I>(g.s_ebase)))) return st;
        if ((st = up(plan.s_actor, g.s_actor))) return st;
        if ((st = up(plan.s_dec, narrow<I>(fs_dec)))) return st;
        if ((st = up(plan.s_coff, s_coff))) return st;
        if ((st = up(plan.qbase, narrow<I>(g.qbase_int)))) return st;
        if ((st = up(plan.owner, g.owner_int))) return st;
        if ((st = up(plan.tiles, tiles))) return st;
        build_layouts(tiles);
        if ((st = up(plan.segs, segs))) return st;
        if ((st = up(plan.deferred, narrow<I>(g.deferred_list)))) return st;
        if ((st = up(plan.dqbase, narrow<long long>(g.dqbase)))) return st;
        if (ncut() > 0) {
            // cut rows are local canonical indices of depth-`cut` nodes (owned or
            // not): their U row is inside their parent slot's child row
            const int cut = sh->cut;
            std::vector<std::pair<int64_t, int64_t>> cb_slot;   // (canonical first child, slot) of depth cut-1
            if (cut >= 1)
                for (int64_t s = g.slot_ptr[cut - 1]; s < g.slot_ptr[cut]; ++s) cb_slot.emplace_back(g.s_cb[s], s);
            std::sort(cb_slot.begin(), cb_slot.end());
            std::vector<long long> rows(sh->cut_row.size());
            for (size_t i = 0; i < rows.size(); ++i) {
                const int64_t k = sh->cut_row[i];
                if (cut == 0) { rows[i] = 0; continue; }
                auto it = std::upper_bound(cb_slot.begin(), cb_slot.end(), std::make_pair(k, INT64_MAX));
                if (it == cb_slot.begin() || k >= (it - 1)->first + g.s_n[(it - 1)->second]) {
                    cfrb_set_error("internal: cut node without a parent slot");
                    return CFR_ERR_INVALID_ARG;
                }
                --it;
                rows[i] = s_cb_u[it->second] + (k - it->first);
            }
            if ((st = up(plan.cutrow, rows))) return st;
            if ((st = up(plan.cutown, sh->cut_owned))) return st;
        }
        if (world > 1 && g.H > 0) {
            // report mask in internal infoset order
            if ((st = up(plan.report, sh->report))) return st;
        }
        // sigma^(1) = 1/|A(h)| and chance probabilities (rounded once, Q14)
        {
            std::vector<R> s0(g.Q + g.C);
            for (int64_t h = 0; h < g.H; ++h) {
                const int64_t n = g.qbase_int[h + 1] - g.qbase_int[h];
                for (int64_t q = g.qbase_int[h]; q < g.qbase_int[h + 1]; ++q) s0[q] = (R)1 / (R)n;
            }
            for (int64_t c = 0; c < g.C; ++c) s0[g.Q + c] = (R)g.chance_vals[c];
            if ((st = up(plan.sig, s0))) return st;
            if ((st = up(plan.sig_eval, s0))) return st;
        }
        CU(cudaMemsetAsync(ws + plan.regret, 0, g.Q * sizeof(R), stream));
        CU(cudaMemsetAsync(ws + plan.snum, 0, g.Q * sizeof(R), stream));
        CU(cudaMemsetAsync(ws + plan.sden, 0, g.H * sizeof(R), stream));
        CU(cudaMemsetAsync(ws + plan.acc_r, 0, acc_bytes(), stream));
        CU(cudaMemsetAsync(ws + plan.lcnt, 0, (4 * (size_t)g.D + 4) * sizeof(unsigned long long), stream));
        CU(cudaMemsetAsync(ws + plan.reach, 0, 2 * (size_t)g.P * g.ND * sizeof(R), stream));
        {
            // root reach factors = 1 (Eq 2 / Eq 4 base case); the root is decision 0
            std::vector<R> one(2 * g.P, (R)1);
            if (g.ND > 0) CU(cudaMemcpyAsync(ws + plan.reach, one.data(), one.size() * sizeof(R), cudaMemcpyHostToDevice,
                                             stream));
            std::vector<long long> ctrl = {0, LLONG_MAX, 0, 0, 0, 0, 0, 0};
            if ((st = up(plan.ctrl, ctrl))) return st;
        }
        CU(cudaStreamSynchronize(stream));
        // kernel attributes (dynamic smem above 48 KB needs opt-in)
        // The attribute is per kernel function, shared by every solver of the
        // process: opt in to the device maximum once (occupancy depends only on the
        // dynamic size requested at launch).
        {
            int dev = 0, optin = 0;
            CU(cudaGetDevice(&dev));
            CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            if (max_smem_stream_ > optin) {
                for (StreamLevel& f : stream_) f.ntiles = 0;   // fall back to the tile kernels
                max_smem_stream_ = 0;
            }
            if (max_smem_ > optin) {
                cfrb_set_error("tile shared-memory layout exceeds the device limit");
                return CFR_ERR_UNSUPPORTED;
            }
            CU(set_smem_attr(optin));
        }
        launches_per_iter = count_launches();
        {
            cfr_status ps = setup_persistent();
            if (ps) return ps;
            if ((ps = setup_tiny())) return ps;
        }
        if (use_graph && g.NS > 0 && !external) {
            CU(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
            cudaGraph_t graph;
            CU(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
            cfr_status ls = launch_iteration(cap_stream, nullptr);
            cudaError_t ce = cudaStreamEndCapture(cap_stream, &graph);
            if (ls != CFR_OK) return ls;
            if (ce != cudaSuccess) {
                cfrb_set_error(std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
                return CFR_ERR_CUDA;
            }
            CU(cudaGraphInstantiate(&gexec, graph, 0));
            cudaGraphDestroy(graph);
        }
        return CFR_OK;
    }

    cudaError_t set_smem_attr(int sm) {
        cudaError_t e = cudaSuccess;
#define SETA(PC)                                                                                        \
    e = cudaFuncSetAttribute(k_bwd<R, I, PC, MODE_CFR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
    if (e) return e;                                                                                    \
    e = cudaFuncSetAttribute(k_bwd_fast<R, I, PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);     \
    if (e) return e;                                                                                    \
    e = cudaFuncSetAttribute(k_bwd_stream<R, I, PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);   \
    if (e) return e;                                                                                    \
    e = cudaFuncSetAttribute(k_bwd_stream<R, I, PC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100); \
    if (e) return e;                                                                                    \
    e = cudaFuncSetAttribute(k_bwd<R, I, PC, MODE_VALUES>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
    if (e) return e;                                                                                    \
    e = cudaFuncSetAttribute(k_bwd<R, I, PC, MODE_BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); \
    if (e) return e;
        switch (gp->Pc) {
            case 1: SETA(1) break;
            case 2: SETA(2) break;
            case 3: SETA(3) break;
            default: SETA(4) break;
        }
#undef SETA
        return e;
    }

    // Persistent mode for small games (opt-in, CFR_FLAG_PERSISTENT): one cooperative
    // launch runs T iterations (k_persist).  Measured slower than the PDL graph on
    // B200 (Kuhn 36.6 vs 24.6 us/it, Leduc 134 vs 108): each level's dependent
    // global-memory chain, not the launch, dominates.  Off for sharded solvers.
    static constexpr int64_t kPersistMaxNodes = int64_t(1) << 22;
    cfr_status setup_persistent() {
        const Game& g = *gp;
        persist_ = false;
        if (world > 1 || external || !(cfg.flags & CFR_FLAG_PERSISTENT) || g.NS == 0 || g.V > kPersistMaxNodes ||
            cfg.variant == CFR_PLUS_ALT)
            return CFR_OK;
        int dev = 0, coop = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        if (!coop) return CFR_OK;
        std::vector<PLevel> lv(g.D + 1);
        long long max_units = 1;
        for (int l = 0; l < g.D; ++l) {
            lv[l].s0 = g.slot_ptr[l];
            lv[l].s1 = g.slot_ptr[l + 1];
            lv[l].t0 = g.tile_ptr[l];
            lv[l].t1 = g.tile_ptr[l + 1];
            lv[l].lay = lay_[l];
            max_units = std::max<long long>(max_units, lv[l].t1 - lv[l].t0);
            max_units = std::max<long long>(max_units, (lv[l].s1 - lv[l].s0 + 1023) / 1024);
        }
        persist_smem_ = std::max(16, max_smem_);
        void* fn = persist_fn();
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, persist_smem_));
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTileSlots, persist_smem_));
        if (per_sm < 1) return CFR_OK;
        persist_grid_ = (int)std::min<long long>((long long)num_sms_ * per_sm, max_units);
        cfr_status st = up(plan.plev, lv);
        if (st) return st;
        CU(cudaMemsetAsync(ws + plan.gbar, 0, 4 * sizeof(unsigned), stream));
        CU(cudaStreamSynchronize(stream));
        persist_ = true;
        return CFR_OK;
    }
    void* persist_fn() const {
        const int Pc = gp->Pc;
        const bool p2 = gp->P == 2;
        switch (Pc) {
            case 1: return p2 ? (void*)k_persist<R, I, 1, 2> : (void*)k_persist<R, I, 1, 0>;
            case 2: return p2 ? (void*)k_persist<R, I, 2, 2> : (void*)k_persist<R, I, 2, 0>;
            case 3: return p2 ? (void*)k_persist<R, I, 3, 2> : (void*)k_persist<R, I, 3, 0>;
            default: return p2 ? (void*)k_persist<R, I, 4, 2> : (void*)k_persist<R, I, 4, 0>;
        }
    }
    cfr_status launch_persistent(int64_t iters) {
        const Game& g = *gp;
        const PLevel* lv = at<PLevel>(plan.plev);
        int D = g.D;
        int has_def = has_def_() ? 1 : 0;
        long long T = (long long)iters;
        unsigned* bar = at<unsigned>(plan.gbar);
        void* args[] = {(void*)&dg, (void*)&lv, (void*)&D, (void*)&has_def, (void*)&T, (void*)&bar};
        CU(cudaLaunchCooperativeKernel(persist_fn(), dim3(persist_grid_), dim3(kTileSlots), args, (size_t)persist_smem_,
                                       stream));
        return CFR_OK;
    }
    bool has_def_() const { return !gp->deferred_list.empty(); }

    void* tiny_fn() const {
        switch (gp->Pc) {
            case 1: return (void*)k_tiny<R, I, 1>;
            case 2: return (void*)k_tiny<R, I, 2>;
            case 3: return (void*)k_tiny<R, I, 3>;
            default: return (void*)k_tiny<R, I, 4>;
        }
    }
    // Tiny-game mode (k_tiny): single-GPU, depth-homogeneous games whose mutable
    // state fits one CTA's shared memory.  On by default (CFR_FLAG_NO_TINY to opt out).
    cfr_status setup_tiny() {
        const Game& g = *gp;
        tiny_ = false;
        if (world > 1 || external || persist_ || (cfg.flags & CFR_FLAG_NO_TINY) || !g.depth_homogeneous || g.NS == 0)
            return CFR_OK;
        const long long nU = (long long)(plan_u_rows()) * g.Pc, nreach = 2LL * g.P * g.NS, nsig = g.Q + g.C;
        TinyPlan tp{};
        long long o = 0;
        auto take = [&](long long n) { const long long r = o; o += (n + 1) & ~1LL; return r; };   // 16-byte aligned
        tp.U = take(nU);
        tp.reach = take(nreach);
        tp.sig = take(nsig);
        tp.reg = take(g.Q);
        tp.snum = take(g.Q);
        tp.sden = take(g.H);
        tp.rt = take(g.Q);
        tp.pib = take(g.H);
        tp.nU = nU;
        tp.nreach = nreach;
        tp.nsig = nsig;
        tp.Q = g.Q;
        tp.H = g.H;
        const long long bytes = o * (long long)sizeof(R);
        int dev = 0, optin = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (bytes > optin - 1024) return CFR_OK;
        tp.bytes = (int)bytes;
        // per level: slots and its (consecutive) infosets; members of each infoset
        std::vector<TinyLevel> lv(g.D + 1, TinyLevel{0, 0, 0, 0});
        std::vector<int64_t> mem(2 * (size_t)g.H + 2, -1);
        for (int L = 0; L < g.D; ++L) {
            lv[L].s0 = g.slot_ptr[L];
            lv[L].s1 = g.slot_ptr[L + 1];
            long long h0 = LLONG_MAX, h1 = -1;
            for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1]; ++t)
                for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1; ++k) {
                    const SegH& sg = g.segs[k];
                    const int64_t h = sg.h;
                    mem[2 * h] = mem[2 * h] < 0 ? sg.sb : std::min<int64_t>(mem[2 * h], sg.sb);
                    mem[2 * h + 1] = std::max<int64_t>(mem[2 * h + 1], sg.se);
                    h0 = std::min<long long>(h0, h);
                    h1 = std::max<long long>(h1, h + 1);
                }
            if (h1 > h0) {
                lv[L].h0 = h0;
                lv[L].h1 = h1;
            }
        }
        for (int64_t h = 0; h < g.H; ++h)
            if (mem[2 * h] < 0) return CFR_OK;
        for (int L = 0; L < g.D; ++L)   // each level's infosets must be a consecutive id range
            for (long long h = lv[L].h0; h < lv[L].h1; ++h)
                if (mem[2 * h] < g.slot_ptr[L] || mem[2 * h + 1] > g.slot_ptr[L + 1]) return CFR_OK;
        CU(cudaFuncSetAttribute(tiny_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, tp.bytes));
        cfr_status st = up(plan.tlev, lv);
        if (st) return st;
        if ((st = up(plan.tmem_of, narrow<I>(mem)))) return st;
        CU(cudaStreamSynchronize(stream));
        tiny_plan_ = tp;
        tiny_ = true;
        return CFR_OK;
    }
    long long plan_u_rows() const { return (long long)u_layout(*gp, sizeof(R)).back(); }
    cfr_status launch_tiny(int64_t iters) {
        const Game& g = *gp;
        const TinyLevel* lv = reinterpret_cast<const TinyLevel*>(ws + plan.tlev);
        const I* mem = reinterpret_cast<const I*>(ws + plan.tmem_of);
        const int D = g.D;
        const long long T = (long long)iters;
        const TinyPlan tp = tiny_plan_;
        switch (g.Pc) {
            case 1: launch(pdl_, k_tiny<R, I, 1>, dim3(1), dim3(1024), (size_t)tp.bytes, stream, dg, lv, mem, D, T, tp); break;
            case 2: launch(pdl_, k_tiny<R, I, 2>, dim3(1), dim3(1024), (size_t)tp.bytes, stream, dg, lv, mem, D, T, tp); break;
            case 3: launch(pdl_, k_tiny<R, I, 3>, dim3(1), dim3(1024), (size_t)tp.bytes, stream, dg, lv, mem, D, T, tp); break;
            default: launch(pdl_, k_tiny<R, I, 4>, dim3(1), dim3(1024), (size_t)tp.bytes, stream, dg, lv, mem, D, T, tp); break;
        }
        CU(cudaGetLastError());
        return CFR_OK;
    }

    int64_t count_launches() const {
        const Game& g = *gp;
        int64_t n = 0;
        for (int l = 1; l < g.D; ++l)
            if (g.slot_ptr[l + 1] > g.slot_ptr[l] && !fwd_fused(l)) ++n;
        for (int L = g.D - 1; L >= 0; --L)
            if (g.tile_ptr[L + 1] > g.tile_ptr[L]) ++n;
        if (!g.deferred_list.empty()) ++n;
        return (cfg.variant == CFR_PLUS_ALT) ? n * g.P : n;   // alternating updates: one pass per player
    }

    // the deepest level's reach rows in compact (actor-only) form: CFR iterations
    // whose backward pass there is the (unfused) streaming kernel, two players
    bool fwd_compact(int l) const {
        return gp->P == 2 && l == gp->D - 1 && use_stream_ && l < (int)stream_.size() && stream_[l].ntiles > 0 &&
               !stream_[l].fused && stream_[l].compact;
    }
    void fwd_level(cudaStream_t st, const R* sig, int l, int compact = 0) {
        const Game& g = *gp;
        const long long s0 = g.slot_ptr[l], s1 = g.slot_ptr[l + 1];   // reach rows = slots
        if (s1 <= s0) return;
        const long long n = s1 - s0;
        const int threads = 256;
        const long long per_block = (g.P == 2) ? threads * CFR_FWD_FW : threads;
        const long long blocks = std::min<long long>((n + per_block - 1) / per_block, 148LL * 16);
        if (g.P == 2)
            launch(pdl_, k_fwd<R, I, 2>, dim3((unsigned)blocks), dim3(threads), 0, st, dg, sig, (long long)s0, (long long)s1,
                   compact);
        else
            launch(pdl_, k_fwd<R, I, 0>, dim3((unsigned)blocks), dim3(threads), 0, st, dg, sig, (long long)s0, (long long)s1,
                   0);
    }

    template <int MODE>
    void bwd_level(cudaStream_t st, const R* sig, int L, int br_player, int last) {
        const Game& g = *gp;
        const long long t0 = g.tile_ptr[L], t1 = g.tile_ptr[L + 1];
        if (t1 <= t0) return;
        if (MODE == MODE_CFR && sig == dg.sig && use_stream_ && stream_[L].ntiles > 0) {
            StreamLevel f = stream_[L];
            f.last = last;
            f.debug = stream_debug_;
            int per_sm = 1;
            switch (g.Pc) {
                case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_stream<R, I, 1>, kStreamThreads, f.bytes); break;
                case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_stream<R, I, 2>, kStreamThreads, f.bytes); break;
                case 3: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_stream<R, I, 3>, kStreamThreads, f.bytes); break;
                default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_stream<R, I, 4>, kStreamThreads, f.bytes); break;
            }
            per_sm = std::max(1, per_sm);
            const unsigned nb = (unsigned)std::min<long long>(f.ntiles, (long long)num_sms_ * per_sm);
            if (std::getenv("CFR_STREAM_VERBOSE"))
                std::fprintf(stderr, "[stream] level %d: %lld tiles, maxm %d, maxseg %d, smem %d B, %d CTA/SM, grid %u\n", L,
                             f.ntiles, f.maxm, f.maxseg, f.bytes, per_sm, nb);
            const int* sp = at<int>(plan.spool);
            switch (g.Pc) {
                case 1: launch(pdl_, k_bwd_stream<R, I, 1>, dim3(nb), dim3(kStreamThreads), (size_t)f.bytes, st, dg, sp, f); break;
                case 2: launch(pdl_, k_bwd_stream<R, I, 2>, dim3(nb), dim3(kStreamThreads), (size_t)f.bytes, st, dg, sp, f); break;
                case 3: launch(pdl_, k_bwd_stream<R, I, 3>, dim3(nb), dim3(kStreamThreads), (size_t)f.bytes, st, dg, sp, f); break;
                default: launch(pdl_, k_bwd_stream<R, I, 4>, dim3(nb), dim3(kStreamThreads), (size_t)f.bytes, st, dg, sp, f); break;
            }
            return;
        }
        // pipelined kernel: measured faster for f64 only (f32 tiles move half the bytes)
        if (MODE == MODE_CFR && sizeof(R) == 8 && sig == dg.sig && use_fast_ && fast_[L].recsize > 0) {
            FastLevel f = fast_[L];
            f.last = last;
            const int bytes = fast_plan(f, g.Pc, (int)sizeof(R)).bytes;
            int per_sm = 1;
            switch (g.Pc) {
                case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_fast<R, I, 1>, 2 * kTileSlots, bytes); break;
                case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_fast<R, I, 2>, 2 * kTileSlots, bytes); break;
                case 3: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_fast<R, I, 3>, 2 * kTileSlots, bytes); break;
                default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_fast<R, I, 4>, 2 * kTileSlots, bytes); break;
            }
            per_sm = std::max(1, per_sm);
            const unsigned nb = (unsigned)std::min<long long>(f.ntiles, (long long)num_sms_ * per_sm);
            switch (g.Pc) {
                case 1: launch(pdl_, k_bwd_fast<R, I, 1>, dim3(nb), dim3(2 * kTileSlots), (size_t)bytes, st, dg, (const unsigned char*)at<unsigned char>(plan.pool), f); break;
                case 2: launch(pdl_, k_bwd_fast<R, I, 2>, dim3(nb), dim3(2 * kTileSlots), (size_t)bytes, st, dg, (const unsigned char*)at<unsigned char>(plan.pool), f); break;
                case 3: launch(pdl_, k_bwd_fast<R, I, 3>, dim3(nb), dim3(2 * kTileSlots), (size_t)bytes, st, dg, (const unsigned char*)at<unsigned char>(plan.pool), f); break;
                default: launch(pdl_, k_bwd_fast<R, I, 4>, dim3(nb), dim3(2 * kTileSlots), (size_t)bytes, st, dg, (const unsigned char*)at<unsigned char>(plan.pool), f); break;
            }
            return;
        }
        const SmemLayout lay = lay_[L];
        const size_t sm = (size_t)lay.bytes;
        const unsigned nb = (unsigned)(t1 - t0);
        switch (g.Pc) {
            case 1: launch(pdl_, k_bwd<R, I, 1, MODE>, dim3(nb), dim3(kTileSlots), sm, st, dg, sig, (long long)t0, br_player, last, lay); break;
            case 2: launch(pdl_, k_bwd<R, I, 2, MODE>, dim3(nb), dim3(kTileSlots), sm, st, dg, sig, (long long)t0, br_player, last, lay); break;
            case 3: launch(pdl_, k_bwd<R, I, 3, MODE>, dim3(nb), dim3(kTileSlots), sm, st, dg, sig, (long long)t0, br_player, last, lay); break;
            default: launch(pdl_, k_bwd<R, I, 4, MODE>, dim3(nb), dim3(kTileSlots), sm, st, dg, sig, (long long)t0, br_player, last, lay); break;
        }
    }

    void deferred_update(cudaStream_t st, int last) {
        const long long n = dg.ndef;
        const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8));
        launch(pdl_, k_deferred<R, I>, dim3(blocks), dim3(256), 0, st, dg, last);
    }

    // ---- iteration phases.  One iteration = lower (forward + backward of the
    // owned levels, down to the cut) -> [exchange 1: cut values] -> upper (trunk
    // backward) -> [exchange 2: deferred exact sums] -> deferred update.  On one
    // GPU the cut is -1: lower is the whole pass and both exchanges vanish.
    // `ev` (optional) collects (tag, level, event) for profiling: tag 0 forward,
    // 1 backward, 2 deferred update, 3 exchange.
    struct Mark {
        int tag, level;
        cudaEvent_t e;
    };
    void mark(cudaStream_t st, std::vector<Mark>* ev, int tag, int level) {
        if (!ev) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev->push_back(Mark{tag, level, e});
    }
    bool has_def() const { return !gp->deferred_list.empty(); }

    // forward level l runs inside the streaming backward kernel of level l
    bool fwd_fused(int l) const { return use_stream_ && l < (int)stream_.size() && stream_[l].ntiles > 0 && stream_[l].fused; }

    void launch_lower(cudaStream_t st, int mode, const R* sig, std::vector<Mark>* ev) {
        const Game& g = *gp;
        if (mode == MODE_CFR)
            for (int l = 1; l < g.D; ++l) {
                if (sig == dg.sig && fwd_fused(l)) continue;
                fwd_level(st, sig, l, (sig == dg.sig && fwd_compact(l)) ? 1 : 0);
                mark(st, ev, 0, l);
            }
        const int stop = sharded() ? sh->cut : 0;
        for (int L = g.D - 1; L >= stop; --L) {
            const int last = (mode == MODE_CFR && L == 0 && !has_def() && pass_final_) ? 1 : 0;
            if (mode == MODE_CFR) bwd_level<MODE_CFR>(st, sig, L, 0, last);
            else bwd_level<MODE_VALUES>(st, sig, L, 0, 0);
            mark(st, ev, 1, L);
        }
        if (sharded()) {
            const long long n = ncut();
            const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148));
            k_cut_pack<R><<<nb, 256, 0, st>>>(dg.U, at<long long>(plan.cutrow), at<unsigned char>(plan.cutown),
                                              at<R>(plan.cutbuf), n, g.Pc);
        }
    }
    void launch_upper(cudaStream_t st, int mode, const R* sig, std::vector<Mark>* ev) {
        const Game& g = *gp;
        if (!sharded()) return;
        const long long n = ncut();
        const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148));
        k_cut_unpack<R><<<nb, 256, 0, st>>>(dg.U, at<long long>(plan.cutrow), at<R>(plan.cutbuf), n, g.Pc);
        for (int L = sh->cut - 1; L >= 0; --L) {
            const int last = (mode == MODE_CFR && L == 0 && !has_def() && pass_final_) ? 1 : 0;
            if (mode == MODE_CFR) bwd_level<MODE_CFR>(st, sig, L, 0, last);
            else bwd_level<MODE_VALUES>(st, sig, L, 0, 0);
            mark(st, ev, 1, L);
        }
    }
    void launch_update(cudaStream_t st, std::vector<Mark>* ev) {
        if (has_def()) {
            deferred_update(st, pass_final_ ? 1 : 0);
            mark(st, ev, 2, -1);
        }
    }
    cfr_status nccl_sum(cudaStream_t st, void* buf, size_t count, ncclDataType_t t) {
        if (!comm || count == 0) return CFR_OK;
        const ncclResult_t r = ncclAllReduce(buf, buf, count, t, ncclSum, comm, st);
        if (r != ncclSuccess) {
            cfrb_set_error(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
            return CFR_ERR_NCCL;
        }
        return CFR_OK;
    }
    static ncclDataType_t rtype() { return sizeof(R) == 8 ? ncclFloat64 : ncclFloat32; }

    // One iteration: one pass, or (alternating updates, variant 4) one pass per
    // player, each a full forward + backward under the current profile updating
    // only that player's infosets (reading Q19).  The iteration counter advances
    // in the last kernel of the final pass.
    int pass_final_ = 1;
    cfr_status launch_iteration(cudaStream_t st, std::vector<Mark>* ev) {
        const Game& g = *gp;
        cfr_status s = CFR_OK;
        const int passes = (cfg.variant == CFR_PLUS_ALT) ? g.P : 1;
        mark(st, ev, -1, 0);
        for (int pass = 1; pass <= passes && !s; ++pass) {
            dg.upd_player = (passes > 1) ? pass : 0;
            pass_final_ = (pass == passes) ? 1 : 0;
            launch_lower(st, MODE_CFR, dg.sig, ev);
            if (sharded()) {
                if ((s = nccl_sum(st, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype()))) break;
                mark(st, ev, 3, -1);
                launch_upper(st, MODE_CFR, dg.sig, ev);
            }
            if (world > 1 && has_def()) {
                if ((s = nccl_sum(st, dg.acc_r, acc_bytes() / 8, ncclInt64))) break;
                mark(st, ev, 3, -1);
            }
            launch_update(st, ev);
        }
        dg.upd_player = 0;
        pass_final_ = 1;
        if (s) return s;
        CU(cudaGetLastError());
        return CFR_OK;
    }

    cfr_status enqueue(int64_t iters) override {
        if (gp->NS == 0) return CFR_OK;   // one-node game: nothing to iterate
        if (external) {
            cfrb_set_error("world_size > 1 without an NCCL id: drive the iteration with cfr_solver_phase");
            return CFR_ERR_UNSUPPORTED;
        }
        if (persist_ && iters > 0) return launch_persistent(iters);
        if (tiny_ && iters > 0) return launch_tiny(iters);
        for (int64_t k = 0; k < iters; ++k) {
            if (gexec) CU(cudaGraphLaunch(gexec, stream));
            else {
                cfr_status s = launch_iteration(stream, nullptr);
                if (s) return s;
            }
        }
        return CFR_OK;
    }

    cfr_status sync() override {
        CU(cudaStreamSynchronize(stream));
        long long c[2];
        CU(cudaMemcpy(c, dg.ctrl, sizeof(c), cudaMemcpyDeviceToHost));
        if (c[1] != LLONG_MAX) {
            cfrb_set_error("NaN/Inf in regrets or strategy at iteration " + std::to_string(c[1]));
            return CFR_ERR_NUMERICAL;
        }
        return CFR_OK;
    }

    cfr_status iteration(int64_t* T) override {
        CU(cudaStreamSynchronize(stream));
        long long c;
        CU(cudaMemcpy(&c, dg.ctrl, sizeof(c), cudaMemcpyDeviceToHost));
        *T = c;
        return CFR_OK;
    }

    // device buffer (internal q order) -> host doubles in caller order
    // Multi-GPU readback combination: every rank zeroes what it does not report
    // (trunk + deferred infosets: rank 0; shard-local infosets: their owner) and a
    // sum-allreduce completes the array (exact: one nonzero contribution).  In the
    // external mode the caller sums the partial arrays itself.
    cfr_status combine_q(R* dptr) {
        const Game& g = *gp;
        if (world <= 1) return CFR_OK;
        const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((g.H + 255) / 256, 148LL * 8));
        if (g.H) k_mask_q<R, I><<<nb, 256, 0, stream>>>(dptr, dg.qbase, at<unsigned char>(plan.report), g.H);
        CU(cudaGetLastError());
        return nccl_sum(stream, dptr, (size_t)g.Q, rtype());
    }
    cfr_status combine_h(R* dptr) {
        const Game& g = *gp;
        if (world <= 1) return CFR_OK;
        const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((g.H + 255) / 256, 148LL * 8));
        if (g.H) k_mask_h<R><<<nb, 256, 0, stream>>>(dptr, at<unsigned char>(plan.report), g.H);
        CU(cudaGetLastError());
        return nccl_sum(stream, dptr, (size_t)g.H, rtype());
    }

    // device buffer (internal q order) -> combined -> host doubles in caller order
    // pinned host staging for readbacks (allocated on first use)
    R* pinned_ = nullptr;
    size_t pinned_n_ = 0;
    cfr_status staging(size_t n, R** out) {
        if (pinned_n_ < n) {
            if (pinned_) cudaFreeHost(pinned_);
            pinned_ = nullptr;
            pinned_n_ = 0;
            CU(cudaMallocHost(&pinned_, std::max<size_t>(n, 1) * sizeof(R)));
            pinned_n_ = n;
        }
        *out = pinned_;
        return CFR_OK;
    }
    cfr_status read_q(const R* dptr, double* out) {
        const Game& g = *gp;
        const R* src = dptr;
        if (world > 1) {
            R* tmpd = at<R>(plan.out);
            if (g.Q) CU(cudaMemcpyAsync(tmpd, dptr, g.Q * sizeof(R), cudaMemcpyDeviceToDevice, stream));
            cfr_status s = combine_q(tmpd);
            if (s) return s;
            src = tmpd;
        }
        R* tmp = nullptr;
        cfr_status s = staging((size_t)g.Q, &tmp);
        if (s) return s;
        if (g.Q) CU(cudaMemcpyAsync(tmp, src, g.Q * sizeof(R), cudaMemcpyDeviceToHost, stream));
        CU(cudaStreamSynchronize(stream));
#pragma omp parallel for schedule(static)
        for (int64_t hc = 0; hc < g.H; ++hc) {
            const int64_t hi = g.h_int_of_caller[hc];
            const int64_t n = g.qbase_caller[hc + 1] - g.qbase_caller[hc];
            for (int64_t a = 0; a < n; ++a) out[g.qbase_caller[hc] + a] = (double)tmp[g.qbase_int[hi] + a];
        }
        return CFR_OK;
    }

    cfr_status compute_average() {
        const Game& g = *gp;
        const long long n = std::max<long long>(g.H, g.C);
        const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8));
        k_average<R, I><<<blocks, 256, 0, stream>>>(dg, at<R>(plan.sig_eval), g.H, g.Q, g.C);
        CU(cudaGetLastError());
        return CFR_OK;
    }

    cfr_status strategy(int which, double* out) override {
        CU(cudaStreamSynchronize(stream));
        if (which == 0) {
            cfr_status s = compute_average();
            if (s) return s;
            return read_q(at<R>(plan.sig_eval), out);
        }
        return read_q(dg.sig, out);
    }

    cfr_status get_state(double* regret, double* snum, double* sden) override {
        const Game& g = *gp;
        cfr_status s;
        if (regret && (s = read_q(dg.regret, regret))) return s;
        if (snum && (s = read_q(dg.snum, snum))) return s;
        if (sden) {
            R* tmpd = at<R>(plan.out);
            if (g.H) CU(cudaMemcpyAsync(tmpd, dg.sden, g.H * sizeof(R), cudaMemcpyDeviceToDevice, stream));
            if ((s = combine_h(tmpd))) return s;
            std::vector<R> tmp(g.H);
            if (g.H) CU(cudaMemcpyAsync(tmp.data(), tmpd, g.H * sizeof(R), cudaMemcpyDeviceToHost, stream));
            CU(cudaStreamSynchronize(stream));
            for (int64_t hc = 0; hc < g.H; ++hc) sden[hc] = (double)tmp[g.h_int_of_caller[hc]];
        }
        return CFR_OK;
    }

    cfr_status read_root(double* out) {
        const Game& g = *gp;
        std::vector<R> r(g.Pc);
        CU(cudaMemcpyAsync(r.data(), dg.U, g.Pc * sizeof(R), cudaMemcpyDeviceToHost, stream));
        CU(cudaStreamSynchronize(stream));
        if (g.zero_sum_2p) {
            out[0] = (double)r[0];
            out[1] = (double)(-r[0]);
        } else {
            for (int j = 0; j < g.P; ++j) out[j] = (double)r[j];
        }
        return CFR_OK;
    }

    // values-only backward pass under `sig` -> root values (P entries, double)
    cfr_status root_values(const R* sig, double* out) {
        const Game& g = *gp;
        launch_lower(stream, MODE_VALUES, sig, nullptr);
        if (sharded()) {
            cfr_status s = nccl_sum(stream, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype());
            if (s) return s;
            launch_upper(stream, MODE_VALUES, sig, nullptr);
        }
        CU(cudaGetLastError());
        return read_root(out);
    }

    cfr_status expected_values(int which, double* out) override {
        if (external) {
            cfrb_set_error("world_size > 1 without an NCCL id: use cfr_solver_phase (EV phases)");
            return CFR_ERR_UNSUPPORTED;
        }
        CU(cudaStreamSynchronize(stream));
        const R* sig = dg.sig;
        if (which == CFR_EV_AVERAGE) {
            cfr_status s = compute_average();
            if (s) return s;
            sig = at<R>(plan.sig_eval);
        }
        return root_values(sig, out);
    }

    cfr_status exploitability(double* nc, double* ex, double* br) override {
        const Game& g = *gp;
        if (world > 1) {
            cfrb_set_error("device best response is single-GPU in this version (DESIGN.md §9)");
            return CFR_ERR_UNSUPPORTED;
        }
        if (!g.depth_homogeneous || !g.deferred_list.empty()) {
            cfrb_set_error("device best response needs every infoset on one depth and inside one tile (reading Q17)");
            return CFR_ERR_UNSUPPORTED;
        }
        CU(cudaStreamSynchronize(stream));
        cfr_status s = compute_average();
        if (s) return s;
        const R* sig = at<R>(plan.sig_eval);
        double ev[16];
        if ((s = root_values(sig, ev))) return s;
        // forward pass under sigma_bar: pi_check(., i) for every player
        for (int l = 1; l < g.D; ++l) fwd_level(stream, sig, l);
        double total = 0.0;
        for (int i = 1; i <= g.P; ++i) {
            for (int L = g.D - 1; L >= 0; --L) bwd_level<MODE_BR>(stream, sig, L, i, 0);
            CU(cudaGetLastError());
            std::vector<R> r(g.Pc);
            CU(cudaMemcpyAsync(r.data(), dg.U, g.Pc * sizeof(R), cudaMemcpyDeviceToHost, stream));
            CU(cudaStreamSynchronize(stream));
            double b;
            if (g.zero_sum_2p) b = (i == 1) ? (double)r[0] : (double)(-r[0]);
            else b = (double)r[i - 1];
            if (br) br[i - 1] = b;
            total = total + (b - ev[i - 1]);
        }
        // restore the reach arrays of the current strategy is unnecessary: every
        // iteration recomputes them.  Root reach stays 1.
        *nc = total;
        *ex = total / (double)g.P;
        return CFR_OK;
    }

    cfr_status launches(int64_t* n) override {
        *n = (persist_ || tiny_) ? 1 : launches_per_iter;   // one launch per enqueue of T iterations
        return CFR_OK;
    }

    cfr_status profile(int64_t iters, double* out) override {
        const Game& g = *gp;
        for (int k = 0; k < 5; ++k) out[k] = 0.0;
        if (g.NS == 0 || iters <= 0) return CFR_OK;
        if (external) {
            cfrb_set_error("profile needs NCCL or a single GPU");
            return CFR_ERR_UNSUPPORTED;
        }
        std::vector<double> per_bwd(g.D, 0.0), per_fwd(g.D, 0.0);
        std::vector<unsigned long long> c0, c1;
        cfr_status cs = read_lcnt(c0);
        if (cs) return cs;
        for (int64_t it = 0; it < iters; ++it) {
            std::vector<Mark> ev;
            cfr_status s = launch_iteration(stream, &ev);
            if (s) return s;
            CU(cudaStreamSynchronize(stream));
            for (size_t e = 1; e < ev.size(); ++e) {
                float ms = 0;
                cudaEventElapsedTime(&ms, ev[e - 1].e, ev[e].e);
                switch (ev[e].tag) {
                    case 0: out[0] += ms; per_fwd[ev[e].level] += ms; break;
                    case 1: out[1] += ms; per_bwd[ev[e].level] += ms; break;
                    case 2: out[2] += ms; break;
                    default: out[2] += ms; break;   // exchanges are reported with the update
                }
            }
            for (auto& m : ev) cudaEventDestroy(m.e);
        }
        if ((cs = read_lcnt(c1))) return cs;
        // live (updated) infosets / pairs per iteration of the streaming levels
        prof_live_.assign(2 * (size_t)g.D, -1.0);
        for (int L = 0; L < g.D; ++L)
            if (c1[4 * L + 2] > c0[4 * L + 2]) {
                prof_live_[2 * L] = (double)(c1[4 * L + 0] - c0[4 * L + 0]) / (double)iters;
                prof_live_[2 * L + 1] = (double)(c1[4 * L + 1] - c0[4 * L + 1]) / (double)iters;
            }
        int dom = 0;
        for (int L = 0; L < g.D; ++L)
            if (per_bwd[L] > per_bwd[dom]) dom = L;
        out[0] /= iters;
        out[1] /= iters;
        out[2] /= iters;
        out[3] = per_bwd[dom] / iters;
        out[4] = dom;
        dom_level = dom;
        prof_fwd_ms_.assign(g.D, 0.0);
        prof_bwd_ms_.assign(g.D, 0.0);
        for (int L = 0; L < g.D; ++L) {
            prof_fwd_ms_[L] = per_fwd[L] / iters;
            prof_bwd_ms_[L] = per_bwd[L] / iters;
        }
        return sync();
    }
    std::vector<double> prof_fwd_ms_, prof_bwd_ms_;   // per level, last profile window
    cfr_status level_profile(double* out, int32_t max_levels, int32_t* num_levels) override {
        const Game& g = *gp;
        *num_levels = g.D;
        for (int L = 0; L < g.D && L < max_levels; ++L) {
            out[4 * L + 0] = L < (int)prof_fwd_ms_.size() ? prof_fwd_ms_[L] : 0.0;
            out[4 * L + 1] = L < (int)prof_bwd_ms_.size() ? prof_bwd_ms_[L] : 0.0;
            out[4 * L + 2] = level_fwd_bytes(L);
            out[4 * L + 3] = (g.tile_ptr[L + 1] > g.tile_ptr[L]) ? level_bwd_bytes(L) : 0.0;
        }
        return CFR_OK;
    }

    // ---- externally driven multi-GPU iteration (tests; world > 1 without NCCL)
    cfr_status phase(int ph, double* out) override {
        const Game& g = *gp;
        if (g.NS == 0) return CFR_OK;
        switch (ph) {
            case 0: launch_lower(stream, MODE_CFR, dg.sig, nullptr); break;
            case 1: launch_upper(stream, MODE_CFR, dg.sig, nullptr); break;
            case 2: launch_update(stream, nullptr); break;
            case 3: {
                cfr_status s = compute_average();
                if (s) return s;
                launch_lower(stream, MODE_VALUES, at<R>(plan.sig_eval), nullptr);
                break;
            }
            case 4: {
                launch_upper(stream, MODE_VALUES, at<R>(plan.sig_eval), nullptr);
                if (out) {
                    cfr_status s = read_root(out);
                    if (s) return s;
                }
                break;
            }
            default:
                cfrb_set_error("bad phase");
                return CFR_ERR_INVALID_ARG;
        }
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(stream));
        return CFR_OK;
    }
    cfr_status exchange_size(int which, size_t* bytes) override {
        if (which == 0) *bytes = (size_t)ncut() * gp->Pc * sizeof(R);
        else if (which == 1) *bytes = acc_bytes();
        else {
            cfrb_set_error("bad exchange id");
            return CFR_ERR_INVALID_ARG;
        }
        return CFR_OK;
    }
    cfr_status exchange(int which, int put, void* host, size_t bytes) override {
        size_t need = 0;
        cfr_status s = exchange_size(which, &need);
        if (s) return s;
        if (bytes != need) {
            cfrb_set_error("exchange buffer size mismatch: need " + std::to_string(need));
            return CFR_ERR_INVALID_ARG;
        }
        if (need == 0) return CFR_OK;
        unsigned char* dev = (which == 0) ? ws + plan.cutbuf : (unsigned char*)dg.acc_r;
        CU(cudaStreamSynchronize(stream));
        if (put) CU(cudaMemcpy(dev, host, need, cudaMemcpyHostToDevice));
        else CU(cudaMemcpy(host, dev, need, cudaMemcpyDeviceToHost));
        return CFR_OK;
    }
    cfr_status shard_info(int64_t* out) override {
        const Game& g = *gp;
        out[0] = sh->cut;
        out[1] = ncut();
        out[2] = sh->owned_nodes;
        out[3] = g.V;
        out[4] = g.NS;
        out[5] = (int64_t)g.deferred_list.size();
        out[6] = g.dqbase.empty() ? 0 : g.dqbase.back();
        out[7] = world;
        return CFR_OK;
    }

    int level_kernel(int L) const {
        const Game& g = *gp;
        if (g.tile_ptr[L + 1] <= g.tile_ptr[L]) return 0;
        if (use_stream_ && stream_[L].ntiles > 0) return 3;
        if (sizeof(R) == 8 && use_fast_ && fast_[L].recsize > 0) return 2;
        return 1;
    }
    cfr_status read_lcnt(std::vector<unsigned long long>& c) {
        c.assign(4 * (size_t)gp->D, 0);
        CU(cudaStreamSynchronize(stream));
        if (!c.empty()) CU(cudaMemcpy(c.data(), dg.lcnt, c.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        return CFR_OK;
    }
    cfr_status counters(int64_t* out, int32_t max_levels, int32_t* num_levels) override {
        std::vector<unsigned long long> c;
        cfr_status st = read_lcnt(c);
        if (st) return st;
        *num_levels = gp->D;
        for (int L = 0; L < gp->D && L < max_levels; ++L)
            for (int k = 0; k < 4; ++k) out[4 * L + k] = (int64_t)c[4 * L + k];
        return CFR_OK;
    }
    cfr_status level_kernels(int32_t* out, int32_t max_levels, int32_t* num_levels) override {
        const Game& g = *gp;
        *num_levels = g.D;
        for (int L = 0; L < g.D && L < max_levels; ++L) out[L] = level_kernel(L);
        return CFR_OK;
    }

    // Algorithmic DRAM bytes per iteration (DESIGN.md §6 byte model).
    int dom_level = -1;   // set by profile(): the backward level with the largest time
    std::vector<double> prof_live_;   // per level: live infosets, live pairs per iteration (last profile), -1 unknown
    // forward pass of depth l: per decision node its parent slot, edge index and
    // parent actor, its 2P factors written (compact: the actor and its 2 factors);
    // every parent's 2P factors read once (parent rows and sigma are gathers made
    // cache-local by the row-order slot numbering; sigma not counted)
    double level_fwd_bytes(int l) const {
        const Game& g = *gp;
        if (l < 1 || l >= g.D || fwd_fused(l)) return 0.0;   // fused: inside the streaming kernel (not modelled)
        const double w = sizeof(R), ix = sizeof(I);
        const int P = g.P;
        const double n = (double)(g.slot_ptr[l + 1] - g.slot_ptr[l]);
        double b = fwd_compact(l) ? n * (2 * ix + 1 + 1 + 2 * w) : n * (2 * ix + 1 + 2 * P * w);
        b += (double)(g.slot_ptr[l] - g.slot_ptr[l - 1]) * 2 * P * w;
        return b;
    }
    double level_bwd_bytes(int L) const {
        const Game& g = *gp;
        const double w = sizeof(R), ix = sizeof(I);
        const int Pc = g.Pc;
        const double parents = (double)(g.slot_ptr[L + 1] - g.slot_ptr[L]);
        const double children = (double)(g.level_ptr[L + 2] - g.level_ptr[L + 1]);
        if (use_stream_ && L < (int)stream_.size() && stream_[L].ntiles > 0) {
            // k_bwd_stream: children's values read once; per member its U row index,
            // value write, the actor's pi_check and pi_hat; per infoset its member
            // start, owner and S_den read; per pair sigma, R, S_num read.  Writes of
            // the update (R, S_num, sigma per pair, S_den per infoset) for LIVE
            // infosets only (the measured count of the last profile window; all
            // infosets if unknown).  The fused forward variant is not modelled.
            double nh = 0, npairs = 0;
            for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1]; ++t)
                for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1; ++k) {
                    nh += 1;
                    npairs += (double)(g.qbase_int[g.segs[k].h + 1] - g.qbase_int[g.segs[k].h]);
                }
            double live_h = nh, live_p = npairs;
            if ((int)prof_live_.size() == 2 * g.D && prof_live_[2 * L] >= 0) {
                live_h = prof_live_[2 * L];
                live_p = prof_live_[2 * L + 1];
            }
            return children * Pc * w + parents * (ix + Pc * w + 2 * w) + npairs * 3 * w + nh * (4 + 1 + w) +
                   live_p * 3 * w + live_h * w;
        }
        // children values read once; parent: node, cb, ebase, dec (ix each), n, coff
        // (4 each), actor (1); value write; the owner's pi_check and pi_hat
        double b = children * Pc * w + parents * (4 * ix + 8 + 1 + Pc * w + 2 * w);
        // fused update of the level's infosets: R, S_num, sigma read + written per
        // pair; S_den read + written per infoset
        double pairs = 0, infosets = 0;
        for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1]; ++t)
            for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1; ++k)
                if (g.segs[k].fused) {
                    pairs += (double)(g.qbase_int[g.segs[k].h + 1] - g.qbase_int[g.segs[k].h]);
                    infosets += 1;
                }
        b += pairs * 6 * w + infosets * 2 * w;
        return b;
    }
    cfr_status model_bytes(double* out) override {
        const Game& g = *gp;
        const double w = sizeof(R), ix = sizeof(I);
        const int P = g.P;
        double fwd = 0, bwd = 0, upd = 0;
        for (int l = 1; l < g.D; ++l) fwd += level_fwd_bytes(l);
        int big = 0;
        for (int L = g.D - 1; L >= 0; --L) {
            bwd += level_bwd_bytes(L);
            if (g.level_ptr[L + 2] - g.level_ptr[L + 1] > g.level_ptr[big + 2] - g.level_ptr[big + 1]) big = L;
        }
        // deferred infosets: slices read + zeroed, R, S_num, sigma r/w per pair; S_den per infoset
        for (int64_t h : g.deferred_list) {
            const double n = (double)(g.qbase_int[h + 1] - g.qbase_int[h]);
            upd += n * (6 * w + 48) + 2 * w + 48;
        }
        out[0] = fwd + bwd + upd;
        out[1] = fwd;
        out[2] = bwd;
        out[3] = upd;
        out[4] = g.D > 0 ? level_bwd_bytes(dom_level >= 0 ? dom_level : big) : 0.0;
        (void)ix;
        return CFR_OK;
    }
};

static bool use_idx32(const Game& g) {
    const int64_t lim = (int64_t(1) << 31) - 2;
    return g.V < lim && (g.Q + g.C) < lim && g.NS < lim;
}

// The game a rank iterates + its shard metadata (world 1: the whole game).
static cfr_status view_for(cfr_game* G, const cfr_dist* dist, const Game** local, const ShardInfo** info,
                           std::shared_ptr<cfr_game::Shard>* keep) {
    static const ShardInfo single{};
    const int world = dist ? dist->world_size : 1;
    const int rank = dist ? dist->rank : 0;
    if (world < 1 || rank < 0 || rank >= world) {
        cfrb_set_error("bad cfr_dist (rank / world_size)");
        return CFR_ERR_INVALID_ARG;
    }
    if (world == 1) {
        if (G->shard_only) {
            cfrb_set_error("a game loaded from a shard file needs its (rank, world_size)");
            return CFR_ERR_INVALID_ARG;
        }
        *local = &G->g;
        *info = &single;
        return CFR_OK;
    }
    auto key = std::make_pair(rank, world);
    auto it = G->shards.find(key);
    if (it == G->shards.end() && G->shard_only) {
        cfrb_set_error("this game was loaded from a shard file for another (rank, world_size)");
        return CFR_ERR_INVALID_ARG;
    }
    if (it == G->shards.end()) {
        auto sh = std::make_shared<cfr_game::Shard>();
        std::string err;
        if (!build_shard(G->g, rank, world, sh->local, sh->info, err)) {
            cfrb_set_error("shard: " + err);
            return CFR_ERR_INVALID_TREE;
        }
        it = G->shards.emplace(key, sh).first;
    }
    *local = &it->second->local;
    *info = &it->second->info;
    *keep = it->second;
    return CFR_OK;
}

static size_t bytes_for(const Game& g, const ShardInfo* sh, int precision) {
    const bool i32 = use_idx32(g);
    if (precision == 64) return i32 ? Plan<double, int>(g, sh).total : Plan<double, long long>(g, sh).total;
    return i32 ? Plan<float, int>(g, sh).total : Plan<float, long long>(g, sh).total;
}

}  // namespace cfrb

using namespace cfrb;

struct cfr_solver {
    std::unique_ptr<SolverBase> impl;
    std::shared_ptr<cfr_game::Shard> keep;   // shard view the solver iterates
};

extern "C" {

cfr_status cfr_solver_workspace_bytes(const cfr_game* g, const cfr_solver_config* cfg, const cfr_dist* dist,
                                      size_t* bytes) {
    if (!g || !cfg || !bytes) { cfrb_set_error("NULL argument"); return CFR_ERR_INVALID_ARG; }
    if (cfg->precision != 64 && cfg->precision != 32) { cfrb_set_error("precision must be 64 or 32"); return CFR_ERR_INVALID_ARG; }
    const Game* local = nullptr;
    const ShardInfo* info = nullptr;
    std::shared_ptr<cfr_game::Shard> keep;
    cfr_status s = view_for(const_cast<cfr_game*>(g), dist, &local, &info, &keep);
    if (s) return s;
    *bytes = bytes_for(*local, info, cfg->precision);
    return CFR_OK;
}

cfr_status cfr_solver_create(const cfr_game* g, const cfr_solver_config* cfg, void* workspace, size_t workspace_bytes,
                             void* stream, const cfr_dist* dist, cfr_solver** out) {
    if (!g || !cfg || !out || !workspace) { cfrb_set_error("NULL argument"); return CFR_ERR_INVALID_ARG; }
    *out = nullptr;
    if (cfg->variant < CFR_VANILLA || cfg->variant > CFR_PLUS_ALT) { cfrb_set_error("bad variant"); return CFR_ERR_INVALID_ARG; }
    if (cfg->precision != 64 && cfg->precision != 32) { cfrb_set_error("precision must be 64 or 32"); return CFR_ERR_INVALID_ARG; }
    const Game* local = nullptr;
    const ShardInfo* info = nullptr;
    std::shared_ptr<cfr_game::Shard> keep;
    cfr_status s = view_for(const_cast<cfr_game*>(g), dist, &local, &info, &keep);
    if (s) return s;
    const size_t need = bytes_for(*local, info, cfg->precision);
    if (workspace_bytes < need) {
        cfrb_set_error("workspace too small: need " + std::to_string(need) + " bytes");
        return CFR_ERR_OOM;
    }
    if (((uintptr_t)workspace & 255) != 0) { cfrb_set_error("workspace must be 256-byte aligned"); return CFR_ERR_INVALID_ARG; }
    const bool i32 = use_idx32(*local);
    std::unique_ptr<SolverBase> impl;
    cudaStream_t st = (cudaStream_t)stream;
    const void* nid = (dist && dist->world_size > 1) ? dist->nccl_unique_id : nullptr;
    if (cfg->precision == 64) {
        if (i32) { auto p = new Solver<double, int>(local, &g->g, info, *cfg, workspace, st); impl.reset(p); s = p->init(nid); }
        else { auto p = new Solver<double, long long>(local, &g->g, info, *cfg, workspace, st); impl.reset(p); s = p->init(nid); }
    } else {
        if (i32) { auto p = new Solver<float, int>(local, &g->g, info, *cfg, workspace, st); impl.reset(p); s = p->init(nid); }
        else { auto p = new Solver<float, long long>(local, &g->g, info, *cfg, workspace, st); impl.reset(p); s = p->init(nid); }
    }
    if (s != CFR_OK) return s;
    *out = new cfr_solver{std::move(impl), keep};
    return CFR_OK;
}

void cfr_solver_destroy(cfr_solver* s) { delete s; }

#define CHK_S(s) \
    if (!(s)) { cfrb_set_error("NULL solver"); return CFR_ERR_INVALID_ARG; }

cfr_status cfr_solver_enqueue(cfr_solver* s, int64_t iterations) {
    CHK_S(s);
    if (iterations < 0) { cfrb_set_error("iterations < 0"); return CFR_ERR_INVALID_ARG; }
    return s->impl->enqueue(iterations);
}
cfr_status cfr_solver_sync(cfr_solver* s) {
    CHK_S(s);
    return s->impl->sync();
}
cfr_status cfr_solver_run(cfr_solver* s, int64_t iterations) {
    CHK_S(s);
    cfr_status st = cfr_solver_enqueue(s, iterations);
    if (st) return st;
    return s->impl->sync();
}
cfr_status cfr_solver_iteration(cfr_solver* s, int64_t* T) {
    CHK_S(s);
    if (!T) { cfrb_set_error("NULL T"); return CFR_ERR_INVALID_ARG; }
    return s->impl->iteration(T);
}
cfr_status cfr_solver_average_strategy(cfr_solver* s, double* out) {
    CHK_S(s);
    if (!out) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->strategy(0, out);
}
cfr_status cfr_solver_current_strategy(cfr_solver* s, double* out) {
    CHK_S(s);
    if (!out) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->strategy(1, out);
}
cfr_status cfr_solver_get_state(cfr_solver* s, double* regret, double* s_num, double* s_den) {
    CHK_S(s);
    return s->impl->get_state(regret, s_num, s_den);
}
cfr_status cfr_solver_expected_values(cfr_solver* s, int32_t which, double* out) {
    CHK_S(s);
    if (!out || (which != CFR_EV_AVERAGE && which != CFR_EV_CURRENT)) { cfrb_set_error("bad argument"); return CFR_ERR_INVALID_ARG; }
    return s->impl->expected_values(which, out);
}
cfr_status cfr_solver_exploitability(cfr_solver* s, double* nash_conv, double* exploitability, double* br) {
    CHK_S(s);
    if (!nash_conv || !exploitability) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->exploitability(nash_conv, exploitability, br);
}
cfr_status cfr_solver_launches_per_iteration(cfr_solver* s, int64_t* launches) {
    CHK_S(s);
    if (!launches) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->launches(launches);
}
cfr_status cfr_solver_profile(cfr_solver* s, int64_t iterations, double* out_ms) {
    CHK_S(s);
    if (!out_ms) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->profile(iterations, out_ms);
}
cfr_status cfr_solver_model_bytes(cfr_solver* s, double* out) {
    CHK_S(s);
    if (!out) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->model_bytes(out);
}
cfr_status cfr_solver_level_kernels(cfr_solver* s, int32_t* out, int32_t max_levels, int32_t* num_levels) {
    CHK_S(s);
    if (!num_levels || (max_levels > 0 && !out)) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->level_kernels(out, max_levels, num_levels);
}
cfr_status cfr_solver_level_profile(cfr_solver* s, double* out, int32_t max_levels, int32_t* num_levels) {
    CHK_S(s);
    if (!num_levels || (max_levels > 0 && !out)) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->level_profile(out, max_levels, num_levels);
}
cfr_status cfr_solver_counters(cfr_solver* s, int64_t* out, int32_t max_levels, int32_t* num_levels) {
    CHK_S(s);
    if (!num_levels || (max_levels > 0 && !out)) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->counters(out, max_levels, num_levels);
}
cfr_status cfr_nccl_unique_id(void* out) {
    if (!out) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        cfrb_set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        return CFR_ERR_NCCL;
    }
    std::memcpy(out, &id, sizeof(id));
    return CFR_OK;
}
cfr_status cfr_game_shard_info(const cfr_game* g, int32_t rank, int32_t world, int64_t* out) {
    if (!g || !out) { cfrb_set_error("NULL argument"); return CFR_ERR_INVALID_ARG; }
    cfr_dist d{rank, world, nullptr};
    const Game* local = nullptr;
    const ShardInfo* info = nullptr;
    std::shared_ptr<cfr_game::Shard> keep;
    cfr_status s = view_for(const_cast<cfr_game*>(g), &d, &local, &info, &keep);
    if (s) return s;
    out[0] = info->cut;
    out[1] = (int64_t)info->cut_row.size();
    out[2] = info->owned_nodes;
    out[3] = local->V;
    out[4] = local->NS;
    out[5] = (int64_t)local->deferred_list.size();
    out[6] = local->dqbase.empty() ? 0 : local->dqbase.back();
    out[7] = world;
    int64_t owned_cut = 0, reported = 0;
    for (auto o : info->cut_owned) owned_cut += o;
    for (auto r : info->report) reported += r;
    out[8] = owned_cut;
    out[9] = world > 1 ? reported : g->g.H;
    return CFR_OK;
}
cfr_status cfr_solver_phase(cfr_solver* s, int32_t phase, double* out) {
    CHK_S(s);
    return s->impl->phase(phase, out);
}
cfr_status cfr_solver_exchange_size(cfr_solver* s, int32_t which, size_t* bytes) {
    CHK_S(s);
    if (!bytes) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->exchange_size(which, bytes);
}
cfr_status cfr_solver_exchange(cfr_solver* s, int32_t which, int32_t put, void* host, size_t bytes) {
    CHK_S(s);
    if (!host && bytes) { cfrb_set_error("NULL buffer"); return CFR_ERR_INVALID_ARG; }
    return s->impl->exchange(which, put, host, bytes);
}
cfr_status cfr_solver_shard_info(cfr_solver* s, int64_t* out) {
    CHK_S(s);
    if (!out) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->shard_info(out);
}

}  // extern "C"
