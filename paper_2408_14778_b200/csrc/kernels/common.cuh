// Shared device definitions of the CFR kernels: tile / segment records, the
// kernel argument block DG, exact slice sums, cp.async / PDL
// helpers, L2 cache-policy loads/stores and the per-iteration update rule.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

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
    int* br_best;                 // [ndef] best-response action of each deferred infoset (MODE_BR passes)
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

}  // namespace cfrb
