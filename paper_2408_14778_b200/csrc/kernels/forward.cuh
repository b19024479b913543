// Forward pass (Eq 2 / Eq 4): k_fwd.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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

}  // namespace cfrb
