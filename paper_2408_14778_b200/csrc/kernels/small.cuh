// Small-game kernel: k_tiny (one CTA, shared memory, T iterations per launch).
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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
    long long U, reach, sig, reg, snum, sden, rt, pib;   // element offsets in shared memory (R units); U < 0: U in global
    long long nU, nreach, nsig, Q, H;
    int bytes;
};

template <class R, class I, int PC>
__global__ void __launch_bounds__(1024) k_tiny(DG<R, I> g, const TinyLevel* __restrict__ lv, const I* __restrict__ mem_of,
                                                int D, long long T, TinyPlan tp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* const sm = reinterpret_cast<R*>(smem_raw);
    R* const U = (tp.U >= 0) ? sm + tp.U : g.U;   // global: this CTA's stores are seen by its later loads
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
    if (tp.U >= 0)
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
    long long bad = LLONG_MAX;   // first iteration of this launch with a non-finite value
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
                            if (!finite_(rtb[q]) || !finite_(nsig) || !finite_(z)) bad = min(bad, t_iter);
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
    // write the state back (readbacks and later launches read it from global)
    if (tp.U >= 0)
        for (long long k = tid; k < tp.nU; k += nth) g.U[k] = U[k];
    for (long long k = tid; k < tp.nreach; k += nth) g.reach[k] = reach[k];
    for (long long k = tid; k < tp.nsig; k += nth) g.sig[k] = sig[k];
    for (long long k = tid; k < tp.Q; k += nth) {
        g.regret[k] = reg[k];
        g.snum[k] = snum[k];
    }
    for (long long k = tid; k < tp.H; k += nth) g.sden[k] = sden[k];
    if (bad != LLONG_MAX) atomicMin(&g.ctrl[1], bad);
    if (tid == 0) g.ctrl[0] = t_iter;
}

}  // namespace cfrb
