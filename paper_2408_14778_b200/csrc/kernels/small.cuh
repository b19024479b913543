// Small-game kernel: k_tiny (one CTA, shared memory, T iterations per launch).
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

// ------------------------------------------------------------- tiny games
// Games whose whole mutable state fits in one CTA's shared memory (Kuhn; Leduc
// with its node values in global memory) are bound by per-level latency, not
// bytes.  k_tiny runs T iterations in ONE CTA: U, reach, sigma, R, S_num, S_den
// (and the per-level r~ / pi_bar) live in shared memory; levels are separated by
// __syncthreads.  The read-only game tables are one int32 block (TinyMeta) that
// is copied into shared memory too when it fits (META; Kuhn), so a level's
// dependent chain is shared-memory loads only, and read through L1 otherwise.
// Same operations, same order as the per-level kernels (requires depth-homogeneous
// infosets: an infoset's members are the contiguous slots mem0[h] .. mem1[h] of
// one level).
struct TinyPlan {
    long long U, reach, sig, reg, snum, sden, rt, pib;   // element offsets in shared memory (R units); U < 0: U in global
    long long nU, nreach, nsig, Q, H;
    int bytes;          // dynamic shared memory
    int meta_off;       // META: byte offset of the TinyMeta copy in shared memory
    int meta_ints;      // ints of the TinyMeta block
    // int offsets inside the TinyMeta block
    int m_lv;           // [4 D]: per depth s0, s1 (slots), h0, h1 (internal infosets)
    int m_slot;         // [7 NS]: parent slot, sigma_ext edge, parent actor, first child U row,
                        //         sigma_ext base, children, node U row
    int m_qb;           // [H + 1] qbase (internal)
    int m_own;          // [H] owner
    int m_mem;          // [2 H] member slot range
    int m_ph;           // [Q] infoset of each (h, a) pair
};

template <class R, class I, int PC, bool META>
__global__ void __launch_bounds__(1024) k_tiny(DG<R, I> g, const int* __restrict__ gmeta, int D, long long T,
                                                TinyPlan tp) {
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
    int* const smeta = reinterpret_cast<int*>(smem_raw + tp.meta_off);
    const int* const M = META ? smeta : gmeta;
    const int* const lv = M + tp.m_lv;
    const int* const sl = M + tp.m_slot;
    const int* const qb_ = M + tp.m_qb;
    const int* const own_ = M + tp.m_own;
    const int* const mem_ = M + tp.m_mem;
    const int* const ph_ = M + tp.m_ph;
    pdl_trigger();
    pdl_wait();
    if (META)
        for (int k = tid; k < tp.meta_ints; k += nth) smeta[k] = gmeta[k];
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
                for (int s = lv[4 * l] + tid; s < lv[4 * l + 1]; s += nth) {
                    const int* e = sl + 7 * s;
                    const int p = e[0];
                    const R x = sig[e[1]];
                    const int act = e[2];
                    for (int j = 0; j < P; ++j) {
                        const R pc = reach[p * 2 * P + j], ph = reach[p * 2 * P + P + j];
                        reach[s * 2 * P + j] = (act != j + 1) ? pc * x : pc;
                        reach[s * 2 * P + P + j] = (act == j + 1) ? ph * x : ph;
                    }
                }
                __syncthreads();
            }
            for (int L = D - 1; L >= 0; --L) {
                for (int s = lv[4 * L] + tid; s < lv[4 * L + 1]; s += nth) {   // values (Eq 1)
                    const int* e = sl + 7 * s;
                    const int cb = e[3], eb = e[4], nch = e[5];
                    R v[PC];
#pragma unroll
                    for (int j = 0; j < PC; ++j) v[j] = (R)0;
                    for (int a = 0; a < nch; ++a) {
                        const R x = sig[eb + a];
#pragma unroll
                        for (int j = 0; j < PC; ++j) v[j] = v[j] + x * U[(long long)(cb + a) * PC + j];
                    }
                    const long long node = e[6];
#pragma unroll
                    for (int j = 0; j < PC; ++j) U[node * PC + j] = v[j];
                }
                __syncthreads();
                const int h0 = lv[4 * L + 2], h1 = lv[4 * L + 3];
                if (h1 > h0) {
                    const int q0 = qb_[h0], q1 = qb_[h1];
                    const int items = (q1 - q0) + (h1 - h0);
                    for (int x = tid; x < items; x += nth) {   // exact sums
                        double c0 = 0, c1 = 0, c2 = 0;
                        if (x < q1 - q0) {
                            const int q = q0 + x;
                            const int h = ph_[q];
                            const int i = own_[h];
                            if (upl != 0 && i != upl) continue;
                            const int a = q - qb_[h];
                            const int col = (PC == 1) ? 0 : i - 1;
                            for (int d = mem_[2 * h]; d < mem_[2 * h + 1]; ++d) {
                                const R pc = reach[d * 2 * P + (i - 1)];
                                if (pc == (R)0) continue;   // exact zero terms
                                const int* e = sl + 7 * d;
                                const R u = U[(long long)(e[3] + a) * PC + col];
                                const R v = U[(long long)e[6] * PC + col];
                                xadd(c0, c1, c2, (double)(pc * (u - v)), g.sc0);
                            }
                            if (PC == 1 && i == 2) { c0 = -c0; c1 = -c1; c2 = -c2; }   // u2 = -u1 storage
                            rtb[q] = (R)xdec(c0, c1, c2, g.rc);
                        } else {
                            const int h = h0 + (x - (q1 - q0));
                            const int i = own_[h];
                            if (upl != 0 && i != upl) continue;
                            for (int d = mem_[2 * h]; d < mem_[2 * h + 1]; ++d)
                                xadd(c0, c1, c2, (double)reach[d * 2 * P + P + (i - 1)], g.scp0);
                            pibb[h] = (R)xdec(c0, c1, c2, g.rcp);
                        }
                    }
                    __syncthreads();
                    for (int h = h0 + tid; h < h1; h += nth) {   // update (Eq 8/15 / CFR+ / Q18, Eq 10, Eq 9)
                        const int i = own_[h];
                        if (upl != 0 && i != upl) continue;
                        const int qb = qb_[h];
                        const int n = qb_[h + 1] - qb;
                        const R wp = w * pibb[h];
                        R z = (R)0;
                        for (int a = 0; a < n; ++a) {
                            const int q = qb + a;
                            const R r = upd_regret(up, reg[q], rtb[q]);
                            reg[q] = r;
                            snum[q] = upd_sum(up, snum[q], wp * sig[q]);
                            z = z + ((r > (R)0) ? r : (R)0);
                        }
                        sden[h] = upd_sum(up, sden[h], wp);
                        for (int a = 0; a < n; ++a) {
                            const int q = qb + a;
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
