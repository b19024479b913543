// Subtree kernel: forward + backward of the subtrees below a
// cut level in ONE launch, their state in shared memory; k_sub_update.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

// ------------------------------------------------------------ subtree fusion
// P:401 partitions the root-to-leaf paths into subgraphs processed separately;
// P:403 chunks the tree into a trunk and subtrees.  Below a cut level c every
// non-terminal node of depth c roots a subtree; one CTA runs the subtree's whole
// forward pass (Eq 2 / Eq 4, reading Q1) and backward pass (Eq 1) with the reach
// factors, node values and terminal utilities of the subtree in shared memory and
// levels separated by __syncthreads -- instead of 2(D - c) level launches, each a
// dependent chain through global memory.  Infosets span subtrees (imperfect
// information), so their regret terms (Eq 7, cancelled form) and pi_hat terms
// (Eq 5) are added as exact 40-bit slices to int64 accumulators
// with global atomics: integer sums, so the result does not depend on the order
// in which subtrees add them.  k_sub_update then decodes the sums and applies the
// update of every infoset below the cut (Eq 8/15 or CFR+, Eq 10, Eq 9: the
// operations and order of k_deferred).  The trunk (depths < c) keeps the level
// kernels; the roots' values are written to their U rows for it.
//
// Tables (int32, built once on the host from the device slot tables, so both
// paths read the same numbers), all staged into shared memory at the start:
//   per subtree b (kSubMeta ints): node0, nodes, term0, terms, lvl0, levels,
//     plv0, root slot, child0, edges, pair0, pairs
//   per local node (two int4): {local parent (-1 root), child-table position of
//     its incoming edge, parent actor | actor << 8 (0 chance), sigma_ext index of
//     its incoming edge} and {sigma_ext base of its children's edges, children,
//     first child-table position (local), internal infoset (-1 chance)}
//   child table (local positions, one per edge): >= 0 local node, < 0 -(1 + k) =
//     the subtree's k-th terminal
//   pair table (int4 per (player node, action)): local node << 8 | action, child
//     reference, sigma / accumulator pair index q, actor
//   per level: local node starts [levels + 1], then local pair starts [levels + 1]
// Terminal utilities in subtree order: tu[(term0 + k) * Pc + j].
// STAGED (the subtrees' tables fit shared memory next to their state): the tables
// are copied in at the start and the edge probabilities of the subtree (sigma of
// its player nodes' infosets, the chance probabilities) gathered once per
// iteration into ev[] (one dependent round trip); every level step after that is
// shared-memory work and a barrier.  Otherwise (larger subtrees at a shallower
// cut) the tables and sigma are read from global memory (L2) in each level step:
// 16-byte records, sigma and child references batched 8 actions at a time.
// -DCFR_SUB_CHECKS builds (tools/sub_checks.sh) trap on any out-of-range table
// entry or shared-memory index: the bounds checks that stand in for
// compute-sanitizer, which is closed on this pool.  Product builds compile them out.
#ifdef CFR_SUB_CHECKS
#define SUB_CHECK(c) do { if (!(c)) __trap(); } while (0)
#else
#define SUB_CHECK(c) do { } while (0)
#endif
constexpr int kSubMeta = 12;
constexpr int kSubRec = 8;
constexpr int kSubThreads = 1024;

struct SubPlan {
    int nsub;          // subtrees (= CTAs)
    int cut;           // cut level c
    long long hc, qc;  // first internal infoset / pair below the cut (accumulator bases)
    long long nh, nq;  // infosets / pairs below the cut
    int bytes;         // dynamic shared memory (the largest subtree)
    int threads;       // CTA size
    int staged;        // 1: tables and edge probabilities staged in shared memory
    int trunk;         // 1: the trunk (depths < c) holds chance nodes only -- k_sub computes each
                       //    root's reach along its path, k_sub_update's last CTA the trunk values
    int m_path;        // trunk: per subtree the sigma_ext edges root path, top-down (cut ints each)
    int m_trunk;       // trunk: per trunk slot {U row of the node, first child U row, sigma_ext base, children}
    int ntrunk;        // trunk slots (levels 0..c-1, level-major)
    int m_sub, m_rec, m_child, m_pair, m_lvl;   // int offsets inside the table block
};

// shared-memory plan of one subtree (host and device agree on it)
struct SubSmem {
    long long reach, val, tv, ev, rec, prs, chl, lvl, total;   // byte offsets
};
__host__ __device__ inline long long sub_al16(long long x) { return (x + 15) & ~15LL; }
__host__ __device__ inline SubSmem sub_smem(long long nn, long long nt, long long ne, long long np, int nlev, int P,
                                            int Pc, int w) {
    SubSmem m;
    long long o = 0;
    m.reach = o; o += sub_al16(nn * 2 * P * w);
    m.val = o; o += sub_al16(nn * Pc * w);
    m.tv = o; o += sub_al16(nt * Pc * w);
    m.ev = o; o += sub_al16(ne * w);
    m.rec = o; o += nlev >= 0 ? nn * 4 * kSubRec : 0;
    m.prs = o; o += np * 16;
    m.chl = o; o += sub_al16(ne * 4);
    m.lvl = o; o += nlev >= 0 ? sub_al16(2LL * (nlev + 1) * 4) : 0;
    m.total = o;
    return m;
}

template <class R, class I, int PC, bool STAGED>
__global__ void __launch_bounds__(kSubThreads) k_sub(DG<R, I> g, const int* __restrict__ T, const R* __restrict__ tu,
                                                     unsigned long long* __restrict__ acc, SubPlan sp) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.x, tid = threadIdx.x, nth = blockDim.x;
    const int P = g.P;
    const int* const mb = T + sp.m_sub + kSubMeta * b;
    const int node0 = mb[0], nn = mb[1], term0 = mb[2], nt = mb[3], lvl0 = mb[4], nlev = mb[5];
    const int root_slot = mb[7], child0 = mb[8], ne = mb[9], pair0 = mb[10], np = mb[11];
    const SubSmem L = sub_smem(nn, nt, STAGED ? ne : 0, STAGED ? np : 0, STAGED ? nlev : -1, P, PC, (int)sizeof(R));
#ifdef CFR_SUB_CHECKS
    {
        unsigned dyn = 0;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        SUB_CHECK(L.total <= (long long)dyn && nn >= 1 && nt >= 0 && ne == nn - 1 + nt && np >= 0 && nlev >= 1);
    }
#endif
    R* const reach = reinterpret_cast<R*>(smem_raw + L.reach);    // [nn][2P]
    R* const val = reinterpret_cast<R*>(smem_raw + L.val);        // [nn][PC]
    R* const tv = reinterpret_cast<R*>(smem_raw + L.tv);          // [nt][PC] terminal utilities
    R* const ev = reinterpret_cast<R*>(smem_raw + L.ev);          // [ne] edge probabilities (STAGED)
    const int4* const grec = reinterpret_cast<const int4*>(T + sp.m_rec + (long long)kSubRec * node0);
    const int4* const gprs = reinterpret_cast<const int4*>(T + sp.m_pair) + pair0;
    const int* const gchl = T + sp.m_child + child0;
    const int* const glv = T + sp.m_lvl + lvl0;
    int4* const srec = reinterpret_cast<int4*>(smem_raw + L.rec);
    int4* const sprs = reinterpret_cast<int4*>(smem_raw + L.prs);
    int* const schl = reinterpret_cast<int*>(smem_raw + L.chl);
    int* const slv = reinterpret_cast<int*>(smem_raw + L.lvl);
    const int4* const rec = STAGED ? srec : grec;                 // [nn][2]
    const int4* const prs = STAGED ? sprs : gprs;                 // [np]
    const int* const chl = STAGED ? schl : gchl;                  // [ne]
    const int* const lv = STAGED ? slv : glv;                     // [nlev + 1] nodes, then [nlev + 1] pairs
    const int* const plv = lv + nlev + 1;
    unsigned long long* const acc_r = acc;                        // [nq][3]
    unsigned long long* const acc_p = acc + 3 * sp.nq;            // [nh][3]
    pdl_trigger();
    // the constant tables and terminal utilities: staged before the dependency wait
    if (STAGED) {
        for (int k = tid; k < 2 * nn; k += nth) srec[k] = grec[k];
        for (int k = tid; k < np; k += nth) sprs[k] = gprs[k];
        for (int k = tid; k < ne; k += nth) schl[k] = gchl[k];
        for (int k = tid; k < 2 * (nlev + 1); k += nth) slv[k] = glv[k];
    }
    for (long long k = tid; k < (long long)nt * PC; k += nth) tv[k] = tu[(long long)term0 * PC + k];
    pdl_wait();
    const long long t_iter = g.ctrl[0] + 1;
    bool bad = false;
    if (STAGED) {
        __syncthreads();
        // edge probabilities of this iteration (sigma is constant during the pass)
        for (int j = tid; j < nn; j += nth) {
            const int4 bb = rec[2 * j + 1];
            SUB_CHECK(bb.z >= 0 && bb.y >= 0 && bb.z + bb.y <= ne && bb.x >= 0);
            for (int a = 0; a < bb.y; ++a) ev[bb.z + a] = g.sig[bb.x + a];
        }
    }
    if (sp.trunk) {
        // chance-only trunk: the root's reach is the path product of its chance edges
        // (k_fwd's operations with a chance parent: every pi_check times the edge's
        // probability, top-down from the root row of ones; pi_hat unchanged)
        if (tid == 0) {
            R pc[8];
            for (int i = 0; i < P; ++i) pc[i] = (R)1;
            const int* path = T + sp.m_path + (long long)sp.cut * b;
            for (int k = 0; k < sp.cut; ++k) {
                const R x = g.sig[path[k]];
                for (int i = 0; i < P; ++i) pc[i] = pc[i] * x;
            }
            for (int i = 0; i < P; ++i) {
                reach[i] = pc[i];
                reach[P + i] = (R)1;
            }
        }
    } else if (tid < 2 * P) {
        reach[tid] = g.reach[(long long)root_slot * 2 * P + tid];   // level-c forward kernel's row
    }
    __syncthreads();
    // ---- forward (Eq 2 / Eq 4 with reading Q1; k_fwd's operations)
    for (int l = 1; l < nlev; ++l) {
        for (int j = lv[l] + tid; j < lv[l + 1]; j += nth) {
            const int4 ea = rec[2 * j];
            const int p = ea.x;
            SUB_CHECK(j < nn && p >= 0 && p < j && ea.y >= 0 && ea.y < ne && ea.w >= 0);
            const R x = STAGED ? ev[ea.y] : g.sig[ea.w];
            const int act = ea.z & 255;
            for (int i = 0; i < P; ++i) {
                const R pc = reach[p * 2 * P + i], ph = reach[p * 2 * P + P + i];
                reach[j * 2 * P + i] = (act != i + 1) ? pc * x : pc;
                reach[j * 2 * P + P + i] = (act == i + 1) ? ph * x : ph;
            }
        }
        __syncthreads();
    }
    // ---- backward, deepest level first
    for (int l = nlev - 1; l >= 0; --l) {
        // values (Eq 1: ascending actions from +0)
        for (int j = lv[l] + tid; j < lv[l + 1]; j += nth) {
            const int4 ea = rec[2 * j];
            const int4 bb = rec[2 * j + 1];
            const int eb = bb.x, nch = bb.y, cp = bb.z;
            SUB_CHECK(j < nn && cp >= 0 && nch >= 0 && cp + nch <= ne);
            R v[PC];
#pragma unroll
            for (int c = 0; c < PC; ++c) v[c] = (R)0;
            if (STAGED) {
                for (int a = 0; a < nch; ++a) {
                    const R x = ev[cp + a];
                    const int ch = chl[cp + a];
                    SUB_CHECK(ch < nn && ch >= -nt && (ch < 0 || ch > j));
                    const R* u = (ch >= 0) ? val + (long long)ch * PC : tv + (long long)(-1 - ch) * PC;
#pragma unroll
                    for (int c = 0; c < PC; ++c) v[c] = v[c] + x * u[c];
                }
            } else {
                for (int a0 = 0; a0 < nch; a0 += 8) {
                    // the batch's sigma and child references in flight together
                    R x[8];
                    int ch[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        x[k] = (a0 + k < nch) ? g.sig[eb + a0 + k] : (R)0;
                        ch[k] = (a0 + k < nch) ? chl[cp + a0 + k] : 0;
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (a0 + k >= nch) break;
                        SUB_CHECK(ch[k] < nn && ch[k] >= -nt && (ch[k] < 0 || ch[k] > j));
                        const R* u = (ch[k] >= 0) ? val + (long long)ch[k] * PC : tv + (long long)(-1 - ch[k]) * PC;
#pragma unroll
                        for (int c = 0; c < PC; ++c) v[c] = v[c] + x[k] * u[c];
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < PC; ++c) val[(long long)j * PC + c] = v[c];
            // exact slices of pi_hat (Eq 5 / Eq 10 weights) of a player node (the
            // reach factors are final since the forward pass)
            const int i = ea.z >> 8;
            if (i != 0 && (g.upd_player == 0 || i == g.upd_player)) {
                const R ph = reach[j * 2 * P + P + (i - 1)];
                if (ph != (R)0) {
                    SUB_CHECK(bb.w >= sp.hc && bb.w < sp.hc + sp.nh && i <= P);
                    double c0 = 0, c1 = 0, c2 = 0;
                    xadd(c0, c1, c2, (double)ph, g.scp0);
                    unsigned long long* ac = acc_p + ((long long)bb.w - sp.hc) * 3;
                    if (c0 != 0.0) atomicAdd(ac + 0, (unsigned long long)(long long)c0);
                    if (c1 != 0.0) atomicAdd(ac + 1, (unsigned long long)(long long)c1);
                    if (c2 != 0.0) atomicAdd(ac + 2, (unsigned long long)(long long)c2);
                }
            }
        }
        __syncthreads();
        // exact slices of the regret terms pi_check * (u(child) - u(node)) of this
        // level's (node, action) pairs; zero terms are exact zeros and skipped
        for (int k = plv[l] + tid; k < plv[l + 1]; k += nth) {
            const int4 pr = prs[k];
            const int j = pr.x >> 8, ch = pr.y, i = pr.w;
            SUB_CHECK(k < np && j >= 0 && j < nn && ch < nn && ch >= -nt && i >= 1 && i <= P && pr.z >= sp.qc &&
                      pr.z < sp.qc + sp.nq);
            if (g.upd_player != 0 && i != g.upd_player) continue;
            const R pc = reach[j * 2 * P + (i - 1)];
            if (pc == (R)0) continue;
            const int col = (PC == 1) ? 0 : i - 1;
            const R u = (ch >= 0) ? val[(long long)ch * PC + col] : tv[(long long)(-1 - ch) * PC + col];
            const R t = pc * (u - val[(long long)j * PC + col]);
            if (!finite_(t)) bad = true;
            double c0 = 0, c1 = 0, c2 = 0;
            xadd(c0, c1, c2, (double)t, g.sc0);
            if (PC == 1 && i == 2) { c0 = -c0; c1 = -c1; c2 = -c2; }   // u2 = -u1 storage
            unsigned long long* ac = acc_r + ((long long)pr.z - sp.qc) * 3;
            if (c0 != 0.0) atomicAdd(ac + 0, (unsigned long long)(long long)c0);
            if (c1 != 0.0) atomicAdd(ac + 1, (unsigned long long)(long long)c1);
            if (c2 != 0.0) atomicAdd(ac + 2, (unsigned long long)(long long)c2);
        }
        // (no barrier: the next level reads only values written before the last one)
    }
    // the root's value into its U row (read by the trunk's backward pass)
    if (tid < PC) {
        const long long row = (long long)g.s_node[root_slot];
        g.U[row * PC + tid] = val[tid];
    }
    if (bad) atomicMin(&g.ctrl[1], t_iter);
}

// Update of every infoset below the cut: decode the exact sums, then Eq 8/15 or
// CFR+ (or Q18), Eq 10, Eq 9 (k_deferred's operations and order); zero the sums.
// A thread per infoset; the infoset's loads (sums, R, S_num, sigma) are all issued
// before its first store (restrict-qualified copies of the state pointers), so
// the chain is one round trip of loads, not one per action.
constexpr int kSubUpdRegs = 8;   // actions kept in registers (wider infosets: generic loop)
template <class R, class I, int PC>
__global__ void __launch_bounds__(256) k_sub_update(DG<R, I> g, unsigned long long* __restrict__ acc, SubPlan sp,
                                                    const int* __restrict__ T, int last) {
    pdl_trigger();
    pdl_wait();
    const long long t_iter = g.ctrl[0] + 1;
    const Upd<R> up = make_upd<R>(g.variant, t_iter);
    const R w = up.w;
    bool bad = false;
    unsigned long long* __restrict__ const acc_r = acc;
    unsigned long long* __restrict__ const acc_p = acc + 3 * sp.nq;
    R* __restrict__ const reg = g.regret;
    R* __restrict__ const snum = g.snum;
    R* __restrict__ const sig = g.sig;
    R* __restrict__ const sden = g.sden;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < sp.nh; x += stride) {
        const long long h = sp.hc + x;
        const long long qb = (long long)g.qbase[h];
        const int n = (int)((long long)g.qbase[h + 1] - qb);
        const long long cq0 = qb - sp.qc;
        if (g.upd_player != 0 && g.owner[h] != g.upd_player) {
            // alternating updates: another player's infoset (its sums are zero)
            continue;
        }
        const long long p0 = (long long)acc_p[x * 3 + 0], p1 = (long long)acc_p[x * 3 + 1], p2 = (long long)acc_p[x * 3 + 2];
        const R sd = sden[h];
        if (n <= kSubUpdRegs) {
            long long c[kSubUpdRegs][3];
            R r0[kSubUpdRegs], s0[kSubUpdRegs], x0[kSubUpdRegs];
#pragma unroll
            for (int a = 0; a < kSubUpdRegs; ++a)
                if (a < n) {
                    const unsigned long long* ac = acc_r + (cq0 + a) * 3;
                    c[a][0] = (long long)ac[0];
                    c[a][1] = (long long)ac[1];
                    c[a][2] = (long long)ac[2];
                    r0[a] = reg[qb + a];
                    s0[a] = snum[qb + a];
                    x0[a] = sig[qb + a];
                }
            acc_p[x * 3 + 0] = 0;
            acc_p[x * 3 + 1] = 0;
            acc_p[x * 3 + 2] = 0;
            const R pib = (R)xdec_ll(p0, p1, p2, g.rcp);
            const R wp = w * pib;
            R z = (R)0;
#pragma unroll
            for (int a = 0; a < kSubUpdRegs; ++a)
                if (a < n) {
                    unsigned long long* ac = acc_r + (cq0 + a) * 3;
                    ac[0] = 0;
                    ac[1] = 0;
                    ac[2] = 0;
                    const R rt = (R)xdec_ll(c[a][0], c[a][1], c[a][2], g.rc);
                    const R r = upd_regret(up, r0[a], rt);
                    r0[a] = r;
                    reg[qb + a] = r;
                    snum[qb + a] = upd_sum(up, s0[a], wp * x0[a]);
                    z = z + ((r > (R)0) ? r : (R)0);
                    if (!finite_(rt)) bad = true;
                }
            sden[h] = upd_sum(up, sd, wp);
#pragma unroll
            for (int a = 0; a < kSubUpdRegs; ++a)
                if (a < n) {
                    const R r = r0[a];
                    const R pos = (r > (R)0) ? r : (R)0;
                    const R nsig = (z > (R)0) ? pos / z : (R)1 / (R)n;
                    sig[qb + a] = nsig;
                    if (!finite_(r) || !finite_(nsig) || !finite_(z)) bad = true;
                }
            continue;
        }
        acc_p[x * 3 + 0] = 0;
        acc_p[x * 3 + 1] = 0;
        acc_p[x * 3 + 2] = 0;
        const R pib = (R)xdec_ll(p0, p1, p2, g.rcp);
        const R wp = w * pib;
        R z = (R)0;
        for (int a = 0; a < n; ++a) {
            const long long q = qb + a;
            unsigned long long* ac = acc_r + (cq0 + a) * 3;
            const long long c0 = (long long)ac[0], c1 = (long long)ac[1], c2 = (long long)ac[2];
            ac[0] = 0;
            ac[1] = 0;
            ac[2] = 0;
            const R rt = (R)xdec_ll(c0, c1, c2, g.rc);
            reg[q] = upd_regret(up, reg[q], rt);
            snum[q] = upd_sum(up, snum[q], wp * sig[q]);
            if (!finite_(rt)) bad = true;
        }
        sden[h] = upd_sum(up, sd, wp);
        for (int a = 0; a < n; ++a) {
            const R r = reg[qb + a];
            z = z + ((r > (R)0) ? r : (R)0);
        }
        for (int a = 0; a < n; ++a) {
            const R r = reg[qb + a];
            const R pos = (r > (R)0) ? r : (R)0;
            const R nsig = (z > (R)0) ? pos / z : (R)1 / (R)n;
            sig[qb + a] = nsig;
            if (!finite_(r) || !finite_(nsig) || !finite_(z)) bad = true;
        }
    }
    if (bad) atomicMin(&g.ctrl[1], t_iter);
    if (sp.trunk || last) {
        // the last CTA to finish: the chance-only trunk's values (Eq 1, depths c-1..0,
        // k_bwd's operations) from the subtree roots' values, then the iteration count
        __shared__ int is_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned long long prev = atomicAdd((unsigned long long*)&g.ctrl[2], 1ULL);
            is_last = (prev == gridDim.x - 1) ? 1 : 0;
        }
        __syncthreads();
        if (is_last) {
            __threadfence();
            if (sp.trunk) {
                const int4* tr = reinterpret_cast<const int4*>(T + sp.m_trunk);
                // trunk slots are level-major: deepest level last, so walk back by level
                for (int L = sp.cut - 1; L >= 0; --L) {
                    for (int k = threadIdx.x; k < sp.ntrunk; k += blockDim.x) {
                        const int4 e = tr[k];   // {node U row, first child U row, sigma_ext base, children | level << 16}
                        if ((e.w >> 16) != L) continue;
                        const int nch = e.w & 0xffff;
                        R v[PC];
#pragma unroll
                        for (int c = 0; c < PC; ++c) v[c] = (R)0;
                        for (int a = 0; a < nch; ++a) {
                            const R x = g.sig[e.z + a];
#pragma unroll
                            for (int c = 0; c < PC; ++c) v[c] = v[c] + x * g.U[(long long)(e.y + a) * PC + c];
                        }
#pragma unroll
                        for (int c = 0; c < PC; ++c) g.U[(long long)e.x * PC + c] = v[c];
                    }
                    __threadfence_block();
                    __syncthreads();
                }
            }
            if (threadIdx.x == 0) {
                if (last) g.ctrl[0] = t_iter;
                g.ctrl[2] = 0;
            }
        }
    }
}


}  // namespace cfrb
