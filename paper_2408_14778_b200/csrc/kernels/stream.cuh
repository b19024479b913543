// Streaming backward kernel (TMA producer warp + consumer warps): k_bwd_stream.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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
    int o_pact, o_fpar, o_fe;   // fused: parent actors, parent slots, incoming sigma_ext edges (TMA); the
                                // reach area holds the consumers' (pi_check, pi_hat) of the actor
    unsigned ndiv_m;        // p / n == (p * ndiv_m) >> ndiv_s (64-bit) for p < 2^16 (host-verified)
    int ndiv_s;
    int umem;               // > 0: every infoset of the level has umem members (m / umem by udiv)
    unsigned udiv_m;
    int udiv_s;
    int o_sv, o_cm, o_rt, o_pos, o_pib, o_zs, o_ccnt, o_bar;          // work arrays / barriers
    int bytes;              // dynamic shared memory
    int last;
    int debug;              // timing experiments only (CFR_STREAM_EXPERIMENTS builds): 1 consumers skip
                            // compute, 2 producer skips loads, 4/8/16/32 skip value writes / updates /
                            // value loop / compaction
    int level;              // parent level (work counters)
    int compact;            // 1: reach rows of this level are compact (pi_check, pi_hat of the actor; k_fwd compact)
    int defer;              // 1: every infoset of the level is deferred (spans ranks): exact partial sums are
                            //    added to the exchange block acc_r / acc_p; the update runs after the all-reduce
    long long dh0, dq0;     // defer: deferred index of the level's first infoset, its compact pair base
};
// The timing-experiment knobs (StreamLevel::debug) exist only in experiment
// builds (-DCFR_STREAM_EXPERIMENTS); the product build compiles them out.
#ifdef CFR_STREAM_EXPERIMENTS
#define STREAM_DEBUG(L) ((L).debug)
#else
#define STREAM_DEBUG(L) 0
#endif
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
// try_wait suspend-time hint: a waiting warp is parked by the hardware until the
// phase completes (or the hint elapses) instead of re-issuing the test, so
// waiting warps do not take issue slots from working ones
#ifndef CFR_WAIT_HINT_NS
#define CFR_WAIT_HINT_NS 1000000
#endif
constexpr unsigned kWaitHintNs = CFR_WAIT_HINT_NS;
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(kWaitHintNs)
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
    int fpo, feo;               // fused: parent-slot / edge window offsets
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
            mbar_init(&full[s], 1);
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
        // Lane 0 arms the stage and issues the TMA bulk copies.
        const int plane = tid - kStreamConsumers;
        if (plane != 0) return;   // lane 0 alone issues
        const int4* recs = reinterpret_cast<const int4*>(pool) + L.rec;
        const int* hs = pool + L.hs;
        long long t = blockIdx.x;
        int4 rec = (t < L.ntiles) ? recs[t] : make_int4(0, 0, 0, 0);
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
            {
                const long long q = L.q0 + (long long)k0 * n;
                const long long h = L.h0 + k0;
                unsigned b_rows, b_reach = 0, b_sig, b_reg, b_snum, b_sden, b_own, b_hs, b_node, b_pact = 0, b_fpar = 0, b_fe = 0;
                int o_rows, o_reach = 0, po, po2, po3, ho, oo, hso, no, pao = 0, fpo = 0, feo = 0;
                const unsigned char* w_fpar = nullptr;
                const unsigned char* w_fe = nullptr;
                const unsigned char* w_rows = window16(g.U + (L.row0 + (long long)m0 * n) * PC, (long long)M * L.rowlen, &b_rows, &o_rows);
                const unsigned char* w_reach = nullptr;
                const unsigned char* w_pact = nullptr;
                if (L.fused) {
                    w_pact = window16(g.f_pact + slot, M, &b_pact, &pao);
                    w_fpar = window16(g.f_parent + slot, M, &b_fpar, &fpo);
                    w_fe = window16(g.f_e + slot, M, &b_fe, &feo);
                }
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
                hd->fpo = fpo;
                hd->feo = feo;
                (void)po2; (void)po3;   // sigma / R / S_num share the pair window offset (same base alignment)
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                if (STREAM_DEBUG(L) == 2) {   // timing experiment: no loads (consumers compute on stale data)
                    mbar_expect_tx(&full[st], 0);
                } else {
                    mbar_expect_tx(&full[st], b_rows + b_reach + b_sig + b_reg + b_snum + b_sden + b_own + b_hs + b_node +
                                                  b_pact + b_fpar + b_fe);
                    bulk_g2s(S + L.o_node, w_node, b_node, &full[st]);
                    bulk_g2s(S + L.o_rows, w_rows, b_rows, &full[st]);
                    if (L.fused) {
                        bulk_g2s(S + L.o_pact, w_pact, b_pact, &full[st]);
                        bulk_g2s(S + L.o_fpar, w_fpar, b_fpar, &full[st]);
                        bulk_g2s(S + L.o_fe, w_fe, b_fe, &full[st]);
                    } else {
                        bulk_g2s(S + L.o_reach, w_reach, b_reach, &full[st]);
                    }
                    bulk_g2s(S + L.o_sig, w_sig, b_sig, &full[st]);
                    bulk_g2s(S + L.o_reg, w_reg, b_reg, &full[st]);
                    bulk_g2s(S + L.o_snum, w_snum, b_snum, &full[st]);
                    bulk_g2s(S + L.o_sden, w_sden, b_sden, &full[st]);
                    bulk_g2s(S + L.o_own, w_own, b_own, &full[st]);
                    bulk_g2s(S + L.o_hs, w_hs, b_hs, &full[st]);
                }
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
    const int rs = (L.compact || L.fused) ? 2 : 2 * P;   // reach row stride in the stage (elements)
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
        const I* fpar = reinterpret_cast<const I*>(S + L.o_fpar) + hd.fpo;                         // fused only
        const I* fedge = reinterpret_cast<const I*>(S + L.o_fe) + hd.feo;                          // fused only
        const int nseg = hd.nseg, M = hd.M, m0 = hd.m0;

        if (STREAM_DEBUG(L) == 1) {   // timing experiment: data movement only
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
                // fused forward (Eq 2 pi_check, Eq 4 pi_hat with reading Q1, the k_fwd
                // arithmetic): the actor's two factors of the parent's reach row and
                // the incoming edge's sigma are loaded now, in flight during the value pass
                R fpc = (R)0, fph = (R)0, fx = (R)0;
                int fact = 0;
                if (L.fused) {
                    const int ia = own[k];
                    const R* prow = g.reach + (long long)fpar[m] * 2 * P;
                    fpc = __ldg(prow + ia - 1);
                    fph = __ldg(prow + P + ia - 1);
                    fx = __ldg(g.sig + (long long)fedge[m]);
                    fact = pact[m];
                }
                R v[PC];
#pragma unroll
                for (int j = 0; j < PC; ++j) v[j] = (R)0;
                const R* row = rows + (long long)m * L.rowlen;
                const R* sg = ssig + k * n;
                if (STREAM_DEBUG(L) & 16) {   // timing experiment: no value loop
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
                        // (f64 only: for float4 rows the selects cost more than the
                        // conflicts -- L10 f32 0.871 vs 0.892 ms without the stagger,
                        // f64 1.385 vs 1.352 ms)
                        const int d = (sizeof(R) == 8) ? ((m >> 2) & 1) : 0;
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
                } else if (PC == 2 && vec_rows) {
                    // two value columns (general-sum two-player games): 16-byte row
                    // reads, four chunks in flight per step; the two columns' sums
                    // are independent chains, each in ascending action order
                    using V = typename std::conditional<sizeof(R) == 8, double2, float4>::type;
                    constexpr int E = 16 / (2 * (int)sizeof(R));   // actions per 16-byte chunk
                    const V* row4 = reinterpret_cast<const V*>(row);
                    const int nc = n / E;
                    int c = 0;
                    for (; c + 4 <= nc; c += 4) {
                        const V p0 = row4[c], p1 = row4[c + 1], p2 = row4[c + 2], p3 = row4[c + 3];
                        const R* u0 = reinterpret_cast<const R*>(&p0);
                        const R* u1 = reinterpret_cast<const R*>(&p1);
                        const R* u2 = reinterpret_cast<const R*>(&p2);
                        const R* u3 = reinterpret_cast<const R*>(&p3);
                        const int a0 = c * E;
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const R x = sg[a0 + e];
                            v[0] = v[0] + x * u0[2 * e];
                            v[1] = v[1] + x * u0[2 * e + 1];
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const R x = sg[a0 + E + e];
                            v[0] = v[0] + x * u1[2 * e];
                            v[1] = v[1] + x * u1[2 * e + 1];
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const R x = sg[a0 + 2 * E + e];
                            v[0] = v[0] + x * u2[2 * e];
                            v[1] = v[1] + x * u2[2 * e + 1];
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            const R x = sg[a0 + 3 * E + e];
                            v[0] = v[0] + x * u3[2 * e];
                            v[1] = v[1] + x * u3[2 * e + 1];
                        }
                    }
                    for (int a = c * E; a < n; ++a) {
                        const R x = sg[a];
                        v[0] = v[0] + x * row[2 * a];
                        v[1] = v[1] + x * row[2 * a + 1];
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
                    if (!(STREAM_DEBUG(L) & 4)) g.U[node * PC + j] = v[j];   // (debug bit 4: timing experiment)
                    sv[m * PC + j] = v[j];
                }
                const int i = own[k];
                if (L.fused) {
                    // the member's (pi_check, pi_hat) of the actor, kept for phase B
                    pc = (fact != i) ? fpc * fx : fpc;
                    ph = (fact == i) ? fph * fx : fph;
                    R* rw = const_cast<R*>(reach) + (long long)m * 2;
                    rw[0] = pc;
                    rw[1] = ph;
                } else {
                    pc = reach[(long long)m * rs + (L.compact ? 0 : i - 1)];
                    ph = reach[(long long)m * rs + (L.compact ? 1 : P + i - 1)];
                }
            }
            SPROF(3);
            if (STREAM_DEBUG(L) & 32) continue;   // timing experiment: no compaction
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
            // (a deferred infoset contributes only nonzero partial sums; its update
            // runs after the exchange)
            const unsigned live = __ballot_sync(
                0xffffffffu, lane < nseg && (L.defer ? (ccnt[lane] != 0 || ccnt[L.maxseg + lane] != 0)
                                                     : (g.upd_player == 0 || own[lane] == g.upd_player) &&
                                                           (all_live || ccnt[lane] != 0 || ccnt[L.maxseg + lane] != 0)));
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
                        double e0 = 0, e1 = 0, e2 = 0;   // second independent slice chain (ILP; a 4-chain variant measured slower)
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
                    if (L.defer) {
                        // exact partial sums of this rank's members (int64 slices, any order)
                        if (part == 0 && itm <= n && (c0 != 0.0 || c1 != 0.0 || c2 != 0.0)) {
                            unsigned long long* acc = (itm < n) ? g.acc_r + (L.dq0 + (long long)(hd.k0 + k) * n + itm) * 3
                                                                : g.acc_p + (L.dh0 + hd.k0 + k) * 3;
                            atomicAdd(acc + 0, (unsigned long long)(long long)c0);
                            atomicAdd(acc + 1, (unsigned long long)(long long)c1);
                            atomicAdd(acc + 2, (unsigned long long)(long long)c2);
                        }
                    } else if (part == 0) {
                        if (itm < n) rt[k * n + itm] = (R)xdec(c0, c1, c2, g.rc);
                        else if (itm == n) pib[k] = (R)xdec(c0, c1, c2, g.rcp);
                    }
                }
                __syncwarp();
                if (L.defer) continue;   // updated by k_deferred after the exchange
                // ---- phase C: Eq 8/15 or CFR+, Eq 10, then Eq 9 (z ascending)
                const R wp = w * pib[k];
                for (int c = 0; c < n; c += 32) {
                    const int a = c + lane;
                    if (a < n) {
                        const int p = k * n + a;
                        const R r_t = rt[p];
                        const R r = upd_regret(up, sreg[p], r_t);   // Eq 8/15 (Q4) / CFR+ (Q6) / Q18
                        if (!(STREAM_DEBUG(L) & 8)) {   // (debug bit 8: timing experiment)
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
                if (lane == 0 && !(STREAM_DEBUG(L) & 8)) g.sden[ht + k] = upd_sum(up, sden[k], wp);   // Eq 10 denominator
                for (int c = 0; c < n; c += 32) {
                    const int a = c + lane;
                    if (a < n) {
                        const int p = k * n + a;
                        const R nsig = (z > (R)0) ? pos[p] / z : inv_n;   // Eq 9
                        if (!(STREAM_DEBUG(L) & 8)) g.sig[qt + p] = nsig;
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

}  // namespace cfrb
