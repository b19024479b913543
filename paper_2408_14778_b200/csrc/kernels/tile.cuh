// Generic backward tile kernel (any game; also EV / best-response modes): k_bwd.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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
            const bool keep = sm.seg[k].fused;
            if (keep) {
                const double x = is_pair ? xdec(c0, c1, c2, g.rc) : xdec(c0, c1, c2, g.rcp);
                if (rd == 0) kr0 = x;
                else if (rd == 1) kr1 = x;
                else if (rd == 2) kr2 = x;
                else if (rd == 3) kr3 = x;
                else kr4 = x;
            } else if (T.contrib) {
                // deferred infoset (spans tiles, depths or ranks): exact partial sums
                // into its global slices (CFR: r~ and pi_bar; BR: the best-response
                // sums of the BR player's infosets, decided by k_br_decide)
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
        // stored sums are negated, so player 2 takes the argmin.  A deferred
        // infoset (not complete in this tile) takes the action k_br_decide chose
        // after the previous pass (reading Q17: the BR passes repeat until every
        // deferred decision below is final; see Solver::best_response).
        for (int k = tid; k < nseg; k += nth) {
            if (sm.seg[k].owner != br_player) continue;
            if (!sm.seg[k].fused) {
                sm.best[k] = g.br_best[sm.seg[k].dh];
                continue;
            }
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

}  // namespace cfrb
