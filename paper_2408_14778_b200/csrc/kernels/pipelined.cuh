// Pipelined cp.async backward kernel for uniform f64 levels: k_bwd_fast.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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

}  // namespace cfrb
