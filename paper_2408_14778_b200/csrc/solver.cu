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

// device code, one header per kernel family
#include "kernels/common.cuh"
#include "kernels/forward.cuh"
#include "kernels/tile.cuh"
#include "kernels/stream.cuh"
#include "kernels/update.cuh"
#include "kernels/small.cuh"
#include "kernels/subtree.cuh"

namespace cfrb {

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
    virtual cfr_status set_state(int64_t T, const double* regret, const double* snum, const double* sden) = 0;
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
    virtual cfr_status br_phase(int ph, int player, double* out) = 0;
    virtual cfr_status br_passes_out(int32_t* n) = 0;
    virtual cfr_status run_tracked(int64_t iters, int64_t every, double* out, int64_t* rows) = 0;
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

// child-row bytes per streaming tile (the n = 40 synthetic's f64 tiles: 240 x 160 B)
constexpr int kStreamRowBytes = 40960;

// Shared-memory plan of k_bwd_stream for one level (stage ring + work arrays +
// barriers).  Every block is 16-byte aligned; windows get 16 bytes of slack.
static void stream_plan(StreamLevel& f, int P, int Pc, int w, int ix, int stages) {
    auto al = [](long long x) { return (int)((x + 15) & ~15ll); };
    const int maxpairs = f.maxm > 0 ? f.maxseg * f.n : 0;
    int o = al(sizeof(StreamHdr));
    f.o_rows = o; o += al((long long)f.maxm * f.rowlen * w + 16);
    f.o_reach = o; o += al((long long)f.maxm * (f.fused ? 2 : 2 * P) * w + 16);   // fused: consumer-written (pc, ph)
    f.o_sig = o; o += al((long long)maxpairs * w + 16);
    f.o_reg = o; o += al((long long)maxpairs * w + 16);
    f.o_snum = o; o += al((long long)maxpairs * w + 16);
    f.o_sden = o; o += al((long long)f.maxseg * w + 16);
    f.o_own = o; o += al((long long)f.maxseg + 16);
    f.o_hs = o; o += al((long long)(f.maxseg + 1) * 4 + 16);
    f.o_node = o; o += al((long long)f.maxm * ix + 16);
    f.o_pact = o; o += f.fused ? al((long long)f.maxm + 16) : 0;
    f.o_fpar = o; o += f.fused ? al((long long)f.maxm * ix + 16) : 0;
    f.o_fe = o; o += f.fused ? al((long long)f.maxm * ix + 16) : 0;
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
                                              bool compact_reach, const std::vector<uint8_t>& contrib) {
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
        // every infoset of the level fused (updated here), or every one deferred
        // (spanning ranks: exact partial sums into the exchange block, updated
        // after the all-reduce) with consecutive deferred indices; a deferred
        // level must lie below the cut (every tile contributes)
        int mode = -1;   // 0 fused, 1 deferred
        for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1] && ok; ++t)
            for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1 && ok; ++k) {
                const SegH& sg = g.segs[k];
                const int nn = (int)(g.qbase_int[sg.h + 1] - g.qbase_int[sg.h]);
                const int m = sg.fused ? 0 : (g.deferred[sg.h] ? 1 : 2);
                if (m == 2 || (mode >= 0 && m != mode) || sg.sb != next || (h_prev >= 0 && sg.h != h_prev + 1) ||
                    (n >= 0 && nn != n) || sg.se - sg.sb > tile_target)
                    ok = false;
                if (m == 1 && h_prev >= 0 && g.dpos[sg.h] != g.dpos[h_prev] + 1) ok = false;
                if (m == 1 && !contrib.empty() && !contrib[t]) ok = false;
                mode = m;
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
        // tiles: greedy runs of whole infosets, <= 32 infosets, at most tile_target
        // members and about kStreamRowBytes of child rows per stage (wide rows --
        // e.g. two value columns of a general-sum game -- get fewer members, so two
        // CTAs with two-stage rings stay resident per SM), never fewer members
        // than the level's largest infoset
        int maxmem = 1;
        for (int k = 0; k < nh; ++k) maxmem = std::max(maxmem, hs[k + 1] - hs[k]);
        const int tt = std::max(maxmem, std::min(tile_target, kStreamRowBytes / std::max(1, n * Pc * w)));
        std::vector<int> tk = {0};
        for (int k = 0; k < nh; ++k) {
            const int k0 = tk.back();
            if (k > k0 && (hs[k + 1] - hs[k0] > tt || k + 1 - k0 > 32)) tk.push_back(k);
        }
        tk.push_back(nh);
        f.ntiles = (long long)tk.size() - 1;
        if (f.ntiles < min_tiles) { out[L] = StreamLevel{}; continue; }
        f.s0 = s0;
        f.h0 = g.segs[g.tiles[g.tile_ptr[L]].seg0].h;
        f.q0 = g.qbase_int[f.h0];
        f.defer = mode == 1 ? 1 : 0;
        if (f.defer) {
            f.dh0 = g.dpos[f.h0];
            f.dq0 = g.dqbase[f.dh0];
        }
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
        f.fused = (fuse_forward && L == g.D - 1) ? 1 : 0;
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

// In-graph exploitability record (cfr_solver_run_tracked): per evaluation one
// row of root values -- EV (Pc columns), then each player's best-response root
// row (Pc columns each), then the iteration count.
constexpr int kRecRows = 1024;
static int rec_width(const Game& g) { return g.Pc + g.P * g.Pc + 1; }

// Subtree mode (k_sub, kernels/subtree.cuh): games up to kSubMaxV nodes reserve
// its tables; at most kSubMaxSub subtrees (CTAs) per cut.
constexpr int64_t kSubMaxV = int64_t(1) << 22;
constexpr int64_t kSubMaxSub = 16384;
constexpr int64_t kSubMinV = 2048;      // default: below this k_tiny (many iterations per launch) wins (Kuhn)
constexpr int64_t kSubMinCTAs = 24;     // preferred minimum of subtrees (CTAs) when choosing the cut
constexpr int64_t kSubStreamV = int64_t(1) << 20;   // above: games with streaming levels keep the level path
static bool sub_candidate(const Game& g) { return g.V <= kSubMaxV && g.D >= 2 && g.NS > 0; }
// ints: per-subtree records, node records, child entries (<= V), pair entries
// (<= V), per-level node and pair starts of every subtree
static size_t sub_table_bound(const Game& g) {
    return (size_t)(kSubMeta * kSubMaxSub + kSubRec * g.NS + 5 * g.V + 2 * kSubMaxSub * (g.D + 2) + 16 * kSubMaxSub +
                    4 * g.NS + 64);
}

template <class R, class I>
struct Plan {
    size_t U, reach, sig, sig_eval, regret, snum, sden, acc_r, acc_p, dqbase;
    size_t f_parent, f_e, f_pact;
    size_t s_node, s_cb, s_n, s_ebase, s_actor, s_dec, s_coff;
    size_t qbase, owner, tiles, segs, deferred, br_best, ctrl, lcnt, out, rec;
    size_t cutbuf, cutrow, cutown, report, spool, tmeta;
    size_t subt, subu, suba;   // subtree mode (k_sub): int32 tables, terminal utilities, exact accumulators
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
        br_best = L.take<int>(g.deferred_list.size() + 1);
        ctrl = L.take<long long>(8);
        lcnt = L.take<unsigned long long>(4 * (size_t)g.D + 4);
        out = L.take<R>(std::max<size_t>(Q + C, (size_t)g.P * 2 + 8));
        const size_t ncut = sh ? sh->cut_row.size() : 0;
        cutbuf = L.take<R>(ncut * g.Pc + 1);
        cutrow = L.take<long long>(ncut + 1);
        cutown = L.take<unsigned char>(ncut + 1);
        report = L.take<unsigned char>(H + 1);
        spool = L.take<int>(stream_pool_bound(g));
        // k_tiny's int32 game tables (TinyMeta), tiny-game candidates only
        tmeta = L.take<int>(g.V <= (int64_t(1) << 20) ? (size_t)(4 * (g.D + 1) + 7 * NS + 4 * H + Q + 16) : 2);
        rec = L.take<double>((size_t)kRecRows * rec_width(g));
        // subtree mode: reserved for candidate games only (sub_candidate)
        const bool sc = sub_candidate(g);
        subt = L.take<int>(sc ? sub_table_bound(g) : 2);
        subu = L.take<R>(sc ? (size_t)g.V * g.Pc + 2 : 2);
        suba = L.take<unsigned long long>(sc ? 3 * (Q + H) + 3 : 3);
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
    bool tiny_ = false;           // tiny game: whole iterations in one CTA, state in shared memory (k_tiny)
    TinyPlan tiny_plan_{};
    bool sub_ = false;            // subtree mode: levels >= cut in one k_sub launch + k_sub_update
    SubPlan sub_plan_{};
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

    // NCCL mode: exchange 2 per level, overlapped with the shallower levels.  A
    // deferred infoset's sums are complete once its shallowest level is done
    // (levels run deep -> shallow); internal ids are assigned level by level, so
    // the deferred infosets first seen at level L are one contiguous range of
    // deferred indices [xr_[L].first, xr_[L].second).
    std::vector<std::pair<int64_t, int64_t>> xr_;
    cudaStream_t xstream_ = nullptr;          // the communication stream
    std::vector<cudaEvent_t> xev_;            // fork / join events (2 per level + 1)

    ~Solver() override {
        // the workspace belongs to the caller: no kernel may still run on it once
        // the handle is gone (the caller frees it after cfr_solver_destroy)
        cudaStreamSynchronize(stream);
        if (xstream_) cudaStreamSynchronize(xstream_);
        for (cudaEvent_t e : xev_) cudaEventDestroy(e);
        if (xstream_) cudaStreamDestroy(xstream_);

        if (pinned_) cudaFreeHost(pinned_);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (eval_exec_) cudaGraphExecDestroy(eval_exec_);
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
        if (comm) {
            // deferred-index range of the infosets first seen at each level
            xr_.assign(g.D, std::make_pair((int64_t)0, (int64_t)0));
            std::vector<int> first(g.H, INT32_MAX);
            for (int L = 0; L < g.D; ++L)
                for (int64_t t = g.tile_ptr[L]; t < g.tile_ptr[L + 1]; ++t)
                    for (int k = g.tiles[t].seg0; k < g.tiles[t].seg1; ++k)
                        first[g.segs[k].h] = std::min(first[g.segs[k].h], L);
            // a rank sees only its own members: the shallowest level of every
            // deferred infoset is the minimum over the ranks (one all-reduce at
            // creation), so every rank derives the same ranges and issues the same
            // sequence of collectives
            const size_t ndef = g.deferred_list.size();
            std::vector<int> fl(ndef + 1, INT32_MAX);
            for (size_t d = 0; d < ndef; ++d) fl[d] = first[g.deferred_list[d]];
            {
                int* dfl = nullptr;
                CU(cudaMalloc(&dfl, fl.size() * sizeof(int)));
                cudaError_t ce = cudaMemcpyAsync(dfl, fl.data(), fl.size() * sizeof(int), cudaMemcpyHostToDevice, stream);
                ncclResult_t nr = ncclSuccess;
                if (!ce) nr = ncclAllReduce(dfl, dfl, fl.size(), ncclInt32, ncclMin, comm, stream);
                if (!ce && nr == ncclSuccess)
                    ce = cudaMemcpyAsync(fl.data(), dfl, fl.size() * sizeof(int), cudaMemcpyDeviceToHost, stream);
                if (!ce) ce = cudaStreamSynchronize(stream);
                cudaFree(dfl);
                if (nr != ncclSuccess) {
                    cfrb_set_error(std::string("ncclAllReduce: ") + ncclGetErrorString(nr));
                    return CFR_ERR_NCCL;
                }
                CU(ce);
            }
            std::vector<int64_t> lo(g.D, INT64_MAX), hi(g.D, -1);
            for (size_t d = 0; d < ndef; ++d) {
                const int L = fl[d];
                if (L == INT32_MAX) continue;
                lo[L] = std::min(lo[L], (int64_t)d);
                hi[L] = std::max(hi[L], (int64_t)d + 1);
            }
            int64_t next = 0;
            bool contiguous = true;
            for (int L = 0; L < g.D; ++L) {   // shallow -> deep: ranges must tile [0, ndef) in order
                if (hi[L] < 0) continue;
                if (lo[L] != next || hi[L] - lo[L] <= 0) contiguous = false;
                xr_[L] = std::make_pair(lo[L], hi[L]);
                next = hi[L];
            }
            if (!contiguous || next != (int64_t)g.deferred_list.size()) xr_.clear();   // one exchange after the pass
            if (!xr_.empty()) {
                CU(cudaStreamCreateWithFlags(&xstream_, cudaStreamNonBlocking));
                xev_.resize(2 * g.D + 2);
                for (cudaEvent_t& e : xev_) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
        }

        if (cfg.flags & CFR_FLAG_PERSISTENT) {
            cfrb_set_error("CFR_FLAG_PERSISTENT (the cooperative single-launch kernel) was removed: measured slower "
                           "than the CUDA-graph iteration on B200; tiny games use k_tiny (DESIGN.md 6.1)");
            return CFR_ERR_UNSUPPORTED;
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
        dg.br_best = at<int>(plan.br_best);
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
            // tables of the streaming levels
            std::vector<int> sp;
            int stages = 2;
            if (const char* e = std::getenv("CFR_STREAM_STAGES")) stages = std::max(2, std::min(8, std::atoi(e)));
#ifdef CFR_STREAM_EXPERIMENTS
            if (const char* e = std::getenv("CFR_STREAM_DEBUG")) stream_debug_ = std::atoi(e);
#endif
            // members per tile: ~240 f64 / ~480 f32 keeps two CTAs (2-stage rings of
            // ~50 KB) resident per SM (measured best, tools/stream_sweep.py)
            int tile = (sizeof(R) == 4 && !(cfg.flags & CFR_FLAG_FUSED_FORWARD)) ? 2 * kStreamConsumers : kStreamConsumers;
            if (const char* e = std::getenv("CFR_STREAM_TILE")) tile = std::max(32, std::min(1024, std::atoi(e)));
            // levels with fewer tiles than min_tiles stay on the tile kernel (CFR_STREAM_MIN_TILES: A/B)
            int min_tiles = num_sms_;
            if (const char* e = std::getenv("CFR_STREAM_MIN_TILES")) min_tiles = std::max(1, std::atoi(e));
            stream_ = stream_levels<R, I>(g, s_cb_u, &sp, (cfg.flags & CFR_FLAG_FORCE_STREAM) ? 1 : min_tiles, stages, tile,
                                          (cfg.flags & CFR_FLAG_FUSED_FORWARD) != 0, std::getenv("CFR_NO_COMPACT") == nullptr,
                                          tile_contrib_);
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
        CU(cudaMemsetAsync(ws + plan.br_best, 0, (g.deferred_list.size() + 1) * sizeof(int), stream));
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
            // subtree mode first (latency-bound games beyond the tiniest), else k_tiny
            cfr_status ps = setup_sub();
            if (ps) return ps;
            if (!sub_ && (ps = setup_tiny())) return ps;
            if (sub_) launches_per_iter = count_launches();
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

    bool has_def_() const { return !gp->deferred_list.empty(); }

    bool tiny_meta_smem_ = false;   // k_tiny's game tables are in shared memory
    void* tiny_fn() const {
        const bool m = tiny_meta_smem_;
        switch (gp->Pc) {
            case 1: return m ? (void*)k_tiny<R, I, 1, true> : (void*)k_tiny<R, I, 1, false>;
            case 2: return m ? (void*)k_tiny<R, I, 2, true> : (void*)k_tiny<R, I, 2, false>;
            case 3: return m ? (void*)k_tiny<R, I, 3, true> : (void*)k_tiny<R, I, 3, false>;
            default: return m ? (void*)k_tiny<R, I, 4, true> : (void*)k_tiny<R, I, 4, false>;
        }
    }
    // Tiny-game mode (k_tiny): single-GPU, depth-homogeneous games whose mutable
    // state fits one CTA's shared memory.  On by default (CFR_FLAG_NO_TINY to opt out).
    cfr_status setup_tiny() {
        const Game& g = *gp;
        tiny_ = false;
        if (world > 1 || external || (cfg.flags & (CFR_FLAG_NO_TINY | CFR_FLAG_FORCE_SUBTREE)) || !g.depth_homogeneous ||
            g.NS == 0)
            return CFR_OK;
        const long long nU = (long long)(plan_u_rows()) * g.Pc, nreach = 2LL * g.P * g.NS, nsig = g.Q + g.C;
        int dev = 0, optin = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        // everything in shared memory if it fits, else node values U stay in global
        // memory (L1 / L2) and the rest is shared (e.g. Leduc in f64)
        TinyPlan tp{};
        long long bytes = 0;
        for (int u_global = 0; u_global <= 1; ++u_global) {
            tp = TinyPlan{};
            long long o = 0;
            auto take = [&](long long n) { const long long r = o; o += (n + 1) & ~1LL; return r; };   // 16-byte aligned
            tp.U = u_global ? -1 : take(nU);
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
            bytes = o * (long long)sizeof(R);
            if (bytes <= optin - 1024) break;
        }
        if (bytes > optin - 1024) return CFR_OK;
        // per level: slots and its (consecutive) infosets; members of each infoset
        std::vector<int64_t> lvv(4 * (size_t)(g.D + 1), 0);
        std::vector<int64_t> mem(2 * (size_t)g.H + 2, -1);
        for (int L = 0; L < g.D; ++L) {
            lvv[4 * L] = g.slot_ptr[L];
            lvv[4 * L + 1] = g.slot_ptr[L + 1];
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
                lvv[4 * L + 2] = h0;
                lvv[4 * L + 3] = h1;
            }
        }
        for (int64_t h = 0; h < g.H; ++h)
            if (mem[2 * h] < 0) return CFR_OK;
        for (int L = 0; L < g.D; ++L)   // each level's infosets must be a consecutive id range
            for (long long h = lvv[4 * L + 2]; h < lvv[4 * L + 3]; ++h)
                if (mem[2 * h] < g.slot_ptr[L] || mem[2 * h + 1] > g.slot_ptr[L + 1]) return CFR_OK;
        // TinyMeta: int32 tables (the slot tables come back from the device
        // arrays the per-level kernels use, so both paths read the same numbers)
        const int64_t NS = g.NS;
        tp.m_lv = 0;
        tp.m_slot = 4 * (g.D + 1);
        tp.m_qb = (int)(tp.m_slot + 7 * NS);
        tp.m_own = (int)(tp.m_qb + g.H + 1);
        tp.m_mem = (int)(tp.m_own + g.H);
        tp.m_ph = (int)(tp.m_mem + 2 * g.H);
        tp.meta_ints = (int)(tp.m_ph + g.Q);
        std::vector<int> meta((size_t)tp.meta_ints, 0);
        for (size_t k = 0; k < lvv.size(); ++k) meta[tp.m_lv + k] = (int)lvv[k];
        {
            std::vector<I> fp(NS), fe(NS), cb(NS), eb(NS), nd(NS);
            std::vector<unsigned char> pa(NS);
            std::vector<int> nn(NS);
            CU(cudaStreamSynchronize(stream));   // the uploads of the device tables are done
            CU(cudaMemcpy(fp.data(), ws + plan.f_parent, NS * sizeof(I), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(fe.data(), ws + plan.f_e, NS * sizeof(I), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(pa.data(), ws + plan.f_pact, NS, cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(cb.data(), ws + plan.s_cb, NS * sizeof(I), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(eb.data(), ws + plan.s_ebase, NS * sizeof(I), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(nn.data(), ws + plan.s_n, NS * sizeof(int), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(nd.data(), ws + plan.s_node, NS * sizeof(I), cudaMemcpyDeviceToHost));
            for (int64_t k = 0; k < NS; ++k) {
                int* e = &meta[tp.m_slot + 7 * k];
                e[0] = (int)fp[k];
                e[1] = (int)fe[k];
                e[2] = (int)pa[k];
                e[3] = (int)cb[k];
                e[4] = (int)eb[k];
                e[5] = nn[k];
                e[6] = (int)nd[k];
            }
        }
        for (int64_t h = 0; h <= g.H; ++h) meta[tp.m_qb + h] = (int)g.qbase_int[h];
        for (int64_t h = 0; h < g.H; ++h) {
            meta[tp.m_own + h] = (int)g.owner_int[h];
            meta[tp.m_mem + 2 * h] = (int)mem[2 * h];
            meta[tp.m_mem + 2 * h + 1] = (int)mem[2 * h + 1];
            for (int64_t q = g.qbase_int[h]; q < g.qbase_int[h + 1]; ++q) meta[tp.m_ph + q] = (int)h;
        }
        // the tables join the state in shared memory when both fit (Kuhn)
        const long long meta_bytes = 4LL * tp.meta_ints;
        tp.meta_off = (int)((bytes + 15) & ~15LL);
        tiny_meta_smem_ = tp.meta_off + meta_bytes <= optin - 1024;
        tp.bytes = tiny_meta_smem_ ? (int)(tp.meta_off + meta_bytes) : (int)bytes;
        CU(cudaFuncSetAttribute(tiny_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, tp.bytes));
        cfr_status st = up(plan.tmeta, meta);
        if (st) return st;
        CU(cudaStreamSynchronize(stream));
        // one thread per slot / item of the widest level (fewer warps = cheaper
        // barriers on games like Kuhn), at most 1024
        int64_t widest = 32;
        for (int L = 0; L < g.D; ++L) {
            widest = std::max<int64_t>(widest, lvv[4 * L + 1] - lvv[4 * L]);
            const int64_t h0 = lvv[4 * L + 2], h1 = lvv[4 * L + 3];
            if (h1 > h0) widest = std::max<int64_t>(widest, (g.qbase_int[h1] - g.qbase_int[h0]) + (h1 - h0));
        }
        tiny_threads_ = (int)std::min<int64_t>(1024, (widest + 31) / 32 * 32);
        tiny_plan_ = tp;
        tiny_ = true;
        return CFR_OK;
    }
    int tiny_threads_ = 1024;
    long long plan_u_rows() const { return (long long)u_layout(*gp, sizeof(R)).back(); }
    cfr_status launch_tiny(int64_t iters) {
        const Game& g = *gp;
        const int* meta = reinterpret_cast<const int*>(ws + plan.tmeta);
        const int D = g.D;
        const long long T = (long long)iters;
        const TinyPlan tp = tiny_plan_;
#define CFRB_TINY(PC)                                                                                              \
    (tiny_meta_smem_ ? launch(pdl_, k_tiny<R, I, PC, true>, dim3(1), dim3(tiny_threads_), (size_t)tp.bytes, stream, dg, meta, D, T, tp) \
                     : launch(pdl_, k_tiny<R, I, PC, false>, dim3(1), dim3(tiny_threads_), (size_t)tp.bytes, stream, dg, meta, D, T, tp))
        switch (g.Pc) {
            case 1: CFRB_TINY(1); break;
            case 2: CFRB_TINY(2); break;
            case 3: CFRB_TINY(3); break;
            default: CFRB_TINY(4); break;
        }
#undef CFRB_TINY
        CU(cudaGetLastError());
        return CFR_OK;
    }

    // Subtree mode (k_sub, kernels/subtree.cuh):
    // single-GPU, depth-homogeneous games of <= kSubMaxV nodes without deferred
    // infosets that are not tiny.  The cut is the shallowest level whose every
    // subtree fits one CTA's shared memory (CFR_SUB_CUT overrides).  On by default
    // for those games (CFR_FLAG_NO_SUBTREE opts out); CFR_FLAG_FORCE_SUBTREE also
    // takes games k_tiny would run.
    void* sub_fn(bool staged) const {
        switch (gp->Pc) {
            case 1: return staged ? (void*)k_sub<R, I, 1, true> : (void*)k_sub<R, I, 1, false>;
            case 2: return staged ? (void*)k_sub<R, I, 2, true> : (void*)k_sub<R, I, 2, false>;
            case 3: return staged ? (void*)k_sub<R, I, 3, true> : (void*)k_sub<R, I, 3, false>;
            default: return staged ? (void*)k_sub<R, I, 4, true> : (void*)k_sub<R, I, 4, false>;
        }
    }
    cfr_status setup_sub() {
        const Game& g = *gp;
        sub_ = false;
        // flags that select another kernel family (tests, A/B) keep it unless forced
        const int other = CFR_FLAG_NO_TINY | CFR_FLAG_NO_STREAM | CFR_FLAG_FORCE_STREAM | CFR_FLAG_FUSED_FORWARD |
                          CFR_FLAG_INDEX64;
        const bool forced = (cfg.flags & CFR_FLAG_FORCE_SUBTREE) != 0;
        if (!forced && (cfg.flags & other)) return CFR_OK;
        if (!forced) {
            // default: latency-bound games only -- not the tiniest (k_tiny runs many
            // iterations per launch there); above kSubStreamV nodes, a game with a
            // level big enough for the streaming kernel keeps the level path when
            // most of its nodes are terminals (bandwidth-bound: Battleship-7, 92 %
            // terminals, 120 vs 190 us/it) and takes k_sub otherwise (Goofspiel-6,
            // 26 % terminals, 163 vs 292 us/it)
            if (g.V < kSubMinV) return CFR_OK;
            if (g.V > kSubStreamV && 2 * g.num_terminals > g.V)
                for (const StreamLevel& f : stream_)
                    if (use_stream_ && f.ntiles > 0) return CFR_OK;
        }
        if (world > 1 || external || (cfg.flags & CFR_FLAG_NO_SUBTREE) || !g.depth_homogeneous || !sub_candidate(g) ||
            g.Pc > 4)
            return CFR_OK;
        const int64_t NS = g.NS;
        const int P = g.P, Pc = g.Pc, w = (int)sizeof(R);
        int dev = 0, optin = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        const long long budget = optin - 1024;
        // the device slot tables (the numbers the level kernels use)
        std::vector<I> fe(NS), cb(NS), eb(NS), nd(NS), fpar(NS);
        std::vector<unsigned char> pa(NS), ac(NS);
        std::vector<int> nn(NS);
        const long long nU = plan_u_rows() * Pc;
        std::vector<R> U((size_t)nU);
        CU(cudaStreamSynchronize(stream));
        CU(cudaMemcpy(fpar.data(), ws + plan.f_parent, NS * sizeof(I), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(fe.data(), ws + plan.f_e, NS * sizeof(I), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(pa.data(), ws + plan.f_pact, NS, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(ac.data(), ws + plan.s_actor, NS, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(cb.data(), ws + plan.s_cb, NS * sizeof(I), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(eb.data(), ws + plan.s_ebase, NS * sizeof(I), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(nn.data(), ws + plan.s_n, NS * sizeof(int), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(nd.data(), ws + plan.s_node, NS * sizeof(I), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(U.data(), ws + plan.U, (size_t)nU * sizeof(R), cudaMemcpyDeviceToHost));
        // U row -> slot (non-terminal rows), slot -> internal infoset
        std::vector<int64_t> rowslot((size_t)plan_u_rows() + 1, -1);
        for (int64_t x = 0; x < NS; ++x) rowslot[(size_t)nd[x]] = x;
        std::vector<int64_t> sh(NS, -1);
        for (const SegH& sg : g.segs)
            for (int64_t x = sg.sb; x < sg.se; ++x) sh[x] = sg.h;
        std::vector<int> lev(NS, 0);
        for (int L = 0; L < g.D; ++L)
            for (int64_t x = g.slot_ptr[L]; x < g.slot_ptr[L + 1]; ++x) lev[x] = L;
        for (int64_t x = 0; x < NS; ++x) {
            if (ac[x] != 0 && (sh[x] < 0 || (int64_t)eb[x] != g.qbase_int[sh[x]])) return CFR_OK;
            if (nn[x] > 256) return CFR_OK;
        }
        // subtree sizes (non-terminal nodes, terminals), deepest level first
        // subtree sizes (non-terminal nodes, terminals, player (node, action) pairs,
        // levels), deepest level first
        std::vector<int64_t> snn(NS, 0), snt(NS, 0), snp(NS, 0), sdep(NS, 0);
        for (int L = g.D - 1; L >= 0; --L)
            for (int64_t x = g.slot_ptr[L]; x < g.slot_ptr[L + 1]; ++x) {
                int64_t a = 1, t = 0, q = ac[x] != 0 ? nn[x] : 0, d = 1;
                for (int k = 0; k < nn[x]; ++k) {
                    const int64_t c = rowslot[(size_t)cb[x] + k];
                    if (c >= 0) { a += snn[c]; t += snt[c]; q += snp[c]; d = std::max(d, 1 + sdep[c]); } else ++t;
                }
                snn[x] = a;
                snt[x] = t;
                snp[x] = q;
                sdep[x] = d;
            }
        auto bytes_of = [&](int64_t x, bool staged) {
            return staged ? sub_smem(snn[x], snt[x], snn[x] - 1 + snt[x], snp[x], (int)sdep[x], P, Pc, w).total
                          : sub_smem(snn[x], snt[x], 0, 0, -1, P, Pc, w).total;
        };
        int forced_cut = -1;
        if (const char* e = std::getenv("CFR_SUB_CUT")) forced_cut = std::atoi(e);
        int forced_staged = -1;
        if (const char* e = std::getenv("CFR_SUB_STAGED")) forced_staged = std::atoi(e);
        // per layout: the shallowest cut whose subtrees fit one CTA and give >=
        // kSubMinCTAs CTAs (else the fitting cut with the most subtrees)
        auto pick = [&](bool staged, long long* need_out) {
            int cut = -1;
            int64_t best_n = -1;
            for (int c = 1; c < g.D; ++c) {
                const int64_t n = g.slot_ptr[c + 1] - g.slot_ptr[c];
                if (n <= 0 || n > kSubMaxSub || (forced_cut >= 0 && c != forced_cut)) continue;
                long long mx = 0;
                for (int64_t x = g.slot_ptr[c]; x < g.slot_ptr[c + 1]; ++x) mx = std::max(mx, bytes_of(x, staged));
                if (mx > budget) continue;
                if (n > best_n) {
                    cut = c;
                    *need_out = mx;
                    best_n = n;
                }
                if (n >= kSubMinCTAs) break;
            }
            return cut;
        };
        long long need_s = 0, need_g = 0;
        const int cut_s = pick(true, &need_s), cut_g = pick(false, &need_g);
        // staged tables unless they need a deeper cut (more trunk launches, e.g.
        // liar's dice in f64, whose per-deal bid trees are large and skewed)
        bool staged = cut_s >= 0 && (cut_g < 0 || cut_s <= cut_g);
        if (forced_staged >= 0) staged = forced_staged != 0 && cut_s >= 0;
        const int cut = staged ? cut_s : cut_g;
        const long long need = staged ? need_s : need_g;
        if (cut < 0) return CFR_OK;
        // infosets below the cut are one id range [hc, H)
        int64_t hc = g.H;
        for (int64_t x = g.slot_ptr[cut]; x < NS; ++x)
            if (sh[x] >= 0) hc = std::min(hc, sh[x]);
        for (int64_t x = 0; x < g.slot_ptr[cut]; ++x)
            if (sh[x] >= hc) return CFR_OK;
        // deferred infosets (member groups split across tiles) are fine below the cut
        // -- every infoset there is accumulated globally and updated by k_sub_update --
        // but not in the trunk, whose level kernels update in-tile
        for (const int64_t h : g.deferred_list)
            if (h < hc) return CFR_OK;
        // tables
        SubPlan sp{};
        sp.cut = cut;
        sp.staged = staged ? 1 : 0;
        sp.nsub = (int)(g.slot_ptr[cut + 1] - g.slot_ptr[cut]);
        sp.hc = hc;
        sp.qc = g.qbase_int[hc];
        sp.nh = g.H - hc;
        sp.nq = g.Q - sp.qc;
        sp.bytes = (int)std::max<long long>(need, 16);
        std::vector<int> meta, recs, chl, prs, lvl;
        std::vector<R> tu;
        meta.reserve((size_t)kSubMeta * sp.nsub);
        std::vector<int64_t> cur, nxt;
        int64_t maxw = 32;   // widest level step (nodes or pairs) of any subtree: the CTA size
        for (int64_t root = g.slot_ptr[cut]; root < g.slot_ptr[cut + 1]; ++root) {
            const int64_t node0 = (int64_t)recs.size() / kSubRec, term0 = (int64_t)tu.size() / Pc;
            const int64_t lvl0 = (int64_t)lvl.size(), child0 = (int64_t)chl.size(), pair0 = (int64_t)prs.size() / 4;
            std::vector<int> lstart, pstart;
            cur.assign(1, root);
            std::vector<int> curpar(1, -1), curin(1, 0);
            int64_t nloc = 0, nterm = 0;
            while (!cur.empty()) {
                lstart.push_back((int)nloc);
                pstart.push_back((int)(prs.size() / 4 - pair0));
                const int64_t p_before = (int64_t)prs.size() / 4;
                nxt.clear();
                std::vector<int> nxtpar, nxtin;
                const int64_t base = nloc;
                for (size_t k = 0; k < cur.size(); ++k) {
                    const int64_t x = cur[k];
                    const int j = (int)(base + (int64_t)k);
                    const int cp = (int)((int64_t)chl.size() - child0);
                    for (int a = 0; a < nn[x]; ++a) {
                        const int64_t row = (int64_t)cb[x] + a;
                        const int64_t c = rowslot[(size_t)row];
                        if (c >= 0) {
                            nxtin.push_back((int)((int64_t)chl.size() - child0));
                            chl.push_back((int)(base + (int64_t)cur.size() + (int64_t)nxt.size()));
                            nxt.push_back(c);
                            nxtpar.push_back(j);
                        } else {
                            chl.push_back((int)(-1 - nterm));
                            for (int q = 0; q < Pc; ++q) tu.push_back(U[(size_t)(row * Pc + q)]);
                            ++nterm;
                        }
                        if (ac[x] != 0) {   // int4: node << 8 | action, child ref, pair index q, actor
                            prs.push_back((j << 8) | a);
                            prs.push_back(chl.back());
                            prs.push_back((int)(eb[x] + a));
                            prs.push_back((int)ac[x]);
                        }
                    }
                    recs.push_back(curpar[k]);
                    recs.push_back(curin[k]);
                    recs.push_back((int)pa[x] | ((int)ac[x] << 8));
                    recs.push_back((int)fe[x]);
                    recs.push_back((int)eb[x]);
                    recs.push_back(nn[x]);
                    recs.push_back(cp);
                    recs.push_back((int)sh[x]);
                }
                maxw = std::max<int64_t>(maxw, std::max<int64_t>((int64_t)cur.size(), (int64_t)prs.size() / 4 - p_before));
                nloc += (int64_t)cur.size();
                cur.swap(nxt);
                curpar.swap(nxtpar);
                curin.swap(nxtin);
            }
            const int nlev = (int)lstart.size();
            lstart.push_back((int)nloc);
            pstart.push_back((int)(prs.size() / 4 - pair0));
            for (int v : lstart) lvl.push_back(v);
            const int64_t plv0 = (int64_t)lvl.size();
            for (int v : pstart) lvl.push_back(v);
            meta.push_back((int)node0);
            meta.push_back((int)nloc);
            meta.push_back((int)term0);
            meta.push_back((int)nterm);
            meta.push_back((int)lvl0);
            meta.push_back(nlev);
            meta.push_back((int)plv0);
            meta.push_back((int)root);
            meta.push_back((int)child0);
            meta.push_back((int)((int64_t)chl.size() - child0));
            meta.push_back((int)pair0);
            meta.push_back((int)((int64_t)prs.size() / 4 - pair0));
            if (nloc != snn[root] || nterm != snt[root] || (int64_t)prs.size() / 4 - pair0 != snp[root] || nlev != sdep[root] ||
                nloc >= (1 << 23))
                return CFR_OK;
        }
        sp.threads = (int)std::min<int64_t>(kSubThreads, (maxw + 31) / 32 * 32);
        // sections start on 16-byte boundaries (int4 copies of records and pairs)
        auto pad4 = [](std::vector<int>& v) { while (v.size() % 4) v.push_back(0); };
        pad4(meta);
        pad4(recs);
        pad4(chl);
        if (chl.size() - (size_t)0 > (size_t)INT32_MAX) return CFR_OK;
        // chance-only trunk (every slot above the cut a chance node): each root's
        // sigma_ext path top-down, and the trunk slots for k_sub_update's last CTA
        std::vector<int> path, trunk;
        {
            bool chance_trunk = P <= 8 && cut <= 16 && g.slot_ptr[cut] <= 65536;
            for (int64_t x = 0; x < g.slot_ptr[cut] && chance_trunk; ++x) chance_trunk = ac[x] == 0;
            if (const char* e = std::getenv("CFR_SUB_TRUNK"))
                if (std::atoi(e) == 0) chance_trunk = false;
            if (chance_trunk) {
                for (int64_t root = g.slot_ptr[cut]; root < g.slot_ptr[cut + 1] && chance_trunk; ++root) {
                    std::vector<int> up;
                    int64_t x = root;
                    for (int k = 0; k < cut; ++k) {
                        if (x <= 0 || lev[x] != cut - k) { chance_trunk = false; break; }
                        up.push_back((int)fe[x]);
                        x = (int64_t)fpar[x];
                    }
                    if (x != 0) chance_trunk = false;
                    for (int k = cut - 1; k >= 0 && chance_trunk; --k) path.push_back(up[k]);
                }
                for (int64_t x = 0; x < g.slot_ptr[cut] && chance_trunk; ++x) {
                    trunk.push_back((int)nd[x]);
                    trunk.push_back((int)cb[x]);
                    trunk.push_back((int)eb[x]);
                    trunk.push_back(nn[x] | (lev[x] << 16));
                }
            }
            sp.trunk = chance_trunk ? 1 : 0;
            if (!chance_trunk) {
                path.clear();
                trunk.clear();
            }
        }
        pad4(lvl);
        pad4(path);
        sp.m_sub = 0;
        sp.m_rec = (int)meta.size();
        sp.m_child = (int)(sp.m_rec + recs.size());
        sp.m_pair = (int)(sp.m_child + chl.size());
        sp.m_lvl = (int)(sp.m_pair + prs.size());
        sp.m_path = (int)(sp.m_lvl + lvl.size());
        sp.m_trunk = (int)(sp.m_path + path.size());
        sp.ntrunk = (int)(trunk.size() / 4);
        const size_t total = (size_t)sp.m_trunk + trunk.size();
        if (total > sub_table_bound(g) || tu.size() > (size_t)g.V * Pc + 2) return CFR_OK;
        std::vector<int> tab;
        tab.reserve(total);
        tab.insert(tab.end(), meta.begin(), meta.end());
        tab.insert(tab.end(), recs.begin(), recs.end());
        tab.insert(tab.end(), chl.begin(), chl.end());
        tab.insert(tab.end(), prs.begin(), prs.end());
        tab.insert(tab.end(), lvl.begin(), lvl.end());
        tab.insert(tab.end(), path.begin(), path.end());
        tab.insert(tab.end(), trunk.begin(), trunk.end());
        cfr_status st = up(plan.subt, tab);
        if (st) return st;
        if ((st = up(plan.subu, tu))) return st;
        CU(cudaMemsetAsync(ws + plan.suba, 0, (size_t)3 * (sp.nq + sp.nh) * sizeof(unsigned long long), stream));
        CU(cudaFuncSetAttribute(sub_fn(sp.staged != 0), cudaFuncAttributeMaxDynamicSharedMemorySize, sp.bytes));
        CU(cudaStreamSynchronize(stream));
        sub_plan_ = sp;
        sub_ = true;
        return CFR_OK;
    }
    int64_t count_launches() const {
        const Game& g = *gp;
        int64_t n = 0;
        if (sub_ && sub_plan_.trunk) return (cfg.variant == CFR_PLUS_ALT) ? 2 * g.P : 2;
        if (sub_) {
            for (int l = 1; l <= sub_plan_.cut; ++l)
                if (g.slot_ptr[l + 1] > g.slot_ptr[l]) ++n;
            n += 2;   // k_sub, k_sub_update
            for (int L = sub_plan_.cut - 1; L >= 0; --L)
                if (g.tile_ptr[L + 1] > g.tile_ptr[L]) ++n;
            return (cfg.variant == CFR_PLUS_ALT) ? n * g.P : n;
        }
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
        // no programmatic (PDL) edge when an NCCL all-reduce precedes it (sharded)
        launch(pdl_ && world == 1, k_deferred<R, I>, dim3(blocks), dim3(256), 0, st, dg, last);
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

    void launch_sub(cudaStream_t st, std::vector<Mark>* ev) {
        const Game& g = *gp;
        const SubPlan sp = sub_plan_;
        if (!sp.trunk)
            for (int l = 1; l <= sp.cut; ++l) {
                fwd_level(st, dg.sig, l, 0);
                mark(st, ev, 0, l);
            }
        const int* tab = at<int>(plan.subt);
        const R* tu = at<R>(plan.subu);
        unsigned long long* acc = at<unsigned long long>(plan.suba);
#define CFRB_SUB(PC)                                                                                               \
    (sp.staged ? launch(pdl_, k_sub<R, I, PC, true>, dim3(sp.nsub), dim3(sp.threads), (size_t)sp.bytes, st, dg, tab, tu, acc, sp) \
               : launch(pdl_, k_sub<R, I, PC, false>, dim3(sp.nsub), dim3(sp.threads), (size_t)sp.bytes, st, dg, tab, tu, acc, sp))
        switch (g.Pc) {
            case 1: CFRB_SUB(1); break;
            case 2: CFRB_SUB(2); break;
            case 3: CFRB_SUB(3); break;
            default: CFRB_SUB(4); break;
        }
#undef CFRB_SUB
        const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((sp.nh + 255) / 256, 4LL * num_sms_));
        const int last = (sp.trunk && pass_final_) ? 1 : 0;
        switch (g.Pc) {
            case 1: launch(pdl_, k_sub_update<R, I, 1>, dim3(nb), dim3(256), 0, st, dg, acc, sp, tab, last); break;
            case 2: launch(pdl_, k_sub_update<R, I, 2>, dim3(nb), dim3(256), 0, st, dg, acc, sp, tab, last); break;
            case 3: launch(pdl_, k_sub_update<R, I, 3>, dim3(nb), dim3(256), 0, st, dg, acc, sp, tab, last); break;
            default: launch(pdl_, k_sub_update<R, I, 4>, dim3(nb), dim3(256), 0, st, dg, acc, sp, tab, last); break;
        }
        mark(st, ev, 1, sp.cut);
        if (sp.trunk) return;   // the trunk's values and the iteration count: k_sub_update's last CTA
        for (int L = sp.cut - 1; L >= 0; --L) {
            bwd_level<MODE_CFR>(st, dg.sig, L, 0, (L == 0 && pass_final_) ? 1 : 0);
            mark(st, ev, 1, L);
        }
    }

    // mode MODE_CFR (forward + backward), MODE_VALUES (values under sig) or
    // MODE_BR (best-response values of player br_player; reach of sig computed before)
    void launch_lower(cudaStream_t st, int mode, const R* sig, std::vector<Mark>* ev, int br_player = 0) {
        const Game& g = *gp;
        if (mode == MODE_CFR && sig == dg.sig && sub_) {
            launch_sub(st, ev);
            return;
        }
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
            else if (mode == MODE_VALUES) bwd_level<MODE_VALUES>(st, sig, L, 0, 0);
            else bwd_level<MODE_BR>(st, sig, L, br_player, 0);
            mark(st, ev, 1, L);
            if (mode == MODE_CFR && overlap_exchange()) xchg_level(st, L);
        }
        if (sharded()) {
            const long long n = ncut();
            const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148));
            k_cut_pack<R><<<nb, 256, 0, st>>>(dg.U, at<long long>(plan.cutrow), at<unsigned char>(plan.cutown),
                                              at<R>(plan.cutbuf), n, g.Pc);
        }
    }
    // exchange 2 of the infosets first seen at level L on the communication
    // stream, forked from `st` after level L's backward kernel (NCCL issues the
    // per-level calls in the same order on every rank: the level schedule is
    // identical).  Returns the NCCL status through xstatus_.
    cfr_status xstatus_ = CFR_OK;
    int xforks_ = 0;
    bool overlap_exchange() const { return comm && xstream_ && world > 1 && has_def(); }
    void xchg_level(cudaStream_t st, int L) {
        const int64_t d0 = xr_[L].first, d1 = xr_[L].second;
        if (d1 <= d0) return;
        cudaEvent_t e = xev_[xforks_++ % xev_.size()];
        cudaEventRecord(e, st);
        cudaStreamWaitEvent(xstream_, e, 0);
        const int64_t q0 = gp->dqbase[d0], q1 = gp->dqbase[d1];
        cfr_status s = nccl_sum(xstream_, dg.acc_r + 3 * q0, (size_t)(3 * (q1 - q0)), ncclInt64);
        if (!s) s = nccl_sum(xstream_, dg.acc_p + 3 * d0, (size_t)(3 * (d1 - d0)), ncclInt64);
        if (s && !xstatus_) xstatus_ = s;
    }
    // join: `st` waits for every exchange issued on the communication stream
    void xchg_join(cudaStream_t st) {
        cudaEvent_t e = xev_.back();
        cudaEventRecord(e, xstream_);
        cudaStreamWaitEvent(st, e, 0);
    }
    void launch_upper(cudaStream_t st, int mode, const R* sig, std::vector<Mark>* ev, int br_player = 0) {
        const Game& g = *gp;
        if (!sharded()) return;
        const long long n = ncut();
        const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148));
        k_cut_unpack<R><<<nb, 256, 0, st>>>(dg.U, at<long long>(plan.cutrow), at<R>(plan.cutbuf), n, g.Pc);
        for (int L = sh->cut - 1; L >= 0; --L) {
            const int last = (mode == MODE_CFR && L == 0 && !has_def() && pass_final_) ? 1 : 0;
            if (mode == MODE_CFR) bwd_level<MODE_CFR>(st, sig, L, 0, last);
            else if (mode == MODE_VALUES) bwd_level<MODE_VALUES>(st, sig, L, 0, 0);
            else bwd_level<MODE_BR>(st, sig, L, br_player, 0);
            mark(st, ev, 1, L);
            if (mode == MODE_CFR && overlap_exchange()) xchg_level(st, L);
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
        xstatus_ = CFR_OK;
        mark(st, ev, -1, 0);
        for (int pass = 1; pass <= passes && !s; ++pass) {
            dg.upd_player = (passes > 1) ? pass : 0;
            pass_final_ = (pass == passes) ? 1 : 0;
            launch_lower(st, MODE_CFR, dg.sig, ev);
            if (sharded()) {
                if (overlap_exchange()) {
                    // every NCCL call of the iteration goes through the one
                    // communication stream, in issue order (no two collectives of
                    // the communicator in flight on different streams)
                    cudaEvent_t e = xev_[xforks_++ % xev_.size()];
                    cudaEventRecord(e, st);
                    cudaStreamWaitEvent(xstream_, e, 0);
                    if ((s = nccl_sum(xstream_, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype()))) break;
                    xchg_join(st);
                } else if ((s = nccl_sum(st, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype()))) {
                    break;
                }
                mark(st, ev, 3, -1);
                launch_upper(st, MODE_CFR, dg.sig, ev);
            }
            if (world > 1 && has_def()) {
                if (overlap_exchange()) {
                    // the per-level exchanges ran on the communication stream
                    if ((s = xstatus_)) break;
                    xchg_join(st);
                } else if ((s = nccl_sum(st, dg.acc_r, acc_bytes() / 8, ncclInt64))) {
                    break;
                }
                mark(st, ev, 3, -1);
            }
            if (!sub_) launch_update(st, ev);   // subtree mode: every deferred infoset is below the cut (k_sub_update)
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

    cfr_status compute_average(cudaStream_t st = nullptr) {
        const Game& g = *gp;
        const long long n = std::max<long long>(g.H, g.C);
        const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8));
        k_average<R, I><<<blocks, 256, 0, st ? st : stream>>>(dg, at<R>(plan.sig_eval), g.H, g.Q, g.C);
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

    // Resume (checkpoint restore): T iterations done, R, S_num (caller (h, a)
    // order), S_den (caller infoset order).  The current strategy is the regret
    // matching of R (Eq 9, z summed in ascending action order, uniform when z = 0)
    // -- what every update rule leaves after its iteration -- computed here with
    // the kernels' operations, so a restored solver continues bit for bit.
    cfr_status set_state(int64_t T, const double* regret, const double* snum, const double* sden) override {
        const Game& g = *gp;
        CU(cudaStreamSynchronize(stream));
        std::vector<R> r(g.Q), sn(g.Q), sd(g.H), sg(g.Q);
        for (int64_t hc = 0; hc < g.H; ++hc) {
            const int64_t hi = g.h_int_of_caller[hc];
            const int64_t n = g.qbase_caller[hc + 1] - g.qbase_caller[hc];
            for (int64_t a = 0; a < n; ++a) {
                r[g.qbase_int[hi] + a] = (R)regret[g.qbase_caller[hc] + a];
                sn[g.qbase_int[hi] + a] = (R)snum[g.qbase_caller[hc] + a];
            }
            sd[hi] = (R)sden[hc];
        }
        for (int64_t h = 0; h < g.H; ++h) {
            const int64_t q0 = g.qbase_int[h], q1 = g.qbase_int[h + 1];
            R z = (R)0;
            for (int64_t q = q0; q < q1; ++q) z = z + ((r[q] > (R)0) ? r[q] : (R)0);
            for (int64_t q = q0; q < q1; ++q) {
                const R pos = (r[q] > (R)0) ? r[q] : (R)0;
                sg[q] = (z > (R)0) ? pos / z : (R)1 / (R)(q1 - q0);
            }
        }
        cfr_status st;
        if ((st = up(plan.regret, r))) return st;
        if ((st = up(plan.snum, sn))) return st;
        if ((st = up(plan.sden, sd))) return st;
        if (g.Q) CU(cudaMemcpyAsync(ws + plan.sig, sg.data(), g.Q * sizeof(R), cudaMemcpyHostToDevice, stream));
        std::vector<long long> ctrl = {(long long)T, LLONG_MAX, 0, 0, 0, 0, 0, 0};
        if ((st = up(plan.ctrl, ctrl))) return st;
        CU(cudaStreamSynchronize(stream));
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

    // ---- best response (reading Q11 / Q17) ------------------------------------
    // BR_i under sig: MODE_BR backward passes (+ the cut exchange when sharded).
    // Infosets complete in one tile decide in-tile, bottom-up, in the same pass.
    // A deferred infoset (its members span tiles, depths or ranks) sums its
    // exact BR terms globally; k_br_decide (after the int64 exchange when
    // sharded) sets its action, which its members use from the next pass on.
    // Under perfect recall the deferred infosets below a member of h have
    // strictly longer own-action sequences than h, so after pass k every
    // deferred infoset whose chain of deferred infosets below is shorter than k
    // has its final action; sequences are at most D long, so D passes decide all
    // and one more pass leaves BR_i at the root (1 pass without deferred infosets).
    int br_passes() const { return (world > 1 || has_def()) ? full->D + 1 : 1; }
    cfr_status br_decide(cudaStream_t st, int i) {
        const long long n = dg.ndef;
        if (n == 0) return CFR_OK;
        if (world > 1) {
            cfr_status s = nccl_sum(st, dg.acc_r, acc_bytes() / 8, ncclInt64);
            if (s) return s;
        }
        const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8));
        k_br_decide<R, I><<<blocks, 256, 0, st>>>(dg, i, (gp->Pc == 1 && i == 2) ? 1 : 0);
        CU(cudaGetLastError());
        return CFR_OK;
    }
    cfr_status br_pass(cudaStream_t st, const R* sig, int i) {
        const Game& g = *gp;
        launch_lower(st, MODE_BR, sig, nullptr, i);
        if (sharded()) {
            cfr_status s = nccl_sum(st, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype());
            if (s) return s;
            launch_upper(st, MODE_BR, sig, nullptr, i);
        }
        return br_decide(st, i);
    }
    // sigma_bar into sig_eval and its forward pass (reach of every level)
    cfr_status eval_setup(cudaStream_t st) {
        const Game& g = *gp;
        cfr_status s = compute_average(st);
        if (s) return s;
        const R* sig = at<R>(plan.sig_eval);
        for (int l = 1; l < g.D; ++l) fwd_level(st, sig, l);
        CU(cudaGetLastError());
        return CFR_OK;
    }
    // root row -> per-player values (u2 = -u1 storage for two-player zero-sum)
    void root_to_players(const R* r, double* out) const {
        const Game& g = *gp;
        if (g.zero_sum_2p) {
            out[0] = (double)r[0];
            out[1] = (double)(-r[0]);
        } else {
            for (int j = 0; j < g.P; ++j) out[j] = (double)r[j];
        }
    }

    cfr_status exploitability(double* nc, double* ex, double* br) override {
        const Game& g = *gp;
        if (external) {
            cfrb_set_error("world_size > 1 without an NCCL id: drive the best response with cfr_solver_br_phase");
            return CFR_ERR_UNSUPPORTED;
        }
        CU(cudaStreamSynchronize(stream));
        cfr_status s;
        double ev[16];
        {
            if ((s = compute_average())) return s;
            if ((s = root_values(at<R>(plan.sig_eval), ev))) return s;
        }
        if ((s = eval_setup(stream))) return s;
        const R* sig = at<R>(plan.sig_eval);
        double total = 0.0;
        const int passes = br_passes();
        for (int i = 1; i <= g.P; ++i) {
            for (int k = 0; k < passes; ++k)
                if ((s = br_pass(stream, sig, i))) return s;
            std::vector<R> r(g.Pc);
            CU(cudaMemcpyAsync(r.data(), dg.U, g.Pc * sizeof(R), cudaMemcpyDeviceToHost, stream));
            CU(cudaStreamSynchronize(stream));
            double v[16];
            root_to_players(r.data(), v);
            const double b = v[i - 1];
            if (br) br[i - 1] = b;
            total = total + (b - ev[i - 1]);
        }
        // the reach arrays of the current strategy need no restoring: every
        // iteration recomputes them (root reach stays 1)
        *nc = total;
        *ex = total / (double)g.P;
        return CFR_OK;
    }

    // externally driven sharded best response (tests; world > 1 without NCCL):
    // 0 setup (sigma_bar + its forward pass), 1 lower pass, 2 upper pass (caller
    // exchanged the cut values), 3 decide (caller exchanged the int64 sums; `out`
    // receives the root values of this pass)
    cfr_status br_phase(int ph, int i, double* out) override {
        const Game& g = *gp;
        if (i < 1 || i > g.P) {
            cfrb_set_error("bad best-response player");
            return CFR_ERR_INVALID_ARG;
        }
        const R* sig = at<R>(plan.sig_eval);
        cfr_status s = CFR_OK;
        switch (ph) {
            case 0: s = eval_setup(stream); break;
            case 1: launch_lower(stream, MODE_BR, sig, nullptr, i); break;
            case 2: launch_upper(stream, MODE_BR, sig, nullptr, i); break;
            case 3: {
                if (dg.ndef > 0) {
                    const unsigned blocks = (unsigned)std::max<long long>(
                        1, std::min<long long>((dg.ndef + 255) / 256, 148LL * 8));
                    k_br_decide<R, I><<<blocks, 256, 0, stream>>>(dg, i, (g.Pc == 1 && i == 2) ? 1 : 0);
                }
                if (out) {
                    CU(cudaGetLastError());
                    std::vector<R> r(g.Pc);
                    CU(cudaMemcpyAsync(r.data(), dg.U, g.Pc * sizeof(R), cudaMemcpyDeviceToHost, stream));
                    CU(cudaStreamSynchronize(stream));
                    root_to_players(r.data(), out);
                }
                break;
            }
            default:
                cfrb_set_error("bad best-response phase");
                return CFR_ERR_INVALID_ARG;
        }
        if (s) return s;
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(stream));
        return CFR_OK;
    }
    cfr_status br_passes_out(int32_t* n) override {
        *n = br_passes();
        return CFR_OK;
    }

    // ---- in-graph exploitability (Fig 3) -------------------
    // One evaluation = sigma_bar, its forward pass, the values pass (EV) and every
    // player's best-response passes, each root row stored on the device into the
    // record (k_root_store): captured once as a CUDA graph and replayed every
    // `every` iterations with no host synchronisation; rows are read back when
    // the record fills up and at the end.
    cudaGraphExec_t eval_exec_ = nullptr;
    cfr_status eval_enqueue(cudaStream_t st) {
        const Game& g = *gp;
        const int width = rec_width(g);
        double* rec = at<double>(plan.rec);
        const R* sig = at<R>(plan.sig_eval);
        cfr_status s;
        if ((s = compute_average(st))) return s;
        launch_lower(st, MODE_VALUES, sig, nullptr);
        if (sharded()) {
            if ((s = nccl_sum(st, at<R>(plan.cutbuf), (size_t)ncut() * g.Pc, rtype()))) return s;
            launch_upper(st, MODE_VALUES, sig, nullptr);
        }
        k_root_store<R><<<1, 32, 0, st>>>(dg.U, rec, dg.ctrl, g.Pc, 0, width, 0, kRecRows);
        for (int l = 1; l < g.D; ++l) fwd_level(st, sig, l);
        const int passes = br_passes();
        for (int i = 1; i <= g.P; ++i) {
            for (int k = 0; k < passes; ++k)
                if ((s = br_pass(st, sig, i))) return s;
            k_root_store<R><<<1, 32, 0, st>>>(dg.U, rec, dg.ctrl, g.Pc, g.Pc * i, width, i == g.P ? 1 : 0, kRecRows);
        }
        CU(cudaGetLastError());
        return CFR_OK;
    }
    cfr_status flush_record(int64_t rows, double* out, int64_t* written) {
        const Game& g = *gp;
        const int width = rec_width(g);
        std::vector<double> buf((size_t)rows * width);
        CU(cudaStreamSynchronize(stream));
        if (rows) CU(cudaMemcpy(buf.data(), at<double>(plan.rec), buf.size() * sizeof(double), cudaMemcpyDeviceToHost));
        long long zero = 0;
        CU(cudaMemcpy(dg.ctrl + 4, &zero, sizeof(zero), cudaMemcpyHostToDevice));
        const int ow = 2 + 2 * g.P;   // out row: T, NashConv, EV_1..P, BR_1..P
        for (int64_t r = 0; r < rows; ++r) {
            const double* row = buf.data() + (size_t)r * width;
            double* o = out + (size_t)(*written + r) * ow;
            std::vector<R> tmp(g.Pc);
            for (int j = 0; j < g.Pc; ++j) tmp[j] = (R)row[j];
            root_to_players(tmp.data(), o + 2);
            double nc = 0.0;
            for (int i = 1; i <= g.P; ++i) {
                for (int j = 0; j < g.Pc; ++j) tmp[j] = (R)row[g.Pc * i + j];
                double v[16];
                root_to_players(tmp.data(), v);
                o[2 + g.P + (i - 1)] = v[i - 1];
                nc = nc + (v[i - 1] - o[2 + (i - 1)]);
            }
            o[0] = row[width - 1];
            o[1] = nc;
        }
        *written += rows;
        return CFR_OK;
    }
    cfr_status run_tracked(int64_t iters, int64_t every, double* out, int64_t* rows_out) override {
        if (external) {
            cfrb_set_error("world_size > 1 without an NCCL id: tracked runs need the in-graph exchanges");
            return CFR_ERR_UNSUPPORTED;
        }
        if (every <= 0 || iters < 0) {
            cfrb_set_error("run_tracked: every must be > 0 and iterations >= 0");
            return CFR_ERR_INVALID_ARG;
        }
        CU(cudaStreamSynchronize(stream));
        if (!eval_exec_ && use_graph) {
            cudaStream_t cs = cap_stream;
            if (!cs) CU(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
            cudaGraph_t graph;
            CU(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
            cfr_status ls = eval_enqueue(cap_stream);
            cudaError_t ce = cudaStreamEndCapture(cap_stream, &graph);
            if (ls != CFR_OK) return ls;
            if (ce != cudaSuccess) {
                cfrb_set_error(std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
                return CFR_ERR_CUDA;
            }
            CU(cudaGraphInstantiate(&eval_exec_, graph, 0));
            cudaGraphDestroy(graph);
        }
        long long zero = 0;
        CU(cudaMemcpy(dg.ctrl + 4, &zero, sizeof(zero), cudaMemcpyHostToDevice));
        int64_t written = 0, pending = 0;
        for (int64_t done = 0; done + every <= iters; done += every) {
            cfr_status s = enqueue(every);
            if (s) return s;
            if (eval_exec_) CU(cudaGraphLaunch(eval_exec_, stream));
            else if ((s = eval_enqueue(stream))) return s;
            if (++pending == kRecRows) {
                if ((s = flush_record(pending, out, &written))) return s;
                pending = 0;
            }
        }
        const int64_t tail = iters % every;
        if (tail) {
            cfr_status s = enqueue(tail);
            if (s) return s;
        }
        cfr_status s = flush_record(pending, out, &written);
        if (s) return s;
        *rows_out = written;
        return sync();
    }

    cfr_status launches(int64_t* n) override {
        *n = tiny_ ? 1 : launches_per_iter;   // k_tiny: one launch per enqueue of T iterations
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
        if (sub_ && L >= sub_plan_.cut) return 4;
        if (use_stream_ && stream_[L].ntiles > 0) return 3;
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

static size_t bytes_for(const Game& g, const ShardInfo* sh, int precision, int flags) {
    const bool i32 = use_idx32(g) && !(flags & CFR_FLAG_INDEX64);
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
    *bytes = bytes_for(*local, info, cfg->precision, cfg->flags);
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
    const size_t need = bytes_for(*local, info, cfg->precision, cfg->flags);
    if (workspace_bytes < need) {
        cfrb_set_error("workspace too small: need " + std::to_string(need) + " bytes");
        return CFR_ERR_OOM;
    }
    if (((uintptr_t)workspace & 255) != 0) { cfrb_set_error("workspace must be 256-byte aligned"); return CFR_ERR_INVALID_ARG; }
    const bool i32 = use_idx32(*local) && !(cfg->flags & CFR_FLAG_INDEX64);
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
cfr_status cfr_solver_set_state(cfr_solver* s, int64_t T, const double* regret, const double* s_num,
                                const double* s_den) {
    CHK_S(s);
    if (T < 0 || !regret || !s_num || !s_den) { cfrb_set_error("bad argument"); return CFR_ERR_INVALID_ARG; }
    return s->impl->set_state(T, regret, s_num, s_den);
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
cfr_status cfr_solver_br_phase(cfr_solver* s, int32_t phase, int32_t player, double* out) {
    CHK_S(s);
    return s->impl->br_phase(phase, player, out);
}
cfr_status cfr_solver_br_passes(cfr_solver* s, int32_t* passes) {
    CHK_S(s);
    if (!passes) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->br_passes_out(passes);
}
cfr_status cfr_solver_run_tracked(cfr_solver* s, int64_t iterations, int64_t every, double* out, int64_t* rows) {
    CHK_S(s);
    if (!out || !rows) { cfrb_set_error("NULL out"); return CFR_ERR_INVALID_ARG; }
    return s->impl->run_tracked(iterations, every, out, rows);
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
