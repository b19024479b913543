// Deferred-infoset update (k_deferred), sigma_bar / multi-GPU exchange and readback-mask kernels.
// Part of the single translation unit solver.cu (included from it only).
#pragma once

namespace cfrb {

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


// Best response (reading Q11 / Q17): after a MODE_BR backward pass, every
// deferred infoset of the BR player (spanning tiles, depths or ranks) decodes its
// exact sums sum_{d in h} pi_check(d, i) V(child(d, a)) and takes the argmax
// (ties to the lowest action; with u2 = -u1 storage player 2 takes the argmin of
// the stored sums), compared in the working precision like the in-tile argmax.
// The accumulators of every deferred infoset are zeroed for the next pass.
template <class R, class I>
__global__ void __launch_bounds__(256) k_br_decide(DG<R, I> g, int br_player, int neg) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < g.ndef; idx += stride) {
        const long long h = (long long)g.deferred[idx];
        const long long qb = (long long)g.qbase[h];
        const int n = (int)((long long)g.qbase[h + 1] - qb);
        const long long dq = g.dqbase[idx];
        const bool mine = g.owner[h] == br_player;
        int best = 0;
        R bv = (R)0;
        for (int a = 0; a < n; ++a) {
            const long long cq = dq + a;
            const long long c0 = (long long)g.acc_r[cq * 3 + 0], c1 = (long long)g.acc_r[cq * 3 + 1],
                            c2 = (long long)g.acc_r[cq * 3 + 2];
            g.acc_r[cq * 3 + 0] = 0;
            g.acc_r[cq * 3 + 1] = 0;
            g.acc_r[cq * 3 + 2] = 0;
            const R x = (R)xdec_ll(c0, c1, c2, g.rc);
            if (a == 0 || (neg ? (x < bv) : (x > bv))) {
                bv = x;
                best = a;
            }
        }
        if (mine) g.br_best[idx] = best;
    }
}

// Root row of U (values of the last backward pass) into slot `slot` of the
// exploitability record `rec` (in-graph exploitability, cfr_solver_run_tracked):
// rec[row * width + slot + j] = U[j], row = ctrl[4]; `advance` closes the row
// (writes the iteration count into its last entry and moves to the next row).
template <class R>
__global__ void k_root_store(const R* __restrict__ U, double* __restrict__ rec, long long* ctrl, int Pc, int slot,
                             int width, int advance, long long cap) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const long long row = ctrl[4];
        if (row < cap) {
            double* r = rec + row * width;
            for (int j = 0; j < Pc; ++j) r[slot + j] = (double)U[j];
            if (advance) r[width - 1] = (double)ctrl[0];
        }
        if (advance) ctrl[4] = row + 1;
    }
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

}  // namespace cfrb
