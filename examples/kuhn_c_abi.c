/* A plain C caller of include/cfr_b200.h: Kuhn poker (Table 7, P:659:
 * 58 nodes, 12 infosets) built as Def. 2.1 arrays, flattened by the
 * library, and -- with the argument "gpu" -- solved with 1000 vanilla CFR
 * iterations in f64 on the current CUDA device (BASELINE.json configs[0]): the
 * value of the average strategy must be within 1e-4 of -1/18 and within its
 * NashConv (the 2-epsilon bound).
 *
 *   gcc -std=c99 -I include examples/kuhn_c_abi.c -L paper_2408_14778_b200 -lcfr_b200 \
 *       -I /usr/local/cuda/include -L /usr/local/cuda/lib64 -lcudart -o kuhn && ./kuhn gpu
 *
 * Without "gpu" only the host half runs (game creation, info, qbase, canonical
 * order), which needs no device. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "cfr_b200.h"

#define MAXV 64
static int64_t parent[MAXV], infoset[MAXV];
static int32_t player[MAXV], action[MAXV];
static double chance_prob[MAXV], utility[MAXV * 2];
static int V = 0;

static int node(int par, int act, double prob) {
    parent[V] = par;
    action[V] = act;
    chance_prob[V] = prob;
    player[V] = -1;
    infoset[V] = -1;
    utility[2 * V] = utility[2 * V + 1] = 0.0;
    return V++;
}
static void terminal(int v, double u1) {
    utility[2 * v] = u1;
    utility[2 * v + 1] = -u1;
}
/* infosets: P1 (card, "") = card, P1 (card, "pb") = 3 + card,
 *           P2 (card, "p") = 6 + card, P2 (card, "b") = 9 + card */
static void deal(int v, int c1, int c2) {
    const double win = c1 > c2 ? 1.0 : -1.0;
    player[v] = 1;
    infoset[v] = c1;
    const int p = node(v, 0, 0), b = node(v, 1, 0);
    player[p] = 2; infoset[p] = 6 + c2;      /* P2 after pass */
    player[b] = 2; infoset[b] = 9 + c2;      /* P2 after bet */
    terminal(node(p, 0, 0), win);            /* pass-pass: showdown for 1 */
    const int pb = node(p, 1, 0);            /* pass-bet */
    player[pb] = 1; infoset[pb] = 3 + c1;
    terminal(node(pb, 0, 0), -1.0);          /* P1 folds */
    terminal(node(pb, 1, 0), 2.0 * win);     /* P1 calls */
    terminal(node(b, 0, 0), 1.0);            /* P2 folds */
    terminal(node(b, 1, 0), 2.0 * win);      /* P2 calls */
}

#define CHECK(x)                                                                          \
    do {                                                                                  \
        cfr_status s_ = (x);                                                              \
        if (s_ != CFR_OK) {                                                               \
            fprintf(stderr, "%s failed: %s: %s\n", #x, cfr_status_string(s_), cfr_last_error()); \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

int main(int argc, char** argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    const int root = node(-1, -1, 0);
    player[root] = 0;
    for (int c1 = 0; c1 < 3; ++c1) {
        const int c = node(root, c1, 1.0 / 3.0);
        player[c] = 0;
        for (int k = 0, c2 = 0; c2 < 3; ++c2) {
            if (c2 == c1) continue;
            deal(node(c, k++, 0.5), c1, c2);
        }
    }
    cfr_game_desc d = {V, 2, parent, player, infoset, action, chance_prob, utility};
    cfr_game* g = NULL;
    CHECK(cfr_game_create(&d, &g));
    cfr_game_info_t info;
    CHECK(cfr_game_info(g, &info));
    printf("kuhn: V=%lld terminals=%lld decision=%lld chance=%lld infosets=%lld pairs=%lld depth=%d\n",
           (long long)info.num_nodes, (long long)info.num_terminals, (long long)info.num_decision,
           (long long)info.num_chance, (long long)info.num_infosets, (long long)info.num_pairs, info.depth);
    if (info.num_nodes != 58 || info.num_terminals != 30 || info.num_chance != 4 || info.num_infosets != 12 ||
        info.num_pairs != 24 || !info.zero_sum_2p) {
        fprintf(stderr, "unexpected Kuhn dimensions (PAPER.md Table 7)\n");
        return 1;
    }
    int64_t qbase[13], canon[MAXV], level_ptr[16];
    CHECK(cfr_game_qbase(g, qbase));
    CHECK(cfr_game_canonical(g, canon, level_ptr));
    if (qbase[12] != 24 || canon[root] != 0 || level_ptr[info.depth + 1] != 58) {
        fprintf(stderr, "bad qbase / canonical order\n");
        return 1;
    }
    if (!gpu) {
        cfr_game_destroy(g);
        printf("host half ok\n");
        return 0;
    }

    cfr_solver_config cfg = {CFR_VANILLA, 64, 0, 0};
    size_t bytes = 0;
    CHECK(cfr_solver_workspace_bytes(g, &cfg, NULL, &bytes));
    void* ws = NULL;
    cudaStream_t stream;
    if (cudaMalloc(&ws, bytes) != cudaSuccess || cudaStreamCreate(&stream) != cudaSuccess) {
        fprintf(stderr, "CUDA allocation failed\n");
        return 1;
    }
    cfr_solver* s = NULL;
    CHECK(cfr_solver_create(g, &cfg, ws, bytes, (void*)stream, NULL, &s));
    CHECK(cfr_solver_run(s, 1000));
    int64_t T = 0;
    double ev[2], nash_conv, expl, br[2], avg[24];
    CHECK(cfr_solver_iteration(s, &T));
    CHECK(cfr_solver_expected_values(s, 0, ev));
    CHECK(cfr_solver_exploitability(s, &nash_conv, &expl, br));
    CHECK(cfr_solver_average_strategy(s, avg));
    const double err = fabs(ev[0] + 1.0 / 18.0);
    printf("T=%lld EV(sigma_bar)=(%.9f, %.9f) |EV1 + 1/18|=%.3g NashConv=%.6g exploitability=%.6g\n",
           (long long)T, ev[0], ev[1], err, nash_conv, expl);
    for (int h = 0; h < 12; ++h) {
        const double z = avg[qbase[h]] + avg[qbase[h] + 1];
        if (fabs(z - 1.0) > 1e-12) {
            fprintf(stderr, "sigma_bar of infoset %d is not a distribution\n", h);
            return 1;
        }
    }
    cfr_solver_destroy(s);
    cfr_game_destroy(g);
    cudaFree(ws);
    cudaStreamDestroy(stream);
    if (T != 1000 || err > 1e-4 || err > nash_conv) {
        fprintf(stderr, "Kuhn value check failed\n");
        return 1;
    }
    printf("gpu half ok\n");
    return 0;
}
