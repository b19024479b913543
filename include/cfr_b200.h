/*
 * cfr_b200.h -- C ABI of the B200-native CFR / CFR+ iteration (arXiv 2408.14778).
 *
 * The library runs whole counterfactual-regret-minimization iterations
 * (§3.2: regret matching, level-by-level forward reach pass,
 * level-by-level backward value pass, per-infoset aggregation, regret and
 * average-strategy accumulation) as hand-written sm_100a CUDA kernels: per-level
 * kernels captured in a CUDA Graph (big levels through the TMA-streamed backward
 * kernel); for latency-bound games the levels below a cut as one subtree launch
 * plus one update launch (the subtree mode, CFR_FLAG_NO_SUBTREE); for games whose
 * state fits one CTA's shared memory, one single-CTA launch per enqueue.  Update rules: CFR, CFR+, linear CFR, DCFR and
 * alternating-update CFR+ (cfr_variant).  Everything below is plain C: host or device pointers and
 * sizes, no C++ or torch types.  No exception ever crosses this boundary; every
 * call returns a cfr_status and, on failure, leaves a message in
 * cfr_last_error() (thread-local).  A handle is not thread-safe; distinct
 * handles are independent.
 */
#ifndef CFR_B200_H
#define CFR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CFR_OK = 0,
    CFR_ERR_INVALID_ARG = 1,   /* NULL pointer, bad size, bad enum value            */
    CFR_ERR_INVALID_TREE = 2,  /* the game arrays violate Def. 2.1        */
    CFR_ERR_UNSUPPORTED = 3,   /* e.g. device best response on an infoset spanning
                                  several depths, or world_size > 1 without NCCL    */
    CFR_ERR_CUDA = 4,          /* a CUDA runtime call failed (message has the name) */
    CFR_ERR_NCCL = 5,          /* an NCCL call failed                               */
    CFR_ERR_OOM = 6,           /* workspace smaller than cfr_solver_workspace_bytes */
    CFR_ERR_NUMERICAL = 7      /* NaN/Inf in the regrets or strategy; message names
                                  the first failing iteration          */
} cfr_status;

/* Human-readable name of a status code (static storage). */
const char* cfr_status_string(cfr_status s);
/* Message of the last failing call on this thread ("" if none). */
const char* cfr_last_error(void);

/* ------------------------------------------------------------------ game --
 * A finite extensive-form game G = <T, H, f_h, A, f_a, I, f_i, sigma_0, u>
 * (Def. 2.1) as flat, caller-owned HOST arrays of V entries
 * each, in ANY node order (the library canonicalises: SURVEY.md Appendix B-1).
 *
 *   parent[v]      f_parents(v); -1 for the unique root v0.
 *   player[v]      -1 terminal (v in T); 0 chance (nature i0); 1..P player i+.
 *   infoset[v]     f_h(v) for player decision nodes, dense ids 0..H+-1 across all
 *                  players; ignored (use -1) at chance and terminal nodes
 *                  (reading Q13: sigma_0 is given per chance edge).
 *   action[v]      f_a(v) = index of the incoming action, -1 at the root.  For
 *                  every decision node d the children's actions are exactly
 *                  0..|S(d)|-1 (the bijection f_{a,d}: S(d) -> A(f_h(d))),
 *                  and |S(d)| = |A(h)| is shared by all nodes of an infoset.
 *   chance_prob[v] sigma_0 of the edge INTO v when parent(v) is a chance node
 *                  (P:35); ignored otherwise.  Each chance node's
 *                  children must sum to 1 within 1e-12.
 *   utility[v*P+i] u(v, i+1) at terminals, row-major [V][P]; ignored at
 *                  decision nodes; must be finite.
 *
 * The library copies what it needs: the caller may free the arrays as soon as
 * cfr_game_create returns.  Validation failures return CFR_ERR_INVALID_TREE
 * with a message naming the offending node or infoset.  Limits: 1 <= P <= 16;
 * at most 2^23 nodes per infoset (exact-accumulation headroom).
 */
typedef struct {
    int64_t num_nodes;          /* V >= 1                    */
    int32_t num_players;        /* P in [1, 16]              */
    const int64_t* parent;
    const int32_t* player;
    const int64_t* infoset;
    const int32_t* action;
    const double* chance_prob;
    const double* utility;      /* [V * P]                   */
} cfr_game_desc;

typedef struct cfr_game cfr_game;

typedef struct {
    int64_t num_nodes;          /* |V|                                           */
    int64_t num_terminals;      /* |T|                                           */
    int64_t num_decision;       /* |D| = chance + player decision nodes          */
    int64_t num_chance;         /* chance decision nodes                         */
    int64_t num_infosets;       /* |H+|                                          */
    int64_t num_pairs;          /* |Q+| = sum_h |A(h)|                           */
    int32_t num_players;        /* |I+|                                          */
    int32_t depth;              /* D = max terminal depth                */
    int64_t max_infoset_nodes;  /* largest infoset                               */
    int32_t depth_homogeneous;  /* 1 if every infoset lies on one depth          */
    int32_t zero_sum_2p;        /* 1 if P == 2 and u2 == -u1 bit-exactly (B-7)   */
} cfr_game_info_t;

cfr_status cfr_game_create(const cfr_game_desc* desc, cfr_game** out);
void cfr_game_destroy(cfr_game* g);
cfr_status cfr_game_info(const cfr_game* g, cfr_game_info_t* out);
/* qbase[h] = sum_{h' < h} |A(h')| over the CALLER's infoset ids, [H+ + 1]; the
 * (infoset, action) pair (h, a) is index qbase[h] + a in every strategy array. */
cfr_status cfr_game_qbase(const cfr_game* g, int64_t* qbase);
/* Canonical flattening (Appendix B-1): canon_of_input[V] maps each input node
 * to its canonical BFS index; level_ptr[D + 2] delimits the depth levels.
 * Either pointer may be NULL. */
cfr_status cfr_game_canonical(const cfr_game* g, int64_t* canon_of_input, int64_t* level_ptr);

/* ---------------------------------------------------------------- solver --
 * Solver state lives in ONE caller-allocated device workspace (e.g. a torch
 * uint8 tensor) that must stay allocated until cfr_solver_destroy.  All work is
 * enqueued on the caller's CUDA stream (cudaStream_t passed as void*; NULL =
 * legacy default stream).
 */
/* CFR_LINEAR (LCFR) and CFR_DISCOUNTED (DCFR with alpha = 3/2, beta = 0, gamma = 2)
 * apply Brown & Sandholm's discounting to Eq 14/15 (DESIGN.md reading
 * Q18): after iteration t, positive regrets x t^a/(t^a+1), the others x
 * t^b/(t^b+1), the average-strategy sums x (t/(t+1))^g; LCFR is a = b = g = 1. */
/* CFR_PLUS_ALT: CFR+ with alternating updates (Tammelin; reading Q19):
 * per iteration one full pass per player, each updating only that player's
 * infosets under the profile current at that point. */
typedef enum { CFR_VANILLA = 0, CFR_PLUS = 1, CFR_LINEAR = 2, CFR_DISCOUNTED = 3, CFR_PLUS_ALT = 4 } cfr_variant;

typedef struct {
    int32_t variant;     /* cfr_variant: CFR (w_t = 1), CFR+ (RM+, w_t = t), LCFR,   */
                         /* DCFR, CFR+ with alternating updates                    */
    int32_t precision;   /* 64 (binary64) or 32 (binary32) working precision      */
    int32_t flags;       /* bit 0: disable CUDA-Graph capture (debug);            */
                         /* bit 1: reserved -- the cooperative single-launch     */
                         /* kernel it selected was removed (slower than the PDL  */
                         /* graph on B200): CFR_ERR_UNSUPPORTED; bit 2: reserved */
                         /* (ignored: the pipelined cp.async backward kernel it  */
                         /* disabled was superseded by the streaming kernel and  */
                         /* removed); bit 3: disable                             */
                         /* programmatic dependent launch; bit 4: disable the     */
                         /* streaming (TMA) backward kernel (A/B comparisons);    */
                         /* bit 5: use the streaming kernel on every eligible     */
                         /* level, however small (tests); bit 6: fuse the         */
                         /* deepest level's forward pass into its streaming       */
                         /* backward kernel (experimental); bit 7: disable the    */
                         /* shared-memory single-CTA kernel of tiny games         */
                         /* (k_tiny, default when the state fits one CTA); bit 8: */
                         /* 64-bit device indices even when 32 bits suffice       */
                         /* (they are used automatically for >= 2^31 entries)     */
                         /* bit 9: disable the subtree kernel (k_sub: the levels  */
                         /* below a cut in one launch, subtree state in shared    */
                         /* memory, exact int64 infoset sums, */
                         /* DESIGN.md §6.3; default for single-GPU, depth-        */
                         /* homogeneous games of 2,048 - 2^22 nodes without       */
                         /* deferred infosets above the cut, and above 2^20 nodes */
                         /* only without streaming-size levels or with fewer than */
                         /* half the nodes terminal; flags 4/5/6/7/8 keep the     */
                         /* level kernels); bit 10: the subtree kernel whenever   */
                         /* a cut fits (also where k_tiny would run)              */
    int32_t reserved;
} cfr_solver_config;

#define CFR_FLAG_NO_GRAPH 1
#define CFR_FLAG_PERSISTENT 2   /* reserved: rejected with CFR_ERR_UNSUPPORTED */
#define CFR_FLAG_NO_PIPELINE 4   /* reserved: ignored */
#define CFR_FLAG_NO_PDL 8
#define CFR_FLAG_NO_STREAM 16
#define CFR_FLAG_FORCE_STREAM 32
#define CFR_FLAG_FUSED_FORWARD 64
#define CFR_FLAG_NO_TINY 128
#define CFR_FLAG_INDEX64 256
#define CFR_FLAG_NO_SUBTREE 512   /* do not use the subtree kernel (k_sub) */
#define CFR_FLAG_FORCE_SUBTREE 1024   /* subtree kernel even where k_tiny fits */

/* Multi-GPU level sharding.  NULL or world_size == 1 means a
 * single GPU.  nccl_unique_id points to the 128-byte ncclUniqueId that rank 0
 * created (cfr_nccl_unique_id) and the caller broadcast (e.g. torch.distributed). */
typedef struct {
    int32_t rank;
    int32_t world_size;
    const void* nccl_unique_id;
} cfr_dist;

typedef struct cfr_solver cfr_solver;

/* Bytes of device workspace the solver needs on this rank. */
cfr_status cfr_solver_workspace_bytes(const cfr_game* g, const cfr_solver_config* cfg,
                                      const cfr_dist* dist, size_t* bytes);
/* Builds the solver in `workspace` (>= bytes, device memory of the current
 * device), uploads the flattened game, initialises sigma^(1) = 1/|A(h)|
 * and captures the iteration graph.  Blocking. */
cfr_status cfr_solver_create(const cfr_game* g, const cfr_solver_config* cfg, void* workspace,
                             size_t workspace_bytes, void* stream, const cfr_dist* dist,
                             cfr_solver** out);
/* (The game must outlive its solvers.) */
void cfr_solver_destroy(cfr_solver* s);

/* Runs `iterations` CFR iterations (T += iterations) and synchronises the stream;
 * CFR_ERR_NUMERICAL if any regret or strategy became NaN/Inf. */
cfr_status cfr_solver_run(cfr_solver* s, int64_t iterations);
/* Enqueues `iterations` iterations on the stream and returns immediately (for
 * event timing); call cfr_solver_sync before reading results. */
cfr_status cfr_solver_enqueue(cfr_solver* s, int64_t iterations);
cfr_status cfr_solver_sync(cfr_solver* s);
/* Iterations completed so far (T). */
cfr_status cfr_solver_iteration(cfr_solver* s, int64_t* T);

/* Host outputs in the caller's (h, a) order (qbase).  sigma_bar (Eq 10):
 * S_num / S_den, uniform where S_den = 0 (reading Q5). */
cfr_status cfr_solver_average_strategy(cfr_solver* s, double* out /* [Q+] */);
/* sigma^(T+1) (Eq 9). */
cfr_status cfr_solver_current_strategy(cfr_solver* s, double* out /* [Q+] */);
/* Raw state for checkpoint/inspection: cumulative regrets R [Q+], S_num [Q+],
 * S_den [H+] (caller order).  Any pointer may be NULL. */
cfr_status cfr_solver_get_state(cfr_solver* s, double* regret, double* s_num, double* s_den);
/* Resume from a checkpoint (SURVEY.md §5 checkpoint/resume): T iterations done, the
 * cumulative regrets R and average-strategy sums S_num (caller (h, a) order, [Q+])
 * and S_den (caller infoset order, [H+]), as cfr_solver_get_state returned them.
 * The current strategy is set to the regret matching of R (Eq 9), which
 * is what every update rule leaves after an iteration, so a restored solver
 * continues bit-identically to one that never stopped.  Values are rounded once to
 * the working precision.  Blocking.  CFR_ERR_INVALID_ARG on T < 0 or NULL. */
cfr_status cfr_solver_set_state(cfr_solver* s, int64_t T, const double* regret, const double* s_num,
                                const double* s_den);

#define CFR_EV_AVERAGE 0
#define CFR_EV_CURRENT 1
/* Per-player expected values u_hat(sigma, i) at the root under the
 * average (Q10) or current strategy, computed on the device, [P]. */
cfr_status cfr_solver_expected_values(cfr_solver* s, int32_t which, double* out /* [P] */);
/* Best response to sigma_bar per player (ties to the lowest action), NashConv =
 * sum_i (BR_i - EV_i) and exploitability = NashConv / P (reading Q11, PAPER.md
 * Fig 3 / P:557-560), on the device, for any perfect-recall game and any world
 * size (sharded solvers need the NCCL id; external mode: cfr_solver_br_phase).
 * Infosets whose members span tiles, depths or ranks are decided after a pass
 * from exact global sums; the pass repeats until every such decision below is
 * final (reading Q17; cfr_solver_br_passes).  br may be NULL. */
cfr_status cfr_solver_exploitability(cfr_solver* s, double* nash_conv, double* exploitability,
                                     double* br /* [P] or NULL */);
/* Exploitability curve (Fig 3): runs `iterations` iterations and, after
 * every `every` of them, evaluates sigma_bar's EV and best responses on the
 * device inside one CUDA graph, without a host synchronisation per evaluation.
 * out (host, caller-owned) receives floor(iterations / every) rows of 2 + 2P
 * doubles: T, NashConv, EV_1..EV_P, BR_1..BR_P; *rows = rows written.  The
 * values equal cfr_solver_exploitability at the same T bit for bit. */
cfr_status cfr_solver_run_tracked(cfr_solver* s, int64_t iterations, int64_t every, double* out,
                                  int64_t* rows);
/* Number of MODE_BR backward passes per player of one best response (1 when no
 * infoset is deferred; D + 1 otherwise). */
cfr_status cfr_solver_br_passes(cfr_solver* s, int32_t* passes);

/* Instrumentation for bench.py: kernels launched per iteration, and the mean
 * per-kernel-class device time (CUDA events on the solver stream, ms) over
 * `iterations` un-graphed iterations: out_ms[0] forward levels, [1] backward
 * levels, [2] deferred update, [3] dominant (largest) backward level, [4] the
 * dominant level's index.  The iterations ARE applied (T advances). */
cfr_status cfr_solver_launches_per_iteration(cfr_solver* s, int64_t* launches);
cfr_status cfr_solver_profile(cfr_solver* s, int64_t iterations, double* out_ms /* [5] */);
/* Algorithmic DRAM bytes of one iteration by the DESIGN.md §6 model: out[0]
 * total, [1] forward, [2] backward, [3] update, [4] dominant backward level. */
cfr_status cfr_solver_model_bytes(cfr_solver* s, double* out /* [5] */);
/* Which backward kernel serves each parent level L = 0..D-1 of the CFR iteration:
 * out[L] = 0 (no slots), 1 k_bwd (tile per CTA), 3 k_bwd_stream (TMA bulk-copy
 * ring); 2 is no longer used (the pipelined cp.async kernel was removed).  `max_levels` bounds out[];
 * *num_levels receives D. */
cfr_status cfr_solver_level_kernels(cfr_solver* s, int32_t* out, int32_t max_levels, int32_t* num_levels);
/* Cumulative work counters of the streaming backward kernel per parent level L
 * (0..D-1) since creation: out[4L+0] infosets updated (live: some member with a
 * nonzero pi_check or pi_hat), out[4L+1] their (h, a) pairs, out[4L+2] infosets
 * visited, out[4L+3] pairs visited (zeros for levels served by other kernels).  A
 * dead infoset's update is the identity (every term an exact zero), so its writes
 * are skipped; cfr_solver_model_bytes counts update writes of live infosets only
 * (live fractions of the last cfr_solver_profile window). */
cfr_status cfr_solver_counters(cfr_solver* s, int64_t* out /* [4 * max_levels] */, int32_t max_levels,
                               int32_t* num_levels);
/* Per level L of the last cfr_solver_profile window: out[4L+0] forward ms (depth L),
 * out[4L+1] backward ms (parent depth L), out[4L+2] / out[4L+3] the DESIGN.md §6
 * model bytes of those two launches. */
cfr_status cfr_solver_level_profile(cfr_solver* s, double* out /* [4 * max_levels] */, int32_t max_levels,
                                    int32_t* num_levels);

/* Writes a fresh ncclUniqueId (128 bytes) to `out` (rank 0 only). */
cfr_status cfr_nccl_unique_id(void* out /* 128 bytes */);

/* ------------------------------------------------------ multi-GPU sharding --
 * With world_size > 1 the tree is level-sharded: depths 0..cut
 * are replicated, the decision nodes of depth `cut` are split into world_size
 * contiguous ranges balanced by subtree size, and each rank owns the descendants
 * of its range.  One iteration has two exchanges, both sum-allreduces that are
 * exact by construction:
 *   CFR_XCHG_CUT  cut-level decision values (R = f64 or f32 elements; each value
 *                 is nonzero on exactly one rank);
 *   CFR_XCHG_ACC  int64 exact-slice partial sums of the deferred infosets.
 * With an NCCL id both run inside the iteration's CUDA Graph.  Without one
 * ("external" mode, used by the tests) the caller drives the phases and performs
 * the two sums itself; readbacks then return this rank's part (zeros for the
 * infosets another rank reports) and the caller sums them.
 * Best response in external mode: CFR_BR_SETUP once, then per player i and per
 * pass (cfr_solver_br_passes): CFR_BR_LOWER, sum CFR_XCHG_CUT, CFR_BR_UPPER, sum
 * CFR_XCHG_ACC, CFR_BR_DECIDE (out = root values [P] of that pass; the last
 * pass's entry i is BR_i). */
#define CFR_PHASE_LOWER 0     /* forward pass + backward of the owned depths (+ cut pack) */
#define CFR_PHASE_UPPER 1     /* cut unpack + trunk backward                              */
#define CFR_PHASE_UPDATE 2    /* deferred-infoset update; ends the iteration (T += 1)     */
#define CFR_PHASE_EV_LOWER 3  /* sigma_bar + values pass of the owned depths (+ cut pack) */
#define CFR_PHASE_EV_UPPER 4  /* cut unpack + trunk values pass; out = root values [P]    */
cfr_status cfr_solver_phase(cfr_solver* s, int32_t phase, double* out /* [P] or NULL */);
#define CFR_BR_SETUP 0        /* sigma_bar + its forward pass (reach of every level)      */
#define CFR_BR_LOWER 1        /* best-response pass of the owned depths (+ cut pack)      */
#define CFR_BR_UPPER 2        /* cut unpack + trunk best-response pass                    */
#define CFR_BR_DECIDE 3       /* deferred infosets' argmax (k_br_decide); out = root [P]  */
cfr_status cfr_solver_br_phase(cfr_solver* s, int32_t phase, int32_t player, double* out /* [P] or NULL */);
#define CFR_XCHG_CUT 0
#define CFR_XCHG_ACC 1
cfr_status cfr_solver_exchange_size(cfr_solver* s, int32_t which, size_t* bytes);
/* put = 0: device -> host copy of the exchange buffer; put = 1: host -> device. */
cfr_status cfr_solver_exchange(cfr_solver* s, int32_t which, int32_t put, void* host, size_t bytes);
/* out[8]: cut depth (-1 = unsharded), cut-level decision nodes, owned nodes below
 * the cut, local nodes, local decision nodes, deferred infosets, deferred (h, a)
 * pairs, world size. */
cfr_status cfr_solver_shard_info(cfr_solver* s, int64_t* out);
/* Host-only view of the same partition for (rank, world): out[10] = the eight
 * fields above, cut-level decision nodes owned by `rank`, infosets `rank` reports
 * in readbacks.  No GPU needed. */
cfr_status cfr_game_shard_info(const cfr_game* g, int32_t rank, int32_t world, int64_t* out);
/* Shard files, so that N ranks of one host do not each hold the whole tree:
 * one process writes `<prefix>.r<rank>of<world>.cfrshard` for every rank; each
 * rank then loads only its own view.  A loaded game serves cfr_game_info,
 * cfr_game_qbase and solvers with exactly that (rank, world_size);
 * cfr_game_canonical returns CFR_ERR_UNSUPPORTED for it. */
cfr_status cfr_game_save_shards(const cfr_game* g, int32_t world, const char* prefix);
cfr_status cfr_game_load_shard(const char* prefix, int32_t rank, int32_t world, cfr_game** out);

#ifdef __cplusplus
}
#endif
#endif /* CFR_B200_H */
