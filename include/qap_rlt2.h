/*
 * qap_rlt2.h — C ABI of the B200 RLT2 dual-ascent lower-bound library (libqaprlt2.so).
 *
 * The library computes the level-2 RLT dual-ascent lower bound of a Koopmans–Beckmann
 * QAP (Gonçalves et al., arXiv 1510.02065; P:n = /root/reference/PAPER.md line n):
 *
 *   min sum_{i,j,k!=i,n!=j} f_ik d_jn x_ij x_kn     over permutation matrices x
 *
 * by Algorithm 1: spread B->C->D, transfer between complementary costs of D,
 * concentrate D->C, transfer C, concentrate C->B, concentrate B->LB, repeated.  Every
 * concentration is an exact linear assignment problem whose residual replaces the
 * submatrix.  All arithmetic runs in sm_100a CUDA kernels; the host code
 * only sequences them.  Readings of the paper's silent points are DESIGN.md §3 R1..R30.
 *
 * Conventions
 *   - Every function returns a qap_status; no exceptions cross the ABI.
 *   - Pointers named *_dev are DEVICE pointers (current device); all others are HOST.
 *   - Inputs are copied; the caller keeps ownership of everything it passes in.
 *   - A handle is single-owner and not thread-safe (one worker at a time).
 *   - All work is enqueued on opts->cuda_stream (NULL: the legacy default stream).
 *     Calls that return host-visible results synchronise that stream.
 *   - On failure, qap_last_error(h) returns a human-readable message.
 *
 * Export layouts (qap_rlt2_dual_copy; identical to the oracle's documented layout):
 *   B : n×n row-major, b_ij
 *   C : n² blocks C_ij in (i,j) row-major order; block (n-1)×(n-1) row-major; row k≠i
 *       at index k-[k>i], column l≠j at index l-[l>j]
 *   D : stored blocks D{ij,kl}, i<k, l≠j, in (i,j,k,l) lexicographic order; block
 *       (n-2)×(n-2) row-major; row p∉{i,k} at p-[p>i]-[p>k], column q∉{j,l} at
 *       q-[q>j]-[q>l].  D{kl,ij} is the same stored block ("complementary submatrices",
 *       P:250-252) and each stored value equals both of its logical entries.
 *   n is the number of FREE facilities at the current node (n = N at the root).
 */
#ifndef QAP_RLT2_H
#define QAP_RLT2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qap_rlt2 qap_rlt2;  /* opaque handle; owns all device memory it allocates */

typedef enum {
    QAP_OK = 0,
    QAP_E_ARG = 1,       /* invalid argument (sizes, negative entries, bad partial assignment) */
    QAP_E_CAPACITY = 2,  /* not enough device memory for N                                     */
    QAP_E_CUDA = 3,      /* a CUDA runtime call failed                                          */
    QAP_E_NCCL = 4,      /* reserved: multi-GPU communicator failure                            */
    QAP_E_NUMERIC = 5,   /* a LAP residual fell below -tau (certificate failure, reading R8)    */
    QAP_E_STATE = 6      /* call not valid in the handle's current state                         */
} qap_status;

/*
 * Host-staged collectives of a sharded bound, an alternative to NCCL: the
 * library copies its exchange buffers to pinned host memory, calls these callbacks (same
 * order on every rank, from the thread that called the library), and copies the results
 * back.  For processes that share one GPU (NCCL refuses two ranks on one device) and for
 * testing the sharded data path over any host transport (e.g. torch.distributed gloo).
 *   exchange: for every peer q != rank with count[q] > 0, send send[off[q] .. off[q] +
 *             count[q]) to q and receive q's range into recv[off[q] .. off[q] + count[q])
 *             (counts and offsets in doubles; both ranks of a pair use the same range size).
 *   allgather: S_all[lo[q] .. lo[q+1]) holds rank q's values on rank q; afterwards every
 *             rank holds all of them (lo has world + 1 entries).
 * Return 0 on success; anything else fails the bound with QAP_E_NCCL.  The pointers are
 * valid only during the call.
 */
typedef struct {
    void *ctx;
    int32_t (*exchange)(void *ctx, const double *send, double *recv, const int64_t *off, const int64_t *count,
                        int32_t world, int32_t rank);
    int32_t (*allgather)(void *ctx, double *S_all, const int64_t *lo, int32_t world, int32_t rank);
} qap_host_transport;

typedef struct {
    int32_t device;       /* CUDA device ordinal; -1 = current device                         */
    void *cuda_stream;    /* cudaStream_t to enqueue on; NULL = legacy default stream          */
    int32_t flags;        /* QAP_FLAG_* bit set                                                */
    int32_t lap_warps;    /* level-2 LAP launch config: warps per CTA (bits 0-7); 0 = default  */
    int32_t world;        /* ranks sharing ONE bound (<= 1: single GPU)         */
    int32_t rank;         /* this process's rank in [0, world)                                 */
    const void *nccl_id;  /* world > 1: 128-byte ncclUniqueId from qap_nccl_unique_id on rank
                             0, broadcast by the caller; every rank then calls create (collective) */
    const qap_host_transport *host_transport;  /* world > 1 and non-NULL: host-staged collectives
                             through these callbacks instead of NCCL (nccl_id unused); copied */
} qap_rlt2_opts;

#define QAP_FLAG_TIME_KERNELS 1   /* record CUDA events around every launch (qap_rlt2_kernel_stats) */
#define QAP_FLAG_NO_GRAPH 4       /* do not replay the iteration loop from a cached CUDA graph     */
#define QAP_FLAG_LDG_TRANSFER 8   /* transfer with per-element loads instead of tensor-map TMA    */
/* other bits are reserved: qap_rlt2_create returns QAP_E_ARG for them                    */

typedef struct {
    double lb;          /* kappa + dual bound after the last iteration run            */
    double lb_glb;      /* bound after iteration 0 = Gilmore–Lawler (reading R1)               */
    int32_t iters;      /* Algorithm-1 iterations run by this call (iteration 0 excluded)      */
    int32_t status;     /* 0 iteration cap, 1 converged (LB'/UB < K), 2 pruned (LB > UB-1+1e-6) */
    double *lb_trace;   /* optional HOST buffer: LB after each iteration of this call          */
    int32_t lb_trace_cap;
    int32_t launches;   /* kernels launched by this call                                       */
} qap_rlt2_result;

/*
 * qap_rlt2_create — P:80-97 (flows f_ik, distances d_jn), P:179-181 (initial costs).
 *   N   problem size, 3 <= N <= 64.
 *   F   N×N row-major int64 flows  f_ik >= 0 (HOST; copied).
 *   D   N×N row-major int64 distances d_jl >= 0 (HOST; copied).
 *   Allocates the dual state for N (B, C and the halved D of P:250-252, ~8·N²(N-1)²(N-2)²/2
 *   bytes) and initialises the root node (no fixed assignment), i.e. calls fix(h, 0, ...).
 * Errors: QAP_E_ARG (N out of range, negative entry, N²·maxF·maxD >= 2^53 so that the
 *   integer costs would not be exact in fp64); QAP_E_CAPACITY; QAP_E_CUDA.
 */
qap_status qap_rlt2_create(int32_t N, const int64_t *F, const int64_t *D,
                           const qap_rlt2_opts *opts, qap_rlt2 **out);

/*
 * qap_rlt2_load — replace the instance of an existing handle by a new one of the same N
 *   (HOST F, D copied host->device), then re-initialise the root node as qap_rlt2_create
 *   does.  Reuses the device allocation (a batch of instances of one size needs one
 *   handle).  Errors as qap_rlt2_create; on error the handle keeps its previous instance.
 */
qap_status qap_rlt2_load(qap_rlt2 *h, const int64_t *F, const int64_t *D);

/*
 * qap_rlt2_fix — set the node's partial assignment Φ = {(fac[t], loc[t]) : t < m}
 *   (facility fac[t] at location loc[t]; HOST arrays of length m; m = 0 is the root).
 *   REPLACES any previous Φ.  Rebuilds the reduced problem of the n = N-m free
 *   facilities/locations (cold child, reading R19): b0 folds the fixed-free costs,
 *   c_ij[kl] = f'_ik d'_jl, D = 0, LB = kappa (the fixed-fixed cost).  The next
 *   qap_rlt2_bound starts with iteration 0.
 * Errors: QAP_E_ARG (index out of range, duplicate facility or location, N-m < 3).
 */
qap_status qap_rlt2_fix(qap_rlt2 *h, int32_t m, const int32_t *fac, const int32_t *loc);

/*
 * qap_rlt2_fold — warm child (reading R31, fold rules of
 *   SPEC S:368 derived from the evaluation identity P:169).  Makes `child`'s node the child
 *   of `parent`'s node that fixes facility `fac` at location `loc` (original 0-based indices,
 *   both free in the parent) and builds its dual state from the parent's CURRENT state
 *   (after qap_rlt2_fix or a completed qap_rlt2_bound):
 *     kappa' = kappa, lb_dual' = lb_dual + b_ab,
 *     b'_xy = (b_xy + c_ab[xy]) + c_xy[ab],
 *     c'_xy[zw] = c_xy[zw] + ((d_{ab,xy,zw} + d_{ab,zw,xy}) + d_{xy,zw,ab}),
 *     D' = D restricted to the remaining indices,
 *   so every completion keeps its cost.  The next qap_rlt2_bound(child, ...) runs iteration 0
 *   (concentrate C -> B -> LB) and then the loop from that state.  Both handles: same device,
 *   same instance, single-GPU; the parent needs n >= 4 free facilities.  Enqueued on the
 *   child's stream, ordered after the parent's pending work and before its later work (no
 *   host synchronisation).  Errors: QAP_E_ARG, QAP_E_STATE (parent mid-iteration).
 */
qap_status qap_rlt2_fold(qap_rlt2 *child, const qap_rlt2 *parent, int32_t fac, int32_t loc);

/*
 * qap_rlt2_bound — run Algorithm 1.
 *   If the node is fresh (after create/fix), iteration 0 (concentrate C->B->LB, reading
 *   R1) runs first; then up to max_iters iterations of the loop body P:185-193.  A later
 *   call continues the ascent from the current dual state.
 *   K   minimum relative progress (reading R14); 0 disables the test.
 *   UB  upper bound (+INFINITY allowed; reading R15).  With UB finite the ascent stops
 *       with status 2 when LB > UB - 1 + 1e-6 and with status 1 when K > 0 and
 *       LB'/UB < K.  The stop test runs on the device after every iteration.
 *   out (HOST, required) receives the bound; out->lb_trace may be NULL.
 *   Synchronises the handle's stream.
 * Errors: QAP_E_NUMERIC (LAP certificate failure), QAP_E_CUDA, QAP_E_ARG.
 */
qap_status qap_rlt2_bound(qap_rlt2 *h, int32_t max_iters, double K, double UB,
                          qap_rlt2_result *out);

/*
 * qap_rlt2_bound_async / qap_rlt2_bound_result — the two halves of qap_rlt2_bound: enqueue
 * the bound on the handle's stream without synchronising, then wait for it and read the
 * result.  Lets a caller run independent bounds on several handles concurrently.
 */
qap_status qap_rlt2_bound_async(qap_rlt2 *h, int32_t max_iters, double K, double UB);
qap_status qap_rlt2_bound_result(qap_rlt2 *h, qap_rlt2_result *out);

/* Entry counts of the export layouts above for the current node (HOST outputs).       */
qap_status qap_rlt2_dual_sizes(const qap_rlt2 *h, int64_t *nB, int64_t *nC, int64_t *nD);

/*
 * qap_rlt2_dual_copy — copy the dual state to HOST buffers in the export layouts above
 *   (any of B, C, D may be NULL to skip).  Also returns kappa + accumulated dual (the
 *   current LB) in *lb if lb != NULL.  Synchronises the handle's stream.
 */
qap_status qap_rlt2_dual_copy(const qap_rlt2 *h, double *B, double *C, double *D, double *lb);

/*
 * qap_rlt2_step — run ONE phase of an iteration (parity testing / profiling):
 *   QAP_PHASE_ITER0       concentrate C->B, B->LB (reading R1)
 *   QAP_PHASE_TRANSFER    spread B->C, spread C->D, transfer D
 *   QAP_PHASE_CONC_D      concentrate D->C
 *   QAP_PHASE_CONC_C      transfer C (exact no-op, reading R13) + concentrate C->B
 *   QAP_PHASE_CONC_B      concentrate B->LB
 * Phases must be called in Algorithm-1 order; otherwise QAP_E_STATE.
 */
#define QAP_PHASE_ITER0 0
#define QAP_PHASE_TRANSFER 1
#define QAP_PHASE_CONC_D 2
#define QAP_PHASE_CONC_C 3
#define QAP_PHASE_CONC_B 4
qap_status qap_rlt2_step(qap_rlt2 *h, int32_t phase);

/*
 * qap_rlt2_kernel_stats — per-kernel launch counts and summed CUDA-event durations (ms)
 *   recorded since the last reset, when the handle was created with
 *   QAP_FLAG_TIME_KERNELS.  Kernel kinds: QAP_K_INIT, QAP_K_SIGMA, QAP_K_TRANSFER,
 *   QAP_K_LAP2, QAP_K_LAP1, QAP_K_LAP0.  Arrays have QAP_K_COUNT entries (HOST).
 *   reset != 0 clears the counters after reading.  Synchronises the stream.
 */
#define QAP_K_INIT 0
#define QAP_K_SIGMA 1
#define QAP_K_TRANSFER 2
#define QAP_K_LAP2 3
#define QAP_K_LAP1 4
#define QAP_K_LAP0 5
#define QAP_K_COUNT 6
qap_status qap_rlt2_kernel_stats(qap_rlt2 *h, int64_t *launches, double *ms, int32_t reset);

/*
 * Multi-GPU sharding of one bound.  With opts->world = G > 1
 * the stored blocks are partitioned by first facility into G contiguous ranges balanced
 * by block count; every rank holds only its range.  Per iteration: the partials of the
 * complementary classes whose members straddle two ranks are exchanged (grouped NCCL
 * send/recv = all-to-all), the level-2 values S are all-gathered (NCCL broadcasts), and
 * the level-1/level-0 concentrations run replicated, so LB bits are identical on every
 * rank and equal to the single-GPU bits.  All calls on a sharded handle are collective.
 * qap_rlt2_dual_copy on a sharded handle writes only this rank's blocks of D.
 */
qap_status qap_nccl_unique_id(void *id128);   /* rank 0; 128 bytes, broadcast by the caller */
/* Shard geometry of h at the current node (any pointer may be NULL).                 */
qap_status qap_rlt2_shard_info(const qap_rlt2 *h, int32_t *world, int32_t *rank, int64_t *blk_lo,
                               int64_t *blk_hi, int64_t *tiles_local, int64_t *tiles_shared,
                               int64_t *slots);
/* Host-only: the shard plan of `rank` among `world` for size n (no GPU needed): block
 * ranges blk_lo[world+1], exchanged tiles per peer peer_slots[world], this rank's tile list
 * (global tile ids, kind | slot<<2) — used to test the partition logic.               */
qap_status qap_shard_plan(int32_t n, int32_t world, int32_t rank, int64_t *blk_lo, int64_t *peer_slots,
                          int32_t *tiles, int32_t *tinfo, int64_t tiles_cap, int64_t *n_tiles);
/* In-process group of G shards (one process; the collectives become device copies) for
 * single-GPU testing of the sharded path: out[G] handles; bound them with
 * qap_rlt2_group_bound (out[G] results); fix each member with qap_rlt2_fix.           */
qap_status qap_rlt2_create_group(int32_t G, int32_t N, const int64_t *F, const int64_t *D,
                                 const qap_rlt2_opts *opts, qap_rlt2 **out);
qap_status qap_rlt2_group_bound(qap_rlt2 *const *hs, int32_t G, int32_t max_iters, double K, double UB,
                                qap_rlt2_result *out);

/* Last error message of h (or of the last failed create when h == NULL).             */
const char *qap_last_error(const qap_rlt2 *h);

/* Release the handle and its device memory; NULL-safe.                               */
void qap_destroy(qap_rlt2 *h);

/*
 * qap_lap_batch — the batched warp LAP solver on its own (one warp per LAP,
 *   P:243-245).  Solves `count` independent m×m problems M_b = M_dev + b*ld (DEVICE,
 *   row-major, fp64, entries finite and >= 0), 1 <= m <= 64, ld >= m*m, ld even, M_dev
 *   16-byte aligned.  Outputs (DEVICE; R_dev required and 16-byte aligned, the others
 *   may be NULL):
 *     R_dev      + b*ld   residual (M - u) - v, clamped as in reading R8 (may alias M_dev;
 *                         the padding double of an odd m*m block may be overwritten)
 *     S_dev      [b]      sum_r M[r][a(r)] in row order (reading R9)
 *     assign_dev + b*m    column of each row (tie rule R6)
 *     u_dev, v_dev + b*m  canonical duals (reading R5)
 *     steps_dev  [b]      Dijkstra steps taken
 *   Enqueued on `stream` (cudaStream_t, NULL = default); does not synchronise.  Returns
 *   QAP_E_NUMERIC only from qap_lap_batch_status after a sync (status word per call).
 */
qap_status qap_lap_batch(int32_t m, int64_t count, int64_t ld, const double *M_dev,
                         double *R_dev, double *S_dev, int32_t *assign_dev, double *u_dev,
                         double *v_dev, int64_t *steps_dev, int32_t *err_dev, void *stream);

/*
 * qap_bnb_solve — minimal deterministic depth-first branch-and-bound (P:236-238 as the
 *   caller of the bound).  Branches on the lowest-index free facility,
 *   children in ascending location order; every node with n' >= 4 free facilities is
 *   fixed (cold) and bounded with `iters` iterations; nodes with n' <= 3 are leaves
 *   solved by enumeration; prune when LB > UB - 1 + 1e-6; the incumbent is replaced
 *   only on strict improvement.  UB0 = +INFINITY for none.
 *   batch > 1: the children of an expanded node are bounded `batch` at a time
 *   concurrently (batch-1 helper handles on their own streams, each sized like h, owned by
 *   h: created on first use, kept with their CUDA graphs for later calls, reloaded by
 *   qap_rlt2_load and freed by qap_destroy); with K = 0 every decision equals the
 *   one-node-at-a-time search.
 *   sb_iters >= 0: strong branching at nodes with n' >= 5: the line chosen by
 *   qap_rlt2_strong_branch is branched on (children in ascending order of the line's other
 *   index) and candidates whose RLT1 estimate exceeds UB - 1 + 1e-6 are cut (*sb_cut).
 *   Outputs (HOST): *opt (or -1 if nothing better than UB0), perm[N], node counts.
 *   The handle's node is left at the last bounded node.
 */
qap_status qap_bnb_solve(qap_rlt2 *h, int32_t iters, double K, double UB0, int32_t batch, int32_t sb_iters,
                         int64_t *opt, int32_t *perm, int64_t *bounded, int64_t *leaves, int64_t *pruned,
                         int64_t *sb_cut);

/*
 * qap_bnb_run — qap_bnb_solve with checkpoint / resume (interruptions of multi-day
 *   solves).  The search state (stack of expanded nodes with their
 *   children's bounds, incumbent, counters) is written atomically (<path>.tmp + rename) to
 *   checkpoint_path every checkpoint_every bounded nodes and when the run stops early
 *   (max_nodes > 0: at most that many nodes bounded by this call).  resume != 0 continues
 *   from checkpoint_path (same instance and parameters, checked by digest); a resumed run
 *   makes exactly the decisions of an uninterrupted one.  out->complete = 1 when the tree
 *   is exhausted.
 *   warm = 1 (NEXT-3 (i), reading R31): every child's state is folded from its parent's
 *   post-bound state (qap_rlt2_fold) instead of rebuilt cold; the root (or `root`) is
 *   bounded cold.  The states of the expanded nodes on the current DFS path are kept in
 *   depth handles owned by h (capacity N - d each, created on first use); a node expanded
 *   after its children were bounded concurrently has its state rebuilt (fold + the same
 *   bound), so with K = 0 the decisions equal the one-node-at-a-time warm search (the
 *   oracle's).  qap_bnb_frontier always bounds cold.
 */
/*
 * qap_bnb_node — an open B&B node: m fixed pairs (facility fac[t] at location loc[t],
 *   0-based, N <= 64) and its RLT2 bound lb (NAN: not bounded yet).
 */
typedef struct {
    int32_t m;
    int32_t fac[64], loc[64];
    double lb;
} qap_bnb_node;

/*
 * Subtree-parallel B&B hooks ("at the first Branch, each cpu_thread takes a subtree
 *   (or node) and execute a depth-first search.  When it finished your subtree, the
 *   cpu_thread takes another node that has not been fathomed"; load balancing of
 *   unbalanced subtrees).  The library runs one worker's search; the
 *   scheduler handing nodes to workers belongs to the caller (one process per GPU with a
 *   shared store, threads, ...).
 *   qap_bnb_sync_fn: called every sync_every bounded nodes and whenever the worker's
 *     incumbent improves, with local_best (-1: none) and its permutation (N entries, NULL
 *     when none).  It writes *global_best (best objective known to any worker, -1: none),
 *     which the worker then prunes with (LB > global_best - 1 + 1e-6), and returns how many
 *     open nodes the scheduler wants donated (0: none; < 0: abort with QAP_E_STATE).
 *   qap_bnb_donate_fn: receives each donated node (bounded, not pruned; the callee copies
 *     it).  Donation gives away the unvisited children of the worker's shallowest expanded
 *     nodes (the largest remaining subtrees), whole nodes at a time, until at least the
 *     requested number went out; donated nodes count as bounded by the donor.
 */
typedef int32_t (*qap_bnb_sync_fn)(void *ctx, int64_t local_best, const int32_t *perm, int64_t *global_best);
typedef void (*qap_bnb_donate_fn)(void *ctx, const qap_bnb_node *node);

typedef struct {
    int32_t iters;            /* RLT2 iterations per node                               */
    double K, UB0;            /* stop parameter, initial upper bound (+INFINITY: none)  */
    int32_t batch;            /* children bounded concurrently                          */
    int32_t sb_iters;         /* >= 0: strong branching with RLT1, else off             */
    const char *checkpoint_path;
    int64_t checkpoint_every; /* bounded nodes between checkpoints (0: only on stop)    */
    int64_t max_nodes;        /* stop after this many bounded nodes (0: no limit)       */
    int32_t resume;
    const qap_bnb_node *root; /* NULL: the instance root; else search only this subtree  */
                              /* (root->lb not NAN: its bound, reused, not recounted)    */
    qap_bnb_sync_fn sync;     /* NULL: none                                             */
    qap_bnb_donate_fn donate; /* NULL: donation requests are ignored                    */
    void *ctx;                /* passed to sync / donate                                */
    int64_t sync_every;       /* bounded nodes between sync calls (<= 0: 32)            */
    int32_t warm;             /* 1: warm children (qap_rlt2_fold of the parent's state, */
                              /* NEXT-3); 0: cold children (qap_rlt2_fix)                */
} qap_bnb_opts;
typedef struct {
    int64_t opt;              /* best objective found (-1: none better than UB0)        */
    int32_t perm[64];
    int64_t bounded, leaves, pruned, sb_cut;
    int32_t complete;
    int32_t depth_max;        /* fixed pairs of the deepest expanded node on the DFS stack now */
    int64_t open;             /* unvisited children on the DFS stack (0 when complete)  */
    int64_t bounded_by_depth[64];  /* bounded nodes by their number of fixed pairs      */
} qap_bnb_result;
qap_status qap_bnb_run(qap_rlt2 *h, const qap_bnb_opts *opts, qap_bnb_result *out);

/*
 * qap_bnb_frontier — breadth-first expansion from opts->root (NULL: the instance root)
 *   with the rules of qap_bnb_solve (bounds, pruning, strong branching, leaves), level by
 *   level, until a level holds >= target open nodes or the tree is exhausted (the first
 *   phase of the subtree-parallel search).  On a sharded handle (world > 1) every
 *   rank makes the same call and gets the same nodes; opts->batch > 1 needs a single-GPU
 *   handle.  Writes the open nodes of the last level, in DFS order, to nodes[0..*n_nodes)
 *   (HOST, capacity cap; QAP_E_CAPACITY if more) and the incumbent and counters of the
 *   expansion to *out (out->complete = 1 when no open node is left).  Checkpoint, sync
 *   and donate fields of opts are ignored.
 */
qap_status qap_bnb_frontier(qap_rlt2 *h, const qap_bnb_opts *opts, int32_t target, qap_bnb_node *nodes,
                            int32_t cap, int32_t *n_nodes, qap_bnb_result *out);

/*
 * qap_rlt2_strong_branch — strong branching with the RLT1 dual: every candidate
 *   child of the handle's current node (free facility I[a] at free location J[b], reduced
 *   indices, n = free facilities >= 4) is bounded by a cold RLT1 ascent (Algorithm 1 without
 *   the D operations; iteration 0 + sb_iters iterations of spread B->C, C pair mean,
 *   concentrate C->B, concentrate B->LB), all children at once on the GPU.
 *   est (HOST, n*n): est[a*n + b] = kappa_child + RLT1 bound.  *kind = 0 (row a) or
 *   1 (column b), *index = the line with the maximal min-estimate (ties: lowest index,
 *   rows first).  Uses a separate workspace (~ n^2 * 8 (n-1)^2 (n-2)^2 bytes); the node's
 *   own dual state is untouched.  Synchronises the stream.
 */
qap_status qap_rlt2_strong_branch(qap_rlt2 *h, int32_t sb_iters, double *est, int32_t *kind, int32_t *index);

#ifdef __cplusplus
}
#endif
#endif /* QAP_RLT2_H */
