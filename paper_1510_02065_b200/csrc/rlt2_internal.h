// rlt2_internal.h — device-state layout and kernel launchers shared by the CUDA kernels
// (rlt2_kernels.cu) and the host control (rlt2_host.cu).  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rlt2 {

constexpr int kMaxN = 64;

// Device-resident control block of one bound (stop test of P:183/P:193 on the device).
struct Ctl {
    double lb_dual;    // sum of all level-0 concentration values (LB - kappa)
    double lbprime;    // LB' of the last iteration
    double lb;         // (double)kappa + lb_dual
    double lb_glb;     // after iteration 0
    double K, UB;      // stop parameters of the current bound call
    long long kappa;   // fixed-fixed cost of the node (int64, exact)
    int iters;         // iterations completed in the current bound call
    int status;        // 0 cap, 1 converged, 2 pruned
    int stopped;       // 1: remaining launches of this call are no-ops
    int err;           // bit 0: LAP residual below -tau (reading R8)
    int trace_cap;
    int pad;
};

// The level-2 LAP work queue (blocks handed out in order to persistent warps); reset by
// k_sigma every iteration.
struct Sched {
    unsigned long long head;
};

// Geometry of the reduced problem at the current node.
struct Geom {
    int n;             // free facilities
    int64_t ldc;       // stride (doubles) of one C block: (n-1)^2 rounded up to even
    int64_t ld2;       // stride (doubles) of one stored D block: (n-2)^2 rounded up to even
    int64_t nblk;      // stored D blocks n^2 (n-1)^2 / 2
    int64_t off[kMaxN + 1];  // first block id of facility i (canonical first facility)
    int ntri;          // facility triples n (n-1) (n-2) / 6
};

// Partial assignment of the node, passed to k_init by value.
struct Node {
    int N, n, m;
    int I[kMaxN], J[kMaxN];        // free facilities / locations ascending
    int fac[kMaxN], loc[kMaxN];    // fixed pairs
};

inline void make_geom(int n, Geom &g)
{
    g.n = n;
    int64_t c = (int64_t)(n - 1) * (n - 1), d = (int64_t)(n - 2) * (n - 2);
    g.ldc = (c + 1) & ~int64_t(1);
    g.ld2 = (d + 1) & ~int64_t(1);
    g.nblk = (int64_t)n * n * (n - 1) * (n - 1) / 2;
    int64_t acc = 0;
    for (int i = 0; i <= n && i <= kMaxN; i++) {
        g.off[i] = acc;
        if (i < n) acc += (int64_t)n * (n - 1 - i) * (n - 1);
    }
    g.ntri = n * (n - 1) * (n - 2) / 6;
}

// LAP launch levels.
enum LapLevel { LAP_L2 = 0, LAP_L1_ACC = 1, LAP_L1_SET = 2, LAP_L0_ITER0 = 3, LAP_L0 = 4, LAP_BATCH = 5,
                LAP_L0_MULTI = 6 };

struct LapBatchOut {
    double *R, *S, *u, *v;
    int32_t *assign;
    int64_t *steps;
    int32_t *err;
};

// Batched RLT1 evaluation of the n^2 candidate children of a node (strong branching).
struct Rlt1Batch {
    int K;            // children (n * n)
    Geom g;           // geometry of a child (n' = n - 1)
    double *C;        // K * n'^2 blocks of stride g.ldc
    double *B;        // K * bstr
    int64_t bstr;     // even >= n'^2
    double *lbd;      // K accumulated concentration sums
    long long *kap;   // K fixed-fixed costs
};

// ---- launchers (rlt2_kernels.cu) -----------------------------------------------------
cudaError_t launch_rlt1_init(const Node &parent, const Rlt1Batch &R, const int64_t *F, const int64_t *Dist,
                             cudaStream_t st);
cudaError_t launch_rlt1_pair(const Rlt1Batch &R, cudaStream_t st);
// level 1 (acc: iteration 0) or level 0 LAPs of every child
cudaError_t launch_rlt1_lap(const Rlt1Batch &R, int level1, int acc, int num_sms, cudaStream_t st);
// warm child (NEXT-3 (i)): parent state (gp) -> child state (gc, n = gp.n - 1)
struct FoldArgs {
    Geom gp, gc;
    int a, b;  // parent-reduced facility / location fixed by the child
    const double *pB, *pC, *pD;
    const Ctl *pctl;
    double *cB, *cC, *cD;
    Ctl *cctl;
    int *triples;  // child's facility-triples table
    int d_zero;    // parent D lazily zero
};
cudaError_t launch_fold(const FoldArgs &f, int num_sms, cudaStream_t st);

cudaError_t launch_init(const Node &node, const Geom &g, const int64_t *F, const int64_t *Dist,
                        double *B, double *C, int *triples, Ctl *ctl, cudaStream_t st);
cudaError_t launch_ctl_begin(Ctl *ctl, double K, double UB, int trace_cap, cudaStream_t st);
cudaError_t launch_sigma(const Geom &g, const double *B, const double *C, double *sigma,
                         const Ctl *ctl, Sched *sched, cudaStream_t st);
constexpr int TT = 8;  // transfer tile edge (locations j, l, q)
// edge of the facility-triple cubes of the TMA transfer's dispatch order (write_triples):
// 1.18 -> 1.13-1.15 ms at N = 30 for edges 2..10 (lexicographic order: 1.18-1.20; one box)
constexpr int kTxCube = 8;

struct TransferArgs {
    Geom g;
    double *D;            // stored blocks of this rank (element dbase of the global layout first)
    const double *sigma;  // all stored blocks
    const int *triples;
    int d_zero;
    const Ctl *ctl;
    Sched *sched;
    int ntile;            // ceil(n / TT)
    unsigned ntile_mul;   // ceil(2^16 / ntile): y / ntile = (y * ntile_mul) >> 16 for y < 64 (set by the launcher)
    // sharded iteration (nullptr tiles: every tile, single rank)
    const int *tiles;     // this rank's tiles (global tile id = triple * ntile^3 + tile)
    const int *tinfo;     // kind | slot << 2 (slot: 512-double unit of the exchange buffers)
    int64_t loc_off[kMaxN];  // local block index = global block id + loc_off[facility] (0: unsharded)
    double *sendbuf;
    const double *recvbuf;
    int pack;             // 1: write this side's partial of AGG/HOLD tiles; 0: apply
};
cudaError_t launch_transfer(const TransferArgs &A, int ntiles_list, cudaStream_t st);
// tensor maps of the stored blocks, one per first facility (k_transfer_tma); box extents
constexpr int kBox0 = TT + 4, kBox1 = TT + 1;  // dim0: TT+2 columns + an even (16-byte) start
// (dim0 = in-block entries, dim1 = second location, dim2 = 1 second facility, dim3 = TT first locations)
struct TmaMaps {
    CUtensorMap m[kMaxN];
};
cudaError_t launch_transfer_tma(const TransferArgs &A, const TmaMaps &M, cudaStream_t st);
int tma_box0(int n);  // dim0 box extent for node size n (TT + 2 when n - 2 is even, else TT + 4)
struct Offsets {
    int64_t off[kMaxN];
};
cudaError_t launch_credit(const Geom &g, const double *S, const Offsets &pos, double *C, const Ctl *ctl,
                          cudaStream_t st);
// Level-2 / level-1 / level-0 concentrations (one warp per LAP).
// sched != nullptr (level 2 only): persistent warps take blocks from the Sched queue.
cudaError_t launch_lap_level(LapLevel lvl, const Geom &g, double *D, double *C, double *B,
                             Ctl *ctl, double *trace, int num_sms, int lap_warps, Sched *sched,
                             cudaStream_t st);
// Level-2 LAPs of `count` local blocks (sharded): S of block b to Sout[b].
cudaError_t launch_lap_l2_local(const Geom &g, double *Dloc, int64_t count, double *Sout, Ctl *ctl, int num_sms,
                                int lap_cfg, Sched *sched, cudaStream_t st);
cudaError_t launch_lap_batch(int m, int64_t count, int64_t ld, const double *M,
                             const LapBatchOut &o, int num_sms, cudaStream_t st);

}  // namespace rlt2
