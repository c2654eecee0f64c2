// rlt2_kernels.cu — sm_100a kernels of the RLT2 dual-ascent bound.
//
// P:n = /root/reference/PAPER.md line n.  Readings R1..R30 are listed in DESIGN.md §3.
//
//   k_init      O0/O1: reduced costs of the node                HBM write of B, C
//   k_sigma     spreading B->C and the per-block C->D spread amount
//   k_transfer  spreading C->D fused with the transfer between complementary
//               costs of D: one CTA per facility triple
//               and 8×8×8 location tile, every class read/written once         HBM-bound
//   k_lap<CPL>  cost concentration: one warp per LAP, cost
//               block staged global->smem by a TMA bulk copy, double buffered;
//               shortest-augmenting-path Hungarian with lane = column, argmin
//               by two redux.sync.min.u32 on an order-preserving fp64 key     issue/HBM-bound
//
// Arithmetic order follows DESIGN.md §3 exactly (same IEEE operations as the paper's
// algorithm written out), so results are reproducible bit for bit; no multiplies
// occur in fp64 after initialisation (compiled with -fmad=false regardless).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "rlt2_internal.h"

namespace rlt2 {

#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------------------------------
// Small PTX helpers: mbarrier + 1-D TMA bulk copy (cp.async.bulk, SASS UBLKCP).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *mbar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(parity)
            : "memory");
    }
}

// Order-preserving map fp64 -> u64 (unsigned order == numeric order, -0 < +0).
__device__ __forceinline__ uint64_t okey(double x)
{
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    uint64_t mask = static_cast<uint64_t>(static_cast<int64_t>(b) >> 63) | 0x8000000000000000ull;
    return b ^ mask;
}
__device__ __forceinline__ double okey_inv(uint64_t k)
{
    uint64_t b = (k & 0x8000000000000000ull) ? (k ^ 0x8000000000000000ull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// Stored-block id of D{ij,kl}, i<k, l!=j (export layout order, include/qap_rlt2.h).
__device__ __forceinline__ int64_t bid_of(const Geom &g, int i, int j, int k, int l)
{
    const int n1 = g.n - 1;
    return g.off[i] + (int64_t)j * (n1 - i) * n1 + (int64_t)(k - i - 1) * n1 + (l - (l > j));
}

// ---------------------------------------------------------------------------------------
// The warp LAP solver (reading R4/R5/R6).  Lane `lane` owns columns
// c = lane + 32 t (t < CPL).  Per column: v (dual), ucol = u of the row matched to the
// column, p (matched row, -1 free), minv / way / used of the current Dijkstra search.
// The dummy column of the textbook formulation (holding the row being inserted) lives in
// warp-uniform registers (ucur).  Every floating-point operation and its order equals the
// written-out algorithm of DESIGN.md §3 (O2), so residuals are reproducible bit for bit.
// ---------------------------------------------------------------------------------------
template <int CPL>
__device__ __forceinline__ void warp_argmin(const double (&minv)[CPL], const bool (&used)[CPL],
                                            const int (&p)[CPL], int lane, int &j1, bool &j1free,
                                            double &delta)
{
    if (CPL == 1) {
        const uint64_t key = used[0] ? ~0ull : okey(minv[0]);
        const uint32_t hi = static_cast<uint32_t>(key >> 32), lo = static_cast<uint32_t>(key);
        const uint32_t mhi = __reduce_min_sync(FULL_MASK, hi);
        const uint32_t mlo = __reduce_min_sync(FULL_MASK, hi == mhi ? lo : 0xffffffffu);
        const bool tie = (hi == mhi) && (lo == mlo);
        const uint32_t ft = __ballot_sync(FULL_MASK, tie && p[0] < 0);
        const uint32_t at = __ballot_sync(FULL_MASK, tie);
        j1 = __ffs(ft ? ft : at) - 1;
        j1free = ft != 0;
        delta = okey_inv((static_cast<uint64_t>(mhi) << 32) | mlo);
    } else {
        // lane-local best by (key, matched, t), then warp-wide
        uint64_t key = ~0ull;
        int rank = 7;
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            const uint64_t k = used[t] ? ~0ull : okey(minv[t]);
            const int r = (p[t] >= 0 ? CPL : 0) + t;
            if (k < key || (k == key && r < rank)) { key = k; rank = r; }
        }
        const uint32_t hi = static_cast<uint32_t>(key >> 32), lo = static_cast<uint32_t>(key);
        const uint32_t mhi = __reduce_min_sync(FULL_MASK, hi);
        const uint32_t mlo = __reduce_min_sync(FULL_MASK, hi == mhi ? lo : 0xffffffffu);
        const bool tie = (hi == mhi) && (lo == mlo);
        const uint32_t mr = __reduce_min_sync(FULL_MASK, tie ? static_cast<uint32_t>(rank) : 0xffu);
        const uint32_t pick = __ballot_sync(FULL_MASK, tie && static_cast<uint32_t>(rank) == mr);
        const int t = static_cast<int>(mr) % CPL;
        j1 = (__ffs(pick) - 1) + 32 * t;
        j1free = static_cast<int>(mr) < CPL;
        delta = okey_inv((static_cast<uint64_t>(mhi) << 32) | mlo);
    }
}

template <int CPL>
__device__ __forceinline__ double sel_t(const double (&a)[CPL], int t)
{
    return (CPL == 1 || t == 0) ? a[0] : a[CPL - 1];
}
template <int CPL>
__device__ __forceinline__ int sel_t(const int (&a)[CPL], int t)
{
    return (CPL == 1 || t == 0) ? a[0] : a[CPL - 1];
}

template <int CPL>
__device__ __forceinline__ void warp_lap_solve(const double *__restrict__ M, int m, int lane, int (&p)[CPL],
                                               double (&v)[CPL], double (&ucol)[CPL], int &steps)
{
    double minv[CPL];
    int way[CPL];
    bool used[CPL];
#pragma unroll
    for (int t = 0; t < CPL; t++) {
        v[t] = 0.0;
        ucol[t] = 0.0;
        p[t] = -1;
        way[t] = -1;
    }
    for (int i = 0; i < m; i++) {  // insert row i (P:205 Hungarian, one augmentation per row)
        double ucur = 0.0;         // u of row i = u[p[dummy]]
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            minv[t] = CUDART_INF;
            used[t] = (lane + 32 * t) >= m;  // columns >= m never take part
        }
        int j0 = -1, i0 = i;
        double ui0 = 0.0;
        int jfree;
        while (true) {
            const double *row = M + i0 * m;
#pragma unroll
            for (int t = 0; t < CPL; t++) {
                if (!used[t]) {
                    const double cur = (row[lane + 32 * t] - ui0) - v[t];
                    if (cur < minv[t]) {
                        minv[t] = cur;
                        way[t] = j0;
                    }
                }
            }
            int j1;
            bool j1free;
            double delta;
            warp_argmin<CPL>(minv, used, p, lane, j1, j1free, delta);
#pragma unroll
            for (int t = 0; t < CPL; t++) {
                if (used[t]) {
                    ucol[t] += delta;
                    v[t] -= delta;
                } else {
                    minv[t] -= delta;
                }
            }
            ucur += delta;
#pragma unroll
            for (int t = 0; t < CPL; t++)
                if (lane + 32 * t == j1) used[t] = true;
            steps++;
            if (j1free) {
                jfree = j1;
                break;
            }
            const int src = j1 & 31, tt = j1 >> 5;
            i0 = __shfl_sync(FULL_MASK, sel_t<CPL>(p, tt), src);
            ui0 = __shfl_sync(FULL_MASK, sel_t<CPL>(ucol, tt), src);
            j0 = j1;
        }
        // augment along way[]: columns on the path take the row (and its u) of way[c]
        bool onp[CPL];
#pragma unroll
        for (int t = 0; t < CPL; t++) onp[t] = false;
        int c = jfree;
        while (c >= 0) {
            const int src = c & 31, tt = c >> 5;
#pragma unroll
            for (int t = 0; t < CPL; t++)
                if (lane == src && t == tt) onp[t] = true;
            c = __shfl_sync(FULL_MASK, sel_t<CPL>(way, tt), src);
        }
        int pold[CPL];
        double uold[CPL];
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            pold[t] = p[t];
            uold[t] = ucol[t];
        }
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            const int w = way[t];
            const int wl = (w < 0 ? 0 : w) & 31, wt = w < 0 ? 0 : (w >> 5);
            int np = i;
            double nu = ucur;
#pragma unroll
            for (int s = 0; s < CPL; s++) {
                const int sp = __shfl_sync(FULL_MASK, pold[s], wl);
                const double su = __shfl_sync(FULL_MASK, uold[s], wl);
                if (w >= 0 && wt == s) {
                    np = sp;
                    nu = su;
                }
            }
            if (onp[t]) {
                p[t] = np;
                ucol[t] = nu;
            }
        }
    }
}

// Residual (reading R8) to global + primal value S (reading R9).  Returns S (all lanes)
// and sets `bad` if some residual fell below -tau.
template <int CPL>
__device__ __forceinline__ double warp_lap_epilogue(const double *__restrict__ M, int m, int lane,
                                                    const int (&p)[CPL], const double (&v)[CPL],
                                                    const double (&ucol)[CPL], double *urow, double *sel,
                                                    double *__restrict__ R, bool &bad)
{
#pragma unroll
    for (int t = 0; t < CPL; t++) {
        const int c = lane + 32 * t;
        if (c < m) {
            urow[p[t]] = ucol[t];
            sel[p[t]] = M[p[t] * m + c];
        }
    }
    __syncwarp();
    double mx = 0.0, mn = 0.0;
    for (int r = 0; r < m; r++) {
        const double ur = urow[r];
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            const int c = lane + 32 * t;
            if (c < m) {
                const double a = M[r * m + c];
                mx = fmax(mx, fabs(a));
                double x = (a - ur) - v[t];
                mn = fmin(mn, x);
                if (x < 0.0) x = 0.0;
                if (p[t] == r) x = 0.0;
                if (x == 0.0) x = 0.0;  // canonical +0
                if (R != nullptr) R[r * m + c] = x;
            }
        }
    }
    double S = 0.0;
    if (lane == 0)
        for (int r = 0; r < m; r++) S = S + sel[r];  // sequential row order (reading R9)
    S = __shfl_sync(FULL_MASK, S, 0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, o));
        mn = fmin(mn, __shfl_xor_sync(FULL_MASK, mn, o));
    }
    const double tau = 1e-9 * fmax(1.0, mx);
    bad = mn < -tau;
    __syncwarp();
    return S;
}

// Shared-memory carve-up per warp: 2 × buffer (TMA destinations), urow[64], sel[64], 2 mbarriers.
__host__ __device__ inline size_t lap_buf_bytes(int64_t ld) { return ((size_t)ld * 8 + 127) & ~size_t(127); }
__host__ __device__ inline size_t lap_warp_smem(int64_t ld) { return 2 * lap_buf_bytes(ld) + 64 * 8 * 2 + 128; }

struct LapArgs {
    LapLevel lvl;
    Geom g;
    int m;
    int64_t count, ld;
    const double *src;
    double *dst;
    double *C, *B;
    Ctl *ctl;
    double *trace;
    LapBatchOut bo;
};

template <int CPL>
__global__ void __launch_bounds__(256) k_lap(const LapArgs a)
{
    if (a.ctl != nullptr && a.ctl->stopped) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int wpc = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t bufb = lap_buf_bytes(a.ld);
    unsigned char *base = smem + (size_t)warp * lap_warp_smem(a.ld);
    double *buf[2] = {reinterpret_cast<double *>(base), reinterpret_cast<double *>(base + bufb)};
    double *urow = reinterpret_cast<double *>(base + 2 * bufb);
    double *sel = urow + 64;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sel + 64);

    const int64_t nw = (int64_t)gridDim.x * wpc;
    int64_t b = (int64_t)blockIdx.x * wpc + warp;
    if (b >= a.count) return;
    const int m = a.m;
    const uint32_t bytes = (uint32_t)(((int64_t)m * m + 1) & ~int64_t(1)) * 8u;
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
        mbar_expect_tx(&mbar[0], bytes);
        tma_load_1d(buf[0], a.src + b * a.ld, bytes, &mbar[0]);
    }
    __syncwarp();

    int icur = 0;  // canonical first facility of block b (L2), advanced monotonically
    bool anybad = false;
    for (int it = 0; b < a.count; b += nw, it++) {
        const int64_t nb = b + nw;
        if (lane == 0 && nb < a.count) {
            fence_proxy_async();
            mbar_expect_tx(&mbar[(it + 1) & 1], bytes);
            tma_load_1d(buf[(it + 1) & 1], a.src + nb * a.ld, bytes, &mbar[(it + 1) & 1]);
        }
        mbar_wait(&mbar[it & 1], (it >> 1) & 1);
        const double *M = buf[it & 1];

        int p[CPL];
        double v[CPL], ucol[CPL];
        int steps = 0;
        warp_lap_solve<CPL>(M, m, lane, p, v, ucol, steps);
        bool bad;
        const double S = warp_lap_epilogue<CPL>(M, m, lane, p, v, ucol, urow, sel,
                                                 a.dst ? a.dst + b * a.ld : nullptr, bad);
        anybad |= bad;

        if (lane == 0) {
            switch (a.lvl) {
            case LAP_L2: {  // credit S to both complementary coefficients (reading R12)
                const Geom &g = a.g;
                while (icur + 1 < g.n && b >= g.off[icur + 1]) icur++;
                const int n = g.n, n1 = n - 1;
                int64_t rem = b - g.off[icur];
                const int per_j = (n1 - icur) * n1;
                const int j = (int)(rem / per_j);
                rem -= (int64_t)j * per_j;
                const int kk = (int)(rem / n1);
                const int li = (int)(rem - (int64_t)kk * n1);
                const int i = icur, k = i + 1 + kk, l = li + (li >= j);
                // C was spread to D and zeroed: c <- 0 + S = S.
                a.C[(int64_t)(i * n + j) * g.ldc + (k - 1) * n1 + (l - (l > j))] = S;
                a.C[(int64_t)(k * n + l) * g.ldc + i * n1 + (j - (j > l))] = S;
                break;
            }
            case LAP_L1_ACC: a.B[b] = a.B[b] + S; break;
            case LAP_L1_SET: a.B[b] = S; break;  // B was spread and zeroed: 0 + S = S
            case LAP_L0_ITER0:
            case LAP_L0: {
                Ctl *c = a.ctl;
                c->lb_dual = c->lb_dual + S;
                const double lb = (double)c->kappa + c->lb_dual;
                c->lb = lb;
                const bool ubf = isfinite(c->UB);
                if (a.lvl == LAP_L0_ITER0) {
                    c->lb_glb = lb;
                    if (ubf && lb > c->UB - 1.0 + 1e-6) {
                        c->status = 2;
                        c->stopped = 1;
                    }
                } else {
                    c->lbprime = S;
                    if (a.trace && c->iters < c->trace_cap) a.trace[c->iters] = lb;
                    c->iters += 1;
                    if (ubf) {
                        if (lb > c->UB - 1.0 + 1e-6) {
                            c->status = 2;
                            c->stopped = 1;
                        } else if (c->K > 0.0 && S / c->UB < c->K) {
                            c->status = 1;
                            c->stopped = 1;
                        }
                    }
                }
                break;
            }
            case LAP_BATCH:
                if (a.bo.S) a.bo.S[b] = S;
                if (a.bo.steps) a.bo.steps[b] = steps;
                break;
            }
        }
        if (a.lvl == LAP_BATCH) {
#pragma unroll
            for (int t = 0; t < CPL; t++) {
                const int c = lane + 32 * t;
                if (c < m) {
                    if (a.bo.assign) a.bo.assign[b * m + p[t]] = c;
                    if (a.bo.u) a.bo.u[b * m + p[t]] = ucol[t];
                    if (a.bo.v) a.bo.v[b * m + c] = v[t];
                }
            }
        }
        __syncwarp();
    }
    if (anybad && lane == 0) {
        if (a.ctl) atomicOr(&a.ctl->err, 1);
        if (a.bo.err) atomicOr(a.bo.err, 1);
    }
}

// ---------------------------------------------------------------------------------------
// k_init — O0/O1: b0 with the fixed-free folds, c_ij[kl] = f'_ik d'_jl,
// kappa; D is NOT written (the next transfer reads it as zero).
// ---------------------------------------------------------------------------------------
__global__ void k_init(const Node nd, const Geom g, const int64_t *__restrict__ F,
                       const int64_t *__restrict__ Dist, double *B, double *C, Ctl *ctl)
{
    const int N = nd.N, n = nd.n, n1 = n - 1;
    const int64_t n4 = (int64_t)n * n * n * n;
    const int64_t tot = n4 + (int64_t)n * n;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
        if (x < n4) {
            const int l = (int)(x % n), k = (int)((x / n) % n), j = (int)((x / n / n) % n), i = (int)(x / n / n / n);
            if (k == i || l == j) continue;
            const int64_t f = F[nd.I[i] * N + nd.I[k]], d = Dist[nd.J[j] * N + nd.J[l]];
            C[(int64_t)(i * n + j) * g.ldc + (k - (k > i)) * n1 + (l - (l > j))] = (double)(f * d);
        } else {
            const int y = (int)(x - n4), a_ = y / n, b_ = y % n;
            const int Ia = nd.I[a_], Jb = nd.J[b_];
            int64_t v = F[Ia * N + Ia] * Dist[Jb * N + Jb];
            for (int t = 0; t < nd.m; t++)
                v += F[nd.fac[t] * N + Ia] * Dist[nd.loc[t] * N + Jb] + F[Ia * N + nd.fac[t]] * Dist[Jb * N + nd.loc[t]];
            B[y] = (double)v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        long long kap = 0;
        for (int t = 0; t < nd.m; t++)
            for (int t2 = 0; t2 < nd.m; t2++) kap += F[nd.fac[t] * N + nd.fac[t2]] * Dist[nd.loc[t] * N + nd.loc[t2]];
        ctl->kappa = kap;
        ctl->lb_dual = 0.0;
        ctl->lbprime = 0.0;
        ctl->lb = (double)kap;
        ctl->lb_glb = (double)kap;
        ctl->iters = 0;
        ctl->status = 0;
        ctl->stopped = 0;
        ctl->err = 0;
    }
}

__global__ void k_ctl_begin(Ctl *ctl, double K, double UB, int trace_cap)
{
    ctl->K = K;
    ctl->UB = UB;
    ctl->iters = 0;
    ctl->status = 0;
    ctl->stopped = 0;
    ctl->trace_cap = trace_cap;
}

// ---------------------------------------------------------------------------------------
// k_sigma — spreading B->C fused with the C->D spread amount (reading
// R12): for each stored block D{ij,kl},
//   sigma = ((c_ij[kl] + b_ij/(n-1)) + (c_kl[ij] + b_kl/(n-1))) / (2(n-2)).
// B and C are then logically zero; both are fully overwritten later in the iteration.
// ---------------------------------------------------------------------------------------
__global__ void k_sigma(const Geom g, const double *__restrict__ B, const double *__restrict__ C,
                        double *__restrict__ sigma, const Ctl *ctl)
{
    if (ctl->stopped) return;
    const int n = g.n, n1 = n - 1;
    const int64_t n4 = (int64_t)n * n * n * n;
    const double div1 = (double)(n - 1), div2 = (double)(2 * (n - 2));
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n4; x += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(x % n), k = (int)((x / n) % n), j = (int)((x / n / n) % n), i = (int)(x / n / n / n);
        if (k <= i || l == j) continue;
        const double bij = B[i * n + j] / div1, bkl = B[k * n + l] / div1;
        const double c1 = C[(int64_t)(i * n + j) * g.ldc + (k - 1) * n1 + (l - (l > j))] + bij;
        const double c2 = C[(int64_t)(k * n + l) * g.ldc + i * n1 + (j - (j > l))] + bkl;
        sigma[bid_of(g, i, j, k, l)] = (c1 + c2) / div2;
    }
}

// ---------------------------------------------------------------------------------------
// k_transfer — spreading C->D fused with the transfer between complementary costs of D
// (reading R11: arithmetic mean of the class).  The class
// {(i,j),(k,l),(p,q)}, i<k<p, has stored members
//   e1 = D{ij,kl}[p-2][q'],  e2 = D{ij,pq}[k-1][l'],  e3 = D{kl,pq}[i][j']
// (primes: column index skipping the block's two locations).  A CTA owns one facility
// triple and an 8×8×8 tile of (j,l,q): each view is read as runs of <= 8 contiguous
// doubles along its own contiguous index, transposed through shared memory, averaged,
// and written back the same way — every stored entry is read once and written once.
// ---------------------------------------------------------------------------------------
constexpr int TT = 8;

__global__ void __launch_bounds__(256) k_transfer(const Geom g, double *__restrict__ D,
                                                  const double *__restrict__ sigma, int d_zero, const Ctl *ctl,
                                                  int ntile)
{
    if (ctl->stopped) return;
    __shared__ double s1[TT * TT * TT], s2[TT * TT * TT], s3[TT * TT * TT];
    const int n = g.n, m2 = n - 2;
    const int64_t ld2 = g.ld2;
    int i = 0, k, p;
    {
        int rem = blockIdx.y;
        while (true) {
            const int c = (n - 1 - i) * (n - 2 - i) / 2;
            if (rem < c) break;
            rem -= c;
            i++;
        }
        k = i + 1;
        while (true) {
            const int c = n - 1 - k;
            if (rem < c) break;
            rem -= c;
            k++;
        }
        p = k + 1 + rem;
    }
    const int tile = blockIdx.x;
    const int q0 = (tile % ntile) * TT, l0 = ((tile / ntile) % ntile) * TT, j0 = (tile / (ntile * ntile)) * TT;

    for (int e = threadIdx.x; e < TT * TT * TT; e += blockDim.x) {
        const int a = e >> 6, b = (e >> 3) & 7, c = e & 7;
        {  // view 1: (j,l,q) = (a,b,c); contiguous along q
            const int j = j0 + a, l = l0 + b, q = q0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q) {
                const int64_t bb = bid_of(g, i, j, k, l);
                const double x = d_zero ? 0.0 : D[bb * ld2 + (int64_t)(p - 2) * m2 + (q - (q > j) - (q > l))];
                s1[e] = x + sigma[bb];
            }
        }
        {  // view 2: (j,q,l) = (a,b,c); contiguous along l
            const int j = j0 + a, q = q0 + b, l = l0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q) {
                const int64_t bb = bid_of(g, i, j, p, q);
                const double x = d_zero ? 0.0 : D[bb * ld2 + (int64_t)(k - 1) * m2 + (l - (l > j) - (l > q))];
                s2[e] = x + sigma[bb];
            }
        }
        {  // view 3: (l,q,j) = (a,b,c); contiguous along j
            const int l = l0 + a, q = q0 + b, j = j0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q) {
                const int64_t bb = bid_of(g, k, l, p, q);
                const double x = d_zero ? 0.0 : D[bb * ld2 + (int64_t)i * m2 + (j - (j > l) - (j > q))];
                s3[e] = x + sigma[bb];
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TT * TT * TT; e += blockDim.x) {
        const int a = e >> 6, b = (e >> 3) & 7, c = e & 7;  // (j,l,q) offsets
        const int j = j0 + a, l = l0 + b, q = q0 + c;
        if (j < n && l < n && q < n && j != l && j != q && l != q) {
            const int e1 = e, e2 = (a << 6) | (c << 3) | b, e3 = (b << 6) | (c << 3) | a;
            const double mu = ((s1[e1] + s2[e2]) + s3[e3]) / 3.0;
            s1[e1] = mu;
            s2[e2] = mu;
            s3[e3] = mu;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TT * TT * TT; e += blockDim.x) {
        const int a = e >> 6, b = (e >> 3) & 7, c = e & 7;
        {
            const int j = j0 + a, l = l0 + b, q = q0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q)
                D[bid_of(g, i, j, k, l) * ld2 + (int64_t)(p - 2) * m2 + (q - (q > j) - (q > l))] = s1[e];
        }
        {
            const int j = j0 + a, q = q0 + b, l = l0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q)
                D[bid_of(g, i, j, p, q) * ld2 + (int64_t)(k - 1) * m2 + (l - (l > j) - (l > q))] = s2[e];
        }
        {
            const int l = l0 + a, q = q0 + b, j = j0 + c;
            if (j < n && l < n && q < n && j != l && j != q && l != q)
                D[bid_of(g, k, l, p, q) * ld2 + (int64_t)i * m2 + (j - (j > l) - (j > q))] = s3[e];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------------------
cudaError_t launch_init(const Node &node, const Geom &g, const int64_t *F, const int64_t *Dist, double *B,
                        double *C, Ctl *ctl, cudaStream_t st)
{
    const int64_t tot = (int64_t)g.n * g.n * g.n * g.n + (int64_t)g.n * g.n;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_init<<<blocks, 256, 0, st>>>(node, g, F, Dist, B, C, ctl);
    return cudaGetLastError();
}

cudaError_t launch_ctl_begin(Ctl *ctl, double K, double UB, int trace_cap, cudaStream_t st)
{
    k_ctl_begin<<<1, 1, 0, st>>>(ctl, K, UB, trace_cap);
    return cudaGetLastError();
}

cudaError_t launch_sigma(const Geom &g, const double *B, const double *C, double *sigma, const Ctl *ctl,
                         cudaStream_t st)
{
    const int64_t tot = (int64_t)g.n * g.n * g.n * g.n;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_sigma<<<blocks, 256, 0, st>>>(g, B, C, sigma, ctl);
    return cudaGetLastError();
}

cudaError_t launch_transfer(const Geom &g, double *D, const double *sigma, int d_zero, const Ctl *ctl,
                            cudaStream_t st)
{
    const int n = g.n;
    const int ntile = (n + TT - 1) / TT;
    const int ntri = n * (n - 1) * (n - 2) / 6;
    dim3 grid(ntile * ntile * ntile, ntri);
    k_transfer<<<grid, 256, 0, st>>>(g, D, sigma, d_zero, ctl, ntile);
    return cudaGetLastError();
}

template <int CPL>
static cudaError_t launch_lap_on(const LapArgs &a, int num_sms, int wpc, cudaStream_t st)
{
    const size_t smem = lap_warp_smem(a.ld) * wpc;
    cudaError_t e = cudaFuncSetAttribute(k_lap<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lap<CPL>, 32 * wpc, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t want = (a.count + wpc - 1) / wpc;
    const int64_t cap = (int64_t)num_sms * per_sm;
    const int grid = (int)(want < cap ? want : cap);
    k_lap<CPL><<<grid, 32 * wpc, smem, st>>>(a);
    return cudaGetLastError();
}

static int pick_wpc(int64_t ld, int requested)
{
    const size_t per = lap_warp_smem(ld);
    int w = requested > 0 ? requested : 4;
    while (w > 1 && per * w > 200 * 1024) w--;
    return w;
}

static cudaError_t dispatch_lap(const LapArgs &a, int num_sms, int wpc, cudaStream_t st)
{
    if (a.m <= 32) return launch_lap_on<1>(a, num_sms, wpc, st);
    if (a.m <= 64) return launch_lap_on<2>(a, num_sms, wpc, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_lap_level(LapLevel lvl, const Geom &g, double *D, double *C, double *B, Ctl *ctl,
                             double *trace, int num_sms, int lap_warps, cudaStream_t st)
{
    LapArgs a{};
    a.lvl = lvl;
    a.g = g;
    a.C = C;
    a.B = B;
    a.ctl = ctl;
    a.trace = trace;
    const int n = g.n;
    int wpc = 1;
    switch (lvl) {
    case LAP_L2:
        a.m = n - 2; a.count = g.nblk; a.ld = g.ld2; a.src = D; a.dst = D;
        wpc = pick_wpc(a.ld, lap_warps);
        break;
    case LAP_L1_ACC:
    case LAP_L1_SET:
        a.m = n - 1; a.count = (int64_t)n * n; a.ld = g.ldc; a.src = C; a.dst = C;
        wpc = pick_wpc(a.ld, 2);
        break;
    case LAP_L0_ITER0:
    case LAP_L0:
        a.m = n; a.count = 1; a.ld = ((int64_t)n * n + 1) & ~int64_t(1); a.src = B; a.dst = B;
        wpc = 1;
        break;
    default: return cudaErrorInvalidValue;
    }
    return dispatch_lap(a, num_sms, wpc, st);
}

cudaError_t launch_lap_batch(int m, int64_t count, int64_t ld, const double *M, const LapBatchOut &o, int num_sms,
                             cudaStream_t st)
{
    LapArgs a{};
    a.lvl = LAP_BATCH;
    a.m = m;
    a.count = count;
    a.ld = ld;
    a.src = M;
    a.dst = o.R;
    a.bo = o;
    a.ctl = nullptr;
    return dispatch_lap(a, num_sms, pick_wpc(ld, 4), st);
}

}  // namespace rlt2
