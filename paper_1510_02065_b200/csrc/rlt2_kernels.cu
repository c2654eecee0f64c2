// rlt2_kernels.cu — sm_100a kernels of the RLT2 dual-ascent bound.
//
// P:n = /root/reference/PAPER.md line n.  Readings R1..R31 are listed in DESIGN.md §3.
//
//   k_init          O0/O1: reduced costs of the node            HBM write of B, C
//   k_sigma         spreading B->C and the per-block C->D spread amount
//   k_transfer_tma  spreading C->D fused with the transfer between complementary
//                   costs of D: one CTA per facility triple and
//                   8x8x8 location tile, the three member views as tensor-map TMA boxes
//   k_transfer      the same with register loads (small nodes, sharded handles)
//   k_lap<CPL>      cost concentration: one warp per LAP, the cost
//                   block staged global->smem by a TMA bulk copy and stored back by one;
//                   Munkres row reduction, then shortest augmenting paths (Jonker-Volgenant
//                   form) with lane = column, argmin by a signed redux.sync on the raw
//                   fp64 high word (the low word and the order-preserving key only on ties
//                   or negative values)                                        issue-bound
//   k_fold_*, k_rlt1_*, k_credit: warm children, strong branching, sharded credit
//
// Arithmetic order follows DESIGN.md §3 exactly (same IEEE operations as the paper's
// algorithm written out), so results are reproducible bit for bit; no multiplies
// occur in fp64 after initialisation (compiled with -fmad=false regardless).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>

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
// 4-D tensor-map TMA load of one box (coordinates in elements, dim0 innermost)
__device__ __forceinline__ void tma_load_4d(void *dst, const void *tmap, int c0, int c1, int c2, int c3,
                                            uint64_t *mbar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity)
{
    uint32_t done = 0, spins = 0;
    while (!done) {
        if (++spins > (1u << 28)) __trap();  // a lost TMA transaction: fail, never hang
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_store_1d(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

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

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// The warp LAP solver (reading R4/R5/R6).  Lane `lane` owns columns
// c = lane + 32 t (t < CPL).  Per column, in registers: v (dual), ucol = u of the row
// matched to the column, poff = byte offset of that row in the smem cost block (-1: free),
// minv / way of the current Dijkstra search.  A settled ("used") column carries
// minv = NaN: `cur < NaN` is false, NaN's order key sorts after every number, and
// `NaN - delta` stays NaN, so the scan and the argmin need no used-test.  The dummy
// column of the textbook formulation (holding the row being inserted) lives in
// warp-uniform registers (ucur).  Every floating-point operation and its order is the
// written-out algorithm of DESIGN.md §3 (O2), so results are reproducible bit for bit.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// Munkres' row reduction (reading R4, oracle O2): u_r = min_s M[r][s] for every row,
// v = 0, and the initial partial assignment on the zeros this creates — row r takes the
// lowest column attaining its minimum unless a lower row took that column.  Lane `lane`
// scans rows lane + 32 u (a row of a lane without one: row 0, unused); `col[t]` is the column
// of the lane's owned slot t.  Returns the row minima (rmin[u] of row lane + 32 u), the masks
// of matched rows (bit r & 31 of rmask[r >> 5]) and, per owned column, poff / ucol of its
// matched row (-1 / 0 when free).  `colrow` is m ints of per-warp shared scratch.
template <int CPL>
__device__ __forceinline__ void munkres_init(const double *M, int m, int lane, const int (&col)[CPL], int *colrow,
                                             int (&poff)[CPL], double (&ucol)[CPL], double (&rmin)[CPL],
                                             uint32_t (&rmask)[CPL])
{
    const int rowb = m * 8;
    int rarg[CPL];
#pragma unroll
    for (int u = 0; u < CPL; u++) {
        const int r = lane + 32 * u;
        const double *rp = M + (r < m ? r : 0) * m;
        double mn = rp[0];
        int am = 0;
#pragma unroll 4
        for (int c = 1; c < m; c++) {  // strict <: the lowest column among equal minima
            const double x = rp[c];
            if (x < mn) {
                mn = x;
                am = c;
            }
        }
        rmin[u] = mn;
        rarg[u] = am;
    }
#pragma unroll
    for (int t = 0; t < CPL; t++)
        if (col[t] < m) colrow[col[t]] = -1;
    __syncwarp();
    // one writer per column within a group of 32 rows (the lowest lane of each match group);
    // the lower group writes last, so the lowest row holding a column's minimum keeps it
#pragma unroll
    for (int u = CPL - 1; u >= 0; u--) {
        const int r = lane + 32 * u;
        const uint32_t grp = __match_any_sync(FULL_MASK, r < m ? rarg[u] : 64 + lane);
        if (r < m && (grp & ((1u << lane) - 1u)) == 0u) colrow[rarg[u]] = r;
        __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < CPL; u++) {
        const int r = lane + 32 * u;
        rmask[u] = __ballot_sync(FULL_MASK, r < m && colrow[rarg[u]] == r);
    }
#pragma unroll
    for (int t = 0; t < CPL; t++) {
        const int r = col[t] < m ? colrow[col[t]] : -1;
        const int src = r < 0 ? 0 : r;
        double ur = __shfl_sync(FULL_MASK, rmin[0], src & 31);
        if (CPL > 1) {
            const double ur1 = __shfl_sync(FULL_MASK, rmin[CPL - 1], src & 31);
            if (src >= 32) ur = ur1;
        }
        poff[t] = r < 0 ? -1 : r * rowb;
        ucol[t] = r < 0 ? 0.0 : ur;
    }
    __syncwarp();  // the scratch is free again
}

// One column per lane (m <= 32): Munkres' row reduction (munkres_init), then the rows left are
// inserted in ascending order, each by one shortest-augmenting-path search (Dijkstra with
// absolute tentative distances; the potentials move once, after the search).  Column c is
// held by lane 31 - c, so that "lowest column index" is the highest set lane bit (one FLO).  The
// argmin takes the order key's high word first (the low word only on ties, a warp-uniform
// branch), then prefers a free column (a lane mask updated once per augmentation), then
// the lowest column; way[] and the augmenting path (one lane mask) are in lane ids.
__device__ __forceinline__ uint32_t tie_low_word(double minv, uint32_t sg, uint32_t hi, uint32_t mhi)
{
    const uint32_t lo = static_cast<uint32_t>(__double2loint(minv)) ^ sg;
    const uint32_t mlo = __reduce_min_sync(FULL_MASK, hi == mhi ? lo : 0xffffffffu);
    return __ballot_sync(FULL_MASK, hi == mhi && lo == mlo);
}
// index of the highest set bit (bfind: one FLO, so that merged values stay FLO results)
__device__ __forceinline__ int hibit(uint32_t x)
{
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
// the argmin's ballot through the full order-preserving key (some minv is negative or -0)
__device__ __noinline__ uint32_t argmin_keyed(double minv)
{
    const uint32_t hb = static_cast<uint32_t>(__double2hiint(minv));
    const uint32_t sg = static_cast<uint32_t>(static_cast<int32_t>(hb) >> 31);
    const uint32_t hi = hb ^ (sg | 0x80000000u);
    const uint32_t mhi = __reduce_min_sync(FULL_MASK, hi);
    uint32_t bal = __ballot_sync(FULL_MASK, hi == mhi);
    if (bal & (bal - 1u)) bal = tie_low_word(minv, sg, hi, mhi);
    return bal;
}
template <bool COUNT>
__device__ __forceinline__ void warp_lap_solve1(const double *M, int m, int lane, int *scratch, int &poff, double &v,
                                                double &ucol, int &steps)
{
    const double *Mlane = M + (31 - lane);
    v = 0.0;
    int way = -1;
    const int rowb = m * 8;  // bytes per cost row
    double minv0 = 31 - lane < m ? CUDART_INF : qnan();
    asm("" : "+d"(minv0));  // keep it in registers (not rematerialised per row)
    int pc[1], col[1] = {31 - lane};
    double uc[1], rm[1];
    uint32_t rmask[1];
    munkres_init<1>(M, m, lane, col, scratch, pc, uc, rm, rmask);
    poff = pc[0];
    ucol = uc[0];
    const double rmin = rm[0];
    // lanes 32-m .. 31 hold columns; those matched by the row reduction are taken
    uint32_t freemask = (m >= 32 ? 0xffffffffu : ~((1u << (32 - m)) - 1u)) & ~__ballot_sync(FULL_MASK, poff >= 0);
    // the rows the row reduction left unmatched, ascending (P:205 Hungarian, one augmentation
    // per row)
    for (uint32_t um = ~rmask[0] & (m >= 32 ? 0xffffffffu : ((1u << m) - 1u)); um; um &= um - 1u) {
        const int i = __ffs(um) - 1;
        const double ui = __shfl_sync(FULL_MASK, rmin, i);  // u of row i: its row minimum
        // Dijkstra from row i with absolute tentative distances (minv); the scanned row i0
        // enters as c = dist(its column) - u[i0]; potentials move once, after the search
        double minv = minv0, c = 0.0 - ui;
        uint32_t dhi = 0xffffffffu;  // settled: high word of the column's distance (low word stays in minv)
        int j0 = -1, i0off = i * rowb, j1;
#pragma unroll 2
        for (;;) {
            const double cur = (*reinterpret_cast<const double *>(reinterpret_cast<const char *>(Mlane) + i0off) - v) + c;
            if (cur < minv) {  // false for settled columns (minv = NaN)
                minv = cur;
                way = j0;
            }
            const double cj = minv - ucol;  // lane j1 (below): dist[j1] - u[p[j1]], the next row's offset
            // argmin of (minv, matched?, column).  While no minv is negative (Dijkstra
            // distances are >= 0 up to rounding; settled columns hold +NaN) the raw high words
            // order the values as signed integers (and equal high words by their low words as
            // unsigned): one signed redux on the common path; a negative minimum (a negative
            // value or -0 somewhere) takes the order-preserving key (warp-uniform branch).
            const int32_t hs = __double2hiint(minv);
            const int32_t mhs = __reduce_min_sync(FULL_MASK, hs);
            uint32_t bal = __ballot_sync(FULL_MASK, hs == mhs);
            j1 = hibit(bal);  // a unique minimum (the common case): the next column
            if (mhs < 0 || (bal & (bal - 1u))) {  // several minima (or a negative one)
                bal = mhs < 0 ? argmin_keyed(minv) : tie_low_word(minv, 0u, (uint32_t)hs, (uint32_t)mhs);
                const uint32_t fb = bal & freemask;
                j1 = hibit(fb ? fb : bal);  // a free column first; highest lane = lowest column
            }
            const uint32_t ft = bal & freemask;
            const double nc = __shfl_sync(FULL_MASK, cj, j1);
            const int nx_off = __shfl_sync(FULL_MASK, poff, j1);
            if (lane == j1) {  // settle column j1: keep its distance's high word, NaN in minv
                dhi = static_cast<uint32_t>(__double2hiint(minv));
                minv = __hiloint2double(0x7ff80000, __double2loint(minv));
            }
            if (COUNT) steps++;
            if (ft) break;
            i0off = nx_off;
            c = nc;
            j0 = j1;
        }
        // potentials: every column settled in this search moves by dfin - dist (the free end
        // column by +0); row i's u by dfin
        const double dfin = __shfl_sync(FULL_MASK, __hiloint2double(static_cast<int>(dhi), __double2loint(minv)), j1);
        if (dhi != 0xffffffffu) {
            const double t = dfin - __hiloint2double(static_cast<int>(dhi), __double2loint(minv));
            ucol = ucol + t;
            v = v - t;
        }
        const double ucur = ui + dfin;
        // augment along way[]: columns on the path take the row (and its u) of way[c]
        freemask &= ~(1u << j1);
        uint32_t onmask = 0u;
        for (int c = j1; c >= 0; c = __shfl_sync(FULL_MASK, way, c)) onmask |= 1u << c;
        const int sp = __shfl_sync(FULL_MASK, poff, way);
        const double su = __shfl_sync(FULL_MASK, ucol, way);
        if ((onmask >> lane) & 1u) {
            poff = way >= 0 ? sp : i * rowb;
            ucol = way >= 0 ? su : ucur;
        }
    }
}

// Two columns per lane (32 < m <= 64): column 32 t + 31 - lane in slot t (the one-column
// solver's reversed order, so the lowest column of a slot is the highest lane: one bfind).
// The same algorithm and floating-point operations as warp_lap_solve1.  Argmin on the common
// path: one signed redux per slot on the raw fp64 high words (non-negative values order as
// signed integers, settled columns hold +NaN); when the two slot minima differ and one lane
// holds the smaller, that lane's column is the minimum; every other case (equal high words,
// a negative value) takes argmin2_keyed, the full (value, matched?, column) order.
__device__ __noinline__ int argmin2_keyed(double m0, double m1, int p0, int p1, int lane)
{
    const uint64_t k0 = okey(m0), k1 = okey(m1);
    const int r0 = p0 >= 0 ? 1 : 0, r1 = p1 >= 0 ? 1 : 0;
    // slot 0 holds the lower column, so it wins equal (key, matched?)
    const bool s1 = k1 < k0 || (k1 == k0 && r1 < r0);
    const uint64_t key = s1 ? k1 : k0;
    const uint32_t rank = static_cast<uint32_t>(s1 ? r1 : r0);
    const uint32_t col = static_cast<uint32_t>((s1 ? 63 : 31) - lane);
    const uint32_t hi = static_cast<uint32_t>(key >> 32), lo = static_cast<uint32_t>(key);
    const uint32_t mhi = __reduce_min_sync(FULL_MASK, hi);
    const uint32_t mlo = __reduce_min_sync(FULL_MASK, hi == mhi ? lo : 0xffffffffu);
    const bool tie = hi == mhi && lo == mlo;
    const uint32_t mr = __reduce_min_sync(FULL_MASK, tie ? rank : 0xffu);
    return static_cast<int>(__reduce_min_sync(FULL_MASK, (tie && rank == mr) ? col : 0xffu));
}
template <bool COUNT>
__device__ __forceinline__ void warp_lap_solve2(const double *M, int m, int lane, int *scratch, int (&poff)[2],
                                                double (&v)[2], double (&ucol)[2], int &steps)
{
    const double *Mlane = M + (31 - lane);  // slot 0; slot 1 is 32 doubles further
    const int rowb = m * 8;
    v[0] = v[1] = 0.0;
    int way0 = -1, way1 = -1;  // predecessor column of each owned column
    const double minv00 = CUDART_INF, minv01 = 63 - lane < m ? CUDART_INF : qnan();
    int col[2] = {31 - lane, 63 - lane};
    double rm[2];
    uint32_t rmask[2];
    munkres_init<2>(M, m, lane, col, scratch, poff, ucol, rm, rmask);
    uint64_t um = ~(static_cast<uint64_t>(rmask[0]) | (static_cast<uint64_t>(rmask[1]) << 32));
    if (m < 64) um &= (1ull << m) - 1ull;
    // the rows the row reduction left unmatched, ascending (P:205 Hungarian, one augmentation
    // per row)
    for (; um; um &= um - 1ull) {
        const int i = __ffsll(static_cast<long long>(um)) - 1;
        const double ui = __shfl_sync(FULL_MASK, i < 32 ? rm[0] : rm[1], i & 31);
        double minv0 = minv00, minv1 = minv01, c = 0.0 - ui;
        uint32_t dhi0 = 0xffffffffu, dhi1 = 0xffffffffu;
        int j0 = -1, i0off = i * rowb, jcol, jl, jt;
#pragma unroll 2
        for (;;) {
            const double *row = reinterpret_cast<const double *>(reinterpret_cast<const char *>(Mlane) + i0off);
            const double cur0 = (row[0] - v[0]) + c, cur1 = (row[32] - v[1]) + c;
            if (cur0 < minv0) {  // false for settled columns (minv = NaN)
                minv0 = cur0;
                way0 = j0;
            }
            if (cur1 < minv1) {
                minv1 = cur1;
                way1 = j0;
            }
            const double cj0 = minv0 - ucol[0], cj1 = minv1 - ucol[1];  // dist - u of the column's row
            const int32_t hs0 = __double2hiint(minv0), hs1 = __double2hiint(minv1);
            const int32_t m0 = __reduce_min_sync(FULL_MASK, hs0), m1 = __reduce_min_sync(FULL_MASK, hs1);
            bool uniq = false;
            if (m0 >= 0 && m1 >= 0 && m0 != m1) {
                const bool t1 = m1 < m0;
                const uint32_t bal = __ballot_sync(FULL_MASK, (t1 ? hs1 : hs0) == (t1 ? m1 : m0));
                if (!(bal & (bal - 1u))) {
                    jcol = (t1 ? 63 : 31) - hibit(bal);
                    uniq = true;
                }
            }
            if (!uniq) jcol = argmin2_keyed(minv0, minv1, poff[0], poff[1], lane);
            jt = jcol >> 5;
            jl = 31 - (jcol & 31);
            const int nx_off = __shfl_sync(FULL_MASK, jt ? poff[1] : poff[0], jl);
            const double nc = __shfl_sync(FULL_MASK, jt ? cj1 : cj0, jl);
            // settle column jcol: keep its distance's high word, NaN in minv (selects, no branch)
            const bool me0 = lane == jl && jt == 0, me1 = lane == jl && jt != 0;
            dhi0 = me0 ? static_cast<uint32_t>(__double2hiint(minv0)) : dhi0;
            dhi1 = me1 ? static_cast<uint32_t>(__double2hiint(minv1)) : dhi1;
            minv0 = __hiloint2double(me0 ? 0x7ff80000 : __double2hiint(minv0), __double2loint(minv0));
            minv1 = __hiloint2double(me1 ? 0x7ff80000 : __double2hiint(minv1), __double2loint(minv1));
            if (COUNT) steps++;
            if (nx_off < 0) break;  // a free column: the augmenting path ends here
            i0off = nx_off;
            c = nc;
            j0 = jcol;
        }
        // potentials: every column settled in this search moves by dfin - dist (the free end
        // column by +0); row i's u by dfin
        const double d0 = __hiloint2double(static_cast<int>(dhi0), __double2loint(minv0)),
                     d1 = __hiloint2double(static_cast<int>(dhi1), __double2loint(minv1));
        const double dfin = __shfl_sync(FULL_MASK, jt ? d1 : d0, jl);
        if (dhi0 != 0xffffffffu) {
            const double tt = dfin - d0;
            ucol[0] = ucol[0] + tt;
            v[0] = v[0] - tt;
        }
        if (dhi1 != 0xffffffffu) {
            const double tt = dfin - d1;
            ucol[1] = ucol[1] + tt;
            v[1] = v[1] - tt;
        }
        const double ucur = ui + dfin;
        // augment along way[]: columns on the path take the row (and its u) of their
        // predecessor column; the path is walked once with warp-uniform values
        uint32_t on0 = 0u, on1 = 0u;
        for (int cc = jcol; cc >= 0;) {
            const int cl = 31 - (cc & 31);
            if (cc >> 5) on1 |= 1u << cl;
            else on0 |= 1u << cl;
            cc = __shfl_sync(FULL_MASK, (cc >> 5) ? way1 : way0, cl);
        }
        const int po0 = poff[0], po1 = poff[1];
        const double uo0 = ucol[0], uo1 = ucol[1];
#pragma unroll
        for (int t = 0; t < 2; t++) {
            const int w = t ? way1 : way0;
            const int wl = 31 - (w & 31);  // w < 0 (the inserted row): values unused below
            const int sp0 = __shfl_sync(FULL_MASK, po0, wl), sp1 = __shfl_sync(FULL_MASK, po1, wl);
            const double su0 = __shfl_sync(FULL_MASK, uo0, wl), su1 = __shfl_sync(FULL_MASK, uo1, wl);
            const int np = w < 0 ? i * rowb : ((w >> 5) ? sp1 : sp0);
            const double nu = w < 0 ? ucur : ((w >> 5) ? su1 : su0);
            if ((((t ? on1 : on0) >> lane) & 1u)) {
                poff[t] = np;
                ucol[t] = nu;
            }
        }
    }
}

// Residual (reading R8), written IN PLACE over the smem cost block, + primal value S
// (reading R9).  Returns S (all lanes) and sets `bad` if some residual fell below -tau.
// p[t] receives the matched row of each owned column.  One pass: the clamp to +0 is
// applied directly; since tau >= 1e-9, the exact tau test (which needs max|M|) is only
// evaluated when some raw residual is below -1e-9, from the original block: Mg(r, t, c)
// returns entry (r, c) from global memory, not yet overwritten — the residual is stored
// back after this returns (called by all lanes; c >= m: value unused).
// Rows of the cost buffer are ldm doubles apart; column c of owned slot t sits at offset
// cofs[t] within a row (the block layout: ldm = m, cofs = c).
template <int CPL, class GVal>
__device__ __forceinline__ double warp_lap_epilogue(double *M, GVal Mg, int m, int ldm, const int (&cofs)[CPL],
                                                    int lane, int col0, const int (&poff)[CPL], int (&p)[CPL],
                                                    const double (&v)[CPL], const double (&ucol)[CPL], double *urow,
                                                    double *sel, int ust, uint32_t rmag, bool &bad)
{
    // poff is a multiple of the row's bytes (8 ldm): the row by a multiply-high with rmag =
    // ceil(2^32 / (8 ldm)) (exact: poff < 2^32 / (8 ldm))
#pragma unroll
    for (int t = 0; t < CPL; t++) {
        const int c = col0 + 32 * t;
        p[t] = c < m ? (int)__umulhi((uint32_t)poff[t], rmag) : -1;
        if (c < m) {
            urow[p[t] * ust] = ucol[t];
            sel[p[t] * ust] = M[p[t] * ldm + cofs[t]];
        }
    }
    __syncwarp();
    // the largest raw high word as unsigned: a value at or above the high word of -1e-9 marks
    // a residual that may fall below -tau (every negative double with |x| >= 1e-9 has it; the
    // rare exact test below decides)
    uint32_t hmax = 0u;
#pragma unroll
    for (int t = 0; t < CPL; t++) {
        const int c = col0 + 32 * t;
        if (c < m) {
            double *Mc = M + cofs[t];
            const double vc = v[t];
#pragma unroll 4
            for (int r = 0; r < m; r++) {
                const double x = (Mc[r * ldm] - urow[r * ust]) - vc;
                // x <= 0 (incl. -0) -> +0, else x (== x > 0.0 ? x : 0.0 for every non-NaN x):
                // clear both words when the sign bit is set
                const int hi = __double2hiint(x), lo = __double2loint(x), keep = ~(hi >> 31);
                hmax = max(hmax, static_cast<uint32_t>(hi));
                Mc[r * ldm] = __hiloint2double(hi & keep, lo & keep);
            }
            Mc[p[t] * ldm] = 0.0;  // assigned cell -> +0
        }
    }
    double S = 0.0;
    if (lane == 0)
        for (int r = 0; r < m; r++) S = S + sel[r * ust];  // sequential row order (reading R9)
    S = __shfl_sync(FULL_MASK, S, 0);
    bad = false;
    if (__any_sync(FULL_MASK, hmax >= 0xBE112E0Bu)) {  // rare (hi(-1e-9)): exact test tau = 1e-9 max(1, max|M|)
        // recompute the raw residuals from the original block (same operations)
        double mx = 0.0, mn = 0.0;
#pragma unroll
        for (int t = 0; t < CPL; t++) {
            const int c = col0 + 32 * t;
            for (int r = 0; r < m; r++) {  // warp-uniform loop: Mg may shuffle
                const double g = Mg(r, t, c);
                if (c < m) {
                    const double x = (g - urow[r * ust]) - v[t];
                    mn = x < mn ? x : mn;
                    mx = fmax(mx, fabs(g));
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(FULL_MASK, mx, o));
            mn = fmin(mn, __shfl_xor_sync(FULL_MASK, mn, o));
        }
        bad = mn < -1e-9 * fmax(1.0, mx);
    }
    fence_proxy_async();  // residual (generic-proxy writes) -> visible to the TMA store
    __syncwarp();
    return S;
}

// Shared memory per warp: the cost buffer (TMA destination; m*m doubles plus 32*CPL - m
// doubles of padding so that every lane may load its column of any row unconditionally),
// urow[m], sel[m], one mbarrier — packed tightly so that 34 warps fit one SM at m = 28.
__host__ __device__ inline size_t lap_buf_bytes(int m, int cpl)
{
    // lanes without a column read entry (r, c >= m) of any row r: the block plus 32 cpl - m
    // doubles of padding keeps every such read inside the buffer
    const int pad = 32 * cpl > m ? 32 * cpl - m : 0;
    return (((size_t)m * m + pad) * 8 + 15) & ~size_t(15);
}
__host__ __device__ inline size_t lap_warp_smem(int m, int cpl)
{
    return lap_buf_bytes(m, cpl) + (((size_t)2 * m * 8 + 15) & ~size_t(15)) + 16;
}

// First (canonical) facility of stored block b; `hint` only moves forward.
__device__ __forceinline__ int facility_of(const Geom &g, int64_t b, int &hint)
{
    while (hint + 1 < g.n && b >= g.off[hint + 1]) hint++;
    return hint;
}

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
    Sched *sched;  // non-null: dynamic work queue (head reset by k_sigma)
    int64_t bdiv, bstr;  // level 1: B index of block b = (b / bdiv) * bstr + b % bdiv (batched RLT1)
    double *lbm;         // LAP_L0_MULTI: lbm[b] += S
    int chunk;           // dynamic mode: blocks per work-queue grab (set by the launcher)
    // level 2: x / d = umulhi(x, ceil(2^32 / d)) (exact for x d < 2^32) for d = n - 1 and
    // d = (n - 1 - i)(n - 1), the block-id decode of the S credit (no integer division)
    uint32_t mag_n1, mag_pj[kMaxN];
};
// Level 2: pairs (i,j), (k,l) of stored block b (i = canonical first facility; `icur` is a
// hint that only moves forward), packed i | j << 8 | k << 16 | l << 24.
__device__ __forceinline__ unsigned decode_l2(const LapArgs &a, int64_t b, int &icur)
{
    const Geom &g = a.g;
    facility_of(g, b, icur);
    const int n = g.n, n1 = n - 1;
    int rem = (int)(b - g.off[icur]);  // < n (n-1)^2
    const int per_j = (n1 - icur) * n1;
    const int j = (int)__umulhi((unsigned)rem, a.mag_pj[icur]);  // rem / per_j
    rem -= j * per_j;
    const int kk = (int)__umulhi((unsigned)rem, a.mag_n1);  // rem / n1
    const int li = rem - kk * n1;
    const int k = icur + 1 + kk, l = li + (li >= j);
    return (unsigned)icur | ((unsigned)j << 8) | ((unsigned)k << 16) | ((unsigned)l << 24);
}

// Control flow is kept provably warp-uniform for ptxas (warp index and the stop flag read
// through a shuffle): otherwise every redux/shfl of the solver is guarded by a BRA.DIV pair
// (~15% of the Dijkstra step's issue).
template <int CPL>
__global__ void __launch_bounds__(1024) k_lap(const LapArgs a)
{
    if (a.ctl != nullptr && __shfl_sync(FULL_MASK, a.ctl->stopped, 0)) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int wpc = blockDim.x >> 5, warp = __shfl_sync(FULL_MASK, (int)(threadIdx.x >> 5), 0),
              lane = threadIdx.x & 31;
    const int col0 = 31 - lane;  // this lane's column in slot 0 (slot t: col0 + 32 t)
    const int m = a.m;
    const size_t bufb = lap_buf_bytes(m, CPL);
    unsigned char *wbase = smem + (size_t)warp * lap_warp_smem(m, CPL);
    double *urow = reinterpret_cast<double *>(wbase + bufb);
    double *sel = urow + m;
    int *const scratch = reinterpret_cast<int *>(sel);  // the solver's row-reduction table (m ints)
    uint64_t *mbar = reinterpret_cast<uint64_t *>(wbase + bufb + (((size_t)2 * m * 8 + 15) & ~size_t(15)));

    const bool dyn = a.sched != nullptr;
    const int CH = a.chunk;  // blocks per work-queue grab (dynamic mode)
    const int64_t nw = (int64_t)gridDim.x * wpc;
    int64_t b, cend;
    if (dyn) {
        int64_t c0 = 0;
        if (lane == 0) c0 = (int64_t)atomicAdd(&a.sched->head, (unsigned long long)CH);
        b = __shfl_sync(FULL_MASK, c0, 0);
        cend = b + CH < a.count ? b + CH : a.count;
    } else {
        b = (int64_t)blockIdx.x * wpc + warp;
        cend = a.count;
    }
    if (b >= a.count) return;
    const uint32_t bytes = (uint32_t)(((int64_t)m * m + 1) & ~int64_t(1)) * 8u;
    const uint32_t rmag = (uint32_t)((0x100000000ull + (uint64_t)(m * 8) - 1ull) / (uint64_t)(m * 8));
    int icur = 0;  // canonical first facility of block b (L2), advanced monotonically
    int cofs[CPL];      // offset of each owned column within a cost-buffer row
#pragma unroll
    for (int t = 0; t < CPL; t++) cofs[t] = col0 + 32 * t;
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        fence_mbar_init();
        mbar_expect_tx(&mbar[0], bytes);
        tma_load_1d(wbase, a.src + b * a.ld, bytes, &mbar[0]);
    }
    __syncwarp();

    bool anybad = false;
    for (int it = 0; b < a.count; it++) {
        int64_t nb;  // next block of this warp
        if (dyn) {
            nb = b + 1;
            if (nb >= cend) {
                int64_t c0 = 0;
                if (lane == 0) c0 = (int64_t)atomicAdd(&a.sched->head, (unsigned long long)CH);
                nb = __shfl_sync(FULL_MASK, c0, 0);
                cend = nb + CH < a.count ? nb + CH : a.count;
            }
        } else {
            nb = b + nw;
        }
        mbar_wait(&mbar[0], it & 1);
        double *M = reinterpret_cast<double *>(wbase);

        int poff[CPL], p[CPL];
        double v[CPL], ucol[CPL];
        int steps = 0;
        if constexpr (CPL == 1) {
            if (a.lvl == LAP_BATCH) warp_lap_solve1<true>(M, m, lane, scratch, poff[0], v[0], ucol[0], steps);
            else warp_lap_solve1<false>(M, m, lane, scratch, poff[0], v[0], ucol[0], steps);
        } else {
            if (a.lvl == LAP_BATCH) warp_lap_solve2<true>(M, m, lane, scratch, poff, v, ucol, steps);
            else warp_lap_solve2<false>(M, m, lane, scratch, poff, v, ucol, steps);
        }
        bool bad;
        const double *Mg = a.src + b * a.ld;
        const double S = warp_lap_epilogue<CPL>(
            M, [&](int r, int t, int c) { return c < m ? Mg[r * m + c] : 0.0; }, m, m, cofs, lane, col0, poff, p, v,
            ucol, urow, sel, 1, rmag, bad);
        anybad |= bad;
        if (lane == 0) {
            tma_store_1d(a.dst + b * a.ld, M, bytes);  // residual block back to global
            if (nb < a.count) {                       // buffer free once the store has read it
                bulk_wait_read();
                mbar_expect_tx(&mbar[0], bytes);
                tma_load_1d(wbase, a.src + nb * a.ld, bytes, &mbar[0]);
            }
        }

        if (lane == 0) {
            switch (a.lvl) {
            case LAP_L2: {  // credit S to both complementary coefficients (reading R12)
                if (a.bo.S) {  // sharded: S is all-gathered and credited by k_credit
                    a.bo.S[b] = S;
                    break;
                }
                const Geom &g = a.g;
                const int n = g.n, n1 = n - 1;
                const unsigned q = decode_l2(a, b, icur);
                const int i = q & 0xff, j = (q >> 8) & 0xff, k = (q >> 16) & 0xff, l = q >> 24;
                // C was spread to D and zeroed: c <- 0 + S = S.
                a.C[(int64_t)(i * n + j) * g.ldc + (k - 1) * n1 + (l - (l > j))] = S;
                a.C[(int64_t)(k * n + l) * g.ldc + i * n1 + (j - (j > l))] = S;
                break;
            }
            case LAP_L1_ACC:
            case LAP_L1_SET: {
                const int64_t bi = a.bdiv ? (b / a.bdiv) * a.bstr + b % a.bdiv : b;
                if (a.lvl == LAP_L1_ACC) a.B[bi] = a.B[bi] + S;
                else a.B[bi] = S;  // B was spread and zeroed: 0 + S = S
                break;
            }
            case LAP_L0_MULTI: a.lbm[b] = a.lbm[b] + S; break;
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
                const int c = col0 + 32 * t;
                if (c < m) {
                    if (a.bo.assign) a.bo.assign[b * m + p[t]] = c;
                    if (a.bo.u) a.bo.u[b * m + p[t]] = ucol[t];
                    if (a.bo.v) a.bo.v[b * m + c] = v[t];
                }
            }
        }
        __syncwarp();
        b = nb;
    }
    if (lane == 0) bulk_wait_all();
    if (anybad && lane == 0) {
        if (a.ctl) atomicOr(&a.ctl->err, 1);
        if (a.bo.err) atomicOr(a.bo.err, 1);
    }
}

// ---------------------------------------------------------------------------------------
// k_init — O0/O1: b0 with the fixed-free folds, c_ij[kl] = f'_ik d'_jl,
// kappa; D is NOT written (the next transfer reads it as zero).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int tx_c2(int a) { return a * (a - 1) / 2; }
__device__ __forceinline__ int tx_c3(int a) { return a * (a - 1) * (a - 2) / 6; }
// triples (i<k<p) of the cube (a, b, c) of edge e (a <= b <= c), node size n
__device__ __forceinline__ int tx_cube_count(int a, int b, int c, int e, int n)
{
    const int sa = min(e, n - a * e), sb = min(e, n - b * e), sc = min(e, n - c * e);
    if (a == b && b == c) return tx_c3(sa);
    if (a == b) return tx_c2(sa) * sc;
    if (b == c) return sa * tx_c2(sb);
    return sa * sb * sc;
}
// facility triples i<k<p: triples[0, ntri) in lexicographic order (the register transfer's
// grid.y and the sharded tile ids), triples[ntri, 2 ntri) grouped into cubes of edge
// kTxCube in (i,k,p) (cubes lexicographic, triples lexicographic within a cube): the TMA
// transfer's dispatch order, so that the CTAs in flight read runs of neighbouring rows of the
// same blocks in all three member views
__device__ void write_triples(int n, int *triples)
{
    const int ntri = n * (n - 1) * (n - 2) / 6, e = kTxCube, nc = (n + e - 1) / e;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntri; t += gridDim.x * blockDim.x) {
        int rem = t, i = 0;
        while (rem >= (n - 1 - i) * (n - 2 - i) / 2) {
            rem -= (n - 1 - i) * (n - 2 - i) / 2;
            i++;
        }
        int k = i + 1;
        while (rem >= n - 1 - k) {
            rem -= n - 1 - k;
            k++;
        }
        const int p = k + 1 + rem;
        const int packed = i | (k << 8) | (p << 16);
        triples[t] = packed;
        const int ci = i / e, ck = k / e, cp = p / e;
        int pos = 0;
        for (int a = 0; a < nc; a++)
            for (int b = a; b < nc; b++)
                for (int c = b; c < nc; c++)
                    if (a < ci || (a == ci && (b < ck || (b == ck && c < cp)))) pos += tx_cube_count(a, b, c, e, n);
        for (int x = ci * e; x < min(n, ci * e + e); x++)
            for (int y = max(x + 1, ck * e); y < min(n, ck * e + e); y++)
                for (int z = max(y + 1, cp * e); z < min(n, cp * e + e); z++)
                    if (x < i || (x == i && (y < k || (y == k && z < p)))) pos++;
        triples[ntri + pos] = packed;
    }
}

__global__ void k_init(const Node nd, const Geom g, const int64_t *__restrict__ F,
                       const int64_t *__restrict__ Dist, double *B, double *C, int *triples, Ctl *ctl)
{
    write_triples(nd.n, triples);
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

// ---------------------------------------------------------------------------------------
// Warm child (reading R31): the state of the child of the parent
// node (gp: n free) that fixes the parent-reduced facility a at location b, built from the
// parent's dual state:
//   kappa' = kappa, lb_dual' = lb_dual + b_ab
//   b'_xy     = (b_xy + c_ab[xy]) + c_xy[ab]
//   c'_xy[zw] = c_xy[zw] + ((d_{ab,xy,zw} + d_{ab,zw,xy}) + d_{xy,zw,ab})   (logical d)
//   d'_{xy,zw}[pq] = d_{xy,zw}[pq]                     (x,z != a; y,w != b; indices shifted)
// k_fold_bc writes B', C', the child's control block and its triples table (one thread per
// entry); k_fold_d copies the restricted D blocks (one warp per child block, lane = column,
// rows streamed).  With the parent's D still lazily zero, the D terms are 0 and D' is left
// lazily zero too.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t cidx_g(const Geom &g, int i, int j, int k, int l)
{
    return (int64_t)(i * g.n + j) * g.ldc + (int64_t)(k - (k > i)) * (g.n - 1) + (l - (l > j));
}
__device__ __forceinline__ double dlogical(const Geom &g, const double *D, int i, int j, int k, int l, int p, int q)
{
    if (i > k) {
        int t = i;
        i = k;
        k = t;
        t = j;
        j = l;
        l = t;
    }
    return D[bid_of(g, i, j, k, l) * g.ld2 + (int64_t)(p - (p > i) - (p > k)) * (g.n - 2) + (q - (q > j) - (q > l))];
}

__global__ void k_fold_bc(const FoldArgs f)
{
    const Geom &gp = f.gp;
    const int n = gp.n, nc = n - 1, nc1 = nc - 1, a = f.a, b = f.b;
    write_triples(nc, f.triples);
    const int nC = nc * nc * nc1 * nc1, tot = nC + nc * nc;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
        if (t < nC) {
            const int lw = t % nc1, kz = (t / nc1) % nc1, y = (t / (nc1 * nc1)) % nc, x = t / (nc1 * nc1 * nc);
            const int z = kz + (kz >= x), w = lw + (lw >= y);  // child indices of the entry
            const int X = x + (x >= a), Y = y + (y >= b), Z = z + (z >= a), W = w + (w >= b);
            double e = 0.0;
            if (!f.d_zero) {
                const double e1 = dlogical(gp, f.pD, a, b, X, Y, Z, W);
                const double e2 = dlogical(gp, f.pD, a, b, Z, W, X, Y);
                const double e3 = dlogical(gp, f.pD, X, Y, Z, W, a, b);
                e = (e1 + e2) + e3;
            } else {
                e = (0.0 + 0.0) + 0.0;
            }
            f.cC[(int64_t)(x * nc + y) * f.gc.ldc + (int64_t)kz * nc1 + lw] = f.pC[cidx_g(gp, X, Y, Z, W)] + e;
        } else {
            const int u = t - nC, x = u / nc, y = u % nc;
            const int X = x + (x >= a), Y = y + (y >= b);
            f.cB[u] = (f.pB[X * n + Y] + f.pC[cidx_g(gp, a, b, X, Y)]) + f.pC[cidx_g(gp, X, Y, a, b)];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Ctl *c = f.cctl;
        c->kappa = f.pctl->kappa;
        c->lb_dual = f.pctl->lb_dual + f.pB[a * n + b];
        c->lbprime = 0.0;
        c->lb = (double)c->kappa + c->lb_dual;
        c->lb_glb = c->lb;
        c->iters = 0;
        c->status = 0;
        c->stopped = 0;
        c->err = 0;
    }
}

__global__ void __launch_bounds__(256) k_fold_d(const FoldArgs f)
{
    const Geom &gp = f.gp, &gc = f.gc;
    const int nc = gc.n, nc1 = nc - 1, mc = nc - 2, mp = gp.n - 2, a = f.a, b = f.b;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    int hint = 0;
    for (int64_t cb = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); cb < gc.nblk; cb += nw) {
        while (hint + 1 < nc && cb >= gc.off[hint + 1]) hint++;
        while (hint > 0 && cb < gc.off[hint]) hint--;
        const int x = hint;
        int rem = (int)(cb - gc.off[x]);
        const int per_y = (nc1 - x) * nc1;
        const int y = rem / per_y;
        rem -= y * per_y;
        const int zz = rem / nc1, wl = rem - zz * nc1;
        const int z = x + 1 + zz, w = wl + (wl >= y);
        const int X = x + (x >= a), Y = y + (y >= b), Z = z + (z >= a), W = w + (w >= b);
        const int ra = a - (a > X) - (a > Z), cbk = b - (b > Y) - (b > W);  // parent row/col dropped
        const double *src = f.pD + bid_of(gp, X, Y, Z, W) * gp.ld2;
        double *dst = f.cD + cb * gc.ld2;
        for (int r = 0; r < mc; r++) {
            const double *sr = src + (int64_t)(r + (r >= ra)) * mp;
            for (int c = lane; c < mc; c += 32) dst[r * mc + c] = sr[c + (c >= cbk)];
        }
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
                        double *__restrict__ sigma, const Ctl *ctl, Sched *sched)
{
    if (ctl->stopped) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) sched->head = 0;
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

// x / 3.0 correctly rounded (reading R11's division) without the IEEE division sequence:
// q0 = RN(x y) with y = RN(1/3) = (1 - 2^-54)/3, r = x - 3 q0 exactly (one FMA), q1 = RN(q0 + r y)
// (one FMA).  Writing d = x/3 - q0, the FMA's exact operand is q0 + r y = x/3 - d 2^-54, within
// 2^-55 ulp of x/3; x/3 is never a rounding midpoint and lies at least ulp/6 away from one
// (a 53-bit x would have to equal 3 M for a 54-bit odd M), so RN(x/3 - d 2^-54) = RN(x/3) for
// every normal x and for 0.  Bit-identical to the oracle's (e1 + e2 + e3) / 3.0.
__device__ __forceinline__ double div3(double x)
{
    const double y = 0x1.5555555555555p-2;  // RN(1/3)
    const double q0 = __dmul_rn(x, y);
    const double r = fma(-3.0, q0, x);
    return fma(r, y, q0);
}

// Shared-memory index of element (x,y,z) of a tile view: rows padded to 9 doubles so
// that the transposed reads of the mean phase are (nearly) bank-conflict free.
__device__ __forceinline__ int tix(int x, int y, int z) { return x * (TT * (TT + 1)) + y * (TT + 1) + z; }
constexpr unsigned NOIDX = 0xffffffffu;

// Tile kinds of a sharded iteration.  A tile of facility triple (i,k,p) has
// its views 0 and 1 (members e1, e2) on owner(i) and its view 2 (member e3) on owner(k).
enum { TK_LOCAL = 0, TK_AGG = 1, TK_HOLD = 2 };

template <bool SHARDED, bool WIDE>  // WIDE: 64-bit per-view bases (>= 2^32 stored entries)
__global__ void __launch_bounds__(256, 6) k_transfer(const TransferArgs A)
{
    if (A.ctl->stopped) return;
    __shared__ double sv[3][TT * TT * (TT + 1)];  // the three member views of the tile's classes
    __shared__ unsigned rbase[3][TT * TT];        // element index of each view row in D (NOIDX: none)
    __shared__ double rsig[3][TT * TT];           // spread amount sigma of the row's block
    const Geom &g = A.g;
    const int n = g.n, m2 = n - 2, ntile = A.ntile;
    const int64_t ld2 = g.ld2;
    int tq, tile, kind = TK_LOCAL, slot = 0;
    if (SHARDED) {  // this rank's tile list
        const int T = A.tiles[blockIdx.x];
        const int nt3 = ntile * ntile * ntile;
        tq = T / nt3;
        tile = T - tq * nt3;
        const int info = A.tinfo[blockIdx.x];
        kind = info & 3;
        slot = info >> 2;
        if (A.pack && kind == TK_LOCAL) return;
    } else {
        tq = blockIdx.y;
        tile = blockIdx.x;
    }
    const int tri = A.triples[tq];  // (i,k,p), i<k<p, packed by k_init
    const int i = tri & 0xff, k = (tri >> 8) & 0xff, p = tri >> 16;
    const int tl = tile / ntile, tj = tl / ntile;
    const int q0 = (tile - tl * ntile) * TT, l0 = (tl - tj * ntile) * TT, j0 = tj * TT;
    const int tid = threadIdx.x;
    // which views live here
    const bool has01 = kind != TK_HOLD, has2 = kind != TK_AGG;
    // 64-bit base block of each view (local numbering); 32-bit row offsets relative to it
    const int n1 = n - 1;
    const int64_t lo_i = SHARDED ? A.loc_off[i] : 0, lo_k = SHARDED ? A.loc_off[k] : 0;
    const int64_t vb0 = WIDE ? g.off[i] + (int64_t)j0 * (n1 - i) * n1 + (int64_t)(k - i - 1) * n1 + lo_i : 0,
                  vb1 = WIDE ? g.off[i] + (int64_t)j0 * (n1 - i) * n1 + (int64_t)(p - i - 1) * n1 + lo_i : 0,
                  vb2 = WIDE ? g.off[k] + (int64_t)l0 * (n1 - k) * n1 + (int64_t)(p - k - 1) * n1 + lo_k : 0;
    auto vbs = [&](int vw) { return vw == 0 ? vb0 : (vw == 1 ? vb1 : vb2); };

    // rows: view 0 = D{ij,kl} row p-2 (rows (j,l)); view 1 = D{ij,pq} row k-1 (rows (j,q));
    //       view 2 = D{kl,pq} row i   (rows (l,q)).  sigma is fetched now, used after the
    //       D loads are in flight.
    double sg = 0.0;
    if (tid < 3 * TT * TT) {
        const int vw = tid >> 6, x = (tid >> 3) & 7, y = tid & 7;
        int r0, r1;
        if (vw == 0) { r0 = j0 + x; r1 = l0 + y; }
        else if (vw == 1) { r0 = j0 + x; r1 = q0 + y; }
        else { r0 = l0 + x; r1 = q0 + y; }
        unsigned base = NOIDX;
        if (r0 < n && r1 < n && r0 != r1 && (vw == 2 ? has2 : has01)) {
            int64_t bb;
            int row;
            if (vw == 0) { bb = bid_of(g, i, r0, k, r1); row = p - 2; }
            else if (vw == 1) { bb = bid_of(g, i, r0, p, r1); row = k - 1; }
            else { bb = bid_of(g, k, r0, p, r1); row = i; }
            sg = A.sigma[bb];
            base = (unsigned)((bb + (SHARDED ? A.loc_off[vw == 2 ? k : i] : 0) - vbs(vw)) * ld2 + row * m2);
        }
        rbase[vw][tid & 63] = base;
    }
    __syncthreads();

    // load: element e = (x,y,z) of view vw is row (x,y), free index z (contiguous in D)
    unsigned addr[2][3];
    double val[2][3];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int e = tid + 256 * h;
        const int x = e >> 6, y = (e >> 3) & 7, z = e & 7;
#pragma unroll
        for (int vw = 0; vw < 3; vw++) {
            // (a, b) = the row's two locations, f = the free (column) location
            const int a = (vw == 2 ? l0 : j0) + x;
            const int b = (vw == 0 ? l0 : q0) + y;
            const int f = (vw == 0 ? q0 : (vw == 1 ? l0 : j0)) + z;
            const unsigned base = rbase[vw][e >> 3];
            unsigned ad = NOIDX;
            if (base != NOIDX && f < n && f != a && f != b) ad = base + (unsigned)(f - (f > a) - (f > b));
            addr[h][vw] = ad;
            val[h][vw] = (ad != NOIDX && !A.d_zero) ? A.D[vbs(vw) * ld2 + ad] : 0.0;
        }
    }
    if (tid < 3 * TT * TT) rsig[tid >> 6][tid & 63] = sg;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int e = tid + 256 * h;
        const int x = e >> 6, y = (e >> 3) & 7, z = e & 7;
#pragma unroll
        for (int vw = 0; vw < 3; vw++) sv[vw][tix(x, y, z)] = val[h][vw] + rsig[vw][e >> 3];
    }
    __syncthreads();
    // mean of each class (j,l,q): e1 = sv0[j][l][q], e2 = sv1[j][q][l], e3 = sv2[l][q][j]
    // (reading R11: ((e1 + e2) + e3) / 3, the same operations on every rank)
    const size_t xo = (size_t)slot * (TT * TT * TT);
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int e = tid + 256 * h;
        const int a = e >> 6, b = (e >> 3) & 7, c = e & 7;
        const int j = j0 + a, l = l0 + b, q = q0 + c;
        if (j < n && l < n && q < n && j != l && j != q && l != q) {
            const int e1 = tix(a, b, c), e2 = tix(a, c, b), e3 = tix(b, c, a);
            if (SHARDED && A.pack) {  // sharded, pass 1: this side's partial of the class
                A.sendbuf[xo + e] = kind == TK_AGG ? sv[0][e1] + sv[1][e2] : sv[2][e3];
            } else {
                const double s12 = (SHARDED && kind == TK_HOLD) ? A.recvbuf[xo + e] : sv[0][e1] + sv[1][e2];
                const double h3 = (SHARDED && kind == TK_AGG) ? A.recvbuf[xo + e] : sv[2][e3];
                const double mu = div3(s12 + h3);
                sv[0][e1] = mu;
                sv[1][e2] = mu;
                sv[2][e3] = mu;
            }
        }
    }
    if (SHARDED && A.pack) return;
    __syncthreads();
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int e = tid + 256 * h;
        const int x = e >> 6, y = (e >> 3) & 7, z = e & 7;
#pragma unroll
        for (int vw = 0; vw < 3; vw++)
            if (addr[h][vw] != NOIDX) A.D[vbs(vw) * ld2 + addr[h][vw]] = sv[vw][tix(x, y, z)];
    }
}

// ---------------------------------------------------------------------------------------
// k_transfer_tma — the same transfer (identical operations per class, reading R11) with the
// three member views of a tile fetched by tensor-map TMA instead of per-element loads.  Per
// first facility f a 4-D tensor map views the stored blocks of f as
//   [j (first location)][k - f - 1 (second facility)][l' (second location, skip-indexed)]
//   [in-block entry]
// (TmaMaps, encoded on the host per node size).  A tile's view is one box of
// TT (j) x 1 x (TT+1) (l') x (TT+4) (entries): the row of the third facility with a window of
// TT+2 columns — wide enough for the skip-indexed positions of every (j, l, q) of the tile —
// started at an even entry (TMA needs 16-byte aligned box starts in the innermost dimension).
// Boxes overlap neighbouring tiles, so results are stored element-wise (coalesced runs of
// <= 8 doubles per view row), only for the tile's own classes.  Unsharded handles only.
// ---------------------------------------------------------------------------------------
// position in view vw's box of the element of class (j,l,q) (tile origin j0, l0, q0).
// The box's dim0 window starts at the even entry at or below (row * m2 + w): TMA needs a
// 16-byte aligned start in the innermost dimension; odd = 1 when it was moved down by one.
template <int BX0>
__device__ __forceinline__ int box_pos(int vw, int j, int l, int q, int j0, int l0, int q0, int odd)
{
    if (vw == 0) {  // D{ij,kl}[p-2][q'] : rows (j, l'), column q'
        const int lp = l - (l > j), qp = q - (q > j) - (q > l);
        const int ls = l0 > 0 ? l0 - 1 : 0, w = q0 > 1 ? q0 - 2 : 0;
        return ((j - j0) * kBox1 + (lp - ls)) * BX0 + (qp - w + odd);
    } else if (vw == 1) {  // D{ij,pq}[k-1][l'] : rows (j, q'), column l'
        const int qp = q - (q > j), lp = l - (l > j) - (l > q);
        const int qs = q0 > 0 ? q0 - 1 : 0, w = l0 > 1 ? l0 - 2 : 0;
        return ((j - j0) * kBox1 + (qp - qs)) * BX0 + (lp - w + odd);
    } else {  // D{kl,pq}[i][j'] : rows (l, q'), column j'
        const int qp = q - (q > l), jp = j - (j > l) - (j > q);
        const int qs = q0 > 0 ? q0 - 1 : 0, w = j0 > 1 ? j0 - 2 : 0;
        return ((l - l0) * kBox1 + (qp - qs)) * BX0 + (jp - w + odd);
    }
}

// WIDE: the stored D has >= 2^32 entries (n >= 47): row offsets relative to 64-bit per-view
// base blocks; otherwise absolute 32-bit element indices (fewer instructions).
// NT = 256: each thread averages 2 classes, the means are parked in a per-class array (8 CTAs
// per SM by threads); NT = 128: 4 classes per thread, the means are written over the members'
// box slots and the store phase reads them from there (no mean array: 11 CTAs per SM).
template <int BX0, bool WIDE, int NT>  // BX0 = TT + 2 (m2 even: window starts are even) or TT + 4
__global__ void __launch_bounds__(NT, NT == 256 ? 8 : 11) k_transfer_tma(const TransferArgs A, const __grid_constant__ TmaMaps M)
{
    constexpr int BOXE = TT * kBox1 * BX0;
    constexpr bool INBOX = NT == 128;
    if (A.ctl->stopped) return;
    __shared__ __align__(128) double box[3][BOXE];
    // class (a,b,c) = (j-j0, l-l0, q-q0) -> its mean at a * MA + b * MB + c (odd strides:
    // the permuted reads of the store phase are bank-conflict free)
    constexpr int MB = TT + 1, MA = TT * MB + 1;
    __shared__ double mean[INBOX ? 1 : TT * MA];
    __shared__ unsigned rbase[3][TT * TT];  // element offset of each view row from the view's base
    __shared__ double rsig[3][TT * TT];
    __shared__ __align__(8) uint64_t mbar;
    const Geom &g = A.g;
    const int n = g.n, m2 = n - 2, ntile = A.ntile;
    const int64_t ld2 = g.ld2;
    const int tri = A.triples[blockIdx.z];
    const int i = tri & 0xff, k = (tri >> 8) & 0xff, p = tri >> 16;
    // grid (q tile, j tile * ntile + l tile, triple); y / ntile by a multiply (y < ntile^2 <= 64)
    const int tj = (int)((blockIdx.y * A.ntile_mul) >> 16), tl = (int)blockIdx.y - tj * ntile;
    const int q0 = (int)blockIdx.x * TT, l0 = tl * TT, j0 = tj * TT;
    // WIDE: 64-bit base block of each view (first row location at the tile origin, second at
    // 0); row offsets relative to it stay below 8 (n-1)^2 blocks, so 32 bits suffice for any n
    const int n1 = n - 1;
    const int64_t vb0 = WIDE ? g.off[i] + (int64_t)j0 * (n1 - i) * n1 + (int64_t)(k - i - 1) * n1 : 0;
    const int64_t vb1 = WIDE ? g.off[i] + (int64_t)j0 * (n1 - i) * n1 + (int64_t)(p - i - 1) * n1 : 0;
    const int64_t vb2 = WIDE ? g.off[k] + (int64_t)l0 * (n1 - k) * n1 + (int64_t)(p - k - 1) * n1 : 0;
    double *const D0 = A.D + vb0 * ld2, *const D1 = A.D + vb1 * ld2, *const D2 = A.D + vb2 * ld2;
    const int tid = threadIdx.x;
    const bool dz = A.d_zero != 0;
    // dim0 window starts (entries) of the three views, before rounding down to even
    const int s0 = (p - 2) * m2 + (q0 > 1 ? q0 - 2 : 0), s1 = (k - 1) * m2 + (l0 > 1 ? l0 - 2 : 0),
              s2 = i * m2 + (j0 > 1 ? j0 - 2 : 0);
    const int o0 = s0 & 1, o1 = s1 & 1, o2 = s2 & 1;
    if (tid == 0 && !dz) {
        mbar_init(&mbar, 1);
        fence_mbar_init();
        mbar_expect_tx(&mbar, 3u * BOXE * 8u);
        tma_load_4d(box[0], &M.m[i], s0 - o0, l0 > 0 ? l0 - 1 : 0, k - i - 1, j0, &mbar);
        tma_load_4d(box[1], &M.m[i], s1 - o1, q0 > 0 ? q0 - 1 : 0, p - i - 1, j0, &mbar);
        tma_load_4d(box[2], &M.m[k], s2 - o2, q0 > 0 ? q0 - 1 : 0, p - k - 1, l0, &mbar);
    }
    // per view row: element index of the row in D (stores) and sigma of its block
    for (int er = tid; er < 3 * TT * TT; er += NT) {
        const int vw = er >> 6, x = (er >> 3) & 7, y = er & 7;
        int r0, r1;
        if (vw == 0) { r0 = j0 + x; r1 = l0 + y; }
        else if (vw == 1) { r0 = j0 + x; r1 = q0 + y; }
        else { r0 = l0 + x; r1 = q0 + y; }
        unsigned base = NOIDX;
        double sg = 0.0;
        if (r0 < n && r1 < n && r0 != r1) {
            // block D{f r0, h r1} (f < h): row `row`; 32-bit arithmetic unless WIDE
            const int f = vw == 2 ? k : i, h = vw == 0 ? k : p, row = vw == 0 ? p - 2 : (vw == 1 ? k - 1 : i);
            const int rel = r0 * (n1 - f) * n1 + (h - f - 1) * n1 + (r1 - (r1 > r0));  // block id - off[f]
            if (WIDE) {
                const int64_t bb = g.off[f] + rel;
                sg = A.sigma[bb];
                base = (unsigned)((bb - (vw == 0 ? vb0 : (vw == 1 ? vb1 : vb2))) * ld2 + row * m2);
            } else {
                const unsigned bb = (unsigned)g.off[f] + (unsigned)rel;
                sg = A.sigma[bb];
                base = bb * (unsigned)ld2 + (unsigned)(row * m2);
            }
        }
        rbase[vw][er & 63] = base;
        rsig[vw][er & 63] = sg;
    }
    __syncthreads();
    if (!dz) mbar_wait(&mbar, 0);
    // mean of each class (j,l,q) of the tile: ((e1 + e2) + e3) / 3 with e = stored + sigma.
    // View 0's store element e is class e itself: stored from the register right away.
#pragma unroll
    for (int h = 0; h < TT * TT * TT / NT; h++) {
        const int e = tid + NT * h;
        const int a = e >> 6, b = (e >> 3) & 7, c = e & 7;
        const int j = j0 + a, l = l0 + b, q = q0 + c;
        if (j < n && l < n && q < n && j != l && j != q && l != q) {
            const int b1 = box_pos<BX0>(1, j, l, q, j0, l0, q0, o1), b2 = box_pos<BX0>(2, j, l, q, j0, l0, q0, o2);
            const double e1 = (dz ? 0.0 : box[0][box_pos<BX0>(0, j, l, q, j0, l0, q0, o0)]) + rsig[0][a * 8 + b];
            const double e2 = (dz ? 0.0 : box[1][b1]) + rsig[1][a * 8 + c];
            const double e3 = (dz ? 0.0 : box[2][b2]) + rsig[2][b * 8 + c];
            const double mu = div3((e1 + e2) + e3);
            if (INBOX) {  // each class owns its slots of the three boxes
                box[1][b1] = mu;
                box[2][b2] = mu;
            } else {
                mean[a * MA + b * MB + c] = mu;
            }
            D0[rbase[0][e >> 3] + (unsigned)(q - (q > j) - (q > l))] = mu;  // row (j,l), column q'
        }
    }
    __syncthreads();
    // views 1 and 2: element (x,y,z) = row (x,y), free index z (contiguous runs in D)
#pragma unroll
    for (int h = 0; h < TT * TT * TT / NT; h++) {
        const int e = tid + NT * h;
        const int x = e >> 6, y = (e >> 3) & 7, z = e & 7;
        {   // view 1: row (j, q) = (j0 + x, q0 + y), free l = l0 + z; class (x, z, y)
            const int a = j0 + x, b = q0 + y, f = l0 + z;
            const unsigned base = rbase[1][e >> 3];
            if (base != NOIDX && f < n && f != a && f != b)
                D1[base + (unsigned)(f - (f > a) - (f > b))] =
                    INBOX ? box[1][box_pos<BX0>(1, a, f, b, j0, l0, q0, o1)] : mean[x * MA + z * MB + y];
        }
        {   // view 2: row (l, q) = (l0 + x, q0 + y), free j = j0 + z; class (z, x, y)
            const int a = l0 + x, b = q0 + y, f = j0 + z;
            const unsigned base = rbase[2][e >> 3];
            if (base != NOIDX && f < n && f != a && f != b)
                D2[base + (unsigned)(f - (f > a) - (f > b))] =
                    INBOX ? box[2][box_pos<BX0>(2, f, a, b, j0, l0, q0, o2)] : mean[z * MA + x * MB + y];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Strong branching: RLT1 bounds of the n^2 candidate children of a node at once.
// Child c = a * n + b fixes free facility I[a] at free location J[b] in addition to the
// node's pairs; its reduced costs are built as in k_init (O0/O1).
// ---------------------------------------------------------------------------------------
__global__ void k_rlt1_init(const Node nd, const Rlt1Batch R, const int64_t *__restrict__ F,
                            const int64_t *__restrict__ Dist)
{
    const int N = nd.N, n = nd.n, c = blockIdx.y, ca = c / n, cb = c - ca * n;
    const int np = n - 1, np1 = np - 1;  // child size n', n'-1
    const int fa = nd.I[ca], la = nd.J[cb];
    const int64_t n4 = (int64_t)np * np * np * np;
    const int64_t tot = n4 + (int64_t)np * np;
    double *C = R.C + (int64_t)c * np * np * R.g.ldc;
    double *B = R.B + (int64_t)c * R.bstr;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
        if (x < n4) {
            const int l = (int)(x % np), k = (int)((x / np) % np), j = (int)((x / np / np) % np),
                      i = (int)(x / np / np / np);
            if (k == i || l == j) continue;
            const int Ii = nd.I[i + (i >= ca)], Ik = nd.I[k + (k >= ca)];
            const int Jj = nd.J[j + (j >= cb)], Jl = nd.J[l + (l >= cb)];
            C[(int64_t)(i * np + j) * R.g.ldc + (k - (k > i)) * np1 + (l - (l > j))] =
                (double)(F[Ii * N + Ik] * Dist[Jj * N + Jl]);
        } else {
            const int y = (int)(x - n4), a_ = y / np, b_ = y % np;
            const int Ia = nd.I[a_ + (a_ >= ca)], Jb = nd.J[b_ + (b_ >= cb)];
            int64_t v = F[Ia * N + Ia] * Dist[Jb * N + Jb];
            for (int t = 0; t < nd.m; t++)
                v += F[nd.fac[t] * N + Ia] * Dist[nd.loc[t] * N + Jb] + F[Ia * N + nd.fac[t]] * Dist[Jb * N + nd.loc[t]];
            v += F[fa * N + Ia] * Dist[la * N + Jb] + F[Ia * N + fa] * Dist[Jb * N + la];
            B[y] = (double)v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // kappa: fixed-fixed cost incl. the new pair
        long long kap = 0;
        for (int t = 0; t <= nd.m; t++) {
            const int f1 = t < nd.m ? nd.fac[t] : fa, l1 = t < nd.m ? nd.loc[t] : la;
            for (int t2 = 0; t2 <= nd.m; t2++) {
                const int f2 = t2 < nd.m ? nd.fac[t2] : fa, l2 = t2 < nd.m ? nd.loc[t2] : la;
                kap += F[f1 * N + f2] * Dist[l1 * N + l2];
            }
        }
        R.kap[c] = kap;
        R.lbd[c] = 0.0;
    }
}

// RLT1 iteration, first half (P:216 spread B->C, then P:189 transfer between the
// complementary costs of C = pair mean, reading R13):
//   a = c_ij[kl] + b_ij/(n'-1), b = c_kl[ij] + b_kl/(n'-1), both <- (a + b) / 2.
__global__ void k_rlt1_pair(const Rlt1Batch R)
{
    const int np = R.g.n, np1 = np - 1;
    const int64_t n4 = (int64_t)np * np * np * np;
    const double div1 = (double)(np - 1);
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n4 * R.K; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = x / n4, y = x - c * n4;
        const int l = (int)(y % np), k = (int)((y / np) % np), j = (int)((y / np / np) % np), i = (int)(y / np / np / np);
        if (k <= i || l == j) continue;
        double *C = R.C + c * np * np * R.g.ldc;
        const double *B = R.B + c * R.bstr;
        double *p1 = C + (int64_t)(i * np + j) * R.g.ldc + (k - 1) * np1 + (l - (l > j));
        double *p2 = C + (int64_t)(k * np + l) * R.g.ldc + i * np1 + (j - (j > l));
        const double a = *p1 + B[i * np + j] / div1;
        const double b = *p2 + B[k * np + l] / div1;
        const double mu = (a + b) / 2.0;
        *p1 = mu;
        *p2 = mu;
    }
}

// Sharded iteration: level-2 values S of every stored block (all-gathered, global block
// order) credited to both complementary coefficients (reading R12), on every rank.
__global__ void k_credit(const Geom g, const double *__restrict__ S, const Offsets pos, double *__restrict__ C,
                         const Ctl *ctl)
{
    if (ctl->stopped) return;
    const int n = g.n, n1 = n - 1;
    const int64_t n4 = (int64_t)n * n * n * n;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n4; x += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(x % n), k = (int)((x / n) % n), j = (int)((x / n / n) % n), i = (int)(x / n / n / n);
        if (k <= i || l == j) continue;
        const double v = S[bid_of(g, i, j, k, l) + pos.off[i]];
        C[(int64_t)(i * n + j) * g.ldc + (k - 1) * n1 + (l - (l > j))] = v;
        C[(int64_t)(k * n + l) * g.ldc + i * n1 + (j - (j > l))] = v;
    }
}

// ---------------------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------------------
cudaError_t launch_init(const Node &node, const Geom &g, const int64_t *F, const int64_t *Dist, double *B,
                        double *C, int *triples, Ctl *ctl, cudaStream_t st)
{
    const int64_t tot = (int64_t)g.n * g.n * g.n * g.n + (int64_t)g.n * g.n;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_init<<<blocks, 256, 0, st>>>(node, g, F, Dist, B, C, triples, ctl);
    return cudaGetLastError();
}

cudaError_t launch_fold(const FoldArgs &f, int num_sms, cudaStream_t st)
{
    const int nc = f.gc.n;
    const int64_t tot = (int64_t)nc * nc * (nc - 1) * (nc - 1) + (int64_t)nc * nc;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > num_sms * 16) blocks = num_sms * 16;
    k_fold_bc<<<blocks, 256, 0, st>>>(f);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || f.d_zero) return e;
    int64_t wb = (f.gc.nblk + 7) / 8;
    const int grid = (int)(wb < (int64_t)num_sms * 8 ? wb : (int64_t)num_sms * 8);
    k_fold_d<<<grid, 256, 0, st>>>(f);
    return cudaGetLastError();
}

cudaError_t launch_ctl_begin(Ctl *ctl, double K, double UB, int trace_cap, cudaStream_t st)
{
    k_ctl_begin<<<1, 1, 0, st>>>(ctl, K, UB, trace_cap);
    return cudaGetLastError();
}

cudaError_t launch_sigma(const Geom &g, const double *B, const double *C, double *sigma, const Ctl *ctl,
                         Sched *sched, cudaStream_t st)
{
    const int64_t tot = (int64_t)g.n * g.n * g.n * g.n;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_sigma<<<blocks, 256, 0, st>>>(g, B, C, sigma, ctl, sched);
    return cudaGetLastError();
}

int tma_box0(int n) { return ((n - 2) & 1) ? kBox0 : kBox0 - 2; }

cudaError_t launch_transfer_tma(const TransferArgs &A, const TmaMaps &M, cudaStream_t st)
{
    const int n = A.g.n;
    const int ntri = n * (n - 1) * (n - 2) / 6;
    if (A.ntile > 8 || ntri > 65535) return cudaErrorInvalidValue;  // n <= kMaxN = 64
    TransferArgs B = A;
    B.ntile_mul = (65536u + (unsigned)A.ntile - 1u) / (unsigned)A.ntile;  // exact y / ntile for y < 64
    B.triples = A.triples + ntri;  // the cube-blocked dispatch order (write_triples)
    dim3 grid(A.ntile, A.ntile * A.ntile, ntri);
    const bool wide = (int64_t)A.g.nblk * A.g.ld2 >= (int64_t(1) << 32);
    constexpr int NT = 128;  // means in the boxes, 11 CTAs per SM
    if (tma_box0(n) == kBox0) {
        if (wide) k_transfer_tma<kBox0, true, NT><<<grid, NT, 0, st>>>(B, M);
        else k_transfer_tma<kBox0, false, NT><<<grid, NT, 0, st>>>(B, M);
    } else {
        if (wide) k_transfer_tma<kBox0 - 2, true, NT><<<grid, NT, 0, st>>>(B, M);
        else k_transfer_tma<kBox0 - 2, false, NT><<<grid, NT, 0, st>>>(B, M);
    }
    return cudaGetLastError();
}

cudaError_t launch_transfer(const TransferArgs &A, int ntiles_list, cudaStream_t st)
{
    const int n = A.g.n;
    const bool wide = (int64_t)A.g.nblk * A.g.ld2 >= (int64_t(1) << 32);  // global size: conservative
    if (A.tiles) {
        if (ntiles_list <= 0) return cudaSuccess;
        if (wide) k_transfer<true, true><<<ntiles_list, 256, 0, st>>>(A);
        else k_transfer<true, false><<<ntiles_list, 256, 0, st>>>(A);
    } else {
        const int ntri = n * (n - 1) * (n - 2) / 6;
        dim3 grid(A.ntile * A.ntile * A.ntile, ntri);
        if (wide) k_transfer<false, true><<<grid, 256, 0, st>>>(A);
        else k_transfer<false, false><<<grid, 256, 0, st>>>(A);
    }
    return cudaGetLastError();
}

cudaError_t launch_credit(const Geom &g, const double *S, const Offsets &pos, double *C, const Ctl *ctl,
                          cudaStream_t st)
{
    const int64_t tot = (int64_t)g.n * g.n * g.n * g.n;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_credit<<<blocks, 256, 0, st>>>(g, S, pos, C, ctl);
    return cudaGetLastError();
}

template <int CPL>
static cudaError_t raise_smem_limit()
{
    // The dynamic-smem limit is a process-wide attribute of the kernel: raise it once per
    // device to the opt-in maximum (setting it per launch to the exact size would race
    // between threads launching different sizes, e.g. concurrent B&B workers).
    static std::mutex mu;
    static uint64_t done_dev = 0;
    int dev = 0;
    cudaError_t e0 = cudaGetDevice(&dev);
    if (e0 != cudaSuccess) return e0;
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 64 || !((done_dev >> dev) & 1)) {
        int mx = 0;
        if ((e0 = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e0;
        if ((e0 = cudaFuncSetAttribute(k_lap<CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx)) != cudaSuccess)
            return e0;
        if (dev < 64) done_dev |= 1ull << dev;
    }
    return cudaSuccess;
}

template <int CPL>
static cudaError_t launch_lap_on(const LapArgs &a, int num_sms, int wpc, int ctas_per_sm, cudaStream_t st)
{
    const size_t smem = lap_warp_smem(a.m, CPL) * wpc;
    cudaError_t e = raise_smem_limit<CPL>();
    if (e != cudaSuccess) return e;
    if (smem > 232448) return cudaErrorInvalidValue;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lap<CPL>, 32 * wpc, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t want = (a.count + wpc - 1) / wpc;
    int64_t cap = (int64_t)num_sms * per_sm;
    if (a.sched) cap = (int64_t)num_sms * (per_sm < ctas_per_sm ? per_sm : ctas_per_sm);
    const int grid = (int)(want < cap ? want : cap);
    // one block per queue grab: the grab's atomic is issued a whole LAP before its block is
    // needed, and single grabs shorten the tail (N = 30: lap2 1.385 -> 1.372 ms, N = 20: 0.1925
    // -> 0.188 ms against grabs of 4; one box, profiles/r02/README.md)
    LapArgs b = a;
    b.chunk = 1;
    k_lap<CPL><<<grid, 32 * wpc, smem, st>>>(b);
    return cudaGetLastError();
}

// c CTAs of k_lap<cpl> with `threads` threads and `smem` dynamic bytes resident per SM?  (The
// occupancy calculator knows the register file's per-sub-partition allocation: 2 CTAs of 18
// warps at 56 registers do not fit although 36 warps would.)
static bool lap_fits(int cpl, int threads, size_t smem, int c)
{
    int per_sm = 0;
    cudaError_t e = cpl == 1
                        ? (raise_smem_limit<1>(), cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lap<1>, threads, smem))
                        : (raise_smem_limit<2>(), cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lap<2>, threads, smem));
    return e == cudaSuccess && per_sm >= c;
}

// lap_cfg: bits 0-7 = warps per CTA (0: default), bits 12-15 = CTAs per SM in dynamic mode
// (0: 1).
static cudaError_t dispatch_lap(const LapArgs &a, int num_sms, int lap_cfg, cudaStream_t st)
{
    const int cpl = a.m <= 32 ? 1 : 2;
    if (a.m > 64) return cudaErrorInvalidValue;
    int wpc = lap_cfg & 0xff;
    int cps = (lap_cfg >> 12) & 0xf;
    if (wpc <= 0 && a.sched) {
        // default level-2 configuration: the most resident warps per SM that shared memory
        // (228 KB per SM, 1 KB reserved per CTA) and the register file allow, e.g. 2 CTAs x 17
        // warps at m = 28; depends on (device, m) only, so searched once and cached.  (Round 2
        // start: shared memory only, and up to 42 warps — at m = 18 that asked for 2 CTAs of 21
        // warps, of which the registers hold one: 21 warps per SM instead of 36.)
        static std::mutex mu;
        static std::map<std::pair<int, int>, std::pair<int, int>> cache;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find({dev, a.m});
        if (it != cache.end()) {
            wpc = it->second.first;
            cps = it->second.second;
        } else {
            const size_t ws = lap_warp_smem(a.m, cpl);
            int best = 0;
            for (int c = 1; c <= 2; c++)
                for (int w = 32; w >= 1; w--)
                    if ((size_t)c * (w * ws + 1024) <= 233472 && w * c > best &&
                        lap_fits(cpl, 32 * w, w * ws, c)) {
                        best = w * c;
                        wpc = w;
                        cps = c;
                    }
            if (best > 0) cache[{dev, a.m}] = {wpc, cps};
        }
    }
    if (wpc <= 0) wpc = a.sched ? 32 : 8;
    if (cps <= 0) cps = 1;
    const size_t cap = a.sched ? (size_t)233472 / cps - 1024 : (size_t)226 * 1024;
    while (wpc > 1 && lap_warp_smem(a.m, cpl) * wpc > cap) wpc--;
    return cpl == 1 ? launch_lap_on<1>(a, num_sms, wpc, cps, st) : launch_lap_on<2>(a, num_sms, wpc, cps, st);
}

cudaError_t launch_lap_level(LapLevel lvl, const Geom &g, double *D, double *C, double *B, Ctl *ctl,
                             double *trace, int num_sms, int lap_warps, Sched *sched, cudaStream_t st)
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
        wpc = lap_warps;
        a.mag_n1 = (uint32_t)((0x100000000ull + (uint64_t)(n - 2)) / (uint64_t)(n - 1));
        for (int i = 0; i + 1 < n; i++) {
            const uint64_t d = (uint64_t)(n - 1 - i) * (uint64_t)(n - 1);
            a.mag_pj[i] = (uint32_t)((0x100000000ull + d - 1) / d);
        }
        a.sched = sched;
        break;
    case LAP_L1_ACC:
    case LAP_L1_SET:
        a.m = n - 1; a.count = (int64_t)n * n; a.ld = g.ldc; a.src = C; a.dst = C;
        wpc = 1;
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

cudaError_t launch_lap_l2_local(const Geom &g, double *Dloc, int64_t count, double *Sout, Ctl *ctl, int num_sms,
                                int lap_cfg, Sched *sched, cudaStream_t st)
{
    if (count <= 0) return cudaSuccess;
    LapArgs a{};
    a.lvl = LAP_L2;
    a.g = g;
    a.ctl = ctl;
    a.m = g.n - 2;
    a.count = count;
    a.ld = g.ld2;
    a.src = Dloc;
    a.dst = Dloc;
    a.bo.S = Sout;
    a.sched = sched;  // dynamic queue (reset by k_sigma)
    return dispatch_lap(a, num_sms, lap_cfg, st);
}

cudaError_t launch_rlt1_init(const Node &parent, const Rlt1Batch &R, const int64_t *F, const int64_t *Dist,
                             cudaStream_t st)
{
    const int np = R.g.n;
    const int64_t tot = (int64_t)np * np * np * np + (int64_t)np * np;
    int bx = (int)((tot + 255) / 256);
    if (bx > 64) bx = 64;
    dim3 grid(bx, R.K);
    k_rlt1_init<<<grid, 256, 0, st>>>(parent, R, F, Dist);
    return cudaGetLastError();
}

cudaError_t launch_rlt1_pair(const Rlt1Batch &R, cudaStream_t st)
{
    const int64_t tot = (int64_t)R.g.n * R.g.n * R.g.n * R.g.n * R.K;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_rlt1_pair<<<blocks, 256, 0, st>>>(R);
    return cudaGetLastError();
}

cudaError_t launch_rlt1_lap(const Rlt1Batch &R, int level1, int acc, int num_sms, cudaStream_t st)
{
    LapArgs a{};
    a.g = R.g;
    const int np = R.g.n;
    if (level1) {
        a.lvl = acc ? LAP_L1_ACC : LAP_L1_SET;
        a.m = np - 1;
        a.count = (int64_t)R.K * np * np;
        a.ld = R.g.ldc;
        a.src = a.dst = R.C;
        a.B = R.B;
        a.bdiv = (int64_t)np * np;
        a.bstr = R.bstr;
        return dispatch_lap(a, num_sms, 8, st);
    }
    a.lvl = LAP_L0_MULTI;
    a.m = np;
    a.count = R.K;
    a.ld = R.bstr;
    a.src = a.dst = R.B;
    a.lbm = R.lbd;
    return dispatch_lap(a, num_sms, 4, st);
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
    return dispatch_lap(a, num_sms, 2, st);
}

}  // namespace rlt2
