/*
 * oracle/rlt2_oracle.c — CPU ORACLE of the RLT2 dual-ascent lower bound.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1510_02065_b200/) never links, imports or executes it, and shares no code,
 * header, table or constant generator with it.
 *
 * Plain, slow, obviously correct: fp64 everywhere (PAPER.md is silent on precision,
 * P:259; reading R16), int64 for the instance data, no blocking, fusion or
 * reordering beyond what the paper's Algorithm 1 states.
 * Compile with -O2 -ffp-contract=off (no FMA contraction; there are no a*b+c
 * patterns in the fp64 arithmetic anyway).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source).
 *   QAP, Eqs. (1)-(4)
 *   RLT2 model, complementary coefficients       P:105-164 (Eqs. rlt2a-rlt2j)
 *   Algorithm 1 (dual ascent)
 *   Cost concentration = LAP + residuals
 *   Cost spreading
 *   Complementary transfer
 *   Complementary submatrices (halved D)
 * Readings of silent / ambiguous points are numbered R1.. in DESIGN.md §3.
 *
 * Layouts (also the export layout of the C ABI's qap_rlt2_dual_copy, which the GPU
 * library implements independently):
 *   B : n×n row-major, b_ij.
 *   C : n² blocks C_ij (i,j row-major), each (n-1)×(n-1) row-major; row k≠i at
 *       index k-[k>i], column l≠j at index l-[l>j].
 *   D : stored blocks D{ij,kl} with i<k, l≠j, enumerated in (i,j,k,l) lexicographic
 *       order; each (n-2)×(n-2) row-major; row p∉{i,k} at p-[p>i]-[p>k], column
 *       q∉{j,l} at q-[q>j]-[q>l].  D{kl,ij} is the SAME stored block.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_E_ARG 1
#define ORC_E_NUMERIC 5
#define ORC_E_STATE 6

/* Host threads for the loops over independent units (blocks, classes, pairs (i,j)): 1 by
 * default (the tests); bench.py's all-cores baseline raises it.  Every unit writes only its
 * own entries and runs its operations in the fixed order below, so the result is
 * bit-identical for every thread count (SURVEY.md §8(d) oracle timing mode (ii)).        */
static int g_threads = 1;
void oracle_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int oracle_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------------- */
/* O2 — one linear assignment problem.                           */
/* ------------------------------------------------------------------------- */
/*
 * Shortest-augmenting-path form of the Hungarian algorithm (P:205 cites Munkres;
 * reading R4: an exact Hungarian-type solver).  Munkres' row reduction first (u = row
 * minima, v = 0, rows matched greedily to the lowest column of their minimum), then the
 * classic O(m^3) potentials form for the rows left: each is inserted, in ascending
 * order, by a Dijkstra search over reduced costs; column 0 is a dummy holding the row
 * being inserted.  v starts at 0 and only Dijkstra distances are taken off it, which
 * yields the canonical dual of reading R5 (v componentwise maximal subject to v <= 0).
 *
 * Tie rule (reading R6): the next column settled is the unused column minimising
 * the key (minv[j], column already matched?, j) lexicographically — smallest
 * tentative distance, then prefer a FREE column, then the lowest index.
 *
 * Outputs (reading R8, R9):
 *   assign[r]  column of row r;
 *   *S         = sum_{r=0..m-1} M[r][assign[r]], summed sequentially in row order;
 *   u, v       the row / column duals;
 *   R[r][s]    = (M[r][s] - u[r]) - v[s]; negatives in [-tau, 0) -> +0, below
 *               -tau -> ORC_E_NUMERIC; R[r][assign[r]] = +0; -0 -> +0;
 *               tau = 1e-9 * max(1, max|M|).
 * R may alias M.  *steps counts Dijkstra steps (settled columns).
 */
int oracle_lap(int m, const double *M, double *R, int32_t *assign, double *u_out,
               double *v_out, double *S_out, int64_t *steps_out)
{
    if (m < 1) return ORC_E_ARG;
    double *u = calloc((size_t)m + 1, sizeof(double));
    double *v = calloc((size_t)m + 1, sizeof(double));
    double *minv = malloc(((size_t)m + 1) * sizeof(double));
    int *p = calloc((size_t)m + 1, sizeof(int));
    int *way = calloc((size_t)m + 1, sizeof(int));
    char *used = malloc((size_t)m + 1);
    int64_t steps = 0;

    /* Munkres' first step (P:205 cites the Hungarian method of Munkres; reading R4): every
     * row is reduced by its minimum, u[r] = min_s M[r][s], v = 0.  Initial partial
     * assignment on the zeros this creates: for r ascending, row r takes the lowest column
     * attaining its minimum unless an earlier row took that column.  The dual stays
     * feasible and v = 0 is untouched, so the final dual is still the canonical one of
     * reading R5 (pinned by Bellman–Ford in tests/test_oracle_lap.py).                   */
    char *rmatched = calloc((size_t)m + 1, 1);
    for (int r = 1; r <= m; r++) {
        int a = 1;
        for (int j = 2; j <= m; j++)
            if (M[(size_t)(r - 1) * m + (j - 1)] < M[(size_t)(r - 1) * m + (a - 1)]) a = j;
        u[r] = M[(size_t)(r - 1) * m + (a - 1)];
        if (p[a] == 0) { p[a] = r; rmatched[r] = 1; }
    }

    /* the remaining rows, ascending, each by one shortest-augmenting-path search: Dijkstra
     * over the reduced costs from row i, with tentative distances minv[j] and the distance
     * dist[j] of every column when it is settled; the potentials change once, at the end of
     * the search (the augmentation of Jonker & Volgenant): every settled column j moves by
     * dfin - dist[j], dfin = the distance of the free column reached.  In exact arithmetic
     * this is the textbook step-by-step update (u[p[j]] += delta, v[j] -= delta for the used
     * columns after every step).                                                          */
    double *dist = malloc(((size_t)m + 1) * sizeof(double));
    for (int i = 1; i <= m; i++) {
        if (rmatched[i]) continue;
        p[0] = i;
        int j0 = 0;
        for (int j = 0; j <= m; j++) { minv[j] = INFINITY; used[j] = 0; }
        dist[0] = 0.0;
        do {
            used[j0] = 1;
            int i0 = p[j0];
            const double c = dist[j0] - u[i0];      /* distance of row i0 minus its potential */
            for (int j = 1; j <= m; j++) {
                if (used[j]) continue;
                double cur = (M[(size_t)(i0 - 1) * m + (j - 1)] - v[j]) + c;
                if (cur < minv[j]) { minv[j] = cur; way[j] = j0; }
            }
            int j1 = -1;
            for (int j = 1; j <= m; j++) {   /* ascending j: lowest index wins exact ties */
                if (used[j]) continue;
                if (j1 < 0 || minv[j] < minv[j1] ||
                    (minv[j] == minv[j1] && p[j] == 0 && p[j1] != 0))
                    j1 = j;
            }
            dist[j1] = minv[j1];
            j0 = j1;
            steps++;
        } while (p[j0] != 0);
        const double dfin = dist[j0];
        for (int j = 0; j <= m; j++) {
            if (!used[j]) continue;
            const double t = dfin - dist[j];
            u[p[j]] = u[p[j]] + t;
            v[j] = v[j] - t;
        }
        do { int j1 = way[j0]; p[j0] = p[j1]; j0 = j1; } while (j0);
    }
    free(dist);

    int32_t *a = malloc((size_t)m * sizeof(int32_t));
    for (int j = 1; j <= m; j++) a[p[j] - 1] = j - 1;
    double S = 0.0;
    for (int r = 0; r < m; r++) S = S + M[(size_t)r * m + a[r]];
    double maxabs = 0.0;
    for (size_t t = 0; t < (size_t)m * m; t++) if (fabs(M[t]) > maxabs) maxabs = fabs(M[t]);
    double tau = 1e-9 * (maxabs > 1.0 ? maxabs : 1.0);
    int st = ORC_OK;
    for (int r = 0; r < m; r++) {
        for (int s = 0; s < m; s++) {
            double x = (M[(size_t)r * m + s] - u[r + 1]) - v[s + 1];
            if (x < 0.0) {
                if (x >= -tau) x = 0.0; else st = ORC_E_NUMERIC;
            }
            if (s == a[r]) x = 0.0;
            if (x == 0.0) x = 0.0;          /* canonicalise -0 to +0 */
            R[(size_t)r * m + s] = x;
        }
    }
    if (assign) memcpy(assign, a, (size_t)m * sizeof(int32_t));
    if (u_out) for (int r = 0; r < m; r++) u_out[r] = u[r + 1];
    if (v_out) for (int s = 0; s < m; s++) v_out[s] = v[s + 1];
    if (S_out) *S_out = S;
    if (steps_out) *steps_out = steps;
    free(u); free(v); free(minv); free(p); free(way); free(used); free(a); free(rmatched);
    return st;
}

/* Brute-force LAP by enumerating all m! assignments (test pin; m <= 10).        */
static void bf_rec(int m, const double *M, int r, int32_t *perm, char *taken,
                   double acc, double *best, int32_t *best_perm)
{
    if (r == m) {
        if (acc < *best) { *best = acc; memcpy(best_perm, perm, (size_t)m * sizeof(int32_t)); }
        return;
    }
    for (int s = 0; s < m; s++) {
        if (taken[s]) continue;
        taken[s] = 1; perm[r] = s;
        bf_rec(m, M, r + 1, perm, taken, acc + M[(size_t)r * m + s], best, best_perm);
        taken[s] = 0;
    }
}

int oracle_lap_bruteforce(int m, const double *M, double *best_out, int32_t *assign)
{
    if (m < 1 || m > 10) return ORC_E_ARG;
    int32_t perm[10], bp[10];
    char taken[10] = {0};
    double best = INFINITY;
    bf_rec(m, M, 0, perm, taken, 0.0, &best, bp);
    *best_out = best;
    if (assign) memcpy(assign, bp, (size_t)m * sizeof(int32_t));
    return ORC_OK;
}

/* Brute-force QAP optimum (test pin, not the method): enumerate all N! permutations in
 * lexicographic order and evaluate the Koopmans–Beckmann objective of P:84,
 * sum_{i,k} f_ik d_{pi(i) pi(k)}, accumulated facility by facility (the terms of facility d
 * with the facilities 0..d fixed before it).  Returns the minimum and the first
 * permutation reaching it.  N <= 13 (13! = 6.2e9 leaves).                            */
typedef struct { int N; const int64_t *F, *Dist; int32_t perm[16]; char used[16];
                 int64_t best; int32_t best_perm[16]; } bfq_ctx;

static void bfq_rec(bfq_ctx *c, int d, int64_t partial)
{
    if (d == c->N) {
        if (partial < c->best) { c->best = partial; memcpy(c->best_perm, c->perm, sizeof c->perm); }
        return;
    }
    const int N = c->N;
    for (int x = 0; x < N; x++) {
        if (c->used[x]) continue;
        int64_t add = c->F[d * N + d] * c->Dist[x * N + x];
        for (int t = 0; t < d; t++)
            add += c->F[d * N + t] * c->Dist[x * N + c->perm[t]] + c->F[t * N + d] * c->Dist[c->perm[t] * N + x];
        c->used[x] = 1; c->perm[d] = x;
        bfq_rec(c, d + 1, partial + add);
        c->used[x] = 0;
    }
}

int oracle_qap_bruteforce(int N, const int64_t *F, const int64_t *Dist, int64_t *best_out, int32_t *perm_out)
{
    if (N < 1 || N > 13) return ORC_E_ARG;
    bfq_ctx c;
    memset(&c, 0, sizeof c);
    c.N = N; c.F = F; c.Dist = Dist; c.best = INT64_MAX;
    bfq_rec(&c, 0, 0);
    *best_out = c.best;
    memcpy(perm_out, c.best_perm, sizeof(int32_t) * N);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Dual state: the matrices B, C, D of P:163-164.                            */
/* ------------------------------------------------------------------------- */
typedef struct {
    int N, n;             /* original size, reduced (free) size                 */
    int nfix;
    int32_t fac[64], loc[64];  /* fixed pairs Φ                                 */
    int32_t I[64], J[64];      /* free facilities / locations, ascending        */
    int64_t kappa;        /* cost among the fixed pairs (int64, exact)          */
    int64_t *Fr, *Dr;     /* reduced F' = F[I][I], D' = Dist[J][J]               */
    int64_t *B0;          /* initial b (int64)                                  */
    double *B, *C, *D;
    int64_t nC, nD, nblk; /* entry counts; number of stored D blocks            */
    int32_t *blk;         /* [i][j][k][l] -> stored block id (i<k, j!=l) or -1   */
    double lb_dual;       /* accumulated concentration sums (LB - kappa)        */
    double lb_glb;
    int fresh;            /* 1: iteration 0 not yet run                          */
} ostate;

static int excl1(int x, int a) { return x - (x > a); }                 /* index skipping a    */
static int excl2(int x, int a, int b) { return x - (x > a) - (x > b); } /* index skipping a, b */

static size_t cidx(const ostate *s, int i, int j, int k, int l)        /* c_ij[kl]            */
{
    int n = s->n;
    return ((size_t)(i * n + j)) * (size_t)(n - 1) * (n - 1) + (size_t)excl1(k, i) * (n - 1) + excl1(l, j);
}

/* Logical level-2 coefficient d_{ij,kl,pq}: stored once per complementary block pair. */
static double *dref(const ostate *s, int i, int j, int k, int l, int p, int q)
{
    int n = s->n;
    if (i > k) { int t = i; i = k; k = t; t = j; j = l; l = t; }
    int32_t b = s->blk[((size_t)(i * n + j) * n + k) * n + l];
    return s->D + (size_t)b * (n - 2) * (n - 2) + (size_t)excl2(p, i, k) * (n - 2) + excl2(q, j, l);
}

void oracle_state_free(ostate *s)
{
    if (!s) return;
    free(s->Fr); free(s->Dr); free(s->B0); free(s->B); free(s->C); free(s->D); free(s->blk);
    free(s);
}

/*
 * O0 reduce + O1 init (reading R2 for b_ij; cold child of reading R19).
 * Fixed pairs Φ = {(fac[t], loc[t])}.  With I, J the free facilities / locations:
 *   b0_ab = f_{I_a I_a} d_{J_b J_b} + sum_t ( f_{fac_t I_a} d_{loc_t J_b} + f_{I_a fac_t} d_{J_b loc_t} )
 *   c_ij[kl] = f'_ik d'_jl
 *   d = 0
 *   kappa = sum_{t,t'} f_{fac_t fac_t'} d_{loc_t loc_t'}   (fixed-fixed cost, diagonal included)
 */
ostate *oracle_state_new(int N, const int64_t *F, const int64_t *Dist, int nfix,
                         const int32_t *fac, const int32_t *loc, int *err)
{
    *err = ORC_E_ARG;
    if (N < 3 || N > 64 || nfix < 0 || N - nfix < 3) return NULL;
    char uf[64] = {0}, ul[64] = {0};
    for (int t = 0; t < nfix; t++) {
        if (fac[t] < 0 || fac[t] >= N || loc[t] < 0 || loc[t] >= N) return NULL;
        if (uf[fac[t]] || ul[loc[t]]) return NULL;
        uf[fac[t]] = ul[loc[t]] = 1;
    }
    ostate *s = calloc(1, sizeof(ostate));
    s->N = N; s->nfix = nfix; s->n = N - nfix;
    int n = s->n;
    for (int t = 0; t < nfix; t++) { s->fac[t] = fac[t]; s->loc[t] = loc[t]; }
    int a = 0, b = 0;
    for (int x = 0; x < N; x++) { if (!uf[x]) s->I[a++] = x; if (!ul[x]) s->J[b++] = x; }

    s->kappa = 0;
    for (int t = 0; t < nfix; t++)
        for (int t2 = 0; t2 < nfix; t2++)
            s->kappa += F[fac[t] * N + fac[t2]] * Dist[loc[t] * N + loc[t2]];

    s->Fr = malloc(sizeof(int64_t) * n * n);
    s->Dr = malloc(sizeof(int64_t) * n * n);
    for (int x = 0; x < n; x++)
        for (int y = 0; y < n; y++) {
            s->Fr[x * n + y] = F[s->I[x] * N + s->I[y]];
            s->Dr[x * n + y] = Dist[s->J[x] * N + s->J[y]];
        }
    s->B0 = malloc(sizeof(int64_t) * n * n);
    for (int x = 0; x < n; x++)
        for (int y = 0; y < n; y++) {
            int64_t v = F[s->I[x] * N + s->I[x]] * Dist[s->J[y] * N + s->J[y]];
            for (int t = 0; t < nfix; t++)
                v += F[fac[t] * N + s->I[x]] * Dist[loc[t] * N + s->J[y]]
                   + F[s->I[x] * N + fac[t]] * Dist[s->J[y] * N + loc[t]];
            s->B0[x * n + y] = v;
        }

    s->nC = (int64_t)n * n * (n - 1) * (n - 1);
    s->nblk = (int64_t)n * n * (n - 1) * (n - 1) / 2;
    s->nD = s->nblk * (n - 2) * (n - 2);
    s->blk = malloc(sizeof(int32_t) * (size_t)n * n * n * n);
    for (size_t t = 0; t < (size_t)n * n * n * n; t++) s->blk[t] = -1;
    int32_t id = 0;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = i + 1; k < n; k++)
                for (int l = 0; l < n; l++)
                    if (l != j) s->blk[((size_t)(i * n + j) * n + k) * n + l] = id++;

    s->B = malloc(sizeof(double) * n * n);
    s->C = malloc(sizeof(double) * (size_t)s->nC);
    s->D = malloc(sizeof(double) * (size_t)s->nD);
    if (!s->B || !s->C || !s->D) { oracle_state_free(s); *err = ORC_E_ARG; return NULL; }
    for (int x = 0; x < n * n; x++) s->B[x] = (double)s->B0[x];
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = 0; k < n; k++)
                for (int l = 0; l < n; l++)
                    if (k != i && l != j)
                        s->C[cidx(s, i, j, k, l)] = (double)(s->Fr[i * n + k] * s->Dr[j * n + l]);
    for (int64_t t = 0; t < s->nD; t++) s->D[t] = 0.0;
    s->lb_dual = 0.0;
    s->lb_glb = 0.0;
    s->fresh = 1;
    *err = ORC_OK;
    return s;
}

/*
 * Warm child (fold rules of SPEC S:368, derived in DESIGN.md
 * reading R31 from the evaluation identity of P:169).  The child of node s fixing the
 * reduced facility a at the reduced location b inherits s's dual state; every completion
 * keeps its cost:
 *   kappa' = kappa,  lb_dual' = lb_dual + b_ab
 *   b'_xy      = (b_xy + c_ab[xy]) + c_xy[ab]
 *   c'_xy[zw]  = c_xy[zw] + ((d_{ab,xy,zw} + d_{ab,zw,xy}) + d_{xy,zw,ab})    (logical d)
 *   d'_{xy,zw}[pq] = d_{xy,zw}[pq]
 * for x, z != a and y, w != b; child indices are the parent's with a and b removed.
 * Entries of assignments that the fix makes infeasible (location b, facility a) are
 * dropped.  The child is "fresh": its next bound starts with iteration 0 (concentrate
 * C -> B -> LB), then the loop.  Returns NULL on bad arguments (*err).
 */
ostate *oracle_state_fold(const ostate *s, int a, int b, int *err)
{
    *err = ORC_E_ARG;
    int n = s->n, n1 = n - 1;
    if (n1 < 3 || a < 0 || a >= n || b < 0 || b >= n) return NULL;
    ostate *c = calloc(1, sizeof(ostate));
    c->N = s->N; c->n = n1; c->nfix = s->nfix + 1;
    for (int t = 0; t < s->nfix; t++) { c->fac[t] = s->fac[t]; c->loc[t] = s->loc[t]; }
    c->fac[s->nfix] = s->I[a]; c->loc[s->nfix] = s->J[b];
    for (int x = 0; x < n1; x++) { c->I[x] = s->I[x + (x >= a)]; c->J[x] = s->J[x + (x >= b)]; }
    c->kappa = s->kappa;
    c->Fr = malloc(sizeof(int64_t) * n1 * n1);
    c->Dr = malloc(sizeof(int64_t) * n1 * n1);
    c->B0 = calloc((size_t)n1 * n1, sizeof(int64_t));
    for (int x = 0; x < n1; x++)
        for (int y = 0; y < n1; y++) {
            c->Fr[x * n1 + y] = s->Fr[(x + (x >= a)) * n + (y + (y >= a))];
            c->Dr[x * n1 + y] = s->Dr[(x + (x >= b)) * n + (y + (y >= b))];
        }
    c->nC = (int64_t)n1 * n1 * (n1 - 1) * (n1 - 1);
    c->nblk = (int64_t)n1 * n1 * (n1 - 1) * (n1 - 1) / 2;
    c->nD = c->nblk * (n1 - 2) * (n1 - 2);
    c->blk = malloc(sizeof(int32_t) * (size_t)n1 * n1 * n1 * n1);
    for (size_t t = 0; t < (size_t)n1 * n1 * n1 * n1; t++) c->blk[t] = -1;
    int32_t id = 0;
    for (int i = 0; i < n1; i++)
        for (int j = 0; j < n1; j++)
            for (int k = i + 1; k < n1; k++)
                for (int l = 0; l < n1; l++)
                    if (l != j) c->blk[((size_t)(i * n1 + j) * n1 + k) * n1 + l] = id++;
    c->B = malloc(sizeof(double) * n1 * n1);
    c->C = malloc(sizeof(double) * (size_t)c->nC);
    c->D = malloc(sizeof(double) * (size_t)(c->nD > 0 ? c->nD : 1));
    if (!c->B || !c->C || !c->D) { oracle_state_free(c); return NULL; }
#define PX(x) ((x) + ((x) >= a))  /* child facility index -> parent */
#define PY(y) ((y) + ((y) >= b))  /* child location index -> parent */
    for (int x = 0; x < n1; x++)
        for (int y = 0; y < n1; y++) {
            int X = PX(x), Y = PY(y);
            c->B[x * n1 + y] = (s->B[X * n + Y] + s->C[cidx(s, a, b, X, Y)]) + s->C[cidx(s, X, Y, a, b)];
        }
    for (int x = 0; x < n1; x++)
        for (int y = 0; y < n1; y++)
            for (int z = 0; z < n1; z++)
                for (int w = 0; w < n1; w++) {
                    if (z == x || w == y) continue;
                    int X = PX(x), Y = PY(y), Z = PX(z), W = PY(w);
                    double e1 = *dref(s, a, b, X, Y, Z, W);
                    double e2 = *dref(s, a, b, Z, W, X, Y);
                    double e3 = *dref(s, X, Y, Z, W, a, b);
                    c->C[cidx(c, x, y, z, w)] = s->C[cidx(s, X, Y, Z, W)] + ((e1 + e2) + e3);
                }
    for (int x = 0; x < n1; x++)
        for (int y = 0; y < n1; y++)
            for (int z = x + 1; z < n1; z++)
                for (int w = 0; w < n1; w++) {
                    if (w == y) continue;
                    for (int p = 0; p < n1; p++) {
                        if (p == x || p == z) continue;
                        for (int q = 0; q < n1; q++) {
                            if (q == y || q == w) continue;
                            *dref(c, x, y, z, w, p, q) = *dref(s, PX(x), PY(y), PX(z), PY(w), PX(p), PY(q));
                        }
                    }
                }
#undef PX
#undef PY
    c->lb_dual = s->lb_dual + s->B[a * n + b];
    c->lb_glb = 0.0;
    c->fresh = 1;
    *err = ORC_OK;
    return c;
}

/* ---- the operations of Algorithm 1 ---------------------------------------- */

/* Cost concentration C -> B ("b_ij <- Concentrate(c_ij)"): for (i,j) in
 * row-major order, LAP on C_ij (size n-1), C_ij <- residual, b_ij += S.          */
int oracle_concentrate_c(ostate *s)
{
    int n = s->n, m = n - 1, err = ORC_OK;
#pragma omp parallel for collapse(2) schedule(dynamic) num_threads(g_threads)
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double *blk = s->C + (size_t)(i * n + j) * m * m;
            double S;
            int st = oracle_lap(m, blk, blk, NULL, NULL, NULL, &S, NULL);
            if (st) {
#pragma omp atomic write
                err = st;
            }
            s->B[i * n + j] = s->B[i * n + j] + S;
        }
    return err;
}

/* Cost concentration B -> LB ("LB' <- Concentrate(B)", "LB <- LB + LB'"). */
int oracle_concentrate_b(ostate *s, double *lbprime)
{
    double S;
    int st = oracle_lap(s->n, s->B, s->B, NULL, NULL, NULL, &S, NULL);
    if (st) return st;
    s->lb_dual = s->lb_dual + S;
    if (lbprime) *lbprime = S;
    return ORC_OK;
}

/* O3 — iteration 0 (reading R1): concentrate C -> B -> LB; the Gilmore–Lawler bound. */
int oracle_iteration0(ostate *s)
{
    int st = oracle_concentrate_c(s);
    if (st) return st;
    st = oracle_concentrate_b(s, NULL);
    if (st) return st;
    s->lb_glb = (double)s->kappa + s->lb_dual;
    s->fresh = 0;
    return ORC_OK;
}

/* O4 — spreading B -> C: c_ijkl += b_ij/(n-1) for all k!=i, l!=j; then b = 0. */
int oracle_spread_b(ostate *s)
{
    int n = s->n, m = n - 1;
#pragma omp parallel for collapse(2) schedule(static) num_threads(g_threads)
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            double beta = s->B[i * n + j] / (double)(n - 1);
            double *blk = s->C + (size_t)(i * n + j) * m * m;
            for (int t = 0; t < m * m; t++) blk[t] = blk[t] + beta;
            s->B[i * n + j] = 0.0;
        }
    return ORC_OK;
}

/* O5 — spreading C -> D followed by the transfer between complementary
 * costs of D.
 *   Spreading with shared storage (reading R12): the stored entry of block
 *   D{ij,kl} (i<k) stands for both logical entries d_{ijkl,pq} and d_{klij,pq}; it
 *   receives sigma = (c_ij[kl] + c_kl[ij]) / (2(n-2)), then C = 0.
 *   Transfer (reading R11): for every class of the 6 complementary coefficients of
 *   Eq. (rlt2g) — i<k<p, distinct j,l,q — the 3 stored members
 *     e1 = d_{ij,kl,pq}, e2 = d_{ij,pq,kl}, e3 = d_{kl,pq,ij}
 *   (spread included) are all set to their mean ((e1+e2)+e3)/3.               */
int oracle_spread_c_transfer_d(ostate *s)
{
    int n = s->n;
    double *sigma = malloc(sizeof(double) * (size_t)s->nblk);
#pragma omp parallel for collapse(2) schedule(static) num_threads(g_threads)
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = i + 1; k < n; k++)
                for (int l = 0; l < n; l++) {
                    if (l == j) continue;
                    int32_t b = s->blk[((size_t)(i * n + j) * n + k) * n + l];
                    sigma[b] = (s->C[cidx(s, i, j, k, l)] + s->C[cidx(s, k, l, i, j)]) / (double)(2 * (n - 2));
                }
    /* every stored entry belongs to exactly one class: the classes are independent, and
       the loop order (here (i, j) outermost for the threads) changes no bit */
#pragma omp parallel for collapse(2) schedule(dynamic) num_threads(g_threads)
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = i + 1; k < n; k++)
                for (int p = k + 1; p < n; p++)
                    for (int l = 0; l < n; l++) {
                        if (l == j) continue;
                        for (int q = 0; q < n; q++) {
                            if (q == j || q == l) continue;
                            double *e1 = dref(s, i, j, k, l, p, q);
                            double *e2 = dref(s, i, j, p, q, k, l);
                            double *e3 = dref(s, k, l, p, q, i, j);
                            double h1 = *e1 + sigma[s->blk[((size_t)(i * n + j) * n + k) * n + l]];
                            double h2 = *e2 + sigma[s->blk[((size_t)(i * n + j) * n + p) * n + q]];
                            double h3 = *e3 + sigma[s->blk[((size_t)(k * n + l) * n + p) * n + q]];
                            double mu = ((h1 + h2) + h3) / 3.0;
                            *e1 = mu; *e2 = mu; *e3 = mu;
                        }
                    }
    for (int64_t t = 0; t < s->nC; t++) s->C[t] = 0.0;
    free(sigma);
    return ORC_OK;
}

/* O6 — cost concentration D -> C (halved per P:250-252): for each
 * stored block, LAP (size n-2), block <- residual, S credited to both complementary
 * coefficients c_ij[kl] and c_kl[ij] (reading R12).                              */
int oracle_concentrate_d(ostate *s)
{
    int n = s->n, m = n - 2, err = ORC_OK;
    /* each block credits only its own two coefficients: blocks are independent */
#pragma omp parallel for collapse(2) schedule(dynamic) num_threads(g_threads)
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = i + 1; k < n; k++)
                for (int l = 0; l < n; l++) {
                    if (l == j) continue;
                    int32_t b = s->blk[((size_t)(i * n + j) * n + k) * n + l];
                    double *blk = s->D + (size_t)b * m * m;
                    double S;
                    int st = oracle_lap(m, blk, blk, NULL, NULL, NULL, &S, NULL);
                    if (st) {
#pragma omp atomic write
                        err = st;
                    }
                    s->C[cidx(s, i, j, k, l)] = s->C[cidx(s, i, j, k, l)] + S;
                    s->C[cidx(s, k, l, i, j)] = s->C[cidx(s, k, l, i, j)] + S;
                }
    return err;
}

/* Transfer between complementary costs of C (reading R13: pair mean).  */
int oracle_transfer_c(ostate *s)
{
    int n = s->n;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++)
            for (int k = i + 1; k < n; k++)
                for (int l = 0; l < n; l++) {
                    if (l == j) continue;
                    double *a = s->C + cidx(s, i, j, k, l), *b = s->C + cidx(s, k, l, i, j);
                    double mu = (*a + *b) / 2.0;
                    *a = mu; *b = mu;
                }
    return ORC_OK;
}

/* One iteration of Algorithm 1's loop body, in the paper's order.     */
int oracle_iteration(ostate *s, double *lbprime)
{
    int st;
    if ((st = oracle_spread_b(s))) return st;
    if ((st = oracle_spread_c_transfer_d(s))) return st;
    if ((st = oracle_concentrate_d(s))) return st;
    if ((st = oracle_transfer_c(s))) return st;
    if ((st = oracle_concentrate_c(s))) return st;
    return oracle_concentrate_b(s, lbprime);
}

/*
 * The bound.  If the state is fresh, iteration 0 (reading R1) runs
 * first; then up to T iterations.  Stop rule (readings R14, R15), with
 * LB = (double)kappa + lb_dual:
 *   UB finite and LB > UB - 1 + 1e-6          -> status 2 (pruned)
 *   UB finite, K > 0 and LB'/UB < K            -> status 1 (converged)
 *   otherwise after T iterations               -> status 0 (iteration cap)
 * lb_trace (optional, length >= T) receives LB after each iteration.
 */
int oracle_bound(ostate *s, int T, double K, double UB, double *lb_out, double *lb_glb_out,
                 int *iters_out, int *status_out, double *lb_trace)
{
    int st, iters = 0, status = 0;
    if (s->fresh && (st = oracle_iteration0(s))) return st;
    double LB = (double)s->kappa + s->lb_dual;
    int ub_finite = isfinite(UB);
    if (ub_finite && LB > UB - 1.0 + 1e-6) status = 2;
    while (status == 0 && iters < T) {
        double lbp;
        if ((st = oracle_iteration(s, &lbp))) return st;
        LB = (double)s->kappa + s->lb_dual;
        if (lb_trace) lb_trace[iters] = LB;
        iters++;
        if (ub_finite) {
            if (LB > UB - 1.0 + 1e-6) status = 2;
            else if (K > 0.0 && lbp / UB < K) status = 1;
        }
    }
    if (lb_out) *lb_out = LB;
    if (lb_glb_out) *lb_glb_out = s->lb_glb;
    if (iters_out) *iters_out = iters;
    if (status_out) *status_out = status;
    return ORC_OK;
}

/*
 * RLT1 dual ascent ("the costs concentration follows the RLT1 dual algorithm similar to
 * Section 4, except by the operations with transfer costs of D matrix"):
 * iteration 0 as above, then per iteration: spread B->C, transfer between the
 * complementary costs of C (pair mean, reading R13 — NOT a no-op here), concentrate
 * C->B, concentrate B->LB.  D is neither read nor written.
 */
int oracle_rlt1_iteration(ostate *s, double *lbprime)
{
    int st;
    if ((st = oracle_spread_b(s))) return st;
    if ((st = oracle_transfer_c(s))) return st;
    if ((st = oracle_concentrate_c(s))) return st;
    return oracle_concentrate_b(s, lbprime);
}

int oracle_rlt1_bound(ostate *s, int T, double *lb_out)
{
    int st;
    if (s->fresh && (st = oracle_iteration0(s))) return st;
    for (int t = 0; t < T; t++) {
        double lbp;
        if ((st = oracle_rlt1_iteration(s, &lbp))) return st;
    }
    *lb_out = (double)s->kappa + s->lb_dual;
    return ORC_OK;
}

/*
 * Strong branching: estimate every candidate child (free facility I[a] at free
 * location J[b]) of the node Φ = (fac, loc) by a cold RLT1 bound with T iterations
 * (est[a*n + b], n = N - nfix), then score each row a by min_b est and each column b by
 * min_a est and select the line with the MAXIMUM score (SPEC S:374-382 max-min reading;
 * ties: lowest index, row preferred over column).  *kind = 0 row / 1 column, *index =
 * reduced index of the line.  Requires n >= 4 (children have >= 3 free facilities).
 */
int oracle_strong_branch(int N, const int64_t *F, const int64_t *Dist, int nfix, const int32_t *fac,
                         const int32_t *loc, int T, double *est, int *kind, int *index)
{
    int n = N - nfix;
    if (n < 4) return ORC_E_ARG;
    char uf[64] = {0}, ul[64] = {0};
    for (int t = 0; t < nfix; t++) { uf[fac[t]] = 1; ul[loc[t]] = 1; }
    int32_t I[64], J[64];
    int ni = 0, nj = 0;
    for (int x = 0; x < N; x++) { if (!uf[x]) I[ni++] = x; if (!ul[x]) J[nj++] = x; }
    int32_t cf[64], cl[64];
    for (int t = 0; t < nfix; t++) { cf[t] = fac[t]; cl[t] = loc[t]; }
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) {
            cf[nfix] = I[a];
            cl[nfix] = J[b];
            int err;
            ostate *s = oracle_state_new(N, F, Dist, nfix + 1, cf, cl, &err);
            if (!s) return err;
            int st = oracle_rlt1_bound(s, T, &est[a * n + b]);
            oracle_state_free(s);
            if (st) return st;
        }
    double best = -INFINITY;
    *kind = 0;
    *index = 0;
    for (int a = 0; a < n; a++) {          /* rows first: a row wins exact ties with a column */
        double sc = INFINITY;
        for (int b = 0; b < n; b++) if (est[a * n + b] < sc) sc = est[a * n + b];
        if (sc > best) { best = sc; *kind = 0; *index = a; }
    }
    for (int b = 0; b < n; b++) {
        double sc = INFINITY;
        for (int a = 0; a < n; a++) if (est[a * n + b] < sc) sc = est[a * n + b];
        if (sc > best) { best = sc; *kind = 1; *index = b; }
    }
    return ORC_OK;
}

/* ---- accessors for the Python wrapper -------------------------------------- */
int oracle_state_n(const ostate *s) { return s->n; }
int64_t oracle_state_kappa(const ostate *s) { return s->kappa; }
double oracle_state_lb_dual(const ostate *s) { return s->lb_dual; }
double oracle_state_lb_glb(const ostate *s) { return s->lb_glb; }
void oracle_state_sizes(const ostate *s, int64_t *nB, int64_t *nC, int64_t *nD)
{
    *nB = (int64_t)s->n * s->n; *nC = s->nC; *nD = s->nD;
}
double *oracle_state_B(ostate *s) { return s->B; }
double *oracle_state_C(ostate *s) { return s->C; }
double *oracle_state_D(ostate *s) { return s->D; }
void oracle_state_free_maps(const ostate *s, int32_t *I, int32_t *J)
{
    for (int x = 0; x < s->n; x++) { I[x] = s->I[x]; J[x] = s->J[x]; }
}

/* ------------------------------------------------------------------------- */
/* Minimal deterministic branch-and-bound (SURVEY.md §8(b) caller). */
/* ------------------------------------------------------------------------- */
/*
 * Depth-first; branch on the lowest-index free facility, children in ascending
 * location order (reading R20); cold children (reading R19): every node is
 * reduced and initialised from scratch, then bounded with T iterations (R18).
 * Nodes with n' <= 3 free facilities are leaves solved by enumerating completions
 * in lexicographic order.  Optional strong branching (sb_iters >= 0) at nodes with
 * n' >= 5: see oracle_strong_branch; children in ascending order of the line's other index.  A node is pruned when LB > UB - 1 + 1e-6 (optima are
 * integral, reading R15); the incumbent is replaced only on strict improvement
 * (reading R22).
 */
typedef struct {
    int N;
    const int64_t *F, *Dist;
    int T;
    int warm;            /* 1: children folded from the parent's post-bound state (NEXT-3)   */
    int sb_iters;        /* >= 0: strong branching with RLT1 (sb_iters iterations); < 0: off */
    int64_t sb_cut;      /* candidates cut by their RLT1 estimate                          */
    double K;
    int64_t best;        /* incumbent value; INT64_MAX = none             */
    int have_best;
    double UB;           /* pruning threshold (incumbent or caller UB0)   */
    int32_t best_perm[64];
    int64_t bounded, leaves, pruned;
    int err;
} bnb_ctx;

static int64_t full_cost(const bnb_ctx *c, const int32_t *perm)
{
    int64_t v = 0;
    for (int i = 0; i < c->N; i++)
        for (int k = 0; k < c->N; k++) v += c->F[i * c->N + k] * c->Dist[perm[i] * c->N + perm[k]];
    return v;
}

static void leaf_rec(bnb_ctx *c, int32_t *perm, const int32_t *ffac, int nf, int t,
                     char *lused, const int32_t *floc)
{
    if (t == nf) {
        int64_t v = full_cost(c, perm);
        if (!c->have_best || v < c->best) {
            c->best = v; c->have_best = 1;
            memcpy(c->best_perm, perm, sizeof(int32_t) * c->N);
            if ((double)v < c->UB) c->UB = (double)v;
        }
        return;
    }
    for (int x = 0; x < nf; x++) {
        if (lused[x]) continue;
        lused[x] = 1; perm[ffac[t]] = floc[x];
        leaf_rec(c, perm, ffac, nf, t + 1, lused, floc);
        lused[x] = 0;
    }
}

/* parent: the expanded parent's state (warm mode), the child fixing its reduced (pa, pb) */
static void bnb_visit(bnb_ctx *c, int nfix, int32_t *fac, int32_t *loc, const ostate *parent, int pa, int pb)
{
    if (c->err) return;
    int N = c->N;
    char uf[64] = {0}, ul[64] = {0};
    for (int t = 0; t < nfix; t++) { uf[fac[t]] = 1; ul[loc[t]] = 1; }
    int32_t ffac[64], floc[64];
    int nf = 0, nl = 0;
    for (int x = 0; x < N; x++) { if (!uf[x]) ffac[nf++] = x; if (!ul[x]) floc[nl++] = x; }
    if (nf <= 3) {
        c->leaves++;
        int32_t perm[64];
        for (int t = 0; t < nfix; t++) perm[fac[t]] = loc[t];
        char lused[64] = {0};
        leaf_rec(c, perm, ffac, nf, 0, lused, floc);
        return;
    }
    int err;
    ostate *s = (c->warm && parent) ? oracle_state_fold(parent, pa, pb, &err)
                                    : oracle_state_new(N, c->F, c->Dist, nfix, fac, loc, &err);
    if (!s) { c->err = err; return; }
    double LB; int iters, status;
    int st = oracle_bound(s, c->T, c->K, c->UB, &LB, NULL, &iters, &status, NULL);
    if (st) { oracle_state_free(s); c->err = st; return; }
    c->bounded++;
    if (LB > c->UB - 1.0 + 1e-6) { c->pruned++; oracle_state_free(s); return; }
    if (!c->warm) { oracle_state_free(s); s = NULL; }  /* cold children: built from (F, D, fixed) */
    const ostate *ps = s;  /* the children's parent state (warm mode) */
    if (c->sb_iters >= 0 && nf >= 5) {
        /* strong branching: branch on the row or column with the highest min-estimate;
           candidates whose RLT1 estimate already exceeds the incumbent are cut */
        double *est = malloc(sizeof(double) * nf * nf);
        int kind, index;
        int st2 = oracle_strong_branch(N, c->F, c->Dist, nfix, fac, loc, c->sb_iters, est, &kind, &index);
        if (st2) { free(est); oracle_state_free(s); c->err = st2; return; }
        for (int x = 0; x < nf; x++) {
            const int a = kind == 0 ? index : x, b = kind == 0 ? x : index;
            if (est[a * nf + b] > c->UB - 1.0 + 1e-6) { c->sb_cut++; continue; }
            fac[nfix] = ffac[a]; loc[nfix] = floc[b];
            bnb_visit(c, nfix + 1, fac, loc, ps, a, b);
        }
        free(est);
        oracle_state_free(s);
        return;
    }
    int f = ffac[0];
    for (int x = 0; x < nl; x++) {
        fac[nfix] = f; loc[nfix] = floc[x];
        bnb_visit(c, nfix + 1, fac, loc, ps, 0, x);  /* f = ffac[0] is reduced facility 0 */
    }
    oracle_state_free(s);
}

int oracle_bnb(int N, const int64_t *F, const int64_t *Dist, int T, double K, double UB0, int sb_iters,
               int warm, int64_t *best_out, int32_t *perm_out, int64_t *bounded_out, int64_t *leaves_out,
               int64_t *pruned_out, int64_t *sb_cut_out)
{
    if (N < 1 || N > 64) return ORC_E_ARG;
    bnb_ctx c;
    memset(&c, 0, sizeof c);
    c.N = N; c.F = F; c.Dist = Dist; c.T = T; c.K = K; c.UB = UB0; c.sb_iters = sb_iters; c.warm = warm;
    int32_t fac[64], loc[64];
    bnb_visit(&c, 0, fac, loc, NULL, 0, 0);
    if (c.err) return c.err;
    *best_out = c.have_best ? c.best : -1;
    if (c.have_best) memcpy(perm_out, c.best_perm, sizeof(int32_t) * N);
    *bounded_out = c.bounded; *leaves_out = c.leaves; *pruned_out = c.pruned;
    if (sb_cut_out) *sb_cut_out = c.sb_cut;
    return ORC_OK;
}
