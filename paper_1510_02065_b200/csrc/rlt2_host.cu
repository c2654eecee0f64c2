// rlt2_host.cu — host control of the RLT2 bound: the C ABI of include/qap_rlt2.h.
//
// The host only validates arguments, owns device memory and enqueues kernels in the
// order of Algorithm 1; every arithmetic step of the bound runs on the GPU.
// The stop test is evaluated on the device after each iteration and turns
// the remaining launches of the call into no-ops, so a bound call synchronises once.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <fcntl.h>
#include <unistd.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/qap_rlt2.h"
#include "rlt2_internal.h"
#include "rlt2_shard.h"

using namespace rlt2;

namespace {

enum Phase { PH_FRESH = -1 };

struct TimedLaunch {
    int kind;
    cudaEvent_t a, b;
};

}  // namespace

struct qap_rlt2 {
    int N = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    int flags = 0;
    int lap_warps = 0;
    int num_sms = 148;
    std::vector<int64_t> F, Dist;
    int64_t *dF = nullptr, *dDist = nullptr;
    double *dB = nullptr, *dC = nullptr, *dD = nullptr, *dSigma = nullptr, *dTrace = nullptr;
    int *dTriples = nullptr;
    Sched *dSched = nullptr;
    cudaEvent_t evJoin = nullptr;  // orders this handle's stream against another's (fold, copy)
    Ctl *dCtl = nullptr;
    int trace_cap = 4096;
    Node node{};
    Geom geom{};
    int next_phase = PH_FRESH;  // PH_FRESH: iteration 0 pending; else the next QAP_PHASE_*
    int d_zero = 1, b_zero = 0, c_zero = 0;
    std::string err;
    // kernel timing (QAP_FLAG_TIME_KERNELS)
    std::vector<TimedLaunch> pending;
    std::vector<cudaEvent_t> pool;
    int64_t launches[QAP_K_COUNT] = {0};
    double ms[QAP_K_COUNT] = {0};
    int call_launches = 0;
    // sharding of one bound over `world` ranks
    int world = 1, rank = 0;
    Transport *tp = nullptr;  // NCCL (one process per GPU); nullptr in an in-process group
    bool loopback = false;    // member of an in-process group: the group driver moves data
    ShardPlan plan;           // for the current n
    int *dTiles = nullptr, *dTinfo = nullptr;
    // the transfer of the local tiles runs on sSide while the shared tiles are exchanged, piece
    // by piece on sComm (evPack: piece packed, evX: piece received)
    cudaStream_t sSide = nullptr, sComm = nullptr;
    cudaEvent_t evFork = nullptr, evLocal = nullptr, evPack[kXChunks] = {}, evX[kXChunks] = {};
    size_t tiles_cap = 0, slots_cap = 0;
    int64_t dblk_cap = 0;     // stored blocks the D allocation can hold
    double *dSend = nullptr, *dRecv = nullptr, *dSall = nullptr;
    // strong-branching workspace (RLT1 children of a node), grown on demand
    double *dRc = nullptr, *dRb = nullptr, *dRlbd = nullptr;
    long long *dRkap = nullptr;
    size_t rc_cap = 0, rb_cap = 0, rk_cap = 0;
    std::vector<double> h_lbd;
    std::vector<long long> h_kap;
    // CUDA graphs of the iteration loop, keyed by (n, iterations, D still zero)
    cudaStream_t sCap = nullptr;
    std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;
    // B&B helper handles (children bounded concurrently), each on its own stream: created
    // on first use, kept (with their graphs) for later B&B calls, freed by qap_destroy
    std::vector<qap_rlt2 *> bnb_helpers;
    std::vector<cudaStream_t> bnb_streams;
    // warm B&B (NEXT-3): bnb_depth[d-1] holds the state of the expanded node at depth d of
    // the current DFS path (capacity N - d, on this handle's stream)
    std::vector<qap_rlt2 *> bnb_depth;
    int n_cap = 0;  // largest node (free facilities) the buffers hold
    // tensor maps of D for k_transfer_tma, encoded for node size tma_n (0: none / failed)
    TmaMaps tma{};
    int tma_n = 0;
};

// NVTX range around the host-side enqueue of a phase / call (SURVEY §5 tracing): visible in
// any NVTX-aware profiler, a no-op without one (header-only nvtx3, no link dependency)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static std::string g_create_error;

static qap_status fail(qap_rlt2 *h, qap_status st, const std::string &msg)
{
    if (h) h->err = msg; else g_create_error = msg;
    return st;
}

static qap_status cuda_fail(qap_rlt2 *h, cudaError_t e, const char *where)
{
    return fail(h, QAP_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static cudaEvent_t ev_get(qap_rlt2 *h)
{
    if (!h->pool.empty()) {
        cudaEvent_t e = h->pool.back();
        h->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Enqueue one kernel through `fn` on stream `st`, bracketed by events when timing is on.
template <class Fn>
static cudaError_t launch(qap_rlt2 *h, int kind, cudaStream_t st, Fn fn)
{
    cudaEvent_t a = nullptr, b = nullptr;
    const bool timed = (h->flags & QAP_FLAG_TIME_KERNELS) != 0;
    if (timed) {
        a = ev_get(h);
        b = ev_get(h);
        cudaEventRecord(a, st);
    }
    cudaError_t e = fn(st);
    if (timed) {
        cudaEventRecord(b, st);
        h->pending.push_back({kind, a, b});
    }
    h->call_launches++;
    return e;
}


static void harvest_timing(qap_rlt2 *h)
{
    for (auto &t : h->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
            h->ms[t.kind] += ms;
            h->launches[t.kind] += 1;
        }
        h->pool.push_back(t.a);
        h->pool.push_back(t.b);
    }
    h->pending.clear();
}

static void free_all(qap_rlt2 *h)
{
    cudaFree(h->dF);
    cudaFree(h->dDist);
    cudaFree(h->dB);
    cudaFree(h->dC);
    cudaFree(h->dD);
    cudaFree(h->dSigma);
    cudaFree(h->dTrace);
    cudaFree(h->dCtl);
    cudaFree(h->dTriples);
    cudaFree(h->dSched);
    if (h->evJoin) cudaEventDestroy(h->evJoin);
    cudaFree(h->dRc);
    cudaFree(h->dRb);
    cudaFree(h->dRlbd);
    cudaFree(h->dRkap);
    for (auto &kv : h->graphs) cudaGraphExecDestroy(kv.second);
    h->graphs.clear();
    if (h->sCap) cudaStreamDestroy(h->sCap);
    cudaFree(h->dTiles);
    cudaFree(h->dTinfo);
    if (h->evFork) cudaEventDestroy(h->evFork);
    if (h->evLocal) cudaEventDestroy(h->evLocal);
    for (int c = 0; c < kXChunks; c++) {
        if (h->evPack[c]) cudaEventDestroy(h->evPack[c]);
        if (h->evX[c]) cudaEventDestroy(h->evX[c]);
    }
    if (h->sSide) cudaStreamDestroy(h->sSide);
    if (h->sComm) cudaStreamDestroy(h->sComm);
    cudaFree(h->dSend);
    cudaFree(h->dRecv);
    cudaFree(h->dSall);
    delete h->tp;
    h->tp = nullptr;
    for (auto &t : h->pending) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    for (auto e : h->pool) cudaEventDestroy(e);
}

static qap_status check_instance(qap_rlt2 *h, int N, const int64_t *F, const int64_t *D)
{
    if (!F || !D) return fail(h, QAP_E_ARG, "F or D is NULL");
    int64_t maxf = 0, maxd = 0;
    for (int64_t t = 0; t < (int64_t)N * N; t++) {
        if (F[t] < 0 || D[t] < 0) return fail(h, QAP_E_ARG, "negative flow or distance entry");
        maxf = F[t] > maxf ? F[t] : maxf;
        maxd = D[t] > maxd ? D[t] : maxd;
    }
    // exactness of integer costs in fp64: N^2 maxF maxD < 2^53
    const long double bound = (long double)N * N * (long double)maxf * (long double)maxd;
    if (bound >= 9007199254740992.0L) return fail(h, QAP_E_ARG, "N^2*maxF*maxD >= 2^53");
    return QAP_OK;
}

extern "C" {

static qap_status create_impl(int32_t N, const int64_t *F, const int64_t *D, const qap_rlt2_opts *opts,
                              qap_rlt2 **out, bool loopback, int n_cap = 0);

qap_status qap_rlt2_create(int32_t N, const int64_t *F, const int64_t *D, const qap_rlt2_opts *opts,
                           qap_rlt2 **out)
{
    return create_impl(N, F, D, opts, out, false);
}

// n_cap (internal, single-GPU): buffers sized for nodes with at most n_cap free facilities
static qap_status create_impl(int32_t N, const int64_t *F, const int64_t *D, const qap_rlt2_opts *opts,
                              qap_rlt2 **out, bool loopback, int n_cap)
{
    if (!out) return fail(nullptr, QAP_E_ARG, "out is NULL");
    *out = nullptr;
    if (N < 3 || N > kMaxN) return fail(nullptr, QAP_E_ARG, "N must be in [3, 64]");
    {
        qap_status st0 = check_instance(nullptr, N, F, D);
        if (st0 != QAP_OK) return st0;
    }

    const int world = (opts && opts->world > 1) ? opts->world : 1;
    const int rank = world > 1 ? opts->rank : 0;
    if (world > 1) {
        if (rank < 0 || rank >= world || world > 64) return fail(nullptr, QAP_E_ARG, "bad rank / world");
        if (!loopback && !opts->nccl_id && !opts->host_transport)
            return fail(nullptr, QAP_E_ARG, "world > 1 needs opts->nccl_id or opts->host_transport");
        if (!loopback && opts->host_transport && (!opts->host_transport->exchange || !opts->host_transport->allgather))
            return fail(nullptr, QAP_E_ARG, "host_transport needs both callbacks");
    }
    if (opts && (opts->flags & ~(QAP_FLAG_TIME_KERNELS | QAP_FLAG_NO_GRAPH | QAP_FLAG_LDG_TRANSFER)))
        return fail(nullptr, QAP_E_ARG, "unknown flag bits");
    qap_rlt2 *h = new qap_rlt2();
    h->N = N;
    h->world = world;
    h->rank = rank;
    h->loopback = loopback;
    h->flags = opts ? opts->flags : 0;
    h->lap_warps = opts ? opts->lap_warps : 0;
    h->stream = opts ? static_cast<cudaStream_t>(opts->cuda_stream) : nullptr;
    cudaError_t e;
    if (opts && opts->device >= 0) {
        if ((e = cudaSetDevice(opts->device)) != cudaSuccess) {
            qap_status s = cuda_fail(nullptr, e, "cudaSetDevice");
            delete h;
            return s;
        }
    }
    cudaGetDevice(&h->device);
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
    h->F.assign(F, F + (size_t)N * N);
    h->Dist.assign(D, D + (size_t)N * N);
    h->n_cap = (n_cap >= 3 && n_cap < N && world == 1) ? n_cap : N;

    Geom gN;
    make_geom(h->n_cap, gN);
    size_t bytesD = (size_t)gN.nblk * gN.ld2 * 8;
    if (world > 1) {  // this rank's block slice, tile list and exchange slots: max over n <= N
        ShardPlan P;
        for (int n = 3; n <= N; n++) {
            make_plan(n, world, rank, P);
            Geom gn;
            make_geom(n, gn);
            const int64_t blk = P.blk_lo[rank + 1] - P.blk_lo[rank];
            const int64_t cap = (blk * gn.ld2 + gN.ld2 - 1) / gN.ld2;  // in N-sized blocks
            h->dblk_cap = h->dblk_cap > cap ? h->dblk_cap : cap;
            h->tiles_cap = h->tiles_cap > P.tiles.size() ? h->tiles_cap : P.tiles.size();
            h->slots_cap = h->slots_cap > (size_t)P.total_slots ? h->slots_cap : (size_t)P.total_slots;
        }
        bytesD = (size_t)(h->dblk_cap > 0 ? h->dblk_cap : 1) * gN.ld2 * 8;
    }
    const size_t bytesC = (size_t)gN.n * gN.n * gN.ldc * 8;
    const size_t bytesB = (((size_t)gN.n * gN.n + 1) & ~size_t(1)) * 8;
    const size_t bytesS = (size_t)gN.nblk * 8;
    size_t freeb = 0, totb = 0;
    if ((e = cudaMemGetInfo(&freeb, &totb)) != cudaSuccess) {
        qap_status s = cuda_fail(nullptr, e, "cudaMemGetInfo");
        delete h;
        return s;
    }
    const size_t need = bytesD + bytesC + bytesB + bytesS + (64u << 20);
    if (need > freeb) {
        delete h;
        char msg[160];
        snprintf(msg, sizeof msg, "needs %.3f GB of device memory, %.3f GB free", need / 1e9, freeb / 1e9);
        return fail(nullptr, QAP_E_CAPACITY, msg);
    }
#define ALLOC(ptr, bytes)                                                       \
    if ((e = cudaMalloc(reinterpret_cast<void **>(&ptr), (bytes))) != cudaSuccess) { \
        free_all(h);                                                            \
        delete h;                                                               \
        return e == cudaErrorMemoryAllocation ? fail(nullptr, QAP_E_CAPACITY, "cudaMalloc failed") \
                                              : cuda_fail(nullptr, e, "cudaMalloc");  \
    }
    ALLOC(h->dF, (size_t)N * N * 8);
    ALLOC(h->dDist, (size_t)N * N * 8);
    ALLOC(h->dB, bytesB);
    ALLOC(h->dC, bytesC);
    ALLOC(h->dD, bytesD);
    ALLOC(h->dSigma, bytesS);
    ALLOC(h->dTrace, (size_t)h->trace_cap * 8);
    ALLOC(h->dCtl, sizeof(Ctl));
    ALLOC(h->dTriples, (size_t)gN.n * (gN.n - 1) * (gN.n - 2) / 6 * 2 * sizeof(int) + 16);  // two orders (write_triples)
    ALLOC(h->dSched, sizeof(Sched));
    if (world > 1) {
        ALLOC(h->dTiles, h->tiles_cap * sizeof(int) + 16);
        ALLOC(h->dTinfo, h->tiles_cap * sizeof(int) + 16);
        ALLOC(h->dSend, h->slots_cap * kSlot * 8 + 16);
        ALLOC(h->dRecv, h->slots_cap * kSlot * 8 + 16);
        ALLOC(h->dSall, (size_t)gN.nblk * 8 + 16);
        for (int c = 0; c < kXChunks && e == cudaSuccess; c++)
            if ((e = cudaEventCreateWithFlags(&h->evPack[c], cudaEventDisableTiming)) == cudaSuccess)
                e = cudaEventCreateWithFlags(&h->evX[c], cudaEventDisableTiming);
        if (e != cudaSuccess || (e = cudaStreamCreateWithFlags(&h->sSide, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&h->sComm, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&h->evFork, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&h->evLocal, cudaEventDisableTiming)) != cudaSuccess) {
            free_all(h);
            delete h;
            return cuda_fail(nullptr, e, "side stream");
        }
        if (!loopback && opts->host_transport) {
            h->tp = make_host_transport(*opts->host_transport, world, rank);
        } else if (!loopback) {
            const char *why = "";
            h->tp = make_nccl_transport(opts->nccl_id, world, rank, h->device, &why);
            if (!h->tp) {
                std::string msg = std::string("NCCL transport: ") + why;
                free_all(h);
                delete h;
                return fail(nullptr, QAP_E_NCCL, msg);
            }
        }
    }
    {
        if ((e = cudaEventCreateWithFlags(&h->evJoin, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&h->sCap, cudaStreamNonBlocking)) != cudaSuccess) {
            free_all(h);
            delete h;
            return cuda_fail(nullptr, e, "streams");
        }
    }
    if ((e = cudaMemcpyAsync(h->dF, F, (size_t)N * N * 8, cudaMemcpyHostToDevice, h->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(h->dDist, D, (size_t)N * N * 8, cudaMemcpyHostToDevice, h->stream)) != cudaSuccess ||
        (e = cudaMemsetAsync(h->dCtl, 0, sizeof(Ctl), h->stream)) != cudaSuccess) {
        free_all(h);
        delete h;
        return cuda_fail(nullptr, e, "upload");
    }
    // the root node (a capacity-limited internal handle gets its nodes by qap_rlt2_fold)
    qap_status s = h->n_cap == N ? qap_rlt2_fix(h, 0, nullptr, nullptr) : QAP_OK;
    if (s != QAP_OK) {
        g_create_error = h->err;
        free_all(h);
        delete h;
        return s;
    }
    *out = h;
    return QAP_OK;
}

qap_status qap_rlt2_load(qap_rlt2 *h, const int64_t *F, const int64_t *D)
{
    if (!h) return QAP_E_ARG;
    const int N = h->N;
    qap_status st = check_instance(h, N, F, D);
    if (st != QAP_OK) return st;
    h->F.assign(F, F + (size_t)N * N);
    h->Dist.assign(D, D + (size_t)N * N);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(h->dF, F, (size_t)N * N * 8, cudaMemcpyHostToDevice, h->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(h->dDist, D, (size_t)N * N * 8, cudaMemcpyHostToDevice, h->stream)) != cudaSuccess)
        return cuda_fail(h, e, "upload");
    for (auto x : h->bnb_helpers)
        if ((st = qap_rlt2_load(x, F, D)) != QAP_OK) return fail(h, st, "bnb helper reload");
    for (auto x : h->bnb_depth)
        if ((st = qap_rlt2_load(x, F, D)) != QAP_OK) return fail(h, st, "bnb depth handle reload");
    if (h->n_cap < N) {  // internal capacity-limited handle: no root node; fold gives it nodes
        h->next_phase = PH_FRESH;
        return QAP_OK;
    }
    return qap_rlt2_fix(h, 0, nullptr, nullptr);
}

qap_status qap_rlt2_fix(qap_rlt2 *h, int32_t m, const int32_t *fac, const int32_t *loc)
{
    NvtxRange nv("qap_rlt2_fix");
    if (!h) return QAP_E_ARG;
    const int N = h->N;
    if (m < 0 || N - m < 3) return fail(h, QAP_E_ARG, "need 0 <= m <= N-3");
    if (N - m > h->n_cap) return fail(h, QAP_E_CAPACITY, "node larger than the handle's capacity");
    if (m > 0 && (!fac || !loc)) return fail(h, QAP_E_ARG, "fac/loc NULL");
    bool uf[kMaxN] = {false}, ul[kMaxN] = {false};
    for (int t = 0; t < m; t++) {
        if (fac[t] < 0 || fac[t] >= N || loc[t] < 0 || loc[t] >= N)
            return fail(h, QAP_E_ARG, "fixed index out of range");
        if (uf[fac[t]] || ul[loc[t]]) return fail(h, QAP_E_ARG, "duplicate facility or location in fixed set");
        uf[fac[t]] = ul[loc[t]] = true;
    }
    Node nd{};
    nd.N = N;
    nd.m = m;
    nd.n = N - m;
    int a = 0, b = 0;
    for (int x = 0; x < N; x++) {
        if (!uf[x]) nd.I[a++] = x;
        if (!ul[x]) nd.J[b++] = x;
    }
    for (int t = 0; t < m; t++) {
        nd.fac[t] = fac[t];
        nd.loc[t] = loc[t];
    }
    if (h->world > 1) {
        make_plan(nd.n, h->world, h->rank, h->plan);
        Geom gn;
        make_geom(nd.n, gn);
        Geom gN;
        make_geom(N, gN);
        const int64_t blk = h->plan.blk_lo[h->rank + 1] - h->plan.blk_lo[h->rank];
        if (blk * gn.ld2 > h->dblk_cap * gN.ld2 || h->plan.tiles.size() > h->tiles_cap ||
            (size_t)h->plan.total_slots > h->slots_cap)
            return fail(h, QAP_E_CAPACITY, "shard buffers too small for this node");
        cudaError_t e0;
        if (!h->plan.tiles.empty() &&
            ((e0 = cudaMemcpy(h->dTiles, h->plan.tiles.data(), h->plan.tiles.size() * sizeof(int),
                              cudaMemcpyHostToDevice)) != cudaSuccess ||
             (e0 = cudaMemcpy(h->dTinfo, h->plan.tinfo.data(), h->plan.tinfo.size() * sizeof(int),
                              cudaMemcpyHostToDevice)) != cudaSuccess))
            return cuda_fail(h, e0, "tile lists");
    }
    h->node = nd;
    make_geom(nd.n, h->geom);
    h->call_launches = 0;
    cudaError_t e = launch(h, QAP_K_INIT, h->stream, [&](cudaStream_t st) {
        return launch_init(h->node, h->geom, h->dF, h->dDist, h->dB, h->dC, h->dTriples, h->dCtl, st);
    });
    if (e != cudaSuccess) return cuda_fail(h, e, "k_init");
    h->next_phase = PH_FRESH;
    h->d_zero = 1;
    h->b_zero = 0;
    h->c_zero = 0;
    return QAP_OK;
}

qap_status qap_rlt2_fold(qap_rlt2 *child, const qap_rlt2 *parent, int32_t fac, int32_t loc)
{
    if (!child || !parent || child == parent) return child ? fail(child, QAP_E_ARG, "bad handles") : QAP_E_ARG;
    if (child->world > 1 || parent->world > 1 || child->loopback || parent->loopback)
        return fail(child, QAP_E_ARG, "fold needs single-GPU handles");
    if (child->device != parent->device) return fail(child, QAP_E_ARG, "fold across devices");
    if (child->N != parent->N || child->F != parent->F || child->Dist != parent->Dist)
        return fail(child, QAP_E_ARG, "fold needs handles of the same instance");
    if (parent->next_phase != PH_FRESH && parent->next_phase != QAP_PHASE_TRANSFER)
        return fail(child, QAP_E_STATE, "parent is in the middle of an iteration");
    const Node &pn = parent->node;
    const int n = pn.n;
    if (n - 1 < 3) return fail(child, QAP_E_ARG, "child would have fewer than 3 free facilities");
    int a = -1, b = -1;
    for (int x = 0; x < n; x++) {
        if (pn.I[x] == fac) a = x;
        if (pn.J[x] == loc) b = x;
    }
    if (a < 0 || b < 0) return fail(child, QAP_E_ARG, "facility or location not free in the parent");
    if (n - 1 > child->n_cap) return fail(child, QAP_E_CAPACITY, "child larger than the handle's capacity");
    Node nd = pn;
    nd.m = pn.m + 1;
    nd.n = n - 1;
    nd.fac[pn.m] = fac;
    nd.loc[pn.m] = loc;
    for (int x = 0; x < n - 1; x++) {
        nd.I[x] = pn.I[x + (x >= a)];
        nd.J[x] = pn.J[x + (x >= b)];
    }
    cudaError_t e = cudaSetDevice(child->device);
    if (e != cudaSuccess) return cuda_fail(child, e, "device");
    // order: parent's pending work -> fold (child stream) -> later parent work
    if ((e = cudaEventRecord(parent->evJoin, parent->stream)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(child->stream, parent->evJoin, 0)) != cudaSuccess)
        return cuda_fail(child, e, "fold ordering");
    child->node = nd;
    make_geom(nd.n, child->geom);
    child->call_launches = 0;
    FoldArgs f{};
    f.gp = parent->geom;
    f.gc = child->geom;
    f.a = a;
    f.b = b;
    f.pB = parent->dB;
    f.pC = parent->dC;
    f.pD = parent->dD;
    f.pctl = parent->dCtl;
    f.cB = child->dB;
    f.cC = child->dC;
    f.cD = child->dD;
    f.cctl = child->dCtl;
    f.triples = child->dTriples;
    f.d_zero = parent->d_zero;
    e = launch(child, QAP_K_INIT, child->stream, [&](cudaStream_t st) { return launch_fold(f, child->num_sms, st); });
    if (e != cudaSuccess) return cuda_fail(child, e, "k_fold");
    if ((e = cudaEventRecord(child->evJoin, child->stream)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(parent->stream, child->evJoin, 0)) != cudaSuccess)
        return cuda_fail(child, e, "fold ordering");
    child->next_phase = PH_FRESH;
    child->d_zero = parent->d_zero;
    child->b_zero = 0;
    child->c_zero = 0;
    return QAP_OK;
}

static TransferArgs transfer_args(qap_rlt2 *h)
{
    TransferArgs A{};
    A.g = h->geom;
    A.D = h->dD;
    A.sigma = h->dSigma;
    A.triples = h->dTriples;
    A.d_zero = h->d_zero;
    A.ctl = h->dCtl;
    A.sched = h->dSched;
    A.ntile = (h->geom.n + TT - 1) / TT;
    if (h->world > 1) {
        A.tiles = h->dTiles;
        A.tinfo = h->dTinfo;
        for (int f = 0; f < h->geom.n; f++) A.loc_off[f] = h->plan.loc_off[f];
        A.sendbuf = h->dSend;
        A.recvbuf = h->dRecv;
    }
    return A;
}

// Sharded iteration, one sub-phase (sub = 0 before the collective, 1 after it):
//   TRANSFER: 0 = sigma + pack the partials of shared tiles, 1 = apply (class means)
//   CONC_D:   0 = level-2 LAPs of the local blocks (S -> S_all slice), 1 = credit all S to C
static cudaError_t run_shard_sub(qap_rlt2 *h, int phase, int sub, cudaStream_t st)
{
    cudaError_t e = cudaSuccess;
    const Geom &g = h->geom;
    const ShardPlan &P = h->plan;
    // the plan lists the local tiles first, then the shared ones by exchange piece (make_plan)
    const int nloc = P.n_local;
    if (phase == QAP_PHASE_TRANSFER && sub == 0) {
        e = launch(h, QAP_K_SIGMA, st, [&](cudaStream_t s) {
            return launch_sigma(g, h->dB, h->dC, h->dSigma, h->dCtl, h->dSched, s);
        });
        if (e) return e;
        // pass 1: this side's partials of the shared tiles, piece by piece (evPack[c]: piece c
        // may go on the wire)
        for (int c = 0; c < kXChunks; c++) {
            TransferArgs A = transfer_args(h);
            A.pack = 1;
            A.tiles += nloc + P.piece_lo[c];
            A.tinfo += nloc + P.piece_lo[c];
            const int cnt = P.piece_lo[c + 1] - P.piece_lo[c];
            if (cnt > 0 &&
                (e = launch(h, QAP_K_TRANSFER, st, [&](cudaStream_t s) { return launch_transfer(A, cnt, s); })) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(h->evPack[c], st)) != cudaSuccess) return e;
        }
        if (nloc == 0) return e;
        // the local tiles need no exchange: transferred on the side stream while the shared
        // tiles' partials are exchanged (joined in sub-phase 1); disjoint classes
        if ((e = cudaEventRecord(h->evFork, st)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(h->sSide, h->evFork, 0)) != cudaSuccess)
            return e;
        TransferArgs L = transfer_args(h);
        e = launch(h, QAP_K_TRANSFER, h->sSide, [&](cudaStream_t s) { return launch_transfer(L, nloc, s); });
        if (e == cudaSuccess) e = cudaEventRecord(h->evLocal, h->sSide);
    } else if (phase == QAP_PHASE_TRANSFER && (sub == 1 || sub >= 16)) {
        // pass 2: the class means of the shared tiles — piece sub - 16 once it has arrived
        // (evX), or every piece (sub = 1: the caller moved all of them)
        const int c0 = sub == 1 ? 0 : sub - 16, c1 = sub == 1 ? kXChunks : c0 + 1;
        if (sub >= 16 && (e = cudaStreamWaitEvent(st, h->evX[c0], 0)) != cudaSuccess) return e;
        TransferArgs A = transfer_args(h);
        A.tiles += nloc + P.piece_lo[c0];
        A.tinfo += nloc + P.piece_lo[c0];
        const int cnt = P.piece_lo[c1] - P.piece_lo[c0];
        if (cnt > 0) e = launch(h, QAP_K_TRANSFER, st, [&](cudaStream_t s) { return launch_transfer(A, cnt, s); });
        if (e != cudaSuccess || (sub >= 16 && c1 < kXChunks)) return e;
        if (nloc > 0 && (e = cudaStreamWaitEvent(st, h->evLocal, 0)) != cudaSuccess) return e;
        h->d_zero = 0;
        h->b_zero = h->c_zero = 1;
    } else if (phase == QAP_PHASE_CONC_D && sub == 0) {
        const int64_t cnt = P.blk_lo[h->rank + 1] - P.blk_lo[h->rank];
        e = launch(h, QAP_K_LAP2, st, [&](cudaStream_t s) {
            return launch_lap_l2_local(g, h->dD, cnt, h->dSall + P.blk_lo[h->rank], h->dCtl, h->num_sms,
                                       h->lap_warps, h->dSched, s);  // S rank-major
        });
    } else if (phase == QAP_PHASE_CONC_D && sub == 1) {
        Offsets pos{};
        for (int f = 0; f < g.n; f++) pos.off[f] = P.pos_off[f];
        e = launch(h, QAP_K_LAP2, st, [&](cudaStream_t s) { return launch_credit(g, h->dSall, pos, h->dC, h->dCtl, s); });
        h->c_zero = 0;
    }
    return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda)
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder()
{
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// tensor maps of the current node's stored blocks (one per first facility f): the blocks of
// f as [j][k - f - 1][l'][entry], strides in bytes; false: use the per-element-load kernel
static bool tma_maps(qap_rlt2 *h)
{
    const Geom &g = h->geom;
    if (h->world > 1 || h->loopback) return false;
    if (h->tma_n == g.n) return true;
    if (h->tma_n == -g.n) return false;  // encoding failed for this size before
    auto enc = tma_encoder();
    const int n = g.n, n1 = n - 1;
    // every box extent within the tensor's: kBox1 <= n - 1, TT <= n (and kBox0 <= ld2)
    bool ok = enc != nullptr && n - 1 >= kBox1 && n >= TT && g.ld2 >= kBox0;
    for (int f = 0; ok && f + 1 < n; f++) {
        const cuuint64_t ld = (cuuint64_t)g.ld2;
        cuuint64_t dims[4] = {ld, (cuuint64_t)n1, (cuuint64_t)(n1 - f), (cuuint64_t)n};
        cuuint64_t strides[3] = {ld * 8, (cuuint64_t)n1 * ld * 8, (cuuint64_t)(n1 - f) * n1 * ld * 8};
        cuuint32_t box[4] = {(cuuint32_t)tma_box0(n), (cuuint32_t)kBox1, 1u, (cuuint32_t)TT};
        cuuint32_t es[4] = {1, 1, 1, 1};
        ok = enc(&h->tma.m[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, h->dD + g.off[f] * g.ld2, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    h->tma_n = ok ? n : -n;
    return ok;
}

// Enqueue one phase of Algorithm 1.  `st` is the stream the call's work is ordered on.
static const char *const kPhaseName[] = {"rlt2 iteration 0 (C->B->LB)", "rlt2 spread + transfer D",
                                         "rlt2 level-2 LAPs (D->C)", "rlt2 level-1 LAPs (C->B)",
                                         "rlt2 level-0 LAP (B->LB)"};

static cudaError_t run_phase(qap_rlt2 *h, int phase, cudaStream_t st, bool fused)
{
    NvtxRange nv(phase >= 0 && phase <= QAP_PHASE_CONC_B ? kPhaseName[phase] : "rlt2 phase");
    cudaError_t e = cudaSuccess;
    const Geom &g = h->geom;
    if (h->world > 1 && (phase == QAP_PHASE_TRANSFER || phase == QAP_PHASE_CONC_D)) {
        // NCCL mode: sub-phase, collective, sub-phase (an in-process group calls the
        // sub-phases itself, see qap_rlt2_group_bound)
        const int p0 = phase, p1 = fused ? QAP_PHASE_CONC_D : phase;
        for (int ph = p0; ph <= p1; ph++) {
            if ((e = run_shard_sub(h, ph, 0, st)) != cudaSuccess) return e;
            if (ph == QAP_PHASE_TRANSFER) {
                // piece c goes on the wire (sComm) once packed; its means are applied (st) once
                // it has arrived, while the next piece is exchanged
                for (int c = 0; c < kXChunks; c++) {
                    if ((e = cudaStreamWaitEvent(h->sComm, h->evPack[c], 0)) != cudaSuccess ||
                        (e = h->tp->exchange(h->plan, h->dSend, h->dRecv, c, h->sComm)) != cudaSuccess ||
                        (e = cudaEventRecord(h->evX[c], h->sComm)) != cudaSuccess ||
                        (e = run_shard_sub(h, ph, 16 + c, st)) != cudaSuccess)
                        return e;
                }
                continue;
            }
            if ((e = h->tp->allgather(h->plan, h->dSall, st)) != cudaSuccess) return e;
            if ((e = run_shard_sub(h, ph, 1, st)) != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    switch (phase) {
    case QAP_PHASE_ITER0:
        e = launch(h, QAP_K_LAP1, st, [&](cudaStream_t s) {
            return launch_lap_level(LAP_L1_ACC, g, h->dD, h->dC, h->dB, h->dCtl, h->dTrace, h->num_sms, 0, nullptr, s);
        });
        if (e) return e;
        e = launch(h, QAP_K_LAP0, st, [&](cudaStream_t s) {
            return launch_lap_level(LAP_L0_ITER0, g, h->dD, h->dC, h->dB, h->dCtl, h->dTrace, h->num_sms, 0, nullptr, s);
        });
        break;
    case QAP_PHASE_TRANSFER:
    case QAP_PHASE_CONC_D: {
        // bound() enqueues TRANSFER and CONC_D together (fused = true); qap_rlt2_step runs
        // them one at a time.
        if (phase == QAP_PHASE_TRANSFER) {
            e = launch(h, QAP_K_SIGMA, st, [&](cudaStream_t s) {
                return launch_sigma(g, h->dB, h->dC, h->dSigma, h->dCtl, h->dSched, s);
            });
            if (e) return e;
            TransferArgs A = transfer_args(h);
            const bool tma = !(h->flags & QAP_FLAG_LDG_TRANSFER) && tma_maps(h);
            e = launch(h, QAP_K_TRANSFER, st, [&](cudaStream_t s) {
                return tma ? launch_transfer_tma(A, h->tma, s) : launch_transfer(A, 0, s);
            });
            if (e) return e;
            h->d_zero = 0;
            h->b_zero = h->c_zero = 1;
            if (!fused) break;
        }
        e = launch(h, QAP_K_LAP2, st, [&](cudaStream_t s) {
            return launch_lap_level(LAP_L2, g, h->dD, h->dC, h->dB, h->dCtl, h->dTrace, h->num_sms, h->lap_warps,
                                    h->dSched, s);
        });
        if (e) return e;
        h->c_zero = 0;
        break;
    }
    case QAP_PHASE_CONC_C:
        // transfer between complementary costs of C: both members hold the same S after
        // CONC_D, so the pair mean is an exact no-op (reading R13); then concentrate C->B.
        e = launch(h, QAP_K_LAP1, st, [&](cudaStream_t s) {
            return launch_lap_level(LAP_L1_SET, g, h->dD, h->dC, h->dB, h->dCtl, h->dTrace, h->num_sms, 0, nullptr, s);
        });
        h->b_zero = 0;
        break;
    case QAP_PHASE_CONC_B:
        e = launch(h, QAP_K_LAP0, st, [&](cudaStream_t s) {
            return launch_lap_level(LAP_L0, g, h->dD, h->dC, h->dB, h->dCtl, h->dTrace, h->num_sms, 0, nullptr, s);
        });
        break;
    default: return cudaErrorInvalidValue;
    }
    return e;
}

static qap_status read_ctl(qap_rlt2 *h, Ctl &c)
{
    cudaError_t e = cudaMemcpyAsync(&c, h->dCtl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "sync");
    if (h->flags & QAP_FLAG_TIME_KERNELS) harvest_timing(h);
    if (c.err) return fail(h, QAP_E_NUMERIC, "LAP residual below -tau (certificate failure)");
    return QAP_OK;
}

qap_status qap_rlt2_step(qap_rlt2 *h, int32_t phase)
{
    if (!h) return QAP_E_ARG;
    if (h->world > 1) return fail(h, QAP_E_STATE, "qap_rlt2_step is single-rank only");
    const int expect = h->next_phase == PH_FRESH ? QAP_PHASE_ITER0 : h->next_phase;
    if (phase != expect) return fail(h, QAP_E_STATE, "phases must run in Algorithm-1 order");
    h->call_launches = 0;
    cudaError_t e = launch_ctl_begin(h->dCtl, 0.0, INFINITY, h->trace_cap, h->stream);
    if (e == cudaSuccess) e = run_phase(h, phase, h->stream, false);
    if (e != cudaSuccess) return cuda_fail(h, e, "step");
    h->next_phase = (phase == QAP_PHASE_CONC_B || phase == QAP_PHASE_ITER0) ? QAP_PHASE_TRANSFER : phase + 1;
    Ctl c;
    return read_ctl(h, c);
}

qap_status qap_rlt2_bound(qap_rlt2 *h, int32_t max_iters, double K, double UB, qap_rlt2_result *out)
{
    if (!h || !out) return h ? fail(h, QAP_E_ARG, "out is NULL") : QAP_E_ARG;
    qap_status s = qap_rlt2_bound_async(h, max_iters, K, UB);
    if (s != QAP_OK) return s;
    return qap_rlt2_bound_result(h, out);
}

qap_status qap_rlt2_bound_async(qap_rlt2 *h, int32_t max_iters, double K, double UB)
{
    NvtxRange nv("qap_rlt2_bound");
    if (!h) return QAP_E_ARG;
    if (max_iters < 0 || !(K >= 0.0) || std::isnan(UB)) return fail(h, QAP_E_ARG, "bad max_iters/K/UB");
    if (h->next_phase != PH_FRESH && h->next_phase != QAP_PHASE_TRANSFER)
        return fail(h, QAP_E_STATE, "bound called in the middle of an iteration");
    if (max_iters > h->trace_cap) return fail(h, QAP_E_ARG, "max_iters above the trace capacity (4096)");
    if (h->loopback) return fail(h, QAP_E_STATE, "in-process group member: use qap_rlt2_group_bound");
    if (h->geom.n < 3) return fail(h, QAP_E_STATE, "the handle holds no node");
    h->call_launches = 0;
    cudaError_t e = launch_ctl_begin(h->dCtl, K, UB, h->trace_cap, h->stream);
    h->call_launches++;
    if (e != cudaSuccess) return cuda_fail(h, e, "ctl");
    if (h->next_phase == PH_FRESH) {
        if ((e = run_phase(h, QAP_PHASE_ITER0, h->stream, true)) != cudaSuccess) return cuda_fail(h, e, "iteration 0");
        h->next_phase = QAP_PHASE_TRANSFER;
    }
    // The iteration loop is replayed from a CUDA graph (one launch instead of 5 per
    // iteration: the B&B's small nodes are launch-bound), except when per-kernel event
    // timing or sharding is on.
    const bool graphable = h->world == 1 && !(h->flags & (QAP_FLAG_TIME_KERNELS | QAP_FLAG_NO_GRAPH));
    if (graphable && max_iters > 0) {
        const auto key = std::make_tuple(h->geom.n, max_iters, h->d_zero);
        auto it = h->graphs.find(key);
        if (it == h->graphs.end()) {
            const int save_launches = h->call_launches, dz = h->d_zero;
            cudaGraph_t graph = nullptr;
            cudaGraphExec_t exec = nullptr;
            if ((e = cudaStreamBeginCapture(h->sCap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
                return cuda_fail(h, e, "graph capture");
            cudaError_t ec = cudaSuccess;
            for (int t = 0; t < max_iters && ec == cudaSuccess; t++)
                for (int ph = QAP_PHASE_TRANSFER; ph <= QAP_PHASE_CONC_B && ec == cudaSuccess; ph++)
                    if (ph != QAP_PHASE_CONC_D) ec = run_phase(h, ph, h->sCap, true);
            e = cudaStreamEndCapture(h->sCap, &graph);
            if (ec != cudaSuccess) return cuda_fail(h, ec, "graph capture (launch)");
            if (e != cudaSuccess) return cuda_fail(h, e, "graph capture (end)");
            e = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) return cuda_fail(h, e, "graph instantiate");
            it = h->graphs.emplace(key, exec).first;
            h->call_launches = save_launches;
            h->d_zero = dz;
        }
        if ((e = cudaGraphLaunch(it->second, h->stream)) != cudaSuccess) return cuda_fail(h, e, "graph launch");
        h->call_launches += 4 * max_iters;  // kernels in the graph: sigma, transfer, lap2, lap1, lap0
        h->call_launches += max_iters;
        h->d_zero = 0;
        h->b_zero = h->c_zero = 0;
    } else {
        for (int t = 0; t < max_iters; t++) {
            for (int ph = QAP_PHASE_TRANSFER; ph <= QAP_PHASE_CONC_B; ph++) {
                if (ph == QAP_PHASE_CONC_D) continue;  // enqueued together with TRANSFER
                if ((e = run_phase(h, ph, h->stream, true)) != cudaSuccess) return cuda_fail(h, e, "iteration");
            }
        }
    }
    return QAP_OK;
}

qap_status qap_rlt2_bound_result(qap_rlt2 *h, qap_rlt2_result *out)
{
    if (!h || !out) return h ? fail(h, QAP_E_ARG, "out is NULL") : QAP_E_ARG;
    cudaError_t e;
    Ctl c;
    qap_status s = read_ctl(h, c);
    if (s != QAP_OK) return s;
    out->lb = c.lb;
    out->lb_glb = c.lb_glb;
    out->iters = c.iters;
    out->status = c.status;
    out->launches = h->call_launches;
    if (out->lb_trace && out->lb_trace_cap > 0 && c.iters > 0) {
        const int cnt = c.iters < out->lb_trace_cap ? c.iters : out->lb_trace_cap;
        e = cudaMemcpy(out->lb_trace, h->dTrace, (size_t)cnt * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(h, e, "trace copy");
    }
    return QAP_OK;
}

static cudaError_t grow(void **p, size_t &cap, size_t bytes)
{
    if (bytes <= cap) return cudaSuccess;
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
}

qap_status qap_rlt2_strong_branch(qap_rlt2 *h, int32_t sb_iters, double *est, int32_t *kind, int32_t *index)
{
    if (!h || !est || !kind || !index || sb_iters < 0) return QAP_E_ARG;
    const int n = h->node.n;
    if (n < 4) return fail(h, QAP_E_ARG, "strong branching needs n >= 4 free facilities");
    Rlt1Batch R{};
    R.K = n * n;
    make_geom(n - 1, R.g);
    R.bstr = ((int64_t)(n - 1) * (n - 1) + 1) & ~int64_t(1);
    cudaError_t e;
    if ((e = grow(reinterpret_cast<void **>(&h->dRc), h->rc_cap, (size_t)R.K * (n - 1) * (n - 1) * R.g.ldc * 8)) ||
        (e = grow(reinterpret_cast<void **>(&h->dRb), h->rb_cap, (size_t)R.K * R.bstr * 8 + 16)) ||
        (e = grow(reinterpret_cast<void **>(&h->dRlbd), h->rk_cap, (size_t)R.K * 8)))
        return e == cudaErrorMemoryAllocation ? fail(h, QAP_E_CAPACITY, "strong-branching workspace")
                                              : cuda_fail(h, e, "strong-branching workspace");
    if (!h->dRkap || h->h_kap.size() < (size_t)R.K) {
        cudaFree(h->dRkap);
        h->dRkap = nullptr;
        if ((e = cudaMalloc(reinterpret_cast<void **>(&h->dRkap), (size_t)R.K * 8)) != cudaSuccess)
            return cuda_fail(h, e, "strong-branching workspace");
        h->h_kap.resize(R.K);
    }
    h->h_lbd.resize(R.K);
    R.C = h->dRc;
    R.B = h->dRb;
    R.lbd = h->dRlbd;
    R.kap = h->dRkap;
    cudaStream_t st = h->stream;
    // RLT1: iteration 0, then sb_iters x (spread + C pair mean,
    // concentrate C->B, concentrate B->LB) for every candidate child at once
    if ((e = launch_rlt1_init(h->node, R, h->dF, h->dDist, st)) ||
        (e = launch_rlt1_lap(R, 1, 1, h->num_sms, st)) || (e = launch_rlt1_lap(R, 0, 0, h->num_sms, st)))
        return cuda_fail(h, e, "rlt1");
    for (int t = 0; t < sb_iters; t++)
        if ((e = launch_rlt1_pair(R, st)) || (e = launch_rlt1_lap(R, 1, 0, h->num_sms, st)) ||
            (e = launch_rlt1_lap(R, 0, 0, h->num_sms, st)))
            return cuda_fail(h, e, "rlt1");
    if ((e = cudaMemcpyAsync(h->h_lbd.data(), R.lbd, (size_t)R.K * 8, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(h->h_kap.data(), R.kap, (size_t)R.K * 8, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaStreamSynchronize(st)))
        return cuda_fail(h, e, "rlt1 result");
    for (int c = 0; c < R.K; c++) est[c] = (double)h->h_kap[c] + h->h_lbd[c];
    // max-min line selection (ties: lowest index, a row before a column)
    double best = -INFINITY;
    *kind = 0;
    *index = 0;
    for (int a2 = 0; a2 < n; a2++) {
        double sc = INFINITY;
        for (int b = 0; b < n; b++) sc = est[a2 * n + b] < sc ? est[a2 * n + b] : sc;
        if (sc > best) {
            best = sc;
            *kind = 0;
            *index = a2;
        }
    }
    for (int b = 0; b < n; b++) {
        double sc = INFINITY;
        for (int a2 = 0; a2 < n; a2++) sc = est[a2 * n + b] < sc ? est[a2 * n + b] : sc;
        if (sc > best) {
            best = sc;
            *kind = 1;
            *index = b;
        }
    }
    return QAP_OK;
}

qap_status qap_rlt2_dual_sizes(const qap_rlt2 *h, int64_t *nB, int64_t *nC, int64_t *nD)
{
    if (!h) return QAP_E_ARG;
    const int64_t n = h->geom.n;
    if (nB) *nB = n * n;
    if (nC) *nC = n * n * (n - 1) * (n - 1);
    if (nD) *nD = h->geom.nblk * (n - 2) * (n - 2);
    return QAP_OK;
}

qap_status qap_rlt2_dual_copy(const qap_rlt2 *hc, double *B, double *C, double *D, double *lb)
{
    qap_rlt2 *h = const_cast<qap_rlt2 *>(hc);
    if (!h) return QAP_E_ARG;
    const Geom &g = h->geom;
    const int64_t n = g.n;
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "sync");
    if (B) {
        if (h->b_zero) memset(B, 0, (size_t)n * n * 8);
        else if ((e = cudaMemcpy(B, h->dB, (size_t)n * n * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_fail(h, e, "copy B");
    }
    if (C) {
        const size_t w = (size_t)(n - 1) * (n - 1) * 8;
        if (h->c_zero) memset(C, 0, w * n * n);
        else if ((e = cudaMemcpy2D(C, w, h->dC, g.ldc * 8, w, n * n, cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_fail(h, e, "copy C");
    }
    if (D) {
        const size_t w = (size_t)(n - 2) * (n - 2) * 8;
        // sharded: only this rank's blocks (at their global positions); the rest is untouched
        for (int f = 0; f < (h->world > 1 ? n : 1); f++) {
            if (h->world > 1 && h->plan.owner[f] != h->rank) continue;
            const int64_t b0 = h->world > 1 ? g.off[f] : 0;
            const int64_t nb = h->world > 1 ? (f + 1 < n ? g.off[f + 1] : g.nblk) - g.off[f] : g.nblk;
            const int64_t l0 = h->world > 1 ? b0 + h->plan.loc_off[f] : 0;
            if (nb <= 0) continue;
            double *Dout = D + (size_t)b0 * (n - 2) * (n - 2);
            if (h->d_zero) memset(Dout, 0, w * nb);
            else if ((e = cudaMemcpy2D(Dout, w, h->dD + (size_t)l0 * g.ld2, g.ld2 * 8, w, nb,
                                       cudaMemcpyDeviceToHost)) != cudaSuccess)
                return cuda_fail(h, e, "copy D");
        }
    }
    if (lb) {
        Ctl c;
        if ((e = cudaMemcpy(&c, h->dCtl, sizeof(Ctl), cudaMemcpyDeviceToHost)) != cudaSuccess)
            return cuda_fail(h, e, "copy ctl");
        *lb = c.lb;
    }
    return QAP_OK;
}

qap_status qap_rlt2_kernel_stats(qap_rlt2 *h, int64_t *launches, double *ms, int32_t reset)
{
    if (!h) return QAP_E_ARG;
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "sync");
    harvest_timing(h);
    for (int k = 0; k < QAP_K_COUNT; k++) {
        if (launches) launches[k] = h->launches[k];
        if (ms) ms[k] = h->ms[k];
        if (reset) {
            h->launches[k] = 0;
            h->ms[k] = 0;
        }
    }
    return QAP_OK;
}

const char *qap_last_error(const qap_rlt2 *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

void qap_destroy(qap_rlt2 *h)
{
    if (!h) return;
    for (auto x : h->bnb_helpers) qap_destroy(x);
    for (auto s : h->bnb_streams) cudaStreamDestroy(s);
    for (auto x : h->bnb_depth) qap_destroy(x);
    cudaStreamSynchronize(h->stream);
    free_all(h);
    delete h;
}

qap_status qap_lap_batch(int32_t m, int64_t count, int64_t ld, const double *M_dev, double *R_dev, double *S_dev,
                         int32_t *assign_dev, double *u_dev, double *v_dev, int64_t *steps_dev, int32_t *err_dev,
                         void *stream)
{
    if (m < 1 || m > 64 || count < 0 || ld < (int64_t)m * m || (ld & 1) || !M_dev || !R_dev) return QAP_E_ARG;
    if ((reinterpret_cast<uintptr_t>(M_dev) | reinterpret_cast<uintptr_t>(R_dev)) & 15) return QAP_E_ARG;
    if (count == 0) return QAP_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    LapBatchOut o{R_dev, S_dev, u_dev, v_dev, assign_dev, steps_dev, err_dev};
    cudaError_t e = launch_lap_batch(m, count, ld, M_dev, o, sms, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
        g_create_error = std::string("qap_lap_batch: ") + cudaGetErrorString(e);
        return QAP_E_CUDA;
    }
    return QAP_OK;
}

}  // extern "C"

// ---- minimal deterministic B&B (P:236-238 caller) ----------------------
// Depth-first over an explicit stack of frames.  A frame is an expanded node: its children
// (branching line), their RLT1 estimates (strong branching) and RLT2 bounds, and the next
// child to visit.  Children of a node are bounded together, `batch` at a time, each on its
// own handle and stream; they are then visited in order and pruned against the CURRENT
// incumbent.  With K = 0 this makes exactly the decisions of the one-node-at-a-time DFS
// (a bound stops early only when LB already exceeds UB - 1 + 1e-6, and LB is
// nondecreasing), so node counts, optimum and permutation equal the oracle's B&B.
// The stack + incumbent + counters are the checkpoint ("checkpoints procedure").
namespace {
struct Frame {
    std::vector<int32_t> fac, loc;  // the expanded node
    std::vector<int32_t> fs, ls;    // its children: fac + fs[c] -> loc + ls[c]
    std::vector<double> est, lb;    // RLT1 estimate (-inf without strong branching), RLT2 bound
    uint32_t next = 0;
    uint8_t child_leaf = 0;
    uint64_t id = 0;  // warm: identifies the frame whose children the pool handles hold
};

struct Bnb {
    std::vector<qap_rlt2 *> pool;  // handles that bound children: cold: the caller's + helpers; warm: helpers
    // warm children (NEXT-3 (i), reading R31): depth[d] holds the dual state of the expanded
    // node with base_m + d fixed pairs on the current DFS path (depth[0] = the caller's handle)
    bool warm = false;
    int base_m = 0;
    std::vector<int32_t> root_fac, root_loc;  // the subtree root's fixed pairs (base_m of them)
    std::vector<qap_rlt2 *> depth;
    // warm: pool handle j holds the post-bound state of child holds[j].second of the frame
    // with id holds[j].first (until the handle is reused): expanding that child copies it
    uint64_t next_id = 1;
    std::vector<std::pair<uint64_t, int>> holds;
    int64_t copies = 0, rederived = 0;
    int N = 0, iters = 0, sb_iters = -1;
    double K = 0.0, UB = INFINITY, UB0 = INFINITY;
    bool have = false;
    int64_t best = -1;
    std::vector<int32_t> best_perm;
    int64_t bounded = 0, leaves = 0, pruned = 0, sb_cut = 0;
    std::vector<int64_t> bdepth = std::vector<int64_t>(65, 0);  // bounded nodes by fixed pairs
    void counted(size_t d)
    {
        bounded++;
        if (d < bdepth.size()) bdepth[d]++;
    }
    std::vector<Frame> stack;
    bool root_done = false;
    qap_status st = QAP_OK;
    // subtree-parallel hooks (include/qap_rlt2.h, NEXT-2)
    qap_bnb_sync_fn sync_fn = nullptr;
    qap_bnb_donate_fn donate_fn = nullptr;
    void *ctx = nullptr;
    int64_t sync_every = 32, since_sync = 0;
    bool improved = false;
    const qap_rlt2 *h0() const { return depth[0]; }  // the caller's handle
    bool cut(double lb) const { return lb > UB - 1.0 + 1e-6; }  // prune rule (R15)

    int64_t cost(const std::vector<int32_t> &perm) const
    {
        int64_t v = 0;
        for (int i = 0; i < N; i++)
            for (int k = 0; k < N; k++) v += h0()->F[i * N + k] * h0()->Dist[perm[i] * N + perm[k]];
        return v;
    }
    void leaf_rec(std::vector<int32_t> &perm, const std::vector<int> &ffac, const std::vector<int> &floc, int t,
                  std::vector<char> &used)
    {
        if (t == (int)ffac.size()) {
            const int64_t v = cost(perm);
            if (!have || v < best) {
                best = v;
                have = true;
                best_perm = perm;
                improved = true;
                if ((double)v < UB) UB = (double)v;
            }
            return;
        }
        for (size_t x = 0; x < floc.size(); x++) {
            if (used[x]) continue;
            used[x] = 1;
            perm[ffac[t]] = floc[x];
            leaf_rec(perm, ffac, floc, t + 1, used);
            used[x] = 0;
        }
    }
    void free_sets(const std::vector<int32_t> &fac, const std::vector<int32_t> &loc, std::vector<int> &ffac,
                   std::vector<int> &floc) const
    {
        std::vector<char> uf(N, 0), ul(N, 0);
        for (size_t t = 0; t < fac.size(); t++) uf[fac[t]] = ul[loc[t]] = 1;
        for (int x = 0; x < N; x++) {
            if (!uf[x]) ffac.push_back(x);
            if (!ul[x]) floc.push_back(x);
        }
    }
    void leaf(const std::vector<int32_t> &fac, const std::vector<int32_t> &loc)
    {
        std::vector<int> ffac, floc;
        free_sets(fac, loc, ffac, floc);
        leaves++;
        std::vector<int32_t> perm(N, 0);
        for (size_t t = 0; t < fac.size(); t++) perm[fac[t]] = loc[t];
        std::vector<char> used(floc.size(), 0);
        leaf_rec(perm, ffac, floc, 0, used);
    }
    // bound the wanted children of F, `pool.size()` at a time concurrently
    bool bound_children(Frame &F, const std::vector<char> &want)
    {
        F.lb.assign(F.fs.size(), INFINITY);
        std::vector<size_t> idx;
        for (size_t c = 0; c < F.fs.size(); c++)
            if (want[c]) idx.push_back(c);
        const size_t B = pool.size();
        std::vector<int32_t> fac = F.fac, loc = F.loc;
        for (size_t c0 = 0; c0 < idx.size(); c0 += B) {
            const size_t c1 = c0 + B < idx.size() ? c0 + B : idx.size();
            for (size_t k = c0; k < c1; k++) {
                qap_rlt2 *h = pool[k - c0];
                if (warm) {
                    st = qap_rlt2_fold(h, depth[F.fac.size() - base_m], F.fs[idx[k]], F.ls[idx[k]]);
                } else {
                    fac.push_back(F.fs[idx[k]]);
                    loc.push_back(F.ls[idx[k]]);
                    st = qap_rlt2_fix(h, (int)fac.size(), fac.data(), loc.data());
                    fac.pop_back();
                    loc.pop_back();
                }
                if (st != QAP_OK) return false;
                if ((st = qap_rlt2_bound_async(h, iters, K, UB)) != QAP_OK) return false;
                if (warm) holds[k - c0] = {F.id, (int)idx[k]};
            }
            for (size_t k = c0; k < c1; k++) {
                qap_rlt2_result r{};
                if ((st = qap_rlt2_bound_result(pool[k - c0], &r)) != QAP_OK) return false;
                F.lb[idx[k]] = r.lb;
            }
        }
        return true;
    }
    // node (fac, loc) is bounded and not pruned: its frame (branching line + child bounds)
    bool make_frame(const std::vector<int32_t> &fac, const std::vector<int32_t> &loc, Frame &F)
    {
        F.fac = fac;
        F.loc = loc;
        std::vector<int> ffac, floc;
        free_sets(fac, loc, ffac, floc);
        const int n = (int)ffac.size();
        F.id = next_id++;
        if (sb_iters >= 0 && n >= 5) {  // strong branching
            if (warm) holds[0] = {0, -1};
            if ((st = qap_rlt2_fix(pool[0], (int)fac.size(), fac.data(), loc.data())) != QAP_OK) return false;
            std::vector<double> e((size_t)n * n);
            int32_t kind = 0, index = 0;
            if ((st = qap_rlt2_strong_branch(pool[0], sb_iters, e.data(), &kind, &index)) != QAP_OK) return false;
            for (int x = 0; x < n; x++) {
                const int a = kind == 0 ? index : x, b = kind == 0 ? x : index;
                F.fs.push_back(ffac[a]);
                F.ls.push_back(floc[b]);
                F.est.push_back(e[(size_t)a * n + b]);
            }
        } else {  // lowest free facility, locations ascending (R20)
            for (int x = 0; x < n; x++) {
                F.fs.push_back(ffac[0]);
                F.ls.push_back(floc[x]);
                F.est.push_back(-INFINITY);
            }
        }
        F.child_leaf = n - 1 <= 3;
        if (F.child_leaf) {
            F.lb.assign(F.fs.size(), -INFINITY);
            return true;
        }
        std::vector<char> want(F.fs.size());
        for (size_t c = 0; c < F.fs.size(); c++) want[c] = !(F.est[c] > UB - 1.0 + 1e-6);
        return bound_children(F, want);
    }
    void start()
    {
        std::vector<int32_t> fac, loc;
        root_done = true;
        if (N <= 3) {
            leaf(fac, loc);
            return;
        }
        if ((st = qap_rlt2_fix(depth[0], 0, nullptr, nullptr)) != QAP_OK) return;
        qap_rlt2_result r{};
        if ((st = qap_rlt2_bound(depth[0], iters, K, UB, &r)) != QAP_OK) return;
        counted(0);
        if (r.lb > UB - 1.0 + 1e-6) {
            pruned++;
            return;
        }
        Frame F;
        if (!make_frame(fac, loc, F)) return;
        stack.push_back(std::move(F));
    }
    // search only the subtree of `root` (its bound reused when given)
    void start_at(const qap_bnb_node *root)
    {
        if (!root) {
            start();
            return;
        }
        root_done = true;
        std::vector<int32_t> fac(root->fac, root->fac + root->m), loc(root->loc, root->loc + root->m);
        if (N - root->m <= 3) {
            leaf(fac, loc);
            return;
        }
        double lb = root->lb;
        if (std::isnan(lb)) {
            if ((st = qap_rlt2_fix(depth[0], root->m, fac.data(), loc.data())) != QAP_OK) return;
            qap_rlt2_result r{};
            if ((st = qap_rlt2_bound(depth[0], iters, K, UB, &r)) != QAP_OK) return;
            counted(root->m);
            lb = r.lb;
        }
        if (cut(lb)) {
            pruned++;
            return;
        }
        // warm: the given root's own state (its bound came from elsewhere): a cold bound here
        if (warm && !std::isnan(root->lb) && !derive(0, fac, loc)) return;
        Frame F;
        if (!make_frame(fac, loc, F)) return;
        stack.push_back(std::move(F));
    }
    // give away the unvisited children of the shallowest expanded nodes (largest subtrees)
    // until at least k went out; they count as bounded (and pruned / cut) here
    void donate(int64_t k)
    {
        int64_t given = 0;
        for (size_t d = 0; d < stack.size() && given < k; d++) {
            Frame &F = stack[d];
            if (F.child_leaf || F.next >= F.fs.size()) continue;  // leaves are cheap: keep them
            for (uint32_t c = F.next; c < F.fs.size(); c++) {
                if (cut(F.est[c])) {
                    sb_cut++;
                    continue;
                }
                counted(F.fac.size() + 1);
                if (cut(F.lb[c])) {
                    pruned++;
                    continue;
                }
                qap_bnb_node nd{};
                nd.m = (int32_t)F.fac.size() + 1;
                for (size_t t = 0; t < F.fac.size(); t++) {
                    nd.fac[t] = F.fac[t];
                    nd.loc[t] = F.loc[t];
                }
                nd.fac[nd.m - 1] = F.fs[c];
                nd.loc[nd.m - 1] = F.ls[c];
                nd.lb = F.lb[c];
                donate_fn(ctx, &nd);
                given++;
            }
            F.next = (uint32_t)F.fs.size();
        }
    }
    // exchange the incumbent with the scheduler; false: abort requested
    bool sync()
    {
        since_sync = 0;
        improved = false;
        int64_t g = -1;
        const int32_t k = sync_fn(ctx, have ? best : -1, have ? best_perm.data() : nullptr, &g);
        if (k < 0) {
            st = QAP_E_STATE;
            return false;
        }
        if (g >= 0 && (double)g < UB) UB = (double)g;
        if (k > 0 && donate_fn) donate(k);
        return true;
    }
    // advance by one child; false when the search is over
    bool step()
    {
        while (!stack.empty() && stack.back().next >= stack.back().fs.size()) stack.pop_back();
        if (stack.empty()) return false;
        Frame &T = stack.back();
        const uint32_t c = T.next++;
        if (T.est[c] > UB - 1.0 + 1e-6) {  // cut by its RLT1 estimate (strong branching)
            sb_cut++;
            return true;
        }
        std::vector<int32_t> fac = T.fac, loc = T.loc;
        fac.push_back(T.fs[c]);
        loc.push_back(T.ls[c]);
        if (T.child_leaf) {
            leaf(fac, loc);
            return true;
        }
        counted(fac.size());
        if (T.lb[c] > UB - 1.0 + 1e-6) {
            pruned++;
            return true;
        }
        if (warm) {
            const size_t d = fac.size() - base_m;
            int j = -1;
            for (size_t q = 0; q < holds.size(); q++)
                if (holds[q].first == T.id && holds[q].second == (int)c) j = (int)q;
            if (j >= 0) {
                if ((st = depth_handle(d)) != QAP_OK) return false;
                if ((st = copy_state(depth[d], pool[j])) != QAP_OK) return false;
                copies++;
            } else {
                if (!derive(d, fac, loc)) return false;
                rederived++;
            }
        }
        Frame F;
        if (!make_frame(fac, loc, F)) return false;
        stack.push_back(std::move(F));
        return true;
    }
    // warm: (re)build depth[d]'s state for node (fac, loc): fold from depth[d-1] (which holds
    // its parent) and run the node's bound again.  With K = 0 the node was bounded with all
    // `iters` iterations when it was not pruned, so UB = +inf reproduces that state exactly.
    // d = 0: the search root, cold (fix + bound).
    bool derive(size_t d, const std::vector<int32_t> &fac, const std::vector<int32_t> &loc)
    {
        qap_rlt2_result r{};
        if (d == 0) {
            if ((st = qap_rlt2_fix(depth[0], (int)fac.size(), fac.data(), loc.data())) != QAP_OK) return false;
        } else {
            if ((st = depth_handle(d)) != QAP_OK) return false;
            if ((st = qap_rlt2_fold(depth[d], depth[d - 1], fac.back(), loc.back())) != QAP_OK) return false;
        }
        return (st = qap_rlt2_bound(depth[d], iters, K, INFINITY, &r)) == QAP_OK;
    }
    qap_status depth_handle(size_t d);
    static qap_status copy_state(qap_rlt2 *dst, const qap_rlt2 *src);
    ~Bnb()
    {
        for (auto x : pool) cudaStreamSynchronize(x->stream);  // helpers: owned by the caller's handle
    }
};

// depth handle d >= 1 of the warm search: owned by the caller's handle (kept across calls),
// capacity N - d free facilities, on the caller's stream
qap_status Bnb::depth_handle(size_t d)
{
    qap_rlt2 *own = depth[0];
    while (depth.size() <= d) {
        const size_t k = depth.size();
        while (own->bnb_depth.size() < k) {
            const size_t kk = own->bnb_depth.size() + 1;
            qap_rlt2_opts op{};
            op.device = own->device;
            op.cuda_stream = own->stream;
            op.flags = own->flags & ~QAP_FLAG_TIME_KERNELS;
            op.lap_warps = own->lap_warps;
            qap_rlt2 *x = nullptr;
            const int cap = own->N - (int)kk;
            if (cap < 3) return fail(own, QAP_E_ARG, "warm depth beyond the last bounded level");
            qap_status s0 = create_impl(own->N, own->F.data(), own->Dist.data(), &op, &x, false, cap);
            if (s0 != QAP_OK) return fail(own, s0, std::string("bnb depth handle: ") + qap_last_error(nullptr));
            own->bnb_depth.push_back(x);
        }
        depth.push_back(own->bnb_depth[k - 1]);
    }
    return QAP_OK;
}

// dst := src's node and dual state (same instance, single GPU, src at an iteration
// boundary), ordered after src's pending work; device-to-device copies on dst's stream
qap_status Bnb::copy_state(qap_rlt2 *dst, const qap_rlt2 *src)
{
    const Geom &g = src->geom;
    if (g.n > dst->n_cap) return fail(dst, QAP_E_CAPACITY, "state copy: node larger than the target");
    cudaError_t e;
    if ((e = cudaEventRecord(src->evJoin, src->stream)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(dst->stream, src->evJoin, 0)) != cudaSuccess)
        return cuda_fail(dst, e, "state copy ordering");
    const size_t nb = (size_t)g.n * g.n * 8, nc = (size_t)g.n * g.n * g.ldc * 8, nd = (size_t)g.nblk * g.ld2 * 8;
    if ((e = cudaMemcpyAsync(dst->dB, src->dB, nb, cudaMemcpyDeviceToDevice, dst->stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(dst->dC, src->dC, nc, cudaMemcpyDeviceToDevice, dst->stream)) != cudaSuccess ||
        (!src->d_zero &&
         (e = cudaMemcpyAsync(dst->dD, src->dD, nd, cudaMemcpyDeviceToDevice, dst->stream)) != cudaSuccess) ||
        (e = cudaMemcpyAsync(dst->dCtl, src->dCtl, sizeof(Ctl), cudaMemcpyDeviceToDevice, dst->stream)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(dst->dTriples, src->dTriples, (size_t)g.n * (g.n - 1) * (g.n - 2) / 6 * 2 * sizeof(int),
                             cudaMemcpyDeviceToDevice, dst->stream)) != cudaSuccess)
        return cuda_fail(dst, e, "state copy");
    if ((e = cudaEventRecord(dst->evJoin, dst->stream)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(src->stream, dst->evJoin, 0)) != cudaSuccess)
        return cuda_fail(dst, e, "state copy ordering");
    dst->node = src->node;
    dst->geom = src->geom;
    dst->next_phase = src->next_phase;
    dst->d_zero = src->d_zero;
    dst->b_zero = src->b_zero;
    dst->c_zero = src->c_zero;
    return QAP_OK;
}

// ---- checkpoint file (binary, little-endian; written to <path>.tmp, fsync'ed, renamed) ----
constexpr uint64_t kCkptMagic = 0x3254504b32544c52ull;  // "RLT2KPT2"
constexpr uint32_t kCkptVersion = 3;  // 3: + format version, subtree root (base_m, its pairs)

uint64_t instance_digest(const qap_rlt2 *h)
{
    uint64_t x = 1469598103934665603ull;  // FNV-1a over N, F, D
    auto mix = [&](uint64_t v) {
        for (int b = 0; b < 8; b++) {
            x ^= (v >> (8 * b)) & 0xff;
            x *= 1099511628211ull;
        }
    };
    mix((uint64_t)h->N);
    for (auto v : h->F) mix((uint64_t)v);
    for (auto v : h->Dist) mix((uint64_t)v);
    return x;
}

template <class T>
void put(std::vector<char> &o, const T &v)
{
    const char *p = reinterpret_cast<const char *>(&v);
    o.insert(o.end(), p, p + sizeof(T));
}
template <class T>
void putv(std::vector<char> &o, const std::vector<T> &v)
{
    put(o, (uint64_t)v.size());
    const char *p = reinterpret_cast<const char *>(v.data());
    o.insert(o.end(), p, p + v.size() * sizeof(T));
}
struct Reader {
    const std::vector<char> &b;
    size_t pos = 0;
    bool ok = true;
    template <class T>
    T get()
    {
        T v{};
        if (pos + sizeof(T) > b.size()) {
            ok = false;
            return v;
        }
        memcpy(&v, b.data() + pos, sizeof(T));
        pos += sizeof(T);
        return v;
    }
    template <class T>
    std::vector<T> getv()
    {
        const uint64_t n = get<uint64_t>();
        std::vector<T> v;
        if (!ok || n > (1ull << 32) || pos + n * sizeof(T) > b.size()) {
            ok = false;
            return v;
        }
        v.resize(n);
        memcpy(v.data(), b.data() + pos, n * sizeof(T));
        pos += n * sizeof(T);
        return v;
    }
};

bool save_checkpoint(const Bnb &B, const char *path, std::string &err)
{
    std::vector<char> o;
    put(o, kCkptMagic);
    put(o, kCkptVersion);
    put(o, instance_digest(B.h0()));
    put(o, (int32_t)B.N);
    put(o, (int32_t)B.iters);
    put(o, (int32_t)B.sb_iters);
    put(o, (int32_t)B.warm);
    put(o, B.K);
    put(o, B.UB0);
    put(o, (int32_t)B.base_m);
    putv(o, B.root_fac);
    putv(o, B.root_loc);
    put(o, B.UB);
    put(o, (uint8_t)B.have);
    put(o, B.best);
    putv(o, B.best_perm);
    put(o, B.bounded);
    put(o, B.leaves);
    put(o, B.pruned);
    put(o, B.sb_cut);
    putv(o, B.bdepth);
    put(o, (uint64_t)B.stack.size());
    for (const Frame &F : B.stack) {
        putv(o, F.fac);
        putv(o, F.loc);
        putv(o, F.fs);
        putv(o, F.ls);
        putv(o, F.est);
        putv(o, F.lb);
        put(o, F.next);
        put(o, F.child_leaf);
    }
    const std::string tmp = std::string(path) + ".tmp";
    FILE *f = fopen(tmp.c_str(), "wb");
    if (!f) {
        err = "cannot open " + tmp;
        return false;
    }
    // the data reaches the disk before the rename publishes it (a crash leaves either the
    // old checkpoint or the new one, never a truncated file under `path`)
    const bool wrote = fwrite(o.data(), 1, o.size(), f) == o.size() && fflush(f) == 0 && fsync(fileno(f)) == 0;
    fclose(f);
    if (!wrote || rename(tmp.c_str(), path) != 0) {
        err = "cannot write checkpoint " + std::string(path);
        return false;
    }
    std::string dir(path);
    const size_t slash = dir.find_last_of('/');
    dir = slash == std::string::npos ? "." : (slash == 0 ? "/" : dir.substr(0, slash));
    const int dfd = open(dir.c_str(), O_RDONLY);
    if (dfd >= 0) {  // the rename itself (best effort: some file systems refuse directory fsync)
        fsync(dfd);
        close(dfd);
    }
    return true;
}

bool load_checkpoint(Bnb &B, const char *path, std::string &err)
{
    FILE *f = fopen(path, "rb");
    if (!f) {
        err = "cannot open " + std::string(path);
        return false;
    }
    std::vector<char> buf;
    char tmp[1 << 16];
    size_t r;
    while ((r = fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + r);
    fclose(f);
    Reader R{buf};
    if (R.get<uint64_t>() != kCkptMagic) {
        err = "not a checkpoint file";
        return false;
    }
    if (R.get<uint32_t>() != kCkptVersion) {
        err = "checkpoint format version mismatch";
        return false;
    }
    if (R.get<uint64_t>() != instance_digest(B.h0()) || R.get<int32_t>() != B.N || R.get<int32_t>() != B.iters ||
        R.get<int32_t>() != B.sb_iters || R.get<int32_t>() != (int32_t)B.warm || R.get<double>() != B.K ||
        R.get<double>() != B.UB0) {
        err = "checkpoint belongs to another instance or parameters";
        return false;
    }
    const int32_t base_m = R.get<int32_t>();
    const std::vector<int32_t> rf = R.getv<int32_t>(), rl = R.getv<int32_t>();
    if (!R.ok || base_m != B.base_m || rf != B.root_fac || rl != B.root_loc) {
        err = "checkpoint belongs to another subtree root";
        return false;
    }
    B.UB = R.get<double>();
    B.have = R.get<uint8_t>() != 0;
    B.best = R.get<int64_t>();
    B.best_perm = R.getv<int32_t>();
    B.bounded = R.get<int64_t>();
    B.leaves = R.get<int64_t>();
    B.pruned = R.get<int64_t>();
    B.sb_cut = R.get<int64_t>();
    B.bdepth = R.getv<int64_t>();
    if (B.bdepth.size() != 65) R.ok = false;
    const uint64_t nf = R.get<uint64_t>();
    B.stack.clear();
    for (uint64_t k = 0; k < nf && R.ok; k++) {
        Frame F;
        F.fac = R.getv<int32_t>();
        F.loc = R.getv<int32_t>();
        F.fs = R.getv<int32_t>();
        F.ls = R.getv<int32_t>();
        F.est = R.getv<double>();
        F.lb = R.getv<double>();
        F.next = R.get<uint32_t>();
        F.child_leaf = R.get<uint8_t>();
        B.stack.push_back(std::move(F));
    }
    if (!R.ok) {
        err = "truncated checkpoint";
        return false;
    }
    // frame k is the expanded node at depth base_m + k on the DFS path, below the root
    for (size_t k = 0; k < B.stack.size(); k++) {
        const Frame &F = B.stack[k];
        bool ok = F.fac.size() == (size_t)B.base_m + k && F.loc.size() == F.fac.size() &&
                  F.ls.size() == F.fs.size() && F.est.size() == F.fs.size() && F.lb.size() == F.fs.size() &&
                  F.next <= F.fs.size() && F.fac.size() < (size_t)B.N;
        for (size_t t = 0; ok && t < (size_t)B.base_m; t++)
            ok = F.fac[t] == B.root_fac[t] && F.loc[t] == B.root_loc[t];
        for (size_t t = 0; ok && t < F.fac.size(); t++)
            ok = F.fac[t] >= 0 && F.fac[t] < B.N && F.loc[t] >= 0 && F.loc[t] < B.N;
        if (!ok) {
            err = "inconsistent checkpoint stack";
            return false;
        }
    }
    B.root_done = true;
    return true;
}

// validated node (N <= 64, distinct facilities and locations in range)
bool node_ok(const qap_rlt2 *h, const qap_bnb_node *nd)
{
    if (nd->m < 0 || nd->m > h->N || h->N > 64) return false;
    std::vector<char> uf(h->N, 0), ul(h->N, 0);
    for (int t = 0; t < nd->m; t++) {
        const int f = nd->fac[t], l = nd->loc[t];
        if (f < 0 || f >= h->N || l < 0 || l >= h->N || uf[f] || ul[l]) return false;
        uf[f] = ul[l] = 1;
    }
    return true;
}

// the caller's handle plus batch-1 helper handles, each on its own stream
qap_status bnb_init(qap_rlt2 *h, const qap_bnb_opts *o, Bnb &b)
{
    if (h->world > 1 && o->batch > 1) return fail(h, QAP_E_ARG, "batched B&B needs a single-GPU handle");
    if (o->root && !node_ok(h, o->root)) return fail(h, QAP_E_ARG, "invalid root node");
    b.N = h->N;
    b.iters = o->iters;
    b.K = o->K;
    b.UB = b.UB0 = o->UB0;
    b.sb_iters = o->sb_iters;
    b.warm = o->warm != 0;
    if (b.warm && h->world > 1) return fail(h, QAP_E_ARG, "warm B&B needs a single-GPU handle");
    b.base_m = o->root ? o->root->m : 0;
    if (o->root) {
        b.root_fac.assign(o->root->fac, o->root->fac + o->root->m);
        b.root_loc.assign(o->root->loc, o->root->loc + o->root->m);
    }
    b.depth.push_back(h);
    const int B = o->batch < 1 ? 1 : (o->batch > b.N ? b.N : o->batch);
    int nh = b.warm ? B : B - 1;  // warm: the caller's handle keeps the root's state
    // helpers bound children (at most N - 1 free facilities), except that the first one also
    // hosts the strong-branching RLT1 batch of an expanded node in warm mode (pool[0]), which
    // needs the node's own size; when device memory runs out (large N: one handle holds the
    // N^6/2 tensor), fewer children are bounded at a time
    while ((int)h->bnb_helpers.size() < nh) {
        cudaStream_t s = nullptr;
        cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(h, e, "bnb stream");
        qap_rlt2_opts op{};
        op.device = h->device;
        op.cuda_stream = s;
        op.flags = h->flags & ~QAP_FLAG_TIME_KERNELS;
        op.lap_warps = h->lap_warps;
        qap_rlt2 *x = nullptr;
        const int cap = h->bnb_helpers.empty() ? h->N : h->N - 1;
        qap_status st = create_impl(h->N, h->F.data(), h->Dist.data(), &op, &x, false, cap);
        if (st != QAP_OK) {
            cudaStreamDestroy(s);
            if (st == QAP_E_CAPACITY && (b.warm ? (int)h->bnb_helpers.size() >= 1 : true)) {
                nh = (int)h->bnb_helpers.size();
                break;
            }
            return fail(h, st, std::string("bnb helper handle: ") + qap_last_error(nullptr));
        }
        h->bnb_streams.push_back(s);
        h->bnb_helpers.push_back(x);
    }
    if (!b.warm) b.pool.push_back(h);
    for (int k = 0; k < nh; k++) b.pool.push_back(h->bnb_helpers[k]);
    b.holds.assign(b.pool.size(), {0, -1});
    return QAP_OK;
}

void bnb_out(const Bnb &b, bool done, qap_bnb_result *out)
{
    out->complete = done ? 1 : 0;
    out->opt = b.have ? b.best : -1;
    for (int x = 0; x < 64; x++) out->perm[x] = (b.have && x < b.N) ? b.best_perm[x] : -1;
    out->bounded = b.bounded;
    out->leaves = b.leaves;
    out->pruned = b.pruned;
    out->sb_cut = b.sb_cut;
    int64_t open = 0;
    for (const Frame &F : b.stack) open += (int64_t)F.fs.size() - (int64_t)F.next;
    out->open = open;
    out->depth_max = (int32_t)(b.base_m + b.stack.size());
    for (int d = 0; d < 64; d++) out->bounded_by_depth[d] = b.bdepth[d];
}
}  // namespace

extern "C" {

qap_status qap_bnb_run(qap_rlt2 *h, const qap_bnb_opts *o, qap_bnb_result *out)
{
    NvtxRange nv("qap_bnb_run");
    if (!h || !o || !out || o->iters < 0) return QAP_E_ARG;
    if ((o->resume || o->checkpoint_every > 0) && !o->checkpoint_path)
        return fail(h, QAP_E_ARG, "checkpointing needs checkpoint_path");
    Bnb b;
    qap_status st0 = bnb_init(h, o, b);
    if (st0 != QAP_OK) return st0;
    b.sync_fn = o->sync;
    b.donate_fn = o->donate;
    b.ctx = o->ctx;
    b.sync_every = o->sync_every > 0 ? o->sync_every : 32;
    std::string err;
    if (o->resume) {
        if (!load_checkpoint(b, o->checkpoint_path, err)) return fail(h, QAP_E_ARG, err);
        // warm: the device states of the expanded nodes on the DFS path are rebuilt
        if (b.warm)
            for (size_t k = 0; k < b.stack.size(); k++)
                if (!b.derive(k, b.stack[k].fac, b.stack[k].loc)) return b.st;
    } else {
        b.start_at(o->root);
        if (b.st != QAP_OK) return b.st;
    }
    if (b.sync_fn && !b.sync()) return fail(h, b.st, "bnb aborted by the sync callback");
    int64_t since = 0;
    bool done = false;
    const int64_t b0 = b.bounded;
    while (true) {
        if (o->max_nodes > 0 && b.bounded - b0 >= o->max_nodes) break;  // budget: stop here
        const int64_t before = b.bounded;
        if (!b.step()) {
            done = b.st == QAP_OK;
            break;
        }
        if (o->checkpoint_every > 0 && (since += b.bounded - before) >= o->checkpoint_every) {
            since = 0;
            if (!save_checkpoint(b, o->checkpoint_path, err)) return fail(h, QAP_E_ARG, err);
        }
        if (b.sync_fn && ((b.since_sync += b.bounded - before) >= b.sync_every || b.improved) && !b.sync())
            return fail(h, b.st, "bnb aborted by the sync callback");
    }
    if (b.st != QAP_OK) return b.st;
    if (b.sync_fn && !b.sync()) return fail(h, b.st, "bnb aborted by the sync callback");
    if (!done && o->checkpoint_path && !save_checkpoint(b, o->checkpoint_path, err)) return fail(h, QAP_E_ARG, err);
    bnb_out(b, done, out);
    return QAP_OK;
}

qap_status qap_bnb_frontier(qap_rlt2 *h, const qap_bnb_opts *o, int32_t target, qap_bnb_node *nodes, int32_t cap,
                            int32_t *n_nodes, qap_bnb_result *out)
{
    if (!h || !o || !out || !n_nodes || o->iters < 0 || cap < 0 || (cap > 0 && !nodes)) return QAP_E_ARG;
    Bnb b;
    qap_bnb_opts oc = *o;
    oc.warm = 0;  // the breadth-first frontier bounds cold (node states are not kept level-wide)
    qap_status st0 = bnb_init(h, &oc, b);
    if (st0 != QAP_OK) return st0;
    qap_bnb_node root{};
    root.lb = NAN;
    if (o->root) root = *o->root;
    std::vector<qap_bnb_node> level;
    auto vecs = [](const qap_bnb_node &nd, std::vector<int32_t> &fac, std::vector<int32_t> &loc) {
        fac.assign(nd.fac, nd.fac + nd.m);
        loc.assign(nd.loc, nd.loc + nd.m);
    };
    std::vector<int32_t> fac, loc;
    vecs(root, fac, loc);
    if (b.N - root.m <= 3) {
        b.leaf(fac, loc);
    } else {
        if (std::isnan(root.lb)) {
            if ((b.st = qap_rlt2_fix(h, root.m, fac.data(), loc.data())) != QAP_OK) return b.st;
            qap_rlt2_result r{};
            if ((b.st = qap_rlt2_bound(h, b.iters, b.K, b.UB, &r)) != QAP_OK) return b.st;
            b.counted(root.m);
            root.lb = r.lb;
        }
        if (b.cut(root.lb)) b.pruned++;
        else level.push_back(root);
    }
    while (!level.empty() && (int64_t)level.size() < (int64_t)target) {
        std::vector<qap_bnb_node> next;
        for (const qap_bnb_node &nd : level) {
            if (b.cut(nd.lb)) {  // the incumbent improved since nd was bounded
                b.pruned++;
                continue;
            }
            vecs(nd, fac, loc);
            Frame F;
            if (!b.make_frame(fac, loc, F)) return b.st;
            for (size_t c = 0; c < F.fs.size(); c++) {
                if (b.cut(F.est[c])) {
                    b.sb_cut++;
                    continue;
                }
                qap_bnb_node ch = nd;
                ch.m = nd.m + 1;
                ch.fac[nd.m] = F.fs[c];
                ch.loc[nd.m] = F.ls[c];
                if (F.child_leaf) {
                    vecs(ch, fac, loc);
                    b.leaf(fac, loc);
                    continue;
                }
                b.counted(ch.m);
                if (b.cut(F.lb[c])) {
                    b.pruned++;
                    continue;
                }
                ch.lb = F.lb[c];
                next.push_back(ch);
            }
        }
        level.swap(next);
    }
    *n_nodes = (int32_t)level.size();
    if ((int64_t)level.size() > (int64_t)cap) return fail(h, QAP_E_CAPACITY, "frontier larger than cap");
    for (size_t k = 0; k < level.size(); k++) nodes[k] = level[k];
    bnb_out(b, level.empty(), out);
    return QAP_OK;
}

qap_status qap_bnb_solve(qap_rlt2 *h, int32_t iters, double K, double UB0, int32_t batch, int32_t sb_iters,
                         int64_t *opt, int32_t *perm, int64_t *bounded, int64_t *leaves, int64_t *pruned,
                         int64_t *sb_cut)
{
    if (!h || !opt || !perm) return QAP_E_ARG;
    qap_bnb_opts o{};
    o.iters = iters;
    o.K = K;
    o.UB0 = UB0;
    o.batch = batch;
    o.sb_iters = sb_iters;
    qap_bnb_result r{};
    qap_status s = qap_bnb_run(h, &o, &r);
    if (s != QAP_OK) return s;
    *opt = r.opt;
    if (r.opt >= 0)
        for (int x = 0; x < h->N; x++) perm[x] = r.perm[x];
    if (bounded) *bounded = r.bounded;
    if (leaves) *leaves = r.leaves;
    if (pruned) *pruned = r.pruned;
    if (sb_cut) *sb_cut = r.sb_cut;
    return QAP_OK;
}

qap_status qap_nccl_unique_id(void *id128)
{
    if (!id128) return QAP_E_ARG;
    const char *why = "";
    if (nccl_unique_id(id128, &why) != 0) return fail(nullptr, QAP_E_NCCL, std::string("ncclGetUniqueId: ") + why);
    return QAP_OK;
}

qap_status qap_rlt2_shard_info(const qap_rlt2 *h, int32_t *world, int32_t *rank, int64_t *blk_lo, int64_t *blk_hi,
                               int64_t *tiles_local, int64_t *tiles_shared, int64_t *slots)
{
    if (!h) return QAP_E_ARG;
    if (world) *world = h->world;
    if (rank) *rank = h->rank;
    const bool sh = h->world > 1;
    if (blk_lo) *blk_lo = sh ? h->plan.blk_lo[h->rank] : 0;
    if (blk_hi) *blk_hi = sh ? h->plan.blk_lo[h->rank + 1] : h->geom.nblk;
    if (tiles_local) *tiles_local = sh ? h->plan.n_local : -1;
    if (tiles_shared) *tiles_shared = sh ? h->plan.n_agg + h->plan.n_hold : 0;
    if (slots) *slots = sh ? h->plan.total_slots : 0;
    return QAP_OK;
}

qap_status qap_shard_plan(int32_t n, int32_t world, int32_t rank, int64_t *blk_lo /*world+1*/, int64_t *peer_slots /*world*/,
                          int32_t *tiles, int32_t *tinfo, int64_t tiles_cap, int64_t *n_tiles)
{
    if (n < 3 || n > kMaxN || world < 1 || world > 64 || rank < 0 || rank >= world) return QAP_E_ARG;
    ShardPlan P;
    make_plan(n, world, rank, P);
    if (blk_lo)
        for (int q = 0; q <= world; q++) blk_lo[q] = P.blk_lo[q];
    if (peer_slots)
        for (int q = 0; q < world; q++) peer_slots[q] = P.peer_slots[q];
    if (n_tiles) *n_tiles = (int64_t)P.tiles.size();
    if (tiles || tinfo) {
        if ((int64_t)P.tiles.size() > tiles_cap) return QAP_E_ARG;
        for (size_t t = 0; t < P.tiles.size(); t++) {
            if (tiles) tiles[t] = P.tiles[t];
            if (tinfo) tinfo[t] = P.tinfo[t];
        }
    }
    return QAP_OK;
}

qap_status qap_rlt2_create_group(int32_t G, int32_t N, const int64_t *F, const int64_t *D, const qap_rlt2_opts *opts,
                                 qap_rlt2 **out)
{
    if (!out || G < 1 || G > 64) return fail(nullptr, QAP_E_ARG, "bad group size");
    for (int r = 0; r < G; r++) out[r] = nullptr;
    qap_rlt2_opts o{};
    if (opts) o = *opts;
    else o.device = -1;
    o.world = G;
    o.nccl_id = nullptr;
    for (int r = 0; r < G; r++) {
        o.rank = r;
        qap_status s = create_impl(N, F, D, &o, &out[r], G > 1);
        if (s != QAP_OK) {
            for (int q = 0; q < r; q++) qap_destroy(out[q]);
            for (int q = 0; q < G; q++) out[q] = nullptr;
            return s;
        }
    }
    return QAP_OK;
}

// In-process group: every rank's phases in turn; the collectives are device copies.
qap_status qap_rlt2_group_bound(qap_rlt2 *const *hs, int32_t G, int32_t max_iters, double K, double UB,
                                qap_rlt2_result *out)
{
    if (!hs || !out || G < 1) return QAP_E_ARG;
    if (G == 1) return qap_rlt2_bound(hs[0], max_iters, K, UB, out);
    for (int r = 0; r < G; r++)
        if (!hs[r] || hs[r]->world != G || hs[r]->rank != r || !hs[r]->loopback) return QAP_E_ARG;
    qap_rlt2 *h0 = hs[0];
    if (max_iters < 0 || !(K >= 0.0) || std::isnan(UB)) return fail(h0, QAP_E_ARG, "bad max_iters/K/UB");
    cudaError_t e = cudaSuccess;
#define GCHK(x)                                              \
    if ((e = (x)) != cudaSuccess) return cuda_fail(h0, e, #x);
    for (int r = 0; r < G; r++) {
        qap_rlt2 *h = hs[r];
        h->call_launches = 0;
        GCHK(launch_ctl_begin(h->dCtl, K, UB, h->trace_cap, h->stream));
        if (h->next_phase == PH_FRESH) {
            GCHK(run_phase(h, QAP_PHASE_ITER0, h->stream, true));
            h->next_phase = QAP_PHASE_TRANSFER;
        }
    }
    for (int t = 0; t < max_iters; t++) {
        for (int ph = QAP_PHASE_TRANSFER; ph <= QAP_PHASE_CONC_D; ph++) {
            for (int r = 0; r < G; r++) GCHK(run_shard_sub(hs[r], ph, 0, hs[r]->stream));
            GCHK(cudaDeviceSynchronize());
            for (int r = 0; r < G; r++) {
                const ShardPlan &P = hs[r]->plan;
                for (int q = 0; q < G; q++) {
                    if (q == r) continue;
                    if (ph == QAP_PHASE_TRANSFER) {  // r receives q's partials of their shared tiles
                        const ShardPlan &Q = hs[q]->plan;
                        const size_t cnt = (size_t)P.peer_slots[q] * kSlot;
                        if (cnt)
                            GCHK(cudaMemcpy(hs[r]->dRecv + (size_t)P.peer_off[q] * kSlot,
                                            hs[q]->dSend + (size_t)Q.peer_off[r] * kSlot, cnt * 8,
                                            cudaMemcpyDeviceToDevice));
                    } else {  // r receives q's level-2 values
                        const size_t cnt = (size_t)(P.blk_lo[q + 1] - P.blk_lo[q]);
                        if (cnt)
                            GCHK(cudaMemcpy(hs[r]->dSall + P.blk_lo[q], hs[q]->dSall + P.blk_lo[q], cnt * 8,
                                            cudaMemcpyDeviceToDevice));
                    }
                }
            }
            for (int r = 0; r < G; r++) GCHK(run_shard_sub(hs[r], ph, 1, hs[r]->stream));
        }
        for (int r = 0; r < G; r++) {
            GCHK(run_phase(hs[r], QAP_PHASE_CONC_C, hs[r]->stream, true));
            GCHK(run_phase(hs[r], QAP_PHASE_CONC_B, hs[r]->stream, true));
        }
    }
#undef GCHK
    for (int r = 0; r < G; r++) {
        Ctl c;
        qap_status s = read_ctl(hs[r], c);
        if (s != QAP_OK) return s;
        out[r].lb = c.lb;
        out[r].lb_glb = c.lb_glb;
        out[r].iters = c.iters;
        out[r].status = c.status;
        out[r].launches = hs[r]->call_launches;
        if (out[r].lb_trace && out[r].lb_trace_cap > 0 && c.iters > 0) {
            const int cnt = c.iters < out[r].lb_trace_cap ? c.iters : out[r].lb_trace_cap;
            e = cudaMemcpy(out[r].lb_trace, hs[r]->dTrace, (size_t)cnt * 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_fail(hs[r], e, "trace copy");
        }
    }
    return QAP_OK;
}

}  // extern "C"

