// rlt2_shard.cu — shard plan and collective transports (see rlt2_shard.h).
#include "rlt2_shard.h"

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#ifdef QAP_HAVE_NCCL
#include <nccl.h>
#endif

namespace rlt2 {

namespace {
// Host-staged collectives (qap_host_transport): pinned staging buffers grown on demand; the
// stream is drained before each callback and after the copies back.
struct HostTransport : Transport {
    qap_host_transport cb{};
    int world = 1, rank = 0;
    double *hsend = nullptr, *hrecv = nullptr;
    size_t cap = 0;
    std::vector<int64_t> off, cnt;
    std::string err;
    ~HostTransport() override
    {
        cudaFreeHost(hsend);
        cudaFreeHost(hrecv);
    }
    cudaError_t grow(size_t n)
    {
        if (n <= cap) return cudaSuccess;
        cudaFreeHost(hsend);
        cudaFreeHost(hrecv);
        hsend = hrecv = nullptr;
        cap = 0;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void **>(&hsend), n * 8);
        if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void **>(&hrecv), n * 8);
        if (e == cudaSuccess) cap = n;
        return e;
    }
    cudaError_t exchange(const ShardPlan &P, const double *send, double *recv, int piece, cudaStream_t st) override
    {
        const size_t tot = (size_t)P.total_slots * kSlot;
        if (tot == 0) return cudaSuccess;
        cudaError_t e = grow(tot);
        if (e != cudaSuccess) return e;
        off.assign(P.G, 0);
        cnt.assign(P.G, 0);
        for (int q = 0; q < P.G; q++) {
            if (q == P.r) continue;
            const int64_t a = xchunk_lo(P.peer_slots[q], piece), b = xchunk_lo(P.peer_slots[q], piece + 1);
            off[q] = (P.peer_off[q] + a) * kSlot;
            cnt[q] = (b - a) * kSlot;
            if (cnt[q] && (e = cudaMemcpyAsync(hsend + off[q], send + off[q], cnt[q] * 8, cudaMemcpyDeviceToHost, st)) !=
                              cudaSuccess)
                return e;
        }
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        if (cb.exchange(cb.ctx, hsend, hrecv, off.data(), cnt.data(), world, rank) != 0) {
            err = "host transport: exchange callback failed";
            return cudaErrorUnknown;
        }
        for (int q = 0; q < P.G; q++)
            if (cnt[q] &&
                (e = cudaMemcpyAsync(recv + off[q], hrecv + off[q], cnt[q] * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess)
                return e;
        return cudaStreamSynchronize(st);
    }
    cudaError_t allgather(const ShardPlan &P, double *S_all, cudaStream_t st) override
    {
        const size_t tot = (size_t)P.blk_lo[P.G];
        if (tot == 0) return cudaSuccess;
        cudaError_t e = grow(tot);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hrecv, S_all, tot * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        if (cb.allgather(cb.ctx, hrecv, P.blk_lo.data(), world, rank) != 0) {
            err = "host transport: allgather callback failed";
            return cudaErrorUnknown;
        }
        if ((e = cudaMemcpyAsync(S_all, hrecv, tot * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
        return cudaStreamSynchronize(st);
    }
    const char *error() const override { return err.c_str(); }
};
}  // namespace

Transport *make_host_transport(const qap_host_transport &cb, int world, int rank)
{
    auto *t = new HostTransport();
    t->cb = cb;
    t->world = world;
    t->rank = rank;
    return t;
}

void make_plan(int n, int G, int r, ShardPlan &P)
{
    Geom g;
    make_geom(n, g);
    P.n = n;
    P.G = G;
    P.r = r;
    // LPT: facilities by decreasing block count, each to the least-loaded rank
    std::vector<int64_t> load(G, 0);
    P.owner.assign(n, 0);
    for (int f = 0; f < n; f++) {  // block counts decrease with f, so index order is LPT order
        int best = 0;
        for (int q = 1; q < G; q++)
            if (load[q] < load[best]) best = q;
        P.owner[f] = best;
        load[best] += g.off[f + 1 < n ? f + 1 : n] - g.off[f];
    }
    P.blk_lo.assign(G + 1, 0);
    for (int q = 0; q < G; q++) P.blk_lo[q + 1] = P.blk_lo[q] + load[q];
    P.pos_off.assign(n, 0);
    P.loc_off.assign(n, 0);
    std::vector<int64_t> fill(G, 0);
    for (int f = 0; f < n; f++) {
        const int q = P.owner[f];
        const int64_t cnt = g.off[f + 1 < n ? f + 1 : n] - g.off[f];
        P.loc_off[f] = fill[q] - g.off[f];
        P.pos_off[f] = P.blk_lo[q] + fill[q] - g.off[f];
        fill[q] += cnt;
    }
    const std::vector<int> &owner = P.owner;

    const int ntile = (n + TT - 1) / TT, nt3 = ntile * ntile * ntile;
    P.tiles.clear();
    P.tinfo.clear();
    P.peer_slots.assign(G, 0);
    P.peer_off.assign(G, 0);
    P.n_local = P.n_agg = P.n_hold = 0;
    // pass 1: count per peer; pass 2: assign slots in ascending global tile id
    for (int pass = 0; pass < 2; pass++) {
        std::vector<int64_t> pos(G, 0);
        int tq = 0;
        for (int i = 0; i < n; i++)
            for (int k = i + 1; k < n; k++)
                for (int p = k + 1; p < n; p++, tq++) {
                    const int A = owner[i], B = owner[k];
                    if (A != r && B != r) continue;
                    const int kind = (A == r && B == r) ? 0 : (A == r ? 1 : 2);
                    const int peer = kind == 1 ? B : A;
                    if (pass == 0) {
                        if (kind != 0) P.peer_slots[peer] += nt3;
                        continue;
                    }
                    for (int t = 0; t < nt3; t++) {
                        P.tiles.push_back(tq * nt3 + t);
                        if (kind == 0) {
                            P.tinfo.push_back(0);
                            P.n_local++;
                        } else {
                            const int64_t slot = P.peer_off[peer] + pos[peer]++;
                            P.tinfo.push_back(kind | (int)(slot << 2));
                            (kind == 1 ? P.n_agg : P.n_hold)++;
                        }
                    }
                }
        if (pass == 0) {
            int64_t acc = 0;
            for (int q = 0; q < G; q++) {
                P.peer_off[q] = acc;
                acc += P.peer_slots[q];
            }
            P.total_slots = acc;
        }
    }
    // local tiles first (they are transferred while the shared ones are exchanged), then the
    // shared ones by exchange piece; ascending global tile id within each group
    std::vector<int> tl, il;
    std::vector<std::vector<int>> ts(kXChunks), is(kXChunks);
    for (size_t t = 0; t < P.tiles.size(); t++) {
        if ((P.tinfo[t] & 3) == 0) {
            tl.push_back(P.tiles[t]);
            il.push_back(P.tinfo[t]);
            continue;
        }
        // the tile's slot relative to its peer's range -> its piece
        const int64_t slot = P.tinfo[t] >> 2;
        int q = 0;  // the peer whose slot range holds it (every shared tile has one)
        while (q + 1 < G && !(slot >= P.peer_off[q] && slot < P.peer_off[q] + P.peer_slots[q])) q++;
        const int64_t rel = slot - P.peer_off[q];
        int c = 0;
        while (c + 1 < kXChunks && rel >= xchunk_lo(P.peer_slots[q], c + 1)) c++;
        ts[c].push_back(P.tiles[t]);
        is[c].push_back(P.tinfo[t]);
    }
    P.piece_lo[0] = 0;
    for (int c = 0; c < kXChunks; c++) {
        tl.insert(tl.end(), ts[c].begin(), ts[c].end());
        il.insert(il.end(), is[c].begin(), is[c].end());
        P.piece_lo[c + 1] = P.piece_lo[c] + (int)ts[c].size();
    }
    P.tiles.swap(tl);
    P.tinfo.swap(il);
}

#ifdef QAP_HAVE_NCCL
namespace {
struct NcclApi {
    void *lib = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclBroadcast) bcast = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    std::string why;
    bool load()
    {
        if (lib) return true;
        // prefer the copy already loaded by the process (torch's), else any on the path
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            why = std::string("dlopen(libnccl.so.2): ") + dlerror();
            return false;
        }
#define SYM(f, name)                                                     \
    f = reinterpret_cast<decltype(f)>(dlsym(lib, name));                 \
    if (!f) {                                                            \
        why = std::string("missing NCCL symbol ") + name;                \
        return false;                                                    \
    }
        SYM(getUniqueId, "ncclGetUniqueId");
        SYM(commInitRank, "ncclCommInitRank");
        SYM(commDestroy, "ncclCommDestroy");
        SYM(send, "ncclSend");
        SYM(recv, "ncclRecv");
        SYM(bcast, "ncclBroadcast");
        SYM(groupStart, "ncclGroupStart");
        SYM(groupEnd, "ncclGroupEnd");
        SYM(errStr, "ncclGetErrorString");
#undef SYM
        return true;
    }
};
NcclApi g_nccl;

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    std::string err;
    ~NcclTransport() override
    {
        if (comm) g_nccl.commDestroy(comm);
    }
    cudaError_t fail(ncclResult_t r)
    {
        err = std::string("NCCL: ") + g_nccl.errStr(r);
        return cudaErrorUnknown;
    }
    cudaError_t exchange(const ShardPlan &P, const double *send, double *recv, int piece, cudaStream_t st) override
    {
        ncclResult_t r;
        if ((r = g_nccl.groupStart()) != ncclSuccess) return fail(r);
        for (int q = 0; q < P.G; q++) {
            const int64_t a = xchunk_lo(P.peer_slots[q], piece), b = xchunk_lo(P.peer_slots[q], piece + 1);
            if (q == P.r || b == a) continue;
            const size_t cnt = (size_t)(b - a) * kSlot;
            const size_t off = (size_t)(P.peer_off[q] + a) * kSlot;
            if ((r = g_nccl.send(send + off, cnt, ncclFloat64, q, comm, st)) != ncclSuccess) return fail(r);
            if ((r = g_nccl.recv(recv + off, cnt, ncclFloat64, q, comm, st)) != ncclSuccess) return fail(r);
        }
        if ((r = g_nccl.groupEnd()) != ncclSuccess) return fail(r);
        return cudaSuccess;
    }
    cudaError_t allgather(const ShardPlan &P, double *S_all, cudaStream_t st) override
    {
        ncclResult_t r;
        if ((r = g_nccl.groupStart()) != ncclSuccess) return fail(r);
        for (int q = 0; q < P.G; q++) {
            const size_t cnt = (size_t)(P.blk_lo[q + 1] - P.blk_lo[q]);
            if (cnt == 0) continue;
            double *p = S_all + P.blk_lo[q];
            if ((r = g_nccl.bcast(p, p, cnt, ncclFloat64, q, comm, st)) != ncclSuccess) return fail(r);
        }
        if ((r = g_nccl.groupEnd()) != ncclSuccess) return fail(r);
        return cudaSuccess;
    }
    const char *error() const override { return err.c_str(); }
};
}  // namespace

Transport *make_nccl_transport(const void *unique_id, int world, int rank, int device, const char **err)
{
    if (!g_nccl.load()) {
        *err = g_nccl.why.c_str();
        return nullptr;
    }
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof id);
    cudaSetDevice(device);
    auto *t = new NcclTransport();
    ncclResult_t r = g_nccl.commInitRank(&t->comm, world, id, rank);
    if (r != ncclSuccess) {
        static std::string msg;
        msg = std::string("ncclCommInitRank: ") + g_nccl.errStr(r);
        *err = msg.c_str();
        t->comm = nullptr;
        delete t;
        return nullptr;
    }
    return t;
}

int nccl_unique_id(void *out128, const char **err)
{
    if (!g_nccl.load()) {
        *err = g_nccl.why.c_str();
        return 1;
    }
    ncclUniqueId id;
    ncclResult_t r = g_nccl.getUniqueId(&id);
    if (r != ncclSuccess) {
        *err = g_nccl.errStr(r);
        return 1;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, sizeof id);
    return 0;
}
#else
Transport *make_nccl_transport(const void *, int, int, int, const char **err)
{
    *err = "built without NCCL headers";
    return nullptr;
}
int nccl_unique_id(void *, const char **err)
{
    *err = "built without NCCL headers";
    return 1;
}
#endif

}  // namespace rlt2
