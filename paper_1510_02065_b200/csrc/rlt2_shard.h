// rlt2_shard.h — multi-GPU sharding of one RLT2 bound (host side).
//
// The stored level-2 blocks D{ij,kl} (i<k) are partitioned by their first FACILITY i:
// facilities are assigned to ranks by longest-processing-time balancing of their block
// counts (ties: lower facility, lower rank).  Rank r keeps its blocks in ascending global
// order (local slice); the level-2 values S are all-gathered rank-major.  The transfer is tiled by
// facility triple (i,k,p) × location tile: members e1, e2 of a tile's classes live on
// owner(i) (the aggregator), e3 on owner(k) (the holder).  Tiles with owner(i) != owner(k)
// are exchanged: for each peer pair the list of shared tiles sorted by global tile id
// fixes a symmetric slot layout of the send/receive buffers (512 doubles per tile).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/qap_rlt2.h"
#include "rlt2_internal.h"

namespace rlt2 {

constexpr int kSlot = TT * TT * TT;  // doubles per exchanged tile (one per class slot)
// The shared tiles are exchanged in kXChunks pieces (pack piece c+1 / apply piece c-1 while piece c
// is on the wire): piece c of the slots a rank pair shares is [floor(c S / K), floor((c+1) S / K))
// of their S common slots, the same range on both sides.
constexpr int kXChunks = 4;
inline int64_t xchunk_lo(int64_t slots, int c) { return slots * c / kXChunks; }

struct ShardPlan {
    int n = 0, G = 1, r = 0;
    std::vector<int> owner;        // n: rank owning the blocks of first facility f
    std::vector<int64_t> blk_lo;   // G+1: rank-major offsets: rank q's blocks are S_rm[blk_lo[q], blk_lo[q+1])
    std::vector<int64_t> pos_off;  // n: rank-major position of global block b of facility f = b + pos_off[f]
    std::vector<int64_t> loc_off;  // n: local index of global block b of a facility f owned here = b + loc_off[f]
    std::vector<int> tiles;        // this rank's tiles (global id): the n_local local ones (ascending), then
                                   // the shared ones by exchange piece (ascending within a piece)
    std::vector<int> tinfo;        // kind | slot << 2
    std::vector<int64_t> peer_slots, peer_off;  // G: exchanged tiles per peer, slot offset
    int64_t total_slots = 0;
    int n_local = 0, n_agg = 0, n_hold = 0;
    int piece_lo[kXChunks + 1] = {0};  // shared tiles of piece c: tiles[n_local + piece_lo[c] .. n_local + piece_lo[c+1])
};

// Partition + tile lists of rank r among G for the reduced size n.
void make_plan(int n, int G, int r, ShardPlan &P);

// Collective transport between the ranks of one sharded bound.
struct Transport {
    virtual ~Transport() {}
    // piece c (xchunk_lo) of send[peer_off[s]*kSlot .. + peer_slots[s]*kSlot) to every peer s,
    // the same range of recv from s; enqueued on st (the host transport returns when it is done)
    virtual cudaError_t exchange(const ShardPlan &P, const double *send, double *recv, int piece, cudaStream_t st) = 0;
    // S_all[blk_lo[q] .. blk_lo[q+1]) of rank q -> every rank (in place)
    virtual cudaError_t allgather(const ShardPlan &P, double *S_all, cudaStream_t st) = 0;
    virtual const char *error() const = 0;
};

// Host-staged: device buffers -> pinned host -> the caller's callbacks -> device.
Transport *make_host_transport(const qap_host_transport &cb, int world, int rank);
// NCCL (dlopen'd libnccl.so.2): nullptr if NCCL is unavailable; `err` says why.
Transport *make_nccl_transport(const void *unique_id, int world, int rank, int device, const char **err);
// 128-byte ncclUniqueId (rank 0 creates it, the caller broadcasts it to the other ranks).
int nccl_unique_id(void *out128, const char **err);

}  // namespace rlt2
