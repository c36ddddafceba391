// am_hashset.cuh -- device-side insert into the state hash set (am_hash.cu) and the per-item
// canonical insert + frontier step of an iteration, shared by k_hash_upsert / k_canon_frontier
// (am_hash.cu) and the narrow composition's tile epilogue (am_narrow.cu).
#pragma once

#include "am_internal.h"

namespace am {

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) { return *reinterpret_cast<const volatile uint64_t*>(p); }

__device__ __forceinline__ bool keys_equal(const uint64_t* a, const uint64_t* b, int kw) {
    for (int i = 0; i < kw; i++)
        if (a[i] != b[i]) return false;
    return true;
}

#define GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// Insert a batch of keys (open addressing, linear probing).  A key that claims an empty slot
// is new: the same thread appends it to the pool right away (key, flags, hint), publishes the
// slot's final value (fingerprint | pool index) after a fence, and queues it.  Until then the
// slot holds a candidate marker (fingerprint | cand bit | batch index) and concurrent inserters
// of the same key compare against the batch copy, so duplicates inside a batch and against the
// table resolve in this one launch (dup_ref: pool index, or -2 - batch index of the winner whose
// pool index lands in pool_idx).
// one key of an upsert launch: item i of the launch (source row ci = idx ? idx[i] : i); returns the
// status (1 new, 0 present) and the new entry's pool index in *pidx (-1 otherwise)
__device__ __forceinline__ int32_t upsert_one(const HashSet& H, const uint64_t* src, const int32_t* idx, int64_t i,
                                              int64_t ci, uint64_t* slot_out, int32_t* dup_ref, uint32_t flag,
                                              int32_t* queue, unsigned long long* q_tail, const double* src_hint,
                                              int32_t* pidx, const int64_t* src_par = nullptr) {
    const uint64_t* key = src + ci * H.KW;
    uint64_t h = key_hash(key, H.KW);
    uint64_t fp = h >> 33;
    uint64_t pos = h & H.mask;
    const uint64_t mine = (fp << 33) | (1ull << 32) | (uint64_t)(uint32_t)i;
    int32_t st = -1, dref = -1;  // -1: table full (host keeps load factor <= 1/2, so unreachable)
    for (uint64_t probe = 0; probe <= H.mask; probe++) {
        uint64_t v = ld_volatile(H.table + pos);
        if (v == kEmpty) {
            unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(H.table + pos),
                                               (unsigned long long)kEmpty, (unsigned long long)mine);
            if (old == kEmpty) {
                st = 1;
                slot_out[ci] = pos;
                break;
            }
            v = old;
        }
        if ((v >> 33) == fp) {
            uint32_t ref = (uint32_t)v;
            const bool cand = (v >> 32) & 1ull;
            const int64_t other_ci = idx ? idx[ref] : (int64_t)ref;
            const uint64_t* other = cand ? src + other_ci * H.KW : H.pool + (int64_t)ref * H.KW;
            if (keys_equal(key, other, H.KW)) {
                st = 0;
                dref = cand ? (int32_t)(-2 - other_ci) : (int32_t)ref;
                break;
            }
        }
        pos = (pos + 1) & H.mask;
    }
    if (dup_ref) dup_ref[ci] = dref;
    *pidx = -1;
    if (st != 1) return st;
    const unsigned long long p = atomicAdd(H.n_pool, 1ull);
    uint64_t* dst = H.pool + (int64_t)p * H.KW;
    for (int w = 0; w < H.KW; w++) dst[w] = key[w];
    H.pool_flags[p] = flag;
    H.pool_vn[p] = -1;
    const double4 hint = src_hint ? reinterpret_cast<const double4*>(src_hint)[ci]
                                  : make_double4(0.0, 0.0, 0.0, __longlong_as_double(0x7ff0000000000000ll));
    reinterpret_cast<double4*>(H.pool_hint)[p] = hint;
    if (H.pool_par) H.pool_par[p] = src_par ? src_par[ci] : 0;
    __threadfence();
    H.table[pos] = (fp << 33) | (uint64_t)(uint32_t)p;
    *pidx = (int32_t)p;
    if (queue) {
        const unsigned long long qi = atomicAdd(q_tail, 1ull);
        queue[qi] = (int32_t)p;
        if (H.queue_par) H.queue_par[qi] = src_par ? src_par[ci] : 0;
    }
    return st;
}

// atomicAdd(ctr, 1) for every converged lane of the warp with one atomic per warp (the frontier
// and visited-cell counters are hit by every batch item): returns this lane's old value
__device__ __forceinline__ unsigned long long warp_agg_inc(unsigned long long* ctr) {
    const unsigned act = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(act) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(act));
    base = __shfl_sync(act, base, leader);
    return base + (unsigned long long)__popc(act & ((1u << lane) - 1u));
}

// One batch item after its composition (reference marching.py:221-245 with the canonical state
// of _refine / canonical_state): a changed (canonicalised) key is inserted (or routed to its
// owner rank); a new state joins the frontier (f_items / f_pool) unless the max_cells cap is
// reached; a deferred cell solved again rejoins it directly.
__device__ __forceinline__ void canon_frontier_one(const HashSet& H, const uint64_t* ckey, int changed, int32_t bp,
                                                   int64_t b, int rank, int world, uint64_t* outbox,
                                                   unsigned long long* n_out, int32_t* canon_pos, int32_t* status2,
                                                   uint64_t* slot2, int32_t* canon_pool, const double* ckey_hint,
                                                   int32_t* f_items, int32_t* f_pool, unsigned long long* ctr,
                                                   long long max_cells) {
    const int KW = H.KW;
    int32_t p = -1;
    const uint32_t fl = H.pool_flags[bp];
    H.pool_flags[bp] = (fl | 2u) & ~kPoolDeferred;   // composed (probe records can resolve)
    if (fl & kPoolDeferred) {   // a deferred cell solved again: visited and counted already
        const unsigned long long kf = warp_agg_inc(ctr + C_NF);
        f_items[kf] = (int32_t)b;
        f_pool[kf] = bp;
        return;
    }
    if (!changed) {
        p = bp;
    } else {
        const uint64_t* k = ckey + b * KW;
        if (world > 1 && key_owner(k, KW, world) != rank) {
            const unsigned long long o = atomicAdd(n_out, 1ull);
            for (int w = 0; w < KW; w++) outbox[o * KW + w] = k[w];
            canon_pos[b] = -2;   // handled by its owner
        } else {
            canon_pos[b] = 1;
            atomicAdd(ctr + C_NX, 1ull);   // canonical inserts (stats)
            int32_t np;
            const int32_t st = upsert_one(H, ckey, nullptr, b, b, slot2, nullptr, 0u, nullptr, nullptr, ckey_hint, &np);
            status2[b] = st;
            canon_pool[b] = np;
            if (st == 1) p = np;
        }
    }
    if (p < 0) return;
    const unsigned long long tot = warp_agg_inc(ctr + C_TOTAL);
    if ((long long)tot >= max_cells) {  // max_cells cap (reference marching.py:240-242)
        atomicAdd(ctr + C_CAPPED, 1ull);
        return;
    }
    const unsigned long long kf = warp_agg_inc(ctr + C_NF);
    H.pool_flags[p] |= 1u;
    f_items[kf] = (int32_t)b;
    f_pool[kf] = p;
}

}  // namespace am
