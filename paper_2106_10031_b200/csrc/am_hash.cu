// am_hash.cu -- on-device open-addressing set of activation states.
//
// Replaces the reference's shared Python set `seen` (reference marching.py:221,
// 235-245).  Slots are 64-bit words  fp(31) | cand(1) | ref(32):
//   cand = 1 : ref indexes the key buffer of the insert launch in flight
//   cand = 0 : ref indexes the key pool
// Insertion is lock-free: a thread claims an empty slot with one CAS carrying a
// reference to its own (already written) key, so concurrent duplicates resolve
// by key comparison without any second round; a fix-up launch then moves the
// winners' keys into the pool and rewrites their slots to pool references.
#include "am_internal.h"

namespace am {

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) { return *reinterpret_cast<const volatile uint64_t*>(p); }

__device__ __forceinline__ bool keys_equal(const uint64_t* a, const uint64_t* b, int kw) {
    for (int i = 0; i < kw; i++)
        if (a[i] != b[i]) return false;
    return true;
}

__global__ void k_hash_insert(HashSet H, const uint64_t* src, const int32_t* idx, int64_t n, int32_t* status,
                              uint64_t* slot_out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t ci = idx ? idx[i] : i;
    const uint64_t* key = src + ci * H.KW;
    uint64_t h = key_hash(key, H.KW);
    uint64_t fp = h >> 33;
    uint64_t pos = h & H.mask;
    const uint64_t mine = (fp << 33) | (1ull << 32) | (uint64_t)(uint32_t)i;
    for (uint64_t probe = 0; probe <= H.mask; probe++) {
        uint64_t v = ld_volatile(H.table + pos);
        if (v == kEmpty) {
            unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(H.table + pos),
                                               (unsigned long long)kEmpty, (unsigned long long)mine);
            if (old == kEmpty) {
                status[i] = 1;
                slot_out[i] = pos;
                return;
            }
            v = old;
        }
        if ((v >> 33) == fp) {
            uint32_t ref = (uint32_t)v;
            const uint64_t* other = ((v >> 32) & 1ull) ? src + (int64_t)(idx ? idx[ref] : (int64_t)ref) * H.KW
                                                       : H.pool + (int64_t)ref * H.KW;
            if (keys_equal(key, other, H.KW)) {
                status[i] = 0;
                return;
            }
        }
        pos = (pos + 1) & H.mask;
    }
    status[i] = -1;  // table full (host keeps load factor <= 1/2, so unreachable)
}

__global__ void k_hash_fixup(HashSet H, const uint64_t* src, const int32_t* idx, int64_t n, const int32_t* status,
                             const uint64_t* slot, uint32_t flag, int32_t* pool_idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (status[i] != 1) {
        if (pool_idx) pool_idx[i] = -1;
        return;
    }
    const int64_t ci = idx ? idx[i] : i;
    const uint64_t* key = src + ci * H.KW;
    unsigned long long p = atomicAdd(H.n_pool, 1ull);
    if ((int64_t)p >= H.cap_pool) {  // host guarantees capacity; keep the slot valid regardless
        if (pool_idx) pool_idx[i] = -1;
        return;
    }
    uint64_t* dst = H.pool + (int64_t)p * H.KW;
    for (int w = 0; w < H.KW; w++) dst[w] = key[w];
    H.pool_flags[p] = flag;
    uint64_t fp = key_hash(key, H.KW) >> 33;
    __threadfence();
    H.table[slot[i]] = (fp << 33) | (uint64_t)(uint32_t)p;
    if (pool_idx) pool_idx[i] = (int32_t)p;
}

__global__ void k_hash_lookup(HashSet H, const uint64_t* src, int64_t n, int32_t* found) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t* key = src + i * H.KW;
    uint64_t h = key_hash(key, H.KW);
    uint64_t fp = h >> 33;
    uint64_t pos = h & H.mask;
    for (uint64_t probe = 0; probe <= H.mask; probe++) {
        uint64_t v = H.table[pos];
        if (v == kEmpty) break;
        if ((v >> 33) == fp && !((v >> 32) & 1ull) && keys_equal(key, H.pool + (int64_t)(uint32_t)v * H.KW, H.KW)) {
            found[i] = (int32_t)(uint32_t)v;
            return;
        }
        pos = (pos + 1) & H.mask;
    }
    found[i] = -1;
}

// rebuild the slot array from the pool (table growth)
__global__ void k_hash_rebuild(HashSet H, int64_t n_pool) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n_pool) return;
    const uint64_t* key = H.pool + p * H.KW;
    uint64_t h = key_hash(key, H.KW);
    uint64_t v = ((h >> 33) << 33) | (uint64_t)(uint32_t)p;
    uint64_t pos = h & H.mask;
    for (;;) {
        unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(H.table + pos),
                                           (unsigned long long)kEmpty, (unsigned long long)v);
        if (old == kEmpty) return;
        pos = (pos + 1) & H.mask;
    }
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

void launch_hash_insert(const HashSet& H, const uint64_t* src, const int32_t* idx, int64_t n, int32_t* status,
                        uint64_t* slot, cudaStream_t s) {
    if (n > 0) { k_hash_insert<<<nblk(n, 256), 256, 0, s>>>(H, src, idx, n, status, slot); ++g_launch_count; }
}
void launch_hash_fixup(const HashSet& H, const uint64_t* src, const int32_t* idx, int64_t n, const int32_t* status,
                       const uint64_t* slot, uint32_t flag, int32_t* pool_idx, cudaStream_t s) {
    if (n > 0) { k_hash_fixup<<<nblk(n, 256), 256, 0, s>>>(H, src, idx, n, status, slot, flag, pool_idx); ++g_launch_count; }
}
void launch_hash_lookup(const HashSet& H, const uint64_t* src, int64_t n, int32_t* found, cudaStream_t s) {
    if (n > 0) { k_hash_lookup<<<nblk(n, 256), 256, 0, s>>>(H, src, n, found); ++g_launch_count; }
}
void launch_hash_rebuild(const HashSet& H, int64_t n_pool, cudaStream_t s) {
    if (n_pool > 0) { k_hash_rebuild<<<nblk(n_pool, 256), 256, 0, s>>>(H, n_pool); ++g_launch_count; }
}

// ------------------------------------------------------------ list utilities
// append i to out (via counter) where flag[i] == want; order within a block is ascending
__global__ void k_compact(const int32_t* flag, int32_t want, int64_t n, int32_t* out, unsigned long long* count) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool take = i < n && flag[i] == want;
    unsigned mask = __ballot_sync(0xffffffffu, take);
    int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0 && mask) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (take) out[base + __popc(mask & ((1u << lane) - 1u))] = (int32_t)i;
}
void launch_compact(const int32_t* flag, int32_t want, int64_t n, int32_t* out, unsigned long long* count,
                    cudaStream_t s) {
    if (n > 0) { k_compact<<<nblk(n, 256), 256, 0, s>>>(flag, want, n, out, count); ++g_launch_count; }
}

// dst[i] = src[idx[i]] (KW words each)
__global__ void k_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t i = t / KW;
    int w = (int)(t - i * KW);
    if (i >= n) return;
    dst[i * KW + w] = src[(int64_t)idx[i] * KW + w];
}
void launch_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst, cudaStream_t s) {
    if (n > 0) { k_gather_keys<<<nblk(n * KW, 256), 256, 0, s>>>(src, idx, n, KW, dst); ++g_launch_count; }
}

// frontier assembly after composition (reference marching.py:280-288: canon == state -> skip;
// canon new -> enqueue).  Raw winners whose canonical key equals the raw key are new cells;
// changed ones are new cells only if their canonical insert won.
__global__ void k_frontier(int64_t nR, const int32_t* changed, const int32_t* R, const int32_t* raw_pool,
                           const int32_t* canon_pos, const int32_t* canon_status, const int32_t* canon_pool,
                           uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool, unsigned long long* nF,
                           int64_t max_new, unsigned long long* capped) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nR) return;
    int32_t p = -1;
    if (!changed[b]) {
        p = raw_pool[R[b]];
    } else {
        int32_t j = canon_pos[b];
        if (j >= 0 && canon_status[j] == 1) p = canon_pool[j];
    }
    if (p < 0) return;
    unsigned long long k = atomicAdd(nF, 1ull);
    if ((int64_t)k >= max_new) {  // max_cells cap (reference marching.py:240-242)
        atomicAdd(capped, 1ull);
        return;
    }
    pool_flags[p] |= 1u;
    f_items[k] = (int32_t)b;
    f_pool[k] = p;
}
void launch_frontier(int64_t nR, const int32_t* changed, const int32_t* R, const int32_t* raw_pool,
                     const int32_t* canon_pos, const int32_t* canon_status, const int32_t* canon_pool,
                     uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool, unsigned long long* nF, int64_t max_new,
                     unsigned long long* capped, cudaStream_t s) {
    if (nR > 0)
        { k_frontier<<<nblk(nR, 256), 256, 0, s>>>(nR, changed, R, raw_pool, canon_pos, canon_status, canon_pool,
                                                   pool_flags, f_items, f_pool, nF, max_new, capped); ++g_launch_count; }
}

// canon_pos[b] = position of b in the changed list X (or -1)
__global__ void k_scatter_pos(const int32_t* X, int64_t nX, int32_t* pos) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nX) pos[X[j]] = (int32_t)j;
}
void launch_scatter_pos(const int32_t* X, int64_t nX, int32_t* pos, cudaStream_t s) {
    if (nX > 0) { k_scatter_pos<<<nblk(nX, 256), 256, 0, s>>>(X, nX, pos); ++g_launch_count; }
}

// owner partition for sharded marching: out_owner[i] = owner(key_i)
__global__ void k_owner(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) owner[i] = key_owner(keys + i * KW, KW, world);
}
void launch_owner(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner, cudaStream_t s) {
    if (n > 0) { k_owner<<<nblk(n, 256), 256, 0, s>>>(keys, n, KW, world, owner); ++g_launch_count; }
}

}  // namespace am
