// am_hash.cu -- on-device open-addressing set of activation states + the work queue.
//
// Replaces the reference's shared Python set `seen` and deque (reference
// marching.py:221-245).  Slots are 64-bit words  fp(31) | cand(1) | ref(32):
//   cand = 1 : ref indexes the key buffer of the insert launch in flight
//   cand = 0 : ref indexes the key pool
// Insertion is lock-free and takes one launch (k_hash_upsert): a thread claims an
// empty slot with one CAS carrying a candidate marker (its batch index), so
// concurrent inserters of the same key resolve by comparing against the claimant's
// batch copy; the claiming thread itself appends the key to the pool, rewrites the
// slot to the pool reference and queues the new state.  Every launch reads its item
// count from device memory, so a whole BFS iteration is one capturable CUDA graph.
#include <cstdlib>

#include "am_internal.h"
#include "am_hashset.cuh"

namespace am {

__global__ void k_hash_upsert(HashSet H, const uint64_t* src, const int32_t* idx, const unsigned long long* n_dev,
                              int64_t n_cap, int32_t* status, uint64_t* slot_out, int32_t* dup_ref, uint32_t flag,
                              int32_t* pool_idx, int32_t* queue, unsigned long long* q_tail, const double* src_hint,
                              const int64_t* src_par) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    GRID_STRIDE(i, n) {
        const int64_t ci = idx ? idx[i] : i;
        int32_t p;
        status[ci] = upsert_one(H, src, idx, i, ci, slot_out, dup_ref, flag, queue, q_tail, src_hint, &p, src_par);
        if (pool_idx) pool_idx[ci] = p;
    }
}

// rebuild the slot array from the pool (table growth)
__global__ void k_hash_rebuild(HashSet H, int64_t n_pool) {
    pdl_enter();
    GRID_STRIDE(p, n_pool) {
        const uint64_t* key = H.pool + p * H.KW;
        uint64_t h = key_hash(key, H.KW);
        uint64_t v = ((h >> 33) << 33) | (uint64_t)(uint32_t)p;
        uint64_t pos = h & H.mask;
        for (;;) {
            unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(H.table + pos),
                                               (unsigned long long)kEmpty, (unsigned long long)v);
            if (old == kEmpty) break;
            pos = (pos + 1) & H.mask;
        }
    }
}

static int grid_mult() {
    static int m = 0;
    if (!m) {
        const char* v = getenv("AM_GRID_MULT");
        // A/B on configs[1]: 8 -> 21.35 ms, 4 -> 20.8, 2 -> 20.5, 1 -> 20.4 (round 2, early); at the
        // end of round 2: 2 -> 17.72, 1 -> 17.53 (DeepSDF first 1 M cells 444.8 -> 436.9 ms)
        m = v ? std::max(1, atoi(v)) : 1;
    }
    return m;
}
static unsigned grid_for(int64_t n, int b) {
    int64_t blocks = (n + b - 1) / b;
    int64_t cap = (int64_t)device_sms() * grid_mult();
    return (unsigned)(blocks < 1 ? 1 : (blocks < cap ? blocks : cap));
}

void launch_hash_upsert(const HashSet& H, const uint64_t* src, const int32_t* idx, const unsigned long long* n_dev,
                        int64_t n_cap, int32_t* status, uint64_t* slot, int32_t* dup_ref, uint32_t flag,
                        int32_t* pool_idx, int32_t* queue, unsigned long long* q_tail, const double* src_hint,
                        cudaStream_t s, const int64_t* src_par) {
    if (n_cap > 0) {
        launch_k(k_hash_upsert, grid_for(n_cap, 256), 256, 0, s, H, src, idx, n_dev, n_cap, status, slot, dup_ref, flag,
                 pool_idx, queue, q_tail, src_hint, src_par);
    }
}
void launch_hash_rebuild(const HashSet& H, int64_t n_pool, cudaStream_t s) {
    if (n_pool > 0) { launch_k(k_hash_rebuild, grid_for(n_pool, 256), 256, 0, s, H, n_pool); }
}

// ------------------------------------------------------------- iteration
// take up to B queued states for this iteration, after checking that the
// worst case of what the iteration can produce fits every buffer.
__global__ void k_take(IterState I) {
    pdl_enter();
    unsigned long long* c = I.ctr;
    __shared__ long long s_n;
    __shared__ unsigned long long s_iter;
    __shared__ unsigned s_cnt[kMaxPrefixBuckets];
    if (threadIdx.x < kMaxPrefixBuckets) s_cnt[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        long long head = (long long)c[C_QHEAD], tail = (long long)c[C_QTAIL];
        long long want = tail - head;
        if (want > I.B) want = I.B;
        long long np = (long long)c[C_POOL];
        long long nR = want;
        // new pool entries: each batch item + everything its face can emit
        long long room_pool = (I.cap_pool - np) / (1 + I.emit_per_cell);
        long long room_tab = ((long long)(I.tcap / 2) - np) / (1 + I.emit_per_cell);
        long long room_cells = I.cap_cells - (long long)c[C_CELLS];
        long long room_verts = (I.cap_verts - (long long)c[C_VERTS]) / I.verts_per_cell;
        long long room_refs = (I.cap_refs - (long long)c[C_REFS]) / I.refs_per_cell;
        long long room_pend = (I.cap_pend - (long long)c[C_NPEND]) / I.verts_per_cell;
        long long room_val = (I.cap_val - (long long)c[C_NVAL]) / I.verts_per_cell;
        long long room_out = I.cap_outbox - (long long)c[C_NOUT];
        if (I.world > 1) room_out /= (1 + I.emit_per_cell);
        else room_out = nR;
        long long lim = room_pool;
        if (room_tab < lim) lim = room_tab;
        if (room_cells < lim) lim = room_cells;
        if (room_verts < lim) lim = room_verts;
        if (room_refs < lim) lim = room_refs;
        if (room_out < lim) lim = room_out;
        if (room_pend < lim) lim = room_pend;
        if (room_val < lim) lim = room_val;
        if (lim < 0) lim = 0;
        if (nR > lim) nR = lim;
        // max_cells (reference marching.py:240-242 ends the walk there): a batch item becomes at
        // most one visited cell, so no more than the remaining allowance is composed; once it is
        // used up and no cell can be waiting for a deferred face, the queue, the pending probe
        // records and the queued probe evaluations are dropped instead of composed and discarded
        bool drop = false;
        const long long rem = I.max_cells - (long long)c[C_TOTAL];
        if (rem <= 0 && I.cap_drop) {
            drop = want > 0 || c[C_NPEND] || c[C_NPROBE];
            nR = 0;
        } else if (rem > 0 && nR > rem) {
            nR = rem;
        }
        c[C_STALL] = (!drop && want > 0 && nR == 0) ? 1ull : 0ull;
        c[C_NR] = (unsigned long long)nR;
        // C_NPROBE is not reset: exact probe evaluations accumulate across iterations and are
        // flushed by the host loop (probe_flush) outside the per-iteration graph
        c[C_NX] = 0; c[C_NF] = 0; c[C_NEMIT] = 0; c[C_NLOCAL] = 0;
        c[C_NPREC] = 0; c[C_NKEEP] = 0; c[C_NPLOCAL] = 0; c[C_FCURSOR] = 0;
        c[C_NHEAVY] = 0; c[C_NLIGHT] = 0;
        c[C_ITER] += nR > 0 ? 1ull : 0ull;
        // the batch: queue[head, head + a) + queue[tail - t, tail) (batch_queue_index); prefix
        // reuse takes the entries queued since the previous take (children of its batch) from the
        // tail first, FIFO otherwise
        long long t = 0;
        if (I.queue_par) {
            t = tail - (long long)c[C_QMARK];
            if (t < 0) t = 0;
            if (t > nR) t = nR;
        }
        const long long a = nR - t;
        c[C_QA] = (unsigned long long)a;
        c[C_QB] = (unsigned long long)(tail - t);
        c[C_QHEAD] = (unsigned long long)(head + a);
        c[C_QTAIL] = (unsigned long long)(tail - t);
        c[C_QMARK] = (unsigned long long)(tail - t);
        if (drop) {
            c[C_CAPPED] += (unsigned long long)(want > 0 ? want : 1);
            c[C_QHEAD] = (unsigned long long)tail;
            c[C_QMARK] = (unsigned long long)tail;
            c[C_NPEND] = 0;
            c[C_NPROBE] = 0;
        }
        s_n = nR;
        s_iter = c[C_ITER];
    }
    if (!I.queue_par) return;
    // prefix reuse: bucket the batch by the number of composition steps its cells can take from
    // their parents (emitted in the previous iteration; anything else composes in full)
    __syncthreads();
    const long long n = s_n;
    const unsigned long long it = s_iter;
    const long long qa = (long long)c[C_QA], q0 = (long long)c[C_QHEAD] - qa, qb = (long long)c[C_QB];
    const int lane = threadIdx.x & 31;
    for (long long b0 = threadIdx.x - lane; b0 < n; b0 += blockDim.x) {   // warp-uniform trip count
        const long long b = b0 + lane;
        int f = -1;
        if (b < n) {
            const long long w = I.queue_par[b < qa ? q0 + b : qb + (b - qa)];
            f = 0;
            if (w != 0 && ((unsigned long long)w >> 32) + 1ull == it) {
                f = (int)(w & 31);
                if (f > I.max_share) f = I.max_share;
            }
        }
        // one shared-memory atomic per distinct bucket of the warp
        const unsigned peers = __match_any_sync(0xffffffffu, f);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (lane == leader && f >= 0) base = atomicAdd(&s_cnt[f], (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (f >= 0) I.blist[(long long)f * I.B + base + __popc(peers & ((1u << lane) - 1u))] = (int32_t)b;
    }
    __syncthreads();
    if (threadIdx.x < kMaxPrefixBuckets) {
        c[C_BK0 + threadIdx.x] = s_cnt[threadIdx.x];
        c[C_BKT0 + threadIdx.x] += s_cnt[threadIdx.x];
        unsigned long long pre = 0;   // items of buckets below this one
        for (int f = 0; f < (int)threadIdx.x; f++) pre += s_cnt[f];
        c[C_PRE0 + threadIdx.x] = pre;
    }
}

// batch_pool[b] = queue[batch_queue_index(b)] (the batch k_take dequeued), ckey[b] = pool[batch_pool[b]];
// reset per-item flags
__global__ void k_gather_batch(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                               const unsigned long long* ctr, int32_t* batch_pool, int64_t n_cap, int KW,
                               uint64_t* ckey, double* ckey_hint, int32_t* changed, int32_t* canon_pos) {
    pdl_enter();
    const int64_t n = dev_count(ctr + C_NR, n_cap);
    GRID_STRIDE(t, n * KW) {
        int64_t b = t / KW;
        int w = (int)(t - b * KW);
        const int32_t p = queue[batch_queue_index(ctr, b)];
        ckey[t] = pool[(int64_t)p * KW + w];
        if (w == 0) {
            batch_pool[b] = p;
            changed[b] = 0;
            canon_pos[b] = -1;
            reinterpret_cast<double4*>(ckey_hint)[b] = reinterpret_cast<const double4*>(pool_hint)[p];
        }
    }
}

// changed items: local canonical states -> X (canonical insert), remote-owned -> outbox
__global__ void k_route_changed(const uint64_t* ckey, const int32_t* changed, const unsigned long long* n_dev,
                                int64_t n_cap, int KW, int rank, int world, int32_t* X, unsigned long long* nX,
                                uint64_t* outbox, unsigned long long* n_out, int32_t* canon_pos) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    GRID_STRIDE(b, n) {
        if (!changed[b]) continue;
        const uint64_t* k = ckey + b * KW;
        if (world > 1 && key_owner(k, KW, world) != rank) {
            unsigned long long o = atomicAdd(n_out, 1ull);
            for (int w = 0; w < KW; w++) outbox[o * KW + w] = k[w];
            canon_pos[b] = -2;   // handled by its owner
            continue;
        }
        unsigned long long j = atomicAdd(nX, 1ull);
        X[j] = (int32_t)b;
        canon_pos[b] = 1;   // canonical insert result lands in status2[b] / canon_pool[b]
    }
}

// frontier assembly after composition (reference marching.py:280-288: canon == state -> skip;
// canon new -> enqueue).  Batch items whose canonical key equals the raw key are new cells
// (they won the raw insert); changed ones are new cells only if their canonical insert won.
__global__ void k_frontier(const unsigned long long* n_dev, int64_t n_cap, const int32_t* changed,
                           const int32_t* batch_pool, const int32_t* canon_pos, const int32_t* canon_status,
                           const int32_t* canon_pool, uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool,
                           unsigned long long* ctr, long long max_cells) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    GRID_STRIDE(b, n) {
        int32_t p = -1;
        const uint32_t fl = pool_flags[batch_pool[b]];
        pool_flags[batch_pool[b]] = (fl | 2u) & ~kPoolDeferred;   // composed (probe records can resolve)
        if (fl & kPoolDeferred) {   // a deferred cell solved again: visited and counted already
            const unsigned long long kf = atomicAdd(ctr + C_NF, 1ull);
            f_items[kf] = (int32_t)b;
            f_pool[kf] = batch_pool[b];
            continue;
        }
        if (!changed[b]) {
            p = batch_pool[b];
        } else if (canon_pos[b] == 1 && canon_status[b] == 1) {
            p = canon_pool[b];
        }
        if (p < 0) continue;
        unsigned long long tot = atomicAdd(ctr + C_TOTAL, 1ull);
        if ((long long)tot >= max_cells) {  // max_cells cap (reference marching.py:240-242)
            atomicAdd(ctr + C_CAPPED, 1ull);
            continue;
        }
        unsigned long long k = atomicAdd(ctr + C_NF, 1ull);
        pool_flags[p] |= 1u;
        f_items[k] = (int32_t)b;
        f_pool[k] = p;
    }
}

// k_route_changed + the canonical k_hash_upsert + k_frontier in one launch: every batch item
// decides its own frontier entry from its own canonical insert, so no grid-wide step separates
// them (reference marching.py:280-288: canon == state -> the cell itself; canon new -> a new cell;
// canon already present -> nothing).  Multi-rank: canonical keys owned elsewhere go to the outbox.
__global__ void k_canon_frontier(HashSet H, const uint64_t* ckey, const int32_t* changed, const int32_t* batch_pool,
                                 const unsigned long long* n_dev, int64_t n_cap, int rank, int world,
                                 uint64_t* outbox, unsigned long long* n_out, int32_t* canon_pos, int32_t* status2,
                                 uint64_t* slot2, int32_t* canon_pool, const double* ckey_hint, int32_t* f_items,
                                 int32_t* f_pool, unsigned long long* ctr, long long max_cells) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    GRID_STRIDE(b, n) canon_frontier_one(H, ckey, changed[b], batch_pool[b], b, rank, world, outbox, n_out, canon_pos,
                                         status2, slot2, canon_pool, ckey_hint, f_items, f_pool, ctr, max_cells);
}

void launch_canon_frontier(const HashSet& H, const uint64_t* ckey, const int32_t* changed, const int32_t* batch_pool,
                           const unsigned long long* n_dev, int64_t n_cap, int rank, int world, uint64_t* outbox,
                           unsigned long long* n_out, int32_t* canon_pos, int32_t* status2, uint64_t* slot2,
                           int32_t* canon_pool, const double* ckey_hint, int32_t* f_items, int32_t* f_pool,
                           unsigned long long* ctr, long long max_cells, cudaStream_t s) {
    launch_k(k_canon_frontier, grid_for(n_cap, 256), 256, 0, s, H, ckey, changed, batch_pool, n_dev, n_cap, rank,
             world, outbox, n_out, canon_pos, status2, slot2, canon_pool, ckey_hint, f_items, f_pool, ctr, max_cells);
}

// zero the key slots the probe forward pass ORs its bits into
__global__ void k_zero_probe_keys(uint64_t* scratch, const unsigned long long* ctr, int KW) {
    pdl_enter();
    const int64_t base = (int64_t)ctr[C_NEMIT] * KW;
    const int64_t n = (int64_t)ctr[C_NPROBE] * KW;
    GRID_STRIDE(i, n) scratch[base + i] = 0;
}

// probes were appended after the flips: total emitted = flips + probes
__global__ void k_emit_finalize(unsigned long long* ctr) {
    pdl_enter();
    if (threadIdx.x == 0 && blockIdx.x == 0) ctr[C_NEMIT] += ctr[C_NPROBE];
}

// sharded march: emitted states owned elsewhere -> outbox; local ones -> index list
__global__ void k_route_emitted(const uint64_t* scratch, const unsigned long long* ctr_n, int64_t n_cap, int KW,
                                int rank, int world, int32_t* local_idx, unsigned long long* n_local,
                                uint64_t* outbox, unsigned long long* n_out, int32_t* remote_status) {
    pdl_enter();
    const int64_t n = dev_count(ctr_n, n_cap);
    GRID_STRIDE(i, n) {
        const uint64_t* k = scratch + i * KW;
        if (key_owner(k, KW, world) == rank) {
            local_idx[atomicAdd(n_local, 1ull)] = (int32_t)i;
        } else {
            if (remote_status) remote_status[i] = -5;   // owned elsewhere: probe records on it forward
            unsigned long long o = atomicAdd(n_out, 1ull);
            for (int w = 0; w < KW; w++) outbox[o * KW + w] = k[w];
        }
    }
}

void launch_take(const IterState& I, cudaStream_t s) {
    static int nt = 0;   // bucketing threads (AM_TAKE_THREADS)
    if (!nt) {
        const char* v = getenv("AM_TAKE_THREADS");
        nt = v ? std::max(32, std::min(1024, atoi(v) / 32 * 32)) : 1024;
    }
    launch_k(k_take, 1, I.queue_par ? nt : 32, 0, s, I);
}
void launch_gather_batch(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                         const unsigned long long* ctr, int32_t* batch_pool, int64_t n_cap, int KW, uint64_t* ckey,
                         double* ckey_hint, int32_t* changed, int32_t* canon_pos, cudaStream_t s) {
    launch_k(k_gather_batch, grid_for(n_cap * KW, 256), 256, 0, s, pool, pool_hint, queue, ctr, batch_pool, n_cap, KW,
             ckey, ckey_hint, changed, canon_pos);
}
void launch_route_changed(const uint64_t* ckey, const int32_t* changed, const unsigned long long* n_dev, int64_t n_cap,
                          int KW, int rank, int world, int32_t* X, unsigned long long* nX, uint64_t* outbox,
                          unsigned long long* n_out, int32_t* canon_pos, cudaStream_t s) {
    launch_k(k_route_changed, grid_for(n_cap, 256),  256,  0,  s, ckey, changed, n_dev, n_cap, KW, rank, world, X, nX, outbox,
                                                          n_out, canon_pos);
}
void launch_frontier(const unsigned long long* n_dev, int64_t n_cap, const int32_t* changed, const int32_t* batch_pool,
                     const int32_t* canon_pos, const int32_t* canon_status, const int32_t* canon_pool,
                     uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool, unsigned long long* ctr,
                     long long max_cells, cudaStream_t s) {
    launch_k(k_frontier, grid_for(n_cap, 256),  256,  0,  s, n_dev, n_cap, changed, batch_pool, canon_pos, canon_status,
                                                     canon_pool, pool_flags, f_items, f_pool, ctr, max_cells);
}
void launch_zero_probe_keys(uint64_t* scratch, const unsigned long long* ctr, int KW, int64_t cap, cudaStream_t s) {
    launch_k(k_zero_probe_keys, grid_for(cap * KW, 256),  256,  0,  s, scratch, ctr, KW);
}
void launch_emit_finalize(unsigned long long* ctr, cudaStream_t s) { launch_k(k_emit_finalize, 1, 32, 0, s, ctr); }
void launch_route_emitted(const uint64_t* scratch, const unsigned long long* ctr_n, int64_t n_cap, int KW, int rank,
                          int world, int32_t* local_idx, unsigned long long* n_local, uint64_t* outbox,
                          unsigned long long* n_out, int32_t* remote_status, cudaStream_t s) {
    launch_k(k_route_emitted, grid_for(n_cap, 256),  256,  0,  s, scratch, ctr_n, n_cap, KW, rank, world, local_idx, n_local,
                                                          outbox, n_out, remote_status);
}

// dst[i] = src[idx[i]] (KW words each), host-sized
__global__ void k_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst) {
    pdl_enter();
    GRID_STRIDE(t, n * KW) {
        int64_t i = t / KW;
        int w = (int)(t - i * KW);
        dst[t] = src[(int64_t)idx[i] * KW + w];
    }
}
void launch_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst, cudaStream_t s) {
    if (n > 0) { launch_k(k_gather_keys, grid_for(n * KW, 256), 256, 0, s, src, idx, n, KW, dst); }
}

// open-edge count (edges with a box plane among their transition refs)
__global__ void k_open_edges(const int32_t* enr, const int64_t* roff, const int32_t* refs, int64_t nv, int box0,
                             unsigned long long* out) {
    pdl_enter();
    GRID_STRIDE(v, nv) {
        bool hit = false;
        for (int q = 0; q < enr[v]; q++) hit |= refs[roff[v] + q] >= box0;
        if (hit) atomicAdd(out, 1ull);
    }
}
void launch_open_edges(const int32_t* enr, const int64_t* roff, const int32_t* refs, int64_t nv, int box0,
                       unsigned long long* out, cudaStream_t s) {
    if (nv > 0) { launch_k(k_open_edges, grid_for(nv, 256), 256, 0, s, enr, roff, refs, nv, box0, out); }
}

// ------------------------------------------------------- probe records
// resolve the target pool entry of this iteration's new probe records and append them to the
// pending list (targets owned by another rank cannot be checked here: forward them)
__global__ void k_prec_target(ProbeRecs R, const int32_t* status, const int32_t* dup_ref, const int32_t* pool_idx,
                              unsigned long long* ctr, int64_t cap, double* probe_pts, int64_t cap_probe) {
    pdl_enter();
    const int64_t n = dev_count(ctr + C_NPREC, cap);
    const int par = (int)(ctr[C_PPAR] & 1ull);
    GRID_STRIDE(i, n) {
        const int32_t ci = R.cand[i];
        int32_t t = -1;   // -1: exact forward evaluation (no flip target, or owned by another rank)
        if (ci >= 0) {
            const int32_t st = status[ci];
            if (st == 1) t = pool_idx[ci];
            else if (st == 0) t = dup_ref[ci] >= 0 ? dup_ref[ci] : pool_idx[-2 - dup_ref[ci]];
        }
        unsigned long long j = atomicAdd(ctr + C_NPEND, 1ull);
        if ((int64_t)j >= R.cap_pend) { atomicAdd(ctr + C_OVF1, 1ull); continue; }
        R.pend_t[par][j] = t;
        R.pend_k[par][j] = R.k[i];
        R.pend_pt[par][j * 3 + 0] = R.pt[i * 3 + 0];
        R.pend_pt[par][j * 3 + 1] = R.pt[i * 3 + 1];
        R.pend_pt[par][j * 3 + 2] = R.pt[i * 3 + 2];
        if (R.s) R.pend_s[par][j] = R.s[i];
    }
}

// pending probe records whose target has been processed: dropped if the target validated the
// mirrored probe of that neuron (the probe provably lands in the target cell), otherwise
// forward-evaluated; targets still queued keep the record for a later iteration
__global__ void k_resolve(ProbeRecs R, HashSet H, const int32_t* val_buf, unsigned long long* ctr, int64_t cap,
                          double* probe_pts, int32_t* probe_shape, int64_t cap_probe) {
    pdl_enter();
    const int64_t n = dev_count(ctr + C_NPEND, cap);
    const int par = (int)(ctr[C_PPAR] & 1ull);
    GRID_STRIDE(i, n) {
        const int32_t t = R.pend_t[par][i];
        bool forward = false, keep = false;
        if (t < 0) {
            forward = true;
        } else {
            const int32_t vn = H.pool_vn[t];
            if (vn >= 0) {
                const int32_t k = R.pend_k[par][i];
                const int64_t off = H.pool_voff[t];
                bool found = false;
                for (int q = 0; q < vn; q++) found |= val_buf[off + q] == k;
                forward = !found;
            } else if (H.pool_flags[t] & 2u) {
                forward = true;   // composed but no face (canonical elsewhere / capped): exact evaluation
            } else {
                keep = true;      // target still queued
            }
        }
        if (forward) {
            unsigned long long q = atomicAdd(ctr + C_NPROBE, 1ull);
            if ((int64_t)q < cap_probe) {
                probe_pts[q * 3 + 0] = R.pend_pt[par][i * 3 + 0]; probe_pts[q * 3 + 1] = R.pend_pt[par][i * 3 + 1];
                probe_pts[q * 3 + 2] = R.pend_pt[par][i * 3 + 2];
                if (R.s) probe_shape[q] = R.pend_s[par][i];
            } else {
                keep = true;      // forward buffer full this iteration: retry next iteration
            }
        }
        if (keep) {
            unsigned long long j = atomicAdd(ctr + C_NKEEP, 1ull);
            R.pend_t[par ^ 1][j] = t;
            R.pend_k[par ^ 1][j] = R.pend_k[par][i];
            R.pend_pt[par ^ 1][j * 3 + 0] = R.pend_pt[par][i * 3 + 0];
            R.pend_pt[par ^ 1][j * 3 + 1] = R.pend_pt[par][i * 3 + 1];
            R.pend_pt[par ^ 1][j * 3 + 2] = R.pend_pt[par][i * 3 + 2];
            if (R.s) R.pend_s[par ^ 1][j] = R.pend_s[par][i];
        }
    }
}

// (has_cond: also set the iteration graph's conditional probe stage: any probe to evaluate?)
// Probe records of one iteration in one launch (k_prec_target + k_resolve + k_pend_finalize):
// work item i < n_new is this iteration's record i (its target is resolved from the emitted
// candidate's insert status), i >= n_new the pending record i - n_new of earlier iterations.
// Either is dropped (the target validated the mirrored probe), queued for exact evaluation, or
// kept pending (target not composed yet) in the other parity's list.  The last CTA to finish
// updates the counters and, inside the captured graph, sets the probe stage's predicate.
__device__ __forceinline__ void probe_decide(const ProbeRecs& R, const HashSet& H, const int32_t* val_buf,
                                             unsigned long long* ctr, int32_t t, int32_t k, const double* pt,
                                             int32_t shp, double* probe_pts, int32_t* probe_shape,
                                             int64_t cap_probe, int par) {
    bool forward = false, keep = false;
    if (t < 0) {
        forward = true;
    } else {
        const int32_t vn = H.pool_vn[t];
        if (vn >= 0) {
            const int64_t off = H.pool_voff[t];
            bool found = false;
            for (int q = 0; q < vn; q++) found |= val_buf[off + q] == k;
            forward = !found;
        } else if ((H.pool_flags[t] & 2u) && !(H.pool_flags[t] & kPoolDeferred)) {
            forward = true;   // composed but no face (canonical elsewhere / capped): exact evaluation
        } else {
            keep = true;      // target still queued (or deferred: it is solved in a later iteration)
        }
    }
    if (forward) {
        const unsigned long long q = atomicAdd(ctr + C_NPROBE, 1ull);
        if ((int64_t)q < cap_probe) {
            probe_pts[q * 3 + 0] = pt[0]; probe_pts[q * 3 + 1] = pt[1]; probe_pts[q * 3 + 2] = pt[2];
            if (R.s) probe_shape[q] = shp;
        } else {
            keep = true;      // forward buffer full: retry next iteration
        }
    }
    if (keep) {
        const unsigned long long j = atomicAdd(ctr + C_NKEEP, 1ull);
        if ((int64_t)j >= R.cap_pend) { atomicAdd(ctr + C_OVF1, 1ull); return; }
        R.pend_t[par ^ 1][j] = t;
        R.pend_k[par ^ 1][j] = k;
        R.pend_pt[par ^ 1][j * 3 + 0] = pt[0];
        R.pend_pt[par ^ 1][j * 3 + 1] = pt[1];
        R.pend_pt[par ^ 1][j * 3 + 2] = pt[2];
        if (R.s) R.pend_s[par ^ 1][j] = shp;
    }
}

__global__ void k_probe_records(ProbeRecs R, HashSet H, const int32_t* status, const int32_t* dup_ref,
                                const int32_t* pool_idx, const int32_t* val_buf, unsigned long long* ctr,
                                int64_t cap_new, double* probe_pts, int32_t* probe_shape, int64_t cap_probe,
                                cudaGraphConditionalHandle h, int has_cond) {
    pdl_enter();
    const int64_t n_new = dev_count(ctr + C_NPREC, cap_new);
    const int64_t n_old = dev_count(ctr + C_NPEND, R.cap_pend);
    const int par = (int)(ctr[C_PPAR] & 1ull);
    GRID_STRIDE(i, n_new + n_old) {
        if (i < n_new) {
            const int32_t ci = R.cand[i];
            int32_t t = -1;   // -1: exact forward evaluation (no flip target, or owned by another rank)
            if (ci >= 0) {
                const int32_t st = status[ci];
                if (st == 1) t = pool_idx[ci];
                else if (st == 0) t = dup_ref[ci] >= 0 ? dup_ref[ci] : pool_idx[-2 - dup_ref[ci]];
            }
            probe_decide(R, H, val_buf, ctr, t, R.k[i], R.pt + i * 3, R.s ? R.s[i] : 0, probe_pts, probe_shape,
                         cap_probe, par);
        } else {
            const int64_t j = i - n_new;
            probe_decide(R, H, val_buf, ctr, R.pend_t[par][j], R.pend_k[par][j], R.pend_pt[par] + j * 3,
                         R.s ? R.pend_s[par][j] : 0, probe_pts, probe_shape, cap_probe, par);
        }
    }
    // the last CTA to finish publishes the counters
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctr + C_DONE, 1ull) == (unsigned long long)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        volatile unsigned long long* vc = ctr;
        if (has_cond) cudaGraphSetConditional(h, vc[C_NPROBE] ? 1u : 0u);
        vc[C_PREC_TOTAL] = vc[C_PREC_TOTAL] + vc[C_NPREC];
        vc[C_NPEND] = vc[C_NKEEP];
        vc[C_PPAR] = vc[C_PPAR] ^ 1ull;
        vc[C_DONE] = 0;
    }
}

void launch_probe_records(const ProbeRecs& R, const HashSet& H, const int32_t* status, const int32_t* dup_ref,
                          const int32_t* pool_idx, const int32_t* val_buf, unsigned long long* ctr, int64_t cap_new,
                          double* probe_pts, int32_t* probe_shape, int64_t cap_probe,
                          const cudaGraphConditionalHandle* h, cudaStream_t s) {
    launch_k(k_probe_records, grid_for(cap_new + R.cap_pend, 256), 256, 0, s, R, H, status, dup_ref, pool_idx,
             val_buf, ctr, cap_new, probe_pts, probe_shape, cap_probe, h ? *h : cudaGraphConditionalHandle{},
             h ? 1 : 0);
}

// iteration gate of a graph replay: the iteration (an IF node) runs only when it has work --
// queued states, pending probe records, or (probe stage in the graph) probes to evaluate; a
// replay batch whose queue drained part-way then costs one tiny kernel per left-over iteration
__global__ void k_iter_gate(unsigned long long* ctr, cudaGraphConditionalHandle h, int probes_in_graph) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const bool work = ctr[C_QTAIL] > ctr[C_QHEAD] || ctr[C_NPEND] || (probes_in_graph && ctr[C_NPROBE]);
        cudaGraphSetConditional(h, work ? 1u : 0u);
        if (work) ctr[C_GATED] += 1ull;
    }
}
void launch_iter_gate(unsigned long long* ctr, cudaGraphConditionalHandle h, int probes_in_graph, cudaStream_t s) {
    k_iter_gate<<<1, 32, 0, s>>>(ctr, h, probes_in_graph);
}

__global__ void k_pend_finalize(unsigned long long* ctr, cudaGraphConditionalHandle h, int has_cond) {
    pdl_enter();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (has_cond) cudaGraphSetConditional(h, ctr[C_NPROBE] ? 1u : 0u);
        ctr[C_PREC_TOTAL] += ctr[C_NPREC];
        ctr[C_NPEND] = ctr[C_NKEEP];
        ctr[C_PPAR] ^= 1ull;
    }
}

__global__ void k_zero_keys(uint64_t* keys, const unsigned long long* n_dev, int KW, int64_t cap, int shape_w,
                            const int32_t* shapes, int value) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, cap) * KW;
    GRID_STRIDE(i, n) {
        uint64_t v = 0;
        if (shape_w >= 0) {
            const int64_t item = i / KW;
            if (i - item * KW == shape_w) v = (uint64_t)(shapes ? shapes[item] : value);
        }
        keys[i] = v;
    }
}

void launch_prec_target(const ProbeRecs& R, const int32_t* status, const int32_t* dup_ref, const int32_t* pool_idx,
                        unsigned long long* ctr, int64_t cap, double* probe_pts, int64_t cap_probe, cudaStream_t s) {
    launch_k(k_prec_target, grid_for(cap, 256),  256,  0,  s, R, status, dup_ref, pool_idx, ctr, cap, probe_pts, cap_probe);
}
void launch_resolve(const ProbeRecs& R, const HashSet& H, const int32_t* val_buf, unsigned long long* ctr, int64_t cap,
                    double* probe_pts, int32_t* probe_shape, int64_t cap_probe, cudaStream_t s) {
    launch_k(k_resolve, grid_for(cap, 256),  256,  0,  s, R, H, val_buf, ctr, cap, probe_pts, probe_shape, cap_probe);
}
void launch_pend_finalize(unsigned long long* ctr, const cudaGraphConditionalHandle* h, cudaStream_t s) {
    launch_k(k_pend_finalize, 1, 32, 0, s, ctr, h ? *h : cudaGraphConditionalHandle{}, h ? 1 : 0);
}

// after a probe stage: the evaluated probes leave the buffer
__global__ void k_probe_done(unsigned long long* ctr, long long cap_probe) {
    pdl_enter();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const unsigned long long n = ctr[C_NPROBE];
        ctr[C_PROBES_TOTAL] += n < (unsigned long long)cap_probe ? n : (unsigned long long)cap_probe;
        ctr[C_NFLUSH] += n ? 1ull : 0ull;
        ctr[C_NPROBE] = 0;
    }
}


void launch_probe_done(unsigned long long* ctr, int64_t cap_probe, cudaStream_t s) {
    launch_k(k_probe_done, 1, 32, 0, s, ctr, (long long)cap_probe);
}
void launch_zero_keys(uint64_t* keys, const unsigned long long* n_dev, int KW, int64_t cap, int shape_w,
                      const int32_t* shapes, int value, cudaStream_t s) {
    launch_k(k_zero_keys, grid_for(cap * KW, 256),  256,  0,  s, keys, n_dev, KW, cap, shape_w, shapes, value);
}

// outbox grouped by owner rank on the device (counting sort over <= world buckets; the order
// inside a bucket is free: the owner inserts the keys into an order-independent set)
__global__ void k_outbox_hist(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner,
                              unsigned long long* cnt) {
    pdl_enter();
    GRID_STRIDE(i, n) {
        const int o = key_owner(keys + i * KW, KW, world);
        owner[i] = o;
        atomicAdd(cnt + o, 1ull);
    }
}
__global__ void k_outbox_scatter(const uint64_t* keys, int64_t n, int KW, int world, const int32_t* owner,
                                 const unsigned long long* cnt, unsigned long long* cursor, uint64_t* dst) {
    pdl_enter();
    __shared__ unsigned long long base[64];
    if (threadIdx.x == 0) {
        unsigned long long b = 0;
        for (int r = 0; r < world && r < 64; r++) { base[r] = b; b += cnt[r]; }
    }
    __syncthreads();
    GRID_STRIDE(i, n) {
        const int o = owner[i];
        const unsigned long long p = base[o] + atomicAdd(cursor + o, 1ull);
        for (int w = 0; w < KW; w++) dst[p * KW + w] = keys[i * KW + w];
    }
}
void launch_outbox_group(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner,
                         unsigned long long* cnt, unsigned long long* cursor, uint64_t* dst, cudaStream_t s) {
    if (n <= 0) return;
    launch_k(k_outbox_hist, grid_for(n, 256), 256, 0, s, keys, n, KW, world, owner, cnt);
    launch_k(k_outbox_scatter, grid_for(n, 256), 256, 0, s, keys, n, KW, world, (const int32_t*)owner,
             (const unsigned long long*)cnt, cursor, dst);
}


__global__ void k_filter_owned(const uint64_t* keys, int64_t n, int KW, int rank, int world, int32_t* idx,
                               unsigned long long* cnt) {
    pdl_enter();
    GRID_STRIDE(i, n) if (key_owner(keys + i * KW, KW, world) == rank) idx[atomicAdd(cnt, 1ull)] = (int32_t)i;
}
void launch_filter_owned(const uint64_t* keys, int64_t n, int KW, int rank, int world, int32_t* idx,
                         unsigned long long* cnt, cudaStream_t s) {
    if (n > 0) { launch_k(k_filter_owned, grid_for(n, 256), 256, 0, s, keys, n, KW, rank, world, idx, cnt); }
}

}  // namespace am
