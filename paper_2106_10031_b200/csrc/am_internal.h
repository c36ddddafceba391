// am_internal.h -- shared declarations of the B200 analytic-marching engine.
//
// Layout in HBM:
//   keys   : [items][KW] uint64, MSB-first packed activation bits (+ branch word)
//   Z      : [items][NB][C] fp64 -- C = 4 (compose: nx, ny, nz, c per neuron row)
//                                    C = 1 (forward: pre-activation per neuron)
//   faces  : [items][M][4] fp64 per-subnetwork face functionals
//   table  : open-addressing hash set, uint64 slots (fp:31 | cand:1 | ref:32)
//   pool   : [cap][KW] uint64 keys referenced by table slots
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/am_b200.h"

namespace am {

int set_error(int code, const char* fmt, ...);   // am_engine.cu; returns code

constexpr double kDegen = 1e-12;   // reference network.py:27 DEGENERATE_NORMAL_TOL
constexpr double kTolDet = 1e-12;  // reference cells.py:32 TOL_DET
constexpr uint64_t kEmpty = ~0ull;

// SM count of the current device (cached per device: one process may drive several GPUs)
inline int device_sms() {
    static int cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

// number of kernels this library launched (bench.py gpu_launches)
extern unsigned long long g_launch_count;

// Programmatic dependent launch: every kernel is launched with programmatic stream
// serialization and starts with pdl_enter() -- it waits for the preceding kernel's memory
// (griddepcontrol.wait) and immediately lets its own dependents begin launching, so the
// ~30 kernels of a BFS iteration overlap their launch latency with the predecessor's tail
// (also inside the captured CUDA graph).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++g_launch_count;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ keys
__host__ __device__ inline int key_bit(const uint64_t* k, int i) {
    return (int)((k[i >> 6] >> (63 - (i & 63))) & 1ull);
}
__host__ __device__ inline uint64_t key_mask(int i) { return 1ull << (63 - (i & 63)); }

__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
__host__ __device__ inline uint64_t key_hash(const uint64_t* k, int kw) {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)kw;
    for (int i = 0; i < kw; i++) {
        uint64_t x = mix64(k[i] + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
        h = (h ^ x) * 0x100000001B3ull;
        h ^= h >> 29;
    }
    return mix64(h);
}
// owner rank of a state (hash mod world) -- the sharding rule of the multi-GPU march
__host__ __device__ inline int key_owner(const uint64_t* k, int kw, int world) {
    return world <= 1 ? 0 : (int)((key_hash(k, kw) >> 7) % (uint64_t)world);
}

// --------------------------------------------------------- per-step args
struct StepDev {
    int n_in, n_out, flags, row_off, in_row_off, sin_row_off, n_sin, sub;
    const double* W;   // padded copy, row stride ldw
    const double* b;
    const double* V;   // padded copy, row stride ldv (or null)
    const double* vb;  // or null
    int ldw, ldv;
    const double* b_shape;    // batch of shapes: per-shape bias [n_shapes][n_out] (null: b shared)
    const double* vb_shape;   // per-shape shortcut bias [n_shapes][n_out] (null: vb shared)
};

// head of one subnetwork: F_j = hw . relu(z_last) + hb
struct SubDev {
    int last_row, last_n;
    const double* hw;
    double hb;
    const double* hb_shape;   // batch of shapes: per-shape head bias [n_shapes] (null: hb shared)
};

// shape of an item (batch-of-shapes engines keep it in key word shape_w; -1: single shape)
__device__ __forceinline__ int item_shape(const uint64_t* key, int shape_w) {
    return shape_w < 0 ? 0 : (int)key[shape_w];
}
__device__ __forceinline__ double step_bias(const StepDev& st, int shape, int r) {
    return st.b_shape ? st.b_shape[(int64_t)shape * st.n_out + r] : st.b[r];
}
__device__ __forceinline__ double head_bias(const SubDev& sd, int shape) {
    return sd.hb_shape ? sd.hb_shape[shape] : sd.hb;
}
__device__ __forceinline__ double step_vbias(const StepDev& st, int shape, int r) {
    return st.vb_shape ? st.vb_shape[(int64_t)shape * st.n_out + r] : (st.vb ? st.vb[r] : 0.0);
}

struct LayerLaunch {
    StepDev st;
    double* Z;            // [items][zs][C]
    uint64_t* keys;       // [items][KW] (offset by *key_off items when key_off is set)
    int* changed;         // compose: per-item canonical-changed flag (may be null)
    const double* pts;    // forward: [items][3]
    const unsigned long long* n_dev;    // item count on the device (null: n_cap items)
    const unsigned long long* key_off;  // optional device offset (items) into keys
    int64_t n_cap;        // capacity / grid sizing
    int KW, zs;           // key words, Z row count per item (>= NB)
    int grid_cap;         // >0: persistent GEMM grid = grid_cap CTAs per SM
    int shape_w;          // key word holding the item's shape (-1: single-shape engine)
    int fp32;             // fp32 mode: round every composed value to fp32
    // prefix reuse: Z double-buffered by iteration parity (*zpar & 1) x zstride doubles (null: Z)
    const unsigned long long* zpar;
    int64_t zstride;
    int nj4;              // 64-row compose tiles with 32 x 32 warp tiles (AM_GEMM_NJ4)
};
__device__ __forceinline__ double* zbase(const LayerLaunch& L) {
    return L.zpar ? L.Z + (int64_t)(*L.zpar & 1ull) * L.zstride : L.Z;
}

// fp32 mode: values kept at fp32 precision (round-to-nearest), fp64 otherwise
__device__ __forceinline__ double prec_round(double v, int fp32) { return fp32 ? (double)__double2float_rn(v) : v; }

__device__ __forceinline__ int64_t dev_count(const unsigned long long* p, int64_t cap) {
    if (!p) return cap;
    int64_t n = (int64_t)*reinterpret_cast<const volatile unsigned long long*>(p);
    return n < cap ? n : cap;
}
__device__ __forceinline__ uint64_t* keys_at(const LayerLaunch& L) {
    return L.key_off ? L.keys + (int64_t)(*L.key_off) * L.KW : L.keys;
}



// result assembly (am_result.cu): sorted cell order + gathered CSR face loops
int assemble_results(const uint64_t* keys, const int32_t* cell_nv, const int64_t* cell_voff, const double* verts,
                     const int32_t* enr, const int64_t* roff, const int32_t* refs, int64_t nc, int64_t nvt, int KW,
                     int shape_w, cudaStream_t s, uint64_t* s_keys, int32_t* s_nv, double* s_verts, int32_t* s_enr,
                     int32_t* s_refs);

// kernels' host-side launchers (am_compose.cu)
void launch_input_step(const LayerLaunch& L, int C, cudaStream_t s);

// every step of a composition in one launch (k_compose_fused)
constexpr int kMaxFusedSteps = 24;
struct FusedCompose {
    CUtensorMap tmW[kMaxFusedSteps];
    CUtensorMap tmV[kMaxFusedSteps];
    StepDev st[kMaxFusedSteps];
    int tmV_ok[kMaxFusedSteps];
    LayerLaunch L;          // common fields (L.st unused)
    int nsteps;
    double* faces;          // [items][n_subs][4]
    const SubDev* subs;
    int n_subs;
};
void launch_compose_fused(const FusedCompose& F, cudaStream_t s);
// hash set (am_hash.cu)
struct HashSet {
    uint64_t* table;      // slots
    uint64_t mask;        // capacity - 1
    uint64_t* pool;       // [cap_pool][KW]
    uint32_t* pool_flags; // bit0 visited cell, bit1 composed, bit2 deferred (queued again, already
                          // counted as visited), bit3 was deferred once
    int32_t* pool_vn;     // validated-neuron count of a visited cell (-1: no face yet)
    int64_t* pool_voff;   // offset of its validated-neuron list
    double* pool_hint;    // [cap][4] a point on the cell's face polygon + search radius (inf: none)
    int64_t* pool_par;    // [cap] prefix_word of the emitting parent (0: none); null: not kept
    int64_t* queue_par;   // [queue cap] the same word per queue entry (k_take's bucketing reads it
                          // coalesced); null: not kept
    unsigned long long* n_pool;  // device counter
    int64_t cap_pool;
    int KW;
};

// whole composition of an iteration (gather + every step + face head) in one launch, for plain
// dense networks of width <= 96 (am_narrow.cu k_compose_narrow)
constexpr int kMaxNarrowSteps = 12;
struct NarrowCompose {
    CUtensorMap tm[kMaxNarrowSteps];   // 96-row W boxes of steps >= 1
    StepDev st[kMaxNarrowSteps];
    int nsteps;
    const SubDev* subs;                // device head table (one subnetwork)
    // iteration state (k_gather_batch's inputs and outputs)
    const uint64_t* pool;
    const double* pool_hint;
    const int32_t* queue;
    const unsigned long long* ctr;
    int32_t* batch_pool;
    int32_t* canon_pos;
    double* ckey_hint;
    // composition outputs
    double* Z;
    uint64_t* keys;
    double* faces;
    int32_t* changed;
    const unsigned long long* n_dev;
    int64_t n_cap;
    int KW, zs, shape_w, fp32;
    int dbg;                           // AM_NARROW_DBG bits (experiments; 8: phase cycle counters)
    int thr8, thr4;                    // tile width by wave size: 8 cells when n >= grid * thr8, 4 when
                                       // n >= grid * thr4, else 2 (AM_NARROW_THR8 / AM_NARROW_THR4)
    int tile_cells;                    // > 0: fixed tile width (AM_NARROW_TILE)
    unsigned long long* prof;          // [8] phase cycles of thread 0 of every CTA (dbg & 8)
    // prefix reuse (prefix != 0): Z is double-buffered by iteration parity (zstride doubles per
    // half), tiles are formed per bucket of blist (IterState), parents' rows read from the
    // other half
    int prefix;
    int snake;                         // boustrophedon tile order (AM_NARROW_SNAKE; with prefix)
    int64_t zstride;
    const int64_t* pool_par;
    const int32_t* blist;
    // near lists of the tile's cells (near_fused != 0; am_near.cuh), indexed by batch item
    int near_fused;
    int NB;
    int32_t* near_n;
    int32_t* near_flags;
    int32_t* near_id;
    double* near_row;
    int near_cap;
    double near_reach, tol_cell, tol_onplane, probe_delta;
    double lo[3], hi[3];
    // canonical insert + frontier of the tile's cells in its epilogue (canon_fused != 0;
    // am_hashset.cuh canon_frontier_one: k_canon_frontier's work without its launch)
    int canon_fused;
    const uint64_t* keys_in;           // non-null: compose these n_cap keys (no queue / pool gather)
    HashSet H;
    int rank, world;
    uint64_t* outbox;
    unsigned long long* n_out;
    int32_t* status2;
    uint64_t* slot2;
    int32_t* canon_pool;
    int32_t* f_items;
    int32_t* f_pool;
    long long max_cells;
};
// point forward on the narrow path (am_narrow.cu k_forward_narrow)
struct ForwardArgs {
    const double* pts;                 // [n][3]
    double* vals;                      // [n] (may be null)
    uint64_t* keys;                    // [n][KW]: in, the shape word (zeroed keys); out, the state bits
    const unsigned long long* n_dev;   // device count (null: n_cap)
    int64_t n_cap;
};
void launch_forward_narrow(const NarrowCompose& P, const ForwardArgs& F, cudaStream_t s);
// sharded march exchange (am_shard.cu)
constexpr int kHdrWords = 8;
void launch_shard_pack(uint64_t* outbox, unsigned long long* ctr, int KW, int world, int64_t cap,
                       int hdr_rows, uint64_t* send, uint64_t* rest, unsigned long long* cnt, int64_t max_keys,
                       cudaStream_t s);
void launch_shard_index(const uint64_t* recv, int KW, int world, int64_t cap, int hdr_rows, int32_t* idx,
                        unsigned long long* n, cudaStream_t s);
// iterative trigger schemes (am_trace.cu)
void launch_trace_init(int64_t n, const double* x0, double* x, double* cur, double step, int32_t* status,
                       int32_t* iters, cudaStream_t s);
void launch_sgd_check(int64_t n, const double* f, int32_t* status, int32_t* iters, int it, double tol,
                      unsigned long long* running, cudaStream_t s);
void launch_sgd_propose(int64_t n, const double* x, const double* f, const double* faces, const uint64_t* keys, int KW,
                        int M, int bw_branch, const double* cur, int32_t* status, double* xn, cudaStream_t s);
void launch_sgd_accept(int64_t n, double* x, double* f, uint64_t* keys, const double* xn, const double* fn,
                       const uint64_t* keysn, int KW, double* cur, const int32_t* status, cudaStream_t s);
void launch_sphere_check(int64_t n, const double* x, const double* f, int32_t* status, int32_t* iters, int it,
                         double tol, double escape, unsigned long long* running, cudaStream_t s);
void launch_sphere_step(int64_t n, double* x, const double* f, const double* faces, const uint64_t* keys, int KW,
                        int M, int bw_branch, double eta, const int32_t* status, cudaStream_t s);
void launch_trace_finish(int64_t n, const double* x, int32_t* status, double* out, cudaStream_t s);
bool narrow_compose_ok(const StepDev* st, int nsteps, int n_subs, int KW);
void launch_compose_narrow(const NarrowCompose& P, cudaStream_t s);
void launch_narrow_check(const double* Z, const double* Z2, const double* F, const double* F2, const uint64_t* K,
                         const uint64_t* K2, const int32_t* ch, const int32_t* ch2, const unsigned long long* n_dev,
                         int64_t n_cap, int NB, int zs, int KW, unsigned long long* dbg, cudaStream_t s);
void launch_gemm_step(const LayerLaunch& L, int C, const CUtensorMap* tmW, const CUtensorMap* tmV,
                      cudaStream_t s, const CUtensorMap* tmW96 = nullptr, const CUtensorMap* tmV96 = nullptr);
int make_tmap_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld_elems,
                 int box_rows = 64);

// device counters shared by the iteration kernels
enum Ctr {
    C_POOL = 0, C_CELLS, C_VERTS, C_REFS, C_OVF0, C_OVF1, C_CAPPED, C_TOTAL, C_QHEAD, C_QTAIL, C_NR, C_NX,
    C_NF, C_NPROBE, C_NEMIT, C_NLOCAL, C_NOUT, C_STALL, C_ITER, C_LIST, C_OPEN, C_NPREC, C_NPEND, C_PPAR,
    C_NKEEP, C_NVAL, C_NPLOCAL, C_PROBES_TOTAL, C_PREC_TOTAL, C_FCURSOR, C_NFLUSH, C_DONE, C_NHEAVY, C_NLIGHT,
    // the batch k_take dequeued: batch items [0, QA) = queue[QHEAD - QA ..), items [QA, nR) =
    // queue[QB ..) (prefix reuse takes the entries queued since the previous take from the
    // tail, so children meet their parents' rows; QMARK = the tail after that take)
    C_QA, C_QB, C_QMARK,
    C_GATED,             // graph-replayed iterations the gate let run (launch accounting)
    C_BK0,               // [kMaxPrefixBuckets] cells of this iteration's batch per shared-step count
    C_BKT0 = C_BK0 + 12, // [kMaxPrefixBuckets] the same, summed over the march's iterations
    C_PRE0 = C_BKT0 + 12,// [kMaxPrefixBuckets] items of buckets f < s (the items step s composes)
    C_N = C_PRE0 + 12
};
constexpr int kMaxPrefixBuckets = 12;
// queue index of batch item b of the current iteration (see C_QA)
__device__ __forceinline__ int64_t batch_queue_index(const unsigned long long* ctr, int64_t b) {
    const int64_t A = (int64_t)ctr[C_QA];
    return b < A ? (int64_t)ctr[C_QHEAD] - A + b : (int64_t)ctr[C_QB] + (b - A);
}

// Prefix reuse of the narrow composition.  A cell emitted by the face stage differs from its
// parent only in the flipped neuron(s): with the first flip in step f, Z rows of steps 0..f are
// the parent's (they depend on the state bits of earlier layers only).  A child composed in the
// iteration right after its parent's copies those rows from the parent's slot of the other
// half of the double-buffered Z and runs the DMMA chain from step f + 1.
//   pool_par / emit_par word: iteration (bits 32..63) | parent batch item (5..31) | f (0..4)
__host__ __device__ __forceinline__ long long prefix_word(unsigned long long iter, long long item, int f) {
    return (long long)((iter << 32) | ((unsigned long long)item << 5) | (unsigned long long)f);
}

// per-item outputs are indexed by source item ci (idx[i] or i): status 1 new / 0 present,
// slot (new), dup_ref (present: pool index, or -2 - launch index of the in-flight winner)
void launch_hash_upsert(const HashSet& H, const uint64_t* src, const int32_t* idx, const unsigned long long* n_dev,
                        int64_t n_cap, int32_t* status, uint64_t* slot, int32_t* dup_ref, uint32_t flag,
                        int32_t* pool_idx, int32_t* queue, unsigned long long* q_tail, const double* src_hint,
                        cudaStream_t s, const int64_t* src_par = nullptr);
void launch_hash_rebuild(const HashSet& H, int64_t n_pool, cudaStream_t s);

// per-iteration guard / queue state (am_hash.cu k_take)
struct IterState {
    unsigned long long* ctr;
    const int32_t* queue;
    int32_t* batch_pool;
    long long B, cap_pool, tcap, cap_cells, cap_verts, cap_refs, cap_outbox, cap_pend, cap_val;
    long long emit_per_cell, verts_per_cell, refs_per_cell;
    int world;
    // prefix reuse (null pool_par: off): the batch's cells are listed per shared-step count
    // (blist[f * B + i], counts in ctr[C_BK0 + f]) for the narrow composition's tiles
    const int64_t* queue_par;   // prefix_word per queue entry (HashSet::queue_par)
    int32_t* blist;
    int max_share;            // largest usable f (nsteps - 1)
    long long max_cells;      // visited-cell cap (this rank's share)
    int cap_drop;             // no deferral: the cap ends the walk (drop what is queued)
};
// probe records: (target pool entry, neuron, point); double-buffered by parity counter
struct ProbeRecs {
    int32_t* cand;        // [cap] emitted-candidate index of the flip the probe belongs to
    int32_t* k;           // [cap] crossed neuron
    double* pt;           // [cap][3]
    int32_t* pend_t[2];   // pending: target pool index
    int32_t* pend_k[2];
    double* pend_pt[2];
    int32_t* s;           // batch of shapes: [cap] shape of the record (null: single shape)
    int32_t* pend_s[2];
    int64_t cap_pend;
};
void launch_prec_target(const ProbeRecs& R, const int32_t* status, const int32_t* dup_ref, const int32_t* pool_idx,
                        unsigned long long* ctr, int64_t cap, double* probe_pts, int64_t cap_probe, cudaStream_t s);
void launch_resolve(const ProbeRecs& R, const HashSet& H, const int32_t* val_buf, unsigned long long* ctr,
                    int64_t cap, double* probe_pts, int32_t* probe_shape, int64_t cap_probe, cudaStream_t s);
void launch_iter_gate(unsigned long long* ctr, cudaGraphConditionalHandle h, int probes_in_graph, cudaStream_t s);
void launch_pend_finalize(unsigned long long* ctr, const cudaGraphConditionalHandle* h, cudaStream_t s);
void launch_probe_records(const ProbeRecs& R, const HashSet& H, const int32_t* status, const int32_t* dup_ref,
                          const int32_t* pool_idx, const int32_t* val_buf, unsigned long long* ctr, int64_t cap_new,
                          double* probe_pts, int32_t* probe_shape, int64_t cap_probe,
                          const cudaGraphConditionalHandle* h, cudaStream_t s);
void launch_probe_done(unsigned long long* ctr, int64_t cap_probe, cudaStream_t s);
void launch_take(const IterState& I, cudaStream_t s);
// k_gather_batch + the first (input) compose step of the batch in one launch (am_compose.cu)
void launch_gather_input(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                         const unsigned long long* ctr, int32_t* batch_pool, double* ckey_hint, int32_t* canon_pos,
                         const LayerLaunch& L, cudaStream_t s, const int32_t* blist = nullptr, int nb = 0);
// prefix reuse on the per-step path (k_prefix_rows): step row table + the bucket counters
struct PrefixRows {
    const unsigned long long* ctr;
    int nb;                       // buckets (= steps)
    int row_off[12], n_out[12];
};
void launch_prefix_rows(const PrefixRows& R, const LayerLaunch& L, const int32_t* batch_pool, const int64_t* pool_par,
                        cudaStream_t s);
void launch_gather_batch(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                         const unsigned long long* ctr, int32_t* batch_pool, int64_t n_cap, int KW, uint64_t* ckey,
                         double* ckey_hint, int32_t* changed, int32_t* canon_pos, cudaStream_t s);
void launch_route_changed(const uint64_t* ckey, const int32_t* changed, const unsigned long long* n_dev, int64_t n_cap,
                          int KW, int rank, int world, int32_t* X, unsigned long long* nX, uint64_t* outbox,
                          unsigned long long* n_out, int32_t* canon_pos, cudaStream_t s);
void launch_frontier(const unsigned long long* n_dev, int64_t n_cap, const int32_t* changed, const int32_t* batch_pool,
                     const int32_t* canon_pos, const int32_t* canon_status, const int32_t* canon_pool,
                     uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool, unsigned long long* ctr,
                     long long max_cells, cudaStream_t s);
// k_route_changed + canonical k_hash_upsert + k_frontier fused (one launch per iteration)
void launch_canon_frontier(const HashSet& H, const uint64_t* ckey, const int32_t* changed, const int32_t* batch_pool,
                           const unsigned long long* n_dev, int64_t n_cap, int rank, int world, uint64_t* outbox,
                           unsigned long long* n_out, int32_t* canon_pos, int32_t* status2, uint64_t* slot2,
                           int32_t* canon_pool, const double* ckey_hint, int32_t* f_items, int32_t* f_pool,
                           unsigned long long* ctr, long long max_cells, cudaStream_t s);
// zero n keys; with shape_w >= 0 word shape_w gets shapes[item] (or `value` when shapes is null)
void launch_zero_keys(uint64_t* keys, const unsigned long long* n_dev, int KW, int64_t cap, int shape_w,
                      const int32_t* shapes, int value, cudaStream_t s);
void launch_zero_probe_keys(uint64_t* scratch, const unsigned long long* ctr, int KW, int64_t cap, cudaStream_t s);
void launch_emit_finalize(unsigned long long* ctr, cudaStream_t s);
void launch_route_emitted(const uint64_t* scratch, const unsigned long long* ctr_n, int64_t n_cap, int KW, int rank,
                          int world, int32_t* local_idx, unsigned long long* n_local, uint64_t* outbox,
                          unsigned long long* n_out, int32_t* remote_status, cudaStream_t s);
void launch_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst, cudaStream_t s);
void launch_open_edges(const int32_t* enr, const int64_t* roff, const int32_t* refs, int64_t nv, int box0,
                       unsigned long long* out, cudaStream_t s);
void launch_face_head_dev(const double* Z, const uint64_t* keys, double* faces, const unsigned long long* n_dev,
                          int64_t n_cap, int zs, int KW, const void* subs, int n_subs, int shape_w, int fp32,
                          cudaStream_t s, const unsigned long long* zpar = nullptr, int64_t zstride = 0);
void launch_forward_head_dev(const double* Z, uint64_t* keys, const unsigned long long* key_off, double* vals,
                             const unsigned long long* n_dev, int64_t n_cap, int zs, int KW, const void* subs,
                             int n_subs, int ensemble, int shape_w, int fp32, cudaStream_t s);

// face extraction (am_face.cu)
struct FaceArgs {
    const double* Z;          // [batch][zs][4]
    const double* faces;      // [batch][M][4]
    const uint64_t* keys;     // canonical keys [batch][KW]
    const int32_t* items;     // frontier: batch slots to process
    const int32_t* pool_idx;  // per frontier entry: pool index of the state
    const double* hints;      // [batch][4] point on the face polygon + search radius (inf: none)
    double* emit_hint;        // [cap_cand][4] hint of every emitted flip (edge midpoint + radius)
    const unsigned long long* n_dev;  // frontier size (device)
    int64_t n_cap;
    int NB, M, KW, zs, ensemble;
    double lo[3], hi[3];
    double tol_cell, tol_weld, tol_onplane, probe_delta;
    // outputs
    int32_t* cell_pool;       // [cap_cells] pool index per visited cell
    int32_t* cell_nv;         // vertex count (0 = empty face)
    int64_t* cell_voff;       // vertex offset
    unsigned long long* n_cells;
    double* verts;            // [cap_verts][3]
    int32_t* edge_nrefs;      // [cap_verts]
    int64_t* edge_roff;       // [cap_verts] offset into edge_refs
    int32_t* edge_refs;       // [cap_refs] global plane ids
    unsigned long long* n_verts;
    unsigned long long* n_refs;
    int64_t cap_cells, cap_verts, cap_refs;
    uint64_t* cand;           // emitted candidate keys [cap_cand][KW] (flips; probes follow)
    unsigned long long* n_cand;
    int64_t cap_cand;
    double* probe_pts;        // [cap_probe][3]
    unsigned long long* n_probe;
    int64_t cap_probe;
    unsigned long long* overflow;  // counters: [0] C-set/polygon overflow, [1] capacity overflow
    // probe records of single-neuron edges + validated mirrored probes
    int32_t* prec_cand;
    int32_t* prec_k;
    double* prec_pt;
    int32_t* prec_s;          // batch of shapes: shape of the record's cell (null: single shape)
    int shape_w;
    unsigned long long* n_prec;
    int64_t cap_prec;
    int32_t* val_buf;
    unsigned long long* n_val;
    int64_t cap_val;
    int32_t* pool_vn;
    int64_t* pool_voff;
    // deferral of cells whose polygon outgrows the near list's reach: instead of the slow
    // streaming attempts, the cell is queued again with its hint radius widened (so the next
    // near list covers it) and solved in a later iteration -- the visited set and every result
    // are order independent.  Once per cell.  null queue: never defer.
    int32_t* queue;
    unsigned long long* q_tail;
    int64_t defer_min;        // defer only in waves of at least this many cells (a lone deferred cell
                              // costs a whole extra iteration at the end of a march)
    uint32_t* pool_flags;
    double* pool_hint;
    unsigned long long* dbg;   // instrumentation (AM_FACE_STATS builds), may be null
    unsigned long long* cursor;   // work-distribution counter (zeroed by k_take each iteration)
    // near lists (k_near -> k_face), per frontier entry: count, flags, ids and raw rows
    int near_cap;
    double tau_mult;          // first hinted attempt: reach = tau_mult x the hint radius
    double near_reach;        // near lists cover near_reach x the hint radius
    int max_attempts;         // hinted attempts before the full path
    double tau_grow;          // reach growth factor between attempts (at least)
    int32_t* near_n;
    int32_t* near_flags;
    // face work order (k_near -> k_face): cells known to take the slow paths (near list overflow,
    // hint point outside the cell, no hint) first, so their long chains start with the wave
    // instead of trailing it; null: frontier order
    int32_t* order;
    unsigned long long* order_ctr;   // [0] heavy cells placed from the front, [1] light from the back
    int32_t* near_id;         // [n_cap][near_cap]
    double* near_row;         // [n_cap][near_cap][4]
    int near_by_item;         // 1: lists indexed by batch item (built by k_compose_narrow), 0: by frontier entry
    int near_depth;           // k_near: 32-row batches in flight per warp (2 or 4; AM_NEAR_DEPTH)
    // prefix reuse: Z half of this iteration (parity of *zpar), and every emitted flip's
    // prefix_word (first flipped step: step_end[f] > its row) -- null zpar / emit_par: off
    const unsigned long long* zpar;
    int64_t zstride;
    int64_t* emit_par;
    int64_t* queue_par;       // deferral re-queues a cell with no parent word (full composition)
    // flips inserted by the face warps themselves (fused_upsert; single rank): per candidate
    // status / slot / dup_ref / pool index, as k_hash_upsert writes them
    int fused_upsert;
    HashSet H;
    int32_t* cand_status;
    uint64_t* cand_slot;
    int32_t* cand_dup;
    int32_t* cand_pool;
    int32_t* ins_queue;
    int nsteps;
    int step_end[12];
};
constexpr uint32_t kPoolDeferred = 4u, kPoolWasDeferred = 8u;
constexpr int kEmitFlipsPerCell = 48;   // face kernel EMAXC
constexpr int kVertsPerCell = 64;       // face kernel QMAX
constexpr int kRefsPerCell = 256;
void launch_face(const FaceArgs& a, cudaStream_t s);
void launch_near(const FaceArgs& a, cudaStream_t s);

}  // namespace am
