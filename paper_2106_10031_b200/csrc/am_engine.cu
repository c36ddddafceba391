// am_engine.cu -- C-ABI engine: breadth-first analytic marching on one GPU.
//
// Replaces the reference's _Marcher (reference marching.py:216-301).  The work
// queue is a device array of pool indices of not-yet-composed states; the
// visited set is the device hash set (am_hash.cu).  One BFS iteration:
//   take     guard capacities, dequeue up to B states            (k_take)
//   compose  all hidden layers for the batch, fp64 DMMA           (am_compose.cu)
//   canon    states whose canonical key differs are re-inserted   (insert/fixup)
//   frontier new cells of this iteration                          (k_frontier)
//   face     polygons + flip candidates + probe points            (am_face.cu)
//   probe    forward pass at the probe points                     (am_compose.cu C=1)
//   enqueue  insert every emitted state; winners join the queue   (insert/fixup)
// Every kernel reads its item count from device counters, so the iteration is
// captured once as a CUDA graph and replayed; the host only synchronises every
// few iterations to test for termination and to grow buffers.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <memory>
#include <vector>

#include "am_internal.h"

namespace am {
unsigned long long g_launch_count = 0;

void launch_seed_project(const double* X, const double* faces, const uint64_t* keys, int KW, int M, int ensemble,
                         int64_t n, const int32_t* active, double* Xp, int32_t* done_flat, cudaStream_t s);
void launch_seed_check(const uint64_t* snew, const uint64_t* canon, int KW, int64_t n, int32_t* active,
                       double* X, const double* Xp, uint64_t* S, uint64_t* result, int32_t* done_flat,
                       cudaStream_t s);
void launch_dichotomy_step(const double* vals, double* xp, double* xn, double* fp, double* fn, double* mid,
                           int32_t* active, double* out, int64_t n, double eps, double seed_tol, int last,
                           cudaStream_t s);
void launch_midpoint(const double* a, const double* b, double* m, int64_t n, cudaStream_t s);
void launch_bisect_tree(const double* xp, const double* xn, const int32_t* active, int64_t n, double* nodes,
                        cudaStream_t s);
void launch_bisect_replay(const double* vals, const double* nodes, double* xp, double* xn, double* fp, double* fn,
                          int32_t* active, double* out, int64_t n, int it0, int max_iters, double eps,
                          double seed_tol, cudaStream_t s);
int bisect_tree_points();
int bisect_tree_depth();
void launch_point_hints(const double* X, int64_t n, double tau, double* hints, cudaStream_t s);
void launch_count_active(const int32_t* active, int64_t n, unsigned long long* cnt, cudaStream_t s);
void launch_outbox_group(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner,
                         unsigned long long* cnt, unsigned long long* cursor, uint64_t* dst, cudaStream_t s);
void launch_filter_owned(const uint64_t* keys, int64_t n, int KW, int rank, int world, int32_t* idx,
                         unsigned long long* cnt, cudaStream_t s);

}  // namespace am

using namespace am;

static thread_local std::string g_err;
// records the message am_last_error() returns; shared by every C-ABI entry point
int am::set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
#define fail am::set_error
#define fail am::set_error
#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess) return fail(AM_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, \
                                           cudaGetErrorString(_e));                            \
    } while (0)
#define RC(x)                  \
    do {                       \
        int _r = (x);          \
        if (_r) return _r;     \
    } while (0)

template <class T>
struct DBuf {
    T* p = nullptr;
    int64_t n = 0;  // capacity in elements
    // grow to >= m elements (2x geometric); keep the first keep_n elements.  Stream-ordered
    // allocation from the device's default memory pool (kept resident, see pool_setup): no
    // device-wide synchronisation, and a re-created engine reuses the pooled memory.
    cudaError_t reserve(int64_t m, cudaStream_t s, bool keep = false, int64_t keep_n = 0, bool* moved = nullptr) {
        if (m <= n) return cudaSuccess;
        int64_t cap = std::max<int64_t>(m, 2 * n);
        T* q = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&q), (size_t)cap * sizeof(T), s);
        if (e != cudaSuccess) return e;
        if (keep && p && keep_n > 0) {
            e = cudaMemcpyAsync(q, p, (size_t)keep_n * sizeof(T), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
        }
        if (p) cudaFreeAsync(p, s);
        p = q;
        n = cap;
        if (moved) *moved = true;
        return cudaSuccess;
    }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
};

struct am_engine {
    int device = 0;
    cudaStream_t stream = 0;
    bool own_stream = false;
    am_march_params P{};
    // network
    int NB = 0, M = 0, KW = 0, ensemble = 0, zs = 0;
    std::vector<int64_t> steps, subs;
    std::vector<StepDev> sdev;
    std::vector<CUtensorMap> tmW, tmV;
    std::vector<int> tmV_ok;
    std::vector<CUtensorMap> tmW96, tmV96;   // 96-row boxes of the compose steps with 64 < n_out <= 96
    std::vector<int> narrow;
    DBuf<double> params, wpad;
    int n_shapes = 1, shape_w = -1, cur_shape = 0;   // batch of shapes (am_engine_set_shape_params)
    int fp32 = 0;                                    // fp32 mode (am_march_params.precision)
    DBuf<double> shape_tab;                          // per-shape bias tables
    std::vector<int64_t> shp_idx;                    // overridden parameter entries ...
    std::vector<double> shp_val;                     // ... and their per-shape values [S][n_idx]
    DBuf<int32_t> probe_shape, prec_s, pend_s[2];    // shapes of probe points / records (batches)
    int64_t n_params = 0;
    std::vector<int64_t> woff, voff;   // padded weight layout (wpad_layout)
    DBuf<uint8_t> subdev;
    double flops_per_cell = 0, flops_per_point = 0;
    // hash set + queue
    DBuf<uint64_t> table, pool;
    DBuf<uint32_t> pool_flags;
    DBuf<int32_t> queue, pool_vn;
    DBuf<int64_t> pool_voff;
    DBuf<double> pool_hint, ckey_hint, emit_hint, near_row;
    DBuf<int32_t> near_n, near_flags, near_id;   // k_near lists per frontier entry
    DBuf<int32_t> f_order;                        // face work order (heavy cells first)
    int64_t defer_min = 0;      // AM_DEFER_MIN: smallest wave that defers
    bool defer = true;          // deferral of cells that outgrow their near list (AM_DEFER=0: stream them)
    bool canon_fused = true;    // k_canon_frontier (AM_CANON_FUSED=0: the three separate kernels)
    bool face_order = false;                      // AM_FACE_ORDER=1: heavy cells first (A/B: 20.15 vs 19.95 ms, off)
    int near_cap = 256;
    double tau_mult = 1.0, near_reach = 4.5;   // near-list reach in hint radii (A/B after the 96-row GEMM: 6 -> 24.7-24.9 ms, 4.5 -> 24.5)
    int max_attempts = 12;                     // hinted attempts (AM_MAX_ATTEMPTS; 5 -> 12: 31 -> 28.3 ms)
    double tau_grow = 2.0;                     // reach growth per failed attempt (AM_TAU_GROW)
    // composition: per-step launches (AM_COMPOSE_FUSED=1: one fused launch for all steps; slower
    // on configs[1] and DeepSDF, kept for experiments)
    bool compose_fused = false;
    std::unique_ptr<FusedCompose> fused{new FusedCompose()};
    // narrow plain networks (every hidden width <= 96): gather + composition + face head of an
    // iteration in one launch (am_narrow.cu; AM_NARROW=0 selects the per-step kernels)
    bool narrow_fused = false;
    bool narrow_check = false;   // AM_NARROW_CHECK=1: also run the per-step path into shadow buffers and compare
    DBuf<double> Z2, faces2;
    DBuf<uint64_t> ckey2;
    DBuf<int32_t> changed2;
    // prefix reuse of the narrow composition (AM_PREFIX=0: off): the iterations' Z rows in two
    // halves by iteration parity, each pool entry's / emitted flip's parent word, and the batch
    // listed per shared-step bucket
    bool prefix = false;
    int near_depth = 2;         // AM_NEAR_DEPTH
    bool narrow_snake = true;   // AM_NARROW_SNAKE
    int gemm_nj4 = 0;           // AM_GEMM_NJ4: 32 x 32 warp tiles in the 64-row compose GEMM
    // flips inserted by the face warps themselves (AM_FACE_UPSERT=1; single rank): bitwise-equal
    // marches but slower (configs[1] BFS 18.55 vs 17.76 ms, a 48-wave small net 3.78 vs 3.57):
    // the hash probes lengthen every cell's chain more than the separate launch costs
    bool face_upsert = false;
    // point forwards through k_forward_narrow on the narrow path (AM_FORWARD_NARROW=0: the
    // per-layer kernels; bitwise equal).  The trigger: sample_seeds 1.43 -> 1.27 ms, e2e -0.3 ms;
    // the BFS is unaffected since the exact probe forwards moved to the host rounds (17.64 vs
    // 17.67 ms; with a per-iteration probe stage it had cost 0.2 ms)
    bool forward_narrow = true;
    bool narrow_explicit = true;   // explicit-key compositions (seeds, affine maps) on k_compose_narrow (AM_NARROW_EXPLICIT)
    bool canon_in_narrow = false;   // canonical insert + frontier in k_compose_narrow (AM_CANON_IN_NARROW)
    bool near_fused = false;    // near lists built by k_compose_narrow (AM_NEAR_FUSED=1; default: k_near)
    DBuf<double> Zi;
    DBuf<int64_t> pool_par, emit_par, queue_par;
    DBuf<int32_t> blist;
    std::unique_ptr<NarrowCompose> ncomp{new NarrowCompose()};   // face-solver reach (tuning: AM_TAU_MULT, AM_NEAR_REACH)
    DBuf<unsigned long long> dbg;   // face-kernel instrumentation counters (AM_FACE_STATS builds)
    uint64_t tcap = 0;
    // counters (device) + host mirror
    DBuf<unsigned long long> ctr;
    unsigned long long hctr[C_N] = {0};
    // batch buffers (capacity B)
    int64_t B = 0, E = 0, PB = 0, PR = 0;   // batch cells, emitted keys, probe points, probe records
    DBuf<double> Z, faces;
    DBuf<uint64_t> ckey, slot, slot2, scratch, outbox;
    DBuf<int32_t> changed, status, status2, canon_pos, canon_pool, X, f_items, f_pool, batch_pool, local_idx;
    DBuf<double> probe_pts, pZ;
    DBuf<uint64_t> pkeys, pslot;
    DBuf<int32_t> pstatus, emit_dup, emit_pool;
    // probe records (single-neuron edges) + pending list + validated-neuron lists
    DBuf<int32_t> prec_cand, prec_k, pend_t[2], pend_k[2], val_buf;
    DBuf<double> prec_pt, pend_pt[2];
    // results
    DBuf<int32_t> cell_pool, cell_nv, edge_nrefs, edge_refs;
    DBuf<int64_t> cell_voff, edge_roff;
    DBuf<double> verts;
    // host-sized scratch (seeding, pushes, primitives)
    DBuf<uint64_t> hkeys;
    DBuf<uint64_t> s_keys;   // sorted results (am_result_copy)
    DBuf<int32_t> s_nv, s_enr, s_refs;
    DBuf<double> s_verts;
    DBuf<int32_t> hstatus;
    DBuf<uint64_t> hslot;
    DBuf<double> sx, sxp, pvals, shint;
    DBuf<uint64_t> ss, ssn, sres;
    DBuf<int32_t> sact, sdone;
    // graph of one iteration
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    bool graph_valid = false;
    cudaStream_t stream2 = nullptr;          // captures the conditional probe-stage body
    cudaStream_t stream3 = nullptr;          // captures the gated iteration body
    // AM_ITER_GATE=1: each graph-replayed iteration behind an IF node set by a gate kernel (no
    // empty iterations at the end of a replay batch).  Bitwise-equal marches but slower (configs[1]
    // BFS 19.16 vs 17.96 ms, small nets +0.5-1 ms): the conditional node costs every iteration
    // more than the few empty iterations it saves, and it cuts the PDL chain
    bool iter_gate = false;
    unsigned long long gate_kernels = 0;     // kernels of one gated iteration body
    bool probe_in_graph = false;             // probe stage inside the iteration graph (sticky)
    // AM_PROBE_AUTO=1: switch the probe stage into the graph once a host round sees many probes.
    // Off: the exact probe forwards of a round are evaluated together at its host synchronisation
    // (complete DeepSDF march 6.56 -> 6.33 s: ~30 probes per iteration paid a whole per-layer
    // forward pipeline and a conditional node -- which cuts the PDL chain -- every iteration)
    bool probe_auto = false;
    bool shard_probe_in_graph = false;       // AM_SHARD_PROBE_IN_GRAPH
    unsigned long long cond_kernels = 0;     // kernels in that body
    // bisection trigger: engine-owned buffers and a captured 8-step graph (am_dichotomy)
    DBuf<double> dxp, dxn, dfp, dfn, dmid, dvals, dout, dtree, dtvals;
    DBuf<int32_t> dact, dshape, dtshape;
    bool bisect_tree = true;   // speculative bisection tree (AM_BISECT_TREE=0: step by step)
    cudaGraphExec_t dgexec = nullptr;
    int64_t dg_n = -1;
    double dg_eps = 0, dg_tol = 0;
    int dg_shapes = -3;   // -2: per-point shapes, else the engine's current shape at capture
    std::vector<const void*> dg_ptrs;
    unsigned long long dg_kernels = 0;
    // speculative-tree bisection graph (all rounds), keyed like the step graph
    cudaGraphExec_t tgexec = nullptr;
    int64_t tg_n = -1;
    double tg_eps = 0, tg_tol = 0;
    int tg_iters = -1, tg_shapes = -3;
    std::vector<const void*> tg_ptrs;
    unsigned long long tg_kernels = 0;
    // seed refinement graph (am_seed_shapes), keyed like the bisection's
    cudaGraphExec_t sgexec = nullptr;
    int64_t sg_n = -1;
    int sg_shape = -3;
    std::vector<const void*> sg_ptrs;
    unsigned long long sg_kernels = 0;
    DBuf<int32_t> sshape;
    bool gather_input = true;   // k_gather_input: batch gather + input step in one launch
    int graph_batch = 32;   // iterations replayed per host synchronisation (A/B: 8 -> 25.7 ms, 16 -> 25.0, 32 -> 24.6)
    int64_t tail_queue = 64;   // fewer queued cells at a synchronisation: replay tail_batch iterations (AM_TAIL_QUEUE)
    int tail_batch = 8;        // AM_TAIL_BATCH
    int grid_cap = 0;    // >0: CTAs per SM for persistent GEMM launches
    unsigned long long graph_kernels = 0;
    // iterative trigger schemes (am_trace): per-start state
    DBuf<double> tx, tf, txn, tfn, tcur;
    DBuf<uint64_t> tk, tkn;
    DBuf<unsigned long long> trun;
    // sharded rounds (am_shard_*): leftover outbox, pack counters, received-row index, headers
    DBuf<uint64_t> sh_rest;
    DBuf<unsigned long long> sh_cnt;
    DBuf<int32_t> sh_idx;
    uint64_t* h_hdr = nullptr;   // pinned [world][kHdrWords] headers of the last exchange
    bool sh_have_hdr = false;
    unsigned long long n_syncs = 0, sh_rounds = 0, sh_sent = 0, sh_recv = 0;
    // stats
    bool timing = false;
    cudaEvent_t ev[6];
    // timing mode: contiguous per-stage buckets of an iteration (am_kernel_times)
    static constexpr int kMarks = 9;
    cudaEvent_t tev[kMarks] = {};
    double t_bucket[12] = {0};
    double n_emit = 0, n_canon = 0, n_prec = 0, n_new = 0, n_timed = 0;
    cudaEvent_t ev_join = nullptr;   // orders the caller's stream and the engine's own stream
    double t_compose = 0, t_face = 0, t_probe = 0, flops = 0, pflops = 0, face_bytes = 0;
    double n_comp_cells = 0, n_face_cells = 0, n_probes = 0;
    int64_t iters = 0;
};

extern "C" const char* am_last_error(void) { return g_err.c_str(); }

extern "C" int am_device_info(int device, int32_t* sm, int32_t* maj, int32_t* min) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) return fail(AM_ERR_NO_DEVICE, "no CUDA device %d", device);
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    *sm = p.multiProcessorCount;
    *maj = p.major;
    *min = p.minor;
    return AM_OK;
}

// ------------------------------------------------------------------ helpers
static int sync_counters(am_engine* e) {
    CK(cudaMemcpyAsync(e->hctr, e->ctr.p, sizeof(e->hctr), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    e->n_syncs++;
    return AM_OK;
}
static int set_counter(am_engine* e, int which, unsigned long long v) {
    e->hctr[which] = v;
    CK(cudaMemcpyAsync(e->ctr.p + which, &e->hctr[which], sizeof(unsigned long long), cudaMemcpyHostToDevice,
                       e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}
static bool gather_fuses_input(const am_engine* e);

static HashSet hs(am_engine* e) {
    HashSet H;
    H.table = e->table.p;
    H.mask = e->tcap - 1;
    H.pool = e->pool.p;
    H.pool_flags = e->pool_flags.p;
    H.pool_vn = e->pool_vn.p;
    H.pool_voff = e->pool_voff.p;
    H.pool_hint = e->pool_hint.p;
    H.pool_par = e->prefix ? e->pool_par.p : nullptr;
    H.queue_par = e->prefix ? e->queue_par.p : nullptr;
    H.n_pool = e->ctr.p + C_POOL;
    H.cap_pool = e->pool.n / e->KW;
    H.KW = e->KW;
    return H;
}
static int64_t emit_per_cell() { return kEmitFlipsPerCell + kVertsPerCell; }

// hash set + queue room for `extra` more states (load factor <= 1/2)
static int ensure_hash(am_engine* e, int64_t extra, bool sync = true) {
    if (sync) RC(sync_counters(e));
    int64_t np = (int64_t)e->hctr[C_POOL];
    int64_t need = np + extra;
    bool moved = false;
    if (e->pool.n / e->KW < need) {
        CK(e->pool.reserve(need * e->KW, e->stream, true, np * e->KW, &moved));
        CK(e->pool_flags.reserve(e->pool.n / e->KW, e->stream, true, np, &moved));
        CK(e->pool_vn.reserve(e->pool.n / e->KW, e->stream, true, np, &moved));
        CK(e->pool_voff.reserve(e->pool.n / e->KW, e->stream, true, np, &moved));
        CK(e->pool_hint.reserve(e->pool.n / e->KW * 4, e->stream, true, np * 4, &moved));
        if (e->prefix) CK(e->pool_par.reserve(e->pool.n / e->KW, e->stream, true, np, &moved));
    }
    // a cell is queued once, plus at most once more when deferred (face solver, status 3)
    CK(e->queue.reserve(2 * (e->pool.n / e->KW), e->stream, true, (int64_t)e->hctr[C_QTAIL], &moved));
    if (e->prefix) CK(e->queue_par.reserve(e->queue.n, e->stream, true, (int64_t)e->hctr[C_QTAIL], &moved));
    if ((int64_t)e->tcap < 2 * need) {
        uint64_t cap = e->tcap ? e->tcap : 1024;
        while ((int64_t)cap < 2 * need) cap <<= 1;
        e->table.release(e->stream);
        CK(e->table.reserve((int64_t)cap, e->stream));
        e->tcap = cap;
        CK(cudaMemsetAsync(e->table.p, 0xff, cap * sizeof(uint64_t), e->stream));
        launch_hash_rebuild(hs(e), np, e->stream);
        CK(cudaGetLastError());
        moved = true;
    }
    if (moved) e->graph_valid = false;
    return AM_OK;
}

// room for `cells` more visited cells; per-vertex buffers (vertices, edge refs, validation and
// pending-probe lists) get worst-case room for `vcells` cells (default: all of them)
static int ensure_results(am_engine* e, int64_t cells, int64_t vcells = -1, bool sync = true) {
    if (sync) RC(sync_counters(e));
    const int64_t cells_all = cells;
    if (vcells >= 0) cells = vcells;
    int64_t nc = (int64_t)e->hctr[C_CELLS], nv = (int64_t)e->hctr[C_VERTS], nr = (int64_t)e->hctr[C_REFS];
    cudaStream_t s = e->stream;
    bool moved = false;
    CK(e->cell_pool.reserve(nc + cells_all, s, true, nc, &moved));
    CK(e->cell_nv.reserve(nc + cells_all, s, true, nc, &moved));
    CK(e->cell_voff.reserve(nc + cells_all, s, true, nc, &moved));
    CK(e->verts.reserve((nv + cells * kVertsPerCell) * 3, s, true, nv * 3, &moved));
    CK(e->edge_nrefs.reserve(nv + cells * kVertsPerCell, s, true, nv, &moved));
    CK(e->edge_roff.reserve(nv + cells * kVertsPerCell, s, true, nv, &moved));
    CK(e->edge_refs.reserve(nr + cells * kRefsPerCell, s, true, nr, &moved));
    int64_t nval = (int64_t)e->hctr[C_NVAL], npend = (int64_t)e->hctr[C_NPEND];
    int par = (int)(e->hctr[C_PPAR] & 1ull);
    CK(e->val_buf.reserve(nval + cells * kVertsPerCell, s, true, nval, &moved));
    int64_t pcap = npend + cells * kVertsPerCell;
    for (int q = 0; q < 2; q++) {
        int64_t keep = q == par ? npend : 0;
        CK(e->pend_t[q].reserve(pcap, s, true, keep, &moved));
        CK(e->pend_k[q].reserve(pcap, s, true, keep, &moved));
        CK(e->pend_pt[q].reserve(pcap * 3, s, true, keep * 3, &moved));
        if (e->shape_w >= 0) CK(e->pend_s[q].reserve(pcap, s, true, keep, &moved));
    }
    if (e->P.world > 1) {
        int64_t no = (int64_t)e->hctr[C_NOUT];
        CK(e->outbox.reserve((no + cells_all * (1 + emit_per_cell())) * e->KW, s, true, no * e->KW, &moved));
    }
    if (moved) e->graph_valid = false;
    return AM_OK;
}

// -------------------------------------------------------------- lifecycle
// padded weight layout: per step, W (and the shortcut V) with a row stride of 16 doubles
static int64_t wpad_layout(am_engine* e, std::vector<int64_t>& woff, std::vector<int64_t>& voff) {
    const int ns = (int)(e->steps.size() / AM_STEP_FIELDS);
    woff.assign(ns, 0);
    voff.assign(ns, -1);
    int64_t tot = 0;
    auto pad = [](int64_t x) { return (x + 15) / 16 * 16; };
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        woff[s] = tot;
        tot += st[1] * pad(st[0]);
        if (st[5] >= 0) { voff[s] = tot; tot += st[1] * pad(st[10]); }
    }
    return tot;
}

// per-shape bias tables of a batch of shapes: every overridden parameter must be a layer bias,
// a shortcut bias or a head bias; each affected vector gets a [n_shapes][n] table holding the
// base values with the shape's overrides applied
static int build_shape_tables(am_engine* e, const double* h_params, std::vector<const double*>* hb_shape) {
    const int ns = (int)(e->steps.size() / AM_STEP_FIELDS), S = e->n_shapes;
    const int64_t n_idx = (int64_t)e->shp_idx.size();
    for (int st = 0; st < ns; st++) { e->sdev[st].b_shape = nullptr; e->sdev[st].vb_shape = nullptr; }
    hb_shape->assign(e->M, nullptr);
    if (n_idx == 0) return AM_OK;
    // (vector kind, owner, offset of the vector in params, length) for each overridden entry
    struct Vec { int kind, owner; int64_t base, len, tab; };
    std::vector<Vec> vecs;
    std::vector<int> vec_of(n_idx, -1), pos_of(n_idx, 0);
    for (int64_t j = 0; j < n_idx; j++) {
        const int64_t ix = e->shp_idx[j];
        int kind = -1, owner = -1;
        int64_t base = 0, len = 0;
        for (int st = 0; st < ns && kind < 0; st++) {
            const int64_t* d = &e->steps[(size_t)st * AM_STEP_FIELDS];
            if (ix >= d[3] && ix < d[3] + d[1]) { kind = 0; owner = st; base = d[3]; len = d[1]; }
            else if (d[6] >= 0 && ix >= d[6] && ix < d[6] + d[1]) { kind = 1; owner = st; base = d[6]; len = d[1]; }
        }
        for (int sb = 0; sb < e->M && kind < 0; sb++)
            if (ix == e->subs[(size_t)sb * AM_SUB_FIELDS + 3]) { kind = 2; owner = sb; base = ix; len = 1; }
        if (kind < 0)
            return fail(AM_ERR_ARG, "shape parameter %lld is not a bias: shapes of a batch must share every weight",
                        (long long)ix);
        int v = -1;
        for (size_t q = 0; q < vecs.size(); q++)
            if (vecs[q].kind == kind && vecs[q].owner == owner) v = (int)q;
        if (v < 0) { vecs.push_back({kind, owner, base, len, 0}); v = (int)vecs.size() - 1; }
        vec_of[j] = v;
        pos_of[j] = (int)(ix - base);
    }
    int64_t tot = 0;
    for (auto& v : vecs) { v.tab = tot; tot += (int64_t)S * v.len; }
    std::vector<double> h(tot);
    for (auto& v : vecs)
        for (int sh = 0; sh < S; sh++)
            memcpy(&h[v.tab + (int64_t)sh * v.len], h_params + v.base, (size_t)v.len * sizeof(double));
    for (int sh = 0; sh < S; sh++)
        for (int64_t j = 0; j < n_idx; j++) {
            const Vec& v = vecs[vec_of[j]];
            h[v.tab + (int64_t)sh * v.len + pos_of[j]] =
                e->fp32 ? (double)(float)e->shp_val[(size_t)sh * n_idx + j] : e->shp_val[(size_t)sh * n_idx + j];
        }
    CK(e->shape_tab.reserve(std::max<int64_t>(tot, 1), e->stream));
    CK(cudaMemcpyAsync(e->shape_tab.p, h.data(), (size_t)tot * sizeof(double), cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (auto& v : vecs) {
        const double* p = e->shape_tab.p + v.tab;
        if (v.kind == 0) e->sdev[v.owner].b_shape = p;
        else if (v.kind == 1) e->sdev[v.owner].vb_shape = p;
        else (*hb_shape)[v.owner] = p;
    }
    e->graph_valid = false;   // captured launches carry the table pointers
    return AM_OK;
}

// network parameters -> device: the flat parameter buffer, the padded per-step weight copies
// the TMA descriptors point at, and the per-subnetwork head table (head bias by value)
static int upload_params(am_engine* e, const double* h_params_in) {
    const int ns = (int)(e->steps.size() / AM_STEP_FIELDS);
    std::vector<double> rounded;          // fp32 mode: the network at fp32 precision
    const double* h_params = h_params_in;
    if (e->fp32) {
        rounded.assign(h_params_in, h_params_in + e->n_params);
        for (double& v : rounded) v = (double)(float)v;
        h_params = rounded.data();
    }
    CK(cudaMemcpyAsync(e->params.p, h_params, (size_t)e->n_params * sizeof(double), cudaMemcpyHostToDevice,
                       e->stream));
    auto pad = [](int64_t x) { return (x + 15) / 16 * 16; };
    std::vector<double> hw((size_t)std::max<int64_t>(e->wpad.n, 1), 0.0);
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        int64_t n_in = st[0], n_out = st[1], ld = pad(n_in);
        for (int64_t r = 0; r < n_out; r++)
            memcpy(&hw[e->woff[s] + r * ld], h_params + st[2] + r * n_in, (size_t)n_in * sizeof(double));
        if (st[5] >= 0) {
            int64_t n_sin = st[10], ldv = pad(n_sin);
            for (int64_t r = 0; r < n_out; r++)
                memcpy(&hw[e->voff[s] + r * ldv], h_params + st[5] + r * n_sin, (size_t)n_sin * sizeof(double));
        }
    }
    CK(cudaMemcpyAsync(e->wpad.p, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice, e->stream));
    std::vector<const double*> hb_shape;
    RC(build_shape_tables(e, h_params, &hb_shape));
    std::vector<SubDev> hsub(e->M);
    for (int j = 0; j < e->M; j++) {
        const int64_t* sb = &e->subs[(size_t)j * AM_SUB_FIELDS];
        int last = (int)(sb[0] + sb[1] - 1);
        const int64_t* st = &e->steps[(size_t)last * AM_STEP_FIELDS];
        hsub[j].last_row = (int)st[7];
        hsub[j].last_n = (int)st[1];
        hsub[j].hw = e->params.p + sb[2];
        hsub[j].hb = h_params[sb[3]];
        hsub[j].hb_shape = hb_shape[j];
    }
    CK(cudaMemcpyAsync(e->subdev.p, hsub.data(), sizeof(SubDev) * e->M, cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));   // host staging vectors go out of scope
    return AM_OK;
}

extern "C" int am_engine_create(am_engine** out, const am_net_desc* net, const am_march_params* p, int device,
                                void* stream) {
    if (!out || !net || !p) return fail(AM_ERR_ARG, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device)
        return fail(AM_ERR_NO_DEVICE, "no CUDA device %d (found %d)", device, ndev);
    CK(cudaSetDevice(device));
    {   // keep freed engine / weld / result memory in the device's default pool
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    am_engine* e = new am_engine();
    e->device = device;
    e->stream = (cudaStream_t)stream;
    if (!e->stream) {  // graphs cannot be captured on the legacy default stream
        CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->own_stream = true;
    }
    CK(cudaStreamCreateWithFlags(&e->stream2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->stream3, cudaStreamNonBlocking));
    e->P = *p;
    if (e->P.world < 1) e->P.world = 1;
    e->NB = net->n_bits;
    e->M = net->n_subs;
    e->ensemble = net->ensemble;
    e->n_shapes = e->P.n_shapes > 1 ? e->P.n_shapes : 1;
    if (e->P.precision != 0 && e->P.precision != 1) return fail(AM_ERR_ARG, "precision must be 0 (fp64) or 1 (fp32)");
    e->fp32 = e->P.precision;
    if (e->n_shapes > 1 && e->ensemble) return fail(AM_ERR_ARG, "a batch of shapes of max-pool ensembles is not supported");
    e->KW = (e->NB + 63) / 64 + (e->ensemble ? 1 : 0) + (e->n_shapes > 1 ? 1 : 0);
    e->shape_w = e->n_shapes > 1 ? e->KW - 1 : -1;
    e->zs = e->NB;
    e->steps.assign(net->h_steps, net->h_steps + (size_t)net->n_steps * AM_STEP_FIELDS);
    e->subs.assign(net->h_subs, net->h_subs + (size_t)net->n_subs * AM_SUB_FIELDS);
    e->n_params = net->n_params;
    CK(e->params.reserve(std::max<int64_t>(net->n_params, 1), e->stream));

    // padded weight copies (row stride multiple of 16 doubles) for TMA
    int ns = net->n_steps;
    int64_t tot = wpad_layout(e, e->woff, e->voff);
    CK(e->wpad.reserve(std::max<int64_t>(tot, 1), e->stream));
    e->sdev.resize(ns);
    e->tmW.resize(ns);
    e->tmV.resize(ns);
    e->tmV_ok.assign(ns, 0);
    e->tmW96.resize(ns);
    e->tmV96.resize(ns);
    e->narrow.assign(ns, 0);
    const char* nv = getenv("AM_NARROW96");
    const bool use96 = !nv || atoi(nv) != 0;
    auto pad = [](int64_t x) { return (x + 15) / 16 * 16; };
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        StepDev& d = e->sdev[s];
        d.n_in = (int)st[0]; d.n_out = (int)st[1]; d.flags = (int)st[4]; d.row_off = (int)st[7];
        d.in_row_off = (int)st[8]; d.sin_row_off = (int)st[9]; d.n_sin = (int)st[10]; d.sub = (int)st[11];
        d.W = e->wpad.p + e->woff[s];
        d.ldw = (int)pad(st[0]);
        d.b = e->params.p + st[3];
        d.V = st[5] >= 0 ? e->wpad.p + e->voff[s] : nullptr;
        d.ldv = st[5] >= 0 ? (int)pad(st[10]) : 0;
        d.vb = st[6] >= 0 ? e->params.p + st[6] : nullptr;
        if (!(d.flags & AM_STEP_FIRST)) {
            if (make_tmap_2d(&e->tmW[s], d.W, d.n_out, d.n_in, d.ldw) != 0)
                return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for step %d", s);
            e->flops_per_cell += 2.0 * d.n_out * d.n_in * 4;
            e->flops_per_point += 2.0 * d.n_out * d.n_in;
            if (use96 && d.n_out > 64 && d.n_out <= 96) {
                if (make_tmap_2d(&e->tmW96[s], d.W, d.n_out, d.n_in, d.ldw, 96) != 0)
                    return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for step %d", s);
                e->narrow[s] = 1;
            }
        }
        if (d.V && !(d.flags & AM_STEP_SC_FROM_INPUT)) {
            if (make_tmap_2d(&e->tmV[s], d.V, d.n_out, d.n_sin, d.ldv) != 0)
                return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for shortcut of step %d", s);
            e->tmV_ok[s] = 1;
            if (e->narrow[s] && make_tmap_2d(&e->tmV96[s], d.V, d.n_out, d.n_sin, d.ldv, 96) != 0)
                return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for shortcut of step %d", s);
            e->flops_per_cell += 2.0 * d.n_out * d.n_sin * 4;
            e->flops_per_point += 2.0 * d.n_out * d.n_sin;
        }
    }
    CK(e->subdev.reserve((int64_t)(sizeof(SubDev) * e->M), e->stream));
    RC(upload_params(e, net->h_params));
    {
        const char* nv = getenv("AM_NARROW");
        const int KWk = (e->NB + 63) / 64 + (e->ensemble ? 1 : 0) + (e->n_shapes > 1 ? 1 : 0);
        if ((!nv || atoi(nv) != 0) && narrow_compose_ok(e->sdev.data(), ns, e->M, KWk)) {
            NarrowCompose& N = *e->ncomp;
            N.nsteps = ns;
            for (int s = 0; s < ns; s++) {
                const StepDev& d = e->sdev[s];
                if (s > 0 && make_tmap_2d(&N.tm[s], d.W, d.n_out, d.n_in, d.ldw, 96) != 0)
                    return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for narrow step %d", s);
            }
            e->narrow_fused = true;
            if (const char* v = getenv("AM_NARROW_CHECK")) e->narrow_check = atoi(v) != 0;
            if (const char* v = getenv("AM_NARROW_DBG")) N.dbg = atoi(v);
            N.thr8 = 12; N.thr4 = 4; N.tile_cells = 0;
            if (const char* v = getenv("AM_NARROW_THR8")) N.thr8 = atoi(v);
            if (const char* v = getenv("AM_NARROW_THR4")) N.thr4 = atoi(v);
            if (const char* v = getenv("AM_NARROW_TILE")) N.tile_cells = atoi(v);
        }
    }
    // batch size from the per-iteration memory budget: compose planes + worst-case probe
    // activations + emitted keys per batch cell
    // Heavy compositions (>= 2 MFLOP per cell, e.g. DeepSDF 512x8) take batches of up to 64 k
    // cells within a 32 GB budget: a wide frontier then composes in fewer, fuller waves and the
    // previous batch's children all fit the next batch (prefix reuse).  Complete DeepSDF march:
    // 16 k -> 8.07 s, 24 k -> 7.55, 32 k -> 7.24, 48 k -> 6.74, 64 k -> 6.74 s (waves 1002 -> 818).
    // Light ones keep 16 k cells in 4 GB (configs[1]'s waves stay below 6 k cells).
    // (sharded engines keep 16 k: the exchange buffers are reserved for a whole round's worst-case
    // emissions, and several ranks may share a device in functional checks)
    const bool heavy = e->flops_per_cell >= 2.0e6 && e->P.world <= 1;
    int64_t budget = e->P.mem_budget > 0 ? e->P.mem_budget : (int64_t)(heavy ? 32 : 4) << 30;
    int64_t per = (int64_t)e->zs * 32 * 3 + (int64_t)e->zs * 8 + emit_per_cell() * e->KW * 8 * 2 +
                  (int64_t)kVertsPerCell * 40 + e->M * 32 + 256;   // Z + both prefix halves
    e->B = e->P.batch_cells > 0 ? e->P.batch_cells
                                : std::max<int64_t>(256, std::min<int64_t>(budget / per, heavy ? 65536 : 16384));
    e->E = e->B * emit_per_cell();
    e->PB = std::max<int64_t>(e->B, 4096);   // exact probe evaluations per iteration (overflow waits in pending)
    e->PR = e->B * kVertsPerCell;           // probe records per iteration (one per edge at most)
    if (e->P.max_cells <= 0) e->P.max_cells = INT64_C(10000000);
    cudaStream_t s = e->stream;
    CK(e->Z.reserve(e->B * e->zs * 4, s));
    CK(e->faces.reserve(e->B * e->M * 4, s));
    CK(e->ckey.reserve(e->B * e->KW, s));
    DBuf<int32_t>* bi[] = {&e->changed, &e->status2, &e->canon_pos, &e->canon_pool, &e->X, &e->f_items, &e->f_pool,
                           &e->batch_pool};
    for (auto* x : bi) CK(x->reserve(e->B, s));
    CK(e->slot2.reserve(e->B, s));
    CK(e->scratch.reserve(e->E * e->KW, s));
    CK(e->status.reserve(e->E, s));
    CK(e->slot.reserve(e->E, s));
    CK(e->local_idx.reserve(e->E, s));
    CK(e->probe_pts.reserve(e->PB * 3, s));
    CK(e->pZ.reserve(e->PB * e->zs, s));
    CK(e->pkeys.reserve(e->PB * e->KW, s));
    CK(e->pslot.reserve(e->PB, s));
    CK(e->pstatus.reserve(e->PB, s));
    CK(e->emit_dup.reserve(e->E, s));
    CK(e->emit_pool.reserve(e->E, s));
    CK(e->emit_hint.reserve(e->E * 4, s));
    CK(e->ckey_hint.reserve(e->B * 4, s));
    if (const char* v = getenv("AM_TAU_MULT")) e->tau_mult = atof(v);
    if (const char* v = getenv("AM_COMPOSE_FUSED")) e->compose_fused = atoi(v) != 0;
    if (const char* v = getenv("AM_PROBE_IN_GRAPH")) e->probe_in_graph = atoi(v) != 0;
    if (const char* v = getenv("AM_PROBE_AUTO")) e->probe_auto = atoi(v) != 0;
    if (const char* v = getenv("AM_SHARD_PROBE_IN_GRAPH")) e->shard_probe_in_graph = atoi(v) != 0;
    if (const char* v = getenv("AM_NEAR_REACH")) e->near_reach = atof(v);
    if (const char* v = getenv("AM_NEAR_CAP")) e->near_cap = atoi(v);
    if (const char* v = getenv("AM_MAX_ATTEMPTS")) e->max_attempts = atoi(v);
    if (const char* v = getenv("AM_TAU_GROW")) e->tau_grow = atof(v);
    if (const char* v = getenv("AM_BISECT_TREE")) e->bisect_tree = atoi(v) != 0;
    if (const char* v = getenv("AM_GRAPH_BATCH")) e->graph_batch = std::max(1, atoi(v));
    if (const char* v = getenv("AM_TAIL_QUEUE")) e->tail_queue = atoll(v);
    if (const char* v = getenv("AM_TAIL_BATCH")) e->tail_batch = std::max(1, atoi(v));
    if (const char* v = getenv("AM_GATHER_INPUT")) e->gather_input = atoi(v) != 0;
    if (e->narrow_check) {
        CK(e->Z2.reserve(e->Z.n, s)); CK(e->faces2.reserve(e->faces.n, s));
        CK(e->ckey2.reserve(e->ckey.n, s)); CK(e->changed2.reserve(e->changed.n, s));
    }
    // narrow path, or the per-step path with the gather fused into the input step where the
    // composition is heavy enough to repay the extra launch (A/B, BFS ms off -> on: DeepSDF
    // 512x8 first 1M cells 722 -> 545, 128-wide 108.8 -> 98.5, 64-wide 19.7 -> 21.5, configs[1]
    // per-step 22.3 -> 23.1)
    e->prefix = (e->narrow_fused ? !e->narrow_check : gather_fuses_input(e) && e->flops_per_cell >= 5.0e5) &&
                (int)e->sdev.size() <= kMaxPrefixBuckets && e->B < (INT64_C(1) << 27);
    if (const char* v = getenv("AM_PREFIX")) e->prefix = e->prefix && atoi(v) != 0;
    if (e->prefix) {
        CK(e->Zi.reserve(2 * e->B * e->zs * 4, s));
        CK(e->emit_par.reserve(e->E, s));
        CK(e->blist.reserve(kMaxPrefixBuckets * e->B, s));
    }
    CK(e->near_n.reserve(e->B, s));
    CK(e->f_order.reserve(e->B, s));
    if (const char* v = getenv("AM_FACE_ORDER")) e->face_order = atoi(v) != 0;
    // near lists inside k_compose_narrow (AM_NEAR_FUSED=1): correct, but slower on configs[1]
    // (BFS 18.58 vs 18.27 ms): 12 warps per SM stream the tile's rows at the end of every tile,
    // where k_near keeps 32 warps per SM of row loads in flight
    if (const char* v = getenv("AM_NEAR_DEPTH")) e->near_depth = atoi(v);
    if (const char* v = getenv("AM_NARROW_SNAKE")) e->narrow_snake = atoi(v) != 0;
    if (const char* v = getenv("AM_ITER_GATE")) e->iter_gate = atoi(v) != 0;
    if (const char* v = getenv("AM_GEMM_NJ4")) e->gemm_nj4 = atoi(v) != 0;
    if (const char* v = getenv("AM_FACE_UPSERT")) e->face_upsert = atoi(v) != 0;
    if (const char* v = getenv("AM_FORWARD_NARROW")) e->forward_narrow = atoi(v) != 0;
    if (const char* v = getenv("AM_NARROW_EXPLICIT")) e->narrow_explicit = atoi(v) != 0;
    if (const char* v = getenv("AM_NEAR_FUSED"))
        e->near_fused = e->narrow_fused && !e->face_order && !e->narrow_check && atoi(v) != 0;
    if (const char* v = getenv("AM_CANON_FUSED")) e->canon_fused = atoi(v) != 0;
    // canonical insert + frontier in k_compose_narrow's tile epilogue (AM_CANON_IN_NARROW=1):
    // correct, but slower on configs[1] (BFS 18.48 vs 17.99 ms)
    if (const char* v = getenv("AM_CANON_IN_NARROW"))
        e->canon_in_narrow = e->narrow_fused && e->canon_fused && atoi(v) != 0;
    // deferral re-composes the deferred cells: worth it where the face solve dominates (narrow
    // nets; configs[1] 19.75 -> 18.85 ms), not where composition does (DeepSDF 512x8: 0.724 ->
    // 0.747 s for the first 1 M cells)
    e->defer = e->flops_per_cell < 2.0e6;
    if (const char* v = getenv("AM_DEFER")) e->defer = atoi(v) != 0;
    if (const char* v = getenv("AM_DEFER_MIN")) e->defer_min = atoll(v);
    CK(e->near_flags.reserve(e->B, s));
    CK(e->near_id.reserve(e->B * e->near_cap, s));
    CK(e->near_row.reserve(e->B * e->near_cap * 4, s));
    CK(e->prec_cand.reserve(e->PR, s));
    CK(e->prec_k.reserve(e->PR, s));
    CK(e->prec_pt.reserve(e->PR * 3, s));
    if (e->shape_w >= 0) {
        CK(e->prec_s.reserve(e->PR, s));
        CK(e->probe_shape.reserve(e->PB, s));
    }
    CK(e->outbox.reserve(e->KW, s));
    CK(e->ctr.reserve(C_N, s));
    CK(cudaMemsetAsync(e->ctr.p, 0, C_N * sizeof(unsigned long long), e->stream));
    CK(e->dbg.reserve(64, s));
    CK(cudaMemsetAsync(e->dbg.p, 0, 64 * sizeof(unsigned long long), e->stream));
    for (int i = 0; i < 6; i++) cudaEventCreate(&e->ev[i]);
    for (int i = 0; i < am_engine::kMarks; i++) cudaEventCreate(&e->tev[i]);
    CK(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    // initial room: the trigger's and one iteration's worth; the march grows it from the observed
    // per-cell growth before every batch of graph replays (ensure_iter_room)
    int64_t init_keys = e->B * 8;
    if (const char* v = getenv("AM_INIT_KEYS")) init_keys = std::max<int64_t>(1024, atoll(v));
    int rc = ensure_hash(e, init_keys);
    if (!rc) rc = ensure_results(e, e->B, std::min<int64_t>(e->B, 4096));
    if (rc) { delete e; return rc; }
    *out = e;
    return AM_OK;
}

extern "C" int am_engine_destroy(am_engine* e) {
    if (!e) return AM_OK;
    cudaStreamSynchronize(e->stream);
    if (e->gexec) cudaGraphExecDestroy(e->gexec);
    if (e->dgexec) cudaGraphExecDestroy(e->dgexec);
    if (e->sgexec) cudaGraphExecDestroy(e->sgexec);
    if (e->tgexec) cudaGraphExecDestroy(e->tgexec);
    e->sshape.release(e->stream);
    for (auto* b : {&e->dxp, &e->dxn, &e->dfp, &e->dfn, &e->dmid, &e->dvals, &e->dout, &e->dtree, &e->dtvals})
        b->release(e->stream);
    e->dact.release(e->stream);
    e->dshape.release(e->stream);
    e->dtshape.release(e->stream);
    if (e->graph) cudaGraphDestroy(e->graph);
    DBuf<double>* dbl[] = {&e->params, &e->wpad, &e->Z, &e->faces, &e->probe_pts, &e->pZ, &e->verts, &e->sx, &e->shint,
                           &e->sxp, &e->pvals, &e->prec_pt, &e->pend_pt[0], &e->pend_pt[1], &e->pool_hint,
                           &e->ckey_hint, &e->emit_hint, &e->s_verts, &e->shape_tab, &e->near_row, &e->Zi,
                           &e->Z2, &e->faces2};
    for (auto* b : dbl) b->release(e->stream);
    DBuf<uint64_t>* u64[] = {&e->table, &e->pool, &e->ckey, &e->slot, &e->slot2, &e->scratch, &e->outbox,
                             &e->hkeys, &e->hslot, &e->ss, &e->ssn, &e->sres, &e->pkeys, &e->pslot, &e->s_keys};
    for (auto* b : u64) b->release(e->stream);
    DBuf<int32_t>* i32[] = {&e->changed, &e->status, &e->status2, &e->canon_pos, &e->canon_pool, &e->X,
                            &e->f_items, &e->f_pool, &e->batch_pool, &e->local_idx, &e->queue, &e->cell_pool,
                            &e->cell_nv, &e->edge_nrefs, &e->edge_refs, &e->hstatus, &e->sact, &e->sdone,
                            &e->pool_vn, &e->pstatus, &e->emit_dup, &e->emit_pool, &e->prec_cand, &e->prec_k,
                            &e->pend_t[0], &e->pend_t[1], &e->pend_k[0], &e->pend_k[1], &e->val_buf, &e->s_nv,
                            &e->near_n, &e->near_flags, &e->near_id,
                            &e->probe_shape, &e->prec_s, &e->pend_s[0], &e->pend_s[1],
                            &e->s_enr, &e->s_refs};
    for (auto* b : i32) b->release(e->stream);
    e->pool_flags.release(e->stream);
    e->pool_voff.release(e->stream);
    e->pool_par.release(e->stream);
    e->emit_par.release(e->stream);
    e->queue_par.release(e->stream);
    e->blist.release(e->stream);
    e->ckey2.release(e->stream);
    e->changed2.release(e->stream);
    e->cell_voff.release(e->stream);
    e->edge_roff.release(e->stream);
    e->subdev.release(e->stream);
    e->ctr.release(e->stream);
    for (int i = 0; i < 6; i++) cudaEventDestroy(e->ev[i]);
    for (int i = 0; i < am_engine::kMarks; i++) if (e->tev[i]) cudaEventDestroy(e->tev[i]);
    if (e->h_hdr) cudaFreeHost(e->h_hdr);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->own_stream) cudaStreamDestroy(e->stream);
    if (e->stream2) cudaStreamDestroy(e->stream2);
    if (e->stream3) cudaStreamDestroy(e->stream3);
    delete e;
    return AM_OK;
}

extern "C" int am_engine_key_words(const am_engine* e) { return e ? e->KW : 0; }

// new weights for an engine built for the same architecture (same step / sub tables and
// parameter count): everything derived from the values is re-uploaded; buffers, TMA descriptors
// and captured graphs (which reference the buffers, not the values) stay valid
extern "C" int am_engine_load_params(am_engine* e, const double* h_params, int64_t n_params) {
    if (!e || !h_params) return fail(AM_ERR_ARG, "null argument");
    if (n_params != e->n_params)
        return fail(AM_ERR_ARG, "parameter count %lld does not match the engine's %lld", (long long)n_params,
                    (long long)e->n_params);
    CK(cudaStreamSynchronize(e->stream));
    return upload_params(e, h_params);
}

extern "C" int am_engine_set_shape_params(am_engine* e, const int64_t* h_param_idx, int64_t n_idx,
                                          const double* h_values) {
    if (!e || n_idx < 0 || (n_idx > 0 && (!h_param_idx || !h_values))) return fail(AM_ERR_ARG, "bad arguments");
    if (e->n_shapes < 2) return fail(AM_ERR_ARG, "engine was created for a single shape (n_shapes < 2)");
    for (int64_t j = 0; j < n_idx; j++)
        if (h_param_idx[j] < 0 || h_param_idx[j] >= e->n_params) return fail(AM_ERR_ARG, "parameter index out of range");
    e->shp_idx.assign(h_param_idx, h_param_idx + n_idx);
    e->shp_val.assign(h_values, h_values + (size_t)n_idx * e->n_shapes);
    std::vector<double> hp((size_t)e->n_params);
    CK(cudaMemcpyAsync(hp.data(), e->params.p, (size_t)e->n_params * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return upload_params(e, hp.data());
}

extern "C" int am_engine_set_shape(am_engine* e, int32_t shape) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    if (shape < 0 || shape >= e->n_shapes) return fail(AM_ERR_ARG, "shape %d out of range [0, %d)", shape, e->n_shapes);
    e->cur_shape = shape;
    return AM_OK;
}

extern "C" int am_engine_reset(am_engine* e) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    CK(cudaMemsetAsync(e->ctr.p, 0, C_N * sizeof(unsigned long long), e->stream));
    CK(cudaMemsetAsync(e->table.p, 0xff, e->tcap * sizeof(uint64_t), e->stream));
    CK(cudaStreamSynchronize(e->stream));
    memset(e->hctr, 0, sizeof e->hctr);
    e->t_compose = e->t_face = e->t_probe = e->flops = e->pflops = e->face_bytes = 0;
    e->n_comp_cells = e->n_face_cells = e->n_probes = 0;
    e->iters = 0;
    e->sh_have_hdr = false;
    e->sh_rounds = 0;
    for (double& t : e->t_bucket) t = 0;
    e->n_emit = e->n_canon = e->n_prec = e->n_new = e->n_timed = 0;
    return AM_OK;
}

// ----------------------------------------------------- compose / forward
// every hidden step for the items; C = 4 (cells) or 1 (points); n_dev null -> n_cap items
static int run_steps(am_engine* e, int C, double* Z, uint64_t* keys, const unsigned long long* key_off,
                     int32_t* changed, const double* pts, const unsigned long long* n_dev, int64_t n_cap,
                     size_t first = 0, const unsigned long long* zpar = nullptr, int64_t zstride = 0,
                     const unsigned long long* n_step = nullptr) {
    for (size_t s = first; s < e->sdev.size(); s++) {
        LayerLaunch L{};
        L.zpar = zpar;
        L.zstride = zstride;
        L.nj4 = e->gemm_nj4;
        L.st = e->sdev[s];
        L.Z = Z;
        L.keys = keys;
        L.key_off = key_off;
        L.changed = changed;
        L.pts = pts;
        L.n_dev = n_step ? n_step + s : n_dev;
        L.n_cap = n_cap;
        L.KW = e->KW;
        L.zs = e->zs;
        L.grid_cap = e->grid_cap;
        L.shape_w = e->shape_w;
        L.fp32 = e->fp32;
        if (L.st.flags & AM_STEP_FIRST) launch_input_step(L, C, e->stream);
        else launch_gemm_step(L, C, &e->tmW[s], e->tmV_ok[s] ? &e->tmV[s] : nullptr, e->stream,
                              e->narrow[s] ? &e->tmW96[s] : nullptr,
                              e->narrow[s] && e->tmV_ok[s] ? &e->tmV96[s] : nullptr);
    }
    CK(cudaGetLastError());
    return AM_OK;
}

// step 0 launch of the compose path (input step: the caller may fuse it with its gather)
static LayerLaunch first_step_launch(am_engine* e, uint64_t* keys, int32_t* changed, double* Z,
                                     const unsigned long long* n_dev, int64_t n_cap) {
    LayerLaunch L{};
    L.st = e->sdev[0];
    L.Z = Z; L.keys = keys; L.key_off = nullptr; L.changed = changed; L.pts = nullptr;
    L.n_dev = n_dev; L.n_cap = n_cap; L.KW = e->KW; L.zs = e->zs; L.grid_cap = e->grid_cap;
    L.shape_w = e->shape_w; L.fp32 = e->fp32;
    return L;
}

static bool gather_fuses_input(const am_engine* e) {
    const int ns = (int)e->sdev.size();
    return e->gather_input && ns > 0 && (e->sdev[0].flags & AM_STEP_FIRST) &&
           !(e->compose_fused && ns <= kMaxFusedSteps);
}

static int compose(am_engine* e, uint64_t* keys, int32_t* changed, double* Z, double* faces,
                   const unsigned long long* n_dev, int64_t n_cap, size_t first = 0) {
    const int ns = (int)e->sdev.size();
    if (e->compose_fused && ns <= kMaxFusedSteps) {
        FusedCompose* F = e->fused.get();
        for (int s = 0; s < ns; s++) {
            F->tmW[s] = e->tmW[s];
            F->tmV[s] = e->tmV_ok[s] ? e->tmV[s] : e->tmW[s];
            F->tmV_ok[s] = e->tmV_ok[s];
            F->st[s] = e->sdev[s];
        }
        LayerLaunch& L = F->L;
        L = LayerLaunch{};
        L.Z = Z; L.keys = keys; L.key_off = nullptr; L.changed = changed; L.pts = nullptr;
        L.n_dev = n_dev; L.n_cap = n_cap; L.KW = e->KW; L.zs = e->zs; L.grid_cap = 0;
        L.shape_w = e->shape_w; L.fp32 = e->fp32;
        F->nsteps = ns; F->faces = faces; F->subs = reinterpret_cast<const SubDev*>(e->subdev.p); F->n_subs = e->M;
        launch_compose_fused(*F, e->stream);
        CK(cudaGetLastError());
        return AM_OK;
    }
    RC(run_steps(e, 4, Z, keys, nullptr, changed, nullptr, n_dev, n_cap, first));
    launch_face_head_dev(Z, keys, faces, n_dev, n_cap, e->zs, e->KW, e->subdev.p, e->M, e->shape_w, e->fp32, e->stream);
    CK(cudaGetLastError());
    return AM_OK;
}

// composition of n explicit keys (in place: canonical keys, changed flags, Z rows, face planes):
// the narrow kernel in explicit-key mode where the net is narrow (one launch for every layer;
// bitwise equal to the per-layer path), else the per-layer kernels
static int compose_keys(am_engine* e, uint64_t* keys, int32_t* changed, double* Z, double* faces, int64_t n) {
    if (n <= 0) return AM_OK;
    if (e->narrow_fused && e->narrow_explicit && !e->narrow_check) {
        NarrowCompose N = *e->ncomp;
        for (int q = 0; q < N.nsteps; q++) N.st[q] = e->sdev[q];
        N.subs = reinterpret_cast<const SubDev*>(e->subdev.p);
        N.keys_in = keys; N.keys = keys; N.Z = Z; N.faces = faces; N.changed = changed;
        N.n_dev = nullptr; N.n_cap = n; N.KW = e->KW; N.zs = e->zs; N.shape_w = e->shape_w; N.fp32 = e->fp32;
        N.prefix = 0; N.snake = 0; N.near_fused = 0; N.canon_fused = 0; N.ctr = e->ctr.p;
        N.prof = e->dbg.p + 32;
        launch_compose_narrow(N, e->stream);
        CK(cudaGetLastError());
        return AM_OK;
    }
    return compose(e, keys, changed, Z, faces, nullptr, n);
}

static int forward(am_engine* e, const double* pts, double* vals, uint64_t* keys, const unsigned long long* key_off,
                   double* Zw, const unsigned long long* n_dev, int64_t n_cap) {
    if (e->narrow_fused && e->forward_narrow && !key_off) {
        // narrow plain nets: every layer + head in one launch (bitwise equal to the per-layer path)
        NarrowCompose& N = *e->ncomp;
        for (int q = 0; q < N.nsteps; q++) N.st[q] = e->sdev[q];
        N.subs = reinterpret_cast<const SubDev*>(e->subdev.p);
        N.KW = e->KW; N.shape_w = e->shape_w; N.fp32 = e->fp32;
        ForwardArgs F{pts, vals, keys, n_dev, n_cap};
        launch_forward_narrow(N, F, e->stream);
        CK(cudaGetLastError());
        return AM_OK;
    }
    RC(run_steps(e, 1, Zw, keys, key_off, nullptr, pts, n_dev, n_cap));
    launch_forward_head_dev(Zw, keys, key_off, vals, n_dev, n_cap, e->zs, e->KW, e->subdev.p, e->M, e->ensemble,
                            e->shape_w, e->fp32,
                            e->stream);
    CK(cudaGetLastError());
    return AM_OK;
}

// host-sized forward in chunks of the probe workspace
// shapes: per-point shape of a batch-of-shapes engine (device, may be null: the current shape)
static int forward_host(am_engine* e, const double* pts, int64_t n, double* vals, uint64_t* keys,
                        const int32_t* shapes = nullptr) {
    for (int64_t o = 0; o < n; o += e->PB) {
        int64_t m = std::min<int64_t>(e->PB, n - o);
        launch_zero_keys(keys + o * e->KW, nullptr, e->KW, m, e->shape_w, shapes ? shapes + o : nullptr, e->cur_shape,
                         e->stream);
        RC(forward(e, pts + o * 3, vals ? vals + o : nullptr, keys + o * e->KW, nullptr, e->pZ.p, nullptr, m));
    }
    return AM_OK;
}

// When the caller passed the legacy default stream (torch's default), the engine runs on a
// stream of its own: the caller's pending work that produced our device inputs must come
// first (the entry points end with a host sync, so outputs are complete on return).
static int join_caller(am_engine* e) {
    if (!e->own_stream) return AM_OK;   // caller's own stream: already ordered
    CK(cudaEventRecord(e->ev_join, cudaStreamLegacy));
    CK(cudaStreamWaitEvent(e->stream, e->ev_join, 0));
    return AM_OK;
}

extern "C" int am_forward_shapes(am_engine* e, const double* d_pts, const int32_t* d_shapes, int64_t n,
                                 double* d_vals, uint64_t* d_keys);
extern "C" int am_forward(am_engine* e, const double* d_pts, int64_t n, double* d_vals, uint64_t* d_keys) {
    return am_forward_shapes(e, d_pts, nullptr, n, d_vals, d_keys);
}
extern "C" int am_forward_shapes(am_engine* e, const double* d_pts, const int32_t* d_shapes, int64_t n,
                                 double* d_vals, uint64_t* d_keys) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    RC(join_caller(e));
    uint64_t* keys = d_keys;
    if (!keys) {
        CK(e->hkeys.reserve(n * e->KW, e->stream));
        keys = e->hkeys.p;
    }
    RC(forward_host(e, d_pts, n, d_vals, keys, d_shapes));
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}

extern "C" int am_affine_maps(am_engine* e, const uint64_t* d_keys, int64_t n, uint64_t* d_canon, double* d_planes,
                              double* d_faces) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    RC(join_caller(e));
    for (int64_t o = 0; o < n; o += e->B) {
        int64_t m = std::min<int64_t>(e->B, n - o);
        CK(cudaMemcpyAsync(e->ckey.p, d_keys + o * e->KW, m * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
        CK(cudaMemsetAsync(e->changed.p, 0, m * sizeof(int32_t), e->stream));
        RC(compose_keys(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, m));
        if (d_canon)
            CK(cudaMemcpyAsync(d_canon + o * e->KW, e->ckey.p, m * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
        if (d_planes)
            CK(cudaMemcpy2DAsync(d_planes + o * e->NB * 4, e->NB * 32, e->Z.p, e->zs * 32, e->NB * 32, m,
                                 cudaMemcpyDeviceToDevice, e->stream));
        if (d_faces)
            CK(cudaMemcpyAsync(d_faces + o * e->M * 4, e->faces.p, m * e->M * 32, cudaMemcpyDeviceToDevice, e->stream));
    }
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}

// ----------------------------------------------------------- iteration
static int launch_probe_stage(am_engine* e);
constexpr unsigned long long kProbeInGraph = 256;   // probes per host round that switch the stage into the graph
static int launch_iteration(am_engine* e) {
    cudaStream_t s = e->stream;
    unsigned long long* c = e->ctr.p;
    const int64_t B = e->B;
    HashSet H = hs(e);
    const bool tm = e->timing;
    IterState I;
    I.ctr = c; I.queue = e->queue.p; I.batch_pool = e->batch_pool.p; I.B = B;
    I.cap_pool = e->pool.n / e->KW; I.tcap = (long long)e->tcap;
    I.cap_cells = e->cell_pool.n; I.cap_verts = e->edge_nrefs.n; I.cap_refs = e->edge_refs.n;
    I.cap_outbox = e->P.world > 1 ? e->outbox.n / e->KW : 0;
    I.cap_pend = e->pend_t[0].n; I.cap_val = e->val_buf.n;
    I.emit_per_cell = emit_per_cell(); I.verts_per_cell = kVertsPerCell; I.refs_per_cell = kRefsPerCell;
    I.world = e->P.world;
    I.queue_par = e->prefix ? e->queue_par.p : nullptr;
    I.blist = e->blist.p;
    I.max_share = (int)e->sdev.size() - 1;
    I.max_cells = (long long)e->P.max_cells;
    I.cap_drop = e->defer ? 0 : 1;
    ProbeRecs R;
    R.cand = e->prec_cand.p; R.k = e->prec_k.p; R.pt = e->prec_pt.p;
    for (int q = 0; q < 2; q++) { R.pend_t[q] = e->pend_t[q].p; R.pend_k[q] = e->pend_k[q].p; R.pend_pt[q] = e->pend_pt[q].p; }
    const bool shapes = e->shape_w >= 0;
    R.s = shapes ? e->prec_s.p : nullptr;
    for (int q = 0; q < 2; q++) R.pend_s[q] = shapes ? e->pend_s[q].p : nullptr;
    R.cap_pend = e->pend_t[0].n;
    const bool multi = e->P.world > 1;
    // timing mode: marks 0..8 cut the iteration into contiguous stages (am_kernel_times)
    auto mark = [&](int i) { if (tm) cudaEventRecord(e->tev[i], s); };

    mark(0);
    launch_take(I, s);
    mark(1);
    const bool fuse_in = gather_fuses_input(e);
    if (e->narrow_fused) {
        if (tm) cudaEventRecord(e->ev[0], s);
        NarrowCompose& N = *e->ncomp;
        for (int q = 0; q < N.nsteps; q++) N.st[q] = e->sdev[q];
        N.subs = reinterpret_cast<const SubDev*>(e->subdev.p);
        N.pool = e->pool.p; N.pool_hint = e->pool_hint.p; N.queue = e->queue.p; N.ctr = c;
        N.batch_pool = e->batch_pool.p; N.canon_pos = e->canon_pos.p; N.ckey_hint = e->ckey_hint.p;
        N.Z = e->prefix ? e->Zi.p : e->Z.p; N.keys = e->ckey.p; N.faces = e->faces.p; N.changed = e->changed.p;
        N.prefix = e->prefix; N.zstride = e->B * e->zs * 4; N.pool_par = e->pool_par.p; N.blist = e->blist.p;
        N.near_fused = e->near_fused; N.NB = e->NB;
        N.snake = e->prefix && e->narrow_snake;
        N.canon_fused = e->canon_in_narrow;
        N.H = H; N.rank = e->P.rank; N.world = e->P.world; N.outbox = e->outbox.p; N.n_out = c + C_NOUT;
        N.status2 = e->status2.p; N.slot2 = e->slot2.p; N.canon_pool = e->canon_pool.p; N.f_items = e->f_items.p;
        N.f_pool = e->f_pool.p; N.max_cells = (long long)e->P.max_cells;
        N.near_n = e->near_n.p; N.near_flags = e->near_flags.p; N.near_id = e->near_id.p; N.near_row = e->near_row.p;
        N.near_cap = e->near_cap; N.near_reach = e->near_reach; N.tol_cell = e->P.tol_cell;
        N.tol_onplane = e->P.tol_onplane; N.probe_delta = e->P.probe_delta;
        for (int k = 0; k < 3; k++) { N.lo[k] = e->P.bbox_lo[k]; N.hi[k] = e->P.bbox_hi[k]; }
        N.n_dev = c + C_NR; N.n_cap = B; N.KW = e->KW; N.zs = e->zs; N.shape_w = e->shape_w; N.fp32 = e->fp32;
        N.prof = e->dbg.p + 32;
        launch_compose_narrow(N, s);
        CK(cudaGetLastError());
        if (e->narrow_check) {
            launch_gather_input(e->pool.p, e->pool_hint.p, e->queue.p, c, e->batch_pool.p, e->ckey_hint.p,
                                e->canon_pos.p, first_step_launch(e, e->ckey2.p, e->changed2.p, e->Z2.p, c + C_NR, B), s);
            RC(compose(e, e->ckey2.p, e->changed2.p, e->Z2.p, e->faces2.p, c + C_NR, B, 1));
            launch_narrow_check(e->Z.p, e->Z2.p, e->faces.p, e->faces2.p, e->ckey.p, e->ckey2.p, e->changed.p,
                                e->changed2.p, c + C_NR, B, e->NB, e->zs, e->KW, e->dbg.p, s);
        }
    } else if (fuse_in && e->prefix) {
        // prefix reuse on the per-step path: gather in bucket order + input step, parents' rows,
        // then each GEMM step over the items that need it (buckets f < s) and the heads
        if (tm) cudaEventRecord(e->ev[0], s);
        LayerLaunch L0 = first_step_launch(e, e->ckey.p, e->changed.p, e->Zi.p, c + C_NR, B);
        L0.zpar = c + C_ITER;
        L0.zstride = B * e->zs * 4;
        launch_gather_input(e->pool.p, e->pool_hint.p, e->queue.p, c, e->batch_pool.p, e->ckey_hint.p,
                            e->canon_pos.p, L0, s, e->blist.p, (int)e->sdev.size());
        PrefixRows R{};
        R.ctr = c;
        R.nb = (int)e->sdev.size();
        for (int q = 0; q < R.nb; q++) { R.row_off[q] = e->sdev[q].row_off; R.n_out[q] = e->sdev[q].n_out; }
        launch_prefix_rows(R, L0, e->batch_pool.p, e->pool_par.p, s);
        RC(run_steps(e, 4, e->Zi.p, e->ckey.p, nullptr, e->changed.p, nullptr, c + C_NR, B, 1, c + C_ITER, L0.zstride,
                     c + C_PRE0));
        launch_face_head_dev(e->Zi.p, e->ckey.p, e->faces.p, c + C_NR, B, e->zs, e->KW, e->subdev.p, e->M,
                             e->shape_w, e->fp32, s, c + C_ITER, L0.zstride);
        CK(cudaGetLastError());
    } else if (fuse_in) {
        if (tm) cudaEventRecord(e->ev[0], s);
        launch_gather_input(e->pool.p, e->pool_hint.p, e->queue.p, c, e->batch_pool.p, e->ckey_hint.p,
                            e->canon_pos.p, first_step_launch(e, e->ckey.p, e->changed.p, e->Z.p, c + C_NR, B), s);
    } else {
        launch_gather_batch(e->pool.p, e->pool_hint.p, e->queue.p, c, e->batch_pool.p, B, e->KW, e->ckey.p,
                            e->ckey_hint.p, e->changed.p, e->canon_pos.p, s);
        if (tm) cudaEventRecord(e->ev[0], s);
    }
    if (!e->narrow_fused && !(fuse_in && e->prefix))
        RC(compose(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, c + C_NR, B, fuse_in ? 1 : 0));
    if (tm) cudaEventRecord(e->ev[1], s);
    mark(2);
    if (e->narrow_fused && e->canon_in_narrow) {
        mark(3);   // done in k_compose_narrow's tile epilogue
    } else if (e->canon_fused) {
        launch_canon_frontier(H, e->ckey.p, e->changed.p, e->batch_pool.p, c + C_NR, B, e->P.rank, e->P.world,
                              e->outbox.p, c + C_NOUT, e->canon_pos.p, e->status2.p, e->slot2.p, e->canon_pool.p,
                              e->ckey_hint.p, e->f_items.p, e->f_pool.p, c, (long long)e->P.max_cells, s);
        mark(3);
    } else {
        launch_route_changed(e->ckey.p, e->changed.p, c + C_NR, B, e->KW, e->P.rank, e->P.world, e->X.p, c + C_NX,
                             e->outbox.p, c + C_NOUT, e->canon_pos.p, s);
        launch_hash_upsert(H, e->ckey.p, e->X.p, c + C_NX, B, e->status2.p, e->slot2.p, nullptr, 0u, e->canon_pool.p, nullptr, nullptr, e->ckey_hint.p, s);
        mark(3);
        launch_frontier(c + C_NR, B, e->changed.p, e->batch_pool.p, e->canon_pos.p, e->status2.p, e->canon_pool.p,
                        e->pool_flags.p, e->f_items.p, e->f_pool.p, c, (long long)e->P.max_cells, s);
    }
    FaceArgs a;
    a.Z = e->Z.p; a.faces = e->faces.p; a.keys = e->ckey.p; a.items = e->f_items.p; a.pool_idx = e->f_pool.p;
    a.hints = e->ckey_hint.p; a.emit_hint = e->emit_hint.p;
    a.n_dev = c + C_NF; a.n_cap = B;
    a.NB = e->NB; a.M = e->M; a.KW = e->KW; a.zs = e->zs; a.ensemble = e->ensemble;
    for (int k = 0; k < 3; k++) { a.lo[k] = e->P.bbox_lo[k]; a.hi[k] = e->P.bbox_hi[k]; }
    a.tol_cell = e->P.tol_cell; a.tol_weld = e->P.tol_weld; a.tol_onplane = e->P.tol_onplane;
    a.probe_delta = e->P.probe_delta;
    a.cell_pool = e->cell_pool.p; a.cell_nv = e->cell_nv.p; a.cell_voff = e->cell_voff.p; a.n_cells = c + C_CELLS;
    a.verts = e->verts.p; a.edge_nrefs = e->edge_nrefs.p; a.edge_roff = e->edge_roff.p; a.edge_refs = e->edge_refs.p;
    a.n_verts = c + C_VERTS; a.n_refs = c + C_REFS;
    a.cap_cells = e->cell_pool.n; a.cap_verts = e->edge_nrefs.n; a.cap_refs = e->edge_refs.n;
    a.cand = e->scratch.p; a.n_cand = c + C_NEMIT; a.cap_cand = e->E;
    a.probe_pts = e->probe_pts.p; a.n_probe = c + C_NPROBE; a.cap_probe = e->PB;
    a.overflow = c + C_OVF0;
    a.prec_cand = e->prec_cand.p; a.prec_k = e->prec_k.p; a.prec_pt = e->prec_pt.p; a.n_prec = c + C_NPREC;
    a.prec_s = shapes ? e->prec_s.p : nullptr; a.shape_w = e->shape_w;
    a.cap_prec = e->PR;
    a.val_buf = e->val_buf.p; a.n_val = c + C_NVAL; a.cap_val = e->val_buf.n;
    a.pool_vn = e->pool_vn.p; a.pool_voff = e->pool_voff.p;
    a.queue = e->defer ? e->queue.p : nullptr; a.q_tail = c + C_QTAIL; a.defer_min = e->defer_min;
    a.pool_flags = e->pool_flags.p; a.pool_hint = e->pool_hint.p;
    a.dbg = e->dbg.p;
    a.cursor = c + C_FCURSOR;
    a.near_cap = e->near_cap; a.near_n = e->near_n.p; a.near_flags = e->near_flags.p;
    a.near_id = e->near_id.p; a.near_row = e->near_row.p; a.near_by_item = e->near_fused ? 1 : 0;
    a.near_depth = e->near_depth;
    a.order = e->face_order ? e->f_order.p : nullptr; a.order_ctr = c + C_NHEAVY;
    a.tau_mult = e->tau_mult; a.near_reach = e->near_reach; a.max_attempts = e->max_attempts;
    a.tau_grow = e->tau_grow;
    a.zpar = nullptr; a.zstride = 0; a.emit_par = nullptr; a.queue_par = nullptr; a.nsteps = 0;
    a.fused_upsert = (e->face_upsert && !multi) ? 1 : 0;
    a.H = H; a.cand_status = e->status.p; a.cand_slot = e->slot.p; a.cand_dup = e->emit_dup.p;
    a.cand_pool = e->emit_pool.p; a.ins_queue = e->queue.p;
    if (e->prefix) {
        a.Z = e->Zi.p;
        a.zpar = c + C_ITER; a.zstride = e->B * e->zs * 4; a.emit_par = e->emit_par.p; a.queue_par = e->queue_par.p;
        a.nsteps = (int)e->sdev.size();
        for (int q = 0; q < a.nsteps; q++) a.step_end[q] = e->sdev[q].row_off + e->sdev[q].n_out;
    }
    if (tm) cudaEventRecord(e->ev[2], s);
    mark(4);
    if (!e->near_fused) launch_near(a, s);
    mark(5);
    launch_face(a, s);
    mark(6);
    if (tm) cudaEventRecord(e->ev[3], s);
    // flips: insert (local) and queue the new states
    if (multi) {
        launch_route_emitted(e->scratch.p, c + C_NEMIT, e->E, e->KW, e->P.rank, e->P.world, e->local_idx.p,
                             c + C_NLOCAL, e->outbox.p, c + C_NOUT, e->status.p, s);
        launch_hash_upsert(H, e->scratch.p, e->local_idx.p, c + C_NLOCAL, e->E, e->status.p, e->slot.p, e->emit_dup.p, 0u, e->emit_pool.p, e->queue.p, c + C_QTAIL, e->emit_hint.p, s, a.emit_par);
    } else if (!a.fused_upsert) {
        launch_hash_upsert(H, e->scratch.p, nullptr, c + C_NEMIT, e->E, e->status.p, e->slot.p, e->emit_dup.p, 0u, e->emit_pool.p, e->queue.p, c + C_QTAIL, e->emit_hint.p, s, a.emit_par);
    }
    mark(7);
    // probe records (this iteration's and the pending ones): drop / forward / keep pending
    // This iteration's exact probe evaluations.  Probe-heavy marches (wide nets, batches of
    // shapes) capture them as a conditional node of the iteration graph whose predicate
    // k_pend_finalize sets, so probe-found states join the next wave.  Marches with only a
    // handful of probes (configs[1]: 15) leave them to the host loop, which evaluates whatever
    // accumulated at each synchronisation point: the visited set does not depend on when a
    // probe's state is inserted, and the graph stays free of the conditional node's cost.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cs));
    const bool capturing = cs == cudaStreamCaptureStatusActive && e->probe_in_graph;
    cudaGraphConditionalHandle h{};
    if (capturing) {
        cudaGraph_t g0 = nullptr;
        CK(cudaStreamGetCaptureInfo_v3(s, &cs, nullptr, &g0, nullptr, nullptr, nullptr));
        CK(cudaGraphConditionalHandleCreate(&h, g0, 0, cudaGraphCondAssignDefault));
    }
    launch_probe_records(R, H, e->status.p, e->emit_dup.p, e->emit_pool.p, e->val_buf.p, c, e->PR, e->probe_pts.p,
                         shapes ? e->probe_shape.p : nullptr, e->PB, capturing ? &h : nullptr, s);
    if (capturing) {
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t* deps = nullptr;
        const cudaGraphEdgeData* ed = nullptr;
        size_t nd = 0;
        unsigned long long cid = 0;
        CK(cudaStreamGetCaptureInfo_v3(s, &cs, &cid, &g, &deps, &ed, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CK(cudaGraphAddNode(&cn, g, deps, nd, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(e->stream2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        const unsigned long long before = g_launch_count;
        e->stream = e->stream2;
        int rc = launch_probe_stage(e);
        e->stream = s;
        e->cond_kernels = g_launch_count - before;
        cudaGraph_t bout = nullptr;
        cudaError_t ce = cudaStreamEndCapture(e->stream2, &bout);
        RC(rc);
        CK(ce);
        CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
    }
    if (tm) cudaEventRecord(e->ev[4], s);
    mark(8);
    CK(cudaGetLastError());
    return AM_OK;
}

// Exact forward evaluation of the probe points this iteration left (reference
// marching.py:271-276) and insertion of their states: launches only, on e->stream.  Inside the
// captured iteration graph it is the body of a conditional node (IF probes > 0): after probe
// validation most iterations have none, and the ~10 launches of the stage are then skipped.
static int launch_probe_stage(am_engine* e) {
    cudaStream_t s = e->stream;
    unsigned long long* c = e->ctr.p;
    const bool shapes = e->shape_w >= 0;
    const bool multi = e->P.world > 1;
    HashSet H = hs(e);
    launch_zero_keys(e->pkeys.p, c + C_NPROBE, e->KW, e->PB, e->shape_w, shapes ? e->probe_shape.p : nullptr, 0, s);
    e->grid_cap = 2;   // a small persistent grid per layer
    int frc = forward(e, e->probe_pts.p, nullptr, e->pkeys.p, nullptr, e->pZ.p, c + C_NPROBE, e->PB);
    e->grid_cap = 0;
    RC(frc);
    if (multi) {
        CK(cudaMemsetAsync(c + C_NPLOCAL, 0, sizeof(unsigned long long), s));
        launch_route_emitted(e->pkeys.p, c + C_NPROBE, e->PB, e->KW, e->P.rank, e->P.world, e->local_idx.p,
                             c + C_NPLOCAL, e->outbox.p, c + C_NOUT, nullptr, s);
        launch_hash_upsert(H, e->pkeys.p, e->local_idx.p, c + C_NPLOCAL, e->PB, e->pstatus.p, e->pslot.p, nullptr, 0u, nullptr, e->queue.p, c + C_QTAIL, nullptr, s);
    } else {
        launch_hash_upsert(H, e->pkeys.p, nullptr, c + C_NPROBE, e->PB, e->pstatus.p, e->pslot.p, nullptr, 0u, nullptr, e->queue.p, c + C_QTAIL, nullptr, s);
    }
    launch_probe_done(c, e->PB, s);
    CK(cudaGetLastError());
    return AM_OK;
}

// the probe stage run from the host (timing mode after every iteration; and whenever probes are
// still waiting at a host synchronisation point, e.g. more than one buffer's worth)
static int probe_flush(am_engine* e) {
    RC(ensure_hash(e, e->PB));
    if (e->timing) cudaEventRecord(e->ev[5], e->stream);
    RC(launch_probe_stage(e));
    if (e->timing) {
        cudaEventRecord(e->ev[4], e->stream);
        CK(cudaEventSynchronize(e->ev[4]));
        float t = 0;
        cudaEventElapsedTime(&t, e->ev[5], e->ev[4]);
        e->t_probe += t;
        e->t_bucket[8] += t;
        const double nP = (double)std::min<unsigned long long>(e->hctr[C_NPROBE], (unsigned long long)e->PB);
        e->pflops += e->flops_per_point * nP;
        e->n_probes += nP;
    }
    return AM_OK;
}

static int capture(am_engine* e) {
    if (e->gexec) { cudaGraphExecDestroy(e->gexec); e->gexec = nullptr; }
    if (e->graph) { cudaGraphDestroy(e->graph); e->graph = nullptr; }
    unsigned long long before = g_launch_count;
    CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    int rc = AM_OK;
    if (e->iter_gate) {
        // gate kernel + IF node whose body is the iteration (captured on stream3)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaGraph_t g0 = nullptr;
        CK(cudaStreamGetCaptureInfo_v3(e->stream, &cs, nullptr, &g0, nullptr, nullptr, nullptr));
        cudaGraphConditionalHandle hg{};
        CK(cudaGraphConditionalHandleCreate(&hg, g0, 0, cudaGraphCondAssignDefault));
        launch_iter_gate(e->ctr.p, hg, e->probe_in_graph ? 1 : 0, e->stream);
        CK(cudaGetLastError());
        const cudaGraphNode_t* deps = nullptr;
        const cudaGraphEdgeData* ed = nullptr;
        size_t nd = 0;
        cudaGraph_t gt = nullptr;
        CK(cudaStreamGetCaptureInfo_v3(e->stream, &cs, nullptr, &gt, &deps, &ed, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hg;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CK(cudaGraphAddNode(&cn, gt, deps, nd, &cp));
        CK(cudaStreamBeginCaptureToGraph(e->stream3, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        cudaStream_t s0 = e->stream;
        e->stream = e->stream3;
        const unsigned long long b0 = g_launch_count;
        rc = launch_iteration(e);
        e->gate_kernels = g_launch_count - b0;
        e->stream = s0;
        cudaGraph_t bout = nullptr;
        cudaError_t be = cudaStreamEndCapture(e->stream3, &bout);
        if (!rc && be != cudaSuccess) rc = fail(AM_ERR_CUDA, "gated iteration capture: %s", cudaGetErrorString(be));
        if (!rc) CK(cudaStreamUpdateCaptureDependencies(e->stream, &cn, 1, cudaStreamSetCaptureDependencies));
    } else {
        rc = launch_iteration(e);
    }
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
    if (rc) { if (g) cudaGraphDestroy(g); return rc; }
    CK(ce);
    e->graph = g;
    e->graph_kernels = g_launch_count - before - e->cond_kernels;   // the conditional body counts per run
    g_launch_count = before;   // captured, not launched
    CK(cudaGraphInstantiate(&e->gexec, e->graph, 0));
    e->graph_valid = true;
    return AM_OK;
}

// make room for `iters` more iterations: the key pool / hash set get one iteration's worst case
// (the unit k_take's capacity guard checks before taking a batch) plus the pool growth per cell
// observed so far (x2, >= 8 keys) for the round's other iterations -- an under-estimate only makes
// the guard take smaller batches (or stall until the next host round grows the buffers), never
// overflows; the worst case for every iteration of a round would reserve ~130 keys per cell
static int ensure_iter_room(am_engine* e, int iters, bool sync = true, int64_t extra_keys = 0) {
    if (sync) RC(sync_counters(e));
    const int64_t per_cell = 1 + emit_per_cell();
    const int64_t np = (int64_t)e->hctr[C_POOL], nc = (int64_t)e->hctr[C_CELLS];
    const int64_t g = nc > 0 ? std::min<int64_t>(per_cell, std::max<int64_t>(8, 2 * ((np + nc - 1) / nc))) : 16;
    RC(ensure_hash(e, e->B * per_cell + (int64_t)(iters - 1) * e->B * g + extra_keys, sync));
    // per-vertex buffers likewise: one worst-case iteration (kVertsPerCell per cell) + observed
    // vertices per cell (x2, >= 8) for the rest
    const int64_t nv = (int64_t)e->hctr[C_VERTS];
    const int64_t gv = nc > 0 ? std::min<int64_t>(kVertsPerCell, std::max<int64_t>(8, 2 * ((nv + nc - 1) / nc))) : 16;
    const int64_t vcells = e->B + ((int64_t)(iters - 1) * e->B * gv + kVertsPerCell - 1) / kVertsPerCell;
    RC(ensure_results(e, (int64_t)iters * e->B, vcells, sync));
    return AM_OK;
}

static int timed_iteration(am_engine* e) {
    const unsigned long long pool0 = e->hctr[C_POOL];
    RC(launch_iteration(e));
    CK(cudaEventSynchronize(e->tev[am_engine::kMarks - 1]));
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, e->ev[0], e->ev[1]);
    cudaEventElapsedTime(&b, e->ev[2], e->ev[3]);
    cudaEventElapsedTime(&c, e->ev[3], e->ev[4]);
    for (int i = 0; i + 1 < am_engine::kMarks; i++) {
        float t = 0;
        cudaEventElapsedTime(&t, e->tev[i], e->tev[i + 1]);
        e->t_bucket[i] += t;
    }
    RC(sync_counters(e));
    e->n_emit += (double)e->hctr[C_NEMIT];
    e->n_canon += (double)e->hctr[C_NX];
    e->n_prec += (double)e->hctr[C_NPREC];
    e->n_new += (double)(e->hctr[C_POOL] - pool0);
    e->n_timed += 1;
    if (e->hctr[C_NPROBE]) RC(probe_flush(e));
    e->t_compose += a;
    e->t_face += b;
    double nR = (double)e->hctr[C_NR], nF = (double)e->hctr[C_NF];
    e->flops += e->flops_per_cell * nR;
    e->n_comp_cells += nR;
    e->n_face_cells += nF;
    if (getenv("AM_TRACE_ITERS")) {
        // AM_FACE_STATS builds: slowest face cell of the iteration (cycles) and full-path cells so far
        unsigned long long dbg[64];
        CK(cudaMemcpy(dbg, e->dbg.p, sizeof dbg, cudaMemcpyDeviceToHost));
        fprintf(stderr, "iter %lld nR %.0f nF %.0f compose %.1f us face %.1f us probe-stage %.1f us | max cell %llu cyc, "
                "full-path %llu streamed %llu | emit %llu prec %llu pend %llu\n", (long long)e->hctr[C_ITER], nR, nF,
                a * 1e3, b * 1e3, c * 1e3, dbg[8], dbg[27], dbg[26], e->hctr[C_NEMIT], e->hctr[C_NPREC],
                e->hctr[C_NPEND]);
        CK(cudaMemset(e->dbg.p + 8, 0, 8));
    }
    e->face_bytes += nF * (e->NB * 32.0 + e->M * 32.0 + e->KW * 8.0);
    return AM_OK;
}

// kernels launched by k replays of the iteration graph of which `ran` passed the gate
static unsigned long long replay_kernels(const am_engine* e, int k, unsigned long long ran) {
    if (!e->iter_gate) return (unsigned long long)k * e->graph_kernels;
    return (unsigned long long)k + ran * (e->graph_kernels - 1);
}

// run up to `max_iters` iterations (graph replays), stopping when the queue drains
static int run_iterations(am_engine* e, int64_t max_iters, int64_t* done) {
    int64_t n = 0;
    bool fresh = false;   // host counters current (the GPU has been idle since they were read)
    while (n < max_iters) {
        if (!fresh) RC(sync_counters(e));
        fresh = false;
        if (e->hctr[C_OVF1]) return fail(AM_ERR_OVERFLOW, "output capacity overflow (%llu events)", e->hctr[C_OVF1]);
        if (e->hctr[C_QHEAD] >= e->hctr[C_QTAIL] && e->hctr[C_NPEND] == 0) {
            if (e->hctr[C_NPROBE] == 0) break;
            RC(probe_flush(e));
            continue;
        }
        int k = (int)std::min<int64_t>(e->graph_batch, max_iters - n);
        // the tail of a march (a few dozen queued cells) ends within a few iterations: a short
        // replay batch there leaves at most 7 empty iterations (~19 us each) instead of up to 31
        const int64_t queued = (int64_t)(e->hctr[C_QTAIL] - e->hctr[C_QHEAD]);
        if (n > 0 && queued < e->tail_queue) k = std::min(k, e->tail_batch);
        RC(ensure_iter_room(e, k + 1, false));   // counters read above; nothing ran since
        if (e->timing) {
            for (int i = 0; i < k; i++) RC(timed_iteration(e));
        } else {
            if (!e->graph_valid) RC(capture(e));
            const unsigned long long fl0 = e->hctr[C_NFLUSH], gt0 = e->hctr[C_GATED];
            for (int i = 0; i < k; i++) CK(cudaGraphLaunch(e->gexec, e->stream));
            RC(sync_counters(e));
            g_launch_count += replay_kernels(e, k, e->hctr[C_GATED] - gt0);
            g_launch_count += (e->hctr[C_NFLUSH] - fl0) * e->cond_kernels;
        }
        n += k;
        if (e->timing) RC(sync_counters(e));
        fresh = true;
        if (e->hctr[C_STALL]) e->graph_valid = false;  // guard fired: the next round grows buffers
        if (e->hctr[C_NPROBE]) {
            // many probes per batch of iterations: evaluate them inside the graph from now on
            if (!e->probe_in_graph && e->probe_auto && e->hctr[C_NPROBE] > kProbeInGraph) {
                e->probe_in_graph = true;
                e->graph_valid = false;
            }
            RC(probe_flush(e));
            RC(sync_counters(e));
        }
    }
    if (!fresh) RC(sync_counters(e));
    e->iters = (int64_t)e->hctr[C_ITER];
    if (done) *done = n;
    return AM_OK;
}

// --------------------------------------------------------------- marching
// insert host-sized keys and queue the new ones
static int push_keys(am_engine* e, const uint64_t* d_keys, int64_t n, const double* d_hints = nullptr) {
    if (n <= 0) return AM_OK;
    RC(ensure_hash(e, n));
    CK(e->hstatus.reserve(n, e->stream));
    CK(e->hslot.reserve(n, e->stream));
    HashSet H = hs(e);
    if (e->P.world > 1) {   // keep only the states this rank owns
        CK(e->local_idx.reserve(n, e->stream));
        CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, 8, e->stream));
        launch_filter_owned(d_keys, n, e->KW, e->P.rank, e->P.world, e->local_idx.p, e->ctr.p + C_LIST, e->stream);
        launch_hash_upsert(H, d_keys, e->local_idx.p, e->ctr.p + C_LIST, n, e->hstatus.p, e->hslot.p, nullptr, 0u, nullptr, e->queue.p, e->ctr.p + C_QTAIL, d_hints, e->stream);
    } else {
        launch_hash_upsert(H, d_keys, nullptr, nullptr, n, e->hstatus.p, e->hslot.p, nullptr, 0u, nullptr, e->queue.p, e->ctr.p + C_QTAIL, d_hints, e->stream);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}

extern "C" int am_push_candidates(am_engine* e, const uint64_t* d_keys, int64_t n) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    RC(join_caller(e));
    return push_keys(e, d_keys, n);
}

extern "C" int am_wave(am_engine* e, int64_t* h_new_cells) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    unsigned long long before = e->hctr[C_TOTAL];
    int64_t done = 0;
    int saved = e->graph_batch;
    e->graph_batch = 1;
    int rc = run_iterations(e, 1, &done);
    e->graph_batch = saved;
    RC(rc);
    if (h_new_cells) *h_new_cells = (int64_t)(e->hctr[C_TOTAL] - before);
    return AM_OK;
}

extern "C" int am_run(am_engine* e, int64_t* h_waves) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(run_iterations(e, INT64_MAX, nullptr));
    if (h_waves) *h_waves = e->iters;
    return AM_OK;
}

extern "C" int am_queue_size(am_engine* e, int64_t* h_n) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    // outstanding work: queued states, pending probe records and unevaluated probes (the
    // sharded loop terminates when this is zero on every rank)
    *h_n = (int64_t)(e->hctr[C_QTAIL] - e->hctr[C_QHEAD]) + (int64_t)e->hctr[C_NPEND] + (int64_t)e->hctr[C_NPROBE];
    return AM_OK;
}

extern "C" int am_outbox_counts(am_engine* e, int64_t* h_total) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    *h_total = (int64_t)e->hctr[C_NOUT];
    return AM_OK;
}

// move the outbox to d_out grouped by owner rank (h_counts[world] keys per owner) and clear it
extern "C" int am_outbox_take(am_engine* e, uint64_t* d_out, int64_t* h_counts) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(join_caller(e));
    RC(sync_counters(e));
    const int world = e->P.world, KW = e->KW;
    int64_t n = (int64_t)e->hctr[C_NOUT];
    for (int r = 0; r < world; r++) h_counts[r] = 0;
    if (n > 0) {
        if (world > 64) return fail(AM_ERR_ARG, "world size %d > 64", world);
        DBuf<int32_t> own;
        DBuf<unsigned long long> cnt;
        CK(own.reserve(n, e->stream));
        CK(cnt.reserve(2 * world, e->stream));
        CK(cudaMemsetAsync(cnt.p, 0, 2 * world * sizeof(unsigned long long), e->stream));
        launch_outbox_group(e->outbox.p, n, KW, world, own.p, cnt.p, cnt.p + world, d_out, e->stream);
        std::vector<unsigned long long> hc(world);
        CK(cudaMemcpyAsync(hc.data(), cnt.p, world * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        for (int r = 0; r < world; r++) h_counts[r] = (int64_t)hc[r];
        own.release(e->stream);
        cnt.release(e->stream);
    }
    RC(set_counter(e, C_NOUT, 0));
    return AM_OK;
}

// ------------------------------------------------------------ trigger schemes
// sgd (scheme 0) and sphere tracing (scheme 1) from n start points, all in lockstep on the device
// (reference seeding.py:35-77); the host looks at the running count every 8 steps only.
extern "C" int am_trace(am_engine* e, const double* d_x0, int64_t n, int scheme, double seed_tol, int max_iters,
                        double param, double escape, double* d_out, int32_t* d_status, int32_t* d_iters) {
    if (!e || n < 0 || (scheme != 0 && scheme != 1) || max_iters < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    if (n > e->B || n > e->PB) return fail(AM_ERR_ARG, "am_trace: at most %lld start points per call",
                                           (long long)std::min(e->B, e->PB));
    RC(join_caller(e));
    cudaStream_t s = e->stream;
    const int KW = e->KW;
    CK(e->tx.reserve(n * 3, s)); CK(e->txn.reserve(n * 3, s));
    CK(e->tf.reserve(n, s)); CK(e->tfn.reserve(n, s)); CK(e->tcur.reserve(n, s));
    CK(e->tk.reserve(n * KW, s)); CK(e->tkn.reserve(n * KW, s));
    CK(e->trun.reserve(1, s));
    const int bw_branch = e->ensemble ? (e->NB + 63) / 64 : -1;
    launch_trace_init(n, d_x0, e->tx.p, e->tcur.p, param, d_status, d_iters, s);
    auto grad = [&]() -> int {   // face planes of the current states -> e->faces
        CK(cudaMemcpyAsync(e->ckey.p, e->tk.p, n * KW * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemsetAsync(e->changed.p, 0, n * sizeof(int32_t), s));
        return compose_keys(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, n);
    };
    if (scheme == 0) RC(forward_host(e, e->tx.p, n, e->tf.p, e->tk.p));
    for (int it = 0; it <= max_iters; it++) {
        CK(cudaMemsetAsync(e->trun.p, 0, sizeof(unsigned long long), s));
        if (scheme == 0) {
            launch_sgd_check(n, e->tf.p, d_status, d_iters, it, seed_tol, e->trun.p, s);
        } else {
            RC(forward_host(e, e->tx.p, n, e->tf.p, e->tk.p));
            launch_sphere_check(n, e->tx.p, e->tf.p, d_status, d_iters, it, seed_tol, escape, e->trun.p, s);
        }
        if (it % 8 == 7) {
            unsigned long long running = 0;
            CK(cudaMemcpyAsync(&running, e->trun.p, sizeof running, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (!running) break;
        }
        RC(grad());
        if (scheme == 0) {
            launch_sgd_propose(n, e->tx.p, e->tf.p, e->faces.p, e->ckey.p, KW, e->M, bw_branch, e->tcur.p, d_status,
                               e->txn.p, s);
            RC(forward_host(e, e->txn.p, n, e->tfn.p, e->tkn.p));
            launch_sgd_accept(n, e->tx.p, e->tf.p, e->tk.p, e->txn.p, e->tfn.p, e->tkn.p, KW, e->tcur.p, d_status, s);
        } else {
            launch_sphere_step(n, e->tx.p, e->tf.p, e->faces.p, e->ckey.p, KW, e->M, bw_branch, param, d_status, s);
        }
        CK(cudaGetLastError());
    }
    launch_trace_finish(n, e->tx.p, d_status, d_out, s);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return AM_OK;
}

// ------------------------------------------------------------ sharded rounds
// One round of the multi-GPU march = am_shard_iterate (the round's only host synchronisation)
// + am_shard_pack + the caller's all-to-all + am_shard_absorb; see include/am_b200.h.
static int shard_hdr_rows(const am_engine* e) { return (kHdrWords + e->KW - 1) / e->KW; }

extern "C" int am_shard_rows(am_engine* e, int64_t cap) {
    if (!e || cap < 1) return fail(AM_ERR_ARG, "bad arguments");
    return shard_hdr_rows(e) + (int)std::min<int64_t>(cap, INT32_MAX / 2);
}

extern "C" int am_shard_iterate(am_engine* e, int iters, int64_t cap, int64_t* h_out) {
    if (!e || iters < 0 || cap < 1 || !h_out) return fail(AM_ERR_ARG, "bad arguments");
    const int world = e->P.world;
    RC(sync_counters(e));   // also completes the previous absorb's header copy
    if (e->hctr[C_OVF1]) return fail(AM_ERR_OVERFLOW, "output capacity overflow (%llu events)", e->hctr[C_OVF1]);
    int64_t done = 0, cap_next = cap, visited = 0, capped = 0;
    if (e->sh_have_hdr) {
        bool idle = true;
        uint64_t demand = 0;
        for (int r = 0; r < world; r++) {
            const uint64_t* h = e->h_hdr + (size_t)r * kHdrWords;
            if (h[7] != 1) return fail(AM_ERR_ARG, "exchange header of rank %d missing", r);
            if (h[1] || h[2] || h[3]) idle = false;
            demand = std::max<uint64_t>(demand, h[4]);
            visited += (int64_t)h[5];
            capped |= h[6] ? 1 : 0;
        }
        done = idle ? 1 : 0;
        // the next exchange must take every rank's largest per-destination demand (identical on
        // every rank: every rank sees every header); grows in powers of two, never shrinks
        while ((uint64_t)cap_next < demand && cap_next < (int64_t)1 << 24) cap_next <<= 1;
    }
    h_out[0] = done;
    h_out[1] = cap_next;
    h_out[2] = visited;
    h_out[3] = capped;
    if (done) return AM_OK;
    // local iterations: capacity from the counters just read (no further synchronisation), plus
    // room for the keys the coming exchange can deliver
    const bool queued = e->hctr[C_QHEAD] < e->hctr[C_QTAIL] || e->hctr[C_NPEND] || e->hctr[C_NPROBE];
    const int k = queued ? iters : 0;
    RC(ensure_iter_room(e, k + 1, false, (int64_t)world * cap_next + e->PB));
    if (k > 0) {
        // the exact probe evaluations queued by the previous round run first (device-side counts:
        // no extra synchronisation); a conditional probe node in every iteration would cut the
        // PDL chain of each one (AM_SHARD_PROBE_IN_GRAPH=1 restores it)
        if (e->shard_probe_in_graph) {
            if (!e->probe_in_graph) { e->probe_in_graph = true; e->graph_valid = false; }
        } else if (e->hctr[C_NPROBE] && !e->probe_in_graph) {
            RC(launch_probe_stage(e));
        }
        if (!e->graph_valid) RC(capture(e));
        for (int i = 0; i < k; i++) CK(cudaGraphLaunch(e->gexec, e->stream));
        g_launch_count += (unsigned long long)k * e->graph_kernels;   // gated: an upper bound (no sync here)
    }
    return AM_OK;
}

extern "C" int am_shard_pack(am_engine* e, uint64_t* d_send, int64_t cap) {
    if (!e || !d_send || cap < 1) return fail(AM_ERR_ARG, "bad arguments");
    const int world = e->P.world;
    const int64_t max_keys = e->outbox.n / e->KW;
    CK(e->sh_rest.reserve(std::max<int64_t>(e->outbox.n, e->KW), e->stream));
    CK(e->sh_cnt.reserve(world + 1, e->stream));
    launch_shard_pack(e->outbox.p, e->ctr.p, e->KW, world, cap, shard_hdr_rows(e), d_send, e->sh_rest.p, e->sh_cnt.p,
                      max_keys, e->stream);
    CK(cudaGetLastError());
    e->sh_rounds++;
    return AM_OK;
}

extern "C" int am_shard_absorb(am_engine* e, const uint64_t* d_recv, int64_t cap) {
    if (!e || !d_recv || cap < 1) return fail(AM_ERR_ARG, "bad arguments");
    const int world = e->P.world, KW = e->KW, hr = shard_hdr_rows(e);
    const int64_t rows = hr + cap;
    if (!e->h_hdr) CK(cudaMallocHost(&e->h_hdr, (size_t)64 * kHdrWords * sizeof(uint64_t)));
    if (world > 64) return fail(AM_ERR_ARG, "world size %d > 64", world);
    CK(e->sh_idx.reserve((int64_t)world * cap, e->stream));
    CK(e->hstatus.reserve((int64_t)world * rows, e->stream));   // upsert outputs are indexed by recv row
    CK(e->hslot.reserve((int64_t)world * rows, e->stream));
    // room for world * cap keys was reserved by am_shard_iterate
    launch_shard_index(d_recv, KW, world, cap, hr, e->sh_idx.p, e->ctr.p + C_LIST, e->stream);
    HashSet H = hs(e);
    launch_hash_upsert(H, d_recv, e->sh_idx.p, e->ctr.p + C_LIST, (int64_t)world * cap, e->hstatus.p, e->hslot.p,
                       nullptr, 0u, nullptr, e->queue.p, e->ctr.p + C_QTAIL, nullptr, e->stream);
    CK(cudaMemcpy2DAsync(e->h_hdr, kHdrWords * sizeof(uint64_t), d_recv, (size_t)rows * KW * sizeof(uint64_t),
                         kHdrWords * sizeof(uint64_t), world, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaGetLastError());
    e->sh_have_hdr = true;
    return AM_OK;
}

// h_out[6]: rounds, host synchronisations, iterations, pool entries, visited cells, outbox
extern "C" int am_shard_stats(am_engine* e, int64_t* h_out) {
    if (!e || !h_out) return fail(AM_ERR_ARG, "bad arguments");
    h_out[0] = (int64_t)e->sh_rounds;
    h_out[1] = (int64_t)e->n_syncs;
    h_out[2] = (int64_t)e->hctr[C_ITER];
    h_out[3] = (int64_t)e->hctr[C_POOL];
    h_out[4] = (int64_t)e->hctr[C_TOTAL];
    h_out[5] = (int64_t)e->hctr[C_NOUT];
    return AM_OK;
}

// ------------------------------------------------------------------ seeding
// reference marching.py:201-213 (_refine_seed_state), batched over seeds
extern "C" int am_seed_shapes(am_engine* e, const double* d_pts, const int32_t* d_shapes, int64_t n);
extern "C" int am_seed(am_engine* e, const double* d_pts, int64_t n) { return am_seed_shapes(e, d_pts, nullptr, n); }
extern "C" int am_seed_shapes(am_engine* e, const double* d_pts, const int32_t* d_shapes, int64_t n) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    RC(join_caller(e));
    if (n > e->B) return fail(AM_ERR_ARG, "too many seeds for one batch (%lld > %lld)", (long long)n, (long long)e->B);
    cudaStream_t s = e->stream;
    int KW = e->KW;
    CK(e->sx.reserve(n * 3, s));
    CK(e->sxp.reserve(n * 3, s));
    CK(e->ss.reserve(n * KW, s));
    CK(e->ssn.reserve(n * KW, s));
    CK(e->sres.reserve(n * KW, s));
    CK(e->sact.reserve(n, s));
    CK(e->sdone.reserve(n, s));
    CK(cudaMemcpyAsync(e->sx.p, d_pts, n * 24, cudaMemcpyDeviceToDevice, s));
    const int32_t* shp = nullptr;
    if (d_shapes) {
        CK(e->sshape.reserve(n, s));
        CK(cudaMemcpyAsync(e->sshape.p, d_shapes, n * 4, cudaMemcpyDeviceToDevice, s));
        shp = e->sshape.p;
    }
    CK(e->shint.reserve(n * 4, s));
    double ext = 0.0;
    for (int k = 0; k < 3; k++) ext = std::max(ext, e->P.bbox_hi[k] - e->P.bbox_lo[k]);
    // the refinement (3 project / re-evaluate rounds + the final composition) is a fixed
    // sequence of ~50 small launches: captured once per (n, buffers) and replayed
    auto body = [&]() -> int {
        RC(forward_host(e, e->sx.p, n, nullptr, e->ss.p, shp));
        CK(cudaMemsetAsync(e->sact.p, 1, n * 4, s));   // active: any non-zero word
        for (int it = 0; it < 3; it++) {
            CK(cudaMemcpyAsync(e->ckey.p, e->ss.p, n * KW * 8, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemsetAsync(e->changed.p, 0, n * 4, s));
            RC(compose_keys(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, n));
            launch_seed_project(e->sx.p, e->faces.p, e->ckey.p, KW, e->M, e->ensemble, n, e->sact.p, e->sxp.p,
                                e->sdone.p, s);
            launch_seed_check(nullptr, e->ckey.p, KW, n, e->sact.p, nullptr, nullptr, nullptr, e->sres.p, e->sdone.p, s);
            RC(forward_host(e, e->sxp.p, n, nullptr, e->ssn.p, shp));
            launch_seed_check(e->ssn.p, e->ckey.p, KW, n, e->sact.p, e->sx.p, e->sxp.p, e->ss.p, e->sres.p, nullptr, s);
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(e->ckey.p, e->ss.p, n * KW * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemsetAsync(e->changed.p, 0, n * 4, s));
        RC(compose_keys(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, n));
        launch_seed_check(nullptr, e->ckey.p, KW, n, e->sact.p, nullptr, nullptr, nullptr, e->sres.p, nullptr, s);
        // the seed point (inside the seed's cell, on the surface up to seed_tol) is the face
        // solver's hint, with a small initial reach that the solver widens as needed
        launch_point_hints(e->sx.p, n, ext / 256.0, e->shint.p, s);
        CK(cudaGetLastError());
        return AM_OK;
    };
    std::vector<const void*> ptrs = {e->sx.p, e->sxp.p, e->ss.p, e->ssn.p, e->sres.p, e->sact.p, e->sdone.p,
                                     e->ckey.p, e->changed.p, e->Z.p, e->faces.p, e->pZ.p, e->shint.p, shp};
    if (!e->sgexec || e->sg_n != n || e->sg_shape != (shp ? -2 : e->cur_shape) || e->sg_ptrs != ptrs) {
        if (e->sgexec) { cudaGraphExecDestroy(e->sgexec); e->sgexec = nullptr; }
        unsigned long long before = g_launch_count;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int rc = body();
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        CK(ce);
        e->sg_kernels = g_launch_count - before;
        g_launch_count = before;
        cudaError_t ie = cudaGraphInstantiate(&e->sgexec, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
        e->sg_n = n; e->sg_shape = shp ? -2 : e->cur_shape; e->sg_ptrs = ptrs;
    }
    CK(cudaGraphLaunch(e->sgexec, s));
    g_launch_count += e->sg_kernels;
    return push_keys(e, e->sres.p, n, e->shint.p);
}

// batched bisection between sign-opposite samples (reference seeding.py:84-112)
extern "C" int am_dichotomy_shapes(am_engine* e, const double* d_xpos, const double* d_xneg, const int32_t* d_shapes,
                                   int64_t n, double eps, double seed_tol, int max_iters, double* d_out);
extern "C" int am_dichotomy(am_engine* e, const double* d_xpos, const double* d_xneg, int64_t n, double eps,
                            double seed_tol, int max_iters, double* d_out) {
    return am_dichotomy_shapes(e, d_xpos, d_xneg, nullptr, n, eps, seed_tol, max_iters, d_out);
}
extern "C" int am_dichotomy_shapes(am_engine* e, const double* d_xpos, const double* d_xneg, const int32_t* d_shapes,
                                   int64_t n, double eps, double seed_tol, int max_iters, double* d_out) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    RC(join_caller(e));
    if (n > e->PB) return fail(AM_ERR_ARG, "too many dichotomy pairs (%lld)", (long long)n);
    cudaStream_t s = e->stream;
    CK(e->dxp.reserve(n * 3, s)); CK(e->dxn.reserve(n * 3, s)); CK(e->dmid.reserve(n * 3, s));
    CK(e->dout.reserve(n * 3, s));
    CK(e->dfp.reserve(n, s)); CK(e->dfn.reserve(n, s)); CK(e->dvals.reserve(n, s)); CK(e->dact.reserve(n, s));
    CK(e->hkeys.reserve(n * e->KW, s));
    const int32_t* shp = nullptr;
    if (d_shapes) {
        CK(e->dshape.reserve(n, s));
        CK(cudaMemcpyAsync(e->dshape.p, d_shapes, n * 4, cudaMemcpyDeviceToDevice, s));
        shp = e->dshape.p;
    }
    CK(cudaMemcpyAsync(e->dxp.p, d_xpos, n * 24, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(e->dxn.p, d_xneg, n * 24, cudaMemcpyDeviceToDevice, s));
    RC(forward_host(e, e->dxp.p, n, e->dfp.p, e->hkeys.p, shp));
    RC(forward_host(e, e->dxn.p, n, e->dfn.p, e->hkeys.p, shp));
    std::vector<int32_t> ones(n, 1);
    CK(cudaMemcpyAsync(e->dact.p, ones.data(), n * 4, cudaMemcpyHostToDevice, s));
    // speculative bisection tree: D exact steps per batched forward (k_bisect_tree / replay);
    // the per-point shapes repeat over each pair's tree points
    const int TN = bisect_tree_points(), TD = bisect_tree_depth();
    if (e->bisect_tree && n * TN <= e->PB) {
        CK(e->dtree.reserve(n * TN * 3, s));
        CK(e->dtvals.reserve(n * TN, s));
        CK(e->hkeys.reserve(n * TN * e->KW, s));
        const int32_t* tshp = nullptr;
        if (shp) {
            std::vector<int32_t> hs(n), ht(n * TN);
            CK(cudaMemcpyAsync(hs.data(), shp, n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (int64_t i = 0; i < n; i++) for (int k = 0; k < TN; k++) ht[i * TN + k] = hs[i];
            CK(e->dtshape.reserve(n * TN, s));
            CK(cudaMemcpyAsync(e->dtshape.p, ht.data(), n * TN * 4, cudaMemcpyHostToDevice, s));
            tshp = e->dtshape.p;
        }
        // the first kGraphRounds rounds of the tree (25 bisection steps: what a pair between
        // sample points needs to reach eps) as one graph, captured per (n, tolerances, buffers),
        // then one host check; any pair still open continues round by round
        constexpr int kGraphRounds = 5;
        auto round = [&](int it0) -> int {
            launch_bisect_tree(e->dxp.p, e->dxn.p, e->dact.p, n, e->dtree.p, s);
            RC(forward_host(e, e->dtree.p, n * TN, e->dtvals.p, e->hkeys.p, tshp));
            launch_bisect_replay(e->dtvals.p, e->dtree.p, e->dxp.p, e->dxn.p, e->dfp.p, e->dfn.p, e->dact.p,
                                 e->dout.p, n, it0, max_iters, eps, seed_tol, s);
            return AM_OK;
        };
        int it0 = 1;
        std::vector<const void*> tptrs = {e->dxp.p, e->dxn.p, e->dfp.p, e->dfn.p, e->dact.p, e->dout.p, e->dtree.p,
                                          e->dtvals.p, e->hkeys.p, e->pZ.p, tshp};
        if (!e->tgexec || e->tg_n != n || e->tg_eps != eps || e->tg_tol != seed_tol || e->tg_iters != max_iters ||
            e->tg_shapes != (tshp ? -2 : e->cur_shape) || e->tg_ptrs != tptrs) {
            if (e->tgexec) { cudaGraphExecDestroy(e->tgexec); e->tgexec = nullptr; }
            unsigned long long before = g_launch_count;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int rc = AM_OK;
            for (int r = 0, i0 = 1; r < kGraphRounds && i0 <= max_iters && !rc; r++, i0 += TD) rc = round(i0);
            cudaGraph_t g = nullptr;
            cudaError_t ce = cudaStreamEndCapture(s, &g);
            if (rc) { if (g) cudaGraphDestroy(g); return rc; }
            CK(ce);
            e->tg_kernels = g_launch_count - before;
            g_launch_count = before;
            cudaError_t ie = cudaGraphInstantiate(&e->tgexec, g, 0);
            cudaGraphDestroy(g);
            CK(ie);
            e->tg_n = n; e->tg_eps = eps; e->tg_tol = seed_tol; e->tg_iters = max_iters;
            e->tg_shapes = tshp ? -2 : e->cur_shape; e->tg_ptrs = tptrs;
        }
        CK(cudaGraphLaunch(e->tgexec, s));
        g_launch_count += e->tg_kernels;
        it0 += kGraphRounds * TD;
        for (; it0 <= max_iters; it0 += TD) {
            CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, 8, s));
            launch_count_active(e->dact.p, n, e->ctr.p + C_LIST, s);
            RC(sync_counters(e));
            if (e->hctr[C_LIST] == 0) break;
            RC(round(it0));
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(d_out, e->dout.p, n * 24, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        return AM_OK;
    }
    launch_midpoint(e->dxp.p, e->dxn.p, e->dmid.p, n, s);
    // one bisection step: F(mid) (the forward kernels) + the step kernel; 8 steps are captured
    // once per (n, tolerances, buffers) and replayed, the host checks convergence between replays
    auto step = [&](int last) -> int {
        RC(forward_host(e, e->dmid.p, n, e->dvals.p, e->hkeys.p, shp));
        launch_dichotomy_step(e->dvals.p, e->dxp.p, e->dxn.p, e->dfp.p, e->dfn.p, e->dmid.p, e->dact.p, e->dout.p,
                              n, eps, seed_tol, last, s);
        return AM_OK;
    };
    std::vector<const void*> ptrs = {e->dxp.p, e->dxn.p, e->dfp.p, e->dfn.p, e->dmid.p, e->dvals.p, e->dact.p,
                                     e->dout.p, e->hkeys.p, e->pZ.p, shp};
    if (!e->dgexec || e->dg_n != n || e->dg_eps != eps || e->dg_tol != seed_tol || e->dg_shapes != (shp ? -2 : e->cur_shape) ||
        e->dg_ptrs != ptrs) {
        if (e->dgexec) { cudaGraphExecDestroy(e->dgexec); e->dgexec = nullptr; }
        unsigned long long before = g_launch_count;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int rc = AM_OK;
        for (int k = 0; k < 8 && !rc; k++) rc = step(0);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        CK(ce);
        e->dg_kernels = g_launch_count - before;
        g_launch_count = before;
        cudaError_t ie = cudaGraphInstantiate(&e->dgexec, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
        e->dg_n = n; e->dg_eps = eps; e->dg_tol = seed_tol; e->dg_shapes = shp ? -2 : e->cur_shape; e->dg_ptrs = ptrs;
    }
    int it = 1;
    bool done = false;
    for (; it + 7 < max_iters && !done; it += 8) {
        CK(cudaGraphLaunch(e->dgexec, s));
        g_launch_count += e->dg_kernels;
        CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, 8, s));
        launch_count_active(e->dact.p, n, e->ctr.p + C_LIST, s);
        RC(sync_counters(e));
        done = e->hctr[C_LIST] == 0;
    }
    for (; it <= max_iters && !done; it++) {   // the tail (the last step finalises every pair)
        RC(step(it == max_iters));
        if (it == max_iters || (it & 7) == 0) {
            CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, 8, s));
            launch_count_active(e->dact.p, n, e->ctr.p + C_LIST, s);
            RC(sync_counters(e));
            done = e->hctr[C_LIST] == 0;
        }
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(d_out, e->dout.p, n * 24, cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    return AM_OK;
}

// ------------------------------------------------------------------ results
extern "C" int am_result_counts(am_engine* e, int64_t* h) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    int64_t nc = (int64_t)e->hctr[C_CELLS], nvt = (int64_t)e->hctr[C_VERTS];
    std::vector<int32_t> nv(nc);
    if (nc) {
        CK(cudaMemcpyAsync(nv.data(), e->cell_nv.p, nc * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
    }
    int64_t faces = 0, empty = 0, verts = 0, ovf = 0;
    for (int64_t i = 0; i < nc; i++) {
        if (nv[i] > 0) { faces++; verts += nv[i]; }
        else if (nv[i] == 0) empty++;
        else ovf++;
    }
    CK(cudaMemsetAsync(e->ctr.p + C_OPEN, 0, 8, e->stream));
    launch_open_edges(e->edge_nrefs.p, e->edge_roff.p, e->edge_refs.p, nvt, e->NB + e->M, e->ctr.p + C_OPEN, e->stream);
    RC(sync_counters(e));
    h[0] = nc; h[1] = faces; h[2] = empty; h[3] = verts; h[4] = (int64_t)e->hctr[C_REFS];
    h[5] = (int64_t)e->hctr[C_OPEN];
    h[6] = e->hctr[C_CAPPED] ? 1 : 0;
    h[7] = ovf;   // every cell past the face solver's limits is recorded once (nverts -1 / -2)
    return AM_OK;
}

// sorted result arrays into device buffers -- see include/am_b200.h
static int result_assemble(am_engine* e, uint64_t* d_keys, int32_t* d_nverts, double* d_verts,
                           int32_t* d_edge_nrefs, int32_t* d_edge_refs) {
    const int KW = e->KW;
    const int64_t nc = (int64_t)e->hctr[C_CELLS], nvt = (int64_t)e->hctr[C_VERTS];
    if (nc == 0) return AM_OK;
    CK(e->hkeys.reserve(nc * KW, e->stream));
    launch_gather_keys(e->pool.p, e->cell_pool.p, nc, KW, e->hkeys.p, e->stream);
    return assemble_results(e->hkeys.p, e->cell_nv.p, e->cell_voff.p, e->verts.p, e->edge_nrefs.p, e->edge_roff.p,
                            e->edge_refs.p, nc, nvt, KW, e->shape_w, e->stream, d_keys, d_nverts, d_verts,
                            d_edge_nrefs, d_edge_refs);
}

extern "C" int am_result_copy_device(am_engine* e, uint64_t* d_keys, int32_t* d_nverts, double* d_verts,
                                     int32_t* d_edge_nrefs, int32_t* d_edge_refs) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(join_caller(e));
    RC(sync_counters(e));
    RC(result_assemble(e, d_keys, d_nverts, d_verts, d_edge_nrefs, d_edge_refs));
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}

extern "C" int am_result_copy(am_engine* e, uint64_t* h_keys, int32_t* h_nverts, double* h_verts,
                              int32_t* h_edge_nrefs, int32_t* h_edge_refs) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    const int KW = e->KW;
    const int64_t nc = (int64_t)e->hctr[C_CELLS], nvt = (int64_t)e->hctr[C_VERTS], nref = (int64_t)e->hctr[C_REFS];
    if (nc == 0) return AM_OK;
    cudaStream_t s = e->stream;
    CK(e->s_keys.reserve(nc * KW, s));
    CK(e->s_nv.reserve(nc, s));
    CK(e->s_verts.reserve(std::max<int64_t>(nvt, 1) * 3, s));
    CK(e->s_enr.reserve(std::max<int64_t>(nvt, 1), s));
    CK(e->s_refs.reserve(std::max<int64_t>(nref, 1), s));
    RC(result_assemble(e, e->s_keys.p, e->s_nv.p, e->s_verts.p, e->s_enr.p, e->s_refs.p));
    CK(cudaMemcpyAsync(h_keys, e->s_keys.p, (size_t)nc * KW * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_nverts, e->s_nv.p, (size_t)nc * 4, cudaMemcpyDeviceToHost, s));
    if (nvt) {
        CK(cudaMemcpyAsync(h_verts, e->s_verts.p, (size_t)nvt * 24, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(h_edge_nrefs, e->s_enr.p, (size_t)nvt * 4, cudaMemcpyDeviceToHost, s));
    }
    if (nref) CK(cudaMemcpyAsync(h_edge_refs, e->s_refs.p, (size_t)nref * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return AM_OK;
}

// face-kernel instrumentation counters (non-zero only in AM_FACE_STATS builds); reset after read
extern "C" int am_debug_counters(am_engine* e, uint64_t* h_out64) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    CK(cudaMemcpyAsync(h_out64, e->dbg.p, 64 * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemsetAsync(e->dbg.p, 0, 64 * 8, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}

extern "C" int am_set_timing(am_engine* e, int enabled) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    e->timing = enabled != 0;
    return AM_OK;
}

// out: [compose_ms, face_ms, compose_flops, face_bytes, composed, faced, batch, flops_per_cell,
//       kernel launches (process-wide), iterations, probe_ms, probe_flops, probes, flops_per_point]
// timing mode (am_set_timing): per-stage device time of the iterations, contiguous stages
// h[0..8] ms: take, compose, canonical insert, frontier, near, face, flip insert, probe records,
// probe forwards; h[9] iterations timed; h[10] flip candidates emitted; h[11] changed canonical
// keys inserted; h[12] probe records; h[13] new pool entries; h[14] key words; h[15] cells composed
extern "C" int am_kernel_times(am_engine* e, double* h) {
    if (!e || !h) return fail(AM_ERR_ARG, "bad arguments");
    for (int i = 0; i < 9; i++) h[i] = e->t_bucket[i];
    h[9] = e->n_timed; h[10] = e->n_emit; h[11] = e->n_canon; h[12] = e->n_prec; h[13] = e->n_new;
    h[14] = (double)e->KW; h[15] = e->n_comp_cells;
    return AM_OK;
}

extern "C" int am_stats(am_engine* e, double* h) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    RC(sync_counters(e));
    h[0] = e->t_compose; h[1] = e->t_face; h[2] = e->flops; h[3] = e->face_bytes;
    h[4] = e->n_comp_cells; h[5] = e->n_face_cells; h[6] = (double)e->B; h[7] = e->flops_per_cell;
    h[8] = (double)g_launch_count; h[9] = (double)e->iters; h[10] = e->t_probe; h[11] = e->pflops;
    h[12] = e->n_probes; h[13] = e->flops_per_point;
    h[14] = (double)e->hctr[C_PROBES_TOTAL]; h[15] = (double)e->hctr[C_PREC_TOTAL];
    // prefix reuse: composition flops not executed (cells x the DMMA steps taken from parents)
    double skipped = 0, step_flops = 0;
    if (e->prefix)
        for (int f = 1; f < (int)e->sdev.size(); f++) {
            const StepDev& d = e->sdev[f];
            step_flops += 2.0 * d.n_out * d.n_in * 4 + (d.V && !(d.flags & AM_STEP_SC_FROM_INPUT) ? 2.0 * d.n_out * d.n_sin * 4 : 0.0);
            skipped += (double)e->hctr[C_BKT0 + f] * step_flops;
        }
    h[16] = skipped; h[17] = e->prefix ? 1.0 : 0.0;
    return AM_OK;
}
