// am_engine.cu -- C-ABI engine: breadth-first analytic marching on one GPU.
//
// Replaces the reference's _Marcher (reference marching.py:216-301): the
// work queue becomes a wave of candidate states in HBM, the visited set the
// on-device hash set (am_hash.cu), per-cell affine maps the batched DMMA
// composition (am_compose.cu) and face extraction the warp-per-cell solver
// (am_face.cu).  A wave:
//   1 insert raw candidates (dedup against everything ever dispatched)
//   2 compose the new ones (all layers, fp64 DMMA) -> planes + canonical states
//   3 insert canonical states whose key changed; build the frontier of new cells
//   4 face-extract the frontier -> polygons, flip candidates, probe points
//   5 forward-evaluate the probe points -> probe candidates
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "am_internal.h"

namespace am {
void launch_hash_rebuild(const HashSet& H, int64_t n_pool, cudaStream_t s);
void launch_compact(const int32_t* flag, int32_t want, int64_t n, int32_t* out, unsigned long long* count,
                    cudaStream_t s);
void launch_gather_keys(const uint64_t* src, const int32_t* idx, int64_t n, int KW, uint64_t* dst, cudaStream_t s);
void launch_frontier(int64_t nR, const int32_t* changed, const int32_t* R, const int32_t* raw_pool,
                     const int32_t* canon_pos, const int32_t* canon_status, const int32_t* canon_pool,
                     uint32_t* pool_flags, int32_t* f_items, int32_t* f_pool, unsigned long long* nF, int64_t max_new,
                     unsigned long long* capped, cudaStream_t s);
void launch_scatter_pos(const int32_t* X, int64_t nX, int32_t* pos, cudaStream_t s);
void launch_owner(const uint64_t* keys, int64_t n, int KW, int world, int32_t* owner, cudaStream_t s);
void launch_face_head_dev(const double* Z, const uint64_t* keys, double* faces, int64_t n_items, int zs, int KW,
                          const void* subs, int n_subs, cudaStream_t s);
void launch_forward_head_dev(const double* Z, uint64_t* keys, double* vals, int64_t n_items, int zs, int KW,
                             const void* subs, int n_subs, int ensemble, cudaStream_t s);
void launch_seed_project(const double* X, const double* faces, const uint64_t* keys, int KW, int M, int ensemble,
                         int64_t n, const int32_t* active, double* Xp, int32_t* done_flat, cudaStream_t s);
void launch_seed_check(const uint64_t* snew, const uint64_t* canon, int KW, int64_t n, int32_t* active,
                       double* X, const double* Xp, uint64_t* S, uint64_t* result, int32_t* done_flat,
                       cudaStream_t s);
void launch_dichotomy_step(const double* vals, double* xp, double* xn, double* fp, double* fn, double* mid,
                           int32_t* active, double* out, int64_t n, double eps, double seed_tol, int last,
                           cudaStream_t s);

void launch_midpoint(const double* a, const double* b, double* m, int64_t n, cudaStream_t s);
void launch_count_active(const int32_t* active, int64_t n, unsigned long long* cnt, cudaStream_t s);

struct SubDev {
    int last_row, last_n;
    const double* hw;
    double hb;
};
}  // namespace am

using namespace am;

namespace am {
unsigned long long g_launch_count = 0;
}

static thread_local std::string g_err;
static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess) return fail(AM_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, \
                                           cudaGetErrorString(_e));                            \
    } while (0)

template <class T>
struct DBuf {
    T* p = nullptr;
    int64_t n = 0;  // capacity in elements
    cudaError_t reserve(int64_t m, cudaStream_t s, bool keep = false, int64_t keep_n = 0) {
        if (m <= n) return cudaSuccess;
        int64_t cap = std::max<int64_t>(m, n + n / 2);
        T* q = nullptr;
        cudaError_t e = cudaMalloc(&q, (size_t)cap * sizeof(T));
        if (e != cudaSuccess) return e;
        if (keep && p && keep_n > 0) {
            e = cudaMemcpyAsync(q, p, (size_t)keep_n * sizeof(T), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
            cudaStreamSynchronize(s);
        }
        if (p) cudaFree(p);
        p = q;
        n = cap;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

enum Ctr {
    C_POOL = 0, C_CELLS, C_VERTS, C_REFS, C_NEXT, C_PROBE, C_OVF0, C_OVF1, C_LIST, C_FRONT, C_CAPPED, C_N
};

struct am_engine {
    int device = 0;
    cudaStream_t stream = 0;
    am_march_params P{};
    // network
    int NB = 0, M = 0, KW = 0, ensemble = 0, zs = 0;
    std::vector<int64_t> steps, subs;
    std::vector<StepDev> sdev;
    std::vector<CUtensorMap> tmW, tmV;
    std::vector<int> tmV_ok;
    DBuf<double> params, wpad;
    DBuf<uint8_t> subdev;
    std::vector<SubDev> hsub;
    double flops_per_cell = 0, flops_per_point = 0;
    // hash set
    DBuf<uint64_t> table, pool;
    DBuf<uint32_t> pool_flags;
    uint64_t tcap = 0;
    // counters (device) + host mirror
    DBuf<unsigned long long> ctr;
    unsigned long long hctr[C_N] = {0};
    // candidates: current wave and next wave
    DBuf<uint64_t> cand, next;
    int64_t n_cand = 0;
    // batch buffers
    int64_t B = 0;
    DBuf<double> Z, faces;
    DBuf<uint64_t> ckey;
    DBuf<int32_t> changed, status, status2, raw_pool, canon_pos, canon_pool, R, X, f_items, f_pool;
    DBuf<uint64_t> slot, slot2;
    // probes
    DBuf<double> probe_pts, probe_vals, pZ;
    // results
    DBuf<int32_t> cell_pool, cell_nv, edge_nrefs, edge_refs;
    DBuf<int64_t> cell_voff, edge_roff;
    DBuf<double> verts;
    // outbox (sharded)
    DBuf<int32_t> owner;
    std::vector<int64_t> outbox_counts;
    DBuf<uint64_t> outbox;
    int64_t n_outbox = 0;
    // seeding scratch
    DBuf<double> sx, sxp;
    DBuf<uint64_t> ss, ssn, sres;
    DBuf<int32_t> sact, sdone;
    // stats
    bool timing = false;
    cudaEvent_t ev[4];
    double t_compose = 0, t_face = 0, flops = 0, face_bytes = 0, n_comp_cells = 0, n_face_cells = 0;
    int64_t cells_total = 0;
    bool capped = false;
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
    return AM_OK;
}
static int set_counter(am_engine* e, int which, unsigned long long v) {
    e->hctr[which] = v;
    CK(cudaMemcpyAsync(e->ctr.p + which, &e->hctr[which], sizeof(unsigned long long), cudaMemcpyHostToDevice,
                       e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return AM_OK;
}
static HashSet hs(am_engine* e) {
    HashSet H;
    H.table = e->table.p;
    H.mask = e->tcap - 1;
    H.pool = e->pool.p;
    H.pool_flags = e->pool_flags.p;
    H.n_pool = e->ctr.p + C_POOL;
    H.cap_pool = e->pool.n / e->KW;
    H.KW = e->KW;
    return H;
}
// ensure room for `extra` more keys in the hash set (load factor <= 1/2)
static int ensure_hash(am_engine* e, int64_t extra) {
    int rc = sync_counters(e);
    if (rc) return rc;
    int64_t np = (int64_t)e->hctr[C_POOL];
    int64_t need = np + extra;
    if ((int64_t)(e->pool.n / e->KW) < need) {
        CK(e->pool.reserve(need * e->KW, e->stream, true, np * e->KW));
        CK(e->pool_flags.reserve(e->pool.n / e->KW, e->stream, true, np));
    }
    if ((int64_t)e->tcap < 2 * need) {
        uint64_t cap = e->tcap ? e->tcap : 1024;
        while ((int64_t)cap < 2 * need) cap <<= 1;
        e->table.release();
        CK(e->table.reserve((int64_t)cap, e->stream));
        e->tcap = cap;
        CK(cudaMemsetAsync(e->table.p, 0xff, cap * sizeof(uint64_t), e->stream));
        launch_hash_rebuild(hs(e), np, e->stream);
        CK(cudaGetLastError());
    }
    return AM_OK;
}

// -------------------------------------------------------------- lifecycle
extern "C" int am_engine_create(am_engine** out, const am_net_desc* net, const am_march_params* p, int device,
                                void* stream) {
    if (!out || !net || !p) return fail(AM_ERR_ARG, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device)
        return fail(AM_ERR_NO_DEVICE, "no CUDA device %d (found %d)", device, ndev);
    CK(cudaSetDevice(device));
    am_engine* e = new am_engine();
    e->device = device;
    e->stream = (cudaStream_t)stream;
    e->P = *p;
    if (e->P.world < 1) e->P.world = 1;
    e->NB = net->n_bits;
    e->M = net->n_subs;
    e->ensemble = net->ensemble;
    e->KW = (e->NB + 63) / 64 + (e->ensemble ? 1 : 0);
    e->zs = e->NB;
    e->steps.assign(net->h_steps, net->h_steps + (size_t)net->n_steps * AM_STEP_FIELDS);
    e->subs.assign(net->h_subs, net->h_subs + (size_t)net->n_subs * AM_SUB_FIELDS);
    CK(e->params.reserve(std::max<int64_t>(net->n_params, 1), e->stream));
    CK(cudaMemcpy(e->params.p, net->h_params, (size_t)net->n_params * sizeof(double), cudaMemcpyHostToDevice));

    // padded weight copies (row stride multiple of 16 doubles) for TMA
    int ns = net->n_steps;
    std::vector<int64_t> woff(ns), voff(ns, -1);
    int64_t tot = 0;
    auto pad = [](int64_t x) { return (x + 15) / 16 * 16; };
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        woff[s] = tot;
        tot += st[1] * pad(st[0]);
        if (st[5] >= 0) { voff[s] = tot; tot += st[1] * pad(st[10]); }
    }
    std::vector<double> hw((size_t)std::max<int64_t>(tot, 1), 0.0);
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        int64_t n_in = st[0], n_out = st[1], ld = pad(n_in);
        for (int64_t r = 0; r < n_out; r++)
            for (int64_t k = 0; k < n_in; k++) hw[woff[s] + r * ld + k] = net->h_params[st[2] + r * n_in + k];
        if (st[5] >= 0) {
            int64_t n_sin = st[10], ldv = pad(n_sin);
            for (int64_t r = 0; r < n_out; r++)
                for (int64_t k = 0; k < n_sin; k++) hw[voff[s] + r * ldv + k] = net->h_params[st[5] + r * n_sin + k];
        }
    }
    CK(e->wpad.reserve((int64_t)hw.size(), e->stream));
    CK(cudaMemcpy(e->wpad.p, hw.data(), hw.size() * sizeof(double), cudaMemcpyHostToDevice));
    e->sdev.resize(ns);
    e->tmW.resize(ns);
    e->tmV.resize(ns);
    e->tmV_ok.assign(ns, 0);
    for (int s = 0; s < ns; s++) {
        const int64_t* st = &e->steps[(size_t)s * AM_STEP_FIELDS];
        StepDev& d = e->sdev[s];
        d.n_in = (int)st[0]; d.n_out = (int)st[1]; d.flags = (int)st[4]; d.row_off = (int)st[7];
        d.in_row_off = (int)st[8]; d.sin_row_off = (int)st[9]; d.n_sin = (int)st[10]; d.sub = (int)st[11];
        d.W = e->wpad.p + woff[s];
        d.ldw = (int)pad(st[0]);
        d.b = e->params.p + st[3];
        d.V = st[5] >= 0 ? e->wpad.p + voff[s] : nullptr;
        d.ldv = st[5] >= 0 ? (int)pad(st[10]) : 0;
        d.vb = st[6] >= 0 ? e->params.p + st[6] : nullptr;
        if (!(d.flags & AM_STEP_FIRST)) {
            if (make_tmap_2d(&e->tmW[s], d.W, d.n_out, d.n_in, d.ldw) != 0)
                return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for step %d", s);
            e->flops_per_cell += 2.0 * d.n_out * d.n_in * 4;
            e->flops_per_point += 2.0 * d.n_out * d.n_in;
        }
        if (d.V && !(d.flags & AM_STEP_SC_FROM_INPUT)) {
            if (make_tmap_2d(&e->tmV[s], d.V, d.n_out, d.n_sin, d.ldv) != 0)
                return fail(AM_ERR_CUDA, "cuTensorMapEncodeTiled failed for shortcut of step %d", s);
            e->tmV_ok[s] = 1;
            e->flops_per_cell += 2.0 * d.n_out * d.n_sin * 4;
            e->flops_per_point += 2.0 * d.n_out * d.n_sin;
        }
    }
    e->hsub.resize(e->M);
    for (int j = 0; j < e->M; j++) {
        const int64_t* sb = &e->subs[(size_t)j * AM_SUB_FIELDS];
        int last = (int)(sb[0] + sb[1] - 1);
        const int64_t* st = &e->steps[(size_t)last * AM_STEP_FIELDS];
        e->hsub[j].last_row = (int)st[7];
        e->hsub[j].last_n = (int)st[1];
        e->hsub[j].hw = e->params.p + sb[2];
        e->hsub[j].hb = net->h_params[sb[3]];
    }
    CK(e->subdev.reserve((int64_t)(sizeof(SubDev) * e->M), e->stream));
    CK(cudaMemcpy(e->subdev.p, e->hsub.data(), sizeof(SubDev) * e->M, cudaMemcpyHostToDevice));

    // batch size from the plane-buffer budget
    int64_t budget = e->P.mem_budget > 0 ? e->P.mem_budget : (int64_t)2 << 30;
    int64_t per = (int64_t)e->zs * 4 * 8 + (int64_t)e->M * 32 + e->KW * 8 + 64;
    e->B = e->P.batch_cells > 0 ? e->P.batch_cells : std::max<int64_t>(64, std::min<int64_t>(budget / per, 1 << 20));
    if (e->P.max_cells <= 0) e->P.max_cells = INT64_C(10000000);

    CK(e->ctr.reserve(C_N, e->stream));
    CK(cudaMemset(e->ctr.p, 0, C_N * sizeof(unsigned long long)));
    for (int i = 0; i < 4; i++) cudaEventCreate(&e->ev[i]);
    int rc = ensure_hash(e, 4096);
    if (rc) { delete e; return rc; }
    e->outbox_counts.assign(e->P.world, 0);
    *out = e;
    return AM_OK;
}

extern "C" int am_engine_destroy(am_engine* e) {
    if (!e) return AM_OK;
    cudaStreamSynchronize(e->stream);
    DBuf<double>* dbl[] = {&e->params, &e->wpad, &e->Z, &e->faces, &e->probe_pts, &e->probe_vals, &e->pZ,
                           &e->verts, &e->sx, &e->sxp};
    for (auto* b : dbl) b->release();
    DBuf<uint64_t>* u64[] = {&e->table, &e->pool, &e->cand, &e->next, &e->ckey, &e->slot, &e->slot2, &e->outbox,
                             &e->ss, &e->ssn, &e->sres};
    for (auto* b : u64) b->release();
    DBuf<int32_t>* i32[] = {&e->changed, &e->status, &e->status2, &e->raw_pool, &e->canon_pos, &e->canon_pool,
                            &e->R, &e->X, &e->f_items, &e->f_pool, &e->cell_pool, &e->cell_nv, &e->edge_nrefs,
                            &e->edge_refs, &e->owner, &e->sact, &e->sdone};
    for (auto* b : i32) b->release();
    e->pool_flags.release();
    e->cell_voff.release();
    e->edge_roff.release();
    e->subdev.release();
    e->ctr.release();
    for (int i = 0; i < 4; i++) cudaEventDestroy(e->ev[i]);
    delete e;
    return AM_OK;
}

extern "C" int am_engine_key_words(const am_engine* e) { return e ? e->KW : 0; }

extern "C" int am_engine_reset(am_engine* e) {
    CK(cudaMemsetAsync(e->ctr.p, 0, C_N * sizeof(unsigned long long), e->stream));
    CK(cudaMemsetAsync(e->table.p, 0xff, e->tcap * sizeof(uint64_t), e->stream));
    CK(cudaStreamSynchronize(e->stream));
    memset(e->hctr, 0, sizeof e->hctr);
    e->n_cand = 0;
    e->n_outbox = 0;
    e->cells_total = 0;
    e->capped = false;
    e->t_compose = e->t_face = e->flops = e->face_bytes = e->n_comp_cells = e->n_face_cells = 0;
    return AM_OK;
}

// ----------------------------------------------------- compose / forward
// run every hidden step for n items; C = 4 (cells) or 1 (points)
static int run_steps(am_engine* e, int C, double* Z, uint64_t* keys, int32_t* changed, const double* pts, int64_t n) {
    for (size_t s = 0; s < e->sdev.size(); s++) {
        LayerLaunch L;
        L.st = e->sdev[s];
        L.Z = Z;
        L.keys = keys;
        L.changed = changed;
        L.pts = pts;
        L.n_items = n;
        L.KW = e->KW;
        L.zs = e->zs;
        if (L.st.flags & AM_STEP_FIRST) launch_input_step(L, C, e->stream);
        else launch_gemm_step(L, C, &e->tmW[s], e->tmV_ok[s] ? &e->tmV[s] : nullptr, e->stream);
    }
    CK(cudaGetLastError());
    return AM_OK;
}

// compose n cell states in place: keys -> canonical keys, Z planes, faces
static int compose(am_engine* e, uint64_t* keys, int32_t* changed, double* Z, double* faces, int64_t n) {
    if (n <= 0) return AM_OK;
    if (e->timing) cudaEventRecord(e->ev[0], e->stream);
    int rc = run_steps(e, 4, Z, keys, changed, nullptr, n);
    if (rc) return rc;
    launch_face_head_dev(Z, keys, faces, n, e->zs, e->KW, e->subdev.p, e->M, e->stream);
    CK(cudaGetLastError());
    if (e->timing) {
        cudaEventRecord(e->ev[1], e->stream);
        cudaEventSynchronize(e->ev[1]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]);
        e->t_compose += ms;
    }
    e->flops += e->flops_per_cell * n;
    e->n_comp_cells += n;
    return AM_OK;
}

// forward n points: vals (may be null) + keys (zeroed here)
static int forward(am_engine* e, const double* pts, int64_t n, double* vals, uint64_t* keys, double* Zw) {
    if (n <= 0) return AM_OK;
    CK(cudaMemsetAsync(keys, 0, (size_t)n * e->KW * sizeof(uint64_t), e->stream));
    int rc = run_steps(e, 1, Zw, keys, nullptr, pts, n);
    if (rc) return rc;
    launch_forward_head_dev(Zw, keys, vals, n, e->zs, e->KW, e->subdev.p, e->M, e->ensemble, e->stream);
    CK(cudaGetLastError());
    return AM_OK;
}

static int ensure_probe_ws(am_engine* e, int64_t n) {
    CK(e->pZ.reserve(n * e->zs, e->stream));
    CK(e->probe_vals.reserve(n, e->stream));
    return AM_OK;
}

extern "C" int am_forward(am_engine* e, const double* d_pts, int64_t n, double* d_vals, uint64_t* d_keys) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, 4 * e->B));
    int rc = ensure_probe_ws(e, chunk);
    if (rc) return rc;
    DBuf<uint64_t> tmpk;
    uint64_t* keys = d_keys;
    if (!keys) {
        CK(tmpk.reserve(chunk * e->KW, e->stream));
    }
    for (int64_t o = 0; o < n; o += chunk) {
        int64_t m = std::min(chunk, n - o);
        uint64_t* k = d_keys ? d_keys + o * e->KW : tmpk.p;
        rc = forward(e, d_pts + o * 3, m, d_vals ? d_vals + o : nullptr, k, e->pZ.p);
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(e->stream));
    tmpk.release();
    return AM_OK;
}

static int ensure_batch(am_engine* e, int64_t b) {
    CK(e->Z.reserve(b * e->zs * 4, e->stream));
    CK(e->faces.reserve(b * e->M * 4, e->stream));
    CK(e->ckey.reserve(b * e->KW, e->stream));
    DBuf<int32_t>* i32[] = {&e->changed, &e->status, &e->status2, &e->raw_pool, &e->canon_pos, &e->canon_pool,
                            &e->R, &e->X, &e->f_items, &e->f_pool};
    for (auto* x : i32) CK(x->reserve(b, e->stream));
    CK(e->slot.reserve(b, e->stream));
    CK(e->slot2.reserve(b, e->stream));
    return AM_OK;
}

extern "C" int am_affine_maps(am_engine* e, const uint64_t* d_keys, int64_t n, uint64_t* d_canon, double* d_planes,
                              double* d_faces) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    int rc = ensure_batch(e, std::min<int64_t>(n, e->B));
    if (rc) return rc;
    for (int64_t o = 0; o < n; o += e->B) {
        int64_t m = std::min<int64_t>(e->B, n - o);
        CK(cudaMemcpyAsync(e->ckey.p, d_keys + o * e->KW, m * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
        CK(cudaMemsetAsync(e->changed.p, 0, m * sizeof(int32_t), e->stream));
        rc = compose(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, m);
        if (rc) return rc;
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

// --------------------------------------------------------------- marching
extern "C" int am_push_candidates(am_engine* e, const uint64_t* d_keys, int64_t n) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    CK(e->cand.reserve((e->n_cand + n) * e->KW, e->stream, true, e->n_cand * e->KW));
    CK(cudaMemcpyAsync(e->cand.p + e->n_cand * e->KW, d_keys, n * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    e->n_cand += n;
    return AM_OK;
}

// one chunk of candidates [o, o+m): steps 1-5
static int absorb_expand(am_engine* e, const uint64_t* cands, int64_t m, int64_t* new_cells) {
    int rc = ensure_hash(e, 2 * m);
    if (rc) return rc;
    rc = ensure_batch(e, m);
    if (rc) return rc;
    HashSet H = hs(e);
    cudaStream_t s = e->stream;
    // 1. raw insert
    launch_hash_insert(H, cands, nullptr, m, e->status.p, e->slot.p, s);
    launch_hash_fixup(H, cands, nullptr, m, e->status.p, e->slot.p, 0u, e->raw_pool.p, s);
    CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, sizeof(unsigned long long), s));
    launch_compact(e->status.p, 1, m, e->R.p, e->ctr.p + C_LIST, s);
    CK(cudaGetLastError());
    if ((rc = sync_counters(e))) return rc;
    int64_t nR = (int64_t)e->hctr[C_LIST];
    if (nR == 0) { *new_cells = 0; return AM_OK; }
    // keep the batch order deterministic (the compaction appends in warp order)
    // 2. compose
    launch_gather_keys(cands, e->R.p, nR, e->KW, e->ckey.p, s);
    CK(cudaMemsetAsync(e->changed.p, 0, nR * sizeof(int32_t), s));
    rc = compose(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, nR);
    if (rc) return rc;
    // 3. canonical inserts for changed keys
    CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, sizeof(unsigned long long), s));
    launch_compact(e->changed.p, 1, nR, e->X.p, e->ctr.p + C_LIST, s);
    if ((rc = sync_counters(e))) return rc;
    int64_t nX = (int64_t)e->hctr[C_LIST];
    CK(cudaMemsetAsync(e->canon_pos.p, 0xff, nR * sizeof(int32_t), s));
    if (nX > 0) {
        launch_hash_insert(H, e->ckey.p, e->X.p, nX, e->status2.p, e->slot2.p, s);
        launch_hash_fixup(H, e->ckey.p, e->X.p, nX, e->status2.p, e->slot2.p, 0u, e->canon_pool.p, s);
        launch_scatter_pos(e->X.p, nX, e->canon_pos.p, s);
    }
    int64_t max_new = e->P.max_cells - e->cells_total;
    if (max_new < 0) max_new = 0;
    CK(cudaMemsetAsync(e->ctr.p + C_FRONT, 0, sizeof(unsigned long long), s));
    launch_frontier(nR, e->changed.p, e->R.p, e->raw_pool.p, e->canon_pos.p, e->status2.p, e->canon_pool.p,
                    e->pool_flags.p, e->f_items.p, e->f_pool.p, e->ctr.p + C_FRONT, max_new, e->ctr.p + C_CAPPED, s);
    CK(cudaGetLastError());
    if ((rc = sync_counters(e))) return rc;
    int64_t nF = std::min<int64_t>((int64_t)e->hctr[C_FRONT], max_new);
    if (e->hctr[C_CAPPED]) e->capped = true;
    *new_cells = nF;
    if (nF == 0) return AM_OK;
    e->cells_total += nF;
    // 4. faces: make room for outputs
    const int64_t VPC = 64, RPC = 256, CPC = 48;
    int64_t nc = (int64_t)e->hctr[C_CELLS], nv = (int64_t)e->hctr[C_VERTS], nrf = (int64_t)e->hctr[C_REFS];
    CK(e->cell_pool.reserve(nc + nF, s, true, nc));
    CK(e->cell_nv.reserve(nc + nF, s, true, nc));
    CK(e->cell_voff.reserve(nc + nF, s, true, nc));
    CK(e->verts.reserve((nv + nF * VPC) * 3, s, true, nv * 3));
    CK(e->edge_nrefs.reserve(nv + nF * VPC, s, true, nv));
    CK(e->edge_roff.reserve(nv + nF * VPC, s, true, nv));
    CK(e->edge_refs.reserve(nrf + nF * RPC, s, true, nrf));
    int64_t nn = (int64_t)e->hctr[C_NEXT], npb = (int64_t)e->hctr[C_PROBE];
    CK(e->next.reserve((nn + nF * CPC) * e->KW, s, true, nn * e->KW));
    CK(e->probe_pts.reserve((npb + nF * VPC) * 3, s, true, npb * 3));
    FaceArgs a;
    a.Z = e->Z.p; a.faces = e->faces.p; a.keys = e->ckey.p; a.items = e->f_items.p; a.pool_idx = e->f_pool.p;
    a.n = nF; a.NB = e->NB; a.M = e->M; a.KW = e->KW; a.zs = e->zs; a.ensemble = e->ensemble;
    for (int k = 0; k < 3; k++) { a.lo[k] = e->P.bbox_lo[k]; a.hi[k] = e->P.bbox_hi[k]; }
    a.tol_cell = e->P.tol_cell; a.tol_weld = e->P.tol_weld; a.tol_onplane = e->P.tol_onplane;
    a.probe_delta = e->P.probe_delta;
    a.cell_pool = e->cell_pool.p; a.cell_nv = e->cell_nv.p; a.cell_voff = e->cell_voff.p;
    a.n_cells = e->ctr.p + C_CELLS;
    a.verts = e->verts.p; a.edge_nrefs = e->edge_nrefs.p; a.edge_roff = e->edge_roff.p; a.edge_refs = e->edge_refs.p;
    a.n_verts = e->ctr.p + C_VERTS; a.n_refs = e->ctr.p + C_REFS;
    a.cap_cells = e->cell_pool.n; a.cap_verts = e->edge_nrefs.n; a.cap_refs = e->edge_refs.n;
    a.cand = e->next.p; a.n_cand = e->ctr.p + C_NEXT; a.cap_cand = e->next.n / e->KW;
    a.probe_pts = e->probe_pts.p; a.n_probe = e->ctr.p + C_PROBE; a.cap_probe = e->probe_pts.n / 3;
    a.overflow = e->ctr.p + C_OVF0;
    if (e->timing) cudaEventRecord(e->ev[2], s);
    launch_face(a, s);
    CK(cudaGetLastError());
    if (e->timing) {
        cudaEventRecord(e->ev[3], s);
        cudaEventSynchronize(e->ev[3]);
        float ms = 0;
        cudaEventElapsedTime(&ms, e->ev[2], e->ev[3]);
        e->t_face += ms;
    }
    e->n_face_cells += nF;
    e->face_bytes += (double)nF * (2.0 * (e->NB * 32.0) + e->M * 32.0);
    return AM_OK;
}

// probes of the wave -> candidate keys appended to next
static int flush_probes(am_engine* e) {
    int rc = sync_counters(e);
    if (rc) return rc;
    int64_t np = (int64_t)e->hctr[C_PROBE];
    if (np == 0) return AM_OK;
    int64_t nn = (int64_t)e->hctr[C_NEXT];
    CK(e->next.reserve((nn + np) * e->KW, e->stream, true, nn * e->KW));
    const int64_t chunk = std::max<int64_t>(1, 4 * e->B);
    if ((rc = ensure_probe_ws(e, std::min(chunk, np)))) return rc;
    for (int64_t o = 0; o < np; o += chunk) {
        int64_t m = std::min(chunk, np - o);
        rc = forward(e, e->probe_pts.p + o * 3, m, nullptr, e->next.p + (nn + o) * e->KW, e->pZ.p);
        if (rc) return rc;
    }
    return set_counter(e, C_NEXT, nn + np) || set_counter(e, C_PROBE, 0);
}

extern "C" int am_wave(am_engine* e, int64_t* h_new_cells) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    int64_t total_new = 0;
    int rc;
    if ((rc = set_counter(e, C_NEXT, 0))) return rc;
    if ((rc = set_counter(e, C_PROBE, 0))) return rc;
    for (int64_t o = 0; o < e->n_cand; o += e->B) {
        int64_t m = std::min<int64_t>(e->B, e->n_cand - o);
        int64_t nw = 0;
        rc = absorb_expand(e, e->cand.p + o * e->KW, m, &nw);
        if (rc) return rc;
        total_new += nw;
        // bound the probe backlog per batch
        if ((rc = flush_probes(e))) return rc;
    }
    if ((rc = sync_counters(e))) return rc;
    if (e->hctr[C_OVF0] || e->hctr[C_OVF1]) {
        // capacity overflow drops work: report loudly instead of returning a silently partial mesh
        if (e->hctr[C_OVF1])
            return fail(AM_ERR_OVERFLOW, "output capacity overflow (%llu events)", e->hctr[C_OVF1]);
    }
    int64_t nn = (int64_t)e->hctr[C_NEXT];
    std::swap(e->cand, e->next);
    e->n_cand = nn;
    if ((rc = set_counter(e, C_NEXT, 0))) return rc;
    // sharded marching: hold back candidates owned by other ranks
    if (e->P.world > 1 && nn > 0) {
        CK(e->owner.reserve(nn, e->stream));
        launch_owner(e->cand.p, nn, e->KW, e->P.world, e->owner.p, e->stream);
        std::vector<int32_t> own(nn);
        CK(cudaMemcpyAsync(own.data(), e->owner.p, nn * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        std::vector<int64_t> order(nn);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return own[a] < own[b]; });
        std::vector<int64_t> cnt(e->P.world, 0);
        for (int64_t i = 0; i < nn; i++) cnt[own[i]]++;
        // keep own, move the rest to the outbox grouped by owner
        std::vector<int32_t> idx(order.begin(), order.end());
        DBuf<int32_t> didx;
        CK(didx.reserve(nn, e->stream));
        CK(cudaMemcpyAsync(didx.p, idx.data(), nn * 4, cudaMemcpyHostToDevice, e->stream));
        DBuf<uint64_t> sorted;
        CK(sorted.reserve(nn * e->KW, e->stream));
        launch_gather_keys(e->cand.p, didx.p, nn, e->KW, sorted.p, e->stream);
        int rank = e->P.rank;
        int64_t before = 0;
        for (int r = 0; r < rank; r++) before += cnt[r];
        int64_t n_mine = cnt[rank];
        int64_t n_out = nn - n_mine;
        CK(e->outbox.reserve(std::max<int64_t>(n_out, 1) * e->KW, e->stream));
        // outbox = sorted without the own block (still grouped by owner, own count 0)
        if (before > 0)
            CK(cudaMemcpyAsync(e->outbox.p, sorted.p, before * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
        if (nn - before - n_mine > 0)
            CK(cudaMemcpyAsync(e->outbox.p + before * e->KW, sorted.p + (before + n_mine) * e->KW,
                               (nn - before - n_mine) * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
        if (n_mine > 0)
            CK(cudaMemcpyAsync(e->cand.p, sorted.p + before * e->KW, n_mine * e->KW * 8, cudaMemcpyDeviceToDevice,
                               e->stream));
        CK(cudaStreamSynchronize(e->stream));
        didx.release();
        sorted.release();
        e->n_cand = n_mine;
        e->n_outbox = n_out;
        for (int r = 0; r < e->P.world; r++) e->outbox_counts[r] = r == rank ? 0 : cnt[r];
    }
    *h_new_cells = total_new;
    return AM_OK;
}

extern "C" int am_run(am_engine* e, int64_t* h_waves) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    int64_t waves = 0;
    while (e->n_cand > 0) {
        int64_t nw = 0;
        int rc = am_wave(e, &nw);
        if (rc) return rc;
        waves++;
    }
    if (h_waves) *h_waves = waves;
    return AM_OK;
}

extern "C" int am_outbox_counts(am_engine* e, int64_t* h_counts) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    for (int r = 0; r < e->P.world; r++) h_counts[r] = e->n_outbox ? e->outbox_counts[r] : 0;
    return AM_OK;
}

extern "C" int am_outbox_take(am_engine* e, uint64_t* d_out) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    if (e->n_outbox > 0)
        CK(cudaMemcpyAsync(d_out, e->outbox.p, e->n_outbox * e->KW * 8, cudaMemcpyDeviceToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    e->n_outbox = 0;
    return AM_OK;
}

// ------------------------------------------------------------------ seeding
// reference marching.py:201-213 (_refine_seed_state), batched over seeds
extern "C" int am_seed(am_engine* e, const double* d_pts, int64_t n) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    cudaStream_t s = e->stream;
    int KW = e->KW, rc;
    CK(e->sx.reserve(n * 3, s));
    CK(e->sxp.reserve(n * 3, s));
    CK(e->ss.reserve(n * KW, s));
    CK(e->ssn.reserve(n * KW, s));
    CK(e->sres.reserve(n * KW, s));
    CK(e->sact.reserve(n, s));
    CK(e->sdone.reserve(n, s));
    if ((rc = ensure_batch(e, std::min<int64_t>(n, e->B)))) return rc;
    if (n > e->B) return fail(AM_ERR_ARG, "too many seeds for one batch (%lld > %lld)", (long long)n, (long long)e->B);
    if ((rc = ensure_probe_ws(e, n))) return rc;
    CK(cudaMemcpyAsync(e->sx.p, d_pts, n * 24, cudaMemcpyDeviceToDevice, s));
    if ((rc = forward(e, e->sx.p, n, nullptr, e->ss.p, e->pZ.p))) return rc;
    std::vector<int32_t> ones(n, 1);
    CK(cudaMemcpyAsync(e->sact.p, ones.data(), n * 4, cudaMemcpyHostToDevice, s));
    for (int it = 0; it < 3; it++) {
        CK(cudaMemcpyAsync(e->ckey.p, e->ss.p, n * KW * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemsetAsync(e->changed.p, 0, n * 4, s));
        if ((rc = compose(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, n))) return rc;
        launch_seed_project(e->sx.p, e->faces.p, e->ckey.p, KW, e->M, e->ensemble, n, e->sact.p, e->sxp.p,
                            e->sdone.p, s);
        // projected-away seeds whose face normal vanished are final: result = canonical
        launch_seed_check(nullptr, e->ckey.p, KW, n, e->sact.p, nullptr, nullptr, nullptr, e->sres.p, e->sdone.p, s);
        if ((rc = forward(e, e->sxp.p, n, nullptr, e->ssn.p, e->pZ.p))) return rc;
        launch_seed_check(e->ssn.p, e->ckey.p, KW, n, e->sact.p, e->sx.p, e->sxp.p, e->ss.p, e->sres.p, nullptr, s);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(e->ckey.p, e->ss.p, n * KW * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(e->changed.p, 0, n * 4, s));
    if ((rc = compose(e, e->ckey.p, e->changed.p, e->Z.p, e->faces.p, n))) return rc;
    // still-active seeds take canonical(s)
    launch_seed_check(nullptr, e->ckey.p, KW, n, e->sact.p, nullptr, nullptr, nullptr, e->sres.p, nullptr, s);
    CK(cudaGetLastError());
    return am_push_candidates(e, e->sres.p, n);
}

// ------------------------------------------------------------------ results
extern "C" int am_result_counts(am_engine* e, int64_t* h) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    int rc = sync_counters(e);
    if (rc) return rc;
    int64_t nc = (int64_t)e->hctr[C_CELLS];
    std::vector<int32_t> nv(nc);
    if (nc) {
        CK(cudaMemcpy(nv.data(), e->cell_nv.p, nc * 4, cudaMemcpyDeviceToHost));
    }
    int64_t faces = 0, empty = 0, verts = 0, ovf = 0;
    for (int64_t i = 0; i < nc; i++) {
        if (nv[i] > 0) { faces++; verts += nv[i]; }
        else if (nv[i] == 0) empty++;
        else ovf++;
    }
    // open edges need the refs; computed in am_result_copy -- report here via a scan
    int64_t nref = (int64_t)e->hctr[C_REFS];
    int64_t open = 0;
    if (verts) {
        int64_t nvt = (int64_t)e->hctr[C_VERTS];
        std::vector<int32_t> enr(nvt);
        std::vector<int64_t> roff(nvt);
        std::vector<int32_t> refs(nref);
        CK(cudaMemcpy(enr.data(), e->edge_nrefs.p, nvt * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(roff.data(), e->edge_roff.p, nvt * 8, cudaMemcpyDeviceToHost));
        if (nref) CK(cudaMemcpy(refs.data(), e->edge_refs.p, nref * 4, cudaMemcpyDeviceToHost));
        const int box0 = e->NB + e->M;
        for (int64_t v = 0; v < nvt; v++) {
            bool hit = false;
            for (int q = 0; q < enr[v]; q++) hit |= refs[roff[v] + q] >= box0;
            open += hit;
        }
    }
    h[0] = nc; h[1] = faces; h[2] = empty; h[3] = verts; h[4] = nref; h[5] = open;
    h[6] = e->capped ? 1 : 0;
    h[7] = ovf + (int64_t)e->hctr[C_OVF0];
    return AM_OK;
}

extern "C" int am_result_copy(am_engine* e, uint64_t* h_keys, int32_t* h_nverts, double* h_verts,
                              int32_t* h_edge_nrefs, int32_t* h_edge_refs) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    int rc = sync_counters(e);
    if (rc) return rc;
    const int KW = e->KW;
    int64_t nc = (int64_t)e->hctr[C_CELLS], nvt = (int64_t)e->hctr[C_VERTS], nref = (int64_t)e->hctr[C_REFS];
    if (nc == 0) return AM_OK;
    std::vector<int32_t> cp(nc), nv(nc);
    std::vector<int64_t> voff(nc);
    CK(cudaMemcpy(cp.data(), e->cell_pool.p, nc * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nv.data(), e->cell_nv.p, nc * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(voff.data(), e->cell_voff.p, nc * 8, cudaMemcpyDeviceToHost));
    // gather the cells' keys on device, then copy
    DBuf<uint64_t> ck;
    DBuf<int32_t> dcp;
    CK(ck.reserve(nc * KW, e->stream));
    CK(dcp.reserve(nc, e->stream));
    CK(cudaMemcpy(dcp.p, cp.data(), nc * 4, cudaMemcpyHostToDevice));
    launch_gather_keys(e->pool.p, dcp.p, nc, KW, ck.p, e->stream);
    std::vector<uint64_t> keys((size_t)nc * KW);
    CK(cudaMemcpyAsync(keys.data(), ck.p, nc * KW * 8, cudaMemcpyDeviceToHost, e->stream));
    std::vector<double> verts((size_t)nvt * 3);
    std::vector<int32_t> enr(nvt), refs(nref);
    std::vector<int64_t> roff(nvt);
    if (nvt) {
        CK(cudaMemcpyAsync(verts.data(), e->verts.p, nvt * 24, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaMemcpyAsync(enr.data(), e->edge_nrefs.p, nvt * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaMemcpyAsync(roff.data(), e->edge_roff.p, nvt * 8, cudaMemcpyDeviceToHost, e->stream));
    }
    if (nref) CK(cudaMemcpyAsync(refs.data(), e->edge_refs.p, nref * 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    ck.release();
    dcp.release();
    std::vector<int64_t> order(nc);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        const uint64_t* ka = &keys[(size_t)a * KW];
        const uint64_t* kb = &keys[(size_t)b * KW];
        for (int w = 0; w < KW; w++)
            if (ka[w] != kb[w]) return ka[w] < kb[w];
        return false;
    });
    int64_t vo = 0, ro = 0;
    for (int64_t i = 0; i < nc; i++) {
        int64_t c = order[i];
        memcpy(h_keys + i * KW, &keys[(size_t)c * KW], KW * 8);
        int n = nv[c] > 0 ? nv[c] : 0;
        h_nverts[i] = nv[c];
        for (int v = 0; v < n; v++) {
            int64_t src = voff[c] + v;
            h_verts[(vo + v) * 3 + 0] = verts[src * 3 + 0];
            h_verts[(vo + v) * 3 + 1] = verts[src * 3 + 1];
            h_verts[(vo + v) * 3 + 2] = verts[src * 3 + 2];
            h_edge_nrefs[vo + v] = enr[src];
            for (int q = 0; q < enr[src]; q++) h_edge_refs[ro++] = refs[roff[src] + q];
        }
        vo += n;
    }
    return AM_OK;
}

extern "C" int am_set_timing(am_engine* e, int enabled) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    e->timing = enabled != 0;
    return AM_OK;
}

// out: [compose_ms, face_ms, compose_flops, face_bytes, composed_items, face_cells, batch, flops_per_cell,
//       kernel launches (process-wide), waves]
extern "C" int am_stats(am_engine* e, double* h) {
    if (!e) return fail(AM_ERR_ARG, "null engine");
    h[0] = e->t_compose; h[1] = e->t_face; h[2] = e->flops; h[3] = e->face_bytes;
    h[4] = e->n_comp_cells; h[5] = e->n_face_cells; h[6] = (double)e->B; h[7] = e->flops_per_cell;
    h[8] = (double)g_launch_count; h[9] = 0;
    return AM_OK;
}

// batched bisection between sign-opposite samples (reference seeding.py:84-112)
extern "C" int am_dichotomy(am_engine* e, const double* d_xpos, const double* d_xneg, int64_t n, double eps,
                            double seed_tol, int max_iters, double* d_out) {
    if (!e || n < 0) return fail(AM_ERR_ARG, "bad arguments");
    if (n == 0) return AM_OK;
    cudaStream_t s = e->stream;
    int rc;
    DBuf<double> xp, xn, fp, fn, mid, vals;
    DBuf<int32_t> act;
    CK(xp.reserve(n * 3, s)); CK(xn.reserve(n * 3, s)); CK(mid.reserve(n * 3, s));
    CK(fp.reserve(n, s)); CK(fn.reserve(n, s)); CK(vals.reserve(n, s)); CK(act.reserve(n, s));
    DBuf<uint64_t> keys;
    CK(keys.reserve(n * e->KW, s));
    if ((rc = ensure_probe_ws(e, n))) return rc;
    CK(cudaMemcpyAsync(xp.p, d_xpos, n * 24, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(xn.p, d_xneg, n * 24, cudaMemcpyDeviceToDevice, s));
    if ((rc = forward(e, xp.p, n, fp.p, keys.p, e->pZ.p))) return rc;
    if ((rc = forward(e, xn.p, n, fn.p, keys.p, e->pZ.p))) return rc;
    std::vector<int32_t> ones(n, 1);
    CK(cudaMemcpyAsync(act.p, ones.data(), n * 4, cudaMemcpyHostToDevice, s));
    launch_midpoint(xp.p, xn.p, mid.p, n, s);
    for (int it = 1; it <= max_iters; it++) {
        if ((rc = forward(e, mid.p, n, vals.p, keys.p, e->pZ.p))) return rc;
        launch_dichotomy_step(vals.p, xp.p, xn.p, fp.p, fn.p, mid.p, act.p, d_out, n, eps, seed_tol,
                              it == max_iters, s);
        CK(cudaGetLastError());
        if ((it & 7) == 0 || it == max_iters) {
            CK(cudaMemsetAsync(e->ctr.p + C_LIST, 0, 8, s));
            launch_count_active(act.p, n, e->ctr.p + C_LIST, s);
            if ((rc = sync_counters(e))) return rc;
            if (e->hctr[C_LIST] == 0) break;
        }
    }
    CK(cudaStreamSynchronize(s));
    xp.release(); xn.release(); fp.release(); fn.release(); mid.release(); vals.release(); act.release();
    keys.release();
    return AM_OK;
}
