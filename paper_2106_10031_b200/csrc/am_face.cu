// am_face.cu -- analytic-face polygon solver, one warp per cell.
//
// For a visited cell the face polygon is { x : F-plane(x) = 0, every oriented
// cell constraint (neuron planes, branch-dominance planes, box faces) <= tol }.
// The reference enumerates it naively (all plane pairs, reference
// cells.py:337-362) or by the pivot walk (cells.py:381-462).  Here:
//
//   pass A  the warp streams all K constraint rows (coalesced 32 B plane rows
//           straight from the composition buffer), projects them into a 2-D
//           frame of the face plane and clips a polygon by every half-plane
//           shifted by tol (32 rows tested per step, cutting rows applied with a
//           warp-parallel Sutherland-Hodgman step, one lane per vertex).  The
//           result is P_tol, the tol-dilated face polygon.
//   pass B  streams the rows again and keeps the set C of rows that come within
//           tol of P_tol.  Every pair whose solution the reference accepts, every
//           incident plane and every edge-midpoint plane lies in C (DESIGN.md
//           §Face solver proves it), and C is tiny (~the polygon's edge count).
//   exact   the reference's own vertex semantics run on C only: canonical-pair
//           3x3 LU solves, tol_cell membership, incident sets, greedy weld-radius
//           dedup with lexicographic representatives, angular ordering, CCW
//           orientation, canonical rotation and per-edge transition planes.
//   expand  each crossable edge emits the neighbour states of
//           reference marching.py:152-186 (flip subsets x branch targets) and a
//           probe 1e-7 across its first plane (marching.py:271-276).  A probe
//           across a single neuron plane is emitted as a *probe record* tied to
//           the flipped state instead of a point to forward-evaluate: the cell on
//           the far side validates the mirrored point against its own planes
//           (below) and a validated probe provably lands in that cell, so it needs
//           no forward pass.  Every other probe is forward-evaluated exactly.
//   validate for each single-neuron edge the mirrored probe point mid - 1e-7 n
//           is checked against every neuron / branch functional of this cell
//           (sign consistent with the canonical state, with margin); the
//           validated neuron ids are published for the cell's pool entry.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "am_internal.h"
#include "am_hashset.cuh"
#include "am_near.cuh"

namespace am {

// optional per-cell instrumentation (build with -DAM_FACE_STATS): A.dbg[0..] accumulates
// cells, clip events (pass 1 / pass 2), C' size, raw vertices, polygon vertices, cycles,
// and a log2 histogram of per-cell cycles in dbg[16..40)
#ifdef AM_FACE_STATS
#define FSTAT(i, v) do { if (lane == 0 && A.dbg) atomicAdd(&A.dbg[i], (unsigned long long)(v)); } while (0)
// phase timers: clock cycles since the previous mark accumulate in dbg[40 + i]
#define PMARK(i) do { long long now_ = clock64(); FSTAT(40 + (i), now_ - t_mark); t_mark = now_; } while (0)
#else
#define FSTAT(i, v) do { } while (0)
#define PMARK(i) do { } while (0)
#endif

constexpr int VMAX = 32;   // clip polygon capacity (one lane per vertex)
constexpr int CMAX = 64;   // candidate plane set capacity (uint64 masks)
constexpr int QMAX = 64;   // accepted raw vertices
constexpr int FW = 4;      // warps per CTA
constexpr int kFaceCtasPerSm = 3;
#ifndef AM_NMAX
#define AM_NMAX 160
#endif
constexpr int NMAX = AM_NMAX;  // hinted path: rows near the hint point (more: the full path)
constexpr double kCDelta = 1e-10;
constexpr double kValMargin = 1e-11;   // sign margin (unit and raw values) for probe validation

// phase-private scratch: near rows (hinted clipping) and polygon assembly never overlap
struct NearPhase {
    int nl[NMAX];                   // near rows (global ids, ascending)
    double nd[NMAX];                // |value at the hint point|
    double na[NMAX], nb[NMAX], ng[NMAX];   // 2-D rows (unshifted)
    int nord[NMAX];                 // clipping order (by distance)
};
struct PolyPhase {
    // the raw vertices die with the dedup; the final loop (written by the ordering) reuses them
    union {
        double qv[QMAX][3];         // accepted raw vertices (triu order)
        double fv[QMAX][3];         // final loop
    };
    union {
        unsigned long long qs[QMAX];    // their incident-plane sets (C-row masks)
        unsigned long long fs[QMAX];    // incident sets of the final loop
    };
    double rv[QMAX][3];             // weld-cluster representatives (lexicographic minimum)
    int rfi[QMAX];                  // first member of each cluster (index into qv)
    unsigned long long rs[QMAX];
    double ang[QMAX];
    int ord[QMAX];
};

constexpr int KWF = 72;     // key words of a cell held in shared memory (larger keys: read from HBM)

struct FaceWarp {
    uint64_t key[KWF];              // the cell's state key: every orientation / bit lookup of the
                                    // solver reads it here instead of from global memory
    double ps[2][VMAX], pt[2][VMAX];
    double cn[NMAX][5];             // unit row (n, o) + raw normal norm (near rows, then C')
    int cid[NMAX];
    unsigned long long core;        // C rows within tol of P_tol (pair / incident candidates)
    int tb[32], tr[32];             // scratch: neuron bits / branch targets of one edge
    union {
        NearPhase np;
        PolyPhase pp;
    } u;
    unsigned long long erow[QMAX];  // per-edge C-row mask of the transition planes
    int eargmin[QMAX];              // per-edge global row when the mask is empty (argmin fallback)
    int eval[QMAX];                 // per edge: 1 if the mirrored probe validated
    int efirst[QMAX], eprec[QMAX];  // per edge: crossable[0], probe-record slot
    // per-edge emission: neuron / branch counts and output offsets (warp scans)
    int e_nb[QMAX], e_nbr[QMAX], e_cdoff[QMAX + 1], e_refoff[QMAX], e_valoff[QMAX];
    long long obase[5];             // reserved bases: verts, refs, validated, candidates, probe records
    double diam;                    // polygon diameter bound (hint radius for the neighbours)
    int n_cd;
    int status;
};

// this iteration's half of the (prefix-reuse double-buffered) composition rows
__device__ __forceinline__ const double* zbase(const FaceArgs& A) {
    return A.zpar ? A.Z + (int64_t)(*A.zpar & 1ull) * A.zstride : A.Z;
}

// unit oriented constraint row of global plane id gr (reference cells.py:127-185); false if dropped.
// *nrm receives the raw normal norm (neuron / branch rows) or 1 (box rows)
__device__ __noinline__ bool get_row(const Ctx& c, int gr, double n[3], double& o, double* nrm_out = nullptr) {
    if (gr < c.NB) {
        const double2* p = reinterpret_cast<const double2*>(c.Z + (int64_t)gr * 4);
        double2 a = __ldg(p), b = __ldg(p + 1);
        double nrm = sqrt((a.x * a.x + a.y * a.y) + b.x * b.x);
        if (nrm_out) *nrm_out = nrm;
        if (!(nrm > kDegen)) return false;
        double orient = key_bit(c.key, gr) ? -1.0 : 1.0;
        n[0] = (a.x * orient) / nrm; n[1] = (a.y * orient) / nrm; n[2] = (b.x * orient) / nrm;
        o = (b.y * orient) / nrm;
        return true;
    }
    if (gr < c.NB + c.M) {
        int t = gr - c.NB;
        if (!c.ensemble || t == c.branch) return false;
        const double* ft = c.faces + t * 4;
        const double* fj = c.faces + c.branch * 4;
        double d0 = ft[0] - fj[0], d1 = ft[1] - fj[1], d2 = ft[2] - fj[2], dc = ft[3] - fj[3];
        double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
        if (nrm_out) *nrm_out = nrm;
        if (!(nrm > kDegen)) return false;
        n[0] = d0 / nrm; n[1] = d1 / nrm; n[2] = d2 / nrm; o = dc / nrm;
        return true;
    }
    if (nrm_out) *nrm_out = 1.0;
    int k = gr - c.NB - c.M;
    int ax = k >> 1;
    n[0] = n[1] = n[2] = 0.0;
    if ((k & 1) == 0) { n[ax] = 1.0; o = -c.hi[ax]; }
    else { n[ax] = -1.0; o = c.lo[ax]; }
    return true;
}

__device__ __forceinline__ double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// 2-D projection (a, b, g) of the oriented unit row in the face-plane frame, with one
// reciprocal per row (the streaming passes only need it to ~1 ulp); *nrm = raw norm
__device__ __forceinline__ bool row2d(const Ctx& c, int gr, const RawRow& r, const double U[3], const double V[3],
                                      const double P0[3], double& a2, double& b2, double& g2, double& nrm) {
    if (r.kind < 0) { nrm = 0.0; return false; }
    nrm = sqrt((r.x * r.x + r.y * r.y) + r.z * r.z);
    if (r.kind != 2 && !(nrm > kDegen)) return false;
    double s = 1.0 / nrm;
    if (r.kind == 0 && key_bit(c.key, gr)) s = -s;
    a2 = ((r.x * U[0] + r.y * U[1]) + r.z * U[2]) * s;
    b2 = ((r.x * V[0] + r.y * V[1]) + r.z * V[2]) * s;
    g2 = (((r.x * P0[0] + r.y * P0[1]) + r.z * P0[2]) + r.c) * s;
    return true;
}

// 3x3 LU with partial pivoting, same operation order as oracle solve3 (LAPACK getf2/getrs)
__device__ double solve3(const double Min[9], const double rin[3], double x[3]) {
    double a[9], b[3];
#pragma unroll
    for (int i = 0; i < 9; i++) a[i] = Min[i];
    b[0] = rin[0]; b[1] = rin[1]; b[2] = rin[2];
    double sign = 1.0;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        int p = k;
        double best = fabs(a[k * 3 + k]);
        for (int i = k + 1; i < 3; i++)
            if (fabs(a[i * 3 + k]) > best) { best = fabs(a[i * 3 + k]); p = i; }
        if (p != k) {
            for (int j = 0; j < 3; j++) { double tt = a[k * 3 + j]; a[k * 3 + j] = a[p * 3 + j]; a[p * 3 + j] = tt; }
            double tt = b[k]; b[k] = b[p]; b[p] = tt;
            sign = -sign;
        }
        double piv = a[k * 3 + k];
        if (piv == 0.0) return 0.0;
        double rp = 1.0 / piv;
        for (int i = k + 1; i < 3; i++) {
            double l = a[i * 3 + k] * rp;
            a[i * 3 + k] = l;
            for (int j = k + 1; j < 3; j++) a[i * 3 + j] -= l * a[k * 3 + j];
            b[i] -= l * b[k];
        }
    }
    double det = fabs(sign * a[0] * a[4] * a[8]);
    x[2] = b[2] / a[8];
    x[1] = (b[1] - a[5] * x[2]) / a[4];
    x[0] = ((b[0] - a[1] * x[1]) - a[2] * x[2]) / a[0];
    return det;
}

__device__ __forceinline__ bool lex_less(const double* a, const double* b) {
    if (a[0] != b[0]) return a[0] < b[0];
    if (a[1] != b[1]) return a[1] < b[1];
    return a[2] < b[2];
}

// current clip polygon of a warp: vertex count, ring buffer index, status (0 ok, 1 empty,
// 2 overflow) and the bounding circle (sc, tc, rho) used by the quick rejection tests
struct Poly { int nv, cur, status; double sc, tc, rho; };

// warp-parallel Sutherland-Hodgman step by (ca, cb, cg) (<= 0 inside), one lane per vertex;
// keeps the bounding circle current.  Out of line so the three call sites share one copy.
__device__ __noinline__ Poly clip_poly(FaceWarp* W, Poly P, double ca, double cb, double cg) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const int nv = P.nv, cur = P.cur;
    double si = 0, ti = 0, di = 0;
    if (lane < nv) { si = W->ps[cur][lane]; ti = W->pt[cur][lane]; di = ca * si + cb * ti + cg; }
    int nx = lane + 1 == nv ? 0 : lane + 1;
    double sj = __shfl_sync(full, si, nx & 31), tj = __shfl_sync(full, ti, nx & 31),
           dj = __shfl_sync(full, di, nx & 31);
    bool in_i = di <= 0.0, in_j = dj <= 0.0;
    if (!__any_sync(full, lane < nv && !in_i)) return P;
    int cnt = lane < nv ? (in_i ? 1 : 0) + (in_i != in_j ? 1 : 0) : 0;
    int pre = cnt;
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
        int y = __shfl_up_sync(full, pre, o2);
        if (lane >= o2) pre += y;
    }
    int total = __shfl_sync(full, pre, 31);
    pre -= cnt;
    if (total > VMAX) { P.status = 2; return P; }
    int dst = cur ^ 1;
    double ns = 0.0, nt = 0.0;
    if (lane < nv) {
        int w = pre;
        if (in_i) { W->ps[dst][w] = si; W->pt[dst][w] = ti; ns += si; nt += ti; w++; }
        if (in_i != in_j) {
            double lam = di / (di - dj);
            double xs = si + lam * (sj - si), xt = ti + lam * (tj - ti);
            W->ps[dst][w] = xs;
            W->pt[dst][w] = xt;
            ns += xs; nt += xt;
        }
    }
    __syncwarp();
    P.cur = dst;
    P.nv = total;
    if (total < 3) { P.status = 1; return P; }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
        ns += __shfl_xor_sync(full, ns, o2);
        nt += __shfl_xor_sync(full, nt, o2);
    }
    P.sc = ns / total; P.tc = nt / total;
    double d2 = 0.0;
    if (lane < total) {
        double ds = W->ps[dst][lane] - P.sc, dt = W->pt[dst][lane] - P.tc;
        d2 = ds * ds + dt * dt;
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) d2 = fmax(d2, __shfl_xor_sync(full, d2, o2));
    P.rho = sqrt(d2) * (1.0 + 1e-9) + 1e-12;
    return P;
}

// exclusive warp scan of v; *total = sum over the warp
__device__ __forceinline__ int warp_excl_scan(int v, int& total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// flip subsets of an edge with 3 neuron planes in the reference's order (itertools.combinations
// by size 0..3): bit i = flip the i-th neuron plane of the edge
__constant__ unsigned kComb3[8] = {0u, 1u, 2u, 4u, 3u, 5u, 6u, 7u};

// polygons with more than 32 vertices: the serial ordering (lane 0)
__device__ __noinline__ void order_serial(FaceWarp* W, int nr, const double* fu) {
    for (int i = 0; i < nr; i++) W->u.pp.ord[i] = i;
    for (int i = 1; i < nr; i++) {   // stable sort by angle (reference np.argsort kind="stable")
        int tt = W->u.pp.ord[i], j = i - 1;
        while (j >= 0 && W->u.pp.ang[W->u.pp.ord[j]] > W->u.pp.ang[tt]) { W->u.pp.ord[j + 1] = W->u.pp.ord[j]; j--; }
        W->u.pp.ord[j + 1] = tt;
    }
    double tot[3] = {0, 0, 0};
    for (int i = 0; i < nr; i++) {
        const double* p = W->u.pp.rv[W->u.pp.ord[i]];
        const double* q = W->u.pp.rv[W->u.pp.ord[(i + 1) % nr]];
        tot[0] += p[1] * q[2] - p[2] * q[1];
        tot[1] += p[2] * q[0] - p[0] * q[2];
        tot[2] += p[0] * q[1] - p[1] * q[0];
    }
    double area = 0.5 * ((tot[0] * fu[0] + tot[1] * fu[1]) + tot[2] * fu[2]);
    if (area < 0.0)
        for (int i = 0, j = nr - 1; i < j; i++, j--) { int tt = W->u.pp.ord[i]; W->u.pp.ord[i] = W->u.pp.ord[j]; W->u.pp.ord[j] = tt; }
    int start = 0;
    for (int k = 1; k < nr; k++)
        if (lex_less(W->u.pp.rv[W->u.pp.ord[k]], W->u.pp.rv[W->u.pp.ord[start]])) start = k;
    for (int k = 0; k < nr; k++) {
        int src = W->u.pp.ord[(k + start) % nr];
        for (int d = 0; d < 3; d++) W->u.pp.fv[k][d] = W->u.pp.rv[src][d];
        W->u.pp.fs[k] = W->u.pp.rs[src];
    }
}

// Full path (cells whose hinted attempts did not converge, or without a hint): pass 1 clips a
// large square by every row (box rows first), pass 2 collects C.  Out of line: rare, and its code
// would otherwise sit between the hot phases in the instruction cache.
struct FullOut { int nv, cur, status; double sc, tc, rho; int nC; unsigned long long core; int risky; };
__device__ __noinline__ FullOut full_path(FaceWarp* W, const Ctx& c, const double* U, const double* Vv,
                                          const double* P0, double tol_c, double tol_max, double band) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const int box0 = c.NB + c.M;
    int nv = 0, cur = 0, status = 0;
    double sc = 0.0, tc = 0.0, rho = 0.0;
    int nC = 0, risky = 0;
    unsigned long long core = 0;
    auto clip = [&](double ca, double cb, double cg) {
        Poly P{nv, cur, status, sc, tc, rho};
        P = clip_poly(W, P, ca, cb, cg);
        nv = P.nv; cur = P.cur; status = P.status; sc = P.sc; tc = P.tc; rho = P.rho;
    };
    auto cuts = [&](double a2, double b2, double g2) -> bool {
        if ((a2 * sc + b2 * tc + g2) + rho <= 0.0) return false;   // |(a2, b2)| <= 1 for a unit row
        double mx = -1e300;
#pragma unroll 1
        for (int v = 0; v < nv; v++) mx = fmax(mx, a2 * W->ps[cur][v] + b2 * W->pt[cur][v] + g2);
        return mx > 0.0;
    };
    {
        // initial square; then pass 1: box rows first, then neurons, then branch rows
        nC = 0; core = 0;
        double R = 64.0;
        for (int k = 0; k < 3; k++) R = fmax(R, 64.0 * fmax(fabs(c.lo[k]), fabs(c.hi[k])));
        if (lane < 4) {
            W->ps[0][lane] = (lane == 0 || lane == 3) ? -R : R;
            W->pt[0][lane] = (lane < 2) ? -R : R;
        }
        nv = 4; cur = 0; sc = 0.0; tc = 0.0;
        rho = R * 1.4142135623730951 * (1.0 + 1e-12);
        __syncwarp();
        auto order = [&](int idx) { return idx < 6 ? box0 + idx : idx - 6; };
        RawRow nxt = load_raw(c, lane < c.K ? order(lane) : c.K);
        for (int base = 0; base < c.K && status == 0; base += 32) {
            const int idx = base + lane;
            const RawRow rr = nxt;
            if (base + 32 < c.K) nxt = load_raw(c, idx + 32 < c.K ? order(idx + 32) : c.K);   // prefetch
            double a2 = 0.0, b2 = 0.0, g2 = 0.0, nrm;
            bool cut = false;
            if (idx < c.K && row2d(c, order(idx), rr, U, Vv, P0, a2, b2, g2, nrm)) {
                g2 -= tol_c;
                cut = cuts(a2, b2, g2);
            }
            unsigned mask = __ballot_sync(full, cut);
            while (mask && status == 0) {
                int src = __ffs(mask) - 1;
                mask &= mask - 1;
                clip(__shfl_sync(full, a2, src), __shfl_sync(full, b2, src), __shfl_sync(full, g2, src));
            }
        }
    }

    // ------------------------------------------------ pass 2: remaining cuts + candidate set C'
    // Every row: clip if it still cuts (rare after a good hint), then keep it in C' if it
    // comes within the band of the current polygon.  Rows seen before a late clip were
    // tested against a larger polygon -- a superset, which is still exact (C' only has to
    // contain every row near the final P_tol).  core rows: within tol of P_tol (the only
    // rows that can carry a vertex, an incident plane or an edge plane); the wider band up
    // to 1.5 probe steps serves probe validation.  `risky` marks near-degenerate rows that
    // make the validation margins meaningless (the cell then publishes nothing).
    for (int attempt = 0; attempt < 2 && status == 0; attempt++) {
        nC = 0;
        core = 0;
        risky = 0;
        RawRow nx1 = load_raw(c, lane), nx2 = load_raw(c, lane + 32);
        for (int base = 0; base < c.K && status == 0; base += 32) {
            const int gr = base + lane;
            const RawRow rr = nx1;
            nx1 = nx2;
            if (base + 64 < c.K) nx2 = load_raw(c, gr + 64);   // prefetch two batches ahead
            double a2 = 0.0, b2 = 0.0, g2 = 0.0, nrm = 0.0;
            bool kept = false;
            if (gr < c.K) {
                kept = row2d(c, gr, rr, U, Vv, P0, a2, b2, g2, nrm);
                // near-degenerate neuron / branch functionals make the validation margins meaningless
                if (rr.kind == 0 && nrm > 0.0 && nrm < kTinyNorm) risky = 1;
                if (rr.kind == 1 && nrm < kTinyNorm) risky = 1;
            }
            bool cut = kept && cuts(a2, b2, g2 - tol_c);
            unsigned cmask_cut = __ballot_sync(full, cut);
            while (cmask_cut && status == 0) {
                int src = __ffs(cmask_cut) - 1;
                cmask_cut &= cmask_cut - 1;
                clip(__shfl_sync(full, a2, src), __shfl_sync(full, b2, src), __shfl_sync(full, g2 - tol_c, src));
            }
            if (status != 0) break;
            bool in = false, is_core = false;
            if (kept && (a2 * sc + b2 * tc + g2) + rho >= -band) {
                double mx = -1e300;
#pragma unroll 1
                for (int v = 0; v < nv; v++) mx = fmax(mx, a2 * W->ps[cur][v] + b2 * W->pt[cur][v] + g2);
                in = mx >= -band;
                is_core = mx >= -tol_max - kCDelta;
            }
            unsigned mask = __ballot_sync(full, in);
            unsigned cmask = __ballot_sync(full, is_core);
            int pos = nC + __popc(mask & ((1u << lane) - 1u));
            if (in && pos < CMAX) {
                // exact unit row, same arithmetic as reference cells.py:146-160
                double n[3], o;
                get_row(c, gr, n, o);
                W->cn[pos][0] = n[0]; W->cn[pos][1] = n[1]; W->cn[pos][2] = n[2]; W->cn[pos][3] = o;
                W->cn[pos][4] = nrm;
                W->cid[pos] = gr;
            }
            // core bits in C order
            unsigned m = mask;
            int k = nC;
            while (m && k < CMAX) {
                int l = __ffs(m) - 1;
                m &= m - 1;
                if ((cmask >> l) & 1u) core |= 1ull << k;
                k++;
            }
            nC += __popc(mask);
        }
        risky = __any_sync(full, risky);
        if (nC <= CMAX) break;   // else: late clips inflated C' -- once more against the final polygon
    }
    return FullOut{nv, cur, status, sc, tc, rho, nC, core, risky};
}

__device__ void face_cell(const FaceArgs& A, FaceWarp* W, int64_t fi, int64_t n_wave) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    const int item = A.items[fi];
#ifdef AM_FACE_STATS
    const long long t_start = clock64();
    long long t_mark = t_start;
    int n_clip1 = 0, n_clip2 = 0;
#endif
    (void)0;

    Ctx c;
    c.Z = zbase(A) + (int64_t)item * A.zs * 4;
    c.faces = A.faces + (int64_t)item * A.M * 4;
    c.key = A.keys + (int64_t)item * A.KW;
    // the cell's independent inputs are requested together, ahead of their first use: hint,
    // near-list header and (single-subnetwork nets) the face row
    const int64_t nslot = A.near_by_item ? (int64_t)item : fi;   // near lists built by the composition: per item
    const double4 hint_in = reinterpret_cast<const double4*>(A.hints)[item];
    const int nflags_in = A.near_flags ? A.near_flags[nslot] : 0;
    const int nn_in = A.near_flags ? A.near_n[nslot] : 0;
    double4 face_in = make_double4(0.0, 0.0, 0.0, 0.0);
    if (!A.ensemble) face_in = *reinterpret_cast<const double4*>(c.faces);
    if (A.KW <= KWF) {   // stage the key: one coalesced load instead of a dependent round trip per lookup
        for (int w = lane; w < A.KW; w += 32) W->key[w] = c.key[w];
        __syncwarp();
        c.key = W->key;
    }
    c.NB = A.NB; c.M = A.M; c.ensemble = A.ensemble;
    c.branch = A.ensemble ? (int)c.key[A.KW - 1] : 0;
    c.K = A.NB + A.M + 6;
    for (int k = 0; k < 3; k++) { c.lo[k] = A.lo[k]; c.hi[k] = A.hi[k]; }
    const double tol_c = A.tol_cell, tol_p = A.tol_onplane;
    const double tol_max = fmax(tol_c, tol_p);
    const int box0 = c.NB + c.M;

    // ------------------------------------------------------ face plane
    if (A.ensemble) face_in = *reinterpret_cast<const double4*>(c.faces + c.branch * 4);
    const double fr[4] = {face_in.x, face_in.y, face_in.z, face_in.w};
    double fn = sqrt((fr[0] * fr[0] + fr[1] * fr[1]) + fr[2] * fr[2]);
    double fu[3] = {0, 0, 0}, fo = 0.0;
    bool face_ok = fn > kDegen;
    if (face_ok) {
        fu[0] = fr[0] / fn; fu[1] = fr[1] / fn; fu[2] = fr[2] / fn; fo = fr[3] / fn;
        face_ok = sqrt((fu[0] * fu[0] + fu[1] * fu[1]) + fu[2] * fu[2]) > kDegen;
    }
    // 2-D frame (same basis as reference cells.py:275-285)
    double ua[3] = {1.0, 0.0, 0.0};
    if (!(fabs(fu[0]) < 0.9)) { ua[0] = 0.0; ua[1] = 1.0; }
    double U[3] = {fu[1] * ua[2] - fu[2] * ua[1], fu[2] * ua[0] - fu[0] * ua[2], fu[0] * ua[1] - fu[1] * ua[0]};
    double un = sqrt((U[0] * U[0] + U[1] * U[1]) + U[2] * U[2]);
    U[0] /= un; U[1] /= un; U[2] /= un;
    double Vv[3] = {fu[1] * U[2] - fu[2] * U[1], fu[2] * U[0] - fu[0] * U[2], fu[0] * U[1] - fu[1] * U[0]};
    double P0[3] = {-fo * fu[0], -fo * fu[1], -fo * fu[2]};

    int nv = 0, cur = 0;
    int status = face_ok ? 0 : 1;  // 0 ok, 1 empty, 2 overflow, 3 deferred

    // hint: a point on this cell's polygon (the edge midpoint through which the cell was
    // found: F is continuous across the shared plane, so it lies on this face plane too)
    // and a search radius.  Pass 1 clips only by rows within that radius, so the polygon
    // is (nearly) final before the full passes.
    // Seeds carry their surface point as the hint; it is projected onto the face plane (a
    // no-op up to rounding for edge midpoints) so the 3-D near test and the 2-D frame agree.
    double4 hint = hint_in;
    const bool have_hint = isfinite(hint.w) && face_ok;
    double s0 = 0.0, t0 = 0.0;
    if (have_hint) {
        const double hd = ((fu[0] * hint.x + fu[1] * hint.y) + fu[2] * hint.z) + fo;
        hint.x -= hd * fu[0]; hint.y -= hd * fu[1]; hint.z -= hd * fu[2];
        double dx[3] = {hint.x - P0[0], hint.y - P0[1], hint.z - P0[2]};
        s0 = dot3(dx, U);
        t0 = dot3(dx, Vv);
    }
    // ---------------------------------------------------- hinted single pass
    // Stream every row once: keep those whose value at the hint point x0 is within
    // lim = tau + band (raw-value test, no sqrt/division).  Each kept row is unit and
    // Lipschitz-1, so a row farther than lim from x0 can neither cut nor come within band
    // of any point within tau of x0.  Clip by the kept rows only (nearest first) inside a
    // square of half-size tau around x0, take C' from them, and accept the result iff
    // every vertex of P_tol lies within tau - band of x0 (else: the full two-pass path).
    bool hinted_done = false;
    double defer_w = 0.0;   // status 3: the widened hint radius of a deferred cell
    int nC = 0;
    unsigned long long core = 0;
    int risky = 0;
    const double band = tol_max + 1.5 * A.probe_delta + 1e-9;
    double tau = A.tau_mult * hint.w;
    // near list from k_near (rows within `reach` of x0): attempts with tau <= reach filter it
    // instead of streaming every row again
    const int list_flags = have_hint ? nflags_in : 0;
    const bool use_list = (list_flags & kNearValid) && !(list_flags & kNearOverflow);
    const int n_list = use_list ? nn_in : 0;
    const double reach = A.near_reach * hint.w;
    FSTAT(14, use_list ? 1 : 0);
    FSTAT(15, (list_flags & kNearOverflow) ? 1 : 0);
    PMARK(0);
#ifdef AM_FACE_STATS
    int n_attempts = 0, n_streamed = 0, fp_reason = 3;   // 1 x0 violates, 2 near rows > NMAX, 3 attempts
#endif
    for (int attempt = 0; attempt < A.max_attempts && status == 0 && have_hint && !hinted_done; attempt++) {
#ifdef AM_FACE_STATS
        n_attempts++;
        if (!(use_list && tau <= reach)) n_streamed++;
#endif
        if (attempt > 0 && use_list && !(tau <= reach) && A.queue && n_wave >= A.defer_min) {
            // the polygon outgrew the near list: defer the cell (queued again with a hint radius
            // whose near list covers this reach) rather than stream every row in this iteration
            const int32_t pq = A.pool_idx[fi];
            if (!(A.pool_flags[pq] & kPoolWasDeferred)) {
                status = 3;
                defer_w = tau / A.tau_mult;
                break;
            }
        }
        const double x0[3] = {hint.x, hint.y, hint.z};
        const double lim = tau + band + 1e-9;
        double dmax_seen = 0.0;
        int nn = 0;
        bool ok = true;
        if (use_list && tau <= reach) {
            // the near kernel's list (rows within `reach` of x0, ascending ids): same test, tighter lim
            const int64_t lb = nslot * (int64_t)A.near_cap;
#pragma unroll 1
            for (int base = 0; base < n_list; base += 32) {
                const int j = base + lane;
                bool near = false;
                int gr = 0;
                double4 rr = make_double4(0.0, 0.0, 0.0, 0.0);
                if (j < n_list) {
                    gr = A.near_id[lb + j];
                    rr = reinterpret_cast<const double4*>(A.near_row)[lb + j];
                    const double n2 = (rr.x * rr.x + rr.y * rr.y) + rr.z * rr.z;
                    double v = ((rr.x * x0[0] + rr.y * x0[1]) + rr.z * x0[2]) + rr.w;
                    if (gr < c.NB && key_bit(c.key, gr)) v = -v;
                    near = v >= 0.0 || v * v <= lim * lim * n2;
                }
                const unsigned mask = __ballot_sync(full, near);
                const int pos = nn + __popc(mask & ((1u << lane) - 1u));
                if (near && pos < NMAX) {
                    W->u.np.nl[pos] = gr;
                    W->cn[pos][0] = rr.x; W->cn[pos][1] = rr.y; W->cn[pos][2] = rr.z; W->cn[pos][3] = rr.w;
                }
                nn += __popc(mask);
            }
            ok = !(list_flags & kNearX0Bad);
            risky = (list_flags & kNearRisky) ? 1 : 0;
        } else {
        RawRow nx1 = load_raw(c, lane), nx2 = load_raw(c, lane + 32);
        for (int base = 0; base < c.K; base += 32) {
            const int gr = base + lane;
            const RawRow rr = nx1;
            nx1 = nx2;
            if (base + 64 < c.K) nx2 = load_raw(c, gr + 64);   // prefetch two batches ahead
            bool near = false;
            if (gr < c.K && rr.kind >= 0) {
                double n2 = (rr.x * rr.x + rr.y * rr.y) + rr.z * rr.z;
                if (rr.kind == 0 && n2 > 0.0 && n2 < kTinyNorm * kTinyNorm) risky = 1;
                if (rr.kind == 1 && n2 < kTinyNorm * kTinyNorm) risky = 1;
                if (rr.kind == 2 || n2 > kDegen * kDegen) {
                    double v = ((rr.x * x0[0] + rr.y * x0[1]) + rr.z * x0[2]) + rr.c;
                    if (rr.kind == 0 && key_bit(c.key, gr)) v = -v;
                    if (v > 0.0 && v * v > 1e-18 * n2) ok = false;   // x0 violates the row by > 1e-9
                    near = v >= 0.0 || v * v <= lim * lim * n2;
                }
            }
            unsigned mask = __ballot_sync(full, near);
            int pos = nn + __popc(mask & ((1u << lane) - 1u));
            if (near && pos < NMAX) {   // keep the raw row: no second global read
                W->u.np.nl[pos] = gr;
                W->cn[pos][0] = rr.x; W->cn[pos][1] = rr.y; W->cn[pos][2] = rr.z; W->cn[pos][3] = rr.c;
            }
            nn += __popc(mask);
        }
        }
        PMARK(1);
        bool x0ok = __all_sync(full, ok);
        ok = x0ok && nn <= NMAX;
        FSTAT(9, x0ok ? 0 : 1);
        FSTAT(10, nn > NMAX ? 1 : 0);
        FSTAT(12, nn);
        risky = __any_sync(full, risky);
        __syncwarp();
        if (ok) {
            // exact unit rows of the near set (get_row arithmetic), 2-D projections and distances
            for (int i = lane; i < nn; i += 32) {
                const int gr = W->u.np.nl[i];
                const double rx = W->cn[i][0], ry = W->cn[i][1], rz = W->cn[i][2], rc = W->cn[i][3];
                double n[3], o, nrm;
                if (gr < box0) {
                    nrm = sqrt((rx * rx + ry * ry) + rz * rz);
                    double orient = (gr < c.NB && key_bit(c.key, gr)) ? -1.0 : 1.0;
                    n[0] = (rx * orient) / nrm; n[1] = (ry * orient) / nrm; n[2] = (rz * orient) / nrm;
                    o = (rc * orient) / nrm;
                } else {
                    nrm = 1.0; n[0] = rx; n[1] = ry; n[2] = rz; o = rc;
                }
                double a2 = dot3(n, U), b2 = dot3(n, Vv), g2 = dot3(n, P0) + o;
                W->u.np.na[i] = a2; W->u.np.nb[i] = b2; W->u.np.ng[i] = g2;
                W->u.np.nd[i] = fabs(dot3(n, x0) + o);
                W->cn[i][0] = n[0]; W->cn[i][1] = n[1]; W->cn[i][2] = n[2]; W->cn[i][3] = o; W->cn[i][4] = nrm;
                W->cid[i] = gr;
            }
            __syncwarp();
            for (int i = lane; i < nn; i += 32) {   // rank sort by distance (ties: lower id first)
                int rk = 0;
#pragma unroll 1
                for (int j = 0; j < nn; j++) rk += (W->u.np.nd[j] < W->u.np.nd[i]) || (W->u.np.nd[j] == W->u.np.nd[i] && j < i);
                W->u.np.nord[rk] = i;
            }
            PMARK(2);
            // start from the square of half-size tau around x0.  The polygon lives in registers
            // (lane v holds vertex v), mirrored in W->ps/pt[cur] for the C' pass below; each near
            // row is one register test + ballot, and a cutting row is a Sutherland-Hodgman step
            // whose output slots come from two ballots.
            const double hw = tau;
            double vs = 0.0, vt = 0.0;
            if (lane < 4) {
                vs = s0 + ((lane == 0 || lane == 3) ? -hw : hw);
                vt = t0 + ((lane < 2) ? -hw : hw);
                W->ps[0][lane] = vs;
                W->pt[0][lane] = vt;
            }
            nv = 4; cur = 0;
            __syncwarp();
            const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
            for (int q = 0; q < nn; q++) {
                const int i = W->u.np.nord[q];
                const double a2 = W->u.np.na[i], b2 = W->u.np.nb[i], g2 = W->u.np.ng[i] - tol_c;
                const bool act = lane < nv;
                const double di = act ? a2 * vs + b2 * vt + g2 : -1.0;
                if (!__any_sync(full, di > 0.0)) continue;
                const int nx = lane + 1 == nv ? 0 : lane + 1;
                const double sj = __shfl_sync(full, vs, nx & 31), tj = __shfl_sync(full, vt, nx & 31),
                             dj = __shfl_sync(full, di, nx & 31);
                const bool in_i = di <= 0.0, in_j = dj <= 0.0;
                const unsigned m_in = __ballot_sync(full, act && in_i), m_x = __ballot_sync(full, act && in_i != in_j);
                const int total = __popc(m_in) + __popc(m_x);
                if (total > VMAX) { status = 2; break; }
                const int dst = cur ^ 1;
                if (act) {
                    int w = __popc(m_in & lt) + __popc(m_x & lt);
                    if (in_i) { W->ps[dst][w] = vs; W->pt[dst][w] = vt; w++; }
                    if (in_i != in_j) {
                        const double lam = di / (di - dj);
                        W->ps[dst][w] = vs + lam * (sj - vs);
                        W->pt[dst][w] = vt + lam * (tj - vt);
                    }
                }
                __syncwarp();
                cur = dst;
                nv = total;
#ifdef AM_FACE_STATS
                n_clip1++;
#endif
                if (nv < 3) { status = 1; break; }
                vs = lane < nv ? W->ps[cur][lane] : 0.0;
                vt = lane < nv ? W->pt[cur][lane] : 0.0;
            }
            if (status == 0) {
                PMARK(3);
                // acceptance: P_tol within tau - band of x0
                double dmax = 0.0;
                if (lane < nv) {
                    double ds = W->ps[cur][lane] - s0, dt = W->pt[cur][lane] - t0;
                    dmax = sqrt(ds * ds + dt * dt);
                }
#pragma unroll
                for (int o2 = 16; o2; o2 >>= 1) dmax = fmax(dmax, __shfl_xor_sync(full, dmax, o2));
                FSTAT(11, dmax + band + 1e-9 <= hw ? 0 : 1);
                dmax_seen = dmax;
                if (dmax + band + 1e-9 <= hw) {
                    // C' and core among the near rows (already in ascending id order)
                    for (int base = 0; base < nn; base += 32) {
                        int i = base + lane;
                        bool in = false, is_core = false;
                        if (i < nn) {
                            double a2 = W->u.np.na[i], b2 = W->u.np.nb[i], g2 = W->u.np.ng[i];
                            double mx = -1e300;
#pragma unroll 1
            #pragma unroll 1
                for (int v = 0; v < nv; v++) mx = fmax(mx, a2 * W->ps[cur][v] + b2 * W->pt[cur][v] + g2);
                            in = mx >= -band;
                            is_core = mx >= -tol_max - kCDelta;
                        }
                        unsigned mask = __ballot_sync(full, in);
                        unsigned cmask = __ballot_sync(full, is_core);
                        // compact in place (positions only move down)
                        int pos = nC + __popc(mask & ((1u << lane) - 1u));
                        double r0 = 0, r1 = 0, r2 = 0, r3 = 0, r4 = 0;
                        int rid = 0;
                        if (in) { r0 = W->cn[i][0]; r1 = W->cn[i][1]; r2 = W->cn[i][2]; r3 = W->cn[i][3]; r4 = W->cn[i][4]; rid = W->cid[i]; }
                        __syncwarp();
                        if (in) {
                            W->cn[pos][0] = r0; W->cn[pos][1] = r1; W->cn[pos][2] = r2; W->cn[pos][3] = r3; W->cn[pos][4] = r4;
                            W->cid[pos] = rid;
                        }
                        __syncwarp();
                        unsigned m = mask;
                        int k = nC;
                        while (m && k < CMAX) {
                            int l = __ffs(m) - 1;
                            m &= m - 1;
                            if ((cmask >> l) & 1u) core |= 1ull << k;
                            k++;
                        }
                        nC += __popc(mask);
                    }
                    hinted_done = true;
                }
            }
#ifdef AM_FACE_STATS
            if (!hinted_done) FSTAT(status == 1 ? 53 : status == 2 ? 54 : 55, 1);   // empty / overflow / reach
#endif
            if (!hinted_done) status = 0;   // outside the hint's reach (or degenerate): retry / full path
        }
#ifdef AM_FACE_STATS
        if (!ok) fp_reason = !x0ok ? 1 : 2;
#endif
        if (!ok) break;                    // x0 not on this polygon, or too many near rows: full path
        tau = fmax(A.tau_grow * tau, 2.5 * dmax_seen);   // the polygon reached the square: widen the reach
    }

    PMARK(4);
    if (status == 0 && !hinted_done) {
        const FullOut fo_ = full_path(W, c, U, Vv, P0, tol_c, tol_max, band);
        nv = fo_.nv; cur = fo_.cur; status = fo_.status;
        nC = fo_.nC; core = fo_.core; risky = fo_.risky;
    }
    PMARK(5);
    if (status == 0 && nC > CMAX) status = 2;
    __syncwarp();

    // ------------------------------------- exact vertex semantics on C (core rows)
    int nq = 0;
    if (status == 0) {
        // core row indices, in C order
        int ncore = __popcll(core);
        int P = ncore * (ncore - 1) / 2;
        if (lane == 0) {
            int k = 0;
            for (int r = 0; r < nC; r++)
                if ((core >> r) & 1ull) W->tb[k++] = r;
        }
        __syncwarp();
        for (int base = 0; base < P; base += 32) {
            int p = base + lane;
            bool valid = false;
            double x[3];
            unsigned long long set = 0;
            if (p < P) {
                // triu order: i from 0, j from i+1 (reference cells.py:344 np.triu_indices)
                int ii = 0, rem = p;
                while (rem >= ncore - 1 - ii) { rem -= ncore - 1 - ii; ii++; }
                int jj = ii + 1 + rem;
                int i = W->tb[ii], j = W->tb[jj];
                double Mx[9] = {W->cn[i][0], W->cn[i][1], W->cn[i][2], W->cn[j][0], W->cn[j][1], W->cn[j][2],
                                fu[0], fu[1], fu[2]};
                double rhs[3] = {-W->cn[i][3], -W->cn[j][3], -fo};
                double det = solve3(Mx, rhs, x);
                if (det >= kTolDet) {
                    valid = true;
#pragma unroll 1
                    for (int r = 0; r < nC; r++) {
                        double val = dot3(W->cn[r], x) + W->cn[r][3];
                        if (!(val <= tol_c)) { valid = false; break; }
                        if (fabs(val) <= tol_p) set |= 1ull << r;
                    }
                    set |= (1ull << i) | (1ull << j);
                }
            }
            unsigned mask = __ballot_sync(full, valid);
            int pos = nq + __popc(mask & ((1u << lane) - 1u));
            if (valid && pos < QMAX) {
                W->u.pp.qv[pos][0] = x[0]; W->u.pp.qv[pos][1] = x[1]; W->u.pp.qv[pos][2] = x[2];
                W->u.pp.qs[pos] = set;
            }
            nq += __popc(mask);
        }
        if (nq > QMAX) status = 2;
        else if (nq < 3) status = 1;
        __syncwarp();
    }

    PMARK(6);
    // dedup + ordering (lane 0; a handful of vertices)
    int nr = 0;
    if (status == 0) {
        if (lane == 0) {
            for (int q = 0; q < nq; q++) {
                const double* x = W->u.pp.qv[q];
                int hit = -1;
                for (int k = 0; k < nr; k++) {
                    const double* f = W->u.pp.qv[W->u.pp.rfi[k]];
                    double d0 = f[0] - x[0], d1 = f[1] - x[1], d2 = f[2] - x[2];
                    if (sqrt((d0 * d0 + d1 * d1) + d2 * d2) <= A.tol_weld) { hit = k; break; }
                }
                if (hit < 0) {
                    hit = nr++;
                    W->u.pp.rfi[hit] = q;
                    for (int d = 0; d < 3; d++) W->u.pp.rv[hit][d] = x[d];
                    W->u.pp.rs[hit] = 0;
                } else if (lex_less(x, W->u.pp.rv[hit])) {
                    for (int d = 0; d < 3; d++) W->u.pp.rv[hit][d] = x[d];
                }
                W->u.pp.rs[hit] |= W->u.pp.qs[q];
            }
            W->status = nr;
        }
        __syncwarp();
        nr = W->status;
        if (nr < 3) status = 1;
    }
    if (status == 0) {
        PMARK(7);
        // centroid (reference cells.py:282: verts.mean), angles in the face frame -- lane per vertex
        double cen[3] = {0, 0, 0};
        for (int k = 0; k < nr; k++) { cen[0] += W->u.pp.rv[k][0]; cen[1] += W->u.pp.rv[k][1]; cen[2] += W->u.pp.rv[k][2]; }
        cen[0] /= nr; cen[1] /= nr; cen[2] /= nr;
        double rk = 0.0;
        for (int k = lane; k < nr; k += 32) {
            double r0 = W->u.pp.rv[k][0] - cen[0], r1 = W->u.pp.rv[k][1] - cen[1], r2 = W->u.pp.rv[k][2] - cen[2];
            rk = fmax(rk, sqrt((r0 * r0 + r1 * r1) + r2 * r2));
            W->u.pp.ang[k] = atan2((r0 * Vv[0] + r1 * Vv[1]) + r2 * Vv[2], (r0 * U[0] + r1 * U[1]) + r2 * U[2]);
        }
#pragma unroll
        for (int o2 = 16; o2; o2 >>= 1) rk = fmax(rk, __shfl_xor_sync(full, rk, o2));
        __syncwarp();
        if (nr <= 32) {
            // lane per vertex: stable rank by angle (reference np.argsort kind="stable"), the
            // orientation sum in sorted order on lane 0 (same terms, same order as the serial
            // loop), CCW reversal and rotation to the lexicographically smallest vertex
            const int k = lane;
            int pos = 0;
            if (k < nr) {
                const double ak = W->u.pp.ang[k];
#pragma unroll 1
                for (int j = 0; j < nr; j++) {
                    const double aj = W->u.pp.ang[j];
                    pos += (aj < ak) || (aj == ak && j < k);
                }
                W->u.pp.ord[pos] = k;
            }
            __syncwarp();
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            if (k < nr) {
                const double* pv = W->u.pp.rv[W->u.pp.ord[k]];
                const double* qv = W->u.pp.rv[W->u.pp.ord[k + 1 == nr ? 0 : k + 1]];
                t0 = pv[1] * qv[2] - pv[2] * qv[1];
                t1 = pv[2] * qv[0] - pv[0] * qv[2];
                t2 = pv[0] * qv[1] - pv[1] * qv[0];
            }
            // serial left-to-right sum (bit-identical sign decision)
            double tot[3] = {0, 0, 0};
#pragma unroll 1
            for (int i = 0; i < nr; i++) {
                tot[0] += __shfl_sync(full, t0, i);
                tot[1] += __shfl_sync(full, t1, i);
                tot[2] += __shfl_sync(full, t2, i);
            }
            const double area = 0.5 * ((tot[0] * fu[0] + tot[1] * fu[1]) + tot[2] * fu[2]);
            if (area < 0.0) pos = nr - 1 - pos;
            // lexicographic minimum (first in the final order on ties)
            double m0 = 1e300, m1 = 1e300, m2 = 1e300;
            int mp = 0x7fffffff;
            if (k < nr) { m0 = W->u.pp.rv[k][0]; m1 = W->u.pp.rv[k][1]; m2 = W->u.pp.rv[k][2]; mp = pos; }
#pragma unroll
            for (int o2 = 16; o2; o2 >>= 1) {
                double o0 = __shfl_xor_sync(full, m0, o2), o1 = __shfl_xor_sync(full, m1, o2),
                       oz = __shfl_xor_sync(full, m2, o2);
                int op = __shfl_xor_sync(full, mp, o2);
                bool take = op != 0x7fffffff &&
                            (mp == 0x7fffffff || o0 < m0 || (o0 == m0 && (o1 < m1 || (o1 == m1 && (oz < m2 || (oz == m2 && op < mp))))));
                if (take) { m0 = o0; m1 = o1; m2 = oz; mp = op; }
            }
            if (k < nr) {
                int f = pos - mp;
                if (f < 0) f += nr;
                W->u.pp.fv[f][0] = W->u.pp.rv[k][0]; W->u.pp.fv[f][1] = W->u.pp.rv[k][1]; W->u.pp.fv[f][2] = W->u.pp.rv[k][2];
                W->u.pp.fs[f] = W->u.pp.rs[k];
            }
            if (lane == 0) W->diam = 2.0 * rk;
        } else if (lane == 0) {
            order_serial(W, nr, fu);
            W->diam = 2.0 * rk;
        }
        __syncwarp();
    }

    PMARK(8);
    // per-edge transition planes + mirrored-probe validation (lane per edge)
    if (status == 0) {
        bool need_argmin = false;
        for (int e = lane; e < nr; e += 32) {
            const double* p = W->u.pp.fv[e];
            const double* q = W->u.pp.fv[(e + 1) % nr];
            double mid[3] = {0.5 * (p[0] + q[0]), 0.5 * (p[1] + q[1]), 0.5 * (p[2] + q[2])};
            unsigned long long on_mid = 0;
#pragma unroll 1
            for (int r = 0; r < nC; r++)
                if (((core >> r) & 1ull) && fabs(dot3(W->cn[r], mid) + W->cn[r][3]) <= tol_p) on_mid |= 1ull << r;
            unsigned long long shared = W->u.pp.fs[e] & W->u.pp.fs[(e + 1) % nr];
            unsigned long long rows = shared & on_mid;
            if (!rows) rows = shared ? shared : on_mid;
            W->erow[e] = rows;
            W->eargmin[e] = -1;
            if (!rows) need_argmin = true;
            // validation: a single crossable neuron plane k -> the neighbour's probe lands at
            // mid - delta * n_k (mirror image); it lands in this cell iff every neuron and
            // branch functional keeps the sign of this cell's state there (with margin)
            int ok = 0;
            if (!risky && rows) {
                int ncross = 0, kr = -1;
                unsigned long long m = rows;
                while (m) {
                    int r = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    if (W->cid[r] < box0) { ncross++; kr = r; }
                }
                if (ncross == 1 && W->cid[kr] < c.NB) {
                    double qp[3] = {mid[0] - A.probe_delta * W->cn[kr][0], mid[1] - A.probe_delta * W->cn[kr][1],
                                    mid[2] - A.probe_delta * W->cn[kr][2]};
                    ok = 1;
#pragma unroll 1
                    for (int r = 0; r < nC && ok; r++) {
                        if (W->cid[r] >= box0) continue;
                        double v = dot3(W->cn[r], qp) + W->cn[r][3];
                        if (!(v < -kValMargin && v * W->cn[r][4] < -kValMargin)) ok = 0;
                    }
                }
            }
            W->eval[e] = ok;
        }
        // rare: no plane within tol of the edge -> argmin over every cell row (reference cells.py:327-328)
        unsigned am_mask = __ballot_sync(full, need_argmin);
        __syncwarp();
        if (am_mask) {
            for (int e = 0; e < nr; e++) {
                if (W->erow[e]) continue;
                const double* p = W->u.pp.fv[e];
                const double* q = W->u.pp.fv[(e + 1) % nr];
                double mid[3] = {0.5 * (p[0] + q[0]), 0.5 * (p[1] + q[1]), 0.5 * (p[2] + q[2])};
                double best = 1e300;
                int bi = 0x7fffffff;
                for (int gr = lane; gr < c.K; gr += 32) {
                    double n[3], o;
                    if (!get_row(c, gr, n, o)) continue;
                    double v = fabs(dot3(n, mid) + o);
                    if (v < best) { best = v; bi = gr; }
                }
                for (int o2 = 16; o2; o2 >>= 1) {
                    double ob = __shfl_xor_sync(full, best, o2);
                    int oi = __shfl_xor_sync(full, bi, o2);
                    if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
                }
                if (lane == 0) W->eargmin[e] = bi;
                __syncwarp();
            }
        }
        __syncwarp();
    }

#ifdef AM_FACE_STATS
    {
        long long dt = clock64() - t_start;
        FSTAT(0, 1); FSTAT(1, n_clip1); FSTAT(2, n_clip2); FSTAT(3, nC); FSTAT(4, nq); FSTAT(5, nr);
        FSTAT(6, dt); FSTAT(7, hinted_done ? 1 : 0); FSTAT(13, have_hint ? 1 : 0);
        // path classes: 0 list, one attempt; 1 list, retries; 2 streamed an attempt; 3 full path
        const int cls = !hinted_done ? 3 : n_streamed ? 2 : n_attempts > 1 ? 1 : 0;
        FSTAT(24 + cls, 1); FSTAT(28 + cls, dt); FSTAT(32 + cls, dt > 100000 ? 1 : 0);
        if (cls == 3) FSTAT(36 + (!have_hint ? 0 : fp_reason), 1);
        int bkt = 0;   // log2 histogram from 2^14 cycles, 8 buckets
        while ((1ll << (bkt + 15)) <= dt && bkt < 7) bkt++;
        FSTAT(16 + bkt, 1);
        if (lane == 0 && A.dbg) atomicMax(&A.dbg[8], (unsigned long long)dt);
    }
#endif
    // ------------------------------------------------------------ emit cell
    // lane 0 builds the neighbour descriptors (reference marching.py:152-186, 262-288), then
    // every output range is reserved with one round of independent atomics
    const int32_t pidx = A.pool_idx[fi];
    if (status == 3) {   // deferred: queued again, no record, nothing emitted or validated yet
        if (lane == 0) {
            A.pool_hint[(int64_t)pidx * 4 + 3] = defer_w;
            atomicOr(&A.pool_flags[pidx], kPoolDeferred | kPoolWasDeferred);
            __threadfence();
            const unsigned long long qi = atomicAdd(A.q_tail, 1ull);
            A.queue[qi] = pidx;
            if (A.queue_par) A.queue_par[qi] = 0;
        }
        return;
    }
    if (status != 0) {
        if (lane == 0) {
            int64_t cell = (int64_t)atomicAdd(A.n_cells, 1ull);
            if (status == 2) atomicAdd(&A.overflow[0], 1ull);
            if (cell < A.cap_cells) {
                A.cell_pool[cell] = pidx;
                A.cell_nv[cell] = status == 2 ? -1 : 0;
                A.cell_voff[cell] = 0;
            } else {
                atomicAdd(&A.overflow[1], 1ull);
            }
            A.pool_vn[pidx] = 0;   // processed, nothing validated
        }
        return;
    }
    PMARK(9);
    // lane per edge: transition refs, validated neuron, probe record and the neighbour states
    // of reference marching.py:152-186, 262-288; warp scans give every output offset and lane 0
    // reserves all ranges with one round of independent atomics
    const int NBl = c.NB;
    int tot_ref = 0, tot_val = 0, tot_cd = 0, tot_prec = 0;
#pragma unroll 1
    for (int eb = 0; eb < nr; eb += 32) {
        const int e = eb + lane;
        int nref = 0, nval = 0, ncd = 0, npr = 0;
        if (e < nr) {
            int first = -1, nb = 0, nbr = 0;   // first: global id of crossable[0]
            unsigned long long m = W->erow[e];
            if (m) {
                nref = __popcll(m);
                while (m) {
                    const int r = __ffsll((long long)m) - 1;
                    m &= m - 1;
                    const int gid = W->cid[r];
                    if (gid >= box0) continue;
                    if (first < 0) first = gid;
                    if (gid < NBl) nb++; else nbr++;
                }
            } else {
                nref = 1;
                const int g = W->eargmin[e];
                if (g < box0) { first = g; if (g < NBl) nb = 1; else nbr = 1; }
            }
            nval = W->eval[e];
            if (first >= 0) {
                // flip subsets: all combinations (nb <= 3) or singles + all + none (nb > 3),
                // times (no branch change + each branch target), minus (none, no change)
                npr = 1;
                ncd = (nb > 3 ? nb + 2 : (1 << nb)) * (nbr + 1) - 1;
            }
            W->efirst[e] = first; W->e_nb[e] = nb; W->e_nbr[e] = nbr;
        }
        int t_ref, t_val, t_cd, t_pr;
        const int o_ref = warp_excl_scan(nref, t_ref), o_val = warp_excl_scan(nval, t_val);
        const int o_cd = warp_excl_scan(ncd, t_cd), o_pr = warp_excl_scan(npr, t_pr);
        if (e < nr) {
            W->e_refoff[e] = tot_ref + o_ref; W->e_valoff[e] = tot_val + o_val;
            W->e_cdoff[e] = tot_cd + o_cd; W->eprec[e] = tot_prec + o_pr;
        }
        tot_ref += t_ref; tot_val += t_val; tot_cd += t_cd; tot_prec += t_pr;
    }
    if (lane == 0) {
        W->e_cdoff[nr] = tot_cd;
        const unsigned long long r_cell = atomicAdd(A.n_cells, 1ull);
        const unsigned long long r_vert = atomicAdd(A.n_verts, (unsigned long long)nr);
        const unsigned long long r_ref = atomicAdd(A.n_refs, (unsigned long long)tot_ref);
        const unsigned long long r_val = tot_val ? atomicAdd(A.n_val, (unsigned long long)tot_val) : 0ull;
        const unsigned long long r_cand = tot_cd ? atomicAdd(A.n_cand, (unsigned long long)tot_cd) : 0ull;
        const unsigned long long r_prec = tot_prec ? atomicAdd(A.n_prec, (unsigned long long)tot_prec) : 0ull;
        const int64_t cell = (int64_t)r_cell;
        const bool fits = cell < A.cap_cells && (int64_t)r_vert + nr <= A.cap_verts &&
                          (int64_t)r_ref + tot_ref <= A.cap_refs && (int64_t)r_val + tot_val <= A.cap_val &&
                          (int64_t)r_cand + tot_cd <= A.cap_cand && (int64_t)r_prec + tot_prec <= A.cap_prec;
        if (!fits) {
            atomicAdd(&A.overflow[1], 1ull);
            if (cell < A.cap_cells) { A.cell_pool[cell] = pidx; A.cell_nv[cell] = -2; A.cell_voff[cell] = 0; }
            A.pool_vn[pidx] = 0;
            W->status = -1;
        } else {
            A.cell_pool[cell] = pidx;
            A.cell_nv[cell] = nr;
            A.cell_voff[cell] = (int64_t)r_vert;
            A.pool_voff[pidx] = (int64_t)r_val;
            A.pool_vn[pidx] = tot_val;
            W->status = 0;
            W->obase[0] = (long long)r_vert; W->obase[1] = (long long)r_ref; W->obase[2] = (long long)r_val;
            W->obase[3] = (long long)r_cand; W->obase[4] = (long long)r_prec;
        }
    }
    __syncwarp();
    if (W->status < 0) return;
    const int64_t voff = W->obase[0], roff = W->obase[1], vloff = W->obase[2], cbase = W->obase[3],
                  pbase = W->obase[4];
    PMARK(10);
    // per-edge records (lane per edge)
#pragma unroll 1
    for (int e = lane; e < nr; e += 32) {
        const double* p = W->u.pp.fv[e];
        const double* q = W->u.pp.fv[e + 1 == nr ? 0 : e + 1];
        A.verts[(voff + e) * 3 + 0] = p[0];
        A.verts[(voff + e) * 3 + 1] = p[1];
        A.verts[(voff + e) * 3 + 2] = p[2];
        int64_t ro = roff + W->e_refoff[e];
        A.edge_roff[voff + e] = ro;
        int cnt = 0, kn = -1;
        unsigned long long m = W->erow[e];
        if (m) {
            while (m) {
                const int r = __ffsll((long long)m) - 1;
                m &= m - 1;
                const int gid = W->cid[r];
                A.edge_refs[ro++] = gid;
                cnt++;
                if (gid < box0) kn = gid;
            }
        } else {
            A.edge_refs[ro++] = W->eargmin[e];
            cnt = 1;
        }
        A.edge_nrefs[voff + e] = cnt;
        if (W->eval[e]) A.val_buf[vloff + W->e_valoff[e]] = kn;   // the edge's single crossable neuron
        const int first = W->efirst[e];
        if (first < 0) continue;
        // probe across crossable[0] (reference marching.py:271-276) as a probe record: a
        // single-neuron edge points at its lone flip (resolved by that cell's mirrored
        // validation); any other edge is a forced exact forward evaluation (cand = -1)
        double pn[3], po_;
        int pr = -1;
#pragma unroll 1
        for (int r = 0; r < nC; r++)
            if (W->cid[r] == first) { pr = r; break; }
        if (pr >= 0) { pn[0] = W->cn[pr][0]; pn[1] = W->cn[pr][1]; pn[2] = W->cn[pr][2]; }
        else get_row(c, first, pn, po_);
        const int64_t po = pbase + W->eprec[e];
        A.prec_pt[po * 3 + 0] = 0.5 * (p[0] + q[0]) + A.probe_delta * pn[0];
        A.prec_pt[po * 3 + 1] = 0.5 * (p[1] + q[1]) + A.probe_delta * pn[1];
        A.prec_pt[po * 3 + 2] = 0.5 * (p[2] + q[2]) + A.probe_delta * pn[2];
        A.prec_k[po] = first;
        const bool single = W->e_nb[e] == 1 && W->e_nbr[e] == 0;
        A.prec_cand[po] = single ? (int32_t)(cbase + W->e_cdoff[e]) : -1;
        if (A.prec_s) A.prec_s[po] = item_shape(c.key, A.shape_w);
    }
    PMARK(11);
    // neighbour keys, one (candidate, word) per thread: coalesced over the cell's candidates
    const int KW = A.KW;
    const int n_words = tot_cd * KW;
#pragma unroll 1
    for (int idx = lane; idx < n_words; idx += 32) {
        const int k = idx / KW, w = idx - k * KW;
        int lo = 0, hi = nr - 1;   // edge of candidate k: last e with e_cdoff[e] <= k
        while (lo < hi) {
            const int md = (lo + hi + 1) >> 1;
            if (W->e_cdoff[md] <= k) lo = md; else hi = md - 1;
        }
        const int e = lo;
        const int j = k - W->e_cdoff[e];
        const int nb = W->e_nb[e], nbr = W->e_nbr[e];
        const bool big = nb > 3;
        // position in the (subset, branch target) enumeration with the skipped (none, no change)
        const int pos = big ? (j < (nb + 1) * (nbr + 1) ? j : j + 1) : j + 1;
        const int si = pos / (nbr + 1), ti = pos % (nbr + 1) - 1;
        const unsigned sub = nb == 3 ? kComb3[si] : (unsigned)si;   // combination order for nb <= 3
        uint64_t word = c.key[w];
        int branch = -1, in_ = 0, ib = 0, gmin = NBl;
        auto visit = [&](int gid) {
            if (gid >= box0) return;
            if (gid < NBl) {
                const bool fl = big ? (si < nb ? in_ == si : si == nb) : ((sub >> in_) & 1u);
                if (fl && (gid >> 6) == w) word ^= key_mask(gid);
                if (fl && gid < gmin) gmin = gid;
                in_++;
            } else {
                if (ib == ti) branch = gid - NBl;
                ib++;
            }
        };
        unsigned long long m = W->erow[e];
        if (m) {
            while (m) {
                const int r = __ffsll((long long)m) - 1;
                m &= m - 1;
                visit(W->cid[r]);
            }
        } else {
            visit(W->eargmin[e]);
        }
        if (A.ensemble && w == KW - 1 && branch >= 0) word = (uint64_t)branch;
        const int64_t ci = cbase + k;
        A.cand[ci * KW + w] = word;
        if (w == 0) {
            // hint for the neighbour: midpoint of the shared edge + search radius
            const double* p = W->u.pp.fv[e];
            const double* q = W->u.pp.fv[e + 1 == nr ? 0 : e + 1];
            reinterpret_cast<double4*>(A.emit_hint)[ci] =
                make_double4(0.5 * (p[0] + q[0]), 0.5 * (p[1] + q[1]), 0.5 * (p[2] + q[2]), 2.0 * W->diam + 1e-9);
            if (A.emit_par) {
                // prefix reuse: the child shares Z rows of steps 0..f with this cell (f: step of
                // its first flipped neuron; a branch-only change shares nothing)
                int f = 0;
                if (gmin < NBl && branch < 0) {
                    while (f + 1 < A.nsteps && A.step_end[f] <= gmin) f++;
                }
                A.emit_par[ci] = f ? prefix_word(*A.zpar, item, f) : 0;
            }
        }
    }
    if (A.fused_upsert && tot_cd) {
        // the flips go straight into the state set (k_hash_upsert's work, one candidate per
        // lane): their key rows must be visible device-wide before a slot marker can point at them
        __threadfence();
        __syncwarp();
#pragma unroll 1
        for (int k = lane; k < tot_cd; k += 32) {
            const int64_t ci = cbase + k;
            int32_t p;
            A.cand_status[ci] = upsert_one(A.H, A.cand, nullptr, ci, ci, A.cand_slot, A.cand_dup, 0u, A.ins_queue,
                                           A.q_tail, A.emit_hint, &p, A.emit_par);
            A.cand_pool[ci] = p;
        }
    }
    PMARK(12);
}

// Near lists: one warp per frontier cell streams every constraint row once (coalesced 32 B
// rows of the composition buffer, the same test as the face solver's hinted pass) and keeps the
// rows within reach = near_reach x the hint radius of the hint point, in ascending id order,
// with their raw functionals.  Full-occupancy warps keep many row loads in flight; the face
// solver then filters ~tens of listed rows per attempt instead of streaming all K rows.
// face work order: heavy cells from the front, light ones from the back (longest chains first)
__device__ __forceinline__ void place_cell(const FaceArgs& A, int64_t n, int64_t fi, bool heavy) {
    if (!A.order) return;
    if (heavy) A.order[atomicAdd(&A.order_ctr[0], 1ull)] = (int32_t)fi;
    else A.order[n - 1 - (int64_t)atomicAdd(&A.order_ctr[1], 1ull)] = (int32_t)fi;
}

template <int D>
#ifndef AM_NEAR_MINB
#define AM_NEAR_MINB 1
#endif
__global__ void __launch_bounds__(256, AM_NEAR_MINB) k_near(FaceArgs A) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int64_t n = dev_count(A.n_dev, A.n_cap);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t fi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; fi < n; fi += nw) {
        const int item = A.items[fi];
        Ctx c;
        c.Z = zbase(A) + (int64_t)item * A.zs * 4;
        c.faces = A.faces + (int64_t)item * A.M * 4;
        c.key = A.keys + (int64_t)item * A.KW;
        c.NB = A.NB; c.M = A.M; c.ensemble = A.ensemble;
        c.branch = A.ensemble ? (int)c.key[A.KW - 1] : 0;
        c.K = A.NB + A.M + 6;
        for (int k = 0; k < 3; k++) { c.lo[k] = A.lo[k]; c.hi[k] = A.hi[k]; }
        NearOut o{A.near_n, A.near_flags, A.near_id, A.near_row, A.near_cap};
        bool heavy = false;
        near_list<true, D>(c, reinterpret_cast<const double4*>(A.hints)[item], A.tol_cell, A.tol_onplane,
                           A.probe_delta, A.near_reach, o, fi, heavy);
        if (lane == 0) place_cell(A, n, fi, heavy);
    }
}

template <int D>
static void launch_near_d(const FaceArgs& a, cudaStream_t s) {
    static int grid_max[64] = {};   // per device
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev >= 0 && dev < 64 ? dev : 0;
    if (!grid_max[di]) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_near<D>, 256, 0);
        if (const char* v = getenv("AM_NEAR_CTAS")) per_sm = std::min(per_sm, std::max(1, atoi(v)));
        grid_max[di] = device_sms() * (per_sm > 0 ? per_sm : 1);
    }
    const int64_t blocks = (a.n_cap + 7) / 8;   // a warp per frontier entry
    launch_k(k_near<D>, (unsigned)(blocks < grid_max[di] ? blocks : grid_max[di]), 256, 0, s, a);
}

void launch_near(const FaceArgs& a, cudaStream_t s) {
    if (a.n_cap <= 0 || !a.near_flags) return;
    if (a.near_depth >= 4) launch_near_d<4>(a, s);
    else launch_near_d<2>(a, s);
}

// persistent: each warp walks the device-resident frontier
__global__ void __launch_bounds__(FW * 32, 4) k_face(FaceArgs A) {
    pdl_enter();
    extern __shared__ uint8_t smem_raw[];
    FaceWarp* W = reinterpret_cast<FaceWarp*>(smem_raw) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int64_t n = dev_count(A.n_dev, A.n_cap);
    // dynamic work distribution: cell latencies vary by 10x, so warps pull cells from a cursor
    for (;;) {
        int64_t fi = 0;
        if (lane == 0) {
            fi = (int64_t)atomicAdd(A.cursor, 1ull);
            if (fi < n && A.order) fi = A.order[fi];
            else if (fi >= n) fi = n;
        }
        fi = __shfl_sync(0xffffffffu, fi, 0);
        if (fi >= n) break;
        face_cell(A, W, fi, n);
        __syncwarp();
    }
}

void launch_face(const FaceArgs& a, cudaStream_t s) {
    if (a.n_cap <= 0) return;
    size_t smem = sizeof(FaceWarp) * FW;
    static int grids[64] = {};   // per device: the smem attribute and occupancy are per device
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev >= 0 && dev < 64 ? dev : 0;
    if (!grids[di]) {
        cudaFuncSetAttribute(k_face, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_face, FW * 32, smem);
        // resident CTAs per SM: the per-cell latency chain, not issue throughput, bounds an
        // iteration (waves of ~2.5 k cells on ~1.8 k warps), and more warps per SM lengthen it
        int want = kFaceCtasPerSm;
        if (const char* v = getenv("AM_FACE_CTAS")) want = atoi(v);
        if (want > 0 && want < per_sm) per_sm = want;
        grids[di] = device_sms() * (per_sm > 0 ? per_sm : 1);
    }
    const int grid = grids[di];
    int64_t need = (a.n_cap + FW - 1) / FW;
    { launch_k(k_face, (unsigned)(need < grid ? need : grid), FW * 32, smem, s, a); }
}

}  // namespace am
