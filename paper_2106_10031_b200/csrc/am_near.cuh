// am_near.cuh -- a cell's constraint rows and its near list, shared by the face solver
// (am_face.cu: k_near, k_face) and the narrow composition (am_narrow.cu), which builds the near
// lists of its tile while the tile's rows are still in L2.
//
// Near list: the rows within reach = near_reach x the hint radius of the hint point projected on
// the face plane, in ascending id order, with their raw functionals (one warp per cell, every
// constraint row streamed once).  The face solver then filters ~tens of listed rows per attempt
// instead of streaming all K rows.
#pragma once

#include "am_internal.h"

namespace am {

constexpr double kTinyNorm = 1e-6;     // rows this thin make validation unreliable
constexpr int kNearValid = 1, kNearX0Bad = 2, kNearRisky = 4, kNearOverflow = 8;

struct Ctx {
    const double* Z;   // this item's rows
    const double* faces;
    const uint64_t* key;
    int NB, M, branch, ensemble, K;
    double lo[3], hi[3];
};

// raw functional of global plane id gr (not normalised, not oriented); kind: 0 neuron,
// 1 branch (valid unless it is the cell's own branch), 2 box, -1 none
struct RawRow { double x, y, z, c; int kind; };
// branch-dominance, box and padding rows (a handful per cell): out of line
static __device__ __noinline__ RawRow load_raw_other(const Ctx& c, int gr) {
    RawRow r;
    if (gr < c.NB + c.M) {
        int t = gr - c.NB;
        r.kind = (!c.ensemble || t == c.branch) ? -1 : 1;
        if (r.kind == 1) {
            const double* ft = c.faces + t * 4;
            const double* fj = c.faces + c.branch * 4;
            r.x = ft[0] - fj[0]; r.y = ft[1] - fj[1]; r.z = ft[2] - fj[2]; r.c = ft[3] - fj[3];
        } else {
            r.x = r.y = r.z = r.c = 0.0;
        }
    } else if (gr < c.K) {
        int k = gr - c.NB - c.M, ax = k >> 1;
        r.x = r.y = r.z = 0.0;
        double sg = (k & 1) ? -1.0 : 1.0;
        if (ax == 0) r.x = sg; else if (ax == 1) r.y = sg; else r.z = sg;
        r.c = (k & 1) ? c.lo[ax] : -c.hi[ax];
        r.kind = 2;
    } else {
        r.x = r.y = r.z = r.c = 0.0;
        r.kind = -1;
    }
    return r;
}
// NC: rows written by an earlier kernel (read-only path); !NC: written earlier in this kernel
template <bool NC = true>
__device__ __forceinline__ RawRow load_raw(const Ctx& c, int gr) {
    if (gr < c.NB) {
        RawRow r;
        const double2* p = reinterpret_cast<const double2*>(c.Z + (int64_t)gr * 4);
        double2 a, b;
        if (NC) { a = __ldg(p); b = __ldg(p + 1); }
        else { a = p[0]; b = p[1]; }
        r.x = a.x; r.y = a.y; r.z = b.x; r.c = b.y; r.kind = 0;
        return r;
    }
    return load_raw_other(c, gr);
}

struct NearOut {
    int32_t* n;
    int32_t* flags;
    int32_t* id;        // [slot][cap]
    double* row;        // [slot][cap][4]
    int cap;
};

// Warp-collective: the near list of the cell in c, written at `slot`.  heavy (lane-uniform):
// the face solver's slow paths are certain (no usable hint with a face, x0 outside the cell, or
// a list overflow).
template <bool NC, int D = 2>   // D: row batches of 32 in flight per warp
__device__ __forceinline__ void near_list(const Ctx& c, double4 hint, double tol_cell, double tol_onplane,
                                          double probe_delta, double near_reach, const NearOut& o, int64_t slot,
                                          bool& heavy) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    // face plane and projected hint point: the face solver's arithmetic
    const double* fr = c.faces + c.branch * 4;
    const double fn = sqrt((fr[0] * fr[0] + fr[1] * fr[1]) + fr[2] * fr[2]);
    double fu[3] = {0, 0, 0}, fo = 0.0;
    bool face_ok = fn > kDegen;
    if (face_ok) {
        fu[0] = fr[0] / fn; fu[1] = fr[1] / fn; fu[2] = fr[2] / fn; fo = fr[3] / fn;
        face_ok = sqrt((fu[0] * fu[0] + fu[1] * fu[1]) + fu[2] * fu[2]) > kDegen;
    }
    if (!(isfinite(hint.w) && face_ok)) {
        if (lane == 0) o.flags[slot] = 0;
        heavy = face_ok;   // no hint: the full two-pass path; empty face: quick
        return;
    }
    const double hd = ((fu[0] * hint.x + fu[1] * hint.y) + fu[2] * hint.z) + fo;
    hint.x -= hd * fu[0]; hint.y -= hd * fu[1]; hint.z -= hd * fu[2];
    const double x0[3] = {hint.x, hint.y, hint.z};
    const double band = fmax(tol_cell, tol_onplane) + 1.5 * probe_delta + 1e-9;
    const double lim = near_reach * hint.w + band + 1e-9;
    const int64_t lb = slot * (int64_t)o.cap;
    int nn = 0, risky = 0;
    bool ok = true;
    RawRow nx[D];
#pragma unroll
    for (int d = 0; d < D; d++) nx[d] = load_raw<NC>(c, lane + 32 * d);
    for (int base = 0; base < c.K; base += 32) {
        const int gr = base + lane;
        const RawRow rr = nx[0];
#pragma unroll
        for (int d = 0; d + 1 < D; d++) nx[d] = nx[d + 1];
        if (base + 32 * D < c.K) nx[D - 1] = load_raw<NC>(c, gr + 32 * D);
        bool near = false;
        if (gr < c.K && rr.kind >= 0) {
            const double n2 = (rr.x * rr.x + rr.y * rr.y) + rr.z * rr.z;
            if (rr.kind == 0 && n2 > 0.0 && n2 < kTinyNorm * kTinyNorm) risky = 1;
            if (rr.kind == 1 && n2 < kTinyNorm * kTinyNorm) risky = 1;
            if (rr.kind == 2 || n2 > kDegen * kDegen) {
                double v = ((rr.x * x0[0] + rr.y * x0[1]) + rr.z * x0[2]) + rr.c;
                if (rr.kind == 0 && key_bit(c.key, gr)) v = -v;
                if (v > 0.0 && v * v > 1e-18 * n2) ok = false;   // x0 violates the row by > 1e-9
                near = v >= 0.0 || v * v <= lim * lim * n2;
            }
        }
        const unsigned mask = __ballot_sync(full, near);
        const int pos = nn + __popc(mask & ((1u << lane) - 1u));
        if (near && pos < o.cap) {
            o.id[lb + pos] = gr;
            reinterpret_cast<double4*>(o.row)[lb + pos] = make_double4(rr.x, rr.y, rr.z, rr.c);
        }
        nn += __popc(mask);
    }
    ok = __all_sync(full, ok);
    risky = __any_sync(full, risky);
    if (lane == 0) {
        o.n[slot] = nn < o.cap ? nn : o.cap;
        o.flags[slot] = kNearValid | (ok ? 0 : kNearX0Bad) | (risky ? kNearRisky : 0) | (nn > o.cap ? kNearOverflow : 0);
    }
    heavy = !ok || nn > o.cap;
}

}  // namespace am
