// am_seed.cu -- seed refinement and bisection triggering, batched over seeds.
// reference marching.py:201-213 (_refine_seed_state), seeding.py:84-112 (seed_dichotomy)
#include "am_internal.h"

namespace am {

static inline unsigned nb(int64_t n) { return (unsigned)((n + 127) / 128); }

// x_proj = x - (n.x + c)/nn * n on the face plane of canonical(s); nn <= 0 -> done
__global__ void k_seed_project(const double* X, const double* faces, const uint64_t* keys, int KW, int M,
                               int ensemble, int64_t n, const int32_t* active, double* Xp, int32_t* done_flat) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    done_flat[i] = 0;
    if (!active[i]) return;
    int br = ensemble ? (int)keys[i * KW + KW - 1] : 0;
    const double* f = faces + (i * M + br) * 4;
    const double* x = X + i * 3;
    double nn = (f[0] * f[0] + f[1] * f[1]) + f[2] * f[2];
    if (nn <= 0.0) { done_flat[i] = 1; return; }
    double t = (((f[0] * x[0] + f[1] * x[1]) + f[2] * x[2]) + f[3]) / nn;
    Xp[i * 3 + 0] = x[0] - t * f[0];
    Xp[i * 3 + 1] = x[1] - t * f[1];
    Xp[i * 3 + 2] = x[2] - t * f[2];
}

// snew == null: finalize active seeds flagged in done_flat (or all active if done_flat null)
// with result = canon.  Otherwise: snew == canon -> result = canon, inactive; else x = xp, s = snew.
__global__ void k_seed_check(const uint64_t* snew, const uint64_t* canon, int KW, int64_t n, int32_t* active,
                             double* X, const double* Xp, uint64_t* S, uint64_t* result, int32_t* done_flat) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !active[i]) return;
    if (!snew) {
        if (done_flat && !done_flat[i]) return;
        for (int w = 0; w < KW; w++) result[i * KW + w] = canon[i * KW + w];
        active[i] = 0;
        return;
    }
    bool eq = true;
    for (int w = 0; w < KW; w++) eq &= snew[i * KW + w] == canon[i * KW + w];
    if (eq) {
        for (int w = 0; w < KW; w++) result[i * KW + w] = canon[i * KW + w];
        active[i] = 0;
    } else {
        X[i * 3 + 0] = Xp[i * 3 + 0]; X[i * 3 + 1] = Xp[i * 3 + 1]; X[i * 3 + 2] = Xp[i * 3 + 2];
        for (int w = 0; w < KW; w++) S[i * KW + w] = snew[i * KW + w];
    }
}

void launch_seed_project(const double* X, const double* faces, const uint64_t* keys, int KW, int M, int ensemble,
                         int64_t n, const int32_t* active, double* Xp, int32_t* done_flat, cudaStream_t s) {
    if (n > 0) { launch_k(k_seed_project, nb(n), 128, 0, s, X, faces, keys, KW, M, ensemble, n, active, Xp, done_flat); }
}
void launch_seed_check(const uint64_t* snew, const uint64_t* canon, int KW, int64_t n, int32_t* active, double* X,
                       const double* Xp, uint64_t* S, uint64_t* result, int32_t* done_flat, cudaStream_t s) {
    if (n > 0) { launch_k(k_seed_check, nb(n), 128, 0, s, snew, canon, KW, n, active, X, Xp, S, result, done_flat); }
}

// one bisection step given F(mid) (reference seeding.py:96-112)
__global__ void k_dichotomy_step(const double* vals, double* xp, double* xn, double* fp, double* fn, double* mid,
                                 int32_t* active, double* out, int64_t n, double eps, double seed_tol, int last) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !active[i]) return;
    double fm = vals[i];
    double* m = mid + i * 3;
    if (fabs(fm) <= seed_tol) {
        out[i * 3 + 0] = m[0]; out[i * 3 + 1] = m[1]; out[i * 3 + 2] = m[2];
        active[i] = 0;
        return;
    }
    if (fm > 0.0) { xp[i * 3] = m[0]; xp[i * 3 + 1] = m[1]; xp[i * 3 + 2] = m[2]; fp[i] = fm; }
    else { xn[i * 3] = m[0]; xn[i * 3 + 1] = m[1]; xn[i * 3 + 2] = m[2]; fn[i] = fm; }
    if (fp[i] - fn[i] <= eps || last) {
        const double* src = fabs(fp[i]) <= fabs(fn[i]) ? xp + i * 3 : xn + i * 3;
        out[i * 3 + 0] = src[0]; out[i * 3 + 1] = src[1]; out[i * 3 + 2] = src[2];
        active[i] = 0;
        return;
    }
    m[0] = 0.5 * (xp[i * 3] + xn[i * 3]);
    m[1] = 0.5 * (xp[i * 3 + 1] + xn[i * 3 + 1]);
    m[2] = 0.5 * (xp[i * 3 + 2] + xn[i * 3 + 2]);
}
void launch_dichotomy_step(const double* vals, double* xp, double* xn, double* fp, double* fn, double* mid,
                           int32_t* active, double* out, int64_t n, double eps, double seed_tol, int last,
                           cudaStream_t s) {
    if (n > 0) { launch_k(k_dichotomy_step, nb(n), 128, 0, s, vals, xp, xn, fp, fn, mid, active, out, n, eps, seed_tol, last); }
}

// ---------------------------------------------- speculative bisection tree (exact)
// The bisection's next D midpoints lie in a binary tree of 2^D - 1 points fixed by (xp, xn):
// node 0 = 0.5 (xp + xn); the children of a node m of interval {a, b} are the midpoints of
// {m, xn-side} (taken when F(m) > 0, xp := m) and {xp-side, m}.  Every node is formed with the
// bisection's own arithmetic (0.5 (l + r); addition commutes, so the midpoint of an interval
// does not depend on which end is xp), and F is evaluated per point, so replaying the
// reference's step rule through the tree (k_bisect_replay) visits exactly the points and values
// of D sequential steps -- with one batched forward instead of D.
constexpr int kTreeD = 5, kTreeN = (1 << kTreeD) - 1;

// node k (heap order: children of k are 2k+1 (F > 0: xp := m) and 2k+2 (F <= 0: xn := m))
__global__ void k_bisect_tree(const double* xp, const double* xn, const int32_t* active, int64_t n, double* nodes) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double* out = nodes + i * kTreeN * 3;
    double lp[kTreeN][3], ln[kTreeN][3];   // interval (xp side, xn side) of every node
    for (int d = 0; d < 3; d++) { lp[0][d] = xp[i * 3 + d]; ln[0][d] = xn[i * 3 + d]; }
    for (int k = 0; k < kTreeN; k++) {
        double m[3];
        for (int d = 0; d < 3; d++) { m[d] = 0.5 * (lp[k][d] + ln[k][d]); out[k * 3 + d] = m[d]; }
        const int c0 = 2 * k + 1, c1 = 2 * k + 2;
        if (c0 < kTreeN) for (int d = 0; d < 3; d++) { lp[c0][d] = m[d]; ln[c0][d] = ln[k][d]; }
        if (c1 < kTreeN) for (int d = 0; d < 3; d++) { lp[c1][d] = lp[k][d]; ln[c1][d] = m[d]; }
    }
    (void)active;
}

// D steps of reference seeding.py:96-112 per active pair along the evaluated tree
__global__ void k_bisect_replay(const double* vals, const double* nodes, double* xp, double* xn, double* fp,
                                double* fn, int32_t* active, double* out, int64_t n, int it0, int max_iters,
                                double eps, double seed_tol) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !active[i]) return;
    int k = 0;
    for (int lvl = 0; lvl < kTreeD; lvl++) {
        const int it = it0 + lvl;
        const double fm = vals[i * kTreeN + k];
        const double* m = nodes + (i * kTreeN + k) * 3;
        if (fabs(fm) <= seed_tol) {
            out[i * 3 + 0] = m[0]; out[i * 3 + 1] = m[1]; out[i * 3 + 2] = m[2];
            active[i] = 0;
            return;
        }
        if (fm > 0.0) { xp[i * 3] = m[0]; xp[i * 3 + 1] = m[1]; xp[i * 3 + 2] = m[2]; fp[i] = fm; k = 2 * k + 1; }
        else { xn[i * 3] = m[0]; xn[i * 3 + 1] = m[1]; xn[i * 3 + 2] = m[2]; fn[i] = fm; k = 2 * k + 2; }
        if (fp[i] - fn[i] <= eps || it == max_iters) {
            const double* src = fabs(fp[i]) <= fabs(fn[i]) ? xp + i * 3 : xn + i * 3;
            out[i * 3 + 0] = src[0]; out[i * 3 + 1] = src[1]; out[i * 3 + 2] = src[2];
            active[i] = 0;
            return;
        }
    }
}

void launch_bisect_tree(const double* xp, const double* xn, const int32_t* active, int64_t n, double* nodes,
                        cudaStream_t s) {
    if (n > 0) { launch_k(k_bisect_tree, nb(n), 128, 0, s, xp, xn, active, n, nodes); }
}
void launch_bisect_replay(const double* vals, const double* nodes, double* xp, double* xn, double* fp, double* fn,
                          int32_t* active, double* out, int64_t n, int it0, int max_iters, double eps,
                          double seed_tol, cudaStream_t s) {
    if (n > 0) {
        launch_k(k_bisect_replay, nb(n), 128, 0, s, vals, nodes, xp, xn, fp, fn, active, out, n, it0, max_iters, eps,
                 seed_tol);
    }
}
int bisect_tree_points() { return kTreeN; }
int bisect_tree_depth() { return kTreeD; }

}  // namespace am

namespace am {
__global__ void k_midpoint(const double* a, const double* b, double* m, int64_t n) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n * 3) m[i] = 0.5 * (a[i] + b[i]);
}
void launch_midpoint(const double* a, const double* b, double* m, int64_t n, cudaStream_t s) {
    if (n > 0) { launch_k(k_midpoint, (unsigned)((n * 3 + 127) / 128), 128, 0, s, a, b, m, n); }
}
// hint records (x, y, z, reach) of points that lie in their cells (seeds)
__global__ void k_point_hints(const double* X, int64_t n, double tau, double* hints) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) reinterpret_cast<double4*>(hints)[i] = make_double4(X[i * 3], X[i * 3 + 1], X[i * 3 + 2], tau);
}
void launch_point_hints(const double* X, int64_t n, double tau, double* hints, cudaStream_t s) {
    if (n > 0) { launch_k(k_point_hints, (unsigned)((n + 127) / 128), 128, 0, s, X, n, tau, hints); }
}
__global__ void k_count_active(const int32_t* active, int64_t n, unsigned long long* cnt) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && active[i]) atomicAdd(cnt, 1ull);
}
void launch_count_active(const int32_t* active, int64_t n, unsigned long long* cnt, cudaStream_t s) {
    if (n > 0) { launch_k(k_count_active, (unsigned)((n + 127) / 128), 128, 0, s, active, n, cnt); }
}
}  // namespace am
