// am_trace.cu -- the iterative trigger schemes on the device (reference seeding.py:35-77).
//
//   sgd           x <- x - cur * sign(F) * g / |g| with g = grad F (the face normal of the region
//                 containing x); cur halves whenever F changes sign; converged when |F| <= tol
//   sphere_trace  x <- x - eta * F * g; converged when |F| <= tol; diverged (the reference
//                 raises) when the iterate leaves escape_scale x the unit box
//
// Every start point is an independent lane of state (x, F, cur, status); the engine drives
// all of them in lockstep with device-resident forwards (F and the activation state) and
// affine-map compositions (the gradient), synchronising with the host only every few steps to
// test whether any start is still running.  The update arithmetic is the reference's, step for
// step and in its evaluation order, compiled with -fmad=false (separately rounded products and
// sums, as numpy evaluates them).
#include "am_internal.h"

namespace am {

namespace {

__device__ __forceinline__ double sgn(double v) { return (double)((v > 0.0) - (v < 0.0)); }

// face normal of the region containing point i: its branch's face functional (ensembles)
__device__ __forceinline__ const double* grad_of(const double* faces, const uint64_t* keys, int64_t i, int KW,
                                                 int M, int bw_branch) {
    const int br = bw_branch >= 0 ? (int)keys[i * KW + bw_branch] : 0;
    return faces + (i * M + br) * 4;
}

// status: 0 running, 1 converged, 2 diverged (sphere tracing), 3 stopped (zero gradient / out of
// iterations)
__global__ void k_trace_init(int64_t n, const double* x0, double* x, double* cur, double step, int32_t* status,
                             int32_t* iters) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int d = 0; d < 3; d++) x[i * 3 + d] = x0[i * 3 + d];
        cur[i] = step;
        status[i] = 0;
        iters[i] = 0;
    }
}

// sgd, top of iteration `it`: converged when |F| <= tol
__global__ void k_sgd_check(int64_t n, const double* f, int32_t* status, int32_t* iters, int it, double tol,
                            unsigned long long* running) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        if (fabs(f[i]) <= tol) { status[i] = 1; iters[i] = it; continue; }
        atomicAdd(running, 1ull);
    }
}

// sgd: proposal x_new = x - cur * sign(f) * g / |g| (reference seeding.py:49-56)
__global__ void k_sgd_propose(int64_t n, const double* x, const double* f, const double* faces, const uint64_t* keys,
                              int KW, int M, int bw_branch, const double* cur, int32_t* status, double* xn) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        const double* g = grad_of(faces, keys, i, KW, M, bw_branch);
        const double gn = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
        if (gn == 0.0) { status[i] = 3; continue; }
        const double a = cur[i] * sgn(f[i]);
        for (int d = 0; d < 3; d++) xn[i * 3 + d] = x[i * 3 + d] - (a * g[d]) / gn;
    }
}

// sgd: accept the proposal; the step halves when F changed sign
__global__ void k_sgd_accept(int64_t n, double* x, double* f, uint64_t* keys, const double* xn, const double* fn,
                             const uint64_t* keysn, int KW, double* cur, const int32_t* status) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        if (sgn(fn[i]) != sgn(f[i])) cur[i] *= 0.5;
        for (int d = 0; d < 3; d++) x[i * 3 + d] = xn[i * 3 + d];
        f[i] = fn[i];
        for (int w = 0; w < KW; w++) keys[i * KW + w] = keysn[i * KW + w];
    }
}

// sphere tracing, after F(x): converged / diverged tests of iteration `it` (reference
// seeding.py:68-76)
__global__ void k_sphere_check(int64_t n, const double* x, const double* f, int32_t* status, int32_t* iters, int it,
                               double tol, double escape, unsigned long long* running) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        if (fabs(f[i]) <= tol) { status[i] = 1; iters[i] = it; continue; }
        const double m = fmax(fmax(fabs(x[i * 3]), fabs(x[i * 3 + 1])), fabs(x[i * 3 + 2]));
        if (m > escape) { status[i] = 2; iters[i] = it; continue; }
        atomicAdd(running, 1ull);
    }
}

// sphere tracing step x <- x - eta * F * g
__global__ void k_sphere_step(int64_t n, double* x, const double* f, const double* faces, const uint64_t* keys,
                              int KW, int M, int bw_branch, double eta, const int32_t* status) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        const double* g = grad_of(faces, keys, i, KW, M, bw_branch);
        const double a = eta * f[i];
        for (int d = 0; d < 3; d++) x[i * 3 + d] = x[i * 3 + d] - a * g[d];
    }
}

__global__ void k_trace_finish(int64_t n, const double* x, int32_t* status, double* out) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (status[i] == 0) status[i] = 3;   // out of iterations
        for (int d = 0; d < 3; d++) out[i * 3 + d] = x[i * 3 + d];
    }
}

unsigned blocks_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 1184)); }

}  // namespace

void launch_trace_init(int64_t n, const double* x0, double* x, double* cur, double step, int32_t* status,
                       int32_t* iters, cudaStream_t s) {
    launch_k(k_trace_init, blocks_for(n), 128, 0, s, n, x0, x, cur, step, status, iters);
}
void launch_sgd_check(int64_t n, const double* f, int32_t* status, int32_t* iters, int it, double tol,
                      unsigned long long* running, cudaStream_t s) {
    launch_k(k_sgd_check, blocks_for(n), 128, 0, s, n, f, status, iters, it, tol, running);
}
void launch_sgd_propose(int64_t n, const double* x, const double* f, const double* faces, const uint64_t* keys, int KW,
                        int M, int bw_branch, const double* cur, int32_t* status, double* xn, cudaStream_t s) {
    launch_k(k_sgd_propose, blocks_for(n), 128, 0, s, n, x, f, faces, keys, KW, M, bw_branch, cur, status, xn);
}
void launch_sgd_accept(int64_t n, double* x, double* f, uint64_t* keys, const double* xn, const double* fn,
                       const uint64_t* keysn, int KW, double* cur, const int32_t* status, cudaStream_t s) {
    launch_k(k_sgd_accept, blocks_for(n), 128, 0, s, n, x, f, keys, xn, fn, keysn, KW, cur, status);
}
void launch_sphere_check(int64_t n, const double* x, const double* f, int32_t* status, int32_t* iters, int it,
                         double tol, double escape, unsigned long long* running, cudaStream_t s) {
    launch_k(k_sphere_check, blocks_for(n), 128, 0, s, n, x, f, status, iters, it, tol, escape, running);
}
void launch_sphere_step(int64_t n, double* x, const double* f, const double* faces, const uint64_t* keys, int KW,
                        int M, int bw_branch, double eta, const int32_t* status, cudaStream_t s) {
    launch_k(k_sphere_step, blocks_for(n), 128, 0, s, n, x, f, faces, keys, KW, M, bw_branch, eta, status);
}
void launch_trace_finish(int64_t n, const double* x, int32_t* status, double* out, cudaStream_t s) {
    launch_k(k_trace_finish, blocks_for(n), 128, 0, s, n, x, status, out);
}

}  // namespace am
