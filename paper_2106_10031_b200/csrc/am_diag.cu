// am_diag.cu -- march diagnostics on the GPU.
//
// am_unique_planes: pairs of face planes proportional within an angle tolerance
// (reference network.py:528-570 check_unique_planes, called by marching.py:361-363 when the
// march has <= unique_planes_limit faces).  Rows H_i = (n_i, d_i) are scaled to unit length
// (a zero row keeps scale 1) and a pair (i < j) is reported when the chord distance
// min(|u_i - u_j|, |u_i + u_j|) <= tol.  The arithmetic is the reference's: the 4-term sums
// of squares are accumulated left to right with separately rounded multiply / add (this file
// is compiled with -fmad=false), then sqrt, so the comparisons see the same doubles numpy does.
#include <algorithm>

#include "am_internal.h"

namespace am {
namespace {

__device__ __forceinline__ double sumsq4(double a, double b, double c, double d) {
    double s = a * a;
    s = s + b * b;
    s = s + c * c;
    return s + d * d;
}

__global__ void k_unit_rows(const double* __restrict__ H, int64_t m, double* __restrict__ U) {
    pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double4 h = reinterpret_cast<const double4*>(H)[i];
        double n = sqrt(sumsq4(h.x, h.y, h.z, h.w));
        if (n == 0.0) n = 1.0;
        reinterpret_cast<double4*>(U)[i] = make_double4(h.x / n, h.y / n, h.z / n, h.w / n);
    }
}

// one warp per row i; lanes stride over j > i; row i stays in registers, rows j stream from L2
__global__ void k_plane_pairs(const double* __restrict__ U, int64_t m, double tol, int32_t* __restrict__ pairs,
                              int64_t cap, unsigned long long* __restrict__ count) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        const double4 u = reinterpret_cast<const double4*>(U)[i];
        for (int64_t j = i + 1 + lane; j < m; j += 32) {
            const double4 v = reinterpret_cast<const double4*>(U)[j];
            const double dm = sqrt(sumsq4(u.x - v.x, u.y - v.y, u.z - v.z, u.w - v.w));
            const double dp = sqrt(sumsq4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w));
            if (fmin(dm, dp) <= tol) {
                const unsigned long long k = atomicAdd(count, 1ull);
                if ((int64_t)k < cap) {
                    pairs[2 * k] = (int32_t)i;
                    pairs[2 * k + 1] = (int32_t)j;
                }
            }
        }
    }
}

}  // namespace
}  // namespace am

using namespace am;

extern "C" int am_unique_planes(const double* d_planes, int64_t m, double tol, int32_t* d_pairs, int64_t cap,
                                void* stream, int64_t* h_count) {
    if (m < 0 || !h_count || (m > 0 && !d_planes) || (cap > 0 && !d_pairs) || m > INT32_MAX)
        return set_error(AM_ERR_ARG, "am_unique_planes: bad arguments");
    *h_count = 0;
    if (m < 2) return AM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    double* U = nullptr;
    unsigned long long* cnt = nullptr;
    auto ck = [](cudaError_t e) { return e == cudaSuccess ? AM_OK : set_error(AM_ERR_CUDA, "am_unique_planes: %s",
                                                                              cudaGetErrorString(e)); };
    int rc = ck(cudaMallocAsync(&U, (size_t)m * 32, s));
    if (!rc) rc = ck(cudaMallocAsync(&cnt, sizeof(unsigned long long), s));
    if (!rc) rc = ck(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    if (!rc) {
        const int g1 = (int)std::min<int64_t>((m + 255) / 256, 1184);
        rc = ck(launch_k(k_unit_rows, dim3(g1), dim3(256), 0, s, d_planes, m, U));
    }
    if (!rc) {
        const int g2 = (int)std::min<int64_t>((m + 7) / 8, 148 * 8);
        rc = ck(launch_k(k_plane_pairs, dim3(g2), dim3(256), 0, s, (const double*)U, m, tol, d_pairs, cap, cnt));
    }
    unsigned long long n = 0;
    if (!rc) rc = ck(cudaMemcpyAsync(&n, cnt, sizeof(n), cudaMemcpyDeviceToHost, s));
    if (U) cudaFreeAsync(U, s);
    if (cnt) cudaFreeAsync(cnt, s);
    if (!rc) rc = ck(cudaStreamSynchronize(s));
    *h_count = (int64_t)n;
    return rc;
}
