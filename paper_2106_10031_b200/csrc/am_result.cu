// am_result.cu -- result assembly on the GPU: the visited cells in the reference's order.
//
// The reference returns its polygons sorted by (state key bytes, branch) (marching.py:356-359);
// packbits key bytes compare like the MSB-first key words, and the ensemble branch is the last
// word, so the order is the word-lexicographic order of the KW-word keys.  It is produced by a
// stable merge sort of the cell indices comparing the KW-word keys most significant word first
// (keys resident in L2; most comparisons resolve in the first words), or with AM_RESULT_RADIX=1
// by an LSD radix sort: one stable (word, index) pair sort per word, last word first.  The cells' face
// loops (vertices, per-edge transition refs) are then gathered into that order as CSR, ready for
// one device->host copy per array or for the GPU weld.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "am_internal.h"

namespace am {

namespace {

__global__ void k_iota(int32_t* o, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = (int32_t)i;
}
__global__ void k_key_word(const uint64_t* keys, const int32_t* ord, int64_t n, int KW, int w, uint64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = keys[(int64_t)ord[i] * KW + w];
}
__global__ void k_sorted_cells(const uint64_t* keys, const int32_t* ord, const int32_t* cell_nv, int64_t n, int KW,
                               uint64_t* s_keys, int32_t* s_nv, int64_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = ord[i];
        for (int w = 0; w < KW; w++) s_keys[i * KW + w] = keys[c * KW + w];
        const int32_t nv = cell_nv[c];
        s_nv[i] = nv;
        cnt[i] = nv > 0 ? nv : 0;
    }
}
__global__ void k_sorted_verts(const int32_t* ord, const int64_t* cnt, const int64_t* svoff, const int64_t* cell_voff,
                               const double* verts, const int32_t* enr, int64_t n, double* s_verts, int64_t* s_enr,
                               int64_t* vsrc) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src0 = cell_voff[ord[i]], dst0 = svoff[i];
        for (int64_t v = 0; v < cnt[i]; v++) {
            const int64_t src = src0 + v, dst = dst0 + v;
            s_verts[dst * 3 + 0] = verts[src * 3 + 0];
            s_verts[dst * 3 + 1] = verts[src * 3 + 1];
            s_verts[dst * 3 + 2] = verts[src * 3 + 2];
            s_enr[dst] = enr[src];
            vsrc[dst] = src;
        }
    }
}
__global__ void k_sorted_refs(const int64_t* vsrc, const int64_t* s_enr, const int64_t* sroff, const int64_t* roff,
                              const int32_t* refs, int64_t nv, int32_t* s_enr32, int32_t* s_refs) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nv; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = vsrc[p], m = s_enr[p], d = sroff[p], r0 = roff[src];
        s_enr32[p] = (int32_t)m;
        for (int64_t q = 0; q < m; q++) s_refs[d + q] = refs[r0 + q];
    }
}

// word q of the sort order -> key word: a batch of shapes is ordered by shape first (its shape
// word is the most significant), then like the reference
__host__ __device__ __forceinline__ int order_word(int q, int shape_w) {
    return shape_w < 0 ? q : (q == 0 ? shape_w : q - 1 + (q - 1 >= shape_w ? 1 : 0));
}

struct KeyLess {
    const uint64_t* keys;
    int KW, shape_w;
    __device__ bool operator()(int32_t a, int32_t b) const {
        const uint64_t* ka = keys + (int64_t)a * KW;
        const uint64_t* kb = keys + (int64_t)b * KW;
        for (int q = 0; q < KW; q++) {
            const int w = order_word(q, shape_w);
            const uint64_t x = __ldg(ka + w), y = __ldg(kb + w);
            if (x != y) return x < y;
        }
        return false;
    }
};

inline unsigned blocks(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

template <typename T>
struct Tmp {
    T* p = nullptr;
    cudaStream_t s;
    explicit Tmp(cudaStream_t st) : s(st) {}
    cudaError_t alloc(int64_t n) { return cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(T), s); }
    ~Tmp() { if (p) cudaFreeAsync(p, s); }
};

#define RCK(x)                                                                                      \
    do {                                                                                            \
        cudaError_t err_ = (x);                                                                     \
        if (err_ != cudaSuccess) return set_error(AM_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(err_)); \
    } while (0)

}  // namespace

// keys: the nc visited cells' keys in discovery order (KW words each).  Outputs (device,
// caller-sized): s_keys [nc*KW], s_nv [nc] (raw counts, <= 0 for empty/overflow cells),
// s_verts [nvt*3], s_enr [nvt], s_refs [nref], all in sorted cell order.
int assemble_results(const uint64_t* keys, const int32_t* cell_nv, const int64_t* cell_voff, const double* verts,
                     const int32_t* enr, const int64_t* roff, const int32_t* refs, int64_t nc, int64_t nvt, int KW,
                     int shape_w, cudaStream_t s, uint64_t* s_keys, int32_t* s_nv, double* s_verts, int32_t* s_enr,
                     int32_t* s_refs) {
    if (nc <= 0) return AM_OK;
    if (nc >= ((int64_t)1 << 31)) return set_error(AM_ERR_ARG, "result assembly: more than 2^31 cells");
    Tmp<int32_t> ord_a(s), ord_b(s);
    Tmp<uint64_t> w_a(s), w_b(s);
    Tmp<int64_t> cnt(s), svoff(s), senr(s), sroff(s), vsrc(s);
    RCK(ord_a.alloc(nc)); RCK(ord_b.alloc(nc)); RCK(w_a.alloc(nc)); RCK(w_b.alloc(nc));
    RCK(cnt.alloc(nc + 1)); RCK(svoff.alloc(nc + 1)); RCK(senr.alloc(nvt + 1)); RCK(sroff.alloc(nvt + 1));
    RCK(vsrc.alloc(nvt));
    static const bool radix = [] { const char* v = getenv("AM_RESULT_RADIX"); return v && atoi(v) != 0; }();
    const KeyLess less{keys, KW, shape_w};
    size_t tb = 0, t2 = 0;
    if (radix) cub::DeviceRadixSort::SortPairs(nullptr, tb, w_a.p, w_b.p, ord_a.p, ord_b.p, (int)nc, 0, 64, s);
    else cub::DeviceMergeSort::StableSortKeys(nullptr, tb, ord_a.p, (int)nc, less, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, cnt.p, svoff.p, nc + 1, s);
    tb = std::max(tb, t2);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, senr.p, sroff.p, nvt + 1, s);
    tb = std::max(tb, t2);
    Tmp<unsigned char> tmp(s);
    RCK(tmp.alloc((int64_t)tb));
    const unsigned G = blocks(nc);
    k_iota<<<G, 256, 0, s>>>(ord_a.p, nc);
    if (radix) {
        // LSD: a stable sort by each word, least significant first
        for (int q = KW - 1; q >= 0; q--) {
            k_key_word<<<G, 256, 0, s>>>(keys, ord_a.p, nc, KW, order_word(q, shape_w), w_a.p);
            size_t t = tb;
            RCK(cub::DeviceRadixSort::SortPairs(tmp.p, t, w_a.p, w_b.p, ord_a.p, ord_b.p, (int)nc, 0, 64, s));
            std::swap(ord_a.p, ord_b.p);
        }
    } else {
        size_t t = tb;
        RCK(cub::DeviceMergeSort::StableSortKeys(tmp.p, t, ord_a.p, (int)nc, less, s));
    }
    k_sorted_cells<<<G, 256, 0, s>>>(keys, ord_a.p, cell_nv, nc, KW, s_keys, s_nv, cnt.p);
    RCK(cudaMemsetAsync(cnt.p + nc, 0, 8, s));
    {
        size_t t = tb;
        RCK(cub::DeviceScan::ExclusiveSum(tmp.p, t, cnt.p, svoff.p, nc + 1, s));
    }
    if (nvt > 0) {
        k_sorted_verts<<<G, 256, 0, s>>>(ord_a.p, cnt.p, svoff.p, cell_voff, verts, enr, nc, s_verts, senr.p, vsrc.p);
        RCK(cudaMemsetAsync(senr.p + nvt, 0, 8, s));
        size_t t = tb;
        RCK(cub::DeviceScan::ExclusiveSum(tmp.p, t, senr.p, sroff.p, nvt + 1, s));
        k_sorted_refs<<<blocks(nvt), 256, 0, s>>>(vsrc.p, senr.p, sroff.p, roff, refs, nvt, s_enr, s_refs);
    }
    RCK(cudaGetLastError());
    return AM_OK;
}

}  // namespace am
