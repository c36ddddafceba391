// am_weld.cu -- mesh assembly: weld the vertices of a polygon soup on the GPU.
//
// Reference semantics (meshes.py:89-148 weld): vertices are visited in order; vertex i merges
// into the FIRST kept vertex met while scanning the 27 grid cells of side tol around it (dx, dy,
// dz each in the order 0, -1, 1) and, inside a cell, kept vertices in insertion (= index) order,
// at euclidean distance <= tol; otherwise i is kept.  tol == 0: exact-coordinate buckets.
//
// That greedy pass is sequential, but its decisions are a fixed point that can be resolved in
// parallel: for every vertex the ordered list of EARLIER vertices within tol in the reference's
// search order (its candidates) is built once; then in rounds, an undecided vertex walks its
// candidates -- merged ones are skipped, the first kept one is its hit, an undecided one blocks
// it until a later round; with no kept candidate it is kept.  The lowest undecided vertex is
// always decidable, so the rounds terminate; on meshes they take a handful.  Everything else is
// data-parallel: a cell hash table (open addressing on a 64-bit tag, full-key verification,
// rehash on a tag collision), a radix sort of (cell, vertex) that lists each cell's vertices in
// index order, scans for the kept ranks and the compacted face loops.  Pure selection and
// index rewriting: the output is bit-identical to the reference's.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "am_internal.h"

namespace am {

namespace {

struct CellKey {
    long long k[3];
};

__host__ __device__ inline unsigned long long mix64(unsigned long long h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    return h ^ (h >> 33);
}
__device__ inline unsigned long long cell_tag(const CellKey& c, unsigned long long seed) {
    unsigned long long h = seed;
    for (int d = 0; d < 3; d++) h = mix64(h ^ (unsigned long long)c.k[d]) + 0x9e3779b97f4a7c15ull;
    return h | 1ull;  // 0 = empty slot
}
__device__ inline long long exact_bits(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 and 0.0 compare equal in the reference's tuple keys
    return __double_as_longlong(x);
}
__device__ inline CellKey key_of(const double* v, double inv, bool exact) {
    CellKey c;
    for (int d = 0; d < 3; d++)
        c.k[d] = exact ? exact_bits(v[d]) : (long long)floor(__dmul_rn(v[d], inv));
    return c;
}

struct Table {
    unsigned long long* tag;
    CellKey* key;
    int* start;   // the cell's vertices are sorted positions [start, end)
    int* end;
    unsigned long long mask, seed;
};

__device__ inline long long table_find(const Table& T, const CellKey& c) {
    const unsigned long long t = cell_tag(c, T.seed);
    for (unsigned long long s = t & T.mask;; s = (s + 1) & T.mask) {
        unsigned long long x = T.tag[s];
        if (x == 0ull) return -1;
        if (x == t) {
            const CellKey& k = T.key[s];
            if (k.k[0] == c.k[0] && k.k[1] == c.k[1] && k.k[2] == c.k[2]) return (long long)s;
        }
    }
}

__global__ void k_weld_insert(const double* v, int n, double inv, int exact, Table T, int* slot) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const CellKey c = key_of(v + (size_t)i * 3, inv, exact);
        const unsigned long long t = cell_tag(c, T.seed);
        for (unsigned long long s = t & T.mask;; s = (s + 1) & T.mask) {
            unsigned long long prev = atomicCAS(&T.tag[s], 0ull, t);
            if (prev == 0ull) { T.key[s] = c; slot[i] = (int)s; break; }   // the claimer writes the key
            if (prev == t) { slot[i] = (int)s; break; }
        }
    }
}

// every vertex re-derives its key and checks the slot's key: a differing key means two cells
// share a 64-bit tag -> rehash with another seed
__global__ void k_weld_verify(const double* v, int n, double inv, int exact, Table T, const int* slot, int* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const CellKey c = key_of(v + (size_t)i * 3, inv, exact);
        const CellKey& k = T.key[slot[i]];
        if (k.k[0] != c.k[0] || k.k[1] != c.k[1] || k.k[2] != c.k[2]) atomicExch(bad, 1);
    }
}

__global__ void k_weld_sortkeys(const int* slot, int n, unsigned long long* sk) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        sk[i] = ((unsigned long long)(unsigned)slot[i] << 32) | (unsigned)i;
}

__global__ void k_weld_ranges(const unsigned long long* sorted, int n, Table T) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        unsigned s = (unsigned)(sorted[p] >> 32);
        if (p == 0 || (unsigned)(sorted[p - 1] >> 32) != s) T.start[s] = p;
        if (p == n - 1 || (unsigned)(sorted[p + 1] >> 32) != s) T.end[s] = p + 1;
    }
}

// candidates of vertex i in the reference's search order; FILL = false counts them
template <bool FILL>
__global__ void k_weld_cands(const double* v, int n, double tol, double inv, int exact, Table T,
                             const unsigned long long* sorted, long long* ncand, const long long* coff, int* cand) {
    const int ord[3] = {0, -1, 1};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double* p = v + (size_t)i * 3;
        const CellKey c = key_of(p, inv, exact);
        int m = 0;
        long long w = FILL ? coff[i] : 0;
        const int nd = exact ? 1 : 27;
        for (int q = 0; q < nd; q++) {
            CellKey c2 = c;
            if (!exact) {
                c2.k[0] += ord[q / 9];
                c2.k[1] += ord[(q / 3) % 3];
                c2.k[2] += ord[q % 3];
            }
            const long long s = table_find(T, c2);
            if (s < 0) continue;
            const int b = T.start[s], e = T.end[s];
            for (int r = b; r < e; r++) {
                const int j = (int)(unsigned)(sorted[r] & 0xffffffffull);
                if (j >= i) break;   // ascending: only earlier vertices exist at i's turn
                const double* o = v + (size_t)j * 3;
                bool near;
                if (exact) {
                    near = o[0] == p[0] && o[1] == p[1] && o[2] == p[2];
                } else {
                    const double d0 = __dsub_rn(o[0], p[0]), d1 = __dsub_rn(o[1], p[1]), d2 = __dsub_rn(o[2], p[2]);
                    near = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2))) <= tol;
                }
                if (!near) continue;
                if (FILL) cand[w++] = j;
                m++;
            }
        }
        if (!FILL) ncand[i] = m;
    }
}

// status: 0 undecided, 1 kept, 2 merged (hit set)
__global__ void k_weld_round(int n, const long long* coff, const int* cand, int* status, int* hit, int* left) {
    int mine = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (status[i] != 0) continue;
        int decided = 1, h = -1;
        for (long long q = coff[i]; q < coff[i + 1]; q++) {
            const int j = cand[q];
            const int sj = *reinterpret_cast<volatile int*>(&status[j]);
            if (sj == 2) continue;
            if (sj == 1) { h = j; break; }
            decided = 0;
            break;
        }
        if (!decided) { mine++; continue; }
        if (h >= 0) { hit[i] = h; __threadfence(); status[i] = 2; }
        else status[i] = 1;
    }
    if (mine) atomicAdd(left, mine);
}

__global__ void k_weld_keptflag(const int* status, int n, int* flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) flag[i] = status[i] == 1;
}

__global__ void k_weld_remap(const double* v, int n, const int* status, const int* hit, const int* rank,
                             long long* remap, double* kept) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (status[i] == 1) {
            const int r = rank[i];
            remap[i] = r;
            kept[(size_t)r * 3 + 0] = v[(size_t)i * 3 + 0];
            kept[(size_t)r * 3 + 1] = v[(size_t)i * 3 + 1];
            kept[(size_t)r * 3 + 2] = v[(size_t)i * 3 + 2];
        } else {
            remap[i] = rank[hit[i]];
        }
    }
}

// one thread per loop: the remapped loop without consecutive and closing repeats
// (reference meshes.py:137-148); a loop with < 3 distinct indices is dropped (length 0).  The
// distinct count of the deduplicated loop equals that of the remapped loop (a removed entry
// equals a neighbour that stays), so it is counted on the latter.
template <bool FILL>
__global__ void k_weld_loops(const long long* loop_off, const long long* loop_idx, int n_loops, const long long* remap,
                             long long* out_n, const long long* out_off, long long* face_idx, const int* src_rank,
                             long long* face_src) {
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n_loops; l += gridDim.x * blockDim.x) {
        const long long a = loop_off[l], b = loop_off[l + 1];
        const long long keep = FILL ? out_n[l] : 0;   // FILL: the counted length (closing repeat excluded)
        if (FILL && keep == 0) continue;
        int m = 0;
        long long first = -1, last = -1;
        long long w = FILL ? out_off[l] : 0;
        for (long long q = a; q < b; q++) {
            const long long x = remap[loop_idx[q]];
            if (m > 0 && x == last) continue;
            if (m == 0) first = x;
            last = x;
            if (FILL && m < keep) face_idx[w++] = x;
            m++;
        }
        if (m > 1 && first == last) m--;
        if (FILL) {
            face_src[src_rank[l]] = l;
            continue;
        }
        int distinct = 0;
        for (long long q = a; q < b && distinct < 3; q++) {
            const long long x = remap[loop_idx[q]];
            bool seen = false;
            for (long long r = a; r < q && !seen; r++) seen = remap[loop_idx[r]] == x;
            distinct += !seen;
        }
        out_n[l] = distinct >= 3 ? m : 0;
    }
}

// compacted face offsets: face r starts where its source loop's output starts
__global__ void k_weld_faceoff(const long long* face_src, int n_faces, const long long* ooff, int n_loops,
                               long long* face_off) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_faces; r += gridDim.x * blockDim.x)
        face_off[r] = r < n_faces ? ooff[face_src[r]] : ooff[n_loops];
}

__global__ void k_flag_nonzero(const long long* a, int n, int* f) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) f[i] = a[i] > 0;
}

template <typename T>
struct Tmp {
    T* p = nullptr;
    cudaStream_t s;
    explicit Tmp(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t n) { return cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s); }
    ~Tmp() { if (p) cudaFreeAsync(p, s); }
};

inline unsigned grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)std::max<long long>(1, std::min<long long>(b, 148LL * 16));
}

}  // namespace

}  // namespace am

using namespace am;

#define WCK(x)                                                                            \
    do {                                                                                  \
        cudaError_t err_ = (x);                                                           \
        if (err_ != cudaSuccess) return set_error(AM_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(err_)); \
    } while (0)

// reference meshes.py:89-148 weld(mesh, tol) -- see include/am_b200.h
extern "C" int am_weld(const double* d_verts, int64_t n_verts, const int64_t* d_loop_off, const int64_t* d_loop_idx,
                       int64_t n_loops, double tol, void* stream, int64_t* d_remap, double* d_kept,
                       int64_t* d_face_off, int64_t* d_face_idx, int64_t* d_face_src, int64_t* h_counts) {
    if (n_verts < 0 || n_loops < 0 || !(tol >= 0) || !h_counts) return set_error(AM_ERR_ARG, "bad weld arguments");
    if (n_verts >= (int64_t)1 << 31 || n_loops >= (int64_t)1 << 31)
        return set_error(AM_ERR_ARG, "weld: more than 2^31 vertices or loops");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int n = (int)n_verts, nl = (int)n_loops;
    const int exact = tol == 0.0;
    const double inv = exact ? 0.0 : 1.0 / tol;
    h_counts[0] = h_counts[1] = h_counts[2] = 0;
    if (n == 0 && nl == 0) {
        WCK(cudaMemsetAsync(d_face_off, 0, 8, s));
        return AM_OK;
    }
    // ---- cell table (rehash with a new seed on a 64-bit tag collision)
    unsigned long long cap = 16;
    while (cap < 2ull * (unsigned long long)n + 2) cap <<= 1;
    Tmp<unsigned long long> tag(s), sk(s), sk2(s);
    Tmp<CellKey> keys(s);
    Tmp<int> start(s), endp(s), slot(s), flag(s), status(s), hit(s), rank(s), oflag(s), orank(s), dev(s);
    Tmp<long long> ncand(s), coff(s), outn(s), ooff(s);
    Tmp<int> cand(s);
    WCK(tag.alloc(cap)); WCK(keys.alloc(cap)); WCK(start.alloc(cap)); WCK(endp.alloc(cap));
    WCK(slot.alloc(n)); WCK(sk.alloc(n)); WCK(sk2.alloc(n)); WCK(flag.alloc(n)); WCK(ncand.alloc(n + 1));
    WCK(status.alloc(n)); WCK(hit.alloc(n)); WCK(rank.alloc(n)); WCK(coff.alloc(n + 1)); WCK(dev.alloc(2));
    WCK(outn.alloc(nl + 1)); WCK(oflag.alloc(nl + 1)); WCK(orank.alloc(nl + 1)); WCK(ooff.alloc(nl + 1));
    Table T{tag.p, keys.p, start.p, endp.p, cap - 1, 0x243f6a8885a308d3ull};
    const unsigned G = grid_for(n);
    for (int attempt = 0;; attempt++) {
        WCK(cudaMemsetAsync(tag.p, 0, cap * 8, s));
        WCK(cudaMemsetAsync(dev.p, 0, 8, s));
        if (n) {
            k_weld_insert<<<G, 256, 0, s>>>(d_verts, n, inv, exact, T, slot.p);
            k_weld_verify<<<G, 256, 0, s>>>(d_verts, n, inv, exact, T, slot.p, dev.p);
        }
        int bad = 0;
        WCK(cudaMemcpyAsync(&bad, dev.p, 4, cudaMemcpyDeviceToHost, s));
        WCK(cudaStreamSynchronize(s));
        if (!bad) break;
        if (attempt == 8) return set_error(AM_ERR_CUDA, "weld: cell table tag collisions persist");
        T.seed = mix64(T.seed + 0x9e3779b97f4a7c15ull);
    }
    // ---- cell member lists in vertex order: radix sort of (slot << 32 | vertex)
    int end_bit = 32;
    while ((1ull << (end_bit - 32)) < cap) end_bit++;
    size_t tmp_bytes = 0, t2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, sk.p, sk2.p, n, 0, end_bit, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, ncand.p, coff.p, n + 1, s);
    tmp_bytes = std::max(tmp_bytes, t2);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, outn.p, ooff.p, nl + 1, s);
    tmp_bytes = std::max(tmp_bytes, t2);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, flag.p, rank.p, n, s);
    tmp_bytes = std::max(tmp_bytes, t2);
    Tmp<unsigned char> cubtmp(s);
    WCK(cubtmp.alloc(tmp_bytes));
    if (n) {
        k_weld_sortkeys<<<G, 256, 0, s>>>(slot.p, n, sk.p);
        WCK(cub::DeviceRadixSort::SortKeys(cubtmp.p, tmp_bytes, sk.p, sk2.p, n, 0, end_bit, s));
        k_weld_ranges<<<G, 256, 0, s>>>(sk2.p, n, T);
        // ---- candidates (count, scan, fill)
        k_weld_cands<false><<<G, 256, 0, s>>>(d_verts, n, tol, inv, exact, T, sk2.p, ncand.p, nullptr, nullptr);
        WCK(cudaMemsetAsync(ncand.p + n, 0, 8, s));
    }
    {
        // int counts -> int64 offsets
        size_t tb = tmp_bytes;
        WCK(cub::DeviceScan::ExclusiveSum(cubtmp.p, tb, ncand.p, coff.p, n + 1, s));
    }
    long long ncand_total = 0;
    WCK(cudaMemcpyAsync(&ncand_total, coff.p + n, 8, cudaMemcpyDeviceToHost, s));
    WCK(cudaStreamSynchronize(s));
    WCK(cand.alloc((size_t)ncand_total));
    if (n) k_weld_cands<true><<<G, 256, 0, s>>>(d_verts, n, tol, inv, exact, T, sk2.p, nullptr, coff.p, cand.p);
    // ---- greedy decisions in rounds
    WCK(cudaMemsetAsync(status.p, 0, (size_t)n * 4, s));
    for (int round = 0; n; round++) {
        WCK(cudaMemsetAsync(dev.p, 0, 4, s));
        k_weld_round<<<G, 256, 0, s>>>(n, coff.p, cand.p, status.p, hit.p, dev.p);
        int left = 0;
        WCK(cudaMemcpyAsync(&left, dev.p, 4, cudaMemcpyDeviceToHost, s));
        WCK(cudaStreamSynchronize(s));
        if (!left) break;
        if (round > n) return set_error(AM_ERR_CUDA, "weld: rounds did not converge");
    }
    // ---- kept ranks, remap, kept vertices
    if (n) {
        k_weld_keptflag<<<G, 256, 0, s>>>(status.p, n, flag.p);
        size_t tb = tmp_bytes;
        WCK(cub::DeviceScan::ExclusiveSum(cubtmp.p, tb, flag.p, rank.p, n, s));
        k_weld_remap<<<G, 256, 0, s>>>(d_verts, n, status.p, hit.p, rank.p, reinterpret_cast<long long*>(d_remap),
                                       d_kept);
    }
    int last_rank = 0, last_flag = 0;
    if (n) {
        WCK(cudaMemcpyAsync(&last_rank, rank.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
        WCK(cudaMemcpyAsync(&last_flag, flag.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
    }
    // ---- loops: kept length per loop, scans, fill
    const unsigned GL = grid_for(nl);
    const long long* lo = reinterpret_cast<const long long*>(d_loop_off);
    const long long* li = reinterpret_cast<const long long*>(d_loop_idx);
    const long long* rm = reinterpret_cast<const long long*>(d_remap);
    WCK(cudaMemsetAsync(outn.p + nl, 0, 8, s));
    if (nl) k_weld_loops<false><<<GL, 256, 0, s>>>(lo, li, nl, rm, outn.p, nullptr, nullptr, nullptr, nullptr);
    {
        size_t tb = tmp_bytes;
        WCK(cub::DeviceScan::ExclusiveSum(cubtmp.p, tb, outn.p, ooff.p, nl + 1, s));
    }
    if (nl) {
        k_flag_nonzero<<<GL, 256, 0, s>>>(outn.p, nl + 1, oflag.p);
        size_t tb = tmp_bytes;
        WCK(cub::DeviceScan::ExclusiveSum(cubtmp.p, tb, oflag.p, orank.p, nl + 1, s));
        k_weld_loops<true><<<GL, 256, 0, s>>>(lo, li, nl, rm, outn.p, ooff.p,
                                              reinterpret_cast<long long*>(d_face_idx), orank.p,
                                              reinterpret_cast<long long*>(d_face_src));
    }
    int n_faces = 0;
    WCK(cudaMemcpyAsync(&n_faces, orank.p + nl, 4, cudaMemcpyDeviceToHost, s));
    WCK(cudaStreamSynchronize(s));
    if (nl == 0) n_faces = 0;
    k_weld_faceoff<<<grid_for(n_faces + 1), 256, 0, s>>>(reinterpret_cast<const long long*>(d_face_src), n_faces,
                                                        ooff.p, nl, reinterpret_cast<long long*>(d_face_off));
    WCK(cudaGetLastError());
    WCK(cudaStreamSynchronize(s));
    h_counts[0] = n ? (int64_t)last_rank + last_flag : 0;
    h_counts[1] = n_faces;
    h_counts[2] = (int64_t)nl - n_faces;
    return AM_OK;
}
