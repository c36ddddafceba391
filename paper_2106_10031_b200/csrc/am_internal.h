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

#include "../../include/am_b200.h"

namespace am {

constexpr double kDegen = 1e-12;   // reference network.py:27 DEGENERATE_NORMAL_TOL
constexpr double kTolDet = 1e-12;  // reference cells.py:32 TOL_DET
constexpr uint64_t kEmpty = ~0ull;

// number of kernels this library launched (bench.py gpu_launches)
extern unsigned long long g_launch_count;

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
};

struct LayerLaunch {
    StepDev st;
    double* Z;            // [items][zs][C]
    uint64_t* keys;       // [items][KW]
    int* changed;         // compose: per-item canonical-changed flag (may be null)
    const double* pts;    // forward: [items][3]
    int64_t n_items;
    int KW, zs;           // key words, Z row count per item (>= NB)
};

// kernels' host-side launchers (am_compose.cu)
void launch_input_step(const LayerLaunch& L, int C, cudaStream_t s);
void launch_gemm_step(const LayerLaunch& L, int C, const CUtensorMap* tmW, const CUtensorMap* tmV,
                      cudaStream_t s);
void launch_face_head(const double* Z, const uint64_t* keys, double* faces, int64_t n_items, int zs,
                      int KW, const int* sub_last_row, const int* sub_last_n, const double* const* head_w,
                      const double* head_b, int n_subs, cudaStream_t s);
void launch_forward_head(const double* Z, uint64_t* keys, double* vals, int64_t n_items, int zs, int KW,
                         const int* sub_last_row, const int* sub_last_n, const double* const* head_w,
                         const double* head_b, int n_subs, int ensemble, cudaStream_t s);
int make_tmap_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld_elems);

// hash set (am_hash.cu)
struct HashSet {
    uint64_t* table;      // slots
    uint64_t mask;        // capacity - 1
    uint64_t* pool;       // [cap_pool][KW]
    uint32_t* pool_flags; // bit0 visited-canonical
    unsigned long long* n_pool;  // device counter
    int64_t cap_pool;
    int KW;
};
// insert src[idx[i]] (or src[i] if idx null) for i < n; status[i] = 1 new / 0 present,
// slot[i] = slot index for new entries (candidate-ref written, fixed up later)
void launch_hash_insert(const HashSet& H, const uint64_t* src, const int32_t* idx, int64_t n,
                        int32_t* status, uint64_t* slot, cudaStream_t s);
// assign pool indices to new entries, copy keys into the pool, rewrite slots
void launch_hash_fixup(const HashSet& H, const uint64_t* src, const int32_t* idx, int64_t n,
                       const int32_t* status, const uint64_t* slot, uint32_t flag, int32_t* pool_idx,
                       cudaStream_t s);
void launch_hash_lookup(const HashSet& H, const uint64_t* src, int64_t n, int32_t* found, cudaStream_t s);

// face extraction (am_face.cu)
struct FaceArgs {
    const double* Z;          // [batch][zs][4]
    const double* faces;      // [batch][M][4]
    const uint64_t* keys;     // canonical keys [batch][KW]
    const int32_t* items;     // frontier: batch slots to process
    const int32_t* pool_idx;  // per frontier entry: pool index of the state
    int64_t n;                // frontier size
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
    uint64_t* cand;           // next-wave candidate keys [cap_cand][KW]
    unsigned long long* n_cand;
    int64_t cap_cand;
    double* probe_pts;        // [cap_probe][3]
    unsigned long long* n_probe;
    int64_t cap_probe;
    unsigned long long* overflow;  // counters: [0] C-set/polygon overflow, [1] capacity overflow
};
void launch_face(const FaceArgs& a, cudaStream_t s);

}  // namespace am
