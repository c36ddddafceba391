// am_compose.cu -- per-cell affine-map composition and batched forward passes.
//
// One kernel launch per hidden layer l computes, for a batch of items,
//     Z_l[item] = W_l · (s_{l-1}[item] ⊙ Z_{l-1}[item]) + shortcut + bias
// where an item is
//   * a cell state (C = 4 columns: the 3 normal components and the offset of
//     every neuron functional, reference network.py:398-443 _region_maps_sub), or
//   * a point (C = 1 column: the pre-activation, reference network.py:320-349).
// Across a batch this is the dense contraction W_l [n_l x n_{l-1}] x [n_{l-1} x C·B],
// run on the fp64 tensor cores (mma.sync m16n8k4 .f64 -> SASS DMMA) with the
// W_l tile staged by TMA (cp.async.bulk.tensor, 128B swizzle) and the masked
// activation tile staged through registers (the mask s_{l-1} is applied while
// staging).  The epilogue adds bias / shortcut, derives the canonical state bit
// of every neuron (constant functionals forced to the sign of their offset,
// reference network.py:421-428) and writes Z_l, which is also the plane buffer
// the face kernel reads.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "am_internal.h"
#include "am_ptx.cuh"

namespace am {

constexpr int BM = 64, BN = 64, TB = 16, BK = 32;   // TB: K width of one TMA box (128 B)
constexpr int kThreads = 256;   // 8 warps: 2 (rows) x 4 (columns), 32 x 16 outputs each

// ----------------------------------------------------------- tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int make_tmap_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld_elems, int box_rows) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return -1;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)(ld_elems * sizeof(double))};
    cuuint32_t box[2] = {TB, (cuuint32_t)box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box,
                          estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

// -------------------------------------------------------- bit utilities
// state bit read through L2: the fused composition kernel updates canonical bits with atomics
// (performed at L2) and reads them back in later layers of the same launch
__device__ __forceinline__ int key_bit_cg(const uint64_t* k, int i) {
    return (int)((__ldcg(k + (i >> 6)) >> (63 - (i & 63))) & 1ull);
}
__device__ __forceinline__ void set_key_bit(uint64_t* key, int row, int bit) {
    uint64_t m = key_mask(row);
    if (bit) atomicOr(reinterpret_cast<unsigned long long*>(key + (row >> 6)), (unsigned long long)m);
    else atomicAnd(reinterpret_cast<unsigned long long*>(key + (row >> 6)), (unsigned long long)~m);
}

// ------------------------------------------------------ input step (l = 1)
// reference network.py:398-443 with A = I, c = 0: pre_A = W[:, :3] (+ shortcut
// from the input), pre_c = (sc + 0) + b.
// reference network.py:398-443 with A = I, c = 0 for one (item, neuron)
template <int C>
__device__ __forceinline__ void input_elem(const LayerLaunch& L, uint64_t* keys, int64_t item, int r) {
    const StepDev& st = L.st;
    const double* w = st.W + (int64_t)r * st.ldw;
    uint64_t* key = keys + item * L.KW;
    int row = st.row_off + r;
    double* z = zbase(L) + (item * L.zs + row) * C;
    bool sc = st.flags & (AM_STEP_SHORTCUT_IDENT | AM_STEP_SHORTCUT_LINEAR);
    const bool has_vb = st.vb || st.vb_shape;
    const int shp = item_shape(key, L.shape_w);
    if (C == 4) {
        double a0 = w[0], a1 = w[1], a2 = w[2], c = 0.0;
        if (sc) {
            double s0, s1, s2, sc_c = 0.0;
            if (st.flags & AM_STEP_SHORTCUT_IDENT) {
                s0 = r == 0; s1 = r == 1; s2 = r == 2;
            } else {
                const double* v = st.V + (int64_t)r * st.ldv;
                s0 = v[0]; s1 = v[1]; s2 = v[2];
                if (has_vb) sc_c = step_vbias(st, shp, r);
            }
            a0 = s0 + a0; a1 = s1 + a1; a2 = s2 + a2;
            c = (sc_c + c) + step_bias(st, shp, r);
        } else {
            c = c + step_bias(st, shp, r);
        }
        a0 = prec_round(a0, L.fp32); a1 = prec_round(a1, L.fp32);
        a2 = prec_round(a2, L.fp32); c = prec_round(c, L.fp32);
        double nrm = sqrt((a0 * a0 + a1 * a1) + a2 * a2);
        if (!(nrm > kDegen)) {
            int bit = c > 0.0;
            if (bit != key_bit(key, row)) {
                set_key_bit(key, row, bit);
                if (L.changed) L.changed[item] = 1;
            }
        }
        reinterpret_cast<double2*>(z)[0] = make_double2(a0, a1);
        reinterpret_cast<double2*>(z)[1] = make_double2(a2, c);
    } else {
        const double* x = L.pts + item * 3;
        double acc = (x[0] * w[0] + x[1] * w[1]) + x[2] * w[2];
        double pre;
        if (sc) {
            double s;
            if (st.flags & AM_STEP_SHORTCUT_IDENT) {
                s = x[r];
            } else {
                const double* v = st.V + (int64_t)r * st.ldv;
                s = (x[0] * v[0] + x[1] * v[1]) + x[2] * v[2];
                if (has_vb) s = s + step_vbias(st, shp, r);
            }
            pre = (s + acc) + step_bias(st, shp, r);
        } else {
            pre = acc + step_bias(st, shp, r);
        }
        pre = prec_round(pre, L.fp32);
        if (pre > 0.0) atomicOr(reinterpret_cast<unsigned long long*>(key + (row >> 6)), (unsigned long long)key_mask(row));
        z[0] = pre;
    }
}

template <int C>
__global__ void k_input_step(LayerLaunch L) {
    pdl_enter();
    const int64_t n = dev_count(L.n_dev, L.n_cap);
    uint64_t* keys = keys_at(L);
    const int64_t total = n * L.st.n_out;
    for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        int64_t item = gid / L.st.n_out;
        input_elem<C>(L, keys, item, (int)(gid - item * L.st.n_out));
    }
}

static int num_sms() { return device_sms(); }

void launch_input_step(const LayerLaunch& L, int C, cudaStream_t s) {
    int64_t total = L.n_cap * L.st.n_out;
    if (total <= 0) return;
    int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * (L.grid_cap > 0 ? L.grid_cap : 8));
    if (C == 4) { launch_k(k_input_step<4>, (unsigned)blocks, 256, 0, s, L); }
    else { launch_k(k_input_step<1>, (unsigned)blocks, 256, 0, s, L); }
}

// ------------------------------------------- batch gather fused with the input step
// One warp per batch item: the item's pool index is read from the queue slice k_take dequeued
// (queue[QHEAD - nR + b]), its key words and hint are gathered (k_gather_batch's work), and the
// warp's lanes then compute the item's layer-1 rows exactly as k_input_step does (input_elem),
// so a BFS iteration launches one kernel less.  __syncwarp orders the gathered key and the reset
// flags before the lanes' canonical-bit updates of the same item.
// batch item b -> (bucket f, position) of the prefix-reuse bucketing (k_take): items are laid out
// bucket after bucket, ascending f
__device__ __forceinline__ int bucket_of(const unsigned long long* ctr, int nb, int64_t b, int64_t& pos) {
    int f = 0;
    int64_t off = 0;
    for (; f < nb - 1; f++) {
        const int64_t c = (int64_t)ctr[C_BK0 + f];
        if (b < off + c) break;
        off += c;
    }
    pos = b - off;
    return f;
}

__global__ void k_gather_input(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                               const unsigned long long* ctr, int32_t* batch_pool, double* ckey_hint,
                               int32_t* canon_pos, LayerLaunch L, const int32_t* blist, int nb) {
    pdl_enter();
    const int64_t n = dev_count(ctr + C_NR, L.n_cap);
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t* keys = L.keys;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < n; b += nw) {
        int64_t q = b;
        if (blist) {   // prefix reuse: bucket order (cells sharing fewer steps first)
            int64_t pos;
            const int f = bucket_of(ctr, nb, b, pos);
            q = blist[(int64_t)f * L.n_cap + pos];
        }
        const int32_t p = queue[batch_queue_index(ctr, q)];
        for (int w = lane; w < L.KW; w += 32) keys[b * L.KW + w] = pool[(int64_t)p * L.KW + w];
        if (lane == 0) {
            batch_pool[b] = p;
            L.changed[b] = 0;
            canon_pos[b] = -1;
            reinterpret_cast<double4*>(ckey_hint)[b] = reinterpret_cast<const double4*>(pool_hint)[p];
        }
        __syncwarp();
        for (int r = lane; r < L.st.n_out; r += 32) input_elem<4>(L, keys, b, r);
        __syncwarp();
    }
}

void launch_gather_input(const uint64_t* pool, const double* pool_hint, const int32_t* queue,
                         const unsigned long long* ctr, int32_t* batch_pool, double* ckey_hint, int32_t* canon_pos,
                         const LayerLaunch& L, cudaStream_t s, const int32_t* blist, int nb) {
    if (L.n_cap <= 0) return;
    const int64_t blocks = std::min<int64_t>((L.n_cap + 7) / 8, (int64_t)num_sms() * 16);
    launch_k(k_gather_input, (unsigned)blocks, 256, 0, s, pool, pool_hint, queue, ctr, batch_pool, ckey_hint,
             canon_pos, L, blist, nb);
}

// Prefix reuse on the per-step path: the items of buckets f >= 1 take the Z rows of steps 1..f
// from their parents (the previous iteration's half of Z) instead of composing them, with the
// canonical test of step f's rows (its flipped neuron: the parent's bits hold for every earlier
// step); the GEMM of step s then runs over the items of buckets f < s only (C_PRE0 + s).  Warp
// per item.
__global__ void k_prefix_rows(PrefixRows R, LayerLaunch L, const int32_t* batch_pool, const int64_t* pool_par) {
    pdl_enter();
    const int64_t n = dev_count(R.ctr + C_NR, L.n_cap);
    const int64_t n0 = (int64_t)R.ctr[C_BK0];
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const unsigned long long par = *L.zpar & 1ull;
    double* Zc = L.Z + (int64_t)par * L.zstride;
    const double* Zp = L.Z + (int64_t)(par ^ 1ull) * L.zstride;
    for (int64_t b = n0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); b < n; b += nw) {
        int64_t pos;
        const int f = bucket_of(R.ctr, R.nb, b, pos);
        const int64_t pi = (int64_t)(((unsigned long long)pool_par[batch_pool[b]] >> 5) & 0x7ffffffull);
        const int r0 = R.row_off[1], rf = R.row_off[f], r1 = rf + R.n_out[f];
        uint64_t* key = L.keys + b * L.KW;
        for (int row = r0 + lane; row < r1; row += 32) {
            const double2* src = reinterpret_cast<const double2*>(Zp + (pi * L.zs + row) * 4);
            const double2 v0 = src[0], v1 = src[1];
            double2* dst = reinterpret_cast<double2*>(Zc + (b * L.zs + row) * 4);
            dst[0] = v0;
            dst[1] = v1;
            if (row >= rf) {
                const double nrm = sqrt((v0.x * v0.x + v0.y * v0.y) + v1.x * v1.x);
                if (!(nrm > kDegen)) {
                    const int bit = v1.y > 0.0;
                    if (bit != key_bit(key, row)) {
                        set_key_bit(key, row, bit);
                        if (L.changed) L.changed[b] = 1;
                    }
                }
            }
        }
    }
}

void launch_prefix_rows(const PrefixRows& R, const LayerLaunch& L, const int32_t* batch_pool, const int64_t* pool_par,
                        cudaStream_t s) {
    if (L.n_cap <= 0) return;
    const int64_t blocks = std::min<int64_t>((L.n_cap + 7) / 8, (int64_t)num_sms() * 16);
    launch_k(k_prefix_rows, (unsigned)blocks, 256, 0, s, R, L, batch_pool, pool_par);
}

// ----------------------------------------------------------- GEMM step

#ifndef AM_NST
#define AM_NST 3
#endif
constexpr int NST = AM_NST;   // pipeline stages (BK = 32 rows of K each)
constexpr int XS4 = BK * 4;   // compose stage: per-item stride (32 rows x 4 components, contiguous as in Z)
constexpr int XS1 = BK + 4;   // forward stage: per-point padded stride (bank-conflict free B fragments)

constexpr int KCW = 10;    // cached state words per item and K segment (K rows <= 576)

// Tile shapes.  TM = 64: 8 warps (2 rows x 4 columns of 32 x 16 warp tiles), 64 x 64 outputs.
// TM = 96 (compose steps with 64 < n_out <= 96, e.g. the 90-wide layers of configs[1]): 6 warps
// (3 x 2), 96 x 32 outputs -- one row tile covers the layer, so the padding rows of a second
// 64-row tile (26 of 64 useful) are not computed and the activation tile is staged once, not twice.
#ifndef AM_NST96
#define AM_NST96 2
#endif
#ifndef AM_CPS96
#define AM_CPS96 2
#endif
// AM_WRES96 (off: measured neutral, 25.8-26.0 vs 25.8-25.9 ms): the 96-row tile keeps the whole layer's W (<= 3 K chunks) resident in shared memory,
// loaded by TMA once per CTA (before the grid dependency wait), instead of re-streaming it per tile
#ifndef AM_WRES96
#define AM_WRES96 0
#endif
// NJ: 8-column fragments per warp (2: 32 x 16 warp tiles; 4: 32 x 32 warp tiles, half the warps
// per CTA for the same 64 x 64 output tile -- twice the DMMAs per A-fragment load, AM_GEMM_NJ4)
#ifndef AM_NJ4_NST
#define AM_NJ4_NST 2
#endif
#ifndef AM_NJ4_CPS
#define AM_NJ4_CPS 3
#endif
template <int C, int TM, int NJ = 2>
struct GT {
    static constexpr int NS = TM == 96 ? AM_NST96 : (NJ == 4 ? AM_NJ4_NST : NST);   // pipeline stages
    static constexpr int CPS = TM == 96 ? AM_CPS96 : (NJ == 4 ? AM_NJ4_CPS : 2);    // resident CTAs per SM
    static constexpr bool WRES = TM == 96 && AM_WRES96;    // W resident for layers of <= WS chunks
    static constexpr int WS = WRES ? (NS > 3 ? NS : 3) : NS;   // W slots
    static constexpr int WM = TM / 32;                // warps along rows
    static constexpr int WN = TM == 64 ? 8 / NJ : 2;  // warps along columns
    static constexpr int NT = 32 * WM * WN;           // threads
    static constexpr int TN = 8 * NJ * WN;            // columns per tile
    static constexpr int NI = C == 4 ? TN / 4 : TN;   // items per tile
};

template <int C, int TM = BM, int NJ = 2>
struct __align__(1024) GemmSmem {
    static constexpr int NI = GT<C, TM, NJ>::NI;   // items per tile
    static constexpr int TN = GT<C, TM, NJ>::TN;
    static constexpr int XSZ = C == 4 ? NI * XS4 : TN * XS1;
    static constexpr int NS = GT<C, TM, NJ>::NS;
    double w[GT<C, TM, NJ>::WS][BK / TB][TM * TB];   // TMA destination: 2 boxes of TM rows x 16 k, 128B-swizzled
    double x[NS][XSZ];            // raw activation tile
    uint32_t mask[NS][TN];        // per item / point: the 32 state bits of the stage's K rows
    uint64_t kc[2][NI][KCW];       // the tile's state words covering each K segment
    uint64_t bar[NS];
    uint64_t wbar;                  // resident W loaded
    unsigned long long bits[TN][2];  // forward epilogue: per-column bit window
};

// 32 state bits of rows [row, row + 32) (MSB-first key words), bit j = row + j; zero beyond `valid`
// (G: key in global memory, read through L2; else the tile's shared-memory word cache)
template <bool G = false>
__device__ __forceinline__ uint32_t bits32(const uint64_t* key, int row, int valid) {
    if (valid <= 0) return 0u;
    int w = row >> 6, off = row & 63;
    uint64_t hi = (G ? __ldcg(key + w) : key[w]) << off;   // bit 63 of hi = state bit of `row`
    if (off > 32 && valid > 64 - off) hi |= (G ? __ldcg(key + w + 1) : key[w + 1]) >> (64 - off);
    uint32_t m = __brev((uint32_t)(hi >> 32));
    if (valid < 32) m &= (1u << valid) - 1u;
    return m;
}

// One TM-row x TN-column output tile of layer L.st (all K chunks + epilogue).
template <int C, int TM = BM, int NJ = 2>
__device__ __forceinline__ void gemm_tile(GemmSmem<C, TM, NJ>& S, const LayerLaunch& L, uint64_t* keys, int64_t n,
                                          const CUtensorMap* tmWp, const CUtensorMap* tmVp, int m0, int64_t n0,
                                          uint32_t& gchunk, bool wres = false) {
    const StepDev& st = L.st;
    double* const Zb = zbase(L);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    using T = GT<C, TM, NJ>;
    static_assert(C == 4 || TM == 64, "the forward stage uses 64-row tiles");
    static_assert(C == 4 || NJ == 2, "the forward stage uses 32 x 16 warp tiles");
    constexpr int WC = 8 * NJ;   // warp tile columns
    const int wm = warp % T::WM, wn = warp / T::WM;   // warp tile: rows wm*32 .. +31, columns wn*WC .. +WC-1
    const bool lin = (st.flags & AM_STEP_SHORTCUT_LINEAR) && !(st.flags & AM_STEP_SC_FROM_INPUT);
    const int kc0 = (st.n_in + BK - 1) / BK;
    const int kc1 = lin ? (st.n_sin + BK - 1) / BK : 0;
    const int nchunks = kc0 + kc1;
    const bool sc_ident = st.flags & AM_STEP_SHORTCUT_IDENT;
    const bool sc_input_lin = (st.flags & AM_STEP_SHORTCUT_LINEAR) && (st.flags & AM_STEP_SC_FROM_INPUT);
    const bool sc_input_id = sc_ident && (st.flags & AM_STEP_SC_FROM_INPUT);
    const bool has_sc = (st.flags & (AM_STEP_SHORTCUT_IDENT | AM_STEP_SHORTCUT_LINEAR)) != 0;
    const bool has_vb = st.vb || st.vb_shape;
    {
        if (C == 1 && tid < BN) { S.bits[tid][0] = 0; S.bits[tid][1] = 0; }
        // state words of the tile's items covering both K segments (no global reads in issue())
        constexpr int NI = GemmSmem<C, TM, NJ>::NI;
        const int64_t item0 = C == 4 ? n0 / 4 : n0;
        int wbeg[2], wcnt[2];
        wbeg[0] = st.in_row_off >> 6;
        wcnt[0] = ((st.in_row_off + st.n_in - 1) >> 6) - wbeg[0] + 1;
        wbeg[1] = lin ? st.sin_row_off >> 6 : 0;
        wcnt[1] = lin ? ((st.sin_row_off + st.n_sin - 1) >> 6) - wbeg[1] + 1 : 0;
        const bool cache_ok = wcnt[0] <= KCW && wcnt[1] <= KCW;
        if (cache_ok) {
            for (int q = tid; q < 2 * NI * KCW; q += T::NT) {
                const int sg = q / (NI * KCW), rem = q % (NI * KCW), il = rem / KCW, w = rem % KCW;
                const int64_t item = item0 + il;
                uint64_t v = 0;
                if (item < n && w < wcnt[sg]) v = __ldcg(keys + item * L.KW + wbeg[sg] + w);
                S.kc[sg][il][w] = v;
            }
        }
        __syncthreads();

        // issue chunk c of this tile into its ring stage
        auto issue = [&](int c) {
            const int stage = (gchunk + c) % T::NS;
            const bool seg0 = c < kc0;
            const int k0 = (seg0 ? c : c - kc0) * BK;
            const int src_row = seg0 ? st.in_row_off : st.sin_row_off;
            const int n_src = seg0 ? st.n_in : st.n_sin;
            const int valid = n_src - k0;
            if (tid == 0 && !wres) {   // boxes past the K extent are zero-filled and still complete their bytes
                mbar_expect_tx(&S.bar[stage], TM * BK * sizeof(double));
#pragma unroll
                for (int bx = 0; bx < BK / TB; bx++)
                    tma_load_2d(S.w[stage][bx], seg0 ? tmWp : tmVp, &S.bar[stage], k0 + bx * TB, m0);
            }
            if (C == 4) {
                // NI items x 1 KB in 16-B pieces
                constexpr int NP = NI * 64;
#pragma unroll
                for (int q = 0; q < (NP + T::NT - 1) / T::NT; q++) {
                    const int piece = q * T::NT + tid;
                    const int it = piece >> 6, j = piece & 63;   // item, 16-B piece within its 1 KB
                    const int64_t item = n0 / 4 + it;
                    const int krow = j >> 1;                 // 2 pieces per row (4 doubles)
                    if ((NP % T::NT == 0 || piece < NP) && item < n && krow < valid)
                        cp_async16(&S.x[stage][it * XS4 + j * 2],
                                   Zb + (item * L.zs + src_row + k0) * 4 + j * 2);
                }
                if (tid < NI) {
                    const int64_t item = n0 / 4 + tid;
                    const int sg = seg0 ? 0 : 1;
                    S.mask[stage][tid] = item >= n ? 0u
                        : cache_ok ? bits32(S.kc[sg][tid], src_row + k0 - wbeg[sg] * 64, valid)
                                   : bits32<true>(keys + item * L.KW, src_row + k0, valid);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int pt = tid >> 2, krow = (tid & 3) * 8 + q;
                    const int64_t item = n0 + pt;
                    if (item < n && krow < valid)
                        cp_async8(&S.x[stage][pt * XS1 + krow], Zb + item * L.zs + src_row + k0 + krow);
                }
                if (tid < BN) {
                    const int64_t item = n0 + tid;
                    const int sg = seg0 ? 0 : 1;
                    S.mask[stage][tid] = item >= n ? 0u
                        : cache_ok ? bits32(S.kc[sg][tid], src_row + k0 - wbeg[sg] * 64, valid)
                                   : bits32<true>(keys + item * L.KW, src_row + k0, valid);
                }
            }
            cp_async_commit();
        };

        double acc[2][NJ][4];
#pragma unroll
        for (int i = 0; i < 2; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++)
#pragma unroll
                for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;

        // NST-1 chunks in flight; the stage refilled at iteration c is the one chunk c-1 used,
        // which every warp has finished once it passes iteration c's barrier (one barrier per chunk)
        constexpr int NST = T::NS;
        const int pro = nchunks < NST - 1 ? nchunks : NST - 1;
        for (int c = 0; c < pro; c++) issue(c);
        // fragment row g reads tile row pg: the 4 rows x 2 16-B chunks of a half-warp then fall on
        // 8 distinct bank groups of the 128B-swizzled W stage
        const int pg = ((g & 3) << 1) | (g >> 2);

        for (int c = 0; c < nchunks; c++) {
            const uint32_t gc = gchunk + c;
            const int s = gc % NST;
            const int committed = (c + NST - 2 < nchunks - 1) ? c + NST - 2 : nchunks - 1;
            cp_async_wait(committed - c);
            if (wres) mbar_wait(&S.wbar, 0);
            else mbar_wait(&S.bar[s], (gc / NST) & 1);
            // the stage refilled below (by TMA, async proxy) was read through the generic proxy
            // in the previous chunk: order those reads before the refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (c + NST - 1 < nchunks) issue(c + NST - 1);
            const double* ws = S.w[wres ? c : s][0];
            const double* xsm = S.x[s];
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[2][2], b[NJ];
#pragma unroll
                for (int mi = 0; mi < 2; mi++) {
                    int r = wm * 32 + mi * 16 + pg;
                    a[mi][0] = ws[(kk / TB) * TM * TB + swz(r, (kk % TB) + t)];
                    a[mi][1] = ws[(kk / TB) * TM * TB + swz(r + 8, (kk % TB) + t)];
                }
#pragma unroll
                for (int nj = 0; nj < NJ; nj++) {
                    const int col = wn * WC + nj * 8 + g;
                    double v;
                    uint32_t mk;
                    if (C == 4) {
                        v = xsm[(col >> 2) * XS4 + (kk + t) * 4 + (col & 3)];
                        mk = S.mask[s][col >> 2];
                    } else {
                        v = xsm[col * XS1 + kk + t];
                        mk = S.mask[s][col];
                    }
                    b[nj] = ((mk >> (kk + t)) & 1u) ? v : 0.0;
                }
#pragma unroll
                for (int mi = 0; mi < 2; mi++)
#pragma unroll
                    for (int nj = 0; nj < NJ; nj++) dmma_16x8x4(acc[mi][nj], a[mi][0], a[mi][1], b[nj]);
            }
        }
        gchunk += nchunks;

    // ------------------------------------------------------ epilogue
        const int wbase = (st.row_off + m0) >> 6;  // forward: first key word the tile touches
#pragma unroll
        for (int mi = 0; mi < 2; mi++) {
#pragma unroll
            for (int half = 0; half < 2; half++) {
                const int rl = wm * 32 + mi * 16 + pg + half * 8;  // local row
                const int r = m0 + rl;
                const bool rok = r < st.n_out;
                const int row = st.row_off + r;
#pragma unroll
                for (int nj = 0; nj < NJ; nj++) {
                    const int64_t col = n0 + wn * WC + nj * 8 + 2 * t;
                    double v0 = acc[mi][nj][half * 2], v1 = acc[mi][nj][half * 2 + 1];
                    if (C == 4) {
                        const int64_t item = col >> 2;
                        const int comp = (int)(col & 3);  // 0 (even t) or 2 (odd t)
                        const bool ok = rok && item < n;
                        const int shp = (ok && L.shape_w >= 0) ? item_shape(keys + item * L.KW, L.shape_w) : 0;
                        if (ok && has_sc) {
                            double s0 = 0.0, s1 = 0.0;
                            if (sc_input_id) {            // A_in = I, c_in = 0 (block starts at x)
                                s0 = (comp == r) ? 1.0 : 0.0;
                                s1 = (comp == 0 && r == 1) ? 1.0 : 0.0;
                            } else if (sc_input_lin) {    // V @ I = V[:, :3], V @ 0 + vb
                                const double* vr = st.V + (int64_t)r * st.ldv;
                                s0 = vr[comp];
                                s1 = comp == 0 ? vr[1] : (has_vb ? step_vbias(st, shp, r) : 0.0);
                            } else if (sc_ident) {        // masked block input rows
                                const uint64_t* key = keys + item * L.KW;
                                int srow = st.sin_row_off + r;
                                if (key_bit_cg(key, srow)) {
                                    double2 p = *reinterpret_cast<const double2*>(Zb + (item * L.zs + srow) * 4 + comp);
                                    s0 = p.x; s1 = p.y;
                                }
                            } else {                      // V @ A_in is in acc (second K segment); add vb
                                s1 = (comp == 2 && has_vb) ? step_vbias(st, shp, r) : 0.0;
                            }
                            v0 = s0 + v0;   // pre_A = sA + W A ; pre_c = (sc + W c) + b
                            v1 = s1 + v1;
                        }
                        if (comp == 2) v1 = v1 + (ok ? step_bias(st, shp, r) : 0.0);
                        v0 = prec_round(v0, L.fp32);
                        v1 = prec_round(v1, L.fp32);
                        // canonical bit: the pair (t, t^1) holds the 4 components of (item, row)
                        double p0 = __shfl_xor_sync(0xffffffffu, v0, 1);
                        double p1 = __shfl_xor_sync(0xffffffffu, v1, 1);
                        if (ok) {
                            if (comp == 0) {
                                double nrm = sqrt((v0 * v0 + v1 * v1) + p0 * p0);
                                if (!(nrm > kDegen)) {
                                    uint64_t* key = keys + item * L.KW;
                                    int bit = p1 > 0.0;
                                    if (bit != key_bit(key, row)) {
                                        set_key_bit(key, row, bit);
                                        if (L.changed) L.changed[item] = 1;
                                    }
                                }
                            }
                            *reinterpret_cast<double2*>(Zb + (item * L.zs + row) * 4 + comp) = make_double2(v0, v1);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const int64_t item = col + e;
                            double v = e ? v1 : v0;
                            if (!(rok && item < n)) continue;
                            const int shp = L.shape_w >= 0 ? item_shape(keys + item * L.KW, L.shape_w) : 0;
                            double pre;
                            if (has_sc) {
                                double sc = 0.0;
                                const double* x = L.pts ? L.pts + item * 3 : nullptr;
                                if (sc_input_id) {
                                    sc = x[r];
                                } else if (sc_input_lin) {
                                    const double* vr = st.V + (int64_t)r * st.ldv;
                                    sc = (x[0] * vr[0] + x[1] * vr[1]) + x[2] * vr[2];
                                    if (has_vb) sc = sc + step_vbias(st, shp, r);
                                } else if (sc_ident) {
                                    int srow = st.sin_row_off + r;
                                    if (key_bit(keys + item * L.KW, srow)) sc = Zb[item * L.zs + srow];
                                } else if (has_vb) {
                                    sc = step_vbias(st, shp, r);  // V h_in is in acc (second K segment)
                                }
                                pre = (sc + v) + step_bias(st, shp, r);   // reference: shortcut(h_in) + h W^T + b
                            } else {
                                pre = v + step_bias(st, shp, r);
                            }
                            pre = prec_round(pre, L.fp32);
                            Zb[item * L.zs + row] = pre;
                            if (pre > 0.0) {
                                int lb = row - wbase * 64;
                                atomicOr(&S.bits[(int)(item - n0)][lb >> 6], (unsigned long long)key_mask(lb));
                            }
                        }
                    }
                }
            }
        }
        if (C == 1) {
            __syncthreads();
            if (tid < BN) {
                int64_t item = n0 + tid;
                if (item < n) {
                    uint64_t* key = keys + item * L.KW;
                    if (S.bits[tid][0]) atomicOr(reinterpret_cast<unsigned long long*>(key + wbase), S.bits[tid][0]);
                    if (S.bits[tid][1] && wbase + 1 < L.KW)
                        atomicOr(reinterpret_cast<unsigned long long*>(key + wbase + 1), S.bits[tid][1]);
                }
            }
            __syncthreads();
        }
    }
}

// Persistent: each CTA walks output tiles (64 neuron rows x 64 item columns) of the
// device-resident item count (graph-capturable).  K is streamed in 16-row chunks through an
// NST-stage ring: W by TMA (mbarrier), the raw activations by cp.async, the state mask of the
// chunk as 16-bit words -- applied when the B fragments are read, so padding rows and
// inactive neurons contribute exact zeros.
template <int C, int TM, int NJ = 2>
__global__ void __launch_bounds__(GT<C, TM, NJ>::NT, GT<C, TM, NJ>::CPS) k_gemm_step(const __grid_constant__ CUtensorMap tmW,
                                                        const __grid_constant__ CUtensorMap tmV, LayerLaunch L) {
    extern __shared__ uint8_t smem_raw[];
    // 1 KB-aligned view derived by pointer arithmetic on the shared array (keeps LDS addressing)
    GemmSmem<C, TM, NJ>& S = *reinterpret_cast<GemmSmem<C, TM, NJ>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    using T = GT<C, TM, NJ>;
    const StepDev& st = L.st;
    const int tid = threadIdx.x;
    const bool lin = (st.flags & AM_STEP_SHORTCUT_LINEAR) && !(st.flags & AM_STEP_SC_FROM_INPUT);
    const int kc0 = (st.n_in + BK - 1) / BK;
    const int nchunks = kc0 + (lin ? (st.n_sin + BK - 1) / BK : 0);
    // W is a weight (not produced by the preceding kernels): its TMA is issued before the grid
    // dependency wait, so it overlaps the predecessor's tail
    const bool wres = T::WRES && st.n_out <= TM && nchunks <= T::WS;

    if (tid < T::NS) mbar_init(&S.bar[tid], 1);
    if (tid == T::NS) mbar_init(&S.wbar, 1);
    if (tid == 0) {
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    }
    __syncthreads();
    if (wres && tid == 0) {
        mbar_expect_tx(&S.wbar, (uint32_t)(nchunks * TM * BK * sizeof(double)));
        for (int c = 0; c < nchunks; c++) {
            const bool seg0 = c < kc0;
            const int k0 = (seg0 ? c : c - kc0) * BK;
#pragma unroll
            for (int bx = 0; bx < BK / TB; bx++)
                tma_load_2d(S.w[c][bx], seg0 ? &tmW : &tmV, &S.wbar, k0 + bx * TB, 0);
        }
    }
    pdl_enter();
    const int64_t n = dev_count(L.n_dev, L.n_cap);
    if (n <= 0) {
        if (wres) mbar_wait(&S.wbar, 0);   // no bulk copy may be in flight when the CTA exits
        return;
    }
    uint64_t* keys = keys_at(L);
    constexpr int TN = T::TN;
    const int64_t ntx = (n * C + TN - 1) / TN;
    const int nty = (st.n_out + TM - 1) / TM;
    const int64_t ntiles = ntx * nty;

    uint32_t gchunk = 0;  // chunks consumed by this CTA so far (stage ring + mbarrier phases)
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // column-block-major: the row tiles of one activation block run on neighbouring CTAs at the
        // same time and share its staging through L2 (row-major re-streamed every activation block
        // once per row tile from DRAM: ~7x the input on DeepSDF 512x8)
        const int m0 = (int)(tile % nty) * TM;
        const int64_t n0 = (tile / nty) * TN;
        gemm_tile<C, TM, NJ>(S, L, keys, n, &tmW, &tmV, m0, n0, gchunk, wres);
    }
    if (wres && blockIdx.x >= ntiles) mbar_wait(&S.wbar, 0);
}

template <int C, int TM, int NJ = 2>
static void launch_gemm_tm(const LayerLaunch& L, const CUtensorMap* tmW, const CUtensorMap* tmV, cudaStream_t s) {
    using T = GT<C, TM, NJ>;
    const int64_t cols = L.n_cap * C;
    const int64_t tiles = ((cols + T::TN - 1) / T::TN) * ((L.st.n_out + TM - 1) / TM);
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)num_sms() * (L.grid_cap > 0 ? L.grid_cap : T::CPS));
    const size_t smem = sizeof(GemmSmem<C, TM, NJ>) + 1024;
    static bool init[64] = {};   // the attribute is per function and device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !init[dev]) {
        cudaFuncSetAttribute(k_gemm_step<C, TM, NJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev < 64) init[dev] = true;
    }
    launch_k(k_gemm_step<C, TM, NJ>, (unsigned)grid, T::NT, smem, s, *tmW, tmV ? *tmV : *tmW, L);
}

void launch_gemm_step(const LayerLaunch& L, int C, const CUtensorMap* tmW, const CUtensorMap* tmV, cudaStream_t s,
                      const CUtensorMap* tmW96, const CUtensorMap* tmV96) {
    if (L.n_cap <= 0) return;
    if (C == 4 && tmW96) launch_gemm_tm<4, 96>(L, tmW96, tmV96, s);
    else if (C == 4 && L.nj4) launch_gemm_tm<4, 64, 4>(L, tmW, tmV, s);
    else if (C == 4) launch_gemm_tm<4, 64>(L, tmW, tmV, s);
    else launch_gemm_tm<1, 64>(L, tmW, tmV, s);
}

// ------------------------------------------------- fused composition (all steps)
// One launch composes every step of a batch of cells and their face functionals: a CTA owns a
// block of 16 cells (64 columns) and walks the steps in order -- the input step elementwise,
// each hidden step as its 64-row output tiles (gemm_tile: TMA-staged W, DMMA, epilogue) -- with
// a barrier between steps, then the heads.  Every step's K extent is the previous steps' rows of
// the same cells, all produced by this CTA, so no grid-wide dependency exists and the ~L+2
// per-layer launches of a BFS iteration (each paying its own pipeline fill) become one.
__global__ void __launch_bounds__(kThreads, 2) k_compose_fused(const __grid_constant__ FusedCompose F) {
    pdl_enter();
    extern __shared__ uint8_t smem_raw[];
    GemmSmem<4>& S = *reinterpret_cast<GemmSmem<4>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = dev_count(F.L.n_dev, F.L.n_cap);
    if (n <= 0) return;
    uint64_t* keys = keys_at(F.L);
    if (tid < NST) mbar_init(&S.bar[tid], 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int64_t nblk = (n * 4 + BN - 1) / BN;
    uint32_t gchunk = 0;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        const int64_t n0 = blk * BN, item0 = n0 / 4;
        for (int s = 0; s < F.nsteps; s++) {
            LayerLaunch L = F.L;
            L.st = F.st[s];
            if (L.st.flags & AM_STEP_FIRST) {
                const int no = L.st.n_out;
                for (int idx = tid; idx < 16 * no; idx += kThreads) {
                    const int64_t item = item0 + idx / no;
                    if (item < n) input_elem<4>(L, keys, item, idx % no);
                }
            } else {
                for (int m0 = 0; m0 < L.st.n_out; m0 += BM)
                    gemm_tile<4>(S, L, keys, n, &F.tmW[s], F.tmV_ok[s] ? &F.tmV[s] : &F.tmW[s], m0, n0, gchunk);
            }
            __threadfence();
            __syncthreads();
        }
        // face functional of every subnetwork (reference network.py:440-442), warp per (cell, sub)
        for (int wid = warp; wid < 16 * F.n_subs; wid += kThreads / 32) {
            const int64_t item = item0 + wid / F.n_subs;
            const int j = wid % F.n_subs;
            if (item >= n) continue;
            const SubDev sd = F.subs[j];
            const uint64_t* key = keys + item * F.L.KW;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            for (int r = lane; r < sd.last_n; r += 32) {
                const int row = sd.last_row + r;
                if (!key_bit_cg(key, row)) continue;
                const double2* p = reinterpret_cast<const double2*>(F.L.Z + (item * F.L.zs + row) * 4);
                const double2 x = p[0], y = p[1];
                const double w = sd.hw[r];
                a0 += w * x.x; a1 += w * x.y; a2 += w * y.x; a3 += w * y.y;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o);
                a3 += __shfl_xor_sync(0xffffffffu, a3, o);
            }
            if (lane == 0) {
                double* f = F.faces + (item * F.n_subs + j) * 4;
                f[0] = prec_round(a0, F.L.fp32); f[1] = prec_round(a1, F.L.fp32); f[2] = prec_round(a2, F.L.fp32);
                f[3] = prec_round(a3 + head_bias(sd, item_shape(key, F.L.shape_w)), F.L.fp32);
            }
        }
        __syncthreads();
    }
}

void launch_compose_fused(const FusedCompose& F, cudaStream_t s) {
    if (F.L.n_cap <= 0) return;
    const int64_t blocks = (F.L.n_cap * 4 + BN - 1) / BN;
    const int64_t grid = std::min<int64_t>(blocks, (int64_t)num_sms() * 2);
    const size_t smem = sizeof(GemmSmem<4>) + 1024;
    static bool init[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !init[dev]) {
        cudaFuncSetAttribute(k_compose_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (dev < 64) init[dev] = true;
    }
    launch_k(k_compose_fused, (unsigned)grid, kThreads, smem, s, F);
}

// ------------------------------------------------------------ head kernels

// face functional of every subnetwork: head_w @ (s ⊙ Z_last) (+ head_b on the offset)
// reference network.py:440-442
__global__ void k_face_head(const double* Z, const uint64_t* keys, double* faces, const unsigned long long* n_dev,
                            int64_t n_cap, int zs, int KW, const SubDev* subs, int n_subs, int shape_w, int fp32,
                            const unsigned long long* zpar, int64_t zstride) {
    pdl_enter();
    if (zpar) Z += (int64_t)(*zpar & 1ull) * zstride;
    const int64_t n = dev_count(n_dev, n_cap);
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wid < n * n_subs; wid += nw) {
        int64_t item = wid / n_subs;
        int j = (int)(wid - item * n_subs);
        const SubDev sd = subs[j];
        const uint64_t* key = keys + item * KW;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        for (int r = lane; r < sd.last_n; r += 32) {
            int row = sd.last_row + r;
            if (!key_bit(key, row)) continue;
            const double2* p = reinterpret_cast<const double2*>(Z + (item * zs + row) * 4);
            double2 x = p[0], y = p[1];
            double w = sd.hw[r];
            a0 += w * x.x; a1 += w * x.y; a2 += w * y.x; a3 += w * y.y;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            a3 += __shfl_xor_sync(0xffffffffu, a3, o);
        }
        if (lane == 0) {
            double* f = faces + (item * n_subs + j) * 4;
            f[0] = prec_round(a0, fp32); f[1] = prec_round(a1, fp32); f[2] = prec_round(a2, fp32);
            f[3] = prec_round(a3 + head_bias(sd, item_shape(key, shape_w)), fp32);
        }
    }
}

// F_j(x) = head_w @ relu(Z_last) + head_b; F = max_j (argmax lowest index) -- reference network.py:352-392
__global__ void k_forward_head(const double* Z, uint64_t* keys_base, const unsigned long long* key_off, double* vals,
                               const unsigned long long* n_dev, int64_t n_cap, int zs, int KW, const SubDev* subs,
                               int n_subs, int ensemble, int shape_w, int fp32) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    uint64_t* keys = key_off ? keys_base + (int64_t)(*key_off) * KW : keys_base;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < n; item += nw) {
        const uint64_t* key = keys + item * KW;
        double best = 0.0;
        int arg = 0;
        for (int j = 0; j < n_subs; j++) {
            const SubDev sd = subs[j];
            double a = 0.0;
            for (int r = lane; r < sd.last_n; r += 32) {
                int row = sd.last_row + r;
                if (key_bit(key, row)) a += Z[item * zs + row] * sd.hw[r];
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            double f = prec_round(a + head_bias(sd, item_shape(key, shape_w)), fp32);
            if (j == 0 || f > best) { best = f; arg = j; }
        }
        if (lane == 0) {
            if (vals) vals[item] = best;
            if (ensemble) keys[item * KW + KW - 1] = (uint64_t)arg;
        }
    }
}

void launch_face_head_dev(const double* Z, const uint64_t* keys, double* faces, const unsigned long long* n_dev,
                          int64_t n_cap, int zs, int KW, const void* subs, int n_subs, int shape_w, int fp32,
                          cudaStream_t s, const unsigned long long* zpar, int64_t zstride) {
    int64_t warps = n_cap * n_subs;
    if (warps <= 0) return;
    int64_t blocks = std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)num_sms() * 8);
    { launch_k(k_face_head, (unsigned)blocks, 256, 0, s, Z, keys, faces, n_dev, n_cap, zs, KW,
                                                 static_cast<const SubDev*>(subs), n_subs, shape_w, fp32, zpar, zstride); }
}
void launch_forward_head_dev(const double* Z, uint64_t* keys, const unsigned long long* key_off, double* vals,
                             const unsigned long long* n_dev, int64_t n_cap, int zs, int KW, const void* subs,
                             int n_subs, int ensemble, int shape_w, int fp32, cudaStream_t s) {
    if (n_cap <= 0) return;
    int64_t blocks = std::min<int64_t>((n_cap * 32 + 255) / 256, (int64_t)num_sms() * 8);
    { launch_k(k_forward_head, (unsigned)blocks, 256, 0, s, Z, keys, key_off, vals, n_dev, n_cap, zs, KW,
                                                    static_cast<const SubDev*>(subs), n_subs, ensemble, shape_w, fp32); }
}

}  // namespace am
