// am_narrow.cu -- the whole composition of a BFS iteration in ONE launch, for narrow plain MLPs.
//
// Networks whose hidden layers are all plain dense layers of width <= 96 (configs[0] 3-60-60-1,
// configs[1] 3-(90x6)-1, the reference's random test nets) compose a cell as a chain of small
// dependent GEMMs: Z_l = W_l (s_{l-1} (.) Z_{l-1}) + b_l, 90 x 90 x 4 per cell and layer
// (reference network.py:398-443 _region_maps_sub).  The per-layer kernels (am_compose.cu
// k_gemm_step) pay a launch, a TMA pipeline fill and a grid-wide drain per layer for a
// K extent of only 96; on configs[1]'s ~2.5 k-cell waves that left the DMMA pipe at 27 %.
//
// Here one persistent CTA owns a tile of 8 cells (32 columns = 8 cells x (nx, ny, nz, c)) and
// walks every layer with the tile's activations resident in shared memory:
//
//   gather   the tile's pool entries from the BFS queue slice (k_gather_batch's work)
//   step 0   A_1 = W_1, c_1 = b_1 elementwise (A_0 = I), canonical bits, Z rows -> HBM
//   step l   96 x 32 x K DMMA tile (mma.sync m16n8k4 f64 -> DMMA.8x8x4): A = W_l from a 4-box
//            TMA ring (96 rows x 16 k, 128B swizzle) fed by a dedicated producer warp through
//            full / empty mbarriers -- the ring runs across layers AND tiles, so W of the next
//            layer streams in while the current one computes and the pipeline fills once per
//            CTA; B = the previous layer's output from shared memory, already masked by the
//            state bits (applied once in the epilogue that wrote it, not per fragment read)
//   epilogue bias, fp32-mode rounding, canonical bit of constant neurons (shared-memory key),
//            raw Z rows -> HBM (the face solver's planes), masked rows -> the other act buffer
//   head     F = head . (s_L (.) Z_L) per cell from shared memory (reference network.py:440-442)
//
// so a BFS iteration's gather + L + 1 launches become one.  With prefix reuse tiles
// are formed per bucket of cells that share steps 0..f with their parents (k_take's blist): such a
// tile copies the parents' rows of steps 1..f from the other half of the double-buffered Z, tests
// step f's rows for constant neurons, and starts the DMMA chain at step f + 1 (the producer skips
// the W boxes of the skipped steps).  6 consumer warps (3 x 2 warp tiles
// of 32 x 16) + 1 producer warp, ~107 KB shared memory, 2 CTAs per SM.  Arithmetic per output
// element is the same as k_gemm_step's (DMMA accumulation over K, then + bias), so the two
// paths agree to the last bit on the same K order; parity is checked against the oracle.
#include <algorithm>

#include "am_internal.h"
#include "am_hashset.cuh"
#include "am_near.cuh"
#include "am_ptx.cuh"

namespace am {

namespace {

constexpr int NR = 96;          // max rows (layer width) of the tile
constexpr int NCELL = 8;        // cells per tile
constexpr int NCOL = NCELL * 4; // columns
constexpr int AS = NCOL + 4;    // act row stride (doubles): conflict-free B fragments
constexpr int KB = 16;          // K per W box (128 B rows)
#ifndef AM_NARROW_NSB
#define AM_NARROW_NSB 4
#endif
#ifndef AM_NARROW_NACT
#define AM_NARROW_NACT 2
#endif
#ifndef AM_NARROW_CPS
#define AM_NARROW_CPS 2
#endif
constexpr int NSB = AM_NARROW_NSB;    // W ring boxes
constexpr int NACT = AM_NARROW_NACT;  // act buffers: 2 = ping-pong (one barrier per layer), 1 = in place (two)
constexpr int CPS = AM_NARROW_CPS;    // resident CTAs per SM
constexpr int NCW = 6;          // consumer warps
constexpr int NCT = NCW * 32;   // consumer threads
constexpr int NT = NCT + 32;    // + producer warp
constexpr int KWMAX = 20;       // key words per cell held in shared memory (<= 1280 state bits)

struct __align__(1024) NarrowSmem {
    double w[NSB][NR * KB];       // TMA destinations (1 KB aligned for the 128B swizzle)
    double act[NACT][NR * AS];    // masked layer outputs [row][col]
    uint64_t key[NCELL][KWMAX];   // the tile's state keys (canonical bits updated in place)
    double p1[NR * 4];            // step 0's planes (W_1[:, :3], b_1) per row, staged once per CTA
    double hw[NR];                // head weights
    uint32_t deg1[NR / 32];       // step-0 rows with a degenerate (zero) normal
    uint64_t full[NSB], empty[NSB];
    int changed[NCELL];
    int32_t bidx[NCELL];          // batch item of each tile cell
    int32_t pitem[NCELL];         // prefix reuse: the parent's batch item (previous iteration)
};

// Tiles of an iteration.  Without prefix reuse: consecutive batch items.  With it: per bucket f
// (cells sharing steps 0..f with their parents, ascending f), each bucket cut into tiles of nc
// cells of blist.  Producer and consumers derive the same (f, cells) from the bucket counts.
struct Tiling {
    int nb;                        // buckets (1 without prefix reuse)
    long long cnt[kMaxPrefixBuckets];
    long long ntiles;
    __device__ void init(const NarrowCompose& P, int64_t n, int nc) {
        if (!P.prefix) { nb = 1; cnt[0] = n; ntiles = (n + nc - 1) / nc; return; }
        nb = P.nsteps < kMaxPrefixBuckets ? P.nsteps : kMaxPrefixBuckets;
        ntiles = 0;
        for (int f = 0; f < nb; f++) {
            cnt[f] = (long long)P.ctr[C_BK0 + f];
            ntiles += (cnt[f] + nc - 1) / nc;
        }
    }
    // tile t -> (bucket f, first position in the bucket, cells)
    __device__ void locate(long long t, int nc, int& f, long long& pos, int& ncell) const {
        f = 0;
        for (; f < nb - 1; f++) {
            const long long tf = (cnt[f] + nc - 1) / nc;
            if (t < tf) break;
            t -= tf;
        }
        pos = t * nc;
        const long long left = cnt[f] - pos;
        ncell = (int)(left < nc ? left : nc);
    }
};

__device__ __forceinline__ int skey_bit(const uint64_t* k, int i) {
    return (int)((k[i >> 6] >> (63 - (i & 63))) & 1ull);
}
__device__ __forceinline__ void skey_set(uint64_t* k, int i, int bit) {
    unsigned long long* w = reinterpret_cast<unsigned long long*>(k + (i >> 6));
    const unsigned long long m = key_mask(i);
    if (bit) atomicOr(w, m);
    else atomicAnd(w, ~m);
}

// !(|(x, y, z)| > 1e-12) -- the reference's constant-functional test (network.py:421-428) -- with
// the square root taken only near the threshold: a squared norm far from 1e-24 decides it alone
__device__ __forceinline__ bool degenerate3(double x, double y, double z) {
    const double ss = (x * x + y * y) + z * z;
    if (ss > 2.0e-24) return false;
    if (ss < 0.5e-24) return true;
    return !(sqrt(ss) > kDegen);
}

// |x| > t (t > 0) on the integer pipe; NaN counts as not greater, so a NaN normal takes the exact
// norm test like every small one
constexpr double kBig = 2e-12;
__device__ __forceinline__ bool fabs_gt(double x, double t) {
    const unsigned long long ax = (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
    return ax > (unsigned long long)__double_as_longlong(t) && ax <= 0x7ff0000000000000ull;
}

// the CTA's k-th tile: round-robin, or (P.snake, with the tiles ordered costliest first by the
// prefix buckets) boustrophedon -- odd rounds run backwards, so the CTAs that drew the full-chain
// tiles of bucket 0 draw the cheapest ones next
__device__ __forceinline__ int64_t tile_of(const NarrowCompose& P, int64_t k) {
    const int64_t g = gridDim.x;
    return k * g + ((P.snake && (k & 1)) ? g - 1 - (int64_t)blockIdx.x : (int64_t)blockIdx.x);
}

// The consumer warps' tile loop for one tile width: MI 16-row fragments x NJ 8-column fragments
// per warp; 6 warps = WR row blocks x WC column blocks; a tile is NC = WC * NJ * 2 cells.
//   MI 2, NJ 2: 3 x 2 warps of 32 x 16, 8 cells (wide waves)
//   MI 1, NJ 2: 6 x 1 warps of 16 x 16, 4 cells
//   MI 1, NJ 1: 6 x 1 warps of 16 x 8,  2 cells (narrow waves: spread over more SMs)
template <int FP32, int MI, int NJ>
__device__ __forceinline__ void consume(NarrowSmem& S, const NarrowCompose& P, int64_t n,
                                        uint32_t& gbox, bool prof, unsigned long long& tprev, double* Zc,
                                        const double* Zp) {
    constexpr int WR = MI == 2 ? 3 : 6, WC = NCW / WR, RB = 16 * MI, CB = 8 * NJ;
    constexpr int NC = WC * NJ * 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ns = P.nsteps;
    const int KW = P.KW;
    Tiling T;
    T.init(P, n, NC);
    const int64_t ntiles = T.ntiles;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = warp % WR, wn = warp / WR;
    const int pg = ((g & 3) << 1) | (g >> 2);   // fragment row permutation (bank-conflict-free W reads)
    constexpr int fp32 = FP32;
    const bool shaped = P.shape_w >= 0;   // batch of shapes: biases per cell's shape
#define PROF(i) do { if (prof) { unsigned long long tn = clock64(); atomicAdd(&P.prof[i], tn - tprev); tprev = tn; } } while (0)

    for (int64_t k = 0; k * gridDim.x < ntiles; k++) {
        const int64_t t = tile_of(P, k);
        if (t >= ntiles) continue;
        int fsh, ncell;
        long long pos0;
        T.locate(t, NC, fsh, pos0, ncell);
        // ---- gather (reference order: the BFS queue slice k_take dequeued)
        for (int q = tid; q < NC * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            uint64_t v = 0;
            if (c < ncell && P.keys_in) {   // explicit keys (seeds, affine maps): no queue, no pool
                const int64_t b = pos0 + c;
                v = P.keys_in[b * KW + w];
                if (w == 0) S.bidx[c] = (int32_t)b;
            } else if (c < ncell) {
                const int64_t b = P.prefix ? (int64_t)P.blist[(int64_t)fsh * P.n_cap + pos0 + c] : pos0 + c;
                const int32_t p = P.queue[batch_queue_index(P.ctr, b)];
                v = P.pool[(int64_t)p * KW + w];
                if (w == 0) {
                    S.bidx[c] = (int32_t)b;
                    if (fsh) S.pitem[c] = (int32_t)(((unsigned long long)P.pool_par[p] >> 5) & 0x7ffffffull);
                    P.batch_pool[b] = p;
                    P.canon_pos[b] = -1;
                    reinterpret_cast<double4*>(P.ckey_hint)[b] = reinterpret_cast<const double4*>(P.pool_hint)[p];
                }
            }
            S.key[c][w] = v;
        }
        if (tid < NCELL) S.changed[tid] = 0;
        bar_sync(1, NCT);
        PROF(0);

        // ---- step 0: A_1 = W_1[:, :3], c_1 = b_1 (reference network.py:398-443 with A = I, c = 0)
        {
            const StepDev& st = P.st[0];
            const int no = st.n_out;
            for (int idx = tid; idx < ncell * no; idx += NCT) {
                const int c = idx / no, r = idx - c * no;
                const int64_t item = S.bidx[c];
                uint64_t* key = S.key[c];
                const int row = st.row_off + r;
                const double2 pa = *reinterpret_cast<const double2*>(&S.p1[r * 4]);
                const double a2 = S.p1[r * 4 + 2];
                double cc = S.p1[r * 4 + 3];
                if (shaped) cc = prec_round(0.0 + step_bias(st, item_shape(key, P.shape_w), r), fp32);
                int bit = skey_bit(key, row);
                if ((S.deg1[r >> 5] >> (r & 31)) & 1u) {
                    const int cb = cc > 0.0;
                    if (cb != bit) { skey_set(key, row, cb); S.changed[c] = 1; bit = cb; }
                }
                double* z = Zc + (item * P.zs + row) * 4;
                reinterpret_cast<double2*>(z)[0] = pa;
                reinterpret_cast<double2*>(z)[1] = make_double2(a2, cc);
                double* ao = &S.act[0][r * AS + c * 4];
                reinterpret_cast<double2*>(ao)[0] = bit ? pa : make_double2(0.0, 0.0);
                reinterpret_cast<double2*>(ao)[1] = bit ? make_double2(a2, cc) : make_double2(0.0, 0.0);
            }
            bar_sync(1, NCT);
            PROF(1);
        }

        // ---- prefix reuse: Z rows of steps 1..fsh are the parent's (same bits in every earlier
        // layer); the masked rows of step fsh (own bits, canonical test of the flipped neuron)
        // feed step fsh + 1
        if (fsh) {
            const StepDev& sf = P.st[fsh];
            const int r0 = P.st[1].row_off, rf = sf.row_off, nrow = rf + sf.n_out - r0;
            for (int idx = tid; idx < ncell * nrow; idx += NCT) {
                const int c = idx / nrow, row = r0 + (idx - c * nrow);
                const double2* src = reinterpret_cast<const double2*>(Zp + ((int64_t)S.pitem[c] * P.zs + row) * 4);
                const double2 v0 = src[0], v1 = src[1];
                double2* dst = reinterpret_cast<double2*>(Zc + ((int64_t)S.bidx[c] * P.zs + row) * 4);
                dst[0] = v0;
                dst[1] = v1;
                if (row >= rf) {
                    int bit = skey_bit(S.key[c], row);
                    if (degenerate3(v0.x, v0.y, v1.x)) {
                        const int cb = v1.y > 0.0;
                        if (cb != bit) { skey_set(S.key[c], row, cb); S.changed[c] = 1; bit = cb; }
                    }
                    double* ao = &S.act[0][(row - rf) * AS + c * 4];
                    reinterpret_cast<double2*>(ao)[0] = bit ? v0 : make_double2(0.0, 0.0);
                    reinterpret_cast<double2*>(ao)[1] = bit ? v1 : make_double2(0.0, 0.0);
                }
            }
            bar_sync(1, NCT);
        }

        // ---- GEMM steps
        int cur = 0;
        for (int s = fsh + 1; s < ns; s++) {
            const StepDev& st = P.st[s];
            const int nb = (st.n_in + KB - 1) / KB;
            double acc[MI][NJ][4];
#pragma unroll
            for (int i = 0; i < MI; i++)
#pragma unroll
                for (int j = 0; j < NJ; j++)
#pragma unroll
                    for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;
            double bias[MI][2];   // this thread's output rows (loads overlap the K loop)
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const int r = wm * RB + mi * 16 + pg + half * 8;
                    bias[mi][half] = (r < st.n_out && !shaped) ? st.b[r] : 0.0;
                }
            const double* xs = S.act[cur];
            for (int b = 0; b < nb; b++, gbox++) {
                const int slot = gbox % NSB;
                const unsigned long long tw = prof ? clock64() : 0ull;
                mbar_wait(&S.full[slot], (gbox / NSB) & 1);
                if (prof) atomicAdd(&P.prof[8], clock64() - tw);
                const double* ws = S.w[slot];
                // (skipping the all-zero k-steps past the layer's K extent measured slower: 20.0 vs
                // 19.65 ms -- the fully unrolled box schedules its fragment loads better)
#pragma unroll
                for (int kk = 0; kk < KB; kk += 4) {
                    double a[MI][2], bf[NJ];
#pragma unroll
                    for (int mi = 0; mi < MI; mi++) {
                        const int r = wm * RB + mi * 16 + pg;
                        a[mi][0] = ws[swz(r, kk + tq)];
                        a[mi][1] = ws[swz(r + 8, kk + tq)];
                    }
                    const int k = b * KB + kk + tq;
#pragma unroll
                    for (int nj = 0; nj < NJ; nj++) bf[nj] = xs[k * AS + wn * CB + nj * 8 + g];
#pragma unroll
                    for (int mi = 0; mi < MI; mi++)
#pragma unroll
                        for (int nj = 0; nj < NJ; nj++) dmma_16x8x4(acc[mi][nj], a[mi][0], a[mi][1], bf[nj]);
                }
                // release the slot: the generic-proxy reads of this box must be ordered before the
                // TMA (async proxy) that will overwrite it -- without the proxy fence a refill was
                // observed to land under the last k-step's fragment loads (rare corrupted tiles)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[slot]);
            }
            PROF(2);
            // epilogue
            if (NACT == 1) bar_sync(1, NCT);   // in place: every warp has read the layer's input
            double* xo = S.act[NACT == 1 ? 0 : cur ^ 1];
#pragma unroll
            for (int mi = 0; mi < MI; mi++) {
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const int r = wm * RB + mi * 16 + pg + half * 8;
                    const bool rok = r < st.n_out;
                    const int row = st.row_off + r;
#pragma unroll
                    for (int nj = 0; nj < NJ; nj++) {
                        const int col = wn * CB + nj * 8 + 2 * tq;
                        const int c = col >> 2, comp = col & 3;   // comp 0 or 2
                        const bool ok = rok && c < ncell;
                        double v0 = acc[mi][nj][half * 2], v1 = acc[mi][nj][half * 2 + 1];
                        if (comp == 2)
                            v1 = v1 + (!ok ? 0.0 : shaped ? step_bias(st, item_shape(S.key[c], P.shape_w), r) : bias[mi][half]);
                        v0 = prec_round(v0, fp32);
                        v1 = prec_round(v1, fp32);
                        // Constant-functional test of (cell, row), whose 4 components sit in the lane
                        // pair (tq, tq ^ 1): a normal component above 2e-12 settles it without fp64
                        // math (|n| >= that component); only pairs with every component below run
                        // the reference's norm test (uniform branch, rare).
                        const bool big = (comp == 0) ? (fabs_gt(v0, kBig) || fabs_gt(v1, kBig)) : fabs_gt(v0, kBig);
                        const unsigned bal = __ballot_sync(0xffffffffu, big);
                        bool deg = !((bal >> lane) & 1u) && !((bal >> (lane ^ 1)) & 1u);
                        if (__any_sync(0xffffffffu, deg && ok)) {
                            const double p0 = __shfl_xor_sync(0xffffffffu, v0, 1);
                            const double p1 = __shfl_xor_sync(0xffffffffu, v1, 1);
                            if (deg) {
                                const double nx = comp == 0 ? v0 : p0, ny = comp == 0 ? v1 : p1;
                                const double nz = comp == 0 ? p0 : v0;
                                deg = degenerate3(nx, ny, nz);
                            }
                            // the sign of the offset decides a constant neuron's bit
                            const double cc = comp == 0 ? p1 : v1;
                            if (ok) {
                                int bit = skey_bit(S.key[c], row);
                                if (deg) {
                                    const int cb = cc > 0.0;
                                    if (cb != bit) {
                                        if (comp == 0) { skey_set(S.key[c], row, cb); S.changed[c] = 1; }
                                        bit = cb;
                                    }
                                }
                                *reinterpret_cast<double2*>(Zc + ((int64_t)S.bidx[c] * P.zs + row) * 4 + comp) = make_double2(v0, v1);
                                *reinterpret_cast<double2*>(xo + r * AS + col) = bit ? make_double2(v0, v1) : make_double2(0.0, 0.0);
                            }
                        } else if (ok) {
                            const int bit = skey_bit(S.key[c], row);
                            *reinterpret_cast<double2*>(Zc + ((int64_t)S.bidx[c] * P.zs + row) * 4 + comp) = make_double2(v0, v1);
                            *reinterpret_cast<double2*>(xo + r * AS + col) = bit ? make_double2(v0, v1) : make_double2(0.0, 0.0);
                        }
                    }
                }
            }
            PROF(3);
            bar_sync(1, NCT);
            PROF(6);
            if (NACT == 2) cur ^= 1;
        }

        // ---- face functional: head . (s_L (.) Z_L) (+ head bias on the offset)
        {
            const SubDev sd = P.subs[0];
            for (int c = warp; c < ncell; c += NCW) {
                double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
                const double* xs = S.act[cur];
                for (int r = lane; r < sd.last_n; r += 32) {
                    const double2 x = *reinterpret_cast<const double2*>(xs + r * AS + c * 4);
                    const double2 y = *reinterpret_cast<const double2*>(xs + r * AS + c * 4 + 2);
                    const double w = S.hw[r];
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
                    double* f = P.faces + (int64_t)S.bidx[c] * 4;
                    f[0] = prec_round(a0, fp32); f[1] = prec_round(a1, fp32); f[2] = prec_round(a2, fp32);
                    f[3] = prec_round(a3 + head_bias(sd, item_shape(S.key[c], P.shape_w)), fp32);
                }
            }
        }
        PROF(4);
        // ---- canonical keys + changed flags out
        for (int q = tid; q < ncell * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            P.keys[(int64_t)S.bidx[c] * KW + w] = S.key[c][w];
        }
        if (tid < ncell) P.changed[S.bidx[tid]] = S.changed[tid];
        // canonical insert + frontier (k_canon_frontier's work): another CTA's inserter may compare
        // against this tile's key rows as soon as a slot marker is published, so they are made
        // visible device-wide first; the per-cell values are read before the barrier (the next
        // tile's gather rewrites them)
        int32_t cf_b = 0, cf_ch = 0;
        if (P.canon_fused) {
            bool anych = false;   // only a changed key is inserted (and read by other CTAs)
            for (int c = 0; c < ncell; c++) anych |= S.changed[c] != 0;
            if (anych) __threadfence();
            if (tid < ncell) { cf_b = S.bidx[tid]; cf_ch = S.changed[tid]; }
        }
        bar_sync(1, NCT);
        if (P.canon_fused && tid < ncell)
            canon_frontier_one(P.H, P.keys, cf_ch, P.batch_pool[cf_b], cf_b, P.rank, P.world, P.outbox, P.n_out,
                               P.canon_pos, P.status2, P.slot2, P.canon_pool, P.ckey_hint, P.f_items, P.f_pool,
                               const_cast<unsigned long long*>(P.ctr), P.max_cells);
        PROF(5);
        if (P.near_fused) {
            // ---- near lists of the tile's cells (the face solver's k_near), while their rows are
            // in L2: warp per cell, the same warp that wrote the cell's face plane
            for (int c = warp; c < ncell; c += NCW) {
                const int64_t b = S.bidx[c];
                Ctx cx;
                cx.Z = Zc + b * P.zs * 4;
                cx.faces = P.faces + b * 4;
                cx.key = S.key[c];
                cx.NB = P.NB; cx.M = 1; cx.branch = 0; cx.ensemble = 0; cx.K = P.NB + 1 + 6;
                for (int k = 0; k < 3; k++) { cx.lo[k] = P.lo[k]; cx.hi[k] = P.hi[k]; }
                const NearOut o{P.near_n, P.near_flags, P.near_id, P.near_row, P.near_cap};
                bool heavy = false;
                near_list<false>(cx, reinterpret_cast<const double4*>(P.ckey_hint)[b], P.tol_cell, P.tol_onplane,
                                 P.probe_delta, P.near_reach, o, b, heavy);
            }
            bar_sync(1, NCT);
            PROF(9);
        }
        if (prof) atomicAdd(&P.prof[7], 1ull);
    }
#undef PROF
}

// cells per tile for a wave of n cells: the widest tile that still gives every CTA slot work
__device__ __forceinline__ int tile_cells(int64_t n, const NarrowCompose& P, int grid) {
    if (P.tile_cells) return P.tile_cells;
    if (n >= (int64_t)grid * P.thr8) return 8;
    if (n >= (int64_t)grid * P.thr4) return 4;
    return 2;
}

template <int FP32>
__global__ void __launch_bounds__(NT, CPS) k_compose_narrow(const __grid_constant__ NarrowCompose P) {
    extern __shared__ uint8_t smem_raw[];
    NarrowSmem& S = *reinterpret_cast<NarrowSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ns = P.nsteps;

    if (tid == 0) {   // one thread initialises every barrier, then makes the inits visible to the async proxy
        for (int i = 0; i < NSB; i++) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < NACT * NR * AS; i += NT) (&S.act[0][0])[i] = 0.0;
    if (tid < NR / 32) S.deg1[tid] = 0u;
    __syncthreads();
    {   // constants of step 0 and the head (weights: not produced by the preceding kernels)
        const StepDev& s0 = P.st[0];
        for (int r = tid; r < s0.n_out; r += NT) {
            const double* w = s0.W + (int64_t)r * s0.ldw;
            const double a0 = prec_round(w[0], FP32), a1 = prec_round(w[1], FP32), a2 = prec_round(w[2], FP32);
            S.p1[r * 4 + 0] = a0; S.p1[r * 4 + 1] = a1; S.p1[r * 4 + 2] = a2;
            S.p1[r * 4 + 3] = s0.b ? prec_round(0.0 + s0.b[r], FP32) : 0.0;
            if (degenerate3(a0, a1, a2)) atomicOr(&S.deg1[r >> 5], 1u << (r & 31));
        }
        const SubDev* sd = P.subs;
        for (int r = tid; r < sd->last_n; r += NT) S.hw[r] = sd->hw[r];
    }
    __syncthreads();

    // boxes per tile: every GEMM step's K extent in 16-wide boxes
    int tile_boxes = 0;
    for (int s = 1; s < ns; s++) tile_boxes += (P.st[s].n_in + KB - 1) / KB;

    if (warp == NCW) {
        // ---------------------------------------------------------------- producer warp
        if (lane != 0) return;
        for (int s = 1; s < ns; s++) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tm[s])) : "memory");
        // the weights are not produced by the preceding kernels: the first boxes are requested
        // before the grid-dependency wait
        uint32_t g = 0;
        auto issue = [&](int s, int b) {
            const int slot = g % NSB;
            if (g >= NSB) mbar_wait(&S.empty[slot], ((g / NSB) - 1) & 1);
            mbar_expect_tx(&S.full[slot], NR * KB * sizeof(double));
            tma_load_2d(S.w[slot], &P.tm[s], &S.full[slot], b * KB, 0);
            g++;
        };
        int ps = 1, pb = 0;   // next (step, box) of the first tile
        const int pre = (P.dbg & 1) ? 0 : (NSB < tile_boxes ? NSB : tile_boxes);
        for (int i = 0; i < pre; i++) {
            issue(ps, pb);
            if (++pb == (P.st[ps].n_in + KB - 1) / KB) { pb = 0; ps++; }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        const int64_t n = dev_count(P.n_dev, P.n_cap);
        const int nc = tile_cells(n, P, gridDim.x);
        Tiling T;
        T.init(P, n, nc);
        const int64_t ntiles = T.ntiles;
        if ((int64_t)blockIdx.x >= ntiles) {
            // no tile for this CTA: let the prefetched boxes land before exiting
            for (uint32_t i = 0; i < g; i++) mbar_wait(&S.full[i % NSB], (i / NSB) & 1);
            return;
        }
        // a first tile that starts past step 1 (prefix reuse) does not use the prefetched boxes:
        // the consumers drain them and the tile's own sequence follows
        int f0, nc0;
        long long pos0;
        T.locate(blockIdx.x, nc, f0, pos0, nc0);
        bool first = f0 == 0;
        for (int64_t k = 0; k * gridDim.x < ntiles; k++) {
            const int64_t t = tile_of(P, k);
            if (t >= ntiles) continue;
            int f, ncell;
            long long pos;
            T.locate(t, nc, f, pos, ncell);
            for (int s = f + 1; s < ns; s++) {
                const int nb = (P.st[s].n_in + KB - 1) / KB;
                for (int b = 0; b < nb; b++) {
                    if (first && (s < ps || (s == ps && b < pb))) continue;   // prefetched
                    issue(s, b);
                }
            }
            first = false;
        }
        return;
    }

    // -------------------------------------------------------------------- consumers
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t n = dev_count(P.n_dev, P.n_cap);
    uint32_t gbox = 0;
    const bool prof = (P.dbg & 8) && P.prof && threadIdx.x == 0;
    unsigned long long tprev = prof ? clock64() : 0;
    const int nc = tile_cells(n, P, gridDim.x);
    double* Zc = P.Z;
    const double* Zp = P.Z;
    if (P.prefix) {
        const unsigned long long par = P.ctr[C_ITER] & 1ull;
        Zc = P.Z + (int64_t)par * P.zstride;
        Zp = P.Z + (int64_t)(par ^ 1ull) * P.zstride;
        Tiling T;
        T.init(P, n, nc);
        int f0, nc0;
        long long pos0;
        T.locate(blockIdx.x, nc, f0, pos0, nc0);
        if ((int64_t)blockIdx.x < T.ntiles && f0 > 0) {   // drain the prefetched boxes (see the producer)
            const uint32_t pre = (P.dbg & 1) ? 0u : (uint32_t)(NSB < tile_boxes ? NSB : tile_boxes);
            for (; gbox < pre; gbox++) {
                mbar_wait(&S.full[gbox % NSB], (gbox / NSB) & 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[gbox % NSB]);
            }
        }
    }
    if (nc == 8) consume<FP32, 2, 2>(S, P, n, gbox, prof, tprev, Zc, Zp);
    else if (nc == 4) consume<FP32, 1, 2>(S, P, n, gbox, prof, tprev, Zc, Zp);
    else consume<FP32, 1, 1>(S, P, n, gbox, prof, tprev, Zc, Zp);
}

// debug (AM_NARROW_CHECK=1): compare the fused kernel's outputs with the per-step path's
__global__ void k_narrow_check(const double* Z, const double* Z2, const double* F, const double* F2,
                               const uint64_t* K, const uint64_t* K2, const int32_t* ch, const int32_t* ch2,
                               const unsigned long long* n_dev, int64_t n_cap, int NB, int zs, int KW,
                               unsigned long long* dbg) {
    pdl_enter();
    const int64_t n = dev_count(n_dev, n_cap);
    const int64_t total = n * NB * 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t item = i / (NB * 4);
        const int rem = (int)(i - item * NB * 4);
        const int64_t off = item * zs * 4 + rem;
        if (__double_as_longlong(Z[off]) != __double_as_longlong(Z2[off])) {
            atomicAdd(&dbg[56], 1ull);
            if (atomicCAS(&dbg[60], 0ull, 1ull) == 0ull) {
                dbg[61] = (unsigned long long)item;
                dbg[62] = (unsigned long long)rem;
                dbg[63] = (unsigned long long)__double_as_longlong(Z[off] - Z2[off]);
            }
        }
        if (rem < 4 && __double_as_longlong(F[item * 4 + rem]) != __double_as_longlong(F2[item * 4 + rem]))
            atomicAdd(&dbg[57], 1ull);
        if (rem < KW && K[item * KW + rem] != K2[item * KW + rem]) atomicAdd(&dbg[58], 1ull);
        if (rem == 0 && (ch[item] != 0) != (ch2[item] != 0)) atomicAdd(&dbg[59], 1ull);
    }
}

}  // namespace

void launch_narrow_check(const double* Z, const double* Z2, const double* F, const double* F2, const uint64_t* K,
                         const uint64_t* K2, const int32_t* ch, const int32_t* ch2, const unsigned long long* n_dev,
                         int64_t n_cap, int NB, int zs, int KW, unsigned long long* dbg, cudaStream_t s) {
    launch_k(k_narrow_check, 148 * 8, 256, 0, s, Z, Z2, F, F2, K, K2, ch, ch2, n_dev, n_cap, NB, zs, KW, dbg);
}

bool narrow_compose_ok(const StepDev* st, int nsteps, int n_subs, int KW) {
    if (n_subs != 1 || nsteps < 2 || nsteps > kMaxNarrowSteps || KW > KWMAX) return false;
    if (!(st[0].flags & AM_STEP_FIRST) || st[0].n_in != 3) return false;
    for (int s = 0; s < nsteps; s++) {
        const int f = st[s].flags & ~AM_STEP_FIRST;
        if (f != 0 || st[s].n_out > NR || st[s].V || st[s].vb || st[s].vb_shape) return false;
        if (s > 0 && ((st[s].flags & AM_STEP_FIRST) || st[s].n_in != st[s - 1].n_out ||
                      st[s].in_row_off != st[s - 1].row_off))
            return false;
    }
    return true;
}

// ---------------------------------------------------------------------------------------
// Point forward of the same narrow networks in one launch (the trigger's samples, bisection
// midpoints, seed refinement and the BFS's exact probe evaluations): a CTA walks tiles of 32
// points (32 columns) through every layer with the activations in shared memory, W streamed by
// the same producer-warp TMA ring.  Per element the arithmetic is the per-layer path's
// (k_input_step<1> / k_gemm_step<1, 64> / k_forward_head: DMMA accumulation in the same K order,
// + bias, relu by the sign bit, the head's lane-strided sums and shuffle tree), so values and
// state bits agree bit for bit with it.
constexpr int FP = 32;   // points per tile
struct __align__(1024) ForwardSmem {
    double w[NSB][NR * KB];
    double act[2][NR * AS];
    double x[FP][3];
    uint64_t key[FP][KWMAX];
    double hw[NR];
    uint64_t full[NSB], empty[NSB];
};

template <int FP32>
__global__ void __launch_bounds__(NT, CPS) k_forward_narrow(const __grid_constant__ NarrowCompose P,
                                                            const __grid_constant__ ForwardArgs F) {
    extern __shared__ uint8_t smem_raw[];
    ForwardSmem& S = *reinterpret_cast<ForwardSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ns = P.nsteps, KW = P.KW;
    if (tid == 0) {
        for (int i = 0; i < NSB; i++) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 2 * NR * AS; i += NT) (&S.act[0][0])[i] = 0.0;
    for (int r = tid; r < P.subs->last_n; r += NT) S.hw[r] = P.subs->hw[r];
    __syncthreads();
    int tile_boxes = 0;
    for (int s = 1; s < ns; s++) tile_boxes += (P.st[s].n_in + KB - 1) / KB;

    if (warp == NCW) {   // producer: every tile streams the W boxes of steps 1..ns-1
        if (lane != 0) return;
        uint32_t g = 0;
        auto issue = [&](int s, int b) {
            const int slot = g % NSB;
            if (g >= NSB) mbar_wait(&S.empty[slot], ((g / NSB) - 1) & 1);
            mbar_expect_tx(&S.full[slot], NR * KB * sizeof(double));
            tma_load_2d(S.w[slot], &P.tm[s], &S.full[slot], b * KB, 0);
            g++;
        };
        int ps = 1, pb = 0;
        const int pre = NSB < tile_boxes ? NSB : tile_boxes;
        for (int i = 0; i < pre; i++) {
            issue(ps, pb);
            if (++pb == (P.st[ps].n_in + KB - 1) / KB) { pb = 0; ps++; }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        const int64_t n = dev_count(F.n_dev, F.n_cap);
        const int64_t ntiles = (n + FP - 1) / FP;
        if ((int64_t)blockIdx.x >= ntiles) {
            for (uint32_t i = 0; i < g; i++) mbar_wait(&S.full[i % NSB], (i / NSB) & 1);
            return;
        }
        bool first = true;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 1; s < ns; s++) {
                const int nb = (P.st[s].n_in + KB - 1) / KB;
                for (int b = 0; b < nb; b++) {
                    if (first && (s < ps || (s == ps && b < pb))) continue;
                    issue(s, b);
                }
            }
            first = false;
        }
        return;
    }

    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t n = dev_count(F.n_dev, F.n_cap);
    const int64_t ntiles = (n + FP - 1) / FP;
    constexpr int MI = 2, NJ = 2, WR = 3, RB = 32, CB = 16;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = warp % WR, wn = warp / WR;
    const int pg = ((g & 3) << 1) | (g >> 2);
    uint32_t gbox = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t p0 = t * FP;
        const int np = (int)(n - p0 < FP ? n - p0 : FP);
        // ---- points and key rows (the shape word, if any, comes with the zeroed keys)
        for (int q = tid; q < FP * 3; q += NCT) {
            const int c = q / 3;
            S.x[c][q - c * 3] = c < np ? F.pts[(p0 + c) * 3 + (q - c * 3)] : 0.0;
        }
        for (int q = tid; q < FP * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            S.key[c][w] = (c < np && w == P.shape_w) ? F.keys[(p0 + c) * KW + w] : 0ull;
        }
        bar_sync(1, NCT);
        // ---- step 0 (k_input_step<1>'s input_elem): pre = x . W_1[r] + b_1[r]
        {
            const StepDev& st = P.st[0];
            for (int idx = tid; idx < np * st.n_out; idx += NCT) {
                const int c = idx / st.n_out, r = idx - c * st.n_out;
                const double* w = st.W + (int64_t)r * st.ldw;
                const double acc = (S.x[c][0] * w[0] + S.x[c][1] * w[1]) + S.x[c][2] * w[2];
                const double pre = prec_round(acc + step_bias(st, item_shape(S.key[c], P.shape_w), r), FP32);
                const int row = st.row_off + r;
                if (pre > 0.0) atomicOr(reinterpret_cast<unsigned long long*>(&S.key[c][row >> 6]), key_mask(row));
                S.act[0][r * AS + c] = pre > 0.0 ? pre : 0.0;
            }
            bar_sync(1, NCT);
        }
        int cur = 0;
        for (int s = 1; s < ns; s++) {
            const StepDev& st = P.st[s];
            const int nb = (st.n_in + KB - 1) / KB;
            double acc[MI][NJ][4];
#pragma unroll
            for (int i = 0; i < MI; i++)
#pragma unroll
                for (int j = 0; j < NJ; j++)
#pragma unroll
                    for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;
            const double* xs = S.act[cur];
            for (int b = 0; b < nb; b++, gbox++) {
                const int slot = gbox % NSB;
                mbar_wait(&S.full[slot], (gbox / NSB) & 1);
                const double* ws = S.w[slot];
#pragma unroll
                for (int kk = 0; kk < KB; kk += 4) {
                    double a[MI][2], bf[NJ];
#pragma unroll
                    for (int mi = 0; mi < MI; mi++) {
                        const int r = wm * RB + mi * 16 + pg;
                        a[mi][0] = ws[swz(r, kk + tq)];
                        a[mi][1] = ws[swz(r + 8, kk + tq)];
                    }
                    const int k = b * KB + kk + tq;
#pragma unroll
                    for (int nj = 0; nj < NJ; nj++) bf[nj] = xs[k * AS + wn * CB + nj * 8 + g];
#pragma unroll
                    for (int mi = 0; mi < MI; mi++)
#pragma unroll
                        for (int nj = 0; nj < NJ; nj++) dmma_16x8x4(acc[mi][nj], a[mi][0], a[mi][1], bf[nj]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[slot]);
            }
            double* xo = S.act[cur ^ 1];
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const int r = wm * RB + mi * 16 + pg + half * 8;
                    if (r >= st.n_out) continue;
                    const int row = st.row_off + r;
#pragma unroll
                    for (int nj = 0; nj < NJ; nj++)
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const int c = wn * CB + nj * 8 + 2 * tq + e;
                            if (c >= np) continue;
                            const double pre = prec_round(
                                acc[mi][nj][half * 2 + e] + step_bias(st, item_shape(S.key[c], P.shape_w), r), FP32);
                            if (pre > 0.0)
                                atomicOr(reinterpret_cast<unsigned long long*>(&S.key[c][row >> 6]), key_mask(row));
                            xo[r * AS + c] = pre > 0.0 ? pre : 0.0;
                        }
                }
            bar_sync(1, NCT);
            cur ^= 1;
        }
        // ---- head (k_forward_head): per point, lane-strided sums over the active rows + tree
        const SubDev sd = *P.subs;
        for (int c = warp; c < np; c += NCW) {
            double a = 0.0;
            for (int r = lane; r < sd.last_n; r += 32) {
                const int row = sd.last_row + r;
                if ((S.key[c][row >> 6] >> (63 - (row & 63))) & 1ull) a += S.act[cur][r * AS + c] * S.hw[r];
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0 && F.vals) F.vals[p0 + c] = prec_round(a + head_bias(sd, item_shape(S.key[c], P.shape_w)), FP32);
        }
        for (int q = tid; q < np * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            F.keys[(p0 + c) * KW + w] = S.key[c][w];
        }
        bar_sync(1, NCT);
    }
}

void launch_forward_narrow(const NarrowCompose& P, const ForwardArgs& F, cudaStream_t s) {
    if (F.n_cap <= 0) return;
    const int64_t tiles = (F.n_cap + FP - 1) / FP;
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t grid = std::min<int64_t>(tiles, (int64_t)device_sms() * CPS);
    const size_t smem = sizeof(ForwardSmem) + 1024;
    static bool init[64] = {};
    if (dev < 64 && !init[dev]) {
        cudaFuncSetAttribute(k_forward_narrow<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_forward_narrow<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        init[dev] = true;
    }
    if (P.fp32) launch_k(k_forward_narrow<1>, (unsigned)grid, NT, smem, s, P, F);
    else launch_k(k_forward_narrow<0>, (unsigned)grid, NT, smem, s, P, F);
}

void launch_compose_narrow(const NarrowCompose& P, cudaStream_t s) {
    if (P.n_cap <= 0) return;
    const int64_t tiles = (P.n_cap + NCELL - 1) / NCELL;
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = device_sms();
    const int64_t grid = (P.dbg & 4) ? tiles : std::min<int64_t>(tiles, (int64_t)sms * CPS);
    const size_t smem = sizeof(NarrowSmem) + 1024;
    // per device: the attribute is a property of the function on the current device
    static bool init[64] = {};
    if (dev < 64 && !init[dev]) {
        cudaFuncSetAttribute(k_compose_narrow<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_compose_narrow<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        init[dev] = true;
    }
    if (P.fp32) launch_k(k_compose_narrow<1>, (unsigned)grid, NT, smem, s, P);
    else launch_k(k_compose_narrow<0>, (unsigned)grid, NT, smem, s, P);
}

}  // namespace am
