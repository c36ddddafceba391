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
// so a BFS iteration's gather + L + 1 launches become one.  6 consumer warps (3 x 2 warp tiles
// of 32 x 16) + 1 producer warp, ~107 KB shared memory, 2 CTAs per SM.  Arithmetic per output
// element is the same as k_gemm_step's (DMMA accumulation over K, then + bias), so the two
// paths agree to the last bit on the same K order; parity is checked against the oracle.
#include <algorithm>

#include "am_internal.h"
#include "am_ptx.cuh"

namespace am {

namespace {

constexpr int NR = 96;          // max rows (layer width) of the tile
constexpr int NCELL = 8;        // cells per tile
constexpr int NCOL = NCELL * 4; // columns
constexpr int AS = NCOL + 4;    // act row stride (doubles): conflict-free B fragments
constexpr int KB = 16;          // K per W box (128 B rows)
constexpr int NSB = 4;          // W ring boxes
constexpr int NCW = 6;          // consumer warps
constexpr int NCT = NCW * 32;   // consumer threads
constexpr int NT = NCT + 32;    // + producer warp
constexpr int KWMAX = 40;       // key words per cell held in shared memory

struct __align__(1024) NarrowSmem {
    double w[NSB][NR * KB];       // TMA destinations (1 KB aligned for the 128B swizzle)
    double act[2][NR * AS];       // masked layer outputs [row][col], ping-pong
    uint64_t key[NCELL][KWMAX];   // the tile's state keys (canonical bits updated in place)
    uint64_t full[NSB], empty[NSB];
    int changed[NCELL];
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

__global__ void __launch_bounds__(NT, 2) k_compose_narrow(const __grid_constant__ NarrowCompose P) {
    extern __shared__ uint8_t smem_raw[];
    NarrowSmem& S = *reinterpret_cast<NarrowSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ns = P.nsteps;
    const int KW = P.KW;

    if (tid == 0) {   // one thread initialises every barrier, then makes the inits visible to the async proxy
        for (int i = 0; i < NSB; i++) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 2 * NR * AS; i += NT) (&S.act[0][0])[i] = 0.0;
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
        const int64_t ntiles = (n + NCELL - 1) / NCELL;
        if ((int64_t)blockIdx.x >= ntiles) {
            // no tile for this CTA: let the prefetched boxes land before exiting
            for (uint32_t i = 0; i < g; i++) mbar_wait(&S.full[i % NSB], (i / NSB) & 1);
            return;
        }
        bool first = true;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 1; s < ns; s++) {
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
    const unsigned long long* ctr = P.ctr;
    const int64_t n = dev_count(P.n_dev, P.n_cap);
    const int64_t ntiles = (n + NCELL - 1) / NCELL;
    const int64_t head0 = (int64_t)ctr[C_QHEAD] - n;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = warp % 3, wn = warp / 3;
    const int pg = ((g & 3) << 1) | (g >> 2);   // fragment row permutation (bank-conflict-free W reads)
    const int fp32 = P.fp32;
    uint32_t gbox = 0;

    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t item0 = t * NCELL;
        const int ncell = (int)(n - item0 < NCELL ? n - item0 : NCELL);
        // ---- gather (reference order: the BFS queue slice k_take dequeued)
        for (int q = tid; q < NCELL * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            uint64_t v = 0;
            if (c < ncell) {
                const int32_t p = P.queue[head0 + item0 + c];
                v = P.pool[(int64_t)p * KW + w];
                if (w == 0) {
                    P.batch_pool[item0 + c] = p;
                    P.canon_pos[item0 + c] = -1;
                    reinterpret_cast<double4*>(P.ckey_hint)[item0 + c] = reinterpret_cast<const double4*>(P.pool_hint)[p];
                }
            }
            S.key[c][w] = v;
        }
        if (tid < NCELL) S.changed[tid] = 0;
        bar_sync(1, NCT);

        // ---- step 0: A_1 = W_1[:, :3], c_1 = b_1 (reference network.py:398-443 with A = I, c = 0)
        {
            const StepDev& st = P.st[0];
            const int no = st.n_out;
            for (int idx = tid; idx < ncell * no; idx += NCT) {
                const int c = idx / no, r = idx - c * no;
                const int64_t item = item0 + c;
                uint64_t* key = S.key[c];
                const int row = st.row_off + r;
                const double* w = st.W + (int64_t)r * st.ldw;
                double a0 = w[0], a1 = w[1], a2 = w[2];
                double cc = 0.0;
                cc = cc + step_bias(st, item_shape(key, P.shape_w), r);
                a0 = prec_round(a0, fp32); a1 = prec_round(a1, fp32);
                a2 = prec_round(a2, fp32); cc = prec_round(cc, fp32);
                const double nrm = sqrt((a0 * a0 + a1 * a1) + a2 * a2);
                int bit = skey_bit(key, row);
                if (!(nrm > kDegen)) {
                    const int cb = cc > 0.0;
                    if (cb != bit) { skey_set(key, row, cb); S.changed[c] = 1; bit = cb; }
                }
                double* z = P.Z + (item * P.zs + row) * 4;
                reinterpret_cast<double2*>(z)[0] = make_double2(a0, a1);
                reinterpret_cast<double2*>(z)[1] = make_double2(a2, cc);
                double* ao = &S.act[0][r * AS + c * 4];
                reinterpret_cast<double2*>(ao)[0] = bit ? make_double2(a0, a1) : make_double2(0.0, 0.0);
                reinterpret_cast<double2*>(ao)[1] = bit ? make_double2(a2, cc) : make_double2(0.0, 0.0);
            }
            bar_sync(1, NCT);
        }

        // ---- GEMM steps
        int cur = 0;
        for (int s = 1; s < ns; s++) {
            const StepDev& st = P.st[s];
            const int nb = (st.n_in + KB - 1) / KB;
            double acc[2][2][4];
#pragma unroll
            for (int i = 0; i < 2; i++)
#pragma unroll
                for (int j = 0; j < 2; j++)
#pragma unroll
                    for (int e = 0; e < 4; e++) acc[i][j][e] = 0.0;
            const double* xs = S.act[cur];
            for (int b = 0; b < nb; b++, gbox++) {
                const int slot = gbox % NSB;
                mbar_wait(&S.full[slot], (gbox / NSB) & 1);
                const double* ws = S.w[slot];
#pragma unroll
                for (int kk = 0; kk < KB; kk += 4) {
                    double a[2][2], bf[2];
#pragma unroll
                    for (int mi = 0; mi < 2; mi++) {
                        const int r = wm * 32 + mi * 16 + pg;
                        a[mi][0] = ws[swz(r, kk + tq)];
                        a[mi][1] = ws[swz(r + 8, kk + tq)];
                    }
                    const int k = b * KB + kk + tq;
#pragma unroll
                    for (int nj = 0; nj < 2; nj++) bf[nj] = xs[k * AS + wn * 16 + nj * 8 + g];
#pragma unroll
                    for (int mi = 0; mi < 2; mi++)
#pragma unroll
                        for (int nj = 0; nj < 2; nj++) dmma_16x8x4(acc[mi][nj], a[mi][0], a[mi][1], bf[nj]);
                }
                // release the slot: the generic-proxy reads of this box must be ordered before the
                // TMA (async proxy) that will overwrite it -- without the proxy fence a refill was
                // observed to land under the last k-step's fragment loads (rare corrupted tiles)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[slot]);
            }
            // epilogue
            double* xo = S.act[cur ^ 1];
#pragma unroll
            for (int mi = 0; mi < 2; mi++) {
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const int r = wm * 32 + mi * 16 + pg + half * 8;
                    const bool rok = r < st.n_out;
                    const int row = st.row_off + r;
#pragma unroll
                    for (int nj = 0; nj < 2; nj++) {
                        const int col = wn * 16 + nj * 8 + 2 * tq;
                        const int c = col >> 2, comp = col & 3;   // comp 0 or 2
                        const bool ok = rok && c < ncell;
                        double v0 = acc[mi][nj][half * 2], v1 = acc[mi][nj][half * 2 + 1];
                        if (comp == 2) v1 = v1 + (ok ? step_bias(st, item_shape(S.key[c], P.shape_w), r) : 0.0);
                        v0 = prec_round(v0, fp32);
                        v1 = prec_round(v1, fp32);
                        // the pair of lanes (tq, tq ^ 1) holds the 4 components of (cell, row)
                        const double p0 = __shfl_xor_sync(0xffffffffu, v0, 1);
                        const double p1 = __shfl_xor_sync(0xffffffffu, v1, 1);
                        if (ok) {
                            const double nx = comp == 0 ? v0 : p0, ny = comp == 0 ? v1 : p1;
                            const double nz = comp == 0 ? p0 : v0, cc = comp == 0 ? p1 : v1;
                            const double nrm = sqrt((nx * nx + ny * ny) + nz * nz);
                            int bit = skey_bit(S.key[c], row);
                            if (!(nrm > kDegen)) {
                                const int cb = cc > 0.0;
                                if (cb != bit) {
                                    if (comp == 0) { skey_set(S.key[c], row, cb); S.changed[c] = 1; }
                                    bit = cb;
                                }
                            }
                            *reinterpret_cast<double2*>(P.Z + ((item0 + c) * P.zs + row) * 4 + comp) = make_double2(v0, v1);
                            *reinterpret_cast<double2*>(xo + r * AS + col) = bit ? make_double2(v0, v1) : make_double2(0.0, 0.0);
                        }
                    }
                }
            }
            bar_sync(1, NCT);
            cur ^= 1;
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
                    double* f = P.faces + (item0 + c) * 4;
                    f[0] = prec_round(a0, fp32); f[1] = prec_round(a1, fp32); f[2] = prec_round(a2, fp32);
                    f[3] = prec_round(a3 + head_bias(sd, item_shape(S.key[c], P.shape_w)), fp32);
                }
            }
        }
        // ---- canonical keys + changed flags out
        for (int q = tid; q < ncell * KW; q += NCT) {
            const int c = q / KW, w = q - c * KW;
            P.keys[(item0 + c) * KW + w] = S.key[c][w];
        }
        if (tid < ncell) P.changed[item0 + tid] = S.changed[tid];
        bar_sync(1, NCT);
    }
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

void launch_compose_narrow(const NarrowCompose& P, cudaStream_t s) {
    if (P.n_cap <= 0) return;
    const int64_t tiles = (P.n_cap + NCELL - 1) / NCELL;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = (P.dbg & 4) ? tiles : std::min<int64_t>(tiles, (int64_t)sms * 2);
    const size_t smem = sizeof(NarrowSmem) + 1024;
    // per device: the attribute is a property of the function on the current device
    static bool init[64] = {};
    if (dev < 64 && !init[dev]) {
        cudaFuncSetAttribute(k_compose_narrow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        init[dev] = true;
    }
    launch_k(k_compose_narrow, (unsigned)grid, NT, smem, s, P);
}

}  // namespace am
