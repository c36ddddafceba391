// am_shard.cu -- device side of the sharded (multi-GPU) march's frontier exchange.
//
// States are owned by key_owner(state) = (hash(state) >> 7) % world.  During a round each rank
// marches its own queue; emitted / canonical states owned elsewhere accumulate in the outbox
// (k_route_emitted / k_route_changed).  Between rounds the outbox is exchanged with ONE
// fixed-size all-to-all whose blocks carry their own count header, so the host never needs the
// counts to size the collective:
//
//   send / recv  [world][rows][KW] uint64, rows = hdr_rows + cap; block r of send goes to rank r
//   header       kHdrWords words at the start of each block:
//                  [0] keys in this block            [1] sender's outstanding work
//                  [2] sender's outbox rest           [3] keys the sender sent in total
//                  [4] sender's largest per-rank demand  [5] sender's visited cells
//                  [6] sender capped                   [7] 1 (valid)
//
// k_shard_scatter moves up to `cap` outbox keys per destination into its block (atomic slot per
// key; order inside a block is irrelevant -- the visited set does not depend on processing
// order) and the overflow into `rest`, which k_shard_copyback returns to the outbox for the
// next round, so no key is ever dropped whatever `cap` is.  k_shard_header fills the headers;
// every rank receives every sender's header, so all ranks take identical decisions (the
// capacity of the next exchange, termination) from the same numbers.
#include "am_internal.h"

namespace am {

namespace {

__global__ void k_shard_scatter(const uint64_t* outbox, const unsigned long long* n_out, int KW, int world,
                                int64_t cap, int hdr_rows, uint64_t* send, uint64_t* rest,
                                unsigned long long* cnt) {
    pdl_enter();
    const int64_t n = (int64_t)*n_out;
    const int64_t rows = hdr_rows + cap;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t* k = outbox + i * KW;
        const int o = key_owner(k, KW, world);
        const unsigned long long pos = atomicAdd(&cnt[o], 1ull);
        uint64_t* dst;
        if ((int64_t)pos < cap) {
            dst = send + ((int64_t)o * rows + hdr_rows + (int64_t)pos) * KW;
        } else {
            dst = rest + (int64_t)atomicAdd(&cnt[world], 1ull) * KW;
        }
        for (int w = 0; w < KW; w++) dst[w] = k[w];
    }
}

__global__ void k_shard_header(unsigned long long* ctr, int KW, int world, int64_t cap, int hdr_rows,
                               uint64_t* send, const unsigned long long* cnt) {
    pdl_enter();
    if (threadIdx.x != 0) return;
    const int64_t rows = hdr_rows + cap;
    unsigned long long sent = 0, demand = 0;
    for (int o = 0; o < world; o++) {
        const unsigned long long c = cnt[o];
        sent += c < (unsigned long long)cap ? c : (unsigned long long)cap;
        demand = c > demand ? c : demand;
    }
    const unsigned long long nrest = cnt[world];
    const unsigned long long outstanding = (ctr[C_QTAIL] - ctr[C_QHEAD]) + ctr[C_NPEND] + ctr[C_NPROBE];
    for (int o = 0; o < world; o++) {
        uint64_t* h = send + (int64_t)o * rows * KW;
        const unsigned long long c = cnt[o];
        h[0] = c < (unsigned long long)cap ? c : (unsigned long long)cap;
        h[1] = outstanding;
        h[2] = nrest;
        h[3] = sent;
        h[4] = demand;
        h[5] = ctr[C_TOTAL];
        h[6] = ctr[C_CAPPED];
        h[7] = 1;
    }
    ctr[C_NOUT] = nrest;   // the rest goes back into the outbox (k_shard_copyback)
}

__global__ void k_shard_copyback(const unsigned long long* ctr, int KW, const uint64_t* rest, uint64_t* outbox) {
    pdl_enter();
    const int64_t n = (int64_t)ctr[C_NOUT] * KW;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        outbox[i] = rest[i];
}

// flat row indices (into recv) of every received key
__global__ void k_shard_index(const uint64_t* recv, int KW, int world, int64_t cap, int hdr_rows, int32_t* idx,
                              unsigned long long* n) {
    pdl_enter();
    const int64_t rows = hdr_rows + cap;
    for (int s = blockIdx.y; s < world; s += gridDim.y) {
        const uint64_t* h = recv + (int64_t)s * rows * KW;
        const int64_t c = h[7] == 1 ? (int64_t)(h[0] < (uint64_t)cap ? h[0] : (uint64_t)cap) : 0;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x)
            idx[atomicAdd(n, 1ull)] = (int32_t)((int64_t)s * rows + hdr_rows + i);
    }
}

}  // namespace

void launch_shard_pack(uint64_t* outbox, unsigned long long* ctr, int KW, int world, int64_t cap,
                       int hdr_rows, uint64_t* send, uint64_t* rest, unsigned long long* cnt, int64_t max_keys,
                       cudaStream_t s) {
    cudaMemsetAsync(cnt, 0, (world + 1) * sizeof(unsigned long long), s);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((max_keys + 255) / 256, (int64_t)device_sms() * 8));
    launch_k(k_shard_scatter, (unsigned)blocks, 256, 0, s, (const uint64_t*)outbox,
             (const unsigned long long*)(ctr + C_NOUT), KW, world, cap, hdr_rows, send, rest, cnt);
    launch_k(k_shard_header, 1, 32, 0, s, ctr, KW, world, cap, hdr_rows, send, (const unsigned long long*)cnt);
    launch_k(k_shard_copyback, (unsigned)blocks, 256, 0, s, (const unsigned long long*)ctr, KW,
             (const uint64_t*)rest, outbox);
}

void launch_shard_index(const uint64_t* recv, int KW, int world, int64_t cap, int hdr_rows, int32_t* idx,
                        unsigned long long* n, cudaStream_t s) {
    cudaMemsetAsync(n, 0, sizeof(unsigned long long), s);
    const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 64));
    launch_k(k_shard_index, dim3(bx, (unsigned)std::min(world, 64)), dim3(256), 0, s, recv, KW, world, cap,
             hdr_rows, idx, n);
}

}  // namespace am
