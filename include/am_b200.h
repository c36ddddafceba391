/*
 * am_b200.h -- C-ABI of the B200 analytic-marching engine (libam_b200.so).
 *
 * The reference (exactmesh, pure Python) exposes the meshing path as
 *     march(net, MarchConfig) -> MarchResult          reference marching.py:304
 * built from per-cell primitives
 *     state_at / forward_many                          reference network.py:352-392
 *     affine_maps (+ canonical state)                  reference network.py:446-489
 *     build_cell + extract_face_{pivot,naive}          reference cells.py:127-462
 *     neighbor transitions + probes                    reference marching.py:152-288
 * The entry points below replace exactly that path; a ctypes binding of them
 * is shown in INTEGRATION.md.  All buffers are plain pointers + sizes; device
 * pointers are marked d_, host pointers h_.  Every function returns 0 on
 * success or a negative AM_ERR_* code (am_last_error() has the message).
 *
 * State keys: n_bits activation bits packed MSB-first into uint64 words
 * (bit i -> word i/64, bit 63 - i%64), so big-endian bytes of the words are
 * exactly the reference's np.packbits key (reference network.py:222); max-pool
 * ensembles append one word holding the branch index.
 */
#ifndef AM_B200_H
#define AM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AM_OK 0
#define AM_ERR_ARG (-1)
#define AM_ERR_CUDA (-2)
#define AM_ERR_CAPACITY (-3)
#define AM_ERR_NO_DEVICE (-4)
#define AM_ERR_OVERFLOW (-5)

/* network step flags (one step = one hidden layer of ReLU neurons) */
#define AM_STEP_SAVE_INPUT 1       /* this step's input is a residual block input */
#define AM_STEP_SHORTCUT_IDENT 2   /* add the saved block input (identity shortcut) */
#define AM_STEP_SHORTCUT_LINEAR 4  /* add V @ saved block input + shortcut bias */
#define AM_STEP_FIRST 8            /* input is the network input x */
#define AM_STEP_SC_FROM_INPUT 16   /* the saved block input is the network input x */

#define AM_STEP_FIELDS 12 /* n_in,n_out,w_off,b_off,flags,v_off,vb_off,row_off,in_row_off,sin_row_off,n_sin,sub */
#define AM_SUB_FIELDS 6   /* first_step,n_steps,head_w_off,head_b_off,row_begin,n_rows */

/* Flattened network: every hidden layer of every subnetwork, in StateVector
 * bit order.  params holds all fp64 weights (row-major W[n_out][n_in]). */
typedef struct {
    const double *h_params;
    int64_t n_params;
    const int64_t *h_steps; /* n_steps x AM_STEP_FIELDS */
    int32_t n_steps;
    const int64_t *h_subs;  /* n_subs x AM_SUB_FIELDS */
    int32_t n_subs;
    int32_t n_bits;         /* total hidden neurons N */
    int32_t ensemble;       /* 1: max-pool union of n_subs subnetworks */
} am_net_desc;

/* MarchConfig fields the GPU path consumes (reference marching.py:52-75) */
typedef struct {
    double bbox_lo[3], bbox_hi[3];
    double tol_cell;      /* 1e-9  cell membership slack      (reference cells.py:33) */
    double tol_weld;      /* 1e-7  vertex dedup radius        (reference cells.py:35) */
    double tol_onplane;   /* 1e-9  point-on-plane slack       (reference cells.py:34) */
    double probe_delta;   /* 1e-7  neighbour probe step       (reference marching.py:67) */
    int64_t max_cells;    /* visited-cell cap                 (reference marching.py:59) */
    int64_t batch_cells;  /* cells composed per batch (0 = size from mem_budget) */
    int64_t mem_budget;   /* bytes for per-batch buffers (0 = 4 GiB; 32 GiB when a cell composes >= 2 MFLOP) */
    int32_t rank, world;  /* state ownership: owner(state) = (hash(state) >> 7) % world */
    int32_t n_shapes;     /* > 1: batch of same-architecture shapes marched together (the key
                           * gains a trailing shape word; see am_engine_set_shape_params) */
    int32_t precision;    /* 0: fp64 (reference arithmetic); 1: fp32 mode -- weights and every
                           * composed affine map / field value rounded to fp32 (products of fp32
                           * operands are exact in the fp64 DMMA accumulation), faces solved from
                           * those fp32-precision planes; pair with the looser tolerances of the
                           * fp32-mode study */
} am_march_params;

typedef struct am_engine am_engine;

/* --- lifecycle ------------------------------------------------------------ */
const char *am_last_error(void);
int am_device_info(int device, int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor);
/* stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream) or 0 */
int am_engine_create(am_engine **out, const am_net_desc *net, const am_march_params *p, int device,
                     void *stream);
int am_engine_destroy(am_engine *e);
int am_engine_key_words(const am_engine *e);
int am_engine_reset(am_engine *e);                       /* clear visited set + results */
/* new weights for an engine of the same architecture (same step / sub tables and parameter
 * count, e.g. another latent code folded into the first layer, or a training checkpoint):
 * re-uploads the values; buffers, TMA descriptors and captured graphs are reused.
 * Replaces re-running the reference's network construction (network.py:131-216) per march. */
int am_engine_load_params(am_engine *e, const double *h_params, int64_t n_params);
/* Batch of shapes (n_shapes > 1): shape s uses the engine's parameters with the n_idx entries
 * h_param_idx[j] replaced by h_values[s * n_idx + j].  Every replaced entry must lie in a bias
 * vector (a layer bias, a shortcut bias or a head bias), so the shapes share every weight
 * matrix and one DMMA contraction serves all of them -- e.g. latent-conditioned decoders with
 * the code folded into the biases it enters (BASELINE configs[4]).  Each shape's march is the
 * reference march (marching.py:304-362) of its own network. */
int am_engine_set_shape_params(am_engine *e, const int64_t *h_param_idx, int64_t n_idx, const double *h_values);
/* shape of the points given to later am_forward / am_dichotomy / am_seed calls */
int am_engine_set_shape(am_engine *e, int32_t shape);

/* --- per-point primitives (replace forward_many / state_at / affine_maps) - */
/* F(x) and the activation state at n points (device buffers; keys may be NULL) */
int am_forward(am_engine *e, const double *d_pts, int64_t n, double *d_vals, uint64_t *d_keys);
/* the same for a batch-of-shapes engine with a per-point shape (device int32 [n]) */
int am_forward_shapes(am_engine *e, const double *d_pts, const int32_t *d_shapes, int64_t n, double *d_vals,
                      uint64_t *d_keys);
/* canonical state, raw neuron planes (n_bits x 4: nx,ny,nz,c) and face planes
 * (n_subs x 4) of n states; device buffers */
int am_affine_maps(am_engine *e, const uint64_t *d_keys, int64_t n, uint64_t *d_canon,
                   double *d_planes, double *d_faces);

/* --- marching (replace _Marcher, reference marching.py:216-301) ---------- */
/* seed points -> refined canonical seed states queued as candidates
 * (reference marching.py:201-213 _refine_seed_state, 322-324) */
int am_seed(am_engine *e, const double *d_pts, int64_t n);
int am_seed_shapes(am_engine *e, const double *d_pts, const int32_t *d_shapes, int64_t n);
/* batched bisection triggering between F>0 and F<0 samples (reference
 * seeding.py:84-112); writes n surface points to d_out */
int am_dichotomy(am_engine *e, const double *d_xpos, const double *d_xneg, int64_t n, double eps,
                 double seed_tol, int max_iters, double *d_out);
int am_dichotomy_shapes(am_engine *e, const double *d_xpos, const double *d_xneg, const int32_t *d_shapes,
                        int64_t n, double eps, double seed_tol, int max_iters, double *d_out);
/* iterative triggers from n start points (device, all in lockstep; reference seeding.py:35-77):
 * scheme 0 = sgd on |F| (param = initial step 0.05), 1 = sphere tracing (param = eta 1.0,
 * escape = 12 x the unit box), at most max_iters steps (1000 / 50).  d_out [n*3] final iterate,
 * d_status [n]: 1 converged, 2 diverged (sphere tracing; the reference raises), 3 not converged
 * (zero gradient / out of iterations); d_iters [n] iterations to convergence.  n <= the
 * engine's batch size. */
int am_trace(am_engine *e, const double *d_x0, int64_t n, int scheme, double seed_tol, int max_iters, double param,
             double escape, double *d_out, int32_t *d_status, int32_t *d_iters);
/* queue n raw candidate states (device keys) for the next absorb */
int am_push_candidates(am_engine *e, const uint64_t *d_keys, int64_t n);
/* one BFS iteration: dequeue up to a batch of states, compose them,
 * canonicalise, extract the faces of the new cells and enqueue every new
 * neighbour state (flips + probes).  *h_new_cells = cells visited. */
int am_wave(am_engine *e, int64_t *h_new_cells);
/* run waves until no candidates remain (single rank); *h_waves = waves run */
int am_run(am_engine *e, int64_t *h_waves);

/* --- sharded marching (owner = (hash >> 7) % world) ----------------------- */
/* with world > 1, states emitted by a wave that another rank owns are held in
 * an outbox instead of being inserted locally.  am_outbox_counts gives the
 * total; am_outbox_take moves them to d_out grouped by owner rank
 * (h_counts[world] per owner) and clears the outbox.  Received states are fed
 * back with am_push_candidates. */
int am_outbox_counts(am_engine *e, int64_t *h_total);
int am_outbox_take(am_engine *e, uint64_t *d_out, int64_t *h_counts);
/* states queued but not yet composed on this rank */
int am_queue_size(am_engine *e, int64_t *h_n);

/* Device-driven rounds (the multi-GPU march's loop; one host synchronisation per round).
 * A round is
 *   am_shard_iterate(e, iters, cap, h_out) -- synchronises once: reads the engine counters and
 *       the headers of the previous exchange.  h_out[0] = 1 when every rank reported no queued
 *       work, no outbox and nothing sent (the march is over on every rank at the same round);
 *       h_out[1] = the exchange capacity (keys per destination) for this round's exchange, agreed
 *       from the headers (>= cap; identical on every rank); h_out[2] = visited cells summed over
 *       ranks, h_out[3] = any rank capped.  Otherwise replays up to `iters` BFS iterations on
 *       the owned queue (asynchronously, on the engine stream);
 *   am_shard_pack(e, d_send, cap)  -- outbox -> d_send, [world][am_shard_rows(e, cap)][KW]
 *       uint64 blocks, block r for rank r, each opening with a count header; keys beyond cap
 *       per destination stay in the outbox for the next round (asynchronous);
 *   the caller's all-to-all of equal blocks d_send -> d_recv (e.g. NCCL over NVLink) on the
 *       engine stream;
 *   am_shard_absorb(e, d_recv, cap) -- queues the received keys (device-side counts) and copies
 *       the headers to the host for the next am_shard_iterate (asynchronous).
 * Replaces the reference's shared visited set + queue of the threaded marcher
 * (reference marching.py:217-316) by a partitioned one. */
int am_shard_rows(am_engine *e, int64_t cap);
int am_shard_iterate(am_engine *e, int iters, int64_t cap, int64_t *h_out);
int am_shard_pack(am_engine *e, uint64_t *d_send, int64_t cap);
int am_shard_absorb(am_engine *e, const uint64_t *d_recv, int64_t cap);
/* h_out[6]: rounds, host synchronisations so far, iterations, pool entries, visited, outbox */
int am_shard_stats(am_engine *e, int64_t *h_out);

/* --- results ------------------------------------------------------------- */
/* h_counts[8]: cells, faces, empty, verts, edge_refs, open_edges, capped, overflow */
int am_result_counts(am_engine *e, int64_t *h_counts);
/* copy results to HOST buffers, cells sorted by (key, branch) like the
 * reference (marching.py:346-349).  edge_refs are global plane ids:
 * id < n_bits neuron, id < n_bits+n_subs branch target, else bbox face. */
int am_result_copy(am_engine *e, uint64_t *h_keys, int32_t *h_nverts, double *h_verts,
                   int32_t *h_edge_nrefs, int32_t *h_edge_refs);
/* the same sorted arrays into DEVICE buffers (sorting and gathering run on the GPU in both
 * calls: LSD radix sort of the key words, CSR gathers); feeds am_weld without a host trip */
int am_result_copy_device(am_engine *e, uint64_t *d_keys, int32_t *d_nverts, double *d_verts,
                          int32_t *d_edge_nrefs, int32_t *d_edge_refs);

/* --- mesh assembly ------------------------------------------------------- */
/* Weld the vertices of a polygon soup: reference meshes.py:89-148 weld(mesh, tol)
 * (MarchResult.welded_mesh, reference marching.py:126-127), bit-identical output.
 * Device inputs: d_verts [n_verts*3] fp64, loops as CSR d_loop_off [n_loops+1] /
 * d_loop_idx [d_loop_off[n_loops]] (int64 vertex indices).  Device outputs (caller-sized):
 * d_remap [n_verts] (vertex -> kept index), d_kept [n_verts*3] (first n_kept rows used),
 * d_face_off [n_loops+1] / d_face_idx [d_loop_off[n_loops]] (kept faces, CSR; loops that
 * collapse below 3 distinct vertices are dropped), d_face_src [n_loops] (source loop of each
 * kept face, for carrying face planes).  h_counts[3] = {n_kept, n_faces, n_dropped}.
 * stream: a cudaStream_t (null = legacy default stream); returns after synchronizing it. */
int am_weld(const double *d_verts, int64_t n_verts, const int64_t *d_loop_off, const int64_t *d_loop_idx,
            int64_t n_loops, double tol, void *stream, int64_t *d_remap, double *d_kept, int64_t *d_face_off,
            int64_t *d_face_idx, int64_t *d_face_src, int64_t *h_counts);

/* --- diagnostics -------------------------------------------------------- */
/* Pairs (i < j) of face planes proportional within chord tol (reference network.py:528-570
 * check_unique_planes; MarchReport.unique_plane_violations, reference marching.py:361-363).
 * d_planes: m rows (nx, ny, nz, d) fp64 on the device.  Up to cap pairs are written to d_pairs
 * (int32 [cap][2], unordered); *h_count = the number of pairs found (may exceed cap: call
 * again with a larger buffer).  stream: a cudaStream_t; returns after synchronizing it. */
int am_unique_planes(const double *d_planes, int64_t m, double tol, int32_t *d_pairs, int64_t cap, void *stream,
                     int64_t *h_count);

/* --- profiling hooks (bench.py roofline) --------------------------------- */
/* cumulative device time (ms) of the compose (DMMA) kernels, of the face
 * kernel, and the algorithmic flop / byte counts they processed; h_out[16] = composition
 * flops taken from parents' rows instead of executed (prefix reuse), h_out[17] = 1 when prefix
 * reuse is on (18 doubles) */
int am_stats(am_engine *e, double *h_out18);
int am_set_timing(am_engine *e, int enabled);
/* timing mode: per-stage device time (ms) of the timed iterations, the stages contiguous so they
 * sum to the iterations' device time: h_out16[0..8] take, compose, canonical insert, frontier,
 * near lists, face solver, flip insert, probe records, exact probe forwards; [9] iterations;
 * [10] flip candidates; [11] changed canonical keys; [12] probe records; [13] new pool entries;
 * [14] key words; [15] cells composed */
int am_kernel_times(am_engine *e, double *h_out16);
/* measured fp64 peaks of this device: h_out2[0] DMMA (tensor) TFLOP/s, [1] DFMA TFLOP/s */
int am_bench_fp64_peak(int device, double *h_out2);
/* face-kernel instrumentation counters (64; non-zero only in -DAM_FACE_STATS builds), reset on read */
int am_debug_counters(am_engine *e, uint64_t *h_out64);

#ifdef __cplusplus
}
#endif
#endif /* AM_B200_H */
