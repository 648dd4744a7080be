/*
 * emb_a2a.h -- C ABI of libemba2a.so: fused EmbeddingBag(sum) + All-to-All for B200 (sm_100a).
 *
 * Method: arXiv 2305.06942 ("fusing computation with communication using GPU-initiated
 * networking").  Citations: P:n = PAPER.md line n (with section); S:n = SPEC.md line n;
 * R#n = reading n in DESIGN.md.
 *
 * What one forward computes: rank r owns T_r embedding tables (model
 * parallel, P:68 / P:135) and sum-pools them for the WHOLE global batch B.  Pooled vector (t, j)
 * belongs to the rank s with p_s <= j < p_{s+1} (contiguous batch blocks) and lands in
 * row i = j - p_s, columns [(toff_r + t) * D, (toff_r + t + 1) * D) of s's output
 * {local batch b_s, numTables G x D}.  The kernel stores every pooled vector straight
 * into the destination GPU's receive buffer over NVLink ("zero-copy", Sec 3.3), signals
 * one per-peer arrival counter per completed slice with system-scope release semantics
 * (the PUT -> fence -> sliceRdy protocol of P:151), and waits for every peer's slices with
 * acquire loads before it exits ("poll on ... sliceRdy flags before exiting").
 *
 * Conventions (all entry points):
 *  - Every call returns an int status (emb_a2a_status).  0 = success.
 *  - A call that fails validation returns before enqueuing any GPU work.
 *  - Asynchronous device failures (receive-wait timeout) are recorded in a mapped host word and
 *    returned by the NEXT call on the handle as EMB_A2A_ETIMEOUT; the handle is then poisoned
 *    (every later call except destroy returns EMB_A2A_ESTATE).
 *  - register_tables, forward, forward_host and destroy are COLLECTIVE: every rank of the group
 *    calls them the same number of times in the same order (as with NCCL).
 *  - A handle is not thread-safe.  Different handles may be used from different threads.
 *  - emb_a2a_last_error() returns a human-readable message for the last failure on a handle.
 */
#ifndef EMB_A2A_H_
#define EMB_A2A_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMB_A2A_ABI_VERSION 1
#define EMB_A2A_MAX_WORLD 64

typedef enum {
    EMB_A2A_OK = 0,
    EMB_A2A_EINVAL = 1,    /* bad argument / inconsistent metadata across ranks */
    EMB_A2A_ESTATE = 2,    /* call out of order, or handle poisoned by an earlier failure */
    EMB_A2A_ECUDA = 3,     /* a CUDA runtime call failed (message in last_error) */
    EMB_A2A_ENOMEM = 4,    /* device or pinned host allocation failed */
    EMB_A2A_EPEER = 5,     /* a peer's buffers cannot be mapped (no P2P / IPC path) */
    EMB_A2A_EBOOT = 6,     /* the caller's all-gather callback failed */
    EMB_A2A_ETIMEOUT = 7,  /* a peer never signalled within timeout_ms (P:151 drain) */
    EMB_A2A_EINDEX = 8     /* validate mode: index out of range / malformed CSR */
} emb_a2a_status;

/* Table element types.  Every element is converted exactly to fp32 before it is accumulated;
 * the output is always fp32 (R#28). */
typedef enum { EMB_A2A_F32 = 0, EMB_A2A_BF16 = 1, EMB_A2A_F16 = 2 } emb_a2a_dtype;
/* Pooling (EmbeddingBag_updateOutputKernel_sum_mean): sum, or sum / bag length with IEEE
 * fp32 division (an empty bag gives +0.0) (R#27). */
typedef enum { EMB_A2A_SUM = 0, EMB_A2A_MEAN = 1 } emb_a2a_pooling;

typedef struct emb_a2a emb_a2a_t;

/* Caller-supplied all-gather over its process group (the bootstrap channel; S:86 problem
 * record exchange).  send: nbytes; recv: world_size * nbytes, rank-ordered.  Return 0 on success.
 * Called synchronously from inside init / register_tables / destroy. */
typedef int (*emb_a2a_allgather_fn)(const void* send, void* recv, size_t nbytes, void* user);

/* Create a handle for rank `rank` of `world_size` (1..EMB_A2A_MAX_WORLD) on CUDA device
 * `cuda_device`.  Several handles may live in one process (virtual ranks for loopback tests),
 * on the same or different devices.  *out receives the handle.  Not collective. */
int emb_a2a_init(int rank, int world_size, int cuda_device, emb_a2a_allgather_fn allgather,
                 void* user, emb_a2a_t** out);

/* Register this rank's tables and the problem shape (collective).
 *  num_local_tables  T_r >= 0 (may differ across ranks; G = sum_r T_r >= 1).
 *  tables            host array of T_r DEVICE pointers, each row-major [rows[t]][dim] float32,
 *                    16-byte aligned.  Borrowed: must stay valid and unchanged during forwards
 *                    until destroy.  Table-wise model parallelism.
 *  rows              host array of T_r row counts, 1 <= rows < 2^31.
 *  dim               D, identical on all ranks, D % 4 == 0, 4 <= D <= 1024 (R#9).
 *  global_batch      B >= 0, identical on all ranks.
 *  batch_partition   host array of W+1 prefix sums p (p_0 = 0, p_W = B, non-decreasing),
 *                    identical on all ranks; NULL = even split (requires B % W == 0) (R#1).
 * Allocates the symmetric receive region (2 buffers [b_r][G*D] float32 + per-peer counters,
 * P:178 "symmetric heap"), exports it with cudaIpcGetMemHandle, maps every peer's region
 * (cudaIpcOpenMemHandle; raw pointer for handles in the same process) -- the roc_shmem_ptr
 * analogue of P:165 -- and all-gathers metadata to check consistency.
 * May be called again to re-register (the old registration is torn down collectively). */
int emb_a2a_register_tables(emb_a2a_t* h, int num_local_tables, const float* const* tables,
                            const int64_t* rows, int dim, int64_t global_batch,
                            const int64_t* batch_partition);

/* register_tables with a table element type (emb_a2a_dtype; tables[t] then points to
 * [rows][dim] elements of that type, dim * element size a multiple of 16 bytes) and a pooling
 * mode (emb_a2a_pooling).  Both must be identical on all ranks (EINVAL otherwise). */
int emb_a2a_register_tables_ex(emb_a2a_t* h, int num_local_tables, const void* const* tables,
                               const int64_t* rows, int dim, int table_dtype, int pooling,
                               int64_t global_batch, const int64_t* batch_partition);

/* One fused forward (collective), asynchronous on `stream` (cudaStream_t; NULL = legacy default).
 *  indices   DEVICE int32[num_indices]: the T_r tables' bags concatenated table-major; values
 *            are local row ids (0 <= idx < rows[t]).  Borrowed until the stream passes the op.
 *  offsets   DEVICE int32[T_r * B + 1]: absolute CSR offsets, offsets[0] = 0, non-decreasing,
 *            offsets[T_r*B] = num_indices (bag (t, j) = indices[offsets[t*B+j] .. offsets[t*B+j+1])).
 *  out       receives a DEVICE pointer to this rank's output [b_r][G*D] row-major, the layout
 *            the interaction op consumes; float32, or -- with set_option("out_dtype")
 *            -- bfloat16 / binary16 elements (the fp32 sum rounded once to nearest even, R#32),
 *            which halves the bytes every peer store moves over NVLink.  Library-owned; valid until the SECOND
 *            following forward on this handle or destroy (double buffer by epoch parity).
 *  out_rows, out_cols  receive b_r and G*D (either may be NULL).
 * Preconditions (fast path, unchecked unless set_option("validate",1)): indices in range,
 * offsets well formed.  The consumer of *out must be ordered before this rank's forward after
 * next (same stream, or an event the stream waits for): a forward adds a credit to every peer
 * when it starts, and no peer stores into this rank's receive half before the credit of the
 * forward that reuses it.  Exception: when a peer runs on this same GPU
 * (virtual ranks, a test mode) the consumer must be ordered before the NEXT forward. */
int emb_a2a_forward(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                    int64_t num_indices, void* stream, float** out, int64_t* out_rows,
                    int64_t* out_cols);

/* forward with per-sample weights: weights = DEVICE float32[num_indices] aligned with indices
 * (NULL = unweighted); pooled value = sum_k fl(w_k * x_k) in bag order (R#26).  Sum pooling only
 * (EINVAL with mean, as torch.nn.functional.embedding_bag). */
int emb_a2a_forward_weighted(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                             const float* weights, int64_t num_indices, void* stream,
                             float** out, int64_t* out_rows, int64_t* out_cols);

/* The same forward fed from HOST memory (the end-to-end path): copies h_indices / h_offsets
 * (host, ideally pinned) into library-owned device staging, runs the fused forward, and copies
 * the [b_r][G*D] result into h_out (host, b_r*G*D elements of the output type).  The forward and the result
 * copy are enqueued on `stream`; the input copy runs on a library-owned copy stream that
 * `stream` waits for, into one of two staging buffers, so consecutive calls overlap the next
 * call's host->device copy with this call's device->host copy.  Returns after enqueuing;
 * synchronise the stream before reading h_out or reusing h_indices / h_offsets (collective). */
int emb_a2a_forward_host(emb_a2a_t* h, const int32_t* h_indices, const int32_t* h_offsets,
                         int64_t num_indices, void* stream, float* h_out);

/* A sequence of nsteps host-buffer forwards, pipelined (collective; every rank passes the same
 * nsteps): step k copies h_indices[k] (num_indices[k] int32) and h_offsets[k] (T_r*B+1 int32)
 * in on one library copy stream, runs the fused forward on `stream`, and copies the result into
 * h_out[k] (b_r*G*D elements of the output type) on a second copy stream -- so step k's result copy overlaps step
 * k+1's forward and step k+2's input copy (the serving loop).  All host buffers ideally pinned,
 * and left untouched until `stream` is synchronised; `stream` completes only after the last
 * result copy.  Returns after enqueuing. */
int emb_a2a_forward_host_batch(emb_a2a_t* h, int nsteps, const int32_t* const* h_indices,
                               const int32_t* const* h_offsets, const int64_t* num_indices,
                               float* const* h_out, void* stream);

/* Unfused baseline, first half (not collective): the same pooling, written with local stores to
 * a caller-owned DEVICE staging buffer `send`, dest-major [W][b_s][T_r][D] elements of the output
 * type (the block of destination s starts at p_s*T_r*D elements).  The second half is the caller's NCCL
 * all_to_all_single (P:250 baseline: embedding kernels + RCCL All-to-All). */
int emb_a2a_pool_local(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                       int64_t num_indices, void* stream, float* send);

/* pool_local with per-sample weights (device float32[num_indices], NULL = unweighted). */
int emb_a2a_pool_local_weighted(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                                const float* weights, int64_t num_indices, void* stream,
                                float* send);

/* ---------------------------------------------------------------- backward
 * The paper leaves the backward pass to future work (Sec 5 "explore ... the backward
 * pass").  What it computes (R#29-R#31; oracle_backward_sgd): rank s holds
 * dL/d(out_s), [b_s][G*D] float32, the gradient of its forward output.  The owner r of table g
 * (local t) applies, for every row x that occurs in g's bags,
 *     W_g[x] = W_g[x] - fl(lr * sum_{k : idx_k = x} c_k)
 *     c_k = grad_s[j - p_s][g*D .. g*D + D)   for lookup k in bag j, s = dest(j)
 *           (fl(w_k * grad) with per-sample weights, fl(grad / L_j) with mean pooling)
 * i.e. the forward's All-to-All reversed (data parallel -> model parallel) followed by the
 * embedding-gradient segment reduction and a sparse SGD step.  Rows that do not occur are not
 * touched.  fp32 tables only (EINVAL otherwise).  The sum over a row's lookups is taken in a
 * fixed, deterministic order (runs of C sorted lookups, then runs in order, R#31), so
 * repeated calls give bitwise-identical tables; it matches the oracle's ascending-order sum
 * within the fp32 rounding bound, and bitwise when every partial sum is exact. */

/* Backward plan (not collective): sorts this rank's lookups by (local table, row) on `stream`
 * (stable LSD radix sort in the library's kernels).  Depends only on the forward's inputs, so it
 * can run as soon as they are known (e.g. on a side stream overlapping the dense layers).
 *  indices, offsets  as for emb_a2a_forward (DEVICE, borrowed: offsets must stay valid until
 *                    the backward that uses this plan has run, for mean pooling).
 *  weights           DEVICE float32[num_indices] per-sample weights, or NULL (sum pooling only).
 * Plan storage is library-owned and grow-only; a new plan replaces the previous one.
 * EINVAL if the sort key t << ceil(log2(max rows)) | row needs more than 32 bits. */
int emb_a2a_backward_plan(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                          const float* weights, int64_t num_indices, void* stream);

/* Fused backward (collective), asynchronous on `stream`, using the last plan.
 *  grad   DEVICE float32 [b_r][G*D] row-major (the forward output's layout): dL/d(out_r).
 *         Borrowed until the stream passes the op.  16-byte aligned.
 *  lr     SGD learning rate.
 * One kernel: every CTA pushes its share of grad's column blocks (owner q's tables) straight
 * into q's library-owned staging buffer over NVLink and releases q's per-source counter
 * (red.release.sys), waits for every source's rows (ld.acquire.sys, bounded by timeout_ms ->
 * ETIMEOUT on the next call), then reduces and updates this rank's tables in place.  The
 * registered table memory is written: nothing else may read or write it until the stream passes
 * the op.  Staging is double-buffered by backward epoch, like the forward's receive buffers. */
int emb_a2a_backward(emb_a2a_t* h, const float* grad, float lr, void* stream);

/* Unfused backward, second half (not collective): the same reduce + update from a caller-owned
 * DEVICE float32 gradient in model-parallel layout [B][T_r][D] (row j = global sample j) -- what
 * NCCL all_to_all_single delivers from the destination ranks' [b_s][T_r*D] column blocks.  The
 * baseline is: pack columns, all_to_all_single, backward_local. */
int emb_a2a_backward_local(emb_a2a_t* h, const float* grad_mp, float lr, void* stream);

/* Cross-rank device barrier on `stream` (collective; benchmark tooling, not part of the op):
 * returns immediately on the host; the stream proceeds once every rank's barrier kernel has
 * arrived (system-scope release/acquire counters in the symmetric region).  Used to align the
 * start of timed regions across GPUs.  Timeout -> ETIMEOUT on the next call. */
int emb_a2a_device_barrier(emb_a2a_t* h, void* stream);

/* NVLink store probe (benchmark tooling, not part of the op): enqueue on `stream` one kernel in
 * which every CTA issues 16-byte st.global.v4 stores -- the fused kernel's store -- into the
 * receive regions of ALL peers at once (512-byte runs, destinations staggered as in row a1).
 * Writes min(bytes_per_peer, the smallest peer region) rounded down to 512 B per peer
 * (*bytes_used); the peers' receive buffers (both halves) are overwritten, so no earlier
 * forward output may still be in use anywhere.  Timed with events by the caller, all ranks
 * together (after a device barrier), it gives the SM-issued peer-store bandwidth the fused
 * kernel's exchange can reach.  W = 1: enqueues nothing, *bytes_used = 0. */
int emb_a2a_peer_store_probe(emb_a2a_t* h, int64_t bytes_per_peer, void* stream,
                             int64_t* bytes_used);

/* Tunables (not collective, but keep them identical on all ranks; "slice" must be):
 *   "slice"        S, pooled vectors per slice, >= 1 (P:147 user parameter; default 32)
 *   "order"        0 comm-aware staggered (default), 1 comm-aware ascending, 2 oblivious
 *                  (set before register_tables)
 *   "out_dtype"    output element type (emb_a2a_dtype): 0 fp32 (default), 1 bf16, 2 fp16 --
 *                  accumulation stays fp32, the result is rounded once (R#32); identical on all
 *                  ranks, set before register_tables (the receive buffers are sized for it)
 *   "chunk"        bags per work ticket, 1..127, or 0 (default): per forward, about 640
 *                  lookups per ticket from the forward's average bag length, 32..127 bags.
 *                  Load-balance granularity, rank-local, independent of the signal slice S --
 *                  a chunk's bags count toward every slice they fall in (set before
 *                  register_tables)
 *   "threads"      consumer threads per CTA, multiple of 32 in [32, 256] (default 256); each
 *                  CTA also has one producer warp
 *   "timeout_ms"   receive-wait timeout (default 10000)
 *   "validate"     1 = check indices/offsets on device before each forward (sync)
 *   "flat_below"   pipeline stages whose average bag length is below this (default 12) pool with a
 *                  row-flattened loop (rows of several short bags in flight at once); longer
 *                  bags use the per-bag loop.  0 = always per-bag, large = always flattened
 *   "l1_rows"      unweighted forwards, LSU gathers: -1 auto (default: when the forward has
 *                  >= 4096 lookups per SM or B >= 4096 bags per table), 0 rows stream past L1
 *                  (L1::no_allocate), 1 rows are
 *                  allocated in L1 (a Zipf-hot row recurring on the same SM is served there).
 *                  Same results either way.  Read back "l1_rows_active" for the last forward's
 *                  choice.
 *   "pdl"          1 = programmatic dependent launch (default): the kernel's CTAs may start while
 *                  the previous kernel on the stream drains; all reads of inputs, counters and
 *                  buffers wait (griddepcontrol.wait) for that kernel to complete
 *   "pdl_rows_early"  1 (default): with one rank (W = 1), a forward's table-row reads and stores
 *                  skip the programmatic wait when this handle has launched no backward since its
 *                  previous forward (the predecessor can then only be a forward, which never
 *                  writes tables or this forward's receive buffer).  Set 0 if a
 *                  kernel of your own that writes the tables and triggers programmatic launch
 *                  (griddepcontrol.launch_dependents) can directly precede a forward on its stream.
 *                  With peers, stores into a peer wait for that peer's credit (it has started
 *                  the same forward, so it consumed the buffer half they overwrite); off when a
 *                  peer shares this GPU (its CTAs could need the slots), 2 = on even then
 *   "debug_credit_lag"  -1 (default): a peer's store into this rank's buffer half waits for this
 *                  rank to have started the same forward (0) -- or, when a peer shares this GPU,
 *                  the previous one (1, the weaker consumer contract); 0 / 1 force it (tests of
 *                  the one-GPU-per-rank protocol on one GPU, with grids small enough to co-reside)
 *                  (tests, small grids)
 *   "vec"          float4s per lane per row, 1/2/4/8 (0 = auto): lanes per bag = D/(4*vec);
 *                  fewer lanes per bag keeps more bags in flight per warp
 *   "tma"          0 = per-lane 16-byte LDG row gathers, indices staged in shared memory (default)
 *                  1 = TMA tile::gather4 of whole rows into shared memory (measured ~2x slower
 *                  for 256 B - 1 KB rows on B200; kept as an option); applies to
 *                  fp32 unweighted forwards only, others use the LDG path
 *   "stage_kb"     TMA mode: KiB of table rows per pipeline stage (default 32); a bag with more
 *                  rows than a stage holds is gathered with LDGs
 *   "stages"       shared-memory pipeline depth per CTA, 2..8 (default 4; reduced to fit 227 KB)
 *   "ctas_per_sm"  persistent grid size per SM: 0 = max occupancy (P:280 occupancy study)
 *   "idx_cap"      LSU mode: indices per pipeline stage (default 2048); a chunk whose bags need
 *                  more is split over several stages, and a single bag longer than this reads
 *                  its indices from global memory
 *   "trace"        N > 0: record up to N per-CTA %globaltimer events per forward (the paper's
 *                  per-WG timeline); 0 = off (default).  Read with emb_a2a_read_trace.
 *   "sort_mode"    backward plan's radix passes: 0 auto (default: the bucket plan (5) for
 *                  65536..524288 lookups with <= 32768 per table, else one kernel per 8-bit
 *                  pass with look-back while the
 *                  tiles fit one wave, else three kernels per pass, reduce-then-scan), 1 always
 *                  one kernel, 2 always three, 3 the segmented plan
 *                  (each table's lookups sorted by row bits only: 2 passes of <= 11-bit digits,
 *                  tiles aligned to tables; needs rows <= 2^22 and T <= 256, else as 0), 4 the
 *                  cluster plan (ONE kernel: a thread-block cluster per table generates and
 *                  sorts the table's lookups by row bits, <= 8-bit digits, digit offsets
 *                  exchanged in distributed shared memory, passes split by cluster barriers), 5
 *                  the bucket plan (one pass on the top 8 key bits, then one CTA per bucket sorts
 *                  it by the low bits in shared memory) -- results identical in every mode
 *   "bucket_cap"   bucket plan: keys a bucket may hold to be sorted in shared memory (default
 *                  4096; multiple of 256 in 256..8192; shared memory per CTA = 16 B x cap, so
 *                  larger caps fit fewer CTAs per SM); larger buckets sort in global memory
 *   "cluster_ctas" cluster plan: CTAs per table cluster, 0 auto (default: the largest of 16, 8,
 *                  4, 2 whose T clusters fit two CTAs per SM, else 1; smaller if the occupancy
 *                  query says a cluster cannot be resident), or 1, 2, 4, 8, 16
 *   "bwd_threads"  backward kernel threads per CTA, multiple of 32 in [32, 128] (default 128;
 *                  the kernel is compiled with __launch_bounds__(128))
 *   "bwd_share"    divide the backward's persistent grid by this (default 1): W virtual ranks on
 *                  one GPU must all be resident at once (loopback sets it to W)
 *   "debug_delay_ns"  test knob: CTAs sleep this long before signalling (stress tests)
 *   "debug_skip_signal_to"  test knob: never signal rank v (>= 0), to exercise ETIMEOUT
 *   "debug_sort_stall"  test knob: the backward plan's first radix tile publishes a stale
 *                  look-back word (onesweep passes), so the look-back times out -> ETIMEOUT */
int emb_a2a_set_option(emb_a2a_t* h, const char* key, int64_t value);
int emb_a2a_get_option(const emb_a2a_t* h, const char* key, int64_t* value);

/* Read-only facts about the current registration:
 *   "rank", "world_size", "device", "epoch" (forwards issued), "local_batch" (b_r),
 *   "total_tables" (G), "table_offset" (toff_r), "dim", "table_dtype", "pooling" (0 sum,
 *   1 mean), "global_batch", "num_slices",
 *   "num_chunks", "chunk_bags" (C),
 *   "expected_in:<src>" (signals rank src sends here per forward), "region_bytes",
 *   "last_grid" (CTAs of the last fused launch), "kernel_launches" (total kernels launched),
 *   "backward_epoch" (fused backwards issued), "plan_lookups" (lookups in the current backward
 *   plan, -1 = none), "bwd_grid" (CTAs of the backward kernel), "bwd_chunk" (lookups per chunk). */
int emb_a2a_query(const emb_a2a_t* h, const char* key, int64_t* value);

/* Introspection for parity tests (synchronous; not on the hot path):
 *  slice_plan:  decode every slice ticket ON THE DEVICE (the same decode the fused kernel uses)
 *               into host out[n][4] = (dst s, local table t, first local row i0, rows nb).
 *  read_flags:  host out[W] = this rank's arrival counters, one per source rank. */
int emb_a2a_slice_plan(emb_a2a_t* h, int32_t* out, int64_t capacity, int64_t* n);
int emb_a2a_read_flags(emb_a2a_t* h, uint64_t* out, int capacity);
/* Trace log (set_option "trace" > 0): synchronises the device, copies the n records logged since
 * the last read into host out[n][2] = {cta << 40 | event << 32 | payload, globaltimer_ns}, and
 * restarts the log.  Events: 0 CTA start, 1 chunk ticket, 2 stage ready, 3 stage released
 * (payload 1 = completed a remote slice and signalled it), 4 consumers done, 5 receive wait done. */
int emb_a2a_read_trace(emb_a2a_t* h, uint64_t* out, int64_t capacity, int64_t* n);

/* Collective teardown: synchronises the device, barriers through the all-gather so no peer is
 * still writing, unmaps peers, frees the region.  h is invalid afterwards. */
int emb_a2a_destroy(emb_a2a_t* h);

/* Poll the asynchronous error word (not collective, no GPU work): EMB_A2A_ETIMEOUT if a receive
 * wait / credit wait / backward exchange wait / sort look-back / barrier timed out since the
 * last check (the handle is then poisoned), EMB_A2A_ESTATE if it already was, else OK.  Synchronise the stream first to see
 * the failures of work enqueued on it. */
int emb_a2a_check(emb_a2a_t* h);

const char* emb_a2a_last_error(const emb_a2a_t* h);
const char* emb_a2a_status_string(int status);
int emb_a2a_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EMB_A2A_H_ */
