/*
 * ag_gemm.h -- C ABI of the fused AllGather + GEMM in libemba2a.so (sm_100a).
 *
 * SURVEY.md Sec 8 row f4 ("other fused collectives ... AllGather+GEMM (FSDP)").  Method:
 * arXiv 2305.06942, P:180 (Sec 3.5 "General Applicability for Collectives"): "In fully-sharded
 * data parallel models, the AllGather collective can be overlapped with the subsequent matrix
 * computations" -- the paper's fused-kernel principle (the producer PUTs each finished
 * slice and sets a per-slice ready flag; the consumer waits only for the slice it needs) applied
 * to AllGather -> GEMM.  Citations: P:n = PAPER.md line n; R#n = reading n in DESIGN.md.
 *
 * What one forward computes on rank r of W (oracle/ag_gemm.py, R#33):
 *     W_gathered[s*N_r + i][k] = W_s[i][k]                     (AllGather, rank-ordered)
 *     Y_r[m][n]                = sum_k X_r[m][k] * W_gathered[n][k]   (a Linear layer, y = x W^T)
 * with bfloat16 operands, fp32 accumulation in tensor memory, and Y rounded once to bfloat16
 * (nearest even) or kept fp32 (R#34).
 *
 * How: ONE persistent kernel per rank.  Its communication warps copy the
 * rank's own shard W_r straight into every peer's gather buffer with 16-byte stores over
 * NVLink (zero-copy PUT), in chunks of one GEMM N-tile, destinations staggered
 * r+1, r+2, ... (comm-aware order); the last piece of a chunk fences at system scope and
 * stores the epoch into the destination's per-(source, chunk) ready flag (sliceRdy).
 * Its GEMM warps (TMA producer, tcgen05 MMA issuer, TMEM epilogue; by default a CTA pair per
 * 256 x BN tile with tcgen05.mma.cta_group::2) take output tiles in the
 * order local shard first, then sources r-1, r-2, ... -- the order the peers' chunks arrive --
 * and the TMA producer waits (ld.acquire.sys) for exactly the chunk a tile's B operand needs.
 *
 * Conventions: every call returns an int status (the emb_a2a_status codes of emb_a2a.h:
 * 0 OK, 1 EINVAL, 2 ESTATE, 3 ECUDA, 4 ENOMEM, 5 EPEER, 6 EBOOT, 7 ETIMEOUT).  Asynchronous
 * device failures (a flag or credit wait that timed out, a pipeline stall) are recorded in a
 * mapped host word and returned by the NEXT call as ETIMEOUT; the handle is then poisoned.
 * register and forward are COLLECTIVE (every rank calls them, same order).  Not thread-safe.
 */
#ifndef AG_GEMM_H_
#define AG_GEMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AG_GEMM_MAX_WORLD 8

typedef struct ag_gemm ag_gemm_t;

/* Caller-supplied all-gather over its process group (bootstrap only): send nbytes, recv
 * world_size * nbytes rank-ordered; return 0 on success.  Same contract as emb_a2a_allgather_fn. */
typedef int (*ag_gemm_allgather_fn)(const void* send, void* recv, size_t nbytes, void* user);

/* Create a handle for rank `rank` of `world_size` (1..AG_GEMM_MAX_WORLD) on `cuda_device`.
 * Several handles may live in one process (virtual ranks).  Not collective. */
int ag_gemm_init(int rank, int world_size, int cuda_device, ag_gemm_allgather_fn allgather,
                 void* user, ag_gemm_t** out);

/* Register the problem shape (collective; identical on all ranks, EINVAL otherwise).
 *  M        rows of X_r (tokens on this rank), M % 128 == 0, M >= 128.
 *  n_local  N_r rows of each rank's weight shard, N_r % 128 == 0; the GEMM N-tile (= the
 *           communication chunk) is 256 rows when N_r % 256 == 0, else 128 (option "bn").
 *           N = W * N_r < 2^31 / K.
 *  K        reduction length, K % 64 == 0, K >= 64.
 *  out_f32  0: Y is bfloat16 (fp32 accumulator rounded once to nearest even); 1: Y is float32.
 * Allocates the symmetric region -- [ready flags W x chunks u32 | credits W x 128 B | gather
 * buffer 0 [N][K] bf16 | gather buffer 1] -- exports it with cudaIpcGetMemHandle and maps every
 * peer's (raw pointer in the same process, cudaIpcOpenMemHandle across processes). */
int ag_gemm_register(ag_gemm_t* h, int64_t M, int64_t n_local, int64_t K, int out_f32);

/* One fused AllGather + GEMM (collective), asynchronous on `stream` (cudaStream_t).
 *  X        DEVICE bf16 [M][K] row-major (K contiguous), 16-B aligned.  Borrowed.
 *  w_local  DEVICE bf16 [N_r][K] row-major: this rank's shard W_r.  Borrowed.
 *  Y        DEVICE [M][W*N_r] row-major, bf16 or f32 per out_f32.  Caller-owned, written only by
 *           this rank's kernel.
 *  w_gathered  receives (if not NULL) a DEVICE pointer to this forward's gather buffer
 *           [W*N_r][K] bf16: every peer's shard, and this rank's own block only when option
 *           "local_copy" is 1 (an FSDP forward reads its own shard in place).  Library-owned;
 *           valid until this rank's NEXT forward starts (double buffer by epoch parity; a peer
 *           overwrites it in the forward after next, gated by this rank's start credit).
 * The kernel first adds one credit to every peer ("this rank started forward e, so its forward
 * e-1 completed"), and stores into peer q's buffer half e&1 only after q's credit shows q
 * started forward e-1. */
int ag_gemm_forward(ag_gemm_t* h, const void* X, const void* w_local, void* Y, void* stream,
                    void** w_gathered);

/* Options (set before or between forwards; identical on all ranks where noted):
 *   "grid"        persistent CTAs (0 = auto: SMs, divided by the number of ranks sharing the GPU)
 *   "local_copy"  1: also copy W_r into this rank's own gather block (default 0)
 *   "order"       0: tiles of the local shard first, then sources r-1, r-2, ... (comm-aware,
 *                 P:151, default); 1: ascending source order 0..W-1 (oblivious)
 *   "group_m"     M-tiles per raster group (default 16)
 *   "piece_kb"    bytes per communication piece, in KiB, power of two 4..1024 (default 64)
 *   "timeout_ms"  bound on every device-side wait (default 10000)
 *   "comm"        0: skip the communication warps (test mode: flags are then never set and a
 *                 remote tile times out) -- default 1
 *   "pair"        1: a cluster of two CTAs (one TPC) per 256 x BN tile, tcgen05.mma.cta_group::2,
 *                 each CTA staging its 128 A rows and half of the B rows (default; used when
 *                 M % 256 == 0); 0: one CTA per 128 x BN tile (cta_group::1)
 *   "bn"          0 (default: 256 when N_r allows), 128 or 256: the N-tile (set before
 *                 register)
 *   "l2hints"     L2 cache-policy bits (default 0 = none): 1 TMA loads of A evict_last, 2 of B
 *                 evict_first, 4 Y written with streaming stores (st.global.cs) -- measured
 *                 neutral to worse */
int ag_gemm_set_option(ag_gemm_t* h, const char* key, int64_t value);
int ag_gemm_get_option(const ag_gemm_t* h, const char* key, int64_t* value);

/* Derived values: "tiles" (output tiles per forward), "grid", "pair" (CTA pairs in use), "bn"
 * (N-tile), "chunks" (per source), "pieces" (per chunk), "epoch", "shared_gpu", "smem_bytes". */
int ag_gemm_query(const ag_gemm_t* h, const char* key, int64_t* value);

/* Copy this rank's ready flags [W][chunks] (u32 epoch stamps) into out (capacity words). */
int ag_gemm_read_flags(ag_gemm_t* h, uint32_t* out, int64_t capacity, int64_t* n);

/* Poll the asynchronous error word (0 or ETIMEOUT). */
int ag_gemm_check(ag_gemm_t* h);

/* Free everything (collective when registered: ranks synchronise before unmapping). */
int ag_gemm_destroy(ag_gemm_t* h);

const char* ag_gemm_last_error(const ag_gemm_t* h);

#ifdef __cplusplus
}
#endif
#endif /* AG_GEMM_H_ */
