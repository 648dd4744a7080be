// emb_a2a_internal.h -- shared between host.cpp (C ABI) and kernels.cu (sm_100a kernels).
// Not installed; the public ABI is include/emb_a2a.h.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/emb_a2a.h"

namespace emba2a {

constexpr int kMaxW = EMB_A2A_MAX_WORLD;
// Per-source arrival counters are padded to 128 B so concurrent writers never share a line.
constexpr int kFlagStride = 16;  // uint64 words
constexpr int kMaxStages = 8;    // shared-memory pipeline depth cap
constexpr int kMaxSmemTables = 256;  // table pointers cached in shared memory per CTA

// A CUtensorMap (TMA descriptor): 128 opaque bytes, 64-B aligned.
struct alignas(64) TmaDesc {
  unsigned char bytes[128];
};

// Where peer s's receive buffers and our counter inside peer s's region live.  Device-resident,
// written once per registration (the roc_shmem_ptr table of).
struct DevPeers {
  float* recv[kMaxW][2];                  // recv_s[parity] base, [b_s][G*D] float32
  unsigned long long* flag_out[kMaxW];    // &flags_s[r]: counter r increments in peer s
  long long n_in[kMaxW];                  // signals expected from source q per forward
  unsigned long long* barrier_out[kMaxW]; // peer q's barrier counter (device barrier)
  // backward (f3): peer q's gradient staging [B][T_q][D] float32 by parity, and our arrival
  // counter inside peer q's region (rows of our batch block pushed to q)
  float* gstage[kMaxW][2];
  unsigned long long* bflag_out[kMaxW];
  // buffer-reuse credits: &credits_q[r] / &bcredits_q[r] inside peer q's region.  A rank adds 1
  // to every peer's slot when a forward (backward) of its starts; a writer stores into peer q's
  // receive half (gradient staging half) only once q's credit proves q has consumed the previous
  // contents
  unsigned long long* credit_out[kMaxW];
  unsigned long long* bcredit_out[kMaxW];
};

// Kernel parameters, passed by value (constant bank).  Scalars + the two small tables the
// slice decode needs; everything per-peer is in DevPeers.
struct KParams {
  const int* indices;
  const int* offsets;
  const float* weights;         // per-sample weights aligned with indices, or NULL
  const void* const* tables;    // device array of T pointers (element type: elem)
  const TmaDesc* tmaps;         // device array of T tensor maps (TMA gather mode)
  float* send;                  // pool_local staging base ([B][T][D] by global row)
  const DevPeers* peers;
  unsigned long long* flags_in; // own counters, index src * kFlagStride
  const unsigned long long* credits_in;  // own credit counters (forwards started by src)
  unsigned int* done;           // CTA completion counter (last-CTA detection)
  unsigned int* ticket;         // next chunk ticket (beyond the first gridDim.x)
  unsigned long long* slice_cnt;// per-slice completed-bag counters (monotone over epochs)
  int* err;                     // device alias of the mapped host error word
  unsigned long long* trace;    // optional %globaltimer event log (NULL = off); [0] = count
  long long trace_cap;          // records (2 words each) after the header
  long long B;
  unsigned long long epoch;     // 1-based forward number
  long long timeout_ns;
  long long delay_ns;
  int W, r, T, D, G, toff, S, C, order, nslices, nchunks, nstages, skip_to, parity;
  int DU;             // 16-byte units per table row (D * element size / 16)
  int elem;           // table element type: 0 fp32, 1 bf16, 2 fp16
  int mean;           // 1: mean pooling (P:119 sum_mean), 0: sum
  int out_dtype;      // output element type: 0 fp32, 1 bf16, 2 fp16 (R#32: rounded once, RNE)
  int oshift;         // log2 of the output element size (2 or 1)
  int tma;            // 1: rows via TMA gather4 into shared memory; 0: per-lane LDG gathers
  int ncb, box4;      // TMA: column blocks per row and float4s per block (DU = ncb * box4)
  int stage_bytes;    // shared memory per pipeline stage
  int payload_off;    // offset of the rows / indices inside a stage
  int payload_cap;    // rows (TMA) or indices (LSU) a stage holds
  int pdl;            // programmatic dependent launch (overlap with the stream predecessor)
  int rows_wait;      // consumers wait for the predecessor before reading table rows
  int pdl_trigger;    // trigger the dependent launch once the predecessor is complete (else
                      // only by exiting)
  int credit_lag;     // a peer's credit must reach epoch - credit_lag before we store into it
  int flat_below;     // stages whose average bag length is below this use row-flattened pooling
  int l1rows;         // unweighted LSU gathers: rows allocated in L1 (instance sets ELEM 3-5)
  long long part[kMaxW + 1];    // batch partition prefix
  int slice_base[kMaxW + 1];    // first slice of destination ordinal k; [W] = nslices
  int chunk_base[kMaxW + 1];    // first chunk of destination ordinal k; [W] = nchunks
};

// Destination rank of ordinal k in rank r's slice order (row a1; R#19).
__host__ __device__ inline int dest_of_ordinal(int order, int r, int W, int k) {
  if (order == 0) return (k < W - 1) ? (r + 1 + k) % W : r;        // staggered remote, local last
  if (order == 1) return (k < W - 1) ? (k < r ? k : k + 1) : r;    // ascending remote, local last
  return k;                                                        // oblivious
}

// Work units of one rank, in issue order (row a1): for destination ordinal k = 0..W-1 (dest
// s = dest_of_ordinal(k)), local table t, then row blocks of `unit` bags of s's batch block.
// With unit = S these are the slices (signal granularity); with unit = C (C | S) they are
// the chunks handed out as tickets (load-balance granularity).  base[k] = first unit of ordinal k.
__host__ __device__ inline void decode_unit(const KParams& P, int ticket, int unit,
                                            const int* base, int& k, int& s, int& t, int& i0,
                                            int& nb) {
  k = 0;
  while (k < P.W - 1 && ticket >= base[k + 1]) ++k;
  s = dest_of_ordinal(P.order, P.r, P.W, k);
  const int q = ticket - base[k];
  const long long b_s = P.part[s + 1] - P.part[s];
  const int nu = (int)((b_s + unit - 1) / unit);
  t = q / nu;
  const int c = q - t * nu;
  i0 = c * unit;
  const long long rem = b_s - i0;
  nb = rem < unit ? (int)rem : unit;
}

__host__ __device__ inline void decode_slice(const KParams& P, int ticket, int& s, int& t,
                                             int& i0, int& nb) {
  int k;
  decode_unit(P, ticket, P.S, P.slice_base, k, s, t, i0, nb);
}

// Global slice id and size of the slice containing chunk (k, s, t, i0).
__host__ __device__ inline void slice_of_chunk(const KParams& P, int k, int s, int t, int i0,
                                               int& slice_id, int& slice_bags) {
  const long long b_s = P.part[s + 1] - P.part[s];
  const int nsl = (int)((b_s + P.S - 1) / P.S);
  const int c = i0 / P.S;
  slice_id = P.slice_base[k] + t * nsl + c;
  const long long rem = b_s - (long long)c * P.S;
  slice_bags = rem < P.S ? (int)rem : P.S;
}

// fp32 rows are gathered through L1 (auto "l1_rows") for forwards with at least kL1RowsPerSm
// lookups per SM or at least kL1RowsBags bags per table: a Zipf-hot row then recurs on the same
// SM often enough that L1 hits beat streaming every row past L1.  Measured (r02ak, W=1, on vs
// off): DLRM-wide 193 -> 162 us, sweep P=32 155.5 -> 133.7, P=8 62.9 -> 59.5, P=4 41.1 -> 38.7,
// P=1 22.6 -> 22.0 (B = 4096 / 8192); DLRM-small 12.4 -> 12.7 and weak 18.8 -> 19.6 (B = 2048 /
// 1024, ~2.2 K lookups per SM) -- left streaming.
constexpr long long kL1RowsPerSm = 4096;
constexpr long long kL1RowsBags = 4096;

// Fill stage_bytes / payload_off / payload_cap for P.tma, P.C, P.D4 (kernels.cu).
void stage_layout(KParams& P, int stage_kb, int idx_cap);

struct LaunchCfg {
  int threads;      // consumer threads per CTA (+1 producer warp)
  int vec;          // float4s per lane (0 auto)
  int ctas_per_sm;  // persistent grid: 0 = max occupancy
};

// A resolved launch: kernel instance, persistent grid, block, shared memory, pipeline depth.
struct LaunchPlan {
  const void* fn = nullptr;
  unsigned grid = 0;
  int threads = 0;
  size_t smem = 0;
  int nstages = 0;
};

// Launchers (kernels.cu).  plan_* resolve a LaunchPlan once (occupancy query etc.);
// launch_planned is the per-forward path.
cudaError_t plan_fused(const KParams& P, const LaunchCfg& c, LaunchPlan* pl);
// per-instance-set planners (inst_*.cu) and the shared resolver (kernels.cu)
cudaError_t plan_with(const void* fn, const KParams& P, const LaunchCfg& c, LaunchPlan* pl);
cudaError_t plan_f32(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl);
cudaError_t plan_f32w(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl);
cudaError_t plan_f32l1(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl);
cudaError_t plan_bf16l1(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl);
cudaError_t plan_f16l1(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl);
cudaError_t plan_bf16(const KParams& P, const LaunchCfg& c, bool fused, bool weighted,
                      LaunchPlan* pl);
cudaError_t plan_f16(const KParams& P, const LaunchCfg& c, bool fused, bool weighted,
                     LaunchPlan* pl);
cudaError_t plan_pool_local(const KParams& P, const LaunchCfg& c, LaunchPlan* pl);
cudaError_t launch_planned(const LaunchPlan& pl, KParams P, cudaStream_t st);
cudaError_t launch_barrier(const DevPeers* peers, unsigned long long* own_counter, int W, int r,
                           unsigned long long target, long long timeout_ns, int* err,
                           cudaStream_t st);
cudaError_t launch_slice_plan(const KParams& P, int* out, cudaStream_t st);
cudaError_t launch_peer_store_probe(const DevPeers* peers, int W, int r, long long runs,
                                    cudaStream_t st);
cudaError_t launch_validate(const int* indices, const int* offsets, long long nnz, long long TB,
                            long long B, int T, const long long* rows_dev, int* err_dev,
                            cudaStream_t st);

// ------------------------------------------------------------------------------ backward (f3)
// Sort plan: this rank's lookups as (key = t << rbits | row, payload = bag id t*B + j [, weight])
// sorted stably by key with an LSD radix sort (8-bit digits, one onesweep pass per digit; the
// last digit may be narrower).
constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;   // keys per onesweep tile
constexpr int kMaxPasses = 4;                          // 32-bit keys
constexpr int kHistWords = kMaxPasses * 256 + kMaxPasses;   // digit counts + tile tickets
constexpr int kLbGroup = 16;                           // onesweep look-back group (tiles)
constexpr int kSegLb = 4;                              // segmented plan: look-back group (tiles)

struct SortParams {
  const int* indices;
  const int* offsets;
  const float* weights;        // NULL = unweighted
  unsigned* keys;              // [n] out (keygen) / pass ping-pong buffers
  int* bags;
  float* wts;
  unsigned* hist;              // [kMaxPasses][256] digit counts + tile tickets (zero at entry)
  unsigned* hist_clear;        // the other half of the plan buffer: zeroed here for the next plan
  long long TB, B;
  int rbits, passes;
  unsigned last_mask;          // digit mask of the last pass (the key may end inside a digit)
  int hshift;                  // bit of pass 0's digit (0; the bucket plan counts the TOP digit)
  unsigned* lbg;               // onesweep group look-back words of every pass (zeroed by keygen)
  long long lbg_words;
  // segmented plan (seg_db > 0): digits are row bits only, counted per (table, digit); the
  // input is table-major, so each table's lookups are sorted in place of its own segment
  int seg_db;                  // digit bits of both passes (the last may be narrower)
  int T;                       // tables (<= 256)
  unsigned* shist;             // [2 passes][T][1 << seg_db] digit counts (zero at entry)
  unsigned* shist_clear;       // the other half, zeroed here for the next plan
  long long shist_words;       // words per half (incl. the 2 tile tickets)
};

struct PassParams {
  const unsigned* keys_in;
  unsigned* keys_out;
  const int* bags_in;
  int* bags_out;
  const float* wts_in;         // NULL = no weight payload
  float* wts_out;
  const unsigned* hist;        // this pass's 256 digit counts
  unsigned* cnt;               // [256][ntiles] tile digit counts -> global digit offsets
  unsigned long long* status;  // onesweep: [ntiles][256] look-back words of this pass
  unsigned* tile_ctr;          // onesweep: this pass's tile ticket (zeroed before keygen)
  unsigned* garrive;           // onesweep: [ngroups] tiles of each look-back group counted in
  unsigned* gsum;              // onesweep: [ngroups][256] digit counts of each group's tiles
  long long ntiles;
  long long n;
  int shift;
  unsigned dmask;              // this pass's digit mask (255, or narrower for the last pass)
  unsigned stamp;              // plan number (30 bits): stale look-back words are ignored
  unsigned long long* trace;   // optional %globaltimer event log (the "trace" option)
  long long trace_cap;
  int* err;                    // device error word (look-back timeout -> EMB_A2A_ETIMEOUT)
  long long timeout_ns;
  int stall;                   // debug: tile 0 publishes a stale stamp (tests the timeout)
  // segmented pass (bwd_onesweep_seg_kernel): tiles never straddle tables
  const int* offsets;          // the plan's CSR offsets: table t's lookups start at offsets[t*B]
  long long B;
  int T;
  const unsigned* shist;       // this pass's [T][NB] per-table digit counts
};

// Cluster plan (sort_mode 4): one thread-block cluster of C CTAs per table generates the keys of
// the table's segment and sorts it by row bits (every LSD pass in one kernel; digit offsets
// exchanged through distributed shared memory, passes separated by cluster barriers).
constexpr int kClusterMaxDB = 11;              // digit bits per pass
struct ClusterSortParams {
  const int* indices;
  const int* offsets;          // absolute CSR offsets [T*B + 1]; table t = [offsets[t*B], ..)
  const float* weights;        // NULL = unweighted
  unsigned* keys[2];           // ping-pong: keygen writes [0]; pass p reads [p&1], writes [p+1&1]
  int* bags[2];
  float* wts[2];
  long long B;
  int C;                       // CTAs per cluster (= per table)
  int rbits;                   // row bits (key = t << rbits | row)
  int passes;                  // LSD passes over the row bits (0 when every row is 0)
  int db;                      // digit bits per pass (the last pass may be narrower)
  unsigned long long* trace;   // optional %globaltimer event log (the "trace" option), NULL = off
  long long trace_cap;
};
cudaError_t launch_sort_plan_cluster(const ClusterSortParams& S, int T, cudaStream_t st);
// Bucket plan (sort_mode 5): after keygen + one onesweep pass on the top 8 key bits, one CTA per
// bucket sorts it by the low bits in shared memory (global memory above `cap` keys).
cudaError_t launch_bucket_sort(const unsigned* keys_in, const int* bags_in, const float* wts_in,
                               unsigned* keys_out, int* bags_out, float* wts_out,
                               const unsigned* hist, int low_bits, int cap, cudaStream_t st);
// CTAs per cluster the cluster plan would use for T tables (0 = cannot launch)
int cluster_plan_size(int T, int db, bool weights);

// The fused backward (exchange + reduce + update) and the unfused reduce share one kernel.
struct BwdParams {
  const float* grad;           // fused: own [b_r][G*D] output gradient; local: [B][T][D] (MP)
  float* stage;                // fused: own staging [B][T][D] for this parity (remote rows)
  const DevPeers* peers;
  unsigned long long* bflags_in;   // own backward arrival counters, src * kFlagStride
  const unsigned long long* bcredits_in;  // own backward credit counters (backwards started)
  const unsigned* keys;        // sorted plan
  const int* bags;
  const float* wts;            // sorted weights (weighted plan) or NULL
  const int* offsets;          // bag lengths for mean pooling
  float* const* tables;        // device array of T fp32 table pointers (updated in place)
  float* scratch;              // [nchunks][2][D] partial sums of runs crossing chunk edges
  unsigned char* info;         // [nchunks] bit 0: owns a crossing run, bit 1: inside one
  unsigned* ticket;            // pass-1 chunk tickets (zeroed before each launch)
  unsigned long long* trace;   // optional %globaltimer event log (the "trace" option), NULL = off
  long long trace_cap;
  int* err;
  long long n;                 // lookups in the plan
  long long B, timeout_ns;
  unsigned long long bepoch;   // 1-based fused-backward number (exchange counters, parity)
  float lr;
  long long nchunks;           // chunks of `chunk` sorted lookups
  int chunk;                   // sorted lookups per pass-1 work unit (a multiple of 32)
  long long wbytes;            // shared memory per warp (finish queue)
  int flist;                   // finish-queue entries per warp
  int W, r, T, D, G, toff, rbits, fused, mean, parity;
  int pdl_fold;                // launch pass 2 with programmatic dependent launch
  long long part[kMaxW + 1];
  int allT[kMaxW];
  int tofs[kMaxW];
};

// mode: 0 auto (onesweep while the tiles fit one wave, else reduce-then-scan), 1 onesweep,
// 2 reduce-then-scan
cudaError_t launch_sort_plan(const SortParams& S, const PassParams* passes, int npasses,
                             long long ntiles, int grid_keygen, int mode, cudaStream_t st);
// Segmented plan: keygen with per-(table, digit) counts, then 2 onesweep passes over row digits
// of seg_db bits, tiles aligned to tables (ntiles_max = ceil(n / tile) + T; surplus CTAs exit).
cudaError_t launch_sort_plan_seg(const SortParams& S, const PassParams* passes, int npasses,
                                 long long ntiles_max, int grid_keygen, cudaStream_t st);
size_t seg_sort_smem(int db, bool weights);
cudaError_t plan_backward(const BwdParams& P, int threads, int share, unsigned* grid,
                          size_t* smem);
cudaError_t launch_backward(const BwdParams& P, unsigned grid, int threads, size_t smem,
                            cudaStream_t st);
// finish-queue entries per warp for dimension D (<= 8 KB of pooled rows); sorted lookups per
// warp work unit
inline int bwd_flist(int D) {
  int c = 2048 / D;
  return c > 16 ? 16 : (c < 2 ? 2 : c);
}
// sorted lookups per pass-1 work unit: 2 sub-batches of 32, 4 for wide rows (fewer crossing
// runs; measured: D=256 415 vs 451 us, D<=128 best at 64)
constexpr int kBwdChunkMin = 64;
inline int bwd_chunk_for(int D) { return D >= 256 ? 128 : 64; }

}  // namespace emba2a
