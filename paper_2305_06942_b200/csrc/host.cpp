// host.cpp -- the C ABI of libemba2a.so (include/emb_a2a.h).
//
// Owns: the symmetric receive region ("symmetric heap"; here a library-owned cudaMalloc
// exported with cudaIpcGetMemHandle), the peer pointer table (roc_shmem_ptr analogue),
// epochs, validation and error state.  Every step of the forward runs in kernels.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "emb_a2a_internal.h"

using namespace emba2a;

namespace {

constexpr uint32_t kMagic = 0xE2BA2A01u;

struct Meta {           // phase-1 all-gather record (problem statement)
  uint32_t magic, abi;
  int32_t rank, world, T, D;
  int64_t B;
  int64_t part[kMaxW + 1];
  int32_t S, dtype, pooling, out_dtype;
};

struct Handles {        // phase-2 all-gather record (symmetric region)
  uint32_t magic;
  int32_t pid;
  int32_t device;
  int32_t pad;
  uint64_t host_id;
  uint64_t raw_ptr;
  uint64_t region_bytes;
  cudaIpcMemHandle_t ipc;
  char bus_id[32];      // PCI bus id of the device: peers on the same physical GPU co-reside
};

uint64_t host_id() {
  char name[256] = {0};
  gethostname(name, sizeof(name) - 1);
  uint64_t h = 1469598103934665603ull;
  for (const char* p = name; *p; ++p) h = (h ^ (uint8_t)*p) * 1099511628211ull;
  return h;
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }
 private:
  int prev_ = 0, dev_ = 0;
};

}  // namespace

struct emb_a2a {
  int rank = 0, W = 1, dev = 0;
  emb_a2a_allgather_fn allgather = nullptr;
  void* user = nullptr;
  bool registered = false, poisoned = false;
  std::string last_error;

  // problem
  int T = 0, D = 0, G = 0, toff = 0;
  int64_t B = 0, b = 0;
  std::vector<int64_t> part;
  std::vector<int32_t> allT;
  std::vector<int64_t> rows;

  // options
  int64_t S = 32, order = 0, threads = 256, timeout_ms = 10000, validate = 0, unroll = 0;
  int64_t delay_ns = 0, skip_to = -1, idx_cap = 2048, stages = 4, ctas_per_sm = 0, tma = 0;
  int64_t stage_kb = 32, vec = 0, pdl = 1, flat_below = 12, rows_early = 1;
  int64_t credit_lag_opt = -1;           // debug: -1 auto (1 iff a peer shares the GPU), 0, 1
  bool tables_dirty = true;              // a table writer may precede the next forward
  bool shared_gpu = false;               // some peer runs on this same GPU
  int64_t chunk = 0;                     // 0 = auto per forward (auto_chunk)
  int64_t trace_cap = 0;                 // records; 0 = tracing off
  unsigned long long* d_trace = nullptr;

  // device state
  char* region = nullptr;
  size_t region_bytes = 0;
  unsigned long long* flags = nullptr;   // own counters
  unsigned long long* credits = nullptr; // own forward credit counters (slot q: written by q)
  unsigned long long* bcredits = nullptr;
  float* recv[2] = {nullptr, nullptr};
  std::vector<void*> opened;             // IPC-opened peer bases
  DevPeers host_peers{};
  DevPeers* d_peers = nullptr;
  const void** d_tables = nullptr;
  int elem = 0;                          // table element type (emb_a2a_dtype)
  int64_t out_dtype = 0;                 // output element type (option "out_dtype", R#32)
  int mean = 0;                          // pooling (emb_a2a_pooling)
  TmaDesc* d_tmaps = nullptr;            // one TMA descriptor per local table
  int ncb = 1, box4 = 1;
  long long* d_rows = nullptr;
  unsigned int* d_done = nullptr;        // [fused done, fused ticket, pool done, pool ticket]
  unsigned long long* d_slice_cnt = nullptr;   // per-slice completed-bag counters
  int* h_err = nullptr;                  // mapped pinned host
  int* d_err = nullptr;
  int* h_verr = nullptr;                 // validate error word (mapped)
  int* d_verr = nullptr;
  // forward_host: double-buffered input staging filled on a copy stream, so the next call's
  // host->device copy overlaps this call's device->host copy (different copy engines)
  int32_t* d_idx_stage[2] = {nullptr, nullptr};
  int32_t* d_off_stage[2] = {nullptr, nullptr};
  size_t idx_stage_cap = 0, off_stage_cap = 0;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  uint64_t host_calls = 0;

  uint64_t epoch = 0;
  uint64_t barrier_epoch = 0;
  int nslices = 0;
  int slice_base[kMaxW + 1] = {0};
  int chunk_base[kMaxW + 1] = {0};
  int C = 8, nchunks = 0;
  int64_t l1_opt = -1;                   // "l1_rows": -1 auto (kL1RowsPerSm), 0 off, 1 on
  int l1_cur = 0;                        // this chunk plan's choice
  int sms = 0;
  int last_grid = 0;
  LaunchPlan plan_fused[2], plan_pool[2]; // cached launch configurations [weighted]
                                          // (fn == nullptr: stale)
  int64_t kernel_launches = 0;

  // backward (f3)
  int64_t bwd_threads = 128, bwd_share = 1, sort_mode = 0, sort_stall = 0;
  int64_t bucket_cap = 4096;             // bucket plan: keys a bucket sorts in shared memory
  int64_t cluster_ctas = 0;              // cluster plan: CTAs per table (0 auto)
  uint64_t bepoch = 0;                   // fused backwards issued (exchange epochs, parity)
  uint32_t plan_no = 0;                  // sort plans (look-back stamps)
  unsigned long long* bflags = nullptr;  // own backward arrival counters
  float* gstage[2] = {nullptr, nullptr}; // own gradient staging [B][T][D] by parity
  unsigned* d_keys[2] = {nullptr, nullptr};
  int* d_bags[2] = {nullptr, nullptr};
  float* d_wts[2] = {nullptr, nullptr};
  size_t plan_cap = 0, wts_cap = 0;
  unsigned* d_hist = nullptr;            // 2 x ([kMaxPasses][256] digit counts + kMaxPasses tile
                                         // tickets) + the backward chunk ticket
  int hist_par = 0;                      // the half the next plan uses (keygen zeroes the other)
  unsigned* d_shist = nullptr;           // segmented plan: 2 x ([2][T][NB] counts + 2 tickets)
  size_t shist_half = 0;                 // words per half
  int last_seg = -1;                     // mode of the previous plan (-1: none yet)
  unsigned* d_cnt = nullptr;             // radix pass: [256][ntiles] tile digit counts
  size_t cnt_cap = 0;
  unsigned long long* d_status = nullptr;  // onesweep look-back words
  unsigned* d_lbg = nullptr;             // onesweep group look-back: [passes][ngroups][1 + 256]
  size_t lbg_cap = 0;
  size_t status_cap = 0;
  float* d_scratch = nullptr;
  unsigned char* d_info = nullptr;       // per-chunk crossing-run flags (backward pass 2)
  size_t chunk_cap = 0;
  bool planned = false, plan_weighted = false;
  int64_t plan_n = 0;
  int plan_buf = 0, rbits = 0;
  const int32_t* plan_offsets = nullptr;
  int bwd_mode = -1;                     // cached launch: mode it was planned for
  unsigned bwd_grid = 0;
  size_t bwd_smem = 0;
};

namespace {

int fail(emb_a2a* h, int code, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    h->last_error = buf;
  }
  return code;
}

#define CUDA_TRY(h, call)                                                                 \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail((h), e_ == cudaErrorMemoryAllocation ? EMB_A2A_ENOMEM : EMB_A2A_ECUDA,  \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);   \
    }                                                                                     \
  } while (0)

// Poll the asynchronous error word; poison the handle on failure.
int check_async(emb_a2a* h) {
  if (h->poisoned) return fail(h, EMB_A2A_ESTATE, "handle poisoned by an earlier failure: %s",
                               h->last_error.c_str());
  if (h->h_err && *(volatile int*)h->h_err != 0) {
    const int v = *(volatile int*)h->h_err;
    h->poisoned = true;
    const char* what =
        (v & 0x4000) ? "backward sort look-back timed out on rank %d (code %d, timeout_ms=%lld): "
                       "a radix tile never published its digit counts"
        : (v & 0x2000) ? "backward credit wait timed out: rank %d waited for rank %d to start its "
                         "previous backward (timeout_ms=%lld)"
        : (v & 0x1000) ? "forward credit wait timed out: rank %d waited for rank %d to start the "
                         "same forward (timeout_ms=%lld)"
        : (v & 0x800) ? "backward chunk fold timed out on rank %d (code %d, timeout_ms=%lld)"
        : (v & 0x400) ? "backward exchange wait timed out: rank %d never received all gradient "
                        "rows from rank %d (timeout_ms=%lld)"
        : (v & 0x200) ? "device barrier timed out on rank %d (code %d, timeout_ms=%lld)"
                      : "receive wait timed out: rank %d never received all slices from "
                        "rank %d (timeout_ms=%lld)";
    return fail(h, EMB_A2A_ETIMEOUT, what, h->rank, v & 0xff, (long long)h->timeout_ms);
  }
  return EMB_A2A_OK;
}

void release_registration(emb_a2a* h) {
  for (void* p : h->opened) cudaIpcCloseMemHandle(p);
  h->opened.clear();
  if (h->region) cudaFree(h->region);
  if (h->d_peers) cudaFree(h->d_peers);
  if (h->d_tables) cudaFree(h->d_tables);
  if (h->d_tmaps) cudaFree(h->d_tmaps);
  h->d_tmaps = nullptr;
  if (h->d_rows) cudaFree(h->d_rows);
  if (h->d_done) cudaFree(h->d_done);
  if (h->d_slice_cnt) cudaFree(h->d_slice_cnt);
  if (h->d_trace) cudaFree(h->d_trace);
  h->d_trace = nullptr;
  h->d_slice_cnt = nullptr;
  for (int x = 0; x < 2; ++x) {
    if (h->d_idx_stage[x]) cudaFree(h->d_idx_stage[x]);
    if (h->d_off_stage[x]) cudaFree(h->d_off_stage[x]);
    h->d_idx_stage[x] = nullptr;
    h->d_off_stage[x] = nullptr;
  }
  for (int x = 0; x < 2; ++x) {
    if (h->d_keys[x]) cudaFree(h->d_keys[x]);
    if (h->d_bags[x]) cudaFree(h->d_bags[x]);
    if (h->d_wts[x]) cudaFree(h->d_wts[x]);
    h->d_keys[x] = nullptr;
    h->d_bags[x] = nullptr;
    h->d_wts[x] = nullptr;
    h->gstage[x] = nullptr;
  }
  h->plan_cap = h->wts_cap = 0;
  if (h->d_hist) cudaFree(h->d_hist);
  if (h->d_shist) cudaFree(h->d_shist);
  h->d_shist = nullptr;
  h->shist_half = 0;
  h->last_seg = -1;
  if (h->d_cnt) cudaFree(h->d_cnt);
  if (h->d_status) cudaFree(h->d_status);
  if (h->d_lbg) cudaFree(h->d_lbg);
  h->d_lbg = nullptr;
  h->d_status = nullptr;
  h->cnt_cap = 0;
  if (h->d_scratch) cudaFree(h->d_scratch);
  if (h->d_info) cudaFree(h->d_info);
  h->d_hist = nullptr;
  h->d_cnt = nullptr;
  h->d_scratch = nullptr;
  h->d_info = nullptr;
  h->status_cap = h->chunk_cap = 0;
  h->planned = false;
  h->bwd_mode = -1;
  h->bflags = nullptr;
  h->region = nullptr;
  h->d_peers = nullptr;
  h->d_tables = nullptr;
  h->d_rows = nullptr;
  h->d_done = nullptr;
  h->idx_stage_cap = h->off_stage_cap = 0;
  h->flags = nullptr;
  h->credits = h->bcredits = nullptr;
  h->recv[0] = h->recv[1] = nullptr;
  h->registered = false;
}

int barrier(emb_a2a* h) {
  std::vector<char> recv(h->W);
  char one = 1;
  if (h->allgather(&one, recv.data(), 1, h->user) != 0)
    return fail(h, EMB_A2A_EBOOT, "all-gather callback failed (barrier)");
  return EMB_A2A_OK;
}

// Chunk size (bags per work unit): the "chunk" option, at most 127 (the producer keeps a chunk's
// offsets in four registers per lane).  Chunks and slices are independent: a stage's bags count
// toward every slice they fall in (fused_kernel.cuh recycle).
int chunk_size(int64_t S, int64_t want) {
  (void)S;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, 127));
}

// Chunk size when the "chunk" option is 0 (default): about 640 lookups per work unit from this
// forward's average bag length, 32..127 bags.  Measured (r02u, one B200, per-rank work at W=1):
// short bags need long chunks (sweep P=1: 31.5 us at 32 bags -> 23.2 us at 127; P=4 44.1 ->
// 41.7), long bags short ones (DLRM-small 12.9 us at 32 vs 14.3 at 64; weak 19.4 vs 23.0;
// DLRM-wide 193 vs 203).  Chunks are rank-local work units: no peer needs to agree.
int auto_chunk(const emb_a2a* h, int64_t nnz) {
  const int64_t bags = (int64_t)h->T * h->B;
  if (bags <= 0 || nnz <= 0) return 127;
  return (int)std::max<int64_t>(32, std::min<int64_t>(127, (640 * bags) / nnz));
}

// Slice and chunk counts per destination ordinal (row a1): T * ceil(b_s / unit).
void compute_slices(emb_a2a* h, int C) {
  h->C = C;
  int64_t acc = 0, accc = 0;
  for (int k = 0; k < h->W; ++k) {
    h->slice_base[k] = (int)acc;
    h->chunk_base[k] = (int)accc;
    const int s = dest_of_ordinal((int)h->order, h->rank, h->W, k);
    const int64_t bs = h->part[s + 1] - h->part[s];
    acc += (int64_t)h->T * ((bs + h->S - 1) / h->S);
    accc += (int64_t)h->T * ((bs + h->C - 1) / h->C);
  }
  h->slice_base[h->W] = (int)acc;
  h->chunk_base[h->W] = (int)accc;
  h->nslices = (int)acc;
  h->nchunks = (int)accc;
  for (int q = 0; q < h->W; ++q) {
    const int64_t nsl = (h->b + h->S - 1) / h->S;
    h->host_peers.n_in[q] = (q == h->rank) ? 0 : (long long)h->allT[q] * nsl;
  }
}

// Re-derive the chunk plan when this forward's chunk size differs from the last one (the
// cached launch configurations depend on it: grid = min(slots, chunks), stage layout).
void ensure_chunk(emb_a2a* h, int64_t nnz) {
  const int C = h->chunk > 0 ? chunk_size(h->S, h->chunk) : auto_chunk(h, nnz);
  if (h->sms <= 0) cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev);
  const int l1 = h->l1_opt >= 0 ? (int)h->l1_opt
                                : ((nnz >= kL1RowsPerSm * std::max(h->sms, 1) ||
                                    (long long)h->B >= kL1RowsBags) ? 1 : 0);
  if (C == h->C && l1 == h->l1_cur) return;
  h->l1_cur = l1;
  if (C != h->C) compute_slices(h, C);
  for (int w = 0; w < 2; ++w) {
    h->plan_fused[w] = LaunchPlan();
    h->plan_pool[w] = LaunchPlan();
  }
}

KParams make_params(emb_a2a* h, const int32_t* indices, const int32_t* offsets,
                    const float* weights) {
  KParams P;
  memset(&P, 0, sizeof(P));
  P.indices = indices;
  P.offsets = offsets;
  P.weights = weights;
  P.elem = h->elem;
  P.mean = h->mean;
  P.out_dtype = (int)h->out_dtype;
  P.oshift = h->out_dtype == EMB_A2A_F32 ? 2 : 1;
  P.tables = h->d_tables;
  P.tmaps = h->d_tmaps;
  P.tma = (h->tma && h->elem == 0 && !weights) ? 1 : 0;   // TMA gather: fp32, unweighted
  P.ncb = h->ncb;
  P.box4 = h->box4;
  P.peers = h->d_peers;
  P.flags_in = h->flags;
  P.credits_in = h->credits;
  P.done = h->d_done;
  P.ticket = h->d_done + 1;
  P.err = h->d_err;
  P.trace = h->d_trace;
  P.trace_cap = h->trace_cap;
  P.B = h->B;
  P.epoch = h->epoch;
  P.timeout_ns = (long long)h->timeout_ms * 1000000ll;
  P.delay_ns = h->delay_ns;
  P.W = h->W;
  P.r = h->rank;
  P.T = h->T;
  P.D = h->D;
  P.DU = h->D * (h->elem == 0 ? 4 : 2) / 16;
  P.G = h->G;
  P.toff = h->toff;
  P.S = (int)h->S;
  P.order = (int)h->order;
  P.nslices = h->nslices;
  P.C = h->C;
  P.nchunks = h->nchunks;
  P.slice_cnt = h->d_slice_cnt;
  P.nstages = (int)h->stages;
  P.pdl = (int)h->pdl;
  P.rows_wait = 1;
  P.pdl_trigger = (h->W > 1 && h->shared_gpu && h->rows_early != 2) ? 0 : 1;
  // A peer on this very GPU (virtual ranks, test mode) only has to have started the previous
  // forward: waiting for the same forward could park our persistent grid on SM slots the
  // peer's kernel needs.  That keeps the weaker contract (a consumer ordered before our next
  // forward); one GPU per rank gives the full one (output valid until the second following
  // forward).
  P.credit_lag = h->credit_lag_opt >= 0 ? (int)h->credit_lag_opt : (h->shared_gpu ? 1 : 0);
  P.flat_below = (int)h->flat_below;
  P.l1rows = h->l1_cur;
  P.skip_to = (int)h->skip_to;
  P.parity = (int)(h->epoch & 1);
  stage_layout(P, (int)h->stage_kb, (int)h->idx_cap);
  for (int s = 0; s <= h->W; ++s) {
    P.part[s] = h->part[s];
    P.slice_base[s] = h->slice_base[s];
    P.chunk_base[s] = h->chunk_base[s];
  }
  return P;
}

// TMA descriptors for the local tables: 2-D [rows][D] fp32, box {box, 1} so that one
// tile::gather4 moves 4 arbitrary rows x box columns.  box = D / ncb <= 256 elements.
int make_tensor_maps(emb_a2a* h, const void* const* tables) {
  h->ncb = 1;
  if (h->elem != 0) return EMB_A2A_OK;   // TMA gather mode is fp32-only
  while (h->D / h->ncb > 256 || h->D % h->ncb != 0 || (h->D / h->ncb) % 4 != 0) ++h->ncb;
  h->box4 = h->D / h->ncb / 4;
  if (h->T == 0) return EMB_A2A_OK;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return fail(h, EMB_A2A_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  std::vector<TmaDesc> maps(h->T);
  for (int t = 0; t < h->T; ++t) {
    cuuint64_t gdim[2] = {(cuuint64_t)h->D, (cuuint64_t)h->rows[t]};
    cuuint64_t gstride[1] = {(cuuint64_t)h->D * 4};
    cuuint32_t box[2] = {(cuuint32_t)(h->box4 * 4), 1};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(&maps[t]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        2, const_cast<void*>(tables[t]), gdim, gstride, box, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(h, EMB_A2A_EINVAL, "cuTensorMapEncodeTiled(table %d) failed (%d)", t, (int)r);
  }
  CUDA_TRY(h, cudaMalloc((void**)&h->d_tmaps, sizeof(TmaDesc) * h->T));
  CUDA_TRY(h, cudaMemcpy(h->d_tmaps, maps.data(), sizeof(TmaDesc) * h->T,
                         cudaMemcpyHostToDevice));
  return EMB_A2A_OK;
}

int push_peers(emb_a2a* h) {
  CUDA_TRY(h, cudaMemcpy(h->d_peers, &h->host_peers, sizeof(DevPeers), cudaMemcpyHostToDevice));
  return EMB_A2A_OK;
}

int run_validate(emb_a2a* h, const int32_t* indices, const int32_t* offsets, int64_t nnz,
                 cudaStream_t st) {
  *(volatile int*)h->h_verr = 0;
  CUDA_TRY(h, launch_validate(indices, offsets, nnz, (long long)h->T * h->B, h->B, h->T,
                              h->d_rows, h->d_verr, st));
  h->kernel_launches++;
  CUDA_TRY(h, cudaStreamSynchronize(st));
  const int v = *(volatile int*)h->h_verr;
  if (v) return fail(h, EMB_A2A_EINDEX, v == 1 ? "malformed offsets" : "index out of range");
  return EMB_A2A_OK;
}

}  // namespace

extern "C" {

int emb_a2a_abi_version(void) { return EMB_A2A_ABI_VERSION; }

const char* emb_a2a_status_string(int s) {
  switch (s) {
    case EMB_A2A_OK: return "EMB_A2A_OK";
    case EMB_A2A_EINVAL: return "EMB_A2A_EINVAL";
    case EMB_A2A_ESTATE: return "EMB_A2A_ESTATE";
    case EMB_A2A_ECUDA: return "EMB_A2A_ECUDA";
    case EMB_A2A_ENOMEM: return "EMB_A2A_ENOMEM";
    case EMB_A2A_EPEER: return "EMB_A2A_EPEER";
    case EMB_A2A_EBOOT: return "EMB_A2A_EBOOT";
    case EMB_A2A_ETIMEOUT: return "EMB_A2A_ETIMEOUT";
    case EMB_A2A_EINDEX: return "EMB_A2A_EINDEX";
    default: return "EMB_A2A_UNKNOWN";
  }
}

const char* emb_a2a_last_error(const emb_a2a_t* h) {
  return h ? h->last_error.c_str() : "null handle";
}

int emb_a2a_init(int rank, int world_size, int cuda_device, emb_a2a_allgather_fn allgather,
                 void* user, emb_a2a_t** out) {
  if (!out) return EMB_A2A_EINVAL;
  *out = nullptr;
  if (world_size < 1 || world_size > kMaxW || rank < 0 || rank >= world_size || !allgather)
    return EMB_A2A_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
    return EMB_A2A_ECUDA;
  emb_a2a* h = new emb_a2a();
  h->rank = rank;
  h->W = world_size;
  h->dev = cuda_device;
  h->allgather = allgather;
  h->user = user;
  DeviceGuard g(cuda_device);
  cudaError_t e = cudaHostAlloc((void**)&h->h_err, 2 * sizeof(int), cudaHostAllocMapped);
  if (e != cudaSuccess) {
    delete h;
    return EMB_A2A_ENOMEM;
  }
  h->h_err[0] = h->h_err[1] = 0;
  h->h_verr = h->h_err + 1;
  if (cudaHostGetDevicePointer((void**)&h->d_err, h->h_err, 0) != cudaSuccess) {
    cudaFreeHost(h->h_err);
    delete h;
    return EMB_A2A_ECUDA;
  }
  h->d_verr = h->d_err + 1;
  *out = h;
  return EMB_A2A_OK;
}

static int register_impl(emb_a2a_t* h, int num_local_tables, const void* const* tables,
                         const int64_t* rows, int dim, int table_dtype, int pooling,
                         int64_t global_batch, const int64_t* batch_partition);

int emb_a2a_register_tables(emb_a2a_t* h, int num_local_tables, const float* const* tables,
                            const int64_t* rows, int dim, int64_t global_batch,
                            const int64_t* batch_partition) {
  return emb_a2a_register_tables_ex(h, num_local_tables, (const void* const*)tables, rows, dim,
                                    EMB_A2A_F32, EMB_A2A_SUM, global_batch, batch_partition);
}

int emb_a2a_register_tables_ex(emb_a2a_t* h, int num_local_tables, const void* const* tables,
                               const int64_t* rows, int dim, int table_dtype, int pooling,
                               int64_t global_batch, const int64_t* batch_partition) {
  if (!h) return EMB_A2A_EINVAL;
  const int rc = register_impl(h, num_local_tables, tables, rows, dim, table_dtype, pooling,
                               global_batch, batch_partition);
  if (rc != EMB_A2A_OK && !h->registered) {
    DeviceGuard guard(h->dev);
    release_registration(h);
  }
  return rc;
}

static int register_impl(emb_a2a_t* h, int num_local_tables, const void* const* tables,
                         const int64_t* rows, int dim, int table_dtype, int pooling,
                         int64_t global_batch, const int64_t* batch_partition) {
  if (h->poisoned) return check_async(h);
  DeviceGuard guard(h->dev);
  if (h->registered) {   // collective re-registration: quiesce, barrier, tear down
    cudaDeviceSynchronize();
    int rc = barrier(h);
    if (rc) return rc;
    release_registration(h);
  }
  // ---- local validation (identical decisions on every rank would be ideal; metadata
  //      mismatches are caught after the all-gather so every rank returns EINVAL together)
  int bad = 0;
  if (num_local_tables < 0 || (num_local_tables > 0 && (!tables || !rows))) bad = 1;
  if (table_dtype < EMB_A2A_F32 || table_dtype > EMB_A2A_F16) bad = 1;
  if (pooling != EMB_A2A_SUM && pooling != EMB_A2A_MEAN) bad = 1;
  const int esize = table_dtype == EMB_A2A_F32 ? 4 : 2;
  if (dim < 4 || dim > 1024 || (dim * esize) % 16 != 0) bad = 1;   // whole 16-byte units (R#9)
  if (global_batch < 0) bad = 1;
  for (int t = 0; !bad && t < num_local_tables; ++t) {
    if (rows[t] < 1 || rows[t] >= (1ll << 31)) bad = 1;
    if (((uintptr_t)tables[t]) % 16 != 0 || !tables[t]) bad = 1;
  }
  Meta me;
  memset(&me, 0, sizeof(me));
  me.magic = kMagic;
  me.abi = EMB_A2A_ABI_VERSION;
  me.rank = h->rank;
  me.world = h->W;
  me.T = num_local_tables;
  me.D = dim;
  me.B = global_batch;
  me.S = (int32_t)h->S;
  me.dtype = table_dtype;
  me.pooling = pooling;
  me.out_dtype = (int32_t)h->out_dtype;
  if (batch_partition) {
    for (int s = 0; s <= h->W; ++s) me.part[s] = batch_partition[s];
  } else if (h->W > 0 && global_batch % h->W == 0) {
    for (int s = 0; s <= h->W; ++s) me.part[s] = global_batch / h->W * s;
  } else {
    bad = 1;
  }
  if (me.part[0] != 0 || me.part[h->W] != global_batch) bad = 1;
  for (int s = 0; s < h->W; ++s)
    if (me.part[s + 1] < me.part[s]) bad = 1;
  if (bad) me.magic = 0;   // tell everyone

  std::vector<Meta> all(h->W);
  if (h->allgather(&me, all.data(), sizeof(Meta), h->user) != 0)
    return fail(h, EMB_A2A_EBOOT, "all-gather callback failed (metadata)");
  int64_t G = 0;
  for (int q = 0; q < h->W; ++q) {
    const Meta& m = all[q];
    if (m.magic != kMagic || m.abi != EMB_A2A_ABI_VERSION || m.rank != q || m.world != h->W)
      return fail(h, EMB_A2A_EINVAL, "rank %d sent invalid registration arguments", q);
    if (m.D != dim || m.B != global_batch || m.S != (int32_t)h->S || m.dtype != table_dtype ||
        m.pooling != pooling || m.out_dtype != (int32_t)h->out_dtype ||
        memcmp(m.part, me.part, sizeof(int64_t) * (h->W + 1)) != 0)
      return fail(h, EMB_A2A_EINVAL,
                  "ranks disagree on dim / global batch / partition / slice / dtypes (rank %d)", q);
    G += m.T;
  }
  if (G < 1) return fail(h, EMB_A2A_EINVAL, "no tables registered on any rank");
  int64_t nnz_tb = (int64_t)num_local_tables * global_batch;
  if (nnz_tb + 1 >= (1ll << 31) || G * (int64_t)dim >= (1ll << 31))
    return fail(h, EMB_A2A_EINVAL, "T*B or G*D too large for int32 CSR / layout (R#8)");

  h->T = num_local_tables;
  h->D = dim;
  h->elem = table_dtype;
  h->mean = pooling == EMB_A2A_MEAN ? 1 : 0;
  h->B = global_batch;
  h->G = (int)G;
  h->part.assign(me.part, me.part + h->W + 1);
  h->b = h->part[h->rank + 1] - h->part[h->rank];
  h->allT.resize(h->W);
  h->toff = 0;
  for (int q = 0; q < h->W; ++q) {
    h->allT[q] = all[q].T;
    if (q < h->rank) h->toff += all[q].T;
  }
  h->rows.assign(rows, rows + num_local_tables);

  // ---- symmetric region: [forward arrival counters W x 128 B | barrier counter 128 B |
  //      backward arrival counters W x 128 B | forward credits W x 128 B | backward credits
  //      W x 128 B | recv0 | recv1 | gstage0 | gstage1], 256-B aligned pieces.  gstage
  //      (backward, fp32 tables only): [B][T_r][D] float32 gradient rows pushed by their
  //      data-parallel owners.  Credits: slot q counts the forwards (backwards) rank q started.
  const size_t flag_bytes = ((size_t)(4 * h->W + 1) * kFlagStride * 8 + 255) / 256 * 256;
  const size_t oes = h->out_dtype == EMB_A2A_F32 ? 4 : 2;   // output element size (R#32)
  const size_t buf_bytes = ((size_t)h->b * G * dim * oes + 255) / 256 * 256;
  auto gstage_bytes = [&](int Tq) -> size_t {
    if (table_dtype != EMB_A2A_F32) return 256;
    return std::max<size_t>(((size_t)Tq * global_batch * dim * 4 + 255) / 256 * 256, 256);
  };
  const size_t gsz = gstage_bytes(num_local_tables);
  h->region_bytes = flag_bytes + 2 * std::max<size_t>(buf_bytes, 256) + 2 * gsz;
  CUDA_TRY(h, cudaMalloc((void**)&h->region, h->region_bytes));
  CUDA_TRY(h, cudaMemset(h->region, 0, h->region_bytes));
  h->flags = (unsigned long long*)h->region;
  h->bflags = h->flags + (size_t)(h->W + 1) * kFlagStride;
  h->credits = h->flags + (size_t)(2 * h->W + 1) * kFlagStride;
  h->bcredits = h->flags + (size_t)(3 * h->W + 1) * kFlagStride;
  h->recv[0] = (float*)(h->region + flag_bytes);
  h->recv[1] = (float*)(h->region + flag_bytes + std::max<size_t>(buf_bytes, 256));
  h->gstage[0] = (float*)(h->region + flag_bytes + 2 * std::max<size_t>(buf_bytes, 256));
  h->gstage[1] = (float*)((char*)h->gstage[0] + gsz);

  Handles mine;
  memset(&mine, 0, sizeof(mine));
  mine.magic = kMagic;
  mine.pid = (int32_t)getpid();
  mine.device = h->dev;
  cudaDeviceGetPCIBusId(mine.bus_id, sizeof(mine.bus_id), h->dev);
  mine.host_id = host_id();
  mine.raw_ptr = (uint64_t)(uintptr_t)h->region;
  mine.region_bytes = h->region_bytes;
  CUDA_TRY(h, cudaIpcGetMemHandle(&mine.ipc, h->region));
  std::vector<Handles> hs(h->W);
  if (h->allgather(&mine, hs.data(), sizeof(Handles), h->user) != 0)
    return fail(h, EMB_A2A_EBOOT, "all-gather callback failed (handles)");

  // ---- map every peer (roc_shmem_ptr gives the peer's virtual address)
  memset(&h->host_peers, 0, sizeof(DevPeers));
  h->shared_gpu = false;
  for (int q = 0; q < h->W; ++q) {
    char* base = nullptr;
    const Handles& o = hs[q];
    if (q != h->rank && o.host_id == mine.host_id &&
        strncmp(o.bus_id, mine.bus_id, sizeof(mine.bus_id)) == 0)
      h->shared_gpu = true;   // a peer on this very GPU (virtual ranks / shared-GPU test mode)
    if (q == h->rank) {
      base = h->region;
    } else if (o.pid == mine.pid && o.host_id == mine.host_id) {
      base = (char*)(uintptr_t)o.raw_ptr;     // same process: raw pointer (loopback / threads)
      if (o.device != h->dev) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, h->dev, o.device);
        if (!can) return fail(h, EMB_A2A_EPEER, "no P2P path from device %d to %d", h->dev,
                              o.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(h, EMB_A2A_EPEER, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
        cudaGetLastError();
      }
    } else {
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, o.ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        return fail(h, EMB_A2A_EPEER, "cudaIpcOpenMemHandle(rank %d): %s", q,
                    cudaGetErrorString(e));
      h->opened.push_back(p);
      base = (char*)p;
    }
    const int64_t bq = h->part[q + 1] - h->part[q];
    const size_t fq = flag_bytes;   // identical layout on every rank (same W)
    const size_t bufq = std::max<size_t>(((size_t)bq * G * dim * oes + 255) / 256 * 256, 256);
    h->host_peers.recv[q][0] = (float*)(base + fq);
    h->host_peers.recv[q][1] = (float*)(base + fq + bufq);
    h->host_peers.flag_out[q] = (unsigned long long*)(base) + (size_t)h->rank * kFlagStride;
    h->host_peers.barrier_out[q] = (unsigned long long*)(base) + (size_t)h->W * kFlagStride;
    h->host_peers.bflag_out[q] =
        (unsigned long long*)(base) + (size_t)(h->W + 1 + h->rank) * kFlagStride;
    h->host_peers.credit_out[q] =
        (unsigned long long*)(base) + (size_t)(2 * h->W + 1 + h->rank) * kFlagStride;
    h->host_peers.bcredit_out[q] =
        (unsigned long long*)(base) + (size_t)(3 * h->W + 1 + h->rank) * kFlagStride;
    h->host_peers.gstage[q][0] = (float*)(base + fq + 2 * bufq);
    h->host_peers.gstage[q][1] = (float*)(base + fq + 2 * bufq + gstage_bytes(all[q].T));
  }

  // ---- device-side tables, plan, counters
  CUDA_TRY(h, cudaMalloc((void**)&h->d_peers, sizeof(DevPeers)));
  CUDA_TRY(h, cudaMalloc((void**)&h->d_tables, sizeof(void*) * std::max(1, h->T)));
  CUDA_TRY(h, cudaMalloc((void**)&h->d_rows, sizeof(long long) * std::max(1, h->T)));
  CUDA_TRY(h, cudaMalloc((void**)&h->d_done, 4 * sizeof(unsigned int)));
  CUDA_TRY(h, cudaMemset(h->d_done, 0, 4 * sizeof(unsigned int)));
  if (h->T > 0) {
    CUDA_TRY(h, cudaMemcpy(h->d_tables, tables, sizeof(void*) * h->T, cudaMemcpyHostToDevice));
    std::vector<long long> r64(rows, rows + h->T);
    CUDA_TRY(h, cudaMemcpy(h->d_rows, r64.data(), sizeof(long long) * h->T,
                           cudaMemcpyHostToDevice));
  }
  compute_slices(h, h->chunk > 0 ? chunk_size(h->S, h->chunk) : 32);
  {
    const int rc_maps = make_tensor_maps(h, tables);
    if (rc_maps) return rc_maps;
  }
  CUDA_TRY(h, cudaMalloc((void**)&h->d_slice_cnt, sizeof(unsigned long long) *
                                                      std::max(1, h->nslices)));
  CUDA_TRY(h, cudaMemset(h->d_slice_cnt, 0, sizeof(unsigned long long) *
                                               std::max(1, h->nslices)));
  int rc = push_peers(h);
  if (rc) return rc;
  CUDA_TRY(h, cudaDeviceSynchronize());
  h->epoch = 0;
  h->barrier_epoch = 0;
  h->bepoch = 0;
  h->planned = false;
  h->bwd_mode = -1;
  h->tables_dirty = true;
  for (int w = 0; w < 2; ++w) {
    h->plan_fused[w] = LaunchPlan();
    h->plan_pool[w] = LaunchPlan();
  }
  h->registered = true;
  return barrier(h);   // nobody forwards before everyone has mapped everyone
}

int emb_a2a_forward(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                    int64_t num_indices, void* stream, float** out, int64_t* out_rows,
                    int64_t* out_cols) {
  return emb_a2a_forward_weighted(h, indices, offsets, nullptr, num_indices, stream, out,
                                  out_rows, out_cols);
}

int emb_a2a_forward_weighted(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                             const float* weights, int64_t num_indices, void* stream,
                             float** out, int64_t* out_rows, int64_t* out_cols) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "forward before register_tables");
  if (!out) return fail(h, EMB_A2A_EINVAL, "out is NULL");
  if (num_indices < 0 || num_indices >= (1ll << 31))
    return fail(h, EMB_A2A_EINVAL, "num_indices out of range (int32 CSR, R#8)");
  if ((h->T > 0 && h->B > 0) && (!offsets || (num_indices > 0 && !indices)))
    return fail(h, EMB_A2A_EINVAL, "indices/offsets are NULL");
  DeviceGuard guard(h->dev);
  cudaStream_t st = (cudaStream_t)stream;
  if (h->validate && h->T > 0 && h->B > 0) {
    rc = run_validate(h, indices, offsets, num_indices, st);
    if (rc) return rc;
  }
  if (weights && h->mean)
    return fail(h, EMB_A2A_EINVAL, "per-sample weights need sum pooling (R#26)");
  if (weights && num_indices > 0 && ((uintptr_t)weights % 4))
    return fail(h, EMB_A2A_EINVAL, "weights must be 4-byte aligned");
  h->epoch += 1;
  const float* w = num_indices > 0 ? weights : nullptr;
  ensure_chunk(h, num_indices);
  KParams P = make_params(h, indices, offsets, w);
  // consumers may gather rows and store before the predecessor completes when no backward of
  // this handle (the only table writer) ran since the previous forward; with peers, the
  // producer holds back the one stage it publishes before its own wait until the destination
  // peer has provably consumed the buffer half (fused_kernel.cuh)
  // (not when a peer shares this GPU: a stage held back for that peer would keep CTAs resident
  // that the peer's own forward may need)
  // ("pdl_rows_early" = 2 forces it on a shared GPU too: tests, with grids small enough to
  // co-reside)
  P.rows_wait = (h->tables_dirty || !h->rows_early ||
                 (h->W > 1 && h->shared_gpu && h->rows_early != 2)) ? 1 : 0;
  h->tables_dirty = false;
  LaunchPlan& pl = h->plan_fused[w ? 1 : 0];
  cudaError_t e = cudaSuccess;
  if (!pl.fn) {
    LaunchCfg c{(int)h->threads, (int)h->vec, (int)h->ctas_per_sm};
    e = plan_fused(P, c, &pl);
  }
  if (e == cudaSuccess) e = launch_planned(pl, P, st);
  h->last_grid = (int)pl.grid;
  if (e != cudaSuccess) {
    h->poisoned = true;
    return fail(h, EMB_A2A_ECUDA, "fused kernel launch: %s", cudaGetErrorString(e));
  }
  h->kernel_launches++;
  *out = h->recv[h->epoch & 1];
  if (out_rows) *out_rows = h->b;
  if (out_cols) *out_cols = (int64_t)h->G * h->D;
  return EMB_A2A_OK;
}

}  // extern "C"

namespace {

// forward_host plumbing: copy streams, events, double-buffered input staging (grow-only).
int host_staging(emb_a2a* h, int64_t num_indices) {
  const size_t nidx = (size_t)std::max<int64_t>(num_indices, 1);
  const size_t noff = (size_t)h->T * h->B + 1;
  if (!h->h2d_stream) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking));
    CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
    for (int x = 0; x < 2; ++x) {
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_free[x], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_done[x], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_out[x], cudaEventDisableTiming));
    }
  }
  // grow-only with headroom: batches vary in size, and cudaFree synchronises the device
  if (nidx > h->idx_stage_cap || noff > h->off_stage_cap) {
    // a regrow waits for earlier calls' copies and forwards (the first call has nothing to
    // wait for -- and must not wait: loopback peers' forwards may still be in flight)
    if (h->idx_stage_cap > 0) CUDA_TRY(h, cudaDeviceSynchronize());
    const size_t icap = std::max(h->idx_stage_cap, nidx + nidx / 4);
    const size_t ocap = std::max(h->off_stage_cap, noff);
    for (int x = 0; x < 2; ++x) {
      if (h->d_idx_stage[x]) cudaFree(h->d_idx_stage[x]);
      if (h->d_off_stage[x]) cudaFree(h->d_off_stage[x]);
      h->d_idx_stage[x] = nullptr;
      h->d_off_stage[x] = nullptr;
    }
    h->idx_stage_cap = h->off_stage_cap = 0;
    for (int x = 0; x < 2; ++x) {
      CUDA_TRY(h, cudaMalloc((void**)&h->d_idx_stage[x], icap * sizeof(int32_t)));
      CUDA_TRY(h, cudaMalloc((void**)&h->d_off_stage[x], ocap * sizeof(int32_t)));
    }
    h->idx_stage_cap = icap;
    h->off_stage_cap = ocap;
  }
  return EMB_A2A_OK;
}

}  // namespace

extern "C" {

int emb_a2a_forward_host(emb_a2a_t* h, const int32_t* h_indices, const int32_t* h_offsets,
                         int64_t num_indices, void* stream, float* h_out) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "forward_host before register_tables");
  if (num_indices < 0 || num_indices >= (1ll << 31))
    return fail(h, EMB_A2A_EINVAL, "num_indices out of range");
  if (!h_out || (!h_offsets && h->T > 0 && h->B > 0) || (num_indices > 0 && !h_indices))
    return fail(h, EMB_A2A_EINVAL, "host buffers are NULL");
  DeviceGuard guard(h->dev);
  cudaStream_t st = (cudaStream_t)stream;
  rc = host_staging(h, num_indices);
  if (rc) return rc;
  const size_t noff = (size_t)h->T * h->B + 1;
  {
  }
  const int par = (int)(h->host_calls++ & 1);
  // staging[par] was last read by the forward two calls ago (ev_free[par]); the copy stream
  // does not wait for this stream's device->host copy of the previous call
  CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_free[par], 0));
  if (num_indices > 0)
    CUDA_TRY(h, cudaMemcpyAsync(h->d_idx_stage[par], h_indices, num_indices * sizeof(int32_t),
                                cudaMemcpyHostToDevice, h->h2d_stream));
  if (h->T > 0 && h->B > 0)
    CUDA_TRY(h, cudaMemcpyAsync(h->d_off_stage[par], h_offsets, noff * sizeof(int32_t),
                                cudaMemcpyHostToDevice, h->h2d_stream));
  CUDA_TRY(h, cudaEventRecord(h->ev_in, h->h2d_stream));
  CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_in, 0));
  float* dout = nullptr;
  rc = emb_a2a_forward(h, h->d_idx_stage[par], h->d_off_stage[par], num_indices, stream, &dout,
                       nullptr, nullptr);
  if (rc) return rc;
  CUDA_TRY(h, cudaEventRecord(h->ev_free[par], st));
  const size_t out_bytes = (size_t)h->b * h->G * h->D * (h->out_dtype == EMB_A2A_F32 ? 4 : 2);
  if (out_bytes) CUDA_TRY(h, cudaMemcpyAsync(h_out, dout, out_bytes, cudaMemcpyDeviceToHost, st));
  return EMB_A2A_OK;
}

int emb_a2a_forward_host_batch(emb_a2a_t* h, int nsteps, const int32_t* const* h_indices,
                               const int32_t* const* h_offsets, const int64_t* num_indices,
                               float* const* h_out, void* stream) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "forward_host_batch before register_tables");
  if (nsteps < 0 || (nsteps > 0 && (!h_indices || !h_offsets || !num_indices || !h_out)))
    return fail(h, EMB_A2A_EINVAL, "bad step arrays");
  int64_t nmax = 0;
  for (int k = 0; k < nsteps; ++k) {
    if (num_indices[k] < 0 || num_indices[k] >= (1ll << 31))
      return fail(h, EMB_A2A_EINVAL, "num_indices[%d] out of range", k);
    if (!h_out[k] || (!h_offsets[k] && h->T > 0 && h->B > 0) ||
        (num_indices[k] > 0 && !h_indices[k]))
      return fail(h, EMB_A2A_EINVAL, "host buffers of step %d are NULL", k);
    nmax = std::max(nmax, num_indices[k]);
  }
  DeviceGuard guard(h->dev);
  cudaStream_t st = (cudaStream_t)stream;
  rc = host_staging(h, nmax);
  if (rc) return rc;
  const size_t noff = (size_t)h->T * h->B + 1;
  const size_t out_bytes = (size_t)h->b * h->G * h->D * (h->out_dtype == EMB_A2A_F32 ? 4 : 2);
  for (int k = 0; k < nsteps; ++k) {
    const int par = (int)(h->host_calls++ & 1);
    // inputs: copy stream, into the staging the forward two steps ago has finished reading
    CUDA_TRY(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_free[par], 0));
    if (num_indices[k] > 0)
      CUDA_TRY(h, cudaMemcpyAsync(h->d_idx_stage[par], h_indices[k],
                                  num_indices[k] * sizeof(int32_t), cudaMemcpyHostToDevice,
                                  h->h2d_stream));
    if (h->T > 0 && h->B > 0)
      CUDA_TRY(h, cudaMemcpyAsync(h->d_off_stage[par], h_offsets[k], noff * sizeof(int32_t),
                                  cudaMemcpyHostToDevice, h->h2d_stream));
    CUDA_TRY(h, cudaEventRecord(h->ev_in, h->h2d_stream));
    // forward on `stream`, once the inputs are in and the receive buffer it will write (the
    // one of two steps ago) has been copied out
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_in, 0));
    CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_out[(h->epoch + 1) & 1], 0));
    // a peer on this same GPU only waits for our previous forward (credit_lag 1): the copy of
    // the previous step's result must then be out before this forward starts
    if (h->W > 1 && h->shared_gpu)
      CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_out[h->epoch & 1], 0));
    float* dout = nullptr;
    rc = emb_a2a_forward(h, h->d_idx_stage[par], h->d_off_stage[par], num_indices[k], stream,
                         &dout, nullptr, nullptr);
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_free[par], st));
    CUDA_TRY(h, cudaEventRecord(h->ev_done[h->epoch & 1], st));
    // result: device->host on the other copy stream, overlapping the next step's forward
    CUDA_TRY(h, cudaStreamWaitEvent(h->d2h_stream, h->ev_done[h->epoch & 1], 0));
    if (out_bytes)
      CUDA_TRY(h, cudaMemcpyAsync(h_out[k], dout, out_bytes, cudaMemcpyDeviceToHost,
                                  h->d2h_stream));
    CUDA_TRY(h, cudaEventRecord(h->ev_out[h->epoch & 1], h->d2h_stream));
  }
  // `stream` completes only after every result copy
  for (int x = 0; x < 2; ++x) CUDA_TRY(h, cudaStreamWaitEvent(st, h->ev_out[x], 0));
  return EMB_A2A_OK;
}

int emb_a2a_pool_local(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                       int64_t num_indices, void* stream, float* send) {
  return emb_a2a_pool_local_weighted(h, indices, offsets, nullptr, num_indices, stream, send);
}

int emb_a2a_pool_local_weighted(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                                const float* weights, int64_t num_indices, void* stream,
                                float* send) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "pool_local before register_tables");
  if (num_indices < 0 || num_indices >= (1ll << 31))
    return fail(h, EMB_A2A_EINVAL, "num_indices out of range");
  if (h->T > 0 && h->B > 0 && (!send || !offsets || (num_indices > 0 && !indices)))
    return fail(h, EMB_A2A_EINVAL, "NULL buffer");
  DeviceGuard guard(h->dev);
  cudaStream_t st = (cudaStream_t)stream;
  if (h->validate && h->T > 0 && h->B > 0) {
    rc = run_validate(h, indices, offsets, num_indices, st);
    if (rc) return rc;
  }
  if (weights && h->mean)
    return fail(h, EMB_A2A_EINVAL, "per-sample weights need sum pooling (R#26)");
  const float* w = num_indices > 0 ? weights : nullptr;
  ensure_chunk(h, num_indices);
  KParams P = make_params(h, indices, offsets, w);
  P.send = send;
  P.done = h->d_done + 2;      // own counters: may run concurrently with a forward's kernel
  P.ticket = h->d_done + 3;
  cudaError_t e = cudaSuccess;
  if (P.nchunks > 0) {
    LaunchPlan& pl = h->plan_pool[w ? 1 : 0];
    if (!pl.fn) {
      LaunchCfg c{(int)h->threads, (int)h->vec, (int)h->ctas_per_sm};
      e = plan_pool_local(P, c, &pl);
    }
    if (e == cudaSuccess) e = launch_planned(pl, P, st);
  }
  if (e != cudaSuccess) return fail(h, EMB_A2A_ECUDA, "pool kernel launch: %s",
                                    cudaGetErrorString(e));
  if (P.nslices > 0) h->kernel_launches++;
  return EMB_A2A_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------ backward (f3)
namespace {

int ceil_log2(int64_t v) {   // bits needed for values 0 .. v-1
  int b = 0;
  while (b < 63 && ((int64_t)1 << b) < v) ++b;
  return b;
}

template <typename T>
int grow(emb_a2a* h, T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  CUDA_TRY(h, cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T)));
  return EMB_A2A_OK;
}

BwdParams bwd_params(emb_a2a* h, const float* grad, float lr, int fused) {
  BwdParams P;
  memset(&P, 0, sizeof(P));
  P.grad = grad;
  P.peers = h->d_peers;
  P.bflags_in = h->bflags;
  P.bcredits_in = h->bcredits;
  P.keys = h->d_keys[h->plan_buf];
  P.bags = h->d_bags[h->plan_buf];
  P.wts = h->plan_weighted ? h->d_wts[h->plan_buf] : nullptr;
  P.offsets = h->plan_offsets;
  P.tables = (float* const*)h->d_tables;
  P.scratch = h->d_scratch;
  P.info = h->d_info;
  P.ticket = h->d_hist + 2 * kHistWords;
  P.trace = h->d_trace;
  P.trace_cap = h->trace_cap;
  P.err = h->d_err;
  P.n = h->planned ? h->plan_n : 0;
  P.B = h->B;
  P.timeout_ns = (long long)h->timeout_ms * 1000000ll;
  P.lr = lr;
  P.W = h->W;
  P.r = h->rank;
  P.T = h->T;
  P.D = h->D;
  P.G = h->G;
  P.toff = h->toff;
  P.chunk = bwd_chunk_for(h->D);
  P.nchunks = (P.n + P.chunk - 1) / P.chunk;
  P.flist = 0;
  // per warp: gradient-row and table-row pointers and scalars of a sub-batch, a carried sum
  P.wbytes = 32 * (8 + 8 + 4) + 2 * (int64_t)h->D * 4;
  P.rbits = h->rbits;
  P.fused = fused;
  P.mean = h->mean;
  int acc = 0;
  for (int q = 0; q < h->W; ++q) {
    P.allT[q] = h->allT[q];
    P.tofs[q] = acc;
    acc += h->allT[q];
  }
  for (int s = 0; s <= h->W; ++s) P.part[s] = h->part[s];
  return P;
}

int run_backward(emb_a2a* h, BwdParams& P, cudaStream_t st) {
  h->tables_dirty = true;   // the next forward's table reads wait for this kernel
  const int mode = P.wts ? 1 : (P.mean ? 2 : 0);
  if (h->bwd_mode != mode) {
    cudaError_t e = plan_backward(P, (int)h->bwd_threads, (int)h->bwd_share, &h->bwd_grid,
                                  &h->bwd_smem);
    if (e != cudaSuccess) return fail(h, EMB_A2A_ECUDA, "backward plan: %s", cudaGetErrorString(e));
    h->bwd_mode = mode;
  }
  // P.ticket: zero when allocated, reset by pass 2 of each launch (no memset between kernels)
  P.pdl_fold = (h->bwd_share <= 1) ? 1 : 0;
  cudaError_t e = launch_backward(P, h->bwd_grid, (int)h->bwd_threads, h->bwd_smem, st);
  if (e != cudaSuccess) {
    h->poisoned = true;
    return fail(h, EMB_A2A_ECUDA, "backward kernel launch: %s", cudaGetErrorString(e));
  }
  h->kernel_launches += (P.T > 0 && P.nchunks > 0) ? 2 : 1;
  return EMB_A2A_OK;
}

int bwd_common_checks(emb_a2a* h, const char* what) {
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "%s before register_tables", what);
  if (h->elem != EMB_A2A_F32)
    return fail(h, EMB_A2A_EINVAL, "%s: backward updates fp32 tables only (R#30)", what);
  return EMB_A2A_OK;
}

}  // namespace

extern "C" {

int emb_a2a_backward_plan(emb_a2a_t* h, const int32_t* indices, const int32_t* offsets,
                          const float* weights, int64_t num_indices, void* stream) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = bwd_common_checks(h, "backward_plan");
  if (rc) return rc;
  if (num_indices < 0 || num_indices >= (1ll << 31))
    return fail(h, EMB_A2A_EINVAL, "num_indices out of range (int32 CSR, R#8)");
  if ((h->T > 0 && h->B > 0) && (!offsets || (num_indices > 0 && !indices)))
    return fail(h, EMB_A2A_EINVAL, "indices/offsets are NULL");
  if (weights && h->mean)
    return fail(h, EMB_A2A_EINVAL, "per-sample weights need sum pooling (R#26)");
  int64_t rmax = 1;
  for (int t = 0; t < h->T; ++t) rmax = std::max<int64_t>(rmax, h->rows[t]);
  const int tbits = ceil_log2(std::max(1, h->T)), rbits = ceil_log2(rmax);
  if (tbits + rbits > 32)
    return fail(h, EMB_A2A_EINVAL, "backward sort key needs %d bits (> 32): T_r * max rows too "
                "large", tbits + rbits);
  DeviceGuard guard(h->dev);
  cudaStream_t st = (cudaStream_t)stream;
  if (h->validate && h->T > 0 && h->B > 0) {
    rc = run_validate(h, indices, offsets, num_indices, st);
    if (rc) return rc;
  }
  const int64_t n = (h->T > 0) ? num_indices : 0;
  // passes over the whole key (table, row).  (Measured: sorting the row bits only -- the input
  // is table-major and the sort stable, so (table, row) runs stay contiguous -- saves a pass for
  // DLRM-wide / sweep / weak, but the (row, table) order it leaves makes the reduction jump
  // between tables: pass 1 of DLRM-wide 401 -> 451 us, more than the plan saved.)
  const int kbits = tbits + rbits;
  // Segmented plan (backward.cu "segmented sort plan"): the input is table-major and the sort
  // stable, so sorting each table's segment by its row bits alone gives the same (table, row)
  // order in 2 passes of <= 11-bit digits where the plain key needs 3 or 4.
  int dev0 = 0, sms0 = 0;
  cudaGetDevice(&dev0);
  cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
  const int seg_db = std::max(8, (rbits + 1) / 2);
  const int64_t ntiles_seg = (num_indices + kSortTile - 1) / kSortTile + h->T;
  // Measured (r02o, ncu launch list): a 10-bit segmented pass costs 16.9 us and an 11-bit one
  // 22.4 us against 12.0 us for an 8-bit pass (publishing and looking back over 4-8x the digit
  // words), so 2 wide passes only tie 3-4 narrow ones; auto keeps the plain plan (option 3 only).
  const bool seg = h->T >= 1 && h->T <= 256 && rbits <= 22 && h->sort_mode == 3;
  (void)sms0;
  // bucket plan (sort_mode 5): one pass on the top 8 key bits, then per-bucket local sorts
  // Auto: 64 K..512 K lookups (<= 2 K keys per bucket on average) and <= 32 K lookups per table
  // (the largest bucket holds a table's Zipf-hot row, ~10 % of its lookups, and the CTA sorting
  // it bounds the kernel).  Measured r02bc (plan, plain -> bucket): sweep P=1 49.7 -> 27.2 us,
  // weak 48.2 -> 42.4, sweep P=4 59.4 -> 56.3; DLRM-small (41 K lookups per table, a ~5 K-key
  // bucket) 39.7 -> 51.3, so it keeps the plain plan.
  const bool bkt = kbits > 8 && (h->sort_mode == 5 ||
                                 (h->sort_mode == 0 && n >= (1 << 16) && n <= (1 << 19) &&
                                  n <= (int64_t)32768 * std::max(h->T, 1)));
  const int passes = seg ? 2 : bkt ? 1 : (kbits + 7) / 8;
  const int64_t nchunks = (n + kBwdChunkMin - 1) / kBwdChunkMin;   // upper bound
  const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const bool wtd = weights != nullptr && n > 0;
  // plan storage (grow-only)
  const size_t ncap = (size_t)n + n / 4 + 4096;   // headroom: batches vary in size
  if ((size_t)n > h->plan_cap) {
    for (int x = 0; x < 2; ++x) {
      if ((rc = grow(h, &h->d_keys[x], ncap))) return rc;
      if ((rc = grow(h, &h->d_bags[x], ncap))) return rc;
    }
    h->plan_cap = ncap;
  }
  if (wtd && (size_t)n > h->wts_cap) {
    for (int x = 0; x < 2; ++x)
      if ((rc = grow(h, &h->d_wts[x], ncap))) return rc;
    h->wts_cap = ncap;
  }
  // [pass histograms | pass tile tickets | backward chunk ticket]
  if (!h->d_hist) {
    if ((rc = grow(h, &h->d_hist, 2 * kHistWords + 1))) return rc;
    CUDA_TRY(h, cudaMemsetAsync(h->d_hist, 0, (2 * kHistWords + 1) * 4, st));
  }
  const size_t ncnt = (size_t)ntiles * 256;      // tile digit counts of one pass
  if (ncnt > h->cnt_cap) {
    const size_t scap = ncnt + ncnt / 4 + 256;
    if ((rc = grow(h, &h->d_cnt, scap))) return rc;
    h->cnt_cap = scap;
  }
  const size_t nb_seg = (size_t)1 << seg_db;
  const long long ngroups_seg = (ntiles_seg + kSegLb - 1) / kSegLb + h->T;
  const size_t nstatus = seg ? (size_t)2 * ntiles_seg * nb_seg
                             : (size_t)passes * ntiles * 256;   // onesweep look-back words
  if (nstatus > h->status_cap) {
    const size_t scap = nstatus + nstatus / 4 + 4 * 256;
    if ((rc = grow(h, &h->d_status, scap))) return rc;
    CUDA_TRY(h, cudaMemsetAsync(h->d_status, 0, scap * 8, st));   // ordered before the plan
    h->status_cap = scap;
  }
  const long long ngroups = (ntiles + kLbGroup - 1) / kLbGroup;
  const size_t nlbg = seg ? (size_t)2 * ngroups_seg * (nb_seg + 1)
                          : (size_t)passes * ngroups * 257;      // zeroed by keygen every plan
  if (nlbg > h->lbg_cap) {
    const size_t scap = nlbg + nlbg / 4 + 257;
    if ((rc = grow(h, &h->d_lbg, scap))) return rc;
    h->lbg_cap = scap;
  }
  if ((size_t)nchunks > h->chunk_cap) {
    const size_t cap = (size_t)nchunks + nchunks / 4 + 64;    // headroom: batches vary in size
    if ((rc = grow(h, &h->d_scratch, cap * 2 * h->D))) return rc;
    if ((rc = grow(h, &h->d_info, cap))) return rc;
    h->chunk_cap = cap;
  }
  if (seg) {
    const size_t half = (size_t)2 * h->T * nb_seg + 2;
    if (half > h->shist_half) {
      if (h->d_shist) cudaFree(h->d_shist);
      h->d_shist = nullptr;
      h->shist_half = 0;
      if ((rc = grow(h, &h->d_shist, 2 * half))) return rc;
      CUDA_TRY(h, cudaMemsetAsync(h->d_shist, 0, 2 * half * 4, st));
      h->shist_half = half;
    }
  }
  if (n > 0 && h->last_seg >= 0 && h->last_seg != (seg ? 1 : 0)) {
    // switching plan kinds breaks the "keygen zeroes the next plan's half" chain: clean both
    CUDA_TRY(h, cudaMemsetAsync(h->d_hist, 0, 2 * kHistWords * sizeof(unsigned), st));
    if (h->d_shist) CUDA_TRY(h, cudaMemsetAsync(h->d_shist, 0, 2 * h->shist_half * 4, st));
  }
  // Cluster plan (sort_mode 4, backward.cu "cluster sort plan"): keygen + every pass in one
  // kernel, one thread-block cluster per table, digit offsets exchanged in distributed shared
  // memory.  Needs the table-major segments of an in-range key (checked above).
  if (h->sort_mode == 4 && n > 0) {
    const int cpasses = rbits == 0 ? 0 : (rbits + kClusterMaxDB - 1) / kClusterMaxDB;
    const int cdb = cpasses ? (rbits + cpasses - 1) / cpasses : 0;
    const int C = h->cluster_ctas > 0 ? (int)h->cluster_ctas : cluster_plan_size(h->T, cdb, wtd);
    if (C <= 0) return fail(h, EMB_A2A_ECUDA, "backward cluster plan: no cluster size fits");
    ClusterSortParams cs;
    memset(&cs, 0, sizeof(cs));
    cs.indices = indices;
    cs.offsets = offsets;
    cs.weights = wtd ? weights : nullptr;
    for (int x = 0; x < 2; ++x) {
      cs.keys[x] = h->d_keys[x];
      cs.bags[x] = h->d_bags[x];
      cs.wts[x] = wtd ? h->d_wts[x] : nullptr;
    }
    cs.B = h->B;
    cs.C = C;
    cs.rbits = rbits;
    cs.passes = cpasses;
    cs.db = cdb;
    cs.trace = h->d_trace;
    cs.trace_cap = h->trace_cap;
    h->planned = false;
    cudaError_t e = launch_sort_plan_cluster(cs, h->T, st);
    if (e != cudaSuccess)
      return fail(h, EMB_A2A_ECUDA, "backward cluster plan launch (C=%d): %s", C,
                  cudaGetErrorString(e));
    h->plan_no += 1;
    h->rbits = rbits;
    h->plan_weighted = wtd;
    h->plan_offsets = offsets;
    h->plan_n = n;
    h->plan_buf = cpasses & 1;
    h->planned = true;
    h->kernel_launches += 1;
    return EMB_A2A_OK;
  }
  h->plan_no += 1;
  h->rbits = rbits;
  h->plan_weighted = wtd;
  h->plan_offsets = offsets;
  h->plan_n = n;
  h->plan_buf = bkt ? 0 : passes & 1;   // the bucket sort writes buffer 0
  h->planned = true;
  if (n == 0) return EMB_A2A_OK;
  // this plan's digit counts and tile tickets: the half zeroed by the previous plan's keygen (or
  // at allocation); this keygen zeroes the other half for the next plan (no memset in the chain)
  unsigned* const hb = h->d_hist + h->hist_par * kHistWords;
  SortParams S;
  memset(&S, 0, sizeof(S));
  S.indices = indices;
  S.offsets = offsets;
  S.weights = wtd ? weights : nullptr;
  S.keys = h->d_keys[0];
  S.bags = h->d_bags[0];
  S.wts = h->d_wts[0];
  S.hist = hb;
  S.hist_clear = h->d_hist + (1 - h->hist_par) * kHistWords;
  S.TB = (long long)h->T * h->B;
  S.B = h->B;
  S.rbits = rbits;
  S.passes = passes;
  S.last_mask = bkt ? 255u : passes > 0 ? (1u << (kbits - 8 * (passes - 1))) - 1u : 0u;
  S.hshift = bkt ? kbits - 8 : 0;
  S.lbg = h->d_lbg;
  S.lbg_words = (long long)nlbg;
  PassParams pp[kMaxPasses];
  for (int p = 0; p < passes; ++p) {
    PassParams& q = pp[p];
    memset(&q, 0, sizeof(q));
    q.keys_in = h->d_keys[p & 1];
    q.keys_out = h->d_keys[(p + 1) & 1];
    q.bags_in = h->d_bags[p & 1];
    q.bags_out = h->d_bags[(p + 1) & 1];
    q.wts_in = wtd ? h->d_wts[p & 1] : nullptr;
    q.wts_out = wtd ? h->d_wts[(p + 1) & 1] : nullptr;
    q.hist = hb + p * 256;
    q.cnt = h->d_cnt;
    q.status = h->d_status + (size_t)p * ntiles * 256;
    q.tile_ctr = hb + kMaxPasses * 256 + p;
    q.garrive = h->d_lbg + (size_t)p * ngroups * 257;
    q.gsum = q.garrive + ngroups;
    q.ntiles = ntiles;
    q.n = n;
    q.shift = bkt ? kbits - 8 : 8 * p;
    q.dmask = p == passes - 1 ? S.last_mask : 255u;
    q.stamp = h->plan_no;
    q.trace = h->d_trace;
    q.trace_cap = h->trace_cap;
    q.err = h->d_err;
    q.timeout_ns = (long long)h->timeout_ms * 1000000ll;
    q.stall = (int)h->sort_stall;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long TB = (long long)h->T * h->B;
  const long long gk = std::min<long long>((TB + 63) / 64, (long long)sms * 8);   // 8 bags/warp
  if (seg) {
    unsigned* const sh = h->d_shist + (size_t)h->hist_par * h->shist_half;
    S.seg_db = seg_db;
    S.T = h->T;
    S.shist = sh;
    S.shist_clear = h->d_shist + (size_t)(1 - h->hist_par) * h->shist_half;
    S.shist_words = (long long)h->shist_half;
    const unsigned m0 = (1u << seg_db) - 1u;
    const unsigned m1 = rbits > seg_db ? (1u << (rbits - seg_db)) - 1u : 0u;
    for (int p = 0; p < 2; ++p) {
      PassParams& q = pp[p];
      q.status = h->d_status + (size_t)p * ntiles_seg * nb_seg;
      q.tile_ctr = sh + (size_t)2 * h->T * nb_seg + p;
      q.garrive = h->d_lbg + (size_t)p * ngroups_seg * (nb_seg + 1);
      q.gsum = q.garrive + ngroups_seg;
      q.ntiles = ntiles_seg;
      q.shift = p * seg_db;
      q.dmask = p == 0 ? m0 : m1;
      q.offsets = offsets;
      q.B = h->B;
      q.T = h->T;
      q.shist = sh + (size_t)p * h->T * nb_seg;
    }
  }
  cudaError_t e = seg ? launch_sort_plan_seg(S, pp, passes, ntiles_seg,
                                             (int)std::max<long long>(gk, 1), st)
                      : launch_sort_plan(S, pp, passes, ntiles, (int)std::max<long long>(gk, 1),
                                         bkt ? 1 : (int)h->sort_mode, st);
  if (e == cudaSuccess && bkt)
    e = launch_bucket_sort(h->d_keys[1], h->d_bags[1], wtd ? h->d_wts[1] : nullptr, h->d_keys[0],
                           h->d_bags[0], wtd ? h->d_wts[0] : nullptr, hb, kbits - 8,
                           (int)h->bucket_cap, st);
  if (e != cudaSuccess) {
    h->planned = false;
    cudaMemsetAsync(h->d_hist, 0, 2 * kHistWords * sizeof(unsigned), st);   // both halves clean
    if (h->d_shist) cudaMemsetAsync(h->d_shist, 0, 2 * h->shist_half * 4, st);
    return fail(h, EMB_A2A_ECUDA, "backward plan launch: %s", cudaGetErrorString(e));
  }
  if (n > 0) h->last_seg = seg ? 1 : 0;
  h->hist_par ^= 1;
  h->kernel_launches += 1 + passes + (bkt ? 1 : 0);
  return EMB_A2A_OK;
}

int emb_a2a_backward(emb_a2a_t* h, const float* grad, float lr, void* stream) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = bwd_common_checks(h, "backward");
  if (rc) return rc;
  if (h->T > 0 && !h->planned)
    return fail(h, EMB_A2A_ESTATE, "backward before backward_plan");
  if (!grad && h->b > 0) return fail(h, EMB_A2A_EINVAL, "grad is NULL");
  if (grad && ((uintptr_t)grad % 16)) return fail(h, EMB_A2A_EINVAL, "grad must be 16-B aligned");
  DeviceGuard guard(h->dev);
  h->bepoch += 1;
  BwdParams P = bwd_params(h, grad, lr, 1);
  P.parity = (int)(h->bepoch & 1);
  P.stage = h->gstage[P.parity];
  P.bepoch = h->bepoch;
  return run_backward(h, P, (cudaStream_t)stream);
}

int emb_a2a_backward_local(emb_a2a_t* h, const float* grad_mp, float lr, void* stream) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = bwd_common_checks(h, "backward_local");
  if (rc) return rc;
  if (h->T == 0) return EMB_A2A_OK;
  if (!h->planned) return fail(h, EMB_A2A_ESTATE, "backward_local before backward_plan");
  if (!grad_mp && h->B > 0) return fail(h, EMB_A2A_EINVAL, "grad_mp is NULL");
  if (grad_mp && ((uintptr_t)grad_mp % 16))
    return fail(h, EMB_A2A_EINVAL, "grad_mp must be 16-B aligned");
  DeviceGuard guard(h->dev);
  BwdParams P = bwd_params(h, grad_mp, lr, 0);
  return run_backward(h, P, (cudaStream_t)stream);
}

int emb_a2a_check(emb_a2a_t* h) {
  if (!h) return EMB_A2A_EINVAL;
  return check_async(h);
}

int emb_a2a_device_barrier(emb_a2a_t* h, void* stream) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "device_barrier before register_tables");
  if (h->W == 1) return EMB_A2A_OK;
  DeviceGuard guard(h->dev);
  h->barrier_epoch += 1;
  CUDA_TRY(h, launch_barrier(h->d_peers, h->flags + (size_t)h->W * kFlagStride, h->W, h->rank,
                             h->barrier_epoch * (unsigned long long)(h->W - 1),
                             (long long)h->timeout_ms * 1000000ll, h->d_err,
                             (cudaStream_t)stream));
  h->kernel_launches++;
  return EMB_A2A_OK;
}

int emb_a2a_peer_store_probe(emb_a2a_t* h, int64_t bytes_per_peer, void* stream,
                             int64_t* bytes_used) {
  if (!h || !bytes_used) return EMB_A2A_EINVAL;
  *bytes_used = 0;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "peer_store_probe before register_tables");
  if (bytes_per_peer < 0) return fail(h, EMB_A2A_EINVAL, "bytes_per_peer < 0");
  if (h->W == 1) return EMB_A2A_OK;
  // the smallest peer receive region (both halves) bounds what may be written: 512-B runs
  int64_t cap = -1;
  for (int q = 0; q < h->W; ++q) {
    if (q == h->rank) continue;
    const int64_t bq = h->part[q + 1] - h->part[q];
    const int64_t oes = h->out_dtype == EMB_A2A_F32 ? 4 : 2;
    const int64_t half = std::max<int64_t>((bq * h->G * h->D * oes + 255) / 256 * 256, 256);
    cap = cap < 0 ? 2 * half : std::min<int64_t>(cap, 2 * half);
  }
  const long long runs = std::min<int64_t>(bytes_per_peer, cap) / 512;
  if (runs <= 0) return EMB_A2A_OK;
  DeviceGuard guard(h->dev);
  CUDA_TRY(h, launch_peer_store_probe(h->d_peers, h->W, h->rank, runs, (cudaStream_t)stream));
  h->kernel_launches++;
  *bytes_used = (int64_t)runs * 512;
  return EMB_A2A_OK;
}

int emb_a2a_set_option(emb_a2a_t* h, const char* key, int64_t v) {
  if (!h || !key) return EMB_A2A_EINVAL;
  for (int w = 0; w < 2; ++w) {   // any option may change the kernel instance / grid / smem
    h->plan_fused[w] = LaunchPlan();
    h->plan_pool[w] = LaunchPlan();
  }
  std::string k(key);
  if (k == "slice") {
    if (v < 1 || v > (1 << 20)) return fail(h, EMB_A2A_EINVAL, "slice must be in [1, 2^20]");
    if (h->registered && v != h->S) {
      // counters are monotone per (epoch x expected count): changing S mid-stream would break
      // the epoch arithmetic, so it is only allowed before register_tables.
      return fail(h, EMB_A2A_ESTATE, "set 'slice' before register_tables");
    }
    h->S = v;
  } else if (k == "order") {
    if (v < 0 || v > 2) return fail(h, EMB_A2A_EINVAL, "order must be 0, 1 or 2");
    if (h->registered && v != h->order)   // slice ids (and their counters) depend on the order
      return fail(h, EMB_A2A_ESTATE, "set 'order' before register_tables");
    h->order = v;
  } else if (k == "out_dtype") {
    if (v < EMB_A2A_F32 || v > EMB_A2A_F16)
      return fail(h, EMB_A2A_EINVAL, "out_dtype: 0 fp32, 1 bf16, 2 fp16");
    if (h->registered && v != h->out_dtype)   // the receive buffers are sized for it
      return fail(h, EMB_A2A_ESTATE, "set 'out_dtype' before register_tables");
    h->out_dtype = v;
  } else if (k == "chunk") {
    if (v < 0 || v > 127) return fail(h, EMB_A2A_EINVAL, "chunk in [0 (auto), 127]");
    if (h->registered && v != h->chunk)
      return fail(h, EMB_A2A_ESTATE, "set 'chunk' before register_tables");
    h->chunk = v;
  } else if (k == "threads") {
    if (v < 32 || v > 256 || v % 32) return fail(h, EMB_A2A_EINVAL, "threads: 32..256, x32");
    h->threads = v;
  } else if (k == "timeout_ms") {
    if (v < 1) return fail(h, EMB_A2A_EINVAL, "timeout_ms >= 1");
    h->timeout_ms = v;
  } else if (k == "validate") {
    h->validate = v ? 1 : 0;
  } else if (k == "idx_cap") {
    if (v < 0 || v > 16384) return fail(h, EMB_A2A_EINVAL, "idx_cap in [0, 16384]");
    h->idx_cap = v;
  } else if (k == "l1_rows") {
    if (v < -1 || v > 1) return fail(h, EMB_A2A_EINVAL, "l1_rows in {-1 (auto), 0, 1}");
    h->l1_opt = v;                     // applied by the next forward's ensure_chunk
  } else if (k == "flat_below") {
    if (v < 0 || v > 1 << 20) return fail(h, EMB_A2A_EINVAL, "flat_below >= 0");
    h->flat_below = v;
  } else if (k == "pdl") {
    h->pdl = v ? 1 : 0;
  } else if (k == "vec") {
    if (!(v == 0 || v == 1 || v == 2 || v == 4 || v == 8))
      return fail(h, EMB_A2A_EINVAL, "vec in {0, 1, 2, 4, 8}");
    h->vec = v;
  } else if (k == "tma") {
    h->tma = v ? 1 : 0;
  } else if (k == "stage_kb") {
    if (v < 1 || v > 200) return fail(h, EMB_A2A_EINVAL, "stage_kb in [1, 200]");
    h->stage_kb = v;
  } else if (k == "stages") {
    if (v < 2 || v > kMaxStages) return fail(h, EMB_A2A_EINVAL, "stages in [2, %d]", kMaxStages);
    h->stages = v;
  } else if (k == "ctas_per_sm") {
    if (v < 0 || v > 32) return fail(h, EMB_A2A_EINVAL, "ctas_per_sm in [0, 32]");
    h->ctas_per_sm = v;
  } else if (k == "trace") {
    if (v < 0 || v > (1 << 24)) return fail(h, EMB_A2A_EINVAL, "trace records in [0, 2^24]");
    DeviceGuard guard(h->dev);
    if (h->d_trace) cudaFree(h->d_trace);
    h->d_trace = nullptr;
    h->trace_cap = 0;
    if (v > 0) {
      CUDA_TRY(h, cudaMalloc((void**)&h->d_trace, (size_t)(2 + 2 * v) * 8));
      CUDA_TRY(h, cudaMemset(h->d_trace, 0, (size_t)(2 + 2 * v) * 8));
      CUDA_TRY(h, cudaDeviceSynchronize());   // legacy-stream memset vs. non-blocking streams
      h->trace_cap = v;
    }
  } else if (k == "pdl_rows_early") {
    if (v < 0 || v > 2) return fail(h, EMB_A2A_EINVAL, "pdl_rows_early in {0, 1, 2}");
    h->rows_early = v;
  } else if (k == "debug_credit_lag") {
    if (v < -1 || v > 1) return fail(h, EMB_A2A_EINVAL, "debug_credit_lag in {-1, 0, 1}");
    h->credit_lag_opt = v;
  } else if (k == "sort_mode") {
    if (v < 0 || v > 5) return fail(h, EMB_A2A_EINVAL, "sort_mode in {0, 1, 2, 3, 4, 5}");
    h->sort_mode = v;
  } else if (k == "bucket_cap") {
    if (v < 256 || v > 8192 || v % 256)
      return fail(h, EMB_A2A_EINVAL, "bucket_cap: 256..8192, multiple of 256");
    h->bucket_cap = v;
  } else if (k == "cluster_ctas") {
    if (v != 0 && v != 1 && v != 2 && v != 4 && v != 8 && v != 16)
      return fail(h, EMB_A2A_EINVAL, "cluster_ctas in {0 (auto), 1, 2, 4, 8, 16}");
    h->cluster_ctas = v;
  } else if (k == "bwd_threads") {
    // bwd_kernel is compiled with __launch_bounds__(128, ...): more threads cannot launch
    if (v < 32 || v > 128 || v % 32) return fail(h, EMB_A2A_EINVAL, "bwd_threads: 32..128, x32");
    h->bwd_threads = v;
    h->bwd_mode = -1;
  } else if (k == "bwd_share") {
    if (v < 1 || v > kMaxW) return fail(h, EMB_A2A_EINVAL, "bwd_share in [1, %d]", kMaxW);
    h->bwd_share = v;
    h->bwd_mode = -1;
  } else if (k == "debug_delay_ns") {
    h->delay_ns = std::max<int64_t>(0, v);
  } else if (k == "debug_sort_stall") {
    h->sort_stall = v ? 1 : 0;
  } else if (k == "debug_skip_signal_to") {
    h->skip_to = v;
  } else {
    return fail(h, EMB_A2A_EINVAL, "unknown option '%s'", key);
  }
  return EMB_A2A_OK;
}

int emb_a2a_get_option(const emb_a2a_t* h, const char* key, int64_t* v) {
  if (!h || !key || !v) return EMB_A2A_EINVAL;
  std::string k(key);
  if (k == "slice") *v = h->S;
  else if (k == "order") *v = h->order;
  else if (k == "threads") *v = h->threads;
  else if (k == "timeout_ms") *v = h->timeout_ms;
  else if (k == "validate") *v = h->validate;
  else if (k == "idx_cap") *v = h->idx_cap;
  else if (k == "stages") *v = h->stages;
  else if (k == "chunk") *v = h->chunk;
  else if (k == "out_dtype") *v = h->out_dtype;
  else if (k == "trace") *v = h->trace_cap;
  else if (k == "tma") *v = h->tma;
  else if (k == "vec") *v = h->vec;
  else if (k == "pdl") *v = h->pdl;
  else if (k == "flat_below") *v = h->flat_below;
  else if (k == "l1_rows") *v = h->l1_opt;
  else if (k == "l1_rows_active") *v = h->l1_cur;
  else if (k == "stage_kb") *v = h->stage_kb;
  else if (k == "ctas_per_sm") *v = h->ctas_per_sm;
  else if (k == "pdl_rows_early") *v = h->rows_early;
  else if (k == "debug_credit_lag") *v = h->credit_lag_opt;
  else if (k == "sort_mode") *v = h->sort_mode;
  else if (k == "cluster_ctas") *v = h->cluster_ctas;
  else if (k == "bucket_cap") *v = h->bucket_cap;
  else if (k == "bwd_threads") *v = h->bwd_threads;
  else if (k == "bwd_share") *v = h->bwd_share;
  else if (k == "debug_delay_ns") *v = h->delay_ns;
  else if (k == "debug_sort_stall") *v = h->sort_stall;
  else if (k == "debug_skip_signal_to") *v = h->skip_to;
  else return EMB_A2A_EINVAL;
  return EMB_A2A_OK;
}

int emb_a2a_query(const emb_a2a_t* h, const char* key, int64_t* v) {
  if (!h || !key || !v) return EMB_A2A_EINVAL;
  std::string k(key);
  if (k == "rank") *v = h->rank;
  else if (k == "world_size") *v = h->W;
  else if (k == "device") *v = h->dev;
  else if (k == "epoch") *v = (int64_t)h->epoch;
  else if (k == "kernel_launches") *v = h->kernel_launches;
  else if (!h->registered) return EMB_A2A_ESTATE;
  else if (k == "local_batch") *v = h->b;
  else if (k == "total_tables") *v = h->G;
  else if (k == "local_tables") *v = h->T;
  else if (k == "table_offset") *v = h->toff;
  else if (k == "dim") *v = h->D;
  else if (k == "table_dtype") *v = h->elem;
  else if (k == "pooling") *v = h->mean;
  else if (k == "global_batch") *v = h->B;
  else if (k == "num_slices") *v = h->nslices;
  else if (k == "num_chunks") *v = h->nchunks;
  else if (k == "chunk_bags") *v = h->C;
  else if (k == "region_bytes") *v = (int64_t)h->region_bytes;
  else if (k == "last_grid") *v = h->last_grid;
  else if (k == "backward_epoch") *v = (int64_t)h->bepoch;
  else if (k == "plan_lookups") *v = h->planned ? h->plan_n : -1;
  else if (k == "bwd_grid") *v = h->bwd_grid;
  else if (k == "bwd_chunk") *v = bwd_chunk_for(h->D);
  else if (k.rfind("expected_in:", 0) == 0) {
    const int q = atoi(k.c_str() + 12);
    if (q < 0 || q >= h->W) return EMB_A2A_EINVAL;
    *v = h->host_peers.n_in[q];
  } else {
    return EMB_A2A_EINVAL;
  }
  return EMB_A2A_OK;
}

int emb_a2a_slice_plan(emb_a2a_t* h, int32_t* out, int64_t capacity, int64_t* n) {
  if (!h || !n) return EMB_A2A_EINVAL;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "not registered");
  *n = h->nslices;
  if (capacity < h->nslices || (!out && h->nslices > 0))
    return fail(h, EMB_A2A_EINVAL, "capacity %lld < %d slices", (long long)capacity,
                h->nslices);
  if (h->nslices == 0) return EMB_A2A_OK;
  DeviceGuard guard(h->dev);
  int* d = nullptr;
  CUDA_TRY(h, cudaMalloc((void**)&d, sizeof(int) * 4 * h->nslices));
  KParams P = make_params(h, nullptr, nullptr, nullptr);
  cudaError_t e = launch_slice_plan(P, d, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(int) * 4 * h->nslices,
                                       cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(h, EMB_A2A_ECUDA, "slice_plan: %s", cudaGetErrorString(e));
  return EMB_A2A_OK;
}

int emb_a2a_read_trace(emb_a2a_t* h, uint64_t* out, int64_t capacity, int64_t* n) {
  if (!h || !n) return EMB_A2A_EINVAL;
  if (!h->d_trace) return fail(h, EMB_A2A_ESTATE, "tracing is off (set_option trace)");
  DeviceGuard guard(h->dev);
  CUDA_TRY(h, cudaDeviceSynchronize());
  unsigned long long cnt = 0;
  CUDA_TRY(h, cudaMemcpy(&cnt, h->d_trace, 8, cudaMemcpyDeviceToHost));
  const int64_t m = std::min<int64_t>((int64_t)cnt, h->trace_cap);
  *n = m;
  if (capacity < m || (!out && m > 0)) return fail(h, EMB_A2A_EINVAL, "capacity < %lld", (long long)m);
  if (m > 0) CUDA_TRY(h, cudaMemcpy(out, h->d_trace + 2, (size_t)m * 16, cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemset(h->d_trace, 0, 8));   // restart the log
  CUDA_TRY(h, cudaDeviceSynchronize());
  return EMB_A2A_OK;
}

int emb_a2a_read_flags(emb_a2a_t* h, uint64_t* out, int capacity) {
  if (!h || !out || capacity < h->W) return EMB_A2A_EINVAL;
  if (!h->registered) return fail(h, EMB_A2A_ESTATE, "not registered");
  DeviceGuard guard(h->dev);
  std::vector<unsigned long long> buf((size_t)h->W * kFlagStride);
  CUDA_TRY(h, cudaMemcpy(buf.data(), h->flags, buf.size() * 8, cudaMemcpyDeviceToHost));
  for (int q = 0; q < h->W; ++q) out[q] = buf[(size_t)q * kFlagStride];
  return EMB_A2A_OK;
}

int emb_a2a_destroy(emb_a2a_t* h) {
  if (!h) return EMB_A2A_EINVAL;
  int rc = EMB_A2A_OK;
  {
    DeviceGuard guard(h->dev);
    if (h->registered) {
      cudaDeviceSynchronize();
      rc = barrier(h);                      // no peer is still writing into our region
      for (void* p : h->opened) cudaIpcCloseMemHandle(p);
      h->opened.clear();
      int rc2 = barrier(h);                 // every peer has unmapped us
      if (!rc) rc = rc2;
      release_registration(h);
    }
    if (h->h_err) cudaFreeHost(h->h_err);
    if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
    if (h->d2h_stream) cudaStreamDestroy(h->d2h_stream);
    if (h->ev_in) cudaEventDestroy(h->ev_in);
    for (int x = 0; x < 2; ++x) {
      if (h->ev_free[x]) cudaEventDestroy(h->ev_free[x]);
      if (h->ev_done[x]) cudaEventDestroy(h->ev_done[x]);
      if (h->ev_out[x]) cudaEventDestroy(h->ev_out[x]);
    }
  }
  delete h;
  return rc;
}

}  // extern "C"
