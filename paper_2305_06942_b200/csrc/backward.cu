// backward.cu -- the backward pass of the fused op (the paper's future work,
// P:318 "we plan to explore ... the backward pass"), sm_100a.
//
// What it computes (oracle/oracle.c oracle_backward_sgd; R#29-R#31): every rank s holds
// the gradient of its forward output, [b_s][G*D] (data parallel).  The owner r of table g needs,
// for every lookup k of g (bag j, row x), the gradient row of bag j -- which lives on the rank
// s = dest(j) that received bag j's pooled vector -- and updates
//     W_g[x] = W_g[x] - lr * sum_{k : idx_k = x} c_k,   c_k = grad_s[j - p_s][g*D ..]
//                                                        (x w_k weighted, / L_j mean)
// i.e. the All-to-All of the forward runs in reverse (DP -> MP) and is followed by the
// embedding-gradient segment reduction and a sparse SGD step.
//
// Kernels:
//   bwd_keygen_kernel    key_k = t << rbits | idx_k, payload bag_k (+ w_k); digit histograms of
//                        every radix pass at once (upfront histogram)
//   bwd_onesweep_kernel  one stable LSD radix pass (8-bit digit) in one kernel, with a two-level
//                        look-back over the tiles (used while the tiles fit one wave)
//   bwd_upsweep_kernel / bwd_scan_kernel / bwd_downsweep_kernel
//                        the same pass as reduce-then-scan: tile digit counts, a per-digit scan
//                        over tiles, then warp-level ranking with match.any and a digit-ordered,
//                        contiguous write-out of each tile (more tiles than one wave)
//   bwd_bucket_sort_kernel  (bucket plan) after a onesweep pass on the top key digit, one CTA
//                        per bucket sorts it by the low bits in shared memory
//   bwd_cluster_sort_kernel (cluster plan, option) keygen + every row-digit pass of a table in
//                        one thread-block cluster, digit counts exchanged through DSMEM
//   bwd_kernel           pass 1 (fused) each CTA first pushes its share of this rank's gradient
//                        rows straight into the owners' staging buffers over NVLink (zero-copy,
//                        the reverse of P:165; a store into owner q waits for q's credit) and
//                        signals the owner's per-source counter with red.release.sys once per
//                        (CTA, owner).  No CTA-wide wait: a warp reads source s's rows only after
//                        s's counter shows all of them landed (ld.acquire.sys, per warp and
//                        source, recorded in shared memory for the CTA's other warps), so the
//                        reduction overlaps the exchange.  Reduce: the sorted lookups are cut
//                        into chunks; a warp walks a chunk's runs 32 lookups at a time (lane
//                        groups take different runs when a row needs fewer than 32 lanes), sums
//                        each run in ascending lookup order and applies the SGD step to rows
//                        whose run starts and ends inside the chunk; a run crossing chunk edges
//                        leaves one partial sum per chunk in scratch.
//                        (local) the same reduce from a caller-owned [B][T][D] gradient -- the
//                        unfused baseline's second half after NCCL all_to_all_single.
//   bwd_fold_kernel / bwd_fold_narrow_kernel
//                        pass 2: the chunk a crossing run starts in folds the partials in chunk
//                        order (fixed order: the result does not depend on timing) and updates
//                        the row.  The kernel boundary orders pass 1's partials before it.
#include "fused_kernel.cuh"

namespace emba2a {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Programmatic dependent launch: the next kernel on the stream may be scheduled while this one
// drains (launch_dependents); a kernel waits (griddepcontrol.wait) for its predecessor's grid
// to complete -- and its writes to be visible -- before it reads anything the predecessor wrote.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void st_f4(float* p, const float4& v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// ------------------------------------------------------------------------------ sort plan
// Keys of this rank's lookups and the digit histograms of every pass.  A warp takes 8
// consecutive bags; their lookups are one contiguous range, walked 32 positions at a time
// (coalesced), each position's bag found by a 3-step binary search over the 8 bag starts.
template <bool WEIGHTED>
__global__ void __launch_bounds__(256) bwd_keygen_kernel(const SortParams S) {
  constexpr int BPW = 8;
  __shared__ unsigned h[kMaxPasses * 256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) h[i] = 0u;
  pdl_wait();     // the caller's indices/offsets and the previous plan's passes are complete
  pdl_trigger();  // pass 0's CTAs may take their slots and wait
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.lbg_words;
       i += (long long)gridDim.x * blockDim.x)
    S.lbg[i] = 0u;                     // the passes' group look-back words (they follow keygen)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kHistWords; i += gridDim.x * blockDim.x)
    S.hist_clear[i] = 0u;              // the next plan's digit counts and tile tickets
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long ngroups = (S.TB + BPW - 1) / BPW;
  const long long nwt = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; grp < ngroups;
       grp += nwt) {
    const long long b0 = grp * BPW;
    const int nb = (S.TB - b0) < BPW ? (int)(S.TB - b0) : BPW;
    const int my_off = lane < nb ? S.offsets[b0 + lane] : 0x7fffffff;
    const int lo = __shfl_sync(kFull, my_off, 0);
    const int hi = S.offsets[b0 + nb];
    // the group's lookups are requested UNROLL x 32 at a time before any key is stored (the
    // stores could alias the loads, so the compiler would not hoist them itself)
    constexpr int UNROLL = 8;
    for (int base0 = lo; base0 < hi; base0 += 32 * UNROLL) {
      int ix[UNROLL];
      float wv[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int p = base0 + 32 * u + lane;
        ix[u] = p < hi ? S.indices[p] : 0;
        if (WEIGHTED) wv[u] = p < hi ? S.weights[p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int p = base0 + 32 * u + lane;
        if (base0 + 32 * u >= hi) break;            // warp-uniform
        int i = 0;
#pragma unroll
        for (int step = BPW / 2; step >= 1; step >>= 1) {
          const int v = __shfl_sync(kFull, my_off, i + step);
          if (i + step < nb && v <= p) i += step;
        }
        if (p < hi) {
          const long long bag = b0 + i;
          const unsigned t = (unsigned)(bag / S.B);
          const unsigned key = (S.rbits >= 32 ? 0u : (t << S.rbits)) | (unsigned)ix[u];
          S.keys[p] = key;
          S.bags[p] = (int)bag;
          if (WEIGHTED) S.wts[p] = wv[u];
          for (int q = 0; q < S.passes; ++q)   // the last digit may be narrower
            atomicAdd(&h[q * 256 + ((key >> (S.hshift + 8 * q)) &
                                    (q == S.passes - 1 ? S.last_mask : 255u))],
                      1u);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S.passes * 256; i += blockDim.x)
    if (h[i]) atomicAdd(S.hist + i, h[i]);
}

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ unsigned block_excl_scan256(unsigned v, unsigned* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  unsigned base = 0;
  for (int i = 0; i < w; ++i) base += s_warp[i];
  return base + x - v;
}

// Per-CTA timeline of a radix pass (the "trace" option): events 30 start, 31 tile loaded,
// 32 ranked, 33 offsets known, 34 scattered; payload = tile.  Thread 0 only.
__device__ __forceinline__ void ptrace(const PassParams& P, unsigned event, unsigned payload) {
  if (P.trace == nullptr || threadIdx.x != 0) return;
  const unsigned long long i = atomicAdd(P.trace, 1ull);
  if ((long long)i >= P.trace_cap) return;
  P.trace[2 + 2 * i] = ((unsigned long long)blockIdx.x << 40) |
                       ((unsigned long long)event << 32) | payload;
  P.trace[3 + 2 * i] = globaltimer();
}

// Look-back words: [63:34] stamp | [33:32] flag (1 = the tile's digit count published) | [31:0] count
__device__ __forceinline__ unsigned long long lb_word(unsigned stamp, unsigned flag,
                                                      unsigned count) {
  return ((unsigned long long)(stamp & 0x3fffffffu) << 34) | ((unsigned long long)flag << 32) |
         count;
}

// One stable LSD radix pass in ONE kernel (onesweep; used when all tiles fit in one wave, so the
// look-back chains are short and the launch count matters more).  Tile = kSortTile keys; warp w owns keys [w*32*I, (w+1)*32*I) of
// the tile (I = kSortItems), item i of lane l at w*32*I + i*32 + l (warp-striped, so "item,
// then lane" is position order and the ranking below is stable).  The ranked tile is reordered
// by digit in shared memory and written out one contiguous run per digit.
template <bool WEIGHTS>
__global__ void __launch_bounds__(kSortThreads) bwd_onesweep_kernel(const PassParams P) {
  constexpr int NW = kSortThreads / 32;
  static_assert(kSortThreads == 256, "one thread per 8-bit digit");
  __shared__ unsigned s_cnt[NW][256];   // running per-warp digit counts -> warp offsets in tile
  __shared__ unsigned s_hist[256];      // the tile's digit counts
  __shared__ unsigned s_gofs[256];
  __shared__ unsigned s_tstart[256];    // first tile-local slot of each digit
  __shared__ unsigned s_warp[NW];
  __shared__ unsigned s_tile;
  __shared__ unsigned s_key[kSortTile];  // the tile, reordered by digit (coalesced write-out)
  __shared__ int s_bag[kSortTile];
  __shared__ float s_wt[WEIGHTS ? kSortTile : 1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pdl_trigger();
  for (int i = tid; i < NW * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0u;
  s_hist[tid] = 0u;
  pdl_wait();
  if (tid == 0) s_tile = atomicAdd(P.tile_ctr, 1u);
  const unsigned hval = P.hist[tid];   // this pass's count of digit tid (for the global base)
  __syncthreads();
  const long long tile = s_tile;
  ptrace(P, 30, (unsigned)tile);
  const long long base = tile * kSortTile + (long long)w * (32 * kSortItems);
  const unsigned lt_mask = (1u << lane) - 1u;

  unsigned key[kSortItems];
  int bag[kSortItems];
  float wt[kSortItems];
  unsigned short rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const bool valid = pos < P.n;
    key[i] = valid ? P.keys_in[pos] : 0u;
    bag[i] = valid ? P.bags_in[pos] : 0;
    if (WEIGHTS) wt[i] = valid ? P.wts_in[pos] : 0.f;
  }
  if (P.trace) {                       // (tracing only: wait for the loads to time them)
    unsigned x = 0;
    for (int i = 0; i < kSortItems; ++i) x ^= key[i];
    if (x == 0xdeadbeefu) s_tile = x;
    ptrace(P, 31, (unsigned)tile);
  }
  // The tile's digit counts first (one shared add per group of equal digits in a warp), so the
  // tile publishes them -- and the look-back of later tiles can complete -- while it ranks.
  const long long ngroups = (P.ntiles + kLbGroup - 1) / kLbGroup;
  const long long J = tile / kLbGroup, j0 = J * kLbGroup;
  unsigned peers[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const unsigned d = pos < P.n ? ((key[i] >> P.shift) & P.dmask) : 256u;
    peers[i] = __match_any_sync(kFull, d);
    if (d < 256u && lane == __ffs(peers[i]) - 1) atomicAdd(&s_hist[d], __popc(peers[i]));
  }
  __syncthreads();
  const unsigned d = tid;
  const unsigned run = s_hist[d];      // the tile's count of digit d
  // Look-back in two levels.  Tile k of group J = k / G (G = kLbGroup tiles) publishes its
  // digit counts twice: as its stamped look-back word (read by the later tiles of its group)
  // and added into the group's sums, after which one thread counts the tile in on the group's
  // arrival counter (fence + add = release).  The exclusive prefix of tile k = the sums of
  // groups 0 .. J-1 (complete once their counters reach G) + the words of tiles J*G .. k-1.
  // All tiles publish at about the same time, so this is ~3 round trips; a chain of 8-tile
  // look-back windows costs ~k/16 of them.  (Tried: a 64-bit word per group and digit carrying
  // its own tile count, no fence: slower -- 256 threads polling words instead of J counters.)
  // Tiles are taken in ticket order, so every tile waited for is running and will publish;
  // the time bound only guards against a broken invariant hanging the GPU.
  // (debug option "debug_sort_stall": tile 0 publishes a stale stamp, so the later tiles of its
  // group never see it -- the look-back must then time out with an error, not hang or go on)
  st_relaxed_gpu(P.status + tile * 256 + d,
                 lb_word(P.stall && tile == 0 ? P.stamp + 1u : P.stamp, 1, run));
  if (J + 1 < ngroups) atomicAdd(P.gsum + J * 256 + d, run);
  __syncthreads();
  if (tid == 0 && J + 1 < ngroups) {
    __threadfence();
    atomicAdd(P.garrive + J, 1u);
  }
  // stable rank of each key within its warp's digit (warp-striped: item, then lane = position)
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const unsigned dd = pos < P.n ? ((key[i] >> P.shift) & P.dmask) : 256u;
    const unsigned c = dd < 256u ? s_cnt[w][dd] : 0u;
    rank[i] = (unsigned short)(c + __popc(peers[i] & lt_mask));
    __syncwarp();
    if (dd < 256u && lane == __ffs(peers[i]) - 1) s_cnt[w][dd] = c + __popc(peers[i]);
    __syncwarp();
  }
  __syncthreads();
  ptrace(P, 32, (unsigned)tile);
  // thread d: exclusive offsets of digit d per warp
  {
    unsigned acc = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const unsigned c = s_cnt[ww][d];
      s_cnt[ww][d] = acc;
      acc += c;
    }
  }
  const unsigned want = P.stamp & 0x3fffffffu;
  const unsigned long long tb = globaltimer();
  unsigned excl = 0, gbase;
  {
    unsigned long long v[kLbGroup - 1];
#pragma unroll
    for (int i = 0; i < kLbGroup - 1; ++i)
      v[i] = (j0 + i < tile) ? ld_relaxed_gpu(P.status + (j0 + i) * 256 + d) : 0ull;
    // while those are in flight: the digit's global base (exclusive scan of the pass
    // histogram) and its first slot in the tile
    gbase = block_excl_scan256(hval, s_warp);
    __syncthreads();                     // s_warp is reused by the next scan
    s_tstart[d] = block_excl_scan256(run, s_warp);
#pragma unroll
    for (int i = 0; i < kLbGroup - 1; ++i) {
      if (j0 + i >= tile) continue;
      unsigned long long w = v[i];
      while ((unsigned)(w >> 34) != want || ((unsigned)(w >> 32) & 3u) == 0u) {
        if (globaltimer() - tb > (unsigned long long)P.timeout_ns) {
          atomicExch(P.err, 0x4000);   // a broken invariant: report it (ETIMEOUT, handle poisoned)
          break;
        }
        w = ld_relaxed_gpu(P.status + (j0 + i) * 256 + d);
      }
      excl += (unsigned)w;
    }
  }
  if (J > 0) {
    for (long long jj = tid; jj < J; jj += kSortThreads) {
      while (ld_acquire_gpu_u32(P.garrive + jj) < (unsigned)kLbGroup)
        if (globaltimer() - tb > (unsigned long long)P.timeout_ns) {
          atomicExch(P.err, 0x4000);
          break;
        }
    }
    __syncthreads();                   // the acquires above order the group sums read below
    long long jj = 0;
    for (; jj + 8 <= J; jj += 8) {
      unsigned g[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = ld_relaxed_gpu_u32(P.gsum + (jj + i) * 256 + d);
#pragma unroll
      for (int i = 0; i < 8; ++i) excl += g[i];
    }
    for (; jj < J; ++jj) excl += ld_relaxed_gpu_u32(P.gsum + jj * 256 + d);
  }
  s_gofs[d] = gbase + excl;
  __syncthreads();
  ptrace(P, 33, (unsigned)tile);
  // reorder the tile by digit in shared memory, then write each digit's run of keys out
  // contiguously (consecutive threads -> consecutive addresses within a run)
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    if (pos < P.n) {
      const unsigned dd = (key[i] >> P.shift) & P.dmask;
      const unsigned lp = s_tstart[dd] + s_cnt[w][dd] + rank[i];
      s_key[lp] = key[i];
      s_bag[lp] = bag[i];
      if (WEIGHTS) s_wt[lp] = wt[i];
    }
  }
  __syncthreads();
  const long long t0 = tile * kSortTile;
  const int tn = (P.n - t0) < kSortTile ? (int)(P.n - t0) : kSortTile;
  for (int i = tid; i < tn; i += kSortThreads) {
    const unsigned k = s_key[i];
    const unsigned dd = (k >> P.shift) & P.dmask;
    const unsigned out = s_gofs[dd] + (unsigned)i - s_tstart[dd];
    P.keys_out[out] = k;
    P.bags_out[out] = s_bag[i];
    if (WEIGHTS) P.wts_out[out] = s_wt[i];
  }
  if (P.trace) {
    __syncthreads();
    ptrace(P, 34, (unsigned)tile);
  }
}

// One stable LSD radix pass = three kernels (reduce-then-scan: no look-back chains, so tiles of
// one wave do not wait on each other).
//   upsweep:   each tile's digit counts -> cnt[digit][tile]
//   scan:      one CTA per digit: cnt[d][t] <- (keys with a smaller digit) + sum_{t' < t} cnt[d][t']
//              = the global position of tile t's first key with digit d (digit-major order)
//   downsweep: rank each key within its tile (stable), reorder the tile by digit in shared
//              memory, write each digit's run to its global position (contiguous writes)
__global__ void __launch_bounds__(kSortThreads) bwd_upsweep_kernel(const PassParams P) {
  __shared__ unsigned h[256];
  const int tid = threadIdx.x;
  pdl_trigger();
  h[tid] = 0u;
  pdl_wait();
  __syncthreads();
  const long long t0 = (long long)blockIdx.x * kSortTile;
  for (int i = tid; i < kSortTile; i += kSortThreads) {
    const long long pos = t0 + i;
    if (pos < P.n) atomicAdd(&h[(P.keys_in[pos] >> P.shift) & P.dmask], 1u);
  }
  __syncthreads();
  P.cnt[(long long)tid * P.ntiles + blockIdx.x] = h[tid];
}

__global__ void __launch_bounds__(256) bwd_scan_kernel(const PassParams P) {
  __shared__ unsigned s_warp[8];
  __shared__ unsigned s_carry;
  const int tid = threadIdx.x, d = blockIdx.x;
  pdl_trigger();
  pdl_wait();
  // keys with a digit below d (the pass histogram from keygen)
  const unsigned below = block_excl_scan256(P.hist[tid], s_warp);
  if (tid == d) s_carry = below;
  __syncthreads();
  unsigned* row = P.cnt + (long long)d * P.ntiles;
  constexpr int K = 4;                       // consecutive tiles per thread
  for (long long t0 = 0; t0 < P.ntiles; t0 += 256 * K) {
    unsigned x[K], sum = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long t = t0 + (long long)tid * K + k;
      x[k] = t < P.ntiles ? row[t] : 0u;
      sum += x[k];
    }
    const unsigned carry = s_carry;
    __syncthreads();                         // s_warp / s_carry reuse below
    const unsigned ex = block_excl_scan256(sum, s_warp);
    unsigned run = carry + ex;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long t = t0 + (long long)tid * K + k;
      if (t < P.ntiles) row[t] = run;
      run += x[k];
    }
    if (tid == 255) s_carry = run;           // = carry + this block's total
    __syncthreads();
  }
}

// Warp-striped tile: warp w owns keys [w*32*I, (w+1)*32*I) of the tile (I = kSortItems), item i
// of lane l at w*32*I + i*32 + l, so "item, then lane" is position order and the ranking is
// stable.
template <bool WEIGHTS>
__global__ void __launch_bounds__(kSortThreads) bwd_downsweep_kernel(const PassParams P) {
  constexpr int NW = kSortThreads / 32;
  static_assert(kSortThreads == 256, "one thread per 8-bit digit");
  __shared__ unsigned s_cnt[NW][256];   // running per-warp digit counts -> warp offsets in tile
  __shared__ unsigned s_gofs[256];
  __shared__ unsigned s_tstart[256];    // first tile-local slot of each digit
  __shared__ unsigned s_warp[NW];
  __shared__ unsigned s_key[kSortTile];  // the tile, reordered by digit (contiguous write-out)
  __shared__ int s_bag[kSortTile];
  __shared__ float s_wt[WEIGHTS ? kSortTile : 1];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long tile = blockIdx.x;
  pdl_trigger();
  for (int i = tid; i < NW * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0u;
  pdl_wait();
  __syncthreads();
  ptrace(P, 30, (unsigned)tile);
  const long long base = tile * kSortTile + (long long)w * (32 * kSortItems);
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned key[kSortItems];
  int bag[kSortItems];
  float wt[kSortItems];
  unsigned short rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const bool valid = pos < P.n;
    key[i] = valid ? P.keys_in[pos] : 0u;
    bag[i] = valid ? P.bags_in[pos] : 0;
    if (WEIGHTS) wt[i] = valid ? P.wts_in[pos] : 0.f;
  }
  const unsigned d = tid;
  const unsigned gofs = P.cnt[(long long)d * P.ntiles + tile];   // scanned by bwd_scan_kernel
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const unsigned dg = pos < P.n ? ((key[i] >> P.shift) & P.dmask) : 256u;
    const unsigned peers = __match_any_sync(kFull, dg);
    const unsigned c = dg < 256u ? s_cnt[w][dg] : 0u;
    rank[i] = (unsigned short)(c + __popc(peers & lt_mask));
    __syncwarp();
    if (dg < 256u && lane == __ffs(peers) - 1) s_cnt[w][dg] = c + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  ptrace(P, 32, (unsigned)tile);
  // thread d: exclusive offsets of digit d per warp, the tile's count of d
  unsigned run = 0;
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) {
    const unsigned c = s_cnt[ww][d];
    s_cnt[ww][d] = run;
    run += c;
  }
  s_gofs[d] = gofs;
  s_tstart[d] = block_excl_scan256(run, s_warp);
  __syncthreads();
  ptrace(P, 33, (unsigned)tile);
  // reorder the tile by digit in shared memory, then write each digit's run of keys out
  // contiguously (consecutive threads -> consecutive addresses within a run)
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    if (pos < P.n) {
      const unsigned dd = (key[i] >> P.shift) & P.dmask;
      const unsigned lp = s_tstart[dd] + s_cnt[w][dd] + rank[i];
      s_key[lp] = key[i];
      s_bag[lp] = bag[i];
      if (WEIGHTS) s_wt[lp] = wt[i];
    }
  }
  __syncthreads();
  const long long t0 = tile * kSortTile;
  const int tn = (P.n - t0) < kSortTile ? (int)(P.n - t0) : kSortTile;
  for (int i = tid; i < tn; i += kSortThreads) {
    const unsigned k = s_key[i];
    const unsigned dd = (k >> P.shift) & P.dmask;
    const unsigned out = s_gofs[dd] + (unsigned)i - s_tstart[dd];
    P.keys_out[out] = k;
    P.bags_out[out] = s_bag[i];
    if (WEIGHTS) P.wts_out[out] = s_wt[i];
  }
  if (P.trace) {
    __syncthreads();
    ptrace(P, 34, (unsigned)tile);
  }
}

// ------------------------------------------------------------------ segmented sort plan
// The input is table-major (table t's lookups are offsets[t*B] .. offsets[(t+1)*B]) and the sort
// is stable, so sorting every table's segment by ROW alone gives exactly the (table, row) order
// of the plain plan while the digits cover only the row bits: 2 passes of <= 11-bit digits for
// tables of up to 4M rows (DLRM-small: 23-bit keys = 3 plain passes).  Digit counts are kept per
// (table, digit); tiles never straddle tables, and the look-back runs over the earlier tiles of
// the same table only.

// Keys/payloads as in bwd_keygen_kernel, plus the per-(table, digit) counts of both passes.  A
// CTA's bag groups are contiguous (one grid-stride step when TB <= 64 x grid), so their tables
// fall in a window of two: counted in shared memory; anything outside goes to global atomics.
template <bool WEIGHTED>
__global__ void __launch_bounds__(256) bwd_keygen_seg_kernel(const SortParams S) {
  constexpr int BPW = 8;
  extern __shared__ unsigned h[];                // [2 window tables][2 passes][NB]
  const int NB = 1 << S.seg_db;
  const int nwin = 4 * NB;
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) h[i] = 0u;
  pdl_wait();     // the caller's indices/offsets and the previous plan's passes are complete
  pdl_trigger();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.lbg_words;
       i += (long long)gridDim.x * blockDim.x)
    S.lbg[i] = 0u;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S.shist_words;
       i += (long long)gridDim.x * blockDim.x)
    S.shist_clear[i] = 0u;                       // the next plan's counts and tile tickets
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned m0 = (1u << S.seg_db) - 1u;
  const unsigned m1 = S.rbits > S.seg_db ? (1u << (S.rbits - S.seg_db)) - 1u : 0u;
  const long long ngroups = (S.TB + BPW - 1) / BPW;
  const long long nwt = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long tw = ((long long)blockIdx.x * (blockDim.x >> 5) * BPW) / S.B;   // window base
  for (long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; grp < ngroups;
       grp += nwt) {
    const long long b0 = grp * BPW;
    const int nb = (S.TB - b0) < BPW ? (int)(S.TB - b0) : BPW;
    const int my_off = lane < nb ? S.offsets[b0 + lane] : 0x7fffffff;
    const int lo = __shfl_sync(kFull, my_off, 0);
    const int hi = S.offsets[b0 + nb];
    constexpr int UNROLL = 8;
    for (int base0 = lo; base0 < hi; base0 += 32 * UNROLL) {
      int ix[UNROLL];
      float wv[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int p = base0 + 32 * u + lane;
        ix[u] = p < hi ? S.indices[p] : 0;
        if (WEIGHTED) wv[u] = p < hi ? S.weights[p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int p = base0 + 32 * u + lane;
        if (base0 + 32 * u >= hi) break;            // warp-uniform
        int i = 0;
#pragma unroll
        for (int step = BPW / 2; step >= 1; step >>= 1) {
          const int v = __shfl_sync(kFull, my_off, i + step);
          if (i + step < nb && v <= p) i += step;
        }
        if (p < hi) {
          const long long bag = b0 + i;
          const unsigned t = (unsigned)(bag / S.B);
          const unsigned row = (unsigned)ix[u];
          S.keys[p] = (t << S.rbits) | row;
          S.bags[p] = (int)bag;
          if (WEIGHTED) S.wts[p] = wv[u];
          const unsigned d0 = row & m0, d1 = (row >> S.seg_db) & m1;
          const long long wl = (long long)t - tw;
          if (wl == 0 || wl == 1) {
            atomicAdd(&h[((int)wl * 2 + 0) * NB + d0], 1u);
            atomicAdd(&h[((int)wl * 2 + 1) * NB + d1], 1u);
          } else {
            atomicAdd(S.shist + ((size_t)t) * NB + d0, 1u);
            atomicAdd(S.shist + ((size_t)S.T + t) * NB + d1, 1u);
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nwin; i += blockDim.x) {
    const unsigned c = h[i];
    if (!c) continue;
    const long long t = tw + i / (2 * NB);
    const int p = (i / NB) & 1, d = i % NB;
    if (t < S.T) atomicAdd(S.shist + ((size_t)p * S.T + t) * NB + d, c);
  }
}

// Exclusive scan over NB = 256 * DPT values, DPT consecutive values per thread: returns each of
// this thread's exclusive prefixes in x[] (in place) and the block total.
template <int DPT>
__device__ __forceinline__ unsigned block_excl_scan_dpt(unsigned (&x)[DPT], unsigned* s_warp) {
  unsigned tot = 0;
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    const unsigned v = x[k];
    x[k] = tot;
    tot += v;
  }
  const unsigned base = block_excl_scan256(tot, s_warp);
#pragma unroll
  for (int k = 0; k < DPT; ++k) x[k] += base;
  __syncthreads();                          // s_warp reused by the caller's next scan
  return base + tot;
}

// One stable LSD pass over the row digit of every table segment (onesweep, tiles aligned to
// tables, taken in ticket order).  Same structure as bwd_onesweep_kernel; NB = 2^DB digits,
// DPT = NB / 256 consecutive digits per thread in the digit-wise steps.
template <bool WEIGHTS, int DB>
__global__ void __launch_bounds__(kSortThreads) bwd_onesweep_seg_kernel(const PassParams P) {
  constexpr int NW = kSortThreads / 32;
  constexpr int NB = 1 << DB;
  constexpr int DPT = NB / kSortThreads;
  static_assert(DPT >= 1 && kSortThreads == 256, "digits per thread");
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned short* s_cnt = reinterpret_cast<unsigned short*>(sm);          // [NW][NB]
  unsigned* s_hist = reinterpret_cast<unsigned*>(sm + (size_t)NW * NB * 2);  // [NB] -> tile start
  unsigned* s_gofs = s_hist + NB;                                          // [NB]
  unsigned* s_key = s_gofs + NB;                                           // [tile]
  int* s_bag = reinterpret_cast<int*>(s_key + kSortTile);
  float* s_wt = reinterpret_cast<float*>(s_bag + kSortTile);
  __shared__ unsigned s_warp[NW];
  __shared__ unsigned s_tile, s_ntiles;
  __shared__ int s_t;
  __shared__ unsigned s_tpre[kSortThreads], s_gpre[kSortThreads];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pdl_trigger();
  for (int i = tid; i < NW * NB / 2; i += kSortThreads) reinterpret_cast<unsigned*>(s_cnt)[i] = 0u;
  for (int i = tid; i < NB; i += kSortThreads) s_hist[i] = 0u;
  pdl_wait();
  if (tid == 0) s_tile = atomicAdd(P.tile_ctr, 1u);
  // table map: tiles and look-back groups per table (T <= 256, one table per thread)
  long long o_t = 0, n_t = 0;
  unsigned nt = 0, ng = 0;
  if (tid < P.T) {
    o_t = P.offsets[(long long)tid * P.B];
    n_t = P.offsets[(long long)(tid + 1) * P.B] - o_t;
    nt = (unsigned)((n_t + kSortTile - 1) / kSortTile);
    ng = (nt + kSegLb - 1) / kSegLb;
  }
  const unsigned tpre = block_excl_scan256(nt, s_warp);
  __syncthreads();
  const unsigned gpre = block_excl_scan256(ng, s_warp);
  s_tpre[tid] = tpre;
  s_gpre[tid] = gpre;
  if (tid == kSortThreads - 1) s_ntiles = tpre + nt;
  __syncthreads();
  const unsigned g = s_tile;
  if (g >= s_ntiles) return;                 // surplus ticket (the grid is an upper bound)
  if (tid < P.T && nt > 0 && g >= tpre && g < tpre + nt) s_t = tid;
  __syncthreads();
  const int t = s_t;
  const long long seg0 = P.offsets[(long long)t * P.B];
  const long long segn = P.offsets[(long long)(t + 1) * P.B] - seg0;
  const unsigned j = g - s_tpre[t];                    // tile index within the table
  const unsigned ntt = (unsigned)((segn + kSortTile - 1) / kSortTile);
  const unsigned ngt = (ntt + kSegLb - 1) / kSegLb;
  const unsigned J = j / kSegLb, j0 = J * kSegLb;      // look-back group within the table
  const unsigned gg = s_gpre[t] + J;                   // its global group id
  const long long start = seg0 + (long long)j * kSortTile;
  const int len = (segn - (long long)j * kSortTile) < kSortTile
                      ? (int)(segn - (long long)j * kSortTile) : kSortTile;
  const int base = w * (32 * kSortItems);
  const unsigned lt_mask = (1u << lane) - 1u;

  unsigned key[kSortItems];
  int bag[kSortItems];
  float wt[kSortItems];
  unsigned short rank[kSortItems];
  unsigned peers[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int pos = base + i * 32 + lane;
    const bool valid = pos < len;
    key[i] = valid ? P.keys_in[start + pos] : 0u;
    bag[i] = valid ? P.bags_in[start + pos] : 0;
    if (WEIGHTS) wt[i] = valid ? P.wts_in[start + pos] : 0.f;
  }
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int pos = base + i * 32 + lane;
    const unsigned d = pos < len ? ((key[i] >> P.shift) & P.dmask) : (unsigned)NB;
    peers[i] = __match_any_sync(kFull, d);
    if (d < (unsigned)NB && lane == __ffs(peers[i]) - 1) atomicAdd(&s_hist[d], __popc(peers[i]));
  }
  __syncthreads();
  unsigned run[DPT];
#pragma unroll
  for (int k = 0; k < DPT; ++k) run[k] = s_hist[tid * DPT + k];
  // publish: the tile's stamped words (read by the later tiles of its group) and, unless this is
  // the table's last group, the group's digit sums + one arrival
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    const unsigned d = tid * DPT + k;
    st_relaxed_gpu(P.status + (size_t)g * NB + d,
                   lb_word(P.stall && g == 0 ? P.stamp + 1u : P.stamp, 1, run[k]));
    if (J + 1 < ngt && run[k]) atomicAdd(P.gsum + (size_t)gg * NB + d, run[k]);
  }
  __syncthreads();
  if (tid == 0 && J + 1 < ngt) {
    __threadfence();
    atomicAdd(P.garrive + gg, 1u);
  }
  // stable rank of each key within its warp's digit
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int pos = base + i * 32 + lane;
    const unsigned dd = pos < len ? ((key[i] >> P.shift) & P.dmask) : (unsigned)NB;
    const unsigned c = dd < (unsigned)NB ? s_cnt[w * NB + dd] : 0u;
    rank[i] = (unsigned short)(c + __popc(peers[i] & lt_mask));
    __syncwarp();
    if (dd < (unsigned)NB && lane == __ffs(peers[i]) - 1)
      s_cnt[w * NB + dd] = (unsigned short)(c + __popc(peers[i]));
    __syncwarp();
  }
  __syncthreads();
  // per-warp exclusive offsets of my digits
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    const int d = tid * DPT + k;
    unsigned acc = 0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      const unsigned c = s_cnt[ww * NB + d];
      s_cnt[ww * NB + d] = (unsigned short)acc;
      acc += c;
    }
  }
  // look-back over the earlier tiles of this table: the words of tiles j0 .. j-1 of its group,
  // then the sums of its earlier (complete) groups
  const unsigned want = P.stamp & 0x3fffffffu;
  const unsigned long long tb = globaltimer();
  unsigned excl[DPT];
#pragma unroll
  for (int k = 0; k < DPT; ++k) excl[k] = 0u;
  {
    unsigned long long v[kSegLb - 1][DPT];
#pragma unroll
    for (int i = 0; i < kSegLb - 1; ++i)
#pragma unroll
      for (int k = 0; k < DPT; ++k)
        v[i][k] = (j0 + i < j) ? ld_relaxed_gpu(P.status + (size_t)(g - (j - j0 - i)) * NB +
                                                tid * DPT + k)
                               : 0ull;
    // while those are in flight: the table's digit base and the tile's first slot per digit
    unsigned gb[DPT], ts[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      gb[k] = P.shist[(size_t)t * NB + tid * DPT + k];
      ts[k] = run[k];
    }
    block_excl_scan_dpt<DPT>(gb, s_warp);
    block_excl_scan_dpt<DPT>(ts, s_warp);
#pragma unroll
    for (int k = 0; k < DPT; ++k) s_hist[tid * DPT + k] = ts[k];   // tile start of each digit
#pragma unroll
    for (int i = 0; i < kSegLb - 1; ++i) {
      if (j0 + i >= j) continue;
#pragma unroll
      for (int k = 0; k < DPT; ++k) {
        unsigned long long x = v[i][k];
        while ((unsigned)(x >> 34) != want || ((unsigned)(x >> 32) & 3u) == 0u) {
          if (globaltimer() - tb > (unsigned long long)P.timeout_ns) {
            atomicExch(P.err, 0x4000);
            break;
          }
          x = ld_relaxed_gpu(P.status + (size_t)(g - (j - j0 - i)) * NB + tid * DPT + k);
        }
        excl[k] += (unsigned)x;
      }
    }
    if (J > 0) {
      const unsigned gfirst = s_gpre[t];
      for (unsigned jj = tid; jj < J; jj += kSortThreads) {
        while (ld_acquire_gpu_u32(P.garrive + gfirst + jj) < (unsigned)kSegLb)
          if (globaltimer() - tb > (unsigned long long)P.timeout_ns) {
            atomicExch(P.err, 0x4000);
            break;
          }
      }
      __syncthreads();                 // the acquires above order the group sums read below
      for (unsigned jj = 0; jj < J; ++jj)
#pragma unroll
        for (int k = 0; k < DPT; ++k)
          excl[k] += ld_relaxed_gpu_u32(P.gsum + (size_t)(gfirst + jj) * NB + tid * DPT + k);
    }
#pragma unroll
    for (int k = 0; k < DPT; ++k)
      s_gofs[tid * DPT + k] = (unsigned)seg0 + gb[k] + excl[k];
  }
  __syncthreads();
  // reorder the tile by digit in shared memory, then write each digit's run out contiguously
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int pos = base + i * 32 + lane;
    if (pos < len) {
      const unsigned dd = (key[i] >> P.shift) & P.dmask;
      const unsigned lp = s_hist[dd] + s_cnt[w * NB + dd] + rank[i];
      s_key[lp] = key[i];
      s_bag[lp] = bag[i];
      if (WEIGHTS) s_wt[lp] = wt[i];
    }
  }
  __syncthreads();
  for (int i = tid; i < len; i += kSortThreads) {
    const unsigned k = s_key[i];
    const unsigned dd = (k >> P.shift) & P.dmask;
    const unsigned out = s_gofs[dd] + (unsigned)i - s_hist[dd];
    P.keys_out[out] = k;
    P.bags_out[out] = s_bag[i];
    if (WEIGHTS) P.wts_out[out] = s_wt[i];
  }
}

// Exclusive scan of one value per thread over a block of NW warps.
template <int NW>
__device__ __forceinline__ unsigned block_excl_scan_nw(unsigned v, unsigned* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  unsigned base = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) base += i < w ? s_warp[i] : 0u;
  __syncthreads();                     // s_warp may be reused right after
  return base + x - v;
}

// ------------------------------------------------------------------- bucket sort plan
// sort_mode 5: keygen (histogram of the TOP 8 key bits only), one stable onesweep pass on that
// top digit -- 256 buckets, each a contiguous, position-ordered range -- then ONE kernel sorts
// every bucket on its own by the remaining low bits (stable LSD passes of 8 bits), one CTA per
// bucket, entirely in shared memory: no cross-CTA coordination after the first pass, so the
// look-back chains and kernel boundaries of passes 2.. disappear.  A bucket larger than the
// shared-memory capacity is sorted the same way in global memory (the plan's ping-pong buffers).
// Same stable order as the plain plan: MSD on the top digit, then LSD within each bucket.
struct BucketParams {
  const unsigned* keys_in;     // after the top-digit pass (buffer 1)
  const int* bags_in;
  const float* wts_in;
  unsigned* keys_out;          // the plan's output (buffer 0)
  int* bags_out;
  float* wts_out;
  const unsigned* hist;        // [256] top-digit counts (keygen)
  int low_bits;                // key bits below the top digit
  int cap;                     // keys a bucket may have to sort in shared memory
};

// 256 threads x 8 keys per tile (measured r02at/r02au: 1024 threads x 4 only moved DLRM-small's
// bucket kernel 30.4 -> 27.4 us and slowed sweep P=1's plan 32.5 -> 38.7 us)
constexpr int kBktThreads = 256;
constexpr int kBktItems = 8;
template <bool WEIGHTS>
__global__ void __launch_bounds__(kBktThreads, 1) bwd_bucket_sort_kernel(const BucketParams P) {
  constexpr int NT = kBktThreads, NW = NT / 32, K = kBktItems, TILE = NT * K;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_base[256], s_run[256], s_tot[256], s_warp[NW];
  __shared__ unsigned short s_cnt[NW][256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  pdl_wait();     // the top-digit pass is complete
  pdl_trigger();
  const unsigned hv = tid < 256 ? P.hist[tid] : 0u;
  const unsigned start = block_excl_scan_nw<NW>(hv, s_warp);
  if (tid == blockIdx.x) s_base[0] = start;            // (s_base reused below)
  __syncthreads();
  const unsigned b0 = s_base[0];
  const int nb = (int)P.hist[blockIdx.x];
  if (nb == 0) return;
  const int passes = (P.low_bits + 7) / 8;
  const bool in_smem = nb <= P.cap;
  // ping-pong: shared memory (two arrays of cap) or the plan's global buffers
  unsigned* sk[2];
  int* sb[2];
  float* sw[2];
  sk[0] = reinterpret_cast<unsigned*>(smem);
  sb[0] = reinterpret_cast<int*>(sk[0] + P.cap);
  sw[0] = reinterpret_cast<float*>(sb[0] + P.cap);
  sk[1] = reinterpret_cast<unsigned*>(sw[0] + (WEIGHTS ? P.cap : 0));
  sb[1] = reinterpret_cast<int*>(sk[1] + P.cap);
  sw[1] = reinterpret_cast<float*>(sb[1] + P.cap);
  unsigned* gk[2] = {const_cast<unsigned*>(P.keys_in) + b0, P.keys_out + b0};
  int* gb[2] = {const_cast<int*>(P.bags_in) + b0, P.bags_out + b0};
  float* gw[2] = {WEIGHTS ? const_cast<float*>(P.wts_in) + b0 : nullptr,
                  WEIGHTS ? P.wts_out + b0 : nullptr};
  int cur = 0;                                  // index of the array holding the current order
  if (in_smem) {
    for (int i = tid; i < nb; i += NT) {
      sk[0][i] = __ldcg(gk[0] + i);
      sb[0][i] = __ldcg(gb[0] + i);
      if (WEIGHTS) sw[0][i] = __ldcg(gw[0] + i);
    }
    __syncthreads();
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    const unsigned dmask = (1u << min(8, P.low_bits - shift)) - 1u;
    // (selects, not runtime indexing: keeps the pointers in registers)
    unsigned* const kin = in_smem ? (cur ? sk[1] : sk[0]) : (cur ? gk[1] : gk[0]);
    int* const bin = in_smem ? (cur ? sb[1] : sb[0]) : (cur ? gb[1] : gb[0]);
    float* const win = in_smem ? (cur ? sw[1] : sw[0]) : (cur ? gw[1] : gw[0]);
    unsigned* const kout = in_smem ? (cur ? sk[0] : sk[1]) : (cur ? gk[0] : gk[1]);
    int* const bout = in_smem ? (cur ? sb[0] : sb[1]) : (cur ? gb[0] : gb[1]);
    float* const wout = in_smem ? (cur ? sw[0] : sw[1]) : (cur ? gw[0] : gw[1]);
    // the bucket's digit counts -> exclusive base per digit
    if (tid < 256) s_tot[tid] = 0u;
    __syncthreads();
    {
      // 8 keys per thread in flight (global path: one round trip per 8 x NT keys)
      constexpr int LB = 8;
      for (int i0 = 0; i0 < nb; i0 += LB * NT) {
        unsigned kk[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int i = i0 + u * NT + tid;
          kk[u] = i < nb ? (in_smem ? kin[i] : __ldcg(kin + i)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < LB; ++u)
          if (i0 + u * NT + tid < nb) atomicAdd(&s_tot[(kk[u] >> shift) & dmask], 1u);
      }
    }
    __syncthreads();
    {
      const unsigned ex = block_excl_scan_nw<NW>(tid < 256 ? s_tot[tid] : 0u, s_warp);
      if (tid < 256) s_run[tid] = ex;
    }
    __syncthreads();
    for (int base = 0; base < nb; base += TILE) {
      unsigned key[K], dg[K];
      int bag[K];
      float wt[K];
      unsigned short rank[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int pos = base + w * (32 * K) + i * 32 + lane;
        const bool valid = pos < nb;
        key[i] = valid ? (in_smem ? kin[pos] : __ldcg(kin + pos)) : 0u;
        bag[i] = valid ? (in_smem ? bin[pos] : __ldcg(bin + pos)) : 0;
        if (WEIGHTS) wt[i] = valid ? (in_smem ? win[pos] : __ldcg(win + pos)) : 0.f;
        dg[i] = valid ? ((key[i] >> shift) & dmask) : 256u;
      }
      for (int i = tid; i < NW * 256 / 2; i += NT)
        reinterpret_cast<unsigned*>(&s_cnt[0][0])[i] = 0u;
      __syncthreads();
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const unsigned peers = __match_any_sync(kFull, dg[i]);
        const unsigned c = dg[i] < 256u ? s_cnt[w][dg[i]] : 0u;
        rank[i] = (unsigned short)(c + __popc(peers & lt_mask));
        __syncwarp();
        if (dg[i] < 256u && lane == __ffs(peers) - 1)
          s_cnt[w][dg[i]] = (unsigned short)(c + __popc(peers));
        __syncwarp();
      }
      __syncthreads();
      if (tid < 256) {
        unsigned acc = 0;
#pragma unroll 8
        for (int ww = 0; ww < NW; ++ww) {
          const unsigned x = s_cnt[ww][tid];
          s_cnt[ww][tid] = (unsigned short)acc;
          acc += x;
        }
        s_tot[tid] = acc;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (dg[i] >= 256u) continue;
        const unsigned o = s_run[dg[i]] + s_cnt[w][dg[i]] + rank[i];
        kout[o] = key[i];
        bout[o] = bag[i];
        if (WEIGHTS) wout[o] = wt[i];
      }
      __syncthreads();
      if (tid < 256) s_run[tid] += s_tot[tid];
      __syncthreads();
    }
    cur ^= 1;
    if (!in_smem) __threadfence_block();
    __syncthreads();
  }
  // the result into the plan's output buffer (global index 1 = keys_out)
  if (in_smem) {
    const unsigned* const fk = cur ? sk[1] : sk[0];
    const int* const fb = cur ? sb[1] : sb[0];
    const float* const fw = cur ? sw[1] : sw[0];
    for (int i = tid; i < nb; i += NT) {
      gk[1][i] = fk[i];
      gb[1][i] = fb[i];
      if (WEIGHTS) gw[1][i] = fw[i];
    }
  } else if (cur == 0) {              // global ping-pong ended in the input buffer: copy over
    for (int i = tid; i < nb; i += NT) {
      gk[1][i] = __ldcg(gk[0] + i);
      gb[1][i] = __ldcg(gb[0] + i);
      if (WEIGHTS) gw[1][i] = __ldcg(gw[0] + i);
    }
  }
}

// ------------------------------------------------------------------- cluster sort plan
// sort_mode 4: the whole plan in ONE kernel, one thread-block cluster of C CTAs per table.  The
// input is table-major and the sort stable, so each table's segment is sorted by its row bits
// alone (the segmented plan's observation) -- and a segment is small enough for one cluster to
// own it, so the digit offsets of every pass are exchanged between the cluster's CTAs through
// distributed shared memory and the passes are separated by cluster barriers: no global
// look-back, no stamped words, no tile tickets and no kernel boundary between keygen and the
// passes (the plain plan's 4 launches and their look-back round trips).
//
// CTA c of table t's cluster owns the strip of the segment made of bags
// [t*B + c*B/C, t*B + (c+1)*B/C) (contiguous positions, strips in CTA order).  It generates those
// keys (counting pass 0's digits as it goes), then in every pass: (1) counts its strip's digits,
// (2) after a cluster barrier reads the C strips' counts (DSMEM) -- digit d of strip c starts at
// seg_lo + (keys of the segment with a smaller digit) + (digit-d keys of strips 0..c-1) --
// and (3) scatters its strip tile by tile in position order with the onesweep kernel's stable
// warp-striped ranks; a cluster barrier (release/acquire at cluster scope: global stores too)
// ends the pass.  Same key order as the plain plan, hence the same plan.

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// DPT consecutive 32-bit words at this CTA's shared address `addr`, read from cluster CTA `rank`
template <int DPT>
__device__ __forceinline__ void ld_dsmem(unsigned addr, unsigned rank, unsigned (&v)[DPT]) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(rank));
  if constexpr (DPT == 1) {
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v[0]) : "r"(ra) : "memory");
  } else if constexpr (DPT == 2) {
    asm volatile("ld.shared::cluster.v2.u32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(ra)
                 : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < DPT; k += 4)
      asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[k]), "=r"(v[k + 1]), "=r"(v[k + 2]), "=r"(v[k + 3])
                   : "r"(ra + 4u * k)
                   : "memory");
  }
}


// Per-CTA timeline of the cluster plan (the "trace" option): events 40 start, 41 keys generated,
// then per pass (payload = pass) 43 the pass's counts complete (cluster barrier), 44 offsets
// known, 45 strip written; 46 the cluster done.  Thread 0 only.
__device__ __forceinline__ void ctrace(const ClusterSortParams& S, unsigned event, unsigned payload) {
  if (S.trace == nullptr || threadIdx.x != 0) return;
  const unsigned long long i = atomicAdd(S.trace, 1ull);
  if ((long long)i >= S.trace_cap) return;
  S.trace[2 + 2 * i] = ((unsigned long long)blockIdx.x << 40) |
                       ((unsigned long long)event << 32) | payload;
  S.trace[3 + 2 * i] = globaltimer();
}

// One CTA = kClThreads threads; a tile = kClThreads * kClItems positions, warp w owning
// [w*32*I, (w+1)*32*I) of it, item i of lane l at w*32*I + i*32 + l (warp-striped: "item, then
// lane" is position order, so the match.any ranks are stable).  A pass over the strip, tile by
// tile: rank (per-warp digit counts), reorder the tile by digit in shared memory, write each
// digit's run out contiguously (coalesced; a 4-byte scatter per key costs the SM one L2 sector
// per key: measured 4-5 us per pass for ~2.5 K keys per CTA), and -- while writing -- count the
// NEXT pass's digit of every key into the counts of the CTA whose strip the key lands in
// (red.shared::cluster), so a pass needs one cluster barrier and no counting sweep.  Counts
// rotate over three buffers: pass p reads buffer p%3, its write-out adds to (p+1)%3, and
// (p+2)%3 -- last read in pass p-1, next written in pass p+1 -- is zeroed during pass p.
constexpr int kClThreads = 256;
constexpr int kClItems = 12;
constexpr int kClTile = kClThreads * kClItems;
constexpr int kClMaxC = 16;
size_t cluster_smem(int db, bool weights) {
  const size_t ND = (size_t)1 << (db <= 8 ? 8 : db);
  return ND * 4 * 6 + (size_t)(kClThreads / 32) * ND * 2 + (size_t)kClTile * (weights ? 12 : 8);
}
template <bool WEIGHTED, int DB>
__global__ void __launch_bounds__(kClThreads, 2) bwd_cluster_sort_kernel(const ClusterSortParams S) {
  constexpr int ND = 1 << DB, NW = kClThreads / 32, K = kClItems, TILE = kClTile;
  constexpr int DPT = ND / kClThreads, BPW = 32;
  static_assert(DPT >= 1 && DPT <= 8, "1..8 digits per thread");
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* s_hist = reinterpret_cast<unsigned*>(smem);   // [3][ND] strip digit counts (cluster)
  unsigned* s_run = s_hist + 3 * ND;                      // [ND] next output slot per digit
  unsigned* s_tstart = s_run + ND;                        // [ND] first tile slot per digit
  unsigned* s_gofs = s_tstart + ND;                       // [ND] output slot of the tile's run
  unsigned short* s_cnt = reinterpret_cast<unsigned short*>(s_gofs + ND);   // [NW][ND]
  unsigned* s_key = reinterpret_cast<unsigned*>(s_cnt + NW * ND);          // [TILE]
  int* s_bag = reinterpret_cast<int*>(s_key + TILE);                       // [TILE]
  float* s_wt = reinterpret_cast<float*>(s_bag + TILE);                    // [TILE] (weighted)
  __shared__ unsigned s_warp[NW];
  __shared__ unsigned s_sb[kClMaxC + 1];                  // strip starts of the cluster's CTAs
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned C = (unsigned)S.C, c = cluster_ctarank();
  const long long t = blockIdx.x / S.C;
  for (int i = tid; i < 3 * ND; i += kClThreads) s_hist[i] = 0u;
  for (int i = tid; i < NW * ND / 2; i += kClThreads) reinterpret_cast<unsigned*>(s_cnt)[i] = 0u;
  pdl_wait();     // the caller's indices/offsets and the previous plan's readers are complete
  pdl_trigger();
  if (tid <= (int)C) s_sb[tid] = (unsigned)S.offsets[t * S.B + ((long long)tid * S.B) / C];
  const long long jlo = t * S.B + ((long long)c * S.B) / C;
  const long long jhi = t * S.B + ((long long)(c + 1) * S.B) / C;
  const long long seg_lo = S.offsets[t * S.B];
  const long long s0 = S.offsets[jlo], s1 = S.offsets[jhi];
  const unsigned mask0 = S.passes > 0 ? (1u << min(S.db, S.rbits)) - 1u : 0u;
  ctrace(S, 40, 0);
  // (every CTA's count buffers are zeroed above, before its pass-0 barrier; remote adds start
  // after that barrier)
  // ---- keygen over this strip's bags: a warp takes 32 bags (one offset per lane), walks their
  //      lookups UNROLL x 32 at a time, finds each lookup's bag by a 5-step search over the
  //      lanes' offsets; pass 0's digit counts on the side
  {
    unsigned* const keys = S.keys[0];
    int* const bags = S.bags[0];
    float* const wts = S.wts[0];
    for (long long b0 = jlo + (long long)w * BPW; b0 < jhi; b0 += (long long)NW * BPW) {
      const int nb = (jhi - b0) < BPW ? (int)(jhi - b0) : BPW;
      const int my_off = lane < nb ? S.offsets[b0 + lane] : 0x7fffffff;
      const int lo = __shfl_sync(kFull, my_off, 0);
      const int hi = S.offsets[b0 + nb];
      constexpr int UNROLL = 12;
      for (int base0 = lo; base0 < hi; base0 += 32 * UNROLL) {
        int ix[UNROLL];
        float wv[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const int p = base0 + 32 * u + lane;
          ix[u] = p < hi ? S.indices[p] : 0;
          if (WEIGHTED) wv[u] = p < hi ? S.weights[p] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          const int p = base0 + 32 * u + lane;
          if (base0 + 32 * u >= hi) break;            // warp-uniform
          int i = 0;
#pragma unroll
          for (int step = BPW / 2; step >= 1; step >>= 1) {
            const int v = __shfl_sync(kFull, my_off, i + step);
            if (i + step < nb && v <= p) i += step;
          }
          const unsigned row = (unsigned)ix[u];
          unsigned d = (unsigned)ND;                   // invalid: counted nowhere
          if (p < hi) {
            const long long bag = b0 + i;
            keys[p] = ((unsigned)(bag / S.B) << S.rbits) | row;
            bags[p] = (int)bag;
            if (WEIGHTED) wts[p] = wv[u];
            d = row & mask0;
          }
          const unsigned peers = __match_any_sync(kFull, d);
          if (d < (unsigned)ND && lane == __ffs(peers) - 1) atomicAdd(&s_hist[d], __popc(peers));
        }
      }
    }
  }
  ctrace(S, 41, 0);
  const unsigned lt_mask = (1u << lane) - 1u;
  const long long wbase = (long long)w * (32 * K);
  for (int p = 0; p < S.passes; ++p) {
    const int shift = p * S.db;
    const unsigned dmask = (1u << min(S.db, S.rbits - shift)) - 1u;
    const bool last = p == S.passes - 1;
    const int shift2 = shift + S.db;
    const unsigned dmask2 = last ? 0u : (1u << min(S.db, S.rbits - shift2)) - 1u;
    const bool odd = p & 1;            // (selects, not indexing: keeps the params in registers)
    const unsigned* const kin = odd ? S.keys[1] : S.keys[0];
    const int* const bin = odd ? S.bags[1] : S.bags[0];
    const float* const win = odd ? S.wts[1] : S.wts[0];
    unsigned* const kout = odd ? S.keys[0] : S.keys[1];
    int* const bout = odd ? S.bags[0] : S.bags[1];
    float* const wout = odd ? S.wts[0] : S.wts[1];
    unsigned* const h_cur = s_hist + (p % 3) * ND;
    const unsigned h_next = smem_u32(s_hist + ((p + 1) % 3) * ND);
    cluster_barrier();                 // counts of this pass complete; pass p-1's keys in place
    ctrace(S, 43, p);
    {
      unsigned* const h_free = s_hist + ((p + 2) % 3) * ND;   // read in pass p-1, written in p+1
      for (int i = tid; i < ND; i += kClThreads) h_free[i] = 0u;
    }
    // digit offsets: thread tid owns digits tid*DPT .. +DPT-1 and reads their counts in every
    // strip of the cluster (DSMEM)
    {
      unsigned tot[DPT], bef[DPT];
#pragma unroll
      for (int k = 0; k < DPT; ++k) tot[k] = bef[k] = 0u;
      const unsigned a = smem_u32(h_cur + tid * DPT);
#pragma unroll 4
      for (unsigned q = 0; q < C; ++q) {
        unsigned v[DPT];
        ld_dsmem<DPT>(a, q, v);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
          tot[k] += v[k];
          if (q < c) bef[k] += v[k];
        }
      }
      block_excl_scan_dpt<DPT>(tot, s_warp);
#pragma unroll
      for (int k = 0; k < DPT; ++k) s_run[tid * DPT + k] = (unsigned)seg_lo + tot[k] + bef[k];
    }
    __syncthreads();
    ctrace(S, 44, p);
    for (long long base = s0; base < s1; base += TILE) {
      unsigned key[K], dg[K];
      int bag[K];
      float wt[K];
      unsigned short rank[K];
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const long long pos = base + wbase + i * 32 + lane;
        const bool valid = pos < s1;
        key[i] = valid ? __ldcg(kin + pos) : 0u;
        bag[i] = valid ? __ldcg(bin + pos) : 0;
        if (WEIGHTED) wt[i] = valid ? __ldcg(win + pos) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const long long pos = base + wbase + i * 32 + lane;
        dg[i] = pos < s1 ? ((key[i] >> shift) & dmask) : (unsigned)ND;
        if (base + wbase + i * 32 >= s1) continue;     // warp-uniform
        const unsigned peers = __match_any_sync(kFull, dg[i]);
        const unsigned cur = dg[i] < (unsigned)ND ? s_cnt[w * ND + dg[i]] : 0u;
        rank[i] = (unsigned short)(cur + __popc(peers & lt_mask));
        __syncwarp();
        if (dg[i] < (unsigned)ND && lane == __ffs(peers) - 1)
          s_cnt[w * ND + dg[i]] = (unsigned short)(cur + __popc(peers));
        __syncwarp();
      }
      __syncthreads();
      {                                // per digit: warp offsets, tile start, output slot
        unsigned cnt[DPT];
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
          const int d = tid * DPT + k;
          unsigned acc = 0;
#pragma unroll
          for (int ww = 0; ww < NW; ++ww) {
            const unsigned x = s_cnt[ww * ND + d];
            s_cnt[ww * ND + d] = (unsigned short)acc;
            acc += x;
          }
          cnt[k] = acc;
        }
        unsigned st[DPT];
#pragma unroll
        for (int k = 0; k < DPT; ++k) st[k] = cnt[k];
        block_excl_scan_dpt<DPT>(st, s_warp);
#pragma unroll
        for (int k = 0; k < DPT; ++k) {
          const int d = tid * DPT + k;
          s_tstart[d] = st[k];
          s_gofs[d] = s_run[d];
          s_run[d] += cnt[k];
        }
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (dg[i] >= (unsigned)ND) continue;
        const unsigned lp = s_tstart[dg[i]] + s_cnt[w * ND + dg[i]] + rank[i];
        s_key[lp] = key[i];
        s_bag[lp] = bag[i];
        if (WEIGHTED) s_wt[lp] = wt[i];
      }
      __syncthreads();
      const int tn = (s1 - base) < TILE ? (int)(s1 - base) : TILE;
      for (int i0 = 0; i0 < tn; i0 += kClThreads) {
        const int i = i0 + tid;
        unsigned k2 = (unsigned)ND, q = 0u;
        if (i < tn) {
          const unsigned k = s_key[i];
          const unsigned dd = (k >> shift) & dmask;
          const unsigned out = s_gofs[dd] + (unsigned)i - s_tstart[dd];
          kout[out] = k;
          bout[out] = s_bag[i];
          if (WEIGHTED) wout[out] = s_wt[i];
          if (!last) {                 // the next pass's digit, counted at the strip it lands in
            unsigned lo = 0u;
#pragma unroll
            for (unsigned stp = kClMaxC / 2; stp >= 1; stp >>= 1)
              if (lo + stp < C && s_sb[lo + stp] <= out) lo += stp;
            q = lo;
            k2 = (k >> shift2) & dmask2;
          }
        }
        if (!last) {
          const unsigned tag = k2 < (unsigned)ND ? (q << 16) | k2 : 0xffffffffu;
          const unsigned peers = __match_any_sync(kFull, tag);
          if (tag != 0xffffffffu && lane == __ffs(peers) - 1) {
            unsigned ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                         : "=r"(ra) : "r"(h_next + 4u * k2), "r"(q));
            asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(ra), "r"(__popc(peers))
                         : "memory");
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < NW * ND / 2; i += kClThreads) reinterpret_cast<unsigned*>(s_cnt)[i] = 0u;
      __syncthreads();
    }
    ctrace(S, 45, p);
  }
  cluster_barrier();                   // no CTA leaves while a peer may still read its counts
  ctrace(S, 46, 0);
}

template <bool W, int DB>
const void* cluster_fn() {
  return reinterpret_cast<const void*>(bwd_cluster_sort_kernel<W, DB>);
}
const void* pick_cluster_fn(int db, bool weights) {
  switch (db <= 8 ? 8 : db) {
    case 8: return weights ? cluster_fn<true, 8>() : cluster_fn<false, 8>();
    case 9: return weights ? cluster_fn<true, 9>() : cluster_fn<false, 9>();
    case 10: return weights ? cluster_fn<true, 10>() : cluster_fn<false, 10>();
    case 11: return weights ? cluster_fn<true, 11>() : cluster_fn<false, 11>();
    default: return nullptr;
  }
}
cudaLaunchConfig_t cluster_cfg(int T, int C, size_t sm, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(T * C));
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cfg;
}
cudaError_t prep_cluster_fn(const void* fn, size_t sm) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

// ------------------------------------------------------------------------- fused backward
// Per-warp timeline of the backward (the "trace" option; read with emb_a2a_read_trace): record
// (warp << 40 | event << 32 | payload, %globaltimer).  Events: 20 warp start, 21 exchange done,
// 22 chunk start (payload = chunk), 23 chunk keys in, 24 sub-batch staged, 25 sub-batch done,
// 26 warp done.  Lane 0 only.
__device__ __forceinline__ void btrace(const BwdParams& P, unsigned event, unsigned payload) {
  if (P.trace == nullptr || (threadIdx.x & 31) != 0) return;
  const unsigned long long i = atomicAdd(P.trace, 1ull);
  if ((long long)i >= P.trace_cap) return;
  P.trace[2 + 2 * i] = ((unsigned long long)(blockIdx.x * 32 + (threadIdx.x >> 5)) << 40) |
                       ((unsigned long long)event << 32) | payload;
  P.trace[3 + 2 * i] = globaltimer();
}
// Sparse SGD step on 4 elements (R#29): w = fl(w - fl(lr * g)).
__device__ __forceinline__ void sgd4(float4& w, float lr, const float4& g) {
  w.x = __fsub_rn(w.x, __fmul_rn(lr, g.x));
  w.y = __fsub_rn(w.y, __fmul_rn(lr, g.y));
  w.z = __fsub_rn(w.z, __fmul_rn(lr, g.z));
  w.w = __fsub_rn(w.w, __fmul_rn(lr, g.w));
}

__device__ __forceinline__ void st_shared_f4(float* p, const float4& v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
template <int NVC, int MODE>
__global__ void __launch_bounds__(128, NVC >= 8 ? 1 : (NVC == 1 ? 6 : 4)) bwd_kernel(const __grid_constant__ BwdParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_pushed[kMaxW];
  __shared__ unsigned long long s_ready;     // sources whose rows of this epoch have all landed
  __shared__ float* s_tab[kMaxSmemTables];   // this rank's table pointers (T <= 256)
  __shared__ long long s_ticket[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int D = P.D, DU = D >> 2;

  if (tid == 0) s_ready = 0ull;
  pdl_wait();     // the plan (sort) and the caller's gradient are complete
  pdl_trigger();
  btrace(P, 20, 0);
  // ---- exchange (fused, W > 1): push this rank's gradient rows to their table owners
  if (P.fused && P.W > 1) {
    // buffer-reuse credit: this backward has passed its wait, so every earlier kernel on the
    // stream -- our backward bepoch - 1, which read the staging half the peers fill next -- is
    // complete
    if (blockIdx.x == 0 && tid < P.W && tid != P.r)
      red_release_sys_add(P.peers->bcredit_out[tid], 1ull);
    for (int q = tid; q < P.W; q += blockDim.x) s_pushed[q] = 0u;
    __syncthreads();
    const long long b_r = P.part[P.r + 1] - P.part[P.r];
    const long long total = (long long)(P.W - 1) * b_r;
    const long long gw = (long long)blockIdx.x * nw + warp, nwt = (long long)gridDim.x * nw;
    int cred_ok = -1;
    for (long long m = gw; m < total; m += nwt) {
      const int k = (int)(m / b_r);
      const long long i = m - k * b_r;
      const int q = (P.r + 1 + k) % P.W;          // staggered destinations (R#19)
      const int Tq = P.allT[q];
      if (Tq == 0) continue;
      if (q != cred_ok) {
        // owner q's staging half bepoch & 1 was last read by q's backward bepoch - 2; q's
        // backward bepoch - 1 having passed its wait proves that one complete
        if (lane == 0) {
          const unsigned long long* f = P.bcredits_in + (size_t)q * kFlagStride;
          const unsigned long long t0 = globaltimer();
          while (ld_acquire_sys(f) + 1ull < P.bepoch) {
            if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
              atomicExch(P.err, 0x2000 | q);
              break;
            }
            __nanosleep(128);
          }
        }
        __syncwarp();
        cred_ok = q;
      }
      const float4* src = reinterpret_cast<const float4*>(P.grad + (i * P.G + P.tofs[q]) * D);
      float* dst = P.peers->gstage[q][P.parity] + (P.part[P.r] + i) * Tq * (long long)D;
      const int n4 = Tq * DU;
      for (int u0 = 0; u0 < n4; u0 += 32 * 4) {
        float4 v[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int u = u0 + x * 32 + lane;
          if (u < n4) v[x] = __ldg(src + u);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int u = u0 + x * 32 + lane;
          if (u < n4) st_f4(dst + 4 * u, v[x]);
        }
      }
      if (lane == 0) atomicAdd(&s_pushed[q], 1u);
    }
    __syncthreads();
    // a7 (reverse): one release per (CTA, owner) after the CTA barrier (R#25)
    for (int q = tid; q < P.W; q += blockDim.x) {
      if (q != P.r && s_pushed[q] > 0u) {
        fence_acq_rel_sys();
        red_release_sys_add(P.peers->bflag_out[q], (unsigned long long)s_pushed[q]);
      }
    }
    // a8 (reverse) is per source and per warp (below): a warp waits for source s's rows only
    // when a lookup of its sub-batch needs them, so the reduction of rows from sources that have
    // arrived (and of this rank's own rows) overlaps the exchange from the others.
  }
  if (P.T == 0 || P.n == 0) return;
  for (int t = tid; t < P.T && t < kMaxSmemTables; t += blockDim.x) s_tab[t] = P.tables[t];
  __syncthreads();
  float* const* tabs = P.T <= kMaxSmemTables ? s_tab : P.tables;

  // ---- reduce + update, pass 1 (R#31).  Work unit = a chunk of P.chunk consecutive sorted
  // lookups per warp, taken 32 at a time (sub-batches).  A sub-batch's runs (pieces of equal
  // keys) are split into NG contiguous ranges, one per lane group (LPG lanes cover a row); a
  // group walks its range in sorted order with UF gradient rows in flight per lane and sums each
  // run in ascending lookup order -- the row-flattened pooling loop of the forward, with runs for
  // bags.  A run going on into the next sub-batch hands its sum over through shared memory.  A
  // run that starts and ends inside the chunk is finished here: queued (row, sum) in the group's
  // registers and applied in batches (all table-row loads in flight together).  The chunk's
  // first run, if it began in an earlier chunk, and its last run, if it goes on into the next
  // chunk, are left as partial sums in the chunk's two scratch slots for pass 2.
  constexpr int UF = NVC >= 8 ? 1 : (NVC == 1 ? 4 : 8 / NVC);   // lookups in flight per lane
  int LPG = 1;
  while (LPG < DU && LPG < 32) LPG <<= 1;
  const int NG = 32 / LPG, grp = lane / LPG, gl = lane - grp * LPG;
  long long* wsrc = reinterpret_cast<long long*>(smem + (size_t)warp * P.wbytes);  // [32] rows
  long long* wtab = wsrc + 32;                                                     // [32] table
  float* wsc = reinterpret_cast<float*>(wtab + 32);                                // [32] scale
  float* carry0 = wsc + 32;                                           // [2][D] carried sums
  const unsigned rmask = P.rbits >= 32 ? 0xffffffffu : ((1u << P.rbits) - 1u);
  const long long gw = (long long)blockIdx.x * nw + warp, nwt = (long long)gridDim.x * nw;
  const long long pr = P.part[P.r];
  const long long n = P.n;
  const unsigned B32 = (unsigned)P.B;
  const unsigned* __restrict__ keys = P.keys;

  // chunk gw first (no atomic), then further chunks by ticket (P.ticket zeroed before the
  // launch), so a warp that drew cheap chunks takes more
  btrace(P, 21, 0);
  for (long long c = gw; c < P.nchunks;) {
    btrace(P, 22, (unsigned)c);
    const long long p0 = c * P.chunk;
    const int clen = (n - p0) < P.chunk ? (int)(n - p0) : P.chunk;
    // sub-batch 0's lookups; the keys just before and just after the chunk
    unsigned key = 0u, nkey = 0u;
    int bag = 0, nbag = 0;
    if (lane < clen) {
      key = keys[p0 + lane];
      bag = P.bags[p0 + lane];
    }
    int cf = 0;
    if (lane == 0) {
      if (p0 > 0 && keys[p0 - 1] == key) cf |= 1;                         // run enters chunk
      if (p0 + clen < n && keys[p0 + clen] == keys[p0 + clen - 1]) cf |= 2;   // run leaves
    }
    cf = __shfl_sync(kFull, cf, 0);
    const bool chunk_in = cf & 1, chunk_out = cf & 2;
    btrace(P, 23, 0);
    bool ob = chunk_in;          // the run entering the current sub-batch began before the chunk
    unsigned prev_last = 0u;     // last key of the previous sub-batch
    const int nsb = (clen + 31) / 32;
    for (int sb = 0; sb < nsb; ++sb) {
      const long long pb = p0 + 32 * sb;
      const int len = (clen - 32 * sb) < 32 ? clen - 32 * sb : 32;
      const bool last_sb = sb == nsb - 1;
      if (!last_sb) {                                // prefetch the next sub-batch
        const int nl = (clen - 32 * (sb + 1)) < 32 ? clen - 32 * (sb + 1) : 32;
        if (lane < nl) {
          nkey = keys[pb + 32 + lane];
          nbag = P.bags[pb + 32 + lane];
        }
      }
      const unsigned kup = __shfl_up_sync(kFull, key, 1);
      const unsigned startm = __ballot_sync(kFull, lane < len && (lane == 0 || key != kup));
      const unsigned key0 = __shfl_sync(kFull, key, 0);
      const unsigned keyl = __shfl_sync(kFull, key, len - 1);
      const bool in_sb = sb == 0 ? chunk_in : (key0 == prev_last);
      const bool out_sb = last_sb ? chunk_out : (__shfl_sync(kFull, nkey, 0) == keyl);
      const int npieces = __popc(startm);
      __syncwarp();                                  // the previous sub-batch's readers are done
      unsigned long long needm = 0ull;               // remote sources this sub-batch reads
      if (lane < len) {
        const unsigned t = P.rbits >= 32 ? 0u : key >> P.rbits;   // bag = t * B + j
        const long long j = (long long)((unsigned)bag - t * B32);
        int s = 0;
        if (P.W > 1)
          while (P.part[s + 1] <= j) ++s;            // destination of bag j
        if (P.fused && s != P.r) needm = 1ull << s;
        const float* src;
        if (P.fused)
          src = (s == P.r) ? P.grad + ((j - pr) * P.G + P.toff + (int)t) * D
                           : P.stage + (j * P.T + (int)t) * D;
        else
          src = P.grad + (j * P.T + (int)t) * D;
        wsrc[lane] = reinterpret_cast<long long>(src);
        float* trow = (P.rbits >= 32) ? tabs[0] + (size_t)key * D
                                      : tabs[(int)(key >> P.rbits)] + (size_t)(key & rmask) * D;
        wtab[lane] = reinterpret_cast<long long>(trow);
        // a run that starts here will read and write its table row at its end: bring the row
        // into L2 now, so the walk's round trips are L2 (gradient rows) rather than HBM
        if (((startm >> lane) & 1u) && !(lane == 0 && in_sb))
          for (int b = 0; b < D * 4; b += 128)
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(
                             reinterpret_cast<const char*>(trow) + b));
        if (MODE == 1) wsc[lane] = P.wts[pb + lane];
        if (MODE == 2) wsc[lane] = (float)(P.offsets[bag + 1] - P.offsets[bag]);
      }
      if (P.fused && P.W > 1) {
        // a8 (reverse), per source: rows from source s are read only once all of s's rows of
        // this epoch have landed (its counter reached bepoch * b_s, ld.acquire.sys); the first
        // warp of the CTA to see it records it for the others
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) needm |= __shfl_xor_sync(kFull, needm, o);
        const unsigned long long miss = needm & ~*(volatile unsigned long long*)&s_ready;
        if (miss) {
          if (lane == 0) {
            for (unsigned long long m = miss; m; m &= m - 1) {
              const int src = __ffsll((long long)m) - 1;
              const unsigned long long target =
                  P.bepoch * (unsigned long long)(P.part[src + 1] - P.part[src]);
              const unsigned long long* f = P.bflags_in + (size_t)src * kFlagStride;
              const unsigned long long t0 = globaltimer();
              unsigned backoff = 32;
              while (ld_acquire_sys(f) < target) {
                if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
                  atomicExch(P.err, 0x400 | src);
                  break;
                }
                __nanosleep(backoff);
                if (backoff < 1024) backoff <<= 1;
              }
            }
            fence_acq_rel_sys();
            atomicOr(&s_ready, miss);
          }
        } else {
          // another warp's acquire covers these sources: order our loads after it
          asm volatile("fence.acq_rel.cta;" ::: "memory");
        }
      }
      if (sb == 0 && lane == 0) {
        const bool inside = chunk_in && chunk_out && npieces == 1 && nsb == 1;
        // pass-2 flags, fixed up below once we know whether the last run began before the chunk
        P.info[c] = (unsigned char)((chunk_out && !inside ? 1 : 0) | (inside ? 2 : 0));
      }
      __syncwarp();
      bool carry_out = false, carry_ob = false;
      const float* cin = carry0 + (size_t)(sb & 1) * D;      // written in sub-batch sb - 1
      float* cout = carry0 + (size_t)((sb + 1) & 1) * D;

      // Finish the piece (run, or part of one) ending at lookup q with sum acc.
      auto finish = [&](float4 (&acc)[NVC], int q, int pi, bool enters, bool has_w,
                        const float4 (&cur_w)[NVC]) {
        const bool leaves = pi == npieces - 1 && out_sb;
        const bool began_before = enters && ob;      // the run began in an earlier chunk
        if (leaves && !last_sb) {                    // hand over to the next sub-batch
          carry_out = true;
          carry_ob = began_before;
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            const int col = gl + LPG * v;
            if (col < DU) st_shared_f4(cout + 4 * col, acc[v]);
          }
        } else if (leaves || began_before) {         // partial for pass 2
          float* slot = P.scratch + ((size_t)c * 2 + (leaves ? 1 : 0)) * D;
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            const int col = gl + LPG * v;
            if (col < DU) st_f4(slot + 4 * col, acc[v]);
          }
          if (leaves && gl == 0)                     // owner iff the run began in this chunk
            P.info[c] = (unsigned char)(began_before ? 2 : 1);
        } else {                                     // finished here: the SGD step
          float* tp = reinterpret_cast<float*>(wtab[q]);
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            const int col = gl + LPG * v;
            if (col < DU) {
              // a run handed over from the previous sub-batch loads its row now
              float4 w = has_w ? cur_w[v] : __ldcg(reinterpret_cast<const float4*>(tp) + col);
              sgd4(w, P.lr, acc[v]);
              st_f4(tp + 4 * col, w);
            }
          }
        }
      };

      // Sum lookups [lo, hi) in order into acc (UF rows in flight per lane); at each run end
      // inside the range call finish (split = false), else just accumulate (split = true).
      // The table row of a run starting in the range is loaded with its first gradient row.
      auto walk = [&](float4 (&acc)[NVC], int lo, int hi, int pi, bool enters, bool split,
                      bool& has_w, float4 (&cur_w)[NVC]) {
        for (int q0 = lo; q0 < hi; q0 += UF) {
          float4 buf[UF][NVC], tw[UF][NVC];
#pragma unroll
          for (int x = 0; x < UF; ++x) {
            const int q = q0 + x;
            const bool ok = q < hi;
            const bool st = ok && ((startm >> q) & 1u) && !(q == 0 && in_sb);
            const float4* rp = reinterpret_cast<const float4*>(wsrc[ok ? q : lo]);
            const float4* tp = reinterpret_cast<const float4*>(wtab[ok ? q : lo]);
#pragma unroll
            for (int v = 0; v < NVC; ++v) {
              const int col = gl + LPG * v;
              buf[x][v] = (ok && col < DU) ? __ldcg(rp + col) : make_float4(0.f, 0.f, 0.f, 0.f);
              tw[x][v] = (st && col < DU) ? __ldcg(tp + col) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int x = 0; x < UF; ++x) {
            const int q = q0 + x;
            if (q >= hi) break;
            if (((startm >> q) & 1u) && !(q == 0 && in_sb)) {
#pragma unroll
              for (int v = 0; v < NVC; ++v) cur_w[v] = tw[x][v];
              has_w = true;
            }
            const float s = (MODE != 0) ? wsc[q] : 1.f;
#pragma unroll
            for (int v = 0; v < NVC; ++v) {
              float4 cv = buf[x][v];
              if (MODE == 1) {
                cv.x = __fmul_rn(s, cv.x); cv.y = __fmul_rn(s, cv.y);
                cv.z = __fmul_rn(s, cv.z); cv.w = __fmul_rn(s, cv.w);
              } else if (MODE == 2) {
                cv.x = __fdiv_rn(cv.x, s); cv.y = __fdiv_rn(cv.y, s);
                cv.z = __fdiv_rn(cv.z, s); cv.w = __fdiv_rn(cv.w, s);
              }
              add4(acc[v], cv);
            }
            if (split || (q + 1 < len && !((startm >> (q + 1)) & 1u))) continue;
            finish(acc, q, pi, enters, has_w, cur_w);
#pragma unroll
            for (int v = 0; v < NVC; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            ++pi;
            enters = false;
            has_w = false;
          }
        }
      };

      float4 acc[NVC], cur_w[NVC];
      bool has_w = false;
#pragma unroll
      for (int v = 0; v < NVC; ++v) {
        acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        cur_w[v] = acc[v];
      }
      btrace(P, 24, (unsigned)sb);
      if (npieces == 1 && NG > 1) {
        // one run fills the sub-batch (a Zipf-hot row): every lane group sums an equal share of
        // its lookups, then the shares are added in group order (after the carried-in sum)
        walk(acc, (len * grp) / NG, (len * (grp + 1)) / NG, 0, false, true, has_w, cur_w);
        const bool enters = in_sb;
        float4 tot[NVC];
#pragma unroll
        for (int v = 0; v < NVC; ++v) {
          const int col = gl + LPG * v;
          tot[v] = (enters && sb > 0 && col < DU) ? lds_f4(smem_u32(cin + 4 * col))
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int g = 0; g < NG; ++g) {
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            float4 p;
            p.x = __shfl_sync(kFull, acc[v].x, g * LPG + gl);
            p.y = __shfl_sync(kFull, acc[v].y, g * LPG + gl);
            p.z = __shfl_sync(kFull, acc[v].z, g * LPG + gl);
            p.w = __shfl_sync(kFull, acc[v].w, g * LPG + gl);
            add4(tot[v], p);
          }
        }
        if (grp == 0) finish(tot, len - 1, 0, enters, has_w, cur_w);
      } else {
        const int pa = (npieces * grp) / NG, pbnd = (npieces * (grp + 1)) / NG;
        if (pa < pbnd) {
          const int lo = __fns(startm, 0, pa + 1);
          const int hi = pbnd < npieces ? (int)__fns(startm, 0, pbnd + 1) : len;
          const bool enters = pa == 0 && in_sb;
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            const int col = gl + LPG * v;
            if (enters && sb > 0 && col < DU) acc[v] = lds_f4(smem_u32(cin + 4 * col));
          }
          walk(acc, lo, hi, pa, enters, false, has_w, cur_w);
        }
      }
      // which group (if any) carried a run over, and whether it began before the chunk
      const unsigned cm = __ballot_sync(kFull, carry_out);
      if (cm) ob = __shfl_sync(kFull, carry_ob, __ffs(cm) - 1);
      else ob = false;
      prev_last = keyl;
      key = nkey;
      bag = nbag;
      btrace(P, 25, (unsigned)sb);
    }
    if (lane == 0) s_ticket[warp] = nwt + (long long)atomicAdd(P.ticket, 1u);
    __syncwarp();
    c = s_ticket[warp];
    __syncwarp();
  }
  btrace(P, 26, 0);
}

// ---- reduce + update, pass 2 (R#31): the runs that cross chunk boundaries.  The chunk a run
// starts in owns it (info bit 0): tot = +0, + its slot-1 partial, + the slot-1 partials of the
// chunks the run covers entirely (info bit 1, read 32 at a time), + the slot-0 partial of the
// chunk it ends in -- in chunk order -- then the SGD step on the row.
template <int NVC>
__global__ void __launch_bounds__(256) bwd_fold_kernel(const __grid_constant__ BwdParams P) {
  const int lane = threadIdx.x & 31;
  const int D = P.D, DU = D >> 2;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  pdl_wait();     // pass 1 complete: partials, info
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x == 0) *P.ticket = 0u;   // pass 1's tickets, for next time
  const unsigned rmask = P.rbits >= 32 ? 0xffffffffu : ((1u << P.rbits) - 1u);
  constexpr int BATCH = NVC >= 16 ? 1 : 16 / NVC;
  for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < P.nchunks;
       c += nw) {
    if (!(P.info[c] & 1)) continue;
    const unsigned K = P.keys[c * P.chunk + P.chunk - 1];
    float4 tot[NVC];
#pragma unroll
    for (int v = 0; v < NVC; ++v) {
      const int col = lane + 32 * v;
      tot[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (col < DU)
        add4(tot[v], __ldcg(reinterpret_cast<const float4*>(P.scratch + (c * 2 + 1) * D) + col));
    }
    long long q = c + 1;
    while (true) {
      const bool in = q + lane < P.nchunks && (P.info[q + lane] & 2);
      const unsigned m = __ballot_sync(kFull, in);
      const int k = (m == kFull) ? 32 : __ffs(~m) - 1;     // chunks q .. q+k-1 lie inside the run
      for (int x0 = 0; x0 < (k < 32 ? k + 1 : 32); x0 += BATCH) {             // ... and chunk q+k ends it
        float4 pv[BATCH][NVC];
#pragma unroll
        for (int x = 0; x < BATCH; ++x) {
          const long long qq = q + x0 + x;
          const bool ok = x0 + x < k || (x0 + x == k && k < 32);
          const float* src = P.scratch + (qq * 2 + (x0 + x < k ? 1 : 0)) * D;
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            const int col = lane + 32 * v;
            pv[x][v] = (ok && col < DU) ? __ldcg(reinterpret_cast<const float4*>(src) + col)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int x = 0; x < BATCH; ++x)
          if (x0 + x < k || (x0 + x == k && k < 32))
#pragma unroll
            for (int v = 0; v < NVC; ++v) add4(tot[v], pv[x][v]);
      }
      if (k < 32) break;
      q += 32;
    }
    float* tp = (P.rbits >= 32) ? P.tables[0] + (size_t)K * D
                                : P.tables[(int)(K >> P.rbits)] + (size_t)(K & rmask) * D;
#pragma unroll
    for (int v = 0; v < NVC; ++v) {
      const int col = lane + 32 * v;
      if (col < DU) {
        float4 w = __ldcg(reinterpret_cast<const float4*>(tp) + col);
        sgd4(w, P.lr, tot[v]);
        st_f4(tp + 4 * col, w);
      }
    }
  }
}

// Pass 2 for rows of at most 32 float4 (D <= 128): the same fold, with the warp cut into NGF =
// 32 / LPG lane groups (LPG lanes cover a row) that load different chunks' partials -- group g
// takes chunks x0 + g, x0 + g + NGF, ... -- so a window of 32 chunks is one round of loads at
// D <= 64; the partials are then added in chunk order from the loading group's lanes
// (shuffles), every group keeping the same running sum.  Same order, same result as the
// one-group fold.
__global__ void __launch_bounds__(256) bwd_fold_narrow_kernel(const __grid_constant__ BwdParams P) {
  const int lane = threadIdx.x & 31;
  const int D = P.D, DU = D >> 2;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  pdl_wait();     // pass 1 complete: partials, info
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x == 0) *P.ticket = 0u;   // pass 1's tickets, for next time
  const unsigned rmask = P.rbits >= 32 ? 0xffffffffu : ((1u << P.rbits) - 1u);
  int LPG = 1;
  while (LPG < DU) LPG <<= 1;
  const int NGF = 32 / LPG, g = lane / LPG, col = lane - g * LPG;
  const bool colok = col < DU;
  constexpr int BATCH = 16;                 // loads in flight per lane
  for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < P.nchunks;
       c += nw) {
    if (!(P.info[c] & 1)) continue;
    const unsigned K = P.keys[c * P.chunk + P.chunk - 1];
    float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
    if (colok) add4(tot, __ldcg(reinterpret_cast<const float4*>(P.scratch + (c * 2 + 1) * D) + col));
    long long q = c + 1;
    bool in = q + lane < P.nchunks && (P.info[q + lane] & 2);
    while (true) {
      const unsigned m = __ballot_sync(kFull, in);
      const int k = (m == kFull) ? 32 : __ffs(~m) - 1;     // chunks q .. q+k-1 lie inside the run
      const int kend = k < 32 ? k + 1 : 32;                // ... and chunk q+k ends it (if k < 32)
      if (k == 32)                                         // the next window's flags, early
        in = q + 32 + lane < P.nchunks && (P.info[q + 32 + lane] & 2);
      for (int x0 = 0; x0 < kend; x0 += BATCH * NGF) {
        float4 pv[BATCH];
#pragma unroll
        for (int s_ = 0; s_ < BATCH; ++s_) {
          const int x = x0 + s_ * NGF + g;
          const float* src = P.scratch + ((q + x) * 2 + (x < k ? 1 : 0)) * D;
          pv[s_] = (x < kend && colok) ? __ldcg(reinterpret_cast<const float4*>(src) + col)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int s_ = 0; s_ < BATCH; ++s_) {
          if (x0 + s_ * NGF >= kend) break;                // warp-uniform
          for (int gg = 0; gg < NGF; ++gg) {
            if (x0 + s_ * NGF + gg >= kend) break;         // warp-uniform
            const int from = gg * LPG + col;
            float4 v;
            v.x = __shfl_sync(kFull, pv[s_].x, from);
            v.y = __shfl_sync(kFull, pv[s_].y, from);
            v.z = __shfl_sync(kFull, pv[s_].z, from);
            v.w = __shfl_sync(kFull, pv[s_].w, from);
            add4(tot, v);
          }
        }
      }
      if (k < 32) break;
      q += 32;
    }
    float* tp = (P.rbits >= 32) ? P.tables[0] + (size_t)K * D
                                : P.tables[(int)(K >> P.rbits)] + (size_t)(K & rmask) * D;
    if (g == 0 && colok) {
      float4 w = __ldcg(reinterpret_cast<const float4*>(tp) + col);
      sgd4(w, P.lr, tot);
      st_f4(tp + 4 * col, w);
    }
  }
}

typedef void (*BwdFn)(const BwdParams);

template <int NVC>
BwdFn pick_bwd_mode(int mode) {
  switch (mode) {
    case 1: return bwd_kernel<NVC, 1>;
    case 2: return bwd_kernel<NVC, 2>;
    default: return bwd_kernel<NVC, 0>;
  }
}

BwdFn pick_bwd(const BwdParams& P) {
  const int DU = P.D / 4;
  const int mode = P.wts ? 1 : (P.mean ? 2 : 0);
  const int nvc = (DU + 31) / 32;
  if (nvc <= 1) return pick_bwd_mode<1>(mode);
  if (nvc <= 2) return pick_bwd_mode<2>(mode);
  if (nvc <= 4) return pick_bwd_mode<4>(mode);
  return pick_bwd_mode<8>(mode);
}

BwdFn pick_fold(const BwdParams& P) {
  const int nvc = (P.D / 4 + 31) / 32;
  return nvc <= 1 ? bwd_fold_narrow_kernel : nvc <= 2 ? bwd_fold_kernel<2>
       : nvc <= 4 ? bwd_fold_kernel<4> : bwd_fold_kernel<8>;
}

cudaError_t launch_pdl(const void* fn, unsigned grid, int threads, size_t smem, cudaStream_t st,
                       void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

size_t bwd_smem(const BwdParams& P, int threads) {
  return (size_t)(threads / 32) * (size_t)P.wbytes;
}

}  // namespace

cudaError_t launch_sort_plan(const SortParams& S, const PassParams* passes, int npasses,
                             long long ntiles, int grid_keygen, int mode, cudaStream_t st) {
  if (S.TB > 0) {
    SortParams s = S;
    void* args[] = {&s};
    const void* fn = S.weights ? reinterpret_cast<const void*>(bwd_keygen_kernel<true>)
                               : reinterpret_cast<const void*>(bwd_keygen_kernel<false>);
    cudaError_t e = launch_pdl(fn, (unsigned)grid_keygen, 256, 0, st, args);
    if (e != cudaSuccess) return e;
  }
  // one wave of tiles: onesweep (1 kernel per pass, short look-back); more: reduce-then-scan
  // (3 kernels per pass, no look-back chains across the tiles of a wave)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool one_wave = mode == 1 || (mode == 0 && ntiles <= 3LL * sms);
  for (int p = 0; p < npasses; ++p) {
    PassParams pp = passes[p];
    void* args[] = {&pp};
    if (one_wave) {
      const void* fn = passes[p].wts_in
                           ? reinterpret_cast<const void*>(bwd_onesweep_kernel<true>)
                           : reinterpret_cast<const void*>(bwd_onesweep_kernel<false>);
      cudaError_t e = launch_pdl(fn, (unsigned)ntiles, kSortThreads, 0, st, args);
      if (e != cudaSuccess) return e;
      continue;
    }
    cudaError_t e = launch_pdl(reinterpret_cast<const void*>(bwd_upsweep_kernel),
                               (unsigned)ntiles, kSortThreads, 0, st, args);
    if (e == cudaSuccess)
      e = launch_pdl(reinterpret_cast<const void*>(bwd_scan_kernel), 256, 256, 0, st, args);
    const void* fn = passes[p].wts_in ? reinterpret_cast<const void*>(bwd_downsweep_kernel<true>)
                                      : reinterpret_cast<const void*>(bwd_downsweep_kernel<false>);
    if (e == cudaSuccess) e = launch_pdl(fn, (unsigned)ntiles, kSortThreads, 0, st, args);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

size_t seg_sort_smem(int db, bool weights) {
  const size_t NB = (size_t)1 << db;
  return (size_t)(kSortThreads / 32) * NB * 2 + 2 * NB * 4 +
         (size_t)kSortTile * (weights ? 12 : 8);
}

namespace {
template <bool W, int DB>
cudaError_t launch_seg_pass(const PassParams& pp, long long grid, cudaStream_t st) {
  const void* fn = reinterpret_cast<const void*>(bwd_onesweep_seg_kernel<W, DB>);
  const size_t sm = seg_sort_smem(DB, W);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  PassParams q = pp;
  void* args[] = {&q};
  return launch_pdl(fn, (unsigned)grid, kSortThreads, sm, st, args);
}
template <bool W>
cudaError_t launch_seg_pass_db(const PassParams& pp, int db, long long grid, cudaStream_t st) {
  switch (db) {
    case 8: return launch_seg_pass<W, 8>(pp, grid, st);
    case 9: return launch_seg_pass<W, 9>(pp, grid, st);
    case 10: return launch_seg_pass<W, 10>(pp, grid, st);
    case 11: return launch_seg_pass<W, 11>(pp, grid, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

cudaError_t launch_sort_plan_seg(const SortParams& S, const PassParams* passes, int npasses,
                                 long long ntiles_max, int grid_keygen, cudaStream_t st) {
  if (S.TB > 0) {
    SortParams s = S;
    void* args[] = {&s};
    const size_t sm = (size_t)4 * ((size_t)1 << S.seg_db) * 4;
    const void* fn = S.weights ? reinterpret_cast<const void*>(bwd_keygen_seg_kernel<true>)
                               : reinterpret_cast<const void*>(bwd_keygen_seg_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess) e = launch_pdl(fn, (unsigned)grid_keygen, 256, sm, st, args);
    if (e != cudaSuccess) return e;
  }
  for (int p = 0; p < npasses; ++p) {
    cudaError_t e = passes[p].wts_in
                        ? launch_seg_pass_db<true>(passes[p], S.seg_db, ntiles_max, st)
                        : launch_seg_pass_db<false>(passes[p], S.seg_db, ntiles_max, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}



cudaError_t launch_bucket_sort(const unsigned* keys_in, const int* bags_in, const float* wts_in,
                               unsigned* keys_out, int* bags_out, float* wts_out,
                               const unsigned* hist, int low_bits, int cap, cudaStream_t st) {
  BucketParams P;
  P.keys_in = keys_in;
  P.bags_in = bags_in;
  P.wts_in = wts_in;
  P.keys_out = keys_out;
  P.bags_out = bags_out;
  P.wts_out = wts_out;
  P.hist = hist;
  P.low_bits = low_bits;
  P.cap = cap;
  const bool w = wts_in != nullptr;
  const void* fn = w ? reinterpret_cast<const void*>(bwd_bucket_sort_kernel<true>)
                     : reinterpret_cast<const void*>(bwd_bucket_sort_kernel<false>);
  const size_t sm = (size_t)2 * cap * (w ? 12 : 8);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  void* args[] = {&P};
  return launch_pdl(fn, 256, kBktThreads, sm, st, args);
}

int cluster_plan_size(int T, int db, bool weights) {
  const void* fn = pick_cluster_fn(db, weights);
  const size_t sm = cluster_smem(db, weights);
  if (!fn || T <= 0 || prep_cluster_fn(fn, sm) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int C = 16; C >= 1; C >>= 1) {
    // the largest cluster whose T copies fit two CTAs per SM (1 if even that is short)
    if (C > 1 && (long long)T * C > 2LL * sms) continue;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = cluster_cfg(T, C, sm, 0, attr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n > 0) return C;
    cudaGetLastError();
  }
  return 0;
}

cudaError_t launch_sort_plan_cluster(const ClusterSortParams& S, int T, cudaStream_t st) {
  if (T <= 0 || S.B <= 0) return cudaSuccess;
  const void* fn = pick_cluster_fn(S.db, S.weights != nullptr);
  if (!fn) return cudaErrorInvalidValue;
  const size_t sm = cluster_smem(S.db, S.weights != nullptr);
  cudaError_t e = prep_cluster_fn(fn, sm);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = cluster_cfg(T, S.C, sm, st, attr);
  ClusterSortParams s = S;
  void* args[] = {&s};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Persistent grid: every CTA must be resident at once (the exchange wait and the chunk fold
// wait on other CTAs).  share > 1 divides it (W virtual ranks on one GPU must co-reside).
cudaError_t plan_backward(const BwdParams& P, int threads, int share, unsigned* grid,
                          size_t* smem) {
  cudaGetLastError();
  BwdFn fn = pick_bwd(P);
  const size_t sm = bwd_smem(P, threads);
  if (sm > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(fn),
                                                    threads, sm);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  // load pass 2's kernel now: with lazy module loading, its first launch behind a running pass 1
  // (whose CTAs spin on the peers' rows) could otherwise stall the launches the peers need
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(pick_fold(P)));
  if (e != cudaSuccess) return e;
  long long g = (long long)sms * occ / (share > 1 ? share : 1);
  if (g < 1) g = 1;
  *grid = (unsigned)g;
  *smem = sm;
  return cudaSuccess;
}

cudaError_t launch_backward(const BwdParams& P, unsigned grid, int threads, size_t smem,
                            cudaStream_t st) {
  BwdFn fn = pick_bwd(P);
  BwdParams Pc = P;
  void* args[] = {&Pc};
  cudaError_t e = launch_pdl(reinterpret_cast<const void*>(fn), grid, threads, smem, st, args);
  if (e != cudaSuccess || P.T == 0 || P.nchunks == 0) return e;
  // pass 2: one warp per chunk (most exit at once)
  const long long blocks = (P.nchunks + 7) / 8;
  const unsigned g2 = (unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16);
  BwdFn f2 = pick_fold(P);
  // pass 2 overlaps pass 1's drain only when this rank has the GPU to itself: with virtual
  // ranks sharing one device, its early CTAs could take the slots a peer's pass 1 still needs
  if (!P.pdl_fold) return cudaLaunchKernel(reinterpret_cast<const void*>(f2), dim3(g2), dim3(256),
                                           args, 0, st);
  return launch_pdl(reinterpret_cast<const void*>(f2), g2, 256, 0, st, args);
}

}  // namespace emba2a
