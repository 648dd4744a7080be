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
//   bwd_onesweep_kernel  one stable LSD radix pass (8-bit digit): warp-level ranking with
//                        match.any, per-digit decoupled look-back across tiles (tiles taken in
//                        ticket order, so every look-back target is already running)
//   bwd_kernel           (fused) each CTA first pushes its share of this rank's gradient rows
//                        straight into the owners' staging buffers over NVLink (zero-copy, the
//                        reverse of P:165) and signals the owner's per-source counter with
//                        red.release.sys; then waits (ld.acquire.sys) for every source's rows;
//                        then reduces: the sorted lookups are cut into chunks of C; a warp
//                        gathers a chunk's gradient rows and the table rows it will update into
//                        shared memory (cp.async), sums each run of equal keys in order, and
//                        updates the row.  A run that crosses chunks is published as a partial
//                        sum per chunk and folded, in chunk order, by the chunk where it ends
//                        (the last-finisher pattern of P:149/P:176, made deterministic).
//                        (local) the same reduce from a caller-owned [B][T][D] gradient -- the
//                        unfused baseline's second half after NCCL all_to_all_single.
#include "fused_kernel.cuh"

namespace emba2a {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void cp_async16_cg(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void st_f4(float* p, const float4& v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// ------------------------------------------------------------------------------ sort plan
// Keys of this rank's lookups and the digit histograms of every pass.  One thread per bag.
template <bool WEIGHTED>
__global__ void __launch_bounds__(256) bwd_keygen_kernel(const SortParams S) {
  __shared__ unsigned h[kMaxPasses * 256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long bag = blockIdx.x * (long long)blockDim.x + threadIdx.x; bag < S.TB;
       bag += stride) {
    const unsigned t = (unsigned)(bag / S.B);
    const int lo = S.offsets[bag], hi = S.offsets[bag + 1];
    for (int k = lo; k < hi; ++k) {
      const unsigned key = (S.rbits >= 32 ? 0u : (t << S.rbits)) | (unsigned)S.indices[k];
      S.keys[k] = key;
      S.bags[k] = (int)bag;
      if (WEIGHTED) S.wts[k] = S.weights[k];
      for (int p = 0; p < S.passes; ++p) atomicAdd(&h[p * 256 + ((key >> (8 * p)) & 255u)], 1u);
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

// Look-back words: [63:34] stamp | [33:32] flag (1 aggregate, 2 inclusive prefix) | [31:0] count
__device__ __forceinline__ unsigned long long lb_word(unsigned stamp, unsigned flag,
                                                      unsigned count) {
  return ((unsigned long long)(stamp & 0x3fffffffu) << 34) | ((unsigned long long)flag << 32) |
         count;
}

// One stable LSD radix pass.  Tile = 4096 keys; warp w owns keys [w*512, (w+1)*512) of the
// tile, item i of lane l at w*512 + i*32 + l (warp-striped, so "item, then lane" is position
// order and the ranking below is stable).
template <bool WEIGHTS>
__global__ void __launch_bounds__(kSortThreads) bwd_onesweep_kernel(const PassParams P) {
  constexpr int NW = kSortThreads / 32;
  __shared__ unsigned s_cnt[NW][256];   // running per-warp digit counts -> warp offsets in tile
  __shared__ unsigned s_gofs[256];
  __shared__ unsigned s_warp[NW];
  __shared__ unsigned s_tile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < NW * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0u;
  if (tid == 0) s_tile = atomicAdd(P.tile_ctr, 1u);
  __syncthreads();
  const long long tile = s_tile;
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
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    const unsigned d = pos < P.n ? ((key[i] >> P.shift) & 255u) : 256u;
    const unsigned peers = __match_any_sync(kFull, d);
    const unsigned c = d < 256u ? s_cnt[w][d] : 0u;
    rank[i] = (unsigned short)(c + __popc(peers & lt_mask));
    __syncwarp();
    if (d < 256u && lane == __ffs(peers) - 1) s_cnt[w][d] = c + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // thread d: exclusive offsets of digit d per warp, the tile's count, the global base
  const unsigned d = tid;
  unsigned run = 0;
#pragma unroll
  for (int ww = 0; ww < NW; ++ww) {
    const unsigned c = s_cnt[ww][d];
    s_cnt[ww][d] = run;
    run += c;
  }
  const unsigned gbase = block_excl_scan256(P.hist[d], s_warp);
  unsigned long long* my = P.status + tile * 256 + d;
  unsigned excl = 0;
  if (tile == 0) {
    st_relaxed_gpu(my, lb_word(P.stamp, 2, run));
  } else {
    st_relaxed_gpu(my, lb_word(P.stamp, 1, run));
    long long look = tile - 1;
    const unsigned want = P.stamp & 0x3fffffffu;
    const unsigned long long t0 = globaltimer();
    while (look >= 0) {
      const unsigned long long v = ld_acquire_gpu(P.status + look * 256 + d);
      const unsigned flag = (unsigned)(v >> 32) & 3u;
      if ((unsigned)(v >> 34) != want || flag == 0u) {   // predecessor not published yet
        // tiles are taken in ticket order, so every predecessor is running and will publish;
        // the bound only guards against a broken invariant turning into a hung GPU
        if (globaltimer() - t0 > 5000000000ull) break;
        continue;
      }
      excl += (unsigned)v;
      if (flag == 2u) break;
      --look;
    }
    st_relaxed_gpu(my, lb_word(P.stamp, 2, excl + run));
  }
  s_gofs[d] = gbase + excl;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const long long pos = base + i * 32 + lane;
    if (pos < P.n) {
      const unsigned dd = (key[i] >> P.shift) & 255u;
      const unsigned out = s_gofs[dd] + s_cnt[w][dd] + rank[i];
      P.keys_out[out] = key[i];
      P.bags_out[out] = bag[i];
      if (WEIGHTS) P.wts_out[out] = wt[i];
    }
  }
}

// ------------------------------------------------------------------------- fused backward
// MODE 0 sum, 1 weighted (c = fl(w * g), R#26), 2 mean (c = fl(g / L), R#27).  NVC = float4
// columns per lane (D / 128 rounded up to 1, 2, 4, 8).
template <int NVC, int MODE>
__global__ void __launch_bounds__(128) bwd_kernel(const __grid_constant__ BwdParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned s_pushed[kMaxW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int D = P.D, DU = D >> 2, C = P.C;

  // ---- exchange (fused, W > 1): push this rank's gradient rows to their table owners
  if (P.fused && P.W > 1) {
    for (int q = tid; q < P.W; q += blockDim.x) s_pushed[q] = 0u;
    __syncthreads();
    const long long b_r = P.part[P.r + 1] - P.part[P.r];
    const long long total = (long long)(P.W - 1) * b_r;
    const long long gw = (long long)blockIdx.x * nw + warp, nwt = (long long)gridDim.x * nw;
    for (long long m = gw; m < total; m += nwt) {
      const int k = (int)(m / b_r);
      const long long i = m - k * b_r;
      const int q = (P.r + 1 + k) % P.W;          // staggered destinations (R#19)
      const int Tq = P.allT[q];
      if (Tq == 0) continue;
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
    // a8 (reverse): every source's rows of this epoch have landed here
    if (tid == 0 && P.T > 0) {
      for (int s = 0; s < P.W; ++s) {
        if (s == P.r) continue;
        const unsigned long long target =
            P.bepoch * (unsigned long long)(P.part[s + 1] - P.part[s]);
        const unsigned long long* f = P.bflags_in + (size_t)s * kFlagStride;
        const unsigned long long t0 = globaltimer();
        unsigned backoff = 32;
        while (ld_acquire_sys(f) < target) {
          if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
            atomicExch(P.err, 0x400 | s);
            break;
          }
          __nanosleep(backoff);
          if (backoff < 1024) backoff <<= 1;
        }
      }
    }
    __syncthreads();
  }
  if (P.T == 0 || P.n == 0) return;

  // ---- reduce + update: warp-level work units (chunks of C sorted lookups)
  const size_t wbytes = (size_t)2 * C * D * 4 + 32 * 4 + 32 * 8;
  unsigned char* wb = smem + warp * wbytes;
  float* sg = reinterpret_cast<float*>(wb);             // [C][D] gradient rows
  float* stb = sg + (size_t)C * D;                      // [C][D] table rows (per piece)
  float* sscal = stb + (size_t)C * D;                   // [C] weight or bag length
  float** stp = reinterpret_cast<float**>(sscal + 32);  // [C] table row pointers (per piece)
  const unsigned rmask = P.rbits >= 32 ? 0xffffffffu : ((1u << P.rbits) - 1u);
  const long long gw = (long long)blockIdx.x * nw + warp, nwt = (long long)gridDim.x * nw;
  const long long pr = P.part[P.r];

  for (long long c = gw; c < P.nchunks; c += nwt) {
    const long long p0 = c * C;
    const int len = (int)((P.n - p0) < C ? (P.n - p0) : C);
    unsigned key = 0u;
    int bag = 0;
    if (lane < len) {
      key = P.keys[p0 + lane];
      bag = P.bags[p0 + lane];
    }
    const unsigned kup = __shfl_up_sync(kFull, key, 1);
    const unsigned startm = __ballot_sync(kFull, lane < len && (lane == 0 || key != kup));
    const unsigned key0 = __shfl_sync(kFull, key, 0);
    const unsigned keyl = __shfl_sync(kFull, key, len - 1);
    int flags = 0;
    if (lane == 0) {
      if (p0 > 0 && P.keys[p0 - 1] == key0) flags |= 1;              // run continues in
      if (p0 + len < P.n && P.keys[p0 + len] == keyl) flags |= 2;    // run continues out
    }
    flags = __shfl_sync(kFull, flags, 0);
    const bool cont_in = flags & 1, cont_out = flags & 2;
    const int npieces = __popc(startm);

    // this lane's lookup: where its gradient row lives, its scalar, the piece's table row
    unsigned long long srow = 0ull;
    if (lane < len) {
      const int t = (int)(bag / P.B);
      const long long j = bag - (long long)t * P.B;
      int s = 0;
      while (P.part[s + 1] <= j) ++s;                  // destination of bag j
      const float* src;
      if (P.fused)
        src = (s == P.r) ? P.grad + ((j - pr) * P.G + P.toff + t) * D
                         : P.stage + (j * P.T + t) * D;
      else
        src = P.grad + (j * P.T + t) * D;
      srow = reinterpret_cast<unsigned long long>(src);
      if (MODE == 1) sscal[lane] = P.wts[p0 + lane];
      if (MODE == 2) sscal[lane] = (float)(P.offsets[bag + 1] - P.offsets[bag]);
      if ((startm >> lane) & 1u) {
        const int pi = __popc(startm & ((1u << lane) - 1u));
        const bool fin_here = !(pi == npieces - 1 && cont_out);
        stp[pi] = fin_here ? P.tables[t] + (size_t)(key & rmask) * D : nullptr;
      }
    }
    __syncwarp();
    // gather the chunk's gradient rows and the table rows it finalises (cp.async, L2 only)
    const int tot = len * DU;
    for (int b = 0; b < tot; b += 32) {
      const int idx = b + lane;
      const int o = idx < tot ? idx / DU : len - 1;
      const float* rp = reinterpret_cast<const float*>(__shfl_sync(kFull, srow, o));
      if (idx < tot) {
        const int u = idx - o * DU;
        cp_async16_cg(smem_u32(sg + o * D + 4 * u), rp + 4 * u);
      }
    }
    const int ttot = npieces * DU;
    for (int idx = lane; idx < ttot; idx += 32) {
      const int pi = idx / DU, u = idx - pi * DU;
      const float* tp = stp[pi];
      if (tp) cp_async16_cg(smem_u32(stb + pi * D + 4 * u), tp + 4 * u);
    }
    cp_async_wait_all();
    __syncwarp();

    float4 acc[NVC];
#pragma unroll
    for (int v = 0; v < NVC; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    int pi = 0;
    for (int o = 0; o < len; ++o) {
      float sc = 1.f;
      if (MODE != 0) sc = sscal[o];
#pragma unroll
      for (int v = 0; v < NVC; ++v) {
        const int u = lane + 32 * v;
        if (u < DU) {
          float4 g = lds_f4(smem_u32(sg + o * D + 4 * u));
          if (MODE == 1) {
            g.x = __fmul_rn(sc, g.x); g.y = __fmul_rn(sc, g.y);
            g.z = __fmul_rn(sc, g.z); g.w = __fmul_rn(sc, g.w);
          } else if (MODE == 2) {
            g.x = __fdiv_rn(g.x, sc); g.y = __fdiv_rn(g.y, sc);
            g.z = __fdiv_rn(g.z, sc); g.w = __fdiv_rn(g.w, sc);
          }
          add4(acc[v], g);
        }
      }
      const bool end = (o == len - 1) || ((startm >> (o + 1)) & 1u);
      if (!end) continue;
      if (pi == npieces - 1 && cont_out) {
        // partial of a run that continues in the next chunk: publish it for the fold
#pragma unroll
        for (int v = 0; v < NVC; ++v) {
          const int u = lane + 32 * v;
          if (u < DU) st_f4(P.scratch + c * D + 4 * u, acc[v]);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(P.chunk_flag + c, P.stamp);
      } else {
        if (pi == 0 && cont_in) {
          // the run started in an earlier chunk: find that chunk c0 (look back over chunk
          // starts, 32 at a time), then fold the published partials of c0 .. c-1 in order
          long long cc = c - 1, c0 = -1;
          while (c0 < 0) {
            const long long q = cc - lane;
            bool starts = false;
            if (q >= 0)
              starts = (q == 0) || P.keys[q * C] != key0 || P.keys[q * C - 1] != key0;
            const unsigned m = __ballot_sync(kFull, starts);
            if (m) c0 = cc - (__ffs(m) - 1);
            else cc -= 32;
          }
          float4 tot4[NVC];
#pragma unroll
          for (int v = 0; v < NVC; ++v) tot4[v] = make_float4(0.f, 0.f, 0.f, 0.f);
          constexpr int BATCH = 8 / NVC;
          for (long long q0 = c0; q0 < c; q0 += BATCH) {
            const int nb = (c - q0) < BATCH ? (int)(c - q0) : BATCH;
            if (lane < nb) {
              const unsigned long long t0 = globaltimer();
              while (ld_acquire_gpu(P.chunk_flag + q0 + lane) != P.stamp) {
                if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
                  atomicExch(P.err, 0x800);
                  break;
                }
              }
            }
            __syncwarp();
            float4 pv[BATCH][NVC];
#pragma unroll
            for (int x = 0; x < BATCH; ++x)
#pragma unroll
              for (int v = 0; v < NVC; ++v) {
                const int u = lane + 32 * v;
                pv[x][v] = (x < nb && u < DU)
                               ? __ldcg(reinterpret_cast<const float4*>(P.scratch +
                                                                        (q0 + x) * D) + u)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
            for (int x = 0; x < BATCH; ++x)
              if (x < nb)
#pragma unroll
                for (int v = 0; v < NVC; ++v) add4(tot4[v], pv[x][v]);
          }
#pragma unroll
          for (int v = 0; v < NVC; ++v) {
            add4(tot4[v], acc[v]);
            acc[v] = tot4[v];
          }
        }
        // sparse SGD step on the row (R#29): W = W - fl(lr * g)
        float* tp = stp[pi];
#pragma unroll
        for (int v = 0; v < NVC; ++v) {
          const int u = lane + 32 * v;
          if (u < DU) {
            float4 w = lds_f4(smem_u32(stb + pi * D + 4 * u));
            w.x = __fsub_rn(w.x, __fmul_rn(P.lr, acc[v].x));
            w.y = __fsub_rn(w.y, __fmul_rn(P.lr, acc[v].y));
            w.z = __fsub_rn(w.z, __fmul_rn(P.lr, acc[v].z));
            w.w = __fsub_rn(w.w, __fmul_rn(P.lr, acc[v].w));
            st_f4(tp + 4 * u, w);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < NVC; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      ++pi;
    }
    __syncwarp();   // the next chunk reuses this warp's shared memory
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

size_t bwd_smem(const BwdParams& P, int threads) {
  return (size_t)(threads / 32) * ((size_t)2 * P.C * P.D * 4 + 32 * 4 + 32 * 8);
}

}  // namespace

cudaError_t launch_sort_plan(const SortParams& S, const PassParams* passes, int npasses,
                             long long ntiles, int grid_keygen, cudaStream_t st) {
  if (S.TB > 0) {
    if (S.weights) bwd_keygen_kernel<true><<<grid_keygen, 256, 0, st>>>(S);
    else bwd_keygen_kernel<false><<<grid_keygen, 256, 0, st>>>(S);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  for (int p = 0; p < npasses; ++p) {
    if (passes[p].wts_in)
      bwd_onesweep_kernel<true><<<(unsigned)ntiles, kSortThreads, 0, st>>>(passes[p]);
    else
      bwd_onesweep_kernel<false><<<(unsigned)ntiles, kSortThreads, 0, st>>>(passes[p]);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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
  return cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(threads), args, smem,
                          st);
}

}  // namespace emba2a
