// ag_gemm.cu -- fused AllGather + GEMM for B200 (sm_100a): SURVEY.md Sec 8 row f4, PAPER.md
// P:180 (FSDP: "the AllGather collective can be overlapped with the subsequent matrix
// computations").  C ABI: include/ag_gemm.h.  Oracle: oracle/ag_gemm.py.  DESIGN.md Sec 14.
//
// One persistent kernel per rank, warp-specialised (384 threads):
//   warp 0      TMA producer: per output tile, waits for the B operand's ready flag (remote
//               shard chunk; ld.acquire.sys + proxy fence), then streams A = X_r and B = W_s
//               K-blocks of 64 into a 4-stage shared-memory ring (SWIZZLE_128B, mbarrier
//               complete_tx)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16 (128 x BN x 16,
//               bf16 in, fp32 accumulate) into one of two TMEM accumulators; tcgen05.commit
//               frees ring stages and hands finished accumulators to the epilogue
//   warp 2      TMEM allocator (2 x BN columns)
//   warps 4-7   epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32(w%4)..+31 = tile rows),
//               round to bf16 (or keep fp32), 16-byte stores of Y
//   warps 8-11  communication: copy W_r into every peer's gather buffer (16-byte loads, 16-byte
//               stores over NVLink), pieces of one chunk (= one N-tile of rows) spread over the
//               CTAs; the CTA completing a chunk fences at system scope and stores the epoch
//               into the destination's ready flag (P:149 sliceRdy, P:151 PUT -> fence -> flag)
// Tiles are taken in the order: local shard, then sources r-1, r-2, ... (the order in which the
// peers' staggered sends r+1, r+2, ... deliver them), M-tiles rastered in groups for L2 reuse.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ag_gemm.h"

namespace aggemm {

constexpr int kMaxW = AG_GEMM_MAX_WORLD;
constexpr int BM = 128;          // tile rows (UMMA M, one TMEM lane per row)
constexpr int BK = 64;           // K per stage: 64 bf16 = 128 B rows (SWIZZLE_128B atom)
constexpr int UK = 16;           // K per tcgen05.mma (kind::f16)
constexpr int kThreads = 384;
constexpr int kCommWarp0 = 8, kCommThreads = 128;
constexpr int kEpiWarp0 = 4;
enum : int { kErrFlag = 0x100, kErrCredit = 0x200, kErrPipe = 0x400 };

struct Params {
  CUtensorMap tmA;          // X_r [M][K]
  CUtensorMap tmB_local;    // W_r [N_r][K]
  CUtensorMap tmB_g;        // this epoch's gather buffer [N][K]
  void* Y;
  long long ldy;            // = N
  int out_f32;
  int M, N_r, K, W, rank;
  int tiles_m, tiles_n, k_blocks, group_m, order;
  unsigned epoch;
  // communication
  const uint4* w_local;
  uint4* dst[kMaxW];                    // peer q's gather half + this rank's block
  unsigned* flag_out[kMaxW];            // &flags_q[rank][0]
  unsigned long long* credit_out[kMaxW];  // &credits_q[rank]
  const unsigned* flag_in;              // own flags [W][flag_stride]
  int flag_stride;
  const unsigned long long* credit_in;  // own credits, slot q at q * 16
  unsigned* piece_ctr;                  // [W][chunks] monotone, local
  int chunks, pieces, comm, local_copy;
  int l2hints;                          // bits: 1 A evict_last, 2 B evict_first, 4 Y streaming stores
  long long piece_u4;
  int* err;
  long long timeout_ns;
};

// ------------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline that never completes (a broken invariant) reports instead of hanging.
__device__ __forceinline__ bool mbar_wait(unsigned bar, unsigned parity, const Params& P) {
  if (mbar_try(bar, parity)) return true;
  const unsigned long long t0 = globaltimer();
  while (!mbar_try(bar, parity)) {
    if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
      atomicExch(P.err, kErrPipe);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, unsigned bar,
                                            int c0, int c1, unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(policy) : "memory");
}
// L2 policies: the A panel of an M-tile group is re-read for every N-tile of the group (keep
// it), a B tile only by the group's consecutive M-tiles and Y is written once (let them go)
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_normal() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_stream_v4(void* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// tcgen05 --------------------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major operand tile in shared memory written by TMA with SWIZZLE_128B: rows of 128 B, 8-row
// swizzle atoms of 1024 B stacked along M/N.  Descriptor: start >> 4 [0,14), leading byte
// offset >> 4 [16,30) (unused for swizzled K-major, canonical 1), stride byte offset >> 4
// [32,46) = 1024 B between 8-row atoms, version 1 [46,48) (sm_100), layout SWIZZLE_128B = 2
// [61,64).  (cute/arch/mma_sm100_desc.hpp SmemDescriptor; cute make_umma_desc<Major::K>.)
__device__ __forceinline__ unsigned long long smem_desc(unsigned addr) {
  return (unsigned long long)((addr & 0x3FFFFu) >> 4) | (1ull << 16) |
         ((unsigned long long)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1, both
// K-major (bits 15, 16 = 0), N >> 3 at [17,23), M >> 4 at [24,29).
template <int UM, int UN>
__device__ __forceinline__ unsigned instr_desc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(UN >> 3) << 17) |
         ((unsigned)(UM >> 4) << 24);
}
template <bool PAIR>
__device__ __forceinline__ void mma_bf16(unsigned tmem_d, unsigned long long a,
                                         unsigned long long b, unsigned idesc, unsigned acc) {
  if (PAIR)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// MMA completion -> mbarrier: one CTA, or (CTA pair) the barrier at the same offset in both CTAs
template <bool PAIR>
__device__ __forceinline__ void mma_commit(unsigned bar) {
  if (PAIR)
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], m;\n\t}" ::"r"(bar) : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(bar) : "memory");
}
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(unsigned taddr, unsigned (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// clusters (CTA pair) ------------------------------------------------------------------------
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the shared::cluster address of `addr` (a shared::cta offset) in CTA `rank` of the cluster
__device__ __forceinline__ unsigned mapa(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// TMA load into this CTA's shared memory whose completion (bytes) is counted on the pair
// leader's mbarrier (cta_group::2: the leader's MMA reads both CTAs' stages)
__device__ __forceinline__ void tma_load_2d_pair(unsigned dst, const CUtensorMap* map,
                                                 unsigned leader_bar, int c0, int c1,
                                                 unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(leader_bar), "l"(policy) : "memory");
}

// ------------------------------------------------------------------------------ tile order
struct Tile { int s, m, n; };
// Tile t of this rank's sequence: sources in the comm-aware order (own shard, then r-1, r-2, ...)
// or ascending; inside a source, groups of group_m M-tiles, N-tiles outer within a group.
__device__ __forceinline__ Tile tile_of(const Params& P, int t) {
  const int per_src = P.tiles_m * P.tiles_n;
  const int o = t / per_src;
  int u = t - o * per_src;
  Tile x;
  x.s = P.order == 0 ? (P.rank - o + P.W) % P.W : o;
  const int gsz = P.group_m * P.tiles_n;
  const int g = u / gsz;
  u -= g * gsz;
  const int gm = min(P.group_m, P.tiles_m - g * P.group_m);
  x.n = u / gm;
  x.m = g * P.group_m + (u - x.n * gm);
  return x;
}

// Per-configuration constants.  PAIR: a cluster of two CTAs (one per SM of a TPC) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and half of
// the tile's B rows (BN/2), the leader issues M = 256 MMAs reading both CTAs' stages, and each
// CTA's TMEM receives its 128 rows x BN accumulator.  Half the B bytes per SM, so more stages.
template <int BN, bool PAIR, int NSTG = 0>
struct Cfg {
  static constexpr int kBRows = PAIR ? BN / 2 : BN;
  static constexpr unsigned kABytes = BM * BK * 2;
  static constexpr unsigned kBBytes = kBRows * BK * 2;
  static constexpr int kStages = NSTG ? NSTG : (PAIR ? (BN == 256 ? 6 : 8) : 4);
  static constexpr int kUM = PAIR ? 2 * BM : BM;
  static constexpr unsigned kTmemCols = 2 * BN;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * (kABytes + kBBytes) +
                                  8 * (2 * kStages + 4) + 16;
};

// ---------------------------------------------------------------------------------- kernel
template <int BN, bool PAIR, int NSTG = 0>
__global__ void __launch_bounds__(kThreads, 1) ag_gemm_kernel(const __grid_constant__ Params P) {
  using C = Cfg<BN, PAIR, NSTG>;
  constexpr int NS = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = smem;
  unsigned char* sb = smem + NS * C::kABytes;
  unsigned long long* bars = (unsigned long long*)(sb + NS * C::kBBytes);
  // bars: full[NS], empty[NS], tfull[2], tempty[2]
  unsigned* tmem_slot = (unsigned*)(bars + 2 * NS + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned crank = PAIR ? cluster_ctarank() : 0u;     // 0 = the pair's leader
  const bool leader = crank == 0;
  const unsigned bar0 = smem_u32(bars);
  auto full_bar = [&](int i) { return bar0 + 8u * i; };
  auto empty_bar = [&](int i) { return bar0 + 8u * (NS + i); };
  auto tfull_bar = [&](int i) { return bar0 + 8u * (2 * NS + i); };
  auto tempty_bar = [&](int i) { return bar0 + 8u * (2 * NS + 2 + i); };

  if (warp == 0 && lane == 0) {
    prefetch_map(&P.tmA);
    prefetch_map(&P.tmB_local);
    prefetch_map(&P.tmB_g);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full_bar(i), 1);   // pair: the leader's expect_tx covers both CTAs' bytes
      mbar_init(empty_bar(i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull_bar(i), 1);
      mbar_init(tempty_bar(i), PAIR ? 8 : 4);   // one arrival per epilogue warp (of both CTAs)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(C::kTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(tmem_slot)), "r"(C::kTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  // this forward started: our previous forward (same stream) has completed, so every peer may
  // overwrite the gather half it used (DESIGN.md Sec 14 buffer reuse)
  if (blockIdx.x == 0 && threadIdx.x == kCommWarp0 * 32 && P.comm)
    for (int q = 0; q < P.W; ++q)
      if (q != P.rank) red_release_sys_add(P.credit_out[q], 1ull);
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const unsigned tmem_base = *tmem_slot;
  const int ntiles = P.W * P.tiles_m * P.tiles_n;
  const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // cluster / CTA index
  const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      int stage = 0;
      unsigned phase = 0;
      int ready_s = -1, ready_n = -1;
      bool ok = true;
      const unsigned lbar0 = PAIR ? mapa(full_bar(0), 0) : full_bar(0);   // leader's full[0]
      const unsigned long long pol_a = (P.l2hints & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
      const unsigned long long pol_b = (P.l2hints & 2) ? l2_policy_evict_first() : l2_policy_evict_normal();
      for (int t = unit; t < ntiles && ok; t += nunits) {
        const Tile x = tile_of(P, t);
        const CUtensorMap* mb = &P.tmB_local;
        int brow = x.n * BN + (int)crank * C::kBRows;
        if (x.s != P.rank) {
          mb = &P.tmB_g;
          brow += x.s * P.N_r;
          if (x.s != ready_s || x.n != ready_n) {
            // consume a slice only after its ready flag; acquire at system scope, then
            // order the async proxy (TMA) after the generic-proxy stores the flag covers
            const unsigned* f = P.flag_in + (size_t)x.s * P.flag_stride + x.n;
            if (ld_acquire_sys(f) < P.epoch) {
              const unsigned long long t0 = globaltimer();
              while (ld_acquire_sys(f) < P.epoch) {
                if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
                  atomicExch(P.err, kErrFlag | x.s);
                  ok = false;
                  break;
                }
              }
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            ready_s = x.s;
            ready_n = x.n;
          }
        }
        const int arow = x.m * C::kUM + (int)crank * BM;
        for (int kb = 0; kb < P.k_blocks && ok; ++kb) {
          if (!mbar_wait(empty_bar(stage), phase ^ 1u, P)) { ok = false; break; }
          const unsigned da = smem_u32(sa + stage * C::kABytes);
          const unsigned db = smem_u32(sb + stage * C::kBBytes);
          if (PAIR) {
            // the peer's bytes may land on the leader's barrier before the leader's expect_tx
            // (a transiently negative tx-count); the phase cannot complete without the leader's
            // arrival, and the peer refills a stage only after the MMA freed it (its own empty
            // barrier, multicast commit).  (A remote arrive per stage was a MEMBAR.GPU each.)
            const unsigned lb = lbar0 + 8u * stage;
            if (leader) mbar_expect_tx(full_bar(stage), 2 * (C::kABytes + C::kBBytes));
            tma_load_2d_pair(da, &P.tmA, lb, kb * BK, arow, pol_a);
            tma_load_2d_pair(db, mb, lb, kb * BK, brow, pol_b);
          } else {
            mbar_expect_tx(full_bar(stage), C::kABytes + C::kBBytes);
            tma_load_2d(da, &P.tmA, full_bar(stage), kb * BK, arow, pol_a);
            tma_load_2d(db, mb, full_bar(stage), kb * BK, brow, pol_b);
          }
          if (++stage == NS) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer (the pair's leader) ============
    if (lane == 0 && leader) {
      const unsigned idesc = instr_desc<C::kUM, BN>();
      int stage = 0;
      unsigned phase = 0;
      int it = 0;
      bool ok = true;
      for (int t = unit; t < ntiles && ok; t += nunits, ++it) {
        const int as = it & 1;
        const unsigned aph = (unsigned)(it >> 1) & 1u;
        if (!mbar_wait(tempty_bar(as), aph ^ 1u, P)) break;
        tc_fence_after();
        const unsigned dacc = tmem_base + (unsigned)(as * BN);
        for (int kb = 0; kb < P.k_blocks; ++kb) {
          if (!mbar_wait(full_bar(stage), phase, P)) { ok = false; break; }
          tc_fence_after();
          const unsigned a0 = smem_u32(sa + stage * C::kABytes);
          const unsigned b0 = smem_u32(sb + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k)   // +32 B along K inside the 128-B swizzled row
            mma_bf16<PAIR>(dacc, smem_desc(a0 + k * UK * 2), smem_desc(b0 + k * UK * 2), idesc,
                           (kb | k) != 0);
          mma_commit<PAIR>(empty_bar(stage));   // frees the stage (in both CTAs of a pair)
          if (++stage == NS) { stage = 0; phase ^= 1u; }
        }
        mma_commit<PAIR>(tfull_bar(as));        // accumulator complete -> epilogue(s)
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
    // ============================== epilogue ==================================
    const int q = warp & 3;                   // TMEM lanes 32q..32q+31 = tile rows
    auto st_y = [&](uint4* p, const uint4& v) {
      if (P.l2hints & 4) st_stream_v4(p, v); // Y is written once: do not displace the A panel
      else *p = v;
    };
    const unsigned lt0 = PAIR ? mapa(tempty_bar(0), 0) : tempty_bar(0);
    int it = 0;
    for (int t = unit; t < ntiles; t += nunits, ++it) {
      const Tile x = tile_of(P, t);
      const int as = it & 1;
      const unsigned aph = (unsigned)(it >> 1) & 1u;
      if (!mbar_wait(tfull_bar(as), aph, P)) break;
      tc_fence_after();
      const long long row = (long long)x.m * C::kUM + (long long)crank * BM + q * 32 + lane;
      const long long col0 = (long long)x.s * P.N_r + (long long)x.n * BN;
      const unsigned taddr = tmem_base + ((unsigned)(q * 32) << 16) + (unsigned)(as * BN);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        unsigned v[32];
        tmem_ld32(taddr + c * 32, v);
        if (P.out_f32) {
          uint4* dst = (uint4*)((float*)P.Y + row * P.ldy + col0 + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st_y(dst + j, make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        } else {
          unsigned pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(v[2 * j]),
                                                      __uint_as_float(v[2 * j + 1]));
            pk[j] = *(unsigned*)&b2;
          }
          uint4* dst = (uint4*)((__nv_bfloat16*)P.Y + row * P.ldy + col0 + c * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_y(dst + j, make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) mbar_arrive_remote(lt0 + 8u * as);   // the leader's MMA reuses both halves
        else mbar_arrive(tempty_bar(as));
      }
    }
  } else if (warp >= kCommWarp0 && P.comm) {
    // ============================== communication =============================
    // unit u = ((dest ordinal d, chunk c), piece p); destination d -> rank (r+1+d) mod W,
    // local copy (if asked) last.  Every CTA walks the same order in lock-step, so chunk
    // (d=0, c=0) completes first (P:151 staggered, remote first).
    const int ctid = threadIdx.x - kCommWarp0 * 32;
    const int ndest = (P.W - 1) + (P.local_copy ? 1 : 0);
    const long long units = (long long)ndest * P.chunks * P.pieces;
    __shared__ int s_credit_ok;
    int credited = -1;
    const long long chunk_u4 = (long long)P.pieces * P.piece_u4;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const int d = (int)(u / ((long long)P.chunks * P.pieces));
      const long long rem = u - (long long)d * P.chunks * P.pieces;
      const int c = (int)(rem / P.pieces);
      const int p = (int)(rem - (long long)c * P.pieces);
      const int dst_rank = d < P.W - 1 ? (P.rank + 1 + d) % P.W : P.rank;
      if (dst_rank != credited) {
        // peer q must have started forward e-1 before anything lands in the half it read in
        // forward e-2 (a forward's credit = its previous forward completed)
        if (ctid == 0) {
          int okc = 1;
          if (dst_rank != P.rank && P.epoch > 1) {
            const unsigned long long* cr = P.credit_in + (size_t)dst_rank * 16;
            const unsigned long long want = P.epoch - 1;
            if (ld_acquire_sys64(cr) < want) {
              const unsigned long long t0 = globaltimer();
              while (ld_acquire_sys64(cr) < want)
                if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
                  atomicExch(P.err, kErrCredit | dst_rank);
                  okc = 0;
                  break;
                }
            }
          }
          s_credit_ok = okc;
        }
        named_bar(1, kCommThreads);
        if (!s_credit_ok) break;
        credited = dst_rank;
      }
      const uint4* src = P.w_local + (long long)c * chunk_u4 + (long long)p * P.piece_u4;
      uint4* dst = P.dst[dst_rank] + (long long)c * chunk_u4 + (long long)p * P.piece_u4;
      constexpr int U = 8;
      for (long long i0 = 0; i0 < P.piece_u4; i0 += (long long)U * kCommThreads) {
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const long long i = i0 + (long long)j * kCommThreads + ctid;
          if (i < P.piece_u4) v[j] = ld_stream(src + i);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const long long i = i0 + (long long)j * kCommThreads + ctid;
          if (i < P.piece_u4) st_v4(dst + i, v[j]);
        }
      }
      named_bar(1, kCommThreads);   // every comm thread's stores of this piece precede ...
      if (ctid == 0 && dst_rank != P.rank) {
        fence_acq_rel_sys();          // ... this system-scope fence (R#25 pattern)
        const unsigned old = atomicAdd(P.piece_ctr + (size_t)dst_rank * P.chunks + c, 1u);
        if (old + 1u == P.epoch * (unsigned)P.pieces) {
          fence_acq_rel_sys();        // acquire the other pieces' fences, then publish
          st_release_sys(P.flag_out[dst_rank] + c, P.epoch);
        }
      }
    }
  }

  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();   // both CTAs done with TMEM and stages
  if (warp == 2) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(C::kTmemCols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(C::kTmemCols) : "memory");
  }
}

}  // namespace aggemm

// =============================================================================== host side
using namespace aggemm;

namespace {
constexpr uint32_t kMagicAG = 0xA6E33A01u;
constexpr int kErrWordsAG = 2;

struct MetaAG {
  uint32_t magic;
  int32_t rank, world, out_f32;
  int64_t M, N_r, K;
  int32_t bn, pad;
};
struct HandlesAG {
  uint32_t magic;
  int32_t pid, device, pad;
  uint64_t host_id, raw_ptr, region_bytes;
  cudaIpcMemHandle_t ipc;
  char bus_id[32];
};
uint64_t host_id_ag() {
  char name[256] = {0};
  gethostname(name, sizeof(name) - 1);
  uint64_t h = 1469598103934665603ull;
  for (const char* p = name; *p; ++p) h = (h ^ (uint8_t)*p) * 1099511628211ull;
  return h;
}
}  // namespace

struct ag_gemm {
  int rank = 0, W = 1, dev = 0;
  ag_gemm_allgather_fn allgather = nullptr;
  void* user = nullptr;
  bool registered = false, poisoned = false, shared_gpu = false;
  std::string last_error;
  int64_t M = 0, N_r = 0, K = 0;
  int out_f32 = 0, BN = 256, chunks = 0, pieces = 0, flag_stride = 0, sms = 0;
  char* region = nullptr;
  size_t region_bytes = 0, flag_bytes = 0, credit_bytes = 0, half_bytes = 0;
  char* peer_base[kMaxW] = {};
  std::vector<void*> opened;
  unsigned* piece_ctr = nullptr;
  unsigned epoch = 0;
  int* h_err = nullptr;
  int* d_err = nullptr;
  int64_t opt_grid = 0, local_copy = 0, order = 0, group_m = 16, piece_kb = 64,
          timeout_ms = 10000, comm = 1, pair = 1, stages = 6, opt_bn = 0, l2hints = 0;
};

namespace {
int fail(ag_gemm* h, int code, const char* fmt, ...) {
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
#define AG_TRY(h, call)                                                                    \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail((h), e_ == cudaErrorMemoryAllocation ? 4 : 3, "%s: %s", #call,            \
                  cudaGetErrorString(e_));                                                 \
  } while (0)

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); }
  ~DevGuard() { cudaSetDevice(prev); }
};

int check_async(ag_gemm* h) {
  if (h->poisoned) return fail(h, 2, "handle poisoned by an earlier failure: %s",
                               h->last_error.c_str());
  if (h->h_err && *(volatile int*)h->h_err != 0) {
    const int v = *(volatile int*)h->h_err;
    h->poisoned = true;
    const char* what = (v & kErrFlag) ? "ready-flag wait timed out (source %d never signalled)"
                       : (v & kErrCredit) ? "credit wait timed out (rank %d never started its "
                                            "previous forward)"
                                          : "pipeline wait timed out (%d)";
    return fail(h, 7, what, v & 0xff);
  }
  return 0;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn(ag_gemm* h) {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      f = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  if (!f) fail(h, 3, "cuTensorMapEncodeTiled unavailable");
  return f;
}

// 2D bf16 K-major tensor [rows][K], box {64, box_rows}, SWIZZLE_128B.
int make_map(ag_gemm* h, CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows) {
  auto f = encode_fn(h);
  if (!f) return 3;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(h, 1, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

template <int BN, bool PAIR, int NSTG = 0>
cudaError_t set_smem_attr() {
  return cudaFuncSetAttribute(ag_gemm_kernel<BN, PAIR, NSTG>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)Cfg<BN, PAIR, NSTG>::kSmem);
}

// CTA pairs (cta_group::2) need M % 256 == 0 and an even grid; option "pair" 0 forces single CTAs
bool use_pair(const ag_gemm* h) { return h->pair && h->M % 256 == 0; }

int64_t grid_of(const ag_gemm* h) {
  const bool pair = use_pair(h);
  const int64_t tiles = (int64_t)h->W * (h->M / (pair ? 256 : 128)) * h->chunks;
  int64_t g = h->opt_grid > 0 ? h->opt_grid : (h->shared_gpu ? h->sms / h->W : h->sms);
  if (pair) {
    g = std::max<int64_t>(1, std::min<int64_t>(g / 2, tiles)) * 2;   // clusters of two CTAs
  } else {
    g = std::max<int64_t>(1, std::min<int64_t>(g, tiles));
  }
  return g;
}

template <int BN, bool PAIR, int NSTG = 0>
cudaError_t launch(const Params& P, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<BN, PAIR, NSTG>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ag_gemm_kernel<BN, PAIR, NSTG>, P);
}

void release(ag_gemm* h) {
  for (void* p : h->opened) cudaIpcCloseMemHandle(p);
  h->opened.clear();
  if (h->region) cudaFree(h->region);
  if (h->piece_ctr) cudaFree(h->piece_ctr);
  h->region = nullptr;
  h->piece_ctr = nullptr;
  h->registered = false;
}
}  // namespace

extern "C" {

int ag_gemm_init(int rank, int world_size, int cuda_device, ag_gemm_allgather_fn allgather,
                 void* user, ag_gemm_t** out) {
  if (!out || world_size < 1 || world_size > kMaxW || rank < 0 || rank >= world_size ||
      (!allgather && world_size > 1))
    return 1;
  *out = nullptr;
  ag_gemm* h = new ag_gemm();
  h->rank = rank;
  h->W = world_size;
  h->dev = cuda_device;
  h->allgather = allgather;
  h->user = user;
  DevGuard g(cuda_device);
  if (cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, cuda_device) !=
      cudaSuccess) {
    delete h;
    return 3;
  }
  if (cudaHostAlloc((void**)&h->h_err, kErrWordsAG * sizeof(int), cudaHostAllocMapped) !=
      cudaSuccess) {
    delete h;
    return 4;
  }
  h->h_err[0] = h->h_err[1] = 0;
  cudaHostGetDevicePointer((void**)&h->d_err, h->h_err, 0);
  *out = h;
  return 0;
}

int ag_gemm_register(ag_gemm_t* h, int64_t M, int64_t n_local, int64_t K, int out_f32) {
  if (!h) return 1;
  if (h->poisoned) return check_async(h);
  DevGuard g(h->dev);
  if (h->registered) {
    cudaDeviceSynchronize();
    release(h);
  }
  if (M < BM || M % BM || n_local < 128 || n_local % 128 || K < BK || K % BK ||
      (out_f32 != 0 && out_f32 != 1) || (int64_t)h->W * n_local * K >= (1ll << 40) ||
      M >= (1ll << 31) || K >= (1ll << 31) || (int64_t)h->W * n_local >= (1ll << 31))
    return fail(h, 1, "shape: need M %% 128 == 0, N_r %% 128 == 0, K %% 64 == 0 (M=%lld N_r=%lld "
                "K=%lld)", (long long)M, (long long)n_local, (long long)K);
  // N-tile (= communication chunk rows): 256 when N_r allows it (option "bn" forces 128).
  // Measured (r02w, ag_small): 128-row tiles fill the last wave of the persistent grid better
  // (98.8 % vs 86.5 %) but run at 977 vs 1469 TFLOP/s -- twice the A traffic per flop.
  const int bn = (h->opt_bn == 128 || n_local % 256 != 0) ? 128 : 256;
  MetaAG me{kMagicAG, h->rank, h->W, out_f32, M, n_local, K, bn};
  std::vector<MetaAG> all(h->W);
  if (h->W > 1) {
    if (h->allgather(&me, all.data(), sizeof(MetaAG), h->user) != 0)
      return fail(h, 6, "all-gather callback failed (metadata)");
    for (int q = 0; q < h->W; ++q)
      if (all[q].magic != kMagicAG || all[q].rank != q || all[q].world != h->W ||
          all[q].M != M || all[q].N_r != n_local || all[q].K != K || all[q].out_f32 != out_f32 ||
          all[q].bn != bn)
        return fail(h, 1, "ranks disagree on the problem shape / N-tile (rank %d)", q);
  }
  h->M = M;
  h->N_r = n_local;
  h->K = K;
  h->out_f32 = out_f32;
  h->BN = bn;
  h->chunks = (int)(n_local / h->BN);
  const int64_t chunk_bytes = (int64_t)h->BN * K * 2;
  int64_t piece = h->piece_kb * 1024;
  while (piece > chunk_bytes) piece >>= 1;
  h->pieces = (int)(chunk_bytes / piece);
  h->flag_stride = (h->chunks + 31) / 32 * 32;
  h->flag_bytes = ((size_t)h->W * h->flag_stride * 4 + 1023) / 1024 * 1024;
  h->credit_bytes = ((size_t)h->W * 128 + 1023) / 1024 * 1024;
  h->half_bytes = ((size_t)h->W * n_local * K * 2 + 1023) / 1024 * 1024;
  h->region_bytes = h->flag_bytes + h->credit_bytes + 2 * h->half_bytes;
  AG_TRY(h, cudaMalloc((void**)&h->region, h->region_bytes));
  AG_TRY(h, cudaMemset(h->region, 0, h->flag_bytes + h->credit_bytes));
  AG_TRY(h, cudaMalloc((void**)&h->piece_ctr, sizeof(unsigned) * h->W * h->chunks));
  AG_TRY(h, cudaMemset(h->piece_ctr, 0, sizeof(unsigned) * h->W * h->chunks));
  h->epoch = 0;

  HandlesAG mine;
  memset(&mine, 0, sizeof(mine));
  mine.magic = kMagicAG;
  mine.pid = (int32_t)getpid();
  mine.device = h->dev;
  cudaDeviceGetPCIBusId(mine.bus_id, sizeof(mine.bus_id), h->dev);
  mine.host_id = host_id_ag();
  mine.raw_ptr = (uint64_t)(uintptr_t)h->region;
  mine.region_bytes = h->region_bytes;
  std::vector<HandlesAG> hs(h->W);
  h->shared_gpu = false;
  if (h->W > 1) {
    AG_TRY(h, cudaIpcGetMemHandle(&mine.ipc, h->region));
    if (h->allgather(&mine, hs.data(), sizeof(HandlesAG), h->user) != 0)
      return fail(h, 6, "all-gather callback failed (handles)");
  } else {
    hs[0] = mine;
  }
  for (int q = 0; q < h->W; ++q) {
    const HandlesAG& o = hs[q];
    if (q != h->rank && o.host_id == mine.host_id &&
        strncmp(o.bus_id, mine.bus_id, sizeof(mine.bus_id)) == 0)
      h->shared_gpu = true;
    if (q == h->rank) {
      h->peer_base[q] = h->region;
    } else if (o.pid == mine.pid && o.host_id == mine.host_id) {
      h->peer_base[q] = (char*)(uintptr_t)o.raw_ptr;
      if (o.device != h->dev) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, h->dev, o.device);
        if (!can) return fail(h, 5, "no P2P path from device %d to %d", h->dev, o.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(h, 5, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
        cudaGetLastError();
      }
    } else {
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, o.ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        return fail(h, 5, "cudaIpcOpenMemHandle(rank %d): %s", q, cudaGetErrorString(e));
      h->opened.push_back(p);
      h->peer_base[q] = (char*)p;
    }
  }
  AG_TRY(h, (set_smem_attr<256, false>()));
  AG_TRY(h, (set_smem_attr<128, false>()));
  AG_TRY(h, (set_smem_attr<256, true>()));
  AG_TRY(h, (set_smem_attr<128, true>()));
  AG_TRY(h, (set_smem_attr<256, true, 7>()));
  h->registered = true;
  return 0;
}

int ag_gemm_forward(ag_gemm_t* h, const void* X, const void* w_local, void* Y, void* stream,
                    void** w_gathered) {
  if (!h) return 1;
  int rc = check_async(h);
  if (rc) return rc;
  if (!h->registered) return fail(h, 2, "forward before register");
  if (!X || !w_local || !Y || ((uintptr_t)X & 15) || ((uintptr_t)w_local & 15) ||
      ((uintptr_t)Y & 15))
    return fail(h, 1, "X, w_local and Y must be non-null, 16-byte aligned device pointers");
  DevGuard g(h->dev);
  const unsigned e = h->epoch + 1;
  const int half = (int)(e & 1u);
  Params P;
  memset(&P, 0, sizeof(P));
  const bool pair = use_pair(h);
  const int brows = pair ? h->BN / 2 : h->BN;   // B rows one CTA stages per tile
  rc = make_map(h, &P.tmA, X, h->M, h->K, BM);
  if (!rc) rc = make_map(h, &P.tmB_local, w_local, h->N_r, h->K, brows);
  char* my_half = h->region + h->flag_bytes + h->credit_bytes + (size_t)half * h->half_bytes;
  if (!rc) rc = make_map(h, &P.tmB_g, my_half, (int64_t)h->W * h->N_r, h->K, brows);
  if (rc) return rc;
  P.Y = Y;
  P.ldy = (long long)h->W * h->N_r;
  P.out_f32 = h->out_f32;
  P.M = (int)h->M;
  P.N_r = (int)h->N_r;
  P.K = (int)h->K;
  P.W = h->W;
  P.rank = h->rank;
  P.tiles_m = (int)(h->M / (pair ? 2 * BM : BM));
  P.tiles_n = h->chunks;
  P.k_blocks = (int)(h->K / BK);
  P.group_m = (int)std::max<int64_t>(1, h->group_m);
  P.order = (int)h->order;
  P.epoch = e;
  P.w_local = (const uint4*)w_local;
  const size_t block_off = (size_t)h->rank * h->N_r * h->K * 2;
  for (int q = 0; q < h->W; ++q) {
    char* b = h->peer_base[q];
    P.dst[q] = (uint4*)(b + h->flag_bytes + h->credit_bytes + (size_t)half * h->half_bytes +
                        block_off);
    P.flag_out[q] = (unsigned*)b + (size_t)h->rank * h->flag_stride;
    P.credit_out[q] = (unsigned long long*)(b + h->flag_bytes) + (size_t)h->rank * 16;
  }
  P.flag_in = (const unsigned*)h->region;
  P.flag_stride = h->flag_stride;
  P.credit_in = (const unsigned long long*)(h->region + h->flag_bytes);
  P.piece_ctr = h->piece_ctr;
  P.chunks = h->chunks;
  P.pieces = h->pieces;
  P.piece_u4 = (long long)h->BN * h->K * 2 / 16 / h->pieces;
  P.comm = (h->W > 1 || h->local_copy) ? (int)h->comm : 0;
  P.local_copy = (int)h->local_copy;
  P.l2hints = (int)h->l2hints;
  P.err = h->d_err;
  P.timeout_ns = h->timeout_ms * 1000000ll;
  const int grid = (int)grid_of(h);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t le;
  if (h->BN == 256)
    le = pair ? (h->stages == 7 ? launch<256, true, 7>(P, grid, st) : launch<256, true>(P, grid, st))
              : launch<256, false>(P, grid, st);
  else le = pair ? launch<128, true>(P, grid, st) : launch<128, false>(P, grid, st);
  if (le != cudaSuccess) return fail(h, 3, "launch: %s", cudaGetErrorString(le));
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) return fail(h, 3, "launch: %s", cudaGetErrorString(ce));
  h->epoch = e;
  if (w_gathered) *w_gathered = my_half;
  return 0;
}

int ag_gemm_set_option(ag_gemm_t* h, const char* key, int64_t v) {
  if (!h || !key) return 1;
  std::string k(key);
  if (k == "grid") { if (v < 0) return fail(h, 1, "grid >= 0"); h->opt_grid = v; }
  else if (k == "local_copy") { if (v != 0 && v != 1) return fail(h, 1, "local_copy 0/1"); h->local_copy = v; }
  else if (k == "order") { if (v != 0 && v != 1) return fail(h, 1, "order 0/1"); h->order = v; }
  else if (k == "group_m") { if (v < 1 || v > 4096) return fail(h, 1, "group_m 1..4096"); h->group_m = v; }
  else if (k == "piece_kb") {
    if (v < 4 || v > 1024 || (v & (v - 1))) return fail(h, 1, "piece_kb: power of two 4..1024");
    if (h->registered) return fail(h, 2, "piece_kb must be set before register");
    h->piece_kb = v;
  }
  else if (k == "timeout_ms") { if (v < 1) return fail(h, 1, "timeout_ms >= 1"); h->timeout_ms = v; }
  else if (k == "comm") { if (v != 0 && v != 1) return fail(h, 1, "comm 0/1"); h->comm = v; }
  else if (k == "pair") { if (v != 0 && v != 1) return fail(h, 1, "pair 0/1"); h->pair = v; }
  else if (k == "l2hints") { if (v < 0 || v > 7) return fail(h, 1, "l2hints: bit mask 0..7"); h->l2hints = v; }
  else if (k == "stages") { if (v != 6 && v != 7) return fail(h, 1, "stages 6/7"); h->stages = v; }
  else if (k == "bn") {
    if (v != 0 && v != 128 && v != 256) return fail(h, 1, "bn: 0 (auto), 128 or 256");
    if (h->registered) return fail(h, 2, "bn must be set before register");
    h->opt_bn = v;
  }
  else return fail(h, 1, "unknown option '%s'", key);
  return 0;
}

int ag_gemm_get_option(const ag_gemm_t* h, const char* key, int64_t* v) {
  if (!h || !key || !v) return 1;
  std::string k(key);
  if (k == "grid") *v = h->opt_grid;
  else if (k == "local_copy") *v = h->local_copy;
  else if (k == "order") *v = h->order;
  else if (k == "group_m") *v = h->group_m;
  else if (k == "piece_kb") *v = h->piece_kb;
  else if (k == "timeout_ms") *v = h->timeout_ms;
  else if (k == "comm") *v = h->comm;
  else if (k == "pair") *v = h->pair;
  else if (k == "l2hints") *v = h->l2hints;
  else if (k == "stages") *v = h->stages;
  else if (k == "bn") *v = h->opt_bn;
  else return 1;
  return 0;
}

int ag_gemm_query(const ag_gemm_t* h, const char* key, int64_t* v) {
  if (!h || !key || !v) return 1;
  std::string k(key);
  const bool pair = h->registered && use_pair(h);
  const int64_t tiles = h->registered ? (int64_t)h->W * (h->M / (pair ? 256 : 128)) * h->chunks : 0;
  if (k == "tiles") *v = tiles;
  else if (k == "grid") *v = h->registered ? grid_of(h) : 0;
  else if (k == "pair") *v = pair ? 1 : 0;
  else if (k == "bn") *v = h->BN;
  else if (k == "chunks") *v = h->chunks;
  else if (k == "pieces") *v = h->pieces;
  else if (k == "epoch") *v = h->epoch;
  else if (k == "shared_gpu") *v = h->shared_gpu ? 1 : 0;
  else if (k == "smem_bytes")
    *v = (int64_t)(h->BN == 256 ? (pair ? (h->stages == 7 ? Cfg<256, true, 7>::kSmem
                                                         : Cfg<256, true>::kSmem)
                                        : Cfg<256, false>::kSmem)
                                : (pair ? Cfg<128, true>::kSmem : Cfg<128, false>::kSmem));
  else return 1;
  return 0;
}

int ag_gemm_read_flags(ag_gemm_t* h, uint32_t* out, int64_t capacity, int64_t* n) {
  if (!h || !out) return 1;
  if (!h->registered) return fail(h, 2, "read_flags before register");
  DevGuard g(h->dev);
  const int64_t need = (int64_t)h->W * h->chunks;
  if (n) *n = need;
  if (capacity < need) return fail(h, 1, "capacity %lld < %lld", (long long)capacity,
                                   (long long)need);
  std::vector<uint32_t> all((size_t)h->W * h->flag_stride);
  AG_TRY(h, cudaMemcpy(all.data(), h->region, all.size() * 4, cudaMemcpyDeviceToHost));
  for (int s = 0; s < h->W; ++s)
    for (int c = 0; c < h->chunks; ++c) out[s * h->chunks + c] = all[(size_t)s * h->flag_stride + c];
  return 0;
}

int ag_gemm_check(ag_gemm_t* h) {
  if (!h) return 1;
  return check_async(h);
}

int ag_gemm_destroy(ag_gemm_t* h) {
  if (!h) return 1;
  {
    DevGuard g(h->dev);
    if (h->registered) {
      cudaDeviceSynchronize();
      if (h->W > 1 && h->allgather) {   // no peer unmaps while another still stores into it
        int one = 1;
        std::vector<int> all(h->W);
        h->allgather(&one, all.data(), sizeof(int), h->user);
      }
    }
    release(h);
    if (h->h_err) cudaFreeHost(h->h_err);
  }
  delete h;
  return 0;
}

const char* ag_gemm_last_error(const ag_gemm_t* h) {
  return h ? h->last_error.c_str() : "null handle";
}

}  // extern "C"
