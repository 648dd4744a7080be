// fused_kernel.cuh -- the fused (and pool) kernel template of libemba2a.so, sm_100a.
// Included by the instantiation units inst_*.cu (one per table element type, compiled in
// parallel) and by kernels.cu (tooling kernels, launch).
//
// The fused kernel performs the rows of SURVEY.md Sec 8(a) for one rank r:
//   a1  walk this rank's work in comm-aware order: remote destinations first, staggered
//       (r+1 .. r+W-1) mod W, local last (R#19); work is handed out as chunks of C bags
//   a2  stage each chunk's CSR offsets in shared memory
//   a3  gather the bags' table rows: TMA tile::gather4 copies whole rows into a shared-memory
//       stage (4 arbitrary rows per instruction, completion counted in bytes on an mbarrier), so
//       every row of a stage is in flight at once -- no per-thread unroll / register budget
//   a4  sum-pool in fp32, ascending bag order, from +0.0 (R#5), reading the stage
//   a5  place: row i = j - p_s, columns (toff + t) * D of s's [b_s][G*D] buffer
//   a6  store straight into the destination GPU's receive buffer (zero-copy)
//   a7  a remote slice of S bags is released once: every CTA that finished part of it makes its
//       stores visible system-wide and adds its bag count to the slice's counter; the CTA whose
//       add completes the slice does red.release.sys on the destination's arrival counter
//       (the last-finisher WG_Done / PUT -> fence -> sliceRdy protocol of P:147-151)
//   a8  the last CTA to finish polls the W-1 incoming counters with ld.acquire.sys until every
//       peer's slices for this epoch have arrived ("poll ... before exiting")
// The unfused baseline kernel (pool_local) runs the same gather body and stores to a local
// dest-major staging buffer instead ("stored into an intermediate buffer").
// A second gather mode (tma = 0) loads rows with per-lane 16-byte LDGs instead of TMA; it is also
// the path for a single bag too large for a shared-memory stage.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "emb_a2a_internal.h"

namespace emba2a {
namespace {

// ------------------------------------------------------------------------------------ PTX
__device__ __forceinline__ void st_out4(float* p, const float4& v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// a5/a6 store of 4 pooled fp32 values at byte address p in the output element type: fp32 as one
// 16-byte st.global.v4; bf16 / fp16 rounded to nearest even (R#32) and stored as 8 bytes.
__device__ __forceinline__ void st_out_e4(char* p, float a, float b, float c, float d, int odt) {
  if (odt == 0) {
    st_out4(reinterpret_cast<float*>(p), make_float4(a, b, c, d));
    return;
  }
  unsigned lo, hi;
  if (odt == 1) {
    const __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
    lo = *reinterpret_cast<const unsigned*>(&x);
    hi = *reinterpret_cast<const unsigned*>(&y);
  } else {
    const __half2 x = __floats2half2_rn(a, b), y = __floats2half2_rn(c, d);
    lo = *reinterpret_cast<const unsigned*>(&x);
    hi = *reinterpret_cast<const unsigned*>(&y);
  }
  asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(lo), "r"(hi) : "memory");
}

__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long atom_add_acqrel_gpu(unsigned long long* p,
                                                                  unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void add4(float4& a, const float4& x) {
  a.x = __fadd_rn(a.x, x.x);
  a.y = __fadd_rn(a.y, x.y);
  a.z = __fadd_rn(a.z, x.z);
  a.w = __fadd_rn(a.w, x.w);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ int lds_s32(unsigned addr) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float4 lds_f4(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Predicated 16-byte read-only row load: when !pred the destination is +0.0 (no memory access).
__device__ __forceinline__ float4 ld_row4_pred(const float4* p, bool pred) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
      : "l"(p), "r"((int)pred));
  return v;
}

// Predicated 16-byte raw load ("unit"): when !pred the destination is all-zero bits, which is +0.0
// in every element type (no memory access).  L1 = false: L1::no_allocate (streams past L1); L1 =
// true: the row is allocated in L1, so a hot (Zipf head) row gathered again by the same SM is
// served there instead of queueing on its L2 slice (the fp32 "L1 rows" instance set, ELEM 3).
template <bool L1>
__device__ __forceinline__ uint4 ld_unit_pred(const uint4* p, bool pred) {
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if constexpr (L1)
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"((int)pred));
  else
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
        : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w)
        : "l"(p), "r"((int)pred));
  return v;
}

__device__ __forceinline__ float lds_f32(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Table element types: 0 = fp32 (4 per 16-byte unit), 1 = bf16, 2 = fp16 (8 per unit); 3, 4, 5 =
// fp32, bf16, fp16 with L1-allocating row loads (ld_unit_pred).  Every element is converted
// EXACTLY to fp32 before it is accumulated (R#28).
template <int ELEM>
struct Elem {
  static constexpr int EPU = (ELEM == 0 || ELEM == 3) ? 4 : 8;
};

template <int ELEM>
__device__ __forceinline__ void unit_to_f(const uint4& u, float (&f)[Elem<ELEM>::EPU]) {
  if constexpr (ELEM == 0 || ELEM == 3) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  } else if constexpr (ELEM == 1 || ELEM == 4) {   // bf16 = top half of binary32
    const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {                            // IEEE binary16
    const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __half2float(__ushort_as_half((unsigned short)(w[i] & 0xFFFFu)));
      f[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(w[i] >> 16)));
    }
  }
}

// ---------------------------------------------------------------------------- mbarrier / TMA
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// .release.cta: orders this thread's prior writes (incl. global stores) before the phase
// completion observed by a waiter.
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// arrive + expect `bytes` of asynchronous (TMA) transactions on the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
// .acquire.cta
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cp_async4(unsigned dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst_smem), "l"(src) : "memory");
}
// Arrive on `bar` once all of this thread's prior cp.async copies have landed (counts as one of
// the barrier's expected arrivals: .noinc).
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// TMA gather4: rows r0..r3 (columns [c0, c0 + box)) of the 2-D tensor `map` -> 4 consecutive
// box-sized rows at dst; completion counted in bytes on `bar`.
__device__ __forceinline__ void tma_gather4(unsigned dst, const void* map, int c0, int r0, int r1,
                                            int r2, int r3, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------------- tooling: trace
// Per-CTA timeline (the paper's WG timeline, Fig. wg_profiled).  A record is
// (cta << 40 | event << 32 | payload, %globaltimer ns).  Events: 0 CTA start, 1 chunk start
// (payload = chunk), 2 stage ready, 3 stage released (payload = 1 if it completed a remote
// slice and signalled), 4 consumers done, 5 receive wait done.
__device__ __forceinline__ void trace_ev(const KParams& P, unsigned event, unsigned payload) {
  if (P.trace == nullptr) return;
  const unsigned long long i = atomicAdd(P.trace, 1ull);
  if ((long long)i >= P.trace_cap) return;
  P.trace[2 + 2 * i] = ((unsigned long long)blockIdx.x << 40) |
                       ((unsigned long long)event << 32) | payload;
  P.trace[3 + 2 * i] = globaltimer();
}

__device__ __forceinline__ int warp_bcast(int v, int src = 0) {
  return __shfl_sync(0xffffffffu, v, src);
}

// ------------------------------------------------------------------- LSU gather + pool (a3, a4)
// One bag per group of LPB lanes; lane c of the group owns 16-byte units c, c+LPB, ... (NV of
// them) of every row.  Per batch of U rows: the U row ids (and weights) are read first (shared
// memory if staged, else global), then all U x NV unit loads are issued (predicated, zero-filled
// past the bag's end), then the adds run in bag order.  acc starts at +0.0 and can never become
// -0.0, so adding the +0.0 padding (weight 0 for padded rows) leaves it unchanged: the result is
// the oracle's ascending-order fp32 sum bit for bit.  Weighted: acc = acc + fl(w * x) (R#26).
template <int ELEM, int LPB, int NV, int U, bool SMEM_IDX, bool WEIGHTED>
__device__ __forceinline__ void pool_bag_lsu(const uint4* __restrict__ tab, int DU,
                                             unsigned idx_s, const int* __restrict__ idx_g,
                                             unsigned w_s, const float* __restrict__ w_g,
                                             int lo, int hi, int lane,
                                             float (&acc)[NV][Elem<ELEM>::EPU]) {
  constexpr int EPU = Elem<ELEM>::EPU;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < EPU; ++e) acc[v][e] = 0.f;
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) colok[v] = (lane + v * LPB) < DU;
  for (int k = lo; k < hi; k += U) {
    const int n = hi - k;
    int row[U];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = (u < n) ? k + u : k;     // always a valid id; the load is predicated off
      row[u] = SMEM_IDX ? lds_s32(idx_s + 4u * (unsigned)kk) : __ldg(idx_g + kk);
      if (WEIGHTED) {
        const float w = SMEM_IDX ? lds_f32(w_s + 4u * (unsigned)kk) : __ldg(w_g + kk);
        wt[u] = (u < n) ? w : 0.f;
      }
    }
    uint4 x[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* r = tab + (size_t)(unsigned)row[u] * DU + lane;
#pragma unroll
      for (int v = 0; v < NV; ++v) x[u][v] = ld_unit_pred<(ELEM >= 3)>(r + v * LPB, colok[v] && (u < n));
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        float f[EPU];
        unit_to_f<ELEM>(x[u][v], f);
#pragma unroll
        for (int e = 0; e < EPU; ++e)
          acc[v][e] = WEIGHTED ? __fadd_rn(acc[v][e], __fmul_rn(wt[u], f[e]))
                               : __fadd_rn(acc[v][e], f[e]);
      }
  }
}

// Row-flattened pooling of a contiguous block of bags [b0, b1) of one stage (the LSU path):
// the group walks the block's rows in batches of U that may cross bag boundaries, so short bags
// (pooling factor 1..4) still keep U rows in flight per lane.  A bag's sum is finished -- mean
// division, store to dst0 + b*stride -- the moment its last row has been added, and the
// accumulator restarts from +0.0, so every bag is summed alone and in ascending order (bitwise
// the oracle's result).  Empty bags store +0.0.
template <int ELEM, int LPB, int NV, int U, bool SMEM_IDX, bool WEIGHTED>
__device__ __forceinline__ void pool_run_lsu(const uint4* __restrict__ tab, int DU,
                                             unsigned idx_s, const int* __restrict__ idx_g,
                                             unsigned w_s, const float* __restrict__ w_g,
                                             const int* so, int base, int b0, int b1, int lane,
                                             bool mean, char* dst0, long long stride, int oshift,
                                             int odt) {
  constexpr int EPU = Elem<ELEM>::EPU;
  float acc[NV][EPU];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < EPU; ++e) acc[v][e] = 0.f;
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) colok[v] = (lane + v * LPB) < DU;
  int cb = b0;
  int cstart = so[b0] - base;
  int cend = so[b0 + 1] - base;
  const int lo_all = cstart;
  const int hi_all = so[b1] - base;
  auto finish = [&]() {
    if (mean && cend > cstart) {   // R#27: IEEE binary32 division by the bag length
      const float L = (float)(cend - cstart);
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < EPU; ++e) acc[v][e] = __fdiv_rn(acc[v][e], L);
    }
    char* dst = dst0 + (long long)cb * stride;
#pragma unroll
    for (int v = 0; v < NV; ++v) {                             // a6: zero-copy store
      const int c = lane + v * LPB;
      if (c < DU) {
#pragma unroll
        for (int e = 0; e < EPU; e += 4)
          st_out_e4(dst + ((long long)(EPU * c + e) << oshift), acc[v][e], acc[v][e + 1],
                    acc[v][e + 2], acc[v][e + 3], odt);
      }
#pragma unroll
      for (int e = 0; e < EPU; ++e) acc[v][e] = 0.f;
    }
    ++cb;
    cstart = cend;
    if (cb < b1) cend = so[cb + 1] - base;
  };
  while (cb < b1 && cend == cstart) finish();       // leading empty bags
  for (int k = lo_all; k < hi_all; k += U) {
    const int n = hi_all - k;
    int row[U];
    float wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = (u < n) ? k + u : k;     // always a valid id; the load is predicated off
      row[u] = SMEM_IDX ? lds_s32(idx_s + 4u * (unsigned)kk) : __ldg(idx_g + kk);
      if (WEIGHTED) {
        const float w = SMEM_IDX ? lds_f32(w_s + 4u * (unsigned)kk) : __ldg(w_g + kk);
        wt[u] = (u < n) ? w : 0.f;
      }
    }
    uint4 x[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* r = tab + (size_t)(unsigned)row[u] * DU + lane;
#pragma unroll
      for (int v = 0; v < NV; ++v) x[u][v] = ld_unit_pred<(ELEM >= 3)>(r + v * LPB, colok[v] && (u < n));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < n) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          float f[EPU];
          unit_to_f<ELEM>(x[u][v], f);
#pragma unroll
          for (int e = 0; e < EPU; ++e)
            acc[v][e] = WEIGHTED ? __fadd_rn(acc[v][e], __fmul_rn(wt[u], f[e]))
                                 : __fadd_rn(acc[v][e], f[e]);
        }
        if (k + u + 1 == cend) {
          finish();
          while (cb < b1 && cend == cstart) finish();   // empty bags after it
        }
      }
    }
  }
}

// ------------------------------------------------------------------- smem-stage pool (a4)
// gather4 writes 4 rows x box columns per column block; TMA destinations are 128-B aligned, so a
// block occupies cbstride = round_up(4 * boxbytes, 128) bytes and a 4-row group ncb * cbstride.
__host__ __device__ inline unsigned cb_stride(int box4) { return ((unsigned)box4 * 64u + 127u) & ~127u; }

// Sum stage rows [lo, hi) in order.  Row q's float4 column c lives at
//   rows + (q/4) * gstride + (c / box4) * cbstride + (q%4) * boxbytes + (c % box4) * 16
template <int LPB, int NV>
__device__ __forceinline__ void pool_bag_smem(unsigned rows, int D4, int box4, unsigned gstride,
                                              int lo, int hi, int lane, float (&acc)[NV][4]) {
  unsigned coff[NV];
  bool colok[NV];
  float4 a[NV];
  const unsigned boxbytes = (unsigned)box4 * 16u;
  const unsigned cbs = cb_stride(box4);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int c = lane + v * LPB;
    colok[v] = c < D4;
    const int cb = c / box4;
    coff[v] = (unsigned)cb * cbs + (unsigned)(c - cb * box4) * 16u;
    a[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int q = lo; q < hi; ++q) {
    const unsigned rq = rows + (unsigned)(q >> 2) * gstride + (unsigned)(q & 3) * boxbytes;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (colok[v]) add4(a[v], lds_f4(rq + coff[v]));
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    acc[v][0] = a[v].x; acc[v][1] = a[v].y; acc[v][2] = a[v].z; acc[v][3] = a[v].w;
  }
}

// One pipeline stage: a run of <= C consecutive bags of one chunk whose rows (TMA mode) or
// indices (LSU mode) fit the stage's payload; or a single oversized bag (staged = 0).
struct StageHdr {
  int end;            // 1: no more work (consumers exit)
  int s, t;           // destination rank, local table
  int row0;           // destination-local row of the stage's first bag
  int nb;             // bags in this stage
  int base;           // offsets value of the first bag (indices[base] is the stage's first)
  int staged;         // payload holds this stage's rows / indices
  int flat;           // short bags: row-flattened pooling (average length < flat_below)
  int remote;         // fused, s != r: count the stage's bags toward its slice when consumed
  int slice_id, slice_bags;   // the slice holding row0 and its bag count
  int bs;             // destination block size b_s (a stage may run on into later slices)
  long long j0;       // global sample of the first bag
  char* out_base;     // fused: recv_s[parity]; pool: send (elements of the output type)
  unsigned long long* flag;
};

constexpr int kHdrBytes = 128;   // header area (StageHdr + padding), keeps payloads 128-B aligned
static_assert(sizeof(StageHdr) <= kHdrBytes, "stage header too large");

// ------------------------------------------------------------------------- fused / pool
// FUSED=true: rows a1..a8.  FUSED=false: the baseline's local-staging pool kernel.
// TMA=true: rows gathered by TMA gather4 into the stage.  TMA=false: stage holds indices, rows
// come from per-lane LDGs.
//
// Persistent, warp-specialised CTA (fixed grid <= max occupancy, a task loop over logical
// work in comm-aware order):
//   warp 0 (producer)  CTA c takes chunks c, c + grid, c + 2*grid, ...  All CTAs walk the chunk
//                      list in lock-step, so chunks start in the remote-first, staggered order of
//                      row a1, with no ticket atomics on the latency-critical path.  Per chunk it
//                      stages the CSR offsets (prefetched one chunk ahead in registers) and issues
//                      the row gathers (or index copies) into a ring of NS shared-memory stages.
//                      When the consumers have released a stage of a remote slice it makes their
//                      stores visible system-wide and adds the stage's bags to the slice's counter;
//                      the CTA whose add completes the slice releases the destination's arrival
//                      counter (a7) -- the paper's last-finisher protocol across CTAs.
//   warps 1..C         pool the bags of each stage (a4), store them (a5, a6) and arrive on the
//   (consumers)        stage's empty barrier; no CTA-wide barrier inside the loop, so a fast lane
//                      group moves on to the next stage while slow ones finish ("make forward
//                      progress after setting WG_Done instead of waiting on an inter-WG barrier",
//                      P:151).
// Register budget of the LDG path: 4 CTAs/SM (<= 56 regs) when a lane holds one 16-byte unit per
// row, 3 CTAs/SM (<= 75 regs) when it holds several (wide rows: 16 units in flight per lane
// would spill at 56 registers).  Measured round 1: DLRM-small (NV=1) 16.4 vs 20.2 us with 3;
// DLRM-wide (NV=2) 222 vs 250 us with 4.
#ifndef EMBA2A_LSU_MINB
#define EMBA2A_LSU_MINB(NV) ((NV) >= 2 ? 3 : 4)
#endif
#ifndef EMBA2A_LSU_UNITS
#define EMBA2A_LSU_UNITS 16
#endif
template <int ELEM, int LPB, int NV, bool FUSED, bool TMA, bool WEIGHTED>
__global__ void __launch_bounds__(288, TMA ? 1 : EMBA2A_LSU_MINB(NV))
    emb_a2a_kernel(const __grid_constant__ KParams P) {
  static_assert(!TMA || (ELEM == 0 && !WEIGHTED), "TMA gather: fp32 unweighted tables only");
  constexpr int EPU = Elem<ELEM>::EPU;
  // LSU rows in flight per lane group: ~16 unit loads per lane for the per-bag loop (long bags),
  // ~8 for the row-flattened loop (short bags; more live state per row)
  constexpr int U = TMA ? 8 : (EMBA2A_LSU_UNITS / NV >= 2 ? EMBA2A_LSU_UNITS / NV : 2);
  constexpr int UF = (8 / NV >= 2 ? 8 / NV : 2);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ unsigned long long full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ int last_cta;
  // per-table and per-destination pointers, read once per CTA (no global round trip per stage)
  __shared__ const uint4* s_tab[kMaxSmemTables];
  __shared__ char* s_out[kMaxW];
  __shared__ unsigned long long* s_flag[kMaxW];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane32 = tid & 31;
  const int NS = P.nstages;
  const int nconsumer = blockDim.x - 32;
  const unsigned stage_bytes = (unsigned)P.stage_bytes;
  const unsigned rowbytes = (unsigned)P.DU * 16u;
  auto hdr = [&](int st) { return reinterpret_cast<StageHdr*>(smem_raw + st * stage_bytes); };
  auto soff = [&](int st) {
    return reinterpret_cast<int*>(smem_raw + st * stage_bytes + kHdrBytes);
  };
  // payload (rows or indices), 128-B aligned
  auto payload = [&](int st) {
    return smem_u32(smem_raw) + st * stage_bytes + (unsigned)P.payload_off;
  };

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      // TMA: 32 producer arrivals (+ transaction bytes); LSU: 32 arrivals + 32 cp.async arrivals
      mbar_init(&full_bar[i], TMA ? 32u : 64u);
      mbar_init(&empty_bar[i], (unsigned)nconsumer);
    }
  }
  // Buffer-reuse credit: this forward has started, so everything the caller
  // ordered before it -- the consumer of our output epoch - 2, which lives in the receive half
  // the peers are about to overwrite -- is complete.  One add per peer, before any waiting.
  if (FUSED && P.W > 1 && blockIdx.x == 0 && tid < P.W && tid != P.r)
    red_release_sys_add(P.peers->credit_out[tid], 1ull);
  for (int i = tid; i < P.T && i < kMaxSmemTables; i += blockDim.x)
    s_tab[i] = reinterpret_cast<const uint4*>(P.tables[i]);
  for (int i = tid; i < P.W; i += blockDim.x) {
    if (FUSED) {
      s_out[i] = reinterpret_cast<char*>(P.peers->recv[i][P.parity]);
      s_flag[i] = P.peers->flag_out[i];
    } else {
      s_out[i] = reinterpret_cast<char*>(P.send);
      s_flag[i] = nullptr;
    }
  }
  __syncthreads();
  // Programmatic dependent launch: everything that reads table rows, counters or buffers a
  // predecessor on the stream may write waits for it (griddepcontrol.wait; a no-op without a
  // programmatic predecessor).  The producer's first reads -- the first chunk's CSR offsets and
  // the first stage's index copy -- touch only the caller's inputs, which no kernel of this
  // library writes (and a caller kernel that does is not a programmatic predecessor: it has
  // completed before this grid launched), so in the LSU mode they go ahead of the wait and
  // overlap the predecessor's drain.

  if (warp == 0) {
    // ===================================================================== producer
    bool waited = !P.pdl;
    // Programmatic dependent launch: the next kernel on the stream may start its CTAs (launch
    // ramp, prologue, the work before its own wait) once every CTA of ours has triggered.  We
    // trigger only after OUR wait has returned, i.e. once our predecessor is complete: a kernel
    // that triggered at entry would let its successor's pre-wait work (rows gathered early, a
    // stage stored early) overlap its PREDECESSOR -- forward e+2 storing into the receive half
    // forward e is still writing, or reading table rows a backward is still updating.
    // (Not when a peer shares this GPU: a rank running ahead would park the waiting CTAs of its
    // next forwards on SM slots a slower peer's forward needs; exiting triggers it then.)
    auto pdl_wait_once = [&]() {
      if (!waited) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
        if (P.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      }
    };
    if (TMA) pdl_wait_once();            // the producer gathers table rows itself
    if (lane32 == 0) trace_ev(P, 0, 0);
    int u = 0;   // stage uses so far
    // wait until consumers released use v; for a remote slice, publish its bags (a7)
    auto recycle = [&](int v) {
      const int st = v % NS;
      mbar_wait(&empty_bar[st], (unsigned)((v / NS) & 1));
      unsigned signalled = 0;
      if (FUSED && lane32 == 0) {
        const StageHdr* h = hdr(st);
        if (h->remote) {
          // every consumer store of this stage happens-before this point (mbarrier
          // release/acquire); make them visible system-wide before counting them (R#25)
          fence_acq_rel_sys();
          // the stage's bags [row0, row0 + nb) count toward each slice they fall in (a chunk
          // may be longer than a slice: chunks are work units, slices signal units)
          int row = h->row0, left = h->nb, sid = h->slice_id, sbags = h->slice_bags;
          while (left > 0) {
            const int in_slice = P.S - row % P.S;
            const int take = left < in_slice ? left : in_slice;
            const unsigned long long old =
                atom_add_acqrel_gpu(P.slice_cnt + sid, (unsigned long long)take);
            if (old + (unsigned long long)take == P.epoch * (unsigned long long)sbags &&
                h->s != P.skip_to) {
              if (P.delay_ns > 0) {
                const unsigned long long t0 = globaltimer();
                while (globaltimer() - t0 < (unsigned long long)P.delay_ns) __nanosleep(1000);
              }
              red_release_sys_add(h->flag, 1ull);   // P:151 PUT -> fence -> sliceRdy
              ++signalled;
            }
            row += take;
            left -= take;
            ++sid;
            sbags = (h->bs - row) < P.S ? h->bs - row : P.S;
          }
        }
      }
      if (lane32 == 0) trace_ev(P, 3, signalled);
      __syncwarp();
    };
    // Credit check (a6 precondition): before the first stage of ours that stores into peer s is
    // published, s must have started its forward epoch - credit_lag.  Chunks
    // come destination by destination, so a producer checks each destination once.
    int cred_ok = -1;
    auto await_credit = [&](int s) {
      if (lane32 == 0) {
        const unsigned long long target = P.epoch - (unsigned long long)P.credit_lag;
        const unsigned long long* f = P.credits_in + (size_t)s * kFlagStride;
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(f) < target) {
          if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
            atomicExch(P.err, 0x1000 | s);
            break;
          }
          __nanosleep(64);
        }
      }
      __syncwarp();
      cred_ok = s;
    };
    int ticket = (int)blockIdx.x;
    int k, s, t, i0, nb;
    // chunk offsets (C <= 127 bags): lane q holds off[q], off[32 + q], off[64 + q], off[96 + q]
    int o0 = 0, o1 = 0, o2 = 0, o3 = 0;
    auto load_offsets = [&](int tk, int& kk, int& ss, int& tt, int& ii, int& nn, int& a,
                            int& b2, int& c2, int& d2) {
      decode_unit(P, tk, P.C, P.chunk_base, kk, ss, tt, ii, nn);
      const int* offg = P.offsets + (long long)tt * P.B + P.part[ss] + ii;
      if (lane32 <= nn) a = __ldg(offg + lane32);
      if (32 + lane32 <= nn) b2 = __ldg(offg + 32 + lane32);
      if (64 + lane32 <= nn) c2 = __ldg(offg + 64 + lane32);
      if (96 + lane32 <= nn) d2 = __ldg(offg + 96 + lane32);
    };
    auto off_at = [&](int e) {
      return warp_bcast(e < 64 ? (e < 32 ? o0 : o1) : (e < 96 ? o2 : o3), e & 31);
    };
    if (ticket < P.nchunks) load_offsets(ticket, k, s, t, i0, nb, o0, o1, o2, o3);
    while (ticket < P.nchunks) {
      const int tk_next = ticket + (int)gridDim.x;
      int k2 = 0, s2 = 0, t2 = 0, i02 = 0, nb2 = 0, p0 = 0, p1 = 0, p2 = 0, p3 = 0;
      if (tk_next < P.nchunks) load_offsets(tk_next, k2, s2, t2, i02, nb2, p0, p1, p2, p3);
      if (lane32 == 0) trace_ev(P, 1, (unsigned)ticket);
      const long long j0 = P.part[s] + i0;
      for (int cb = 0; cb < nb;) {    // usually one stage per chunk
        const int st = u % NS;
        if (u >= NS) recycle(u - NS);
        int* so = soff(st);
        int n = nb - cb;
        const int base = off_at(cb);
        int cnt = off_at(nb) - base;
        int staged = 1;
        if (cnt > P.payload_cap) {   // shrink the run to what fits; a lone huge bag -> LSU
          int m = 0;
          for (int q = 1; q <= n; ++q)
            if (off_at(cb + q) - base <= P.payload_cap) m = q;
          if (m == 0) { m = 1; staged = 0; }
          n = m;
          cnt = off_at(cb + n) - base;
        }
        // stage-local offsets
        if (lane32 >= cb && lane32 <= cb + n) so[lane32 - cb] = o0;
        if (32 + lane32 >= cb && 32 + lane32 <= cb + n) so[32 + lane32 - cb] = o1;
        if (64 + lane32 >= cb && 64 + lane32 <= cb + n) so[64 + lane32 - cb] = o2;
        if (96 + lane32 >= cb && 96 + lane32 <= cb + n) so[96 + lane32 - cb] = o3;
        int slice_id = 0, slice_bags = 0;
        if (FUSED) slice_of_chunk(P, k, s, t, i0 + cb, slice_id, slice_bags);
        if (lane32 == 0) {
          StageHdr* h = hdr(st);
          h->end = 0; h->s = s; h->t = t; h->row0 = i0 + cb; h->nb = n; h->base = base;
          h->staged = staged; h->j0 = j0 + cb;
          h->flat = cnt < P.flat_below * n ? 1 : 0;
          h->remote = (FUSED && s != P.r) ? 1 : 0;
          h->slice_id = slice_id;
          h->slice_bags = slice_bags;
          h->bs = (int)(P.part[s + 1] - P.part[s]);
          h->out_base = s_out[s];
          h->flag = s_flag[s];
        }
        __syncwarp();
        if (FUSED && s != P.r && s != cred_ok) await_credit(s);
        const int* ig = P.indices + base;
        if (TMA) {
          // a3: gather4 groups of rows; rows past cnt (padding to a multiple of 4) read row 0
          const int groups = staged ? (cnt + 3) >> 2 : 0;
          if (lane32 == 0)   // bytes actually moved: 4 rows x box per column block
            mbar_arrive_expect_tx(&full_bar[st], (unsigned)groups * 4u * rowbytes);
          else
            mbar_arrive(&full_bar[st]);
          const void* map = P.tmaps + t;
          const unsigned dst0 = payload(st);
          const unsigned cbs = cb_stride(P.box4);
          for (int g = lane32; g < groups; g += 32) {
            const int q = 4 * g;
            const int r0 = __ldg(ig + q);
            const int r1 = q + 1 < cnt ? __ldg(ig + q + 1) : 0;
            const int r2 = q + 2 < cnt ? __ldg(ig + q + 2) : 0;
            const int r3 = q + 3 < cnt ? __ldg(ig + q + 3) : 0;
            const unsigned dst = dst0 + (unsigned)g * (unsigned)P.ncb * cbs;
            for (int c = 0; c < P.ncb; ++c)
              tma_gather4(dst + (unsigned)c * cbs, map, c * P.box4 * 4, r0, r1, r2, r3,
                          &full_bar[st]);
          }
        } else {
          if (staged) {   // asynchronous, coalesced index copy; completion on full_bar[st]
            const unsigned si = payload(st);
            for (int q = lane32; q < cnt; q += 32) cp_async4(si + 4u * (unsigned)q, ig + q);
            if (WEIGHTED) {   // per-sample weights ride along, right after the indices
              const float* wg = P.weights + base;
              const unsigned sw = si + 4u * (unsigned)P.payload_cap;
              for (int q = lane32; q < cnt; q += 32) cp_async4(sw + 4u * (unsigned)q, wg + q);
            }
          }
          mbar_arrive(&full_bar[st]);
          cp_async_mbar_arrive(&full_bar[st]);
        }
        pdl_wait_once();                 // before any recycle (counters) or a next stage
        if (lane32 == 0) trace_ev(P, 2, (unsigned)u);
        cb += n;
        ++u;
      }
      ticket = tk_next;
      k = k2; s = s2; t = t2; i0 = i02; nb = nb2; o0 = p0; o1 = p1; o2 = p2; o3 = p3;
    }
    // end marker, then drain: every outstanding stage is consumed and published
    pdl_wait_once();
    {
      const int st = u % NS;
      if (u >= NS) recycle(u - NS);
      if (lane32 == 0) hdr(st)->end = 1;
      __syncwarp();
      mbar_arrive(&full_bar[st]);
      if (!TMA) cp_async_mbar_arrive(&full_bar[st]);
      for (int v = (u - NS + 1 > 0 ? u - NS + 1 : 0); v < u; ++v) recycle(v);
    }
  } else {
    // ===================================================================== consumers
    // table rows and receive-buffer stores: wait for the predecessor unless the host found it
    // harmless (one rank, no backward of this handle since its previous forward; option
    // "pdl_rows_early"); the counters are the producer's, and it always waits
    if (P.pdl && P.rows_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ctid = tid - 32;
    const int lane = ctid % LPB;
    const int group = ctid / LPB;
    const int ngroups = nconsumer / LPB;
    const int D = P.D;
    for (int u = 0;; ++u) {
      const int st = u % NS;
      mbar_wait(&full_bar[st], (unsigned)((u / NS) & 1));
      const StageHdr* h = hdr(st);
      if (h->end) break;
      const int nb = h->nb, base = h->base, t = h->t;
      const int* so = soff(st);
      const bool staged = h->staged;
      const unsigned pay = payload(st);
      const unsigned wpay = pay + 4u * (unsigned)P.payload_cap;
      const uint4* tab = t < kMaxSmemTables ? s_tab[t]
                                            : reinterpret_cast<const uint4*>(P.tables[t]);
      // a5: bag b of this stage goes to row (row0 + b) of s's [b_s][G*D], column block
      // g = toff + t (fused), or to staging row (j0 + b), table t (pool)
      // (byte addresses: the output element is 4 or 2 bytes, P.oshift)
      const int osh = P.oshift, odt = P.out_dtype;
      char* dst0;
      long long stride;
      if (FUSED) {
        dst0 = h->out_base + ((((long long)h->row0 * P.G + (P.toff + t)) * D) << osh);
        stride = ((long long)P.G * D) << osh;
      } else {
        dst0 = h->out_base + (((h->j0 * P.T + t) * (long long)D) << osh);
        stride = ((long long)P.T * D) << osh;
      }
      if (TMA && staged) {
        for (int b = group; b < nb; b += ngroups) {
          float acc[NV][EPU];
          const int lo = so[b] - base, hi = so[b + 1] - base;
          if constexpr (TMA)
            pool_bag_smem<LPB, NV>(pay, P.DU, P.box4, (unsigned)P.ncb * cb_stride(P.box4), lo,
                                   hi, lane, acc);
          if (P.mean && hi > lo) {   // R#27: IEEE binary32 division by the bag length
            const float L = (float)(hi - lo);
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int e = 0; e < EPU; ++e) acc[v][e] = __fdiv_rn(acc[v][e], L);
          }
          char* dst = dst0 + (long long)b * stride;
#pragma unroll
          for (int v = 0; v < NV; ++v) {                         // a6: zero-copy store
            const int c = lane + v * LPB;
            if (c < P.DU) {
#pragma unroll
              for (int e = 0; e < EPU; e += 4)
                st_out_e4(dst + ((long long)(EPU * c + e) << osh), acc[v][e], acc[v][e + 1],
                          acc[v][e + 2], acc[v][e + 3], odt);
            }
          }
        }
      } else if (h->flat) {
        // short bags: contiguous block of bags per lane group, rows walked across bag
        // boundaries so U rows stay in flight
        const int q = nb / ngroups, rmd = nb - q * ngroups;
        const int b0 = group * q + (group < rmd ? group : rmd);
        const int b1 = b0 + q + (group < rmd ? 1 : 0);
        if (b0 < b1) {
          if (staged)
            pool_run_lsu<ELEM, LPB, NV, UF, true, WEIGHTED>(tab, P.DU, pay, nullptr, wpay, nullptr,
                                                            so, base, b0, b1, lane, P.mean != 0,
                                                            dst0, stride, osh, odt);
          else
            pool_run_lsu<ELEM, LPB, NV, UF, false, WEIGHTED>(
                tab, P.DU, 0u, P.indices + base, 0u, WEIGHTED ? P.weights + base : nullptr, so,
                base, b0, b1, lane, P.mean != 0, dst0, stride, osh, odt);
        }
      } else {
        // long bags: one bag per lane group at a time, round robin, U rows in flight
        for (int b = group; b < nb; b += ngroups) {
          float acc[NV][EPU];
          const int lo = so[b] - base, hi = so[b + 1] - base;
          if (staged)
            pool_bag_lsu<ELEM, LPB, NV, U, true, WEIGHTED>(tab, P.DU, pay, nullptr, wpay,
                                                           nullptr, lo, hi, lane, acc);
          else
            pool_bag_lsu<ELEM, LPB, NV, U, false, WEIGHTED>(
                tab, P.DU, 0u, P.indices + base, 0u, WEIGHTED ? P.weights + base : nullptr, lo,
                hi, lane, acc);
          if (P.mean && hi > lo) {   // R#27: IEEE binary32 division by the bag length
            const float L = (float)(hi - lo);
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
              for (int e = 0; e < EPU; ++e) acc[v][e] = __fdiv_rn(acc[v][e], L);
          }
          char* dst = dst0 + (long long)b * stride;
#pragma unroll
          for (int v = 0; v < NV; ++v) {                         // a6: zero-copy store
            const int c = lane + v * LPB;
            if (c < P.DU) {
#pragma unroll
              for (int e = 0; e < EPU; e += 4)
                st_out_e4(dst + ((long long)(EPU * c + e) << osh), acc[v][e], acc[v][e + 1],
                          acc[v][e + 2], acc[v][e + 3], odt);
            }
          }
        }
      }
      mbar_arrive(&empty_bar[st]);
    }
    if (ctid == 0) trace_ev(P, 4, 0);
  }

  // last-finisher detection over CTAs (the WG_Done role): the atomic's return value
  // decides (R#18).  The last CTA resets the done counter for the next launch.  Only needed when
  // there is a receive wait (fused, W > 1).
  if (!FUSED || P.W == 1) return;
  __syncthreads();
  if (tid == 0) {
    const unsigned int prev = atomicAdd(P.done, 1u);
    last_cta = (prev == (unsigned int)gridDim.x - 1u);
    if (last_cta) *P.done = 0u;
  }
  __syncthreads();
  if constexpr (FUSED) {
    if (P.W == 1 || !last_cta) return;
    // a8: receive-side completion wait, one thread per source rank
    for (int src = tid; src < P.W; src += blockDim.x) {
      if (src == P.r) continue;
      const unsigned long long target = P.epoch * (unsigned long long)P.peers->n_in[src];
      const unsigned long long* f = P.flags_in + (size_t)src * kFlagStride;
      const unsigned long long t0 = globaltimer();
      unsigned int backoff = 32;
      while (ld_acquire_sys(f) < target) {
        if (globaltimer() - t0 > (unsigned long long)P.timeout_ns) {
          atomicExch(P.err, 0x100 | src);   // surfaces as EMB_A2A_ETIMEOUT on the next call
          break;
        }
        __nanosleep(backoff);
        if (backoff < 1024) backoff <<= 1;
      }
    }
    if (tid == 0) trace_ev(P, 5, 0);
  }
}

// ------------------------------------------------------------------------- dispatch
typedef void (*KernelFn)(const KParams);

template <int ELEM, int LPB, int NV, bool FUSED, bool WEIGHTED>
KernelFn pick_mode(bool tma) {
  if constexpr (ELEM == 0 && !WEIGHTED) {
    if (tma) return emb_a2a_kernel<ELEM, LPB, NV, FUSED, true, WEIGHTED>;
  }
  return emb_a2a_kernel<ELEM, LPB, NV, FUSED, false, WEIGHTED>;
}

// units (16 B) per lane NV (1, 2, 4, 8; 0 = auto: 1 up to 32 units per row, else
// ceil(DU/32)); lanes per bag LPB = next_pow2(ceil(DU / NV)) <= 32.  Fewer lanes per bag = more
// bags in flight per warp.
inline int choose_nv(int DU, int want, int max_nv) {
  int nv = want > 0 ? want : (DU + 31) / 32;
  if (nv <= 1) nv = 1;
  else if (nv <= 2) nv = 2;
  else if (nv <= 4) nv = 4;
  else nv = 8;
  while (nv < max_nv && (DU + nv - 1) / nv > 32) nv <<= 1;   // LPB <= 32 must cover the row
  return nv > max_nv ? max_nv : nv;
}

template <int ELEM, int NV, bool FUSED, bool WEIGHTED>
KernelFn pick_lpb(int DU, bool tma) {
  const int per = (DU + NV - 1) / NV;
  int lpb = 1;
  while (lpb < per && lpb < 32) lpb <<= 1;
  switch (lpb) {
    case 1: return pick_mode<ELEM, 1, NV, FUSED, WEIGHTED>(tma);
    case 2: return pick_mode<ELEM, 2, NV, FUSED, WEIGHTED>(tma);
    case 4: return pick_mode<ELEM, 4, NV, FUSED, WEIGHTED>(tma);
    case 8: return pick_mode<ELEM, 8, NV, FUSED, WEIGHTED>(tma);
    case 16: return pick_mode<ELEM, 16, NV, FUSED, WEIGHTED>(tma);
    default: return pick_mode<ELEM, 32, NV, FUSED, WEIGHTED>(tma);
  }
}

// fp32 tables: NV in {1,2,4,8} (D <= 1024); 16-bit tables: NV in {1,2,4} (8 elements per unit)
template <int ELEM, bool FUSED, bool WEIGHTED>
KernelFn pick(int DU, int nv_want, bool tma) {
  constexpr int kMaxNV = (ELEM == 0 || ELEM == 3) ? 8 : 4;
  switch (choose_nv(DU, nv_want, kMaxNV)) {
    case 1: return pick_lpb<ELEM, 1, FUSED, WEIGHTED>(DU, tma);
    case 2: return pick_lpb<ELEM, 2, FUSED, WEIGHTED>(DU, tma);
    case 4: return pick_lpb<ELEM, 4, FUSED, WEIGHTED>(DU, tma);
    default:
      if constexpr (kMaxNV == 8) return pick_lpb<ELEM, 8, FUSED, WEIGHTED>(DU, tma);
      return pick_lpb<ELEM, 4, FUSED, WEIGHTED>(DU, tma);
  }
}

template <int ELEM, bool WEIGHTED>
cudaError_t plan_elem(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl) {
  const bool tma = ELEM == 0 && !WEIGHTED && P.tma != 0;
  KernelFn fn = fused ? pick<ELEM, true, WEIGHTED>(P.DU, c.vec, tma)
                      : pick<ELEM, false, WEIGHTED>(P.DU, c.vec, tma);
  return plan_with(reinterpret_cast<const void*>(fn), P, c, pl);
}

}  // namespace
}  // namespace emba2a
