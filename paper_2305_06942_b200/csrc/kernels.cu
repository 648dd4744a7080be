// kernels.cu -- tooling kernels (device barrier, slice-plan decode, validation), the launch path
// and the stage layout of libemba2a.so.  The fused / pool kernel template lives in
// fused_kernel.cuh; its instances are compiled in inst_*.cu.
#include "fused_kernel.cuh"

namespace emba2a {
namespace {

// Cross-rank device barrier (bench tooling, not the hot path): every rank adds 1 to each peer's
// barrier counter with release semantics, then waits for W-1 arrivals on its own counter.  Lets
// all ranks' timed regions start within the fabric round trip instead of host launch jitter.
__global__ void barrier_kernel(const DevPeers* __restrict__ peers, unsigned long long* own, int W,
                               int r, unsigned long long target, long long timeout_ns, int* err) {
  const int q = threadIdx.x;
  if (q < W && q != r) red_release_sys_add(peers->barrier_out[q], 1ull);
  if (q == 0) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(own) < target) {
      if (globaltimer() - t0 > (unsigned long long)timeout_ns) {
        atomicExch(err, 0x200);
        break;
      }
      __nanosleep(64);
    }
  }
}

// NVLink store probe (bench tooling, not the hot path): every CTA streams 16-byte st.global.v4
// stores -- the fused kernel's store instruction -- into the receive regions of all peers at
// once, 512-byte runs per warp, consecutive warps on different peers (staggered like row a1).
// Measures what SM-issued peer stores sustain with every rank sending to every peer.
__global__ void __launch_bounds__(256) peer_store_probe_kernel(const DevPeers* __restrict__ peers,
                                                               int W, int r, long long runs) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long total = runs * (W - 1);
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (long long c = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < total;
       c += nwarps) {
    const int k = (int)(c % (W - 1));
    const long long run = c / (W - 1);
    const int q = (r + 1 + k) % W;
    float* dst = peers->recv[q][0] + run * 128 + lane * 4;
    st_out4(dst, v);
  }
}

__global__ void slice_plan_kernel(const __grid_constant__ KParams P, int* out) {
  const int ticket = blockIdx.x * blockDim.x + threadIdx.x;
  if (ticket >= P.nslices) return;   // slice-level decode (the signal units)
  int s, t, i0, nb;
  decode_slice(P, ticket, s, t, i0, nb);
  out[4 * ticket + 0] = s;
  out[4 * ticket + 1] = t;
  out[4 * ticket + 2] = i0;
  out[4 * ticket + 3] = nb;
}

// Validate mode: offsets[0] = 0, non-decreasing, offsets[TB] = nnz, 0 <= idx < rows[t].
__global__ void validate_kernel(const int* __restrict__ indices, const int* __restrict__ offsets,
                                long long nnz, long long TB, long long B,
                                const long long* __restrict__ rows, int* err) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q < TB) {
    const int lo = offsets[q], hi = offsets[q + 1];
    if (hi < lo || lo < 0 || (long long)hi > nnz) { atomicExch(err, 1); return; }
    const long long rmax = rows[q / B];
    for (int k = lo; k < hi; ++k) {
      const int v = indices[k];
      if (v < 0 || (long long)v >= rmax) { atomicExch(err, 2); return; }
    }
  }
  if (q == 0 && (offsets[0] != 0 || (long long)offsets[TB] != nnz)) atomicExch(err, 1);
}

}  // namespace

// Resolve shared memory, pipeline depth and the persistent grid for kernel instance `fn` once;
// the result is cached by the host per handle (no occupancy query on the per-forward path).
cudaError_t plan_with(const void* fn, const KParams& P, const LaunchCfg& c, LaunchPlan* pl) {
  cudaGetLastError();   // never report someone else's stale error as ours
  // pipeline depth: as requested, but never more than fits the 227 KB per-CTA limit (>= 2)
  int ns = P.nstages;
  while (ns > 2 && (size_t)P.stage_bytes * ns > 227 * 1024) --ns;
  const size_t smem = (size_t)P.stage_bytes * ns;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;   // even 2 stages do not fit
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
  }
  const int threads = c.threads + 32;      // consumers + one producer warp
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  if (c.ctas_per_sm > 0 && c.ctas_per_sm < occ) occ = c.ctas_per_sm;
  long long grid = (long long)sms * occ;
  const long long want = P.nchunks > 0 ? P.nchunks : 1;
  if (grid > want) grid = want;
  pl->fn = fn;
  pl->grid = (unsigned)grid;
  pl->threads = threads;
  pl->smem = smem;
  pl->nstages = ns;
  return cudaSuccess;
}

static cudaError_t plan_any(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl) {
  const bool weighted = P.weights != nullptr;
  switch (P.elem) {
    case 0:
      if (weighted) return plan_f32w(P, c, fused, pl);
      return (P.l1rows && !P.tma) ? plan_f32l1(P, c, fused, pl) : plan_f32(P, c, fused, pl);
    case 1:
      return (P.l1rows && !weighted) ? plan_bf16l1(P, c, fused, pl)
                                     : plan_bf16(P, c, fused, weighted, pl);
    case 2:
      return (P.l1rows && !weighted) ? plan_f16l1(P, c, fused, pl)
                                     : plan_f16(P, c, fused, weighted, pl);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t plan_fused(const KParams& P, const LaunchCfg& c, LaunchPlan* pl) {
  return plan_any(P, c, true, pl);
}

cudaError_t plan_pool_local(const KParams& P, const LaunchCfg& c, LaunchPlan* pl) {
  return plan_any(P, c, false, pl);
}

cudaError_t launch_planned(const LaunchPlan& pl, KParams P, cudaStream_t st) {
  P.nstages = pl.nstages;
  void* args[] = {&P};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(pl.threads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, pl.fn, args);
}

cudaError_t launch_barrier(const DevPeers* peers, unsigned long long* own_counter, int W, int r,
                           unsigned long long target, long long timeout_ns, int* err,
                           cudaStream_t st) {
  barrier_kernel<<<1, ((W + 31) / 32) * 32, 0, st>>>(peers, own_counter, W, r, target, timeout_ns,
                                                     err);
  return cudaGetLastError();
}

cudaError_t launch_peer_store_probe(const DevPeers* peers, int W, int r, long long runs,
                                    cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  peer_store_probe_kernel<<<sms * 4, 256, 0, st>>>(peers, W, r, runs);
  return cudaGetLastError();
}

cudaError_t launch_slice_plan(const KParams& P, int* out, cudaStream_t st) {
  if (P.nslices == 0) return cudaSuccess;
  slice_plan_kernel<<<(P.nslices + 255) / 256, 256, 0, st>>>(P, out);
  return cudaGetLastError();
}

cudaError_t launch_validate(const int* indices, const int* offsets, long long nnz, long long TB,
                            long long B, int T, const long long* rows_dev, int* err_dev,
                            cudaStream_t st) {
  (void)T;
  const long long blocks = (TB + 255) / 256;
  validate_kernel<<<(unsigned)(blocks > 0 ? blocks : 1), 256, 0, st>>>(indices, offsets, nnz, TB,
                                                                        B, rows_dev, err_dev);
  return cudaGetLastError();
}

// Stage layout: [header 128 B | offsets (C+1) ints, padded to 128 B | payload].
// TMA: payload = payload_cap rows (a multiple of 4) of D floats, from `kb` KiB; LSU: payload =
// idx_cap indices (+ idx_cap per-sample weights when weighted).
void stage_layout(KParams& P, int kb, int idx_cap) {
  const int off_bytes = ((P.C + 1) * 4 + 127) / 128 * 128;
  P.payload_off = kHdrBytes + off_bytes;
  int payload;
  if (P.tma) {
    const int gbytes = P.ncb * (int)cb_stride(P.box4);   // one 4-row gather group
    int groups = kb * 1024 / gbytes;
    if (groups < 1) groups = 1;
    P.payload_cap = groups * 4;
    payload = groups * gbytes;
  } else {
    // weighted: indices and weights share the same payload bytes (half the entries each), so
    // the stage -- and the CTAs per SM -- stay the same size
    P.payload_cap = P.weights ? (idx_cap + 1) / 2 : idx_cap;
    payload = (idx_cap * 4 + 127) / 128 * 128 + (P.weights ? 128 : 0);
  }
  P.stage_bytes = P.payload_off + payload;
}

}  // namespace emba2a
