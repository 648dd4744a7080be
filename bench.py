"""Benchmark: fused EmbeddingBag(sum) + All-to-All on B200 vs the unfused pool + NCCL baseline.

Metric (BASELINE.json): "fused emb+All-to-All us & lookups/s at 1/2/4/8 B200 vs unfused
emb+NCCL".  One step = one fused forward (rows a1-a8: pool this rank's tables for the whole
global batch, zero-copy store to every destination, signal, receive wait) over one batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dlrm_small] [--impl fused|reference]

N=1 runs the config's per-rank work at W=1; under torchrun each rank
owns one GPU and the config runs at W=N (W-scaling rule: T_r, rows, D, B, pooling fixed).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0      # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json absent)
NVLINK_GBS = 770.0             # measured peer copy per direction (B200_PROFILING.md); 900 nominal
L2_FLUSH_BYTES = 512 << 20     # > 126 MB L2
METRIC = "fused emb+All-to-All lookups/s (us/step in ms_per_step)"   # both arms


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="dlrm_small")
    ap.add_argument("--impl", default="fused", choices=["fused", "reference"])
    ap.add_argument("--alpha", type=float, default=1.05)
    ap.add_argument("--slice", type=int, default=0, help="slice size S (0 = library default)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--vec", type=int, default=0)
    ap.add_argument("--opt", action="append", default=[],
                    help="key=value library option for the fused op's handle (repeatable)")
    ap.add_argument("--order", type=int, default=-1)
    ap.add_argument("--ctas-per-sm", type=int, default=0, help="persistent grid per SM (E3)")
    ap.add_argument("--skew-us", type=float, default=0.0,
                    help="E5: the last rank sleeps this long on the GPU before each forward")
    ap.add_argument("--batches", type=int, default=16,
                    help="distinct pre-generated batches rotated through the timed steps")
    ap.add_argument("--timing", default="b2b", choices=["b2b", "flushed"],
                    help="b2b: K back-to-back steps between one event pair, rotating batches whose "
                         "working set exceeds L2; flushed: L2 flush + per-step events")
    ap.add_argument("--no-baseline", action="store_true", help="skip the unfused NCCL baseline")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle timing")
    ap.add_argument("--no-backward", action="store_true", help="skip the f3 backward timing")
    ap.add_argument("--table-dtype", default="f32", choices=["f32", "bf16", "f16"],
                    help="table element type (f2; fp32 accumulation and output either way)")
    ap.add_argument("--pooling", default="sum", choices=["sum", "mean"], help="f2: mean pooling")
    ap.add_argument("--out-dtype", default="f32", choices=["f32", "bf16", "f16"],
                    help="f2: output element type (fp32 sum rounded once, R#32; halves TX bytes)")
    ap.add_argument("--weighted", action="store_true", help="f2: per-sample weights")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-alpha0", action="store_true",
                    help="skip the alpha = 0 (uniform, cold-cache) control leg")
    ap.add_argument("--alpha0-batches", type=int, default=4)
    ap.add_argument("--out", default="", help="also append the JSON line to this file")
    ap.add_argument("--path", default="emb_a2a", choices=["emb_a2a", "ag_gemm"],
                    help="emb_a2a: the north-star fused embedding + All-to-All (default); "
                         "ag_gemm: SURVEY Sec 8 row f4, the fused AllGather + GEMM (P:180)")
    ap.add_argument("--ag-config", default="ag_ffn", help="ag_gemm workload (synth/gemm_gen.py)")
    ap.add_argument("--ag-order", type=int, default=-1, help="ag_gemm tile order (0 comm-aware, 1 ascending)")
    ap.add_argument("--ag-grid", type=int, default=0, help="ag_gemm persistent CTAs (0 = auto)")
    ap.add_argument("--ag-leg", type=int, default=1,
                    help="add the f4 AllGather+GEMM measurement to the main line as 'ag_gemm' "
                         "(1 = at every N, default; -1 = only at N=1; 0 = never)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg):
    kind, p = cfg.pool
    pool = f"L={p}" if kind == "fixed" else f"L~U{{1..{2 * p - 1}}}"
    return (f"{cfg.name} at W={cfg.W}: {cfg.T[0]} tables/rank x {cfg.R} rows x D={cfg.D}, "
            f"global batch {cfg.B}, {pool}, Zipf alpha={cfg.alpha}, fp32")


def algorithmic_bytes(cfg, r, nnz, esize=4, weighted=False, oes=4):
    """Per-rank algorithmic bytes of one forward: gathered rows (esize bytes
    per element) + indices (+ weights) + offsets + this rank's receive buffer; and the bytes it
    must send over NVLink."""
    b = int(cfg.part[r + 1] - cfg.part[r])
    T = cfg.T[r]
    hbm = nnz * cfg.D * esize + nnz * (8 if weighted else 4) + (T * cfg.B + 1) * 4 + \
        b * cfg.G * cfg.D * oes
    tx = (cfg.B - b) * T * cfg.D * oes
    return hbm, tx


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every ~2 ms during the timed region
    (the kernels are microseconds long, so nvidia-smi's >= 50 ms period would see nothing)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:      # no NVML: report that instead of inventing clocks
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self.t.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class NvlinkCounters:
    """This GPU's NVLink data-TX byte counter through NVML field values (summed over links) --
    the non-profiler evidence of NVLink traffic (ncu cannot wrap the multi-rank run: its
    serialised replay deadlocks the receive wait).  None where NVML has no such counter."""

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.ok = self.read() is not None
        except Exception:
            self.ok = False

    def read(self):
        try:
            nv = self.nv
            fid = nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX
            vals = nv.nvmlDeviceGetFieldValues(self.h, [(fid, link) for link in range(18)])
            tot, seen = 0, False
            for v in vals:
                if getattr(v, "nvmlReturn", 1) == 0:
                    tot += int(v.value.ullVal)
                    seen = True
            return tot * 1024 if seen else None
        except Exception:
            return None


# ---------------------------------------------------------------------------- oracle timing

def host_cpu():
    """The host's CPU model and logical core count (stated beside every oracle timing)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cpu": model, "host_cpu_count": os.cpu_count()}


def oracle_rows_pass(cfg, csr, s, rows=None, weights=None, pooling="sum"):
    """The oracle as it stands (single-threaded C, procedural tables): rank s's output rows
    (all b_s of them, or `rows`), computed from every rank's CSR.  Returns (lookups, seconds)."""
    import oracle
    idx = [c[0] for c in csr]
    off = [c[1] for c in csr]
    b = int(cfg.part[s + 1] - cfg.part[s])
    sel = np.arange(b) if rows is None else np.asarray(rows, np.int64)
    t0 = time.perf_counter()
    oracle.emb_a2a_rows(cfg.table_seed, cfg.value_mode, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                        idx, off, s, sel, check_inputs=False, weights=weights,
                        pooling=oracle.MEAN if pooling == "mean" else oracle.SUM)
    secs = time.perf_counter() - t0
    lookups = 0
    js = cfg.part[s] + sel
    for r in range(cfg.W):
        o = off[r].astype(np.int64)
        for t in range(cfg.T[r]):
            lookups += int((o[t * cfg.B + js + 1] - o[t * cfg.B + js]).sum())
    return lookups, secs


def oracle_pass(cfg, csr, rows_per_call=None):
    """Every destination's rows (the whole forward of all W ranks): the reference arm."""
    lookups, secs = 0, 0.0
    for s in range(cfg.W):
        b = int(cfg.part[s + 1] - cfg.part[s])
        rows = None if rows_per_call is None else np.arange(min(b, rows_per_call))
        l, t = oracle_rows_pass(cfg, csr, s, rows)
        lookups += l
        secs += t
    return lookups, secs


def cpu_baseline(cfg, rank, N, csr_batches, budget_s, gather, weights=None, pooling="sum"):
    """Bounded sample, every rank in parallel on its own host core: whole-output oracle passes
    for THIS rank's rows over the given batches until ~budget_s.  value = all ranks' lookups /
    the slowest rank's seconds (N single-threaded processes, N cores); single_core_value =
    lookups / summed seconds."""
    lookups, secs, passes = 0, 0.0, 0
    while secs < budget_s and passes < 256:
        k = passes % len(csr_batches)
        l, t = oracle_rows_pass(cfg, csr_batches[k], rank,
                                weights=None if weights is None else weights[k], pooling=pooling)
        lookups += l
        secs += t
        passes += 1
    per = gather([float(lookups), secs, float(passes)])
    tot_l = sum(p[0] for p in per)
    tot_s = sum(p[1] for p in per)
    max_s = max(p[1] for p in per)
    return dict({"value": tot_l / max_s, "unit": "lookups/s", "cores": N, "kind": "oracle",
                 "single_core_value": tot_l / tot_s,
                 "per_rank": [{"lookups": int(p[0]), "seconds": p[1], "passes": int(p[2])}
                              for p in per],
                 "sample": f"each of {N} rank process(es) ran the single-threaded C oracle over "
                           f"all of its own output rows (procedural tables) for ~{budget_s:g} s: "
                           f"{int(tot_l)} lookups, {tot_s:.2f} core-seconds"}, **host_cpu())


def run_reference(args):
    """--impl reference: the CPU oracle is this tier's reference arm (no installable reference
    exists; PAPER.md ships no code).  Rank 0 only."""
    import synth
    rank, world, _ = dist_env()
    if rank != 0:
        return
    N = max(args.gpus, world)
    cfg = synth.config_for(args.config, W=N, alpha=args.alpha)
    csrs = [synth.gen_all_csr(cfg, k) for k in range(min(args.batches, 2))]
    for w in range(args.warmup):
        oracle_pass(cfg, csrs[w % len(csrs)], rows_per_call=8)
    lookups, secs = 0, 0.0
    for k in range(args.steps):
        l, s = oracle_pass(cfg, csrs[k % len(csrs)])
        lookups += l
        secs += s
    v = lookups / secs
    line = {"metric": METRIC, "value": v, "unit": "lookups/s",
            "impl": "reference", "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "global_batch": cfg.B,
                       "tables_per_rank": cfg.T[0], "rows": cfg.R, "dim": cfg.D},
            "cpu_baseline": dict({"value": v, "unit": "lookups/s", "cores": 1, "kind": "oracle",
                                  "sample": f"{args.steps} full forwards of the workload (all W "
                                            "ranks' outputs), single-threaded C oracle"},
                                 **host_cpu()),
            "e2e": {"value": v, "unit": "lookups/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm

def main():
    args = parse()
    if args.path == "ag_gemm":
        import bench_ag_gemm
        return bench_ag_gemm.main(args, ROOT, {"ClockSampler": ClockSampler, "host_cpu": host_cpu,
                                               "dist_env": dist_env})
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import synth
    import synth.device as sdev
    from paper_2305_06942_b200 import EmbA2A, torch_allgather

    rank, world, local = dist_env()
    N = world
    if args.gpus != world and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    # EMBA2A_SHARED_GPU=1: test mode for the N>1 code path on a one-GPU box -- every rank runs on
    # cuda:0 (cross-process cudaIpc still used), gloo bootstrap, baseline exchange via host copies.
    # Numbers from this mode are not bench values (ranks time-share one GPU).
    shared = os.environ.get("EMBA2A_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            import socket
            s = socket.socket()
            s.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(s.getsockname()[1])
            s.close()
        if shared:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    cfg = synth.config_for(args.config, W=N, alpha=args.alpha)
    # ---- inputs (all resident in HBM before timing; rotating batches).  Batch 0 of EVERY rank
    # is generated here too: the oracle needs all ranks' bags for this rank's output rows
    # (parity check, cpu_baseline).
    csr0_all = synth.gen_all_csr(cfg, 0)
    mine = [csr0_all[rank]] + [synth.gen_rank_csr(cfg, rank, k) for k in range(1, args.batches)]
    d_in = [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev)) for i, o in mine]
    h_in = [(torch.from_numpy(i).pin_memory(), torch.from_numpy(o).pin_memory()) for i, o in mine]
    nnz_all = []   # global lookups per batch
    for k in range(args.batches):
        t = torch.tensor([mine[k][0].size], dtype=torch.int64, device="cpu" if shared else dev)
        dist.all_reduce(t)
        nnz_all.append(int(t.item()))
    tables = sdev.rank_tables(cfg, rank, dev)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[args.table_dtype]
    if tdt != torch.float32:      # exact conversion of the procedural fp32 values (R#28)
        tables = [t.to(tdt) for t in tables]
    d_w = None
    if args.weighted:
        d_w = [torch.from_numpy(synth.gen_weights(cfg, rank, mine[k][0].size, batch=k)).to(dev)
               for k in range(args.batches)]
    torch.cuda.synchronize()

    h = EmbA2A(rank, N, dev, torch_allgather(None, dev), {"timeout_ms": 60000} if shared else None)
    if args.slice:
        h.set_option("slice", args.slice)
    if args.threads:
        h.set_option("threads", args.threads)
    if args.chunk:
        h.set_option("chunk", args.chunk)
    if args.vec:
        h.set_option("vec", args.vec)
    if args.order >= 0:
        h.set_option("order", args.order)
    if args.ctas_per_sm:
        h.set_option("ctas_per_sm", args.ctas_per_sm)
    for kv in args.opt:
        k_, v_ = kv.split("=")
        h.set_option(k_, int(v_))
    ODT = {"f32": 0, "bf16": 1, "f16": 2}[args.out_dtype]
    oes = 4 if ODT == 0 else 2
    if ODT:
        h.set_option("out_dtype", ODT)
    h.register_tables(tables, cfg.B, pooling=args.pooling)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def b2b_loop(step_fn, K, W):
        """W warm-up steps, then K back-to-back steps between ONE event pair on the launching
        stream (inputs rotate over args.batches batches whose working set exceeds L2), bracketed
        by barrier + synchronize.  Returns this rank's total ms."""
        for w in range(W):
            step_fn(w % args.batches)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h.device_barrier(stream)          # align rank starts on the device (no-op at W = 1)
        a.record(stream)
        for k in range(K):
            step_fn(k % args.batches)
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def timed_loop(step_fn, K, W, with_barrier=True):
        """W warm-up steps, then K steps; per step: L2 flush, device barrier, events around the
        step on the launching stream.  Returns per-step ms (this rank)."""
        for w in range(W):
            step_fn(w % args.batches)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
        for k in range(K):
            flush.zero_()
            if with_barrier:
                h.device_barrier(stream)
            evs[k][0].record(stream)
            step_fn(k % args.batches)
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- fused (the product)
    skew_cycles = int(args.skew_us * 1965) if (args.skew_us > 0 and rank == N - 1) else 0

    def fused_step(k):
        if skew_cycles:                   # E5: a late rank (its peers wait for its slices)
            torch.cuda._sleep(skew_cycles)
        return h.forward(d_in[k][0], d_in[k][1], stream,
                         per_sample_weights=None if d_w is None else d_w[k])
    launches0 = h.query("kernel_launches")
    clk = ClockSampler(local)
    nvc = NvlinkCounters(local) if (N > 1 and not shared) else None
    tx0 = nvc.read() if nvc else None
    clk.start()
    b2b_ms = b2b_loop(fused_step, args.steps, args.warmup)
    clocks = clk.stop()
    tx1 = nvc.read() if nvc else None
    launches = h.query("kernel_launches") - launches0 - args.warmup
    launches -= 1 if N > 1 else 0          # the device barrier before the timed region
    ms = timed_loop(fused_step, args.steps, args.warmup)     # flushed, per-step events
    lookups = sum(nnz_all[k % args.batches] for k in range(args.steps))
    b2b_total = max_over_ranks(b2b_ms)
    flushed_total = max_over_ranks(sum(ms))
    total_ms = b2b_total if args.timing == "b2b" else flushed_total
    value = lookups / (total_ms / 1e3)
    ms_step = total_ms / args.steps

    # dominant kernel = the fused kernel (one launch per step); per-launch time from the same
    # events over the timed region
    nnz_mean = float(np.mean([mine[k % args.batches][0].size for k in range(args.steps)]))
    hbm_b, tx_b = algorithmic_bytes(cfg, rank, nnz_mean, 4 if args.table_dtype == "f32" else 2,
                                    args.weighted, oes)
    peak_hbm, peak_src = measured_peaks()
    t_hbm = hbm_b / (peak_hbm * 1e9)
    t_nvl = tx_b / (NVLINK_GBS * 1e9)

    def roofline(kern_s):
        if t_nvl > t_hbm:
            r = {"bound": "nvlink", "achieved": tx_b / kern_s / 1e9, "peak": NVLINK_GBS,
                 "unit": "GB/s", "peak_source": "measured peer copy (B200_PROFILING.md)"}
        else:
            r = {"bound": "hbm", "achieved": hbm_b / kern_s / 1e9, "peak": peak_hbm,
                 "unit": "GB/s", "peak_source": peak_src}
        r["frac"] = r["achieved"] / r["peak"]
        return r

    roof = roofline(ms_step / 1e3)
    roof["algorithmic_bytes_per_launch"] = hbm_b
    roof["nvlink_tx_bytes_per_launch"] = tx_b
    # the committed capture is of the default variant (fp32 sum, unweighted, default alpha)
    default_variant = (args.table_dtype == "f32" and args.pooling == "sum" and not args.weighted
                       and args.alpha == 1.05)
    roof["traffic"] = ncu_traffic(cfg) if default_variant else None
    roof["roofline_us"] = max(t_hbm, t_nvl) * 1e6
    flushed = {"us_per_step": flushed_total / args.steps * 1e3,
               "us_p50": float(np.median(ms)) * 1e3, "us_p90": float(np.percentile(ms, 90)) * 1e3,
               "lookups_per_s": lookups / (flushed_total / 1e3),
               "roofline_frac": roofline(flushed_total / args.steps / 1e3)["frac"],
               "note": "L2 flushed (512 MiB write) + device barrier before each step, CUDA events "
                       "around each forward (includes ~5 us event overhead per step)"}

    # ---- parity (outside every timed region, before the backward section updates the
    # tables): a fresh forward of batch 0, >= 96 sampled output rows of THIS rank recomputed one
    # by one by the oracle from every rank's bags; a mismatch fails the run
    w_all0 = None
    if args.weighted:
        w_all0 = [synth.gen_weights(cfg, r, csr0_all[r][0].size, batch=0) for r in range(N)]
    parity = parity_check(args, cfg, h, csr0_all, w_all0, rank, dev, stream, d_in[0],
                          None if d_w is None else d_w[0])

    # ---- the same step against compulsory bytes and DRAM traffic, and the alpha = 0 control
    esize = 4 if args.table_dtype == "f32" else 2
    comp_b = float(np.mean([compulsory_bytes(cfg, rank, mine[k % args.batches][0],
                                             mine[k % args.batches][1], esize, args.weighted, oes)
                            for k in range(min(args.steps, args.batches))]))
    kern_s = ms_step / 1e3
    roof["compulsory_bytes_per_launch"] = comp_b
    roof["frac_compulsory"] = comp_b / kern_s / 1e9 / peak_hbm
    roof["dram_frac"] = (roof["traffic"] / kern_s / 1e9 / peak_hbm) if roof["traffic"] else None
    roof["readings"] = ("frac: algorithmic bytes (every lookup's row counted, SURVEY 8(d)); "
                        "frac_compulsory: distinct (table,row) rows + indices + offsets + "
                        "receive buffer; dram_frac: ncu dram__bytes of the committed capture "
                        "(cold, serialised) over this run's step time")
    alpha0 = None
    if not args.no_alpha0 and args.alpha != 0.0:
        alpha0 = alpha0_leg(args, cfg, h, rank, N, dev, stream, b2b_loop, max_over_ranks,
                            peak_hbm, esize, oes)
    nvl = None
    if N > 1 and not shared:
        nvl = nvlink_probe(h, N, stream, max_over_ranks) or {}
        if tx0 is not None and tx1 is not None:
            steps_in = args.steps + args.warmup     # the counters saw warm-up steps too
            nvl["nvml_tx_bytes_per_step"] = (tx1 - tx0) / steps_in
            nvl["algorithmic_tx_bytes_per_step"] = tx_b
            nvl["nvml_tx_gbs_during_b2b"] = (tx1 - tx0) / steps_in * args.steps / (b2b_ms / 1e3) / 1e9
            nvl["nvml_note"] = ("NVML NVLink data-TX counters (KiB granularity, all links) "
                                "around the warm-up + timed back-to-back loop, this rank")
        if nvl and nvl.get("tx_gbs_per_gpu") and roof["bound"] == "nvlink":
            roof["peak_measured_probe"] = nvl["tx_gbs_per_gpu"]
            roof["frac_vs_probe"] = roof["achieved"] / nvl["tx_gbs_per_gpu"]

    # ---- end to end through the public API: pinned host inputs -> device -> host result
    b = h.b
    h_out = torch.empty((b, h.G * h.D), dtype=h.out_dtype).pin_memory()
    # the pipelined serving loop (emb_a2a_forward_host_batch): every step copies its inputs in
    # and its result out; neighbouring steps' copies overlap the forwards
    h_outs = [h_out, torch.empty_like(h_out).pin_memory()]
    ks_w = [w % args.batches for w in range(args.warmup)]
    ks = [k % args.batches for k in range(args.steps)]
    h.forward_host_batch([h_in[k][0] for k in ks_w], [h_in[k][1] for k in ks_w],
                         [h_outs[i & 1] for i in range(len(ks_w))], stream)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h.device_barrier(stream)
    ea.record(stream)
    h.forward_host_batch([h_in[k][0] for k in ks], [h_in[k][1] for k in ks],
                         [h_outs[i & 1] for i in range(len(ks))], stream)
    eb.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    e2e_total = max_over_ranks(ea.elapsed_time(eb))
    h2d = float(np.mean([(mine[k % args.batches][0].size + mine[k % args.batches][1].size) * 4
                         for k in range(args.steps)]))
    e2e = {"value": lookups / (e2e_total / 1e3), "unit": "lookups/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(b * h.G * h.D * oes),
           "ms_per_step": e2e_total / args.steps,
           "api": "emb_a2a_forward_host_batch (pinned host in/out, copies overlapped across steps)"}
    if args.weighted:
        e2e["note"] = "forward_host has no per-sample-weight variant: e2e is the unweighted forward"

    # ---- unfused baseline: same pooling kernel -> staging, then NCCL all_to_all_single
    unfused = None
    if not args.no_baseline:
        T = cfg.T[rank]
        send = torch.empty((cfg.B, T, cfg.D), dtype=h.out_dtype, device=dev)
        recv = torch.empty((N, b, T, cfg.D), dtype=h.out_dtype, device=dev)
        final = torch.empty((b, cfg.G * cfg.D), dtype=h.out_dtype, device=dev)

        def unfused_step(k, permute):
            h.pool_local(d_in[k][0], d_in[k][1], send, stream,
                         per_sample_weights=None if d_w is None else d_w[k])
            if shared:     # gloo: exchange through host memory (test mode only)
                r_cpu = torch.empty(recv.numel(), dtype=recv.dtype)
                dist.all_to_all_single(r_cpu, send.view(-1).cpu())
                recv.view(-1).copy_(r_cpu)
            else:
                dist.all_to_all_single(recv.view(-1), send.view(-1))
            if permute:   # [src][i][t][d] -> [i][src*T+t][d] (R#17)
                final.view(b, N, T, cfg.D).copy_(recv.permute(1, 0, 2, 3))

        if args.timing == "b2b":
            un_np_ms = max_over_ranks(b2b_loop(lambda k: unfused_step(k, False), args.steps,
                                               args.warmup)) / args.steps
            un_p_ms = max_over_ranks(b2b_loop(lambda k: unfused_step(k, True), args.steps,
                                              args.warmup)) / args.steps
        else:
            un_np_ms = max_over_ranks(sum(timed_loop(lambda k: unfused_step(k, False), args.steps,
                                                     args.warmup))) / args.steps
            un_p_ms = max_over_ranks(sum(timed_loop(lambda k: unfused_step(k, True), args.steps,
                                                    args.warmup))) / args.steps
        # parity of the two paths on the last batch (cheap, outside timing)
        k = 0
        out_f = fused_step(k).clone()
        unfused_step(k, True)
        torch.cuda.synchronize()
        same = bool(torch.equal(out_f, final))
        unfused = {"us_no_permute": un_np_ms * 1e3, "us_with_permute": un_p_ms * 1e3,
                   "lookups_per_s_no_permute": lookups / (un_np_ms * args.steps / 1e3),
                   "fused_speedup_vs_no_permute": un_np_ms / ms_step,
                   "fused_speedup_vs_permute": un_p_ms / ms_step,
                   "fused_equals_unfused_bitwise": same}

    backward = None
    if not args.no_backward and args.table_dtype == "f32":
        backward = backward_section(args, cfg, h, d_in, mine, dev, stream, N, rank, shared,
                                    b2b_loop, max_over_ranks, peak_hbm, peak_src, d_w)

    cpu = None
    if not args.no_cpu:
        budget = args.cpu_seconds if N == 1 else args.cpu_seconds / 2
        cpu = cpu_baseline(cfg, rank, N, [csr0_all], budget,
                           lambda v: all_gather_floats(v, dist, shared, dev),
                           weights=None if w_all0 is None else [w_all0], pooling=args.pooling)

    ag = None
    if (args.ag_leg == 1 or (args.ag_leg == -1 and N == 1)) and args.timing == "b2b":
        # the fused AllGather + GEMM, its own metric (TFLOP/s); the full
        # line is `bench.py --path ag_gemm`.  Measured after the main path, outside its timing.
        try:
            import bench_ag_gemm
            agl = bench_ag_gemm.measure(args, ROOT, dev, rank, N, shared, ClockSampler, host_cpu,
                                        "ag_tiny" if shared else args.ag_config,
                                        min(args.steps, 10), 3, with_e2e=False, with_cpu=False)
            ag = agl if "error" in agl else {
                  "metric": agl["metric"], "value": agl["value"], "unit": agl["unit"],
                  "ms_per_step": agl["ms_per_step"], "workload": agl["config"]["workload"],
                  "roofline": agl["roofline"], "unfused": agl["unfused"],
                  "parity_all_ranks": agl["parity_all_ranks"], "clocks": agl["clocks"],
                  "gpu_launches": agl["gpu_launches"], "full_line": "bench.py --path ag_gemm"}
        except Exception as e:     # reported, never fatal for the main path's line
            ag = {"error": repr(e)[:400]}
    line = {
        "metric": METRIC,
        "value": value, "unit": "lookups/s", "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "us_per_step": ms_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": ("f32" if args.table_dtype == "f32" else f"{args.table_dtype}-tables/f32-accumulate")
                 + ("" if ODT == 0 else f"/{args.out_dtype}-output"),
        "data": "synthetic (seeded Zipf indices, procedural fp32 tables; DESIGN.md Input recipe)",
        "config": {"workload": workload_desc(cfg), "global_batch": cfg.B,
                   "tables_per_rank": cfg.T[0], "rows": cfg.R, "dim": cfg.D,
                   "pooling": list(cfg.pool), "alpha": cfg.alpha, "world": N,
                   "table_dtype": args.table_dtype, "pooling_mode": args.pooling,
                   "out_dtype": args.out_dtype,
                   "per_sample_weights": bool(args.weighted),
                   "parallelism": f"table-wise MP x{N} -> batch DP x{N}",
                   "slice": h.get_option("slice"), "threads": h.get_option("threads"),
                   "order": h.get_option("order"), "ctas_per_sm": h.get_option("ctas_per_sm"),
                   "chunk_bags": h.query("chunk_bags"),
                   "l1_rows": h.get_option("l1_rows_active"), "opts": list(args.opt),
                   "skew_us_last_rank": args.skew_us,
                   "l2": ("inputs larger than L2: %d rotating batches (~%.0f MB of indices + "
                          "distinct rows) over %.1f GB of tables, K back-to-back steps" %
                          (args.batches, args.batches * working_set_mb(cfg, mine[0][0], mine[0][1]),
                           cfg.T[rank] * cfg.R * cfg.D * 4 / 1e9))
                   if args.timing == "b2b" else
                   f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                   "batches": args.batches,
                   "step_timing": ("one CUDA event pair around K back-to-back forwards on the "
                                   "launching stream, after barrier + device barrier; max over ranks")
                   if args.timing == "b2b" else
                   "CUDA events around each forward after L2 flush + device barrier; sum over K; "
                   "max over ranks"},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "unfused": unfused,
        "parity": parity, "alpha0": alpha0, "nvlink_probe": nvl,
        "flushed": flushed, "clocks": clocks, "gpu_launches": int(launches),
        "backward": backward,
        "ag_gemm": ag,
    }
    if shared:
        line["test_mode"] = "EMBA2A_SHARED_GPU=1: all ranks on one GPU; not a bench value"
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    ok = parity is None or parity.get("skipped") or parity["within_tol"]
    h.destroy()
    dist.barrier()
    dist.destroy_process_group()
    if not ok:
        raise SystemExit(f"rank {rank}: fused output differs from the oracle: {parity}")


def backward_section(args, cfg, h, d_in, mine, dev, stream, N, rank, shared, b2b_loop,
                     max_over_ranks, peak_hbm, peak_src, d_w=None):
    """f3: one training-step backward = sort plan of the batch's lookups + the
    fused backward kernel (gradient exchange DP -> MP over peer memory, segment reduce, sparse
    SGD on the tables).  Baseline: pack the owners' column blocks, NCCL all_to_all_single, then
    the same reduce (backward_local).  Both are timed back to back over the rotating batches;
    the tables are updated in place (lr tiny) and restored before the parity check."""
    import torch
    import torch.distributed as dist
    T, D, b = cfg.T[rank], cfg.D, h.b
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    grad = torch.randn((b, h.G * D), generator=gen, device=dev, dtype=torch.float32)
    lr = 1e-6
    W_ = (lambda k: None) if d_w is None else (lambda k: d_w[k])  # noqa: E731
    plan_step = lambda k: h.backward_plan(d_in[k][0], d_in[k][1], stream,  # noqa: E731
                                          per_sample_weights=W_(k))

    def fused_step(k):
        plan_step(k)
        h.backward(grad, lr, stream)

    send = torch.empty((N, b, T * D), dtype=torch.float32, device=dev)
    recv = torch.empty((cfg.B, T * D), dtype=torch.float32, device=dev)

    def unfused_step(k):
        plan_step(k)
        send.copy_(grad.view(b, N, T * D).permute(1, 0, 2))      # owners' column blocks
        if shared:
            r_cpu = torch.empty(recv.numel(), dtype=recv.dtype)
            dist.all_to_all_single(r_cpu, send.view(-1).cpu())
            recv.view(-1).copy_(r_cpu)
        else:
            dist.all_to_all_single(recv.view(-1), send.view(-1))
        h.backward_local(recv, lr, stream)

    K, W = args.steps, args.warmup
    l0 = h.query("kernel_launches")
    step_ms = max_over_ranks(b2b_loop(fused_step, K, W)) / K
    launches = (h.query("kernel_launches") - l0) // (K + W)
    plan_ms = max_over_ranks(b2b_loop(plan_step, K, W)) / K
    plan_step(0)
    kern_ms = max_over_ranks(b2b_loop(lambda k: h.backward(grad, lr, stream), K, W)) / K
    un_ms = max_over_ranks(b2b_loop(unfused_step, K, W)) / K
    # parity: fused vs unfused from the same tables on batch 0 (bitwise: same plan, same order);
    # only the rows batch 0 touches can change (sparse SGD), so only those are snapshotted
    idx0, off0 = mine[0]
    rows = [torch.from_numpy(np.unique(idx0[off0[t * cfg.B]:off0[(t + 1) * cfg.B]]).astype(np.int64))
            .to(dev) for t in range(T)]
    snap = [tab[r].clone() for tab, r in zip(h._tables, rows)]
    fused_step(0)
    after_f = [tab[r].clone() for tab, r in zip(h._tables, rows)]
    for tab, r, s0 in zip(h._tables, rows, snap):
        tab[r] = s0
    unfused_step(0)
    torch.cuda.synchronize()
    same = all(bool(torch.equal(a, tab[r])) for a, tab, r in zip(after_f, h._tables, rows))
    # algorithmic bytes of the backward kernel (per launch, batch 0): gradient rows read once
    # (B * T_r * D * 4 at the owner + the pushed share), the sorted lookup list (key + bag,
    # 8 B per lookup), each distinct (table, row) read and written once
    idx, off = mine[0]
    uniq = sum(np.unique(idx[off[t * cfg.B]:off[(t + 1) * cfg.B]]).size for t in range(T))
    tx = (cfg.B - b) * T * D * 4 if N > 1 else 0
    alg = cfg.B * T * D * 4 + idx.size * 8 + 2 * uniq * D * 4 + b * (h.G - T) * D * 4 * (N > 1)
    kern_s = kern_ms / 1e3
    return {"what": "plan (radix sort by table,row) + fused backward (DP->MP gradient exchange, "
                    "segment reduce, sparse SGD) per step",
            "us_per_step": step_ms * 1e3, "us_plan": plan_ms * 1e3, "us_kernel": kern_ms * 1e3,
            "lookups_per_s": float(np.mean([m[0].size for m in mine])) * N / (step_ms / 1e3),
            "unfused_us_per_step": un_ms * 1e3,
            "unfused": "plan + pack column blocks + NCCL all_to_all_single + backward_local",
            "fused_speedup": un_ms / step_ms, "fused_equals_unfused_bitwise": same,
            "gpu_launches_per_step": int(launches),
            "roofline": {"bound": "hbm", "kernel": "bwd_kernel", "achieved": alg / kern_s / 1e9,
                         "peak": peak_hbm, "unit": "GB/s", "peak_source": peak_src,
                         "frac": alg / kern_s / 1e9 / peak_hbm, "algorithmic_bytes": int(alg),
                         "traffic": ncu_traffic(cfg, "_backward") if (
                             d_w is None and args.pooling == "sum" and args.alpha == 1.05) else None,
                         "distinct_rows": int(uniq), "nvlink_tx_bytes": int(tx)}}


def all_gather_floats(vals, dist, shared, dev):
    """Every rank's list of floats, rank-ordered."""
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else dev)
    outs = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(outs, t)
    return [o.cpu().tolist() for o in outs]


def parity_check(args, cfg, h, csr_all, w_all, rank, dev, stream, d_in0, d_w0, nsample=96):
    """A fresh fused forward of batch 0; nsample output rows of this rank (first, last, random)
    against the oracle, element by element: max |err|, bitwise, within the north-star
    tolerance (|err| <= 1e-6 + 1e-5 |ref|)."""
    import torch
    import oracle
    if args.table_dtype != "f32":
        return {"skipped": "16-bit tables hold rounded procedural values; the bench's parity "
                           "check needs the oracle's exact fp32 tables (tests cover bf16/fp16)"}
    out = h.forward(d_in0[0], d_in0[1], stream, per_sample_weights=d_w0).clone()
    torch.cuda.synchronize()
    b = h.b
    if b == 0:
        return {"rows": 0, "max_abs_err": 0.0, "bitwise": True, "within_tol": True}
    rng = np.random.default_rng(1000 + rank)
    sel = np.unique(np.concatenate([[0, b - 1], rng.integers(0, b, max(nsample - 2, 0))]))
    while sel.size < min(nsample, b):
        sel = np.unique(np.concatenate([sel, rng.integers(0, b, nsample)]))[:min(nsample, b)]
    t0 = time.perf_counter()
    odt = {torch.float32: oracle.F32, torch.bfloat16: oracle.BF16, torch.float16: oracle.F16}[h.out_dtype]
    ref = oracle.emb_a2a_rows(cfg.table_seed, cfg.value_mode, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                              [c[0] for c in csr_all], [c[1] for c in csr_all], rank, sel,
                              check_inputs=False, weights=w_all,
                              pooling=oracle.MEAN if args.pooling == "mean" else oracle.SUM,
                              out_dtype=odt)
    secs = time.perf_counter() - t0
    got_t = out[torch.from_numpy(sel).to(dev)]
    if odt == oracle.F32:
        got = got_t.cpu().numpy()
        bitwise = bool(np.array_equal(got.view(np.uint32), ref.view(np.uint32)))
        tol = 1e-6 + 1e-5 * np.abs(ref.astype(np.float64))
    else:   # 16-bit output: the rounded oracle value, bit for bit (R#32)
        bits = got_t.view(torch.int16).cpu().numpy().view(np.uint16)
        bitwise = bool(np.array_equal(bits, ref))
        got = got_t.float().cpu().numpy()
        ref = torch.from_numpy(ref.view(np.int16)).view(h.out_dtype).float().numpy()
        tol = np.zeros(ref.shape)
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    return {"rows": int(sel.size), "cols": int(ref.shape[1]), "max_abs_err": float(err.max()),
            "bitwise": bitwise, "within_tol": bool((err <= tol).all()) and (odt == oracle.F32 or bitwise),
            "oracle_seconds": secs,
            "what": "fresh fused forward of batch 0; sampled rows of this rank's output vs "
                    "oracle.emb_a2a_rows (every rank checks its own; the line shows rank 0's)"}


def compulsory_bytes(cfg, r, idx, off, esize=4, weighted=False, oes=4):
    """Bytes one forward cannot avoid moving: each DISTINCT (table, row) once + indices (+
    weights) + offsets + this rank's receive buffer (SURVEY 8(d) "Zipf caveat")."""
    T = cfg.T[r]
    b = int(cfg.part[r + 1] - cfg.part[r])
    uniq = sum(np.unique(idx[off[t * cfg.B]:off[(t + 1) * cfg.B]]).size for t in range(T))
    return uniq * cfg.D * esize + idx.size * (8 if weighted else 4) + (T * cfg.B + 1) * 4 + \
        b * cfg.G * cfg.D * oes


def alpha0_leg(args, cfg, h, rank, N, dev, stream, b2b_loop, max_over_ranks, peak_hbm, esize,
               oes=4):
    """The same fused step on uniform indices (alpha = 0: no Zipf reuse, the cold-cache control
    of SURVEY 8(d)), args.alpha0_batches rotating batches, timed like the headline."""
    import torch
    import synth
    cfg0 = synth.config_for(args.config, W=N, alpha=0.0)
    nb = max(1, args.alpha0_batches)
    mine0 = [synth.gen_rank_csr(cfg0, rank, k) for k in range(nb)]
    d0 = [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev)) for i, o in mine0]
    torch.cuda.synchronize()
    step = lambda k: h.forward(d0[k % nb][0], d0[k % nb][1], stream)  # noqa: E731
    ms = max_over_ranks(b2b_loop(step, args.steps, args.warmup)) / args.steps
    nnz = float(np.mean([mine0[k % nb][0].size for k in range(args.steps)]))
    hbm_b, _ = algorithmic_bytes(cfg0, rank, nnz, esize, False, oes)
    comp = float(np.mean([compulsory_bytes(cfg0, rank, i, o, esize, False, oes) for i, o in mine0]))
    del d0
    return {"us_per_step": ms * 1e3, "frac": hbm_b / (ms / 1e3) / 1e9 / peak_hbm,
            "frac_compulsory": comp / (ms / 1e3) / 1e9 / peak_hbm,
            "algorithmic_bytes_per_launch": hbm_b, "compulsory_bytes_per_launch": comp,
            "batches": nb, "note": "uniform indices (alpha = 0), unweighted sum, same tables"}


def nvlink_probe(h, N, stream, max_over_ranks, nbytes=8 << 20, reps=5):
    """SM-issued st.global.v4 stores from every rank into every peer at once (the fused
    kernel's store pattern without the gather): TX GB/s per GPU, max over ranks, best of reps."""
    import torch
    best = None
    used = 0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h.device_barrier(stream)
        a.record(stream)
        used = h.peer_store_probe(nbytes, stream)
        b.record(stream)
        torch.cuda.synchronize()
        t = max_over_ranks(a.elapsed_time(b))
        best = t if best is None else min(best, t)
    if not used or not best:
        return None
    gbs = (N - 1) * used / (best / 1e3) / 1e9
    return {"tx_gbs_per_gpu": gbs, "bytes_per_peer": used, "peers": N - 1, "ms": best,
            "frac_of_nominal_900": gbs / 900.0, "guide_peer_copy_gbs": NVLINK_GBS,
            "what": "one kernel, all SMs, 16-B peer stores to all N-1 peers concurrently "
                    "(emb_a2a_peer_store_probe), CUDA events, max over ranks, best of %d" % reps}


def working_set_mb(cfg, idx, off):
    """Indices + distinct table rows one batch touches on this rank (MB): the part of the input
    that could stay in L2 between steps."""
    T = (off.size - 1) // cfg.B if cfg.B else 0
    rows = sum(np.unique(idx[off[t * cfg.B]:off[(t + 1) * cfg.B]]).size for t in range(T))
    return (idx.size * 4 + off.size * 4 + rows * cfg.D * 4) / 1e6


def ncu_traffic(cfg, suffix=""):
    """DRAM bytes per fused launch from a committed ncu --set full capture, if one exists for
    this workload (profiles/ncu_traffic.json written from the .ncu-rep by tools)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    key = f"{cfg.name}_W{cfg.W}{suffix}"
    v = d.get(key)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else v


if __name__ == "__main__":
    main()
