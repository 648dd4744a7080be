"""``python bench.py --path ag_gemm``: the fused AllGather + GEMM (SURVEY.md Sec 8 row f4,
PAPER.md P:180 -- FSDP: "the AllGather collective can be overlapped with the subsequent matrix
computations").  Same launch contract and JSON line as the main bench (bench.py).

One step = one fused forward on every rank: rank r gathers the layer weight from the W shards
(its own N/W rows and the peers', PUT into its gather buffer over NVLink by the peers' kernels)
and computes Y_r = X_r W^T, bf16 in, fp32 accumulation, bf16 out.  W-scaling rule (R#36): M, K
and the full weight [N][K] are fixed, so every rank's GEMM is the same size at any W ("weak").
N=1 is the config's per-rank work (a plain GEMM: nothing to gather), compared with cuBLAS;
under torchrun the unfused baseline is NCCL all_gather_into_tensor + cuBLAS (torch.matmul).
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

METRIC_AG = "fused AllGather+GEMM TFLOP/s (ms/step) vs NCCL all_gather + cuBLAS"


def tensor_peaks(root):
    p = os.path.join(root, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return (float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "measured (MEASURED_PEAKS.json bf16_tflops: cuBLAS bf16 8192^3, burst)")
    return 2250.0, 2250.0, "fallback (nominal dense bf16 2.25 PFLOP/s)"


def ncu_traffic(root, cfg):
    """DRAM bytes per launch of ag_gemm_kernel for this workload from the committed ncu capture
    (tools/ncu_traffic.sh -> profiles/ncu_traffic.json), or None."""
    p = os.path.join(root, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    v = json.load(open(p)).get(f"{cfg.name}_W{cfg.W}")
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else None


def workload_desc(cfg):
    return (f"{cfg.name} at W={cfg.W}: X_r [{cfg.M}][{cfg.K}] x AllGather(W_s [{cfg.N_r}][{cfg.K}], "
            f"s<{cfg.W}) -> Y_r [{cfg.M}][{cfg.N}], bf16 in / fp32 accumulate / bf16 out")


def oracle_sample(cfg, rank, budget_s):
    """The oracle (numpy float64 matmul, as it stands) on a bounded sample of the workload:
    16 rows of X_r against 1024 gathered weight rows (all K), repeated for ~budget_s.  Returns
    (flop/s, cores, sample description)."""
    from oracle import ag_gemm as O
    from synth import gemm_gen as G
    rows_m, rows_n = 16, 1024
    X = G.values(G.X_TENSOR + rank, np.arange(rows_m), np.arange(cfg.K))
    shards = [G.values(G.W_TENSOR + s, np.arange(rows_n // cfg.W), np.arange(cfg.K))
              for s in range(cfg.W)]
    flops, secs, reps = 0.0, 0.0, 0
    while secs < budget_s or reps < 1:
        t0 = time.perf_counter()
        O.ag_gemm(X, shards)
        secs += time.perf_counter() - t0
        flops += 2.0 * rows_m * rows_n * cfg.K
        reps += 1
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count() or 1
    return flops / secs, cores, (f"{reps} oracle calls of {rows_m} X rows x {rows_n} gathered "
                                 f"weight rows x K={cfg.K} (numpy float64 matmul), {secs:.1f} s")


def run_reference(args, root, host_cpu):
    """--impl reference on this path: the oracle, rank 0 only."""
    from synth import gemm_gen as G
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    cfg = G.gemm_config(args.ag_config, N)
    per_step = max(0.5, min(20.0, 60.0 / max(args.steps + args.warmup, 1)))
    v, cores, sample = oracle_sample(cfg, 0, per_step * args.steps)
    line = {"metric": METRIC_AG, "value": v / 1e12, "unit": "TFLOP/s", "impl": "reference",
            "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cfg.flops_per_rank() / v * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg)},
            "cpu_baseline": dict({"value": v / 1e12, "unit": "TFLOP/s", "cores": cores,
                                  "kind": "oracle", "sample": sample}, **host_cpu()),
            "e2e": {"value": v / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure(args, root, dev, rank, N, shared, ClockSampler, host_cpu, cfg_name, steps, warmup,
            with_e2e=True, with_cpu=True):
    """One AllGather + GEMM measurement on an initialised process group; returns the JSON dict
    (rank 0's view; timings are max over ranks, parity is min over ranks)."""
    import torch
    import torch.distributed as dist

    from oracle import ag_gemm as O
    from paper_2305_06942_b200 import AgGemm, torch_allgather
    from synth import gemm_gen as G
    from synth.device import fill_gemm_bf16

    local = dev.index or 0
    cfg = G.gemm_config(cfg_name, N, mode=0)
    X = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device=dev)
    Wr = torch.empty((cfg.N_r, cfg.K), dtype=torch.bfloat16, device=dev)
    fill_gemm_bf16(X, G.X_TENSOR + rank, G.GEMM_SEED, 0)
    fill_gemm_bf16(Wr, G.W_TENSOR + rank, G.GEMM_SEED, 0)
    Y = torch.empty((cfg.M, cfg.N), dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()

    def agree(ok):
        """Every rank's verdict on the phase just run (MIN over ranks): a failure on one rank
        stops all of them at the same point instead of leaving the others in a collective."""
        t = torch.tensor([1 if ok else 0], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    h = AgGemm(rank, N, dev, torch_allgather(None, dev), {"timeout_ms": 60000} if shared else None)
    if getattr(args, "ag_order", -1) >= 0:
        h.set_option("order", args.ag_order)
    if getattr(args, "ag_grid", 0):
        h.set_option("grid", args.ag_grid)
    h.register(cfg.M, cfg.N_r, cfg.K)
    stream = torch.cuda.current_stream(dev)
    failed = {}

    def bail(where, err):
        failed["where"] = where
        failed["error"] = err
        h.destroy()                  # collective; every rank reaches it at the same phase
        return {"metric": METRIC_AG, "error": f"{where}: {err}"[:400], "n_gpus": N,
                "config": {"workload": workload_desc(cfg)}, "parity_all_ranks": False}

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def b2b(step, K, W):
        for _ in range(W):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(K):
            step()
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def fused():
        h.forward(X, Wr, Y, stream)

    clk = ClockSampler(local)
    err = ""
    try:
        for _ in range(warmup):
            fused()
        torch.cuda.synchronize()
    except Exception as e:          # host-side failure on this rank
        err = repr(e)
    if not agree(not err and h.status() == 0):
        return bail("warm-up", err or f"device status {h.status()} (rank {rank})")
    clk.start()
    ms = b2b(fused, steps, 0)
    clocks = clk.stop()
    if not agree(h.status() == 0):
        return bail("timed forwards", f"device status {h.status()} (rank {rank})")
    ms_step = max_over_ranks(ms) / steps
    flops = cfg.flops_per_rank()
    value = N * flops / (ms_step * 1e-3) / 1e12
    peak, peak_sus, peak_src = tensor_peaks(root)
    achieved = flops / (ms_step * 1e-3) / 1e12

    # ---- parity: a fresh forward, sampled entries against one-at-a-time oracle dot products
    Yp, Wg = h.forward(X, Wr, None, stream)
    torch.cuda.synchronize()
    if not agree(h.status() == 0):
        return bail("parity forward", f"device status {h.status()} (rank {rank})")
    rng = np.random.default_rng(1000 + rank)
    m = rng.integers(0, cfg.M, 128)
    n = rng.integers(0, cfg.N, 128)
    t0 = time.perf_counter()
    xr = G.values(G.X_TENSOR + rank, m, np.arange(cfg.K))
    wr = np.stack([G.values(G.W_TENSOR + nn // cfg.N_r, [nn % cfg.N_r], np.arange(cfg.K))[0]
                   for nn in n])
    want = O.ag_gemm_entries(xr, wr)
    got = Yp[torch.from_numpy(m).to(dev), torch.from_numpy(n).to(dev)].float().cpu().numpy()
    absdot = np.einsum("ik,ik->i", np.abs(xr), np.abs(wr))
    bound = 2.0 * cfg.K * 2.0 ** -24 * absdot * (1 + 2 ** -8) + 2.0 ** -8 * np.abs(want)
    err = np.abs(got - want)
    ok = bool(np.all(err <= bound + 1e-30))
    remote = [int(nn) for nn in n if nn // cfg.N_r != rank][:16]
    gathered_ok = True
    for nn in remote:
        row = Wg[nn:nn + 1].view(torch.int16).cpu().numpy().view(np.uint16)[0]
        ref = G.to_bf16_bits_exact(G.values(G.W_TENSOR + nn // cfg.N_r, [nn % cfg.N_r],
                                            np.arange(cfg.K))[0])
        gathered_ok &= bool(np.array_equal(row, ref))
    parity = {"entries": int(len(m)), "max_abs_err": float(err.max()),
              "max_err_over_bound": float((err / (bound + 1e-30)).max()),
              "within_bound": ok, "gathered_rows_checked": len(remote),
              "gathered_bitwise": gathered_ok, "oracle_seconds": time.perf_counter() - t0,
              "what": "sampled Y entries vs oracle.ag_gemm_entries within the R#37 bound; "
                      "sampled remote rows of the gather buffer bitwise"}
    okt = torch.tensor([1 if (ok and gathered_ok) else 0], device="cpu" if shared else dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    del Yp

    # ---- unfused baseline: NCCL all_gather_into_tensor + cuBLAS
    Wfull = torch.empty((cfg.N, cfg.K), dtype=torch.bfloat16, device=dev) if N > 1 else Wr
    Yb = torch.empty_like(Y)

    def unfused():
        if N > 1:
            if shared:   # gloo test mode: host round trip (not a bench value)
                parts = [torch.empty_like(Wr).cpu() for _ in range(N)]
                dist.all_gather(parts, Wr.cpu())
                Wfull.copy_(torch.cat(parts).to(dev))
            else:
                dist.all_gather_into_tensor(Wfull, Wr)
        torch.matmul(X, Wfull.t(), out=Yb)

    ms_b = max_over_ranks(b2b(unfused, steps, warmup)) / steps
    ms_gemm = max_over_ranks(b2b(lambda: torch.matmul(X, Wfull.t(), out=Yb), steps, 2)) / steps
    e2e = None
    if with_e2e:
        # end to end through the public API: X from pinned host memory in, Y back to pinned host
        Xh = X.cpu().pin_memory()
        Yh = torch.empty((cfg.M, cfg.N), dtype=torch.bfloat16).pin_memory()
        Xd = torch.empty_like(X)
        e2e_steps = max(2, min(steps, 5))

        def e2e_step():
            Xd.copy_(Xh, non_blocking=True)
            h.forward(Xd, Wr, Y, stream)
            Yh.copy_(Y, non_blocking=True)
        ms_e2e = max_over_ranks(b2b(e2e_step, e2e_steps, 1)) / e2e_steps
        e2e = {"value": N * flops / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": cfg.M * cfg.K * 2, "d2h_bytes_per_step": cfg.M * cfg.N * 2,
               "ms_per_step": ms_e2e,
               "api": "ag_gemm_forward with X copied from pinned host and Y copied back each step"}
    cpu = None
    if with_cpu and rank == 0:
        v, cores, sample = oracle_sample(cfg, 0, min(args.cpu_seconds, 10.0))
        cpu = dict({"value": v / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                    "sample": sample}, **host_cpu())
    line = {
        "metric": METRIC_AG, "value": value, "unit": "TFLOP/s", "n_gpus": N,
        "steps": steps, "warmup": warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-based bf16-exact operands, synth/gemm_gen.py)",
        "config": {"workload": workload_desc(cfg), "M": cfg.M, "N": cfg.N, "K": cfg.K,
                   "N_local": cfg.N_r, "world": N, "parallelism": f"FSDP weight shards x{N}",
                   "bn": h.query("bn"), "grid": h.query("grid"), "order": h.get_option("order"),
                   "l2": f"operands {(cfg.M * cfg.K + cfg.N * cfg.K) * 2 / 2**20:.0f} MiB + "
                         f"output {cfg.M * cfg.N * 2 / 2**20:.0f} MiB > 126 MB L2; K back-to-back steps"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "peak_source": peak_src, "frac": achieved / peak,
                     "frac_vs_sustained": achieved / peak_sus,
                     "flops_per_launch": flops, "traffic": ncu_traffic(root, cfg),
                     "compulsory_bytes": 2 * (cfg.M * cfg.K + cfg.N * cfg.K + cfg.M * cfg.N),
                     "traffic_note": "dram__bytes_read + write per launch from the committed ncu "
                                     "capture (profiles/ncu_traffic.json), cold and serialised"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "unfused": {"ms_per_step": ms_b, "what": ("NCCL all_gather_into_tensor + torch.matmul "
                                                 "(cuBLAS)" if N > 1 else "torch.matmul (cuBLAS)"),
                    "tflops": N * flops / (ms_b * 1e-3) / 1e12, "fused_speedup": ms_b / ms_step,
                    "cublas_gemm_only_ms": ms_gemm},
        "parity": parity, "parity_all_ranks": bool(okt.item()),
        "clocks": clocks, "gpu_launches": steps,
    }
    h.destroy()
    del X, Wr, Y, Yb, Wfull
    torch.cuda.empty_cache()
    return line


def main(args, root, helpers):
    import torch
    import torch.distributed as dist

    ClockSampler, host_cpu, dist_env = helpers["ClockSampler"], helpers["host_cpu"], helpers["dist_env"]
    if args.impl == "reference":
        return run_reference(args, root, host_cpu)
    rank, world, local = dist_env()
    N = world
    if args.gpus != world and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
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
    line = measure(args, root, dev, rank, N, shared, ClockSampler, host_cpu, args.ag_config,
                   args.steps, args.warmup, with_e2e=True, with_cpu=not args.no_cpu)
    line.setdefault("value", 0.0)
    line.setdefault("unit", "TFLOP/s")
    if shared:
        line["test_mode"] = "EMBA2A_SHARED_GPU=1: all ranks on one GPU; not a bench value"
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    ok = line["parity_all_ranks"]
    dist.barrier()
    dist.destroy_process_group()
    if not ok:
        raise SystemExit("ag_gemm parity check FAILED")
