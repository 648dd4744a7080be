"""The paper's ablations on real GPUs, one process per GPU, as ONE command:

    python tools/ablations_torchrun.py --gpus 8 [--config dlrm_small] [--out f.jsonl]

Each point is a `bench.py` run under torchrun (max-over-ranks device timing, the same protocol
and JSON line as the headline bench), printed as one JSON line with an "ablation" key:

  E4  slice size S (signals per slice vs overlap granularity)
  E3  persistent CTAs per SM (occupancy vs memory contention)
  E5  comm-aware staggered / ascending / oblivious order, without and with a
      late rank (the last rank sleeps --skew-us on the GPU before each forward)
  AG  the fused AllGather + GEMM: comm-aware tile order (own shard first, then
      sources in arrival order) vs ascending source order, N > 1 only

--gpus 1 runs bench.py directly (no peers: E5 is then meaningless and skipped).  With
EMBA2A_SHARED_GPU=1 every rank shares cuda:0 (a test of the command, not a measurement).
"""
import argparse
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_point(args, extra, tag):
    base = [os.path.join(ROOT, "bench.py"), "--gpus", str(args.gpus), "--steps", str(args.steps),
            "--warmup", str(args.warmup), "--config", args.config, "--no-baseline",
            "--no-backward", "--no-cpu", "--no-alpha0", "--ag-leg", "0",
            "--batches", str(args.batches)] + extra
    if args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(free_port())] + base
    else:
        cmd = [sys.executable] + base
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=args.timeout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if r.returncode != 0 or len(lines) != 1:
        rec = {"ablation": tag, "error": (r.stderr or r.stdout)[-1500:], "rc": r.returncode}
    else:
        d = json.loads(lines[0])
        rec = {"ablation": tag, "n_gpus": d["n_gpus"], "us_per_step": d.get("us_per_step"),
               "ms_per_step": d.get("ms_per_step"),
               "value": d["value"], "unit": d["unit"], "roofline": d["roofline"],
               "parity": d.get("parity"), "clocks": d.get("clocks"), "config": d["config"]}
        if isinstance(d.get("unfused"), dict) and "fused_speedup" in d["unfused"]:
            rec["fused_speedup"] = d["unfused"]["fused_speedup"]
    print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--config", default="dlrm_small")
    ap.add_argument("--which", default="E4,E3,E5,AG")
    ap.add_argument("--ag-config", default="ag_ffn")
    ap.add_argument("--slices", default="1,4,8,16,32,64,128,256")
    ap.add_argument("--ctas", default="1,2,3,4")
    ap.add_argument("--skew-us", type=float, default=20.0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--timeout", type=int, default=900)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    which = args.which.split(",")
    if "E4" in which:
        for S in [int(x) for x in args.slices.split(",")]:
            run_point(args, ["--slice", str(S)], {"E4": {"slice": S}})
    if "E3" in which:
        for c in [int(x) for x in args.ctas.split(",")]:
            run_point(args, ["--ctas-per-sm", str(c)], {"E3": {"ctas_per_sm": c}})
    if "E5" in which and args.gpus > 1:
        for order in (0, 1, 2):
            for skew in (0.0, args.skew_us):
                run_point(args, ["--order", str(order), "--skew-us", str(skew)],
                          {"E5": {"order": ["staggered", "ascending", "oblivious"][order],
                                  "skew_us_last_rank": skew}})
    if "AG" in which and args.gpus > 1:
        for order in (0, 1):
            run_point(args, ["--path", "ag_gemm", "--ag-config", args.ag_config,
                             "--ag-order", str(order)],
                      {"AG": {"order": ["comm-aware", "ascending"][order]}})


if __name__ == "__main__":
    main()
