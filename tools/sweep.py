"""Tuning sweep of the fused kernel on one GPU (W=1 per-rank work of a config).

  python tools/sweep.py --config dlrm_small --grid 'slice=8,16,32;minb=2,4;unroll=4,8'
Prints one JSON line per option set: median / p10 / p90 us over --steps timed forwards, each
after an L2 flush, plus the HBM roofline fraction.
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import synth.device as sdev  # noqa: E402
from paper_2305_06942_b200 import EmbA2A, LocalGroup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dlrm_small")
    ap.add_argument("--W", type=int, default=1)
    ap.add_argument("--grid", default="slice=32")
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--alpha", type=float, default=1.05)
    ap.add_argument("--pool", action="store_true", help="also time pool_local")
    ap.add_argument("--B", type=int, default=0, help="override the global batch")
    ap.add_argument("--R", type=int, default=0, help="override rows per table")
    ap.add_argument("--P", type=int, default=0, help="override: fixed pooling factor")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "f16"])
    ap.add_argument("--weighted", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--flush-mode", default="write", choices=["write", "read", "sleep"])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    over = {"B": args.B} if args.B else {}
    if args.R:
        over["R"] = args.R
    if args.P:
        over["pool"] = ("fixed", args.P)
    cfg = synth.config_for(args.config, W=args.W, alpha=args.alpha, **over)
    assert cfg.W == 1, "sweep runs one real rank"
    batches = [synth.gen_rank_csr(cfg, 0, k) for k in range(args.batches)]
    d_in = [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev)) for i, o in batches]
    nnz = np.mean([i.size for i, _ in batches])
    tables = sdev.rank_tables(cfg, 0, dev)
    esize = 4
    if args.dtype != "f32":
        tables = [t.to({"bf16": torch.bfloat16, "f16": torch.float16}[args.dtype]) for t in tables]
        esize = 2
    d_w = [torch.from_numpy(synth.gen_weights(cfg, 0, i.size, batch=k)).to(dev)
           for k, (i, _) in enumerate(batches)] if args.weighted else None
    flush = torch.zeros(128 << 20, dtype=torch.float32, device=dev)
    sink = torch.zeros((), device=dev)
    hbm = nnz * cfg.D * esize + nnz * (8 if args.weighted else 4) + (cfg.T[0] * cfg.B + 1) * 4 + cfg.B * cfg.G * cfg.D * 4
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    keys, vals = [], []
    for part in args.grid.split(";"):
        k, v = part.split("=")
        keys.append(k)
        vals.append([int(x) for x in v.split(",")])
    for combo in itertools.product(*vals):
        opts = dict(zip(keys, combo))
        h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
        try:
            for k, v in opts.items():
                h.set_option(k, v)
            h.register_tables(tables, cfg.B)
            h.forward(d_in[0][0], d_in[0][1], per_sample_weights=None if d_w is None else d_w[0])
        except Exception as e:   # invalid combination (e.g. too much shared memory)
            print(json.dumps({"config": cfg.name, "opts": opts, "error": str(e)[:200]}), flush=True)
            continue
        st = torch.cuda.current_stream()

        def run(fn):
            for k in range(5):
                fn(k % args.batches)
            ts = []
            for k in range(args.steps):
                if not args.no_flush:
                    if args.flush_mode == "write":
                        flush.zero_()
                    elif args.flush_mode == "sleep":   # warm caches, launch still queued
                        torch.cuda._sleep(200000)
                    else:
                        sink.copy_(flush.sum())
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                fn(k % args.batches)
                b.record(st)
                ts.append((a, b))
            torch.cuda.synchronize()
            return np.array([a.elapsed_time(b) * 1e3 for a, b in ts])

        us = run(lambda k: h.forward(d_in[k][0], d_in[k][1], st,
                                     per_sample_weights=None if d_w is None else d_w[k]))
        rec = {"config": cfg.name, "opts": opts, "grid": h.query("last_grid"),
               "us_p50": float(np.median(us)), "us_p10": float(np.percentile(us, 10)),
               "us_p90": float(np.percentile(us, 90)), "us_mean": float(us.mean()),
               "frac_p50": hbm / (np.median(us) * 1e-6) / 1e9 / peak}
        if args.pool:
            send = torch.empty((cfg.B, cfg.T[0], cfg.D), device=dev)
            up = run(lambda k: h.pool_local(d_in[k][0], d_in[k][1], send, st))
            rec["pool_us_p50"] = float(np.median(up))
        print(json.dumps(rec), flush=True)
        h.destroy()


if __name__ == "__main__":
    main()
