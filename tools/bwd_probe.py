"""Backward (f3) component timing on one GPU: sort plan and backward kernel, per BASELINE config
at W=1, back-to-back over rotating batches (cold) and on one repeated batch (warm).  Also the
target for `ncu` (one plan + one backward per batch).

  python tools/bwd_probe.py [config ...] [--reps N]
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["dlrm_small"])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--batches", type=int, default=8)
ap.add_argument("--opt", action="append", default=[], help="key=value backward option")
args = ap.parse_args()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(0)
    torch.cuda.synchronize()
    a.record(st)
    for k in range(n):
        fn(k)
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n


for name in args.configs:
    cfg = synth.config_for(name, W=1)
    batches = [synth.gen_rank_csr(cfg, 0, k) for k in range(args.batches)]
    d_in = [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev)) for i, o in batches]
    tables = sdev.rank_tables(cfg, 0, dev)
    h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
    for kv in args.opt:
        k, v = kv.split("=")
        h.set_option(k, int(v))
    h.register_tables(tables, cfg.B)
    grad = torch.randn((h.b, h.G * h.D), device=dev)
    nb = len(d_in)
    plan = lambda k: h.backward_plan(d_in[k % nb][0], d_in[k % nb][1], st)  # noqa: E731
    bwd = lambda k: h.backward(grad, 1e-6, st)  # noqa: E731

    def step(k):
        plan(k)
        bwd(k)

    res = {"config": name, "lookups": int(np.mean([b[0].size for b in batches])),
           "plan_us": timed(plan, args.reps), "step_us": timed(step, args.reps)}
    plan(0)
    res["kernel_warm_us"] = timed(bwd, args.reps)
    res["grid"] = h.query("bwd_grid")
    res["chunk"] = h.query("bwd_chunk")
    print(json.dumps(res), flush=True)
    h.destroy()
    del tables
    torch.cuda.empty_cache()
