"""Per-CTA timeline of one fused forward (the paper's Fig. wg_profiled).

  python tools/timeline.py --config dlrm_small [--W 1] [--chrome out.json] [--opts chunk=16,...]
Prints when CTAs start, when their first stage is ready, when consumers finish, and the launch
-> finish span, from %globaltimer records written by the kernel (set_option trace).
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
from paper_2305_06942_b200 import LoopbackGroup  # noqa: E402

EV = {0: "cta_start", 1: "ticket", 2: "stage_ready", 3: "stage_released", 4: "consumers_done",
      5: "recv_wait_done"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dlrm_small")
    ap.add_argument("--W", type=int, default=1)
    ap.add_argument("--opts", default="")
    ap.add_argument("--chrome", default="")
    ap.add_argument("--B", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    over = {"B": args.B} if args.B else {}
    cfg = synth.config_for(args.config, W=args.W, **over)
    opts = {k: int(v) for k, v in (kv.split("=") for kv in args.opts.split(",") if kv)}
    opts["trace"] = 1 << 20
    grp = LoopbackGroup(cfg.W, dev, opts)
    grp.register_tables([sdev.rank_tables(cfg, r, dev) for r in range(cfg.W)], cfg.B)
    csr = synth.gen_all_csr(cfg, 0)
    idx = [torch.from_numpy(c[0]).to(dev) for c in csr]
    off = [torch.from_numpy(c[1]).to(dev) for c in csr]
    flush = torch.empty(128 << 20, device=dev)
    for _ in range(3):
        grp.forward(idx, off)
    for h in grp.handles:
        h.read_trace()
    flush.zero_()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    grp.forward(idx, off, sync=False)
    ev[1].record()
    torch.cuda.synchronize()
    report = {"config": cfg.name, "W": cfg.W, "opts": opts, "event_us": ev[0].elapsed_time(ev[1]) * 1e3}
    chrome = []
    for r, h in enumerate(grp.handles):
        tr = h.read_trace()
        t0 = tr["t_ns"].min()
        t = (tr["t_ns"] - t0) / 1e3
        by = {n: t[tr["event"] == e] for e, n in EV.items()}
        first_ready = {}
        for c, e, tt in zip(tr["cta"], tr["event"], t):
            if e == 2 and c not in first_ready:
                first_ready[c] = tt
        rep = {"grid": int(tr["cta"].max()) + 1, "span_us": float(t.max()),
               "tickets": int((tr["event"] == 1).sum())}
        for n, v in by.items():
            if v.size:
                rep[n] = {"min": float(v.min()), "p50": float(np.median(v)), "max": float(v.max()),
                          "n": int(v.size)}
        fr = np.array(list(first_ready.values()))
        if fr.size:
            rep["first_stage_ready"] = {"min": float(fr.min()), "p50": float(np.median(fr)),
                                        "max": float(fr.max())}
        report[f"rank{r}"] = rep
        for c, e, p, tt in zip(tr["cta"], tr["event"], tr["payload"], t):
            chrome.append({"name": EV[int(e)], "ph": "i", "s": "t", "ts": float(tt), "pid": r,
                           "tid": int(c), "args": {"payload": int(p)}})
    print(json.dumps(report), flush=True)
    if args.chrome:
        with open(args.chrome, "w") as f:
            json.dump({"traceEvents": chrome}, f)
    grp.destroy()


if __name__ == "__main__":
    main()
