"""The paper's ablations on one B200.

E4 slice size, E3 occupancy, E5 comm-aware vs oblivious order and rank skew
(P:286), E1 per-CTA timeline.  Multi-rank runs use W virtual ranks on the one GPU
(LoopbackGroup: real counters, sys-scope fences, releases and waits; "peer" stores land in the
same HBM), so they measure protocol overhead and scheduling, not NVLink.  Prints JSON lines.
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

dev = torch.device("cuda:0")


def setup(cfg, opts, nb=4):
    grp = LoopbackGroup(cfg.W, dev, opts)
    grp.register_tables([sdev.rank_tables(cfg, r, dev) for r in range(cfg.W)], cfg.B)
    batches = []
    for k in range(nb):
        csr = synth.gen_all_csr(cfg, k)
        batches.append(([torch.from_numpy(c[0]).to(dev) for c in csr],
                        [torch.from_numpy(c[1]).to(dev) for c in csr]))
    return grp, batches


def time_fwd(grp, batches, steps=30):
    for k in range(5):
        grp.forward(*batches[k % len(batches)], sync=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(steps):
        grp.forward(*batches[k % len(batches)], sync=False)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dlrm_small")
    ap.add_argument("--W", type=int, default=4)
    ap.add_argument("--which", default="E4,E3,E5,E1")
    ap.add_argument("--opts", default="", help="extra options for E5/E1, e.g. ctas_per_sm=1")
    args = ap.parse_args()
    which = args.which.split(",")
    cfg = synth.config_for(args.config, W=args.W)
    tabs_cache = None

    if "E4" in which:   # slice size: signals per slice vs overlap granularity
        for S in (1, 2, 4, 8, 16, 32, 64, 128, 256):
            grp, batches = setup(cfg, {"slice": S, "chunk": min(S, 32)})
            us = time_fwd(grp, batches)
            n = grp.handles[0].query("num_slices")
            print(json.dumps({"exp": "E4_slice", "W": cfg.W, "slice": S, "us": round(us, 2),
                              "slices_per_rank": n}), flush=True)
            grp.destroy()
            torch.cuda.empty_cache()

    if "E3" in which:   # occupancy: persistent CTAs per SM
        for W in (1, cfg.W):
            c = synth.config_for(args.config, W=W)
            for k in (1, 2, 3, 4):
                grp, batches = setup(c, {"ctas_per_sm": k})
                us = time_fwd(grp, batches)
                print(json.dumps({"exp": "E3_occupancy", "W": W, "ctas_per_sm": k,
                                  "grid": grp.handles[0].query("last_grid"), "us": round(us, 2)}),
                      flush=True)
                grp.destroy()
                torch.cuda.empty_cache()

    if "E5" in which or "E1" in which:   # order + skew, timeline
        for order in ((0, 1, 2, 0) if "E5" in which else (0,)):
            extra = {k: int(v) for k, v in (kv.split("=") for kv in args.opts.split(",") if kv)}
            grp, batches = setup(cfg, dict(extra, order=order, trace=1 << 20))
            us = time_fwd(grp, batches, steps=10)
            for h in grp.handles:
                h.read_trace()
            torch.cuda.synchronize()
            grp.forward(*batches[0], sync=True, aligned=True)
            traces = [h.read_trace() for h in grp.handles]
            t0 = min(int(tr["t_ns"].min()) for tr in traces)
            ends, first_sig, last_sig, recv_done = [], [], [], []
            for tr in traces:
                t = (tr["t_ns"] - t0) / 1e3
                ends.append(float(t.max()))
                sig = t[(tr["event"] == 3) & (tr["payload"] == 1)]
                first_sig.append(float(sig.min()) if sig.size else None)
                last_sig.append(float(sig.max()) if sig.size else None)
                rd = t[tr["event"] == 5]
                recv_done.append(float(rd.max()) if rd.size else None)
            e = np.array(ends)
            print(json.dumps({"exp": "E5_order", "W": cfg.W, "order": order, "opts": extra,
                              "us_per_fwd": round(us, 2),
                              "rank_end_us": [round(x, 2) for x in ends],
                              "skew_pct": round(float((e.max() - e.min()) / e.mean() * 100), 2),
                              "first_signal_us": first_sig, "last_signal_us": last_sig,
                              "recv_wait_done_us": recv_done}), flush=True)
            if order == 0 and "E1" in which:
                chrome = []
                names = {0: "cta_start", 1: "chunk", 2: "stage_ready", 3: "stage_released",
                         4: "consumers_done", 5: "recv_wait_done"}
                for r, tr in enumerate(traces):
                    for c, ev, pl, tt in zip(tr["cta"], tr["event"], tr["payload"], tr["t_ns"]):
                        chrome.append({"name": names[int(ev)] + ("_signal" if ev == 3 and pl else ""),
                                       "ph": "i", "s": "t", "ts": (int(tt) - t0) / 1e3, "pid": r,
                                       "tid": int(c)})
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                with open(os.path.join(ROOT, "gpurun_out", "timeline_W%d.json" % cfg.W), "w") as f:
                    json.dump({"traceEvents": chrome}, f)
            grp.destroy()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
