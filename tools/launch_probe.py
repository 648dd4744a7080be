"""Where does the fixed per-forward cost go?  Host time per call, and GPU event time with a long
GPU-side sleep before the start event (so host enqueue cost cannot leak into the window)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import synth.device as sdev  # noqa: E402
from paper_2305_06942_b200 import EmbA2A, LocalGroup  # noqa: E402

dev = torch.device("cuda:0")
res = {}
for B, P in ((2048, 20), (2048, 1), (8, 1)):
    cfg = synth.config_for("dlrm_small", W=1, B=B, pool=("fixed", P))
    idx, off = synth.gen_rank_csr(cfg, 0, 0)
    di, do = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
    tables = sdev.rank_tables(cfg, 0, dev)
    h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
    h.register_tables(tables, cfg.B)
    st = torch.cuda.current_stream()
    for _ in range(10):
        h.forward(di, do, st)
    torch.cuda.synchronize()
    # host cost per call (GPU kept busy by a long sleep so calls never block)
    torch.cuda._sleep(50_000_000)
    t0 = time.perf_counter()
    for _ in range(50):
        h.forward(di, do, st)
    host_us = (time.perf_counter() - t0) / 50 * 1e6
    torch.cuda.synchronize()
    for sleep_cycles in (200_000, 4_000_000):
        ts = []
        for _ in range(30):
            torch.cuda._sleep(sleep_cycles)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            h.forward(di, do, st)
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        us = [x.elapsed_time(y) * 1e3 for x, y in ts]
        res[f"B{B}_P{P}_sleep{sleep_cycles}"] = round(float(np.median(us)), 2)
    # back-to-back throughput: 200 forwards, no sleep
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(200):
        h.forward(di, do, st)
    b.record(st)
    torch.cuda.synchronize()
    res[f"B{B}_P{P}_b2b_us"] = round(a.elapsed_time(b) * 1e3 / 200, 2)
    res[f"B{B}_P{P}_host_us"] = round(host_us, 2)
    # an empty torch kernel for the event floor
    h.destroy()
    del tables
    torch.cuda.empty_cache()
x = torch.zeros(1, device=dev)
ts = []
for _ in range(30):
    torch.cuda._sleep(4_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x.add_(1)
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
res["torch_tiny_kernel_us"] = round(float(np.median([p.elapsed_time(q) * 1e3 for p, q in ts])), 2)
print(json.dumps(res))

# ---- CUDA graph replay (W = 1: epoch only selects the output buffer, so a captured launch is
# functionally fine for timing)
cfg = synth.config_for("dlrm_small", W=1)
idx, off = synth.gen_rank_csr(cfg, 0, 0)
di, do = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
tables = sdev.rank_tables(cfg, 0, dev)
h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
h.register_tables(tables, cfg.B)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        h.forward(di, do, s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    h.forward(di, do, s)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    torch.cuda._sleep(4_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
res2 = {"graph_replay_dlrm_small_us": round(float(np.median([p.elapsed_time(q) * 1e3 for p, q in ts])), 2)}
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=s):
    x.add_(1)
ts = []
for _ in range(30):
    torch.cuda._sleep(4_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g2.replay()
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
res2["graph_replay_tiny_us"] = round(float(np.median([p.elapsed_time(q) * 1e3 for p, q in ts])), 2)
# two tiny kernels back to back between events: marginal cost of one more launch
ts = []
for _ in range(30):
    torch.cuda._sleep(4_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x.add_(1)
    x.add_(1)
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
res2["torch_two_tiny_kernels_us"] = round(float(np.median([p.elapsed_time(q) * 1e3 for p, q in ts])), 2)
print(json.dumps(res2))
