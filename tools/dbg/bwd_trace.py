import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, synth.device as sdev
from paper_2305_06942_b200 import EmbA2A, LocalGroup
dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
cfg = synth.config_for(name, W=1)
idx, off = synth.gen_rank_csr(cfg, 0, 0)
di, do = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
tables = sdev.rank_tables(cfg, 0, dev)
h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
h.register_tables(tables, cfg.B)
grad = torch.randn((h.b, h.G * h.D), device=dev)
for _ in range(3):
    h.backward_plan(di, do); h.backward(grad, 1e-6)
torch.cuda.synchronize()
h.set_option("trace", 1 << 20)
h.backward_plan(di, do)
torch.cuda.synchronize()
h.read_trace()
h.backward(grad, 1e-6)
tr = h.read_trace()
t0 = tr["t_ns"].min()
ev = {}
for e in (20, 21, 22, 23, 24, 25, 26):
    m = tr["event"] == e
    if m.any():
        ev[e] = ((tr["t_ns"][m] - t0) / 1000.0)
        print(e, "n", m.sum(), "first %.2f us  median %.2f  last %.2f" % (ev[e].min(), np.median(ev[e]), ev[e].max()))
# per warp: chunk durations
warps = {}
for rec in tr:
    warps.setdefault(rec["cta"], []).append((rec["t_ns"] - t0, rec["event"], rec["payload"]))
durs = []
for w, lst in warps.items():
    lst.sort()
    st = None
    for t, e, pl in lst:
        if e == 22: st = t
        if e in (22, 26) and st is not None and t != st:
            pass
    ts = {e: t for t, e, pl in lst}
busy = [max(t for t, e, p in lst) - min(t for t, e, p in lst) for lst in warps.values()]
print("warps", len(warps), "busy us: median %.2f max %.2f" % (np.median(busy) / 1e3, max(busy) / 1e3))
# the slowest warp's timeline
w = max(warps, key=lambda k: max(t for t, e, p in warps[k]) - min(t for t, e, p in warps[k]))
print("slowest warp", w, [(round(t / 1e3, 2), e, p) for t, e, p in sorted(warps[w])][:40])
h.destroy()
