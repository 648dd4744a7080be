import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, synth.device as sdev
from paper_2305_06942_b200 import EmbA2A, LocalGroup
dev = torch.device("cuda:0")
cfg = synth.config_for(sys.argv[1] if len(sys.argv) > 1 else "dlrm_small", W=1)
idx, off = synth.gen_rank_csr(cfg, 0, 0)
di, do = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
tables = sdev.rank_tables(cfg, 0, dev)
h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
h.register_tables(tables, cfg.B)
for _ in range(3): h.backward_plan(di, do)
torch.cuda.synchronize()
h.set_option("trace", 1 << 20)
h.backward_plan(di, do)
tr = h.read_trace()
t0 = tr["t_ns"].min()
# per pass: passes are sequential; split by large gaps in event-30 times
for e in (30, 31, 32, 33, 34):
    m = tr["event"] == e
    t = (tr["t_ns"][m] - t0) / 1e3
    print(e, "n", m.sum(), "min %.2f med %.2f max %.2f" % (t.min(), np.median(t), t.max()) if m.any() else "")
# per tile durations (per pass: sort by time)
recs = sorted([(int(r["t_ns"]) - int(t0), int(r["event"]), int(r["cta"]), int(r["payload"])) for r in tr])
starts = [r for r in recs if r[1] == 30]
print("first/last start per 1/3:", [round(x[0] / 1e3, 2) for x in starts[::max(1, len(starts) // 9)]])
# phase durations (pair events by (cta, order))
from collections import defaultdict
ev = defaultdict(list)
for t, e, c, p in recs:
    ev[(c, e)].append(t)
for a, b in ((30, 31), (31, 32), (32, 33), (33, 34)):
    d = [tb - ta for c in set(k[0] for k in ev) for ta, tb in zip(ev.get((c, a), []), ev.get((c, b), []))]
    if d: print(f"{a}->{b}: median {np.median(d)/1e3:.2f} us  max {max(d)/1e3:.2f} us")
h.destroy()
