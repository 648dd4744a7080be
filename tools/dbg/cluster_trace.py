"""Phase timeline of the cluster sort plan (sort_mode 4) from its trace events (40..46)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, synth.device as sdev
from paper_2305_06942_b200 import EmbA2A, LocalGroup
dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "dlrm_small"
opts = dict(kv.split("=") for kv in sys.argv[2:])
cfg = synth.config_for(name, W=1)
idx, off = synth.gen_rank_csr(cfg, 0, 0)
di, do = torch.from_numpy(idx).to(dev), torch.from_numpy(off).to(dev)
tables = sdev.rank_tables(cfg, 0, dev)
h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
h.set_option("sort_mode", 4)
for k, v in opts.items():
    h.set_option(k, int(v))
h.register_tables(tables, cfg.B)
for _ in range(3): h.backward_plan(di, do)
torch.cuda.synchronize()
h.set_option("trace", 1 << 16)
h.read_trace()
h.backward_plan(di, do)
torch.cuda.synchronize()
tr = h.read_trace()
t0 = tr["t_ns"].min()
print(name, opts, "records", len(tr), "ctas", len(set(tr["cta"])))
for e in range(40, 47):
    for p in sorted(set(tr["payload"][tr["event"] == e])):
        m = (tr["event"] == e) & (tr["payload"] == p)
        t = (tr["t_ns"][m] - t0) / 1e3
        print(f"event {e} pass {p}: n {m.sum():4d}  min {t.min():7.2f}  med {np.median(t):7.2f}  max {t.max():7.2f} us")
h.destroy()
