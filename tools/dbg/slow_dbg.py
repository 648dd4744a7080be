import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth
from tests._problems import from_config
from tests.test_gpu_parity import dev_csr, oracle_out
from paper_2305_06942_b200 import LoopbackGroup
W = int(os.environ.get("W", "4")); early = int(os.environ.get("EARLY", "0")); pdl = int(os.environ.get("PDL", "1"))
cfg = synth.config_for("tiny", W=W, B=64)
probs = [from_config(cfg, k) for k in range(4)]
g = LoopbackGroup(W, torch.device("cuda:0"), {"slice": 4, "chunk": 2, "pdl_rows_early": early, "timeout_ms": 4000, "pdl": pdl})
tabs = [[torch.from_numpy(t).to("cuda") for t in probs[0].rank_tables(r)] for r in range(W)]
g.register_tables(tabs, cfg.B, cfg.part)
csr = [dev_csr(pr) for pr in probs]
torch.cuda._sleep(10); torch.zeros(4, device="cuda").clone(); torch.cuda.synchronize()
cur = torch.cuda.current_stream()
for s_ in g.streams: s_.wait_stream(cur)
copies = []
for e in range(4):
    for r, h in enumerate(g.handles):
        st = g.streams[r]
        out = h.forward(csr[e][0][r], csr[e][1][r], stream=st)
        if r == 0:
            with torch.cuda.stream(st):
                torch.cuda._sleep(20_000_000)
                copies.append(out.clone())
for s_ in g.streams: cur.wait_stream(s_)
torch.cuda.synchronize()
T = cfg.T[0]; D = cfg.D
for e in range(4):
    got = copies[e].cpu().numpy(); ref = oracle_out(probs[e])[0]
    bad = []
    for src in range(W):
        cols = slice(src * T * D, (src + 1) * T * D)
        if not np.array_equal(got[:, cols], ref[:, cols]):
            # which epoch's data is it?
            match = [k for k in range(4) if np.array_equal(got[:, cols], oracle_out(probs[k])[0][:, cols])]
            bad.append((src, match))
    print("W", W, "early", early, "pdl", pdl, "epoch", e, "bad src blocks (src, matches epoch)", bad, flush=True)
g.destroy()
