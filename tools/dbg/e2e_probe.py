import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, synth.device as sdev
from paper_2305_06942_b200 import EmbA2A, LocalGroup
dev = torch.device("cuda:0")
cfg = synth.config_for("dlrm_small", W=1)
mine = [synth.gen_rank_csr(cfg, 0, k) for k in range(4)]
h_in = [(torch.from_numpy(i).pin_memory(), torch.from_numpy(o).pin_memory()) for i, o in mine]
tables = sdev.rank_tables(cfg, 0, dev)
h = EmbA2A(0, 1, dev, LocalGroup(1).allgather_for(0))
h.register_tables(tables, cfg.B)
out = torch.empty((h.b, h.G * h.D), dtype=torch.float32).pin_memory()
st = torch.cuda.current_stream()
for k in range(5): h.forward_host(h_in[k % 4][0], h_in[k % 4][1], out, st)
torch.cuda.synchronize()
K = 50
t0 = time.perf_counter()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for k in range(K): h.forward_host(h_in[k % 4][0], h_in[k % 4][1], out, st)
b.record(st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("gpu us/step", a.elapsed_time(b) * 1e3 / K, "host us/call", (t1 - t0) / K * 1e6)
# with the host ahead: sleep first
torch.cuda._sleep(100_000_000)
a.record(st)
for k in range(K): h.forward_host(h_in[k % 4][0], h_in[k % 4][1], out, st)
b.record(st)
torch.cuda.synchronize()
print("gpu us/step (host ahead)", a.elapsed_time(b) * 1e3 / K)
print("bytes h2d", mine[0][0].nbytes + mine[0][1].nbytes, "d2h", out.numel() * 4)
h.destroy()
