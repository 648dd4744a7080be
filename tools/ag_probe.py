"""AllGather+GEMM launch-shape probe (W=1): time the fused kernel at several grids / pair modes."""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from synth import gemm_gen as G
from synth.device import fill_gemm_bf16
from paper_2305_06942_b200 import AgGemm, LocalGroup
cfgname = sys.argv[1] if len(sys.argv) > 1 else "ag_ffn"
cfg = G.gemm_config(cfgname, 1)
dev = torch.device("cuda:0")
X = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device=dev)
Wr = torch.empty((cfg.N_r, cfg.K), dtype=torch.bfloat16, device=dev)
fill_gemm_bf16(X, G.X_TENSOR, G.GEMM_SEED, 0); fill_gemm_bf16(Wr, G.W_TENSOR, G.GEMM_SEED, 0)
Y = torch.empty((cfg.M, cfg.N), dtype=torch.bfloat16, device=dev)
h = AgGemm(0, 1, dev, LocalGroup(1).allgather_for(0))
if len(sys.argv) > 3:
    h.set_option("bn", int(sys.argv[3]))
h.register(cfg.M, cfg.N_r, cfg.K)
print(json.dumps({"bn": h.query("bn"), "pair": h.query("pair")}))
def t(steps=10):
    for _ in range(3): h.forward(X, Wr, Y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps): h.forward(X, Wr, Y)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / steps
flops = cfg.flops_per_rank()
mode = sys.argv[2] if len(sys.argv) > 2 else "grid"
if mode.startswith("grid_h"):                 # a few forwards with l2hints 0/1 (ncu target)
    h.set_option("l2hints", int(mode[-1]))
    for _ in range(6):
        h.forward(X, Wr, Y)
    torch.cuda.synchronize()
elif mode == "grid":
    for pair in (1, 0):
        for grid in (148, 146, 144, 140, 128, 112, 96, 74, 64):
            h.set_option("pair", pair); h.set_option("grid", grid)
            ms = t()
            print(json.dumps({"pair": pair, "grid": h.query("grid"), "ms": round(ms, 4),
                              "tflops": round(flops / ms / 1e9, 1)}), flush=True)
elif mode == "ab":
    # interleaved A/B: every config measured once per round, 5 rounds; min and median reported
    import statistics
    confs = [dict(pair=1, l2hints=0), dict(pair=1, l2hints=1), dict(pair=1, l2hints=4),
             dict(pair=1, l2hints=5), dict(pair=1, l2hints=7), "cublas"]
    Yb = torch.empty_like(Y)
    res = {i: [] for i in range(len(confs))}
    for rnd in range(5):
        for i, c in enumerate(confs):
            if c == "cublas":
                for _ in range(3): torch.matmul(X, Wr.t(), out=Yb)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(10): torch.matmul(X, Wr.t(), out=Yb)
                b.record(); torch.cuda.synchronize()
                res[i].append(a.elapsed_time(b) / 10)
            else:
                for k, v in c.items(): h.set_option(k, v)
                res[i].append(t(10))
    for i, c in enumerate(confs):
        print(json.dumps({"conf": c, "ms_min": round(min(res[i]), 4),
                          "ms_med": round(statistics.median(res[i]), 4),
                          "tflops_best": round(flops / min(res[i]) / 1e9, 1)}), flush=True)
else:
    for gm in (2, 4, 8, 16, 32, 64):
        h.set_option("group_m", gm)
        ms = t(20)
        print(json.dumps({"pair": h.query("pair"), "group_m": gm, "ms": round(ms, 4),
                          "tflops": round(flops / ms / 1e9, 1)}), flush=True)
    Yb = torch.empty_like(Y)
    for _ in range(3): torch.matmul(X, Wr.t(), out=Yb)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): torch.matmul(X, Wr.t(), out=Yb)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(json.dumps({"cublas_ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1)}))
h.destroy()
