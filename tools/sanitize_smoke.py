"""Small forwards and backwards of every kernel path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  W = 1 by default (the sanitizer serialises kernels, which would stall a cross-rank
receive wait); --W 2 for memcheck of the loopback protocol.  Each output is checked against the
oracle, so a sanitizer-induced difference would also show."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2305_06942_b200 import LoopbackGroup  # noqa: E402
from tests._problems import random_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--W", type=int, default=1)
args = ap.parse_args()
dev = torch.device("cuda:0")
cases = [({}, "sum"), ({"tma": 1}, "sum"), ({"flat_below": 1000}, "sum"), ({"vec": 2}, "mean"),
         ({"idx_cap": 3}, "sum"), ({"tma": 1, "stage_kb": 1}, "sum"),
         ({}, "sum")]   # 60 K lookups: 30 sort tiles (two look-back groups), long runs
n = 0
for seed, (opts, pooling) in enumerate(cases):
    if seed == 6:
        p = random_problem(2004, W=args.W, value_mode=1, max_B=2048, max_D=64)
    else:
        p = random_problem(900 + seed, W=args.W, value_mode=1, max_B=64, max_D=64)
    if args.W > 1:
        opts = dict(opts, timeout_ms=120000)
    g = LoopbackGroup(p.W, dev, opts)
    g.register_tables([[torch.from_numpy(t).to(dev) for t in p.rank_tables(r)] for r in range(p.W)],
                      p.B, p.part, dim=p.D, pooling=pooling)
    idx = [torch.from_numpy(i).to(dev) for i in p.indices]
    off = [torch.from_numpy(o).to(dev) for o in p.offsets]
    w = None
    if pooling == "sum" and seed % 2 == 0:
        w = [torch.ones(i.size, dtype=torch.float32, device=dev) for i in p.indices]
    for _ in range(2):
        outs = g.forward(idx, off, weights=w)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets,
                         pooling=oracle.MEAN if pooling == "mean" else oracle.SUM)
    for o, r in zip(outs, ref):
        assert np.array_equal(o.cpu().numpy(), r), (opts, pooling)
    for r, h in enumerate(g.handles):   # the unfused pool kernel too
        send = torch.zeros((p.B, p.T[r], p.D), device=dev)
        h.pool_local(idx[r], off[r], send)
    torch.cuda.synchronize()
    # the backward (f3): sort plan, fused exchange + reduce + SGD (pass 1), cross-chunk fold
    # (pass 2), twice (staging parity); integer gradients -> the oracle's tables bitwise
    rng = np.random.default_rng(seed)
    grads = [rng.integers(-4, 4, (p.b(s_), p.G * p.D)).astype(np.float32) for s_ in range(p.W)]
    kw = {"pooling": oracle.MEAN} if pooling == "mean" else {}
    if w is not None:
        kw["weights"] = [np.ones(i.size, np.float32) for i in p.indices]
    want = [t.copy() for t in p.tables]
    for _ in range(2):
        g.backward(idx, off, [torch.from_numpy(x).to(dev) for x in grads], 0.5, weights=w)
        want = oracle.backward_sgd(p.part, p.D, p.B, p.T, want, p.indices, p.offsets, grads, 0.5,
                                   **kw)
    got = [t.cpu().numpy() for r in range(p.W) for t in g.handles[r]._tables]
    for a_, b_ in zip(got, want):
        if pooling == "mean":   # fl(g / L) is inexact: the summation order shows (R#31)
            assert np.allclose(a_, b_, rtol=1e-6, atol=1e-5), ("backward", opts, pooling)
        else:
            assert np.array_equal(a_, b_), ("backward", opts, pooling)
    g.destroy()
    n += 1
# f4: the fused AllGather + GEMM (TMA, mbarriers, tcgen05 MMA/TMEM, communication warps), exact
# ints -> Y is the oracle's sum rounded once to bf16, bitwise; BN = 256 and BN = 128 shapes
from oracle import ag_gemm as OAG  # noqa: E402
from synth import gemm_gen as GG  # noqa: E402
from synth.device import fill_gemm_bf16  # noqa: E402
from paper_2305_06942_b200 import AgGemmLoopback  # noqa: E402
for (M, Nr, K) in ((256, 256, 192), (128, 384, 128)):
    gc = GG.GemmConfig("san", args.W, M, Nr, K, 1)
    grp = AgGemmLoopback(args.W, dev, {"timeout_ms": 120000, "local_copy": 1})
    grp.register(M, Nr, K)
    ops = []
    for r in range(args.W):
        X = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
        Wr = torch.empty((Nr, K), dtype=torch.bfloat16, device=dev)
        fill_gemm_bf16(X, GG.X_TENSOR + r, GG.GEMM_SEED, 1)
        fill_gemm_bf16(Wr, GG.W_TENSOR + r, GG.GEMM_SEED, 1)
        ops.append((X, Wr))
    for _ in range(2):
        outs = grp.forward([o[0] for o in ops], [o[1] for o in ops])
    shards = [GG.rank_inputs(gc, s)[1] for s in range(args.W)]
    for r in range(args.W):
        Wf, Yref = OAG.ag_gemm(GG.rank_inputs(gc, r)[0], shards)
        assert np.array_equal(outs[r][0].view(torch.int16).cpu().numpy().view(np.uint16),
                              OAG.bf16_rne_bits(Yref)), ("ag_gemm", M, Nr, K, r)
        assert np.array_equal(outs[r][1].view(torch.int16).cpu().numpy().view(np.uint16),
                              GG.to_bf16_bits_exact(Wf)), ("ag_gemm gathered", r)
    grp.destroy()
    n += 1
print(f"sanitize_smoke: {n} cases OK (W={args.W}), forward + backward + AllGather+GEMM")
