import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from tests._problems import random_problem
from tests.test_oracle_backward import grads_for
from tests.test_gpu_backward import Run
dev = torch.device("cuda:0")
seed = int(os.environ.get("SEED", "5602"))
p0 = random_problem(seed, value_mode=1, ragged=True, max_B=128, max_D=64)
print("W", p0.W, "T", p0.T, "D", p0.D, "B", p0.B, "part", list(p0.part), flush=True)
grads = grads_for(p0, 2, 1)
want = oracle.backward_sgd(p0.part, p0.D, p0.B, p0.T, p0.tables, p0.indices, p0.offsets, grads, 2.0)
full = np.concatenate(grads, axis=0).reshape(p0.B, p0.G, p0.D)
for mode in ("fused", "local", "fused_sync"):
    fails = 0
    for it in range(8):
        run = Run(p0)
        if mode == "fused":
            run.backward(grads, 2.0)
        elif mode == "fused_sync":
            # plans first, synchronise, then the backwards
            for r, h in enumerate(run.g.handles):
                h.set_option("bwd_share", p0.W)
                h.backward_plan(run.idx[r], run.off[r])
            torch.cuda.synchronize()
            run.backward(grads, 2.0, plan=False)
        else:
            for r, h in enumerate(run.g.handles):
                h.backward_plan(run.idx[r], run.off[r])
                mp = torch.from_numpy(np.ascontiguousarray(full[:, p0.toff(r):p0.toff(r) + p0.T[r], :])).to(dev)
                h.backward_local(mp, 2.0)
            torch.cuda.synchronize()
        got = run.tables()
        run.destroy()
        bad = [g for g, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        if bad:
            fails += 1
            print(mode, it, "bad tables", bad, flush=True)
    print(mode, "fails", fails, "/ 8", flush=True)
