import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from tests._problems import random_problem
from tests.test_oracle_backward import grads_for
from tests.test_gpu_backward import Run
for seed in [int(x) for x in os.environ.get('SEEDS','0 1 2 3').split()]:
    for unit in (0,):
        p = random_problem(5000 + seed, value_mode=1, ragged=seed % 2 == 1, max_B=128, max_D=64)
        grads = grads_for(p, seed, 1)
        lr = -1.0
        zero = [np.zeros_like(t) for t in p.tables] if os.environ.get("ZERO") else p.tables
        want = oracle.backward_sgd(p.part, p.D, p.B, p.T, zero, p.indices, p.offsets, grads, lr)
        p.tables = zero
        run = Run(p, opts={"bwd_unit": unit})
        run.backward(grads, lr)
        got = run.tables()
        u = run.g.handles[0].query("bwd_unit")
        run.destroy()
        bad = [(g, int(np.sum(np.any(a != b, axis=1))), a.shape[0]) for g, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        print(seed, unit, u, "W", p.W, "T", p.T, "D", p.D, "B", p.B, "nnz", [i.size for i in p.indices], "bad", bad[:6], flush=True)
        if bad:
            g = bad[0][0]
            a, b = got[g], want[g]
            rows = np.nonzero(np.any(a != b, axis=1))[0][:3]
            for r in rows:
                print("   row", r, "got", a[r][:6], "want", b[r][:6])
