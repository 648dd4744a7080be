"""GPU parity of the backward: sort plan + fused exchange/reduce/SGD kernel
through the C ABI, against oracle.backward_sgd, element by element.

Tolerance.  The oracle sums a row's contributions in ascending lookup order (R#29); the kernel
sums runs of C sorted lookups, then the runs in order (R#31) -- a different rounding order of
the same sum.  Each side's error is at most gamma_n * S (S = sum of |c_k| for that element,
computed by the oracle on |grad|, |w|; n = lookups of that row), so the gate is
    |gpu - oracle| <= 2 * gamma_n * |lr| * S + 2u * (|W_new| + |lr * acc|)      (u = 2^-24)
(the last term covers the two sides rounding fl(lr * acc) and W - step independently).  In
exact-integer mode every partial sum is exact, so the result must be bitwise equal.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._problems import Problem, csr_from_bags, from_config, random_problem
from tests.test_oracle_backward import grads_for

pytestmark = pytest.mark.gpu

U = 2.0 ** -24


def dev():
    return torch.device("cuda:0")


class Run:
    """Loopback group with this problem's tables on the device (updated in place)."""

    def __init__(self, p: Problem, pooling="sum", opts=None):
        from paper_2305_06942_b200 import LoopbackGroup
        self.p = p
        self.g = LoopbackGroup(p.W, dev(), opts)
        self.tabs = [[torch.from_numpy(np.ascontiguousarray(t)).to(dev()) for t in p.rank_tables(r)]
                     for r in range(p.W)]
        self.g.register_tables(self.tabs, p.B, p.part, dim=p.D, pooling=pooling)
        self.idx = [torch.from_numpy(np.ascontiguousarray(i)).to(dev()) for i in p.indices]
        self.off = [torch.from_numpy(np.ascontiguousarray(o)).to(dev()) for o in p.offsets]

    def backward(self, grads, lr, weights=None, plan=True):
        gd = [torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(dev()) for x in grads]
        w = None if weights is None else [torch.from_numpy(x).to(dev()) for x in weights]
        self.g.backward(self.idx, self.off, gd, lr, weights=w, plan=plan)

    def tables(self):
        return [t.cpu().numpy() for r in range(self.p.W) for t in self.tabs[r]]

    def forward(self):
        return [o.cpu().numpy() for o in self.g.forward(self.idx, self.off)]

    def destroy(self):
        self.g.destroy()


def occurrences(p: Problem):
    """Per global table: count of lookups of each row (n for gamma_n)."""
    out = []
    for r in range(p.W):
        for t in range(p.T[r]):
            o = p.offsets[r]
            seg = p.indices[r][o[t * p.B]: o[(t + 1) * p.B]]
            out.append(np.bincount(seg, minlength=p.tables[p.toff(r) + t].shape[0]))
    return out


def bound_check(p, got, want, grads, lr, weights=None, pooling=oracle.SUM):
    zero = [np.zeros_like(t) for t in p.tables]
    absw = None if weights is None else [np.abs(w) for w in weights]
    S = oracle.backward_sgd(p.part, p.D, p.B, p.T, zero, p.indices, p.offsets,
                            [np.abs(g) for g in grads], -1.0, weights=absw, pooling=pooling)
    acc = oracle.backward_sgd(p.part, p.D, p.B, p.T, zero, p.indices, p.offsets, grads, -1.0,
                              weights=weights, pooling=pooling)
    for g, (a, b, s, ac, n) in enumerate(zip(got, want, S, acc, occurrences(p))):
        nn = n[:, None].astype(np.float64)
        gam = nn * U / (1 - nn * U)
        tol = 2 * gam * abs(lr) * s.astype(np.float64) + \
            2 * U * (np.abs(b).astype(np.float64) + abs(lr) * np.abs(ac).astype(np.float64)) + 1e-30
        err = np.abs(a.astype(np.float64) - b.astype(np.float64))
        bad = err > tol
        assert not bad.any(), (g, np.argwhere(bad)[:5], err[bad][:5], tol[bad][:5])
        untouched = n == 0
        np.testing.assert_array_equal(a[untouched], p.tables[g][untouched])


# ------------------------------------------------------------------------------- exact mode

@pytest.mark.parametrize("seed", range(8))
def test_backward_exact_int_bitwise(seed):
    """Integer tables and gradients, lr = -1 / 0.5: every sum is exact -> bitwise equal."""
    p = random_problem(5000 + seed, value_mode=1, ragged=seed % 2 == 1, max_B=128, max_D=64)
    grads = grads_for(p, seed, 1)
    lr = -1.0 if seed % 2 == 0 else 0.5
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, lr)
    run = Run(p)
    run.backward(grads, lr)
    got = run.tables()
    run.destroy()
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


def test_tiny_config_backward_exact():
    cfg = synth.config_for("tiny", value_mode=1)
    p = from_config(cfg)
    grads = grads_for(p, 7, 1)
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 0.25)
    run = Run(p)
    run.backward(grads, 0.25)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


# ------------------------------------------------------------------------------- fp32 mode

@pytest.mark.parametrize("sort_mode", [1, 2])
@pytest.mark.parametrize("seed", range(3))
def test_both_radix_schemes_exact(seed, sort_mode):
    """The plan's radix passes as one kernel with look-back (1) or as upsweep / scan /
    downsweep (2): same sorted plan, so the same tables bitwise (exact-int), incl. weights."""
    p = random_problem(5800 + seed, value_mode=1, ragged=seed == 1, max_B=128, max_D=64)
    grads = grads_for(p, seed, 1)
    weights = None
    kw = {}
    if seed == 2:
        cfg = synth.config_for("tiny")
        weights = [np.ones(i.size, np.float32) * 2 for i in p.indices]
        kw["weights"] = weights
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 1.0, **kw)
    run = Run(p, opts={"sort_mode": sort_mode})
    run.backward(grads, 1.0, weights=weights)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


def test_reduce_then_scan_many_tiles():
    """More than a wave of radix tiles (auto mode switches to reduce-then-scan): ~1.2 M lookups
    over 2 small tables, exact-int."""
    rng = np.random.default_rng(59)
    D, B = 8, 8192
    R = [48, 33]
    tables = [rng.integers(-8, 8, (r, D)).astype(np.float32) for r in R]
    bags = [[list(rng.integers(0, R[t], rng.integers(50, 100))) for _ in range(B)] for t in range(2)]
    i, o = csr_from_bags(bags)
    assert i.size > 3 * 148 * 2048
    p = Problem(1, [2], D, B, np.array([0, B]), tables, [i], [o])
    grads = grads_for(p, 9, 1)
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, 0.5)
    run = Run(p)
    run.backward(grads, 0.5)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


@pytest.mark.parametrize("seed", range(8))
def test_backward_fp32_within_rounding_bound(seed):
    p = random_problem(5100 + seed, value_mode=0, ragged=seed % 3 == 1, max_B=128, max_D=128)
    grads = grads_for(p, seed, 0)
    lr = 0.05
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, lr)
    run = Run(p)
    run.backward(grads, lr)
    got = run.tables()
    run.destroy()
    bound_check(p, got, want, grads, lr)


@pytest.mark.parametrize("mode", ["weighted", "mean"])
def test_backward_variants(mode):
    p = random_problem(5200, value_mode=0, max_B=128, max_D=64)
    grads = grads_for(p, 3, 0)
    weights = pooling = None
    kw = {}
    if mode == "weighted":
        cfg = synth.config_for("tiny")
        weights = [synth.gen_weights(cfg, r, p.indices[r].size) for r in range(p.W)]
        kw["weights"] = weights
        pooling = oracle.SUM
    else:
        pooling = oracle.MEAN
        kw["pooling"] = oracle.MEAN
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 0.1, **kw)
    run = Run(p, pooling="mean" if mode == "mean" else "sum")
    run.backward(grads, 0.1, weights=weights)
    got = run.tables()
    run.destroy()
    bound_check(p, got, want, grads, 0.1, weights=weights, pooling=pooling)


@pytest.mark.parametrize("threads", [128, 32])
@pytest.mark.parametrize("D", [4, 64, 256, 1024])
def test_hot_row_spanning_many_chunks(D, threads):
    """One row looked up thousands of times (a Zipf head): its run crosses hundreds of chunks
    and more than one 32-chunk look-back window; exact-int grads -> bitwise."""
    B, W = 256, 2
    rng = np.random.default_rng(D)
    bags = [[[5] * 12 + list(rng.integers(0, 40, 3)) for _ in range(B)]]
    i, o = csr_from_bags(bags)
    tab = rng.integers(-8, 8, (40, D)).astype(np.float32)
    tab2 = rng.integers(-8, 8, (40, D)).astype(np.float32)
    i2, o2 = csr_from_bags([[[7] * 3 for _ in range(B)]])
    p = Problem(W, [1, 1], D, B, synth.even_partition(B, W), [tab, tab2], [i, i2], [o, o2])
    grads = grads_for(p, 1, 1)
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, 1.0)
    run = Run(p, opts={"bwd_threads": threads})
    run.backward(grads, 1.0)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


@pytest.mark.parametrize("shift", [0, 1, 17, 31])
def test_runs_around_chunk_edges(shift):
    """Runs of length C-1, C, C+1, 2C+3, 33C, 64C+5 (C = 32 lookups per sub-batch; chunks are
    4 sub-batches) shifted so that they start and end at every offset: runs inside a chunk are
    finished there (handed over between sub-batches), runs that cross chunk edges are folded
    from per-chunk partials (pass 2).  Exact-int -> bitwise."""
    D, B = 8, 64
    unit = 32
    lens = [shift + 1, unit - 1, 3, unit, unit + 1, 2, 2 * unit + 3, 5, unit - 1, unit + 1, 7,
            33 * unit, 1, 1, 64 * unit + 5]
    rows = []
    for x, L in enumerate(lens):
        rows += [x] * L
    # spread the lookups over the bags in order (one table), several per bag
    per = (len(rows) + B - 1) // B
    bags = [rows[j * per:(j + 1) * per] for j in range(B)]
    i, o = csr_from_bags([bags])
    rng = np.random.default_rng(unit)
    tab = rng.integers(-8, 8, (len(lens), D)).astype(np.float32)
    p = Problem(1, [1], D, B, np.array([0, B]), [tab], [i], [o])
    grads = grads_for(p, 2, 1)
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, -1.0)
    run = Run(p)
    run.backward(grads, -1.0)
    np.testing.assert_array_equal(run.tables()[0], want[0])
    assert run.g.handles[0].query("bwd_chunk") % unit == 0
    run.destroy()


@pytest.mark.parametrize("threads", [128, 64])
@pytest.mark.parametrize("seed", range(4))
def test_random_exact_any_grid(seed, threads):
    p = random_problem(5600 + seed, value_mode=1, ragged=True, max_B=128, max_D=64)
    grads = grads_for(p, seed, 1)
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 2.0)
    run = Run(p, opts={"bwd_threads": threads})
    run.backward(grads, 2.0)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


def test_deterministic_and_fused_equals_local():
    """Two identical backwards give bitwise-identical tables; the unfused backward_local from the
    model-parallel gradient layout gives the same bits as the fused exchange."""
    p = random_problem(5300, W=4, value_mode=0, max_B=128, max_D=64)
    grads = grads_for(p, 5, 0)
    res = []
    for _ in range(2):
        run = Run(p)
        run.backward(grads, 0.03)
        res.append(run.tables())
        run.destroy()
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)
    # unfused: grad_mp[r] = [B][T_r][D] gathered on the host (the all_to_all's output layout)
    full = np.concatenate(grads, axis=0).reshape(p.B, p.G, p.D)
    run = Run(p)
    for r, h in enumerate(run.g.handles):
        h.backward_plan(run.idx[r], run.off[r])
        mp = torch.from_numpy(np.ascontiguousarray(full[:, p.toff(r):p.toff(r) + p.T[r], :])).to(dev())
        h.backward_local(mp, 0.03)
    torch.cuda.synchronize()
    for a, b in zip(run.tables(), res[0]):
        np.testing.assert_array_equal(a, b)
    run.destroy()


def test_training_steps_forward_backward_interleaved():
    """forward -> backward -> forward ... over 3 steps on the same handle (exchange epochs, staging
    parity, chunk stamps, plan reuse); each forward sees the previous step's updated tables."""
    p = random_problem(5400, W=2, value_mode=1, max_B=64, max_D=32)
    run = Run(p)
    tabs = [t.copy() for t in p.tables]
    for step in range(3):
        outs = run.forward()
        ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, tabs, p.indices, p.offsets)
        for a, b in zip(outs, ref):
            np.testing.assert_array_equal(a, b)
        grads = grads_for(p, 10 + step, 1)
        tabs = oracle.backward_sgd(p.part, p.D, p.B, p.T, tabs, p.indices, p.offsets, grads, 1.0)
        run.backward(grads, 1.0, plan=(step != 2) or True)
        for a, b in zip(run.tables(), tabs):
            np.testing.assert_array_equal(a, b)
    run.destroy()


def test_single_rank_forward_backward_forward_no_sync():
    """W=1, one stream, no host sync: forward, forward (its table reads may overlap the previous
    forward's drain), plan + backward (writes the tables), forward (must see the update: its
    reads wait for the backward), forward.  Every output equals the oracle on the tables of its
    time, bitwise (exact-int)."""
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    p = random_problem(5700, W=1, value_mode=1, max_B=128, max_D=64)
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0))
    tabs = [torch.from_numpy(np.ascontiguousarray(t)).to(dev()) for t in p.tables]
    h.register_tables(tabs, p.B)
    idx = torch.from_numpy(p.indices[0]).to(dev())
    off = torch.from_numpy(p.offsets[0]).to(dev())
    grads = grads_for(p, 3, 1)
    g = torch.from_numpy(grads[0]).to(dev())
    outs = []
    for k in range(2):
        outs.append(h.forward(idx, off).clone())
    h.backward_plan(idx, off)
    h.backward(g, -1.0)
    for k in range(2):
        outs.append(h.forward(idx, off).clone())
    torch.cuda.synchronize()
    ref0 = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets)[0]
    new = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, -1.0)
    ref1 = oracle.emb_a2a(p.part, p.D, p.B, p.T, new, p.indices, p.offsets)[0]
    for k, o in enumerate(outs):
        np.testing.assert_array_equal(o.cpu().numpy(), ref0 if k < 2 else ref1)
    h.destroy()


def test_empty_plan_and_empty_blocks():
    """No lookups at all on one rank, a rank with an empty batch block, all-empty bags."""
    D, B = 8, 6
    tab = np.arange(10 * D, dtype=np.float32).reshape(10, D)
    i0, o0 = csr_from_bags([[[1, 2], [], [3], [], [], [1]]])
    i1, o1 = csr_from_bags([[[] for _ in range(B)]])
    p = Problem(2, [1, 1], D, B, np.array([0, 0, B]), [tab, tab.copy()], [i0, i1], [o0, o1])
    grads = [np.zeros((0, 2 * D), np.float32), np.ones((B, 2 * D), np.float32)]
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, 1.0)
    run = Run(p)
    run.backward(grads, 1.0)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


def test_rank_without_tables_and_uneven_tables():
    """W=3, T = [2, 0, 3], ragged partition: the rank without tables still pushes its gradient
    rows to the owners; every owner's tables match the oracle bitwise (exact-int)."""
    rng = np.random.default_rng(11)
    D, B = 12, 30
    T = [2, 0, 3]
    part = np.array([0, 7, 19, 30])
    R = [17, 5, 23, 9, 40]
    tables = [rng.integers(-8, 8, (r, D)).astype(np.float32) for r in R]
    idx, off = [], []
    g = 0
    for r in range(3):
        bags = []
        for t in range(T[r]):
            bags.append([list(rng.integers(0, R[g], rng.integers(0, 9))) for _ in range(B)])
            g += 1
        i, o = csr_from_bags(bags) if bags else (np.zeros(0, np.int32), np.zeros(1, np.int32))
        idx.append(i)
        off.append(o)
    p = Problem(3, T, D, B, part, tables, idx, off)
    grads = grads_for(p, 4, 1)
    want = oracle.backward_sgd(p.part, D, B, T, p.tables, p.indices, p.offsets, grads, -1.0)
    run = Run(p)
    for step in range(2):
        run.backward(grads, -1.0)
        for a, b in zip(run.tables(), want):
            np.testing.assert_array_equal(a, b)
        want = oracle.backward_sgd(p.part, D, B, T, want, p.indices, p.offsets, grads, -1.0)
    run.destroy()


def test_backward_plan_validate_mode_rejects_bad_indices():
    """validate=1: an out-of-range index or malformed offsets fail the plan with EINDEX
    before any sort work is enqueued."""
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    from paper_2305_06942_b200.emb_a2a import EmbA2AError
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), {"validate": 1})
    t = torch.zeros(10, 8, device=dev())
    h.register_tables([t], 4)
    idx = torch.tensor([1, 2, 10, 3], dtype=torch.int32, device=dev())      # 10 >= rows
    off = torch.tensor([0, 1, 2, 3, 4], dtype=torch.int32, device=dev())
    with pytest.raises(EmbA2AError) as e:
        h.backward_plan(idx, off)
    assert e.value.status == 8   # EMB_A2A_EINDEX
    bad_off = torch.tensor([0, 3, 2, 3, 4], dtype=torch.int32, device=dev())  # decreasing
    with pytest.raises(EmbA2AError) as e:
        h.backward_plan(torch.tensor([1, 2, 3, 4], dtype=torch.int32, device=dev()), bad_off)
    assert e.value.status == 8
    h.destroy()


def test_backward_rejects_half_tables_and_missing_plan():
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    from paper_2305_06942_b200.emb_a2a import EmbA2AError
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0))
    t = torch.zeros(10, 8, device=dev())
    h.register_tables([t], 4)
    g = torch.zeros(4, 8, device=dev())
    with pytest.raises(EmbA2AError):
        h.backward(g, 1.0)                  # no plan yet
    h.register_tables([t.to(torch.bfloat16)], 4)
    with pytest.raises(EmbA2AError):
        h.backward_plan(torch.zeros(4, dtype=torch.int32, device=dev()),
                        torch.arange(5, dtype=torch.int32, device=dev()))
    h.destroy()


def test_plans_in_any_sequence_use_clean_buffers():
    """The plan's digit counts and tile tickets live in two halves, each keygen zeroing the
    other half for the next plan (no memset in the plan chain).  Plans replaced before any
    backward, empty plans in between (no keygen), and plans big enough for several onesweep
    tiles and two look-back groups must each leave the next plan a clean half: every backward
    matches the oracle bitwise (exact-int) for the plan it follows."""
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    rng = np.random.default_rng(5)
    D, B, T, R = 8, 512, 4, 300
    tab0 = [rng.integers(-8, 8, (R, D)).astype(np.float32) for _ in range(T)]
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0))
    tabs = [torch.from_numpy(t).to(dev()) for t in tab0]
    h.register_tables(tabs, B)

    def csr(maxL):
        bags = [[list(rng.integers(0, R, rng.integers(0, maxL + 1))) for _ in range(B)]
                for _ in range(T)]
        return csr_from_bags(bags)

    plans = {"small": csr(3), "big": csr(40), "empty": csr(0)}
    assert plans["big"][0].size > 16 * 2048      # > 16 onesweep tiles: two look-back groups
    d_in = {k: (torch.from_numpy(i).to(dev()), torch.from_numpy(o).to(dev()))
            for k, (i, o) in plans.items()}
    want = [t.copy() for t in tab0]
    seq = [["small", "big"], ["empty", "big"], ["big", "empty", "small"], ["big"], ["big", "big"],
           ["empty", "empty", "small"], ["small"]]
    for step, names in enumerate(seq):
        for nm in names:
            h.backward_plan(*d_in[nm])
        last = names[-1]
        grad = rng.integers(-4, 4, (B, T * D)).astype(np.float32)
        h.backward(torch.from_numpy(grad).to(dev()), 0.5)
        i, o = plans[last]
        want = oracle.backward_sgd([0, B], D, B, [T], want, [i], [o], [grad], 0.5)
        torch.cuda.synchronize()
        for a, b in zip(tabs, want):
            np.testing.assert_array_equal(a.cpu().numpy(), b, err_msg=f"step {step} {names}")
    h.destroy()


@pytest.mark.parametrize("name", ["dlrm_small", "weak", "sweep_p1", "sweep_p8", "dlrm_wide"])
def test_full_size_backward_sampled_rows(name):
    """BASELINE config at full size (W=1 per-rank work, as bench.py times it): the plan sorts
    every lookup; check the updated table on sampled rows against the oracle on just the
    lookups of those rows (the sum over a row depends only on that row's lookups).  DLRM-small
    and weak sort in one wave of onesweep tiles, sweep P=8 and DLRM-wide (1-2 M lookups) take
    the reduce-then-scan passes; DLRM-wide (D = 256) takes 128-lookup chunks."""
    cfg = synth.config_for(name, W=1)
    csr = synth.gen_all_csr(cfg, 0)
    idx_h, off_h = csr[0]
    rng = np.random.default_rng(0)
    grad = (rng.integers(-(1 << 20), 1 << 20, (cfg.B, cfg.G * cfg.D)) * 2.0 ** -20).astype(np.float32)
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0))
    tabs = [torch.zeros(cfg.R, cfg.D, device=dev()) for _ in range(cfg.T[0])]
    h.register_tables(tabs, cfg.B)
    idx = torch.from_numpy(idx_h).to(dev())
    off = torch.from_numpy(off_h).to(dev())
    h.backward_plan(idx, off)
    h.backward(torch.from_numpy(grad).to(dev()), -1.0)     # zero tables, lr=-1: table = dL/dW
    torch.cuda.synchronize()
    for t in (0, cfg.T[0] - 1):
        o = off_h[t * cfg.B:(t + 1) * cfg.B + 1]
        seg = idx_h[o[0]:o[-1]]
        uniq, cnt = np.unique(seg, return_counts=True)
        pick = np.unique(np.concatenate([uniq[np.argsort(-cnt)[:4]], rng.choice(uniq, 12, replace=False)]))
        got = tabs[t][torch.from_numpy(pick.astype(np.int64)).to(dev())].cpu().numpy()
        # oracle on the sub-problem of just these rows (remapped to 0..len(pick)-1)
        bags = []
        where = {int(x): k for k, x in enumerate(pick)}
        for j in range(cfg.B):
            rows = seg[o[j] - o[0]:o[j + 1] - o[0]]
            bags.append([where[int(x)] for x in rows if int(x) in where])
        si, so = csr_from_bags([bags])
        sub_grad = [grad[:, t * cfg.D:(t + 1) * cfg.D]]
        want = oracle.backward_sgd([0, cfg.B], cfg.D, cfg.B, [1], [np.zeros((len(pick), cfg.D), np.float32)],
                                   [si], [so], sub_grad, -1.0)[0]
        S = oracle.backward_sgd([0, cfg.B], cfg.D, cfg.B, [1], [np.zeros((len(pick), cfg.D), np.float32)],
                                [si], [so], [np.abs(sub_grad[0])], -1.0)[0]
        n = np.array([np.sum(seg == x) for x in pick], np.float64)[:, None]
        tol = 2 * (n * U / (1 - n * U)) * S + 4 * U * np.abs(want) + 1e-30
        assert np.all(np.abs(got.astype(np.float64) - want) <= tol), t
    h.destroy()


def _seg_problem(seed, W, weighted=False, rows=(300, 4000)):
    """Several sort tiles per table (look-back groups of 4 tiles), Zipf-like repeats, exact-int
    values; rows drawn from `rows` (2^17..2^22 reaches every segmented digit width)."""
    rng = np.random.default_rng(seed)
    T = [int(rng.integers(1, 4)) for _ in range(W)]
    D = 8
    B = 1024 * W
    G = sum(T)
    R = [int(rng.integers(rows[0], rows[1])) for _ in range(G)]
    tables = [rng.integers(-8, 8, size=(R[g], D)).astype(np.float32) for g in range(G)]
    indices, offsets = [], []
    g = 0
    for r in range(W):
        bags_t = []
        for t in range(T[r]):
            L = rng.integers(0, 24, size=B)
            hot = rng.integers(0, R[g], size=16)          # repeated rows, runs across tiles
            flat = np.where(rng.random(int(L.sum())) < 0.3, rng.choice(hot, size=int(L.sum())),
                            rng.integers(0, R[g], size=int(L.sum())))
            cuts = np.concatenate([[0], np.cumsum(L)])
            bags_t.append([list(flat[cuts[b]:cuts[b + 1]]) for b in range(B)])
            g += 1
        i, o = csr_from_bags(bags_t)
        indices.append(i)
        offsets.append(o)
    p = Problem(W, T, D, B, synth.even_partition(B, W), tables, indices, offsets)
    w = [rng.integers(1, 4, size=i.size).astype(np.float32) for i in indices] if weighted else None
    return p, w


@pytest.mark.parametrize("seed,W,weighted", [(0, 1, False), (1, 1, True), (2, 2, False),
                                             (3, 4, False)])
def test_segmented_plan_exact_vs_oracle(seed, W, weighted):
    """The segmented sort plan (sort_mode 3: each table's segment sorted by row bits only, 2
    passes, tiles aligned to tables) gives the oracle's tables bitwise in exact-int mode."""
    p, w = _seg_problem(7100 + seed, W, weighted)
    grads = grads_for(p, seed, 1)
    kw = {} if w is None else {"weights": w}
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 0.5, **kw)
    run = Run(p, opts={"sort_mode": 3})
    run.backward(grads, 0.5, weights=w)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


@pytest.mark.parametrize("seed,W,weighted,rows", [(0, 1, False, (1 << 16, 1 << 18)),
                                                  (1, 1, True, (1 << 18, 1 << 20)),
                                                  (2, 2, False, (1 << 20, 1 << 22)),
                                                  (3, 1, False, (1 << 21, 1 << 22))])
def test_segmented_plan_equals_plain_plan_wide_digits(seed, W, weighted, rows):
    """17..22 row bits (digit widths 9, 10, 11): the segmented plan (sort_mode 3) produces the
    plain (table, row) plan's order, so the updated tables are bitwise those of
    sort_mode 1 (the plain plan is pinned to the oracle by the tests above)."""
    p, w = _seg_problem(7150 + seed, W, weighted, rows)
    grads = grads_for(p, seed, 1)
    outs = []
    for mode in (1, 3):
        run = Run(p, opts={"sort_mode": mode})
        run.backward(grads, 0.5, weights=w)
        outs.append(run.tables())
        run.destroy()
    for got in outs[1:]:
        for a, b in zip(got, outs[0]):
            np.testing.assert_array_equal(a, b)


def test_segmented_plan_stall_reports_timeout():
    """The segmented look-back's broken-invariant path (debug_sort_stall) reports ETIMEOUT."""
    from paper_2305_06942_b200 import EmbA2AError
    p, _ = _seg_problem(7200, 1)
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), {"sort_mode": 3, "timeout_ms": 300})
    tabs = [torch.from_numpy(t).to(dev()) for t in p.tables]
    h.register_tables(tabs, p.B)
    idx = torch.from_numpy(p.indices[0]).to(dev())
    off = torch.from_numpy(p.offsets[0]).to(dev())
    h.backward_plan(idx, off)
    torch.cuda.synchronize()
    h.check()
    h.set_option("debug_sort_stall", 1)
    h.backward_plan(idx, off)
    torch.cuda.synchronize()
    with pytest.raises(EmbA2AError) as e:
        h.check()
    assert "ETIMEOUT" in str(e.value)
    h.destroy()


# ------------------------------------------------------------------ cluster plan (sort_mode 4)

@pytest.mark.parametrize("ctas", [0, 1, 4, 16])
@pytest.mark.parametrize("seed,W,weighted", [(0, 1, False), (1, 1, True), (2, 2, False),
                                             (3, 4, False), (4, 2, True)])
def test_cluster_plan_exact_vs_oracle(seed, W, weighted, ctas):
    """The cluster plan (sort_mode 4: one kernel, a thread-block cluster per table, keygen and
    every row-digit pass, offsets exchanged in distributed shared memory) gives the oracle's
    tables bitwise in exact-int mode, at every cluster size (strips of 1..16 CTAs per table)."""
    p, w = _seg_problem(7300 + seed, W, weighted)
    grads = grads_for(p, seed, 1)
    kw = {} if w is None else {"weights": w}
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 0.5, **kw)
    run = Run(p, opts={"sort_mode": 4, "cluster_ctas": ctas})
    run.backward(grads, 0.5, weights=w)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


@pytest.mark.parametrize("seed,W,weighted,rows", [(0, 1, False, (1 << 16, 1 << 18)),
                                                  (1, 1, True, (1 << 18, 1 << 20)),
                                                  (2, 2, False, (1 << 20, 1 << 22)),
                                                  (3, 1, False, (1 << 21, 1 << 22)),
                                                  (4, 1, False, (1 << 8, 1 << 9)),
                                                  (5, 1, True, (1 << 11, 1 << 12))])
def test_cluster_plan_equals_plain_plan_digit_widths(seed, W, weighted, rows):
    """9..22 row bits (2 passes of 5-bit digits .. 3 passes of 8): the cluster plan gives the
    plain (table, row) plan's order, so the updated tables are bitwise those of sort_mode 1
    (fp32 values: any other order would change the rounding somewhere)."""
    p, w = _seg_problem(7350 + seed, W, weighted, rows)
    grads = grads_for(p, seed, 0)
    outs = []
    for mode in (1, 4):
        run = Run(p, opts={"sort_mode": mode})
        run.backward(grads, 0.5, weights=w)
        outs.append(run.tables())
        run.destroy()
    for a, b in zip(outs[1], outs[0]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("case", ["one_row", "tiny_batch", "empty_bags", "one_table", "mean"])
def test_cluster_plan_degenerate(case):
    """Edge cases of the cluster plan vs the oracle (exact-int): every row 0 (no radix pass at
    all: keygen only), fewer bags than cluster CTAs (empty strips), mostly empty bags, a single
    table (one cluster), and mean pooling (per-bag division in pass 1)."""
    rng = np.random.default_rng(77)
    D, T, R, B, maxL = 8, 3, 500, 256, 12
    pooling = "sum"
    if case == "one_row":
        R = 1
    elif case == "tiny_batch":
        B = 3
    elif case == "empty_bags":
        maxL = 1
    elif case == "one_table":
        T = 1
    elif case == "mean":
        pooling = "mean"
    tables = [rng.integers(-8, 8, (R, D)).astype(np.float32) for _ in range(T)]
    bags = [[list(rng.integers(0, R, rng.integers(0, maxL + 1))) for _ in range(B)] for _ in range(T)]
    i, o = csr_from_bags(bags)
    p = Problem(1, [T], D, B, np.array([0, B]), tables, [i], [o])
    grads = grads_for(p, 3, 1)
    kw = {"pooling": oracle.MEAN} if pooling == "mean" else {}
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, 0.5, **kw)
    run = Run(p, pooling=pooling, opts={"sort_mode": 4, "cluster_ctas": 16})
    run.backward(grads, 0.5)
    got = run.tables()
    run.destroy()
    if pooling == "mean":
        bound_check(p, got, want, grads, 0.5, pooling=oracle.MEAN)
    else:
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)


def test_cluster_plan_switching_plan_kinds():
    """Cluster, plain and segmented plans in any order on one handle: the plain plans' two
    digit-count halves (each keygen zeroing the other) are untouched by the cluster plan, so
    every backward still matches the oracle bitwise for the plan it follows."""
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    rng = np.random.default_rng(6)
    D, B, T, R = 8, 512, 4, 3000
    tab0 = [rng.integers(-8, 8, (R, D)).astype(np.float32) for _ in range(T)]
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0))
    tabs = [torch.from_numpy(t).to(dev()) for t in tab0]
    h.register_tables(tabs, B)
    want = [t.copy() for t in tab0]
    for step, mode in enumerate([4, 0, 4, 4, 3, 4, 1, 0, 4]):
        bags = [[list(rng.integers(0, R, rng.integers(0, 30))) for _ in range(B)] for _ in range(T)]
        i, o = csr_from_bags(bags)
        h.set_option("sort_mode", mode)
        h.backward_plan(torch.from_numpy(i).to(dev()), torch.from_numpy(o).to(dev()))
        grad = rng.integers(-4, 4, (B, T * D)).astype(np.float32)
        h.backward(torch.from_numpy(grad).to(dev()), 0.5)
        want = oracle.backward_sgd([0, B], D, B, [T], want, [i], [o], [grad], 0.5)
        torch.cuda.synchronize()
        h.check()
        for a, b in zip(tabs, want):
            np.testing.assert_array_equal(a.cpu().numpy(), b, err_msg=f"step {step} mode {mode}")
    h.destroy()


@pytest.mark.parametrize("name", ["dlrm_small", "weak", "sweep_p8", "dlrm_wide"])
def test_cluster_plan_full_size_equals_plain(name):
    """BASELINE configs at full size (W=1 per-rank work): the cluster plan's tables are bitwise
    those of the plain plan (fp32 gradients, so equal results need the same lookup order; the
    plain plan is pinned to the oracle on sampled rows by test_full_size_backward_sampled_rows)."""
    cfg = synth.config_for(name, W=1)
    idx_h, off_h = synth.gen_all_csr(cfg, 0)[0]
    rng = np.random.default_rng(1)
    grad = torch.from_numpy(rng.standard_normal((cfg.B, cfg.G * cfg.D)).astype(np.float32)).to(dev())
    idx = torch.from_numpy(idx_h).to(dev())
    off = torch.from_numpy(off_h).to(dev())
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    outs = []
    for mode in (0, 4):
        h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), {"sort_mode": mode})
        tabs = [torch.zeros(cfg.R, cfg.D, device=dev()) for _ in range(cfg.T[0])]
        h.register_tables(tabs, cfg.B)
        h.backward_plan(idx, off)
        h.backward(grad, -1.0)
        torch.cuda.synchronize()
        h.check()
        outs.append(tabs)
        h.destroy()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    del outs
    torch.cuda.empty_cache()


# ------------------------------------------------------------------- bucket plan (sort_mode 5)

@pytest.mark.parametrize("cap", [8192, 256])
@pytest.mark.parametrize("seed,W,weighted", [(0, 1, False), (1, 1, True), (2, 2, False),
                                             (3, 4, False), (4, 2, True)])
def test_bucket_plan_exact_vs_oracle(seed, W, weighted, cap):
    """The bucket plan (sort_mode 5: a pass on the top key digit, then every bucket sorted by
    its low bits in shared memory, or in global memory above bucket_cap) gives the oracle's
    tables bitwise in exact-int mode."""
    p, w = _seg_problem(7400 + seed, W, weighted)
    grads = grads_for(p, seed, 1)
    kw = {} if w is None else {"weights": w}
    want = oracle.backward_sgd(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, grads, 0.5, **kw)
    run = Run(p, opts={"sort_mode": 5, "bucket_cap": cap})
    run.backward(grads, 0.5, weights=w)
    for a, b in zip(run.tables(), want):
        np.testing.assert_array_equal(a, b)
    run.destroy()


@pytest.mark.parametrize("cap", [8192, 512])
@pytest.mark.parametrize("seed,W,weighted,rows", [(0, 1, False, (1 << 16, 1 << 18)),
                                                  (1, 1, True, (1 << 18, 1 << 20)),
                                                  (2, 2, False, (1 << 20, 1 << 22)),
                                                  (4, 1, False, (1 << 8, 1 << 9)),
                                                  (5, 1, True, (40, 200))])
def test_bucket_plan_equals_plain_plan(seed, W, weighted, rows, cap):
    """Key widths from 8 to 24 bits (0 to 3 local passes per bucket): the bucket plan's order is
    the plain plan's, so the updated tables are bitwise those of sort_mode 1 (fp32 values)."""
    p, w = _seg_problem(7450 + seed, W, weighted, rows)
    grads = grads_for(p, seed, 0)
    outs = []
    for mode, opts in ((1, {}), (5, {"bucket_cap": cap})):
        run = Run(p, opts=dict(opts, sort_mode=mode))
        run.backward(grads, 0.5, weights=w)
        outs.append(run.tables())
        run.destroy()
    for a, b in zip(outs[1], outs[0]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("case", ["one_row", "tiny_batch", "empty_bags", "one_table", "mean",
                                  "hot_row"])
def test_bucket_plan_degenerate(case):
    """Edge cases of the bucket plan vs the oracle (exact-int): every row 0 (a key of the table
    bits only), 3 bags, mostly empty bags, one table, mean pooling, and one row looked up by
    every bag (a bucket above the shared-memory capacity: the global-memory path)."""
    rng = np.random.default_rng(78)
    D, T, R, B, maxL = 8, 3, 500, 256, 12
    pooling = "sum"
    if case == "one_row":
        R = 1
    elif case == "tiny_batch":
        B = 3
    elif case == "empty_bags":
        maxL = 1
    elif case == "one_table":
        T = 1
    elif case == "mean":
        pooling = "mean"
    tables = [rng.integers(-8, 8, (R, D)).astype(np.float32) for _ in range(T)]
    if case == "hot_row":
        B = 2048
        bags = [[[5] * int(rng.integers(2, 8)) + list(rng.integers(0, R, 2)) for _ in range(B)]
                for _ in range(T)]
    else:
        bags = [[list(rng.integers(0, R, rng.integers(0, maxL + 1))) for _ in range(B)]
                for _ in range(T)]
    i, o = csr_from_bags(bags)
    p = Problem(1, [T], D, B, np.array([0, B]), tables, [i], [o])
    grads = grads_for(p, 3, 1)
    kw = {"pooling": oracle.MEAN} if pooling == "mean" else {}
    want = oracle.backward_sgd(p.part, D, B, p.T, p.tables, p.indices, p.offsets, grads, 0.5, **kw)
    run = Run(p, pooling=pooling, opts={"sort_mode": 5, "bucket_cap": 1024})
    run.backward(grads, 0.5)
    got = run.tables()
    run.destroy()
    if pooling == "mean":
        bound_check(p, got, want, grads, 0.5, pooling=oracle.MEAN)
    else:
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", ["dlrm_small", "weak", "sweep_p1", "sweep_p8", "dlrm_wide"])
def test_bucket_plan_full_size_equals_plain(name):
    """BASELINE configs at full size: the bucket plan's tables are bitwise those of the plain
    plan (fp32 gradients: equal results need the same lookup order); weak and sweep P=1 take
    the bucket plan by default (auto), the others are forced."""
    cfg = synth.config_for(name, W=1)
    idx_h, off_h = synth.gen_all_csr(cfg, 0)[0]
    rng = np.random.default_rng(1)
    grad = torch.from_numpy(rng.standard_normal((cfg.B, cfg.G * cfg.D)).astype(np.float32)).to(dev())
    idx = torch.from_numpy(idx_h).to(dev())
    off = torch.from_numpy(off_h).to(dev())
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    outs = []
    for mode in (1, 5):
        h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), {"sort_mode": mode})
        tabs = [torch.zeros(cfg.R, cfg.D, device=dev()) for _ in range(cfg.T[0])]
        h.register_tables(tabs, cfg.B)
        h.backward_plan(idx, off)
        h.backward(grad, -1.0)
        torch.cuda.synchronize()
        h.check()
        outs.append(tabs)
        h.destroy()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    del outs
    torch.cuda.empty_cache()
