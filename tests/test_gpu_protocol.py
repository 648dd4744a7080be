"""GPU tests of the exchange protocol's ordering guarantees (Sec 12), through the
C ABI, against the CPU oracle:

- programmatic dependent launch: a kernel triggers its successor only after its own wait, so
  the successor's early work never overlaps the kernel BEFORE it (backward -> forward -> forward
  with no host sync and no kernel in between, small grids so the three can co-reside);
- buffer-reuse credits: a writer stores into a peer's receive half (gradient staging half) only
  once that peer has started the forward (backward) that reuses it -- also when the writer has
  no reason to wait otherwise (it receives nothing: an empty batch block, or owns no tables);
- the pipelined host path at W > 1; the trace option's event counts; error words of the sort
  look-back and of the option ranges.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._problems import Problem, csr_from_bags, from_config, random_problem
from tests.test_oracle_backward import grads_for

pytestmark = pytest.mark.gpu


def dev():
    return torch.device("cuda:0")


def oracle_out(p: Problem, tables=None):
    return oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables if tables is None else tables,
                          p.indices, p.offsets)


def _single(p: Problem, opts=None):
    from paper_2305_06942_b200 import EmbA2A, LocalGroup
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), opts)
    tabs = [torch.from_numpy(np.ascontiguousarray(t)).to(dev()) for t in p.tables]
    h.register_tables(tabs, p.B)
    return h, tabs


def _load_torch_kernels():
    # a lazily loaded module queued behind a forward that waits for a peer on this same GPU
    # would stall that peer: load the torch kernels the tests use first
    torch.cuda._sleep(10)
    torch.zeros(4, device=dev()).clone()
    torch.cuda.synchronize()


# ------------------------------------------------------------------ programmatic launch order

@pytest.mark.parametrize("ctas", [1, 2])
def test_backward_forward_forward_chain_small_grid(ctas):
    """W=1, one stream, no host sync and nothing between the kernels: plan, backward (writes the
    tables), forward A (waits for it), forward B (rows may be read before A completes -- but
    never before the backward completes), forward A again (stores into the half forward A
    filled: never before forward A completes).  Small persistent grids, so the kernels can
    co-reside.  Bitwise equal to the oracle on the tables of their time (exact-int)."""
    pa = random_problem(7100, W=1, value_mode=1, max_B=256, max_D=64)
    rng = np.random.default_rng(7)
    R = [t.shape[0] for t in pa.tables]
    bags = [[list(rng.integers(0, R[t], rng.integers(0, 30))) for _ in range(pa.B)]
            for t in range(len(pa.tables))]
    ib, ob = csr_from_bags(bags)
    pb = Problem(1, pa.T, pa.D, pa.B, pa.part, pa.tables, [ib], [ob])
    h, tabs = _single(pa, {"ctas_per_sm": ctas, "slice": 4, "chunk": 2})
    ia, oa = torch.from_numpy(pa.indices[0]).to(dev()), torch.from_numpy(pa.offsets[0]).to(dev())
    ibd, obd = torch.from_numpy(ib).to(dev()), torch.from_numpy(ob).to(dev())
    grads = grads_for(pa, 11, 1)
    g = torch.from_numpy(grads[0]).to(dev())
    new = oracle.backward_sgd(pa.part, pa.D, pa.B, pa.T, pa.tables, pa.indices, pa.offsets,
                              grads, -1.0)
    ref_a, ref_b = oracle_out(pa, new)[0], oracle_out(pb, new)[0]
    for rep in range(3):
        h.backward_plan(ia, oa)
        h.backward(g, -1.0)
        oa1 = h.forward(ia, oa)
        ob1 = h.forward(ibd, obd)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(oa1.cpu().numpy(), ref_a)
        np.testing.assert_array_equal(ob1.cpu().numpy(), ref_b)
        h.backward(-g, -1.0)                  # undo the update (exact-int): tables back to start
        x1 = h.forward(ia, oa)
        x2 = h.forward(ibd, obd)
        x3 = h.forward(ia, oa)               # stores into x1's half
        torch.cuda.synchronize()
        np.testing.assert_array_equal(x2.cpu().numpy(), oracle_out(pb)[0])
        np.testing.assert_array_equal(x3.cpu().numpy(), oracle_out(pa)[0])
        assert x1.data_ptr() == x3.data_ptr()
    h.destroy()


# ------------------------------------------------------------------ buffer-reuse credits

def _slow_consumer_run(W, part, T, slow, nfwd=5, opts=None):
    """Rank `slow` consumes each output after a long GPU sleep on its stream; every other rank
    issues forward after forward.  Returns the slow rank's copies and the problems."""
    from paper_2305_06942_b200 import LoopbackGroup
    B = int(part[-1])
    probs = []
    for k in range(nfwd):
        rng = np.random.default_rng(100 + k)
        tables = [rng.integers(-8, 8, size=(37, 8)).astype(np.float32) for _ in range(sum(T))]
        idx, off = [], []
        for r in range(W):
            i, o = csr_from_bags([[list(rng.integers(0, 37, size=rng.integers(0, 6)))
                                   for _ in range(B)] for _ in range(T[r])])
            idx.append(i)
            off.append(o if o.size else np.zeros(1, np.int32))
        probs.append(Problem(W, list(T), 8, B, np.asarray(part, np.int64), tables if k == 0 else
                             probs[0].tables, idx, off))
    g = LoopbackGroup(W, dev(), dict({"slice": 4, "chunk": 2, "timeout_ms": 8000}, **(opts or {})))
    tabs = [[torch.from_numpy(t).to(dev()) for t in probs[0].tables[sum(T[:r]):sum(T[:r + 1])]]
            for r in range(W)]
    g.register_tables(tabs, B, part, dim=8)
    _load_torch_kernels()
    csr = [([torch.from_numpy(i).to(dev()) for i in p.indices],
            [torch.from_numpy(o).to(dev()) for o in p.offsets]) for p in probs]
    cur = torch.cuda.current_stream()
    for s_ in g.streams:
        s_.wait_stream(cur)
    copies = []
    for e in range(nfwd):
        for r, h in enumerate(g.handles):
            st = g.streams[r]
            out = h.forward(csr[e][0][r], csr[e][1][r], stream=st)
            if r == slow:
                with torch.cuda.stream(st):
                    torch.cuda._sleep(20_000_000)
                    copies.append(out.clone())
    for s_ in g.streams:
        cur.wait_stream(s_)
    torch.cuda.synchronize()
    for h in g.handles:
        h.check()
    g.destroy()
    return copies, probs


@pytest.mark.parametrize("case", ["sender_receives_nothing", "sender_owns_tables_only",
                                  "receiver_without_tables"])
def test_credits_bound_run_ahead_of_non_receiving_rank(case):
    """a rank that receives nothing never waits in its receive wait, so
    without backpressure it would run forwards ahead and overwrite the slow rank's receive
    half before the slow rank copied it out.  The credit (the slow rank started the forward that
    reuses the half) bounds it: every copy equals the oracle."""
    if case == "sender_receives_nothing":       # rank 0: b_0 = 0, owns tables
        W, part, T, slow = 2, [0, 0, 8], [2, 1], 1
    elif case == "sender_owns_tables_only":     # rank 1 sends, receives nothing; rank 0 no tables
        W, part, T, slow = 2, [0, 8, 8], [0, 2], 0
    else:                                       # 3 ranks; the slow one owns no tables
        W, part, T, slow = 3, [0, 4, 4, 12], [2, 1, 0], 2
    copies, probs = _slow_consumer_run(W, part, T, slow)
    for e, c in enumerate(copies):
        np.testing.assert_array_equal(c.cpu().numpy(), oracle_out(probs[e])[slow])


def test_backward_credits_table_less_rank_runs_ahead():
    """ADVICE r1 (medium), backward: rank 1 owns no tables, so its backward pushes gradient rows
    and never waits for anything.  Rank 0 (the owner) starts each backward late (GPU sleep).
    Without the backward credit, rank 1's backward e+2 would overwrite the staging half rank 0's
    backward e has not reduced yet.  Tables after 5 steps (different integer gradients each
    step) equal the oracle's 5 sequential SGD steps bitwise."""
    from paper_2305_06942_b200 import LoopbackGroup
    rng = np.random.default_rng(42)
    W, T, B, D, R = 2, [2, 0], 16, 8, 23
    tables = [rng.integers(-8, 8, size=(R, D)).astype(np.float32) for _ in range(2)]
    i0, o0 = csr_from_bags([[list(rng.integers(0, R, size=rng.integers(1, 5))) for _ in range(B)]
                            for _ in range(2)])
    i1, o1 = np.zeros(0, np.int32), np.zeros(1, np.int32)
    p = Problem(W, T, D, B, synth.even_partition(B, W), tables, [i0, i1], [o0, o1])
    g = LoopbackGroup(W, dev(), {"timeout_ms": 8000})
    tabs = [[torch.from_numpy(t.copy()).to(dev()) for t in tables], []]
    g.register_tables(tabs, B, dim=D)
    for h in g.handles:
        h.set_option("bwd_share", W + 1)
    _load_torch_kernels()
    idx = [torch.from_numpy(i0).to(dev()), torch.zeros(1, dtype=torch.int32, device=dev())]
    off = [torch.from_numpy(o0).to(dev()), torch.from_numpy(o1).to(dev())]
    g.handles[0].backward_plan(idx[0], off[0], stream=g.streams[0])
    g.handles[1].backward_plan(idx[1][:0], off[1], stream=g.streams[1])
    torch.cuda.synchronize()
    steps = 5
    grads = [[rng.integers(-4, 4, (B // W, 2 * D)).astype(np.float32) for _ in range(W)]
             for _ in range(steps)]
    dgr = [[torch.from_numpy(x).to(dev()) for x in gs] for gs in grads]
    for e in range(steps):
        with torch.cuda.stream(g.streams[0]):
            torch.cuda._sleep(20_000_000)
        for r, h in enumerate(g.handles):
            h.backward(dgr[e][r], -1.0, stream=g.streams[r])
    torch.cuda.synchronize()
    for h in g.handles:
        h.check()
    want = [t.copy() for t in tables]
    for e in range(steps):
        want = oracle.backward_sgd(p.part, D, B, T, want, p.indices, p.offsets, grads[e], -1.0)
    for t in range(2):
        np.testing.assert_array_equal(tabs[0][t].cpu().numpy(), want[t])
    g.destroy()


def test_forward_host_batch_multi_rank_loopback():
    """The pipelined serving loop at W > 1 (forward_host_batch on every virtual rank): every
    step's host copy equals the oracle (exact-int), over two rounds."""
    from paper_2305_06942_b200 import LoopbackGroup
    cfg = synth.config_for("tiny", W=2, value_mode=1)
    probs = [from_config(cfg, k) for k in range(4)]
    g = LoopbackGroup(2, dev())
    tabs = [[torch.from_numpy(t).to(dev()) for t in probs[0].rank_tables(r)] for r in range(2)]
    g.register_tables(tabs, cfg.B)
    hin = [[(torch.from_numpy(p.indices[r]).pin_memory(), torch.from_numpy(p.offsets[r]).pin_memory())
            for p in probs] for r in range(2)]
    outs = [[torch.zeros((probs[0].b(r), cfg.G * cfg.D), dtype=torch.float32).pin_memory()
             for _ in probs] for r in range(2)]
    from paper_2305_06942_b200 import run_ranks
    for rnd in range(2):
        # the W calls are collective and enqueue only: issue them from W host threads
        run_ranks(lambda r: g.handles[r].forward_host_batch(
            [x[0] for x in hin[r]], [x[1] for x in hin[r]], outs[r], stream=g.streams[r]), 2)
        torch.cuda.synchronize()
        for k, p in enumerate(probs):
            ref = oracle_out(p)
            for r in range(2):
                np.testing.assert_array_equal(outs[r][k].numpy(), ref[r])
                outs[r][k].zero_()
    g.destroy()


# ------------------------------------------------------------------ trace (E1) and counts

@pytest.mark.parametrize("W,S,C", [(2, 4, 0), (4, 7, 0), (2, 4, 16), (4, 7, 20)])
def test_trace_invariance_and_signal_counts(W, S, C):
    """The trace option (P:239-258 per-WG timeline) changes no result: outputs with trace on
    equal the trace-off outputs and the oracle bitwise.  Each rank's trace logs exactly one
    release per remote slice (event 3, payload = slices released by that stage; a chunk C
    longer than a slice S releases several): sum over s != r of T_r * ceil(b_s / S),
    which is also what the destinations' counters grew by."""
    from paper_2305_06942_b200 import LoopbackGroup
    cfg = synth.config_for("tiny", W=W, B=64 if W == 2 else 96)
    p = from_config(cfg, 0)
    ref = oracle_out(p)
    outs = {}
    for trace in (0, 1 << 16):
        opts = {"slice": S, "trace": trace}
        if C:
            opts["chunk"] = C
        g = LoopbackGroup(W, dev(), opts)
        tabs = [[torch.from_numpy(t).to(dev()) for t in p.rank_tables(r)] for r in range(W)]
        g.register_tables(tabs, cfg.B)
        idx = [torch.from_numpy(i).to(dev()) for i in p.indices]
        off = [torch.from_numpy(o).to(dev()) for o in p.offsets]
        nfwd = 3
        for _ in range(nfwd):
            o = g.forward(idx, off)
        outs[trace] = [x.cpu().numpy() for x in o]
        if trace:
            for r, h in enumerate(g.handles):
                tr = h.read_trace()
                assert tr.size < (1 << 16)
                sent = int(tr["payload"][tr["event"] == 3].sum())
                want = sum(oracle.signal_count(r, s, cfg.T, cfg.part, S) for s in range(W) if s != r)
                assert sent == nfwd * want, (r, sent, want)
                # one receive-wait-done record per forward (the last CTA), for W > 1
                assert int((tr["event"] == 5).sum()) == nfwd
            for r, h in enumerate(g.handles):
                fl = h.read_flags()
                for src in range(W):
                    assert int(fl[src]) == nfwd * oracle.signal_count(src, r, cfg.T, cfg.part, S)
        g.destroy()
    for s in range(W):
        np.testing.assert_array_equal(outs[0][s], ref[s])
        np.testing.assert_array_equal(outs[1 << 16][s], outs[0][s])


# ------------------------------------------------------------------ error words, option ranges

def test_sort_lookback_stall_reports_timeout():
    """A broken look-back invariant (debug knob: tile 0 publishes a stale word) must surface as
    EMB_A2A_ETIMEOUT on the next call and poison the handle -- not hang, not go on silently."""
    from paper_2305_06942_b200 import EmbA2AError
    rng = np.random.default_rng(7300)
    B, D, R = 512, 8, 300
    tables = [rng.integers(-8, 8, size=(R, D)).astype(np.float32) for _ in range(2)]
    i, o = csr_from_bags([[list(rng.integers(0, R, size=rng.integers(10, 20))) for _ in range(B)]
                          for _ in range(2)])
    p = Problem(1, [2], D, B, synth.even_partition(B, 1), tables, [i], [o])
    h, _ = _single(p, {"sort_mode": 1, "timeout_ms": 300})
    assert p.indices[0].size > 2 * 2048        # several radix tiles (one look-back group)
    idx = torch.from_numpy(p.indices[0]).to(dev())
    off = torch.from_numpy(p.offsets[0]).to(dev())
    h.backward_plan(idx, off)                  # clean plan first
    torch.cuda.synchronize()
    h.check()
    h.set_option("debug_sort_stall", 1)
    h.backward_plan(idx, off)
    torch.cuda.synchronize()
    with pytest.raises(EmbA2AError) as e:
        h.check()
    assert "ETIMEOUT" in str(e.value) and "look-back" in str(e.value)
    with pytest.raises(EmbA2AError) as e:
        h.backward_plan(idx, off)
    assert "ESTATE" in str(e.value)
    h.destroy()


def test_bwd_threads_option_range():
    """the backward kernel is compiled for at most 128 threads; larger values
    are rejected up front instead of failing every backward with ECUDA."""
    from paper_2305_06942_b200 import EmbA2AError
    p = random_problem(7400, W=1, value_mode=1, max_B=64, max_D=32)
    h, _ = _single(p)
    for bad in (160, 256, 16, 100):
        with pytest.raises(EmbA2AError):
            h.set_option("bwd_threads", bad)
    for ok in (32, 64, 96, 128):
        h.set_option("bwd_threads", ok)
        h.backward_plan(torch.from_numpy(p.indices[0]).to(dev()),
                        torch.from_numpy(p.offsets[0]).to(dev()))
        h.backward(torch.zeros((p.B, p.G * p.D), device=dev()), 1.0)
        torch.cuda.synchronize()
        h.check()
    h.destroy()
