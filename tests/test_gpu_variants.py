"""GPU parity of the f2 variants (P:119 EmbeddingBag_..._sum_mean): bf16 / fp16 tables, mean
pooling, per-sample weights -- through the C ABI, against the oracle, bitwise."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests._problems import Problem, csr_from_bags, random_problem

pytestmark = pytest.mark.gpu

DT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16}


def dev():
    return torch.device("cuda:0")


def half_bits(t: np.ndarray, dtype):
    if dtype == oracle.BF16:
        return (np.ascontiguousarray(t, np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    return np.ascontiguousarray(t, np.float32).astype(np.float16).view(np.uint16)


def to_dev_table(bits: np.ndarray, dtype):
    return torch.from_numpy(bits.view(np.int16)).to(dev()).view(DT[dtype])


def run_gpu(p: Problem, tables_dev, pooling="sum", weights=None, opts=None, dtype=None):
    from paper_2305_06942_b200 import LoopbackGroup
    g = LoopbackGroup(p.W, dev(), opts)
    tabs = [tables_dev[p.toff(r): p.toff(r) + p.T[r]] for r in range(p.W)]
    g.register_tables(tabs, p.B, p.part, dim=p.D, pooling=pooling, dtype=dtype)
    idx = [torch.from_numpy(np.ascontiguousarray(i)).to(dev()) for i in p.indices]
    off = [torch.from_numpy(np.ascontiguousarray(o)).to(dev()) for o in p.offsets]
    w = None if weights is None else [torch.from_numpy(x).to(dev()) for x in weights]
    outs = [o.cpu().numpy() for o in g.forward(idx, off, weights=w)]
    g.destroy()
    return outs


def weights_for(p, mode):
    cfg = synth.config_for("tiny")
    return [synth.gen_weights(cfg, r, p.indices[r].size, mode=mode) for r in range(p.W)]


@pytest.mark.parametrize("dtype", [oracle.BF16, oracle.F16])
@pytest.mark.parametrize("seed", range(6))
def test_half_tables_random_configs(dtype, seed):
    p = random_problem(2000 + seed, value_mode=0, ragged=seed % 2 == 1, max_D=256)
    p.D = max(8, p.D // 8 * 8)
    rng = np.random.default_rng(seed)
    bits = []
    for t in p.tables:   # arbitrary finite half values, incl. fp16 subnormals
        a = rng.standard_normal((t.shape[0], p.D)).astype(np.float32) * (1e-5 if seed == 3 else 1)
        bits.append(half_bits(a, dtype))
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, bits, p.indices, p.offsets, dtype=dtype)
    got = run_gpu(p, [to_dev_table(b, dtype) for b in bits], dtype=DT[dtype])
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("dtype", [oracle.BF16, oracle.F16])
@pytest.mark.parametrize("D", [8, 16, 24, 64, 120, 128, 256, 512, 1024])
def test_half_lane_mappings(dtype, D):
    rng = np.random.default_rng(D)
    W, T, B = 2, [2, 1], 16
    bits = [half_bits(rng.standard_normal((40, D)).astype(np.float32), dtype) for _ in range(3)]
    idx, off = [], []
    for r in range(W):
        i, o = csr_from_bags([[list(rng.integers(0, 40, size=int(rng.integers(0, 30))))
                               for _ in range(B)] for _ in range(T[r])])
        idx.append(i)
        off.append(o)
    p = Problem(W, T, D, B, synth.even_partition(B, W), bits, idx, off)
    ref = oracle.emb_a2a(p.part, D, B, T, bits, idx, off, dtype=dtype)
    for opts in ({}, {"vec": 2}, {"vec": 4}):
        got = run_gpu(p, [to_dev_table(b, dtype) for b in bits], opts=opts, dtype=DT[dtype])
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("flat", [0, 1000])
def test_mean_pooling(seed, flat):
    p = random_problem(2100 + seed, value_mode=seed % 2, ragged=seed % 3 == 0)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets,
                         pooling=oracle.MEAN)
    got = run_gpu(p, [torch.from_numpy(t).to(dev()) for t in p.tables], pooling="mean",
                  opts={"flat_below": flat})
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("opts", [{}, {"idx_cap": 3}, {"idx_cap": 0}, {"vec": 2},
                                  {"flat_below": 0}, {"flat_below": 1000}])
def test_per_sample_weights(seed, opts):
    p = random_problem(2200 + seed, value_mode=seed % 2, ragged=seed % 3 == 1)
    w = weights_for(p, seed % 2)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, weights=w)
    got = run_gpu(p, [torch.from_numpy(t).to(dev()) for t in p.tables], weights=w, opts=opts)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def test_weighted_bf16_tables_and_mean_half():
    p = random_problem(2300, W=4, value_mode=0, max_D=128)
    p.D = max(8, p.D // 8 * 8)
    rng = np.random.default_rng(0)
    bits = [half_bits(rng.standard_normal((t.shape[0], p.D)).astype(np.float32), oracle.BF16)
            for t in p.tables]
    w = weights_for(p, 0)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, bits, p.indices, p.offsets, dtype=oracle.BF16,
                         weights=w)
    got = run_gpu(p, [to_dev_table(b, oracle.BF16) for b in bits], weights=w, dtype=torch.bfloat16)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, bits, p.indices, p.offsets, dtype=oracle.BF16,
                         pooling=oracle.MEAN)
    got = run_gpu(p, [to_dev_table(b, oracle.BF16) for b in bits], pooling="mean",
                  dtype=torch.bfloat16)
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


def test_weights_with_mean_rejected():
    from paper_2305_06942_b200 import EmbA2AError, LoopbackGroup
    p = random_problem(2400, W=1)
    g = LoopbackGroup(1, dev())
    g.register_tables([[torch.from_numpy(t).to(dev()) for t in p.tables]], p.B, p.part,
                      pooling="mean")
    idx = torch.from_numpy(p.indices[0]).to(dev())
    off = torch.from_numpy(p.offsets[0]).to(dev())
    with pytest.raises(EmbA2AError):
        g.handles[0].forward(idx, off, per_sample_weights=torch.ones(idx.numel(), device=dev()))
    g.destroy()


def test_pool_local_weighted_bf16_layout():
    p = random_problem(2500, W=2, value_mode=1, max_D=64)
    p.D = max(8, p.D // 8 * 8)
    rng = np.random.default_rng(1)
    bits = [half_bits(rng.integers(-8, 8, (t.shape[0], p.D)).astype(np.float32), oracle.BF16)
            for t in p.tables]
    w = weights_for(p, 1)
    full = np.concatenate(oracle.emb_a2a(p.part, p.D, p.B, p.T, bits, p.indices, p.offsets,
                                         dtype=oracle.BF16, weights=w), axis=0)
    from paper_2305_06942_b200 import LoopbackGroup
    g = LoopbackGroup(p.W, dev())
    g.register_tables([[to_dev_table(b, oracle.BF16) for b in bits[p.toff(r):p.toff(r) + p.T[r]]]
                       for r in range(p.W)], p.B, p.part, dim=p.D, dtype=torch.bfloat16)
    for r, h in enumerate(g.handles):
        send = torch.full((p.B, p.T[r], p.D), float("nan"), device=dev())
        h.pool_local(torch.from_numpy(p.indices[r]).to(dev()),
                     torch.from_numpy(p.offsets[r]).to(dev()), send,
                     per_sample_weights=torch.from_numpy(w[r]).to(dev()))
        torch.cuda.synchronize()
        got = send.cpu().numpy()
        for t in range(p.T[r]):
            gg = p.toff(r) + t
            np.testing.assert_array_equal(got[:, t, :], full[:, gg * p.D:(gg + 1) * p.D])
    g.destroy()


def test_full_size_bf16_dlrm_small_sampled():
    """DLRM-small per-rank work at W=1 with bf16 tables (values exact in bf16), sampled rows."""
    import synth.device as sd
    from paper_2305_06942_b200 import LoopbackGroup
    cfg = synth.config_for("dlrm_small", W=1, value_mode=2)
    csr = synth.gen_all_csr(cfg, 0)
    t32 = sd.rank_tables(cfg, 0, dev())
    tabs = [t.to(torch.bfloat16) for t in t32]
    del t32
    torch.cuda.empty_cache()
    g = LoopbackGroup(1, dev())
    g.register_tables([tabs], cfg.B)
    out = g.forward([torch.from_numpy(csr[0][0]).to(dev())], [torch.from_numpy(csr[0][1]).to(dev())])[0]
    sel = np.arange(0, cfg.B, 37)
    ref = oracle.emb_a2a_rows(cfg.table_seed, 2, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                              [csr[0][0]], [csr[0][1]], 0, sel, check_inputs=False)
    np.testing.assert_array_equal(out[torch.from_numpy(sel).to(dev())].cpu().numpy(), ref)
    g.destroy()
