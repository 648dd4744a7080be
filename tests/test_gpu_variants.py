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
    for opts in ({}, {"vec": 2}, {"vec": 4}, {"l1_rows": 1}, {"l1_rows": 1, "vec": 4},
                 {"l1_rows": 1, "flat_below": 1000}):
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


# ------------------------------------------------------------------ 16-bit output (R#32)

OUT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16}


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("out_dtype", [oracle.BF16, oracle.F16])
@pytest.mark.parametrize("seed", range(8))
def test_half_output_random_configs(out_dtype, seed):
    """fp32 tables, bf16 / fp16 output (option "out_dtype"): every element is the oracle's fp32
    sum rounded once to nearest even -- bitwise, across W in {1,2,4,8}, ragged partitions,
    lane mappings D = 4..256, both pooling loops."""
    from paper_2305_06942_b200 import LoopbackGroup
    p = random_problem(4000 + seed, value_mode=0, ragged=seed % 2 == 1, max_D=256)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets, out_dtype=out_dtype)
    opts = {"out_dtype": out_dtype}
    if seed % 3 == 2:
        opts.update({"flat_below": 1 << 20, "slice": 5})
    g = LoopbackGroup(p.W, dev(), opts)
    g.register_tables([[torch.from_numpy(t).to(dev()) for t in p.rank_tables(r)] for r in range(p.W)],
                      p.B, p.part, dim=p.D)
    idx = [torch.from_numpy(i).to(dev()) for i in p.indices]
    off = [torch.from_numpy(o).to(dev()) for o in p.offsets]
    for rep in range(2):       # both halves of the (half-size) double buffer
        outs = g.forward(idx, off)
        for s, o in enumerate(outs):
            assert o.dtype == OUT[out_dtype] and tuple(o.shape) == ref[s].shape
            np.testing.assert_array_equal(_bits(o), ref[s])
    g.destroy()


@pytest.mark.parametrize("tdt,odt,pooling,weighted", [
    (oracle.BF16, oracle.BF16, "sum", False), (oracle.F16, oracle.F16, "mean", False),
    (oracle.BF16, oracle.F16, "sum", True), (oracle.F32, oracle.BF16, "mean", False),
    (oracle.F32, oracle.F16, "sum", True)])
def test_half_output_variants(tdt, odt, pooling, weighted):
    """16-bit output combined with 16-bit tables, mean pooling and per-sample weights."""
    from paper_2305_06942_b200 import LoopbackGroup
    p = random_problem(4100 + 3 * tdt + odt, W=2, value_mode=0, max_D=128)
    p.D = max(8, p.D // 8 * 8)
    rng = np.random.default_rng(3)
    if tdt == oracle.F32:
        tabs = [rng.standard_normal((t.shape[0], p.D)).astype(np.float32) for t in p.tables]
        dev_tabs = [torch.from_numpy(t).to(dev()) for t in tabs]
    else:
        tabs = [half_bits(rng.standard_normal((t.shape[0], p.D)).astype(np.float32), tdt)
                for t in p.tables]
        dev_tabs = [to_dev_table(b, tdt) for b in tabs]
    w = weights_for(p, 0) if weighted else None
    pm = oracle.MEAN if pooling == "mean" else oracle.SUM
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, tabs, p.indices, p.offsets, dtype=tdt, weights=w,
                         pooling=pm, out_dtype=odt)
    g = LoopbackGroup(p.W, dev(), {"out_dtype": odt})
    g.register_tables([dev_tabs[p.toff(r):p.toff(r) + p.T[r]] for r in range(p.W)], p.B, p.part,
                      dim=p.D, pooling=pooling)
    idx = [torch.from_numpy(i).to(dev()) for i in p.indices]
    off = [torch.from_numpy(o).to(dev()) for o in p.offsets]
    outs = g.forward(idx, off, weights=None if w is None else [torch.from_numpy(x).to(dev()) for x in w])
    for s, o in enumerate(outs):
        np.testing.assert_array_equal(_bits(o), ref[s])
    # the unfused baseline's pool kernel writes the same type, dest-major
    full = np.concatenate(ref, axis=0)
    for r, h in enumerate(g.handles):
        send = torch.zeros((p.B, p.T[r], p.D), dtype=OUT[odt], device=dev())
        h.pool_local(idx[r], off[r], send,
                     per_sample_weights=None if w is None else torch.from_numpy(w[r]).to(dev()))
        torch.cuda.synchronize()
        got = _bits(send)
        for t in range(p.T[r]):
            gg = p.toff(r) + t
            np.testing.assert_array_equal(got[:, t, :], full[:, gg * p.D:(gg + 1) * p.D])
    g.destroy()


def test_half_output_host_paths_and_rejections():
    """forward_host / forward_host_batch copy 16-bit results into 16-bit host buffers; ranks
    disagreeing on out_dtype fail registration together; out_dtype cannot change after it."""
    from paper_2305_06942_b200 import EmbA2A, EmbA2AError, LocalGroup, LoopbackGroup
    p = random_problem(4200, W=1, value_mode=1, max_B=64, max_D=64)
    ref = oracle.emb_a2a(p.part, p.D, p.B, p.T, p.tables, p.indices, p.offsets,
                         out_dtype=oracle.BF16)[0]
    h = EmbA2A(0, 1, dev(), LocalGroup(1).allgather_for(0), {"out_dtype": oracle.BF16})
    h.register_tables([torch.from_numpy(t).to(dev()) for t in p.tables], p.B)
    hi = torch.from_numpy(p.indices[0]).pin_memory()
    ho = torch.from_numpy(p.offsets[0]).pin_memory()
    out = torch.zeros((p.B, p.G * p.D), dtype=torch.bfloat16).pin_memory()
    h.forward_host(hi, ho, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.view(torch.int16).numpy().view(np.uint16), ref)
    outs = [torch.zeros_like(out).pin_memory() for _ in range(3)]
    h.forward_host_batch([hi] * 3, [ho] * 3, outs)
    torch.cuda.synchronize()
    for o in outs:
        np.testing.assert_array_equal(o.view(torch.int16).numpy().view(np.uint16), ref)
    with pytest.raises(ValueError):          # a float32 host buffer for a bf16 output
        h.forward_host(hi, ho, torch.zeros((p.B, p.G * p.D)).pin_memory())
    with pytest.raises(EmbA2AError):
        h.set_option("out_dtype", oracle.F32)
    h.destroy()
    q = random_problem(4201, W=2, value_mode=1, max_B=16, max_D=16)
    g = LoopbackGroup(2, dev())
    g.handles[1].set_option("out_dtype", oracle.F16)
    with pytest.raises(EmbA2AError):
        g.register_tables([[torch.from_numpy(t).to(dev()) for t in q.rank_tables(r)]
                           for r in range(2)], q.B, q.part, dim=q.D)
    g.destroy()


def test_full_size_half_output_dlrm_small_sampled():
    """DLRM-small per-rank work at W=1, bf16 output, sampled rows vs the rounded oracle."""
    import synth.device as sd
    from paper_2305_06942_b200 import LoopbackGroup
    cfg = synth.config_for("dlrm_small", W=1)
    csr = synth.gen_all_csr(cfg, 0)
    g = LoopbackGroup(1, dev(), {"out_dtype": oracle.BF16})
    g.register_tables([sd.rank_tables(cfg, 0, dev())], cfg.B)
    out = g.forward([torch.from_numpy(csr[0][0]).to(dev())], [torch.from_numpy(csr[0][1]).to(dev())])[0]
    sel = np.arange(0, cfg.B, 41)
    ref = oracle.emb_a2a_rows(cfg.table_seed, cfg.value_mode, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                              [csr[0][0]], [csr[0][1]], 0, sel, check_inputs=False,
                              out_dtype=oracle.BF16)
    np.testing.assert_array_equal(_bits(out[torch.from_numpy(sel).to(dev())]), ref)
    g.destroy()
