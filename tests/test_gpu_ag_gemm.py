"""GPU parity of the fused AllGather + GEMM against the
oracle (oracle/ag_gemm.py), through the C ABI (include/ag_gemm.h).

Exact-int operands (synth/gemm_gen.py mode 1) make every fp32 partial sum exact, so Y must equal
the oracle's sum rounded once to bf16 (nearest even, R#34) BITWISE, and the fp32-output variant
must equal the exact sum; grid-valued operands (mode 0) are checked against the stated bound
(R#37).  The gathered weight is compared bitwise (routing / layout).  Multi-rank cases run W
virtual ranks on the one GPU (AgGemmLoopback): real flags, credits, waits and peer stores.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import ag_gemm as O  # noqa: E402
from synth import gemm_gen as G  # noqa: E402


def dev():
    return torch.device("cuda:0")


def operands(cfg, r):
    """(X_r, W_r) bf16 on the device, from the device fill (input generator)."""
    from synth.device import fill_gemm_bf16
    X = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device=dev())
    Wr = torch.empty((cfg.N_r, cfg.K), dtype=torch.bfloat16, device=dev())
    fill_gemm_bf16(X, G.X_TENSOR + r, G.GEMM_SEED, cfg.mode)
    fill_gemm_bf16(Wr, G.W_TENSOR + r, G.GEMM_SEED, cfg.mode)
    return X, Wr


def bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def check_rank(cfg, r, Y, Wg, local_copy=False, out_f32=False):
    Xh, _ = G.rank_inputs(cfg, r)
    shards = [G.rank_inputs(cfg, s)[1] for s in range(cfg.W)]
    Wf, Yref = O.ag_gemm(Xh, shards)
    # gathered weight: every remote block (and the own block with local_copy) bitwise
    wg = bits(Wg)
    for s in range(cfg.W):
        if s == r and not local_copy:
            continue
        blk = slice(s * cfg.N_r, (s + 1) * cfg.N_r)
        np.testing.assert_array_equal(wg[blk], G.to_bf16_bits_exact(Wf[blk]), err_msg=f"block {s}")
    if cfg.mode == 1:
        if out_f32:
            np.testing.assert_array_equal(Y.cpu().numpy().astype(np.float64), Yref)
        else:
            np.testing.assert_array_equal(bits(Y), O.bf16_rne_bits(Yref))
    else:
        got = Y.float().cpu().numpy().astype(np.float64)
        bound = O.error_bound(Xh, Wf, out_bits=32 if out_f32 else 16)
        err = np.abs(got - Yref)
        assert np.all(err <= bound), f"max excess {np.max(err - bound)}"


def run_loopback(cfg, opts=None, out_f32=False, forwards=1):
    from paper_2305_06942_b200 import AgGemmLoopback
    grp = AgGemmLoopback(cfg.W, dev(), opts)
    try:
        grp.register(cfg.M, cfg.N_r, cfg.K, torch.float32 if out_f32 else torch.bfloat16)
        ops = [operands(cfg, r) for r in range(cfg.W)]
        outs = None
        for _ in range(forwards):
            outs = grp.forward([o[0] for o in ops], [o[1] for o in ops])
        for r in range(cfg.W):
            check_rank(cfg, r, outs[r][0], outs[r][1], bool((opts or {}).get("local_copy")),
                       out_f32)
        return grp.handles[0].read_flags()
    finally:
        grp.destroy()


def cfg_of(W, M, N_r, K, mode=1):
    return G.GemmConfig("t", W, M, N_r, K, mode)


def test_device_fill_matches_host_generator():
    from synth.device import fill_gemm_bf16
    for mode in (0, 1):
        t = torch.empty((300, 1000), dtype=torch.bfloat16, device=dev())
        fill_gemm_bf16(t, G.W_TENSOR + 5, G.GEMM_SEED, mode, row0=77)
        want = G.to_bf16_bits_exact(G.matrix(G.W_TENSOR + 5, 300, 1000, mode=mode, row0=77))
        np.testing.assert_array_equal(bits(t), want)


@pytest.mark.parametrize("M,N_r,K", [(128, 256, 64), (128, 128, 128), (256, 512, 512),
                                     (384, 384, 192), (640, 768, 1024), (128, 256, 4096)])
def test_single_rank_exact(M, N_r, K):
    run_loopback(cfg_of(1, M, N_r, K))


def test_single_rank_fp32_output_exact():
    run_loopback(cfg_of(1, 256, 512, 512), out_f32=True)


@pytest.mark.parametrize("M,N_r,K", [(256, 512, 512), (512, 1024, 2048)])
def test_single_rank_grid_values_within_bound(M, N_r, K):
    run_loopback(cfg_of(1, M, N_r, K, mode=0))


def test_persistent_loop_small_grid_and_many_forwards():
    """grid 3 < tiles: every CTA walks many tiles through both TMEM accumulators and the ring."""
    run_loopback(cfg_of(1, 512, 1024, 320), opts={"grid": 3}, forwards=3)


def test_local_copy_single_rank():
    run_loopback(cfg_of(1, 128, 256, 128), opts={"local_copy": 1})


@pytest.mark.parametrize("W", [2, 4, 8])
def test_loopback_exact(W):
    flags = run_loopback(cfg_of(W, 256, 512, 512), forwards=1)
    # rank 0 received every remote chunk of epoch 1; its own row is never signalled
    assert (flags[1:] == 1).all() and (flags[0] == 0).all()


@pytest.mark.parametrize("opts", [{"order": 1}, {"piece_kb": 4}, {"grid": 5},
                                  {"local_copy": 1}, {"group_m": 1}])
def test_loopback_tunables_invariant(opts):
    run_loopback(cfg_of(2, 384, 256, 256), opts=dict(opts))


def test_loopback_epochs_double_buffer():
    flags = run_loopback(cfg_of(2, 256, 256, 256), forwards=5)
    assert (flags[1] == 5).all()


def test_loopback_bn128_and_grid_values():
    run_loopback(cfg_of(4, 256, 128, 512, mode=0))


def test_loopback_fp32_output():
    run_loopback(cfg_of(2, 128, 256, 256), out_f32=True)


def test_missing_peer_times_out_then_poisons():
    """comm=0: no chunk is ever signalled, so the first remote tile's wait times out; the next
    call reports ETIMEOUT and the handle is poisoned (no hang, no silent garbage)."""
    from paper_2305_06942_b200 import AgGemmLoopback, EmbA2AError
    cfg = cfg_of(2, 128, 256, 128)
    grp = AgGemmLoopback(2, dev(), {"comm": 0, "timeout_ms": 300})
    try:
        grp.register(cfg.M, cfg.N_r, cfg.K)
        ops = [operands(cfg, r) for r in range(2)]
        with pytest.raises(EmbA2AError) as e:
            grp.forward([o[0] for o in ops], [o[1] for o in ops])
        assert e.value.status == 7
        with pytest.raises(EmbA2AError) as e2:
            grp.handles[0].check()
        assert e2.value.status == 2
    finally:
        grp.destroy()


def test_bad_shapes_rejected():
    from paper_2305_06942_b200 import AgGemm, EmbA2AError, LocalGroup
    h = AgGemm(0, 1, dev(), LocalGroup(1).allgather_for(0))
    try:
        for M, N_r, K in ((100, 256, 64), (128, 200, 64), (128, 256, 100), (0, 256, 64)):
            with pytest.raises(EmbA2AError) as e:
                h.register(M, N_r, K)
            assert e.value.status == 1
    finally:
        h.destroy()


@pytest.mark.parametrize("name,W", [("ag_small", 1), ("ag_small", 2), ("ag_ffn", 1)])
def test_full_size_sampled_entries(name, W):
    """Bench-size problems: sampled Y entries (and sampled gathered rows) against one-at-a-time
    oracle dot products from the generator's rows (grid values: within the R#37 bound)."""
    from paper_2305_06942_b200 import AgGemmLoopback
    cfg = G.gemm_config(name, W, mode=0)
    grp = AgGemmLoopback(W, dev())
    try:
        grp.register(cfg.M, cfg.N_r, cfg.K)
        ops = [operands(cfg, r) for r in range(W)]
        outs = grp.forward([o[0] for o in ops], [o[1] for o in ops])
        rng = np.random.default_rng(17)
        for r in range(W):
            Y, Wg = outs[r]
            m = rng.integers(0, cfg.M, 256)
            n = rng.integers(0, cfg.N, 256)
            xr = G.values(G.X_TENSOR + r, m, np.arange(cfg.K))
            wr = np.stack([G.values(G.W_TENSOR + nn // cfg.N_r, [nn % cfg.N_r], np.arange(cfg.K))[0]
                           for nn in n])
            want = O.ag_gemm_entries(xr, wr)
            got = Y[torch.from_numpy(m).to(dev()), torch.from_numpy(n).to(dev())].float().cpu().numpy()
            absdot = np.einsum("ik,ik->i", np.abs(xr), np.abs(wr))
            bound = 2.0 * cfg.K * 2.0 ** -24 * absdot * (1 + 2 ** -8) + 2.0 ** -8 * np.abs(want)
            assert np.all(np.abs(got - want) <= bound + 1e-30)
            rem = [nn for nn in n if nn // cfg.N_r != r][:32]
            for nn in rem:
                row = bits(Wg[nn:nn + 1])[0]
                ref = G.to_bf16_bits_exact(G.values(G.W_TENSOR + nn // cfg.N_r, [nn % cfg.N_r],
                                                    np.arange(cfg.K))[0])
                np.testing.assert_array_equal(row, ref)
    finally:
        grp.destroy()


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("M,N_r,K,W", [(256, 256, 512, 1), (512, 384, 256, 1), (768, 512, 320, 2),
                                       (256, 128, 128, 4)])
def test_cta_pair_and_single_cta_paths(pair, M, N_r, K, W):
    """tcgen05.mma.cta_group::2 (a CTA pair per 256 x BN tile, each CTA staging half of B) and
    the single-CTA path give the same bitwise result; the query reports which one ran."""
    flags = run_loopback(cfg_of(W, M, N_r, K), opts={"pair": pair, "grid": 6})
    assert flags.shape == (W, N_r // (256 if N_r % 256 == 0 else 128))


def test_pair_query_and_odd_grid():
    from paper_2305_06942_b200 import AgGemm, LocalGroup
    h = AgGemm(0, 1, dev(), LocalGroup(1).allgather_for(0), {"grid": 7})
    try:
        h.register(512, 1024, 128)                                # 2 x 4 pair tiles
        assert h.query("pair") == 1 and h.query("grid") == 6      # even: clusters of two
        h.set_option("pair", 0)
        assert h.query("pair") == 0 and h.query("grid") == 7
        h.register(384, 256, 128)                                 # M % 256 != 0: single CTAs
        h.set_option("pair", 1)
        assert h.query("pair") == 0
    finally:
        h.destroy()
