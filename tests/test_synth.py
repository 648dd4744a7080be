"""The seeded input generator: determinism and distribution."""
import numpy as np

import synth


def test_same_seed_same_bytes_and_batches_differ():
    cfg = synth.config_for("tiny")
    a = synth.gen_all_csr(cfg, 0)
    b = synth.gen_all_csr(cfg, 0)
    c = synth.gen_all_csr(cfg, 1)
    for (ia, oa), (ib, ob) in zip(a, b):
        assert ia.tobytes() == ib.tobytes() and oa.tobytes() == ob.tobytes()
    assert any(ia.tobytes() != ic.tobytes() for (ia, _), (ic, _) in zip(a, c))


def test_csr_shapes_and_ranges():
    cfg = synth.config_for("dlrm_small", W=2, R=5000)   # reduced R for speed
    for r in range(cfg.W):
        idx, off = synth.gen_rank_csr(cfg, r)
        assert off.dtype == np.int32 and idx.dtype == np.int32
        assert off.size == cfg.T[r] * cfg.B + 1 and off[0] == 0 and off[-1] == idx.size
        L = np.diff(off)
        assert L.min() >= 1 and L.max() <= 39
        assert abs(L.mean() - 20) < 0.5                   # mean pooling ~ Pbar
        assert idx.min() >= 0 and idx.max() < cfg.R


def test_fixed_pooling_factor():
    cfg = synth.config_for("tiny")
    idx, off = synth.gen_rank_csr(cfg, 0)
    assert np.all(np.diff(off) == 4)


def test_zipf_rank_frequency_slope():
    """log-frequency vs log-rank slope of the top ranks ~ -alpha.  The rank -> row bijection
    (A, C drawn per (batch, table) substream) only renames rows, so the sorted row frequencies of
    one (batch, table) draw are the rank frequencies."""
    cfg = synth.config_for("dlrm_small", W=1, R=100_000, B=20000)
    L, rows = synth.dlrm_gen.gen_table_bags(cfg, 0, 0)
    cnt = np.sort(np.bincount(rows, minlength=cfg.R))[::-1].astype(np.float64)
    k = np.arange(1, 101)
    slope = np.polyfit(np.log(k), np.log(cnt[:100]), 1)[0]
    assert abs(slope + 1.05) < 0.15, slope


def test_uniform_control_alpha0():
    cfg = synth.config_for("dlrm_small", W=1, R=1000, B=4000, alpha=0.0)
    _, rows = synth.dlrm_gen.gen_table_bags(cfg, 0, 0)
    cnt = np.bincount(rows, minlength=cfg.R)
    assert cnt.max() < 3 * cnt.mean()


def test_table_values_host_modes():
    v = synth.table_values_host(7, 0, 3, 100, 16)
    assert v.dtype == np.float32 and v.shape == (100, 16)
    assert v.min() >= -1 and v.max() < 1 and abs(v.mean()) < 0.05
    w = synth.table_values_host(7, 1, 3, 100, 16)
    assert set(np.unique(w).tolist()) <= set(range(-8, 8))


def test_weak_scaling_batch_grows_with_w():
    for W in (1, 2, 4, 8):
        cfg = synth.config_for("weak", W=W)
        assert cfg.B == 1024 * W and cfg.part[1] - cfg.part[0] == 1024
