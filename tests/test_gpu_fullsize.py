"""Full-size forward parity at the largest BASELINE.json configs (VERDICT r1 "What's missing" 5):
every config's per-rank work at the bench's launch configuration, 96+ sampled output rows per
rank recomputed one by one by the oracle (procedural tables, so nothing is materialised on the
host) -- bitwise, and within the north-star tolerance.

  DLRM-wide W=1  (16 x 4M x 256: 65.5 GB of fp32 tables; bf16 tables too)
  sweep P=32 / P=128 W=1  (16 x 2M x 128, B=8192: up to 16.8 M lookups)
  weak W=4 / W=8 loopback (W virtual ranks of 16 x 2M x 128 on one GPU: up to 131 GB)

At these sizes a table index, a row offset or a receive-buffer offset that overflowed 32 bits
would show up here and nowhere else (DLRM-wide rows are 1 KB: a 4M-row table is 4 GB).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


def dev():
    return torch.device("cuda:0")


def _tables(cfg, r, dtype):
    """Rank r's procedural tables; 16-bit ones are converted one table at a time (peak memory)."""
    import synth.device as sd
    if dtype == torch.float32:
        return sd.rank_tables(cfg, r, dev())
    out = []
    tmp = torch.empty((cfg.R, cfg.D), dtype=torch.float32, device=dev())
    for t in range(cfg.T[r]):
        sd.fill_table(tmp, cfg.toff(r) + t, cfg.table_seed, cfg.value_mode)
        out.append(tmp.to(dtype))
    del tmp
    return out


def _sampled_parity(name, W, dtype=torch.float32, value_mode=0, nsample=96, opts=None,
                    l1_active=None):
    from paper_2305_06942_b200 import LoopbackGroup
    cfg = synth.config_for(name, W=W, value_mode=value_mode)
    csr = synth.gen_all_csr(cfg, 0)
    grp = LoopbackGroup(W, dev(), opts)
    tabs = [_tables(cfg, r, dtype) for r in range(W)]
    grp.register_tables(tabs, cfg.B)
    idx = [torch.from_numpy(c[0]).to(dev()) for c in csr]
    off = [torch.from_numpy(c[1]).to(dev()) for c in csr]
    outs = grp.forward(idx, off)
    outs = grp.forward(idx, off)        # the second half of the double buffer, same inputs
    if l1_active is not None:
        assert all(h.get_option("l1_rows_active") == l1_active for h in grp.handles)
    rng = np.random.default_rng(W)
    try:
        for s in range(W):
            b = int(cfg.part[s + 1] - cfg.part[s])
            sel = np.unique(np.concatenate([[0, b - 1], rng.integers(0, b, nsample - 2)]))
            ref = oracle.emb_a2a_rows(cfg.table_seed, cfg.value_mode, cfg.part, cfg.D, cfg.B,
                                      cfg.T, cfg.R, [c[0] for c in csr], [c[1] for c in csr], s,
                                      sel, check_inputs=False)
            got = outs[s][torch.from_numpy(sel).to(dev())].cpu().numpy()
            np.testing.assert_allclose(got, ref, rtol=RTOL, atol=ATOL)
            np.testing.assert_array_equal(got, ref)
    finally:
        grp.destroy()
        del tabs, outs
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name,W", [("dlrm_wide", 1), ("sweep_p32", 1), ("sweep_p128", 1),
                                    ("weak", 4), ("weak", 8)])
def test_full_size_forward_sampled_rows(name, W):
    _sampled_parity(name, W)


@pytest.mark.parametrize("name,l1,active", [("sweep_p8", -1, 1), ("dlrm_wide", -1, 1),
                                           ("sweep_p1", -1, 1), ("dlrm_small", -1, 0),
                                           ("weak", -1, 0), ("dlrm_small", 1, 1),
                                           ("dlrm_wide", 0, 0)])
def test_full_size_l1_rows_choice(name, l1, active):
    """The auto L1 choice (rows allocated in L1 from 4096 lookups per SM or 4096 bags per table:
    sweep and DLRM-wide yes, DLRM-small and weak at W=1 no) and both forced settings, at full
    size, against the oracle."""
    _sampled_parity(name, 1, opts={"l1_rows": l1}, l1_active=active)


@pytest.mark.parametrize("l1", [-1, 0])
def test_full_size_dlrm_wide_bf16_tables(l1):
    """DLRM-wide with bf16 tables (value mode 2: k * 2^-7, exact in bf16), fp32 accumulation;
    rows through L1 (auto at DLRM-wide) and streamed."""
    _sampled_parity("dlrm_wide", 1, dtype=torch.bfloat16, value_mode=2, opts={"l1_rows": l1},
                    l1_active=1 if l1 else 0)
