"""Pins for the oracle's backward + SGD update (f3) against torch autograd and closed forms."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from tests._problems import Problem, csr_from_bags, random_problem


def grads_for(p: Problem, seed, mode):
    rng = np.random.default_rng(seed)
    out = []
    for s in range(p.W):
        b = p.b(s)
        if mode == 1:
            out.append(rng.integers(-4, 4, (b, p.G * p.D)).astype(np.float32))
        else:
            out.append((rng.integers(-(1 << 20), 1 << 20, (b, p.G * p.D)) * 2.0 ** -20).astype(np.float32))
    return out


def torch_table_grads(p: Problem, grad, mode="sum", weights=None):
    """Autograd of L = sum(out * grad) through F.embedding_bag per table: dL/dW_g."""
    full = np.concatenate(grad, axis=0)             # [B, G*D] in global row order
    res = []
    for r in range(p.W):
        for t in range(p.T[r]):
            g = p.toff(r) + t
            Wt = torch.from_numpy(p.tables[g].astype(np.float64)).requires_grad_(True)
            off = p.offsets[r][t * p.B:(t + 1) * p.B + 1].astype(np.int64)
            idx = torch.from_numpy(p.indices[r][off[0]:off[-1]].astype(np.int64))
            psw = None if weights is None else torch.from_numpy(
                weights[r][off[0]:off[-1]].astype(np.float64))
            out = F.embedding_bag(idx, Wt, torch.from_numpy(off - off[0]), mode=mode,
                                  include_last_offset=True, per_sample_weights=psw)
            (out * torch.from_numpy(full[:, g * p.D:(g + 1) * p.D].astype(np.float64))).sum().backward()
            res.append(Wt.grad.numpy())
    return res


def run_grad(p, grad, **kw):
    """gradient = backward_sgd on zero tables with lr = -1 (W' = 0 - fl(-1 * acc) = acc)."""
    zero = [np.zeros_like(t) for t in p.tables]
    return oracle.backward_sgd(p.part, p.D, p.B, p.T, zero, p.indices, p.offsets, grad, -1.0, **kw)


@pytest.mark.parametrize("seed", range(6))
def test_gradient_equals_torch_autograd_exact_int(seed):
    """Integer grads: every sum is exact, so the oracle's gradient equals autograd's bitwise."""
    p = random_problem(3000 + seed, value_mode=1, ragged=seed % 2 == 1, max_B=64, max_D=32)
    grad = grads_for(p, seed, 1)
    got = run_grad(p, grad)
    for a, b in zip(got, torch_table_grads(p, grad)):
        np.testing.assert_array_equal(a, b.astype(np.float32))


def test_weighted_and_mean_gradients_vs_autograd():
    p = random_problem(3100, value_mode=0, max_B=64, max_D=32)
    grad = grads_for(p, 1, 0)
    cfg = synth.config_for("tiny")
    w = [synth.gen_weights(cfg, r, p.indices[r].size) for r in range(p.W)]
    for kw, mode, ww in (({"weights": w}, "sum", w), ({"pooling": oracle.MEAN}, "mean", None)):
        got = run_grad(p, grad, **kw)
        for a, b in zip(got, torch_table_grads(p, grad, mode, ww)):
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_sgd_update_closed_form_single_occurrence():
    """A row used exactly once gets W - lr * g; unused rows are untouched (bitwise)."""
    D, B = 4, 4
    tab = np.arange(40, dtype=np.float32).reshape(10, D) / 8
    i, o = csr_from_bags([[[3], [7, 3], [], [5]]])
    p = Problem(1, [1], D, B, np.array([0, B]), [tab], [i], [o])
    g = np.array([[1, 2, 3, 4], [10, 20, 30, 40], [9, 9, 9, 9], [0.5, 0.25, -1, 2]], np.float32)
    new = oracle.backward_sgd(p.part, D, B, [1], [tab], [i], [o], [g], 0.5)[0]
    want = tab.copy()
    want[3] = tab[3] - np.float32(0.5) * (g[0] + g[1])
    want[7] = tab[7] - np.float32(0.5) * g[1]
    want[5] = tab[5] - np.float32(0.5) * g[3]
    np.testing.assert_array_equal(new, want)


def test_ascending_occurrence_order_is_the_definition():
    """Three occurrences of one row: acc = ((+0 + c0) + c1) + c2 in position order."""
    D, B = 1, 3
    tab = np.zeros((2, 1), np.float32)
    i, o = csr_from_bags([[[1], [1], [1]]])
    g = np.array([[1e8], [1.0], [-1e8]], np.float32)
    new = oracle.backward_sgd([0, B], D, B, [1], [tab], [i], [o], [g], -1.0)[0]
    want = np.float32(np.float32(np.float32(0) + np.float32(1e8)) + np.float32(1.0)) + np.float32(-1e8)
    assert new[1, 0] == want and new[0, 0] == 0
