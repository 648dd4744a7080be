"""Pins for the AllGather + GEMM oracle (oracle/ag_gemm.py).

Each check compares the oracle with something other than itself: a hand-worked example, Python
integer brute force, closed forms (identity / constant / one-hot operands), torch's own bf16
cast, and a simulated fp32 accumulation against the stated error bound (and a deliberately
wrong result against it).  CPU only.
"""
import json
import os

import numpy as np
import pytest

from oracle import ag_gemm as O
from synth import gemm_gen as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ag_gemm_hand.json")


def test_hand_example():
    g = json.load(open(GOLDEN))
    shards = [np.array(s, dtype=np.float64) for s in g["shards"]]
    Wf, Y = O.ag_gemm(np.array(g["X_0"], dtype=np.float64), shards)
    np.testing.assert_array_equal(Wf, np.array(g["W_gathered"]))
    np.testing.assert_array_equal(Y, np.array(g["Y_0"]))


@pytest.mark.parametrize("W,Nr,K,M", [(1, 3, 5, 2), (2, 2, 7, 3), (3, 1, 4, 4), (4, 3, 2, 1)])
def test_brute_force_python_ints(W, Nr, K, M):
    rng = np.random.default_rng(100 * W + K)
    X = rng.integers(-9, 10, size=(M, K))
    shards = [rng.integers(-9, 10, size=(Nr, K)) for _ in range(W)]
    Wf, Y = O.ag_gemm(X.astype(np.float64), [s.astype(np.float64) for s in shards])
    for s in range(W):
        for i in range(Nr):
            for k in range(K):
                assert Wf[s * Nr + i][k] == int(shards[s][i][k])
    for m in range(M):
        for s in range(W):
            for i in range(Nr):
                acc = 0
                for k in range(K):
                    acc += int(X[m][k]) * int(shards[s][i][k])
                assert Y[m][s * Nr + i] == acc


def test_identity_activations_give_the_transposed_weight():
    K, W, Nr = 6, 3, 2
    rng = np.random.default_rng(7)
    shards = [rng.integers(-5, 6, size=(Nr, K)).astype(np.float64) for _ in range(W)]
    Wf, Y = O.ag_gemm(np.eye(K), shards)
    assert Y.shape == (K, W * Nr)
    for n in range(W * Nr):
        for k in range(K):
            assert Y[k][n] == shards[n // Nr][n % Nr][k]


def test_rank_order_constant_shards():
    """Shard s filled with s + 1: column block s of Y is (s + 1) * rowsum(X) -- a swapped or
    mis-offset rank block fails."""
    M, K, W, Nr = 3, 5, 4, 2
    X = np.arange(M * K, dtype=np.float64).reshape(M, K) - 6
    shards = [np.full((Nr, K), s + 1.0) for s in range(W)]
    _, Y = O.ag_gemm(X, shards)
    rs = X.sum(axis=1)
    for s in range(W):
        for i in range(Nr):
            np.testing.assert_array_equal(Y[:, s * Nr + i], (s + 1) * rs)


def test_one_hot_weights_select_columns():
    """Gathered row n is e_{(3n+1) mod K}: Y[m][n] = X[m][(3n+1) mod K] (an index or transpose
    slip selects the wrong column)."""
    M, K, W, Nr = 4, 7, 2, 5
    shards = []
    for s in range(W):
        sh = np.zeros((Nr, K))
        for i in range(Nr):
            sh[i, (3 * (s * Nr + i) + 1) % K] = 1.0
        shards.append(sh)
    X = np.arange(M * K, dtype=np.float64).reshape(M, K) * 1.5
    _, Y = O.ag_gemm(X, shards)
    for m in range(M):
        for n in range(W * Nr):
            assert Y[m][n] == X[m][(3 * n + 1) % K]


def test_sampled_entries_match_the_dense_result():
    cfg = G.gemm_config("ag_tiny", 2, mode=1)
    X0, W0 = G.rank_inputs(cfg, 0)
    _, W1 = G.rank_inputs(cfg, 1)
    Wf, Y = O.ag_gemm(X0, [W0, W1])
    rng = np.random.default_rng(3)
    m = rng.integers(0, cfg.M, 50)
    n = rng.integers(0, cfg.N, 50)
    # brute force with Python ints for the sampled pairs (exact-int mode)
    for mi, ni in zip(m[:10], n[:10]):
        acc = sum(int(a) * int(b) for a, b in zip(X0[mi], Wf[ni]))
        assert Y[mi, ni] == acc
    np.testing.assert_array_equal(O.ag_gemm_entries(X0[m], Wf[n]), Y[m, n])


def test_bf16_rne_matches_torch_cast():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    f = rng.standard_normal(200_000).astype(np.float32) * np.float32(2.0) ** rng.integers(-20, 20, 200_000).astype(np.float32)
    # ties: bf16 value + exactly half an ulp, both parities of the kept lsb
    base = rng.integers(0, 1 << 15, 20_000).astype(np.uint32) << np.uint32(16)
    ties = (base | np.uint32(0x8000)).view(np.float32)
    ints = np.arange(-(1 << 20), 1 << 20, 37).astype(np.float32)   # exact integers (exact-int mode)
    vals = np.concatenate([f, ties, ints, np.float32([0.0, -0.0, 1.0, -1.0, 255.0, 257.0, 259.0])])
    vals = vals[np.isfinite(vals)]
    ours = O.bf16_rne_bits(vals.astype(np.float64))
    ref = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)
    np.testing.assert_array_equal(O.bf16_bits_to_f64(ours),
                                  torch.from_numpy(vals).to(torch.bfloat16).double().numpy())


def test_bf16_rne_hand_ties():
    # 257 = 1.00000001b * 2^8: halfway between 256 and 258 -> ties to even mantissa: 256
    # 259 = halfway between 258 and 260 -> 260 (258 has odd mantissa lsb)
    assert O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([257.0, 259.0, -257.0])))[0] == 256.0
    assert O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([259.0])))[0] == 260.0
    assert O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([-257.0])))[0] == -256.0


def test_error_bound_holds_for_fp32_accumulation_and_rejects_a_dropped_term():
    """A float32 accumulation of the exact products in a shuffled order (any order the tensor
    core may use), rounded to bf16, stays inside error_bound; the same sum with one term
    dropped does not (for some entry)."""
    cfg = G.gemm_config("ag_tiny", 1, mode=0)
    X, W0 = G.rank_inputs(cfg, 0)
    X, W0 = X[:16], W0[:64]
    Y = O.gemm_nt(X, W0)
    bound = O.error_bound(X, W0, out_bits=16)
    rng = np.random.default_rng(5)
    bad = False
    for m in range(X.shape[0]):
        for n in range(W0.shape[0]):
            prods = (X[m] * W0[n]).astype(np.float32)          # exact: 7x7-bit products
            order = rng.permutation(len(prods))
            acc = np.float32(0.0)
            for k in order:
                acc = np.float32(acc + prods[k])
            y16 = O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([float(acc)])))[0]
            assert abs(y16 - Y[m, n]) <= bound[m, n]
            drop = float(acc) - float(prods[order[0]])
            y16d = O.bf16_bits_to_f64(O.bf16_rne_bits(np.array([float(np.float32(drop))])))[0]
            bad |= abs(y16d - Y[m, n]) > bound[m, n]
    assert bad


def test_generator_values_are_bf16_exact_and_in_range():
    for mode, lo, hi in ((0, -1.0, 1.0 - 2 ** -6), (1, -4.0, 3.0)):
        v = G.matrix(G.W_TENSOR + 3, 64, 300, mode=mode)
        assert v.min() >= lo and v.max() <= hi
        G.to_bf16_bits_exact(v)                      # raises if any value is not bf16-exact
        assert len(np.unique(v)) == (128 if mode == 0 else 8)
    a = G.matrix(G.X_TENSOR, 4, 8)
    b = G.values(G.X_TENSOR, np.arange(2, 4), np.arange(8))
    np.testing.assert_array_equal(a[2:4], b)        # counter-based: any row slice agrees
    assert not np.array_equal(G.matrix(G.X_TENSOR, 4, 8), G.matrix(G.X_TENSOR + 1, 4, 8))
