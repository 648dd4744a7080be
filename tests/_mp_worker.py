"""Worker bodies for multi-process tests (spawned; must be importable)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def init_gloo(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def cpu_allgather_worker(rank, world, port, q):
    """Host logic of the N>1 path on CPU: the torch.distributed bootstrap all-gather and the
    per-rank sampled oracle check that bench/tests use (each rank checks its own rows)."""
    import numpy as np
    dist = init_gloo(rank, world, port)
    from paper_2305_06942_b200.emb_a2a import torch_allgather   # noqa: E402
    import oracle
    import synth
    ag = torch_allgather()
    payload = bytes([rank]) * 7
    out = ag(payload)
    ok_ag = out == b"".join(bytes([r]) * 7 for r in range(world))
    cfg = synth.config_for("tiny", W=world)
    csr = synth.gen_all_csr(cfg, 0)
    tabs = [synth.table_values_host(cfg.table_seed, 0, g, cfg.R, cfg.D) for g in range(cfg.G)]
    full = oracle.emb_a2a(cfg.part, cfg.D, cfg.B, cfg.T, tabs, [c[0] for c in csr],
                          [c[1] for c in csr])
    b = int(cfg.part[rank + 1] - cfg.part[rank])
    mine = oracle.emb_a2a_rows(cfg.table_seed, 0, cfg.part, cfg.D, cfg.B, cfg.T, cfg.R,
                               [c[0] for c in csr], [c[1] for c in csr], rank, np.arange(b))
    ok_rows = bool(np.array_equal(mine, full[rank]))
    # max-over-ranks reduction as bench.py does it
    import torch
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok_max = float(t.item()) == float(world)
    q.put((rank, ok_ag, ok_rows, ok_max))
    dist.destroy_process_group()


def gpu_ipc_worker(rank, world, port, q):
    """Real cross-process cudaIpc path: W processes on ONE GPU, gloo bootstrap."""
    import numpy as np
    import torch
    dist = init_gloo(rank, world, port)
    import oracle
    import synth
    from paper_2305_06942_b200 import EmbA2A, torch_allgather
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = synth.config_for("tiny", W=world)
    csr = synth.gen_all_csr(cfg, 0)
    tabs_host = [synth.table_values_host(cfg.table_seed, 0, g, cfg.R, cfg.D) for g in range(cfg.G)]
    h = EmbA2A(rank, world, dev, torch_allgather(), {"timeout_ms": 60000, "slice": 5})
    mine = [torch.from_numpy(tabs_host[cfg.toff(rank) + t]).to(dev) for t in range(cfg.T[rank])]
    h.register_tables(mine, cfg.B)
    ref = oracle.emb_a2a(cfg.part, cfg.D, cfg.B, cfg.T, tabs_host, [c[0] for c in csr],
                         [c[1] for c in csr])
    idx = torch.from_numpy(csr[rank][0]).to(dev)
    off = torch.from_numpy(csr[rank][1]).to(dev)
    ok = True
    for e in range(3):
        out = h.forward(idx, off)
        torch.cuda.synchronize()
        ok &= bool(np.array_equal(out.cpu().numpy(), ref[rank]))
    flags = h.read_flags()
    ok_flags = all(int(flags[src]) == 3 * oracle.signal_count(src, rank, cfg.T, cfg.part, 5)
                   for src in range(world))
    # backward (f3) across processes: gradient rows pushed into the peer's IPC-mapped staging,
    # counters across the process boundary; two steps against the oracle (integer gradients:
    # every sum is exact, so the updated tables are bitwise equal)
    rng = np.random.default_rng(77)
    cur = [t.copy() for t in tabs_host]
    ok_bwd = True
    for step in range(2):
        grads = [rng.integers(-4, 4, (int(cfg.part[s + 1] - cfg.part[s]), cfg.G * cfg.D))
                 .astype(np.float32) for s in range(world)]
        cur = oracle.backward_sgd(cfg.part, cfg.D, cfg.B, cfg.T, cur, [c[0] for c in csr],
                                  [c[1] for c in csr], grads, -1.0)
        h.backward_plan(idx, off)
        h.backward(torch.from_numpy(grads[rank]).to(dev), -1.0)
        torch.cuda.synchronize()
        h.check()
        for t in range(cfg.T[rank]):
            ok_bwd &= bool(np.array_equal(mine[t].cpu().numpy(), cur[cfg.toff(rank) + t]))
    h.destroy()
    q.put((rank, ok and ok_bwd, ok_flags))
    dist.destroy_process_group()


def gpu_ag_ipc_worker(rank, world, port, q):
    """Fused AllGather + GEMM across processes on ONE GPU: each process maps
    the other's gather buffer with cudaIpcOpenMemHandle; exact-int operands, three forwards
    (both buffer halves, credits across the process boundary), bitwise against the oracle."""
    import numpy as np
    import torch
    dist = init_gloo(rank, world, port)
    from oracle import ag_gemm as O
    from synth import gemm_gen as G
    from synth.device import fill_gemm_bf16
    from paper_2305_06942_b200 import AgGemm, torch_allgather
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = G.GemmConfig("mp", world, 256, 256, 512, 1)
    X = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device=dev)
    Wr = torch.empty((cfg.N_r, cfg.K), dtype=torch.bfloat16, device=dev)
    fill_gemm_bf16(X, G.X_TENSOR + rank, G.GEMM_SEED, 1)
    fill_gemm_bf16(Wr, G.W_TENSOR + rank, G.GEMM_SEED, 1)
    h = AgGemm(rank, world, dev, torch_allgather(), {"timeout_ms": 60000})
    h.register(cfg.M, cfg.N_r, cfg.K)
    shared = h.query("shared_gpu") == 1
    ok = True
    Xh, _ = G.rank_inputs(cfg, rank)
    Wf, Yref = O.ag_gemm(Xh, [G.rank_inputs(cfg, s)[1] for s in range(world)])
    for _ in range(3):
        Y, Wg = h.forward(X, Wr)
        torch.cuda.synchronize()
        h.check()
        ok &= bool(np.array_equal(Y.view(torch.int16).cpu().numpy().view(np.uint16),
                                  O.bf16_rne_bits(Yref)))
        wg = Wg.view(torch.int16).cpu().numpy().view(np.uint16)
        for s in range(world):
            if s != rank:
                blk = slice(s * cfg.N_r, (s + 1) * cfg.N_r)
                ok &= bool(np.array_equal(wg[blk], G.to_bf16_bits_exact(Wf[blk])))
        dist.barrier()
    flags = h.read_flags()
    ok_flags = bool(all((flags[s] == 3).all() for s in range(world) if s != rank))
    h.destroy()
    q.put((rank, ok and shared, ok_flags))
    dist.destroy_process_group()
