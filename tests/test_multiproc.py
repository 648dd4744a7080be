"""Multi-process tests of the N>1 path: host logic over gloo on CPU (world size 2), and the real
cross-process cudaIpc path with two processes sharing one GPU."""
import socket

import pytest
import torch.multiprocessing as mp

from tests import _mp_worker


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run(fn, world, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=timeout) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


def test_gloo_world2_bootstrap_and_rank_local_oracle_check():
    for rank, ok_ag, ok_rows, ok_max in run(_mp_worker.cpu_allgather_worker, 2):
        assert ok_ag and ok_rows and ok_max, rank


@pytest.mark.gpu
def test_two_processes_one_gpu_cuda_ipc_path():
    """Each process maps the other's receive region with cudaIpcOpenMemHandle; fused forwards
    (3 epochs) match the oracle bitwise and the arrival counters equal epoch * n(src->dst); then
    two fused backward steps (gradient rows pushed across the process boundary) update the
    tables exactly as the oracle does."""
    for rank, ok, ok_flags in run(_mp_worker.gpu_ipc_worker, 2, timeout=300):
        assert ok and ok_flags, rank


@pytest.mark.gpu
def test_two_processes_one_gpu_ag_gemm_cuda_ipc():
    """f4 across processes: chunk PUTs into the other process's gather buffer, ready flags and
    credits through cudaIpc mappings; three forwards bitwise equal to the oracle."""
    for rank, ok, ok_flags in run(_mp_worker.gpu_ag_ipc_worker, 2, timeout=300):
        assert ok and ok_flags, rank
