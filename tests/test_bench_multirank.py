"""The N>1 bench path (torchrun, one process per rank) on a one-GPU box: all ranks share cuda:0
(EMBA2A_SHARED_GPU=1), real cross-process cudaIpc, device barrier, back-to-back and flushed
timing loops, max-over-ranks, the unfused baseline and its bitwise check."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4])
def test_bench_torchrun_shared_gpu(n):
    env = dict(os.environ, EMBA2A_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "4", "--warmup", "3",
           "--config", "tiny", "--batches", "2", "--cpu-seconds", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["value"] > 0
    assert line["unfused"]["fused_equals_unfused_bitwise"] is True
    assert line["gpu_launches"] == 4
    bwd = line["backward"]          # f3 across processes: fused exchange vs pack + all_to_all
    assert bwd["fused_equals_unfused_bitwise"] is True and bwd["us_per_step"] > 0
    par = line["parity"]            # every rank checked its own rows against the oracle
    assert par["within_tol"] is True and par["bitwise"] is True and par["rows"] >= 16
    cpu = line["cpu_baseline"]      # N single-threaded oracle processes, one per rank
    assert cpu["cores"] == n and len(cpu["per_rank"]) == n and cpu["value"] > 0
    assert cpu["host_cpu_count"] >= 1
    roof = line["roofline"]
    assert roof["compulsory_bytes_per_launch"] <= roof["algorithmic_bytes_per_launch"]
    assert 0 < roof["frac_compulsory"] <= roof["frac"]
    assert line["alpha0"]["us_per_step"] > 0
    ag = line["ag_gemm"]            # f4 leg at N ranks: fused AllGather + GEMM, parity on every rank
    assert "error" not in ag, ag
    assert ag["parity_all_ranks"] is True and ag["value"] > 0 and ag["roofline"]["bound"] == "tensor"


@pytest.mark.gpu
def test_ablations_command_torchrun_shared_gpu():
    """f1 as one driver-runnable command (tools/ablations_torchrun.py): every point is a torchrun
    bench run that prints a JSON line with its ablation key, parity-checked."""
    env = dict(os.environ, EMBA2A_SHARED_GPU="1")
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ablations_torchrun.py"), "--gpus", "2",
           "--config", "tiny", "--slices", "4,32", "--ctas", "1", "--steps", "3", "--warmup", "3",
           "--batches", "2", "--skew-us", "5", "--ag-config", "ag_tiny"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    recs = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(recs) == 2 + 1 + 6 + 2, r.stdout[-2000:]
    for rec in recs:
        assert "error" not in rec, rec
        if "AG" in rec["ablation"]:       # f4 points: TFLOP/s lines, oracle bound on every rank
            assert rec["ms_per_step"] > 0 and rec["parity"]["within_bound"] is True
        else:
            assert rec["us_per_step"] > 0 and rec["parity"]["within_tol"] is True
    kinds = [next(iter(rec["ablation"])) for rec in recs]
    assert kinds == ["E4", "E4", "E3"] + ["E5"] * 6 + ["AG"] * 2


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2])
def test_bench_ag_gemm_torchrun_shared_gpu(n):
    """bench.py --path ag_gemm under torchrun (f4): per-rank oracle parity, the NCCL-style
    baseline leg, e2e and the tensor roofline keys, max over ranks."""
    env = dict(os.environ, EMBA2A_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--path", "ag_gemm", "--ag-config", "ag_tiny",
           "--gpus", str(n), "--steps", "4", "--warmup", "3", "--cpu-seconds", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["value"] > 0 and line["unit"] == "TFLOP/s"
    assert line["parity_all_ranks"] is True and line["parity"]["gathered_bitwise"] is True
    assert line["roofline"]["bound"] == "tensor" and line["roofline"]["frac"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["cpu_baseline"]["value"] > 0
    assert line["unfused"]["ms_per_step"] > 0
