"""Host<->device copy bandwidth of pinned buffers allocated from different CPU sets: no affinity,
the GPU-local CPUs NVML reports (nvmlDeviceGetCpuAffinity), and the other CPUs.  Each variant
runs in a fresh subprocess (first-touch NUMA placement follows the allocating thread)."""
import json, os, subprocess, sys

CHILD = r'''
import json, os, sys, time, torch
cpus = json.loads(sys.argv[1])
if cpus: os.sched_setaffinity(0, cpus)
dev = torch.device("cuda:0")
out = {"cpus": len(cpus) if cpus else "all"}
for nbytes in (1_376_618, 4_194_304):
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    for _ in range(5): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    a, b, c = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    a.record()
    for _ in range(50): d.copy_(h, non_blocking=True)
    b.record()
    for _ in range(50): h.copy_(d, non_blocking=True)
    c.record(); torch.cuda.synchronize()
    out[f"h2d_gbs_{nbytes}"] = round(nbytes * 50 / a.elapsed_time(b) / 1e6, 1)
    out[f"d2h_gbs_{nbytes}"] = round(nbytes * 50 / b.elapsed_time(c) / 1e6, 1)
print(json.dumps(out))
'''

def main():
    import pynvml
    pynvml.nvmlInit()
    hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
    n = os.cpu_count()
    words = pynvml.nvmlDeviceGetCpuAffinity(hdl, (n + 63) // 64)
    local = [i for i in range(n) if (words[i // 64] >> (i % 64)) & 1]
    remote = [i for i in range(n) if i not in local]
    print("cpu_count", n, "gpu-local cpus", len(local), local[:4], "...")
    os.system("lscpu | grep -i numa")
    for name, cpus in (("none", []), ("local", local), ("remote", remote)):
        if name == "remote" and not remote:
            continue
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(cpus)], capture_output=True,
                           text=True)
        print(name, r.stdout.strip() or r.stderr[-500:])

main()
