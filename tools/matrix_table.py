"""Markdown table of a bench matrix (tools/bench_matrix.sh output), as in BASELINE.md §6.2.

  python tools/matrix_table.py profiles/r01g_bench_matrix_W1.jsonl
"""
import json
import sys


def variant(c):
    if c.get("out_dtype", "f32") != "f32":
        return f"{c['out_dtype']} output"
    if c.get("table_dtype", "f32") != "f32":
        return c["table_dtype"]
    if c.get("pooling_mode") == "mean":
        return "mean"
    if c.get("per_sample_weights"):
        return "weights"
    if c.get("alpha", 1.05) == 0:
        return "α=0.0"
    return "f32 sum"


print("| config (per-rank work, W=1, one B200) | variant | fused µs/step | G lookups/s | roofline frac "
      "| frac (compulsory bytes) | DRAM frac (ncu) | α=0 µs (frac) "
      "| unfused pool + NCCL µs | fused speed-up | flushed-mode µs | backward step µs (plan + kernels) "
      "| unfused backward µs | backward kernel frac | oracle parity | fused == unfused |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    c = d["config"]
    u = d["unfused"]
    b = d.get("backward") or {}
    name = c["workload"].split(" ")[0]
    bw = "— (fp32 tables only, R#30)"
    ub = bf = "—"
    if "us_per_step" in b:
        bw = f"{b['us_per_step']:.1f} ({b['us_plan']:.1f} + {b['us_kernel']:.1f})"
        ub = f"{b['unfused_us_per_step']:.1f}"
        bf = f"{b['roofline']['frac']:.2f}"
    eq = u["fused_equals_unfused_bitwise"] and b.get("fused_equals_unfused_bitwise", True)
    r = d["roofline"]
    fc = f"{r['frac_compulsory']:.2f}" if r.get("frac_compulsory") is not None else "—"
    df = f"{r['dram_frac']:.2f}" if r.get("dram_frac") is not None else "—"
    a0 = d.get("alpha0")
    a0s = f"{a0['us_per_step']:.1f} ({a0['frac']:.2f})" if a0 else "—"
    par = d.get("parity") or {}
    ps = ("bitwise" if par.get("bitwise") else ("within tol" if par.get("within_tol") else "FAIL")) \
        if "rows" in par else "—"
    print(f"| {name} | {variant(c)} | {d['us_per_step']:.1f} | {d['value'] / 1e9:.2f} | "
          f"{r['frac']:.2f} | {fc} | {df} | {a0s} | {u['us_no_permute']:.1f} | "
          f"{u['us_no_permute'] / d['us_per_step']:.2f}× | {d['flushed']['us_per_step']:.1f} | {bw} | "
          f"{ub} | {bf} | {ps} | {'bitwise' if eq else 'DIFFERS'} |")
