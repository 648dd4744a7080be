"""Collect tools/ncu_traffic.sh captures into profiles/ncu_traffic.json (DRAM bytes per launch of
the fused kernel, key "<config>_W1", and of the backward's pass-1 kernel, "<config>_W1_backward").

  python tools/ncu_traffic.py gpurun_out/ncu_r02 [profiles/ncu_traffic.json]
"""
import csv
import glob
import json
import os
import sys


def read(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    vals = {}
    name = None
    for r in rows:
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                     "usecond": 1, "msecond": 1e3}.get(unit, 1)
            vals[d["Metric Name"]] = v * scale
    if not vals:
        return None
    return {"kernel": name, "dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0) +
            vals.get("dram__bytes_write.sum", 0),
            "dram_read": vals.get("dram__bytes_read.sum"), "dram_write": vals.get("dram__bytes_write.sum"),
            "us_cold_serialised": vals.get("gpu__time_duration.sum"),
            "l2_hit_pct": vals.get("lts__t_sector_hit_rate.pct"),
            "warps_active_pct": vals.get("sm__warps_active.avg.pct_of_peak_sustained_active")}


def main():
    src = sys.argv[1]
    dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    for p in sorted(glob.glob(os.path.join(src, "*.csv"))):
        base = os.path.basename(p)[:-4]
        rec = read(p)
        if rec is None:
            continue
        cfg = base.replace("_backward", "")
        key = f"{cfg}_W1" + ("_backward" if base.endswith("_backward") else "")
        rec["source"] = f"{src}/{os.path.basename(p)} (ncu --metrics, -s 3 -c 1, --clock-control none)"
        out[key] = rec
    with open(dst, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
