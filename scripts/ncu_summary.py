"""Summarise an `ncu --set full` capture of the step-1 evaluation kernels (A, B, C) into the
per-launch traffic record bench.py reads (profiles/traffic_<config>.json).

    python scripts/ncu_summary.py gpurun_out/p16_full_c4.ncu-rep c4 "<what>" > profiles/traffic_c4.json
"""
import csv
import json
import subprocess
import sys

ALG = {"c4": 7288202781.131464}
SHORT = {"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
         "lts__t_sector_hit_rate.pct": "l2_hit_pct", "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
         "launch__registers_per_thread": "regs"}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    rep, cfg, what = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    kernels, total, ms = {}, 0.0, 0.0
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0]
        t = float(r[col["gpu__time_duration.sum"]])
        tu = units[col["gpu__time_duration.sum"]]
        k = {"ms": t * {"us": 1e-3, "ms": 1.0, "ns": 1e-6}[tu]}
        for m, s in SHORT.items():
            v = float(r[col[m]])
            k[s] = v * UNIT.get(units[col[m]], 1.0) if "bytes" in m else v
        k["dram_GBps"] = (k["dram_read_bytes"] + k["dram_write_bytes"]) / k["ms"] / 1e6
        kernels[name] = k
        total += k["dram_read_bytes"] + k["dram_write_bytes"]
        ms += k["ms"]
    rec = {"config": cfg, "round": 2, "what": what, "kernels": kernels,
           "dram_bytes_per_launch": total, "algorithmic_bytes": ALG.get(cfg),
           "traffic_over_algorithmic": total / ALG[cfg] if cfg in ALG else None,
           "eval_ms_cold": ms}
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
