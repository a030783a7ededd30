"""Summarise ncu captures for profiles/ (run here, on the CPU, after gpurun).

  python tools/ncu_summary.py full <report.ncu-rep> <out.json>
      per-kernel key counters of a `--set full` capture
  python tools/ncu_summary.py launches <launches.csv> <out.json>
      per-kernel totals of a `--metrics gpu__time_duration.sum` launch list
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, short in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                d[short] = _num(r[i])
                if units[i]:
                    d[short + "_unit"] = units[i]
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(d["kernel"][-40:], {k: d.get(k) for k in ("duration", "dram_read", "dram_pct", "l2_hit_pct",
                                                         "occupancy_pct", "dmma_pipe_pct")})


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, {"launches": 0, "ns": 0.0})
        a["launches"] += 1
        a["ns"] += v
    tot = sum(a["ns"] for a in agg.values())
    res = {"total_ms": tot / 1e6,
           "kernels": {k: {"launches": v["launches"], "ms": v["ns"] / 1e6, "share": v["ns"] / tot}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["ns"])}}
    json.dump(res, open(out, "w"), indent=1)
    print(f"total {tot / 1e6:.3f} ms")
    for k, v in list(res["kernels"].items())[:15]:
        print(f"  {v['ms']:8.3f} ms {v['launches']:5d}  {v['share'] * 100:5.1f}%  {k[-60:]}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
