"""Per-source-line stall summary of an ncu source-page CSV
(`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > f.csv`):
python tools/ncu_lines.py f.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[2]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


cur = None
agg = collections.defaultdict(lambda: collections.Counter())
txt = {}
for r in rows[3:]:
    if len(r) <= iI:
        continue
    if r[0]:
        try:
            cur = int(r[0])
            txt[cur] = r[1].strip()[:90]
        except ValueError:
            pass
    if r[2].startswith("0x") and cur is not None:
        a = agg[cur]
        a["samples"] += f(r[iS])
        a["instr"] += f(r[iI])
        for i, h in stalls:
            a[h] += f(r[i])
T = sum(a["samples"] for a in agg.values())
I = sum(a["instr"] for a in agg.values())
print(f"samples {T:.0f}  warp instructions {I:.0f}")
for ln, a in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
    st = sorted(((a[h], h[6:]) for _, h in stalls if a[h] > 0), reverse=True)[:3]
    sts = " ".join(f"{n}:{v / max(a['samples'], 1) * 100:.0f}%" for v, n in st)
    print(f"{a['samples'] / T * 100:5.1f}% {a['instr'] / I * 100:5.1f}%  L{ln}: {txt.get(ln, '')[:70]}  [{sts}]")
